"""Synthetic traces (input only) and the five BASELINE.json configurations.

Generation runs in host C++ (``e2_generate`` in the product library,
``csrc/workload_gen.cpp``); for the reference archetypes it produces the same
tokens, ids, arrivals and output lengths as ``kvsched::generate`` +
``assign_poisson_arrivals`` (workload.cpp:235-327, 486-497) — pinned by
``tests/test_workload.py`` against the reference shim.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np

from . import abi
from .scheduler import DriverConfig, GlobalPolicy, SchedulerConfig

ARCH = {
    "custom": 0,
    "toolbench": 1,
    "embodied_agent": 2,
    "programming": 3,
    "video_qa": 4,
    "doc_qa": 5,
    "tree_of_thought": 6,
}


@dataclasses.dataclass
class Trace:
    tokens: np.ndarray  # int32 CSR arena
    offsets: np.ndarray  # int64 [n+1]
    ids: np.ndarray  # int64
    arrivals: np.ndarray  # float64 ms
    output_lens: np.ndarray  # int64

    @property
    def n(self) -> int:
        return len(self.ids)

    def prompt(self, i: int) -> np.ndarray:
        return self.tokens[self.offsets[i] : self.offsets[i + 1]]

    def head(self, n: int) -> "Trace":
        end = int(self.offsets[n])
        return Trace(
            self.tokens[:end].copy(), self.offsets[: n + 1].copy(), self.ids[:n].copy(), self.arrivals[:n].copy(),
            self.output_lens[:n].copy(),
        )

    @property
    def nbytes(self) -> int:
        return int(self.tokens.nbytes + self.offsets.nbytes + self.ids.nbytes + self.arrivals.nbytes + self.output_lens.nbytes)


def default_spec(archetype: str, lib: Optional[ctypes.CDLL] = None) -> abi.WorkloadSpecC:
    lib = lib or abi.product_lib()
    s = abi.WorkloadSpecC()
    lib.e2_workload_default(ARCH[archetype], ctypes.byref(s))
    return s


def generate(spec: abi.WorkloadSpecC, seed: int, rps: float, arrival_seed: int, lib: Optional[ctypes.CDLL] = None) -> Trace:
    lib = lib or abi.product_lib()
    n, nt = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.e2_generate(ctypes.byref(spec), seed, rps, arrival_seed, ctypes.byref(n), ctypes.byref(nt), None, None, None, None, None)
    if rc != abi.E2_OK:
        raise ValueError(lib.e2_last_error(None).decode())
    tokens = np.zeros(nt.value + 64, dtype=np.int32)  # slack for vector loads
    offsets = np.zeros(n.value + 1, dtype=np.int64)
    ids = np.zeros(n.value, dtype=np.int64)
    arr = np.zeros(n.value, dtype=np.float64)
    outl = np.zeros(n.value, dtype=np.int64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    rc = lib.e2_generate(ctypes.byref(spec), seed, rps, arrival_seed, ctypes.byref(n), ctypes.byref(nt), p(tokens), p(offsets), p(ids), p(arr), p(outl))
    if rc != abi.E2_OK:
        raise ValueError(lib.e2_last_error(None).decode())
    return Trace(tokens[: nt.value], offsets, ids, arr, outl)


@dataclasses.dataclass
class Config:
    name: str
    archetype: str
    n_requests: int
    n_gpus: int
    sched: SchedulerConfig
    driver: DriverConfig
    seed: int = 13
    rps: float = 2000.0
    arrival_seed: int = 14
    spec_overrides: dict = dataclasses.field(default_factory=dict)
    policy: Optional[GlobalPolicy] = None

    def spec(self, lib=None) -> abi.WorkloadSpecC:
        s = default_spec(self.archetype, lib)
        s.request_count = self.n_requests
        for k, v in self.spec_overrides.items():
            setattr(s, k, v)
        return s

    def trace(self, lib=None, n_requests: Optional[int] = None) -> Trace:
        s = self.spec(lib)
        if n_requests is not None:
            s.request_count = n_requests
        return generate(s, self.seed, self.rps, self.arrival_seed, lib)


def mix(traces, token_strides) -> Trace:
    """Interleave several traces by arrival time (config 5's mixed workload).

    Each component's token ids are shifted by its stride so unrelated
    archetypes do not alias; ids stay int32 (the reference's TokenId)."""
    parts = []
    for t, stride in zip(traces, token_strides):
        lens = np.diff(t.offsets)
        toks = t.tokens.astype(np.int64) + stride
        if toks.size and (toks.max() > np.iinfo(np.int32).max or toks.min() < 0):
            raise ValueError("token id space exhausted by the mixture")
        parts.append((t.arrivals, lens, toks.astype(np.int32), t.output_lens))
    arr = np.concatenate([p[0] for p in parts])
    order = np.argsort(arr, kind="stable")
    lens = np.concatenate([p[1] for p in parts])
    starts = np.concatenate([np.concatenate([[0], np.cumsum(p[1])[:-1]]) + sum(len(q[2]) for q in parts[:i])
                             for i, p in enumerate(parts)])
    toks_all = np.concatenate([p[2] for p in parts])
    outl = np.concatenate([p[3] for p in parts])
    n = len(arr)
    new_off = np.zeros(n + 1, dtype=np.int64)
    new_off[1:] = np.cumsum(lens[order])
    tokens = np.empty(int(new_off[-1]), dtype=np.int32)
    for k, i in enumerate(order):
        tokens[new_off[k]:new_off[k + 1]] = toks_all[starts[i]:starts[i] + lens[i]]
    return Trace(tokens, new_off, np.arange(1, n + 1, dtype=np.int64), arr[order].copy(), outl[order].copy())


class MixConfig(Config):
    """Config 5: toolbench + doc-QA + programming + tree-of-thought + embodied
    chains, interleaved by arrival time, on 64 instances with a small cache
    so the eviction term is active on most decisions."""

    COMPONENTS = (("toolbench", 0.4, {}), ("doc_qa", 0.1, {}), ("programming", 0.2, {}),
                  ("tree_of_thought", 0.2, {}), ("embodied_agent", 0.1, {}))

    def trace(self, lib=None, n_requests: Optional[int] = None) -> Trace:
        n = n_requests if n_requests is not None else self.n_requests
        traces, strides = [], []
        for k, (arch, frac, over) in enumerate(self.COMPONENTS):
            s = default_spec(arch, lib)
            s.request_count = max(1, int(round(n * frac)))
            for a, v in over.items():
                setattr(s, a, v)
            traces.append(generate(s, self.seed + k, self.rps * frac, self.arrival_seed + k, lib))
            strides.append(k * 20_000_000)
        t = mix(traces, strides)
        return t.head(min(n, t.n)) if t.n > n else t


def _cs2_sched(cap=200000):
    # criterion-7 settings: cap 200000, H = 10 s (acceptance_main.cpp:380-383)
    return SchedulerConfig(kv_capacity_tokens=cap, history_window_ms=10000.0)


CONFIGS = {
    # C1: criterion-7 loop exactly (FIFO-tail eviction at 150000 = 0.75 cap).
    "c1": Config(
        "c1_toolbench_1k_4inst", "toolbench", 1000, 4, _cs2_sched(),
        DriverConfig(eviction=abi.E2_EVICT_FIFO_TAIL, trunk_len=1860, high_water=150000, finish_lag=2000),
    ),
    # C2: toolbench Zipf(1.1)/16 branches, 100k requests, 8 instances, mirror-LRU driver.
    "c2": Config(
        "c2_toolbench_100k_8inst", "toolbench", 100000, 8, _cs2_sched(),
        DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=1860, high_water=150000, finish_lag=2000),
    ),
    # C3: LooGLE-shape doc QA: docs U[20000,40000], questions U[200,300], 1+Poisson(5) per doc,
    # 16 instances; cap 100k / high-water 0.9 so the eviction term M is active.
    "c3": Config(
        "c3_docqa_20k-40k_16inst", "doc_qa", 10000, 16, _cs2_sched(cap=100000),
        DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=90000, finish_lag=2000),
        spec_overrides=dict(branch_len=20000, branch_len_max=40000),
    ),
    # C4: tree-of-thought / programming-style deep branching: 64-request problems, fanout 3,
    # depth <= 8 thought segments of 40-120 tokens; 1M requests (parity on prefixes).
    "c4": Config(
        "c4_tree_of_thought_1M_16inst", "tree_of_thought", 1_000_000, 16, _cs2_sched(cap=20000),
        DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=19000, finish_lag=2000),
    ),
    # C5: mixed multi-workload, 10M requests, 64 instances, heavy eviction (cap 30k, high-water 0.95).
    "c5": MixConfig(
        "c5_mixed_10M_64inst", "mixed", 10_000_000, 64, _cs2_sched(cap=30000),
        DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=28500, finish_lag=2000),
    ),
}
