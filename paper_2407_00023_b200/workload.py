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


def concat(traces) -> Trace:
    """Concatenate traces (chunks of one stream) into one."""
    lens = [t.offsets[-1] - t.offsets[0] for t in traces]
    offs = [traces[0].offsets[:1] * 0]
    base = 0
    for t, ln in zip(traces, lens):
        offs.append(t.offsets[1:] - t.offsets[0] + base)
        base += ln
    return Trace(np.concatenate([t.tokens[t.offsets[0]:t.offsets[-1]] for t in traces]), np.concatenate(offs),
                 np.concatenate([t.ids for t in traces]), np.concatenate([t.arrivals for t in traces]),
                 np.concatenate([t.output_lens for t in traces]))


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


FRESH_BASE = 500_000_000  # the generator's fresh-id region (workload.cpp:25-28)
FRESH_SPAN = 2_147_483_647 - FRESH_BASE


class MixConfig(Config):
    """Config 5: toolbench + doc-QA + programming + tree-of-thought + embodied
    chains on 64 instances with a small cache, so the eviction term is active
    on most decisions — generated as a STREAM of independent chunks.

    The reference's generator hands out fresh token ids from one counter
    (workload.cpp:44) and runs out of int32 ids long before 10M requests.
    Here chunk c (CHUNK requests) is generated by the same archetype
    generators with seeds derived from (seed, c, component) and then:
      * shared-prefix ids (system prompts, tool branches, documents, problem
        trunks: below 5e8) are kept, shifted per component — they recur
        across chunks like a real corpus;
      * fresh ids (unique suffixes, thoughts, observations: >= 5e8) are
        REUSED: remapped by a 64-bit hash of (id, chunk, component) into
        [5e8, 2^31-1), so id space never runs out;
      * the components are interleaved by arrival time inside the chunk and
        the chunk's arrivals are placed in its own time slot, so arrival
        times increase across chunks; request ids are the stream index + 1.
    Chunks are independent, so chunk c can be generated directly (random
    access) and the stream never has to be held in memory: the replay takes
    it chunk by chunk (e2_replay_set_continue)."""

    COMPONENTS = (("toolbench", 0.4, {}), ("doc_qa", 0.1, {}), ("programming", 0.2, {}),
                  ("tree_of_thought", 0.2, {}), ("embodied_agent", 0.1, {}))
    CHUNK = 65536

    def _counts(self, q: int):
        fr = np.array([f for _, f, _ in self.COMPONENTS])
        base = np.floor(q * fr).astype(np.int64)
        rem = q * fr - base
        for i in np.argsort(-rem, kind="stable")[: q - int(base.sum())]:
            base[i] += 1
        return base

    def chunk(self, c: int, lib=None, q: int = None) -> Trace:
        """Chunk c of the stream: requests [c*CHUNK, c*CHUNK + q)."""
        Q = self.CHUNK
        q = q if q is not None else min(Q, self.n_requests - c * Q)
        if q <= 0:
            raise ValueError("chunk index past the end of the stream")
        parts = []
        for k, ((arch, frac, over), cnt) in enumerate(zip(self.COMPONENTS, self._counts(q))):
            if cnt == 0:
                continue
            s = default_spec(arch, lib)
            s.request_count = int(cnt)
            for a, v in over.items():
                setattr(s, a, v)
            t = generate(s, self.seed + 7919 * c + k, self.rps * frac, self.arrival_seed + 7919 * c + k, lib)
            tok = t.tokens.astype(np.int64)
            fresh = tok >= FRESH_BASE
            salt = np.uint64((c * 64 + k + 1) * 0x9E3779B97F4A7C15 & 0xFFFFFFFFFFFFFFFF)
            h = _splitmix(tok[fresh].astype(np.uint64) ^ salt)
            tok[fresh] = FRESH_BASE + (h % np.uint64(FRESH_SPAN)).astype(np.int64)
            tok[~fresh] += k * 20_000_000
            parts.append((t.arrivals, np.diff(t.offsets), tok.astype(np.int32), t.output_lens))
        arr = np.concatenate([p[0] for p in parts])
        lens = np.concatenate([p[1] for p in parts])
        toks = np.concatenate([p[2] for p in parts])
        outl = np.concatenate([p[3] for p in parts])
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
        order = np.argsort(arr, kind="stable")
        lens_o = lens[order]
        off = np.zeros(q + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens_o)
        idx = np.repeat(starts[order] - off[:-1], lens_o) + np.arange(off[-1], dtype=np.int64)
        span = 1000.0 * Q / self.rps  # the chunk's time slot (ms)
        a = arr[order]
        rel = a / (a[-1] + 1000.0 / self.rps)  # in [0, 1), increasing
        arrivals = c * span + span * rel
        ids = np.arange(c * Q + 1, c * Q + q + 1, dtype=np.int64)
        return Trace(toks[idx], off, ids, arrivals, outl[order].copy())

    def chunks(self, n_requests=None, lib=None):
        """The stream's chunks, in order, up to n_requests (default: all)."""
        n = n_requests if n_requests is not None else self.n_requests
        Q = self.CHUNK
        for c in range((n + Q - 1) // Q):
            yield self.chunk(c, lib, q=min(Q, n - c * Q))

    def trace(self, lib=None, n_requests: Optional[int] = None) -> Trace:
        n = n_requests if n_requests is not None else self.n_requests
        if n > 8 * self.CHUNK:
            raise ValueError("config 5 is a stream: use chunks() and a continued replay beyond 8 chunks")
        return concat(list(self.chunks(n, lib)))


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
    # Device batches of 2048: partial evictions split ~1 node per request, so
    # K1's path hints age fast; smaller batches refresh them (C5 +30 % vs 16384,
    # C2/C4 insensitive: scripts/ab_batch.py).
    "c5": MixConfig(
        "c5_mixed_10M_64inst", "mixed", 10_000_000, 64, _cs2_sched(cap=30000),
        DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=28500, finish_lag=2000, batch=2048),
    ),
}


# --------------------------------------------------------------------------
# corpus / trace files and the corpus study (workload.cpp:329-601), C ABI
# --------------------------------------------------------------------------
def _lib_err(lib, rc):
    if rc != abi.E2_OK:
        msg = lib.e2_last_error(None).decode()
        raise ValueError(msg) if rc == abi.E2_ERR_ARG else RuntimeError(msg)


def write_corpus(path: str, trace: Trace, with_arrivals: bool = True, lib=None) -> None:
    lib = lib or abi.product_lib()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    toks = np.ascontiguousarray(trace.tokens, dtype=np.int32)
    rc = lib.e2_corpus_write(path.encode(), p(toks), p(trace.offsets), p(trace.ids),
                             p(trace.arrivals) if with_arrivals else None, None, p(trace.output_lens), trace.n)
    _lib_err(lib, rc)


def read_corpus(path: str, lib=None):
    """(Trace, has_arrival) of a corpus file; arrivals are 0 where absent."""
    lib = lib or abi.product_lib()
    n, nt = ctypes.c_int64(), ctypes.c_int64()
    _lib_err(lib, lib.e2_corpus_read(path.encode(), ctypes.byref(n), ctypes.byref(nt), None, None, None, None, None,
                                     None))
    toks = np.zeros(nt.value + 64, dtype=np.int32)
    off = np.zeros(n.value + 1, dtype=np.int64)
    ids = np.zeros(n.value, dtype=np.int64)
    arr = np.zeros(n.value, dtype=np.float64)
    has = np.zeros(n.value, dtype=np.int32)
    outl = np.zeros(n.value, dtype=np.int64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _lib_err(lib, lib.e2_corpus_read(path.encode(), ctypes.byref(n), ctypes.byref(nt), p(toks), p(off), p(ids), p(arr),
                                     p(has), p(outl)))
    return Trace(toks[: nt.value], off, ids, arr, outl), has


def read_trace(path: str, lib=None):
    """(arrival_s, prompt_len, output_len) of a request-trace CSV, by arrival."""
    lib = lib or abi.product_lib()
    n = ctypes.c_int64()
    _lib_err(lib, lib.e2_trace_read(path.encode(), ctypes.byref(n), None, None, None))
    a = np.zeros(n.value, dtype=np.float64)
    pl = np.zeros(n.value, dtype=np.int64)
    ol = np.zeros(n.value, dtype=np.int64)
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    _lib_err(lib, lib.e2_trace_read(path.encode(), ctypes.byref(n), p(a), p(pl), p(ol)))
    return a, pl, ol


def synthesize_from_trace(arrival_s, prompt_len, output_len, content: abi.WorkloadSpecC, seed: int, lib=None) -> Trace:
    lib = lib or abi.product_lib()
    a = np.ascontiguousarray(arrival_s, dtype=np.float64)
    pl = np.ascontiguousarray(prompt_len, dtype=np.int64)
    ol = np.ascontiguousarray(output_len, dtype=np.int64)
    n = len(a)
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    nt = ctypes.c_int64()
    args = [ctypes.byref(content), seed, p(a), p(pl), p(ol), n, ctypes.byref(nt)]
    _lib_err(lib, lib.e2_synthesize_from_trace(*args, None, None, None, None, None))
    toks = np.zeros(nt.value + 64, dtype=np.int32)
    off = np.zeros(n + 1, dtype=np.int64)
    ids = np.zeros(n, dtype=np.int64)
    arr = np.zeros(n, dtype=np.float64)
    outl = np.zeros(n, dtype=np.int64)
    _lib_err(lib, lib.e2_synthesize_from_trace(*args, p(toks), p(off), p(ids), p(arr), p(outl)))
    return Trace(toks[: nt.value], off, ids, arr, outl)


def analyze(trace: Trace, lib=None) -> dict:
    """The corpus study (StudyReport, workload.hpp:126-141) as a dict."""
    lib = lib or abi.product_lib()
    st = abi.StudyC()
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    toks = np.ascontiguousarray(trace.tokens, dtype=np.int32)
    _lib_err(lib, lib.e2_analyze(p(toks), p(trace.offsets), p(trace.output_lens), trace.n, ctypes.byref(st)))

    def conv(x):
        if isinstance(x, abi.DistC):
            return {f: getattr(x, f) for f, _ in abi.DistC._fields_}
        return x

    return {f: conv(getattr(st, f)) for f, _ in abi.StudyC._fields_}
