"""A replay that fails part-way must stop exactly where the reference stops.

The reference's CS2-style loop (acceptance_main.cpp:367-416) calls
schedule_request per request; a prompt longer than the KV capacity makes
decide throw NoAdmissibleGpu (global_scheduler.cpp:77-80), and every earlier
request has already been scheduled, prefilled, evicted for and finished.
The product's replay (the pipelined kernel on the GPU) must report the same
error at the same request index and the same decisions before it."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import DriverConfig, NoAdmissibleGpu, SchedulerConfig
from paper_2407_00023_b200.workload import Trace

from parity import diff_decisions, replay


def _with_long_prompt(tr: Trace, k: int, length: int) -> Trace:
    """Replace request k's prompt by `length` fresh tokens."""
    lens = np.diff(tr.offsets)
    prompts = [tr.prompt(i) for i in range(tr.n)]
    prompts[k] = np.arange(900_000_000, 900_000_000 + length, dtype=np.int32)
    lens[k] = length
    off = np.zeros(tr.n + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    return Trace(np.concatenate(prompts).astype(np.int32), off, tr.ids.copy(), tr.arrivals.copy(), tr.output_lens.copy())


def _case(gen_lib, n, k, batch):
    cfg = dataclasses.replace(
        W.CONFIGS["c2"],
        n_requests=n,
        sched=SchedulerConfig(kv_capacity_tokens=20000, history_window_ms=10000.0),
        driver=DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=15000, finish_lag=200,
                            batch=batch),
    )
    tr = _with_long_prompt(cfg.trace(lib=gen_lib), k, 25000)
    return cfg, tr


def _check(lib, ref_lib, cfg, tr, k):
    _, a = replay(ref_lib, cfg, tr)
    _, b = replay(lib, cfg, tr)
    assert isinstance(getattr(a, "error", None), NoAdmissibleGpu), getattr(a, "error", None)
    assert isinstance(getattr(b, "error", None), NoAdmissibleGpu), getattr(b, "error", None)
    assert a.n_done == b.n_done == k
    assert diff_decisions(a, b) is None


@pytest.mark.parametrize("n,k,batch", [(600, 437, 0), (600, 0, 0), (600, 300, 64)])
def test_replay_error_hostsim(hostsim_lib, ref_lib, gen_lib, n, k, batch):
    cfg, tr = _case(gen_lib, n, k, batch)
    _check(hostsim_lib, ref_lib, cfg, tr, k)


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,batch", [(3000, 2457, 0), (3000, 0, 0), (3000, 1, 0), (3000, 1500, 256)])
def test_replay_error_b200(b200_lib, ref_lib, gen_lib, n, k, batch):
    cfg, tr = _case(gen_lib, n, k, batch)
    _check(b200_lib, ref_lib, cfg, tr, k)


@pytest.mark.parametrize("n", [1, 2, 3, 33])
def test_tiny_replays_hostsim(hostsim_lib, ref_lib, gen_lib, n):
    cfg = dataclasses.replace(W.CONFIGS["c1"], n_requests=n)
    tr = cfg.trace(lib=gen_lib)
    _, a = replay(ref_lib, cfg, tr)
    _, b = replay(hostsim_lib, cfg, tr)
    assert a.n_done == b.n_done == n
    assert diff_decisions(a, b) is None


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 33, 2049])
def test_tiny_replays_b200(b200_lib, ref_lib, gen_lib, n):
    """Pipeline start-up and drain with fewer requests than pipeline stages
    (and one request past the first ramp batch)."""
    cfg = dataclasses.replace(W.CONFIGS["c1"], n_requests=n)
    tr = cfg.trace(lib=gen_lib)
    _, a = replay(ref_lib, cfg, tr)
    _, b = replay(b200_lib, cfg, tr)
    assert a.n_done == b.n_done == n
    assert diff_decisions(a, b) is None
