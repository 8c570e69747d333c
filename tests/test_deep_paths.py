"""Deep radix paths: a chain whose every request extends the previous one,
so request i's path has i levels.  Past kMaxPath (512) levels the engine keeps path
levels in its global overflow arrays, K1 grows its hint stride between
batches, and hit stamps are undone through the path log — all of it must
still match the reference bit for bit (decisions, costs, final mirror).

C5-shaped traces reach such depths: partial LRU evictions split hot chains
again and again (depth ~1.4k after 120k requests)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2407_00023_b200 import abi
from paper_2407_00023_b200.scheduler import DriverConfig, SchedulerConfig
from paper_2407_00023_b200.workload import Config, Trace

from parity import assert_same_state, diff_decisions, replay


def chain_trace(n: int, seg: int = 10, every: int = 5, seed: int = 7) -> Trace:
    """Request i = the first seg*(i+1) tokens of one chain; every `every`-th
    request is instead an unrelated short prompt (explore traffic)."""
    rng = np.random.default_rng(seed)
    chain = np.arange(1_000_000, 1_000_000 + seg * (n + 1), dtype=np.int32)
    prompts, k = [], 0
    for i in range(n):
        if i % every == every - 1:
            prompts.append(rng.integers(5_000_000, 6_000_000, size=int(rng.integers(50, 400)), dtype=np.int32))
        else:
            k += 1
            prompts.append(chain[: seg * k])
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    toks = np.concatenate(prompts).astype(np.int32)
    arr = np.cumsum(rng.exponential(0.5, size=n))
    outl = rng.integers(20, 40, size=n).astype(np.int64)
    return Trace(toks, off, np.arange(1, n + 1, dtype=np.int64), arr, outl)


def _cfg(n, cap, hw, batch, G=4, H=200.0):
    c = Config("deep_chain", "custom", n, G, SchedulerConfig(kv_capacity_tokens=cap, history_window_ms=H),
               DriverConfig(eviction=abi.E2_EVICT_MIRROR_LRU, trunk_len=0, high_water=hw, finish_lag=300,
                            batch=batch))
    c.policy = None
    return c


def _check(lib, ref_lib, n, cap, hw, batch):
    cfg = _cfg(n, cap, hw, batch)
    tr = chain_trace(n)
    sa, a = replay(ref_lib, cfg, tr)
    sb, b = replay(lib, cfg, tr)
    assert getattr(a, "error", None) is None, a.error
    d = diff_decisions(a, b)
    assert d is None, f"first mismatch at request {d[0]} field {d[1]}"
    assert a.n_done == tr.n
    assert_same_state(sa, sb, float(tr.arrivals[-1]))


def test_deep_chain_hostsim(hostsim_lib, ref_lib):
    # 1400 requests: the chain path reaches ~1120 levels (> kMaxPath = 512);
    # the tight capacity makes the eviction term and hit catch-up run on it
    _check(hostsim_lib, ref_lib, 1400, 20000, 16000, 256)


@pytest.mark.gpu
@pytest.mark.parametrize("cap,hw", [(200000, 150000), (20000, 16000)])
def test_deep_chain_b200(b200_lib, ref_lib, cap, hw):
    _check(b200_lib, ref_lib, 1400, cap, hw, 256)
