"""Golden vectors recorded from the unmodified reference (make_golden.py):
the engine must reproduce them where the reference itself is unavailable."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2407_00023_b200.scheduler import GlobalScheduler, ReplayResult

from parity import diff_decisions

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
import sys

sys.path.insert(0, HERE)
from make_golden import CASES  # noqa: E402


def check(lib, gen_lib, name):
    g = np.load(os.path.join(HERE, f"{name}.npz"))
    cfg, n = CASES[name]
    trace = cfg.trace(lib=gen_lib, n_requests=n)
    assert trace.n == int(g["n_requests"])
    assert int(trace.tokens.astype(np.int64).sum()) == int(g["token_checksum"])
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
    r = s.replay(trace, cfg.driver, want_costs=True, want_ratios=True)
    want = ReplayResult(g["decisions"], g["costs"], g["ratios"], trace.n)
    d = diff_decisions(want, r)
    assert d is None, f"first mismatch at request {d[0]} field {d[1]}"
    st = s.stats()
    assert [st.exploit, st.explore, st.decode_pressure, st.round_robin, st.redirected, st.rebalance_installs,
            st.autoscale_events, st.tree_reads] == g["stats"].tolist()
    nodes, toks, la, hits = s.export_arrays(float(trace.arrivals[-1]))
    got = np.frombuffer(nodes, dtype=np.uint64).reshape(len(nodes), -1)
    cols = [0, 1, 3, 4, 5]
    assert np.array_equal(got[:, cols], g["nodes"][:, cols])
    assert np.array_equal(toks, g["edge_tokens"])
    assert la.tobytes() == g["last_access"].tobytes()
    assert np.array_equal(hits, g["hits"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_hostsim(hostsim_lib, gen_lib, name):
    check(hostsim_lib, gen_lib, name)


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_checker(ref_lib, gen_lib, name):
    """The checker library itself (reference shim, or the C restatement where
    the shim is absent) reproduces the golden vectors."""
    check(ref_lib, gen_lib, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_b200(b200_lib, gen_lib, name):
    check(b200_lib, gen_lib, name)
