"""Pin the plain-C restatement (oracle/e2_oracle.c): it must reproduce the
golden vectors recorded from the unmodified reference, the reference's own
known-answer behaviour, and the live reference on randomized op streams."""
from __future__ import annotations

import pytest

import test_fuzz
import test_golden
from parity import assert_same_state, diff_decisions, replay
from test_parity import CASES


@pytest.mark.parametrize("name", sorted(test_golden.CASES))
def test_oracle_golden(oracle_lib, gen_lib, name):
    test_golden.check(oracle_lib, gen_lib, name)


@pytest.mark.parametrize("case", ["c1", "c1_batch7", "docqa_mterm", "programming_infeasible", "embodied_chains",
                                  "videoqa_fifo", "round_robin", "short_window"])
def test_oracle_replay_vs_reference(oracle_lib, true_ref_lib, gen_lib, case):
    cfg = CASES[case]
    trace = cfg.trace(lib=gen_lib)
    sa, a = replay(true_ref_lib, cfg, trace)
    sb, b = replay(oracle_lib, cfg, trace)
    d = diff_decisions(a, b)
    assert d is None, f"first mismatch at request {d[0]} field {d[1]}"
    assert_same_state(sa, sb, float(trace.arrivals[-1]))


def test_oracle_fuzz_vs_reference(oracle_lib, true_ref_lib):
    test_fuzz._fuzz(oracle_lib, true_ref_lib, 150, 20260815)
