"""Randomized placement fidelity through the per-call API.

Mirrors the reference's own criterion-1 harness (tests/oracle/
reference_scheduler.cpp:271-436, acceptance_main.cpp:63-78): random cluster
scenarios (2-4 instances, random H / capacity / time model / policy), random
interleavings of schedule_request, note_admitted + note_prefill_cached,
note_finished and legal note_eviction, then standalone load_cost probes
(including missed totals past capacity, which exercise the infeasible flag).
Every decision field and cost term is compared bit-for-bit against the
unmodified reference driven with the same op stream, and the final mirrors
are compared node by node.
"""
from __future__ import annotations

import random

import pytest

from paper_2407_00023_b200.scheduler import (
    EvictedRange,
    GlobalPolicy,
    GlobalScheduler,
    Request,
    SchedulerConfig,
    TimeModel,
)

from parity import export_diff, snapshot_diff


def _same_decision(a, b):
    if (a.branch, a.gpu, a.redirected, a.pre_redirect_gpu, a.cached_len, a.missed_len, a.missed_on_chosen,
            a.matched_len) != (b.branch, b.gpu, b.redirected, b.pre_redirect_gpu, b.cached_len, b.missed_len,
                               b.missed_on_chosen, b.matched_len):
        return False
    if len(a.costs) != len(b.costs):
        return False
    for x, y in zip(a.costs, b.costs):
        if x.gpu != y.gpu or x.cost != y.cost:  # dataclass == compares the doubles exactly
            return False
    return a.decode_ratios == b.decode_ratios


def run_case(lib, ref_lib, seed, stats):
    rng = random.Random(seed)
    snap = hasattr(lib, "e2_export_hit_stamps")  # the plain-C oracle has no snapshot()
    n = 2 + rng.randrange(3)
    cfg = SchedulerConfig(
        history_window_ms=rng.choice([600.0, 3000.0, 20000.0]),
        imbal_ratio=rng.choice([0.5, 0.9]),
        kv_capacity_tokens=rng.choice([120, 300, 900, 4000]),
        default_output_len=rng.choice([8, 32]),
    )
    model = TimeModel(rng.choice([0.0, 4.0, 5.0]), rng.choice([0.25, 0.5, 1.0]), rng.choice([1.0, 8.0, 15.0]), 8.0)
    pol = GlobalPolicy(rebalance=rng.random() < 0.5, autoscale=rng.random() < 0.5, pd_balance=rng.random() < 0.5)
    A = GlobalScheduler(n, cfg, model, pol, lib=ref_lib)
    B = GlobalScheduler(n, cfg, model, pol, lib=lib)
    stems = []
    for s in range(2 + rng.randrange(4)):
        stems.append([(s + 1) * 1000 + j for j in range(4 + rng.randrange(37))])
    live, cached_paths, issued = [], [], []
    t, next_id, unique = 0.0, 1, 9000000
    for op in range(12 + rng.randrange(24)):
        t += 1.0 + rng.randrange(1000) / 10.0
        roll = rng.randrange(100)
        if roll < 55 or not live:
            if issued and rng.randrange(100) < 25:
                prompt = list(rng.choice(issued))
            else:
                stem = rng.choice(stems)
                take = len(stem) if rng.randrange(100) < 70 else 1 + rng.randrange(len(stem))
                prompt = stem[:take]
                if rng.random() < 0.5:
                    extra = 1 + rng.randrange(15)
                    prompt += list(range(unique, unique + extra))
                    unique += extra
            if snap and rng.randrange(4) == 0:  # the reference harness snapshots before each decision (:333)
                stats["snapshots"] += 1
                msg = snapshot_diff(A, B, t)
                assert msg is None, (seed, op, msg)
            req = Request(next_id, prompt, t, 1 + rng.randrange(40))
            errs = []
            outs = []
            for S in (A, B):
                try:
                    outs.append(S.schedule_request(req, t))
                    errs.append(None)
                except Exception as e:
                    outs.append(None)
                    errs.append(type(e).__name__)
            assert errs[0] == errs[1], (seed, op, errs)
            if errs[0] is None:
                assert _same_decision(outs[0], outs[1]), (seed, op, outs[0], outs[1])
                d = outs[0]
                stats["decisions"] += 1
                stats["exploit"] += d.branch == 0
                stats["pressure"] += d.branch == 2
                stats["redirected"] += d.redirected
                live.append((next_id, prompt, d.gpu))
                issued.append(prompt)
            next_id += 1
        elif roll < 70:
            rid, prompt, g = live[rng.randrange(len(live))]
            for S in (A, B):
                S.note_admitted(rid, t)
                S.note_prefill_cached(prompt, g, t)
            cached_paths.append((list(prompt), g))
        elif roll < 85:
            i = rng.randrange(len(live))
            out = 1 + rng.randrange(40)
            for S in (A, B):
                S.note_finished(live[i][0], t, out)
            live.pop(i)
        elif cached_paths:
            # legal eviction range: below the deepest branch point with any
            # other cached path on the same instance (reference_scheduler.cpp:375-404)
            i = rng.randrange(len(cached_paths))
            seq, g = cached_paths[i]
            shared = 0
            for j, (other, og) in enumerate(cached_paths):
                if j == i or og != g or other == seq:
                    continue
                lcp = 0
                while lcp < len(seq) and lcp < len(other) and seq[lcp] == other[lcp]:
                    lcp += 1
                shared = max(shared, lcp)
            if shared < len(seq):
                tail = 1 + rng.randrange(len(seq) - shared)
                for S in (A, B):
                    S.note_eviction(EvictedRange(seq, tail), g, t)
                remain = len(seq) - tail
                if remain == 0:
                    cached_paths.pop(i)
                else:
                    cached_paths[i] = (seq[:remain], g)
    # standalone cost probes (reference_scheduler.cpp:407-433)
    for g in range(n):
        for missed in (0, 1, 7, rng.randrange(2 * cfg.kv_capacity_tokens)):
            ca, cb = A.load_cost(g, missed, t), B.load_cost(g, missed, t)
            assert ca == cb, (seed, g, missed, ca, cb)
            stats["probes"] += 1
            stats["infeasible"] += ca.eviction_infeasible
    assert A.stats() == B.stats(), seed
    assert A.redirects() == B.redirects()
    msg = export_diff(A, B, t)
    assert msg is None, (seed, msg)
    if snap:
        msg = snapshot_diff(A, B, t)
        assert msg is None, (seed, msg)
    A.close()
    B.close()


def _fuzz(lib, ref_lib, cases, base):
    stats = dict(snapshots=0, decisions=0, exploit=0, pressure=0, redirected=0, probes=0, infeasible=0)
    for c in range(cases):
        run_case(lib, ref_lib, base * 1000003 + c, stats)
    # the comparison must not be vacuous (test_scheduler_oracle.cpp:17-21)
    assert stats["decisions"] > 5 * cases
    assert stats["exploit"] > 0 and stats["redirected"] > 0 and stats["pressure"] > 0 and stats["infeasible"] > 0, stats
    return stats


def test_fuzz_hostsim(hostsim_lib, true_ref_lib):
    _fuzz(hostsim_lib, true_ref_lib, 1000, 20260815)  # criterion 1 runs 1000 scenarios (acceptance_main.cpp:63-78)


@pytest.mark.gpu
def test_fuzz_b200(b200_lib, true_ref_lib):
    _fuzz(b200_lib, true_ref_lib, 1000, 20260815)


def _redirect_probe(lib, ref_lib):
    """test_scheduler_oracle.cpp:26-66: an installed redirect diverts an
    exploit placement and the target's cost joins the audited list."""
    cfg = SchedulerConfig(history_window_ms=5000, kv_capacity_tokens=4000, th_bal=1.5)
    pol = GlobalPolicy(rebalance=True, autoscale=False, pd_balance=False)
    stem = [100 + j for j in range(32)]
    outs = []
    for L in (ref_lib, lib):
        s = GlobalScheduler(2, cfg, TimeModel(), pol, lib=L)
        first = s.schedule_request(Request(1, stem, 0.0, 8), 1.0)
        assert first.gpu == 0
        s.note_prefill_cached(stem, first.gpu, 2.0)
        got = s.schedule_request(Request(99, stem + [999], 0.0, 8), 5.0)
        assert got.branch == 0 and got.redirected and got.pre_redirect_gpu == 0 and got.gpu == 1
        assert len(got.costs) == 2
        outs.append(got)
    assert _same_decision(outs[0], outs[1])


def test_redirect_probe_hostsim(hostsim_lib, true_ref_lib):
    _redirect_probe(hostsim_lib, true_ref_lib)


@pytest.mark.gpu
def test_redirect_probe_b200(b200_lib, true_ref_lib):
    _redirect_probe(b200_lib, true_ref_lib)
