"""Known-answer tests of the reference, restated against the C-ABI mirror.

Each test follows one TEST_CASE of proj/tests/test_global_scheduler.cpp /
test_prefix_tree.cpp / test_cost_model.cpp (cited per test) and runs on
every backend: the reference shim itself (pins the restatement), the host
emulation of the product engine, and — marked gpu — libe2sched.so.
"""
from __future__ import annotations

import pytest

from paper_2407_00023_b200.scheduler import (
    ConfigError,
    EvictedRange,
    GlobalPolicy,
    GlobalScheduler,
    NoAdmissibleGpu,
    Request,
    SchedulerConfig,
    SimError,
    TimeModel,
)

BACKENDS = ["ref", "oracle", "hostsim", pytest.param("b200", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def lib(request):
    return request.getfixturevalue({"ref": "true_ref_lib", "oracle": "oracle_lib", "hostsim": "hostsim_lib", "b200": "b200_lib"}[request.param])


def identity():  # test_global_scheduler.cpp:11-18
    return TimeModel(0.0, 1.0, 0.0, 8.0)


def seq(base, n):
    return list(range(base, base + n))


def req(i, prompt, arrival=0.0):
    return Request(i, prompt, arrival, 8)


def mk(lib, n, cfg=None, model=None, pol=None):
    return GlobalScheduler(n, cfg or SchedulerConfig(), model or identity(), pol or GlobalPolicy(), lib=lib)


def approx(a, b):
    return abs(a - b) <= 1e-9 * max(1.0, abs(b))


def test_exploit_routes_to_longest_extent(lib):  # :42-58
    s = mk(lib, 4)
    s.note_prefill_cached(seq(100, 63), 2, 0.0)
    d = s.schedule_request(req(1, seq(100, 100)), 1.0)
    assert d.branch == 0 and d.gpu == 2
    assert (d.cached_len, d.missed_len, d.missed_on_chosen) == (63, 37, 37)
    assert not d.redirected and d.decode_ratios == {}
    assert [c.gpu for c in d.costs] == [2]
    assert s.stats().exploit == 1 and s.stats().tree_reads == 1


def test_explore_ties_lowest_gpu(lib):  # :60-67
    s = mk(lib, 4)
    d = s.schedule_request(req(1, seq(500, 40)), 0.0)
    assert d.branch == 1 and d.gpu == 0 and len(d.costs) == 4
    assert all(approx(c.cost.total_ms(), 40.0) for c in d.costs)


def test_explore_lowest_total(lib):  # :69-80
    s = mk(lib, 2)
    s.schedule_request(req(1, seq(1000, 60)), 0.0)
    s.schedule_request(req(2, seq(2000, 35)), 1.0)
    d = s.schedule_request(req(3, seq(3000, 40)), 2.0)
    assert d.branch == 1 and len(d.costs) == 2
    assert approx(d.costs[0].cost.total_ms(), 100.0) and approx(d.costs[1].cost.total_ms(), 75.0)
    assert d.gpu == 1


@pytest.mark.parametrize("pd", [True, False])
def test_decode_pressure(lib, pd):  # :82-111
    s = mk(lib, 4, pol=GlobalPolicy(rebalance=False, autoscale=False, pd_balance=pd))
    s.note_prefill_cached(seq(40000, 1000), 3, 0.0)
    s.note_prefill_cached(seq(41000, 95), 3, 0.0)
    s.schedule_request(req(1, seq(40000, 1000) + seq(42000, 500)), 0.0)
    s.schedule_request(req(2, seq(41000, 95) + seq(43000, 5)), 1.0)
    s.note_finished(1, 2.0, 8)
    if pd:
        assert approx(s.decode_ratio(3), 0.95)
    d = s.schedule_request(req(3, seq(44000, 50)), 3.0)
    if pd:
        assert d.branch == 2 and d.gpu == 3 and d.costs == []
        assert approx(d.decode_ratios[3], 0.95) and s.stats().decode_pressure == 1
    else:
        assert d.branch == 1 and d.gpu == 0


def test_decode_ratio_weights(lib):  # :113-133
    s = mk(lib, 1)
    assert s.decode_ratio(0) == 0.0
    x = seq(50000, 50)
    s.note_prefill_cached(x, 0, 0.0)
    s.schedule_request(req(1, x), 1.0)
    assert approx(s.decode_ratio(0), 1.0)
    y = seq(50000, 10) + seq(51000, 40)
    s.schedule_request(req(2, y), 2.0)
    assert approx(s.decode_ratio(0), 0.6)
    s.note_prefill_cached(y, 0, 3.0)
    assert approx(s.decode_ratio(0), 0.6)
    s.note_finished(1, 4.0, 8)
    s.note_finished(2, 5.0, 8)
    assert s.decode_ratio(0) == 0.0


def test_rebalance_threshold(lib):  # :135-159
    s = mk(lib, 2)
    s.schedule_request(req(1, seq(1000, 100)), 0.0)
    s.schedule_request(req(2, seq(2000, 60)), 1.0)
    s.schedule_request(req(3, seq(3000, 1)), 2.0)
    assert s.redirects() == {}
    s = mk(lib, 2)
    s.schedule_request(req(1, seq(1000, 250)), 0.0)
    s.schedule_request(req(2, seq(2000, 100)), 1.0)
    d = s.schedule_request(req(3, seq(3000, 1)), 2.0)
    assert s.redirects() == {0: 1} and s.stats().rebalance_installs == 1 and not d.redirected
    s.schedule_request(req(4, seq(4000, 1)), 3.0)
    assert s.stats().rebalance_installs == 1


def test_redirect_follow_and_expire(lib):  # :161-190
    s = mk(lib, 2)
    p = seq(10000, 100)
    s.note_prefill_cached(p, 0, 0.0)
    q1 = s.schedule_request(req(1, p + seq(11000, 400)), 0.0)
    assert q1.branch == 1 and q1.gpu == 0
    q2 = s.schedule_request(req(2, p + seq(12000, 50)), 1.0)
    assert q2.branch == 0 and q2.redirected and q2.pre_redirect_gpu == 0 and q2.gpu == 1
    assert q2.missed_on_chosen == 150 and s.stats().rebalance_installs == 1
    q3 = s.schedule_request(req(3, p + seq(13000, 20)), 2.0)
    assert q3.redirected and q3.gpu == 1 and s.stats().redirected == 2
    q4 = s.schedule_request(req(4, seq(14000, 30)), 3.0)
    assert s.redirects() == {} and not q4.redirected and q4.gpu == 1


def test_single_gpu_never_redirects(lib):  # :192-200
    s = mk(lib, 1)
    for i in range(5):
        assert s.schedule_request(req(i + 1, seq(1000 * (i + 1), 50)), float(i)).gpu == 0
    assert s.redirects() == {} and s.stats().rebalance_installs == 0


@pytest.mark.parametrize("delay,rebalance,events", [(85.0, True, 1), (70.0, True, 0), (85.0, False, 0)])
def test_autoscale_replication(lib, delay, rebalance, events):  # :202-257
    H = 180000.0
    r, s_, t = seq(60000, 50), seq(61000, 300), seq(62000, 300)
    sch = mk(lib, 2, pol=GlobalPolicy(rebalance=rebalance))
    sch.note_prefill_cached(r, 0, 0.0)
    sch.note_prefill_cached(s_, 0, 0.0)
    sch.note_prefill_cached(t, 1, 0.0)
    sch.schedule_request(Request(1, t + seq(64000, 10), 1000.0, 8), 1000.0)
    sch.schedule_request(Request(2, r + seq(63000, 10), 1001.0, 8), 1001.0)
    sch.note_admitted(2, 1041.0)
    sch.schedule_request(Request(3, s_ + seq(65000, 200), H + 100, 8), H + 100)
    sch.schedule_request(Request(4, r + seq(66000, 10), H + 200, 8), H + 200)
    sch.note_admitted(4, H + 200 + delay)
    sch.schedule_request(Request(5, seq(67000, 20), H + 300, 8), H + 300)
    assert sch.stats().autoscale_events == events
    if not rebalance:
        assert sch.redirects() == {}
    if events:
        nodes = {n.edge[0]: n for n in sch.export_nodes(H + 300) if n.edge}
        rn = nodes[60000]
        assert set(rn.caching_gpus) == {0, 1}
        assert nodes[63000].caching_gpus == ()
        assert nodes[66000].caching_gpus == (1,)
        sch.schedule_request(Request(6, seq(68000, 20), H + 400, 8), H + 400)
        assert sch.stats().autoscale_events == 1


def test_round_robin(lib):  # :259-275
    s = mk(lib, 3, pol=GlobalPolicy(mode=1))
    for i in range(7):
        d = s.schedule_request(req(i + 1, seq(1000 * (i + 1), 30)), float(i))
        assert d.branch == 3 and d.gpu == i % 3 and d.missed_on_chosen == 30
    st = s.stats()
    assert st.round_robin == 7 and st.tree_reads == 0 and s.node_count() == 0
    assert s.gpu_load_ms(0, 10.0) == 0.0
    s.note_finished(1, 10.0, 8)
    assert s.decode_ratio(0) == 0.0


def test_capacity_rejects(lib):  # :277-288
    cfg = SchedulerConfig(kv_capacity_tokens=100)
    s = mk(lib, 2, cfg)
    with pytest.raises(NoAdmissibleGpu):
        s.schedule_request(req(1, seq(1000, 101)), 0.0)
    s.schedule_request(req(2, seq(2000, 100)), 1.0)
    rr = mk(lib, 2, cfg, pol=GlobalPolicy(mode=1))
    with pytest.raises(NoAdmissibleGpu):
        rr.schedule_request(req(3, seq(3000, 101)), 0.0)


def test_window_landing(lib):  # :290-305
    s = mk(lib, 2)
    s.schedule_request(req(1, seq(1000, 100)), 5.0)
    assert approx(s.gpu_load_ms(0, 5.0), 100.0) and s.gpu_load_ms(1, 5.0) == 0.0
    assert s.window_sizes(0, 5.0)[:2] == (1, 0) and s.window_sizes(1, 5.0)[:2] == (0, 0)
    assert s.redirects() == {} and s.node_count() > 0


def test_config_validation(lib):  # :307-319
    for cfg in (SchedulerConfig(th_bal=1.0), SchedulerConfig(imbal_ratio=1.5), SchedulerConfig(kv_capacity_tokens=0)):
        with pytest.raises(ConfigError):
            mk(lib, 2, cfg)
    with pytest.raises(ConfigError):
        mk(lib, 0)


def test_non_contiguous_exploit_fails(lib):  # :321-336
    s = mk(lib, 2)
    full = seq(100, 40)
    s.note_prefill_cached(full, 0, 1.0)
    s.note_eviction(EvictedRange(full[:10], 10), 0, 2.0)
    with pytest.raises(SimError):
        s.schedule_request(req(7, full), 3.0)


# --- prefix tree behaviour observable through the scheduler ------------------
def test_contiguity_and_cached_len(lib):  # test_prefix_tree.cpp:100-129
    s = mk(lib, 2)
    s.note_prefill_cached([1, 2], 0, 10.0)
    s.note_prefill_cached([1, 2, 3, 4], 1, 20.0)
    m, c, per = s.match([1, 2, 3, 4])
    assert (m, c, per) == (4, 4, {0: 2, 1: 4})
    s.note_eviction(EvictedRange([1, 2], 2), 1, 21.0)
    m, c, per = s.match([1, 2, 3, 4])
    assert per == {0: 2} and c == 4 and s.cached_tokens(1) == 2
    s.note_eviction(EvictedRange([1, 2], 2), 0, 22.0)
    m, c, per = s.match([1, 2, 3, 4])
    assert c == 2 and per == {}


def test_uncache_suffix_split_and_idempotent(lib):  # test_prefix_tree.cpp:288-300
    s = mk(lib, 1)
    p = list(range(1, 11))
    s.note_prefill_cached(p, 0, 10.0)
    s.note_eviction(EvictedRange(p, 3), 0, 11.0)
    assert s.cached_tokens(0) == 7
    m, c, per = s.match(p)
    assert m == 10 and per == {0: 7}
    s.note_eviction(EvictedRange(p, 3), 0, 12.0)
    assert s.cached_tokens(0) == 7


def test_dead_node_window_boundary(lib):  # test_prefix_tree.cpp:248-261, via hits-only inserts
    cfg = SchedulerConfig(history_window_ms=180000.0)
    s = mk(lib, 1, cfg)
    s.schedule_request(req(1, [1, 2]), 0.0)
    s.schedule_request(req(2, [3, 4]), 1.0)
    s.note_prefill_cached([5, 6], 0, 500.0)
    assert s.prune_dead_nodes(180001.0) == 1
    edges = {tuple(n.edge) for n in s.export_nodes(180001.0)}
    assert (1, 2) not in edges and (3, 4) in edges and (5, 6) in edges


def test_debug_dump_golden(lib):  # test_prefix_tree.cpp:302-313 (insert semantics via the scheduler)
    s = mk(lib, 2, pol=GlobalPolicy(rebalance=False, autoscale=False, pd_balance=False))
    s.note_prefill_cached([1, 2, 3], 0, 10.0)
    s.note_prefill_cached([1, 2, 4], 1, 20.0)
    assert s.debug_dump(30.0) == (
        "d0 len=0 gpus=[] hits=[]\n"
        "  d1 len=2 gpus=[0,1] hits=[]\n"
        "    d2 len=1 gpus=[0] hits=[]\n"
        "    d2 len=1 gpus=[1] hits=[]\n"
    )
    s.schedule_request(req(1, [1, 2, 3]), 30.0)
    dump = s.debug_dump(30.0)
    assert dump.splitlines()[1].endswith("hits=[0:1]")
