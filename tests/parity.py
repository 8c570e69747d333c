"""Comparison helpers shared by the parity tests (decision streams, cost
terms bit-for-bit, and mirror exports)."""
from __future__ import annotations

import numpy as np

from paper_2407_00023_b200.scheduler import GlobalScheduler


def replay(lib, cfg, trace, driver=None, want_ratios=True):
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=getattr(cfg, "policy", None), lib=lib)
    try:
        r = s.replay(trace, driver or cfg.driver, want_costs=True, want_ratios=want_ratios)
    except Exception as e:  # keep the partial stream for the diff
        r = getattr(e, "partial", None)
        if r is None:
            raise
        r.error = e
    return s, r


def diff_decisions(a, b, n=None):
    """First mismatching (index, field) between two ReplayResults, or None."""
    if a.n_done != b.n_done:
        return (min(a.n_done, b.n_done), "n_done")
    nd = a.n_done if n is None else min(n, a.n_done)
    for f in a.decisions.dtype.names:
        bad = np.nonzero(a.decisions[f][:nd] != b.decisions[f][:nd])[0]
        if len(bad):
            return (int(bad[0]), f)
    # costs: only the evaluated entries, compared as raw bytes (bitwise doubles)
    for i in np.nonzero(a.decisions["n_costs"][:nd] > 0)[0]:
        k = int(a.decisions["n_costs"][i])
        if a.costs[i, :k].tobytes() != b.costs[i, :k].tobytes():
            return (int(i), "costs")
    if a.ratios is not None and b.ratios is not None:
        for i in np.nonzero(a.decisions["has_ratios"][:nd] > 0)[0]:
            if a.ratios[i].tobytes() != b.ratios[i].tobytes():
                return (int(i), "ratios")
    return None


def export_diff(sa: GlobalScheduler, sb: GlobalScheduler, now: float):
    """Compare mirror exports (ids, parents, edges, caching sets, last_access
    presence+bits, windowed hit counts).  Returns a message or None."""
    na, ta, la_a, ha = sa.export_arrays(now)
    nb, tb, la_b, hb = sb.export_arrays(now)
    if len(na) != len(nb):
        return f"node count {len(na)} != {len(nb)}"
    fa = np.frombuffer(na, dtype=np.uint64).reshape(len(na), -1)
    fb = np.frombuffer(nb, dtype=np.uint64).reshape(len(nb), -1)
    for col, name in [(0, "id"), (1, "parent_id"), (3, "edge_len"), (4, "caching"), (5, "last_access_mask")]:
        bad = np.nonzero(fa[:, col] != fb[:, col])[0]
        if len(bad):
            return f"{name} differs at export index {bad[0]}: {fa[bad[0]]} vs {fb[bad[0]]}"
    if not np.array_equal(ta, tb):
        return "edge tokens differ"
    if la_a.tobytes() != la_b.tobytes():
        return "last_access differs"
    if not np.array_equal(ha, hb):
        i = np.argwhere(ha != hb)[0]
        return f"windowed hits differ at node {i[0]} gpu {i[1]}: {ha[i[0], i[1]]} vs {hb[i[0], i[1]]}"
    return None


def snapshot_diff(sa: GlobalScheduler, sb: GlobalScheduler, now: float):
    """Compare snapshot(now) (global_scheduler.cpp:375-394) field by field,
    doubles as raw bits (== on floats; no NaNs occur).  Message or None."""
    a, b = sa.snapshot(now), sb.snapshot(now)
    if (a.now, a.n_gpus, a.redirects) != (b.now, b.n_gpus, b.redirects):
        return "header/redirects differ"
    if len(a.nodes) != len(b.nodes):
        return f"node count {len(a.nodes)} != {len(b.nodes)}"
    for i, (x, y) in enumerate(zip(a.nodes, b.nodes)):
        if x != y:
            return f"node {i}: {x} vs {y}"
    for x, y in zip(a.gpus, b.gpus):
        if x != y:
            return f"gpu {x.id}: {x} vs {y}"
    return None


def assert_same_state(sa, sb, now):
    assert sa.stats() == sb.stats()
    assert sa.node_count() == sb.node_count()
    assert sa.redirects() == sb.redirects()
    for g in range(sa.n_gpus()):
        assert sa.cached_tokens(g) == sb.cached_tokens(g), g
        assert sa.window_sizes(g, now) == sb.window_sizes(g, now), g
    msg = export_diff(sa, sb, now)
    assert msg is None, msg
