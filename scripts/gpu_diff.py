"""Dev check: replay a config prefix on the product library and on the
reference shim, report first mismatch and timings."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler

def exports_equal(a, b, now):
    na, ta, la_a, ha = a.export_arrays(now)
    nb, tb, la_b, hb = b.export_arrays(now)
    if len(na) != len(nb):
        print("export node count", len(na), len(nb)); return False
    fa = np.frombuffer(na, dtype=np.uint64).reshape(len(na), -1)
    fb = np.frombuffer(nb, dtype=np.uint64).reshape(len(nb), -1)
    ok = True
    for col, name in [(0, 'id'), (1, 'parent'), (3, 'edge_len'), (4, 'caching'), (5, 'la_mask')]:
        bad = np.nonzero(fa[:, col] != fb[:, col])[0]
        if len(bad):
            print("export", name, "first mismatch node", bad[0], fa[bad[0]], fb[bad[0]]); ok = False
    if not np.array_equal(ta, tb): print("export tokens differ"); ok = False
    if not np.array_equal(la_a.view(np.uint64), la_b.view(np.uint64)): print("export last_access differ"); ok = False
    if not np.array_equal(ha, hb):
        bad = np.argwhere(ha != hb)[0]; print("export hits differ", bad, ha[bad[0]], hb[bad[0]]); ok = False
    return ok

def main(name, n, other=None, batch=0):
    ref = abi.load_library(abi.REF_SO)
    prod = abi.load_library(other) if other else abi.product_lib()
    cfg = W.CONFIGS[name]
    tr = cfg.trace(lib=prod, n_requests=n)
    drv = cfg.driver
    drv.batch = batch
    out = {}
    for nm, lib in [('ref', ref), ('prod', prod)]:
        s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
        t0 = time.time()
        try:
            r = s.replay(tr, drv)
        except Exception as e:
            print(nm, "ERROR", e, flush=True); r = e.partial
        dt = time.time() - t0
        print(f"{nm} {s.backend}: {dt:.3f}s {r.n_done/dt:.0f} req/s done={r.n_done}", s.stats(), s.node_count(), flush=True)
        out[nm] = (s, r)
    a, b = out['ref'][1], out['prod'][1]
    nd = min(a.n_done, b.n_done)
    ok = a.n_done == b.n_done
    for f in a.decisions.dtype.names:
        x, y = a.decisions[f][:nd], b.decisions[f][:nd]
        bad = np.nonzero(x != y)[0]
        if len(bad):
            ok = False
            print("field", f, "first mismatch at", bad[0], x[bad[0]], y[bad[0]])
    cb = np.nonzero((a.costs[:nd].view(np.uint8).reshape(nd, -1) != b.costs[:nd].view(np.uint8).reshape(nd, -1)).any(1))[0]
    if len(cb):
        ok = False
        print("costs first mismatch", cb[0], a.costs[cb[0]], b.costs[cb[0]])
    now = float(tr.arrivals[-1])
    # reference debug_dump erases map entries while iterating once a GPU's hit
    # deque fully expires (prefix_tree.cpp:423-424 with :37-43): compare exports.
    de = exports_equal(out['ref'][0], out['prod'][0], now)
    print(f"RESULT {name} n={n} decisions_equal={ok} dump_equal={de}", flush=True)
    return ok and de

if __name__ == "__main__":
    name = sys.argv[1]; n = int(sys.argv[2])
    other = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != '-' else None
    batch = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    sys.exit(0 if main(name, n, other, batch) else 1)
