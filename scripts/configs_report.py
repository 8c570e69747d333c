"""All five BASELINE.json configs on the B200: decisions/s of the product
(device-resident replay, CUDA-event kernel time) beside the unmodified
reference on the same trace on the host core, and a bit-exact decision
check on the overlap.  Writes one JSON line per config to stdout."""
import ctypes, json, os, sys, time
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
from parity import diff_decisions

SIZES = {"c1": (1000, 1000), "c2": (100000, 100000), "c3": (10000, 10000), "c4": (1000000, 100000), "c5": (200000, 100000)}


def main(names):
    prod = abi.product_lib()
    ref = abi.load_library(abi.REF_SO)
    for name in names:
        n, n_ref = SIZES[name]
        cfg = W.CONFIGS[name]
        tr = cfg.trace(lib=prod, n_requests=n)
        s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=prod)
        s.replay(tr.head(min(n, 2000)), cfg.driver)  # warm-up (allocations, module load)
        prod.e2_reset(s._h)
        prod.e2_profile_reset(s._h, 1)
        t0 = time.perf_counter()
        b = s.replay(tr, cfg.driver)
        wall = time.perf_counter() - t0
        prof = abi.ProfileC()
        prod.e2_profile_get(s._h, ctypes.byref(prof))
        kms = sum(prof.ms)
        r = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=ref)
        trr = tr.head(n_ref) if n_ref < n else tr
        t0 = time.perf_counter()
        a = r.replay(trr, cfg.driver)
        cpu = time.perf_counter() - t0
        bb = type(b)(b.decisions[:trr.n], b.costs[:trr.n], None, min(b.n_done, trr.n))
        d = diff_decisions(a, bb)
        nodes = s.node_count()
        # the product on exactly the reference's prefix (same work on both sides)
        same = None
        if trr.n < tr.n:
            prod.e2_reset(s._h)
            prod.e2_profile_reset(s._h, 1)
            s.replay(trr, cfg.driver)
            p2 = abi.ProfileC()
            prod.e2_profile_get(s._h, ctypes.byref(p2))
            same = trr.n / (sum(p2.ms) / 1000)
        print(json.dumps({
            "config": cfg.name, "requests": tr.n, "instances": cfg.n_gpus,
            "b200_decisions_per_s_kernel": tr.n / (kms / 1000), "b200_decisions_per_s_wall": tr.n / wall,
            "kernel_ms": {k: prof.ms[i] for i, k in enumerate(["match", "group", "serial", "other"])},
            "match_gbps": (prof.match_bytes / 1e9) / (prof.ms[0] / 1e3) if prof.ms[0] else None,
            "reference_requests": trr.n, "reference_decisions_per_s": trr.n / cpu,
            "b200_decisions_per_s_on_reference_prefix": same if same is not None else tr.n / (kms / 1000),
            "bit_exact_on_reference_prefix": d is None, "first_mismatch": d,
            "nodes": nodes,
        }), flush=True)
        s.close(); r.close()


if __name__ == "__main__":
    main(sys.argv[1:] or list(SIZES))
