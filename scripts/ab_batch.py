"""dev: batch-size sweep (decisions/s of whole replays, wall clock around the synchronous call)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import DriverConfig, GlobalScheduler
lib = abi.product_lib()
for spec in sys.argv[1:]:
    name, n, sizes = spec.split(":")
    n = int(n)
    cfg = W.CONFIGS[name]
    tr = cfg.trace(lib=lib, n_requests=n)
    for B in [int(x) for x in sizes.split(",")]:
        drv = DriverConfig(**{**cfg.driver.__dict__, "batch": B})
        s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
        s.replay(tr.head(2000), drv)
        best = 0
        for _ in range(2):
            lib.e2_reset(s._h)
            t0 = time.perf_counter()
            s.replay(tr, drv, want_costs=False)
            best = max(best, n / (time.perf_counter() - t0))
        print(name, n, "batch", B, round(best), flush=True)
        s.close()
