import ctypes, os, sys
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
lib = abi.load_library("build/libbase.so")
for name, n in [("c2", 100000), ("c4", 50000)]:
    cfg = W.CONFIGS[name]
    tr = cfg.trace(lib=lib, n_requests=n)
    for B in [8192, 16384, 32768, 65536]:
        cfg.driver.batch = B
        s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
        s.replay(tr.head(2000), cfg.driver)
        best = 0
        for _ in range(2):
            lib.e2_reset(s._h); lib.e2_profile_reset(s._h, 1)
            s.replay(tr, cfg.driver)
            p = abi.ProfileC(); lib.e2_profile_get(s._h, ctypes.byref(p))
            best = max(best, n / (sum(p.ms) / 1000))
        print(name, "batch", B, round(best), flush=True)
        s.close()
