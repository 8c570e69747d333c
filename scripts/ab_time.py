"""dev: decisions/s (CUDA-event kernel time) of a replay with a given library; for A/B runs on one box."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
name = sys.argv[2]; n = int(sys.argv[3]); reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = W.CONFIGS[name]
for path in sys.argv[1].split(","):
    lib = abi.load_library(path)
    tr = cfg.trace(lib=lib, n_requests=n)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    s.replay(tr.head(min(n, 2000)), cfg.driver)
    best = 0
    for _ in range(reps):
        lib.e2_reset(s._h)
        lib.e2_profile_reset(s._h, 1)
        s.replay(tr, cfg.driver)
        p = abi.ProfileC()
        lib.e2_profile_get(s._h, ctypes.byref(p))
        best = max(best, n / (sum(p.ms) / 1000))
    print(f"{path} {name} n={n} decisions/s {best:.0f}", flush=True)
    s.close()
