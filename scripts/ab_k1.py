"""dev: K1 (k_match) per-launch time and algorithmic GB/s for several library builds, one box."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
name = sys.argv[2]; n = int(sys.argv[3])
cfg = W.CONFIGS[name]
for path in sys.argv[1].split(","):
    lib = abi.load_library(path)
    tr = cfg.trace(lib=lib, n_requests=n)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    s.replay(tr.head(min(n, 2000)), cfg.driver)
    res = []
    for _ in range(2):
        lib.e2_reset(s._h)
        lib.e2_profile_reset(s._h, 1)
        s.replay(tr, cfg.driver, want_costs=False)
        p = abi.ProfileC()
        lib.e2_profile_get(s._h, ctypes.byref(p))
        ms = p.ms[0] / max(1, p.launches[0])
        res.append((ms, p.match_bytes / 1e9 / (p.ms[0] / 1e3), n / (sum(p.ms) / 1e3)))
    ms, gbs, dps = min(res)
    print(f"{os.path.basename(path)} top={'off' if os.environ.get('E2_NO_TOP') == '1' else 'on'} {name} n={n} "
          f"k1_ms/launch {ms:.4f} k1_GB/s {gbs:.0f} decisions/s {dps:.0f}", flush=True)
    s.close()
