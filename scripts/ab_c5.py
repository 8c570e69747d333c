"""dev: C5 streamed chunk by chunk with several libraries (A/B): decisions/s per chunk (kernel time)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
cfg = W.CONFIGS["c5"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 196608
for path in sys.argv[1].split(","):
    lib = abi.load_library(path)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    lib.e2_replay_set_continue(s._h, 1)
    lib.e2_profile_reset(s._h, 1)
    prev, rates, done = 0.0, [], 0
    for ch in cfg.chunks(n, lib=lib):
        r = s.replay(ch, cfg.driver, want_costs=False)
        p = abi.ProfileC(); lib.e2_profile_get(s._h, ctypes.byref(p))
        tot = sum(p.ms); rates.append(ch.n / ((tot - prev) / 1e3)); prev = tot; done += r.n_done
    print(f"{path} c5 n={done}: per chunk " + " ".join(f"{x:.0f}" for x in rates) + f" | overall {done / (prev / 1e3):.0f} decisions/s", flush=True)
    s.close()
