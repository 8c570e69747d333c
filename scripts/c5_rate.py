"""dev: C5 decisions/s over a long prefix, per 16k-request window of the replay."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
lib = abi.product_lib()
cfg = W.CONFIGS["c5"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
lib.e2_replay_set_continue(s._h, 1)
lib.e2_profile_reset(s._h, 1)
done = 0; prev = 0.0
for ch in cfg.chunks(n, lib=lib):
    r = s.replay(ch, cfg.driver, want_costs=False)
    p = abi.ProfileC(); lib.e2_profile_get(s._h, ctypes.byref(p))
    tot = sum(p.ms)
    done += r.n_done
    print(f"requests {done}: chunk {ch.n / ((tot - prev) / 1e3):.0f} decisions/s, cumulative {done / (tot / 1e3):.0f}, nodes {s.node_count()}", flush=True)
    prev = tot
