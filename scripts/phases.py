"""dev: per-phase cycles of the serial replay (E2_PHASES build)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
lib = abi.load_library(sys.argv[1])
lib.e2_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
name = sys.argv[2]; n = int(sys.argv[3])
cfg = W.CONFIGS[name]
tr = cfg.trace(lib=lib, n_requests=n)
s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
r = s.replay(tr, cfg.driver)
buf = (ctypes.c_uint64 * 8)()
lib.e2_debug_phases(s._h, buf)
names = ["redirects", "decide", "commit(+mark)", "decision_out", "eviction", "finished"]
tot = sum(buf[:6])
print(name, n, "cycles/request total %.0f" % (tot / n), " ".join("%s=%.0f" % (names[i], buf[i] / n) for i in range(6)))
