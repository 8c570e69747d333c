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
buf = (ctypes.c_uint64 * 48)()
lib.e2_debug_phases(s._h, buf)
names = ["redirects", "decide_other", "commit_other", "decision_out", "evict_apply", "finished", "walk", "cost_prep",
         "cost_pick", "ensure_path", "path_update", "evict_plan", "", "", "", ""]
tot = sum(buf[:12]) + buf[16] + buf[18] + buf[30] + sum(buf[32:38])
print(name, n, "cycles/request total %.0f" % (tot / n), " ".join("%s=%.0f" % (names[i], buf[i] / n) for i in range(16) if names[i]), "wait_evict=%.0f wait_bar2=%.0f wait_books=%.0f" % (buf[16] / n, buf[18] / n, buf[30] / n), "spec_redo=%.3f" % (buf[17] / n),
      "| warp1: fix_wait=%.0f fixes=%.0f evict=%.0f out=%.0f spin=%.0f books=%.0f" % tuple(buf[k] / n for k in (31, 20, 21, 22, 29, 19)),
      "| evict: plan=%.0f tail_pre=%.0f split=%.0f tail_post=%.0f whole=%.0f" % tuple(buf[k] / n for k in (24, 28, 25, 26, 27)),
      "| decide: prologue=%.0f cands=%.0f | validate=%.0f handoff=%.0f hint_row=%.0f post=%.0f" % tuple(buf[k] / n for k in (32, 33, 34, 35, 36, 37)),
      "| per request: walk_fallback_probes=%.3f evict_tail=%.3f evict_whole=%.3f" % (buf[12] / n, buf[13] / n, buf[14] / n),
      "| walk: hinted=%.0f leader_switch=%.0f climb=%.0f probes=%.0f extents=%.0f" % tuple(buf[k] / n for k in (38, 39, 40, 41, 6)),
      "| redo: spec_fail=%.4f conflict=%.4f" % (buf[42] / n, buf[43] / n),
      "| explore: ratios=%.0f prepare=%.0f costs=%.0f" % (buf[46] / n, buf[44] / n, buf[45] / n))
