"""dev: per-phase cycles per request of each C5 chunk (E2_PHASES build), streamed."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
lib = abi.load_library(sys.argv[1])
lib.e2_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cfg = W.CONFIGS["c5"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 260000
s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
lib.e2_replay_set_continue(s._h, 1)
prev = [0] * 48
names = {6: "extents", 7: "cost_prep", 8: "cost_pick", 9: "ensure", 10: "path_upd", 16: "wait_evict", 24: "w1_plan",
         25: "w1_split", 26: "w1_tail", 27: "w1_whole", 20: "w1_fixes", 31: "w1_fixwait", 38: "walk_hint", 39: "walk_leader",
         40: "walk_climb", 41: "walk_probe", 44: "expl_prep", 45: "expl_cost", 33: "cands", 32: "prologue", 34: "validate",
         35: "handoff", 37: "post", 2: "commit_other", 1: "decide_other", 17: "redo_cnt", 12: "probe_cnt"}
for ch in cfg.chunks(n, lib=lib):
    r = s.replay(ch, cfg.driver, want_costs=False)
    buf = (ctypes.c_uint64 * 48)()
    lib.e2_debug_phases(s._h, buf)
    d = [buf[i] - prev[i] for i in range(48)]
    prev = list(buf)
    k = ch.n
    print(f"chunk of {k}: nodes {s.node_count()} " + " ".join(f"{v}={d[i] / k:.0f}" for i, v in sorted(names.items())), flush=True)
