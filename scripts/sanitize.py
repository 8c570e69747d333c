"""dev: one C2 replay prefix through the product under compute-sanitizer (the
four-warp pipelined k_serial, K1 and the leader rounds)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler
name, n = sys.argv[1], int(sys.argv[2])
lib = abi.product_lib()
cfg = W.CONFIGS[name]
tr = cfg.trace(lib=lib, n_requests=n)
s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
r = s.replay(tr, cfg.driver)
print("replayed", r.n_done, "of", tr.n)
