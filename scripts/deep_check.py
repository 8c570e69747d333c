"""dev: deep-chain parity (tests/test_deep_paths.py) against a given library, repeated."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2407_00023_b200 import abi
from test_deep_paths import _cfg, chain_trace
from parity import diff_decisions, replay
lib = abi.load_library(sys.argv[1]); ref = abi.load_library(abi.REF_SO)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for cap, hw in [(200000, 150000), (20000, 16000)]:
    cfg = _cfg(1400, cap, hw, 256); tr = chain_trace(1400)
    _, a = replay(ref, cfg, tr)
    res = []
    for k in range(reps):
        _, b = replay(lib, cfg, tr)
        res.append(diff_decisions(a, b))
    print(sys.argv[1], os.environ.get("E2_NO_PIPE", "0"), cap, res, flush=True)
