"""dev: the deep-chain parity case with the product's error message."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2407_00023_b200 import abi
from test_deep_paths import _cfg, chain_trace
from parity import replay, diff_decisions
lib = abi.product_lib()
ref = abi.load_library(abi.REF_SO)
cfg = _cfg(1400, 200000, 150000, 256)
tr = chain_trace(1400)
sa, a = replay(ref, cfg, tr)
sb, b = replay(lib, cfg, tr)
print("ref", a.n_done, getattr(a, "error", None))
print("b200", b.n_done, getattr(b, "error", None))
print("diff", diff_decisions(a, b))
