"""dev: one parity case on the product with the error message."""
import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from paper_2407_00023_b200 import abi
from test_parity import CASES
from parity import replay, diff_decisions
import conftest
lib = abi.product_lib(); ref = abi.load_library(abi.REF_SO); gen = abi.load_library(conftest.build_hostsim())
for name in sys.argv[1:]:
    cfg = CASES[name]; tr = cfg.trace(lib=gen)
    sa, a = replay(ref, cfg, tr); sb, b = replay(lib, cfg, tr)
    print(name, a.n_done, b.n_done, getattr(b, "error", None), diff_decisions(a, b))
