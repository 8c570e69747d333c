"""Trace generation (input only) is bit-identical to kvsched::generate +
assign_poisson_arrivals (workload.cpp:235-327, 486-497) for every reference
archetype, and the config-3/4 extensions are deterministic."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2407_00023_b200 import workload as W


@pytest.mark.parametrize("arch,n", [("toolbench", 3000), ("programming", 500), ("video_qa", 300), ("doc_qa", 600),
                                    ("embodied_agent", 800)])
def test_generator_matches_reference(gen_lib, true_ref_lib, arch, n):
    spec = W.default_spec(arch, gen_lib)
    spec.request_count = n
    a = W.generate(spec, 13, 2000.0, 14, lib=gen_lib)
    b = W.generate(spec, 13, 2000.0, 14, lib=true_ref_lib)
    for f in ("tokens", "offsets", "ids", "arrivals", "output_lens"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_defaults_match_reference(gen_lib, true_ref_lib):
    for arch in ("toolbench", "programming", "video_qa", "doc_qa", "embodied_agent"):
        a, b = W.default_spec(arch, gen_lib), W.default_spec(arch, true_ref_lib)
        for f, _ in a._fields_:
            assert getattr(a, f) == getattr(b, f), (arch, f)


def test_extensions_deterministic(gen_lib):
    c3 = W.CONFIGS["c3"]
    t1, t2 = c3.trace(lib=gen_lib, n_requests=200), c3.trace(lib=gen_lib, n_requests=200)
    assert np.array_equal(t1.tokens, t2.tokens)
    lens = np.diff(t1.offsets)
    assert lens.min() >= 13 + 20000 + 200 and lens.max() <= 13 + 40000 + 300
    spec = W.default_spec("tree_of_thought", gen_lib)
    spec.request_count = 300
    t = W.generate(spec, 5, 1000.0, 6, lib=gen_lib)
    assert t.n == 300 and np.all(np.diff(t.arrivals) > 0)
