"""corpus / trace files and the corpus study
(workload.cpp:329-601) — the product's implementation against the unmodified
reference on the same inputs: files byte-identical, parsed contents and
error messages identical, study reports equal field for field (doubles
bitwise)."""
from __future__ import annotations

import random
import struct

import numpy as np
import pytest

from paper_2407_00023_b200 import abi, workload as W


def _trace_from_prompts(prompts, outs=None):
    off = np.zeros(len(prompts) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    toks = np.array([t for p in prompts for t in p], dtype=np.int32)
    n = len(prompts)
    outs = outs if outs is not None else [1 + (i * 7) % 40 for i in range(n)]
    return W.Trace(toks, off, np.arange(1, n + 1, dtype=np.int64), np.arange(n, dtype=np.float64) * 1.25,
                   np.array(outs, dtype=np.int64))


def _same_study(a, b):
    for k in a:
        if isinstance(a[k], dict):
            for f in a[k]:
                assert struct.pack("d", float(a[k][f])) == struct.pack("d", float(b[k][f])), (k, f, a[k][f], b[k][f])
        else:
            assert struct.pack("d", float(a[k])) == struct.pack("d", float(b[k])), (k, a[k], b[k])


def _random_corpus(seed, n):
    rng = random.Random(seed)
    stems = [[rng.randrange(50) for _ in range(rng.randrange(1, 30))] for _ in range(4)]
    prompts = []
    for i in range(n):
        roll = rng.randrange(10)
        if roll < 2 and prompts:
            p = list(prompts[rng.randrange(len(prompts))])  # duplicate
        elif roll < 4 and prompts:
            q = prompts[rng.randrange(len(prompts))]
            p = list(q[: rng.randrange(1, len(q) + 1)])  # prefix of an earlier prompt
        else:
            s = stems[rng.randrange(len(stems))]
            p = s[: rng.randrange(1, len(s) + 1)] + [rng.randrange(6) for _ in range(rng.randrange(0, 12))]
        prompts.append(p)
    return _trace_from_prompts(prompts)


@pytest.mark.parametrize("seed", range(40))
def test_study_random_corpora(hostsim_lib, true_ref_lib, seed):
    t = _random_corpus(seed, 5 + seed * 3)
    _same_study(W.analyze(t, lib=true_ref_lib), W.analyze(t, lib=hostsim_lib))


@pytest.mark.parametrize("arch", ["toolbench", "doc_qa", "programming", "embodied_agent", "video_qa",
                                  "tree_of_thought"])
def test_study_archetypes(hostsim_lib, true_ref_lib, arch):
    s = W.default_spec(arch, hostsim_lib)
    s.request_count = 1500
    t = W.generate(s, 13, 2000.0, 14, lib=hostsim_lib)
    a, b = W.analyze(t, lib=true_ref_lib), W.analyze(t, lib=hostsim_lib)
    assert a["requests"] == 1500 and a["key_portion_count"] > 0
    _same_study(a, b)


def test_corpus_files_roundtrip(tmp_path, hostsim_lib, true_ref_lib):
    t = W.CONFIGS["c1"].trace(lib=hostsim_lib, n_requests=300)
    for with_arr in (True, False):
        pa, pb = str(tmp_path / f"ref{with_arr}.txt"), str(tmp_path / f"new{with_arr}.txt")
        W.write_corpus(pa, t, with_arr, lib=true_ref_lib)
        W.write_corpus(pb, t, with_arr, lib=hostsim_lib)
        assert open(pa, "rb").read() == open(pb, "rb").read()
        (ra, ha), (rb, hb) = W.read_corpus(pa, lib=true_ref_lib), W.read_corpus(pa, lib=hostsim_lib)
        for f in ("tokens", "offsets", "ids", "arrivals", "output_lens"):
            assert np.array_equal(getattr(ra, f), getattr(rb, f)), f
        assert np.array_equal(ha, hb) and bool(ha.all()) == with_arr
        assert np.array_equal(rb.tokens, t.tokens) and np.array_equal(rb.offsets, t.offsets)


BAD_CORPORA = ["1 2\n", "x 5 6 7\n", "1 0.5 7\n", "1 -3.0 5 6 7\n", "1 5 6 0\n", "1 5 99999999999 3\n",
               "\n\n1 2 3 4\n2 a 3\n"]


@pytest.mark.parametrize("text", BAD_CORPORA)
def test_corpus_errors_match(tmp_path, hostsim_lib, true_ref_lib, text):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    errs = []
    for lib in (true_ref_lib, hostsim_lib):
        with pytest.raises(ValueError) as e:
            W.read_corpus(str(p), lib=lib)
        errs.append(str(e.value))
    assert errs[0] == errs[1]


TRACES = ["arrival_s,prompt_len,output_len\n3.5,100,10\n1.0,50,5\n1.0,60,6\n\n2.25 , 70 , 7\n",
          "t,p,o\n0,1,1\n"]
BAD_TRACES = ["", "1.0,2,3\n", "a,b,c\n1.0,2\n", "a,b,c\n-1,2,3\n", "a,b,c\n1,0,3\n", "a,b,c\n1,2,x\n"]


@pytest.mark.parametrize("text", TRACES)
def test_trace_files(tmp_path, hostsim_lib, true_ref_lib, text):
    p = tmp_path / "t.csv"
    p.write_text(text)
    a, b = W.read_trace(str(p), lib=true_ref_lib), W.read_trace(str(p), lib=hostsim_lib)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    spec = W.default_spec("toolbench", hostsim_lib)
    ta = W.synthesize_from_trace(*a, spec, 99, lib=true_ref_lib)
    tb = W.synthesize_from_trace(*b, spec, 99, lib=hostsim_lib)
    for f in ("tokens", "offsets", "ids", "arrivals", "output_lens"):
        assert np.array_equal(getattr(ta, f), getattr(tb, f)), f


@pytest.mark.parametrize("text", BAD_TRACES)
def test_trace_errors_match(tmp_path, hostsim_lib, true_ref_lib, text):
    p = tmp_path / "t.csv"
    p.write_text(text)
    errs = []
    for lib in (true_ref_lib, hostsim_lib):
        with pytest.raises(ValueError) as e:
            W.read_trace(str(p), lib=lib)
        errs.append(str(e.value))
    assert errs[0] == errs[1]


def test_synthesize_zipf_lengths(hostsim_lib, true_ref_lib):
    rng = np.random.default_rng(5)
    n = 2000
    a = np.sort(rng.uniform(0, 100, n))
    pl = rng.integers(1, 4000, n)
    ol = rng.integers(1, 300, n)
    spec = W.default_spec("toolbench", hostsim_lib)
    ta = W.synthesize_from_trace(a, pl, ol, spec, 7, lib=true_ref_lib)
    tb = W.synthesize_from_trace(a, pl, ol, spec, 7, lib=hostsim_lib)
    assert np.array_equal(ta.tokens, tb.tokens) and np.array_equal(ta.offsets, tb.offsets)
    assert np.array_equal(np.diff(tb.offsets), pl)
    _same_study(W.analyze(ta, lib=true_ref_lib), W.analyze(tb, lib=hostsim_lib))
