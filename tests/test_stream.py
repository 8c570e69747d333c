"""Config 5 as a stream: chunked generation with token-id reuse,
and a replay continued chunk by chunk (e2_replay_set_continue) that equals
one replay of the concatenated trace — on the host emulation against the
unmodified reference here, and on the B200 under -m gpu at >=100k requests."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from paper_2407_00023_b200 import workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler, ReplayResult

from parity import assert_same_state, diff_decisions, replay


def _small_stream(n, chunk):
    base = W.CONFIGS["c5"]
    cfg = W.MixConfig(**{f.name: getattr(base, f.name) for f in dataclasses.fields(W.Config) if f.name != "n_requests"},
                      n_requests=n)
    cfg.CHUNK = chunk
    return cfg


def streamed_replay(lib, cfg, chunks, driver=None):
    """Replay the chunks one call each on one handle (continued)."""
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    assert lib.e2_replay_set_continue(s._h, 1) == 0
    parts = [s.replay(ch, driver or cfg.driver, want_costs=True) for ch in chunks]
    dec = np.concatenate([p.decisions for p in parts])
    cost = np.concatenate([p.costs for p in parts])
    return s, ReplayResult(dec, cost, None, sum(p.n_done for p in parts))


def test_chunks_random_access_and_id_space(gen_lib):
    cfg = _small_stream(2300, 800)
    seq = list(cfg.chunks(lib=gen_lib))
    assert [c.n for c in seq] == [800, 800, 700]
    direct = cfg.chunk(1, lib=gen_lib)
    assert np.array_equal(direct.tokens, seq[1].tokens) and np.array_equal(direct.offsets, seq[1].offsets)
    t = W.concat(seq)
    assert t.n == 2300 and np.array_equal(t.ids, np.arange(1, 2301))
    assert np.all(np.diff(t.arrivals) >= 0)
    assert t.tokens.min() >= 0 and t.tokens.max() < 2**31 - 1


def test_last_chunk_of_10M_stream_is_generable(gen_lib):
    """The reference's single fresh-id counter exhausts int32 long before 10M
    requests; the stream's last chunk is generated directly."""
    cfg = W.CONFIGS["c5"]
    last = (cfg.n_requests - 1) // cfg.CHUNK
    ch = cfg.chunk(last, lib=gen_lib)
    assert ch.ids[-1] == cfg.n_requests
    assert ch.n == cfg.n_requests - last * cfg.CHUNK
    assert ch.tokens.max() < 2**31 - 1 and ch.tokens.min() >= 0
    assert ch.arrivals[0] > cfg.chunk(last - 1, lib=gen_lib, q=10).arrivals[-1]


def _stream_parity(lib, ref_lib, gen_lib, cfg):
    chunks = list(cfg.chunks(lib=gen_lib))
    whole = W.concat(chunks)
    sa, a = replay(ref_lib, cfg, whole, want_ratios=False)
    sb, b = streamed_replay(lib, cfg, chunks)
    assert getattr(a, "error", None) is None, a.error
    d = diff_decisions(a, b)
    assert d is None, f"first mismatch at request {d[0]} field {d[1]}"
    assert a.n_done == b.n_done == whole.n
    assert_same_state(sa, sb, float(whole.arrivals[-1]))


def test_streamed_replay_equals_one_replay_hostsim(hostsim_lib, ref_lib, gen_lib):
    cfg = _small_stream(2600, 700)
    cfg.driver = dataclasses.replace(cfg.driver, finish_lag=900)  # the lag spans a whole chunk
    _stream_parity(hostsim_lib, ref_lib, gen_lib, cfg)


@pytest.mark.gpu
def test_streamed_c5_parity_b200(b200_lib, ref_lib, gen_lib):
    """C5 as streamed on the B200: 3 chunks of 16384 vs the reference
    replaying the concatenation in one go (C5 at 100k requests in one replay:
    test_parity.py)."""
    _stream_parity(b200_lib, ref_lib, gen_lib, _small_stream(3 * 16384, 16384))
