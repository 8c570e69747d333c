"""Regenerate the committed golden vectors from the UNMODIFIED reference
(oracle/_ref/libe2ref.so, built from /root/reference by oracle/Makefile).

  python tests/golden/make_golden.py

Writes tests/golden/<case>.npz: the reference's decision stream, cost terms,
decode ratios, final stats and mirror export for small configurations, so
parity tests can run where /root/reference is absent (the GPU box).
"""
from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from paper_2407_00023_b200 import abi, workload as W  # noqa: E402
from paper_2407_00023_b200.scheduler import GlobalScheduler  # noqa: E402

CASES = {
    "c1": (W.CONFIGS["c1"], None),
    "c2_3k": (W.CONFIGS["c2"], 3000),
    "c3_200": (W.CONFIGS["c3"], 200),
}


def main():
    ref = abi.load_library(abi.REF_SO)
    for name, (cfg, n) in CASES.items():
        trace = cfg.trace(lib=ref if cfg.archetype != "doc_qa" or not cfg.spec_overrides else None, n_requests=n)
        s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=ref)
        r = s.replay(trace, cfg.driver, want_costs=True, want_ratios=True)
        now = float(trace.arrivals[-1])
        nodes, toks, la, hits = s.export_arrays(now)
        st = s.stats()
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            decisions=r.decisions,
            costs=r.costs,
            ratios=r.ratios,
            stats=np.array([getattr(st, f.name) for f in dataclasses.fields(st)], dtype=np.int64),
            nodes=np.frombuffer(nodes, dtype=np.uint64).reshape(len(nodes), -1),
            edge_tokens=toks,
            last_access=la,
            hits=hits,
            n_requests=np.int64(trace.n),
            token_checksum=np.int64(int(trace.tokens.astype(np.int64).sum())),
        )
        print(name, trace.n, "decisions", st)


if __name__ == "__main__":
    main()
