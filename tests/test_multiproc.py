"""N>1 path of the bench (replicas only) with the gloo backend
at world size 2 on CPU: each rank replays its own copy of a trace on its own
engine instance; replicas agree bit-for-bit and the job throughput uses the
max-over-ranks step time."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, lib_path, out_dir):
    import time

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2407_00023_b200 import abi, replicas, workload
    from paper_2407_00023_b200.scheduler import GlobalScheduler

    lib = abi.load_library(lib_path)
    cfg = workload.CONFIGS["c1"]
    trace = cfg.trace(lib=lib, n_requests=600)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
    dist.barrier()
    t0 = time.perf_counter()
    r = s.replay(trace, cfg.driver)
    ms = 1000 * (time.perf_counter() - t0) + rank  # ranks differ: max must win
    (ms_max,) = replicas.max_over_ranks([ms])
    assert abs(ms_max - max(ms, ms_max)) < 1e-9
    np.save(os.path.join(out_dir, f"dec{rank}.npy"), r.decisions)
    np.save(os.path.join(out_dir, f"ms{rank}.npy"), np.array([ms, ms_max]))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo(tmp_path, hostsim_lib):
    from conftest import HOSTSIM_SO

    mp.spawn(_worker, args=(2, _free_port(), HOSTSIM_SO, str(tmp_path)), nprocs=2, join=True)
    d0, d1 = np.load(tmp_path / "dec0.npy"), np.load(tmp_path / "dec1.npy")
    assert np.array_equal(d0, d1)
    m0, m1 = np.load(tmp_path / "ms0.npy"), np.load(tmp_path / "ms1.npy")
    assert m0[1] == m1[1] == max(m0[0], m1[0])
    from paper_2407_00023_b200.replicas import job_throughput

    assert job_throughput(2, 600, m0[1]) == pytest.approx(2 * 600 / (m0[1] / 1000))
