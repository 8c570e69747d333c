"""SURVEY 8(e) sharded replay at world size 2 with the gloo backend on CPU
(the host emulation of the product engine stands in for the B200).

Each batch: both ranks run K1 on their half, the summaries are all-gathered,
rank 0 commits and broadcasts the state delta, rank 1 applies it.  Checked:
after EVERY batch rank 1's replicated state (digest of every region and the
hot counters) equals rank 0's; the decisions equal a plain single-process
replay of the same trace; the final tree exports are identical."""
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


def _worker(rank, ws, port, lib_path, out_dir, cfg_name, n_req, batch, device="cpu"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2407_00023_b200 import abi, sharded, workload
    from paper_2407_00023_b200.scheduler import DriverConfig, GlobalScheduler

    lib = abi.load_library(lib_path)
    cfg = workload.CONFIGS[cfg_name]
    trace = cfg.trace(lib=lib, n_requests=n_req)
    drv = DriverConfig(**{**cfg.driver.__dict__, "batch": batch})
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    dev = torch.device(device)
    if dev.type == "cuda":
        torch.cuda.set_device(dev)
        st = torch.cuda.Stream(dev)
        torch.cuda.set_stream(st)
        lib.e2_set_stream(s._h, st.cuda_stream)
    rep = sharded.ShardedReplay(s, sharded.trace_tensors(trace, dev), drv, dev, rank, ws)
    digests = []

    def on_batch(b0, nb):
        d = torch.from_numpy(s.state_digest().view(np.int64).copy())
        allv = [torch.zeros_like(d) for _ in range(ws)]
        dist.all_gather(allv, d)
        digests.append([a.numpy().copy() for a in allv])

    done = rep.run(on_batch)
    assert done == trace.n
    for k, per_rank in enumerate(digests):
        for r in range(1, ws):
            assert np.array_equal(per_rank[0], per_rank[r]), f"batch {k}: rank {r} diverged from rank 0"
    nodes, toks, la, hits = s.export_arrays(float(trace.arrivals[-1]) + 1.0)
    np.save(os.path.join(out_dir, f"nodes{rank}.npy"), np.frombuffer(bytes(nodes), dtype=np.uint8))
    np.save(os.path.join(out_dir, f"la{rank}.npy"), la)
    np.save(os.path.join(out_dir, f"hits{rank}.npy"), hits)
    np.save(os.path.join(out_dir, f"nb{rank}.npy"), np.array([len(digests), rep.delta_bytes]))
    if rank == 0:
        np.save(os.path.join(out_dir, "dec.npy"), rep.decisions())
        np.save(os.path.join(out_dir, "cost.npy"), rep.costs())
    s.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name,n_req,batch", [("c1", 700, 256), ("c4", 3000, 1024), ("c3", 240, 64)])
def test_sharded_replay_two_ranks_gloo(tmp_path, hostsim_lib, cfg_name, n_req, batch):
    from conftest import HOSTSIM_SO
    from paper_2407_00023_b200 import workload
    from paper_2407_00023_b200.scheduler import DriverConfig, GlobalScheduler

    mp.spawn(_worker, args=(2, _free_port(), HOSTSIM_SO, str(tmp_path), cfg_name, n_req, batch), nprocs=2, join=True)
    nb0, nb1 = np.load(tmp_path / "nb0.npy"), np.load(tmp_path / "nb1.npy")
    assert nb0[0] == nb1[0] >= 2, "the replay must span several batches"
    assert nb0[1] > 0
    for f in ("nodes", "la", "hits"):
        assert np.array_equal(np.load(tmp_path / f"{f}0.npy"), np.load(tmp_path / f"{f}1.npy")), f
    # decisions equal the unsharded replay of the same trace on one engine
    cfg = workload.CONFIGS[cfg_name]
    trace = cfg.trace(lib=hostsim_lib, n_requests=n_req)
    drv = DriverConfig(**{**cfg.driver.__dict__, "batch": batch})
    ref = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=hostsim_lib).replay(trace, drv)
    dec = np.load(tmp_path / "dec.npy")
    assert np.array_equal(dec, ref.decisions)
    assert np.array_equal(np.load(tmp_path / "cost.npy").view(np.uint8), ref.costs.view(np.uint8))


def test_max_over_ranks_single_process():
    from paper_2407_00023_b200.sharded import max_over_ranks

    assert max_over_ranks([1.5, 2.0]) == [1.5, 2.0]


@pytest.mark.gpu
def test_sharded_replay_two_ranks_b200():
    """The device path of the sharded replay (K1 slices, summary pack/unpack,
    delta diff/apply kernels) with two ranks sharing cuda:0; gloo moves the
    CUDA tensors (NCCL needs one GPU per rank).  Same checks as on CPU."""
    import tempfile
    from pathlib import Path

    from paper_2407_00023_b200 import abi, workload
    from paper_2407_00023_b200.scheduler import DriverConfig, GlobalScheduler

    lib = abi.product_lib()
    with tempfile.TemporaryDirectory() as d:
        tmp = Path(d)
        n_req, batch = 40000, 4096
        mp.spawn(_worker, args=(2, _free_port(), abi.PRODUCT_SO, d, "c4", n_req, batch, "cuda:0"), nprocs=2,
                 join=True)
        for f in ("nodes", "la", "hits"):
            assert np.array_equal(np.load(tmp / f"{f}0.npy"), np.load(tmp / f"{f}1.npy")), f
        cfg = workload.CONFIGS["c4"]
        trace = cfg.trace(lib=lib, n_requests=n_req)
        drv = DriverConfig(**{**cfg.driver.__dict__, "batch": batch})
        ref = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib).replay(trace, drv)
        assert np.array_equal(np.load(tmp / "dec.npy"), ref.decisions)
