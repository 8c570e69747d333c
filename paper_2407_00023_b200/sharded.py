"""Multi-GPU replay: tree replicated, K1 sharded, commit on rank 0.

One process per GPU (torchrun).  Every rank holds the whole trace and a
replica of the scheduler state in its own HBM.  Per batch of the replay
(the same batch schedule as ``e2_replay``):

1. every rank runs K1 (the read-only prefix match, ``prefix_tree.cpp:79-120``)
   on its contiguous slice of the batch and packs the per-request summaries
   (snapshot match length, divergence point, path hints);
2. the slices are all-gathered (NCCL over NVLink; gloo on CPU in the tests);
3. rank 0 runs the leader rounds and the serial decide/commit pass
   (``global_scheduler.cpp:76-192``) and diffs its state against what the
   replicas hold: 64-byte chunks of the node pool, child table, LRU pages,
   windows and inflight map that changed, plus the hot counters;
4. rank 0 broadcasts the delta; the replicas scatter it, after which every
   replica equals rank 0 byte for byte and can match the next batch.

The commit is serial by construction (every decision reads the state left by
all earlier ones), so decisions/s of ONE trace is the metric at every N.
The C-ABI steps are ``e2_shard_*`` (include/e2sched.h); this module only
moves their buffers through ``torch.distributed``.
"""
from __future__ import annotations

import ctypes
import json
import os
import statistics
import time

import numpy as np

from . import abi
from .scheduler import COST_DTYPE, DECISION_DTYPE, DriverConfig, GlobalScheduler


def dist_env():
    return (
        int(os.environ.get("WORLD_SIZE", "1")),
        int(os.environ.get("RANK", "0")),
        int(os.environ.get("LOCAL_RANK", "0")),
    )


def max_over_ranks(values, device=None):
    """Element-wise max of per-rank floats (barrier semantics of all_reduce)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


class _Buf:
    """A growable byte tensor on the replay's device."""

    def __init__(self, device):
        import torch

        self.torch, self.device, self.t = torch, device, None

    def get(self, nbytes: int):
        if self.t is None or self.t.numel() < nbytes:
            cap = max(int(nbytes * 1.25) + 64, 1 << 16)
            self.t = self.torch.empty(cap, dtype=self.torch.uint8, device=self.device)
        return self.t[:nbytes]


class ShardedReplay:
    """Drives one sharded replay of a resident trace through ``e2_shard_*``."""

    def __init__(self, sched: GlobalScheduler, tensors, driver: DriverConfig, device, rank: int, world: int,
                 want_costs: bool = True):
        import torch

        self.torch, self.s, self.lib, self.h = torch, sched, sched._lib, sched._h
        self.tok, self.off, self.ids, self.arr, self.outl = tensors
        self.n = int(self.ids.numel())
        self.G = sched.n_gpus()
        self.drv = driver.to_c()
        self.device, self.rank, self.world = device, rank, world
        self.dec = self.cost = None
        if rank == 0:
            self.dec = torch.empty(self.n * DECISION_DTYPE.itemsize, dtype=torch.uint8, device=device)
            if want_costs:
                self.cost = torch.zeros(self.n * (self.G + 1) * COST_DTYPE.itemsize, dtype=torch.uint8,
                                        device=device)
        self.send, self.recv, self.delta = _Buf(device), _Buf(device), _Buf(device)
        self.meta = torch.zeros(2, dtype=torch.int64, device=device)
        self.batches = 0
        self.delta_bytes = 0

    def _check(self, rc):
        if rc != abi.E2_OK:
            raise RuntimeError(self.lib.e2_last_error(self.h).decode())

    def _settle(self):
        """Collectives complete on the device asynchronously; the library's
        next step reads their output on its own stream: wait for them."""
        if self.torch.device(self.device).type == "cuda":
            self.torch.cuda.current_stream(self.device).synchronize()

    def _all_gather(self, send, nbytes):
        import torch.distributed as dist

        recv = self.recv.get(nbytes * self.world)
        if self.world == 1:
            recv.copy_(send)
            return recv
        if send.is_cuda and dist.get_backend() == "gloo":
            # gloo has no CUDA all-gather (tests sharing one GPU): stage on the host
            host = send.cpu()
            parts = [self.torch.empty_like(host) for _ in range(self.world)]
            dist.all_gather(parts, host)
            recv.copy_(self.torch.cat(parts))
            return recv
        parts = [recv[k * nbytes:(k + 1) * nbytes] for k in range(self.world)]
        dist.all_gather(parts, send)
        return recv

    def run(self, on_batch=None) -> int:
        """The whole replay; returns the number of requests decided.
        ``on_batch(b0, nb)`` runs on every rank after each batch's delta."""
        import torch.distributed as dist

        lib, h, rank, world = self.lib, self.h, self.rank, self.world
        p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
        self._check(lib.e2_shard_begin(h, p(self.tok), p(self.off), p(self.ids), p(self.arr), p(self.outl), self.n,
                                       ctypes.byref(self.drv), p(self.dec), p(self.cost), None, rank, world))
        b0, nb, rb, db = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        failed = None
        while True:
            self._check(lib.e2_shard_next(h, ctypes.byref(b0), ctypes.byref(nb), ctypes.byref(rb)))
            if nb.value == 0:
                break
            per = -(-nb.value // world)
            lo = rank * per
            cnt = max(0, min(per, nb.value - lo))
            slice_bytes = 16 + per * rb.value
            send = self.send.get(slice_bytes)
            self._check(lib.e2_shard_match(h, lo, cnt, p(send)))
            recv = self._all_gather(send, slice_bytes)
            self._settle()
            if rank == 0:
                rc = lib.e2_shard_commit(h, p(recv), per, ctypes.byref(db))
                if rc != abi.E2_OK:
                    failed = lib.e2_last_error(h).decode()
                    self.meta[0], self.meta[1] = -1, rc
                else:
                    self.meta[0], self.meta[1] = db.value, 0
            if world > 1:
                dist.broadcast(self.meta, 0)
            size = int(self.meta[0].item())
            if size < 0:
                raise RuntimeError(failed or f"rank 0 failed to commit a batch (code {int(self.meta[1])})")
            delta = self.delta.get(size)
            if rank == 0:
                self._check(lib.e2_shard_delta_copy(h, p(delta)))
            if world > 1:
                dist.broadcast(delta, 0)
                self._settle()
            if rank != 0:
                self._check(lib.e2_shard_apply(h, p(delta), size))
            self.batches += 1
            self.delta_bytes += size
            if on_batch is not None:
                on_batch(b0.value, nb.value)
        done = ctypes.c_int64()
        rc = lib.e2_shard_end(h, ctypes.byref(done))
        if rc != abi.E2_OK:
            err = RuntimeError(lib.e2_last_error(h).decode())
            err.n_done = done.value
            raise err
        return done.value

    def decisions(self) -> np.ndarray:
        return np.frombuffer(self.dec.cpu().numpy().tobytes(), dtype=DECISION_DTYPE)

    def costs(self) -> np.ndarray:
        return np.frombuffer(self.cost.cpu().numpy().tobytes(), dtype=COST_DTYPE).reshape(self.n, self.G + 1)


def trace_tensors(trace, device):
    import torch

    return tuple(torch.from_numpy(np.ascontiguousarray(a)).to(device)
                 for a in (trace.tokens, trace.offsets, trace.ids, trace.arrivals, trace.output_lens))


# --------------------------------------------------------------------------
# bench.py --gpus N (N > 1)
# --------------------------------------------------------------------------
def bench_main(args, metric, unit, config_dict, clock_sampler):
    """One sharded replay of the config's trace per step on every rank.
    value = decisions of the trace / max-over-ranks step time (CUDA events)."""
    import torch
    import torch.distributed as dist

    from . import workload

    ws, rank, local = dist_env()
    if getattr(args, "same_device", False):
        local = 0  # dev check of the N>1 path on a one-GPU box (with --dist-backend gloo)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = getattr(args, "dist_backend", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    cfg = workload.CONFIGS[args.config]
    lib = abi.product_lib()
    trace = cfg.trace(lib=lib)
    n, G = trace.n, cfg.n_gpus
    drv = DriverConfig(**{**cfg.driver.__dict__, "batch": args.batch or cfg.driver.batch or 16384})
    sched = GlobalScheduler(G, cfg.sched, policy=cfg.policy, lib=lib)
    stream = torch.cuda.Stream(dev)  # the library and the timing events share it
    torch.cuda.set_stream(stream)     # the collectives order against it too
    lib.e2_set_stream(sched._h, ctypes.c_void_p(stream.cuda_stream))
    tens = trace_tensors(trace, dev)
    rep = ShardedReplay(sched, tens, drv, dev, rank, ws, want_costs=True)

    def step():
        assert lib.e2_reset(sched._h) == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = rep.run()
        e1.record(stream)
        assert done == n, (done, n)
        return e0, e1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib.e2_profile_reset(sched._h, 1)
    dist.barrier()
    torch.cuda.synchronize()
    with clock_sampler(local) as clk:
        evs = [step() for _ in range(args.steps)]
        torch.cuda.synchronize()
    dist.barrier()
    ms_local = statistics.mean(a.elapsed_time(b) for a, b in evs)
    prof = abi.ProfileC()
    lib.e2_profile_get(sched._h, ctypes.byref(prof))
    launches_local = int(sum(prof.launches))
    ms_max, launches_max = max_over_ranks([ms_local, float(launches_local)], dev)

    # e2e: pinned host trace -> every rank's HBM, decisions back to rank 0's host
    pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
           for a in (trace.tokens, trace.offsets, trace.ids, trace.arrivals, trace.output_lens)]
    h_dec = torch.empty(rep.dec.numel() if rank == 0 else 1, dtype=torch.uint8).pin_memory()
    e2e_ms = []
    for k in range(2):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for dst, src in zip(tens, pin):
            dst.copy_(src, non_blocking=True)
        step()
        if rank == 0:
            h_dec.copy_(rep.dec, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if k > 0:
            e2e_ms.append(1000 * dt)
    (e2e_max,) = max_over_ranks([statistics.mean(e2e_ms)], dev)
    ok = True
    if rank == 0:
        # the sharded decisions equal the single-GPU replay's (same library, same trace)
        single = GlobalScheduler(G, cfg.sched, policy=cfg.policy, lib=lib)
        r = single.replay(trace.head(min(n, 200000)), drv, want_costs=False)
        dec = rep.decisions()
        ok = bool(np.array_equal(dec[:r.n_done], r.decisions[:r.n_done]))
        single.close()
    nodes = sched.node_count()
    if rank == 0:
        value = n / (ms_max / 1000.0)
        line = {
            "metric": metric,
            "value": value,
            "unit": unit,
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "i32 tokens / f64 costs",
            "data": "synthetic",
            "config": dict(config_dict(cfg, n, args, ws), prompt_tokens=int(len(trace.tokens)), tree_nodes=nodes),
            "e2e": {"value": n / (e2e_max / 1000.0), "unit": unit,
                    "h2d_bytes_per_step": int(trace.nbytes) * ws,
                    "d2h_bytes_per_step": int(n * DECISION_DTYPE.itemsize)},
            "sharding": {
                "batches_per_step": rep.batches // max(1, args.steps + args.warmup + 2),
                "delta_bytes_per_step": prof.delta_bytes / max(1, args.steps),
                "delta_chunks_per_step": prof.delta_chunks / max(1, args.steps),
                "decisions_equal_single_gpu_replay": ok,
            },
            "kernel_ms_per_step_rank0": {nm: prof.ms[i] / args.steps
                                         for i, nm in enumerate(["match_k1", "group_rounds", "serial_commit", "other"])},
            "gpu_launches": int(launches_max),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    sched.close()
    dist.destroy_process_group()
    return 0
