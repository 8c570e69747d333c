#!/usr/bin/env python
"""bench.py — E2 global-scheduler hot path (Preble, arXiv 2407.00023) on B200.

Metric (BASELINE.json): scheduling decisions/s, with the prefix-match
kernel's algorithmic GB/s as a fraction of HBM peak.  A "step" is one full
replay of the config's synthetic trace (the generalised criterion-7 loop,
e2sched.h) from an empty scheduler.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

N > 1 (torchrun, one process per GPU): the serial commit does not shard, so
every rank runs an independent replica on its own GPU ("replicas only",
DESIGN.md); value = decisions of all ranks / max-over-ranks step time.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2407_00023_b200 import abi, replicas, workload  # noqa: E402
from paper_2407_00023_b200.scheduler import COST_DTYPE, DECISION_DTYPE, GlobalScheduler  # noqa: E402

METRIC = "scheduling decisions/sec (E2 placement replay)"
UNIT = "decisions/s"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = (
        "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": mx,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


dist_env = replicas.dist_env


def cpu_reference_replay(cfg, trace, repeats_s: float = 10.0, max_runs: int = 3):
    """The unmodified reference (oracle/_ref) on the host: decisions/s samples."""
    lib = abi.load_library(abi.REF_SO) if os.path.exists(abi.REF_SO) else abi.load_library(abi.ORACLE_SO)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
    rates = []
    t_total = 0.0
    while len(rates) < max_runs and (t_total < repeats_s or not rates):
        s._lib.e2_reset(s._h)
        t0 = time.perf_counter()
        r = s.replay(trace, cfg.driver, want_costs=False)
        dt = time.perf_counter() - t0
        assert r.n_done == trace.n
        rates.append(trace.n / dt)
        t_total += dt
    kind = "reference" if s.backend == "reference" else "port"
    return rates, kind


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = workload.CONFIGS[args.config]
    prod = abi.product_lib()
    trace = cfg.trace(lib=prod)
    lib = abi.load_library(abi.REF_SO) if os.path.exists(abi.REF_SO) else abi.load_library(abi.ORACLE_SO)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
    times = []
    for k in range(args.warmup + args.steps):
        s._lib.e2_reset(s._h)
        t0 = time.perf_counter()
        r = s.replay(trace, cfg.driver, want_costs=False)
        dt = time.perf_counter() - t0
        assert r.n_done == trace.n
        if k >= args.warmup:
            times.append(dt)
    ms = 1000.0 * statistics.mean(times)
    value = trace.n / (ms / 1000.0)
    kind = "reference" if s.backend == "reference" else "port"
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "i32 tokens / f64 costs",
        "data": "synthetic",
        "config": _config_dict(cfg, trace, args, ws),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": 1,
            "kind": kind,
            "sample": f"full {cfg.name} trace ({trace.n} requests) per step, single-threaded (the reference is serial)",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(cfg, trace, args, ws):
    return {
        "workload": cfg.name,
        "requests": trace.n,
        "instances": cfg.n_gpus,
        "prompt_tokens": int(len(trace.tokens)),
        "eviction": {0: "none", 1: "fifo_tail", 2: "mirror_lru"}[cfg.driver.eviction],
        "high_water": cfg.driver.high_water,
        "finish_lag": cfg.driver.finish_lag,
        "kv_capacity": cfg.sched.kv_capacity_tokens,
        "history_window_ms": cfg.sched.history_window_ms,
        "batch": args.batch,
        "parallelism": f"replicas{ws}" if ws > 1 else "single",
        "l2": "inputs larger than L2 (prompt arena > 126 MB), no flush",
    }


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = workload.CONFIGS[args.config]
    cfg.driver.batch = args.batch
    lib = abi.product_lib()
    trace = cfg.trace(lib=lib)
    n, G = trace.n, cfg.n_gpus

    # device-resident inputs / outputs (value) ---------------------------------
    t_tok = torch.from_numpy(np.ascontiguousarray(trace.tokens)).to(dev)
    t_off = torch.from_numpy(trace.offsets).to(dev)
    t_ids = torch.from_numpy(trace.ids).to(dev)
    t_arr = torch.from_numpy(trace.arrivals).to(dev)
    t_out = torch.from_numpy(trace.output_lens).to(dev)
    o_dec = torch.empty(n * DECISION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    o_cost = torch.empty(n * (G + 1) * COST_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sched = GlobalScheduler(G, cfg.sched, lib=lib)
    h = sched._h
    lib.e2_set_stream(h, ctypes.c_void_p(stream.cuda_stream))
    drv = cfg.driver.to_c()
    done = ctypes.c_int64()

    def step_device():
        rc = lib.e2_reset(h)
        assert rc == 0, lib.e2_last_error(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        rc = lib.e2_replay_device(
            h, t_tok.data_ptr(), t_off.data_ptr(), t_ids.data_ptr(), t_arr.data_ptr(), t_out.data_ptr(), n,
            ctypes.byref(drv), o_dec.data_ptr(), o_cost.data_ptr(), None, ctypes.c_void_p(stream.cuda_stream),
            ctypes.byref(done),
        )
        ev1.record(stream)
        assert rc == 0 and done.value == n, lib.e2_last_error(h)
        return ev0, ev1

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    lib.e2_profile_reset(h, 1)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            evs.append(step_device())
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = statistics.mean(step_ms)
    prof = abi.ProfileC()
    lib.e2_profile_get(h, ctypes.byref(prof))

    # correctness guard on the timed output: first decisions vs a host replay
    dec = np.frombuffer(o_dec.cpu().numpy().tobytes(), dtype=DECISION_DTYPE)

    # end to end through the C ABI with host (pinned) buffers ------------------
    pin = lambda a: torch.from_numpy(a).pin_memory()
    h_tok, h_off, h_ids, h_arr, h_out = map(pin, (np.ascontiguousarray(trace.tokens), trace.offsets, trace.ids,
                                                  trace.arrivals, trace.output_lens))
    h_dec = torch.empty(n * DECISION_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    h_cost = torch.empty(n * (G + 1) * COST_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    e2e_ms = []
    for k in range(max(1, min(args.steps, 3)) + 1):
        lib.e2_reset(h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.e2_replay(
            h, h_tok.data_ptr(), h_off.data_ptr(), h_ids.data_ptr(), h_arr.data_ptr(), h_out.data_ptr(), n,
            ctypes.byref(drv), h_dec.data_ptr(), h_cost.data_ptr(), None, ctypes.byref(done),
        )
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert rc == 0 and done.value == n, lib.e2_last_error(h)
        if k > 0:
            e2e_ms.append(1000 * dt)
    dec_e2e = np.frombuffer(h_dec.numpy().tobytes(), dtype=DECISION_DTYPE)
    assert np.array_equal(dec, dec_e2e), "device-resident and host-buffer replays disagree"

    # max over ranks
    ms, e2e_max = replicas.max_over_ranks([ms, statistics.mean(e2e_ms)], device=dev)
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    value = replicas.job_throughput(ws, n, ms)
    e2e_value = replicas.job_throughput(ws, n, e2e_max)
    peak, peak_kind = _peaks()
    steps = args.steps
    match_ms = prof.ms[abi.E2_K_MATCH] / max(1, prof.launches[abi.E2_K_MATCH])
    match_bytes = prof.match_bytes / max(1, prof.launches[abi.E2_K_MATCH])
    achieved = (match_bytes / 1e9) / (match_ms / 1e3) if match_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(REPO, "profiles", "match_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                per_req = json.load(f).get("dram_bytes_per_request")
            # same per-launch normalisation as `achieved`
            traffic = per_req * prof.match_requests / max(1, prof.launches[abi.E2_K_MATCH])
        except Exception:
            traffic = None
    total_kernel_ms = sum(prof.ms)
    shares = {
        nm: (prof.ms[i] / total_kernel_ms if total_kernel_ms else None)
        for i, nm in enumerate(["match_k1", "group_rounds", "serial_commit", "other"])
    }
    h2d = int(trace.nbytes)
    d2h = int(n * DECISION_DTYPE.itemsize + n * (G + 1) * COST_DTYPE.itemsize)
    cpu_rates, cpu_kind = cpu_reference_replay(cfg, trace)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "i32 tokens / f64 costs",
        "data": "synthetic",
        "config": _config_dict(cfg, trace, args, ws),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": {
            "kernel": "k_match (K1 batched prefix match)",
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved / peak if peak else None,
            "traffic": traffic,
            "algorithmic_bytes_per_launch": match_bytes,
            "avg_launch_ms": match_ms,
        },
        "kernel_share": shares,
        "kernel_ms_per_step": {nm: prof.ms[i] / steps for i, nm in enumerate(["match_k1", "group_rounds", "serial_commit", "other"])},
        "gpu_launches": int(sum(prof.launches)),
        "clocks": clk.summary(),
        "cpu_baseline": {
            "value": statistics.median(cpu_rates),
            "unit": UNIT,
            "cores": 1,
            "kind": cpu_kind,
            "sample": f"full {cfg.name} trace ({n} requests) x {len(cpu_rates)} runs on the host, single-threaded reference",
        },
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
