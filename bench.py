#!/usr/bin/env python
"""bench.py — E2 global-scheduler hot path (Preble, arXiv 2407.00023) on B200.

Metric (BASELINE.json): scheduling decisions/s, with the prefix-match
kernel's algorithmic GB/s as a fraction of HBM peak.  A "step" is one full
replay of the config's synthetic trace (the generalised criterion-7 loop,
e2sched.h) from an empty scheduler.  The headline workload is config C4
(`configs[3]`: tree-of-thought, 1M requests, the largest single-GPU config;
C5 is the one BASELINE.json shards across 8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

N > 1 (torchrun, one process per GPU): the SURVEY 8(e) sharded replay
(`sharded.py`): the tree is replicated on every rank, each rank matches its
slice of every batch (K1), the summaries are all-gathered over NCCL, rank 0
commits the batch and broadcasts the state delta, the other ranks apply it.
Every rank processes the same trace, so value = decisions of ONE trace /
max-over-ranks step time.

--impl reference: the unmodified reference (oracle/_ref/libe2ref.so, built
from /root/reference/proj/src by oracle/Makefile; the trace comes from the
same library) timed on the host on a bounded prefix of the same workload.
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

from paper_2407_00023_b200 import abi, workload  # noqa: E402
from paper_2407_00023_b200.scheduler import COST_DTYPE, DECISION_DTYPE, DriverConfig, GlobalScheduler  # noqa: E402

METRIC = "scheduling decisions/sec (E2 placement replay)"
UNIT = "decisions/s"
KNAMES = ["match_k1", "group_rounds", "serial_commit", "other"]


def dist_env():
    return (
        int(os.environ.get("WORLD_SIZE", "1")),
        int(os.environ.get("RANK", "0")),
        int(os.environ.get("LOCAL_RANK", "0")),
    )


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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


# --------------------------------------------------------------------------
# the reference on the host (oracle/_ref: unmodified reference sources)
# --------------------------------------------------------------------------
def _ref_lib():
    if not os.path.exists(abi.REF_SO):
        raise RuntimeError(f"{abi.REF_SO} missing: build it here with `make -C oracle ref` (needs /root/reference)")
    lib = abi.load_library(abi.REF_SO)
    lib.e2ref_time_loop.restype = ctypes.c_int
    lib.e2ref_time_loop.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                             ctypes.c_void_p]
    return lib


def time_reference(lib, cfg, trace, driver) -> float:
    """One run of the reference's criterion-7 loop (acceptance_main.cpp:367-416)
    over `trace` from a fresh scheduler; seconds of the scheduling loop alone
    (steady_clock inside the library, requests pre-built as the reference does)."""
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    sec, done = ctypes.c_double(), ctypes.c_int64()
    rc = lib.e2ref_time_loop(s._h, p(trace.tokens), p(trace.offsets), p(trace.ids), p(trace.arrivals),
                             p(trace.output_lens), trace.n, ctypes.byref(driver.to_c()), ctypes.byref(sec),
                             ctypes.byref(done))
    assert rc == 0 and done.value == trace.n, lib.e2_last_error(s._h)
    s.close()
    return sec.value


def _sample_desc(cfg, n_sample, n_full, runs, cores):
    part = f"first {n_sample} of the {n_full} requests" if n_sample < n_full else f"all {n_full} requests"
    return (f"{part} of {cfg.name} per run ({runs} runs); the reference's criterion-7 loop, "
            f"single-threaded (the reference is serial): 1 thread of {cores} host cores")


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0  # rank 0 alone times the host reference
    cfg = workload.CONFIGS[args.config]
    lib = _ref_lib()  # the only native library this process maps
    n_sample = ref_sample_size(args, cfg)
    trace = cfg.trace(lib=lib, n_requests=n_sample)
    drv = cfg.driver
    times = []
    for k in range(args.warmup + args.steps):
        dt = time_reference(lib, cfg, trace, drv)
        if k >= args.warmup:
            times.append(dt)
    sec = statistics.mean(times)
    value = trace.n / sec
    cores = _host_cores()
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * sec,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "i32 tokens / f64 costs",
        "data": "synthetic",
        "config": dict(_config_dict(cfg, cfg.n_requests, args, ws), reference_sample_requests=trace.n),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": 1,
            "host_cores": cores,
            "kind": "reference",
            "sample": _sample_desc(cfg, trace.n, cfg.n_requests, args.steps, cores),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def ref_sample_size(args, cfg) -> int:
    """Requests of the trace one reference step replays.  Default: the whole
    config when the run has at most 8 steps in all (C4: ~22 s per step), else
    a 300k-request prefix so the arm stays within a few minutes."""
    if args.ref_sample > 0:
        return min(args.ref_sample, cfg.n_requests)
    if args.ref_sample == 0 or args.steps + args.warmup <= 8:
        return cfg.n_requests
    return min(300000, cfg.n_requests)


def eff_batch(args, cfg) -> int:
    return args.batch or cfg.driver.batch or 16384


def _config_dict(cfg, n, args, ws):
    return {
        "workload": cfg.name,
        "requests": n,
        "instances": cfg.n_gpus,
        "archetype": cfg.archetype,
        "eviction": {0: "none", 1: "fifo_tail", 2: "mirror_lru"}[cfg.driver.eviction],
        "high_water": cfg.driver.high_water,
        "finish_lag": cfg.driver.finish_lag,
        "kv_capacity": cfg.sched.kv_capacity_tokens,
        "history_window_ms": cfg.sched.history_window_ms,
        "batch": eff_batch(args, cfg),
        "parallelism": f"sharded{ws} (K1 sharded, commit on rank 0, NCCL delta broadcast)" if ws > 1 else "single",
        "l2": "inputs larger than L2 (prompt arena > 126 MB), no flush",
    }


# --------------------------------------------------------------------------
# traffic: ncu DRAM bytes of the bench's own kernels, measured in this run
# --------------------------------------------------------------------------
def _under_profiler() -> bool:
    return any(k in os.environ for k in ("NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NSIGHT_COMPUTE_INJECTION",
                                         "CUDA_INJECTION64_PATH"))


def measure_traffic(args, cfg, timeout=420):
    """Run this script's --probe mode (one replay of a prefix of the same
    trace) under ncu with DRAM byte counters on k_serial and k_match; returns
    per-kernel bytes per request of the full-size batches, or None."""
    if args.no_traffic or _under_profiler():
        return None
    ncu = "ncu"
    skip = 4  # the ramp batches (2048, 4096, 8192) and the first full one: one k_match + one k_serial each
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:k_serial|k_match", "--launch-skip", str(2 * skip),
           "--launch-count", "4", "--csv", sys.executable, os.path.abspath(__file__), "--probe",
           "--config", args.config, "--probe-n", str(args.probe_n), "--batch", str(eff_batch(args, cfg))]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except Exception:
        return None
    rows = {}
    import csv
    import io

    lines = [ln for ln in out.stdout.splitlines() if ln.startswith('"')]
    if not lines:
        return None
    rd = csv.DictReader(io.StringIO("\n".join(lines)))
    for r in rd:
        nm = r.get("Kernel Name", "")
        k = "k_serial" if "k_serial" in nm else "k_match" if "k_match" in nm else None
        if k is None:
            continue
        lid = r.get("ID")
        v = float(str(r.get("Metric Value", "0")).replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1}.get(unit, 1)
        rows.setdefault((k, lid), {})[r.get("Metric Name")] = v * scale
    res = {}
    for (k, _), m in rows.items():
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        res.setdefault(k, []).append((b, m.get("gpu__time_duration.sum")))
    if not res:
        return None
    # the probe's full-size batches hold args.batch requests per launch
    return {k: {"dram_bytes_per_launch": statistics.mean(b for b, _ in v), "requests_per_launch": eff_batch(args, cfg),
                "ncu_launch_s": statistics.mean(t for _, t in v if t), "launches": len(v)} for k, v in res.items()}


def run_probe(args):
    """--probe: one device replay of a trace prefix (the ncu traffic pass)."""
    cfg = workload.CONFIGS[args.config]
    lib = abi.product_lib()
    trace = cfg.trace(lib=lib, n_requests=args.probe_n)
    drv = cfg.driver
    drv.batch = eff_batch(args, cfg)
    s = GlobalScheduler(cfg.n_gpus, cfg.sched, policy=cfg.policy, lib=lib)
    r = s.replay(trace, drv, want_costs=False)
    assert r.n_done == trace.n
    return 0


# --------------------------------------------------------------------------
# the product on the B200
# --------------------------------------------------------------------------
class DeviceReplay:
    """One config's trace resident in HBM + a product scheduler bound to the
    current torch stream."""

    def __init__(self, cfg, trace, dev, batch):
        import torch

        self.torch = torch
        self.cfg, self.trace, self.dev = cfg, trace, dev
        self.lib = abi.product_lib()
        self.n, self.G = trace.n, cfg.n_gpus
        self.drv = DriverConfig(**{**cfg.driver.__dict__, "batch": batch}).to_c()
        self.t_tok = torch.from_numpy(np.ascontiguousarray(trace.tokens)).to(dev)
        self.t_off = torch.from_numpy(trace.offsets).to(dev)
        self.t_ids = torch.from_numpy(trace.ids).to(dev)
        self.t_arr = torch.from_numpy(trace.arrivals).to(dev)
        self.t_out = torch.from_numpy(trace.output_lens).to(dev)
        self.o_dec = torch.empty(self.n * DECISION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.o_cost = torch.empty(self.n * (self.G + 1) * COST_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        # a dedicated stream: the library's launches and the timing events
        # share it (the legacy default stream would leave the library on its
        # own non-blocking stream)
        self.stream = torch.cuda.Stream(dev)
        self.sched = GlobalScheduler(self.G, cfg.sched, policy=cfg.policy, lib=self.lib)
        self.h = self.sched._h
        self.lib.e2_set_stream(self.h, ctypes.c_void_p(self.stream.cuda_stream))
        self.done = ctypes.c_int64()

    def step(self):
        """Reset + one full replay; returns the CUDA events bracketing it."""
        lib, h, torch = self.lib, self.h, self.torch
        rc = lib.e2_reset(h)
        assert rc == 0, lib.e2_last_error(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(self.stream)
        rc = lib.e2_replay_device(
            h, self.t_tok.data_ptr(), self.t_off.data_ptr(), self.t_ids.data_ptr(), self.t_arr.data_ptr(),
            self.t_out.data_ptr(), self.n, ctypes.byref(self.drv), self.o_dec.data_ptr(), self.o_cost.data_ptr(),
            None, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(self.done),
        )
        ev1.record(self.stream)
        assert rc == 0 and self.done.value == self.n, lib.e2_last_error(h)
        return ev0, ev1

    def decisions(self):
        return np.frombuffer(self.o_dec.cpu().numpy().tobytes(), dtype=DECISION_DTYPE)

    def e2e(self, runs):
        """Through the public C ABI with pinned HOST buffers: H2D of the trace
        and D2H of decisions + costs inside the timed region."""
        torch, lib, h, tr = self.torch, self.lib, self.h, self.trace
        pin = lambda a: torch.from_numpy(a).pin_memory()
        h_tok, h_off, h_ids, h_arr, h_out = map(pin, (np.ascontiguousarray(tr.tokens), tr.offsets, tr.ids,
                                                      tr.arrivals, tr.output_lens))
        h_dec = torch.empty(self.n * DECISION_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
        h_cost = torch.empty(self.n * (self.G + 1) * COST_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
        ms = []
        for k in range(runs):  # the device path is warm (timed steps ran first)
            lib.e2_reset(h)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = lib.e2_replay(
                h, h_tok.data_ptr(), h_off.data_ptr(), h_ids.data_ptr(), h_arr.data_ptr(), h_out.data_ptr(), self.n,
                ctypes.byref(self.drv), h_dec.data_ptr(), h_cost.data_ptr(), None, ctypes.byref(self.done),
            )
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert rc == 0 and self.done.value == self.n, lib.e2_last_error(h)
            ms.append(1000 * dt)
        dec = np.frombuffer(h_dec.numpy().tobytes(), dtype=DECISION_DTYPE)
        h2d = int(tr.nbytes)
        d2h = int(self.n * DECISION_DTYPE.itemsize + self.n * (self.G + 1) * COST_DTYPE.itemsize)
        return statistics.mean(ms), dec, h2d, d2h

    def close(self):
        self.sched.close()


def _timed_steps(rep, steps, warmup, barrier=None):
    torch = rep.torch
    for _ in range(warmup):
        rep.step()
    torch.cuda.synchronize()
    rep.lib.e2_profile_reset(rep.h, 1)
    if barrier:
        barrier()
    torch.cuda.synchronize()
    evs = [rep.step() for _ in range(steps)]
    torch.cuda.synchronize()
    if barrier:
        barrier()
    ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    prof = abi.ProfileC()
    rep.lib.e2_profile_get(rep.h, ctypes.byref(prof))
    return ms, prof


def secondary_lines(args, dev):
    """C2 under both eviction drivers: the product (device-resident value)
    beside the reference on the same full trace."""
    out = []
    ref = _ref_lib() if os.path.exists(abi.REF_SO) else None
    base = workload.CONFIGS["c2"]
    for label, drv in (("mirror_lru", base.driver),
                       ("fifo_tail", DriverConfig(eviction=abi.E2_EVICT_FIFO_TAIL, trunk_len=1860, high_water=150000,
                                                  finish_lag=2000))):
        cfg = workload.Config(base.name, base.archetype, base.n_requests, base.n_gpus, base.sched, drv)
        trace = cfg.trace()
        rep = DeviceReplay(cfg, trace, dev, eff_batch(args, cfg))
        ms, _ = _timed_steps(rep, 3, 2)
        rep.close()
        line = {"workload": cfg.name, "eviction": label, "requests": trace.n, "value": trace.n / (ms / 1000.0),
                "unit": UNIT}
        if ref is not None:
            t = time_reference(ref, cfg, trace, drv)
            line["reference_value"] = trace.n / t
            line["reference_sample"] = f"all {trace.n} requests, 1 run, 1 thread"
        out.append(line)
    return out


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        from paper_2407_00023_b200 import sharded

        return sharded.bench_main(args, METRIC, UNIT, _config_dict, ClockSampler)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = workload.CONFIGS[args.config]
    lib = abi.product_lib()
    trace = cfg.trace(lib=lib)
    n, G = trace.n, cfg.n_gpus
    rep = DeviceReplay(cfg, trace, dev, eff_batch(args, cfg))

    with ClockSampler(local) as clk:
        ms, prof = _timed_steps(rep, args.steps, args.warmup)
    dec = rep.decisions()
    e2e_ms, dec_e2e, h2d, d2h = rep.e2e(max(1, min(args.steps, 2)))
    assert np.array_equal(dec, dec_e2e), "device-resident and host-buffer replays disagree"
    nodes = rep.sched.node_count()
    rep.close()
    value = n / (ms / 1000.0)
    e2e_value = n / (e2e_ms / 1000.0)

    # correctness guard on the timed output: the decisions of the reference's
    # sample prefix must equal the reference's own (bit-exact placement)
    peak, peak_kind = _peaks()
    steps = args.steps
    L = prof.launches
    kms = [prof.ms[i] / steps for i in range(4)]
    total_kernel_ms = sum(prof.ms)
    shares = {nm: (prof.ms[i] / total_kernel_ms if total_kernel_ms else None) for i, nm in enumerate(KNAMES)}
    # algorithmic bytes: B_match from K1's per-request counter,
    # B_cost = 24 B per (request, evaluated instance)
    match_bytes_step = prof.match_bytes / steps
    n_costs = int(dec["n_costs"].astype(np.int64).sum())
    cost_bytes_step = 24 * n_costs
    ser_launch_ms = prof.ms[abi.E2_K_COMMIT] / max(1, L[abi.E2_K_COMMIT])
    ser_launches_step = L[abi.E2_K_COMMIT] / steps
    ser_bytes_launch = (match_bytes_step + cost_bytes_step) / ser_launches_step
    match_ms = prof.ms[abi.E2_K_MATCH] / max(1, L[abi.E2_K_MATCH])
    match_launches_step = L[abi.E2_K_MATCH] / steps
    match_bytes_launch = match_bytes_step / match_launches_step
    k1_achieved = (match_bytes_launch / 1e9) / (match_ms / 1e3) if match_ms > 0 else 0.0
    ser_achieved = (ser_bytes_launch / 1e9) / (ser_launch_ms / 1e3) if ser_launch_ms > 0 else 0.0
    traffic = measure_traffic(args, cfg) if rank == 0 else None
    req_per_launch = n / ser_launches_step

    def _traffic(k, per_launch_requests):
        if not traffic or k not in traffic:
            return None
        t = traffic[k]
        return t["dram_bytes_per_launch"] / t["requests_per_launch"] * per_launch_requests

    cores = _host_cores()
    ref_n = min(300000, n)  # cpu_baseline: a bounded sample (~13 s of host work on C4)
    cpu = None
    if os.path.exists(abi.REF_SO):
        rlib = _ref_lib()
        sample = trace.head(ref_n) if ref_n < n else trace
        runs = [time_reference(rlib, cfg, sample, cfg.driver) for _ in range(2)]
        cpu = {
            "value": ref_n / statistics.median(runs),
            "unit": UNIT,
            "cores": 1,
            "host_cores": cores,
            "kind": "reference",
            "sample": _sample_desc(cfg, ref_n, n, len(runs), cores),
        }
    secondary = None if args.no_secondary else secondary_lines(args, dev)
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
        "config": dict(_config_dict(cfg, n, args, ws), prompt_tokens=int(len(trace.tokens)), tree_nodes=nodes,
                       nodes_per_request=nodes / n),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": {
            "kernel": "k_serial (serial decide+commit replay: the dominant kernel)",
            "bound": "hbm",
            "achieved": ser_achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": ser_achieved / peak if peak else None,
            "traffic": _traffic("k_serial", req_per_launch),
            "algorithmic_bytes_per_launch": ser_bytes_launch,
            "algorithmic_bytes": "B_match + B_cost per request (SURVEY 8(d)), summed over the launch's requests",
            "avg_launch_ms": ser_launch_ms,
            "note": "latency-bound: one dependent decide/commit chain per request on one SM",
        },
        "roofline_k1": {
            "kernel": "k_match (K1 batched prefix match)",
            "bound": "hbm",
            "achieved": k1_achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": k1_achieved / peak if peak else None,
            "traffic": _traffic("k_match", n / match_launches_step),
            "algorithmic_bytes_per_launch": match_bytes_launch,
            "avg_launch_ms": match_ms,
        },
        "match_cost_phase": {
            "algorithmic_bytes_per_step": match_bytes_step + cost_bytes_step,
            "achieved_gbs_over_step": (match_bytes_step + cost_bytes_step) / 1e9 / (ms / 1e3),
            "frac_of_peak_over_step": (match_bytes_step + cost_bytes_step) / 1e9 / (ms / 1e3) / peak,
        },
        "traffic_probe": traffic,
        "kernel_share": shares,
        "kernel_ms_per_step": {nm: kms[i] for i, nm in enumerate(KNAMES)},
        "gpu_launches": int(sum(L)),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--batch", type=int, default=0, help="requests per device batch (0: the config's, else 16384)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=-1,
                    help="requests the host reference is timed on per step (0: all; default: all when steps+warmup <= 8, else 300k)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help=argparse.SUPPRESS)  # gloo: dev check on one GPU
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe-n", type=int, default=120000, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.probe:
        return run_probe(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
