"""dev: per-call API latency on the product (e2_schedule + note_prefill_cached +
note_finished per request, a C1-shaped trace): wall time per call and the
serial kernel's share."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2407_00023_b200 import abi, workload as W
from paper_2407_00023_b200.scheduler import GlobalScheduler, Request
lib = abi.product_lib()
cfg = W.CONFIGS["c1"]
tr = cfg.trace(lib=lib, n_requests=int(sys.argv[1]) if len(sys.argv) > 1 else 2000)
s = GlobalScheduler(cfg.n_gpus, cfg.sched, lib=lib)
reqs = [Request(int(tr.ids[i]), tr.prompt(i), float(tr.arrivals[i]), int(tr.output_lens[i])) for i in range(tr.n)]
for r in reqs[:200]:
    d = s.schedule_request(r, r.arrival_ms)
lib.e2_reset(s._h)
lib.e2_profile_reset(s._h, 1)
t0 = time.perf_counter(); calls = 0
for i, r in enumerate(reqs):
    d = s.schedule_request(r, r.arrival_ms); calls += 1
    s.note_prefill_cached(r.prompt, d.gpu, r.arrival_ms); calls += 1
    if i >= 500:
        o = reqs[i - 500]; s.note_finished(o.id, r.arrival_ms, o.output_len); calls += 1
dt = time.perf_counter() - t0
p = abi.ProfileC(); lib.e2_profile_get(s._h, ctypes.byref(p))
print(f"{calls} calls in {dt:.3f} s: {1e6 * dt / calls:.1f} us/call wall; serial kernel {1e3 * p.ms[3] / max(1, p.launches[3]):.1f} us/launch "
      f"({p.launches[3]} launches, {100 * p.ms[3] / 1e3 / dt:.0f}% of wall)")
s.close()
