"""the reference's own callers drive the product.

The reference's experiment harness, discrete-event simulator and per-instance
LocalSchedulers (harness.cpp, simulator.cpp:60-240, local_scheduler.cpp:
165-266 — the LocalScheduler's partial-tail LRU eviction and prefill
completion are the source of every note_eviction / note_prefill_cached) are
compiled UNCHANGED from /root/reference, with oracle/dropin/ shadowing
kvsched/global_scheduler.hpp so that kvsched::GlobalScheduler is the drop-in
class of include/e2sched.hpp over the C ABI.  On the experiment configs of
acceptance criteria 4-6 the metrics reports (JSON + per-request CSV) must be
byte-identical to the same harness linked against the reference's own
GlobalScheduler.  CPU: the host emulation; -m gpu: libe2sched.so."""
from __future__ import annotations

import filecmp
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(REPO, "oracle")
REF_BIN = os.path.join(ORACLE, "_ref", "e2e_ref")


def _make(target):
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", target], cwd=ORACLE, check=True)
    path = os.path.join(ORACLE, target)
    if not os.path.exists(path):
        pytest.skip(f"{target} not built (needs /root/reference here, or the prebuilt binary)")
    return path


def _run(binary, out):
    os.makedirs(out, exist_ok=True)
    r = subprocess.run([binary, out], capture_output=True, text=True, timeout=900, check=True)
    return {ln.split()[0]: float(ln.split()[1]) for ln in r.stdout.splitlines() if ln.strip()}


def _compare(dropin_bin, tmp_path):
    ref_bin = _make("_ref/e2e_ref")
    # the drop-in binary keeps no reference GlobalScheduler member (gc-sections)
    syms = subprocess.run(["nm", "-C", dropin_bin], capture_output=True, text=True).stdout
    assert "kvsched::GlobalScheduler::" not in syms
    t_ref = _run(ref_bin, str(tmp_path / "ref"))
    t_new = _run(dropin_bin, str(tmp_path / "dropin"))
    assert set(t_ref) == set(t_new) and len(t_ref) == 8
    names = sorted(os.listdir(tmp_path / "ref"))
    assert len(names) == 16
    _, mismatch, errors = filecmp.cmpfiles(tmp_path / "ref", tmp_path / "dropin", names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)
    return t_ref, t_new


def test_reference_harness_on_hostsim(tmp_path, hostsim_lib):
    _compare(_make("_ref/e2e_dropin_hostsim"), tmp_path)


@pytest.mark.gpu
def test_reference_harness_on_b200(tmp_path, b200_lib):
    t_ref, t_new = _compare(_make("_ref/e2e_dropin_b200"), tmp_path)
    print("e2e seconds (reference scheduler, drop-in B200):",
          {k: (round(t_ref[k], 3), round(t_new[k], 3)) for k in sorted(t_ref)})
