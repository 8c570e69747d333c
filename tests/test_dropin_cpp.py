"""The C++ drop-in wrapper (include/e2sched.hpp) replaces
kvsched::GlobalScheduler in the reference's own criterion-7 loop with no other
change: built against the reference headers and sources, run in lock step."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import BUILD, REPO, build_hostsim

REF = "/root/reference/proj"


def _build(lib_path, out):
    srcs = [os.path.join(REF, "src", f) for f in ("prefix_tree.cpp", "cost_model.cpp", "global_scheduler.cpp",
                                                   "workload.cpp")]
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-ffp-contract=off", "-w", "-I" + os.path.join(REPO, "include"),
           "-I" + os.path.join(REF, "include"), os.path.join(REPO, "tests", "cpp", "drop_in_main.cpp"), *srcs,
           lib_path, "-Wl,-rpath," + os.path.dirname(lib_path), "-o", out]
    subprocess.run(cmd, check=True)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")
def test_dropin_hostsim():
    lib = build_hostsim()
    exe = os.path.join(BUILD, "drop_in_hostsim")
    _build(lib, exe)
    out = subprocess.run([exe, "3000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "drop-in OK" in out.stdout


@pytest.mark.gpu
def test_dropin_b200():
    """The same lock-step loop with the drop-in on libe2sched.so (prebuilt by
    `make -C oracle e2e` where the reference sources are)."""
    exe = os.path.join(REPO, "oracle", "_ref", "drop_in_b200")
    if os.path.isdir(REF):
        subprocess.run(["make", "-s", "_ref/drop_in_b200"], cwd=os.path.join(REPO, "oracle"), check=True)
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/drop_in_b200 not built")
    out = subprocess.run([exe, "3000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "drop-in OK" in out.stdout and "b200 backend" in out.stdout
    print(out.stdout.strip().splitlines()[-1])
