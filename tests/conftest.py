"""Shared fixtures.

Backends (all implement include/e2sched.h):
  ref      oracle/_ref/libe2ref.so   — the unmodified reference (test-only)
  oracle   oracle/libe2oracle.so     — plain-C restatement (test-only)
  hostsim  tests/_build/libe2hostsim.so — the product engine source compiled
           for the host with a warp width of 1 (test double for CPU CI only)
  b200     paper_2407_00023_b200/libe2sched.so — the product (GPU tests)
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2407_00023_b200 import abi  # noqa: E402

BUILD = os.path.join(REPO, "tests", "_build")
HOSTSIM_SO = os.path.join(BUILD, "libe2hostsim.so")
CSRC = os.path.join(REPO, "paper_2407_00023_b200", "csrc")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the product library)")
    config.addinivalue_line("markers", "slow: larger parity cases")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_hostsim() -> str:
    srcs = [os.path.join(CSRC, "e2_lib.cu"), os.path.join(CSRC, "workload_gen.cpp"), os.path.join(CSRC, "corpus.cpp")]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(REPO, "include", "e2sched.h")]
    if _stale(HOSTSIM_SO, deps):
        os.makedirs(BUILD, exist_ok=True)
        tmp = HOSTSIM_SO + f".{os.getpid()}.tmp"
        cmd = [
            "/usr/bin/g++", "-x", "c++", "-std=c++17", "-O2", "-DE2_HOSTSIM", "-ffp-contract=off", "-fPIC", "-shared",
            "-I" + os.path.join(REPO, "include"), "-I" + CSRC, "-o", tmp, srcs[0], "-x", "c++", srcs[1], srcs[2],
        ]
        subprocess.run(cmd, check=True)
        os.replace(tmp, HOSTSIM_SO)
    return HOSTSIM_SO


def build_ref() -> str | None:
    if not os.path.exists(abi.REF_SO) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "ref"], cwd=os.path.join(REPO, "oracle"), check=True)
    return abi.REF_SO if os.path.exists(abi.REF_SO) else None


def build_oracle() -> str | None:
    src = os.path.join(REPO, "oracle", "e2_oracle.c")
    if os.path.exists(src) and _stale(abi.ORACLE_SO, [src, os.path.join(REPO, "include", "e2sched.h")]):
        subprocess.run(["make", "-s", "oracle"], cwd=os.path.join(REPO, "oracle"), check=True)
    return abi.ORACLE_SO if os.path.exists(abi.ORACLE_SO) else None


@pytest.fixture(scope="session")
def ref_lib():
    """The checker: the real reference when built, else the C restatement."""
    p = build_ref() or build_oracle()
    if p is None:
        pytest.skip("no reference/oracle library available")
    return abi.load_library(p)


@pytest.fixture(scope="session")
def true_ref_lib():
    p = build_ref()
    if p is None:
        pytest.skip("reference shim not built (needs /root/reference or a prebuilt oracle/_ref)")
    return abi.load_library(p)


@pytest.fixture(scope="session")
def oracle_lib():
    p = build_oracle()
    if p is None:
        pytest.skip("C oracle not built")
    return abi.load_library(p)


@pytest.fixture(scope="session")
def hostsim_lib():
    return abi.load_library(build_hostsim())


@pytest.fixture(scope="session")
def b200_lib():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    lib = abi.product_lib()
    assert lib.e2_backend().decode() == "b200"
    return lib


@pytest.fixture(scope="session")
def gen_lib(hostsim_lib):
    """Trace generation is host code shared by every product build."""
    return hostsim_lib
