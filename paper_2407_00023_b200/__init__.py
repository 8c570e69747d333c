"""B200-native E2 global-scheduler hot path (Preble, arXiv 2407.00023).

The product is ``libe2sched.so`` (device-resident radix tree + sm_100a
kernels) behind the C ABI in ``include/e2sched.h``; this package is its
Python mirror of the reference's ``kvsched::GlobalScheduler`` API.
"""
from . import abi
from .scheduler import (
    ConfigError,
    CostBreakdown,
    Decision,
    DriverConfig,
    EvictedRange,
    GlobalPolicy,
    GlobalScheduler,
    NoAdmissibleGpu,
    Request,
    SchedulerConfig,
    SimError,
    TimeModel,
)

__all__ = [
    "abi",
    "ConfigError",
    "CostBreakdown",
    "Decision",
    "DriverConfig",
    "EvictedRange",
    "GlobalPolicy",
    "GlobalScheduler",
    "NoAdmissibleGpu",
    "Request",
    "SchedulerConfig",
    "SimError",
    "TimeModel",
]
