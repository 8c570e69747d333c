"""ctypes declarations for the C-ABI boundary (include/e2sched.h).

The same ABI is exported by three libraries:

* ``paper_2407_00023_b200/libe2sched.so`` — the product (device-resident tree,
  sm_100a kernels).  :func:`product_lib` loads it and raises if it is missing:
  there is no CPU fallback.
* ``oracle/_ref/libe2ref.so`` and ``oracle/libe2oracle.so`` — test-only
  checkers, loaded only by ``tests/``, ``bench.py`` and ``__graft_entry__``
  through :func:`load_library`.
"""
from __future__ import annotations

import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
PRODUCT_SO = os.path.join(PKG_DIR, "libe2sched.so")
REF_SO = os.path.join(REPO_DIR, "oracle", "_ref", "libe2ref.so")
ORACLE_SO = os.path.join(REPO_DIR, "oracle", "libe2oracle.so")

E2_OK = 0
E2_ERR_CONFIG = 1
E2_ERR_NO_ADMISSIBLE = 2
E2_ERR_SIM = 3
E2_ERR_CUDA = 4
E2_ERR_ARG = 5
E2_MAX_GPUS = 64

E2_EVICT_NONE = 0
E2_EVICT_FIFO_TAIL = 1
E2_EVICT_MIRROR_LRU = 2

E2_K_MATCH, E2_K_GROUP, E2_K_COMMIT, E2_K_OTHER = 0, 1, 2, 3
E2_K_COUNT = 4


class SchedCfg(ctypes.Structure):
    _fields_ = [
        ("history_window_ms", ctypes.c_double),
        ("th_bal", ctypes.c_double),
        ("imbal_ratio", ctypes.c_double),
        ("priority_groups", ctypes.c_int64),
        ("kv_capacity_tokens", ctypes.c_int64),
        ("default_output_len", ctypes.c_int64),
    ]


class TimeModelC(ctypes.Structure):
    _fields_ = [
        ("prefill_base_ms", ctypes.c_double),
        ("prefill_per_token_ms", ctypes.c_double),
        ("decode_per_token_ms", ctypes.c_double),
        ("iteration_base_ms", ctypes.c_double),
    ]


class PolicyC(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("rebalance", ctypes.c_int32),
        ("autoscale", ctypes.c_int32),
        ("pd_balance", ctypes.c_int32),
    ]


class CostC(ctypes.Structure):
    _fields_ = [
        ("gpu", ctypes.c_int32),
        ("eviction_infeasible", ctypes.c_int32),
        ("current_load_ms", ctypes.c_double),
        ("eviction_ms", ctypes.c_double),
        ("prefill_ms", ctypes.c_double),
    ]


class DecisionC(ctypes.Structure):
    _fields_ = [
        ("request", ctypes.c_int64),
        ("branch", ctypes.c_int32),
        ("gpu", ctypes.c_int32),
        ("redirected", ctypes.c_int32),
        ("pre_redirect_gpu", ctypes.c_int32),
        ("n_costs", ctypes.c_int32),
        ("has_ratios", ctypes.c_int32),
        ("cached_len", ctypes.c_int64),
        ("missed_len", ctypes.c_int64),
        ("missed_on_chosen", ctypes.c_int64),
        ("matched_len", ctypes.c_int64),
    ]


class StatsC(ctypes.Structure):
    _fields_ = [
        (n, ctypes.c_int64)
        for n in (
            "exploit",
            "explore",
            "decode_pressure",
            "round_robin",
            "redirected",
            "rebalance_installs",
            "autoscale_events",
            "tree_reads",
        )
    ]


class NodeC(ctypes.Structure):
    _fields_ = [
        ("id", ctypes.c_uint64),
        ("parent_id", ctypes.c_uint64),
        ("edge_off", ctypes.c_int64),
        ("edge_len", ctypes.c_int64),
        ("caching_mask", ctypes.c_uint64),
        ("last_access_mask", ctypes.c_uint64),
        ("pin_count", ctypes.c_int64),
    ]


class DriverCfg(ctypes.Structure):
    _fields_ = [
        ("eviction", ctypes.c_int32),
        ("prefill_cached", ctypes.c_int32),
        ("trunk_len", ctypes.c_int64),
        ("high_water", ctypes.c_int64),
        ("finish_lag", ctypes.c_int64),
        ("batch", ctypes.c_int64),
        ("prune_interval_ms", ctypes.c_double),
    ]


class ProfileC(ctypes.Structure):
    _fields_ = [
        ("ms", ctypes.c_double * E2_K_COUNT),
        ("launches", ctypes.c_int64 * E2_K_COUNT),
        ("match_bytes", ctypes.c_int64),
        ("match_requests", ctypes.c_int64),
        ("group_retries", ctypes.c_int64),
        ("delta_bytes", ctypes.c_int64),
        ("delta_chunks", ctypes.c_int64),
    ]


class WorkloadSpecC(ctypes.Structure):
    _fields_ = [
        ("archetype", ctypes.c_int32),
        ("zipf", ctypes.c_int32),
        ("request_count", ctypes.c_int64),
        ("system_prompt_len", ctypes.c_int64),
        ("branch_count", ctypes.c_int64),
        ("branch_len", ctypes.c_int64),
        ("branch_len_max", ctypes.c_int64),
        ("zipf_s", ctypes.c_double),
        ("unique_min", ctypes.c_int64),
        ("unique_max", ctypes.c_int64),
        ("output_min", ctypes.c_int64),
        ("output_max", ctypes.c_int64),
        ("requests_per_group", ctypes.c_double),
        ("chain_mean_len", ctypes.c_double),
        ("observation_len", ctypes.c_int64),
        ("fanout", ctypes.c_int64),
        ("depth", ctypes.c_int64),
    ]


P = ctypes.POINTER
_vp = ctypes.c_void_p
_h = ctypes.c_void_p
_i32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double

_SIGS = {
    "e2_create": (ctypes.c_int, [_i32, P(SchedCfg), P(TimeModelC), P(PolicyC), P(_h)]),
    "e2_destroy": (None, [_h]),
    "e2_reset": (ctypes.c_int, [_h]),
    "e2_set_stream": (ctypes.c_int, [_h, _vp]),
    "e2_last_error": (ctypes.c_char_p, [_h]),
    "e2_backend": (ctypes.c_char_p, []),
    "e2_schedule": (ctypes.c_int, [_h, _vp, _i64, _i64, _f64, _f64, P(DecisionC), _vp, _vp]),
    "e2_decide": (ctypes.c_int, [_h, _vp, _i64, _i64, _f64, P(DecisionC), _vp, _vp]),
    "e2_note_admitted": (ctypes.c_int, [_h, _i64, _f64]),
    "e2_note_prefill_cached": (ctypes.c_int, [_h, _vp, _i64, _i32, _f64]),
    "e2_note_eviction": (ctypes.c_int, [_h, _vp, _i64, _i64, _i32, _f64]),
    "e2_note_finished": (ctypes.c_int, [_h, _i64, _f64, _i64]),
    "e2_decode_ratio": (ctypes.c_int, [_h, _i32, P(_f64)]),
    "e2_gpu_load_ms": (ctypes.c_int, [_h, _i32, _f64, P(_f64)]),
    "e2_prune_dead_nodes": (ctypes.c_int, [_h, _f64, P(_i64)]),
    "e2_cached_tokens": (ctypes.c_int, [_h, _i32, P(_i64)]),
    "e2_node_count": (ctypes.c_int, [_h, P(_i64)]),
    "e2_redirects": (ctypes.c_int, [_h, _vp]),
    "e2_get_stats": (ctypes.c_int, [_h, P(StatsC)]),
    "e2_load_cost": (ctypes.c_int, [_h, _i32, _i64, _f64, P(CostC)]),
    "e2_match": (ctypes.c_int, [_h, _vp, _i64, P(_i64), P(_i64), _vp]),
    "e2_export_size": (ctypes.c_int, [_h, P(_i64), P(_i64)]),
    "e2_export": (ctypes.c_int, [_h, _f64, _vp, _vp, _vp, _vp]),
    "e2_debug_dump": (ctypes.c_int, [_h, _f64, ctypes.c_char_p, ctypes.c_size_t, P(ctypes.c_size_t)]),
    "e2_window_sizes": (ctypes.c_int, [_h, _i32, _f64, P(_i64), P(_i64), P(_i64), P(_i64)]),
    "e2_replay": (ctypes.c_int, [_h, _vp, _vp, _vp, _vp, _vp, _i64, P(DriverCfg), _vp, _vp, _vp, P(_i64)]),
    "e2_replay_device": (
        ctypes.c_int,
        [_h, _vp, _vp, _vp, _vp, _vp, _i64, P(DriverCfg), _vp, _vp, _vp, _vp, P(_i64)],
    ),
    "e2_profile_get": (ctypes.c_int, [_h, P(ProfileC)]),
    "e2_profile_reset": (ctypes.c_int, [_h, _i32]),
    "e2_workload_default": (None, [_i32, P(WorkloadSpecC)]),
    "e2_generate": (
        ctypes.c_int,
        [P(WorkloadSpecC), _u64, _f64, _u64, P(_i64), P(_i64), _vp, _vp, _vp, _vp, _vp],
    ),
}

#: Product-only entry points (the sharded replay); attached when
#: the library exports them.
_PRODUCT_SIGS = {
    "e2_shard_begin": (
        ctypes.c_int,
        [_h, _vp, _vp, _vp, _vp, _vp, _i64, P(DriverCfg), _vp, _vp, _vp, _i32, _i32],
    ),
    "e2_shard_next": (ctypes.c_int, [_h, P(_i64), P(_i64), P(_i64)]),
    "e2_shard_match": (ctypes.c_int, [_h, _i64, _i64, _vp]),
    "e2_shard_commit": (ctypes.c_int, [_h, _vp, _i64, P(_i64)]),
    "e2_shard_delta_copy": (ctypes.c_int, [_h, _vp]),
    "e2_shard_apply": (ctypes.c_int, [_h, _vp, _i64]),
    "e2_shard_end": (ctypes.c_int, [_h, P(_i64)]),
    "e2_state_digest": (ctypes.c_int, [_h, _vp, _i32, P(_i32)]),
    "e2_replay_set_continue": (ctypes.c_int, [_h, _i32]),
}

class DistC(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64)] + [(n, ctypes.c_double) for n in ("mean", "p50", "p99", "min", "max")]


class StudyC(ctypes.Structure):
    _fields_ = [
        ("requests", ctypes.c_int64),
        ("total_prompt_tokens", ctypes.c_int64),
        ("total_output_tokens", ctypes.c_int64),
        ("total_shared_tokens", ctypes.c_int64),
        ("shared_token_fraction", ctypes.c_double),
        ("mean_request_shared_fraction", ctypes.c_double),
        ("mean_prompt_output_ratio", ctypes.c_double),
        ("prompt_len", DistC),
        ("output_len", DistC),
        ("key_portion_count", ctypes.c_int64),
        ("mean_key_portion_len", ctypes.c_double),
        ("requests_per_shared_sequence", DistC),
    ]


#: Corpus / trace files and the study (product and reference shim).
_CORPUS_SIGS = {
    "e2_corpus_write": (ctypes.c_int, [ctypes.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp, _i64]),
    "e2_corpus_read": (ctypes.c_int, [ctypes.c_char_p, P(_i64), P(_i64), _vp, _vp, _vp, _vp, _vp, _vp]),
    "e2_trace_read": (ctypes.c_int, [ctypes.c_char_p, P(_i64), _vp, _vp, _vp]),
    "e2_synthesize_from_trace": (
        ctypes.c_int,
        [P(WorkloadSpecC), _u64, _vp, _vp, _vp, _i64, P(_i64), _vp, _vp, _vp, _vp, _vp],
    ),
    "e2_analyze": (ctypes.c_int, [_vp, _vp, _vp, _i64, P(StudyC)]),
}
#: Entry points only the product (and its host emulation) exports: the
#: checkers have no sharded or streamed replay.
PRODUCT_ONLY = tuple(_PRODUCT_SIGS)
_PRODUCT_SIGS.update(_CORPUS_SIGS)
#: snapshot() pieces beyond export/window sizes (product and reference shim;
#: the plain-C oracle has no snapshot).
_PRODUCT_SIGS.update({
    "e2_window_entries": (ctypes.c_int, [_h, _i32, _f64, _vp, _vp, _vp, _vp, _vp]),
    "e2_export_hit_stamps": (ctypes.c_int, [_h, _f64, _vp, _i64, P(_i64)]),
})

#: Every symbol include/e2sched.h declares (checked by the CPU test suite).
DECLARED_SYMBOLS = tuple(_SIGS) + tuple(_PRODUCT_SIGS)

_cache: dict[str, ctypes.CDLL] = {}


def load_library(path: str) -> ctypes.CDLL:
    """Load one implementation of the ABI and attach signatures."""
    path = os.path.abspath(path)
    if path in _cache:
        return _cache[path]
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    for name, (res, args) in _PRODUCT_SIGS.items():
        if hasattr(lib, name):
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
    _cache[path] = lib
    return lib


def product_lib() -> ctypes.CDLL:
    """The B200 library.  Fails loudly when the CUDA extension is not built."""
    if not os.path.exists(PRODUCT_SO):
        raise RuntimeError(
            f"CUDA extension {PRODUCT_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    return load_library(PRODUCT_SO)
