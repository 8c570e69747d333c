"""Python mirror of the reference's ``kvsched::GlobalScheduler`` interface.

Same names, argument meaning and error behaviour as
``proj/include/kvsched/global_scheduler.hpp:99-161`` so that tests read like
the reference's own (``proj/tests/test_global_scheduler.cpp``).  Every call
goes through the C ABI (include/e2sched.h); by default that is the product
library ``libe2sched.so`` whose state lives in HBM.  ``lib=`` selects a
test-only checker instead (reference shim / C oracle).
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import abi


# --- reference exception types (types.hpp:32-46, global_scheduler.hpp:14-16) ---
class ConfigError(RuntimeError):
    pass


class SimError(RuntimeError):
    pass


class NoAdmissibleGpu(SimError):
    pass


class BackendError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == abi.E2_ERR_CONFIG:
        raise ConfigError(msg)
    if code == abi.E2_ERR_NO_ADMISSIBLE:
        raise NoAdmissibleGpu(msg)
    if code == abi.E2_ERR_SIM:
        raise SimError(msg)
    raise BackendError(f"e2 error {code}: {msg}")


@dataclasses.dataclass
class SchedulerConfig:  # global_scheduler.hpp:18-27
    history_window_ms: float = 180000.0
    th_bal: float = 2.0
    imbal_ratio: float = 0.9
    priority_groups: int = 10
    kv_capacity_tokens: int = 200000
    default_output_len: int = 32

    def to_c(self) -> abi.SchedCfg:
        return abi.SchedCfg(
            self.history_window_ms,
            self.th_bal,
            self.imbal_ratio,
            self.priority_groups,
            self.kv_capacity_tokens,
            self.default_output_len,
        )


@dataclasses.dataclass
class TimeModel:  # cost_model.hpp:12-17
    prefill_base_ms: float = 5.0
    prefill_per_token_ms: float = 0.25
    decode_per_token_ms: float = 15.0
    iteration_base_ms: float = 8.0

    def to_c(self) -> abi.TimeModelC:
        return abi.TimeModelC(
            self.prefill_base_ms, self.prefill_per_token_ms, self.decode_per_token_ms, self.iteration_base_ms
        )


PREFIX_AWARE = 0
ROUND_ROBIN = 1


@dataclasses.dataclass
class GlobalPolicy:  # global_scheduler.hpp:31-36
    mode: int = PREFIX_AWARE
    rebalance: bool = True
    autoscale: bool = True
    pd_balance: bool = True

    def to_c(self) -> abi.PolicyC:
        return abi.PolicyC(self.mode, int(self.rebalance), int(self.autoscale), int(self.pd_balance))


EXPLOIT, EXPLORE, DECODE_PRESSURE, ROUND_ROBIN_BRANCH = 0, 1, 2, 3
BRANCH_NAMES = {0: "exploit", 1: "explore", 2: "decode_pressure", 3: "round_robin"}


@dataclasses.dataclass
class CostBreakdown:  # cost_model.hpp:73-82
    current_load_ms: float = 0.0
    eviction_ms: float = 0.0
    prefill_ms: float = 0.0
    eviction_infeasible: bool = False

    def total_ms(self) -> float:
        return (self.current_load_ms + self.eviction_ms) + self.prefill_ms


@dataclasses.dataclass
class GpuCandidateCost:
    gpu: int
    cost: CostBreakdown


@dataclasses.dataclass
class Decision:  # global_scheduler.hpp:53-64 (+ matched_len)
    request: int = 0
    branch: int = EXPLORE
    gpu: int = -1
    redirected: bool = False
    pre_redirect_gpu: int = -1
    cached_len: int = 0
    missed_len: int = 0
    missed_on_chosen: int = 0
    matched_len: int = 0
    costs: List[GpuCandidateCost] = dataclasses.field(default_factory=list)
    decode_ratios: Dict[int, float] = dataclasses.field(default_factory=dict)


@dataclasses.dataclass
class Request:  # types.hpp:23-28
    id: int
    prompt: Sequence[int]
    arrival_ms: float = 0.0
    output_len: int = 0


@dataclasses.dataclass
class EvictedRange:  # prefix_tree.hpp:84-89
    seq: Sequence[int]
    tail_len: int


@dataclasses.dataclass
class GlobalStats:  # global_scheduler.hpp:85-94
    exploit: int = 0
    explore: int = 0
    decode_pressure: int = 0
    round_robin: int = 0
    redirected: int = 0
    rebalance_installs: int = 0
    autoscale_events: int = 0
    tree_reads: int = 0


@dataclasses.dataclass
class NodeExport:  # PrefixTree::NodeSnapshot (prefix_tree.hpp:186-194), hits as windowed counts
    id: int
    parent_id: int
    edge: tuple
    caching_gpus: tuple
    last_access: Dict[int, float]
    hits: Dict[int, int]
    pin_count: int


@dataclasses.dataclass
class NodeSnapshot:  # PrefixTree::NodeSnapshot (prefix_tree.hpp:170-178); hits: in-window stamps
    id: int
    parent_id: int
    edge: tuple
    caching_gpus: tuple
    hits: Dict[int, List[float]]
    last_access: Dict[int, float]
    pin_count: int


@dataclasses.dataclass
class GpuSnap:  # ClusterSnapshot::GpuSnap (global_scheduler.hpp:74-80)
    id: int
    scheduled: List[tuple]  # LoadWindow::Scheduled (t, missed, est_output)
    completed: List[tuple]  # LoadWindow::Completed (t, output)
    inflight_cached: int
    inflight_prompt: int


@dataclasses.dataclass
class ClusterSnapshot:  # global_scheduler.hpp:67-83 (config/model/policy: the scheduler's own)
    now: float
    n_gpus: int
    nodes: List[NodeSnapshot]
    gpus: List[GpuSnap]
    redirects: Dict[int, int]


def _tokens(seq) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int32))
    return a


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class GlobalScheduler:
    """``kvsched::GlobalScheduler`` over the C ABI (global_scheduler.hpp:99-161)."""

    def __init__(
        self,
        n_gpus: int,
        config: Optional[SchedulerConfig] = None,
        model: Optional[TimeModel] = None,
        policy: Optional[GlobalPolicy] = None,
        lib: Optional[ctypes.CDLL] = None,
    ):
        self._lib = lib if lib is not None else abi.product_lib()
        self.config = config or SchedulerConfig()
        self.model = model or TimeModel()
        self.policy = policy or GlobalPolicy()
        self._n = int(n_gpus)
        h = ctypes.c_void_p()
        rc = self._lib.e2_create(
            self._n,
            ctypes.byref(self.config.to_c()),
            ctypes.byref(self.model.to_c()),
            ctypes.byref(self.policy.to_c()),
            ctypes.byref(h),
        )
        if rc != abi.E2_OK:
            _raise(rc, self._lib.e2_last_error(None).decode())
        self._h = h
        self._costs = (abi.CostC * (self._n + 1))()
        self._ratios = np.zeros(max(self._n, 1), dtype=np.float64)

    # -- lifetime -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.e2_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def backend(self) -> str:
        return self._lib.e2_backend().decode()

    def n_gpus(self) -> int:
        return self._n

    def _check(self, rc: int):
        if rc != abi.E2_OK:
            _raise(rc, self._lib.e2_last_error(self._h).decode())

    # -- decisions ------------------------------------------------------
    def _decision(self, d: abi.DecisionC) -> Decision:
        out = Decision(
            request=d.request,
            branch=d.branch,
            gpu=d.gpu,
            redirected=bool(d.redirected),
            pre_redirect_gpu=d.pre_redirect_gpu,
            cached_len=d.cached_len,
            missed_len=d.missed_len,
            missed_on_chosen=d.missed_on_chosen,
            matched_len=d.matched_len,
        )
        for i in range(d.n_costs):
            c = self._costs[i]
            out.costs.append(
                GpuCandidateCost(
                    c.gpu,
                    CostBreakdown(c.current_load_ms, c.eviction_ms, c.prefill_ms, bool(c.eviction_infeasible)),
                )
            )
        if d.has_ratios:
            out.decode_ratios = {g: float(self._ratios[g]) for g in range(self._n)}
        return out

    def schedule_request(self, req: Request, now: float) -> Decision:
        p = _tokens(req.prompt)
        d = abi.DecisionC()
        rc = self._lib.e2_schedule(
            self._h, _ptr(p), len(p), int(req.id), float(req.arrival_ms), float(now), ctypes.byref(d),
            ctypes.cast(self._costs, ctypes.c_void_p), _ptr(self._ratios),
        )
        self._check(rc)
        return self._decision(d)

    def decide(self, req: Request, now: float) -> Decision:
        p = _tokens(req.prompt)
        d = abi.DecisionC()
        rc = self._lib.e2_decide(
            self._h, _ptr(p), len(p), int(req.id), float(now), ctypes.byref(d),
            ctypes.cast(self._costs, ctypes.c_void_p), _ptr(self._ratios),
        )
        self._check(rc)
        return self._decision(d)

    # -- callbacks ------------------------------------------------------
    def note_admitted(self, request_id: int, now: float):
        self._check(self._lib.e2_note_admitted(self._h, int(request_id), float(now)))

    def note_prefill_cached(self, prompt, gpu: int, now: float):
        p = _tokens(prompt)
        self._check(self._lib.e2_note_prefill_cached(self._h, _ptr(p), len(p), int(gpu), float(now)))

    def note_eviction(self, rng: EvictedRange, gpu: int, now: float):
        s = _tokens(rng.seq)
        self._check(self._lib.e2_note_eviction(self._h, _ptr(s), len(s), int(rng.tail_len), int(gpu), float(now)))

    def note_finished(self, request_id: int, now: float, output_len: int):
        self._check(self._lib.e2_note_finished(self._h, int(request_id), float(now), int(output_len)))

    # -- queries --------------------------------------------------------
    def decode_ratio(self, gpu: int) -> float:
        v = ctypes.c_double()
        self._check(self._lib.e2_decode_ratio(self._h, int(gpu), ctypes.byref(v)))
        return v.value

    def gpu_load_ms(self, gpu: int, now: float) -> float:
        v = ctypes.c_double()
        self._check(self._lib.e2_gpu_load_ms(self._h, int(gpu), float(now), ctypes.byref(v)))
        return v.value

    def prune_dead_nodes(self, now: float) -> int:
        v = ctypes.c_int64()
        self._check(self._lib.e2_prune_dead_nodes(self._h, float(now), ctypes.byref(v)))
        return v.value

    def cached_tokens(self, gpu: int) -> int:
        v = ctypes.c_int64()
        self._check(self._lib.e2_cached_tokens(self._h, int(gpu), ctypes.byref(v)))
        return v.value

    def node_count(self) -> int:
        v = ctypes.c_int64()
        self._check(self._lib.e2_node_count(self._h, ctypes.byref(v)))
        return v.value

    def redirects(self) -> Dict[int, int]:
        a = np.full(self._n, -1, dtype=np.int32)
        self._check(self._lib.e2_redirects(self._h, _ptr(a)))
        return {g: int(t) for g, t in enumerate(a) if t >= 0}

    def stats(self) -> GlobalStats:
        s = abi.StatsC()
        self._check(self._lib.e2_get_stats(self._h, ctypes.byref(s)))
        return GlobalStats(*[getattr(s, f) for f, _ in abi.StatsC._fields_])

    def load_cost(self, gpu: int, missed_tokens: int, now: float) -> CostBreakdown:
        c = abi.CostC()
        self._check(self._lib.e2_load_cost(self._h, int(gpu), int(missed_tokens), float(now), ctypes.byref(c)))
        return CostBreakdown(c.current_load_ms, c.eviction_ms, c.prefill_ms, bool(c.eviction_infeasible))

    def match(self, seq):
        """Read-only mirror().match(seq): (matched_len, cached_len, {gpu: extent})."""
        s = _tokens(seq)
        m, c = ctypes.c_int64(), ctypes.c_int64()
        per = np.zeros(self._n, dtype=np.int64)
        self._check(self._lib.e2_match(self._h, _ptr(s), len(s), ctypes.byref(m), ctypes.byref(c), _ptr(per)))
        return m.value, c.value, {g: int(v) for g, v in enumerate(per) if v > 0}

    def window_sizes(self, gpu: int, now: float):
        a = [ctypes.c_int64() for _ in range(4)]
        self._check(self._lib.e2_window_sizes(self._h, int(gpu), float(now), *[ctypes.byref(x) for x in a]))
        return tuple(x.value for x in a)

    def export_arrays(self, now: float):
        """Raw export: (nodes structured array, tokens, last_access[n,G], hits[n,G])."""
        nn, nt = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.e2_export_size(self._h, ctypes.byref(nn), ctypes.byref(nt)))
        nodes = (abi.NodeC * nn.value)()
        toks = np.zeros(max(nt.value, 1), dtype=np.int32)
        la = np.zeros((nn.value, self._n), dtype=np.float64)
        hits = np.zeros((nn.value, self._n), dtype=np.int64)
        self._check(
            self._lib.e2_export(self._h, float(now), ctypes.cast(nodes, ctypes.c_void_p), _ptr(toks), _ptr(la), _ptr(hits))
        )
        return nodes, toks, la, hits

    def export_nodes(self, now: float) -> List[NodeExport]:
        nodes, toks, la, hits = self.export_arrays(now)
        out = []
        for i, n in enumerate(nodes):
            gpus = tuple(g for g in range(self._n) if (n.caching_mask >> g) & 1)
            lam = {g: float(la[i, g]) for g in range(self._n) if (n.last_access_mask >> g) & 1}
            hm = {g: int(hits[i, g]) for g in range(self._n) if hits[i, g] > 0}
            out.append(
                NodeExport(
                    n.id, n.parent_id, tuple(toks[n.edge_off : n.edge_off + n.edge_len].tolist()), gpus, lam, hm,
                    n.pin_count,
                )
            )
        return out

    def snapshot(self, now: float) -> ClusterSnapshot:
        """snapshot(now) (global_scheduler.cpp:375-394).  Node hits hold the
        in-window stamps (t >= now - H), which is what the reference's reads
        see after their lazy prune; its raw deques may hold older ones."""
        gpus = []
        for g in range(self._n):
            ns, nc, ic, ip = self.window_sizes(g, now)
            st, sm, se = np.zeros(ns), np.zeros(ns, dtype=np.int64), np.zeros(ns, dtype=np.int64)
            ct, co = np.zeros(nc), np.zeros(nc, dtype=np.int64)
            self._check(self._lib.e2_window_entries(self._h, g, float(now), _ptr(st), _ptr(sm), _ptr(se), _ptr(ct), _ptr(co)))
            gpus.append(GpuSnap(g, list(zip(st.tolist(), sm.tolist(), se.tolist())), list(zip(ct.tolist(), co.tolist())), ic, ip))
        nodes, toks, la, hits = self.export_arrays(now)
        total = ctypes.c_int64()
        self._check(self._lib.e2_export_hit_stamps(self._h, float(now), None, 0, ctypes.byref(total)))
        stamps = np.zeros(max(total.value, 1))
        self._check(self._lib.e2_export_hit_stamps(self._h, float(now), _ptr(stamps), total.value, ctypes.byref(total)))
        out, k = [], 0
        for i, n in enumerate(nodes):
            hm = {}
            for g in range(self._n):
                c = int(hits[i, g])
                if c:
                    hm[g] = stamps[k : k + c].tolist()
                    k += c
            out.append(NodeSnapshot(
                n.id, n.parent_id, tuple(toks[n.edge_off : n.edge_off + n.edge_len].tolist()),
                tuple(g for g in range(self._n) if (n.caching_mask >> g) & 1), hm,
                {g: float(la[i, g]) for g in range(self._n) if (n.last_access_mask >> g) & 1}, n.pin_count))
        if k != total.value:
            raise SimError(f"snapshot: {total.value} hit stamps for {k} windowed hits")
        return ClusterSnapshot(float(now), self._n, out, gpus, self.redirects())

    def debug_dump(self, now: float) -> str:
        need = ctypes.c_size_t()
        self._check(self._lib.e2_debug_dump(self._h, float(now), None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value + 1)
        self._check(self._lib.e2_debug_dump(self._h, float(now), buf, need.value + 1, ctypes.byref(need)))
        return buf.value.decode()

    def state_digest(self) -> np.ndarray:
        """Non-mutating digest of the replicated state regions (product only)."""
        out = np.zeros(32, dtype=np.uint64)
        n = ctypes.c_int32()
        self._check(self._lib.e2_state_digest(self._h, _ptr(out), 32, ctypes.byref(n)))
        return out[: n.value].copy()

    # -- batched trace driver ---------------------------------------------
    def replay(self, trace, driver, want_costs: bool = True, want_ratios: bool = False):
        """e2_replay over a :class:`workload.Trace`; returns a :class:`ReplayResult`."""
        n = trace.n
        out = np.zeros(n, dtype=DECISION_DTYPE)
        costs = np.zeros((n, self._n + 1), dtype=COST_DTYPE) if want_costs else None
        ratios = np.zeros((n, self._n), dtype=np.float64) if want_ratios else None
        done = ctypes.c_int64()
        rc = self._lib.e2_replay(
            self._h, _ptr(trace.tokens), _ptr(trace.offsets), _ptr(trace.ids), _ptr(trace.arrivals),
            _ptr(trace.output_lens), n, ctypes.byref(driver.to_c()), _ptr(out), _ptr(costs), _ptr(ratios),
            ctypes.byref(done),
        )
        res = ReplayResult(out, costs, ratios, done.value)
        if rc != abi.E2_OK:
            err = self._lib.e2_last_error(self._h).decode()
            try:
                _raise(rc, err)
            except Exception as e:  # attach partial results
                e.partial = res
                raise
        return res


DECISION_DTYPE = np.dtype(
    [
        ("request", "<i8"),
        ("branch", "<i4"),
        ("gpu", "<i4"),
        ("redirected", "<i4"),
        ("pre_redirect_gpu", "<i4"),
        ("n_costs", "<i4"),
        ("has_ratios", "<i4"),
        ("cached_len", "<i8"),
        ("missed_len", "<i8"),
        ("missed_on_chosen", "<i8"),
        ("matched_len", "<i8"),
    ]
)
assert DECISION_DTYPE.itemsize == ctypes.sizeof(abi.DecisionC)

COST_DTYPE = np.dtype(
    [
        ("gpu", "<i4"),
        ("eviction_infeasible", "<i4"),
        ("current_load_ms", "<f8"),
        ("eviction_ms", "<f8"),
        ("prefill_ms", "<f8"),
    ]
)
assert COST_DTYPE.itemsize == ctypes.sizeof(abi.CostC)


@dataclasses.dataclass
class ReplayResult:
    decisions: np.ndarray
    costs: Optional[np.ndarray]
    ratios: Optional[np.ndarray]
    n_done: int


@dataclasses.dataclass
class DriverConfig:
    """e2_driver_cfg: the generalised criterion-7 loop (acceptance_main.cpp:367-416)."""

    eviction: int = abi.E2_EVICT_FIFO_TAIL
    prefill_cached: bool = True
    trunk_len: int = 1860
    high_water: int = 150000
    finish_lag: int = 2000
    batch: int = 0
    prune_interval_ms: float = 0.0  # > 0: prune_dead_nodes at every tick k*interval <= now (simulator cadence H/2)

    def to_c(self) -> abi.DriverCfg:
        return abi.DriverCfg(
            self.eviction, int(self.prefill_cached), self.trunk_len, self.high_water, self.finish_lag, self.batch,
            float(self.prune_interval_ms),
        )
