"""Python mirror of the reference's host API (namespace pipefreeze), over libpf_host.so.

Names, argument meaning and error classes follow /root/reference/proj/include/pipefreeze:
  build_schedule / stage_to_rank        schedule.hpp:30,41
  build_dag / longest_path_start_times  dag.hpp:69,80
  phase_of / actual_freeze_ratio        freezectl.hpp:31,35
  sample_mask / reconcile_mask          freezectl.hpp:63,68
  run_freezing_masks                    freezectl.hpp:124
  build_lp + solve_lp + extract_freeze_plan, verify_solution  lp.hpp:52-114
  aggregate_monitoring                  timing.hpp:83
Errors: ConfigError (config_error, CLI exit 2), DomainError (std::domain_error,
exit 2), NumericalError (numerical_error, exit 3).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native

KINDS = {"gpipe": 0, "1f1b": 1, "interleaved-1f1b": 2, "interleaved": 2, "zbv": 3, "zbv-split": 4}
KIND_NAMES = {0: "gpipe", 1: "1f1b", 2: "interleaved-1f1b", 3: "zbv", 4: "zbv-split"}
SPLIT_KINDS = {4}  # backward split into b (dX) and w (dW) actions; not in the reference


class ConfigError(ValueError):
    pass


class DomainError(ValueError):
    pass


class NumericalError(RuntimeError):
    pass


def _check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {_native.host().pf_last_error().decode()}"
    if rc == _native.PF_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _native.PF_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == _native.PF_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise _native.PfError(rc, msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _kind(kind) -> int:
    if isinstance(kind, int):
        return kind
    try:
        return KINDS[kind]
    except KeyError:
        raise ConfigError(f"unknown schedule kind: '{kind}'") from None


class Phase(enum.IntEnum):
    Warmup = 0
    MonitorUpper = 1
    MonitorLower = 2
    Solve = 3
    ProgressiveFreeze = 4
    StableFreeze = 5


@dataclass(frozen=True, order=True)
class ActionId:
    """(kind, stage, microbatch) order as the reference's operator<=> (types.hpp:20-24)."""

    kind: int  # 0 forward, 1 backward, 2 weight gradient (zbv-split only)
    stage: int
    microbatch: int

    def __str__(self) -> str:
        return f"{'fbw'[self.kind]}({self.microbatch},{self.stage})"


def forward_action(m: int, s: int) -> ActionId:
    return ActionId(0, s, m)


def backward_action(m: int, s: int) -> ActionId:
    return ActionId(1, s, m)


def weight_action(m: int, s: int) -> ActionId:
    return ActionId(2, s, m)


@dataclass(frozen=True)
class PipelineConfig:
    schedule_kind: str = "gpipe"
    num_ranks: int = 1
    stages_per_rank: int = 1
    num_microbatches: int = 1

    @property
    def total_stages(self) -> int:
        return self.num_ranks * self.stages_per_rank

    def key(self):
        return (_kind(self.schedule_kind), self.num_ranks, self.stages_per_rank, self.num_microbatches)

    @property
    def split_weight(self) -> bool:
        return _kind(self.schedule_kind) in SPLIT_KINDS

    @property
    def kinds(self) -> int:
        """Action kinds per (m, s) cell: 2 (f, b) or 3 (f, b, w)."""
        return 3 if self.split_weight else 2

    def freeze_node(self, m: int, s: int) -> ActionId:
        return weight_action(m, s) if self.split_weight else backward_action(m, s)


@dataclass
class RankTimeline:
    config: PipelineConfig
    rank_order: list  # list[list[ActionId]]

    def rank_of(self, stage: int) -> int:
        return stage_to_rank(self.config, stage)


def build_schedule(config: PipelineConfig) -> RankTimeline:
    k, R, C, M = config.key()
    per = config.kinds * M * C
    acts = np.zeros(max(1, R) * per * 3 + 3, dtype=np.int32)
    lens = np.zeros(max(1, R), dtype=np.int32)
    _check(_native.host().pf_schedule_build(k, R, C, M, _p(acts), _p(lens)), "build_schedule")
    order, i = [], 0
    for r in range(R):
        lst = []
        for _ in range(int(lens[r])):
            kind, m, s = (int(x) for x in acts[i:i + 3])
            lst.append(ActionId(kind, s, m))
            i += 3
        order.append(lst)
    return RankTimeline(config, order)


def stage_to_rank(config: PipelineConfig, stage: int) -> int:
    out = ctypes.c_int(0)
    _check(_native.host().pf_stage_to_rank(*config.key(), stage, ctypes.byref(out)), "stage_to_rank")
    return out.value


def issue_program(config: PipelineConfig, rank: int) -> list[tuple[ActionId, int, int]]:
    """The rank's issue program (libpf_host issue_program, the one trainer.cpp walks): its actions
    in schedule order, each with the rank to receive from before it and the rank to send to after
    it (-1: none) for the cross-rank DAG rule-3 edges (dag.cpp:90-93)."""
    cap = config.kinds * config.num_microbatches * config.stages_per_rank
    ops = np.zeros(5 * cap, dtype=np.int32)
    n = ctypes.c_int(0)
    _check(_native.host().pf_issue_program(*config.key(), rank, _p(ops), ctypes.byref(n)), "issue_program")
    out = []
    for i in range(n.value):
        k, m, s, rf, st = (int(x) for x in ops[5 * i:5 * i + 5])
        out.append((ActionId(k, s, m), rf, st))
    return out


def p2p_links(config: PipelineConfig) -> list[tuple[int, int, int]]:
    """Cross-rank classes of DAG rule-3 edges (dag.cpp:90-93), one NCCL link each, in the device
    trainer's order (trainer.cpp): for s = 1..S-1 with rank(s) != rank(s+1), the activation link
    (0, rank(s), rank(s+1)) then the gradient link (1, rank(s+1), rank(s)), first occurrence kept."""
    out = []
    for s in range(1, config.total_stages):
        a, b = stage_to_rank(config, s), stage_to_rank(config, s + 1)
        if a == b:
            continue
        for link in ((0, a, b), (1, b, a)):
            if link not in out:
                out.append(link)
    return out


class PipelineDag:
    """Node ids: 0 = src, 1 + kind*M*S + (s-1)*M + (m-1), N-1 = dst (dag.cpp:18-23; kind 2 = w
    exists only for zbv-split)."""

    def __init__(self, config: PipelineConfig):
        self.config = config
        k, R, C, M = config.key()
        self.M, self.S = M, R * C
        n = self.node_count
        cap = 10 * n + 16
        e = np.zeros(2 * cap, dtype=np.int32)
        ne = ctypes.c_int(0)
        topo = np.zeros(n, dtype=np.int32)
        _check(_native.host().pf_dag_build(k, R, C, M, _p(e), cap, ctypes.byref(ne), _p(topo), None, 0), "build_dag")
        self.edges = [(int(e[2 * i]), int(e[2 * i + 1])) for i in range(ne.value)]
        self.topological_order = topo.tolist()

    @property
    def node_count(self) -> int:
        return self.config.kinds * self.M * self.S + 2

    @property
    def source(self) -> int:
        return 0

    @property
    def destination(self) -> int:
        return self.node_count - 1

    def index_of(self, a: ActionId) -> int:
        return 1 + a.kind * self.M * self.S + (a.stage - 1) * self.M + (a.microbatch - 1)

    def action_at(self, node: int) -> ActionId:
        k = node - 1
        per = self.M * self.S
        w = k % per
        return ActionId(k // per, w // self.M + 1, w % self.M + 1)

    def json_text(self) -> str:
        k, R, C, M = self.config.key()
        buf = ctypes.create_string_buffer(1 << 22)
        _check(_native.host().pf_dag_build(k, R, C, M, None, 0, None, None, buf, 1 << 22), "dag_to_json_text")
        return buf.value.decode()


def build_dag(timeline_or_config) -> PipelineDag:
    cfg = timeline_or_config.config if isinstance(timeline_or_config, RankTimeline) else timeline_or_config
    return PipelineDag(cfg)


@dataclass
class StartTimes:
    start: np.ndarray
    makespan: float


def longest_path_start_times(dag: PipelineDag, weights) -> StartTimes:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if w.shape != (dag.node_count,):
        raise DomainError("weights must cover every dag node")
    start = np.zeros(dag.node_count)
    ms = ctypes.c_double(0)
    _check(_native.host().pf_longest_path(*dag.config.key(), _p(w), _p(start), ctypes.byref(ms)), "longest_path")
    return StartTimes(start, ms.value)


def critical_path(dag: PipelineDag, weights) -> list[int]:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    nodes = np.zeros(dag.node_count, dtype=np.int32)
    ln = ctypes.c_int(0)
    _check(_native.host().pf_critical_path(*dag.config.key(), _p(w), _p(nodes), ctypes.byref(ln)), "critical_path")
    return nodes[: ln.value].tolist()


@dataclass(frozen=True)
class PhasePlan:
    t_warmup: int
    t_monitor: int
    t_freeze: int
    t_total: int

    def arr(self) -> np.ndarray:
        return np.array([self.t_warmup, self.t_monitor, self.t_freeze, self.t_total], dtype=np.int32)

    @property
    def t_mid(self) -> int:
        return self.t_warmup + (self.t_monitor - self.t_warmup + 1) // 2


def phase_of(t: int, plan: PhasePlan) -> Phase:
    out = ctypes.c_int(0)
    _check(_native.host().pf_phase_of(t, _p(plan.arr()), ctypes.byref(out)), "phase_of")
    return Phase(out.value)


def actual_freeze_ratio(t: int, plan: PhasePlan, expected_ratio: float) -> float:
    out = ctypes.c_double(0)
    _check(_native.host().pf_actual_freeze_ratio(t, _p(plan.arr()), expected_ratio, ctypes.byref(out)),
           "actual_freeze_ratio")
    return out.value


def afr_at(t: int, plan: PhasePlan, expected_ratio: float) -> float:
    return 0.0 if t <= plan.t_monitor else actual_freeze_ratio(t, plan, expected_ratio)


def rng_u64(seed: int, n: int) -> list[int]:
    out = np.zeros(n, dtype=np.uint64)
    _check(_native.host().pf_rng_u64(seed, n, _p(out)), "rng")
    return [int(x) for x in out]


def words_per_mask(n: int) -> int:
    return (n + 63) // 64


def sample_masks(seed: int, n_units: int, ratios) -> np.ndarray:
    """len(ratios) consecutive sample_mask calls on one Rng(seed) stream -> [count, words] uint64."""
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    w = words_per_mask(n_units)
    out = np.zeros((len(r), max(w, 1)), dtype=np.uint64)
    _check(_native.host().pf_sample_masks(seed, n_units, len(r), _p(r), _p(out)), "sample_mask")
    return out[:, :w]


def reconcile_mask(seed: int, n_units: int, base_words, target: int) -> np.ndarray:
    b = np.ascontiguousarray(base_words, dtype=np.uint64)
    out = np.zeros(max(1, words_per_mask(n_units)), dtype=np.uint64)
    _check(_native.host().pf_reconcile_mask(seed, n_units, _p(b), target, _p(out)), "reconcile_mask")
    return out[: words_per_mask(n_units)]


def unpack_mask(words: np.ndarray, n: int) -> np.ndarray:
    bits = np.unpackbits(np.ascontiguousarray(words, dtype="<u8").view(np.uint8), bitorder="little")
    return bits[:n].astype(bool)


def popcount(words: np.ndarray) -> int:
    return int(np.unpackbits(np.ascontiguousarray(words, dtype="<u8").view(np.uint8)).sum())


def run_freezing_masks(ratios, plan: PhasePlan, M: int, S: int, n_units: int, seed: int):
    """Reference controller horizon -> (popcounts[t,s,m], stage_counts[S, n])."""
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    pop = np.zeros(plan.t_total * S * M, dtype=np.int32)
    sc = np.zeros(S * n_units, dtype=np.int64)
    _check(_native.host().pf_freezing_masks_horizon(M, S, _p(plan.arr()), _p(r), n_units, seed, _p(pop), _p(sc)),
           "run_freezing_masks")
    return pop.reshape(plan.t_total, S, M), sc.reshape(S, n_units)


class MaskStream:
    """Random access into run_freezing_masks' single stream (t -> s -> m), by jump-ahead."""

    def __init__(self, ratios, plan: PhasePlan, M: int, S: int, n_units, seed: int):
        """n_units: one count for every stage, or a list of S per-stage counts."""
        self.ratios = np.ascontiguousarray(ratios, dtype=np.float64)
        self.plan, self.M, self.S, self.seed = plan, M, S, seed
        self.stage_units = None if np.isscalar(n_units) else np.ascontiguousarray(n_units, dtype=np.int32)
        self.n = int(n_units) if self.stage_units is None else None
        self.words = words_per_mask(self.n) if self.n is not None else None

    def stage_step(self, t: int, s: int, threads: int = 0) -> np.ndarray:
        n = self.n if self.stage_units is None else int(self.stage_units[s - 1])
        words = words_per_mask(n)
        out = np.zeros((self.M, max(1, words)), dtype=np.uint64)
        exact = ctypes.c_int(0)
        lib = _native.host()
        if self.stage_units is None:
            rc = lib.pf_mask_stream_stage_step(self.M, self.S, _p(self.plan.arr()), _p(self.ratios), n, self.seed, t, s,
                                               _p(out), threads, ctypes.byref(exact))
        else:
            rc = lib.pf_mask_stream_stage_step_units(self.M, self.S, _p(self.plan.arr()), _p(self.ratios),
                                                     _p(self.stage_units), self.seed, t, s, _p(out), threads,
                                                     ctypes.byref(exact))
        _check(rc, "mask_stream")
        return out[:, :words]

    def offset(self, t: int, s: int, m: int) -> int:
        out = ctypes.c_uint64(0)
        _check(_native.host().pf_mask_stream_offset(self.M, self.S, _p(self.plan.arr()), _p(self.ratios), self.n,
                                                    self.seed, t, s, m, ctypes.byref(out)), "mask_stream_offset")
        return out.value


@dataclass
class FreezePlan:
    ratios: np.ndarray          # [(s-1)*M + (m-1)]
    durations: np.ndarray       # per action node (node id - 1)
    makespan_base: float
    makespan_opt: float
    makespan_floor: float
    lp_makespan: float
    iterations: int
    stage_avg: np.ndarray
    r_max: float
    w_min: np.ndarray = field(repr=False, default=None)
    w_max: np.ndarray = field(repr=False, default=None)


def stage_default_bounds(M: int, S: int, fwd, bact, bparam, split: bool = False):
    """TimingProfile::from_stage_defaults (timing.cpp:13-27) as per-node bound arrays; split=True is
    from_stage_defaults_split (zbv-split: b = [act, act], w = [0, param])."""
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,))
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,))
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,))
    if split:
        wmin = np.concatenate([np.repeat(f, M), np.repeat(a, M), np.zeros(S * M)])
        wmax = np.concatenate([np.repeat(f, M), np.repeat(a, M), np.repeat(b, M)])
        return wmin, wmax
    wmin = np.concatenate([np.repeat(f, M), np.repeat(a, M)])
    wmax = np.concatenate([np.repeat(f, M), np.repeat(a + b, M)])
    return wmin, wmax


def solve_plan(config: PipelineConfig, w_min, w_max, r_max: float, lambda_mode: int = 0,
               budget_all: bool = False) -> FreezePlan:
    k, R, C, M = config.key()
    S = R * C
    wmin = np.ascontiguousarray(w_min, dtype=np.float64)
    wmax = np.ascontiguousarray(w_max, dtype=np.float64)
    ratios = np.zeros(S * M)
    dur = np.zeros(config.kinds * S * M)
    out5 = np.zeros(5)
    savg = np.zeros(S)
    _check(_native.host().pf_plan_solve(k, R, C, M, _p(wmin), _p(wmax), r_max, lambda_mode, int(budget_all),
                                        _p(ratios), _p(dur), _p(out5), _p(savg)), "solve_lp")
    return FreezePlan(ratios, dur, out5[0], out5[1], out5[2], out5[3], int(out5[4]), savg, r_max, wmin, wmax)


def verify_solution(config: PipelineConfig, plan: FreezePlan) -> tuple[bool, float]:
    ok = ctypes.c_int(0)
    rec = ctypes.c_double(0)
    _check(_native.host().pf_plan_verify(*config.key(), _p(plan.w_min), _p(plan.w_max), plan.r_max,
                                         _p(np.ascontiguousarray(plan.ratios)), _p(np.ascontiguousarray(plan.durations)),
                                         plan.makespan_opt, ctypes.byref(ok), ctypes.byref(rec)), "verify_solution")
    return bool(ok.value), rec.value


def plan_weights(config: PipelineConfig, plan: FreezePlan, afr_scale: float = 1.0) -> np.ndarray:
    n = config.kinds * config.num_microbatches * config.total_stages + 2
    out = np.zeros(n)
    _check(_native.host().pf_plan_weights(*config.key(), _p(plan.w_min), _p(plan.w_max),
                                          _p(np.ascontiguousarray(plan.ratios)), afr_scale, _p(out)), "plan_weights")
    return out


def aggregate_monitoring(M: int, S: int, node, step, sample_ms, frozen):
    """node = dag node id - 1; ids >= 2*M*S are w nodes of a zbv-split dag (3*M*S bounds out)."""
    node = np.ascontiguousarray(node, dtype=np.int32)
    step = np.ascontiguousarray(step, dtype=np.int32)
    ms = np.ascontiguousarray(sample_ms, dtype=np.float64)
    fz = np.ascontiguousarray(frozen, dtype=np.int32)
    kinds = 3 if len(node) and int(node.max()) >= 2 * M * S else 2
    wmin = np.zeros(kinds * M * S)
    wmax = np.zeros(kinds * M * S)
    _check(_native.host().pf_monitor_aggregate(M, S, len(node), _p(node), _p(step), _p(ms), _p(fz), _p(wmin), _p(wmax)),
           "aggregate_monitoring")
    return wmin, wmax


def simulate_monitoring(M: int, S: int, fwd, bact, bparam, plan: PhasePlan, sigma: float, seed: int):
    f = np.ascontiguousarray(np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)))
    a = np.ascontiguousarray(np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)))
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)))
    wmin = np.zeros(2 * M * S)
    wmax = np.zeros(2 * M * S)
    _check(_native.host().pf_simulate_monitoring(M, S, _p(f), _p(a), _p(b), _p(plan.arr()), sigma, seed,
                                                 _p(wmin), _p(wmax)), "run_monitoring")
    return wmin, wmax


def run_masked_sgd_quadratic(diag, theta0, eta: float, microbatches: int, steps: int, sigma: float, policy: int,
                             param: float, seed: int):
    """run_masked_sgd (sandbox.cpp:191-257) on a diagonal quadratic -> (theta_final, grad_sq_norms)."""
    dg = np.ascontiguousarray(diag, dtype=np.float64)
    t0 = np.ascontiguousarray(theta0, dtype=np.float64)
    th = np.zeros_like(t0)
    gs = np.zeros(steps)
    _check(_native.host().pf_masked_sgd_host(len(dg), _p(dg), _p(t0), eta, microbatches, steps, sigma, policy, param,
                                             seed, _p(th), _p(gs)), "run_masked_sgd")
    return th, gs


def run_masked_sgd_plan_quadratic(diag, theta0, eta: float, microbatches: int, steps: int, sigma: float, S: int,
                                  ratios, phases, step: int, seed: int):
    """run_masked_sgd with MaskPolicy::plan_driven (sandbox.cpp:97-115,158) on a diagonal quadratic:
    coordinate j belongs to stage block min(S-1, j*S/d) and is frozen in microbatch m with
    probability AFR(step, phases, ratio of b(m, s)). ratios[(s-1)*M + (m-1)]; step < 0 = t_total."""
    dg = np.ascontiguousarray(diag, dtype=np.float64)
    t0 = np.ascontiguousarray(theta0, dtype=np.float64)
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    ph = np.ascontiguousarray(phases, dtype=np.int32)
    th = np.zeros_like(t0)
    gs = np.zeros(steps)
    _check(_native.host().pf_masked_sgd_plan_host(len(dg), _p(dg), _p(t0), eta, microbatches, steps, sigma, S, _p(r),
                                                  _p(ph), step, seed, _p(th), _p(gs)), "run_masked_sgd(plan_driven)")
    return th, gs


def autofreeze_score(norm_prev: float, norm_cur: float) -> float:
    """AutoFreeze layer score (freezectl.cpp:116-122)."""
    out = ctypes.c_double(0)
    _check(_native.host().pf_autofreeze_score(norm_prev, norm_cur, ctypes.byref(out)), "autofreeze_score")
    return out.value


def autofreeze_select(scores, frozen_prefix_len: int, percentile: float) -> int:
    """AutoFreeze prefix selection by nearest-rank percentile (freezectl.cpp:124-136)."""
    sc = np.ascontiguousarray(scores, dtype=np.float64)
    out = ctypes.c_int(0)
    _check(_native.host().pf_autofreeze_select(_p(sc), len(sc), frozen_prefix_len, percentile, ctypes.byref(out)),
           "autofreeze_select")
    return out.value


def apf_update_host(ema: np.ndarray, ema_abs: np.ndarray, delta, alpha: float = 0.9) -> np.ndarray:
    d = np.ascontiguousarray(delta, dtype=np.float64)
    sc = np.zeros_like(d)
    _check(_native.host().pf_apf_update_host(len(d), alpha, _p(ema), _p(ema_abs), _p(d), _p(sc)), "apf_update")
    return sc
