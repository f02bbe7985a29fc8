"""Artifact I/O compatible with the reference's JSON files.

Schemas follow proj/src/config.cpp and proj/src/gantt.cpp exactly (keys, nesting,
ordering); values come from this build's host layer:
  plan.json         freeze_plan_to_json_text      config.cpp:188-198
  report.json       throughput_report_to_json_text config.cpp:240-257 (+ build_report, analysis.cpp:33-71)
  timeline json     gantt_to_json_text            gantt.cpp:34-48 (planned or CUDA-event measured)
  masks.json        mask_history_to_json_text     config.cpp:278-287
  timing profile    timing_profile_to_json_text   config.cpp:166-175
so a plan written by the reference's `pipefreeze optimize` can drive the device
trainer, and this build's plans/timelines can be read by the reference CLI.
"""
from __future__ import annotations

import json

import numpy as np

from . import pipefreeze as pf


def _dump(doc) -> str:
    return json.dumps(doc, indent=2, sort_keys=True) + "\n"


def kappa(r_max: float, pd_min: float, pd_max: float) -> float:
    """analysis.cpp:9-14."""
    if not (0.0 <= r_max <= 1.0):
        raise pf.DomainError("r_max must be in [0, 1]")
    if not (0.0 < pd_min <= pd_max):
        raise pf.DomainError("makespan envelopes must satisfy 0 < pd_min <= pd_max")
    return (1.0 - r_max) + r_max * pd_min / pd_max


def plan_to_json(plan, M: int, S: int) -> str:
    """FreezePlan (pipefreeze.solve_plan result, or a dict with ratios/makespans/r_max) -> plan.json text."""
    get = (lambda k: plan[k]) if isinstance(plan, dict) else (lambda k: getattr(plan, k))
    ratios = np.asarray(get("ratios"), dtype=np.float64)
    rows = [{"m": m, "r": float(ratios[(s - 1) * M + (m - 1)]), "s": s} for s in range(1, S + 1) for m in range(1, M + 1)]
    doc = {"makespan_base": float(get("makespan_base")), "makespan_floor": float(get("makespan_floor")),
           "makespan_opt": float(get("makespan_opt")), "r_max": float(get("r_max")), "ratios": rows}
    return _dump(doc)


def plan_from_json(text: str, M: int, S: int) -> dict:
    """plan.json text (reference or ours) -> {ratios[(s-1)*M+(m-1)], makespans, r_max, stage_avg}."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise pf.ConfigError(f"plan is not valid json: {e}") from None
    ratios = np.zeros(S * M)
    seen = np.zeros(S * M, dtype=bool)
    for ent in doc["ratios"]:
        m, s = int(ent["m"]), int(ent["s"])
        if not (1 <= m <= M and 1 <= s <= S):
            raise pf.ConfigError(f"plan entry b({m},{s}) is outside the configured pipeline")
        ratios[(s - 1) * M + (m - 1)] = float(ent["r"])
        seen[(s - 1) * M + (m - 1)] = True
    if not seen.all():
        raise pf.ConfigError(f"plan has {int(seen.sum())} ratios but the config expects {S * M}")
    return {"ratios": ratios, "makespan_opt": float(doc["makespan_opt"]), "makespan_base": float(doc["makespan_base"]),
            "makespan_floor": float(doc["makespan_floor"]), "r_max": float(doc.get("r_max", 0.0)),
            "stage_avg": ratios.reshape(S, M).mean(axis=1)}


def report_to_json(plan, M: int, S: int, avg_freeze_ratio: float | None = None,
                   reference_gain_pct: float | None = None) -> str:
    """build_report + throughput_report_to_json_text (analysis.cpp:33-71, config.cpp:240-257)."""
    get = (lambda k: plan[k]) if isinstance(plan, dict) else (lambda k: getattr(plan, k))
    base, opt, floor, r_max = (float(get(k)) for k in ("makespan_base", "makespan_opt", "makespan_floor", "r_max"))
    if not (floor <= opt + 1e-9 and opt <= base + 1e-9):
        raise pf.DomainError("inconsistent plan makespans")
    ratios = np.asarray(get("ratios"), dtype=np.float64).reshape(S, M)
    k = kappa(r_max, floor, base)
    p_eff = None if avg_freeze_ratio is None or avg_freeze_ratio >= 1.0 else 1.0 - avg_freeze_ratio
    doc = {"avg_freeze_ratio": avg_freeze_ratio, "kappa": k, "makespan_base_ms": base, "makespan_floor_ms": floor,
           "makespan_opt_ms": opt, "p_eff": p_eff, "predicted_tta_ratio": (k / p_eff) if p_eff else None,
           "r_max": r_max, "reduction_pct": 100.0 * (1.0 - opt / base), "reference_gain_pct": reference_gain_pct,
           "stage_avg_freeze_ratio": {str(s + 1): float(ratios[s].mean()) for s in range(S)},
           "throughput_gain_pct": 100.0 * (base / opt - 1.0)}
    return _dump(doc)


def gantt(config: pf.PipelineConfig, weights) -> dict:
    """build_gantt (gantt.cpp:12-32): blocks from longest-path start times, rank lanes from the schedule."""
    dag = pf.build_dag(config)
    w = np.asarray(weights, dtype=np.float64)
    st = pf.longest_path_start_times(dag, w)
    blocks = []
    for rank, lst in enumerate(pf.build_schedule(config).rank_order):
        for a in lst:
            v = dag.index_of(a)
            blocks.append({"end_ms": float(st.start[v] + w[v]), "kind": "fbw"[a.kind], "microbatch": a.microbatch,
                           "rank": rank, "stage": a.stage, "start_ms": float(st.start[v])})
    return {"blocks": blocks, "makespan_ms": float(st.makespan), "num_ranks": config.num_ranks}


def measured_gantt(trainer, rank: int | None = None, group=None) -> dict:
    """Timeline of the trainer's last step in the reference's gantt schema (gantt.cpp:12-48), from
    the CUDA-event action times (start/end relative to the step's origin event).

    Multi-rank (torch.distributed initialised): every rank's blocks are gathered (a collective:
    call it on every rank) and num_ranks is the world size. The ranks share one time axis when
    they barriered right before the step (pf_trainer_step records the origin event first); the
    makespan is the latest end over all ranks."""
    import torch.distributed as dist

    start, end, kinds, mbs, stages = trainer.action_times()
    multi = dist.is_available() and dist.is_initialized()
    if rank is None:
        rank = dist.get_rank(group) if multi else 0
    blocks = [{"end_ms": float(e), "kind": "fbw"[int(k)], "microbatch": int(m), "rank": int(rank), "stage": int(s),
               "start_ms": float(b)} for b, e, k, m, s in zip(start, end, kinds, mbs, stages)]
    world = 1
    if multi:
        world = dist.get_world_size(group)
        parts = [None] * world
        dist.all_gather_object(parts, blocks, group=group)
        blocks = [b for part in parts for b in part]
    blocks.sort(key=lambda b: (b["rank"], b["start_ms"]))
    return {"blocks": blocks, "makespan_ms": float(max((b["end_ms"] for b in blocks), default=0.0)),
            "num_ranks": world}


def gantt_to_json(doc: dict) -> str:
    return _dump(doc)


def gantt_from_json(text: str) -> dict:
    return json.loads(text)


def mask_history_to_json(popcounts: np.ndarray, n_units: int) -> str:
    """popcounts[t, s, m] (pipefreeze.run_freezing_masks) -> masks.json rows (config.cpp:278-287)."""
    Tt, S, M = popcounts.shape
    rows = [{"action": f"b({m + 1},{s + 1})", "n_params": n_units, "popcount": int(popcounts[t, s, m]),
             "stage": s + 1, "step": t + 1} for t in range(Tt) for s in range(S) for m in range(M)]
    return _dump({"rows": rows})


def timing_profile_to_json(w_min, w_max, M: int, S: int) -> str:
    """Per-node bounds in ActionId order -> timing profile json (config.cpp:166-175)."""
    nodes = []
    for kind in range(len(w_min) // (S * M)):  # f, b (, w for a split backward)
        for s in range(1, S + 1):
            for m in range(1, M + 1):
                i = kind * S * M + (s - 1) * M + (m - 1)
                nodes.append({"kind": "fbw"[kind], "m": m, "s": s, "w_max": float(w_max[i]), "w_min": float(w_min[i])})
    return _dump({"per_node": nodes})
