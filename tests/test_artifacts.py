"""Artifact I/O vs the reference's own JSON writers (config.cpp, gantt.cpp, analysis.cpp),
golden texts in tests/golden/artifacts.json (oracle/gen_golden.py artifacts)."""
import json
import os

import numpy as np
import pytest

from paper_2602_05754_b200 import artifacts as art
from paper_2602_05754_b200 import pipefreeze as pf

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _fx(name):
    f = gold("fixtures.json")[name]
    pl = f["pipeline"]
    t = f["timing"]["per_stage"]
    return f, pl, t


@pytest.mark.parametrize("idx", range(4))
def test_plan_json_roundtrip_and_reference_compat(idx):
    case = gold("artifacts.json")[idx]
    f, pl, t = _fx(case["fixture"])
    R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
    S = R * C
    cfg = pf.PipelineConfig(pl["schedule"], R, C, M)
    # the reference's plan.json parses into a full ratio vector that reproduces its makespan
    ref_plan = art.plan_from_json(case["plan_json"], M, S)
    wmin, wmax = pf.stage_default_bounds(M, S, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"])
    dag = pf.build_dag(cfg)
    w = np.r_[0.0, wmax, 0.0]
    w[1 + M * S: 1 + 2 * M * S] = wmax[M * S:] - ref_plan["ratios"] * (wmax[M * S:] - wmin[M * S:])
    ms = pf.longest_path_start_times(dag, w).makespan
    assert abs(ms - ref_plan["makespan_opt"]) <= 1e-7 * ref_plan["makespan_base"]
    # our plan.json has the reference's schema and values within the LP tolerance
    ours = pf.solve_plan(cfg, wmin, wmax, f["r_max"])
    doc = json.loads(art.plan_to_json(ours, M, S))
    rdoc = json.loads(case["plan_json"])
    assert sorted(doc) == sorted(rdoc)
    assert [(e["m"], e["s"]) for e in doc["ratios"]] == [(e["m"], e["s"]) for e in rdoc["ratios"]]
    for k in ("makespan_base", "makespan_floor", "makespan_opt", "r_max"):
        assert abs(doc[k] - rdoc[k]) <= 1e-7 * max(1.0, rdoc["makespan_base"]), k
    back = art.plan_from_json(art.plan_to_json(ours, M, S), M, S)
    assert np.array_equal(back["ratios"], ours.ratios)
    # report.json: same schema; makespan-derived fields agree
    rep = json.loads(art.report_to_json(ours, M, S))
    rrep = json.loads(case["report_json"])
    assert sorted(rep) == sorted(rrep)
    for k in ("makespan_base_ms", "makespan_floor_ms", "kappa", "r_max"):
        assert rep[k] == pytest.approx(rrep[k], rel=1e-12), k
    for k in ("makespan_opt_ms", "reduction_pct", "throughput_gain_pct"):
        assert rep[k] == pytest.approx(rrep[k], rel=1e-6), k


@pytest.mark.parametrize("idx", range(4))
def test_gantt_json_matches_reference(idx):
    case = gold("artifacts.json")[idx]
    f, pl, t = _fx(case["fixture"])
    R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
    S = R * C
    cfg = pf.PipelineConfig(pl["schedule"], R, C, M)
    w = np.array([0.0] + [t["forward_ms"]] * (M * S) + [t["backward_act_ms"] + t["backward_param_ms"]] * (M * S) + [0.0])
    ours = art.gantt(cfg, w)
    ref = json.loads(case["gantt_json"])
    assert ours == ref  # identical blocks, start/end floats and makespan
    assert art.gantt_from_json(art.gantt_to_json(ours)) == ours


def test_mask_history_and_profile_json_match_reference():
    for case in gold("artifacts.json"):
        f, pl, t = _fx(case["fixture"])
        R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
        S = R * C
        ref_plan = art.plan_from_json(case["plan_json"], M, S)
        pop, _ = pf.run_freezing_masks(ref_plan["ratios"], pf.PhasePlan(2, 8, 10, 20), M, S, 500, f["seed"])
        # the reference plan.json carries ratios printed to 17 significant digits; the mask
        # counts floor(r * n) are reproduced from it
        assert json.loads(art.mask_history_to_json(pop, 500)) == json.loads(case["masks_json"])
        wmin, wmax = pf.stage_default_bounds(M, S, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"])
        assert json.loads(art.timing_profile_to_json(wmin, wmax, M, S)) == json.loads(case["profile_json"])


def test_bad_plan_json_raises_config_error():
    with pytest.raises(pf.ConfigError):
        art.plan_from_json("{not json", 2, 2)
    with pytest.raises(pf.ConfigError):
        art.plan_from_json(json.dumps({"makespan_opt": 1, "makespan_base": 1, "makespan_floor": 1,
                                       "ratios": [{"m": 3, "s": 1, "r": 0.5}]}), 2, 1)


def _gantt_worker(rank, world, kind, C, M, port, errq, outq):
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = pf.PipelineConfig(kind, world, C, M)
        dag = pf.build_dag(cfg)
        rng = np.random.default_rng(5)
        w = rng.uniform(0.5, 2.0, size=dag.node_count)
        w[0] = w[-1] = 0.0
        st = pf.longest_path_start_times(dag, w)

        class FakeTrainer:  # this rank's CUDA-event action times = the DAG schedule of w
            def action_times(self):
                acts = [a for a, _, _ in pf.issue_program(cfg, rank)]
                v = np.array([dag.index_of(a) for a in acts])
                return (st.start[v], st.start[v] + w[v], np.array([a.kind for a in acts]),
                        np.array([a.microbatch for a in acts]), np.array([a.stage for a in acts]))

        doc = art.measured_gantt(FakeTrainer())
        if rank == 0:
            outq.put((doc, art.gantt(cfg, w)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


@pytest.mark.parametrize("kind,world,C,M", [("1f1b", 2, 1, 4), ("interleaved-1f1b", 2, 2, 4)])
def test_measured_gantt_gathers_every_rank(kind, world, C, M):
    """Multi-rank measured Gantt (gantt.cpp:12-48 schema): blocks of every rank gathered over the
    process group, num_ranks = world size; with action times equal to the DAG schedule it is the
    reference's build_gantt of the same weights, block for block."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    errq, outq = ctx.Queue(), ctx.Queue()
    port = 31000 + (abs(hash((kind, world, C, M))) % 2000)
    procs = [ctx.Process(target=_gantt_worker, args=(r, world, kind, C, M, port, errq, outq)) for r in range(world)]
    for p in procs:
        p.start()
    doc, ref = outq.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert doc["num_ranks"] == world
    key = lambda b: (b["rank"], b["start_ms"], b["stage"], b["microbatch"], b["kind"])  # noqa: E731
    assert sorted(doc["blocks"], key=key) == sorted(ref["blocks"], key=key)
    assert doc["makespan_ms"] == ref["makespan_ms"]
