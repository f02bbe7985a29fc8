"""ZBV with the backward split into B (dX) and W (dW) actions.

The reference keeps one combined b node per cell, so there are no golden vectors
for this schedule: these tests pin its structural properties (every action exactly once, the
per-cell and per-stage orders, a valid DAG) and what the split is for (a shorter base makespan
than combined ZBV under the same total backward time, an LP plan over the w nodes that
verifies). Host-only: run on CPU."""
import numpy as np
import pytest

from paper_2602_05754_b200 import pipefreeze as pf

CASES = [(1, 4), (2, 4), (2, 8), (4, 8), (4, 16)]


@pytest.mark.parametrize("R,M", CASES)
def test_schedule_emits_each_action_once_in_dependency_order(R, M):
    cfg = pf.PipelineConfig("zbv-split", R, 2, M)
    tl = pf.build_schedule(cfg)
    S = 2 * R
    seen = {}
    for r, lst in enumerate(tl.rank_order):
        assert len(lst) == 3 * M * 2
        for i, a in enumerate(lst):
            assert pf.stage_to_rank(cfg, a.stage) == r
            assert a not in seen
            seen[a] = (r, i)
        pos = {a: i for i, a in enumerate(lst)}
        for s in {a.stage for a in lst}:
            for m in range(1, M + 1):
                f, b, w = pf.forward_action(m, s), pf.backward_action(m, s), pf.weight_action(m, s)
                assert pos[f] < pos[b] < pos[w]
                if m > 1:
                    assert pos[pf.weight_action(m - 1, s)] < pos[w]
    assert len(seen) == 3 * M * S


@pytest.mark.parametrize("R,M", CASES)
def test_dag_has_w_nodes_and_validates(R, M):
    cfg = pf.PipelineConfig("zbv-split", R, 2, M)
    dag = pf.build_dag(cfg)
    S = 2 * R
    assert dag.node_count == 3 * M * S + 2
    edges = set(dag.edges)
    for s in range(1, S + 1):
        for m in range(1, M + 1):
            b, w = dag.index_of(pf.backward_action(m, s)), dag.index_of(pf.weight_action(m, s))
            assert (b, w) in edges
            assert dag.action_at(w) == pf.weight_action(m, s)
        assert (dag.index_of(pf.weight_action(M, s)), dag.destination) in edges
    assert sorted(dag.topological_order) == list(range(dag.node_count))
    assert '"w(1,1)"' in dag.json_text()


@pytest.mark.parametrize("R,M", [(2, 4), (2, 8), (4, 8), (4, 16)])
def test_split_shortens_base_makespan_and_plan_verifies(R, M):
    S = 2 * R
    fwd, act, param = 1.0, 1.0, 1.0
    split = pf.PipelineConfig("zbv-split", R, 2, M)
    comb = pf.PipelineConfig("zbv", R, 2, M)
    wmin_s, wmax_s = pf.stage_default_bounds(M, S, fwd, act, param, split=True)
    wmin_c, wmax_c = pf.stage_default_bounds(M, S, fwd, act, param)
    base_s = pf.longest_path_start_times(pf.build_dag(split), np.r_[0.0, wmax_s, 0.0]).makespan
    base_c = pf.longest_path_start_times(pf.build_dag(comb), np.r_[0.0, wmax_c, 0.0]).makespan
    assert base_s < base_c  # W fills pipeline bubbles
    plan = pf.solve_plan(split, wmin_s, wmax_s, 0.8)
    assert np.all(plan.ratios >= -1e-9) and np.all(plan.ratios <= 1 + 1e-9)
    assert np.all(plan.stage_avg <= 0.8 + 1e-7)
    assert plan.makespan_opt <= base_s + 1e-9
    ok, rec = pf.verify_solution(split, plan)
    assert ok and abs(rec - plan.makespan_opt) < 1e-6 * max(1.0, base_s)
    plan_c = pf.solve_plan(comb, wmin_c, wmax_c, 0.8)
    assert plan.makespan_opt <= plan_c.makespan_opt + 1e-6
    # b nodes are fixed: only w durations move
    dur = plan.durations.reshape(3, S, M)
    assert np.allclose(dur[1], act)
    w = pf.plan_weights(split, plan)
    assert abs(pf.longest_path_start_times(pf.build_dag(split), w).makespan - plan.makespan_opt) < 1e-6 * base_s


def test_monitoring_keeps_split_b_fixed():
    M, S = 2, 2
    dag = pf.build_dag(pf.PipelineConfig("zbv-split", 1, 2, M))
    node, step, ms, fz = [], [], [], []
    for t, frozen in ((1, 0), (2, 0), (3, 1), (4, 1)):
        for s in range(1, S + 1):
            for m in range(1, M + 1):
                for a, base in ((pf.forward_action(m, s), 2.0), (pf.backward_action(m, s), 3.0),
                                (pf.weight_action(m, s), 4.0)):
                    node.append(dag.index_of(a) - 1)
                    step.append(t)
                    is_w = a.kind == 2
                    ms.append(base * (0.25 if (frozen and is_w) else 1.0) + 0.01 * t)
                    fz.append(int(frozen and is_w))
    wmin, wmax = pf.aggregate_monitoring(M, S, node, step, ms, fz)
    assert len(wmin) == 3 * M * S
    n = M * S
    assert np.allclose(wmin[:2 * n], wmax[:2 * n])  # f and b fixed (b includes the frozen-phase samples)
    assert np.all(wmin[2 * n:] < wmax[2 * n:])


def test_unknown_kind_rejected():
    with pytest.raises(pf.ConfigError):
        pf.build_schedule(pf.PipelineConfig("zbv-split", 2, 1, 4))
