"""Pin the Python restatement oracle (oracle/pforacle.py) to the reference's own golden vectors."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pforacle as po  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def unhex(a):
    return [float.fromhex(x) for x in a]


def test_rng_restatement():
    g = gold("rng.json")
    r = po.Rng(42)
    assert [r.next_u64() for _ in range(16)] == [int(x) for x in g["seed42_u64"]]
    r = po.Rng(0)
    assert [r.next_u64() for _ in range(4)] == [int(x) for x in g["seed0_u64"]]
    mx = g["mixed_seed7"]
    r = po.Rng(7)
    for b, i, u, gs in zip(mx["bounds"], mx["index"], mx["unit"], mx["gauss"]):
        assert r.index_below(int(b)) == int(i)
        assert r.unit() == float.fromhex(u)
        assert r.gaussian() == float.fromhex(gs)


@pytest.mark.parametrize("case", range(16))
def test_schedule_dag_restatement(case):
    row = gold("schedules.json")[case]
    k, R, C, M = row["kind"], row["R"], row["C"], row["M"]
    assert [[list(a) for a in lst] for lst in po.schedule(k, R, C, M)] == row["rank_order"]
    edges, topo = po.dag(k, R, C, M)
    assert [list(e) for e in edges] == row["edges"]
    assert topo == row["topo"]
    start, ms = po.longest_path(edges, topo, unhex(row["weights"]))
    assert [x.hex() for x in start] == row["start"]
    assert ms.hex() == row["makespan"]


def test_phase_restatement():
    for row in gold("phases.json"):
        p = tuple(row["plan"])
        assert [po.phase_of(t, p) for t in range(1, p[3] + 1)] == row["phases"]
        for r, vals in row["afr_from_tm_plus_1"].items():
            assert [po.actual_freeze_ratio(t, p, float(r)).hex() for t in range(p[1] + 1, p[3] + 1)] == vals


def test_mask_restatement_small_cases():
    for case in gold("masks.json")["sample"]:
        if case["n"] > 1000:
            continue
        r = po.Rng(case["seed"])
        for ratio, wrow in zip(unhex(case["ratios"]), case["words"]):
            idx = po.sample_mask(case["n"], ratio, r)
            words = [0] * len(wrow)
            for i in idx:
                words[i >> 6] |= 1 << (i & 63)
            assert [str(w) for w in words] == wrow


def test_apf_restatement():
    for case in gold("apf.json"):
        n = case["n"]
        d = np.array(unhex(case["deltas"])).reshape(-1, n)
        e, a = np.zeros(n), np.zeros(n)
        for row in d:
            s = po.apf_update(e, a, row, case["alpha"])
        assert [x.hex() for x in e] == case["ema"]
        assert [x.hex() for x in a] == case["ema_abs"]
        assert [x.hex() for x in s] == case["scores"]


def test_masked_sgd_restatement_matches_reference_trajectory():
    """Replay run_masked_sgd's exact-count policy with the restated primitives (sandbox.cpp:222-253)."""
    for case in gold("sgd.json")["runs"]:
        if case["policy"] != 2:
            continue
        d, M = case["d"], case["M"]
        diag = np.array(unhex(case["diag"]))
        theta = np.array(unhex(case["theta0"]))
        rng = po.Rng(case["seed"])
        for _ in range(case["steps"]):
            grad = diag * theta
            gs, us = [], []
            for _m in range(M):
                g = grad.copy()
                if case["sigma"] > 0:
                    for j in range(d):
                        g[j] += case["sigma"] * rng.gaussian()
                u = np.ones(d)
                u[po.sample_mask(d, case["param"], rng)] = 0.0
                gs.append(g)
                us.append(u)
            theta = po.masked_sgd_update(theta, gs, us, case["eta"])
        np.testing.assert_allclose(theta, np.array(unhex(case["theta"])), rtol=1e-12, atol=1e-15)
