"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/*.json from the compiled reference.

Run in the build container (needs /root/reference for the fixtures and
oracle/_ref/libpfref.so from `make -C oracle`):

    python oracle/gen_golden.py            # everything but the two below
    python oracle/gen_golden.py artifacts  # tests/golden/artifacts.json
    python oracle/gen_golden.py lp_big     # tests/golden/lp_big.json (reference simplex, ~7 min)

Every number here comes from the reference's own functions (oracle/ref_harness.cpp).
Floats that must match bit-exactly are stored as float.hex() strings.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import ref  # noqa: E402

FIXTURES = "/root/reference/proj/fixtures"
OUT = os.path.join(ROOT, "tests", "golden")


def hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dump(name, obj):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print("wrote", name)


def fixtures():
    out = {}
    for fn in sorted(os.listdir(FIXTURES)):
        with open(os.path.join(FIXTURES, fn)) as f:
            out[fn[:-5]] = json.load(f)
    return out


SCHED_CASES = [
    ("gpipe", 2, 1, 2), ("gpipe", 4, 1, 8), ("1f1b", 2, 1, 2), ("1f1b", 4, 1, 8), ("1f1b", 3, 1, 2),
    ("1f1b", 8, 1, 32), ("gpipe", 2, 1, 8), ("gpipe", 4, 1, 1), ("interleaved-1f1b", 2, 2, 4),
    ("interleaved-1f1b", 4, 2, 8), ("interleaved-1f1b", 8, 2, 32), ("interleaved-1f1b", 3, 3, 5),
    ("zbv", 2, 2, 4), ("zbv", 4, 2, 8), ("zbv", 1, 2, 3), ("1f1b", 1, 1, 4),
]


def gen_rng():
    bounds = [10, 3, 1, 7, 1000, 53248, 2, 5, 1 << 40, 17] * 3
    idx, unit, gauss = ref.rng_mixed(7, bounds)
    dump("rng.json", {
        "seed42_u64": [str(x) for x in ref.rng_u64(42, 16)],
        "seed0_u64": [str(x) for x in ref.rng_u64(0, 4)],
        "mixed_seed7": {"bounds": [str(b) for b in bounds], "index": [str(i) for i in idx],
                        "unit": hx(unit), "gauss": hx(gauss)},
    })


def gen_schedules():
    rows = []
    for kind, R, C, M in SCHED_CASES:
        order = ref.schedule(kind, R, C, M)
        edges, topo, js = ref.dag(kind, R, C, M, with_json=(2 * M * R * C + 2) <= 66)
        n = 2 * M * R * C + 2
        rng = np.random.default_rng(R * 1000 + C * 100 + M)
        w = rng.uniform(0.5, 3.0, size=n)
        w[0] = 0.0
        w[-1] = 0.0
        start, ms = ref.longest_path(kind, R, C, M, w)
        rows.append({"kind": kind, "R": R, "C": C, "M": M, "rank_order": order, "edges": edges, "topo": topo,
                     "json": js, "weights": hx(w), "start": hx(start), "makespan": float(ms).hex(),
                     "stage_to_rank": [ref.lib().ref_stage_to_rank(ref.KIND[kind], R, C, M, s) for s in range(1, R * C + 1)]})
    dump("schedules.json", rows)


def gen_phases():
    plans = [[160, 200, 250, 400], [2, 8, 10, 20], [1, 2, 2, 5], [2, 4, 9, 12], [3, 10, 10, 10], [100, 200, 200, 300]]
    out = []
    for p in plans:
        ph = [ref.phase_of(t, p) for t in range(1, p[3] + 1)]
        afr = {str(r): hx([ref.afr(t, p, r) for t in range(p[1] + 1, p[3] + 1)]) for r in (0.8, 0.65, 0.3, 1.0)}
        out.append({"plan": p, "phases": ph, "afr_from_tm_plus_1": afr})
    dump("phases.json", out)


def gen_masks(fx):
    cases = []
    for seed, n, ratios in [(42, 16, [0.5]), (42, 10, [0.0, 1.0, 0.5, 0.56, 0.0]), (9, 1000, list(np.linspace(0, 1, 21))),
                            (123, 53248, [0.6, 0.35]), (5, 64, [0.99, 0.01, 0.5]), (11, 1, [1.0, 0.5]), (3, 0, [0.5])]:
        words = ref.sample_masks(seed, n, ratios)
        cases.append({"seed": seed, "n": n, "ratios": hx(ratios),
                      "words": [[str(int(x)) for x in row] for row in words] if n <= 1000 else None,
                      "sha": sha(words), "popcounts": [int(sum(bin(int(x)).count("1") for x in row)) for row in words]})
    rec = []
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(1, 200))
        base = ref.sample_masks(trial + 100, n, [float(rng.uniform())])[0]
        target = int(rng.integers(0, n + 1))
        out = ref.reconcile(trial + 7, n, base, target)
        rec.append({"n": n, "seed": trial + 7, "base": [str(int(x)) for x in base], "target": target,
                    "out": [str(int(x)) for x in out]})
    base = np.zeros(1, dtype=np.uint64)
    base[0] = (1 << 0) | (1 << 2) | (1 << 4)
    rec.append({"n": 10, "seed": 7, "base": [str(int(base[0]))], "target": 5,
                "out": [str(int(x)) for x in ref.reconcile(7, 10, base, 5)]})
    # full-horizon controller on two fixtures, using the reference's own LP plan
    horizon = []
    for name, n, plan_override, t_from, t_to in [("default_1f1b_s4m8", 10000, None, 199, 203),
                                                  ("gpipe_s2m2", 300, [2, 8, 10, 20], 1, 20),
                                                  ("interleaved_r2c2m4", 2000, [2, 6, 9, 14], 6, 10)]:
        f = fx[name]
        pl = f["pipeline"]
        R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
        t = f["timing"]["per_stage"]
        pr = ref.plan(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"], f["r_max"])
        ph = plan_override or [f["phases"][k] for k in ("t_warmup", "t_monitor", "t_freeze", "t_total")]
        pop, sc, w = ref.freezing_masks(M, R * C, ph, pr["ratios"], n, f["seed"], t_from, t_to)
        horizon.append({"fixture": name, "n": n, "phases": ph, "seed": f["seed"], "ratios": hx(pr["ratios"]),
                        "popcounts": pop.tolist(), "stage_counts_sha": sha(sc.astype(np.int64)),
                        "stage_counts_sum": [int(x) for x in sc.sum(axis=1)],
                        "t_from": t_from, "t_to": t_to, "words_sha": sha(w),
                        "words": [[str(int(x)) for x in row] for row in w] if n <= 300 else None})
    dump("masks.json", {"sample": cases, "reconcile": rec, "horizon": horizon})


def gen_apf():
    rng = np.random.default_rng(17)
    out = []
    for n, alpha, steps in [(64, 0.9, 5), (257, 0.5, 12), (1000, 0.99, 3)]:
        d = rng.normal(scale=1e-3, size=(steps, n))
        d[:, :3] = 0.0  # E_abs == 0 -> score 1 branch
        e, ea, s = ref.apf(n, alpha, d)
        out.append({"n": n, "alpha": alpha, "deltas": hx(d), "ema": hx(e), "ema_abs": hx(ea), "scores": hx(s)})
    e, ea, s = ref.apf(1, 0.9, np.array([[1.0], [-1.0]]))
    out.append({"n": 1, "alpha": 0.9, "deltas": hx([1.0, -1.0]), "ema": hx(e), "ema_abs": hx(ea), "scores": hx(s)})
    dump("apf.json", out)


def gen_lp(fx):
    rows = []
    for name, f in fx.items():
        pl = f["pipeline"]
        t = f["timing"]["per_stage"]
        R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
        for lam in (0, 1):
            p = ref.plan(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"], f["r_max"], lam)
            rows.append({"name": name, "kind": pl["schedule"], "R": R, "C": C, "M": M,
                         "fwd": [t["forward_ms"]] * (R * C), "bact": [t["backward_act_ms"]] * (R * C),
                         "bparam": [t["backward_param_ms"]] * (R * C), "r_max": f["r_max"], "lambda_mode": lam,
                         "budget_all": 0, **{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in p.items()}})
    # heterogeneous stages (LP fodder: embedding-heavy first stage, LM-head-heavy last stage)
    extra = [("1f1b", 4, 1, 8, [12.0, 10.0, 10.0, 16.0], [13.0, 10.0, 10.0, 18.0], [15.0, 12.0, 12.0, 20.0], 0.7),
             ("gpipe", 4, 1, 8, [12.0, 10.0, 10.0, 16.0], [13.0, 10.0, 10.0, 18.0], [15.0, 12.0, 12.0, 20.0], 0.5),
             ("gpipe", 2, 1, 8, [5.0, 6.0], [5.0, 7.0], [6.0, 8.0], 0.8),
             ("1f1b", 8, 1, 8, [10.0] * 8, [10.0] * 8, [12.0] * 8, 0.8),
             ("interleaved-1f1b", 2, 2, 4, [7.0, 8.0, 7.5, 9.0], [7.0, 8.0, 8.0, 9.0], [9.0, 9.5, 9.0, 11.0], 0.6),
             ("1f1b", 2, 1, 2, [1.0, 1.0], [1.0, 1.0], [1.0, 1.0], 1.0),
             ("1f1b", 2, 1, 2, [1.0, 1.0], [1.0, 1.0], [1.0, 1.0], 0.0)]
    for kind, R, C, M, fw, ba, bp, rmax in extra:
        for budget_all in (0, 1):
            p = ref.plan(kind, R, C, M, fw, ba, bp, rmax, 0, budget_all)
            rows.append({"name": f"{kind}_r{R}c{C}m{M}_het", "kind": kind, "R": R, "C": C, "M": M, "fwd": fw, "bact": ba,
                         "bparam": bp, "r_max": rmax, "lambda_mode": 0, "budget_all": budget_all,
                         **{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in p.items()}})
    dump("lp.json", rows)


BIG_LP_CASES = [
    # (kind, R, C, M): 258-node and 514-node-class DAGs the dense simplex still finishes (90-190 s each);
    # embedding-heavy first stage, LM-head-heavy last stage (the heterogeneous rows of gen_lp, scaled up)
    ("1f1b", 8, 1, 16), ("interleaved-1f1b", 8, 2, 8), ("1f1b", 4, 1, 32),
]


def _het(S):
    fw = [12.0] + [10.0] * (S - 2) + [16.0]
    ba = [13.0] + [10.0] * (S - 2) + [18.0]
    bp = [15.0] + [12.0] * (S - 2) + [20.0]
    return fw, ba, bp


def gen_lp_big():
    """tests/golden/lp_big.json: reference solves of 258-node pipelines (slow: ~7 min in total)."""
    import time

    rows = []
    for kind, R, C, M in BIG_LP_CASES:
        fw, ba, bp = _het(R * C)
        w0 = time.time()
        p = ref.plan(kind, R, C, M, fw, ba, bp, 0.8, 0, 0)
        rows.append({"name": f"{kind}_r{R}c{C}m{M}_big", "kind": kind, "R": R, "C": C, "M": M, "fwd": fw, "bact": ba,
                     "bparam": bp, "r_max": 0.8, "lambda_mode": 0, "budget_all": 0,
                     **{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in p.items()},
                     "wall_s": time.time() - w0})
    dump("lp_big.json", rows)


def gen_monitor():
    out = []
    for M, S, fw, ba, bp, plan, sigma, seed in [(2, 2, [1.0, 2.0], [1.0, 1.5], [1.0, 2.5], [160, 200, 250, 400], 0.0, 13),
                                                (4, 3, [3.0, 2.0, 4.0], [2.0, 2.5, 3.0], [4.0, 3.0, 5.0], [2, 8, 10, 20], 0.05, 42),
                                                (1, 1, [1.0], [1.0], [1.0], [10, 20, 25, 30], 0.2, 5)]:
        wmin, wmax = ref.monitor(M, S, fw, ba, bp, plan, sigma, seed)
        out.append({"M": M, "S": S, "fwd": fw, "bact": ba, "bparam": bp, "plan": plan, "sigma": sigma, "seed": seed,
                    "w_min": hx(wmin), "w_max": hx(wmax)})
    dump("monitor.json", out)


def gen_sgd():
    out = []
    for d, M, steps, eta, sigma, policy, param, seed in [(100, 4, 30, 0.1, 0.0, 1, 0.5, 42), (64, 8, 10, 0.05, 0.1, 2, 0.6, 9),
                                                         (16, 3, 20, 0.05, 0.2, 2, 0.4, 99), (8, 2, 5, 0.2, 0.0, 0, 0.0, 7)]:
        diag = np.linspace(0.5, 2.0, d)
        theta0 = np.linspace(-1.0, 1.0, d)
        th, gs = ref.masked_sgd(diag, theta0, eta, M, steps, sigma, policy, param, seed)
        out.append({"d": d, "M": M, "steps": steps, "eta": eta, "sigma": sigma, "policy": policy, "param": param,
                    "seed": seed, "diag": hx(diag), "theta0": hx(theta0), "theta": hx(th), "grad_sq": hx(gs)})
    # MaskPolicy::plan_driven (sandbox.cpp:97-115): the reference's own LP plan of two fixtures,
    # AFR at a ramp step and at t_total
    fx = fixtures()
    plan_rows = []
    for name, d, steps, eta, sigma, step, seed in [("gpipe_s2m2", 40, 12, 0.05, 0.1, 15, 3),
                                                   ("default_1f1b_s4m8", 64, 8, 0.02, 0.0, -1, 21)]:
        f = fx[name]
        pl = f["pipeline"]
        R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
        t = f["timing"]["per_stage"]
        pr = ref.plan(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"], f["r_max"])
        phases = [2, 8, 10, 20]
        diag = np.linspace(0.5, 2.0, d)
        theta0 = np.linspace(-1.0, 1.0, d)
        th, gs = ref.masked_sgd_plan(diag, theta0, eta, M, steps, sigma, R * C, pr["ratios"], phases, step, seed)
        plan_rows.append({"fixture": name, "d": d, "M": M, "S": R * C, "steps": steps, "eta": eta, "sigma": sigma,
                          "ratios": hx(pr["ratios"]), "phases": phases, "step": step, "seed": seed, "diag": hx(diag),
                          "theta0": hx(theta0), "theta": hx(th), "grad_sq": hx(gs)})
    dump("sgd.json", {"runs": out, "plan_driven": plan_rows})


if __name__ == "__main__" and len(sys.argv) == 1:
    fx = fixtures()
    dump("fixtures.json", fx)
    gen_rng()
    gen_schedules()
    gen_phases()
    gen_masks(fx)
    gen_apf()
    gen_lp(fx)
    gen_monitor()
    gen_sgd()


def gen_artifacts(fx):
    """Reference JSON artifacts (plan.json, report.json, gantt timelines, mask history, timing profile)."""
    out = []
    for name in ("default_1f1b_s4m8", "gpipe_s2m2", "interleaved_r2c2m4", "zbv_r2m4"):
        f = fx[name]
        pl = f["pipeline"]
        R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
        S = R * C
        t = f["timing"]["per_stage"]
        plan_txt, report_txt = ref.plan_json(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"],
                                             t["backward_param_ms"], f["r_max"])
        n = 2 * M * S + 2
        w = np.array([0.0] + [t["forward_ms"]] * (M * S) + [t["backward_act_ms"] + t["backward_param_ms"]] * (M * S) + [0.0])
        pr = ref.plan(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"], t["backward_param_ms"], f["r_max"])
        masks_txt = ref.masks_json(M, S, [2, 8, 10, 20], pr["ratios"], 500, f["seed"])
        out.append({"fixture": name, "plan_json": plan_txt, "report_json": report_txt,
                    "gantt_json": ref.gantt_json(pl["schedule"], R, C, M, w),
                    "masks_json": masks_txt, "profile_json": ref.profile_json(M, S, t["forward_ms"], t["backward_act_ms"],
                                                                               t["backward_param_ms"])})
    dump("artifacts.json", out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "artifacts":
    gen_artifacts(fixtures())

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "lp_big":
    gen_lp_big()


def gen_boundary(fx):
    """Device-boundary case (tests/test_boundary_gpu.py): the reference's plan.json for the C1
    fixture, whose stage-2 row (8 ratios) is injected with pf_trainer_set_plan into a 1-stage,
    8-microbatch trainer of the tiny preset (160 units); the expected masks are the reference's
    run_freezing_masks words for that single stage (freezectl.cpp:185-211) over t = 1..T."""
    f = fx["default_1f1b_s4m8"]
    pl = f["pipeline"]
    R, C, M = pl["num_ranks"], pl["stages_per_rank"], pl["num_microbatches"]
    t = f["timing"]["per_stage"]
    plan_txt, _ = ref.plan_json(pl["schedule"], R, C, M, t["forward_ms"], t["backward_act_ms"],
                                t["backward_param_ms"], f["r_max"])
    doc = json.loads(plan_txt)
    ratios = np.zeros(M)
    for e in doc["ratios"]:
        if e["s"] == 2:
            ratios[e["m"] - 1] = e["r"]
    phases, n, seed, T = [1, 3, 4, 9], 160, 17, 9
    _, _, words = ref.freezing_masks(M, 1, phases, ratios, n, seed, 1, T)
    dump("boundary.json", {"fixture": "default_1f1b_s4m8", "plan_json": plan_txt, "stage": 2, "M": M,
                           "phases": phases, "n_units": n, "seed": seed, "steps": T,
                           "words": [[str(int(x)) for x in row] for row in words]})


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "boundary":
    gen_boundary(fixtures())
