"""TEST INFRASTRUCTURE ONLY: ctypes view of the compiled reference (oracle/_ref/libpfref.so).

The library is the unmodified reference source (/root/reference/proj/src) built by
oracle/Makefile. Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline arm may use this module, and only as the checker or the timed
reference — never as a product code path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpfref.so")

KIND = {"gpipe": 0, "1f1b": 1, "interleaved-1f1b": 2, "interleaved": 2, "zbv": 3}

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_param_pass.restype = ctypes.c_double
        L.ref_param_pass.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int, ctypes.c_long, ctypes.c_double]
        L.ref_controller_step.restype = ctypes.c_double
        L.ref_controller_step.argtypes = [ctypes.c_int] * 5 + [ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p]
        L.ref_cpu_step.restype = ctypes.c_double
        L.ref_cpu_step.argtypes = [ctypes.c_int] * 5 + [ctypes.c_long, ctypes.c_double, ctypes.c_uint64]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def rng_u64(seed: int, n: int) -> list[int]:
    out = np.zeros(n, dtype=np.uint64)
    lib().ref_rng_u64(ctypes.c_uint64(seed), n, _p(out))
    return [int(x) for x in out]


def rng_mixed(seed: int, bounds: list[int]):
    n = len(bounds)
    b = np.array(bounds, dtype=np.uint64)
    idx = np.zeros(n, dtype=np.uint64)
    unit = np.zeros(n)
    gauss = np.zeros(n)
    _chk(lib().ref_rng_mixed(ctypes.c_uint64(seed), n, _p(b), _p(idx), _p(unit), _p(gauss)))
    return [int(x) for x in idx], unit.tolist(), gauss.tolist()


def schedule(kind: str, R: int, C: int, M: int) -> list[list[tuple[int, int, int]]]:
    per = 2 * M * C
    out = np.zeros(R * per * 3 + 3 * R, dtype=np.int32)
    lens = np.zeros(R, dtype=np.int32)
    _chk(lib().ref_schedule(KIND[kind], R, C, M, _p(out), _p(lens)))
    res, k = [], 0
    for r in range(R):
        lst = []
        for _ in range(int(lens[r])):
            lst.append((int(out[k]), int(out[k + 1]), int(out[k + 2])))
            k += 3
        res.append(lst)
    return res


def dag(kind: str, R: int, C: int, M: int, with_json: bool = False):
    n = 2 * M * R * C + 2
    cap = 8 * n
    edges = np.zeros(2 * cap, dtype=np.int32)
    ne = ctypes.c_int(0)
    topo = np.zeros(n, dtype=np.int32)
    jcap = 1 << 22 if with_json else 0
    buf = ctypes.create_string_buffer(jcap) if with_json else None
    _chk(lib().ref_dag(KIND[kind], R, C, M, _p(edges), cap, ctypes.byref(ne), _p(topo), buf, jcap))
    e = [(int(edges[2 * i]), int(edges[2 * i + 1])) for i in range(ne.value)]
    return e, topo.tolist(), (buf.value.decode() if with_json else None)


def longest_path(kind: str, R: int, C: int, M: int, weights: np.ndarray):
    n = 2 * M * R * C + 2
    w = np.ascontiguousarray(weights, dtype=np.float64)
    start = np.zeros(n)
    ms = ctypes.c_double(0)
    _chk(lib().ref_longest_path(KIND[kind], R, C, M, _p(w), _p(start), ctypes.byref(ms)))
    return start, ms.value


def phase_of(t: int, plan) -> int:
    p = np.array(plan, dtype=np.int32)
    return lib().ref_phase_of(t, _p(p))


def afr(t: int, plan, r: float) -> float:
    p = np.array(plan, dtype=np.int32)
    out = ctypes.c_double(0)
    _chk(lib().ref_afr(t, _p(p), ctypes.c_double(r), ctypes.byref(out)))
    return out.value


def sample_masks(seed: int, n: int, ratios) -> np.ndarray:
    r = np.array(ratios, dtype=np.float64)
    words = (n + 63) // 64
    out = np.zeros(len(r) * max(words, 1), dtype=np.uint64)
    _chk(lib().ref_sample_masks(ctypes.c_uint64(seed), n, len(r), _p(r), _p(out)))
    return out.reshape(len(r), max(words, 1))[:, :words]


def reconcile(seed: int, n: int, base_words: np.ndarray, target: int) -> np.ndarray:
    words = (n + 63) // 64
    b = np.ascontiguousarray(base_words, dtype=np.uint64)
    out = np.zeros(words, dtype=np.uint64)
    _chk(lib().ref_reconcile(ctypes.c_uint64(seed), n, _p(b), target, _p(out)))
    return out


def freezing_masks(M, S, plan, ratios, n, seed, t_from=1, t_to=0):
    p = np.array(plan, dtype=np.int32)
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    cells = plan[3] * S * M
    pop = np.zeros(cells, dtype=np.int32)
    sc = np.zeros(S * n, dtype=np.int64)
    nsel = max(0, t_to - t_from + 1) * S * M
    words = (n + 63) // 64
    w = np.zeros(max(1, nsel * words), dtype=np.uint64)
    _chk(lib().ref_freezing_masks(M, S, _p(p), _p(r), n, ctypes.c_uint64(seed), _p(pop), _p(sc),
                                  t_from, t_to, _p(w) if nsel else None))
    return pop, sc.reshape(S, n), w[: nsel * words].reshape(nsel, words) if nsel else None


def apf(n: int, alpha: float, deltas: np.ndarray):
    d = np.ascontiguousarray(deltas, dtype=np.float64)
    steps = d.shape[0]
    e, ea, s = np.zeros(n), np.zeros(n), np.zeros(n)
    _chk(lib().ref_apf(n, ctypes.c_double(alpha), steps, _p(d), _p(e), _p(ea), _p(s)))
    return e, ea, s


def plan(kind, R, C, M, fwd, bact, bparam, r_max, lambda_mode=0, budget_all=0):
    S = R * C
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)).copy()
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)).copy()
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)).copy()
    ratios = np.zeros(S * M)
    dur = np.zeros(2 * S * M)
    out5 = np.zeros(5)
    savg = np.zeros(S)
    secs = ctypes.c_double(0)
    _chk(lib().ref_plan(KIND[kind], R, C, M, _p(f), _p(a), _p(b), ctypes.c_double(r_max), lambda_mode, budget_all,
                        _p(ratios), _p(dur), _p(out5), _p(savg), ctypes.byref(secs)))
    return dict(ratios=ratios, durations=dur, makespan_base=out5[0], makespan_opt=out5[1],
                makespan_floor=out5[2], lp_makespan=out5[3], iterations=int(out5[4]),
                stage_avg=savg, solve_seconds=secs.value)


def verify(kind, R, C, M, fwd, bact, bparam, r_max, ratios, durations, makespan_opt):
    S = R * C
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)).copy()
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)).copy()
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)).copy()
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    d = np.ascontiguousarray(durations, dtype=np.float64)
    ok = ctypes.c_int(0)
    rec = ctypes.c_double(0)
    _chk(lib().ref_verify(KIND[kind], R, C, M, _p(f), _p(a), _p(b), ctypes.c_double(r_max), _p(r), _p(d),
                          ctypes.c_double(makespan_opt), ctypes.byref(ok), ctypes.byref(rec)))
    return bool(ok.value), rec.value


def monitor(M, S, fwd, bact, bparam, plan, sigma, seed):
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)).copy()
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)).copy()
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)).copy()
    p = np.array(plan, dtype=np.int32)
    wmin = np.zeros(2 * S * M)
    wmax = np.zeros(2 * S * M)
    _chk(lib().ref_monitor(M, S, _p(f), _p(a), _p(b), _p(p), ctypes.c_double(sigma), ctypes.c_uint64(seed),
                           _p(wmin), _p(wmax)))
    return wmin, wmax


def masked_sgd(diag, theta0, eta, M, steps, sigma, policy, param, seed):
    d = len(diag)
    dg = np.ascontiguousarray(diag, dtype=np.float64)
    t0 = np.ascontiguousarray(theta0, dtype=np.float64)
    th = np.zeros(d)
    gs = np.zeros(steps)
    _chk(lib().ref_masked_sgd(d, _p(dg), _p(t0), ctypes.c_double(eta), M, steps, ctypes.c_double(sigma), policy,
                              ctypes.c_double(param), ctypes.c_uint64(seed), _p(th), _p(gs)))
    return th, gs


def masked_sgd_plan(diag, theta0, eta, M, steps, sigma, S, ratios, phases, step, seed):
    """run_masked_sgd with MaskPolicy::plan_driven (sandbox.cpp:97-115)."""
    d = len(diag)
    dg = np.ascontiguousarray(diag, dtype=np.float64)
    t0 = np.ascontiguousarray(theta0, dtype=np.float64)
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    ph = np.ascontiguousarray(phases, dtype=np.int32)
    th = np.zeros(d)
    gs = np.zeros(steps)
    _chk(lib().ref_masked_sgd_plan(d, _p(dg), _p(t0), ctypes.c_double(eta), M, steps, ctypes.c_double(sigma), S,
                                   _p(r), _p(ph), step, ctypes.c_uint64(seed), _p(th), _p(gs)))
    return th, gs


def autofreeze_score(prev: float, cur: float) -> float:
    f = lib().ref_autofreeze_score
    f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double, ctypes.c_double]
    return f(prev, cur)


def autofreeze_select(scores, prefix: int, pct: float) -> int:
    sc = np.ascontiguousarray(scores, dtype=np.float64)
    out = ctypes.c_int(0)
    _chk(lib().ref_autofreeze_select(_p(sc), len(sc), prefix, ctypes.c_double(pct), ctypes.byref(out)))
    return out.value


def param_pass_seconds(begin, end, block, masks, per_unit, lr=0.01) -> float:
    """ref_param_pass: elements [begin, end) of the reference per-parameter step (apf_update +
    masked accumulation + SGD) over the M x words masks."""
    m = np.ascontiguousarray(masks, dtype=np.uint64)
    return lib().ref_param_pass(begin, end, block, m.shape[0], _p(m), m.shape[1], per_unit, lr)


def controller_step(kind, R, C, M, n_units, ratio, seed=42):
    """ref_controller_step: schedule + DAG + longest path + S*M sample_mask; (seconds, stage-1 masks)."""
    out = np.zeros((M, (n_units + 63) // 64), dtype=np.uint64)
    secs = lib().ref_controller_step(KIND[kind], R, C, M, n_units, ratio, seed, _p(out))
    return secs, out


def cpu_step_seconds(kind, R, C, M, n_units, n_params, ratio, seed=42) -> float:
    return lib().ref_cpu_step(KIND[kind], R, C, M, n_units, n_params, ratio, seed)


def _text(fn, *args, cap=1 << 24):
    buf = ctypes.create_string_buffer(cap)
    _chk(fn(*args, buf, cap))
    return buf.value.decode()


def plan_json(kind, R, C, M, fwd, bact, bparam, r_max):
    """freeze_plan_to_json_text + throughput_report_to_json_text of the reference plan (config.cpp:188-257)."""
    S = R * C
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)).copy()
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)).copy()
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)).copy()
    pb = ctypes.create_string_buffer(1 << 22)
    rb = ctypes.create_string_buffer(1 << 20)
    _chk(lib().ref_plan_json(KIND[kind], R, C, M, _p(f), _p(a), _p(b), ctypes.c_double(r_max), pb, 1 << 22, rb, 1 << 20))
    return pb.value.decode(), rb.value.decode()


def gantt_json(kind, R, C, M, weights):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    return _text(lib().ref_gantt_json, KIND[kind], R, C, M, _p(w))


def masks_json(M, S, plan, ratios, n, seed):
    p = np.array(plan, dtype=np.int32)
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    return _text(lib().ref_masks_json, M, S, _p(p), _p(r), n, ctypes.c_uint64(seed))


def profile_json(M, S, fwd, bact, bparam):
    f = np.broadcast_to(np.asarray(fwd, dtype=np.float64), (S,)).copy()
    a = np.broadcast_to(np.asarray(bact, dtype=np.float64), (S,)).copy()
    b = np.broadcast_to(np.asarray(bparam, dtype=np.float64), (S,)).copy()
    return _text(lib().ref_profile_json, M, S, _p(f), _p(a), _p(b))
