"""TEST INFRASTRUCTURE ONLY — CPU restatement (pure Python / numpy) of the reference's
hot-path algorithms, used as a checker by tests/ and never by the product.

Each function cites the reference file:line it restates (paths relative to the
reference's proj/ directory). The restatement is pinned against tests/golden/*.json,
which oracle/gen_golden.py produces from the reference itself compiled in
oracle/_ref (tests/test_oracle_restatement.py).
"""
from __future__ import annotations

import heapq
import math

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


class Rng:
    """splitmix64 stream, include/pipefreeze/types.hpp:46-82."""

    def __init__(self, seed: int):
        self.state = seed if seed else GAMMA  # types.hpp:48

    def next_u64(self) -> int:  # types.hpp:50-56
        self.state = (self.state + GAMMA) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def unit(self) -> float:  # types.hpp:59
        return (self.next_u64() >> 11) * 2.0 ** -53

    def index_below(self, n: int) -> int:  # types.hpp:62-68
        if n == 0:
            raise ValueError("index_below: n must be positive")
        limit = MASK64 - MASK64 % n
        x = self.next_u64()
        while x >= limit:
            x = self.next_u64()
        return x % n

    def gaussian(self) -> float:  # types.hpp:73-78
        u1 = self.unit()
        u2 = self.unit()
        while u1 <= 0.0:
            u1 = self.unit()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)


def sample_mask(n: int, ratio: float, rng: Rng) -> list[int]:
    """Exact-count subset (sorted indices), src/freezectl.cpp:77-98 (partial Fisher-Yates)."""
    k = int(math.floor(ratio * n))
    if k == 0:
        return []
    pool = list(range(n))
    for i in range(k):
        j = i + rng.index_below(n - i)
        pool[i], pool[j] = pool[j], pool[i]
    return sorted(pool[:k])


def phase_of(t: int, plan) -> int:
    """src/freezectl.cpp:28-38; plan = (T_w, T_m, T_f, T_total); returns the Phase enum index."""
    tw, tm, tf, tt = plan
    if t < 1 or t > tt:
        raise ValueError("step outside horizon")
    tmid = tw + (tm - tw + 1) // 2
    if t <= tw:
        return 0
    if t == tm:
        return 3
    if t <= tmid:
        return 1
    if t < tm:
        return 2
    return 4 if t <= tf else 5


def actual_freeze_ratio(t: int, plan, r: float) -> float:
    """src/freezectl.cpp:40-47."""
    tw, tm, tf, tt = plan
    if tf == tm:
        return r
    ramp = float(t - tm) / float(tf - tm)
    return min(r, r * ramp)


def schedule(kind: str, R: int, C: int, M: int) -> list[list[tuple[int, int, int]]]:
    """Rank action lists (kind 0/1, microbatch, stage), src/schedule.cpp:48-197."""
    S = R * C

    def rank_of(s):  # schedule.cpp:48-64
        if kind in ("gpipe", "1f1b"):
            return s - 1
        if kind.startswith("interleaved"):
            return (s - 1) % R
        return s - 1 if s <= R else 2 * R - s

    order = []
    for r in range(R):
        stages = [s for s in range(1, S + 1) if rank_of(s) == r]
        if kind == "gpipe":  # schedule.cpp:77-86
            order.append([(0, m, r + 1) for m in range(1, M + 1)] + [(1, m, r + 1) for m in range(1, M + 1)])
            continue
        if kind == "zbv":
            order.append(None)
            continue
        fwd = [(0, m, s) for s in stages for m in range(1, M + 1)]  # schedule.cpp:117-120
        bwd = [(1, m, s) for s in reversed(stages) for m in range(1, M + 1)]
        warm = (C - 1) * M + min(R - r, M)  # schedule.cpp:123 (C = 1: :94)
        lst = fwd[:warm]
        f = min(warm, len(fwd))
        for b in bwd:
            lst.append(b)
            if f < len(fwd):
                lst.append(fwd[f])
                f += 1
        order.append(lst)
    if kind == "zbv":  # schedule.cpp:145-197 greedy rounds
        done, emitted = set(), set()
        order = [[] for _ in range(R)]
        total = 2 * M * S

        def ready(a):
            k, m, s = a
            if a in emitted:
                return False
            if k == 0:
                return not ((m > 1 and (0, m - 1, s) not in done) or (s > 1 and (0, m, s - 1) not in done))
            return not ((0, m, s) not in done or (m > 1 and (1, m - 1, s) not in done)
                        or (s < S and (1, m, s + 1) not in done))

        while len(emitted) < total:
            rnd = []
            for r in range(R):
                stages = sorted((s for s in range(1, S + 1) if rank_of(s) == r), reverse=True)
                pick = next(((k, m, s) for k in (1, 0) for s in stages for m in range(1, M + 1) if ready((k, m, s))),
                            None)
                if pick:
                    order[r].append(pick)
                    emitted.add(pick)
                    rnd.append(pick)
            if not rnd:
                raise RuntimeError("zbv stalled")
            done.update(rnd)
    return order


def dag(kind: str, R: int, C: int, M: int):
    """Edges (insertion order) and min-index Kahn order, src/dag.cpp:18-106."""
    S = R * C
    n = 2 * M * S + 2

    def idx(k, m, s):
        return 1 + (M * S if k else 0) + (s - 1) * M + (m - 1)

    edges, seen = [], set()

    def add(a, b):
        if (a, b) not in seen:
            seen.add((a, b))
            edges.append((a, b))

    add(0, idx(0, 1, 1))
    add(idx(1, M, 1), n - 1)
    for s in range(1, S + 1):
        for m in range(1, M + 1):
            if m < M:
                add(idx(0, m, s), idx(0, m + 1, s))
                add(idx(1, m, s), idx(1, m + 1, s))
            add(idx(0, m, s), idx(1, m, s))
            if s < S:
                add(idx(0, m, s), idx(0, m, s + 1))
            if s > 1:
                add(idx(1, m, s), idx(1, m, s - 1))
    for lst in schedule(kind, R, C, M):
        for a, b in zip(lst, lst[1:]):
            add(idx(*a), idx(*b))
    out = [[] for _ in range(n)]
    indeg = [0] * n
    for a, b in edges:
        out[a].append(b)
        indeg[b] += 1
    heap = [v for v in range(n) if indeg[v] == 0]
    heapq.heapify(heap)
    topo = []
    while heap:
        v = heapq.heappop(heap)
        topo.append(v)
        for w in out[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(heap, w)
    return edges, topo


def longest_path(edges, topo, weights) -> tuple[list[float], float]:
    """src/dag.cpp:142-161: start[w] = max(start[w], start[v] + w_v) in topological order."""
    n = len(topo)
    out = [[] for _ in range(n)]
    for a, b in edges:
        out[a].append(b)
    start = [0.0] * n
    for v in topo:
        for w in out[v]:
            start[w] = max(start[w], start[v] + weights[v])
    return start, start[n - 1]


def apf_update(ema: np.ndarray, ema_abs: np.ndarray, delta: np.ndarray, alpha: float) -> np.ndarray:
    """src/freezectl.cpp:147-156 (fp64): E <- aE + (1-a)d, E_abs <- aE_abs + (1-a)|d|, score |E|/E_abs."""
    ema *= alpha
    ema += (1.0 - alpha) * delta
    ema_abs *= alpha
    ema_abs += (1.0 - alpha) * np.abs(delta)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(ema_abs == 0.0, 1.0, np.abs(ema) / ema_abs)


def masked_sgd_update(theta: np.ndarray, grads: list[np.ndarray], update_masks: list[np.ndarray],
                      eta: float) -> np.ndarray:
    """src/sandbox.cpp:221,232-250: theta -= (eta/M) * sum_m U_m * g_m (divisor M, not the unfrozen count)."""
    total = np.zeros_like(theta)
    for g, u in zip(grads, update_masks):
        total += u * g
    return theta - (eta / len(grads)) * total
