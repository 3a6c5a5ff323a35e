"""Variable-batch dynamic program and the fixed-batch baseline
(P:L756-757), plus a brute-force chain enumerator that pins the DP.

Definitions:
  Time(i,B), IN(i,B), OUT(i,B), WS(i), TOT.
  <i,B,A> feasible  <=>  A + IN(i,B) + WS(i) + OUT(i,B) <= TOT.
Recurrence:
  OPT(1,B,A) = Time(1,B) if feasible else inf
  OPT(i,B,A) = Time(i,B) + min_{b <= B, b | B} (B/b) * OPT(i-1, b, A + IN(i, B-b))
               subject to <i,B,A> feasible
Objective: min_B OPT(f,B,0) / B.
Latency extension: OPT(i,B,A) <- inf when it exceeds the threshold.
Remainder: if the chosen B* does not divide K, run floor(K/B*) rounds
  and plan again for the remaining K mod B* inputs.
Readings: C-26 ties -> larger b, then larger B; C-27 latency = OPT(f,B,0);
C-32 batch grid = 1..K for the DP, fixed baseline over all of 1..K.
The oracle DP uses EXACT byte values of A (memoised top-down).
"""
from __future__ import annotations

import dataclasses
import functools
import math
from typing import Dict, List, Optional, Sequence, Tuple

INF = math.inf


@dataclasses.dataclass
class Problem:
    time: Sequence[Dict[int, float]]   # time[i][B] for i = 0..f-1 (layer L_{i+1})
    in_bytes: Sequence[int]            # IN(i,B) = in_bytes[i] * B
    out_bytes: Sequence[int]           # OUT(i,B) = out_bytes[i] * B
    ws: Sequence[int]                  # WS(i)
    tot: int                           # TOT
    latency: Optional[float] = None    # threshold (ms or any unit of time)

    @property
    def f(self) -> int:
        return len(self.time)

    def IN(self, i: int, B: int) -> int:
        return self.in_bytes[i] * B

    def OUT(self, i: int, B: int) -> int:
        return self.out_bytes[i] * B

    def feasible(self, i: int, B: int, A: int) -> bool:
        return A + self.IN(i, B) + self.ws[i] + self.OUT(i, B) <= self.tot


@dataclasses.dataclass
class Plan:
    batches: List[int]          # B_1..B_f
    time: float                 # OPT(f, B_f, 0)  (one outermost batch)
    per_image: float            # time / B_f


def divisors(B: int) -> List[int]:
    return [b for b in range(1, B + 1) if B % b == 0]


def dp_plan(p: Problem, Bmax: int) -> Optional[Plan]:
    """The recurrence of P:L694-710, memoised over exact A, batch grid 1..Bmax."""

    @functools.lru_cache(maxsize=None)
    def opt(i: int, B: int, A: int) -> Tuple[float, int]:
        if not p.feasible(i, B, A):
            return INF, 0
        if i == 0:
            v = p.time[0][B]
            best_b = 0
        else:
            best, best_b = INF, 0
            for b in sorted(divisors(B), reverse=True):          # C-26: larger b first
                sub, _ = opt(i - 1, b, A + p.IN(i, B - b))
                cand = (B // b) * sub
                if cand < best:
                    best, best_b = cand, b
            v = p.time[i][B] + best if best < INF else INF
        if p.latency is not None and v > p.latency:
            v = INF
        return v, best_b

    best: Optional[Plan] = None
    for B in range(Bmax, 0, -1):                                 # C-26: larger B on ties
        v, _ = opt(p.f - 1, B, 0)
        if v == INF:
            continue
        if best is None or v / B < best.per_image:
            # backtrack
            batches = [B]
            A = 0
            Bi = B
            for i in range(p.f - 1, 0, -1):
                _, b = opt(i, Bi, A)
                A = A + p.IN(i, Bi - b)
                Bi = b
                batches.append(b)
            best = Plan(batches[::-1], v, v / B)
    opt.cache_clear()
    return best


def chain_cost(p: Problem, batches: Sequence[int]) -> float:
    """Closed form of the unrolled recurrence for a divisor chain
    B_1 | B_2 | ... | B_f (SURVEY §8(c) planner pin):
      OPT_i = Time(i,B_i) + (B_i/B_{i-1}) OPT_{i-1}
      A_f = 0, A_{j-1} = A_j + IN(j, B_j - B_{j-1})
      feasible iff A_j + IN(j,B_j) + WS(j) + OUT(j,B_j) <= TOT for all j
    Returns INF when infeasible or over the latency threshold."""
    f = p.f
    A = [0] * f
    for j in range(f - 1, 0, -1):
        A[j - 1] = A[j] + p.IN(j, batches[j] - batches[j - 1])
    for j in range(f):
        if not p.feasible(j, batches[j], A[j]):
            return INF
    t = 0.0
    for j in range(f):
        t = p.time[j][batches[j]] + ((batches[j] // batches[j - 1]) * t if j > 0 else 0.0)
        if p.latency is not None and t > p.latency:
            return INF
    return t


def brute_force(p: Problem, Bmax: int) -> Optional[Plan]:
    """Enumerate every monotone divisor chain with B_f <= Bmax."""
    best: Optional[Plan] = None

    def rec(j: int, suffix: List[int]):
        nonlocal best
        if j < 0:
            chain = suffix[::-1]
            t = chain_cost(p, chain)
            if t < INF:
                per = t / chain[-1]
                if best is None or per < best.per_image:
                    best = Plan(list(chain), t, per)
            return
        for b in divisors(suffix[-1]):
            rec(j - 1, suffix + [b])

    for B in range(1, Bmax + 1):
        rec(p.f - 2, [B])
    return best


def fixed_batch(p: Problem, Bmax: int) -> Optional[Plan]:
    """Baseline: one B for every layer such that (i) no layer
    violates the memory constraint at that B and (ii) throughput is maximal."""
    best: Optional[Plan] = None
    for B in range(1, Bmax + 1):
        if not all(p.feasible(i, B, 0) for i in range(p.f)):
            continue
        t = sum(p.time[i][B] for i in range(p.f))
        if p.latency is not None and t > p.latency:
            continue
        if best is None or t / B < best.per_image:
            best = Plan([B] * p.f, t, t / B)
    return best


def plan_requests(p: Problem, K: int, planner=dp_plan) -> Tuple[List[Tuple[int, Plan]], float]:
    """Plan K requested inputs: floor(K/B*) rounds of the best plan, then plan
    again for the remainder.  Returns ([(rounds, plan), ...], total)."""
    out: List[Tuple[int, Plan]] = []
    total = 0.0
    while K > 0:
        pl = planner(p, K)
        if pl is None:
            raise ValueError("infeasible")
        B = pl.batches[-1]
        rounds = K // B
        out.append((rounds, pl))
        total += rounds * pl.time
        K -= rounds * B
    return out, total


def table_bytes(f: int, n_batch: int, tot: int, step: int, cell_bytes: int = 4) -> int:
    """Size of a discretised OPT table: f x |B grid| x |A grid| cells."""
    return f * n_batch * (tot // step) * cell_bytes
