"""Oracle for SURVEY §8(f) NEXT-3: the profiling space (Eq. 2) and the dynamic
profiling time budget.

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench.py's cpu_baseline /
`--impl reference` legs, never by the product package.  Plain Python and
numpy; shares no code with the CUDA path.

Eq. 2: the number of programs to compile and profile is
    sum_i ( prod_j S_{i,j} + sum_j sum_{(l,k) in D_{i,j}} S_{i,l} * S_{j,k} )
over the N distinct segments i.  In this repo's problem model a distinct
segment is a segment type (its K blocks have radices D_j = S_{i,j}); a
cross-segment dependency pair (l, k) of segments (i, j) is a cross edge of
the transition (i -> j) from i's output block l to j's consumer block k
(SURVEY Q2), so its term is D_in * D_k.

Budget ("a dynamic profiling time budget, which is continuously
updated based on the fastest observed parallelism plans, aggressively
trimming the profiling of inefficient or stalled executions"; S:411-419
"abandoned and marked pruned once its accumulating cost exceeds f x best
completed cost for the same segment type").  Readings (DESIGN.md R-B1..R-B4):
  R-B1  the plan tasks of one type run one after another in canonical
        (big-endian mixed-radix) index order; `best` before task i is the
        least finite cost among the completed tasks 0..i-1, which equals the
        least finite cost among all of them because f >= 1 (a pruned task
        exceeded f x best >= best, so it could not have lowered it);
  R-B2  f = num / den (integers, 1 <= den <= num <= 65535); task i is pruned
        iff a best exists and W[i] * den > best * num (exact integer
        comparison); a pruned task costs its budget floor(best * num / den)
        of profiling time;
  R-B3  CFP_INF32 entries are infeasible programs (e.g. out of memory): they
        cost no profiling time, are never pruned and never become the best;
  R-B4  the best is reported with the least index attaining it.
"""
from __future__ import annotations

from typing import Dict, Iterator, List, Tuple

import numpy as np

from synth.problem import INF32, Problem

INF64 = (1 << 64) - 1
NOIDX = INF64


# ---------------------------------------------------------------- Eq. 2


def profile_space(prob: Problem) -> Dict:
    """Eq. 2 term by term.  Returns the left term per distinct segment
    (`type_plans[i]` = prod_j S_{i,j}), the right term per dependent segment
    pair (`trans_pairs[x]` = sum over the cross edges of transition x of
    S_{pred, out} * S_{type, k}; 0 for a chain start) and their sum."""
    type_plans = []
    for ty in prob.types:
        n = 1
        for d in ty.radix:
            n *= int(d)
        type_plans.append(n)
    trans_pairs = []
    for x, tr in enumerate(prob.transitions):
        if tr.pred_type < 0:
            trans_pairs.append(0)
            continue
        pt = prob.types[tr.pred_type]
        s_l = int(pt.radix[pt.out_block])
        ty = prob.types[tr.type]
        trans_pairs.append(sum(s_l * int(ty.radix[e.dst]) for e in tr.in_edges))
    return dict(type_plans=type_plans, trans_pairs=trans_pairs,
                total=sum(type_plans) + sum(trans_pairs))


def profile_tasks(prob: Problem) -> Iterator[Tuple]:
    """The task list itself (tiny problems): ("plan", type, index) for every
    whole-segment plan, then ("reshard", transition, edge, s_l, s_k) for every
    strategy pair of every cross-segment dependency."""
    for t, ty in enumerate(prob.types):
        n = 1
        for d in ty.radix:
            n *= int(d)
        for idx in range(n):
            yield ("plan", t, idx)
    for x, tr in enumerate(prob.transitions):
        if tr.pred_type < 0:
            continue
        pt = prob.types[tr.pred_type]
        s_l = int(pt.radix[pt.out_block])
        for e_i, e in enumerate(tr.in_edges):
            for a in range(s_l):
                for b in range(int(prob.types[tr.type].radix[e.dst])):
                    yield ("reshard", x, e_i, a, b)


# ---------------------------------------------------------------- budget


def budget_loop(W, num: int, den: int) -> Dict:
    """R-B1..R-B4 as a plain sequential loop (small inputs)."""
    if not (1 <= den <= num <= 65535):
        raise ValueError("budget factor num/den: need 1 <= den <= num <= 65535")
    best, best_idx = None, NOIDX
    pruned = infeasible = spent = full = 0
    for i, w in enumerate(np.asarray(W, dtype=np.uint32).tolist()):
        if w == INF32:
            infeasible += 1
            continue
        full += w
        if best is not None and w * den > best * num:
            pruned += 1
            spent += best * num // den
            continue
        spent += w
        if best is None or w < best:
            best, best_idx = w, i
    return dict(tasks=len(W), pruned=pruned, infeasible=infeasible, spent=spent, full=full,
                best=INF64 if best is None else best, best_index=best_idx)


def budget(W, num: int, den: int) -> Dict:
    """The same definition with numpy primitives (any size that fits host
    memory): best-before-i is an exclusive prefix minimum
    (np.minimum.accumulate) with CFP_INF32 as the identity (R-B3)."""
    if not (1 <= den <= num <= 65535):
        raise ValueError("budget factor num/den: need 1 <= den <= num <= 65535")
    W = np.asarray(W, dtype=np.uint32)
    n = int(W.size)
    if n == 0:
        return dict(tasks=0, pruned=0, infeasible=0, spent=0, full=0, best=INF64, best_index=NOIDX)
    incl = np.minimum.accumulate(W)
    prev = np.empty(n, dtype=np.uint64)
    prev[0] = INF32
    prev[1:] = incl[:-1]
    W64 = W.astype(np.uint64)
    finite = W != np.uint32(INF32)
    has_best = prev != np.uint64(INF32)
    pruned = finite & has_best & (W64 * np.uint64(den) > prev * np.uint64(num))
    budget_ns = (prev * np.uint64(num)) // np.uint64(den)
    cost = np.where(pruned, budget_ns, np.where(finite, W64, np.uint64(0)))
    best = int(incl[-1])
    if best == INF32:
        best_out, best_idx = INF64, NOIDX
    else:
        best_out, best_idx = best, int(np.argmax(W == np.uint32(best)))
    # exact sums: per-element values < 2^48, chunks of <= ~2^14 elements in uint64
    spent = sum(int(c.sum(dtype=np.uint64)) for c in np.array_split(cost, max(1, n >> 14)))
    fullv = np.where(finite, W64, np.uint64(0))
    full = sum(int(c.sum(dtype=np.uint64)) for c in np.array_split(fullv, max(1, n >> 14)))
    return dict(tasks=n, pruned=int(pruned.sum()), infeasible=int((~finite).sum()), spent=spent,
                full=full, best=best_out, best_index=best_idx)
