"""Pins of the dense per-plan-table oracle (P:572-574,
P:608: profiled time per whole-segment plan) against things other than itself:

  * the already-pinned factored oracle: a dense table filled with each plan's
    factored cost (sum of p_j + c_j and intra reshards, written out here with
    numpy from the input tables) must give the factored (A, I) and plan;
  * an independent Python brute force over every global plan;
  * closed forms: no cross edges -> A[0][v] = min over the plans with s_o = v,
    I = least such index (numpy argmin on the reshaped table);
  * the synthetic generator is deterministic and prefix-consistent.
"""
import numpy as np
import pytest

from oracle import oracle as O
from synth import generators as G
from synth.problem import INF32


def _factored_dense(ty) -> np.ndarray:
    """W[idx] = sum_j (p_j + c_j)[s_j] + sum_edges R[s_a][s_b] (INF absorbing), by numpy broadcasting."""
    K = len(ty.radix)
    shape = tuple(int(d) for d in ty.radix)
    tot = np.zeros(shape, dtype=np.uint64)
    bad = np.zeros(shape, dtype=bool)
    for j in range(K):
        p = ty.comp(j).astype(np.uint64)
        c = ty.comm(j).astype(np.uint64)
        inf = (ty.comp(j) == INF32) | (ty.comm(j) == INF32)
        sh = [1] * K
        sh[j] = shape[j]
        tot = tot + (p + c).reshape(sh)
        bad = bad | inf.reshape(sh)
    for e in ty.edges:
        sh = [1] * K
        sh[e.src], sh[e.dst] = shape[e.src], shape[e.dst]
        tab = e.table if e.src < e.dst else e.table.T
        tot = tot + tab.astype(np.uint64).reshape(sh)
        bad = bad | (tab == INF32).reshape(sh)
    big = tot >= np.uint64(INF32)
    w = np.where(bad | big, np.uint64(INF32), tot).astype(np.uint32).ravel()
    return w, bool(big[~bad].any()) if (~bad).any() else False


@pytest.mark.parametrize("seed", range(60))
def test_dense_equals_factored(oracle_lib, seed):
    p = G.tiny_random(6000 + seed, mode="random")
    Ws = []
    for ty in p.types:
        w, overflow = _factored_dense(ty)
        if overflow:
            pytest.skip("factored plan cost does not fit uint32")
        Ws.append(w)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        A, I = O.segment_table(p, tr, m=m)
        Ad, Id = O.dense_segment_table(p, tr, Ws[p.transitions[tr].type], m=m)
        assert np.array_equal(A, Ad) and np.array_equal(I, Id)
    try:
        want = O.search_plan(p)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        with pytest.raises(O.OracleError):
            O.dense_search_plan(p, Ws)
        return
    got = O.dense_search_plan(p, Ws)
    assert got["total"] == want["total"]
    assert got["seg_index"].tolist() == want["seg_index"].tolist()
    assert got["seg_ns"].tolist() == want["seg_ns"].tolist()


@pytest.mark.parametrize("seed", range(120))
def test_dense_plan_equals_brute_force(oracle_lib, seed):
    p = G.tiny_random(6200 + seed, max_plans=20000)
    Ws = [G.dense_table(seed, t, p.num_combinations(t)) % np.uint32(97) if seed % 3 == 0
          else G.dense_table(seed, t, p.num_combinations(t)) for t in range(len(p.types))]
    for w in Ws:                       # a few infeasible plans in every table
        w[::7] = np.uint32(INF32)
    b = O.brute_force_dense(p, Ws, limit=20000)
    try:
        got = O.dense_search_plan(p, Ws)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE and b["total"] is None
        return
    assert got["total"] == b["total"]
    assert got["seg_index"].tolist() == b["seg_index"].tolist()


@pytest.mark.parametrize("seed", range(30))
def test_dense_closed_form_no_cross(oracle_lib, seed):
    p = G.tiny_random(6400 + seed, max_d=5)
    for tr in sorted({int(t) for t in p.instances}):
        T = p.transitions[tr]
        if T.in_edges:
            continue
        ty = p.types[T.type]
        W = G.dense_table(seed, T.type, p.num_combinations(T.type))
        A, I = O.dense_segment_table(p, tr, W)
        o = ty.out_block
        Wm = np.moveaxis(W.reshape(tuple(int(d) for d in ty.radix)), o, -1).reshape(-1, int(ty.radix[o]))
        # least index with the minimum: canonical order of the remaining digits is preserved by moveaxis
        idx = np.moveaxis(np.arange(W.size).reshape(W.shape[0] if False else tuple(int(d) for d in ty.radix)),
                          o, -1).reshape(-1, int(ty.radix[o]))
        mn = Wm.min(axis=0).astype(np.uint64)
        first = np.array([idx[np.flatnonzero(Wm[:, v] == Wm[:, v].min())[0], v] for v in range(Wm.shape[1])])
        for u in range(A.shape[0]):
            exp = np.where(mn == np.uint64(INF32), np.uint64(O.INF64), mn)
            assert np.array_equal(A[u], exp)
            expi = np.where(mn == np.uint64(INF32), np.uint64(O.NOIDX), first.astype(np.uint64))
            assert np.array_equal(I[u], expi)


def test_dense_generator_deterministic_and_windowed():
    a = G.dense_table(3, 2, 1000)
    assert np.array_equal(a, G.dense_table(3, 2, 1000))
    assert np.array_equal(a[400:700], G.dense_table(3, 2, 300, lo=400))
    assert not np.array_equal(a, G.dense_table(3, 1, 1000))
    assert (a == INF32).sum() < 10 and a[a != INF32].max() < (1 << 24)
