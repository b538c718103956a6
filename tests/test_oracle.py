"""Pins for the CPU oracle (runs without a GPU).

The oracle is checked against things other than itself (task ③):
  * hand-worked examples with citations (tests/golden/*.json);
  * closed forms that reduce to numpy library reductions;
  * the chain DP against scipy's shortest path on the layered DAG;
  * the min-plus product against numpy broadcasting;
  * an independent pure-Python brute force over all global plans.
"""
import numpy as np
import pytest

from golden_util import load, problem_from
from synth import generators as G
from synth.problem import INF32, CrossEdge, Edge, Problem, SegmentType, Transition

INF64 = (1 << 64) - 1


# ---------------------------------------------------------------- golden
def test_h1_tables_chain_plan(oracle_lib):
    O = oracle_lib
    g = load("h1")
    p = problem_from(g["problem"])
    for tr in ("0", "1"):
        A, I = O.segment_table(p, int(tr))
        assert A.tolist() == g["expect"]["A"][tr]
        assert I.tolist() == g["expect"]["I"][tr]
    A0, I0 = O.segment_table(p, 0)
    A1, I1 = O.segment_table(p, 1)
    Gs = O.chain([A0, A1])
    assert Gs[1].tolist() == g["expect"]["G1"]
    assert int(Gs[0][0]) == g["expect"]["total"]
    r = O.search_plan(p)
    assert r["total"] == g["expect"]["total"]
    assert r["seg_index"].tolist() == g["expect"]["seg_index"]
    assert r["seg_ns"].tolist() == g["expect"]["seg_ns"]
    assert r["digits"].tolist() == g["expect"]["digits"]


@pytest.mark.parametrize("name", ["h2", "h2p"])
def test_spec_crafted_example(oracle_lib, name):
    O = oracle_lib
    g = load(name)
    p = problem_from(g["problem"])
    r = O.search_plan(p)
    assert r["total"] == g["expect"]["total"]
    assert r["seg_index"].tolist() == g["expect"]["seg_index"]
    assert r["seg_ns"].tolist() == g["expect"]["seg_ns"]
    m = O.Marshalled(p)
    for key, T in g["expect"]["all_plans"].items():
        a, b = (int(x) for x in key.split(","))
        # Eq. 3 for the two-segment plan (a, b): C_1(0, a) + C_2(a, b)
        assert O.cost_index(p, 0, 0, a, m) + O.cost_index(p, 1, a, b, m) == T
        assert O.py_cost(p, 0, 0, [a]) + O.py_cost(p, 1, a, [b]) == T
    bf = O.brute_force(p)
    assert bf["total"] == g["expect"]["total"]
    assert bf["seg_index"].tolist() == g["expect"]["seg_index"]


def test_h3_merge_invariance(oracle_lib):
    O = oracle_lib
    g = load("h3")
    p = problem_from(g["problem"])
    r = O.search_plan(p)
    assert r["total"] == g["expect"]["total"]
    assert r["seg_index"].tolist() == g["expect"]["seg_index"]
    assert r["digits"].tolist() == g["expect"]["digits"]
    h1 = O.search_plan(problem_from(load("h1")["problem"]))
    assert h1["total"] == r["total"]
    assert h1["digits"].ravel().tolist() == r["digits"].ravel().tolist()


def test_cx_canonical_not_midpoint(oracle_lib):
    O = oracle_lib
    g = load("cx")
    mats = [np.array(M, np.uint64) for M in g["chain"]["mats"]]
    idxs = [np.tile(np.arange(M.shape[1], dtype=np.uint64), (M.shape[0], 1)) for M in mats]
    Gs = O.chain(mats)
    assert [x.tolist() for x in Gs] == g["expect"]["G"]
    v, ix, cost = O.reconstruct(mats, idxs, Gs)
    assert v.tolist() == g["expect"]["v"]
    assert int(cost.sum()) == g["expect"]["total"]


def test_paper_counts():
    """P:815-817 and P:591 counts on the generated C2 structure."""
    g = load("counts")["expect"]
    p = G.make_config("C2")
    L = p.types[2]
    assert p.num_combinations(2) == g["plans_per_gpt_segment"]
    # Eq. 2: per distinct layer segment prod S_j, plus per layer transition
    # (L1->L, L->L) the cross pairs S_out * S_in (boundary-only, J_in={0}).
    layer_types = [1, 2]
    layer_trans = [2, 3]
    n = sum(p.num_combinations(t) for t in layer_types)
    for t in layer_trans:
        tr = p.transitions[t]
        for x in tr.in_edges:
            n += x.table.shape[0] * x.table.shape[1]
    assert n == g["programs_c2"]
    # best case (single repeated segment, last -> first dependency) = 81 + 9
    assert p.num_combinations(2) + int(L.radix[0]) * int(L.radix[-1]) == g["best_case_single_segment"]


# ---------------------------------------------------------------- closed forms
def _rand_type(rng, K, D, edges=(), o=None, inf=False, comm=True):
    radix = np.array(D, np.int32)
    sD = int(radix.sum())
    comp = rng.integers(0, 1000, sD).astype(np.uint32)
    cm = rng.integers(0, 1000, sD).astype(np.uint32) if comm else None
    if inf:
        comp[rng.random(sD) < 0.15] = INF32
    E = [Edge(a, b, rng.integers(0, 1000, (D[a], D[b])).astype(np.uint32)) for a, b in edges]
    return SegmentType(radix, comp, cm, E, int(rng.integers(0, K)) if o is None else o)


def _w(ty, j):
    p = ty.comp(j).astype(np.float64)
    c = ty.comm(j).astype(np.float64)
    w = p + c
    w[(ty.comp(j) == INF32) | (ty.comm(j) == INF32)] = np.inf
    return w


@pytest.mark.parametrize("seed", range(12))
def test_closed_form_separable(oracle_lib, seed):
    """(i) no edges, no cross terms: A[u][v] = sum_{j!=o} min w_j + w_o[v];
    I = per-block first argmins composed big-endian."""
    O = oracle_lib
    rng = np.random.default_rng(seed)
    K = int(rng.integers(1, 4))
    D = [int(x) for x in rng.integers(1, 5, K)]
    ty = _rand_type(rng, K, D, inf=seed % 2 == 1)
    p = Problem((1,), [ty], [Transition(-1, 0, [])], np.array([0], np.int32))
    A, I = O.segment_table(p, 0)
    o = ty.out_block
    rest = sum(np.min(_w(ty, j)) for j in range(K) if j != o)
    for v in range(D[o]):
        exp = rest + _w(ty, o)[v]
        if np.isinf(exp):
            assert int(A[0, v]) == INF64 and int(I[0, v]) == INF64
            continue
        assert int(A[0, v]) == int(exp)
        idx = 0
        for j in range(K):
            dj = v if j == o else int(np.argmin(_w(ty, j)))
            idx = idx * D[j] + dj
        assert int(I[0, v]) == idx


@pytest.mark.parametrize("seed", range(8))
def test_closed_form_single_block(oracle_lib, seed):
    """(ii) K = 1 with one cross edge: A[u][v] = Q[u][v] + w[v], I[u][v] = v."""
    O = oracle_lib
    rng = np.random.default_rng(100 + seed)
    d_in, d = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    pred = SegmentType(np.array([d_in], np.int32), np.zeros(d_in, np.uint32), None, [], 0)
    ty = _rand_type(rng, 1, [d], o=0)
    Q = rng.integers(0, 1000, (d_in, d)).astype(np.uint32)
    Q[rng.random((d_in, d)) < 0.2] = INF32
    p = Problem((1,), [pred, ty], [Transition(-1, 0, []), Transition(0, 1, [CrossEdge(0, Q)])],
                np.array([0, 1], np.int32))
    A, I = O.segment_table(p, 1)
    Qf = Q.astype(np.float64)
    Qf[Q == INF32] = np.inf
    exp = Qf + _w(ty, 0)[None, :]
    for u in range(d_in):
        for v in range(d):
            if np.isinf(exp[u, v]):
                assert int(A[u, v]) == INF64 and int(I[u, v]) == INF64
            else:
                assert int(A[u, v]) == int(exp[u, v]) and int(I[u, v]) == v


@pytest.mark.parametrize("direction", ["fwd", "bwd"])
@pytest.mark.parametrize("seed", range(6))
def test_closed_form_one_edge(oracle_lib, seed, direction):
    """(iv) K = 2, one (asymmetric) edge, o = 1: A[v] = min_{s0} w0[s0] + w1[v]
    + R(s0, v) -- numpy min/argmin over the broadcast sum; catches a
    transposed R or a dropped term."""
    O = oracle_lib
    rng = np.random.default_rng(200 + seed)
    D = [int(x) for x in rng.integers(2, 6, 2)]
    e = (0, 1) if direction == "fwd" else (1, 0)
    ty = _rand_type(rng, 2, D, edges=[e], o=1)
    p = Problem((1,), [ty], [Transition(-1, 0, [])], np.array([0], np.int32))
    A, I = O.segment_table(p, 0)
    R = ty.edges[0].table.astype(np.float64)
    Rs = R if direction == "fwd" else R.T          # indexed [s0][s1]
    tot = _w(ty, 0)[:, None] + _w(ty, 1)[None, :] + Rs
    for v in range(D[1]):
        assert int(A[0, v]) == int(np.min(tot[:, v]))
        assert int(I[0, v]) == int(np.argmin(tot[:, v])) * D[1] + v


@pytest.mark.parametrize("seed", range(6))
def test_closed_form_all_equal(oracle_lib, seed):
    """(iii) all costs equal: I[u][v] = lowest index of bucket v = v * stride_o."""
    O = oracle_lib
    rng = np.random.default_rng(300 + seed)
    K = int(rng.integers(1, 4))
    D = [int(x) for x in rng.integers(1, 5, K)]
    edges = [(0, K - 1)] if K > 1 else []
    ty = _rand_type(rng, K, D, edges=edges)
    ty.comp_ns[:] = 7
    ty.comm_ns[:] = 0
    for e in ty.edges:
        e.table[:] = 1
    p = Problem((1,), [ty], [Transition(-1, 0, [])], np.array([0], np.int32))
    A, I = O.segment_table(p, 0)
    o = ty.out_block
    stride = int(np.prod(D[o + 1:])) if o + 1 < K else 1
    for v in range(D[o]):
        assert int(A[0, v]) == 7 * K + len(edges)
        assert int(I[0, v]) == v * stride


# ---------------------------------------------------------------- chain / min-plus
def _rand_mats(rng, N, inf_p=0.2, maxv=50):
    dims = [1] + [int(x) for x in rng.integers(1, 5, N)]
    mats = []
    for n in range(N):
        M = rng.integers(0, maxv, (dims[n], dims[n + 1])).astype(np.uint64)
        M[rng.random(M.shape) < inf_p] = np.uint64(INF64)
        mats.append(M)
    return mats


@pytest.mark.parametrize("seed", range(20))
def test_chain_vs_scipy_shortest_path(oracle_lib, seed):
    from scipy.sparse.csgraph import csgraph_from_dense, dijkstra
    O = oracle_lib
    rng = np.random.default_rng(400 + seed)
    N = int(rng.integers(1, 7))
    mats = _rand_mats(rng, N)
    # layered DAG: node 0 = source (u_1 = 0), then each layer's states, then sink
    sizes = [M.shape[1] for M in mats]
    base = np.cumsum([1] + sizes)
    n_nodes = int(base[-1]) + 1
    Wd = np.full((n_nodes, n_nodes), np.inf)
    prev_nodes = [0]
    for n, M in enumerate(mats):
        cur = [int(base[n]) + v for v in range(M.shape[1])]
        for u, pu in enumerate(prev_nodes):
            for v, cv in enumerate(cur):
                if int(M[u, v]) != INF64:
                    Wd[pu, cv] = float(M[u, v])
        prev_nodes = cur
    for pu in prev_nodes:
        Wd[pu, n_nodes - 1] = 0.0
    dist = dijkstra(csgraph_from_dense(Wd, null_value=np.inf), indices=0)[n_nodes - 1]
    Gs = O.chain(mats)
    if np.isinf(dist):
        assert int(Gs[0][0]) == INF64
    else:
        assert int(Gs[0][0]) == int(dist)


@pytest.mark.parametrize("seed", range(10))
def test_minplus_vs_numpy(oracle_lib, seed):
    O = oracle_lib
    rng = np.random.default_rng(500 + seed)
    m, k, n = (int(x) for x in rng.integers(1, 9, 3))
    A = rng.integers(0, 30, (m, k)).astype(np.uint64)
    B = rng.integers(0, 30, (k, n)).astype(np.uint64)
    A[rng.random(A.shape) < 0.2] = np.uint64(INF64)
    B[rng.random(B.shape) < 0.2] = np.uint64(INF64)
    Cm, arg = O.minplus(A, B)
    Af = A.astype(np.float64)
    Af[A == np.uint64(INF64)] = np.inf
    Bf = B.astype(np.float64)
    Bf[B == np.uint64(INF64)] = np.inf
    S = Af[:, :, None] + Bf[None, :, :]
    ref = S.min(axis=1)
    am = S.argmin(axis=1)
    for i in range(m):
        for j in range(n):
            if np.isinf(ref[i, j]):
                assert int(Cm[i, j]) == INF64 and int(arg[i, j]) == INF64
            else:
                assert int(Cm[i, j]) == int(ref[i, j]) and int(arg[i, j]) == int(am[i, j])


def test_powers_associative(oracle_lib):
    """M^a (x) M^b = M^(a+b) (the identity repeated squaring relies on)."""
    O = oracle_lib
    rng = np.random.default_rng(7)
    M = rng.integers(0, 100, (5, 5)).astype(np.uint64)
    M[rng.random(M.shape) < 0.2] = np.uint64(INF64)
    P = [M]
    for _ in range(6):
        P.append(O.minplus(P[-1], M)[0])       # P[k] = M^(k+1)
    for a in range(1, 4):
        for b in range(1, 4):
            assert np.array_equal(O.minplus(P[a - 1], P[b - 1])[0], P[a + b - 1])


# ---------------------------------------------------------------- brute force corpus
MODES = ("ties", "random", "nearmax")


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("block", range(6))
def test_oracle_vs_brute_force_corpus(oracle_lib, mode, block):
    """>= 500 random tiny problems (6 blocks x 30 seeds x 3 modes = 540)."""
    O = oracle_lib
    for seed in range(block * 30, block * 30 + 30):
        p = G.tiny_random(seed * 7 + MODES.index(mode), mode=mode, max_plans=20000)
        bf = O.brute_force(p)
        if bf["total"] is None:
            with pytest.raises(O.OracleError) as ei:
                O.search_plan(p, nthreads=1)
            assert ei.value.rc == O.ORC_EINFEASIBLE
            continue
        r = O.search_plan(p, nthreads=2)
        assert r["total"] == bf["total"], p.name
        assert r["seg_index"].tolist() == bf["seg_index"].tolist(), p.name
        assert r["seg_ns"].tolist() == bf["seg_ns"].tolist(), p.name


@pytest.mark.parametrize("seed", range(60))
def test_segment_table_vs_python_enumeration(oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(9000 + seed, mode=MODES[seed % 3], max_plans=None, max_n=3)
    m = O.Marshalled(p)
    for tr in range(len(p.transitions)):
        A, I = O.segment_table(p, tr, nthreads=3, m=m)
        A2, I2 = O.brute_force_table(p, tr)
        assert np.array_equal(A, A2) and np.array_equal(I, I2)
        for u in range(A.shape[0]):
            for v in range(A.shape[1]):
                assert O.bucket(p, tr, u, v, nthreads=2, m=m) == (int(A[u, v]), int(I[u, v]))


def test_determinism(oracle_lib):
    O = oracle_lib
    p = G.make_config("C2", seed=1, dist="ties")
    a = O.search_plan(p, nthreads=3)
    b = O.search_plan(p, nthreads=5)
    assert a["total"] == b["total"]
    for k in ("seg_index", "digits", "seg_ns"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("cfg", ["C1", "C2"])
@pytest.mark.parametrize("dist", ["shaped", "random", "ties"])
def test_small_configs_eq3_recompute(oracle_lib, cfg, dist):
    """Oracle plan's Eq. 3 total recomputed in Python from its tuple."""
    O = oracle_lib
    p = G.make_config(cfg, seed=0, dist=dist)
    r = O.search_plan(p)
    u, tot = 0, 0
    for n, t in enumerate(p.instances):
        ty = p.types[p.transitions[int(t)].type]
        s = O._digits(ty.radix, int(r["seg_index"][n]))
        c = O.py_cost(p, int(t), u, s)
        assert c == int(r["seg_ns"][n])
        tot += c
        u = s[ty.out_block]
    assert tot == r["total"]
    if cfg == "C1":
        bf = O.brute_force(p)
        assert bf["total"] == r["total"] and bf["seg_index"].tolist() == r["seg_index"].tolist()
