"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit-exact.

Costs are integer ns, so every comparison is exact equality (north_star:
"GPU and oracle plans and costs must be bit-exact with lowest-index
tie-break").
"""
import numpy as np
import pytest

from golden_util import load, problem_from
from synth import generators as G
from synth.problem import INF32, CrossEdge, Problem, SegmentType, Transition

pytestmark = pytest.mark.gpu
INF64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def ctx():
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    c = cfp.Context(device=0)
    yield c
    c.close()


def _cfp():
    from paper_2504_00598_b200 import cfp
    return cfp


def _assert_plan(got, want, name=""):
    assert got.total_ns == want["total"], (name, got.total_ns, want["total"])
    assert got.seg_index.tolist() == want["seg_index"].tolist(), name
    assert got.seg_ns.tolist() == want["seg_ns"].tolist(), name
    k = min(got.digits.shape[1], want["digits"].shape[1])
    assert np.array_equal(got.digits[:, :k], want["digits"][:, :k]), name


def _search_or_infeasible(ctx, oracle_lib, prob):
    O = oracle_lib
    cfp = _cfp()
    try:
        want = O.search_plan(prob)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        with pytest.raises(cfp.CfpError) as ei:
            ctx.search_plan(prob)
        assert ei.value.status == cfp.CFP_EINFEASIBLE
        return None
    got = ctx.search_plan(prob)
    _assert_plan(got, want, prob.name)
    return got


# ---------------------------------------------------------------- golden
@pytest.mark.parametrize("name", ["h1", "h2", "h2p", "h3"])
def test_golden_plans(ctx, name):
    g = load(name)
    p = problem_from(g["problem"])
    got = ctx.search_plan(p)
    assert got.total_ns == g["expect"]["total"]
    assert got.seg_index.tolist() == g["expect"]["seg_index"]
    assert got.seg_ns.tolist() == g["expect"]["seg_ns"]


def test_golden_h1_tables(ctx):
    g = load("h1")
    p = problem_from(g["problem"])
    A, I = ctx.segment_costs(p.types[0], None, 1)
    assert A.tolist() == g["expect"]["A"]["0"] and I.tolist() == g["expect"]["I"]["0"]
    A, I = ctx.segment_costs(p.types[0], p.transitions[1], 3)
    assert A.tolist() == g["expect"]["A"]["1"] and I.tolist() == g["expect"]["I"]["1"]


def test_golden_cx_chain(ctx):
    g = load("cx")
    mats = [np.array(M, np.uint64) for M in g["chain"]["mats"]]
    opt, Gs = ctx.minplus_chain(mats, [(0, 1), (1, 1)])
    assert opt == g["expect"]["total"]
    assert [x.tolist() for x in Gs] == g["expect"]["G"]


# ---------------------------------------------------------------- corpus
MODES = ("ties", "random", "nearmax")


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("block", range(4))
def test_random_corpus_search(ctx, oracle_lib, mode, block):
    for seed in range(block * 25, block * 25 + 25):
        p = G.tiny_random(seed * 7 + MODES.index(mode), mode=mode, max_plans=None, max_n=6)
        _search_or_infeasible(ctx, oracle_lib, p)


@pytest.mark.parametrize("seed", range(40))
def test_random_segment_tables(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(5000 + seed, mode=MODES[seed % 3], max_plans=None, max_n=4, max_k=4)
    for tr_id, tr in enumerate(p.transitions):
        A0, I0 = O.segment_table(p, tr_id)
        ty = p.types[tr.type]
        A, I = ctx.segment_costs(ty, tr, p.d_in(tr_id))
        assert np.array_equal(A, A0), (seed, tr_id)
        assert np.array_equal(I, I0), (seed, tr_id)


@pytest.mark.parametrize("seed", range(12))
def test_larger_random_segment_tables(ctx, oracle_lib, seed):
    """K up to 6, D up to 6 -- exercises the M/A/B schedules and multi-CTA
    grids (several tiles, ragged tails)."""
    O = oracle_lib
    p = G.tiny_random(7000 + seed, mode=("ties", "random")[seed % 2], max_plans=None, max_n=3,
                      max_k=6, max_d=6, max_edges=6, p_inf=0.03)
    for tr_id, tr in enumerate(p.transitions):
        A0, I0 = O.segment_table(p, tr_id)
        ty = p.types[tr.type]
        A, I = ctx.segment_costs(ty, tr, p.d_in(tr_id))
        assert np.array_equal(A, A0), (seed, tr_id)
        assert np.array_equal(I, I0), (seed, tr_id)


@pytest.mark.parametrize("seed", range(10))
def test_long_runs_repeated_squaring(ctx, oracle_lib, seed):
    """Chains with long runs of one transition (repeated squaring + doubling)."""
    p = G.tiny_random(8000 + seed, mode=MODES[seed % 3], max_plans=None, max_n=40, max_types=2,
                      max_run=37)
    _search_or_infeasible(ctx, oracle_lib, p)


# ---------------------------------------------------------------- chain / product
@pytest.mark.parametrize("seed", range(10))
def test_minplus_product(ctx, oracle_lib, seed):
    rng = np.random.default_rng(seed)
    m, k, n = (int(x) for x in rng.integers(1, 40, 3))
    A = rng.integers(0, 1000, (m, k)).astype(np.uint64)
    B = rng.integers(0, 1000, (k, n)).astype(np.uint64)
    A[rng.random(A.shape) < 0.2] = np.uint64(INF64)
    B[rng.random(B.shape) < 0.2] = np.uint64(INF64)
    C0, a0 = oracle_lib.minplus(A, B)
    C1, a1 = ctx.minplus_product(A, B)
    assert np.array_equal(C0, C1) and np.array_equal(a0, a1)


@pytest.mark.parametrize("shape,maxv", [((130, 257, 129), 1 << 20), ((64, 300, 200), 1 << 40),
                                         ((1, 500, 3), 1000), ((200, 17, 1), 1 << 29)])
def test_minplus_product_tiled(ctx, oracle_lib, shape, maxv):
    """Multi-tile (min,+) products with ragged edges, narrow (< 2^31) and
    wide (2^40) values, INF entries, least-k argmin."""
    rng = np.random.default_rng(sum(shape))
    m, k, n = shape
    A = rng.integers(0, maxv, (m, k), dtype=np.uint64)
    B = rng.integers(0, maxv, (k, n), dtype=np.uint64)
    A[rng.random(A.shape) < 0.1] = np.uint64(INF64)
    B[rng.random(B.shape) < 0.1] = np.uint64(INF64)
    B[:, 0] = np.uint64(INF64)                      # an all-INF column
    C0, a0 = oracle_lib.minplus(A, B)
    C1, a1 = ctx.minplus_product(A, B)
    assert np.array_equal(C0, C1) and np.array_equal(a0, a1)


def test_minplus_bench_runs(ctx):
    ms, ops = ctx.minplus_bench(256, wide=False, argk=False, iters=2)
    assert ms > 0 and ops > 0


@pytest.mark.parametrize("seed", range(10))
def test_minplus_chain_runs(ctx, oracle_lib, seed):
    rng = np.random.default_rng(100 + seed)
    S = int(rng.integers(1, 30))
    M0 = rng.integers(0, 1 << 20, (1, S)).astype(np.uint64)
    M1 = rng.integers(0, 1 << 20, (S, S)).astype(np.uint64)
    M1[rng.random(M1.shape) < 0.3] = np.uint64(INF64)
    L = int(rng.integers(1, 100))
    term = rng.integers(0, 1000, S).astype(np.uint64)
    opt, Gs = ctx.minplus_chain([M0, M1], [(0, 1), (1, L)], terminal=term)
    want = oracle_lib.chain([M0] + [M1] * L, terminal=term)
    assert opt == int(want[0][0])
    for a, b in zip(Gs, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("S,L,maxv", [(100, 13, 1 << 20), (200, 9, 1 << 40), (65, 40, 1000)])
def test_minplus_chain_large_states(ctx, oracle_lib, S, L, maxv):
    """State spaces too large for the shared-memory chain kernel: squarings by
    the tiled (min,+) kernel, doubling by batched matrix-vector launches."""
    rng = np.random.default_rng(S + L)
    M0 = rng.integers(0, maxv, (3, S), dtype=np.uint64)
    M1 = rng.integers(0, maxv, (S, S), dtype=np.uint64)
    M1[rng.random(M1.shape) < 0.3] = np.uint64(INF64)
    M2 = rng.integers(0, maxv, (S, 7), dtype=np.uint64)
    opt, Gs = ctx.minplus_chain([M0, M1, M2], [(0, 1), (1, L), (2, 1)])
    want = oracle_lib.chain([M0] + [M1] * L + [M2])
    assert opt == int(want[0][0])
    for a, b in zip(Gs, want):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- configs
@pytest.mark.parametrize("cfg", ["C1", "C2"])
@pytest.mark.parametrize("dist", ["shaped", "random", "ties"])
@pytest.mark.parametrize("seed", [0, 1])
def test_small_configs_full_parity(ctx, oracle_lib, cfg, dist, seed):
    p = G.make_config(cfg, seed=seed, dist=dist)
    got = _search_or_infeasible(ctx, oracle_lib, p)
    assert got is not None


def _check_table_properties(O, p, tr_id, A, I, m, samples):
    """Full-size A/I: every entry's index decodes to its bucket and re-evaluates
    (oracle, Eq. 3 terms) to exactly A; sampled buckets are recomputed by the
    oracle's exhaustive enumeration (value and least index)."""
    ty = p.types[p.transitions[tr_id].type]
    din, dout = A.shape
    for u in range(din):
        for v in range(dout):
            if int(A[u, v]) == INF64:
                assert int(I[u, v]) == INF64
                continue
            s = O._digits(ty.radix, int(I[u, v]))
            assert s[ty.out_block] == v
            assert O.cost_index(p, tr_id, u, int(I[u, v]), m) == int(A[u, v])
    for (u, v) in samples:
        a, i = O.bucket(p, tr_id, u, v, m=m)
        assert (int(A[u, v]), int(I[u, v])) == (a, i), (tr_id, u, v)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_large_config_tables_sampled(ctx, oracle_lib, cfg):
    O = oracle_lib
    p = G.make_config(cfg, seed=0, dist="shaped")
    m = O.Marshalled(p)
    rng = np.random.default_rng(1)
    tr_id = 3                                    # L -> L
    tr = p.transitions[tr_id]
    A, I = ctx.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
    samples = [(int(rng.integers(0, A.shape[0])), int(rng.integers(0, A.shape[1]))) for _ in range(2)]
    _check_table_properties(O, p, tr_id, A, I, m, samples)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_large_config_plan(ctx, oracle_lib, cfg):
    """Full-size plan: Eq. 3 recomputation of the GPU tuple equals its total,
    and the oracle's chain DP + reconstruction over the GPU's per-transition
    tables gives the same OPT and plan."""
    O = oracle_lib
    p = G.make_config(cfg, seed=0, dist="shaped")
    got = ctx.search_plan(p)
    m = O.Marshalled(p)
    u, tot = 0, 0
    for n, t in enumerate(p.instances):
        ty = p.types[p.transitions[int(t)].type]
        c = O.cost_index(p, int(t), u, int(got.seg_index[n]), m)
        assert c == int(got.seg_ns[n])
        tot += c
        u = O._digits(ty.radix, int(got.seg_index[n]))[ty.out_block]
    assert tot == got.total_ns
    tabs = {}
    for tr_id, tr in enumerate(p.transitions):
        tabs[tr_id] = ctx.segment_costs(p.types[tr.type], tr,
                                        p.d_in(tr_id))
    mats = [tabs[int(t)][0] for t in p.instances]
    idxs = [tabs[int(t)][1] for t in p.instances]
    Gs = O.chain(mats)
    assert int(Gs[0][0]) == got.total_ns
    v, ix, cost = O.reconstruct(mats, idxs, Gs)
    assert ix.tolist() == got.seg_index.tolist()


# ---------------------------------------------------------------- errors
def test_errors(ctx):
    cfp = _cfp()
    p = problem_from(load("h1")["problem"])
    bad = problem_from(load("h1")["problem"])
    bad.instances = np.array([1, 1], np.int32)            # chain must start with pred -1
    with pytest.raises(cfp.CfpError) as ei:
        ctx.search_plan(bad)
    assert ei.value.status == cfp.CFP_EINVAL
    bad = problem_from(load("h1")["problem"])
    bad.types[0].out_block = 5
    with pytest.raises(cfp.CfpError) as ei:
        ctx.search_plan(bad)
    assert ei.value.status == cfp.CFP_EINVAL
    bad = problem_from(load("h1")["problem"])
    bad.types[0].edges[0].dst = 0                          # self edge
    with pytest.raises(cfp.CfpError) as ei:
        ctx.search_plan(bad)
    assert ei.value.status == cfp.CFP_EINVAL
    inf = problem_from(load("h1")["problem"])
    inf.types[0].comp_ns[3:6] = INF32                      # block 1 all infeasible
    with pytest.raises(cfp.CfpError) as ei:
        ctx.search_plan(inf)
    assert ei.value.status == cfp.CFP_EINFEASIBLE
    assert ctx.search_plan(p).total_ns == 6


def test_determinism(ctx):
    p = G.make_config("C2", seed=2, dist="ties")
    a = ctx.search_plan(p)
    b = ctx.search_plan(p)
    assert a.total_ns == b.total_ns
    assert np.array_equal(a.seg_index, b.seg_index) and np.array_equal(a.digits, b.digits)


def test_prepared_execute_matches(ctx, oracle_lib):
    p = G.make_config("C2", seed=0, dist="shaped")
    prep = ctx.prepare(p)
    for _ in range(3):
        prep.execute()
    got = prep.fetch()
    want = oracle_lib.search_plan(p)
    _assert_plan(got, want)
    info = prep.info()
    assert info.combos == 3 + 81 + 81 + 3
    prep.close()


# ---------------------------------------------------------------- sharded enumeration (one GPU)
def _merge_shards(parts):
    """Lexicographic (cost, index) min over the ranks' shard-local tables."""
    A = parts[0][0].copy()
    I = parts[0][1].copy()
    for a, i in parts[1:]:
        take = (a < A) | ((a == A) & (i < I))
        A = np.where(take, a, A)
        I = np.where(take, i, I)
    return A, I


def _shard_tables(cfp, ty, tr, din, world):
    parts = []
    for r in range(world):
        c = cfp.Context(device=0, world=world, rank=r)       # no unique id: shard simulation
        parts.append(c.segment_costs(ty, tr, din))
        c.close()
    return _merge_shards(parts)


@pytest.mark.parametrize("seed", range(12))
def test_shard_simulation_random(ctx, oracle_lib, seed):
    """The world > 1 enumeration path (shard ranges, rank-local fold, minima and
    least indices) on one GPU: every world size's merged shards == world 1."""
    cfp = _cfp()
    p = G.tiny_random(8800 + seed, max_k=6, max_d=6, max_plans=None)
    for tr in sorted({int(t) for t in p.instances}):
        ty = p.types[p.transitions[tr].type]
        A1, I1 = ctx.segment_costs(ty, p.transitions[tr], p.d_in(tr))
        for world in (2, 3, 8):
            A, I = _shard_tables(cfp, ty, p.transitions[tr], p.d_in(tr), world)
            assert np.array_equal(A, A1) and np.array_equal(I, I1), (seed, tr, world)


@pytest.mark.parametrize("cfg,world", [("C2", 4), ("C3", 2), ("C3", 8), ("C5", 3)])
def test_shard_simulation_configs(ctx, cfg, world):
    cfp = _cfp()
    p = G.make_config(cfg, 0, "shaped")
    for tr in sorted({int(t) for t in p.instances}):
        ty = p.types[p.transitions[tr].type]
        A1, I1 = ctx.segment_costs(ty, p.transitions[tr], p.d_in(tr))
        A, I = _shard_tables(cfp, ty, p.transitions[tr], p.d_in(tr), world)
        assert np.array_equal(A, A1) and np.array_equal(I, I1), (cfg, tr, world)


# ---------------------------------------------------------------- M split
# The enumeration's M-split path (two threads per prefix, each taking half of
# the M loop, merged in shared memory before the fold) runs by default only
# for long M loops (nM >= 128, C4); a ctx created with
# CFP_ENUM_MSPLIT_MIN_M=2 takes it for every eligible type.


@pytest.fixture(scope="module")
def ctx_ms():
    import os
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    old = os.environ.get("CFP_ENUM_MSPLIT_MIN_M")
    os.environ["CFP_ENUM_MSPLIT_MIN_M"] = "2"
    try:
        c = cfp.Context(device=0)
    finally:
        if old is None:
            del os.environ["CFP_ENUM_MSPLIT_MIN_M"]
        else:
            os.environ["CFP_ENUM_MSPLIT_MIN_M"] = old
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(12))
def test_msplit_random_segment_tables(ctx_ms, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(7000 + seed, mode=("ties", "random")[seed % 2], max_plans=None, max_n=3,
                      max_k=6, max_d=6, max_edges=6, p_inf=0.03)
    for tr_id, tr in enumerate(p.transitions):
        A0, I0 = O.segment_table(p, tr_id)
        A, I = ctx_ms.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
        assert np.array_equal(A, A0), (seed, tr_id)
        assert np.array_equal(I, I0), (seed, tr_id)


@pytest.mark.parametrize("cfg,dist", [("C1", "shaped"), ("C2", "random"), ("C2", "ties")])
def test_msplit_small_configs(ctx_ms, oracle_lib, cfg, dist):
    p = G.make_config(cfg, seed=1, dist=dist)
    _search_or_infeasible(ctx_ms, oracle_lib, p)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_msplit_large_config(ctx_ms, oracle_lib, cfg):
    """Full-size C3/C5 with the split on: sampled buckets against the oracle
    and the plan's Eq. 3 recomputation."""
    O = oracle_lib
    p = G.make_config(cfg, seed=0, dist="shaped")
    m = O.Marshalled(p)
    rng = np.random.default_rng(2)
    tr_id = 3
    tr = p.transitions[tr_id]
    A, I = ctx_ms.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
    samples = [(int(rng.integers(0, A.shape[0])), int(rng.integers(0, A.shape[1]))) for _ in range(2)]
    _check_table_properties(O, p, tr_id, A, I, m, samples)
    got = ctx_ms.search_plan(p)
    u, tot = 0, 0
    for n, t in enumerate(p.instances):
        ty = p.types[p.transitions[int(t)].type]
        c = O.cost_index(p, int(t), u, int(got.seg_index[n]), m)
        assert c == int(got.seg_ns[n])
        tot += c
        u = O._digits(ty.radix, int(got.seg_index[n]))[ty.out_block]
    assert tot == got.total_ns


# ---------------------------------------------------------------- NCCL merge path
# A ctx with world = 1 and an ncclUniqueId builds a one-rank communicator and
# runs the sharded path (rank-local tables, ncclAllReduce(ncclMin) of the
# bucket minima, masked least indices, second ncclAllReduce) on one GPU.


@pytest.fixture(scope="module")
def ctx_nccl():
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    c = cfp.Context(device=0, world=1, rank=0, nccl_unique_id=cfp.nccl_unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(8))
def test_nccl_one_rank_tables_and_plans(ctx_nccl, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(7300 + seed, mode=("ties", "random")[seed % 2], max_plans=None, max_n=3,
                      max_k=5, max_d=5, max_edges=5, p_inf=0.03)
    for tr_id, tr in enumerate(p.transitions):
        A0, I0 = O.segment_table(p, tr_id)
        A, I = ctx_nccl.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
        assert np.array_equal(A, A0) and np.array_equal(I, I0), (seed, tr_id)
    _search_or_infeasible(ctx_nccl, oracle_lib, p)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C5"])
def test_nccl_one_rank_configs(ctx, ctx_nccl, cfg):
    p = G.make_config(cfg, seed=0, dist="shaped")
    a, b = ctx.search_plan(p), ctx_nccl.search_plan(p)
    assert a.total_ns == b.total_ns
    assert a.seg_index.tolist() == b.seg_index.tolist() and a.seg_ns.tolist() == b.seg_ns.tolist()


# ---------------------------------------------------------------- transition dedup
# Transitions into the same type with identical predecessor output strategies,
# consumers and cross tables share one fold (C3/C5: L1 -> L and L -> L).


@pytest.fixture(scope="module")
def ctx_nodedup():
    import os
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    old = os.environ.get("CFP_DEDUP")
    os.environ["CFP_DEDUP"] = "0"
    try:
        c = cfp.Context(device=0)
    finally:
        if old is None:
            del os.environ["CFP_DEDUP"]
        else:
            os.environ["CFP_DEDUP"] = old
    yield c
    c.close()


@pytest.mark.parametrize("cfg", ["C2", "C3", "C5"])
def test_dedup_configs_equal_undeduplicated(ctx, ctx_nodedup, cfg):
    p = G.make_config(cfg, seed=0, dist="shaped")
    a, b = ctx.search_plan(p), ctx_nodedup.search_plan(p)
    assert a.total_ns == b.total_ns
    assert a.seg_index.tolist() == b.seg_index.tolist() and a.seg_ns.tolist() == b.seg_ns.tolist()


@pytest.mark.parametrize("seed", range(10))
def test_dedup_duplicated_transitions_random(ctx, oracle_lib, seed):
    """A chain E -> T, T -> T whose T -> T copy is byte-identical to a second
    transition from a different predecessor type with the same output radix."""
    import copy
    rng = np.random.default_rng(seed)
    p = copy.deepcopy(G.tiny_random(7700 + seed, mode="random", max_plans=None, max_n=2, max_k=4,
                                    max_d=4, max_edges=4, p_inf=0.0))
    # make every transition into the same type with the same D_in share its
    # first sibling's cross edges
    first = {}
    for tr_id, tr in enumerate(p.transitions):
        key = (tr.type, p.d_in(tr_id))
        if key in first and rng.random() < 0.8:
            tr.in_edges = copy.deepcopy(p.transitions[first[key]].in_edges)
        first.setdefault(key, tr_id)
    _search_or_infeasible(ctx, oracle_lib, p)


# ---------------------------------------------------------------- plan reuse
# cfp_search_plan reuses the previous call's prepared plan when the structure
# (shapes, feasible sets, term maxima, deduplicated instances) is unchanged
# and uploads only the new values: alternate problems that share a structure
# but not their values (finite entries permuted within each table, so every
# maximum is unchanged), and problems that do not.


def _permuted(p, seed):
    import copy
    q = copy.deepcopy(p)
    rng = np.random.default_rng(seed)
    for ty in q.types:
        comp = np.array(ty.comp_ns, np.uint32)
        comm = None if ty.comm_ns is None else np.array(ty.comm_ns, np.uint32)
        off = 0
        for d in ty.radix:                    # one permutation per block, shared by p and c
            d = int(d)
            perm = rng.permutation(d)
            comp[off:off + d] = comp[off:off + d][perm]
            if comm is not None:
                comm[off:off + d] = comm[off:off + d][perm]
            off += d
        ty.comp_ns, ty.comm_ns = comp, comm
        for e in ty.edges:
            e.table = rng.permutation(e.table.ravel()).reshape(e.table.shape).astype(np.uint32)
    for tr in q.transitions:
        for x in tr.in_edges:
            x.table = rng.permutation(x.table.ravel()).reshape(x.table.shape).astype(np.uint32)
    return q


@pytest.mark.parametrize("seed", range(6))
def test_plan_reuse_same_structure_new_values(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(7900 + seed, mode="random", max_plans=None, max_n=4, max_k=4, max_d=4,
                      max_edges=4, p_inf=0.0)
    variants = [p, _permuted(p, seed), _permuted(p, seed + 100), p]
    for q in variants:
        _search_or_infeasible(ctx, O, q)


def test_plan_reuse_alternating_configs(ctx, oracle_lib):
    O = oracle_lib
    probs = [G.make_config("C2", 0, "shaped"), G.make_config("C1", 0, "shaped"),
             G.make_config("C2", 1, "random"), G.make_config("C2", 0, "shaped")]
    for q in probs:
        _search_or_infeasible(ctx, O, q)


# ---------------------------------------------------------------- fused tail
# World 1 runs bucket minima, chain, argmin and backtrack as one cooperative
# launch; CFP_FUSED_TAIL=0 keeps the separate launches.  Both must agree with
# the oracle (and each other) bit for bit.


@pytest.fixture(scope="module")
def ctx_split():
    import os
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    old = os.environ.get("CFP_FUSED_TAIL")
    os.environ["CFP_FUSED_TAIL"] = "0"
    try:
        c = cfp.Context(device=0)
    finally:
        if old is None:
            del os.environ["CFP_FUSED_TAIL"]
        else:
            os.environ["CFP_FUSED_TAIL"] = old
    yield c
    c.close()


@pytest.mark.parametrize("mode", MODES)
def test_split_tail_corpus_search(ctx_split, oracle_lib, mode):
    for seed in range(40):
        p = G.tiny_random(seed * 11 + 3 + MODES.index(mode), mode=mode, max_plans=None, max_n=6)
        _search_or_infeasible(ctx_split, oracle_lib, p)


@pytest.mark.parametrize("seed", range(10))
def test_split_tail_segment_tables(ctx_split, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(9100 + seed, mode=MODES[seed % 3], max_plans=None, max_n=3, max_k=5, max_d=5)
    for tr_id, tr in enumerate(p.transitions):
        A0, I0 = O.segment_table(p, tr_id)
        A, I = ctx_split.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
        assert np.array_equal(A, A0) and np.array_equal(I, I0), (seed, tr_id)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_fused_tail_taken_and_equal_split(ctx, ctx_split, cfg):
    """The bench configurations take the fused tail (one launch after the
    enumeration), and it returns the split path's plan byte for byte."""
    p = G.make_config(cfg, seed=0, dist="shaped")
    prep = ctx.prepare(p)
    info = prep.info()
    assert info.fused_tail and info.tail_grid >= 2
    prep.execute()
    a = prep.fetch()
    prep.close()
    b = ctx_split.search_plan(p)
    assert a.total_ns == b.total_ns
    assert np.array_equal(a.seg_index, b.seg_index) and np.array_equal(a.seg_ns, b.seg_ns)
    assert np.array_equal(a.digits, b.digits)


def test_fused_tail_repeated_executes(ctx, oracle_lib):
    """The grid barrier words are left zero by every launch: many executes in
    a row (and phase timing on) keep returning the oracle's plan."""
    p = G.make_config("C2", seed=1, dist="ties")
    want = oracle_lib.search_plan(p)
    prep = ctx.prepare(p)
    prep.time_kernels(2)
    for _ in range(25):
        prep.execute()
        ph = prep.phase_ms()
        assert all(v >= 0 for v in ph.values())
    _assert_plan(prep.fetch(), want, "C2 repeated")
    prep.close()


@pytest.fixture(scope="module")
def ctx_sq():
    import os
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    old = os.environ.get("CFP_TAIL_SQUARING")
    os.environ["CFP_TAIL_SQUARING"] = "1"
    try:
        c = cfp.Context(device=0)
    finally:
        if old is None:
            del os.environ["CFP_TAIL_SQUARING"]
        else:
            os.environ["CFP_TAIL_SQUARING"] = old
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(12))
def test_fused_squaring_long_runs(ctx_sq, oracle_lib, seed):
    """The fused tail's repeated squaring + doubling variant (CFP_TAIL_SQUARING=1)."""
    p = G.tiny_random(8300 + seed, mode=MODES[seed % 3], max_plans=None, max_n=40, max_types=2, max_run=37)
    _search_or_infeasible(ctx_sq, oracle_lib, p)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C5"])
def test_fused_squaring_configs(ctx, ctx_sq, cfg):
    p = G.make_config(cfg, seed=0, dist="shaped")
    a, b = ctx.search_plan(p), ctx_sq.search_plan(p)
    assert a.total_ns == b.total_ns and np.array_equal(a.seg_index, b.seg_index)
    assert np.array_equal(a.seg_ns, b.seg_ns) and np.array_equal(a.digits, b.digits)


def test_marshal_cache_sees_in_place_changes(ctx, oracle_lib):
    """search_plan on the same problem object after in-place value changes:
    the cached marshalling refills its tables, so the plan follows the values."""
    import copy
    p = copy.deepcopy(G.make_config("C2", seed=2, dist="random"))
    _assert_plan(ctx.search_plan(p), oracle_lib.search_plan(p), "C2 before")
    rng = np.random.default_rng(0)
    for t in p.types:
        t.comp_ns[:] = rng.integers(0, 1 << 20, t.comp_ns.shape, dtype=np.uint32)
        for e in t.edges:
            e.table[...] = rng.integers(0, 1 << 20, e.table.shape, dtype=np.uint32)
    for tr in p.transitions:
        for x in tr.in_edges:
            x.table[...] = rng.integers(0, 1 << 20, x.table.shape, dtype=np.uint32)
    _assert_plan(ctx.search_plan(p), oracle_lib.search_plan(p), "C2 after in-place change")
