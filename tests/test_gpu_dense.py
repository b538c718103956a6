"""GPU parity of the dense per-plan-table search (P:572-574,
P:608) through the C-ABI vs the CPU oracle, bit-exact.

Cases: the device generator equals synth.dense_table; full tables of random
tiny problems (o anywhere, cross edges on any block, start transitions with
cross edges, INF plans, 16-byte and scalar row paths); random searches
(feasible and infeasible); C1/C2 graphs with hashed dense tables; C3 at the
bench's full size (every emitted segment's cost recomputed from the generator
and the cross tables, and the oracle's chain + reconstruction over the GPU's
per-transition tables).
"""
import numpy as np
import pytest

from synth import generators as G
from synth.problem import INF32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    c = cfp.Context(device=0)
    yield c
    c.close()


def _dev(W):
    import torch
    return torch.from_numpy(np.ascontiguousarray(W, np.uint32).view(np.int32)).cuda()


def _tables(p, seed, inf_every=0):
    Ws = []
    for t in range(len(p.types)):
        w = G.dense_table(seed, t, p.num_combinations(t))
        if seed % 3 == 0:
            w = np.where(w == INF32, w, w % np.uint32(61)).astype(np.uint32)   # ties
        if inf_every:
            w[::inf_every] = np.uint32(INF32)
        Ws.append(w)
    return Ws


def test_device_generator_matches_synth(ctx):
    import torch
    n = 100003
    buf = torch.empty(n + 8, dtype=torch.int32, device="cuda")
    base = G.dense_base(7, 3)
    ctx.dense_fill(buf.data_ptr(), n, base)
    got = buf[:n].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, G.dense_table(7, 3, n))
    ctx.dense_fill(buf.data_ptr() + 4, 1000, base)          # unaligned start: scalar path
    # element e of the stream is a function of e alone; the window starting at
    # the second word is W[0..1000) again
    assert np.array_equal(buf[1:1001].cpu().numpy().view(np.uint32), G.dense_table(7, 3, 1000))


@pytest.mark.parametrize("seed", range(40))
def test_dense_tables_random(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(7000 + seed, max_k=4, max_d=6)
    Ws = _tables(p, seed, inf_every=11 if seed % 4 == 1 else 0)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        t = p.transitions[tr].type
        A, I = O.dense_segment_table(p, tr, Ws[t], m=m)
        d = _dev(Ws[t])
        Ag, Ig = ctx.segment_costs_dense(p.types[t], d.data_ptr(), p.transitions[tr], p.d_in(tr))
        assert np.array_equal(Ag, A), (seed, tr)
        assert np.array_equal(Ig, I), (seed, tr)


@pytest.mark.parametrize("seed", range(120))
def test_dense_search_random(ctx, oracle_lib, seed):
    O = oracle_lib
    from paper_2504_00598_b200 import cfp
    p = G.tiny_random(7200 + seed)
    Ws = _tables(p, seed, inf_every=5 if seed % 5 == 0 else 0)
    devs = [_dev(w) for w in Ws]
    ptrs = [d.data_ptr() for d in devs]
    try:
        want = O.dense_search_plan(p, Ws)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        with pytest.raises(cfp.CfpError) as ei:
            ctx.search_plan_dense(p, ptrs)
        assert ei.value.status == cfp.CFP_EINFEASIBLE
        return
    got = ctx.search_plan_dense(p, ptrs)
    assert got.total_ns == want["total"]
    assert got.seg_index.tolist() == want["seg_index"].tolist()
    assert got.seg_ns.tolist() == want["seg_ns"].tolist()
    k = min(got.digits.shape[1], want["digits"].shape[1])
    assert np.array_equal(got.digits[:, :k], want["digits"][:, :k])


@pytest.mark.parametrize("cfg,seed", [("C1", 0), ("C1", 3), ("C2", 0), ("C2", 1)])
def test_dense_configs(ctx, oracle_lib, cfg, seed):
    O = oracle_lib
    p = G.make_config(cfg, seed, "shaped")
    Ws = _tables(p, seed + 1)
    devs = [_dev(w) for w in Ws]
    want = O.dense_search_plan(p, Ws)
    got = ctx.search_plan_dense(p, [d.data_ptr() for d in devs])
    assert got.total_ns == want["total"]
    assert got.seg_index.tolist() == want["seg_index"].tolist()


def test_dense_c3_full_size(ctx, oracle_lib):
    """C3 with hashed dense tables at full size (2 x 4.59e9 plans, 36.7 GB)."""
    import torch
    O = oracle_lib
    p = G.make_config("C3", 0, "shaped")
    seed = 0
    bufs = []
    for t in range(len(p.types)):
        n = p.num_combinations(t)
        b = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.dense_fill(b.data_ptr(), n, G.dense_base(seed, t))
        bufs.append(b)
    got = ctx.search_plan_dense(p, [b.data_ptr() for b in bufs])
    u, tot = 0, 0
    for n, t in enumerate(p.instances):
        T = p.transitions[int(t)]
        ty = p.types[T.type]
        idx = int(got.seg_index[n])
        w = int(G.dense_table(seed, T.type, 1, lo=idx)[0])
        assert w != int(INF32)
        s = got.digits[n][: len(ty.radix)]
        c = w + sum(int(x.table[u, s[x.dst]]) for x in T.in_edges)
        assert c == int(got.seg_ns[n])
        tot += c
        u = int(s[ty.out_block])
    assert tot == got.total_ns
    # oracle chain + reconstruction over the GPU's per-transition tables
    tabs = {}
    for tr in sorted({int(t) for t in p.instances}):
        T = p.transitions[tr]
        tabs[tr] = ctx.segment_costs_dense(p.types[T.type], bufs[T.type].data_ptr(), T, p.d_in(tr))
    mats = [tabs[int(t)][0] for t in p.instances]
    idxs = [tabs[int(t)][1] for t in p.instances]
    Gs = O.chain(mats)
    assert int(Gs[0][0]) == got.total_ns
    rec = O.reconstruct(mats, idxs, Gs)
    assert [int(x) for x in rec[1]] == got.seg_index.tolist()
    del bufs
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- world > 1
# Every rank holds the rows of a block-0 strategy range (cfp_dense_shard) and
# answers with rank-local (A, least global index); the lexicographic (cost,
# index) min over the ranks -- what the NCCL merge computes -- must equal the
# single-GPU tables.  Shard simulation: world > 1 contexts without a
# communicator on one GPU.


def _merge(parts):
    A, I = parts[0][0].copy(), parts[0][1].copy()
    for a, i in parts[1:]:
        take = (a < A) | ((a == A) & (i < I))
        A, I = np.where(take, a, A), np.where(take, i, I)
    return A, I


def _dense_shards(cfp, ty, W, tr, din, world):
    d = _dev(W)
    parts, covered = [], 0
    for r in range(world):
        c = cfp.Context(device=0, world=world, rank=r)
        first, count = c.dense_shard(ty)
        assert first == covered                          # contiguous, in rank order
        covered += count
        parts.append(c.segment_costs_dense(ty, d.data_ptr() + 4 * first, tr, din))
        c.close()
    assert covered == len(W)
    return _merge(parts)


@pytest.mark.parametrize("seed", range(16))
def test_dense_shard_simulation_random(ctx, seed):
    from paper_2504_00598_b200 import cfp
    p = G.tiny_random(7300 + seed, max_k=4, max_d=6)
    Ws = _tables(p, seed, inf_every=7 if seed % 3 == 1 else 0)
    for tr in sorted({int(t) for t in p.instances}):
        t = p.transitions[tr].type
        d = _dev(Ws[t])
        A1, I1 = ctx.segment_costs_dense(p.types[t], d.data_ptr(), p.transitions[tr], p.d_in(tr))
        for world in (2, 3, 8):
            A, I = _dense_shards(cfp, p.types[t], Ws[t], p.transitions[tr], p.d_in(tr), world)
            assert np.array_equal(A, A1) and np.array_equal(I, I1), (seed, tr, world)


def test_dense_shard_simulation_c2(ctx):
    from paper_2504_00598_b200 import cfp
    p = G.make_config("C2", 0, "shaped")
    Ws = _tables(p, 5)
    for tr in sorted({int(t) for t in p.instances}):
        t = p.transitions[tr].type
        d = _dev(Ws[t])
        A1, I1 = ctx.segment_costs_dense(p.types[t], d.data_ptr(), p.transitions[tr], p.d_in(tr))
        A, I = _dense_shards(cfp, p.types[t], Ws[t], p.transitions[tr], p.d_in(tr), 4)
        assert np.array_equal(A, A1) and np.array_equal(I, I1), tr


def test_dense_shard_simulation_search_refused(ctx):
    from paper_2504_00598_b200 import cfp
    p = G.tiny_random(7301, max_k=3, max_d=4)
    Ws = _tables(p, 1)
    ds = [_dev(w) for w in Ws]
    c = cfp.Context(device=0, world=2, rank=0)
    with pytest.raises(cfp.CfpError):
        c.search_plan_dense(p, [d.data_ptr() for d in ds])
    c.close()


@pytest.fixture(scope="module")
def ctx_nccl():
    from paper_2504_00598_b200 import cfp
    c = cfp.Context(device=0, world=1, rank=0, nccl_unique_id=cfp.nccl_unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(10))
def test_dense_nccl_one_rank(ctx_nccl, oracle_lib, seed):
    """The world > 1 merge code (NCCL MIN of A, masked MIN of the least
    indices) on a 1-rank communicator: tables and plans == the oracle."""
    O = oracle_lib
    p = G.tiny_random(7400 + seed, max_k=4, max_d=5)
    Ws = _tables(p, seed)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        t = p.transitions[tr].type
        A, I = O.dense_segment_table(p, tr, Ws[t], m=m)
        d = _dev(Ws[t])
        Ag, Ig = ctx_nccl.segment_costs_dense(p.types[t], d.data_ptr(), p.transitions[tr], p.d_in(tr))
        assert np.array_equal(Ag, A) and np.array_equal(Ig, I), (seed, tr)
    devs = [_dev(w) for w in Ws]
    try:
        want = O.dense_search_plan(p, Ws)
    except O.OracleError:
        return
    got = ctx_nccl.search_plan_dense(p, [d.data_ptr() for d in devs])
    assert got.total_ns == want["total"] and got.seg_index.tolist() == want["seg_index"].tolist()
