"""GPU parity of the dynamic profiling budget (P:601,
readings R-B1..R-B4) through the C-ABI vs the CPU oracle (oracle/profiling.py),
exact: integer counts, 128-bit ns sums, best and its least index.

Cases: empty, single task, one partial tile, tile boundaries +- 1, many tiles
(the decoupled look-back crosses tens of thousands of tiles), random / tie /
monotone / INF-heavy / all-INF tables, factors from 1 to 65535, the device
generator's dense tables up to 2^26 tasks compared with the oracle in full,
and the bench's full C3 table (24^7 tasks, 18.3 GB) checked by properties that
hold at any size (the reported best is the table's minimum, attained first at
the reported index; counts add up; spent <= full).
"""
import numpy as np
import pytest

from oracle import profiling as PR
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
    W = np.ascontiguousarray(W, np.uint32)
    t = torch.empty(max(1, W.size) + 4, dtype=torch.int32, device="cuda")
    if W.size:
        t[:W.size] = torch.from_numpy(W.view(np.int32)).cuda()
    return t


def _run(ctx, W, num, den):
    t = _dev(W)
    return ctx.profile_budget(t.data_ptr(), len(W), num, den)


SIZES = [0, 1, 3, 4095, 4096, 4097, 8191, 8193, 12345, 40961, 1 << 20, (1 << 20) + 17]
FACTORS = [(1, 1), (2, 1), (3, 2), (65535, 1), (65535, 65534), (101, 100)]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", ["random", "ties", "dec", "inf"])
def test_budget_matches_oracle(ctx, n, dist):
    rng = np.random.default_rng(n * 7 + len(dist))
    if dist == "random":
        W = rng.integers(0, 1 << 24, size=n, dtype=np.uint64).astype(np.uint32)
    elif dist == "ties":
        W = rng.integers(0, 4, size=n, dtype=np.uint64).astype(np.uint32)
    elif dist == "dec":                      # a new best in (almost) every tile: look-back + rare path
        W = (np.uint32(1 << 30) - np.arange(n, dtype=np.uint32) * np.uint32(3)
             + rng.integers(0, 5, size=n, dtype=np.uint64).astype(np.uint32))
    else:
        W = rng.integers(0, (1 << 32) - 1, size=n, dtype=np.uint64).astype(np.uint32)
        W[rng.random(n) < 0.4] = INF32
    for num, den in FACTORS[: 3 if n > 100000 else len(FACTORS)]:
        assert _run(ctx, W, num, den) == PR.budget(W, num, den), (n, dist, num, den)


def test_budget_all_infeasible_and_empty(ctx):
    W = np.full(10000, INF32, np.uint32)
    assert _run(ctx, W, 2, 1) == PR.budget(W, 2, 1)
    import torch
    t = torch.empty(4, dtype=torch.int32, device="cuda")
    assert ctx.profile_budget(t.data_ptr(), 0, 2, 1) == PR.budget(np.zeros(0, np.uint32), 2, 1)


def test_budget_small_loop_brute(ctx):
    """Against the plain sequential loop too (R-B1 as written)."""
    for seed in range(6):
        rng = np.random.default_rng(seed)
        W = rng.integers(0, 50, size=5000, dtype=np.uint64).astype(np.uint32)
        W[rng.random(5000) < 0.1] = INF32
        assert _run(ctx, W, 3, 2) == PR.budget_loop(W, 3, 2)


def test_budget_errors(ctx):
    from paper_2504_00598_b200 import cfp
    t = _dev(np.arange(100, dtype=np.uint32))
    for num, den in [(1, 2), (0, 0), (70000, 1)]:
        with pytest.raises(cfp.CfpError) as ei:
            ctx.profile_budget(t.data_ptr(), 100, num, den)
        assert ei.value.status == cfp.CFP_EINVAL
    with pytest.raises(cfp.CfpError) as ei:
        ctx.profile_budget(t.data_ptr() + 4, 10, 2, 1)          # not 16-byte aligned
    assert ei.value.status == cfp.CFP_EINVAL
    with pytest.raises(cfp.CfpError) as ei:
        ctx.profile_budget(t.data_ptr(), 1 << 44, 2, 1)
    assert ei.value.status == cfp.CFP_ETOOBIG


@pytest.mark.parametrize("n,seed", [(24 ** 5, 0), ((1 << 26) + 1000, 3)])
def test_budget_dense_generator_tables(ctx, n, seed):
    """The synthetic dense tables of NEXT-2 (device generator == synth), in full."""
    import torch
    buf = torch.empty(n + 8, dtype=torch.int32, device="cuda")
    base = G.dense_base(seed, 1)
    ctx.dense_fill(buf.data_ptr(), n, base)
    W = G.dense_table(seed, 1, n)
    for num, den in [(2, 1), (5, 4)]:
        assert ctx.profile_budget(buf.data_ptr(), n, num, den) == PR.budget(W, num, den)


@pytest.mark.slow
def test_budget_full_c3_table_properties(ctx):
    """BASELINE config C3's layer type: 24^7 = 4.59e9 tasks (18.3 GB), the
    launch configuration bench.py --budget times."""
    import torch
    n = 24 ** 7
    buf = torch.empty(n + 8, dtype=torch.int32, device="cuda")
    ctx.dense_fill(buf.data_ptr(), n, G.dense_base(0, 1))
    r = ctx.profile_budget(buf.data_ptr(), n, 2, 1)
    assert r["tasks"] == n and r["pruned"] + r["infeasible"] <= n and r["spent"] <= r["full"]
    # best = the table minimum, first attained at best_index (chunked on the GPU)
    u = lambda x: x.to(torch.int64) & 0xFFFFFFFF                    # noqa: E731
    gmin, first = None, None
    step = 1 << 28
    for lo in range(0, n, step):
        c = u(buf[lo:min(n, lo + step)])
        m = int(c.min())
        if gmin is None or m < gmin:
            gmin, first = m, lo + int(torch.nonzero(c == m)[0])
    assert (r["best"], r["best_index"]) == (gmin, first)
    # the prefix up to 2^26 tasks against the oracle: the same counts as a
    # separate call on that prefix (the scan is causal)
    m = 1 << 26
    assert ctx.profile_budget(buf.data_ptr(), m, 2, 1) == PR.budget(G.dense_table(0, 1, m), 2, 1)
    del buf
    torch.cuda.empty_cache()
