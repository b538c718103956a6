"""GPU parity of the memory-constrained search through
the C-ABI (cfp_search_plan_mem, cfp_segment_costs_mem) vs the CPU oracle,
bit-exact: integer ns costs, integer quanta, least-index tie-break.

Cases: the hand-worked golden examples M1/M2 and M3/M4 (P:628:
each plan's memory quantised as a whole -- answers that differ from a
per-block ceiling); memory-bucketed
segment tables of random tiny problems (ragged digit splits, INF entries,
narrow and wide paths, o inside and outside the prefix); full searches with a
limit drawn between the smallest and largest plan memory (binding or
infeasible) at quantum 1-3; C1/C2 with their shaped memory tables; C3 at full
size on sampled buckets recomputed by the oracle.
"""
import numpy as np
import pytest

from golden_util import load, problem_from
from synth import generators as G

pytestmark = pytest.mark.gpu


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


def _qtotals(O, p, quantum):
    m = O.Marshalled(p)
    lo = hi = 0
    for t in p.instances:
        a, b = O.mem_range(p, p.transitions[int(t)].type, quantum, m)
        lo, hi = lo + a, hi + b
    return lo, hi


def _compare(ctx, O, p, quantum, limit, name=""):
    cfp = _cfp()
    try:
        want = O.search_plan_mem(p, quantum, limit)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        with pytest.raises(cfp.CfpError) as ei:
            ctx.search_plan_mem(p, quantum, limit)
        assert ei.value.status == cfp.CFP_EINFEASIBLE, name
        return None
    got = ctx.search_plan_mem(p, quantum, limit)
    assert got.total_ns == want["total"], (name, got.total_ns, want["total"])
    assert got.seg_index.tolist() == want["seg_index"].tolist(), name
    assert got.seg_ns.tolist() == want["seg_ns"].tolist(), name
    assert got.seg_q.tolist() == want["seg_q"].tolist(), name
    assert got.total_q == want["total_q"], name
    k = min(got.digits.shape[1], want["digits"].shape[1])
    assert np.array_equal(got.digits[:, :k], want["digits"][:, :k]), name
    return got


@pytest.mark.parametrize("name", ["m1", "m2", "m3", "m4"])
def test_golden_mem(ctx, oracle_lib, name):
    d = load(name)
    p = problem_from(d["problem"])
    cfp = _cfp()
    for c in d["cases"]:
        if c["total"] is None:
            with pytest.raises(cfp.CfpError) as ei:
                ctx.search_plan_mem(p, c["quantum"], c["mem_limit"])
            assert ei.value.status == cfp.CFP_EINFEASIBLE
            continue
        got = ctx.search_plan_mem(p, c["quantum"], c["mem_limit"])
        assert got.total_ns == c["total"], c
        assert got.seg_index.tolist() == c["seg_index"], c
        assert got.total_q == c["total_q"], c


@pytest.mark.parametrize("seed", range(40))
def test_tables_mem_random(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(4000 + seed, max_k=4, max_d=5)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        ty = p.types[p.transitions[tr].type]
        din = p.d_in(tr)
        x = p.transitions[tr]           # a chain start may carry cross edges (one row, u = 0)
        for quantum in (1, 2, 5):
            A, I, qlo = O.segment_table_mem(p, tr, quantum, m=m)
            Ag, Ig, qlog = ctx.segment_costs_mem(ty, quantum, x, din)
            assert qlog == qlo, (seed, tr, quantum)
            assert Ag.shape == A.shape
            assert np.array_equal(Ag, A), (seed, tr, quantum)
            assert np.array_equal(Ig, I), (seed, tr, quantum)


@pytest.mark.parametrize("seed", range(150))
def test_search_mem_random(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(5000 + seed)
    rng = np.random.default_rng(seed)
    quantum = int(1 + seed % 3)
    lo, hi = _qtotals(O, p, quantum)
    limit = int(rng.integers(max(lo - 1, 0), hi + 2)) * quantum + int(rng.integers(0, quantum))
    _compare(ctx, O, p, quantum, limit, f"seed{seed}")


@pytest.mark.parametrize("seed", range(20))
def test_search_mem_unbinding_equals_unconstrained(ctx, oracle_lib, seed):
    O = oracle_lib
    p = G.tiny_random(5400 + seed)
    lo, hi = _qtotals(O, p, 1)
    try:
        ref = O.search_plan(p)
    except O.OracleError:
        return
    got = ctx.search_plan_mem(p, 1, hi)
    assert got.total_ns == ref["total"]
    assert got.seg_index.tolist() == ref["seg_index"].tolist()


@pytest.mark.parametrize("cfg,seed,dist", [("C1", 0, "shaped"), ("C1", 1, "ties"), ("C2", 0, "shaped"),
                                           ("C2", 2, "random"), ("C2", 1, "ties")])
def test_configs_mem(ctx, oracle_lib, cfg, seed, dist):
    O = oracle_lib
    p = G.make_config(cfg, seed, dist)
    lo, hi = _qtotals(O, p, 1)
    quantum = max(1, (hi - lo) // 64 or 1)
    lo, hi = _qtotals(O, p, quantum)
    for frac in (0.0, 0.3, 0.7, 1.0):
        limit = int((lo + frac * (hi - lo)) * quantum)
        _compare(ctx, O, p, quantum, limit, f"{cfg}/{frac}")


def test_c3_mem_full_size_sampled(ctx, oracle_lib):
    """C3 (LLaMA-7B shaped) at full size, the bench's configuration: every
    emitted segment's Eq. 3 cost and quantised memory recomputed by the oracle
    from its combination index; the oracle's (layout, memory) DP and greedy
    reconstruction over the GPU's per-transition tables give the same OPT and
    the same plan."""
    O = oracle_lib
    from synth.memcfg import mem_workload
    p, quantum, limit = mem_workload("C3", 0, "shaped")
    got = ctx.search_plan_mem(p, quantum, limit)
    m = O.Marshalled(p)
    # every emitted segment: the oracle's cost of that combination index and its memory
    u = 0
    tot = 0
    for n, t in enumerate(p.instances):
        tr = int(t)
        c = O.cost_index(p, tr, u, int(got.seg_index[n]), m=m)
        assert c == int(got.seg_ns[n])
        ty = p.types[p.transitions[tr].type]
        dg = got.digits[n][: len(ty.radix)]
        assert O.py_mem_q(ty, dg, quantum) == int(got.seg_q[n])
        tot += c
        u = int(dg[ty.out_block])
    assert tot == got.total_ns
    assert got.total_q * quantum <= limit
    # oracle DP + reconstruction over the GPU's tables
    tabs = {}
    for tr in sorted({int(t) for t in p.instances}):
        ty = p.types[p.transitions[tr].type]
        tabs[tr] = ctx.segment_costs_mem(ty, quantum, p.transitions[tr], p.d_in(tr))
    mats = [tabs[int(t)][0] for t in p.instances]
    idxs = [tabs[int(t)][1] for t in p.instances]
    qlos = [tabs[int(t)][2] for t in p.instances]
    Qmax = limit // quantum
    Gs = O.chain_mem(mats, qlos, Qmax)
    assert int(Gs[0][0, 0]) == got.total_ns
    _, q, ix, cost = O.reconstruct_mem(mats, idxs, qlos, Qmax, Gs)
    assert ix.tolist() == got.seg_index.tolist()
    assert cost.tolist() == got.seg_ns.tolist() and q.tolist() == got.seg_q.tolist()


@pytest.mark.parametrize("fold", ["u", "4x4"])     # mem_fold_u_kernel (default) / the 4 x 4 fold
@pytest.mark.parametrize("cfg,keep", [("C3", [3, 4, 5, 6]), ("C5", [3, 4, 5, 6])])
def test_midsize_mem_tables_every_bucket(ctx, oracle_lib, cfg, keep, fold, monkeypatch):
    """Mid-size cuts of the bench graphs with their memory tables: many prefix
    memory groups and suffix memories per class, so the per-plan class runs
    start and end anywhere in the sorted suffix row; every (u, v, q) bucket of
    every transition vs the oracle, then the search."""
    if fold == "4x4":
        monkeypatch.setenv("CFP_MEM_FOLD4", "1")      # read at each fold launch
    O = oracle_lib
    from synth.generators import midsize
    p = midsize(cfg, keep, n_layers=5)
    lo, hi = _qtotals(O, p, 1)                       # exact chain memory range
    m = O.Marshalled(p)
    top = max(O.mem_range(p, p.transitions[int(t)].type, 1, m)[1] for t in p.instances)
    for quantum in (max(1, top // 300), max(1, top // 40)):   # ~300 / ~40 levels per segment
        for tr in sorted({int(t) for t in p.instances}):
            A, I, qlo = O.segment_table_mem(p, tr, quantum, m=m)
            Ag, Ig, qlog = ctx.segment_costs_mem(p.types[p.transitions[tr].type], quantum, p.transitions[tr], p.d_in(tr))
            assert qlog == qlo and np.array_equal(Ag, A) and np.array_equal(Ig, I), (cfg, quantum, tr)
        qlo_t, qhi_t = _qtotals(O, p, quantum)
        for frac in (0.3, 0.7):
            limit = int((qlo_t + frac * (qhi_t - qlo_t)) * quantum)
            _compare(ctx, O, p, quantum, limit, f"{cfg} midsize q{quantum} {frac}")


def test_mem_plan_reuse_alternating(ctx, oracle_lib):
    """cfp_search_plan_mem keeps the last prepared search: calls with the same
    structure / memory profile / quantum / limit but new cost values reuse it
    (values re-uploaded, K0 / T rebuilt on the device), anything else
    re-prepares; every answer matches the oracle."""
    import copy
    O = oracle_lib
    from synth.memcfg import mem_workload
    base, quantum, limit = mem_workload("C2", 0, "shaped")
    other, quantum1, limit1 = mem_workload("C1", 0, "shaped")
    variants = []
    for k in range(3):
        q = copy.deepcopy(base)
        rng = np.random.default_rng(k)
        for t in q.types:
            t.comp_ns[:] = rng.integers(0, 1 << 20, t.comp_ns.shape, dtype=np.uint32)
        variants.append(q)
    for p, q, lim in [(variants[0], quantum, limit), (variants[1], quantum, limit), (other, quantum1, limit1),
                      (variants[2], quantum, limit), (variants[2], quantum, limit + quantum * 7),
                      (variants[0], quantum, limit)]:
        _compare(ctx, O, p, q, lim, "reuse")


def test_mem_infeasible_diagnostic_names_least_memory_plan(ctx, oracle_lib):
    """EINFEASIBLE carries the least-memory plan's memory and quanta."""
    from golden_util import load, problem_from
    cfp = _cfp()
    p = problem_from(load("m4")["problem"])
    with pytest.raises(cfp.CfpError) as ei:
        ctx.search_plan_mem(p, 4, 7)            # M4: each of the 2 segments needs >= 1 quantum, Qmax = 1
    assert ei.value.status == cfp.CFP_EINFEASIBLE
    msg = str(ei.value)
    assert "least-memory plan (0,0) (0,0)" in msg and "needs 4 memory units = 2 quanta" in msg and "Qmax = 1" in msg, msg
