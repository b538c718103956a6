"""Pins of the memory-constrained oracle against things
other than itself:

  * hand-worked examples M1/M2 (tests/golden/m*.json);
  * an independent pure-Python brute force over every global plan with the
    memory constraint ("matches dp_search with quantum = 1");
  * the already-pinned unconstrained oracle: with a limit that never binds the
    memory DP must return the unconstrained OPT and canonical plan;
  * invariants: never falsely feasible, monotone in the limit,
    coarser quantum never beats quantum = 1;
  * closed form: zero memory -> one memory class, Am[..., 0] == A.
"""
import numpy as np
import pytest

from golden_util import load, problem_from
from oracle import oracle as O
from synth import generators as G


def _qhi_total(p, quantum):
    m = O.Marshalled(p)
    return sum(O.mem_range(p, p.transitions[int(t)].type, quantum, m)[1] for t in p.instances)


def _qlo_total(p, quantum):
    m = O.Marshalled(p)
    return sum(O.mem_range(p, p.transitions[int(t)].type, quantum, m)[0] for t in p.instances)


def _search(p, quantum, limit):
    try:
        return O.search_plan_mem(p, quantum, limit)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        return dict(total=None)


@pytest.mark.parametrize("name", ["m1", "m2", "m3", "m4"])
def test_golden_mixed_plans(oracle_lib, name):
    d = load(name)
    p = problem_from(d["problem"])
    for c in d["cases"]:
        r = _search(p, c["quantum"], c["mem_limit"])
        assert r["total"] == c["total"], c
        if c["total"] is not None:
            assert r["seg_index"].tolist() == c["seg_index"], c
            assert r["total_q"] == c["total_q"], c
        b = O.brute_force_mem(p, c["quantum"], c["mem_limit"])
        assert b["total"] == c["total"], c


def test_mem_range_by_hand(oracle_lib):
    p = problem_from(load("m1")["problem"])
    assert O.mem_range(p, 0, 1) == (3, 6)
    assert O.mem_range(p, 0, 2) == (2, 3)
    assert O.mem_range(p, 0, 4) == (1, 2)
    assert O.mem_range(p, 0, 7) == (1, 1)
    # M3: plan memories 2..10 quantised per plan: ceil(2/4) = 1,
    # ceil(10/4) = 3 -- per-block ceilings would give (2, 4)
    p = problem_from(load("m3")["problem"])
    assert O.mem_range(p, 0, 4) == (1, 3)
    assert O.mem_range(p, 0, 1) == (2, 10)


def test_m3_table_by_hand(oracle_lib):
    """M3's table at quantum 4: bucket (u=0, v=s1, q): plan 0 (v 0, q 1, T 20),
    plan 1 (v 1, q 2, T 14), plan 2 (v 0, q 2, T 14), plan 3 (v 1, q 3, T 8)."""
    p = problem_from(load("m3")["problem"])
    A, I, qlo = O.segment_table_mem(p, 0, 4)
    INF = O.INF64
    assert qlo == 1 and A.shape == (1, 2, 3)
    assert A[0].tolist() == [[20, 14, INF], [INF, 14, 8]]
    assert I[0].tolist() == [[0, 2, INF], [INF, 1, 3]]


@pytest.mark.parametrize("seed", range(60))
def test_table_mem_matches_python(oracle_lib, seed):
    p = G.tiny_random(2000 + seed, max_d=3)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        for quantum in (1, 2):
            A, I, qlo = O.segment_table_mem(p, tr, quantum, m=m)
            A2, I2, qlo2 = O.brute_force_table_mem(p, tr, quantum)
            assert qlo == qlo2
            assert np.array_equal(A, A2) and np.array_equal(I, I2)


@pytest.mark.parametrize("seed", range(40))
def test_table_mem_projects_to_plain_table(oracle_lib, seed):
    """min over the memory coordinate of (Am, Im) is (A, I): the lowest index
    among the equal-cost classes is the plain bucket's lowest index."""
    p = G.tiny_random(2100 + seed)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        A, I = O.segment_table(p, tr, m=m)
        Am, Im, _ = O.segment_table_mem(p, tr, 1, m=m)
        amin = Am.min(axis=2)
        assert np.array_equal(amin, A)
        Imask = np.where(Am == amin[..., None], Im, np.uint64(O.NOIDX))
        assert np.array_equal(Imask.min(axis=2), I)


def test_zero_memory_closed_form(oracle_lib):
    p = G.tiny_random(7, max_d=4)
    for ty in p.types:
        ty.mem = None
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        A, I = O.segment_table(p, tr, m=m)
        Am, Im, qlo = O.segment_table_mem(p, tr, 3, m=m)
        assert qlo == 0 and Am.shape[2] == 1
        assert np.array_equal(Am[..., 0], A) and np.array_equal(Im[..., 0], I)


@pytest.mark.parametrize("seed", range(120))
def test_unbinding_limit_equals_unconstrained(oracle_lib, seed):
    p = G.tiny_random(2200 + seed)
    try:
        ref = O.search_plan(p)
    except O.OracleError as e:
        assert e.rc == O.ORC_EINFEASIBLE
        ref = dict(total=None)
    quantum = 1 + seed % 3
    r = _search(p, quantum, quantum * _qhi_total(p, quantum))
    assert r["total"] == ref["total"]
    if ref["total"] is not None:
        assert r["seg_index"].tolist() == ref["seg_index"].tolist()
        assert r["seg_ns"].tolist() == ref["seg_ns"].tolist()


@pytest.mark.parametrize("seed", range(300))
def test_dp_equals_brute_force(oracle_lib, seed):
    """DP with quantum = 1 == exhaustive search, at a limit drawn between
    the smallest and largest plan memory (so it binds, or just fails)."""
    p = G.tiny_random(2500 + seed, max_plans=20000)
    rng = np.random.default_rng(seed)
    lo, hi = _qlo_total(p, 1), _qhi_total(p, 1)
    limit = int(rng.integers(max(lo - 1, 0), hi + 1))
    r = _search(p, 1, limit)
    b = O.brute_force_mem(p, 1, limit, limit=20000)
    assert r["total"] == b["total"]
    if b["total"] is not None:
        assert r["seg_index"].tolist() == b["seg_index"].tolist()
        assert r["seg_ns"].tolist() == b["seg_ns"].tolist()
        assert r["seg_q"].tolist() == b["seg_q"].tolist()
        assert r["total_q"] == b["total_q"] <= limit


@pytest.mark.parametrize("seed", range(80))
def test_coarse_quantum_sound(oracle_lib, seed):
    """quantised memory over-approximates -> the returned plan's exact
    memory fits; a coarser quantum can only lose plans (T >= T at quantum 1);
    the DP still equals brute force at that quantum."""
    p = G.tiny_random(2900 + seed, max_plans=20000)
    rng = np.random.default_rng(seed)
    lo, hi = _qlo_total(p, 1), _qhi_total(p, 1)
    limit = int(rng.integers(lo, hi + 1))
    exact = _search(p, 1, limit)
    for quantum in (2, 3):
        r = _search(p, quantum, limit)
        b = O.brute_force_mem(p, quantum, limit, limit=20000)
        assert r["total"] == b["total"]
        if r["total"] is None:
            continue
        assert exact["total"] is not None and r["total"] >= exact["total"]
        assert r["seg_index"].tolist() == b["seg_index"].tolist()
        assert b["mem_exact"] <= limit
        assert r["total_q"] * quantum >= b["mem_exact"]


@pytest.mark.parametrize("seed", range(30))
def test_monotone_in_limit(oracle_lib, seed):
    """raising mem_limit never increases the returned T."""
    p = G.tiny_random(3100 + seed, max_plans=50000)
    lo, hi = _qlo_total(p, 1), _qhi_total(p, 1)
    prev = None
    for limit in range(max(lo - 1, 0), hi + 2):
        r = _search(p, 1, limit)
        t = r["total"]
        if prev is not None:
            assert t is not None and t <= prev
        if t is not None:
            prev = t
    assert limit >= hi


def test_infeasible_below_minimum(oracle_lib):
    p = G.tiny_random(11)
    lo = _qlo_total(p, 1)
    if lo == 0:
        pytest.skip("zero-memory plan exists")
    with pytest.raises(O.OracleError) as e:
        O.search_plan_mem(p, 1, lo - 1)
    assert e.value.rc == O.ORC_EINFEASIBLE


def test_chain_mem_zero_memory_is_plain_chain(oracle_lib):
    """With every q = 0 each G_n(., c) is the plain suffix vector G_n for all c."""
    rng = np.random.default_rng(5)
    mats = [rng.integers(0, 50, size=(1 if n == 0 else 4, 4)).astype(np.uint64) for n in range(5)]
    mats[2][1, 3] = np.uint64(O.INF64)
    Gp = O.chain(mats)
    Gm = O.chain_mem([M[..., None] for M in mats], [0] * 5, 3)
    for a, b in zip(Gp, Gm):
        assert np.array_equal(np.repeat(a[:, None], 4, axis=1), b)


@pytest.mark.parametrize("seed", range(10))
def test_table_mem_range_pieces(oracle_lib, seed):
    """Ranges [0, k) and [k, S) merged by (cost, index) give the full table."""
    p = G.tiny_random(3300 + seed, max_d=4)
    m = O.Marshalled(p)
    for tr in sorted({int(t) for t in p.instances}):
        S = p.num_combinations(p.transitions[tr].type)
        A, I, qlo = O.segment_table_mem(p, tr, 1, m=m)
        k = S // 3
        A1, I1, _ = O.segment_table_mem_range(p, tr, 1, 0, k, m=m)
        A2, I2, _ = O.segment_table_mem_range(p, tr, 1, k, S, m=m)
        take2 = A2 < A1
        assert np.array_equal(np.where(take2, A2, A1), A)
        assert np.array_equal(np.where(take2, I2, I1), I)
