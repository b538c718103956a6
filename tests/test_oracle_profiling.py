"""Pins of the NEXT-3 oracle (oracle/profiling.py) against things other than
itself:

  * the paper's printed counts: 2 x 81 + 2 x 9 = 180 programs for the GPT
    layer segments, the best case prod S_j + S_1 * S_K = 81 + 9 = 90
    (P:591), the worst case prod_{j=1}^{M} S_j, SPEC's trivial 3
    (S:381);
  * the explicit task list has exactly Eq. 2's length (brute enumeration);
  * the budget: SPEC's example (a plan 10x worse than the best with f = 2 is
    pruned), closed forms for monotone sequences, a generous budget
    prunes nothing, all-infeasible input, ties keep the least index; the
    numpy prefix-minimum form equals the sequential loop on random inputs.
"""
import numpy as np
import pytest

from oracle import profiling as PR
from synth import generators as G
from synth.problem import INF32, CrossEdge, Problem, SegmentType, Transition


def _type(radix, out_block):
    K = len(radix)
    D = int(sum(radix))
    return SegmentType(radix=np.array(radix, np.int32), comp_ns=np.zeros(D, np.uint32), comm_ns=None,
                       edges=[], out_block=out_block)


def test_paper_count_180_gpt_layers():
    """two layer segments of 4 blocks x 3 strategies -> 81 plans
    each, two boundary reshard groups (L1 -> L, L -> L) of 3 x 3 -> 180."""
    p = G.make_config("C2", 0, "shaped")
    sp = PR.profile_space(p)
    names = [t.name for t in p.types]
    tnames = [t.name for t in p.transitions]
    layers = sp["type_plans"][names.index("L1")] + sp["type_plans"][names.index("L")]
    pairs = sp["trans_pairs"][tnames.index("L1->L")] + sp["trans_pairs"][tnames.index("L->L")]
    assert (layers, pairs) == (2 * 81, 2 * 9)
    assert layers + pairs == 180
    # the embedding / head segments (K = 1, S = 3) and their boundaries add
    # 3 + 3 + 9 + 9 -- the paper counts the layers only
    assert sp["total"] == 180 + 3 + 3 + 9 + 9


def test_best_case_90():
    """a single distinct segment repeated, cross dependency from the
    last block to the first: prod_j S_j + S_1 * S_K = 81 + 9."""
    ty = _type([3, 3, 3, 3], out_block=3)
    q = np.zeros((3, 3), np.uint32)
    p = Problem(mesh=(4,), types=[ty],
                transitions=[Transition(-1, 0), Transition(0, 0, [CrossEdge(0, q)])],
                instances=np.array([0, 1, 1, 1], np.int32))
    assert PR.profile_space(p)["total"] == 90


@pytest.mark.parametrize("radix", [[3], [2, 5], [4, 3, 2, 2, 3]])
def test_worst_case_single_segment(radix):
    """the whole model as one distinct segment: prod_{j=1}^{M} S_j."""
    p = Problem(mesh=(2,), types=[_type(radix, len(radix) - 1)], transitions=[Transition(-1, 0)],
                instances=np.array([0], np.int32))
    assert PR.profile_space(p)["total"] == int(np.prod(radix))


def test_trivial_3():
    p = Problem(mesh=(2,), types=[_type([3], 0)], transitions=[Transition(-1, 0)],
                instances=np.array([0], np.int32))
    assert PR.profile_space(p)["total"] == 3


@pytest.mark.parametrize("seed", range(20))
def test_task_list_length_is_eq2(seed):
    p = G.tiny_random(9100 + seed, max_plans=None, max_n=4, max_k=4)
    tasks = list(PR.profile_tasks(p))
    assert len(tasks) == PR.profile_space(p)["total"]
    assert len(set(tasks)) == len(tasks)


def test_budget_spec_example():
    """one plan 10x worse than the best with f = 2.0 -> pruned, cut at
    its budget 2 x best."""
    r = PR.budget_loop([100, 1000], 2, 1)
    assert r["pruned"] == 1 and r["spent"] == 100 + 200 and r["full"] == 1100
    assert (r["best"], r["best_index"]) == (100, 0)


def test_budget_closed_forms():
    dec = np.arange(1000, 0, -1, dtype=np.uint32)      # every task is a new best
    r = PR.budget_loop(dec, 1, 1)
    assert r["pruned"] == 0 and r["spent"] == r["full"] == int(dec.sum())
    assert (r["best"], r["best_index"]) == (1, 999)
    inc = np.arange(7, 1007, dtype=np.uint32)           # f = 1: all but the first pruned at W[0]
    r = PR.budget_loop(inc, 1, 1)
    assert r["pruned"] == 999 and r["spent"] == 1000 * 7
    r = PR.budget_loop(inc, 3, 2)                       # f = 1.5: pruned iff w > 10.5
    assert r["pruned"] == int((inc > 10).sum()) and r["spent"] == int(inc[inc <= 10].sum()) + 10 * int((inc > 10).sum())
    r = PR.budget_loop(inc, 65535, 1)                   # generous: nothing pruned
    assert r["pruned"] == 0 and r["spent"] == r["full"]


def test_budget_infeasible_and_ties():
    r = PR.budget_loop(np.full(5, INF32, np.uint32), 2, 1)
    assert r == dict(tasks=5, pruned=0, infeasible=5, spent=0, full=0, best=PR.INF64, best_index=PR.NOIDX)
    r = PR.budget_loop(np.array([INF32, 5, 5, INF32, 5, 11], np.uint32), 2, 1)
    assert r["best_index"] == 1 and r["infeasible"] == 2 and r["pruned"] == 1 and r["spent"] == 25
    assert PR.budget([], 2, 1)["best_index"] == PR.NOIDX


def test_budget_factor_validated():
    for num, den in [(1, 2), (0, 1), (70000, 1), (2, 0)]:
        with pytest.raises(ValueError):
            PR.budget_loop([1, 2], num, den)
        with pytest.raises(ValueError):
            PR.budget([1, 2], num, den)


@pytest.mark.parametrize("seed", range(30))
def test_budget_numpy_equals_loop(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 3000))
    hi = int(rng.choice([4, 1000, 1 << 24, (1 << 32) - 1]))
    W = rng.integers(0, hi, size=n, dtype=np.uint64).astype(np.uint32)
    W[rng.random(n) < 0.05] = INF32
    num = int(rng.integers(1, 65536))
    den = int(rng.integers(1, num + 1))
    assert PR.budget(W, num, den) == PR.budget_loop(W, num, den)


def test_budget_dense_table_sample():
    """The synthetic dense table the GPU tests use, loop == numpy form."""
    W = G.dense_table(0, 1, 20000)
    assert PR.budget(W, 2, 1) == PR.budget_loop(W, 2, 1)
