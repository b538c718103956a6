"""C-ABI surface checks that need no GPU: the library builds, loads and exports
every function include/cfp.h declares; host-only helpers behave; without a
GPU the context refuses loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cfp():
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp as m
    return m


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cfp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cfp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    fns = declared_functions()
    for name in ("cfp_segment_costs", "cfp_minplus_chain", "cfp_search_plan"):
        assert name in fns


def test_library_exports_every_declared_symbol(cfp):
    L = C.CDLL(cfp.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert sorted(cfp.EXPORTS) == sorted(declared_functions())


def test_no_cpu_fallback(cfp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cfp.CfpError) as ei:
        cfp.Context(device=0)
    assert ei.value.status == cfp.CFP_ECUDA


@pytest.mark.parametrize("units,align,world", [(100, 1, 3), (100, 8, 3), (7, 4, 8), (0, 1, 2),
                                               (23 ** 4, 23, 8), (5, 1, 8)])
def test_shard_range_partitions(cfp, units, align, world):
    prev = 0
    for r in range(world):
        lo, hi = cfp.shard_range(units, align, world, r)
        assert lo == prev and lo <= hi
        assert lo % align == 0 or lo == units
        prev = hi
    assert prev == units


def test_pack_unpack_roundtrip_and_order(cfp):
    rng = np.random.default_rng(0)
    cost = rng.integers(0, 1 << 30, 1000).astype(np.uint64)
    idx = rng.integers(0, 1 << 33, 1000).astype(np.uint64)
    cost[::17] = np.uint64((1 << 64) - 1)
    keys = cfp.pack_keys(cost, idx, 33)
    c2, i2 = cfp.unpack_keys(keys, 33)
    fin = cost != np.uint64((1 << 64) - 1)
    assert np.array_equal(c2[fin], cost[fin]) and np.array_equal(i2[fin], idx[fin])
    assert np.all(i2[~fin] == np.uint64((1 << 64) - 1))
    # unsigned key order == lexicographic (cost, idx) order
    order = np.argsort(keys, kind="stable")
    lex = sorted(range(1000), key=lambda i: (int(cost[i]), int(idx[i])))
    assert [int(keys[i]) for i in order] == [int(keys[i]) for i in lex]


def test_pack_rejects_overflow(cfp):
    with pytest.raises(cfp.CfpError) as ei:
        cfp.pack_keys(np.array([1 << 40], np.uint64), np.array([0], np.uint64), 33)
    assert ei.value.status == cfp.CFP_EOVERFLOW


# ---------------------------------------------------------------- NEXT-3 counts
# cfp_profile_space is host arithmetic behind the C-ABI: checked here (no GPU)
# against the pinned oracle (tests/test_oracle_profiling.py).


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_profile_space_configs(cfp, cfg):
    from oracle import profiling as PR
    from synth import make_config
    p = make_config(cfg, 0, "shaped")
    assert cfp.profile_space(p) == PR.profile_space(p)


@pytest.mark.parametrize("seed", range(25))
def test_profile_space_random(cfp, seed):
    from oracle import profiling as PR
    from synth import generators as G
    p = G.tiny_random(9300 + seed, max_plans=None, max_n=4, max_k=5)
    assert cfp.profile_space(p) == PR.profile_space(p)


def test_profile_space_errors(cfp):
    import copy

    from synth import make_config
    p = copy.deepcopy(make_config("C2", 0, "shaped"))   # make_config caches: never mutate its result
    p.transitions[2].in_edges[0].dst = 9          # consumer block out of range
    with pytest.raises(cfp.CfpError) as ei:
        cfp.profile_space(p)
    assert ei.value.status == cfp.CFP_EINVAL
    p = copy.deepcopy(make_config("C2", 0, "shaped"))
    p.transitions[1].pred_type = 7
    with pytest.raises(cfp.CfpError) as ei:
        cfp.profile_space(p)
    assert ei.value.status == cfp.CFP_EINVAL


def test_marshal_cache_refills_values_in_place():
    """The binding caches a problem's marshalled structs; the edge / cross
    tables it hands to the C-ABI must follow in-place value changes and a
    replaced table object must invalidate the cache (no GPU needed)."""
    import copy
    import ctypes as C
    import numpy as np
    from paper_2504_00598_b200 import cfp
    from synth import make_config
    p = copy.deepcopy(make_config("C3", 0, "shaped"))
    cfp._Marshal().problem(p)
    t = p.types[2]
    off = sum(e.table.size for e in t.edges[:3])
    t.edges[3].table.flat[5] += 7
    s = cfp._Marshal().problem(p)
    assert C.cast(s.types[2].edge_ns, C.POINTER(C.c_uint32))[off + 5] == int(t.edges[3].table.flat[5])
    x = p.transitions[2].in_edges[1]
    x.table.flat[3] += 9
    s = cfp._Marshal().problem(p)
    off2 = p.transitions[2].in_edges[0].table.size
    assert C.cast(s.transitions[2].in_ns, C.POINTER(C.c_uint32))[off2 + 3] == int(x.table.flat[3])
    new = x.table.copy()
    new.flat[0] += 1
    x.table = new                                  # a new object: the cache must not be used
    s = cfp._Marshal().problem(p)
    assert C.cast(s.transitions[2].in_ns, C.POINTER(C.c_uint32))[off2] == int(new.flat[0])
    assert copy.deepcopy(p) is not None            # the cache does not ride on the object
