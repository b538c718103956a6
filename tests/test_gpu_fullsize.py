"""Parity of the exact enumeration kernels the bench times, bucket by bucket.

The bench configurations run the fully unrolled A-loop enumeration variant
(`enum_kernel<u32, 24|23, 2, 1, 24|23>`, NB = D of the output block) with the
output block in the register group (C3, C5: o_mode 0) or in the M loop (C4:
o_mode 1).  The random corpora use D <= 6 and never reach those instantiations,
so here:

* mid-size problems cut from the configs' own graphs (synth.generators.midsize:
  the same D = 24 / 23-feasible radices, tables, edges and cross tables on a
  subset of each layer's blocks), forced onto the bench's schedule where the
  planner would pick another one for the smaller prefix space
  (CFP_ENUM_NB / CFP_ENUM_O_IN_M / CFP_ENUM_P), the schedule asserted through
  cfp_prepared_query, and EVERY bucket's (A, I) of every used transition -- read
  through the prepared search itself (cfp_prepared_tables) -- compared with the
  oracle's exhaustive table (Eq. 3, least index SURVEY App. A);
* the full-size C3 / C5 problems against oracle goldens written by
  tests/golden/make_full_golden.py (oracle/ only): every bucket of every
  transition and the plan; C4 against exhaustively enumerated oracle buckets.
"""
import json
import os

import numpy as np
import pytest

from synth import make_config
from synth.generators import midsize

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _ctx(env):
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return cfp.Context(device=0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


# (config, kept blocks, overrides, expected o_mode of the layer types, NB)
MIDSIZE = [
    ("C3", [3, 4, 5, 6], {"CFP_ENUM_NB": "24"}, 0, 24),
    ("C5", [3, 4, 5, 6], {}, 0, 23),
    ("C5", [2, 3, 4, 5, 6], {}, 0, 23),
    ("C4", [1, 4, 5, 6, 7], {"CFP_ENUM_NB": "23", "CFP_ENUM_O_IN_M": "1", "CFP_ENUM_P": "1"}, 1, 23),
    ("C3", [2, 3, 4, 5, 6], {"CFP_ENUM_NB": "24"}, 0, 24),
]


# the layer loop's instruction mix (CFP_ENUM_MIX): default two-pipe groups of
# 3 A values, groups of 4, and the ALU-only loop
@pytest.mark.parametrize("mix", ["3", "4", "0"])
@pytest.mark.parametrize("case", MIDSIZE, ids=lambda c: f"{c[0]}-{len(c[1])}blocks")
def test_midsize_every_bucket_bench_kernel(oracle_lib, case, mix):
    cfg, keep, env, o_mode, nb = case
    if mix != "3" and o_mode == 0 and len(keep) > 4:
        pytest.skip("mix variants on the 4-block o_mode-0 problems and C4's layout (time)")
    O = oracle_lib
    ctx = _ctx({**env, "CFP_ENUM_MIX": mix})
    p = midsize(cfg, keep, n_layers=6)
    prep = ctx.prepare(p)
    info = prep.info()
    # types: E, L1', L', H -> the two layer types run the bench's kernel variant
    for slot in (1, 2):
        assert info.full_a[slot] == 1, (cfg, keep, info)
        assert info.o_mode[slot] == o_mode, (cfg, keep, info)
        assert info.schedule[slot][1] == nb and info.schedule[slot][2] == 1, (cfg, keep, info)
    assert info.fused_tail
    m = O.Marshalled(p)
    for tr in sorted(set(int(t) for t in p.instances)):
        A0, I0 = O.segment_table(p, tr, m=m)
        A, I = prep.tables(tr, p.d_in(tr), p.d_out(tr))
        assert np.array_equal(A, A0), (cfg, keep, tr)
        assert np.array_equal(I, I0), (cfg, keep, tr)
    want = O.search_plan(p)
    prep.execute()
    got = prep.fetch()
    assert got.total_ns == want["total"]
    assert got.seg_index.tolist() == want["seg_index"].tolist()
    assert got.seg_ns.tolist() == want["seg_ns"].tolist()
    prep.close()
    ctx.close()


def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"missing golden {name}: run tests/golden/make_full_golden.py")
    with open(path) as f:
        return json.load(f)


def _sha(prob):
    import importlib.util
    spec = importlib.util.spec_from_file_location("mkg", os.path.join(GOLDEN, "make_full_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.problem_sha256(prob)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_full_size_every_bucket_and_plan_vs_oracle_golden(ctx, cfg):
    """Every bucket (A, I) of every used transition and the canonical plan at
    full size, against the oracle's exhaustive tables and chain."""
    g = _golden(f"full_{cfg}_shaped_s0.json")
    p = make_config(cfg, 0, "shaped")
    assert g["problem_sha256"] == _sha(p), "generator changed since the golden was written"
    prep = ctx.prepare(p)
    info = prep.info()
    assert info.full_a[1] == 1 and info.full_a[2] == 1
    for tr, tab in g["tables"].items():
        tr = int(tr)
        A, I = prep.tables(tr, p.d_in(tr), p.d_out(tr))
        assert A.tolist() == tab["A"], (cfg, tr)
        assert I.tolist() == tab["I"], (cfg, tr)
    prep.execute()
    got = prep.fetch()
    assert got.total_ns == g["total"]
    assert got.seg_index.tolist() == g["seg_index"]
    assert got.seg_ns.tolist() == g["seg_ns"]
    prep.close()
    plan = ctx.search_plan(p)                      # the public call, same answer
    assert plan.total_ns == g["total"] and plan.seg_index.tolist() == g["seg_index"]


@pytest.mark.slow
def test_c4_sampled_buckets_vs_oracle_golden(ctx):
    """C4 (1.57e11 combinations; whole tables are out of the oracle's reach):
    seeded buckets of every layer transition, each enumerated exhaustively by
    the oracle, against the bench schedule's tables (o in M, NB = 23)."""
    g = _golden("buckets_C4_shaped_s0.json")
    p = make_config("C4", 0, "shaped")
    assert g["problem_sha256"] == _sha(p)
    prep = ctx.prepare(p)
    info = prep.info()
    assert info.full_a[1] == 1 and info.full_a[2] == 1 and info.o_mode[1] == 1 and info.o_mode[2] == 1
    tabs = {}
    for b in g["buckets"]:
        tr = b["tr"]
        if tr not in tabs:
            tabs[tr] = prep.tables(tr, p.d_in(tr), p.d_out(tr))
        A, I = tabs[tr]
        assert int(A[b["u"], b["v"]]) == b["A"], b
        assert int(I[b["u"], b["v"]]) == b["I"], b
    prep.close()


@pytest.fixture(scope="module")
def ctx():
    c = _ctx({})
    yield c
    c.close()
