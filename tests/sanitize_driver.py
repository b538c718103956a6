"""Small end-to-end run of every CUDA path, for compute-sanitizer (memcheck,
racecheck, synccheck) -- driven by tests/test_gpu_sanitizer.py.

Each path runs on tiny inputs and is checked against the oracle, so a
sanitizer run also fails on a wrong answer.  Exit status 0 = every check held.
Usage: python tests/sanitize_driver.py [plain|mem|dense|budget|all]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from synth import generators as G  # noqa: E402


def check_plan(got, want, name):
    assert got.total_ns == want["total"], (name, got.total_ns, want["total"])
    assert got.seg_index.tolist() == want["seg_index"].tolist(), name


def plain(cfp):
    for env in ({}, {"CFP_FUSED_TAIL": "0"}, {"CFP_TAIL_SQUARING": "1"}):
        os.environ.update(env)
        ctx = cfp.Context(device=0)
        for k in env:
            del os.environ[k]
        probs = [G.make_config("C1", 0, "shaped"), G.make_config("C2", 1, "ties")]
        probs += [G.tiny_random(s, mode=("ties", "random", "nearmax")[s % 3], max_plans=None, max_n=8,
                                max_k=4, max_d=5) for s in range(6)]
        for p in probs:
            try:
                want = O.search_plan(p)
            except O.OracleError:
                continue
            check_plan(ctx.search_plan(p), want, p.name)
        p = G.tiny_random(3, max_k=4, max_d=5, max_plans=None)
        for tr_id, tr in enumerate(p.transitions):
            A0, I0 = O.segment_table(p, tr_id)
            A, I = ctx.segment_costs(p.types[tr.type], tr, p.d_in(tr_id))
            assert np.array_equal(A, A0) and np.array_equal(I, I0)
        rng = np.random.default_rng(1)
        mats = [rng.integers(0, 100, size=(1 if n == 0 else 5, 5)).astype(np.uint64) for n in range(2)]
        opt, _ = ctx.minplus_chain(mats, [(0, 1), (1, 6)])
        Gs = O.chain([mats[0]] + [mats[1]] * 6)
        assert opt == int(Gs[0][0])
        ctx.close()


def mem(cfp):
    ctx = cfp.Context(device=0)
    for s in range(6):
        p = G.tiny_random(2500 + s, max_plans=None, max_k=4, max_d=4)
        for quantum, frac in ((1, 0.5), (3, 0.7)):
            m = O.Marshalled(p)
            lo = sum(O.mem_range(p, p.transitions[int(t)].type, quantum, m)[0] for t in p.instances)
            hi = sum(O.mem_range(p, p.transitions[int(t)].type, quantum, m)[1] for t in p.instances)
            limit = int((lo + frac * (hi - lo)) * quantum)
            try:
                want = O.search_plan_mem(p, quantum, limit)
            except O.OracleError:
                continue
            got = ctx.search_plan_mem(p, quantum, limit)
            assert got.total_ns == want["total"] and got.seg_index.tolist() == want["seg_index"].tolist()
    ctx.close()


def dense(cfp):
    import torch
    ctx = cfp.Context(device=0)
    for s in range(4):
        p = G.tiny_random(7200 + s, max_plans=None, max_k=3, max_d=5)
        rng = np.random.default_rng(s)
        Ws = [rng.integers(0, 1 << 20, size=p.num_combinations(t), dtype=np.uint64).astype(np.uint32)
              for t in range(len(p.types))]
        devs = [torch.from_numpy(w.view(np.int32)).cuda() for w in Ws]
        try:
            want = O.dense_search_plan(p, Ws)
        except O.OracleError:
            continue
        got = ctx.search_plan_dense(p, [d.data_ptr() for d in devs])
        check_plan(got, want, p.name)
    ctx.close()


def budget(cfp):
    import torch

    from oracle import profiling as PR
    ctx = cfp.Context(device=0)
    rng = np.random.default_rng(0)
    for n in (1, 4097, 70001):
        W = rng.integers(0, 1 << 24, size=n, dtype=np.uint64).astype(np.uint32)
        W[rng.random(n) < 0.1] = np.uint32(0xFFFFFFFF)
        t = torch.from_numpy(W.view(np.int32)).cuda()
        assert ctx.profile_budget(t.data_ptr(), n, 3, 2) == PR.budget(W, 3, 2)
    ctx.close()


def main():
    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    O.build()
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("plain", plain), ("mem", mem), ("dense", dense), ("budget", budget)):
        if which in (name, "all"):
            fn(cfp)
            print(f"{name}: ok", flush=True)


if __name__ == "__main__":
    main()
