"""Write full-size oracle goldens for the bench configurations (TEST INFRASTRUCTURE).

Calls only `oracle/` (and `synth/` for the seeded inputs): every value this
script stores is computed by the plain C oracle -- nothing comes from the CUDA
path (task rule: "a stored value is ... written by a committed script that
calls only oracle/").

  full_<cfg>_<dist>_s<seed>.json
    * `problem_sha256`: digest of every input array, so a generator change is
      detected instead of silently comparing against stale values;
    * for every transition the instance list uses: the whole segment table
      A_tau[u][v] / I_tau[u][v] (Eq. 3, S = prod D P:477)
      from `orc_segment_table` -- every (u, s) recomputed from scratch;
    * the textbook backward DP and forward-greedy reconstruction
      over those tables: OPT, the canonical plan (seg_index, seg_ns).
  buckets_<cfg>_<dist>_s<seed>.json (configs too large for whole tables, C4)
    * `orc_bucket` for a seeded sample of (transition, u, v) buckets of every
      large used transition: exhaustive enumeration of the bucket's sub-space.

Cost (8 host cores): C3 ~2.5 h, C5 ~2 h, C4 buckets ~1.5 min each.  Run once:
    nice -n 19 python tests/golden/make_full_golden.py C3 C5
    nice -n 19 python tests/golden/make_full_golden.py --buckets C4
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from synth import make_config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def problem_sha256(prob) -> str:
    """Digest of every input array of the problem, in a fixed order."""
    h = hashlib.sha256()

    def add(a):
        if a is None:
            h.update(b"none")
        else:
            a = np.ascontiguousarray(a)
            h.update(str(a.dtype).encode() + str(a.shape).encode())
            h.update(a.tobytes())

    for t in prob.types:
        add(t.radix), add(t.comp_ns), add(t.comm_ns), add(np.array([t.out_block]))
        for e in t.edges:
            add(np.array([e.src, e.dst])), add(e.table)
    for tr in prob.transitions:
        add(np.array([tr.pred_type, tr.type]))
        for x in tr.in_edges:
            add(np.array([x.dst])), add(x.table)
    add(prob.instances)
    return h.hexdigest()


def full(cfg: str, seed: int, dist: str, nthreads: int) -> None:
    prob = make_config(cfg, seed, dist)
    m = O.Marshalled(prob)
    used = sorted(set(int(t) for t in prob.instances))
    tables = {}
    for tr in used:
        t0 = time.time()
        A, I = O.segment_table(prob, tr, nthreads=nthreads, m=m)
        tables[tr] = (A, I)
        print(f"{cfg} transition {tr}: {time.time() - t0:.0f} s", flush=True)
    mats = [tables[int(t)][0] for t in prob.instances]
    idxs = [tables[int(t)][1] for t in prob.instances]
    G = O.chain(mats)
    v, ix, cost = O.reconstruct(mats, idxs, G)
    out = {
        "what": f"oracle segment tables + plan for {cfg} ({dist}, seed {seed}); "
                "written by tests/golden/make_full_golden.py (oracle/ only)",
        "cite": "Eq. 3 P:613; S = prod D P:477; DP P:625-627; canonical plan SURVEY App. A",
        "config": cfg, "seed": seed, "dist": dist,
        "problem_sha256": problem_sha256(prob),
        "tables": {str(tr): {"A": [[int(x) for x in row] for row in tables[tr][0]],
                             "I": [[int(x) for x in row] for row in tables[tr][1]]} for tr in used},
        "total": int(G[0][0]),
        "seg_index": [int(x) for x in ix],
        "seg_ns": [int(x) for x in cost],
    }
    path = os.path.join(HERE, f"full_{cfg}_{dist}_s{seed}.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, flush=True)


def buckets(cfg: str, seed: int, dist: str, nthreads: int, per_tr: int) -> None:
    prob = make_config(cfg, seed, dist)
    m = O.Marshalled(prob)
    used = sorted(set(int(t) for t in prob.instances))
    rng = np.random.default_rng(12345)
    big = [tr for tr in used if prob.types[prob.transitions[tr].type].radix.size > 1]
    rows = []
    for tr in big:
        din, dout = prob.d_in(tr), prob.d_out(tr)
        for _ in range(per_tr):
            u, v = int(rng.integers(din)), int(rng.integers(dout))
            t0 = time.time()
            a, i = O.bucket(prob, tr, u, v, nthreads=nthreads, m=m)
            rows.append({"tr": tr, "u": u, "v": v, "A": a, "I": i})
            print(f"{cfg} tr {tr} ({u},{v}) -> {a} @ {i}: {time.time() - t0:.0f} s", flush=True)
    out = {
        "what": f"oracle buckets (exhaustive) for {cfg} ({dist}, seed {seed}); "
                "written by tests/golden/make_full_golden.py (oracle/ only)",
        "cite": "A[u][v] = min over s with s_o = v of Eq. 3 (P:613), least index (SURVEY App. A)",
        "config": cfg, "seed": seed, "dist": dist,
        "problem_sha256": problem_sha256(prob),
        "buckets": rows,
    }
    path = os.path.join(HERE, f"buckets_{cfg}_{dist}_s{seed}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dist", default="shaped")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--buckets", action="store_true")
    ap.add_argument("--per-transition", type=int, default=4)
    args = ap.parse_args()
    O.build()
    for cfg in args.configs:
        if args.buckets:
            buckets(cfg, args.seed, args.dist, args.threads, args.per_transition)
        else:
            full(cfg, args.seed, args.dist, args.threads)


if __name__ == "__main__":
    main()
