"""Seeded synthetic problem generators (inputs only; no method arithmetic).

Configs C1..C5 follow BASELINE.json `configs` made concrete in SURVEY.md §8(d)
and Appendix C.  Tables are produced by a documented counter-based hash
(splitmix64 of (seed, table id, entry)), so every input is reproducible from
(config, seed, dist) on any machine.  The "shaped" recipe prices each
ParallelBlock strategy with an alpha-beta model of the collectives it implies
(App. C); "random" draws U[0, 2^20); "ties" draws U[0, 3] to stress the
lowest-index tie-break.  Infeasible (divisibility-violating)
strategies are INF in every distribution.

The tiny random corpus (SURVEY §8(c) "Property-test corpus") uses numpy's
PCG64 generator seeded per problem.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .problem import (INF32, CrossEdge, Edge, Problem, SegmentType,
                      Transition)

U64 = np.uint64
MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------------
# counter-based hash
# --------------------------------------------------------------------------
def _splitmix64_int(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def _splitmix64_arr(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x.astype(U64) + U64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
        return z ^ (z >> U64(31))


def hash_stream(seed: int, table_id: int, n: int) -> np.ndarray:
    """h(seed, table_id, e) for e = 0..n-1 as uint64."""
    base = _splitmix64_int(_splitmix64_int(seed & MASK64) ^ (table_id & MASK64))
    e = np.arange(n, dtype=U64)
    return _splitmix64_arr(e ^ U64(base))


# --------------------------------------------------------------------------
# strategies on a mesh (App. C)
# --------------------------------------------------------------------------
DIMS_2D = ("B", "S", "N", "K", None)
DIMS_1D = ("M", "N", "K")


def strategies_for(mesh: Tuple[int, ...]) -> List[Tuple[Optional[str], ...]]:
    """Strategy = per-mesh-axis choice of the block head's partitioned dim.

    1-D mesh: D = 3 candidates {M (row), N (column), K (split-K)} (P:130-137,
    P:815).  2-D mesh: each axis picks one of {B, S, N, K, none}, the fully
    replicated choice excluded: D = 5^2 - 1 = 24."""
    if len(mesh) == 1:
        return [(d,) for d in DIMS_1D]
    assert len(mesh) == 2
    out = []
    for a in DIMS_2D:
        for b in DIMS_2D:
            if a is None and b is None:
                continue
            out.append((a, b))
    return out


class BlockShape:
    """Head matmul [M = B*S, K] x [K, N] of a ParallelBlock (bf16)."""

    def __init__(self, name: str, B: int, S: int, K: int, N: int):
        self.name, self.B, self.S, self.K, self.N = name, B, S, K, N

    def extent(self, dim: str) -> int:
        return {"B": self.B, "S": self.S, "M": self.B * self.S,
                "N": self.N, "K": self.K}[dim]


ALPHA_NS = 10_000.0          # 10 us
BETA_BYTES_PER_NS = 100.0    # 100 GB/s
FLOP_RATE = 1e14             # nominal FLOP/s
CAP_UNARY = 1 << 25          # p <= 2^25 and c <= 2^25  =>  p + c <= 2^26
CAP_PAIR = 1 << 24


def _split(strategy, mesh, dim_set) -> int:
    p = 1
    for ax, d in enumerate(strategy):
        if d in dim_set:
            p *= mesh[ax]
    return p


def feasible(shape: BlockShape, strategy, mesh) -> bool:
    for d in ("B", "S", "M", "N", "K"):
        p = _split(strategy, mesh, (d,))
        if p > 1 and shape.extent(d) % p != 0:
            return False
    return True


def unary_costs(shape: BlockShape, strategy, mesh, jitter: float) -> Tuple[int, int]:
    """(p, c) in integer ns for one block strategy (App. C shaped recipe)."""
    pm = _split(strategy, mesh, ("B", "S", "M"))
    pn = _split(strategy, mesh, ("N",))
    pk = _split(strategy, mesh, ("K",))
    M = shape.B * shape.S
    flops = 6.0 * M * shape.N * shape.K / (pm * pn * pk)
    p = math.ceil(flops / FLOP_RATE * 1e9 * (1.0 + 0.03 * jitter))
    c = 0.0
    wbytes = 2.0 * shape.K * shape.N / (pn * pk)
    for ax, d in enumerate(strategy):
        P = mesh[ax]
        if P == 1:
            continue
        if d not in ("K", "N"):      # weight replicated along this axis
            c += ALPHA_NS + 2.0 * (P - 1) / P * wbytes / BETA_BYTES_PER_NS
        if d == "K":                 # split-K partial output all-reduce
            obytes = 2.0 * M * shape.N / (pm * pn)
            c += ALPHA_NS + 2.0 * (P - 1) / P * obytes / BETA_BYTES_PER_NS
    return min(int(p), CAP_UNARY), min(int(math.ceil(c)), CAP_UNARY)


def block_memory_kib(shape: BlockShape, strategy, mesh) -> int:
    """Peak memory of one block strategy in KiB (NEXT-1 memory model, App. C
    style): bf16 weight + fp32 master copy + Adam moments = 16 B per parameter,
    sharded by the strategy's N and K splits, plus the bf16 output activation
    kept for backward, sharded by its M and N splits."""
    pm = _split(strategy, mesh, ("B", "S", "M"))
    pn = _split(strategy, mesh, ("N",))
    pk = _split(strategy, mesh, ("K",))
    M = shape.B * shape.S
    wstate = 16.0 * shape.K * shape.N / (pn * pk)
    act = 2.0 * M * shape.N / (pm * pn)
    return int(math.ceil((wstate + act) / 1024.0))


def _out_layout(d):
    return {"B": "B", "S": "S", "M": "M", "N": "H", "K": "P", None: "R"}[d]


def _in_layout(d):
    return {"B": "B", "S": "S", "M": "M", "K": "H", "N": "R", None: "R"}[d]


def reshard_cost(src_strategy, dst_strategy, mesh, act_bytes: float) -> int:
    """Sum over mesh axes of the primitive converting the producer's output
    layout to the consumer's expected input layout (App. C)."""
    out = [_out_layout(d) for d in src_strategy]
    inp = [_in_layout(d) for d in dst_strategy]
    total = 0.0
    for ax in range(len(mesh)):
        P = mesh[ax]
        a, b = out[ax], inp[ax]
        if a == b or P == 1:
            continue
        bytes_ = act_bytes
        for ox in range(len(mesh)):
            if ox != ax and out[ox] not in ("R", "P"):
                bytes_ /= mesh[ox]
        if a == "R":
            continue                         # replicated -> sharded: local slice
        if b == "R":
            f = 2.0 * (P - 1) / P if a == "P" else (P - 1) / P
        elif a == "P":
            f = (P - 1) / P                  # reduce-scatter
        else:
            f = (P - 1) / (P * P)            # all-to-all
        total += ALPHA_NS + f * bytes_ / BETA_BYTES_PER_NS
    return min(int(math.ceil(total)), CAP_PAIR)


# --------------------------------------------------------------------------
# config structures (App. C)
# --------------------------------------------------------------------------
CONFIGS = ("C1", "C2", "C3", "C4", "C5")
CONFIG_NAMES = {
    "C1": "toy 2-layer MLP graph (4 ParallelBlocks, 3 strategies each) on a 2x2 mesh",
    "C2": "GPT-2 small graph: 12 repeated segments, 1D mesh of 8 devices",
    "C3": "LLaMA-7B graph on 2D mesh 2x4, full segment enumeration",
    "C4": "GPT-3 13B graph on 4x8 mesh, large per-segment strategy spaces",
    "C5": "LLaMA-70B-shaped graph on 8x8 mesh, repeated-squaring chain over 80 layers",
}


def _gpt_layer(B, S, h, f):
    return [BlockShape("qkv+attn", B, S, h, 3 * h), BlockShape("o+res", B, S, h, h),
            BlockShape("fc1+gelu", B, S, h, f), BlockShape("fc2+res", B, S, f, h)]


def _llama_layer(B, S, h, f, kv):
    return [BlockShape("q+rope+attn", B, S, h, h), BlockShape("k+rope", B, S, h, kv),
            BlockShape("v", B, S, h, kv), BlockShape("o+res", B, S, h, h),
            BlockShape("gate+silu*mul", B, S, h, f), BlockShape("up", B, S, h, f),
            BlockShape("down+res", B, S, f, h)]


GPT_EDGES = [(0, 1), (1, 2), (2, 3), (1, 3)]
LLAMA_EDGES = [(1, 0), (2, 0), (0, 3), (3, 4), (3, 5), (5, 4), (4, 6), (3, 6)]


def _spec(cfg: str):
    """Returns (mesh, h, B, S, layer_shapes, edges, j_in, out_block, n_layers,
    vocab, toy_strategies)."""
    if cfg == "C1":
        B, S, h, f = 8, 128, 256, 1024
        shapes = [BlockShape("fc1+act", B, S, h, f), BlockShape("fc2", B, S, f, h)]
        return dict(mesh=(2, 2), h=h, B=B, S=S, layer=shapes, edges=[(0, 1)],
                    j_in=[0], out=1, layers=2, vocab=None, flat_mesh=(4,))
    if cfg == "C2":
        B, S, h, f = 8, 1024, 768, 3072
        return dict(mesh=(8,), h=h, B=B, S=S, layer=_gpt_layer(B, S, h, f),
                    edges=GPT_EDGES, j_in=[0], out=3, layers=12, vocab=50304)
    if cfg == "C3":
        B, S, h, f = 8, 2048, 4096, 11008
        return dict(mesh=(2, 4), h=h, B=B, S=S, layer=_llama_layer(B, S, h, f, h),
                    edges=LLAMA_EDGES, j_in=[0, 1, 2, 3], out=6, layers=32, vocab=32000)
    if cfg == "C4":
        B, S, h, f = 16, 2048, 5120, 20480
        two = _gpt_layer(B, S, h, f) + _gpt_layer(B, S, h, f)
        edges = GPT_EDGES + [(a + 4, b + 4) for a, b in GPT_EDGES] + [(3, 4), (3, 5)]
        return dict(mesh=(4, 8), h=h, B=B, S=S, layer=two, edges=edges,
                    j_in=[0, 1], out=7, layers=20, vocab=50304)
    if cfg == "C5":
        B, S, h, f, kv = 8, 4096, 8192, 28672, 1024
        return dict(mesh=(8, 8), h=h, B=B, S=S, layer=_llama_layer(B, S, h, f, kv),
                    edges=LLAMA_EDGES, j_in=[0, 1, 2, 3], out=6, layers=80, vocab=32000)
    raise ValueError(cfg)


class _Tables:
    """Per-(config, seed, dist) table factory; every table gets a unique id."""

    def __init__(self, seed: int, dist: str):
        self.seed, self.dist, self.next_id = seed, dist, 1

    def _tid(self) -> int:
        t = self.next_id
        self.next_id += 1
        return t

    def redraw(self, vals: np.ndarray, inf_mask: np.ndarray) -> np.ndarray:
        """Apply the distribution: shaped keeps `vals`; random/ties redraw
        every finite entry from the hash stream.  INF stays INF."""
        tid = self._tid()
        out = vals.astype(np.uint64).copy()
        if self.dist == "random":
            out = hash_stream(self.seed, tid, out.size).reshape(out.shape) % U64(1 << 20)
        elif self.dist == "ties":
            out = hash_stream(self.seed, tid, out.size).reshape(out.shape) % U64(4)
        elif self.dist != "shaped":
            raise ValueError(self.dist)
        out = out.astype(np.uint32)
        out[inf_mask] = INF32
        return out

    def jitter(self, n: int) -> np.ndarray:
        h = hash_stream(self.seed, self._tid(), n)
        return (h % U64(2001)).astype(np.float64) / 1000.0 - 1.0


def _block_strats(cfg_mesh, spec):
    mesh = spec.get("flat_mesh", cfg_mesh)
    return mesh, strategies_for(mesh)


def _segment_type(tables: _Tables, spec, shapes, edges, out_block, name) -> SegmentType:
    mesh, strats = _block_strats(spec["mesh"], spec)
    comp, comm, mem = [], [], []
    feas = []
    for shape in shapes:
        mem.append(np.array([block_memory_kib(shape, s, mesh) for s in strats], dtype=np.uint32))
        jit = tables.jitter(len(strats))
        f = np.array([feasible(shape, s, mesh) for s in strats])
        pc = [unary_costs(shape, s, mesh, jit[i]) for i, s in enumerate(strats)]
        p = np.array([x[0] for x in pc], dtype=np.uint64)
        c = np.array([x[1] for x in pc], dtype=np.uint64)
        comp.append(tables.redraw(p, ~f))
        comm.append(tables.redraw(c, ~f))
        feas.append(f)
    act = 2.0 * spec["B"] * spec["S"] * spec["h"]
    E = []
    for a, b in edges:
        R = np.array([[reshard_cost(sa, sb, mesh, act) for sb in strats] for sa in strats],
                     dtype=np.uint64)
        inf = ~(feas[a][:, None] & feas[b][None, :])
        E.append(Edge(a, b, tables.redraw(R, inf)))
    return SegmentType(radix=np.full(len(shapes), len(strats), dtype=np.int32),
                       comp_ns=np.concatenate(comp), comm_ns=np.concatenate(comm),
                       edges=E, out_block=out_block, name=name,
                       mem=np.concatenate(mem)), feas


def _cross(tables: _Tables, spec, pred_feas, pred_out, dst_feas, j_in) -> List[CrossEdge]:
    mesh, strats = _block_strats(spec["mesh"], spec)
    act = 2.0 * spec["B"] * spec["S"] * spec["h"]
    out = []
    for j in j_in:
        Q = np.array([[reshard_cost(sa, sb, mesh, act) for sb in strats] for sa in strats],
                     dtype=np.uint64)
        inf = ~(pred_feas[pred_out][:, None] & dst_feas[j][None, :])
        out.append(CrossEdge(j, tables.redraw(Q, inf)))
    return out


_CACHE: Dict[Tuple[str, int, str], Problem] = {}


def make_config(cfg: str, seed: int = 0, dist: str = "shaped") -> Problem:
    """Build config C1..C5.  Chain (App. C): E, L1, L x (layers-1), H for
    C2-C5 (types E=0, L1=1, L=2, H=3; transitions start->E, E->L1, L1->L,
    L->L, L->H); C1 is two instances of one MLP-layer type."""
    key = (cfg, seed, dist)
    if key in _CACHE:
        return _CACHE[key]
    spec = _spec(cfg)
    tables = _Tables(seed * 1_000_003 + CONFIGS.index(cfg) + 1, dist)
    mesh = spec["mesh"]
    if cfg == "C1":
        T, feas = _segment_type(tables, spec, spec["layer"], spec["edges"], spec["out"], "T")
        start = Transition(-1, 0, [], "start->T")
        tt = Transition(0, 0, _cross(tables, spec, feas, spec["out"], feas, spec["j_in"]), "T->T")
        prob = Problem(mesh, [T], [start, tt], np.array([0, 1], dtype=np.int32), cfg)
        _CACHE[key] = prob
        return prob
    B, S, h = spec["B"], spec["S"], spec["h"]
    emb = [BlockShape("embed", B, S, h, h)]
    head = [BlockShape("lm_head", B, S, h, spec["vocab"])]
    E, fe = _segment_type(tables, spec, emb, [], 0, "E")
    L1, f1 = _segment_type(tables, spec, spec["layer"], spec["edges"], spec["out"], "L1")
    L, fl = _segment_type(tables, spec, spec["layer"], spec["edges"], spec["out"], "L")
    H, fh = _segment_type(tables, spec, head, [], 0, "H")
    o = spec["out"]
    trs = [Transition(-1, 0, [], "start->E"),
           Transition(0, 1, _cross(tables, spec, fe, 0, f1, spec["j_in"]), "E->L1"),
           Transition(1, 2, _cross(tables, spec, f1, o, fl, spec["j_in"]), "L1->L"),
           Transition(2, 2, _cross(tables, spec, fl, o, fl, spec["j_in"]), "L->L"),
           Transition(2, 3, _cross(tables, spec, fl, o, fh, [0]), "L->H")]
    n_layers = spec["layers"]   # C4: 20 two-layer segments (GPT-3 13B: 40 layers)
    inst = [0, 1, 2] + [3] * (n_layers - 2) + [4]
    prob = Problem(mesh, [E, L1, L, H], trs, np.array(inst, dtype=np.int32), cfg)
    _CACHE[key] = prob
    return prob


def midsize(cfg: str, keep, n_layers: int = 6, seed: int = 0, dist: str = "shaped") -> Problem:
    """A config's graph with its layer types restricted to the blocks `keep`
    (renumbered in order), for parity tests of the full-size kernels at a size
    the oracle enumerates in seconds: the same radices (D = 24, or 23 feasible
    with the (B,B) strategy infeasible at C4/C5), value tables, edges among the
    kept blocks, cross tables of the kept consumer blocks and output block.
    Pure slicing of the config's inputs."""
    base = make_config(cfg, seed, dist)
    keep = list(keep)
    pos = {b: i for i, b in enumerate(keep)}

    def cut(t: SegmentType) -> SegmentType:
        o = t.offsets()
        sl = lambda a: None if a is None else np.concatenate([a[o[j]:o[j + 1]] for j in keep])
        edges = [Edge(pos[e.src], pos[e.dst], e.table) for e in t.edges if e.src in pos and e.dst in pos]
        return SegmentType(radix=t.radix[keep].copy(), comp_ns=sl(t.comp_ns), comm_ns=sl(t.comm_ns),
                           edges=edges, out_block=pos[t.out_block], name=t.name + "'", mem=sl(t.mem))

    E, L1, L, H = base.types
    types = [E, cut(L1), cut(L), H]
    trs = []
    for tr in base.transitions:
        if tr.type in (1, 2):
            xs = [CrossEdge(pos[x.dst], x.table) for x in tr.in_edges if x.dst in pos]
        else:
            xs = list(tr.in_edges)
        trs.append(Transition(tr.pred_type, tr.type, xs, tr.name))
    inst = [0, 1, 2] + [3] * (n_layers - 2) + [4]
    return Problem(base.mesh, types, trs, np.array(inst, dtype=np.int32),
                   f"{cfg}[{','.join(map(str, keep))}]x{n_layers}")


# --------------------------------------------------------------------------
# tiny random corpus
# --------------------------------------------------------------------------
def _draw_values(rng, shape, mode, p_inf=0.05):
    if mode == "ties":
        v = rng.integers(0, 4, size=shape, dtype=np.uint64)
    elif mode == "random":
        v = rng.integers(0, 1 << 20, size=shape, dtype=np.uint64)
    elif mode == "nearmax":
        v = rng.integers((1 << 31) - (1 << 10), 1 << 31, size=shape, dtype=np.uint64)
    elif mode == "wide":
        v = rng.integers(0, (1 << 32) - 1, size=shape, dtype=np.uint64)
    else:
        raise ValueError(mode)
    v = v.astype(np.uint32)
    if p_inf > 0:
        v[rng.random(shape) < p_inf] = INF32
    return v


def tiny_random(seed: int, mode: Optional[str] = None, max_n: int = 4, max_k: int = 3,
                max_d: int = 4, max_edges: int = 3, max_types: int = 3,
                max_run: int = 9, p_inf: float = 0.05,
                max_plans: Optional[int] = 10 ** 6) -> Problem:
    """Random small problem.  Structure: any J_in subset (incl. the output block
    and duplicates), o anywhere, both edge directions and multi-edges, mixed
    types, repeated transitions.  Values: ties / random / nearmax (forces the
    64-bit path), each entry INF w.p. p_inf, plus occasional whole-INF rows.
    If `max_plans` is set, N is reduced until the global plan count <= it."""
    rng = np.random.default_rng(seed)
    if mode is None:
        mode = ("ties", "random", "nearmax")[int(rng.integers(0, 3))]
    T = int(rng.integers(1, max_types + 1))
    types = []
    for t in range(T):
        K = int(rng.integers(1, max_k + 1))
        radix = rng.integers(1, max_d + 1, size=K).astype(np.int32)
        sD = int(radix.sum())
        comp = _draw_values(rng, (sD,), mode, p_inf)
        comm = _draw_values(rng, (sD,), mode, p_inf) if rng.random() < 0.7 else None
        edges = []
        if K > 1:
            for _ in range(int(rng.integers(0, max_edges + 1))):
                a, b = rng.choice(K, size=2, replace=False)
                tab = _draw_values(rng, (int(radix[a]), int(radix[b])), mode, p_inf)
                if rng.random() < 0.1:
                    tab[int(rng.integers(0, radix[a]))] = INF32
                edges.append(Edge(int(a), int(b), tab))
        o = int(rng.integers(0, K))
        # memory tables from a separate stream (keeps the cost streams of
        # earlier corpus versions unchanged): small integers so quantum = 1
        # brute force stays meaningful; None (all 0) w.p. 0.15
        mrng = np.random.default_rng([seed, 7, t])
        mem = (None if mrng.random() < 0.15 else
               mrng.integers(0, 6, size=sD).astype(np.uint32))
        types.append(SegmentType(radix, comp, comm, edges, o, f"T{t}", mem=mem))
    # chain of types with runs
    seq = []
    N_target = int(rng.integers(1, max_n + 1))
    while len(seq) < N_target:
        t = int(rng.integers(0, T))
        run = int(rng.integers(1, max_run + 1))
        seq.extend([t] * run)
    seq = seq[:N_target]
    # plan-count guard for brute force
    if max_plans is not None:
        while True:
            cnt = 1
            for t in seq:
                cnt *= int(np.prod([int(d) for d in types[t].radix]))
            if cnt <= max_plans or len(seq) == 1:
                break
            seq = seq[:-1]
    trans, tid = [], {}
    inst = []
    prev = -1
    for t in seq:
        key = (prev, t)
        if key not in tid:
            ty = types[t]
            d_in = 1 if prev < 0 else int(types[prev].radix[types[prev].out_block])
            X = []
            nx = int(rng.integers(0, min(ty.K, 3) + 1))
            for _ in range(nx):
                j = int(rng.integers(0, ty.K))
                tab = _draw_values(rng, (d_in, int(ty.radix[j])), mode, p_inf)
                if rng.random() < 0.1:
                    tab[:, int(rng.integers(0, ty.radix[j]))] = INF32
                X.append(CrossEdge(j, tab))
            tid[key] = len(trans)
            trans.append(Transition(prev, t, X, f"{prev}->{t}"))
        inst.append(tid[key])
        prev = t
    return Problem((2, 2), types, trans, np.array(inst, dtype=np.int32), f"tiny{seed}:{mode}")


def global_plan_count(p: Problem) -> int:
    n = 1
    for t in p.instances:
        n *= p.num_combinations(p.transitions[int(t)].type)
    return n


# --------------------------------------------------------------------------
# dense per-plan tables: one profiled time per
# whole-segment plan.  W[idx] from the counter-based hash of
# (seed, DENSE_TABLE_ID + type, idx): 24-bit ns, INF when the low 12 bits are 0
# (about one plan in 4096 infeasible).  The library's device generator
# (cfp_dense_fill) implements the same splitmix64 stream from dense_base().
# --------------------------------------------------------------------------
DENSE_TABLE_ID = 1 << 32


def dense_base(seed: int, type_id: int) -> int:
    return _splitmix64_int(_splitmix64_int(seed & MASK64) ^ ((DENSE_TABLE_ID + type_id) & MASK64))


def dense_table(seed: int, type_id: int, n: int, lo: int = 0) -> np.ndarray:
    """W[lo .. lo + n) of type `type_id` as uint32."""
    e = np.arange(lo, lo + n, dtype=U64)
    h = _splitmix64_arr(e ^ U64(dense_base(seed, type_id)))
    w = (h >> U64(40)).astype(np.uint32)
    w[(h & U64(0xFFF)) == U64(0)] = np.uint32(INF32)
    return w

