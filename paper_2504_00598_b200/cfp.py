"""Thin ctypes binding of include/cfp.h (argument marshalling only).

Every step of the search runs in libcfp.so's sm_100a kernels; this module
only converts numpy arrays / problem objects to the C structs and back.  There
is no CPU fallback: if the library or a CUDA device is missing, the calls
raise CfpError.

Problem objects are duck-typed: anything with `.types` (radix, comp_ns,
comm_ns, edges[(src, dst, table)], out_block), `.transitions` (pred_type,
type, in_edges[(dst, table)]), `.instances` and `.mesh` -- e.g.
`synth.Problem`.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcfp.so")

CFP_ABI_VERSION = 1
INF64 = (1 << 64) - 1
NOIDX = INF64
STATUS = {0: "CFP_OK", 1: "CFP_EINVAL", 2: "CFP_EOVERFLOW", 3: "CFP_EINFEASIBLE",
          4: "CFP_ETOOBIG", 5: "CFP_ECUDA", 6: "CFP_ENCCL", 7: "CFP_ENOMEM", 8: "CFP_EVERSION"}
CFP_OK, CFP_EINVAL, CFP_EOVERFLOW, CFP_EINFEASIBLE, CFP_ETOOBIG = 0, 1, 2, 3, 4
CFP_ECUDA, CFP_ENCCL, CFP_ENOMEM, CFP_EVERSION = 5, 6, 7, 8


class CfpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


P = C.POINTER


class cfp_mesh(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("axes", P(C.c_int32))]


# pointer members are declared c_void_p (same ABI as the typed pointers of
# cfp.h) so that marshalling assigns raw addresses without ctypes casts
class cfp_segment_type(C.Structure):
    _fields_ = [("num_blocks", C.c_int32), ("radix", C.c_void_p), ("comp_ns", C.c_void_p),
                ("comm_ns", C.c_void_p), ("num_edges", C.c_int32), ("edge_src", C.c_void_p),
                ("edge_dst", C.c_void_p), ("edge_ns", C.c_void_p), ("out_block", C.c_int32)]


class cfp_transition(C.Structure):
    _fields_ = [("pred_type", C.c_int32), ("type", C.c_int32), ("num_in_edges", C.c_int32),
                ("in_dst", C.c_void_p), ("in_ns", C.c_void_p)]


class cfp_problem(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("mesh", cfp_mesh), ("num_types", C.c_int32),
                ("types", P(cfp_segment_type)), ("num_transitions", C.c_int32),
                ("transitions", P(cfp_transition)), ("num_instances", C.c_int32),
                ("inst_transition", C.c_void_p)]


class cfp_plan(C.Structure):
    _fields_ = [("total_ns", C.c_uint64), ("seg_index", P(C.c_uint64)), ("digits", P(C.c_int32)),
                ("kmax", C.c_int32), ("seg_ns", P(C.c_uint64))]


class cfp_mem_model(C.Structure):
    _fields_ = [("quantum", C.c_uint64), ("mem_limit", C.c_uint64), ("type_mem", P(P(C.c_uint32)))]


class cfp_budget_result(C.Structure):
    _fields_ = [("tasks", C.c_uint64), ("pruned", C.c_uint64), ("infeasible", C.c_uint64),
                ("spent_lo", C.c_uint64), ("spent_hi", C.c_uint64), ("full_lo", C.c_uint64),
                ("full_hi", C.c_uint64), ("best", C.c_uint64), ("best_index", C.c_uint64)]


class cfp_ctx_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("cuda_stream", C.c_void_p), ("world", C.c_int32),
                ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p)]


class cfp_prepared_info(C.Structure):
    _fields_ = [("combos", C.c_double), ("combos_local", C.c_double), ("evals", C.c_double),
                ("num_types", C.c_int32), ("num_transitions", C.c_int32), ("wide_types", C.c_int32),
                ("kernel_launches", C.c_int32), ("prefix_len", C.c_int32 * 32),
                ("nb", C.c_int32 * 32), ("na", C.c_int32 * 32), ("fused_tail", C.c_int32),
                ("tail_grid", C.c_int32), ("o_mode", C.c_int32 * 32), ("full_a", C.c_int32 * 32)]


EXPORTS = ["cfp_ctx_create", "cfp_ctx_destroy", "cfp_last_error", "cfp_nccl_unique_id",
           "cfp_segment_costs", "cfp_minplus_chain", "cfp_search_plan", "cfp_minplus_product",
           "cfp_prepare", "cfp_execute", "cfp_fetch_plan", "cfp_prepared_free",
           "cfp_ctx_nccl_info", "cfp_prepared_tables", "cfp_prepared_query", "cfp_prepared_time_kernels", "cfp_prepared_kernel_ms", "cfp_prepared_phase_ms",
           "cfp_shard_range", "cfp_pack_keys", "cfp_unpack_keys", "cfp_intpipe_bench",
           "cfp_minplus_bench", "cfp_search_plan_mem", "cfp_segment_costs_mem", "cfp_mem_prepare",
           "cfp_mem_execute", "cfp_mem_fetch_plan", "cfp_mem_free", "cfp_mem_time_kernels",
           "cfp_mem_kernel_ms", "cfp_mem_fold_ops", "cfp_dense_fill", "cfp_dense_shard", "cfp_search_plan_dense",
           "cfp_segment_costs_dense", "cfp_dense_prepare", "cfp_dense_execute", "cfp_dense_fetch_plan",
           "cfp_dense_free", "cfp_dense_time_kernels", "cfp_dense_kernel_ms", "cfp_profile_space",
           "cfp_profile_budget"]

_lib = None


def lib() -> C.CDLL:
    """Load libcfp.so (built in-tree by paper_2504_00598_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CfpError(CFP_ECUDA, f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.cfp_ctx_create.argtypes = [P(vp), P(cfp_ctx_opts)]
    L.cfp_ctx_destroy.argtypes = [vp]
    L.cfp_ctx_destroy.restype = None
    L.cfp_last_error.restype = C.c_char_p
    L.cfp_nccl_unique_id.argtypes = [vp]
    L.cfp_segment_costs.argtypes = [vp, P(cfp_segment_type), P(cfp_transition), C.c_int32,
                                    P(C.c_uint64), P(C.c_uint64)]
    L.cfp_minplus_chain.argtypes = [vp, C.c_int32, P(C.c_int32), P(C.c_int32), P(P(C.c_uint64)),
                                    C.c_int32, P(C.c_int32), P(C.c_int64), P(C.c_uint64),
                                    P(C.c_uint64), P(C.c_uint64)]
    L.cfp_search_plan.argtypes = [vp, P(cfp_problem), P(cfp_plan)]
    L.cfp_minplus_product.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, P(C.c_uint64),
                                      P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]
    L.cfp_prepare.argtypes = [vp, P(cfp_problem), P(vp)]
    L.cfp_execute.argtypes = [vp, vp]
    L.cfp_fetch_plan.argtypes = [vp, vp, P(cfp_plan)]
    L.cfp_prepared_free.argtypes = [vp]
    L.cfp_prepared_free.restype = None
    L.cfp_prepared_query.argtypes = [vp, P(cfp_prepared_info)]
    L.cfp_prepared_time_kernels.argtypes = [vp, C.c_int32]
    L.cfp_prepared_kernel_ms.argtypes = [vp, P(C.c_double), P(C.c_double)]
    L.cfp_prepared_phase_ms.argtypes = [vp, P(C.c_double)]
    L.cfp_ctx_nccl_info.argtypes = [vp, P(C.c_int32), P(C.c_int32)]
    L.cfp_prepared_tables.argtypes = [vp, vp, C.c_int32, P(C.c_uint64), P(C.c_uint64)]
    L.cfp_shard_range.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, P(C.c_int64), P(C.c_int64)]
    L.cfp_pack_keys.argtypes = [C.c_int64, P(C.c_uint64), P(C.c_uint64), C.c_int32, P(C.c_uint64)]
    L.cfp_unpack_keys.argtypes = [C.c_int64, P(C.c_uint64), C.c_int32, P(C.c_uint64), P(C.c_uint64)]
    L.cfp_intpipe_bench.argtypes = [vp, C.c_int32, C.c_int32, P(C.c_double), P(C.c_double)]
    L.cfp_minplus_bench.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_double),
                                    P(C.c_double)]
    L.cfp_search_plan_mem.argtypes = [vp, P(cfp_problem), P(cfp_mem_model), P(cfp_plan), P(C.c_int64),
                                      P(C.c_int64)]
    L.cfp_segment_costs_mem.argtypes = [vp, P(cfp_segment_type), P(C.c_uint32), C.c_uint64,
                                        P(cfp_transition), C.c_int32, P(C.c_int64), P(C.c_int32),
                                        P(C.c_uint64), P(C.c_uint64)]
    L.cfp_mem_prepare.argtypes = [vp, P(cfp_problem), P(cfp_mem_model), P(vp)]
    L.cfp_mem_execute.argtypes = [vp, vp]
    L.cfp_mem_fetch_plan.argtypes = [vp, vp, P(cfp_plan), P(C.c_int64), P(C.c_int64)]
    L.cfp_mem_free.argtypes = [vp]
    L.cfp_mem_free.restype = None
    L.cfp_mem_time_kernels.argtypes = [vp, C.c_int32]
    L.cfp_mem_kernel_ms.argtypes = [vp, P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
                                    P(C.c_int32)]
    L.cfp_mem_fold_ops.argtypes = [vp, P(C.c_double)]
    L.cfp_dense_fill.argtypes = [vp, vp, C.c_uint64, C.c_uint64]
    L.cfp_dense_shard.argtypes = [vp, P(cfp_segment_type), P(C.c_int64), P(C.c_int64)]
    L.cfp_search_plan_dense.argtypes = [vp, P(cfp_problem), P(vp), P(cfp_plan)]
    L.cfp_segment_costs_dense.argtypes = [vp, P(cfp_segment_type), vp, P(cfp_transition), C.c_int32,
                                          P(C.c_uint64), P(C.c_uint64)]
    L.cfp_dense_prepare.argtypes = [vp, P(cfp_problem), P(vp), P(vp)]
    L.cfp_dense_execute.argtypes = [vp, vp]
    L.cfp_dense_fetch_plan.argtypes = [vp, vp, P(cfp_plan)]
    L.cfp_dense_free.argtypes = [vp]
    L.cfp_dense_free.restype = None
    L.cfp_dense_time_kernels.argtypes = [vp, C.c_int32]
    L.cfp_dense_kernel_ms.argtypes = [vp, P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
                                      P(C.c_int32)]
    L.cfp_profile_space.argtypes = [P(cfp_problem), P(C.c_int64), P(C.c_int64), P(C.c_int64)]
    L.cfp_profile_budget.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, P(cfp_budget_result),
                                     P(C.c_double)]
    _lib = L
    return L


def _check(status: int):
    if status != CFP_OK:
        raise CfpError(status, lib().cfp_last_error().decode(errors="replace"))


def _p(a: Optional[np.ndarray], ct):
    return None if a is None else a.ctypes.data_as(P(ct))


def _a(a: Optional[np.ndarray]) -> Optional[int]:
    """Raw address of a contiguous array (for c_void_p members)."""
    return None if a is None else a.__array_interface__["data"][0]


# ---------------------------------------------------------------- marshalling
class _Marshal:
    def __init__(self):
        self.keep = []
        self.concat = []        # concatenated edge / cross tables, in marshalling order

    def arr(self, a, dtype):
        if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
            a = np.ascontiguousarray(a, dtype=dtype)
        self.keep.append(a)
        return a

    def segment_type(self, ty) -> cfp_segment_type:
        radix = self.arr(ty.radix, np.int32)
        comp = self.arr(ty.comp_ns, np.uint32)
        comm = None if ty.comm_ns is None else self.arr(ty.comm_ns, np.uint32)
        edges = list(ty.edges)
        src = self.arr([_e(e)[0] for e in edges] or [0], np.int32)
        dst = self.arr([_e(e)[1] for e in edges] or [0], np.int32)
        tab = self.arr(np.concatenate([np.asarray(_e(e)[2], np.uint32).ravel() for e in edges])
                       if edges else np.zeros(1, np.uint32), np.uint32)
        if edges:
            self.concat.append(tab)
        return cfp_segment_type(len(radix), _a(radix), _a(comp), _a(comm), len(edges), _a(src),
                                _a(dst), _a(tab), int(ty.out_block))

    def transition(self, tr) -> cfp_transition:
        xs = list(tr.in_edges)
        dst = self.arr([_x(x)[0] for x in xs] or [0], np.int32)
        tab = self.arr(np.concatenate([np.asarray(_x(x)[1], np.uint32).ravel() for x in xs])
                       if xs else np.zeros(1, np.uint32), np.uint32)
        if xs:
            self.concat.append(tab)
        return cfp_transition(int(tr.pred_type), int(tr.type), len(xs), _a(dst), _a(tab))

    def problem(self, prob) -> cfp_problem:
        cached = _cached_problem(prob)
        if cached is not None:
            self.keep.append(cached[1])
            return cached[0]
        types = (cfp_segment_type * len(prob.types))(*[self.segment_type(t) for t in prob.types])
        trans = (cfp_transition * len(prob.transitions))(*[self.transition(t) for t in prob.transitions])
        self.keep += [types, trans]
        mesh = self.arr(list(prob.mesh) or [1], np.int32)
        inst = self.arr(prob.instances, np.int32)
        struct = cfp_problem(CFP_ABI_VERSION, cfp_mesh(len(prob.mesh), _p(mesh, C.c_int32)),
                             len(prob.types), types, len(prob.transitions), trans, len(inst), _a(inst))
        _cache_problem(prob, self, struct)
        return struct


# Marshalled problems are cached on the problem object: a repeated call with the
# same array objects (shapes, dtypes, contiguity unchanged) reuses the ctypes
# structs; the concatenated edge / cross tables are refilled from the current
# arrays on every call (np.concatenate(out=...)), and every other pointer is
# the caller's own array, so in-place value changes are always seen.
def _sig(prob):
    """Identity / shape signature of every array the marshalled struct refers to."""
    s = [len(prob.types), len(prob.transitions), id(prob.instances), prob.instances.shape, tuple(prob.mesh)]
    for t in prob.types:
        s += [id(t.radix), id(t.comp_ns), id(t.comm_ns), t.comp_ns.shape, t.out_block, len(t.edges)]
        s += [id(e.table) if hasattr(e, "table") else id(e[2]) for e in t.edges]
    for tr in prob.transitions:
        s += [tr.pred_type, tr.type, len(tr.in_edges)]
        s += [id(x.table) if hasattr(x, "table") else id(x[1]) for x in tr.in_edges]
    return tuple(s)


_MCACHE = {}        # id(problem) -> (weakref, entry); entries die with their problem


def _cached_problem(prob):
    hit = _MCACHE.get(id(prob))
    if hit is None or hit[0]() is not prob:
        return None
    c = hit[1]
    if c[0] != _sig(prob):
        return None
    _, struct, keep, views, buf = c
    if views:
        np.concatenate(views, out=buf)    # current values of every edge / cross table
    return struct, keep


def _cache_problem(prob, m: "_Marshal", struct):
    """Remember the marshalled struct (called after a fresh marshal): all
    concatenated tables move into one buffer refilled by a single concatenate."""
    srcs = [[_e(e)[2] for e in t.edges] for t in prob.types if t.edges]
    srcs += [[_x(x)[1] for x in tr.in_edges] for tr in prob.transitions if tr.in_edges]
    if len(srcs) != len(m.concat):
        return
    # the cache may only point at arrays it keeps alive and that are the caller's own
    for t in prob.types:
        for a in (t.radix, t.comp_ns, t.comm_ns):
            if a is not None and not any(a is k for k in m.keep):
                return                  # converted copy: a later in-place change would be missed
    if not any(prob.instances is k for k in m.keep):
        return
    views = []
    for group in srcs:
        for a in group:
            if not (isinstance(a, np.ndarray) and a.dtype == np.uint32 and a.flags.c_contiguous):
                return
            views.append(a.reshape(-1))
    buf = np.concatenate(views) if views else np.zeros(1, np.uint32)
    # re-point the structs at slices of the shared buffer
    off = 0
    slots = [(struct.types[i], "edge_ns") for i, t in enumerate(prob.types) if t.edges]
    slots += [(struct.transitions[i], "in_ns") for i, tr in enumerate(prob.transitions) if tr.in_edges]
    base = buf.__array_interface__["data"][0]
    for (obj, field), cat in zip(slots, m.concat):
        setattr(obj, field, base + off * 4)
        off += cat.size
    try:
        ref = weakref.ref(prob)
        weakref.finalize(prob, _MCACHE.pop, id(prob), None)
    except TypeError:           # objects without weak references: no cache
        return
    _MCACHE[id(prob)] = (ref, (_sig(prob), struct, list(m.keep) + [buf], views, buf))


def _mem_model(m: "_Marshal", prob, quantum: int, mem_limit: int) -> cfp_mem_model:
    """Per-type m_j[s] tables (P:573 peak memory per strategy; NEXT-1)."""
    ptrs = []
    for t in prob.types:
        mem = getattr(t, "mem", None)
        ptrs.append(None if mem is None else _p(m.arr(mem, np.uint32), C.c_uint32))
    arr = (P(C.c_uint32) * len(ptrs))(*ptrs)
    m.keep.append(arr)
    return cfp_mem_model(int(quantum), int(mem_limit), arr)


def _e(e):
    return (e.src, e.dst, e.table) if hasattr(e, "src") else e


def _x(x):
    return (x.dst, x.table) if hasattr(x, "dst") else x


def profile_space(prob) -> dict:
    """Eq. 2 counts through the C-ABI (host arithmetic, no GPU):
    whole-segment plans per type, reshard pairs per transition, total."""
    m = _Marshal()
    p = m.problem(prob)
    tp = np.zeros(len(prob.types), np.int64)
    xp = np.zeros(len(prob.transitions), np.int64)
    tot = C.c_int64(0)
    _check(lib().cfp_profile_space(C.byref(p), _p(tp, C.c_int64), _p(xp, C.c_int64), C.byref(tot)))
    return dict(type_plans=[int(x) for x in tp], trans_pairs=[int(x) for x in xp], total=int(tot.value))


@dataclass
class Plan:
    total_ns: int
    seg_index: np.ndarray      # uint64 [N]
    digits: np.ndarray         # int32 [N, kmax]
    seg_ns: np.ndarray         # uint64 [N]


@dataclass
class PlanMem:
    total_ns: int
    seg_index: np.ndarray      # uint64 [N]
    digits: np.ndarray         # int32 [N, kmax]
    seg_ns: np.ndarray         # uint64 [N]
    seg_q: np.ndarray          # int64 [N] quantised memory of each segment
    total_q: int


@dataclass
class PreparedInfo:
    combos: float
    combos_local: float
    evals: float
    num_types: int
    num_transitions: int
    wide_types: int
    kernel_launches: int
    schedule: List[Tuple[int, int, int, int]]   # per type (prefix_len, NB, VG, na)
    fused_tail: bool = False
    tail_grid: int = 0
    o_mode: Tuple[int, ...] = ()      # per type: output block in B (0), M (1), prefix (2)
    full_a: Tuple[int, ...] = ()      # per type: 1 = fully unrolled A-loop enumeration kernel


class Context:
    """cfp_ctx wrapper: one per process / GPU."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, world: int = 1, rank: int = 0,
                 nccl_unique_id: Optional[bytes] = None):
        L = lib()
        self._h = C.c_void_p()
        uid = None
        if nccl_unique_id is not None:     # world > 1 without one: shard simulation (cfp.h)
            if len(nccl_unique_id) != 128:
                raise CfpError(CFP_EINVAL, "the nccl unique id has 128 bytes")
            uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
        opts = cfp_ctx_opts(device, stream, world, rank, C.cast(uid, C.c_void_p) if uid else None)
        _check(L.cfp_ctx_create(C.byref(self._h), C.byref(opts)))
        self.world, self.rank, self.device = world, rank, device

    def nccl_info(self) -> Tuple[int, int]:
        """(ranks of the ctx's communicator, NCCL version code); (0, 0) without one."""
        n, v = C.c_int32(), C.c_int32()
        _check(lib().cfp_ctx_nccl_info(self._h, C.byref(n), C.byref(v)))
        return n.value, v.value

    def close(self):
        if self._h:
            lib().cfp_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- (1)
    def segment_costs(self, seg_type, transition=None, d_in: int = 1) -> Tuple[np.ndarray, np.ndarray]:
        m = _Marshal()
        t = m.segment_type(seg_type)
        tr = m.transition(transition) if transition is not None else None
        do = int(np.asarray(seg_type.radix)[int(seg_type.out_block)])
        A = np.empty((d_in, do), np.uint64)
        I = np.empty((d_in, do), np.uint64)
        _check(lib().cfp_segment_costs(self._h, C.byref(t), C.byref(tr) if tr is not None else None,
                                       d_in, _p(A, C.c_uint64), _p(I, C.c_uint64)))
        return A, I

    # -- (2)
    def minplus_chain(self, mats: Sequence[np.ndarray], runs: Sequence[Tuple[int, int]],
                      terminal: Optional[np.ndarray] = None, suffix: bool = True):
        mats = [np.ascontiguousarray(M, dtype=np.uint64) for M in mats]
        rows = np.array([M.shape[0] for M in mats], np.int32)
        cols = np.array([M.shape[1] for M in mats], np.int32)
        ptrs = (P(C.c_uint64) * len(mats))(*[_p(M, C.c_uint64) for M in mats])
        run_mat = np.array([r[0] for r in runs], np.int32)
        run_len = np.array([r[1] for r in runs], np.int64)
        N = int(run_len.sum())
        term = None if terminal is None else np.ascontiguousarray(terminal, dtype=np.uint64)
        opt = np.zeros(1, np.uint64)
        total = int(rows[run_mat[0]]) + int(sum(int(cols[run_mat[r]]) * int(run_len[r])
                                                 for r in range(len(runs))))
        suf = np.empty(total, np.uint64) if suffix else None
        _check(lib().cfp_minplus_chain(self._h, len(mats), _p(rows, C.c_int32), _p(cols, C.c_int32),
                                       ptrs, len(runs), _p(run_mat, C.c_int32), _p(run_len, C.c_int64),
                                       _p(term, C.c_uint64), _p(opt, C.c_uint64), _p(suf, C.c_uint64)))
        if not suffix:
            return int(opt[0]), None
        out, off = [suf[:rows[run_mat[0]]]], int(rows[run_mat[0]])
        for r in range(len(runs)):
            c = int(cols[run_mat[r]])
            for _ in range(int(run_len[r])):
                out.append(suf[off:off + c])
                off += c
        assert len(out) == N + 1
        return int(opt[0]), out

    # -- (3)
    def search_plan(self, prob) -> Plan:
        m = _Marshal()
        p = m.problem(prob)
        N = len(prob.instances)
        kmax = max(int(len(t.radix)) for t in prob.types)
        idx = np.empty(N, np.uint64)
        dig = np.empty(N * kmax, np.int32)
        seg = np.empty(N, np.uint64)
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_search_plan(self._h, C.byref(p), C.byref(plan)))
        return Plan(int(plan.total_ns), idx, dig.reshape(N, kmax), seg)

    def minplus_product(self, A: np.ndarray, B: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        A = np.ascontiguousarray(A, dtype=np.uint64)
        B = np.ascontiguousarray(B, dtype=np.uint64)
        m, k = A.shape
        k2, n = B.shape
        if k != k2:
            raise CfpError(CFP_EINVAL, "inner dimensions differ")
        Cm = np.empty((m, n), np.uint64)
        arg = np.empty((m, n), np.uint64)
        _check(lib().cfp_minplus_product(self._h, m, k, n, _p(A, C.c_uint64), _p(B, C.c_uint64),
                                         _p(Cm, C.c_uint64), _p(arg, C.c_uint64)))
        return Cm, arg

    def prepare(self, prob) -> "Prepared":
        return Prepared(self, prob)

    # -- memory-constrained search (NEXT-1)
    def search_plan_mem(self, prob, quantum: int, mem_limit: int) -> PlanMem:
        m = _Marshal()
        p = m.problem(prob)
        mm = _mem_model(m, prob, quantum, mem_limit)
        N = len(prob.instances)
        kmax = max(int(len(t.radix)) for t in prob.types)
        idx = np.empty(N, np.uint64)
        dig = np.empty(N * kmax, np.int32)
        seg = np.empty(N, np.uint64)
        sq = np.empty(N, np.int64)
        tq = C.c_int64()
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_search_plan_mem(self._h, C.byref(p), C.byref(mm), C.byref(plan),
                                         _p(sq, C.c_int64), C.byref(tq)))
        return PlanMem(int(plan.total_ns), idx, dig.reshape(N, kmax), seg, sq, tq.value)

    def segment_costs_mem(self, seg_type, quantum: int, transition=None, d_in: int = 1):
        """(Am [d_in][D_o][nq], Im, qlo) of one transition (memory-bucketed)."""
        m = _Marshal()
        t = m.segment_type(seg_type)
        tr = m.transition(transition) if transition is not None else None
        mem = getattr(seg_type, "mem", None)
        mp = None if mem is None else _p(m.arr(mem, np.uint32), C.c_uint32)
        qlo, nq = C.c_int64(), C.c_int32()
        trp = C.byref(tr) if tr is not None else None
        _check(lib().cfp_segment_costs_mem(self._h, C.byref(t), mp, int(quantum), trp, d_in,
                                           C.byref(qlo), C.byref(nq), None, None))
        do = int(np.asarray(seg_type.radix)[int(seg_type.out_block)])
        A = np.empty((d_in, do, nq.value), np.uint64)
        I = np.empty((d_in, do, nq.value), np.uint64)
        _check(lib().cfp_segment_costs_mem(self._h, C.byref(t), mp, int(quantum), trp, d_in,
                                           C.byref(qlo), C.byref(nq), _p(A, C.c_uint64), _p(I, C.c_uint64)))
        return A, I, qlo.value

    def prepare_mem(self, prob, quantum: int, mem_limit: int) -> "PreparedMem":
        return PreparedMem(self, prob, quantum, mem_limit)

    # -- dense per-plan tables (NEXT-2); W arguments are device pointers (int)
    def dense_fill(self, w_ptr: int, n: int, base: int):
        _check(lib().cfp_dense_fill(self._h, C.c_void_p(w_ptr), n, base))

    def dense_shard(self, seg_type) -> Tuple[int, int]:
        """(first, count): the combination indices of seg_type's dense table
        this rank holds (world > 1; (0, prod D) at world 1)."""
        m = _Marshal()
        t = m.segment_type(seg_type)
        first, count = C.c_int64(), C.c_int64()
        _check(lib().cfp_dense_shard(self._h, C.byref(t), C.byref(first), C.byref(count)))
        return first.value, count.value

    def search_plan_dense(self, prob, w_ptrs: Sequence[Optional[int]]) -> Plan:
        m = _Marshal()
        p = m.problem(prob)
        arr = (C.c_void_p * len(w_ptrs))(*[C.c_void_p(x) if x else None for x in w_ptrs])
        N = len(prob.instances)
        kmax = max(int(len(t.radix)) for t in prob.types)
        idx = np.empty(N, np.uint64)
        dig = np.empty(N * kmax, np.int32)
        seg = np.empty(N, np.uint64)
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_search_plan_dense(self._h, C.byref(p), C.cast(arr, P(C.c_void_p)), C.byref(plan)))
        return Plan(int(plan.total_ns), idx, dig.reshape(N, kmax), seg)

    def segment_costs_dense(self, seg_type, w_ptr: int, transition=None, d_in: int = 1):
        m = _Marshal()
        t = m.segment_type(seg_type)
        tr = m.transition(transition) if transition is not None else None
        do = int(np.asarray(seg_type.radix)[int(seg_type.out_block)])
        A = np.empty((d_in, do), np.uint64)
        I = np.empty((d_in, do), np.uint64)
        _check(lib().cfp_segment_costs_dense(self._h, C.byref(t), C.c_void_p(w_ptr),
                                             C.byref(tr) if tr is not None else None, d_in,
                                             _p(A, C.c_uint64), _p(I, C.c_uint64)))
        return A, I

    def prepare_dense(self, prob, w_ptrs) -> "PreparedDense":
        return PreparedDense(self, prob, w_ptrs)

    # -- dynamic profiling budget (NEXT-3); W is a device pointer (int)
    def profile_budget(self, w_ptr: int, n: int, num: int, den: int, timed: bool = False):
        """Budgeted profiling of one type's dense table in index order; returns
        a dict (tasks, pruned, infeasible, spent, full, best, best_index) and,
        with timed=True, also the device ms of the call's kernels."""
        r = cfp_budget_result()
        ms = C.c_double(0.0)
        _check(lib().cfp_profile_budget(self._h, C.c_void_p(w_ptr) if w_ptr else None, int(n), int(num),
                                        int(den), C.byref(r), C.byref(ms) if timed else None))
        out = dict(tasks=int(r.tasks), pruned=int(r.pruned), infeasible=int(r.infeasible),
                   spent=(int(r.spent_hi) << 64) | int(r.spent_lo),
                   full=(int(r.full_hi) << 64) | int(r.full_lo),
                   best=int(r.best), best_index=int(r.best_index))
        return (out, ms.value) if timed else out

    def minplus_bench(self, S: int, wide: bool = False, argk: bool = False, iters: int = 5):
        """(ms per launch, add+min ops per second) of an S^3 (min,+) product."""
        ms, ops = C.c_double(), C.c_double()
        _check(lib().cfp_minplus_bench(self._h, S, int(wide), int(argk), iters, C.byref(ms), C.byref(ops)))
        return ms.value, ops.value

    def intpipe_bench(self, op: int = 0, iters: int = 20000) -> Tuple[float, float]:
        ops, ms = C.c_double(), C.c_double()
        _check(lib().cfp_intpipe_bench(self._h, op, iters, C.byref(ops), C.byref(ms)))
        return ops.value, ms.value


class Prepared:
    """Device-resident problem: prepare once, execute many times."""

    def __init__(self, ctx: Context, prob):
        self.ctx = ctx
        self._m = _Marshal()
        p = self._m.problem(prob)
        self._h = C.c_void_p()
        _check(lib().cfp_prepare(ctx._h, C.byref(p), C.byref(self._h)))
        self.N = len(prob.instances)
        self.kmax = max(int(len(t.radix)) for t in prob.types)

    def execute(self):
        _check(lib().cfp_execute(self.ctx._h, self._h))

    def fetch(self) -> Plan:
        idx = np.empty(self.N, np.uint64)
        dig = np.empty(self.N * self.kmax, np.int32)
        seg = np.empty(self.N, np.uint64)
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), self.kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_fetch_plan(self.ctx._h, self._h, C.byref(plan)))
        return Plan(int(plan.total_ns), idx, dig.reshape(self.N, self.kmax), seg)

    def info(self) -> PreparedInfo:
        i = cfp_prepared_info()
        _check(lib().cfp_prepared_query(self._h, C.byref(i)))
        sched = [(i.prefix_len[t], i.nb[t] // 100, i.nb[t] % 100, i.na[t]) for t in range(i.num_types)]
        return PreparedInfo(i.combos, i.combos_local, i.evals, i.num_types, i.num_transitions,
                            i.wide_types, i.kernel_launches, sched, bool(i.fused_tail), i.tail_grid,
                            tuple(i.o_mode[t] for t in range(i.num_types)),
                            tuple(i.full_a[t] for t in range(i.num_types)))

    def tables(self, transition: int, d_in: int, d_out: int) -> Tuple[np.ndarray, np.ndarray]:
        """(A, I) of one transition through this prepared search's schedule and kernels."""
        A = np.empty((d_in, d_out), np.uint64)
        I = np.empty((d_in, d_out), np.uint64)
        _check(lib().cfp_prepared_tables(self.ctx._h, self._h, transition, _p(A, C.c_uint64), _p(I, C.c_uint64)))
        return A, I

    def time_kernels(self, on=True):
        """0 off, 1 (True): events around a0 / enumeration / whole path, 2: + every phase."""
        _check(lib().cfp_prepared_time_kernels(self._h, int(on)))

    PHASES = ("a0_stage", "a1_enumerate", "a1_reduce_a2_allreduce", "a3_chain", "a1_argmin_a2_merge",
              "a4_backtrack")

    def phase_ms(self) -> Dict[str, float]:
        """Device ms of each hot-path phase of the last execute (timing level 2)."""
        ms = (C.c_double * 6)()
        _check(lib().cfp_prepared_phase_ms(self._h, ms))
        return {k: float(v) for k, v in zip(self.PHASES, ms)}

    def kernel_ms(self) -> Tuple[float, float]:
        a, b = C.c_double(), C.c_double()
        _check(lib().cfp_prepared_kernel_ms(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if self._h:
            lib().cfp_prepared_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PreparedMem:
    """Device-resident memory-constrained search: prepare once, execute many times."""

    def __init__(self, ctx: Context, prob, quantum: int, mem_limit: int):
        self.ctx = ctx
        self._m = _Marshal()
        p = self._m.problem(prob)
        mm = _mem_model(self._m, prob, quantum, mem_limit)
        self._h = C.c_void_p()
        _check(lib().cfp_mem_prepare(ctx._h, C.byref(p), C.byref(mm), C.byref(self._h)))
        self.N = len(prob.instances)
        self.kmax = max(int(len(t.radix)) for t in prob.types)

    def execute(self):
        _check(lib().cfp_mem_execute(self.ctx._h, self._h))

    def fetch(self) -> PlanMem:
        idx = np.empty(self.N, np.uint64)
        dig = np.empty(self.N * self.kmax, np.int32)
        seg = np.empty(self.N, np.uint64)
        sq = np.empty(self.N, np.int64)
        tq = C.c_int64()
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), self.kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_mem_fetch_plan(self.ctx._h, self._h, C.byref(plan), _p(sq, C.c_int64),
                                        C.byref(tq)))
        return PlanMem(int(plan.total_ns), idx, dig.reshape(self.N, self.kmax), seg, sq, tq.value)

    def time_kernels(self, on: bool = True):
        _check(lib().cfp_mem_time_kernels(self._h, 1 if on else 0))

    def kernel_ms(self):
        """(enumeration ms, enumeration+fold+minima ms, total ms, combinations per
        execute, kernel launches) of the last execute."""
        e, a, b, c, n = C.c_double(), C.c_double(), C.c_double(), C.c_double(), C.c_int32()
        _check(lib().cfp_mem_kernel_ms(self._h, C.byref(e), C.byref(a), C.byref(b), C.byref(c), C.byref(n)))
        return e.value, a.value, b.value, c.value, n.value

    def fold_ops(self) -> float:
        f = C.c_double()
        _check(lib().cfp_mem_fold_ops(self._h, C.byref(f)))
        return f.value

    def close(self):
        if self._h:
            lib().cfp_mem_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PreparedDense:
    """Device-resident dense-table search (tables stay where the caller put them)."""

    def __init__(self, ctx: Context, prob, w_ptrs):
        self.ctx = ctx
        self._m = _Marshal()
        p = self._m.problem(prob)
        self._arr = (C.c_void_p * len(w_ptrs))(*[C.c_void_p(x) if x else None for x in w_ptrs])
        self._h = C.c_void_p()
        _check(lib().cfp_dense_prepare(ctx._h, C.byref(p), C.cast(self._arr, P(C.c_void_p)), C.byref(self._h)))
        self.N = len(prob.instances)
        self.kmax = max(int(len(t.radix)) for t in prob.types)

    def execute(self):
        _check(lib().cfp_dense_execute(self.ctx._h, self._h))

    def fetch(self) -> Plan:
        idx = np.empty(self.N, np.uint64)
        dig = np.empty(self.N * self.kmax, np.int32)
        seg = np.empty(self.N, np.uint64)
        plan = cfp_plan(0, _p(idx, C.c_uint64), _p(dig, C.c_int32), self.kmax, _p(seg, C.c_uint64))
        _check(lib().cfp_dense_fetch_plan(self.ctx._h, self._h, C.byref(plan)))
        return Plan(int(plan.total_ns), idx, dig.reshape(self.N, self.kmax), seg)

    def time_kernels(self, on: bool = True):
        _check(lib().cfp_dense_time_kernels(self._h, 1 if on else 0))

    def kernel_ms(self):
        """(table-stream ms, total ms, combinations, table bytes, kernel launches)."""
        a, b, c, d, n = C.c_double(), C.c_double(), C.c_double(), C.c_double(), C.c_int32()
        _check(lib().cfp_dense_kernel_ms(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d), C.byref(n)))
        return a.value, b.value, c.value, d.value, n.value

    def close(self):
        if self._h:
            lib().cfp_dense_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- host-only helpers
def shard_range(units: int, align: int, world: int, rank: int) -> Tuple[int, int]:
    lo, hi = C.c_int64(), C.c_int64()
    _check(lib().cfp_shard_range(units, align, world, rank, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def pack_keys(cost: np.ndarray, idx: np.ndarray, idx_bits: int) -> np.ndarray:
    cost = np.ascontiguousarray(cost, np.uint64)
    idx = np.ascontiguousarray(idx, np.uint64)
    keys = np.empty_like(cost)
    _check(lib().cfp_pack_keys(cost.size, _p(cost, C.c_uint64), _p(idx, C.c_uint64), idx_bits,
                               _p(keys, C.c_uint64)))
    return keys


def unpack_keys(keys: np.ndarray, idx_bits: int) -> Tuple[np.ndarray, np.ndarray]:
    keys = np.ascontiguousarray(keys, np.uint64)
    cost = np.empty_like(keys)
    idx = np.empty_like(keys)
    _check(lib().cfp_unpack_keys(keys.size, _p(keys, C.c_uint64), idx_bits, _p(cost, C.c_uint64),
                                 _p(idx, C.c_uint64)))
    return cost, idx


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().cfp_nccl_unique_id(buf))
    return buf.raw
