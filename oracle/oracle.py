"""ctypes front end of the C oracle + a pure-Python brute force.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs; never by the product
package.  Marshals `synth.Problem` into the oracle's own structs
(oracle/cfp_oracle.h) -- no code is shared with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from itertools import product
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from synth.problem import INF32, Problem

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcfp_oracle.so")
INF64 = (1 << 64) - 1
NOIDX = INF64

ORC_OK, ORC_EINVAL, ORC_EINFEASIBLE, ORC_ETOOBIG, ORC_ENOMEM = 0, 1, 3, 4, 7


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "cfp_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "cfp_oracle.h"))):
        tmp = LIB_PATH + ".tmp"   # rename into place: a running process keeps its mapping
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, src])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Type(C.Structure):
    _fields_ = [("K", C.c_int32), ("radix", C.POINTER(C.c_int32)),
                ("comp", C.POINTER(C.c_uint32)), ("comm", C.POINTER(C.c_uint32)),
                ("E", C.c_int32), ("esrc", C.POINTER(C.c_int32)),
                ("edst", C.POINTER(C.c_int32)), ("etab", C.POINTER(C.c_uint32)),
                ("out_block", C.c_int32), ("mem", C.POINTER(C.c_uint32))]


class _Trans(C.Structure):
    _fields_ = [("pred", C.c_int32), ("type", C.c_int32), ("X", C.c_int32),
                ("xdst", C.POINTER(C.c_int32)), ("xtab", C.POINTER(C.c_uint32))]


class _Problem(C.Structure):
    _fields_ = [("ntypes", C.c_int32), ("types", C.POINTER(_Type)),
                ("ntrans", C.c_int32), ("trans", C.POINTER(_Trans)),
                ("N", C.c_int32), ("inst", C.POINTER(C.c_int32))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.orc_cost_index.restype = C.c_uint64
        L.orc_cost_index.argtypes = [P(_Problem), C.c_int32, C.c_int32, C.c_uint64]
        L.orc_segment_table.argtypes = [P(_Problem), C.c_int32, P(C.c_uint64), P(C.c_uint64), C.c_int]
        L.orc_segment_table_range.argtypes = [P(_Problem), C.c_int32, C.c_uint64, C.c_uint64,
                                              P(C.c_uint64), P(C.c_uint64), C.c_int]
        L.orc_bucket.argtypes = [P(_Problem), C.c_int32, C.c_int32, C.c_int32,
                                 P(C.c_uint64), P(C.c_uint64), C.c_int]
        L.orc_chain.argtypes = [C.c_int32, P(C.c_int32), P(C.c_int32), P(P(C.c_uint64)),
                                P(C.c_uint64), P(C.c_uint64)]
        L.orc_reconstruct.argtypes = [C.c_int32, P(C.c_int32), P(C.c_int32), P(P(C.c_uint64)),
                                      P(P(C.c_uint64)), P(C.c_uint64), P(C.c_int32),
                                      P(C.c_uint64), P(C.c_uint64)]
        L.orc_search_plan.argtypes = [P(_Problem), C.c_int, P(C.c_uint64), P(C.c_uint64),
                                      P(C.c_int32), C.c_int32, P(C.c_uint64)]
        L.orc_segment_table_mem_range.argtypes = [P(_Problem), C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64,
                                                  P(C.c_uint64), P(C.c_uint64), C.c_int]
        L.orc_dense_segment_table.argtypes = [P(_Problem), C.c_int32, P(C.c_uint32), P(C.c_uint64),
                                              P(C.c_uint64), C.c_int]
        L.orc_dense_search_plan.argtypes = [P(_Problem), P(P(C.c_uint32)), C.c_int, P(C.c_uint64),
                                            P(C.c_uint64), P(C.c_int32), C.c_int32, P(C.c_uint64)]
        L.orc_minplus.argtypes = [C.c_int32, C.c_int32, C.c_int32, P(C.c_uint64), P(C.c_uint64),
                                  P(C.c_uint64), P(C.c_uint64)]
        L.orc_mem_range.argtypes = [P(_Type), C.c_uint64, P(C.c_int64), P(C.c_int64)]
        L.orc_segment_table_mem.argtypes = [P(_Problem), C.c_int32, C.c_uint64, P(C.c_uint64),
                                            P(C.c_uint64), C.c_int]
        L.orc_chain_mem.argtypes = [C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                    P(C.c_int64), P(P(C.c_uint64)), C.c_int64, P(C.c_uint64)]
        L.orc_reconstruct_mem.argtypes = [C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                          P(C.c_int64), P(P(C.c_uint64)), P(P(C.c_uint64)),
                                          C.c_int64, P(C.c_uint64), P(C.c_int32), P(C.c_int64),
                                          P(C.c_uint64), P(C.c_uint64)]
        L.orc_search_plan_mem.argtypes = [P(_Problem), C.c_uint64, C.c_uint64, C.c_int,
                                          P(C.c_uint64), P(C.c_uint64), P(C.c_int32), C.c_int32,
                                          P(C.c_uint64), P(C.c_int64), P(C.c_int64)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Marshalled:
    """Keeps numpy buffers alive for the lifetime of the C struct."""

    def __init__(self, prob: Problem):
        self.keep: List[np.ndarray] = []
        types = (_Type * len(prob.types))()
        for i, ty in enumerate(prob.types):
            radix = self._k(np.ascontiguousarray(ty.radix, dtype=np.int32))
            comp = self._k(np.ascontiguousarray(ty.comp_ns, dtype=np.uint32))
            comm = None if ty.comm_ns is None else self._k(
                np.ascontiguousarray(ty.comm_ns, dtype=np.uint32))
            esrc = self._k(np.array([e.src for e in ty.edges] or [0], dtype=np.int32))
            edst = self._k(np.array([e.dst for e in ty.edges] or [0], dtype=np.int32))
            etab = self._k(np.concatenate([np.ascontiguousarray(e.table, dtype=np.uint32).ravel()
                                           for e in ty.edges]) if ty.edges
                           else np.zeros(1, np.uint32))
            mem = None if ty.mem is None else self._k(np.ascontiguousarray(ty.mem, dtype=np.uint32))
            types[i] = _Type(ty.K, _ptr(radix, C.c_int32), _ptr(comp, C.c_uint32),
                             _ptr(comm, C.c_uint32) if comm is not None else None,
                             len(ty.edges), _ptr(esrc, C.c_int32), _ptr(edst, C.c_int32),
                             _ptr(etab, C.c_uint32), ty.out_block,
                             _ptr(mem, C.c_uint32) if mem is not None else None)
        trans = (_Trans * len(prob.transitions))()
        for i, tr in enumerate(prob.transitions):
            xdst = self._k(np.array([x.dst for x in tr.in_edges] or [0], dtype=np.int32))
            xtab = self._k(np.concatenate([np.ascontiguousarray(x.table, dtype=np.uint32).ravel()
                                           for x in tr.in_edges]) if tr.in_edges
                           else np.zeros(1, np.uint32))
            trans[i] = _Trans(tr.pred_type, tr.type, len(tr.in_edges), _ptr(xdst, C.c_int32),
                              _ptr(xtab, C.c_uint32))
        inst = self._k(np.ascontiguousarray(prob.instances, dtype=np.int32))
        self.types, self.trans = types, trans
        self.s = _Problem(len(prob.types), types, len(prob.transitions), trans,
                          len(prob.instances), _ptr(inst, C.c_int32))

    def _k(self, a):
        self.keep.append(a)
        return a

    @property
    def ref(self):
        return C.byref(self.s)


def _check(rc: int, what: str):
    if rc != ORC_OK:
        raise OracleError(rc, what)


class OracleError(RuntimeError):
    def __init__(self, rc, what):
        super().__init__(f"oracle {what} failed with status {rc}")
        self.rc = rc


def cost_index(prob: Problem, tr: int, u: int, idx: int, m: Optional[Marshalled] = None) -> int:
    m = m or Marshalled(prob)
    return int(lib().orc_cost_index(m.ref, tr, u, idx))


def segment_table(prob: Problem, tr: int, nthreads: int = 0,
                  m: Optional[Marshalled] = None) -> Tuple[np.ndarray, np.ndarray]:
    m = m or Marshalled(prob)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.empty((din, dout), dtype=np.uint64)
    I = np.empty((din, dout), dtype=np.uint64)
    _check(lib().orc_segment_table(m.ref, tr, _ptr(A, C.c_uint64), _ptr(I, C.c_uint64), nthreads),
           "segment_table")
    return A, I


def segment_table_range(prob: Problem, tr: int, lo: int, hi: int, nthreads: int = 0,
                        m: Optional[Marshalled] = None) -> Tuple[np.ndarray, np.ndarray]:
    """A/I restricted to combination indices [lo, hi) (all input states u)."""
    m = m or Marshalled(prob)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.empty((din, dout), dtype=np.uint64)
    I = np.empty((din, dout), dtype=np.uint64)
    _check(lib().orc_segment_table_range(m.ref, tr, lo, hi, _ptr(A, C.c_uint64), _ptr(I, C.c_uint64),
                                         nthreads), "segment_table_range")
    return A, I


def bucket(prob: Problem, tr: int, u: int, v: int, nthreads: int = 0,
           m: Optional[Marshalled] = None) -> Tuple[int, int]:
    m = m or Marshalled(prob)
    a, i = C.c_uint64(), C.c_uint64()
    _check(lib().orc_bucket(m.ref, tr, u, v, C.byref(a), C.byref(i), nthreads), "bucket")
    return int(a.value), int(i.value)


def _mat_ptrs(mats: Sequence[np.ndarray]):
    arr = (C.POINTER(C.c_uint64) * len(mats))()
    for i, M in enumerate(mats):
        arr[i] = _ptr(M, C.c_uint64)
    return arr


def chain(mats: Sequence[np.ndarray], terminal: Optional[np.ndarray] = None) -> List[np.ndarray]:
    """Backward DP; returns [G_0, G_1, ..., G_N]."""
    mats = [np.ascontiguousarray(M, dtype=np.uint64) for M in mats]
    N = len(mats)
    rows = np.array([M.shape[0] for M in mats], dtype=np.int32)
    cols = np.array([M.shape[1] for M in mats], dtype=np.int32)
    G = np.empty(int(rows[0] + cols.sum()), dtype=np.uint64)
    term = None
    if terminal is not None:
        term = np.ascontiguousarray(terminal, dtype=np.uint64)
    _check(lib().orc_chain(N, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32), _mat_ptrs(mats),
                           _ptr(term, C.c_uint64) if term is not None else None,
                           _ptr(G, C.c_uint64)), "chain")
    out, off = [G[:rows[0]]], int(rows[0])
    for c in cols:
        out.append(G[off:off + int(c)])
        off += int(c)
    return out


def reconstruct(mats, idxs, G: List[np.ndarray]):
    mats = [np.ascontiguousarray(M, dtype=np.uint64) for M in mats]
    idxs = [np.ascontiguousarray(M, dtype=np.uint64) for M in idxs]
    N = len(mats)
    rows = np.array([M.shape[0] for M in mats], dtype=np.int32)
    cols = np.array([M.shape[1] for M in mats], dtype=np.int32)
    Gf = np.ascontiguousarray(np.concatenate(G), dtype=np.uint64)
    v = np.empty(N, np.int32)
    ix = np.empty(N, np.uint64)
    cost = np.empty(N, np.uint64)
    _check(lib().orc_reconstruct(N, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32),
                                 _mat_ptrs(mats), _mat_ptrs(idxs), _ptr(Gf, C.c_uint64),
                                 _ptr(v, C.c_int32), _ptr(ix, C.c_uint64), _ptr(cost, C.c_uint64)),
           "reconstruct")
    return v, ix, cost


def search_plan(prob: Problem, nthreads: int = 0) -> Dict:
    m = Marshalled(prob)
    N = len(prob.instances)
    kmax = prob.k_max()
    total = C.c_uint64()
    idx = np.empty(N, np.uint64)
    dig = np.empty(N * kmax, np.int32)
    seg = np.empty(N, np.uint64)
    _check(lib().orc_search_plan(m.ref, nthreads, C.byref(total), _ptr(idx, C.c_uint64),
                                 _ptr(dig, C.c_int32), kmax, _ptr(seg, C.c_uint64)), "search_plan")
    return dict(total=int(total.value), seg_index=idx, digits=dig.reshape(N, kmax), seg_ns=seg)


def minplus(A: np.ndarray, B: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    Cm = np.empty((m, n), np.uint64)
    arg = np.empty((m, n), np.uint64)
    _check(lib().orc_minplus(m, k, n, _ptr(A, C.c_uint64), _ptr(B, C.c_uint64),
                             _ptr(Cm, C.c_uint64), _ptr(arg, C.c_uint64)), "minplus")
    return Cm, arg


# ---------------------------------------------------------------------------
# brute force over all global plans (tiny problems only) -- pure Python,
# independent of the C code above.  Eq. 3 evaluated directly on each
# plan tuple; the lexicographically smallest optimal tuple is kept.
# ---------------------------------------------------------------------------
def _digits(radix, idx):
    out = [0] * len(radix)
    for j in range(len(radix) - 1, -1, -1):
        out[j] = idx % int(radix[j])
        idx //= int(radix[j])
    return out


def py_cost(prob: Problem, tr: int, u: int, s: Sequence[int]) -> Optional[int]:
    """C_n(u, s) from the definition; None = infeasible."""
    T = prob.transitions[tr]
    ty = prob.types[T.type]
    total = 0
    for j in range(ty.K):
        p = int(ty.comp(j)[s[j]])
        c = int(ty.comm(j)[s[j]])
        if p == int(INF32) or c == int(INF32):
            return None
        total += p + c
    for e in ty.edges:
        r = int(e.table[s[e.src], s[e.dst]])
        if r == int(INF32):
            return None
        total += r
    for x in T.in_edges:
        r = int(x.table[u, s[x.dst]])
        if r == int(INF32):
            return None
        total += r
    return total


def brute_force(prob: Problem, limit: int = 10 ** 6) -> Dict:
    """All global plans (idx_1..idx_N) in lexicographic order; T(i) per Eq. 3."""
    spaces = []
    for t in prob.instances:
        ty = prob.types[prob.transitions[int(t)].type]
        spaces.append(range(int(np.prod([int(d) for d in ty.radix]))))
    n_plans = 1
    for s in spaces:
        n_plans *= len(s)
    if n_plans > limit:
        raise ValueError(f"brute force guard: {n_plans} plans > {limit}")
    best, best_plan, best_seg = None, None, None
    for plan in product(*spaces):               # lexicographic order
        u = 0
        total = 0
        segs = []
        ok = True
        for n, idx in enumerate(plan):
            tr = int(prob.instances[n])
            ty = prob.types[prob.transitions[tr].type]
            s = _digits(ty.radix, idx)
            c = py_cost(prob, tr, u, s)
            if c is None:
                ok = False
                break
            segs.append(c)
            total += c
            u = s[ty.out_block]
        if ok and (best is None or total < best):
            best, best_plan, best_seg = total, plan, segs
    if best is None:
        return dict(total=None)
    return dict(total=best, seg_index=np.array(best_plan, dtype=np.uint64),
                seg_ns=np.array(best_seg, dtype=np.uint64))


def brute_force_table(prob: Problem, tr: int) -> Tuple[np.ndarray, np.ndarray]:
    """A/I of one transition by direct enumeration in Python (tiny only)."""
    ty = prob.types[prob.transitions[tr].type]
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.full((din, dout), INF64, dtype=np.uint64)
    I = np.full((din, dout), NOIDX, dtype=np.uint64)
    S = int(np.prod([int(d) for d in ty.radix]))
    for u in range(din):
        for idx in range(S):
            s = _digits(ty.radix, idx)
            c = py_cost(prob, tr, u, s)
            if c is None:
                continue
            v = s[ty.out_block]
            if c < int(A[u, v]):
                A[u, v] = c
                I[u, v] = idx
    return A, I


# ---------------------------------------------------------------------------
# memory-constrained search (Eq. 4)
# ---------------------------------------------------------------------------
def mem_range(prob: Problem, type_id: int, quantum: int, m: Optional[Marshalled] = None) -> Tuple[int, int]:
    """(qlo, qhi) = sum_j min/max_s ceil(m_j[s] / quantum)."""
    m = m or Marshalled(prob)
    lo, hi = C.c_int64(), C.c_int64()
    _check(lib().orc_mem_range(C.byref(m.types[type_id]), quantum, C.byref(lo), C.byref(hi)),
           "mem_range")
    return int(lo.value), int(hi.value)


def segment_table_mem(prob: Problem, tr: int, quantum: int, nthreads: int = 0,
                      m: Optional[Marshalled] = None) -> Tuple[np.ndarray, np.ndarray, int]:
    """Am, Im [D_in][D_o][nq] and qlo (Am[u][v][q - qlo])."""
    m = m or Marshalled(prob)
    ty = prob.transitions[tr].type
    qlo, qhi = mem_range(prob, ty, quantum, m)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.empty((din, dout, qhi - qlo + 1), dtype=np.uint64)
    I = np.empty_like(A)
    _check(lib().orc_segment_table_mem(m.ref, tr, quantum, _ptr(A, C.c_uint64), _ptr(I, C.c_uint64),
                                       nthreads), "segment_table_mem")
    return A, I, qlo


def segment_table_mem_range(prob: Problem, tr: int, quantum: int, lo: int, hi: int, nthreads: int = 0,
                            m: Optional[Marshalled] = None):
    """segment_table_mem over the combination-index range [lo, hi) only."""
    m = m or Marshalled(prob)
    ty = prob.transitions[tr].type
    qlo, qhi = mem_range(prob, ty, quantum, m)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.empty((din, dout, qhi - qlo + 1), dtype=np.uint64)
    I = np.empty_like(A)
    _check(lib().orc_segment_table_mem_range(m.ref, tr, quantum, lo, hi, _ptr(A, C.c_uint64),
                                             _ptr(I, C.c_uint64), nthreads), "segment_table_mem_range")
    return A, I, qlo


def chain_mem(mats: Sequence[np.ndarray], qlos: Sequence[int], Qmax: int) -> List[np.ndarray]:
    """Backward DP over (u, c); returns [G_0, ..., G_N], G_n of shape [S][Qmax+1]."""
    mats = [np.ascontiguousarray(M, dtype=np.uint64) for M in mats]
    N = len(mats)
    rows = np.array([M.shape[0] for M in mats], dtype=np.int32)
    cols = np.array([M.shape[1] for M in mats], dtype=np.int32)
    nq = np.array([M.shape[2] for M in mats], dtype=np.int32)
    qlo = np.ascontiguousarray(qlos, dtype=np.int64)
    G = np.empty(int(rows[0] + cols.sum()) * (Qmax + 1), dtype=np.uint64)
    _check(lib().orc_chain_mem(N, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32), _ptr(nq, C.c_int32),
                               _ptr(qlo, C.c_int64), _mat_ptrs(mats), Qmax, _ptr(G, C.c_uint64)),
           "chain_mem")
    out, off = [G[:rows[0] * (Qmax + 1)].reshape(rows[0], Qmax + 1)], int(rows[0]) * (Qmax + 1)
    for c in cols:
        out.append(G[off:off + int(c) * (Qmax + 1)].reshape(int(c), Qmax + 1))
        off += int(c) * (Qmax + 1)
    return out


def reconstruct_mem(mats, idxs, qlos, Qmax: int, G: List[np.ndarray]):
    mats = [np.ascontiguousarray(M, dtype=np.uint64) for M in mats]
    idxs = [np.ascontiguousarray(M, dtype=np.uint64) for M in idxs]
    N = len(mats)
    rows = np.array([M.shape[0] for M in mats], dtype=np.int32)
    cols = np.array([M.shape[1] for M in mats], dtype=np.int32)
    nq = np.array([M.shape[2] for M in mats], dtype=np.int32)
    qlo = np.ascontiguousarray(qlos, dtype=np.int64)
    Gf = np.ascontiguousarray(np.concatenate([g.ravel() for g in G]), dtype=np.uint64)
    v = np.empty(N, np.int32)
    q = np.empty(N, np.int64)
    ix = np.empty(N, np.uint64)
    cost = np.empty(N, np.uint64)
    _check(lib().orc_reconstruct_mem(N, _ptr(rows, C.c_int32), _ptr(cols, C.c_int32),
                                     _ptr(nq, C.c_int32), _ptr(qlo, C.c_int64), _mat_ptrs(mats),
                                     _mat_ptrs(idxs), Qmax, _ptr(Gf, C.c_uint64), _ptr(v, C.c_int32),
                                     _ptr(q, C.c_int64), _ptr(ix, C.c_uint64), _ptr(cost, C.c_uint64)),
           "reconstruct_mem")
    return v, q, ix, cost


def search_plan_mem(prob: Problem, quantum: int, mem_limit: int, nthreads: int = 0) -> Dict:
    m = Marshalled(prob)
    N = len(prob.instances)
    kmax = prob.k_max()
    total, total_q = C.c_uint64(), C.c_int64()
    idx = np.empty(N, np.uint64)
    dig = np.empty(N * kmax, np.int32)
    seg = np.empty(N, np.uint64)
    segq = np.empty(N, np.int64)
    _check(lib().orc_search_plan_mem(m.ref, quantum, mem_limit, nthreads, C.byref(total),
                                     _ptr(idx, C.c_uint64), _ptr(dig, C.c_int32), kmax,
                                     _ptr(seg, C.c_uint64), _ptr(segq, C.c_int64), C.byref(total_q)),
           "search_plan_mem")
    return dict(total=int(total.value), seg_index=idx, digits=dig.reshape(N, kmax), seg_ns=seg,
                seg_q=segq, total_q=int(total_q.value))


def py_mem_q(ty, s: Sequence[int], quantum: int) -> int:
    """q(s) = ceil(sum_j m_j[s_j] / quantum): the segment plan's memory
    quantised as a whole, P:628 (pure Python, independent of the C code)."""
    return -(-sum(int(ty.mem_of(j)[s[j]]) for j in range(ty.K)) // quantum)


def py_mem_exact(ty, s: Sequence[int]) -> int:
    return sum(int(ty.mem_of(j)[s[j]]) for j in range(ty.K))


def brute_force_mem(prob: Problem, quantum: int, mem_limit: int, limit: int = 10 ** 6) -> Dict:
    """All global plans in lexicographic order; feasible iff
    sum_n q_n <= floor(mem_limit / quantum), q_n = ceil(m_n(i_n) / quantum) (Eq. 4);
    minimal Eq. 3 total, lexicographically smallest tuple."""
    Qmax = mem_limit // quantum
    spaces = []
    for t in prob.instances:
        ty = prob.types[prob.transitions[int(t)].type]
        spaces.append(range(int(np.prod([int(d) for d in ty.radix]))))
    n_plans = 1
    for sp in spaces:
        n_plans *= len(sp)
    if n_plans > limit:
        raise ValueError(f"brute force guard: {n_plans} plans > {limit}")
    best = None
    for plan in product(*spaces):
        u, total, mq, mex = 0, 0, 0, 0
        segs, qs = [], []
        ok = True
        for n, idx in enumerate(plan):
            tr = int(prob.instances[n])
            ty = prob.types[prob.transitions[tr].type]
            s = _digits(ty.radix, idx)
            c = py_cost(prob, tr, u, s)
            if c is None:
                ok = False
                break
            q = py_mem_q(ty, s, quantum)
            segs.append(c)
            qs.append(q)
            total += c
            mq += q
            mex += py_mem_exact(ty, s)
            u = s[ty.out_block]
        if not ok or mq > Qmax:
            continue
        if best is None or total < best[0]:
            best = (total, plan, segs, qs, mq, mex)
    if best is None:
        return dict(total=None)
    total, plan, segs, qs, mq, mex = best
    return dict(total=total, seg_index=np.array(plan, dtype=np.uint64),
                seg_ns=np.array(segs, dtype=np.uint64), seg_q=np.array(qs, dtype=np.int64),
                total_q=mq, mem_exact=mex)


def brute_force_table_mem(prob: Problem, tr: int, quantum: int):
    """Am/Im of one transition by direct enumeration in Python (tiny only)."""
    ty = prob.types[prob.transitions[tr].type]
    lo = sum(min(int(x) for x in ty.mem_of(j)) for j in range(ty.K))
    hi = sum(max(int(x) for x in ty.mem_of(j)) for j in range(ty.K))
    qlo, qhi = -(-lo // quantum), -(-hi // quantum)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.full((din, dout, qhi - qlo + 1), INF64, dtype=np.uint64)
    I = np.full_like(A, NOIDX)
    S = int(np.prod([int(d) for d in ty.radix]))
    for u in range(din):
        for idx in range(S):
            s = _digits(ty.radix, idx)
            c = py_cost(prob, tr, u, s)
            if c is None:
                continue
            k = py_mem_q(ty, s, quantum) - qlo
            v = s[ty.out_block]
            if c < int(A[u, v, k]):
                A[u, v, k] = c
                I[u, v, k] = idx
    return A, I, qlo


# ---------------------------------------------------------------- dense per-plan tables (NEXT-2)
def dense_segment_table(prob: Problem, tr: int, W: np.ndarray, nthreads: int = 0,
                        m: Optional[Marshalled] = None) -> Tuple[np.ndarray, np.ndarray]:
    """A, I [D_in][D_o] with C(u, s) = W[idx(s)] + cross terms."""
    m = m or Marshalled(prob)
    W = np.ascontiguousarray(W, dtype=np.uint32)
    din, dout = prob.d_in(tr), prob.d_out(tr)
    A = np.empty((din, dout), dtype=np.uint64)
    I = np.empty_like(A)
    _check(lib().orc_dense_segment_table(m.ref, tr, _ptr(W, C.c_uint32), _ptr(A, C.c_uint64),
                                         _ptr(I, C.c_uint64), nthreads), "dense_segment_table")
    return A, I


def dense_search_plan(prob: Problem, Ws: Sequence[Optional[np.ndarray]], nthreads: int = 0) -> Dict:
    m = Marshalled(prob)
    N = len(prob.instances)
    kmax = prob.k_max()
    Ws = [None if w is None else np.ascontiguousarray(w, dtype=np.uint32) for w in Ws]
    ptrs = (C.POINTER(C.c_uint32) * len(Ws))(*[None if w is None else _ptr(w, C.c_uint32) for w in Ws])
    total = C.c_uint64()
    idx = np.empty(N, np.uint64)
    dig = np.empty(N * kmax, np.int32)
    seg = np.empty(N, np.uint64)
    _check(lib().orc_dense_search_plan(m.ref, ptrs, nthreads, C.byref(total), _ptr(idx, C.c_uint64),
                                       _ptr(dig, C.c_int32), kmax, _ptr(seg, C.c_uint64)), "dense_search_plan")
    return dict(total=int(total.value), seg_index=idx, digits=dig.reshape(N, kmax), seg_ns=seg)


def brute_force_dense(prob: Problem, Ws, limit: int = 10 ** 6) -> Dict:
    """All global plans in lexicographic order, T = sum_n W[idx_n] + cross terms."""
    spaces = []
    for t in prob.instances:
        ty = prob.types[prob.transitions[int(t)].type]
        spaces.append(range(int(np.prod([int(d) for d in ty.radix]))))
    n_plans = 1
    for sp in spaces:
        n_plans *= len(sp)
    if n_plans > limit:
        raise ValueError(f"brute force guard: {n_plans} plans > {limit}")
    best = None
    for plan in product(*spaces):
        u, total, ok = 0, 0, True
        for n, idx in enumerate(plan):
            tr = int(prob.instances[n])
            T = prob.transitions[tr]
            ty = prob.types[T.type]
            w = int(Ws[T.type][idx])
            if w == int(INF32):
                ok = False
                break
            s = _digits(ty.radix, idx)
            total += w
            for x in T.in_edges:
                r = int(x.table[u, s[x.dst]])
                if r == int(INF32):
                    ok = False
                    break
                total += r
            if not ok:
                break
            u = s[ty.out_block]
        if ok and (best is None or total < best[0]):
            best = (total, plan)
    if best is None:
        return dict(total=None)
    return dict(total=best[0], seg_index=np.array(best[1], dtype=np.uint64))

