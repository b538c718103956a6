"""Problem data model shared by the oracle and the CUDA path as *inputs only*.

This module holds containers and validation-free plumbing: no cost arithmetic of
the method (no Eq. 3 sums, no minimisation) lives here.  Both `oracle/` and the
product package marshal these numpy arrays into their own, independent C
structures.

Vocabulary follows PAPER.md (`P:n` = /root/reference/PAPER.md line n):
  * SegmentType   -- one distinct segment (fingerprint class): K
                     ParallelBlocks with D_j strategies each,
                     per-strategy profiled compute/comm time
                     and intra-segment PB->PB resharding tables.
  * Transition    -- (predecessor type -> type) with the cross-segment resharding
                     tables between the predecessor's output block and consumer
                     blocks of `type`.
  * Problem       -- the instance sequence n = 1..N as transition ids.

All costs are uint32 integer nanoseconds; INF32 (0xFFFFFFFF) marks an
infeasible strategy / pair and is absorbing.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

INF32 = np.uint32(0xFFFFFFFF)
INF64 = np.uint64(0xFFFFFFFFFFFFFFFF)
NOIDX = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class Edge:
    """Intra-segment dependency src -> dst with reshard table R[D_src][D_dst]."""
    src: int
    dst: int
    table: np.ndarray  # uint32 [D_src, D_dst]


@dataclass
class SegmentType:
    radix: np.ndarray                 # int32 [K]
    comp_ns: np.ndarray               # uint32 [sum D]   p_j[s]
    comm_ns: Optional[np.ndarray]     # uint32 [sum D]   c_j[s] (None -> 0)
    edges: List[Edge]
    out_block: int
    name: str = ""
    # per-strategy peak memory m_j[s] of each ParallelBlock ("peak memory
    # consumption", P:608 m_n; NEXT-1), uint32 in caller-chosen units (the
    # generators use KiB); None -> 0.  Eq. 4 sums it over the plan.
    mem: Optional[np.ndarray] = None

    def mem_of(self, j: int) -> np.ndarray:
        o = self.offsets()
        if self.mem is None:
            return np.zeros(int(self.radix[j]), dtype=np.uint32)
        return self.mem[o[j]:o[j + 1]]

    @property
    def K(self) -> int:
        return int(len(self.radix))

    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.radix)]).astype(np.int64)

    def comp(self, j: int) -> np.ndarray:
        o = self.offsets()
        return self.comp_ns[o[j]:o[j + 1]]

    def comm(self, j: int) -> np.ndarray:
        o = self.offsets()
        if self.comm_ns is None:
            return np.zeros(int(self.radix[j]), dtype=np.uint32)
        return self.comm_ns[o[j]:o[j + 1]]


@dataclass
class CrossEdge:
    """Cross-segment edge into consumer block `dst` with table Q[D_in][D_dst]."""
    dst: int
    table: np.ndarray  # uint32 [D_in, D_dst]


@dataclass
class Transition:
    pred_type: int          # -1 = chain start (D_in = 1)
    type: int
    in_edges: List[CrossEdge] = field(default_factory=list)
    name: str = ""


@dataclass
class Problem:
    mesh: Tuple[int, ...]
    types: List[SegmentType]
    transitions: List[Transition]
    instances: np.ndarray   # int32 [N] transition id per instance
    name: str = ""

    def d_in(self, t: int) -> int:
        tr = self.transitions[t]
        if tr.pred_type < 0:
            return 1
        pt = self.types[tr.pred_type]
        return int(pt.radix[pt.out_block])

    def d_out(self, t: int) -> int:
        ty = self.types[self.transitions[t].type]
        return int(ty.radix[ty.out_block])

    def k_max(self) -> int:
        return max(ty.K for ty in self.types)

    def num_combinations(self, type_id: int) -> int:
        return int(np.prod([int(d) for d in self.types[type_id].radix], dtype=object))

    def feasible_combinations(self, type_id: int) -> int:
        """prod_j (#strategies of block j whose own p+c is not INF) -- the
        enumerated space after pruning infeasible strategies."""
        ty = self.types[type_id]
        n = 1
        for j in range(ty.K):
            c = ty.comp(j)
            m = ty.comm(j)
            n *= int(np.sum((c != INF32) & (m != INF32)))
        return n

    def used_types(self) -> List[int]:
        return sorted({self.transitions[int(t)].type for t in self.instances})
