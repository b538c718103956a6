/*
 * cfp_oracle.h -- plain, slow, obviously-correct CPU oracle for the CFP
 * plan-search hot path (arXiv 2504.00598).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2504_00598_b200/, include/cfp.h).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY = SURVEY.md.
 *
 * Definitions implemented (the normative reading):
 *  - cost of combination s of a segment instance under input state u
 *      C(u,s) = sum_j (p_j[s_j] + c_j[s_j])               (Eq. 3 p_n + c_n)
 *             + sum_{intra edges (a,b,R)} R[s_a][s_b]     (reshard between PBs)
 *             + sum_{cross edges (j,Q)}  Q[u][s_j]        (Eq. 3 r_n)
 *    computed exactly in uint64; any INF (0xFFFFFFFF) term makes C = INF.
 *  - combination index: big-endian mixed radix, block 0 most significant
 *    (S = prod_i D_i; order = SURVEY Q5).
 *  - A[u][v] = min_{s: s_o = v} C(u,s); I[u][v] = least index attaining it
 *    (NOIDX if the bucket is all-INF).
 *  - chain (textbook backward DP, P:625-627 with the state of S:501):
 *      G_N = terminal (0); G_{n-1}(u) = min_v A_n[u][v] + G_n(v); OPT = G_0(0).
 *  - reconstruction: forward greedy choosing, among optimal successors, the
 *    least combination index (lexicographically smallest plan tuple).
 *
 * Memory-constrained search (Eq. 4):
 *  - per-block peak memory m_j[s], quantised per block with a
 *    ceiling: q_j[s] = ceil(m_j[s] / quantum)  (reading R-M1 in DESIGN.md:
 *    the factored model's profile unit is the ParallelBlock; the
 *    ceiling over-approximates, so a plan is never falsely feasible);
 *    segment memory q(s) = sum_j q_j[s_j]  (Eq. 4 restricted to a segment);
 *  - Am[u][v][q - qlo] = min_{s: s_o = v, q(s) = q} C(u,s), Im = least index;
 *    qlo/qhi = sum_j min/max_s q_j[s] over all strategies;
 *  - chain state (u, c), c = quantised memory used so far:
 *      G_N(v, c) = 0 for c <= Qmax = floor(mem_limit / quantum);
 *      G_{n-1}(u, c) = min_{v, q: c + q <= Qmax} Am_n[u][v][q] + G_n(v, c + q);
 *      OPT = G_0(0, 0);
 *  - reconstruction: forward greedy from (u, c) = (0, 0) choosing, among the
 *    optimal successors (v, q), the least combination index.
 */
#ifndef CFP_ORACLE_H
#define CFP_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_INF32 0xFFFFFFFFu
#define ORC_INF64 0xFFFFFFFFFFFFFFFFull
#define ORC_NOIDX 0xFFFFFFFFFFFFFFFFull

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EINFEASIBLE = 3, ORC_ETOOBIG = 4, ORC_ENOMEM = 7 };

typedef struct {
  int32_t K;
  const int32_t* radix;     /* [K] */
  const uint32_t* comp;     /* [sum D] p_j[s] */
  const uint32_t* comm;     /* [sum D] c_j[s], nullable = 0 */
  int32_t E;
  const int32_t* esrc;      /* [E] */
  const int32_t* edst;      /* [E] */
  const uint32_t* etab;     /* concat row-major [D_src][D_dst] */
  int32_t out_block;
  const uint32_t* mem;      /* [sum D] m_j[s] (NEXT-1), nullable = 0 */
} orc_type;

typedef struct {
  int32_t pred;             /* -1 = chain start, D_in = 1 */
  int32_t type;
  int32_t X;
  const int32_t* xdst;      /* [X] consumer block */
  const uint32_t* xtab;     /* concat row-major [D_in][D_dst] */
} orc_trans;

typedef struct {
  int32_t ntypes;
  const orc_type* types;
  int32_t ntrans;
  const orc_trans* trans;
  int32_t N;
  const int32_t* inst;      /* [N] transition id per instance */
} orc_problem;

/* C(u, s) for digit vector s (length K of the transition's type). */
uint64_t orc_cost(const orc_problem* p, int32_t tr, int32_t u, const int32_t* s);
/* C(u, s) for s given as big-endian index. */
uint64_t orc_cost_index(const orc_problem* p, int32_t tr, int32_t u, uint64_t idx);
/* Full A/I table of one transition: A, I are [D_in][D_o]. */
int orc_segment_table(const orc_problem* p, int32_t tr, uint64_t* A, uint64_t* I, int nthreads);
/* Same over the index sub-range [lo, hi) only (bounded CPU-baseline samples). */
int orc_segment_table_range(const orc_problem* p, int32_t tr, uint64_t lo, uint64_t hi,
                            uint64_t* A, uint64_t* I, int nthreads);
/* One bucket (u, v): enumerates every s with s_o = v in index order. */
int orc_bucket(const orc_problem* p, int32_t tr, int32_t u, int32_t v,
               uint64_t* a, uint64_t* i, int nthreads);
/* Backward DP over N instance matrices (rows[n] x cols[n], row-major).
 * G receives (N+1) ragged vectors: G_0 (rows[0]) then G_n (cols[n-1]).
 * terminal: cols[N-1] values or NULL (= 0). */
int orc_chain(int32_t N, const int32_t* rows, const int32_t* cols,
              const uint64_t* const* A, const uint64_t* terminal, uint64_t* G);
/* Forward greedy reconstruction from u_1 = 0. Outputs per instance the chosen
 * column v_n, index I_n[u][v_n] and cost A_n[u][v_n]. Returns EINFEASIBLE if
 * G_0(0) is INF. */
int orc_reconstruct(int32_t N, const int32_t* rows, const int32_t* cols,
                    const uint64_t* const* A, const uint64_t* const* I,
                    const uint64_t* G, int32_t* v_out, uint64_t* idx_out, uint64_t* cost_out);
/* Full search: tables for every transition used, chain, reconstruction.
 * digits: [N * kmax] padded with -1. */
int orc_search_plan(const orc_problem* p, int nthreads, uint64_t* total,
                    uint64_t* seg_index, int32_t* digits, int32_t kmax, uint64_t* seg_ns);
/* (A (x) B)[i][j] = min_k A[i][k] + B[k][j]; argk = least k (NOIDX if INF). */
int orc_minplus(int32_t m, int32_t k, int32_t n, const uint64_t* A, const uint64_t* B,
                uint64_t* C, uint64_t* argk);
/* ---- memory-constrained search (NEXT-1) ---- */
/* qlo/qhi of a type: ceil(sum_j min_s m_j[s] / quantum), ceil(sum_j max_s m_j[s] / quantum). */
int orc_mem_range(const orc_type* t, uint64_t quantum, int64_t* qlo, int64_t* qhi);
/* m(s) = sum_j m_j[s_j]: the segment plan's memory (Eq. 4 within a segment). */
uint64_t orc_mem_exact(const orc_type* t, const int32_t* s);
/* q(s) = ceil(m(s) / quantum): each plan's memory quantised. */
uint64_t orc_mem_q(const orc_type* t, const int32_t* s, uint64_t quantum);
/* Am, Im: [D_in][D_o][qhi - qlo + 1]. */
int orc_segment_table_mem(const orc_problem* p, int32_t tr, uint64_t quantum,
                          uint64_t* Am, uint64_t* Im, int nthreads);
int orc_segment_table_mem_range(const orc_problem* p, int32_t tr, uint64_t quantum, uint64_t lo_idx,
                                uint64_t hi_idx, uint64_t* Am, uint64_t* Im, int nthreads);
/* Backward DP over (u, c).  Instance n has matrix Am[n] of shape
 * rows[n] x cols[n] x nq[n] with memory offset qlo[n].  G receives N+1 blocks
 * [S][Qmax + 1]: G_0 (rows[0]) then G_n (cols[n-1]). */
int orc_chain_mem(int32_t N, const int32_t* rows, const int32_t* cols, const int32_t* nq,
                  const int64_t* qlo, const uint64_t* const* Am, int64_t Qmax, uint64_t* G);
/* Forward greedy from (0, 0): per instance the chosen v, q (absolute), index
 * and cost.  EINFEASIBLE if G_0(0, 0) is INF. */
int orc_reconstruct_mem(int32_t N, const int32_t* rows, const int32_t* cols, const int32_t* nq,
                        const int64_t* qlo, const uint64_t* const* Am, const uint64_t* const* Im,
                        int64_t Qmax, const uint64_t* G, int32_t* v_out, int64_t* q_out,
                        uint64_t* idx_out, uint64_t* cost_out);
/* Full memory-constrained search; seg_q[n] = q of segment n, total_q = sum. */
int orc_search_plan_mem(const orc_problem* p, uint64_t quantum, uint64_t mem_limit, int nthreads,
                        uint64_t* total, uint64_t* seg_index, int32_t* digits, int32_t kmax,
                        uint64_t* seg_ns, int64_t* seg_q, int64_t* total_q);

/* ---- dense per-plan tables (NEXT-2) ----
 * W: [prod D] profiled time of every whole-segment plan (INF = 0xFFFFFFFF);
 * C(u, s) = W[idx(s)] + sum_cross Q_j[u][s_j]; tables/chain/plan as above. */
int orc_dense_segment_table(const orc_problem* p, int32_t tr, const uint32_t* W, uint64_t* A, uint64_t* I,
                            int nthreads);
/* W[t] = dense table of type t (NULL for unused types). */
int orc_dense_search_plan(const orc_problem* p, const uint32_t* const* W, int nthreads, uint64_t* total,
                          uint64_t* seg_index, int32_t* digits, int32_t kmax, uint64_t* seg_ns);

/* Big-endian mixed-radix decode. */
void orc_decode(int32_t K, const int32_t* radix, uint64_t idx, int32_t* digits);

#ifdef __cplusplus
}
#endif
#endif
