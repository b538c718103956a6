/*
 * cfp.h -- C-ABI of the B200-native CFP plan-search hot path (arXiv 2504.00598).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * SURVEY = /root/repo/SURVEY.md (its §8 is the scope contract).
 *
 * What is computed (the data-parallel hot path of "ComposeSearch"):
 *   (1) cfp_segment_costs -- for one distinct segment type and one
 *       incoming transition, evaluate EVERY strategy combination of its
 *       ParallelBlocks (S = prod_i D_i; "combines all ParallelBlocks'
 *       strategies") under every input layout u of the predecessor's
 *       output block, with the Eq. 3 cost terms:
 *          C(u,s) = sum_j (p_j[s_j] + c_j[s_j])
 *                 + sum_{intra edges a->b} R_ab[s_a][s_b]
 *                 + sum_{cross edges ->j}  Q_j[u][s_j]
 *       and reduce to A[u][v] = min_{s: s_o = v} C(u,s) with the least
 *       big-endian combination index I[u][v] attaining it.
 *   (2) cfp_minplus_chain -- the segment DP as tropical (min,+)
 *       products: G_N = terminal, G_{n-1} = A_n (x) G_n, using repeated squaring
 *       for runs of identical transitions.
 *   (3) cfp_search_plan -- (1) for every distinct segment type + (2) + the
 *       forward-greedy backtrack that emits the canonical optimal plan tuple
 *       (i_1..i_N), lexicographically smallest among optimal.
 *
 * Conventions:
 *  - Costs are integer nanoseconds.  Table entries are uint32; CFP_INF32 marks
 *    an infeasible strategy / pair and is absorbing.  Results are exact uint64;
 *    CFP_INF64 = unreachable.  CFP_NOIDX = argmin of an all-infeasible bucket.
 *  - Combination index: big-endian mixed radix, block 0 most significant:
 *    idx(s) = ((s_0*D_1 + s_1)*D_2 + ...)*D_{K-1} + s_{K-1}.
 *  - Ownership: every input pointer is caller-owned HOST memory, read only
 *    during the call and never retained.  Outputs are caller-allocated HOST
 *    memory; their contents are unspecified when the call fails.  Device
 *    scratch belongs to the ctx.
 *  - Errors: every function returns cfp_status (0 = CFP_OK) and never throws
 *    across the ABI; cfp_last_error() gives a thread-local message.
 *      CFP_EINVAL      structural problem (K<1, D<1, bad block id, self edge,
 *                      D_in mismatch with the predecessor's output radix, N<1,
 *                      chain not starting with pred_type=-1, ...)
 *      CFP_EOVERFLOW   a finite sum could reach 2^63
 *      CFP_EINFEASIBLE OPT = infinity (message names the first instance with
 *                      no finite completion)
 *      CFP_ETOOBIG     prod D > 2^48, K > 32, or device scratch too large
 *      CFP_ECUDA / CFP_ENCCL  wrapped runtime failures
 *      CFP_EVERSION    abi_version != CFP_ABI_VERSION
 *    There is no CPU fallback: without a usable CUDA device cfp_ctx_create
 *    fails with CFP_ECUDA.
 *  - Determinism: identical inputs give byte-identical outputs,
 *    independent of the world size.
 *  - Threading: a ctx is not thread-safe.  With world > 1 every rank must make
 *    the same calls with identical inputs (SPMD / NCCL semantics).
 */
#ifndef CFP_H
#define CFP_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define CFP_ABI_VERSION 1
#define CFP_INF32 0xFFFFFFFFu
#define CFP_INF64 0xFFFFFFFFFFFFFFFFull
#define CFP_NOIDX 0xFFFFFFFFFFFFFFFFull
#define CFP_MAX_BLOCKS 32

typedef enum {
  CFP_OK = 0, CFP_EINVAL = 1, CFP_EOVERFLOW = 2, CFP_EINFEASIBLE = 3, CFP_ETOOBIG = 4,
  CFP_ECUDA = 5, CFP_ENCCL = 6, CFP_ENOMEM = 7, CFP_EVERSION = 8
} cfp_status;

/* TARGET training mesh being planned for.  Metadata only: it
 * determined the strategy counts D_j upstream; the search never reads it. */
typedef struct { int32_t ndim; const int32_t* axes; } cfp_mesh;

/* One distinct segment type (fingerprint class). */
typedef struct {
  int32_t num_blocks;          /* K, 1..CFP_MAX_BLOCKS ParallelBlocks */
  const int32_t* radix;        /* [K] D_j >= 1 strategies per block */
  const uint32_t* comp_ns;     /* [sum D_j] profiled compute time p_j[s] */
  const uint32_t* comm_ns;     /* [sum D_j] profiled comm time c_j[s]; NULL = 0 */
  int32_t num_edges;           /* intra-segment PB->PB dependencies */
  const int32_t* edge_src;     /* [E] producer block */
  const int32_t* edge_dst;     /* [E] consumer block, != src */
  const uint32_t* edge_ns;     /* concat of row-major [D_src][D_dst] reshard tables */
  int32_t out_block;           /* o: its strategy is the segment's output layout */
} cfp_segment_type;

/* Transition type tau = (pred_type -> type) with its cross-segment reshard
 * tables from the predecessor's output block. */
typedef struct {
  int32_t pred_type;           /* -1 = chain start (D_in = 1) */
  int32_t type;
  int32_t num_in_edges;
  const int32_t* in_dst;       /* [X] consumer blocks of `type` */
  const uint32_t* in_ns;       /* concat of row-major [D_in][D_dst] tables */
} cfp_transition;

typedef struct {
  int32_t abi_version;         /* must equal CFP_ABI_VERSION */
  cfp_mesh mesh;
  int32_t num_types;        const cfp_segment_type* types;
  int32_t num_transitions;  const cfp_transition* transitions;
  int32_t num_instances;    const int32_t* inst_transition;  /* [N] */
} cfp_problem;

typedef struct {               /* caller-allocated outputs */
  uint64_t total_ns;           /* OPT = Eq. 3 of the emitted plan */
  uint64_t* seg_index;         /* [N] big-endian combination index i_n */
  int32_t* digits;             /* [N * kmax] per-block strategy, rows padded with -1 */
  int32_t kmax;                /* row stride of digits (>= max K of used types) */
  uint64_t* seg_ns;            /* [N] C_n(u_n, s_n) incl. incoming cross terms */
} cfp_plan;

typedef struct {
  int32_t device;              /* CUDA device ordinal */
  void* cuda_stream;           /* cudaStream_t; NULL = a stream owned by the ctx */
  int32_t world, rank;         /* world > 1: enumeration sharded over ranks */
  const void* nccl_unique_id;  /* world > 1: 128-byte ncclUniqueId (same on all ranks).
                                * NULL with world > 1 = shard simulation (test hook, one
                                * process): no collective; cfp_segment_costs returns this
                                * rank's shard-local (cost, least index) per bucket, whose
                                * lexicographic min over ranks is the world-1 result;
                                * cfp_search_plan / cfp_prepare are rejected (EINVAL).
                                * world == 1 with an id: a one-rank communicator; the
                                * sharded path (rank-local tables, NCCL min-all-reduce
                                * merge) runs on one GPU with results identical to
                                * world == 1 without an id. */
} cfp_ctx_opts;

typedef struct cfp_ctx cfp_ctx;
typedef struct cfp_prepared cfp_prepared;

cfp_status  cfp_ctx_create(cfp_ctx** ctx, const cfp_ctx_opts* opts);
void        cfp_ctx_destroy(cfp_ctx* ctx);
const char* cfp_last_error(void);
/* Writes a fresh 128-byte ncclUniqueId (call on one rank, broadcast it). */
cfp_status  cfp_nccl_unique_id(void* out128);
/* The ctx's communicator: ranks (ncclCommCount) and NCCL version code;
 * both 0 when the ctx has no communicator.  EINVAL on null arguments. */
cfp_status  cfp_ctx_nccl_info(cfp_ctx* ctx, int32_t* nranks, int32_t* version);

/* (1) One transition: cost_out/index_out are [d_in][D_o] row-major.
 * tr == NULL: no cross edges and d_in must be 1.  Collective if world > 1. */
cfp_status cfp_segment_costs(cfp_ctx* ctx, const cfp_segment_type* t, const cfp_transition* tr,
                             int32_t d_in, uint64_t* cost_out, uint64_t* index_out);

/* (2) Chain over run-length-encoded matrices.  mats[m] is rows[m] x cols[m]
 * row-major uint64 (CFP_INF64 = no edge).  Instance sequence = run r repeats
 * matrix run_mat[r] run_len[r] times (square when run_len > 1); consecutive
 * matrices must chain (cols of one = rows of the next); rows of the first = 1
 * is NOT required: G_0 has rows of the first matrix.
 * terminal: [cols of the last matrix] or NULL (= 0).
 * opt_out: G_0[0].  suffix_out (nullable): G_0, G_1, ..., G_N concatenated
 * (G_0 has rows(first) entries, G_n has cols(matrix of instance n) entries). */
cfp_status cfp_minplus_chain(cfp_ctx* ctx, int32_t num_mats, const int32_t* rows,
                             const int32_t* cols, const uint64_t* const* mats,
                             int32_t num_runs, const int32_t* run_mat, const int64_t* run_len,
                             const uint64_t* terminal, uint64_t* opt_out, uint64_t* suffix_out);

/* (3) Full search: identical result on every rank. */
cfp_status cfp_search_plan(cfp_ctx* ctx, const cfp_problem* p, cfp_plan* out);
/* cfp_search_plan keeps the last call's prepared plan in the ctx (schedule,
 * device buffers; freed by the next structural miss or cfp_ctx_destroy): a
 * call whose problem has the same structure -- shapes, feasible strategy
 * sets, term maxima, deduplicated instances -- uploads only its table values
 * and re-runs the path.  CFP_PLAN_CACHE=0 in the environment at ctx creation
 * disables it. */

/* One (min,+) product C = A (x) B with the least k attaining each entry
 * (CFP_NOIDX if the row/column pair is all-infinite).  argk nullable.
 * Finite entries must satisfy max(A) + max(B) < 2^63 - 1 (else
 * CFP_EOVERFLOW); when max(A) + max(B) < 2^31 - 1 the uint32 fused add+min
 * path runs, else uint64 -- identical results. */
cfp_status cfp_minplus_product(cfp_ctx* ctx, int32_t m, int32_t k, int32_t n,
                               const uint64_t* A, const uint64_t* B,
                               uint64_t* C, uint64_t* argk);

/* (min,+) product microbenchmark: S x S x S on device-resident synthetic
 * operands (values < 2^20); wide = 0 -> uint32 VIADDMNMX path, 1 -> uint64;
 * with_argk = 1 also tracks the least k.  Reports ms per launch and
 * add+min operations per second (S^3 / time). */
cfp_status cfp_minplus_bench(cfp_ctx* ctx, int32_t S, int32_t wide, int32_t with_argk, int32_t iters,
                             double* ms_per_launch, double* addmins_per_s);

/* ---- device-resident execution (used by the bench to time the hot path
 * with inputs already in HBM) ---------------------------------------------
 * cfp_prepare validates, prunes and stages the problem on the device (H2D);
 * cfp_execute runs the whole hot path (enumeration, merge, chain, backtrack)
 * on the ctx stream WITHOUT host synchronisation or copies; cfp_fetch_plan
 * synchronises and copies the plan to host memory. */
cfp_status cfp_prepare(cfp_ctx* ctx, const cfp_problem* p, cfp_prepared** out);
cfp_status cfp_execute(cfp_ctx* ctx, cfp_prepared* prep);
cfp_status cfp_fetch_plan(cfp_ctx* ctx, cfp_prepared* prep, cfp_plan* out);
void       cfp_prepared_free(cfp_prepared* prep);

typedef struct {
  double combos;               /* sum over distinct used types of prod_j feasible D_j */
  double combos_local;         /* this rank's share */
  double evals;                /* sum over used transitions of combos(type) x D_in */
  int32_t num_types, num_transitions, wide_types;  /* wide = 64-bit path */
  int32_t kernel_launches;     /* kernels launched by one cfp_execute */
  int32_t prefix_len[CFP_MAX_BLOCKS];   /* per type: enumeration schedule summary */
  int32_t nb[CFP_MAX_BLOCKS], na[CFP_MAX_BLOCKS];
  int32_t fused_tail;          /* 1: bucket minima + chain + argmin + backtrack run as one
                                  cooperative launch (world 1); 0: separate launches */
  int32_t tail_grid;           /* CTAs of that launch */
  int32_t o_mode[CFP_MAX_BLOCKS];   /* per type: output block in the register group (0), the M
                                       loop (1) or the prefix (2) of the enumeration schedule */
  int32_t full_a[CFP_MAX_BLOCKS];   /* per type: 1 = the fully unrolled A-loop kernel variant runs */
} cfp_prepared_info;
cfp_status cfp_prepared_query(const cfp_prepared* prep, cfp_prepared_info* info);
/* Segment tables of one transition through a prepared search's own schedule
 * and kernels (the enumeration variant the search runs; parity tests at full
 * size): re-executes the enumeration, then the least-index argmin of every
 * bucket instead of the chain.  Outputs as cfp_segment_costs: caller-allocated
 * host [d_in][D_o] cost and index (Eq. 3).  A transition
 * merged with an identical earlier one (same cross tables) returns that one's
 * tables.  EINVAL: the transition is not used by the instance list. */
cfp_status cfp_prepared_tables(cfp_ctx* ctx, cfp_prepared* prep, int32_t transition,
                               uint64_t* cost_out, uint64_t* index_out);
/* Record CUDA events on the ctx stream during the next cfp_execute calls
 * (bench instrumentation).  on = 0: off; 1: events at the start, after a0
 * staging, after the enumeration (all side lanes joined) and at the end --
 * cfp_prepared_kernel_ms reports enumeration ms and whole-path ms; 2: also an
 * event after every later phase -- cfp_prepared_phase_ms reports ms[6] =
 * {a0 stage, a1 enumerate, a1 bucket minima + a2 all-reduce of A, a3 chain,
 * a1 argmin + a2 index merge, a4 backtrack} of the last execute (SURVEY §8(d)
 * per-phase breakdown).  EINVAL: on outside [0, 2], or the level needed for
 * the query was not enabled.  Both queries synchronise on the end event. */
cfp_status cfp_prepared_time_kernels(cfp_prepared* prep, int32_t on);
cfp_status cfp_prepared_kernel_ms(cfp_prepared* prep, double* enum_ms, double* total_ms);
cfp_status cfp_prepared_phase_ms(cfp_prepared* prep, double* ms /* [6] */);

/* ---- memory-constrained search ----------------------
 * The paper's DP carries a memory constraint: Eq. 4 sums the profiled
 * peak memory of the chosen strategies, and the search keeps plans whose
 * memory fits the device.  Reading R-M1
 * (DESIGN.md): memory is profiled per ParallelBlock strategy, m_j[s]; a
 * segment plan's memory is their sum m(s) = sum_j m_j[s_j] (Eq. 4 within the
 * segment), and "we quantize the memory usage of each parallelism plan"
 * (P:628): q(s) = ceil(m(s) / quantum) -- a ceiling, so the quantised
 * total never under-estimates (never falsely feasible).
 *   segment table  Am[u][v][q - qlo] = min_{s: s_o = v, q(s) = q} C(u,s)
 *                  Im = least big-endian index attaining it (CFP_NOIDX if none),
 *                  qlo/qhi = ceil(sum_j min_s m_j[s] / quantum) and
 *                  ceil(sum_j max_s m_j[s] / quantum) over ALL strategies;
 *   chain          states (u, c), c = quantised memory used so far,
 *                  G_N(v, c) = 0 for c <= Qmax = floor(mem_limit / quantum),
 *                  G_{n-1}(u, c) = min_{v, q: c + q <= Qmax} Am_n[u][v][q] + G_n(v, c + q),
 *                  OPT = G_0(0, 0);
 *   plan           forward greedy from (0, 0), least combination index among
 *                  the optimal successors (v, q) -- the canonical plan.
 * Same conventions as above (host memory, caller-allocated outputs, status
 * codes).  Single-GPU: world > 1 gives CFP_EINVAL.  Limits (else CFP_ETOOBIG):
 * Qmax < 65536, qhi - qlo < 65536 per segment, D_o x (qhi - qlo + 1) of a
 * segment fits the DP's shared-memory row (coarser quantum otherwise). */
typedef struct {
  uint64_t quantum;                 /* >= 1, unit of m_j (e.g. KiB) */
  uint64_t mem_limit;               /* per-device limit in the same unit */
  const uint32_t* const* type_mem;  /* [num_types] -> [sum D_j] m_j[s]; NULL (array or entry) = 0 */
} cfp_mem_model;

/* Full memory-constrained search.  out as cfp_search_plan (seg_ns = Am of the
 * chosen bucket); seg_q [N] receives q of each segment, total_q their sum.
 * CFP_EINFEASIBLE when no plan fits the limit. */
cfp_status cfp_search_plan_mem(cfp_ctx* ctx, const cfp_problem* p, const cfp_mem_model* mem,
                               cfp_plan* out, int64_t* seg_q, int64_t* total_q);
/* Device-resident split of cfp_search_plan_mem (the bench times execute with
 * the tables already in HBM): prepare validates and stages, execute runs the
 * whole path on the ctx stream without host synchronisation, fetch copies the
 * plan out.  cfp_mem_time_kernels(prep, 1) before execute records events;
 * cfp_mem_kernel_ms then reports, for the last execute, the ms of the
 * enumeration kernels, of enumeration + folds + bucket minima, and of the
 * whole path, plus the combinations per execute and the kernel launches. */
typedef struct cfp_mem_prepared cfp_mem_prepared;
cfp_status cfp_mem_prepare(cfp_ctx* ctx, const cfp_problem* p, const cfp_mem_model* mem,
                           cfp_mem_prepared** out);
cfp_status cfp_mem_execute(cfp_ctx* ctx, cfp_mem_prepared* prep);
cfp_status cfp_mem_fetch_plan(cfp_ctx* ctx, cfp_mem_prepared* prep, cfp_plan* out, int64_t* seg_q,
                              int64_t* total_q);
void       cfp_mem_free(cfp_mem_prepared* prep);
cfp_status cfp_mem_time_kernels(cfp_mem_prepared* prep, int32_t on);
cfp_status cfp_mem_kernel_ms(cfp_mem_prepared* prep, double* enum_ms, double* tables_ms,
                             double* total_ms, double* combos, int32_t* launches);
/* Algorithmic (min,+) work of the cross-term folds of one execute: one fused
 * add+min per (prefix, input state, suffix class) per transition. */
cfp_status cfp_mem_fold_ops(const cfp_mem_prepared* prep, double* fold_addmins);

/* One transition's memory-bucketed table: cost_out / index_out are
 * [d_in][D_o][nq] row-major with nq = qhi - qlo + 1.  Pass cost_out =
 * index_out = NULL to query qlo_out / nq_out only (no device work). */
cfp_status cfp_segment_costs_mem(cfp_ctx* ctx, const cfp_segment_type* t, const uint32_t* mem,
                                 uint64_t quantum, const cfp_transition* tr, int32_t d_in,
                                 int64_t* qlo_out, int32_t* nq_out,
                                 uint64_t* cost_out, uint64_t* index_out);

/* ---- dense per-plan tables ---------------------------
 * The paper profiles whole-segment plans: p_n(i_n) and c_n(i_n) are measured
 * per plan i_n of a segment, so the cost of a type is a
 * dense table W_t[idx] over every combination index (uint32 ns, CFP_INF32 =
 * infeasible; intra-segment resharding included).  The cross-segment term
 * stays Q2's factored r_n:  C(u, s) = W_t[idx(s)] + sum_cross Q_j[u][s_j].
 * Buckets, least index, chain and canonical plan are those of (1)-(3).
 * Nothing factorises, so every entry is read once: an HBM stream of 4 bytes
 * per combination (C3: 2 x 18.3 GB).
 * W arguments are DEVICE pointers (the tables are tens of GB; the caller
 * allocates them on ctx's device and keeps them resident), 16-byte aligned
 * for the vector path; the types' comp/comm/edge tables are ignored (comp_ns
 * must still be non-NULL for validation); output block with <= 64
 * strategies (else ETOOBIG).
 * world > 1 (C4's two 313 GB tables fit only on 8 GPUs): every rank holds the
 * rows of a contiguous range of block 0's strategies -- combination indices
 * [first, first + count) of cfp_dense_shard -- and W points at the first of
 * them; each rank streams its rows, its least indices are global, and the
 * buckets are merged as the plain path's (NCCL MIN all-reduce of A, then of
 * the least index among the ranks attaining it); the chain is replicated.  A
 * shard-simulation ctx (world > 1 without nccl_unique_id) answers
 * cfp_segment_costs_dense with the rank-local tables only. */
/* This rank's share of a type's dense table: combination indices
 * [*first, *first + *count) (a block-0 strategy range, cfp_shard_range over
 * D_0; count may be 0).  EINVAL: null or malformed type. */
cfp_status cfp_dense_shard(cfp_ctx* ctx, const cfp_segment_type* t, int64_t* first, int64_t* count);
/* Synthetic tables: W[e] = splitmix64 stream of (e ^ base), 24-bit ns,
 * CFP_INF32 when the low 12 bits are zero (synth.generators.dense_table). */
cfp_status cfp_dense_fill(cfp_ctx* ctx, uint32_t* W_dev, uint64_t n, uint64_t base);
cfp_status cfp_search_plan_dense(cfp_ctx* ctx, const cfp_problem* p, const uint32_t* const* W_dev,
                                 cfp_plan* out);
/* One transition: cost_out/index_out [d_in][D_o] (host). */
cfp_status cfp_segment_costs_dense(cfp_ctx* ctx, const cfp_segment_type* t, const uint32_t* W_dev,
                                   const cfp_transition* tr, int32_t d_in, uint64_t* cost_out,
                                   uint64_t* index_out);
typedef struct cfp_dense_prepared cfp_dense_prepared;
cfp_status cfp_dense_prepare(cfp_ctx* ctx, const cfp_problem* p, const uint32_t* const* W_dev,
                             cfp_dense_prepared** out);
cfp_status cfp_dense_execute(cfp_ctx* ctx, cfp_dense_prepared* prep);
cfp_status cfp_dense_fetch_plan(cfp_ctx* ctx, cfp_dense_prepared* prep, cfp_plan* out);
void       cfp_dense_free(cfp_dense_prepared* prep);
cfp_status cfp_dense_time_kernels(cfp_dense_prepared* prep, int32_t on);
/* ms of the table stream (row minima; window from the first type's stream
 * start to the last one's end -- the types stream concurrently) and of the
 * whole path of the last execute; combinations and table bytes per execute;
 * kernel launches. */
cfp_status cfp_dense_kernel_ms(cfp_dense_prepared* prep, double* stream_ms, double* total_ms,
                               double* combos, double* bytes, int32_t* launches);

/* ---- profiling space and dynamic profiling budget ----
 * cfp_profile_space: Eq. 2 term by term, host arithmetic (callable
 * without a GPU):  type_plans[t] = prod_j D_j of type t (the whole-segment
 * plans to profile), trans_pairs[x] = sum over the cross edges (o_pred -> k)
 * of transition x of D_{pred,o} * D_k (the reshard kernel groups; 0 for a
 * chain start), total = their sum.  type_plans [num_types] and trans_pairs
 * [num_transitions] are nullable caller-owned host arrays.  EINVAL for bad
 * ids / radices, ETOOBIG when a count exceeds 2^62.
 * Pins: 2 x 81 + 2 x 9 = 180 for the GPT layer segments,
 * prod S_j + S_1 * S_K.
 *
 * cfp_profile_budget: the dynamic profiling time budget ("continuously
 * updated based on the fastest observed parallelism plans, aggressively
 * trimming the profiling of inefficient or stalled executions") over one
 * type's dense per-plan table W [n] (DEVICE pointer, 16-byte aligned, uint32
 * ns, CFP_INF32 = infeasible program), tasks run in canonical index order
 * (DESIGN R-B1..R-B4): with best_i = min_{j<i} W[j], task i is pruned iff
 * W[i] and best_i are finite and W[i] * den > best_i * num (f = num/den,
 * 1 <= den <= num <= 65535, else EINVAL); a pruned task costs
 * floor(best_i * num / den), a completed one W[i], an infeasible one 0.
 * One read of W (a single-pass prefix-minimum scan).  n < 2^44 (ETOOBIG);
 * single GPU.  kernel_ms (nullable): device time of the call's kernels. */
typedef struct {
  uint64_t tasks;                     /* n */
  uint64_t pruned;                    /* tasks trimmed by the budget */
  uint64_t infeasible;                /* CFP_INF32 entries */
  uint64_t spent_lo, spent_hi;        /* profiling ns under the budget (128-bit) */
  uint64_t full_lo, full_hi;          /* profiling ns without it: sum of finite W (128-bit) */
  uint64_t best;                      /* least finite W, CFP_INF64 if none */
  uint64_t best_index;                /* least index attaining it, CFP_NOIDX if none */
} cfp_budget_result;
cfp_status cfp_profile_space(const cfp_problem* p, int64_t* type_plans, int64_t* trans_pairs,
                             int64_t* total);
cfp_status cfp_profile_budget(cfp_ctx* ctx, const uint32_t* W_dev, uint64_t n, uint32_t num,
                              uint32_t den, cfp_budget_result* out, double* kernel_ms);

/* ---- host-only helpers (no device work; callable without a GPU) ---------- */
/* Contiguous, balanced share [lo, hi) of `units` items for `rank` of `world`
 * in multiples of `align`. */
cfp_status cfp_shard_range(int64_t units, int64_t align, int32_t world, int32_t rank,
                           int64_t* lo, int64_t* hi);
/* Packed merge key (cost << idx_bits) | idx, CFP_INF64 for (INF, NOIDX). */
cfp_status cfp_pack_keys(int64_t n, const uint64_t* cost, const uint64_t* idx, int32_t idx_bits,
                         uint64_t* keys);
cfp_status cfp_unpack_keys(int64_t n, const uint64_t* keys, int32_t idx_bits,
                           uint64_t* cost, uint64_t* idx);

/* ---- N5 integer-pipe microbenchmark (roofline denominator) --------------
 * op 0: VIADDMNMX.U32 (fused add+min), op 1: IADD3, op 2: 64-bit add+min,
 * op 3: the enumeration's two-pipe group (VIADDMNMX + two FMA-pipe IMAD adds
 * + VIMNMX3: three add+mins in four instructions over the ALU and FMA pipes).
 * Reports lane-ops/s (op 3: add+mins/s) and the elapsed ms of one launch. */
cfp_status cfp_intpipe_bench(cfp_ctx* ctx, int32_t op, int32_t iters, double* ops_per_s,
                             double* ms);

#ifdef __cplusplus
}
#endif
#endif
