// cfp_internal.h -- structures shared by the host runtime (cfp_host.cu) and the
// sm_100a kernels (cfp_kernels.cu).  Not part of the ABI.
//
// Vocabulary: a segment type has K blocks ("digits"); a
// combination s is a mixed-radix number, block 0 most significant.  After
// pruning strategies whose own p+c is infeasible (monotone remap),
// every block j has D'_j >= 1 "compact" strategies.
//
// Enumeration schedule of one type (chosen by the host planner):
//   digits [0, P)  = prefix: one GPU thread (or VG threads) per prefix value;
//                    every fold digit (consumer block of a cross edge) is here.
//   suffix digits  = M (loop) | A (broadcast operand) | B (register operand),
//                    no intra edge between an A digit and a B digit.
// For a prefix p and an M value m, every combination (p, m, a, b) costs
//      C = K0[p] + Z[ctxZ] + X[ctxA][a] + Y[ctxB][b]
// (each cost term of Eq. 3 is assigned to exactly one of the four tables), so
// one fused add+min (VIADDMNMX) per combination evaluates and reduces it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfp {

constexpr int kMaxDigits = 32;
constexpr int kMaxTerms = 96;
constexpr int kMaxCross = 16;    // cross edges per transition
constexpr int kBlock = 256;          // threads per CTA of the enumeration kernel
constexpr int kBuildChunk = 1024;    // table entries per CTA of build_table_kernel
constexpr uint32_t kCap32 = 0x7FFFFFFFu;            // narrow "infinity" (>= CAP => INF)
constexpr uint64_t kCap64 = 0x7FFFFFFFFFFFFFFFull;  // wide "infinity"
constexpr uint64_t kInf64 = 0xFFFFFFFFFFFFFFFFull;

// A cost term over the digits of a table's index space.
//   kind 0: unary   W[off + s_a]
//   kind 1: pair    R[off + s_a * db + s_b]
//   kind 2: cross   Q[off + u * db + s_b]      (fold only; u = input state)
struct Term {
  int32_t kind;
  int32_t a, b;      // positions in the owning index space (or block ids)
  int32_t db;        // row length of the pair table
  int64_t off;       // element offset into the value blob
};

// A table T[e] over the mixed-radix space of `ndig` digits (last fastest),
// entry = saturated sum of `nterm` terms.  Rows may be padded: the last digit
// group spans `row` entries of which `row_valid` are real (the rest = CAP).
struct TableSpec {
  int32_t ndig;
  int32_t radix[kMaxDigits];
  int32_t nterm;
  Term term[kMaxTerms];
  int64_t rows;        // product of radices of the leading (row) digits
  int32_t row_digits;  // number of trailing digits forming one row
  int64_t row_valid;   // product of radices of the row digits
  int64_t row;         // padded row length
  int64_t out_off;     // element offset of T in the derived blob
  int64_t block0, nblocks;   // this table's CTAs in the build launch (1024 entries each)
};

// A transition folded in the enumeration epilogue (cross terms into this type).
struct EpiTau {
  int32_t Din;
  int32_t nq;
  Term q[kMaxCross];            // kind 2: a = prefix position of the consumer, db, off
  int64_t qt[kMaxCross];        // transposed copies Q^T[s][DinP] (16-byte aligned rows)
  void* chunkmin;               // [Din * Do][nchunks]
};

struct EnumParams {
  // prefix mapping: p = h * W + l, thread t -> (l, vg) = t / Gpad, h = h0 + t % Gpad
  int32_t P;                    // prefix length
  int32_t pre_radix[kMaxDigits];
  int64_t W;                    // size of the low prefix part (canonical last digits)
  int64_t G, Gpad, h0;          // high values handled, padded to a multiple of CH
  int32_t VG;                   // register groups per prefix (B split)
  int32_t MS;                   // M-loop split: 1, or 2 (threads t and t + CH share a prefix
                                // and take the two halves of the M values; B = {o} only)
  int32_t CH;                   // prefixes per CTA (= chunk) = kBlock / MS
  int32_t no_full_a;            // 1: do not take the fully unrolled A loop (A/B tests)
  int64_t pre_sx[kMaxDigits], pre_sy[kMaxDigits], pre_sz[kMaxDigits];  // ctx strides
  int64_t nM;                   // |M space| (mtab rows)
  int32_t na, na_pad;           // |A space| (XT row length), padded
  int32_t nb;                   // |B space|
  int32_t nb_pad;               // YT row length = VG * NB
  int32_t o_mode;               // 0: o in B, 1: o in M, 2: o in prefix
  int32_t o_pre;                // o's prefix position (mode 2)
  int32_t o_bstride, o_bradix;  // v(j) = (j / o_bstride) % o_bradix (mode 0)
  int32_t Do;                   // compact output radix
  int32_t staged;               // 1: tables sliced into shared memory per CTA
  int32_t ymerge;               // 1 (staged only): Z folded into per-m Y rows in smem
  int32_t ym_inplace;           // 1: ... in place (the slice's Y rows are the M values in order)
  int32_t init_row;             // 1: B_p row must be pre-filled with CAP
  int64_t xspan, yspan, zspan;  // slice lengths (staged)
  // device pointers (element type = the path's value type)
  const void* XT; const void* YT; const void* ZT; const void* K0;
  const int4* mtab;             // [nM] (x, y, z, v_o)
  void* Bp;                     // [G*W][Do] local canonical prefixes
  // epilogue fold of the cross-segment terms (one chunk = one CTA's prefixes)
  int64_t pre_stride[kMaxDigits];
  int32_t ntau;
  const EpiTau* taus;           // device [ntau]
  const void* vals;             // value blob (compact Q tables)
  int64_t nchunks;              // W * (Gpad / CH)
  int32_t smem_epi;             // bytes of the epilogue region
  int32_t one;                  // 1 (the FMA-pipe adds' multiplier, opaque to the compiler)
  int32_t mix;                  // 1: full-A loop on two pipes (ALU + FMA), 0: VIADDMNMX only
  int32_t xs_off;               // elements from the region start to the cross rows Xs
  int32_t dinp_max;             // largest padded D_in of the incoming transitions
};

struct FoldParams {
  int32_t P;
  int32_t pre_radix[kMaxDigits];
  int64_t pre_stride[kMaxDigits];   // prod of the radices after each prefix digit
  int64_t p_lo;                 // global canonical prefix of local row 0
  int64_t nPl;                  // local prefixes
  int32_t Din, Do;
  int32_t nq;                   // cross terms: a = prefix position of consumer, db, off
  Term q[kMaxCross];
  int32_t CH;                   // prefixes per chunk
  int64_t nchunks;
  int32_t tma;                  // 1: B_p chunk rows are 16-byte multiples (bulk copy)
  int32_t qelems;               // sum of D_in * D_j over cross terms (smem copy)
  const void* Bp;
  const void* vals;             // value blob (compact Q tables)
  void* chunkmin;               // [Din * Do][nchunks]
  // chunk -> rows: chunk = l * nhb + hb holds local rows (hb*CH + i) * W + l
  int64_t W, G, h0, nhb;
};

// Generic evaluation of all intra terms of a compact combination (argmin
// recovery) -- terms reference block ids directly.
struct EvalSpec {
  int32_t K;
  int32_t radix[kMaxDigits];    // compact
  int32_t P;                    // prefix length
  int32_t o;                    // output block
  int32_t nterm;
  Term term[kMaxTerms];         // kind 0/1 over block ids
  int64_t nsuffix;              // prod of suffix radices
  int64_t tab_lo;               // the type's compact W/R tables: [tab_lo, tab_lo + tab_n)
  int32_t tab_n;
};

struct ArgminParams {
  FoldParams f;
  EvalSpec e;
  const void* K0;               // unused (full evaluation)
  int32_t map_off[kMaxDigits];  // compact -> original strategy maps (int32 blob)
  int32_t orig_radix[kMaxDigits];
  int32_t Do_orig;
  const int32_t* maps;
  const int32_t* vmap;          // compact v -> original v of the output block
  uint64_t* A_out;              // [Din][Do_orig] uint64
  uint64_t* I_out;
  uint64_t* key_out;            // [Din][Do_orig] local (cost, idx) for merge (nullable)
  int64_t* pstar;               // scratch [Din*Do]
  const int32_t* vinv;          // original v -> compact v (-1 = pruned)
  const uint64_t* A_glob;       // [Din][Do_orig] merged bucket minima (amin + all-reduce)
  int32_t wide;                 // value type of this transition's type (0 u32, 1 u64)
  int32_t slot;                 // transition slot (list entries)
};

struct ArgminEntry { int32_t slot, pair; };   // pair = u * Do + compact v

struct ChainInst {
  const uint64_t* A;            // [rows][cols]
  const uint64_t* I;            // nullable
  int32_t mat;                  // distinct matrix id (staging)
  int32_t rows, cols;
  int32_t K;                    // digits of the instance's type (plan decode)
  int32_t radix_off;            // offset into radix blob
};

struct ChainRun {
  int32_t first;                // first instance (0-based)
  int32_t len;                  // instances in the run (same matrix)
};

struct CompactJob {
  int32_t kind;          // 0 unary, 1 pair (rows & cols remapped), 2 cross (cols remapped),
                         // 3 cross transposed: out[c][rows_pad], rows >= `rows` padded with CAP
  int32_t rows, cols;    // compact shape (unary: rows = 1)
  int32_t rows_pad;      // kind 3 row length of the transposed table
  int32_t raw_cols;      // raw row length
  int64_t raw_off, raw_off2;   // comp / comm (unary), table (pair/cross); raw_off2 < 0: no comm
  int32_t map_r, map_c;  // offsets into the map blob (-1 = identity)
  int64_t out_off;
};

struct ChainParams {
  int32_t N;
  int32_t nruns;
  const ChainInst* inst;        // [N]
  const ChainRun* runs;         // [nruns], in instance order
  const uint64_t* terminal;     // nullable
  uint64_t* G;                  // ragged (N+1) vectors
  const int64_t* goff;          // [N+2] offsets of G_0..G_N (+end)
  uint64_t* powers;             // scratch
  int64_t powers_cap;           // elements available
  int32_t backtrack;
  // plan outputs (backtrack)
  uint64_t* total;
  uint64_t* seg_index;
  uint64_t* seg_ns;
  int32_t* digits;
  int32_t kmax;
  const int32_t* radix_blob;
  int32_t* status;              // 0 ok, 3 infeasible, 4 scratch too small
  // shared-memory staging (all distinct matrices, G and powers fit)
  int32_t nmat;
  const ChainInst* mats;        // [nmat] distinct matrices (A, I, rows, cols)
  const int64_t* moff;          // [nmat] element offsets in the staged area
  int64_t mat_elems;            // sum rows*cols
  int64_t smem_bytes;           // 0 = global mode
  int32_t levels_max, smax;
  int32_t mode;                 // 0 G + backtrack, 1 G + optimal-edge list, 2 backtrack (G given)
  int32_t* edge_flag;           // mode 1: [sum Din*Do_orig] dedupe flags (zeroed)
  const int64_t* flag_off;      // mode 1: per distinct matrix offset into edge_flag
  ArgminEntry* edge_list;       // mode 1: reachable optimal edges (slot, u * Do_orig + v_orig)
  uint8_t* reach;               // [goff[N]] state u reachable before instance n (set by mode 1)
  int32_t* edge_count;
  const uint64_t* baseA;        // all distinct A matrices, contiguous (moff offsets)
  const uint64_t* baseI;        // same for I (backtrack)
};

#ifndef CFP_TAIL_THREADS
#define CFP_TAIL_THREADS 512
#endif
constexpr int kTailThreads = CFP_TAIL_THREADS;   // threads per CTA of the fused tail kernel

// Shared-memory layout of the fused tail's chain (CTA 0; every state count
// <= 32).  Host and device compute it from the same numbers.
struct FusedChainLayout {
  int64_t sA, sG, sP, sgoff, smoff, sinst, om, rmask, ebits, nxt, vseq, bytes;
  __host__ __device__ static int64_t al(int64_t x) { return (x + 15) & ~int64_t(15); }
  __host__ __device__ FusedChainLayout(int64_t mat_elems, int64_t gtot, int64_t goffN, int N, int nmat,
                                       int levels, int S) {
    int64_t o = 0;
    sA = o;    o = al(o + mat_elems * 8);
    sG = o;    o = al(o + gtot * 8);
    sP = o;    o = al(o + (int64_t)(levels + 1) * S * S * 8);   // P_0 .. P_levels (big encoding)
    sgoff = o; o = al(o + (int64_t)(N + 2) * 8);
    smoff = o; o = al(o + (int64_t)nmat * 8);
    sinst = o; o = al(o + (int64_t)N * 16);
    om = o;    o = al(o + goffN * 4);
    rmask = o; o = al(o + (int64_t)N * 4);
    ebits = o; o = al(o + ((mat_elems + 31) / 32) * 4);
    nxt = o;   o = al(o + goffN * 1);
    vseq = o;  o = al(o + (int64_t)N * 4);
    bytes = o;
  }
};

// Fused tail of one execute (world 1): bucket minima of every transition,
// then (chain = 1) suffix vectors + reachable optimal edges on CTA 0, the
// least-index argmin of those buckets on the other CTAs, and the backtrack on
// CTA 0 -- one cooperative launch with grid barriers between the phases
// (chain = 0: the argmin of every bucket, cfp_segment_costs).
struct TailParams {
  const ArgminParams* aps;      // [nslot]
  const int64_t* pair_off;      // [nslot + 1] compact buckets (Din * Do) per slot
  const int64_t* orig_off;      // [nslot + 1] caller-layout buckets (Din * Do_orig) per slot
  int32_t nslot;
  int32_t chain;
  ChainParams cp;               // shared-memory chain (cp.mode set per part by the kernel)
  unsigned int* sync;           // [4] zero between launches (the kernel leaves them zero)
  uint64_t* phase_ts;           // nullable: %globaltimer of CTA 0 at each phase boundary [5]
  int32_t squaring;             // chain: 1 repeated squaring + doubling for runs, 0 sequential recurrence
  int32_t levels;               // chain: largest squaring level of a run (P_0 .. P_levels)
  int32_t smax;                 // chain: largest state count (<= 32)
  int32_t kmax_arg;             // argmin: largest K (digit scratch [K][1024] u16)
  int64_t arg_tab_off[32];      // argmin: byte offset of slot s's staged W/R tables (16-aligned), nslot <= 32
  int64_t arg_desc_off;         // argmin: byte offset of the descriptor copies [nslot]
};


// ---------------------------------------------------------------------------
// Memory-constrained search (cfp_mem.cu).
// A type's digits split into a prefix [0, P) (every cross-edge consumer is
// here) and a suffix [P, K).  ctx = prefix digits sharing an intra edge with a
// suffix digit.  For ctx value c and suffix combination sigma the host
// tabulates T[c][sigma] = every Eq. 3 term touching a suffix digit; K0[p] =
// every term inside the prefix.  Cost of combination (p, sigma) =
// K0[p] + T[ctx(p)][sigma].  Buckets: output layout v and quantised plan
// memory q = ceil((mP(p) + mS(sigma)) / quantum) (each plan's memory is
// quantised).  Prefixes are grouped by exact mP; for group g the suffix class
// is cls = vslot * RQs + rs, rs = q - q0(g), q0(g) = ceil((mP_g + mS_min) /
// quantum), vslot = s_o when o is a suffix digit, else 0 (v then comes from
// the prefix).  Suffixes sorted by (vslot, mS): every class of a group is one
// contiguous run of that order.
// ---------------------------------------------------------------------------
constexpr int kMemFoldRows = 64;     // rows staged per fold step
constexpr int kMemFoldStage = 128;   // fold rows per stage x sizeof(V) (32 u32 rows, 16 u64 rows)
constexpr int kMemFoldQuads = 48;    // class quads per fold CTA at most (smem, copies per thread)
constexpr int kMemNPF = 4;           // prefixes per enumeration thread

struct MemPrefixMap {
  int32_t P;
  int32_t radix[kMaxDigits];
  int64_t stride[kMaxDigits];        // natural (big-endian) stride of each prefix digit
  int32_t nctx;                      // ctx digits (canonical order)
  int32_t ctx_pos[kMaxDigits];
  int32_t nnon;                      // other prefix digits (canonical order)
  int32_t non_pos[kMaxDigits];
};

// Prefix rows are ordered by position pos: prefixes sorted by (ctx value,
// prefix-memory class, p) -- perm[pos] = p.  Enumeration tiles (<= 1024
// positions) and fold tiles (<= kMemFoldTile positions) never straddle a ctx
// value resp. a (ctx, class) group.  B is class-quad-major: B[cls/4][pos][cls%4]
// (coalesced enumeration stores, 16-byte fold loads).
constexpr int kMemFoldTile = 512;

// a0 of the memory-constrained search: the per-prefix K0 and the per-ctx
// suffix tables (canonical Tc and the (slot, memory)-sorted Ts) summed on the
// device from the raw input values (every execute; the host keeps only the
// structure).  One job = one table of one type.
struct MemValTerm {
  int32_t kind;                      // 0 unary block a: raw comp (+ comm) ; 1 pair R[d_a][d_b]
  int32_t a, b;                      // block ids
  int32_t db;                        // pair: row length (radix of b)
  int64_t off, off2;                 // raw offsets: comp / table; comm (< 0: none)
};
struct MemValJob {
  int32_t kind;                      // 0: K0[p] over the prefix; 1: Tc[c][sigma]; 2: Ts[c][i], sigma = order[i]
  int32_t P, K;                      // prefix length, blocks
  int32_t radix[kMaxDigits];         // original radices of the blocks
  int32_t nctx, ctx_pos[kMaxDigits]; // ctx blocks (canonical order)
  int32_t nterm;
  MemValTerm term[48];
  int64_t n;                         // entries
  int64_t nS, Tlen;                  // suffix combinations, sorted row length
  const int32_t* order;              // kind 2: [nS] sigma of sorted position i
  void* out;
  int64_t block0;                    // first CTA of this job in the launch
};

struct MemEnumParams {
  int32_t Wc;                        // classes per prefix row
  int32_t Tlen;                      // padded sorted row length (multiple of 4)
  int64_t nP;
  const void* Ts;                    // [nC][Tlen] suffixes sorted by (vslot, exact memory), CAP padded
  const int2* runs;                  // [ngroups][Wc] class runs [start, end) of the sorted row
  const int4* ctiles;                // CTA: (first warp tile, warp tiles <= 8, ctx, 0)
  const int4* wtiles;                // warp: (pos_start, count <= 32 * NPF, prefix group, 0)
  const int32_t* perm;
  const void* K0;                    // [nP] natural prefix order
  void* B;                           // [Wc/4][nP][4] out: K0[p] + min over the class
  uint32_t one;                      // 1 (the FMA-pipe adds' multiplier, opaque to the compiler)
};

struct MemFoldParams {
  MemPrefixMap pm;
  int32_t Din, DinP;
  int32_t nq;                        // cross terms
  int32_t q_pos[kMaxCross];          // prefix position of each consumer
  int64_t q_off[kMaxCross];          // element offset of Q^T[s][DinP] in `vals`
  const void* vals;
  int32_t Wc, ncolblk, fc;           // fc: columns per block (balanced, multiple of 4)
  int64_t nP;
  const int4* tiles;                 // [ntiles] (pos_start, rows, rowclass, 0)
  const int32_t* perm;               // [nP] position -> prefix
  const void* B;                     // [Wc/4][nP][4]
  void* X;                           // [nP][DinP] cross terms per position (mem_xrows_kernel)
  void* chunk;                       // [ntiles][Din][Wc] out
};

struct MemAminParams {
  int32_t Din, Do, nq;               // output [Din][Do][nq] (u64)
  int32_t RQs, nVp;                  // nVp = Do if o is a prefix digit, else 1
  int32_t o_in_prefix;
  int32_t ntiles, Wc;
  const int4* tiles;
  const void* chunk;
  uint64_t* Am;
};

struct MemArgEntry { int32_t slot, u, v, qi; };

struct MemArgSlot {                  // one transition (argmin side)
  MemPrefixMap pm;
  int32_t Din, DinP, Do, nq, RQs, nVp, o_in_prefix, Wc, ntiles;
  int32_t nqx;
  int64_t nP;
  int32_t q_pos[kMaxCross];
  int64_t q_off[kMaxCross];
  const void* vals;
  const int4* tiles;
  const int32_t* perm;
  const void* B;
  const void* chunk;
  const void* K0;
  const void* Tc;                    // [nC][nS] canonical suffix order
  const int32_t* svs;                // [nS] output slot of each suffix combination
  const uint64_t* sms;               // [nS] its exact memory mS
  const int32_t* gP;                 // [nP] prefix group (natural prefix order)
  const uint64_t* gmem;              // [ngroups] group memory mP_g
  const int32_t* gq0;                // [ngroups] q0(g)
  uint64_t quantum;
  int64_t nS;
  const uint64_t* Am;
  uint64_t* Im;                      // [Din][Do][nq]
};

struct MemInst {                     // one chain instance
  int32_t slot, rows, cols, nq;
  int32_t qlo;
  int32_t K;
  int32_t radix_off;                 // into MemChainParams::radix
  int32_t pad_;
  const uint64_t* Am;
  const uint64_t* Im;
};

struct MemChainParams {
  int32_t N;
  int32_t C;                         // Qmax + 1
  const MemInst* inst;
  const int64_t* goff;               // [N + 2] row offsets (times C)
  uint64_t* G;
  // BFS / argmin list
  uint32_t* need;                    // bitsets per slot
  const int64_t* need_off;           // [nslot + 1] word offsets
  int32_t nslot;
  MemArgEntry* list;
  int32_t* count;
  int32_t list_cap;
  // plan outputs (device)
  const int32_t* radix;
  int32_t kmax;
  uint64_t* total;
  uint64_t* seg_index;
  uint64_t* seg_ns;
  int64_t* seg_q;
  int32_t* digits;
  int32_t* status;
};

// ---------------------------------------------------------------------------
// Dense per-plan tables (cfp_dense.cu).  W_t[idx] is the
// profiled time of whole-segment plan idx (uint32, 0xFFFFFFFF = infeasible).
// Rows: prefix p = the cross-edge consumer digits (and the output digit when
// it is not the last one); row p = the prod(suffix) consecutive entries.
// ---------------------------------------------------------------------------
constexpr int kDenseChunk = 128;     // prefixes per fold chunk

struct DenseRowParams {
  const uint32_t* W;
  int64_t nP, nS;
  int32_t nVs;                       // Do (output digit last) or 1 (output digit in the prefix)
  int32_t T;                         // threads per CTA used (4T or T a multiple of Do)
  int32_t vec;                       // 16-byte loads
  uint32_t* B;                       // [nP][nVs]
};

struct DenseSlotParams {             // one transition
  const uint32_t* W;
  int64_t nP, nS;
  int64_t p_lo;                      // global prefix row of local row 0 (rank's shard; 0 at world 1)
  int32_t Din, Do, nVs;
  int64_t o_stride;                  // output digit's stride in the prefix index (nVs == 1)
  int32_t nq;
  int64_t q_off[kMaxCross];          // offset of Q_i [Din][radix_i] in Q
  int64_t q_stride[kMaxCross];       // consumer digit's stride in the prefix index
  int32_t q_radix[kMaxCross];
  const uint32_t* Q;
  const uint32_t* B;
  int64_t nchunks;                   // ceil(nP / kDenseChunk)
  uint64_t* chunk;                   // [nchunks][Din][Do]
  uint64_t* A;                       // [Din][Do]
  uint64_t* I;
};

struct DenseInst {
  int32_t rows, cols, K, radix_off;
  const uint64_t* A;
  const uint64_t* I;
};

struct DenseChainParams {
  int32_t N, kmax;
  const DenseInst* inst;
  const int64_t* goff;               // [N + 2]
  uint64_t* G;
  const int32_t* radix;
  uint64_t* total;
  int32_t* status;
  uint64_t* seg_index;
  uint64_t* seg_ns;
  int32_t* digits;
};

}  // namespace cfp
