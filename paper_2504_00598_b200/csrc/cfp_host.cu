// cfp_host.cu -- host runtime behind include/cfp.h.
//
// Responsibilities (no cost arithmetic of the method happens here -- every
// sum and min is computed by the kernels in cfp_kernels.cu):
//   * validation of the problem structure (EINVAL/ETOOBIG/EVERSION);
//   * pruning: strategies whose own p_j+c_j is infeasible are removed with a
//     monotone index remap, so the lowest-index rule is kept;
//   * precision choice: the narrow (uint32) path is used when the sum of the
//     finite maxima of every term of a combination is < 2^31-1, else uint64;
//   * the enumeration schedule of each segment type (prefix / M / A / B split,
//     register blocking, thread mapping), from a small cost model;
//   * device staging, kernel launch order, the NCCL merge (world > 1) and the
//     chain/backtrack launch.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cfp.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu timelines (no-ops untraced)
#include "cfp_internal.h"

namespace cfp {
template <typename V> cudaError_t launch_compact(const CompactJob*, int, const uint32_t*, const int32_t*, V*, cudaStream_t);
template <typename V> cudaError_t launch_build_tables(const TableSpec*, int, int64_t, const V*, V*, cudaStream_t);
template <typename V> cudaError_t launch_fill(V*, int64_t, V, cudaStream_t);
template <typename V> cudaError_t launch_enum(const EnumParams&, int, int64_t, size_t, cudaStream_t);
template <typename V> cudaError_t launch_argmin(const ArgminParams*, const ArgminEntry*, const int32_t*, int, int, int, cudaStream_t);
cudaError_t launch_chain(const ChainParams&, cudaStream_t);
cudaError_t launch_tail(const TailParams&, int, size_t, cudaStream_t);
cudaError_t tail_max_blocks(size_t, int*);
cudaError_t launch_intpipe(int, int, int, uint32_t*, cudaStream_t);
template <typename V> cudaError_t launch_amin(const ArgminParams*, const int64_t*, int, int64_t, cudaStream_t);
cudaError_t launch_all_pairs(const int64_t*, int, int64_t, ArgminEntry*, int32_t*, cudaStream_t);
cudaError_t launch_edges_to_pairs(const ArgminParams*, ArgminEntry*, const int32_t*, int64_t, cudaStream_t);
template <typename V> cudaError_t launch_minplus_tiled(int, int, int, const V*, const V*, V*, uint32_t*, cudaStream_t);
template <typename V> cudaError_t launch_to_path(const uint64_t*, V*, int64_t, cudaStream_t);
template <typename V> cudaError_t launch_from_path(const V*, const uint32_t*, uint64_t*, uint64_t*, int64_t, cudaStream_t);
template <typename V> cudaError_t launch_fill_random(V*, int64_t, uint64_t, cudaStream_t);
cudaError_t launch_matvec_batch(const uint64_t*, int, int, const uint64_t*, const int64_t*, const int64_t*, uint64_t*,
                                int, cudaStream_t);
}  // namespace cfp

using namespace cfp;

// NVTX range for the duration of a scope (host-side phases of prepare /
// execute / fetch; a profiler attaches the GPU work enqueued inside)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;
static cfp_status fail(cfp_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return fail(CFP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
  } while (0)
#define NCCL_TRY(x)                                                                     \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      return fail(CFP_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_));         \
  } while (0)
#define TRY(x)                             \
  do {                                     \
    cfp_status s_ = (x);                   \
    if (s_ != CFP_OK) return s_;           \
  } while (0)

extern "C" const char* cfp_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- ctx
struct cfp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  int sms = 148;
  bool sim = false;                 // world > 1 without a communicator: shard simulation (test hook)
  bool sharded = false;             // rank-local tables + merge path (world > 1, or a 1-rank communicator)
  bool plan_cache = true;           // CFP_PLAN_CACHE=0: no structure-keyed reuse in cfp_search_plan
  bool fused_tail = true;           // CFP_FUSED_TAIL=0: separate launches after the enumeration (A/B, tests)
  bool tail_squaring = false;       // CFP_TAIL_SQUARING=1: fused chain by repeated squaring (A/B, tests)
  int force_nb = 0;                 // CFP_ENUM_NB: register group size of the enumeration (tuning, tests)
  bool force_o_m = false;           // CFP_ENUM_O_IN_M=1: output block in the M loop (tests)
  int force_p = 0;                  // CFP_ENUM_P: prefix length of the enumeration schedule (tests)
  cfp_prepared* cached = nullptr;   // last cfp_search_plan's prepared plan (device buffers, schedule)
  struct cfp_mem_prepared* mem_cached = nullptr;   // last cfp_search_plan_mem's prepared search
  std::vector<int64_t> cached_key;  //   and its structural key (plan_key)
  bool mem_chain_fused = true;      // CFP_MEM_CHAIN_FUSED=0: one launch per DP step (A/B tests)
  bool dedup = true;                // CFP_DEDUP=0: fold identical transitions separately (A/B tests)
  std::vector<uint32_t> raw_pool;   // host value blob reused across cfp_search_plan calls (its
                                    // pages stay mapped: a fresh 70 KB+ blob page-faulted every call)
  bool no_ym_inplace = false;       // CFP_YM_INPLACE=0: merged Y' rows in their own region (A/B)
  int enum_mix = 3;                 // CFP_ENUM_MIX: full-A loop (B = {o}) on two pipes in groups of 3 or 4
                                    // A values; 0 = ALU pipe only (A/B, tests)
  bool no_full_a = false;           // CFP_ENUM_FULL_A=0: runtime-length A loop only (A/B tests)
  int64_t msplit_min_m = 128;       // M split when nM >= this (CFP_ENUM_MSPLIT_MIN_M; tests force 2)
  // side streams for concurrent per-type enumerations (fork/join by events):
  // the types are independent until the bucket reduction, and running them
  // side by side packs their CTAs into the same waves (no per-launch tail)
  void* pinned = nullptr;           // pinned host staging (value uploads, plan downloads)
  size_t pinned_bytes = 0;
  static constexpr int kLanes = 3;
  cudaStream_t lane[kLanes] = {};
  cudaEvent_t fork = nullptr, join[kLanes] = {};
};

extern "C" cfp_status cfp_nccl_unique_id(void* out128) {
  if (!out128) return fail(CFP_EINVAL, "null output");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return CFP_OK;
}

extern "C" cfp_status cfp_ctx_create(cfp_ctx** out, const cfp_ctx_opts* opts) {
  if (!out) return fail(CFP_EINVAL, "null ctx pointer");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(CFP_ECUDA, std::string("no CUDA device (no CPU fallback exists): ") +
                               (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  std::unique_ptr<cfp_ctx> c(new cfp_ctx());
  if (opts) {
    c->device = opts->device;
    c->world = opts->world < 1 ? 1 : opts->world;
    c->rank = opts->rank;
  }
  if (c->rank < 0 || c->rank >= c->world) return fail(CFP_EINVAL, "rank out of range");
  if (c->device < 0 || c->device >= ndev) return fail(CFP_EINVAL, "device out of range");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, c->device));
  if (prop.major < 10)
    return fail(CFP_ECUDA, "this library is built for sm_100a (B200); found sm_" +
                               std::to_string(prop.major) + std::to_string(prop.minor));
  c->sms = prop.multiProcessorCount;
  if (const char* fa = getenv("CFP_ENUM_FULL_A")) c->no_full_a = atoi(fa) == 0;
  if (const char* yi = getenv("CFP_YM_INPLACE")) c->no_ym_inplace = atoi(yi) == 0;
  if (const char* mx = getenv("CFP_ENUM_MIX")) c->enum_mix = atoi(mx) == 4 ? 4 : atoi(mx) == 0 ? 0 : 3;
  if (const char* dd = getenv("CFP_DEDUP")) c->dedup = atoi(dd) != 0;
  if (const char* mf = getenv("CFP_MEM_CHAIN_FUSED")) c->mem_chain_fused = atoi(mf) != 0;
  if (const char* pc = getenv("CFP_PLAN_CACHE")) c->plan_cache = atoi(pc) != 0;
  if (const char* ft = getenv("CFP_FUSED_TAIL")) c->fused_tail = atoi(ft) != 0;
  if (const char* sq = getenv("CFP_TAIL_SQUARING")) c->tail_squaring = atoi(sq) != 0;
  if (const char* nb = getenv("CFP_ENUM_NB")) c->force_nb = atoi(nb);
  if (const char* om = getenv("CFP_ENUM_O_IN_M")) c->force_o_m = atoi(om) != 0;
  if (const char* fp = getenv("CFP_ENUM_P")) c->force_p = atoi(fp);
  if (const char* ms = getenv("CFP_ENUM_MSPLIT_MIN_M")) c->msplit_min_m = std::max(2LL, atoll(ms));
  if (opts && opts->cuda_stream) {
    c->stream = (cudaStream_t)opts->cuda_stream;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  for (int i = 0; i < cfp_ctx::kLanes; ++i) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->lane[i], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->join[i], cudaEventDisableTiming));
  }
  CUDA_TRY(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  {
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, c->device));
    uint64_t thr = ~0ull;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  if (c->world > 1 && !opts->nccl_unique_id) {
    c->sim = true;                  // single-process shard simulation: no collective
    c->sharded = true;
  } else if (opts && opts->nccl_unique_id) {
    // world > 1: one rank per GPU; world == 1 with an id: a one-rank
    // communicator, so the merge path and its NCCL calls run on one GPU
    ncclUniqueId id;
    memcpy(&id, opts->nccl_unique_id, sizeof(id));
    NCCL_TRY(ncclCommInitRank(&c->comm, c->world, id, c->rank));
    c->sharded = true;
  }
  *out = c.release();
  return CFP_OK;
}

// grow the ctx's pinned staging buffer to at least `bytes` (the previous
// call's copies have completed: every user of it synchronises)
static cfp_status ctx_pinned(cfp_ctx* c, size_t bytes) {
  if (c->pinned_bytes >= bytes) return CFP_OK;
  if (c->pinned) CUDA_TRY(cudaFreeHost(c->pinned));
  c->pinned = nullptr;
  c->pinned_bytes = 0;
  const size_t nb = std::max<size_t>(bytes, 64 * 1024);
  CUDA_TRY(cudaMallocHost(&c->pinned, nb));
  c->pinned_bytes = nb;
  return CFP_OK;
}

extern "C" cfp_status cfp_ctx_nccl_info(cfp_ctx* c, int32_t* nranks, int32_t* version) {
  if (!c || !nranks || !version) return fail(CFP_EINVAL, "null argument");
  *nranks = 0;
  *version = 0;
  if (!c->comm) return CFP_OK;
  int n = 0, v = 0;
  NCCL_TRY(ncclCommCount(c->comm, &n));
  NCCL_TRY(ncclGetVersion(&v));
  *nranks = n;
  *version = v;
  return CFP_OK;
}

extern "C" void cfp_ctx_destroy(cfp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->cached) cfp_prepared_free(c->cached);     // frees on c->stream: before the streams go
  if (c->mem_cached) cfp_mem_free(c->mem_cached);
  if (c->comm) ncclCommDestroy(c->comm);
  for (int i = 0; i < cfp_ctx::kLanes; ++i) {
    if (c->lane[i]) cudaStreamDestroy(c->lane[i]);
    if (c->join[i]) cudaEventDestroy(c->join[i]);
  }
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// ---------------------------------------------------------------- host helpers
extern "C" cfp_status cfp_shard_range(int64_t units, int64_t align, int32_t world, int32_t rank,
                                      int64_t* lo, int64_t* hi) {
  if (units < 0 || align < 1 || world < 1 || rank < 0 || rank >= world || !lo || !hi)
    return fail(CFP_EINVAL, "bad shard arguments");
  const int64_t blocks = (units + align - 1) / align;
  const int64_t b0 = blocks * rank / world, b1 = blocks * (rank + 1) / world;
  *lo = std::min(units, b0 * align);
  *hi = std::min(units, b1 * align);
  return CFP_OK;
}

extern "C" cfp_status cfp_pack_keys(int64_t n, const uint64_t* cost, const uint64_t* idx,
                                    int32_t idx_bits, uint64_t* keys) {
  if (n < 0 || idx_bits < 1 || idx_bits > 63) return fail(CFP_EINVAL, "bad pack arguments");
  const uint64_t imask = (idx_bits == 64) ? ~0ull : ((1ull << idx_bits) - 1);
  for (int64_t i = 0; i < n; ++i) {
    if (cost[i] == CFP_INF64) { keys[i] = CFP_INF64; continue; }
    if ((cost[i] >> (64 - idx_bits)) != 0 || idx[i] > imask)
      return fail(CFP_EOVERFLOW, "key does not fit the packed layout");
    keys[i] = (cost[i] << idx_bits) | idx[i];
  }
  return CFP_OK;
}

extern "C" cfp_status cfp_unpack_keys(int64_t n, const uint64_t* keys, int32_t idx_bits,
                                      uint64_t* cost, uint64_t* idx) {
  if (n < 0 || idx_bits < 1 || idx_bits > 63) return fail(CFP_EINVAL, "bad unpack arguments");
  const uint64_t imask = (1ull << idx_bits) - 1;
  for (int64_t i = 0; i < n; ++i) {
    if (keys[i] == CFP_INF64) { cost[i] = CFP_INF64; idx[i] = CFP_NOIDX; continue; }
    cost[i] = keys[i] >> idx_bits;
    idx[i] = keys[i] & imask;
  }
  return CFP_OK;
}

// ---------------------------------------------------------------- device buffer
// Stream-ordered allocations from the device's default memory pool (release
// threshold raised at ctx creation), so repeated prepare/search calls reuse
// memory instead of paying cudaMalloc/cudaFree.
static thread_local cudaStream_t g_alloc_stream = nullptr;
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf& o) : n(0), st(nullptr) {    // copies never share ownership:
    (void)o;                                        // a copy of an allocated buffer is empty
    if (o.p) std::abort();                          // (copying a live buffer is a bug)
  }
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  cudaError_t alloc(size_t bytes) {
    release();
    n = bytes;
    st = g_alloc_stream;
    return cudaMallocAsync(&p, bytes ? bytes : 16, st);
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------- problem model
namespace {

struct HostType {
  int K = 0;
  std::vector<int> radix;                   // original
  std::vector<int64_t> comp_off;            // raw blob offsets per block
  std::vector<int64_t> comm_off;            // -1 = none
  int E = 0;
  std::vector<int> esrc, edst;
  std::vector<int64_t> e_off;               // raw blob offset per edge table
  int o = 0;
  // pruning
  std::vector<std::vector<int>> keep;       // compact -> original
  std::vector<int> radix_c;
  bool empty = false;                       // some block has no feasible strategy
  std::vector<uint64_t> wmax, emax;         // finite maxima (bound check)
  bool used = false;
};

struct HostTrans {
  int pred = -1, type = 0, X = 0;
  std::vector<int> xdst;
  std::vector<int64_t> x_off;
  int Din = 1;
  std::vector<uint64_t> xmax;
  bool used = false;
};

int64_t prod(const std::vector<int>& r, int lo, int hi) {
  int64_t n = 1;
  for (int i = lo; i < hi; ++i) n *= r[i];
  return n;
}

}  // namespace

// All device state of a prepared problem.
struct TypeExec {
  int id = 0;
  bool wide = false;
  bool empty = false;
  int K = 0, o = 0, P = 0, NB = 4;
  std::vector<int> role;                    // 0 prefix 1 M 2 A 3 B
  EnumParams ep{};
  int64_t nthreads = 0;
  size_t smem = 0;
  int64_t H = 0;                            // high-part units (sharding)
  int64_t nPl = 0;                          // local prefixes
  std::vector<int> w_off, e_off;            // value blob offsets (elements)
  int64_t xt_off = 0, yt_off = 0, zt_off = 0, k0_off = 0, mtab_off = 0, bp_off = 0;
  std::vector<int> trans;                   // incoming transitions (used)
  int epi_off = 0;                          // first EpiTau of this type
  EvalSpec es{};
  double combos = 0, combos_local = 0;
};

struct TransExec {
  int id = 0, type = 0, Din = 1, Do = 1, Do_orig = 1;
  std::vector<int64_t> q_off;               // value blob offsets of compact Q tables
  std::vector<int64_t> qt_off;              // ... and of their transposed copies
  FoldParams fp{};
  ArgminParams ap{};
  int64_t chunk_off = 0, aval_off = 0, pstar_off = 0;  // scratch offsets (bytes)
  int64_t out_off = 0;                      // offset (elements) of A/I in the out blob
};

struct cfp_prepared {
  cfp_ctx* ctx = nullptr;
  int N = 0, kmax = 0;
  bool do_chain = true;
  std::vector<TypeExec> types;
  std::vector<TransExec> trans;
  std::vector<int> inst;
  std::vector<int> canon;                   // dedup: transition -> canonical identical transition
  // device memory
  DevBuf raw, maps, vals32, vals64, jobs32, jobs64, specs32, specs64, mtab, bp, scratch,
      outAI, chain_inst, chain_runs, chain_mats, chain_moff, chain_G, chain_goff, chain_pow, plan, radix_blob, status,
      merge_keys;
  int njobs32 = 0, njobs64 = 0, nspecs32 = 0, nspecs64 = 0;
  int64_t spec_max32 = 0, spec_max64 = 0;
  std::vector<CompactJob> hjobs32, hjobs64;
  std::vector<EpiTau> epi_host;
  DevBuf epi, aps, pair_off, locAI, edges, reach;
  // fused tail (world 1): one cooperative launch after the enumeration
  bool fused_tail = false;
  int tail_grid = 0, tail_per_sm = 1;
  size_t tail_smem = 0;
  TailParams tp{};
  DevBuf orig_off, tail_sync, phase_ts;
  int64_t reach_bytes = 0;
  int64_t ai = 0, npairs = 0;
  bool has32 = false, has64 = false, use_edges = false;
  int kmax_arg = 1, tabn_max = 1;
  std::vector<TableSpec> hspecs32, hspecs64;
  ChainParams cp{};
  int nruns = 0;
  int launches = 0;
  double combos = 0, combos_local = 0, evals = 0;
  // host-side copies for diagnostics
  std::vector<int> inst_rows, inst_cols;
  // timing
  size_t plan_bytes = 0;          // plan buffer: total, seg_index, seg_ns, digits (status word after it)
  int timing = 0;                 // 1: events around a0 / enumeration / whole; 2: + every phase
  cudaEvent_t ev[7] = {};         // 0 start, 1 a0 done, 2 enumeration done, 3 end,
                                  // 4 bucket minima (+ all-reduce), 5 chain, 6 argmin (+ merge)
  ~cfp_prepared() {
    for (auto& e : ev) if (e) cudaEventDestroy(e);
  }
};

extern "C" void cfp_prepared_free(cfp_prepared* p) { delete p; }

// ---------------------------------------------------------------- planner
namespace {

struct Schedule {
  int P = 0;
  std::vector<int> role;
  int NB = 4, VG = 1;
  double cost = 1e300;
};

// neighbours of a digit set (intra edges) outside the set
std::vector<int> ctx_of(const std::vector<int>& set_mask, const HostType& t) {
  std::vector<int> nb(t.K, 0);
  for (int e = 0; e < t.E; ++e) {
    int a = t.esrc[e], b = t.edst[e];
    if (set_mask[a] && !set_mask[b]) nb[b] = 1;
    if (set_mask[b] && !set_mask[a]) nb[a] = 1;
  }
  return nb;
}

int round_up(int64_t x, int64_t m) { return (int)((x + m - 1) / m * m); }

// Estimated ALU cycles (arbitrary units) of a schedule -- enumeration + fold.
double schedule_cost(const HostType& t, int P, const std::vector<int>& role, int NB, int VG,
                     int ntrans_in, int sms, int din_max) {
  const auto& r = t.radix_c;
  int64_t nP = prod(r, 0, P);
  int64_t nM = 1, na = 1, nb = 1;
  for (int d = P; d < t.K; ++d) {
    if (role[d] == 1) nM *= r[d];
    if (role[d] == 2) na *= r[d];
    if (role[d] == 3) nb *= r[d];
  }
  const int na_pad = round_up(na, 4);
  // low part: ctx prefix digits
  std::vector<int> A(t.K, 0), B(t.K, 0), Mm(t.K, 0);
  for (int d = 0; d < t.K; ++d) { A[d] = role[d] == 2; B[d] = role[d] == 3; Mm[d] = role[d] == 1; }
  auto ca = ctx_of(A, t), cb = ctx_of(B, t);
  int lmin = P;
  for (int d = 0; d < P; ++d) if (ca[d] || cb[d]) { lmin = d; break; }
  // Z ctx (terms touching M only) may also pull prefix digits in; approximate
  for (int e = 0; e < t.E; ++e) {
    int a = t.esrc[e], b = t.edst[e];
    bool touchM = Mm[a] || Mm[b];
    bool touchAB = A[a] || A[b] || B[a] || B[b];
    if (touchM && !touchAB) {
      if (a < P) lmin = std::min(lmin, a);
      if (b < P) lmin = std::min(lmin, b);
    }
  }
  int64_t W = prod(r, lmin, P);
  int64_t Hh = nP / W;
  int64_t Gpad = (Hh + kBlock - 1) / kBlock * kBlock;
  double threads = (double)Gpad * W * VG;
  double per_thread = (double)nM * ((double)NB * na + NB + 10.0) + 40.0;
  (void)na_pad;
  int regs = NB <= 8 ? 40 : NB <= 16 ? 56 : NB <= 24 ? 72 : 96;
  int ctas_per_sm = std::max(1, std::min(8, 65536 / (regs * kBlock)));
  double slots = (double)sms * ctas_per_sm * kBlock;
  double waves = threads / slots;
  double eff_waves = std::max(1.0, std::ceil(waves * 4.0) / 4.0);
  // lanes in a warp run together: per-SMSP issue of NB*na VIADDMNMX at 16 lanes/clk
  double enum_cost = per_thread * eff_waves * slots / (sms * 64.0);
  double fold_cost = (double)ntrans_in * nP * din_max * r[t.o] * 2.0 / (sms * 64.0) + nP * 0.002;
  return enum_cost + fold_cost;
}

Schedule plan_schedule(const HostType& t, const std::vector<int>& fold_digits, int ntrans_in,
                       int sms, int din_max, int force_nb, bool force_o_m, int force_p) {
  const auto& r = t.radix_c;
  int Pmin = 0;
  for (int d : fold_digits) Pmin = std::max(Pmin, d + 1);
  Schedule best;
  // force_nb (CFP_ENUM_NB): register group size override; force_o_m
  // (CFP_ENUM_O_IN_M=1): only schedules with the output block in the M loop
  // -- tuning / test overrides read at ctx creation
  int64_t nP = prod(r, 0, Pmin);
  for (int P = Pmin; P <= t.K; ++P) {
    if (P > Pmin) nP *= r[P - 1];
    if (nP > (int64_t)1 << 26) break;
    if (force_p > 0 && P != std::max(force_p, Pmin)) continue;   // CFP_ENUM_P (tests)
    const int S = t.K - P;
    std::vector<int> role(t.K, 0);
    // enumerate roles of suffix digits (base-3 counter over M/A/B); cap size
    int64_t combos = 1;
    for (int i = 0; i < S; ++i) combos *= 3;
    if (combos > 59049) combos = 59049;
    for (int64_t code = 0; code < combos; ++code) {
      int64_t c = code;
      int na_d = 0, nb_d = 0;
      for (int d = P; d < t.K; ++d) {
        role[d] = 1 + (int)(c % 3);
        c /= 3;
        na_d += role[d] == 2;
        nb_d += role[d] == 3;
      }
      if (S > 9 && (na_d > 2 || nb_d > 2)) continue;
      if (role[t.o] == 2) continue;                    // o never in A
      if (force_o_m && t.o >= P && role[t.o] != 1) continue;
      bool ok = true;
      for (int e = 0; e < t.E && ok; ++e) {
        int a = t.esrc[e], b = t.edst[e];
        if ((role[a] == 2 && role[b] == 3) || (role[a] == 3 && role[b] == 2)) ok = false;
      }
      if (!ok) continue;
      int64_t na = 1, nb = 1;
      for (int d = P; d < t.K; ++d) {
        if (role[d] == 2) na *= r[d];
        if (role[d] == 3) nb *= r[d];
      }
      if (na > 4096 || nb > 32) continue;
      const bool b_is_o = nb_d == 1 && role[t.o] == 3;
      for (int NB : {4, 8, 12, 16, 23, 24, 32}) {
        if (force_nb > 0 && NB != force_nb && nb >= force_nb) continue;   // tuning override
        int VG = (int)((nb + NB - 1) / NB);
        if (VG > 1 && !b_is_o) continue;
        if (NB % 4 != 0 && VG > 1) continue;             // register groups start on 16-byte rows
        if (NB > 4 && NB >= 2 * nb && NB != 4) continue;
        double cost = schedule_cost(t, P, role, NB, VG, ntrans_in, sms, din_max);
        if (cost < best.cost * 0.999) {
          best.cost = cost;
          best.P = P;
          best.role = role;
          best.NB = NB;
          best.VG = VG;
        }
      }
    }
  }
  return best;
}

}  // namespace

// ---------------------------------------------------------------- prepare
namespace {

struct Builder {
  // raw uint32 blob
  std::vector<uint32_t> raw;
  std::vector<int32_t> maps;
  int64_t vals32 = 0, vals64 = 0;          // element counts
  int64_t der32 = 0, der64 = 0;            // derived table sizes (appended after vals)

  int64_t put_raw(const uint32_t* p, int64_t n) {
    int64_t off = (int64_t)raw.size();
    raw.insert(raw.end(), p, p + n);
    return off;
  }
  int put_map(const std::vector<int>& m) {
    int off = (int)maps.size();
    maps.insert(maps.end(), m.begin(), m.end());
    return off;
  }
  int64_t& vcount(bool wide) { return wide ? vals64 : vals32; }
};


}  // namespace

// largest finite (!= CFP_INF32) entry of t[0, n), 0 if none: 8 independent
// lanes, so the host compiler vectorises it (a serial max chain was most of a
// reused-plan call's host model time)
static inline uint32_t max_finite(const uint32_t* t, int64_t n) {
  uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t q = 0;
  for (; q + 8 <= n; q += 8)
    for (int k = 0; k < 8; ++k) {
      const uint32_t v = t[q + k] == CFP_INF32 ? 0u : t[q + k];
      m[k] = m[k] > v ? m[k] : v;
    }
  uint32_t r = 0;
  for (int k = 0; k < 8; ++k) r = r > m[k] ? r : m[k];
  for (; q < n; ++q) {
    const uint32_t v = t[q] == CFP_INF32 ? 0u : t[q];
    r = r > v ? r : v;
  }
  return r;
}

static cfp_status validate_and_model(const cfp_problem* p, std::vector<HostType>& T,
                                     std::vector<HostTrans>& X, Builder& b, bool chain) {
  if (!p) return fail(CFP_EINVAL, "null problem");
  if (p->abi_version != CFP_ABI_VERSION)
    return fail(CFP_EVERSION, "abi_version " + std::to_string(p->abi_version) + " != " +
                                  std::to_string(CFP_ABI_VERSION));
  if (p->num_types < 1 || !p->types) return fail(CFP_EINVAL, "num_types < 1");
  if (p->num_transitions < 1 || !p->transitions) return fail(CFP_EINVAL, "num_transitions < 1");
  if (p->num_instances < 1 || !p->inst_transition) return fail(CFP_EINVAL, "num_instances < 1");
  T.resize(p->num_types);
  for (int i = 0; i < p->num_types; ++i) {
    const cfp_segment_type& s = p->types[i];
    HostType& h = T[i];
    if (s.num_blocks < 1) return fail(CFP_EINVAL, "type " + std::to_string(i) + ": K < 1");
    if (s.num_blocks > CFP_MAX_BLOCKS) return fail(CFP_ETOOBIG, "type " + std::to_string(i) + ": K > 32");
    if (!s.radix || !s.comp_ns) return fail(CFP_EINVAL, "type " + std::to_string(i) + ": null table");
    h.K = s.num_blocks;
    h.radix.assign(s.radix, s.radix + h.K);
    double space = 1;
    for (int d : h.radix) {
      if (d < 1) return fail(CFP_EINVAL, "type " + std::to_string(i) + ": radix < 1");
      space *= d;
    }
    if (space > 281474976710656.0) return fail(CFP_ETOOBIG, "type " + std::to_string(i) + ": prod D > 2^48");
    if (s.out_block < 0 || s.out_block >= h.K)
      return fail(CFP_EINVAL, "type " + std::to_string(i) + ": out_block out of range");
    h.o = s.out_block;
    if (s.num_edges < 0 || (s.num_edges > 0 && (!s.edge_src || !s.edge_dst || !s.edge_ns)))
      return fail(CFP_EINVAL, "type " + std::to_string(i) + ": bad edges");
    h.E = s.num_edges;
    int64_t off = 0;
    for (int j = 0; j < h.K; ++j) {
      h.comp_off.push_back(b.put_raw(s.comp_ns + off, h.radix[j]));
      h.comm_off.push_back(s.comm_ns ? b.put_raw(s.comm_ns + off, h.radix[j]) : -1);
      off += h.radix[j];
    }
    int64_t eoff = 0;
    for (int e = 0; e < h.E; ++e) {
      int a = s.edge_src[e], c = s.edge_dst[e];
      if (a < 0 || a >= h.K || c < 0 || c >= h.K || a == c)
        return fail(CFP_EINVAL, "type " + std::to_string(i) + ": bad edge " + std::to_string(e));
      h.esrc.push_back(a);
      h.edst.push_back(c);
      int64_t n = (int64_t)h.radix[a] * h.radix[c];
      h.e_off.push_back(b.put_raw(s.edge_ns + eoff, n));
      eoff += n;
    }
    // pruning + maxima
    h.keep.resize(h.K);
    h.radix_c.resize(h.K);
    h.wmax.assign(h.K, 0);
    off = 0;
    for (int j = 0; j < h.K; ++j) {
      h.keep[j].reserve(h.radix[j]);
      for (int q = 0; q < h.radix[j]; ++q) {
        uint32_t pc = s.comp_ns[off + q], cc = s.comm_ns ? s.comm_ns[off + q] : 0;
        if (pc == CFP_INF32 || cc == CFP_INF32) continue;
        h.keep[j].push_back(q);
        h.wmax[j] = std::max<uint64_t>(h.wmax[j], (uint64_t)pc + cc);
      }
      h.radix_c[j] = (int)h.keep[j].size();
      if (h.radix_c[j] == 0) h.empty = true;
      off += h.radix[j];
    }
    eoff = 0;
    for (int e = 0; e < h.E; ++e) {
      int a = h.esrc[e], c = h.edst[e];
      uint64_t m = 0;
      if ((int)h.keep[a].size() == h.radix[a] && (int)h.keep[c].size() == h.radix[c]) {
        // every strategy feasible: one branch-free pass over the table (INF -> 0)
        const uint32_t* t = s.edge_ns + eoff;
        const int64_t n = (int64_t)h.radix[a] * h.radix[c];
        uint32_t mm = 0;
        mm = max_finite(t, n);
        m = mm;
      } else {
        for (int x : h.keep[a])
          for (int y : h.keep[c]) {
            uint32_t v = s.edge_ns[eoff + (int64_t)x * h.radix[c] + y];
            if (v != CFP_INF32) m = std::max<uint64_t>(m, v);
          }
      }
      h.emax.push_back(m);
      eoff += (int64_t)h.radix[a] * h.radix[c];
    }
  }
  X.resize(p->num_transitions);
  for (int i = 0; i < p->num_transitions; ++i) {
    const cfp_transition& s = p->transitions[i];
    HostTrans& h = X[i];
    if (s.type < 0 || s.type >= p->num_types)
      return fail(CFP_EINVAL, "transition " + std::to_string(i) + ": bad type");
    if (s.pred_type < -1 || s.pred_type >= p->num_types)
      return fail(CFP_EINVAL, "transition " + std::to_string(i) + ": bad pred_type");
    h.pred = s.pred_type;
    h.type = s.type;
    h.Din = s.pred_type < 0 ? 1 : T[s.pred_type].radix[T[s.pred_type].o];
    if (s.num_in_edges < 0 || (s.num_in_edges > 0 && (!s.in_dst || !s.in_ns)))
      return fail(CFP_EINVAL, "transition " + std::to_string(i) + ": bad cross edges");
    h.X = s.num_in_edges;
    const HostType& ty = T[h.type];
    int64_t off = 0;
    for (int x = 0; x < h.X; ++x) {
      int j = s.in_dst[x];
      if (j < 0 || j >= ty.K)
        return fail(CFP_EINVAL, "transition " + std::to_string(i) + ": bad in_dst");
      h.xdst.push_back(j);
      int64_t n = (int64_t)h.Din * ty.radix[j];
      h.x_off.push_back(b.put_raw(s.in_ns + off, n));
      uint64_t m = 0;
      if ((int)ty.keep[j].size() == ty.radix[j]) {
        const uint32_t* t = s.in_ns + off;
        uint32_t mm = 0;
        mm = max_finite(t, n);
        m = mm;
      } else {
        for (int u = 0; u < h.Din; ++u)
          for (int y : ty.keep[j]) {
            uint32_t v = s.in_ns[off + (int64_t)u * ty.radix[j] + y];
            if (v != CFP_INF32) m = std::max<uint64_t>(m, v);
          }
      }
      h.xmax.push_back(m);
      off += n;
    }
  }
  for (int n = 0; n < p->num_instances; ++n) {
    int tr = p->inst_transition[n];
    if (tr < 0 || tr >= p->num_transitions)
      return fail(CFP_EINVAL, "instance " + std::to_string(n) + ": bad transition id");
    const HostTrans& h = X[tr];
    if (chain && n == 0 && h.pred != -1)
      return fail(CFP_EINVAL, "instance 0 must use a chain-start transition (pred_type = -1)");
    if (chain && n > 0) {
      int prev_type = X[p->inst_transition[n - 1]].type;
      if (h.pred != prev_type)
        return fail(CFP_EINVAL, "instance " + std::to_string(n) + ": pred_type " +
                                    std::to_string(h.pred) + " != type of instance " +
                                    std::to_string(n - 1) + " (" + std::to_string(prev_type) + ")");
    }
    X[tr].used = true;
    T[h.type].used = true;
  }
  return CFP_OK;
}

// Identical transitions.  Two used transitions into the same type with the
// same predecessor output strategies (radix and feasible set), the same
// consumer blocks and byte-identical cross tables have identical segment
// tables (A, I): instances of the later one are pointed at the first, and the
// later one is marked unused (not folded).  C3/C5: L1 -> L and L -> L carry
// the same reshard profiles.
static std::vector<int> dedup_transitions(const std::vector<HostType>& T, std::vector<HostTrans>& X,
                                          const Builder& b, std::vector<int>& inst) {
  auto out_keep = [&](int pred) {
    return pred < 0 ? std::vector<int>{0} : T[pred].keep[T[pred].o];
  };
  std::vector<int> canon(X.size());
  for (int x = 0; x < (int)X.size(); ++x) {
    canon[x] = x;
    if (!X[x].used) continue;
    for (int y = 0; y < x; ++y) {
      const HostTrans& a = X[x];
      const HostTrans& c = X[y];
      if (!c.used || canon[y] != y || a.type != c.type || a.Din != c.Din || a.X != c.X || a.xdst != c.xdst)
        continue;
      if (out_keep(a.pred) != out_keep(c.pred)) continue;
      bool same = true;
      for (int q = 0; q < a.X && same; ++q) {
        const int64_t n = (int64_t)a.Din * T[a.type].radix[a.xdst[q]];
        same = std::equal(b.raw.begin() + a.x_off[q], b.raw.begin() + a.x_off[q] + n, b.raw.begin() + c.x_off[q]);
      }
      if (same) { canon[x] = y; break; }
    }
  }
  for (int& t : inst) t = canon[t];
  for (int x = 0; x < (int)X.size(); ++x)
    if (canon[x] != x) X[x].used = false;
  return canon;
}

// Precision of a type: narrow (uint32) iff the sum of the finite maxima of
// every term of one combination (unary, intra, worst incoming cross) < CAP32.
static bool type_is_wide(const std::vector<HostType>& T, const std::vector<HostTrans>& X, int i) {
  long double bound = 0;
  for (auto v : T[i].wmax) bound += v;
  for (auto v : T[i].emax) bound += v;
  long double xb = 0;
  for (const HostTrans& x : X) {
    if (!x.used || x.type != i) continue;
    long double s = 0;
    for (auto v : x.xmax) s += v;
    xb = std::max(xb, s);
  }
  bound += xb;
  return !(bound < (long double)kCap32);
}

// Chain overflow guard: the sum over instances of every term's finite maximum < 2^63.
static cfp_status check_chain_overflow(const std::vector<HostType>& T, const std::vector<HostTrans>& X,
                                       const std::vector<int>& inst) {
  long double tot = 0;
  for (int t : inst) {
    const HostTrans& h = X[t];
    const HostType& ty = T[h.type];
    long double s = 0;
    for (auto v : ty.wmax) s += v;
    for (auto v : ty.emax) s += v;
    for (auto v : h.xmax) s += v;
    tot += s;
  }
  if (tot >= 9.2e18L) return fail(CFP_EOVERFLOW, "a finite plan cost could reach 2^63");
  return CFP_OK;
}

// Structural key of a validated problem for cfp_search_plan's plan reuse.
// Everything prepare derives on the host from the problem -- shapes, the
// feasible strategy sets (INF pattern), the term maxima (precision and
// overflow decisions), the deduplicated instance list -- is in the key; the
// table values themselves reach the device through the raw blob, which is
// uploaded again on every call.
static std::vector<int64_t> plan_key(const cfp_problem* p, const std::vector<HostType>& T,
                                     const std::vector<HostTrans>& X, const std::vector<int>& inst,
                                     const Builder& b) {
  std::vector<int64_t> k;
  k.push_back((int64_t)T.size());
  k.push_back((int64_t)X.size());
  k.push_back((int64_t)b.raw.size());
  k.push_back((int64_t)p->mesh.ndim);
  for (const HostType& h : T) {
    k.push_back(h.K);
    k.push_back(h.o);
    k.push_back(h.E);
    k.insert(k.end(), h.radix.begin(), h.radix.end());
    k.insert(k.end(), h.esrc.begin(), h.esrc.end());
    k.insert(k.end(), h.edst.begin(), h.edst.end());
    for (int64_t o : h.comm_off) k.push_back(o < 0 ? -1 : 1);
    for (const auto& kp : h.keep) {
      k.push_back((int64_t)kp.size());
      k.insert(k.end(), kp.begin(), kp.end());
    }
    k.push_back(h.used ? 1 : 0);
  }
  for (const HostTrans& x : X) {
    k.push_back(x.pred);
    k.push_back(x.type);
    k.push_back(x.X);
    k.push_back(x.Din);
    k.push_back(x.used ? 1 : 0);
    k.insert(k.end(), x.xdst.begin(), x.xdst.end());
  }
  // the term maxima enter only through the precision of each type
  for (int i = 0; i < (int)T.size(); ++i) k.push_back(T[i].used ? (int64_t)type_is_wide(T, X, i) : -1);
  k.push_back((int64_t)inst.size());
  k.insert(k.end(), inst.begin(), inst.end());
  return k;
}

// Derived-table spec over an ordered digit list.  `row_digits` trailing digits
// form a row, padded to `row_pad` entries.
static TableSpec make_spec(const std::vector<int>& digits, const std::vector<int>& radix_c,
                           int row_digits, int64_t row_pad) {
  TableSpec s{};
  s.ndig = (int)digits.size();
  for (int i = 0; i < s.ndig; ++i) s.radix[i] = radix_c[digits[i]];
  int64_t rv = 1, rows = 1;
  for (int i = 0; i < s.ndig; ++i) {
    if (i >= s.ndig - row_digits) rv *= s.radix[i];
    else rows *= s.radix[i];
  }
  s.row_digits = row_digits;
  s.row_valid = rv;
  s.rows = rows;
  s.row = std::max<int64_t>(row_pad, rv);
  return s;
}

static cfp_status add_term(TableSpec& s, const std::vector<int>& digits, int kind, int a, int b,
                           int db, int64_t off) {
  if (s.nterm >= kMaxTerms) return fail(CFP_ETOOBIG, "too many cost terms in one table");
  Term t{};
  t.kind = kind;
  t.a = (int)(std::find(digits.begin(), digits.end(), a) - digits.begin());
  t.b = kind == 1 ? (int)(std::find(digits.begin(), digits.end(), b) - digits.begin()) : 0;
  t.db = db;
  t.off = off;
  s.term[s.nterm++] = t;
  return CFP_OK;
}

static int64_t stride_in(const TableSpec& s, int pos) {
  // stride of digit position `pos` in the padded table layout
  int64_t st = 1;
  const int first_row = s.ndig - s.row_digits;
  if (pos >= first_row) {
    for (int i = s.ndig - 1; i > pos; --i) st *= s.radix[i];
    return st;
  }
  st = s.row;
  for (int i = first_row - 1; i > pos; --i) st *= s.radix[i];
  return st;
}

// Distinct matrices + shared-memory budget of the single-CTA chain kernel.
static cfp_status setup_chain_staging(ChainParams& cp, const std::vector<ChainInst>& mats, int64_t g_elems,
                                      int levels_max, int smax, DevBuf& dmats, DevBuf& dmoff,
                                      cudaStream_t st) {
  std::vector<int64_t> moff(mats.size());
  int64_t tot = 0;
  for (size_t m = 0; m < mats.size(); ++m) {
    moff[m] = tot;
    tot += (int64_t)mats[m].rows * mats[m].cols;
  }
  CUDA_TRY(dmats.alloc(std::max<size_t>(1, mats.size()) * sizeof(ChainInst)));
  CUDA_TRY(dmoff.alloc(std::max<size_t>(1, mats.size()) * sizeof(int64_t)));
  if (!mats.empty()) {
    CUDA_TRY(cudaMemcpyAsync(dmats.p, mats.data(), mats.size() * sizeof(ChainInst), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dmoff.p, moff.data(), moff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  cp.nmat = (int)mats.size();
  cp.mats = dmats.as<ChainInst>();
  cp.baseA = mats.empty() ? nullptr : mats[0].A;     // matrices are contiguous in moff order
  cp.baseI = mats.empty() ? nullptr : mats[0].I;
  cp.moff = dmoff.as<int64_t>();
  cp.mat_elems = tot;
  cp.levels_max = levels_max;
  cp.smax = smax;
  const int64_t need = (tot * (cp.backtrack ? 2 : 1) + g_elems + (int64_t)levels_max * smax * smax) * 8 +
                       (int64_t)(cp.N + 2) * 8 + (int64_t)mats.size() * 8 + (int64_t)cp.N * 16 + 128 +
                       g_elems * 2 + 16 + (int64_t)cp.N * 4 + 16 + ((tot + 31) / 32) * 4 + 16 +
                       g_elems * 4 + (int64_t)cp.N * 4 + 16;        // successor / reach masks
  cp.smem_bytes = need <= 200 * 1024 ? need : 0;
  return CFP_OK;
}

// CFP_DEBUG_PREP=1: host-side phase times of prepare (stderr)
struct PrepTimer {
  bool on = getenv("CFP_DEBUG_PREP") != nullptr;
  std::vector<std::pair<const char*, double>> marks;
  double t0 = now();
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
  }
  void mark(const char* what) { if (on) marks.emplace_back(what, now()); }
  ~PrepTimer() {
    if (!on) return;
    double prev = t0;
    fprintf(stderr, "prepare (us):");
    for (auto& m : marks) { fprintf(stderr, " %s %.1f", m.first, m.second - prev); prev = m.second; }
    fprintf(stderr, "\n");
  }
};

// The validated host model of a problem (validate_and_model + dedup): built
// once per cfp_search_plan call and handed to prepare_impl on a cache miss.
struct HostModel {
  std::vector<HostType> T;
  std::vector<HostTrans> X;
  Builder b;
  std::vector<int> inst;
  std::vector<int> canon;       // transition -> the identical transition whose tables it shares
};

static cfp_status build_model(cfp_ctx* ctx, const cfp_problem* p, bool do_chain, HostModel& m) {
  TRY(validate_and_model(p, m.T, m.X, m.b, do_chain));
  m.inst.assign(p->inst_transition, p->inst_transition + p->num_instances);
  if (ctx->dedup) m.canon = dedup_transitions(m.T, m.X, m.b, m.inst);
  return CFP_OK;
}

static cfp_status prepare_impl(cfp_ctx* ctx, const cfp_problem* p, bool do_chain,
                               cfp_prepared** out, HostModel* pre = nullptr) {
  NvtxRange nv("cfp_prepare");
  PrepTimer tm;
  *out = nullptr;
  g_alloc_stream = ctx->stream;
  HostModel local;
  if (!pre) {
    TRY(build_model(ctx, p, do_chain, local));
    pre = &local;
  }
  std::vector<HostType>& T = pre->T;
  std::vector<HostTrans>& X = pre->X;
  Builder& b = pre->b;
  tm.mark("validate");
  std::unique_ptr<cfp_prepared> P(new cfp_prepared());
  P->ctx = ctx;
  P->do_chain = do_chain;
  P->N = p->num_instances;
  P->inst = pre->inst;
  P->canon = pre->canon;
  const int world = ctx->world, rank = ctx->rank;

  TRY(check_chain_overflow(T, X, P->inst));

  // ---- per type: precision, schedule, value-blob layout
  std::map<int, int> type_slot, trans_slot;
  for (int i = 0; i < (int)T.size(); ++i) {
    if (!T[i].used) continue;
    TypeExec te;
    te.id = i;
    te.K = T[i].K;
    te.o = T[i].o;
    te.empty = T[i].empty;
    for (int x = 0; x < (int)X.size(); ++x)
      if (X[x].used && X[x].type == i) te.trans.push_back(x);
    te.wide = type_is_wide(T, X, i);
    double c = 1;
    for (int d : T[i].radix_c) c *= d;
    te.combos = te.empty ? 0 : c;
    type_slot[i] = (int)P->types.size();
    P->types.push_back(te);
  }
  for (int x = 0; x < (int)X.size(); ++x) {
    if (!X[x].used) continue;
    TransExec tx;
    tx.id = x;
    tx.type = X[x].type;
    tx.Din = X[x].Din;
    tx.Do = T[tx.type].radix_c[T[tx.type].o];
    tx.Do_orig = T[tx.type].radix[T[tx.type].o];
    trans_slot[x] = (int)P->trans.size();
    P->trans.push_back(tx);
  }
  // compaction jobs + value blob offsets
  for (TypeExec& te : P->types) {
    const HostType& t = T[te.id];
    if (te.empty) continue;
    auto& jobs = te.wide ? P->hjobs64 : P->hjobs32;
    int64_t& vc = b.vcount(te.wide);
    std::vector<int> mo(t.K);
    for (int j = 0; j < t.K; ++j) mo[j] = b.put_map(t.keep[j]);
    for (int j = 0; j < t.K; ++j) {
      CompactJob cj{};
      cj.kind = 0; cj.rows = 1; cj.cols = t.radix_c[j]; cj.raw_cols = t.radix[j];
      cj.raw_off = t.comp_off[j]; cj.raw_off2 = t.comm_off[j];
      cj.map_r = -1; cj.map_c = mo[j]; cj.out_off = vc;
      te.w_off.push_back((int)vc);
      vc += cj.cols;
      jobs.push_back(cj);
    }
    for (int e = 0; e < t.E; ++e) {
      int a = t.esrc[e], c = t.edst[e];
      CompactJob cj{};
      cj.kind = 1; cj.rows = t.radix_c[a]; cj.cols = t.radix_c[c]; cj.raw_cols = t.radix[c];
      cj.raw_off = t.e_off[e]; cj.raw_off2 = -1; cj.map_r = mo[a]; cj.map_c = mo[c]; cj.out_off = vc;
      te.e_off.push_back((int)vc);
      vc += (int64_t)cj.rows * cj.cols;
      jobs.push_back(cj);
    }
    for (int x : te.trans) {
      TransExec& tx = P->trans[trans_slot[x]];
      const HostTrans& h = X[x];
      for (int q = 0; q < h.X; ++q) {
        int j = h.xdst[q];
        CompactJob cj{};
        cj.kind = 2; cj.rows = h.Din; cj.cols = t.radix_c[j]; cj.raw_cols = t.radix[j];
        cj.raw_off = h.x_off[q]; cj.raw_off2 = -1; cj.map_r = -1; cj.map_c = mo[j]; cj.out_off = vc;
        tx.q_off.push_back(vc);
        vc += (int64_t)cj.rows * cj.cols;
        jobs.push_back(cj);
        // transposed copy for the enumeration epilogue (16-byte aligned rows)
        vc = (vc + 3) & ~3LL;
        CompactJob ct = cj;
        ct.kind = 3; ct.rows_pad = (h.Din + 3) & ~3; ct.out_off = vc;
        tx.qt_off.push_back(vc);
        vc += (int64_t)ct.rows_pad * ct.cols;
        jobs.push_back(ct);
      }
    }
    // map offsets for argmin remap
    for (int x : te.trans) {
      TransExec& tx = P->trans[trans_slot[x]];
      for (int j = 0; j < t.K; ++j) {
        tx.ap.map_off[j] = mo[j];
        tx.ap.orig_radix[j] = t.radix[j];
      }
    }
  }

  tm.mark("types");
  // ---- schedules + derived tables
  std::vector<int4> mtab_all;
  int64_t bp_bytes = 0, scratch_bytes = 0;
  for (TypeExec& te : P->types) {
    if (te.empty) continue;
    const HostType& t = T[te.id];
    const auto& r = t.radix_c;
    std::vector<int> fold;
    int din_max = 1;
    for (int x : te.trans) {
      for (int j : X[x].xdst) fold.push_back(j);
      din_max = std::max(din_max, X[x].Din);
    }
    Schedule sc = plan_schedule(t, fold, (int)te.trans.size(), ctx->sms, din_max, ctx->force_nb, ctx->force_o_m,
                                ctx->force_p);
    if (sc.cost >= 1e299) return fail(CFP_ETOOBIG, "no enumeration schedule for type " + std::to_string(te.id));
    te.P = sc.P;
    te.role = sc.role;
    te.NB = sc.NB;
    const int K = t.K, Pp = sc.P;
    std::vector<int> A(K, 0), B(K, 0), M(K, 0), PR(K, 0);
    for (int d = 0; d < K; ++d) {
      PR[d] = d < Pp;
      M[d] = d >= Pp && sc.role[d] == 1;
      A[d] = d >= Pp && sc.role[d] == 2;
      B[d] = d >= Pp && sc.role[d] == 3;
    }
    auto ca = ctx_of(A, t), cb = ctx_of(B, t);
    // term assignment: 0 K0, 1 X, 2 Y, 3 Z
    struct TermRef { int kind, a, b, db; int64_t off; int dest; };
    std::vector<TermRef> terms;
    for (int j = 0; j < K; ++j) terms.push_back({0, j, j, 0, te.w_off[j], -1});
    for (int e = 0; e < t.E; ++e)
      terms.push_back({1, t.esrc[e], t.edst[e], r[t.edst[e]], te.e_off[e], -1});
    std::vector<int> domX(K, 0), domY(K, 0), ctxZ(K, 0);
    for (int d = 0; d < K; ++d) { domX[d] = A[d] || ca[d]; domY[d] = B[d] || cb[d]; }
    for (auto& tm : terms) {
      bool allP = PR[tm.a] && PR[tm.b];
      bool tA = A[tm.a] || A[tm.b], tB = B[tm.a] || B[tm.b];
      if (allP) tm.dest = 0;
      else if (tA) tm.dest = 1;
      else if (tB) tm.dest = 2;
      else if (domX[tm.a] && domX[tm.b]) tm.dest = 1;
      else if (domY[tm.a] && domY[tm.b]) tm.dest = 2;
      else { tm.dest = 3; ctxZ[tm.a] = 1; ctxZ[tm.b] = 1; }
    }
    // digit lists: prefix ctx (canonical), M ctx (canonical), own (canonical)
    auto digits_of = [&](const std::vector<int>& ctxmask, const std::vector<int>& own) {
      std::vector<int> d;
      for (int i = 0; i < Pp; ++i) if (ctxmask[i] && !own[i]) d.push_back(i);
      for (int i = Pp; i < K; ++i) if (ctxmask[i] && !own[i] && M[i]) d.push_back(i);
      for (int i = Pp; i < K; ++i) if (own[i]) d.push_back(i);
      return d;
    };
    std::vector<int> zero(K, 0);
    std::vector<int> dx = digits_of(ca, A), dy = digits_of(cb, B), dz = digits_of(ctxZ, zero);
    int nA = 0, nBd = 0;
    for (int d = 0; d < K; ++d) { nA += A[d]; nBd += B[d]; }
    int64_t na = 1, nb = 1, nM = 1;
    for (int d = Pp; d < K; ++d) {
      if (A[d]) na *= r[d];
      if (B[d]) nb *= r[d];
      if (M[d]) nM *= r[d];
    }
    if (nM >= INT32_MAX) return fail(CFP_ETOOBIG, "M loop space >= 2^31");
    const int VG = sc.VG, NB = sc.NB;
    const int na_pad = round_up(na, 4);
    const int nb_pad = round_up((int64_t)VG * NB, 4);
    TableSpec sx = make_spec(dx, r, nA, na_pad);
    TableSpec sy = make_spec(dy, r, nBd, nb_pad);
    TableSpec sz = make_spec(dz, r, 0, 1);
    std::vector<int> dk;
    for (int i = 0; i < Pp; ++i) dk.push_back(i);
    TableSpec sk = make_spec(dk, r, 0, 1);
    for (auto& tm : terms) {
      TableSpec* s = tm.dest == 0 ? &sk : tm.dest == 1 ? &sx : tm.dest == 2 ? &sy : &sz;
      const std::vector<int>& dl = tm.dest == 0 ? dk : tm.dest == 1 ? dx : tm.dest == 2 ? dy : dz;
      TRY(add_term(*s, dl, tm.kind, tm.a, tm.b, tm.db, tm.off));
    }
    // derived blob layout (after the compact values)
    int64_t& dc = te.wide ? b.der64 : b.der32;
    auto place = [&](TableSpec& s) {
      s.out_off = dc;                          // relative; rebased after vals are sized
      int64_t n = s.rows * s.row;
      dc += (n + 3) & ~3LL;
      return s.out_off;
    };
    te.xt_off = place(sx);
    te.yt_off = place(sy);
    te.zt_off = place(sz);
    auto& specs = te.wide ? P->hspecs64 : P->hspecs32;
    specs.push_back(sx); specs.push_back(sy); specs.push_back(sz);
    // thread mapping
    EnumParams& ep = te.ep;
    te.k0_off = place(sk);
    specs.push_back(sk);
    ep.P = Pp;
    for (int i = 0; i < Pp; ++i) ep.pre_radix[i] = r[i];
    int lmin = Pp;
    for (int i = 0; i < Pp; ++i)
      if (ca[i] || cb[i] || ctxZ[i]) { lmin = i; break; }
    ep.W = prod(r, lmin, Pp);
    te.H = prod(r, 0, Pp) / ep.W;
    int64_t h0, h1;
    TRY(cfp_shard_range(te.H, 1, world, rank, &h0, &h1));
    ep.h0 = h0;
    ep.G = h1 - h0;
    ep.Gpad = (ep.G + kBlock - 1) / kBlock * kBlock;
    ep.VG = VG;
    te.nPl = ep.G * ep.W;
    te.combos_local = te.combos * (double)te.nPl / (double)prod(r, 0, Pp);
    for (int i = 0; i < Pp; ++i) {
      auto pos = [&](const std::vector<int>& dl, int d) {
        return (int)(std::find(dl.begin(), dl.end(), d) - dl.begin());
      };
      int px = pos(dx, i), py = pos(dy, i), pz = pos(dz, i);
      ep.pre_sx[i] = px < (int)dx.size() ? stride_in(sx, px) : 0;
      ep.pre_sy[i] = py < (int)dy.size() ? stride_in(sy, py) : 0;
      ep.pre_sz[i] = pz < (int)dz.size() ? stride_in(sz, pz) : 0;
    }
    // mtab over the M digits (canonical order)
    std::vector<int> md;
    for (int i = Pp; i < K; ++i) if (M[i]) md.push_back(i);
    te.mtab_off = (int64_t)mtab_all.size();
    int64_t xspan_m = 0, yspan_m = 0, zspan_m = 0;
    for (int64_t m = 0; m < nM; ++m) {
      int64_t q = m;
      int4 e{0, 0, 0, 0};
      int64_t xo = 0, yo = 0, zo = 0;
      for (int k = (int)md.size() - 1; k >= 0; --k) {
        int d = md[k];
        int dig = (int)(q % r[d]);
        q /= r[d];
        auto pos = [&](const std::vector<int>& dl) {
          return (int)(std::find(dl.begin(), dl.end(), d) - dl.begin());
        };
        int px = pos(dx), py = pos(dy), pz = pos(dz);
        if (px < (int)dx.size()) xo += dig * stride_in(sx, px);
        if (py < (int)dy.size()) yo += dig * stride_in(sy, py);
        if (pz < (int)dz.size()) zo += dig * stride_in(sz, pz);
        if (d == t.o) e.w = dig;
      }
      if (xo > INT32_MAX || yo > INT32_MAX || zo > INT32_MAX)
        return fail(CFP_ETOOBIG, "derived table too large");
      e.x = (int)xo; e.y = (int)yo; e.z = (int)zo;
      xspan_m = std::max(xspan_m, xo);
      yspan_m = std::max(yspan_m, yo);
      zspan_m = std::max(zspan_m, zo);
      mtab_all.push_back(e);
    }
    ep.nM = nM;
    ep.na = (int)na;
    ep.na_pad = na_pad;
    ep.nb = (int)nb;
    ep.nb_pad = nb_pad;
    ep.Do = r[t.o];
    if (t.o < Pp) { ep.o_mode = 2; ep.o_pre = t.o; }
    else if (M[t.o]) { ep.o_mode = 1; ep.o_pre = -1; }
    else {
      ep.o_mode = 0; ep.o_pre = -1;
      // stride of o inside the B row (canonical order of B digits)
      int64_t st = 1;
      for (int i = K - 1; i > t.o; --i) if (B[i]) st *= r[i];
      ep.o_bstride = (int)st;
      ep.o_bradix = r[t.o];
    }
    ep.xspan = xspan_m + sx.row;
    ep.yspan = yspan_m + sy.row;
    ep.zspan = zspan_m + 1;
    // slices are contiguous because prefix ctx digits are the most significant
    const size_t vbytes = te.wide ? 8 : 4;
    size_t smem = (size_t)(ep.xspan + ep.yspan + ((ep.zspan + 3) & ~3LL)) * vbytes + (size_t)nM * 16;
    ep.staged = smem <= 160 * 1024;
    {
      // merged Y'[m][j] = Y + Z rows: in place when the slice's Y rows are
      // exactly the M values in order (Y depends on every M digit: C3, C4),
      // else a second region
      bool inplace = ep.yspan == nM * ep.nb_pad;
      for (int64_t m = 0; inplace && m < nM; ++m) inplace = mtab_all[te.mtab_off + m].y == m * ep.nb_pad;
      const size_t ymb = inplace ? 0 : (size_t)nM * ep.nb_pad * vbytes;
      ep.ymerge = ep.staged && ymb <= 64 * 1024 && smem + ymb <= 160 * 1024;
      ep.ym_inplace = ep.ymerge && inplace && !ctx->no_ym_inplace;
      if (ep.ymerge && !ep.ym_inplace) smem += (size_t)nM * ep.nb_pad * vbytes;
    }
    ep.init_row = ep.o_mode != 0 || !(ep.o_bstride == 1 && ep.o_bradix == ep.nb);
    // M split (B = {o}): two threads per prefix halve the work unit, so the
    // CTAs of a launch fill the last wave of 148 x 4 slots twice as finely.
    // It doubles the CTAs' fixed costs (staging, fold epilogue), so it pays
    // only for long M loops (measured: C4 nM = 529 10.35 -> 10.21 ms; C3/C5
    // nM = 24/23 0.69 -> 0.75 ms)
    ep.MS = (!ep.init_row && ep.o_mode == 0 && nM >= ctx->msplit_min_m && ep.staged && ep.ymerge) ? 2 : 1;
    ep.CH = kBlock / ep.MS;
    ep.no_full_a = ctx->no_full_a ? 1 : 0;
    ep.one = 1;
    ep.mix = 0;
    if (ctx->enum_mix) ep.mix = (int32_t)ctx->enum_mix;
    ep.Gpad = (ep.G + ep.CH - 1) / ep.CH * ep.CH;
    te.smem = ep.staged ? smem : 0;
    te.nthreads = ep.Gpad * ep.W * ep.VG * ep.MS;
    if (te.nthreads / kBlock > 0x7FFFFFFF) return fail(CFP_ETOOBIG, "grid too large");
    te.bp_off = bp_bytes;
    bp_bytes += ((te.nPl * ep.Do * vbytes) + 255) & ~255LL;
    for (int i = 0; i < Pp; ++i) ep.pre_stride[i] = prod(r, i + 1, Pp);
    ep.nchunks = ep.W * (ep.Gpad / ep.CH);
    // eval spec for argmin recovery
    EvalSpec& es = te.es;
    es.K = K;
    for (int d = 0; d < K; ++d) es.radix[d] = r[d];
    es.P = Pp;
    es.o = t.o;
    es.nsuffix = prod(r, Pp, K);
    {
      int64_t lo = INT64_MAX, hi = 0;
      for (int j = 0; j < K; ++j) { lo = std::min<int64_t>(lo, te.w_off[j]); hi = std::max<int64_t>(hi, te.w_off[j] + r[j]); }
      for (int e2 = 0; e2 < t.E; ++e2) {
        lo = std::min<int64_t>(lo, te.e_off[e2]);
        hi = std::max<int64_t>(hi, te.e_off[e2] + (int64_t)r[t.esrc[e2]] * r[t.edst[e2]]);
      }
      if ((hi - lo) * (int64_t)vbytes > 160 * 1024) return fail(CFP_ETOOBIG, "segment tables too large");
      es.tab_lo = lo;
      es.tab_n = (int32_t)(hi - lo);
    }
    for (int d = 0; d < K; ++d)
      if (r[d] > 65535) return fail(CFP_ETOOBIG, "more than 65535 feasible strategies for one block");
    for (auto& tm : terms) {
      if (es.nterm >= kMaxTerms) return fail(CFP_ETOOBIG, "too many terms");
      Term x{};
      x.kind = tm.kind; x.a = tm.a; x.b = tm.b; x.db = tm.db; x.off = tm.off;
      es.term[es.nterm++] = x;
    }
    // fold / argmin per incoming transition
    for (int x : te.trans) {
      TransExec& tx = P->trans[trans_slot[x]];
      FoldParams& f = tx.fp;
      f.P = Pp;
      for (int i = 0; i < Pp; ++i) {
        f.pre_radix[i] = r[i];
        f.pre_stride[i] = prod(r, i + 1, Pp);
      }
      f.p_lo = ep.h0 * ep.W;
      f.nPl = te.nPl;
      f.Din = tx.Din;
      f.Do = ep.Do;
      for (int q = 0; q < X[x].X; ++q) {
        if (f.nq >= kMaxCross) return fail(CFP_ETOOBIG, "more than 16 cross edges in one transition");
        Term tq{};
        tq.kind = 2; tq.a = X[x].xdst[q]; tq.db = r[X[x].xdst[q]]; tq.off = tx.q_off[q];
        f.q[f.nq++] = tq;
      }
      f.qelems = 0;
      for (int q = 0; q < f.nq; ++q) f.qelems += f.Din * f.q[q].db;
      f.tma = ((int64_t)f.Do * (int64_t)vbytes) % 16 == 0 ? 1 : 0;
      tx.ap.e = es;
      tx.ap.Do_orig = tx.Do_orig;
    }
    // cross-term fold in the enumeration epilogue: one chunk = one CTA
    {
      const bool simple = ep.o_mode == 0 && ep.o_bstride == 1 && ep.o_bradix == ep.nb;
      const int64_t VP = simple ? ((te.NB + 3) & ~3) : ((ep.Do + 3) & ~3);   // = the kernel's VP bound
      int64_t dinp_max = 4;
      for (int x : te.trans) dinp_max = std::max<int64_t>(dinp_max, (P->trans[trans_slot[x]].Din + 3) & ~3);
      // [B_p rows CH x VP (over the staged tables) | cross rows CH x DinP |
      // fold minima DinP x VP]
      ep.xs_off = (int32_t)(ep.CH * VP);
      ep.dinp_max = (int32_t)dinp_max;
      const int64_t epi = ep.xs_off + ep.CH * dinp_max + dinp_max * VP;
      ep.smem_epi = (int32_t)(te.trans.empty() ? 0 : epi * (int64_t)vbytes);
      if (ep.smem_epi > 200 * 1024) return fail(CFP_ETOOBIG, "D_in x D_o too large for the fold epilogue");
      ep.ntau = (int)te.trans.size();
      te.epi_off = (int)P->epi_host.size();
      for (int x : te.trans) {
        TransExec& tx = P->trans[trans_slot[x]];
        EpiTau et{};
        et.Din = tx.Din;
        et.nq = tx.fp.nq;
        for (int q = 0; q < tx.fp.nq; ++q) {
          et.q[q] = tx.fp.q[q];
          et.qt[q] = tx.qt_off[q];
        }
        P->epi_host.push_back(et);
        tx.fp.CH = ep.CH;
        tx.fp.nchunks = ep.nchunks;
        tx.fp.W = ep.W;
        tx.fp.G = ep.G;
        tx.fp.h0 = ep.h0;
        tx.fp.nhb = ep.Gpad / ep.CH;
        tx.chunk_off = scratch_bytes;
        scratch_bytes += ((ep.nchunks * tx.fp.Din * tx.fp.Do * vbytes) + 255) & ~255LL;
        tx.aval_off = scratch_bytes;
        scratch_bytes += ((int64_t)tx.fp.Din * tx.fp.Do * 8 + 255) & ~255LL;
        tx.pstar_off = scratch_bytes;
        scratch_bytes += ((int64_t)tx.fp.Din * tx.fp.Do * 8 + 255) & ~255LL;
      }
    }
  }
  tm.mark("schedules");
  // ---- device allocation + H2D
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(P->raw.alloc(b.raw.size() * 4));
  CUDA_TRY(cudaMemcpyAsync(P->raw.p, b.raw.data(), b.raw.size() * 4, cudaMemcpyHostToDevice, st));
  // vmap per transition = keep list of output block; stored in maps blob
  for (TransExec& tx : P->trans) {
    const HostType& t = T[tx.type];
    if (t.empty) continue;
    int off = b.put_map(t.keep[t.o]);
    tx.ap.vmap = reinterpret_cast<const int32_t*>((intptr_t)off);   // rebased below
    std::vector<int> inv(t.radix[t.o], -1);
    for (size_t c = 0; c < t.keep[t.o].size(); ++c) inv[t.keep[t.o][c]] = (int)c;
    int ioff = b.put_map(inv);
    tx.ap.vinv = reinterpret_cast<const int32_t*>((intptr_t)ioff);
  }
  CUDA_TRY(P->maps.alloc(std::max<size_t>(1, b.maps.size()) * 4));
  CUDA_TRY(cudaMemcpyAsync(P->maps.p, b.maps.data(), b.maps.size() * 4, cudaMemcpyHostToDevice, st));
  const int64_t v32 = (b.vals32 + 3) & ~3LL, v64 = (b.vals64 + 3) & ~3LL;
  CUDA_TRY(P->vals32.alloc((size_t)(v32 + b.der32) * 4));
  CUDA_TRY(P->vals64.alloc((size_t)(v64 + b.der64) * 8));
  for (auto& s : P->hspecs32) {
    s.out_off += v32;
    s.block0 = P->spec_max32;
    s.nblocks = std::max<int64_t>(1, (s.rows * s.row + kBuildChunk - 1) / kBuildChunk);
    P->spec_max32 += s.nblocks;                       // total CTAs of the build launch
  }
  for (auto& s : P->hspecs64) {
    s.out_off += v64;
    s.block0 = P->spec_max64;
    s.nblocks = std::max<int64_t>(1, (s.rows * s.row + kBuildChunk - 1) / kBuildChunk);
    P->spec_max64 += s.nblocks;
  }
  // epilogue transition descriptors (chunkmin pointers patched below)
  CUDA_TRY(P->epi.alloc(std::max<size_t>(1, P->epi_host.size()) * sizeof(EpiTau)));
  P->njobs32 = (int)P->hjobs32.size();
  P->njobs64 = (int)P->hjobs64.size();
  P->nspecs32 = (int)P->hspecs32.size();
  P->nspecs64 = (int)P->hspecs64.size();
  CUDA_TRY(P->jobs32.alloc(std::max<size_t>(1, P->hjobs32.size()) * sizeof(CompactJob)));
  CUDA_TRY(P->jobs64.alloc(std::max<size_t>(1, P->hjobs64.size()) * sizeof(CompactJob)));
  CUDA_TRY(P->specs32.alloc(std::max<size_t>(1, P->hspecs32.size()) * sizeof(TableSpec)));
  CUDA_TRY(P->specs64.alloc(std::max<size_t>(1, P->hspecs64.size()) * sizeof(TableSpec)));
  if (!P->hjobs32.empty())
    CUDA_TRY(cudaMemcpyAsync(P->jobs32.p, P->hjobs32.data(), P->hjobs32.size() * sizeof(CompactJob), cudaMemcpyHostToDevice, st));
  if (!P->hjobs64.empty())
    CUDA_TRY(cudaMemcpyAsync(P->jobs64.p, P->hjobs64.data(), P->hjobs64.size() * sizeof(CompactJob), cudaMemcpyHostToDevice, st));
  if (!P->hspecs32.empty())
    CUDA_TRY(cudaMemcpyAsync(P->specs32.p, P->hspecs32.data(), P->hspecs32.size() * sizeof(TableSpec), cudaMemcpyHostToDevice, st));
  if (!P->hspecs64.empty())
    CUDA_TRY(cudaMemcpyAsync(P->specs64.p, P->hspecs64.data(), P->hspecs64.size() * sizeof(TableSpec), cudaMemcpyHostToDevice, st));
  CUDA_TRY(P->mtab.alloc(std::max<size_t>(1, mtab_all.size()) * sizeof(int4)));
  if (!mtab_all.empty())
    CUDA_TRY(cudaMemcpyAsync(P->mtab.p, mtab_all.data(), mtab_all.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(P->bp.alloc((size_t)std::max<int64_t>(bp_bytes, 256)));
  CUDA_TRY(P->scratch.alloc((size_t)std::max<int64_t>(scratch_bytes, 256)));
  // A/I outputs for every used transition
  int64_t ai = 0;
  for (TransExec& tx : P->trans) { tx.out_off = ai; ai += (int64_t)tx.Din * tx.Do_orig; }
  CUDA_TRY(P->outAI.alloc((size_t)ai * 16 + 16));
  CUDA_TRY(P->merge_keys.alloc((size_t)ai * 8 + 16));
  CUDA_TRY(P->locAI.alloc((size_t)ai * 16 + 16));            // rank-local (A, I) before the merge
  CUDA_TRY(P->edges.alloc((size_t)(ai + 1) * sizeof(ArgminEntry) + (size_t)(ai + 1) * 4 + 16));
  P->ai = ai;
  uint64_t* outA = P->outAI.as<uint64_t>();
  uint64_t* outI = outA + ai;
  uint64_t* argA = ctx->sharded ? P->locAI.as<uint64_t>() : outA;
  uint64_t* argI = ctx->sharded ? P->locAI.as<uint64_t>() + ai : outI;
  // rebase pointers
  for (TypeExec& te : P->types) {
    if (te.empty) continue;
    const int64_t base = te.wide ? v64 : v32;
    const size_t vb = te.wide ? 8 : 4;
    char* vals = te.wide ? (char*)P->vals64.p : (char*)P->vals32.p;
    EnumParams& ep = te.ep;
    ep.XT = vals + (base + te.xt_off) * vb;
    ep.YT = vals + (base + te.yt_off) * vb;
    ep.ZT = vals + (base + te.zt_off) * vb;
    ep.K0 = vals + (base + te.k0_off) * vb;
    ep.mtab = P->mtab.as<int4>() + te.mtab_off;
    ep.Bp = (char*)P->bp.p + te.bp_off;
    for (int x : te.trans) {
      TransExec& tx = P->trans[trans_slot[x]];
      tx.fp.Bp = ep.Bp;
      tx.fp.vals = vals;
      tx.fp.chunkmin = (char*)P->scratch.p + tx.chunk_off;
      tx.ap.f = tx.fp;
      tx.ap.maps = P->maps.as<int32_t>();
      tx.ap.vmap = P->maps.as<int32_t>() + (intptr_t)tx.ap.vmap;
      tx.ap.vinv = P->maps.as<int32_t>() + (intptr_t)tx.ap.vinv;
      tx.ap.A_out = argA + tx.out_off;
      tx.ap.I_out = argI + tx.out_off;
      tx.ap.A_glob = outA + tx.out_off;
      tx.ap.wide = te.wide ? 1 : 0;
      tx.ap.slot = trans_slot[x];
      tx.ap.pstar = reinterpret_cast<int64_t*>((char*)P->scratch.p + tx.pstar_off);
    }
    for (size_t q = 0; q < te.trans.size(); ++q)
      P->epi_host[te.epi_off + q].chunkmin = P->trans[trans_slot[te.trans[q]]].fp.chunkmin;
    ep.taus = P->epi.as<EpiTau>() + te.epi_off;
    ep.vals = vals;
  }
  for (size_t q = 0; q < P->trans.size(); ++q) {   // outputs of every transition, empty types included
    TransExec& tx = P->trans[q];
    tx.ap.A_out = argA + tx.out_off;
    tx.ap.I_out = argI + tx.out_off;
    tx.ap.A_glob = outA + tx.out_off;
    tx.ap.slot = (int)q;
    tx.ap.Do_orig = tx.Do_orig;
  }
  {
    // device copies of the per-transition argmin descriptors + bucket offsets
    std::vector<ArgminParams> aps(P->trans.size());
    std::vector<int64_t> poff(P->trans.size() + 1, 0);
    for (size_t q = 0; q < P->trans.size(); ++q) {
      TransExec& tx = P->trans[q];
      aps[q] = tx.ap;
      const TypeExec& te = P->types[type_slot[tx.type]];
      const bool live = !te.empty && te.nPl > 0;
      if (!live) aps[q].f.nchunks = 0;
      poff[q + 1] = poff[q] + (live ? (int64_t)tx.fp.Din * tx.fp.Do : 0);
      P->has32 |= live && !te.wide;
      P->has64 |= live && te.wide;
      P->kmax_arg = std::max(P->kmax_arg, te.K);
      P->tabn_max = std::max(P->tabn_max, (int)te.es.tab_n);
    }
    P->npairs = poff.back();
    CUDA_TRY(P->aps.alloc(std::max<size_t>(1, aps.size()) * sizeof(ArgminParams)));
    CUDA_TRY(P->pair_off.alloc(poff.size() * 8));
    if (!aps.empty())
      CUDA_TRY(cudaMemcpyAsync(P->aps.p, aps.data(), aps.size() * sizeof(ArgminParams), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(P->pair_off.p, poff.data(), poff.size() * 8, cudaMemcpyHostToDevice, st));
  }
  if (!P->epi_host.empty())
    CUDA_TRY(cudaMemcpyAsync(P->epi.p, P->epi_host.data(), P->epi_host.size() * sizeof(EpiTau),
                             cudaMemcpyHostToDevice, st));
  for (TransExec& tx : P->trans) {
    const TypeExec& te = P->types[type_slot[tx.type]];
    P->evals += te.combos * (double)tx.Din;          // (combination, input state) costs minimised over
  }
  for (TypeExec& te : P->types) {
    P->combos += te.combos;
    P->combos_local += te.combos_local;
  }
  tm.mark("alloc+h2d");
  // ---- chain setup
  if (do_chain) {
    const int N = P->N;
    std::vector<ChainInst> ci(N);
    std::vector<int32_t> radix_blob;
    std::vector<int64_t> goff(N + 2);
    int kmax = 1;
    goff[0] = 0;
    for (int n = 0; n < N; ++n) {
      const TransExec& tx = P->trans[trans_slot[P->inst[n]]];
      const HostType& t = T[tx.type];
      ci[n].A = outA + tx.out_off;
      ci[n].I = outI + tx.out_off;
      ci[n].mat = trans_slot[P->inst[n]];
      ci[n].rows = tx.Din;
      ci[n].cols = tx.Do_orig;
      ci[n].K = t.K;
      ci[n].radix_off = (int)radix_blob.size();
      radix_blob.insert(radix_blob.end(), t.radix.begin(), t.radix.end());
      kmax = std::max(kmax, t.K);
      P->inst_rows.push_back(tx.Din);
      P->inst_cols.push_back(tx.Do_orig);
    }
    goff[1] = ci[0].rows;
    for (int n = 1; n <= N; ++n) goff[n + 1] = goff[n] + ci[n - 1].cols;
    std::vector<ChainRun> runs;
    int64_t pow_need = 0;
    for (int n = 0; n < N;) {
      int m = n + 1;
      while (m < N && P->inst[m] == P->inst[n] && ci[n].rows == ci[n].cols) ++m;
      runs.push_back({n, m - n});
      if (m - n > 1) {
        int levels = 0;
        while ((1 << (levels + 1)) <= m - n) ++levels;
        pow_need = std::max<int64_t>(pow_need, (int64_t)ci[n].rows * ci[n].rows * levels);
      }
      n = m;
    }
    P->kmax = kmax;
    P->nruns = (int)runs.size();
    CUDA_TRY(P->chain_inst.alloc(N * sizeof(ChainInst)));
    CUDA_TRY(cudaMemcpyAsync(P->chain_inst.p, ci.data(), N * sizeof(ChainInst), cudaMemcpyHostToDevice, st));
    CUDA_TRY(P->chain_runs.alloc(runs.size() * sizeof(ChainRun)));
    CUDA_TRY(cudaMemcpyAsync(P->chain_runs.p, runs.data(), runs.size() * sizeof(ChainRun), cudaMemcpyHostToDevice, st));
    CUDA_TRY(P->chain_goff.alloc((N + 2) * sizeof(int64_t)));
    CUDA_TRY(cudaMemcpyAsync(P->chain_goff.p, goff.data(), (N + 2) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(P->chain_G.alloc((size_t)goff[N + 1] * 8));
    CUDA_TRY(P->chain_pow.alloc((size_t)std::max<int64_t>(pow_need, 1) * 8));
    CUDA_TRY(P->radix_blob.alloc(radix_blob.size() * 4));
    CUDA_TRY(cudaMemcpyAsync(P->radix_blob.p, radix_blob.data(), radix_blob.size() * 4, cudaMemcpyHostToDevice, st));
    // plan: total, seg_index[N], seg_ns[N], digits[N*kmax], status
    // plan: total, seg_index[N], seg_ns[N], digits[N*kmax], then the status word
    P->plan_bytes = 8 + (size_t)N * 16 + (size_t)N * kmax * 4;
    CUDA_TRY(P->plan.alloc(P->plan_bytes + 16));
    ChainParams& cp = P->cp;
    cp.N = N;
    cp.nruns = P->nruns;
    cp.inst = P->chain_inst.as<ChainInst>();
    cp.runs = P->chain_runs.as<ChainRun>();
    cp.terminal = nullptr;
    cp.G = P->chain_G.as<uint64_t>();
    cp.goff = P->chain_goff.as<int64_t>();
    cp.powers = P->chain_pow.as<uint64_t>();
    cp.powers_cap = std::max<int64_t>(pow_need, 1);
    cp.backtrack = 1;
    char* pl = (char*)P->plan.p;
    cp.total = reinterpret_cast<uint64_t*>(pl);
    cp.seg_index = reinterpret_cast<uint64_t*>(pl + 8);
    cp.seg_ns = reinterpret_cast<uint64_t*>(pl + 8 + (size_t)N * 8);
    cp.digits = reinterpret_cast<int32_t*>(pl + 8 + (size_t)N * 16);
    cp.kmax = kmax;
    cp.radix_blob = P->radix_blob.as<int32_t>();
    cp.status = reinterpret_cast<int32_t*>(pl + P->plan_bytes);
    {
      std::vector<ChainInst> mats(P->trans.size());
      int lv = 0, smax = 1;
      for (size_t q = 0; q < P->trans.size(); ++q) {
        const TransExec& tx = P->trans[q];
        mats[q] = ChainInst{outA + tx.out_off, outI + tx.out_off, (int)q, tx.Din, tx.Do_orig, 0, 0};
        smax = std::max(smax, std::max(tx.Din, tx.Do_orig));
      }
      for (auto& r : runs) {
        int levels = 0;
        while ((1 << (levels + 1)) <= r.len) ++levels;
        if (r.len > 1) lv = std::max(lv, levels);
      }
      TRY(setup_chain_staging(cp, mats, goff[N + 1], lv, smax, P->chain_mats, P->chain_moff, st));
      // argmin only on optimal edges reachable from the chain start (<= 256 states)
      P->use_edges = smax <= 256;
      cp.edge_list = P->edges.as<ArgminEntry>();
      cp.edge_count = reinterpret_cast<int32_t*>(P->edges.as<char>() + (size_t)(P->ai + 1) * sizeof(ArgminEntry));
      cp.edge_flag = reinterpret_cast<int32_t*>(P->merge_keys.p);      // ai ints, zeroed per execute
      CUDA_TRY(P->reach.alloc((size_t)goff[N] + 16));
      cp.reach = P->reach.as<uint8_t>();
      P->reach_bytes = goff[N];
    }
  }
  // ---- fused tail (world 1): bucket minima, chain, argmin, backtrack in one launch
  int chain_levels = 0, chain_smax = 1;
  if (do_chain) {
    for (const TransExec& tx : P->trans) chain_smax = std::max(chain_smax, std::max(tx.Din, tx.Do_orig));
    for (int n = 0; n < P->N;) {                     // runs as the chain setup forms them
      int m = n + 1;
      while (m < P->N && P->inst[m] == P->inst[n] && P->inst_rows[n] == P->inst_cols[n]) ++m;
      int levels = 0;
      while ((1 << (levels + 1)) <= m - n) ++levels;
      if (m - n > 1) chain_levels = std::max(chain_levels, levels);
      n = m;
    }
  }
  if (ctx->fused_tail && !ctx->sharded && P->trans.size() <= 32 &&
      (!do_chain || (P->use_edges && chain_smax <= 32))) {
    // worker CTAs: digit scratch [K][threads] u16, descriptor copies, every slot's W/R tables
    auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
    size_t off = al((size_t)P->kmax_arg * kTailThreads * 2);
    const size_t desc_off = off;
    off = al(off + P->trans.size() * sizeof(ArgminParams));
    std::vector<int64_t> tab_off(P->trans.size(), 0);
    for (size_t q = 0; q < P->trans.size(); ++q) {
      const TypeExec& te = P->types[type_slot[P->trans[q].type]];
      tab_off[q] = (int64_t)off;
      off = al(off + (size_t)te.es.tab_n * (te.wide ? 8 : 4));
    }
    size_t smem = off;
    if (do_chain) {
      const FusedChainLayout L(P->cp.mat_elems, P->inst_rows[0] + [&] {
        int64_t c = 0;
        for (int n = 0; n < P->N; ++n) c += P->inst_cols[n];
        return c;
      }(), [&] {
        int64_t r = 0;
        for (int n = 0; n < P->N; ++n) r += P->inst_rows[n];
        return r;
      }(), P->N, P->cp.nmat, chain_levels, chain_smax);
      smem = std::max(smem, (size_t)L.bytes);
    }
    int optin = 0, per_sm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    if (smem + 40 * 1024 <= (size_t)optin) CUDA_TRY(tail_max_blocks(smem, &per_sm));
    if (per_sm >= 1 && ctx->sms >= 2) {              // co-resident CTAs (cooperative launch)
      std::vector<int64_t> oo(P->trans.size() + 1, 0);
      for (size_t q = 0; q < P->trans.size(); ++q)
        oo[q + 1] = oo[q] + (int64_t)P->trans[q].Din * P->trans[q].Do_orig;
      CUDA_TRY(P->orig_off.alloc(oo.size() * 8));
      CUDA_TRY(cudaMemcpyAsync(P->orig_off.p, oo.data(), oo.size() * 8, cudaMemcpyHostToDevice, st));
      CUDA_TRY(P->tail_sync.alloc(16));
      CUDA_TRY(cudaMemsetAsync(P->tail_sync.p, 0, 16, st));
      CUDA_TRY(P->phase_ts.alloc(8 * 8));
      TailParams& tp = P->tp;
      tp.aps = P->aps.as<ArgminParams>();
      tp.pair_off = P->pair_off.as<int64_t>();
      tp.orig_off = P->orig_off.as<int64_t>();
      tp.nslot = (int)P->trans.size();
      tp.chain = do_chain ? 1 : 0;
      if (do_chain) tp.cp = P->cp;
      tp.sync = P->tail_sync.as<unsigned int>();
      tp.phase_ts = nullptr;
      tp.squaring = ctx->tail_squaring ? 1 : 0;
      tp.levels = chain_levels;
      tp.smax = chain_smax;
      tp.kmax_arg = P->kmax_arg;
      tp.arg_desc_off = (int64_t)desc_off;
      for (size_t q = 0; q < P->trans.size(); ++q) tp.arg_tab_off[q] = tab_off[q];
      const int64_t warps = oo.back();                // phase 1: a warp per bucket
      const int64_t wpc = kTailThreads / 32;
      int64_t g = do_chain ? std::max<int64_t>(8, (warps + wpc - 1) / wpc + 1) : std::max<int64_t>(1, P->npairs);
      g = std::max<int64_t>(2, std::min<int64_t>(g, (int64_t)ctx->sms * per_sm));
      P->tail_grid = (int)g;
      P->tail_per_sm = per_sm;
      P->tail_smem = smem;
      P->fused_tail = true;
    }
  }
  tm.mark("chain");
  CUDA_TRY(cudaStreamSynchronize(st));
  tm.mark("sync");
  *out = P.release();
  return CFP_OK;
}

// ---------------------------------------------------------------- execute
template <typename V> constexpr V VTcap();
template <> constexpr uint32_t VTcap<uint32_t>() { return kCap32; }
template <> constexpr uint64_t VTcap<uint64_t>() { return kCap64; }

template <typename V>
static cfp_status run_type_kernels(cfp_prepared* P, TypeExec& te, cudaStream_t st, bool first_of_prec) {
  (void)first_of_prec;
  static const bool dbg = getenv("CFP_DEBUG_ENUM") != nullptr;
  if (dbg) {
    const EnumParams& e = te.ep;
    fprintf(stderr, "enum: P=%d W=%lld G=%lld NB=%d VG=%d nM=%lld na=%d nb=%d staged=%d ymerge=%d MS=%d "
            "CH=%d full_a=%d ntau=%d smem=%zu epi=%d\n", e.P, (long long)e.W, (long long)e.G, te.NB, e.VG,
            (long long)e.nM, e.na, e.nb, e.staged, e.ymerge, e.MS, e.CH,
            (int)(sizeof(V) == 4 && e.MS == 1 && e.staged && e.ymerge && e.na == te.NB &&
                  (te.NB == 23 || te.NB == 24) && !e.no_full_a),
            e.ntau, te.smem, e.smem_epi);
  }
  CUDA_TRY(launch_enum<V>(te.ep, te.NB, te.nthreads, te.smem, st));
  P->launches += 1;
  return CFP_OK;
}

static cfp_status merge_ranks(cfp_prepared* P, cudaStream_t st);

// all_tables: every bucket's least index (as cfp_segment_costs) instead of the
// chain + backtrack -- cfp_prepared_tables reads the tables of the exact
// schedule / kernels a search runs
static cfp_status execute_impl(cfp_ctx* ctx, cfp_prepared* P, bool all_tables = false) {
  CUDA_TRY(cudaSetDevice(ctx->device));
  NvtxRange nv("cfp_execute");
  cudaStream_t st = ctx->stream;
  P->launches = 0;
  if (P->timing) {
    for (auto& e : P->ev) if (!e) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(P->ev[0], st));
  }
  auto phase = [&](int i) -> cudaError_t {
    return P->timing >= 2 ? cudaEventRecord(P->ev[i], st) : cudaSuccess;
  };
  // a0: compaction + derived tables
  if (P->njobs32) {
    CUDA_TRY(launch_compact<uint32_t>(P->jobs32.as<CompactJob>(), P->njobs32, P->raw.as<uint32_t>(),
                                      P->maps.as<int32_t>(), P->vals32.as<uint32_t>(), st));
    P->launches++;
  }
  if (P->njobs64) {
    CUDA_TRY(launch_compact<uint64_t>(P->jobs64.as<CompactJob>(), P->njobs64, P->raw.as<uint32_t>(),
                                      P->maps.as<int32_t>(), P->vals64.as<uint64_t>(), st));
    P->launches++;
  }
  if (P->nspecs32) {
    CUDA_TRY(launch_build_tables<uint32_t>(P->specs32.as<TableSpec>(), P->nspecs32, P->spec_max32,
                                           P->vals32.as<uint32_t>(), P->vals32.as<uint32_t>(), st));
    P->launches++;
  }
  if (P->nspecs64) {
    CUDA_TRY(launch_build_tables<uint64_t>(P->specs64.as<TableSpec>(), P->nspecs64, P->spec_max64,
                                           P->vals64.as<uint64_t>(), P->vals64.as<uint64_t>(), st));
    P->launches++;
  }
  // a1: enumeration per type (largest first), then fold + argmin per transition
  if (P->timing) CUDA_TRY(cudaEventRecord(P->ev[1], st));
  {
    // types (largest first) round-robin over the caller's stream and the side
    // lanes; they write disjoint scratch (own B_p, own transitions' chunks)
    int nlive = 0;
    for (TypeExec& te : P->types) nlive += !(te.empty || te.nPl == 0);
    const int nl = std::min(nlive, cfp_ctx::kLanes + 1);
    if (nl > 1) {
      CUDA_TRY(cudaEventRecord(ctx->fork, st));
      for (int i = 0; i + 1 < nl; ++i) CUDA_TRY(cudaStreamWaitEvent(ctx->lane[i], ctx->fork, 0));
    }
    int k = 0;
    for (TypeExec& te : P->types) {
      if (te.empty || te.nPl == 0) continue;
      cudaStream_t ls = (k % nl) == 0 ? st : ctx->lane[(k % nl) - 1];
      ++k;
      if (te.wide) TRY(run_type_kernels<uint64_t>(P, te, ls, false));
      else TRY(run_type_kernels<uint32_t>(P, te, ls, false));
    }
    for (int i = 0; i + 1 < nl; ++i) {
      CUDA_TRY(cudaEventRecord(ctx->join[i], ctx->lane[i]));
      CUDA_TRY(cudaStreamWaitEvent(st, ctx->join[i], 0));
    }
  }
  if (P->timing) CUDA_TRY(cudaEventRecord(P->ev[2], st));
  if (P->fused_tail) {
    TailParams tp = P->tp;
    tp.phase_ts = P->timing >= 2 ? P->phase_ts.as<uint64_t>() : nullptr;
    int grid = P->tail_grid;
    if (all_tables && tp.chain) {
      tp.chain = 0;
      tp.phase_ts = nullptr;
      grid = (int)std::max<int64_t>(2, std::min<int64_t>(P->npairs, (int64_t)ctx->sms * P->tail_per_sm));
    }
    CUDA_TRY(launch_tail(tp, grid, P->tail_smem, st));
    P->launches++;
    CUDA_TRY(phase(4));
    CUDA_TRY(phase(5));
    CUDA_TRY(phase(6));
    if (P->timing) CUDA_TRY(cudaEventRecord(P->ev[3], st));
    return CFP_OK;
  }
  uint64_t* outA = P->outAI.as<uint64_t>();
  const int64_t ai = P->ai;
  // outputs default to (INF, NOIDX): covers pruned output strategies, empty types
  CUDA_TRY(launch_fill<uint64_t>(outA, ai * 2, kInf64, st));
  P->launches++;
  if (ctx->sharded) {
    CUDA_TRY(launch_fill<uint64_t>(P->locAI.as<uint64_t>(), ai * 2, kInf64, st));
    P->launches++;
  }
  const ArgminParams* aps = P->aps.as<ArgminParams>();
  const int nslot = (int)P->trans.size();
  // a1: bucket minima A (values)
  if (P->has32) { CUDA_TRY(launch_amin<uint32_t>(aps, P->pair_off.as<int64_t>(), nslot, P->npairs, st)); P->launches++; }
  if (P->has64) { CUDA_TRY(launch_amin<uint64_t>(aps, P->pair_off.as<int64_t>(), nslot, P->npairs, st)); P->launches++; }
  if (ctx->sharded) {
    // rank-local minima were written to locA by the argmin descriptors; amin wrote
    // them there too -- reduce into the global A (shard simulation: the local A)
    if (ctx->comm) NCCL_TRY(ncclAllReduce(P->locAI.p, outA, ai, ncclUint64, ncclMin, ctx->comm, st));
    else CUDA_TRY(cudaMemcpyAsync(outA, P->locAI.p, (size_t)ai * 8, cudaMemcpyDeviceToDevice, st));
  }
  CUDA_TRY(phase(4));
  ArgminEntry* list = P->edges.as<ArgminEntry>();
  int32_t* count = reinterpret_cast<int32_t*>(P->edges.as<char>() + (size_t)(ai + 1) * sizeof(ArgminEntry));
  const bool edges = P->do_chain && P->use_edges && !all_tables;
  if (edges) {
    // a3: suffix vectors + the optimal edges reachable from the chain start
    CUDA_TRY(cudaMemsetAsync(P->cp.status, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(count, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(P->merge_keys.p, 0, (size_t)ai * 4, st));
    CUDA_TRY(cudaMemsetAsync(P->reach.p, 0, (size_t)P->reach_bytes, st));
    ChainParams c1 = P->cp;
    c1.mode = 1;
    CUDA_TRY(launch_chain(c1, st));
    CUDA_TRY(launch_edges_to_pairs(aps, list, count, ai, st));
    P->launches += 2;
  } else {
    CUDA_TRY(launch_all_pairs(P->pair_off.as<int64_t>(), nslot, P->npairs, list, count, st));
    P->launches++;
  }
  CUDA_TRY(phase(5));
  // a1: least combination index of the listed buckets
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(edges ? 64 : P->npairs, P->npairs));
  if (P->has32) { CUDA_TRY(launch_argmin<uint32_t>(aps, list, count, grid, P->kmax_arg, P->tabn_max, st)); P->launches++; }
  if (P->has64) { CUDA_TRY(launch_argmin<uint64_t>(aps, list, count, grid, P->kmax_arg, P->tabn_max, st)); P->launches++; }
  // a2: merge across ranks
  if (ctx->sharded) TRY(merge_ranks(P, st));
  CUDA_TRY(phase(6));
  // a4 (+ a3 when the edge list is not used)
  if (P->do_chain && !all_tables) {
    if (!edges) CUDA_TRY(cudaMemsetAsync(P->cp.status, 0, 4, st));
    ChainParams c2 = P->cp;
    c2.mode = edges ? 2 : 0;
    CUDA_TRY(launch_chain(c2, st));
    P->launches++;
  }
  if (P->timing) CUDA_TRY(cudaEventRecord(P->ev[3], st));
  return CFP_OK;
}

// Rank merge: packed keys (cost << b | idx) when they fit, else two rounds.
__global__ void pack_kernel(const uint64_t* A, const uint64_t* I, int64_t n, int bits, uint64_t* keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = A[i] == kInf64 ? kInf64 : ((A[i] << bits) | I[i]);
}
__global__ void unpack_kernel(const uint64_t* keys, int64_t n, int bits, uint64_t* A, uint64_t* I) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (keys[i] == kInf64) { A[i] = kInf64; I[i] = kInf64; return; }
  A[i] = keys[i] >> bits;
  I[i] = keys[i] & ((1ull << bits) - 1);
}
__global__ void mask_idx_kernel(const uint64_t* A, const uint64_t* Amin, const uint64_t* I, int64_t n,
                                uint64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (A[i] == Amin[i]) ? I[i] : kInf64;
}

static cfp_status merge_ranks(cfp_prepared* P, cudaStream_t st) {
  // (cost, index) lexicographic min over ranks of the rank-local argmins:
  // round 1 min cost (already the global A in outA), round 2 min index among
  // ranks attaining it.
  cfp_ctx* ctx = P->ctx;
  const int64_t ai = P->ai;
  uint64_t* A = P->outAI.as<uint64_t>();
  uint64_t* I = A + ai;
  const uint64_t* locA = P->locAI.as<uint64_t>();
  const uint64_t* locI = locA + ai;
  const unsigned nb = (unsigned)((ai + 255) / 256);
  mask_idx_kernel<<<nb, 256, 0, st>>>(locA, A, locI, ai, I);
  CUDA_TRY(cudaGetLastError());
  if (ctx->comm) NCCL_TRY(ncclAllReduce(I, I, ai, ncclUint64, ncclMin, ctx->comm, st));
  P->launches += 1;
  return CFP_OK;
}

// ---------------------------------------------------------------- fetch
static cfp_status fetch_impl(cfp_ctx* ctx, cfp_prepared* P, cfp_plan* out) {
  NvtxRange nv("cfp_fetch_plan");
  cudaStream_t st = ctx->stream;
  const int N = P->N;
  // plan + status word in one copy, through the ctx's pinned staging buffer
  const size_t nb = P->plan_bytes + 4;
  TRY(ctx_pinned(ctx, nb));
  CUDA_TRY(cudaMemcpyAsync(ctx->pinned, P->plan.p, nb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const char* buf = static_cast<const char*>(ctx->pinned);
  int32_t status = 0;
  memcpy(&status, buf + P->plan_bytes, 4);
  if (status == 4) return fail(CFP_ETOOBIG, "chain scratch too small");
  if (status == 3) {
    // diagnostic: forward reachability over finite entries of A_n
    int64_t ai = 0;
    for (TransExec& tx : P->trans) ai += (int64_t)tx.Din * tx.Do_orig;
    std::vector<uint64_t> A(ai);
    CUDA_TRY(cudaMemcpy(A.data(), P->outAI.p, ai * 8, cudaMemcpyDeviceToHost));
    std::vector<char> reach(1, 1);
    int bad = N;
    for (int n = 0; n < N; ++n) {
      const TransExec* tx = nullptr;
      for (auto& t : P->trans) if (t.id == P->inst[n]) tx = &t;
      std::vector<char> nx(tx->Do_orig, 0);
      bool any = false;
      for (int u = 0; u < tx->Din && u < (int)reach.size(); ++u)
        if (reach[u])
          for (int v = 0; v < tx->Do_orig; ++v)
            if (A[tx->out_off + (int64_t)u * tx->Do_orig + v] != kInf64) { nx[v] = 1; any = true; }
      if (!any) { bad = n; break; }
      reach.swap(nx);
    }
    return fail(CFP_EINFEASIBLE, "no feasible plan: instance " + std::to_string(bad) +
                                     " has no finite strategy combination reachable from the chain start");
  }
  if (!out) return CFP_OK;
  if (out->kmax < P->kmax) return fail(CFP_EINVAL, "plan.kmax smaller than the largest K");
  memcpy(&out->total_ns, buf, 8);
  if (out->seg_index) memcpy(out->seg_index, buf + 8, (size_t)N * 8);
  if (out->seg_ns) memcpy(out->seg_ns, buf + 8 + (size_t)N * 8, (size_t)N * 8);
  if (out->digits) {
    const int32_t* d = reinterpret_cast<const int32_t*>(buf + 8 + (size_t)N * 16);
    for (int n = 0; n < N; ++n)
      for (int j = 0; j < out->kmax; ++j)
        out->digits[(int64_t)n * out->kmax + j] = j < P->kmax ? d[(int64_t)n * P->kmax + j] : -1;
  }
  return CFP_OK;
}

// ---------------------------------------------------------------- public API
extern "C" cfp_status cfp_prepare(cfp_ctx* ctx, const cfp_problem* p, cfp_prepared** out) {
  if (!ctx || !out) return fail(CFP_EINVAL, "null argument");
  if (ctx->sim) return fail(CFP_EINVAL, "shard simulation ctx (world > 1 without nccl_unique_id): tables only");
  return prepare_impl(ctx, p, true, out);
}

extern "C" cfp_status cfp_execute(cfp_ctx* ctx, cfp_prepared* prep) {
  if (!ctx || !prep) return fail(CFP_EINVAL, "null argument");
  return execute_impl(ctx, prep);
}

extern "C" cfp_status cfp_fetch_plan(cfp_ctx* ctx, cfp_prepared* prep, cfp_plan* out) {
  if (!ctx || !prep) return fail(CFP_EINVAL, "null argument");
  return fetch_impl(ctx, prep, out);
}

extern "C" cfp_status cfp_search_plan(cfp_ctx* ctx, const cfp_problem* p, cfp_plan* out) {
  if (!ctx || !p || !out) return fail(CFP_EINVAL, "null argument");
  if (ctx->sim) return fail(CFP_EINVAL, "shard simulation ctx (world > 1 without nccl_unique_id): tables only");
  NvtxRange nv("cfp_search_plan");
  std::vector<int64_t> key;
  HostModel model;
  model.b.raw.swap(ctx->raw_pool);
  model.b.raw.clear();
  struct PoolBack {
    cfp_ctx* c; Builder& b;
    ~PoolBack() { c->raw_pool.swap(b.raw); }
  } pool_back{ctx, model.b};
  static const bool dbg = getenv("CFP_DEBUG_E2E") != nullptr;
  PrepTimer tm;
  TRY(build_model(ctx, p, true, model));
  if (dbg) tm.mark("build_model");
  if (ctx->plan_cache) {
    // the same structure as the last call: reuse its prepared plan (schedule,
    // device buffers, chain setup) and upload only this call's values
    key = plan_key(p, model.T, model.X, model.inst, model.b);
    if (dbg) tm.mark("plan_key");
    if (ctx->cached && key == ctx->cached_key) {
      TRY(check_chain_overflow(model.T, model.X, model.inst));
      CUDA_TRY(cudaSetDevice(ctx->device));
      g_alloc_stream = ctx->stream;
      cfp_prepared* P = ctx->cached;
      const size_t nb = model.b.raw.size() * 4;      // this call's values, via pinned staging
      TRY(ctx_pinned(ctx, nb));
      memcpy(ctx->pinned, model.b.raw.data(), nb);
      CUDA_TRY(cudaMemcpyAsync(P->raw.p, ctx->pinned, nb, cudaMemcpyHostToDevice, ctx->stream));
      if (dbg) tm.mark("h2d_submit");
      TRY(execute_impl(ctx, P));
      if (dbg) tm.mark("execute_submit");
      cfp_status st = fetch_impl(ctx, P, out);
      if (dbg) tm.mark("fetch");
      return st;
    }
  }
  // structure changed: release the previous plan's device buffers first, so a
  // search that fits the device alone never needs old + new plan at once
  if (ctx->cached) {
    cfp_prepared_free(ctx->cached);
    ctx->cached = nullptr;
    ctx->cached_key.clear();
  }
  cfp_prepared* prep = nullptr;
  TRY(prepare_impl(ctx, p, true, &prep, &model));
  std::unique_ptr<cfp_prepared> guard(prep);
  TRY(execute_impl(ctx, prep));
  TRY(fetch_impl(ctx, prep, out));
  if (ctx->plan_cache) {
    ctx->cached = guard.release();
    ctx->cached_key = std::move(key);
  }
  return CFP_OK;
}

extern "C" cfp_status cfp_prepared_tables(cfp_ctx* ctx, cfp_prepared* P, int32_t transition, uint64_t* cost_out,
                                          uint64_t* index_out) {
  if (!ctx || !P || !cost_out || !index_out) return fail(CFP_EINVAL, "null argument");
  const TransExec* tx = nullptr;
  if (transition >= 0 && transition < (int)P->canon.size()) transition = P->canon[transition];
  for (const TransExec& t : P->trans) if (t.id == transition) tx = &t;
  if (!tx) return fail(CFP_EINVAL, "transition " + std::to_string(transition) +
                                       " is not used by the instance list (or was merged with an identical one)");
  TRY(execute_impl(ctx, P, true));
  const int64_t n = (int64_t)tx->Din * tx->Do_orig;
  CUDA_TRY(cudaMemcpyAsync(cost_out, P->outAI.as<uint64_t>() + tx->out_off, n * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(index_out, P->outAI.as<uint64_t>() + P->ai + tx->out_off, n * 8,
                           cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CFP_OK;
}

extern "C" cfp_status cfp_prepared_query(const cfp_prepared* P, cfp_prepared_info* info) {
  if (!P || !info) return fail(CFP_EINVAL, "null argument");
  memset(info, 0, sizeof(*info));
  info->combos = P->combos;
  info->combos_local = P->combos_local;
  info->evals = P->evals;
  info->num_types = (int)P->types.size();
  info->num_transitions = (int)P->trans.size();
  info->kernel_launches = P->launches;
  info->fused_tail = P->fused_tail ? 1 : 0;
  info->tail_grid = P->tail_grid;
  for (size_t i = 0; i < P->types.size() && i < CFP_MAX_BLOCKS; ++i) {
    info->wide_types += P->types[i].wide;
    info->prefix_len[i] = P->types[i].P;
    info->nb[i] = P->types[i].NB * 100 + P->types[i].ep.VG;
    info->na[i] = P->types[i].ep.na;
    const EnumParams& e = P->types[i].ep;
    info->o_mode[i] = e.o_mode;
    info->full_a[i] = (!P->types[i].wide && e.MS == 1 && e.staged && e.ymerge && e.na == P->types[i].NB &&
                       (P->types[i].NB == 23 || P->types[i].NB == 24) && !e.no_full_a &&
                       e.na_pad >= (P->types[i].NB + 3) / 4 * 4) ? 1 : 0;
  }
  return CFP_OK;
}

extern "C" cfp_status cfp_prepared_time_kernels(cfp_prepared* P, int32_t on) {
  if (!P) return fail(CFP_EINVAL, "null argument");
  if (on < 0 || on > 2) return fail(CFP_EINVAL, "timing level must be 0, 1 or 2");
  P->timing = on;
  return CFP_OK;
}

extern "C" cfp_status cfp_prepared_phase_ms(cfp_prepared* P, double* ms) {
  if (!P || !ms) return fail(CFP_EINVAL, "null argument");
  if (P->timing < 2 || !P->ev[6]) return fail(CFP_EINVAL, "phase timing (level 2) not enabled");
  CUDA_TRY(cudaEventSynchronize(P->ev[3]));
  const int from[6] = {0, 1, 2, 4, 5, 6}, to[6] = {1, 2, 4, 5, 6, 3};
  for (int i = 0; i < 6; ++i) {
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, P->ev[from[i]], P->ev[to[i]]));
    ms[i] = t;
  }
  if (P->fused_tail && P->tp.chain) {
    // one launch: split its event time by CTA 0's %globaltimer marks (phase
    // boundaries: start, bucket minima done, chain done, argmins done, end)
    uint64_t t[5];
    CUDA_TRY(cudaMemcpy(t, P->phase_ts.p, sizeof(t), cudaMemcpyDeviceToHost));
    const double tail = ms[2];
    const double tot = (double)(t[4] - t[0]);
    const double f[4] = {(double)(t[1] - t[0]), (double)(t[2] - t[1]), (double)(t[3] - t[2]), (double)(t[4] - t[3])};
    for (int i = 0; i < 4; ++i) ms[2 + i] = tot > 0 ? tail * f[i] / tot : 0.0;
  }
  return CFP_OK;
}

extern "C" cfp_status cfp_prepared_kernel_ms(cfp_prepared* P, double* enum_ms, double* total_ms) {
  if (!P || !P->timing || !P->ev[0]) return fail(CFP_EINVAL, "timing not enabled");
  CUDA_TRY(cudaEventSynchronize(P->ev[3]));
  float a = 0, b = 0;
  CUDA_TRY(cudaEventElapsedTime(&a, P->ev[1], P->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&b, P->ev[0], P->ev[3]));
  if (enum_ms) *enum_ms = a;
  if (total_ms) *total_ms = b;
  return CFP_OK;
}

extern "C" cfp_status cfp_segment_costs(cfp_ctx* ctx, const cfp_segment_type* t, const cfp_transition* tr,
                                        int32_t d_in, uint64_t* cost_out, uint64_t* index_out) {
  if (!ctx || !t || !cost_out || !index_out) return fail(CFP_EINVAL, "null argument");
  if (d_in < 1) return fail(CFP_EINVAL, "d_in < 1");
  if (!tr && d_in != 1) return fail(CFP_EINVAL, "tr == NULL requires d_in == 1");
  // problem = [type, pred stub with one block of d_in strategies]
  cfp_segment_type types[2];
  types[0] = *t;
  std::vector<int32_t> stub_radix{d_in};
  std::vector<uint32_t> stub_comp(d_in, 0);
  types[1] = cfp_segment_type{1, stub_radix.data(), stub_comp.data(), nullptr, 0, nullptr, nullptr, nullptr, 0};
  cfp_transition x{};
  if (tr) {
    x = *tr;
    x.type = 0;
    x.pred_type = 1;
  } else {
    x = cfp_transition{-1, 0, 0, nullptr, nullptr};
  }
  int32_t inst = 0;
  cfp_problem p{};
  p.abi_version = CFP_ABI_VERSION;
  p.num_types = 2;
  p.types = types;
  p.num_transitions = 1;
  p.transitions = &x;
  p.num_instances = 1;
  p.inst_transition = &inst;
  cfp_prepared* prep = nullptr;
  cfp_status s;
  s = prepare_impl(ctx, &p, false, &prep);
  if (s != CFP_OK) return s;
  std::unique_ptr<cfp_prepared> guard(prep);
  TRY(execute_impl(ctx, prep));
  const TransExec& tx = prep->trans[0];
  const int64_t n = (int64_t)tx.Din * tx.Do_orig;
  int64_t ai = n;
  CUDA_TRY(cudaMemcpyAsync(cost_out, prep->outAI.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(index_out, prep->outAI.as<uint64_t>() + ai, n * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CFP_OK;
}

// ---------------------------------------------------------------- chain API
// Large-S chain (shared-memory staging impossible): repeated squaring with the
// tiled (min,+) kernel, doubling stages as batched matrix-vector launches.
static cfp_status chain_large(const std::vector<ChainInst>& ci, const std::vector<ChainRun>& runs,
                              const std::vector<int64_t>& goff, uint64_t* G, bool narrow, cudaStream_t st) {
  int64_t maxS2 = 1, maxL = 1;
  for (const ChainRun& r : runs) {
    maxS2 = std::max<int64_t>(maxS2, (int64_t)ci[r.first].rows * ci[r.first].cols);
    maxL = std::max<int64_t>(maxL, r.len);
  }
  int levels_max = 0;
  while ((1ll << (levels_max + 1)) <= maxL) ++levels_max;
  DevBuf pw, pa, pc, offs;
  CUDA_TRY(pw.alloc((size_t)std::max(1, levels_max) * maxS2 * 8));
  CUDA_TRY(pa.alloc((size_t)maxS2 * 8));
  CUDA_TRY(pc.alloc((size_t)maxS2 * 8));
  CUDA_TRY(offs.alloc((size_t)(2 * maxL + 2) * 8));
  std::vector<int64_t> ho(2 * maxL + 2);
  auto batch = [&](const uint64_t* P, int R, int C, const std::vector<std::pair<int64_t, int64_t>>& sd) -> cfp_status {
    const int nv = (int)sd.size();
    for (int i = 0; i < nv; ++i) { ho[i] = sd[i].first; ho[maxL + 1 + i] = sd[i].second; }
    CUDA_TRY(cudaMemcpyAsync(offs.p, ho.data(), ho.size() * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));     // host vector is reused by the next batch
    CUDA_TRY(launch_matvec_batch(P, R, C, G, offs.as<int64_t>(), offs.as<int64_t>() + maxL + 1, G, nv, st));
    return CFP_OK;
  };
  for (int r = (int)runs.size() - 1; r >= 0; --r) {
    const ChainRun run = runs[r];
    const ChainInst& in = ci[run.first];
    const int e = run.first + run.len;
    if (run.len == 1) {
      TRY(batch(in.A, in.rows, in.cols, {{goff[e], goff[e - 1]}}));
      continue;
    }
    const int S = in.rows;
    int levels = 0;
    while ((1 << (levels + 1)) <= run.len) ++levels;
    const int64_t S2 = (int64_t)S * S;
    for (int j = 1; j <= levels; ++j) {
      const uint64_t* src = j == 1 ? in.A : pw.as<uint64_t>() + (j - 2) * S2;
      uint64_t* dst = pw.as<uint64_t>() + (j - 1) * S2;
      if (narrow) {
        CUDA_TRY(launch_to_path<uint32_t>(src, pa.as<uint32_t>(), S2, st));
        CUDA_TRY(launch_minplus_tiled<uint32_t>(S, S, S, pa.as<uint32_t>(), pa.as<uint32_t>(), pc.as<uint32_t>(),
                                                nullptr, st));
        CUDA_TRY(launch_from_path<uint32_t>(pc.as<uint32_t>(), nullptr, dst, nullptr, S2, st));
      } else {
        CUDA_TRY(launch_to_path<uint64_t>(src, pa.as<uint64_t>(), S2, st));
        CUDA_TRY(launch_minplus_tiled<uint64_t>(S, S, S, pa.as<uint64_t>(), pa.as<uint64_t>(), pc.as<uint64_t>(),
                                                nullptr, st));
        CUDA_TRY(launch_from_path<uint64_t>(pc.as<uint64_t>(), nullptr, dst, nullptr, S2, st));
      }
    }
    for (int j = 0; j <= levels; ++j) {
      const uint64_t* Pj = j == 0 ? in.A : pw.as<uint64_t>() + (j - 1) * S2;
      const int k_lo = 1 << j, k_hi = std::min(1 << (j + 1), run.len + 1);
      std::vector<std::pair<int64_t, int64_t>> sd;
      for (int k = k_lo; k < k_hi; ++k) sd.push_back({goff[e - k + (1 << j)], goff[e - k]});
      TRY(batch(Pj, S, S, sd));
    }
  }
  return CFP_OK;
}

extern "C" cfp_status cfp_minplus_chain(cfp_ctx* ctx, int32_t num_mats, const int32_t* rows,
                                        const int32_t* cols, const uint64_t* const* mats,
                                        int32_t num_runs, const int32_t* run_mat, const int64_t* run_len,
                                        const uint64_t* terminal, uint64_t* opt_out, uint64_t* suffix_out) {
  if (!ctx || num_mats < 1 || !rows || !cols || !mats || num_runs < 1 || !run_mat || !run_len || !opt_out)
    return fail(CFP_EINVAL, "bad chain arguments");
  for (int m = 0; m < num_mats; ++m)
    if (rows[m] < 1 || cols[m] < 1 || !mats[m]) return fail(CFP_EINVAL, "bad matrix " + std::to_string(m));
  int64_t N = 0;
  for (int r = 0; r < num_runs; ++r) {
    if (run_mat[r] < 0 || run_mat[r] >= num_mats || run_len[r] < 1)
      return fail(CFP_EINVAL, "bad run " + std::to_string(r));
    if (run_len[r] > 1 && rows[run_mat[r]] != cols[run_mat[r]])
      return fail(CFP_EINVAL, "run " + std::to_string(r) + " repeats a non-square matrix");
    if (r > 0 && rows[run_mat[r]] != cols[run_mat[r - 1]])
      return fail(CFP_EINVAL, "run " + std::to_string(r) + " does not chain");
    N += run_len[r];
  }
  if (N > (1 << 26)) return fail(CFP_ETOOBIG, "chain too long");
  long double chain_bound = 0;
  // overflow guard: sum of per-instance maximum finite entries < 2^63
  {
    long double tot = 0;
    for (int r = 0; r < num_runs; ++r) {
      const int m = run_mat[r];
      uint64_t mx = 0;
      for (int64_t i = 0; i < (int64_t)rows[m] * cols[m]; ++i)
        if (mats[m][i] != CFP_INF64) mx = std::max(mx, mats[m][i]);
      tot += (long double)mx * run_len[r];
    }
    if (terminal)
      for (int v = 0; v < cols[run_mat[num_runs - 1]]; ++v)
        if (terminal[v] != CFP_INF64) tot += terminal[v];
    if (tot >= 9.2e18L) return fail(CFP_EOVERFLOW, "a finite chain cost could reach 2^63");
    chain_bound = tot;
  }
  g_alloc_stream = ctx->stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf dm, dinst, druns, dgoff, dG, dpow, dterm, dstatus;
  std::vector<int64_t> moff(num_mats + 1, 0);
  for (int m = 0; m < num_mats; ++m) moff[m + 1] = moff[m] + (int64_t)rows[m] * cols[m];
  CUDA_TRY(dm.alloc(moff[num_mats] * 8));
  for (int m = 0; m < num_mats; ++m)
    CUDA_TRY(cudaMemcpyAsync(dm.as<uint64_t>() + moff[m], mats[m], (size_t)(moff[m + 1] - moff[m]) * 8,
                             cudaMemcpyHostToDevice, st));
  std::vector<ChainInst> ci;
  std::vector<ChainRun> runs;
  int64_t pow_need = 1;
  int maxS = 0;
  for (int r = 0; r < num_runs; ++r) {
    const int m = run_mat[r];
    runs.push_back({(int)ci.size(), (int)run_len[r]});
    for (int64_t k = 0; k < run_len[r]; ++k)
      ci.push_back({dm.as<uint64_t>() + moff[m], nullptr, m, rows[m], cols[m], 0, 0});
    if (run_len[r] > 1) {
      int levels = 0;
      while ((1ll << (levels + 1)) <= run_len[r]) ++levels;
      pow_need = std::max<int64_t>(pow_need, (int64_t)rows[m] * rows[m] * levels);
    }
    maxS = std::max(maxS, std::max(rows[m], cols[m]));
  }
  std::vector<int64_t> goff(N + 2);
  goff[0] = 0;
  goff[1] = ci[0].rows;
  for (int64_t n = 1; n <= N; ++n) goff[n + 1] = goff[n] + ci[n - 1].cols;
  CUDA_TRY(dinst.alloc(ci.size() * sizeof(ChainInst)));
  CUDA_TRY(cudaMemcpyAsync(dinst.p, ci.data(), ci.size() * sizeof(ChainInst), cudaMemcpyHostToDevice, st));
  CUDA_TRY(druns.alloc(runs.size() * sizeof(ChainRun)));
  CUDA_TRY(cudaMemcpyAsync(druns.p, runs.data(), runs.size() * sizeof(ChainRun), cudaMemcpyHostToDevice, st));
  CUDA_TRY(dgoff.alloc((N + 2) * 8));
  CUDA_TRY(cudaMemcpyAsync(dgoff.p, goff.data(), (N + 2) * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(dG.alloc(goff[N + 1] * 8));
  CUDA_TRY(dpow.alloc(pow_need * 8));
  CUDA_TRY(dstatus.alloc(16));
  CUDA_TRY(cudaMemsetAsync(dstatus.p, 0, 4, st));
  if (terminal) {
    CUDA_TRY(dterm.alloc((size_t)ci.back().cols * 8));
    CUDA_TRY(cudaMemcpyAsync(dterm.p, terminal, (size_t)ci.back().cols * 8, cudaMemcpyHostToDevice, st));
  }
  ChainParams cp{};
  cp.N = (int)N;
  cp.nruns = num_runs;
  cp.inst = dinst.as<ChainInst>();
  cp.runs = druns.as<ChainRun>();
  cp.terminal = terminal ? dterm.as<uint64_t>() : nullptr;
  cp.G = dG.as<uint64_t>();
  cp.goff = dgoff.as<int64_t>();
  cp.powers = dpow.as<uint64_t>();
  cp.powers_cap = pow_need;
  cp.backtrack = 0;
  cp.status = dstatus.as<int32_t>();
  DevBuf dmats, dmoff;
  {
    std::vector<ChainInst> umats(num_mats);
    int lv = 0;
    for (int m = 0; m < num_mats; ++m)
      umats[m] = ChainInst{dm.as<uint64_t>() + moff[m], nullptr, m, rows[m], cols[m], 0, 0};
    for (int r = 0; r < num_runs; ++r) {
      int levels = 0;
      while ((1ll << (levels + 1)) <= run_len[r]) ++levels;
      if (run_len[r] > 1) lv = std::max(lv, levels);
    }
    TRY(setup_chain_staging(cp, umats, goff[N + 1], lv, maxS, dmats, dmoff, st));
  }
  if (cp.smem_bytes == 0 && maxS > 64) {
    if (terminal)
      CUDA_TRY(cudaMemcpyAsync(dG.as<uint64_t>() + goff[N], terminal, (size_t)ci.back().cols * 8,
                               cudaMemcpyHostToDevice, st));
    else
      CUDA_TRY(cudaMemsetAsync(dG.as<uint64_t>() + goff[N], 0, (size_t)ci.back().cols * 8, st));
    TRY(chain_large(ci, runs, goff, dG.as<uint64_t>(), chain_bound < (long double)kCap32, st));
  } else {
    CUDA_TRY(launch_chain(cp, st));
  }
  int32_t status = 0;
  CUDA_TRY(cudaMemcpyAsync(&status, dstatus.p, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(opt_out, dG.p, 8, cudaMemcpyDeviceToHost, st));
  if (suffix_out)
    CUDA_TRY(cudaMemcpyAsync(suffix_out, dG.p, goff[N + 1] * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (status == 4) return fail(CFP_ETOOBIG, "chain scratch too small");
  return CFP_OK;
}

// Narrow (uint32, VIADDMNMX) when every finite a + b < 2^31 - 1, else uint64.
extern "C" cfp_status cfp_minplus_product(cfp_ctx* ctx, int32_t m, int32_t k, int32_t n, const uint64_t* A,
                                          const uint64_t* B, uint64_t* C, uint64_t* argk) {
  if (!ctx || m < 1 || k < 1 || n < 1 || !A || !B || !C) return fail(CFP_EINVAL, "bad product arguments");
  uint64_t ma = 0, mb = 0;
  for (int64_t i = 0; i < (int64_t)m * k; ++i) if (A[i] != CFP_INF64) ma = std::max(ma, A[i]);
  for (int64_t i = 0; i < (int64_t)k * n; ++i) if (B[i] != CFP_INF64) mb = std::max(mb, B[i]);
  if ((long double)ma + mb >= (long double)kCap64) return fail(CFP_EOVERFLOW, "a finite sum could reach 2^63");
  const bool narrow = (long double)ma + mb < (long double)kCap32;
  g_alloc_stream = ctx->stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t vb = narrow ? 4 : 8;
  DevBuf dA, dB, dC, dK, dA8, dB8, dC8, dK8;
  CUDA_TRY(dA8.alloc((size_t)m * k * 8));
  CUDA_TRY(dB8.alloc((size_t)k * n * 8));
  CUDA_TRY(dC8.alloc((size_t)m * n * 8));
  CUDA_TRY(dK8.alloc((size_t)m * n * 8));
  CUDA_TRY(dA.alloc((size_t)m * k * vb));
  CUDA_TRY(dB.alloc((size_t)k * n * vb));
  CUDA_TRY(dC.alloc((size_t)m * n * vb));
  CUDA_TRY(dK.alloc((size_t)m * n * 4));
  CUDA_TRY(cudaMemcpyAsync(dA8.p, A, (size_t)m * k * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dB8.p, B, (size_t)k * n * 8, cudaMemcpyHostToDevice, st));
  uint32_t* kp = argk ? dK.as<uint32_t>() : nullptr;
  if (narrow) {
    CUDA_TRY(launch_to_path<uint32_t>(dA8.as<uint64_t>(), dA.as<uint32_t>(), (int64_t)m * k, st));
    CUDA_TRY(launch_to_path<uint32_t>(dB8.as<uint64_t>(), dB.as<uint32_t>(), (int64_t)k * n, st));
    CUDA_TRY(launch_minplus_tiled<uint32_t>(m, k, n, dA.as<uint32_t>(), dB.as<uint32_t>(), dC.as<uint32_t>(), kp, st));
    CUDA_TRY(launch_from_path<uint32_t>(dC.as<uint32_t>(), kp, dC8.as<uint64_t>(), argk ? dK8.as<uint64_t>() : nullptr,
                                        (int64_t)m * n, st));
  } else {
    CUDA_TRY(launch_to_path<uint64_t>(dA8.as<uint64_t>(), dA.as<uint64_t>(), (int64_t)m * k, st));
    CUDA_TRY(launch_to_path<uint64_t>(dB8.as<uint64_t>(), dB.as<uint64_t>(), (int64_t)k * n, st));
    CUDA_TRY(launch_minplus_tiled<uint64_t>(m, k, n, dA.as<uint64_t>(), dB.as<uint64_t>(), dC.as<uint64_t>(), kp, st));
    CUDA_TRY(launch_from_path<uint64_t>(dC.as<uint64_t>(), kp, dC8.as<uint64_t>(), argk ? dK8.as<uint64_t>() : nullptr,
                                        (int64_t)m * n, st));
  }
  CUDA_TRY(cudaMemcpyAsync(C, dC8.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost, st));
  if (argk) CUDA_TRY(cudaMemcpyAsync(argk, dK8.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return CFP_OK;
}

// Device-resident (min,+) product microbenchmark: S x S x S,
// hash-generated operands < 2^20, `iters` timed launches after one warm-up.
extern "C" cfp_status cfp_minplus_bench(cfp_ctx* ctx, int32_t S, int32_t wide, int32_t with_argk, int32_t iters,
                                        double* ms_per_launch, double* addmins_per_s) {
  if (!ctx || S < 1 || S > 65536 || iters < 1) return fail(CFP_EINVAL, "bad minplus bench arguments");
  g_alloc_stream = ctx->stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t vb = wide ? 8 : 4;
  const int64_t n2 = (int64_t)S * S;
  DevBuf dA, dB, dC, dK;
  CUDA_TRY(dA.alloc(n2 * vb));
  CUDA_TRY(dB.alloc(n2 * vb));
  CUDA_TRY(dC.alloc(n2 * vb));
  CUDA_TRY(dK.alloc(with_argk ? n2 * 4 : 16));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  uint32_t* kp = with_argk ? dK.as<uint32_t>() : nullptr;
  auto run = [&]() -> cudaError_t {
    if (wide) return launch_minplus_tiled<uint64_t>(S, S, S, dA.as<uint64_t>(), dB.as<uint64_t>(), dC.as<uint64_t>(), kp, st);
    return launch_minplus_tiled<uint32_t>(S, S, S, dA.as<uint32_t>(), dB.as<uint32_t>(), dC.as<uint32_t>(), kp, st);
  };
  if (wide) {
    CUDA_TRY(launch_fill_random<uint64_t>(dA.as<uint64_t>(), n2, 1, st));
    CUDA_TRY(launch_fill_random<uint64_t>(dB.as<uint64_t>(), n2, 2, st));
  } else {
    CUDA_TRY(launch_fill_random<uint32_t>(dA.as<uint32_t>(), n2, 1, st));
    CUDA_TRY(launch_fill_random<uint32_t>(dB.as<uint32_t>(), n2, 2, st));
  }
  CUDA_TRY(run());
  CUDA_TRY(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) CUDA_TRY(run());
  CUDA_TRY(cudaEventRecord(e1, st));
  CUDA_TRY(cudaEventSynchronize(e1));
  float t = 0;
  CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double per = t / iters;
  if (ms_per_launch) *ms_per_launch = per;
  if (addmins_per_s) *addmins_per_s = (double)S * S * S / (per * 1e-3);
  return CFP_OK;
}

extern "C" cfp_status cfp_intpipe_bench(cfp_ctx* ctx, int32_t op, int32_t iters, double* ops_per_s, double* ms) {
  if (!ctx || op < 0 || op > 3 || iters < 1) return fail(CFP_EINVAL, "bad intpipe arguments");
  g_alloc_stream = ctx->stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf out;
  CUDA_TRY(out.alloc(4096 * 4));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = ctx->sms * 2;
  CUDA_TRY(launch_intpipe(op, blocks, iters, out.as<uint32_t>(), st));   // warm-up
  CUDA_TRY(cudaEventRecord(e0, st));
  CUDA_TRY(launch_intpipe(op, blocks, iters, out.as<uint32_t>(), st));
  CUDA_TRY(cudaEventRecord(e1, st));
  CUDA_TRY(cudaEventSynchronize(e1));
  float t = 0;
  CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // op 3: 2 * blocks CTAs x 256 threads x 576 add+mins per step
  const double ops = op == 3 ? (double)blocks * 2 * 256 * iters * 576 : (double)blocks * 1024 * iters * 64;
  if (ops_per_s) *ops_per_s = ops / (t * 1e-3);
  if (ms) *ms = t;
  return CFP_OK;
}

// memory-constrained search (NEXT-1)
#include "cfp_mem_host.inc"

// dense per-plan tables (NEXT-2)
#include "cfp_dense_host.inc"

// profiling space and dynamic profiling budget (NEXT-3)
#include "cfp_profile_host.inc"

