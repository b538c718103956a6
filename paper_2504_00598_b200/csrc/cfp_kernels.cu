// cfp_kernels.cu -- sm_100a kernels of the CFP plan-search hot path.
//
// Hot path and where each step lives:
//   a0 stage:      compact_kernel (prune + p+c), build_table_kernel (X/Y/Z/K0)
//   a1 enumerate:  enum_kernel -- one fused add+min per strategy combination
//                  (VIADDMNMX, or for 2 of 3 an FMA-pipe IMAD + VIMNMX3); its
//                  epilogue folds the cross-segment terms of every incoming
//                  transition into per-CTA chunk minima
//   a1 reduce:     amin_kernel -- A[u][v] = min over chunk minima
//   a3 chain:      chain_kernel mode 1 -- (min,+) powers by repeated squaring,
//                  suffix vectors by doubling, optimal edges reachable from
//                  the chain start
//   a1 argmin:     argmin_kernel -- least combination index of those buckets
//                  (every bucket for cfp_segment_costs)
//   a2 merge:      NCCL min-allreduce (host side, world > 1)
//   a4 backtrack:  chain_kernel mode 2 -- forward greedy + plan decode
// Everything is exact integer arithmetic; the narrow path keeps values in
// [0, CAP32] with CAP32 = 2^31-1 meaning "infeasible" (any sum >= CAP is
// infeasible, guaranteed by the host's bound check), so the fused
// add+min never wraps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "cfp_internal.h"

namespace cfp {

// Development-only phase trace of the fused tail (build with -DCFP_TAIL_TRACE;
// compiled out of the library otherwise).
#ifdef CFP_TAIL_TRACE
__device__ uint64_t g_trace[64];
__device__ uint64_t g_trace_cta[256];
__device__ uint64_t g_enum_trace[4096 * 8];     // per CTA of one enum launch: phase marks
#define ETRACE(i)                                                                              \
  do {                                                                                         \
    if (threadIdx.x == 0 && p.ntau > 0 && blockIdx.x < 4096) {                                 \
      uint64_t t_;                                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      g_enum_trace[blockIdx.x * 8 + (i)] = t_;                                                 \
    }                                                                                          \
  } while (0)
#define TTRACE(cta, i)                                                                      \
  do {                                                                                     \
    if (threadIdx.x == 0 && blockIdx.x == (cta)) {                                         \
      uint64_t t_;                                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      g_trace[(i)] = t_;                                                                   \
    }                                                                                      \
  } while (0)
#else
#define TTRACE(cta, i) do { } while (0)
#define ETRACE(i) do { } while (0)
#endif

template <typename V> struct VT;
template <> struct VT<uint32_t> {
  static constexpr uint32_t CAP = kCap32;
  static __device__ __forceinline__ uint32_t addmin(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_u32(a, b, c);          // VIADDMNMX.U32: min(a + b, c)
  }
  static __device__ __forceinline__ uint32_t sat(uint32_t a, uint32_t b) {
    return __viaddmin_u32(a, b, CAP);
  }
  static __device__ __forceinline__ uint32_t mn(uint32_t a, uint32_t b) { return a < b ? a : b; }
};
template <> struct VT<uint64_t> {
  static constexpr uint64_t CAP = kCap64;
  static __device__ __forceinline__ uint64_t addmin(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t s = a + b;
    return s < c ? s : c;
  }
  static __device__ __forceinline__ uint64_t sat(uint64_t a, uint64_t b) {
    uint64_t s = a + b;
    return s < CAP ? s : CAP;
  }
  static __device__ __forceinline__ uint64_t mn(uint64_t a, uint64_t b) { return a < b ? a : b; }
};

// x * one + y as an IMAD on the FMA pipe (one = 1 at run time, so ptxas can
// neither fold it to an ALU IADD3 nor to a VIADDMNMX)
__device__ __forceinline__ uint32_t mad_fma(uint32_t x, uint32_t one, uint32_t y) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(y));
  return r;
}

// --------------------------------------------------------------------------
// TMA 1-D bulk copies (cp.async.bulk, SASS UBLKCP) with mbarrier completion.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// digit at canonical position `pos` of prefix value pg (block 0 most significant)
__device__ __forceinline__ int prefix_digit(int64_t pg, int pos, int P, const int32_t* radix) {
  if (pg < 0x7FFFFFFF) {
    uint32_t q = (uint32_t)pg;
    uint32_t dig = 0;
    for (int d = P - 1; d >= pos; --d) {
      const uint32_t r = (uint32_t)radix[d];
      dig = q % r;
      q /= r;
    }
    return (int)dig;
  }
  int64_t q = pg;
  int dig = 0;
  for (int d = P - 1; d >= pos; --d) {
    dig = (int)(q % radix[d]);
    q /= radix[d];
  }
  return dig;
}

// --------------------------------------------------------------------------
// a0: compaction.  Each job gathers one table of the pruned problem from the
// raw uint32 inputs: unary w = p + c (INF absorbing), pair / cross
// tables with rows/cols remapped to the surviving strategies.  INF -> CAP.
// --------------------------------------------------------------------------


template <typename V>
__global__ void compact_kernel(const CompactJob* __restrict__ jobs, const uint32_t* __restrict__ raw,
                               const int32_t* __restrict__ maps, V* __restrict__ out) {
  const CompactJob j = jobs[blockIdx.x];
  if (j.kind == 3) {                              // transposed cross table Q^T[s][u]
    const int64_t n = (int64_t)j.cols * j.rows_pad;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
      const int32_t c = (int32_t)((uint32_t)e / (uint32_t)j.rows_pad), r = (int32_t)((uint32_t)e % (uint32_t)j.rows_pad);
      V v = VT<V>::CAP;
      if (r < j.rows) {
        const int32_t rc = j.map_c >= 0 ? maps[j.map_c + c] : c;
        const uint32_t x = raw[j.raw_off + (int64_t)r * j.raw_cols + rc];
        v = (x == 0xFFFFFFFFu || (uint64_t)x >= (uint64_t)VT<V>::CAP) ? VT<V>::CAP : (V)x;
      }
      out[j.out_off + e] = v;
    }
    return;
  }
  const int64_t n = (int64_t)j.rows * j.cols;       // tables are small: 32-bit index math
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int32_t r = (int32_t)((uint32_t)e / (uint32_t)j.cols), c = (int32_t)((uint32_t)e % (uint32_t)j.cols);
    const int32_t rc = j.map_c >= 0 ? maps[j.map_c + c] : c;
    V v;
    if (j.kind == 0) {
      const uint32_t pc = raw[j.raw_off + rc];
      const uint32_t cc = j.raw_off2 >= 0 ? raw[j.raw_off2 + rc] : 0u;
      if (pc == 0xFFFFFFFFu || cc == 0xFFFFFFFFu) v = VT<V>::CAP;
      else {
        const uint64_t s = (uint64_t)pc + cc;
        v = s >= (uint64_t)VT<V>::CAP ? VT<V>::CAP : (V)s;
      }
    } else {
      const int32_t rr = (j.kind == 1 && j.map_r >= 0) ? maps[j.map_r + r] : r;
      const uint32_t x = raw[j.raw_off + (int64_t)rr * j.raw_cols + rc];
      v = (x == 0xFFFFFFFFu || (uint64_t)x >= (uint64_t)VT<V>::CAP) ? VT<V>::CAP : (V)x;
    }
    out[j.out_off + e] = v;
  }
}

// --------------------------------------------------------------------------
// a0: derived tables X / Y / Z / K0 -- saturated sums of the cost terms the
// host assigned to each table, over the table's mixed-radix index space.
// --------------------------------------------------------------------------
template <typename V>
__global__ void build_table_kernel(const TableSpec* __restrict__ specs, int nspecs, const V* __restrict__ vals,
                                   V* __restrict__ out) {
  // block -> table: the specs' block ranges tested in parallel (one round trip)
  __shared__ int s_si;
  if (threadIdx.x < 32) {
    int found = -1;
    for (int base = 0; found < 0 && base < nspecs; base += 32) {
      const int i = base + (int)threadIdx.x;
      const bool in = i < nspecs && (int64_t)blockIdx.x >= specs[i].block0 &&
                      (int64_t)blockIdx.x < specs[i].block0 + specs[i].nblocks;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (m) found = base + __ffs(m) - 1;
    }
    if (threadIdx.x == 0) s_si = found;
  }
  __syncthreads();
  const int si = s_si;
  // the spec (radices, term list) in shared memory: the per-entry loop reads
  // it for every term, and a global read per field made that a chain of
  // dependent L1/L2 round trips
  __shared__ __align__(16) TableSpec s;
  {
    const int words = (int)(sizeof(TableSpec) / 4);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(specs + si);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&s);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int64_t total = min(s.rows * s.row, (int64_t)(blockIdx.x - s.block0 + 1) * kBuildChunk);
  __shared__ int32_t sdig[kMaxDigits][256];       // per-thread digits (dynamic index)
  const bool small = total < 0x7FFFFFFF && s.row < 0x7FFFFFFF;
  for (int64_t e = (blockIdx.x - s.block0) * kBuildChunk + threadIdx.x; e < total; e += blockDim.x) {
    int64_t r, c;
    if (small) {
      r = (uint32_t)e / (uint32_t)s.row;
      c = (uint32_t)e - (uint32_t)r * (uint32_t)s.row;
    } else {
      r = e / s.row;
      c = e % s.row;
    }
    V acc = 0;
    if (c >= s.row_valid) {
      acc = VT<V>::CAP;
    } else {
      int32_t* dig = &sdig[0][threadIdx.x];
      const int64_t q0 = r * s.row_valid + c;
      if (q0 < 0x7FFFFFFF) {
        uint32_t q = (uint32_t)q0;
        for (int d = s.ndig - 1; d >= 0; --d) {
          const uint32_t rd = (uint32_t)s.radix[d];
          dig[d * 256] = (int32_t)(q % rd);
          q /= rd;
        }
      } else {
        int64_t q = q0;
        for (int d = s.ndig - 1; d >= 0; --d) {
          dig[d * 256] = (int32_t)(q % s.radix[d]);
          q /= s.radix[d];
        }
      }
      for (int t = 0; t < s.nterm; ++t) {
        const Term& tm = s.term[t];
        const V v = tm.kind == 0 ? vals[tm.off + dig[tm.a * 256]]
                                 : vals[tm.off + (int64_t)dig[tm.a * 256] * tm.db + dig[tm.b * 256]];
        acc = VT<V>::sat(acc, v);
      }
    }
    out[s.out_off + e] = acc;
  }
}

template <typename V>
__global__ void fill_kernel(V* __restrict__ p, int64_t n, V v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// --------------------------------------------------------------------------
// a1: exhaustive enumeration.  Thread = (prefix p, register group vg).  For
// each M value: Y[j] = YT[..][j] + K0[p] + Z (NB registers), then for every A
// value x = XT[..][a] (a warp-uniform shared-memory broadcast) and every
// register slot j:  acc[j] = min(x + Y[j], acc[j])  -- one VIADDMNMX per
// combination (p, m, a, b_j).  acc[j] ends as min over the combination's
// bucket; the per-prefix bucket minima B_p[v] go to global memory.
// --------------------------------------------------------------------------
template <typename V> struct Vec4;
template <> struct Vec4<uint32_t> { using T = uint4; static constexpr int N = 4; };
template <> struct Vec4<uint64_t> { using T = ulonglong2; static constexpr int N = 2; };

template <typename V>
__device__ __forceinline__ void load_vec(const V* p, V* out);
template <>
__device__ __forceinline__ void load_vec<uint32_t>(const uint32_t* p, uint32_t* out) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <>
__device__ __forceinline__ void load_vec<uint64_t>(const uint64_t* p, uint64_t* out) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
  out[0] = v.x; out[1] = v.y;
}
template <typename V>
__device__ __forceinline__ void store_vec(V* p, const V* in);
template <>
__device__ __forceinline__ void store_vec<uint32_t>(uint32_t* p, const uint32_t* in) {
  *reinterpret_cast<uint4*>(p) = make_uint4(in[0], in[1], in[2], in[3]);
}
template <>
__device__ __forceinline__ void store_vec<uint64_t>(uint64_t* p, const uint64_t* in) {
  *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(in[0], in[1]);
}

template <typename V>
__device__ __forceinline__ void atomic_min_v(V* p, V v);
template <>
__device__ __forceinline__ void atomic_min_v<uint32_t>(uint32_t* p, uint32_t v) { atomicMin(p, v); }
template <>
__device__ __forceinline__ void atomic_min_v<uint64_t>(uint64_t* p, uint64_t v) {
  atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// X^t_p[u] = sum_i Q_i[u][s_i(p)] (Eq. 3 r_n) for prefix pg into
// xrow[0, DinP): each term is one contiguous row Q_i^T[s_i(p)][0..DinP) of the
// transposed copy, read 16 bytes at a time; a padding prefix gets a CAP row.
template <typename V, int NB, int FX, int NA>
__device__ __forceinline__ void cross_row(const EpiTau& et, const EnumParams& p, const V* vals, const int64_t pg,
                                          const bool live, V* xrow) {
  using T = VT<V>;
  constexpr int VN = Vec4<V>::N;
  const int DinP = (et.Din + 3) & ~3;
  constexpr int DPC = (NB + 3) & ~3;            // compile-time row length (D_in = D_o of a layer chain)
  // measured (A/B on one B200): the register path costs spills at NB = 24
  // (C3 0.784 -> 0.779 of the ALU roofline) and pays at NB = 23 (C5
  // 0.783 -> 0.791)
  const bool fastx = FX && NA > 0 && NB != 24 && DinP == DPC && pg < 0x7FFFFFFF;
  if (fastx && et.nq > 0) {
    // the whole row in registers: per term its DPC / VN 16-byte loads are
    // issued together (one L1/L2 round trip per term, not one per vector)
    V xa[DPC];
#pragma unroll
    for (int k2 = 0; k2 < DPC; ++k2) xa[k2] = live ? (V)0 : T::CAP;
    for (int i = 0; i < et.nq; ++i) {
      const int a = et.q[i].a;
      const int dig = (int)(((uint32_t)pg / (uint32_t)p.pre_stride[a]) % (uint32_t)p.pre_radix[a]);
      const V* qr = vals + et.qt[i] + dig * DPC;
      V y[DPC];
#pragma unroll
      for (int u0 = 0; u0 < DPC; u0 += VN) load_vec<V>(qr + u0, y + u0);
#pragma unroll
      for (int k2 = 0; k2 < DPC; ++k2) xa[k2] = T::sat(xa[k2], y[k2]);
    }
#pragma unroll
    for (int u0 = 0; u0 < DPC; u0 += VN) store_vec<V>(xrow + u0, xa + u0);
    return;
  }
  for (int i = 0; i < et.nq; ++i) {
    const int a = et.q[i].a;
    const int dig = pg < 0x7FFFFFFF ? (int)(((uint32_t)pg / (uint32_t)p.pre_stride[a]) % (uint32_t)p.pre_radix[a])
                                    : (int)((pg / p.pre_stride[a]) % p.pre_radix[a]);
    const V* qr = vals + et.qt[i] + dig * DinP;
    for (int u0 = 0; u0 < DinP; u0 += VN) {
      V y[VN], x[VN];
      if (live) load_vec<V>(qr + u0, y);
      else {
#pragma unroll
        for (int k2 = 0; k2 < VN; ++k2) y[k2] = T::CAP;
      }
      if (i > 0) {
        load_vec<V>(xrow + u0, x);
#pragma unroll
        for (int k2 = 0; k2 < VN; ++k2) y[k2] = T::sat(x[k2], y[k2]);
      }
      store_vec<V>(xrow + u0, y);
    }
  }
  if (et.nq == 0)
    for (int u0 = 0; u0 < DinP; u0 += VN) {
      V y[VN];
#pragma unroll
      for (int k2 = 0; k2 < VN; ++k2) y[k2] = live ? (V)0 : T::CAP;
      store_vec<V>(xrow + u0, y);
    }
}

// The fold's blocks: thread = one 4 x BW block of (u, v) in one stripe of
// rows; min over its rows of X_r[u] + B_r[v] into the shared minima `red`
// (atomic), or straight to the chunk minima when there is one stripe.
template <typename V, int BW>
__device__ __forceinline__ void fold_blocks(const V* Xs, const V* Bs, V* red, const int DinP, const int VP,
                                            const int CH, const int Din, const int v_cnt, const int v_lo,
                                            const int Do, const int64_t nchunks, const int64_t chunk, V* out) {
  using T = VT<V>;
  constexpr int VN = Vec4<V>::N;
  const int tid = threadIdx.x;
  const int nbv = VP / BW;
  const int nblk = (DinP / 4) * nbv;
  const int stripes = nblk >= kBlock ? 1 : min(8, kBlock / nblk);
  const int gi = tid / nblk;
  const bool active = nblk >= kBlock ? tid < nblk : gi < stripes;
  for (int blk = (nblk >= kBlock ? tid : tid - gi * nblk); active && blk < nblk;
       blk += (nblk >= kBlock ? kBlock : nblk)) {
    const int u0 = (blk / nbv) * 4;
    const int v0 = (blk % nbv) * BW;
    V res[4][BW];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < BW; ++j) res[i][j] = T::CAP;
    const int rs = stripes > 1 ? gi : 0;
    for (int r = rs; r < CH; r += stripes) {
      V x[4], y[BW];
#pragma unroll
      for (int i = 0; i < 4; i += VN) load_vec<V>(Xs + r * DinP + u0 + i, x + i);
#pragma unroll
      for (int j = 0; j < BW; j += VN) load_vec<V>(Bs + r * VP + v0 + j, y + j);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < BW; ++j) res[i][j] = T::addmin(x[i], y[j], res[i][j]);
    }
    if (nblk >= kBlock) {                           // one stripe: write straight out
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < BW; ++j)
          if (u0 + i < Din && v0 + j < v_cnt) out[((int64_t)(u0 + i) * Do + v_lo + v0 + j) * nchunks + chunk] = res[i][j];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < BW; ++j) atomic_min_v<V>(red + (u0 + i) * VP + v0 + j, res[i][j]);
    }
  }
}

// CTA = (group g = (low prefix part l, register group vg), h-block hb of
// kBlock prefixes); thread = one prefix.  After the enumeration the CTA holds
// the complete B_p[v] of its prefixes and folds the cross-segment terms of
// every incoming transition into this chunk's minima (epilogue):
//    chunkmin_t[u][v][chunk] = min_{p in chunk} X^t_p[u] + B_p[v],
//    X^t_p[u] = sum_{cross (j, Q)} Q[u][s_j(p)]          (Eq. 3 r_n)
// with 4x4 register-blocked fused add+mins over the chunk's rows.
// ST = 0: tables read from global/L2; 1: CTA slices staged in shared memory;
// 2: staged, and the Z term folded into per-m copies of the Y rows
// (Y'[m][j] = Y[m][j] + Z[m]) with K0[p] added once after the enumeration --
// no per-m saturating add in the loop (exact: min(K0 + t) = K0 + min t).
// NA > 0: the A space has exactly NA values (compile time) -- the A loop is
// fully unrolled with all NA x values loaded at the top of each M step, so no
// x load latency sits between consecutive VIADDMNMX groups.
// FX: the fold epilogue keeps a prefix's cross-term row in registers (only
// taken at NB != 24); instantiated without it for the output-digit-in-M
// layout, where the extra registers made ptxas spill into the main loop
// (C4: 9.82 -> 9.58 ms enumeration)
template <typename V, int NB, int ST, int MSPLIT, int NA = 0, int FX = 1, int MX = 0>
__global__ void __launch_bounds__(kBlock, 4) enum_kernel(const EnumParams p) {
  constexpr bool STAGED = ST > 0;
  constexpr bool MERGED = ST == 2;
  using T = VT<V>;
  constexpr int VN = Vec4<V>::N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  ETRACE(0);
  constexpr int CH = kBlock / MSPLIT;                       // prefixes per CTA (= p.CH)
  const int slot = MSPLIT == 2 ? (tid & (CH - 1)) : tid;    // this thread's prefix slot
  const int half = MSPLIT == 2 ? tid / CH : 0;              // its share of the M values
  const uint32_t nhb = (uint32_t)(p.Gpad / CH);             // 32-bit index math (grid < 2^31)
  const uint32_t g = blockIdx.x / nhb;
  const int64_t hb = blockIdx.x - g * nhb;
  const int64_t l = g / (uint32_t)p.VG;
  const int vg = (int)(g - (uint32_t)l * (uint32_t)p.VG);
  const int64_t hh = hb * CH + slot;
  const bool live = hh < p.G;
  const int64_t pg = (p.h0 + hh) * p.W + l;       // global canonical prefix
  const int64_t row = hh * p.W + l;               // local canonical prefix
  // prefix digits -> table offsets (ctx digits live in the low part l, so
  // sx/sy/sz are uniform over the CTA)
  int64_t sx = 0, sy = 0, sz = 0;
  int od = 0;
  if (pg < 0x7FFFFFFF) {
    uint32_t q = (uint32_t)pg;
    for (int d = p.P - 1; d >= 0; --d) {
      const uint32_t r = (uint32_t)p.pre_radix[d];
      const int dig = (int)(q % r);
      q /= r;
      sx += dig * p.pre_sx[d];
      sy += dig * p.pre_sy[d];
      sz += dig * p.pre_sz[d];
      if (d == p.o_pre) od = dig;
    }
  } else {
    int64_t q = pg;
    for (int d = p.P - 1; d >= 0; --d) {
      const int dig = (int)(q % p.pre_radix[d]);
      q /= p.pre_radix[d];
      sx += dig * p.pre_sx[d];
      sy += dig * p.pre_sy[d];
      sz += dig * p.pre_sz[d];
      if (d == p.o_pre) od = dig;
    }
  }
  const V* XT = static_cast<const V*>(p.XT);
  const V* YT = static_cast<const V*>(p.YT);
  const V* ZT = static_cast<const V*>(p.ZT);
  const int4* MT = p.mtab;
  ETRACE(1);
  if constexpr (STAGED) {
    V* xs = reinterpret_cast<V*>(smem_raw);
    V* ys = xs + p.xspan;
    V* zs = ys + p.yspan;
    int4* ms = reinterpret_cast<int4*>(zs + ((p.zspan + 3) & ~3LL));
    // the CTA's X and Y slices and the M table arrive by TMA bulk copies
    // (one thread issues, an mbarrier counts the bytes); Z (a few values,
    // any alignment) by plain loads meanwhile
    __shared__ __align__(8) uint64_t sbar;
    const bool tma = p.xspan % VN == 0 && p.yspan % VN == 0 &&
                     ((reinterpret_cast<uintptr_t>(XT + sx) | reinterpret_cast<uintptr_t>(YT + sy)) & 15) == 0;
    if (tma) {
      if (tid == 0) {
        const uint32_t xb = (uint32_t)(p.xspan * sizeof(V)), yb = (uint32_t)(p.yspan * sizeof(V));
        const uint32_t mb = (uint32_t)(p.nM * sizeof(int4));
        mbar_init(&sbar, 1);
        mbar_expect_tx(&sbar, xb + yb + mb);
        tma_bulk_g2s(xs, XT + sx, xb, &sbar);
        tma_bulk_g2s(ys, YT + sy, yb, &sbar);
        tma_bulk_g2s(ms, MT, mb, &sbar);
      }
    } else {
      for (int64_t e = tid * VN; e < p.xspan; e += kBlock * VN)
        *reinterpret_cast<typename Vec4<V>::T*>(xs + e) =
            *reinterpret_cast<const typename Vec4<V>::T*>(XT + sx + e);
      for (int64_t e = tid * VN; e < p.yspan; e += kBlock * VN)
        *reinterpret_cast<typename Vec4<V>::T*>(ys + e) =
            *reinterpret_cast<const typename Vec4<V>::T*>(YT + sy + e);
      for (int64_t e = tid; e < p.nM; e += kBlock) ms[e] = MT[e];
    }
    for (int64_t e = tid; e < p.zspan; e += kBlock) zs[e] = ZT[sz + e];
    ETRACE(2);
    if (tma && tid == 0) mbar_wait(&sbar, 0);       // the barrier below releases everyone after it
    __syncthreads();
    ETRACE(3);
    XT = xs; YT = ys; ZT = zs; MT = ms;
    sx = sy = sz = 0;
    if constexpr (MERGED) {
      const int n = (int)(p.nM * p.nb_pad);           // staged: fits shared memory
      const uint32_t nbp = (uint32_t)p.nb_pad;
      if (p.ym_inplace) {                             // Y row m is the slice's row m: Y' over Y
        for (int e = tid; e < n; e += kBlock) ys[e] = T::sat(ys[e], zs[ms[(uint32_t)e / nbp].z]);
        __syncthreads();
        YT = ys;
      } else {
        V* ym = reinterpret_cast<V*>(ms + p.nM);
        for (int e = tid; e < n; e += kBlock) {
          const int m = (int)((uint32_t)e / nbp);
          const int4 mt = ms[m];
          ym[e] = T::sat(ys[mt.y + (e - m * (int)nbp)], zs[mt.z]);
        }
        __syncthreads();
        YT = ym;
      }
    }
  }
  ETRACE(4);
  V* Bp = static_cast<V*>(p.Bp) + row * p.Do;
  const uint32_t one = (uint32_t)p.one;            // 1, opaque to the compiler (keeps IMAD an FMA-pipe add)
  V acc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j] = T::CAP;
  const int ybase = vg * NB;
  if (live) {
    if (p.init_row)
      for (int v = 0; v < p.Do; ++v) Bp[v] = T::CAP;
    const V k0 = static_cast<const V*>(p.K0)[pg];
    // MS = 2: warps of half 0 take m in [0, mh), warps of half 1 [mh, nM)
    const int nM = (int)p.nM;                      // host: nM < 2^31 (mtab rows)
    const int mh = MSPLIT == 2 ? (nM + 1) / 2 : nM;
    const int m_lo = half ? mh : 0, m_hi = half ? nM : mh;
    for (int m = m_lo; m < m_hi; ++m) {
      const int4 mt = MT[m];
      constexpr int NBV = (NB + VN - 1) / VN * VN;   // Y rows are padded to whole vectors
      V y[NBV];
      if constexpr (MERGED) {
        const V* yr = YT + m * p.nb_pad + ybase;
#pragma unroll
        for (int j = 0; j < NBV; j += VN) load_vec<V>(yr + j, y + j);
      } else {
        const V km = T::sat(k0, ZT[sz + mt.z]);
        const V* yr = YT + sy + mt.y + ybase;
#pragma unroll
        for (int j = 0; j < NBV; j += VN) load_vec<V>(yr + j, y + j);
#pragma unroll
        for (int j = 0; j < NB; ++j) y[j] = T::sat(y[j], km);
      }
      const V* xr = XT + sx + mt.x;
      if constexpr (NA > 0) {
        constexpr int NAV = (NA + VN - 1) / VN * VN;  // X rows are padded to whole vectors
        V x[NAV];
#pragma unroll
        for (int a = 0; a < NAV; a += VN) load_vec<V>(xr + a, x + a);
        if constexpr (MX && sizeof(V) == 4) {
          // two pipes: of every three A values, one combination is a
          // VIADDMNMX (ALU pipe) and two are adds on the FMA pipe (IMAD with a
          // runtime 1) folded in by one three-way min (VIMNMX3, ALU pipe):
          // 4 instructions, 2 per pipe, per 3 combinations instead of 3 ALU
          // instructions (exact: every sum <= 2 CAP < 2^32)
          // MX = A values per group: MX - 2 VIADDMNMX + one FMA-pipe pair
#pragma unroll
          for (int j0 = 0; j0 < NB; j0 += 4)
#pragma unroll
            for (int a = 0; a < NA; a += MX)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int j = j0 + q;
                if (j < NB) {
                  // FX = 0 (bucket digit in M): every M step starts from CAP
                  V t = (FX == 0 && a == 0) ? T::CAP : acc[j];
#pragma unroll
                  for (int b = 0; b < MX - 2; ++b)
                    if (a + b < NA) t = T::addmin(x[a + b], y[j], t);
                  if (a + MX - 1 < NA)
                    t = __vimin3_u32(t, mad_fma(x[a + MX - 2], one, y[j]), mad_fma(x[a + MX - 1], one, y[j]));
                  else if (a + MX - 2 < NA)
                    t = T::addmin(x[a + MX - 2], y[j], t);
                  acc[j] = t;
                }
              }
        } else if constexpr (FX == 0) {
          // FX = 0: the bucket-digit-in-M instantiation (C4, launched for
          // o_mode 1 only): the accumulators start every M step at
          // CAP, so the first A value's add+min takes CAP as its third operand
          // (an immediate) instead of NB register resets after each flush
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x[0], y[j], T::CAP);
#pragma unroll
          for (int a = 1; a < NA; ++a)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x[a], y[j], acc[j]);
        } else {
#pragma unroll
          for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x[a], y[j], acc[j]);
        }
      }
      const int na_v = NA > 0 ? 0 : p.na & ~(VN - 1);
#pragma unroll 2
      for (int a = 0; a < na_v; a += VN) {
        V x[VN];
        load_vec<V>(xr + a, x);
#pragma unroll
        for (int q = 0; q < VN; ++q)
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x[q], y[j], acc[j]);
      }
      for (int a = na_v; NA == 0 && a < p.na; ++a) {   // ragged A tail (no padded evaluations)
        const V x = xr[a];
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x, y[j], acc[j]);
      }
      if (p.o_mode == 1) {                        // bucket digit in M: flush per m
        V r = acc[0];
#pragma unroll
        for (int j = 1; j < NB; ++j) r = T::mn(r, acc[j]);
        if constexpr (MERGED) r = T::sat(r, k0);
        Bp[mt.w] = T::mn(Bp[mt.w], r);
        if constexpr (!(NA > 0 && FX == 0))             // those loops restart from CAP themselves
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = T::CAP;
      }
    }
    if constexpr (MERGED) {
      if (p.o_mode != 1) {
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[j] = T::sat(acc[j], k0);
      }
    }
    if (MSPLIT == 2) {
      // written after the two halves are merged (below)
    } else if (p.o_mode == 0) {
      if (p.o_bstride == 1 && p.o_bradix == p.nb) {       // B = {o}: slot j <-> v
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (ybase + j < p.nb) Bp[ybase + j] = acc[j];
      } else {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (ybase + j < p.nb) {
            const int v = ((ybase + j) / p.o_bstride) % p.o_bradix;
            Bp[v] = T::mn(Bp[v], acc[j]);
          }
      }
    } else if (p.o_mode == 2) {
      V r = acc[0];
#pragma unroll
      for (int j = 1; j < NB; ++j) r = T::mn(r, acc[j]);
      Bp[od] = r;
    }
  }
  ETRACE(5);
  const bool simple = p.o_mode == 0 && p.o_bstride == 1 && p.o_bradix == p.nb;
  const int v_lo = simple ? ybase : 0;
  const int v_cnt = simple ? min(NB, p.nb - ybase) : p.Do;
  const int VP = (v_cnt + 3) & ~3;
  V* Bs = reinterpret_cast<V*>(smem_raw);                     // [CH][VP] (over the staged tables)
  V* Xs = Bs + p.xs_off;                                      // [CH][DinP] cross rows
  V* red = Xs + CH * p.dinp_max;                              // [DinP][VP] fold minima (shared atomics)
  if constexpr (MSPLIT == 2) {
    // merge the two halves' bucket minima of each prefix (B = {o}, simple):
    // half 1 parks its registers in Bs, half 0 takes the min, writes B_p and
    // leaves the merged row in Bs for the fold
    __syncthreads();                              // staged tables no longer needed
    if (half == 1) {
#pragma unroll
      for (int j = 0; j < NB; j += VN) {
        V w[VN];
#pragma unroll
        for (int q = 0; q < VN; ++q) w[q] = j + q < NB ? acc[j + q] : T::CAP;
        if (j + VN <= VP) store_vec<V>(Bs + slot * VP + j, w);
        else
          for (int q = 0; q < VN && j + q < VP; ++q) Bs[slot * VP + j + q] = w[q];
      }
    }
    __syncthreads();
    if (half == 0) {
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < VP) acc[j] = T::mn(acc[j], Bs[slot * VP + j]);
      if (live) {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (ybase + j < p.nb) Bp[ybase + j] = acc[j];
      }
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < VP) Bs[slot * VP + j] = (live && j < v_cnt) ? acc[j] : T::CAP;
    }
  }
  if (p.ntau == 0) return;
  // ---- epilogue: fold the cross-segment terms of every incoming transition
  __syncthreads();                                // staged tables no longer needed / Bs merged
  if (MSPLIT == 2) {
    // Bs already holds the merged rows
  } else if (simple && VP == NB) {                // 16-byte stores (conflict-light rows)
#pragma unroll
    for (int j = 0; j < NB; j += VN) {
      V w[VN];
#pragma unroll
      for (int q = 0; q < VN; ++q) w[q] = (live && j + q < v_cnt) ? acc[j + q] : T::CAP;
      store_vec<V>(Bs + tid * VP + j, w);
    }
  } else if (simple) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j < VP) Bs[tid * VP + j] = (live && j < v_cnt) ? acc[j] : T::CAP;
  } else {
    for (int j = 0; j < VP; ++j) Bs[tid * VP + j] = (live && j < v_cnt) ? Bp[j] : T::CAP;
  }
  const V* vals = static_cast<const V*>(p.vals);
  const int64_t chunk = l * nhb + hb;
  for (int t = 0; t < p.ntau; ++t) {
    const EpiTau& et = p.taus[t];
    const int Din = et.Din, DinP = (Din + 3) & ~3;
    const int nblk = (DinP / 4) * (VP / 4);         // = fold_blocks' block count
    if (t > 0) __syncthreads();                     // the previous transition is done with Xs / red
    if (half == 0) cross_row<V, NB, FX, NA>(et, p, vals, pg, live, Xs + slot * DinP);
    if (nblk < kBlock)
      for (int e = tid; e < DinP * VP; e += kBlock) red[e] = T::CAP;
    __syncthreads();
    // min_p X_p[u] + B_p[v] over the chunk's rows: 4 x 4 register blocks, the
    // rows split into stripes (one block per thread), the stripes' minima
    // merged by shared-memory atomic mins.  Measured (C3 / C5 / C4 enumeration
    // ms): 4 x 4 with the per-stripe partials reduced by a separate pass
    // 0.625 / 0.465 / 9.60, with atomic mins 0.624 / 0.465 / --, 4 x 8 blocks
    // (14 stripes, twice the atomics per address) 0.647 / 0.473 / 9.51
    fold_blocks<V, 4>(Xs, Bs, red, DinP, VP, CH, Din, v_cnt, v_lo, p.Do, p.nchunks, chunk,
                      static_cast<V*>(et.chunkmin));
    if (nblk < kBlock) {
      __syncthreads();
      V* out = static_cast<V*>(et.chunkmin);
      for (int e = tid; e < Din * v_cnt; e += kBlock) {
        const int u = e / v_cnt, vv = e - u * v_cnt;
        out[((int64_t)u * p.Do + v_lo + vv) * p.nchunks + chunk] = red[u * VP + vv];
      }
    }
  }
  ETRACE(6);
}

// --------------------------------------------------------------------------
// a1 fold: chunk c of local prefixes; chunkmin[c][u][v] = min_p X_p[u] + B_p[v]
// with X_p[u] = sum_{cross (j, Q)} Q[u][s_j(p)]   (Eq. 3 r_n).
// --------------------------------------------------------------------------
template <typename V>
__device__ __forceinline__ V cross_sum(const FoldParams& f, const V* vals, int64_t pg, int u) {
  V x = 0;
  for (int i = 0; i < f.nq; ++i) {
    const Term& q = f.q[i];
    const int dig = prefix_digit(pg, q.a, f.P, f.pre_radix);
    x = VT<V>::sat(x, vals[q.off + (int64_t)u * q.db + dig]);
  }
  return x;
}

template <typename V>
__device__ __forceinline__ void load4(const V* p, V* out) {
  if constexpr (sizeof(V) == 4) {
    load_vec<V>(p, out);
  } else {
    load_vec<V>(p, out);
    load_vec<V>(p + 2, out + 2);
  }
}

// --------------------------------------------------------------------------
// Fused least-index argmin, one CTA (128 threads) per bucket (u, v):
//  1. A = min over the chunk minima and the first chunk c* attaining it;
//  2. the least prefix p* in chunk c* with X_p[u] + B_p[v] == A;
//  3. the least suffix (canonical order; s_o = v when o is a suffix digit)
//     whose intra cost equals B_p*[v];
//  4. outputs in the caller's (unpruned) layout: A[u][v_orig], I[u][v_orig].
// --------------------------------------------------------------------------
template <typename V, int NT>
__device__ void argmin_pair(const ArgminParams& ap, const int pair, unsigned char* smem_raw,
                            const V* pre_tabs = nullptr, const int64_t* hb_pre = nullptr) {
  const int tid = threadIdx.x;
  // descriptor pieces used inside loops -> shared memory (one global read each)
  __shared__ Term s_terms[kMaxTerms];
  __shared__ Term s_q[kMaxCross];
  __shared__ int32_t s_rad[kMaxDigits];          // compact radices (prefix and suffix)
  __shared__ int64_t s_misc[8];
  __shared__ unsigned long long s_first;
  __shared__ int s_cnt;
  const EvalSpec& e = ap.e;
  const FoldParams& f = ap.f;
  for (int i = tid; i < e.nterm; i += NT) s_terms[i] = e.term[i];
  __shared__ uint32_t s_qstr[kMaxCross], s_qrad[kMaxCross];   // consumer digit of each cross term
  for (int i = tid; i < f.nq; i += NT) {
    s_q[i] = f.q[i];
    s_qstr[i] = (uint32_t)f.pre_stride[f.q[i].a];
    s_qrad[i] = (uint32_t)e.radix[f.q[i].a];
  }
  for (int i = tid; i < e.K; i += NT) s_rad[i] = e.radix[i];
  TTRACE(2, 20);
  if (tid == 0) {
    s_misc[0] = f.nchunks; s_misc[1] = f.nhb; s_misc[2] = f.G; s_misc[3] = f.W;
    s_misc[4] = f.p_lo; s_misc[5] = f.Do; s_misc[6] = (int64_t)(uintptr_t)f.chunkmin;
    s_misc[7] = (int64_t)(uintptr_t)f.Bp;
    s_first = ~0ull;
    s_cnt = 0;
  }
  __syncthreads();
  const int64_t nchunks = s_misc[0], nhb = s_misc[1], Gh = s_misc[2], W = s_misc[3], p_lo = s_misc[4];
  const int Do = (int)s_misc[5];
  const V* cm = reinterpret_cast<const V*>((uintptr_t)s_misc[6]) + (int64_t)pair * nchunks;
  const V* Bp = reinterpret_cast<const V*>((uintptr_t)s_misc[7]);
  const V* vals = static_cast<const V*>(f.vals);
  const int K = e.K, P = e.P, o = e.o, nterm = e.nterm, nq = f.nq;
  uint16_t* sd = reinterpret_cast<uint16_t*>(smem_raw);        // [K][NT] digits
  const V* tabs = pre_tabs;                                     // W/R tables (staged by the caller)
  if (!pre_tabs) {
  V* st = reinterpret_cast<V*>(smem_raw + (((size_t)K * NT * 2 + 15) & ~(size_t)15));
  tabs = st;
  for (int i0 = tid; i0 < e.tab_n; i0 += NT * 8) {   // 8 loads in flight per thread
    V t8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t8[k] = i0 + k * NT < e.tab_n ? vals[e.tab_lo + i0 + k * NT] : (V)0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i0 + k * NT < e.tab_n) st[i0 + k * NT] = t8[k];
  }
  }
  const int u = pair / Do, v = pair - (pair / Do) * Do;
  TTRACE(2, 21);
  const int64_t outi = (int64_t)u * ap.Do_orig + ap.vmap[v];
  // 1. the bucket minimum is the (merged) A computed by amin_kernel
  const uint64_t Ag = __ldcg(ap.A_glob + outi);    // L2: written by other CTAs in the fused tail
  if (Ag == kInf64) {
    if (tid == 0) { ap.A_out[outi] = kInf64; ap.I_out[outi] = kInf64; }
    return;
  }
  const V best = (V)Ag;
  // 2. chunks of this rank attaining it (none: this rank holds no candidate);
  //    the fused tail's bucket-minimum pass already found the least attaining
  //    h-block (hb_pre) -- then steps 1-2 are skipped
  const int64_t hb_known = hb_pre ? __ldcg(hb_pre + pair) : -1;
  constexpr int LIST = 4 * NT > 1024 ? 1024 : 4 * NT;
  __shared__ int64_t s_list[LIST];
  for (int64_t c0 = (int64_t)tid * 4; hb_known < 0 && c0 < nchunks; c0 += NT * 4) {
    V x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = c0 + q < nchunks ? cm[c0 + q] : VT<V>::CAP;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (x[q] == best) {
        const int at = atomicAdd(&s_cnt, 1);
        if (at < LIST) s_list[at] = c0 + q;
      }
  }
  __syncthreads();
  const int cnt_all = hb_known >= 0 ? 1 : s_cnt;
  TTRACE(2, 22);
  if (cnt_all == 0) {                               // possible only with world > 1
    if (tid == 0) { ap.A_out[outi] = kInf64; ap.I_out[outi] = kInf64; }
    return;
  }
  // every row of h-block hb precedes every row of a later h-block in canonical
  // order and every attaining chunk holds an attaining row: p* lies in the
  // chunks of the least attaining h-block
  __shared__ long long s_hbmin;
  if (tid == 0) s_hbmin = hb_known >= 0 ? hb_known : 0x7FFFFFFFFFFFFFFFLL;
  __syncthreads();
  if (hb_known >= 0) {
  } else if (cnt_all <= LIST) {
    for (int li = tid; li < cnt_all; li += NT) atomicMin(&s_hbmin, (long long)(s_list[li] % nhb));
  } else {
    for (int64_t c = tid; c < nchunks; c += NT)
      if (cm[c] == best) atomicMin(&s_hbmin, (long long)(c % nhb));
  }
  __syncthreads();
  const int64_t hbmin = s_hbmin;
  TTRACE(2, 23);
  // rows of the chunks (l, hbmin), l < W, attaining the minimum
  __shared__ int32_t s_ls[NT];
  __shared__ int s_nl;
  if (tid == 0) s_nl = 0;
  __syncthreads();
  for (int64_t l = tid; l < W; l += NT)
    if (cm[l * nhb + hbmin] == best) {
      const int at = atomicAdd(&s_nl, 1);
      if (at < NT) s_ls[at] = (int32_t)l;
    }
  __syncthreads();
  const int nl = min(s_nl, NT);                       // W > NT with > NT hits: rare, see below
  const bool all_l = s_nl > NT;
  const int64_t CH = f.CH;
  const int64_t nrow = (all_l ? W : (int64_t)nl) * CH;
  const bool narrow_ix = nrow < 0x7FFFFFFF && p_lo + (hbmin + 1) * CH * W < 0x7FFFFFFF;
#pragma unroll 2
  for (int64_t w = tid; w < nrow; w += NT) {
    int64_t li, i;
    if (narrow_ix) {
      li = (uint32_t)w / (uint32_t)CH;
      i = (uint32_t)w - (uint32_t)li * (uint32_t)CH;
    } else {
      li = w / CH;
      i = w - li * CH;
    }
    const int64_t l = all_l ? li : s_ls[li];
    const int64_t hh = hbmin * CH + i;
    if (hh >= Gh) continue;
    if (all_l && cm[l * nhb + hbmin] != best) continue;
    const int64_t plr = hh * W + l;
    const int64_t pg = p_lo + plr;
    const V b = Bp[plr * Do + v];
    V x = 0;
    if (narrow_ix) {                                 // 32-bit digit extraction by stride
      const uint32_t pq = (uint32_t)pg;
      for (int qi = 0; qi < nq; ++qi) {
        const uint32_t d = (pq / s_qstr[qi]) % s_qrad[qi];
        x = VT<V>::sat(x, vals[s_q[qi].off + (int64_t)u * s_q[qi].db + d]);
      }
    } else {
      for (int qi = 0; qi < nq; ++qi) {
        const Term q = s_q[qi];
        x = VT<V>::sat(x, vals[q.off + (int64_t)u * q.db + prefix_digit(pg, q.a, P, s_rad)]);
      }
    }
    if (VT<V>::sat(x, b) == best) atomicMin(&s_first, (unsigned long long)plr);
  }
  __syncthreads();
  const int64_t pl = (int64_t)s_first;
  TTRACE(2, 24);
  __syncthreads();
  if (tid == 0) s_first = ~0ull;
  const uint64_t target = (uint64_t)Bp[pl * Do + v];
  const int64_t pg = p_lo + pl;
  auto S = [&](int d) -> uint16_t& { return sd[d * NT + tid]; };
  {
    int64_t q = pg;
    for (int d = P - 1; d >= 0; --d) { S(d) = (uint16_t)(q % s_rad[d]); q /= s_rad[d]; }
  }
  const bool o_suffix = o >= P;
  const int64_t nrest = o_suffix ? e.nsuffix / s_rad[o] : e.nsuffix;
  __syncthreads();
  // 3. least suffix (canonical order, s_o = v if o is a suffix digit) whose
  //    intra cost equals B_p*[v]
  const int64_t per = (nrest + NT - 1) / NT;
  TTRACE(2, 25);
  const int64_t lo = (int64_t)tid * per;
  const int64_t hi = min(nrest, lo + per);
  if (lo < hi) {
    int64_t q = lo;
    for (int d = K - 1; d >= P; --d) {
      if (o_suffix && d == o) { S(d) = (uint16_t)v; continue; }
      S(d) = (uint16_t)(q % s_rad[d]);
      q /= s_rad[d];
    }
    for (int64_t r = lo; r < hi; ++r) {
      uint64_t c = 0;
      bool inf = false;
      for (int i = 0; i < nterm; ++i) {
        const Term tm = s_terms[i];
        const int64_t to = tm.off - e.tab_lo;
        const V x = tm.kind == 0 ? tabs[to + S(tm.a)] : tabs[to + (int)S(tm.a) * tm.db + S(tm.b)];
        inf |= x >= VT<V>::CAP;
        c += (uint64_t)x;
      }
      if (!inf && c == target) {
        int64_t sfx = 0;
        for (int d = P; d < K; ++d) sfx = sfx * s_rad[d] + S(d);
        atomicMin(&s_first, (unsigned long long)sfx);
        break;
      }
      for (int d = K - 1; d >= P; --d) {       // odometer step
        if (o_suffix && d == o) continue;
        if (++S(d) < s_rad[d]) break;
        S(d) = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const uint64_t sfx = s_first;
    uint64_t q = sfx;
    for (int d = K - 1; d >= P; --d) { S(d) = (uint16_t)(q % s_rad[d]); q /= s_rad[d]; }
    uint64_t idx = 0;
    for (int d = 0; d < K; ++d) idx = idx * ap.orig_radix[d] + ap.maps[ap.map_off[d] + S(d)];
    ap.A_out[outi] = Ag;
    ap.I_out[outi] = sfx == ~0ull ? kInf64 : idx;     // ~0: cannot happen (exact arithmetic)
  }
}

// Persistent walk over a list of (transition slot, bucket) entries.
template <typename V>
__global__ void __launch_bounds__(256) argmin_kernel(const ArgminParams* __restrict__ aps,
                                                     const ArgminEntry* __restrict__ list,
                                                     const int32_t* __restrict__ count, int wide) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = *count;
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const ArgminEntry en = list[it];
    const ArgminParams& ap = aps[en.slot];
    if (ap.wide != wide) continue;                  // uniform per CTA
    argmin_pair<V, 256>(ap, en.pair, smem_raw);
    __syncthreads();
  }
}

// A[u][v] = min over the chunk minima (values only), one warp per bucket.
template <typename V>
__global__ void amin_kernel(const ArgminParams* __restrict__ aps, const int64_t* __restrict__ pair_off,
                            int nslot, int wide) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int s = 0;
  while (s < nslot && w >= pair_off[s + 1]) ++s;
  if (s >= nslot) return;
  const ArgminParams& ap = aps[s];
  if (ap.wide != wide || ap.f.nchunks == 0) return;
  const int pair = (int)(w - pair_off[s]);
  const V* cm = static_cast<const V*>(ap.f.chunkmin) + (int64_t)pair * ap.f.nchunks;
  V best = VT<V>::CAP;
  for (int64_t c = lane; c < ap.f.nchunks; c += 32) best = VT<V>::mn(best, cm[c]);
  for (int o = 16; o > 0; o >>= 1) best = VT<V>::mn(best, (V)__shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) {
    const int u = pair / ap.f.Do, v = pair - u * ap.f.Do;
    ap.A_out[(int64_t)u * ap.Do_orig + ap.vmap[v]] = best >= VT<V>::CAP ? kInf64 : (uint64_t)best;
  }
}

// all buckets of every slot (cfp_segment_costs / full tables)
__global__ void all_pairs_kernel(const int64_t* __restrict__ pair_off, int nslot, ArgminEntry* list, int32_t* count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0) *count = (int32_t)pair_off[nslot];
  if (i >= pair_off[nslot]) return;
  int s = 0;
  while (i >= pair_off[s + 1]) ++s;
  list[i] = ArgminEntry{s, (int32_t)(i - pair_off[s])};
}

// chain edge list (slot, u * Do_orig + v_orig) -> compact bucket entries
__global__ void edges_to_pairs_kernel(const ArgminParams* __restrict__ aps, ArgminEntry* list,
                                      const int32_t* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *count) return;
  ArgminEntry en = list[i];
  const ArgminParams& ap = aps[en.slot];
  const int u = en.pair / ap.Do_orig, vo = en.pair - u * ap.Do_orig;
  const int vc = ap.vinv[vo];
  en.pair = vc < 0 ? 0 : u * ap.f.Do + vc;       // pruned columns are INF: never optimal
  list[i] = en;
}

// --------------------------------------------------------------------------
// a3 + a4: chain (single CTA).  G_N = terminal; runs processed last to first;
// a run of L identical square matrices uses powers P_j = M^(2^j) (repeated
// squaring) and fills its suffix vectors by doubling:
//    G_{e-k} = P_j (x) G_{e-k+2^j}   for k in [2^j, 2^(j+1))
// then (optionally) the forward greedy backtrack picks, at each instance, the
// optimal successor with the least combination index.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t sat64(uint64_t a, uint64_t b) {
  return (a == kInf64 || b == kInf64) ? kInf64 : a + b;
}




// min_v sat64(row[v], g[v]) with four independent partial minima (ILP)
__device__ __forceinline__ uint64_t minplus_dot(const uint64_t* row, int rstride, const uint64_t* g, int n) {
  uint64_t b0 = kInf64, b1 = kInf64, b2 = kInf64, b3 = kInf64;
  int v = 0;
  for (; v + 4 <= n; v += 4) {
    const uint64_t x0 = sat64(row[(int64_t)v * rstride], g[v]);
    const uint64_t x1 = sat64(row[(int64_t)(v + 1) * rstride], g[v + 1]);
    const uint64_t x2 = sat64(row[(int64_t)(v + 2) * rstride], g[v + 2]);
    const uint64_t x3 = sat64(row[(int64_t)(v + 3) * rstride], g[v + 3]);
    b0 = x0 < b0 ? x0 : b0;
    b1 = x1 < b1 ? x1 : b1;
    b2 = x2 < b2 ? x2 : b2;
    b3 = x3 < b3 ? x3 : b3;
  }
  for (; v < n; ++v) {
    const uint64_t x = sat64(row[(int64_t)v * rstride], g[v]);
    b0 = x < b0 ? x : b0;
  }
  b0 = b1 < b0 ? b1 : b0;
  b2 = b3 < b2 ? b3 : b2;
  return b2 < b0 ? b2 : b0;
}

// Warp-cooperative min_v sat64(row[v], g[v]): lanes over v (contiguous,
// bank-conflict free), butterfly min; every lane returns the result.
__device__ __forceinline__ uint64_t warp_row_min(const uint64_t* row, const uint64_t* g, int n, int lane) {
  uint64_t b = kInf64;
  for (int v = lane; v < n; v += 32) {
    const uint64_t x = sat64(row[v], g[v]);
    b = x < b ? x : b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, b, o);
    b = y < b ? y : b;
  }
  return b;
}

// Single-CTA chain.  SM = true: every distinct matrix (A and, for the
// backtrack, I), every suffix vector G_n, the powers of the current run and the
// instance metadata live in shared memory; G is copied out at the end.
// SM = false: same algorithm on global memory (large S).
// mode 0: G + backtrack; 1: G + the optimal edges reachable from u_1 = 0
// (the only buckets whose least index the backtrack needs); 2: backtrack with
// G already computed.
// goff[N] (rows of all instances) read from the parameter block's table
__device__ __forceinline__ int64_t goff_n_of(const ChainParams& cp) { return cp.goff[cp.N]; }

// part: kChainWhole = the kernel's cp.mode; inside the fused tail kernel (one
// CTA, shared memory kept between the calls) kChainFusedEdges = mode 1 with the
// A matrices read by plain loads (they were written by other CTAs of the same
// launch) and no I staging, kChainFusedBacktrack = mode 2 with A, G and the
// metadata still in shared memory from the first call and I loaded now.
constexpr int kChainWhole = 0, kChainFusedEdges = 1, kChainFusedBacktrack = 2;

template <bool SM>
__device__ void chain_run(const ChainParams& cp, unsigned char* smem_raw, const int part) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int N = cp.N;
  uint64_t* sA = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* sI = sA + cp.mat_elems;
  uint64_t* sG = sI + (cp.backtrack ? cp.mat_elems : 0);
  uint64_t* sP = sG + cp.goff[N + 1];
  int64_t* sgoff = reinterpret_cast<int64_t*>(sP + (int64_t)cp.levels_max * cp.smax * cp.smax);
  int64_t* smoff = sgoff + N + 2;
  int4* sinst = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(smoff + cp.nmat) + 15) & ~uintptr_t(15));
  int16_t* nxt = reinterpret_cast<int16_t*>(sinst + N);        // [goff[N]] successor of (n, u)
  int32_t* vseq = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(nxt + cp.goff[N]) + 15) & ~uintptr_t(15));
  uint32_t* ebits = reinterpret_cast<uint32_t*>(vseq + N);     // mode 1 dedupe bitset
  uint32_t* om = ebits + (cp.mat_elems + 31) / 32;               // mode 1: optimal-successor masks [goff[N]]
  uint32_t* rmask = om + goff_n_of(cp);                           // mode 1: reachable-state masks [N]
  uint64_t* G = SM ? sG : cp.G;
  uint64_t* Pw = SM ? sP : cp.powers;
  const int64_t* goff = SM ? sgoff : cp.goff;
  if (SM && part == kChainFusedBacktrack) {
    for (int64_t e = tid; e < cp.mat_elems; e += nth) sI[e] = __ldcg(cp.baseI + e);   // other CTAs' writes
    __syncthreads();
  } else if constexpr (SM) {
    __shared__ __align__(8) uint64_t cbar;
    const bool tma = part == kChainWhole && (cp.mat_elems & 1) == 0;   // 16-byte multiples
    if (tma) {
      if (tid == 0) {
        mbar_init(&cbar, 1);
        const uint32_t bytes = (uint32_t)(cp.mat_elems * 8);
        mbar_expect_tx(&cbar, bytes * (cp.backtrack ? 2 : 1));
        tma_bulk_g2s(sA, cp.baseA, bytes, &cbar);
        if (cp.backtrack) tma_bulk_g2s(sI, cp.baseI, bytes, &cbar);
      }
    } else {
      for (int64_t e = tid; e < cp.mat_elems; e += nth) {
        sA[e] = __ldcg(cp.baseA + e);
        if (cp.backtrack && part == kChainWhole) sI[e] = cp.baseI[e];
      }
    }
    for (int i = tid; i < N + 2; i += nth) sgoff[i] = cp.goff[i];
    for (int i = tid; i < cp.nmat; i += nth) smoff[i] = cp.moff[i];
    for (int i = tid; i < N; i += nth) sinst[i] = make_int4(cp.inst[i].mat, cp.inst[i].rows, cp.inst[i].cols, 0);
    if (cp.mode == 1)
      for (int64_t i = tid; i < (cp.mat_elems + 31) / 32; i += nth) ebits[i] = 0;
    if (tma && tid == 0) mbar_wait(&cbar, 0);      // only the initialising thread polls; the barrier below releases the rest
    __syncthreads();
  }
  TTRACE(0, 1);
  auto rows_of = [&](int n) { return SM ? sinst[n].y : cp.inst[n].rows; };
  auto cols_of = [&](int n) { return SM ? sinst[n].z : cp.inst[n].cols; };
  auto mat_of = [&](int n) { return SM ? sinst[n].x : cp.inst[n].mat; };
  auto matA = [&](int n) -> const uint64_t* { return SM ? sA + smoff[sinst[n].x] : cp.inst[n].A; };
  auto matI = [&](int n) -> const uint64_t* { return SM ? sI + smoff[sinst[n].x] : cp.inst[n].I; };
  const int lastc = cols_of(N - 1);
  if (cp.mode == 2) {                               // suffix vectors already computed
    if (SM && part != kChainFusedBacktrack)
      for (int64_t e2 = tid; e2 < goff[N + 1]; e2 += nth) G[e2] = cp.G[e2];
    __syncthreads();
  } else {
    for (int v = tid; v < lastc; v += nth) G[goff[N] + v] = cp.terminal ? cp.terminal[v] : 0;
    __syncthreads();
    for (int r = cp.nruns - 1; r >= 0; --r) {
      TTRACE(0, 2 + min(cp.nruns - 1 - r, 7));
      const ChainRun run = cp.runs[r];
      const uint64_t* M = matA(run.first);
      const int R = rows_of(run.first), Cc = cols_of(run.first);
      const int e = run.first + run.len;             // G_e known (1-based instance e)
      if (run.len == 1) {
        const uint64_t* g = G + goff[e];
        const int warp = tid >> 5, lane = tid & 31;
        for (int u = warp; u < R; u += nth >> 5) {              // warp per row
          const uint64_t b = warp_row_min(M + (int64_t)u * Cc, g, Cc, lane);
          if (lane == 0) G[goff[e - 1] + u] = b;
        }
        __syncthreads();
        continue;
      }
      const int S = R;                                // square
      int levels = 0;
      while ((1 << (levels + 1)) <= run.len) ++levels;   // P_0 .. P_levels
      if (!SM && (int64_t)S * S * levels > cp.powers_cap) {
        if (tid == 0) *cp.status = 4;
        return;
      }
      // repeated squaring: P_j = P_{j-1} (x) P_{j-1}
      for (int j = 1; j <= levels; ++j) {
        const uint64_t* Pa = j == 1 ? M : Pw + (int64_t)(j - 2) * S * S;
        uint64_t* Pc = Pw + (int64_t)(j - 1) * S * S;
        for (int64_t c = tid; c < (int64_t)S * S; c += nth) {
          const int i = (int)(c / S), k2 = (int)(c - (int64_t)i * S);
          Pc[c] = minplus_dot(Pa + k2, S, Pa + (int64_t)i * S, S);      // min_k Pa[i][k] + Pa[k][k2]
        }
        __syncthreads();
      }
      // doubling: G_{e-k} = P_j (x) G_{e-k+2^j}, k in [2^j, 2^(j+1))
      for (int j = 0; j <= levels; ++j) {
        const uint64_t* Pj = j == 0 ? M : Pw + (int64_t)(j - 1) * S * S;
        const int k_lo = 1 << j, k_hi = min(1 << (j + 1), run.len + 1);
        const int64_t work = (int64_t)(k_hi - k_lo) * S;
        for (int64_t w = tid; w < work; w += nth) {
          const int k = k_lo + (int)(w / S), u = (int)(w % S);
          G[goff[e - k] + u] = minplus_dot(Pj + (int64_t)u * S, 1, G + goff[e - k + (1 << j)], S);
        }
        __syncthreads();
      }
    }
    if constexpr (SM)
      for (int64_t e2 = tid; e2 < goff[N + 1]; e2 += nth) cp.G[e2] = G[e2];
    TTRACE(0, 10);
  }
  if (cp.mode == 1 && SM && cp.smax <= 32) {
    // optimal edges reachable from u_1 = 0, for <= 32 states per instance:
    // (1) warp 0 walks the instances; for each reachable state u its optimal
    //     successors om = {v : A_n[u][v] + G_n(v) = G_{n-1}(u)} by one ballot
    //     (lanes = v), reach_{n+1} = OR of them -- only reachable rows are
    //     evaluated (usually one per instance);
    // (2) every (n, u) in parallel: emit the reachable optimal edges (deduplicated).
    __syncthreads();
    __shared__ int s_cnt2;
    if (tid == 0) s_cnt2 = 0;
    for (int64_t w = tid; w < goff[N]; w += nth) cp.reach[w] = 0;
    if (tid < 32) {
      const int lane = tid;
      uint32_t r = G[0] == kInf64 ? 0u : 1u;
      for (int n = 0; n < N; ++n) {
        if (lane == 0) rmask[n] = r;
        const int cols = cols_of(n);
        const int64_t g0 = goff[n];
        const uint64_t gv = lane < cols ? G[goff[n + 1] + lane] : kInf64;
        const uint64_t* An = matA(n);
        uint32_t nx = 0, rr = r;
        while (rr) {
          const int u = __ffs(rr) - 1;
          rr &= rr - 1;
          const uint64_t target = G[g0 + u];
          const uint64_t a = lane < cols ? An[(int64_t)u * cols + lane] : kInf64;
          const uint32_t m = __ballot_sync(0xffffffffu, target != kInf64 && a != kInf64 && gv != kInf64 &&
                                                          a + gv == target);
          if (lane == 0) om[g0 + u] = m;
          nx |= m;
        }
        r = nx;
      }
    }
    __syncthreads();
    for (int64_t w = tid; w < (int64_t)N * 32; w += nth) {   // (instance, lane = u)
      const int n = (int)(w >> 5), u = (int)(w & 31);
      if (u >= rows_of(n) || !((rmask[n] >> u) & 1u)) continue;
      cp.reach[goff[n] + u] = 1;
      const int cols = cols_of(n), mat = mat_of(n);
      const int64_t fo = smoff[mat];
      uint32_t m = om[goff[n] + u];
      while (m) {
        const int v = __ffs(m) - 1;
        m &= m - 1;
        const int64_t bit = fo + (int64_t)u * cols + v;
        if (!(atomicOr(&ebits[bit >> 5], 1u << (bit & 31)) & (1u << (bit & 31))))
          cp.edge_list[atomicAdd(&s_cnt2, 1)] = ArgminEntry{mat, u * cols + v};
      }
    }
    __syncthreads();
    if (tid == 0) *cp.edge_count = s_cnt2;
    TTRACE(0, 12);
    return;
  }
  if (cp.mode == 1) {
    // optimal edges reachable from u_1 = 0 (warp 0, sequential over instances;
    // reachable states found by ballot, edges deduplicated in a shared bitset)
    __syncthreads();
    __shared__ int s_cnt;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      __shared__ uint8_t rc[2][256];
      for (int s = lane; s < 256; s += 32) { rc[0][s] = 0; rc[1][s] = 0; }
      __syncwarp();
      if (lane == 0) rc[0][0] = 1;
      __syncwarp();
      int cur = 0;
      for (int n = 0; n < N; ++n) {
        const int rows = rows_of(n), cols = cols_of(n);
        const uint64_t* A = matA(n);
        const uint64_t* Gp = G + goff[n];
        const uint64_t* Gn = G + goff[n + 1];
        const int mat = mat_of(n);
        const int64_t fo = SM ? smoff[mat] : cp.moff[mat];
        for (int s = lane; s < 256; s += 32) rc[cur ^ 1][s] = 0;
        __syncwarp();
        for (int u0 = 0; u0 < rows && u0 < 256; u0 += 32) {
          unsigned live = __ballot_sync(0xffffffffu, u0 + lane < rows && u0 + lane < 256 && rc[cur][u0 + lane] &&
                                                         Gp[min(u0 + lane, rows - 1)] != kInf64);
          if ((live >> lane) & 1u) cp.reach[goff[n] + u0 + lane] = 1;
          while (live) {
            const int u = u0 + __ffs(live) - 1;
            live &= live - 1;
            const uint64_t target = Gp[u];
            for (int v = lane; v < cols; v += 32) {
              const uint64_t a = A[(int64_t)u * cols + v];
              if (a == kInf64 || Gn[v] == kInf64 || a + Gn[v] != target) continue;
              if (v < 256) rc[cur ^ 1][v] = 1;
              const int64_t bit = fo + (int64_t)u * cols + v;
              bool fresh;
              if constexpr (SM) {
                fresh = !(atomicOr(&ebits[bit >> 5], 1u << (bit & 31)) & (1u << (bit & 31)));
              } else {
                fresh = atomicExch(cp.edge_flag + bit, 1) == 0;
              }
              if (fresh) cp.edge_list[atomicAdd(&s_cnt, 1)] = ArgminEntry{mat, u * cols + v};
            }
          }
        }
        __syncwarp();
        cur ^= 1;
      }
      if (lane == 0) *cp.edge_count = s_cnt;
    }
    return;
  }
  if (!cp.backtrack) return;
  TTRACE(0, 13);
  // forward greedy: at each instance the optimal successor with the least
  // combination index.  SM mode: the successor of every (n, u) is tabulated in
  // parallel first, then the walk from u_1 = 0 is a chain of shared loads.
  __shared__ int s_status;
  if (tid == 0) s_status = 0;
  __syncthreads();
  if (SM && cp.mode == 2) {
    // successor of every reachable (n, u) (recorded by mode 1): one warp per
    // instance, lanes over v; then the walk from u_1 = 0 is a chain of loads
    for (int64_t w = tid; w < goff[N]; w += nth) nxt[w] = -1;   // unreachable / no successor
    __syncthreads();
    {
      const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
      for (int n = warp; n < N; n += nw) {
        const int rows = rows_of(n), cols = cols_of(n);
        const uint64_t* Gn = G + goff[n + 1];
        for (int u0 = 0; u0 < rows; u0 += 32) {
         // reachable states of this instance, 32 at a time (one coalesced load)
         unsigned rmask = __ballot_sync(0xffffffffu, u0 + lane < rows && cp.reach[goff[n] + u0 + lane]);
         while (rmask) {
          const int u = u0 + __ffs(rmask) - 1;
          rmask &= rmask - 1;
          const uint64_t* A = matA(n) + (int64_t)u * cols;
          const uint64_t* I = matI(n) + (int64_t)u * cols;
          const uint64_t target = G[goff[n] + u];
          uint64_t bi = kInf64;
          int bv = -1;
          for (int v = lane; v < cols; v += 32) {
            const uint64_t a = A[v], gv = Gn[v];
            if (a == kInf64 || gv == kInf64 || a + gv != target) continue;
            const uint64_t ix = I[v];
            if (ix < bi) { bi = ix; bv = v; }
          }
          for (int off = 16; off > 0; off >>= 1) {
            const uint64_t ob = __shfl_xor_sync(0xffffffffu, bi, off);
            const int ov = __shfl_xor_sync(0xffffffffu, bv, off);
            if (ov >= 0 && (bv < 0 || ob < bi || (ob == bi && ov < bv))) { bi = ob; bv = ov; }
          }
          if (lane == 0) nxt[goff[n] + u] = (int16_t)bv;
         }
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      if (G[0] == kInf64) {
        s_status = 3;
      } else {
        int u = 0;
        for (int n = 0; n < N; ++n) {
          const int v = nxt[goff[n] + u];           // shared-memory chain only
          if (v < 0) { s_status = 3; break; }
          vseq[n] = (u << 16) | v;
          u = v;
        }
      }
    }
    __syncthreads();
    TTRACE(0, 14);
    if (tid == 0) *cp.total = s_status ? kInf64 : G[0];
    if (s_status == 0)
      for (int n = tid; n < N; n += nth) {
        const int u = vseq[n] >> 16, v = vseq[n] & 0xFFFF, cols = cols_of(n);
        cp.seg_index[n] = matI(n)[(int64_t)u * cols + v];
        cp.seg_ns[n] = matA(n)[(int64_t)u * cols + v];
      }
  } else if (tid < 32) {
    const int lane = tid;
    int u = 0;
    if (G[0] == kInf64) {
      if (lane == 0) { s_status = 3; *cp.total = kInf64; }
    } else {
      if (lane == 0) *cp.total = G[0];
      for (int n = 1; n <= N; ++n) {
        const uint64_t* A = matA(n - 1);
        const uint64_t* I = matI(n - 1);
        const int cols = cols_of(n - 1);
        const uint64_t target = G[goff[n - 1] + u];
        const uint64_t* Gn = G + goff[n];
        uint64_t bi = kInf64;
        int bv = -1;
        for (int v = lane; v < cols; v += 32) {
          const uint64_t a = A[(int64_t)u * cols + v];
          if (a == kInf64 || Gn[v] == kInf64 || a + Gn[v] != target) continue;
          const uint64_t ix = I[(int64_t)u * cols + v];
          if (ix < bi) { bi = ix; bv = v; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t ob = __shfl_xor_sync(0xffffffffu, bi, o);
          const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
          if (ob < bi || (ob == bi && ov >= 0 && (bv < 0 || ov < bv))) { bi = ob; bv = ov; }
        }
        if (bv < 0) {
          if (lane == 0) s_status = 3;
          break;
        }
        if (lane == 0) {
          cp.seg_index[n - 1] = bi;
          cp.seg_ns[n - 1] = A[(int64_t)u * cols + bv];
        }
        u = bv;
      }
    }
  }
  __syncthreads();
  TTRACE(0, 15);
  if (tid == 0) *cp.status = s_status;
  if (s_status != 0) return;
  __syncthreads();
  for (int64_t w = tid; w < (int64_t)N * cp.kmax; w += nth) {
    const int n = (int)(w / cp.kmax), j = (int)(w % cp.kmax);
    const ChainInst in = cp.inst[n];
    int32_t dval = -1;
    if (j < in.K) {
      uint64_t stride = 1;
      for (int d = in.K - 1; d > j; --d) stride *= (uint64_t)cp.radix_blob[in.radix_off + d];
      dval = (int32_t)((cp.seg_index[n] / stride) % (uint64_t)cp.radix_blob[in.radix_off + j]);
    }
    cp.digits[w] = dval;
  }
  TTRACE(0, 16);
  __syncthreads();
}

template <bool SM>
__global__ void __launch_bounds__(1024) chain_kernel(const ChainParams cp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  chain_run<SM>(cp, smem_raw, kChainWhole);
}

// --------------------------------------------------------------------------
// Fused tail: the chain on CTA 0 for state counts <= 32 (every layer graph of
// the configs).  Values by repeated squaring + doubling in
// the "big" encoding (INF -> 2^63 - 1, so an add never wraps and needs no INF
// test; results >= 2^63 - 1 are INF); optimal-successor masks of every (n, u)
// by warp ballots in parallel; reachability from u_1 = 0 as a bit walk; the
// reachable optimal edges -> the argmin list.  The backtrack picks, per
// reachable (n, u), the optimal successor with the least combination index.
// --------------------------------------------------------------------------
constexpr uint64_t kBigC = (1ull << 63) - 1;
__device__ __forceinline__ uint64_t big_of(uint64_t x) { return x == kInf64 ? kBigC : x; }
__device__ __forceinline__ uint64_t inf_of(uint64_t x) { return x >= kBigC ? kInf64 : x; }

struct FusedChainSmem {
  uint64_t *A, *G, *P;
  int64_t *goff, *moff;
  int4* inst;                   // (mat, rows, cols, K)
  uint32_t *om, *rmask, *ebits;
  int8_t* nxt;
  int32_t* vseq;
};

__device__ __forceinline__ FusedChainSmem fused_chain_smem(const TailParams& tp, unsigned char* smem) {
  const ChainParams& cp = tp.cp;
  // goff[N] / goff[N + 1] are read from global here (metadata staged below)
  const FusedChainLayout L(cp.mat_elems, cp.goff[cp.N + 1], cp.goff[cp.N], cp.N, cp.nmat, tp.levels, tp.smax);
  FusedChainSmem s;
  s.A = reinterpret_cast<uint64_t*>(smem + L.sA);
  s.G = reinterpret_cast<uint64_t*>(smem + L.sG);
  s.P = reinterpret_cast<uint64_t*>(smem + L.sP);
  s.goff = reinterpret_cast<int64_t*>(smem + L.sgoff);
  s.moff = reinterpret_cast<int64_t*>(smem + L.smoff);
  s.inst = reinterpret_cast<int4*>(smem + L.sinst);
  s.om = reinterpret_cast<uint32_t*>(smem + L.om);
  s.rmask = reinterpret_cast<uint32_t*>(smem + L.rmask);
  s.ebits = reinterpret_cast<uint32_t*>(smem + L.ebits);
  s.nxt = reinterpret_cast<int8_t*>(smem + L.nxt);
  s.vseq = reinterpret_cast<int32_t*>(smem + L.vseq);
  return s;
}

// metadata only (independent of this launch's A): staged before the first barrier
__device__ void fused_chain_meta(const TailParams& tp, const FusedChainSmem& s) {
  const ChainParams& cp = tp.cp;
  const int tid = threadIdx.x, nth = blockDim.x, N = cp.N;
  for (int i = tid; i < N + 2; i += nth) s.goff[i] = cp.goff[i];
  for (int i = tid; i < cp.nmat; i += nth) s.moff[i] = cp.moff[i];
  for (int i = tid; i < N; i += nth) s.inst[i] = make_int4(cp.inst[i].mat, cp.inst[i].rows, cp.inst[i].cols, cp.inst[i].K);
  for (int64_t i = tid; i < (cp.mat_elems + 31) / 32; i += nth) s.ebits[i] = 0;
}

// G_{e-1}[u] = min_v M[u][v] + G_e[v] for one instance (warp per row, lanes = v)
__device__ __forceinline__ void fused_matvec(const uint64_t* M, int R, int Cc, const uint64_t* g, uint64_t* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = warp; u < R; u += (int)(blockDim.x >> 5)) {
    uint64_t x = kBigC;
    if (lane < Cc) x = big_of(M[u * Cc + lane]) + big_of(g[lane]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t y = __shfl_xor_sync(0xffffffffu, x, o);
      x = y < x ? y : x;
    }
    if (lane == 0) out[u] = inf_of(x);
  }
}

__device__ void fused_chain_values(const TailParams& tp, const FusedChainSmem& s) {
  const ChainParams& cp = tp.cp;
  const int tid = threadIdx.x, nth = blockDim.x, N = cp.N;
  for (int64_t e = tid; e < cp.mat_elems; e += nth) s.A[e] = __ldcg(cp.baseA + e);   // other CTAs' writes
  const int lastc = s.inst[N - 1].z;
  for (int v = tid; v < lastc; v += nth) s.G[s.goff[N] + v] = 0;                      // terminal 0 (Q8)
  __syncthreads();
  TTRACE(0, 40);
  for (int r = cp.nruns - 1; r >= 0; --r) {
    const ChainRun run = cp.runs[r];
    TTRACE(0, 41 + min(cp.nruns - 1 - r, 3));
    const int4 in = s.inst[run.first];
    const uint64_t* M = s.A + s.moff[in.x];
    const int R = in.y, Cc = in.z;
    const int e = run.first + run.len;               // G_e known (1-based instance e)
    if (run.len == 1) {
      fused_matvec(M, R, Cc, s.G + s.goff[e], s.G + s.goff[e - 1]);
      __syncthreads();
      continue;
    }
    const int S = R;                                 // square (host: runs need rows == cols)
    int levels = 0;
    while ((1 << (levels + 1)) <= run.len) ++levels;
    const int SS = S * S;
    for (int c = tid; c < SS; c += nth) s.P[c] = big_of(M[c]);
    __syncthreads();
    for (int j = 1; j <= levels; ++j) {              // repeated squaring: P_j = P_{j-1} (x) P_{j-1}
      const uint64_t* Pa = s.P + (int64_t)(j - 1) * SS;
      uint64_t* Pc = s.P + (int64_t)j * SS;
      for (int c = tid; c < SS; c += nth) {
        const int i = c / S, k2 = c - i * S;
        uint64_t b0 = kBigC, b1 = kBigC;
        int k = 0;
        for (; k + 2 <= S; k += 2) {
          const uint64_t x0 = Pa[i * S + k] + Pa[k * S + k2];
          const uint64_t x1 = Pa[i * S + k + 1] + Pa[(k + 1) * S + k2];
          b0 = x0 < b0 ? x0 : b0;
          b1 = x1 < b1 ? x1 : b1;
        }
        if (k < S) { const uint64_t x0 = Pa[i * S + k] + Pa[k * S + k2]; b0 = x0 < b0 ? x0 : b0; }
        b0 = b1 < b0 ? b1 : b0;
        Pc[c] = b0 < kBigC ? b0 : kBigC;
      }
      __syncthreads();
    }
    TTRACE(0, 45);
    for (int j = 0; j <= levels; ++j) {              // doubling: G_{e-k} = P_j (x) G_{e-k+2^j}
      const uint64_t* Pj = s.P + (int64_t)j * SS;
      const int k_lo = 1 << j, k_hi = min(1 << (j + 1), run.len + 1);
      const int work = (k_hi - k_lo) * S;
      for (int w = tid; w < work; w += nth) {
        const int k = k_lo + w / S, u = w - (w / S) * S;
        const uint64_t* g = s.G + s.goff[e - k + (1 << j)];
        const uint64_t* row = Pj + u * S;
        uint64_t b0 = kBigC, b1 = kBigC;
        int v = 0;
        for (; v + 2 <= S; v += 2) {
          const uint64_t x0 = row[v] + big_of(g[v]);
          const uint64_t x1 = row[v + 1] + big_of(g[v + 1]);
          b0 = x0 < b0 ? x0 : b0;
          b1 = x1 < b1 ? x1 : b1;
        }
        if (v < S) { const uint64_t x0 = row[v] + big_of(g[v]); b0 = x0 < b0 ? x0 : b0; }
        b0 = b1 < b0 ? b1 : b0;
        s.G[s.goff[e - k] + u] = inf_of(b0);
      }
      __syncthreads();
    }
  }
  TTRACE(0, 46);
  for (int64_t e2 = tid; e2 < s.goff[N + 1]; e2 += nth) cp.G[e2] = s.G[e2];
}

// u64 minimum over the warp: two 32-bit CREDUX.MIN (high words, then the low
// words of the lanes holding the least high word)
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t x) {
  const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
  const uint32_t hm = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t lm = __reduce_min_sync(0xffffffffu, hi == hm ? lo : 0xFFFFFFFFu);
  return ((uint64_t)hm << 32) | lm;
}

// Sequential backward recurrence G_n(u) = min_v A_n[u][v] + G_{n+1}(v) (the
// textbook DP) with the optimal-successor mask of every (n, u) from
// the same reduction (lanes v attaining the minimum): one warp per row, the
// rows of the current matrix kept in registers across a run of identical
// transitions, one CTA barrier per instance.  On one SM with <= 32 states this
// is cheaper than repeated squaring + doubling (S^3 log L vs S^2 L work, both
// latency-bound): measured in DESIGN.md §5.
__device__ void fused_chain_values_seq(const TailParams& tp, const FusedChainSmem& s) {
  constexpr int NW = kTailThreads / 32;
  constexpr int RPW = (32 + NW - 1) / NW;              // rows per warp (<= 32 rows)
  const ChainParams& cp = tp.cp;
  const int tid = threadIdx.x, nth = blockDim.x, N = cp.N;
  const int warp = tid >> 5, lane = tid & 31;
  for (int64_t e = tid; e < cp.mat_elems; e += nth) s.A[e] = __ldcg(cp.baseA + e);   // other CTAs' writes
  const int lastc = s.inst[N - 1].z;
  for (int v = tid; v < lastc; v += nth) s.G[s.goff[N] + v] = 0;                      // terminal 0 (Q8)
  __syncthreads();
  TTRACE(0, 40);
  int cur = -1;
  uint64_t a[RPW];
  for (int n = N - 1; n >= 0; --n) {
    const int4 in = s.inst[n];
    if (in.x != cur) {
      const uint64_t* M = s.A + s.moff[in.x];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int u = warp + r * NW;
        a[r] = (u < in.y && lane < in.z) ? big_of(M[u * in.z + lane]) : kBigC;
      }
      cur = in.x;
    }
    const int64_t g0 = s.goff[n];
    const uint64_t gv = lane < in.z ? big_of(s.G[s.goff[n + 1] + lane]) : kBigC;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int u = warp + r * NW;
      if (u < in.y) {
        const uint64_t x = a[r] + gv;                  // <= 2^64 - 2: no wrap
        const uint64_t m = warp_min_u64(x);
        const uint32_t mask = __ballot_sync(0xffffffffu, x == m && m < kBigC);
        if (lane == 0) {
          s.G[g0 + u] = inf_of(m);
          s.om[g0 + u] = mask;
        }
      }
    }
    __syncthreads();
  }
  TTRACE(0, 46);
  for (int64_t e2 = tid; e2 < s.goff[N + 1]; e2 += nth) cp.G[e2] = s.G[e2];
}

// optimal-successor masks of every (n, u), reachability from u_1 = 0, and the
// reachable optimal edges (deduplicated per distinct matrix) -> argmin list
__device__ void fused_chain_edges(const TailParams& tp, const FusedChainSmem& s, bool have_om) {
  const ChainParams& cp = tp.cp;
  const int tid = threadIdx.x, nth = blockDim.x, N = cp.N;
  const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
  __shared__ int s_ecnt;
  if (tid == 0) s_ecnt = 0;
  for (int n = have_om ? N : warp; n < N; n += nw) {  // warp per instance, lanes = v
    const int4 in = s.inst[n];
    const int64_t g0 = s.goff[n];
    const uint64_t gv = lane < in.z ? s.G[s.goff[n + 1] + lane] : kInf64;
    const uint64_t* Am = s.A + s.moff[in.x];
    for (int u = 0; u < in.y; ++u) {
      const uint64_t target = s.G[g0 + u];
      const uint64_t a = lane < in.z ? Am[u * in.z + lane] : kInf64;
      const uint32_t m = __ballot_sync(0xffffffffu, target != kInf64 && a != kInf64 && gv != kInf64 &&
                                                        a + gv == target);
      if (lane == 0) s.om[g0 + u] = m;
    }
  }
  __syncthreads();
  TTRACE(0, 47);
  if (tid == 0) {
    uint32_t r = s.G[0] == kInf64 ? 0u : 1u;
    for (int n = 0; n < N; ++n) {
      s.rmask[n] = r;
      uint32_t nx = 0, rr = r;
      const int64_t g0 = s.goff[n];
      while (rr) {
        const int u = __ffs(rr) - 1;
        rr &= rr - 1;
        nx |= s.om[g0 + u];
      }
      r = nx;
    }
  }
  __syncthreads();
  TTRACE(0, 48);
  for (int64_t w = tid; w < (int64_t)N * 32; w += nth) {   // (instance, lane = u)
    const int n = (int)(w >> 5), u = (int)(w & 31);
    if (!((s.rmask[n] >> u) & 1u)) continue;
    const int4 in = s.inst[n];
    const int64_t fo = s.moff[in.x];
    uint32_t m = s.om[s.goff[n] + u];
    while (m) {
      const int v = __ffs(m) - 1;
      m &= m - 1;
      const int64_t bit = fo + (int64_t)u * in.z + v;
      if (!(atomicOr(&s.ebits[bit >> 5], 1u << (bit & 31)) & (1u << (bit & 31))))
        cp.edge_list[atomicAdd(&s_ecnt, 1)] = ArgminEntry{in.x, u * in.z + v};
    }
  }
  __syncthreads();
  if (tid == 0) *cp.edge_count = s_ecnt;
}

// forward greedy: per reachable (n, u) the optimal successor with the least
// combination index (I of the listed buckets, written by the argmin CTAs),
// then the walk from u_1 = 0, the plan outputs and the digit decode
__device__ void fused_backtrack(const TailParams& tp, const FusedChainSmem& s) {
  const ChainParams& cp = tp.cp;
  const int tid = threadIdx.x, nth = blockDim.x, N = cp.N;
  __shared__ int s_stat;
  for (int64_t w = tid; w < (int64_t)N * 32; w += nth) {
    const int n = (int)(w >> 5), u = (int)(w & 31);
    if (!((s.rmask[n] >> u) & 1u)) continue;
    const int4 in = s.inst[n];
    const uint64_t* I = cp.baseI + s.moff[in.x] + (int64_t)u * in.z;
    uint32_t m = s.om[s.goff[n] + u];
    uint64_t bi = kInf64;
    int bv = -1;
    while (m) {
      const int v = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t ix = __ldcg(I + v);             // other CTAs' writes
      if (bv < 0 || ix < bi) { bi = ix; bv = v; }
    }
    s.nxt[s.goff[n] + u] = (int8_t)bv;
  }
  __syncthreads();
  if (tid == 0) {
    int st = 0;
    if (s.G[0] == kInf64) {
      st = 3;
    } else {
      int u = 0;
      for (int n = 0; n < N; ++n) {
        const int v = s.nxt[s.goff[n] + u];
        if (v < 0) { st = 3; break; }
        s.vseq[n] = (u << 16) | v;
        u = v;
      }
    }
    s_stat = st;
    *cp.total = st ? kInf64 : s.G[0];
    *cp.status = st;
  }
  __syncthreads();
  if (s_stat != 0) return;
  for (int n = tid; n < N; n += nth) {
    const int u = s.vseq[n] >> 16, v = s.vseq[n] & 0xFFFF;
    const int4 in = s.inst[n];
    const int64_t at = s.moff[in.x] + (int64_t)u * in.z + v;
    cp.seg_index[n] = __ldcg(cp.baseI + at);
    cp.seg_ns[n] = s.A[at];
  }
  __syncthreads();
  for (int64_t w = tid; w < (int64_t)N * cp.kmax; w += nth) {
    const int n = (int)(w / cp.kmax), j = (int)(w % cp.kmax);
    const int4 in = s.inst[n];
    int32_t dval = -1;
    if (j < in.w) {
      const int ro = cp.inst[n].radix_off;
      uint64_t stride = 1;
      for (int d = in.w - 1; d > j; --d) stride *= (uint64_t)cp.radix_blob[ro + d];
      dval = (int32_t)((cp.seg_index[n] / stride) % (uint64_t)cp.radix_blob[ro + j]);
    }
    cp.digits[w] = dval;
  }
}

// --------------------------------------------------------------------------
// Fused tail (world 1).  One cooperative launch replaces bucket-minima,
// chain mode 1, edge conversion, argmin and chain mode 2 (and the fills and
// memsets between them): the steps are latency-bound and each separate launch
// cost a few microseconds of fixed overhead.
//   phase 1 (all CTAs): A[u][v] = min over the chunk minima for every bucket
//            of every transition in the caller's layout (INF for pruned
//            strategies), I = NOIDX;
//   grid barrier;
//   chain = 1: CTA 0 suffix vectors + reachable optimal edges (shared memory);
//            grid barrier; CTAs 1.. least index of the listed buckets; CTA 0
//            waits for them and runs the forward greedy + digit decode;
//   chain = 0: every CTA takes buckets of the full list (segment tables).
// Grid barrier: arrival counter + generation word; co-residency is
// guaranteed by the cooperative launch.  The kernel leaves sync[] zero.
// --------------------------------------------------------------------------
__device__ __forceinline__ void tail_grid_sync(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  ++gen;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == nblocks * gen) {
      atomicExch(bar + 1, gen);
    } else {
      while (*reinterpret_cast<volatile unsigned int*>(bar + 1) < gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t tail_timer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// min over one bucket's chunk minima: 16-byte loads, several in flight per
// lane (the loop is latency-bound otherwise), then a butterfly min
template <typename V>
__device__ __forceinline__ uint64_t bucket_min(const ArgminParams& ap, int pair, int lane) {
  const V* cm = static_cast<const V*>(ap.f.chunkmin) + (int64_t)pair * ap.f.nchunks;
  const int64_t n = ap.f.nchunks;
  constexpr int VN = Vec4<V>::N;
  V b[4] = {VT<V>::CAP, VT<V>::CAP, VT<V>::CAP, VT<V>::CAP};
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(cm) & 15) == 0) {
    const int64_t nv = n / VN;
    const typename Vec4<V>::T* cv = reinterpret_cast<const typename Vec4<V>::T*>(cm);
#pragma unroll 4
    for (int64_t i = lane; i < nv; i += 32) {
      V x[VN];
      load_vec<V>(reinterpret_cast<const V*>(cv + i), x);
#pragma unroll
      for (int q = 0; q < VN; ++q) b[q] = VT<V>::mn(b[q], x[q]);
    }
    done = nv * VN;
  }
#pragma unroll 4
  for (int64_t c = done + lane; c < n; c += 32) b[0] = VT<V>::mn(b[0], cm[c]);
  V best = VT<V>::mn(VT<V>::mn(b[0], b[1]), VT<V>::mn(b[2], b[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = VT<V>::mn(best, (V)__shfl_xor_sync(0xffffffffu, best, o));
  return best >= VT<V>::CAP ? kInf64 : (uint64_t)best;
}

template <typename V>
__device__ __forceinline__ void tail_argmin(const ArgminParams& ap, int pair, unsigned char* smem, const void* tabs) {
  argmin_pair<V, kTailThreads>(ap, pair, smem, static_cast<const V*>(tabs), sizeof(V) == 4 ? ap.pstar : nullptr);
}

// narrow buckets: the minimum and the least h-block of a chunk attaining it,
// as one min over the keys (value << 32 | hb) -- chunk c = l * nhb + hb
__device__ __forceinline__ uint64_t bucket_min_hb(const ArgminParams& ap, int pair, int lane, int64_t* hb_out) {
  const uint32_t* cm = static_cast<const uint32_t*>(ap.f.chunkmin) + (int64_t)pair * ap.f.nchunks;
  const uint32_t n = (uint32_t)ap.f.nchunks, nhb = (uint32_t)ap.f.nhb;
  uint64_t k0 = ~0ull, k1 = ~0ull;
  uint32_t c = (uint32_t)lane;
#pragma unroll 4
  for (; c + 32 < n; c += 64) {
    const uint32_t x0 = cm[c], x1 = cm[c + 32];
    const uint64_t y0 = ((uint64_t)x0 << 32) | (c % nhb), y1 = ((uint64_t)x1 << 32) | ((c + 32) % nhb);
    k0 = y0 < k0 ? y0 : k0;
    k1 = y1 < k1 ? y1 : k1;
  }
  if (c < n) {
    const uint64_t y0 = ((uint64_t)cm[c] << 32) | (c % nhb);
    k0 = y0 < k0 ? y0 : k0;
  }
  k0 = k1 < k0 ? k1 : k0;
  k0 = warp_min_u64(k0);
  const uint32_t best = (uint32_t)(k0 >> 32);
  *hb_out = best >= kCap32 ? -1 : (int64_t)(k0 & 0xFFFFFFFFu);
  return best >= kCap32 ? kInf64 : (uint64_t)best;
}

// worker CTAs: copies of every slot's argmin descriptor and W/R tables in
// shared memory (done while CTA 0 runs the chain, off the critical path)
__device__ void tail_stage_argmin(const TailParams& tp, unsigned char* smem) {
  const int tid = threadIdx.x, nth = blockDim.x;
  ArgminParams* desc = reinterpret_cast<ArgminParams*>(smem + tp.arg_desc_off);
  {
    const int words = (int)(sizeof(ArgminParams) / 4) * tp.nslot;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(tp.aps);
    uint32_t* dst = reinterpret_cast<uint32_t*>(desc);
    for (int i = tid; i < words; i += nth) dst[i] = src[i];
  }
  for (int q = 0; q < tp.nslot; ++q) {
    const ArgminParams& ap = tp.aps[q];
    if (ap.f.nchunks == 0) continue;
    const int n = ap.e.tab_n;
    if (ap.wide) {
      const uint64_t* v = static_cast<const uint64_t*>(ap.f.vals) + ap.e.tab_lo;
      uint64_t* d = reinterpret_cast<uint64_t*>(smem + tp.arg_tab_off[q]);
      for (int i = tid; i < n; i += nth) d[i] = v[i];
    } else {
      const uint32_t* v = static_cast<const uint32_t*>(ap.f.vals) + ap.e.tab_lo;
      uint32_t* d = reinterpret_cast<uint32_t*>(smem + tp.arg_tab_off[q]);
      for (int i = tid; i < n; i += nth) d[i] = v[i];
    }
  }
}

__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(const TailParams tp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned int G = gridDim.x;
  unsigned int gen = 0;
  const bool ts = tp.phase_ts != nullptr && blockIdx.x == 0 && tid == 0;
  if (ts) tp.phase_ts[0] = tail_timer();
  TTRACE(0, 30);
  FusedChainSmem cs{};
  if (tp.chain && blockIdx.x == 0) {
    cs = fused_chain_smem(tp, smem_raw);
    fused_chain_meta(tp, cs);                       // independent of this launch's A
  }
  // ---- phase 1: bucket minima (warp per caller-layout bucket), I = NOIDX
  {
    const int64_t total = tp.orig_off[tp.nslot];
    const int64_t nw = (int64_t)G * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (tid >> 5); w < total; w += nw) {
      int s = 0;
      while (w >= tp.orig_off[s + 1]) ++s;
      const ArgminParams& ap = tp.aps[s];
      const int po = (int)(w - tp.orig_off[s]);
      const int u = po / ap.Do_orig, vo = po - u * ap.Do_orig;
      const int vc = ap.f.nchunks > 0 ? ap.vinv[vo] : -1;   // empty types: no maps
      uint64_t a = kInf64;
      if (vc >= 0) {
        const int pair = u * ap.f.Do + vc;
        if (ap.wide) {
          a = bucket_min<uint64_t>(ap, pair, lane);
        } else {
          int64_t hb;
          a = bucket_min_hb(ap, pair, lane, &hb);
          if (lane == 0) ap.pstar[pair] = hb;
        }
      }
      if (lane == 0) {
        ap.A_out[po] = a;
        ap.I_out[po] = kInf64;
      }
    }
  }
  if (!tp.chain) {
    tail_stage_argmin(tp, smem_raw);
  }
  tail_grid_sync(tp.sync, G, gen);
  if (ts) tp.phase_ts[1] = tail_timer();
  TTRACE(0, 31);
  if (tp.chain) {
    if (blockIdx.x == 0) {
      if (tp.squaring) fused_chain_values(tp, cs);
      else fused_chain_values_seq(tp, cs);
      TTRACE(0, 10);
      fused_chain_edges(tp, cs, !tp.squaring);
      TTRACE(0, 12);
    } else {
      tail_stage_argmin(tp, smem_raw);
    }
    tail_grid_sync(tp.sync, G, gen);
    if (ts) tp.phase_ts[2] = tail_timer();
    TTRACE(0, 32);
    TTRACE(1, 33);
    if (blockIdx.x > 0) {
#ifdef CFP_TAIL_TRACE
      uint64_t t_w0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w0));
#endif
      const ArgminParams* desc = reinterpret_cast<const ArgminParams*>(smem_raw + tp.arg_desc_off);
      const int n = __ldcg(tp.cp.edge_count);
      for (int it = (int)blockIdx.x - 1; it < n; it += (int)G - 1) {
        const long long raw = __ldcg(reinterpret_cast<const long long*>(tp.cp.edge_list) + it);   // CTA 0's writes
        const ArgminEntry en{(int32_t)(raw & 0xFFFFFFFFll), (int32_t)(raw >> 32)};
        const ArgminParams& ap = desc[en.slot];
        const int u = en.pair / ap.Do_orig, vo = en.pair - u * ap.Do_orig;
        const int vc = ap.vinv[vo];
        const int pair = vc < 0 ? 0 : u * ap.f.Do + vc;     // pruned columns are INF: never optimal
        const void* tabs = smem_raw + tp.arg_tab_off[en.slot];
        if (ap.wide) tail_argmin<uint64_t>(ap, pair, smem_raw, tabs);
        else tail_argmin<uint32_t>(ap, pair, smem_raw, tabs);
        __syncthreads();
      }
      __syncthreads();
      TTRACE(1, 36);
#ifdef CFP_TAIL_TRACE
      if (tid == 0 && blockIdx.x < 256) {
        uint64_t t_w1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w1));
        g_trace_cta[blockIdx.x] = t_w1 - t_w0;
      }
#endif
      if (tid == 0) {
        __threadfence();
        atomicAdd(tp.sync + 2, 1u);
      }
      return;
    }
    if (tid == 0) {
      while (*reinterpret_cast<volatile unsigned int*>(tp.sync + 2) < G - 1) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    if (ts) tp.phase_ts[3] = tail_timer();
    TTRACE(0, 34);
    fused_backtrack(tp, cs);
    __syncthreads();
    if (tid == 0) {                                 // every other CTA is past its last barrier
      tp.sync[0] = 0u;
      tp.sync[1] = 0u;
      tp.sync[2] = 0u;
      if (ts) tp.phase_ts[4] = tail_timer();
    }
    TTRACE(0, 35);
    return;
  }
  const ArgminParams* desc = reinterpret_cast<const ArgminParams*>(smem_raw + tp.arg_desc_off);
  const int64_t npairs = tp.pair_off[tp.nslot];
  for (int64_t it = blockIdx.x; it < npairs; it += G) {
    int s = 0;
    while (it >= tp.pair_off[s + 1]) ++s;
    const ArgminParams& ap = desc[s];
    const int pair = (int)(it - tp.pair_off[s]);
    const void* tabs = smem_raw + tp.arg_tab_off[s];
    if (ap.wide) tail_argmin<uint64_t>(ap, pair, smem_raw, tabs);
    else tail_argmin<uint32_t>(ap, pair, smem_raw, tabs);
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(tp.sync + 2, 1u) == G - 1) {      // last CTA: everyone is past the barriers
      tp.sync[0] = 0u;
      tp.sync[1] = 0u;
      tp.sync[2] = 0u;
    }
  }
}

// --------------------------------------------------------------------------
// N5: integer-pipe microbenchmark (roofline denominator).
// --------------------------------------------------------------------------
template <int OP>
__global__ void __launch_bounds__(1024) intpipe_kernel(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[8], y[8];
  uint64_t a64[8], y64[8];
  uint32_t x = seed ^ (threadIdx.x * 2654435761u) ^ (uint32_t)clock64();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = 0xFFFFFFFFu - i * x; y[i] = x * (i + 3);
    a64[i] = ~0ull - i * (uint64_t)x; y64[i] = (uint64_t)x * (i + 5);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = __viaddmin_u32(x, y[i], a[i]);
        else if (OP == 1) a[i] = a[i] + y[i] + x;
        else { const uint64_t s = (uint64_t)x + y64[i]; a64[i] = s < a64[i] ? s : a64[i]; }
      }
      x += 0x9E3779B9u;
      if (OP == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] ^= a[i];
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i] ^ (uint32_t)a64[i];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

// N5 op 3: the enumeration's full-A step on two pipes, as in enum_kernel
// (24 accumulators, the step's 24 x values in registers, y rows streamed from
// shared memory 4 at a time; per 3 combinations one VIADDMNMX, two FMA-pipe
// IMAD adds and one VIMNMX3), 4 CTAs x 256 threads per SM.  576 add+mins per
// step.
__global__ void __launch_bounds__(256, 4) intpipe_mix_kernel(uint32_t* out, int iters, uint32_t one) {
  __shared__ __align__(16) uint32_t xs[64 * 24];
  __shared__ __align__(16) uint32_t ys[64 * 24];
  for (int i = threadIdx.x; i < 64 * 24; i += 256) {
    xs[i] = (i * 2654435761u) & 0x3FFFFFFFu;
    ys[i] = (i * 40503u + 17u) & 0x3FFFFFFFu;
  }
  __syncthreads();
  uint32_t acc[24];
#pragma unroll
  for (int j = 0; j < 24; ++j) acc[j] = 0x7FFFFFFFu - threadIdx.x - j;
  for (int it = 0; it < iters; ++it) {
    const int m = it & 63;
    uint32_t x[24];
#pragma unroll
    for (int a = 0; a < 24; a += 4) load_vec<uint32_t>(xs + m * 24 + a, x + a);
#pragma unroll
    for (int j0 = 0; j0 < 24; j0 += 4) {
      uint32_t y[4];
      load_vec<uint32_t>(ys + m * 24 + j0, y);
#pragma unroll
      for (int a = 0; a < 24; a += 3)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          acc[j0 + q] = __vimin3_u32(__viaddmin_u32(x[a], y[q], acc[j0 + q]), mad_fma(x[a + 1], one, y[q]),
                                     mad_fma(x[a + 2], one, y[q]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 24; ++j) s ^= acc[j];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

// ===================== launchers (called from cfp_host.cu) =================
#define CFP_LAUNCH_CHECK() do { cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return e_; } while (0)

template <typename V>
cudaError_t launch_compact(const CompactJob* jobs, int njobs, const uint32_t* raw, const int32_t* maps,
                           V* out, cudaStream_t st) {
  if (njobs == 0) return cudaSuccess;
  compact_kernel<V><<<njobs, 256, 0, st>>>(jobs, raw, maps, out);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template <typename V>
cudaError_t launch_build_tables(const TableSpec* specs, int nspecs, int64_t max_entries, const V* vals,
                                V* out, cudaStream_t st) {
  if (nspecs == 0) return cudaSuccess;
  // max_entries carries the total CTA count (sum of the tables' nblocks)
  build_table_kernel<V><<<(unsigned)max_entries, 256, 0, st>>>(specs, nspecs, vals, out);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template <typename V>
cudaError_t launch_fill(V* p, int64_t n, V v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  fill_kernel<V><<<(unsigned)blocks, 256, 0, st>>>(p, n, v);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template <typename V, int NB>
cudaError_t launch_enum_nb(const EnumParams& p, int64_t nthreads, size_t smem, cudaStream_t st) {
  (void)nthreads;
  const int64_t blocks = p.W * p.VG * (p.Gpad / p.CH);
  if (blocks <= 0) return cudaSuccess;
  const size_t sm = std::max(smem, (size_t)p.smem_epi);
  auto launch = [&](auto kern) -> cudaError_t {
    if (sm > 40 * 1024) {                          // opt in above the 48 KB default (static smem counts too)
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
    }
    // maximum shared-memory carveout: four CTAs of the fold epilogue per SM
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e2 != cudaSuccess) return e2;
    kern<<<(unsigned)blocks, kBlock, sm, st>>>(p);
    return cudaGetLastError();
  };
  if (p.MS == 2) {                                  // host: B = {o}, staged + merged Y
    if (!(p.staged && p.ymerge)) return cudaErrorInvalidValue;
    return launch(enum_kernel<V, NB, 2, 2>);
  }
  if constexpr (sizeof(V) == 4 && (NB == 23 || NB == 24)) {
    if (p.staged && p.ymerge && p.na == NB && p.na_pad >= (NB + 3) / 4 * 4 && !p.no_full_a) {
      if (p.mix == 3 && NB == 23 && p.o_mode == 1) return launch(enum_kernel<V, NB, 2, 1, NB, 0, 3>);
      if (p.mix == 3) return launch(enum_kernel<V, NB, 2, 1, NB, 1, 3>);
      if (p.mix == 4) return launch(enum_kernel<V, NB, 2, 1, NB, 1, 4>);
      if (NB == 23 && p.o_mode == 1) return launch(enum_kernel<V, NB, 2, 1, NB, 0>);
      return launch(enum_kernel<V, NB, 2, 1, NB>);
    }
  }
  if (p.staged && p.ymerge) return launch(enum_kernel<V, NB, 2, 1>);
  if (p.staged) return launch(enum_kernel<V, NB, 1, 1>);
  return launch(enum_kernel<V, NB, 0, 1>);
}

template <typename V>
cudaError_t launch_enum(const EnumParams& p, int NB, int64_t nthreads, size_t smem, cudaStream_t st) {
  switch (NB) {
    case 4: return launch_enum_nb<V, 4>(p, nthreads, smem, st);
    case 8: return launch_enum_nb<V, 8>(p, nthreads, smem, st);
    case 12: return launch_enum_nb<V, 12>(p, nthreads, smem, st);
    case 16: return launch_enum_nb<V, 16>(p, nthreads, smem, st);
    case 23: return launch_enum_nb<V, 23>(p, nthreads, smem, st);
    case 24: return launch_enum_nb<V, 24>(p, nthreads, smem, st);
    case 32: return launch_enum_nb<V, 32>(p, nthreads, smem, st);
    default: return cudaErrorInvalidValue;
  }
}



template <typename V>
cudaError_t launch_argmin(const ArgminParams* aps, const ArgminEntry* list, const int32_t* count, int grid,
                          int kmax, int tabn_max, cudaStream_t st) {
  const size_t smem = (((size_t)kmax * 256 * 2 + 15) & ~(size_t)15) + (size_t)tabn_max * sizeof(V) + 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(argmin_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  argmin_kernel<V><<<grid, 256, smem, st>>>(aps, list, count, sizeof(V) == 8 ? 1 : 0);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template <typename V>
cudaError_t launch_amin(const ArgminParams* aps, const int64_t* pair_off, int nslot, int64_t total,
                        cudaStream_t st) {
  if (total <= 0) return cudaSuccess;
  amin_kernel<V><<<(unsigned)((total * 32 + 255) / 256), 256, 0, st>>>(aps, pair_off, nslot, sizeof(V) == 8 ? 1 : 0);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

cudaError_t launch_all_pairs(const int64_t* pair_off, int nslot, int64_t total, ArgminEntry* list, int32_t* count,
                             cudaStream_t st) {
  all_pairs_kernel<<<(unsigned)((total + 255) / 256 + 1), 256, 0, st>>>(pair_off, nslot, list, count);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

cudaError_t launch_edges_to_pairs(const ArgminParams* aps, ArgminEntry* list, const int32_t* count, int64_t cap,
                                  cudaStream_t st) {
  edges_to_pairs_kernel<<<(unsigned)((cap + 255) / 256 + 1), 256, 0, st>>>(aps, list, count);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

cudaError_t launch_chain(const ChainParams& cp, cudaStream_t st) {
  if (cp.smem_bytes > 0) {
    if (cp.smem_bytes > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)cp.smem_bytes);
      if (e != cudaSuccess) return e;
    }
    chain_kernel<true><<<1, 1024, (size_t)cp.smem_bytes, st>>>(cp);
  } else {
    chain_kernel<false><<<1, 1024, 0, st>>>(cp);
  }
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}



// co-resident CTAs of the tail kernel for a dynamic shared-memory size (cooperative launch bound)
cudaError_t tail_max_blocks(size_t smem, int* per_sm) {
  cudaError_t e = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, tail_kernel, kTailThreads, smem);
}

// one cooperative launch (grid <= co-resident CTAs, checked by the host)
cudaError_t launch_tail(const TailParams& tp, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<TailParams*>(&tp)};
  return cudaLaunchCooperativeKernel((void*)tail_kernel, dim3((unsigned)grid), dim3(kTailThreads), args, smem, st);
}

#ifdef CFP_TAIL_TRACE
extern "C" int cfp_debug_trace(uint64_t* out64) {
  int e = (int)cudaMemcpyFromSymbol(out64, g_trace, 64 * sizeof(uint64_t));
  if (e) return e;
  e = (int)cudaMemcpyFromSymbol(out64 + 64, g_trace_cta, 256 * sizeof(uint64_t));
  if (e) return e;
  return (int)cudaMemcpyFromSymbol(out64 + 320, g_enum_trace, 4096 * 8 * sizeof(uint64_t));
}
#endif

cudaError_t launch_intpipe(int op, int blocks, int iters, uint32_t* out, cudaStream_t st) {
  if (op == 0) intpipe_kernel<0><<<blocks, 1024, 0, st>>>(out, iters, 7u);
  else if (op == 1) intpipe_kernel<1><<<blocks, 1024, 0, st>>>(out, iters, 7u);
  else if (op == 3) intpipe_mix_kernel<<<blocks * 2, 256, 0, st>>>(out, iters, 1u);   // 4 x 256 per SM
  else intpipe_kernel<2><<<blocks, 1024, 0, st>>>(out, iters, 7u);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template cudaError_t launch_compact<uint32_t>(const CompactJob*, int, const uint32_t*, const int32_t*, uint32_t*, cudaStream_t);
template cudaError_t launch_compact<uint64_t>(const CompactJob*, int, const uint32_t*, const int32_t*, uint64_t*, cudaStream_t);
template cudaError_t launch_build_tables<uint32_t>(const TableSpec*, int, int64_t, const uint32_t*, uint32_t*, cudaStream_t);
template cudaError_t launch_build_tables<uint64_t>(const TableSpec*, int, int64_t, const uint64_t*, uint64_t*, cudaStream_t);
template cudaError_t launch_fill<uint32_t>(uint32_t*, int64_t, uint32_t, cudaStream_t);
template cudaError_t launch_fill<uint64_t>(uint64_t*, int64_t, uint64_t, cudaStream_t);
template cudaError_t launch_enum<uint32_t>(const EnumParams&, int, int64_t, size_t, cudaStream_t);
template cudaError_t launch_enum<uint64_t>(const EnumParams&, int, int64_t, size_t, cudaStream_t);
template cudaError_t launch_argmin<uint32_t>(const ArgminParams*, const ArgminEntry*, const int32_t*, int, int, int, cudaStream_t);
template cudaError_t launch_argmin<uint64_t>(const ArgminParams*, const ArgminEntry*, const int32_t*, int, int, int, cudaStream_t);
template cudaError_t launch_amin<uint32_t>(const ArgminParams*, const int64_t*, int, int64_t, cudaStream_t);
template cudaError_t launch_amin<uint64_t>(const ArgminParams*, const int64_t*, int, int64_t, cudaStream_t);

}  // namespace cfp
