// cfp_kernels.cu -- sm_100a kernels of the CFP plan-search hot path.
//
// Hot path and where each step lives:
//   a0 stage:       compact_kernel (prune + p+c), build_table_kernel (X/Y/Z/K0)
//   a1 enumerate:   enum_kernel  -- one VIADDMNMX per strategy combination
//   a1 fold:        fold_kernel  -- cross-segment terms Q_j[u][s_j] folded per
//                                   prefix: A[u][v] = min_p X_p[u] + B_p[v]
//   a1 argmin:      fold_reduce_kernel + suffix_argmin_kernel -- least index
//   a2 merge:       NCCL min-allreduce on packed keys (host side, world > 1)
//   a3 chain:       chain_kernel -- (min,+) powers by repeated squaring,
//                                   suffix vectors by doubling
//   a4 backtrack:   chain_kernel (forward greedy) + plan decode
// Everything is exact integer arithmetic; the narrow path keeps values in
// [0, CAP32] with CAP32 = 2^31-1 meaning "infeasible" (any sum >= CAP is
// infeasible, guaranteed by the host's bound check), so the fused
// add+min never wraps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cfp_internal.h"

namespace cfp {

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
  const int64_t n = (int64_t)j.rows * j.cols;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int32_t r = (int32_t)(e / j.cols), c = (int32_t)(e % j.cols);
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
__global__ void build_table_kernel(const TableSpec* __restrict__ specs, const V* __restrict__ vals,
                                   V* __restrict__ out) {
  const TableSpec& s = specs[blockIdx.y];
  const int64_t total = s.rows * s.row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / s.row, c = e % s.row;
    V acc = 0;
    if (c >= s.row_valid) {
      acc = VT<V>::CAP;
    } else {
      int32_t dig[kMaxDigits];
      int64_t q = r * s.row_valid + c;
      for (int d = s.ndig - 1; d >= 0; --d) {
        dig[d] = (int32_t)(q % s.radix[d]);
        q /= s.radix[d];
      }
      for (int t = 0; t < s.nterm; ++t) {
        const Term& tm = s.term[t];
        const V v = tm.kind == 0 ? vals[tm.off + dig[tm.a]]
                                 : vals[tm.off + (int64_t)dig[tm.a] * tm.db + dig[tm.b]];
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
__device__ __forceinline__ void atomic_min_v(V* p, V v);
template <>
__device__ __forceinline__ void atomic_min_v<uint32_t>(uint32_t* p, uint32_t v) { atomicMin(p, v); }
template <>
__device__ __forceinline__ void atomic_min_v<uint64_t>(uint64_t* p, uint64_t v) {
  atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// CTA = (group g = (low prefix part l, register group vg), h-block hb of
// kBlock prefixes); thread = one prefix.  After the enumeration the CTA holds
// the complete B_p[v] of its prefixes and folds the cross-segment terms of
// every incoming transition into this chunk's minima (epilogue):
//    chunkmin_t[u][v][chunk] = min_{p in chunk} X^t_p[u] + B_p[v],
//    X^t_p[u] = sum_{cross (j, Q)} Q[u][s_j(p)]          (Eq. 3 r_n)
// with 4x4 register-blocked fused add+mins over the chunk's rows.
template <typename V, int NB, bool STAGED>
__global__ void __launch_bounds__(kBlock) enum_kernel(const EnumParams p) {
  using T = VT<V>;
  constexpr int VN = Vec4<V>::N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int64_t nhb = p.Gpad / kBlock;
  const int64_t g = blockIdx.x / nhb;
  const int64_t hb = blockIdx.x - g * nhb;
  const int64_t l = g / p.VG;
  const int vg = (int)(g - l * p.VG);
  const int64_t hh = hb * kBlock + tid;
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
  if constexpr (STAGED) {
    V* xs = reinterpret_cast<V*>(smem_raw);
    V* ys = xs + p.xspan;
    V* zs = ys + p.yspan;
    int4* ms = reinterpret_cast<int4*>(zs + ((p.zspan + 3) & ~3LL));
    for (int64_t e = tid * VN; e < p.xspan; e += kBlock * VN)
      *reinterpret_cast<typename Vec4<V>::T*>(xs + e) =
          *reinterpret_cast<const typename Vec4<V>::T*>(XT + sx + e);
    for (int64_t e = tid * VN; e < p.yspan; e += kBlock * VN)
      *reinterpret_cast<typename Vec4<V>::T*>(ys + e) =
          *reinterpret_cast<const typename Vec4<V>::T*>(YT + sy + e);
    for (int64_t e = tid; e < p.zspan; e += kBlock) zs[e] = ZT[sz + e];
    for (int64_t e = tid; e < p.nM; e += kBlock) ms[e] = MT[e];
    __syncthreads();
    XT = xs; YT = ys; ZT = zs; MT = ms;
    sx = sy = sz = 0;
  }
  V* Bp = static_cast<V*>(p.Bp) + row * p.Do;
  V acc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j] = T::CAP;
  const int ybase = vg * NB;
  if (live) {
    if (p.init_row)
      for (int v = 0; v < p.Do; ++v) Bp[v] = T::CAP;
    const V k0 = static_cast<const V*>(p.K0)[pg];
    for (int64_t m = 0; m < p.nM; ++m) {
      const int4 mt = MT[m];
      const V km = T::sat(k0, ZT[sz + mt.z]);
      const V* yr = YT + sy + mt.y + ybase;
      V y[NB];
#pragma unroll
      for (int j = 0; j < NB; j += VN) load_vec<V>(yr + j, y + j);
#pragma unroll
      for (int j = 0; j < NB; ++j) y[j] = T::sat(y[j], km);
      const V* xr = XT + sx + mt.x;
#pragma unroll 2
      for (int a = 0; a < p.na_pad; a += VN) {
        V x[VN];
        load_vec<V>(xr + a, x);
#pragma unroll
        for (int q = 0; q < VN; ++q)
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = T::addmin(x[q], y[j], acc[j]);
      }
      if (p.o_mode == 1) {                        // bucket digit in M: flush per m
        V r = acc[0];
#pragma unroll
        for (int j = 1; j < NB; ++j) r = T::mn(r, acc[j]);
        Bp[mt.w] = T::mn(Bp[mt.w], r);
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[j] = T::CAP;
      }
    }
    if (p.o_mode == 0) {
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
  if (p.ntau == 0) return;
  // ---- epilogue: fold the cross-segment terms of every incoming transition
  __syncthreads();                                // staged tables no longer needed
  const bool simple = p.o_mode == 0 && p.o_bstride == 1 && p.o_bradix == p.nb;
  const int v_lo = simple ? ybase : 0;
  const int v_cnt = simple ? min(NB, p.nb - ybase) : p.Do;
  const int VP = (v_cnt + 3) & ~3;
  V* Bs = reinterpret_cast<V*>(smem_raw);                     // [kBlock][VP]
  V* Xs = Bs + kBlock * VP;                                   // [kBlock][DinP] (red afterwards)
  if (simple) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j < VP) Bs[tid * VP + j] = (live && j < v_cnt) ? acc[j] : T::CAP;
  } else {
    for (int j = 0; j < VP; ++j) Bs[tid * VP + j] = (live && j < v_cnt) ? Bp[j] : T::CAP;
  }
  const V* vals = static_cast<const V*>(p.vals);
  const int64_t chunk = l * nhb + hb;
  int dinp_max = 4;
  for (int t = 0; t < p.ntau; ++t) dinp_max = max(dinp_max, (p.taus[t].Din + 3) & ~3);
  for (int t = 0; t < p.ntau; ++t) {
    const EpiTau& et = p.taus[t];
    const int Din = et.Din, DinP = (Din + 3) & ~3;
    for (int u = 0; u < DinP; ++u) Xs[tid * DinP + u] = T::CAP;
    if (live) {
      for (int u = 0; u < Din; ++u) Xs[tid * DinP + u] = 0;
      for (int i = 0; i < et.nq; ++i) {
        const Term& q = et.q[i];
        const int dig = pg < 0x7FFFFFFF
                            ? (int)(((uint32_t)pg / (uint32_t)p.pre_stride[q.a]) % (uint32_t)p.pre_radix[q.a])
                            : (int)((pg / p.pre_stride[q.a]) % p.pre_radix[q.a]);
        const V* Q = vals + q.off + dig;
        for (int u = 0; u < Din; ++u) Xs[tid * DinP + u] = T::sat(Xs[tid * DinP + u], Q[(int64_t)u * q.db]);
      }
    }
    __syncthreads();
    const int nblk = (DinP / 4) * (VP / 4);
    const int stripes = nblk >= kBlock ? 1 : min(8, kBlock / nblk);
    V res[4][4];
    int u0 = 0, v0 = 0;
    const int gi = tid / nblk;
    const bool active = nblk >= kBlock ? tid < nblk : gi < stripes;
    // (nblk > kBlock handled by the loop below)
    for (int blk = (nblk >= kBlock ? tid : tid - gi * nblk); active && blk < nblk;
         blk += (nblk >= kBlock ? kBlock : nblk)) {
      u0 = (blk / (VP / 4)) * 4;
      v0 = (blk % (VP / 4)) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) res[i][j] = T::CAP;
      const int rs = stripes > 1 ? gi : 0;
      for (int r = rs; r < kBlock; r += stripes) {
        V x[4], y[4];
        load_vec<V>(Xs + r * DinP + u0, x);
        if (VN == 2) load_vec<V>(Xs + r * DinP + u0 + 2, x + 2);
        load_vec<V>(Bs + r * VP + v0, y);
        if (VN == 2) load_vec<V>(Bs + r * VP + v0 + 2, y + 2);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) res[i][j] = T::addmin(x[i], y[j], res[i][j]);
      }
      if (nblk >= kBlock) {                         // one stripe: write straight out
        V* out = static_cast<V*>(et.chunkmin);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (u0 + i < Din && v0 + j < v_cnt)
              out[((int64_t)(u0 + i) * p.Do + v_lo + v0 + j) * p.nchunks + chunk] = res[i][j];
      }
      if (stripes > 1) break;
    }
    __syncthreads();                                 // Xs free -> stripe partials
    if (nblk < kBlock) {
      V* red = stripes * VP <= kBlock ? Xs : Xs + kBlock * dinp_max;   // [stripes][DinP][VP]
      if (active) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) red[(gi * DinP + u0 + i) * VP + v0 + j] = res[i][j];
      }
      __syncthreads();
      V* out = static_cast<V*>(et.chunkmin);
      for (int e = tid; e < Din * v_cnt; e += kBlock) {
        const int u = e / v_cnt, vv = e - u * v_cnt;
        V m = red[u * VP + vv];
        for (int s = 1; s < stripes; ++s) m = T::mn(m, red[(s * DinP + u) * VP + vv]);
        out[((int64_t)u * p.Do + v_lo + vv) * p.nchunks + chunk] = m;
      }
      __syncthreads();
    }
  }
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

// Persistent fold over all transitions into one segment type (they share
// B_p).  The local prefixes are cut into chunks of CH rows; CTA c owns a
// contiguous run of chunks.  Per chunk: B_p rows arrive by double-buffered
// TMA bulk copies; X_p[u] is built from the prefix's digit structure -- rows
// sharing all but the last prefix digit ("group") share Xhi[u] = the cross
// terms on the other digits, so X_p[u] = Xhi[u] + sum of the last-digit terms
// (1-2 shared loads per entry); then each thread folds a 4x4 (u, v) block
// over a stripe of the rows (two 4-wide shared loads per 16 fused add+mins)
// and the stripes are reduced into chunkmin_t[(u * Do + v) * nchunks + chunk].
template <typename V>
__global__ void __launch_bounds__(256) fold_kernel(const FoldMulti fm) {
  using T = VT<V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FoldSmem L = fold_layout(fm, (int)sizeof(V));
  const FoldParams& f0 = fm.f[0];
  const int Do = f0.Do, DoP = L.DoP, CH = L.CH, Dl = L.Dl, P = f0.P;
  V* bs = reinterpret_cast<V*>(smem_raw + L.bs);
  __shared__ __align__(8) uint64_t mbar[2];
  const int tid = threadIdx.x;
  const int64_t nch = f0.nchunks;
  const int64_t c_lo = blockIdx.x * nch / gridDim.x, c_hi = (blockIdx.x + 1) * nch / gridDim.x;
  const V* Bp = static_cast<const V*>(f0.Bp);
  const V* vals = static_cast<const V*>(f0.vals);
  const bool tma = f0.tma && DoP == Do;
  for (int t = 0; t < fm.ntau; ++t) {                 // Q tables -> smem
    const FoldParams& f = fm.f[t];
    V* qs = reinterpret_cast<V*>(smem_raw + L.qs[t]);
    int qo = 0;
    for (int i = 0; i < f.nq; ++i) {
      const int ne = f.Din * f.q[i].db;
      for (int e = tid; e < ne; e += 256) qs[qo + e] = vals[f.q[i].off + e];
      qo += ne;
    }
  }
  if (tma && tid == 0) { mbar_init(&mbar[0], 1); mbar_init(&mbar[1], 1); }
  __syncthreads();
  for (int t = 0; t < fm.ntau; ++t) {                 // QL[u][s]: cross terms on the last digit
    const FoldParams& f = fm.f[t];
    const V* qs = reinterpret_cast<const V*>(smem_raw + L.qs[t]);
    V* ql = reinterpret_cast<V*>(smem_raw + L.ql[t]);      // [s][u] (u contiguous)
    for (int e = tid; e < L.DinP[t] * Dl; e += 256) {
      const int s = e / L.DinP[t], u = e - s * L.DinP[t];
      V x = u < f.Din ? (V)0 : T::CAP;
      if (u < f.Din) {
        int qo = 0;
        for (int i = 0; i < f.nq; ++i) {
          if (f.q[i].a == P - 1) x = T::sat(x, qs[qo + u * f.q[i].db + s]);
          qo += f.Din * f.q[i].db;
        }
      }
      ql[e] = x;
    }
  }
  int32_t* rg = reinterpret_cast<int32_t*>(smem_raw + L.rows);
  int32_t* rs = rg + CH;
  int32_t* gdig = reinterpret_cast<int32_t*>(smem_raw + L.gdig);
  auto rows_of = [&](int64_t ch) { return (int)min((int64_t)CH, f0.nPl - ch * CH); };
  auto issue = [&](int64_t ch, int buf) {             // B_p rows of chunk ch -> bs[buf]
    const int64_t p0 = ch * CH;
    const int n = rows_of(ch);
    V* dst = bs + (int64_t)buf * CH * DoP;
    if (tma) {
      if (tid == 0) {
        const uint32_t bytes = (uint32_t)((int64_t)n * Do * sizeof(V));
        mbar_expect_tx(&mbar[buf], bytes);
        tma_bulk_g2s(dst, Bp + p0 * Do, bytes, &mbar[buf]);
      }
    } else {
      for (int e = tid; e < n * DoP; e += 256) {
        const int pi = e / DoP, v = e - pi * DoP;
        dst[e] = v < Do ? Bp[(p0 + pi) * Do + v] : T::CAP;
      }
    }
  };
  if (c_lo < c_hi) issue(c_lo, 0);
  uint32_t phases = 0;                               // bit b = parity of mbar[b]
  const int gi = tid / L.nblk_all;
  for (int64_t ch = c_lo; ch < c_hi; ++ch) {
    const int buf = (int)((ch - c_lo) & 1);
    const int64_t p0 = ch * CH;
    const int n = rows_of(ch);
    if (ch + 1 < c_hi) issue(ch + 1, buf ^ 1);         // buffer freed by the previous chunk's last sync
    const int64_t pg0 = f0.p_lo + p0;
    const int64_t grp0 = pg0 / Dl;
    const int ng = (int)((pg0 + n - 1) / Dl - grp0 + 1);
    // per row: (group, last digit); per group: the digits the other cross terms read
    const int s0 = (int)(pg0 - grp0 * Dl);          // last digit of the chunk's first row
    for (int pi = tid; pi < n; pi += 256) {
      const int g = (s0 + pi) / Dl;
      rg[pi] = g;
      rs[pi] = s0 + pi - g * Dl;
    }
    for (int t = 0, col = 0; t < fm.ntau; ++t)
      for (int i = 0; i < fm.f[t].nq; ++i, ++col) {
        const int a = fm.f[t].q[i].a;
        if (a >= P - 1) continue;
        const int64_t st = f0.pre_stride[a] / Dl;
        for (int g = tid; g < ng; g += 256) {
          const int64_t ghi = grp0 + g;             // prefix value without its last digit
          gdig[g * kMaxFoldTau * kMaxCross + col] =
              (ghi < 0x7FFFFFFF && st < 0x7FFFFFFF)
                  ? (int)(((uint32_t)ghi / (uint32_t)st) % (uint32_t)f0.pre_radix[a])
                  : (int)((ghi / st) % f0.pre_radix[a]);
        }
      }
    __syncthreads();
    for (int t = 0, col0 = 0; t < fm.ntau; ++t) {     // Xhi[g][u]
      const FoldParams& f = fm.f[t];
      V* xh = reinterpret_cast<V*>(smem_raw + L.xh[t]);
      const V* qs = reinterpret_cast<const V*>(smem_raw + L.qs[t]);
      for (int g = tid >> 5; g < ng; g += 8)
        for (int u = tid & 31; u < L.DinP[t]; u += 32) {
          V x = u < f.Din ? (V)0 : T::CAP;
          if (u < f.Din) {
            int qo = 0;
            for (int i = 0; i < f.nq; ++i) {
              if (f.q[i].a < P - 1)
                x = T::sat(x, qs[qo + u * f.q[i].db + gdig[g * kMaxFoldTau * kMaxCross + col0 + i]]);
              qo += f.Din * f.q[i].db;
            }
          }
          xh[g * L.DinP[t] + u] = x;
        }
      col0 += f.nq;
    }
    __syncthreads();
    for (int t = 0; t < fm.ntau; ++t) {                // X_p[u] = Xhi[g][u] + QL[s][u], 4 u at a time
      V* xs = reinterpret_cast<V*>(smem_raw + L.xs[t]);
      const V* xh = reinterpret_cast<const V*>(smem_raw + L.xh[t]);
      const V* ql = reinterpret_cast<const V*>(smem_raw + L.ql[t]);
      const int DinP = L.DinP[t], nq4 = DinP / 4;
      for (int e = tid; e < n * nq4; e += 256) {
        const int pi = e / nq4, u0 = (e - pi * nq4) * 4;
        V a[4], b[4];
        load4<V>(xh + rg[pi] * DinP + u0, a);
        load4<V>(ql + rs[pi] * DinP + u0, b);
#pragma unroll
        for (int i = 0; i < 4; ++i) xs[pi * DinP + u0 + i] = T::sat(a[i], b[i]);
      }
    }
    if (tma) { mbar_wait(&mbar[buf], (phases >> buf) & 1u); phases ^= 1u << buf; }
    __syncthreads();
    const V* b = bs + (int64_t)buf * CH * DoP;
    auto fold_block = [&](int gblk, int pstart, int pstep, int grp) {
      int t = 0;
      while (t + 1 < fm.ntau && gblk >= L.blk0[t + 1]) ++t;
      const int blk = gblk - L.blk0[t];
      const int DinP = L.DinP[t];
      const V* xs = reinterpret_cast<const V*>(smem_raw + L.xs[t]);
      V* red = reinterpret_cast<V*>(smem_raw + L.red[t]) + (int64_t)grp * DinP * DoP;
      const int u0 = (blk / (DoP / 4)) * 4, v0 = (blk % (DoP / 4)) * 4;
      V acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T::CAP;
      const V* xp = xs + pstart * DinP + u0;
      const V* bp = b + pstart * DoP + v0;
      for (int pi = pstart; pi < n; pi += pstep, xp += pstep * DinP, bp += pstep * DoP) {
        V x[4], y[4];
        load4<V>(xp, x);
        load4<V>(bp, y);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = T::addmin(x[i], y[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[(u0 + i) * DoP + v0 + j] = acc[i][j];
    };
    if (L.groups > 1) {
      if (gi < L.groups) fold_block(tid - gi * L.nblk_all, gi, L.groups, gi);
    } else {
      for (int gb = tid; gb < L.nblk_all; gb += 256) fold_block(gb, 0, 1, 0);
    }
    __syncthreads();
    for (int t = 0; t < fm.ntau; ++t) {              // stripes -> this chunk's minima
      const FoldParams& f = fm.f[t];
      const V* red = reinterpret_cast<const V*>(smem_raw + L.red[t]);
      V* out = static_cast<V*>(f.chunkmin);
      const int DinP = L.DinP[t];
      for (int u = tid >> 5; u < f.Din; u += 8)
        for (int v = tid & 31; v < Do; v += 32) {
          V m = red[u * DoP + v];
          for (int g2 = 1; g2 < L.groups; ++g2) m = T::mn(m, red[(int64_t)g2 * DinP * DoP + u * DoP + v]);
          out[(int64_t)(u * Do + v) * nch + ch] = m;
        }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// argmin phase 1: per (u, v): A = min over chunks; the first chunk attaining
// it, then the least local prefix in that chunk with X_p[u] + B_p[v] == A.
// One warp per (u, v); chunk minima are contiguous per pair.
// --------------------------------------------------------------------------
template <typename V>
__global__ void fold_reduce_kernel(const FoldParams f, V* __restrict__ Aval, int64_t* __restrict__ pstar) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= f.Din * f.Do) return;
  const int u = warp / f.Do, v = warp % f.Do;
  const V* cm = static_cast<const V*>(f.chunkmin) + (int64_t)warp * f.nchunks;
  V best = VT<V>::CAP;
  int64_t bc = INT64_MAX;
  for (int64_t c = lane; c < f.nchunks; c += 32) {
    const V x = cm[c];
    if (x < best) { best = x; bc = c; }       // c increasing per lane: first wins
  }
  for (int o = 16; o > 0; o >>= 1) {
    const V ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
    if (ob < best || (ob == best && oc < bc)) { best = ob; bc = oc; }
  }
  if (best >= VT<V>::CAP) {
    if (lane == 0) { Aval[warp] = VT<V>::CAP; pstar[warp] = -1; }
    return;
  }
  const V* Bp = static_cast<const V*>(f.Bp);
  const V* vals = static_cast<const V*>(f.vals);
  const int64_t p0 = bc * f.CH;
  const int n = (int)min((int64_t)f.CH, f.nPl - p0);
  int64_t first = INT64_MAX;
  for (int pi = lane; pi < n; pi += 32) {
    const int64_t pl = p0 + pi;
    const V x = cross_sum<V>(f, vals, f.p_lo + pl, u);
    if (VT<V>::sat(x, Bp[pl * f.Do + v]) == best) { first = pl; break; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t of = __shfl_xor_sync(0xffffffffu, first, o);
    first = of < first ? of : first;
  }
  if (lane == 0) { Aval[warp] = best; pstar[warp] = first; }
}

// --------------------------------------------------------------------------
// argmin phase 2: least suffix (in canonical order, restricted to s_o = v when
// o is a suffix digit) whose intra cost equals B_p*[v]; then the original
// combination index and the outputs in the caller's (unpruned) layout.
// --------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) suffix_argmin_kernel(const ArgminParams ap,
                                                            const V* __restrict__ Aval,
                                                            const V* __restrict__ vals) {
  const FoldParams& f = ap.f;
  const EvalSpec& e = ap.e;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tabs = reinterpret_cast<V*>(smem_raw);                                   // W/R tables
  uint16_t* sd = reinterpret_cast<uint16_t*>(tabs + ((e.tab_n + 1) & ~1));    // [K][blockDim]
  const int pair = blockIdx.x;
  const int u = pair / f.Do, v = pair % f.Do;
  const int vo = ap.vmap[v];
  const int64_t outi = (int64_t)u * ap.Do_orig + vo;
  const int64_t pl = ap.pstar[pair];
  __shared__ unsigned long long s_first;
  if (pl < 0) {
    if (threadIdx.x == 0) {
      ap.A_out[outi] = kInf64;
      ap.I_out[outi] = kInf64;
    }
    return;
  }
  for (int i = threadIdx.x; i < e.tab_n; i += blockDim.x) tabs[i] = vals[e.tab_lo + i];
  const V* Bp = static_cast<const V*>(f.Bp);
  const uint64_t target = (uint64_t)Bp[pl * f.Do + v];
  const int64_t pg = f.p_lo + pl;
  const int tid = threadIdx.x, nth = blockDim.x;
  auto S = [&](int d) -> uint16_t& { return sd[d * nth + tid]; };
  {
    int64_t q = pg;
    for (int d = e.P - 1; d >= 0; --d) { S(d) = (uint16_t)(q % e.radix[d]); q /= e.radix[d]; }
  }
  const bool o_suffix = e.o >= e.P;
  const int64_t nrest = o_suffix ? e.nsuffix / e.radix[e.o] : e.nsuffix;
  if (tid == 0) s_first = ~0ull;
  __syncthreads();
  const int64_t per = (nrest + nth - 1) / nth;
  const int64_t lo = (int64_t)tid * per;
  const int64_t hi = min(nrest, lo + per);
  if (lo < hi) {
    // decode lo over the free suffix digits (canonical order, o fixed to v)
    int64_t q = lo;
    for (int d = e.K - 1; d >= e.P; --d) {
      if (o_suffix && d == e.o) { S(d) = (uint16_t)v; continue; }
      S(d) = (uint16_t)(q % e.radix[d]);
      q /= e.radix[d];
    }
    for (int64_t r = lo; r < hi; ++r) {
      uint64_t c = 0;
      bool inf = false;
      for (int i = 0; i < e.nterm; ++i) {
        const Term& tm = e.term[i];
        const int64_t o = tm.off - e.tab_lo;
        const V x = tm.kind == 0 ? tabs[o + S(tm.a)] : tabs[o + (int)S(tm.a) * tm.db + S(tm.b)];
        inf |= x >= VT<V>::CAP;
        c += (uint64_t)x;
      }
      if (!inf && c == target) {
        int64_t sfx = 0;                       // suffix index in canonical order
        for (int d = e.P; d < e.K; ++d) sfx = sfx * e.radix[d] + S(d);
        atomicMin(&s_first, (unsigned long long)sfx);
        break;
      }
      for (int d = e.K - 1; d >= e.P; --d) {   // odometer step
        if (o_suffix && d == e.o) continue;
        if (++S(d) < e.radix[d]) break;
        S(d) = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const uint64_t sfx = s_first;
    uint64_t q = sfx;
    for (int d = e.K - 1; d >= e.P; --d) { S(d) = (uint16_t)(q % e.radix[d]); q /= e.radix[d]; }
    uint64_t idx = 0;
    for (int d = 0; d < e.K; ++d) idx = idx * ap.orig_radix[d] + ap.maps[ap.map_off[d] + S(d)];
    ap.A_out[outi] = (uint64_t)Aval[pair];
    ap.I_out[outi] = sfx == ~0ull ? kInf64 : idx;     // ~0: cannot happen (exact arithmetic)
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
template <typename V>
__global__ void __launch_bounds__(128) argmin_kernel(const ArgminParams ap, const V* __restrict__ vals) {
  const FoldParams& f = ap.f;
  const EvalSpec& e = ap.e;
  constexpr int NT = 128;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* sd = reinterpret_cast<uint16_t*>(smem_raw);        // [K][NT] digits
  __shared__ V s_best[4];
  __shared__ int64_t s_bc[4];
  __shared__ unsigned long long s_first;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const int u = pair / f.Do, v = pair - (pair / f.Do) * f.Do;
  const int64_t outi = (int64_t)u * ap.Do_orig + ap.vmap[v];
  // 1. chunk minima of this pair are contiguous
  const V* cm = static_cast<const V*>(f.chunkmin) + (int64_t)pair * f.nchunks;
  V best = VT<V>::CAP;
  int64_t bc = INT64_MAX;
  for (int64_t c = tid; c < f.nchunks; c += NT) {
    const V x = cm[c];
    if (x < best) { best = x; bc = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const V ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
    if (ob < best || (ob == best && oc < bc)) { best = ob; bc = oc; }
  }
  if (lane == 0) { s_best[warp] = best; s_bc[warp] = bc; }
  if (tid == 0) s_first = ~0ull;
  __syncthreads();
  best = s_best[0];
  bc = s_bc[0];
  for (int w = 1; w < NT / 32; ++w)
    if (s_best[w] < best || (s_best[w] == best && s_bc[w] < bc)) { best = s_best[w]; bc = s_bc[w]; }
  if (best >= VT<V>::CAP) {
    if (tid == 0) { ap.A_out[outi] = kInf64; ap.I_out[outi] = kInf64; }
    return;
  }
  // 2. least canonical prefix over every chunk attaining the minimum
  //    (chunk c = (l, hb) holds local rows (hb * kBlock + i) * W + l)
  const V* Bp = static_cast<const V*>(f.Bp);
  __shared__ int64_t s_list[NT];
  __shared__ int s_cnt;
  for (int64_t base = 0; base < f.nchunks; base += NT) {
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    const int64_t c = base + tid;
    if (c < f.nchunks && cm[c] == best) s_list[atomicAdd(&s_cnt, 1)] = c;
    __syncthreads();
    const int cnt = s_cnt;
    for (int li = 0; li < cnt; ++li) {
      const int64_t cc = s_list[li];
      const int64_t l = cc / f.nhb, hb = cc - l * f.nhb;
      for (int i = tid; i < kBlock; i += NT) {
        const int64_t hh = hb * kBlock + i;
        if (hh >= f.G) break;
        const int64_t plr = hh * f.W + l;
        const V x = cross_sum<V>(f, vals, f.p_lo + plr, u);
        if (VT<V>::sat(x, Bp[plr * f.Do + v]) == best) {
          atomicMin(&s_first, (unsigned long long)plr);   // local order == canonical order
          break;
        }
      }
    }
    __syncthreads();
  }
  const int64_t pl = (int64_t)s_first;
  __syncthreads();
  if (tid == 0) s_first = ~0ull;
  const uint64_t target = (uint64_t)Bp[pl * f.Do + v];
  const int64_t pg = f.p_lo + pl;
  auto S = [&](int d) -> uint16_t& { return sd[d * NT + tid]; };
  {
    int64_t q = pg;
    for (int d = e.P - 1; d >= 0; --d) { S(d) = (uint16_t)(q % e.radix[d]); q /= e.radix[d]; }
  }
  const bool o_suffix = e.o >= e.P;
  const int64_t nrest = o_suffix ? e.nsuffix / e.radix[e.o] : e.nsuffix;
  __syncthreads();
  // 3. least suffix with intra cost == B_p*[v]
  const int64_t per = (nrest + NT - 1) / NT;
  const int64_t lo = (int64_t)tid * per;
  const int64_t hi = min(nrest, lo + per);
  if (lo < hi) {
    int64_t q = lo;
    for (int d = e.K - 1; d >= e.P; --d) {
      if (o_suffix && d == e.o) { S(d) = (uint16_t)v; continue; }
      S(d) = (uint16_t)(q % e.radix[d]);
      q /= e.radix[d];
    }
    for (int64_t r = lo; r < hi; ++r) {
      uint64_t c = 0;
      bool inf = false;
      for (int i = 0; i < e.nterm; ++i) {
        const Term& tm = e.term[i];
        const V x = tm.kind == 0 ? vals[tm.off + S(tm.a)] : vals[tm.off + (int)S(tm.a) * tm.db + S(tm.b)];
        inf |= x >= VT<V>::CAP;
        c += (uint64_t)x;
      }
      if (!inf && c == target) {
        int64_t sfx = 0;
        for (int d = e.P; d < e.K; ++d) sfx = sfx * e.radix[d] + S(d);
        atomicMin(&s_first, (unsigned long long)sfx);
        break;
      }
      for (int d = e.K - 1; d >= e.P; --d) {       // odometer step
        if (o_suffix && d == e.o) continue;
        if (++S(d) < e.radix[d]) break;
        S(d) = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const uint64_t sfx = s_first;
    uint64_t q = sfx;
    for (int d = e.K - 1; d >= e.P; --d) { S(d) = (uint16_t)(q % e.radix[d]); q /= e.radix[d]; }
    uint64_t idx = 0;
    for (int d = 0; d < e.K; ++d) idx = idx * ap.orig_radix[d] + ap.maps[ap.map_off[d] + S(d)];
    ap.A_out[outi] = (uint64_t)best;
    ap.I_out[outi] = sfx == ~0ull ? kInf64 : idx;     // ~0: cannot happen (exact arithmetic)
  }
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



__device__ void matvec(const uint64_t* M, int rows, int cols, const uint64_t* g, uint64_t* out,
                       int tid, int nth) {
  for (int u = tid; u < rows; u += nth) {
    uint64_t best = kInf64;
    for (int v = 0; v < cols; ++v) {
      const uint64_t c = sat64(M[(int64_t)u * cols + v], g[v]);
      best = c < best ? c : best;
    }
    out[u] = best;
  }
}

// Single-CTA chain.  SM = true: every distinct matrix (A and, for the
// backtrack, I), every suffix vector G_n, the powers of the current run and the
// instance metadata live in shared memory; G is copied out at the end.
// SM = false: same algorithm on global memory (large S).
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool SM>
__global__ void __launch_bounds__(1024) chain_kernel(const ChainParams cp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int dbg_i = 0;
  auto mark = [&]() { if (cp.dbg && threadIdx.x == 0 && dbg_i < 64) cp.dbg[dbg_i++] = gtimer(); };
  mark();
  const int tid = threadIdx.x, nth = blockDim.x;
  const int N = cp.N;
  uint64_t* sA = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* sI = sA + cp.mat_elems;
  uint64_t* sG = sI + (cp.backtrack ? cp.mat_elems : 0);
  uint64_t* sP = sG + cp.goff[N + 1];
  int64_t* sgoff = reinterpret_cast<int64_t*>(sP + (int64_t)cp.levels_max * cp.smax * cp.smax);
  int4* sinst = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(sgoff + N + 2) + 15) & ~uintptr_t(15));
  uint64_t* G = SM ? sG : cp.G;
  uint64_t* Pw = SM ? sP : cp.powers;
  const int64_t* goff = SM ? sgoff : cp.goff;
  if constexpr (SM) {
    __shared__ __align__(8) uint64_t cbar;
    const bool tma = (cp.mat_elems & 1) == 0;          // 16-byte multiples
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
        sA[e] = cp.baseA[e];
        if (cp.backtrack) sI[e] = cp.baseI[e];
      }
    }
    for (int i = tid; i < N + 2; i += nth) sgoff[i] = cp.goff[i];
    for (int i = tid; i < N; i += nth) sinst[i] = make_int4(cp.inst[i].mat, cp.inst[i].rows, cp.inst[i].cols, 0);
    if (tma) mbar_wait(&cbar, 0);
    __syncthreads();
  }
  mark();
  auto rows_of = [&](int n) { return SM ? sinst[n].y : cp.inst[n].rows; };
  auto cols_of = [&](int n) { return SM ? sinst[n].z : cp.inst[n].cols; };
  auto matA = [&](int n) -> const uint64_t* { return SM ? sA + cp.moff[sinst[n].x] : cp.inst[n].A; };
  auto matI = [&](int n) -> const uint64_t* { return SM ? sI + cp.moff[sinst[n].x] : cp.inst[n].I; };
  const int lastc = cols_of(N - 1);
  for (int v = tid; v < lastc; v += nth) G[goff[N] + v] = cp.terminal ? cp.terminal[v] : 0;
  __syncthreads();
  for (int r = cp.nruns - 1; r >= 0; --r) {
    const ChainRun run = cp.runs[r];
    const uint64_t* M = matA(run.first);
    const int R = rows_of(run.first), Cc = cols_of(run.first);
    const int e = run.first + run.len;             // G_e known (1-based instance e)
    if (run.len == 1) {
      const uint64_t* g = G + goff[e];
      for (int u = tid; u < R; u += nth) {
        uint64_t best = kInf64;
        for (int v = 0; v < Cc; ++v) {
          const uint64_t c = sat64(M[(int64_t)u * Cc + v], g[v]);
          best = c < best ? c : best;
        }
        G[goff[e - 1] + u] = best;
      }
      __syncthreads();
      mark();
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
        const int i = (int)(c / S), k2 = (int)(c % S);
        uint64_t best = kInf64;
        for (int k = 0; k < S; ++k) {
          const uint64_t x = sat64(Pa[(int64_t)i * S + k], Pa[(int64_t)k * S + k2]);
          best = x < best ? x : best;
        }
        Pc[c] = best;
      }
      __syncthreads();
      mark();
    }
    // doubling: G_{e-k} = P_j (x) G_{e-k+2^j}, k in [2^j, 2^(j+1))
    for (int j = 0; j <= levels; ++j) {
      const uint64_t* Pj = j == 0 ? M : Pw + (int64_t)(j - 1) * S * S;
      const int k_lo = 1 << j, k_hi = min(1 << (j + 1), run.len + 1);
      const int64_t work = (int64_t)(k_hi - k_lo) * S;
      for (int64_t w = tid; w < work; w += nth) {
        const int k = k_lo + (int)(w / S), u = (int)(w % S);
        const uint64_t* g = G + goff[e - k + (1 << j)];
        uint64_t best = kInf64;
        for (int v = 0; v < S; ++v) {
          const uint64_t x = sat64(Pj[(int64_t)u * S + v], g[v]);
          best = x < best ? x : best;
        }
        G[goff[e - k] + u] = best;
      }
      __syncthreads();
      mark();
    }
  }
  if constexpr (SM)
    for (int64_t e2 = tid; e2 < goff[N + 1]; e2 += nth) cp.G[e2] = G[e2];
  if (!cp.backtrack) return;
  // forward greedy: at each instance the optimal successor with the least
  // combination index.  SM mode: the successor of every (n, u) is tabulated in
  // parallel first, then the walk from u_1 = 0 is a chain of shared loads.
  __shared__ int s_status;
  if (tid == 0) s_status = 0;
  __syncthreads();
  if constexpr (SM) {
    int16_t* nxt = reinterpret_cast<int16_t*>(sinst + N);   // [goff[N]] successor of (n, u)
    const int smax = cp.smax;
    for (int64_t w = tid; w < (int64_t)N * smax; w += nth) {
      const int n = (int)(w / smax), u = (int)(w - (int64_t)n * smax);   // instance n + 1
      if (u >= rows_of(n)) continue;
      const uint64_t* A = matA(n);
      const uint64_t* I = matI(n);
      const int cols = cols_of(n);
      const uint64_t target = G[goff[n] + u];
      const uint64_t* Gn = G + goff[n + 1];
      uint64_t bi = kInf64;
      int bv = -1;
      if (target != kInf64)
        for (int v = 0; v < cols; ++v) {
          const uint64_t a = A[(int64_t)u * cols + v];
          if (a == kInf64 || Gn[v] == kInf64 || a + Gn[v] != target) continue;
          const uint64_t ix = I[(int64_t)u * cols + v];
          if (bv < 0 || ix < bi) { bi = ix; bv = v; }
        }
      nxt[goff[n] + u] = (int16_t)bv;
    }
    __syncthreads();
    mark();
    if (tid == 0) {
      if (G[0] == kInf64) {
        s_status = 3;
        *cp.total = kInf64;
      } else {
        *cp.total = G[0];
        int u = 0;
        for (int n = 0; n < N; ++n) {
          const int v = nxt[goff[n] + u];
          if (v < 0) { s_status = 3; break; }
          const int cols = cols_of(n);
          cp.seg_index[n] = matI(n)[(int64_t)u * cols + v];
          cp.seg_ns[n] = matA(n)[(int64_t)u * cols + v];
          u = v;
        }
      }
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
  mark();
  if (tid == 0) *cp.status = s_status;
  if (s_status != 0) return;
  for (int64_t w = tid; w < (int64_t)N * cp.kmax; w += nth) {
    const int n = (int)(w / cp.kmax), j = (int)(w % cp.kmax);
    const ChainInst in = cp.inst[n];
    int32_t dval = -1;
    if (j < in.K) {
      uint64_t q = cp.seg_index[n];
      for (int d = in.K - 1; d > j; --d) q /= (uint64_t)cp.radix_blob[in.radix_off + d];
      dval = (int32_t)(q % (uint64_t)cp.radix_blob[in.radix_off + j]);
    }
    cp.digits[w] = dval;
  }
  __syncthreads();
  mark();
  if (cp.dbg && tid == 0) cp.dbg[63] = dbg_i;
}

// --------------------------------------------------------------------------
// (min,+) product with least-k argmin (cfp_minplus_product; also the large-S
// chain path).  16x16 output tile per CTA, K staged through shared memory.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) minplus_kernel(int m, int k, int n, const uint64_t* __restrict__ A,
                                                      const uint64_t* __restrict__ B, uint64_t* __restrict__ C,
                                                      uint64_t* __restrict__ argk) {
  __shared__ uint64_t As[16][17], Bs[16][17];
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const int i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  uint64_t best = kInf64, bk = kInf64;
  for (int k0 = 0; k0 < k; k0 += 16) {
    As[ty][tx] = (i < m && k0 + tx < k) ? A[(int64_t)i * k + k0 + tx] : kInf64;
    Bs[ty][tx] = (k0 + ty < k && j < n) ? B[(int64_t)(k0 + ty) * n + j] : kInf64;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint64_t x = sat64(As[ty][q], Bs[q][tx]);
      if (x < best) { best = x; bk = (uint64_t)(k0 + q); }
    }
    __syncthreads();
  }
  if (i < m && j < n) {
    C[(int64_t)i * n + j] = best;
    if (argk) argk[(int64_t)i * n + j] = best == kInf64 ? kInf64 : bk;
  }
}

__global__ void matvec_kernel(const uint64_t* __restrict__ M, int rows, int cols,
                              const uint64_t* __restrict__ g, uint64_t* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= rows) return;
  uint64_t best = kInf64;
  for (int v = 0; v < cols; ++v) {
    const uint64_t c = sat64(M[(int64_t)u * cols + v], g[v]);
    best = c < best ? c : best;
  }
  out[u] = best;
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
  int64_t blocks = (max_entries + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  build_table_kernel<V><<<dim3((unsigned)blocks, nspecs), 256, 0, st>>>(specs, vals, out);
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
  const int64_t blocks = p.W * p.VG * (p.Gpad / kBlock);
  if (blocks <= 0) return cudaSuccess;
  const size_t sm = std::max(smem, (size_t)p.smem_epi);
  auto launch = [&](auto kern) -> cudaError_t {
    if (sm > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)blocks, kBlock, sm, st>>>(p);
    return cudaGetLastError();
  };
  if (p.staged) return launch(enum_kernel<V, NB, true>);
  return launch(enum_kernel<V, NB, false>);
}

template <typename V>
cudaError_t launch_enum(const EnumParams& p, int NB, int64_t nthreads, size_t smem, cudaStream_t st) {
  switch (NB) {
    case 4: return launch_enum_nb<V, 4>(p, nthreads, smem, st);
    case 8: return launch_enum_nb<V, 8>(p, nthreads, smem, st);
    case 12: return launch_enum_nb<V, 12>(p, nthreads, smem, st);
    case 16: return launch_enum_nb<V, 16>(p, nthreads, smem, st);
    case 24: return launch_enum_nb<V, 24>(p, nthreads, smem, st);
    case 32: return launch_enum_nb<V, 32>(p, nthreads, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename V>
cudaError_t launch_fold(const FoldMulti& fm, int grid, cudaStream_t st) {
  const FoldSmem L = fold_layout(fm, (int)sizeof(V));
  const size_t smem = (size_t)L.total;
  auto k = fold_kernel<V>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)grid, 256, smem, st>>>(fm);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

template <typename V>
cudaError_t launch_argmin(const ArgminParams& ap, V* Aval, const V* vals, cudaStream_t st) {
  (void)Aval;
  const int pairs = ap.f.Din * ap.f.Do;
  const size_t smem = (size_t)ap.e.K * 128 * 2 + 16;
  argmin_kernel<V><<<pairs, 128, smem, st>>>(ap, vals);
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

cudaError_t launch_minplus(int m, int k, int n, const uint64_t* A, const uint64_t* B, uint64_t* C,
                           uint64_t* argk, cudaStream_t st) {
  dim3 grid((n + 15) / 16, (m + 15) / 16);
  minplus_kernel<<<grid, 256, 0, st>>>(m, k, n, A, B, C, argk);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

cudaError_t launch_matvec(const uint64_t* M, int rows, int cols, const uint64_t* g, uint64_t* out,
                          cudaStream_t st) {
  matvec_kernel<<<(rows + 255) / 256, 256, 0, st>>>(M, rows, cols, g, out);
  CFP_LAUNCH_CHECK();
  return cudaSuccess;
}

cudaError_t launch_intpipe(int op, int blocks, int iters, uint32_t* out, cudaStream_t st) {
  if (op == 0) intpipe_kernel<0><<<blocks, 1024, 0, st>>>(out, iters, 7u);
  else if (op == 1) intpipe_kernel<1><<<blocks, 1024, 0, st>>>(out, iters, 7u);
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
template cudaError_t launch_fold<uint32_t>(const FoldMulti&, int, cudaStream_t);
template cudaError_t launch_fold<uint64_t>(const FoldMulti&, int, cudaStream_t);
template cudaError_t launch_argmin<uint32_t>(const ArgminParams&, uint32_t*, const uint32_t*, cudaStream_t);
template cudaError_t launch_argmin<uint64_t>(const ArgminParams&, uint64_t*, const uint64_t*, cudaStream_t);

}  // namespace cfp
