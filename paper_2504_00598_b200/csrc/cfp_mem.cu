// cfp_mem.cu -- sm_100a kernels of the memory-constrained search (SURVEY
// §8(f) NEXT-1: Eq. 4, DP P:625-628).
//
// Steps (host side in cfp_mem_host.inc):
//   mem_enum_kernel   every combination (p, sigma) of a type: cost
//                     K0[p] + T[ctx(p)][sigma] formed and min-reduced into its
//                     suffix class (output layout slot, suffix memory) with one
//                     fused add+min (VIADDMNMX) per combination; the suffix
//                     combinations of a class are contiguous in the
//                     class-sorted table staged in shared memory.
//   mem_fold_kernel   cross terms of one transition folded over the prefixes
//                     of one prefix-memory class (a tile): a (min,+) product
//                     chunk[u][cls] = min_p X_p[u] + B_p[cls], 4x4 register
//                     blocks, rows staged through shared memory.
//   mem_amin_kernel   Am[u][v][q] = min over tiles (tile memory k + class rs = q).
//   mem_chain_kernel  one backward step of the (layout, memory) DP.
//   mem_bfs_kernel    optimal edges reachable from (0, 0) -> needed buckets.
//   mem_argmin_kernel least combination index of every needed bucket: least
//                     prefix among the attaining tiles' rows, then the least
//                     suffix combination of that prefix.
//   mem_greedy_kernel forward greedy walk + digit decode.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "cfp_internal.h"

namespace cfp {

template <typename V> struct MT;
template <> struct MT<uint32_t> {
  static constexpr uint32_t CAP = kCap32;
  __device__ static __forceinline__ uint32_t addmin(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_u32(a, b, c);                 // min(a + b, c): VIADDMNMX.U32
  }
  __device__ static __forceinline__ uint32_t sat(uint32_t a, uint32_t b) { return __viaddmin_u32(a, b, CAP); }
  __device__ static __forceinline__ void load4(const uint32_t* p, uint32_t* v) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct MT<uint64_t> {
  static constexpr uint64_t CAP = kCap64;
  __device__ static __forceinline__ uint64_t addmin(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t s = a + b;                       // a, b <= CAP: no wrap
    return s < c ? s : c;
  }
  __device__ static __forceinline__ uint64_t sat(uint64_t a, uint64_t b) { return addmin(a, b, CAP); }
  __device__ static __forceinline__ void load4(const uint64_t* p, uint64_t* v) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(p);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};

// x * one + y on the FMA pipe (one = 1 at run time: ptxas keeps the IMAD)
__device__ __forceinline__ uint32_t mem_mad(uint32_t x, uint32_t one, uint32_t y) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(y));
  return r;
}
__device__ __forceinline__ uint64_t mem_mad(uint64_t x, uint32_t, uint64_t y) { return x + y; }

// Natural prefix index from (ctx value, other-digit value).
__device__ __forceinline__ int64_t mem_prefix(const MemPrefixMap& m, int64_t c, int64_t n) {
  int64_t p = 0;
  for (int i = m.nctx - 1; i >= 0; --i) {
    const int pos = m.ctx_pos[i];
    const int64_t r = m.radix[pos];
    p += (c % r) * m.stride[pos];
    c /= r;
  }
  for (int i = m.nnon - 1; i >= 0; --i) {
    const int pos = m.non_pos[i];
    const int64_t r = m.radix[pos];
    p += (n % r) * m.stride[pos];
    n /= r;
  }
  return p;
}
__device__ __forceinline__ int mem_digit(const MemPrefixMap& m, int64_t p, int pos) {
  return (int)((p / m.stride[pos]) % m.radix[pos]);
}
__device__ __forceinline__ int mem_digit32(const MemPrefixMap& m, uint32_t p, int pos) {
  return (int)((p / (uint32_t)m.stride[pos]) % (uint32_t)m.radix[pos]);   // prefix space < 2^31
}
__device__ __forceinline__ int64_t mem_ctx(const MemPrefixMap& m, int64_t p) {
  int64_t c = 0;
  for (int i = 0; i < m.nctx; ++i) c = c * m.radix[m.ctx_pos[i]] + mem_digit(m, p, m.ctx_pos[i]);
  return c;
}

// --------------------------------------------------------------------------
// a0: K0 / Tc / Ts of every type from the raw input values (saturating uint64
// sums, INF absorbing, clamped to the path's CAP).  Grid-stride over the jobs'
// entries; a CTA belongs to one job (block0 ranges).
// --------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) mem_values_kernel(const MemValJob* __restrict__ jobs, int njobs,
                                                         const uint32_t* __restrict__ raw) {
  __shared__ int s_j;
  if (threadIdx.x == 0) {
    int j = 0;
    while (j + 1 < njobs && (int64_t)blockIdx.x >= jobs[j + 1].block0) ++j;
    s_j = j;
  }
  __syncthreads();
  const MemValJob& J = jobs[s_j];
  const int64_t nblk = (s_j + 1 < njobs ? jobs[s_j + 1].block0 : (int64_t)gridDim.x) - J.block0;
  V* out = static_cast<V*>(J.out);
  for (int64_t e = (blockIdx.x - J.block0) * (int64_t)blockDim.x + threadIdx.x; e < J.n;
       e += nblk * blockDim.x) {
    int dig[kMaxDigits];
    uint64_t acc = 0;
    bool pad = false;
    if (J.kind == 0) {                                   // prefix p, natural order
      int64_t q = e;
      for (int d = J.P - 1; d >= 0; --d) { dig[d] = (int)(q % J.radix[d]); q /= J.radix[d]; }
    } else {
      const int64_t row = J.kind == 1 ? J.nS : J.Tlen;
      int64_t c = e / row, i = e - c * row;
      if (J.kind == 2) {
        if (i >= J.nS) pad = true;
        else i = J.order[i];
      }
      for (int d = J.K - 1; d >= J.P; --d) { dig[d] = (int)(i % J.radix[d]); i /= J.radix[d]; }
      for (int t = J.nctx - 1; t >= 0; --t) {
        const int b = J.ctx_pos[t];
        dig[b] = (int)(c % J.radix[b]);
        c /= J.radix[b];
      }
    }
    if (!pad) {
      for (int t = 0; t < J.nterm && acc != kInf64; ++t) {
        const MemValTerm tm = J.term[t];
        uint64_t x;
        if (tm.kind == 0) {
          const uint32_t pc = raw[tm.off + dig[tm.a]];
          const uint32_t cc = tm.off2 >= 0 ? raw[tm.off2 + dig[tm.a]] : 0u;
          x = (pc == 0xFFFFFFFFu || cc == 0xFFFFFFFFu) ? kInf64 : (uint64_t)pc + cc;
        } else {
          const uint32_t r = raw[tm.off + (int64_t)dig[tm.a] * tm.db + dig[tm.b]];
          x = r == 0xFFFFFFFFu ? kInf64 : (uint64_t)r;
        }
        acc = x == kInf64 ? kInf64 : acc + x;
      }
    }
    const uint64_t cap = MT<V>::CAP;
    out[e] = (V)((pad || acc >= cap) ? cap : acc);
  }
}

// --------------------------------------------------------------------------
// Enumeration.  CTA = up to 8 warp tiles of one ctx value c; warp tile = up to
// 32 * NPF consecutive prefix positions of one prefix-memory group g (so one
// set of suffix class runs); lane = NPF positions.  T[c] (suffixes sorted by
// (output slot, exact memory), CAP padded) is staged in shared memory; every
// combination of a class run is one VIADDMNMX per prefix:
// acc_i = min(K0[p_i] + T[c][e], acc_i).  The runs start anywhere in the row:
// a scalar head up to the next 16-byte boundary, 16-byte loads (warp-uniform
// addresses: broadcasts), a scalar tail.  B[cls][pos] stores are coalesced.
// --------------------------------------------------------------------------
template <typename V, int NPF>
__global__ void __launch_bounds__(256) mem_enum_kernel(const MemEnumParams p) {
  using M = MT<V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* ts = reinterpret_cast<V*>(smem_raw);
  const int4 ct = p.ctiles[blockIdx.x];
  const V* src = static_cast<const V*>(p.Ts) + (int64_t)ct.z * p.Tlen;
  for (int e = threadIdx.x * 4; e < p.Tlen; e += 256 * 4) {
    V t[4];
    M::load4(src + e, t);
#pragma unroll
    for (int q = 0; q < 4; ++q) ts[e + q] = t[q];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= ct.y) return;                          // no barrier below
  const int4 wt = p.wtiles[ct.x + warp];
  int64_t pos[NPF];
  V k0[NPF];
  bool live[NPF];
#pragma unroll
  for (int i = 0; i < NPF; ++i) {
    const int r = i * 32 + lane;
    live[i] = r < wt.y;
    pos[i] = (int64_t)wt.x + r;
    k0[i] = live[i] ? static_cast<const V*>(p.K0)[p.perm[pos[i]]] : M::CAP;
  }
  const int2* rg = p.runs + (int64_t)wt.z * p.Wc;
  V* B = static_cast<V*>(p.B);
  for (int c0 = 0; c0 < p.Wc; c0 += 32) {
    const int2 myrun = c0 + lane < p.Wc ? rg[c0 + lane] : make_int2(0, 0);   // one coalesced load per 32 classes
    const int nc = min(32, p.Wc - c0);
    for (int ci = 0; ci < nc; ++ci) {
      const int s0 = __shfl_sync(0xffffffffu, myrun.x, ci), s1 = __shfl_sync(0xffffffffu, myrun.y, ci);
      V acc[NPF];
#pragma unroll
      for (int i = 0; i < NPF; ++i) acc[i] = M::CAP;
      const int a0 = min((s0 + 3) & ~3, s1), a1 = max(a0, s1 & ~3);
      for (int e = s0; e < a0; ++e) {                  // head
        const V t = ts[e];
#pragma unroll
        for (int i = 0; i < NPF; ++i) acc[i] = M::addmin(k0[i], t, acc[i]);
      }
#pragma unroll 2
      for (int e = a0; e < a1; e += 4) {               // 16-byte body
        V t[4];
        M::load4(ts + e, t);
        if constexpr (sizeof(V) == 4) {
          // two pipes (as enum_kernel's loop): per 4 combinations two
          // VIADDMNMX (ALU) and two FMA-pipe IMAD adds folded by one VIMNMX3
#pragma unroll
          for (int i = 0; i < NPF; ++i) {
            V a = M::addmin(k0[i], t[0], acc[i]);
            a = M::addmin(k0[i], t[1], a);
            acc[i] = __vimin3_u32(a, mem_mad(k0[i], p.one, t[2]), mem_mad(k0[i], p.one, t[3]));
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < NPF; ++i) acc[i] = M::addmin(k0[i], t[q], acc[i]);
        }
      }
      for (int e = a1; e < s1; ++e) {                  // tail
        const V t = ts[e];
#pragma unroll
        for (int i = 0; i < NPF; ++i) acc[i] = M::addmin(k0[i], t, acc[i]);
      }
      const int cls = c0 + ci;
      V* row = B + (int64_t)(cls >> 2) * p.nP * 4 + (cls & 3);     // B[cls/4][pos][cls%4]
#pragma unroll
      for (int i = 0; i < NPF; ++i)
        if (live[i]) row[pos[i] * 4] = acc[i];
    }
  }
}

// --------------------------------------------------------------------------
// Cross terms of every prefix position: X[pos][u] = sum_i Q_i[u][s_i(perm[pos])]
// (Eq. 3 r_n), saturated; one thread per (position, u quad).
// --------------------------------------------------------------------------
template <typename V>
__global__ void mem_xrows_kernel(const MemFoldParams p) {
  using M = MT<V>;
  const int nuq = p.DinP >> 2;
  const int64_t total = p.nP * nuq;
  const V* vals = static_cast<const V*>(p.vals);
  V* X = static_cast<V*>(p.X);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = e / nuq;
    const int uq = (int)(e - pos * nuq);
    const uint32_t pr = (uint32_t)p.perm[pos];
    V x[4] = {0, 0, 0, 0};
    for (int i = 0; i < p.nq; ++i) {
      V y[4];
      M::load4(vals + p.q_off[i] + (int64_t)mem_digit32(p.pm, pr, p.q_pos[i]) * p.DinP + uq * 4, y);
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = M::sat(x[k], y[k]);
    }
    V* o = X + pos * p.DinP + uq * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = x[k];
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// --------------------------------------------------------------------------
// Fold of one transition.  CTA = (tile of <= kMemFoldTile positions of one
// (ctx, prefix-memory class) group, balanced block of classes).  Thread = 4
// input states x 4 classes, 16 fused add+mins per row.  X rows and B rows are
// staged by cp.async into a two-stage shared-memory ring: the copies of
// chunk c+1 overlap the (min,+) work on chunk c.
// --------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) mem_fold_kernel(const MemFoldParams p) {
  using M = MT<V>;
  constexpr int R = kMemFoldStage / (int)sizeof(V);   // rows per stage
  constexpr int VPU = 16 / sizeof(V);               // elements per 16-byte copy
  extern __shared__ __align__(16) unsigned char fsm[];
  const int fc = p.fc;
  const int FP = fc + 4;                            // Bs row pitch (+4: conflict-free row stores)
  V* Xs = reinterpret_cast<V*>(fsm);                // [2][R][32]
  V* Bs = Xs + 2 * R * 32;                          // [2][R][FP]
  const int4 tile = p.tiles[blockIdx.x];
  const int col0 = blockIdx.y * fc;
  const int ncols = min(fc, p.Wc - col0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int ncq = (ncols + 3) >> 2;                 // class quads of this block
  const int tu = tid / ncq, tc = tid - tu * ncq;    // thread = (u quad, class quad)
  const V* B = static_cast<const V*>(p.B);
  const V* X = static_cast<const V*>(p.X);
  V* out = static_cast<V*>(p.chunk) + (int64_t)blockIdx.x * p.Din * p.Wc;
  const int nchunk = (tile.y + R - 1) / R;
  // this thread's 16-byte copies of a full stage, (row, column unit) pairs
  // computed once (the per-stage index math was a quarter of the kernel's
  // instructions); a short last stage skips rows >= its row count
  constexpr int MAXB = (kMemFoldStage / 4) * kMemFoldQuads * 2 / 256 + 1;   // >= R x (16-byte units per row) / threads
  int brow[MAXB], bcol[MAXB];
  const int nbq = ncq * (4 / VPU);                  // 16-byte units per B row
  int nbc = 0;
  const bool pre = R * nbq <= MAXB * nth;          // else (few threads, wide block) index per copy
#pragma unroll
  for (int i = 0; i < MAXB; ++i) {                  // fully unrolled: brow / bcol stay in registers
    const int e = tid + i * nth;
    brow[i] = pre && e < R * nbq ? e % R : R;       // R = no copy
    bcol[i] = e / R;
  }
  (void)nbc;
  for (int ub = 0; ub < p.Din; ub += 32) {          // input states in blocks of 32
    const int ucnt = min(32, p.DinP - ub);
    const int xu = ucnt / VPU;                      // 16-byte units per X row
    auto issue = [&](int st, int c) {
      const int64_t pos0 = (int64_t)tile.x + (int64_t)c * R;
      const int nr = min(R, tile.y - c * R);
      for (int e = tid; e < nr * xu; e += nth) {
        const int r = e / xu, k = e - r * xu;
        cp_async16(Xs + (st * R + r) * 32 + k * VPU, X + (pos0 + r) * p.DinP + ub + k * VPU);
      }
#pragma unroll
      for (int i = 0; i < MAXB; ++i) {
        if (brow[i] >= nr) continue;
        const int cq = bcol[i] / (4 / VPU), h = bcol[i] - cq * (4 / VPU);
        cp_async16(Bs + (st * R + brow[i]) * FP + cq * 4 + h * VPU,
                   B + ((int64_t)(col0 / 4 + cq) * p.nP + pos0 + brow[i]) * 4 + h * VPU);
      }
      for (int e = tid; !pre && e < nr * nbq; e += nth) {
        const int r = e % nr, q = e / nr;
        const int cq = q / (4 / VPU), h = q - cq * (4 / VPU);
        cp_async16(Bs + (st * R + r) * FP + cq * 4 + h * VPU, B + ((int64_t)(col0 / 4 + cq) * p.nP + pos0 + r) * 4 + h * VPU);
      }
      cp_async_commit();
    };
    V res[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) res[i][j] = M::CAP;
    issue(0, 0);
    for (int c = 0; c < nchunk; ++c) {
      if (c + 1 < nchunk) {
        issue((c + 1) & 1, c + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const int st = c & 1;
      const int nr = min(R, tile.y - c * R);
      if (tu < 8 && tu * 4 < ucnt) {
        const V* xr = Xs + st * R * 32 + tu * 4;
        const V* br = Bs + st * R * FP + tc * 4;
#pragma unroll 4
        for (int r = 0; r < nr; ++r) {
          V x[4], y[4];
          M::load4(xr + r * 32, x);
          M::load4(br + r * FP, y);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) res[i][j] = M::addmin(x[i], y[j], res[i][j]);
        }
      }
      __syncthreads();                               // stage st is refilled by the next issue
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int u = ub + tu * 4 + i, cl = col0 + tc * 4 + j;
        if (tu < 8 && u < p.Din && cl < col0 + ncols && tu * 4 + i < ucnt) out[(int64_t)u * p.Wc + cl] = res[i][j];
      }
  }
}

// --------------------------------------------------------------------------
// Fold of one transition, 32-bit path.  CTA = (tile of <= kMemFoldTile
// positions, block of fc classes); thread = U input states x 4 classes:
// per row U/4 X loads (warp broadcasts: a warp spans <= 2 state groups) and
// one 16-byte B load feed 4U fused add+mins (C3: U = 12, 48 per 4 loads --
// the 4 x 4 kernel above needs 2 loads per 16).  Rows arrive by cp.async in
// a 3-stage shared-memory ring.
// --------------------------------------------------------------------------
constexpr int kFoldUR = 16;      // rows per stage (3 x 16 rows of C3: 56 KB, 4 CTAs per SM)
constexpr int kFoldUS = 3;       // stages (2: C3 0.622 ms, C5 1.321 ms; 3: 0.630, 1.144)
template <int U>
__global__ void __launch_bounds__(256) mem_fold_u_kernel(const MemFoldParams p) {
  using M = MT<uint32_t>;
  constexpr int R = kFoldUR, NS = kFoldUS;
  extern __shared__ __align__(16) unsigned char fsm[];
  const int fc = p.fc, FP = fc + 4, XP = p.DinP;
  uint32_t* Xs = reinterpret_cast<uint32_t*>(fsm);  // [NS][R][XP]
  uint32_t* Bs = Xs + NS * R * XP;                  // [NS][R][FP]
  const int4 tile = p.tiles[blockIdx.x];
  const int col0 = blockIdx.y * fc;
  const int ncols = min(fc, p.Wc - col0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int ncq = (ncols + 3) >> 2;
  const int ngu = (p.DinP + U - 1) / U;
  const int tg = tid / ncq, tc = tid - tg * ncq;    // thread = (state group, class quad)
  const bool act = tg < ngu;
  const uint32_t* B = static_cast<const uint32_t*>(p.B);
  const uint32_t* X = static_cast<const uint32_t*>(p.X);
  const int nchunk = (tile.y + R - 1) / R;
  const int xu = XP / 4;
  // this thread's X copies of a stage, (row, 16-byte unit) fixed over the
  // stages (index math once, not per copy); B copies are (quad, row) =
  // (e / R, e % R) with R a power of two
  constexpr int MAXX = 2;
  int xr_[MAXX], xk_[MAXX];
#pragma unroll
  for (int i = 0; i < MAXX; ++i) {
    const int e = tid + i * nth;
    xr_[i] = e < R * xu ? e / xu : R;               // R = no copy
    xk_[i] = e - (e / xu) * xu;
  }
  const bool xfew = R * xu <= MAXX * nth;
  const int64_t bq_stride = (int64_t)p.nP * 4;
  const uint32_t* Bc = B + (int64_t)(col0 / 4) * bq_stride;
  auto issue = [&](int st, int c) {
    if (c < nchunk) {
      const int64_t pos0 = (int64_t)tile.x + (int64_t)c * R;
      const int nr = min(R, tile.y - c * R);
      if (xfew) {
#pragma unroll
        for (int i = 0; i < MAXX; ++i)
          if (xr_[i] < nr) cp_async16(Xs + (st * R + xr_[i]) * XP + xk_[i] * 4, X + (pos0 + xr_[i]) * XP + xk_[i] * 4);
      } else {
        for (int e = tid; e < nr * xu; e += nth) {
          const int r = e / xu, k = e - r * xu;
          cp_async16(Xs + (st * R + r) * XP + k * 4, X + (pos0 + r) * XP + k * 4);
        }
      }
      const uint32_t* Bp0 = Bc + pos0 * 4;
      for (int e = tid; e < R * ncq; e += nth) {
        const int q = e / R, r = e % R;             // consecutive threads: consecutive positions
        if (r < nr) cp_async16(Bs + (st * R + r) * FP + q * 4, Bp0 + q * bq_stride + r * 4);
      }
    }
    cp_async_commit();                              // (an empty group past the last chunk)
  };
  uint32_t res[U][4];
#pragma unroll
  for (int i = 0; i < U; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) res[i][j] = M::CAP;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(s, s);
  for (int c = 0; c < nchunk; ++c) {
    issue((c + NS - 1) % NS, c + NS - 1);
    cp_async_wait<NS - 1>();
    __syncthreads();
    const int st = c % NS;
    const int nr = min(R, tile.y - c * R);
    if (act) {
      const uint32_t* xr = Xs + st * R * XP + tg * U;
      const uint32_t* br = Bs + st * R * FP + tc * 4;
#pragma unroll 2
      for (int r = 0; r < nr; ++r) {
        uint32_t x[U], y[4];
#pragma unroll
        for (int i = 0; i < U; i += 4) M::load4(xr + r * XP + i, x + i);
        M::load4(br + r * FP, y);
#pragma unroll
        for (int i = 0; i < U; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) res[i][j] = M::addmin(x[i], y[j], res[i][j]);
      }
    }
    __syncthreads();                                 // stage st is refilled by a later issue
  }
  if (!act) return;
  uint32_t* out = static_cast<uint32_t*>(p.chunk) + (int64_t)blockIdx.x * p.Din * p.Wc;
#pragma unroll
  for (int i = 0; i < U; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int u = tg * U + i, cl = col0 + tc * 4 + j;
      if (u < p.Din && cl < col0 + ncols) out[(int64_t)u * p.Wc + cl] = res[i][j];
    }
}

// --------------------------------------------------------------------------
// Am[u][v][qi] = min over tiles of the tile's chunk at class (vslot, qi - k).
// One warp per output entry.
// --------------------------------------------------------------------------
template <typename V>
__global__ void mem_amin_kernel(const MemAminParams p) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)p.Din * p.Do * p.nq;
  if (e >= total) return;
  const int qi = (int)(e % p.nq);
  const int v = (int)((e / p.nq) % p.Do);
  const int u = (int)(e / ((int64_t)p.nq * p.Do));
  const V* ch = static_cast<const V*>(p.chunk);
  V best = MT<V>::CAP;
  for (int t = lane; t < p.ntiles; t += 32) {
    const int rc = p.tiles[t].z;
    const int k = rc / p.nVp, vp = rc % p.nVp;
    int vslot = v;
    if (p.o_in_prefix) {
      if (vp != v) continue;
      vslot = 0;
    }
    const int rs = qi - k;
    if (rs < 0 || rs >= p.RQs) continue;
    const V x = ch[((int64_t)t * p.Din + u) * p.Wc + vslot * p.RQs + rs];
    best = x < best ? x : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const V y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y < best ? y : best;
  }
  if (lane == 0) p.Am[e] = best >= MT<V>::CAP ? kInf64 : (uint64_t)best;
}

// --------------------------------------------------------------------------
// One backward DP step (P:625-628 with the memory state of S:466-474):
// G_n(u, c) = min_{v, q: c + q <= Qmax} Am[u][v][q - qlo] + G_{n+1}(v, c + q).
// CTA = (u, 64 memory states); thread = (state, v group of 4); Am row u in
// shared memory; the four v-group partial minima are reduced in shared memory.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) mem_chain_kernel(const MemChainParams cp, int n, int win) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t part[4][64];
  uint64_t* arow = reinterpret_cast<uint64_t*>(smem_raw);
  const MemInst in = cp.inst[n];
  const int u = blockIdx.x;
  const int C = cp.C;
  const int rowlen = in.cols * in.nq;
  const int c0 = blockIdx.y * 64;
  const uint64_t* Gn = cp.G + cp.goff[n + 1] * C;
  for (int e = threadIdx.x; e < rowlen; e += blockDim.x) arow[e] = in.Am[(int64_t)u * rowlen + e];
  // window of G_{n+1}: columns [c0 + qlo, c0 + qlo + win) of every row v
  uint64_t* gw = arow + ((rowlen + 1) & ~1);
  if (win > 0)
    for (int e = threadIdx.x; e < in.cols * win; e += blockDim.x) {
      const int v = e / win, k = e - v * win;
      const int cc = c0 + in.qlo + k;
      gw[e] = cc < C ? Gn[(int64_t)v * C + cc] : kInf64;
    }
  __syncthreads();
  const int cl = threadIdx.x & 63, vg = threadIdx.x >> 6;
  const int c = c0 + cl;
  uint64_t best = kInf64;
  if (c < C) {
    const int qmax = min(in.nq, C - c - in.qlo);    // c + qlo + qi <= Qmax = C - 1
    for (int v = vg; v < in.cols; v += 4) {
      const uint64_t* gv = win > 0 ? gw + v * win + cl : Gn + (int64_t)v * C + c + in.qlo;
      const uint64_t* av = arow + v * in.nq;
      for (int qi = 0; qi < qmax; ++qi) {
        const uint64_t a = av[qi], g = gv[qi];
        if (a == kInf64 || g == kInf64) continue;
        const uint64_t s = a + g;
        best = s < best ? s : best;
      }
    }
  }
  part[vg][cl] = best;
  __syncthreads();
  if (vg == 0 && c < C) {
    uint64_t b = part[0][cl];
#pragma unroll
    for (int k = 1; k < 4; ++k) b = part[k][cl] < b ? part[k][cl] : b;
    cp.G[(cp.goff[n] + u) * C + c] = b;
  }
}

// --------------------------------------------------------------------------
// All N backward DP steps in one persistent launch: the (row u, 64-column
// block) tiles of instance n are spread over the co-resident CTAs (the same
// arithmetic as mem_chain_kernel), then a grid barrier, then instance n - 1.
// One launch instead of N (each step is a few microseconds of work).
// --------------------------------------------------------------------------
constexpr uint64_t kBig = (1ull << 63) - 1;   // kBig + kBig < 2^64: no wrap
__device__ __forceinline__ uint64_t to_big(uint64_t x) { return x == kInf64 ? kBig : x; }

__device__ __forceinline__ void mem_grid_sync(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    const unsigned int arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == nblocks * gen) {
      atomicExch(bar + 1, gen);
    } else {
      while (*reinterpret_cast<volatile unsigned int*>(bar + 1) < gen) __nanosleep(64);
    }
    __threadfence();
  } else {
    ++gen;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) mem_chain_all_kernel(const MemChainParams cp, size_t smem_bytes,
                                                            unsigned int* bar) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t part[4][64];
  uint64_t* arow = reinterpret_cast<uint64_t*>(smem_raw);
  const int C = cp.C;
  const int nblk = (C + 63) / 64;
  unsigned int gen = 0;
  for (int n = cp.N - 1; n >= 0; --n) {
    const MemInst in = cp.inst[n];
    const int rowlen = in.cols * in.nq;
    int win = 64 + in.nq - 1;                       // as launch_mem_chain_step, against this launch's smem
    if ((size_t)((rowlen + 1) & ~1) * 8 + (size_t)in.cols * win * 8 + 16 > smem_bytes) win = 0;
    const uint64_t* Gn = cp.G + cp.goff[n + 1] * C;
    for (int tile = blockIdx.x; tile < in.rows * nblk; tile += gridDim.x) {
      const int u = tile / nblk;
      const int c0 = (tile - u * nblk) * 64;
      // staged with INF -> kBig = 2^63 - 1: finite sums stay below it (the
      // EOVERFLOW guard bounds every plan total by 9.2e18), a + g never wraps
      // (2 kBig < 2^64) and a sum >= kBig means INF -- the inner loop is a
      // plain add and min
      for (int e = threadIdx.x; e < rowlen; e += blockDim.x) arow[e] = to_big(in.Am[(int64_t)u * rowlen + e]);
      uint64_t* gw = arow + ((rowlen + 1) & ~1);
      if (win > 0)
        for (int e = threadIdx.x; e < in.cols * win; e += blockDim.x) {
          const int v = e / win, k = e - v * win;
          const int cc = c0 + in.qlo + k;
          gw[e] = cc < C ? to_big(Gn[(int64_t)v * C + cc]) : kBig;
        }
      __syncthreads();
      const int cl = threadIdx.x & 63, vg = threadIdx.x >> 6;
      const int c = c0 + cl;
      uint64_t best = kBig;
      if (c < C) {
        const int qmax = min(in.nq, C - c - in.qlo);
        for (int v = vg; v < in.cols; v += 4) {
          const uint64_t* av = arow + v * in.nq;
          if (win > 0) {
            const uint64_t* gv = gw + v * win + cl;
#pragma unroll 4
            for (int qi = 0; qi < qmax; ++qi) {
              const uint64_t s2 = av[qi] + gv[qi];
              best = s2 < best ? s2 : best;
            }
          } else {
            const uint64_t* gv = Gn + (int64_t)v * C + c + in.qlo;
            for (int qi = 0; qi < qmax; ++qi) {
              const uint64_t s2 = av[qi] + to_big(gv[qi]);
              best = s2 < best ? s2 : best;
            }
          }
        }
      }
      part[vg][cl] = best;
      __syncthreads();
      if (vg == 0 && c < C) {
        uint64_t b = part[0][cl];
#pragma unroll
        for (int k = 1; k < 4; ++k) b = part[k][cl] < b ? part[k][cl] : b;
        cp.G[(cp.goff[n] + u) * C + c] = b >= kBig ? kInf64 : b;
      }
      __syncthreads();                              // arow / gw / part reused by the next tile
    }
    if (n > 0) mem_grid_sync(bar, gridDim.x, gen);  // G_n complete before step n - 1 reads it
  }
}

// --------------------------------------------------------------------------
// Optimal edges reachable from (u, c) = (0, 0): single CTA, instance by
// instance.  The reachable states of level n are listed (ballot compaction),
// then every (state, v, q) candidate is checked in parallel; optimal ones set
// the next level's reach bit and their bucket's `need` bit.  All levels'
// reach bitsets are kept (reach + goff[n] * C bits) for the successor table.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) mem_bfs_kernel(const MemChainParams cp, uint32_t* reach,
                                                       int32_t* slist, int64_t slist_cap, int maxw) {
  // the current and next levels' reach bits live in shared memory (the
  // global copy, for mem_succ_kernel, is written alongside)
  extern __shared__ uint32_t sbits[];
  uint32_t* cur = sbits;
  uint32_t* nxt = sbits + maxw;
  __shared__ int s_n;
  const int C = cp.C;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int w = tid; w < maxw; w += nth) cur[w] = 0;
  __syncthreads();
  if (tid == 0 && cp.G[0] != kInf64) { reach[0] = 1u; cur[0] = 1u; }   // (u, c) = (0, 0) at level 0
  for (int n = 0; n < cp.N; ++n) {
    const MemInst in = cp.inst[n];
    const int64_t base = cp.goff[n] * C, nbase = cp.goff[n + 1] * C;
    const int nw_cur = (int)(((int64_t)in.rows * C + 31) / 32);
    const int nw_nxt = (int)(((int64_t)in.cols * C + 31) / 32);
    for (int w = tid; w < nw_nxt; w += nth) nxt[w] = 0;
    if (tid == 0) s_n = 0;
    __syncthreads();
    for (int w = tid; w < nw_cur; w += nth) {          // list the reachable states, a word at a time
      uint32_t m = cur[w];
      if (!m) continue;
      int k = atomicAdd(&s_n, __popc(m));
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        if (k < slist_cap) slist[k] = w * 32 + b;
        ++k;
      }
    }
    __syncthreads();
    const int ns = (int)min((int64_t)s_n, slist_cap);
    const uint64_t* Gp = cp.G + base;
    const uint64_t* Gn = cp.G + nbase;
    uint32_t* need = cp.need + cp.need_off[in.slot];
    const int per = in.cols * in.nq;
    const int64_t work = (int64_t)ns * per;
    for (int64_t w = tid; w < work; w += nth) {
      const int si = (int)(w / per), r = (int)(w - (int64_t)si * per);
      const int v = r / in.nq, qi = r - v * in.nq;
      const int s = slist[si];
      const int u = s / C, c = s - u * C;
      const int cc = c + in.qlo + qi;
      if (cc >= C) continue;
      const int64_t cell = ((int64_t)u * in.cols + v) * in.nq + qi;
      const uint64_t a = in.Am[cell], g = Gn[(int64_t)v * C + cc];
      if (a == kInf64 || g == kInf64 || a + g != Gp[s]) continue;
      const int tl = v * C + cc;
      atomicOr(&nxt[tl >> 5], 1u << (tl & 31));
      const int64_t t = nbase + tl;
      atomicOr(&reach[t >> 5], 1u << (t & 31));
      atomicOr(&need[cell >> 5], 1u << (cell & 31));
    }
    __syncthreads();
    uint32_t* tmp = cur; cur = nxt; nxt = tmp;
  }
  // list the needed buckets
  for (int sl = 0; sl < cp.nslot; ++sl) {
    const int64_t w0 = cp.need_off[sl], w1 = cp.need_off[sl + 1];
    for (int64_t w = w0 + tid; w < w1; w += nth) {
      uint32_t m = cp.need[w];
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int64_t cell = (w - w0) * 32 + b;
        const int k = atomicAdd(cp.count, 1);
        if (k < cp.list_cap) cp.list[k] = MemArgEntry{sl, (int32_t)cell, 0, 0};   // decoded by the argmin
      }
    }
  }
}

// --------------------------------------------------------------------------
// Successor of every reachable state (all levels in parallel, one warp per
// state): among the optimal (v, q) the least combination index.
// succ[(goff[n] + u) * C + c] = v * nq + qi, -1 = none.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) mem_succ_kernel(const MemChainParams cp, const uint32_t* reach,
                                                       int32_t* succ) {
  const int C = cp.C;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = cp.goff[cp.N] * C;        // states of levels 0..N-1
  for (int64_t b = warp; b < total; b += nwarps) {
    if (!((reach[b >> 5] >> (b & 31)) & 1u)) continue;            // warp-uniform
    int n = 0;
    while (cp.goff[n + 1] * C <= b) ++n;
    const MemInst in = cp.inst[n];
    const int64_t s = b - cp.goff[n] * C;
    const int u = (int)(s / C), c = (int)(s % C);
    const uint64_t target = cp.G[b];
    const uint64_t* Gn = cp.G + cp.goff[n + 1] * C;
    uint64_t bi = kInf64;
    int bp = -1;
    for (int pr = lane; pr < in.cols * in.nq; pr += 32) {
      const int v = pr / in.nq, qi = pr % in.nq;
      const int cc = c + in.qlo + qi;
      if (cc >= C) continue;
      const int64_t cell = ((int64_t)u * in.cols + v) * in.nq + qi;
      const uint64_t a = in.Am[cell], g = Gn[(int64_t)v * C + cc];
      if (a == kInf64 || g == kInf64 || a + g != target) continue;
      const uint64_t ix = in.Im[cell];
      if (ix < bi) { bi = ix; bp = pr; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ob = __shfl_xor_sync(0xffffffffu, bi, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (op >= 0 && (bp < 0 || ob < bi || (ob == bi && op < bp))) { bi = ob; bp = op; }
    }
    if (lane == 0) succ[b] = bp;
  }
}

// --------------------------------------------------------------------------
// Least combination index of listed buckets.  One CTA per entry (grid-stride).
// --------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) mem_argmin_kernel(const MemArgSlot* __restrict__ slots,
                                                         const MemArgEntry* __restrict__ list,
                                                         const int32_t* __restrict__ count, int cell_mode) {
  using M = MT<V>;
  __shared__ int32_t s_tiles[1024];
  __shared__ int s_nt, s_over;
  __shared__ unsigned long long s_best, s_sig;
  const int tid = threadIdx.x;
  const int total = *count;
  for (int e = blockIdx.x; e < total; e += gridDim.x) {
    const MemArgEntry ent = list[e];
    const MemArgSlot& S = slots[ent.slot];
    int u, v, qi;
    int64_t cell;
    if (cell_mode) {                                 // entry = (slot, cell)
      cell = ent.u;
      qi = (int)(cell % S.nq);
      v = (int)((cell / S.nq) % S.Do);
      u = (int)(cell / ((int64_t)S.nq * S.Do));
    } else {
      u = ent.u; v = ent.v; qi = ent.qi;
      cell = ((int64_t)u * S.Do + v) * S.nq + qi;
    }
    const uint64_t A = S.Am[cell];
    if (A == kInf64) {
      if (tid == 0) S.Im[cell] = kInf64;
      continue;
    }
    const V target = (V)A;
    const int vslot = S.o_in_prefix ? 0 : v;
    if (tid == 0) { s_nt = 0; s_over = 0; s_best = ~0ull; s_sig = ~0ull; }
    __syncthreads();
    const V* ch = static_cast<const V*>(S.chunk);
    for (int t = tid; t < S.ntiles; t += 256) {
      const int rc = S.tiles[t].z;
      const int k = rc / S.nVp, vp = rc % S.nVp;
      if (S.o_in_prefix && vp != v) continue;
      const int rs = qi - k;
      if (rs < 0 || rs >= S.RQs) continue;
      if (ch[((int64_t)t * S.Din + u) * S.Wc + vslot * S.RQs + rs] == target) {
        const int k2 = atomicAdd(&s_nt, 1);
        if (k2 < 1024) s_tiles[k2] = t;
        else s_over = 1;
      }
    }
    __syncthreads();
    const int nt = s_over ? S.ntiles : s_nt;
    const V* vals = static_cast<const V*>(S.vals);
    const V* B = static_cast<const V*>(S.B);
    for (int i = 0; i < nt; ++i) {
      const int t = s_over ? i : s_tiles[i];
      const int4 tl = S.tiles[t];
      const int k = tl.z / S.nVp, vp = tl.z % S.nVp;
      if (S.o_in_prefix && vp != v) continue;
      const int rs = qi - k;
      if (rs < 0 || rs >= S.RQs) continue;
      for (int r = tid; r < tl.y; r += 256) {
        const int64_t pr = S.perm[tl.x + r];
        V x = 0;
        for (int j = 0; j < S.nqx; ++j)
          x = M::sat(x, vals[S.q_off[j] + (int64_t)mem_digit(S.pm, pr, S.q_pos[j]) * S.DinP + u]);
        const int cl = vslot * S.RQs + rs;
        const uint64_t b = (uint64_t)B[((int64_t)(cl >> 2) * S.nP + tl.x + r) * 4 + (cl & 3)];
        if ((uint64_t)x + b == (uint64_t)target)
          atomicMin(&s_best, (unsigned long long)(((uint64_t)pr << 32) | (uint64_t)t));
      }
    }
    __syncthreads();
    if (s_best == ~0ull) {                           // cannot happen for a finite A
      if (tid == 0) S.Im[cell] = kInf64;
      __syncthreads();
      continue;
    }
    const int64_t pstar = (int64_t)(s_best >> 32);
    const int rc = S.tiles[(int)(s_best & 0xFFFFFFFFu)].z;
    const int rs = qi - rc / S.nVp;
    const int cls = vslot * S.RQs + rs;
    const int64_t c = mem_ctx(S.pm, pstar);
    V xs = 0;                                        // X_{p*}[u]
    for (int j = 0; j < S.nqx; ++j)
      xs = M::sat(xs, vals[S.q_off[j] + (int64_t)mem_digit(S.pm, pstar, S.q_pos[j]) * S.DinP + u]);
    // the least suffix of p* in class (vslot, rs) -- plan memory
    // ceil((mP_g + mS) / quantum) = q0(g) + rs -- whose cost
    // K0[p*] + T[c][s] = A - X_{p*}[u]
    const V rel = target - xs - static_cast<const V*>(S.K0)[pstar];
    const V* T = static_cast<const V*>(S.Tc) + c * S.nS;
    const int g = S.gP[pstar];
    const uint64_t mPg = S.gmem[g];
    const int64_t qwant = (int64_t)S.gq0[g] + rs;
    (void)cls;
    for (int64_t s = tid; s < S.nS; s += 256)
      if (S.svs[s] == vslot && T[s] == rel) {
        const uint64_t m = mPg + S.sms[s];
        if ((int64_t)(m / S.quantum + (m % S.quantum != 0)) == qwant) atomicMin(&s_sig, (unsigned long long)s);
      }
    __syncthreads();
    if (tid == 0) S.Im[cell] = s_sig == ~0ull ? kInf64 : (uint64_t)pstar * (uint64_t)S.nS + s_sig;
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// Forward greedy from (0, 0) through the successor table (the least
// combination index among the optimal successors = canonical plan), then the
// digits (big-endian decode), one warp.
// --------------------------------------------------------------------------
__global__ void mem_greedy_kernel(const MemChainParams cp, const int32_t* succ) {
  const int lane = threadIdx.x;
  const int C = cp.C;
  if (lane == 0) {
    int status = cp.G[0] == kInf64 ? 3 : 0;
    int u = 0, c = 0;
    for (int n = 0; n < cp.N && status == 0; ++n) {
      const MemInst in = cp.inst[n];
      const int bp = succ[(cp.goff[n] + u) * C + c];
      if (bp < 0) { status = 3; break; }
      const int v = bp / in.nq, qi = bp % in.nq;
      const int64_t cell = ((int64_t)u * in.cols + v) * in.nq + qi;
      cp.seg_index[n] = in.Im[cell];
      cp.seg_ns[n] = in.Am[cell];
      cp.seg_q[n] = in.qlo + qi;
      u = v;
      c += in.qlo + qi;
    }
    *cp.status = status;
    *cp.total = status ? kInf64 : cp.G[0];
  }
  __syncwarp();
  if (*cp.status) return;
  for (int64_t w = lane; w < (int64_t)cp.N * cp.kmax; w += 32) {
    const int n = (int)(w / cp.kmax), j = (int)(w % cp.kmax);
    const MemInst in = cp.inst[n];
    int32_t d = -1;
    if (j < in.K) {
      uint64_t st = 1;
      for (int k = in.K - 1; k > j; --k) st *= (uint64_t)cp.radix[in.radix_off + k];
      d = (int32_t)((cp.seg_index[n] / st) % (uint64_t)cp.radix[in.radix_off + j]);
    }
    cp.digits[w] = d;
  }
}

// ---------------------------------------------------------------- launchers
template <typename V>
cudaError_t launch_mem_enum(const MemEnumParams& p, int64_t ntiles, int npf, cudaStream_t st) {
  const size_t smem = (size_t)p.Tlen * sizeof(V) + 16;
  if (ntiles <= 0) return cudaSuccess;
  auto go = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)ntiles, 256, smem, st>>>(p);
    return cudaGetLastError();
  };
  if (npf == 4) return go(mem_enum_kernel<V, 4>);
  if (npf == 2) return go(mem_enum_kernel<V, 2>);
  return go(mem_enum_kernel<V, 1>);
}
template <typename V>
cudaError_t launch_mem_values(const MemValJob* jobs, int njobs, int64_t nblocks, const uint32_t* raw,
                              cudaStream_t st) {
  if (njobs <= 0 || nblocks <= 0) return cudaSuccess;
  mem_values_kernel<V><<<(unsigned)nblocks, 256, 0, st>>>(jobs, njobs, raw);
  return cudaGetLastError();
}
template <typename V>
cudaError_t launch_mem_fold(const MemFoldParams& p, int64_t ntiles, cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  const int64_t xthreads = p.nP * (p.DinP / 4);
  mem_xrows_kernel<V><<<(unsigned)std::min<int64_t>(148 * 16, (xthreads + 255) / 256), 256, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (sizeof(V) == 4 && !getenv("CFP_MEM_FOLD4") && p.DinP <= 48) {
    // U states x 4 classes per thread (U = 12 / 8 / 4 dividing D_in padded);
    // column blocks so that (state groups) x (class quads) <= 256 threads
    const int U = p.DinP % 12 == 0 ? 12 : p.DinP % 8 == 0 ? 8 : 4;
    const int ngu = p.DinP / U;
    // <= 64 KB of stages per CTA
    const int fcmax = (int)(64 * 1024 / (kFoldUS * kFoldUR * sizeof(uint32_t))) - p.DinP - 4;
    const int ncq = (p.Wc + 3) / 4, qmax = std::max(1, std::min(256 / ngu, fcmax / 4));
    // (a column-block / CTAs-per-SM choice for whole waves was measured
    // slower on both C3 and C5 and dropped)
    MemFoldParams q = p;
    q.ncolblk = (ncq + qmax - 1) / qmax;
    q.fc = ((ncq + q.ncolblk - 1) / q.ncolblk) * 4;
    const int nthr = (ngu * (q.fc / 4) + 31) / 32 * 32;
    const size_t smem = (size_t)kFoldUS * kFoldUR * (p.DinP + q.fc + 4) * sizeof(uint32_t);
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e2 != cudaSuccess) return e2;
      kern<<<dim3((unsigned)ntiles, (unsigned)q.ncolblk), nthr, smem, st>>>(q);
      return cudaGetLastError();
    };
    if (U == 12) return go(mem_fold_u_kernel<12>);
    if (U == 8) return go(mem_fold_u_kernel<8>);
    return go(mem_fold_u_kernel<4>);
  }
  // threads = (u quads of one 32-state block) x (class quads): no idle threads
  // when D_in < 32 (C3: 6 x 30 -> 192 instead of 256 with 76 idle)
  const int ntu = std::min(8, (std::min(32, p.DinP) + 3) / 4);
  const int nthr = std::min(256, (ntu * ((p.fc + 3) / 4) + 31) / 32 * 32);
  constexpr int R = kMemFoldStage / (int)sizeof(V);
  const size_t smem = (size_t)2 * R * 32 * sizeof(V) + (size_t)2 * R * (p.fc + 4) * sizeof(V);
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(mem_fold_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  mem_fold_kernel<V><<<dim3((unsigned)ntiles, (unsigned)p.ncolblk), nthr, smem, st>>>(p);
  return cudaGetLastError();
}
template <typename V>
cudaError_t launch_mem_amin(const MemAminParams& p, cudaStream_t st) {
  const int64_t total = (int64_t)p.Din * p.Do * p.nq;
  if (total <= 0) return cudaSuccess;
  mem_amin_kernel<V><<<(unsigned)((total * 32 + 255) / 256), 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_mem_chain_step(const MemChainParams& cp, int n, int rows, int cols, int nq, cudaStream_t st) {
  const int rowlen = cols * nq;
  int win = 64 + nq - 1;                            // G_{n+1} window per CTA in shared memory
  size_t smem = (size_t)((rowlen + 1) & ~1) * 8 + (size_t)cols * win * 8 + 16;
  if (smem > 160 * 1024) {                          // too wide: read G_{n+1} from L2
    win = 0;
    smem = (size_t)((rowlen + 1) & ~1) * 8 + 16;
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mem_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  mem_chain_kernel<<<dim3((unsigned)rows, (unsigned)((cp.C + 63) / 64)), 256, smem, st>>>(cp, n, win);
  return cudaGetLastError();
}
// every step of the backward DP in one cooperative launch; bar: 2 zeroed words
cudaError_t launch_mem_chain_all(const MemChainParams& cp, int max_rowlen, int max_cols, int max_nq, int max_rows,
                                 unsigned int* bar, int sms, cudaStream_t st) {
  size_t smem = (size_t)((max_rowlen + 1) & ~1) * 8 + (size_t)max_cols * (64 + max_nq - 1) * 8 + 16;
  if (smem > 160 * 1024) smem = (size_t)((max_rowlen + 1) & ~1) * 8 + 16;   // windows off for the widest
  cudaError_t e = cudaFuncSetAttribute(mem_chain_all_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mem_chain_all_kernel, 256, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int tiles = max_rows * ((cp.C + 63) / 64);
  int grid = std::min(sms * per_sm, tiles);
  if (grid < 1) grid = 1;
  e = cudaMemsetAsync(bar, 0, 8, st);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<MemChainParams*>(&cp), &smem, &bar};
  return cudaLaunchCooperativeKernel((void*)mem_chain_all_kernel, dim3((unsigned)grid), dim3(256), args, smem, st);
}
cudaError_t launch_mem_bfs(const MemChainParams& cp, uint32_t* reach, int32_t* slist, int64_t slist_cap,
                           int max_dim, cudaStream_t st) {
  const int maxw = (int)(((int64_t)max_dim * cp.C + 31) / 32);
  const size_t smem = (size_t)maxw * 2 * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mem_bfs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  mem_bfs_kernel<<<1, 1024, smem, st>>>(cp, reach, slist, slist_cap, maxw);
  return cudaGetLastError();
}
cudaError_t launch_mem_succ(const MemChainParams& cp, const uint32_t* reach, int32_t* succ, int64_t states,
                            cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(4096, (states * 32 + 255) / 256 + 1);
  mem_succ_kernel<<<(unsigned)blocks, 256, 0, st>>>(cp, reach, succ);
  return cudaGetLastError();
}
template <typename V>
cudaError_t launch_mem_argmin(const MemArgSlot* slots, const MemArgEntry* list, const int32_t* count, int grid,
                              int cell_mode, cudaStream_t st) {
  mem_argmin_kernel<V><<<grid, 256, 0, st>>>(slots, list, count, cell_mode);
  return cudaGetLastError();
}
cudaError_t launch_mem_greedy(const MemChainParams& cp, const int32_t* succ, cudaStream_t st) {
  mem_greedy_kernel<<<1, 32, 0, st>>>(cp, succ);
  return cudaGetLastError();
}

template cudaError_t launch_mem_values<uint32_t>(const MemValJob*, int, int64_t, const uint32_t*, cudaStream_t);
template cudaError_t launch_mem_values<uint64_t>(const MemValJob*, int, int64_t, const uint32_t*, cudaStream_t);
template cudaError_t launch_mem_enum<uint32_t>(const MemEnumParams&, int64_t, int, cudaStream_t);
template cudaError_t launch_mem_enum<uint64_t>(const MemEnumParams&, int64_t, int, cudaStream_t);
template cudaError_t launch_mem_fold<uint32_t>(const MemFoldParams&, int64_t, cudaStream_t);
template cudaError_t launch_mem_fold<uint64_t>(const MemFoldParams&, int64_t, cudaStream_t);
template cudaError_t launch_mem_amin<uint32_t>(const MemAminParams&, cudaStream_t);
template cudaError_t launch_mem_amin<uint64_t>(const MemAminParams&, cudaStream_t);
template cudaError_t launch_mem_argmin<uint32_t>(const MemArgSlot*, const MemArgEntry*, const int32_t*, int, int,
                                                 cudaStream_t);
template cudaError_t launch_mem_argmin<uint64_t>(const MemArgSlot*, const MemArgEntry*, const int32_t*, int, int,
                                                 cudaStream_t);

}  // namespace cfp
