// cfp_dense.cu -- sm_100a kernels of the dense per-plan-table search
// (the paper profiles every
// whole-segment plan, so a segment type's cost table W_t[idx] has one entry
// per strategy combination and nothing factorises -- the enumeration must
// read every entry: an HBM stream, 4 bytes per combination).
//
//   dense_fill_kernel   synthetic tables (counter-based splitmix64, the same
//                       stream as synth.generators.dense_table)
//   dense_rows_kernel   B_p[v] = min over prefix p's row of W with s_o = v
//                       (one coalesced 16-byte load per 4 combinations, one
//                       IMNMX per combination; persistent CTAs)
//   dense_fold_kernel   cross terms: chunk[u][v] = min_p X_p[u] + B_p[v]
//   dense_amin_kernel   A[u][v] = min over chunks
//   dense_argmin_kernel least combination index: first attaining chunk,
//                       least prefix in it, least suffix of that prefix
//   dense_chain_kernel  G_N = 0, G_{n-1}(u) = min_v A[u][v] + G_n(v); forward
//                       greedy with the least index among optimal successors
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cfp_internal.h"

namespace cfp {

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t dense_value(uint64_t e, uint64_t base) {
  const uint64_t h = d_splitmix64(e ^ base);
  return (h & 0xFFFull) == 0 ? 0xFFFFFFFFu : (uint32_t)(h >> 40);
}

__global__ void dense_fill_kernel(uint32_t* __restrict__ W, uint64_t n, uint64_t base) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t e = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; e < n; e += stride) {
    if (e + 4 <= n && (reinterpret_cast<uintptr_t>(W + e) & 15) == 0) {
      uint4 v;
      v.x = dense_value(e, base);
      v.y = dense_value(e + 1, base);
      v.z = dense_value(e + 2, base);
      v.w = dense_value(e + 3, base);
      *reinterpret_cast<uint4*>(W + e) = v;
    } else {
      for (uint64_t k = e; k < e + 4 && k < n; ++k) W[k] = dense_value(k, base);
    }
  }
}

// --------------------------------------------------------------------------
// Row minima.  Row p = the nS consecutive entries of prefix p.  Mode A (the
// output block is the last digit): v(e) = e % Do; the CTA uses T threads with
// 4T a multiple of Do, so each thread's four lanes of every 16-byte load keep
// fixed v's and the reduction needs four registers per thread.  Mode B (the
// output digit is in the prefix): one minimum per row.
// --------------------------------------------------------------------------
template <bool VEC>
__global__ void __launch_bounds__(256) dense_rows_kernel(const DenseRowParams p) {
  __shared__ uint32_t smin[2][64];
  const int tid = threadIdx.x;
  const int T = p.T;
  const bool act = tid < T;
  const int nv = p.nVs;
  int buf = 0;
  for (int64_t r = blockIdx.x; r < p.nP; r += gridDim.x) {
    const uint32_t* row = p.W + r * p.nS;
    if (tid < nv) smin[buf][tid] = 0xFFFFFFFFu;
    uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, a2 = 0xFFFFFFFFu, a3 = 0xFFFFFFFFu;
    if (act) {
      if constexpr (VEC) {
        const uint4* row4 = reinterpret_cast<const uint4*>(row);
        const int64_t n4 = p.nS >> 2;
#pragma unroll 4
        for (int64_t j = tid; j < n4; j += T) {
          const uint4 x = __ldcs(row4 + j);          // streamed once: evict-first
          a0 = min(a0, x.x);
          a1 = min(a1, x.y);
          a2 = min(a2, x.z);
          a3 = min(a3, x.w);
        }
      } else {
#pragma unroll 4
        for (int64_t j = tid; j < p.nS; j += T) a0 = min(a0, __ldcs(row + j));
      }
    }
    __syncthreads();
    if (act) {
      if (nv == 1) {
        atomicMin(&smin[buf][0], min(min(a0, a1), min(a2, a3)));
      } else if constexpr (VEC) {
        atomicMin(&smin[buf][(4 * tid) % nv], a0);
        atomicMin(&smin[buf][(4 * tid + 1) % nv], a1);
        atomicMin(&smin[buf][(4 * tid + 2) % nv], a2);
        atomicMin(&smin[buf][(4 * tid + 3) % nv], a3);
      } else {
        atomicMin(&smin[buf][tid % nv], a0);
      }
    }
    __syncthreads();
    if (tid < nv) p.B[r * nv + tid] = smin[buf][tid];
    buf ^= 1;                                          // next row reduces into the other buffer
  }
}

// X_p[u] = sum_cross Q_j[u][s_j(p)] (INF absorbing, u64)
__device__ __forceinline__ uint64_t dense_x(const DenseSlotParams& s, int64_t p, int u) {
  uint64_t x = 0;
  for (int i = 0; i < s.nq; ++i) {
    const int dig = (int)((p / s.q_stride[i]) % s.q_radix[i]);
    const uint32_t q = s.Q[s.q_off[i] + (int64_t)u * s.q_radix[i] + dig];
    if (q == 0xFFFFFFFFu) return kInf64;
    x += q;
  }
  return x;
}
__device__ __forceinline__ int dense_vp(const DenseSlotParams& s, int64_t p) {
  return s.nVs == 1 ? (int)((p / s.o_stride) % s.Do) : -1;
}

// --------------------------------------------------------------------------
// Fold: chunk c = prefixes [c * kDenseChunk, ...).  Thread = (u, v) pairs.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dense_fold_kernel(const DenseSlotParams s) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int R = kDenseChunk;
  uint64_t (*Xs)[32] = reinterpret_cast<uint64_t (*)[32]>(smem_raw);           // [R][32]
  uint32_t* Bs = reinterpret_cast<uint32_t*>(smem_raw + R * 32 * 8);            // [R][nVs]
  int32_t* vps = reinterpret_cast<int32_t*>(Bs + R * s.nVs);                    // [R]
  const int64_t p0 = (int64_t)blockIdx.x * R;
  const int rows = s.nP - p0 < R ? (int)(s.nP - p0) : R;
  const int tid = threadIdx.x;
  for (int ub = 0; ub < s.Din; ub += 32) {
    const int uc = min(32, s.Din - ub);
    for (int r = tid; r < rows; r += 256) {          // digits once per row, then every u
      const int64_t p = s.p_lo + p0 + r;             // global prefix (digits)
      int64_t base[kMaxCross];
      for (int i = 0; i < s.nq; ++i)
        base[i] = s.q_off[i] + (int64_t)((p / s.q_stride[i]) % s.q_radix[i]);
      for (int u = 0; u < uc; ++u) {
        uint64_t x = 0;
        for (int i = 0; i < s.nq && x != kInf64; ++i) {
          const uint32_t q = s.Q[base[i] + (int64_t)(ub + u) * s.q_radix[i]];
          x = q == 0xFFFFFFFFu ? kInf64 : x + q;
        }
        Xs[r][u] = x;
      }
    }
    for (int e = tid; e < rows * s.nVs; e += 256) {
      const int r = e / s.nVs, v = e % s.nVs;
      Bs[r * s.nVs + v] = s.B[(p0 + r) * s.nVs + v];
    }
    for (int r = tid; r < rows; r += 256) vps[r] = dense_vp(s, s.p_lo + p0 + r);
    __syncthreads();
    for (int e = tid; e < uc * s.Do; e += 256) {
      const int u = e / s.Do, v = e % s.Do;
      uint64_t best = kInf64;
      for (int r = 0; r < rows; ++r) {
        const uint64_t x = Xs[r][u];
        uint32_t b;
        if (s.nVs == 1) {
          if (vps[r] != v) continue;
          b = Bs[r];
        } else {
          b = Bs[r * s.nVs + v];
        }
        if (x == kInf64 || b == 0xFFFFFFFFu) continue;
        const uint64_t c = x + b;
        best = c < best ? c : best;
      }
      s.chunk[((int64_t)blockIdx.x * s.Din + ub + u) * s.Do + v] = best;
    }
    __syncthreads();
  }
}

__global__ void dense_amin_kernel(const DenseSlotParams s) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= (int64_t)s.Din * s.Do) return;
  uint64_t best = kInf64;
  for (int64_t c = lane; c < s.nchunks; c += 32) {
    const uint64_t x = s.chunk[c * s.Din * s.Do + e];
    best = x < best ? x : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y < best ? y : best;
  }
  if (lane == 0) s.A[e] = best;
}

// --------------------------------------------------------------------------
// Least index of bucket (u, v): first chunk attaining A, least prefix of it
// with X_p[u] + B_p[v] = A, least suffix of that prefix with W = B_p[v] and
// output digit v.  One CTA per bucket (grid-stride over all buckets).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dense_argmin_kernel(const DenseSlotParams* __restrict__ slots,
                                                           const int2* __restrict__ list, int count) {
  __shared__ unsigned long long s_c, s_p, s_s;
  const int tid = threadIdx.x;
  for (int e = blockIdx.x; e < count; e += gridDim.x) {
    const DenseSlotParams& s = slots[list[e].x];
    const int cell = list[e].y;
    const int u = cell / s.Do, v = cell % s.Do;
    const uint64_t A = s.A[cell];
    if (A == kInf64) {
      if (tid == 0) s.I[cell] = kInf64;
      continue;
    }
    if (tid == 0) { s_c = ~0ull; s_p = ~0ull; s_s = ~0ull; }
    __syncthreads();
    for (int64_t c = tid; c < s.nchunks; c += 256)
      if (s.chunk[(c * s.Din + u) * s.Do + v] == A) atomicMin(&s_c, (unsigned long long)c);
    __syncthreads();
    const int64_t p0 = (int64_t)s_c * kDenseChunk;
    const int rows = s.nP - p0 < kDenseChunk ? (int)(s.nP - p0) : kDenseChunk;
    for (int r = tid; r < rows; r += 256) {
      const int64_t p = p0 + r;                      // local row; digits of the global prefix
      if (s.nVs == 1 && dense_vp(s, s.p_lo + p) != v) continue;
      const uint64_t x = dense_x(s, s.p_lo + p, u);
      const uint32_t b = s.B[p * s.nVs + (s.nVs == 1 ? 0 : v)];
      if (x != kInf64 && b != 0xFFFFFFFFu && x + b == A) atomicMin(&s_p, (unsigned long long)p);
    }
    __syncthreads();
    const int64_t ps = (int64_t)s_p;
    const uint32_t b = s.B[ps * s.nVs + (s.nVs == 1 ? 0 : v)];
    const uint32_t* row = s.W + ps * s.nS;
    for (int64_t j = tid; j < s.nS; j += 256)
      if (row[j] == b && (s.nVs == 1 || (int)(j % s.Do) == v)) atomicMin(&s_s, (unsigned long long)j);
    __syncthreads();
    if (tid == 0) s.I[cell] = (uint64_t)(s.p_lo + ps) * (uint64_t)s.nS + s_s;
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// Chain + plan, one CTA: backward DP (warp per state), forward greedy.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) dense_chain_kernel(const DenseChainParams cp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int N = cp.N;
  for (int v = tid; v < cp.inst[N - 1].cols; v += blockDim.x) cp.G[cp.goff[N] + v] = 0;
  __syncthreads();
  for (int n = N - 1; n >= 0; --n) {
    const DenseInst in = cp.inst[n];
    const uint64_t* Gn = cp.G + cp.goff[n + 1];
    for (int u = warp; u < in.rows; u += nw) {
      uint64_t b = kInf64;
      for (int v = lane; v < in.cols; v += 32) {
        const uint64_t a = in.A[(int64_t)u * in.cols + v], g = Gn[v];
        if (a != kInf64 && g != kInf64 && a + g < b) b = a + g;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, b, o);
        b = y < b ? y : b;
      }
      if (lane == 0) cp.G[cp.goff[n] + u] = b;
    }
    __syncthreads();
  }
  if (warp != 0) return;
  int status = cp.G[0] == kInf64 ? 3 : 0;
  int u = 0;
  for (int n = 0; n < N && status == 0; ++n) {
    const DenseInst in = cp.inst[n];
    const uint64_t target = cp.G[cp.goff[n] + u];
    const uint64_t* Gn = cp.G + cp.goff[n + 1];
    uint64_t bi = kInf64;
    int bv = -1;
    for (int v = lane; v < in.cols; v += 32) {
      const uint64_t a = in.A[(int64_t)u * in.cols + v], g = Gn[v];
      if (a == kInf64 || g == kInf64 || a + g != target) continue;
      const uint64_t ix = in.I[(int64_t)u * in.cols + v];
      if (ix < bi) { bi = ix; bv = v; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ob = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
      if (ov >= 0 && (bv < 0 || ob < bi || (ob == bi && ov < bv))) { bi = ob; bv = ov; }
    }
    if (bv < 0) { status = 3; break; }
    if (lane == 0) {
      cp.seg_index[n] = bi;
      cp.seg_ns[n] = in.A[(int64_t)u * in.cols + bv];
    }
    u = bv;
  }
  if (lane == 0) {
    *cp.status = status;
    *cp.total = status ? kInf64 : cp.G[0];
  }
  __syncwarp();
  if (status) return;
  for (int64_t w = lane; w < (int64_t)N * cp.kmax; w += 32) {
    const int n = (int)(w / cp.kmax), j = (int)(w % cp.kmax);
    const DenseInst in = cp.inst[n];
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
cudaError_t launch_dense_fill(uint32_t* W, uint64_t n, uint64_t base, cudaStream_t st) {
  const uint64_t blocks = std::min<uint64_t>(148ull * 16, (n / 4 + 255) / 256 + 1);
  dense_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(W, n, base);
  return cudaGetLastError();
}
cudaError_t launch_dense_rows(const DenseRowParams& p, int sms, cudaStream_t st) {
  const int64_t grid = std::min<int64_t>(p.nP, (int64_t)sms * 8);
  if (grid <= 0) return cudaSuccess;
  if (p.vec) dense_rows_kernel<true><<<(unsigned)grid, 256, 0, st>>>(p);
  else dense_rows_kernel<false><<<(unsigned)grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_dense_fold(const DenseSlotParams& s, cudaStream_t st) {
  const size_t smem = kDenseChunk * 32 * 8 + (size_t)kDenseChunk * s.nVs * 4 + kDenseChunk * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(dense_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (s.nchunks > 0) {                               // (an empty shard: A = INF from the minima below)
    dense_fold_kernel<<<(unsigned)s.nchunks, 256, smem, st>>>(s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int64_t tot = (int64_t)s.Din * s.Do;
  dense_amin_kernel<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, st>>>(s);
  return cudaGetLastError();
}
cudaError_t launch_dense_argmin(const DenseSlotParams* slots, const int2* list, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dense_argmin_kernel<<<std::min(count, 1184), 256, 0, st>>>(slots, list, count);
  return cudaGetLastError();
}
cudaError_t launch_dense_chain(const DenseChainParams& cp, cudaStream_t st) {
  dense_chain_kernel<<<1, 1024, 0, st>>>(cp);
  return cudaGetLastError();
}

}  // namespace cfp
