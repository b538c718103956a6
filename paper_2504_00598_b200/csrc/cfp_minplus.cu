// cfp_minplus.cu -- N2: tiled tropical (min,+) product on the integer ALU pipe.
//
//   C[i][j] = min_k A[i][k] + B[k][j]
//
// This is a GEMM-shaped loop nest but not a multiply-add contraction, so it
// runs on the ALU pipe, not the tensor cores: one fused add+min
// (VIADDMNMX.U32) per (i, j, k) in the narrow path.  128x128 output tile per
// CTA, 256 threads x (8x8) register-blocked accumulators, 16-deep k slices
// staged through double-buffered shared memory: per k step a thread issues
// four LDS.128 and 64 VIADDMNMX.
//
// Narrow path: entries in [0, CAP32], CAP32 = 2^31-1 = infinity; the host only
// selects it when every finite a + b < CAP32.  Wide path: uint64 with
// CAP64 = 2^63-1.  ARGK variant tracks the least k attaining each minimum
// (strict '<' in increasing k).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cfp_internal.h"

namespace cfp {

namespace mp {

template <typename V> struct Ops;
template <> struct Ops<uint32_t> {
  static constexpr uint32_t CAP = kCap32;
  static __device__ __forceinline__ uint32_t addmin(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_u32(a, b, c);
  }
};
template <> struct Ops<uint64_t> {
  static constexpr uint64_t CAP = kCap64;
  static __device__ __forceinline__ uint64_t addmin(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t s = a + b;
    return s < c ? s : c;
  }
};

constexpr int BM = 128, BN = 128, BK32 = 16, BK64 = 8, TM = 8, TN = 8;

template <typename V>
__device__ __forceinline__ void lds4(const V* p, V* o) {
  if constexpr (sizeof(V) == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
    const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(p);
    const ulonglong2 v1 = *reinterpret_cast<const ulonglong2*>(p + 2);
    o[0] = v0.x; o[1] = v0.y; o[2] = v1.x; o[3] = v1.y;
  }
}

template <typename V, bool ARGK>
__global__ void __launch_bounds__(256, sizeof(V) == 4 ? 2 : 1) minplus_tiled_kernel(int m, int k, int n, const V* __restrict__ A,
                                                            const V* __restrict__ B, V* __restrict__ C,
                                                            uint32_t* __restrict__ argk) {
  using O = Ops<V>;
  constexpr int BK = sizeof(V) == 4 ? BK32 : BK64;   // 64 KB of static smem max
  constexpr int LQ = BK * BM / 256;                  // staged elements per thread per operand
  __shared__ __align__(16) V As[2][BK][BM];
  __shared__ __align__(16) V Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int bm = blockIdx.y * BM, bn = blockIdx.x * BN;
  // global -> register staging: A: row = tid / (BK/LQ), LQ consecutive k;
  //                             B: kk = tid / (BN/LQ), LQ consecutive cols
  const int a_row = tid / (BK / LQ), a_k = (tid % (BK / LQ)) * LQ;
  const int b_k = tid / (BN / LQ), b_col = (tid % (BN / LQ)) * LQ;
  V ra[LQ], rb[LQ];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < LQ; ++q) {
      const int gi = bm + a_row, gk = k0 + a_k + q;
      ra[q] = (gi < m && gk < k) ? A[(int64_t)gi * k + gk] : O::CAP;
      const int gk2 = k0 + b_k, gj = bn + b_col + q;
      rb[q] = (gk2 < k && gj < n) ? B[(int64_t)gk2 * n + gj] : O::CAP;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < LQ; ++q) As[buf][a_k + q][a_row] = ra[q];
#pragma unroll
    for (int q = 0; q < LQ; ++q) Bs[buf][b_k][b_col + q] = rb[q];
  };
  V acc[TM][TN];
  uint32_t idx[ARGK ? TM : 1][ARGK ? TN : 1];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      acc[i][j] = O::CAP;
      if constexpr (ARGK) idx[i][j] = 0xFFFFFFFFu;
    }
  const int nk = (k + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load_tile((t + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      V a[TM], b[TN];
      lds4<V>(&As[buf][kk][ty * 4], a);
      lds4<V>(&As[buf][kk][64 + ty * 4], a + 4);
      lds4<V>(&Bs[buf][kk][tx * 4], b);
      lds4<V>(&Bs[buf][kk][64 + tx * 4], b + 4);
      if constexpr (ARGK) {
        const uint32_t kg = (uint32_t)(t * BK + kk);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            const V s = a[i] + b[j];
            if (s < acc[i][j]) { acc[i][j] = s; idx[i][j] = kg; }
          }
      } else {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = O::addmin(a[i], b[j], acc[i][j]);
      }
    }
    if (t + 1 < nk) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gi = bm + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gi >= m) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gj = bn + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gj >= n) continue;
      C[(int64_t)gi * n + gj] = acc[i][j];
      if constexpr (ARGK) argk[(int64_t)gi * n + gj] = acc[i][j] >= O::CAP ? 0xFFFFFFFFu : idx[i][j];
    }
  }
}

// uint64 (INF64 = no edge) <-> path values (CAP = no edge)
template <typename V>
__global__ void to_path_kernel(const uint64_t* __restrict__ in, V* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] == kInf64 ? Ops<V>::CAP : (V)in[i];
}
template <typename V>
__global__ void from_path_kernel(const V* __restrict__ in, const uint32_t* __restrict__ ak, uint64_t* __restrict__ out,
                                 uint64_t* __restrict__ aout, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool inf = in[i] >= Ops<V>::CAP;
    out[i] = inf ? kInf64 : (uint64_t)in[i];
    if (aout) aout[i] = (inf || ak[i] == 0xFFFFFFFFu) ? kInf64 : (uint64_t)ak[i];
  }
}

// synthetic operands for the microbenchmark: hash-generated, values < 2^20
template <typename V>
__global__ void fill_random_kernel(V* __restrict__ p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (V)(z & 0xFFFFF);
  }
}

// batched (min,+) matrix-vector products of the large-S chain:
// out_k = P (x) g_k for a batch of vectors (one warp per output row)
__global__ void matvec_batch_kernel(const uint64_t* __restrict__ P, int rows, int cols,
                                    const uint64_t* __restrict__ G, const int64_t* __restrict__ src_off,
                                    const int64_t* __restrict__ dst_off, uint64_t* __restrict__ Gout, int nvec) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)nvec * rows) return;
  const int vec = (int)(w / rows), u = (int)(w % rows);
  const uint64_t* g = G + src_off[vec];
  uint64_t best = kInf64;
  for (int v = lane; v < cols; v += 32) {
    const uint64_t a = P[(int64_t)u * cols + v], b = g[v];
    const uint64_t s = (a == kInf64 || b == kInf64) ? kInf64 : a + b;
    best = s < best ? s : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
    best = ob < best ? ob : best;
  }
  if (lane == 0) Gout[dst_off[vec] + u] = best;
}

}  // namespace mp

template <typename V>
cudaError_t launch_minplus_tiled(int m, int k, int n, const V* A, const V* B, V* C, uint32_t* argk,
                                 cudaStream_t st) {
  dim3 grid((n + mp::BN - 1) / mp::BN, (m + mp::BM - 1) / mp::BM);
  if (argk) mp::minplus_tiled_kernel<V, true><<<grid, 256, 0, st>>>(m, k, n, A, B, C, argk);
  else mp::minplus_tiled_kernel<V, false><<<grid, 256, 0, st>>>(m, k, n, A, B, C, nullptr);
  return cudaGetLastError();
}

template <typename V>
cudaError_t launch_to_path(const uint64_t* in, V* out, int64_t n, cudaStream_t st) {
  mp::to_path_kernel<V><<<(unsigned)std::min<int64_t>(4096, (n + 255) / 256 + 1), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

template <typename V>
cudaError_t launch_from_path(const V* in, const uint32_t* ak, uint64_t* out, uint64_t* aout, int64_t n,
                             cudaStream_t st) {
  mp::from_path_kernel<V><<<(unsigned)std::min<int64_t>(4096, (n + 255) / 256 + 1), 256, 0, st>>>(in, ak, out,
                                                                                                  aout, n);
  return cudaGetLastError();
}

template <typename V>
cudaError_t launch_fill_random(V* p, int64_t n, uint64_t seed, cudaStream_t st) {
  mp::fill_random_kernel<V><<<(unsigned)std::min<int64_t>(4096, (n + 255) / 256 + 1), 256, 0, st>>>(p, n, seed);
  return cudaGetLastError();
}

cudaError_t launch_matvec_batch(const uint64_t* P, int rows, int cols, const uint64_t* G, const int64_t* src_off,
                                const int64_t* dst_off, uint64_t* Gout, int nvec, cudaStream_t st) {
  const int64_t warps = (int64_t)nvec * rows;
  mp::matvec_batch_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(P, rows, cols, G, src_off, dst_off,
                                                                                Gout, nvec);
  return cudaGetLastError();
}

template cudaError_t launch_minplus_tiled<uint32_t>(int, int, int, const uint32_t*, const uint32_t*, uint32_t*,
                                                    uint32_t*, cudaStream_t);
template cudaError_t launch_minplus_tiled<uint64_t>(int, int, int, const uint64_t*, const uint64_t*, uint64_t*,
                                                    uint32_t*, cudaStream_t);
template cudaError_t launch_to_path<uint32_t>(const uint64_t*, uint32_t*, int64_t, cudaStream_t);
template cudaError_t launch_to_path<uint64_t>(const uint64_t*, uint64_t*, int64_t, cudaStream_t);
template cudaError_t launch_from_path<uint32_t>(const uint32_t*, const uint32_t*, uint64_t*, uint64_t*, int64_t,
                                                cudaStream_t);
template cudaError_t launch_from_path<uint64_t>(const uint64_t*, const uint32_t*, uint64_t*, uint64_t*, int64_t,
                                                cudaStream_t);
template cudaError_t launch_fill_random<uint32_t>(uint32_t*, int64_t, uint64_t, cudaStream_t);
template cudaError_t launch_fill_random<uint64_t>(uint64_t*, int64_t, uint64_t, cudaStream_t);

}  // namespace cfp
