// cfp_profile.cu -- SURVEY §8(f) NEXT-3 on sm_100a: the dynamic profiling
// time budget ("continuously updated based on the fastest observed
// parallelism plans, aggressively trimming the profiling of inefficient or
// stalled executions") over a type's dense per-plan table W[idx] (uint32 ns,
// CFP_INF32 = infeasible program), in canonical index order (DESIGN R-B1..4):
//
//    best_i  = min_{j < i} W[j]                      (exclusive prefix minimum)
//    thr_i   = floor(best_i * num / den)              (f = num / den >= 1)
//    pruned  = W[i] finite, best_i finite, W[i] > thr_i  (== W*den > best*num)
//    spent  += pruned ? thr_i : (W[i] finite ? W[i] : 0)
//
// HBM sees each task once (up to the pass-2 L2 misses below): a persistent
// grid takes kBudSlice-task slices (49152 tasks = 192 KB) in index order from
// a ticket counter; pass 1 streams the slice from HBM for
// its minimum (published at once), a decoupled look-back over the earlier
// slices' status words (aggregate published before the look-back, inclusive
// prefix after it) gives the minimum of everything before the slice, and pass
// 2 re-reads the slice from L2 for the per-task decisions.
// The exclusive minimum changes only at a strict new best (rare): the
// division for thr runs there, every other task costs a few ops.
#include <cuda_runtime.h>

#include <cstdint>

#include "cfp_internal.h"

namespace cfp {

constexpr int kBudThreads = 256;
constexpr int kBudPer = 16;                          // tasks per thread per tile
constexpr int kBudTile = kBudThreads * kBudPer;      // 4096
constexpr int kBudSlice = 12 * kBudTile;            // 49152 tasks = 192 KB per ticket (measured: 128 KB 0.616, 192 KB 0.645, 256 KB 0.631 of HBM -- L2 residency of the slices in flight)
constexpr uint32_t kInf32 = 0xFFFFFFFFu;

struct BudgetParams {
  const uint32_t* W;
  uint64_t n;
  uint32_t ntiles;              // slices of kBudSlice tasks
  uint32_t num, den;
  unsigned long long* status;   // [ntiles]: (flag << 32) | min; flag 1 = slice aggregate, 2 = inclusive prefix
  unsigned int* ticket;         // next slice
  unsigned long long* acc;      // [8]: pruned, infeasible, spent lo/hi, full lo/hi, best (min), best index (max)
};

__device__ __forceinline__ uint32_t budget_thr(uint32_t best, uint32_t num, uint32_t den) {
  if (best == kInf32) return kInf32;                 // no completed task yet: nothing is pruned
  const uint64_t t = (uint64_t)best * num / den;
  return t >= kInf32 ? kInf32 - 1 : (uint32_t)t;     // >= every finite W: nothing is pruned
}

__device__ __forceinline__ void add128(uint64_t& lo, uint64_t& hi, uint64_t x) {
  lo += x;
  hi += lo < x ? 1 : 0;
}

__device__ __forceinline__ uint4 ld_stream(const uint32_t* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}

// Blocked layout for the decision pass: lane l of warp w holds the 16
// consecutive tasks tbase + w*512 + l*16 .. +15 (four 16-byte loads through
// L1, so the lines the warp touches are fetched from L2 once).
__device__ __forceinline__ void budget_load(const BudgetParams& p, uint64_t tbase, int warp, int lane,
                                            uint32_t (&v)[16]) {
  const uint64_t base = tbase + (uint64_t)warp * 512 + (uint64_t)lane * 16;
  if (tbase + kBudTile <= p.n) {
    const uint4* q = reinterpret_cast<const uint4*>(p.W + base);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 x = __ldg(q + j);
      v[4 * j] = x.x; v[4 * j + 1] = x.y; v[4 * j + 2] = x.z; v[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = base + k < p.n ? p.W[base + k] : kInf32;   // padding = min identity
  }
}

// A CTA takes a slice of kBudSlice tasks (ticket order) and reads it twice
// (16 loads of 16 bytes in flight per thread in pass 1; pass 2 prefetches
// the next tile):
// pass 1 streams it from HBM for its minimum (published at once for the
// look-back of later slices), pass 2 re-reads it -- mostly L2-resident: the
// slices in flight total <= grid x kBudSlice x 4 B (444 CTAs x 192 KB =
// 85 MB of the 126 MB L2; ncu: 22.3 GB of DRAM reads for an 18.35 GB table,
// i.e. ~18 % of the pass-2 re-reads miss, profiles/r02_ncu_budget_v8.json).
// The ticket, look-back and barriers are paid per slice instead of per tile.
__global__ void __launch_bounds__(kBudThreads, 3) budget_kernel(const BudgetParams p) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned FULL = 0xFFFFFFFFu;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wtot[kBudThreads / 32];
  __shared__ uint32_t s_excl;
  uint64_t spent_lo = 0, spent_hi = 0, full_lo = 0, full_hi = 0;
  uint32_t pruned = 0, infeasible = 0;
  uint64_t bidx = 0;
  bool found = false;
  uint32_t cta_min = kInf32;
  uint32_t thr_basis = kInf32, thr = kInf32;          // thr = budget_thr(thr_basis)
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const uint32_t slice = s_tile;
    if (slice >= p.ntiles) break;
    const uint64_t sbase = (uint64_t)slice * kBudSlice;
    const uint64_t send = min(p.n, sbase + kBudSlice);
    // ---- pass 1: slice minimum (16-byte streaming loads, 8 in flight per thread)
    uint32_t m = kInf32;
    if (send - sbase == (uint64_t)kBudSlice) {
      const uint4* q = reinterpret_cast<const uint4*>(p.W + sbase);
#pragma unroll
      for (int i0 = 0; i0 < kBudSlice / 4 / kBudThreads; i0 += 16) {
        uint4 x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = q[(i0 + i) * kBudThreads + tid];
#pragma unroll
        for (int i = 0; i < 16; ++i) m = min(m, min(min(x[i].x, x[i].y), min(x[i].z, x[i].w)));
      }
    } else {
      for (uint64_t i = sbase + tid; i < send; i += kBudThreads) m = min(m, p.W[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(FULL, m, o));
    if (lane == 0) s_wtot[warp] = m;
    __syncthreads();
    // ---- decoupled look-back over slices (warp 0)
    if (warp == 0) {
      uint32_t agg = lane < kBudThreads / 32 ? s_wtot[lane] : kInf32;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) agg = min(agg, __shfl_xor_sync(FULL, agg, o));
      uint32_t excl = kInf32;
      if (slice == 0) {
        if (lane == 0) atomicExch(p.status, (2ull << 32) | agg);
      } else {
        if (lane == 0) atomicExch(p.status + slice, (1ull << 32) | agg);
        int64_t pred = (int64_t)slice - 1;
        for (;;) {
          const int64_t at = pred - lane;
          unsigned long long st;
          for (;;) {
            st = at >= 0 ? *reinterpret_cast<volatile unsigned long long*>(p.status + at)
                         : ((2ull << 32) | kInf32);
            if (__all_sync(FULL, (st >> 32) != 0)) break;
          }
          const unsigned incl = __ballot_sync(FULL, (st >> 32) == 2);
          uint32_t val = (uint32_t)st;
          const int stop = incl ? __ffs(incl) - 1 : 31;   // lanes 0..stop contribute
          if (lane > stop) val = kInf32;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) val = min(val, __shfl_xor_sync(FULL, val, o));
          excl = min(excl, val);
          if (incl) break;
          pred -= 32;
        }
        if (lane == 0) atomicExch(p.status + slice, (2ull << 32) | min(excl, agg));
      }
      if (lane == 0) {
        s_excl = excl;
        cta_min = min(cta_min, agg);
      }
    }
    __syncthreads();
    uint32_t slice_run = s_excl;                       // every task before the current tile
    // ---- pass 2: per-task decisions, tile by tile (L2 re-read)
    uint32_t vn[16];
    budget_load(p, sbase, warp, lane, vn);
    for (uint64_t tbase = sbase; tbase < send; tbase += kBudTile) {
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = vn[k];
      if (tbase + kBudTile < send) budget_load(p, tbase + kBudTile, warp, lane, vn);   // prefetch
      const uint64_t base = tbase + (uint64_t)warp * 512 + (uint64_t)lane * 16;
      uint32_t lmin = v[0];
#pragma unroll
      for (int k = 1; k < 16; ++k) lmin = min(lmin, v[k]);
      uint32_t incl = lmin;                            // warp inclusive scan of the lanes' minima
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl = min(incl, y);
      }
      uint32_t ex = __shfl_up_sync(FULL, incl, 1);
      if (lane == 0) ex = kInf32;
      if (lane == 31) s_wtot[warp] = incl;
      __syncthreads();
      uint32_t before = slice_run, tile_min = kInf32;
#pragma unroll
      for (int w = 0; w < kBudThreads / 32; ++w) {
        if (w < warp) before = min(before, s_wtot[w]);
        tile_min = min(tile_min, s_wtot[w]);
      }
      slice_run = min(slice_run, tile_min);
      uint32_t run = min(before, ex);                  // best before this lane's 16 tasks
      if (run != thr_basis) { thr_basis = run; thr = budget_thr(run, p.num, p.den); }
      // With w' = (W finite ? W : 0) and thr >= the current best a task costs
      // min(w', thr) (pruned iff w' > thr); a new best w < best costs
      // w = min(w, thr) as well; an infeasible one min(0, thr) = 0.
      uint64_t t_spent = 0, t_full = 0;
      uint32_t t_inf = 0, t_pr = 0;
      if (lmin < run) {                                // a new best among the 16 (rare)
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
          const uint32_t w = v[k];
          if (w < run) {
            t_spent += w;
            t_full += w;
            run = w;
            thr_basis = run;
            thr = budget_thr(run, p.num, p.den);
            bidx = base + k;
            found = true;
            continue;
          }
          const uint32_t wf = w == kInf32 ? 0u : w;
          t_inf += w == kInf32 ? 1u : 0u;
          t_pr += wf > thr ? 1u : 0u;
          t_spent += min(wf, thr);
          t_full += wf;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t w = v[k];
          const uint32_t wf = min(w, w + 1u);          // INF + 1 wraps to 0: w' in one op
          t_inf += w == kInf32 ? 1u : 0u;
          t_pr += wf > thr ? 1u : 0u;
          t_spent += min(wf, thr);
          t_full += wf;
        }
      }
      if (tbase + kBudTile > p.n) {                    // ragged tile: padding is not infeasible
#pragma unroll 1
        for (int k = 0; k < 16; ++k) t_inf -= base + k >= p.n ? 1u : 0u;
      }
      infeasible += t_inf;
      pruned += t_pr;
      add128(spent_lo, spent_hi, t_spent);
      add128(full_lo, full_hi, t_full);
      __syncthreads();                                 // s_wtot reused by the next tile
    }
  }
  // ---- CTA reduction, then one set of global atomics per CTA
  __shared__ unsigned long long s_acc[8];
  if (tid < 8) s_acc[tid] = tid == 6 ? ~0ull : 0ull;
  __syncthreads();
  atomicAdd(&s_acc[0], (unsigned long long)pruned);
  atomicAdd(&s_acc[1], (unsigned long long)infeasible);
  {
    const unsigned long long o = atomicAdd(&s_acc[2], (unsigned long long)spent_lo);
    atomicAdd(&s_acc[3], (unsigned long long)(spent_hi + (o + spent_lo < o ? 1 : 0)));
    const unsigned long long f = atomicAdd(&s_acc[4], (unsigned long long)full_lo);
    atomicAdd(&s_acc[5], (unsigned long long)(full_hi + (f + full_lo < f ? 1 : 0)));
  }
  if (tid == 0) atomicMin(&s_acc[6], (unsigned long long)cta_min);
  if (found) atomicMax(&s_acc[7], (unsigned long long)bidx);
  __syncthreads();
  if (tid == 0) {
    atomicAdd(p.acc + 0, s_acc[0]);
    atomicAdd(p.acc + 1, s_acc[1]);
    unsigned long long o = atomicAdd(p.acc + 2, s_acc[2]);
    atomicAdd(p.acc + 3, s_acc[3] + (o + s_acc[2] < o ? 1 : 0));
    o = atomicAdd(p.acc + 4, s_acc[4]);
    atomicAdd(p.acc + 5, s_acc[5] + (o + s_acc[4] < o ? 1 : 0));
    atomicMin(p.acc + 6, s_acc[6]);
    atomicMax(p.acc + 7, s_acc[7]);
  }
}

cudaError_t launch_budget(const uint32_t* W, uint64_t n, uint32_t num, uint32_t den, void* scratch,
                          int sms, cudaStream_t st) {
  // scratch: [8] accumulators, [1] ticket (+ pad), then [ntiles] status words
  BudgetParams p{};
  p.W = W;
  p.n = n;
  p.ntiles = (uint32_t)((n + kBudSlice - 1) / kBudSlice);     // slices
  p.num = num;
  p.den = den;
  p.acc = static_cast<unsigned long long*>(scratch);
  p.ticket = reinterpret_cast<unsigned int*>(p.acc + 8);
  p.status = p.acc + 10;
  cudaError_t e = cudaMemsetAsync(scratch, 0, (10 + (size_t)p.ntiles) * 8, st);
  if (e != cudaSuccess) return e;
  // acc[6] (best) starts at +inf: written by the kernel's atomicMin identity
  e = cudaMemsetAsync(p.acc + 6, 0xFF, 8, st);
  if (e != cudaSuccess) return e;
  if (p.ntiles == 0) return cudaSuccess;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, budget_kernel, kBudThreads, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > (int64_t)p.ntiles) grid = p.ntiles;
  budget_kernel<<<(unsigned)grid, kBudThreads, 0, st>>>(p);
  return cudaGetLastError();
}

size_t budget_scratch_bytes(uint64_t n) {
  return (10 + (size_t)((n + kBudSlice - 1) / kBudSlice)) * 8;
}

}  // namespace cfp
