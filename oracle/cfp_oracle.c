/*
 * cfp_oracle.c -- TEST INFRASTRUCTURE ONLY (see cfp_oracle.h).
 *
 * Plain definitions, written for checkability rather than speed:
 *  - every combination's cost is recomputed from scratch from Eq. 3's terms
 *     -- no hoisting, no blocking, no reordering of the minimisation;
 *  - the only parallelism is splitting the index range into contiguous chunks
 *    (one per thread) and merging the per-chunk (A, I) in chunk order with a
 *    strict '<', which is the same as one sequential pass in index order.
 */
#include "cfp_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* w_j[s] = p_j[s] + c_j[s]; INF if either is INF (Q7).  Returns 0 if INF. */
static int unary(const orc_type* t, int32_t j, int32_t s, uint64_t* w) {
  int64_t off = 0;
  for (int32_t q = 0; q < j; ++q) off += t->radix[q];
  uint32_t p = t->comp[off + s];
  uint32_t c = t->comm ? t->comm[off + s] : 0u;
  if (p == ORC_INF32 || c == ORC_INF32) return 0;
  *w = (uint64_t)p + (uint64_t)c;
  return 1;
}

static const uint32_t* edge_table(const orc_type* t, int32_t e) {
  int64_t off = 0;
  for (int32_t q = 0; q < e; ++q) off += (int64_t)t->radix[t->esrc[q]] * t->radix[t->edst[q]];
  return t->etab + off;
}

static int32_t d_in_of(const orc_problem* p, int32_t tr) {
  const orc_trans* x = &p->trans[tr];
  if (x->pred < 0) return 1;
  const orc_type* pt = &p->types[x->pred];
  return pt->radix[pt->out_block];
}

static const uint32_t* cross_table(const orc_problem* p, int32_t tr, int32_t x) {
  const orc_trans* T = &p->trans[tr];
  const orc_type* t = &p->types[T->type];
  int64_t din = d_in_of(p, tr);
  int64_t off = 0;
  for (int32_t q = 0; q < x; ++q) off += din * t->radix[T->xdst[q]];
  return T->xtab + off;
}

uint64_t orc_cost(const orc_problem* p, int32_t tr, int32_t u, const int32_t* s) {
  const orc_trans* T = &p->trans[tr];
  const orc_type* t = &p->types[T->type];
  uint64_t total = 0, w;
  /* sum_j (p_j + c_j)  -- Eq. 3 first term, per ParallelBlock */
  for (int32_t j = 0; j < t->K; ++j) {
    if (!unary(t, j, s[j], &w)) return ORC_INF64;
    total += w;
  }
  /* intra-segment resharding between connected ParallelBlocks */
  for (int32_t e = 0; e < t->E; ++e) {
    const uint32_t* R = edge_table(t, e);
    uint32_t r = R[(int64_t)s[t->esrc[e]] * t->radix[t->edst[e]] + s[t->edst[e]]];
    if (r == ORC_INF32) return ORC_INF64;
    total += r;
  }
  /* cross-segment resharding r_n (Eq. 3 second term) */
  for (int32_t x = 0; x < T->X; ++x) {
    const uint32_t* Q = cross_table(p, tr, x);
    int32_t j = T->xdst[x];
    uint32_t r = Q[(int64_t)u * t->radix[j] + s[j]];
    if (r == ORC_INF32) return ORC_INF64;
    total += r;
  }
  return total;
}

void orc_decode(int32_t K, const int32_t* radix, uint64_t idx, int32_t* digits) {
  for (int32_t j = K - 1; j >= 0; --j) {
    digits[j] = (int32_t)(idx % (uint64_t)radix[j]);
    idx /= (uint64_t)radix[j];
  }
}

uint64_t orc_cost_index(const orc_problem* p, int32_t tr, int32_t u, uint64_t idx) {
  const orc_type* t = &p->types[p->trans[tr].type];
  int32_t s[64];
  orc_decode(t->K, t->radix, idx, s);
  return orc_cost(p, tr, u, s);
}

static uint64_t space_size(const orc_type* t) {
  uint64_t n = 1;
  for (int32_t j = 0; j < t->K; ++j) n *= (uint64_t)t->radix[j];
  return n;
}

static int nthreads_or_default(int n) {
#ifdef _OPENMP
  if (n <= 0) n = omp_get_max_threads();
#else
  n = 1;
#endif
  return n < 1 ? 1 : n;
}

int orc_segment_table_range(const orc_problem* p, int32_t tr, uint64_t lo_idx, uint64_t hi_idx,
                            uint64_t* A, uint64_t* I, int nthreads) {
  if (tr < 0 || tr >= p->ntrans) return ORC_EINVAL;
  const orc_type* t = &p->types[p->trans[tr].type];
  if (t->K > 64) return ORC_ETOOBIG;
  const int32_t din = d_in_of(p, tr);
  const int32_t dout = t->radix[t->out_block];
  const uint64_t S0 = space_size(t);
  if (hi_idx > S0) hi_idx = S0;
  if (lo_idx > hi_idx) lo_idx = hi_idx;
  const uint64_t S = hi_idx - lo_idx;
  const int nt = nthreads_or_default(nthreads);
  const size_t cells = (size_t)din * dout;
  uint64_t* LA = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  uint64_t* LI = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  if (!LA || !LI) { free(LA); free(LI); return ORC_ENOMEM; }
  for (size_t c = 0; c < cells * nt; ++c) { LA[c] = ORC_INF64; LI[c] = ORC_NOIDX; }
#pragma omp parallel for schedule(static, 1) num_threads(nt)
  for (int ch = 0; ch < nt; ++ch) {
    uint64_t lo = lo_idx + S * (uint64_t)ch / nt, hi = lo_idx + S * (uint64_t)(ch + 1) / nt;
    uint64_t* a = LA + cells * ch;
    uint64_t* ix = LI + cells * ch;
    int32_t s[64];
    for (int32_t u = 0; u < din; ++u) {
      for (uint64_t idx = lo; idx < hi; ++idx) {
        orc_decode(t->K, t->radix, idx, s);
        uint64_t c = orc_cost(p, tr, u, s);
        size_t cell = (size_t)u * dout + s[t->out_block];
        if (c < a[cell]) { a[cell] = c; ix[cell] = idx; }
      }
    }
  }
  for (size_t c = 0; c < cells; ++c) { A[c] = ORC_INF64; I[c] = ORC_NOIDX; }
  for (int ch = 0; ch < nt; ++ch)            /* chunk order == index order */
    for (size_t c = 0; c < cells; ++c)
      if (LA[cells * ch + c] < A[c]) { A[c] = LA[cells * ch + c]; I[c] = LI[cells * ch + c]; }
  free(LA); free(LI);
  return ORC_OK;
}

int orc_segment_table(const orc_problem* p, int32_t tr, uint64_t* A, uint64_t* I, int nthreads) {
  if (tr < 0 || tr >= p->ntrans) return ORC_EINVAL;
  return orc_segment_table_range(p, tr, 0, space_size(&p->types[p->trans[tr].type]), A, I, nthreads);
}

int orc_bucket(const orc_problem* p, int32_t tr, int32_t u, int32_t v,
               uint64_t* a_out, uint64_t* i_out, int nthreads) {
  if (tr < 0 || tr >= p->ntrans) return ORC_EINVAL;
  const orc_type* t = &p->types[p->trans[tr].type];
  if (t->K > 64) return ORC_ETOOBIG;
  const int32_t o = t->out_block;
  if (u < 0 || u >= d_in_of(p, tr) || v < 0 || v >= t->radix[o]) return ORC_EINVAL;
  /* the sub-space s_o = v, indexed by the remaining digits in the same order */
  int32_t rr[64];
  int32_t K2 = 0;
  for (int32_t j = 0; j < t->K; ++j) if (j != o) rr[K2++] = t->radix[j];
  uint64_t S2 = 1;
  for (int32_t j = 0; j < K2; ++j) S2 *= (uint64_t)rr[j];
  const int nt = nthreads_or_default(nthreads);
  uint64_t* LA = (uint64_t*)malloc(sizeof(uint64_t) * nt);
  uint64_t* LI = (uint64_t*)malloc(sizeof(uint64_t) * nt);
  if (!LA || !LI) { free(LA); free(LI); return ORC_ENOMEM; }
#pragma omp parallel for schedule(static, 1) num_threads(nt)
  for (int ch = 0; ch < nt; ++ch) {
    uint64_t lo = S2 * (uint64_t)ch / nt, hi = S2 * (uint64_t)(ch + 1) / nt;
    uint64_t best = ORC_INF64, bi = ORC_NOIDX;
    int32_t q[64], s[64];
    for (uint64_t k = lo; k < hi; ++k) {
      orc_decode(K2, rr, k, q);
      for (int32_t j = 0, m = 0; j < t->K; ++j) s[j] = (j == o) ? v : q[m++];
      uint64_t c = orc_cost(p, tr, u, s);
      if (c < best) {
        uint64_t idx = 0;
        for (int32_t j = 0; j < t->K; ++j) idx = idx * (uint64_t)t->radix[j] + (uint64_t)s[j];
        best = c; bi = idx;
      }
    }
    LA[ch] = best; LI[ch] = bi;
  }
  uint64_t A = ORC_INF64, I = ORC_NOIDX;
  for (int ch = 0; ch < nt; ++ch) if (LA[ch] < A) { A = LA[ch]; I = LI[ch]; }
  free(LA); free(LI);
  *a_out = A; *i_out = I;
  return ORC_OK;
}

static uint64_t add_inf(uint64_t a, uint64_t b) {
  return (a == ORC_INF64 || b == ORC_INF64) ? ORC_INF64 : a + b;
}

int orc_chain(int32_t N, const int32_t* rows, const int32_t* cols,
              const uint64_t* const* A, const uint64_t* terminal, uint64_t* G) {
  if (N < 1) return ORC_EINVAL;
  for (int32_t n = 1; n < N; ++n) if (rows[n] != cols[n - 1]) return ORC_EINVAL;
  /* offsets of G_0..G_N in the ragged output */
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (N + 2));
  if (!off) return ORC_ENOMEM;
  off[0] = 0;
  off[1] = rows[0];
  for (int32_t n = 1; n <= N; ++n) off[n + 1] = off[n] + cols[n - 1];
  uint64_t* GN = G + off[N];
  for (int32_t v = 0; v < cols[N - 1]; ++v) GN[v] = terminal ? terminal[v] : 0;
  for (int32_t n = N; n >= 1; --n) {           /* G_{n-1}(u) = min_v A_n[u][v] + G_n(v) */
    const uint64_t* M = A[n - 1];
    const uint64_t* Gn = G + off[n];
    uint64_t* Gp = G + off[n - 1];
    for (int32_t u = 0; u < rows[n - 1]; ++u) {
      uint64_t best = ORC_INF64;
      for (int32_t v = 0; v < cols[n - 1]; ++v) {
        uint64_t c = add_inf(M[(int64_t)u * cols[n - 1] + v], Gn[v]);
        if (c < best) best = c;
      }
      Gp[u] = best;
    }
  }
  free(off);
  return ORC_OK;
}

int orc_reconstruct(int32_t N, const int32_t* rows, const int32_t* cols,
                    const uint64_t* const* A, const uint64_t* const* I,
                    const uint64_t* G, int32_t* v_out, uint64_t* idx_out, uint64_t* cost_out) {
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (N + 2));
  if (!off) return ORC_ENOMEM;
  off[0] = 0;
  off[1] = rows[0];
  for (int32_t n = 1; n <= N; ++n) off[n + 1] = off[n] + cols[n - 1];
  if (G[0] == ORC_INF64) { free(off); return ORC_EINFEASIBLE; }
  int32_t u = 0;                               /* u_1 = 0 (chain start, Q8) */
  for (int32_t n = 1; n <= N; ++n) {
    const uint64_t* M = A[n - 1];
    const uint64_t* Ix = I[n - 1];
    const uint64_t target = G[off[n - 1] + u];
    const uint64_t* Gn = G + off[n];
    int32_t best = -1;
    for (int32_t v = 0; v < cols[n - 1]; ++v) {
      uint64_t a = M[(int64_t)u * cols[n - 1] + v];
      if (a == ORC_INF64 || Gn[v] == ORC_INF64) continue;
      if (a + Gn[v] != target) continue;
      if (best < 0 || Ix[(int64_t)u * cols[n - 1] + v] < Ix[(int64_t)u * cols[n - 1] + best]) best = v;
    }
    if (best < 0) { free(off); return ORC_EINFEASIBLE; }
    v_out[n - 1] = best;
    idx_out[n - 1] = Ix[(int64_t)u * cols[n - 1] + best];
    cost_out[n - 1] = M[(int64_t)u * cols[n - 1] + best];
    u = best;
  }
  free(off);
  return ORC_OK;
}

int orc_search_plan(const orc_problem* p, int nthreads, uint64_t* total,
                    uint64_t* seg_index, int32_t* digits, int32_t kmax, uint64_t* seg_ns) {
  const int32_t N = p->N;
  if (N < 1) return ORC_EINVAL;
  uint64_t** At = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  uint64_t** It = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  const uint64_t** An = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  const uint64_t** In = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* vsel = (int32_t*)malloc(sizeof(int32_t) * N);
  int rc = ORC_OK;
  uint64_t* G = NULL;
  if (!At || !It || !An || !In || !rows || !cols || !vsel) { rc = ORC_ENOMEM; goto done; }
  int64_t gsz = 1;
  for (int32_t n = 0; n < N; ++n) {
    int32_t tr = p->inst[n];
    if (tr < 0 || tr >= p->ntrans) { rc = ORC_EINVAL; goto done; }
    const orc_type* t = &p->types[p->trans[tr].type];
    rows[n] = d_in_of(p, tr);
    cols[n] = t->radix[t->out_block];
    gsz += cols[n];
    if (!At[tr]) {
      size_t cells = (size_t)rows[n] * cols[n];
      At[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      It[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      if (!At[tr] || !It[tr]) { rc = ORC_ENOMEM; goto done; }
      rc = orc_segment_table(p, tr, At[tr], It[tr], nthreads);
      if (rc) goto done;
    }
    An[n] = At[tr];
    In[n] = It[tr];
  }
  G = (uint64_t*)malloc(sizeof(uint64_t) * (gsz + rows[0]));
  if (!G) { rc = ORC_ENOMEM; goto done; }
  rc = orc_chain(N, rows, cols, An, NULL, G);
  if (rc) goto done;
  *total = G[0];
  rc = orc_reconstruct(N, rows, cols, An, In, G, vsel, seg_index, seg_ns);
  if (rc) goto done;
  for (int32_t n = 0; n < N; ++n) {
    const orc_type* t = &p->types[p->trans[p->inst[n]].type];
    for (int32_t j = 0; j < kmax; ++j) digits[(int64_t)n * kmax + j] = -1;
    orc_decode(t->K, t->radix, seg_index[n], digits + (int64_t)n * kmax);
  }
done:
  if (At) for (int32_t q = 0; q < p->ntrans; ++q) free(At[q]);
  if (It) for (int32_t q = 0; q < p->ntrans; ++q) free(It[q]);
  free(At); free(It); free(An); free(In); free(rows); free(cols); free(vsel); free(G);
  return rc;
}

int orc_minplus(int32_t m, int32_t k, int32_t n, const uint64_t* A, const uint64_t* B,
                uint64_t* C, uint64_t* argk) {
  if (m < 0 || k < 0 || n < 0) return ORC_EINVAL;
  for (int32_t i = 0; i < m; ++i)
    for (int32_t j = 0; j < n; ++j) {
      uint64_t best = ORC_INF64, bk = ORC_NOIDX;
      for (int32_t q = 0; q < k; ++q) {
        uint64_t c = add_inf(A[(int64_t)i * k + q], B[(int64_t)q * n + j]);
        if (c < best) { best = c; bk = (uint64_t)q; }
      }
      C[(int64_t)i * n + j] = best;
      if (argk) argk[(int64_t)i * n + j] = bk;
    }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Memory-constrained search (NEXT-1).  Same plain style: every combination's
 * cost and quantised memory recomputed from the definition.
 * ------------------------------------------------------------------------- */
static uint64_t ceil_div(uint64_t a, uint64_t b) { return a / b + (a % b != 0); }

static uint64_t block_mem(const orc_type* t, int32_t j, int32_t s) {
  if (!t->mem) return 0;
  int64_t off = 0;
  for (int32_t q = 0; q < j; ++q) off += t->radix[q];
  return (uint64_t)t->mem[off + s];
}

/* m_n(i_n): the segment plan's peak memory, Eq. 4 restricted to one segment
 * (the sum of its ParallelBlocks' profiled memories, reading R-M1). */
uint64_t orc_mem_exact(const orc_type* t, const int32_t* s) {
  uint64_t m = 0;
  for (int32_t j = 0; j < t->K; ++j) m += block_mem(t, j, s[j]);
  return m;
}

/* "we quantize the memory usage of each parallelism plan": the
 * plan's quanta q = ceil(m_n(i_n) / quantum) (ceiling; R-M1). */
uint64_t orc_mem_q(const orc_type* t, const int32_t* s, uint64_t quantum) {
  return ceil_div(orc_mem_exact(t, s), quantum);
}

/* [qlo, qhi] of a type: the ceilings of the smallest and largest plan memory
 * over ALL strategies (R-M3; ceil is monotone, so every plan lies inside). */
int orc_mem_range(const orc_type* t, uint64_t quantum, int64_t* qlo, int64_t* qhi) {
  if (quantum == 0) return ORC_EINVAL;
  uint64_t lo = 0, hi = 0;
  for (int32_t j = 0; j < t->K; ++j) {
    uint64_t mn = ORC_INF64, mx = 0;
    for (int32_t s = 0; s < t->radix[j]; ++s) {
      uint64_t m = block_mem(t, j, s);
      if (m < mn) mn = m;
      if (m > mx) mx = m;
    }
    lo += mn;
    hi += mx;
  }
  *qlo = (int64_t)ceil_div(lo, quantum);
  *qhi = (int64_t)ceil_div(hi, quantum);
  return ORC_OK;
}

int orc_segment_table_mem(const orc_problem* p, int32_t tr, uint64_t quantum,
                          uint64_t* Am, uint64_t* Im, int nthreads) {
  if (tr < 0 || tr >= p->ntrans) return ORC_EINVAL;
  return orc_segment_table_mem_range(p, tr, quantum, 0, space_size(&p->types[p->trans[tr].type]),
                                     Am, Im, nthreads);
}

/* The same over the combination-index range [lo_idx, hi_idx) only (the
 * bench's bounded cpu_baseline sample); arithmetic identical. */
int orc_segment_table_mem_range(const orc_problem* p, int32_t tr, uint64_t quantum, uint64_t lo_idx,
                                uint64_t hi_idx, uint64_t* Am, uint64_t* Im, int nthreads) {
  if (tr < 0 || tr >= p->ntrans || quantum == 0) return ORC_EINVAL;
  const orc_type* t = &p->types[p->trans[tr].type];
  if (t->K > 64) return ORC_ETOOBIG;
  int64_t qlo, qhi;
  orc_mem_range(t, quantum, &qlo, &qhi);
  const int64_t nq = qhi - qlo + 1;
  const int32_t din = d_in_of(p, tr);
  const int32_t dout = t->radix[t->out_block];
  const uint64_t S0 = space_size(t);
  if (hi_idx > S0) hi_idx = S0;
  if (lo_idx > hi_idx) lo_idx = hi_idx;
  const uint64_t S = hi_idx - lo_idx;
  const int nt = nthreads_or_default(nthreads);
  const size_t cells = (size_t)din * dout * nq;
  uint64_t* LA = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  uint64_t* LI = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  if (!LA || !LI) { free(LA); free(LI); return ORC_ENOMEM; }
  for (size_t c = 0; c < cells * nt; ++c) { LA[c] = ORC_INF64; LI[c] = ORC_NOIDX; }
#pragma omp parallel for schedule(static, 1) num_threads(nt)
  for (int ch = 0; ch < nt; ++ch) {
    uint64_t lo = lo_idx + S * (uint64_t)ch / nt, hi = lo_idx + S * (uint64_t)(ch + 1) / nt;
    uint64_t* a = LA + cells * ch;
    uint64_t* ix = LI + cells * ch;
    int32_t s[64];
    for (int32_t u = 0; u < din; ++u) {
      for (uint64_t idx = lo; idx < hi; ++idx) {
        orc_decode(t->K, t->radix, idx, s);
        uint64_t c = orc_cost(p, tr, u, s);
        int64_t q = (int64_t)orc_mem_q(t, s, quantum);
        size_t cell = ((size_t)u * dout + s[t->out_block]) * nq + (size_t)(q - qlo);
        if (c < a[cell]) { a[cell] = c; ix[cell] = idx; }
      }
    }
  }
  for (size_t c = 0; c < cells; ++c) { Am[c] = ORC_INF64; Im[c] = ORC_NOIDX; }
  for (int ch = 0; ch < nt; ++ch)            /* chunk order == index order */
    for (size_t c = 0; c < cells; ++c)
      if (LA[cells * ch + c] < Am[c]) { Am[c] = LA[cells * ch + c]; Im[c] = LI[cells * ch + c]; }
  free(LA); free(LI);
  return ORC_OK;
}

static int64_t* mem_offsets(int32_t N, const int32_t* rows, const int32_t* cols, int64_t Qmax) {
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (N + 2));
  if (!off) return NULL;
  off[0] = 0;
  off[1] = (int64_t)rows[0] * (Qmax + 1);
  for (int32_t n = 1; n <= N; ++n) off[n + 1] = off[n] + (int64_t)cols[n - 1] * (Qmax + 1);
  return off;
}

int orc_chain_mem(int32_t N, const int32_t* rows, const int32_t* cols, const int32_t* nq,
                  const int64_t* qlo, const uint64_t* const* Am, int64_t Qmax, uint64_t* G) {
  if (N < 1 || Qmax < 0) return ORC_EINVAL;
  for (int32_t n = 1; n < N; ++n) if (rows[n] != cols[n - 1]) return ORC_EINVAL;
  int64_t* off = mem_offsets(N, rows, cols, Qmax);
  if (!off) return ORC_ENOMEM;
  const int64_t C = Qmax + 1;
  uint64_t* GN = G + off[N];
  for (int64_t i = 0; i < (int64_t)cols[N - 1] * C; ++i) GN[i] = 0;   /* free final layout */
  for (int32_t n = N; n >= 1; --n) {
    /* G_{n-1}(u, c) = min_{v, q : c + q <= Qmax} Am_n[u][v][q] + G_n(v, c + q) */
    const uint64_t* M = Am[n - 1];
    const uint64_t* Gn = G + off[n];
    uint64_t* Gp = G + off[n - 1];
    const int32_t D = cols[n - 1], Q = nq[n - 1];
    for (int32_t u = 0; u < rows[n - 1]; ++u)
      for (int64_t c = 0; c < C; ++c) {
        uint64_t best = ORC_INF64;
        for (int32_t v = 0; v < D; ++v)
          for (int32_t k = 0; k < Q; ++k) {
            const int64_t q = qlo[n - 1] + k;
            if (c + q > Qmax) continue;
            uint64_t x = add_inf(M[((int64_t)u * D + v) * Q + k], Gn[(int64_t)v * C + c + q]);
            if (x < best) best = x;
          }
        Gp[(int64_t)u * C + c] = best;
      }
  }
  free(off);
  return ORC_OK;
}

int orc_reconstruct_mem(int32_t N, const int32_t* rows, const int32_t* cols, const int32_t* nq,
                        const int64_t* qlo, const uint64_t* const* Am, const uint64_t* const* Im,
                        int64_t Qmax, const uint64_t* G, int32_t* v_out, int64_t* q_out,
                        uint64_t* idx_out, uint64_t* cost_out) {
  int64_t* off = mem_offsets(N, rows, cols, Qmax);
  if (!off) return ORC_ENOMEM;
  const int64_t C = Qmax + 1;
  if (G[0] == ORC_INF64) { free(off); return ORC_EINFEASIBLE; }
  int32_t u = 0;                               /* (u_1, c) = (0, 0) */
  int64_t c = 0;
  for (int32_t n = 1; n <= N; ++n) {
    const uint64_t* M = Am[n - 1];
    const uint64_t* Ix = Im[n - 1];
    const int32_t D = cols[n - 1], Q = nq[n - 1];
    const uint64_t target = G[off[n - 1] + (int64_t)u * C + c];
    const uint64_t* Gn = G + off[n];
    int64_t best = -1;
    for (int32_t v = 0; v < D; ++v)
      for (int32_t k = 0; k < Q; ++k) {
        const int64_t q = qlo[n - 1] + k;
        if (c + q > Qmax) continue;
        const int64_t cell = ((int64_t)u * D + v) * Q + k;
        uint64_t a = M[cell], g = Gn[(int64_t)v * C + c + q];
        if (a == ORC_INF64 || g == ORC_INF64 || a + g != target) continue;
        if (best < 0 || Ix[cell] < Ix[best]) best = cell;
      }
    if (best < 0) { free(off); return ORC_EINFEASIBLE; }
    const int32_t v = (int32_t)((best / Q) % D);
    const int64_t q = qlo[n - 1] + best % Q;
    v_out[n - 1] = v;
    q_out[n - 1] = q;
    idx_out[n - 1] = Ix[best];
    cost_out[n - 1] = M[best];
    u = v;
    c += q;
  }
  free(off);
  return ORC_OK;
}

int orc_search_plan_mem(const orc_problem* p, uint64_t quantum, uint64_t mem_limit, int nthreads,
                        uint64_t* total, uint64_t* seg_index, int32_t* digits, int32_t kmax,
                        uint64_t* seg_ns, int64_t* seg_q, int64_t* total_q) {
  const int32_t N = p->N;
  if (N < 1 || quantum == 0) return ORC_EINVAL;
  const int64_t Qmax = (int64_t)(mem_limit / quantum);
  if (Qmax > (1 << 22)) return ORC_ETOOBIG;
  uint64_t** At = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  uint64_t** It = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  const uint64_t** An = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  const uint64_t** In = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* nq = (int32_t*)malloc(sizeof(int32_t) * N);
  int64_t* qlo = (int64_t*)malloc(sizeof(int64_t) * N);
  int32_t* vsel = (int32_t*)malloc(sizeof(int32_t) * N);
  int rc = ORC_OK;
  uint64_t* G = NULL;
  if (!At || !It || !An || !In || !rows || !cols || !nq || !qlo || !vsel) { rc = ORC_ENOMEM; goto done; }
  int64_t gsz = 0;
  for (int32_t n = 0; n < N; ++n) {
    int32_t tr = p->inst[n];
    if (tr < 0 || tr >= p->ntrans) { rc = ORC_EINVAL; goto done; }
    const orc_type* t = &p->types[p->trans[tr].type];
    int64_t lo, hi;
    orc_mem_range(t, quantum, &lo, &hi);
    rows[n] = d_in_of(p, tr);
    cols[n] = t->radix[t->out_block];
    nq[n] = (int32_t)(hi - lo + 1);
    qlo[n] = lo;
    gsz += cols[n];
    if (!At[tr]) {
      size_t cells = (size_t)rows[n] * cols[n] * nq[n];
      At[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      It[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      if (!At[tr] || !It[tr]) { rc = ORC_ENOMEM; goto done; }
      rc = orc_segment_table_mem(p, tr, quantum, At[tr], It[tr], nthreads);
      if (rc) goto done;
    }
    An[n] = At[tr];
    In[n] = It[tr];
  }
  G = (uint64_t*)malloc(sizeof(uint64_t) * (gsz + rows[0]) * (Qmax + 1));
  if (!G) { rc = ORC_ENOMEM; goto done; }
  rc = orc_chain_mem(N, rows, cols, nq, qlo, An, Qmax, G);
  if (rc) goto done;
  *total = G[0];
  rc = orc_reconstruct_mem(N, rows, cols, nq, qlo, An, In, Qmax, G, vsel, seg_q, seg_index, seg_ns);
  if (rc) goto done;
  *total_q = 0;
  for (int32_t n = 0; n < N; ++n) {
    const orc_type* t = &p->types[p->trans[p->inst[n]].type];
    for (int32_t j = 0; j < kmax; ++j) digits[(int64_t)n * kmax + j] = -1;
    orc_decode(t->K, t->radix, seg_index[n], digits + (int64_t)n * kmax);
    *total_q += seg_q[n];
  }
done:
  if (At) for (int32_t q = 0; q < p->ntrans; ++q) free(At[q]);
  if (It) for (int32_t q = 0; q < p->ntrans; ++q) free(It[q]);
  free(At); free(It); free(An); free(In); free(rows); free(cols); free(nq); free(qlo); free(vsel); free(G);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Dense per-plan tables.  The
 * paper profiles whole-segment plans: W_t[idx] is the profiled time of plan
 * idx of segment type t (its p_n(i_n) + c_n(i_n), intra-segment resharding
 * included), INF = 0xFFFFFFFF.  The cross-segment term stays Q2's:
 *   C(u, s) = W_t[idx(s)] + sum_{cross (j, Q)} Q_j[u][s_j]
 * everything else (buckets, least index, chain, plan) as the factored model.
 * ------------------------------------------------------------------------- */
static uint64_t dense_cost(const orc_problem* p, int32_t tr, const uint32_t* W, int32_t u, uint64_t idx,
                           const int32_t* s) {
  const orc_trans* T = &p->trans[tr];
  const orc_type* t = &p->types[T->type];
  if (W[idx] == ORC_INF32) return ORC_INF64;
  uint64_t total = W[idx];
  for (int32_t x = 0; x < T->X; ++x) {
    const uint32_t* Q = cross_table(p, tr, x);
    int32_t j = T->xdst[x];
    uint32_t r = Q[(int64_t)u * t->radix[j] + s[j]];
    if (r == ORC_INF32) return ORC_INF64;
    total += r;
  }
  return total;
}

int orc_dense_segment_table(const orc_problem* p, int32_t tr, const uint32_t* W, uint64_t* A, uint64_t* I,
                            int nthreads) {
  if (tr < 0 || tr >= p->ntrans || !W) return ORC_EINVAL;
  const orc_type* t = &p->types[p->trans[tr].type];
  if (t->K > 64) return ORC_ETOOBIG;
  const int32_t din = d_in_of(p, tr);
  const int32_t dout = t->radix[t->out_block];
  const uint64_t S = space_size(t);
  const int nt = nthreads_or_default(nthreads);
  const size_t cells = (size_t)din * dout;
  uint64_t* LA = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  uint64_t* LI = (uint64_t*)malloc(sizeof(uint64_t) * cells * nt);
  if (!LA || !LI) { free(LA); free(LI); return ORC_ENOMEM; }
  for (size_t c = 0; c < cells * nt; ++c) { LA[c] = ORC_INF64; LI[c] = ORC_NOIDX; }
#pragma omp parallel for schedule(static, 1) num_threads(nt)
  for (int ch = 0; ch < nt; ++ch) {
    uint64_t lo = S * (uint64_t)ch / nt, hi = S * (uint64_t)(ch + 1) / nt;
    uint64_t* a = LA + cells * ch;
    uint64_t* ix = LI + cells * ch;
    int32_t s[64];
    for (int32_t u = 0; u < din; ++u)
      for (uint64_t idx = lo; idx < hi; ++idx) {
        orc_decode(t->K, t->radix, idx, s);
        uint64_t c = dense_cost(p, tr, W, u, idx, s);
        size_t cell = (size_t)u * dout + s[t->out_block];
        if (c < a[cell]) { a[cell] = c; ix[cell] = idx; }
      }
  }
  for (size_t c = 0; c < cells; ++c) { A[c] = ORC_INF64; I[c] = ORC_NOIDX; }
  for (int ch = 0; ch < nt; ++ch)            /* chunk order == index order */
    for (size_t c = 0; c < cells; ++c)
      if (LA[cells * ch + c] < A[c]) { A[c] = LA[cells * ch + c]; I[c] = LI[cells * ch + c]; }
  free(LA); free(LI);
  return ORC_OK;
}

int orc_dense_search_plan(const orc_problem* p, const uint32_t* const* W, int nthreads, uint64_t* total,
                          uint64_t* seg_index, int32_t* digits, int32_t kmax, uint64_t* seg_ns) {
  const int32_t N = p->N;
  if (N < 1 || !W) return ORC_EINVAL;
  uint64_t** At = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  uint64_t** It = (uint64_t**)calloc(p->ntrans, sizeof(uint64_t*));
  const uint64_t** An = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  const uint64_t** In = (const uint64_t**)malloc(sizeof(uint64_t*) * N);
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* vsel = (int32_t*)malloc(sizeof(int32_t) * N);
  int rc = ORC_OK;
  uint64_t* G = NULL;
  if (!At || !It || !An || !In || !rows || !cols || !vsel) { rc = ORC_ENOMEM; goto done; }
  int64_t gsz = 0;
  for (int32_t n = 0; n < N; ++n) {
    int32_t tr = p->inst[n];
    if (tr < 0 || tr >= p->ntrans) { rc = ORC_EINVAL; goto done; }
    const orc_type* t = &p->types[p->trans[tr].type];
    rows[n] = d_in_of(p, tr);
    cols[n] = t->radix[t->out_block];
    gsz += cols[n];
    if (!At[tr]) {
      size_t cells = (size_t)rows[n] * cols[n];
      At[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      It[tr] = (uint64_t*)malloc(sizeof(uint64_t) * cells);
      if (!At[tr] || !It[tr]) { rc = ORC_ENOMEM; goto done; }
      rc = orc_dense_segment_table(p, tr, W[p->trans[tr].type], At[tr], It[tr], nthreads);
      if (rc) goto done;
    }
    An[n] = At[tr];
    In[n] = It[tr];
  }
  G = (uint64_t*)malloc(sizeof(uint64_t) * (gsz + rows[0]));
  if (!G) { rc = ORC_ENOMEM; goto done; }
  rc = orc_chain(N, rows, cols, An, NULL, G);
  if (rc) goto done;
  *total = G[0];
  rc = orc_reconstruct(N, rows, cols, An, In, G, vsel, seg_index, seg_ns);
  if (rc) goto done;
  for (int32_t n = 0; n < N; ++n) {
    const orc_type* t = &p->types[p->trans[p->inst[n]].type];
    for (int32_t j = 0; j < kmax; ++j) digits[(int64_t)n * kmax + j] = -1;
    orc_decode(t->K, t->radix, seg_index[n], digits + (int64_t)n * kmax);
  }
done:
  if (At) for (int32_t q = 0; q < p->ntrans; ++q) free(At[q]);
  if (It) for (int32_t q = 0; q < p->ntrans; ++q) free(It[q]);
  free(At); free(It); free(An); free(In); free(rows); free(cols); free(vsel); free(G);
  return rc;
}

