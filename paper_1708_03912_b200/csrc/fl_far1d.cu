// 1D far field.  In 1D a disjoint pair carries only k x k cross evaluations and 6 k tail
// evaluations (k = 2 for ~90% of the pairs of the graded BASELINE mesh), so per-pair cost —
// not arithmetic — dominates.  The 1D kernels therefore use lean, barrier-free layouts:
//
//  * tail1d:  one warp per target cell, one LANE per source cell, six per-lane accumulators
//             (the six cell-rule nodes), a single warp reduction at the end.  Source data is
//             read from structure-of-arrays (coalesced, no 128-B record loads).
//  * cross1d (fused, default): a CTA owns a 32 x 32 tile of DoFs (upper triangle, mirrored),
//             computes the 2x2 blocks M^{K,L} (cross_matrices, assembly.py:172-229, orders in
//             the reference's (min, max) orientation) of the <= 40 x 40 cell pairs behind it
//             into shared memory, bucketed by order so each warp runs one fixed-k unrolled
//             block, and forms A[i][j] = -C sum_{K∋i, L∋j} M[a][b] (assembly.py:723-725) with
//             the sum in one canonical order for (i, j) and (j, i): exactly symmetric.
//  * cross1d (pairs, fallback when a tile has > 40 cells, or FRACLAP_CROSS1D=pairs): every
//             unordered pair's block once into a packed triangular buffer, then a tiled gather
//             with the same canonical order; bitwise identical results.
// Row-block (multi-GPU) mode computes the ordered pairs (K in the owned rows' cells, all L)
// into a rectangular buffer instead.
#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

#include <climits>
#include <memory>
#include <cstdlib>
#include <string>

#ifndef FL_TAIL1D_MINB
#define FL_TAIL1D_MINB 4     // resident 128-thread CTAs per SM the tail is compiled for
#endif
#ifndef FL_TAIL1D_NT
#define FL_TAIL1D_NT 1       // target cells per warp in the 1D tail (2 measured slower: registers)
#endif
#ifndef FL_TILE1D_MINB
#define FL_TILE1D_MINB 3     // resident 256-thread CTAs per SM of the fused cross tiles
#endif

namespace fl {

// one 32-byte record per cell for the tail's source stream (two 16-byte loads per source);
// lo/hi/h are recomputed exactly: min/max of the end points and |x1 - x0| (fl_prep.cu diam)
struct __align__(16) Rec1D {
  double x0, x1;
  int v0, v1;
  float lnhf, lhf;
};

struct Src1D {
  const Rec1D* rec;
  const double *x0, *x1, *lo, *hi, *h, *lh;
  const int *v0, *v1;
  const float *lnhf, *lhf;      // __logf((float)h), (float)|ln h| for the fp32 order estimate
  const double* cstat;          // per 32-cell chunk: CSTAT doubles (chunk_order)
};

// Per chunk of 32 consecutive cells: x extent (lo, hi), max h, min / max |ln h|, ln(max h), min h,
// ln(min h).
constexpr int CSTAT = 8;

__global__ void build_src1d_kernel(DevMesh m, Rec1D* rec, double* x0, double* x1, double* lo, double* hi, double* h,
                                   double* lh, int* v0, int* v1, float* lnhf, float* lhf, double* cstat) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;   // blockDim a multiple of 32: warp = chunk
  {
    double clo = 1e300, chi = -1e300, hmx = 0.0, hmn = 1e300, lmn = 1e300, lmx = 0.0;
    if (c < m.nc) {
      const CellGeo& g = m.geo[c];
      clo = fmin(g.p[0][0], g.p[1][0]);
      chi = fmax(g.p[0][0], g.p[1][0]);
      hmx = hmn = g.diam;
      lmn = lmx = g.ldiam;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      clo = fmin(clo, __shfl_xor_sync(0xffffffffu, clo, o));
      chi = fmax(chi, __shfl_xor_sync(0xffffffffu, chi, o));
      hmx = fmax(hmx, __shfl_xor_sync(0xffffffffu, hmx, o));
      hmn = fmin(hmn, __shfl_xor_sync(0xffffffffu, hmn, o));
      lmn = fmin(lmn, __shfl_xor_sync(0xffffffffu, lmn, o));
      lmx = fmax(lmx, __shfl_xor_sync(0xffffffffu, lmx, o));
    }
    if ((c & 31) == 0 && c < m.nc) {
      double* cs = cstat + (size_t)CSTAT * (c >> 5);
      cs[0] = clo; cs[1] = chi; cs[2] = hmx; cs[3] = lmn; cs[4] = lmx; cs[5] = log(hmx); cs[6] = hmn;
      cs[7] = log(hmn);
    }
  }
  if (c >= m.nc) return;
  const CellGeo& g = m.geo[c];
  x0[c] = g.p[0][0];
  x1[c] = g.p[1][0];
  lo[c] = fmin(g.p[0][0], g.p[1][0]);
  hi[c] = fmax(g.p[0][0], g.p[1][0]);
  h[c] = g.diam;
  lh[c] = g.ldiam;
  v0[c] = g.v[0];
  v1[c] = g.v[1];
  lnhf[c] = __logf((float)g.diam);
  lhf[c] = (float)g.ldiam;
  Rec1D r;
  r.x0 = g.p[0][0];
  r.x1 = g.p[1][0];
  r.v0 = g.v[0];
  r.v1 = g.v[1];
  r.lnhf = lnhf[c];
  r.lhf = lhf[c];
  rec[c] = r;
}

// the exact fp64 order (rare: the fp32 estimate is within ORDER_DELTA of an integer), kept out
// of line so its registers do not count against the hot loops
static __device__ __noinline__ int order_exact1d(const OrderConsts& oc, double coff, double hA, double lA, double hB,
                                                 double lB, double dist) {
  return order_disjoint_s(oc, coff, hA, lA, hB, lB, dist);
}

// ------------------------------------------------------------------ tail
// The tail order shared by every source of a 32-cell chunk (target cell alo, ahi, |ln h| = alh,
// ln h = lah), or 0.  Upper bound: the gap D between the target and the chunk's x extent bounds
// every pair distance from below, so the disjoint order formula with the tail's C_offset - 4
// (quadrature.py:159-168, assembly.py:997) is bounded above term by term (numerator up,
// denominator down).  Lower bound of its first branch: numerator down (|ln h_B| at its chunk
// maximum in the (s-1) term, ln(dist / h_B) with the farthest gap and the smallest h_B),
// denominator up (the farthest gap).  When ceil() of both bounds (1e-9 margins) agree — and so
// every order between them — the chunk's order is that value.  D > 0 also excludes K and every
// cell sharing a vertex with it (N(K), assembly.py:999-1009).
__device__ __forceinline__ int chunk_order(const OrderConsts& oc, double alo, double ahi, double alh, double lah,
                                           const double* __restrict__ cs) {
  const double D = fmax(cs[0] - ahi, alo - cs[1]);
  if (!(D > 0.0)) return 0;
  const double lmn = fmin(alh, cs[3]), lmx = fmax(alh, cs[4]), lhmx = fmax(lah, cs[5]);
  const double lD = log(D);
  const double num_u = oc.lead_lnn + oc.sm1 * lmn + lmx - oc.s * lD + oc.s * lhmx - oc.coff_tail;
  const double den_l = fmax(lD - lhmx, 0.0) + oc.ln_rho2;
  const double up = num_u > 0.0 ? num_u / den_l : 0.0;
  if (up <= 2.0 - 1e-9) return 2;
  const double Dmax = cs[0] > ahi ? cs[1] - ahi : alo - cs[0];         // farthest gap to the chunk
  const double lDx = log(Dmax);
  const double num_l = oc.lead_lnn + oc.sm1 * cs[4] + fmax(alh, cs[3]) - oc.s * lDx + oc.s * cs[7] - oc.coff_tail;
  if (!(num_l > 0.0)) return 0;
  const double lo = num_l / (fmax(lDx - lah, 0.0) + oc.ln_rho2);
  const double kl = fmin(fmax(ceil(lo - 1e-9), 2.0), (double)oc.cap_disjoint);
  const double ku = fmin(fmax(ceil(up + 1e-9), 2.0), (double)oc.cap_disjoint);
  return kl == ku ? (int)kl : 0;
}

// one source of uniform order k on a known side of the target: k nodes x 6 target nodes
template <int E4, bool RIGHT>
__device__ __forceinline__ void tail1d_source_side(const double* __restrict__ nd, int k, double ex,
                                                   const double (&xq)[6], double (&acc)[6], double x0, double e,
                                                   double J) {
  for (int r = 0; r < k; ++r) {
    const double y = x0 + __ldg(nd + r * NODE) * e;
    const double jw = J * __ldg(nd + r * NODE + 2);
#pragma unroll
    for (int q = 0; q < 6; ++q) acc[q] = fma(jw, kpow_pos<E4>(RIGHT ? y - xq[q] : xq[q] - y, ex), acc[q]);
  }
}

template <int E4>
__device__ __forceinline__ void tail1d_source(const double* __restrict__ tab, const DevTables& dir, double ex,
                                              const double (&xq)[6], double (&acc)[6], double x0, double e, double J,
                                              int k) {
  const RuleRef rr = dir.rule(T_DISJ, k);
  for (int r = 0; r < k; ++r) {
    const double* nd = tab + (size_t)(rr.off + r) * NODE;
    const double y = x0 + nd[0] * e;
    const double jw = J * nd[2];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double d = xq[q] - y;
      acc[q] = fma(jw, kpow_abs<E4>(d, ex), acc[q]);
    }
  }
}

// Warp per NT target cells (NT = 2 by default), lane per source cell.  The source record, its two
// order-2 nodes and weights are shared by the NT targets; sources of order 2 for a target (~80%)
// are evaluated inline with the rule in registers, the others are compacted (ballot,
// deterministic order) into that target's per-warp queue and evaluated 32 at a time.  Per target
// the accumulation order is the same as with one target per warp.
template <int E4, int NT>
__global__ void __launch_bounds__(128, FL_TAIL1D_MINB) tail1d_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                     OrderConsts oc, double ex, Src1D S,
                                                     const int* __restrict__ targets,
                                                     const int* __restrict__ d_ntargets,
                                                     double* __restrict__ psi,
                                                     unsigned long long* __restrict__ evals) {
  constexpr int Q = 6;
  __shared__ int qs[4][NT][64], qk[4][NT][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wi = blockIdx.x * (blockDim.x >> 5) + w;
  const int ntargets = *d_ntargets;             // device count: launched before the host knows it
  if (wi * NT >= ntargets) return;
  int K[NT], av0[NT], av1[NT];
  bool valid[NT];
  double alo[NT], ahi[NT], ah[NT], alh[NT], alg[NT];
  float alnf[NT], alhf[NT];
  double xq[NT][Q], acc[NT][Q];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int ti = wi * NT + t;
    valid[t] = ti < ntargets;
    K[t] = targets[valid[t] ? ti : wi * NT];
    alo[t] = S.lo[K[t]]; ahi[t] = S.hi[K[t]]; ah[t] = S.h[K[t]]; alh[t] = S.lh[K[t]];
    alg[t] = log(ah[t]);
    alnf[t] = S.lnhf[K[t]]; alhf[t] = S.lhf[K[t]];
    av0[t] = S.v0[K[t]]; av1[t] = S.v1[K[t]];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      xq[t][q] = m.X[(size_t)K[t] * Q + q];
      acc[t][q] = 0.0;
    }
  }
  const double* n2 = tab + (size_t)dir.rule(T_DISJ, 2).off * NODE;
  const double t0 = n2[0], w0 = n2[2], t1 = n2[NODE], w1 = n2[NODE + 2];
  unsigned nodes[NT], rmask[NT];
  int ck[NT];                                   // per lane: the order of chunk (ci & ~31) + lane
  int qn[NT];                                   // warp-uniform queue lengths
  const int nchunks = (m.nc + 31) >> 5;
#pragma unroll
  for (int t = 0; t < NT; ++t) { nodes[t] = 0; qn[t] = 0; ck[t] = 0; rmask[t] = 0; }
  const unsigned lt = (1u << lane) - 1u;
  const int4* R = reinterpret_cast<const int4*>(S.rec);
  int4 na = make_int4(0, 0, 0, 0), nb = na;     // prefetched record of the next source
  if (lane < m.nc) { na = __ldg(R + 2 * lane); nb = __ldg(R + 2 * lane + 1); }
  for (int s0 = 0; s0 < m.nc; s0 += 32) {
    const int s = s0 + lane;
    const int4 ra = na, rb = nb;
    if (s + 32 < m.nc) { na = __ldg(R + 2 * (s + 32)); nb = __ldg(R + 2 * (s + 32) + 1); }
    const double sx0 = __hiloint2double(ra.y, ra.x), sx1 = __hiloint2double(ra.w, ra.z);
    const int bv0 = rb.x, bv1 = rb.y;
    const double blo = fmin(sx0, sx1), bhi = fmax(sx0, sx1);
    const double e = sx1 - sx0, J = fabs(e);
    const double y0 = sx0 + t0 * e, y1 = sx0 + t1 * e;
    const double j0 = J * w0, j1 = J * w1;
    const int ci = s0 >> 5;
    if ((ci & 31) == 0) {                       // order-2 flags of the next 32 chunks, one per lane
      const int cj = ci + lane;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        ck[t] = cj < nchunks ? chunk_order(oc, alo[t], ahi[t], alh[t], alg[t], S.cstat + (size_t)CSTAT * cj) : 0;
        rmask[t] = __ballot_sync(0xffffffffu, cj < nchunks && S.cstat[(size_t)CSTAT * cj] > ahi[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int kc = __shfl_sync(0xffffffffu, ck[t], ci & 31);   // warp-uniform chunk order (0: mixed)
      if (kc > 2) {                             // the whole chunk has order kc: no per-source orders
        if (s < m.nc) {
          const double* nd = tab + (size_t)dir.rule(T_DISJ, kc).off * NODE;
          if ((rmask[t] >> (ci & 31)) & 1u) tail1d_source_side<E4, true>(nd, kc, ex, xq[t], acc[t], sx0, e, J);
          else tail1d_source_side<E4, false>(nd, kc, ex, xq[t], acc[t], sx0, e, J);
          nodes[t] += kc;
        }
        continue;
      }
      if (kc == 2) {                            // warp-uniform: the whole chunk is k = 2
        // the chunk lies on one side of the target (gap > 0): the distance is y - x or x - y,
        // positive, so the kernel power needs no |.| (bitwise the same values)
        if (s < m.nc) {
          if ((rmask[t] >> (ci & 31)) & 1u) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              acc[t][q] = fma(j0, kpow_pos<E4>(y0 - xq[t][q], ex), acc[t][q]);
              acc[t][q] = fma(j1, kpow_pos<E4>(y1 - xq[t][q], ex), acc[t][q]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              acc[t][q] = fma(j0, kpow_pos<E4>(xq[t][q] - y0, ex), acc[t][q]);
              acc[t][q] = fma(j1, kpow_pos<E4>(xq[t][q] - y1, ex), acc[t][q]);
            }
          }
          nodes[t] += 2;
        }
        continue;
      }
      int k = -1;                               // -1: not a tail source of target t
      if (s < m.nc && !(s == K[t] || bv0 == av0[t] || bv0 == av1[t] || bv1 == av0[t] || bv1 == av1[t])) {  // N(K) (:999-1009)
        const double dist = fmax(fmax(__dsub_rn(blo, ahi[t]), __dsub_rn(alo[t], bhi)), 0.0);   // (:750-752)
        k = 0;
        if (dist > 1e-30)
          k = order_from_estimate(order_estimate_f(oc, oc.coff_tail_f, alnf[t], alhf[t], __int_as_float(rb.z),
                                                   __int_as_float(rb.w), __logf((float)dist)), oc.cap_disjoint);
      }
      if (k == 2) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double d0 = xq[t][q] - y0;
          acc[t][q] = fma(j0, kpow_abs<E4>(d0, ex), acc[t][q]);
          const double d1 = xq[t][q] - y1;
          acc[t][q] = fma(j1, kpow_abs<E4>(d1, ex), acc[t][q]);
        }
        nodes[t] += 2;
      }
      const bool dq = k == 0 || k > 2;
      const unsigned bm = __ballot_sync(0xffffffffu, dq);
      if (dq) {
        const int pos = qn[t] + __popc(bm & lt);
        qs[w][t][pos] = s;
        qk[w][t][pos] = k;
      }
      qn[t] += __popc(bm);
      if (qn[t] >= 32) {
        __syncwarp();
        const int ss = qs[w][t][lane];
        int kk = qk[w][t][lane];
        const double qx0 = S.x0[ss], qJ = S.h[ss];
        if (!kk) {
          const double dist = fmax(fmax(__dsub_rn(S.lo[ss], ahi[t]), __dsub_rn(alo[t], S.hi[ss])), 0.0);
          kk = order_exact1d(oc, oc.coff_tail, ah[t], alh[t], qJ, S.lh[ss], dist);
        }
        tail1d_source<E4>(tab, dir, ex, xq[t], acc[t], qx0, S.x1[ss] - qx0, qJ, kk);
        nodes[t] += kk;
        __syncwarp();
        if (lane < qn[t] - 32) {
          qs[w][t][lane] = qs[w][t][32 + lane];
          qk[w][t][lane] = qk[w][t][32 + lane];
        }
        __syncwarp();
        qn[t] -= 32;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (lane < qn[t]) {
      const int ss = qs[w][t][lane];
      int kk = qk[w][t][lane];
      const double qx0 = S.x0[ss], qJ = S.h[ss];
      if (!kk) {
        const double dist = fmax(fmax(__dsub_rn(S.lo[ss], ahi[t]), __dsub_rn(alo[t], S.hi[ss])), 0.0);
        kk = order_exact1d(oc, oc.coff_tail, ah[t], alh[t], qJ, S.lh[ss], dist);
      }
      tail1d_source<E4>(tab, dir, ex, xq[t], acc[t], qx0, S.x1[ss] - qx0, qJ, kk);
      nodes[t] += kk;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double v = warp_sum(acc[t][q]);
      if (lane == 0 && valid[t]) psi[(size_t)K[t] * Q + q] = v;
    }
    if (evals && valid[t]) {
      unsigned long long nd = nodes[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(0xffffffffu, nd, o);
      if (lane == 0) atomicAdd(evals, nd * Q);
    }
  }
}

// ------------------------------------------------------------------ cross: pair blocks
__device__ __forceinline__ int64_t tri_index(int K, int L, int nc) {
  return (int64_t)K * nc - (int64_t)K * (K + 1) / 2 + (L - K - 1);
}

template <int E4>
__device__ __forceinline__ double4 block1d(const double* __restrict__ tab, RuleRef rr, double kx0, double ke,
                                           double lx0, double le, double JJ, double ex) {
  double m00 = 0, m01 = 0, m10 = 0, m11 = 0;
  for (int x = 0; x < rr.cnt; ++x) {
    const double* nx = tab + (size_t)(rr.off + x) * NODE;
    const double X = kx0 + nx[0] * ke;
    double t0 = 0.0, t1 = 0.0;
    for (int y = 0; y < rr.cnt; ++y) {
      const double* ny = tab + (size_t)(rr.off + y) * NODE;
      const double d = X - (lx0 + ny[0] * le);
      const double v = kpow_abs<E4>(d, ex);
      t0 = fma(v, ny[3], t0);
      t1 = fma(v, ny[4], t1);
    }
    m00 = fma(nx[3], t0, m00);
    m01 = fma(nx[3], t1, m01);
    m10 = fma(nx[4], t0, m10);
    m11 = fma(nx[4], t1, m11);
  }
  return make_double4(m00 * JJ, m01 * JJ, m10 * JJ, m11 * JJ);
}

// symmetric mode: block K computes M^{K,L} for all L > K into the packed buffer
template <int E4>
__global__ void __launch_bounds__(256) cross1d_pairs_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                            OrderConsts oc, double ex, Src1D S,
                                                            double4* __restrict__ G,
                                                            unsigned long long* __restrict__ evals) {
  const int K = blockIdx.x;
  const double alo = S.lo[K], ahi = S.hi[K], ah = S.h[K], alh = S.lh[K], kx0 = S.x0[K];
  const double ke = S.x1[K] - kx0;
  const int av0 = S.v0[K], av1 = S.v1[K];
  unsigned long long my = 0;
  for (int L = K + 1 + threadIdx.x; L < m.nc; L += blockDim.x) {
    const int bv0 = S.v0[L], bv1 = S.v1[L];
    double4 out = make_double4(0, 0, 0, 0);
    if (!(bv0 == av0 || bv0 == av1 || bv1 == av0 || bv1 == av1)) {
      const double dist = fmax(fmax(__dsub_rn(S.lo[L], ahi), __dsub_rn(alo, S.hi[L])), 0.0);
      const int k = order_disjoint_fast_s(oc, oc.coff, ah, alh, S.h[L], S.lh[L], dist);
      const double lx0 = S.x0[L];
      out = block1d<E4>(tab, dir.rule(T_DISJ, k), kx0, ke, lx0, S.x1[L] - lx0, ah * S.h[L], ex);
      my += (unsigned long long)(k * k);
    }
    G[tri_index(K, L, m.nc)] = out;
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(evals, my);
  }
}

// row-block mode: block t computes M^{K,L} (K = targets[t]) for every L
template <int E4>
__global__ void __launch_bounds__(256) cross1d_rect_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                           OrderConsts oc, double ex, Src1D S,
                                                           const int* __restrict__ targets, double4* __restrict__ G,
                                                           unsigned long long* __restrict__ evals) {
  const int K = targets[blockIdx.x];
  const int av0 = S.v0[K], av1 = S.v1[K];
  unsigned long long my = 0;
  for (int L = threadIdx.x; L < m.nc; L += blockDim.x) {
    const int bv0 = S.v0[L], bv1 = S.v1[L];
    double4 out = make_double4(0, 0, 0, 0);
    if (L != K && !(bv0 == av0 || bv0 == av1 || bv1 == av0 || bv1 == av1)) {
      // order and block in the reference's (min, max) orientation, stored with K first
      const int P = min(K, L), Qc = max(K, L);
      const double dist = fmax(fmax(__dsub_rn(S.lo[Qc], S.hi[P]), __dsub_rn(S.lo[P], S.hi[Qc])), 0.0);
      const int k = order_disjoint_fast_s(oc, oc.coff, S.h[P], S.lh[P], S.h[Qc], S.lh[Qc], dist);
      const double px0 = S.x0[P], qx0 = S.x0[Qc];
      const double4 g = block1d<E4>(tab, dir.rule(T_DISJ, k), px0, S.x1[P] - px0, qx0, S.x1[Qc] - qx0,
                                    S.h[P] * S.h[Qc], ex);
      out = K < L ? g : make_double4(g.x, g.z, g.y, g.w);
      my += (unsigned long long)(k * k);
    }
    G[(int64_t)blockIdx.x * m.nc + L] = out;
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(evals, my);
  }
}

// ------------------------------------------------------------------ cross: gather
__device__ __forceinline__ double comp(const double4& g, int a, int b) {
  return a == 0 ? (b == 0 ? g.x : g.y) : (b == 0 ? g.z : g.w);
}

// ------------------------------------------------------------------ cross: fused DoF tiles
// The fused path never materialises the pair blocks: a CTA owns a T1 x T1 tile of DoFs
// (bi <= bj, mirrored), computes the blocks M^{K,L} of the <= T1C x T1C cell pairs behind it
// into shared memory and sums them into the tile in the same canonical order as gather1d.
// Cell pairs are bucketed by order inside the CTA so every warp evaluates 32 pairs of one
// order with the rule nodes in registers (no divergence, fully unrolled for k <= 6).
#ifndef FL_T1
#define FL_T1 32         // 64 measured slower (one 512-thread CTA per SM)
#endif
constexpr int T1 = FL_T1;                     // DoFs per tile side (32 or 64)
constexpr int T1C = T1 + 8;                   // max cells behind one DoF tile on the fused path
constexpr int T1X = T1 == 64 ? 512 : 256;     // threads of a tile CTA
constexpr int T1B = T1 == 64 ? 1 : FL_TILE1D_MINB;   // resident tile CTAs per SM
constexpr int T1K = 33;      // order buckets (KDIR)
constexpr int TSTAT = 8;     // doubles of tile statistics: x extent, max h, min / max |ln h|, ln(max h)

// one warp per DoF tile: sorted unique cells of the patches of its DoFs; per DoF the
// (slot << 1 | basis) of each patch cell (-1 = none); the owning tile of every cell
// (tiling of the DoF range [off, off + len): tile t = DoFs off + 32 t ...; dslot is indexed
// relative to off)
__global__ void tile1d_cells_kernel(DevMesh m, const int* __restrict__ dof_vertex, int off, int len, int nt,
                                    int* __restrict__ tcnt, int* __restrict__ tcell, int* __restrict__ dslot,
                                    int* __restrict__ owner, double* __restrict__ tstat, int* __restrict__ maxcnt) {
  constexpr int DPL = T1 / 32;                  // DoFs per lane
  constexpr int NCAND = 2 * T1;                 // candidate position q = (u * 2 + h) * 32 + lane
  __shared__ int cand[4][NCAND];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 4 + w;
  if (t >= nt) return;
  int c[DPL][2], vi[DPL];
  bool anyover = false;
#pragma unroll
  for (int u = 0; u < DPL; ++u) {
    const int li = t * T1 + u * 32 + lane;
    c[u][0] = c[u][1] = INT_MAX;
    vi[u] = -1;
    if (li < len) {
      vi[u] = dof_vertex[off + li];
      const int b = m.patch_off[vi[u]];
      const int np = m.patch_off[vi[u] + 1] - b;
      if (np > 0) c[u][0] = m.patch_cells[b];
      if (np > 1) c[u][1] = m.patch_cells[b + 1];
      anyover |= np > 2;
    }
  }
  if (__any_sync(0xffffffffu, anyover)) {       // not an interval mesh patch: no fused path
    if (lane == 0) atomicMax(maxcnt, 1 << 20);
    return;
  }
#pragma unroll
  for (int u = 0; u < DPL; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) cand[w][(u * 2 + h) * 32 + lane] = c[u][h];
  __syncwarp();
  // first occurrence flags (per 32-candidate group), then unique rank = distinct values below
  bool first[DPL][2];
  unsigned fm[2 * DPL];
#pragma unroll
  for (int u = 0; u < DPL; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = c[u][h], me = (u * 2 + h) * 32 + lane;
      bool f = true;
      for (int q = 0; q < me; ++q) f = f && (cand[w][q] != v);
      first[u][h] = f;
      fm[u * 2 + h] = __ballot_sync(0xffffffffu, f);
    }
  int rk[DPL][2];
  int nuniq = 0;
#pragma unroll
  for (int u = 0; u < DPL; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = c[u][h];
      int r = 0;
      for (int q = 0; q < NCAND; ++q) r += (((fm[q >> 5] >> (q & 31)) & 1u) && cand[w][q] < v);
      rk[u][h] = r;
      nuniq += (v != INT_MAX && first[u][h]);
    }
  const int ncand_unique = __reduce_add_sync(0xffffffffu, nuniq);
  {   // tile statistics for the order bound: x extent of the cells, max h, min / max |ln h|
    double lo = 1e300, hi = -1e300, hmx = 0.0, lmn = 1e300, lmx = 0.0;
#pragma unroll
    for (int u = 0; u < DPL; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = c[u][h];
        if (cc != INT_MAX) {
          const CellGeo& g = m.geo[cc];
          lo = fmin(lo, fmin(g.p[0][0], g.p[1][0]));
          hi = fmax(hi, fmax(g.p[0][0], g.p[1][0]));
          hmx = fmax(hmx, g.diam);
          lmn = fmin(lmn, g.ldiam);
          lmx = fmax(lmx, g.ldiam);
        }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      hmx = fmax(hmx, __shfl_xor_sync(0xffffffffu, hmx, o));
      lmn = fmin(lmn, __shfl_xor_sync(0xffffffffu, lmn, o));
      lmx = fmax(lmx, __shfl_xor_sync(0xffffffffu, lmx, o));
    }
    if (lane == 0) {
      double* st = tstat + TSTAT * t;
      st[0] = lo; st[1] = hi; st[2] = hmx; st[3] = lmn; st[4] = lmx; st[5] = log(hmx); st[6] = 0.0; st[7] = 0.0;
    }
  }
  if (lane == 0) {
    tcnt[t] = ncand_unique;
    atomicMax(maxcnt, ncand_unique);
  }
  if (ncand_unique > T1C) return;
#pragma unroll
  for (int u = 0; u < DPL; ++u) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (c[u][h] != INT_MAX && first[u][h]) {
        tcell[(size_t)t * T1C + rk[u][h]] = c[u][h];
        atomicMin(&owner[c[u][h]], t);
      }
    const int li = t * T1 + u * 32 + lane;
    if (li < len) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        dslot[2 * li + h] = c[u][h] != INT_MAX ? (rk[u][h] << 1 | (m.cells[2 * c[u][h]] == vi[u] ? 0 : 1)) : -1;
    }
  }
}

template <int KK, int E4>
__device__ __forceinline__ double4 block1d_k(const double* __restrict__ nd, double kx0, double ke, double lx0,
                                             double le, double JJ, double ex) {
  double tq[KK], w0[KK], w1[KK], Y[KK];
#pragma unroll
  for (int r = 0; r < KK; ++r) {
    tq[r] = nd[r * NODE];
    w0[r] = nd[r * NODE + 3];
    w1[r] = nd[r * NODE + 4];
    Y[r] = lx0 + tq[r] * le;
  }
  double m00 = 0, m01 = 0, m10 = 0, m11 = 0;
#pragma unroll
  for (int x = 0; x < KK; ++x) {
    const double X = kx0 + tq[x] * ke;
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int y = 0; y < KK; ++y) {
      const double d = X - Y[y];
      const double v = kpow_abs<E4>(d, ex);
      t0 = fma(v, w0[y], t0);
      t1 = fma(v, w1[y], t1);
    }
    m00 = fma(w0[x], t0, m00);
    m01 = fma(w0[x], t1, m01);
    m10 = fma(w1[x], t0, m10);
    m11 = fma(w1[x], t1, m11);
  }
  return make_double4(m00 * JJ, m01 * JJ, m10 * JJ, m11 * JJ);
}

// the order-2 rule held in registers (loaded once per CTA instead of once per pair)
struct Rule2 {
  double tq[2], w0[2], w1[2];
  __device__ explicit Rule2(const double* __restrict__ nd) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      tq[r] = __ldg(nd + r * NODE);
      w0[r] = __ldg(nd + r * NODE + 3);
      w1[r] = __ldg(nd + r * NODE + 4);
    }
  }
};
template <int E4>
__device__ __forceinline__ double4 block1d_2(const Rule2& R2, double kx0, double ke, double lx0, double le, double JJ,
                                             double ex) {
  const double Y0 = lx0 + R2.tq[0] * le, Y1 = lx0 + R2.tq[1] * le;
  double m00 = 0, m01 = 0, m10 = 0, m11 = 0;
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const double X = kx0 + R2.tq[x] * ke;
    const double v0 = kpow_abs<E4>(X - Y0, ex), v1 = kpow_abs<E4>(X - Y1, ex);
    const double t0 = fma(v1, R2.w0[1], v0 * R2.w0[0]);
    const double t1 = fma(v1, R2.w1[1], v0 * R2.w1[0]);
    m00 = fma(R2.w0[x], t0, m00);
    m01 = fma(R2.w0[x], t1, m01);
    m10 = fma(R2.w1[x], t0, m10);
    m11 = fma(R2.w1[x], t1, m11);
  }
  return make_double4(m00 * JJ, m01 * JJ, m10 * JJ, m11 * JJ);
}

struct Cell1S {   // shared-memory copy of a tile's cells
  double x0[T1C], x1[T1C], lo[T1C], hi[T1C], h[T1C], lh[T1C];
  float lnhf[T1C], lhf[T1C];
  int id[T1C], v0[T1C], v1[T1C], own[T1C];
};

// fp32 order estimate of the disjoint pair (P, Q) = (min, max) of two tile cells (reference
// orientation); 0 = ambiguous (resolved by order_exact1d outside the hot loop)
__device__ __forceinline__ int order_est1d(const OrderConsts& oc, const Cell1S& P, int ip, const Cell1S& Q, int iq,
                                           double& dist) {
  const double d1 = __dsub_rn(Q.lo[iq], P.hi[ip]), d2 = __dsub_rn(P.lo[ip], Q.hi[iq]);
  dist = fmax(fmax(d1, d2), 0.0);
  if (!(dist > 1e-30)) return 0;
  return order_from_estimate(order_estimate_f(oc, oc.coff_f, P.lnhf[ip], P.lhf[ip], Q.lnhf[iq], Q.lhf[iq],
                                              __logf((float)dist)), oc.cap_disjoint);
}

struct PairGeo1D {
  double px0, pe, qx0, qe, JJ;
  bool kl;
};
__device__ __forceinline__ PairGeo1D pair_geo1d(const Cell1S& cr, int a, const Cell1S& cc, int b) {
  PairGeo1D g;
  g.kl = cr.id[a] < cc.id[b];
  const Cell1S& P = g.kl ? cr : cc;
  const Cell1S& Q = g.kl ? cc : cr;
  const int ip = g.kl ? a : b, iq = g.kl ? b : a;
  g.px0 = P.x0[ip];
  g.pe = P.x1[ip] - g.px0;
  g.qx0 = Q.x0[iq];
  g.qe = Q.x1[iq] - g.qx0;
  g.JJ = P.h[ip] * Q.h[iq];
  return g;
}
// stored row cell first: Mp[aK * 2 + bL]
__device__ __forceinline__ void store_block1d(double* __restrict__ Mp, const double4& g, bool kl) {
  Mp[0] = g.x;
  Mp[1] = kl ? g.y : g.z;
  Mp[2] = kl ? g.z : g.y;
  Mp[3] = g.w;
}

template <int E4>
__device__ __forceinline__ double4 block1d_small(const double* __restrict__ tab, const DevTables& dir, double ex,
                                                 const PairGeo1D& q, int k) {
  const RuleRef rr = dir.rule(T_DISJ, k);
  const double* nd = tab + (size_t)rr.off * NODE;
  switch (k) {
    case 2: return block1d_k<2, E4>(nd, q.px0, q.pe, q.qx0, q.qe, q.JJ, ex);
    case 3: return block1d_k<3, E4>(nd, q.px0, q.pe, q.qx0, q.qe, q.JJ, ex);
    case 4: return block1d_k<4, E4>(nd, q.px0, q.pe, q.qx0, q.qe, q.JJ, ex);
    case 5: return block1d_k<5, E4>(nd, q.px0, q.pe, q.qx0, q.qe, q.JJ, ex);
    default: return block1d<E4>(tab, rr, q.px0, q.pe, q.qx0, q.qe, q.JJ, ex);
  }
}

// One pair, one warp (large k, up to 32^2 evaluations): lane x owns the x-node row of block1d,
// then every lane folds the rows in x order — the same operations in the same order as
// block1d, so the result is bitwise identical to the thread-per-pair path.
template <int E4>
__device__ __forceinline__ double4 block1d_warp(const double* __restrict__ tab, RuleRef rr, double kx0, double ke,
                                                double lx0, double le, double JJ, double ex, int lane) {
  double t0 = 0.0, t1 = 0.0;
  if (lane < rr.cnt) {
    const double* nx = tab + (size_t)(rr.off + lane) * NODE;
    const double X = kx0 + nx[0] * ke;
    for (int y = 0; y < rr.cnt; ++y) {
      const double* ny = tab + (size_t)(rr.off + y) * NODE;
      const double d = X - (lx0 + ny[0] * le);
      const double v = kpow_abs<E4>(d, ex);
      t0 = fma(v, ny[3], t0);
      t1 = fma(v, ny[4], t1);
    }
  }
  double m00 = 0, m01 = 0, m10 = 0, m11 = 0;
  for (int x = 0; x < rr.cnt; ++x) {
    const double* nx = tab + (size_t)(rr.off + x) * NODE;
    const double a0 = __shfl_sync(0xffffffffu, t0, x), a1 = __shfl_sync(0xffffffffu, t1, x);
    m00 = fma(nx[3], a0, m00);
    m01 = fma(nx[3], a1, m01);
    m10 = fma(nx[4], a0, m10);
    m11 = fma(nx[4], a1, m11);
  }
  return make_double4(m00 * JJ, m01 * JJ, m10 * JJ, m11 * JJ);
}

constexpr int T1WARP = 6;    // orders >= this get a warp per pair

// a tile's cell as the cross tiles stage it: one 80-byte record, tile-contiguous (one round trip)
struct __align__(16) TileCell {
  double x0, x1, lo, hi, h, lh;
  int id, v0, v1, own;
  float lnhf, lhf;
  int pad[2];
};

// one DoF tiling (rows or columns): cells per tile, per-DoF (slot << 1 | basis), cell owners
struct Tiling1D {
  const int *cnt, *cell, *dslot, *owner;
  const double* stat;    // per tile: x extent (lo, hi) of its cells, max h, min / max |ln h|, ln max h
  const TileCell* rec;   // per tile: T1C packed cell records
  int off, len, nt;
};

// True when every disjoint cell pair of the two tiles provably has order 2: the gap D between
// the tiles' x extents bounds every pair distance from below and the disjoint order formula
// (quadrature.py:159-168) from above (each numerator term bounded above, the denominator below);
// 1e-9 of margin absorbs rounding, so the reference's ceil() is 2 as well (clip floor).
// (ln(max h) comes precomputed per tile: one log per tile pair)
__device__ __forceinline__ bool tile_pair_all_k2(const OrderConsts& oc, const double* a, const double* b) {
  const double D = fmax(b[0] - a[1], a[0] - b[1]);
  if (!(D > 0.0)) return false;
  const double lhmx = fmax(a[5], b[5]), lmn = fmin(a[3], b[3]), lmx = fmax(a[4], b[4]);
  const double lD = log(D);
  const double num = oc.lead_lnn + oc.sm1 * lmn + lmx - oc.s * lD + oc.s * lhmx - oc.coff;
  const double den = fmax(lD - lhmx, 0.0) + oc.ln_rho2;
  return (num > 0.0 ? num / den : 0.0) <= 2.0 - 1e-9;
}

// RECT = false: the symmetric whole matrix, upper-triangular tile pairs (diagonal-major,
// heavy first), each off-diagonal tile mirrored.  RECT = true: rows [R.off, R.off + R.len)
// (one GPU's row block) x all columns, every tile pair computed (owner computes).  Both give
// bitwise the same entries: the pair blocks are computed in the reference orientation and
// summed in gather1d's canonical order.
template <int E4, bool RECT>
__global__ void __launch_bounds__(T1X, T1B) cross1d_tile_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                           OrderConsts oc, double ex, Src1D S, Tiling1D R,
                                                           Tiling1D Cn, int mc, double negC, double* __restrict__ A,
                                                           int64_t lda, unsigned long long* __restrict__ evals,
                                                           int band0, int band1,
                                                           const unsigned char* __restrict__ k2flags) {
  extern __shared__ __align__(16) unsigned char smem1d[];
  __shared__ Cell1S cr, cc;
  __shared__ int bcnt[T1K], boff[T1K + 1], ndefer, uni2;
  __shared__ int rA[T1][2], cB[T1][2];
  const int64_t bx = blockIdx.x;
  int bi, bj;
  if (RECT) {
    bi = (int)(bx / Cn.nt);
    bj = (int)(bx - (int64_t)bi * Cn.nt);
  } else if (band1 > band0) {
    // band of tile rows [band0, band1): row-major over the upper-triangular tile pairs of those
    // rows (the diagonal tile, the heaviest, first in each row); the rows of the band are final
    // once the earlier bands (their mirrors) and this one have run
    const int nt = R.nt;
    auto cum = [&](int64_t r) { return (r - band0) * nt - (r * (r - 1) - (int64_t)band0 * (band0 - 1)) / 2; };
    // cum(r) = bx  <=>  r^2 - (2 nt + 1) r + 2 bx + 2 b0 nt - b0 (b0 - 1) = 0; then fix up
    const double q2 = 2.0 * nt + 1.0, b0 = band0;
    const double disc = q2 * q2 - 4.0 * (2.0 * (double)bx + 2.0 * b0 * nt - b0 * (b0 - 1.0));
    int r = (int)((q2 - sqrt(fmax(disc, 0.0))) * 0.5);
    r = max(band0, min(r, band1 - 1));
    while (r > band0 && cum(r) > bx) --r;
    while (r + 1 < band1 && cum(r + 1) <= bx) ++r;
    bi = r;
    bj = bi + (int)(bx - cum(r));
  } else {
    // diagonal-major tile order (near-diagonal tiles hold the high orders: heavy first)
    const int nt = R.nt;
    const double q2 = 2.0 * nt + 1.0;
    int dg = (int)((q2 - sqrt(q2 * q2 - 8.0 * (double)bx)) * 0.5);
    auto cum = [&](int64_t e) { return e * nt - e * (e - 1) / 2; };
    while (dg > 0 && cum(dg) > bx) --dg;
    while (cum(dg + 1) <= bx) ++dg;
    bi = (int)(bx - cum(dg));
    bj = bi + dg;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = R.cnt[bi], ncl = Cn.cnt[bj];
  const int np = nr * ncl;
  const unsigned inv = ((1u << 20) + ncl - 1) / ncl;                 // p / ncl for p < 1600
  double* M = reinterpret_cast<double*>(smem1d);                      // [np][2][2]
  int* defer = reinterpret_cast<int*>(smem1d + sizeof(double) * 4 * (size_t)mc * mc);
  int* sorted = defer + mc * mc;

  for (int q = tid; q < 2 * T1C; q += blockDim.x) {
    Cell1S& C = q < T1C ? cr : cc;
    const int a = q < T1C ? q : q - T1C;
    // every slot is staged (slots past the tile's count hold zeros and are never read), so the
    // record loads do not wait for the count
    const TileCell t = q < T1C ? R.rec[(size_t)bi * T1C + a] : Cn.rec[(size_t)bj * T1C + a];
    C.id[a] = t.id; C.x0[a] = t.x0; C.x1[a] = t.x1; C.lo[a] = t.lo; C.hi[a] = t.hi;
    C.h[a] = t.h; C.lh[a] = t.lh; C.v0[a] = t.v0; C.v1[a] = t.v1;
    C.lnhf[a] = t.lnhf; C.lhf[a] = t.lhf; C.own[a] = t.own;
  }
  if (tid < T1K) bcnt[tid] = 0;
  if (tid == 0) {
    ndefer = 0;
    uni2 = k2flags[(size_t)bi * Cn.nt + bj];     // tile_pair_all_k2, precomputed (tile_flags_kernel)
  }
  if (tid < 2 * T1) {
    // per DoF and patch cell: its part of the M offset (row DoFs: slot row + basis a; column
    // DoFs: slot column + basis b), -1 = no such cell
    const int h = tid / T1, a = tid % T1;
    const int li = bi * T1 + a, lj = bj * T1 + a;
    const int si = li < R.len ? R.dslot[2 * li + h] : -1, sj = lj < Cn.len ? Cn.dslot[2 * lj + h] : -1;
    rA[a][h] = si < 0 ? -1 : 4 * (si >> 1) * ncl + 2 * (si & 1);
    cB[a][h] = sj < 0 ? -1 : 4 * (sj >> 1) + (sj & 1);
  }
  __syncthreads();

  // phase 1: every cell pair's order; k = 2 pairs (~95%) get their block right away.  Tile pairs
  // whose pairs are all provably of order 2 (~92% at c2) skip the orders (and have no touching pair)
  unsigned my = 0;
  const Rule2 R2(tab + (size_t)dir.rule(T_DISJ, 2).off * NODE);
  if (uni2) {
    for (int p = tid; p < np; p += blockDim.x) {
      const int a = (int)(((unsigned)p * inv) >> 20), b = p - a * ncl;
      const PairGeo1D g = pair_geo1d(cr, a, cc, b);
      store_block1d(M + 4 * p, block1d_2<E4>(R2, g.px0, g.pe, g.qx0, g.qe, g.JJ, ex), g.kl);
      const int oK = cr.own[a], oL = cc.own[b];
      if (g.kl && (RECT ? (oK == bi && oL == bj) : (min(oK, oL) == bi && max(oK, oL) == bj))) my += 4u;
    }
  }
  for (int p = uni2 ? np : tid; p < np; p += blockDim.x) {
    const int a = (int)(((unsigned)p * inv) >> 20), b = p - a * ncl;
    const int K = cr.id[a], L = cc.id[b];
    const int kv0 = cr.v0[a], kv1 = cr.v1[a], lv0 = cc.v0[b], lv1 = cc.v1[b];
    double* Mp = M + 4 * p;
    if (K == L || lv0 == kv0 || lv0 == kv1 || lv1 == kv0 || lv1 == kv1) {
      Mp[0] = 0.0; Mp[1] = 0.0; Mp[2] = 0.0; Mp[3] = 0.0;
      continue;
    }
    double dist;
    const int k = K < L ? order_est1d(oc, cr, a, cc, b, dist) : order_est1d(oc, cc, b, cr, a, dist);
    // algorithmic count: each unordered pair once, in the tile of its cells' owners
    const int oK = cr.own[a], oL = cc.own[b];
    const bool owned = K < L && (RECT ? (oK == bi && oL == bj) : (min(oK, oL) == bi && max(oK, oL) == bj));
    if (k == 2) {
      const PairGeo1D g = pair_geo1d(cr, a, cc, b);
      store_block1d(Mp, block1d_2<E4>(R2, g.px0, g.pe, g.qx0, g.qe, g.JJ, ex), g.kl);
      my += owned ? 4u : 0u;
    } else {
      if (k) {
        atomicAdd(&bcnt[k], 1);
        my += owned ? (unsigned)(k * k) : 0u;
      }
      defer[atomicAdd(&ndefer, 1)] = p | (k << 16);
    }
  }
  __syncthreads();
  const int nd = ndefer;
  if (nd > 0) {
    // ambiguous estimates: the exact fp64 order
    for (int it = tid; it < nd; it += blockDim.x) {
      const int e = defer[it];
      if (e >> 16) continue;
      const int p = e & 0xffff;
      const int a = (int)(((unsigned)p * inv) >> 20), b = p - a * ncl;
      const bool kl = cr.id[a] < cc.id[b];
      const Cell1S& P = kl ? cr : cc;
      const Cell1S& Q = kl ? cc : cr;
      const int ip = kl ? a : b, iq = kl ? b : a;
      const double dist = fmax(fmax(__dsub_rn(Q.lo[iq], P.hi[ip]), __dsub_rn(P.lo[ip], Q.hi[iq])), 0.0);
      const int k = order_exact1d(oc, oc.coff, P.h[ip], P.lh[ip], Q.h[iq], Q.lh[iq], dist);
      defer[it] = p | (k << 16);
      atomicAdd(&bcnt[k], 1);
      const int oK = cr.own[a], oL = cc.own[b];
      if (kl && (RECT ? (oK == bi && oL == bj) : (min(oK, oL) == bi && max(oK, oL) == bj))) my += (unsigned)(k * k);
    }
    __syncthreads();
    // sort by order: ascending k, so [0, nsmall) are thread-per-pair and the rest warp-per-pair
    if (tid < 32) {
      const int c = bcnt[tid];
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      boff[tid] = x - c;
      if (tid == 31) boff[32] = x;
    }
    __syncthreads();
    const int nsmall = boff[T1WARP];
    __syncthreads();
    for (int it = tid; it < nd; it += blockDim.x) {
      const int e = defer[it];
      sorted[atomicAdd(&boff[e >> 16], 1)] = e;
    }
    __syncthreads();
    for (int it = nsmall + warp; it < nd; it += blockDim.x >> 5) {
      const int e = sorted[it];
      const int p = e & 0xffff, k = e >> 16;
      const int a = (int)(((unsigned)p * inv) >> 20), b = p - a * ncl;
      const PairGeo1D g = pair_geo1d(cr, a, cc, b);
      const double4 v = block1d_warp<E4>(tab, dir.rule(T_DISJ, k), g.px0, g.pe, g.qx0, g.qe, g.JJ, ex, lane);
      if (lane == 0) store_block1d(M + 4 * p, v, g.kl);
    }
    for (int it = tid; it < nsmall; it += blockDim.x) {
      const int e = sorted[it];
      const int p = e & 0xffff, k = e >> 16;
      const int a = (int)(((unsigned)p * inv) >> 20), b = p - a * ncl;
      const PairGeo1D g = pair_geo1d(cr, a, cc, b);
      store_block1d(M + 4 * p, block1d_small<E4>(tab, dir, ex, g, k), g.kl);
    }
  }
  __syncthreads();

  // phase 3: A[i][j] = -C sum_{K in P(p)} sum_{L in P(q)} M, p = min(i, j), q = max(i, j)
  // (gather1d's canonical order; touching / identical pairs hold zeros, which add nothing)
  constexpr int EPT = T1 * T1 / T1X;            // entries per thread
  double v[EPT];
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int idx = tid + q * T1X, rr_ = idx / T1, tx = idx % T1;
    const int i = R.off + bi * T1 + rr_, j = Cn.off + bj * T1 + tx;
    const int o0 = rA[rr_][0], o1 = rA[rr_][1], i0 = cB[tx][0], i1 = cB[tx][1];
    double x = 0.0;
    if (i <= j) {                                // cells of i outer
      if (o0 >= 0 && i0 >= 0) x += negC * M[o0 + i0];
      if (o0 >= 0 && i1 >= 0) x += negC * M[o0 + i1];
      if (o1 >= 0 && i0 >= 0) x += negC * M[o1 + i0];
      if (o1 >= 0 && i1 >= 0) x += negC * M[o1 + i1];
    } else {                                     // cells of j outer
      if (o0 >= 0 && i0 >= 0) x += negC * M[o0 + i0];
      if (o1 >= 0 && i0 >= 0) x += negC * M[o1 + i0];
      if (o0 >= 0 && i1 >= 0) x += negC * M[o0 + i1];
      if (o1 >= 0 && i1 >= 0) x += negC * M[o1 + i1];
    }
    v[q] = x;
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int idx = tid + q * T1X, rr_ = idx / T1, tx = idx % T1;
    const int li = bi * T1 + rr_, lj = bj * T1 + tx;
    if (li < R.len && lj < Cn.len) A[(int64_t)(RECT ? li : R.off + li) * lda + Cn.off + lj] = v[q];
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
    if (lane == 0 && my) atomicAdd(evals, (unsigned long long)my);
  }
  if (RECT || bi == bj) return;
  // mirror through shared memory (reusing the pair-block buffer once every entry is read)
  __syncthreads();
  double* tt = M;                                // [T1][T1 + 1]
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int idx = tid + q * T1X, rr_ = idx / T1, tx = idx % T1;
    tt[rr_ * (T1 + 1) + tx] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int idx = tid + q * T1X, rr_ = idx / T1, tx = idx % T1;
    const int lj = bj * T1 + rr_, li = bi * T1 + tx;       // A[j][i] = tt[i][j]
    if (li < R.len && lj < Cn.len) A[(int64_t)lj * lda + li] = tt[tx * (T1 + 1) + rr_];
  }
}

// value of the cross part at (p, q), p <= q, in the canonical order (cells of p outer)
__device__ __forceinline__ double gather1d(const DevMesh& m, const Src1D& S, const double4* __restrict__ G,
                                           const int* __restrict__ dof_vertex, int p, int q, double negC) {
  const int vp = dof_vertex[p], vq = dof_vertex[q];
  double val = 0.0;
  for (int a_ = m.patch_off[vp]; a_ < m.patch_off[vp + 1]; ++a_) {
    const int K = m.patch_cells[a_];
    const int kv0 = S.v0[K], kv1 = S.v1[K];
    const int a = (kv0 == vp) ? 0 : 1;
    for (int b_ = m.patch_off[vq]; b_ < m.patch_off[vq + 1]; ++b_) {
      const int L = m.patch_cells[b_];
      const int lv0 = S.v0[L], lv1 = S.v1[L];
      if (K == L || lv0 == kv0 || lv0 == kv1 || lv1 == kv0 || lv1 == kv1) continue;
      const int b = (lv0 == vq) ? 0 : 1;
      const double g = (K < L) ? comp(G[tri_index(K, L, m.nc)], a, b) : comp(G[tri_index(L, K, m.nc)], b, a);
      val += negC * g;
    }
  }
  return val;
}

__global__ void __launch_bounds__(256) cross1d_gather_kernel(DevMesh m, Src1D S, const double4* __restrict__ G,
                                                             const int* __restrict__ dof_vertex, int n, double negC,
                                                             double* __restrict__ A, int64_t lda) {
  __shared__ double t[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bi > bj) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = bi * 32 + r, j = bj * 32 + tx;
    double v = 0.0;
    if (i < n && j < n) v = (i <= j) ? gather1d(m, S, G, dof_vertex, i, j, negC) : gather1d(m, S, G, dof_vertex, j, i, negC);
    t[r][tx] = v;
    if (i < n && j < n) A[(int64_t)i * lda + j] = v;
  }
  if (bi == bj) return;
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = bj * 32 + r, i = bi * 32 + tx;      // mirror: A[j][i] = t[i][j]
    if (i < n && j < n) A[(int64_t)j * lda + i] = t[tx][r];
  }
}

__global__ void __launch_bounds__(256) cross1d_gather_rows_kernel(DevMesh m, Src1D S, const double4* __restrict__ G,
                                                                  const int* __restrict__ tpos,
                                                                  const int* __restrict__ dof_vertex, int n, int r0,
                                                                  int r1, double negC, double* __restrict__ A,
                                                                  int64_t lda) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = r1 - r0;
  if (idx >= rows * n) return;
  const int i = r0 + (int)(idx / n), j = (int)(idx % n);
  const int vi = dof_vertex[i], vj = dof_vertex[j];
  // gather1d's canonical order: the cells of min(i, j) outer; G rows are i's (target) cells
  const bool sw = i > j;
  const int vo = sw ? vj : vi, vn = sw ? vi : vj;
  double val = 0.0;
  for (int a_ = m.patch_off[vo]; a_ < m.patch_off[vo + 1]; ++a_) {
    const int K = m.patch_cells[a_];
    const int kv0 = S.v0[K], kv1 = S.v1[K];
    const int a = (kv0 == vo) ? 0 : 1;
    for (int b_ = m.patch_off[vn]; b_ < m.patch_off[vn + 1]; ++b_) {
      const int L = m.patch_cells[b_];
      const int lv0 = S.v0[L], lv1 = S.v1[L];
      if (K == L || lv0 == kv0 || lv0 == kv1 || lv1 == kv0 || lv1 == kv1) continue;
      const int b = (lv0 == vn) ? 0 : 1;
      val += negC * (sw ? comp(G[(int64_t)tpos[L] * m.nc + K], b, a) : comp(G[(int64_t)tpos[K] * m.nc + L], a, b));
    }
  }
  A[(int64_t)(i - r0) * lda + j] = val;
}

__global__ void tpos_kernel(const int* targets, int nt, int* tpos) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nt) tpos[targets[t]] = t;
}

// ------------------------------------------------------------------ launchers
#define FL_E4_SWITCH1(e4, ...)                                \
  switch (e4) {                                               \
    case 6: { constexpr int E4 = 6; __VA_ARGS__; } break;     \
    case 8: { constexpr int E4 = 8; __VA_ARGS__; } break;     \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

struct Src1DBuf {
  DBuf<double> x0, x1, lo, hi, h, lh;
  DBuf<int> v0, v1;
  DBuf<float> lnhf, lhf;
  DBuf<Rec1D> rec;
  DBuf<double> cstat;
  Src1D view() const { return Src1D{rec.p, x0.p, x1.p, lo.p, hi.p, h.p, lh.p, v0.p, v1.p, lnhf.p, lhf.p, cstat.p}; }
};

static void build_src1d(const DevMesh& m, Src1DBuf& B, cudaStream_t st) {
  const int nc = m.nc;
  B.x0.alloc(nc); B.x1.alloc(nc); B.lo.alloc(nc); B.hi.alloc(nc); B.h.alloc(nc); B.lh.alloc(nc);
  B.v0.alloc(nc); B.v1.alloc(nc); B.lnhf.alloc(nc); B.lhf.alloc(nc); B.rec.alloc(nc);
  B.cstat.alloc((size_t)CSTAT * ((nc + 31) / 32));
  build_src1d_kernel<<<(nc + 255) / 256, 256, 0, st>>>(m, B.rec.p, B.x0.p, B.x1.p, B.lo.p, B.hi.p, B.h.p, B.lh.p, B.v0.p,
                                                        B.v1.p, B.lnhf.p, B.lhf.p, B.cstat.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

struct TilingBuf {
  DBuf<int> cnt, cell, dslot, owner;
  DBuf<double> stat;
  DBuf<TileCell> rec;
  int off = 0, len = 0, nt = 0;
  Tiling1D view() const { return Tiling1D{cnt.p, cell.p, dslot.p, owner.p, stat.p, rec.p, off, len, nt}; }
};

// the packed records of every tile's cells (after the owners are final)
__global__ void pack_tile_cells_kernel(Src1D S, const int* __restrict__ tcnt, const int* __restrict__ tcell,
                                       const int* __restrict__ owner, int nt, TileCell* __restrict__ rec) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)nt * T1C) return;
  const int t = (int)(q / T1C), a = (int)(q % T1C);
  if (tcnt[t] > T1C || a >= tcnt[t]) return;      // (over-full tiles: no fused path)
  const int c = tcell[q];
  TileCell r;
  r.x0 = S.x0[c]; r.x1 = S.x1[c]; r.lo = S.lo[c]; r.hi = S.hi[c]; r.h = S.h[c]; r.lh = S.lh[c];
  r.id = c; r.v0 = S.v0[c]; r.v1 = S.v1[c]; r.own = owner[c];
  r.lnhf = S.lnhf[c]; r.lhf = S.lhf[c]; r.pad[0] = r.pad[1] = 0;
  rec[q] = r;
}

// Everything the 1D far field needs from the mesh, enqueued without host synchronisation: the
// source records and, for the fused cross tiles, the DoF tilings with the max cells per tile on
// the device (read back together with the other sizes).
struct Plan1D {
  Src1DBuf B;
  TilingBuf TR, TC;
  DBuf<int> mx;
  bool fused = false, symmetric = true;
  int row_begin = 0, row_end = 0;
};

Plan1D* plan1d_create(const DevMesh& m, const int* dof_vertex, bool symmetric, int row_begin, int row_end,
                      cudaStream_t st) {
  std::unique_ptr<Plan1D> P(new Plan1D());
  P->symmetric = symmetric;
  P->row_begin = row_begin;
  P->row_end = row_end;
  build_src1d(m, P->B, st);
  P->mx.alloc(1);
  FL_CUDA(cudaMemsetAsync(P->mx.p, 0, sizeof(int), st));
  const char* path = getenv("FRACLAP_CROSS1D");
  const bool force_pairs = path && std::string(path) == "pairs";
  P->fused = !force_pairs && m.n > 0 && row_end > row_begin;
  if (P->fused) {
    auto make = [&](TilingBuf& T, int off, int len) {
      T.off = off; T.len = len; T.nt = (len + T1 - 1) / T1;
      T.cnt.alloc(T.nt); T.cell.alloc((size_t)T.nt * T1C); T.dslot.alloc((size_t)2 * len); T.owner.alloc(m.nc);
      T.stat.alloc((size_t)T.nt * TSTAT);
      FL_CUDA(cudaMemsetAsync(T.owner.p, 0x7f, sizeof(int) * m.nc, st));
      tile1d_cells_kernel<<<(T.nt + 3) / 4, 128, 0, st>>>(m, dof_vertex, off, len, T.nt, T.cnt.p, T.cell.p, T.dslot.p,
                                                          T.owner.p, T.stat.p, P->mx.p),
          ::fl::note_launch();
      T.rec.alloc((size_t)T.nt * T1C);
      FL_CUDA(cudaMemsetAsync(T.rec.p, 0, (size_t)T.nt * T1C * sizeof(TileCell), st));
      pack_tile_cells_kernel<<<(unsigned)(((int64_t)T.nt * T1C + 255) / 256), 256, 0, st>>>(
          P->B.view(), T.cnt.p, T.cell.p, T.owner.p, T.nt, T.rec.p),
          ::fl::note_launch();
      FL_CHECK_LAUNCH();
    };
    make(P->TC, 0, m.n);
    if (!symmetric) make(P->TR, row_begin, row_end - row_begin);
  }
  return P.release();
}
void plan1d_free(Plan1D* P) { delete P; }
const int* plan1d_maxcells(const Plan1D* P) { return P->mx.p; }

void launch_tail1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, const Plan1D* P,
                   const int* targets, const int* d_ntargets, int ntargets_ub, double* psi,
                   unsigned long long* evals, cudaStream_t st) {
  if (ntargets_ub <= 0) return;
  const Src1D S = P->B.view();
  constexpr int NT = FL_TAIL1D_NT;
  const int grid = (ntargets_ub + 4 * NT - 1) / (4 * NT);
  FL_E4_SWITCH1(e4, (tail1d_kernel<E4, NT><<<grid, 128, 0, st>>>(m, t.data, t, oc, ex, S, targets, d_ntargets, psi,
                                                                 evals),
                     ::fl::note_launch()));
  FL_CHECK_LAUNCH();
}

bool cross1d_fits(const DevMesh& m, int64_t ntargets, bool symmetric) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  const double need = symmetric ? 32.0 * (double)m.nc * (m.nc - 1) / 2 : 32.0 * (double)ntargets * m.nc;
  return need < 0.5 * (double)fr;
}

// tile_pair_all_k2 of every (row tile, column tile) in row tiles [r0, r1), ahead of the tile kernel
// (its fp64 log would otherwise sit on one thread in front of the tile's first barrier)
__global__ void tile_flags_kernel(OrderConsts oc, const double* __restrict__ rstat, const double* __restrict__ cstat,
                                  int r0, int r1, int ntc, unsigned char* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)(r1 - r0) * ntc) return;
  const int bi = r0 + (int)(t / ntc), bj = (int)(t % ntc);
  flags[(size_t)bi * ntc + bj] = tile_pair_all_k2(oc, rstat + TSTAT * bi, cstat + TSTAT * bj) ? 1 : 0;
}

bool cross1d_fused(const Plan1D* P, int maxcells) { return P->fused && maxcells <= T1C; }
int cross1d_tile_dofs() { return T1; }

bool launch_cross1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                    const Plan1D* P, int maxcells, const int* targets, int ntargets, const int* dof_vertex,
                    double* A, int64_t lda, unsigned long long* evals, cudaStream_t st, int band_row0,
                    int band_row1) {
  const Src1D S = P->B.view();
  const bool symmetric = P->symmetric;
  const int row_begin = P->row_begin, row_end = P->row_end;
  const double negC = -Cds;   // (C/2) * (-2) (assembly.py:723, :1100)
  if (P->fused && maxcells <= T1C) {
    // fused DoF tiles: every tile's cells fit the shared-memory pair table
    const int mc = std::max(maxcells, 1);
    const size_t smem = std::max((sizeof(double4) + 2 * sizeof(int)) * (size_t)mc * mc,
                                 sizeof(double) * (size_t)T1 * (T1 + 1));   // tt aliases the blocks
    const Tiling1D cv = P->TC.view(), rv = symmetric ? cv : P->TR.view();
    int64_t ntp = symmetric ? (int64_t)cv.nt * (cv.nt + 1) / 2 : (int64_t)rv.nt * cv.nt;
    int b0 = 0, b1 = 0;   // band of tile rows (symmetric whole matrix only; b1 = 0: all tiles)
    if (symmetric && band_row1 > band_row0) {
      if (band_row0 % T1) throw Error(FL_E_CUDA, "internal: band start not tile aligned");
      b0 = band_row0 / T1;
      b1 = std::min(cv.nt, (band_row1 + T1 - 1) / T1);
      ntp = (int64_t)(b1 - b0) * cv.nt - ((int64_t)b1 * (b1 - 1) - (int64_t)b0 * (b0 - 1)) / 2;
      if (ntp <= 0) return true;
    }
    DBuf<unsigned char> flags((size_t)rv.nt * cv.nt);
    {
      const int r0 = b1 > b0 ? b0 : 0, r1 = b1 > b0 ? b1 : rv.nt;
      const int64_t tot = (int64_t)(r1 - r0) * cv.nt;
      tile_flags_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(oc, rv.stat, cv.stat, r0, r1, cv.nt, flags.p);
      ::fl::note_launch();
    }
    FL_E4_SWITCH1(e4, {
      if (symmetric) {
        auto kern = cross1d_tile_kernel<E4, false>;
        FL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)ntp, T1X, smem, st>>>(m, t.data, t, oc, ex, S, rv, cv, mc, negC, A, lda, evals, b0, b1,
                                               flags.p);
      } else {
        auto kern = cross1d_tile_kernel<E4, true>;
        FL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)ntp, T1X, smem, st>>>(m, t.data, t, oc, ex, S, rv, cv, mc, negC, A, lda, evals, 0, 0,
                                               flags.p);
      }
      ::fl::note_launch();
    });
    FL_CHECK_LAUNCH();
    return true;
  }
  if (band_row1 > band_row0) throw Error(FL_E_CUDA, "internal: banded cross term needs the fused tiles");
  if (!cross1d_fits(m, ntargets, symmetric)) return false;   // pair buffer too large: caller uses tiles
  if (symmetric) {
    DBuf<double4> G((size_t)std::max<int64_t>((int64_t)m.nc * (m.nc - 1) / 2, 1));
    FL_E4_SWITCH1(e4, (cross1d_pairs_kernel<E4><<<m.nc, 256, 0, st>>>(m, t.data, t, oc, ex, S, G.p, evals),
                       ::fl::note_launch()));
    FL_CHECK_LAUNCH();
    const int nt = (m.n + 31) / 32;
    cross1d_gather_kernel<<<dim3(nt, nt), 256, 0, st>>>(m, S, G.p, dof_vertex, m.n, negC, A, lda),
        ::fl::note_launch();
    FL_CHECK_LAUNCH();
  } else {
    DBuf<double4> G((size_t)std::max<int64_t>((int64_t)ntargets * m.nc, 1));
    DBuf<int> tpos(m.nc);
    tpos_kernel<<<(ntargets + 255) / 256, 256, 0, st>>>(targets, ntargets, tpos.p), ::fl::note_launch();
    FL_E4_SWITCH1(e4, (cross1d_rect_kernel<E4><<<ntargets, 256, 0, st>>>(m, t.data, t, oc, ex, S, targets, G.p, evals),
                       ::fl::note_launch()));
    FL_CHECK_LAUNCH();
    const int64_t tot = (int64_t)(row_end - row_begin) * m.n;
    cross1d_gather_rows_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(m, S, G.p, tpos.p, dof_vertex, m.n,
                                                                         row_begin, row_end, negC, A, lda),
        ::fl::note_launch();
    FL_CHECK_LAUNCH();
  }
  return true;
}

}  // namespace fl
