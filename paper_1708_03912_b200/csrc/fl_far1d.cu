// 1D far field.  In 1D a disjoint pair carries only k x k cross evaluations and 6 k tail
// evaluations (k = 2 for ~90% of the pairs of the graded BASELINE mesh), so per-pair cost —
// not arithmetic — dominates.  The 1D kernels therefore use lean, barrier-free layouts:
//
//  * tail1d:  one warp per target cell, one LANE per source cell, six per-lane accumulators
//             (the six cell-rule nodes), a single warp reduction at the end.  Source data is
//             read from structure-of-arrays (coalesced, no 128-B record loads).
//  * cross1d: every unordered disjoint pair (K < L) gets its 2x2 block M^{K,L} once
//             (cross_matrices, assembly.py:172-229, orders in the reference's (min, max)
//             orientation) into a packed triangular buffer; a tiled gather then forms
//             A[i][j] = -C sum_{K∋i, L∋j} M[a][b] (assembly.py:723-725) with the sum taken in
//             one canonical order for (i, j) and (j, i): the cross part is exactly symmetric
//             and no halo pair is ever evaluated twice.
// Row-block (multi-GPU) mode computes the ordered pairs (K in the owned rows' cells, all L)
// into a rectangular buffer instead.
#include "fl_internal.h"

namespace fl {

struct Src1D {
  const double *x0, *x1, *lo, *hi, *h, *lh;
  const int *v0, *v1;
};

__global__ void build_src1d_kernel(DevMesh m, double* x0, double* x1, double* lo, double* hi, double* h,
                                   double* lh, int* v0, int* v1) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
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
}

// ------------------------------------------------------------------ tail
template <int E4>
__global__ void __launch_bounds__(128, 4) tail1d_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                     OrderConsts oc, double ex, Src1D S,
                                                     const int* __restrict__ targets, int ntargets,
                                                     double* __restrict__ psi,
                                                     unsigned long long* __restrict__ evals) {
  constexpr int Q = 6;
  const int lane = threadIdx.x & 31;
  const int ti = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ti >= ntargets) return;
  const int K = targets[ti];
  const double alo = S.lo[K], ahi = S.hi[K], ah = S.h[K], alh = S.lh[K];
  const int av0 = S.v0[K], av1 = S.v1[K];
  double xq[Q], acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    xq[q] = m.X[(size_t)K * Q + q];
    acc[q] = 0.0;
  }
  unsigned long long nodes = 0;
  for (int s = lane; s < m.nc; s += 32) {
    const int bv0 = S.v0[s], bv1 = S.v1[s];
    if (s == K || bv0 == av0 || bv0 == av1 || bv1 == av0 || bv1 == av1) continue;   // N(K) (:999-1009)
    const double blo = S.lo[s], bhi = S.hi[s];
    const double dist = fmax(fmax(__dsub_rn(blo, ahi), __dsub_rn(alo, bhi)), 0.0);   // (:750-752)
    const int k = order_disjoint_fast_s(oc, oc.coff_tail, ah, alh, S.h[s], S.lh[s], dist);
    const RuleRef rr = dir.rule(T_DISJ, k);
    const double x0 = S.x0[s], e = S.x1[s] - x0, J = S.h[s];
    nodes += (unsigned long long)k;
    for (int r = 0; r < k; ++r) {
      const double* nd = tab + (size_t)(rr.off + r) * NODE;
      const double y = x0 + nd[0] * e;
      const double jw = J * nd[2];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double d = xq[q] - y;
        acc[q] = fma(jw, kpow<E4>(d * d, ex), acc[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double v = warp_sum(acc[q]);
    if (lane == 0) psi[(size_t)K * Q + q] = v;
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nodes += __shfl_xor_sync(0xffffffffu, nodes, o);
    if (lane == 0) atomicAdd(evals, nodes * Q);
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
      const double v = kpow<E4>(d * d, ex);
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
  const double alo = S.lo[K], ahi = S.hi[K], ah = S.h[K], alh = S.lh[K], kx0 = S.x0[K];
  const double ke = S.x1[K] - kx0;
  const int av0 = S.v0[K], av1 = S.v1[K];
  unsigned long long my = 0;
  for (int L = threadIdx.x; L < m.nc; L += blockDim.x) {
    const int bv0 = S.v0[L], bv1 = S.v1[L];
    double4 out = make_double4(0, 0, 0, 0);
    if (L != K && !(bv0 == av0 || bv0 == av1 || bv1 == av0 || bv1 == av1)) {
      // order in the reference's (min, max) orientation; block with K as the x cell
      const int P = min(K, L), Qc = max(K, L);
      const double dist = fmax(fmax(__dsub_rn(S.lo[Qc], S.hi[P]), __dsub_rn(S.lo[P], S.hi[Qc])), 0.0);
      const int k = order_disjoint_fast_s(oc, oc.coff, S.h[P], S.lh[P], S.h[Qc], S.lh[Qc], dist);
      const double lx0 = S.x0[L];
      out = block1d<E4>(tab, dir.rule(T_DISJ, k), kx0, ke, lx0, S.x1[L] - lx0, ah * S.h[L], ex);
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
  double val = 0.0;
  for (int a_ = m.patch_off[vi]; a_ < m.patch_off[vi + 1]; ++a_) {
    const int K = m.patch_cells[a_];
    const int kv0 = S.v0[K], kv1 = S.v1[K];
    const int a = (kv0 == vi) ? 0 : 1;
    for (int b_ = m.patch_off[vj]; b_ < m.patch_off[vj + 1]; ++b_) {
      const int L = m.patch_cells[b_];
      const int lv0 = S.v0[L], lv1 = S.v1[L];
      if (K == L || lv0 == kv0 || lv0 == kv1 || lv1 == kv0 || lv1 == kv1) continue;
      const int b = (lv0 == vj) ? 0 : 1;
      val += negC * comp(G[(int64_t)tpos[K] * m.nc + L], a, b);
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
  Src1D view() const { return Src1D{x0.p, x1.p, lo.p, hi.p, h.p, lh.p, v0.p, v1.p}; }
};

static void build_src1d(const DevMesh& m, Src1DBuf& B, cudaStream_t st) {
  const int nc = m.nc;
  B.x0.alloc(nc); B.x1.alloc(nc); B.lo.alloc(nc); B.hi.alloc(nc); B.h.alloc(nc); B.lh.alloc(nc);
  B.v0.alloc(nc); B.v1.alloc(nc);
  build_src1d_kernel<<<(nc + 255) / 256, 256, 0, st>>>(m, B.x0.p, B.x1.p, B.lo.p, B.hi.p, B.h.p, B.lh.p, B.v0.p,
                                                        B.v1.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

void launch_tail1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                   const int* targets, int ntargets, double* psi, unsigned long long* evals, cudaStream_t st) {
  if (ntargets <= 0) return;
  Src1DBuf B;
  build_src1d(m, B, st);
  const Src1D S = B.view();
  const int grid = (ntargets + 3) / 4;
  FL_E4_SWITCH1(e4, (tail1d_kernel<E4><<<grid, 128, 0, st>>>(m, t.data, t, oc, ex, S, targets, ntargets, psi, evals),
                     ::fl::note_launch()));
  FL_CHECK_LAUNCH();
}

bool cross1d_fits(const DevMesh& m, int64_t ntargets, bool symmetric) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  const double need = symmetric ? 32.0 * (double)m.nc * (m.nc - 1) / 2 : 32.0 * (double)ntargets * m.nc;
  return need < 0.5 * (double)fr;
}

void launch_cross1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                    const int* targets, int ntargets, const int* dof_vertex, bool symmetric, int row_begin,
                    int row_end, double* A, int64_t lda, unsigned long long* evals, cudaStream_t st) {
  Src1DBuf B;
  build_src1d(m, B, st);
  const Src1D S = B.view();
  const double negC = -Cds;   // (C/2) * (-2) (assembly.py:723, :1100)
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
  FL_CUDA(cudaStreamSynchronize(st));
}

}  // namespace fl
