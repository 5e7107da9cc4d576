// Singular near-field quadrature: one warp per element pair, lanes stride over the rule's
// nodes, 15 symmetric accumulators reduced with warp shuffles.
//
//  * touching pairs (IDENTICAL / COMMON_EDGE / COMMON_VERTEX): pair_matrices
//    (assembly.py:143-169) with the hat-difference matrices of _hat_difference (:99-126);
//  * boundary (cell, edge) pairs EDGE_OF_CELL / TOUCHING_EDGE: boundary_pair_matrices
//    (assembly.py:232-277), inward normal, 1D point form (:242-259).
// Coordinates are mapped to ABSOLUTE positions before the difference, exactly like
// _map_points (:129-132) — required for parity on the graded mesh (SURVEY.md §0 hazard 4).
#include "fl_internal.h"

namespace fl {

template <int D>
__device__ __forceinline__ void map_pt(const double (&P)[3][2], double u0, double u1, double& X0, double& X1) {
  if constexpr (D == 1) {
    X0 = P[0][0] + u0 * (P[1][0] - P[0][0]);
    X1 = 0.0;
  } else {
    const double e00 = P[1][0] - P[0][0], e01 = P[1][1] - P[0][1];
    const double e10 = P[2][0] - P[0][0], e11 = P[2][1] - P[0][1];
    X0 = P[0][0] + (u0 * e00 + u1 * e10);
    X1 = P[0][1] + (u0 * e01 + u1 * e11);
  }
}

template <int D>
__device__ __forceinline__ double jac(const double (&P)[3][2]) {
  if constexpr (D == 1) {
    return fabs(__dsub_rn(P[1][0], P[0][0]));
  } else {
    const double ax = __dsub_rn(P[1][0], P[0][0]), ay = __dsub_rn(P[1][1], P[0][1]);
    const double bx = __dsub_rn(P[2][0], P[0][0]), by = __dsub_rn(P[2][1], P[0][1]);
    return fabs(__dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx)));
  }
}

// Hat differences D[n, a] (assembly.py:104-126) for one node.
template <int D, int TOPO>
__device__ __forceinline__ int hat_diff(double x0, double x1, double y0, double y1, double (&Dv)[5]) {
  if constexpr (D == 1) {
    if constexpr (TOPO == T_IDENT) {
      Dv[0] = (1.0 - x0) - (1.0 - y0); Dv[1] = x0 - y0; return 2;
    } else {  // COMMON_VERTEX
      Dv[0] = (1.0 - x0) - (1.0 - y0); Dv[1] = x0; Dv[2] = -y0; return 3;
    }
  } else {
    const double lx0 = (1.0 - x0) - x1, ly0 = (1.0 - y0) - y1;
    if constexpr (TOPO == T_IDENT) {
      Dv[0] = lx0 - ly0; Dv[1] = x0 - y0; Dv[2] = x1 - y1; return 3;
    } else if constexpr (TOPO == T_CE) {
      Dv[0] = lx0 - ly0; Dv[1] = x0 - y0; Dv[2] = x1; Dv[3] = -y1; return 4;
    } else {  // T_CV
      Dv[0] = lx0 - ly0; Dv[1] = x0; Dv[2] = x1; Dv[3] = -y0; Dv[4] = -y1; return 5;
    }
  }
}

template <int NL>
__device__ __forceinline__ void reduce_store(double (&acc)[15], double scale, double* out) {
  int idx = 0;
#pragma unroll
  for (int a = 0; a < NL; ++a)
#pragma unroll
    for (int b = a; b < NL; ++b) {
      const double v = warp_sum(acc[idx++]) * scale;
      if ((threadIdx.x & 31) == 0) { out[a * 5 + b] = v; out[b * 5 + a] = v; }
    }
}

// One (canonical) touching pair: PK, PK2 in canonical vertex order.
template <int D, int E4, int TOPO>
__device__ void pair_quad(const double* __restrict__ tab, RuleRef r, const double (&PK)[3][2],
                          const double (&PK2)[3][2], double ex, double scale, double* out) {
  constexpr int NL = (D == 1) ? (TOPO == T_IDENT ? 2 : 3) : (TOPO == T_IDENT ? 3 : (TOPO == T_CE ? 4 : 5));
  double acc[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) acc[i] = 0.0;
  const int lane = threadIdx.x & 31;
  for (int n = lane; n < r.cnt; n += 32) {
    const double* nd = tab + (size_t)(r.off + n) * NODE;
    const double x0 = nd[0], x1 = nd[1], y0 = nd[2], y1 = nd[3], w = nd[4];
    double X0, X1, Y0, Y1;
    map_pt<D>(PK, x0, x1, X0, X1);
    map_pt<D>(PK2, y0, y1, Y0, Y1);
    const double dx = X0 - Y0, dy = X1 - Y1;
    const double r2 = (D == 1) ? __dmul_rn(dx, dx) : __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    const double kern = kpow<E4>(r2, ex);
    double Dv[5];
    hat_diff<D, TOPO>(x0, x1, y0, y1, Dv);
    int idx = 0;
#pragma unroll
    for (int a = 0; a < NL; ++a) {
      const double ka = kern * (Dv[a] * w);
#pragma unroll
      for (int b = a; b < NL; ++b) acc[idx++] += ka * Dv[b];
    }
  }
  reduce_store<NL>(acc, scale, out);
}

template <int D, int E4>
__global__ void __launch_bounds__(128) touching_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                       double ex, const TouchPair* __restrict__ pairs,
                                                       int64_t npairs, double* out) {
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p >= npairs) return;
  const TouchPair tp = pairs[p];
  double PK[3][2] = {}, PK2[3][2] = {};
  for (int i = 0; i <= D; ++i)
    for (int j = 0; j < D; ++j) {
      PK[i][j] = m.vert[tp.vK[i] * D + j];
      PK2[i][j] = m.vert[tp.vK2[i] * D + j];
    }
  const double scale = jac<D>(PK) * jac<D>(PK2);
  const RuleRef r = dir.rule(tp.topo, tp.k);
  if (r.cnt == 0) { if ((threadIdx.x & 31) == 0) atomicOr(m.err, 1); return; }
  double* o = out + p * 25;
  if (tp.topo == T_CE) {
    if constexpr (D == 2) pair_quad<D, E4, T_CE>(tab, r, PK, PK2, ex, scale, o);
  } else {
    pair_quad<D, E4, T_CV>(tab, r, PK, PK2, ex, scale, o);
  }
}

template <int D, int E4>
__global__ void __launch_bounds__(128) identical_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                        double ex, const int* __restrict__ ident_k, double* out) {
  const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= m.nc) return;
  const CellGeo g = m.geo[c];
  double PK[3][2];
  for (int i = 0; i < 3; ++i) { PK[i][0] = g.p[i][0]; PK[i][1] = g.p[i][1]; }
  const double J = jac<D>(PK);
  const RuleRef r = dir.rule(T_IDENT, D == 1 ? 0 : ident_k[c]);
  if (r.cnt == 0) { if ((threadIdx.x & 31) == 0) atomicOr(m.err, 1); return; }
  double tmp[25];
  __shared__ double sh[4][25];
  double* o = sh[threadIdx.x >> 5];
  pair_quad<D, E4, T_IDENT>(tab, r, PK, PK, ex, J * J, o);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  if (lane < (D + 1) * (D + 1)) {
    const int a = lane / (D + 1), b = lane % (D + 1);
    out[(size_t)c * 9 + a * 3 + b] = o[a * 5 + b];
  }
  (void)tmp;
}

template <int D, int E4>
__global__ void __launch_bounds__(128) boundary_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                       double ex, const BndPair* __restrict__ items,
                                                       int64_t nitems, double* out) {
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p >= nitems) return;
  const BndPair it = items[p];
  double PK[3][2] = {};
  for (int i = 0; i <= D; ++i)
    for (int j = 0; j < D; ++j) PK[i][j] = m.vert[it.locs[i] * D + j];
  const RuleRef r = dir.rule(it.topo, D == 1 ? 0 : it.k);
  if (r.cnt == 0) { if ((threadIdx.x & 31) == 0) atomicOr(m.err, 1); return; }
  double acc[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) acc[i] = 0.0;
  const int lane = threadIdx.x & 31;
  double scale;
  if constexpr (D == 1) {
    const double pnt = it.pe[0][0];
    const double far = PK[1][0];                 // PK[0] is the boundary point (:252)
    for (int n = lane; n < r.cnt; n += 32) {
      const double* nd = tab + (size_t)(r.off + n) * NODE;
      const double xh = nd[0], w = nd[3];
      const double X = pnt + xh * (far - pnt);
      const double diff = X - pnt;               // absolute, then subtract (:253-254)
      const double ndot = it.ne[0] * diff;
      const double kern = kpow<E4>(__dmul_rn(diff, diff), ex) * ndot;
      const double lam[2] = {1.0 - xh, xh};
      acc[0] += kern * (lam[0] * w) * lam[0];
      acc[1] += kern * (lam[0] * w) * lam[1];
      acc[2] += kern * (lam[1] * w) * lam[1];
    }
    scale = jac<1>(PK);
    const double v00 = warp_sum(acc[0]) * scale, v01 = warp_sum(acc[1]) * scale, v11 = warp_sum(acc[2]) * scale;
    if (lane == 0) {
      double* o = out + p * 9;
      o[0] = v00; o[1] = v01; o[3] = v01; o[4] = v11;
      o[2] = o[5] = o[6] = o[7] = o[8] = 0.0;
    }
  } else {
    const double ex0 = it.pe[1][0] - it.pe[0][0], ex1 = it.pe[1][1] - it.pe[0][1];
    for (int n = lane; n < r.cnt; n += 32) {
      const double* nd = tab + (size_t)(r.off + n) * NODE;
      const double x0 = nd[0], x1 = nd[1], a = nd[2], w = nd[3];
      double X0, X1;
      map_pt<2>(PK, x0, x1, X0, X1);
      const double Y0 = it.pe[0][0] + a * ex0, Y1 = it.pe[0][1] + a * ex1;
      const double dx = X0 - Y0, dy = X1 - Y1;
      const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      const double ndot = dx * it.ne[0] + dy * it.ne[1];
      const double kern = kpow<E4>(r2, ex) * ndot;
      const double lam[3] = {(1.0 - x0) - x1, x0, x1};
      int idx = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double ka = kern * (lam[i] * w);
#pragma unroll
        for (int j = i; j < 3; ++j) acc[idx++] += ka * lam[j];
      }
    }
    const double LE = norm2d(ex0, ex1);
    scale = jac<2>(PK) * LE;
    double* o = out + p * 9;
    int idx = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) {
        const double v = warp_sum(acc[idx++]) * scale;
        if (lane == 0) { o[i * 3 + j] = v; o[j * 3 + i] = v; }
      }
  }
}

#define FL_E4_DISPATCH(e4, D, KERNEL, GRID, BLOCK, ST, ...)                           \
  switch (e4) {                                                                        \
    case 6: KERNEL<D, 6><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                  \
    case 8: KERNEL<D, 8><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                  \
    case 10: KERNEL<D, 10><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                \
    case 12: KERNEL<D, 12><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                \
    case 14: KERNEL<D, 14><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                \
    default: KERNEL<D, 0><<<GRID, BLOCK, 0, ST>>>(__VA_ARGS__), ::fl::note_launch(); break;                 \
  }

void launch_singular_touching(const DevMesh& m, const DevTables& t, double ex, int e4,
                              const TouchPair* pairs, int64_t npairs, double* out, cudaStream_t st) {
  if (npairs <= 0) return;
  const int grid = (int)((npairs + 3) / 4);
  if (m.d == 1) { FL_E4_DISPATCH(e4, 1, touching_kernel, grid, 128, st, m, t.data, t, ex, pairs, npairs, out); }
  else { FL_E4_DISPATCH(e4, 2, touching_kernel, grid, 128, st, m, t.data, t, ex, pairs, npairs, out); }
  FL_CHECK_LAUNCH();
}

void launch_singular_identical(const DevMesh& m, const DevTables& t, double ex, int e4,
                               const int* ident_k, double* out, cudaStream_t st) {
  const int grid = (m.nc + 3) / 4;
  if (m.d == 1) { FL_E4_DISPATCH(e4, 1, identical_kernel, grid, 128, st, m, t.data, t, ex, ident_k, out); }
  else { FL_E4_DISPATCH(e4, 2, identical_kernel, grid, 128, st, m, t.data, t, ex, ident_k, out); }
  FL_CHECK_LAUNCH();
}

void launch_singular_boundary(const DevMesh& m, const DevTables& t, double ex, int e4,
                              const BndPair* items, int64_t nitems, double* out, cudaStream_t st) {
  if (nitems <= 0) return;
  const int grid = (int)((nitems + 3) / 4);
  if (m.d == 1) { FL_E4_DISPATCH(e4, 1, boundary_kernel, grid, 128, st, m, t.data, t, ex, items, nitems, out); }
  else { FL_E4_DISPATCH(e4, 2, boundary_kernel, grid, 128, st, m, t.data, t, ex, items, nitems, out); }
  FL_CHECK_LAUNCH();
}

}  // namespace fl
