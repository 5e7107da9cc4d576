// Far field: the kernel tail Psi_K (direct_tail_potential, assembly.py:985-1025), the
// boundary flux of the non-touching edges at cell nodes (edge_flux_potential :303-333 with
// W_in = touch_T - V, :1082-1094) and the disjoint cross term (cross_matrices :172-229,
// scattered by _cross_triplets :693-725) written straight into dense DoF tiles.
//
// Tail:  one warp per target cell K.  Lanes own target nodes x_q (16 in 2D, 6 in 1D); the
//        32 sources of a chunk get their order k (select_order with C_offset-4) in parallel,
//        their k^d mapped nodes are staged in shared memory and the half-warps (2D) / lane
//        groups (1D) sweep that node list: uniform work, no divergence on k.
// Cross: one CTA per (row tile, column tile) of 64 DoFs.  Cells touching the row tile are
//        processed colour class by colour class (vertex-disjoint => their rows are disjoint);
//        a warp owns one row cell, lanes own column cells, and the column-cell updates are
//        applied colour by colour inside the warp.  Every A entry therefore receives its <=36
//        contributions in the fixed (row colour, column colour) order: deterministic and free
//        of atomics; the tile is written to HBM once (and mirrored when symmetric).
#include "fl_internal.h"

namespace fl {

// ====================================================================== tail Psi_K
constexpr int TAIL_WARPS = 4;
constexpr int TAIL_WIN = 256;

template <int D, int E4>
__global__ void __launch_bounds__(TAIL_WARPS * 32) tail_kernel(DevMesh m, const double* __restrict__ tab,
                                                               DevTables dir, OrderConsts oc, double ex,
                                                               const int* __restrict__ targets, int ntargets,
                                                               double* __restrict__ psi,
                                                               unsigned long long* __restrict__ evals) {
  constexpr int Q = (D == 1) ? 6 : 16;
  constexpr int G = 32 / Q;
  __shared__ double2 s_y[TAIL_WARPS][TAIL_WIN];
  __shared__ double s_jw[TAIL_WARPS][TAIL_WIN];
  __shared__ double s_src[TAIL_WARPS][32][8];   // P0 (2), E (4), J, pad
  __shared__ int s_off[TAIL_WARPS][33];
  __shared__ int s_k[TAIL_WARPS][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ti = blockIdx.x * TAIL_WARPS + w;
  if (ti >= ntargets) return;
  const int K = targets[ti];
  const CellGeo A = m.geo[K];
  const int q = lane % Q, g = lane / Q;
  const bool active = lane < G * Q;
  double xq0 = 0.0, xq1 = 0.0;
  if (active) {
    xq0 = m.X[((size_t)K * Q + q) * D + 0];
    if (D == 2) xq1 = m.X[((size_t)K * Q + q) * D + 1];
  }
  double acc = 0.0;
  unsigned long long nodes = 0;
  for (int s0 = 0; s0 < m.nc; s0 += 32) {
    const int src = s0 + lane;
    int k = 0, nn = 0;
    if (src < m.nc && src != K) {
      const CellGeo B = m.geo[src];
      if (!touching<D>(A, B)) {
        const double dist = dist_estimate<D>(A, B);            // (target, source) orientation
        k = order_disjoint(oc, oc.coff_tail, A, B, dist);      // boosted orders (:997)
        nn = (D == 1) ? k : k * k;
        double* sg = s_src[w][lane];
        sg[0] = B.p[0][0];
        sg[1] = B.p[0][1];
        sg[2] = B.p[1][0] - B.p[0][0];
        sg[3] = B.p[1][1] - B.p[0][1];
        sg[4] = B.p[2][0] - B.p[0][0];
        sg[5] = B.p[2][1] - B.p[0][1];
        sg[6] = B.J;
      }
    }
    // warp exclusive scan of node counts
    int incl = nn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    s_off[w][lane] = incl - nn;
    s_k[w][lane] = k;
    if (lane == 31) s_off[w][32] = total;
    nodes += (unsigned long long)total;
    __syncwarp();
    for (int base = 0; base < total; base += TAIL_WIN) {
      const int cnt = min(TAIL_WIN, total - base);
      for (int idx = lane; idx < cnt; idx += 32) {
        const int gi = base + idx;
        int lo = 0;                                            // owner: last j with off[j] <= gi
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (lo + step < 32 && s_off[w][lo + step] <= gi) lo += step;
        while (s_k[w][lo] == 0 || s_off[w][lo + 1] <= gi) ++lo;   // skip empty sources
        const int r = gi - s_off[w][lo];
        const RuleRef rr = dir.rule(T_DISJ, s_k[w][lo]);
        const double* nd = tab + (size_t)(rr.off + r) * NODE;
        const double* sg = s_src[w][lo];
        double y0, y1 = 0.0;
        if (D == 1) {
          y0 = sg[0] + nd[0] * sg[2];
        } else {
          y0 = sg[0] + (nd[0] * sg[2] + nd[1] * sg[4]);
          y1 = sg[1] + (nd[0] * sg[3] + nd[1] * sg[5]);
        }
        s_y[w][idx] = make_double2(y0, y1);
        s_jw[w][idx] = sg[6] * nd[2];
      }
      __syncwarp();
      if (active) {
        for (int p = g; p < cnt; p += G) {
          const double2 y = s_y[w][p];
          const double d0 = xq0 - y.x;
          double r2;
          if (D == 1) {
            r2 = d0 * d0;
          } else {
            const double d1 = xq1 - y.y;
            r2 = fma(d1, d1, d0 * d0);
          }
          acc = fma(s_jw[w][p], kpow<E4>(r2, ex), acc);
        }
      }
      __syncwarp();
    }
  }
  // combine the G groups of each target node in a fixed order
  double tot = acc;
#pragma unroll
  for (int gg = 1; gg < G; ++gg) tot += __shfl_sync(0xffffffffu, acc, (lane + gg * Q) & 31);
  if (lane < Q) psi[(size_t)K * Q + q] = tot;
  if (lane == 0 && evals) atomicAdd(evals, nodes * Q);
}

// ====================================================================== boundary flux
// W_in(x) = -(sum over boundary edges NOT touching K of the GL8 outward flux) (:1092)
template <int D, int E4>
__global__ void __launch_bounds__(128) flux_kernel(DevMesh m, const double* __restrict__ tab, RuleRef gl,
                                                   double ex, const int* __restrict__ targets, int ntargets,
                                                   double* __restrict__ win) {
  constexpr int Q = (D == 1) ? 6 : 16;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntargets * Q) return;
  const int K = targets[i / Q], q = i % Q;
  const CellGeo A = m.geo[K];
  const double x0 = m.X[((size_t)K * Q + q) * D + 0];
  const double x1 = (D == 2) ? m.X[((size_t)K * Q + q) * D + 1] : 0.0;
  double acc = 0.0;
  for (int e = 0; e < m.nb; ++e) {
    const int v0 = m.bedges[e * D], v1 = (D == 2) ? m.bedges[e * D + 1] : v0;
    bool t = false;
#pragma unroll
    for (int j = 0; j <= D; ++j) t |= (A.v[j] == v0) | (A.v[j] == v1);
    if (t) continue;
    if constexpr (D == 1) {
      const double diff = x0 - m.vert[v0];
      const double nd = diff * m.bnorm[e];
      acc += nd * kpow<E4>(diff * diff, ex);
    } else {
      const double p0x = m.vert[2 * v0], p0y = m.vert[2 * v0 + 1];
      const double ux = m.vert[2 * v1] - p0x, uy = m.vert[2 * v1 + 1] - p0y;
      const double L = norm2d(ux, uy);
      const double n0 = m.bnorm[2 * e], n1 = m.bnorm[2 * e + 1];
      double s = 0.0;
      for (int gq = 0; gq < gl.cnt; ++gq) {
        const double* nd = tab + (size_t)(gl.off + gq) * NODE;
        const double yx = p0x + nd[0] * ux, yy = p0y + nd[0] * uy;
        const double dx = x0 - yx, dy = x1 - yy;
        const double r2 = fma(dy, dy, dx * dx);
        const double ndot = fma(dy, n1, dx * n0);
        s = fma(nd[1], ndot * kpow<E4>(r2, ex), s);
      }
      acc = fma(s, L, acc);
    }
  }
  win[(size_t)K * Q + q] = -acc;
}

// ====================================================================== cross tiles
constexpr int XW = 4;   // warps per cross CTA

struct TileView {
  const int* dofs; const int* ncell; const int* cells; const int* slots; const int* cstart;
};

template <int D, int E4>
__device__ __forceinline__ void cross_block(const double* __restrict__ tab, RuleRef rr, const CellGeo& K,
                                            const CellGeo& L, double ex, double (&Gm)[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Gm[a][b] = 0.0;
  const double ke00 = K.p[1][0] - K.p[0][0], ke01 = K.p[1][1] - K.p[0][1];
  const double ke10 = K.p[2][0] - K.p[0][0], ke11 = K.p[2][1] - K.p[0][1];
  const double le00 = L.p[1][0] - L.p[0][0], le01 = L.p[1][1] - L.p[0][1];
  const double le10 = L.p[2][0] - L.p[0][0], le11 = L.p[2][1] - L.p[0][1];
  for (int x = 0; x < rr.cnt; ++x) {
    const double* nx = tab + (size_t)(rr.off + x) * NODE;
    double X0, X1 = 0.0;
    if (D == 1) {
      X0 = K.p[0][0] + nx[0] * ke00;
    } else {
      X0 = K.p[0][0] + (nx[0] * ke00 + nx[1] * ke10);
      X1 = K.p[0][1] + (nx[0] * ke01 + nx[1] * ke11);
    }
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int y = 0; y < rr.cnt; ++y) {
      const double* ny = tab + (size_t)(rr.off + y) * NODE;
      double r2;
      if (D == 1) {
        const double Y0 = L.p[0][0] + ny[0] * le00;
        const double d0 = X0 - Y0;
        r2 = d0 * d0;
      } else {
        const double Y0 = L.p[0][0] + (ny[0] * le00 + ny[1] * le10);
        const double Y1 = L.p[0][1] + (ny[0] * le01 + ny[1] * le11);
        const double d0 = X0 - Y0, d1 = X1 - Y1;
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
      t0 = fma(v, ny[3], t0);
      t1 = fma(v, ny[4], t1);
      if (D == 2) t2 = fma(v, ny[5], t2);
    }
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      const double lx = nx[3 + a];
      Gm[a][0] = fma(lx, t0, Gm[a][0]);
      Gm[a][1] = fma(lx, t1, Gm[a][1]);
      if (D == 2) Gm[a][2] = fma(lx, t2, Gm[a][2]);
    }
  }
  const double JJ = K.J * L.J;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Gm[a][b] *= JJ;
}

template <int D, int E4>
__global__ void __launch_bounds__(XW * 32) cross_tile_kernel(DevMesh m, const double* __restrict__ tab,
                                                             DevTables dir, OrderConsts oc, double ex,
                                                             double negC, TileView R, TileView Cv,
                                                             const int2* __restrict__ tpairs, int ncolors,
                                                             int symmetric, int row_begin, int row_end,
                                                             double* __restrict__ Aout, int64_t lda,
                                                             unsigned long long* __restrict__ evals) {
  unsigned long long my_evals = 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double (*At)[TILE + 1] = reinterpret_cast<double (*)[TILE + 1]>(smem_raw);
  CellGeo* sR = reinterpret_cast<CellGeo*>(smem_raw + sizeof(double) * TILE * (TILE + 1));
  CellGeo* sC = sR + TILE_MAXC;
  int* sRs = reinterpret_cast<int*>(sC + TILE_MAXC);      // TILE_MAXC*3
  int* sCs = sRs + TILE_MAXC * 3;
  int* sRd = sCs + TILE_MAXC * 3;                           // TILE dofs
  int* sCd = sRd + TILE;
  const int2 tp = tpairs[blockIdx.x];
  const int tr = tp.x, tc = tp.y;
  const int nR = R.ncell[tr], nC = Cv.ncell[tc];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < nR; i += blockDim.x) {
    sR[i] = m.geo[R.cells[tr * TILE_MAXC + i]];
    for (int a = 0; a < 3; ++a) sRs[i * 3 + a] = R.slots[(tr * TILE_MAXC + i) * 3 + a];
  }
  for (int i = tid; i < nC; i += blockDim.x) {
    sC[i] = m.geo[Cv.cells[tc * TILE_MAXC + i]];
    for (int a = 0; a < 3; ++a) sCs[i * 3 + a] = Cv.slots[(tc * TILE_MAXC + i) * 3 + a];
  }
  for (int i = tid; i < TILE; i += blockDim.x) {
    sRd[i] = R.dofs[tr * TILE + i];
    sCd[i] = Cv.dofs[tc * TILE + i];
  }
  for (int i = tid; i < TILE * (TILE + 1); i += blockDim.x) (&At[0][0])[i] = 0.0;
  __syncthreads();

  for (int cr = 0; cr < ncolors; ++cr) {
    const int a0 = R.cstart[tr * (MAXCOLORS + 1) + cr], a1 = R.cstart[tr * (MAXCOLORS + 1) + cr + 1];
    for (int ri = a0 + wid; ri < a1; ri += XW) {
      const CellGeo& K = sR[ri];
      const int lr0 = sRs[ri * 3 + 0], lr1 = sRs[ri * 3 + 1], lr2 = sRs[ri * 3 + 2];
      for (int cj0 = 0; cj0 < nC; cj0 += 32) {
        const int cj = cj0 + lane;
        double Gm[3][3];
        bool have = false;
        int mycol = MAXCOLORS;
        if (cj < nC) {
          const CellGeo& L = sC[cj];
          mycol = L.color;
          if (!touching<D>(K, L)) {
            // reference orientation of the order: (min id, max id) (assembly.py:973-982, :705)
            const int idK = R.cells[tr * TILE_MAXC + ri], idL = Cv.cells[tc * TILE_MAXC + cj];
            const CellGeo& P = (idK < idL) ? K : L;
            const CellGeo& Qc = (idK < idL) ? L : K;
            const double dist = dist_estimate<D>(P, Qc);
            const int k = order_disjoint(oc, oc.coff, P, Qc, dist);
            cross_block<D, E4>(tab, dir.rule(T_DISJ, k), K, L, ex, Gm);
            my_evals += (D == 1) ? (unsigned long long)(k * k) : (unsigned long long)(k * k * k * k);
            have = true;
          }
        }
        // apply column colour classes one after another (vertex-disjoint within a class)
        unsigned pending = __ballot_sync(0xffffffffu, have);
        while (pending) {
          const int cmin = __reduce_min_sync(0xffffffffu, have ? mycol : MAXCOLORS);
          const bool mine = have && mycol == cmin;
          if (mine) {
            const int lc0 = sCs[cj * 3 + 0], lc1 = sCs[cj * 3 + 1], lc2 = sCs[cj * 3 + 2];
            const int lr[3] = {lr0, lr1, lr2}, lc[3] = {lc0, lc1, lc2};
#pragma unroll
            for (int a = 0; a <= D; ++a) {
              if (lr[a] < 0) continue;
#pragma unroll
              for (int b = 0; b <= D; ++b)
                if (lc[b] >= 0) At[lr[a]][lc[b]] += negC * Gm[a][b];
            }
            have = false;
          }
          __syncwarp();
          pending = __ballot_sync(0xffffffffu, have);
        }
      }
    }
    __syncthreads();
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_evals += __shfl_xor_sync(0xffffffffu, my_evals, o);
    if (lane == 0) atomicAdd(evals, my_evals);
  }
  // write the tile (and its mirror) once
  for (int idx = tid; idx < TILE * TILE; idx += blockDim.x) {
    const int r = idx / TILE, c = idx % TILE;
    const int i = sRd[r], j = sCd[c];
    if (i >= row_begin && i < row_end && j >= 0) Aout[(int64_t)(i - row_begin) * lda + j] = At[r][c];
  }
  if (symmetric && tr != tc) {
    for (int idx = tid; idx < TILE * TILE; idx += blockDim.x) {
      const int c = idx / TILE, r = idx % TILE;
      const int i = sRd[r], j = sCd[c];
      if (i >= 0 && j >= row_begin && j < row_end) Aout[(int64_t)(j - row_begin) * lda + i] = At[r][c];
    }
  }
}

size_t cross_smem_bytes() {
  return sizeof(double) * TILE * (TILE + 1) + sizeof(CellGeo) * 2 * TILE_MAXC + sizeof(int) * TILE_MAXC * 6 +
         sizeof(int) * TILE * 2;
}

// ====================================================================== debug: orders
template <int D>
__global__ void orders_kernel(DevMesh m, OrderConsts oc, int8_t* cross_k, int8_t* tail_k) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)m.nc * m.nc) return;
  const int a = (int)(idx / m.nc), b = (int)(idx % m.nc);
  int8_t kc = 0, kt = 0;
  if (a != b) {
    const CellGeo A = m.geo[a], B = m.geo[b];
    if (!touching<D>(A, B)) {
      const double dt = dist_estimate<D>(A, B);
      kt = (int8_t)order_disjoint(oc, oc.coff_tail, A, B, dt);
      if (a < b) kc = (int8_t)order_disjoint(oc, oc.coff, A, B, dt);
    }
  }
  cross_k[idx] = kc;
  tail_k[idx] = kt;
}

// ====================================================================== launchers
#define FL_E4_SWITCH(e4, ...)                                 \
  switch (e4) {                                               \
    case 6: { constexpr int E4 = 6; __VA_ARGS__; } break;     \
    case 8: { constexpr int E4 = 8; __VA_ARGS__; } break;     \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

void launch_tail(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                 const int* targets, int ntargets, double* psi, unsigned long long* evals, cudaStream_t st) {
  if (ntargets <= 0) return;
  const int grid = (ntargets + TAIL_WARPS - 1) / TAIL_WARPS;
  if (m.d == 1) {
    FL_E4_SWITCH(e4, (tail_kernel<1, E4><<<grid, TAIL_WARPS * 32, 0, st>>>(m, t.data, t, oc, ex, targets, ntargets, psi, evals), ::fl::note_launch()));
  } else {
    FL_E4_SWITCH(e4, (tail_kernel<2, E4><<<grid, TAIL_WARPS * 32, 0, st>>>(m, t.data, t, oc, ex, targets, ntargets, psi, evals), ::fl::note_launch()));
  }
  FL_CHECK_LAUNCH();
}

void launch_flux(const DevMesh& m, const DevTables& t, double ex, int e4, const int* targets, int ntargets,
                 double* win, cudaStream_t st) {
  if (ntargets <= 0) return;
  const int Q = m.q, tot = ntargets * Q, grid = (tot + 127) / 128;
  const RuleRef gl = t.rule(T_EGL, 0);
  if (m.d == 1) {
    FL_E4_SWITCH(e4, (flux_kernel<1, E4><<<grid, 128, 0, st>>>(m, t.data, gl, ex, targets, ntargets, win), ::fl::note_launch()));
  } else {
    FL_E4_SWITCH(e4, (flux_kernel<2, E4><<<grid, 128, 0, st>>>(m, t.data, gl, ex, targets, ntargets, win), ::fl::note_launch()));
  }
  FL_CHECK_LAUNCH();
}

void launch_cross_tiles(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                        double Cds, const Tiles& rows, const Tiles& cols, bool symmetric, int row_begin,
                        int row_end, double* A, int64_t lda, int ncolors, int64_t& ntilepairs,
                        unsigned long long* evals, cudaStream_t st) {
  std::vector<int2> hp;
  for (int r = 0; r < rows.ntiles; ++r)
    for (int c = symmetric ? r : 0; c < cols.ntiles; ++c) hp.push_back(make_int2(r, c));
  ntilepairs = (int64_t)hp.size();
  if (hp.empty()) return;
  DBuf<int2> dp(hp.size());
  FL_CUDA(cudaMemcpyAsync(dp.p, hp.data(), hp.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  TileView R{rows.dofs.p, rows.ncell.p, rows.cells.p, rows.slots.p, rows.cstart.p};
  TileView C{cols.dofs.p, cols.ncell.p, cols.cells.p, cols.slots.p, cols.cstart.p};
  const size_t smem = cross_smem_bytes();
  const double negC = -Cds;   // (C/2) * (-2)  (assembly.py:723, :1100)
  const int64_t np_ = (int64_t)hp.size();
  for (int64_t base = 0; base < np_; base += 2147483647LL) {
    const int grid = (int)std::min<int64_t>(np_ - base, 2147483647LL);
    if (m.d == 1) {
      FL_E4_SWITCH(e4, {
        FL_CUDA(cudaFuncSetAttribute(cross_tile_kernel<1, E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cross_tile_kernel<1, E4><<<grid, XW * 32, smem, st>>>(m, t.data, t, oc, ex, negC, R, C, dp.p + base, ncolors,
                                                            symmetric ? 1 : 0, row_begin, row_end, A, lda, evals), ::fl::note_launch();
      });
    } else {
      FL_E4_SWITCH(e4, {
        FL_CUDA(cudaFuncSetAttribute(cross_tile_kernel<2, E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cross_tile_kernel<2, E4><<<grid, XW * 32, smem, st>>>(m, t.data, t, oc, ex, negC, R, C, dp.p + base, ncolors,
                                                            symmetric ? 1 : 0, row_begin, row_end, A, lda, evals), ::fl::note_launch();
      });
    }
    FL_CHECK_LAUNCH();
  }
  FL_CUDA(cudaStreamSynchronize(st));   // dp is freed on return
}

// Exact per-order histograms of the disjoint pairs: cross (unordered, normal orders) and
// tail (ordered, C_offset-4); integer atomics => exact totals at any mesh size.
template <int D>
__global__ void order_hist_kernel(DevMesh m, OrderConsts oc, unsigned long long* hc, unsigned long long* ht) {
  __shared__ unsigned long long sc[KDIR], stl[KDIR];
  for (int i = threadIdx.x; i < KDIR; i += blockDim.x) { sc[i] = 0; stl[i] = 0; }
  __syncthreads();
  const int a = blockIdx.x;
  const CellGeo A = m.geo[a];
  for (int b = threadIdx.x; b < m.nc; b += blockDim.x) {
    if (b == a) continue;
    const CellGeo B = m.geo[b];
    if (touching<D>(A, B)) continue;
    const double dt = dist_estimate<D>(A, B);
    atomicAdd(&stl[order_disjoint(oc, oc.coff_tail, A, B, dt)], 1ull);
    if (a < b) atomicAdd(&sc[order_disjoint(oc, oc.coff, A, B, dt)], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < KDIR; i += blockDim.x) {
    if (sc[i]) atomicAdd(&hc[i], sc[i]);
    if (stl[i]) atomicAdd(&ht[i], stl[i]);
  }
}

void launch_order_hist(const DevMesh& m, const OrderConsts& oc, unsigned long long* hc, unsigned long long* ht,
                       cudaStream_t st) {
  if (m.d == 1) order_hist_kernel<1><<<m.nc, 256, 0, st>>>(m, oc, hc, ht), ::fl::note_launch();
  else order_hist_kernel<2><<<m.nc, 256, 0, st>>>(m, oc, hc, ht), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// FP64 peak probe: 8 independent DFMA chains per thread, 148*8 CTAs of 256 threads.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

double probe_fp64_tflops(cudaStream_t st) {
  DBuf<double> out(1);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * 8, iters = 4096;
  dfma_probe_kernel<<<grid, 256, 0, st>>>(out.p, 64, 0.999999, 1e-7), ::fl::note_launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    dfma_probe_kernel<<<grid, 256, 0, st>>>(out.p, iters, 0.999999, 1e-7), ::fl::note_launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  FL_CHECK_LAUNCH();
  const double flops = 2.0 * 8.0 * iters * 256.0 * grid;
  return flops / (best * 1e-3) / 1e12;
}

void launch_debug_orders(const DevMesh& m, const OrderConsts& oc, int8_t* cross_k, int8_t* tail_k,
                         cudaStream_t st) {
  const int64_t tot = (int64_t)m.nc * m.nc;
  const int grid = (int)((tot + 255) / 256);
  if (m.d == 1) orders_kernel<1><<<grid, 256, 0, st>>>(m, oc, cross_k, tail_k), ::fl::note_launch();
  else orders_kernel<2><<<grid, 256, 0, st>>>(m, oc, cross_k, tail_k), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

}  // namespace fl
