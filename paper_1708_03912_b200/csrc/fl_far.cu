// Far field: the kernel tail Psi_K (direct_tail_potential, assembly.py:985-1025), the
// boundary flux of the non-touching edges at cell nodes (edge_flux_potential :303-333 with
// W_in = touch_T - V, :1082-1094) and the disjoint cross term (cross_matrices :172-229,
// scattered by _cross_triplets :693-725) written straight into dense DoF tiles.
//
// Tail:  one warp per target cell K.  Lanes own target nodes x_q (16 in 2D, 6 in 1D); the
//        32 sources of a chunk get their order k (select_order with C_offset-4) in parallel,
//        their k^d mapped nodes are staged in shared memory (padded to the unroll width) and
//        the half-warps (2D) / lane groups (1D) sweep that node list 4 nodes at a time:
//        uniform work, no divergence on k, independent evaluations in flight.
// Cross: one CTA per (row tile, column tile) of 64 DoFs.  The cells touching the two tiles
//        are taken 16 x 32 at a time: (A) every pair gets its order k, (B) the pairs are
//        sorted by k and their 3x3 blocks M^{K,K~} computed into shared memory — a whole
//        warp per pair for large k (lanes over the x nodes), one thread per pair otherwise —
//        (C) each tile row is owned by 4 threads (disjoint column classes) that add the
//        blocks of its cells in a fixed order.  No atomics on values: every A entry receives
//        its contributions in the same order on every run; the tile is written to HBM once
//        (and mirrored when the assembly is symmetric).
#include "fl_internal.h"

namespace fl {

// ====================================================================== tail Psi_K
constexpr int TAIL_WARPS = 4;
constexpr int TAIL_WIN = 256;
#ifndef FL_TAIL_U
#define FL_TAIL_U 4
#endif
#ifndef FL_TAIL_MINB
#define FL_TAIL_MINB 5
#endif
constexpr int TAIL_U = FL_TAIL_U;   // source nodes per lane per step
constexpr int TAIL_T = 2;           // target nodes per lane

// Block-ordered, node-major staging arrays of the mapped disjoint-rule nodes (node r of slot c of
// block Q at [r * 32 + c] of the order's segment): orders 2-4 in Blocks2D::un (shared with the cross
// term), orders 5-9 in the tail's own array uhi (fl_tail2d.cu, hi_nodes_kernel)
__device__ __forceinline__ const double2* staged_nodes(const double2* __restrict__ un, const double2* __restrict__ uhi,
                                                       int Q, int k) {
  return k <= 4 ? un + (size_t)Q * UNODES2D + (k == 2 ? 0 : (k == 3 ? 128 : 416))
                : uhi + (size_t)Q * UHI2D + uhi_seg(k);
}

// FOLD (2D, behind the block kernel): the source weight J w is folded into the staged coordinates —
// s_jw = sc = (J w)^(1/(2 ex)) (cell factor ujh per block slot, rule factor wh per node), s_y =
// -sc (y - c_K) with c_K the target cell's centroid, targets held as x - c_K — so that
// d' = fma(x', sc, s_y) = sc (x - y), r2' = |d'|^2 = (J w)^(1/ex) r2 and (J w) r2^ex = r2'^ex is added
// by kpow_acc: 10 FP64 instructions per evaluation instead of 11.  Centring on the target cell keeps
// the cancellation factor |y - c_K| / |x - y| of a non-touching pair to a few units.
template <int D, int E4, bool FOLD>
__global__ void __launch_bounds__(TAIL_WARPS * 32, FL_TAIL_MINB) tail_kernel(DevMesh m, const double* __restrict__ tab,
                                                                  DevTables dir, OrderConsts oc, double ex,
                                                                  const int* __restrict__ targets, int ntargets,
                                                                  double* __restrict__ psi,
                                                                  unsigned long long* __restrict__ evals,
                                                                  const int8_t* __restrict__ kuni,
                                                                  const int* __restrict__ blk_of,
                                                                  const int* __restrict__ bcells, int nb,
                                                                  const int8_t* __restrict__ kcell,
                                                                  const unsigned long long* __restrict__ psifx,
                                                                  double fxinv,
                                                                  const double* __restrict__ ujh,
                                                                  const double* __restrict__ wh,
                                                                  const double2* __restrict__ un,
                                                                  const double2* __restrict__ uhi) {
  constexpr int Q = (D == 1) ? 6 : 16;     // cell quadrature nodes (XQ_ORDER)
  constexpr int L = Q / TAIL_T;            // lanes per group (8 in 2D, 3 in 1D)
  constexpr int G = 32 / L;                // groups sweeping disjoint source nodes (4 / 10)
  constexpr int STEP = TAIL_U * G;
  constexpr int PADW = TAIL_WIN + STEP;
  __shared__ double2 s_y[TAIL_WARPS][PADW];
  __shared__ double s_jw[TAIL_WARPS][PADW];
  __shared__ double s_src[TAIL_WARPS][7][32];    // SoA: P0x P0y E00 E01 E10 E11 J of the chunk
  __shared__ CellGeo s_tgt[TAIL_WARPS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ti = blockIdx.x * TAIL_WARPS + w;
  if (ti >= ntargets) return;
  const int K = targets[ti];
  if (lane < (int)(sizeof(CellGeo) / 8))
    reinterpret_cast<double*>(&s_tgt[w])[lane] = reinterpret_cast<const double*>(&m.geo[K])[lane];
  __syncwarp();
  const CellGeo& A = s_tgt[w];
  const int j = lane % L, g = lane / L;
  const bool active = lane < G * L;
  double x0[TAIL_T], x1[TAIL_T];
#pragma unroll
  for (int t = 0; t < TAIL_T; ++t) {
    const int q = j + t * L;
    x0[t] = active ? m.X[((size_t)K * Q + q) * D + 0] : 0.0;
    x1[t] = (active && D == 2) ? m.X[((size_t)K * Q + q) * D + 1] : 0.0;
    if (FOLD) {
      x0[t] -= A.cx;
      x1[t] -= A.cy;
    }
  }
  double acc[TAIL_T][2] = {};
  unsigned long long nodes = 0;
  // sources: every cell in chunks of 32, or (kuni) only the Morton source blocks of K's block
  // whose orders the block bounds did not fix (kuni == 0; the others were evaluated by
  // tail2d_block_kernel, whose psi this kernel then adds to)
  const int8_t* krow = kuni ? kuni + (size_t)blk_of[K] * nb : nullptr;
  const int nchunk = kuni ? nb : (m.nc + 31) / 32;
  unsigned pend = 0;
  int cbase = -32;
  for (;;) {
    int ci;
    if (kuni) {
      while (!pend) {
        cbase += 32;
        if (cbase >= nchunk) break;
        const int kq = cbase + lane < nchunk ? (int)krow[cbase + lane] : 1;
        // 0: the whole source block is ours; -1: ours unless K alone has one order for it
        // (then tail2d_block_kernel took it, by the same bitwise decision)
        const bool mine = kq == 0 || (kq < 0 && kcell[(size_t)K * nb + cbase + lane] == 0);
        pend = __ballot_sync(0xffffffffu, mine);
      }
      if (!pend) break;
      ci = cbase + __ffs(pend) - 1;
      pend &= pend - 1;
    } else {
      cbase += 32;
      if (cbase >= m.nc) break;
      ci = cbase >> 5;
    }
    const int src = kuni ? bcells[ci * 32 + lane] : ci * 32 + lane;
    int k = 0, nn = 0;
    if (src >= 0 && src < m.nc && src != K) {
      const CellGeo& B = m.geo[src];
      if (!touching<D>(A, B)) {
        const double dist = dist_estimate<D>(A, B);            // (target, source) orientation
        k = order_disjoint_fast(oc, oc.coff_tail, A, B, dist);      // boosted orders (:997)
        nn = (D == 1) ? k : k * k;
        s_src[w][0][lane] = B.p[0][0];
        s_src[w][1][lane] = B.p[0][1];
        s_src[w][2][lane] = B.p[1][0] - B.p[0][0];
        s_src[w][3][lane] = B.p[1][1] - B.p[0][1];
        s_src[w][4][lane] = B.p[2][0] - B.p[0][0];
        s_src[w][5][lane] = B.p[2][1] - B.p[0][1];
        s_src[w][6][lane] = FOLD ? ujh[ci * 32 + lane] : B.J;
      }
    }
    // the warp's evaluation of one staged window: G groups of L lanes sweep disjoint nodes
    auto eval_window = [&](int cntp) {
      if (!active) return;
#pragma unroll 1
      for (int p = g; p < cntp; p += STEP) {
        double2 y[TAIL_U];
        double jw[TAIL_U];
#pragma unroll
        for (int u = 0; u < TAIL_U; ++u) {
          y[u] = s_y[w][p + u * G];
          jw[u] = s_jw[w][p + u * G];
        }
#pragma unroll
        for (int t = 0; t < TAIL_T; ++t) {
#pragma unroll
          for (int u = 0; u < TAIL_U; ++u) {
            if (FOLD) {
              const double e0 = fma(x0[t], jw[u], y[u].x), e1 = fma(x1[t], jw[u], y[u].y);
              acc[t][u & 1] = kpow_acc<E4>(fma(e1, e1, e0 * e0), ex, acc[t][u & 1]);
              continue;
            }
            const double d0 = x0[t] - y[u].x;
            double r2;
            if (D == 1) {
              r2 = d0 * d0;
            } else {
              const double d1 = x1[t] - y[u].y;
              r2 = fma(d1, d1, d0 * d0);
            }
            acc[t][u & 1] = fma(jw[u], kpow<E4>(r2, ex), acc[t][u & 1]);
          }
        }
      }
    };
    if (FOLD) {
      // one order for every cell of the source block (and none touching K): the block's mapped
      // nodes lie node-major in the staging arrays, so the lanes copy them coalesced, 8 nodes of
      // every cell per window, each lane its own slot's weight factor
      const bool slot_ok = src >= 0;
      const unsigned act = __ballot_sync(0xffffffffu, nn > 0);
      const int k0 = __shfl_sync(0xffffffffu, k, act ? __ffs(act) - 1 : 0);
      if (act && __all_sync(0xffffffffu, slot_ok ? (nn > 0 && k == k0) : true)) {
        const int kk = k0 * k0;
        const double Jh = slot_ok ? s_src[w][6][lane] : 0.0;
        const double2* __restrict__ ub = staged_nodes(un, uhi, ci, k0) + lane;
        const double* __restrict__ whk = wh + disj_roff(k0);
        nodes += (unsigned long long)__popc(act) * kk;
        __syncwarp();
        for (int rb = 0; rb < kk; rb += TAIL_WIN / 32) {
          const int nr = min(TAIL_WIN / 32, kk - rb);
#pragma unroll 4
          for (int r = 0; r < nr; ++r) {
            const double2 yv = ub[(rb + r) * 32];
            const double sc = Jh * __ldg(whk + rb + r);
            s_y[w][r * 32 + lane] = slot_ok ? make_double2(-sc * (yv.x - A.cx), -sc * (yv.y - A.cy))
                                            : make_double2(1e150, 1e150);
            s_jw[w][r * 32 + lane] = slot_ok ? sc : 1.0;
          }
          __syncwarp();
          eval_window(nr * 32);
          __syncwarp();
        }
        continue;
      }
      // mixed orders (or touching cells in the block): rounds of up to 8 nodes per cell, the
      // nodes of a round packed node-major (ballot ranks), so every lane stages in every round
      // and a window never exceeds 256 nodes
      const int nmax = __reduce_max_sync(0xffffffffu, nn);
      const double Jh = nn > 0 ? s_src[w][6][lane] : 0.0;
      const int ks = nn > 0 ? k : 2;
      const double2* __restrict__ ub = staged_nodes(un, uhi, ci, ks) + lane;
      const double* __restrict__ whk = wh + disj_roff(ks);
      const unsigned lt = (1u << lane) - 1u;
      __syncwarp();
      for (int rb = 0; rb < nmax; rb += TAIL_WIN / 32) {
        const int c = min(TAIL_WIN / 32, nn - rb), cm = min(TAIL_WIN / 32, nmax - rb);
        int tot = 0;
#pragma unroll 4
        for (int r = 0; r < cm; ++r) {
          const bool on = r < c;
          const unsigned bal = __ballot_sync(0xffffffffu, on);
          if (on) {
            const double2 yv = ub[(rb + r) * 32];
            const double sc = Jh * __ldg(whk + rb + r);
            const int pos = tot + __popc(bal & lt);
            s_y[w][pos] = make_double2(-sc * (yv.x - A.cx), -sc * (yv.y - A.cy));
            s_jw[w][pos] = sc;
          }
          tot += __popc(bal);
        }
        nodes += (unsigned long long)tot;
        const int cntp = (tot + STEP - 1) / STEP * STEP;
        for (int idx = tot + lane; idx < cntp; idx += 32) {      // padding: far away, sc = 1
          s_y[w][idx] = make_double2(1e150, 1e150);
          s_jw[w][idx] = 1.0;
        }
        __syncwarp();
        eval_window(cntp);
        __syncwarp();
      }
      continue;
    }
    int incl = nn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    nodes += (unsigned long long)total;
    __syncwarp();
    for (int base = 0; base < total; base += TAIL_WIN) {
      const int cnt = min(TAIL_WIN, total - base);
      const int cntp = (cnt + STEP - 1) / STEP * STEP;
      // every lane maps its own source's nodes that fall into this window
      if (nn > 0) {
        const int my0 = incl - nn - base;
        const int r0 = max(0, -my0), r1 = min(nn, cnt - my0);
        if (r0 < r1) {
          const RuleRef rr = dir.rule(T_DISJ, k);
          const double p0x = s_src[w][0][lane], p0y = s_src[w][1][lane];
          const double e00 = s_src[w][2][lane], e01 = s_src[w][3][lane];
          const double e10 = s_src[w][4][lane], e11 = s_src[w][5][lane], J = s_src[w][6][lane];
          {
            for (int r = r0; r < r1; ++r) {
              const double* nd = tab + (size_t)(rr.off + r) * NODE;
              double y0, y1 = 0.0;
              if (D == 1) {
                y0 = p0x + nd[0] * e00;
              } else {
                y0 = p0x + (nd[0] * e00 + nd[1] * e10);
                y1 = p0y + (nd[0] * e01 + nd[1] * e11);
              }
              s_y[w][my0 + r] = make_double2(y0, y1);
              s_jw[w][my0 + r] = J * nd[2];
            }
          }
        }
      }
      for (int idx = cnt + lane; idx < cntp; idx += 32) {      // padding: far away, zero weight
        s_y[w][idx] = FOLD ? make_double2(1e150, 1e150) : make_double2(1e100, 1e100);   // folded: sc = 1
        s_jw[w][idx] = FOLD ? 1.0 : 0.0;
      }
      __syncwarp();
      eval_window(cntp);
      __syncwarp();
    }
  }
  // combine the two accumulators and the G groups of each target node in a fixed order
#pragma unroll
  for (int t = 0; t < TAIL_T; ++t) {
    const double a = acc[t][0] + acc[t][1];
    double tot = a;
#pragma unroll
    for (int gg = 1; gg < G; ++gg) tot += __shfl_sync(0xffffffffu, a, (lane + gg * L) & 31);
    // kuni: the block kernel's sums (double part, then the sym4 fixed-point part) plus ours
    if (lane < L)
      psi[(size_t)K * Q + j + t * L] =
          kuni ? (psi[(size_t)K * Q + j + t * L] + (psifx ? (double)(long long)psifx[(size_t)K * Q + j + t * L] * fxinv : 0.0)) + tot
               : tot;
  }
  if (lane == 0 && evals) atomicAdd(evals, nodes * Q);
}

// ====================================================================== cross tiles
#ifndef FL_PERSISTENT
#define FL_PERSISTENT 1
#endif
constexpr int XT = 256;                 // threads per cross CTA
constexpr int NEAR_MARK = 255;          // pk of a near pair whose block came from fl_near.cu
constexpr int SBR = 16, SBC = 32, SBP = SBR * SBC;
constexpr int ROWL = MAX_VALENCE;       // max (cell, slot) entries of one tile row
constexpr int KPRE = 3;                 // node coordinates precomputed per sub-block for k <= KPRE
constexpr int NPRE = 4 + 9;             // sum_{k=2}^{KPRE} k^2 (2D; 1D uses the first 5)

struct TileView {
  const int* dofs; const int* ncell; const int* cells; const int* slots;
};

struct CrossShared {
  double At[TILE][TILE + 1];
  double Gs[SBP][9];
  double2 nodes[SBR + SBC][NPRE];       // mapped nodes (k <= KPRE) of the sub-block's row / column cells
  int rowc[TILE_MAXC], colc[TILE_MAXC];
  signed char rslot[TILE_MAXC][3], cslot[TILE_MAXC][3];
  short rowl[TILE][ROWL];
  unsigned char rown[TILE];
  short plist[SBP];
  unsigned char pk[SBP];
  int hist[KDIR + 1], cursor[KDIR + 1];
  int qlarge, qsmall, nlarge, nsmall, tile;
  int rdof[TILE], cdof[TILE];
  int kofs[KDIR];
  // phase-C entry lists: per tile column its (column cell, slot) entries in the current column
  // sub-block; per tile row its rowl range in the current row sub-block; touched rows / columns
  short cent[TILE][ROWL];
  unsigned char ccnt[TILE];
  short rr0[TILE], rr1[TILE];
  unsigned char trow[TILE], tcol[TILE];
  int ntr, ntc;
  // order inputs staged per tile (rows) / per column sub-block (columns): centroid, radius,
  // fp32 ln h and |ln h| (2D fast order path)
  double rcx[TILE_MAXC], rcy[TILE_MAXC], rrad[TILE_MAXC], rJ[TILE_MAXC];
  float rlnh[TILE_MAXC], rlh[TILE_MAXC];
  double ccx[SBC], ccy[SBC], crad[SBC], cJ[SBC];
  float clnh[SBC], clh[SBC];
  // phase-B chunks of far pairs of one order: a warp takes 32 / L pairs, L lanes per pair
  short chs[SBP / 4 + 8];
  unsigned char chn[SBP / 4 + 8], chk[SBP / 4 + 8];
  int nchunk;
  // followed by the packed disjoint rules: per node u0 u1 lw0 lw1 lw2 (5 doubles)
};

template <int D>
__device__ __forceinline__ int pre_off(int k) {   // offset of order k in CrossShared::nodes
  return D == 1 ? (k == 2 ? 0 : k == 3 ? 2 : 5) : (k == 2 ? 0 : k == 3 ? 4 : 13);
}

// fully unrolled block for small fixed k: column-cell nodes and weights held in registers
template <int D, int E4, int KK>
__device__ __forceinline__ void cross_fixed(const double2* __restrict__ Xn, const double2* __restrict__ Yn,
                                            const double* __restrict__ rt, double JJ, double ex,
                                            double* __restrict__ out) {
  constexpr int NN = (D == 1) ? KK : KK * KK;
  double2 y[NN];
  double ly[NN][D + 1];
#pragma unroll
  for (int j = 0; j < NN; ++j) {
    y[j] = Yn[j];
#pragma unroll
    for (int b = 0; b <= D; ++b) ly[j][b] = rt[5 * j + 2 + b];
  }
  double Gm[D + 1][D + 1] = {};
#pragma unroll
  for (int i = 0; i < NN; ++i) {
    const double2 X = Xn[i];
    double t[D + 1] = {};
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      const double d0 = X.x - y[j].x;
      double r2;
      if (D == 1) {
        r2 = d0 * d0;
      } else {
        const double d1 = X.y - y[j].y;
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
#pragma unroll
      for (int b = 0; b <= D; ++b) t[b] = fma(v, ly[j][b], t[b]);
    }
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      const double lx = rt[5 * i + 2 + a];
#pragma unroll
      for (int b = 0; b <= D; ++b) Gm[a][b] = fma(lx, t[b], Gm[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) out[a * 3 + b] = (a <= D && b <= D) ? Gm[a < D + 1 ? a : 0][b < D + 1 ? b : 0] * JJ : 0.0;
}

// on-the-fly mapping (any k); `lanes` = 32 (warp-cooperative over x nodes) or 1 (one thread)
template <int D, int E4>
__device__ __forceinline__ void cross_gen(const double* __restrict__ rt, int nn, const CellGeo& K, const CellGeo& L,
                                          double ex, double* __restrict__ out, bool warp) {
  const int lane = threadIdx.x & 31;
  double Gm[3][3] = {};
  const double ke00 = K.p[1][0] - K.p[0][0], ke01 = K.p[1][1] - K.p[0][1];
  const double ke10 = K.p[2][0] - K.p[0][0], ke11 = K.p[2][1] - K.p[0][1];
  const double le00 = L.p[1][0] - L.p[0][0], le01 = L.p[1][1] - L.p[0][1];
  const double le10 = L.p[2][0] - L.p[0][0], le11 = L.p[2][1] - L.p[0][1];
  for (int x = warp ? lane : 0; x < nn; x += warp ? 32 : 1) {
    const double* nx = rt + 5 * x;
    double X0, X1 = 0.0;
    if (D == 1) {
      X0 = K.p[0][0] + nx[0] * ke00;
    } else {
      X0 = K.p[0][0] + (nx[0] * ke00 + nx[1] * ke10);
      X1 = K.p[0][1] + (nx[0] * ke01 + nx[1] * ke11);
    }
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 2
    for (int y = 0; y < nn; ++y) {
      const double* ny = rt + 5 * y;
      double r2;
      if (D == 1) {
        const double d0 = X0 - (L.p[0][0] + ny[0] * le00);
        r2 = d0 * d0;
      } else {
        const double d0 = X0 - (L.p[0][0] + (ny[0] * le00 + ny[1] * le10));
        const double d1 = X1 - (L.p[0][1] + (ny[0] * le01 + ny[1] * le11));
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
      t0 = fma(v, ny[2], t0);
      t1 = fma(v, ny[3], t1);
      if (D == 2) t2 = fma(v, ny[4], t2);
    }
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      const double lx = nx[2 + a];
      Gm[a][0] = fma(lx, t0, Gm[a][0]);
      Gm[a][1] = fma(lx, t1, Gm[a][1]);
      if (D == 2) Gm[a][2] = fma(lx, t2, Gm[a][2]);
    }
  }
  const double JJ = K.J * L.J;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double s = warp ? warp_sum(Gm[a][b]) : Gm[a][b];
      if (!warp || lane == 0) out[a * 3 + b] = s * JJ;
    }
}

// lanes sharing one far pair in phase B (2D: 16 / 81 / 256 evaluations for k = 2 / 3 / 4)
template <int D>
__device__ __forceinline__ int lanes_per_pair(int k) {
  return D == 2 ? (k <= 2 ? 1 : k == 3 ? 3 : 8) : 1;
}

// partial 3x3 block over the x nodes x0, x0 + xs, ... (precomputed node coordinates)
template <int D, int E4>
__device__ __forceinline__ void cross_part_pre(const double2* __restrict__ Xn, const double2* __restrict__ Yn,
                                               const double* __restrict__ rt, int nn, int x0, int xs, double ex,
                                               double (&Gm)[3][3]) {
  for (int i = x0; i < nn; i += xs) {
    const double2 X = Xn[i];
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 2
    for (int j = 0; j < nn; ++j) {
      const double2 Y = Yn[j];
      const double d0 = X.x - Y.x;
      double r2;
      if (D == 1) {
        r2 = d0 * d0;
      } else {
        const double d1 = X.y - Y.y;
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
      const double* ny = rt + 5 * j;
      t0 = fma(v, ny[2], t0);
      t1 = fma(v, ny[3], t1);
      if (D == 2) t2 = fma(v, ny[4], t2);
    }
    const double* nx = rt + 5 * i;
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      Gm[a][0] = fma(nx[2 + a], t0, Gm[a][0]);
      Gm[a][1] = fma(nx[2 + a], t1, Gm[a][1]);
      if (D == 2) Gm[a][2] = fma(nx[2 + a], t2, Gm[a][2]);
    }
  }
}

// y-outer variant for the multi-lane orders (2D k = 3: 3 lanes x 3 x-nodes; k = 4: 8 lanes x 2
// x-nodes): each y node (and its weights) is loaded / mapped once and reused for the lane's NX
// x nodes.  Per x node the sums over y run in the same order as cross_part_pre.
template <int E4, int NX, bool PRE>
__device__ __forceinline__ void cross_part_yo(const double2* __restrict__ Xn, const double2* __restrict__ Yn,
                                              const double* __restrict__ rt, int nn, int x0, int xs,
                                              const CellGeo& K, const CellGeo& L, double ex, double (&Gm)[3][3]) {
  double X0[NX], X1[NX], t[NX][3];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    const int x = x0 + i * xs;
    if (PRE) {
      X0[i] = Xn[x].x;
      X1[i] = Xn[x].y;
    } else {
      const double* nx = rt + 5 * x;
      X0[i] = K.p[0][0] + (nx[0] * (K.p[1][0] - K.p[0][0]) + nx[1] * (K.p[2][0] - K.p[0][0]));
      X1[i] = K.p[0][1] + (nx[0] * (K.p[1][1] - K.p[0][1]) + nx[1] * (K.p[2][1] - K.p[0][1]));
    }
    t[i][0] = t[i][1] = t[i][2] = 0.0;
  }
  double le00 = 0, le01 = 0, le10 = 0, le11 = 0;
  if (!PRE) {
    le00 = L.p[1][0] - L.p[0][0]; le01 = L.p[1][1] - L.p[0][1];
    le10 = L.p[2][0] - L.p[0][0]; le11 = L.p[2][1] - L.p[0][1];
  }
  for (int y = 0; y < nn; ++y) {
    const double* ny = rt + 5 * y;
    double Y0, Y1;
    if (PRE) {
      const double2 Y = Yn[y];
      Y0 = Y.x;
      Y1 = Y.y;
    } else {
      Y0 = L.p[0][0] + (ny[0] * le00 + ny[1] * le10);
      Y1 = L.p[0][1] + (ny[0] * le01 + ny[1] * le11);
    }
    const double w0 = ny[2], w1 = ny[3], w2 = ny[4];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      const double d0 = X0[i] - Y0, d1 = X1[i] - Y1;
      const double v = kpow<E4>(fma(d1, d1, d0 * d0), ex);
      t[i][0] = fma(v, w0, t[i][0]);
      t[i][1] = fma(v, w1, t[i][1]);
      t[i][2] = fma(v, w2, t[i][2]);
    }
  }
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    const double* nx = rt + 5 * (x0 + i * xs);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Gm[a][0] = fma(nx[2 + a], t[i][0], Gm[a][0]);
      Gm[a][1] = fma(nx[2 + a], t[i][1], Gm[a][1]);
      Gm[a][2] = fma(nx[2 + a], t[i][2], Gm[a][2]);
    }
  }
}

// same with the nodes mapped on the fly (orders above KPRE)
template <int D, int E4>
__device__ __forceinline__ void cross_part_gen(const double* __restrict__ rt, int nn, int x0, int xs,
                                               const CellGeo& K, const CellGeo& L, double ex, double (&Gm)[3][3]) {
  const double ke00 = K.p[1][0] - K.p[0][0], ke01 = K.p[1][1] - K.p[0][1];
  const double ke10 = K.p[2][0] - K.p[0][0], ke11 = K.p[2][1] - K.p[0][1];
  const double le00 = L.p[1][0] - L.p[0][0], le01 = L.p[1][1] - L.p[0][1];
  const double le10 = L.p[2][0] - L.p[0][0], le11 = L.p[2][1] - L.p[0][1];
  for (int x = x0; x < nn; x += xs) {
    const double* nx = rt + 5 * x;
    double X0, X1 = 0.0;
    if (D == 1) {
      X0 = K.p[0][0] + nx[0] * ke00;
    } else {
      X0 = K.p[0][0] + (nx[0] * ke00 + nx[1] * ke10);
      X1 = K.p[0][1] + (nx[0] * ke01 + nx[1] * ke11);
    }
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 2
    for (int y = 0; y < nn; ++y) {
      const double* ny = rt + 5 * y;
      double r2;
      if (D == 1) {
        const double d0 = X0 - (L.p[0][0] + ny[0] * le00);
        r2 = d0 * d0;
      } else {
        const double d0 = X0 - (L.p[0][0] + (ny[0] * le00 + ny[1] * le10));
        const double d1 = X1 - (L.p[0][1] + (ny[0] * le01 + ny[1] * le11));
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
      t0 = fma(v, ny[2], t0);
      t1 = fma(v, ny[3], t1);
      if (D == 2) t2 = fma(v, ny[4], t2);
    }
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      const double lx = nx[2 + a];
      Gm[a][0] = fma(lx, t0, Gm[a][0]);
      Gm[a][1] = fma(lx, t1, Gm[a][1]);
      if (D == 2) Gm[a][2] = fma(lx, t2, Gm[a][2]);
    }
  }
}

template <int D, int E4>
__global__ void __launch_bounds__(XT, 2) cross_tile_kernel(DevMesh m, const double* __restrict__ tab,
                                                           DevTables dir, OrderConsts oc, double ex,
                                                           double negC, TileView R, TileView Cv,
                                                           const int2* __restrict__ tpairs, int ntp,
                                                           int* __restrict__ queue, int kmax, int symmetric,
                                                           int row_begin, int row_end,
                                                           double* __restrict__ Aout, int64_t lda,
                                                           unsigned long long* __restrict__ evals,
                                                           unsigned long long* __restrict__ near_keys,
                                                           unsigned int* __restrict__ near_count,
                                                           unsigned int near_cap, int discover,
                                                           const unsigned long long* __restrict__ nearH,
                                                           const int* __restrict__ nearI, unsigned long long hmask,
                                                           const double* __restrict__ nearG) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CrossShared& S = *reinterpret_cast<CrossShared*>(smem_raw);
  double* rtab = reinterpret_cast<double*>(smem_raw + ((sizeof(CrossShared) + 15) / 16) * 16);
  const int KW = (D == 1) ? KW1D : KW2D;   // near pairs (k >= KW) go to fl_near.cu when a list is given
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long my_evals = 0;

  // ---- the disjoint rules, once per CTA
  if (tid == 0) {
    int off = 0;
    for (int k = 0; k < KDIR; ++k) {
      S.kofs[k] = off;
      off += (k >= 2 && k <= kmax) ? dir.rule(T_DISJ, k).cnt : 0;
    }
  }
  __syncthreads();
  for (int k = 2; k <= kmax; ++k) {
    const RuleRef rr = dir.rule(T_DISJ, k);
    for (int i = tid; i < rr.cnt; i += XT) {
      const double* nd = tab + (size_t)(rr.off + i) * NODE;
      double* o = rtab + 5 * (S.kofs[k] + i);
      o[0] = nd[0]; o[1] = nd[1]; o[2] = nd[3]; o[3] = nd[4]; o[4] = nd[5];
    }
  }

  for (;;) {
    if (tid == 0) S.tile = atomicAdd(queue, 1);       // tile pairs come heavy (near) first
    __syncthreads();
    const int ti = S.tile;
    if (ti >= ntp) break;
    const int2 tp = tpairs[ti];
    const int tr = tp.x, tc = tp.y;
    const int nR = R.ncell[tr], nC = Cv.ncell[tc];

    // ---- stage the tile metadata
    for (int i = tid; i < nR; i += XT) {
      const int c = R.cells[tr * TILE_MAXC + i];
      S.rowc[i] = c;
      for (int a = 0; a < 3; ++a) S.rslot[i][a] = (signed char)R.slots[(tr * TILE_MAXC + i) * 3 + a];
      if (D == 2) {
        const CellGeo& g = m.geo[c];
        S.rcx[i] = g.cx; S.rcy[i] = g.cy; S.rrad[i] = g.rad; S.rJ[i] = g.J;
        S.rlnh[i] = __logf((float)g.diam); S.rlh[i] = (float)g.ldiam;
      }
    }
    for (int i = tid; i < nC; i += XT) {
      S.colc[i] = Cv.cells[tc * TILE_MAXC + i];
      for (int a = 0; a < 3; ++a) S.cslot[i][a] = (signed char)Cv.slots[(tc * TILE_MAXC + i) * 3 + a];
    }
    for (int i = tid; i < TILE; i += XT) {
      S.rdof[i] = R.dofs[tr * TILE + i];
      S.cdof[i] = Cv.dofs[tc * TILE + i];
    }
    for (int i = tid; i < TILE * (TILE + 1); i += XT) (&S.At[0][0])[i] = 0.0;
    __syncthreads();
    if (tid < TILE) {                    // tile row r -> its (row cell, slot) entries, in cell-list order
      int c = 0;
      for (int i = 0; i < nR; ++i)
        for (int a = 0; a <= D; ++a)
          if (S.rslot[i][a] == tid && c < ROWL) S.rowl[tid][c++] = (short)(i * 4 + a);
      S.rown[tid] = (unsigned char)c;
    }
    __syncthreads();                     // rowl / rown are read by other warps below

    for (int cs0 = 0; cs0 < nC; cs0 += SBC) {
      if (D == 2 && tid >= 32 && tid < 32 + SBC && cs0 + tid - 32 < nC) {
        const int i = tid - 32;
        const CellGeo& g = m.geo[S.colc[cs0 + i]];
        S.ccx[i] = g.cx; S.ccy[i] = g.cy; S.crad[i] = g.rad; S.cJ[i] = g.J;
        S.clnh[i] = __logf((float)g.diam); S.clh[i] = (float)g.ldiam;
      }
      if (tid >= 64 && tid < 64 + TILE) {   // tile column -> its (column cell, slot) entries here
        const int col = tid - 64;
        int c = 0;
        for (int cc = 0; cc < SBC && cs0 + cc < nC; ++cc)
          for (int b = 0; b <= D; ++b)
            if (S.cslot[cs0 + cc][b] == col && c < ROWL) S.cent[col][c++] = (short)(cc * 4 + b);
        S.ccnt[col] = (unsigned char)c;
      }
      for (int rs0 = 0; rs0 < nR; rs0 += SBR) {
        // ---- (A) orders of the 512 pairs of this sub-block
        if (tid <= KDIR) S.hist[tid] = 0;
        if (tid >= 64 && tid < 64 + TILE) {   // tile row -> its rowl range in this row sub-block
          const int r = tid - 64;
          int e0 = 0;
          while (e0 < S.rown[r] && (S.rowl[r][e0] >> 2) < rs0) ++e0;
          int e1 = e0;
          while (e1 < S.rown[r] && (S.rowl[r][e1] >> 2) < rs0 + SBR) ++e1;
          S.rr0[r] = (short)e0;
          S.rr1[r] = (short)e1;
        }
        __syncthreads();
        if (tid < 32) {                       // touched rows / columns, ascending
          const bool r0 = S.rr1[tid] > S.rr0[tid], r1 = S.rr1[tid + 32] > S.rr0[tid + 32];
          const bool c0 = S.ccnt[tid] > 0, c1 = S.ccnt[tid + 32] > 0;
          const unsigned br0 = __ballot_sync(0xffffffffu, r0), br1 = __ballot_sync(0xffffffffu, r1);
          const unsigned bc0 = __ballot_sync(0xffffffffu, c0), bc1 = __ballot_sync(0xffffffffu, c1);
          const unsigned lt = (1u << tid) - 1u;
          if (r0) S.trow[__popc(br0 & lt)] = (unsigned char)tid;
          if (r1) S.trow[__popc(br0) + __popc(br1 & lt)] = (unsigned char)(tid + 32);
          if (c0) S.tcol[__popc(bc0 & lt)] = (unsigned char)tid;
          if (c1) S.tcol[__popc(bc0) + __popc(bc1 & lt)] = (unsigned char)(tid + 32);
          if (tid == 0) { S.ntr = __popc(br0) + __popc(br1); S.ntc = __popc(bc0) + __popc(bc1); }
        }
        for (int p = tid; p < SBP; p += XT) {
          const int rc = rs0 + p / SBC, cc = cs0 + p % SBC;
          int k = 0;
          if (rc < nR && cc < nC) {
            const int idK = S.rowc[rc], idL = S.colc[cc];
            int kf = 0;
            if (D == 2) {
              const int lc = p % SBC;
              kf = order2d_fast(oc, S.rcx[rc] - S.ccx[lc], S.rcy[rc] - S.ccy[lc], S.rrad[rc], S.crad[lc],
                                S.rlnh[rc], S.rlh[rc], S.clnh[lc], S.clh[lc]);
            }
            bool disjoint = kf > 0;
            if (!disjoint) {
              // close / ambiguous pair: exact reference arithmetic on the cell records; the
              // reference orders a disjoint pair as (min id, max id) (assembly.py:973-982, :705)
              const CellGeo& Kg = m.geo[idK];
              const CellGeo& Lg = m.geo[idL];
              if (!touching<D>(Kg, Lg)) {
                const CellGeo& P = (idK < idL) ? Kg : Lg;
                const CellGeo& Qg = (idK < idL) ? Lg : Kg;
                kf = order_disjoint_fast(oc, oc.coff, P, Qg, dist_estimate<D>(P, Qg));
                disjoint = true;
              }
            }
            if (disjoint) {
              k = kf;
              if (k >= KW && (discover || nearG != nullptr)) {
                // near pair: its block is computed once by the near-pair kernel (fl_near.cu)
                const unsigned long long key = near_key(idK, idL, k);
                if (discover) {
                  // warp-aggregated append (one atomic per warp and sub-block pass)
                  const unsigned am = __activemask();
                  const int leader = __ffs(am) - 1;
                  unsigned int base = 0;
                  if (lane == leader) base = atomicAdd(near_count, (unsigned)__popc(am));
                  base = __shfl_sync(am, base, leader);
                  const unsigned int slot = base + __popc(am & ((1u << lane) - 1u));
                  if (slot < near_cap) near_keys[slot] = key;
                  k = 0;
                } else {
                  unsigned long long h = near_hash(key) & hmask;   // open-addressing lookup
                  unsigned long long hk;
                  while ((hk = nearH[h]) != key && hk != NEAR_EMPTY) h = (h + 1) & hmask;
                  int64_t lo = 0;
                  if (hk == key) lo = nearI[h];
                  else atomicOr(m.err, 4);                         // cannot happen: same orders as discovery
                  const double* g = nearG + lo * 9;
                  const bool tr = idK > idL;                     // M^{min,max}: transpose when K is the max
#pragma unroll
                  for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) S.Gs[p][a * 3 + b] = tr ? g[b * 3 + a] : g[a * 3 + b];
                  k = NEAR_MARK;
                }
              }
            }
          }
          S.pk[p] = (unsigned char)k;
          if (k != NEAR_MARK) atomicAdd(&S.hist[k], 1);
        }
        __syncthreads();
        if (discover) continue;
        if (tid == 0) {                  // descending k: large (warp) pairs first
          int off = 0;
          for (int k = KDIR - 1; k >= 1; --k) { S.cursor[k] = off; off += S.hist[k]; }
          int nl = 0;
          for (int k = KDIR - 1; k >= KW; --k) nl += S.hist[k];
          S.nlarge = nl;
          S.nsmall = off - nl;
          S.qlarge = 0;
          S.qsmall = 0;
          int nch = 0;
          for (int k = KW - 1; k >= 2; --k) {
            const int ppc = 32 / lanes_per_pair<D>(k);
            for (int s0 = 0; s0 < S.hist[k]; s0 += ppc) {
              S.chs[nch] = (short)(S.cursor[k] + s0);
              S.chn[nch] = (unsigned char)min(ppc, S.hist[k] - s0);
              S.chk[nch] = (unsigned char)k;
              ++nch;
            }
          }
          S.nchunk = nch;
        }
        // ---- (A2) node coordinates of the sub-block's cells for the small orders present
        for (int k = 2; k <= KPRE; ++k) {
          if (S.hist[k] == 0) continue;
          const int nn = (D == 1) ? k : k * k;
          const double* rt = rtab + 5 * S.kofs[k];
          for (int idx = tid; idx < (SBR + SBC) * nn; idx += XT) {
            const int c = idx / nn, x = idx % nn;
            const int cl = (c < SBR) ? rs0 + c : cs0 + (c - SBR);
            if ((c < SBR && cl >= nR) || (c >= SBR && cl >= nC)) continue;
            const CellGeo& g = m.geo[(c < SBR) ? S.rowc[cl] : S.colc[cl]];
            double X0, X1 = 0.0;
            if (D == 1) {
              X0 = g.p[0][0] + rt[5 * x] * (g.p[1][0] - g.p[0][0]);
            } else {
              X0 = g.p[0][0] + (rt[5 * x] * (g.p[1][0] - g.p[0][0]) + rt[5 * x + 1] * (g.p[2][0] - g.p[0][0]));
              X1 = g.p[0][1] + (rt[5 * x] * (g.p[1][1] - g.p[0][1]) + rt[5 * x + 1] * (g.p[2][1] - g.p[0][1]));
            }
            S.nodes[c][pre_off<D>(k) + x] = make_double2(X0, X1);
          }
        }
        __syncthreads();
        for (int p = tid; p < SBP; p += XT) {
          const int k = S.pk[p];
          if (k > 0 && k != NEAR_MARK) S.plist[atomicAdd(&S.cursor[k], 1)] = (short)p;
        }
        __syncthreads();
        // ---- (B) the 3x3 blocks, pairs sorted by k
        const int nl = S.nlarge, ns = S.nsmall;
        for (;;) {
          int i = 0;
          if (lane == 0) i = atomicAdd(&S.qlarge, 1);
          i = __shfl_sync(0xffffffffu, i, 0);
          if (i >= nl) break;
          const int p = S.plist[i];
          const int k = S.pk[p];
          const int nn = (D == 1) ? k : k * k;
          cross_gen<D, E4>(rtab + 5 * S.kofs[k], nn, m.geo[S.rowc[rs0 + p / SBC]], m.geo[S.colc[cs0 + p % SBC]],
                           ex, S.Gs[p], true);
          if (lane == 0) my_evals += (unsigned long long)nn * nn;
        }
        for (;;) {
          int ch = 0;
          if (lane == 0) ch = atomicAdd(&S.qsmall, 1);
          ch = __shfl_sync(0xffffffffu, ch, 0);
          if (ch >= S.nchunk) break;
          const int k = S.chk[ch];
          const int L = lanes_per_pair<D>(k);
          const int g = lane / L, sub = lane - g * L;
          const bool act = g < S.chn[ch];
          const int p = act ? S.plist[S.chs[ch] + g] : 0;
          const int nn = (D == 1) ? k : k * k;
          const int r = p / SBC, c = p % SBC;
          const double* rt = rtab + 5 * S.kofs[k];
          if (k == 2) {                       // one lane per pair, fully unrolled
            if (act) {
              const double JJ = D == 2 ? S.rJ[rs0 + r] * S.cJ[c] : m.geo[S.rowc[rs0 + r]].J * m.geo[S.colc[cs0 + c]].J;
              cross_fixed<D, E4, 2>(&S.nodes[r][pre_off<D>(2)], &S.nodes[SBR + c][pre_off<D>(2)], rt, JJ, ex, S.Gs[p]);
              my_evals += (unsigned long long)nn * nn;
            }
            continue;
          }
          double Gm[3][3] = {};
          if (act) {
            if (D == 2 && k == 3) {
              cross_part_yo<E4, 3, true>(&S.nodes[r][pre_off<D>(3)], &S.nodes[SBR + c][pre_off<D>(3)], rt, nn, sub,
                                         L, m.geo[0], m.geo[0], ex, Gm);
            } else if (D == 2 && k == 4) {
              cross_part_yo<E4, 2, false>(nullptr, nullptr, rt, nn, sub, L, m.geo[S.rowc[rs0 + r]],
                                          m.geo[S.colc[cs0 + c]], ex, Gm);
            } else if (k <= KPRE) {
              cross_part_pre<D, E4>(&S.nodes[r][pre_off<D>(k)], &S.nodes[SBR + c][pre_off<D>(k)], rt, nn, sub, L, ex,
                                    Gm);
            } else {
              cross_part_gen<D, E4>(rt, nn, sub, L, m.geo[S.rowc[rs0 + r]], m.geo[S.colc[cs0 + c]], ex, Gm);
            }
          }
          // fixed-order reduction over the L lanes of the pair (L = 1, 3 or 8)
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              double v = Gm[a][b];
              if (L == 3) {
                const double v1 = __shfl_down_sync(0xffffffffu, v, 1), v2 = __shfl_down_sync(0xffffffffu, v, 2);
                v = (v + v1) + v2;
              } else if (L == 8) {
                v += __shfl_down_sync(0xffffffffu, v, 4);
                v += __shfl_down_sync(0xffffffffu, v, 2);
                v += __shfl_down_sync(0xffffffffu, v, 1);
              }
              Gm[a][b] = v;
            }
          if (act && sub == 0) {
            const double JJ = D == 2 ? S.rJ[rs0 + r] * S.cJ[c] : m.geo[S.rowc[rs0 + r]].J * m.geo[S.colc[cs0 + c]].J;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) S.Gs[p][a * 3 + b] = Gm[a][b] * JJ;
            my_evals += (unsigned long long)nn * nn;
          }
        }
        __syncthreads();
        // ---- (C) entry-parallel scatter: every touched (row, column) of the tile sums its
        // terms of this sub-block in (row entry, column entry) order, then adds once
        {
          const int ntr = S.ntr, ntc = S.ntc, nit = ntr * ntc;
          const unsigned long long mg = ntc ? ((1ull << 32) + ntc - 1) / (unsigned)ntc : 0;   // it / ntc, it < 2^16
          for (int it = tid; it < nit; it += XT) {
            const int ri = (int)(((unsigned long long)it * mg) >> 32), ci = it - ri * ntc;
            const int r = S.trow[ri], c = S.tcol[ci];
            const int nce = S.ccnt[c];
            double v = 0.0;
            for (int e = S.rr0[r]; e < S.rr1[r]; ++e) {
              const int rc = S.rowl[r][e] >> 2, a = S.rowl[r][e] & 3;
              const int pr = (rc - rs0) * SBC;
              for (int f = 0; f < nce; ++f) {
                const int ent = S.cent[c][f];
                const int p = pr + (ent >> 2);
                if (S.pk[p] == 0) continue;
                v += negC * S.Gs[p][a * 3 + (ent & 3)];
              }
            }
            S.At[r][c] += v;
          }
        }
        __syncthreads();
      }
    }
    // ---- write the tile (and its mirror) once
    if (discover) { __syncthreads(); continue; }
    for (int idx = tid; idx < TILE * TILE; idx += XT) {
      const int r = idx / TILE, c = idx % TILE;
      const int i = S.rdof[r], j = S.cdof[c];
      if (i >= row_begin && i < row_end && j >= 0) Aout[(int64_t)(i - row_begin) * lda + j] = S.At[r][c];
    }
    if (symmetric && tr != tc) {
      for (int idx = tid; idx < TILE * TILE; idx += XT) {
        const int c = idx / TILE, r = idx % TILE;
        const int i = S.rdof[r], j = S.cdof[c];
        if (i >= 0 && j >= row_begin && j < row_end) Aout[(int64_t)(j - row_begin) * lda + i] = S.At[r][c];
      }
    }
    __syncthreads();
  }
  if (evals) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_evals += __shfl_xor_sync(0xffffffffu, my_evals, o);
    if (lane == 0) atomicAdd(evals, my_evals);
  }
}

// two CTAs per SM (2 x 113.5 KB of the 228 KB) must fit for the 2D tiles
static_assert(((sizeof(CrossShared) + 15) / 16) * 16 + sizeof(double) * 5 * (9 * 10 * 19 / 6 - 1) <= 113 * 1024,
              "cross_tile_kernel shared memory exceeds two CTAs per SM");
size_t cross_smem_bytes(int d) {
  const int nodes = (d == 1) ? (32 * 33 / 2 - 1) : (9 * 10 * 19 / 6 - 1);   // sum_{k=2}^{kmax} k^d
  return ((sizeof(CrossShared) + 15) / 16) * 16 + sizeof(double) * 5 * nodes;
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
      // the kernels use the fast path; it must agree with the exact reference arithmetic
      const double dt = dist_estimate<D>(A, B);
      kt = (int8_t)order_disjoint_fast(oc, oc.coff_tail, A, B, dt);
      if (kt != order_disjoint(oc, oc.coff_tail, A, B, dt)) atomicOr(m.err, 2);
      if (a < b) {
        kc = (int8_t)order_disjoint_fast(oc, oc.coff, A, B, dt);
        if (kc != order_disjoint(oc, oc.coff, A, B, dt)) atomicOr(m.err, 2);
      }
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

// FRACLAP_TAIL_FOLD_WARP=0: the warp tail behind the block kernel keeps plain weights (A/B switch)
static bool tail_fold_warp() {
  static const bool on = [] {
    const char* v = getenv("FRACLAP_TAIL_FOLD_WARP");
    return !(v && v[0] == '0');
  }();
  return on;
}

void launch_tail(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                 const int* targets, int ntargets, double* psi, unsigned long long* evals, cudaStream_t st,
                 const int8_t* kuni, const int* blk_of, const int* bcells, int nb, const int8_t* kcell,
                 const unsigned long long* psifx, double fxinv, const double* ujh, const double* wh,
                 const double2* un, const double2* uhi) {
  if (ntargets <= 0) return;
  const int grid = (ntargets + TAIL_WARPS - 1) / TAIL_WARPS;
  if (m.d == 1) {
    FL_E4_SWITCH(e4, (tail_kernel<1, E4, false><<<grid, TAIL_WARPS * 32, 0, st>>>(m, t.data, t, oc, ex, targets, ntargets, psi, evals, nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr), ::fl::note_launch()));
  } else if (kuni && ujh && wh && un && uhi && oc.cap_disjoint <= 9 && tail_fold_warp()) {
    FL_E4_SWITCH(e4, (tail_kernel<2, E4, true><<<grid, TAIL_WARPS * 32, 0, st>>>(m, t.data, t, oc, ex, targets, ntargets, psi, evals, kuni, blk_of, bcells, nb, kcell, psifx, fxinv, ujh, wh, un, uhi), ::fl::note_launch()));
  } else {
    FL_E4_SWITCH(e4, (tail_kernel<2, E4, false><<<grid, TAIL_WARPS * 32, 0, st>>>(m, t.data, t, oc, ex, targets, ntargets, psi, evals, kuni, blk_of, bcells, nb, kcell, psifx, fxinv, nullptr, nullptr, nullptr, nullptr), ::fl::note_launch()));
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
                        double Cds, const Tiles& rows, const Tiles& cols, const int2* tpairs, int ntp,
                        bool symmetric, int row_begin, int row_end, double* A, int64_t lda,
                        unsigned long long* evals, unsigned long long* near_keys, unsigned int* near_count,
                        unsigned int near_cap, int discover, const unsigned long long* nearH, const int* nearI,
                        unsigned long long hmask, const double* nearG, cudaStream_t st) {
  if (ntp <= 0) return;
  TileView R{rows.dofs.p, rows.ncell.p, rows.cells.p, rows.slots.p};
  TileView C{cols.dofs.p, cols.ncell.p, cols.cells.p, cols.slots.p};
  const size_t smem = cross_smem_bytes(m.d);
  const double negC = -Cds;   // (C/2) * (-2)  (assembly.py:723, :1100)
  const int kmax = oc.cap_disjoint;
  DBuf<int> queue(1);
  FL_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(int), st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = FL_PERSISTENT ? std::min(ntp, 2 * sms) : ntp;   // persistent: 2 CTAs per SM
  if (m.d == 1) {
    FL_E4_SWITCH(e4, {
      FL_CUDA(cudaFuncSetAttribute(cross_tile_kernel<1, E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cross_tile_kernel<1, E4><<<grid, XT, smem, st>>>(m, t.data, t, oc, ex, negC, R, C, tpairs, ntp, queue.p, kmax,
                                                     symmetric ? 1 : 0, row_begin, row_end, A, lda, evals, near_keys,
                                                     near_count, near_cap, discover, nearH, nearI, hmask, nearG),
          ::fl::note_launch();
    });
  } else {
    FL_E4_SWITCH(e4, {
      FL_CUDA(cudaFuncSetAttribute(cross_tile_kernel<2, E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cross_tile_kernel<2, E4><<<grid, XT, smem, st>>>(m, t.data, t, oc, ex, negC, R, C, tpairs, ntp, queue.p, kmax,
                                                     symmetric ? 1 : 0, row_begin, row_end, A, lda, evals, near_keys,
                                                     near_count, near_cap, discover, nearH, nearI, hmask, nearG),
          ::fl::note_launch();
    });
  }
  FL_CHECK_LAUNCH();
}

void launch_debug_orders(const DevMesh& m, const OrderConsts& oc, int8_t* cross_k, int8_t* tail_k,
                         cudaStream_t st) {
  const int64_t tot = (int64_t)m.nc * m.nc;
  const int grid = (int)((tot + 255) / 256);
  if (m.d == 1) orders_kernel<1><<<grid, 256, 0, st>>>(m, oc, cross_k, tail_k), ::fl::note_launch();
  else orders_kernel<2><<<grid, 256, 0, st>>>(m, oc, cross_k, tail_k), ::fl::note_launch();
  FL_CHECK_LAUNCH();
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
    const int kt = order_disjoint_fast(oc, oc.coff_tail, A, B, dt);
    if (kt != order_disjoint(oc, oc.coff_tail, A, B, dt)) atomicOr(m.err, 2);
    atomicAdd(&stl[kt], 1ull);
    if (a < b) {
      const int kc = order_disjoint_fast(oc, oc.coff, A, B, dt);
      if (kc != order_disjoint(oc, oc.coff, A, B, dt)) atomicOr(m.err, 2);
      atomicAdd(&sc[kc], 1ull);
    }
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

// FP64 peak probe: 8 independent DFMA chains per thread, 148*8 CTAs of 256 threads, best of 5.
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
  // ~5 ms per launch: long enough that launch and ramp are < 1 % (a 0.6 ms probe read ~8 % low)
  const int grid = sms * 8, iters = 32768;
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

}  // namespace fl

namespace fl {
template <int E4>
__global__ void kpow_probe_kernel(int d, const double* x, int64_t n, double ex, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = d == 1 ? kpow_abs<E4>(x[i], ex) : (d == 12 ? kpow_acc<E4>(x[i], ex, 0.0) : kpow<E4>(x[i], ex));
}
void launch_kpow_probe(int d, int e4, const double* x, int64_t n, double ex, double* out, cudaStream_t st) {
  const int grid = (int)((n + 255) / 256);
  FL_E4_SWITCH(e4, (kpow_probe_kernel<E4><<<grid, 256, 0, st>>>(d, x, n, ex, out), ::fl::note_launch()));
  FL_CHECK_LAUNCH();
}
}  // namespace fl
