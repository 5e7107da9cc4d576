// 2D kernel tail Psi_K(x_q) (direct_tail_potential, assembly.py:985-1025) by Morton block pairs.
//
// Psi_K(x_q) = sum over the cells L not touching K of J_L sum_y w_y |x_q - y|^(-d-2s), y the
// Gauss nodes of L's order k(K, L) (select_order with C_offset - 4, :997).  The cells are cut
// into the Morton blocks of the cross term (Blocks2D, 32 cells).  For an ordered pair of blocks
// (P targets, Q sources) rigorous bounds of the order formula over all 32 x 32 cell pairs
// (tail_kuni_kernel) either prove one order kuni for every pair — the blocks are then disjoint,
// so no pair touches — or not (kuni = 0).
//
// tail2d_block_kernel: one CTA per target block P, 256 threads holding the 512 target nodes
// (32 cells x 16 XQ nodes, 2 per thread) in registers.  It walks the uniform source blocks Q in
// ascending order: the next block's geometry is loaded into registers while the current one is
// evaluated, its k^2 mapped nodes per cell (absolute coordinates, as _map_points) and J*w are
// staged in shared memory, and every thread sweeps them against its two targets, 4 sources per
// step — a pure FP64 stream, every shared load a broadcast.  The remaining source blocks of P
// (kuni = 0: nearby blocks, P itself, blocks straddling an order boundary) are evaluated cell
// pair by cell pair by fl_far.cu's warp-per-target tail_kernel, which adds its sums to these.
// Deterministic: every target node sums its sources in a fixed order (Q ascending, then the
// block's nodes), independent of how the rows are split over GPUs.
#include <cstring>

#include "fl_internal.h"

namespace fl {

namespace {

constexpr int TB = CB2D;           // cells per block
constexpr int TQN = 16;            // target nodes per cell (XQ_ORDER 4 in 2D, assembly.py:635)
constexpr int TT = 256;            // threads per CTA: 2 target nodes each
constexpr int TWIN = 1024;         // source nodes per shared-memory window
constexpr int TU = 4;              // source nodes per thread per step
#ifndef FL_TUF
#define FL_TUF 8
#endif
constexpr int TUF = FL_TUF;        // ... of the folded sweep (window sizes are multiples of 8)
constexpr int RULE_NODES = DISJ_RULE_NODES;   // sum_{k=2}^{9} k^2
constexpr int RS = 4;              // doubles per staged rule node: u0, u1, w, w^(1/(2 ex))
__host__ __device__ constexpr int useg(int k) { return k == 2 ? 0 : (k == 3 ? 128 : 416); }   // Blocks2D::un
__host__ __device__ constexpr int roff(int k) { return disj_roff(k); }   // sum_{j=2}^{k-1} j^2

__global__ void tail_flag_kernel(const int* __restrict__ targets, int ntargets, const int* __restrict__ blk_of,
                                 int* __restrict__ tflag, int* __restrict__ tcell) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ntargets) {
    tflag[blk_of[targets[i]]] = 1;
    tcell[targets[i]] = 1;
  }
}

// kuni[P * nb + Q] for the target blocks P: one order for every (target in P, source in Q) pair
// when the bounds of the boosted order formula agree; -1 when the blocks are disjoint but the
// orders are not uniform (then decided per target cell, cell_block_korder); 0 otherwise
__global__ void tail_kuni_kernel(OrderConsts oc, const double* __restrict__ bs, const int* __restrict__ tflag, int nb,
                                 int mixed, int8_t* __restrict__ kuni, unsigned long long* __restrict__ dmin4,
                                 int* __restrict__ run) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * nb) return;
  const int P = (int)(i / nb), Q = (int)(i - (int64_t)P * nb);
  int k = 0;
  // every row (not only the target blocks'): the sym4 split must not depend on the row range
  if (P != Q) {
    const double* a = bs + 8 * P;
    const double* b = bs + 8 * Q;
    const double dc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
    const double Dmin = (dc - a[2] - b[2]) * (1.0 - 1e-12) - 1e-300;
    const double Dmax = (dc + a[2] + b[2]) * (1.0 + 1e-12);
    // disjoint bounding circles (no pair touches), at least either block's radius apart: the
    // centred r2 expansion of the block kernel then loses at most a factor 9 of relative accuracy;
    // every operation is symmetric in (P, Q), so kuni[P][Q] == kuni[Q][P] bitwise
    if (Dmin > 0.0 && Dmin >= fmax(a[2], b[2])) {
      const double hmn = fmin(a[3], b[3]), hmx = fmax(a[4], b[4]), lmn = fmin(a[5], b[5]), lmx = fmax(a[6], b[6]);
      const double hi = order_bound_hi(oc, oc.coff_tail, Dmin, hmn, hmx, lmn, lmx);
      const double lo = order_bound_lo(oc, oc.coff_tail, Dmin, Dmax, hmn, hmx, lmn, lmx);
      const double c0 = fmin(fmax(ceil(lo - 1e-9), 2.0), (double)oc.cap_disjoint);
      const double c1 = fmin(fmax(ceil(hi + 1e-9), 2.0), (double)oc.cap_disjoint);
      k = c0 == c1 ? (int)c0 : (mixed ? -1 : 0);  // -1: per target cell (cell_block_korder)
      if (k == 4) {
        atomicMin(dmin4, (unsigned long long)__double_as_longlong(Dmin));
        if (Q > P && tflag[Q]) run[P] = 1;   // P's CTA evaluates (P, Q) for target block Q
      }
    }
  }
  kuni[i] = (int8_t)k;
}

// The block pairs the circle bounds left open (kuni == 0, disjoint, at least a block radius
// apart) get a second try with the exact range of the 32 x 32 pairs' distance estimates
// (block_pair_dist_range): a warp per unordered pair P < Q, both entries written with the same
// order, so kuni stays symmetric; the order-4 bookkeeping as in tail_kuni_kernel.
__global__ void tail_refine_kernel(OrderConsts oc, DevMesh m, const int* __restrict__ bcells,
                                   const double* __restrict__ bs, const int* __restrict__ tflag, int nb,
                                   int8_t* __restrict__ kuni, unsigned long long* __restrict__ dmin4,
                                   int* __restrict__ run) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)nb * nb) return;
  const int P = (int)(w / nb), Q = (int)(w - (int64_t)P * nb);
  if (P >= Q || kuni[w] != 0) return;
  const double* a = bs + 8 * P;
  const double* b = bs + 8 * Q;
  const double dc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
  const double Dmin = (dc - a[2] - b[2]) * (1.0 - 1e-12) - 1e-300;
  if (!(Dmin > 0.0 && Dmin >= fmax(a[2], b[2]))) return;
  double lo, hi;
  block_pair_dist_range(m, bcells, P, Q, lane, lo, hi);
  const int k = block_uniform_order(oc, oc.coff_tail, lo * (1.0 - 1e-12) - 1e-300, hi * (1.0 + 1e-12), a, b);
  if (k == 0 || lane) return;
  kuni[w] = (int8_t)k;
  kuni[(size_t)Q * nb + P] = (int8_t)k;
  if (k == 4) {
    atomicMin(dmin4, (unsigned long long)__double_as_longlong(Dmin));
    if (tflag[Q]) run[P] = 1;
  }
}

// per block slot J^(1/(2 ex)) (0 for an empty slot): the cell factor of the folded source weights
// c = (J w)^(1/ex) = (J^(1/(2 ex)) w^(1/(2 ex)))^2 of sweep_fold and of the warp tail's folded path
__global__ void fold_slots_kernel(DevMesh m, const int* __restrict__ bcells, int nslots, double hex,
                                  double* __restrict__ ujh) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nslots) return;
  const int c = bcells[i];
  ujh[i] = c >= 0 ? pow(m.geo[c].J, hex) : 0.0;
}

// per node of the disjoint rules k = 2..9: w^(1/(2 ex)) (0 when the rule is missing)
__global__ void fold_rules_kernel(const double* __restrict__ tab, DevTables dir, double hex, double* __restrict__ wh) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= RULE_NODES) return;
  int k = 2;
  while (roff(k + 1) <= i) ++k;
  const RuleRef rr = dir.rule(T_DISJ, k);
  wh[i] = rr.cnt == k * k ? pow(tab[(size_t)(rr.off + i - roff(k)) * NODE + 2], hex) : 0.0;
}

// mapped nodes of the disjoint rules k = 5..9 for every block slot, node-major per order (the warp
// tail copies them instead of mapping them per (target, source) pair); the mapping is _map_points'
// y = P0 + u0 (P1 - P0) + u1 (P2 - P0) in the warp tail's own operation order
__global__ void hi_nodes_kernel(DevMesh m, const int* __restrict__ bcells, int nb, const double* __restrict__ tab,
                                DevTables dir, double2* __restrict__ uhi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * UHI2D) return;
  const int b = (int)(i / UHI2D), x = (int)(i % UHI2D);
  int k = 5;
  while (k < 9 && uhi_seg(k + 1) <= x) ++k;
  const int loc = x - uhi_seg(k), r = loc / TB, c = loc % TB;
  const int cell = bcells[b * TB + c];
  const RuleRef rr = dir.rule(T_DISJ, k);
  double2 y = make_double2(0.0, 0.0);
  if (cell >= 0 && rr.cnt == k * k) {
    const CellGeo& g = m.geo[cell];
    const double* nd = tab + (size_t)(rr.off + r) * NODE;
    y.x = g.p[0][0] + (nd[0] * (g.p[1][0] - g.p[0][0]) + nd[1] * (g.p[2][0] - g.p[0][0]));
    y.y = g.p[0][1] + (nd[0] * (g.p[1][1] - g.p[0][1]) + nd[1] * (g.p[2][1] - g.p[0][1]));
  }
  uhi[i] = y;
}

// sum of the Jacobians in units of jmax / 2^30 (an integer sum: the same whatever the order)
__global__ void jsum_kernel(DevMesh m, double units, unsigned long long* __restrict__ jsum) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = c < m.nc ? (unsigned long long)__double2ll_ru(m.geo[c].J * units) : 0ull;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(jsum, v);
}

// sym4: an order-4 uniform block pair (P, Q) is evaluated once, by the CTA of min(P, Q); its
// kernel values serve both directions, because the order-4 source rule is the 16-node target rule
// itself (simplex_rule(2, 4) == XQ, assembly.py:635, :1012).  The split depends on the mesh only,
// not on the row range, so row blocks stay bitwise the whole matrix's rows: a block that holds no
// target still runs (as a helper) when it is the smaller block of an order-4 pair with a target block.
__device__ __forceinline__ int sym4_mode(int T, int S, int k) {
  if (k != 4) return 0;                // 0: ordinary source block
  return S > T ? 1 : -1;               // 1: this CTA takes both directions; -1: S's CTA does
}

// per target cell K and mixed source block Q (kuni == -1): K's own order for the block, or 0
__global__ void tail_kcell_kernel(OrderConsts oc, DevMesh m, const int* __restrict__ targets, int ntargets,
                                  const int* __restrict__ blk_of, const int8_t* __restrict__ kuni,
                                  const double* __restrict__ bs, int nb, int8_t* __restrict__ kcell) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ntargets * nb) return;
  const int t = (int)(i / nb), Q = (int)(i - (int64_t)t * nb);
  const int K = targets[t];
  if (kuni[(size_t)blk_of[K] * nb + Q] != -1) return;
  kcell[(size_t)K * nb + Q] = (int8_t)cell_block_korder(oc, oc.coff_tail, m.geo[K], bs + 8 * Q);
}

// geometry field f of cell slot c of block Q: P0x P0y (P1-P0)x (P1-P0)y (P2-P0)x (P2-P0)y J valid
// (the last field is J^(1/(2 ex)) of the folded weights, nonzero exactly for a valid slot)
__device__ __forceinline__ double geo_field(const DevMesh& m, const int* __restrict__ bcells,
                                            const double* __restrict__ ujh, int Q, int t) {
  const int c = bcells[Q * TB + (t >> 3)], f = t & 7;
  if (c < 0) return 0.0;
  const CellGeo& g = m.geo[c];
  switch (f) {
    case 0: return g.p[0][0];
    case 1: return g.p[0][1];
    case 2: return g.p[1][0] - g.p[0][0];
    case 3: return g.p[1][1] - g.p[0][1];
    case 4: return g.p[2][0] - g.p[0][0];
    case 5: return g.p[2][1] - g.p[0][1];
    case 6: return g.J;
    default: return ujh[Q * TB + (t >> 3)];
  }
}

// the thread's two targets against the nwp staged source nodes, TU per step (MASK: weights times
// wsel, 0 for a thread whose cell takes another order from this block).  Coordinates are relative
// to the target block's centre c and r2 = |x'|^2 + |y'|^2 - 2 x'.y' = fma(x0', -2y0', fma(x1', -2y1',
// |x'|^2 + |y'|^2)): 3 FP64 instructions instead of 4.  The cancellation factor (|x'| + |y'|)^2 / r2
// stays below ~3 for a uniform source block (its distance exceeds the target block's radius), so r2
// keeps a few-ulp relative accuracy.
template <int E4, bool MASK>
__device__ __forceinline__ void sweep(const double2* __restrict__ sM, const double2* __restrict__ sQ, int nwp,
                                      const double (&x0)[2], const double (&x1)[2], const double (&xx)[2],
                                      double wsel, double ex, double (&acc)[2][2]) {
#pragma unroll 1
  for (int p = 0; p < nwp; p += TU) {
    double2 my[TU], qw[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      my[u] = sM[p + u];             // (-2 y0', -2 y1')
      qw[u] = sQ[p + u];             // (|y'|^2, J w)
      if (MASK) qw[u].y *= wsel;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const double r2 = fma(x0[t], my[u].x, fma(x1[t], my[u].y, xx[t] + qw[u].x));
        acc[t][u & 1] = fma(qw[u].y, kpow<E4>(r2, ex), acc[t][u & 1]);
      }
  }
}

// The same sweep with the source weight folded into the staged coordinates (kpow_acc): sM = -2 c y',
// sQ = (c |y'|^2, c), c = (J w)^(1/ex), so r2' = c r2 = fma(x0', sM.x, fma(x1', sM.y, fma(|x'|^2, c,
// sQ.x))) and (J w) r2^ex = r2'^ex is added with the fused correction: 9 FP64 instructions per
// evaluation instead of 10.  Padding nodes sit at 1e150 with c = 1: their term underflows to an exact 0.
template <int E4>
__device__ __forceinline__ void sweep_fold(const double2* __restrict__ sM, const double2* __restrict__ sQ, int nwp,
                                           const double (&x0)[2], const double (&x1)[2], const double (&xx)[2],
                                           double ex, double (&acc)[2][2]) {
#pragma unroll 1
  for (int p = 0; p < nwp; p += TUF) {
    double2 my[TUF], qw[TUF];
#pragma unroll
    for (int u = 0; u < TUF; ++u) {
      my[u] = sM[p + u];             // (-2 c y0', -2 c y1')
      qw[u] = sQ[p + u];             // (c |y'|^2, c)
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < TUF; ++u) {
        const double r2 = fma(x0[t], my[u].x, fma(x1[t], my[u].y, fma(xx[t], qw[u].y, qw[u].x)));
        acc[t][u & 1] = kpow_acc<E4>(r2, ex, acc[t][u & 1]);
      }
  }
}

// sym4 sweep: also the column sums sum_t w_t v(t, y) of every source node y over the warp's 64
// targets (two per lane), reduced across the warp with a 4-value butterfly (lanes 0/8/16/24 end up
// with the four columns of a step) and stored per warp in colw[y]
template <int E4>
__device__ __forceinline__ void sweep_sym(const double2* __restrict__ sM, const double2* __restrict__ sQ, int nwp,
                                          const double (&x0)[2], const double (&x1)[2], const double (&xx)[2],
                                          const double (&wt)[2], double ex, double (&acc)[2][2],
                                          double* __restrict__ colw, int lane) {
#pragma unroll 1
  for (int p = 0; p < nwp; p += TU) {
    double2 my[TU], qw[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      my[u] = sM[p + u];
      qw[u] = sQ[p + u];
    }
    double c[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      double cu = 0.0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double v = kpow<E4>(fma(x0[t], my[u].x, fma(x1[t], my[u].y, xx[t] + qw[u].x)), ex);
        acc[t][u & 1] = fma(qw[u].y, v, acc[t][u & 1]);
        cu = fma(wt[t], v, cu);
      }
      c[u] = cu;
    }
    const bool h16 = lane & 16, h8 = lane & 8;
    double k0 = h16 ? c[2] : c[0], k1 = h16 ? c[3] : c[1];
    k0 += __shfl_xor_sync(0xffffffffu, h16 ? c[0] : c[2], 16);
    k1 += __shfl_xor_sync(0xffffffffu, h16 ? c[1] : c[3], 16);
    double kk = h8 ? k1 : k0;
    kk += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
    kk += __shfl_xor_sync(0xffffffffu, kk, 4);
    kk += __shfl_xor_sync(0xffffffffu, kk, 2);
    kk += __shfl_xor_sync(0xffffffffu, kk, 1);
    if ((lane & 7) == 0) colw[p + (lane >> 3)] = kk;   // lane 0: column p, 8: p + 1, 16: p + 2, 24: p + 3
  }
}

template <int E4>
__global__ void __launch_bounds__(TT, 2) tail2d_block_kernel(DevMesh m, const double* __restrict__ tab, DevTables dir,
                                                            OrderConsts oc, double ex,
                                                            const int8_t* __restrict__ kuni,
                                                            const int* __restrict__ tflag,
                                                            const int* __restrict__ run,
                                                            const int* __restrict__ tcell,
                                                            const int* __restrict__ bcells,
                                                            const int8_t* __restrict__ kcell,
                                                            const double* __restrict__ bstat,
                                                            const double2* __restrict__ un,
                                                            const double* __restrict__ uj,
                                                            const double* __restrict__ ujh,
                                                            const double* __restrict__ wh, int nb,
                                                            unsigned long long* __restrict__ psifx, double fxscale,
                                                            double* __restrict__ psi,
                                                            unsigned long long* __restrict__ evals,
                                                            unsigned long long* __restrict__ evals_sym) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sM = reinterpret_cast<double2*>(smem_raw);          // TWIN source nodes: -2 y' (centred)
  double2* sQ = sM + TWIN;                                     // TWIN: |y'|^2, J * w
  double* sR = reinterpret_cast<double*>(sQ + TWIN);           // RULE_NODES x (u0, u1, w, w^(1/(2 ex)))
  double* sG = sR + RS * RULE_NODES;                           // TB x 8 geometry fields
  double* colbuf = sG + 8 * TB;                                // [8 warps][512] sym4 column partials
  int* sL = reinterpret_cast<int*>(colbuf + (TT / 32) * (TWIN / 2));   // source blocks: Q | (k & 0xff) << 24
  __shared__ int s_wsum[TT / 32];
  __shared__ int s_nq;
  __shared__ int s_kc[TB];                                     // per target cell order (mixed blocks)
  const int P = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (!run[P]) return;
  const bool helper = !tflag[P];       // no target here: only the order-4 pairs with target blocks
  // ---- the disjoint rules k = 2..9 (reference nodes and weights)
  for (int i = tid; i < RULE_NODES; i += TT) {
    int k = 2;
    while (roff(k + 1) <= i) ++k;
    const RuleRef rr = dir.rule(T_DISJ, k);
    const int r = i - roff(k);
    if (rr.cnt == k * k) {
      const double* nd = tab + (size_t)(rr.off + r) * NODE;
      sR[RS * i] = nd[0]; sR[RS * i + 1] = nd[1]; sR[RS * i + 2] = nd[2];
      sR[RS * i + 3] = wh[i];
    } else {
      sR[RS * i] = sR[RS * i + 1] = sR[RS * i + 2] = sR[RS * i + 3] = 0.0;
    }
  }
  // ---- the source blocks of P handled here (uniform or mixed), ascending (ordered compaction)
  const int8_t* krow = kuni + (size_t)P * nb;
  if (tid == 0) s_nq = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += TT) {
    const int Q = base + tid;
    int k = Q < nb ? (int)krow[Q] : 0;
    if (k && sym4_mode(P, Q, k) < 0) k = 0;          // (Q, P) evaluated by Q's CTA for both
    if (k && helper && !(sym4_mode(P, Q, k) > 0 && tflag[Q])) k = 0;
    const unsigned bal = __ballot_sync(0xffffffffu, k != 0);
    if (lane == 0) s_wsum[wid] = __popc(bal);
    __syncthreads();
    int off = s_nq;
    for (int w = 0; w < wid; ++w) off += s_wsum[w];
    if (k) sL[off + __popc(bal & ((1u << lane) - 1u))] = Q | ((k & 0xff) << 24);
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < TT / 32; ++w) tot += s_wsum[w];
      s_nq += tot;
    }
    __syncthreads();
  }
  const int nq = s_nq;
  // ---- the thread's two target nodes: cell tid / 8, nodes tid % 8 and tid % 8 + 8
  const int cme = tid >> 3, q0 = tid & 7;
  const int Kv = bcells[P * TB + cme];               // the cell (-1: an empty slot of a partial block)
  const int Kc = Kv >= 0 && tcell[Kv] ? Kv : -1;     // ... if its psi is wanted (a target)
  const double ccx = bstat[8 * P], ccy = bstat[8 * P + 1];   // the target block's centre
  double x0[2], x1[2], xx[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    // every cell's nodes, targets or not: they are also the sources of the sym4 column sums
    x0[t] = Kv >= 0 ? m.X[((size_t)Kv * TQN + q0 + 8 * t) * 2 + 0] - ccx : -1e100;
    x1[t] = Kv >= 0 ? m.X[((size_t)Kv * TQN + q0 + 8 * t) * 2 + 1] - ccy : -1e100;
    xx[t] = fma(x1[t], x1[t], x0[t] * x0[t]);
  }
  double wt[2];                      // J_K w_q of the thread's targets (sym4 column sums; 0: no target)
#pragma unroll
  for (int t = 0; t < 2; ++t) wt[t] = Kv >= 0 ? m.geo[Kv].J * sR[RS * (roff(4) + q0 + 8 * t) + 2] : 0.0;
  int ntv = 0, nvp = 0;              // target cells / cells of the block (evaluation counts)
  if (tid == 0)
    for (int c = 0; c < TB; ++c) {
      const int K = bcells[P * TB + c];
      ntv += K >= 0 && tcell[K];
      nvp += K >= 0;
    }
  const int Kw = tid < TB ? bcells[P * TB + tid] : -1;     // thread c < 32: target cell c (orders)
  const bool Kw_t = Kw >= 0 && tcell[Kw];
  double acc[2][2] = {};
  unsigned long long nev = 0, nsy = 0;
  bool missing = false;
  // fast path: uniform order k <= 4, the whole block's 32 k^2 nodes in one half of the window
  // (node-major from the block-ordered staging array un / uj), software-pipelined: the next fast
  // block's nodes are loaded into registers before the sweep of the current one and written to the
  // other half after it — one barrier per source block
  auto kof = [&](int qi) { return (int)(int8_t)(sL[qi] >> 24); };
  auto is_fast = [&](int qi) { return qi < nq && kof(qi) >= 2 && kof(qi) <= 4; };
  double2 py[2];
  double pj[2];
  // a sym4 pair keeps plain weights J w (its kernel values also feed the column sums); every
  // other block is staged with the weight folded into the coordinates (sweep_fold)
  auto prefetch = [&](int qi) {
    const int Q = sL[qi] & 0xffffff, k = kof(qi), nn = TB * k * k;
    const double* __restrict__ jsrc = sym4_mode(P, Q, k) > 0 ? uj : ujh;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int idx = tid + TT * t;
      if (idx < nn) {
        py[t] = un[(size_t)Q * UNODES2D + useg(k) + idx];
        pj[t] = jsrc[(size_t)Q * TB + (idx & (TB - 1))];
      }
    }
  };
  auto put_nodes = [&](int qi, int half) {
    const int k = kof(qi), kk = k * k, nn = TB * kk;
    const double* R = sR + RS * roff(k);
    const bool sy4 = sym4_mode(P, sL[qi] & 0xffffff, k) > 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int idx = tid + TT * t;
      if (idx < nn) {
        const bool ok = pj[t] != 0.0;            // an empty slot of a partial block: far, weight 0
        if (sy4) {
          const double yx = (ok ? py[t].x : 1e100) - ccx, yy = (ok ? py[t].y : 1e100) - ccy;
          sM[half * (TWIN / 2) + idx] = make_double2(-2.0 * yx, -2.0 * yy);
          sQ[half * (TWIN / 2) + idx] = make_double2(fma(yy, yy, yx * yx), pj[t] * R[RS * (idx >> 5) + 2]);
        } else {
          const double yx = (ok ? py[t].x : 1e150) - ccx, yy = (ok ? py[t].y : 1e150) - ccy;
          const double sc = pj[t] * R[RS * (idx >> 5) + 3], c = ok ? sc * sc : 1.0;
          sM[half * (TWIN / 2) + idx] = make_double2(-2.0 * c * yx, -2.0 * c * yy);
          sQ[half * (TWIN / 2) + idx] = make_double2(c * fma(yy, yy, yx * yx), c);
        }
      }
    }
    if (wid == 0) {                              // evaluation count: valid source cells (lanes = row 0)
      const int nvs = __popc(__ballot_sync(0xffffffffu, pj[0] != 0.0));
      // sym4: every cell of the block is swept (its nodes are the sources of the column sums)
      const bool sy = sym4_mode(P, sL[qi] & 0xffffff, k) > 0;
      if (lane == 0) {
        nev += (unsigned long long)nvs * kk * (sy ? nvp : ntv) * TQN;
        if (sy) nsy += (unsigned long long)nvs * kk * nvp * TQN;
      }
    }
    if (tid == 0 && dir.rule(T_DISJ, k).cnt != kk) missing = true;
  };
  int half = 0;
  bool staged = false;
  for (int qi = 0; qi < nq; ++qi) {
    const int Q = sL[qi] & 0xffffff;
    const int kq = kof(qi);          // > 0: uniform, -1: per target cell
    if (is_fast(qi)) {
      if (!staged) {
        prefetch(qi);
        put_nodes(qi, half);
        __syncthreads();
      }
      const bool nf = is_fast(qi + 1);
      if (nf) prefetch(qi + 1);      // in flight during the sweep
      const bool sym = sym4_mode(P, Q, kq) > 0;
      if (sym)
        sweep_sym<E4>(sM + half * (TWIN / 2), sQ + half * (TWIN / 2), TB * 16, x0, x1, xx, wt, ex, acc,
                      colbuf + wid * (TWIN / 2), lane);
      else
        sweep_fold<E4>(sM + half * (TWIN / 2), sQ + half * (TWIN / 2), TB * kq * kq, x0, x1, xx, ex, acc);
      if (nf) put_nodes(qi + 1, half ^ 1);
      __syncthreads();
      if (sym) {
        // Q's target nodes: node r of cell c (node-major idx = 32 r + c) is Q's XQ node r; the 8
        // warps' partials summed in a fixed order, added to Q's psi in exact fixed point
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int idx = tid + TT * t, c = idx & (TB - 1), r = idx >> 5;
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < TT / 32; ++w) v += colbuf[w * (TWIN / 2) + idx];
          const int Kq = bcells[Q * TB + c];
          if (Kq >= 0) atomicAdd(psifx + (size_t)Kq * TQN + r, (unsigned long long)__double2ll_rn(v * fxscale));
        }
        __syncthreads();               // colbuf consumed
      }
      staged = nf;
      if (nf) half ^= 1;
      continue;
    }
    staged = false;
    // general path: order >= 5 (windows) or per-target-cell orders; geometry through sG
    sG[tid] = geo_field(m, bcells, ujh, Q, tid);
    if (kq < 0 && tid < TB) s_kc[tid] = Kw_t ? (int)kcell[(size_t)Kw * nb + Q] : 0;
    __syncthreads();
    unsigned kset;                   // bit k: some target cell takes order k from this block here
    if (kq > 0) {
      kset = 1u << kq;
    } else {
      kset = 0;
      for (int c = 0; c < TB; ++c) kset |= (1u << s_kc[c]);
      kset &= ~1u;                   // order 0: that cell leaves the block to the warp tail
    }
    const int kmine = kq > 0 ? kq : s_kc[cme];
    for (unsigned ks = kset; ks; ks &= ks - 1) {
      const int k = __ffs(ks) - 1, kk = k * k;
      if (tid == 0 && dir.rule(T_DISJ, k).cnt != kk) missing = true;
      int ntk = ntv;                 // target cells evaluated at order k
      if (kq < 0 && tid == 0) {
        ntk = 0;
        for (int c = 0; c < TB; ++c) ntk += s_kc[c] == k;
      }
      // warps with none of their 4 cells at order k skip the sweep; a thread of such a warp
      // whose own cell is at another order adds exact zeros (weight 0)
      const bool wact = __any_sync(0xffffffffu, kmine == k);
      const double wsel = kmine == k ? 1.0 : 0.0;
      const double* R = sR + RS * roff(k);
      const int cpw = TWIN / kk;     // cells per window (>= 12)
      for (int c0 = 0; c0 < TB; c0 += cpw) {
        const int c1 = min(TB, c0 + cpw), nw = (c1 - c0) * kk, nwp = (nw + 7) / 8 * 8;
        if (c0 > 0 || ks != kset) __syncthreads();
        const double far = kq > 0 ? 1e150 : 1e100;
        for (int idx = tid; idx < nwp; idx += TT) {
          double2 y = make_double2(far, far);       // padding: far away, weight 0 (folded: c = 1)
          double w = kq > 0 ? 1.0 : 0.0;
          if (idx < nw) {
            const int c = c0 + idx / kk, r = idx - (idx / kk) * kk;
            const double* g = sG + 8 * c;
            if (g[7] != 0.0) {
              const double u0 = R[RS * r], u1 = R[RS * r + 1];
              y.x = g[0] + (u0 * g[2] + u1 * g[4]);
              y.y = g[1] + (u0 * g[3] + u1 * g[5]);
              const double sc = g[7] * R[RS * r + 3];
              w = kq > 0 ? sc * sc : g[6] * R[RS * r + 2];
            }
          }
          const double yx = y.x - ccx, yy = y.y - ccy;
          if (kq > 0) {                             // uniform order: weight folded (sweep_fold)
            sM[idx] = make_double2(-2.0 * w * yx, -2.0 * w * yy);
            sQ[idx] = make_double2(w * fma(yy, yy, yx * yx), w);
          } else {
            sM[idx] = make_double2(-2.0 * yx, -2.0 * yy);
            sQ[idx] = make_double2(fma(yy, yy, yx * yx), w);
          }
        }
        if (tid == 0) {
          int nvs = 0;
          for (int c = c0; c < c1; ++c) nvs += sG[8 * c + 7] != 0.0;
          nev += (unsigned long long)nvs * kk * ntk * TQN;
        }
        __syncthreads();
        if (!wact) continue;
        if (kq > 0) sweep_fold<E4>(sM, sQ, nwp, x0, x1, xx, ex, acc);
        else sweep<E4, true>(sM, sQ, nwp, x0, x1, xx, wsel, ex, acc);
      }
    }
    __syncthreads();                 // the window is consumed before the next block reuses it
  }
  if (Kc >= 0) {
#pragma unroll
    for (int t = 0; t < 2; ++t) psi[(size_t)Kc * TQN + q0 + 8 * t] = acc[t][0] + acc[t][1];
  }
  if (tid == 0) {
    if (missing) atomicOr(m.err, 1);
    if (evals && nev) atomicAdd(evals, nev);
    if (evals_sym && nsy) atomicAdd(evals_sym, nsy);
  }
}

#define FL_E4_SWITCH_T(e4, ...)                               \
  switch (e4) {                                               \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

}  // namespace

void launch_tail2d_blocks(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                          const Blocks2D& B, const int* targets, int ntargets, double* psi,
                          unsigned long long* evals, cudaStream_t st, unsigned long long* evals_block,
                          cudaEvent_t e0, cudaEvent_t e1, unsigned long long* evals_sym) {
  if (ntargets <= 0) return;
  const int nb = B.nb;
  const size_t smem = (size_t)TWIN * 32 + (size_t)(TT / 32) * (TWIN / 2) * 8 + (size_t)RS * RULE_NODES * 8 + (size_t)8 * TB * 8 + (size_t)nb * 4;
  if (m.d != 2 || m.q != TQN || smem > 200 * 1024) {      // out of this path's shape: pair by pair
    launch_tail(m, t, oc, ex, e4, targets, ntargets, psi, evals, st);
    return;
  }
  DBuf<int> tflag(nb), tcell(m.nc);
  FL_CUDA(cudaMemsetAsync(tflag.p, 0, (size_t)nb * sizeof(int), st));
  FL_CUDA(cudaMemsetAsync(tcell.p, 0, (size_t)m.nc * sizeof(int), st));
  tail_flag_kernel<<<(ntargets + 255) / 256, 256, 0, st>>>(targets, ntargets, B.blk_of.p, tflag.p, tcell.p),
      note_launch();
  DBuf<int> run(nb);                   // CTAs that run: target blocks and sym4 helpers
  FL_CUDA(cudaMemcpyAsync(run.p, tflag.p, (size_t)nb * sizeof(int), cudaMemcpyDeviceToDevice, st));
  DBuf<int8_t> kuni((size_t)nb * nb);
  const int64_t nn = (int64_t)nb * nb;
  // FRACLAP_TAIL2D_MIXED=1: disjoint non-uniform block pairs split per target cell (measured slower
  // at c5: the masked two-order sweeps cost what the warp tail does)
  static const bool mixed = [] {
    const char* v = getenv("FRACLAP_TAIL2D_MIXED");
    return v && std::string(v) == "1";
  }();
  // smallest block distance of the order-4 uniform pairs and the largest Jacobian: the bound of the
  // sym4 column sums that sets the fixed-point scale of psifx
  DBuf<unsigned long long> red(2);
  {
    const double big = 1e300;
    unsigned long long init[2] = {0ull, 0ull};
    std::memcpy(&init[0], &big, 8);
    FL_CUDA(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  tail_kuni_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(oc, B.bstat.p, tflag.p, nb, mixed ? 1 : 0, kuni.p,
                                                                 red.p, run.p),
      note_launch();
  // FRACLAP_EXACT_RANGE=0: circle bounds only (round-2 behaviour before the exact ranges)
  static const bool exact_range = [] {
    const char* v = getenv("FRACLAP_EXACT_RANGE");
    return !(v && std::string(v) == "0");
  }();
  if (exact_range && !mixed)
    tail_refine_kernel<<<(unsigned)((nn * 32 + 255) / 256), 256, 0, st>>>(oc, m, B.bcells.p, B.bstat.p, tflag.p, nb,
                                                                          kuni.p, red.p, run.p),
        note_launch();
  const double jmax = B.jmax;
  jsum_kernel<<<(m.nc + 255) / 256, 256, 0, st>>>(m, jmax > 0.0 ? std::ldexp(1.0, 30) / jmax : 0.0, red.p + 1),
      note_launch();
  unsigned long long hred[2];
  FL_CUDA(cudaMemcpyAsync(hred, red.p, sizeof(hred), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  double dmin4;
  std::memcpy(&dmin4, &hred[0], 8);
  // |column sum| <= sum_K J_K / 2 * dmin4^(2 ex) (every target cell at most once per source node, at
  // least dmin4 away; sum_K J_K / 2 = the area of the mesh, summed in integer units rounded up);
  // scale: that -> 2^60
  double fxscale = 1.0;
  if (dmin4 < 1e299 && jmax > 0.0) {
    const double jsum = (double)hred[1] * jmax * std::ldexp(1.0, -30) * (1.0 + 1e-9);
    const double bound = jsum * 0.5 * std::pow(dmin4, 2.0 * ex);
    int S = 60 - (int)std::ceil(std::log2(std::max(bound, 1e-300)));
    S = std::max(-1000, std::min(1000, S));
    fxscale = std::ldexp(1.0, S);
  }
  DBuf<unsigned long long> psifx((size_t)m.nc * TQN);
  FL_CUDA(cudaMemsetAsync(psifx.p, 0, (size_t)m.nc * TQN * sizeof(unsigned long long), st));
  // per target cell orders of the mixed block pairs (read by both tail kernels: one decision)
  DBuf<int8_t> kcell(mixed ? (size_t)m.nc * nb : 1);
  if (mixed) {
    const int64_t nt = (int64_t)ntargets * nb;
    tail_kcell_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(oc, m, targets, ntargets, B.blk_of.p, kuni.p,
                                                                    B.bstat.p, nb, kcell.p),
        note_launch();
  }
  const double hex = 0.5 / ex;         // exponent of the folded weight factors
  DBuf<double> ujh((size_t)nb * TB);
  DBuf<double> wh(RULE_NODES);
  fold_slots_kernel<<<(nb * TB + 255) / 256, 256, 0, st>>>(m, B.bcells.p, nb * TB, hex, ujh.p), note_launch();
  fold_rules_kernel<<<(RULE_NODES + 255) / 256, 256, 0, st>>>(t.data, t, hex, wh.p), note_launch();
  // orders 5-9 staged for the warp tail (130 KB per block; skipped beyond 8 GB: it then maps per pair)
  DBuf<double2> uhi;
  if ((size_t)nb * UHI2D * sizeof(double2) <= ((size_t)8 << 30) && oc.cap_disjoint <= 9) {
    uhi.alloc((size_t)nb * UHI2D);
    hi_nodes_kernel<<<(unsigned)(((int64_t)nb * UHI2D + 255) / 256), 256, 0, st>>>(m, B.bcells.p, nb, t.data, t, uhi.p),
        note_launch();
  }
  if (e0) FL_CUDA(cudaEventRecord(e0, st));
  FL_E4_SWITCH_T(e4, {
    FL_CUDA(cudaFuncSetAttribute(tail2d_block_kernel<E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    tail2d_block_kernel<E4><<<nb, TT, smem, st>>>(m, t.data, t, oc, ex, kuni.p, tflag.p, run.p, tcell.p, B.bcells.p,
                                                  kcell.p, B.bstat.p, B.un.p, B.uj.p, ujh.p, wh.p, nb, psifx.p, fxscale, psi,
                                                  evals_block ? evals_block : evals, evals_sym),
        note_launch();
  });
  FL_CHECK_LAUNCH();
  if (e1) FL_CUDA(cudaEventRecord(e1, st));
  launch_tail(m, t, oc, ex, e4, targets, ntargets, psi, evals, st, kuni.p, B.blk_of.p, B.bcells.p, nb, kcell.p,
              psifx.p, 1.0 / fxscale, ujh.p, wh.p, B.un.p, uhi.p);
}

}  // namespace fl
