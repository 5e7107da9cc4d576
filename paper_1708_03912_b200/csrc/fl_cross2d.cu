// 2D disjoint cross term (cross_matrices, assembly.py:172-229, scattered by _cross_triplets
// :693-725) by CELL-BLOCK PAIRS with exact fixed-point accumulation.
//
// Layout.  The cells are sorted along a Morton curve of their centroids and cut into blocks of
// CB = 32 cells; every block keeps the sorted list of the DoFs of its cells (<= BRMAX) and each
// cell the local slot of its vertices in that list.  A CTA owns one unordered block pair
// {P, Q} (P <= Q) at a time (persistent queue, heaviest pairs first):
//   (A) the Gauss order of its <= 1024 cell pairs (select_order, quadrature.py:138-179; the
//       fast fp32 path with the exact fp64 fallback, or one order for the whole block pair
//       when rigorous bounds of the order formula agree), touching pairs skipped;
//   (B) every disjoint pair evaluated ONCE: k = 2, 3, 4 one thread per pair with the mapped
//       nodes of both cells staged in shared memory (heaviest orders first), k >= 5 (rare,
//       near pairs) looked up from the near-block table computed by fl_near.cu;
//   (C) -C * M^{K,L} added into an int64 tile of the block pair's DoF rectangle in shared
//       memory, and the tile (plus its transpose for P != Q) added into A with 64-bit integer
//       atomics.
// Determinism.  Every contribution is converted to a fixed-point integer with a global scale
// 2^S chosen from a rigorous bound of the largest entry (S leaves ~2^8 headroom); integer
// addition is associative, so every entry is the exact sum of its rounded contributions in
// ANY order: bitwise reproducible run to run, and identical for any split of the rows over
// GPUs (a rank processes the block pairs touching its rows and keeps only its rows).  The
// resolution is ~2^-54 of the bound — finer than an fp64 ulp of the largest entries.  No cell
// pair is evaluated twice (the DoF-tile kernel of round 1 recomputed ~1.5x at the halo).
#include <cstring>

#include <chrono>
#include <cstdio>
#include <cub/cub.cuh>

#include "fl_internal.h"

namespace fl {

namespace {

constexpr int CB = CB2D;          // cells per block
constexpr int BRMAX = 64;         // DoFs per block (more: the mesh is refused by this path)
constexpr int TCAP = 48 * 48;     // int64 tile capacity; larger rectangles go straight to HBM
constexpr int X2T = 256;          // threads per CTA
constexpr int NPRE2 = 29;         // mapped nodes per cell: k = 2, 3, 4 (4 + 9 + 16)
__host__ __device__ constexpr int poff(int k) { return k == 2 ? 0 : (k == 3 ? 4 : 13); }

struct XRec {                     // per staged cell: order inputs
  double cx, cy, rad, J;
  float lnh, lh;
  int id, pad;
};

struct XShared {
  double2 nd[2 * CB][NPRE2];      // mapped nodes (absolute coordinates, as _map_points)
  unsigned long long tile[TCAP];
  XRec r[2 * CB];
  double wl[NPRE2][3];            // w * lambda_a of the rules k = 2, 3, 4
  int dofP[BRMAX], dofQ[BRMAX];
  signed char sl[2 * CB][3];      // local DoF slot of each staged cell's vertices
  unsigned short plist[CB * CB];
  unsigned char pk[CB * CB];
  int hist[8], cursor[8];
  short chs[CB * CB / 4 + 8];       // chunks of same-order pairs: start in plist, count, order
  unsigned char chn[CB * CB / 4 + 8], chk[CB * CB / 4 + 8];
  int nchunk;
  int bp, nP, nQ, q;
  unsigned long long evals;
};

// ---------------------------------------------------------------- preparation
__device__ __forceinline__ uint32_t spread16b(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
__global__ void cell_morton_kernel(DevMesh m, double x0, double y0, double sx, double sy, uint32_t* keys,
                                   int* vals) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m.nc) return;
  const CellGeo& g = m.geo[c];
  const uint32_t qx = (uint32_t)fmin(fmax((g.cx - x0) * sx, 0.0), 65535.0);
  const uint32_t qy = (uint32_t)fmin(fmax((g.cy - y0) * sy, 0.0), 65535.0);
  keys[c] = spread16b(qx) | (spread16b(qy) << 1);
  vals[c] = c;
}

// one CTA (128 threads) per block: cells, sorted DoF list, vertex slots, block statistics
__global__ void __launch_bounds__(128) block_build_kernel(DevMesh m, const int* __restrict__ sorted, int nb,
                                                          int r0, int r1, int* __restrict__ bcells,
                                                          int* __restrict__ bdofs, int* __restrict__ bndof,
                                                          signed char* __restrict__ slot, double* __restrict__ bstat,
                                                          int* __restrict__ rowflag, int* __restrict__ err) {
  const int b = blockIdx.x, t = threadIdx.x;
  __shared__ int key[128];
  __shared__ int list[128];
  __shared__ int nu, cells[CB];
  if (t < CB) {
    const int i = b * CB + t;
    cells[t] = i < m.nc ? sorted[i] : -1;
    bcells[b * CB + t] = cells[t];
  }
  __syncthreads();
  key[t] = 0x7fffffff;
  if (t < 3 * CB) {
    const int c = cells[t / 3];
    if (c >= 0) {
      const int dof = m.geo[c].dof[t % 3];
      if (dof >= 0) key[t] = dof;
    }
  }
  __syncthreads();
  for (int k = 2; k <= 128; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int ixj = t ^ j;
      if (ixj > t) {
        const bool up = (t & k) == 0;
        const int a = key[t], c = key[ixj];
        if ((a > c) == up) { key[t] = c; key[ixj] = a; }
      }
      __syncthreads();
    }
  if (t == 0) {
    int u = 0;
    for (int i = 0; i < 128 && key[i] != 0x7fffffff; ++i)
      if (i == 0 || key[i] != key[i - 1]) list[u++] = key[i];
    nu = u;
    if (u > BRMAX) atomicAdd(err, 1);
    bndof[b] = min(u, BRMAX);
  }
  __syncthreads();
  const int n = min(nu, BRMAX);
  if (t < BRMAX) bdofs[b * BRMAX + t] = t < n ? list[t] : -1;
  if (t < 3 * CB) {
    const int c = cells[t / 3];
    if (c >= 0) {
      const int dof = m.geo[c].dof[t % 3];
      int s = -1;
      for (int i = 0; i < n; ++i)
        if (list[i] == dof) s = i;
      slot[c * 3 + t % 3] = (signed char)(dof >= 0 ? s : -1);
    }
  }
  if (t == 0) {
    int fl = 0;
    for (int i = 0; i < n; ++i) fl |= (list[i] >= r0 && list[i] < r1);
    rowflag[b] = fl;
    double cx = 0, cy = 0;
    int cnt = 0;
    for (int i = 0; i < CB; ++i)
      if (cells[i] >= 0) { cx += m.geo[cells[i]].cx; cy += m.geo[cells[i]].cy; ++cnt; }
    cx /= max(cnt, 1);
    cy /= max(cnt, 1);
    double R = 0, hmn = 1e300, hmx = 0, lmn = 1e300, lmx = 0;
    for (int i = 0; i < CB; ++i) {
      if (cells[i] < 0) continue;
      const CellGeo& g = m.geo[cells[i]];
      const double dx = g.cx - cx, dy = g.cy - cy;
      R = fmax(R, sqrt(dx * dx + dy * dy) * (1.0 + 1e-12) + g.rad);
      hmn = fmin(hmn, g.diam); hmx = fmax(hmx, g.diam);
      lmn = fmin(lmn, g.ldiam); lmx = fmax(lmx, g.ldiam);
    }
    double* st = bstat + 8 * b;
    st[0] = cx; st[1] = cy; st[2] = R * (1.0 + 1e-12); st[3] = hmn; st[4] = hmx; st[5] = lmn; st[6] = lmx; st[7] = 0;
  }
}

__global__ void block_of_kernel(const int* __restrict__ sorted, int nc, int* __restrict__ blk_of) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) blk_of[sorted[i]] = i / CB;
}

// mapped nodes of the rules k = 2, 3, 4 for every cell: X = P0 + (u0 (P1 - P0) + u1 (P2 - P0))
__global__ void cell_nodes2_kernel(DevMesh m, const double* __restrict__ tab, RuleRef r2, RuleRef r3, RuleRef r4,
                                   double2* __restrict__ nodes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)m.nc * NPRE2) return;
  const int c = (int)(i / NPRE2), x = (int)(i % NPRE2);
  const RuleRef rr = x < 4 ? r2 : (x < 13 ? r3 : r4);
  const int xl = x < 4 ? x : (x < 13 ? x - 4 : x - 13);
  const double* nd = tab + (size_t)(rr.off + xl) * NODE;
  const CellGeo& g = m.geo[c];
  const double X0 = g.p[0][0] + (nd[0] * (g.p[1][0] - g.p[0][0]) + nd[1] * (g.p[2][0] - g.p[0][0]));
  const double X1 = g.p[0][1] + (nd[0] * (g.p[1][1] - g.p[0][1]) + nd[1] * (g.p[2][1] - g.p[0][1]));
  nodes[i] = make_double2(X0, X1);
}

// Bound of the largest cross entry: the closest disjoint cell to K lies in its second ring (a
// segment from K to any cell not sharing a vertex with K leaves the star of K through an edge
// whose outer cell is in that ring), so dmin = min over K of the exact distance to its
// second-ring disjoint cells bounds every disjoint pair's node distance from below.
__global__ void dmin_kernel(DevMesh m, unsigned long long* __restrict__ dmin_bits,
                            unsigned long long* __restrict__ jmax_bits, unsigned long long* __restrict__ rmax_bits,
                            double e, unsigned long long* __restrict__ beta_bits) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K >= m.nc) return;
  const CellGeo& A = m.geo[K];
  atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(A.rad));
  double best = 1e300;
  for (int a = 0; a < 3; ++a) {
    const int v = A.v[a];
    for (int p = m.patch_off[v]; p < m.patch_off[v + 1]; ++p) {
      const CellGeo& N = m.geo[m.patch_cells[p]];
      for (int b = 0; b < 3; ++b) {
        const int u = N.v[b];
        for (int q = m.patch_off[u]; q < m.patch_off[u + 1]; ++q) {
          const int L = m.patch_cells[q];
          const CellGeo& B = m.geo[L];
          if (touching<2>(A, B)) continue;
          best = fmin(best, exact_tri_dist(A, B));
        }
      }
    }
  }
  // beta = max over the cells of J_K^2 d_K^(-(d+2s)), d_K = best: a disjoint pair (K, L) lies at least
  // max(d_K, d_L) apart (the segment between them leaves the star of either cell through its second
  // ring), so J_K J_L dist^(-e) <= sqrt(J_K^2 d_K^(-e) J_L^2 d_L^(-e)) <= beta — tighter than
  // Jmax^2 dmin^(-e) on graded meshes
  if (best < 1e300) {
    atomicMin(dmin_bits, (unsigned long long)__double_as_longlong(best));
    atomicMax(beta_bits, (unsigned long long)__double_as_longlong(A.J * A.J * pow(best, -e)));
  }
  atomicMax(jmax_bits, (unsigned long long)__double_as_longlong(A.J));
}

__device__ __forceinline__ double bound_hi(const OrderConsts& oc, double Dmin, double hmn, double hmx, double lmn,
                                           double lmx) {
  return order_bound_hi(oc, oc.coff, Dmin, hmn, hmx, lmn, lmx);
}
__device__ __forceinline__ double bound_lo(const OrderConsts& oc, double Dmin, double Dmax, double hmn, double hmx,
                                           double lmn, double lmx) {
  return order_bound_lo(oc, oc.coff, Dmin, Dmax, hmn, hmx, lmn, lmx);
}

__global__ void block_pairs_kernel(OrderConsts oc, const double* __restrict__ bs, const int* __restrict__ rowflag,
                                   int nb, int full, int64_t ncand, int4* __restrict__ pairs,
                                   unsigned* __restrict__ key, int* __restrict__ keep, int* __restrict__ nearflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncand) return;
  // row-major upper triangle (P <= Q)
  const double qq = 2.0 * nb + 1.0;
  int P = (int)((qq - sqrt(qq * qq - 8.0 * (double)i)) * 0.5);
  auto cum = [&](int64_t e) { return e * nb - e * (e - 1) / 2; };
  while (P > 0 && cum(P) > i) --P;
  while (cum(P + 1) <= i) ++P;
  const int Q = P + (int)(i - cum(P));
  const double* a = bs + 8 * P;
  const double* b = bs + 8 * Q;
  const double dc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
  const double Dmin = (dc - a[2] - b[2]) * (1.0 - 1e-12) - 1e-300;
  const double Dmax = (dc + a[2] + b[2]) * (1.0 + 1e-12);
  const double hmn = fmin(a[3], b[3]), hmx = fmax(a[4], b[4]), lmn = fmin(a[5], b[5]), lmx = fmax(a[6], b[6]);
  int kuni = 0;
  const double hi = bound_hi(oc, Dmin, hmn, hmx, lmn, lmx);
  if (P != Q && Dmin > 0.0) {
    const double lo = bound_lo(oc, Dmin, Dmax, hmn, hmx, lmn, lmx);
    const double c0 = fmin(fmax(ceil(lo - 1e-9), 2.0), (double)oc.cap_disjoint);
    const double c1 = fmin(fmax(ceil(hi + 1e-9), 2.0), (double)oc.cap_disjoint);
    if (c0 == c1) kuni = (int)c0;
  }
  pairs[i] = make_int4(P, Q, kuni, 0);
  keep[i] = full ? 1 : (rowflag[P] | rowflag[Q]);
  nearflag[i] = (kuni == 0 && hi + 1e-9 > (double)(KW2D - 1)) || kuni >= KW2D ? 1 : 0;
  key[i] = __float_as_uint((float)fmax(Dmin, 0.0));      // heavy first: ascending gap
}

// The disjoint block pairs the circle bounds left open (kuni == 0) get a second try with the exact
// range of their 32 x 32 pairs' distance estimates (block_pair_dist_range): a warp per pair.
__global__ void cross_refine_kernel(OrderConsts oc, DevMesh m, const int* __restrict__ bcells,
                                    const double* __restrict__ bs, int64_t ncand, int4* __restrict__ pairs,
                                    int* __restrict__ nearflag) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncand) return;
  const int4 p = pairs[w];
  if (p.z != 0 || p.x == p.y) return;
  const double* a = bs + 8 * p.x;
  const double* b = bs + 8 * p.y;
  const double dc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
  const double Dmin = (dc - a[2] - b[2]) * (1.0 - 1e-12) - 1e-300;
  if (!(Dmin > 0.0)) return;
  double lo, hi;
  block_pair_dist_range(m, bcells, p.x, p.y, lane, lo, hi);
  const int k = block_uniform_order(oc, oc.coff, lo * (1.0 - 1e-12) - 1e-300, hi * (1.0 + 1e-12), a, b);
  if (k == 0 || lane) return;
  pairs[w].z = k;
  nearflag[w] = k >= KW2D ? 1 : 0;
}

__global__ void clear_kuni_kernel(int4* __restrict__ pairs, int* __restrict__ nearflag, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pairs[i].z = 0;
  nearflag[i] = 1;          // any pair may hold near pairs: the discovery pass looks at all of them
}

// 64-bit fixed-point add into a shared-memory tile word with two native 32-bit shared atomics
// (a 64-bit shared atomicAdd compiles to a compare-and-swap loop): the low words add modulo 2^32
// and the carry read from the returned old value goes into the high word, so once every add has
// landed the word holds the exact 64-bit sum, whatever the order.
__device__ __forceinline__ void tile_add(unsigned long long* w, unsigned long long q) {
  unsigned* p = reinterpret_cast<unsigned*>(w);
  const unsigned ql = (unsigned)q, qh = (unsigned)(q >> 32);
  const unsigned old = atomicAdd(p, ql);
  const unsigned hi = qh + ((unsigned)(old + ql) < old ? 1u : 0u);
  if (hi) atomicAdd(p + 1, hi);
}

// ---------------------------------------------------------------- the block-pair kernel
// Partial 3x3 block of one cell pair from the lane's NX x nodes x0, x0 + XS, ... (node
// coordinates and w*lambda staged in shared memory): each y node and its weights are loaded
// once and used for the NX x nodes.
template <int E4, int NN, int NX, int XS>
__device__ __forceinline__ void blk_part(const double2* __restrict__ Xn, const double2* __restrict__ Yn,
                                         const double (*__restrict__ w)[3], int x0, double ex, double (&M)[3][3]) {
  double X0[NX], X1[NX], t[NX][3];
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const int x = min(x0 + u * XS, NN - 1);
    X0[u] = Xn[x].x;
    X1[u] = Xn[x].y;
    t[u][0] = t[u][1] = t[u][2] = 0.0;
  }
#pragma unroll(NN <= 4 ? NN : 3)
  for (int y = 0; y < NN; ++y) {
    const double2 Y = Yn[y];
    const double w0 = w[y][0], w1 = w[y][1], w2 = w[y][2];
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const double d0 = X0[u] - Y.x, d1 = X1[u] - Y.y;
      const double v = kpow<E4>(fma(d1, d1, d0 * d0), ex);
      t[u][0] = fma(v, w0, t[u][0]);
      t[u][1] = fma(v, w1, t[u][1]);
      t[u][2] = fma(v, w2, t[u][2]);
    }
  }
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    if (x0 + u * XS >= NN) continue;
    const int x = x0 + u * XS;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      M[a][0] = fma(w[x][a], t[u][0], M[a][0]);
      M[a][1] = fma(w[x][a], t[u][1], M[a][1]);
      M[a][2] = fma(w[x][a], t[u][2], M[a][2]);
    }
  }
}

struct XArgs {
  DevMesh m;
  OrderConsts oc;
  double ex, cs;                      // cs = -C * 2^S
  double lim;                         // |scaled contribution| must stay below this (headroom check)
  const int* bcells;
  const int* bdofs;
  const int* bndof;
  const signed char* slot;
  const double2* nodes;
  const int4* bpairs;
  int nbp;
  int* queue;
  unsigned long long* A;              // int64 view of the rank's rows [r0, r1) (leading dim lda)
  int64_t lda;
  int r0, r1;
  unsigned long long* evals;
  int* ovf;
  // near pairs (k >= KW2D): discovery output or the precomputed table
  unsigned long long* near_keys;
  unsigned int* near_count;
  unsigned int near_cap;
  const unsigned long long* nearH;
  const int* nearI;
  unsigned long long hmask;
  const double* nearG;
};

#ifndef FL_X2_MINB
#define FL_X2_MINB 3
#endif
template <int E4, bool DISC>
__global__ void __launch_bounds__(X2T, FL_X2_MINB) cross2d_kernel(XArgs a, const double* __restrict__ wl_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  XShared& S = *reinterpret_cast<XShared*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  const OrderConsts& oc = a.oc;
  if (!DISC && (*a.ovf & 2)) return;             // fixed-point unit too coarse for this mesh (coarse_flag_kernel)
  for (int i = tid; i < NPRE2 * 3; i += X2T) (&S.wl[0][0])[i] = wl_g[i];
  if (tid == 0) S.evals = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) S.bp = atomicAdd(a.queue, 1);
    __syncthreads();
    const int bp = S.bp;
    if (bp >= a.nbp) break;
    const int4 pr = a.bpairs[bp];
    const int P = pr.x, Q = pr.y, kuni = pr.z;
    const bool diag = P == Q;
    // ---- stage the two blocks
    if (tid < 2 * CB) {
      const int c = a.bcells[(tid < CB ? P : Q) * CB + (tid & (CB - 1))];
      XRec r;
      r.id = c;
      if (c >= 0) {
        const CellGeo& g = a.m.geo[c];
        r.cx = g.cx; r.cy = g.cy; r.rad = g.rad; r.J = g.J;
        r.lnh = __logf((float)g.diam); r.lh = (float)g.ldiam;
        for (int v = 0; v < 3; ++v) S.sl[tid][v] = a.slot[c * 3 + v];
      } else {
        r.cx = r.cy = r.rad = r.J = 0.0; r.lnh = r.lh = 0.f;
        for (int v = 0; v < 3; ++v) S.sl[tid][v] = -1;
      }
      S.r[tid] = r;
    }
    if (tid == 0) { S.nP = a.bndof[P]; S.nQ = a.bndof[Q]; S.q = 0; }
    if (tid < BRMAX) { S.dofP[tid] = a.bdofs[P * BRMAX + tid]; S.dofQ[tid] = a.bdofs[Q * BRMAX + tid]; }
    if (tid < 8) S.hist[tid] = 0;
    __syncthreads();
    const int nP = S.nP, nQ = S.nQ;
    const bool in_tile = nP * nQ <= TCAP;
    if (!DISC) {
      for (int i = tid; i < 2 * CB * NPRE2; i += X2T) {
        const int c = S.r[i / NPRE2].id;
        if (c >= 0) S.nd[i / NPRE2][i % NPRE2] = a.nodes[(int64_t)c * NPRE2 + i % NPRE2];
      }
      if (in_tile)
        for (int i = tid; i < nP * nQ; i += X2T) S.tile[i] = 0ull;
    }
    __syncthreads();
    // contribution of pair (row cell i of P, column cell j of Q), M in the reference's (min, max)
    // orientation: entry (slot of i's vertex a, slot of j's vertex b) gets M[a][b] if i is the min cell
    auto put = [&](int i, int j, bool imin, const double (&M)[3][3]) {
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) {
          const int si = S.sl[i][imin ? x : y], sj = S.sl[CB + j][imin ? y : x];
          if (si < 0 || sj < 0) continue;
          const double v = M[x][y] * a.cs;
          if (!(fabs(v) < a.lim)) atomicOr(a.ovf, 1);
          const unsigned long long q = (unsigned long long)__double2ll_rn(v);
          if (in_tile) {
            tile_add(&S.tile[si * nQ + sj], q);
            if (diag) tile_add(&S.tile[sj * nQ + si], q);
          } else {
            const int gi = S.dofP[si], gj = S.dofQ[sj];
            if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
            if (gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
          }
        }
    };
    if (!DISC && kuni >= 2 && kuni < KW2D) {
      // ---- one order for the whole block pair (disjoint blocks): no per-pair orders, no sort.
      // A warp takes one row cell i and the 32 column cells j (lane), so the row cell's nodes
      // are broadcast loads; each lane computes its whole pair in registers (the row cell's x
      // nodes NX at a time against the column cell's y nodes).
      const int k = kuni;
      unsigned long long my = 0;
      const int wid = tid >> 5;
#pragma unroll 1
      for (int i = wid; i < CB; i += X2T / 32) {
        const int j = lane;
        if (S.r[i].id < 0 || S.r[CB + j].id < 0) continue;
        const double2* Xn = S.nd[i];
        const double2* Yn = S.nd[CB + j];
        double M[3][3] = {};
        if (k == 2) {
          blk_part<E4, 4, 4, 1>(Xn + poff(2), Yn + poff(2), S.wl + poff(2), 0, a.ex, M);
        } else if (k == 3) {
#pragma unroll 1
          for (int xs = 0; xs < 3; ++xs) blk_part<E4, 9, 3, 3>(Xn + poff(3), Yn + poff(3), S.wl + poff(3), xs, a.ex, M);
        } else {
#pragma unroll 1
          for (int xs = 0; xs < 4; ++xs) blk_part<E4, 16, 4, 4>(Xn + poff(4), Yn + poff(4), S.wl + poff(4), xs, a.ex, M);
        }
        const double JJ = S.r[i].J * S.r[CB + j].J;
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) M[x][y] *= JJ;
        put(i, j, true, M);
        my += (unsigned long long)(k * k) * (k * k);
      }
      if (my) atomicAdd(&S.evals, my);
      __syncthreads();
      if (in_tile) {
        for (int idx = tid; idx < nP * nQ; idx += X2T) {
          const unsigned long long q = S.tile[idx];
          if (!q) continue;
          const int r = idx / nQ, c = idx - r * nQ;
          const int gi = S.dofP[r], gj = S.dofQ[c];
          if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
          if (gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
        }
      }
      continue;
    }
    // ---- (A) orders
    for (int p = tid; p < CB * CB; p += X2T) {
      const int i = p / CB, j = p % CB;
      const XRec& rK = S.r[i];
      const XRec& rL = S.r[CB + j];
      int k = 0;
      if (rK.id >= 0 && rL.id >= 0 && (!diag || i < j)) {
        if (kuni) {
          k = kuni;
        } else {
          k = order2d_fast(oc, rK.cx - rL.cx, rK.cy - rL.cy, rK.rad, rL.rad, rK.lnh, rK.lh, rL.lnh, rL.lh);
          if (k == 0) {
            const CellGeo& gK = a.m.geo[rK.id];
            const CellGeo& gL = a.m.geo[rL.id];
            if (!touching<2>(gK, gL)) {
              const CellGeo& lo = rK.id < rL.id ? gK : gL;
              const CellGeo& hi = rK.id < rL.id ? gL : gK;
              k = order_disjoint_fast(oc, oc.coff, lo, hi, dist_estimate<2>(lo, hi));
            }
          }
        }
      }
      if (k >= KW2D) {
        const unsigned long long key = near_key(rK.id, rL.id, k);
        if (DISC) {
          const unsigned am = __activemask();
          const int leader = __ffs(am) - 1;
          unsigned int base = 0;
          if (lane == leader) base = atomicAdd(a.near_count, (unsigned)__popc(am));
          base = __shfl_sync(am, base, leader);
          const unsigned int slotn = base + __popc(am & ((1u << lane) - 1u));
          if (slotn < a.near_cap) a.near_keys[slotn] = key;
        } else {
          unsigned long long h = near_hash(key) & a.hmask, hk;
          while ((hk = a.nearH[h]) != key && hk != NEAR_EMPTY) h = (h + 1) & a.hmask;
          int64_t lo = 0;
          if (hk == key) lo = a.nearI[h];
          else atomicOr(a.m.err, 4);
          const double* g = a.nearG + lo * 9;
          double M[3][3];
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int y = 0; y < 3; ++y) M[x][y] = g[x * 3 + y];
          put(i, j, rK.id < rL.id, M);
        }
        k = 0;
      }
      if (!DISC) {
        S.pk[p] = (unsigned char)k;
        if (k) atomicAdd(&S.hist[k], 1);
      }
    }
    if (DISC) continue;
    __syncthreads();
    if (tid == 0) {                  // descending k: the heaviest pairs are taken first
      int off = 0, nch = 0;
      for (int k = 4; k >= 2; --k) {
        S.cursor[k] = off;
        const int ppc = k == 4 ? 4 : (k == 3 ? 10 : 32);      // pairs per warp: 8 / 3 / 1 lanes each
        for (int s0 = 0; s0 < S.hist[k]; s0 += ppc) {
          S.chs[nch] = (short)(off + s0);
          S.chn[nch] = (unsigned char)min(ppc, S.hist[k] - s0);
          S.chk[nch] = (unsigned char)k;
          ++nch;
        }
        off += S.hist[k];
      }
      S.nchunk = nch;
    }
    __syncthreads();
    for (int p = tid; p < CB * CB; p += X2T) {
      const int k = S.pk[p];
      if (k) S.plist[atomicAdd(&S.cursor[k], 1)] = (unsigned short)p;
    }
    __syncthreads();
    // ---- (B) blocks: a warp takes one chunk of same-order pairs at a time; k = 2: a lane per
    // pair, k = 3: 3 lanes (3 x nodes each), k = 4: 8 lanes (2 x nodes each), fixed-order
    // shuffle reduction over the lanes of a pair
    unsigned long long my = 0;
    for (;;) {
      int ch = 0;
      if (lane == 0) ch = atomicAdd(&S.q, 1);
      ch = __shfl_sync(0xffffffffu, ch, 0);
      if (ch >= S.nchunk) break;
      const int k = S.chk[ch];
      const int L = k == 4 ? 8 : (k == 3 ? 3 : 1);
      const int g = lane / L, sub = lane - g * L;
      const bool act = g < S.chn[ch];
      const int p = act ? S.plist[S.chs[ch] + g] : 0;
      const int i = p / CB, j = p % CB;
      const bool imin = S.r[i].id < S.r[CB + j].id;
      const double2* Xn = S.nd[imin ? i : CB + j];
      const double2* Yn = S.nd[imin ? CB + j : i];
      double M[3][3] = {};
      if (act) {
        if (k == 2) blk_part<E4, 4, 4, 1>(Xn + poff(2), Yn + poff(2), S.wl + poff(2), 0, a.ex, M);
        else if (k == 3) blk_part<E4, 9, 3, 3>(Xn + poff(3), Yn + poff(3), S.wl + poff(3), sub, a.ex, M);
        else blk_part<E4, 16, 2, 8>(Xn + poff(4), Yn + poff(4), S.wl + poff(4), sub, a.ex, M);
      }
      if (k > 2) {
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) {
            double v = M[x][y];
            if (k == 3) {
              const double v1 = __shfl_down_sync(0xffffffffu, v, 1), v2 = __shfl_down_sync(0xffffffffu, v, 2);
              v = (v + v1) + v2;
            } else {
              v += __shfl_down_sync(0xffffffffu, v, 4);
              v += __shfl_down_sync(0xffffffffu, v, 2);
              v += __shfl_down_sync(0xffffffffu, v, 1);
            }
            M[x][y] = v;
          }
      }
      if (act && sub == 0) {
        const double JJ = S.r[i].J * S.r[CB + j].J;
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) M[x][y] *= JJ;
        put(i, j, imin, M);
        my += (unsigned long long)(k * k) * (k * k);
      }
    }
    if (my) atomicAdd(&S.evals, my);
    __syncthreads();
    // ---- (C) the tile (and its transpose) into HBM
    if (in_tile) {
      for (int idx = tid; idx < nP * nQ; idx += X2T) {
        const unsigned long long q = S.tile[idx];
        if (!q) continue;
        const int r = idx / nQ, c = idx - r * nQ;
        const int gi = S.dofP[r], gj = S.dofQ[c];
        if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
        if (!diag && gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
      }
    }
  }
  if (tid == 0 && S.evals && a.evals) atomicAdd(a.evals, S.evals);
}

// ---------------------------------------------------------------- uniform-order block pairs
// Block pairs whose bounds fix one order k in {2, 3, 4} for all 32 x 32 cell pairs (disjoint
// blocks) are the bulk of the work; cross2d_uni_kernel streams them.  Everything a block pair
// needs is stored block-ordered (UData) so the next pair's data is copied into the second half
// of a double buffer with cp.async while the current pair is computed: the mapped nodes of the
// order k of both blocks (node-major: node r of cell c at [r][c], so the 32 lanes of a warp —
// one column cell each — read consecutive 16-byte words), J per cell, the vertex slots and the
// DoF lists.  Pairs are dealt round-robin over the CTAs (heaviest first), a warp takes one row
// cell i against the 32 column cells, each lane its whole pair; contributions go to the int64
// tile as in cross2d_kernel (fixed point, order-free), flushed to A once per pair.
constexpr int UNODES = 928;                // per block: k = 2, 3, 4 segments of 32 k^2 nodes
__host__ __device__ constexpr int useg(int k) { return k == 2 ? 0 : (k == 3 ? 128 : 416); }

__global__ void block_unodes_kernel(const int* __restrict__ bcells, const double2* __restrict__ nodes, int nb,
                                    const DevMesh m, const signed char* __restrict__ slot,
                                    double2* __restrict__ un, double* __restrict__ uj, int* __restrict__ us) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * UNODES) return;
  const int b = (int)(i / UNODES), x = (int)(i % UNODES);
  const int k = x < 128 ? 2 : (x < 416 ? 3 : 4);
  const int loc = x - useg(k), r = loc / CB, c = loc % CB;
  const int cell = bcells[b * CB + c];
  un[i] = cell >= 0 ? nodes[(int64_t)cell * NPRE2 + poff(k) + r] : make_double2(0.0, 0.0);
  if (x < CB) {
    const int cc = bcells[b * CB + x];
    uj[b * CB + x] = cc >= 0 ? m.geo[cc].J : 0.0;
    int pk = 0xffffff;                         // three slot bytes (0xff: not a DoF of the block)
    if (cc >= 0)
      for (int v = 0; v < 3; ++v) pk = (pk & ~(0xff << (8 * v))) | ((int)(unsigned char)slot[cc * 3 + v] << (8 * v));
    us[b * CB + x] = pk;
  }
}

#ifndef FL_XU_COLDOF
#define FL_XU_COLDOF 0      // 1: column-DoF exchange epilogue in cross2d_uni_kernel (measured neutral)
#endif
// Column-DoF lists of every block: for DoF slot c of block b the (cell slot j, vertex v) pairs with
// slot(j, v) == c, ascending, packed in 16 bytes: byte 0 = count (<= 15), then j * 3 + v.
__global__ void block_colmap_kernel(const int* __restrict__ us, int nb, uint4* __restrict__ ucol, int* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb * BRMAX) return;
  const int b = i / BRMAX, c = i % BRMAX;
  unsigned char e[16] = {};
  int n = 0;
  for (int j = 0; j < CB; ++j) {
    const int pk = us[b * CB + j];
    for (int v = 0; v < 3; ++v)
      if (((pk >> (8 * v)) & 0xff) == c) {
        if (n < 15) e[1 + n] = (unsigned char)(j * 3 + v);
        ++n;
      }
  }
  if (n > 15) atomicAdd(err, 1);
  e[0] = (unsigned char)min(n, 15);
  uint4 o;
  memcpy(&o, e, 16);
  ucol[i] = o;
}

struct UArgs {
  const int4* bpairs;                 // (P, Q, k, nP | nQ << 16)
  int nbp;
  const double2* un;
  const double* uj;
  const int* us;
  const int* bdofs;
  const uint4* ucol;                  // per block and DoF slot: count + (cell * 3 + vertex) entries (block_colmap_kernel)
  double ex, cs, lim;
  long long limq;                     // lim as an integer: |scaled contribution| < limq
  unsigned long long* A;
  int64_t lda;
  int r0, r1;
  unsigned long long* evals;
  int* ovf;
};

struct UBuf {
  double2 nd[2][16 * CB];             // [block][node r * 32 + cell]
  double J[2][CB];
  int sl[2][CB];
  int dof[2][BRMAX];
#if FL_XU_COLDOF
  uint4 col[BRMAX];                   // the column block's DoF -> (cell, vertex) lists
#endif
};
struct UShared {
  UBuf b[2];
#if FL_XU_COLDOF
  double mx[X2T / 32][9][CB];         // per warp: the 32 lanes' scaled 3x3 blocks (column-DoF exchange)
#endif
  unsigned long long tile[TCAP];
  double wl[NPRE2][3];
  unsigned long long evals;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// issue the copies of block pair `pr` into buffer B (every thread its share of 16-byte chunks)
__device__ __forceinline__ void u_stage(const UArgs& a, UBuf& B, int4 pr, int tid) {
  const int k = pr.z, nn = CB * k * k;           // nodes per block (16-byte chunks)
  const int tot = 2 * nn + 2 * 16 + 2 * 8 + 2 * 16 + (FL_XU_COLDOF ? BRMAX : 0);
  for (int c = tid; c < tot; c += X2T) {
    int x = c;
    if (x < 2 * nn) {
      const int side = x >= nn, r = x - side * nn;
      cp_async16(&B.nd[side][r], a.un + (int64_t)(side ? pr.y : pr.x) * UNODES + useg(k) + r);
      continue;
    }
    x -= 2 * nn;
    if (x < 32) {
      const int side = x >= 16, r = x - side * 16;
      cp_async16(&B.J[side][2 * r], a.uj + (int64_t)(side ? pr.y : pr.x) * CB + 2 * r);
      continue;
    }
    x -= 32;
    if (x < 16) {
      const int side = x >= 8, r = x - side * 8;
      cp_async16(&B.sl[side][4 * r], a.us + (int64_t)(side ? pr.y : pr.x) * CB + 4 * r);
      continue;
    }
    x -= 16;
    if (x < 32) {
      const int side = x >= 16, r = x - side * 16;
      cp_async16(&B.dof[side][4 * r], a.bdofs + (int64_t)(side ? pr.y : pr.x) * BRMAX + 4 * r);
      continue;
    }
#if FL_XU_COLDOF
    x -= 32;
    cp_async16(&B.col[x], a.ucol + (int64_t)pr.y * BRMAX + x);
#endif
  }
}

#ifndef FL_XU_YUNROLL
#define FL_XU_YUNROLL 3
#endif
constexpr int XU_YUNROLL = FL_XU_YUNROLL;      // y-loop unroll of the k = 3, 4 blocks

// partial 3x3 block from the NX x nodes x0, x0 + XS, ... of row cell i against all NN y nodes of
// column cell j (node-major staging: node r of cell c at [r * 32 + c])
template <int E4, int NN, int NX, int XS>
__device__ __forceinline__ void blk_part_nm(const double2* __restrict__ Xb, const double2* __restrict__ Yb, int i,
                                            int j, const double (*__restrict__ w)[3], int x0, double ex,
                                            double (&M)[3][3]) {
  double X0[NX], X1[NX], t[NX][3];
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const double2 X = Xb[(x0 + u * XS) * CB + i];
    X0[u] = X.x;
    X1[u] = X.y;
    t[u][0] = t[u][1] = t[u][2] = 0.0;
  }
#pragma unroll(NN <= 4 ? NN : XU_YUNROLL)
  for (int y = 0; y < NN; ++y) {
    const double2 Y = Yb[y * CB + j];
    const double w0 = w[y][0], w1 = w[y][1], w2 = w[y][2];
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const double d0 = X0[u] - Y.x, d1 = X1[u] - Y.y;
      const double v = kpow<E4>(fma(d1, d1, d0 * d0), ex);
      t[u][0] = fma(v, w0, t[u][0]);
      t[u][1] = fma(v, w1, t[u][1]);
      t[u][2] = fma(v, w2, t[u][2]);
    }
  }
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const int x = x0 + u * XS;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      M[a][0] = fma(w[x][a], t[u][0], M[a][0]);
      M[a][1] = fma(w[x][a], t[u][1], M[a][1]);
      M[a][2] = fma(w[x][a], t[u][2], M[a][2]);
    }
  }
}

// w * lambda_a of the rules k = 2, 3, 4 (the same numbers for every assembly: reference-element
// rules) in constant memory: the FP64 instructions of blk_regy read them as constant-bank operands
__constant__ double c_wl[NPRE2 * 3];

// Whole 3x3 block of (row cell i, the lane's column cell) for k = 2, 3: the column cell's NN mapped
// nodes stay in registers for every row cell of the block pair (Yr, loaded once per pair), the row
// cell's nodes are broadcast one at a time, the rule weights come from constant memory — no shared
// load inside the y sweep.  Two accumulator sets (even / odd y) shorten the FMA chains.
template <int E4, int NN>
__device__ __forceinline__ void blk_regy(const double2* __restrict__ Xb, const double2 (&Yr)[9], int i, int wo,
                                         double ex, double (&M)[3][3]) {
#pragma unroll 1
  for (int x = 0; x < NN; ++x) {
    const double2 X = Xb[x * CB + i];
    double t[2][3] = {};
#pragma unroll
    for (int y = 0; y < NN; ++y) {
      const double d0 = X.x - Yr[y].x, d1 = X.y - Yr[y].y;
      const double v = kpow<E4>(fma(d1, d1, d0 * d0), ex);
      t[y & 1][0] = fma(v, c_wl[(wo + y) * 3 + 0], t[y & 1][0]);
      t[y & 1][1] = fma(v, c_wl[(wo + y) * 3 + 1], t[y & 1][1]);
      t[y & 1][2] = fma(v, c_wl[(wo + y) * 3 + 2], t[y & 1][2]);
    }
    const double t0 = t[0][0] + t[1][0], t1 = t[0][1] + t[1][1], t2 = t[0][2] + t[1][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double wa = c_wl[(wo + x) * 3 + a];
      M[a][0] = fma(wa, t0, M[a][0]);
      M[a][1] = fma(wa, t1, M[a][1]);
      M[a][2] = fma(wa, t2, M[a][2]);
    }
  }
}

#ifndef FL_XU_MINB
#define FL_XU_MINB 2
#endif
#ifndef FL_XU_REGY
#define FL_XU_REGY 0
#endif

template <int E4>
__global__ void __launch_bounds__(X2T, FL_XU_MINB) cross2d_uni_kernel(UArgs a, const double* __restrict__ wl_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UShared& S = *reinterpret_cast<UShared*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < NPRE2 * 3; i += X2T) (&S.wl[0][0])[i] = wl_g[i];
  for (int i = tid; i < TCAP; i += X2T) S.tile[i] = 0ull;
  if (tid == 0) S.evals = 0;
  int it = blockIdx.x;
  if (it >= a.nbp || (*a.ovf & 2)) return;       // (bit 1: unit too coarse, coarse_flag_kernel)
  int4 cur = a.bpairs[it];
  u_stage(a, S.b[0], cur, tid);
  cp_async_commit();
  int4 nxt = it + (int)gridDim.x < a.nbp ? a.bpairs[it + gridDim.x] : make_int4(0, 0, 0, 0);
  unsigned long long my = 0;
  int bsel = 0;
  for (; it < a.nbp; it += gridDim.x) {
    cp_async_wait_all();
    __syncthreads();                             // buffer bsel holds `cur`; the tile is flushed
    const bool more = it + (int)gridDim.x < a.nbp;
    if (more) u_stage(a, S.b[bsel ^ 1], nxt, tid);
    cp_async_commit();
    const int4 pr = cur;
    cur = nxt;
    if (it + 2 * (int)gridDim.x < a.nbp) nxt = a.bpairs[it + 2 * gridDim.x];   // record two ahead
    const UBuf& B = S.b[bsel];
    const int k = pr.z, nP = pr.w & 0xffff, nQ = pr.w >> 16;
    const bool in_tile = nP * nQ <= TCAP;
    double2 Yr[9];                               // the lane's column cell nodes (k = 2, 3)
    if (FL_XU_REGY && k <= 3) {
#pragma unroll
      for (int y = 0; y < 9; ++y)
        if (y < k * k) Yr[y] = B.nd[1][y * CB + lane];
    }
#pragma unroll 1
    for (int i = wid; i < CB; i += X2T / 32) {
      const int j = lane;
      const double JJ = B.J[0][i] * B.J[1][j];
#if FL_XU_COLDOF
      if (B.J[0][i] == 0.0) continue;            // an empty row slot (warp-uniform)
      double M[3][3] = {};
      if (JJ == 0.0) {                           // an empty column slot: zeros into the exchange
      } else
#else
      if (JJ == 0.0) continue;                   // an empty slot of a partial block
      double M[3][3] = {};
#endif
      if (FL_XU_REGY && k == 2) {
        blk_regy<E4, 4>(B.nd[0], Yr, i, poff(2), a.ex, M);
      } else if (FL_XU_REGY && k == 3) {
        blk_regy<E4, 9>(B.nd[0], Yr, i, poff(3), a.ex, M);
      } else if (k == 2) {
        blk_part_nm<E4, 4, 4, 1>(B.nd[0], B.nd[1], i, j, S.wl + poff(2), 0, a.ex, M);
      } else if (k == 3) {
#pragma unroll 1
        for (int xs = 0; xs < 3; ++xs) blk_part_nm<E4, 9, 3, 3>(B.nd[0], B.nd[1], i, j, S.wl + poff(3), xs, a.ex, M);
      } else {
#pragma unroll 1
        for (int xs = 0; xs < 4; ++xs)
          blk_part_nm<E4, 16, 4, 4>(B.nd[0], B.nd[1], i, j, S.wl + poff(4), xs, a.ex, M);
      }
#if FL_XU_COLDOF
      // column-DoF exchange: the lanes' scaled blocks go to shared memory, then lane c sums the
      // (cell, vertex) entries of column DoF c in their fixed list order — one rounding and three
      // tile adds per (row cell, column DoF) instead of nine per cell pair, no address conflicts
      // inside the warp
      const int spk = B.sl[0][i];
      {
        const double sc = JJ * a.cs;
        double(*mx)[CB] = S.mx[wid];
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) mx[x * 3 + y][lane] = M[x][y] * sc;
      }
      __syncwarp();
      bool bad = false;
      for (int c = lane; c < nQ; c += 32) {
        const uint4 cm = B.col[c];
        const unsigned char* e = reinterpret_cast<const unsigned char*>(&cm);
        const int n = e[0];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int m = 0; m < n; ++m) {
          const int jv = e[1 + m], jj = jv / 3, v = jv - jj * 3;
          s0 += S.mx[wid][v][jj];
          s1 += S.mx[wid][3 + v][jj];
          s2 += S.mx[wid][6 + v][jj];
        }
        const double sv[3] = {s0, s1, s2};
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          const int si = (spk >> (8 * x)) & 0xff;
          if (si == 0xff) continue;
          const long long qs = __double2ll_rn(sv[x]);
          // at most 15 contributions, each below limq
          bad |= (unsigned long long)(qs + 16 * a.limq) > 32ull * (unsigned long long)a.limq;
          const unsigned long long q = (unsigned long long)qs;
          if (!q) continue;
          if (in_tile) {
            tile_add(&S.tile[si * nQ + c], q);
          } else {
            const int gi = B.dof[0][si], gj = B.dof[1][c];
            if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
            if (gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
          }
        }
      }
      __syncwarp();                              // mx is rewritten for the next row cell
      if (bad) atomicOr(a.ovf, 1);
      if (JJ != 0.0) my += (unsigned long long)(k * k) * (k * k);
      continue;
#else
      const int spk = B.sl[0][i], tpk = B.sl[1][j];
      const double sc = JJ * a.cs;
      bool bad = false;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const int si = (spk >> (8 * x)) & 0xff;
        if (si == 0xff) continue;
#pragma unroll
        for (int y = 0; y < 3; ++y) {
          const int sj = (tpk >> (8 * y)) & 0xff;
          if (sj == 0xff) continue;
          const long long qs = __double2ll_rn(M[x][y] * sc);
          bad |= (unsigned long long)(qs + a.limq) > 2ull * (unsigned long long)a.limq;   // |q| >= limq, NaN
          const unsigned long long q = (unsigned long long)qs;
          if (in_tile) {
            tile_add(&S.tile[si * nQ + sj], q);
          } else {
            const int gi = B.dof[0][si], gj = B.dof[1][sj];
            if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
            if (gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
          }
        }
      }
#endif
      if (bad) atomicOr(a.ovf, 1);
      my += (unsigned long long)(k * k) * (k * k);
    }
    __syncthreads();
    if (in_tile) {
      for (int idx = tid; idx < nP * nQ; idx += X2T) {
        const unsigned long long q = S.tile[idx];
        if (!q) continue;
        S.tile[idx] = 0ull;
        const int r = idx / nQ, c = idx - r * nQ;
        const int gi = B.dof[0][r], gj = B.dof[1][c];
        if (gi >= a.r0 && gi < a.r1) atomicAdd(&a.A[(int64_t)(gi - a.r0) * a.lda + gj], q);
        if (gj >= a.r0 && gj < a.r1) atomicAdd(&a.A[(int64_t)(gj - a.r0) * a.lda + gi], q);
      }
    }
    bsel ^= 1;
  }
  cp_async_wait_all();
  if (my) atomicAdd(&S.evals, my);
  __syncthreads();
  if (tid == 0 && S.evals && a.evals) atomicAdd(a.evals, S.evals);
}

__global__ void pair_morton_kernel(const int4* __restrict__ pr, int n, unsigned* __restrict__ key,
                                   int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = spread16b((uint32_t)pr[i].x) | (spread16b((uint32_t)pr[i].y) << 1);
  idx[i] = i;
}
__global__ void gather_int4_kernel(const int4* __restrict__ src, const int* __restrict__ idx, int n,
                                   int4* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void uni_flag_kernel(const int4* __restrict__ all, int n, const int* __restrict__ bndof,
                                int4* __restrict__ allw, int* __restrict__ uf, int* __restrict__ rf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 p = all[i];
  p.w = bndof[p.x] | (bndof[p.y] << 16);
  allw[i] = p;
  const int u = p.z >= 2 && p.z < KW2D;
  uf[i] = u;
  rf[i] = !u;
}

__global__ void iota_kernel64(int* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int)i;
}
__global__ void gather4_kernel(const int4* __restrict__ raw, const int* __restrict__ keep, const int* __restrict__ nf,
                               const int* __restrict__ idx, int64_t n, int4* __restrict__ out, int* __restrict__ okeep,
                               int* __restrict__ onear) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = idx[i];
  out[i] = raw[j];
  okeep[i] = keep[j];
  onear[i] = keep[j] & nf[j];
}

__global__ void fixed_to_double_kernel(unsigned long long* A, int64_t count, double inv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = (long long)A[i];
    reinterpret_cast<double*>(A)[i] = (double)v * inv;
  }
}

#define FL_E4_SWITCH2(e4, ...)                                \
  switch (e4) {                                               \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

}  // namespace

// The whole 2D cross term of rows [row_begin, row_end) into A (double, leading dim lda): A is
// overwritten (zeroed first).  Near pairs (k >= KW2D) are discovered here and computed once by
// near_pairs_build into `near`.  t_disc / t_near: events recorded after discovery and after the
// near blocks (phase timing).
void build_blocks2d(const DevMesh& m, const DevTables& t, double e, int row_begin, int row_end, Blocks2D& B,
                    cudaStream_t st) {
  const int nc = m.nc;
  const int nb = (nc + CB - 1) / CB;
  B.nb = nb;
  // ---- Morton order of the cells
  std::vector<double> hv((size_t)m.nv * 2);
  FL_CUDA(cudaMemcpyAsync(hv.data(), m.vert, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  double bb[4] = {hv[0], hv[0], hv[1], hv[1]};
  for (int v = 0; v < m.nv; ++v) {
    bb[0] = std::min(bb[0], hv[2 * v]); bb[1] = std::max(bb[1], hv[2 * v]);
    bb[2] = std::min(bb[2], hv[2 * v + 1]); bb[3] = std::max(bb[3], hv[2 * v + 1]);
  }
  const double sx = 65535.0 / std::max(bb[1] - bb[0], 1e-300), sy = 65535.0 / std::max(bb[3] - bb[2], 1e-300);
  DBuf<uint32_t> keys(nc), keys2(nc);
  DBuf<int> vals(nc), vals2(nc);
  cell_morton_kernel<<<(nc + 255) / 256, 256, 0, st>>>(m, bb[0], bb[2], sx, sy, keys.p, vals.p), note_launch();
  {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, keys2.p, vals.p, vals2.p, nc, 0, 32, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, keys.p, keys2.p, vals.p, vals2.p, nc, 0, 32, st));
  }
  // ---- blocks
  B.bcells.alloc((size_t)nb * CB); B.bdofs.alloc((size_t)nb * BRMAX); B.bndof.alloc(nb); B.rowflag.alloc(nb);
  B.err.alloc(1); B.slot.alloc((size_t)nc * 3); B.bstat.alloc((size_t)nb * 8); B.blk_of.alloc(nc);
  FL_CUDA(cudaMemsetAsync(B.err.p, 0, sizeof(int), st));
  block_build_kernel<<<nb, 128, 0, st>>>(m, vals2.p, nb, row_begin, row_end, B.bcells.p, B.bdofs.p, B.bndof.p,
                                         B.slot.p, B.bstat.p, B.rowflag.p, B.err.p), note_launch();
  block_of_kernel<<<(nc + 255) / 256, 256, 0, st>>>(vals2.p, nc, B.blk_of.p), note_launch();
  // mapped nodes of the orders 2, 3, 4: per cell (cross2d_kernel) and block-ordered node-major with
  // J and the vertex slots (cross2d_uni_kernel, tail2d_block_kernel)
  const RuleRef r2 = t.rule(T_DISJ, 2), r3 = t.rule(T_DISJ, 3), r4 = t.rule(T_DISJ, 4);
  if (r2.cnt != 4 || r3.cnt != 9 || r4.cnt != 16) throw Error(-3, "disjoint rules k = 2, 3, 4 missing");
  B.nodes.alloc((size_t)nc * NPRE2);
  cell_nodes2_kernel<<<(unsigned)(((int64_t)nc * NPRE2 + 255) / 256), 256, 0, st>>>(m, t.data, r2, r3, r4, B.nodes.p),
      note_launch();
  B.un.alloc((size_t)nb * UNODES); B.uj.alloc((size_t)nb * CB); B.us.alloc((size_t)nb * CB);
  block_unodes_kernel<<<(unsigned)(((int64_t)nb * UNODES + 255) / 256), 256, 0, st>>>(B.bcells.p, B.nodes.p, nb, m,
                                                                                    B.slot.p, B.un.p, B.uj.p, B.us.p),
      note_launch();
#if FL_XU_COLDOF
  B.ucol.alloc((size_t)nb * BRMAX);
  block_colmap_kernel<<<(nb * BRMAX + 255) / 256, 256, 0, st>>>(B.us.p, nb, B.ucol.p, B.err.p), note_launch();
#endif
  // smallest distance of two disjoint cells (second-ring scan), largest Jacobian and cell radius
  DBuf<unsigned long long> bnd(4);
  unsigned long long init[4] = {0ull, 0ull, 0ull, 0ull};
  const double big = 1e300;
  std::memcpy(&init[0], &big, 8);
  FL_CUDA(cudaMemcpyAsync(bnd.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  dmin_kernel<<<(nc + 127) / 128, 128, 0, st>>>(m, bnd.p, bnd.p + 1, bnd.p + 2, e, bnd.p + 3), note_launch();
  unsigned long long hb[4];
  FL_CUDA(cudaMemcpyAsync(hb, bnd.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  std::memcpy(&B.dmin, &hb[0], 8);
  std::memcpy(&B.jmax, &hb[1], 8);
  std::memcpy(&B.radmax, &hb[2], 8);
  std::memcpy(&B.beta, &hb[3], 8);
  FL_CHECK_LAUNCH();
}

// largest |entry| of the near blocks (already scaled by J_K J_L)
__global__ void absmax_kernel(const double* __restrict__ G, int64_t n, unsigned long long* __restrict__ out) {
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v = fmax(v, fabs(G[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

// sets bit 1 of *flag when an entry's worst rounding error (err_units of 2^-S) could reach 1e-12 of
// the largest near block entry times C (ref_scale * gmax): pass 2 then adds nothing
__global__ void coarse_flag_kernel(const unsigned long long* __restrict__ gmax_bits, double err, double ref_scale,
                                   int force, int* __restrict__ flag) {
  const double gmax = __longlong_as_double((long long)*gmax_bits);
  if (force || err > ref_scale * gmax) atomicOr(flag, 2);
}

void assemble_cross2d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                      const Blocks2D& B, int row_begin, int row_end, double* A, int64_t lda,
                      unsigned long long* evals, NearPairs& near, Cross2DInfo& info, cudaEvent_t t_disc,
                      cudaEvent_t t_near, cudaStream_t st, unsigned long long* evals_near) {
  const int nc = m.nc;
  const int nb = B.nb;
  const int64_t rows = row_end - row_begin;
  const DBuf<int>& bcells = B.bcells;
  const DBuf<int>& bdofs = B.bdofs;
  const DBuf<int>& bndof = B.bndof;
  const DBuf<int>& rowflag = B.rowflag;
  const DBuf<int>& err = B.err;
  const DBuf<signed char>& slot = B.slot;
  const DBuf<double>& bstat = B.bstat;
  // ---- mapped nodes, rule weights, scale bound
  const RuleRef r2 = t.rule(T_DISJ, 2), r3 = t.rule(T_DISJ, 3), r4 = t.rule(T_DISJ, 4);
  const DBuf<double2>& nodes = B.nodes;
  std::vector<double> hw(NPRE2 * 3), hrow(NODE);
  for (int x = 0; x < NPRE2; ++x) {
    const RuleRef rr = x < 4 ? r2 : (x < 13 ? r3 : r4);
    const int xl = x < 4 ? x : (x < 13 ? x - 4 : x - 13);
    FL_CUDA(cudaMemcpyAsync(hrow.data(), t.data + (size_t)(rr.off + xl) * NODE, NODE * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < 3; ++c) hw[x * 3 + c] = hrow[3 + c];
  }
  DBuf<double> wl(NPRE2 * 3);
  FL_CUDA(cudaMemcpyAsync(wl.p, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyToSymbolAsync(c_wl, hw.data(), hw.size() * sizeof(double), 0, cudaMemcpyHostToDevice, st));
  int herr = 0;
  FL_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  static const bool force_early = [] {           // FRACLAP_CROSS2D_FALLBACK=early: take this exit (test switch)
    const char* v = getenv("FRACLAP_CROSS2D_FALLBACK");
    return v && std::string(v) == "early";
  }();
  if (herr || force_early) {  // a Morton block of 32 cells touches more than 64 DoFs: the DoF-tile kernel takes over
    info.fallback = 1;
    return;
  }
  const double dmin = B.dmin;
  // one pair's |contribution| <= C * (1/6)^2 * J_K J_L dist^(-(d+2s)) <= C beta / 36 (sum of
  // w*lambda over the reference triangle = 1/6; beta_kernel); an entry sums at most vmax^2 pairs
  // (vmax cells around a vertex).  Scale: vmax^2 * that -> 2^61, so every contribution stays below
  // lim = 2^62 / vmax^2 (checked in the kernels) and every sum below 2^62.
  const double e = -2.0 * ex;                      // d + 2s
  const double vmax = (double)MAX_VALENCE;
  const double beta = B.beta;
  const double bound = beta > 0.0 ? vmax * vmax * Cds * beta / 36.0 : 1.0;
  int S = 61 - (int)std::ceil(std::log2(std::max(bound, 1e-300)));
  S = std::max(-1000, std::min(1000, S));
  const double scale = std::ldexp(1.0, S);
  info.scale_exp = S;
  info.dmin = dmin;
  // ---- block pairs, heavy first
  const int64_t ncand = (int64_t)nb * (nb + 1) / 2;
  DBuf<int4> raw(ncand);
  DBuf<unsigned> key(ncand), key2(ncand);
  DBuf<int> keep(ncand), nflag(ncand);
  block_pairs_kernel<<<(unsigned)((ncand + 255) / 256), 256, 0, st>>>(oc, bstat.p, rowflag.p, nb,
                                                                     (row_begin == 0 && row_end == m.n) ? 1 : 0,
                                                                     ncand, raw.p, key.p, keep.p, nflag.p),
      note_launch();
  // FRACLAP_EXACT_RANGE=0: circle bounds only
  static const bool exact_range = [] {
    const char* v = getenv("FRACLAP_EXACT_RANGE");
    return !(v && std::string(v) == "0");
  }();
  // FRACLAP_CROSS2D_KUNI=0 (diagnostic): no block-uniform orders, every pair gets its own order
  static const bool kuni_off = [] {
    const char* v = getenv("FRACLAP_CROSS2D_KUNI");
    return v && std::string(v) == "0";
  }();
  if (kuni_off) clear_kuni_kernel<<<(unsigned)((ncand + 255) / 256), 256, 0, st>>>(raw.p, nflag.p, ncand), note_launch();
  if (exact_range && !kuni_off)
    cross_refine_kernel<<<(unsigned)((ncand * 32 + 255) / 256), 256, 0, st>>>(oc, m, bcells.p, bstat.p, ncand, raw.p,
                                                                            nflag.p),
        note_launch();
  DBuf<int> idx(ncand), idx2(ncand);
  iota_kernel64<<<(unsigned)((ncand + 255) / 256), 256, 0, st>>>(idx.p, ncand), note_launch();
  {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, idx2.p, (int)ncand, 0, 32, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, key.p, key2.p, idx.p, idx2.p, (int)ncand, 0, 32, st));
  }
  // gather in sorted order, then keep (rows) / near subsets
  DBuf<int4> sorted(ncand);
  DBuf<int> skeep(ncand), snear(ncand), nsel(2);
  gather4_kernel<<<(unsigned)((ncand + 255) / 256), 256, 0, st>>>(raw.p, keep.p, nflag.p, idx2.p, ncand, sorted.p,
                                                                  skeep.p, snear.p), note_launch();
  DBuf<int4> all(ncand), nearl(ncand);
  {
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, sorted.p, skeep.p, all.p, nsel.p, (int)ncand, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, sorted.p, skeep.p, all.p, nsel.p, (int)ncand, st));
    // near candidates among the kept pairs
    FL_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, sorted.p, snear.p, nearl.p, nsel.p + 1, (int)ncand, st));
  }
  int hn[2];
  FL_CUDA(cudaMemcpyAsync(hn, nsel.p, sizeof(hn), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  const int nall = hn[0], nnear = hn[1];
  // uniform-order block pairs (k = 2..4) for the streaming kernel, the rest for cross2d_kernel
  static const bool uni_off = [] {             // FRACLAP_CROSS2D_UNI=0: every pair through cross2d_kernel
    const char* v = getenv("FRACLAP_CROSS2D_UNI");
    return v && std::string(v) == "0";
  }();
  DBuf<int4> allw(std::max(nall, 1)), ulist(std::max(nall, 1)), rlist(std::max(nall, 1));
  DBuf<int> uf(std::max(nall, 1)), rf(std::max(nall, 1)), nsel2(2);
  int hu[2] = {0, nall};
  if (nall > 0 && !uni_off) {
    uni_flag_kernel<<<(nall + 255) / 256, 256, 0, st>>>(all.p, nall, bndof.p, allw.p, uf.p, rf.p), note_launch();
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, allw.p, uf.p, ulist.p, nsel2.p, nall, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, allw.p, uf.p, ulist.p, nsel2.p, nall, st));
    FL_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, allw.p, rf.p, rlist.p, nsel2.p + 1, nall, st));
    FL_CUDA(cudaMemcpyAsync(hu, nsel2.p, sizeof(hu), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
  }
  const int nuni = hu[0], nrest = hu[1];
  const int4* rest = (nall > 0 && !uni_off) ? rlist.p : all.p;
  // the uniform pairs in 2D Morton order of (P, Q): CTAs working at the same time touch a compact
  // region of A, so the integer atomics of neighbouring block pairs meet in L2 instead of DRAM
  static const bool uni_heavy = [] {          // FRACLAP_CROSS2D_UNI_ORDER=heavy: keep the heavy-first order
    const char* v = getenv("FRACLAP_CROSS2D_UNI_ORDER");
    return v && std::string(v) == "heavy";
  }();
  DBuf<int4> ulist2;
  const int4* uorder = ulist.p;
  if (nuni > 1 && !uni_heavy) {
    DBuf<unsigned> mk(nuni), mk2(nuni);
    DBuf<int> mi(nuni), mi2(nuni);
    pair_morton_kernel<<<(nuni + 255) / 256, 256, 0, st>>>(ulist.p, nuni, mk.p, mi.p), note_launch();
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, mk.p, mk2.p, mi.p, mi2.p, nuni, 0, 32, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, mk.p, mk2.p, mi.p, mi2.p, nuni, 0, 32, st));
    ulist2.alloc(nuni);
    gather_int4_kernel<<<(nuni + 255) / 256, 256, 0, st>>>(ulist.p, mi2.p, nuni, ulist2.p), note_launch();
    uorder = ulist2.p;
  }
  const DBuf<double2>& un = B.un;
  const DBuf<double>& uj = B.uj;
  const DBuf<int>& us = B.us;
  info.block_pairs = nall;
  info.near_block_pairs = nnear;
  // ---- A (int64 view) zeroed
  unsigned long long* Ai = reinterpret_cast<unsigned long long*>(A);
  if (rows > 0) FL_CUDA(cudaMemsetAsync(A, 0, (size_t)rows * lda * sizeof(double), st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(XShared);
  DBuf<int> queue(1), ovf(1);
  FL_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), st));
  XArgs xa{};
  xa.m = m; xa.oc = oc; xa.ex = ex; xa.cs = -Cds * scale; xa.lim = std::ldexp(1.0, 62) / (vmax * vmax);
  xa.bcells = bcells.p; xa.bdofs = bdofs.p; xa.bndof = bndof.p; xa.slot = slot.p; xa.nodes = nodes.p;
  xa.A = Ai; xa.lda = lda; xa.r0 = row_begin; xa.r1 = row_end; xa.evals = evals; xa.ovf = ovf.p;
  // ---- pass 1: discovery of the near pairs (block pairs whose bound reaches KW2D)
  unsigned int cap = (unsigned int)std::max<int64_t>(
      1024, std::min<int64_t>({(int64_t)nnear * CB * CB, (int64_t)nc * 4096, ((int64_t)1 << 31) - 1}));
  DBuf<unsigned long long> near_keys;
  DBuf<unsigned int> near_cnt(1);
  int64_t nkeys = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    near_keys.alloc(cap);
    FL_CUDA(cudaMemsetAsync(near_cnt.p, 0, sizeof(unsigned int), st));
    FL_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(int), st));
    xa.bpairs = nearl.p; xa.nbp = nnear; xa.queue = queue.p;
    xa.near_keys = near_keys.p; xa.near_count = near_cnt.p; xa.near_cap = cap;
    if (nnear > 0) {
      const int grid = std::min(nnear, FL_X2_MINB * sms);
      FL_E4_SWITCH2(e4, {
        FL_CUDA(cudaFuncSetAttribute(cross2d_kernel<E4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cross2d_kernel<E4, true><<<grid, X2T, smem, st>>>(xa, wl.p), note_launch();
      });
      FL_CHECK_LAUNCH();
    }
    unsigned int cnt = 0;
    FL_CUDA(cudaMemcpyAsync(&cnt, near_cnt.p, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    nkeys = cnt;
    if (cnt <= cap) break;
    cap = cnt;
  }
  if (t_disc) FL_CUDA(cudaEventRecord(t_disc, st));
  near_pairs_build(m, t, oc, ex, e4, near_keys.p, nkeys, near, evals_near ? evals_near : evals, st);
  near_keys.free();
  if (t_near) FL_CUDA(cudaEventRecord(t_near, st));
  // ---- is the fixed-point unit fine enough?  An entry's rounding error is at most vmax^2 / 2
  // units of 2^-S; the largest near block entry (times C) is of the size of A's significant
  // off-diagonal entries.  When the units could reach 1e-12 of it (cells sharing no vertex that
  // almost touch: the bound above is then far above every real contribution) pass 2 adds nothing
  // (bit 1 of ovf) and the caller assembles the cross term with the DoF-tile kernel (exact double
  // sums, any mesh).
  if (near.n > 0) {
    static const bool force_fb = [] {              // FRACLAP_CROSS2D_FALLBACK=1: take the fallback (test switch)
      const char* v = getenv("FRACLAP_CROSS2D_FALLBACK");
      return v && std::string(v) == "1";
    }();
    DBuf<unsigned long long> gmax(1);
    FL_CUDA(cudaMemsetAsync(gmax.p, 0, sizeof(unsigned long long), st));
    absmax_kernel<<<4 * sms, 256, 0, st>>>(near.G.p, (int64_t)near.n * 9, gmax.p), note_launch();
    // decided on the device (no host synchronisation here): pass 2 returns at once when the flag is set
    coarse_flag_kernel<<<1, 1, 0, st>>>(gmax.p, 0.5 * vmax * vmax * std::ldexp(1.0, -S), 1e-12 * Cds, force_fb ? 1 : 0,
                                        ovf.p), note_launch();
  }
  // ---- pass 2: every block pair
  FL_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(int), st));
  xa.bpairs = rest; xa.nbp = nrest; xa.queue = queue.p;
  xa.near_keys = nullptr; xa.near_count = nullptr; xa.near_cap = 0;
  xa.nearH = near.hkey.p; xa.nearI = near.hidx.p; xa.hmask = near.hmask; xa.nearG = near.G.p;
  if (nuni > 0) {
    UArgs ua{};
    ua.bpairs = uorder; ua.nbp = nuni; ua.un = un.p; ua.uj = uj.p; ua.us = us.p; ua.bdofs = bdofs.p; ua.ucol = B.ucol.p;
    ua.ex = ex; ua.cs = xa.cs; ua.lim = xa.lim; ua.limq = (long long)xa.lim; ua.A = Ai; ua.lda = lda; ua.r0 = row_begin; ua.r1 = row_end;
    ua.evals = evals; ua.ovf = ovf.p;
    const size_t usm = sizeof(UShared);
    const int grid = std::min(nuni, FL_XU_MINB * sms);
    FL_E4_SWITCH2(e4, {
      FL_CUDA(cudaFuncSetAttribute(cross2d_uni_kernel<E4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
      cross2d_uni_kernel<E4><<<grid, X2T, usm, st>>>(ua, wl.p), note_launch();
    });
    FL_CHECK_LAUNCH();
  }
  if (nrest > 0) {
    const int grid = std::min(nrest, FL_X2_MINB * sms);
    FL_E4_SWITCH2(e4, {
      FL_CUDA(cudaFuncSetAttribute(cross2d_kernel<E4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cross2d_kernel<E4, false><<<grid, X2T, smem, st>>>(xa, wl.p), note_launch();
    });
    FL_CHECK_LAUNCH();
  }
  // ---- fixed point -> double, in place
  if (rows > 0) {
    fixed_to_double_kernel<<<4 * sms, 256, 0, st>>>(Ai, rows * lda, std::ldexp(1.0, -S)), note_launch();
    FL_CHECK_LAUNCH();
  }
  int hovf = 0;
  FL_CUDA(cudaMemcpyAsync(&hovf, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (hovf & 2) {
    info.fallback = 1;
    return;
  }
  if (hovf) throw Error(-5, "internal: a cross contribution exceeded the fixed-point bound");
}

}  // namespace fl
