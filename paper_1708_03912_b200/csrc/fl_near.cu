// Near disjoint pairs: the few cell pairs whose Gauss order k >= KW (k^(2d) >= 625 nodes in 2D)
// carry most of the cross-term work (cross_matrices, assembly.py:172-229) but are rare.  The
// cross tiles only record them; here they are de-duplicated (sort + unique of the (min, max)
// key — the reference's own orientation, assembly.py:973-982), each block is computed ONCE by a
// warp with the column cell's mapped nodes staged in shared memory (no barriers, no halo
// redundancy), and CSR indexes let the row-owner pull (fl_local.cu) add -C*M to every entry
// in a fixed order.
#include <cub/cub.cuh>

#include "fl_internal.h"

namespace fl {

constexpr int NW = 8;          // warps per CTA
constexpr int NMAXN = 81;      // max k^d nodes (2D cap 9; 1D k <= 32)

// One pair's 3x3 block: lane l takes the x nodes l, l + 32, l + 64 (NX of them) and sweeps all y
// nodes, which every lane reads at the same address (broadcast shared loads); NX = 1 keeps four
// accumulator sets (y mod 4) for independent chains.  Fixed summation order.
template <int D, int E4, int NX>
__device__ __forceinline__ void near_pair(const CellGeo& A, const double* __restrict__ tab, RuleRef rr, int nn,
                                          const double4* __restrict__ syw, const double* __restrict__ sw2, int lane,
                                          double ex, double (&Gm)[3][3]) {
  constexpr int HS = NX == 1 ? 4 : 1;          // accumulator sets (independent chains when a lane has one x)
  double X0[NX], X1[NX], t[NX][HS][3];
  bool ok[NX];
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const int x = lane + 32 * u;
    ok[u] = x < nn;
    const double* nx = tab + (size_t)(rr.off + (ok[u] ? x : 0)) * NODE;
    if (D == 1) {
      X0[u] = A.p[0][0] + nx[0] * (A.p[1][0] - A.p[0][0]);
      X1[u] = 0.0;
    } else {
      X0[u] = A.p[0][0] + (nx[0] * (A.p[1][0] - A.p[0][0]) + nx[1] * (A.p[2][0] - A.p[0][0]));
      X1[u] = A.p[0][1] + (nx[0] * (A.p[1][1] - A.p[0][1]) + nx[1] * (A.p[2][1] - A.p[0][1]));
    }
#pragma unroll
    for (int h = 0; h < HS; ++h) t[u][h][0] = t[u][h][1] = t[u][h][2] = 0.0;
  }
  auto eval = [&](int y, int h) {
    const double4 Y = syw[y];
    const double w2 = D == 2 ? sw2[y] : 0.0;
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const double d0 = X0[u] - Y.x;
      double r2;
      if (D == 1) {
        r2 = d0 * d0;
      } else {
        const double d1 = X1[u] - Y.y;
        r2 = fma(d1, d1, d0 * d0);
      }
      const double v = kpow<E4>(r2, ex);
      t[u][h][0] = fma(v, Y.z, t[u][h][0]);
      t[u][h][1] = fma(v, Y.w, t[u][h][1]);
      if (D == 2) t[u][h][2] = fma(v, w2, t[u][h][2]);
    }
  };
  int y = 0;
  if (NX == 1) {
#pragma unroll 1
    for (; y + 3 < nn; y += 4) {
      eval(y, 0);
      eval(y + 1, HS > 1 ? 1 : 0);
      eval(y + 2, HS > 2 ? 2 : 0);
      eval(y + 3, HS > 3 ? 3 : 0);
    }
    for (; y < nn; ++y) eval(y, 0);
  } else {
#pragma unroll 2
    for (; y < nn; ++y) eval(y, 0);
  }
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    if (!ok[u]) continue;
    const double* nx = tab + (size_t)(rr.off + lane + 32 * u) * NODE;
    double t0 = t[u][0][0], t1 = t[u][0][1], t2 = t[u][0][2];
#pragma unroll
    for (int h = 1; h < HS; ++h) { t0 += t[u][h][0]; t1 += t[u][h][1]; t2 += t[u][h][2]; }
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      const double lx = nx[3 + a];
      Gm[a][0] = fma(lx, t0, Gm[a][0]);
      Gm[a][1] = fma(lx, t1, Gm[a][1]);
      if (D == 2) Gm[a][2] = fma(lx, t2, Gm[a][2]);
    }
  }
}

template <int D, int E4>
__global__ void __launch_bounds__(NW * 32) near_block_kernel(DevMesh m, const double* __restrict__ tab,
                                                             DevTables dir, OrderConsts oc, double ex,
                                                             const int* __restrict__ P, const int* __restrict__ Q,
                                                             const int* __restrict__ KK, int64_t n,
                                                             double* __restrict__ G,
                                                             unsigned long long* __restrict__ evals) {
  __shared__ double4 syw[NW][NMAXN];   // y node (x, y) and w*lambda_0, w*lambda_1
  __shared__ double sw2[NW][NMAXN];    // w*lambda_2
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long my = 0;
  for (int64_t pi = (int64_t)blockIdx.x * NW + w; pi < n; pi += (int64_t)gridDim.x * NW) {
    const CellGeo& A = m.geo[P[pi]];
    const CellGeo& B = m.geo[Q[pi]];
    const int k = KK[pi];                 // the order found by the cross tiles (reference orientation)
    const RuleRef rr = dir.rule(T_DISJ, k);
    const int nn = rr.cnt;
    // stage the y (column cell) nodes, absolute coordinates as _map_points forms them
    for (int y = lane; y < nn; y += 32) {
      const double* nd = tab + (size_t)(rr.off + y) * NODE;
      double Y0, Y1 = 0.0;
      if (D == 1) {
        Y0 = B.p[0][0] + nd[0] * (B.p[1][0] - B.p[0][0]);
      } else {
        Y0 = B.p[0][0] + (nd[0] * (B.p[1][0] - B.p[0][0]) + nd[1] * (B.p[2][0] - B.p[0][0]));
        Y1 = B.p[0][1] + (nd[0] * (B.p[1][1] - B.p[0][1]) + nd[1] * (B.p[2][1] - B.p[0][1]));
      }
      syw[w][y] = make_double4(Y0, Y1, nd[3], nd[4]);
      sw2[w][y] = nd[5];
    }
    __syncwarp();
    double Gm[3][3] = {};
    if (nn <= 32) near_pair<D, E4, 1>(A, tab, rr, nn, syw[w], sw2[w], lane, ex, Gm);
    else if (nn <= 64) near_pair<D, E4, 2>(A, tab, rr, nn, syw[w], sw2[w], lane, ex, Gm);
    else near_pair<D, E4, 3>(A, tab, rr, nn, syw[w], sw2[w], lane, ex, Gm);
    const double JJ = A.J * B.J;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double s = warp_sum(Gm[a][b]);
        if (lane == 0) G[pi * 9 + a * 3 + b] = s * JJ;
      }
    if (lane == 0) my += (unsigned long long)nn * nn;
    __syncwarp();
  }
  if (lane == 0 && evals && my) atomicAdd(evals, my);
}

__global__ void split_keys_kernel(const unsigned long long* keys, int64_t n, int* P, int* Q, int* K,
                                  unsigned long long* hkey, int* hidx, unsigned long long hmask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long key = keys[i];
  P[i] = (int)(key >> 34);
  Q[i] = (int)((key >> 6) & ((1ull << 28) - 1));
  K[i] = (int)(key & 63);
  unsigned long long h = near_hash(key) & hmask;
  for (;;) {
    const unsigned long long prev = atomicCAS(&hkey[h], NEAR_EMPTY, key);
    if (prev == NEAR_EMPTY) { hidx[h] = (int)i; break; }
    h = (h + 1) & hmask;
  }
}
#define FL_E4_SWITCHN(e4, ...)                                \
  switch (e4) {                                               \
    case 6: { constexpr int E4 = 6; __VA_ARGS__; } break;     \
    case 8: { constexpr int E4 = 8; __VA_ARGS__; } break;     \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

void near_pairs_build(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                      unsigned long long* keys, int64_t nkeys, NearPairs& np, unsigned long long* evals,
                      cudaStream_t st) {
  np.n = 0;
  if (nkeys <= 0) {
    np.U.alloc(1); np.P.alloc(1); np.Q.alloc(1); np.K.alloc(1); np.G.alloc(1);
    np.hkey.alloc(1); np.hidx.alloc(1); np.hmask = 0;
    FL_CUDA(cudaMemsetAsync(np.hkey.p, 0xff, sizeof(unsigned long long), st));
    return;
  }
  // sort + unique of the (min, max) keys: deterministic order of the pairs
  DBuf<unsigned long long> sorted(nkeys);
  np.U.alloc(nkeys);
  DBuf<int> nsel(1);
  {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, sorted.p, (int)nkeys, 0, 64, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, tmp, keys, sorted.p, (int)nkeys, 0, 64, st));
    size_t tmp2 = 0;
    cub::DeviceSelect::Unique(nullptr, tmp2, sorted.p, np.U.p, nsel.p, (int)nkeys, st);
    DBuf<unsigned char> tb2(tmp2);
    FL_CUDA(cub::DeviceSelect::Unique(tb2.p, tmp2, sorted.p, np.U.p, nsel.p, (int)nkeys, st));
  }
  int nu = 0;
  FL_CUDA(cudaMemcpyAsync(&nu, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  np.n = nu;
  np.P.alloc(nu); np.Q.alloc(nu); np.K.alloc(nu); np.G.alloc((size_t)nu * 9);
  unsigned long long cap = 1024;
  while (cap < 2ull * (unsigned long long)nu) cap <<= 1;
  np.hmask = cap - 1;
  np.hkey.alloc(cap); np.hidx.alloc(cap);
  FL_CUDA(cudaMemsetAsync(np.hkey.p, 0xff, cap * sizeof(unsigned long long), st));
  split_keys_kernel<<<(nu + 255) / 256, 256, 0, st>>>(np.U.p, nu, np.P.p, np.Q.p, np.K.p, np.hkey.p, np.hidx.p,
                                                       np.hmask), ::fl::note_launch();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((nu + NW - 1) / NW, (int64_t)sms * 8);
  if (m.d == 1) {
    FL_E4_SWITCHN(e4, (near_block_kernel<1, E4><<<grid, NW * 32, 0, st>>>(m, t.data, t, oc, ex, np.P.p, np.Q.p, np.K.p,
                                                                         nu, np.G.p, evals), ::fl::note_launch()));
  } else {
    FL_E4_SWITCHN(e4, (near_block_kernel<2, E4><<<grid, NW * 32, 0, st>>>(m, t.data, t, oc, ex, np.P.p, np.Q.p, np.K.p,
                                                                         nu, np.G.p, evals), ::fl::note_launch()));
  }
  FL_CHECK_LAUNCH();
}

void launch_near_blocks(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                        const int* P, const int* Q, const int* K, int64_t n, double* G, unsigned long long* evals,
                        cudaStream_t st) {
  if (n <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n + NW - 1) / NW, (int64_t)sms * 8);
  if (m.d == 1) {
    FL_E4_SWITCHN(e4, (near_block_kernel<1, E4><<<grid, NW * 32, 0, st>>>(m, t.data, t, oc, ex, P, Q, K, n, G, evals),
                       ::fl::note_launch()));
  } else {
    FL_E4_SWITCHN(e4, (near_block_kernel<2, E4><<<grid, NW * 32, 0, st>>>(m, t.data, t, oc, ex, P, Q, K, n, G, evals),
                       ::fl::note_launch()));
  }
  FL_CHECK_LAUNCH();
}

}  // namespace fl
