// Cluster (H-matrix) operator on the device: ClusterOperator.matvec (cluster.py:417-456) —
// y = A_near x - C * far(x) with the Chebyshev far field of cluster.compress (:667-712):
//
//   leaf moments   mom[leaf] = sum_{i in leaf} x_i basis_coef[i, :]            (_moments, :427-434)
//   upward pass    mom[parent] += S_child mom[child]   (2D: S0 V S1^T)        (ChebData.push_up, :339-356)
//   far blocks     F[a] += B_p mom[b],  F[b] += B_p^T mom[a]  over far pairs  (_far_potentials, :436-447)
//   downward pass  F[child] += S_child^T F[parent]   (2D: S0^T V S1)         (ChebData.push_down, :358-374)
//   evaluation     y_far[i] = basis_coef[i, :] . F[leaf(i)]                   (far_apply, :449-457)
//
// Every accumulation has the reference's order (children of a parent in reversed BFS order;
// far contributions first as the pair's first node in pair order, then as its second node), so
// results are deterministic; the near CSR product is a warp-per-row fixed-order reduction.
// The far blocks B_p = |xi_a - xi_b|^(2 ex) at the Chebyshev points (compress, :683-694) are
// either uploaded or built here (one thread per block entry).
#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include <cooperative_groups.h>

#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

struct fl_cluster {
  int device = 0, d = 1, m = 0, M = 0;
  int64_t n = 0, nn = 0, np = 0;
  double C = 0.0;
  fl::DBuf<int64_t> indptr;
  fl::DBuf<int> indices;
  fl::DBuf<double> data, diag;
  fl::DBuf<double> shift, bc, blocks, mom, F, Fp, x, y, yfar;
  fl::DBuf<int> leaf_nodes, leaf_lo, leaf_hi, dof_perm, leaf_of_dof, children, parent, pairs, plist_off, plist,
      level_nodes;
  std::vector<int64_t> level_off_up, level_off_down;   // offsets into level_nodes (host copies)
  fl::DBuf<int64_t> d_off_up, d_off_down;               // ... and device copies (fused far field)
  fl::DBuf<double> center, half, ref;                   // node boxes and Chebyshev nodes (point evaluation)
  bool fused = false;
  int coop_blocks = 0;                                  // resident blocks of the cooperative far field
  int nleaves = 0;
  // fused schedule: subtrees of <= S nodes, each finished by one block (moments, upward and
  // downward passes, evaluation) with block barriers; the nodes above them ("top") by block 0
  fl::DBuf<int> sub_info, grp_off, grp_nodes, sub_leaves;
  int nsub = 0, top_g0 = 0, top_g1 = 0;
  fl::DBuf<int> early, late;                            // far pairs before / after the top levels
  int64_t n_early = 0, n_late = 0;
  cudaStream_t stream = nullptr;
  ~fl_cluster() {
    for (auto* b : {&data, &diag, &shift, &bc, &blocks, &mom, &F, &Fp, &x, &y, &yfar}) b->free();
    for (auto* b : {&leaf_nodes, &leaf_lo, &leaf_hi, &dof_perm, &leaf_of_dof, &children, &parent, &pairs, &plist_off,
                    &plist, &level_nodes})
      b->free();
    indptr.free();
    indices.free();
    d_off_up.free();
    d_off_down.free();
    center.free();
    half.free();
    ref.free();
    if (stream) fl::release_stream(device, stream);
  }
};

namespace fl {
namespace {

int grid_of(int64_t m, int b = 256) { return (int)std::max<int64_t>(1, (m + b - 1) / b); }

__global__ void csr_spmv_kernel(int64_t n, const int64_t* __restrict__ indptr, const int* __restrict__ idx,
                                const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) s = fma(val[e], x[idx[e]], s);
  s = warp_sum(s);
  if (lane == 0) y[i] = s;
}

// mom[leaf] = x[dofs] @ basis_coef[dofs]   (dofs in dof_perm order); other nodes zeroed
__global__ void moments_kernel(int nleaves, const int* __restrict__ leaf_nodes, const int* __restrict__ lo,
                               const int* __restrict__ hi, const int* __restrict__ perm, const double* __restrict__ x,
                               const double* __restrict__ bc, int M, double* __restrict__ mom) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nleaves * M) return;
  const int l = (int)(t / M), a = (int)(t % M);
  double s = 0.0;
  for (int r = lo[l]; r < hi[l]; ++r) {
    const int i = perm[r];
    s = fma(x[i], bc[(int64_t)i * M + a], s);
  }
  mom[(int64_t)leaf_nodes[l] * M + a] = s;
}

// out[a0, a1] += sum_b1 S1[a1, b1] (sum_b0 S0[a0, b0] V[b0, b1])   (2D; 1D: sum_b S0[a, b] v[b])
template <int D>
__device__ __forceinline__ double shift_apply(const double* __restrict__ S, const double* __restrict__ v, int m,
                                              int a, bool transpose) {
  if (D == 1) {
    double s = 0.0;
    for (int b = 0; b < m; ++b) s = fma(transpose ? S[b * m + a] : S[a * m + b], v[b], s);
    return s;
  } else {
    const double* S0 = S;
    const double* S1 = S + m * m;
    const int a0 = a / m, a1 = a % m;
    double s = 0.0;
    for (int b1 = 0; b1 < m; ++b1) {
      double t = 0.0;
      for (int b0 = 0; b0 < m; ++b0) t = fma(transpose ? S0[b0 * m + a0] : S0[a0 * m + b0], v[b0 * m + b1], t);
      s = fma(t, transpose ? S1[b1 * m + a1] : S1[a1 * m + b1], s);
    }
    return s;
  }
}

// 1D, m <= 16: the operands of one shift product (a row / column of S and the vector) loaded into
// registers before the FMA chain, so a level costs one memory round trip instead of one per
// unrolled chunk; the FMA order is shift_apply<1>'s
struct Row16 {
  double s[16], v[16];
};
__device__ __forceinline__ void load_row16(Row16& r, const double* __restrict__ S, const double* __restrict__ v, int m,
                                           int a, bool transpose) {
#pragma unroll
  for (int b = 0; b < 16; ++b)
    if (b < m) {
      r.s[b] = transpose ? S[b * m + a] : S[a * m + b];
      r.v[b] = v[b];
    }
}
__device__ __forceinline__ double dot_row16(const Row16& r, int m) {
  double s = 0.0;
#pragma unroll
  for (int b = 0; b < 16; ++b)
    if (b < m) s = fma(r.s[b], r.v[b], s);
  return s;
}

// 2D, m <= 6: the same for S0 V S1^T (shift_apply<2>'s order)
struct Mat6 {
  double s0[6], s1[6], v[36];
};
__device__ __forceinline__ void load_mat6(Mat6& r, const double* __restrict__ S, const double* __restrict__ v, int m,
                                          int a, bool transpose) {
  const double* S0 = S;
  const double* S1 = S + m * m;
  const int a0 = a / m, a1 = a % m;
#pragma unroll
  for (int b = 0; b < 6; ++b)
    if (b < m) {
      r.s0[b] = transpose ? S0[b * m + a0] : S0[a0 * m + b];
      r.s1[b] = transpose ? S1[b * m + a1] : S1[a1 * m + b];
    }
#pragma unroll
  for (int b0 = 0; b0 < 6; ++b0)
#pragma unroll
    for (int b1 = 0; b1 < 6; ++b1)
      if (b0 < m && b1 < m) r.v[b0 * 6 + b1] = v[b0 * m + b1];
}
__device__ __forceinline__ double dot_mat6(const Mat6& r, int m) {
  double s = 0.0;
#pragma unroll
  for (int b1 = 0; b1 < 6; ++b1)
    if (b1 < m) {
      double t = 0.0;
#pragma unroll
      for (int b0 = 0; b0 < 6; ++b0)
        if (b0 < m) t = fma(r.s0[b0], r.v[b0 * 6 + b1], t);
      s = fma(t, r.s1[b1], s);
    }
  return s;
}

// shift_apply<D> with the operands in registers first where they fit (same FMA order)
template <int D>
__device__ __forceinline__ double shift_apply_fast(const double* __restrict__ S, const double* __restrict__ v, int m,
                                                   int a, bool transpose) {
  if (D == 1 && m <= 16) {
    Row16 r;
    load_row16(r, S, v, m, a, transpose);
    return dot_row16(r, m);
  }
  if (D == 2 && m <= 6) {
    Mat6 r;
    load_mat6(r, S, v, m, a, transpose);
    return dot_mat6(r, m);
  }
  return shift_apply<D>(S, v, m, a, transpose);
}

// upward: one thread per (parent, alpha): children in reversed BFS order (second child first)
template <int D>
__global__ void up_kernel(const int* __restrict__ nodes, int cnt, const int* __restrict__ children,
                          const double* __restrict__ shift, int m, int M, double* __restrict__ mom) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)cnt * M) return;
  const int p = nodes[t / M], a = (int)(t % M);
  double acc = mom[(int64_t)p * M + a];
  for (int k = 1; k >= 0; --k) {
    const int c = children[2 * p + k];
    if (c < 0) continue;
    acc += shift_apply_fast<D>(shift + (int64_t)c * D * m * m, mom + (int64_t)c * M, m, a, false);
  }
  mom[(int64_t)p * M + a] = acc;
}

// far pairs: Fp[p] = (B mom[b], B^T mom[a])
__global__ void far_pair_kernel(int64_t np, const int* __restrict__ pairs, const double* __restrict__ B, int M,
                                const double* __restrict__ mom, double* __restrict__ Fp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np * 2 * M) return;
  const int64_t p = t / (2 * M);
  const int r = (int)(t % (2 * M));
  const double* Bp = B + p * M * M;
  double s = 0.0;
  if (r < M) {
    const double* mb = mom + (int64_t)pairs[2 * p + 1] * M;
    for (int b = 0; b < M; ++b) s = fma(Bp[(int64_t)r * M + b], mb[b], s);
  } else {
    const int c = r - M;
    const double* ma = mom + (int64_t)pairs[2 * p] * M;
    for (int a = 0; a < M; ++a) s = fma(Bp[(int64_t)a * M + c], ma[a], s);
  }
  Fp[t] = s;
}
// F[node] = sum over its pair list (as first node, pair order, then as second node, pair order)
__global__ void far_gather_kernel(int64_t nn, const int* __restrict__ off, const int* __restrict__ lst, int M,
                                  const double* __restrict__ Fp, double* __restrict__ F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nn * M) return;
  const int64_t nd = t / M;
  const int a = (int)(t % M);
  double s = 0.0;
  for (int k = off[nd]; k < off[nd + 1]; ++k) {
    const int e = lst[k];                  // 2 p + role
    s += Fp[(int64_t)(e >> 1) * 2 * M + (e & 1) * M + a];
  }
  F[t] = s;
}

// downward: one thread per (child, alpha): F[child] += S^T F[parent]
template <int D>
__global__ void down_kernel(const int* __restrict__ nodes, int cnt, const int* __restrict__ parent,
                            const double* __restrict__ shift, int m, int M, double* __restrict__ F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)cnt * M) return;
  const int c = nodes[t / M], a = (int)(t % M);
  F[(int64_t)c * M + a] += shift_apply_fast<D>(shift + (int64_t)c * D * m * m, F + (int64_t)parent[c] * M, m, a, true);
}

// y[i] = y_near[i] - C * basis_coef[i, :] . F[leaf(i)]
__global__ void eval_kernel(int64_t n, const int* __restrict__ leaf_of_dof, const double* __restrict__ bc, int M,
                            const double* __restrict__ F, double negC, double* __restrict__ y,
                            double* __restrict__ yfar) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* f = F + (int64_t)leaf_of_dof[i] * M;
  double s = 0.0;
  for (int a = 0; a < M; ++a) s = fma(bc[i * M + a], f[a], s);
  const double v = negC * s;
  yfar[i] = v;
  y[i] += v;
}

// The whole far field in ONE cooperative launch (small / medium operators, e.g. 1D at c2: ~2k
// nodes, M <= 12): the same phases and accumulation orders as the kernels above, separated by
// grid-wide barriers instead of ~2 x depth + 4 launches.
// one level group of the upward pass inside a block: mom[p] += S_c mom[c] over both children
template <int D>
__device__ __forceinline__ void up_group(const int* __restrict__ nodes, int cnt, const int* __restrict__ children,
                                         const double* __restrict__ shift, int m, int M, double* __restrict__ mom,
                                         bool internal_zero) {
  for (int t = threadIdx.x; t < cnt * M; t += blockDim.x) {
    const int p = nodes[t / M], a = t % M;
    double acc = internal_zero ? 0.0 : mom[(int64_t)p * M + a];
    if (D == 1 && m <= 16) {
      const int c1 = children[2 * p + 1], c0 = children[2 * p];
      Row16 r1, r0;
      if (c1 >= 0) load_row16(r1, shift + (int64_t)c1 * m * m, mom + (int64_t)c1 * M, m, a, false);
      if (c0 >= 0) load_row16(r0, shift + (int64_t)c0 * m * m, mom + (int64_t)c0 * M, m, a, false);
      if (c1 >= 0) acc += dot_row16(r1, m);
      if (c0 >= 0) acc += dot_row16(r0, m);
    } else if (D == 2 && m <= 6) {
      const int c1 = children[2 * p + 1], c0 = children[2 * p];
      Mat6 r1, r0;
      if (c1 >= 0) load_mat6(r1, shift + (int64_t)c1 * 2 * m * m, mom + (int64_t)c1 * M, m, a, false);
      if (c0 >= 0) load_mat6(r0, shift + (int64_t)c0 * 2 * m * m, mom + (int64_t)c0 * M, m, a, false);
      if (c1 >= 0) acc += dot_mat6(r1, m);
      if (c0 >= 0) acc += dot_mat6(r0, m);
    } else {
      for (int k = 1; k >= 0; --k) {
        const int c = children[2 * p + k];
        if (c >= 0) acc += shift_apply<D>(shift + (int64_t)c * D * m * m, mom + (int64_t)c * M, m, a, false);
      }
    }
    mom[(int64_t)p * M + a] = acc;
  }
}
// one level group of the downward pass: F[c] += S_c^T F[p] for both children of every p
template <int D>
__device__ __forceinline__ void down_group(const int* __restrict__ nodes, int cnt, const int* __restrict__ children,
                                           const double* __restrict__ shift, int m, int M, double* __restrict__ F) {
  for (int t = threadIdx.x; t < cnt * 2 * M; t += blockDim.x) {
    const int p = nodes[t / (2 * M)], k = (t / M) & 1, a = t % M;
    const int c = children[2 * p + k];
    if (c < 0) continue;
    if (D == 1 && m <= 16) {
      Row16 r;
      load_row16(r, shift + (int64_t)c * m * m, F + (int64_t)p * M, m, a, true);
      const double f = F[(int64_t)c * M + a];
      F[(int64_t)c * M + a] = f + dot_row16(r, m);
    } else if (D == 2 && m <= 6) {
      Mat6 r;
      load_mat6(r, shift + (int64_t)c * 2 * m * m, F + (int64_t)p * M, m, a, true);
      const double f = F[(int64_t)c * M + a];
      F[(int64_t)c * M + a] = f + dot_mat6(r, m);
    } else {
      F[(int64_t)c * M + a] += shift_apply<D>(shift + (int64_t)c * D * m * m, F + (int64_t)p * M, m, a, true);
    }
  }
}

// Fp[p] = (B_p mom[b], B_p^T mom[a]) for the pairs listed  (_far_potentials, cluster.py:436-447)
__device__ __forceinline__ void far_pair_items(int64_t cnt, const int* __restrict__ list, const int* __restrict__ pairs,
                                               const double* __restrict__ B, int M, const double* __restrict__ mom,
                                               double* __restrict__ Fp, int64_t tid, int64_t nt) {
  for (int64_t t = tid; t < cnt * 2 * M; t += nt) {
    const int64_t p = list[t / (2 * M)];
    const int r = (int)(t % (2 * M));
    const double* Bp = B + p * M * M;
    double s = 0.0;
    if (r < M) {
      const double* mb = mom + (int64_t)pairs[2 * p + 1] * M;
      for (int b = 0; b < M; ++b) s = fma(Bp[(int64_t)r * M + b], mb[b], s);
    } else {
      const double* ma = mom + (int64_t)pairs[2 * p] * M;
      for (int a = 0; a < M; ++a) s = fma(Bp[(int64_t)a * M + (r - M)], ma[a], s);
    }
    Fp[p * 2 * M + r] = s;
  }
}

// The whole far field in one cooperative launch with five grid barriers.  Per node the arithmetic
// (and so the result) is that of the level-by-level passes (ChebData.push_up / push_down,
// cluster.py:339-374): the schedule only changes which block runs a node, and when.
//   sub_info[6j..]: group range [g0, g1) (deepest first), leaf range [l0, l1) of sub_leaves,
//   dof range [r0, r1) of dof_perm;  groups: grp_nodes[grp_off[g] .. grp_off[g+1]) (parents only)
template <int D>
__global__ void __launch_bounds__(256) far_fused_kernel(
    int nsub, const int* __restrict__ sub_info, const int* __restrict__ grp_off, const int* __restrict__ grp_nodes,
    const int* __restrict__ sub_leaves, int top_g0, int top_g1, const int* __restrict__ leaf_nodes,
    const int* __restrict__ lo, const int* __restrict__ hi, const int* __restrict__ perm, const double* __restrict__ x,
    const double* __restrict__ bc, int m, int M, int64_t nn, const int* __restrict__ children,
    const double* __restrict__ shift, int64_t np, const int* __restrict__ pairs, const double* __restrict__ B,
    const int* __restrict__ poff, const int* __restrict__ plist, double* __restrict__ mom, double* __restrict__ Fp,
    double* __restrict__ F, const int* __restrict__ leaf_of_dof, double negC, double* __restrict__ y,
    double* __restrict__ yfar, int64_t n, const int64_t* __restrict__ indptr, const int* __restrict__ idx,
    const double* __restrict__ val, int64_t n_early, const int* __restrict__ early, int64_t n_late,
    const int* __restrict__ late) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  // 1. subtrees: leaf moments, then the upward pass to the subtree root
  for (int j = blockIdx.x; j < nsub; j += gridDim.x) {
    const int* I = sub_info + 6 * j;
    for (int t = threadIdx.x; t < (I[3] - I[2]) * M; t += blockDim.x) {
      const int l = sub_leaves[I[2] + t / M], a = t % M;
      double s = 0.0;
      for (int r = lo[l]; r < hi[l]; ++r) s = fma(x[perm[r]], bc[(int64_t)perm[r] * M + a], s);
      mom[(int64_t)leaf_nodes[l] * M + a] = s;
    }
    for (int g = I[0]; g < I[1]; ++g) {
      __syncthreads();
      up_group<D>(grp_nodes + grp_off[g], grp_off[g + 1] - grp_off[g], children, shift, m, M, mom, true);
    }
    __syncthreads();
  }
  grid.sync();
  // 2. block 0: the nodes above the subtrees; the other blocks meanwhile: the near CSR product
  //    (warp per row, as csr_spmv_kernel) and the far pairs whose two nodes are final already
  const bool has_top = top_g1 > top_g0, split = has_top && gridDim.x > 1;
  if (has_top && blockIdx.x == 0) {
    for (int g = top_g0; g < top_g1; ++g) {
      up_group<D>(grp_nodes + grp_off[g], grp_off[g + 1] - grp_off[g], children, shift, m, M, mom, true);
      __syncthreads();
    }
  }
  if (!split || blockIdx.x != 0) {
    const int64_t b0 = split ? 1 : 0;
    const int64_t ltid = (int64_t)(blockIdx.x - b0) * blockDim.x + threadIdx.x;
    const int64_t lnt = (int64_t)(gridDim.x - b0) * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t w = ltid >> 5; w < n; w += lnt >> 5) {
      double s = 0.0;
      for (int64_t e = indptr[w] + lane; e < indptr[w + 1]; e += 32) s = fma(val[e], x[idx[e]], s);
      s = warp_sum(s);
      if (lane == 0) y[w] = s;
    }
    far_pair_items(n_early, early, pairs, B, M, mom, Fp, ltid, lnt);
  }
  grid.sync();
  // 3. the remaining far pairs
  far_pair_items(n_late, late, pairs, B, M, mom, Fp, tid, nt);
  grid.sync();
  // 4. gather the pair contributions of every node
  for (int64_t t = tid; t < nn * M; t += nt) {
    const int64_t nd = t / M;
    const int a = (int)(t % M);
    double s = 0.0;
    for (int k = poff[nd]; k < poff[nd + 1]; ++k) {
      const int e = plist[k];
      s += Fp[(int64_t)(e >> 1) * 2 * M + (e & 1) * M + a];
    }
    F[t] = s;
  }
  grid.sync();
  // 5. downward pass above the subtrees (down to the subtree roots), one block
  if (top_g1 > top_g0) {
    if (blockIdx.x == 0)
      for (int g = top_g1 - 1; g >= top_g0; --g) {
        down_group<D>(grp_nodes + grp_off[g], grp_off[g + 1] - grp_off[g], children, shift, m, M, F);
        __syncthreads();
      }
    grid.sync();
  }
  // 6. subtrees: downward pass to the leaves, then y_far = -C basis_coef . F[leaf]
  for (int j = blockIdx.x; j < nsub; j += gridDim.x) {
    const int* I = sub_info + 6 * j;
    for (int g = I[1] - 1; g >= I[0]; --g) {
      down_group<D>(grp_nodes + grp_off[g], grp_off[g + 1] - grp_off[g], children, shift, m, M, F);
      __syncthreads();
    }
    for (int r = I[4] + threadIdx.x; r < I[5]; r += blockDim.x) {
      const int i = perm[r];
      const double* f = F + (int64_t)leaf_of_dof[i] * M;
      double s = 0.0;
      for (int a = 0; a < M; ++a) s = fma(bc[(int64_t)i * M + a], f[a], s);
      const double v = negC * s;
      yfar[i] = v;
      y[i] += v;
    }
    __syncthreads();
  }
}

template <int E4>
__global__ void far_blocks_kernel(int64_t np, const int* __restrict__ pairs, const double* __restrict__ pts, int d,
                                  int M, double ex, double* __restrict__ B) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np * M * M) return;
  const int64_t p = t / ((int64_t)M * M);
  const int r = (int)(t % ((int64_t)M * M)), a = r / M, b = r % M;
  const double* Pa = pts + ((int64_t)pairs[2 * p] * M + a) * d;
  const double* Pb = pts + ((int64_t)pairs[2 * p + 1] * M + b) * d;
  double r2 = 0.0;
  for (int j = 0; j < d; ++j) {
    const double df = Pa[j] - Pb[j];
    r2 = __dadd_rn(r2, __dmul_rn(df, df));
  }
  B[t] = kpow<E4>(r2, ex);
}

}  // namespace

int32_t cluster_create(const fl_cluster_desc* Dd, int device, fl_cluster** out) {
  const fl_cluster_desc& D = *Dd;
  if (D.d != 1 && D.d != 2) throw Error(FL_E_ARG, "cluster: d must be 1 or 2");
  if (D.m < 1 || D.n < 0 || D.num_nodes < 1) throw Error(FL_E_ARG, "cluster: bad sizes");
  const int d = D.d, m = D.m;
  const int M = d == 1 ? m : m * m;
  const int64_t n = D.n, nn = D.num_nodes, np = D.npairs;
  if (n >= (1LL << 31) || nn >= (1LL << 30) || np >= (1LL << 30)) throw Error(FL_E_ARG, "cluster: too large");
  // host-side structure: children, levels, leaves, per-node pair lists (validated)
  std::vector<int> children(2 * nn, -1), par(nn), depth(nn, -1);
  for (int64_t k = 0; k < nn; ++k) {
    const int64_t p = D.parent[k];
    if (p < -1 || p >= nn) throw Error(FL_E_ARG, "cluster: parent out of range");
    par[k] = (int)p;
  }
  for (int64_t t = 0; t < nn; ++t) {                 // BFS order: children appended in order
    const int64_t k = D.topo_order[t];
    if (k < 0 || k >= nn) throw Error(FL_E_ARG, "cluster: topo_order out of range");
    if (par[k] < 0) { depth[k] = 0; continue; }
    const int p = par[k];
    if (depth[p] < 0) throw Error(FL_E_ARG, "cluster: topo_order lists a child before its parent");
    depth[k] = depth[p] + 1;
    if (children[2 * p] < 0) children[2 * p] = (int)k;
    else if (children[2 * p + 1] < 0) children[2 * p + 1] = (int)k;
    else throw Error(FL_E_ARG, "cluster: more than two children");
  }
  int maxd = 0;
  for (int64_t k = 0; k < nn; ++k) maxd = std::max(maxd, depth[k]);
  std::vector<int> leaf_nodes, lo, hi, lod(std::max<int64_t>(n, 1), -1);
  for (int64_t k = 0; k < nn; ++k) {
    if (children[2 * k] >= 0) continue;
    const int64_t a = D.ranges[2 * k], b = D.ranges[2 * k + 1];
    if (a < 0 || b > n || a > b) throw Error(FL_E_ARG, "cluster: node range out of bounds");
    leaf_nodes.push_back((int)k);
    lo.push_back((int)a);
    hi.push_back((int)b);
    for (int64_t r = a; r < b; ++r) {
      const int64_t i = D.dof_perm[r];
      if (i < 0 || i >= n) throw Error(FL_E_ARG, "cluster: dof_perm out of range");
      lod[i] = (int)k;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (lod[i] < 0) throw Error(FL_E_ARG, "cluster: a DoF lies in no leaf");
  // levels: parents with children at depth L (upward, deepest first); nodes at depth L (downward)
  std::vector<int> lvl_nodes;
  std::vector<int64_t> off_up{0}, off_down;
  for (int L = maxd - 1; L >= 0; --L) {
    for (int64_t t = 0; t < nn; ++t) {
      const int64_t k = D.topo_order[t];
      if (depth[k] == L && children[2 * k] >= 0) lvl_nodes.push_back((int)k);
    }
    off_up.push_back((int64_t)lvl_nodes.size());
  }
  off_down.push_back((int64_t)lvl_nodes.size());
  for (int L = 1; L <= maxd; ++L) {
    for (int64_t t = 0; t < nn; ++t) {
      const int64_t k = D.topo_order[t];
      if (depth[k] == L) lvl_nodes.push_back((int)k);
    }
    off_down.push_back((int64_t)lvl_nodes.size());
  }
  // fused schedule: subtree roots = maximal nodes of <= S nodes; their internal nodes grouped by
  // depth (deepest first), then the nodes above them ("top") grouped the same way
  const int S = getenv("FRACLAP_SUBTREE_NODES") ? std::max(1, atoi(getenv("FRACLAP_SUBTREE_NODES")))
                                                 : (int)std::max<int64_t>(32, nn / 128);
  std::vector<int64_t> tsize(nn, 1);
  for (int64_t t = nn - 1; t >= 0; --t) {
    const int64_t k = D.topo_order[t];
    if (par[k] >= 0) tsize[par[k]] += tsize[k];
  }
  std::vector<int> leaf_index(nn, -1);
  for (size_t l = 0; l < leaf_nodes.size(); ++l) leaf_index[leaf_nodes[l]] = (int)l;
  std::vector<int> sub_info, grp_off{0}, grp_nodes, sub_leaves;
  int64_t covered = 0;
  for (int64_t t = 0; t < nn; ++t) {
    const int64_t root = D.topo_order[t];
    if (tsize[root] > S || (par[root] >= 0 && tsize[par[root]] <= S)) continue;
    std::vector<int> bfs{(int)root};
    for (size_t u = 0; u < bfs.size(); ++u)
      for (int k = 0; k < 2; ++k)
        if (children[2 * bfs[u] + k] >= 0) bfs.push_back(children[2 * bfs[u] + k]);
    int dmax = depth[root];
    for (int k : bfs) dmax = std::max(dmax, depth[k]);
    sub_info.push_back((int)grp_off.size() - 1);
    for (int L = dmax - 1; L >= depth[root]; --L) {
      size_t before = grp_nodes.size();
      for (int k : bfs)
        if (depth[k] == L && children[2 * k] >= 0) grp_nodes.push_back(k);
      if (grp_nodes.size() > before) grp_off.push_back((int)grp_nodes.size());
    }
    sub_info.push_back((int)grp_off.size() - 1);
    sub_info.push_back((int)sub_leaves.size());
    for (int k : bfs)
      if (leaf_index[k] >= 0) sub_leaves.push_back(leaf_index[k]);
    sub_info.push_back((int)sub_leaves.size());
    sub_info.push_back((int)D.ranges[2 * root]);
    sub_info.push_back((int)D.ranges[2 * root + 1]);
    covered += D.ranges[2 * root + 1] - D.ranges[2 * root];
  }
  const int top_g0 = (int)grp_off.size() - 1;
  for (int L = maxd - 1; L >= 0; --L) {
    size_t before = grp_nodes.size();
    for (int64_t t = 0; t < nn; ++t) {
      const int64_t k = D.topo_order[t];
      if (depth[k] == L && tsize[k] > S && children[2 * k] >= 0) grp_nodes.push_back((int)k);
    }
    if (grp_nodes.size() > before) grp_off.push_back((int)grp_nodes.size());
  }
  const int top_g1 = (int)grp_off.size() - 1;
  // pair lists per node: first-node roles in pair order, then second-node roles
  std::vector<int> prs(std::max<int64_t>(2 * np, 1)), cnt(nn + 1, 0);
  for (int64_t p = 0; p < np; ++p) {
    const int64_t a = D.far_pairs[2 * p], b = D.far_pairs[2 * p + 1];
    if (a < 0 || b < 0 || a >= nn || b >= nn) throw Error(FL_E_ARG, "cluster: far pair out of range");
    prs[2 * p] = (int)a;
    prs[2 * p + 1] = (int)b;
    cnt[a + 1]++;
    cnt[b + 1]++;
  }
  for (int64_t k = 0; k < nn; ++k) cnt[k + 1] += cnt[k];
  std::vector<int> lst(std::max<int64_t>(2 * np, 1)), fill(cnt.begin(), cnt.end() - 1);
  for (int role = 0; role < 2; ++role)
    for (int64_t p = 0; p < np; ++p) lst[fill[prs[2 * p + role]]++] = (int)(2 * p + role);
  // far pairs whose nodes are both inside subtrees run while block 0 does the top levels
  std::vector<int> early, late;
  for (int64_t p = 0; p < np; ++p)
    (tsize[prs[2 * p]] > S || tsize[prs[2 * p + 1]] > S ? late : early).push_back((int)p);

  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  std::unique_ptr<fl_cluster> C(new fl_cluster());
  C->device = device;
  C->stream = acquire_stream(device);
  cudaStream_t st = C->stream;
  StreamScope scope(st);
  C->d = d; C->m = m; C->M = M; C->n = n; C->nn = nn; C->np = np; C->C = D.C;
  C->nleaves = (int)leaf_nodes.size();
  C->level_off_up = off_up;
  C->level_off_down = off_down;
  auto up_i = [&](DBuf<int>& b, const std::vector<int>& h) {
    b.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty()) FL_CUDA(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  };
  auto up_d = [&](DBuf<double>& b, const double* h, size_t cnt_) {
    b.alloc(std::max<size_t>(cnt_, 1));
    if (cnt_) FL_CUDA(cudaMemcpyAsync(b.p, h, cnt_ * sizeof(double), cudaMemcpyHostToDevice, st));
  };
  std::vector<int> perm(std::max<int64_t>(n, 1));
  for (int64_t r = 0; r < n; ++r) perm[r] = (int)D.dof_perm[r];
  up_i(C->leaf_nodes, leaf_nodes); up_i(C->leaf_lo, lo); up_i(C->leaf_hi, hi); up_i(C->dof_perm, perm);
  up_i(C->leaf_of_dof, lod); up_i(C->children, children); up_i(C->parent, par); up_i(C->pairs, prs);
  up_i(C->plist_off, cnt); up_i(C->plist, lst); up_i(C->level_nodes, lvl_nodes);
  up_i(C->early, early); up_i(C->late, late);
  C->n_early = (int64_t)early.size();
  C->n_late = (int64_t)late.size();
  up_i(C->sub_info, sub_info); up_i(C->grp_off, grp_off); up_i(C->grp_nodes, grp_nodes);
  up_i(C->sub_leaves, sub_leaves);
  C->nsub = (int)(sub_info.size() / 6);
  C->top_g0 = top_g0;
  C->top_g1 = top_g1;
  up_d(C->shift, D.shift, (size_t)nn * d * m * m);
  up_d(C->bc, D.basis_coef, (size_t)n * M);
  if (D.center && D.half && D.ref) {
    up_d(C->center, D.center, (size_t)nn * d);
    up_d(C->half, D.half, (size_t)nn);
    up_d(C->ref, D.ref, (size_t)m);
  }
  // near CSR
  if (D.nnz < 0 || (D.nnz > 0 && (!D.indptr || !D.indices || !D.data))) throw Error(FL_E_ARG, "cluster: bad near CSR");
  C->indptr.alloc(n + 1);
  FL_CUDA(cudaMemcpyAsync(C->indptr.p, D.indptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  std::vector<int> ci(std::max<int64_t>(D.nnz, 1));
  for (int64_t e = 0; e < D.nnz; ++e) {
    if (D.indices[e] < 0 || D.indices[e] >= n) throw Error(FL_E_ARG, "cluster: near column out of range");
    ci[e] = (int)D.indices[e];
  }
  up_i(C->indices, ci);
  up_d(C->data, D.data, (size_t)D.nnz);
  // far blocks: uploaded, or built from the Chebyshev points
  C->blocks.alloc(std::max<int64_t>(np * M * M, 1));
  if (np > 0) {
    if (D.far_blocks) {
      FL_CUDA(cudaMemcpyAsync(C->blocks.p, D.far_blocks, (size_t)np * M * M * sizeof(double), cudaMemcpyHostToDevice,
                              st));
    } else {
      if (!D.points) throw Error(FL_E_ARG, "cluster: neither far blocks nor Chebyshev points given");
      DBuf<double> pts;
      up_d(pts, D.points, (size_t)nn * M * d);
      const double ex = -(d / 2.0 + D.s);
      const int e4 = (D.s == 0.25 || D.s == 0.5 || D.s == 0.75) ? (int)std::lround(4.0 * (d + 2.0 * D.s)) : 0;
      const int64_t tot = np * M * M;
      switch (e4) {
        case 6: far_blocks_kernel<6><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
        case 8: far_blocks_kernel<8><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
        case 10: far_blocks_kernel<10><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
        case 12: far_blocks_kernel<12><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
        case 14: far_blocks_kernel<14><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
        default: far_blocks_kernel<0><<<grid_of(tot), 256, 0, st>>>(np, C->pairs.p, pts.p, d, M, ex, C->blocks.p); break;
      }
      note_launch();
      FL_CHECK_LAUNCH();
      FL_CUDA(cudaStreamSynchronize(st));
    }
  }
  auto up_l = [&](DBuf<int64_t>& b, const std::vector<int64_t>& h) {
    b.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty()) FL_CUDA(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  };
  up_l(C->d_off_up, off_up);
  up_l(C->d_off_down, off_down);
  // one block does the far field when it is small (work ~ far blocks + shifts), else level kernels
  C->fused = (double)np * M * M + (double)nn * M * m * (d == 2 ? m : 1) <=
             (getenv("FRACLAP_FUSED_WORK") ? atof(getenv("FRACLAP_FUSED_WORK")) : 8.0e6);
  if (C->fused) {
    int sms = 148, per = 0, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, d == 1 ? (const void*)far_fused_kernel<1>
                                                               : (const void*)far_fused_kernel<2>, 256, 0);
    C->coop_blocks = sms * std::min(per, getenv("FRACLAP_COOP_PER_SM") ? atoi(getenv("FRACLAP_COOP_PER_SM")) : 1);
    C->fused = coop && C->coop_blocks > 0 && covered == n && (int64_t)sub_leaves.size() == (int64_t)leaf_nodes.size();
  }
  C->mom.alloc((size_t)nn * M);
  C->F.alloc((size_t)nn * M);
  C->Fp.alloc(std::max<int64_t>(np * 2 * M, 1));
  C->x.alloc(std::max<int64_t>(n, 1));
  C->y.alloc(std::max<int64_t>(n, 1));
  C->yfar.alloc(std::max<int64_t>(n, 1));
  FL_CUDA(cudaStreamSynchronize(st));
  *out = C.release();
  return FL_OK;
}

void far_potentials(fl_cluster* C, const double* x, cudaStream_t st);

int32_t cluster_matvec_dev(fl_cluster* C, const double* x, double* y, double* yfar, cudaStream_t st) {
  const int64_t n = C->n, nn = C->nn, np = C->np;
  const int M = C->M, m = C->m;
  if (n == 0) return FL_OK;
  if (C->fused) {                                      // the near product runs inside the fused kernel
    double negC = -C->C;
    int64_t nn_ = nn, np_ = np, n_ = n;
    int m_ = m, M_ = M;
    void* args[] = {&C->nsub, &C->sub_info.p, &C->grp_off.p, &C->grp_nodes.p, &C->sub_leaves.p, &C->top_g0,
                    &C->top_g1, &C->leaf_nodes.p, &C->leaf_lo.p, &C->leaf_hi.p, &C->dof_perm.p, &x, &C->bc.p, &m_,
                    &M_, &nn_, &C->children.p, &C->shift.p, &np_, &C->pairs.p, &C->blocks.p, &C->plist_off.p,
                    &C->plist.p, &C->mom.p, &C->Fp.p, &C->F.p, &C->leaf_of_dof.p, &negC, &y, &yfar, &n_, &C->indptr.p,
                    &C->indices.p, &C->data.p, &C->n_early, &C->early.p, &C->n_late, &C->late.p};
    const void* fn = C->d == 1 ? (const void*)far_fused_kernel<1> : (const void*)far_fused_kernel<2>;
    FL_CUDA(cudaLaunchCooperativeKernel(fn, dim3(C->coop_blocks), dim3(256), args, 0, st));
    note_launch();
    FL_CHECK_LAUNCH();
    return FL_OK;
  }
  csr_spmv_kernel<<<grid_of(n * 32), 256, 0, st>>>(n, C->indptr.p, C->indices.p, C->data.p, x, y), note_launch();
  far_potentials(C, x, st);
  eval_kernel<<<grid_of(n), 256, 0, st>>>(n, C->leaf_of_dof.p, C->bc.p, M, C->F.p, -C->C, y, yfar), note_launch();
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// F = the far potentials of x at every tree node (moments, upward pass, far pairs, downward pass)
void far_potentials(fl_cluster* C, const double* x, cudaStream_t st) {
  const int64_t nn = C->nn, np = C->np;
  const int M = C->M, m = C->m;
  FL_CUDA(cudaMemsetAsync(C->mom.p, 0, (size_t)nn * M * sizeof(double), st));
  moments_kernel<<<grid_of((int64_t)C->nleaves * M), 256, 0, st>>>(C->nleaves, C->leaf_nodes.p, C->leaf_lo.p,
                                                                   C->leaf_hi.p, C->dof_perm.p, x, C->bc.p, M,
                                                                   C->mom.p), note_launch();
  for (size_t L = 0; L + 1 < C->level_off_up.size(); ++L) {
    const int64_t a = C->level_off_up[L], cnt = C->level_off_up[L + 1] - a;
    if (cnt <= 0) continue;
    if (C->d == 1)
      up_kernel<1><<<grid_of(cnt * M), 256, 0, st>>>(C->level_nodes.p + a, (int)cnt, C->children.p, C->shift.p, m, M,
                                                     C->mom.p);
    else
      up_kernel<2><<<grid_of(cnt * M), 256, 0, st>>>(C->level_nodes.p + a, (int)cnt, C->children.p, C->shift.p, m, M,
                                                     C->mom.p);
    note_launch();
  }
  if (np > 0)
    far_pair_kernel<<<grid_of(np * 2 * M), 256, 0, st>>>(np, C->pairs.p, C->blocks.p, M, C->mom.p, C->Fp.p),
        note_launch();
  far_gather_kernel<<<grid_of(nn * M), 256, 0, st>>>(nn, C->plist_off.p, C->plist.p, M, C->Fp.p, C->F.p),
      note_launch();
  for (size_t L = 0; L + 1 < C->level_off_down.size(); ++L) {
    const int64_t a = C->level_off_down[L], cnt = C->level_off_down[L + 1] - a;
    if (cnt <= 0) continue;
    if (C->d == 1)
      down_kernel<1><<<grid_of(cnt * M), 256, 0, st>>>(C->level_nodes.p + a, (int)cnt, C->parent.p, C->shift.p, m, M,
                                                       C->F.p);
    else
      down_kernel<2><<<grid_of(cnt * M), 256, 0, st>>>(C->level_nodes.p + a, (int)cnt, C->parent.p, C->shift.p, m, M,
                                                       C->F.p);
    note_launch();
  }
  FL_CHECK_LAUNCH();
}

}  // namespace fl

// ------------------------------------------------------------------ strong form (adapt.py:81-214)
namespace fl {
namespace {

// Lagrange basis at the Chebyshev nodes `ref` (lagrange_eval, cluster.py:276-287): products in order
__device__ __forceinline__ double lagrange1(const double* __restrict__ ref, int m, double t, int a) {
  double num = 1.0, den = 1.0;
  for (int b = 0; b < m; ++b) {
    if (b == a) continue;
    num *= t - ref[b];
    den *= ref[a] - ref[b];
  }
  return num / den;
}

// -C * L(x) . F[owner]   (evaluate_far_field_at_points, cluster.py:469-485; eval_basis :327-337)
template <int D>
__global__ void far_points_kernel(int64_t npts, int q, const double* __restrict__ X,
                                  const int64_t* __restrict__ cell_leaf, const double* __restrict__ center,
                                  const double* __restrict__ half, const double* __restrict__ ref, int m, int M,
                                  const double* __restrict__ F, double negC, double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int64_t nd = cell_leaf[p / q];             // the owning leaf of the point's cell
  double l0[16], l1[16];
  const double t0 = (X[p * D] - center[nd * D]) / half[nd];
  for (int a = 0; a < m; ++a) l0[a] = lagrange1(ref, m, t0, a);
  if (D == 2) {
    const double t1 = (X[p * D + 1] - center[nd * D + 1]) / half[nd];
    for (int a = 0; a < m; ++a) l1[a] = lagrange1(ref, m, t1, a);
  }
  const double* f = F + nd * M;
  double s = 0.0;
  for (int a = 0; a < M; ++a) s = fma(D == 1 ? l0[a] : l0[a / m] * l1[a % m], f[a], s);
  out[p] = negC * s;
}

struct CellSurf {                     // one cell's vertices, hat values and gradient
  double P[3][2], v[3], g[2];
};
// grad u_K from the vertex values: 1D (v1 - v0) / (P1 - P0); 2D the reference's
// inv(E^T) [v1 - v0, v2 - v0] with E rows the edge vectors (_cell_gradients_fixed, adapt.py:45-54)
template <int D>
__device__ __forceinline__ void cell_grad(CellSurf& c) {
  if (D == 1) {
    c.g[0] = (c.v[1] - c.v[0]) / (c.P[1][0] - c.P[0][0]);
  } else {
    const double e1x = c.P[1][0] - c.P[0][0], e1y = c.P[1][1] - c.P[0][1];
    const double e2x = c.P[2][0] - c.P[0][0], e2y = c.P[2][1] - c.P[0][1];
    const double r0 = c.v[1] - c.v[0], r1 = c.v[2] - c.v[0];
    const double det = e1x * e2y - e2x * e1y;           // E^T = [[e1x, e2x], [e1y, e2y]]
    c.g[0] = (e2y * r0 - e2x * r1) / det;
    c.g[1] = (e1x * r1 - e1y * r0) / det;
  }
}

struct SurfConsts {
  double s, ex_flux, p_grad, cgrad_near, cgrad_own;   // gradient-term divisors of the near / own formulas
  int log_case, ngl;
  const double* glx;
  const double* glw;
};

// Powers of the strong form, specialised for s in {1/4, 1/2, 3/4} (SQ = 4s; 0: general pow) with
// the assembly's seed-corrected kernel powers: gradient term r^(2-d-2s) (1D: of r = |x - y|;
// 2D: r2^(-s)), flux term |x-y|^(-d-2s) (1D: of r; 2D: r2^(-(1+s))).
template <int D, int SQ>
__device__ __forceinline__ double sf_grad(double rr, double p_grad) {
  if constexpr (SQ == 0) {
    return D == 1 ? pow(rr, p_grad) : pow(rr, 0.5 * p_grad);
  } else if constexpr (D == 1) {
    if constexpr (SQ == 1) return rr * rpow_half<1>(rr);        // r^(1/2)
    else return rpow_half<1>(rr);                               // s = 3/4: r^(-1/2) (s = 1/2: log case)
  } else {
    if constexpr (SQ == 2) return rpow_half<1>(rr);             // r2^(-1/2)
    else return rpow_quarter<SQ>(rr);                           // r2^(-1/4), r2^(-3/4)
  }
}
template <int D, int SQ>
__device__ __forceinline__ double sf_flux(double rr, double s) {
  if constexpr (SQ == 0) {
    return D == 1 ? pow(rr, -1.0 - 2.0 * s) : pow(rr, -(1.0 + s));
  } else if constexpr (D == 1) {
    return rpow_half<2 + SQ>(rr);          // r^(-(1 + 2s)) = r^(-(2 + SQ) / 2)
  } else {
    return kpow<8 + 2 * SQ>(rr, 0.0);      // r2^(-(1 + s)) = r2^(-(8 + 2 SQ) / 8)
  }
}

// surface terms of cell c at point x: returns (gradient term, flux term) sums over the cell's edges
// (1D: its two end points), the flux term WITHOUT the u factor when `flux_only` (own cell)
template <int D, int SQ>
__device__ void surf_terms(const CellSurf& c, double x0, double x1, const SurfConsts& K, bool own, double& tg,
                           double& tf) {
  tg = 0.0;
  tf = 0.0;
  if (D == 1) {
    const double sg = c.P[1][0] - c.P[0][0] > 0.0 ? 1.0 : (c.P[1][0] - c.P[0][0] < 0.0 ? -1.0 : 0.0);
    for (int e = 0; e < 2; ++e) {
      const double pn = e == 0 ? -sg : sg;
      const double diff = x0 - c.P[e][0], r = fabs(diff);
      const double gp = c.g[0] * pn;
      tg += K.log_case ? gp * log(1.0 / r) : gp * sf_grad<D, SQ>(r, K.p_grad);
      const double fl = pn * diff * sf_flux<D, SQ>(r, K.s);
      tf += own ? fl : c.v[e] * fl;
    }
  } else {
    const double cx = (c.P[0][0] + c.P[1][0] + c.P[2][0]) / 3.0, cy = (c.P[0][1] + c.P[1][1] + c.P[2][1]) / 3.0;
    for (int e = 0; e < 3; ++e) {
      const int a = e, b = (e + 1) % 3;
      const double tx = c.P[b][0] - c.P[a][0], ty = c.P[b][1] - c.P[a][1];
      const double EL = sqrt(tx * tx + ty * ty);
      double nx = ty / EL, ny = -tx / EL;
      const double mx = 0.5 * (c.P[a][0] + c.P[b][0]) - cx, my = 0.5 * (c.P[a][1] + c.P[b][1]) - cy;
      if (mx * nx + my * ny < 0.0) { nx = -nx; ny = -ny; }
      const double gn = c.g[0] * nx + c.g[1] * ny;
      double sg = 0.0, sf = 0.0;
      for (int qq = 0; qq < K.ngl; ++qq) {
        const double t = K.glx[qq], w = K.glw[qq];
        const double yx = c.P[a][0] + t * tx, yy = c.P[a][1] + t * ty;
        const double dx = x0 - yx, dy = x1 - yy;
        const double r2 = dx * dx + dy * dy;
        sg += w * (K.log_case ? -0.5 * log(r2) : sf_grad<D, SQ>(r2, K.p_grad));
        const double uY = own ? 1.0 : c.v[a] * (1.0 - t) + c.v[b] * t;
        sf += w * uY * (dx * nx + dy * ny) * sf_flux<D, SQ>(r2, K.s);
      }
      tg += gn * sg * EL;
      tf += sf * EL;
    }
  }
}

// warp per point: near cells of the owning leaf (lanes; u restricted to the near DoFs, the point's
// own cell excluded) + the own cell with the full u; out = far + C * contrib
template <int D, int SQ>
__global__ void __launch_bounds__(256) strong_near_kernel(
    DevMesh m, int64_t npts, int q, const double* __restrict__ X, const int64_t* __restrict__ cell_leaf,
    const int64_t* __restrict__ near_off, const int64_t* __restrict__ near_val, const int64_t* __restrict__ ncell_off,
    const int64_t* __restrict__ ncell_val, const int* __restrict__ leaf_of_dof, const double* __restrict__ u,
    SurfConsts K, double Cds, const double* __restrict__ far, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= npts) return;
  const int c = (int)(p / q);
  const int64_t leaf = cell_leaf[c];
  const double x0 = X[p * D], x1 = D == 2 ? X[p * D + 1] : 0.0;
  const int64_t nl0 = near_off[leaf], nl1 = near_off[leaf + 1];
  double acc = 0.0;
  for (int64_t k = ncell_off[leaf] + lane; k < ncell_off[leaf + 1]; k += 32) {
    const int Kc = (int)ncell_val[k];
    if (Kc == c) continue;
    CellSurf cs;
    for (int j = 0; j <= D; ++j) {
      const int v = m.cells[Kc * (D + 1) + j];
      cs.P[j][0] = m.vert[v * D];
      cs.P[j][1] = D == 2 ? m.vert[v * D + 1] : 0.0;
      const int dof = m.v2d[v];
      double val = 0.0;
      if (dof >= 0) {                            // u restricted to the DoFs of the near leaves
        const int64_t lf = leaf_of_dof[dof];
        int64_t a = nl0, b = nl1;
        while (a < b) {
          const int64_t mid = (a + b) >> 1;
          if (near_val[mid] < lf) a = mid + 1; else b = mid;
        }
        if (a < nl1 && near_val[a] == lf) val = u[dof];
      }
      cs.v[j] = val;
    }
    cell_grad<D>(cs);
    double tg, tf;
    surf_terms<D, SQ>(cs, x0, x1, K, false, tg, tf);
    acc += tg / K.cgrad_near - tf / (2.0 * K.s);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    CellSurf cs;
    for (int j = 0; j <= D; ++j) {
      const int v = m.cells[c * (D + 1) + j];
      cs.P[j][0] = m.vert[v * D];
      cs.P[j][1] = D == 2 ? m.vert[v * D + 1] : 0.0;
      const int dof = m.v2d[v];
      cs.v[j] = dof >= 0 ? u[dof] : 0.0;
    }
    cell_grad<D>(cs);
    double tg, tf;
    surf_terms<D, SQ>(cs, x0, x1, K, true, tg, tf);
    double ux;                                   // the affine u_c at x (_affine_on_cells, adapt.py:217-233)
    if (D == 1) {
      const double t = (x0 - cs.P[0][0]) / (cs.P[1][0] - cs.P[0][0]);
      ux = cs.v[0] * (1.0 - t) + cs.v[1] * t;
    } else {
      const double e1x = cs.P[1][0] - cs.P[0][0], e1y = cs.P[1][1] - cs.P[0][1];
      const double e2x = cs.P[2][0] - cs.P[0][0], e2y = cs.P[2][1] - cs.P[0][1];
      const double rx = x0 - cs.P[0][0], ry = x1 - cs.P[0][1];
      const double det = e1x * e2y - e2x * e1y;
      const double a1 = (rx * e2y - ry * e2x) / det, a2 = (e1x * ry - e1y * rx) / det;
      ux = cs.v[0] * (1.0 - a1 - a2) + cs.v[1] * a1 + cs.v[2] * a2;
    }
    acc += tg / K.cgrad_own - ux * tf / (2.0 * K.s);
    out[p] = far[p] + Cds * acc;
  }
}

}  // namespace

// -C * L(x) . F[owner(x)] at arbitrary points (owner = the leaf node per point)
void cluster_far_points(fl_cluster* C, const double* u_dev, int64_t npts, const double* X_dev,
                        const int64_t* owner_dev, double* out_dev, cudaStream_t st) {
  far_potentials(C, u_dev, st);
  if (C->d == 1)
    far_points_kernel<1><<<grid_of(npts), 256, 0, st>>>(npts, 1, X_dev, owner_dev, C->center.p, C->half.p, C->ref.p,
                                                        C->m, C->M, C->F.p, -C->C, out_dev);
  else
    far_points_kernel<2><<<grid_of(npts), 256, 0, st>>>(npts, 1, X_dev, owner_dev, C->center.p, C->half.p, C->ref.p,
                                                        C->m, C->M, C->F.p, -C->C, out_dev);
  note_launch();
  FL_CHECK_LAUNCH();
}

int32_t cluster_strong_form(fl_cluster* C, const DevMesh& m, double s, const double* u_dev, int64_t q,
                            const double* X_dev, const int64_t* cell_leaf, const int64_t* near_off,
                            const int64_t* near_val, const int64_t* ncell_off, const int64_t* ncell_val,
                            const double* glx, const double* glw, int ngl, double* out_dev, double* far_dev,
                            cudaStream_t st) {
  const int d = m.d;
  const int64_t npts = (int64_t)m.nc * q;
  if (!C->center.p || !C->ref.p) throw Error(FL_E_ARG, "cluster: strong form needs the node boxes (center, half, ref)");
  if (C->m > 16) throw Error(FL_E_ARG, "cluster: Chebyshev order above 16");
  far_potentials(C, u_dev, st);
  if (d == 1)
    far_points_kernel<1><<<grid_of(npts), 256, 0, st>>>(npts, (int)q, X_dev, cell_leaf, C->center.p, C->half.p, C->ref.p,
                                                        C->m, C->M, C->F.p, -C->C, far_dev);
  else
    far_points_kernel<2><<<grid_of(npts), 256, 0, st>>>(npts, (int)q, X_dev, cell_leaf, C->center.p, C->half.p, C->ref.p,
                                                        C->m, C->M, C->F.p, -C->C, far_dev);
  note_launch();
  SurfConsts K;
  K.s = s;
  K.ex_flux = -(d / 2.0 + s);
  K.p_grad = 2.0 - d - 2.0 * s;
  K.log_case = std::fabs(s - (1.0 - d / 2.0)) < 1e-12;      // LOG_CASE_TOL (adapt.py:25)
  K.cgrad_near = K.log_case ? 2.0 * s : 2.0 * s * (d + 2.0 * s - 2.0);
  K.cgrad_own = K.log_case ? 1.0 : (d + 2.0 * s - 2.0);
  K.ngl = ngl;
  K.glx = glx;
  K.glw = glw;
  const int sq = (s == 0.25 || s == 0.5 || s == 0.75) ? (int)std::lround(4.0 * s) : 0;
#define FL_SF_LAUNCH(DD, SS)                                                                                   \
  strong_near_kernel<DD, SS><<<grid_of(npts * 32), 256, 0, st>>>(m, npts, (int)q, X_dev, cell_leaf, near_off,   \
                                                                 near_val, ncell_off, ncell_val,              \
                                                                 C->leaf_of_dof.p, u_dev, K, C->C, far_dev,   \
                                                                 out_dev)
  if (d == 1) {
    if (sq == 1) FL_SF_LAUNCH(1, 1);
    else if (sq == 3) FL_SF_LAUNCH(1, 3);
    else FL_SF_LAUNCH(1, 0);                  // s = 1/2 is the log case in 1D
  } else {
    if (sq == 1) FL_SF_LAUNCH(2, 1);
    else if (sq == 2) FL_SF_LAUNCH(2, 2);
    else if (sq == 3) FL_SF_LAUNCH(2, 3);
    else FL_SF_LAUNCH(2, 0);
  }
#undef FL_SF_LAUNCH
  note_launch();
  FL_CHECK_LAUNCH();
  return FL_OK;
}

}  // namespace fl

// ------------------------------------------------------------------ C ABI

// near part of the dual-tree boundary flux (boundary_flux_at_nodes, cluster.py:586-592): every
// point of a DoF leaf sums edge_flux_potential (assembly.py:303-333) over the edges of that leaf's
// near edge-tree nodes, in the order given.  One thread per point; points are grouped by leaf so
// a warp walks one edge list.
__global__ void __launch_bounds__(128) near_edge_flux_kernel(int64_t npts, const double* __restrict__ X,
                                                             int64_t ngroups, const int64_t* __restrict__ poff,
                                                             const int64_t* __restrict__ eoff,
                                                             const int* __restrict__ eid,
                                                             const double* __restrict__ seg,
                                                             const double* __restrict__ glx,
                                                             const double* __restrict__ glw, int ngl, double ex,
                                                             double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  int64_t a = 0, b = ngroups;                       // group g: poff[g] <= p < poff[g + 1]
  while (b - a > 1) {
    const int64_t mid = (a + b) >> 1;
    if (poff[mid] <= p) a = mid; else b = mid;
  }
  const double x0 = X[2 * p], x1 = X[2 * p + 1];
  double acc = 0.0;
  for (int64_t k = eoff[a]; k < eoff[a + 1]; ++k) {
    const double* e = seg + (size_t)7 * eid[k];     // p0x p0y ux uy nx ny |e|
    double s = 0.0;
    for (int g = 0; g < ngl; ++g) {
      const double dx = x0 - (e[0] + glx[g] * e[2]), dy = x1 - (e[1] + glx[g] * e[3]);
      s = fma(glw[g], fma(dy, e[5], dx * e[4]) * pow(fma(dy, dy, dx * dx), ex), s);
    }
    acc = fma(s, e[6], acc);
  }
  out[p] = acc;
}

#define FL_TRY try {
#define FL_CATCH                                                                   \
  }                                                                                \
  catch (const fl::Error& e) { return fl::api_fail(e.code, e.what()); }            \
  catch (const std::bad_alloc&) { return fl::api_fail(FL_E_OOM, "host allocation failed"); } \
  catch (const std::exception& e) { return fl::api_fail(FL_E_CUDA, e.what()); }

extern "C" {

int32_t fl_cluster_create(const fl_cluster_desc* desc, int32_t device, fl_cluster** out) {
  FL_TRY
  if (!desc || !out) return fl::api_fail(FL_E_ARG, "null argument");
  *out = nullptr;
  if (!desc->parent || !desc->topo_order || !desc->ranges || !desc->dof_perm || !desc->shift || !desc->basis_coef ||
      (desc->npairs > 0 && !desc->far_pairs))
    return fl::api_fail(FL_E_ARG, "cluster: null array");
  return fl::cluster_create(desc, device, out);
  FL_CATCH
}

int32_t fl_cluster_matvec(fl_cluster* C, const double* x, double* y, double* y_far, int32_t ptr_kind) {
  FL_TRY
  if (!C || !x || !y) return fl::api_fail(FL_E_ARG, "null argument");
  fl::DeviceScope dev(C->device);
  cudaStream_t st = C->stream;
  fl::StreamScope scope(st);
  const int64_t n = C->n;
  if (ptr_kind == 1) {
    fl::cluster_matvec_dev(C, x, y, y_far ? y_far : C->yfar.p, st);
    FL_CUDA(cudaStreamSynchronize(st));
    return FL_OK;
  }
  FL_CUDA(cudaMemcpyAsync(C->x.p, x, n * sizeof(double), cudaMemcpyHostToDevice, st));
  fl::cluster_matvec_dev(C, C->x.p, C->y.p, C->yfar.p, st);
  FL_CUDA(cudaMemcpyAsync(y, C->y.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (y_far) FL_CUDA(cudaMemcpyAsync(y_far, C->yfar.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
  FL_CATCH
}

int32_t fl_cluster_matvec_async(fl_cluster* C, const double* x, double* y, void* stream) {
  FL_TRY
  if (!C || !x || !y) return fl::api_fail(FL_E_ARG, "null argument");
  fl::DeviceScope dev(C->device);
  cudaStream_t st = (cudaStream_t)stream;             // NULL: the legacy default stream
  fl::StreamScope scope(st);
  // The operator's scratch (mom, F, Fp, yfar) is shared with the synchronous entry points and
  // released on C->stream: order this matvec after everything pending on C->stream, and
  // everything later on C->stream after this matvec.
  if (st != C->stream) {
    cudaEvent_t e0, e1;
    FL_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    FL_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    FL_CUDA(cudaEventRecord(e0, C->stream));
    FL_CUDA(cudaStreamWaitEvent(st, e0, 0));
    fl::cluster_matvec_dev(C, x, y, C->yfar.p, st);
    FL_CUDA(cudaEventRecord(e1, st));
    FL_CUDA(cudaStreamWaitEvent(C->stream, e1, 0));
    cudaEventDestroy(e0);   // (destruction is deferred by the runtime until the events complete)
    cudaEventDestroy(e1);
  } else {
    fl::cluster_matvec_dev(C, x, y, C->yfar.p, st);
  }
  return FL_OK;
  FL_CATCH
}

int32_t fl_cluster_strong_form(fl_cluster* C, const fl_mesh* mesh, const fl_dofmap* dofmap, double s,
                               const double* u, int64_t q, const double* X, const int64_t* cell_leaf,
                               const int64_t* near_off, const int64_t* near_val, const int64_t* ncell_off,
                               const int64_t* ncell_val, const double* gl_x, const double* gl_w, int64_t ngl,
                               double* out, double* far_out) {
  FL_TRY
  if (!C || !mesh || !dofmap || !u || !X || !cell_leaf || !near_off || !near_val || !ncell_off || !ncell_val ||
      !gl_x || !gl_w || !out)
    return fl::api_fail(FL_E_ARG, "null argument");
  if (!(s > 0.0 && s < 1.0)) return fl::api_fail(FL_E_ARG, "s must lie in (0,1)");
  const int d = mesh->d;
  if (d != C->d || dofmap->n != C->n || q <= 0 || ngl <= 0 || ngl > 64) return fl::api_fail(FL_E_ARG, "bad sizes");
  const int64_t nv = mesh->nv, nc = mesh->nc, nn = C->nn;
  for (int64_t c = 0; c < nc; ++c)
    if (cell_leaf[c] < 0 || cell_leaf[c] >= nn) return fl::api_fail(FL_E_ARG, "cell leaf out of range");
  if (near_off[0] != 0 || ncell_off[0] != 0) return fl::api_fail(FL_E_ARG, "near lists must start at 0");
  for (int64_t k = 0; k < nn; ++k)
    if (near_off[k + 1] < near_off[k] || ncell_off[k + 1] < ncell_off[k])
      return fl::api_fail(FL_E_ARG, "near list offsets must be non-decreasing");
  for (int64_t e = 0; e < near_off[nn]; ++e)
    if (near_val[e] < 0 || near_val[e] >= nn || (e > 0 && near_val[e] < near_val[e - 1] &&
                                                 !std::binary_search(near_off, near_off + nn + 1, e)))
      return fl::api_fail(FL_E_ARG, "near leaves must be node ids, ascending per node");
  for (int64_t e = 0; e < ncell_off[nn]; ++e)
    if (ncell_val[e] < 0 || ncell_val[e] >= nc) return fl::api_fail(FL_E_ARG, "near cell out of range");
  FL_CUDA(cudaSetDevice(C->device));
  cudaStream_t st = C->stream;
  fl::StreamScope scope(st);
  std::vector<int> cells((size_t)nc * (d + 1)), v2d((size_t)nv);
  for (int64_t i = 0; i < nc * (d + 1); ++i) {
    if (mesh->cells[i] < 0 || mesh->cells[i] >= nv) return fl::api_fail(FL_E_ARG, "cell vertex index out of range");
    cells[i] = (int)mesh->cells[i];
  }
  for (int64_t v = 0; v < nv; ++v) v2d[v] = (int)dofmap->vertex_to_dof[v];
  fl::DBuf<double> dvert((size_t)nv * d), du((size_t)std::max<int64_t>(C->n, 1)), dX((size_t)nc * q * d),
      dglx(ngl), dglw(ngl), dout((size_t)nc * q), dfar((size_t)nc * q);
  fl::DBuf<int> dcells(cells.size()), dv2d(v2d.size());
  fl::DBuf<int64_t> dleaf(nc), dnoff(nn + 1), dnval, dcoff(nn + 1), dcval;
  const int64_t nnv = near_off[nn], ncv = ncell_off[nn];
  dnval.alloc(std::max<int64_t>(nnv, 1));
  dcval.alloc(std::max<int64_t>(ncv, 1));
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) FL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  };
  h2d(dvert.p, mesh->vertices, (size_t)nv * d * 8);
  h2d(du.p, u, (size_t)C->n * 8);
  h2d(dX.p, X, (size_t)nc * q * d * 8);
  h2d(dglx.p, gl_x, (size_t)ngl * 8);
  h2d(dglw.p, gl_w, (size_t)ngl * 8);
  h2d(dcells.p, cells.data(), cells.size() * 4);
  h2d(dv2d.p, v2d.data(), v2d.size() * 4);
  h2d(dleaf.p, cell_leaf, (size_t)nc * 8);
  h2d(dnoff.p, near_off, (size_t)(nn + 1) * 8);
  h2d(dnval.p, near_val, (size_t)nnv * 8);
  h2d(dcoff.p, ncell_off, (size_t)(nn + 1) * 8);
  h2d(dcval.p, ncell_val, (size_t)ncv * 8);
  fl::DevMesh m;
  m.d = d; m.nv = (int)nv; m.nc = (int)nc; m.n = (int)C->n;
  m.vert = dvert.p; m.cells = dcells.p; m.v2d = dv2d.p;
  fl::cluster_strong_form(C, m, s, du.p, q, dX.p, dleaf.p, dnoff.p, dnval.p, dcoff.p, dcval.p, dglx.p, dglw.p,
                          (int)ngl, dout.p, dfar.p, st);
  FL_CUDA(cudaMemcpyAsync(out, dout.p, (size_t)nc * q * 8, cudaMemcpyDeviceToHost, st));
  if (far_out) FL_CUDA(cudaMemcpyAsync(far_out, dfar.p, (size_t)nc * q * 8, cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
  FL_CATCH
}

int32_t fl_cluster_far_at_points(fl_cluster* C, const double* u, int64_t npts, const double* points,
                                 const int64_t* owner, double* out) {
  FL_TRY
  if (!C || !u || (npts > 0 && (!points || !owner || !out))) return fl::api_fail(FL_E_ARG, "null argument");
  if (!C->center.p || !C->ref.p) return fl::api_fail(FL_E_ARG, "cluster: the operator has no node boxes");
  if (C->m > 16) return fl::api_fail(FL_E_ARG, "cluster: Chebyshev order above 16");
  for (int64_t p = 0; p < npts; ++p)
    if (owner[p] < 0 || owner[p] >= C->nn) return fl::api_fail(FL_E_ARG, "owner node out of range");
  FL_CUDA(cudaSetDevice(C->device));
  cudaStream_t st = C->stream;
  fl::StreamScope scope(st);
  if (npts == 0) return FL_OK;
  fl::DBuf<double> du(std::max<int64_t>(C->n, 1)), dX((size_t)npts * C->d), dout(npts);
  fl::DBuf<int64_t> down(npts);
  if (C->n) FL_CUDA(cudaMemcpyAsync(du.p, u, C->n * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dX.p, points, (size_t)npts * C->d * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(down.p, owner, npts * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  fl::cluster_far_points(C, du.p, npts, dX.p, down.p, dout.p, st);
  FL_CUDA(cudaMemcpyAsync(out, dout.p, npts * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
  FL_CATCH
}

int32_t fl_cluster_far_blocks(const fl_cluster* C, double* blocks_out) {
  FL_TRY
  if (!C || !blocks_out) return fl::api_fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(C->device));
  if (C->np > 0)
    FL_CUDA(cudaMemcpyAsync(blocks_out, C->blocks.p, (size_t)C->np * C->M * C->M * sizeof(double),
                            cudaMemcpyDeviceToHost, C->stream));
  FL_CUDA(cudaStreamSynchronize(C->stream));
  return FL_OK;
  FL_CATCH
}

int32_t fl_boundary_flux_near(int32_t device, double s, int64_t npts, const double* X, int64_t ngroups,
                              const int64_t* poff, const int64_t* eoff, const int64_t* eid, int64_t nb,
                              const double* p0, const double* p1, const double* normals, const double* gl_x,
                              const double* gl_w, int64_t ngl, double* out) {
  FL_TRY
  if (npts < 0 || ngroups < 0 || nb < 0 || ngl <= 0 || ngl > 64 || !(s > 0.0 && s < 1.0))
    return fl::api_fail(FL_E_ARG, "bad argument");
  if (npts == 0) return FL_OK;
  if (!X || !poff || !eoff || !out || !gl_x || !gl_w || ngroups == 0)
    return fl::api_fail(FL_E_ARG, "null argument");
  if (poff[0] != 0 || poff[ngroups] != npts || eoff[0] != 0) return fl::api_fail(FL_E_ARG, "bad group offsets");
  for (int64_t g = 0; g < ngroups; ++g)
    if (poff[g + 1] < poff[g] || eoff[g + 1] < eoff[g]) return fl::api_fail(FL_E_ARG, "bad group offsets");
  const int64_t ne = eoff[ngroups];
  if (ne > 0 && (!eid || !p0 || !p1 || !normals)) return fl::api_fail(FL_E_ARG, "null argument");
  std::vector<int> ei((size_t)std::max<int64_t>(ne, 1));
  for (int64_t k = 0; k < ne; ++k) {
    if (eid[k] < 0 || eid[k] >= nb) return fl::api_fail(FL_E_ARG, "edge index out of range");
    ei[k] = (int)eid[k];
  }
  std::vector<double> seg((size_t)std::max<int64_t>(7 * nb, 1));
  for (int64_t e = 0; e < nb; ++e) {
    const double ux = p1[2 * e] - p0[2 * e], uy = p1[2 * e + 1] - p0[2 * e + 1];
    double* r = &seg[7 * e];
    r[0] = p0[2 * e]; r[1] = p0[2 * e + 1]; r[2] = ux; r[3] = uy;
    r[4] = normals[2 * e]; r[5] = normals[2 * e + 1]; r[6] = std::sqrt(ux * ux + uy * uy);
  }
  FL_CUDA(cudaSetDevice(device));
  fl::OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  fl::StreamScope scope(st);
  fl::DBuf<double> dX((size_t)2 * npts), dseg(seg.size()), dgx(ngl), dgw(ngl), dout(npts);
  fl::DBuf<int64_t> dpo(ngroups + 1), deo(ngroups + 1);
  fl::DBuf<int> dei(ei.size());
  FL_CUDA(cudaMemcpyAsync(dX.p, X, (size_t)2 * npts * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dseg.p, seg.data(), seg.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dgx.p, gl_x, ngl * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dgw.p, gl_w, ngl * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dpo.p, poff, (ngroups + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(deo.p, eoff, (ngroups + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dei.p, ei.data(), ei.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  near_edge_flux_kernel<<<(unsigned)((npts + 127) / 128), 128, 0, st>>>(npts, dX.p, ngroups, dpo.p, deo.p, dei.p,
                                                                         dseg.p, dgx.p, dgw.p, (int)ngl,
                                                                         -(1.0 + s), dout.p);
  FL_CUDA(cudaGetLastError());
  FL_CUDA(cudaMemcpyAsync(out, dout.p, npts * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
  FL_CATCH
}

void fl_cluster_free(fl_cluster* C) {
  if (!C) return;
  cudaSetDevice(C->device);
  delete C;
}

}  // extern "C"
