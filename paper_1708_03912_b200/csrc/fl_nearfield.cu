// Near-field (cluster) assembly: assemble_near_field (assembly.py:860-970), the sparse matrix
// of the non-admissible DoF pairs that feeds the paper's quasi-linear cluster solver.
//
// It reuses the dense path's pair kernels (classification, singular rules, the one-block-per-
// pair disjoint kernel of fl_near.cu, the cell-local matrices and the row pull of fl_local.cu)
// and replaces two things:
//  * the tail Psi_K by the divergence identity Psi = (V - ring flux of dN(K)) / (2s)
//    (tail_potential / ring_boundaries, assembly.py:336-396): per cell, the boundary of its
//    one-ring patch is found on the device (edges of N(K) used once, outward from the patch's
//    vertex mean), and the GL8 flux of those edges and of the domain boundary is evaluated at
//    the cell nodes (edge_flux_potential, assembly.py:303-333);
//  * the dense rows by CSR rows whose pattern is every DoF pair of a near leaf pair (every such
//    entry receives a triplet in the reference, so the patterns agree), with the cross term
//    -C sum M^{K,L} of every disjoint cell pair behind the entry gathered in a fixed order from
//    the de-duplicated pair blocks (hash lookup) — deterministic, no atomics on values.
#include <cub/cub.cuh>

#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

namespace fl {
namespace {

constexpr int NK_MAX = 64;      // cells in one patch N(K)
constexpr int RING_MAX = 64;    // edges on dN(K)
constexpr unsigned long long NONE = ~0ull;

int grid_of(int64_t m, int b = 256) { return (int)std::max<int64_t>(1, (m + b - 1) / b); }

// ------------------------------------------------------------------ ring of N(K)
// Ring edges as (p0x, p0y, p1x, p1y, nx, ny); 1D: the two end points of N(K) with normals -1, +1.
template <int D>
__device__ int ring_of(const DevMesh& m, int K, double* out /* RING_MAX*6 or null */, int* err) {
  const CellGeo& g = m.geo[K];
  int nk = 0;
  int nbr[NK_MAX];
  for (int j = 0; j <= D; ++j) {
    const int v = g.v[j];
    for (int p = m.patch_off[v]; p < m.patch_off[v + 1]; ++p) {
      const int c = m.patch_cells[p];
      bool seen = false;
      for (int u = 0; u < nk; ++u) seen |= nbr[u] == c;
      if (!seen) {
        if (nk == NK_MAX) { atomicOr(err, 16); return 0; }
        nbr[nk++] = c;
      }
    }
  }
  if constexpr (D == 1) {
    double lo = 1e300, hi = -1e300;
    for (int u = 0; u < nk; ++u) {
      const CellGeo& c = m.geo[nbr[u]];
      lo = fmin(lo, fmin(c.p[0][0], c.p[1][0]));
      hi = fmax(hi, fmax(c.p[0][0], c.p[1][0]));
    }
    if (out) {
      out[0] = lo; out[1] = 0.0; out[2] = lo; out[3] = 0.0; out[4] = -1.0; out[5] = 0.0;
      out[6] = hi; out[7] = 0.0; out[8] = hi; out[9] = 0.0; out[10] = 1.0; out[11] = 0.0;
    }
    return 2;
  } else {
    // vertex mean of the unique vertices of N(K), in ascending vertex order (np.unique, then a
    // sequential axis-0 mean)
    int vs[3 * NK_MAX];
    int nvu = 0;
    for (int u = 0; u < nk; ++u)
      for (int j = 0; j < 3; ++j) {
        const int v = m.geo[nbr[u]].v[j];
        bool seen = false;
        for (int w = 0; w < nvu; ++w) seen |= vs[w] == v;
        if (!seen) vs[nvu++] = v;
      }
    for (int a = 1; a < nvu; ++a) {            // insertion sort (small)
      const int x = vs[a];
      int b = a - 1;
      while (b >= 0 && vs[b] > x) { vs[b + 1] = vs[b]; --b; }
      vs[b + 1] = x;
    }
    double cx = 0.0, cy = 0.0;
    for (int w = 0; w < nvu; ++w) {
      cx = __dadd_rn(cx, m.vert[2 * vs[w]]);
      cy = __dadd_rn(cy, m.vert[2 * vs[w] + 1]);
    }
    cx = __ddiv_rn(cx, (double)nvu);
    cy = __ddiv_rn(cy, (double)nvu);
    int nr = 0;
    for (int u = 0; u < nk; ++u) {
      const CellGeo& c = m.geo[nbr[u]];
      for (int j = 0; j < 3; ++j) {
        const int a0 = c.v[j], b0 = c.v[(j + 1) % 3];
        const int a = min(a0, b0), b = max(a0, b0);
        int cnt = 0;                         // how many cells of N(K) hold the edge
        for (int u2 = 0; u2 < nk; ++u2) {
          const CellGeo& c2 = m.geo[nbr[u2]];
          bool ha = false, hb = false;
          for (int j2 = 0; j2 < 3; ++j2) { ha |= c2.v[j2] == a; hb |= c2.v[j2] == b; }
          cnt += ha && hb;
        }
        if (cnt != 1) continue;
        if (nr == RING_MAX) { atomicOr(err, 16); return 0; }
        if (out) {
          const double pax = m.vert[2 * a], pay = m.vert[2 * a + 1], pbx = m.vert[2 * b], pby = m.vert[2 * b + 1];
          const double tx = __dsub_rn(pbx, pax), ty = __dsub_rn(pby, pay);
          double nx = ty, ny = -tx;
          const double nr2 = norm2d(nx, ny);
          nx = __ddiv_rn(nx, nr2);
          ny = __ddiv_rn(ny, nr2);
          const double mx = __dsub_rn(__dmul_rn(0.5, __dadd_rn(pax, pbx)), cx);
          const double my = __dsub_rn(__dmul_rn(0.5, __dadd_rn(pay, pby)), cy);
          if (__dadd_rn(__dmul_rn(mx, nx), __dmul_rn(my, ny)) < 0.0) { nx = -nx; ny = -ny; }
          double* o = out + 6 * nr;
          o[0] = pax; o[1] = pay; o[2] = pbx; o[3] = pby; o[4] = nx; o[5] = ny;
        }
        ++nr;
      }
    }
    return nr;
  }
}

template <int D>
__global__ void ring_count_kernel(DevMesh m, int* cnt) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K < m.nc) cnt[K] = ring_of<D>(m, K, nullptr, m.err);
}
template <int D>
__global__ void ring_fill_kernel(DevMesh m, const int* off, double* ring) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K < m.nc) ring_of<D>(m, K, ring + (size_t)6 * off[K], m.err);
}

// GL8 flux of one edge (p0, p1, outward n) at x: |e| sum_g w_g n.(x - y_g) |x - y_g|^(2 ex)
template <int D, int E4>
__device__ __forceinline__ double edge_flux(const double* tab, RuleRef gl, double ex, double x0, double x1,
                                            double p0x, double p0y, double p1x, double p1y, double nx, double ny) {
  if constexpr (D == 1) {
    const double diff = x0 - p0x;
    return diff * nx * kpow<E4>(diff * diff, ex);
  } else {
    const double ux = p1x - p0x, uy = p1y - p0y;
    const double L = norm2d(ux, uy);
    double s = 0.0;
    for (int gq = 0; gq < gl.cnt; ++gq) {
      const double* nd = tab + (size_t)(gl.off + gq) * NODE;
      const double dx = x0 - (p0x + nd[0] * ux), dy = x1 - (p0y + nd[0] * uy);
      s = fma(nd[1], fma(dy, ny, dx * nx) * kpow<E4>(fma(dy, dy, dx * dx), ex), s);
    }
    return s * L;
  }
}

// psi = (V - ring) / (2s)  (tail_potential, assembly.py:388-396);  win = T - V  (:1092): the
// inward flux of the boundary edges not touching K — summed directly when V is computed here
template <int D, int E4>
__global__ void __launch_bounds__(128) ring_tail_kernel(DevMesh m, const double* __restrict__ tab, RuleRef gl,
                                                        double ex, double two_s, const double* __restrict__ Vgiven,
                                                        int integral, const int* __restrict__ roff,
                                                        const double* __restrict__ ring, double* __restrict__ psi,
                                                        double* __restrict__ win) {
  const int Q = m.q;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nc * Q) return;
  const int K = i / Q;
  const CellGeo& A = m.geo[K];
  const double x0 = m.X[(size_t)i * D], x1 = D == 2 ? m.X[(size_t)i * D + 1] : 0.0;
  double V = 0.0, T = 0.0, N = 0.0;
  if (!Vgiven || integral) {
    for (int e = 0; e < m.nb; ++e) {
      const int v0 = m.bedges[e * D], v1 = D == 2 ? m.bedges[e * D + 1] : v0;
      bool t = false;
#pragma unroll
      for (int j = 0; j <= D; ++j) t |= (A.v[j] == v0) | (A.v[j] == v1);
      const double f = D == 1 ? edge_flux<D, E4>(tab, gl, ex, x0, x1, m.vert[v0], 0.0, 0.0, 0.0, m.bnorm[e], 0.0)
                              : edge_flux<D, E4>(tab, gl, ex, x0, x1, m.vert[2 * v0], m.vert[2 * v0 + 1],
                                                 m.vert[2 * v1], m.vert[2 * v1 + 1], m.bnorm[2 * e], m.bnorm[2 * e + 1]);
      V += f;
      if (t) T += f; else N += f;
    }
  }
  if (Vgiven) V = Vgiven[i];
  double R = 0.0;
  for (int r = roff[K]; r < roff[K + 1]; ++r) {
    const double* o = ring + (size_t)6 * r;
    R += edge_flux<D, E4>(tab, gl, ex, x0, x1, o[0], o[1], o[2], o[3], o[4], o[5]);
  }
  psi[i] = (V - R) / two_s;
  win[i] = integral ? (Vgiven ? T - V : -N) : 0.0;
}

// ------------------------------------------------------------------ structure
__global__ void seg_offsets_kernel(const unsigned long long* keys, int64_t m, int nseg, int64_t* off) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l > nseg) return;
  const unsigned long long t = (unsigned long long)l << 32;
  int64_t a = 0, b = m;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (keys[mid] < t) a = mid + 1; else b = mid;
  }
  off[l] = a;
}
__global__ void dofleaf_keys_kernel(const int* leaf_of_dof, int n, unsigned long long* key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = ((unsigned long long)leaf_of_dof[i] << 32) | (unsigned)i;
}
// cells supporting each leaf's DoFs (_leaf_cells, cluster.py:511-522): one key per patch entry
__global__ void leafcell_keys_kernel(DevMesh m, const int* leaf_of_dof, int64_t tot, unsigned long long* key) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  int a = 0, b = m.nv;                       // vertex of patch entry e: last v with patch_off[v] <= e
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (m.patch_off[mid] <= e) a = mid; else b = mid;
  }
  const int dof = m.v2d[a];
  key[e] = dof < 0 ? NONE : (((unsigned long long)leaf_of_dof[dof] << 32) | (unsigned)m.patch_cells[e]);
}
__global__ void pair_count_kernel(const int* pairs, int64_t np, const int64_t* lco, int64_t* cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int a = pairs[2 * p], b = pairs[2 * p + 1];
  cnt[p] = (lco[a + 1] - lco[a]) * (lco[b + 1] - lco[b]);
}
template <int D>
__global__ void cand_keys_kernel(DevMesh m, const int* pairs, int64_t np, const int64_t* lco,
                                 const unsigned long long* lcell, const int64_t* coff, int64_t tot,
                                 unsigned long long* key) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tot) return;
  int64_t lo = 0, hi = np;                   // pair p: coff[p] <= t < coff[p + 1]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (coff[mid] <= t) lo = mid; else hi = mid;
  }
  const int a = pairs[2 * lo], b = pairs[2 * lo + 1];
  const int64_t r = t - coff[lo], nb = lco[b + 1] - lco[b];
  const int K = (int)(lcell[lco[a] + r / nb] & 0xffffffffu), L = (int)(lcell[lco[b] + r % nb] & 0xffffffffu);
  if (K == L || touching<D>(m.geo[K], m.geo[L])) { key[t] = NONE; return; }
  key[t] = ((unsigned long long)min(K, L) << 32) | (unsigned)max(K, L);
}
// order of each unique pair in the reference orientation (pa = min, pb = max; _cross_triplets,
// assembly.py:702-706) with the exact fp64 select_order arithmetic; hash (P, Q) -> index
template <int D>
__global__ void near_orders_kernel(DevMesh m, OrderConsts oc, const unsigned long long* U, int64_t nu, int* P, int* Q,
                                   int* K, unsigned long long* hkey, int* hidx, unsigned long long hmask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  const unsigned long long key = U[i];
  const int p = (int)(key >> 32), q = (int)(key & 0xffffffffu);
  P[i] = p;
  Q[i] = q;
  const CellGeo& A = m.geo[p];
  const CellGeo& B = m.geo[q];
  K[i] = order_disjoint(oc, oc.coff, A, B, dist_estimate<D>(A, B));
  unsigned long long h = near_hash(key) & hmask;
  for (;;) {
    const unsigned long long prev = atomicCAS(&hkey[h], NEAR_EMPTY, key);
    if (prev == NEAR_EMPTY) { hidx[h] = (int)i; break; }
    h = (h + 1) & hmask;
  }
}
// directed leaf adjacency (a, b) and (b, a); its column keys (a, dof of b)
__global__ void adj_count_kernel(const int* pairs, int64_t np, const int64_t* ldo, int64_t* cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int a = pairs[2 * p], b = pairs[2 * p + 1];
  cnt[p] = (ldo[b + 1] - ldo[b]) + (a != b ? (ldo[a + 1] - ldo[a]) : 0);
}
__global__ void col_keys_kernel(const int* pairs, int64_t np, const int64_t* ldo, const unsigned long long* ldof,
                                const int64_t* coff, int64_t tot, unsigned long long* key) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tot) return;
  int64_t lo = 0, hi = np;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (coff[mid] <= t) lo = mid; else hi = mid;
  }
  const int a = pairs[2 * lo], b = pairs[2 * lo + 1];
  int64_t r = t - coff[lo];
  const int64_t nb = ldo[b + 1] - ldo[b];
  int row = a, col = b;
  if (r >= nb) { r -= nb; row = b; col = a; }
  const unsigned dof = (unsigned)(ldof[ldo[col] + r] & 0xffffffffu);
  key[t] = ((unsigned long long)row << 32) | dof;
}
__global__ void row_len_kernel(const int* leaf_of_dof, int n, const int64_t* lcol, int64_t* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] = lcol[leaf_of_dof[i] + 1] - lcol[leaf_of_dof[i]];
}

// cross values: warp per row; entry (i, j) = -C sum_{K in patch(i)} sum_{L in patch(j)} M^{K,L}_{ab}
// over disjoint pairs, ascending K then L (both patches ascending)
template <int D>
__global__ void __launch_bounds__(256) near_values_kernel(DevMesh m, const int* __restrict__ leaf_of_dof,
                                                          const int64_t* __restrict__ lcol,
                                                          const unsigned long long* __restrict__ ckeys,
                                                          const int* __restrict__ row_vertex,
                                                          const int64_t* __restrict__ indptr, int* __restrict__ indices,
                                                          double* __restrict__ data, const unsigned long long* hkey,
                                                          const int* hidx, unsigned long long hmask,
                                                          const double* __restrict__ G, double negC) {
  const int lane = threadIdx.x & 31;
  const int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= m.n) return;
  const int vi = row_vertex[i];
  const int64_t c0 = lcol[leaf_of_dof[i]], e0 = indptr[i], len = indptr[i + 1] - e0;
  for (int64_t t = lane; t < len; t += 32) {
    const int j = (int)(ckeys[c0 + t] & 0xffffffffu);
    indices[e0 + t] = j;
    const int vj = row_vertex[j];
    double acc = 0.0;
    for (int pk = m.patch_off[vi]; pk < m.patch_off[vi + 1]; ++pk) {
      const int K = m.patch_cells[pk];
      const CellGeo& gk = m.geo[K];
      int a = 0;
#pragma unroll
      for (int u = 0; u <= D; ++u) if (gk.v[u] == vi) a = u;
      for (int pl = m.patch_off[vj]; pl < m.patch_off[vj + 1]; ++pl) {
        const int L = m.patch_cells[pl];
        if (L == K) continue;
        const CellGeo& gl = m.geo[L];
        if (touching<D>(gk, gl)) continue;
        int b = 0;
#pragma unroll
        for (int u = 0; u <= D; ++u) if (gl.v[u] == vj) b = u;
        const unsigned long long key = ((unsigned long long)min(K, L) << 32) | (unsigned)max(K, L);
        unsigned long long h = near_hash(key) & hmask;
        int idx = -1;
        for (;;) {
          const unsigned long long hk = hkey[h];
          if (hk == key) { idx = hidx[h]; break; }
          if (hk == NEAR_EMPTY) break;
          h = (h + 1) & hmask;
        }
        if (idx < 0) { atomicOr(m.err, 4); continue; }
        acc += K < L ? G[(size_t)idx * 9 + a * 3 + b] : G[(size_t)idx * 9 + b * 3 + a];
      }
    }
    data[e0 + t] = negC * acc;
  }
}

template <class T>
void sort_keys(DBuf<T>& in, DBuf<T>& out, int64_t m, cudaStream_t st) {
  out.alloc(std::max<int64_t>(m, 1));
  if (m <= 0) return;
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, in.p, out.p, (int)m, 0, 64, st);
  DBuf<unsigned char> tb(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, tmp, in.p, out.p, (int)m, 0, 64, st));
}
int64_t excl_scan(const int64_t* in, int64_t* out, int64_t m, cudaStream_t st) {   // out has m + 1 entries
  FL_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
  if (m > 0) {
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, (int)m, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceScan::InclusiveSum(tb.p, tmp, in, out + 1, (int)m, st));
  }
  int64_t tot = 0;
  FL_CUDA(cudaMemcpyAsync(&tot, out + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return tot;
}

#define FL_E4_SWITCHF(e4, ...)                                \
  switch (e4) {                                               \
    case 6: { constexpr int E4 = 6; __VA_ARGS__; } break;     \
    case 8: { constexpr int E4 = 8; __VA_ARGS__; } break;     \
    case 10: { constexpr int E4 = 10; __VA_ARGS__; } break;   \
    case 12: { constexpr int E4 = 12; __VA_ARGS__; } break;   \
    case 14: { constexpr int E4 = 14; __VA_ARGS__; } break;   \
    default: { constexpr int E4 = 0; __VA_ARGS__; } break;    \
  }

}  // namespace

void launch_ring_tail(const DevMesh& m, const DevTables& t, double s, double ex, int e4, const double* Vgiven,
                      bool integral, double* psi, double* win, cudaStream_t st) {
  const int nc = m.nc;
  DBuf<int> cnt(nc);
  DBuf<int> off(nc + 1);
  if (m.d == 1) ring_count_kernel<1><<<grid_of(nc, 128), 128, 0, st>>>(m, cnt.p), note_launch();
  else ring_count_kernel<2><<<grid_of(nc, 128), 128, 0, st>>>(m, cnt.p), note_launch();
  FL_CUDA(cudaMemsetAsync(off.p, 0, sizeof(int), st));
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.p, off.p + 1, nc, st);
  DBuf<unsigned char> tb(tmp);
  FL_CUDA(cub::DeviceScan::InclusiveSum(tb.p, tmp, cnt.p, off.p + 1, nc, st));
  int nr = 0;
  FL_CUDA(cudaMemcpyAsync(&nr, off.p + nc, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  DBuf<double> ring((size_t)6 * std::max(nr, 1));
  if (m.d == 1) ring_fill_kernel<1><<<grid_of(nc, 128), 128, 0, st>>>(m, off.p, ring.p), note_launch();
  else ring_fill_kernel<2><<<grid_of(nc, 128), 128, 0, st>>>(m, off.p, ring.p), note_launch();
  const RuleRef gl = t.rule(T_EGL, 0);
  const int tot = nc * m.q;
  if (m.d == 1) {
    FL_E4_SWITCHF(e4, (ring_tail_kernel<1, E4><<<grid_of(tot, 128), 128, 0, st>>>(
                           m, t.data, gl, ex, 2.0 * s, Vgiven, integral ? 1 : 0, off.p, ring.p, psi, win),
                       note_launch()));
  } else {
    FL_E4_SWITCHF(e4, (ring_tail_kernel<2, E4><<<grid_of(tot, 128), 128, 0, st>>>(
                           m, t.data, gl, ex, 2.0 * s, Vgiven, integral ? 1 : 0, off.p, ring.p, psi, win),
                       note_launch()));
  }
  FL_CHECK_LAUNCH();
}

void near_field_cross(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                      const NearInput& in, const int* row_vertex, CsrOut& out, int64_t* npairs_out,
                      unsigned long long* evals, cudaStream_t st) {
  const int n = m.n, nl = in.nleaves;
  const int64_t np = in.npairs;
  // DoFs of every leaf (ascending), and the cells supporting them
  DBuf<unsigned long long> k0(std::max(n, 1)), ldof;
  dofleaf_keys_kernel<<<grid_of(n), 256, 0, st>>>(in.leaf_of_dof, n, k0.p), note_launch();
  sort_keys(k0, ldof, n, st);
  DBuf<int64_t> ldo(nl + 1), lco(nl + 1), lcol(nl + 1);
  seg_offsets_kernel<<<grid_of(nl + 1), 256, 0, st>>>(ldof.p, n, nl, ldo.p), note_launch();
  const int64_t npe = (int64_t)m.nc * (m.d + 1);
  DBuf<unsigned long long> k1(npe), k1s, lcell(npe);
  DBuf<int> nuniq(1);
  leafcell_keys_kernel<<<grid_of(npe), 256, 0, st>>>(m, in.leaf_of_dof, npe, k1.p), note_launch();
  sort_keys(k1, k1s, npe, st);
  {
    size_t tmp = 0;
    cub::DeviceSelect::Unique(nullptr, tmp, k1s.p, lcell.p, nuniq.p, (int)npe, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceSelect::Unique(tb.p, tmp, k1s.p, lcell.p, nuniq.p, (int)npe, st));
  }
  int nlc = 0;
  FL_CUDA(cudaMemcpyAsync(&nlc, nuniq.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  seg_offsets_kernel<<<grid_of(nl + 1), 256, 0, st>>>(lcell.p, nlc, nl, lco.p), note_launch();
  // candidate cell pairs of the near leaf pairs -> unique disjoint (min, max) pairs
  DBuf<int64_t> pc(std::max<int64_t>(np, 1)), poff(np + 1);
  pair_count_kernel<<<grid_of(np), 256, 0, st>>>(in.pairs, np, lco.p, pc.p), note_launch();
  const int64_t ncand = excl_scan(pc.p, poff.p, np, st);
  if (ncand >= (1LL << 31)) throw Error(FL_E_ASSEMBLY, "near field too large (candidate pairs >= 2^31)");
  DBuf<unsigned long long> ck(std::max<int64_t>(ncand, 1)), cks, U(std::max<int64_t>(ncand, 1));
  if (m.d == 1)
    cand_keys_kernel<1><<<grid_of(ncand), 256, 0, st>>>(m, in.pairs, np, lco.p, lcell.p, poff.p, ncand, ck.p), note_launch();
  else
    cand_keys_kernel<2><<<grid_of(ncand), 256, 0, st>>>(m, in.pairs, np, lco.p, lcell.p, poff.p, ncand, ck.p), note_launch();
  sort_keys(ck, cks, ncand, st);
  int nu = 0;
  if (ncand > 0) {
    size_t tmp = 0;
    cub::DeviceSelect::Unique(nullptr, tmp, cks.p, U.p, nuniq.p, (int)ncand, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceSelect::Unique(tb.p, tmp, cks.p, U.p, nuniq.p, (int)ncand, st));
    unsigned long long last = 0;
    FL_CUDA(cudaMemcpyAsync(&nu, nuniq.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    if (nu > 0) {
      FL_CUDA(cudaMemcpyAsync(&last, U.p + nu - 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      FL_CUDA(cudaStreamSynchronize(st));
      if (last == NONE) --nu;                 // the non-disjoint marker sorts last
    }
  }
  *npairs_out = nu;
  // orders, hash, one block per pair
  DBuf<int> P(std::max(nu, 1)), Qc(std::max(nu, 1)), Kc(std::max(nu, 1));
  DBuf<double> G((size_t)9 * std::max(nu, 1));
  unsigned long long cap = 1024;
  while (cap < 2ull * (unsigned long long)nu) cap <<= 1;
  DBuf<unsigned long long> hkey(cap);
  DBuf<int> hidx(cap);
  FL_CUDA(cudaMemsetAsync(hkey.p, 0xff, cap * sizeof(unsigned long long), st));
  if (nu > 0) {
    if (m.d == 1)
      near_orders_kernel<1><<<grid_of(nu), 256, 0, st>>>(m, oc, U.p, nu, P.p, Qc.p, Kc.p, hkey.p, hidx.p, cap - 1), note_launch();
    else
      near_orders_kernel<2><<<grid_of(nu), 256, 0, st>>>(m, oc, U.p, nu, P.p, Qc.p, Kc.p, hkey.p, hidx.p, cap - 1), note_launch();
    launch_near_blocks(m, t, oc, ex, e4, P.p, Qc.p, Kc.p, nu, G.p, evals, st);
  }
  // CSR pattern: row i holds the DoFs of every leaf near leaf(i), ascending
  DBuf<int64_t> ac(std::max<int64_t>(np, 1)), aoff(np + 1);
  adj_count_kernel<<<grid_of(np), 256, 0, st>>>(in.pairs, np, ldo.p, ac.p), note_launch();
  const int64_t ncol = excl_scan(ac.p, aoff.p, np, st);
  if (ncol >= (1LL << 31)) throw Error(FL_E_ASSEMBLY, "near field too large (leaf columns >= 2^31)");
  DBuf<unsigned long long> colk(std::max<int64_t>(ncol, 1)), cols;
  col_keys_kernel<<<grid_of(ncol), 256, 0, st>>>(in.pairs, np, ldo.p, ldof.p, aoff.p, ncol, colk.p), note_launch();
  sort_keys(colk, cols, ncol, st);
  seg_offsets_kernel<<<grid_of(nl + 1), 256, 0, st>>>(cols.p, ncol, nl, lcol.p), note_launch();
  DBuf<int64_t> rl(std::max(n, 1));
  out.indptr.alloc(n + 1);
  row_len_kernel<<<grid_of(n), 256, 0, st>>>(in.leaf_of_dof, n, lcol.p, rl.p), note_launch();
  out.nnz = excl_scan(rl.p, out.indptr.p, n, st);
  out.indices.alloc(std::max<int64_t>(out.nnz, 1));
  out.data.alloc(std::max<int64_t>(out.nnz, 1));
  if (m.d == 1)
    near_values_kernel<1><<<grid_of((int64_t)n * 32), 256, 0, st>>>(m, in.leaf_of_dof, lcol.p, cols.p, row_vertex,
                                                                  out.indptr.p, out.indices.p, out.data.p, hkey.p,
                                                                  hidx.p, cap - 1, G.p, -Cds), note_launch();
  else
    near_values_kernel<2><<<grid_of((int64_t)n * 32), 256, 0, st>>>(m, in.leaf_of_dof, lcol.p, cols.p, row_vertex,
                                                                  out.indptr.p, out.indices.p, out.data.p, hkey.p,
                                                                  hidx.p, cap - 1, G.p, -Cds), note_launch();
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaStreamSynchronize(st));   // the work buffers above are released on return
}

}  // namespace fl
