// Mesh preparation on the device: per-cell geometry, cell quadrature nodes, vertex patches,
// touching-pair / boundary-pair classification and the DoF tiles
// of the cross kernel.
//
// Reference: mesh.py:76-130 (diameters, patches), assembly.py:282-298 (cell rule),
// assembly.py:412-473 (enumerate/canonicalize touching pairs), assembly.py:784-841
// (boundary pairs), quadrature.py:90-110 (classification), :138-179 (orders).
#include <cub/cub.cuh>

#include "fl_internal.h"

namespace fl {

// ---------------------------------------------------------------- per-cell geometry
template <int D>
__global__ void prep_cells_kernel(DevMesh m, CellGeo* geo) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m.nc) return;
  CellGeo g;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    g.v[i] = -1; g.dof[i] = -1; g.p[i][0] = 0.0; g.p[i][1] = 0.0;
  }
#pragma unroll
  for (int i = 0; i <= D; ++i) {
    const int v = m.cells[c * (D + 1) + i];
    g.v[i] = v;
    g.dof[i] = m.v2d[v];
#pragma unroll
    for (int j = 0; j < D; ++j) g.p[i][j] = m.vert[v * D + j];
  }
  if constexpr (D == 1) {
    g.diam = fabs(__dsub_rn(g.p[1][0], g.p[0][0]));           // mesh.py:80
    g.J = g.diam;                                              // assembly.py:137
    g.cx = __dmul_rn(0.5, __dadd_rn(g.p[0][0], g.p[1][0]));
    g.cy = 0.0;
    g.rad = __dmul_rn(0.5, g.diam);
  } else {
    const double e0 = norm2d(__dsub_rn(g.p[1][0], g.p[0][0]), __dsub_rn(g.p[1][1], g.p[0][1]));
    const double e1 = norm2d(__dsub_rn(g.p[2][0], g.p[1][0]), __dsub_rn(g.p[2][1], g.p[1][1]));
    const double e2 = norm2d(__dsub_rn(g.p[0][0], g.p[2][0]), __dsub_rn(g.p[0][1], g.p[2][1]));
    g.diam = fmax(e0, fmax(e1, e2));                           // mesh.py:82-85
    const double ax = __dsub_rn(g.p[1][0], g.p[0][0]), ay = __dsub_rn(g.p[1][1], g.p[0][1]);
    const double bx = __dsub_rn(g.p[2][0], g.p[0][0]), by = __dsub_rn(g.p[2][1], g.p[0][1]);
    g.J = fabs(__dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx)));   // assembly.py:138-140
    g.cx = __ddiv_rn(__dadd_rn(__dadd_rn(g.p[0][0], g.p[1][0]), g.p[2][0]), 3.0);   // :771
    g.cy = __ddiv_rn(__dadd_rn(__dadd_rn(g.p[0][1], g.p[1][1]), g.p[2][1]), 3.0);
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) r = fmax(r, norm2d(__dsub_rn(g.p[i][0], g.cx), __dsub_rn(g.p[i][1], g.cy)));
    g.rad = r;                                                 // :773
  }
  g.ldiam = fabs(log(g.diam));
  g.pad = 0;
  geo[c] = g;
}

void launch_prep_cells(const DevMesh& m, CellGeo* geo, cudaStream_t st) {
  const int tb = 128, nb = (m.nc + tb - 1) / tb;
  if (m.d == 1) prep_cells_kernel<1><<<nb, tb, 0, st>>>(m, geo), ::fl::note_launch();
  else prep_cells_kernel<2><<<nb, tb, 0, st>>>(m, geo), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- cell quadrature nodes
template <int D>
__global__ void cell_nodes_kernel(DevMesh m, const double* __restrict__ tab, RuleRef r,
                                  double* X, double* W) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nc * r.cnt) return;
  const int c = i / r.cnt, q = i % r.cnt;
  const CellGeo g = m.geo[c];
  const double* nd = tab + (size_t)(r.off + q) * NODE;
  if constexpr (D == 1) {
    const double e = __dsub_rn(g.p[1][0], g.p[0][0]);
    X[i] = g.p[0][0] + nd[0] * e;
  } else {
    const double e00 = __dsub_rn(g.p[1][0], g.p[0][0]), e01 = __dsub_rn(g.p[1][1], g.p[0][1]);
    const double e10 = __dsub_rn(g.p[2][0], g.p[0][0]), e11 = __dsub_rn(g.p[2][1], g.p[0][1]);
    X[2 * i + 0] = g.p[0][0] + (nd[0] * e00 + nd[1] * e10);
    X[2 * i + 1] = g.p[0][1] + (nd[0] * e01 + nd[1] * e11);
  }
  W[i] = __dmul_rn(g.J, nd[2]);                                 // np.outer(J, w)
}

void launch_cell_nodes(const DevMesh& m, const DevTables& t, double* X, double* W, cudaStream_t st) {
  const RuleRef r = t.rule(T_CELL, 0);
  const int tot = m.nc * r.cnt, tb = 256;
  if (m.d == 1) cell_nodes_kernel<1><<<(tot + tb - 1) / tb, tb, 0, st>>>(m, t.data, r, X, W), ::fl::note_launch();
  else cell_nodes_kernel<2><<<(tot + tb - 1) / tb, tb, 0, st>>>(m, t.data, r, X, W), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- vertex patches (CSR)
__global__ void iota_kernel(int* a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
// mesh.py:114-125: argsort(cells.ravel(), kind="stable") -> per vertex, ascending cell ids.
__global__ void max_valence_kernel(const int* off, int nv, int* mx) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  int val = v < nv ? off[v + 1] - off[v] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) val = max(val, __shfl_xor_sync(0xffffffffu, val, o));
  if ((threadIdx.x & 31) == 0 && val > 0) atomicMax(mx, val);
}
void launch_max_valence(const int* off, int nv, int* mx, cudaStream_t st) {
  max_valence_kernel<<<(nv + 255) / 256, 256, 0, st>>>(off, nv, mx), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// vertex -> cells CSR by counting (valences are small): counts, one scan, a fill by atomic slot
// claims, then each vertex's few cells sorted ascending — the order of
// argsort(cells.ravel(), kind="stable") (mesh.py:114-125) without a device-wide radix sort
__global__ void patch_count_kernel(const int* __restrict__ cells, int m, int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) atomicAdd(&cnt[cells[i]], 1);
}
__global__ void patch_fill_kernel(const int* __restrict__ cells, int m, int dp1, const int* __restrict__ off,
                                  int* __restrict__ cursor, int* __restrict__ data) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int v = cells[i];
  data[off[v] + atomicAdd(&cursor[v], 1)] = i / dp1;
}
__global__ void patch_sort_kernel(const int* __restrict__ off, int nv, int* __restrict__ data) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int a = off[v], b = off[v + 1];
  for (int i = a + 1; i < b; ++i) {
    const int x = data[i];
    int j = i - 1;
    while (j >= a && data[j] > x) { data[j + 1] = data[j]; --j; }
    data[j + 1] = x;
  }
}

void build_patches(int nv, int nc, int d, const int* cells, DBuf<int>& off, DBuf<int>& data,
                   cudaStream_t st) {
  const int m = nc * (d + 1);
  DBuf<int> cnt(nv + 1), cursor(nv);
  off.alloc(nv + 1);
  data.alloc(m);
  FL_CUDA(cudaMemsetAsync(cnt.p, 0, (nv + 1) * sizeof(int), st));
  FL_CUDA(cudaMemsetAsync(cursor.p, 0, nv * sizeof(int), st));
  patch_count_kernel<<<(m + 255) / 256, 256, 0, st>>>(cells, m, cnt.p), ::fl::note_launch();
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, off.p, nv + 1, st);
  DBuf<unsigned char> t(tmp);
  FL_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.p, off.p, nv + 1, st));
  patch_fill_kernel<<<(m + 255) / 256, 256, 0, st>>>(cells, m, d + 1, off.p, cursor.p, data.p), ::fl::note_launch();
  patch_sort_kernel<<<(nv + 255) / 256, 256, 0, st>>>(off.p, nv, data.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- touching pairs
constexpr int MAXNB = 96;   // distinct neighbours of one cell

template <int D>
__device__ int neighbours_above(const DevMesh& m, int K, int* out) {
  int cnt = 0;
  for (int i = 0; i <= D; ++i) {
    const int v = m.cells[K * (D + 1) + i];
    for (int p = m.patch_off[v]; p < m.patch_off[v + 1]; ++p) {
      const int o = m.patch_cells[p];
      if (o <= K) continue;
      bool seen = false;
      for (int j = 0; j < cnt; ++j) seen |= (out[j] == o);
      if (!seen && cnt < MAXNB) out[cnt++] = o;
    }
  }
  // insertion sort: pairs sorted by (min, max) as sorted(set) in assembly.py:423
  for (int i = 1; i < cnt; ++i) {
    const int x = out[i];
    int j = i - 1;
    while (j >= 0 && out[j] > x) { out[j + 1] = out[j]; --j; }
    out[j + 1] = x;
  }
  return cnt;
}

template <int D>
__global__ void touch_count_kernel(DevMesh m, int* counts) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K >= m.nc) return;
  int nb[MAXNB];
  counts[K] = neighbours_above<D>(m, K, nb);
}

template <int D>
__global__ void touch_fill_kernel(DevMesh m, OrderConsts oc, const int* offs, TouchPair* pairs, int* ident_k) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K >= m.nc) return;
  const CellGeo A = m.geo[K];
  ident_k[K] = order_touching(oc, A.diam, A.ldiam, false);   // assembly.py:658
  int nb[MAXNB];
  const int cnt = neighbours_above<D>(m, K, nb);
  int o = offs[K];
  for (int t = 0; t < cnt; ++t) {
    const int K2 = nb[t];
    const CellGeo B = m.geo[K2];
    TouchPair tp;
    tp.c0 = K; tp.c1 = K2;
    for (int i = 0; i < 5; ++i) tp.locs[i] = -1;
    for (int i = 0; i < 3; ++i) { tp.vK[i] = -1; tp.vK2[i] = -1; }
    // hmin = np.minimum(h_K, h_K2) -> |log hmin| (quadrature.py:154-155)
    const double lmin = (A.diam <= B.diam) ? A.ldiam : B.ldiam;
    tp.k = order_touching(oc, fmin(A.diam, B.diam), lmin, false);
    if constexpr (D == 1) {
      // assembly.py:435-446: shared vertex first in both cells
      int sh = -1;
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          if (A.v[i] == B.v[j]) sh = max(sh, A.v[i]);
      tp.topo = T_CV;
      tp.vK[0] = sh; tp.vK[1] = (A.v[0] == sh) ? A.v[1] : A.v[0];
      tp.vK2[0] = sh; tp.vK2[1] = (B.v[0] == sh) ? B.v[1] : B.v[0];
      tp.locs[0] = sh; tp.locs[1] = tp.vK[1]; tp.locs[2] = tp.vK2[1];
      tp.nloc = 3;
    } else {
      // assembly.py:452-472: common = sorted(shared); vK = common + restA; vK2 = common + restB
      int common[3], nc_ = 0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          if (A.v[i] == B.v[j]) common[nc_++] = A.v[i];
      if (nc_ == 2 && common[0] > common[1]) { const int x = common[0]; common[0] = common[1]; common[1] = x; }
      int ka = 0, kb = 0;
      for (int i = 0; i < nc_; ++i) { tp.vK[ka++] = common[i]; tp.vK2[kb++] = common[i]; }
      for (int i = 0; i < 3; ++i) {
        bool inA = false, inB = false;
        for (int j = 0; j < nc_; ++j) { inA |= (A.v[i] == common[j]); inB |= (B.v[i] == common[j]); }
        if (!inA) tp.vK[ka++] = A.v[i];
        if (!inB) tp.vK2[kb++] = B.v[i];
      }
      if (nc_ == 2) {                                  // COMMON_EDGE, 4 locals (:469)
        tp.topo = T_CE;
        tp.locs[0] = tp.vK[0]; tp.locs[1] = tp.vK[1]; tp.locs[2] = tp.vK[2]; tp.locs[3] = tp.vK2[2];
        tp.nloc = 4;
      } else {                                         // COMMON_VERTEX, 5 locals (:471)
        tp.topo = T_CV;
        tp.locs[0] = tp.vK[0]; tp.locs[1] = tp.vK[1]; tp.locs[2] = tp.vK[2];
        tp.locs[3] = tp.vK2[1]; tp.locs[4] = tp.vK2[2];
        tp.nloc = 5;
      }
    }
    pairs[o + t] = tp;
  }
}

void touching_count(const DevMesh& m, DBuf<int>& counts, DBuf<int>& offs, cudaStream_t st) {
  const int tb = 128, nb = (m.nc + tb - 1) / tb;
  counts.alloc(m.nc + 1);
  offs.alloc(m.nc + 1);
  FL_CUDA(cudaMemsetAsync(counts.p, 0, (m.nc + 1) * sizeof(int), st));
  if (m.d == 1) touch_count_kernel<1><<<nb, tb, 0, st>>>(m, counts.p), ::fl::note_launch();
  else touch_count_kernel<2><<<nb, tb, 0, st>>>(m, counts.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts.p, offs.p, m.nc + 1, st);
  DBuf<unsigned char> t(tmp);
  FL_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, counts.p, offs.p, m.nc + 1, st));
}

void touching_fill(const DevMesh& m, const OrderConsts& oc, const DBuf<int>& offs, int64_t total,
                   DBuf<TouchPair>& pairs, DBuf<int>& ident_k, cudaStream_t st) {
  const int tb = 128, nb = (m.nc + tb - 1) / tb;
  pairs.alloc(total > 0 ? total : 1);
  ident_k.alloc(m.nc);
  if (m.d == 1) touch_fill_kernel<1><<<nb, tb, 0, st>>>(m, oc, offs.p, pairs.p, ident_k.p), ::fl::note_launch();
  else touch_fill_kernel<2><<<nb, tb, 0, st>>>(m, oc, offs.p, pairs.p, ident_k.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

void classify_touching(const DevMesh& m, const OrderConsts& oc, DBuf<TouchPair>& pairs,
                       int64_t& npairs, DBuf<int>& ident_k, cudaStream_t st) {
  DBuf<int> counts, offs;
  touching_count(m, counts, offs, st);
  int total = 0;
  FL_CUDA(cudaMemcpyAsync(&total, offs.p + m.nc, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  npairs = total;
  touching_fill(m, oc, offs, total, pairs, ident_k, st);
}

// ---------------------------------------------------------------- boundary pairs
template <int D>
__device__ int edge_cells(const DevMesh& m, int e, int* out) {
  int cnt = 0;
  for (int i = 0; i < D; ++i) {
    const int v = m.bedges[e * D + i];
    for (int p = m.patch_off[v]; p < m.patch_off[v + 1]; ++p) {
      const int o = m.patch_cells[p];
      bool seen = false;
      for (int j = 0; j < cnt; ++j) seen |= (out[j] == o);
      if (!seen && cnt < MAXNB) out[cnt++] = o;
    }
  }
  for (int i = 1; i < cnt; ++i) {   // np.unique -> ascending (assembly.py:799)
    const int x = out[i];
    int j = i - 1;
    while (j >= 0 && out[j] > x) { out[j + 1] = out[j]; --j; }
    out[j + 1] = x;
  }
  return cnt;
}

template <int D>
__global__ void bnd_count_kernel(DevMesh m, int* counts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.nb) return;
  int cs[MAXNB];
  counts[e] = edge_cells<D>(m, e, cs);    // every patch cell shares >= 1 vertex
}

template <int D>
__global__ void bnd_fill_kernel(DevMesh m, OrderConsts oc, const int* offs, BndPair* items) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.nb) return;
  int cs[MAXNB];
  const int cnt = edge_cells<D>(m, e, cs);
  int ev[2] = {m.bedges[e * D + 0], D == 2 ? m.bedges[e * D + 1] : -1};
  for (int t = 0; t < cnt; ++t) {
    const int c = cs[t];
    const CellGeo g = m.geo[c];
    BndPair it;
    it.cell = c; it.edge = e;
    int shared[2], ns = 0;
    for (int i = 0; i < D; ++i)
      for (int j = 0; j <= D; ++j)
        if (ev[i] == g.v[j]) shared[ns++] = ev[i];
    if (ns == 2 && shared[0] > shared[1]) { const int x = shared[0]; shared[0] = shared[1]; shared[1] = x; }
    int order[3] = {-1, -1, -1};
    int pe[2] = {-1, -1};
    if (D == 1) {                                  // 1D: boundary point first (:832-835)
      it.topo = T_EOC;
      order[0] = ev[0];
      order[1] = (g.v[0] == ev[0]) ? g.v[1] : g.v[0];
      pe[0] = ev[0];
      it.nloc = 2;
    } else if (ns == 2) {                          // EDGE_OF_CELL (:824-826)
      it.topo = T_EOC;
      order[0] = ev[0]; order[1] = ev[1];
      for (int j = 0; j < 3; ++j)
        if (g.v[j] != ev[0] && g.v[j] != ev[1]) order[2] = g.v[j];
      pe[0] = ev[0]; pe[1] = ev[1];
      it.nloc = 3;
    } else {                                       // TOUCHING_EDGE (:827-831)
      it.topo = T_TE;
      const int sv = shared[0];
      order[0] = sv;
      int k = 1;
      for (int j = 0; j < 3; ++j)
        if (g.v[j] != sv) order[k++] = g.v[j];
      pe[0] = sv;
      pe[1] = (ev[0] == sv) ? ev[1] : ev[0];
      it.nloc = 3;
    }
    for (int j = 0; j < 3; ++j) it.locs[j] = order[j];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        it.pe[i][j] = (pe[i] >= 0 && j < D) ? m.vert[pe[i] * D + j] : 0.0;
    it.ne[0] = -m.bnorm[e * D + 0];
    it.ne[1] = (D == 2) ? -m.bnorm[e * D + 1] : 0.0;
    it.k = order_touching(oc, g.diam, g.ldiam, true);      // select_order(..., boundary=True) :815
    items[offs[e] + t] = it;
  }
}

void boundary_count(const DevMesh& m, DBuf<int>& counts, DBuf<int>& offs, cudaStream_t st) {
  const int tb = 64, nb = (m.nb + tb - 1) / tb;
  counts.alloc(m.nb + 1);
  offs.alloc(m.nb + 1);
  FL_CUDA(cudaMemsetAsync(counts.p, 0, (m.nb + 1) * sizeof(int), st));
  if (m.d == 1) bnd_count_kernel<1><<<nb, tb, 0, st>>>(m, counts.p), ::fl::note_launch();
  else bnd_count_kernel<2><<<nb, tb, 0, st>>>(m, counts.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts.p, offs.p, m.nb + 1, st);
  DBuf<unsigned char> t(tmp);
  FL_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, counts.p, offs.p, m.nb + 1, st));
}

void boundary_fill(const DevMesh& m, const OrderConsts& oc, const DBuf<int>& offs, int64_t total,
                   DBuf<BndPair>& items, cudaStream_t st) {
  const int tb = 64, nb = (m.nb + tb - 1) / tb;
  items.alloc(total > 0 ? total : 1);
  if (m.d == 1) bnd_fill_kernel<1><<<nb, tb, 0, st>>>(m, oc, offs.p, items.p), ::fl::note_launch();
  else bnd_fill_kernel<2><<<nb, tb, 0, st>>>(m, oc, offs.p, items.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

void classify_boundary(const DevMesh& m, const OrderConsts& oc, DBuf<BndPair>& items,
                       int64_t& nitems, cudaStream_t st) {
  nitems = 0;
  if (m.nb == 0) { items.alloc(1); return; }
  DBuf<int> counts, offs;
  boundary_count(m, counts, offs, st);
  int total = 0;
  FL_CUDA(cudaMemcpyAsync(&total, offs.p + m.nb, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  nitems = total;
  boundary_fill(m, oc, offs, total, items, st);
}

// ---------------------------------------------------------------- DoF tiles
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
__global__ void dof_vertex_kernel(DevMesh m, int* dof_vertex) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m.nv) return;
  const int d = m.v2d[v];
  if (d >= 0) dof_vertex[d] = v;
}
__global__ void morton_kernel(DevMesh m, const int* dof_vertex, int r0, int r1, double x0, double y0,
                              double sx, double sy, uint32_t* keys, int* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1 - r0) return;
  const int dof = r0 + i;
  const int v = dof_vertex[dof];
  uint32_t key;
  if (m.d == 1) {
    key = (uint32_t)i;
  } else {
    const double fx = (m.vert[2 * v] - x0) * sx, fy = (m.vert[2 * v + 1] - y0) * sy;
    const uint32_t qx = (uint32_t)fmin(fmax(fx, 0.0), 65535.0);
    const uint32_t qy = (uint32_t)fmin(fmax(fy, 0.0), 65535.0);
    key = spread16(qx) | (spread16(qy) << 1);
  }
  keys[i] = key;
  vals[i] = dof;
}

constexpr int CAND = 1024;
__global__ void __launch_bounds__(256) tile_cells_kernel(DevMesh m, const int* sorted_dofs, int nrows,
                                                         const int* dof_vertex, int* tdofs, int* tncell,
                                                         int* tcells, int* tslots, double* tgeo,
                                                         double* tstat, int* err) {
  const int t = blockIdx.x;
  __shared__ int sd[TILE];
  __shared__ unsigned long long key[CAND];
  __shared__ int ncand;
  const int tid = threadIdx.x;
  if (tid < TILE) {
    const int i = t * TILE + tid;
    sd[tid] = (i < nrows) ? sorted_dofs[i] : -1;
    tdofs[t * TILE + tid] = sd[tid];
  }
  if (tid == 0) {
    ncand = 0;
    double cx = 0, cy = 0, r = 0;
    int c = 0;
    for (int i = 0; i < TILE; ++i)
      if (sd[i] >= 0) {
        const int v = dof_vertex[sd[i]];
        cx += m.vert[v * m.d];
        cy += (m.d == 2) ? m.vert[v * m.d + 1] : 0.0;
        ++c;
      }
    cx /= max(c, 1);
    cy /= max(c, 1);
    for (int i = 0; i < TILE; ++i)
      if (sd[i] >= 0) {
        const int v = dof_vertex[sd[i]];
        const double dx = m.vert[v * m.d] - cx, dy = (m.d == 2) ? m.vert[v * m.d + 1] - cy : 0.0;
        r = fmax(r, sqrt(dx * dx + dy * dy));
      }
    tgeo[3 * t] = cx;
    tgeo[3 * t + 1] = cy;
    tgeo[3 * t + 2] = r;
  }
  __syncthreads();
  if (tid < TILE && sd[tid] >= 0) {
    const int v = dof_vertex[sd[tid]];
    for (int p = m.patch_off[v]; p < m.patch_off[v + 1]; ++p) {
      const int c = m.patch_cells[p];
      const int slot = atomicAdd(&ncand, 1);
      if (slot < CAND) key[slot] = (unsigned long long)(unsigned)c;
    }
  }
  __syncthreads();
  const int nc_ = ncand;
  if (nc_ > CAND) { if (tid == 0) atomicAdd(err, 1); return; }
  for (int i = nc_ + tid; i < CAND; i += blockDim.x) key[i] = ~0ull;
  __syncthreads();
  // bitonic sort of the CAND candidate cell ids
  for (int k = 2; k <= CAND; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < CAND; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = ((i & k) == 0);
          const unsigned long long a = key[i], b = key[ixj];
          if ((a > b) == up) { key[i] = b; key[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  // unique (serial; <= CAND entries, once per tile)
  __shared__ int nuniq;
  if (tid == 0) {
    int u = 0;
    for (int i = 0; i < nc_; ++i)
      if (i == 0 || key[i] != key[i - 1]) key[u++] = key[i];
    nuniq = u;
  }
  __syncthreads();
  const int nu = nuniq;
  if (nu > TILE_MAXC) { if (tid == 0) atomicAdd(err, 1); return; }
  if (tid == 0) tncell[t] = nu;
  for (int i = tid; i < nu; i += blockDim.x) {
    const int c = (int)(key[i] & 0xffffffffu);
    tcells[t * TILE_MAXC + i] = c;
    for (int a = 0; a < 3; ++a) {
      int slot = -1;
      if (a <= m.d) {
        const int dof = m.v2d[m.cells[c * (m.d + 1) + a]];
        if (dof >= 0)
          for (int r = 0; r < TILE; ++r)
            if (sd[r] == dof) slot = r;
      }
      tslots[(t * TILE_MAXC + i) * 3 + a] = slot;
    }
  }
  // tile statistics for the order bounds: cell-covering radius about the DoF centre, h and |ln h| ranges
  {
    __shared__ double red[5][256];
    double R = 0.0, hmn = 1e300, hmx = 0.0, lmn = 1e300, lmx = 0.0;
    const double cx = tgeo[3 * t], cy = tgeo[3 * t + 1];
    for (int i = tid; i < nu; i += blockDim.x) {
      const CellGeo& g = m.geo[(int)(key[i] & 0xffffffffu)];
      const double dx = g.cx - cx, dy = g.cy - cy;
      R = fmax(R, sqrt(dx * dx + dy * dy) * (1.0 + 1e-12) + g.rad);
      hmn = fmin(hmn, g.diam); hmx = fmax(hmx, g.diam);
      lmn = fmin(lmn, g.ldiam); lmx = fmax(lmx, g.ldiam);
    }
    red[0][tid] = R; red[1][tid] = -hmn; red[2][tid] = hmx; red[3][tid] = -lmn; red[4][tid] = lmx;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (tid < o)
        for (int q = 0; q < 5; ++q) red[q][tid] = fmax(red[q][tid], red[q][tid + o]);
      __syncthreads();
    }
    if (tid == 0) {
      double* st = tstat + 8 * t;
      st[0] = cx; st[1] = cy; st[2] = red[0][0]; st[3] = -red[1][0]; st[4] = red[2][0];
      st[5] = -red[3][0]; st[6] = red[4][0]; st[7] = 0.0;
    }
  }
}

void build_tiles(const DevMesh& m, int row_begin, int row_end, Tiles& T, cudaStream_t st) {
  const int nrows = row_end - row_begin;
  T.ntiles = (nrows + TILE - 1) / TILE;
  DBuf<int> dof_vertex(m.n > 0 ? m.n : 1);
  dof_vertex_kernel<<<(m.nv + 255) / 256, 256, 0, st>>>(m, dof_vertex.p), ::fl::note_launch();
  // bounding box of the vertices (host copy is not available here; reduce on device)
  double bb[4] = {0, 1, 0, 1};
  if (m.d == 2) {
    std::vector<double> hv((size_t)m.nv * 2);
    FL_CUDA(cudaMemcpyAsync(hv.data(), m.vert, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    bb[0] = bb[1] = hv[0]; bb[2] = bb[3] = hv[1];
    for (int v = 0; v < m.nv; ++v) {
      bb[0] = std::min(bb[0], hv[2 * v]); bb[1] = std::max(bb[1], hv[2 * v]);
      bb[2] = std::min(bb[2], hv[2 * v + 1]); bb[3] = std::max(bb[3], hv[2 * v + 1]);
    }
  }
  const double sx = 65535.0 / std::max(bb[1] - bb[0], 1e-300), sy = 65535.0 / std::max(bb[3] - bb[2], 1e-300);
  DBuf<uint32_t> keys(nrows), keys2(nrows);
  DBuf<int> vals(nrows), vals2(nrows);
  morton_kernel<<<(nrows + 255) / 256, 256, 0, st>>>(m, dof_vertex.p, row_begin, row_end, bb[0], bb[2],
                                                    sx, sy, keys.p, vals.p), ::fl::note_launch();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, keys2.p, vals.p, vals2.p, nrows, 0, 32, st);
  DBuf<unsigned char> tb(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, keys.p, keys2.p, vals.p, vals2.p, nrows, 0, 32, st));
  T.dofs.alloc((size_t)T.ntiles * TILE);
  T.ncell.alloc(T.ntiles);
  T.cells.alloc((size_t)T.ntiles * TILE_MAXC);
  T.slots.alloc((size_t)T.ntiles * TILE_MAXC * 3);
  T.geo3.alloc((size_t)T.ntiles * 3);
  T.stat.alloc((size_t)T.ntiles * 8);
  DBuf<int> err(1);
  FL_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), st));
  tile_cells_kernel<<<T.ntiles, 256, 0, st>>>(m, vals2.p, nrows, dof_vertex.p, T.dofs.p, T.ncell.p,
                                              T.cells.p, T.slots.p, T.geo3.p, T.stat.p, err.p),
      ::fl::note_launch();
  FL_CHECK_LAUNCH();
  int herr = 0;
  FL_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (herr) throw Error(-2, "DoF tile touches more than 256 cells (vertex valence too high)");
}

__global__ void pair_cells_kernel(const int2* pairs, const int* n, const int* rcnt, const int* ccnt,
                                  unsigned long long* sum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (i < *n) v = (unsigned long long)rcnt[pairs[i].x] * (unsigned long long)ccnt[pairs[i].y];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(sum, v);
}
__global__ void gather_pairs_kernel(const int2* raw, const int* flag, const int* idx, int n, int2* out, int* oflag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { out[i] = raw[idx[i]]; oflag[i] = flag[idx[i]]; }
}

// Upper bound of select_order's disjoint formula (quadrature.py:159-168) over all pairs of two
// tiles: dist >= Dmin (the reference's estimate is >= the centroid gap minus the radii, which is
// >= the tile gap), h in [hmin, hmax], |ln h| in [lmin, lmax]; every term of the numerator is
// bounded above and the denominator below (it is >= ln rho2 > 0).
__device__ double order_bound_hi(const OrderConsts& oc, double Dmin, double hmin, double hmax, double lmin,
                                 double lmax) {
  (void)hmin;
  if (!(Dmin > 0.0)) return 1e30;
  const double num = oc.lead_lnn + oc.sm1 * lmin + lmax - oc.s * log(Dmin) + oc.s * log(hmax) - oc.coff;
  const double den = fmax(log(Dmin / hmax), 0.0) + oc.ln_rho2;
  return num > 0.0 ? num / den : 0.0;
}

__global__ void tile_pairs_kernel(OrderConsts oc, const double* __restrict__ rs, const double* __restrict__ cs,
                                  int nrt, int nct, int symmetric, int kw, int64_t npairs, int2* __restrict__ pairs,
                                  unsigned* __restrict__ key, int* __restrict__ nearflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  int r, c;
  if (symmetric) {   // row-major upper triangle
    const double q = 2.0 * nrt + 1.0;
    r = (int)((q - sqrt(q * q - 8.0 * (double)i)) * 0.5);
    auto cum = [&](int64_t e) { return e * nrt - e * (e - 1) / 2; };
    while (r > 0 && cum(r) > i) --r;
    while (cum(r + 1) <= i) ++r;
    c = r + (int)(i - cum(r));
  } else {
    r = (int)(i / nct);
    c = (int)(i - (int64_t)r * nct);
  }
  const double* a = rs + 8 * r;
  const double* b = cs + 8 * c;
  const double dc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
  const double Dmin = (dc - a[2] - b[2]) * (1.0 - 1e-12) - 1e-300;
  const double hmn = fmin(a[3], b[3]), hmx = fmax(a[4], b[4]), lmn = fmin(a[5], b[5]), lmx = fmax(a[6], b[6]);
  const double bh = order_bound_hi(oc, Dmin, hmn, hmx, lmn, lmx);
  pairs[i] = make_int2(r, c);
  nearflag[i] = (bh + 1e-9 > (double)(kw - 1)) ? 1 : 0;
  // heavy first: ascending tile gap (float bits of a non-negative float are monotonic)
  key[i] = __float_as_uint((float)fmax(Dmin, 0.0));
}

void build_tile_pairs(const DevMesh& m, const OrderConsts& oc, const Tiles& rows, const Tiles& cols, bool symmetric,
                      int kw, TilePairs& tp, cudaStream_t st) {
  (void)m;
  const int nrt = rows.ntiles, nct = cols.ntiles;
  const int64_t np = symmetric ? (int64_t)nrt * (nrt + 1) / 2 : (int64_t)nrt * nct;
  tp.nall = (int)np;
  tp.all.alloc(std::max<int64_t>(np, 1));
  tp.near.alloc(std::max<int64_t>(np, 1));
  tp.nnear = 0;
  if (np == 0) return;
  DBuf<int2> raw(np);
  DBuf<unsigned> key(np), key2(np);
  DBuf<int> flag(np), flag2(np), nsel(1);
  tile_pairs_kernel<<<(int)((np + 255) / 256), 256, 0, st>>>(oc, rows.stat.p, cols.stat.p, nrt, nct, symmetric ? 1 : 0,
                                                              kw, np, raw.p, key.p, flag.p), ::fl::note_launch();
  FL_CHECK_LAUNCH();
  // stable radix sort of (key -> pair, flag): deterministic heavy-first order
  DBuf<int> idx(np), idx2(np);
  iota_kernel<<<(int)((np + 255) / 256), 256, 0, st>>>(idx.p, (int)np), ::fl::note_launch();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, idx2.p, (int)np, 0, 32, st);
  DBuf<unsigned char> tb(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, key.p, key2.p, idx.p, idx2.p, (int)np, 0, 32, st));
  gather_pairs_kernel<<<(int)((np + 255) / 256), 256, 0, st>>>(raw.p, flag.p, idx2.p, (int)np, tp.all.p, flag2.p),
      ::fl::note_launch();
  size_t tmp2 = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp2, tp.all.p, flag2.p, tp.near.p, nsel.p, (int)np, st);
  DBuf<unsigned char> tb2(tmp2);
  FL_CUDA(cub::DeviceSelect::Flagged(tb2.p, tmp2, tp.all.p, flag2.p, tp.near.p, nsel.p, (int)np, st));
  // upper bound of the near keys the discovery pass can emit: sum of nR * nC over its tile pairs
  DBuf<unsigned long long> cand(1);
  FL_CUDA(cudaMemsetAsync(cand.p, 0, sizeof(unsigned long long), st));
  pair_cells_kernel<<<(int)((np + 255) / 256), 256, 0, st>>>(tp.near.p, nsel.p, rows.ncell.p, cols.ncell.p, cand.p),
      ::fl::note_launch();
  FL_CHECK_LAUNCH();
  unsigned long long hc = 0;
  FL_CUDA(cudaMemcpyAsync(&tp.nnear, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&hc, cand.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  tp.near_candidates = (int64_t)hc;
}

}  // namespace fl
