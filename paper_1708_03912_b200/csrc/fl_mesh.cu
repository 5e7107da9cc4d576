// Host-side O(n) steps of the reference's driver moved onto the device:
//
//  * fl_finish_polygon_mesh — _finish_polygon_mesh + _boundary_of (mesh.py:351-403): CCW
//    orientation, refinement (longest) edge first with the vertex-pair tie break, boundary
//    edges (undirected edges of exactly one cell, lexicographic order like np.unique) with
//    outward unit normals;
//  * fl_dofmap — DofMap (mesh.py:200-240): all vertices for s < 1/2, interior ones otherwise,
//    DoFs numbered in vertex order;
//  * fl_cell_rule_nodes / fl_load_vector — load_vector (assembly.py:550-570): per-cell rule
//    nodes X = P0 + u E (_map_points, assembly.py:129-132) for the caller's f, then
//    b_i = sum_K sum_q J_K w_q f(X_q) lambda_a(q), accumulated per DoF over its cells in
//    ascending cell order (the order of np.add.at over the flattened cell_dofs).
// Floating-point steps use explicit round-to-nearest intrinsics where numpy's operation order
// decides a discrete choice (orientation sign, longest edge, normal flip).
#include <cub/cub.cuh>

#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

namespace fl {
namespace {

// ------------------------------------------------------------------ finish_polygon_mesh
__device__ __forceinline__ double edge_len(const double* V, int64_t a, int64_t b) {
  const double dx = __dsub_rn(V[2 * b], V[2 * a]), dy = __dsub_rn(V[2 * b + 1], V[2 * a + 1]);
  return sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));        // np.linalg.norm(axis=1)
}

// CCW orientation (mesh.py:356-359) and the three edge lengths (mesh.py:362-363)
__global__ void orient_kernel(const double* __restrict__ V, const int64_t* __restrict__ cin, int64_t nc,
                              int64_t* __restrict__ c, double* __restrict__ lens) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  int64_t v0 = cin[3 * k], v1 = cin[3 * k + 1], v2 = cin[3 * k + 2];
  const double ax = __dsub_rn(V[2 * v1], V[2 * v0]), ay = __dsub_rn(V[2 * v1 + 1], V[2 * v0 + 1]);
  const double bx = __dsub_rn(V[2 * v2], V[2 * v0]), by = __dsub_rn(V[2 * v2 + 1], V[2 * v0 + 1]);
  if (__dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx)) < 0.0) { const int64_t t = v1; v1 = v2; v2 = t; }
  c[3 * k] = v0; c[3 * k + 1] = v1; c[3 * k + 2] = v2;
  lens[3 * k] = edge_len(V, v0, v1);
  lens[3 * k + 1] = edge_len(V, v1, v2);
  lens[3 * k + 2] = edge_len(V, v2, v0);
}

// longest edge first: argmax of round(len / max len, 12) * 4 nv^2 + lo * 2 nv + hi (mesh.py:364-372),
// the first maximal local edge on ties (np.argmax); then the undirected edge keys of the rolled cell
__global__ void roll_kernel(const double* __restrict__ lens, const double* __restrict__ lmax, int64_t nc, int64_t nv,
                            int64_t* __restrict__ c, unsigned long long* __restrict__ ekey, int* __restrict__ eidx) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  const int64_t v[3] = {c[3 * k], c[3 * k + 1], c[3 * k + 2]};
  const double L = *lmax, nn4 = (double)nv * (double)nv * 4.0, n2 = 2.0 * (double)nv;
  int r = 0;
  double best = 0.0;
  for (int i = 0; i < 3; ++i) {
    const int64_t a = v[i], b = v[(i + 1) % 3];
    const double lo = (double)(a < b ? a : b), hi = (double)(a < b ? b : a);
    const double q = __ddiv_rn(rint(__dmul_rn(__ddiv_rn(lens[3 * k + i], L), 1e12)), 1e12);   // np.round(x, 12)
    const double key = __dadd_rn(__dadd_rn(__dmul_rn(q, nn4), __dmul_rn(lo, n2)), hi);
    if (i == 0 || key > best) { best = key; r = i; }
  }
  int64_t w[3];
  for (int i = 0; i < 3; ++i) w[i] = v[(i + r) % 3];
  for (int i = 0; i < 3; ++i) {
    c[3 * k + i] = w[i];
    const int64_t a = w[i], b = w[(i + 1) % 3];
    ekey[3 * k + i] = (unsigned long long)(a < b ? a : b) * (unsigned long long)nv + (unsigned long long)(a < b ? b : a);
    eidx[3 * k + i] = (int)k;
  }
}

// sorted edge keys: an edge of count 1 (its neighbours differ) is a boundary edge; its owner is
// the single cell holding it (mesh.py:388-391)
__global__ void bflag_kernel(const unsigned long long* __restrict__ key, int64_t m, int* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const bool a = i > 0 && key[i - 1] == key[i], b = i + 1 < m && key[i + 1] == key[i];
  flag[i] = !(a || b);
}

__global__ void bnormal_kernel(const double* __restrict__ V, const int64_t* __restrict__ c,
                               const unsigned long long* __restrict__ key, const int* __restrict__ owner,
                               const int* __restrict__ sel, const int* __restrict__ nsel, int64_t nv,
                               int64_t* __restrict__ be, double* __restrict__ bn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *nsel) return;
  const int j = sel[i];
  const int64_t a = (int64_t)(key[j] / (unsigned long long)nv), b = (int64_t)(key[j] % (unsigned long long)nv);
  be[2 * i] = a;
  be[2 * i + 1] = b;
  const double px = V[2 * a], py = V[2 * a + 1], qx = V[2 * b], qy = V[2 * b + 1];
  const double tx = __dsub_rn(qx, px), ty = __dsub_rn(qy, py);
  double nx = ty, ny = -tx;
  const double nr = sqrt(__dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny)));
  nx = __ddiv_rn(nx, nr);
  ny = __ddiv_rn(ny, nr);
  const int64_t k = owner[j];
  // centroid = vertex mean (np.mean over 3: pairwise sum then divide)
  const int64_t v0 = c[3 * k], v1 = c[3 * k + 1], v2 = c[3 * k + 2];
  const double cx = __ddiv_rn(__dadd_rn(__dadd_rn(V[2 * v0], V[2 * v1]), V[2 * v2]), 3.0);
  const double cy = __ddiv_rn(__dadd_rn(__dadd_rn(V[2 * v0 + 1], V[2 * v1 + 1]), V[2 * v2 + 1]), 3.0);
  const double mx = __dsub_rn(__dmul_rn(0.5, __dadd_rn(px, qx)), cx);
  const double my = __dsub_rn(__dmul_rn(0.5, __dadd_rn(py, qy)), cy);
  if (__dadd_rn(__dmul_rn(mx, nx), __dmul_rn(my, ny)) < 0.0) { nx = -nx; ny = -ny; }
  bn[2 * i] = nx;
  bn[2 * i + 1] = ny;
}

// ------------------------------------------------------------------ DofMap
__global__ void bmark_kernel(const int64_t* __restrict__ be, int64_t m, int64_t nv, int* __restrict__ mark) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m && be[i] >= 0 && be[i] < nv) mark[be[i]] = 1;
}
__global__ void take_kernel(const int* __restrict__ mark, int64_t nv, int all, int* __restrict__ take) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) take[v] = all ? 1 : !mark[v];
}
__global__ void v2d_kernel(const int* __restrict__ take, const int* __restrict__ pos, int64_t nv,
                           int64_t* __restrict__ v2d) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) v2d[v] = take[v] ? (int64_t)pos[v] : -1;
}

// ------------------------------------------------------------------ load vector
__device__ __forceinline__ void map_node(const double* V, const int64_t* cell, int d, const double* u, double* x) {
  if (d == 1) {
    const double p0 = V[cell[0]], e = __dsub_rn(V[cell[1]], p0);
    x[0] = __dadd_rn(p0, __dmul_rn(u[0], e));
  } else {
    const double* P0 = V + 2 * cell[0];
    const double* P1 = V + 2 * cell[1];
    const double* P2 = V + 2 * cell[2];
    for (int k = 0; k < 2; ++k) {   // u @ E: u0 E0k + u1 E1k, then + P0k
      const double e0 = __dsub_rn(P1[k], P0[k]), e1 = __dsub_rn(P2[k], P0[k]);
      x[k] = __dadd_rn(P0[k], __dadd_rn(__dmul_rn(u[0], e0), __dmul_rn(u[1], e1)));
    }
  }
}

__global__ void nodes_kernel(const double* __restrict__ V, const int64_t* __restrict__ cells, int64_t nc, int d,
                             const double* __restrict__ pts, int q, double* __restrict__ X) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc * q) return;
  const int64_t k = i / q;
  const int r = (int)(i - k * q);
  map_node(V, cells + (d + 1) * k, d, pts + d * r, X + d * i);
}

// loc[K][a] = sum_q (J_K w_q f_q) lambda_a(q)   (assembly.py:561-563, _jacobians :135-140)
__global__ void load_local_kernel(const double* __restrict__ V, const int64_t* __restrict__ cells, int64_t nc, int d,
                                  const double* __restrict__ pts, const double* __restrict__ w, int q,
                                  const double* __restrict__ fv, double fconst, double* __restrict__ loc) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  const int64_t* c = cells + (d + 1) * k;
  double J;
  if (d == 1) {
    J = fabs(__dsub_rn(V[c[1]], V[c[0]]));
  } else {
    const double ax = __dsub_rn(V[2 * c[1]], V[2 * c[0]]), ay = __dsub_rn(V[2 * c[1] + 1], V[2 * c[0] + 1]);
    const double bx = __dsub_rn(V[2 * c[2]], V[2 * c[0]]), by = __dsub_rn(V[2 * c[2] + 1], V[2 * c[0] + 1]);
    J = fabs(__dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx)));
  }
  double acc[3] = {0.0, 0.0, 0.0};
  for (int r = 0; r < q; ++r) {
    const double f = fv ? fv[k * q + r] : fconst;
    const double wf = __dmul_rn(__dmul_rn(J, w[r]), f);
    const double u0 = pts[d * r], u1 = d == 2 ? pts[d * r + 1] : 0.0;
    const double lam0 = d == 1 ? __dsub_rn(1.0, u0) : __dsub_rn(__dsub_rn(1.0, u0), u1);
    acc[0] = __dadd_rn(acc[0], __dmul_rn(wf, lam0));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(wf, u0));
    if (d == 2) acc[2] = __dadd_rn(acc[2], __dmul_rn(wf, u1));
  }
  for (int a = 0; a <= d; ++a) loc[(d + 1) * k + a] = acc[a];
}

// (dof, flat index) pairs sorted by dof then flat index = cell-major np.add.at order
__global__ void dofkey_kernel(const int64_t* __restrict__ cells, const int64_t* __restrict__ v2d, int64_t m,
                              unsigned long long* __restrict__ key, int* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t dof = v2d[cells[i]];
  key[i] = dof < 0 ? ~0ull : ((unsigned long long)dof << 32) | (unsigned long long)i;
  idx[i] = (int)i;
}
__global__ void load_pull_kernel(const unsigned long long* __restrict__ key, const int* __restrict__ idx, int64_t m,
                                 const double* __restrict__ loc, double* __restrict__ b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || key[i] == ~0ull) return;
  const unsigned long long dof = key[i] >> 32;
  if (i > 0 && (key[i - 1] >> 32) == dof && key[i - 1] != ~0ull) return;   // not the first of its run
  double s = 0.0;
  for (int64_t j = i; j < m && key[j] != ~0ull && (key[j] >> 32) == dof; ++j) s = __dadd_rn(s, loc[idx[j]]);
  b[dof] = s;
}

__global__ void seq_kernel(int* a, int64_t m) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) a[i] = (int)i;
}

template <class T>
void h2d(DBuf<T>& d, const T* h, size_t cnt, cudaStream_t st) {
  d.alloc(cnt ? cnt : 1);
  if (cnt) FL_CUDA(cudaMemcpyAsync(d.p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, st));
}

int grid_of(int64_t m) { return (int)std::max<int64_t>(1, (m + 255) / 256); }

}  // namespace

int32_t finish_polygon_mesh(const double* V, int64_t nv, const int64_t* cells_in, int64_t nc, int device,
                            int64_t* cells_out, int64_t* be_out, double* bn_out, int64_t cap, int64_t* nb_out) {
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  StreamScope scope(st);
  DBuf<double> dV, lens(3 * nc), lmax(1);
  DBuf<int64_t> dcin, dc(3 * nc);
  h2d(dV, V, 2 * nv, st);
  h2d(dcin, cells_in, 3 * nc, st);
  orient_kernel<<<grid_of(nc), 256, 0, st>>>(dV.p, dcin.p, nc, dc.p, lens.p), note_launch();
  size_t tmp = 0;
  cub::DeviceReduce::Max(nullptr, tmp, lens.p, lmax.p, 3 * nc, st);
  DBuf<unsigned char> t1(tmp);
  FL_CUDA(cub::DeviceReduce::Max(t1.p, tmp, lens.p, lmax.p, 3 * nc, st));
  const int64_t m = 3 * nc;
  DBuf<unsigned long long> key(m), key2(m);
  DBuf<int> own(m), own2(m), flag(m), sel(m), nsel(1);
  roll_kernel<<<grid_of(nc), 256, 0, st>>>(lens.p, lmax.p, nc, nv, dc.p, key.p, own.p), note_launch();
  tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, own.p, own2.p, (int)m, 0, 64, st);
  DBuf<unsigned char> t2(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortPairs(t2.p, tmp, key.p, key2.p, own.p, own2.p, (int)m, 0, 64, st));
  bflag_kernel<<<grid_of(m), 256, 0, st>>>(key2.p, m, flag.p), note_launch();
  DBuf<int> iota(m);
  seq_kernel<<<grid_of(m), 256, 0, st>>>(iota.p, m), note_launch();
  tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, iota.p, flag.p, sel.p, nsel.p, (int)m, st);
  DBuf<unsigned char> t3(tmp);
  FL_CUDA(cub::DeviceSelect::Flagged(t3.p, tmp, iota.p, flag.p, sel.p, nsel.p, (int)m, st));
  DBuf<int64_t> be(2 * m);
  DBuf<double> bn(2 * m);
  bnormal_kernel<<<grid_of(m), 256, 0, st>>>(dV.p, dc.p, key2.p, own2.p, sel.p, nsel.p, nv, be.p, bn.p), note_launch();
  FL_CHECK_LAUNCH();
  int nb = 0;
  FL_CUDA(cudaMemcpyAsync(&nb, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(cells_out, dc.p, 3 * nc * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  *nb_out = nb;
  if (nb > cap) return FL_E_ARG;
  if (nb) {
    FL_CUDA(cudaMemcpyAsync(be_out, be.p, 2 * (size_t)nb * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaMemcpyAsync(bn_out, bn.p, 2 * (size_t)nb * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
}

int32_t dofmap_build(const int64_t* be, int64_t nb, int d, int64_t nv, double s, int device, int64_t* v2d_out,
                     int64_t* n_out) {
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  StreamScope scope(st);
  DBuf<int64_t> dbe, v2d(nv);
  h2d(dbe, be, nb * d, st);
  DBuf<int> mark(nv), take(nv), pos(nv), tot(1);
  FL_CUDA(cudaMemsetAsync(mark.p, 0, nv * sizeof(int), st));
  bmark_kernel<<<grid_of(nb * d), 256, 0, st>>>(dbe.p, nb * d, nv, mark.p), note_launch();
  take_kernel<<<grid_of(nv), 256, 0, st>>>(mark.p, nv, s < 0.5 ? 1 : 0, take.p), note_launch();   // mesh.py:225
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, take.p, pos.p, (int)nv, st);
  DBuf<unsigned char> t1(tmp);
  FL_CUDA(cub::DeviceScan::ExclusiveSum(t1.p, tmp, take.p, pos.p, (int)nv, st));
  v2d_kernel<<<grid_of(nv), 256, 0, st>>>(take.p, pos.p, nv, v2d.p), note_launch();
  FL_CHECK_LAUNCH();
  int last_pos = 0, last_take = 0;
  FL_CUDA(cudaMemcpyAsync(&last_pos, pos.p + nv - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&last_take, take.p + nv - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(v2d_out, v2d.p, nv * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  *n_out = (int64_t)last_pos + last_take;
  return FL_OK;
}

int32_t cell_rule_nodes(const fl_mesh* mesh, const double* pts, int64_t q, int device, double* X_out) {
  const int d = mesh->d;
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  StreamScope scope(st);
  DBuf<double> dV, dp, X((size_t)mesh->nc * q * d);
  DBuf<int64_t> dc;
  h2d(dV, mesh->vertices, mesh->nv * d, st);
  h2d(dc, mesh->cells, mesh->nc * (d + 1), st);
  h2d(dp, pts, q * d, st);
  nodes_kernel<<<grid_of(mesh->nc * q), 256, 0, st>>>(dV.p, dc.p, mesh->nc, d, dp.p, (int)q, X.p), note_launch();
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaMemcpyAsync(X_out, X.p, X.n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
}

int32_t load_vector(const fl_mesh* mesh, const fl_dofmap* dm, const double* pts, const double* w, int64_t q,
                    const double* fvals, double fconst, int device, double* b_out) {
  const int d = mesh->d;
  const int64_t nc = mesh->nc, n = dm->n, m = nc * (d + 1);
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  StreamScope scope(st);
  DBuf<double> dV, dp, dw, dfv, loc(m), b(std::max<int64_t>(n, 1));
  DBuf<int64_t> dc, dv2d;
  h2d(dV, mesh->vertices, mesh->nv * d, st);
  h2d(dc, mesh->cells, m, st);
  h2d(dv2d, dm->vertex_to_dof, mesh->nv, st);
  h2d(dp, pts, q * d, st);
  h2d(dw, w, q, st);
  if (fvals) h2d(dfv, fvals, nc * q, st);
  FL_CUDA(cudaMemsetAsync(b.p, 0, b.n * sizeof(double), st));
  load_local_kernel<<<grid_of(nc), 256, 0, st>>>(dV.p, dc.p, nc, d, dp.p, dw.p, (int)q, fvals ? dfv.p : nullptr,
                                                 fconst, loc.p), note_launch();
  DBuf<unsigned long long> key(m), key2(m);
  DBuf<int> idx(m), idx2(m);
  dofkey_kernel<<<grid_of(m), 256, 0, st>>>(dc.p, dv2d.p, m, key.p, idx.p), note_launch();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, idx2.p, (int)m, 0, 64, st);
  DBuf<unsigned char> t1(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortPairs(t1.p, tmp, key.p, key2.p, idx.p, idx2.p, (int)m, 0, 64, st));
  load_pull_kernel<<<grid_of(m), 256, 0, st>>>(key2.p, idx2.p, m, loc.p, b.p), note_launch();
  FL_CHECK_LAUNCH();
  if (n) FL_CUDA(cudaMemcpyAsync(b_out, b.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
}

}  // namespace fl
