// Local (sparse) contributions and their deterministic accumulation into the dense rows.
//
//  * cell-local matrices  Lc_K = (C/2) S^{KK} + C * int_K phi phi Psi_K + (C/2s) int_K phi phi W_in
//    (identical pair :658-667, weighted_mass_triplets :399-407 used at :1079-1080 and :1093-1094);
//  * touching pairs (weight C = (C/2)*2, :690) and boundary singular pairs (C/2s, :850, :1103).
// The pull kernel gives every DoF row to one thread, which walks the vertex patch in CSR order
// and adds its entries in a fixed order: race-free and bitwise reproducible (no atomics).
#include <cub/cub.cuh>

#include "fl_internal.h"

namespace fl {

template <int D>
__global__ void cell_local_kernel(DevMesh m, const double* __restrict__ tab, RuleRef cr, double Cds, double s,
                                  int integral, const int* __restrict__ targets, int ntargets,
                                  const double* __restrict__ ident, const double* __restrict__ psi,
                                  const double* __restrict__ win, double* __restrict__ Lc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntargets) return;
  const int K = targets[i];
  constexpr int NL = D + 1;
  double mp[NL][NL] = {}, mb[NL][NL] = {};
  const int Q = cr.cnt;
  for (int q = 0; q < Q; ++q) {
    const double* nd = tab + (size_t)(cr.off + q) * NODE;
    const double Wq = m.W[(size_t)K * Q + q];
    const double vp = Wq * psi[(size_t)K * Q + q];
    const double vb = integral ? Wq * win[(size_t)K * Q + q] : 0.0;
#pragma unroll
    for (int a = 0; a < NL; ++a)
#pragma unroll
      for (int b = 0; b < NL; ++b) {
        const double ll = nd[3 + a] * nd[3 + b];
        mp[a][b] = fma(vp, ll, mp[a][b]);
        mb[a][b] = fma(vb, ll, mb[a][b]);
      }
  }
  const double half = 0.5 * Cds, cb = Cds / (2.0 * s);
#pragma unroll
  for (int a = 0; a < NL; ++a)
#pragma unroll
    for (int b = 0; b < NL; ++b)
      Lc[(size_t)K * 9 + a * 3 + b] = half * ident[(size_t)K * 9 + a * 3 + b] + Cds * mp[a][b] + cb * mb[a][b];
}

void launch_cell_local(const DevMesh& m, const DevTables& t, double Cds, double s, bool integral,
                       const int* targets, int ntargets, const double* ident, const double* psi,
                       const double* win, double* Lc, cudaStream_t st) {
  if (ntargets <= 0) return;
  const RuleRef cr = t.rule(T_CELL, 0);
  const int grid = (ntargets + 127) / 128;
  if (m.d == 1)
    cell_local_kernel<1><<<grid, 128, 0, st>>>(m, t.data, cr, Cds, s, integral ? 1 : 0, targets, ntargets, ident,
                                               psi, win, Lc), ::fl::note_launch();
  else
    cell_local_kernel<2><<<grid, 128, 0, st>>>(m, t.data, cr, Cds, s, integral ? 1 : 0, targets, ntargets, ident,
                                               psi, win, Lc), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ index build
__global__ void pair_keys_kernel(const TouchPair* pairs, int64_t np, int* k0, int* k1, int* idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  k0[i] = pairs[i].c0;
  k1[i] = pairs[i].c1;
  idx[i] = (int)i;
}
__global__ void item_keys_kernel(const BndPair* items, int64_t ni, int* k, int* idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ni) return;
  k[i] = items[i].cell;
  idx[i] = (int)i;
}
// offsets of a sorted key array: off[v] = #keys < v, v = 0..nk (one binary search per v: no
// thread walks a long run of empty keys, e.g. the two boundary items of a 1D mesh over nc cells)
__global__ void offsets_kernel(const int* keys, int m, int nk, int* off) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > nk) return;
  int a = 0, b = m;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (keys[mid] < v) a = mid + 1; else b = mid;
  }
  off[v] = a;
}

static void sort_by_key(const int* keys, const int* vals, int* keys_out, int* vals_out, int m, int maxkey,
                        cudaStream_t st) {
  size_t tmp = 0;
  int bits = 1;
  while ((1 << bits) < maxkey + 1) ++bits;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys_out, vals, vals_out, m, 0, bits, st);
  DBuf<unsigned char> t(tmp);
  FL_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys, keys_out, vals, vals_out, m, 0, bits, st));
}

void build_sparse_index(const DevMesh& m, const TouchPair* pairs, int64_t npairs, const BndPair* items,
                        int64_t nitems, SparseIndex& si, cudaStream_t st) {
  const int nc = m.nc;
  si.tp_first_off.alloc(nc + 1);
  si.tp_second_off.alloc(nc + 1);
  si.bp_off.alloc(nc + 1);
  const int np = (int)npairs;
  if (np > 0) {
    DBuf<int> k0(np), k1(np), idx(np), k1s(np);
    si.tp_second.alloc(np);
    pair_keys_kernel<<<(np + 255) / 256, 256, 0, st>>>(pairs, np, k0.p, k1.p, idx.p), ::fl::note_launch();
    offsets_kernel<<<(nc + 1 + 255) / 256, 256, 0, st>>>(k0.p, np, nc, si.tp_first_off.p), ::fl::note_launch();  // already sorted by c0
    sort_by_key(k1.p, idx.p, k1s.p, si.tp_second.p, np, nc, st);                           // stable
    offsets_kernel<<<(nc + 1 + 255) / 256, 256, 0, st>>>(k1s.p, np, nc, si.tp_second_off.p), ::fl::note_launch();
  } else {
    si.tp_second.alloc(1);
    FL_CUDA(cudaMemsetAsync(si.tp_first_off.p, 0, (nc + 1) * sizeof(int), st));
    FL_CUDA(cudaMemsetAsync(si.tp_second_off.p, 0, (nc + 1) * sizeof(int), st));
  }
  const int ni = (int)nitems;
  if (ni > 0) {
    DBuf<int> k(ni), idx(ni), ks(ni);
    si.bp_idx.alloc(ni);
    item_keys_kernel<<<(ni + 255) / 256, 256, 0, st>>>(items, ni, k.p, idx.p), ::fl::note_launch();
    sort_by_key(k.p, idx.p, ks.p, si.bp_idx.p, ni, nc, st);
    offsets_kernel<<<(nc + 1 + 255) / 256, 256, 0, st>>>(ks.p, ni, nc, si.bp_off.p), ::fl::note_launch();
  } else {
    si.bp_idx.alloc(1);
    FL_CUDA(cudaMemsetAsync(si.bp_off.p, 0, (nc + 1) * sizeof(int), st));
  }
  FL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ the pull
// Where a row's local entries go: a dense row (the dense path), or a CSR row with sorted
// column indices (the near-field path; every local entry lies inside the row's pattern).
struct DenseRowSink {
  double* Ar;
  __device__ void add(int j, double v) { Ar[j] += v; }
};
struct CsrRowSink {
  const int* idx;
  double* val;
  int64_t lo, hi;
  __device__ void add(int j, double v) {
    int64_t a = lo, b = hi;                 // lower_bound of j in idx[lo, hi)
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (idx[mid] < j) a = mid + 1; else b = mid;
    }
    val[a] += v;
  }
};
struct DenseRows {
  double* A;
  int64_t lda;
  int row_begin;
  __device__ DenseRowSink row(int i) const { return DenseRowSink{A + (int64_t)(i - row_begin) * lda}; }
};
struct CsrRows {
  const int64_t* indptr;
  const int* idx;
  double* val;
  __device__ CsrRowSink row(int i) const { return CsrRowSink{idx, val, indptr[i], indptr[i + 1]}; }
};

template <int D, class Rows>
__global__ void sparse_pull_kernel(DevMesh m, double Cds, double cb, const double* __restrict__ Lc,
                                   const TouchPair* __restrict__ pairs, const double* __restrict__ tloc,
                                   const BndPair* __restrict__ items, const double* __restrict__ bloc,
                                   const int* __restrict__ tf_off, const int* __restrict__ ts_off,
                                   const int* __restrict__ ts_idx, const int* __restrict__ bp_off,
                                   const int* __restrict__ bp_idx, const int* __restrict__ row_vertex,
                                   int row_begin, int row_end, Rows rows) {
  const int i = row_begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= row_end) return;
  const int v = row_vertex[i];
  auto Ar = rows.row(i);
  for (int pp = m.patch_off[v]; pp < m.patch_off[v + 1]; ++pp) {
    const int K = m.patch_cells[pp];
    const CellGeo g = m.geo[K];
    int a = 0;
#pragma unroll
    for (int j = 0; j <= D; ++j)
      if (g.v[j] == v) a = j;
#pragma unroll
    for (int b = 0; b <= D; ++b)
      if (g.dof[b] >= 0) Ar.add(g.dof[b], Lc[(size_t)K * 9 + a * 3 + b]);
    // touching pairs with K as the first (smaller) cell
    for (int t = tf_off[K]; t < tf_off[K + 1]; ++t) {
      const TouchPair& tp = pairs[t];
      int sa = -1;
      for (int j = 0; j < tp.nloc; ++j)
        if (tp.locs[j] == v) sa = j;
      if (sa < 0) continue;
      const double* T = tloc + (size_t)t * 25 + sa * 5;
      for (int b = 0; b < tp.nloc; ++b) {
        const int dj = m.v2d[tp.locs[b]];
        if (dj >= 0) Ar.add(dj, Cds * T[b]);
      }
    }
    // ... and as the second cell, unless v also lies in the first cell (counted there)
    for (int u = ts_off[K]; u < ts_off[K + 1]; ++u) {
      const int t = ts_idx[u];
      const TouchPair& tp = pairs[t];
      const CellGeo g0 = m.geo[tp.c0];
      bool in0 = false;
#pragma unroll
      for (int j = 0; j <= D; ++j) in0 |= (g0.v[j] == v);
      if (in0) continue;
      int sa = -1;
      for (int j = 0; j < tp.nloc; ++j)
        if (tp.locs[j] == v) sa = j;
      if (sa < 0) continue;
      const double* T = tloc + (size_t)t * 25 + sa * 5;
      for (int b = 0; b < tp.nloc; ++b) {
        const int dj = m.v2d[tp.locs[b]];
        if (dj >= 0) Ar.add(dj, Cds * T[b]);
      }
    }
    // singular boundary pairs (cell K, edge e)
    if (bloc != nullptr) {
      for (int u = bp_off[K]; u < bp_off[K + 1]; ++u) {
        const int t = bp_idx[u];
        const BndPair& it = items[t];
        int sa = -1;
        for (int j = 0; j < it.nloc; ++j)
          if (it.locs[j] == v) sa = j;
        if (sa < 0) continue;
        for (int b = 0; b < it.nloc; ++b) {
          const int dj = m.v2d[it.locs[b]];
          if (dj >= 0) Ar.add(dj, cb * bloc[(size_t)t * 9 + sa * 3 + b]);
        }
      }
    }
  }
}

void launch_sparse_pull(const DevMesh& m, double Cds, double s, const double* Lc, const TouchPair* pairs,
                        const double* tloc, const BndPair* items, const double* bloc, const SparseIndex& si,
                        const int* row_vertex, int row_begin, int row_end, double* A, int64_t lda,
                        cudaStream_t st) {
  const int rows = row_end - row_begin;
  if (rows <= 0) return;
  const int grid = (rows + 127) / 128;
  const double cb = Cds / (2.0 * s);
  const DenseRows R{A, lda, row_begin};
  if (m.d == 1)
    sparse_pull_kernel<1><<<grid, 128, 0, st>>>(m, Cds, cb, Lc, pairs, tloc, items, bloc, si.tp_first_off.p,
                                                si.tp_second_off.p, si.tp_second.p, si.bp_off.p, si.bp_idx.p,
                                                row_vertex, row_begin, row_end, R), ::fl::note_launch();
  else
    sparse_pull_kernel<2><<<grid, 128, 0, st>>>(m, Cds, cb, Lc, pairs, tloc, items, bloc, si.tp_first_off.p,
                                                si.tp_second_off.p, si.tp_second.p, si.bp_off.p, si.bp_idx.p,
                                                row_vertex, row_begin, row_end, R), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

void launch_sparse_pull_csr(const DevMesh& m, double Cds, double s, const double* Lc, const TouchPair* pairs,
                            const double* tloc, const BndPair* items, const double* bloc, const SparseIndex& si,
                            const int* row_vertex, int nrows, const int64_t* indptr, const int* indices,
                            double* data, cudaStream_t st) {
  if (nrows <= 0) return;
  const int grid = (nrows + 127) / 128;
  const double cb = Cds / (2.0 * s);
  const CsrRows R{indptr, indices, data};
  if (m.d == 1)
    sparse_pull_kernel<1><<<grid, 128, 0, st>>>(m, Cds, cb, Lc, pairs, tloc, items, bloc, si.tp_first_off.p,
                                                si.tp_second_off.p, si.tp_second.p, si.bp_off.p, si.bp_idx.p,
                                                row_vertex, 0, nrows, R), ::fl::note_launch();
  else
    sparse_pull_kernel<2><<<grid, 128, 0, st>>>(m, Cds, cb, Lc, pairs, tloc, items, bloc, si.tp_first_off.p,
                                                si.tp_second_off.p, si.tp_second.p, si.bp_off.p, si.bp_idx.p,
                                                row_vertex, 0, nrows, R), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

}  // namespace fl
