// Dense fp64 matvec (HBM-bound, 128-bit streaming loads) and the Jacobi-PCG of solve.pcg
// (solve.py:52-109) with the scalars on the device.
//
// Partition-independent reductions.  Every reduction of the solve is defined over FIXED GLOBAL
// CHUNKS of VCH = 512 entries, so its result does not depend on how the rows are split over
// GPUs (row blocks are multiples of VCH) nor on which kernel variant computed it:
//   * a matvec row y_r = fold_c S_c(r), S_c(r) = xor-butterfly over the 32 lanes of the lane's
//     sequential FMA chain over its 8 double2 of chunk c; fold = sequential left-to-right sum;
//   * a dot product = fold_c P_c, P_c = fixed block tree over the chunk's 512 products.
// A rank computes S_c / P_c for its own chunks; the partial sums of all ranks are gathered and
// every rank folds them in the same global order, so 1, 2, 4 or 8 GPUs give bitwise the same
// CG iterates, and the row-block matvec equals the rows of the whole-matrix matvec bitwise.
// The host polls a `done` flag every few iterations; kernels after convergence are no-ops.
#include <cstdlib>

#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

namespace fl {

// ----------------------------------------------------------------- chunked matvec
// lane l of the warp: S_c partial = sum_{u<8} A[row, c*512 + 2(l + 32u) + {0,1}] x[...]
__device__ __forceinline__ double chunk_lane(const double2* __restrict__ a2, const double2* __restrict__ x2,
                                             int64_t c, int64_t ncol2, int lane) {
  const int64_t j0 = c * (VCH / 2) + lane;
  double2 av[8], xv[8];
  if (j0 + 32 * 7 < ncol2) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      av[u] = __ldcs(a2 + j0 + 32 * u);
      xv[u] = __ldg(x2 + j0 + 32 * u);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool in = j0 + 32 * u < ncol2;
      av[u] = in ? __ldcs(a2 + j0 + 32 * u) : make_double2(0.0, 0.0);
      xv[u] = in ? __ldg(x2 + j0 + 32 * u) : make_double2(0.0, 0.0);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) acc = fma(av[u].y, xv[u].y, fma(av[u].x, xv[u].x, acc));
  return acc;
}

// MODE 0: y = A x over all chunks.  MODE 1: part[row, c - c_lo] = S_c for c in [c_lo, c_hi),
// x addressed from chunk c_lo (the rank's own slice of the vector).  MODE 2: y = fold over all
// chunks, S_c of [c_lo, c_hi) taken from part (written by MODE 1).
struct MvArgs {
  const double* A;
  int64_t rows, ncol2, lda;
  const double* x;     // MODE 0/2: the whole vector (>= 2*ncol2 entries); MODE 1: from column c_lo*VCH
  double* y;
  double* part;
  int64_t c_lo, c_hi, nch;
  const int* done;
};

// warp per RPW rows (many rows)
template <int RPW, int MODE>
__global__ void __launch_bounds__(256) mv_rows_kernel(MvArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t r0 = warp * RPW;
  if (r0 >= a.rows) return;
  const double2* a2[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) a2[r] = reinterpret_cast<const double2*>(a.A + min(r0 + r, a.rows - 1) * a.lda);
  const double2* x2 = reinterpret_cast<const double2*>(a.x);
  const int64_t nw = a.c_hi - a.c_lo;
  if constexpr (MODE == 1) {
    const double2* xl = x2 - a.c_lo * (VCH / 2);
    for (int64_t c = a.c_lo; c < a.c_hi; ++c)
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const double s = warp_sum(chunk_lane(a2[r], xl, c, a.ncol2, lane));
        if (lane == 0 && r0 + r < a.rows) a.part[(r0 + r) * nw + (c - a.c_lo)] = s;
      }
  } else {
  double t[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) t[r] = 0.0;
  for (int64_t c = 0; c < a.nch; ++c) {
    if (MODE == 2 && c >= a.c_lo && c < a.c_hi) {
#pragma unroll
      for (int r = 0; r < RPW; ++r) t[r] += a.part[min(r0 + r, a.rows - 1) * nw + (c - a.c_lo)];
      continue;
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) t[r] += warp_sum(chunk_lane(a2[r], x2, c, a.ncol2, lane));
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
    if (lane == 0 && r0 + r < a.rows) a.y[r0 + r] = t[r];
  }
}

// one CTA (8 warps) per row (up to ~40k rows): warp w computes the chunks c = w (mod 8), the
// S_c land in shared memory and thread 0 folds them in chunk order — the same numbers as above
constexpr int MV_CTA_MAXCH = 4096;
template <int MODE>
__global__ void __launch_bounds__(256) mv_cta_kernel(MvArgs a) {
  if (a.done != nullptr && *a.done) return;
  extern __shared__ double sS[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row = blockIdx.x;
  const double2* a2 = reinterpret_cast<const double2*>(a.A + row * a.lda);
  const double2* x2 = reinterpret_cast<const double2*>(a.x);
  const int64_t nw = a.c_hi - a.c_lo;
  if constexpr (MODE == 1) {
    const double2* xl = x2 - a.c_lo * (VCH / 2);
    for (int64_t c = a.c_lo + w; c < a.c_hi; c += 8) {
      const double s = warp_sum(chunk_lane(a2, xl, c, a.ncol2, lane));
      if (lane == 0) a.part[row * nw + (c - a.c_lo)] = s;
    }
  } else {
  for (int64_t c = w; c < a.nch; c += 8) {
    double s;
    if (MODE == 2 && c >= a.c_lo && c < a.c_hi) s = a.part[row * nw + (c - a.c_lo)];
    else s = warp_sum(chunk_lane(a2, x2, c, a.ncol2, lane));
    if (lane == 0) sS[c] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int64_t c = 0; c < a.nch; ++c) t += sS[c];
    a.y[row] = t;
  }
  }
}

static void launch_mv(int mode, const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, double* y,
                      double* part, int64_t c_lo, int64_t c_hi, const int* done, cudaStream_t st) {
  if (rows <= 0) return;
  MvArgs a{A, rows, (n + 1) / 2, lda, x, y, part, c_lo, c_hi, (n + VCH - 1) / VCH, done};
  static const int var_env = [] { const char* v = getenv("FL_MV_RPW"); return v ? atoi(v) : 0; }();
  // CTA per row: fastest at c2 (537 MB) and c4 (2.2 GB); a warp per 4 rows for very many rows
  // (c5: 65k rows of 520 KB)
  int rpw = var_env ? var_env : (rows >= 148LL * 64 * 4 ? 4 : 8);
  if (a.nch > MV_CTA_MAXCH && rpw == 8) rpw = 4;
  if (rpw == 8) {
    const size_t sm = (size_t)a.nch * sizeof(double);
    if (mode == 0) mv_cta_kernel<0><<<(unsigned)rows, 256, sm, st>>>(a);
    else if (mode == 1) mv_cta_kernel<1><<<(unsigned)rows, 256, 0, st>>>(a);
    else mv_cta_kernel<2><<<(unsigned)rows, 256, sm, st>>>(a);
  } else {
    const int R = rpw >= 4 ? 4 : (rpw >= 2 ? 2 : 1);
    const int64_t warps = (rows + R - 1) / R;
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
#define FL_MV_LAUNCH(RR)                                                   \
    if (mode == 0) mv_rows_kernel<RR, 0><<<grid, 256, 0, st>>>(a);         \
    else if (mode == 1) mv_rows_kernel<RR, 1><<<grid, 256, 0, st>>>(a);    \
    else mv_rows_kernel<RR, 2><<<grid, 256, 0, st>>>(a);
    if (R == 4) { FL_MV_LAUNCH(4) } else if (R == 2) { FL_MV_LAUNCH(2) } else { FL_MV_LAUNCH(1) }
#undef FL_MV_LAUNCH
  }
  note_launch();
  FL_CHECK_LAUNCH();
}

void launch_matvec(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, double* y,
                   cudaStream_t st) {
  launch_mv(0, A, rows, n, lda, x, y, nullptr, 0, 0, nullptr, st);
}

__global__ void diag_kernel(const double* A, int64_t rows, int64_t row0, int64_t lda, double* d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) d[i] = A[i * lda + row0 + i];
}
void launch_diag(const double* A, int64_t rows, int64_t row0, int64_t lda, double* d, cudaStream_t st) {
  if (rows <= 0) return;
  diag_kernel<<<(int)((rows + 255) / 256), 256, 0, st>>>(A, rows, row0, lda, d), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}

// ----------------------------------------------------------------- chunked vector kernels
// One 256-thread block per chunk of VCH = 512 entries; thread t owns entries t and t + 256 of
// the chunk (fma in that order), then a fixed block tree.  part[c] = the chunk's sum.
__device__ __forceinline__ double chunk_block_sum(double v) {
  __shared__ double sh[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (lane < 8) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

__global__ void __launch_bounds__(256) dot_chunk_kernel(int64_t m, const double* __restrict__ a,
                                                        const double* __restrict__ b, double* __restrict__ part,
                                                        const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  const int64_t i0 = (int64_t)blockIdx.x * VCH + threadIdx.x, i1 = i0 + VCH / 2;
  double s = 0.0;
  if (i0 < m) s = fma(a[i0], b[i0], s);
  if (i1 < m) s = fma(a[i1], b[i1], s);
  s = chunk_block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// z = minv r; p = z; part = chunk sums of r.z
__global__ void __launch_bounds__(256) precond_chunk_kernel(int64_t m, const double* __restrict__ r,
                                                            const double* __restrict__ minv, double* __restrict__ z,
                                                            double* __restrict__ p, double* __restrict__ part) {
  const int64_t i0 = (int64_t)blockIdx.x * VCH + threadIdx.x;
  double s = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + h * (VCH / 2);
    if (i < m) {
      const double zi = minv[i] * r[i];
      z[i] = zi;
      p[i] = zi;
      s = fma(r[i], zi, s);
    }
  }
  s = chunk_block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// device CG scalars
struct CgScalars {
  double rz, rz_new, pAp, alpha, beta, norm0, tol;
  long long it, max_iter;
  int done, error, converged, pad;
};

// x += alpha p; r -= alpha Ap; z = minv r; part = chunk sums of r.z
__global__ void __launch_bounds__(256) update_chunk_kernel(int64_t m, const CgScalars* __restrict__ sc,
                                                           double* __restrict__ x, double* __restrict__ r,
                                                           double* __restrict__ z, const double* __restrict__ p,
                                                           const double* __restrict__ Ap,
                                                           const double* __restrict__ minv, double* __restrict__ part,
                                                           const int* __restrict__ done) {
  if (*done) return;
  const double alpha = sc->alpha;
  const int64_t i0 = (int64_t)blockIdx.x * VCH + threadIdx.x;
  double s = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + h * (VCH / 2);
    if (i < m) {
      x[i] += alpha * p[i];
      const double ri = r[i] - alpha * Ap[i];
      r[i] = ri;
      const double zi = minv[i] * ri;
      z[i] = zi;
      s = fma(ri, zi, s);
    }
  }
  s = chunk_block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void xpby_chunk_kernel(int64_t m, const double* __restrict__ z, const CgScalars* __restrict__ sc,
                                  double* __restrict__ p, const int* __restrict__ done) {
  if (*done) return;
  const double beta = sc->beta;
  const int64_t i0 = (int64_t)blockIdx.x * VCH + threadIdx.x;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + h * (VCH / 2);
    if (i < m) p[i] = z[i] + beta * p[i];
  }
}

__global__ void sub_kernel(int64_t m, double* __restrict__ r, const double* __restrict__ Ap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    r[i] -= Ap[i];
}

// Sequential fold of the gathered chunk sums in global chunk order: rank g's slot holds L
// entries of which its first ceil(rows_g / VCH) are real.
struct FoldGeom {
  int64_t n, blk, L;
  int world;
};
__device__ double fold_parts(const double* __restrict__ parts, FoldGeom g) {
  double t = 0.0;
  for (int k = 0; k < g.world; ++k) {
    const int64_t r0 = (int64_t)k * g.blk, r1 = min(g.n, r0 + g.blk);
    const int64_t cnt = r1 > r0 ? (r1 - r0 + VCH - 1) / VCH : 0;
    for (int64_t c = 0; c < cnt; ++c) t += parts[(int64_t)k * g.L + c];
  }
  return t;
}

__global__ void cg_init_kernel(CgScalars* sc, const double* parts, FoldGeom g, int* done) {
  const double rz = fold_parts(parts, g);
  sc->rz = rz;
  sc->norm0 = sqrt(fabs(rz));
  sc->it = 0;
  sc->error = 0;
  sc->converged = 0;
  sc->done = 0;
  *done = 0;
  if (sc->norm0 == 0.0 || sc->max_iter <= 0) {     // b = 0: x0 is the answer (solve.py:78-79)
    sc->converged = sc->norm0 == 0.0;
    sc->done = 1;
    *done = 1;
  }
}
__global__ void cg_alpha_kernel(CgScalars* sc, const double* parts, FoldGeom g, int* done) {
  if (*done) return;
  sc->pAp = fold_parts(parts, g);
  if (!(sc->pAp > 0.0)) {            // pAp <= 0 (or NaN): SolverError (solve.py:87-88)
    sc->error = 1;
    *done = 1;
    sc->done = 1;
    return;
  }
  sc->alpha = sc->rz / sc->pAp;
}
__global__ void cg_beta_kernel(CgScalars* sc, const double* parts, FoldGeom g, int* done) {
  if (*done) return;
  sc->rz_new = fold_parts(parts, g);
  sc->it += 1;
  if (sqrt(fabs(sc->rz_new)) <= sc->tol * sc->norm0) {   // solve.py:96
    sc->converged = 1;
    sc->rz = sc->rz_new;
    *done = 1;
    sc->done = 1;
    return;
  }
  sc->beta = sc->rz_new / sc->rz;
  sc->rz = sc->rz_new;
  if (sc->it >= sc->max_iter) { *done = 1; sc->done = 1; }
}

}  // namespace fl

// ----------------------------------------------------------------- CG state (one rank)
struct fl_cg {
  int device = 0;
  int64_t n = 0, m = 0, blk = 0, L = 0, row0 = 0;
  int world = 1;
  fl::DBuf<fl::CgScalars> sc;
  fl::DBuf<int> done;
  fl::DBuf<double> local, all;       // chunk sums: this rank's (L) and all ranks' (world * L)
  fl::DBuf<double> dpart;            // diagonal-block chunk sums of the split matvec (m x chunks)
  int64_t dch = 0;
  double* ext = nullptr;             // caller-owned buffer for this rank's chunk sums (fl_cg_bind_parts)
  double* lp() const { return ext ? ext : local.p; }
  fl::FoldGeom geom() const { return fl::FoldGeom{n, blk, L, world}; }
  int64_t nloc() const { return (m + fl::VCH - 1) / fl::VCH; }
};

namespace fl {

fl_cg* cg_create(int64_t n, int64_t m, int64_t blk, int world, int rank, double tol, long long max_iter,
                 int device) {
  if (n <= 0 || m < 0 || world < 1 || rank < 0 || rank >= world || blk <= 0 || blk % VCH != 0 ||
      (int64_t)world * blk < n || m > blk)
    throw Error(-1, "bad CG geometry (row blocks must be equal multiples of 512 rows)");
  auto* S = new fl_cg();
  S->device = device;
  S->n = n;
  S->m = m;
  S->blk = blk;
  S->L = blk / VCH;
  S->world = world;
  S->row0 = std::min<int64_t>((int64_t)rank * blk, n);   // (an empty block sits at n)
  S->sc.alloc(1);
  S->done.alloc(1);
  S->local.alloc(S->L);
  S->all.alloc((size_t)S->L * world);
  // chunks of the diagonal block: [row0 / VCH, ceil(min(row0 + m, n) / VCH))
  S->dch = (m + VCH - 1) / VCH;
  if (world > 1 && m > 0) S->dpart.alloc((size_t)m * S->dch);
  CgScalars h{};
  h.tol = tol;
  h.max_iter = max_iter;
  cudaStream_t st = cur_stream();
  FL_CUDA(cudaMemcpyAsync(S->sc.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemsetAsync(S->done.p, 0, sizeof(int), st));
  FL_CUDA(cudaMemsetAsync(S->local.p, 0, S->L * sizeof(double), st));
  FL_CUDA(cudaMemsetAsync(S->all.p, 0, S->L * world * sizeof(double), st));
  return S;
}

static unsigned nblk(int64_t m) { return (unsigned)std::max<int64_t>(1, (m + VCH - 1) / VCH); }

void cg_begin(fl_cg* S, const double* r, const double* minv, double* z, double* p, cudaStream_t st) {
  if (S->m > 0) precond_chunk_kernel<<<nblk(S->m), 256, 0, st>>>(S->m, r, minv, z, p, S->lp()), note_launch();
  FL_CHECK_LAUNCH();
}
void cg_init(fl_cg* S, const double* parts, cudaStream_t st) {
  cg_init_kernel<<<1, 1, 0, st>>>(S->sc.p, parts, S->geom(), S->done.p), note_launch();
  FL_CHECK_LAUNCH();
}
// diagonal-block chunks of the rank's rows (x = this rank's slice of the vector)
void cg_matvec_diag(fl_cg* S, const double* A, int64_t lda, const double* x_local, cudaStream_t st) {
  if (S->world == 1 || S->m == 0) return;
  const int64_t c_lo = S->row0 / VCH;
  launch_mv(1, A, S->m, S->n, lda, x_local, nullptr, S->dpart.p, c_lo, c_lo + S->dch, S->done.p, st);
}
// the rest of the matvec (whole vector gathered) + chunk sums of p.Ap
void cg_matvec_rest(fl_cg* S, const double* A, int64_t lda, const double* x_full, const double* p_local,
                    double* Ap, cudaStream_t st) {
  if (S->m == 0) return;
  if (S->world == 1) {
    launch_mv(0, A, S->m, S->n, lda, x_full, Ap, nullptr, 0, 0, S->done.p, st);
  } else {
    const int64_t c_lo = S->row0 / VCH;
    launch_mv(2, A, S->m, S->n, lda, x_full, Ap, S->dpart.p, c_lo, c_lo + S->dch, S->done.p, st);
  }
  dot_chunk_kernel<<<nblk(S->m), 256, 0, st>>>(S->m, p_local, Ap, S->lp(), S->done.p), note_launch();
  FL_CHECK_LAUNCH();
}
void cg_dot_parts(fl_cg* S, const double* a, const double* b, cudaStream_t st) {
  if (S->m == 0) return;
  dot_chunk_kernel<<<nblk(S->m), 256, 0, st>>>(S->m, a, b, S->lp(), S->done.p), note_launch();
  FL_CHECK_LAUNCH();
}
void cg_alpha_update(fl_cg* S, const double* parts, double* x, double* r, double* z, const double* p,
                     const double* Ap, const double* minv, cudaStream_t st) {
  cg_alpha_kernel<<<1, 1, 0, st>>>(S->sc.p, parts, S->geom(), S->done.p), note_launch();
  if (S->m > 0)
    update_chunk_kernel<<<nblk(S->m), 256, 0, st>>>(S->m, S->sc.p, x, r, z, p, Ap, minv, S->lp(), S->done.p),
        note_launch();
  FL_CHECK_LAUNCH();
}
void cg_beta_xpby(fl_cg* S, const double* parts, const double* z, double* p, cudaStream_t st) {
  cg_beta_kernel<<<1, 1, 0, st>>>(S->sc.p, parts, S->geom(), S->done.p), note_launch();
  if (S->m > 0) xpby_chunk_kernel<<<nblk(S->m), 256, 0, st>>>(S->m, z, S->sc.p, p, S->done.p), note_launch();
  FL_CHECK_LAUNCH();
}
void cg_status(fl_cg* S, fl_cg_status* out, cudaStream_t st) {
  CgScalars h{};
  FL_CUDA(cudaMemcpyAsync(&h, S->sc.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  out->iterations = h.it;
  out->rz = h.rz;
  out->norm0 = h.norm0;
  out->done = h.done;
  out->converged = h.converged;
  out->error = h.error;
  out->pad_ = 0;
}
double* cg_local_parts(fl_cg* S) { return S->lp(); }
void cg_bind_parts(fl_cg* S, double* ext) { S->ext = ext; }
double* cg_all_parts(fl_cg* S) { return S->all.p; }
int64_t cg_chunks(fl_cg* S) { return S->L; }
void cg_free(fl_cg* S) { delete S; }
int cg_device(const fl_cg* S) { return S->device; }
void cg_info(const fl_cg* S, int* device, int64_t* n, int64_t* row0, int64_t* m) {
  *device = S->device;
  *n = S->n;
  *row0 = S->row0;
  *m = S->m;
}

// Single-device Jacobi PCG on a whole matrix (n x n, leading dim lda): the world-1 instance of
// the sharded solver above (same kernels, same fold), CHK iterations per CUDA graph replay.
// Vectors are device buffers of length >= the 512-rounded n (zero padded).
PcgResult run_pcg(const double* A, int64_t n, int64_t lda, const double* minv, double* x, double* r, double* z,
                  double* p, double* Ap, double tol, long long max_iter, bool have_x0, cudaStream_t st) {
  const int64_t blk = (n + VCH - 1) / VCH * VCH;
  fl_cg* S = nullptr;
  {
    StreamScope scope(st);
    S = cg_create(n, n, blk, 1, 0, tol, max_iter, -1);
  }
  struct Del { fl_cg* s; ~Del() { delete s; } } del{S};
  // r = b - A x0 (b is passed in r) (solve.py:74), z = minv r, p = z, rz = r.z (:75-77)
  if (have_x0) {
    launch_matvec(A, n, n, lda, x, Ap, st);
    sub_kernel<<<DOT_BLOCKS, 256, 0, st>>>(n, r, Ap), ::fl::note_launch();
  }
  cg_begin(S, r, minv, z, p, st);
  cg_init(S, S->local.p, st);
  fl_cg_status h{};
  cg_status(S, &h, st);
  PcgResult res{0, h.rz, h.norm0, h.converged, 0};
  if (h.done) return res;
  // one CG iteration = matvec + dot, alpha + update(+dot), beta + xpby; CHK per graph
  constexpr int CHK = 8;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cs;
  FL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const long long before = launch_counter();
  FL_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < CHK; ++k) {
    cg_matvec_rest(S, A, lda, p, p, Ap, cs);
    cg_alpha_update(S, S->local.p, x, r, z, p, Ap, minv, cs);
    cg_beta_xpby(S, S->local.p, z, p, cs);
  }
  FL_CUDA(cudaStreamEndCapture(cs, &graph));
  FL_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  const long long per_graph = launch_counter() - before;   // kernels per replay
  launch_counter() = before;
  for (;;) {
    FL_CUDA(cudaGraphLaunch(exec, cs));
    note_launch(per_graph);
    cg_status(S, &h, cs);
    if (h.done) break;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  res.it = h.iterations;
  res.rz = h.rz;
  res.converged = h.converged;
  res.error = h.error;
  return res;
}

}  // namespace fl
