// Dense fp64 matvec (HBM-bound, 128-bit streaming loads, warp-shuffle row reduction) and the
// fused Jacobi-PCG of solve.pcg (solve.py:52-109).  All reductions use a fixed tree
// (fixed grid, fixed per-thread order, fixed shuffle pattern): results are bitwise
// reproducible.  The CG scalars live on the device; the host polls a `done` flag every few
// iterations, so the iteration count is exactly the reference's.
#include <cstdlib>

#include "fl_internal.h"

#ifndef FL_MV_U
#define FL_MV_U 4      // double2 loads per lane in flight per row and main-loop step
#endif

namespace fl {

// ----------------------------------------------------------------- matvec
// y[r] = sum_j A[r, j] x[j];  lda is a multiple of 32 doubles, columns >= n are zero.
template <int RPW>
__global__ void __launch_bounds__(256) matvec_kernel(const double* __restrict__ A, int64_t rows, int64_t ncol2,
                                                     int64_t lda, const double* __restrict__ x,
                                                     double* __restrict__ y, const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t r0 = warp * RPW;
  if (r0 >= rows) return;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const double2* a2[RPW];
  double acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int64_t row = min(r0 + r, rows - 1);
    a2[r] = reinterpret_cast<const double2*>(A + row * lda);
    acc[r] = 0.0;
  }
  constexpr int U = FL_MV_U;
  int64_t j = lane;
  for (; j + 32 * (U - 1) < ncol2; j += 32 * U) {
    double2 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x2 + j + 32 * u);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      double2 av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) av[u] = __ldcs(a2[r] + j + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) acc[r] = fma(av[u].y, xv[u].y, fma(av[u].x, xv[u].x, acc[r]));
    }
  }
  for (; j < ncol2; j += 32) {
    const double2 xv = __ldg(x2 + j);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const double2 av = __ldcs(a2[r] + j);
      acc[r] = fma(av.y, xv.y, fma(av.x, xv.x, acc[r]));
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const double s = warp_sum(acc[r]);
    if (lane == 0 && r0 + r < rows) y[r0 + r] = s;
  }
}

// One CTA (256 threads) per row: short rows (n ~ 8k) are split over 8 warps, so a matrix of a
// few hundred MB streams in many small, evenly sized pieces (fixed per-thread column sets and a
// fixed reduction tree: deterministic).
__global__ void __launch_bounds__(256) matvec_rowcta_kernel(const double* __restrict__ A, int64_t rows,
                                                            int64_t ncol2, int64_t lda, const double* __restrict__ x,
                                                            double* __restrict__ y, const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double2* a2 = reinterpret_cast<const double2*>(A + r * lda);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double acc = 0.0;
  int64_t j = threadIdx.x;
  for (; j + 256 * 3 < ncol2; j += 256 * 4) {
    double2 av[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { av[u] = __ldcs(a2 + j + 256 * u); xv[u] = __ldg(x2 + j + 256 * u); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = fma(av[u].y, xv[u].y, fma(av[u].x, xv[u].x, acc));
  }
  for (; j < ncol2; j += 256) {
    const double2 av = __ldcs(a2 + j), xv = __ldg(x2 + j);
    acc = fma(av.y, xv.y, fma(av.x, xv.x, acc));
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) y[r] = v;
  }
}

void launch_matvec_flag(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, double* y,
                        const int* done, cudaStream_t st) {
  if (rows <= 0) return;
  const int64_t ncol2 = (n + 1) / 2;
  static const int rpw_env = [] { const char* v = getenv("FL_MV_RPW"); return v ? atoi(v) : 0; }();
  // CTA per row: fastest at c2 (537 MB, 6.1 vs 5.1 TB/s) and c4 (2.2 GB); a warp per 4 rows for
  // very many rows (c5, 65k rows of 520 KB: 6.94 vs 6.80 TB/s)
  const int rpw = rpw_env ? rpw_env : (rows >= 148LL * 64 * 4 ? 4 : 8);
  if (rpw == 8) {      // (FL_MV_RPW=8: the CTA-per-row variant)
    matvec_rowcta_kernel<<<(unsigned)rows, 256, 0, st>>>(A, rows, ncol2, lda, x, y, done), ::fl::note_launch();
  } else if (rpw == 4) {
    const int64_t warps = (rows + 3) / 4;
    const int grid = (int)((warps * 32 + 255) / 256);
    matvec_kernel<4><<<grid, 256, 0, st>>>(A, rows, ncol2, lda, x, y, done), ::fl::note_launch();
  } else if (rpw == 2) {
    const int64_t warps = (rows + 1) / 2;
    const int grid = (int)((warps * 32 + 255) / 256);
    matvec_kernel<2><<<grid, 256, 0, st>>>(A, rows, ncol2, lda, x, y, done), ::fl::note_launch();
  } else {
    const int64_t warps = rows;
    const int grid = (int)((warps * 32 + 255) / 256);
    matvec_kernel<1><<<grid, 256, 0, st>>>(A, rows, ncol2, lda, x, y, done), ::fl::note_launch();
  }
  FL_CHECK_LAUNCH();
}

void launch_matvec(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, double* y,
                   cudaStream_t st) {
  launch_matvec_flag(A, rows, n, lda, x, y, nullptr, st);
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

// ----------------------------------------------------------------- reductions
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = 0.0;
  if (w == 0) {
    t = (lane < nw) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) dot_partial_kernel(int64_t m, const double* __restrict__ a,
                                                          const double* __restrict__ b, double* part,
                                                          const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void __launch_bounds__(256) sum_final_kernel(const double* part, int np, double* out,
                                                        const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

void launch_dot_flag(int64_t m, const double* a, const double* b, double* out, double* scratch, const int* done,
                     cudaStream_t st) {
  dot_partial_kernel<<<DOT_BLOCKS, 256, 0, st>>>(m, a, b, scratch, done), ::fl::note_launch();
  sum_final_kernel<<<1, 256, 0, st>>>(scratch, DOT_BLOCKS, out, done), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}
void launch_dot(int64_t m, const double* a, const double* b, double* out, double* scratch, cudaStream_t st) {
  launch_dot_flag(m, a, b, out, scratch, nullptr, st);
}

// x += alpha p; r -= alpha Ap; z = minv r; partial r.z
__global__ void __launch_bounds__(256) cg_update_kernel(int64_t m, double alpha_h, const double* alpha_dev,
                                                        double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ z, const double* __restrict__ p,
                                                        const double* __restrict__ Ap,
                                                        const double* __restrict__ minv, double* part,
                                                        const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  const double alpha = alpha_dev ? *alpha_dev : alpha_h;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    const double zi = minv[i] * ri;
    z[i] = zi;
    s = fma(ri, zi, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void launch_cg_update_flag(int64_t m, double alpha, const double* alpha_dev, double* x, double* r, double* z,
                           const double* p, const double* Ap, const double* minv, double* out, double* scratch,
                           const int* done, cudaStream_t st) {
  cg_update_kernel<<<DOT_BLOCKS, 256, 0, st>>>(m, alpha, alpha_dev, x, r, z, p, Ap, minv, scratch, done), ::fl::note_launch();
  sum_final_kernel<<<1, 256, 0, st>>>(scratch, DOT_BLOCKS, out, done), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}
void launch_cg_update(int64_t m, double alpha, const double* alpha_dev, double* x, double* r, double* z,
                      const double* p, const double* Ap, const double* minv, double* out, double* scratch,
                      cudaStream_t st) {
  launch_cg_update_flag(m, alpha, alpha_dev, x, r, z, p, Ap, minv, out, scratch, nullptr, st);
}

__global__ void xpby_kernel(int64_t m, const double* __restrict__ z, double beta_h, const double* beta_dev,
                            double* __restrict__ p, const int* __restrict__ done) {
  if (done != nullptr && *done) return;
  const double beta = beta_dev ? *beta_dev : beta_h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
void launch_xpby_flag(int64_t m, const double* z, double beta, const double* beta_dev, double* p, const int* done,
                      cudaStream_t st) {
  xpby_kernel<<<DOT_BLOCKS, 256, 0, st>>>(m, z, beta, beta_dev, p, done), ::fl::note_launch();
  FL_CHECK_LAUNCH();
}
void launch_xpby(int64_t m, const double* z, double beta, const double* beta_dev, double* p, cudaStream_t st) {
  launch_xpby_flag(m, z, beta, beta_dev, p, nullptr, st);
}

__global__ void sub_kernel(int64_t m, double* __restrict__ r, const double* __restrict__ Ap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    r[i] -= Ap[i];
}
// z = minv r; p = z; partial r.z
__global__ void __launch_bounds__(256) precond_kernel(int64_t m, const double* __restrict__ r,
                                                      const double* __restrict__ minv, double* __restrict__ z,
                                                      double* __restrict__ p, double* part) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = minv[i] * r[i];
    z[i] = zi;
    p[i] = zi;
    s = fma(r[i], zi, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ----------------------------------------------------------------- device-side PCG control
struct CgScalars {
  double rz, rz_new, pAp, alpha, beta, norm0, tol;
  long long it, max_iter;
  int done, error, converged, pad;
};

__global__ void cg_alpha_kernel(CgScalars* sc, int* done) {
  if (*done) return;
  if (!(sc->pAp > 0.0)) {            // pAp <= 0 (or NaN): SolverError (solve.py:87-88)
    sc->error = 1;
    *done = 1;
    sc->done = 1;
    return;
  }
  sc->alpha = sc->rz / sc->pAp;
}
__global__ void cg_beta_kernel(CgScalars* sc, int* done) {
  if (*done) return;
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

// Single-device Jacobi PCG on a whole matrix (n x n, leading dim lda).  Vectors are device
// buffers of length >= lda (zero padded).  Returns iterations etc. in the host report.
PcgResult run_pcg(const double* A, int64_t n, int64_t lda, const double* minv, double* x, double* r, double* z,
                  double* p, double* Ap, double tol, long long max_iter, bool have_x0, cudaStream_t st) {
  DBuf<double> scratch(DOT_BLOCKS);
  DBuf<CgScalars> sc(1);
  DBuf<int> done(1);
  CgScalars h{};
  h.tol = tol;
  h.max_iter = max_iter;
  FL_CUDA(cudaMemsetAsync(done.p, 0, sizeof(int), st));
  // r = b - A x0 (b is passed in r) (solve.py:74), z = minv r, p = z, rz = r.z (:75-77)
  if (have_x0) {
    launch_matvec(A, n, n, lda, x, Ap, st);
    sub_kernel<<<DOT_BLOCKS, 256, 0, st>>>(n, r, Ap), ::fl::note_launch();
  }
  precond_kernel<<<DOT_BLOCKS, 256, 0, st>>>(n, r, minv, z, p, scratch.p), ::fl::note_launch();
  sum_final_kernel<<<1, 256, 0, st>>>(scratch.p, DOT_BLOCKS, &sc.p->rz, nullptr), ::fl::note_launch();
  FL_CHECK_LAUNCH();
  double rz0 = 0.0;
  FL_CUDA(cudaMemcpyAsync(&rz0, &sc.p->rz, sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  PcgResult res{0, rz0, std::sqrt(std::fabs(rz0)), 0, 0};
  if (res.norm0 == 0.0) return res;
  h.rz = rz0;
  h.norm0 = res.norm0;
  FL_CUDA(cudaMemcpyAsync(sc.p, &h, sizeof(CgScalars), cudaMemcpyHostToDevice, st));
  if (max_iter <= 0) return res;
  // one CG iteration = matvec, dot, alpha, update(+dot), beta, xpby; captured as a graph of CHK
  constexpr int CHK = 8;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cs;
  FL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  FL_CUDA(cudaStreamSynchronize(st));
  const long long before = launch_counter();
  FL_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < CHK; ++k) {
    launch_matvec_flag(A, n, n, lda, p, Ap, done.p, cs);
    launch_dot_flag(n, p, Ap, &sc.p->pAp, scratch.p, done.p, cs);
    cg_alpha_kernel<<<1, 1, 0, cs>>>(sc.p, done.p), ::fl::note_launch();
    launch_cg_update_flag(n, 0.0, &sc.p->alpha, x, r, z, p, Ap, minv, &sc.p->rz_new, scratch.p, done.p, cs);
    cg_beta_kernel<<<1, 1, 0, cs>>>(sc.p, done.p), ::fl::note_launch();
    launch_xpby_flag(n, z, 0.0, &sc.p->beta, p, done.p, cs);
  }
  FL_CUDA(cudaStreamEndCapture(cs, &graph));
  FL_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  const long long per_graph = launch_counter() - before;   // kernels per replay
  launch_counter() = before;
  for (long long launched = 0;; launched += CHK) {
    FL_CUDA(cudaGraphLaunch(exec, cs));
    note_launch(per_graph);
    FL_CUDA(cudaMemcpyAsync(&h, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, cs));
    FL_CUDA(cudaStreamSynchronize(cs));
    if (h.done) break;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  res.it = h.it;
  res.rz = h.rz;
  res.converged = h.converged;
  res.error = h.error;
  return res;
}

}  // namespace fl
