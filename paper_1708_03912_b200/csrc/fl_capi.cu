// C ABI of fraclap_b200 (include/fraclap_b200.h): argument checks with the reference's error
// semantics, host->device upload of the borrowed mesh arrays, and the orchestration of the
// assembly phases of assemble_dense (assembly.py:1059-1104) on one stream.
#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/fraclap_b200.h"
#include "fl_internal.h"

using namespace fl;

namespace fl {
long long& launch_counter() {
  static long long c = 0;
  return c;
}
cudaStream_t& cur_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
void init_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;   // keep freed blocks cached: repeated assemblies reuse them
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}
}  // namespace fl

namespace fl {
// Recycled non-blocking streams per device (an operator's own stream, the side stream of an
// assembly): creating a stream costs more than the small phases of a 1D assembly.
std::mutex g_stream_mu;
std::map<int, std::vector<cudaStream_t>> g_stream_pool;
cudaStream_t acquire_stream(int device) {
  {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    auto& v = g_stream_pool[device];
    if (!v.empty()) {
      cudaStream_t s = v.back();
      v.pop_back();
      return s;
    }
  }
  cudaStream_t s = nullptr;
  FL_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}
void release_stream(int device, cudaStream_t s) {   // pending stream-ordered work stays ordered
  if (!s) return;
  std::lock_guard<std::mutex> lk(g_stream_mu);
  g_stream_pool[device].push_back(s);
}
}  // namespace fl

struct fl_dense {
  int device = 0;
  int64_t n = 0, row0 = 0, row1 = 0, lda = 0;
  DBuf<double> A;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  fl_assembly_stats stats{};
  ~fl_dense() {
    A.free();
    if (own_stream && stream) fl::release_stream(device, stream);
  }
};

struct fl_sparse {                     // CSR (n x n), int64 row pointers, int32 column indices
  int device = 0;
  int64_t n = 0, nnz = 0, pairs = 0;
  DBuf<int64_t> indptr;
  DBuf<int> indices;
  DBuf<double> data;
  cudaStream_t stream = nullptr;
  ~fl_sparse() {
    indptr.free();
    indices.free();
    data.free();
    if (stream) fl::release_stream(device, stream);
  }
};

static thread_local std::string g_err;

static int32_t fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace fl {
int32_t api_fail(int code, const char* msg) { return fail(code, msg ? msg : ""); }
}  // namespace fl

#define FL_API_BEGIN try {
#define FL_API_END                                              \
  }                                                             \
  catch (const Error& e) { return fail(e.code, e.what()); }     \
  catch (const std::bad_alloc&) { return fail(FL_E_OOM, "host allocation failed"); } \
  catch (const std::exception& e) { return fail(FL_E_CUDA, e.what()); }

extern "C" {

int32_t fl_abi_version(void) { return FL_ABI_VERSION; }
int64_t fl_launch_count(void) { return launch_counter(); }
const char* fl_last_error(void) { return g_err.c_str(); }
int32_t fl_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

}  // extern "C"

namespace {

int e4_of(int d, double s) {
  // e = d + 2s; specialised for s in {1/4, 1/2, 3/4}
  const double e = d + 2.0 * s;
  const double e4 = 4.0 * e;
  if (std::fabs(e4 - std::round(e4)) == 0.0 && (s == 0.25 || s == 0.5 || s == 0.75)) return (int)std::lround(e4);
  return 0;
}

OrderConsts make_order_consts(const fl_order_params& p, int d, double s, int64_t n) {
  OrderConsts oc{};
  const double ln_n = std::log(std::max((double)n, 2.0));          // quadrature.py:145
  oc.lead_lnn = (p.alpha / 2 + 0.5) * ln_n;                         // :149
  oc.lead_lnn_b = (p.alpha / 2 + 0.25) * ln_n;
  oc.s = s;
  oc.sm1 = s - 1;
  oc.ln_rho1 = std::log(p.rho1);
  oc.ln_rho2 = std::log(p.rho2);
  oc.ln_rho3 = std::log(p.rho3);
  oc.coff = p.C_offset;
  oc.coff_tail = p.C_offset - 4;                                    // assembly.py:985, :997
  oc.cap_disjoint = (d == 2) ? 9 : KMAX;                            // quadrature.py:171-175
  oc.lead_f = (float)oc.lead_lnn;
  oc.s_f = (float)oc.s;
  oc.sm1_f = (float)oc.sm1;
  oc.lr2_f = (float)oc.ln_rho2;
  oc.coff_f = (float)oc.coff;
  oc.coff_tail_f = (float)oc.coff_tail;
  return oc;
}

void check_inputs(const fl_mesh* mesh, const fl_dofmap* dm, const fl_kernel* k, const fl_order_params* p,
                  const fl_tables* t) {
  if (!mesh || !dm || !k || !p || !t) throw Error(FL_E_ARG, "null argument");
  if (mesh->d != 1 && mesh->d != 2) throw Error(FL_E_ARG, "mesh dimension must be 1 or 2");
  if (k->d != mesh->d) throw Error(FL_E_ARG, "kernel dimension does not match the mesh");
  if (!(k->s > 0.0 && k->s < 1.0)) throw Error(FL_E_ARG, "s must lie in (0,1)");   // assembly.py:59-60
  if (std::min(std::min(p->rho1, p->rho2), std::min(p->rho3, p->rho4)) <= 1)
    throw Error(FL_E_ARG, "all rho parameters must exceed 1");                      // quadrature.py:125-126
  if (mesh->nv <= 0 || mesh->nc <= 0 || mesh->nv >= (1LL << 31) || mesh->nc >= (1LL << 28))
    throw Error(FL_E_ARG, "mesh size out of range");
  if (!mesh->vertices || !mesh->cells || (mesh->nb > 0 && (!mesh->boundary_edges || !mesh->boundary_normals)))
    throw Error(FL_E_ARG, "missing mesh arrays");
  if (!dm->vertex_to_dof || dm->n < 0) throw Error(FL_E_ARG, "bad dofmap");
  if (!t->dir || !t->data || t->ndata <= 0) throw Error(FL_E_ARG, "missing quadrature tables");
}

// grow-only pinned staging area per host thread (one H2D copy per assembly); the copy has
// completed before the next call on this thread reuses it (every call synchronises its stream)
unsigned char* pinned_stage(size_t bytes) {
  thread_local void* p = nullptr;
  thread_local size_t cap = 0;
  if (cap < bytes) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = bytes + bytes / 4 + 4096;
    FL_CUDA(cudaHostAlloc(&p, want, cudaHostAllocDefault));
    cap = want;
  }
  return static_cast<unsigned char*>(p);
}

struct Uploaded {
  DBuf<unsigned char> blob;           // vertices | normals | tables | cells | v2d | edges
  DBuf<double> X, W;
  DBuf<int> patch_off, patch_cells, err, maxv;
  DBuf<CellGeo> geo;
  DevMesh m;
  DevTables t;
};

void upload(const fl_mesh* mesh, const fl_dofmap* dm, const fl_tables* tb, Uploaded& U, cudaStream_t st) {
  const int d = mesh->d;
  const int64_t nv = mesh->nv, nc = mesh->nc, nb = mesh->nb;
  // everything goes up in ONE copy from a pinned staging area: doubles first (vertices,
  // boundary normals, quadrature tables), then the int32 index arrays (cells, vertex->DoF,
  // boundary edges)
  const size_t n_vert = (size_t)nv * d, n_bn = (size_t)std::max<int64_t>(nb, 1) * d, n_tab = (size_t)tb->ndata;
  const size_t n_cells = (size_t)nc * (d + 1), n_v2d = (size_t)nv, n_be = (size_t)std::max<int64_t>(nb, 1) * d;
  const size_t dbytes = 8 * (n_vert + n_bn + n_tab), ibytes = 4 * (n_cells + n_v2d + n_be);
  unsigned char* stage = pinned_stage(dbytes + ibytes);
  double* hvert = reinterpret_cast<double*>(stage);
  double* hbn = hvert + n_vert;
  double* htab = hbn + n_bn;
  int* hc = reinterpret_cast<int*>(stage + dbytes);
  int* hv2d = hc + n_cells;
  int* hbe = hv2d + n_v2d;
  std::memcpy(hvert, mesh->vertices, n_vert * sizeof(double));
  if (nb > 0) std::memcpy(hbn, mesh->boundary_normals, (size_t)nb * d * sizeof(double));
  else std::fill(hbn, hbn + n_bn, 0.0);
  std::memcpy(htab, tb->data, n_tab * sizeof(double));
  for (size_t i = 0; i < n_cells; ++i) {
    const int64_t c = mesh->cells[i];
    if (c < 0 || c >= nv) throw Error(FL_E_ARG, "cell vertex index out of range");
    hc[i] = (int)c;
  }
  int64_t maxdof = -1;
  for (int64_t v = 0; v < nv; ++v) {
    hv2d[v] = (int)dm->vertex_to_dof[v];
    maxdof = std::max<int64_t>(maxdof, dm->vertex_to_dof[v]);
  }
  if (maxdof + 1 != dm->n) throw Error(FL_E_ARG, "dofmap.n does not match vertex_to_dof");
  for (size_t i = 0; i < n_be; ++i) hbe[i] = i < (size_t)nb * d ? (int)mesh->boundary_edges[i] : 0;
  U.blob.alloc(dbytes + ibytes);
  FL_CUDA(cudaMemcpyAsync(U.blob.p, stage, dbytes + ibytes, cudaMemcpyHostToDevice, st));
  const double* dvert = reinterpret_cast<const double*>(U.blob.p);
  const double* dbn = dvert + n_vert;
  const double* dtab = dbn + n_bn;
  const int* dcells = reinterpret_cast<const int*>(U.blob.p + dbytes);
  const int* dv2d = dcells + n_cells;
  const int* dbe = dv2d + n_v2d;
  for (int i = 0; i < NTOPO * KDIR; ++i) {
    const int64_t off = tb->dir[2 * i], cnt = tb->dir[2 * i + 1];
    if (cnt < 0 || off < 0 || (off + cnt) * NODE > tb->ndata) throw Error(FL_E_ARG, "corrupt quadrature table");
    U.t.dir[i] = RuleRef{(int)off, (int)cnt};
  }
  U.t.data = dtab;
  if (U.t.rule(T_CELL, 0).cnt <= 0) throw Error(FL_E_ARG, "missing cell rule");
  DevMesh& m = U.m;
  m.d = d; m.nv = (int)nv; m.nc = (int)nc; m.nb = (int)nb; m.n = (int)dm->n;
  m.q = U.t.rule(T_CELL, 0).cnt;
  if (m.q != (d == 1 ? 6 : 16)) throw Error(FL_E_ARG, "cell rule must have 6 (1D) / 16 (2D) nodes (XQ_ORDER)");
  m.vert = dvert; m.cells = dcells; m.v2d = dv2d; m.bedges = dbe; m.bnorm = dbn;
  U.err.alloc(1);
  FL_CUDA(cudaMemsetAsync(U.err.p, 0, sizeof(int), st));
  m.err = U.err.p;
  build_patches((int)nv, (int)nc, d, dcells, U.patch_off, U.patch_cells, st);
  m.patch_off = U.patch_off.p;
  m.patch_cells = U.patch_cells.p;
  // max vertex valence on the device; checked (check_valence / the size read-back of
  // fl_assemble_dense) before anything that depends on it is used — every kernel guards its
  // valence-bounded lists, so a too-high valence fails loudly and never writes out of bounds
  U.maxv.alloc(1);
  FL_CUDA(cudaMemsetAsync(U.maxv.p, 0, sizeof(int), st));
  launch_max_valence(U.patch_off.p, (int)nv, U.maxv.p, st);
  U.geo.alloc(nc);
  launch_prep_cells(m, U.geo.p, st);
  m.geo = U.geo.p;
  U.X.alloc((size_t)nc * m.q * d);
  U.W.alloc((size_t)nc * m.q);
  launch_cell_nodes(m, U.t, U.X.p, U.W.p, st);
  m.X = U.X.p;
  m.W = U.W.p;
}

void valence_error(int mv) {
  if (mv > MAX_VALENCE)
    throw Error(FL_E_ASSEMBLY, "vertex valence " + std::to_string(mv) + " exceeds " + std::to_string(MAX_VALENCE));
}
void check_valence(const Uploaded& U, cudaStream_t st) {
  int mv = 0;
  FL_CUDA(cudaMemcpyAsync(&mv, U.maxv.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  valence_error(mv);
}

// small pinned read-back area per host thread (sizes read back together with one sync)
int* pinned_scratch() {
  thread_local int* hs = nullptr;
  if (!hs) FL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hs), 64 * sizeof(int), cudaHostAllocDefault));
  return hs;
}

__global__ void zero_pad_kernel(double* A, int64_t rows, int64_t n, int64_t lda) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, w = lda - n;
  if (i < rows * w) A[(i / w) * lda + n + i % w] = 0.0;
}

__global__ void flag_target_cells(DevMesh m, int r0, int r1, int* flags) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m.nc) return;
  int f = 0;
  for (int i = 0; i <= m.d; ++i) {
    const int dof = m.v2d[m.cells[c * (m.d + 1) + i]];
    f |= (dof >= r0 && dof < r1);
  }
  flags[c] = f;
}
// every cell into the target list of each row band holding one of its vertex DoFs (cut: band starts)
__global__ void band_targets_kernel(DevMesh m, const int* __restrict__ cut, int nbands, int* __restrict__ lists,
                                    int* __restrict__ cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m.nc) return;
  int seen[3] = {-1, -1, -1};
  for (int i = 0; i <= m.d; ++i) {
    const int dof = m.v2d[m.cells[c * (m.d + 1) + i]];
    if (dof < 0) continue;
    int a = 0, b = nbands;                       // the band of dof: cut[band] <= dof < cut[band + 1]
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (cut[mid] <= dof) a = mid; else b = mid;
    }
    bool dup = false;
    for (int j = 0; j < i; ++j) dup |= seen[j] == a;
    seen[i] = a;
    if (!dup) lists[(size_t)a * m.nc + atomicAdd(&cnt[a], 1)] = c;
  }
}
__global__ void iota2(int* a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
__global__ void dof_vertex2(DevMesh m, int* dv) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < m.nv && m.v2d[v] >= 0) dv[m.v2d[v]] = v;
}

struct OwnedStream {          // destroyed after every buffer declared later in the scope
  cudaStream_t s = nullptr;
  OwnedStream() { FL_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~OwnedStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

struct Timer {
  cudaEvent_t* e;                      // per host thread and device, created once (calls are synchronous)
  int k = 0;
  cudaStream_t st;
  explicit Timer(cudaStream_t s) : st(s) {
    thread_local std::map<int, std::vector<cudaEvent_t>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    auto& v = cache[dev];
    if (v.empty()) {
      v.resize(12);
      for (auto& x : v) cudaEventCreate(&x);
    }
    e = v.data();
  }
  // FRACLAP_TRACE=1: host-side timestamps of every mark (to find host gaps between launches)
  std::chrono::steady_clock::time_point h0 = std::chrono::steady_clock::now(), hm[16];
  bool trace = getenv("FRACLAP_TRACE") != nullptr;
  void mark() {
    if (trace) hm[k] = std::chrono::steady_clock::now();
    cudaEventRecord(e[k++], st);
  }
  void report() {
    if (!trace) return;
    fprintf(stderr, "[fl trace] host us at marks:");
    for (int i = 0; i < k; ++i)
      fprintf(stderr, " %.1f", std::chrono::duration<double, std::micro>(hm[i] - h0).count());
    fprintf(stderr, " | end %.1f\n",
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count());
  }
  double ms(int a, int b) {
    float f = 0;
    cudaEventElapsedTime(&f, e[a], e[b]);
    return f;
  }
};

}  // namespace

extern "C" {

}  // extern "C"

// The assembly.  host != nullptr (whole matrix, 1D, fused cross tiles): the rows are finished
// band by band (tail, cell-local matrices, cross tiles and the local pull of one DoF row band)
// and each band is copied to `host` on a copy stream while the next band is assembled, so the
// PCIe copy — ~4x the assembly at c2 — starts after the first band instead of after the whole
// matrix.  The entries are bitwise those of the unbanded assembly.
static int32_t assemble_impl(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                             const fl_order_params* params, const fl_tables* tables, int64_t n_limit,
                             int64_t row_begin, int64_t row_end, int32_t device, void* stream, fl_dense** out,
                             double* host, bool* host_done) {
  FL_API_BEGIN
  if (host_done) *host_done = false;
  const auto t_enter = std::chrono::steady_clock::now();
  if (!out) return fail(FL_E_ARG, "null output handle");
  *out = nullptr;
  check_inputs(mesh, dofmap, kernel, params, tables);
  if (kernel->variant == FL_VARIANT_SYMMETRIZED)
    return fail(FL_E_ASSEMBLY, "symmetrized kernels are out of scope of the dense device path");
  if (n_limit >= 0 && dofmap->n > n_limit)
    return fail(FL_E_ASSEMBLY, "dense assembly refused beyond " + std::to_string(n_limit) + " dofs");
  const int64_t n = dofmap->n;
  if (row_begin < 0 || row_end > n || row_begin > row_end) return fail(FL_E_ARG, "row range out of bounds");
  FL_CUDA(cudaSetDevice(device));
  std::unique_ptr<fl_dense> D(new fl_dense());
  D->device = device;
  D->n = n;
  D->row0 = row_begin;
  D->row1 = row_end;
  // host output: rows packed (lda = n), so every device->host copy is one contiguous transfer
  // (a pitched copy of n = 8191 rows measured ~6 % slower); the operator is never used for matvecs
  D->lda = host ? n : ((n + 31) / 32) * 32;
  init_pool(device);
  D->stream = acquire_stream(device);                                      // the operator's own stream
  D->own_stream = true;
  cudaStream_t st = stream ? (cudaStream_t)stream : D->stream;             // the assembly's stream
  StreamScope scope(st);
  const int d = mesh->d;
  const double s = kernel->s, C = kernel->C_ds;
  const double ex = -(d / 2.0 + s);
  const int e4 = e4_of(d, s);
  const bool integral = kernel->variant == FL_VARIANT_INTEGRAL;
  const int64_t rows = row_end - row_begin;
  if (rows == 0 && !host) {        // an empty row block (a rank past the last row): nothing to assemble
    D->A.alloc(D->lda);
    FL_CUDA(cudaMemsetAsync(D->A.p, 0, D->lda * sizeof(double), st));
    FL_CUDA(cudaStreamSynchronize(st));
    *out = D.release();
    return FL_OK;
  }

  Timer tm(st);
  tm.h0 = t_enter;
  tm.mark();  // 0
  Uploaded U;
  upload(mesh, dofmap, tables, U, st);
  DevMesh& m = U.m;
  const int ncolors = 0;   // (the cross tiles no longer need a cell colouring)
  OrderConsts oc = make_order_consts(*params, d, s, n);
  DBuf<unsigned long long> ties(1);          // k-flip guard counter (fl_device.cuh order_near_tie)
  FL_CUDA(cudaMemsetAsync(ties.p, 0, sizeof(unsigned long long), st));
  oc.ties = ties.p;

  // target cells: cells with a vertex DoF in the owned rows
  DBuf<int> flags(m.nc), all(m.nc), targets(m.nc), nsel(1);
  flag_target_cells<<<(m.nc + 255) / 256, 256, 0, st>>>(m, (int)row_begin, (int)row_end, flags.p), ::fl::note_launch();
  iota2<<<(m.nc + 255) / 256, 256, 0, st>>>(all.p, m.nc), ::fl::note_launch();
  {
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, all.p, flags.p, targets.p, nsel.p, m.nc, st);
    DBuf<unsigned char> tb(tmp);
    FL_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, all.p, flags.p, targets.p, nsel.p, m.nc, st));
    FL_CHECK_LAUNCH();
  }
  DBuf<int> row_vertex(n > 0 ? n : 1);
  dof_vertex2<<<(m.nv + 255) / 256, 256, 0, st>>>(m, row_vertex.p), ::fl::note_launch();

  // classification (quadrature.py:90-110, assembly.py:412-473, :784-841): counts, then one
  // read-back of every size (targets, touching pairs, boundary items, max valence), then fills
  DBuf<TouchPair> tpairs;
  DBuf<int> ident_k, tcounts, toffs, bcounts, boffs;
  int64_t npairs = 0, nitems = 0;
  const bool do_bnd = integral && m.nb > 0;
  // 1D: the far-field mesh data (source records, DoF tilings) is built here too, and the tail —
  // which needs nothing the host has to know — is enqueued before the host waits for the sizes,
  // so the host-side work below overlaps the tail instead of leaving the GPU idle
  int nbands = 0;
  if (host && d == 1 && row_begin == 0 && row_end == n) {
    const char* env = getenv("FRACLAP_HOST_BANDS");
    nbands = env ? atoi(env) : (n >= 2048 ? 8 : 0);
    if (nbands < 2) nbands = 0;
  }
  // band cut points: a short first band (the copy starts early), then equal tile-aligned bands
  std::vector<int> cut;
  if (nbands) {
    const int T = cross1d_tile_dofs();
    static const int first_tiles = [] { const char* v = getenv("FRACLAP_BAND0_TILES"); return v ? std::max(1, atoi(v)) : 16; }();
    const int first = std::min<int>((int)n, first_tiles * T);
    const int rest = (int)((n - first + nbands - 2) / (nbands - 1));
    const int blk = std::max(T, (rest + T - 1) / T * T);
    cut.push_back(0);
    cut.push_back(first);
    while (cut.back() < n) cut.push_back(std::min<int>((int)n, cut.back() + blk));
    nbands = (int)cut.size() - 1;
    if (nbands > 48) throw Error(FL_E_CUDA, "internal: too many host bands");
  }
  const bool early_tail = d == 1 && !nbands;
  std::unique_ptr<Plan1D, void (*)(Plan1D*)> P1(nullptr, plan1d_free);
  if (d == 1) P1.reset(plan1d_create(m, row_vertex.p, row_begin == 0 && row_end == n, (int)row_begin,
                                     (int)row_end, st));
  // banded: the target cells of every band (cells with a vertex DoF in the band), counts read
  // back with the other sizes
  // (one pass, atomic appends: the per-target results do not depend on the list order)
  DBuf<int> btgt_all((size_t)std::max(nbands, 1) * m.nc), bcnt(std::max(nbands, 1)), dcut(nbands + 1);
  std::vector<const int*> btgt(nbands);
  if (nbands) {
    FL_CUDA(cudaMemsetAsync(bcnt.p, 0, nbands * sizeof(int), st));
    FL_CUDA(cudaMemcpyAsync(dcut.p, cut.data(), (nbands + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    band_targets_kernel<<<(m.nc + 255) / 256, 256, 0, st>>>(m, dcut.p, nbands, btgt_all.p, bcnt.p),
        ::fl::note_launch();
    FL_CHECK_LAUNCH();
    for (int b = 0; b < nbands; ++b) btgt[b] = btgt_all.p + (size_t)b * m.nc;
  }
  touching_count(m, tcounts, toffs, st);
  if (do_bnd) boundary_count(m, bcounts, boffs, st);
  int* hs = pinned_scratch();
  hs[2] = 0;
  hs[5] = 0;
  FL_CUDA(cudaMemcpyAsync(&hs[0], nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&hs[1], toffs.p + m.nc, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (do_bnd) FL_CUDA(cudaMemcpyAsync(&hs[2], boffs.p + m.nb, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&hs[3], U.maxv.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (d == 1) FL_CUDA(cudaMemcpyAsync(&hs[5], plan1d_maxcells(P1.get()), sizeof(int), cudaMemcpyDeviceToHost, st));
  if (nbands) FL_CUDA(cudaMemcpyAsync(&hs[16], bcnt.p, nbands * sizeof(int), cudaMemcpyDeviceToHost, st));
  cudaEvent_t ev_sizes = tm.e[11];                 // (the last timing event doubles as the size fence)
  FL_CUDA(cudaEventRecord(ev_sizes, st));
  // evaluation counters: tail (all), cross (all), tail by the block-pair kernel, cross near blocks
  DBuf<unsigned long long> evc(5);      // [4]: the sym4 part of [2]
  FL_CUDA(cudaMemsetAsync(evc.p, 0, 5 * sizeof(unsigned long long), st));
  DBuf<double> psi((size_t)m.nc * m.q), win((size_t)m.nc * m.q);
  FL_CUDA(cudaMemsetAsync(win.p, 0, win.n * sizeof(double), st));
  // 1D: the tail runs on its own stream, so the cross tiles (issued on `st` once the sizes are
  // back) fill the SMs its last partial wave leaves idle; joined before the cell-local matrices
  struct TailStream {
    int dev; cudaStream_t s = nullptr; cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    TailStream(int d, bool on) : dev(d) {
      if (!on) return;
      s = acquire_stream(d);
      for (auto& x : e) FL_CUDA(cudaEventCreate(&x));
    }
    ~TailStream() {
      for (auto& x : e)
        if (x) cudaEventDestroy(x);
      if (s) release_stream(dev, s);
    }
  };
  static const bool tail_concurrent = [] {
    const char* v = getenv("FRACLAP_TAIL_CONCURRENT");
    return !v || atoi(v) != 0;
  }();
  static const bool tail2d_warp = [] {        // FRACLAP_TAIL2D=warp: round-1 warp-per-target tail only
    const char* v = getenv("FRACLAP_TAIL2D");
    return v && std::string(v) == "warp";
  }();
  // 1D: the tail on its own stream beside the cross tiles.  2D: FRACLAP_TAIL2D_STREAM=1 puts the
  // block-pair tail beside the cross term (measured: no gain at c5 — the block scheduler drains the
  // tail's CTAs first — and the phase timings then overlap), default off
  static const bool tail2d_stream = [] {
    const char* v = getenv("FRACLAP_TAIL2D_STREAM");
    return v && atoi(v) != 0;
  }();
  TailStream tstream(device, ((early_tail || (d == 2 && !tail2d_warp && tail2d_stream)) && tail_concurrent) ||
                                 nbands > 0);
  if (nbands) {
    // banded: the first band's tail runs while the host waits for the sizes (the band's copy
    // cannot start before it); the other bands' tails follow in the band loop
    FL_CUDA(cudaEventRecord(tstream.e[0], st));
    FL_CUDA(cudaStreamWaitEvent(tstream.s, tstream.e[0], 0));
    FL_CUDA(cudaEventRecord(tstream.e[1], tstream.s));
    launch_tail1d(m, U.t, oc, ex, e4, P1.get(), btgt[0], bcnt.p, m.nc, psi.p, evc.p, tstream.s);
    FL_CUDA(cudaEventRecord(tstream.e[2], tstream.s));
  }
  if (early_tail) {
    tm.mark();  // 1
    if (tstream.s) {
      FL_CUDA(cudaEventRecord(tstream.e[0], st));
      FL_CUDA(cudaStreamWaitEvent(tstream.s, tstream.e[0], 0));
      FL_CUDA(cudaEventRecord(tstream.e[1], tstream.s));
      launch_tail1d(m, U.t, oc, ex, e4, P1.get(), targets.p, nsel.p, m.nc, psi.p, evc.p, tstream.s);
      FL_CUDA(cudaEventRecord(tstream.e[2], tstream.s));
    } else {
      launch_tail1d(m, U.t, oc, ex, e4, P1.get(), targets.p, nsel.p, m.nc, psi.p, evc.p, st);
    }
    tm.mark();  // 2
  }
  FL_CUDA(cudaEventSynchronize(ev_sizes));
  const int ntargets = hs[0];
  npairs = hs[1];
  nitems = hs[2];
  valence_error(hs[3]);
  const int maxcells1d = hs[5];
  if (nbands && !cross1d_fused(P1.get(), maxcells1d)) nbands = 0;   // not fused: unbanded, late tail
  touching_fill(m, oc, toffs, npairs, tpairs, ident_k, st);
  DBuf<BndPair> bitems;
  if (do_bnd) boundary_fill(m, oc, boffs, nitems, bitems, st);
  else bitems.alloc(1);
  if (!early_tail) tm.mark();  // 1
  // the CSR indexes of the local pull depend only on the classification: built on a side stream
  // while the main stream runs the singular / tail / cross kernels, joined before the pull.
  // (SparseIndex is destroyed after the final synchronisation, so its stream-ordered frees on
  // the side stream cannot overtake the pull.)
  struct SideStream {                  // returned to the pool after everything declared later
    int dev; cudaStream_t s; cudaEvent_t e[2] = {nullptr, nullptr};
    explicit SideStream(int d) : dev(d), s(acquire_stream(d)) {
      for (auto& x : e) FL_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    ~SideStream() {
      for (auto& x : e)
        if (x) cudaEventDestroy(x);
      release_stream(dev, s);
    }
  } sides(device);
  SparseIndex si;
  cudaStream_t side = sides.s;
  cudaEvent_t ev_cls = sides.e[0], ev_si = sides.e[1];
  FL_CUDA(cudaEventRecord(ev_cls, st));
  FL_CUDA(cudaStreamWaitEvent(side, ev_cls, 0));
  {
    StreamScope sc(side);
    build_sparse_index(m, tpairs.p, npairs, bitems.p, nitems, si, side);
  }
  FL_CUDA(cudaEventRecord(ev_si, side));

  // singular pairs
  DBuf<double> ident((size_t)m.nc * 9), tloc((size_t)std::max<int64_t>(npairs, 1) * 25),
      bloc((size_t)std::max<int64_t>(nitems, 1) * 9);
  launch_singular_identical(m, U.t, ex, e4, ident_k.p, ident.p, st);
  launch_singular_touching(m, U.t, ex, e4, tpairs.p, npairs, tloc.p, st);
  if (do_bnd) launch_singular_boundary(m, U.t, ex, e4, bitems.p, nitems, bloc.p, st);
  // 2D: the Morton cell blocks shared by the tail and the cross term
  Blocks2D blocks;
  struct EvPair {                      // events around the 2D block-pair tail kernel
    cudaEvent_t e[2] = {nullptr, nullptr};
    cudaEvent_t& operator[](int i) { return e[i]; }
    ~EvPair() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } tbev;
  if (d == 2) build_blocks2d(m, U.t, -2.0 * ex, (int)row_begin, (int)row_end, blocks, st);
  if (!early_tail) {
    tm.mark();  // 2
    // tail at the nodes of the target cells (banded 1D: per band, below)
    if (d == 2 && tail2d_warp) launch_tail(m, U.t, oc, ex, e4, targets.p, ntargets, psi.p, evc.p, st);
    else if (d == 2) {
      cudaEventCreate(&tbev[0]);
      cudaEventCreate(&tbev[1]);
      cudaStream_t ts = st;
      if (tstream.s) {                  // joined before the cell-local matrices (psi complete)
        FL_CUDA(cudaEventRecord(tstream.e[0], st));
        FL_CUDA(cudaStreamWaitEvent(tstream.s, tstream.e[0], 0));
        FL_CUDA(cudaEventRecord(tstream.e[1], tstream.s));
        ts = tstream.s;
      }
      {
        StreamScope sc(ts);             // the tail's temporaries are freed in its own stream order
        launch_tail2d_blocks(m, U.t, oc, ex, e4, blocks, targets.p, ntargets, psi.p, evc.p, ts, evc.p + 2, tbev[0],
                             tbev[1], evc.p + 4);
      }
      if (tstream.s) FL_CUDA(cudaEventRecord(tstream.e[2], tstream.s));
    }
    else if (!nbands) launch_tail1d(m, U.t, oc, ex, e4, P1.get(), targets.p, nsel.p, m.nc, psi.p, evc.p, st);
  }
  tm.mark();  // 3
  if (do_bnd) launch_flux(m, U.t, ex, e4, targets.p, ntargets, win.p, st);
  tm.mark();  // 4

  // dense rows: cross term tiles, then the local/sparse pull
  D->A.alloc((size_t)std::max<int64_t>(rows, 1) * D->lda);
  D->A.st = D->stream;
  if (D->lda > n && rows > 0) {
    const int64_t padn = (int64_t)rows * (D->lda - n);
    zero_pad_kernel<<<(unsigned)((padn + 255) / 256), 256, 0, st>>>(D->A.p, rows, n, D->lda), ::fl::note_launch();
    FL_CHECK_LAUNCH();
  }
  const bool full = (row_begin == 0 && row_end == n);
  int64_t ntp = 0, nkeys = 0;
  int ntiles = 0;
  DBuf<unsigned long long> near_keys;
  DBuf<unsigned int> near_cnt(1);
  NearPairs near;
  cudaEvent_t xev[2] = {nullptr, nullptr};
  bool done1d = false;
  DBuf<double> Lc((size_t)m.nc * 9);
  struct CopyStream {                  // device -> host copies of finished bands
    int dev; cudaStream_t s = nullptr; std::vector<cudaEvent_t> e, t;   // t: FRACLAP_TRACE copy spans
    CopyStream(int d, int nb, bool trace) : dev(d) {
      if (!nb) return;
      s = acquire_stream(d);
      e.resize(nb, nullptr);
      for (auto& x : e) FL_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      if (trace) {
        t.resize(2 * nb, nullptr);
        for (auto& x : t) FL_CUDA(cudaEventCreate(&x));
      }
    }
    ~CopyStream() {
      if (!s) return;
      cudaStreamSynchronize(s);
      for (auto* v : {&e, &t})
        for (auto& x : *v)
          if (x) cudaEventDestroy(x);
      release_stream(dev, s);
    }
  } cps(device, nbands, tm.trace);
  if (nbands) {
    tm.mark();  // 5
    for (int b = 0; b < nbands; ++b) {
      const int nt_b = hs[16 + b];
      if (b == 0) FL_CUDA(cudaStreamWaitEvent(st, tstream.e[2], 0));     // launched before the size sync
      else launch_tail1d(m, U.t, oc, ex, e4, P1.get(), btgt[b], bcnt.p + b, nt_b, psi.p, evc.p, st);
      launch_cell_local(m, U.t, C, s, integral && m.nb > 0, btgt[b], nt_b, ident.p, psi.p, win.p, Lc.p, st);
      launch_cross1d(m, U.t, oc, ex, e4, C, P1.get(), maxcells1d, targets.p, ntargets, row_vertex.p, D->A.p, D->lda,
                     evc.p + 1, st, cut[b], cut[b + 1]);
      if (b == 0) FL_CUDA(cudaStreamWaitEvent(st, ev_si, 0));
      launch_sparse_pull(m, C, s, Lc.p, tpairs.p, tloc.p, bitems.p, do_bnd ? bloc.p : nullptr, si, row_vertex.p,
                         cut[b], cut[b + 1], D->A.p + (int64_t)cut[b] * D->lda, D->lda, st);   // (rows from cut[b])
      FL_CUDA(cudaEventRecord(cps.e[b], st));
      FL_CUDA(cudaStreamWaitEvent(cps.s, cps.e[b], 0));
      if (tm.trace) cudaEventRecord(cps.t[2 * b], cps.s);
      FL_CUDA(cudaMemcpyAsync(host + (int64_t)cut[b] * n, D->A.p + (int64_t)cut[b] * n,
                              (size_t)(cut[b + 1] - cut[b]) * n * sizeof(double), cudaMemcpyDeviceToHost, cps.s));
      if (tm.trace) cudaEventRecord(cps.t[2 * b + 1], cps.s);
    }
    done1d = true;
  } else if (d == 1) {
    tm.mark();  // 5
    done1d = launch_cross1d(m, U.t, oc, ex, e4, C, P1.get(), maxcells1d, targets.p, ntargets, row_vertex.p, D->A.p,
                            D->lda, evc.p + 1, st);
  }
  static const bool cross2d_tiles = [] {      // FRACLAP_CROSS2D=tiles: the round-1 DoF-tile kernel
    const char* v = getenv("FRACLAP_CROSS2D");
    return v && std::string(v) == "tiles";
  }();
  Cross2DInfo x2{};
  if (!done1d && d == 2 && !cross2d_tiles) {
    cudaEventCreate(&xev[0]);
    cudaEventCreate(&xev[1]);
    tm.mark();  // 5
    assemble_cross2d(m, U.t, oc, ex, e4, C, blocks, (int)row_begin, (int)row_end, D->A.p, D->lda, evc.p + 1, near, x2,
                     xev[0], xev[1], st, evc.p + 3);
    ntiles = -1;
    done1d = true;
    if (x2.fallback) {
      // the mesh is too irregular for the fixed-point accumulation (Cross2DInfo::fallback): nothing
      // was added to A; the DoF-tile kernel below assembles the cross term (its own near pairs)
      done1d = false;
      cudaEventDestroy(xev[0]);
      cudaEventDestroy(xev[1]);
      FL_CUDA(cudaMemsetAsync(evc.p + 1, 0, sizeof(unsigned long long), st));
      FL_CUDA(cudaMemsetAsync(evc.p + 3, 0, sizeof(unsigned long long), st));
    }
  }
  if (!done1d) {
    cudaEventCreate(&xev[0]);
    cudaEventCreate(&xev[1]);
    Tiles trow, tcol;
    build_tiles(m, (int)row_begin, (int)row_end, trow, st);
    if (!full) build_tiles(m, 0, (int)n, tcol, st);
    ntiles = trow.ntiles;
    TilePairs tps;
    build_tile_pairs(m, oc, trow, full ? trow : tcol, full, d == 1 ? KW1D : KW2D, tps, st);
    ntp = tps.nall;
    if (d != 1 && !x2.fallback) tm.mark();  // 5 (1D fallback / 2D fixed-point fallback: already marked)
    // pass 1 (discovery): orders of the pairs of the tile pairs that can hold near pairs (order
    // >= KW, by the tile bound); near pairs are recorded.  Near-key list (with halo duplicates):
    // generous, bounded by a quarter of the free memory
    // capacity: the exact bound from the tile pairs (a pair is scanned once per tile pair holding
    // it), capped; a rare overflow grows the list and rediscovers
    unsigned int cap = (unsigned int)std::max<int64_t>(
        1024, std::min<int64_t>({tps.near_candidates, (int64_t)m.nc * 4096, ((int64_t)1 << 31) - 1}));
    for (int attempt = 0; attempt < 2; ++attempt) {
      near_keys.alloc(cap);
      FL_CUDA(cudaMemsetAsync(near_cnt.p, 0, sizeof(unsigned int), st));
      launch_cross_tiles(m, U.t, oc, ex, e4, C, trow, full ? trow : tcol, tps.near.p, tps.nnear, full,
                         (int)row_begin, (int)row_end, D->A.p, D->lda, evc.p + 1, near_keys.p, near_cnt.p, cap, 1,
                         nullptr, nullptr, 0, nullptr, st);
      unsigned int cnt = 0;
      FL_CUDA(cudaMemcpyAsync(&cnt, near_cnt.p, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
      FL_CUDA(cudaStreamSynchronize(st));
      nkeys = cnt;
      if (cnt <= cap) break;
      cap = cnt;                                 // rare: grow the list and rediscover
    }
    cudaEventRecord(xev[0], st);
    // each near block once (warp per pair), then pass 2 computes the rest and scatters all
    near_pairs_build(m, U.t, oc, ex, e4, near_keys.p, nkeys, near, evc.p + 1, st);
    near_keys.free();
    cudaEventRecord(xev[1], st);
    launch_cross_tiles(m, U.t, oc, ex, e4, C, trow, full ? trow : tcol, tps.all.p, tps.nall, full, (int)row_begin,
                       (int)row_end, D->A.p, D->lda, evc.p + 1, nullptr, nullptr, 0, 0, near.hkey.p, near.hidx.p,
                       near.hmask, near.G.p, st);
  }
  tm.mark();  // 6
  if (tstream.s) FL_CUDA(cudaStreamWaitEvent(st, tstream.e[2], 0));   // psi complete
  if (!nbands) {
    launch_cell_local(m, U.t, C, s, integral && m.nb > 0, targets.p, ntargets, ident.p, psi.p, win.p, Lc.p, st);
    FL_CUDA(cudaStreamWaitEvent(st, ev_si, 0));
    launch_sparse_pull(m, C, s, Lc.p, tpairs.p, tloc.p, bitems.p, do_bnd ? bloc.p : nullptr, si, row_vertex.p,
                       (int)row_begin, (int)row_end, D->A.p, D->lda, st);
  }
  tm.mark();  // 7
  unsigned long long* hev = reinterpret_cast<unsigned long long*>(hs + 32);
  FL_CUDA(cudaMemcpyAsync(hev, evc.p, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&hs[4], m.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  unsigned long long hties = 0;
  FL_CUDA(cudaMemcpyAsync(&hties, ties.p, sizeof(hties), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (nbands) {
    FL_CUDA(cudaStreamSynchronize(cps.s));
    if (host_done) *host_done = true;
  }
  const int herr = hs[4];
  if (herr & 1) throw Error(FL_E_QUAD, "a quadrature rule for a selected order is missing from the tables");
  if (herr & 4) throw Error(FL_E_CUDA, "internal: a near pair missing from the discovery pass");

  fl_assembly_stats& S = D->stats;
  const int64_t nc = m.nc;
  S.pairs_identical = nc;
  S.pairs_touching = npairs;
  S.pairs_cross = nc * (nc - 1) / 2 - npairs;
  S.pairs_tail = nc * (nc - 1) - 2 * npairs;
  S.pairs_boundary_singular = nitems;
  S.pairs_boundary_flux = integral ? nc * m.nb : 0;
  S.evals_tail = (double)hev[0] + (double)hev[2];     // warp-per-target pairs + block-pair kernel
  S.order_ties = (int64_t)hties;
  S.evals_cross = (double)hev[1] + (double)hev[3];    // far blocks + near blocks
  S.evals_tail_block = (double)hev[2];
  S.evals_near = (double)hev[3];
  S.evals_tail_sym = (double)hev[4];
  S.ms_tail_block = 0.0;
  if (tbev[1]) {
    float a = 0.f;
    cudaEventElapsedTime(&a, tbev[0], tbev[1]);
    S.ms_tail_block = a;
  }
  S.ms_prep = tm.ms(0, 1);
  S.ms_singular = early_tail ? tm.ms(2, 3) : tm.ms(1, 2);   // 1D: tail (1 -> 2) runs before the singular kernels
  S.ms_tail = early_tail ? tm.ms(1, 2) : tm.ms(2, 3);
  if (tstream.s) {   // concurrent tail: its own span on its stream
    float a = 0.f;
    cudaEventElapsedTime(&a, tstream.e[1], tstream.e[2]);
    S.ms_tail = a;
  }
  S.ms_flux = tm.ms(3, 4);
  S.ms_tiles = tm.ms(4, 5);
  S.ms_cross = tm.ms(5, 6);
  S.ms_local = tm.ms(6, 7);
  S.ms_total = tm.ms(0, 7);
  tm.report();
  if (tm.trace && nbands) {
    fprintf(stderr, "[fl trace] band copies (ms from mark 0, start-end):");
    for (int b = 0; b < nbands; ++b) {
      float a = 0.f, z = 0.f;
      cudaEventElapsedTime(&a, tm.e[0], cps.t[2 * b]);
      cudaEventElapsedTime(&z, tm.e[0], cps.t[2 * b + 1]);
      fprintf(stderr, " %.3f-%.3f", a, z);
    }
    fprintf(stderr, "\n");
  }
  S.cross_tile_pairs = ntp;
  S.near_pairs = near.n;
  if (ntiles > 0 || ntiles == -1) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, tm.e[5], xev[0]);
    cudaEventElapsedTime(&b, xev[0], xev[1]);
    cudaEventElapsedTime(&c, xev[1], tm.e[6]);
    S.ms_discover = a; S.ms_near = b; S.ms_cross_compute = c;
  }
  for (auto& e : xev)
    if (e) cudaEventDestroy(e);
  S.ncolors = ncolors;
  S.ntiles = ntiles;
  if (ntiles == -1) {
    S.cross_tile_pairs = x2.block_pairs;
    S.ntiles = 0;
    S.cross_scale_exp = x2.scale_exp;
  }
  S.cross_fallback = x2.fallback;
  *out = D.release();
  return FL_OK;
  FL_API_END
}

extern "C" {

int32_t fl_assemble_dense(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                          const fl_order_params* params, const fl_tables* tables, int64_t n_limit,
                          int64_t row_begin, int64_t row_end, int32_t device, void* stream, fl_dense** out) {
  return assemble_impl(mesh, dofmap, kernel, params, tables, n_limit, row_begin, row_end, device, stream, out,
                       nullptr, nullptr);
}

// Whole matrix straight into host memory: the ndarray assembly.assemble_dense returns
// (assembly.py:1059-1104).  1D: banded, each finished row band copied while the next one is
// assembled (assemble_impl); otherwise one assembly, then one pitched device->host copy.
int32_t fl_assemble_dense_host(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                               const fl_order_params* params, const fl_tables* tables, int64_t n_limit,
                               int32_t device, double* host) {
  if (!host || !dofmap) return fail(FL_E_ARG, "null argument");
  fl_dense* D = nullptr;
  bool copied = false;
  int32_t rc = assemble_impl(mesh, dofmap, kernel, params, tables, n_limit, 0, dofmap->n, device, nullptr, &D, host,
                             &copied);
  if (rc != FL_OK) return rc;
  if (!copied) rc = fl_dense_to_host(D, host);
  fl_dense_free(D);
  return rc;
}

// ------------------------------------------------------------- host O(n) steps on the device
int32_t fl_finish_polygon_mesh(const double* vertices, int64_t nv, const int64_t* cells_in, int64_t nc,
                               int32_t device, int64_t* cells_out, int64_t* boundary_edges_out,
                               double* boundary_normals_out, int64_t capacity, int64_t* nb_out) {
  FL_API_BEGIN
  if (!vertices || !cells_in || !cells_out || !nb_out || nv <= 0 || nc <= 0) return fail(FL_E_ARG, "bad argument");
  if (3 * nc >= (1LL << 31) || nv >= (1LL << 31)) return fail(FL_E_ARG, "mesh too large");
  for (int64_t i = 0; i < 3 * nc; ++i)
    if (cells_in[i] < 0 || cells_in[i] >= nv) return fail(FL_E_ARG, "cell vertex index out of range");
  const int32_t rc = fl::finish_polygon_mesh(vertices, nv, cells_in, nc, device, cells_out, boundary_edges_out,
                                             boundary_normals_out, capacity, nb_out);
  if (rc != FL_OK) return fail(rc, "boundary edge capacity too small");
  return FL_OK;
  FL_API_END
}

int32_t fl_build_dofmap(const fl_mesh* mesh, double s, int32_t device, int64_t* vertex_to_dof_out, int64_t* n_out) {
  FL_API_BEGIN
  if (!mesh || !vertex_to_dof_out || !n_out) return fail(FL_E_ARG, "null argument");
  if (!(s > 0.0 && s < 1.0)) return fail(FL_E_ARG, "fractional order s must lie in (0,1)");   // mesh.py:208-209
  if (mesh->nv <= 0 || mesh->nv >= (1LL << 31)) return fail(FL_E_ARG, "bad vertex count");
  return fl::dofmap_build(mesh->boundary_edges, mesh->nb, mesh->d, mesh->nv, s, device, vertex_to_dof_out, n_out);
  FL_API_END
}

int32_t fl_cell_rule_nodes(const fl_mesh* mesh, const double* pts, int64_t q, int32_t device, double* X_out) {
  FL_API_BEGIN
  if (!mesh || !pts || !X_out || q <= 0 || (mesh->d != 1 && mesh->d != 2)) return fail(FL_E_ARG, "bad argument");
  return fl::cell_rule_nodes(mesh, pts, q, device, X_out);
  FL_API_END
}

int32_t fl_load_vector(const fl_mesh* mesh, const fl_dofmap* dofmap, const double* pts, const double* w, int64_t q,
                       const double* f_values, double f_const, int32_t device, double* b_out) {
  FL_API_BEGIN
  if (!mesh || !dofmap || !pts || !w || !b_out || q <= 0 || (mesh->d != 1 && mesh->d != 2))
    return fail(FL_E_ARG, "bad argument");
  if (mesh->nc * (mesh->d + 1) >= (1LL << 31) || dofmap->n >= (1LL << 31)) return fail(FL_E_ARG, "mesh too large");
  return fl::load_vector(mesh, dofmap, pts, w, q, f_values, f_const, device, b_out);
  FL_API_END
}

// ------------------------------------------------------------- near field (cluster path)
int32_t fl_assemble_near_field(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                               const fl_order_params* params, const fl_tables* tables,
                               const fl_near_structure* near, const double* V_nodes, int32_t device,
                               fl_sparse** out) {
  FL_API_BEGIN
  if (!out || !near) return fail(FL_E_ARG, "null argument");
  *out = nullptr;
  check_inputs(mesh, dofmap, kernel, params, tables);
  if (kernel->variant == FL_VARIANT_SYMMETRIZED)
    return fail(FL_E_ASSEMBLY, "symmetrized kernels are assembled densely");          // assembly.py:870-871
  const int64_t n = dofmap->n, nl = near->nleaves, np = near->npairs;
  if (nl <= 0 || nl >= (1LL << 31) || np < 0 || (np > 0 && !near->pairs) || (n > 0 && !near->leaf_of_dof))
    return fail(FL_E_ARG, "bad near structure");
  std::vector<int> lod((size_t)std::max<int64_t>(n, 1)), prs((size_t)std::max<int64_t>(2 * np, 1));
  for (int64_t i = 0; i < n; ++i) {
    if (near->leaf_of_dof[i] < 0 || near->leaf_of_dof[i] >= nl) return fail(FL_E_ARG, "leaf index out of range");
    lod[i] = (int)near->leaf_of_dof[i];
  }
  for (int64_t p = 0; p < np; ++p) {
    int64_t a = near->pairs[2 * p], b = near->pairs[2 * p + 1];
    if (a < 0 || b < 0 || a >= nl || b >= nl) return fail(FL_E_ARG, "near leaf pair out of range");
    prs[2 * p] = (int)std::min(a, b);
    prs[2 * p + 1] = (int)std::max(a, b);
  }
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  std::unique_ptr<fl_sparse> S(new fl_sparse());
  S->device = device;
  S->n = n;
  S->stream = acquire_stream(device);
  cudaStream_t st = S->stream;
  StreamScope scope(st);
  const int d = mesh->d;
  const double s = kernel->s, C = kernel->C_ds;
  const double ex = -(d / 2.0 + s);
  const int e4 = e4_of(d, s);
  const bool integral = kernel->variant == FL_VARIANT_INTEGRAL;
  Uploaded U;
  upload(mesh, dofmap, tables, U, st);
  DevMesh& m = U.m;
  const OrderConsts oc = make_order_consts(*params, d, s, n);
  DBuf<int> dlod(lod.size()), dprs(prs.size());
  FL_CUDA(cudaMemcpyAsync(dlod.p, lod.data(), lod.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dprs.p, prs.data(), prs.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  DBuf<double> dV;
  if (V_nodes) {
    dV.alloc((size_t)m.nc * m.q);
    FL_CUDA(cudaMemcpyAsync(dV.p, V_nodes, dV.n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  DBuf<int> row_vertex(n > 0 ? n : 1), all(m.nc);
  dof_vertex2<<<(m.nv + 255) / 256, 256, 0, st>>>(m, row_vertex.p), ::fl::note_launch();
  iota2<<<(m.nc + 255) / 256, 256, 0, st>>>(all.p, m.nc), ::fl::note_launch();
  // classification + singular pairs exactly as the dense path (the touching triplets are not
  // masked, assembly.py:885; touching pairs are never admissible)
  DBuf<TouchPair> tpairs;
  DBuf<int> ident_k, tcounts, toffs, bcounts, boffs;
  const bool do_bnd = integral && m.nb > 0;
  touching_count(m, tcounts, toffs, st);
  if (do_bnd) boundary_count(m, bcounts, boffs, st);
  int* hs = pinned_scratch();
  hs[2] = 0;
  FL_CUDA(cudaMemcpyAsync(&hs[1], toffs.p + m.nc, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (do_bnd) FL_CUDA(cudaMemcpyAsync(&hs[2], boffs.p + m.nb, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(&hs[3], U.maxv.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  const int64_t npairs = hs[1], nitems = hs[2];
  valence_error(hs[3]);
  touching_fill(m, oc, toffs, npairs, tpairs, ident_k, st);
  DBuf<BndPair> bitems;
  if (do_bnd) boundary_fill(m, oc, boffs, nitems, bitems, st);
  else bitems.alloc(1);
  SparseIndex si;
  build_sparse_index(m, tpairs.p, npairs, bitems.p, nitems, si, st);
  DBuf<double> ident((size_t)m.nc * 9), tloc((size_t)std::max<int64_t>(npairs, 1) * 25),
      bloc((size_t)std::max<int64_t>(nitems, 1) * 9);
  launch_singular_identical(m, U.t, ex, e4, ident_k.p, ident.p, st);
  launch_singular_touching(m, U.t, ex, e4, tpairs.p, npairs, tloc.p, st);
  if (do_bnd) launch_singular_boundary(m, U.t, ex, e4, bitems.p, nitems, bloc.p, st);
  // tail through the one-ring boundary, and the boundary mass potential
  DBuf<double> psi((size_t)m.nc * m.q), win((size_t)m.nc * m.q);
  launch_ring_tail(m, U.t, s, ex, e4, V_nodes ? dV.p : nullptr, do_bnd, psi.p, win.p, st);
  DBuf<double> Lc((size_t)m.nc * 9);
  launch_cell_local(m, U.t, C, s, do_bnd, all.p, m.nc, ident.p, psi.p, win.p, Lc.p, st);
  // near disjoint pairs, CSR pattern and cross values, then the local entries
  NearInput in;
  in.nleaves = (int)nl;
  in.npairs = np;
  in.leaf_of_dof = dlod.p;
  in.pairs = dprs.p;
  CsrOut csr;
  DBuf<unsigned long long> evc(1);
  FL_CUDA(cudaMemsetAsync(evc.p, 0, sizeof(unsigned long long), st));
  int64_t ncross = 0;
  near_field_cross(m, U.t, oc, ex, e4, C, in, row_vertex.p, csr, &ncross, evc.p, st);
  launch_sparse_pull_csr(m, C, s, Lc.p, tpairs.p, tloc.p, bitems.p, do_bnd ? bloc.p : nullptr, si, row_vertex.p,
                         (int)n, csr.indptr.p, csr.indices.p, csr.data.p, st);
  FL_CUDA(cudaMemcpyAsync(&hs[4], m.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (hs[4] & 1) throw Error(FL_E_QUAD, "a quadrature rule for a selected order is missing from the tables");
  if (hs[4] & 4) throw Error(FL_E_CUDA, "internal: a near-field pair block is missing");
  if (hs[4] & 16) throw Error(FL_E_ASSEMBLY, "one-ring patch too large for the device ring lists");
  S->nnz = csr.nnz;
  S->pairs = ncross;
  S->indptr = std::move(csr.indptr);
  S->indices = std::move(csr.indices);
  S->data = std::move(csr.data);
  *out = S.release();
  return FL_OK;
  FL_API_END
}

// psi (tail_potential) and W_in at the (nc, q) cell nodes, as fl_assemble_near_field forms them
int32_t fl_debug_ring_tail(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                           const fl_order_params* params, const fl_tables* tables, const double* V_nodes,
                           int32_t device, double* psi_out, double* win_out) {
  FL_API_BEGIN
  if (!psi_out || !win_out) return fail(FL_E_ARG, "null argument");
  check_inputs(mesh, dofmap, kernel, params, tables);
  FL_CUDA(cudaSetDevice(device));
  init_pool(device);
  OwnedStreamLease lease(device);
  cudaStream_t st = lease.s;
  StreamScope scope(st);
  const int d = mesh->d;
  const double s = kernel->s;
  Uploaded U;
  upload(mesh, dofmap, tables, U, st);
  DevMesh& m = U.m;
  check_valence(U, st);
  DBuf<double> dV, psi((size_t)m.nc * m.q), win((size_t)m.nc * m.q);
  if (V_nodes) {
    dV.alloc((size_t)m.nc * m.q);
    FL_CUDA(cudaMemcpyAsync(dV.p, V_nodes, dV.n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  launch_ring_tail(m, U.t, s, -(d / 2.0 + s), e4_of(d, s), V_nodes ? dV.p : nullptr,
                   kernel->variant == FL_VARIANT_INTEGRAL && m.nb > 0, psi.p, win.p, st);
  FL_CUDA(cudaMemcpyAsync(psi_out, psi.p, psi.n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(win_out, win.p, win.n * sizeof(double), cudaMemcpyDeviceToHost, st));
  int err = 0;
  FL_CUDA(cudaMemcpyAsync(&err, m.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (err & 16) throw Error(FL_E_ASSEMBLY, "one-ring patch too large for the device ring lists");
  return FL_OK;
  FL_API_END
}

int32_t fl_sparse_info(const fl_sparse* A, int64_t* n, int64_t* nnz, int64_t* cross_pairs) {
  if (!A) return fail(FL_E_ARG, "null handle");
  if (n) *n = A->n;
  if (nnz) *nnz = A->nnz;
  if (cross_pairs) *cross_pairs = A->pairs;
  return FL_OK;
}

int32_t fl_sparse_to_host(const fl_sparse* A, int64_t* indptr, int32_t* indices, double* data) {
  FL_API_BEGIN
  if (!A || !indptr || (A->nnz > 0 && (!indices || !data))) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(A->device));
  FL_CUDA(cudaMemcpyAsync(indptr, A->indptr.p, (A->n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, A->stream));
  if (A->nnz > 0) {
    FL_CUDA(cudaMemcpyAsync(indices, A->indices.p, A->nnz * sizeof(int), cudaMemcpyDeviceToHost, A->stream));
    FL_CUDA(cudaMemcpyAsync(data, A->data.p, A->nnz * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  }
  FL_CUDA(cudaStreamSynchronize(A->stream));
  return FL_OK;
  FL_API_END
}

void fl_sparse_free(fl_sparse* A) {
  if (!A) return;
  cudaSetDevice(A->device);
  delete A;
}

int32_t fl_dense_from_host_rows(const double* rows_host, int64_t n, int64_t row_begin, int64_t row_end,
                                int32_t device, fl_dense** out) {
  FL_API_BEGIN
  if (!out) return fail(FL_E_ARG, "null output handle");
  *out = nullptr;
  if (n <= 0 || row_begin < 0 || row_end < row_begin || row_end > n || (row_end > row_begin && !rows_host))
    return fail(FL_E_ARG, "bad argument");
  DeviceScope dev(device);
  std::unique_ptr<fl_dense> D(new fl_dense());
  D->device = device;
  D->n = n;
  D->row0 = row_begin;
  D->row1 = row_end;
  D->lda = ((n + 31) / 32) * 32;
  const int64_t rows = row_end - row_begin;
  init_pool(device);
  D->stream = acquire_stream(device);
  D->own_stream = true;
  StreamScope scope(D->stream);
  D->A.alloc((size_t)std::max<int64_t>(rows, 1) * D->lda);
  FL_CUDA(cudaMemsetAsync(D->A.p, 0, (size_t)std::max<int64_t>(rows, 1) * D->lda * sizeof(double), D->stream));
  if (rows > 0)
    FL_CUDA(cudaMemcpy2DAsync(D->A.p, D->lda * sizeof(double), rows_host, n * sizeof(double), n * sizeof(double),
                              rows, cudaMemcpyHostToDevice, D->stream));
  FL_CUDA(cudaStreamSynchronize(D->stream));
  *out = D.release();
  return FL_OK;
  FL_API_END
}

int32_t fl_dense_from_host(const double* A, int64_t n, int32_t device, fl_dense** out) {
  if (!A) return fail(FL_E_ARG, "bad argument");
  return fl_dense_from_host_rows(A, n, 0, n, device, out);
}

void fl_dense_free(fl_dense* A) {
  if (!A) return;
  cudaSetDevice(A->device);
  delete A;
}

int32_t fl_dense_info(const fl_dense* A, int64_t* n, int64_t* r0, int64_t* r1, double** ptr) {
  if (!A) return fail(FL_E_ARG, "null handle");
  if (n) *n = A->n;
  if (r0) *r0 = A->row0;
  if (r1) *r1 = A->row1;
  if (ptr) *ptr = A->A.p;
  return FL_OK;
}

int32_t fl_dense_stats(const fl_dense* A, fl_assembly_stats* s) {
  if (!A || !s) return fail(FL_E_ARG, "null argument");
  *s = A->stats;
  return FL_OK;
}

int32_t fl_dense_to_host(const fl_dense* A, double* host) {
  FL_API_BEGIN
  if (!A || !host) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(A->device));
  StreamScope scope(A->stream);
  const int64_t rows = A->row1 - A->row0;
  if (rows == 0 || A->n == 0) return FL_OK;
  if (A->lda == A->n)
    FL_CUDA(cudaMemcpyAsync(host, A->A.p, (size_t)rows * A->n * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  else
    FL_CUDA(cudaMemcpy2DAsync(host, A->n * sizeof(double), A->A.p, A->lda * sizeof(double), A->n * sizeof(double),
                              rows, cudaMemcpyDeviceToHost, A->stream));
  FL_CUDA(cudaStreamSynchronize(A->stream));
  return FL_OK;
  FL_API_END
}

int32_t fl_dense_rows(const fl_dense* A, int64_t nrows, const int64_t* rows, double* host_out) {
  FL_API_BEGIN
  if (!A || (nrows > 0 && (!rows || !host_out))) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(A->device));
  StreamScope scope(A->stream);
  for (int64_t r = 0; r < nrows; ++r)
    if (rows[r] < A->row0 || rows[r] >= A->row1) return fail(FL_E_ARG, "row outside the operator's rows");
  for (int64_t r = 0; r < nrows; ++r)
    FL_CUDA(cudaMemcpyAsync(host_out + r * A->n, A->A.p + (rows[r] - A->row0) * A->lda, A->n * sizeof(double),
                            cudaMemcpyDeviceToHost, A->stream));
  FL_CUDA(cudaStreamSynchronize(A->stream));
  return FL_OK;
  FL_API_END
}

int32_t fl_dense_diag(const fl_dense* A, double* host_diag) {
  FL_API_BEGIN
  if (!A || !host_diag) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(A->device));
  StreamScope scope(A->stream);
  const int64_t rows = A->row1 - A->row0;
  if (rows == 0) return FL_OK;
  DBuf<double> d(rows);
  launch_diag(A->A.p, rows, A->row0, A->lda, d.p, A->stream);
  FL_CUDA(cudaMemcpyAsync(host_diag, d.p, rows * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  FL_CUDA(cudaStreamSynchronize(A->stream));
  return FL_OK;
  FL_API_END
}

int32_t fl_matvec_async(const fl_dense* A, const double* x_dev, double* y_dev, void* stream) {
  FL_API_BEGIN
  if (!A || !x_dev || !y_dev) return fail(FL_E_ARG, "null argument");
  cudaStream_t st = stream ? (cudaStream_t)stream : A->stream;
  launch_matvec(A->A.p, A->row1 - A->row0, A->n, A->lda, x_dev, y_dev, st);
  return FL_OK;
  FL_API_END
}

int32_t fl_matvec(const fl_dense* A, const double* x, double* y, int32_t ptr_kind) {
  FL_API_BEGIN
  if (!A || !x || !y) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(A->device));
  StreamScope scope(A->stream);
  const int64_t rows = A->row1 - A->row0;
  if (ptr_kind == 1) {
    launch_matvec(A->A.p, rows, A->n, A->lda, x, y, A->stream);
    FL_CUDA(cudaStreamSynchronize(A->stream));
    return FL_OK;
  }
  DBuf<double> xd(A->lda), yd(std::max<int64_t>(rows, 1));
  FL_CUDA(cudaMemsetAsync(xd.p, 0, A->lda * sizeof(double), A->stream));
  FL_CUDA(cudaMemcpyAsync(xd.p, x, A->n * sizeof(double), cudaMemcpyHostToDevice, A->stream));
  launch_matvec(A->A.p, rows, A->n, A->lda, xd.p, yd.p, A->stream);
  FL_CUDA(cudaMemcpyAsync(y, yd.p, rows * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
  FL_CUDA(cudaStreamSynchronize(A->stream));
  return FL_OK;
  FL_API_END
}

int32_t fl_pcg(const fl_dense* A, const double* b, const double* x0, double tol, int64_t max_iter, int32_t precond,
               double* x, fl_solve_report* rep) {
  FL_API_BEGIN
  if (!A || !b || !x || !rep) return fail(FL_E_ARG, "null argument");
  if (A->row0 != 0 || A->row1 != A->n) return fail(FL_E_ARG, "fl_pcg needs the whole matrix on one device");
  FL_CUDA(cudaSetDevice(A->device));
  StreamScope scope(A->stream);
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n = A->n, L = A->lda;
  cudaStream_t st = A->stream;
  std::vector<double> diag(n), minv(n);
  if (precond == 1) {
    DBuf<double> d(std::max<int64_t>(n, 1));
    launch_diag(A->A.p, n, 0, L, d.p, st);
    FL_CUDA(cudaMemcpyAsync(diag.data(), d.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < n; ++i) {
      if (!(diag[i] > 0)) return fail(FL_E_SOLVER, "nonpositive diagonal; operator not SPD");   // solve.py:67-68
      minv[i] = 1.0 / diag[i];
    }
  } else {
    for (int64_t i = 0; i < n; ++i) minv[i] = 1.0;
  }
  DBuf<double> dminv(L), dx(L), dr(L), dz(L), dp(L), dAp(L), db(L);
  for (auto* buf : {&dminv, &dx, &dr, &dz, &dp, &dAp, &db}) FL_CUDA(cudaMemsetAsync(buf->p, 0, L * sizeof(double), st));
  FL_CUDA(cudaMemcpyAsync(dminv.p, minv.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(dr.p, b, n * sizeof(double), cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice, st));
  if (x0) FL_CUDA(cudaMemcpyAsync(dx.p, x0, n * sizeof(double), cudaMemcpyHostToDevice, st));
  const long long mi = max_iter;
  PcgResult r = run_pcg(A->A.p, n, L, dminv.p, dx.p, dr.p, dz.p, dp.p, dAp.p, tol, mi, x0 != nullptr, st);
  if (r.error) return fail(FL_E_SOLVER, "p^T A p <= 0: operator not SPD");                  // solve.py:87-88
  FL_CUDA(cudaMemcpyAsync(x, dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  // true residual ||b - A x|| / ||b|| reported beside the reference's preconditioned one
  launch_matvec(A->A.p, n, n, L, dx.p, dAp.p, st);
  std::vector<double> ax(n);
  FL_CUDA(cudaMemcpyAsync(ax.data(), dAp.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  double nr = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    nr += (b[i] - ax[i]) * (b[i] - ax[i]);
    nb += b[i] * b[i];
  }
  const auto t1 = std::chrono::steady_clock::now();
  rep->iterations = r.it;
  rep->residual = (r.norm0 == 0.0) ? 0.0 : std::sqrt(std::fabs(r.rz)) / r.norm0;
  rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  rep->converged = (r.norm0 == 0.0) ? 1 : r.converged;
  rep->true_residual = nb > 0 ? std::sqrt(nr / nb) : 0.0;
  return FL_OK;
  FL_API_END
}

int32_t fl_cg_create(int64_t n, int64_t m_local, int64_t block_rows, int32_t world, int32_t rank, double tol,
                     int64_t max_iter, int32_t device, void* stream, fl_cg** out) {
  FL_API_BEGIN
  if (!out) return fail(FL_E_ARG, "null argument");
  *out = nullptr;
  DeviceScope dev(device);
  StreamScope scope((cudaStream_t)stream);
  *out = cg_create(n, m_local, block_rows, world, rank, tol, (long long)max_iter, device);
  return FL_OK;
  FL_API_END
}

int32_t fl_cg_buffers(fl_cg* S, double** local_parts, double** all_parts, int64_t* chunks_per_rank) {
  FL_API_BEGIN
  if (!S) return fail(FL_E_ARG, "null argument");
  if (local_parts) *local_parts = cg_local_parts(S);
  if (all_parts) *all_parts = cg_all_parts(S);
  if (chunks_per_rank) *chunks_per_rank = cg_chunks(S);
  return FL_OK;
  FL_API_END
}

int32_t fl_cg_bind_parts(fl_cg* S, double* local_parts) {
  FL_API_BEGIN
  if (!S) return fail(FL_E_ARG, "null argument");
  cg_bind_parts(S, local_parts);
  return FL_OK;
  FL_API_END
}

#define FL_CG_CALL(cond, body)                                          \
  FL_API_BEGIN                                                         \
  if (!S || !(cond)) return fail(FL_E_ARG, "null argument");           \
  DeviceScope dev(cg_device(S));                                       \
  cudaStream_t st = (cudaStream_t)stream;                              \
  StreamScope scope(st);                                               \
  body;                                                                \
  return FL_OK;                                                        \
  FL_API_END

static void cg_check_rows(const fl_cg* S, const fl_dense* A) {
  int dev;
  int64_t n, row0, m;
  cg_info(S, &dev, &n, &row0, &m);
  if (A->device != dev || A->n != n || A->row0 != row0 || A->row1 - A->row0 != m)
    throw Error(FL_E_ARG, "operator rows do not match the CG rank's row block");
}

int32_t fl_cg_begin(fl_cg* S, const double* r, const double* minv, double* z, double* p, void* stream) {
  FL_CG_CALL(r && minv && z && p, cg_begin(S, r, minv, z, p, st))
}
int32_t fl_cg_init(fl_cg* S, const double* all_parts, void* stream) {
  FL_CG_CALL(all_parts, cg_init(S, all_parts, st))
}
int32_t fl_cg_matvec_diag(fl_cg* S, const fl_dense* A, const double* p_local, void* stream) {
  FL_CG_CALL(A && p_local, (cg_check_rows(S, A), cg_matvec_diag(S, A->A.p, A->lda, p_local, st)))
}
int32_t fl_cg_matvec_rest(fl_cg* S, const fl_dense* A, const double* p_full, const double* p_local, double* Ap,
                          void* stream) {
  FL_CG_CALL(A && p_full && p_local && Ap, (cg_check_rows(S, A), cg_matvec_rest(S, A->A.p, A->lda, p_full, p_local, Ap, st)))
}
int32_t fl_cg_dot_parts(fl_cg* S, const double* a, const double* b, void* stream) {
  FL_CG_CALL(a && b, cg_dot_parts(S, a, b, st))
}
int32_t fl_cg_alpha_update(fl_cg* S, const double* all_parts, double* x, double* r, double* z, const double* p,
                           const double* Ap, const double* minv, void* stream) {
  FL_CG_CALL(all_parts && x && r && z && p && Ap && minv, cg_alpha_update(S, all_parts, x, r, z, p, Ap, minv, st))
}
int32_t fl_cg_beta_xpby(fl_cg* S, const double* all_parts, const double* z, double* p, void* stream) {
  FL_CG_CALL(all_parts && z && p, cg_beta_xpby(S, all_parts, z, p, st))
}
int32_t fl_cg_poll(fl_cg* S, fl_cg_status* status, void* stream) {
  FL_CG_CALL(status, cg_status(S, status, st))
}
#undef FL_CG_CALL

void fl_cg_free(fl_cg* S) {
  if (!S) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(cg_device(S));
  cg_free(S);
  if (prev >= 0) cudaSetDevice(prev);
}

int32_t fl_debug_orders(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                        const fl_order_params* params, int32_t device, int8_t* cross_k, int8_t* tail_k) {
  FL_API_BEGIN
  if (!mesh || !dofmap || !kernel || !params || !cross_k || !tail_k) return fail(FL_E_ARG, "null argument");
  if (kernel->d != mesh->d || !(kernel->s > 0 && kernel->s < 1)) return fail(FL_E_ARG, "bad kernel");
  FL_CUDA(cudaSetDevice(device));
  OwnedStream os_;
  cudaStream_t st = os_.s;
  StreamScope scope(st);
  // minimal table: the cell rule is needed by upload(); fake a 1-node rule of the right size
  std::vector<int64_t> dir(NTOPO * KDIR * 2, 0);
  const int q = mesh->d == 1 ? 6 : 16;
  std::vector<double> data((size_t)q * NODE, 0.0);
  dir[2 * (T_CELL * KDIR + 0) + 1] = q;
  fl_tables t{dir.data(), data.data(), (int64_t)data.size()};
  Uploaded U;
  upload(mesh, dofmap, &t, U, st);
  check_valence(U, st);
  const OrderConsts oc = make_order_consts(*params, mesh->d, kernel->s, dofmap->n);
  const int64_t tot = mesh->nc * mesh->nc;
  DBuf<int8_t> ck(tot), tk(tot);
  launch_debug_orders(U.m, oc, ck.p, tk.p, st);
  FL_CUDA(cudaMemcpyAsync(cross_k, ck.p, tot, cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaMemcpyAsync(tail_k, tk.p, tot, cudaMemcpyDeviceToHost, st));
  int herr = 0;
  FL_CUDA(cudaMemcpyAsync(&herr, U.m.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (herr & 2) return fail(FL_E_QUAD, "fast order path disagrees with the exact select_order arithmetic");
  return FL_OK;
  FL_API_END
}

int32_t fl_debug_order_hist(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                            const fl_order_params* params, int32_t device, int64_t* cross_hist, int64_t* tail_hist) {
  FL_API_BEGIN
  if (!mesh || !dofmap || !kernel || !params || !cross_hist || !tail_hist) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(device));
  OwnedStream os_;
  cudaStream_t st = os_.s;
  StreamScope scope(st);
  std::vector<int64_t> dir(NTOPO * KDIR * 2, 0);
  const int q = mesh->d == 1 ? 6 : 16;
  std::vector<double> data((size_t)q * NODE, 0.0);
  dir[2 * (T_CELL * KDIR + 0) + 1] = q;
  fl_tables t{dir.data(), data.data(), (int64_t)data.size()};
  Uploaded U;
  upload(mesh, dofmap, &t, U, st);
  check_valence(U, st);
  const OrderConsts oc = make_order_consts(*params, mesh->d, kernel->s, dofmap->n);
  DBuf<unsigned long long> h(2 * KDIR);
  FL_CUDA(cudaMemsetAsync(h.p, 0, 2 * KDIR * sizeof(unsigned long long), st));
  launch_order_hist(U.m, oc, h.p, h.p + KDIR, st);
  std::vector<unsigned long long> hh(2 * KDIR);
  FL_CUDA(cudaMemcpyAsync(hh.data(), h.p, hh.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  int herr = 0;
  FL_CUDA(cudaMemcpyAsync(&herr, U.m.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if (herr & 2) return fail(FL_E_QUAD, "fast order path disagrees with the exact select_order arithmetic");
  for (int i = 0; i < KDIR; ++i) {
    cross_hist[i] = (int64_t)hh[i];
    tail_hist[i] = (int64_t)hh[KDIR + i];
  }
  return FL_OK;
  FL_API_END
}

int32_t fl_debug_kpow(int32_t d, double s, const double* r2, int64_t n, double* out, int32_t device) {
  FL_API_BEGIN
  if (!r2 || !out || n < 0 || (d != 1 && d != 2 && d != 11 && d != 12)) return fail(FL_E_ARG, "bad argument");
  FL_CUDA(cudaSetDevice(device));
  OwnedStream os_;
  cudaStream_t st = os_.s;
  StreamScope scope(st);
  DBuf<double> a(std::max<int64_t>(n, 1)), b(std::max<int64_t>(n, 1));
  FL_CUDA(cudaMemcpyAsync(a.p, r2, n * sizeof(double), cudaMemcpyHostToDevice, st));
  const int dd = d == 11 ? 1 : (d == 12 ? 2 : d);
  launch_kpow_probe(d, e4_of(dd, s), a.p, n, -(dd / 2.0 + s), b.p, st);
  FL_CUDA(cudaMemcpyAsync(out, b.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
  FL_API_END
}

int32_t fl_probe_fp64_peak(int32_t device, double* tflops) {
  FL_API_BEGIN
  if (!tflops) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(device));
  OwnedStream os_;
  cudaStream_t st = os_.s;
  StreamScope scope(st);
  *tflops = probe_fp64_tflops(st);
  return FL_OK;
  FL_API_END
}

int32_t fl_debug_touching(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                          const fl_order_params* params, int32_t device, int64_t* npairs, int64_t* pairs,
                          int32_t* topo, int32_t* k, int32_t* ident_k) {
  FL_API_BEGIN
  if (!mesh || !dofmap || !kernel || !params || !npairs) return fail(FL_E_ARG, "null argument");
  FL_CUDA(cudaSetDevice(device));
  OwnedStream os_;
  cudaStream_t st = os_.s;
  StreamScope scope(st);
  std::vector<int64_t> dir(NTOPO * KDIR * 2, 0);
  const int q = mesh->d == 1 ? 6 : 16;
  std::vector<double> data((size_t)q * NODE, 0.0);
  dir[2 * (T_CELL * KDIR + 0) + 1] = q;
  fl_tables t{dir.data(), data.data(), (int64_t)data.size()};
  Uploaded U;
  upload(mesh, dofmap, &t, U, st);
  check_valence(U, st);
  const OrderConsts oc = make_order_consts(*params, mesh->d, kernel->s, dofmap->n);
  DBuf<TouchPair> tp;
  DBuf<int> ik;
  int64_t np = 0;
  classify_touching(U.m, oc, tp, np, ik, st);
  FL_CUDA(cudaStreamSynchronize(st));
  const int64_t cap = *npairs;
  *npairs = np;
  if (pairs && topo && k && cap >= np) {
    std::vector<TouchPair> h(np);
    if (np) FL_CUDA(cudaMemcpy(h.data(), tp.p, np * sizeof(TouchPair), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < np; ++i) {
      pairs[2 * i] = h[i].c0;
      pairs[2 * i + 1] = h[i].c1;
      topo[i] = h[i].topo;
      k[i] = h[i].k;
    }
    if (ident_k) FL_CUDA(cudaMemcpy(ident_k, ik.p, mesh->nc * sizeof(int), cudaMemcpyDeviceToHost));
  }
  return FL_OK;
  FL_API_END
}

}  // extern "C"
