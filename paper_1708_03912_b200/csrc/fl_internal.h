// Internal host-side declarations shared by the fraclap_b200 translation units.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "fl_device.cuh"

namespace fl {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FL_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::fl::Error(e_ == cudaErrorMemoryAllocation ? -6 : -5,                     \
                        std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)

#define FL_CHECK_LAUNCH() FL_CUDA(cudaGetLastError())

// Host-side count of kernel launches issued by this library (fl_launch_count()).
long long& launch_counter();
inline void note_launch(long long k = 1) { launch_counter() += k; }

// The stream the current API call works on; device buffers are allocated and released
// stream-ordered from the device's memory pool (no device-wide sync on free).
cudaStream_t& cur_stream();
void init_pool(int device);

// Recycled non-blocking streams per device (fl_capi.cu); a lease returns its stream on scope exit
// (declare it before the buffers allocated on it, so their stream-ordered frees come first).
cudaStream_t acquire_stream(int device);
void release_stream(int device, cudaStream_t s);
struct OwnedStreamLease {
  int dev;
  cudaStream_t s;
  explicit OwnedStreamLease(int d) : dev(d), s(acquire_stream(d)) {}
  ~OwnedStreamLease() { release_stream(dev, s); }
  OwnedStreamLease(const OwnedStreamLease&) = delete;
  OwnedStreamLease& operator=(const OwnedStreamLease&) = delete;
};

// Makes `device` current for the scope of an API call and restores the caller's device on exit.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    FL_CUDA(cudaSetDevice(device));
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(cur_stream()) { cur_stream() = s; }
  ~StreamScope() { cur_stream() = prev; }
};

// Device buffer with RAII.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DBuf() = default;
  explicit DBuf(size_t cnt) { alloc(cnt); }
  void alloc(size_t cnt) {
    free();
    n = cnt;
    st = cur_stream();
    if (cnt) FL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), cnt * sizeof(T), st));
  }
  void free() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    free();
    p = o.p; n = o.n; st = o.st; o.p = nullptr; o.n = 0;
    return *this;
  }
};

// Device view of the mesh + derived per-cell data (all int32 indices; nv, nc < 2^31).
struct DevMesh {
  int d = 0, nv = 0, nc = 0, nb = 0, n = 0, q = 0;
  const double* vert = nullptr;    // nv*d
  const int* cells = nullptr;      // nc*(d+1)
  const int* v2d = nullptr;        // nv
  const int* bedges = nullptr;     // nb*d
  const double* bnorm = nullptr;   // nb*d (outward)
  const CellGeo* geo = nullptr;    // nc
  const int* patch_off = nullptr;  // nv+1
  const int* patch_cells = nullptr;// nc*(d+1), ascending cell id per vertex (mesh.py:114-125)
  const double* X = nullptr;       // nc*q*d  cell quadrature nodes (assembly.py:292-298)
  const double* W = nullptr;       // nc*q
  int* err = nullptr;              // device error word (bit 0: a quadrature rule was missing)
};

struct DevTables {
  const double* data = nullptr;
  RuleRef dir[NTOPO * KDIR];
  __host__ __device__ RuleRef rule(int topo, int k) const { return dir[topo * KDIR + k]; }
};

// Touching pair record (assembly.py:412-473 + the order of :680).
struct TouchPair {
  int c0, c1;       // c0 < c1  (sorted unordered pair)
  int topo;         // T_CE / T_CV
  int k;
  int vK[3], vK2[3];// canonical vertex orders
  int locs[5];      // global vertex behind each local basis slot
  int nloc;
};

// Boundary (cell, edge) singular pair (assembly.py:796-841).
struct BndPair {
  int cell, edge, topo, k;
  int locs[3];      // canonical cell vertex order
  int nloc;
  double pe[2][2];  // canonical edge points (1D: pe[0][0])
  double ne[2];     // INWARD normal (assembly.py:792)
};

// ------------------------------------------------------------ launchers (by file)
// fl_prep.cu
void launch_prep_cells(const DevMesh& m, CellGeo* geo, cudaStream_t st);
void launch_cell_nodes(const DevMesh& m, const DevTables& t, double* X, double* W, cudaStream_t st);
void build_patches(int nv, int nc, int d, const int* cells, DBuf<int>& off, DBuf<int>& data,
                   cudaStream_t st);
void touching_count(const DevMesh& m, DBuf<int>& counts, DBuf<int>& offs, cudaStream_t st);
void touching_fill(const DevMesh& m, const OrderConsts& oc, const DBuf<int>& offs, int64_t total,
                   DBuf<TouchPair>& pairs, DBuf<int>& ident_k, cudaStream_t st);
void boundary_count(const DevMesh& m, DBuf<int>& counts, DBuf<int>& offs, cudaStream_t st);
void boundary_fill(const DevMesh& m, const OrderConsts& oc, const DBuf<int>& offs, int64_t total,
                   DBuf<BndPair>& items, cudaStream_t st);
void launch_max_valence(const int* off, int nv, int* mx, cudaStream_t st);
void classify_touching(const DevMesh& m, const OrderConsts& oc, DBuf<TouchPair>& pairs,
                       int64_t& npairs, DBuf<int>& ident_k, cudaStream_t st);
void classify_boundary(const DevMesh& m, const OrderConsts& oc, DBuf<BndPair>& items,
                       int64_t& nitems, cudaStream_t st);
// DoF tiles of TILE dofs in Morton order; per tile the sorted id list of cells that
// touch one of its DoFs, with the tile-local slot of each cell vertex.
constexpr int TILE = 64;
constexpr int TILE_MAXC = 256;
constexpr int MAX_VALENCE = 12;   // cells around one vertex (cross-tile row lists)
struct Tiles {
  int ntiles = 0;
  DBuf<int> dofs;     // ntiles*TILE (-1 pad)
  DBuf<int> ncell;    // ntiles
  DBuf<int> cells;    // ntiles*TILE_MAXC
  DBuf<int> slots;    // ntiles*TILE_MAXC*3 (-1: vertex not a DoF of this tile)
  DBuf<double> geo3;  // ntiles*3: centre (x, y) and radius of the tile's DoF vertices
  DBuf<double> stat;  // ntiles*8: centre (x, y), R = max |c_K - centre| + rad_K, h min/max, |ln h| min/max
};

// Tile pairs of the cross term, heavy first (sorted by the tile gap), and the subset that can
// hold near pairs (a rigorous upper bound of the disjoint order formula reaches KW).
struct TilePairs {
  DBuf<int2> all, near;
  int nall = 0, nnear = 0;
  int64_t near_candidates = 0;   // sum of nR * nC over `near`: bound of the discovery's near keys
};
void build_tile_pairs(const DevMesh& m, const OrderConsts& oc, const Tiles& rows, const Tiles& cols, bool symmetric,
                      int kw, TilePairs& tp, cudaStream_t st);
void build_tiles(const DevMesh& m, int row_begin, int row_end, Tiles& t, cudaStream_t st);

// fl_singular.cu
void launch_singular_touching(const DevMesh& m, const DevTables& t, double ex, int e4,
                              const TouchPair* pairs, int64_t npairs, double* out /*npairs*25*/,
                              cudaStream_t st);
void launch_singular_identical(const DevMesh& m, const DevTables& t, double ex, int e4,
                               const int* ident_k, double* out /*nc*9*/, cudaStream_t st);
void launch_singular_boundary(const DevMesh& m, const DevTables& t, double ex, int e4,
                              const BndPair* items, int64_t nitems, double* out /*nitems*9*/,
                              cudaStream_t st);

// fl_far.cu
void launch_tail(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                 const int* targets, int ntargets, double* psi /*nc*q*/, unsigned long long* evals,
                 cudaStream_t st, const int8_t* kuni = nullptr, const int* blk_of = nullptr,
                 const int* bcells = nullptr, int nb = 0, const int8_t* kcell = nullptr,
                 const unsigned long long* psifx = nullptr, double fxinv = 0.0,
                 const double* ujh = nullptr, const double* wh = nullptr, const double2* un = nullptr,
                 const double2* uhi = nullptr);
void launch_flux(const DevMesh& m, const DevTables& t, double ex, int e4, const int* targets,
                 int ntargets, double* win /*nc*q*/, cudaStream_t st);
void launch_cross_tiles(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex,
                        int e4, double Cds, const Tiles& rows, const Tiles& cols, const int2* tpairs, int ntp,
                        bool symmetric, int row_begin, int row_end, double* A, int64_t lda,
                        unsigned long long* evals, unsigned long long* near_keys,
                        unsigned int* near_count, unsigned int near_cap, int discover,
                        const unsigned long long* nearH, const int* nearI, unsigned long long hmask,
                        const double* nearG, cudaStream_t st);
// fl_near.cu: near disjoint pairs (order >= KW) collected by the cross tiles, one block each
constexpr int KW2D = 5, KW1D = 12;
// near-pair key: (min cell << 34) | (max cell << 6) | k  (cells < 2^28, k <= 32): sorting by key
// is sorting by the reference's (min, max) orientation
__host__ __device__ inline unsigned long long near_key(int a, int b, int k) {
  const unsigned long long lo = (unsigned)(a < b ? a : b), hi = (unsigned)(a < b ? b : a);
  return (lo << 34) | (hi << 6) | (unsigned long long)k;
}
__host__ __device__ inline unsigned long long near_hash(unsigned long long x) {   // splitmix64 finaliser
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
constexpr unsigned long long NEAR_EMPTY = ~0ull;

struct NearPairs {
  int64_t n = 0;
  DBuf<unsigned long long> U;           // sorted unique keys (near_key)
  DBuf<int> P, Q, K;                    // the two cells and the order of each key
  DBuf<double> G;                       // n*9: M^{P,Q} (cross_matrices orientation)
  DBuf<unsigned long long> hkey;        // open-addressing table key -> index (linear probing)
  DBuf<int> hidx;
  unsigned long long hmask = 0;
};
void near_pairs_build(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                      unsigned long long* keys, int64_t nkeys, NearPairs& np, unsigned long long* evals,
                      cudaStream_t st);
// fl_cross2d.cu: the 2D cross term by cell-block pairs, exact fixed-point accumulation
struct Cross2DInfo {
  int scale_exp = 0;          // contributions are accumulated as integers of 2^-scale_exp
  double dmin = 0.0;          // smallest disjoint cell distance
  int64_t block_pairs = 0, near_block_pairs = 0;
  int fallback = 0;           // 1: the fixed-point unit is too coarse for this mesh, nothing was added to A
                              // (the caller runs the DoF-tile cross kernel instead)
};
// Morton blocks of CB2D cells (sorted along the Morton curve of the centroids): per block its
// cells, the sorted DoFs of its cells (<= 64) with each cell vertex's slot, a bounding circle and
// h / |ln h| ranges (bstat: cx cy R hmin hmax lmin lmax), whether it holds a DoF of the row range;
// blk_of: the block of every cell.  Shared by the cross term and the tail.
constexpr int CB2D = 32;
struct Blocks2D {
  int nb = 0;
  DBuf<int> bcells, bdofs, bndof, rowflag, err, blk_of;
  DBuf<signed char> slot;
  DBuf<double> bstat;
  // mapped nodes of the orders 2, 3, 4: per cell (29 each), and per block node-major
  // (un[b][seg(k) + r * 32 + c], seg = 0 / 128 / 416, 928 per block) with J and packed vertex slots
  DBuf<double2> nodes, un;
  DBuf<double> uj;
  DBuf<int> us;
  DBuf<uint4> ucol;       // per block and DoF slot: count + (cell slot * 3 + vertex) entries, 16 bytes
  double dmin = 1e300;    // smallest distance of two cells sharing no vertex (second-ring scan)
  double jmax = 0.0;      // largest Jacobian
  double radmax = 0.0;    // largest cell radius (vertex - centroid)
  double beta = 0.0;      // max_K J_K^2 d_K^(-(d+2s)), d_K the smallest distance from K to a cell sharing no vertex
};
constexpr int UNODES2D = 928;
// the 2D tail's staging array of the orders 5-9: per block 32 * (25 + 36 + 49 + 64 + 81) nodes
constexpr int UHI2D = 8160;
__host__ __device__ constexpr int uhi_seg(int k) {
  return k == 5 ? 0 : (k == 6 ? 800 : (k == 7 ? 1952 : (k == 8 ? 3520 : 5568)));
}
static_assert(uhi_seg(6) == 32 * 25 && uhi_seg(7) == uhi_seg(6) + 32 * 36 && uhi_seg(8) == uhi_seg(7) + 32 * 49 &&
                  uhi_seg(9) == uhi_seg(8) + 32 * 64 && UHI2D == uhi_seg(9) + 32 * 81,
              "uhi segments: 32 k^2 nodes per order");
static_assert(disj_roff(2) == 0 && disj_roff(3) == 4 && disj_roff(10) == DISJ_RULE_NODES, "disjoint rule offsets");

// Exact range, over the 32 x 32 cell pairs of Morton blocks P and Q, of the distance estimate that
// select_order is fed (assembly.py:764-781): every pair's estimate lies in [lo, hi] with
// lo = min (|cK - cL| - (rK + rL)) (the estimate of a close pair is the exact triangle distance,
// >= that) and hi = max of the same value, or |cK - cL| for a close pair (the triangles hold their
// centroids, so their distance is <= it).  The block bounding circles give only
// dc -+ (R_P + R_Q); these exact values let the order bounds prove one order for more block pairs.
// Warp-cooperative (every lane returns the result); empty slots of partial blocks are skipped.
// Symmetric in (P, Q) bitwise: (-d)^2 == d^2 and rK + rL == rL + rK.
__device__ __forceinline__ void block_pair_dist_range(const DevMesh& m, const int* __restrict__ bcells, int P, int Q,
                                                      int lane, double& lo, double& hi) {
  const int cp = bcells[P * CB2D + lane], cq = bcells[Q * CB2D + lane];
  double px = 0.0, py = 0.0, pr = 0.0, qx = 0.0, qy = 0.0, qr = 0.0;
  if (cp >= 0) { const CellGeo& g = m.geo[cp]; px = g.cx; py = g.cy; pr = g.rad; }
  if (cq >= 0) { const CellGeo& g = m.geo[cq]; qx = g.cx; qy = g.cy; qr = g.rad; }
  const unsigned qvalid = __ballot_sync(0xffffffffu, cq >= 0);
  double l = 1e300, h = -1e300;
  for (int j = 0; j < CB2D; ++j) {
    const double x = __shfl_sync(0xffffffffu, qx, j), y = __shfl_sync(0xffffffffu, qy, j);
    const double r = __shfl_sync(0xffffffffu, qr, j);
    if (cp < 0 || !((qvalid >> j) & 1u)) continue;
    const double dx = __dsub_rn(px, x), dy = __dsub_rn(py, y);
    const double dc = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    const double rr = __dadd_rn(pr, r);
    const double low = __dsub_rn(dc, rr);
    l = fmin(l, low);
    h = fmax(h, low < 2.0 * rr ? dc : low);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
    h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
  }
  lo = l;
  hi = h;
}
// One order for every cell pair of blocks a, b (bstat records: cx cy R hmin hmax |ln h|min
// |ln h|max) whose distance estimates lie in [Dmin, Dmax], or 0: the rigorous bounds of the order
// formula (coff = C_offset or C_offset - 4) with 1e-9 margins around the ceil.
__device__ __forceinline__ int block_uniform_order(const OrderConsts& oc, double coff, double Dmin, double Dmax,
                                                   const double* a, const double* b) {
  if (!(Dmin > 0.0)) return 0;
  const double hmn = fmin(a[3], b[3]), hmx = fmax(a[4], b[4]), lmn = fmin(a[5], b[5]), lmx = fmax(a[6], b[6]);
  const double hi = order_bound_hi(oc, coff, Dmin, hmn, hmx, lmn, lmx);
  const double lo = order_bound_lo(oc, coff, Dmin, Dmax, hmn, hmx, lmn, lmx);
  const double c0 = fmin(fmax(ceil(lo - 1e-9), 2.0), (double)oc.cap_disjoint);
  const double c1 = fmin(fmax(ceil(hi + 1e-9), 2.0), (double)oc.cap_disjoint);
  return c0 == c1 ? (int)c0 : 0;
}
void build_blocks2d(const DevMesh& m, const DevTables& t, double e /* d + 2s */, int row_begin, int row_end,
                    Blocks2D& B, cudaStream_t st);
void assemble_cross2d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                      const Blocks2D& B, int row_begin, int row_end, double* A, int64_t lda,
                      unsigned long long* evals, NearPairs& near, Cross2DInfo& info, cudaEvent_t t_disc,
                      cudaEvent_t t_near, cudaStream_t st, unsigned long long* evals_near = nullptr);
// fl_tail2d.cu: the 2D tail by Morton block pairs.  Per ordered (target block, source block) the
// rigorous bounds of the boosted order formula either prove one order for all 32 x 32 cell pairs
// (kuni, the source block's nodes are evaluated against all 512 target nodes of the block) or
// not (0: the warp-per-target tail_kernel evaluates those source blocks pair by pair and adds).
void launch_tail2d_blocks(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                          const Blocks2D& B, const int* targets, int ntargets, double* psi,
                          unsigned long long* evals, cudaStream_t st, unsigned long long* evals_block = nullptr,
                          cudaEvent_t e0 = nullptr, cudaEvent_t e1 = nullptr,
                          unsigned long long* evals_sym = nullptr);
void launch_debug_orders(const DevMesh& m, const OrderConsts& oc, int8_t* cross_k, int8_t* tail_k,
                         cudaStream_t st);
// fl_far1d.cu (1D: lean tail, packed pair-block cross + gather)
struct Plan1D;   // 1D far-field mesh data (fl_far1d.cu), built without host synchronisation
Plan1D* plan1d_create(const DevMesh& m, const int* dof_vertex, bool symmetric, int row_begin, int row_end,
                      cudaStream_t st);
void plan1d_free(Plan1D* P);
const int* plan1d_maxcells(const Plan1D* P);   // device: max cells behind one DoF tile
void launch_tail1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, const Plan1D* P,
                   const int* targets, const int* d_ntargets, int ntargets_ub, double* psi,
                   unsigned long long* evals, cudaStream_t st);
bool cross1d_fits(const DevMesh& m, int64_t ntargets, bool symmetric);
// band_row0 < band_row1 (tile-aligned start): only the upper-triangular tile pairs whose row tile
// lies in that DoF row band (needs the fused tiles: cross1d_fused)
bool launch_cross1d(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                    const Plan1D* P, int maxcells, const int* targets, int ntargets, const int* dof_vertex,
                    double* A, int64_t lda, unsigned long long* evals, cudaStream_t st, int band_row0 = 0,
                    int band_row1 = 0);
bool cross1d_fused(const Plan1D* P, int maxcells);
int cross1d_tile_dofs();
void launch_order_hist(const DevMesh& m, const OrderConsts& oc, unsigned long long* hc, unsigned long long* ht,
                       cudaStream_t st);
double probe_fp64_tflops(cudaStream_t st);
void launch_kpow_probe(int d, int e4, const double* x, int64_t n, double ex, double* out, cudaStream_t st);

// fl_local.cu
void launch_cell_local(const DevMesh& m, const DevTables& t, double Cds, double s, bool integral,
                       const int* targets, int ntargets, const double* ident, const double* psi,
                       const double* win, double* Lc /*nc*9*/, cudaStream_t st);
struct SparseIndex {
  DBuf<int> tp_first_off, tp_second_off, tp_second;   // touching pairs by first / second cell
  DBuf<int> bp_off, bp_idx;                           // boundary items by cell
};
void build_sparse_index(const DevMesh& m, const TouchPair* pairs, int64_t npairs,
                        const BndPair* items, int64_t nitems, SparseIndex& si, cudaStream_t st);
void launch_sparse_pull(const DevMesh& m, double Cds, double s, const double* Lc,
                        const TouchPair* pairs, const double* tloc, const BndPair* items,
                        const double* bloc, const SparseIndex& si, const int* row_vertex,
                        int row_begin, int row_end, double* A, int64_t lda, cudaStream_t st);

// fl_mesh.cu (host O(n) driver steps on the device)
int32_t finish_polygon_mesh(const double* V, int64_t nv, const int64_t* cells_in, int64_t nc, int device,
                            int64_t* cells_out, int64_t* be_out, double* bn_out, int64_t cap, int64_t* nb_out);
int32_t dofmap_build(const int64_t* be, int64_t nb, int d, int64_t nv, double s, int device, int64_t* v2d_out,
                     int64_t* n_out);
}  // namespace fl
struct fl_mesh;
struct fl_dofmap;
namespace fl {
int32_t cell_rule_nodes(const ::fl_mesh* mesh, const double* pts, int64_t q, int device, double* X_out);
int32_t load_vector(const ::fl_mesh* mesh, const ::fl_dofmap* dm, const double* pts, const double* w, int64_t q,
                    const double* fvals, double fconst, int device, double* b_out);

// the same pull into CSR rows 0..nrows-1 (sorted column indices covering every local entry)
void launch_sparse_pull_csr(const DevMesh& m, double Cds, double s, const double* Lc, const TouchPair* pairs,
                            const double* tloc, const BndPair* items, const double* bloc, const SparseIndex& si,
                            const int* row_vertex, int nrows, const int64_t* indptr, const int* indices,
                            double* data, cudaStream_t st);

// fl_near.cu: one block per (P, Q, K) pair (warp per pair), G = n x 9 in the (P, Q) orientation
void launch_near_blocks(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4,
                        const int* P, const int* Q, const int* K, int64_t n, double* G, unsigned long long* evals,
                        cudaStream_t st);

// fl_nearfield.cu: the near-field (cluster) assembly, assemble_near_field (assembly.py:860-970)
struct NearField;   // device CSR + work buffers
struct NearInput {
  int nleaves = 0;
  int64_t npairs = 0;
  const int* leaf_of_dof = nullptr;  // device (n)
  const int* pairs = nullptr;        // device (npairs*2), a <= b
  const double* V = nullptr;         // device (nc*q) boundary flux potential, or null: direct GL8
};
struct CsrOut {
  DBuf<int64_t> indptr;
  DBuf<int> indices;
  DBuf<double> data;
  int64_t nnz = 0;
};
// psi = (V - ring flux of N(K)) / (2s) and win = T - V at the cell nodes (tail_potential,
// ring_boundaries, assembly.py:336-396, :1074-1094)
void launch_ring_tail(const DevMesh& m, const DevTables& t, double s, double ex, int e4, const double* Vgiven,
                      bool integral, double* psi, double* win, cudaStream_t st);
// near disjoint cell pairs of the leaf pairs, their blocks, the CSR pattern and the cross values
void near_field_cross(const DevMesh& m, const DevTables& t, const OrderConsts& oc, double ex, int e4, double Cds,
                      const NearInput& in, const int* row_vertex, CsrOut& out, int64_t* npairs_out,
                      unsigned long long* evals, cudaStream_t st);

// fl_cluster.cu: the cluster (H-matrix) operator
}  // namespace fl
struct fl_cluster;
struct fl_cg;
struct fl_cg_status;
struct fl_cluster_desc;
namespace fl {
int32_t cluster_create(const ::fl_cluster_desc* D, int device, ::fl_cluster** out);
int32_t cluster_matvec_dev(::fl_cluster* C, const double* x, double* y, double* yfar, cudaStream_t st);
void cluster_far_points(::fl_cluster* C, const double* u_dev, int64_t npts, const double* X_dev,
                        const int64_t* owner_dev, double* out_dev, cudaStream_t st);
// sets fl_last_error() and returns code (fl_capi.cu)
int32_t api_fail(int code, const char* msg);

// fl_solve.cu
constexpr int VCH = 512;   // fixed global vector chunk of every solve reduction; row blocks are multiples of it
void launch_matvec(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, double* y,
                   cudaStream_t st);
void launch_diag(const double* A, int64_t rows, int64_t row0, int64_t lda, double* d, cudaStream_t st);
struct PcgResult {
  long long it;
  double rz, norm0;
  int converged, error;
};
PcgResult run_pcg(const double* A, int64_t n, int64_t lda, const double* minv, double* x, double* r, double* z,
                  double* p, double* Ap, double tol, long long max_iter, bool have_x0, cudaStream_t st);
fl_cg* cg_create(int64_t n, int64_t m, int64_t blk, int world, int rank, double tol, long long max_iter, int device);
void cg_begin(fl_cg* S, const double* r, const double* minv, double* z, double* p, cudaStream_t st);
void cg_init(fl_cg* S, const double* parts, cudaStream_t st);
void cg_matvec_diag(fl_cg* S, const double* A, int64_t lda, const double* x_local, cudaStream_t st);
void cg_matvec_rest(fl_cg* S, const double* A, int64_t lda, const double* x_full, const double* p_local,
                    double* Ap, cudaStream_t st);
void cg_dot_parts(fl_cg* S, const double* a, const double* b, cudaStream_t st);
void cg_alpha_update(fl_cg* S, const double* parts, double* x, double* r, double* z, const double* p,
                     const double* Ap, const double* minv, cudaStream_t st);
void cg_beta_xpby(fl_cg* S, const double* parts, const double* z, double* p, cudaStream_t st);
void cg_status(fl_cg* S, fl_cg_status* out, cudaStream_t st);
double* cg_local_parts(fl_cg* S);
void cg_bind_parts(fl_cg* S, double* ext);
double* cg_all_parts(fl_cg* S);
int64_t cg_chunks(fl_cg* S);
void cg_free(fl_cg* S);
int cg_device(const fl_cg* S);
void cg_info(const fl_cg* S, int* device, int64_t* n, int64_t* row0, int64_t* m);
constexpr int DOT_BLOCKS = 296;   // 2 x 148 SMs; fixed => deterministic reduction tree

}  // namespace fl
