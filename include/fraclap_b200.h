/*
 * fraclap_b200 — C ABI of the B200 (sm_100a) implementation of the dense hot path of
 * Ainsworth & Glusa's FEM for the integral fractional Laplacian (reference package
 * `fraclap`, /root/reference/pkg/src/fraclap).
 *
 * The path:  assemble_dense (assembly.py:1059-1104)  ->  pcg with the dense matvec
 *            `lambda x: Ad @ x` (solve.py:27-32, 52-109).
 *
 * Conventions
 *   - Plain pointers + int64 sizes, row-major, no torch types.  Host arrays are BORROWED
 *     for the duration of a call.  `fl_dense` OWNS its device matrix and workspaces.
 *   - Every entry point returns 0 (FL_OK) or a negative FL_E_* code; `fl_last_error()`
 *     returns a thread-local message for the last failure.  No partial outputs on error.
 *   - The mapping of codes onto the reference's exceptions is 1:1:
 *       FL_E_ARG      -> ValueError      (assembly.py:59-60, mesh.py:208-209)
 *       FL_E_ASSEMBLY -> AssemblyError   (assembly.py:1062-1063, :871)
 *       FL_E_QUAD     -> QuadratureError (quadrature.py:157-158, :405-406)
 *       FL_E_SOLVER   -> SolverError     (solve.py:67-68, :87-88)
 *       FL_E_CUDA / FL_E_OOM -> RuntimeError
 */
#ifndef FRACLAP_B200_H
#define FRACLAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_ABI_VERSION 1

#define FL_OK 0
#define FL_E_ARG (-1)
#define FL_E_ASSEMBLY (-2)
#define FL_E_QUAD (-3)
#define FL_E_SOLVER (-4)
#define FL_E_CUDA (-5)
#define FL_E_OOM (-6)

/* kernel variants (assembly.py:47-50) */
#define FL_VARIANT_INTEGRAL 0
#define FL_VARIANT_REGIONAL 1
#define FL_VARIANT_SYMMETRIZED 2 /* refused with FL_E_ASSEMBLY: out of scope */

/* rule-table topologies (quadrature.py:38-46) plus the two per-cell rules */
#define FL_TOPO_IDENTICAL 0
#define FL_TOPO_COMMON_EDGE 1
#define FL_TOPO_COMMON_VERTEX 2
#define FL_TOPO_DISJOINT 3      /* ONE-cell simplex_rule(d,k) (quadrature.py:81-85) */
#define FL_TOPO_EDGE_OF_CELL 4
#define FL_TOPO_TOUCHING_EDGE 5
#define FL_TOPO_CELL 6          /* cell rule XQ_ORDER[d] (assembly.py:282-298, :635) */
#define FL_TOPO_EDGE_GL 7       /* GL rule of order EDGE_GL_ORDER on [0,1] (assembly.py:43) */
#define FL_NTOPO 8
#define FL_KDIR 33              /* k = 0..32 (K_MAX = 32, quadrature.py:35) */
#define FL_NODE_STRIDE 8        /* doubles per packed node record */

/* Mesh input contract (mesh.py:24-197).  `boundary_normals` are OUTWARD unit normals. */
typedef struct fl_mesh {
  int32_t d;                        /* 1 or 2 */
  int32_t pad_;
  int64_t nv, nc, nb;
  const double* vertices;           /* (nv, d) */
  const int64_t* cells;             /* (nc, d+1); in 2D CCW with the refinement edge first */
  const int64_t* boundary_edges;    /* (nb, d) */
  const double* boundary_normals;   /* (nb, d) outward */
} fl_mesh;

/* DofMap (mesh.py:200-240): vertex -> dof, -1 for a non-DoF vertex. */
typedef struct fl_dofmap {
  int64_t n;
  const int64_t* vertex_to_dof;     /* (nv,) */
} fl_dofmap;

/* FractionalKernel (assembly.py:66-94).  C_ds = normalisation(d, s) (assembly.py:57-63). */
typedef struct fl_kernel {
  int32_t d;
  int32_t variant;
  double s;
  double C_ds;
} fl_kernel;

/* OrderParams (quadrature.py:115-131) with alpha already resolved by target_alpha(d, s). */
typedef struct fl_order_params {
  double rho1, rho2, rho3, rho4;
  double C_offset;
  double alpha;
} fl_order_params;

/* Packed quadrature tables, built host-side from the same Gauss-Legendre / Gauss-Jacobi
 * node sets the reference uses (quadrature.py:53-420).  `dir` has FL_NTOPO*FL_KDIR*2 int64:
 * dir[2*(topo*FL_KDIR+k)+0] = first node, dir[...+1] = node count (0: rule absent).  Node
 * records are FL_NODE_STRIDE doubles in `data`:
 *   IDENTICAL / COMMON_EDGE / COMMON_VERTEX : x0 x1 y0 y1 w           (1D: x y in slots 0/2)
 *   EDGE_OF_CELL / TOUCHING_EDGE            : x0 x1 a w               (1D: x in slot 0)
 *   DISJOINT (one cell, order k)            : u0 u1 w lw0 lw1 lw2     (lw_a = lambda_a(u) w)
 *   CELL                                    : u0 u1 w lam0 lam1 lam2
 *   EDGE_GL                                 : t w
 * IDENTICAL 1D and EDGE_OF_CELL 1D ignore k and are stored at k = 0. */
typedef struct fl_tables {
  const int64_t* dir;
  const double* data;
  int64_t ndata;                    /* doubles in data */
} fl_tables;

typedef struct fl_dense fl_dense;   /* opaque: device rows [row_begin,row_end) x n of A */
typedef struct fl_sparse fl_sparse; /* opaque: device CSR (n x n), the near-field matrix */

/* The near-field leaf-pair structure of the cluster tree (cluster.NearStructure,
 * cluster.py:743-777): every DoF's leaf index and the unordered near leaf pairs. */
typedef struct fl_near_structure {
  int64_t nleaves;
  const int64_t* leaf_of_dof;       /* (n,) leaf index in [0, nleaves) (NearStructure.leaf_idx_of_dof) */
  int64_t npairs;
  const int64_t* pairs;             /* (npairs, 2) near leaf pairs (nl_pairs as leaf indices) */
} fl_near_structure;

typedef struct fl_solve_report {
  int64_t iterations;
  double residual;                  /* sqrt|r.z| / sqrt|r0.z0| (solve.py:104) */
  double seconds;
  int32_t converged;
  int32_t pad_;
  double true_residual;             /* ||b - A x|| / ||b||, reported beside the reference's */
} fl_solve_report;

typedef struct fl_assembly_stats {
  /* element-pair quadratures, counted as the reference does */
  int64_t pairs_identical, pairs_touching, pairs_cross, pairs_tail;
  int64_t pairs_boundary_singular, pairs_boundary_flux;
  /* kernel evaluations (quadrature node pairs) actually performed */
  double evals_cross, evals_tail, evals_singular, evals_boundary;
  /* device milliseconds per phase (CUDA events on the assembly stream) */
  double ms_prep, ms_singular, ms_tail, ms_flux, ms_tiles, ms_cross, ms_local, ms_total;
  int64_t cross_tile_pairs;
  int32_t ncolors, ntiles;
  /* cross term split: discovery pass (orders only), near blocks, compute pass; near pair count */
  double ms_discover, ms_near, ms_cross_compute;
  int64_t near_pairs;
  /* pairs whose pre-ceil Gauss order lay within 1e-12 of an integer (recomputed with a
   * correctly rounded log; SURVEY.md §8(d) k-flip guard) */
  int64_t order_ties;
  /* 2D cross term: contributions accumulated as integers of 2^-cross_scale_exp (exact, order-free) */
  int32_t cross_scale_exp, cross_fallback; /* cross_fallback = 1: the 2D fixed-point cross accumulation was too coarse for this mesh, the DoF-tile kernel assembled the cross term */
  /* 2D: the part of evals_tail done by the block-pair tail kernel and its device ms; the part of
   * evals_cross done by the near blocks (k >= 5, ms_near) */
  double evals_tail_block, ms_tail_block, evals_near;
  /* 2D: the part of evals_tail_block swept for an order-4 block pair once for both directions
   * (each such evaluation also adds to the partner cell's psi: 2 more FLOPs) */
  double evals_tail_sym;
} fl_assembly_stats;

/* ---------------------------------------------------------------- library */
int32_t fl_abi_version(void);
const char* fl_last_error(void);
int32_t fl_device_count(void);
/* number of CUDA kernel launches this library has issued so far (graph replays included) */
int64_t fl_launch_count(void);

/* ------------------------------------------------------------- assembly
 * Replaces assembly.assemble_dense (assembly.py:1059-1104) for the rows
 * [row_begin, row_end) of the (n x n) matrix; (0, n) = the whole matrix.
 * n_limit reproduces the refusal at assembly.py:1062-1063 (pass <0 to disable).
 * stream: a cudaStream_t (NULL = the library's own stream). */
int32_t fl_assemble_dense(const fl_mesh* mesh, const fl_dofmap* dofmap,
                          const fl_kernel* kernel, const fl_order_params* params,
                          const fl_tables* tables, int64_t n_limit,
                          int64_t row_begin, int64_t row_end,
                          int32_t device, void* stream, fl_dense** out);

/* The whole (n x n) matrix written straight into host memory `A_host` (row-major, n*n doubles):
 * the ndarray that assembly.assemble_dense returns (assembly.py:1059-1104, :1096-1104).
 * Page-locked A_host copies at full PCIe rate.  On error A_host is left unspecified. */
int32_t fl_assemble_dense_host(const fl_mesh* mesh, const fl_dofmap* dofmap,
                               const fl_kernel* kernel, const fl_order_params* params,
                               const fl_tables* tables, int64_t n_limit, int32_t device,
                               double* A_host);

/* Wrap an existing dense host matrix (n x n, row-major) as a device operator — the
 * `Ad = np.asarray(A)` branch of LinearOperatorHandle.from_matrix (solve.py:31-32). */
int32_t fl_dense_from_host(const double* A, int64_t n, int32_t device, fl_dense** out);
/* rows [row_begin, row_end) of an (n x n) host matrix (row-major, (row_end - row_begin) x n) as a
 * row-block operator, e.g. one rank's block of a matrix assembled elsewhere */
int32_t fl_dense_from_host_rows(const double* rows, int64_t n, int64_t row_begin, int64_t row_end,
                                int32_t device, fl_dense** out);

void fl_dense_free(fl_dense* A);
int32_t fl_dense_info(const fl_dense* A, int64_t* n, int64_t* row_begin, int64_t* row_end,
                      double** device_ptr);
int32_t fl_dense_stats(const fl_dense* A, fl_assembly_stats* stats);
/* copy the owned rows (row-major, (row_end-row_begin) x n) to host memory */
int32_t fl_dense_to_host(const fl_dense* A, double* host_rows);
/* copy selected global rows (each within [row_begin, row_end)) to host, nrows x n */
int32_t fl_dense_rows(const fl_dense* A, int64_t nrows, const int64_t* rows, double* host_out);
/* diagonal entries of the owned rows (host) */
int32_t fl_dense_diag(const fl_dense* A, double* host_diag);

/* ------------------------------------------------------------- near field (cluster path)
 * Replaces assembly.assemble_near_field (assembly.py:860-970): the sparse matrix of every DoF pair
 * (i, j) whose leaves form a near pair — touching / identical singular pairs, the disjoint cross
 * terms of the near leaf pairs' cells, the tail through the one-ring boundary
 * Psi = (V - ring flux)/(2s) (tail_potential / ring_boundaries, :336-396) and, for the integral
 * variant, the boundary pairs and the boundary mass term (:1074-1094).  V_nodes: the boundary
 * flux potential at the (nc, q) cell nodes (cell_quadrature(XQ_ORDER)), e.g. the cluster far
 * field's boundary_flux_at_nodes (cluster.py:525); NULL = direct GL8 over every boundary edge. */
int32_t fl_assemble_near_field(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                               const fl_order_params* params, const fl_tables* tables,
                               const fl_near_structure* near, const double* V_nodes, int32_t device,
                               fl_sparse** out);
/* Diagnostics: Psi = (V - ring flux)/(2s) (tail_potential, assembly.py:388-396) and W_in (:1092)
 * at the (nc, q) cell nodes as the near-field assembly forms them; host arrays of nc*q. */
int32_t fl_debug_ring_tail(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                           const fl_order_params* params, const fl_tables* tables, const double* V_nodes,
                           int32_t device, double* psi_out, double* win_out);
/* n, stored entries, and the number of distinct disjoint cell pairs evaluated */
int32_t fl_sparse_info(const fl_sparse* A, int64_t* n, int64_t* nnz, int64_t* cross_pairs);
/* canonical CSR (sorted column indices, no duplicates): indptr (n+1), indices/data (nnz) */
int32_t fl_sparse_to_host(const fl_sparse* A, int64_t* indptr, int32_t* indices, double* data);
void fl_sparse_free(fl_sparse* A);

/* ------------------------------------------------------------- cluster operator (H-matrix)
 * The operator cluster.compress builds (cluster.py:667-712) and its matvec (ClusterOperator.matvec,
 * cluster.py:417-456): y = A_near x - C * far(x), far(x) through the leaf moments, the upward
 * shifts, the far-pair kernel blocks, the downward shifts and the leaf evaluation.  Arrays are the
 * operator's own (tree.parent / topo_order / ranges / dof_perm, cheb.shift, basis_coef,
 * far_pairs, far_blocks, near CSR).  far_blocks NULL: built on the device from `points`
 * (cheb.points, (num_nodes, M, d)) as |xi_a - xi_b|^(-d-2s) (compress, :683-694). */
typedef struct fl_cluster fl_cluster;
typedef struct fl_cluster_desc {
  int32_t d, m;                     /* dimension; Chebyshev points per direction (M = m^d) */
  int64_t n, num_nodes;
  const int64_t* parent;            /* (num_nodes,) -1 at the root */
  const int64_t* topo_order;        /* (num_nodes,) breadth-first, root first */
  const int64_t* ranges;            /* (num_nodes, 2) slices of dof_perm */
  const int64_t* dof_perm;          /* (n,) */
  const double* shift;              /* (num_nodes, d, m, m): S[j][alpha, beta] = L_alpha^parent(xi_beta^node) */
  const double* basis_coef;         /* (n, M): int phi_i L_alpha^leaf(i) */
  int64_t npairs;
  const int64_t* far_pairs;         /* (npairs, 2) unordered admissible node pairs */
  const double* far_blocks;         /* (npairs, M, M) or NULL */
  const double* points;             /* (num_nodes, M, d) or NULL */
  double s, C;                      /* fractional order (device-built blocks); C(d, s) */
  int64_t nnz;                      /* near field CSR (n x n) */
  const int64_t* indptr;
  const int64_t* indices;
  const double* data;
  /* optional (point evaluation, fl_cluster_strong_form): node boxes and the Chebyshev nodes */
  const double* center;             /* (num_nodes, d) tree.center */
  const double* half;               /* (num_nodes,) tree.half */
  const double* ref;                /* (m,) cheb.ref = cos((2j+1) pi / 2m) */
} fl_cluster_desc;
int32_t fl_cluster_create(const fl_cluster_desc* desc, int32_t device, fl_cluster** out);
/* y = A x (and y_far = the far part alone, if non-NULL); ptr_kind 0: host arrays, 1: device */
int32_t fl_cluster_matvec(fl_cluster* C, const double* x, double* y, double* y_far, int32_t ptr_kind);
/* (-Delta)^s u_h at per-cell nodes X (nc, q, d): adapt.strong_form_at (adapt.py:81-214) — the
 * cluster far field evaluated at the points (evaluate_far_field_at_points, cluster.py:469-485) plus
 * the surface terms of the owning leaf's near cells (u restricted to the near DoFs) and of the
 * point's own cell.  cell_leaf: leaf node of every cell (_cell_leaf_assignment); near leaf nodes of
 * every node as CSR (near_off (num_nodes+1), near_val; ClusterOperator.near_dof_leaves); near cells
 * of every node as CSR (ncell_off, ncell_val; cells supporting the near leaves' DoFs); the edge
 * rule (gl_x, gl_w on [0, 1]).  out / far_out: (nc, q). */
int32_t fl_cluster_strong_form(fl_cluster* C, const fl_mesh* mesh, const fl_dofmap* dofmap, double s,
                               const double* u, int64_t q, const double* X, const int64_t* cell_leaf,
                               const int64_t* near_off, const int64_t* near_val, const int64_t* ncell_off,
                               const int64_t* ncell_val, const double* gl_x, const double* gl_w, int64_t ngl,
                               double* out, double* far_out);
/* The far field of u at arbitrary points (ClusterOperator.evaluate_far_field_at_points,
 * cluster.py:469-485): -C * sum L_alpha^owner(x) F[owner], owner = the leaf node of each point. */
int32_t fl_cluster_far_at_points(fl_cluster* C, const double* u, int64_t npts, const double* points,
                                 const int64_t* owner, double* out);
/* the device far blocks (npairs, M, M) */
int32_t fl_cluster_far_blocks(const fl_cluster* C, double* blocks_out);
/* y = A x on device pointers, enqueued on `stream` (NULL: the default stream) without a host
 * synchronisation — the matvec inside the cluster Jacobi-PCG (solve.py:112-214 with the
 * operator's matvec, cluster.py:417-456).  One matvec per operator at a time.  The call is
 * ordered after all work pending on the operator's internal stream, and later synchronous calls
 * and fl_cluster_free are ordered after it (event joins), so no host sync is needed around it.
 * x and y must not alias (the fused kernel writes y while other blocks still read x).  The
 * caller's current device is restored on return. */
int32_t fl_cluster_matvec_async(fl_cluster* C, const double* x, double* y, void* stream);
void fl_cluster_free(fl_cluster* C);
/* Near part of the dual-tree boundary flux at the cell nodes (boundary_flux_at_nodes,
 * cluster.py:586-592; 2D): out[p] = sum over the edges eid[eoff[g]:eoff[g+1]] of the point's group g
 * (poff[g] <= p < poff[g+1]) of edge_flux_potential (assembly.py:303-333) with the rule (gl_x, gl_w)
 * on [0, 1].  X: (npts, 2) grouped by DoF leaf; p0, p1, normals: (nb, 2) boundary edges. */
int32_t fl_boundary_flux_near(int32_t device, double s, int64_t npts, const double* X, int64_t ngroups,
                              const int64_t* poff, const int64_t* eoff, const int64_t* eid, int64_t nb,
                              const double* p0, const double* p1, const double* normals, const double* gl_x,
                              const double* gl_w, int64_t ngl, double* out);

/* ------------------------------------------------------------- driver steps (host O(n) in the
 * reference), on the device
 * _finish_polygon_mesh + _boundary_of (mesh.py:351-403): cells_out (nc x 3) CCW with the longest
 * (refinement) edge first; boundary edges (lexicographic (lo, hi), as np.unique) with outward unit
 * normals.  capacity = rows available in the edge/normal outputs; *nb_out is always set and
 * FL_E_ARG is returned when it exceeds capacity (3*nc always suffices). */
int32_t fl_finish_polygon_mesh(const double* vertices, int64_t nv, const int64_t* cells_in, int64_t nc,
                               int32_t device, int64_t* cells_out, int64_t* boundary_edges_out,
                               double* boundary_normals_out, int64_t capacity, int64_t* nb_out);
/* DofMap (mesh.py:200-240, no `identify`): all vertices for s < 1/2, else the vertices on no
 * boundary edge; vertex_to_dof_out (nv,) with -1 for a non-DoF, *n_out = DoF count. */
int32_t fl_build_dofmap(const fl_mesh* mesh, double s, int32_t device, int64_t* vertex_to_dof_out, int64_t* n_out);
/* Physical nodes of a per-cell reference rule (q nodes `pts`, q x d): X_out (nc, q, d)
 * (cell_quadrature / _map_points, assembly.py:129-132, :290-298) — where the caller evaluates f. */
int32_t fl_cell_rule_nodes(const fl_mesh* mesh, const double* pts, int64_t q, int32_t device, double* X_out);
/* load_vector (assembly.py:550-570, no discontinuity splitting): b_i = sum_K sum_q J_K w_q f_q
 * lambda_a(q) with f_q = f_values[K*q + r] (nc x q, at fl_cell_rule_nodes' nodes) or f_const
 * when f_values is NULL; per DoF in ascending cell order (np.add.at). b_out (n,). */
int32_t fl_load_vector(const fl_mesh* mesh, const fl_dofmap* dofmap, const double* pts, const double* w,
                       int64_t q, const double* f_values, double f_const, int32_t device, double* b_out);

/* ------------------------------------------------------------- matvec
 * y[rows] = A[rows, :] @ x  (solve.py:31-32).  ptr_kind 0: host pointers, 1: device. */
int32_t fl_matvec(const fl_dense* A, const double* x, double* y, int32_t ptr_kind);
/* device-pointer matvec on an explicit stream (used by the sharded CG) */
int32_t fl_matvec_async(const fl_dense* A, const double* x_dev, double* y_dev, void* stream);

/* ------------------------------------------------------------- solve
 * Jacobi-preconditioned CG of solve.pcg (solve.py:52-109) on a whole-matrix fl_dense.
 * precond: 0 none, 1 jacobi.  x0 may be NULL.  b, x0, x are host arrays of length n. */
int32_t fl_pcg(const fl_dense* A, const double* b, const double* x0, double tol,
               int64_t max_iter, int32_t precond, double* x, fl_solve_report* report);

/* Row-block sharded Jacobi-PCG (solve.py:52-109 over row blocks): the
 * per-rank device state and steps; the exchanges between the steps (all-gather of the search
 * direction and of the chunk sums) are the caller's (torch.distributed / NCCL).  Rank g owns
 * rows [g*block_rows, min(n, (g+1)*block_rows)); block_rows is a multiple of 512.  Every
 * reduction is over fixed global chunks of 512 entries and the gathered chunk sums are folded
 * in global order, so the iterates are bitwise the same for any number of ranks and equal to
 * fl_pcg's.  Scalars stay on the device; fl_cg_poll reads them (one host sync).  Vector
 * arguments are device pointers of length >= block_rows (zero padded); p_full >= world*block_rows.
 * One iteration:  [diag] gather(p) [rest] gather(parts) [alpha_update] gather(parts) [beta_xpby]. */
typedef struct fl_cg fl_cg;
typedef struct fl_cg_status {
  int64_t iterations;
  double rz, norm0;                 /* current r.z and sqrt|r0.z0| */
  int32_t done, converged, error, pad_;   /* error 1: p^T A p <= 0 (solve.py:87-88) */
} fl_cg_status;
int32_t fl_cg_create(int64_t n, int64_t m_local, int64_t block_rows, int32_t world, int32_t rank, double tol,
                     int64_t max_iter, int32_t device, void* stream, fl_cg** out);
/* the rank's chunk sums (chunks_per_rank doubles) and the gathered ones (world * chunks_per_rank) */
int32_t fl_cg_buffers(fl_cg* S, double** local_parts, double** all_parts, int64_t* chunks_per_rank);
/* write this rank's chunk sums into a caller-owned device buffer (chunks_per_rank doubles, e.g. the
 * input of the caller's all-gather) instead of the state's own; NULL restores the default */
int32_t fl_cg_bind_parts(fl_cg* S, double* local_parts);
/* z = minv r, p = z; local chunk sums of r.z (solve.py:75-77) */
int32_t fl_cg_begin(fl_cg* S, const double* r, const double* minv, double* z, double* p, void* stream);
/* rz, norm0 from the gathered chunk sums; done at once if b = 0 */
int32_t fl_cg_init(fl_cg* S, const double* all_parts, void* stream);
/* the diagonal block's chunks of A[rows, :] p from the rank's own slice of p (overlaps the all-gather) */
int32_t fl_cg_matvec_diag(fl_cg* S, const fl_dense* A, const double* p_local, void* stream);
/* Ap = A[rows, :] p_full (diagonal chunks from fl_cg_matvec_diag when world > 1); local chunk sums of p.Ap */
int32_t fl_cg_matvec_rest(fl_cg* S, const fl_dense* A, const double* p_full, const double* p_local, double* Ap,
                          void* stream);
/* local chunk sums of a.b (for operators whose matvec is not an fl_dense, e.g. the cluster operator) */
int32_t fl_cg_dot_parts(fl_cg* S, const double* a, const double* b, void* stream);
/* alpha = rz / pAp (pAp folded from all_parts); x += alpha p; r -= alpha Ap; z = minv r; local sums of r.z */
int32_t fl_cg_alpha_update(fl_cg* S, const double* all_parts, double* x, double* r, double* z, const double* p,
                           const double* Ap, const double* minv, void* stream);
/* rz_new folded from all_parts; stopping rule of solve.py:96; beta; p = z + beta p */
int32_t fl_cg_beta_xpby(fl_cg* S, const double* all_parts, const double* z, double* p, void* stream);
int32_t fl_cg_poll(fl_cg* S, fl_cg_status* status, void* stream);
void fl_cg_free(fl_cg* S);

/* ------------------------------------------------------------- parity / diagnostics
 * Per-pair Gauss orders exactly as select_order computes them (quadrature.py:138-179):
 *   cross_k[a*nc+b] (a<b disjoint, assembly.py:705-706), tail_k[t*nc+s] (C_offset-4,
 *   assembly.py:997, :1010-1012); 0 elsewhere.  Host int8 arrays of nc*nc. */
int32_t fl_debug_orders(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                        const fl_order_params* params, int32_t device,
                        int8_t* cross_k, int8_t* tail_k);
/* Exact histograms (index = k, 33 bins) of the same orders, accumulated on the device —
 * usable at every BASELINE size (no nc*nc host arrays). */
int32_t fl_debug_order_hist(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                            const fl_order_params* params, int32_t device, int64_t* cross_hist,
                            int64_t* tail_hist);
/* The device's specialised kernel power on n host values (parity of the building block every
 * quadrature uses): d = 2: x = r2, out = r2^(-(1+s)); d = 1: x = |x - y| (the 1D far field
 * works on the distance itself), out = |x - y|^(-(1+2s)); d = 11: x = r2 with the 1D exponent,
 * out = r2^(-(1/2+s)) (the 1D singular rules); d = 12: the 2D power through the fused
 * accumulate form of the tail kernels (0 + r2^(-(1+s)), kpow_acc). */
int32_t fl_debug_kpow(int32_t d, double s, const double* x, int64_t n, double* out, int32_t device);
/* Measured FP64 FMA peak of the device (TFLOP/s), the roofline denominator of assembly. */
int32_t fl_probe_fp64_peak(int32_t device, double* tflops);
/* Touching pairs as classify/canonicalize produce them (assembly.py:412-473):
 * host outputs sized by *npairs (call with pairs==NULL first to get the count). */
int32_t fl_debug_touching(const fl_mesh* mesh, const fl_dofmap* dofmap, const fl_kernel* kernel,
                          const fl_order_params* params, int32_t device, int64_t* npairs,
                          int64_t* pairs, int32_t* topo, int32_t* k, int32_t* ident_k);

#ifdef __cplusplus
}
#endif
#endif /* FRACLAP_B200_H */
