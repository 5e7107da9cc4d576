"""ctypes binding of libfraclap_b200.so (include/fraclap_b200.h).

There is no CPU fallback: if the shared library is missing or cannot be loaded, every
entry point raises.  Error codes map 1:1 onto the reference's exceptions.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FRACLAP_B200_LIB") or os.path.join(_HERE, "lib", "libfraclap_b200.so")

FL_OK, FL_E_ARG, FL_E_ASSEMBLY, FL_E_QUAD, FL_E_SOLVER, FL_E_CUDA, FL_E_OOM = 0, -1, -2, -3, -4, -5, -6
VARIANT_ID = {"integral": 0, "regional": 1, "symmetrized": 2}

EXPORTS = ["fl_abi_version", "fl_last_error", "fl_device_count", "fl_launch_count", "fl_assemble_dense",
           "fl_assemble_dense_host", "fl_finish_polygon_mesh", "fl_build_dofmap", "fl_cell_rule_nodes",
           "fl_load_vector", "fl_assemble_near_field", "fl_sparse_info", "fl_sparse_to_host", "fl_sparse_free",
           "fl_debug_ring_tail", "fl_cluster_create", "fl_cluster_matvec", "fl_cluster_far_blocks", "fl_cluster_free",
           "fl_cluster_strong_form", "fl_cluster_far_at_points", "fl_boundary_flux_near", "fl_cluster_matvec_async",
           "fl_dense_from_host", "fl_dense_from_host_rows",
           "fl_dense_free",
           "fl_dense_info", "fl_dense_stats", "fl_dense_to_host", "fl_dense_rows", "fl_dense_diag", "fl_matvec",
           "fl_matvec_async", "fl_pcg", "fl_cg_create", "fl_cg_buffers", "fl_cg_bind_parts", "fl_cg_begin", "fl_cg_init",
           "fl_cg_matvec_diag", "fl_cg_matvec_rest", "fl_cg_dot_parts", "fl_cg_alpha_update", "fl_cg_beta_xpby",
           "fl_cg_poll", "fl_cg_free",
           "fl_debug_orders", "fl_debug_order_hist", "fl_debug_kpow", "fl_probe_fp64_peak", "fl_debug_touching"]


class fl_mesh(C.Structure):
    _fields_ = [("d", C.c_int32), ("pad_", C.c_int32), ("nv", C.c_int64), ("nc", C.c_int64),
                ("nb", C.c_int64), ("vertices", C.c_void_p), ("cells", C.c_void_p),
                ("boundary_edges", C.c_void_p), ("boundary_normals", C.c_void_p)]


class fl_dofmap(C.Structure):
    _fields_ = [("n", C.c_int64), ("vertex_to_dof", C.c_void_p)]


class fl_kernel(C.Structure):
    _fields_ = [("d", C.c_int32), ("variant", C.c_int32), ("s", C.c_double), ("C_ds", C.c_double)]


class fl_order_params(C.Structure):
    _fields_ = [("rho1", C.c_double), ("rho2", C.c_double), ("rho3", C.c_double), ("rho4", C.c_double),
                ("C_offset", C.c_double), ("alpha", C.c_double)]


class fl_tables(C.Structure):
    _fields_ = [("dir", C.c_void_p), ("data", C.c_void_p), ("ndata", C.c_int64)]


class fl_cg_status(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("rz", C.c_double), ("norm0", C.c_double), ("done", C.c_int32),
                ("converged", C.c_int32), ("error", C.c_int32), ("pad_", C.c_int32)]


class fl_near_structure(C.Structure):
    _fields_ = [("nleaves", C.c_int64), ("leaf_of_dof", C.c_void_p), ("npairs", C.c_int64), ("pairs", C.c_void_p)]


class fl_cluster_desc(C.Structure):
    _fields_ = [("d", C.c_int32), ("m", C.c_int32), ("n", C.c_int64), ("num_nodes", C.c_int64),
                ("parent", C.c_void_p), ("topo_order", C.c_void_p), ("ranges", C.c_void_p), ("dof_perm", C.c_void_p),
                ("shift", C.c_void_p), ("basis_coef", C.c_void_p), ("npairs", C.c_int64), ("far_pairs", C.c_void_p),
                ("far_blocks", C.c_void_p), ("points", C.c_void_p), ("s", C.c_double), ("C", C.c_double),
                ("nnz", C.c_int64), ("indptr", C.c_void_p), ("indices", C.c_void_p), ("data", C.c_void_p),
                ("center", C.c_void_p), ("half", C.c_void_p), ("ref", C.c_void_p)]


class fl_solve_report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double), ("seconds", C.c_double),
                ("converged", C.c_int32), ("pad_", C.c_int32), ("true_residual", C.c_double)]


class fl_assembly_stats(C.Structure):
    _fields_ = [("pairs_identical", C.c_int64), ("pairs_touching", C.c_int64), ("pairs_cross", C.c_int64),
                ("pairs_tail", C.c_int64), ("pairs_boundary_singular", C.c_int64),
                ("pairs_boundary_flux", C.c_int64), ("evals_cross", C.c_double), ("evals_tail", C.c_double),
                ("evals_singular", C.c_double), ("evals_boundary", C.c_double), ("ms_prep", C.c_double),
                ("ms_singular", C.c_double), ("ms_tail", C.c_double), ("ms_flux", C.c_double),
                ("ms_tiles", C.c_double), ("ms_cross", C.c_double),
                ("ms_local", C.c_double), ("ms_total", C.c_double), ("cross_tile_pairs", C.c_int64),
                ("ncolors", C.c_int32), ("ntiles", C.c_int32), ("ms_discover", C.c_double),
                ("ms_near", C.c_double), ("ms_cross_compute", C.c_double), ("near_pairs", C.c_int64),
                ("order_ties", C.c_int64), ("cross_scale_exp", C.c_int32), ("cross_fallback", C.c_int32),
                ("evals_tail_block", C.c_double), ("ms_tail_block", C.c_double), ("evals_near", C.c_double),
                ("evals_tail_sym", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load():
    """Load the extension; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("fraclap_b200 CUDA library not built: %s (run __graft_entry__.build())" % LIB_PATH)
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "fl_abi_version": (C.c_int32, []),
        "fl_last_error": (C.c_char_p, []),
        "fl_device_count": (C.c_int32, []),
        "fl_launch_count": (C.c_int64, []),
        "fl_assemble_dense": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params),
                                          P(fl_tables), C.c_int64, C.c_int64, C.c_int64, C.c_int32, vp,
                                          P(vp)]),
        "fl_assemble_dense_host": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params),
                                               P(fl_tables), C.c_int64, C.c_int32, vp]),
        "fl_finish_polygon_mesh": (C.c_int32, [vp, C.c_int64, vp, C.c_int64, C.c_int32, vp, vp, vp, C.c_int64,
                                               P(C.c_int64)]),
        "fl_build_dofmap": (C.c_int32, [P(fl_mesh), C.c_double, C.c_int32, vp, P(C.c_int64)]),
        "fl_cell_rule_nodes": (C.c_int32, [P(fl_mesh), vp, C.c_int64, C.c_int32, vp]),
        "fl_load_vector": (C.c_int32, [P(fl_mesh), P(fl_dofmap), vp, vp, C.c_int64, vp, C.c_double, C.c_int32, vp]),
        "fl_assemble_near_field": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params),
                                               P(fl_tables), P(fl_near_structure), vp, C.c_int32, P(vp)]),
        "fl_sparse_info": (C.c_int32, [vp, P(C.c_int64), P(C.c_int64), P(C.c_int64)]),
        "fl_sparse_to_host": (C.c_int32, [vp, vp, vp, vp]),
        "fl_sparse_free": (None, [vp]),
        "fl_cluster_create": (C.c_int32, [P(fl_cluster_desc), C.c_int32, P(vp)]),
        "fl_cluster_matvec": (C.c_int32, [vp, vp, vp, vp, C.c_int32]),
        "fl_cluster_far_blocks": (C.c_int32, [vp, vp]),
        "fl_cluster_free": (None, [vp]),
        "fl_cluster_far_at_points": (C.c_int32, [vp, vp, C.c_int64, vp, vp, vp]),
        "fl_cluster_matvec_async": (C.c_int32, [vp, vp, vp, vp]),
        "fl_boundary_flux_near": (C.c_int32, [C.c_int32, C.c_double, C.c_int64, vp, C.c_int64, vp, vp, vp,
                                              C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp]),
        "fl_cluster_strong_form": (C.c_int32, [vp, P(fl_mesh), P(fl_dofmap), C.c_double, vp, C.c_int64, vp, vp, vp,
                                               vp, vp, vp, vp, vp, C.c_int64, vp, vp]),
        "fl_debug_ring_tail": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params), P(fl_tables),
                                           vp, C.c_int32, vp, vp]),
        "fl_dense_from_host": (C.c_int32, [vp, C.c_int64, C.c_int32, P(vp)]),
        "fl_dense_from_host_rows": (C.c_int32, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, P(vp)]),
        "fl_dense_free": (None, [vp]),
        "fl_dense_info": (C.c_int32, [vp, P(C.c_int64), P(C.c_int64), P(C.c_int64), P(vp)]),
        "fl_dense_stats": (C.c_int32, [vp, P(fl_assembly_stats)]),
        "fl_dense_to_host": (C.c_int32, [vp, vp]),
        "fl_dense_diag": (C.c_int32, [vp, vp]),
        "fl_dense_rows": (C.c_int32, [vp, C.c_int64, vp, vp]),
        "fl_matvec": (C.c_int32, [vp, vp, vp, C.c_int32]),
        "fl_matvec_async": (C.c_int32, [vp, vp, vp, vp]),
        "fl_pcg": (C.c_int32, [vp, vp, vp, C.c_double, C.c_int64, C.c_int32, vp, P(fl_solve_report)]),
        "fl_cg_create": (C.c_int32, [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_int64,
                                     C.c_int32, vp, P(vp)]),
        "fl_cg_buffers": (C.c_int32, [vp, P(vp), P(vp), P(C.c_int64)]),
        "fl_cg_bind_parts": (C.c_int32, [vp, vp]),
        "fl_cg_begin": (C.c_int32, [vp, vp, vp, vp, vp, vp]),
        "fl_cg_init": (C.c_int32, [vp, vp, vp]),
        "fl_cg_matvec_diag": (C.c_int32, [vp, vp, vp, vp]),
        "fl_cg_matvec_rest": (C.c_int32, [vp, vp, vp, vp, vp, vp]),
        "fl_cg_dot_parts": (C.c_int32, [vp, vp, vp, vp]),
        "fl_cg_alpha_update": (C.c_int32, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "fl_cg_beta_xpby": (C.c_int32, [vp, vp, vp, vp, vp]),
        "fl_cg_poll": (C.c_int32, [vp, P(fl_cg_status), vp]),
        "fl_cg_free": (None, [vp]),
        "fl_debug_orders": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params), C.c_int32,
                                        vp, vp]),
        "fl_debug_order_hist": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params),
                                            C.c_int32, vp, vp]),
        "fl_probe_fp64_peak": (C.c_int32, [C.c_int32, P(C.c_double)]),
        "fl_debug_kpow": (C.c_int32, [C.c_int32, C.c_double, vp, C.c_int64, vp, C.c_int32]),
        "fl_debug_touching": (C.c_int32, [P(fl_mesh), P(fl_dofmap), P(fl_kernel), P(fl_order_params), C.c_int32,
                                          P(C.c_int64), vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(code):
    """Raise the reference's exception for a negative FL_E_* code."""
    if code == FL_OK:
        return
    msg = load().fl_last_error().decode(errors="replace")
    if code == FL_E_ARG:
        raise ValueError(msg)
    if code == FL_E_ASSEMBLY:
        from .assembly import AssemblyError
        raise AssemblyError(msg)
    if code == FL_E_QUAD:
        from .quadrature import QuadratureError
        raise QuadratureError(msg)
    if code == FL_E_SOLVER:
        from .solve import SolverError
        raise SolverError(msg)
    if code == FL_E_OOM:
        raise MemoryError(msg)
    raise RuntimeError("fraclap_b200 CUDA error: %s" % msg)


CUDA_STREAM_LEGACY = 0x1


def stream_arg(stream):
    """None -> the library's own stream; 0 (torch's default stream) -> cudaStreamLegacy;
    a torch.cuda.Stream or a raw handle -> that stream."""
    if stream is None:
        return None
    stream = getattr(stream, "cuda_stream", stream)
    return C.c_void_p(CUDA_STREAM_LEGACY if int(stream) == 0 else int(stream))


def ptr(a):
    return a.ctypes.data if a is not None else None


class Marshal:
    """Keeps the contiguous host arrays alive for the duration of one C call."""

    def __init__(self, mesh, dofmap, kernel, params):
        from .quadrature import OrderParams
        d = int(mesh.vertices.shape[1])
        self.vertices = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        self.cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
        be = np.asarray(mesh.boundary_edges, dtype=np.int64).reshape(-1, d)
        bn = np.asarray(mesh.boundary_normals, dtype=np.float64).reshape(-1, d)
        self.bedges = np.ascontiguousarray(be)
        self.bnormals = np.ascontiguousarray(bn)
        self.v2d = np.ascontiguousarray(dofmap.vertex_to_dof, dtype=np.int64)
        self.mesh = fl_mesh(d, 0, len(self.vertices), len(self.cells), len(self.bedges), ptr(self.vertices),
                            ptr(self.cells), ptr(self.bedges) if len(self.bedges) else None,
                            ptr(self.bnormals) if len(self.bnormals) else None)
        self.dofmap = fl_dofmap(int(dofmap.n), ptr(self.v2d))
        variant = getattr(kernel, "variant", "integral")
        variant = getattr(variant, "value", variant)
        self.kernel = fl_kernel(int(kernel.d), VARIANT_ID[str(variant)], float(kernel.s), float(kernel.C_ds))
        params = params if params is not None else OrderParams()
        self.params = fl_order_params(params.rho1, params.rho2, params.rho3, params.rho4, params.C_offset,
                                      float(params.target_alpha(d, float(kernel.s))))
        self.d = d
