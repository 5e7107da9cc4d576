"""DenseDeviceOperator: the assembled matrix (or one row block of it) resident in HBM.

Duck-types the operator contract of the reference solvers (solve.py:19-35): `.matvec(x)`
returns A x for host vectors and `.diag()` the exact diagonal, so it can be handed to the
reference's own pcg / multigrid / heat_step unchanged, or to this package's `solve.pcg`,
which keeps the whole CG loop on the device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class DenseDeviceOperator:
    def __init__(self, handle, n, row_begin, row_end):
        self._h = handle
        self.n = int(n)
        self.row_begin = int(row_begin)
        self.row_end = int(row_end)

    @classmethod
    def from_host(cls, A, device=0):
        """Upload a dense (n, n) host matrix (e.g. the reference's assemble_dense output)."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("A must be square")
        h = C.c_void_p()
        _lib.check(_lib.load().fl_dense_from_host(A.ctypes.data, A.shape[0], int(device), C.byref(h)))
        return cls(h, A.shape[0], 0, A.shape[0])

    @classmethod
    def from_host_rows(cls, rows, n, row_begin, device=0):
        """Rows [row_begin, row_begin + len(rows)) of an (n, n) host matrix as a row-block operator."""
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, int(n))
        h = C.c_void_p()
        _lib.check(_lib.load().fl_dense_from_host_rows(rows.ctypes.data, int(n), int(row_begin),
                                                       int(row_begin) + len(rows), int(device), C.byref(h)))
        return cls(h, n, row_begin, row_begin + len(rows))

    # ------------------------------------------------------------ lifetime
    def free(self):
        if self._h is not None and self._h.value:
            _lib.load().fl_dense_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("operator already freed")
        return self._h

    @property
    def shape(self):
        return (self.row_end - self.row_begin, self.n)

    @property
    def full(self):
        return self.row_begin == 0 and self.row_end == self.n

    # ------------------------------------------------------------ data access
    def device_ptr(self):
        p = C.c_void_p()
        _lib.check(_lib.load().fl_dense_info(self.handle, None, None, None, C.byref(p)))
        return p.value

    def stats(self):
        s = _lib.fl_assembly_stats()
        _lib.check(_lib.load().fl_dense_stats(self.handle, C.byref(s)))
        return s.as_dict()

    def to_host(self, out=None):
        shape = (self.row_end - self.row_begin, self.n)
        if out is None:
            out = np.empty(shape)
        elif out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array of shape %r" % (shape,))
        _lib.check(_lib.load().fl_dense_to_host(self.handle, out.ctypes.data))
        return out

    def rows(self, idx):
        """Copy the global rows `idx` (inside this operator's row range) to the host."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty((len(idx), self.n))
        _lib.check(_lib.load().fl_dense_rows(self.handle, len(idx), idx.ctypes.data, out.ctypes.data))
        return out

    def diag(self):
        out = np.empty(self.row_end - self.row_begin)
        _lib.check(_lib.load().fl_dense_diag(self.handle, out.ctypes.data))
        return out

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("x must have shape (%d,)" % self.n)
        y = np.empty(self.row_end - self.row_begin)
        _lib.check(_lib.load().fl_matvec(self.handle, x.ctypes.data, y.ctypes.data, 0))
        return y

    def matvec_device(self, x_ptr, y_ptr, stream=None):
        """y[rows] = A[rows, :] x on device pointers (x padded to a multiple of 32 entries)."""
        _lib.check(_lib.load().fl_matvec_async(self.handle, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                               _lib.stream_arg(stream)))

    def __matmul__(self, x):
        return self.matvec(x)
