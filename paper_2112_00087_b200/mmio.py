"""Matrix Market I/O at scale (read_matrix_market / write_matrix_market,
mmio.cpp:10-63 of the reference) over the library's
multi-threaded host reader and writer (csrc/cvk_mmio.cu).  Same CSR as the
reference's reader + csr_from_triplets, bit for bit; the writer's output is
byte-identical to the reference's."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .cavac import CsrMatrix

P = C.c_void_p


class CvkMmMatrix(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row_offsets", C.POINTER(C.c_uint64)), ("col_indices", C.POINTER(C.c_uint64)),
                ("values", C.POINTER(C.c_double))]


def _bind(L):
    if getattr(L, "_mm_bound", False):
        return
    L.cvk_mm_read.argtypes = [C.c_char_p, C.c_int, C.POINTER(CvkMmMatrix)]
    L.cvk_mm_read.restype = C.c_int
    L.cvk_mm_free.argtypes = [C.POINTER(CvkMmMatrix)]
    L.cvk_mm_free.restype = None
    L.cvk_mm_write.argtypes = [C.c_char_p, C.POINTER(CvkMmMatrix), C.c_int]
    L.cvk_mm_write.restype = C.c_int
    L._mm_bound = True


def read_matrix_market(path: str, nthreads: int = 0) -> CsrMatrix:
    """mmio.cpp:28-63 + csr_from_triplets (numkit.cpp:41-75); errors raise
    ValueError with the reference's messages."""
    L = _lib.load()
    _bind(L)
    m = CvkMmMatrix()
    code = L.cvk_mm_read(str(path).encode(), int(nthreads), C.byref(m))
    if code != 0:
        raise ValueError(_lib.last_error())
    n, ncols, nnz = m.nrows, m.ncols, m.nnz
    try:
        rp = np.ctypeslib.as_array(m.row_offsets, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(m.col_indices, shape=(max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(m.values, shape=(max(2 * nnz, 2),))[:2 * nnz].copy().view(np.complex128)
    finally:
        L.cvk_mm_free(C.byref(m))
    return CsrMatrix(n, ncols, rp, ci, v)


def write_matrix_market(path: str, A: CsrMatrix, nthreads: int = 0) -> None:
    """mmio.cpp:10-21: "%.17g" values, 1-based indices, row by row."""
    L = _lib.load()
    _bind(L)
    rp = np.ascontiguousarray(A.row_offsets, np.uint64)
    ci = np.ascontiguousarray(A.col_indices, np.uint64)
    v = np.ascontiguousarray(A.values, np.complex128)
    m = CvkMmMatrix(A.nrows, A.ncols, len(ci), rp.ctypes.data_as(C.POINTER(C.c_uint64)),
                    ci.ctypes.data_as(C.POINTER(C.c_uint64)), v.ctypes.data_as(C.POINTER(C.c_double)))
    code = L.cvk_mm_write(str(path).encode(), C.byref(m), int(nthreads))
    if code != 0:
        raise ValueError(_lib.last_error())
