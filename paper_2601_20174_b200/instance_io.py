"""The reference's on-disk inputs for the solver path, through
libnlsp_io.so (include/nlsp_io.h, host C++):

    load_matrix_market(path)  -> SparseCsrMatrix   sparse.hpp:168-194
    save_matrix_market(a, path)                    sparse.hpp:148-166
    load_instance(dir)        -> PdeInstance       instance_io.hpp:137-185

The loaders mirror the reference's names, arguments and error classes
(IoError for unreadable / malformed files, ValidationError for bad indices,
manifests or families). The returned matrix feeds the GPU solver unchanged:
``pcg(inst.matrix, inst.rhs, TwoLevelPreconditioner(...), ...)``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .nlsp import NlspError, SparseCsrMatrix, ValidationError

FAMILIES = ("diffusion", "anisotropic", "screened_poisson")  # fem.hpp:18-35


class IoError(NlspError):
    """errors.hpp:47-50."""


def _raise(status: int):
    msg = L.io_lib().nlsp_io_last_error().decode(errors="replace")
    if status == L.NLSP_E_IO:
        raise IoError(msg)
    raise ValidationError(msg)


def _csr_from_c(h: L.HostCsrC) -> SparseCsrMatrix:
    n, nnz = int(h.n), int(h.nnz)
    rp = np.ctypeslib.as_array(h.row_ptr, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(h.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(h.values, shape=(max(nnz, 1),))[:nnz].copy()
    return SparseCsrMatrix(n, rp, ci, v)


def load_matrix_market(path: str) -> SparseCsrMatrix:
    """load_matrix_market (sparse.hpp:168-194)."""
    lib = L.io_lib()
    h = L.HostCsrC()
    st = lib.nlsp_io_load_matrix_market(str(path).encode(), C.byref(h))
    if st:
        _raise(st)
    try:
        return _csr_from_c(h)
    finally:
        lib.nlsp_io_csr_free(C.byref(h))


def save_matrix_market(a: SparseCsrMatrix, path: str) -> None:
    """save_matrix_market (sparse.hpp:148-166): lower triangle, %.17g."""
    rp = np.ascontiguousarray(a.row_ptr(), np.uint64)
    ci = np.ascontiguousarray(a.col_idx(), np.uint64)
    v = np.ascontiguousarray(a.values(), np.float64)
    h = L.HostCsrC(a.dim(), a.nnz(), L.u64ptr(rp), L.u64ptr(ci) if ci.size else None,
                   L.dptr(v) if v.size else None)
    st = L.io_lib().nlsp_io_save_matrix_market(C.byref(h), str(path).encode())
    if st:
        _raise(st)


@dataclass
class PdeInstance:
    """PdeInstance (fem.hpp:202-211) as load_instance reads it."""
    family: str
    grid_n: int
    seed: int
    jitter: float
    alpha: float
    matrix: SparseCsrMatrix
    rhs: np.ndarray
    vertices: np.ndarray       # n x 2
    boundary_mask: np.ndarray  # n, uint8 (the mask of generate_smoothed_vectors)
    triangles: np.ndarray      # t x 3
    coefficients: np.ndarray   # t x (1 | 3)


def load_instance(dir_path: str) -> PdeInstance:
    """load_instance (instance_io.hpp:137-185)."""
    lib = L.io_lib()
    h = L.InstanceC()
    st = lib.nlsp_io_load_instance(str(dir_path).encode(), C.byref(h))
    if st:
        _raise(st)
    try:
        a = _csr_from_c(h.matrix)
        nv, nt, cc = int(h.n_vertices), int(h.n_triangles), int(h.coeff_cols)

        def arr(ptr, count, shape):
            if count == 0:
                return np.zeros(shape, dtype=np.ctypeslib.as_array(ptr, shape=(1,)).dtype)
            return np.ctypeslib.as_array(ptr, shape=(count,)).copy().reshape(shape)

        return PdeInstance(
            family=FAMILIES[h.family], grid_n=int(h.grid_n), seed=int(h.seed), jitter=float(h.jitter),
            alpha=float(h.alpha), matrix=a, rhs=arr(h.rhs, a.dim(), (a.dim(),)),
            vertices=arr(h.vertices, 2 * nv, (nv, 2)), boundary_mask=arr(h.boundary_mask, nv, (nv,)),
            triangles=arr(h.triangles, 3 * nt, (nt, 3)), coefficients=arr(h.coefficients, cc * nt, (nt, cc)))
    finally:
        lib.nlsp_io_instance_free(C.byref(h))
