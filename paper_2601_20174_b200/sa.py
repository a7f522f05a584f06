"""The SA coarse space, mirroring sa.hpp: aggregate_nodes
(host) and sa_prolongator (aggregation on the host, P assembled on the device),
whose dense P feeds TwoLevelPreconditioner like any basis (coarse dimensions up
to 2048: the wide restriction / prolongation kernels)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .nlsp import DeviceDense, SparseCsrMatrix, ValidationError, _check, default_context


def aggregate_nodes(a: SparseCsrMatrix, theta: float = 0.25):
    """aggregate_nodes (sa.hpp:18-76): (aggregate id per node, count)."""
    n = a.dim()
    agg = np.empty(max(n, 1), np.uint64)
    nc = C.c_uint64(0)
    st = L.gpu_lib().nlsp_sa_aggregate(n, a.nnz(), L.u64ptr(a.row_ptr()), L.u64ptr(a.col_idx()),
                                       L.dptr(a.values()), theta, L.u64ptr(agg), C.byref(nc))
    if st:
        raise ValidationError("aggregate_nodes: bad CSR arrays")
    return agg[:n], int(nc.value)


def sa_prolongator(a: SparseCsrMatrix, theta: float = 0.25, omega: float = 0.66, ctx=None) -> DeviceDense:
    """sa_prolongator (sa.hpp:78-109): dense n x n_c on the device."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(ctx, L.gpu_lib().nlsp_sa_prolongator(ctx.handle, a.dim(), a.nnz(), L.u64ptr(a.row_ptr()),
                                                L.u64ptr(a.col_idx()), L.dptr(a.values()), theta, omega,
                                                C.byref(h)))
    return DeviceDense(ctx, h)
