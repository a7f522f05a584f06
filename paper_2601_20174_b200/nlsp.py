"""Host-side mirror of the reference's solver / preconditioner interface
(/root/reference/proj/include/nlsp/: sparse.hpp, smoothing.hpp, svd.hpp,
two_level.hpp, errors.hpp) over the B200 C-ABI (include/nlsp_gpu.h).

Same names, argument meaning and error behaviour as the reference, so the
parity tests read like the reference's own GoogleTest suites:

    a = SparseCsrMatrix.from_triplets(n, triplets)           # sparse.hpp:24-53
    sv = generate_smoothed_vectors(a, mask, K, s1, w, seed)   # smoothing.hpp:81-100
    u, sigma = svd_basis(sv.s, k)                             # first_cols(svd_oracle(S).U, k)
    m = TwoLevelPreconditioner(a, u, w, nu1, nu2)             # two_level.hpp:24-53
    res = pcg(a, b, m, delta, max_iters)                      # two_level.hpp:141-191

Every numeric call runs on the GPU through libnlsp_gpu.so; nothing here
computes on the host except CSR normalisation of user triplets.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors --
class NlspError(RuntimeError):
    pass


class ValidationError(NlspError):
    """errors.hpp:12-16 (CLI exit code 1)."""


class NumericError(NlspError):
    """errors.hpp:19-23 (CLI exit code 2)."""


class RankDeficiencyError(NumericError):
    pass


class NotSpdError(NumericError):
    pass


class ConvergenceError(NumericError):
    pass


class CudaError(NlspError):
    pass


_STATUS = {
    L.NLSP_E_VALIDATION: ValidationError,
    L.NLSP_E_NUMERIC: NumericError,
    L.NLSP_E_NOT_SPD: NotSpdError,
    L.NLSP_E_RANK_DEFICIENT: RankDeficiencyError,
    L.NLSP_E_CONVERGENCE: ConvergenceError,
    L.NLSP_E_CUDA: CudaError,
    L.NLSP_E_OOM: CudaError,
}


def _check(ctx, status):
    if status != L.NLSP_OK:
        msg = L.gpu_lib().nlsp_last_error(ctx.handle if ctx else None) if ctx else b""
        raise _STATUS.get(status, NlspError)((msg or b"").decode() or f"nlsp status {status}")


# ----------------------------------------------------------------- context --
class Context:
    """One CUDA stream + workspace (nlsp_ctx). One per host thread."""

    def __init__(self, device: int = 0):
        lib = L.gpu_lib()
        h = C.c_void_p()
        st = lib.nlsp_ctx_create(device, C.byref(h))
        if st != L.NLSP_OK:
            raise CudaError(f"nlsp_ctx_create(device={device}) failed with status {st}: "
                            "no usable sm_100 GPU (there is no CPU fallback)")
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        return L.gpu_lib().nlsp_ctx_stream(self.handle) or 0

    def kernel_launches(self) -> int:
        return int(L.gpu_lib().nlsp_ctx_kernel_launches(self.handle))

    def synchronize(self):
        _check(self, L.gpu_lib().nlsp_ctx_synchronize(self.handle))

    def set_s0_draw(self, where: str):
        """Where generate_smoothed_vectors draws S^(0): "host" (default,
        bit-identical to the reference's Rng stream) or "device" (the same
        mt19937_64 words by jump-ahead, CUDA's log / sincos in Box-Muller)."""
        modes = {"host": L.NLSP_S0_DRAW_HOST, "device": L.NLSP_S0_DRAW_DEVICE}
        if where not in modes:
            raise ValidationError("set_s0_draw: 'host' or 'device'")
        _check(self, L.gpu_lib().nlsp_ctx_set_s0_draw(self.handle, modes[where]))

    def last_s0_draw(self) -> str:
        return "device" if L.gpu_lib().nlsp_ctx_last_s0_draw(self.handle) == L.NLSP_S0_DRAW_DEVICE else "host"

    def mt19937_64_words(self, seed: int, count: int) -> np.ndarray:
        """The first `count` outputs of std::mt19937_64(seed) from the device jump tree."""
        out = np.empty(count, dtype=np.uint64)
        _check(self, L.gpu_lib().nlsp_mt19937_64_words(self.handle, seed, count, L.u64ptr(out)))
        return out

    def close(self):
        if self.handle:
            L.gpu_lib().nlsp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


# --------------------------------------------------------------------- CSR --
class SparseCsrMatrix:
    """Square CSR, columns sorted within a row, no duplicates, no stored zeros
    (sparse.hpp:17-19,108-112). Host arrays in the reference's size_t layout;
    the device copy (int32 indices) is uploaded lazily per context."""

    def __init__(self, dim: int, row_ptr, col_idx, values):
        self._dim = int(dim)
        self._rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        self._ci = np.ascontiguousarray(col_idx, dtype=np.uint64)
        self._v = np.ascontiguousarray(values, dtype=np.float64)
        if self._rp.shape != (self._dim + 1,):
            raise ValidationError("row_ptr must have dim + 1 entries")
        self._dev = {}

    @staticmethod
    def from_triplets(dim: int, triplets) -> "SparseCsrMatrix":
        """sparse.hpp:24-53: range check, sort by (i, j), sum duplicates, drop zeros."""
        t = list(triplets)
        if t:
            i = np.array([x[0] for x in t], dtype=np.int64)
            j = np.array([x[1] for x in t], dtype=np.int64)
            v = np.array([x[2] for x in t], dtype=np.float64)
        else:
            i = j = np.zeros(0, np.int64)
            v = np.zeros(0)
        return SparseCsrMatrix.from_coo(dim, i, j, v)

    @staticmethod
    def from_coo(dim: int, i, j, v) -> "SparseCsrMatrix":
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        if i.size and (i.min() < 0 or j.min() < 0 or i.max() >= dim or j.max() >= dim):
            raise ValidationError("triplet index out of range")
        order = np.lexsort((j, i), axis=0) if i.size else np.zeros(0, np.int64)
        i, j, v = i[order], j[order], v[order]
        if i.size:
            new = np.ones(i.size, bool)
            new[1:] = (i[1:] != i[:-1]) | (j[1:] != j[:-1])
            starts = np.flatnonzero(new)
            # duplicates summed left to right from 0.0, as the reference loop does
            # (sparse.hpp:40-44); the sort above is stable, so input order holds
            sums = 0.0 + v[starts]
            if (~new).any():
                ends = np.append(starts[1:], i.size)
                for g in np.flatnonzero(ends - starts > 1):
                    acc = 0.0
                    for t in v[starts[g]:ends[g]]:
                        acc += float(t)
                    sums[g] = acc
            ui, uj = i[starts], j[starts]
            keep = sums != 0.0
            ui, uj, sums = ui[keep], uj[keep], sums[keep]
        else:
            ui = uj = np.zeros(0, np.int64)
            sums = np.zeros(0)
        rp = np.zeros(dim + 1, np.uint64)
        np.add.at(rp, ui + 1, 1)
        rp = np.cumsum(rp, dtype=np.uint64)
        return SparseCsrMatrix(dim, rp, uj.astype(np.uint64), sums)

    @staticmethod
    def identity(dim: int) -> "SparseCsrMatrix":
        return SparseCsrMatrix(dim, np.arange(dim + 1, dtype=np.uint64),
                               np.arange(dim, dtype=np.uint64), np.ones(dim))

    def dim(self) -> int:
        return self._dim

    def nnz(self) -> int:
        return int(self._v.size)

    def row_ptr(self):
        return self._rp

    def col_idx(self):
        return self._ci

    def values(self):
        return self._v

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self._dim, self._dim))
        rows = np.repeat(np.arange(self._dim), np.diff(self._rp.astype(np.int64)))
        d[rows, self._ci.astype(np.int64)] = self._v
        return d

    def device(self, ctx: Context | None = None) -> "DeviceCsr":
        ctx = ctx or default_context()
        key = id(ctx)
        dev = self._dev.get(key)
        if dev is None or dev.ctx is not ctx:
            dev = DeviceCsr.upload(ctx, self)
            self._dev[key] = dev
        return dev

    def diagonal(self) -> np.ndarray:
        dev = self.device()
        d = np.empty(self._dim)
        _check(dev.ctx, L.gpu_lib().nlsp_csr_diagonal(dev.ctx.handle, dev.handle, L.dptr(d)))
        return d


class DeviceCsr:
    """nlsp_csr: the device-resident copy (int32 row_ptr/col_idx, fp64 values)."""

    def __init__(self, ctx, handle, n, nnz):
        self.ctx, self.handle, self.n, self.nnz = ctx, handle, n, nnz

    @staticmethod
    def upload(ctx: Context, a: SparseCsrMatrix) -> "DeviceCsr":
        h = C.c_void_p()
        _check(ctx, L.gpu_lib().nlsp_csr_upload(ctx.handle, a.dim(), a.nnz(), L.u64ptr(a.row_ptr()),
                                                L.u64ptr(a.col_idx()), L.dptr(a.values()),
                                                C.byref(h)))
        return DeviceCsr(ctx, h, a.dim(), a.nnz())

    def format(self):
        """(kind, offsets, pass_bytes) of nlsp_csr_format: 0 CSR, 1 constant
        diagonal form, 2 diagonal form with per-row values, 3 CSR with implicit
        columns (one presence mask per row in place of the column indices)."""
        kind, offs, pb = C.c_int32(0), C.c_int32(0), C.c_uint64(0)
        _check(self.ctx, L.gpu_lib().nlsp_csr_format(self.handle, C.byref(kind), C.byref(offs), C.byref(pb)))
        return int(kind.value), int(offs.value), int(pb.value)

    def geometry(self):
        """(plane, halo, march) of nlsp_csr_geometry: the structured-grid
        geometry of the diagonal form and whether the loop runs plane marches."""
        pl, h, mr = C.c_uint64(0), C.c_int32(0), C.c_int32(0)
        _check(self.ctx, L.gpu_lib().nlsp_csr_geometry(self.ctx.handle, self.handle, C.byref(pl), C.byref(h),
                                                       C.byref(mr)))
        return int(pl.value), int(h.value), bool(mr.value)

    def __del__(self):
        try:
            if self.handle:
                L.gpu_lib().nlsp_csr_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def _dev(a, ctx=None) -> DeviceCsr:
    if isinstance(a, DeviceCsr):
        return a
    return a.device(ctx)


def spmv(a: SparseCsrMatrix, x) -> np.ndarray:
    """y = A x (sparse.hpp:116-128); ValidationError on a dimension mismatch."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (a.dim(),):
        raise ValidationError("spmv: dimension mismatch")
    dev = _dev(a)
    y = np.empty(a.dim())
    _check(dev.ctx, L.gpu_lib().nlsp_spmv(dev.ctx.handle, dev.handle, L.dptr(x), L.dptr(y)))
    return y


# ------------------------------------------------------------------- dense --
class DeviceDense:
    """nlsp_dense: a row-major fp64 matrix resident on the device."""

    def __init__(self, ctx, handle):
        self.ctx, self.handle = ctx, handle
        r, c = C.c_uint64(), C.c_uint64()
        L.gpu_lib().nlsp_dense_dims(handle, C.byref(r), C.byref(c))
        self.rows, self.cols = int(r.value), int(c.value)

    @staticmethod
    def upload(arr, ctx: Context | None = None) -> "DeviceDense":
        ctx = ctx or default_context()
        a = np.ascontiguousarray(arr, dtype=np.float64)
        if a.ndim != 2:
            raise ValidationError("dense matrix must be 2-D")
        h = C.c_void_p()
        _check(ctx, L.gpu_lib().nlsp_dense_upload(ctx.handle, a.shape[0], a.shape[1], L.dptr(a),
                                                  C.byref(h)))
        return DeviceDense(ctx, h)

    def numpy(self) -> np.ndarray:
        out = np.empty((self.rows, self.cols))
        _check(self.ctx, L.gpu_lib().nlsp_dense_export(self.ctx.handle, self.handle, L.dptr(out)))
        return out

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def data_ptr(self) -> int:
        """Device address of the row-major data."""
        return L.gpu_lib().nlsp_dense_data(self.handle) or 0

    def __del__(self):
        try:
            if self.handle:
                L.gpu_lib().nlsp_dense_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def _dense(x, ctx) -> DeviceDense:
    return x if isinstance(x, DeviceDense) else DeviceDense.upload(x, ctx)


# --------------------------------------------------------------- smoothing --
class JacobiSmoother:
    """Weighted Jacobi x <- x + w D^-1 (b - A x) (smoothing.hpp:15-61)."""

    def __init__(self, a: SparseCsrMatrix, omega: float):
        if omega < 0.0 or omega > 1.0:
            raise ValidationError("jacobi: omega must lie in [0, 1]")
        d = a.diagonal()
        if (d <= 0.0).any():
            raise NumericError(f"jacobi: non-positive diagonal at row {int(np.argmax(d <= 0.0))}")
        self._omega = float(omega)
        self._inv_diag = 1.0 / d

    def omega(self) -> float:
        return self._omega

    def inv_diag(self) -> np.ndarray:
        return self._inv_diag

    def sweep(self, a: SparseCsrMatrix, x: np.ndarray, b=None, sweeps: int = 1) -> None:
        """In place, like the reference's vector sweep (b given) or block sweep
        (x 2-D, homogeneous)."""
        if x.ndim == 2:
            if b is not None:
                raise ValidationError("block sweep with b is not on the hot path")
            s = DeviceDense.upload(x, _dev(a).ctx)
            smooth_vectors(a, s, sweeps, self._omega)
            x[...] = s.numpy()
            return
        if x.shape != (a.dim(),) or b is None or np.asarray(b).shape != (a.dim(),):
            raise ValidationError("jacobi sweep: dimension mismatch")
        dev = _dev(a)
        xb = np.ascontiguousarray(x, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        _check(dev.ctx, L.gpu_lib().nlsp_jacobi_sweeps(dev.ctx.handle, dev.handle, self._omega, sweeps,
                                                       L.dptr(xb), L.dptr(bb)))
        x[...] = xb


def smooth_vectors(a: SparseCsrMatrix, s: DeviceDense, sweeps: int, omega: float) -> DeviceDense:
    """`sweeps` homogeneous block sweeps on a device-resident S (smoothing.hpp:50-60)."""
    dev = _dev(a)
    _check(dev.ctx, L.gpu_lib().nlsp_smooth_vectors(dev.ctx.handle, dev.handle, s.handle, sweeps, omega))
    return s


@dataclass
class SmoothedVectorSet:
    """smoothing.hpp:70-75; `s` stays on the device (call .numpy() to copy)."""
    s: DeviceDense
    sweeps_applied: int = 0
    omega: float = 0.66
    source_seed: int = 0


def generate_smoothed_vectors(a: SparseCsrMatrix, boundary_mask, k: int, sweeps: int,
                              omega: float, seed: int) -> SmoothedVectorSet:
    """smoothing.hpp:81-100: S^(0) from Rng(mix_seed(seed, "smoo")), Dirichlet
    rows zero, `sweeps` homogeneous Jacobi sweeps on the device."""
    if k < 1:
        raise ValidationError("generate_smoothed_vectors: K must be positive")
    if boundary_mask is not None and len(boundary_mask) != a.dim():
        raise ValidationError("generate_smoothed_vectors: mask size mismatch")
    dev = _dev(a)
    mask = None
    mp = None
    if boundary_mask is not None:
        mask = np.ascontiguousarray(np.asarray(boundary_mask, dtype=bool).astype(np.uint8))
        mp = L.u8ptr(mask)
    h = C.c_void_p()
    _check(dev.ctx, L.gpu_lib().nlsp_generate_smoothed_vectors(dev.ctx.handle, dev.handle, mp, k, sweeps,
                                                               omega, seed, C.byref(h)))
    return SmoothedVectorSet(DeviceDense(dev.ctx, h), sweeps, omega, seed)


# --------------------------------------------------------------- SVD basis --
def svd_basis(s, k: int, ctx: Context | None = None):
    """first_cols(svd_oracle(S).left_vectors, k) (svd.hpp:155-227, dense.hpp:158-164)
    on the device. Returns (P as DeviceDense, singular values, eigensolver sweeps)."""
    ctx = ctx or (s.ctx if isinstance(s, DeviceDense) else default_context())
    sd = _dense(s, ctx)
    h = C.c_void_p()
    sig = np.zeros(max(sd.cols, 1))
    sweeps = C.c_int32(0)
    _check(ctx, L.gpu_lib().nlsp_svd_basis(ctx.handle, sd.handle, k, C.byref(h), L.dptr(sig),
                                           C.byref(sweeps)))
    return DeviceDense(ctx, h), sig[: min(sd.rows, sd.cols)], int(sweeps.value)


# -------------------------------------------------------------- two-level --
class IdentityPreconditioner:
    """two_level.hpp:103-106."""
    kind = L.PRECOND_IDENTITY


class JacobiPreconditioner:
    """two_level.hpp:107-118."""
    kind = L.PRECOND_JACOBI


class TwoLevelPreconditioner:
    """TwoLevelPreconditioner(a, basis_any, omega, nu1, nu2) (two_level.hpp:22-89).
    The basis may be a numpy array (n x k) or a DeviceDense."""

    kind = L.PRECOND_TWOLEVEL

    def __init__(self, a: SparseCsrMatrix, basis_any, omega: float, nu1: int, nu2: int,
                 ctx: Context | None = None):
        # the context of a device-resident basis unless one is given
        ctx = ctx or (basis_any.ctx if isinstance(basis_any, DeviceDense) else None)
        dev = _dev(a, ctx)
        self.ctx = dev.ctx
        if not isinstance(basis_any, DeviceDense):
            basis_any = np.asarray(basis_any, dtype=np.float64)
            if basis_any.ndim != 2:
                raise ValidationError("two-level: basis must be 2-D")
        b = _dense(basis_any, dev.ctx) if (not isinstance(basis_any, np.ndarray) or basis_any.size) \
            else None
        h = C.c_void_p()
        if b is None:  # an n x 0 basis
            if omega < 0.0 or omega > 1.0:
                raise ValidationError("jacobi: omega must lie in [0, 1]")
            raise ValidationError("two-level: empty coarse space")
        _check(dev.ctx, L.gpu_lib().nlsp_twolevel_build(dev.ctx.handle, dev.handle, b.handle, omega,
                                                        nu1, nu2, C.byref(h)))
        self.handle = h
        self._n = a.dim()
        self._k = b.cols
        self._nu1, self._nu2, self._omega = nu1, nu2, omega

    def coarse_dim(self) -> int:
        return self._k

    def cycle(self) -> str:
        """The PCG schedule of this operator (nlsp_twolevel_cycle): "literal",
        "folded", "onepass" or "lean" (the one-pass cycle with beta known before
        and alpha right after the pass over W)."""
        return {0: "literal", 1: "folded", 2: "onepass", 3: "lean"}[L.gpu_lib().nlsp_twolevel_cycle(self.handle)]

    def nu1(self) -> int:
        return self._nu1

    def nu2(self) -> int:
        return self._nu2

    def _export(self):
        basis = np.empty((self._n, self._k))
        chol = np.empty((self._k, self._k))
        coarse = np.empty((self._k, self._k))
        _check(self.ctx, L.gpu_lib().nlsp_twolevel_export(self.ctx.handle, self.handle, L.dptr(basis),
                                                          L.dptr(chol), L.dptr(coarse)))
        return basis, chol, coarse

    def basis(self) -> np.ndarray:
        return self._export()[0]

    def coarse_operator(self) -> np.ndarray:
        """The symmetrised Galerkin operator P^T A P (two_level.hpp:33-51)."""
        return self._export()[2]

    def cholesky_factor(self) -> np.ndarray:
        return self._export()[1]

    def apply(self, a: SparseCsrMatrix, rhs) -> np.ndarray:
        r = np.ascontiguousarray(rhs, dtype=np.float64)
        if r.shape != (a.dim(),):
            raise ValidationError("two-level apply: dimension mismatch")
        dev = _dev(a, self.ctx)
        z = np.empty(a.dim())
        _check(self.ctx, L.gpu_lib().nlsp_twolevel_apply(self.ctx.handle, self.handle, dev.handle,
                                                         L.dptr(r), L.dptr(z)))
        return z

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                L.gpu_lib().nlsp_twolevel_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def build_preconditioner(a, basis, omega, nu1, nu2) -> TwoLevelPreconditioner:
    """two_level.hpp:91-95."""
    return TwoLevelPreconditioner(a, basis, omega, nu1, nu2)


def apply_two_level(m: TwoLevelPreconditioner, a, rhs) -> np.ndarray:
    """two_level.hpp:97-101."""
    return m.apply(a, rhs)


@dataclass
class SolveReport:
    """two_level.hpp:121-132."""
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    true_relative_residual: float = 0.0
    inference_ms: float = 0.0
    setup_ms: float = 0.0
    solve_ms: float = 0.0
    total_ms: float = 0.0
    method: str = ""
    coarse_dim: int = 0
    kernel_launches: int = 0
    onepass_drift: float = 0.0   # one-pass guard: max |c_rec - W^T r| / |W^T r|
    cycle_fallback: bool = False  # the solve was re-run on the folded cycle


@dataclass
class PcgResult:
    """two_level.hpp:134-137."""
    solution: np.ndarray
    report: SolveReport


def pcg(a: SparseCsrMatrix, b, m, delta: float, max_iters: int) -> PcgResult:
    """Preconditioned CG from x0 = 0 with the recurrence-residual stop
    ||r|| / ||b|| < delta (two_level.hpp:141-191), the whole loop on the device."""
    bb = np.ascontiguousarray(b, dtype=np.float64)
    if bb.shape != (a.dim(),):
        raise ValidationError("pcg: dimension mismatch")
    kind = getattr(m, "kind", None)
    if kind is None:
        raise ValidationError("pcg: unsupported preconditioner type")
    dev = _dev(a, getattr(m, "ctx", None))
    x = np.empty(a.dim())
    rep = L.SolveReportC()
    mh = m.handle if kind == L.PRECOND_TWOLEVEL else None
    lib = L.gpu_lib()
    # max_iters is size_t in the reference: clamp Python ints beyond 2^64 - 1
    _check(dev.ctx, lib.nlsp_pcg(dev.ctx.handle, dev.handle, kind, mh, L.dptr(bb), delta,
                                 min(int(max_iters), 2**64 - 1), L.dptr(x), C.byref(rep), None))
    # the history, sized by the iterations run (nlsp_pcg_history)
    hist = np.empty(int(rep.iterations))
    cnt = C.c_uint64(0)
    _check(dev.ctx, lib.nlsp_pcg_history(dev.ctx.handle, L.dptr(hist) if hist.size else None,
                                         hist.size, C.byref(cnt)))
    r = SolveReport(iterations=int(rep.iterations),
                    residual_history=hist[: int(rep.iterations)].copy(),
                    converged=bool(rep.converged),
                    true_relative_residual=float(rep.true_relative_residual),
                    solve_ms=float(rep.solve_ms), total_ms=float(rep.total_ms),
                    coarse_dim=int(rep.coarse_dim), kernel_launches=int(rep.kernel_launches),
                    onepass_drift=float(rep.onepass_drift), cycle_fallback=bool(rep.cycle_fallback),
                    method={0: "plain", 1: "jacobi", 2: "two_level"}[kind])
    return PcgResult(x, r)


def pcg_batch(systems, delta: float, max_iters: int, return_statuses: bool = False):
    """Independent two-level PCG solves in one launch (nlsp_pcg_batch): one
    single-cluster solver per system. `systems` is a sequence of (a, b, m) with
    m a TwoLevelPreconditioner; returns a list of PcgResult (no residual
    history), plus the per-system statuses when asked."""
    systems = list(systems)
    count = len(systems)
    if count == 0:
        return ([], []) if return_statuses else []
    ctx = systems[0][2].ctx
    keep = []
    ah, mh, bp, xp = (C.c_void_p * count)(), (C.c_void_p * count)(), (L.P_dbl * count)(), (L.P_dbl * count)()
    xs = []
    for i, (a, b, m) in enumerate(systems):
        if getattr(m, "kind", None) != L.PRECOND_TWOLEVEL:
            raise ValidationError("pcg_batch: two-level preconditioners only")
        if m.ctx is not ctx:
            raise ValidationError("pcg_batch: all systems must share one context")
        bb = np.ascontiguousarray(b, dtype=np.float64)
        if bb.shape != (a.dim(),):
            raise ValidationError("pcg: dimension mismatch")
        dev = _dev(a, ctx)
        x = np.empty(a.dim())
        keep += [bb, dev]
        xs.append(x)
        ah[i], mh[i] = dev.handle, m.handle
        bp[i], xp[i] = L.dptr(bb), L.dptr(x)
    reps = (L.SolveReportC * count)()
    sts = (C.c_int32 * count)()
    st = L.gpu_lib().nlsp_pcg_batch(ctx.handle, count, ah, mh, bp, delta, int(max_iters), xp, reps, sts)
    if st and not return_statuses:
        _check(ctx, st)
    out = []
    for i in range(count):
        r = reps[i]
        out.append(PcgResult(xs[i], SolveReport(iterations=int(r.iterations), converged=bool(r.converged),
                                                true_relative_residual=float(r.true_relative_residual),
                                                solve_ms=float(r.solve_ms), total_ms=float(r.total_ms),
                                                coarse_dim=int(r.coarse_dim),
                                                kernel_launches=int(r.kernel_launches), method="two_level")))
    return (out, [int(s) for s in sts]) if return_statuses else out
