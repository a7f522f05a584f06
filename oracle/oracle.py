"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY: Python access to the CPU checkers.

  Oracle()            oracle/build/libnlsp_oracle.so — the plain-C restatement
                      (oracle/nlsp_oracle.c), always available once built;
  Reference(strict)   oracle/_ref/libnlsp_ref[_strict].so — the reference's own
                      headers behind oracle/ref_driver.cpp (built only where
                      /root/reference exists; the .so travels to the GPU box).

Both expose the same methods (spmv, inv_diag, jacobi_sweep, block_sweeps,
generate_smoothed_vectors, svd, qr_thin, cholesky, twolevel, pcg). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
use this module, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libnlsp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnlsp_ref.so")
REF_STRICT_SO = os.path.join(HERE, "_ref", "libnlsp_ref_strict.so")
REF_V4_SO = os.path.join(HERE, "_ref", "libnlsp_ref_v4.so")
_V4_FLAGS = ("avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl")


def host_isa() -> str:
    """x86-64-v4 when this host advertises AVX-512 F/BW/CD/DQ/VL, else v3."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = set(line.split(":", 1)[1].split())
                    return "x86-64-v4" if all(x in fl for x in _V4_FLAGS) else "x86-64-v3"
    except OSError:
        pass
    return "x86-64-v3"

u64, dbl, vp = C.c_uint64, C.c_double, C.c_void_p
Pu64, Pdbl, Pu8, Pi32 = (C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                         C.POINTER(C.c_int))

STATUS_NAMES = {0: "ok", 1: "validation", 2: "numeric", 3: "not_spd", 4: "rank_deficient",
                5: "convergence", 8: "io", 9: "other"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.message = msg
        self.kind = STATUS_NAMES.get(code, str(code))


def _d(a):
    return a.ctypes.data_as(Pdbl)


def _u(a):
    return a.ctypes.data_as(Pu64)


def _csr(a):
    """(n, row_ptr u64, col_idx u64, values f64) from a SparseCsrMatrix-like or tuple."""
    if isinstance(a, tuple):
        n, rp, ci, v = a
    else:
        n, rp, ci, v = a.dim(), a.row_ptr(), a.col_idx(), a.values()
    return (int(n), np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint64),
            np.ascontiguousarray(v, np.float64))


@dataclass
class PcgOut:
    x: np.ndarray
    iterations: int
    converged: bool
    true_relative_residual: float
    history: np.ndarray
    solve_ms: float = 0.0


class _TwoLevel:
    def __init__(self, owner, handle, n, k, csr):
        self.owner, self.handle, self.n, self.k, self.csr = owner, handle, n, k, csr

    def export(self):
        basis = np.empty((self.n, self.k))
        chol = np.empty((self.k, self.k))
        coarse = np.empty((self.k, self.k))
        self.owner._export(self, basis, chol, coarse)
        return basis, chol, coarse

    def apply(self, r):
        return self.owner._apply(self, np.ascontiguousarray(r, np.float64))

    def __del__(self):
        try:
            self.owner._destroy(self)
        except Exception:
            pass


class Oracle:
    """The plain-C restatement (oracle/nlsp_oracle.c)."""

    name = "oracle"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {HERE} oracle`")
        lib = C.CDLL(path)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_mix_seed": (u64, [u64, u64]),
            "orc_rng_u64_fill": (None, [u64, u64, Pu64]),
            "orc_rng_normal_fill": (None, [u64, u64, Pdbl]),
            "orc_rng_uniform_fill": (None, [u64, u64, dbl, dbl, Pdbl]),
            "orc_spmv": (C.c_int, [u64, Pu64, Pu64, Pdbl, Pdbl, Pdbl]),
            "orc_inv_diag": (C.c_int, [u64, Pu64, Pu64, Pdbl, dbl, Pdbl]),
            "orc_jacobi_sweep": (C.c_int, [u64, Pu64, Pu64, Pdbl, dbl, u64, Pdbl, Pdbl]),
            "orc_block_sweeps": (C.c_int, [u64, Pu64, Pu64, Pdbl, u64, Pdbl, u64, dbl]),
            "orc_generate_smoothed_vectors": (C.c_int, [u64, Pu64, Pu64, Pdbl, Pu8, u64, u64, dbl, u64, Pdbl]),
            "orc_matmul_tn": (None, [u64, u64, u64, Pdbl, Pdbl, Pdbl]),
            "orc_orthonormality_defect": (dbl, [u64, u64, Pdbl]),
            "orc_jacobi_eigh": (C.c_int, [u64, Pdbl, Pdbl, Pdbl, Pi32]),
            "orc_svd": (C.c_int, [u64, u64, Pdbl, Pdbl, Pdbl, Pdbl, Pi32]),
            "orc_qr_thin": (C.c_int, [u64, u64, Pdbl, Pdbl, Pdbl]),
            "orc_cholesky": (C.c_int, [u64, Pdbl, Pdbl]),
            "orc_cholesky_solve_factored": (None, [u64, Pdbl, Pdbl, Pdbl]),
            "orc_twolevel_create": (C.c_int, [u64, Pu64, Pu64, Pdbl, u64, Pdbl, dbl, u64, u64, C.POINTER(vp)]),
            "orc_twolevel_destroy": (None, [vp]),
            "orc_twolevel_from_parts": (C.c_int, [u64, Pu64, Pu64, Pdbl, u64, Pdbl, Pdbl, dbl, u64, u64,
                                                  C.POINTER(vp)]),
            "orc_twolevel_export": (None, [vp, Pdbl, Pdbl, Pdbl]),
            "orc_twolevel_apply": (C.c_int, [vp, u64, Pu64, Pu64, Pdbl, Pdbl, Pdbl]),
            "orc_pcg": (C.c_int, [u64, Pu64, Pu64, Pdbl, C.c_int, vp, Pdbl, dbl, u64, Pdbl, Pdbl, u64,
                                  Pu64, Pi32, Pdbl]),
        }
        for k, (r, a) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a
        self.lib = lib

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.orc_last_error().decode())

    # rng.hpp
    def mix_seed(self, seed, tag):
        return int(self.lib.orc_mix_seed(seed, tag))

    def rng_normal(self, seed, count):
        out = np.empty(count)
        self.lib.orc_rng_normal_fill(seed, count, _d(out))
        return out

    def rng_uniform(self, seed, count, lo, hi):
        out = np.empty(count)
        self.lib.orc_rng_uniform_fill(seed, count, lo, hi, _d(out))
        return out

    def rng_u64(self, seed, count):
        out = np.empty(count, np.uint64)
        self.lib.orc_rng_u64_fill(seed, count, _u(out))
        return out

    # sparse / smoothing
    def spmv(self, a, x):
        n, rp, ci, v = _csr(a)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(n)
        self._chk(self.lib.orc_spmv(n, _u(rp), _u(ci), _d(v), _d(x), _d(y)))
        return y

    def inv_diag(self, a, omega):
        n, rp, ci, v = _csr(a)
        d = np.empty(n)
        self._chk(self.lib.orc_inv_diag(n, _u(rp), _u(ci), _d(v), omega, _d(d)))
        return d

    def jacobi_sweep(self, a, omega, sweeps, x, b):
        n, rp, ci, v = _csr(a)
        x = np.array(x, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        self._chk(self.lib.orc_jacobi_sweep(n, _u(rp), _u(ci), _d(v), omega, sweeps, _d(x), _d(b)))
        return x

    def block_sweeps(self, a, s, sweeps, omega):
        n, rp, ci, v = _csr(a)
        s = np.array(s, np.float64, order="C")
        self._chk(self.lib.orc_block_sweeps(n, _u(rp), _u(ci), _d(v), s.shape[1], _d(s), sweeps, omega))
        return s

    def generate_smoothed_vectors(self, a, mask, k, sweeps, omega, seed):
        n, rp, ci, v = _csr(a)
        s = np.empty((n, k))
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(np.asarray(mask, bool).astype(np.uint8))
            mp = mask.ctypes.data_as(Pu8)
        self._chk(self.lib.orc_generate_smoothed_vectors(n, _u(rp), _u(ci), _d(v), mp, k, sweeps,
                                                         omega, seed, _d(s)))
        return s

    # dense
    def matmul_tn(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.empty((a.shape[1], b.shape[1]))
        self.lib.orc_matmul_tn(a.shape[0], a.shape[1], b.shape[1], _d(a), _d(b), _d(c))
        return c

    def orthonormality_defect(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return float(self.lib.orc_orthonormality_defect(a.shape[0], a.shape[1], _d(a)))

    def jacobi_eigh(self, g):
        g = np.ascontiguousarray(g, np.float64)
        n = g.shape[0]
        ev, vec, sw = np.empty(n), np.empty((n, n)), C.c_int(0)
        self._chk(self.lib.orc_jacobi_eigh(n, _d(g), _d(ev), _d(vec), C.byref(sw)))
        return ev, vec, sw.value

    def svd(self, s):
        s = np.ascontiguousarray(s, np.float64)
        n, m = s.shape
        r = min(n, m)
        u, sig, vv, sw = np.empty((n, r)), np.empty(r), np.empty((m, r)), C.c_int(0)
        self._chk(self.lib.orc_svd(n, m, _d(s), _d(u), _d(sig), _d(vv), C.byref(sw)))
        return u, sig, vv, sw.value

    def qr_thin(self, m):
        m = np.ascontiguousarray(m, np.float64)
        n, k = m.shape
        q, r = np.empty((n, k)), np.empty((k, k))
        self._chk(self.lib.orc_qr_thin(n, k, _d(m), _d(q), _d(r)))
        return q, r

    def cholesky(self, a):
        a = np.ascontiguousarray(a, np.float64)
        l = np.empty_like(a)
        self._chk(self.lib.orc_cholesky(a.shape[0], _d(a), _d(l)))
        return l

    def cholesky_solve(self, a, rhs):
        l = self.cholesky(a)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.empty_like(rhs)
        self.lib.orc_cholesky_solve_factored(l.shape[0], _d(l), _d(rhs), _d(x))
        return x

    # two-level / pcg
    def twolevel(self, a, basis, omega, nu1, nu2):
        csr = _csr(a)
        n, rp, ci, v = csr
        basis = np.ascontiguousarray(basis, np.float64)
        k = basis.shape[1] if basis.ndim == 2 else 0
        h = vp()
        self._chk(self.lib.orc_twolevel_create(n, _u(rp), _u(ci), _d(v), k, _d(basis), omega, nu1,
                                               nu2, C.byref(h)))
        return _TwoLevel(self, h, n, k, csr)

    def twolevel_from_parts(self, a, basis, coarse, omega, nu1, nu2):
        csr = _csr(a)
        n, rp, ci, v = csr
        basis = np.ascontiguousarray(basis, np.float64)
        coarse = np.ascontiguousarray(coarse, np.float64)
        h = vp()
        self._chk(self.lib.orc_twolevel_from_parts(n, _u(rp), _u(ci), _d(v), basis.shape[1], _d(basis),
                                                   _d(coarse), omega, nu1, nu2, C.byref(h)))
        return _TwoLevel(self, h, n, basis.shape[1], csr)

    def _export(self, t, basis, chol, coarse):
        self.lib.orc_twolevel_export(t.handle, _d(basis), _d(chol), _d(coarse))

    def _apply(self, t, r):
        n, rp, ci, v = t.csr
        z = np.empty(n)
        self._chk(self.lib.orc_twolevel_apply(t.handle, n, _u(rp), _u(ci), _d(v), _d(r), _d(z)))
        return z

    def _destroy(self, t):
        if t.handle:
            self.lib.orc_twolevel_destroy(t.handle)
            t.handle = None

    def pcg(self, a, b, kind, t, delta, max_iters):
        n, rp, ci, v = _csr(a)
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(n)
        cap = int(min(max_iters, 10_000_000))
        hist = np.empty(max(cap, 1))
        it, conv, tr = C.c_uint64(0), C.c_int(0), C.c_double(0.0)
        import time
        t0 = time.perf_counter()
        self._chk(self.lib.orc_pcg(n, _u(rp), _u(ci), _d(v), kind, t.handle if t else None, _d(b),
                                   delta, max_iters, _d(x), _d(hist), cap, C.byref(it),
                                   C.byref(conv), C.byref(tr)))
        ms = (time.perf_counter() - t0) * 1e3
        return PcgOut(x, int(it.value), bool(conv.value), float(tr.value),
                      hist[: min(int(it.value), cap)].copy(), ms)


def reference_available(strict: bool = False) -> bool:
    return os.path.exists(REF_STRICT_SO if strict else REF_SO)


class Reference:
    """The reference's own code (oracle/_ref), default or -ffp-contract=off build."""

    def __init__(self, strict: bool = False, native: bool = False):
        """native: the build closest to the reference's -march=native on this
        host (x86-64-v4 where AVX-512 is present) — the CPU baselines use it."""
        path = REF_STRICT_SO if strict else REF_SO
        self.isa = "x86-64-v3"
        if native and not strict and host_isa() == "x86-64-v4" and os.path.exists(REF_V4_SO):
            path, self.isa = REF_V4_SO, "x86-64-v4"
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {HERE} ref` where /root/reference exists")
        self.name = "ref_strict" if strict else "ref"
        lib = C.CDLL(path)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_csr_create": (vp, [u64, u64, Pu64, Pu64, Pdbl]),
            "ref_csr_destroy": (None, [vp]),
            "ref_csr_nnz": (u64, [vp]),
            "ref_csr_dim": (u64, [vp]),
            "ref_csr_export": (None, [vp, Pu64, Pu64, Pdbl]),
            "ref_csr_from_triplets": (vp, [u64, u64, Pu64, Pu64, Pdbl, Pi32]),
            "ref_spmv": (C.c_int, [vp, u64, Pdbl, Pdbl]),
            "ref_fem_instance": (C.c_int, [C.c_int, u64, dbl, u64, Pu64, Pu64, Pu64, Pu64, Pdbl, Pdbl, Pu8]),
            "ref_mix_seed": (u64, [u64, u64]),
            "ref_save_instance": (C.c_int, [C.c_int, u64, dbl, u64, C.c_char_p]),
            "ref_aggregate_nodes": (C.c_int, [vp, dbl, Pu64, Pu64]),
            "ref_mlp_create_save": (C.c_int, [Pu64, u64, u64, C.c_char_p]),
            "ref_mlp_params": (C.c_int, [C.c_char_p, Pu64, Pdbl]),
            "ref_mlp_forward": (C.c_int, [C.c_char_p, Pdbl, Pdbl]),
            "ref_infer_basis": (C.c_int, [C.c_char_p, u64, u64, Pdbl, Pdbl, Pu64, Pdbl]),
            "ref_sa_prolongator": (C.c_int, [vp, dbl, dbl, Pu64, Pdbl]),
            "ref_load_matrix_market": (vp, [C.c_char_p, Pi32]),
            "ref_save_matrix_market": (C.c_int, [vp, C.c_char_p]),
            "ref_load_instance": (vp, [C.c_char_p, Pi32]),
            "ref_instance_destroy": (None, [vp]),
            "ref_instance_meta": (None, [vp, Pi32, Pu64, Pu64, Pdbl, Pdbl, Pu64, Pu64, Pu64]),
            "ref_instance_matrix": (vp, [vp]),
            "ref_instance_arrays": (None, [vp, Pdbl, Pu8, Pdbl, Pu64, Pdbl]),
            "ref_rng_normal": (None, [u64, u64, Pdbl]),
            "ref_rng_uniform": (None, [u64, u64, dbl, dbl, Pdbl]),
            "ref_rng_u64": (None, [u64, u64, Pu64]),
            "ref_jacobi_inv_diag": (C.c_int, [vp, dbl, Pdbl]),
            "ref_jacobi_sweep": (C.c_int, [vp, dbl, u64, Pdbl, Pdbl]),
            "ref_generate_smoothed_vectors": (C.c_int, [vp, Pu8, u64, u64, dbl, u64, Pdbl]),
            "ref_block_sweeps": (C.c_int, [vp, u64, Pdbl, u64, dbl]),
            "ref_matmul_tn": (C.c_int, [u64, u64, u64, Pdbl, Pdbl, Pdbl]),
            "ref_jacobi_eigh": (C.c_int, [u64, Pdbl, Pdbl, Pdbl, Pi32]),
            "ref_svd": (C.c_int, [u64, u64, Pdbl, Pdbl, Pdbl, Pdbl, Pi32]),
            "ref_orthonormality_defect": (dbl, [u64, u64, Pdbl]),
            "ref_principal_angles": (C.c_int, [u64, u64, Pdbl, Pdbl, Pdbl]),
            "ref_captured_energy": (dbl, [u64, u64, u64, Pdbl, Pdbl]),
            "ref_qr_thin": (C.c_int, [u64, u64, Pdbl, Pdbl, Pdbl]),
            "ref_cholesky": (C.c_int, [u64, Pdbl, Pdbl]),
            "ref_cholesky_solve": (C.c_int, [u64, Pdbl, Pdbl, Pdbl]),
            "ref_twolevel_create": (vp, [vp, u64, Pdbl, dbl, u64, u64, Pi32]),
            "ref_twolevel_destroy": (None, [vp]),
            "ref_twolevel_from_parts": (vp, [vp, u64, Pdbl, Pdbl, dbl, u64, u64, Pi32]),
            "ref_pcg_parallel": (C.c_int, [vp, C.c_int, vp, Pdbl, dbl, u64, C.c_int, Pdbl, Pu64]),
            "ref_twolevel_export": (None, [vp, Pdbl, Pdbl, Pdbl]),
            "ref_twolevel_galerkin": (None, [vp, vp, Pdbl]),
            "ref_twolevel_apply": (C.c_int, [vp, vp, Pdbl, Pdbl]),
            "ref_pcg": (C.c_int, [vp, C.c_int, vp, Pdbl, dbl, u64, Pdbl, Pdbl, u64, Pu64, Pi32, Pdbl, Pdbl]),
        }
        for k, (r, a) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a
        self.lib = lib
        self._csr_cache = {}

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def handle(self, a):
        key = id(a)
        hit = self._csr_cache.get(key)
        if hit is not None and hit[0] is a:
            return hit[1]
        n, rp, ci, v = _csr(a)
        h = self.lib.ref_csr_create(n, v.size, _u(rp), _u(ci), _d(v))
        if not h:
            raise OracleError(1, self.lib.ref_last_error().decode())
        self._csr_cache[key] = (a, h)
        return h

    def mix_seed(self, seed, tag):
        return int(self.lib.ref_mix_seed(seed, tag))

    def rng_normal(self, seed, count):
        out = np.empty(count)
        self.lib.ref_rng_normal(seed, count, _d(out))
        return out

    def rng_uniform(self, seed, count, lo, hi):
        out = np.empty(count)
        self.lib.ref_rng_uniform(seed, count, lo, hi, _d(out))
        return out

    def rng_u64(self, seed, count):
        out = np.empty(count, np.uint64)
        self.lib.ref_rng_u64(seed, count, _u(out))
        return out

    def fem_instance(self, family, grid_n, jitter, seed):
        n, nnz = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.ref_fem_instance(family, grid_n, jitter, seed, C.byref(n), C.byref(nnz),
                                            None, None, None, None, None))
        n, nnz = n.value, nnz.value
        rp, ci = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint64)
        v, rhs, mask = np.empty(nnz), np.empty(n), np.empty(n, np.uint8)
        self._chk(self.lib.ref_fem_instance(family, grid_n, jitter, seed, C.byref(C.c_uint64()),
                                            C.byref(C.c_uint64()), _u(rp), _u(ci), _d(v), _d(rhs),
                                            mask.ctypes.data_as(Pu8)))
        return (int(n), rp, ci, v), rhs, mask

    # --- on-disk inputs (sparse.hpp:148-194, instance_io.hpp:99-185) ---------
    def _csr_out(self, h, dim):
        nnz = self.lib.ref_csr_nnz(h)
        rp, ci, v = np.empty(dim + 1, np.uint64), np.empty(nnz, np.uint64), np.empty(nnz)
        self.lib.ref_csr_export(h, _u(rp), _u(ci), _d(v))
        return (dim, rp, ci, v)

    # --- MLP inference (mlp.hpp, train.hpp) --------------------------------
    def mlp_create_save(self, widths, seed, path):
        w = np.ascontiguousarray(widths, np.uint64)
        self._chk(self.lib.ref_mlp_create_save(_u(w), w.size, seed, str(path).encode()))

    def mlp_params(self, path):
        np_ = C.c_uint64(0)
        self._chk(self.lib.ref_mlp_params(str(path).encode(), C.byref(np_), None))
        out = np.empty(np_.value)
        self._chk(self.lib.ref_mlp_params(str(path).encode(), C.byref(np_), _d(out)))
        return out

    def mlp_forward(self, path, x, out_width):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(out_width)
        self._chk(self.lib.ref_mlp_forward(str(path).encode(), _d(x), _d(y)))
        return y

    def infer_basis(self, path, s, r):
        """infer_basis (train.hpp:52-62) -> (q n x r, ms of the call)."""
        s = np.ascontiguousarray(s, np.float64)
        n, k = s.shape
        q = np.empty((n, r))
        rr, ms = C.c_uint64(0), C.c_double(0)
        self._chk(self.lib.ref_infer_basis(str(path).encode(), n, k, _d(s), _d(q), C.byref(rr), C.byref(ms)))
        assert rr.value == r
        return q, float(ms.value)

    def aggregate_nodes(self, a, theta):
        """aggregate_nodes (sa.hpp:18-76): (aggregate id per node, count)."""
        n = _csr(a)[0]
        agg, nc = np.empty(n, np.uint64), C.c_uint64(0)
        self._chk(self.lib.ref_aggregate_nodes(self.handle(a), theta, _u(agg), C.byref(nc)))
        return agg, int(nc.value)

    def sa_prolongator(self, a, theta=0.25, omega=0.66):
        """sa_prolongator (sa.hpp:78-109): dense n x nc."""
        n = _csr(a)[0]
        nc = C.c_uint64(0)
        self._chk(self.lib.ref_sa_prolongator(self.handle(a), theta, omega, C.byref(nc), None))
        p = np.empty((n, nc.value))
        self._chk(self.lib.ref_sa_prolongator(self.handle(a), theta, omega, C.byref(nc), _d(p)))
        return p

    def save_instance(self, family, grid_n, jitter, seed, path):
        self._chk(self.lib.ref_save_instance(family, grid_n, jitter, seed, str(path).encode()))

    def load_matrix_market(self, path):
        """(n, rp, ci, v) or OracleError(status, message)."""
        st = C.c_int32(0)
        h = self.lib.ref_load_matrix_market(str(path).encode(), C.byref(st))
        self._chk(st.value)
        try:
            return self._csr_out(h, int(self.lib.ref_csr_dim(h)))
        finally:
            self.lib.ref_csr_destroy(h)

    def save_matrix_market(self, a, path):
        self._chk(self.lib.ref_save_matrix_market(self.handle(a), str(path).encode()))

    def load_instance(self, path):
        st = C.c_int32(0)
        h = self.lib.ref_load_instance(str(path).encode(), C.byref(st))
        self._chk(st.value)
        try:
            fam, gn, seed = C.c_int32(0), C.c_uint64(0), C.c_uint64(0)
            jit, alpha = C.c_double(0), C.c_double(0)
            n, nv, nt = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
            self.lib.ref_instance_meta(h, C.byref(fam), C.byref(gn), C.byref(seed), C.byref(jit),
                                       C.byref(alpha), C.byref(n), C.byref(nv), C.byref(nt))
            n, nv, nt = n.value, nv.value, nt.value
            cc = 3 if fam.value == 1 else 1
            rhs, mask = np.empty(n), np.empty(nv, np.uint8)
            vert, tri, coeff = np.empty((nv, 2)), np.empty((nt, 3), np.uint64), np.empty((nt, cc))
            self.lib.ref_instance_arrays(h, _d(rhs), mask.ctypes.data_as(Pu8), _d(vert), _u(tri), _d(coeff))
            mh = self.lib.ref_instance_matrix(h)
            try:
                a = self._csr_out(mh, n)
            finally:
                self.lib.ref_csr_destroy(mh)
            return dict(family=fam.value, grid_n=gn.value, seed=seed.value, jitter=jit.value,
                        alpha=alpha.value, matrix=a, rhs=rhs, mask=mask, vertices=vert, triangles=tri,
                        coefficients=coeff)
        finally:
            self.lib.ref_instance_destroy(h)

    def from_triplets(self, n, i, j, v):
        i = np.ascontiguousarray(i, np.uint64)
        j = np.ascontiguousarray(j, np.uint64)
        v = np.ascontiguousarray(v, np.float64)
        st = C.c_int(0)
        h = self.lib.ref_csr_from_triplets(n, v.size, _u(i), _u(j), _d(v), C.byref(st))
        self._chk(st.value)
        nnz = int(self.lib.ref_csr_nnz(h))
        rp, ci, vv = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint64), np.empty(nnz)
        self.lib.ref_csr_export(h, _u(rp), _u(ci), _d(vv))
        self.lib.ref_csr_destroy(h)
        return (n, rp, ci, vv)

    def spmv(self, a, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(_csr(a)[0])
        self._chk(self.lib.ref_spmv(self.handle(a), x.size, _d(x), _d(y)))
        return y

    def inv_diag(self, a, omega):
        d = np.empty(_csr(a)[0])
        self._chk(self.lib.ref_jacobi_inv_diag(self.handle(a), omega, _d(d)))
        return d

    def jacobi_sweep(self, a, omega, sweeps, x, b):
        x = np.array(x, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        self._chk(self.lib.ref_jacobi_sweep(self.handle(a), omega, sweeps, _d(x), _d(b)))
        return x

    def block_sweeps(self, a, s, sweeps, omega):
        s = np.array(s, np.float64, order="C")
        self._chk(self.lib.ref_block_sweeps(self.handle(a), s.shape[1], _d(s), sweeps, omega))
        return s

    def generate_smoothed_vectors(self, a, mask, k, sweeps, omega, seed):
        n = _csr(a)[0]
        s = np.empty((n, k))
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(np.asarray(mask, bool).astype(np.uint8))
            mp = mask.ctypes.data_as(Pu8)
        self._chk(self.lib.ref_generate_smoothed_vectors(self.handle(a), mp, k, sweeps, omega, seed, _d(s)))
        return s

    def matmul_tn(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.empty((a.shape[1], b.shape[1]))
        self._chk(self.lib.ref_matmul_tn(a.shape[0], a.shape[1], b.shape[1], _d(a), _d(b), _d(c)))
        return c

    def orthonormality_defect(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return float(self.lib.ref_orthonormality_defect(a.shape[0], a.shape[1], _d(a)))

    def principal_angles(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(a.shape[1])
        self._chk(self.lib.ref_principal_angles(a.shape[0], a.shape[1], _d(a), _d(b), _d(out)))
        return out

    def captured_energy(self, p, s):
        p = np.ascontiguousarray(p, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        return float(self.lib.ref_captured_energy(p.shape[0], p.shape[1], s.shape[1], _d(p), _d(s)))

    def jacobi_eigh(self, g):
        g = np.ascontiguousarray(g, np.float64)
        n = g.shape[0]
        ev, vec, sw = np.empty(n), np.empty((n, n)), C.c_int(0)
        self._chk(self.lib.ref_jacobi_eigh(n, _d(g), _d(ev), _d(vec), C.byref(sw)))
        return ev, vec, sw.value

    def svd(self, s):
        s = np.ascontiguousarray(s, np.float64)
        n, m = s.shape
        r = min(n, m)
        u, sig, vv, sw = np.empty((n, r)), np.empty(r), np.empty((m, r)), C.c_int(0)
        self._chk(self.lib.ref_svd(n, m, _d(s), _d(u), _d(sig), _d(vv), C.byref(sw)))
        return u, sig, vv, sw.value

    def qr_thin(self, m):
        m = np.ascontiguousarray(m, np.float64)
        n, k = m.shape
        q, r = np.empty((n, k)), np.empty((k, k))
        self._chk(self.lib.ref_qr_thin(n, k, _d(m), _d(q), _d(r)))
        return q, r

    def cholesky(self, a):
        a = np.ascontiguousarray(a, np.float64)
        l = np.empty_like(a)
        self._chk(self.lib.ref_cholesky(a.shape[0], _d(a), _d(l)))
        return l

    def cholesky_solve(self, a, rhs):
        a = np.ascontiguousarray(a, np.float64)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.empty_like(rhs)
        self._chk(self.lib.ref_cholesky_solve(a.shape[0], _d(a), _d(rhs), _d(x)))
        return x

    def twolevel(self, a, basis, omega, nu1, nu2):
        basis = np.ascontiguousarray(basis, np.float64)
        k = basis.shape[1] if basis.ndim == 2 else 0
        st = C.c_int(0)
        h = self.lib.ref_twolevel_create(self.handle(a), k, _d(basis), omega, nu1, nu2, C.byref(st))
        self._chk(st.value)
        return _TwoLevel(self, h, _csr(a)[0], k, a)

    def twolevel_from_parts(self, a, basis, coarse, omega, nu1, nu2):
        """Reference TwoLevelPreconditioner with basis_/coarse_/smoother_ seated
        from given parts (the constructor body is bypassed; see ref_driver.cpp)."""
        basis = np.ascontiguousarray(basis, np.float64)
        coarse = np.ascontiguousarray(coarse, np.float64)
        st = C.c_int(0)
        h = self.lib.ref_twolevel_from_parts(self.handle(a), basis.shape[1], _d(basis), _d(coarse),
                                             omega, nu1, nu2, C.byref(st))
        self._chk(st.value)
        return _TwoLevel(self, h, _csr(a)[0], basis.shape[1], a)

    def pcg_parallel(self, a, b, kind, t, delta, max_iters, threads):
        """`threads` concurrent reference pcg solves; returns (wall ms, iterations)."""
        b = np.ascontiguousarray(b, np.float64)
        ms, it = C.c_double(0.0), C.c_uint64(0)
        self._chk(self.lib.ref_pcg_parallel(self.handle(a), kind, t.handle if t else None, _d(b), delta,
                                            max_iters, threads, C.byref(ms), C.byref(it)))
        return float(ms.value), int(it.value)

    def galerkin(self, t):
        out = np.empty((t.k, t.k))
        self.lib.ref_twolevel_galerkin(t.handle, self.handle(t.csr), _d(out))
        return out

    def _export(self, t, basis, chol, coarse):
        self.lib.ref_twolevel_export(t.handle, _d(basis), _d(chol), _d(coarse))

    def _apply(self, t, r):
        z = np.empty(t.n)
        self._chk(self.lib.ref_twolevel_apply(t.handle, self.handle(t.csr), _d(r), _d(z)))
        return z

    def _destroy(self, t):
        if t.handle:
            self.lib.ref_twolevel_destroy(t.handle)
            t.handle = None

    def pcg(self, a, b, kind, t, delta, max_iters):
        b = np.ascontiguousarray(b, np.float64)
        n = _csr(a)[0]
        x = np.empty(n)
        cap = int(min(max_iters, 10_000_000))
        hist = np.empty(max(cap, 1))
        it, conv, tr, ms = C.c_uint64(0), C.c_int(0), C.c_double(0.0), C.c_double(0.0)
        self._chk(self.lib.ref_pcg(self.handle(a), kind, t.handle if t else None, _d(b), delta,
                                   max_iters, _d(x), _d(hist), cap, C.byref(it), C.byref(conv),
                                   C.byref(tr), C.byref(ms)))
        return PcgOut(x, int(it.value), bool(conv.value), float(tr.value),
                      hist[: min(int(it.value), cap)].copy(), float(ms.value))

    def __del__(self):
        try:
            for _, h in self._csr_cache.values():
                self.lib.ref_csr_destroy(h)
        except Exception:
            pass
