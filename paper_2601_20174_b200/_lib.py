"""ctypes bindings for libnlsp_gpu.so (include/nlsp_gpu.h) and libnlsp_inputs.so
(include/nlsp_inputs.h).

The libraries are built in-tree by ``make -C paper_2601_20174_b200`` (or
``__graft_entry__.build()``). Loading fails loudly when they are missing: there
is no Python or CPU fallback for the solver path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
GPU_LIB_PATH = os.environ.get("NLSP_GPU_LIB") or os.path.join(HERE, "libnlsp_gpu.so")
INPUTS_LIB_PATH = os.path.join(HERE, "libnlsp_inputs.so")
IO_LIB_PATH = os.path.join(HERE, "libnlsp_io.so")

c_u64 = C.c_uint64
c_i32 = C.c_int32
c_dbl = C.c_double
P_u64 = C.POINTER(C.c_uint64)
P_dbl = C.POINTER(C.c_double)
P_u8 = C.POINTER(C.c_uint8)
P_i32 = C.POINTER(C.c_int32)
vp = C.c_void_p

# nlsp_status
NLSP_OK = 0
NLSP_E_VALIDATION = 1
NLSP_E_NUMERIC = 2
NLSP_E_NOT_SPD = 3
NLSP_E_RANK_DEFICIENT = 4
NLSP_E_CONVERGENCE = 5
NLSP_E_CUDA = 6
NLSP_E_OOM = 7
NLSP_E_IO = 8  # nlsp::IoError (include/nlsp_io.h)

PRECOND_IDENTITY = 0
PRECOND_JACOBI = 1
PRECOND_TWOLEVEL = 2
NLSP_S0_DRAW_HOST = 0
NLSP_S0_DRAW_DEVICE = 1


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", c_u64),
        ("converged", c_i32),
        ("precond_kind", c_i32),
        ("true_relative_residual", c_dbl),
        ("final_relative_residual", c_dbl),
        ("solve_ms", c_dbl),
        ("total_ms", c_dbl),
        ("coarse_dim", c_u64),
        ("kernel_launches", c_u64),
        ("h2d_bytes", c_u64),
        ("d2h_bytes", c_u64),
        ("onepass_drift", c_dbl),
        ("cycle_fallback", c_i32),
        ("reserved", c_i32),
    ]


class KernelStatC(C.Structure):
    _fields_ = [
        ("name", C.c_char * 32),
        ("launches", c_u64),
        ("total_ms", c_dbl),
        ("bytes_per_launch", c_dbl),
    ]


class ProblemSpecC(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("nx", c_u64),
        ("ny", c_u64),
        ("nz", c_u64),
        ("seed", c_u64),
        ("epsilon", c_dbl),
        ("theta", c_dbl),
        ("corr_len", c_dbl),
        ("variance", c_dbl),
        ("blocks", c_u64),
        ("young_lo", c_dbl),
        ("young_hi", c_dbl),
        ("poisson", c_dbl),
        ("rhs_uniform", C.c_int),
    ]


# (name, restype, argtypes) for every symbol include/nlsp_gpu.h declares
GPU_SYMBOLS = [
    ("nlsp_version", C.c_char_p, []),
    ("nlsp_ctx_create", C.c_int, [C.c_int, C.POINTER(vp)]),
    ("nlsp_ctx_destroy", None, [vp]),
    ("nlsp_last_error", C.c_char_p, [vp]),
    ("nlsp_ctx_stream", vp, [vp]),
    ("nlsp_ctx_synchronize", C.c_int, [vp]),
    ("nlsp_ctx_kernel_launches", c_u64, [vp]),
    ("nlsp_csr_upload", C.c_int, [vp, c_u64, c_u64, P_u64, P_u64, P_dbl, C.POINTER(vp)]),
    ("nlsp_csr_destroy", None, [vp]),
    ("nlsp_csr_dims", None, [vp, P_u64, P_u64]),
    ("nlsp_csr_format", c_i32, [vp, P_i32, P_i32, P_u64]),
    ("nlsp_csr_geometry", c_i32, [vp, vp, P_u64, P_i32, P_i32]),
    ("nlsp_pcg_batch", c_i32, [vp, c_u64, C.POINTER(vp), C.POINTER(vp), C.POINTER(P_dbl), c_dbl, c_u64,
                                C.POINTER(P_dbl), C.POINTER(SolveReportC), P_i32]),
    ("nlsp_sa_aggregate", c_i32, [c_u64, c_u64, P_u64, P_u64, P_dbl, c_dbl, P_u64, P_u64]),
    ("nlsp_sa_prolongator", c_i32, [vp, c_u64, c_u64, P_u64, P_u64, P_dbl, c_dbl, c_dbl, C.POINTER(vp)]),
    ("nlsp_mlp_upload", c_i32, [vp, P_u64, c_u64, P_dbl, c_u64, C.POINTER(vp)]),
    ("nlsp_mlp_destroy", None, [vp]),
    ("nlsp_mlp_forward", c_i32, [vp, vp, P_dbl, P_dbl]),
    ("nlsp_mlp_infer_basis", c_i32, [vp, vp, vp, C.POINTER(vp)]),
    ("nlsp_spmv", C.c_int, [vp, vp, P_dbl, P_dbl]),
    ("nlsp_spmv_device", C.c_int, [vp, vp, vp, vp]),
    ("nlsp_csr_diagonal", C.c_int, [vp, vp, P_dbl]),
    ("nlsp_dense_upload", C.c_int, [vp, c_u64, c_u64, P_dbl, C.POINTER(vp)]),
    ("nlsp_dense_export", C.c_int, [vp, vp, P_dbl]),
    ("nlsp_dense_dims", None, [vp, P_u64, P_u64]),
    ("nlsp_dense_destroy", None, [vp]),
    ("nlsp_dense_data", vp, [vp]),
    ("nlsp_jacobi_sweeps", C.c_int, [vp, vp, c_dbl, c_u64, P_dbl, P_dbl]),
    ("nlsp_smooth_vectors", C.c_int, [vp, vp, vp, c_u64, c_dbl]),
    ("nlsp_generate_smoothed_vectors", C.c_int, [vp, vp, P_u8, c_u64, c_u64, c_dbl, c_u64, C.POINTER(vp)]),
    ("nlsp_ctx_set_s0_draw", C.c_int, [vp, c_i32]),
    ("nlsp_ctx_last_s0_draw", c_i32, [vp]),
    ("nlsp_mt19937_64_words", C.c_int, [vp, c_u64, c_u64, P_u64]),
    ("nlsp_svd_basis", C.c_int, [vp, vp, c_u64, C.POINTER(vp), P_dbl, P_i32]),
    ("nlsp_twolevel_build", C.c_int, [vp, vp, vp, c_dbl, c_u64, c_u64, C.POINTER(vp)]),
    ("nlsp_twolevel_destroy", None, [vp]),
    ("nlsp_twolevel_dims", None, [vp, P_u64, P_u64]),
    ("nlsp_twolevel_cycle", C.c_int, [vp]),
    ("nlsp_twolevel_export", C.c_int, [vp, vp, P_dbl, P_dbl, P_dbl]),
    ("nlsp_twolevel_apply", C.c_int, [vp, vp, vp, P_dbl, P_dbl]),
    ("nlsp_pcg", C.c_int, [vp, vp, C.c_int, vp, P_dbl, c_dbl, c_u64, P_dbl, C.POINTER(SolveReportC), P_dbl]),
    ("nlsp_pcg_device", C.c_int, [vp, vp, C.c_int, vp, vp, c_dbl, c_u64, vp, C.POINTER(SolveReportC), P_dbl]),
    ("nlsp_pcg_history", C.c_int, [vp, P_dbl, c_u64, C.POINTER(c_u64)]),
    ("nlsp_pcg_profile", C.c_int, [vp, vp, C.c_int, vp, vp, c_u64, C.POINTER(KernelStatC), C.c_int]),
]

INPUT_SYMBOLS = [
    ("nlsp_problem_create", C.c_int, [C.POINTER(ProblemSpecC), C.POINTER(vp)]),
    ("nlsp_problem_destroy", None, [vp]),
    ("nlsp_problem_n", c_u64, [vp]),
    ("nlsp_problem_nnz", c_u64, [vp]),
    ("nlsp_problem_export", None, [vp, P_u64, P_u64, P_dbl, P_dbl, P_u8]),
    ("nlsp_problem_coef_len", c_u64, [vp]),
    ("nlsp_problem_export_coef", None, [vp, P_dbl]),
    ("nlsp_inputs_last_error", C.c_char_p, []),
    ("nlsp_mix_seed", c_u64, [c_u64, c_u64]),
    ("nlsp_rng_normal_fill", None, [c_u64, c_u64, P_dbl]),
    ("nlsp_rng_uniform_fill", None, [c_u64, c_u64, c_dbl, c_dbl, P_dbl]),
    ("nlsp_rng_normal_serial", None, [c_u64, c_u64, c_dbl, P_dbl]),
    ("nlsp_rng_normal_chunks", None, [c_u64, c_u64, c_u64, c_dbl, C.c_uint32, P_dbl]),
    ("nlsp_mt19937_64_fill", None, [c_u64, c_u64, c_u64, P_u64]),
    ("nlsp_mt19937_64_jump_fill", C.c_int, [c_u64, c_u64, c_u64, P_u64]),
    ("nlsp_smoothed_s0", None, [c_u64, c_u64, c_u64, P_u8, P_dbl]),
]



class HostCsrC(C.Structure):
    """nlsp_host_csr (include/nlsp_io.h)."""
    _fields_ = [("n", c_u64), ("nnz", c_u64), ("row_ptr", P_u64), ("col_idx", P_u64), ("values", P_dbl)]


class InstanceC(C.Structure):
    """nlsp_instance (include/nlsp_io.h)."""
    _fields_ = [
        ("family", C.c_int),
        ("grid_n", c_u64),
        ("seed", c_u64),
        ("jitter", c_dbl),
        ("alpha", c_dbl),
        ("matrix", HostCsrC),
        ("rhs", P_dbl),
        ("n_vertices", c_u64),
        ("vertices", P_dbl),
        ("boundary_mask", P_u8),
        ("n_triangles", c_u64),
        ("triangles", P_u64),
        ("coeff_cols", c_u64),
        ("coefficients", P_dbl),
    ]


class HostMlpC(C.Structure):
    """nlsp_host_mlp (include/nlsp_io.h)."""
    _fields_ = [("nwidths", c_u64), ("widths", P_u64), ("nparams", c_u64), ("params", P_dbl),
                ("manifest", C.c_char_p)]


IO_SYMBOLS = [
    ("nlsp_io_load_matrix_market", C.c_int, [C.c_char_p, C.POINTER(HostCsrC)]),
    ("nlsp_io_save_matrix_market", C.c_int, [C.POINTER(HostCsrC), C.c_char_p]),
    ("nlsp_io_csr_free", None, [C.POINTER(HostCsrC)]),
    ("nlsp_io_load_instance", C.c_int, [C.c_char_p, C.POINTER(InstanceC)]),
    ("nlsp_io_instance_free", None, [C.POINTER(InstanceC)]),
    ("nlsp_io_mlp_load", C.c_int, [C.c_char_p, C.POINTER(HostMlpC)]),
    ("nlsp_io_mlp_save", C.c_int, [C.POINTER(HostMlpC), C.c_char_p]),
    ("nlsp_io_mlp_init", C.c_int, [P_u64, c_u64, c_u64, C.POINTER(HostMlpC)]),
    ("nlsp_io_mlp_free", None, [C.POINTER(HostMlpC)]),
    ("nlsp_io_last_error", C.c_char_p, []),
]

_lock = threading.Lock()
_gpu = None
_inputs = None
_io = None


def _bind(lib, table):
    for name, res, args in table:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def gpu_lib():
    """libnlsp_gpu.so with every declared symbol bound. Raises if not built."""
    global _gpu
    with _lock:
        if _gpu is None:
            if not os.path.exists(GPU_LIB_PATH):
                raise RuntimeError(
                    f"{GPU_LIB_PATH} is missing: build it with `make -C {HERE}` "
                    "(there is no CPU fallback for the solver)")
            _gpu = _bind(C.CDLL(GPU_LIB_PATH), GPU_SYMBOLS)
        return _gpu


def inputs_lib():
    global _inputs
    with _lock:
        if _inputs is None:
            if not os.path.exists(INPUTS_LIB_PATH):
                raise RuntimeError(f"{INPUTS_LIB_PATH} is missing: build it with `make -C {HERE}`")
            _inputs = _bind(C.CDLL(INPUTS_LIB_PATH), INPUT_SYMBOLS)
        return _inputs


def io_lib():
    """libnlsp_io.so (host C++ loaders, include/nlsp_io.h)."""
    global _io
    with _lock:
        if _io is None:
            if not os.path.exists(IO_LIB_PATH):
                raise RuntimeError(f"{IO_LIB_PATH} is missing: build it with `make -C {HERE}`")
            _io = _bind(C.CDLL(IO_LIB_PATH), IO_SYMBOLS)
        return _io


def dptr(a):
    return a.ctypes.data_as(P_dbl)


def u64ptr(a):
    return a.ctypes.data_as(P_u64)


def u8ptr(a):
    return a.ctypes.data_as(P_u8)
