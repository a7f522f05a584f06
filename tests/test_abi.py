"""The drop-in boundary without a GPU: the C-ABI libraries load, export every
symbol include/*.h declares, the ctypes table matches the headers, and the
product fails loudly (no CPU fallback) when no sm_100 device is present."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2601_20174_b200 import _lib as L

HEADERS = {"nlsp_gpu.h": L.GPU_LIB_PATH, "nlsp_inputs.h": L.INPUTS_LIB_PATH, "nlsp_io.h": L.IO_LIB_PATH}


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = set(re.findall(r"\b(nlsp_[a-z0-9_]+)\s*\(", txt))
    return names


@pytest.mark.parametrize("header", sorted(HEADERS))
def test_library_exports_every_declared_symbol(header):
    lib = C.CDLL(HEADERS[header])
    names = declared(header)
    assert names, header
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", HEADERS[header]], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (nlsp_[a-z0-9_]+)", out))
    assert names <= exported


def test_ctypes_table_covers_headers():
    assert declared("nlsp_gpu.h") == {n for n, _, _ in L.GPU_SYMBOLS}
    assert declared("nlsp_inputs.h") == {n for n, _, _ in L.INPUT_SYMBOLS}
    assert declared("nlsp_io.h") == {n for n, _, _ in L.IO_SYMBOLS}


def test_gpu_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", L.GPU_LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = L.gpu_lib()
    h = C.c_void_p()
    assert lib.nlsp_ctx_create(0, C.byref(h)) == L.NLSP_E_CUDA
    from paper_2601_20174_b200 import nlsp
    with pytest.raises(nlsp.CudaError):
        nlsp.Context(0)


def test_version_string():
    assert b"sm_100a" in L.gpu_lib().nlsp_version()


def test_product_does_not_link_the_oracle():
    for so in HEADERS.values():
        out = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
        assert "oracle" not in out and "nlsp_ref" not in out
        syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
        assert "orc_" not in syms and "ref_pcg" not in syms


def test_null_handle_queries_are_safe():
    """Handle queries need no device: a null operator has no schedule (-1) and
    zero dimensions."""
    lib = L.gpu_lib()
    assert lib.nlsp_twolevel_cycle(None) == -1
    n, k = C.c_uint64(7), C.c_uint64(7)
    lib.nlsp_twolevel_dims(None, C.byref(n), C.byref(k))
    assert n.value == 0 and k.value == 0
