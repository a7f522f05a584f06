"""NLSS basis through MLP inference, mirroring the reference's
names: MlpModel (mlp.hpp:47-320; checkpoints and seeded initialisation through
libnlsp_io.so, host) and infer_basis (train.hpp:52-62; the forward pass and the
orthonormalisation on the device, libnlsp_gpu.so)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .instance_io import IoError
from .nlsp import DeviceDense, ValidationError, _check, default_context


def default_hidden_widths(n: int):
    """train.hpp:28-32: four hidden layers for large grids, one otherwise."""
    return [128, 256, 256, 128] if n >= 33 * 33 else [128]


def _raise_io(st):
    msg = L.io_lib().nlsp_io_last_error().decode(errors="replace")
    raise (IoError if st == L.NLSP_E_IO else ValidationError)(msg)


class MlpModel:
    """Widths + the flat parameter buffer in the reference's layout."""

    def __init__(self, widths, params, manifest: str = ""):
        self.widths = [int(w) for w in widths]
        self.params = np.ascontiguousarray(params, np.float64)
        self.manifest = manifest
        self._dev = {}

    @staticmethod
    def _from_c(h):
        w = np.ctypeslib.as_array(h.widths, shape=(h.nwidths,)).copy()
        p = np.ctypeslib.as_array(h.params, shape=(h.nparams,)).copy()
        return MlpModel(w, p, (h.manifest or b"").decode(errors="replace"))

    @staticmethod
    def init(widths, seed: int) -> "MlpModel":
        """MlpModel(widths, seed) (mlp.hpp:57-88), bit-identical He initialisation."""
        lib = L.io_lib()
        w = np.ascontiguousarray(widths, np.uint64)
        h = L.HostMlpC()
        st = lib.nlsp_io_mlp_init(L.u64ptr(w), w.size, seed, C.byref(h))
        if st:
            _raise_io(st)
        try:
            return MlpModel._from_c(h)
        finally:
            lib.nlsp_io_mlp_free(C.byref(h))

    @staticmethod
    def load(path: str) -> "MlpModel":
        """MlpModel::load (mlp.hpp:276-303)."""
        lib = L.io_lib()
        h = L.HostMlpC()
        st = lib.nlsp_io_mlp_load(str(path).encode(), C.byref(h))
        if st:
            _raise_io(st)
        try:
            return MlpModel._from_c(h)
        finally:
            lib.nlsp_io_mlp_free(C.byref(h))

    def save(self, path: str, manifest: str = "") -> None:
        """MlpModel::save (mlp.hpp:255-274), zero Adam state."""
        w = np.ascontiguousarray(self.widths, np.uint64)
        h = L.HostMlpC(w.size, L.u64ptr(w), self.params.size, L.dptr(self.params), manifest.encode())
        st = L.io_lib().nlsp_io_mlp_save(C.byref(h), str(path).encode())
        if st:
            _raise_io(st)

    def input_width(self) -> int:
        return self.widths[0]

    def output_width(self) -> int:
        return self.widths[-1]

    def device(self, ctx=None):
        ctx = ctx or default_context()
        h = self._dev.get(id(ctx))
        if h is None:
            w = np.ascontiguousarray(self.widths, np.uint64)
            hh = C.c_void_p()
            _check(ctx, L.gpu_lib().nlsp_mlp_upload(ctx.handle, L.u64ptr(w), w.size, L.dptr(self.params),
                                                    self.params.size, C.byref(hh)))
            h = _DevMlp(ctx, hh)
            self._dev[id(ctx)] = h
        return h

    def forward(self, x, ctx=None) -> np.ndarray:
        """MlpModel::forward (mlp.hpp:113-161) on the device."""
        d = self.device(ctx)
        x = np.ascontiguousarray(x, np.float64)
        if x.shape != (self.input_width(),):
            raise ValidationError("mlp forward: width mismatch")
        y = np.empty(self.output_width())
        _check(d.ctx, L.gpu_lib().nlsp_mlp_forward(d.ctx.handle, d.handle, L.dptr(x), L.dptr(y)))
        return y


class _DevMlp:
    def __init__(self, ctx, handle):
        self.ctx, self.handle = ctx, handle

    def __del__(self):
        try:
            if self.handle:
                L.gpu_lib().nlsp_mlp_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def infer_basis(model: MlpModel, s, ctx=None) -> DeviceDense:
    """infer_basis (train.hpp:52-62): Q (n x r) on the device."""
    ctx = ctx or (s.ctx if isinstance(s, DeviceDense) else default_context())
    sd = s if isinstance(s, DeviceDense) else DeviceDense.upload(np.ascontiguousarray(s, np.float64), ctx)
    d = model.device(ctx)
    h = C.c_void_p()
    _check(ctx, L.gpu_lib().nlsp_mlp_infer_basis(ctx.handle, d.handle, sd.handle, C.byref(h)))
    return DeviceDense(ctx, h)
