"""TEST / BASELINE INFRASTRUCTURE ONLY — ctypes wrapper of oracle/cpu_layer.c (fp32 C + OpenMP
restatement of the encoder-layer training step; see that file's header).  Used by
tests/test_cpu_layer.py (checked against layer_oracle.py) and by bench.py's CPU baseline and
`--impl reference` legs.  Never imported by the product package."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_cpu", "libcpu_layer.so")
_L = None

# canonical per-layer parameter order inside the flat block (cpu_layer.c carve())
ORDER = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1",
         "w_2", "b_2")


def lib():
    global _L
    if _L is None:
        if not os.path.exists(SO):
            subprocess.run(["make", "-s", "-C", HERE, "cpu"], check=True)
        L = ctypes.CDLL(SO)
        vp, f, i, u64 = ctypes.c_void_p, ctypes.c_float, ctypes.c_int, ctypes.c_uint64
        L.cpu_model_create.restype = vp
        L.cpu_model_create.argtypes = [i, i, i, i, i, i, f, f, u64]
        L.cpu_model_destroy.argtypes = [vp]
        L.cpu_model_params.restype = ctypes.POINTER(ctypes.c_float)
        L.cpu_model_params.argtypes = [vp, i]
        L.cpu_model_grads.restype = ctypes.POINTER(ctypes.c_float)
        L.cpu_model_grads.argtypes = [vp, i]
        L.cpu_model_step.restype = f
        L.cpu_model_step.argtypes = [vp, vp, vp, vp, vp, i, f, f, f, f, f]
        L.cpu_layer_param_count.restype = ctypes.c_int64
        L.cpu_layer_param_count.argtypes = [i, i]
        L.cpu_threads.restype = i
        _L = L
    return _L


def shapes(h, f):
    return {"ln1_g": (h,), "ln1_b": (h,), "w_qkv": (3 * h, h), "b_qkv": (3 * h,),
            "w_o": (h, h), "b_o": (h,), "ln2_g": (h,), "ln2_b": (h,), "w_1": (f, h),
            "b_1": (f,), "w_2": (h, f), "b_2": (h,)}


class CpuModel:
    """A stack of `layers` encoder layers (hidden h, heads, seq, ffn) for `samples` samples."""

    def __init__(self, layers, samples, seq, hidden, heads, ffn, p_attn=0.0, p_hidden=0.0,
                 seed=1234):
        self.L, self.n, self.s, self.h, self.f = layers, samples, seq, hidden, ffn
        self._m = lib().cpu_model_create(layers, samples, seq, hidden, heads, ffn, p_attn,
                                         p_hidden, seed)
        self.np = lib().cpu_layer_param_count(hidden, ffn)

    def close(self):
        if self._m:
            lib().cpu_model_destroy(self._m)
            self._m = None

    def __del__(self):
        self.close()

    def _view(self, ptr):
        return np.ctypeslib.as_array(ptr, shape=(self.np,))

    def set_layer(self, layer, P: dict):
        flat = self._view(lib().cpu_model_params(self._m, layer))
        off = 0
        for k, shp in shapes(self.h, self.f).items():
            n = int(np.prod(shp))
            flat[off:off + n] = np.asarray(P[k], np.float32).ravel()
            off += n

    def _unflat(self, flat):
        out, off = {}, 0
        for k, shp in shapes(self.h, self.f).items():
            n = int(np.prod(shp))
            out[k] = flat[off:off + n].reshape(shp).copy()
            off += n
        return out

    def layer_params(self, layer):
        return self._unflat(self._view(lib().cpu_model_params(self._m, layer)))

    def layer_grads(self, layer):
        return self._unflat(self._view(lib().cpu_model_grads(self._m, layer)))

    def step(self, x, target, optimizer=True, lr=1e-4, b1=0.9, b2=0.999, eps=1e-8, wd=0.0,
             want=False):
        x = np.ascontiguousarray(x, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        y = np.empty_like(x) if want else None
        dx = np.empty_like(x) if want else None
        loss = lib().cpu_model_step(self._m, x.ctypes.data, t.ctypes.data,
                                    y.ctypes.data if want else None,
                                    dx.ctypes.data if want else None, int(optimizer), lr, b1,
                                    b2, eps, wd)
        return (loss, y, dx) if want else loss


def threads() -> int:
    return lib().cpu_threads()
