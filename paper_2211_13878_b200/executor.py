"""Python handle over the C++ plan executor (gx_exec_* in include/gx.h).

The executor is C++/CUDA; this module only marshals JSON configs and host arrays across
the C ABI (plans in the reference's PlanToJson schema, proj/src/planner.cc:483-521).
"""
from __future__ import annotations

import ctypes
import json
from typing import Optional, Sequence

import numpy as np

from . import _lib

CANONICAL_ORDER = ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_qkv", "b_o", "b_1", "b_2",
                   "w_qkv", "w_o", "w_1", "w_2")
MERGE_ORDER = ("mln_g", "mln_b", "w_m")  # patch-merging layers only, after w_2
CROSS_ORDER = ("ln3_g", "ln3_b", "b_q2", "b_kv2", "b_o2", "w_q2", "w_kv2", "w_o2")  # decoders


def pack_canonical(P: dict) -> np.ndarray:
    """Layer parameter dict (oracle naming) -> canonical flat fp32 vector."""
    keys = CANONICAL_ORDER + (MERGE_ORDER if "w_m" in P else ()) + \
        (CROSS_ORDER if "w_q2" in P else ()) + (("rpb",) if "rpb" in P else ()) + \
        (("relb",) if "relb" in P else ())
    return np.concatenate([np.asarray(P[k], dtype=np.float32).ravel() for k in keys])


def unpack_canonical(flat: np.ndarray, hidden: int, ffn: int, merge: bool = False,
                     cross: bool = False, rpb=None, relb=None) -> dict:
    """rpb: (heads, entries per head) of a Swin relative-position-bias table, or None;
    relb: (heads, buckets) of a T5 relative attention bias table, or None."""
    h, f = hidden, ffn
    shapes = {"ln1_g": (h,), "ln1_b": (h,), "ln2_g": (h,), "ln2_b": (h,), "b_qkv": (3 * h,),
              "b_o": (h,), "b_1": (f,), "b_2": (h,), "w_qkv": (3 * h, h), "w_o": (h, h),
              "w_1": (f, h), "w_2": (h, f),
              "mln_g": (2 * h,), "mln_b": (2 * h,), "w_m": (h, 2 * h),
              "ln3_g": (h,), "ln3_b": (h,), "b_q2": (h,), "b_kv2": (2 * h,), "b_o2": (h,),
              "w_q2": (h, h), "w_kv2": (2 * h, h), "w_o2": (h, h)}
    out, off = {}, 0
    if rpb is not None:
        shapes["rpb"] = tuple(rpb)
    if relb is not None:
        shapes["relb"] = tuple(relb)
    for k in CANONICAL_ORDER + (MERGE_ORDER if merge else ()) + (CROSS_ORDER if cross else ()) + \
            (("rpb",) if rpb is not None else ()) + (("relb",) if relb is not None else ()):
        n = int(np.prod(shapes[k]))
        out[k] = flat[off:off + n].reshape(shapes[k])
        off += n
    return out


def make_plan(strategies: Sequence[str], batch_size: int, pp_degree: int = 1,
              micro_batches: int = 1, stage_bounds: Optional[Sequence[int]] = None) -> dict:
    """Hand-authored plan in the PlanToJson schema (fields the executor reads)."""
    L = len(strategies)
    if stage_bounds is None:
        per = L // pp_degree
        stage_bounds = [i * per for i in range(pp_degree)] + [L]
    stages = []
    for s in range(pp_degree):
        b, e = stage_bounds[s], stage_bounds[s + 1]
        stages.append({"layer_range": [b, e],
                       "layers": [{"id": i, "strategy": strategies[i]} for i in range(b, e)]})
    return {"pp_degree": pp_degree, "micro_batches": micro_batches, "batch_size": batch_size,
            "stages": stages}


def topology(plan: dict, model: dict, world_size: int, local_ranks) -> dict:
    """Device-free view of what each local rank will do (groups, chunks, PP transfers)."""
    cfg = {"plan": plan, "model": model, "world_size": world_size,
           "local_ranks": list(local_ranks), "comm": "dryrun"}
    need = ctypes.c_size_t()
    txt = json.dumps(cfg).encode()
    _lib.check(_lib.lib().gx_exec_topology(txt, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _lib.check(_lib.lib().gx_exec_topology(txt, buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def nccl_unique_id() -> str:
    buf = ctypes.create_string_buffer(257)
    _lib.check(_lib.lib().gx_nccl_unique_id(buf, 257))
    return buf.value.decode()


class PlanExecutor:
    def __init__(self, plan: dict, model: dict, world_size: int, local_ranks=None,
                 comm: str = "sim", nccl_id_hex: str = "", dropout_attn=0.0, dropout_hidden=0.0,
                 seed=1234, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                 optimizer=True, forward_only=False, splitk=True, **options):
        cfg = {"plan": plan, "model": model, "world_size": world_size, "comm": comm,
               "dropout_attn": dropout_attn, "dropout_hidden": dropout_hidden, "seed": seed,
               "lr": lr, "beta1": beta1, "beta2": beta2, "eps": eps,
               "weight_decay": weight_decay, "optimizer": optimizer,
               "forward_only": forward_only, "splitk": splitk}
        cfg.update(options)  # executor knobs, e.g. wgrad_stream=False
        if local_ranks is not None:
            cfg["local_ranks"] = list(local_ranks)
        if comm == "nccl":
            cfg["nccl_id_hex"] = nccl_id_hex
        self.plan, self.model = plan, model
        self.shapes = [l["shape"] for l in model["layers"]]
        self._h = ctypes.c_void_p()
        _lib.check(_lib.lib().gx_exec_create(json.dumps(cfg).encode(), ctypes.byref(self._h)))

    def close(self):
        if self._h:
            _lib.lib().gx_exec_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _canon_n(self, layer):
        s = self.shapes[layer]
        n = ctypes.c_int64()
        _lib.lib().gx_exec_canonical_size(s["hidden"], s["ffn"], ctypes.byref(n))
        h = s["hidden"]
        rp = self._rpb_shape(s)
        rb = self._relb_shape(s)
        return n.value + (4 * h + 2 * h * h if s.get("merge") else 0) + \
            (6 * h + 4 * h * h if s.get("kind") == "decoder" else 0) + \
            (rp[0] * rp[1] if rp else 0) + (rb[0] * rb[1] if rb else 0)

    @staticmethod
    def _relb_shape(s):
        b = int(s.get("rel_bias", 0) or 0)
        return (s["heads"], b) if b > 0 and s.get("kind") != "window" else None

    @staticmethod
    def _rpb_shape(s):
        if s.get("kind") != "window" or not s.get("rel_pos"):
            return None
        side = int(round(s.get("window", 49) ** 0.5))
        return (s["heads"], (2 * side - 1) ** 2)

    def set_layer_params(self, layer: int, P: dict):
        flat = np.ascontiguousarray(pack_canonical(P))
        _lib.check(_lib.lib().gx_exec_set_layer_params(
            self._h, layer, flat.ctypes.data_as(ctypes.c_void_p), flat.size))

    def export_layer(self, layer: int, what: str = "params") -> dict:
        n = self._canon_n(layer)
        out = np.empty(n, dtype=np.float32)
        _lib.check(_lib.lib().gx_exec_export_layer(
            self._h, layer, {"params": 0, "grads": 1, "bf16": 2}[what],
            out.ctypes.data_as(ctypes.c_void_p), n))
        s = self.shapes[layer]
        return unpack_canonical(out, s["hidden"], s["ffn"], bool(s.get("merge")),
                                s.get("kind") == "decoder", self._rpb_shape(s),
                                self._relb_shape(s))

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        _lib.check(_lib.lib().gx_exec_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def load_batch(self, x_host, target_host):
        """x / target: host arrays of bf16 bit patterns (uint16/int16) or torch CPU tensors."""
        _lib.check(_lib.lib().gx_exec_load_batch(self._h, _host_ptr(x_host), _host_ptr(target_host)))

    def load_batch_device(self, x_dev, target_dev):
        import torch
        for t in (x_dev, target_dev):  # produced on torch's stream; the executor's is separate
            if t is not None:
                torch.cuda.current_stream(t.device).synchronize()
        _lib.check(_lib.lib().gx_exec_load_batch_device(
            self._h, x_dev.data_ptr() if x_dev is not None else None,
            target_dev.data_ptr() if target_dev is not None else None))

    def run(self, use_graph=False, profile=False):
        _lib.check(_lib.lib().gx_exec_run(self._h, int(use_graph) | (2 if profile else 0)))

    def profile_report(self) -> dict:
        need = ctypes.c_size_t()
        _lib.check(_lib.lib().gx_exec_profile_report(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _lib.check(_lib.lib().gx_exec_profile_report(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def init_params(self, seed=1, std=0.02):
        _lib.check(_lib.lib().gx_exec_init_params(self._h, seed, std))

    def sync(self, timeout_ms: int = 600000):
        """Wait for the executor's stream; a communicator failure or hang raises GxError."""
        _lib.check(_lib.lib().gx_exec_sync(self._h, int(timeout_ms)))

    def loss(self) -> float:
        v = ctypes.c_float()
        _lib.check(_lib.lib().gx_exec_loss(self._h, ctypes.byref(v)))
        return v.value

    def step(self, x_host, target_host, use_graph=False) -> float:
        v = ctypes.c_float()
        _lib.check(_lib.lib().gx_exec_step(self._h, _host_ptr(x_host), _host_ptr(target_host),
                                           int(use_graph), ctypes.byref(v)))
        return v.value

    def export_output(self, what="y") -> np.ndarray:
        """"y" = model output, "dx" = input gradient, int l = output of layer l."""
        s = self.shapes[-1] if what == "y" else (self.shapes[0] if what == "dx" else self.shapes[what])
        code = 0 if what == "y" else (1 if what == "dx" else 2 + int(what))
        rows = self.plan["batch_size"] * s["seq"]
        out = np.zeros((rows, s["hidden"]), dtype=np.uint16)
        _lib.check(_lib.lib().gx_exec_export_output(self._h, code,
                                                    out.ctypes.data_as(ctypes.c_void_p)))
        return bf16_bits_to_f32(out)

    def info(self) -> dict:
        need = ctypes.c_size_t()
        _lib.check(_lib.lib().gx_exec_info(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _lib.check(_lib.lib().gx_exec_info(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())


def _host_ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if a.is_cuda:
            raise ValueError("load_batch takes host memory; use load_batch_device")
        return a.data_ptr()
    return np.ascontiguousarray(a).ctypes.data_as(ctypes.c_void_p)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)
