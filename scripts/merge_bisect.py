"""Debug: activation-level oracle errors of a Swin stage boundary (window layer -> merging
layer) at real widths, to localise the merging layer's forward error."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import layer_oracle as lo  # noqa: E402
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from tests.test_executor_gpu import _oshape, rel  # noqa: E402
from scripts.swin_bisect import sw, model  # noqa: E402


def export(ex, buf, code):
    import ctypes
    from paper_2211_13878_b200 import _lib
    _lib.check(_lib.lib().gx_exec_export_output(ex._h, code, buf.ctypes.data_as(ctypes.c_void_p)))


def run(name, shapes, p_drop):
    m = model(shapes)
    osh = [_oshape(s) for s in shapes]
    rng = np.random.default_rng(6)
    params = [{k: v.astype(np.float32).astype(np.float64)
               for k, v in lo.init_layer_params(o, rng, 0.02).items()} for o in osh]
    B = 1
    x32 = rng.standard_normal((B * osh[0].seq, osh[0].hidden)).astype(np.float32)
    xb = gxe.f32_to_bf16_bits(x32)
    x = gxe.bf16_bits_to_f32(xb).astype(np.float64)
    ex = gxe.PlanExecutor(gxe.make_plan([""] * len(shapes), B), m, 1, dropout_attn=p_drop,
                          dropout_hidden=p_drop, seed=77, optimizer=False, forward_only=True)
    for l in range(len(shapes)):
        ex.set_layer_params(l, params[l])
    tb = np.zeros(B * osh[-1].seq * osh[-1].hidden, dtype=np.uint16)
    ex.load_batch(xb, tb)
    ex.run(False)
    drop = lo.Dropout(p_drop, p_drop, 77)
    h = x
    out = {}
    for l, o in enumerate(osh):
        y, c = lo.layer_forward(params[l], h, o, l, drop)
        for k, nm, width in ((0, "x", o.hidden), (1, "ln1", o.hidden), (2, "x1", o.hidden),
                             (3, "ln2", o.hidden), (4, "gel", o.ffn), (5, "y", o.hidden)):
            buf = np.empty(B * o.seq * width, dtype=np.uint16)
            export(ex, buf, 1000 + 16 * l + k)
            got = gxe.bf16_bits_to_f32(buf).reshape(B * o.seq, width)
            ref = {"x": c["x"], "ln1": c["a"] if c["perm"] is None else None, "x1": c["x1"],
                   "ln2": c["c"], "gel": c["g"], "y": y}[nm]
            if ref is not None:
                out[f"L{l}.{nm}"] = round(rel(got, ref), 5)
        # feed the next layer the GPU's own output, so each layer is judged on its own
        buf = np.empty(B * o.seq * o.hidden, dtype=np.uint16)
        export(ex, buf, 1000 + 16 * l + 5)
        h = gxe.bf16_bits_to_f32(buf).reshape(B * o.seq, o.hidden).astype(np.float64)
    ex.close()
    print(json.dumps({"case": name, "p": p_drop, "errs": out}), flush=True)


for p in (0.0, 0.1):
    run("w320 g56 -> merge 640 g28", [sw(320, 56), sw(640, 28, merge=True)], p)
    run("w320 g56 -> merge 640 g28 no-rpb", [sw(320, 56, rel_pos=False), sw(640, 28, merge=True, rel_pos=False)], p)
    run("w64 g28 -> merge 128 g14", [sw(64, 28), sw(128, 14, merge=True)], p)
