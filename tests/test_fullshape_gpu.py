"""Executor parity at the BASELINE configs' real layer shapes (VERDICT r1 "next" item 1):
the layers the bench times (BERT-Huge: h 1280, 20 x 64, s 512, ffn 5120), ViT-Huge (16 x 80,
s 257: tail masking), T5-Large encoder + decoder layers across a pipeline split, and a Swin
stage boundary at real widths (320 -> 640: patch merging, SW-MSA, relative-position bias,
grid 56 -> 28).  Each runs in the simulated world on one B200 against the float64 oracle
(oracle/layer_oracle.py) with dropout 0.1, and the errors are printed.

Tolerance: ||got - ref||_2 / ||ref||_2 <= 1e-2 for the output, the input
gradient and every parameter gradient; loss within 1e-2 relative.
"""
import numpy as np
import pytest

from paper_2211_13878_b200 import executor as gxe

from .test_executor_gpu import TOL, _run_case, rel

pytestmark = pytest.mark.gpu


def _model(shapes):
    return {"dtype_bytes": 4, "layers": [
        {"param_bytes": 1, "activation_bytes_per_sample": 1, "fwd_time_per_sample_ms": 1.0,
         "shape": dict(s)} for s in shapes]}


def _enc(h, heads, seq, ffn, kind="encoder"):
    return {"hidden": h, "heads": heads, "head_dim": h // heads, "seq": seq, "ffn": ffn,
            "kind": kind}


def _swin(h, grid, merge=False, shift=False):
    s = _enc(h, h // 32, grid * grid, 4 * h, "window")
    s.update(window=49, rel_pos=True)
    if merge:
        s["merge"] = True
    if shift:
        s["shift"] = True
    return s


def _check_print(name, out):
    got, ref = out["loss"]
    errs = {"loss": abs(got - ref) / abs(ref), "y": rel(*out["y"]), "dx": rel(*out["dx"])}
    worst = ("", 0.0)
    for l, (g, r) in enumerate(out["grads"]):
        for k in r:
            assert not np.isnan(g[k]).any(), (l, k)
            e = rel(g[k], r[k])
            if e > worst[1]:
                worst = (f"L{l}.{k}", e)
    errs["worst_grad"] = worst
    print(f"\n{name}: {errs}")
    assert errs["loss"] <= 1e-2 and errs["y"] <= TOL and errs["dx"] <= TOL, errs
    assert worst[1] <= TOL, errs
    out["ex"].close()


BERT = _enc(1280, 20, 512, 5120)


@pytest.mark.parametrize("world,strategy,B", [(1, "", 1), (2, "sdp:2", 2), (2, "tp:2", 2)],
                         ids=["serial-B1", "sdp2-B2", "tp2-B2"])
def test_bert_huge_layers(cuda, world, strategy, B):
    plan = gxe.make_plan([strategy] * 2, B)
    _check_print(f"bert-huge x2 [{strategy or 'serial'}] B={B}",
                 _run_case(plan, _model([BERT, BERT]), world, 0.1, seed=3))


def test_vit_huge_layers_tp2_sdp4(cuda):
    vit = _enc(1280, 16, 257, 5120)
    plan = gxe.make_plan(["tp:2,sdp:4"] * 2, 4)
    _check_print("vit-huge x2 [tp:2,sdp:4] B=4 (8 sim ranks)",
                 _run_case(plan, _model([vit, vit]), 8, 0.1, seed=4))


def test_t5_large_encoder_decoder_pipeline(cuda):
    """T5-Large layers proper (RMSNorm, 32-bucket relative attention bias) across P = 2."""
    enc, dec = _enc(1024, 16, 512, 4096), _enc(1024, 16, 512, 4096, "decoder")
    for sh in (enc, dec):
        sh.update(norm="rms", rel_bias=32)
    plan = gxe.make_plan(["", "", "", ""], 2, pp_degree=2, micro_batches=2)
    _check_print("t5-large (rms, rel-bias) 2 enc + 2 dec, P=2 m=2 B=2",
                 _run_case(plan, _model([enc, enc, dec, dec]), 2, 0.1, seed=5))


def test_swin_stage_boundary_real_widths(cuda):
    shapes = [_swin(320, 56), _swin(640, 28, merge=True), _swin(640, 28, shift=True)]
    plan = gxe.make_plan(["dp:2", "sdp:2", "tp:2"], 2)
    _check_print("swin 320->640 (merge, SW-MSA, rel-pos) [dp:2|sdp:2|tp:2] B=2",
                 _run_case(plan, _model(shapes), 2, 0.1, seed=6))
