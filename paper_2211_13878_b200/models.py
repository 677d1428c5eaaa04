"""Model descriptions for the BASELINE configs: planner JSON + per-layer executor shapes.

The planner sees the reference's model schema (proj/src/model_ir.cc:69-95):
``{"dtype_bytes", "layers": [{param_bytes, activation_bytes_per_sample,
fwd_time_per_sample_ms, name?}]}``.  Each layer additionally carries a ``"shape"`` object
(hidden, heads, head_dim, seq, ffn, kind) that the reference loader ignores (unknown keys
are skipped, model_ir.cc:78-87) and the executor uses to build the layer.

Planner numbers:
  * bert-huge-32 — the reference fixture values (configs/models/bert-huge-32.json:5-36):
    32 x {84,000,000 B, 103,199,211 B/sample, 1.5 ms}.
  * swin-like — the reference fixture (configs/models/swin-like-heterogeneous.json).
  * bert-base-2, vit-huge-32, t5-large-48 — no reference fixture exists; authored as in
    SURVEY.md Appendix B (UniformModel of the paper's Table 2 totals).
Executor shapes (not in the reference; chosen here): BERT-Huge h=1280 as 20 heads x 64,
s=512, ffn 5120; BERT-base h=768, 12 x 64, s=128, ffn 3072; ViT-Huge h=1280, 16 x 80,
s=257, ffn 5120; T5-Large h=1024, 16 x 64, s=512, ffn 4096, 24 encoder + 24 decoder layers
("kind": "decoder": causal self-attention + cross-attention).  Swin-like (Swin-H at
224 px, the fixture's 2/2/26/2 stages): hidden 320/640/1280/2560 as heads x 32, token grids
56/28/14/7 stored window-major with 7x7 windows ("kind": "window", W-MSA; odd blocks
"shift": true, SW-MSA), ffn 4h; the first layer of stages 2-4 starts with patch merging
("merge": true).
"""
from __future__ import annotations

import copy
import json
from typing import Optional

MiB = 1 << 20
GiB = 1 << 30


def _shape(hidden, heads, seq, ffn, kind="encoder"):
    return {"hidden": hidden, "heads": heads, "head_dim": hidden // heads, "seq": seq,
            "ffn": ffn, "kind": kind}


def _uniform(n, param_bytes, act_bytes, fwd_ms, shape, names=None):
    layers = []
    for i in range(n):
        d = {"param_bytes": int(param_bytes), "activation_bytes_per_sample": int(act_bytes),
             "fwd_time_per_sample_ms": float(fwd_ms), "shape": dict(shape)}
        if names:
            d["name"] = names[i]
        layers.append(d)
    return {"dtype_bytes": 4, "layers": layers}


def layer_param_count(shape) -> int:
    """Parameters of one pre-LN encoder layer: QKV, out-proj, MLP (+biases), 2 LayerNorms."""
    h, f = shape["hidden"], shape["ffn"]
    return 3 * h * h + 3 * h + h * h + h + h * f + f + f * h + h + 4 * h


def _t5(n, param_bytes, act_bytes, fwd_ms, shape):
    """T5 flattened into one layer list: n/2 encoder layers, then n/2 decoder
    layers (causal self-attention + cross-attention over the encoder output + MLP), with T5's
    RMSNorm and the bucketed relative attention bias in every self-attention (bidirectional in
    the encoder, causal in the decoder; each layer owns its table).  The planner numbers stay
    uniform, as in the paper's Table 2 totals."""
    m = _uniform(n, param_bytes, act_bytes, fwd_ms, shape)
    for layer in m["layers"]:
        layer["shape"]["norm"] = "rms"      # T5LayerNorm (gain only)
        layer["shape"]["rel_bias"] = 32     # bucketed relative attention bias, max distance 128
    for layer in m["layers"][n // 2:]:
        layer["shape"]["kind"] = "decoder"
    return m


def _swin():
    spec = [  # (count, hidden, param_bytes, act_bytes, fwd_ms) per reference fixture stage
        (2, 320, 4915200, 78142034, 0.9),
        (2, 640, 19660800, 39071017, 0.95),
        (26, 1280, 78643200, 19535508, 1.0),
        (2, 2560, 314572800, 9767754, 1.1),
    ]
    layers = []
    for st, (n, h, p, a, t) in enumerate(spec):
        grid = 56 >> st
        for i in range(n):
            shape = _shape(h, h // 32, grid * grid, 4 * h, kind="window")
            shape["window"] = 49
            if st > 0 and i == 0:
                shape["merge"] = True
            if i % 2 == 1:
                shape["shift"] = True  # SW-MSA on odd blocks (the 7x7 last stage skips it)
            shape["rel_pos"] = True    # learned relative-position bias per head
            layers.append({"param_bytes": p, "activation_bytes_per_sample": a,
                           "fwd_time_per_sample_ms": t, "name": f"stage{st}.{i}",
                           "shape": shape})
    return {"dtype_bytes": 4, "layers": layers}


_CATALOG = {
    "bert-base-2": lambda: _uniform(2, 28351488, 4325376, 0.1, _shape(768, 12, 128, 3072)),
    "bert-huge-32": lambda: _uniform(32, 84000000, 103199211, 1.5, _shape(1280, 20, 512, 5120)),
    "vit-huge-32": lambda: _uniform(32, 632e6 * 4 / 32, 646.5 * MiB / 32, 1.5,
                                    _shape(1280, 16, 257, 5120)),
    "t5-large-48": lambda: _t5(48, 737e6 * 4 / 48, 6107.75 * MiB / 48, 1.5,
                               _shape(1024, 16, 512, 4096)),
    "swin-like": _swin,
}

MODELS = tuple(_CATALOG)


def model(name: str, num_layers: Optional[int] = None) -> dict:
    """Planner-schema model dict (with executor shapes); optionally truncated to N layers."""
    m = copy.deepcopy(_CATALOG[name]())
    if num_layers is not None:
        m["layers"] = m["layers"][:num_layers]
    return m


def cluster(num_devices: int, budget_gib: float, bw_gbps: float = 13.0,
            island_size: Optional[int] = None) -> dict:
    """Reference cluster schema (single-node-8gpu.json shape with N, E overridden)."""
    return {"num_devices": int(num_devices), "memory_budget_bytes": int(budget_gib * GiB),
            "island_size": int(island_size or num_devices), "intra_island_bw_gbps": float(bw_gbps),
            "inter_island_bw_gbps": float(bw_gbps)}


def planner_json(m: dict) -> str:
    return json.dumps(m)
