"""Debug: per-tensor oracle errors of T5-style (encoder + decoder) stacks at several shapes,
to localise a shape-dependent executor error (std 0.02 weights, dropout 0.1)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from tests.test_executor_gpu import _run_case, rel  # noqa: E402


def model(kinds, h, heads, s, f):
    return {"dtype_bytes": 4, "layers": [
        {"param_bytes": 1, "activation_bytes_per_sample": 1, "fwd_time_per_sample_ms": 1.0,
         "shape": {"hidden": h, "heads": heads, "head_dim": h // heads, "seq": s, "ffn": f,
                   "kind": k}} for k in kinds]}


cases = [
    ("enc+dec h1024 s512 f4096", ["encoder", "decoder"], 1024, 16, 512, 4096),
    ("enc+dec h1024 s128 f4096", ["encoder", "decoder"], 1024, 16, 128, 4096),
    ("enc+dec h256 s512 f1024", ["encoder", "decoder"], 256, 4, 512, 1024),
    ("enc+dec h256 s128 f4096", ["encoder", "decoder"], 256, 4, 128, 4096),
    ("enc+dec h256 s256 f1024", ["encoder", "decoder"], 256, 4, 256, 1024),
    ("causal h256 s512 f1024", ["causal", "causal"], 256, 4, 512, 1024),
    ("enc h256 s512 f1024", ["encoder", "encoder"], 256, 4, 512, 1024),
]
for name, kinds, h, H, s, f in cases:
    plan = gxe.make_plan([""] * len(kinds), 1)
    out = _run_case(plan, model(kinds, h, H, s, f), 1, 0.1, seed=5, std=0.02)
    errs = {"y": rel(*out["y"]), "dx": rel(*out["dx"])}
    for l, (g, r) in enumerate(out["grads"]):
        for k in r:
            errs[f"L{l}.{k}"] = rel(g[k], r[k])
    out["ex"].close()
    print(json.dumps({"case": name, "errs": {k: round(v, 5) for k, v in errs.items()}}), flush=True)
