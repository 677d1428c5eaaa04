"""Debug: per-layer oracle errors of Swin window layers at real widths, feature by feature."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from tests.test_executor_gpu import _run_case, rel  # noqa: E402


def sw(h, grid, merge=False, shift=False, rel_pos=True):
    s = {"hidden": h, "heads": h // 32, "head_dim": 32, "seq": grid * grid, "ffn": 4 * h,
         "kind": "window", "window": 49, "rel_pos": rel_pos}
    if merge:
        s["merge"] = True
    if shift:
        s["shift"] = True
    return s


def model(shapes):
    return {"dtype_bytes": 4, "layers": [{"param_bytes": 1, "activation_bytes_per_sample": 1,
                                          "fwd_time_per_sample_ms": 1.0, "shape": s} for s in shapes]}


cases = [
    ("w320 g56 plain", [sw(320, 56, rel_pos=False)], [""]),
    ("w320 g56 rpb", [sw(320, 56)], [""]),
    ("w320 g56 shift", [sw(320, 56, shift=True, rel_pos=False)], [""]),
    ("w320 g56 shift+rpb", [sw(320, 56, shift=True)], [""]),
    ("w64 g14 shift+rpb", [sw(64, 14, shift=True)], [""]),
    ("w320 g56 -> merge 640 g28", [sw(320, 56), sw(640, 28, merge=True)], ["", ""]),
    ("full boundary serial", [sw(320, 56), sw(640, 28, merge=True), sw(640, 28, shift=True)], ["", "", ""]),
]
for name, shapes, strat in cases:
    plan = gxe.make_plan(strat, 1)
    out = _run_case(plan, model(shapes), 1, 0.1, seed=6)
    errs = {"y": rel(*out["y"]), "dx": rel(*out["dx"])}
    for l, (g, r) in enumerate(out["grads"]):
        for k in r:
            errs[f"L{l}.{k}"] = rel(g[k], r[k])
    out["ex"].close()
    print(json.dumps({"case": name, "errs": {k: round(v, 5) for k, v in errs.items()}}), flush=True)
