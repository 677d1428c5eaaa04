"""Per-layer B200 profiler that feeds measured inputs back into the plan search.

The reference takes layer times as inputs ("no automatic profiling (times are inputs)",
SPEC.md:76; LayerSpec.fwd_time_per_sample_ms, model_ir.h:34; CostProfile.backward_multiplier,
cost_model.h:46).  This module measures them on the device with the executor itself:

  * fwd_time_per_sample_ms  — forward of one layer of each distinct shape, serial strategy,
                              `batch` samples, CUDA-graph replay timed with CUDA events;
  * backward_multiplier     — (fwd+bwd) / fwd of the same layer (optimizer excluded);

and returns a model JSON / profile JSON in the reference's schemas, so `Optimize` (this
repo's or the reference's) runs on B200-measured inputs.  Bandwidths (ClusterSpec) are
measured by `bus_bandwidth_gbps` when a multi-GPU NCCL world is available; on one GPU the
given cluster values are kept.

    python -m paper_2211_13878_b200.profiler --model bert-huge-32 --batch 4 --out prof.json
"""
from __future__ import annotations

import argparse
import copy
import json
from typing import Optional

from . import executor as gxe
from . import models


def _time_layers(shapes: list, batch: int, forward_only: bool, steps: int = 20,
                 warmup: int = 3) -> float:
    """ms per replay of these layers in sequence (serial plan) at `batch` samples."""
    import torch
    m = {"dtype_bytes": 4, "layers": [{"param_bytes": 1, "activation_bytes_per_sample": 1,
                                        "fwd_time_per_sample_ms": 1.0, "shape": dict(sh)}
                                       for sh in shapes]}
    plan = gxe.make_plan([""] * len(shapes), batch)
    ex = gxe.PlanExecutor(plan, m, 1, forward_only=forward_only, optimizer=False,
                          dropout_attn=0.1, dropout_hidden=0.1)
    ex.init_params(seed=1, std=0.02)
    first, last = shapes[0], shapes[-1]
    x = torch.randn(batch * first["seq"], first["hidden"], device="cuda").to(torch.bfloat16)
    y = torch.randn(batch * last["seq"], last["hidden"], device="cuda").to(torch.bfloat16)
    ex.load_batch_device(x, y)
    stream = torch.cuda.ExternalStream(ex.stream)
    for _ in range(warmup):
        ex.run(use_graph=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        ex.run(use_graph=True)
    b.record(stream)
    torch.cuda.synchronize()
    ex.close()
    return a.elapsed_time(b) / steps


def _time_layer(shape: dict, batch: int, forward_only: bool, prev: Optional[dict] = None) -> float:
    """ms of one layer.  A patch-merging layer cannot start a model (its input is the
    previous stage's grid), so it is timed behind its predecessor and the predecessor's own
    time is subtracted."""
    if not shape.get("merge"):
        return _time_layers([shape], batch, forward_only)
    assert prev is not None, "a merging layer needs its predecessor's shape"
    return (_time_layers([prev, shape], batch, forward_only)
            - _time_layers([prev], batch, forward_only))


def profile_model(model: dict, batch: int = 4) -> tuple[dict, dict, dict]:
    """Returns (model with measured fwd_time_per_sample_ms, profile json, raw measurements)."""
    out = copy.deepcopy(model)
    cache: dict = {}
    raw = []
    prev = None
    for layer in out["layers"]:
        key = json.dumps(layer["shape"], sort_keys=True)
        if key not in cache:
            fwd = _time_layer(layer["shape"], batch, True, prev)
            full = _time_layer(layer["shape"], batch, False, prev)
            cache[key] = (fwd, full)
            raw.append({"shape": layer["shape"], "batch": batch, "fwd_ms": fwd, "fwd_bwd_ms": full})
        fwd, full = cache[key]
        layer["fwd_time_per_sample_ms"] = round(fwd / batch, 6)
        prev = layer["shape"]
    ratios = [(full - fwd) / fwd for fwd, full in cache.values() if fwd > 0]
    profile = {"backward_multiplier": round(sum(ratios) / len(ratios), 4)}
    return out, profile, {"layers": raw}


def bus_bandwidth_gbps(group_size: int, nbytes: int = 1 << 28) -> Optional[float]:
    """NCCL all-reduce bus bandwidth (2(g-1)/g * bytes / time, the A6 volume convention of
    cost_model.cc:97-117) over the current torch.distributed world; None on one GPU."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() < 2:
        return None
    t = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        dist.all_reduce(t)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        dist.all_reduce(t)
    b.record()
    torch.cuda.synchronize()
    s = a.elapsed_time(b) / 10 / 1e3
    g = dist.get_world_size()
    return 2 * (g - 1) / g * nbytes / s / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert-huge-32")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    m, prof, raw = profile_model(models.model(args.model), args.batch)
    res = {"model": m, "profile": prof, "raw": raw}
    txt = json.dumps(res, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)
    print(json.dumps({"backward_multiplier": prof["backward_multiplier"],
                      "fwd_time_per_sample_ms": sorted({l["fwd_time_per_sample_ms"] for l in m["layers"]}),
                      "raw": raw["layers"]}))


if __name__ == "__main__":
    main()
