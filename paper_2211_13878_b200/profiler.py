"""Per-layer B200 profiler that feeds measured inputs back into the plan search.

The reference takes layer times as inputs ("no automatic profiling (times are inputs)",
SPEC.md:76; LayerSpec.fwd_time_per_sample_ms, model_ir.h:34; CostProfile.backward_multiplier,
cost_model.h:46).  This module measures them on the device with the executor itself:

  * fwd_time_per_sample_ms  — forward of one layer of each distinct shape, serial strategy,
                              `batch` samples, CUDA-graph replay timed with CUDA events;
  * backward_multiplier     — (fwd+bwd) / fwd of the same layer (optimizer excluded);
  * overlap_slowdown        — the cost model's k in max(bwd, comm) * k (cost_model.cc:200-206,
                              CostProfile.overlap_slowdown, cost_model.h:45-53; PAPER.md:327
                              measured 1.3): the layer's training step and a gradient
                              collective of comparable length launched together on two
                              streams, T_both / max(T_step, T_comm).  Under torchrun (N > 1)
                              the collective is an NCCL reduce-scatter of the layer's fp32
                              gradients over the world; on one GPU it is an SM-driven proxy
                              (an elementwise reduction kernel moving the same bytes through
                              HBM), reported as such;
  * intra_island_bw_gbps    — NCCL all-reduce bus GB/s over the world (ClusterSpec,
                              cluster.h:30-38), when N > 1;

and returns a model JSON / profile JSON (and a cluster JSON) in the reference's schemas, so
`Optimize` (this repo's or the reference's) runs on B200-measured inputs.

    python -m paper_2211_13878_b200.profiler --model bert-huge-32 --batch 4 --out prof.json
"""
from __future__ import annotations

import argparse
import copy
import json
import os
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


def profile_model(model: dict, batch: int = 4, overlap: bool = True) -> tuple[dict, dict, dict]:
    """Returns (model with measured fwd_time_per_sample_ms, profile json, raw measurements).
    With `overlap`, the profile also carries the measured overlap_slowdown (of the model's
    most frequent layer shape)."""
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
    res = {"layers": raw}
    if overlap:
        shapes = [json.dumps(l["shape"], sort_keys=True) for l in out["layers"]]
        common = json.loads(max(set(shapes), key=shapes.count))
        if not common.get("merge"):
            ov = overlap_slowdown(common, batch)
            profile["overlap_slowdown"] = ov["overlap_slowdown"]
            res["overlap"] = ov
    return out, profile, res


def _layer_grad_bytes(shape: dict) -> int:
    """fp32 bytes of one layer's gradients (the collective the overlap rule covers)."""
    h, f = shape["hidden"], shape["ffn"]
    return 4 * (4 * h * h + 2 * h * f + 9 * h + f)


def overlap_slowdown(shape: dict, batch: int, reps: int = 10, warmup: int = 3) -> dict:
    """k of EstimateLayerCost's overlapped schedule for one layer shape (see module doc)."""
    import torch
    import torch.distributed as dist
    m = {"dtype_bytes": 4, "layers": [{"param_bytes": 1, "activation_bytes_per_sample": 1,
                                        "fwd_time_per_sample_ms": 1.0, "shape": dict(shape)}]}
    ex = gxe.PlanExecutor(gxe.make_plan([""], batch), m, 1, forward_only=False, optimizer=False,
                          dropout_attn=0.1, dropout_hidden=0.1)
    ex.init_params(seed=1, std=0.02)
    x = torch.randn(batch * shape["seq"], shape["hidden"], device="cuda").to(torch.bfloat16)
    ex.load_batch_device(x, x)
    ex_stream = torch.cuda.ExternalStream(ex.stream)
    comm_stream = torch.cuda.Stream()
    nbytes = _layer_grad_bytes(shape)
    nccl = dist.is_initialized() and dist.get_world_size() > 1
    if nccl:
        world = dist.get_world_size()
        n = (nbytes // 4 + world - 1) // world * world
        src = torch.randn(n, device="cuda")
        dst = torch.empty(n // world, device="cuda")

        def comm():
            dist.reduce_scatter_tensor(dst, src)
        kind = f"nccl reduce_scatter_tensor fp32 over {world} ranks"
    else:
        a = torch.randn(nbytes // 4, device="cuda")
        b = torch.randn_like(a)
        c = torch.empty_like(a)

        def comm():
            torch.add(a, b, out=c)
        kind = "proxy (1 GPU): elementwise fp32 reduction kernel over the same bytes"

    def timed(run_step, run_comm, n_comm):
        start = torch.cuda.Event(enable_timing=True)
        ends = []
        torch.cuda.synchronize()
        start.record(torch.cuda.current_stream())
        if run_comm:
            comm_stream.wait_event(start)
            with torch.cuda.stream(comm_stream):
                for _ in range(n_comm):
                    comm()
            e = torch.cuda.Event(enable_timing=True)
            e.record(comm_stream)
            ends.append(e)
        if run_step:
            ex_stream.wait_event(start)
            for _ in range(reps):
                ex.run(use_graph=True)
            e = torch.cuda.Event(enable_timing=True)
            e.record(ex_stream)
            ends.append(e)
        torch.cuda.synchronize()
        return max(start.elapsed_time(e) for e in ends)

    for _ in range(warmup):
        ex.run(use_graph=True)
        comm()
    t_step = timed(True, False, 0)
    t_one = timed(False, True, 1)
    n_comm = max(1, round(t_step / max(t_one, 1e-6)))  # a collective as long as the steps
    t_comm = timed(False, True, n_comm)
    t_both = timed(True, True, n_comm)
    ex.close()
    k = t_both / max(t_step, t_comm)
    return {"overlap_slowdown": round(max(k, 1.0), 4), "raw_ratio": round(k, 4),
            "t_step_ms": round(t_step / reps, 4), "t_comm_ms": round(t_comm / reps, 4),
            "t_both_ms": round(t_both / reps, 4), "comm_bytes": nbytes * n_comm // reps,
            "comm": kind, "batch": batch, "shape": shape}


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
    ap.add_argument("--budget-gib", type=float, default=16.0)
    args = ap.parse_args()
    import torch.distributed as dist
    if os.environ.get("WORLD_SIZE", "1") != "1" and not dist.is_initialized():
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    m, prof, raw = profile_model(models.model(args.model), args.batch)
    world = dist.get_world_size() if dist.is_initialized() else 1
    bw = bus_bandwidth_gbps(world)
    cluster = models.cluster(world, args.budget_gib, bw if bw is not None else 13.0)
    res = {"model": m, "profile": prof, "cluster": cluster, "raw": raw,
           "bus_gbps": bw, "bus_gbps_note": None if bw is not None else
           "one GPU: no NCCL peers; the reference cluster's 13 GB/s is kept"}
    if dist.is_initialized() and dist.get_rank() != 0:
        return
    txt = json.dumps(res, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)
    print(json.dumps({"backward_multiplier": prof["backward_multiplier"],
                      "overlap_slowdown": prof.get("overlap_slowdown"), "bus_gbps": bw,
                      "fwd_time_per_sample_ms": sorted({l["fwd_time_per_sample_ms"] for l in m["layers"]}),
                      "raw": raw["layers"]}))


if __name__ == "__main__":
    main()
