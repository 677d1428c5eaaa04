"""Execute the BASELINE configs' plans end to end on one GPU (all ranks simulated).

  config 3  ViT-Huge-32 (s 257, 16 x 80 heads): hand plan [tp:2,sdp:4] x32
  config 4  T5-Large-48 (24 encoder + 24 decoder layers, flattened per SPEC.md:67): the
            searched 8-GPU / 8 GiB plan (P=2, m=8, decoder = stage 1) and hand P=4 / P=8 splits
            (the memory travels with the activations across the decoder's stage boundaries)
  config 5  Swin fixture: the searched [dp:8] x6 | [sdp:8] x24 | [tp:2,sdp:4] x2 (B=64)

Every rank of the world runs in this process on cuda:0 (comm "sim"), so ms/step is the sum
over ranks -- a functional check of the plan's kernels, relayouts and PP schedule at full
model size, not cluster throughput.  One JSON line per run.

    python scripts/config_runs.py [--steps 2] [--only vit,t5p2,...]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from paper_2211_13878_b200 import models, planner  # noqa: E402


def _runs():
    api = planner.api()
    t5 = models.model("t5-large-48")
    swin = models.model("swin-like")
    return {
        "vit": ("config 3: ViT-Huge-32", models.model("vit-huge-32"),
                gxe.make_plan(["tp:2,sdp:4"] * 32, 8), 8),
        "t5p2": ("config 4: T5-Large-48 searched (8 GPUs, 8 GiB)", t5,
                 api.optimize(t5, models.cluster(8, 8)).plan, 8),
        "t5p4": ("config 4: T5-Large-48 P=4", t5,
                 gxe.make_plan(["sdp:2"] * 48, 8, pp_degree=4, micro_batches=8), 8),
        "t5p8": ("config 4: T5-Large-48 P=8", t5,
                 gxe.make_plan([""] * 48, 8, pp_degree=8, micro_batches=8), 8),
        "swin": ("config 5: Swin fixture searched (8 GPUs, 8 GiB)", swin,
                 api.optimize(swin, models.cluster(8, 8)).plan, 8),
    }


def run_one(label, model, plan, world, steps):
    t0 = time.time()
    ex = gxe.PlanExecutor(plan, model, world, dropout_attn=0.1, dropout_hidden=0.1)
    ex.init_params(seed=1, std=0.02)
    first, last = model["layers"][0]["shape"], model["layers"][-1]["shape"]
    B = plan["batch_size"]
    x = torch.randn(B * first["seq"], first["hidden"], device="cuda").to(torch.bfloat16)
    t = torch.randn(B * last["seq"], last["hidden"], device="cuda").to(torch.bfloat16)
    ex.load_batch_device(x, t)
    ex.run(use_graph=True)
    torch.cuda.synchronize()
    setup = time.time() - t0
    st = torch.cuda.ExternalStream(ex.stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        ex.run(use_graph=True)
    b.record(st)
    torch.cuda.synchronize()
    loss = ex.loss()
    info = ex.info()
    ex.close()
    return {"run": label, "plan": planner.ribbon(plan).replace("||", "|| "), "batch_size": B,
            "pp_degree": plan["pp_degree"], "micro_batches": plan["micro_batches"],
            "world": world, "comm": "sim (all ranks on cuda:0)",
            "ms_per_step": round(a.elapsed_time(b) / steps, 3), "loss": loss,
            "loss_finite": math.isfinite(loss),
            "device_gib_all_ranks": round(sum(r["device_bytes"] for r in info["ranks"]) / 2**30, 2),
            "setup_s": round(setup, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    runs = _runs()
    keys = [k for k in runs if not args.only or k in args.only.split(",")]
    ok = True
    for k in keys:
        label, model, plan, world = runs[k]
        try:
            res = run_one(label, model, plan, world, args.steps)
            ok &= res["loss_finite"]
        except Exception as e:  # report and continue with the next config
            res = {"run": label, "error": str(e)[:300]}
            ok = False
        torch.cuda.empty_cache()
        print(json.dumps(res), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
