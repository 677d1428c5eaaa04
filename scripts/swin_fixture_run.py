"""Run the Swin fixture (BASELINE config 5) end to end under the plan the search picks.

The reference's swin-like-heterogeneous model (2/2/26/2 layers, hidden 320 -> 2560) on the
8-GPU / 8 GiB cluster plans as [dp:8] x6 | [sdp:8] x24 | [tp:2,sdp:4] x2 at B=64 (SURVEY.md
§8(a) golden table), which exercises window attention (head_dim 32), three patch-merging
layers (the last one a 5120-wide LayerNorm) and two strategy transitions (dp -> sdp: same
data layout; sdp:8 -> tp:2,sdp:4: all-gather of k=2 sub-chunks).  All eight ranks run in this
process on one GPU (comm "sim"), so the step time is a functional check, not cluster
throughput.

    python scripts/swin_fixture_run.py [--steps 3] [--budget-gib 8] [--batch B]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--budget-gib", type=float, default=8)
    ap.add_argument("--batch", type=int, default=0, help="override the searched batch size")
    args = ap.parse_args()
    model = models.model("swin-like")
    out = planner.api().optimize(model, models.cluster(8, args.budget_gib))
    plan = out.plan
    assert plan is not None, out.diagnostic
    if args.batch:
        plan = dict(plan, batch_size=args.batch)
    ribbon = planner.ribbon(plan)
    torch.cuda.set_device(0)
    t0 = time.time()
    ex = gxe.PlanExecutor(plan, model, 8, dropout_attn=0.1, dropout_hidden=0.1)
    ex.init_params(seed=1, std=0.02)
    first, last = model["layers"][0]["shape"], model["layers"][-1]["shape"]
    B = plan["batch_size"]
    x = torch.randn(B * first["seq"], first["hidden"], device="cuda").to(torch.bfloat16)
    t = torch.randn(B * last["seq"], last["hidden"], device="cuda").to(torch.bfloat16)
    ex.load_batch_device(x, t)
    ex.run(use_graph=True)  # capture + first step
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    stream = torch.cuda.ExternalStream(ex.stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        ex.run(use_graph=True)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    loss = ex.loss()
    info = ex.info()
    dev_bytes = sum(r["device_bytes"] for r in info["ranks"])
    print(json.dumps({"model": "swin-like (Swin-H fixture)", "plan": ribbon, "batch_size": B,
                      "world": 8, "comm": "sim (8 ranks on one GPU)", "ms_per_step": round(ms, 3),
                      "loss": loss, "loss_finite": math.isfinite(loss),
                      "device_gib_all_ranks": round(dev_bytes / 2**30, 2),
                      "setup_s": round(setup_s, 1)}))
    ex.close()
    assert math.isfinite(loss)


if __name__ == "__main__":
    main()
