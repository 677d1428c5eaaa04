"""Runs the bench workload eagerly (no graph): W warm-up steps then 1 step, for ncu launch
lists of exactly one step (skip the warm-up launches with ncu -s; the count is printed)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
import bench  # noqa: E402

W = int(os.environ.get("WARMUP", "2"))
from paper_2211_13878_b200 import planner  # noqa: E402
model, plan, _ = bench.search(planner.api(), os.environ.get("MODEL", "bert-huge-32"), 1, 16.0)
sh = model["layers"][0]["shape"]
x = torch.randn(plan["batch_size"] * sh["seq"], sh["hidden"]).to(torch.bfloat16)
ex = gxe.PlanExecutor(plan, model, 1, dropout_attn=0.1, dropout_hidden=0.1)
ex.init_params(seed=7, std=0.02)
ex.load_batch(x.view(torch.int16), x.view(torch.int16))
for _ in range(W):
    ex.run(False)
torch.cuda.synchronize()
print("launches_per_step", ex.info()["launches_per_step"], file=sys.stderr)
ex.run(False)
torch.cuda.synchronize()
