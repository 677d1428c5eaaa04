"""One BASELINE config's plan (all ranks simulated on one GPU) run eagerly: W warm-up steps
then 1 step, for ncu launch lists of exactly one step (the launch count goes to stderr):
  CONFIG=vit WARMUP=2 python scripts/config_step_once.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from scripts.config_runs import _runs  # noqa: E402

W = int(os.environ.get("WARMUP", "2"))
title, model, plan, world = _runs()[os.environ.get("CONFIG", "vit")][:4]
ex = gxe.PlanExecutor(plan, model, world, dropout_attn=0.1, dropout_hidden=0.1, seed=1, lr=1e-4)
ex.init_params(seed=7, std=0.02)
B = plan["batch_size"]
sh, shl = model["layers"][0]["shape"], model["layers"][-1]["shape"]
ex.load_batch(torch.zeros(B * sh["seq"], sh["hidden"], dtype=torch.int16),
              torch.zeros(B * shl["seq"], shl["hidden"], dtype=torch.int16))
for _ in range(W):
    ex.run(False)
torch.cuda.synchronize()
info = ex.info()
print("launches_per_step", info["launches_per_step"], file=sys.stderr)
ex.run(False)
torch.cuda.synchronize()
