"""Per-category device time (instrumented replay) of one BASELINE config's plan on one GPU
(all ranks simulated): python scripts/config_profile.py t5p8|swin|vit"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
from scripts.config_runs import _runs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "t5p8"
title, model, plan, world = _runs()[name][:4]
ex = gxe.PlanExecutor(plan, model, world, dropout_attn=0.1, dropout_hidden=0.1, seed=1, lr=1e-4)
ex.init_params(seed=7, std=0.02)
B = plan["batch_size"]
sh, shl = model["layers"][0]["shape"], model["layers"][-1]["shape"]
x = torch.zeros(B * sh["seq"], sh["hidden"], dtype=torch.int16)
t = torch.zeros(B * shl["seq"], shl["hidden"], dtype=torch.int16)
ex.load_batch(x, t)
for _ in range(2):
    ex.run(False, profile=True)
rep = ex.profile_report()
cats = {k: round(v["ms"], 3) for k, v in rep["categories"].items()}
print(json.dumps({"run": title, "sum_ms": round(rep["sum_ms"], 3), "categories_ms": cats}))
