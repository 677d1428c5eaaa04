"""Eager-mode timeline of one bench step: layer backward starts vs optimizer start/end."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
import bench  # noqa: E402
from paper_2211_13878_b200 import planner  # noqa: E402
model, plan, _ = bench.search(planner.api(), "bert-huge-32", 1, 16.0)
sh = model["layers"][0]["shape"]
x = torch.randn(plan["batch_size"] * sh["seq"], sh["hidden"]).to(torch.bfloat16)
kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
ex = gxe.PlanExecutor(plan, model, 1, dropout_attn=0.1, dropout_hidden=0.1, trace=True, **kw)
ex.init_params(seed=7, std=0.02)
ex.load_batch(x.view(torch.int16), x.view(torch.int16))
for _ in range(3):
    ex.run(False)
torch.cuda.synchronize()
ex.run(False)
tr = ex.profile_report()["trace"]
print(" ".join(f"{n}={t:.2f}" for n, t in tr))
