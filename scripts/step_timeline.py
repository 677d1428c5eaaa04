"""Eager-mode timeline of one bench step (executor cfg "trace": CUDA events at phase marks):
when the forward, each layer's backward and each layer's AdamW begin / end (ms since the
step's first mark).  python scripts/step_timeline.py ['{"opt": ...}']"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_13878_b200 import planner  # noqa: E402
from paper_2211_13878_b200 import executor as gxe  # noqa: E402

opts = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
model, plan, _ = bench.search(planner.api(), "bert-huge-32", 1, 16.0)
ex = gxe.PlanExecutor(plan, model, 1, dropout_attn=0.1, dropout_hidden=0.1, seed=1234, lr=1e-4,
                      trace=True, **opts)
ex.init_params(seed=7, std=0.02)
sh = model["layers"][0]["shape"]
x = torch.randn(plan["batch_size"] * sh["seq"], sh["hidden"], device="cuda").to(torch.bfloat16)
ex.load_batch_device(x, x)
for _ in range(3):
    ex.run(use_graph=False)
torch.cuda.synchronize()
rep = ex.profile_report()
print(json.dumps(rep.get("timeline", rep))[:6000])
