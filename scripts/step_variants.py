"""Graph-replayed step time of the bench workload under executor variants (what bounds the step)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import executor as gxe  # noqa: E402
import bench  # noqa: E402

model, plan, _ = bench.choose_plan(1, 16.0, "bert-huge-32")
B = plan["batch_size"]
sh = model["layers"][0]["shape"]
rows, h = B * sh["seq"], sh["hidden"]
x = torch.randn(rows, h).to(torch.bfloat16)
variants = [("default", {}), ("no_optimizer", {"optimizer": False}),
            ("forward_only", {"forward_only": True}), ("no_wgrad_stream", {"wgrad_stream": False}),
            ("no_splitk", {"splitk": False}),
            ("opt_blocks_148", {"optimizer_blocks": 148}),
            ("opt_blocks_592", {"optimizer_blocks": 592}),
            ("opt_blocks_1184", {"optimizer_blocks": 1184}),
            ("opt_blocks_4736", {"optimizer_blocks": 4736}),
            ("opt_blocks_16384", {"optimizer_blocks": 16384}),
            ("opt_group2_4736", {"optimizer_blocks": 4736, "optimizer_group": 2}),
            ("defer_4736", {"optimizer_blocks": 4736, "defer_optimizer": True})]
for name in (sys.argv[1:] or [v[0] for v in variants]):
    kw = dict(variants)[name]
    ex = gxe.PlanExecutor(plan, model, 1, dropout_attn=0.1, dropout_hidden=0.1, **kw)
    ex.init_params(seed=7, std=0.02)
    ex.load_batch(x.view(torch.int16), x.view(torch.int16))
    st = torch.cuda.ExternalStream(ex.stream)
    for _ in range(3):
        ex.run(True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10):
        ex.run(True)
    b.record(st)
    torch.cuda.synchronize()
    print(json.dumps({"variant": name, "ms_per_step": round(a.elapsed_time(b) / 10, 4),
                      "loss": ex.loss()}), flush=True)
    ex.close()
