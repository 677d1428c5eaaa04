"""Measures BERT-Huge-32 layer times (and the GEMM || collective overlap slowdown) on this
B200 and re-plans with the product planner.  (The reference planner's identical choice on
measured inputs is asserted in tests/test_profiler_gpu.py.)"""
import json, sys
sys.path.insert(0, ".")
from paper_2211_13878_b200 import models, planner, profiler
m, prof, raw = profiler.profile_model(models.model("bert-huge-32"), batch=4)
out = {"measured": raw, "profile": prof, "fwd_time_per_sample_ms": m["layers"][0]["fwd_time_per_sample_ms"],
       "plans": []}
for n in (1, 2, 4, 8):
    for e in (8, 16):
        for bw in (13.0, 700.0):
            c = models.cluster(n, e, bw)
            a = planner.api().optimize(m, c, prof)
            if a.plan is None:
                a = planner.api().optimize(m, c, prof, list(range(1, 513)))
            out["plans"].append({"N": n, "budget_gib": e, "bw_gbps": bw,
                                 "plan": planner.ribbon(a.plan) if a.plan else None,
                                 "B": a.plan["batch_size"] if a.plan else None,
                                 "pp": a.plan["pp_degree"] if a.plan else None,
                                 "predicted_samples_per_s": a.plan["throughput_samples_per_s"] if a.plan else None})
print(json.dumps(out, indent=1))
