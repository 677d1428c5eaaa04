"""A/B of executor options on the bench workload (BERT-Huge-32, the searched N = 1 plan):
graph-replayed ms per step for each option set, alternating, two rounds.

  python scripts/knob_ab.py '{}' '{"splitk": false}'
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_13878_b200 import _lib, planner  # noqa: E402
from paper_2211_13878_b200 import executor as gxe  # noqa: E402


def step_ms(opts, model_name="bert-huge-32", n=1, budget=16.0):
    model, plan, _ = bench.search(planner.api(), model_name, n, budget)
    ex = gxe.PlanExecutor(plan, model, 1, dropout_attn=0.1, dropout_hidden=0.1, seed=1234,
                          lr=1e-4, **opts)
    ex.init_params(seed=7, std=0.02)
    sh = model["layers"][0]["shape"]
    x = torch.randn(plan["batch_size"] * sh["seq"], sh["hidden"], device="cuda").to(torch.bfloat16)
    ex.load_batch_device(x, x)
    ms = ctypes.c_double()
    _lib.check(_lib.lib().gx_exec_time(ex._h, 1, 5, 20, ctypes.byref(ms)))
    ex.close()
    return ms.value


if __name__ == "__main__":
    variants = [json.loads(a) for a in sys.argv[1:]] or [{}]
    for rnd in range(2):
        for v in variants:
            print(json.dumps({"round": rnd, "opts": v, "ms_per_step": round(step_ms(v), 4)}),
                  flush=True)
