"""Regenerates tests/golden/ref_plans.json from the REFERENCE planner (oracle/_ref, built
from /root/reference by oracle/Makefile).  Run in the build container:

    make -C oracle && python tests/golden/make_ref_plans.py

Each case records the reference's PlanToJson text (or its infeasibility diagnostic) for the
BASELINE configs; tests/test_plan_parity.py requires the product planner to reproduce the
text byte for byte (doubles included).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref_planner  # noqa: E402
from paper_2211_13878_b200 import models  # noqa: E402

ONE_TO_512 = list(range(1, 513))


def cases():
    out = []
    for n in (1, 2, 4, 8):
        for e in (8, 16):
            out.append(("bert-huge-32", n, e, None, 13.0))
            out.append(("bert-huge-32", n, e, ONE_TO_512, 13.0))
    for e in (8, 16):
        out.append(("swin-like", 8, e, None, 13.0))
        out.append(("vit-huge-32", 8, e, None, 13.0))
        out.append(("t5-large-48", 8, e, None, 13.0))
        out.append(("bert-huge-32", 8, e, None, 700.0))   # B200-like bandwidth
    out.append(("bert-base-2", 8, 8, [8], 13.0))
    out.append(("t5-large-48", 4, 16, None, 13.0))
    out.append(("t5-large-48", 2, 16, None, 13.0))
    return out


def main():
    api = ref_planner.api()
    res = []
    for name, n, e, batches, bw in cases():
        m = models.model(name)
        c = models.cluster(n, e, bw)
        o = api.optimize(m, c, None, batches)
        res.append({"model": name, "num_devices": n, "budget_gib": e, "bw_gbps": bw,
                    "batches": "1..512" if batches == ONE_TO_512 else batches,
                    "plan_text": o.plan_text, "diagnostic": o.diagnostic})
        print(name, n, e, bw, "OOM" if o.plan is None else
              f"B={o.plan['batch_size']} P={o.plan['pp_degree']} m={o.plan['micro_batches']}")
    with open(os.path.join(ROOT, "tests", "golden", "ref_plans.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
