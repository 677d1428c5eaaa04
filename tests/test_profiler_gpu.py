"""Profiler loop: B200-measured layer times feed the search; this repo's
planner and the reference planner (oracle/_ref) must pick the identical plan on them, and
the executor must run it."""
import json

import pytest

from paper_2211_13878_b200 import executor as gxe
from oracle import ref_planner
from paper_2211_13878_b200 import models, planner, profiler

pytestmark = pytest.mark.gpu


def _small(L=4):
    shape = {"hidden": 256, "heads": 4, "head_dim": 64, "seq": 128, "ffn": 1024, "kind": "encoder"}
    p = 4 * (12 * 256 * 256 + 13 * 256)
    return {"dtype_bytes": 4, "layers": [{"param_bytes": p, "activation_bytes_per_sample": 4 * 128 * 256 * 20,
                                          "fwd_time_per_sample_ms": 1.0, "shape": dict(shape)}
                                         for _ in range(L)]}


def test_profile_feeds_search(cuda):
    m, prof, raw = profiler.profile_model(_small(), batch=4)
    t = m["layers"][0]["fwd_time_per_sample_ms"]
    assert 0 < t < 1.0
    assert 0.5 < prof["backward_multiplier"] < 10
    # GEMM || collective slowdown (cost_model.cc:200-206), measured with the 1-GPU proxy here
    assert 1.0 <= prof["overlap_slowdown"] < 4.0, raw["overlap"]
    assert raw["overlap"]["t_both_ms"] >= raw["overlap"]["t_step_ms"] * 0.95
    print("\noverlap:", json.dumps(raw["overlap"]))
    cluster = models.cluster(4, 0.25, 700.0)
    a = planner.api().optimize(m, cluster, prof, [4, 8, 16])
    if ref_planner.available():
        b = ref_planner.api().optimize(m, cluster, prof, [4, 8, 16])
        assert a.plan_text == b.plan_text
    assert a.plan is not None
    # the measured knobs (backward_multiplier, overlap_slowdown) re-plan BERT-Huge-32 at every
    # (N, budget) of the metric identically in both planners
    if ref_planner.available():
        bert = models.model("bert-huge-32")
        for n in (1, 2, 4, 8):
            for e in (8, 16):
                c = models.cluster(n, e, 700.0)
                for batches in (None, list(range(1, 65))):
                    x = planner.api().optimize(bert, c, prof, batches)
                    y = ref_planner.api().optimize(bert, c, prof, batches)
                    assert x.plan_text == y.plan_text and x.diagnostic == y.diagnostic, (n, e)
    ex = gxe.PlanExecutor(a.plan, m, 4, optimizer=True)
    ex.init_params(seed=3, std=0.02)
    import torch
    rows = a.plan["batch_size"] * 128
    x = torch.randn(rows, 256).to(torch.bfloat16)
    loss = ex.step(x.view(torch.int16).numpy(), x.view(torch.int16).numpy())
    assert loss == loss and loss > 0


def test_nccl_world_of_one_matches_sim(cuda):
    """The NCCL backend (one rank) runs the same step as the simulated world."""
    import numpy as np
    m = _small(2)
    plan = gxe.make_plan(["", ""], 2)
    outs = []
    for comm in ("sim", "nccl"):
        kw = {"comm": comm}
        if comm == "nccl":
            kw["nccl_id_hex"] = gxe.nccl_unique_id()
            kw["local_ranks"] = [0]
        ex = gxe.PlanExecutor(plan, m, 1, optimizer=False, **kw)
        ex.init_params(seed=5, std=0.02)
        rng = np.random.default_rng(0)
        xb = gxe.f32_to_bf16_bits(rng.standard_normal((2 * 128, 256)).astype(np.float32))
        outs.append((ex.step(xb, xb), ex.export_output("y")))
        ex.close()
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])


def test_profile_swin_merging_layer(cuda):
    """A patch-merging layer is timed behind its predecessor (minus the predecessor)."""
    from tests.test_cli_gpu import _swin_small
    m, prof, raw = profiler.profile_model(_swin_small(), batch=2, overlap=False)
    times = [l["fwd_time_per_sample_ms"] for l in m["layers"]]
    assert all(t > 0 for t in times), times
    assert 0.3 < prof["backward_multiplier"] < 10
