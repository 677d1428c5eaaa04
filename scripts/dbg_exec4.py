import sys, ctypes, numpy as np
sys.path.insert(0, ".")
from tests.test_executor_gpu import _small_model, rel
from oracle import layer_oracle as lo
from paper_2211_13878_b200 import executor as gxe, _lib
world, strat, B, L = (2, ["dp:2"]*4, 4, 4)
for trial in range(6):
    plan = gxe.make_plan(strat, B)
    model = _small_model(L=L)
    shp = model["layers"][0]["shape"]
    osh = lo.LayerShape(shp["hidden"], shp["heads"], shp["seq"], shp["ffn"])
    rng = np.random.default_rng(11)
    params = [lo.init_layer_params(osh, rng, std=0.05) for _ in range(L)]
    params = [{k: v.astype(np.float32).astype(np.float64) for k, v in P.items()} for P in params]
    rows = B * osh.seq
    xb = gxe.f32_to_bf16_bits(rng.standard_normal((rows, osh.hidden)).astype(np.float32))
    tb = gxe.f32_to_bf16_bits(rng.standard_normal((rows, osh.hidden)).astype(np.float32))
    ex = gxe.PlanExecutor(plan, model, world, optimizer=False, forward_only=True)
    for l in range(L):
        ex.set_layer_params(l, params[l])
    bad0 = [(l, k) for l in range(L) for k, v in ex.export_layer(l, "bf16").items() if rel(v, params[l][k]) > 1e-2]
    ex.step(xb, tb)
    bad1 = [(l, k) for l in range(L) for k, v in ex.export_layer(l, "bf16").items() if rel(v, params[l][k]) > 1e-2]
    print("trial", trial, "bad after set", bad0, "bad after step", bad1, flush=True)
    ex.close()
