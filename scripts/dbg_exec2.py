import sys, numpy as np
sys.path.insert(0, ".")
from tests.test_executor_gpu import _small_model, rel
from oracle import layer_oracle as lo
from paper_2211_13878_b200 import executor as gxe
for fo in [True, False]:
  for world, strat, B, L in [(2, ["dp:2"]*4, 4, 4), (2, ["sdp:2"]*2, 4, 2)]:
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
    x = gxe.bf16_bits_to_f32(xb).astype(np.float64)
    ex = gxe.PlanExecutor(plan, model, world, optimizer=False, forward_only=fo)
    for l in range(L):
        ex.set_layer_params(l, params[l])
    for rep in range(2):
        ex.step(xb, tb)
        hcur = x
        res = []
        for l in range(L):
            hcur, _ = lo.layer_forward(params[l], hcur, osh, l)
            y = ex.export_output(l)
            res.append([round(rel(y[i*osh.seq:(i+1)*osh.seq], hcur[i*osh.seq:(i+1)*osh.seq]),4) for i in range(B)])
        print("fwd_only" if fo else "full", world, strat[0], "rep", rep, res)
