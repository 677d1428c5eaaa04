import sys, ctypes, numpy as np
sys.path.insert(0, ".")
from tests.test_executor_gpu import _small_model, rel
from oracle import layer_oracle as lo
from paper_2211_13878_b200 import executor as gxe, _lib
def act(ex, l, k, rows, w):
    out = np.zeros((rows, w), dtype=np.uint16)
    _lib.check(_lib.lib().gx_exec_export_output(ex._h, 1000 + 16 * l + k, out.ctypes.data_as(ctypes.c_void_p)))
    return gxe.bf16_bits_to_f32(out)
world, strat, B, L = (2, ["dp:2"]*4, 4, 4)
for trial in range(3):
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
    ex = gxe.PlanExecutor(plan, model, world, optimizer=False, forward_only=True)
    for l in range(L):
        ex.set_layer_params(l, params[l])
    ex.step(xb, tb)
    hcur = x
    for l in range(L):
        inp = hcur
        hcur, c = lo.layer_forward(params[l], hcur, osh, l)
        names = ["x", "ln1", "x1", "ln2", "gel", "y"]
        refs = [inp, c["a"], c["x1"], c["c"], c["g"], hcur]
        res = {}
        for k, (nm, rf) in enumerate(zip(names, refs)):
            g = act(ex, l, k, rows, rf.shape[1])
            res[nm] = [round(rel(g[i*64:(i+1)*64], rf[i*64:(i+1)*64]), 3) for i in range(B)]
        print("trial", trial, "layer", l, res)
    ex.close()
