"""The fp32 C + OpenMP CPU restatement (oracle/cpu_layer.c: the CPU baseline of bench.py and
BASELINE.md §4.2) agrees with the float64 numpy oracle (oracle/layer_oracle.py, itself pinned
to torch.autograd): outputs, input gradient, every parameter gradient, dropout masks
(bit-identical Philox keep decisions, or the errors would be O(1)) and the AdamW update."""
import numpy as np
import pytest

from oracle import cpu_layer as cl
from oracle import layer_oracle as lo


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("p_drop", [0.0, 0.1])
@pytest.mark.parametrize("seq", [64, 80])
def test_cpu_layer_matches_oracle(p_drop, seq):
    h, H, f, n, L = 128, 4, 512, 2, 2
    sh = lo.LayerShape(h, H, seq, f)
    rng = np.random.default_rng(1)
    params = [{k: v.astype(np.float32).astype(np.float64)
               for k, v in lo.init_layer_params(sh, rng, 0.05).items()} for _ in range(L)]
    x = rng.standard_normal((n * seq, h))
    t = rng.standard_normal((n * seq, h))
    m = cl.CpuModel(L, n, seq, h, H, f, p_drop, p_drop, 3)
    for li in range(L):
        m.set_layer(li, params[li])
    loss, y, dx = m.step(x, t, optimizer=False, want=True)
    rl, ry, rdx, rg = lo.model_step(params, x, t, sh, lo.Dropout(p_drop, p_drop, 3))
    assert abs(loss - rl) <= 1e-5 * abs(rl)
    assert rel(y, ry) < 2e-6 and rel(dx, rdx) < 2e-6
    for li in range(L):
        g = m.layer_grads(li)
        for k in g:
            assert rel(g[k], rg[li][k]) < 5e-6, (li, k)
    m.close()


def test_cpu_adamw_matches_reference():
    h, H, s, f = 64, 2, 32, 128
    sh = lo.LayerShape(h, H, s, f)
    rng = np.random.default_rng(4)
    P = {k: v.astype(np.float32) for k, v in lo.init_layer_params(sh, rng, 0.05).items()}
    x = rng.standard_normal((s, h)).astype(np.float32)
    m = cl.CpuModel(1, 1, s, h, H, f)
    m.set_layer(0, P)
    m.step(x, x, optimizer=True, lr=1e-3, wd=0.01)
    g = m.layer_grads(0)
    after = m.layer_params(0)
    for k in P:
        ref, _, _ = lo.adamw_reference(P[k].astype(np.float64), g[k].astype(np.float64),
                                       0.0, 0.0, 1, 1e-3, 0.9, 0.999, 1e-8, 0.01)
        assert np.allclose(after[k], ref, rtol=1e-5, atol=1e-6), k
    m.close()
