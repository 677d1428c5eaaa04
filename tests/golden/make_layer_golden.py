"""Writes tests/golden/layer_small.npz: one small layer fwd/bwd of the CPU oracle with
Philox dropout (p=0.1), after the oracle was checked against torch.autograd
(tests/test_layer_oracle.py).  Re-run only when the layer definition changes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import layer_oracle as lo  # noqa: E402

rng = np.random.default_rng(20261017)
shape = lo.LayerShape(hidden=64, heads=2, seq=16, ffn=256)
P = lo.init_layer_params(shape, rng, std=0.05)
x = rng.standard_normal((2 * shape.seq, shape.hidden))
dy = rng.standard_normal(x.shape)
drop = lo.Dropout(0.1, 0.1, 1234)
y, cache = lo.layer_forward(P, x, shape, 1, drop, 0)
dx, G = lo.layer_backward(P, dy, cache, shape)
out = {"shape": np.array([shape.hidden, shape.heads, shape.seq, shape.ffn]), "p": 0.1,
       "seed": 1234, "x": x, "dy": dy, "y": y, "dx": dx}
out.update({"P_" + k: v for k, v in P.items()})
out.update({"G_" + k: v for k, v in G.items()})
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "layer_small.npz"), **out)
print("wrote layer_small.npz")
