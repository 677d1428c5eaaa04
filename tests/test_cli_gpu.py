"""`parplan run` / `parplan profile` on the B200 (the executor-facing CLI subcommands of
SURVEY.md §8(f)1): the searched plan executes through libgx.so, its loss agrees with the
Python front-end on the same batch, and the profile output feeds back into `parplan plan`."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2211_13878_b200 import executor as gxe

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2211_13878_b200", "parplan")
H, HEADS, SEQ, FFN = 256, 4, 64, 1024
SHAPE = {"hidden": H, "heads": HEADS, "head_dim": H // HEADS, "seq": SEQ, "ffn": FFN,
         "kind": "encoder"}


def _model(L=2, shape=True):
    pbytes = 4 * (12 * H * H + 13 * H)
    layers = []
    for _ in range(L):
        d = {"param_bytes": pbytes, "activation_bytes_per_sample": 4 * SEQ * H * 20,
             "fwd_time_per_sample_ms": 0.05}
        if shape:
            d["shape"] = dict(SHAPE)
        layers.append(d)
    return {"dtype_bytes": 4, "layers": layers}


def _cluster(n):
    return {"num_devices": n, "memory_budget_bytes": 16 << 30, "island_size": n,
            "intra_island_bw_gbps": 13.0, "inter_island_bw_gbps": 13.0}


def _run(*args, timeout=600):
    assert os.path.exists(CLI), "parplan binary not built (make)"
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def _dump(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj))
    return str(p)


def _synthetic_bf16(n, seed):
    """parplan_cli.cc synthetic_bf16: 64-bit LCG + Box-Muller, fp32 -> bf16 (RNE) bits."""
    A, C, M = 6364136223846793005, 1442695040888963407, (1 << 64) - 1
    s = (seed * A + C) & M
    u = np.empty(2 * n)
    for i in range(2 * n):
        s = (s * A + C) & M
        u[i] = ((s >> 11) + 0.5) * (1.0 / 9007199254740992.0)
    x = (np.sqrt(-2.0 * np.log(u[0::2])) * np.cos(6.283185307179586 * u[1::2])).astype(np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def test_run_searched_plan_one_device(tmp_path):
    m = _dump(tmp_path, "m.json", _model())
    c = _dump(tmp_path, "c.json", _cluster(1))
    rep = tmp_path / "rep.json"
    code, so, se = _run("run", "--model", m, "--cluster", c, "--batches", "2,4", "--steps", 3,
                        "--warmup", 2, "--report", rep)
    assert code == 0, se
    assert "throughput" in so and "step time" in so and "[serial] x2" in so
    r = json.loads(rep.read_text())
    assert r["ms_per_step"] > 0 and r["e2e_ms_per_step"] > 0
    assert math.isfinite(r["loss"]) and r["plan"]["batch_size"] in (2, 4)
    assert r["info"]["ranks"][0]["device_bytes"] > 0


def test_run_loss_matches_python_executor(tmp_path):
    """Same plan, data, seed and parameters through the CLI and through PlanExecutor."""
    model = _model()
    plan = gxe.make_plan(["", ""], 2)
    m = _dump(tmp_path, "m.json", model)
    c = _dump(tmp_path, "c.json", _cluster(1))
    p = _dump(tmp_path, "p.json", plan)
    rep = tmp_path / "rep.json"
    code, _, se = _run("run", "--model", m, "--cluster", c, "--plan", p, "--steps", 1,
                       "--warmup", 0, "--no-graph", "--seed", 1234, "--report", rep)
    assert code == 0, se
    cli_loss = json.loads(rep.read_text())["loss"]
    rows = 2 * SEQ
    x = _synthetic_bf16(rows * H, 1)
    y = _synthetic_bf16(rows * H, 2)
    ex = gxe.PlanExecutor(plan, model, 1, seed=1234, lr=1e-4)
    ex.init_params(seed=1234, std=0.02)
    ex.load_batch(x, y)
    ex.run(use_graph=False)
    py_loss = ex.loss()
    ex.close()
    assert abs(cli_loss - py_loss) <= 1e-5 * abs(py_loss), (cli_loss, py_loss)


def test_run_is_deterministic_and_simulates_two_ranks(tmp_path):
    m = _dump(tmp_path, "m.json", _model())
    c = _dump(tmp_path, "c.json", _cluster(2))
    losses = []
    for i in range(2):
        rep = tmp_path / f"r{i}.json"
        code, so, se = _run("run", "--model", m, "--cluster", c, "--batches", "4", "--steps", 2,
                            "--warmup", 1, "--dropout", 0.1, "--report", rep)
        assert code == 0, se
        assert "world 2" in so
        losses.append(json.loads(rep.read_text())["loss"])
    assert losses[0] == losses[1]


def test_run_enforce_budget_too_small_is_infeasible(tmp_path):
    m = _dump(tmp_path, "m.json", _model())
    cl = _cluster(1)
    p = _dump(tmp_path, "p.json", gxe.make_plan(["", ""], 2))
    cl["memory_budget_bytes"] = 1 << 20
    c = _dump(tmp_path, "c.json", cl)
    code, _, se = _run("run", "--model", m, "--cluster", c, "--plan", p, "--enforce-budget",
                       "--steps", 1, "--warmup", 0)
    assert code == 2, se
    assert se.startswith("infeasible:")


def test_profile_feeds_the_search(tmp_path):
    m = _dump(tmp_path, "m.json", _model(L=3, shape=False))
    om, op = tmp_path / "mm.json", tmp_path / "pp.json"
    code, so, se = _run("profile", "--model", m, "--shape", f"{H},{HEADS},{SEQ},{FFN}",
                        "--batch", 4, "--steps", 5, "--warmup", 2, "--out-model", om,
                        "--out-profile", op)
    assert code == 0, se
    mm, pp = json.loads(om.read_text()), json.loads(op.read_text())
    assert so.count("shape ") == 1  # one distinct shape measured once
    t = {l["fwd_time_per_sample_ms"] for l in mm["layers"]}
    assert len(t) == 1 and 0 < t.pop() < 5.0
    assert 0.5 < pp["backward_multiplier"] < 10.0
    assert all(l["shape"]["hidden"] == H for l in mm["layers"])
    c = _dump(tmp_path, "c.json", _cluster(8))
    code, so, se = _run("plan", "--model", om, "--cluster", c, "--profile", op, "--batches", "8,16")
    assert code == 0, se
    assert "throughput" in so


def _swin_small():
    layers = []
    for st, (h, heads, grid) in enumerate(((64, 2, 14), (128, 4, 7))):
        for i in range(2):
            sh = {"hidden": h, "heads": heads, "head_dim": 32, "seq": grid * grid, "ffn": 2 * h,
                  "kind": "window", "window": 49}
            if st == 1 and i == 0:
                sh["merge"] = True
            if i == 1:
                sh["shift"] = True
            layers.append({"param_bytes": 4 * (12 * h * h + 13 * h),
                           "activation_bytes_per_sample": 4 * grid * grid * h * 20,
                           "fwd_time_per_sample_ms": 0.05, "shape": sh})
    return {"dtype_bytes": 4, "layers": layers}


def _t5_small():
    m = _model(L=4)
    for layer in m["layers"][2:]:
        layer["shape"]["kind"] = "decoder"
    return m


@pytest.mark.parametrize("name", ["swin", "t5"])
def test_run_and_profile_other_layer_families(tmp_path, name):
    """`run` executes Swin (windows, SW-MSA, merging) and T5 (decoder) models; `profile`
    times a merging layer behind its predecessor and writes planner-loadable inputs."""
    model = _swin_small() if name == "swin" else _t5_small()
    m = _dump(tmp_path, "m.json", model)
    c = _dump(tmp_path, "c.json", _cluster(2))
    rep = tmp_path / "rep.json"
    code, so, se = _run("run", "--model", m, "--cluster", c, "--batches", "2,4", "--steps", 2,
                        "--warmup", 1, "--dropout", 0.1, "--report", rep)
    assert code == 0, se
    assert math.isfinite(json.loads(rep.read_text())["loss"])
    om, op = tmp_path / "mm.json", tmp_path / "pp.json"
    code, so, se = _run("profile", "--model", m, "--batch", 2, "--steps", 3, "--warmup", 1,
                        "--out-model", om, "--out-profile", op)
    assert code == 0, se
    times = [l["fwd_time_per_sample_ms"] for l in json.loads(om.read_text())["layers"]]
    assert all(t > 0 for t in times), times
    code, _, se = _run("plan", "--model", om, "--cluster", c, "--profile", op, "--batches", "2,4")
    assert code == 0, se
