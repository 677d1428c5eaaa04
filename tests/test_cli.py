"""The `parplan` command line (paper_2211_13878_b200/csrc/tools/parplan_cli.cc) against the
reference CLI's contract (proj/tools/parplan_main.cc): subcommands, flags, exit codes 0/1/2,
summary text, plan JSON, CSV.  The reference CLI itself cannot be built here (CLI11 is
absent), so parity is anchored on (1) the reference's golden PlanToJson texts
(tests/golden/ref_plans.json, made by the reference library), (2) the product planner's C
surface for estimate / enumerate / sweep values, and (3) the reference's own cli_test.cc,
compiled against this binary in tests/test_reference_suites.py.
"""
import json
import os
import subprocess

import pytest

from paper_2211_13878_b200 import models, planner

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2211_13878_b200", "parplan")
GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_plans.json")


@pytest.fixture(scope="module")
def cli():
    r = subprocess.run(["make", "-s", "-C", ROOT, "paper_2211_13878_b200/parplan"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return CLI


def run(cli, *args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300, env=e)
    return r.returncode, r.stdout, r.stderr


def dump(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj))
    return str(p)


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _ribbon(stage):
    out, i, s = [], 0, [l["strategy"] for l in stage["layers"]]
    while i < len(s):
        j = i
        while j < len(s) and s[j] == s[i]:
            j += 1
        out.append(f"[{s[i] or 'serial'}] x{j - i}")
        i = j
    return " | ".join(out)


def _summary(p):
    lines = [f"batch size       {p['batch_size']}",
             f"pp degree        {p['pp_degree']}  (micro-batches: {p['micro_batches']})",
             f"iteration time   {p['iteration_time_ms']:.3f} ms",
             f"throughput       {p['throughput_samples_per_s']:.3f} samples/s"]
    for i, st in enumerate(p["stages"]):
        b, e = st["layer_range"]
        lines.append(f"stage {i}  layers [{b},{e})  cost {st['stage_cost_ms']:.3f} ms  "
                     f"peak {st['peak_memory_bytes'] / (1 << 30):.2f} GiB")
        lines.append(f"  {_ribbon(st)}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("case", _golden(),
                         ids=lambda c: f"{c['model']}-N{c['num_devices']}-E{c['budget_gib']}-"
                                       f"bw{c['bw_gbps']}-{c['batches']}")
def test_plan_reproduces_reference_golden(cli, tmp_path, case):
    batches = list(range(1, 513)) if case["batches"] == "1..512" else case["batches"]
    m = dump(tmp_path, "m.json", models.model(case["model"]))
    c = dump(tmp_path, "c.json", models.cluster(case["num_devices"], case["budget_gib"],
                                                case["bw_gbps"]))
    out = tmp_path / "plan.json"
    args = ["plan", "--model", m, "--cluster", c, "--out", out]
    if batches:
        args += ["--batches", ",".join(map(str, batches))]
    code, so, se = run(cli, *args)
    if case["plan_text"] is None:
        assert code == 2
        assert se == f"infeasible: {case['diagnostic']}\n"
        assert not out.exists()
    else:
        assert code == 0, se
        ref = json.loads(case["plan_text"])
        assert json.loads(out.read_text()) == ref
        assert so == _summary(ref)


def test_plan_without_out_prints_summary_then_json(cli, tmp_path):
    m = dump(tmp_path, "m.json", models.model("bert-huge-32"))
    c = dump(tmp_path, "c.json", models.cluster(8, 8))
    code, so, _ = run(cli, "plan", "--model", m, "--cluster", c)
    assert code == 0
    ref = planner.api().optimize(models.model("bert-huge-32"), models.cluster(8, 8)).plan
    summary = _summary(ref)
    assert so.startswith(summary)
    assert json.loads(so[len(summary):]) == ref
    assert "[sdp:8] x32" in so


def test_flag_spellings(cli, tmp_path):
    """--flag=value, space-separated lists and the guideline choices, as CLI11 accepts them."""
    m = dump(tmp_path, "m.json", models.model("swin-like"))
    c = dump(tmp_path, "c.json", models.cluster(8, 8))
    outs = []
    for i, spelling in enumerate((["--batches", "8,16"], ["--batches=8,16"], ["--batches", "8", "16"])):
        p = tmp_path / f"p{i}.json"
        code, _, se = run(cli, "plan", f"--model={m}", "--cluster", c, *spelling, "--out", p)
        assert code == 0, se
        outs.append(json.loads(p.read_text()))
    assert outs[0] == outs[1] == outs[2]
    ref = planner.api().optimize(models.model("swin-like"), models.cluster(8, 8), None, [8, 16]).plan
    assert outs[0] == ref
    for g in ("layers", "params", "memory", "time"):
        p = tmp_path / f"g{g}.json"
        code, _, se = run(cli, "plan", "--model", m, "--cluster", c, "--batches", "8",
                          "--pp-guideline", g, "--no-prune", "--out", p)
        assert code == 0, se
        want = planner.api().optimize(models.model("swin-like"), models.cluster(8, 8), None, [8],
                                      prune=False, guideline=g).plan
        assert json.loads(p.read_text()) == want


@pytest.mark.parametrize("args,needle", [
    ([], "usage"),
    (["frobnicate"], "unknown subcommand"),
    (["plan"], "--model is required"),
    (["plan", "--model", "x.json"], "--cluster is required"),
    (["plan", "--model", "x", "--cluster", "y", "--pp-guideline", "depth"], "pp-guideline"),
    (["plan", "--model", "x", "--cluster", "y", "--bogus"], "unknown option --bogus"),
    (["plan", "--model", "x", "--cluster", "y", "--batches", "8,x"], "not an integer"),
    (["enumerate"], "--group-size is required"),
    (["enumerate", "--group-size", "3"], "power of two"),
    (["enumerate", "--group-size", "8", "--no-prune=1"], "takes no value"),
    (["sweep", "--model", "x", "--cluster", "y"], "--budgets is required"),
    (["plan", "--model", "/nonexistent/m.json", "--cluster", "y"], "model"),
])
def test_usage_and_config_errors_exit_1(cli, args, needle):
    code, so, se = run(cli, *args)
    assert code == 1
    assert needle in se


def test_help_exits_0(cli):
    for args in (["--help"], ["plan", "--help"], ["run", "--help"], ["profile", "-h"]):
        code, so, _ = run(cli, *args)
        assert code == 0 and "usage" in so


@pytest.mark.parametrize("group,prune", [(1, True), (2, True), (4, False), (8, True), (8, False),
                                         (16, True)])
def test_enumerate_matches_library(cli, tmp_path, group, prune):
    args = ["enumerate", "--group-size", group] + ([] if prune else ["--no-prune"])
    code, so, _ = run(cli, *args)
    assert code == 0
    assert json.loads(so) == planner.api().enumerate(group, prune)
    p = tmp_path / "e.json"
    assert run(cli, *args, "--out", p)[0] == 0
    assert json.loads(p.read_text()) == json.loads(so)


@pytest.mark.parametrize("strategy,batch", [("", 1), ("dp:8", 16), ("sdp:2", 8), ("tp:2,sdp:4", 8),
                                            ("tp:4,dp:2", 32)])
def test_estimate_csv_matches_cost_model(cli, tmp_path, strategy, batch):
    mj = models.model("swin-like")
    m = dump(tmp_path, "m.json", mj)
    cj = models.cluster(8, 8)
    c = dump(tmp_path, "c.json", cj)
    csv = tmp_path / "e.csv"
    code, so, se = run(cli, "estimate", "--model", m, "--cluster", c, "--strategy", strategy,
                       "--batch", batch, "--csv", csv)
    assert code == 0, se
    api = planner.api()
    group = 1
    for part in filter(None, strategy.split(",")):
        group *= int(part.split(":")[1])
    bw = api.bandwidth(cj, group)
    assert so.splitlines()[0] == f"strategy {strategy or 'serial'}  batch {batch}  bandwidth {bw:.1f} GB/s"
    rows = csv.read_text().splitlines()
    assert rows[0] == ("layer,forward_ms,backward_ms,comm_ms_unoverlapped,total_ms,params_bytes,"
                       "grads_bytes,optimizer_bytes,activation_bytes,total_bytes")
    assert len(rows) == 1 + len(mj["layers"]) and len(so.splitlines()) == 2 + len(mj["layers"])
    for i, (row, layer) in enumerate(zip(rows[1:], mj["layers"])):
        e = api.estimate(layer["param_bytes"], layer["activation_bytes_per_sample"],
                         layer["fwd_time_per_sample_ms"], strategy, batch, bw)
        want = [str(i)] + ["%.9g" % e[k] for k in (
            "forward_ms", "backward_ms", "comm_ms_unoverlapped", "total_ms", "params_bytes",
            "grads_bytes", "optimizer_bytes", "activation_bytes", "total_bytes")]
        assert row.split(",") == want


def test_estimate_indivisible_batch_is_infeasible(cli, tmp_path):
    m = dump(tmp_path, "m.json", models.model("bert-huge-32"))
    c = dump(tmp_path, "c.json", models.cluster(8, 8))
    code, _, se = run(cli, "estimate", "--model", m, "--cluster", c, "--strategy", "dp:8",
                      "--batch", 4)
    assert code == 2 and se.startswith("infeasible: batch 4")


def test_sweep_rows_match_optimize(cli, tmp_path):
    mj = models.model("bert-huge-32")
    m = dump(tmp_path, "m.json", mj)
    c = dump(tmp_path, "c.json", models.cluster(8, 8))
    csv = tmp_path / "s.csv"
    code, so, se = run(cli, "sweep", "--model", m, "--cluster", c, "--budgets", "0.5,8,12.5,16",
                       "--csv", csv)
    assert code == 0, se
    assert csv.read_text() == so
    rows = so.splitlines()
    assert rows[0] == "budget_gb,batch_size,pp_degree,throughput_samples_per_s"
    for row, gb in zip(rows[1:], (0.5, 8, 12.5, 16)):
        cl = models.cluster(8, 8)
        cl["memory_budget_bytes"] = int(gb * (1 << 30))
        o = planner.api().optimize(mj, cl)
        if o.plan is None:
            assert row == f"{gb:g},OOM,OOM,OOM"
        else:
            p = o.plan
            assert row == f"{gb:g},{p['batch_size']},{p['pp_degree']},{p['throughput_samples_per_s']:.6f}"
    assert run(cli, "sweep", "--model", m, "--cluster", c, "--budgets", "8,-1")[0] == 1


def test_oracle_plan_matches_plan_on_small_instances(cli, tmp_path):
    mj = {"dtype_bytes": 4, "layers": [
        {"param_bytes": 16 << 20, "activation_bytes_per_sample": 4 << 20, "fwd_time_per_sample_ms": 1.0},
        {"param_bytes": 32 << 20, "activation_bytes_per_sample": 2 << 20, "fwd_time_per_sample_ms": 1.5},
        {"param_bytes": 8 << 20, "activation_bytes_per_sample": 6 << 20, "fwd_time_per_sample_ms": 0.5}]}
    m = dump(tmp_path, "m.json", mj)
    for n, gib in ((2, 2), (4, 1)):
        c = dump(tmp_path, "c.json", models.cluster(n, gib, 12.0))
        a, b = tmp_path / "a.json", tmp_path / "b.json"
        ca, sa, _ = run(cli, "plan", "--model", m, "--cluster", c, "--batches", "2,4", "--out", a)
        cb, sb, _ = run(cli, "oracle-plan", "--model", m, "--cluster", c, "--batches", "2,4",
                        "--out", b)
        assert ca == cb == 0 and sa == sb
        assert json.loads(a.read_text()) == json.loads(b.read_text())


def test_planner_threads_env_is_plan_invariant(cli, tmp_path):
    m = dump(tmp_path, "m.json", models.model("bert-huge-32"))
    c = dump(tmp_path, "c.json", models.cluster(8, 16))
    texts = []
    for t in ("1", "3", "8"):
        p = tmp_path / f"t{t}.json"
        assert run(cli, "plan", "--model", m, "--cluster", c, "--out", p,
                   env={"PLANNER_THREADS": t})[0] == 0
        texts.append(p.read_text())
    assert texts[0] == texts[1] == texts[2]


def test_run_and_profile_validate_inputs_before_touching_a_device(cli, tmp_path):
    """Shape errors are configuration errors (exit 1) found on the host."""
    ref_model = {"dtype_bytes": 4, "layers": [
        {"param_bytes": 1 << 20, "activation_bytes_per_sample": 1 << 20, "fwd_time_per_sample_ms": 1.0}]}
    m = dump(tmp_path, "m.json", ref_model)
    c = dump(tmp_path, "c.json", models.cluster(1, 16))
    code, _, se = run(cli, "run", "--model", m, "--cluster", c, "--batches", "1")
    assert code == 1 and "shape" in se
    code, _, se = run(cli, "run", "--model", m, "--cluster", c, "--shape", "1280,3,512,5120")
    assert code == 1 and "--shape" in se
    code, _, se = run(cli, "profile", "--model", m)
    assert code == 1 and "shape" in se
    code, _, se = run(cli, "run", "--model", m, "--cluster", c, "--plan", "/nonexistent/p.json",
                      "--shape", "256,4,64,1024")
    assert code == 1 and "plan" in se


def test_run_nccl_id_rendezvous_between_two_processes(cli, tmp_path):
    """WORLD_SIZE=2: rank 0 publishes the NCCL id through the file, rank 1 picks it up and
    both reach executor creation (which fails here: no GPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only check (on a GPU box rank 0 would block in NCCL init)")
    m = dump(tmp_path, "m.json", {"dtype_bytes": 4, "layers": [
        {"param_bytes": 1 << 20, "activation_bytes_per_sample": 1 << 20,
         "fwd_time_per_sample_ms": 1.0,
         "shape": {"hidden": 256, "heads": 4, "seq": 64, "ffn": 1024}}] * 2})
    c = dump(tmp_path, "c.json", models.cluster(2, 8))
    idf = tmp_path / "nccl.id"
    # a leftover id of an earlier launch on the same path must never be read
    idf.write_text("earlier-launch " + "0" * 256)
    procs = []
    for rank in (1, 0):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(rank), LOCAL_RANK=str(rank),
                   PARPLAN_LAUNCH_ID="this-launch")
        procs.append(subprocess.Popen([cli, "run", "--model", m, "--cluster", c, "--batches", "4",
                                       "--nccl-id-file", str(idf)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 1
        assert "gx_exec_create" in se and "timed out" not in se
    assert "[dp:2] x2" in outs[1][0] and outs[0][0] == ""  # only rank 0 prints
    tag, hex_id = idf.read_text().split()  # left in place: the communicator never formed
    assert tag == "this-launch" and len(hex_id) == 256 and hex_id != "0" * 256
    # WORLD_SIZE must agree with the cluster
    env = dict(os.environ, WORLD_SIZE="4", RANK="0")
    r = subprocess.run([cli, "run", "--model", m, "--cluster", c, "--batches", "4"], env=env,
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 1 and "num_devices" in r.stderr
