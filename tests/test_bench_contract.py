"""bench.py's reference arm (CPU) keeps the driver's JSON-line contract: one line, the
metric / unit / direction of the gx arm, an e2e object and a cpu_baseline describing the run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert d["config"]["model"] == "bert-huge-32"
    assert d["ms_per_step"] * d["steps"] / 1e3 <= 600  # the process's own time: fits its run
    # the reference process maps only oracle/ libraries (the reference planner, the CPU port)
    assert "reference_planner_optimize_ms" in d and "gx_planner_optimize_ms" not in d
    assert set(d["reference_planner_optimize_ms"]) >= {"config2-bert-huge-32/n8/8gib",
                                                        "config5-swin-like/n8/16gib"}


def test_multi_gpu_launch_fails_loudly_without_gpus():
    """--gpus 2 outside a launcher re-launches under torchrun only when 2 GPUs are visible;
    here there are none, so it must refuse instead of silently running N = 1."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "GPU(s) visible" in r.stderr


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
