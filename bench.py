#!/usr/bin/env python
"""bench.py — samples/s of one Galvatron-plan training step on B200.

Workload (BASELINE.json configs[1]): BERT-Huge-32 (h 1280, s 512, 20 heads x 64, ffn 5120,
32 layers) under the plan the search picks for N GPUs and a per-GPU memory budget, with the
reference's cluster inputs (island = N, 13 GB/s, configs/clusters/single-node-8gpu.json) and
default profile.  Batch candidates are the reference's DefaultBatchCandidates (8..512 step
8); where the reference search reports OOM for them, 1..512, and where it
is still OOM the budget is reported as OOM.  The headline is the --budget-gib budget
(default 16 GiB; at N = 1 that plan is [serial] x32 with B = 1); the other budget of the
metric's pair (8 / 16 GiB) is measured and reported under "budgets".

One step = forward + MSE loss + backward + gradient synchronisation + AdamW over every layer,
replayed as one CUDA graph, with the per-rank device arena capped at the budget
(memory_cap_bytes, E15).  `value` = B / step time (inputs resident in HBM); `e2e` = the same
through gx_exec_step with pinned host inputs copied in and the loss read back every step.
The working set per step (params + grads + optimizer state, ~10 GB per GPU at N = 1) is far
above the 126 MB L2, so no explicit L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--budget-gib 16] [--impl gx|reference]

--gpus N > 1 without WORLD_SIZE in the environment re-launches itself under torchrun with N
ranks (one per GPU, NCCL); fewer visible GPUs than N is an error.  Rank 0 prints the line.
--impl reference times the reference path's CPU implementation: the
reference is a planner only, so its samples/s leg is the repo's fp32 C + OpenMP restatement
of the layer step (oracle/cpu_layer.c, kind "port"), plus the reference planner's own
Optimize (oracle/_ref, built from the reference sources) on every BASELINE config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (8xB200, per memory budget) + tensor-pipe % of peak vs CPU ref"
BUDGETS = (8.0, 16.0)
NVLINK_GBS = 900.0  # NVLink 5 per GPU per direction
# BASELINE configs whose search time is the reference CPU path:
# (name, model, N, batches or None = DefaultBatchCandidates)
PLANNER_CONFIGS = (("config1-bert-base-2", "bert-base-2", 8, [8]),
                   ("config2-bert-huge-32", "bert-huge-32", 8, None),
                   ("config3-vit-huge-32", "vit-huge-32", 8, None),
                   ("config4-t5-large-48", "t5-large-48", 8, None),
                   ("config5-swin-like", "swin-like", 8, None))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    # B200_PROFILING.md fallback figures
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                self.samples.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------ plans
def search(api, model_name: str, n_gpus: int, budget_gib: float, batches=None):
    """The plan the reference search picks (api: this repo's planner or oracle/_ref's).
    Returns (model, plan or None, batch list description)."""
    from paper_2211_13878_b200 import models
    m = models.model(model_name)
    c = models.cluster(n_gpus, budget_gib, 13.0)
    if batches is not None:
        out = api.optimize(m, c, None, batches)
        return m, out.plan, f"{batches}"
    out = api.optimize(m, c)
    if out.plan is not None:
        return m, out.plan, "8..512 step 8 (DefaultBatchCandidates)"
    out = api.optimize(m, c, None, list(range(1, 513)))
    if out.plan is not None:
        return m, out.plan, "1..512 (reference search OOM at 8..512)"
    return m, None, "OOM at 8..512 and 1..512 (reference search)"


def planner_timings(api, cores: int) -> dict:
    """Optimize wall time (median of 7) at PLANNER_THREADS = 1 and = nproc for every
    BASELINE config and both budgets."""
    from paper_2211_13878_b200 import models
    out = {}
    for name, model_name, n, batches in PLANNER_CONFIGS:
        m = models.model(model_name)
        for budget in BUDGETS:
            c = models.cluster(n, budget, 13.0)
            row = {}
            for threads in (1, cores):
                ts = []
                for _ in range(7):
                    t0 = time.perf_counter()
                    api.optimize(m, c, None, batches, num_threads=threads)
                    ts.append((time.perf_counter() - t0) * 1e3)
                row[f"threads_{threads}"] = round(statistics.median(ts), 3)
            out[f"{name}/n{n}/{int(budget)}gib"] = row
    return out


# ------------------------------------------------------------------------ CPU baseline
def cpu_step_sample(model_name: str, p_drop: float, warmup: int, reps: int):
    """One sample through the model's full training step (fwd + bwd + AdamW over every
    layer) on the host cores: oracle/cpu_layer.c, fp32, OpenMP.  Returns (seconds per step
    list, threads, description)."""
    import numpy as np
    from oracle import cpu_layer
    from paper_2211_13878_b200 import models
    m = models.model(model_name)
    sh = m["layers"][0]["shape"]
    L = len(m["layers"])
    cm = cpu_layer.CpuModel(L, 1, sh["seq"], sh["hidden"], sh["heads"], sh["ffn"], p_drop,
                            p_drop, 1234)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((sh["seq"], sh["hidden"])).astype(np.float32)
    t = rng.standard_normal((sh["seq"], sh["hidden"])).astype(np.float32)
    for _ in range(warmup):
        cm.step(x, t)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        cm.step(x, t)
        ts.append(time.perf_counter() - t0)
    cm.close()
    desc = (f"1 sample through all {L} {model_name} layers: fwd + MSE + bwd + AdamW "
            f"(oracle/cpu_layer.c, fp32 C + OpenMP, dropout {p_drop})")
    return ts, cpu_layer.threads(), desc


def cpu_config1(p_drop: float) -> dict:
    """config 1 (2-layer BERT-base shape, s 128, B 8) fwd+bwd on the host."""
    import numpy as np
    from oracle import cpu_layer
    cm = cpu_layer.CpuModel(2, 8, 128, 768, 12, 3072, p_drop, p_drop, 1234)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((8 * 128, 768)).astype(np.float32)
    cm.step(x, x, optimizer=False)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        cm.step(x, x, optimizer=False)
        ts.append(time.perf_counter() - t0)
    cm.close()
    med = statistics.median(ts)
    return {"ms_fwd_bwd": round(med * 1e3, 3), "samples_per_s": round(8 / med, 3),
            "threads": cpu_layer.threads()}


# ----------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the reference path's CPU implementation on the host cores.  Rank 0
    alone runs; one step = one sample of the gx arm's workload (BERT-Huge-32, all 32 layers,
    fwd + bwd + AdamW) -- a bounded sample of the global batch, so `value` is samples/s of
    exactly this CPU computation and ms_per_step x steps is this process's own time."""
    if rank != 0:
        return
    from oracle import cpu_layer, ref_planner
    cores = os.cpu_count()
    _, plan, batches = search(ref_planner.api(), args.model, world, args.budget_gib) \
        if ref_planner.available() else (None, None, "oracle/_ref not built")
    cpu_layer.lib()  # build / load before the clock starts
    ts, threads, desc = cpu_step_sample(args.model, args.dropout, args.warmup, args.steps)
    total = sum(ts)
    value = args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.model} train step (fwd+bwd+AdamW), 1 sample per step, "
                                   f"host CPU", "model": args.model, "global_batch": 1,
                       "budget_gib": args.budget_gib,
                       "gx_arm_plan_global_batch": plan["batch_size"] if plan else None,
                       "batches": batches},
            "cpu_baseline": {"value": round(value, 6), "unit": "samples/s", "cores": threads,
                             "kind": "port", "sample": desc},
            "e2e": {"value": round(value, 6), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if ref_planner.available():
        # the reference's own CPU path: parplan_ref::Optimize (reference sources, oracle/_ref)
        line["reference_planner_optimize_ms"] = planner_timings(ref_planner.api(), cores)
        line["reference_plan_predicted_samples_per_s"] = plan["throughput_samples_per_s"] if plan else None
    line["cpu_config1_fwd_bwd"] = cpu_config1(args.dropout)
    line["host"] = {"cores": cores, "cpu": _cpu_model()}
    print(json.dumps(line), flush=True)


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- gx arm
def _roofline_rows(prof: dict, peaks: dict, world: int) -> dict:
    """Per-category achieved vs peak from the instrumented replay (algorithmic flops / bytes
    of every launch / its CUDA-event duration)."""
    cats = prof["categories"]
    rows = {}
    for cat, bound in (("gemm", "tensor"), ("attention_fwd", "tensor"), ("attention_bwd", "tensor"),
                       ("layernorm", "hbm"), ("elementwise", "hbm"), ("optimizer", "hbm")):
        c = cats.get(cat)
        if not c or c["ms"] <= 0:
            continue
        if bound == "tensor":
            a, p, u = c["flops"] / (c["ms"] * 1e-3) / 1e12, float(peaks["bf16_tflops"]), "TFLOP/s"
        else:
            a, p, u = c["bytes"] / (c["ms"] * 1e-3) / 1e9, float(peaks["hbm_gbs"]), "GB/s"
        rows[cat] = {"bound": bound, "achieved": round(a, 2), "peak": p, "unit": u,
                     "frac": round(a / p, 4), "ms_per_step": round(c["ms"], 4),
                     "launches_per_step": c["launches"]}
    if world > 1:
        for kind, c in prof.get("comm_kinds", {}).items():
            if c["ms"] > 0:
                bus = c["bus_bytes"] / (c["ms"] * 1e-3) / 1e9
                rows["nccl_" + kind] = {"bound": "nvlink", "achieved": round(bus, 2),
                                        "peak": NVLINK_GBS, "unit": "GB/s (bus)",
                                        "frac": round(bus / NVLINK_GBS, 4),
                                        "ms_per_step": round(c["ms"], 4),
                                        "launches_per_step": c["launches"]}
    return rows


def _measure(ex, stream, world, dev, steps, warmup, use_graph):
    import torch

    def barrier():
        ex.sync()
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(warmup):
        ex.run(use_graph)
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        ex.run(use_graph)
    end.record(stream)
    barrier()
    return start.elapsed_time(end) / steps


def run_gx(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2211_13878_b200 import executor as gxe
    from paper_2211_13878_b200 import planner

    nccl_id = ""
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        obj = [gxe.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peaks, peak_src = _peaks()
    api = planner.api()
    use_graph = not args.no_graph
    budgets = {}
    headline = None
    for budget in sorted(set(BUDGETS) | {args.budget_gib}, key=lambda b: b != args.budget_gib):
        model, plan, batches = search(api, args.model, world, budget)
        if plan is None:
            budgets[f"{budget:g}"] = {"status": "OOM", "batches": batches}
            continue
        ex = gxe.PlanExecutor(plan, model, world, local_ranks=[rank],
                              comm="nccl" if world > 1 else "sim", nccl_id_hex=nccl_id,
                              dropout_attn=args.dropout, dropout_hidden=args.dropout, seed=1234,
                              lr=1e-4, memory_cap_bytes=int(budget * (1 << 30)))
        ex.init_params(seed=7, std=0.02)
        B = plan["batch_size"]
        sh, shl = model["layers"][0]["shape"], model["layers"][-1]["shape"]
        g = torch.Generator().manual_seed(0)
        x_host = torch.randn(B * sh["seq"], sh["hidden"], generator=g).to(torch.bfloat16).pin_memory()
        t_host = torch.randn(B * shl["seq"], shl["hidden"], generator=g).to(torch.bfloat16).pin_memory()
        ex.load_batch(x_host.view(torch.int16), t_host.view(torch.int16))
        stream = torch.cuda.ExternalStream(ex.stream, device=dev)
        is_head = budget == args.budget_gib
        with ClockSampler(local_rank) as clocks:
            ms = max_over_ranks(_measure(ex, stream, world, dev, args.steps, args.warmup, use_graph))
        info = ex.info()
        r0 = info["ranks"][0]
        entry = {"status": "ok", "value": round(B / (ms / 1e3), 4), "ms_per_step": round(ms, 4),
                 "global_batch": B, "plan": planner.ribbon(plan), "pp_degree": plan["pp_degree"],
                 "micro_batches": plan["micro_batches"], "batches": batches,
                 "device_bytes_rank": r0["device_bytes"],
                 "plan_estimate_bytes_rank": r0.get("plan_estimate_bytes"),
                 "memory_cap_bytes": r0.get("memory_cap_bytes")}
        budgets[f"{budget:g}"] = entry
        if is_head:
            loss = ex.loss()
            launches = int(info["launches_per_step"])
            # end to end: host batch in, loss out, every step, through the public C ABI call
            ex.sync()
            torch.cuda.synchronize()
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                ex.step(x_host.view(torch.int16), t_host.view(torch.int16), use_graph)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
            stage0 = r0["stage"] == 0
            last = r0["stage"] == plan["pp_degree"] - 1
            h2d = (r0.get("input_rows", 0) * sh["hidden"] * 2 if stage0 else 0) + \
                  (r0.get("target_rows", 0) * shl["hidden"] * 2 if last else 0)
            # per-launch device timing of the same kernels (instrumented graph replay)
            for _ in range(2):
                ex.run(use_graph, profile=True)
            prof = ex.profile_report()
            headline = dict(ms=ms, e2e_ms=e2e_ms, B=B, plan=plan, batches=batches, loss=loss,
                            launches=launches, clocks=clocks.summary(), h2d=h2d, prof=prof,
                            sh=sh, model=model, info=info)
        ex.close()

    if headline is None:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "samples/s",
                              "n_gpus": world, "error": "no feasible plan at the headline budget",
                              "budgets": budgets}), flush=True)
        return

    # per-GPU proxy of the 8-GPU plans (rank 0 alone, N = 1 runs only): one rank's share of
    # the N = 8 plan with no-op collectives -- the GEMM shapes an 8-GPU run sees.  Reported
    # separately, never as the headline.
    proxy = None
    if world == 1 and not args.no_proxy:
        proxy = {}
        for budget in BUDGETS:
            model, plan, batches = search(api, args.model, 8, budget)
            if plan is None:
                continue
            ex = gxe.PlanExecutor(plan, model, 8, local_ranks=[0], comm="null",
                                  dropout_attn=args.dropout, dropout_hidden=args.dropout,
                                  seed=1234, lr=1e-4, memory_cap_bytes=int(budget * (1 << 30)))
            ex.init_params(seed=7, std=0.02)
            B = plan["batch_size"]
            sh = model["layers"][0]["shape"]
            xh = torch.zeros(B * sh["seq"], sh["hidden"], dtype=torch.int16)
            ex.load_batch(xh, xh)
            stream = torch.cuda.ExternalStream(ex.stream, device=dev)
            pms = _measure(ex, stream, 1, dev, args.steps, args.warmup, use_graph)
            for _ in range(2):
                ex.run(use_graph, profile=True)
            pp = ex.profile_report()
            gm = pp["categories"]["gemm"]
            gt = gm["flops"] / (gm["ms"] * 1e-3) / 1e12 if gm["ms"] > 0 else 0.0
            proxy[f"{budget:g}"] = {
                "plan": planner.ribbon(plan), "global_batch": B,
                "rank0_rows": ex.info()["ranks"][0].get("input_rows"),
                "ms_per_step_rank0_compute": round(pms, 4),
                "projected_samples_per_s_8gpu_if_comm_hidden": round(B / (pms / 1e3), 3),
                "gemm_tflops": round(gt, 2), "gemm_frac_of_burst": round(gt / float(peaks["bf16_tflops"]), 4),
                "kernels": _roofline_rows(pp, peaks, 1)}
            ex.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ts, threads, desc = cpu_step_sample(args.model, args.dropout, 1, 2)
        cpu = {"value": round(1.0 / statistics.median(ts), 6), "unit": "samples/s",
               "cores": threads, "kind": "port", "sample": desc + ", median of 2 after 1 warm-up"}

    if rank != 0:
        return
    H = headline
    prof = H["prof"]
    rows = _roofline_rows(prof, peaks, world)
    gemm = rows.get("gemm", {"achieved": 0.0, "peak": float(peaks["bf16_tflops"]), "frac": 0.0})
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        traffic_note = (f"ncu dram bytes of one {tj.get('kernel')} launch; algorithmic "
                        f"{tj.get('algorithmic_bytes_per_launch')} B")
    B, ms, sh = H["B"], H["ms"], H["sh"]
    line = {
        "metric": METRIC, "value": round(B / (ms / 1e3), 4), "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{args.model} train step (fwd+bwd+AdamW) under the searched plan",
                   "model": args.model, "global_batch": B, "seq_len": sh["seq"],
                   "hidden": sh["hidden"], "layers": len(H["model"]["layers"]),
                   "budget_gib": args.budget_gib, "batches": H["batches"],
                   "plan": planner.ribbon(H["plan"]), "pp_degree": H["plan"]["pp_degree"],
                   "micro_batches": H["plan"]["micro_batches"],
                   "parallelism": f"plan:{planner.ribbon(H['plan'])}",
                   "dropout": args.dropout, "cuda_graph": use_graph,
                   "memory_cap_bytes": int(args.budget_gib * (1 << 30)),
                   "l2": "working set > L2 (params+grads+Adam state ~10 GB/GPU); no flush"},
        "e2e": {"value": round(B / (H["e2e_ms"] / 1e3), 4), "unit": "samples/s",
                "h2d_bytes_per_step": int(H["h2d"]), "d2h_bytes_per_step": 4},
        "roofline": {"bound": "tensor", "achieved": gemm["achieved"], "peak": gemm["peak"],
                     "unit": "TFLOP/s", "frac": gemm["frac"], "traffic": traffic,
                     "traffic_note": traffic_note,
                     "kernel": "gemm_pair_kernel / gemm_tcgen05_kernel (all layer GEMMs)",
                     "peak_source": f"{peak_src} bf16_tflops (burst: kernels timed per launch)",
                     "gemm_launches_per_step": prof["categories"]["gemm"]["launches"],
                     "gemm_ms_per_step": round(prof["categories"]["gemm"]["ms"], 4),
                     "gemm_share_of_step": round(prof["categories"]["gemm"]["ms"] / ms, 4)},
        "kernels": rows,
        "step_breakdown_ms": {k: round(v["ms"], 4) for k, v in prof["categories"].items()},
        "budgets": budgets,
        "loss": H["loss"],
        "gpu_launches": H["launches"] * args.steps,
        "gpu_launches_per_step": H["launches"],
        "clocks": H["clocks"],
        "cpu_baseline": cpu,
        "memory": {"device_bytes_rank0": H["info"]["ranks"][0]["device_bytes"],
                   "plan_estimate_bytes_rank0": H["info"]["ranks"][0].get("plan_estimate_bytes"),
                   "budget_bytes": int(args.budget_gib * (1 << 30))},
    }
    if proxy is not None:
        line["proxy_n8_rank0"] = proxy
    line["gx_planner_optimize_ms"] = planner_timings(api, os.cpu_count())
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gx", "reference"], default="gx")
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--model", default="bert-huge-32")
    ap.add_argument("--dropout", type=float, default=0.1)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-proxy", action="store_true")
    args = ap.parse_args()
    if args.impl == "gx" and args.warmup < 3:
        raise SystemExit("bench.py: --warmup must be >= 3")
    in_launcher = "WORLD_SIZE" in os.environ
    if not in_launcher and args.gpus > 1:
        if args.impl == "reference":  # rank 0 alone runs the CPU reference: no GPUs needed
            run_reference(args, 0, args.gpus)
            return
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_gx(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
