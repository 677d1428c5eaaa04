#!/usr/bin/env python
"""bench.py — samples/s of one Galvatron-plan training step on B200.

Workload (BASELINE.json configs[1]): BERT-Huge-32 (h 1280, s 512, 20 heads x 64, ffn 5120,
32 layers) under the plan the search picks for N GPUs and a per-GPU budget (default
16 GiB), with the reference's cluster inputs (island = N, 13 GB/s,
configs/clusters/single-node-8gpu.json) and default profile.  Batch candidates are the
reference's DefaultBatchCandidates (8..512 step 8); when the reference search reports OOM
for them (N=1, N=2) the list 1..512 is used, as BASELINE.md §4.3 prescribes.  At N=1 / 16 GiB
that plan is [serial] x32 with B=1.

One step = forward + MSE loss + backward + gradient synchronisation + AdamW over every
layer, replayed as one CUDA graph.  `value` = B / step time (inputs resident in HBM);
`e2e` = the same through gx_exec_step with pinned host inputs copied in and the loss read
back every step.  Working set per step (params + grads + optimizer state) is ~10 GB per GPU
at N=1, far above the 126 MB L2, so no explicit L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--budget-gib 16] [--impl gx|reference]
Under torchrun (N>1) every rank runs one executor over NCCL; rank 0 prints the JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (8xB200, per memory budget) + tensor-pipe % of peak vs CPU ref"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
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


def choose_plan(n_gpus: int, budget_gib: float, model_name: str):
    from paper_2211_13878_b200 import models, planner
    m = models.model(model_name)
    c = models.cluster(n_gpus, budget_gib, 13.0)
    out = planner.api().optimize(m, c)
    batches = "8..512 step 8 (DefaultBatchCandidates)"
    if out.plan is None:
        out = planner.api().optimize(m, c, None, list(range(1, 513)))
        batches = "1..512 (reference search OOM at 8..512)"
    if out.plan is None:
        raise SystemExit(f"no feasible plan: {out.diagnostic}")
    return m, out.plan, batches


def cpu_layer_sample(model_name: str, reps: int, p_drop: float):
    """Times the CPU port of one layer fwd+bwd at one sample (numpy fp32, all host cores)."""
    import numpy as np
    from oracle import layer_oracle as lo
    from paper_2211_13878_b200 import models
    sh = models.model(model_name)["layers"][0]["shape"]
    shape = lo.LayerShape(sh["hidden"], sh["heads"], sh["seq"], sh["ffn"])
    rng = np.random.default_rng(0)
    P = {k: v.astype(np.float32) for k, v in lo.init_layer_params(shape, rng).items()}
    x = rng.standard_normal((shape.seq, shape.hidden)).astype(np.float32)
    dy = rng.standard_normal((shape.seq, shape.hidden)).astype(np.float32)
    drop = lo.Dropout(p_drop, p_drop, 1234)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        y, cache = lo.layer_forward(P, x, shape, 0, drop)
        lo.layer_backward(P, dy, cache, shape)
        times.append(time.perf_counter() - t0)
    return times, shape


def run_reference(args, rank):
    """--impl reference: the reference path's CPU implementation on the host cores.

    The reference (arxiv/paper_2211_13878, proj/) is a planner with no executor, so its
    CPU 'path' for samples/s is this repo's CPU port of the layer math (oracle/, kind
    "port"); the reference planner's own Optimize time on the same config is reported
    alongside when oracle/_ref is built."""
    if rank != 0:
        return
    n_layers = 32
    cores = os.cpu_count()
    t_all = []
    for _ in range(args.warmup):
        cpu_layer_sample(args.model, 1, args.dropout)
    for _ in range(args.steps):
        times, _ = cpu_layer_sample(args.model, 1, args.dropout)
        t_all.extend(times)
    t_layer = statistics.median(t_all)
    value = 1.0 / (n_layers * t_layer)
    extra = {}
    try:
        from oracle import ref_planner
        from paper_2211_13878_b200 import models
        if ref_planner.available():
            from paper_2211_13878_b200 import planner as gx_planner
            m = models.model(args.model)
            c = models.cluster(args.gpus, args.budget_gib, 13.0)
            o = ref_planner.api().optimize(m, c)
            batches = None
            if o.plan is None:
                batches = list(range(1, 513))
                o = ref_planner.api().optimize(m, c, None, batches)
            extra["reference_plan_predicted_samples_per_s"] = o.plan["throughput_samples_per_s"] if o.plan else None

            def med7(api, threads):  # median of 7, PLANNER_THREADS = 1 and = nproc
                ts = []
                for _ in range(7):
                    t0 = time.perf_counter()
                    api.optimize(m, c, None, batches, num_threads=threads)
                    ts.append((time.perf_counter() - t0) * 1e3)
                return round(statistics.median(ts), 3)
            extra["reference_planner_optimize_ms"] = {"threads_1": med7(ref_planner.api(), 1),
                                                      f"threads_{cores}": med7(ref_planner.api(), cores)}
            extra["gx_planner_optimize_ms"] = {"threads_1": med7(gx_planner.api(), 1),
                                               f"threads_{cores}": med7(gx_planner.api(), cores)}
    except Exception as e:  # the planner timing is informational only
        extra["reference_planner_error"] = str(e)[:200]
    sample = (f"1 {args.model} layer fwd+bwd at 1 sample (numpy fp32, dropout {args.dropout}) per step, "
              f"extrapolated x{n_layers} layers; median of {len(t_all)}")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_layer * n_layers * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.model} fwd+bwd, CPU port", "model": args.model,
                       "budget_gib": args.budget_gib},
            "cpu_baseline": {"value": round(value, 6), "unit": "samples/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 6), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    line.update(extra)
    print(json.dumps(line), flush=True)


def run_gx(args, rank, world, local_rank):
    import numpy as np
    import torch
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2211_13878_b200 import executor as gxe

    nccl_id = ""
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        obj = [gxe.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    model, plan, batches = choose_plan(world, args.budget_gib, args.model)
    ex = gxe.PlanExecutor(plan, model, world, local_ranks=[rank],
                          comm="nccl" if world > 1 else "sim", nccl_id_hex=nccl_id,
                          dropout_attn=args.dropout, dropout_hidden=args.dropout, seed=1234,
                          lr=1e-4)
    ex.init_params(seed=7, std=0.02)
    B = plan["batch_size"]
    sh = model["layers"][0]["shape"]
    rows, h = B * sh["seq"], sh["hidden"]
    g = torch.Generator().manual_seed(0)
    x_host = torch.randn(rows, h, generator=g).to(torch.bfloat16).pin_memory()
    t_host = torch.randn(rows, h, generator=g).to(torch.bfloat16).pin_memory()
    ex.load_batch(x_host.view(torch.int16), t_host.view(torch.int16))
    stream = torch.cuda.ExternalStream(ex.stream, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    use_graph = not args.no_graph
    for _ in range(args.warmup):
        ex.run(use_graph)
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            ex.run(use_graph)
        end.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(start.elapsed_time(end) / args.steps)
    loss = ex.loss()
    info = ex.info()
    launches = int(info["launches_per_step"]) * args.steps

    # end to end: host batch in, loss out, every step, through the public C ABI call
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ex.step(x_host.view(torch.int16), t_host.view(torch.int16), use_graph)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    r0 = info["ranks"][0]
    stage0 = r0["stage"] == 0
    last = r0["stage"] == plan["pp_degree"] - 1
    my_rows = rows // max(1, world // plan["pp_degree"])  # approx. when data-split is uneven
    h2d = (my_rows * h * 2 if stage0 else 0) + (my_rows * h * 2 if last else 0)

    # per-launch device timing of the same kernels (instrumented graph replay)
    for _ in range(2):
        ex.run(use_graph, profile=True)
    prof = ex.profile_report()
    gemm = prof["categories"]["gemm"]
    gemm_tflops = gemm["flops"] / (gemm["ms"] * 1e-3) / 1e12 if gemm["ms"] > 0 else 0.0
    peaks, peak_src = _peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        traffic_note = (f"ncu dram bytes of one {tj.get('kernel')} launch; algorithmic "
                        f"{tj.get('algorithmic_bytes_per_launch')} B")
    cats = {k: round(v["ms"], 4) for k, v in prof["categories"].items()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times, _ = cpu_layer_sample(args.model, 3, args.dropout)
        t_layer = statistics.median(times)
        cpu = {"value": round(1.0 / (len(model["layers"]) * t_layer), 6), "unit": "samples/s",
               "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 layer fwd+bwd at 1 sample (numpy fp32, dropout {args.dropout}), "
                         f"median of 3, extrapolated x{len(model['layers'])} layers"}

    if rank == 0:
        from paper_2211_13878_b200 import planner
        line = {
            "metric": METRIC, "value": round(B / (ms / 1e3), 4), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.model} train step (fwd+bwd+AdamW) under the searched plan",
                       "model": args.model, "global_batch": B, "seq_len": sh["seq"],
                       "hidden": h, "layers": len(model["layers"]),
                       "budget_gib": args.budget_gib, "batches": batches,
                       "plan": planner.ribbon(plan), "pp_degree": plan["pp_degree"],
                       "micro_batches": plan["micro_batches"],
                       "parallelism": f"plan:{planner.ribbon(plan)}",
                       "dropout": args.dropout, "cuda_graph": use_graph,
                       "l2": "working set > L2 (params+grads+Adam state ~10 GB/GPU); no flush"},
            "e2e": {"value": round(B / (e2e_ms / 1e3), 4), "unit": "samples/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4},
            "roofline": {"bound": "tensor", "achieved": round(gemm_tflops, 2), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(gemm_tflops / peak, 4),
                         "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": "gemm_pair_kernel / gemm_tcgen05_kernel (all layer GEMMs)",
                         "peak_source": f"{peak_src} bf16_tflops_sustained",
                         "gemm_launches_per_step": gemm["launches"],
                         "gemm_ms_per_step": round(gemm["ms"], 4),
                         "gemm_share_of_step": round(gemm["ms"] / ms, 4) if ms else None},
            "step_breakdown_ms": cats,
            "loss": loss,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "memory": {"device_bytes_rank0": info["ranks"][0]["device_bytes"],
                       "plan_estimate_bytes_rank0": info["ranks"][0].get("plan_estimate_bytes"),
                       "budget_bytes": int(args.budget_gib * (1 << 30))},
        }
        print(json.dumps(line), flush=True)
    ex.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


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
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_gx(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
