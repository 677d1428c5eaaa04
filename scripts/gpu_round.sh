#!/bin/bash
# One GPU evidence pass: smoke, the GPU test suite, the bench line, a warm one-step launch
# list under ncu (serialised), and graph-timed per-kernel numbers at M = 512 / 2048.
# Usage (on the box): bash scripts/gpu_round.sh [tests|bench|all]
what=${1:-all}
mkdir -p gpurun_out
if [ "$what" = all ] || [ "$what" = tests ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
  timeout 2400 python -m pytest tests -m gpu -q -s -rf -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"
  tail -5 gpurun_out/gputest.log
fi
if [ "$what" = all ] || [ "$what" = bench ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 600 gpurun_out/bench.err
  WARMUP=2 timeout 120 python scripts/step_once.py 2> gpurun_out/lps.txt
  L=$(grep launches_per_step gpurun_out/lps.txt | awk '{print $2}')
  WARMUP=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    -s $((2 * L)) -c $L --csv --log-file gpurun_out/launches_warm.csv python scripts/step_once.py > /dev/null 2>&1
  python scripts/summarize_launches.py gpurun_out/launches_warm.csv > gpurun_out/launch_summary.txt
  head -30 gpurun_out/launch_summary.txt
  timeout 300 python scripts/layer_kernels.py 512 > gpurun_out/kernels_m512.jsonl 2>&1
  timeout 300 python scripts/layer_kernels.py 2048 > gpurun_out/kernels_m2048.jsonl 2>&1
fi
