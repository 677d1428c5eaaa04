#!/bin/bash
# Launch list (device time per kernel, cold-cache, serialised) of 2 bench steps after warm-up.
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    -s 1750 -c 805 python bench.py --steps 2 --warmup 2 --no-graph --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1 || true
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt
