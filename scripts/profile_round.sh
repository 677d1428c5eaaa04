#!/bin/bash
# Round evidence: bench line, one-step ncu launch list (warm caches, serialised), and
# ncu --set full captures of the top GEMM and the tcgen05 attention kernels.
mkdir -p gpurun_out/ncu
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
WARMUP=1 timeout 120 python scripts/step_once.py 2> gpurun_out/lps.txt
L=$(awk '{print $2}' gpurun_out/lps.txt)
WARMUP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  -s $L -c $L --csv --log-file gpurun_out/launches_warm.csv python scripts/step_once.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_warm.csv > gpurun_out/launch_summary.txt
for k in qkv_fwd up_fwd dgrad_down wgrad_up; do
  ONLY=$k timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -c 1 \
    -o gpurun_out/ncu/$k python scripts/layer_kernels.py 512 > /dev/null 2>&1
done
for k in attn_fwd attn_bwd; do
  ONLY=$k timeout 300 ncu --set full --import-source on --clock-control none -k regex:${k}_tc -c 1 \
    -o gpurun_out/ncu/$k python scripts/layer_kernels.py 512 > /dev/null 2>&1
done
ls gpurun_out/ncu
