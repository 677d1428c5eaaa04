#!/bin/bash
# Round-2 evidence pass (on the GPU box): bench line, the ncu launch list of a short bench
# command, one warm step's launch list, ncu --set full captures of the top kernels, and the
# graph-timed per-kernel numbers at M = 512 / 2048.  Outputs under gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O/ncu
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-proxy \
  --no-cpu-baseline > $O/bench_under_ncu.json 2>&1; echo "ncu bench rc=$?"
python scripts/summarize_launches.py $O/bench_launches.csv > $O/bench_launch_summary.txt
WARMUP=2 timeout 120 python scripts/step_once.py 2> $O/lps.txt
L=$(grep launches_per_step $O/lps.txt | awk '{print $2}')
WARMUP=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  -s $((2 * L)) -c $L --csv --log-file $O/step_launches_warm.csv python scripts/step_once.py > /dev/null 2>&1
python scripts/summarize_launches.py $O/step_launches_warm.csv > $O/step_launch_summary.txt
for k in qkv_fwd "up_fwd(bias+gelu)" "dgrad_down(gelu_bwd)" "wgrad_up dW1" "out_fwd(bias+drop+res)"; do
  f=$(echo "$k" | tr -c 'a-zA-Z0-9_\n' '_')
  ONLY="$k" timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -c 1 \
    -o $O/ncu/$f python scripts/layer_kernels.py 512 > /dev/null 2>&1
  python scripts/ncu_metrics.py $O/ncu/$f.ncu-rep "$k" >> $O/ncu_full_kernels.jsonl
done
for k in attn_fwd attn_bwd; do
  ONLY=$k timeout 300 ncu --set full --import-source on --clock-control none -k regex:${k}_tc -c 1 \
    -o $O/ncu/$k python scripts/layer_kernels.py 512 > /dev/null 2>&1
  python scripts/ncu_metrics.py $O/ncu/$k.ncu-rep $k >> $O/ncu_full_kernels.jsonl
done
timeout 300 python scripts/layer_kernels.py 512 > $O/kernels_m512.jsonl 2>&1
timeout 300 python scripts/layer_kernels.py 2048 > $O/kernels_m2048.jsonl 2>&1
timeout 200 python scripts/attn_bench.py > $O/attn_bench.jsonl 2>&1
ls $O $O/ncu
# gpurun copies back at most 64 MiB: keep the summaries, compress the launch lists
rm -rf $O/ncu
gzip -f $O/*.csv
du -sh $O
