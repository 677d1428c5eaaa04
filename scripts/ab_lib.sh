#!/bin/bash
# A/B of two builds of libgx.so on one box: the tree's build (B) against libgx_base.so (A),
# per-kernel times at M = 512 and the bench step, alternating A / B twice.
# Usage (on the box): bash scripts/ab_lib.sh  -> gpurun_out/ab/
set -u
O=gpurun_out/ab; mkdir -p $O
L=paper_2211_13878_b200/libgx.so
cp $L $O/../libgx_new.so
for v in new base new base; do
  if [ $v = base ]; then cp libgx_base.so $L; else cp $O/../libgx_new.so $L; fi
  timeout 300 python scripts/layer_kernels.py 512 > $O/k_$v.jsonl 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-proxy --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['ms_per_step'])" >> $O/steps.txt
done
cp $O/../libgx_new.so $L
cat $O/steps.txt
python - <<'PY'
import json
a={json.loads(l)["kernel"]:json.loads(l)["us"] for l in open("gpurun_out/ab/k_base.jsonl") if '"kernel"' in l}
b={json.loads(l)["kernel"]:json.loads(l)["us"] for l in open("gpurun_out/ab/k_new.jsonl") if '"kernel"' in l}
for k in a: print(f"{k:28s} base {a[k]:8.2f}  new {b.get(k, float('nan')):8.2f}")
PY
