#!/bin/bash
# bench step time under executor knobs (one line per setting)
for cfg in "GX_OPT_BLOCKS=0" "GX_OPT_BLOCKS=32" "GX_OPT_BLOCKS=64" "GX_OPT_BLOCKS=148" "GX_SPLITK=0 GX_OPT_BLOCKS=64" "GX_PDL=0 GX_OPT_BLOCKS=64"; do
  r=$(env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])" 2>&1)
  echo "$cfg -> $r"
done
