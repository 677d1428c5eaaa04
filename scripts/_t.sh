timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python scripts/step_variants.py default no_optimizer
WARMUP=1 timeout 120 python scripts/step_once.py 2> gpurun_out/lps.txt
L=$(awk '{print $2}' gpurun_out/lps.txt)
WARMUP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s $L -c $L --csv --log-file gpurun_out/launches_warm.csv python scripts/step_once.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_warm.csv | grep -i "layernorm\|total"
