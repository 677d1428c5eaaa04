timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2 3; do timeout 300 python -m pytest tests/test_profiler_gpu.py -x -q -k nccl_world 2>&1 | tail -1; done
timeout 200 python scripts/step_variants.py default no_optimizer
