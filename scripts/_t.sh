timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -1
timeout 200 python scripts/attn_trace.py
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do timeout 200 python scripts/step_variants.py default no_optimizer; done
