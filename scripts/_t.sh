timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
timeout 300 python scripts/layer_kernels.py 512 2>&1 | grep -E "attn"
timeout 200 python scripts/step_variants.py default no_optimizer
