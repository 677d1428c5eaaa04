timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/layer_kernels.py 512 2>&1 | grep -vE "attn|ln_|adamw|dropout"
timeout 200 python scripts/step_variants.py default no_optimizer no_splitk
