timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python scripts/step_variants.py default no_optimizer
