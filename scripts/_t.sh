timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
for i in 1 2; do timeout 200 python scripts/step_variants.py default no_optimizer; done
