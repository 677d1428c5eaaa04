timeout 600 python -m pytest tests/test_executor_gpu.py -x -q 2>&1 | tail -2
for g in 1 2 4 8; do GX_OPT_GROUP=$g timeout 200 python scripts/step_variants.py default | sed "s/^/group$g /"; done
