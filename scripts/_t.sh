timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -2
timeout 200 python scripts/gemm_trace.py
timeout 200 python scripts/step_variants.py default no_optimizer
