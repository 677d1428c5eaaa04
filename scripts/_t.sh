GX_OPT_SMS=16 timeout 300 python -m pytest tests/test_executor_gpu.py -x -q -k "optimizer or deferred" 2>&1 | tail -1
for n in 8 16 24 32 48; do GX_OPT_SMS=$n timeout 120 python scripts/step_variants.py default | sed "s/^/sms$n /"; done
timeout 120 python scripts/step_variants.py default
