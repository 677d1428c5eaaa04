mkdir -p gpurun_out/ncu
ONLY=ln_bwd timeout 300 ncu --set full --import-source on --clock-control none -k regex:layernorm_bwd -c 2 -o gpurun_out/ncu/ln_bwd python scripts/layer_kernels.py 512 > gpurun_out/ncu/ln_bwd.log 2>&1
ONLY=up_fwd timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -c 1 -o gpurun_out/ncu/up_fwd python scripts/layer_kernels.py 512 > gpurun_out/ncu/up_fwd.log 2>&1
ONLY=attn_fwd timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn -c 1 -o gpurun_out/ncu/attn_fwd python scripts/layer_kernels.py 512 > gpurun_out/ncu/attn_fwd.log 2>&1
ls -la gpurun_out/ncu
