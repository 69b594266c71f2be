# full ncu captures of one launch of each hot kernel in the batch-32 FULLY_QUANT forward
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attention|embed|pooler" -s 70 -c 8 \
    -o gpurun_out/prof_b32 python tools/profile_kernels.py --batch 32 --plans FULLY_QUANT:12 --iters 1 > gpurun_out/ncu_b32.log 2>&1
tail -2 gpurun_out/ncu_b32.log
