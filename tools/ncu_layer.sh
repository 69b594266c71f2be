# one full-set ncu capture of each kernel of one mid-stack layer (batch-32 FULLY_QUANT)
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attention_kernel" -s 5 -c 5 \
    -o gpurun_out/prof_layer python tools/profile_kernels.py --batch 32 --plans FULLY_QUANT:12 --iters 1 > gpurun_out/ncu_layer.log 2>&1
tail -1 gpurun_out/ncu_layer.log
