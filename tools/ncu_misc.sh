ncu --set full --clock-control none --import-source on -k regex:"embed|pooler|classifier|attention" -s 0 -c 6 \
    -o gpurun_out/prof_misc python tools/profile_kernels.py --batch 32 --plans FULLY_QUANT:12 --iters 1 > gpurun_out/ncu_misc.log 2>&1
tail -1 gpurun_out/ncu_misc.log
