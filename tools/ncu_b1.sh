# launch list + full captures for the batch-1 FULLY_QUANT forward
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -s 120 -c 140 --csv --log-file gpurun_out/b1_launches.csv \
    python tools/profile_kernels.py --batch 1 --plans FULLY_QUANT:12 --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|embed|classify|attention" -s 200 -c 6 \
    -o gpurun_out/prof_b1 python tools/profile_kernels.py --batch 1 --plans FULLY_QUANT:12 --iters 2 > gpurun_out/ncu_b1.log 2>&1
tail -3 gpurun_out/ncu_b1.log
