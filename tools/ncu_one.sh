# ncu --set full on one launch of kernels matching $1 in the batch-32 FULLY_QUANT forward
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1" -s ${2:-2} -c 1 \
    -o gpurun_out/prof_$3 python tools/profile_kernels.py --batch 32 --plans FULLY_QUANT:12 --iters 1 > gpurun_out/ncu_$3.log 2>&1
tail -1 gpurun_out/ncu_$3.log
