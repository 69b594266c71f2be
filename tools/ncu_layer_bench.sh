# ncu --set full (+ L2 sector counters) on the 5 encoder kernels of one layer of the bench
# forward (second forward, layer 0): QKV, attention, out-proj+LN, FFN1+GELU, FFN2+LN.
# usage: tools/ncu_layer_bench.sh <tag> [extra bench args]
TAG=${1:-layer}; shift
ncu --set full --clock-control none --import-source on \
    --metrics lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum \
    -k regex:"gemm_kernel|gemm_persistent_kernel|attention_kernel" -s 65 -c 5 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --lat-iters 1 --no-cpu "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
