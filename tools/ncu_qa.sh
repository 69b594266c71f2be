# ncu --set full on one fused QKV+attention launch of the bench forward (layer 0 of the 2nd forward)
TAG=${1:-qa}; shift
ncu --set full --clock-control none --import-source on -k regex:"qkv_attention_kernel" -s 12 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --lat-iters 1 --no-cpu "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
