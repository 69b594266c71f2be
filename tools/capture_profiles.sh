# Evidence for profiles/: (1) the per-launch device-time list of the bench command,
# (2) one ncu --set full capture of each hot kernel (one mid-stack layer).
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|attention_kernel|embed_kernel|pooler_kernel|classifier_kernel" \
    -c 400 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attention_kernel|embed_kernel|pooler_kernel|classifier_kernel" \
    -s 62 -c 7 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --lat-iters 1 --no-cpu > gpurun_out/ncu_full.log 2>&1
echo done
