# Evidence for profiles/: (1) the per-launch device-time list of the bench command,
# (2) one ncu --set full capture of each hot kernel: launches 61..68 of the run are the
# first forward's pooler + classifier and the second forward's embed, QKV, attention,
# out-proj(+LN), FFN1(+GELU), FFN2(+LN) (63 launches per BERT-base forward).
set -e
mkdir -p gpurun_out
K='regex:gemm_kernel|gemm_persistent_kernel|attention_kernel|embed_kernel|pooler_kernel|classifier_kernel'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" \
    -c 400 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k "$K" \
    -s 61 -c 8 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --lat-iters 1 --no-cpu > gpurun_out/ncu_full.log 2>&1
echo done
