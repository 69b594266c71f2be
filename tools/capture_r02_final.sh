# End-of-round-2 ncu evidence (kernels changed late in the round): C2 one layer (fused
# QKV+attention, out-proj, FFN1, FFN2), C4 FFN1 (shared-table persistent layout) and the
# bench launch list (gpu__time_duration per launch).  Demangled-name filters.
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$NCU -k regex:"qkv_attention_kernel|gemm_kernel|gemm_persistent_kernel" -s 52 -c 4 -o gpurun_out/prof_r02f_c2 \
    python tools/profile_forward.py --workload c2 --iters 2 > gpurun_out/ncu_r02f_c2.log 2>&1
$NCU -k regex:"gemm_persistent_kernel<\(int\)0, \(int\)128, \(int\)3, \(int\)8, samp::EpiGeluQuantT" -s 30 -c 1 -o gpurun_out/prof_r02f_c4ffn1 \
    python tools/profile_forward.py --workload c4 --iters 2 > gpurun_out/ncu_r02f_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02f.csv \
    python bench.py --steps 2 --warmup 1 --lat-iters 1 --no-cpu > gpurun_out/launches_r02f.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02f_c2.ncu-rep > gpurun_out/ncu_r02f_c2.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02f_c4ffn1.ncu-rep > gpurun_out/ncu_r02f_c4ffn1.txt 2>&1
