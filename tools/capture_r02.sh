# Round-2 ncu evidence: one --set full capture of each hot kernel of the configurations
# BASELINE.json names (C1 FP16 batch 1, C2 fused INT8, C4 BERT-large attention, C5 FP16 MHA
# + INT8 FFN), all with source correlation.  Kernel filters match demangled names.
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
# C2: one layer of the second forward (4 kernels per layer: fused QKV+attention, out-proj, FFN1, FFN2)
$NCU -k regex:"qkv_attention_kernel|gemm_kernel|gemm_persistent_kernel" -s 52 -c 4 -o gpurun_out/prof_r02_c2 \
    python tools/profile_forward.py --workload c2 --iters 2 > gpurun_out/ncu_r02_c2.log 2>&1
# C1: batch 1 x 128, every layer FP16 with fp16 storage (5 kernels per layer)
$NCU -k regex:"gemm_kernel|gemm_persistent_kernel|attention_kernel" -s 65 -c 5 -o gpurun_out/prof_r02_c1 \
    python tools/profile_forward.py --workload c2 --batch 1 --mode FP --fp16-storage --iters 2 > gpurun_out/ncu_r02_c1.log 2>&1
# C4: BERT-large 64 x 256 FULLY_QUANT: the INT8 attention (S = 256: two-kernel path)
$NCU -k regex:"attention_kernel" -s 30 -c 1 -o gpurun_out/prof_r02_c4att \
    python tools/profile_forward.py --workload c4 --iters 2 > gpurun_out/ncu_r02_c4.log 2>&1
# C5: 4096 x 64 text matching FFN_ONLY: f16 QKV, attention (packed S = 64), out-proj; INT8 FFN
$NCU -k regex:"gemm_kernel|gemm_persistent_kernel|attention_kernel" -s 65 -c 5 -o gpurun_out/prof_r02_c5 \
    python tools/profile_forward.py --workload c5 --iters 2 > gpurun_out/ncu_r02_c5.log 2>&1
tail -2 gpurun_out/ncu_r02_*.log
