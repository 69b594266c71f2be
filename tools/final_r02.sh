# End-of-round-2 verification and evidence: full GPU suite, smoke, bench lines (C2/C4/C5 and
# the reference arm), the bench's ncu launch list and one ncu --set full capture of a C2
# layer (FFN1's epilogue changed late in the round).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final_gt.log 2>&1; tail -2 gpurun_out/final_gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_c2.log 2>&1
timeout 600 python bench.py --workload c4 > gpurun_out/final_c4.log 2>&1
timeout 600 python bench.py --workload c5 > gpurun_out/final_c5.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k regex:"qkv_attention_kernel|gemm_kernel|gemm_persistent_kernel" -s 52 -c 4 -o gpurun_out/prof_r02e_c2 \
    python tools/profile_forward.py --workload c2 --iters 2 > gpurun_out/ncu_r02e_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02e.csv \
    python bench.py --steps 2 --warmup 1 --lat-iters 1 --no-cpu > gpurun_out/launches_r02e.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02e_c2.ncu-rep > gpurun_out/ncu_r02e_c2.txt 2>&1
