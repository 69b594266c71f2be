# End-of-round-2 final state: GPU suite, smoke, bench lines (C2/C4/C3/C5, reference arm),
# the bench's ncu launch list and an ncu --set full capture of one C2 layer and of C4's attention
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gt.log 2>&1; tail -1 gpurun_out/fin_gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 600 python bench.py > gpurun_out/fin_c2.log 2>&1
timeout 600 python bench.py --workload c4 > gpurun_out/fin_c4.log 2>&1
timeout 600 python bench.py --workload c3 > gpurun_out/fin_c3.log 2>&1
timeout 900 python bench.py --workload c5 > gpurun_out/fin_c5.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fin.csv \
    python bench.py --steps 2 --warmup 1 --lat-iters 1 --no-cpu > gpurun_out/launches_fin.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k regex:"qkv_attention_kernel|gemm_kernel|gemm_persistent_kernel" -s 52 -c 4 -o gpurun_out/prof_fin_c2 \
    python tools/profile_forward.py --workload c2 --iters 2 > gpurun_out/ncu_fin_c2.log 2>&1
timeout 900 $NCU -k regex:"attention_kernel" -s 30 -c 1 -o gpurun_out/prof_fin_c4att \
    python tools/profile_forward.py --workload c4 --iters 2 > gpurun_out/ncu_fin_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_fin_c2.ncu-rep > gpurun_out/ncu_fin_c2.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_fin_c4att.ncu-rep > gpurun_out/ncu_fin_c4att.txt 2>&1
