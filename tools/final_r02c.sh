# Final check after the attention pass-2 change: full GPU suite, smoke, C2 / C4 / C3 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final3_gt.log 2>&1; tail -1 gpurun_out/final3_gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; tail -1 gpurun_out/final3_smoke.log
timeout 600 python bench.py > gpurun_out/final3_c2.log 2>&1
timeout 600 python bench.py --workload c4 > gpurun_out/final3_c4.log 2>&1
timeout 600 python bench.py --workload c3 > gpurun_out/final3_c3.log 2>&1
