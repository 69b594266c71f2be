# scratch A/B driver (edited per experiment): INT8 ctx codes on FFMA2 pairs
timeout 900 python -m pytest -q -x tests/test_gpu_fused_attention.py tests/test_gpu_engine.py > gpurun_out/abt.log 2>&1; tail -1 gpurun_out/abt.log
bash tools/ab_lib.sh "c2 c4" base= ctxs=abtest/ctxs/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
bash tools/ab_lat.sh "X=1" "SAMP_B200_LIB=abtest/ctxs/libsamp_b200.so" 2 > gpurun_out/ab_lat.txt 2>&1
