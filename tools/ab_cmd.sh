# scratch A/B driver (edited per experiment): EpiF16Out with GELU / amax compiled per launch
timeout 900 python -m pytest -q -x tests/test_gpu_engine.py tests/test_gpu_taps_fp16.py tests/test_gpu_logits_stats.py > gpurun_out/abt.log 2>&1; tail -1 gpurun_out/abt.log
bash tools/ab_lat.sh "X=1" "SAMP_B200_LIB=abtest/f16old/libsamp_b200.so" 3 > gpurun_out/ab_lat.txt 2>&1
bash tools/ab_lib.sh "c5" base= f16old=abtest/f16old/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
