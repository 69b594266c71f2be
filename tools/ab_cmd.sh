# scratch A/B driver (edited per experiment): embed gamma/beta prefetch
timeout 900 python -m pytest -q -x tests/test_gpu_engine.py tests/test_gpu_kernels.py -k "embed or bit_exact or golden" > gpurun_out/abt.log 2>&1; tail -1 gpurun_out/abt.log
bash tools/ab_lib.sh "c2" base= embold=abtest/embold/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
