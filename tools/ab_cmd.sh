# scratch A/B driver (edited per experiment): attention pass-2 clean-chunk path without selects
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_configs.py -k "attention or c4 or varlen" > gpurun_out/abt.log 2>&1; tail -1 gpurun_out/abt.log
bash tools/ab_lib.sh "c4 c3" base= csel=abtest/csel/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
