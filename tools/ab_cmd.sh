# scratch A/B driver (edited per experiment): fused-kernel att_expo32_fast without per-key selects
timeout 900 python -m pytest -q -x tests/test_gpu_fused_attention.py > gpurun_out/abt.log 2>&1; tail -1 gpurun_out/abt.log
timeout 300 python tools/qa_phases.py > gpurun_out/qa_phases_base.txt 2>&1
bash tools/ab_lib.sh "c2" base= csel=abtest/csel/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
bash tools/ab_lat.sh "X=1" "SAMP_B200_LIB=abtest/csel/libsamp_b200.so" 2 > gpurun_out/ab_lat.txt 2>&1
