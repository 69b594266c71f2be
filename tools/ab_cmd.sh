# scratch A/B driver (edited per experiment): GELU chunk 32 vs 16
timeout 300 python tools/persist_phases.py --workload c2 > gpurun_out/pp_base.txt 2>&1
SAMP_B200_LIB=abtest/ch32/libsamp_b200.so timeout 300 python tools/persist_phases.py --workload c2 > gpurun_out/pp_ch32.txt 2>&1
bash tools/ab_lib.sh "c2 c4" base= ch32=abtest/ch32/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
