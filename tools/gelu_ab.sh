# FFN1 GELU epilogue A/B: per-tile phases and C2/C4 bench for the in-tree build against
# abtest/$1 (tools/build_variant.py); workloads in $2 (default c2)
timeout 300 python tools/persist_phases.py --workload c2 > gpurun_out/pp_base.txt 2>&1
SAMP_B200_LIB=abtest/$1/libsamp_b200.so timeout 300 python tools/persist_phases.py --workload c2 > gpurun_out/pp_$1.txt 2>&1
bash tools/ab_lib.sh "${2:-c2}" base= $1=abtest/$1/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
