# fused-kernel phase stamps + C2 bench for the in-tree build and abtest/$1
timeout 300 python tools/qa_phases.py > gpurun_out/qa_phases_base.txt 2>&1
SAMP_B200_LIB=abtest/$1/libsamp_b200.so timeout 300 python tools/qa_phases.py > gpurun_out/qa_phases_$1.txt 2>&1
bash tools/ab_lib.sh "c2" base= $1=abtest/$1/libsamp_b200.so > gpurun_out/al_summary.txt 2>&1
