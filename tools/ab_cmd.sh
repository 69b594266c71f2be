timeout 300 python -m pytest tests/test_gpu_kernels.py -k gelu_fast_admission -x -q -s > gpurun_out/gadm_new.txt 2>&1
SAMP_B200_LIB=abtest/flags/libsamp_b200.so timeout 300 python tools/gelu_flag_rate.py > gpurun_out/gflags.txt 2>&1
bash tools/gelu_ab.sh marginv2 "c2 c4"
