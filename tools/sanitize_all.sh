# compute-sanitizer memcheck / racecheck / synccheck on tools/sanitizer_case.py -> gpurun_out/san_*.txt
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitizer_case.py > gpurun_out/san_$tool.txt 2>&1
done
