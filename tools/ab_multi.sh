#!/bin/bash
# A/B/C... timing of several builds of the engine library: tools/ab_multi.sh ROUNDS lib1.so lib2.so ...
# Each arm runs bench.py (device-timed, no CPU baseline) in turn; prints value + per-kernel us.
R=$1; shift
for r in $(seq $R); do
  for lib in "$@"; do
    SAMP_B200_LIB=$lib python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-2], d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items()})"
  done
done
