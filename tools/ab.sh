#!/bin/bash
# A/B timing of two builds of the engine library: tools/ab.sh <libA.so> <libB.so> [rounds]
# Each arm runs bench.py (device-timed, no CPU baseline) alternately; prints value + kernels.
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for arm in A B; do
    lib=$A; [ $arm = B ] && lib=$B
    SAMP_B200_LIB=$lib python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$arm', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('latency_b1_p50_ms'), {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items()})"
  done
done
