#!/bin/bash
# A/B timing of one build under two environments: tools/ab_env.sh "<envA>" "<envB>" [rounds]
# e.g. tools/ab_env.sh "" "SAMP_NO_PDL=1" 2
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for arm in A B; do
    envs=$A; [ $arm = B ] && envs=$B
    env $envs python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$arm', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('latency_b1_p50_ms'), {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items()})"
  done
done
