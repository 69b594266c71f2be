# Batch-1 latency A/B of one build under two environments: tools/ab_lat.sh "<envA>" "<envB>" [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for arm in A B; do
    envs=$A; [ $arm = B ] && envs=$B
    env $envs python bench.py --no-cpu --steps 5 --warmup 3 --lat-iters 60 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$arm', d['value'], d.get('latency_b1_p50_ms'))"
  done
done
