# A/B of env settings on C2 + batch-1: tools/ab_env3.sh "VAR=1 VAR2=1" "VAR=0" ... (one quoted set per arm)
i=0
for rep in 1 2; do
  for arm in "$@"; do
    i=$((i+1))
    env $arm timeout 300 python bench.py --steps 20 --warmup 5 --lat-iters 20 --no-cpu > gpurun_out/ae_$i.log 2>&1
    tail -1 gpurun_out/ae_$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('[$arm]', d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
  done
done
