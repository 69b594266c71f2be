# A/B of env settings on C4: tools/ab_env_c4.sh "VAR=1" "X=1" ...
i=0
for rep in 1 2; do
  for arm in "$@"; do
    i=$((i+1))
    env $arm timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/aec4_$i.log 2>&1
    tail -1 gpurun_out/aec4_$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('[$arm]', d['value'], d['ms_per_step'], {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
  done
done
