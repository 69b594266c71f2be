# A/B of an env switch on the default bench (C2 + batch-1 latency): tools/ab_env2.sh VAR
for i in 1 2; do
  for v in 0 1; do
    env $1=$v timeout 300 python bench.py --steps 20 --warmup 5 --lat-iters 20 --no-cpu > gpurun_out/ab_$1_$v.log 2>&1
    tail -1 gpurun_out/ab_$1_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1=$v', d['value'], d['ms_per_step'], d['latency_b1_p50_ms'])"
  done
done
