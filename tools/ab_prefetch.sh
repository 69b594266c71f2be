# A/B of the L2 weight prefetch: bench C2 + batch-1 latency with and without it (twice each)
for i in 1 2; do
  for v in 0 1; do
    SAMP_NO_PREFETCH=$v timeout 300 python bench.py --steps 20 --warmup 5 --lat-iters 20 --no-cpu > gpurun_out/ab_pf_$v.log 2>&1
    tail -1 gpurun_out/ab_pf_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_PREFETCH=$v', d['value'], d['ms_per_step'], d['latency_b1_p50_ms'])"
  done
done
