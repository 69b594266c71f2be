# HEAD C4 + C2 bench lines (two passes) -> gpurun_out/q_*.log + summary
for i in 1 2; do
  timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/q_c4_$i.log 2>&1
  timeout 400 python bench.py --workload c2 --steps 20 --warmup 5 --lat-iters 10 --no-cpu > gpurun_out/q_c2_$i.log 2>&1
done
for f in gpurun_out/q_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
