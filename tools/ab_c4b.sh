for i in 1 2; do
  for d in w_bf4e19d w_d39e322; do
    (cd abtest/$d && timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > ../../gpurun_out/c4b_${d}_$i.log 2>&1)
  done
  timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/c4b_head_$i.log 2>&1
done
for f in gpurun_out/c4b_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
