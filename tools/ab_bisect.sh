# Same-box bisection: each abtest/w_<commit> worktree runs its own bench at C4 / C2 (per-kernel event times).
for w in c4 c2; do
  for d in abtest/r1 abtest/w_* .; do
    n=$(basename $d)
    (cd $d && timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --lat-iters 3 --no-cpu > /root/repo/gpurun_out/bis_${n}_${w}.log 2>&1)
  done
done
for f in gpurun_out/bis_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
