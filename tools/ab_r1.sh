# Same-box A/B of the round-1 tree (abtest/r1, a git worktree) against HEAD at C4 and C2.
# Prints per-kernel times from each tree's own bench line.
for w in c4 c2; do
  for i in 1 2; do
    (cd abtest/r1 && timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --lat-iters 3 --no-cpu > ../../gpurun_out/abr1_r1_${w}_$i.log 2>&1)
    timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/abr1_head_${w}_$i.log 2>&1
  done
done
for f in gpurun_out/abr1_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
