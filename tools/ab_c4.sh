# C4 A/B: HEAD vs variant builds / env switches / an older worktree, two passes each.
run() {  # name, then env assignments
  n=$1; shift
  for i in 1 2; do
    env "$@" timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > gpurun_out/c4_${n}_$i.log 2>&1
  done
}
run head X=0
run nonf SAMP_B200_LIB=abtest/nonf/libsamp_b200.so
run scal SAMP_B200_LIB=abtest/scal/libsamp_b200.so
run nocarve SAMP_NO_CARVEOUT=1
for i in 1 2; do (cd abtest/w_bf4e19d && timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > ../../gpurun_out/c4_bf4e19d_$i.log 2>&1); done
for i in 1 2; do (cd abtest/w_35b949f && timeout 400 python bench.py --workload c4 --steps 5 --warmup 3 --lat-iters 3 --no-cpu > ../../gpurun_out/c4_35b949f_$i.log 2>&1); done
for f in gpurun_out/c4_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
