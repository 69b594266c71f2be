# three passes of tools/ab_lib.sh-style runs: tools/ab_lib3.sh "<workloads>" name=lib ...
W=$1; shift
for i in 1 2 3; do
  for w in $W; do
    for nv in "$@"; do
      n=${nv%%=*}; l=${nv#*=}
      SAMP_B200_LIB=$l timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --lat-iters 20 --no-cpu > gpurun_out/al_${n}_${w}_$i.log 2>&1
    done
  done
done
for f in gpurun_out/al_*.log; do
  tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
print('$f', d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {a: b['avg_us'] for a,b in k.items()})" 2>&1 | tail -1
done
