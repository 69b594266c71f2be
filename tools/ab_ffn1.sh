# FFN1 tile-width / occupancy variants (tools/build_variant.py f64x3 SAMP_FFN1_64X3=1)
for v in "base:" "bn64:SAMP_FFN1_BN=64" "bn128:SAMP_FFN1_BN=128" "f64x3:SAMP_FFN1_BN=64 SAMP_B200_LIB=abtest/f64x3/libsamp_b200.so"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['ms_per_step'], {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items() if 'ffn1' in k})"
done
