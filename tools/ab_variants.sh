for v in ne16 ch32 cta2 ne16ch32; do
  SAMP_B200_LIB=abtest/$v/libsamp_b200.so python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items() if 'ffn1' in k})"
done
python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base', d['value'], d['ms_per_step'], d.get('latency_b1_p50_ms'), {k:round(v['avg_us'],2) for k,v in d.get('kernels',{}).items() if 'ffn1' in k})"
