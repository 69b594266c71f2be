for s in "" attention_i8 ffn1_i8 ffn2_i8 outproj_i8 qkv_i8 "qkv_i8,attention_i8,outproj_i8,ffn1_i8,ffn2_i8"; do
  SAMP_SKIP=$s python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$s', d['ms_per_step'])"
done
