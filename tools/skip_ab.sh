# C2 critical-path cost per kernel: step time with each kernel's launches dropped
# (SAMP_SKIP; results garbage) against the full step.  tools/skip_ab.sh
for s in "" qkv_attention_i8 ffn1_i8 ffn2_i8 outproj_i8 embed head "qkv_attention_i8,outproj_i8,ffn1_i8,ffn2_i8"; do
  SAMP_SKIP=$s python bench.py --no-cpu --steps 30 --warmup 5 --lat-iters 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$s', d['ms_per_step'])"
done
