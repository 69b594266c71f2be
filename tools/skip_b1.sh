# Batch-1 critical-path cost per kernel: p50 latency (cold L2) with each kernel's launches
# dropped (SAMP_SKIP; results garbage) minus the full forward's.  tools/skip_b1.sh [MODE]
MODE=${1:-FULLY_QUANT}
for k in none embed qkv_attention_i8 outproj_i8 ffn1_i8 ffn2_i8 head qkv_f16 attention_f16 outproj_f16 ffn1_f16 ffn2_f16; do
  if [ "$MODE" = FP ] && [[ "$k" == *_i8 ]]; then continue; fi
  if [ "$MODE" != FP ] && [[ "$k" == *_f16 ]]; then continue; fi
  echo -n "skip=$k: "
  SAMP_SKIP=$k python tools/l2_probe.py --mode $MODE 2>/dev/null | tail -1 | sed 's/, warm.*//'
done
