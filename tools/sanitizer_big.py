# synccheck repro: the 192-wide 4-CTA-cluster LN GEMM at 40 row tiles (tools/sanitizer_case.py's last case alone)
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.quantization import CalibrationTable
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.tokenization import EncodedInput
from paper_2209_09130_b200.engine import Engine
from oracle import samp_oracle as orc
vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
arch = build_archive(num_layers=1, hidden=768, num_heads=12, intermediate=3072, max_position=512, seed=3,
                     weight_scale=0.02, vocab=vocab, task="classification")
model = orc.Model.from_manifest(arch.manifest, arch.tensors)
table = CalibrationTable(model_fingerprint=arch.fingerprint)
ids = list(range(4, 100)); taps = {}
orc.run(model, ids, [0]*len(ids), len(ids), orc.plan_prefix("FP", 1, 0), taps=taps)
for s, v in taps.items(): table.observe(s, v)
arch.calibration = table
eng = Engine(arch)
rng = np.random.default_rng(0)
big = [EncodedInput(rng.integers(4, 1000, 128).tolist(), [0] * 128, 128) for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40)]
r = eng.run_batch(big, PrecisionPlan.prefix("FULLY_QUANT", 1, 1))
print("big ok", float(np.abs(r.hidden_states).sum()))
