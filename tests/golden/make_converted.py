"""Converter interop fixture (build container only; needs /root/reference, torch, transformers).

    python tests/golden/make_converted.py

A tiny HF ``BertForSequenceClassification`` at GPU-legal shapes (head_dim 64: hidden 128,
2 heads, 2 layers, intermediate 256, gelu_new = the reference's tanh GELU) is converted by
the REFERENCE's own converter (``samp_convert.convert.convert_checkpoint``,
pkg/converter/src/samp_convert/convert.py:180) into tests/golden/converted_bert/, and the
reference's parity fixture (``samp_convert.fixture.emit_parity_fixture``, fixture.py:50: 5
fixed-seed texts + torch logits) is written next to it — the same acceptance check the
reference runs (pkg/converter/tests/test_convert.py:176-193), here consumed by
tests/test_gpu_converter.py on the B200 engine.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "converted_bert"
sys.path.insert(0, "/root/reference/pkg/converter/src")

WORDS = ["the", "a", "quick", "brown", "fox", "jump", "over", "lazy", "dog", "cat", "run", "walk", "good",
         "bad", "fast", "slow", "model", "layer", "text", "match", "un", "able", "to", "and", "or", "not",
         "is", "was", "big", "small", "red", "blue", "green", "old", "new", "day", "night", "sun", "moon",
         "star", "tree", "bird", "fish", "stone", "river", "hill"]


def main():
    import torch
    from transformers import BertConfig, BertForSequenceClassification

    from samp_convert.convert import convert_checkpoint
    from samp_convert.fixture import emit_parity_fixture

    src = Path(tempfile.mkdtemp(prefix="hf_bert_"))
    tokens = ["[PAD]", "[UNK]", "[CLS]", "[SEP]"] + WORDS + ["##s"]
    config = BertConfig(vocab_size=len(tokens), hidden_size=128, num_hidden_layers=2, num_attention_heads=2,
                        intermediate_size=256, max_position_embeddings=64, type_vocab_size=2,
                        hidden_act="gelu_new", num_labels=2, initializer_range=0.05)
    torch.manual_seed(0)
    model = BertForSequenceClassification(config).eval()
    model.save_pretrained(src)
    (src / "vocab.txt").write_text("\n".join(tokens) + "\n", encoding="utf-8")
    if OUT.exists():
        shutil.rmtree(OUT)
    report = convert_checkpoint(src, OUT, "classification", 2)
    assert report.missing_required == []
    doc = emit_parity_fixture(src, OUT / "parity.json", count=16, seed=1234)
    print("wrote", OUT, "inputs", len(doc["inputs"]), "bytes", sum(f.stat().st_size for f in OUT.iterdir()))
    shutil.rmtree(src)


if __name__ == "__main__":
    main()
