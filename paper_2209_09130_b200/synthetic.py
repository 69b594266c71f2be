"""Deterministic random-init archives (the "identical random-init weights").

``build_archive`` draws every tensor from one ``numpy.random.default_rng(seed)``
in ``expected_shapes`` order with the reference's distributions
(reference: pkg/src/samp/synthetic.py:38-79): LayerNorm gamma ~ 1 + 0.1 N,
beta ~ 0.05 N, biases ~ 0.1 N, weights ~ weight_scale * N.  Equal seeds give
byte-identical archives (checked by fingerprint against the reference in
tests/golden).  ``bert_archive`` sizes it as BERT-base / BERT-large.
"""

from __future__ import annotations

import numpy as np

from .archive import ModelArchive, ModelManifest, compute_fingerprint, expected_shapes
from .tokenization import SPECIAL_TOKENS, Vocab

DEFAULT_WORDS = [
    "the", "a", "quick", "brown", "fox", "jump", "##s", "##ing", "##ed",
    "over", "lazy", "dog", "cat", "run", "walk", "un", "##able", "match",
    "text", "good", "bad", "fast", "slow", "model", "layer", "quant",
    "0", "1", "2", "3", "4", "5", "6", "7", "8", "9", ",", ".", "!", "?",
]

SAMPLE_TEXTS = [
    "the quick brown fox jumps over the lazy dog",
    "a lazy cat walks over the slow dog",
    "quant the model layer by layer",
    "good fast model , bad slow model !",
    "unable to match the text ?",
    "the dog runs . the fox walks !",
]

BERT_SHAPES = {
    "bert-base": dict(num_layers=12, hidden=768, num_heads=12, intermediate=3072),
    "bert-large": dict(num_layers=24, hidden=1024, num_heads=16, intermediate=4096),
}


def tiny_vocab(max_seq_len: int = 16, extra_tokens=None, **kwargs) -> Vocab:
    return Vocab.from_tokens(list(SPECIAL_TOKENS) + DEFAULT_WORDS + list(extra_tokens or []),
                             max_seq_len=max_seq_len, **kwargs)


def padded_vocab(size: int, max_seq_len: int) -> Vocab:
    """tiny_vocab grown with filler tokens to ``size`` entries (30522 for BERT)."""
    base = len(SPECIAL_TOKENS) + len(DEFAULT_WORDS)
    return tiny_vocab(max_seq_len, [f"[unused{i}]" for i in range(size - base)])


def _draw(rng, key: str, shape, weight_scale: float) -> np.ndarray:
    if key.endswith("layernorm.gamma"):
        v = 1.0 + 0.1 * rng.standard_normal(shape)
    elif key.endswith("layernorm.beta"):
        v = 0.05 * rng.standard_normal(shape)
    elif key.endswith((".bias", ".b1", ".b2")):
        v = 0.1 * rng.standard_normal(shape)
    else:
        v = weight_scale * rng.standard_normal(shape)
    return v.astype(np.float32)


def build_archive(num_layers: int = 2, hidden: int = 8, num_heads: int = 2, intermediate: int = 16,
                  task: str = "classification", num_labels: int = 2, max_position: int = 16,
                  seed: int = 0, weight_scale: float = 0.35, vocab: Vocab | None = None) -> ModelArchive:
    vocab = vocab or tiny_vocab(max_seq_len=max_position)
    manifest = ModelManifest(num_layers=num_layers, hidden=hidden, num_heads=num_heads,
                             intermediate=intermediate, vocab_size=len(vocab),
                             max_position=max_position, type_vocab_size=2, layernorm_eps=1e-12,
                             task=task, num_labels=num_labels)
    rng = np.random.default_rng(seed)
    tensors = {key: _draw(rng, key, shape, weight_scale)
               for key, shape in expected_shapes(manifest).items()}
    archive = ModelArchive(manifest, tensors, vocab)
    archive.validate()
    archive.fingerprint = compute_fingerprint(manifest, tensors)
    return archive


def bert_archive(model: str = "bert-base", task: str = "classification", num_labels: int = 2,
                 seed: int = 0, weight_scale: float = 0.02, vocab_size: int = 30522,
                 max_position: int = 512) -> ModelArchive:
    """BERT-shaped random-init archive (SURVEY.md §8(d) weights recipe)."""
    return build_archive(task=task, num_labels=num_labels, max_position=max_position, seed=seed,
                         weight_scale=weight_scale, vocab=padded_vocab(vocab_size, max_position),
                         **BERT_SHAPES[model])
