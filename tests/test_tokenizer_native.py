"""Native multi-threaded tokenizer (csrc/tokenizer_host.cu) == the Python encoder, row by
row, on random texts exercising every rule: case, ASCII punctuation, \\t\\n\\r and other
control characters, long words (> 100 chars -> [UNK]), unknown pieces, pair truncation,
padding segments; non-ASCII texts go through the Python path inside encode_batch."""

import time

import numpy as np
import pytest

from paper_2209_09130_b200.synthetic import tiny_vocab
from paper_2209_09130_b200.tokenization import Vocab, encode, encode_batch

WORDS = ["the", "quick", "brown", "fox", "jump", "##s", "##ed", "over", "lazy", "dog", "un", "##believ",
         "##able", "a", "##b", "##c", "hello", "world", ",", ".", "!", "?", "'", "(", ")", "-", "##ing",
         "run", "walk", "##er", "x", "##y", "1", "2", "##3", "ab", "##cd"]


def _vocab(max_seq_len=32, **kw):
    base = set(tiny_vocab(max_seq_len=16).token_to_id)
    extra = []
    for w in WORDS:
        if w not in base and w not in extra:
            extra.append(w)
    return tiny_vocab(max_seq_len=max_seq_len, extra_tokens=extra, **kw)


def _random_text(rng, ascii_only=True):
    parts = []
    for _ in range(rng.integers(0, 25)):
        r = rng.random()
        if r < 0.5:
            w = str(rng.choice([w.lstrip("#") for w in WORDS]))
            if rng.random() < 0.3:
                w = w.upper()
            if rng.random() < 0.2:
                w += str(rng.choice(["s", "ed", "ing", "abc", "zz"]))
            parts.append(w)
        elif r < 0.6:
            parts.append("".join(rng.choice(list("abcdefghij"), size=int(rng.integers(95, 110)))))
        elif r < 0.8:
            parts.append(str(rng.choice(list(",.!?'()-;:[]{}~`\\\"/@#$%^&*_+=|<>"))))
        else:
            parts.append(str(rng.choice(["\t", "\n", "\r", "\x0b", "\x0c", "\x07", "\x7f", "  "])))
    sep = [" ", "", "\t"]
    text = "".join(p + str(rng.choice(sep)) for p in parts)
    if not ascii_only:
        text += str(rng.choice(["café", "naïve", "中文", "Ångström", " x"]))
    return text


@pytest.mark.parametrize("max_len,lower,char_mode", [(32, True, False), (16, False, False), (12, True, True),
                                                     (128, True, False)])
def test_native_batch_equals_python_encode(max_len, lower, char_mode):
    vocab = _vocab(max_seq_len=max_len, do_lower_case=lower, char_mode=char_mode)
    rng = np.random.default_rng(max_len)
    a = [_random_text(rng, ascii_only=rng.random() < 0.9) for _ in range(300)]
    b = [None if rng.random() < 0.3 else _random_text(rng) for _ in range(300)]
    for texts_b in (None, b):
        ids, segs, att = encode_batch(vocab, a, texts_b, threads=4)
        for i in range(len(a)):
            want = encode(vocab, a[i], None if texts_b is None else texts_b[i])
            assert ids[i].tolist() == want.token_ids, (a[i], None if texts_b is None else texts_b[i])
            assert segs[i].tolist() == want.segment_ids
            assert att[i] == want.attention_length


def test_native_edge_cases():
    vocab = _vocab(max_seq_len=10)
    cases = [("", None), ("", ""), ("a\x00b", None), ("x" * 101, None), ("x" * 100, None), ("HELLO,World!", "dog"),
             ("the quick brown fox jumps over the lazy dog", "the quick brown fox"), ("\t\n\r", "\x0b\x0c")]
    ids, segs, att = encode_batch(vocab, [c[0] for c in cases], [c[1] for c in cases], threads=2)
    for i, (ta, tb) in enumerate(cases):
        want = encode(vocab, ta, tb)
        assert (ids[i].tolist(), segs[i].tolist(), int(att[i])) == (want.token_ids, want.segment_ids,
                                                                     want.attention_length)


def test_native_throughput_report():
    """Not a gate: prints native vs Python texts/s on this host."""
    vocab = _vocab(max_seq_len=128)
    rng = np.random.default_rng(0)
    texts = [_random_text(rng) for _ in range(2000)]
    t0 = time.perf_counter()
    encode_batch(vocab, texts, threads=8)
    t1 = time.perf_counter()
    for t in texts[:500]:
        encode(vocab, t)
    t2 = time.perf_counter()
    print(f"native {len(texts) / (t1 - t0):.0f} texts/s, python {500 / (t2 - t1):.0f} texts/s")
