"""BERT-style host tokenizer: basic split + greedy wordpiece + pair encoding.

The reference snapshot does not ship its ``samp/tokenization.py`` although
five of its modules import it (reference: pkg/src/samp/__init__.py:33,
encoder.py:41, archive.py:26, synthetic.py:14, cli.py:31).  This module is
restated from the behavioural spec (reference: SPEC.md:230-286) and the
reference's own tests (reference: pkg/tests/test_tokenization.py:22-162).
It is host preprocessing, not part of the GPU hot path.  The restatement is
pinned by regenerating the reference's ``tiny_cls`` calibration table and
matching all of its amax values bit-exactly (tests/golden/make_golden.py),
which requires identical token ids for the sample texts.
"""

from __future__ import annotations

import ctypes
import os
import unicodedata
import weakref
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

SPECIAL_TOKENS = ("[CLS]", "[SEP]", "[PAD]", "[UNK]")
MAX_WORD_CHARS = 100
_CONT = "##"


@dataclass(frozen=True)
class EncodedInput:
    """One encoded sequence: ids, segment ids and the non-pad prefix length."""

    token_ids: list
    segment_ids: list
    attention_length: int


class Vocab:
    """Dense token -> id map with the four special tokens and encode limits."""

    def __init__(self, token_to_id: dict, do_lower_case: bool = True,
                 max_seq_len: int = 128, char_mode: bool = False):
        ids = sorted(token_to_id.values())
        if ids != list(range(len(ids))):
            raise ConfigurationError("vocab ids must be unique and dense from 0")
        absent = [t for t in SPECIAL_TOKENS if t not in token_to_id]
        if absent:
            raise ConfigurationError(f"vocab lacks special tokens: {', '.join(absent)}")
        if max_seq_len < 2:
            raise ConfigurationError(f"max_seq_len must be >= 2, got {max_seq_len}")
        self.token_to_id = dict(token_to_id)
        self.id_to_token = {i: t for t, i in self.token_to_id.items()}
        self.do_lower_case = bool(do_lower_case)
        self.max_seq_len = int(max_seq_len)
        self.char_mode = bool(char_mode)

    @classmethod
    def from_tokens(cls, tokens, **kwargs) -> "Vocab":
        mapping = {}
        for tok in tokens:
            if tok in mapping:
                raise ConfigurationError(f"duplicate vocab token {tok!r}")
            mapping[tok] = len(mapping)
        return cls(mapping, **kwargs)

    @classmethod
    def load(cls, path, max_seq_len: int = 128, **kwargs) -> "Vocab":
        with open(path, encoding="utf-8") as fh:
            tokens = [line.rstrip("\n").rstrip("\r") for line in fh]
        while tokens and tokens[-1] == "":
            tokens.pop()
        return cls.from_tokens(tokens, max_seq_len=max_seq_len, **kwargs)

    def save(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            for i in range(len(self)):
                fh.write(self.id_to_token[i] + "\n")

    def __len__(self) -> int:
        return len(self.token_to_id)

    def __contains__(self, token) -> bool:
        return token in self.token_to_id

    @property
    def cls_id(self) -> int:
        return self.token_to_id["[CLS]"]

    @property
    def sep_id(self) -> int:
        return self.token_to_id["[SEP]"]

    @property
    def pad_id(self) -> int:
        return self.token_to_id["[PAD]"]

    @property
    def unk_id(self) -> int:
        return self.token_to_id["[UNK]"]


def _is_space(ch: str) -> bool:
    return ch in " \t\n\r" or unicodedata.category(ch) == "Zs"


def _is_control(ch: str) -> bool:
    if ch in "\t\n\r":
        return False
    return unicodedata.category(ch) in ("Cc", "Cf")


def _is_punct(ch: str) -> bool:
    cp = ord(ch)
    if 33 <= cp <= 47 or 58 <= cp <= 64 or 91 <= cp <= 96 or 123 <= cp <= 126:
        return True
    return unicodedata.category(ch).startswith("P")


_CJK_RANGES = (
    (0x4E00, 0x9FFF), (0x3400, 0x4DBF), (0x20000, 0x2A6DF), (0x2A700, 0x2B73F),
    (0x2B740, 0x2B81F), (0x2B820, 0x2CEAF), (0xF900, 0xFAFF), (0x2F800, 0x2FA1F),
)


def _is_cjk(ch: str) -> bool:
    cp = ord(ch)
    return any(lo <= cp <= hi for lo, hi in _CJK_RANGES)


def _normalize(vocab: Vocab, text: str) -> str:
    text = unicodedata.normalize("NFC", text)
    text = "".join(" " if _is_space(c) else c for c in text
                   if c not in ("\x00", "�") and not _is_control(c))
    if vocab.do_lower_case:
        text = unicodedata.normalize("NFD", text.lower())
        text = "".join(c for c in text if unicodedata.category(c) != "Mn")
    return text


def _basic_words(vocab: Vocab, text: str) -> list:
    """Whitespace split with punctuation and CJK codepoints isolated."""
    words: list = []
    current: list = []

    def flush():
        if current:
            words.append("".join(current))
            current.clear()

    for ch in _normalize(vocab, text):
        if ch == " ":
            flush()
        elif vocab.char_mode or _is_punct(ch) or _is_cjk(ch):
            flush()
            words.append(ch)
        else:
            current.append(ch)
    flush()
    return words


def wordpiece(vocab: Vocab, word: str) -> list:
    """Greedy longest-match-first split with '##' continuation pieces."""
    if len(word) > MAX_WORD_CHARS:
        return ["[UNK]"]
    pieces = []
    pos = 0
    while pos < len(word):
        match = None
        for end in range(len(word), pos, -1):
            cand = word[pos:end] if pos == 0 else _CONT + word[pos:end]
            if cand in vocab.token_to_id:
                match = cand
                pos = end
                break
        if match is None:
            return ["[UNK]"]
        pieces.append(match)
    return pieces


def tokenize(vocab: Vocab, text: str) -> list:
    out = []
    for word in _basic_words(vocab, text):
        out.extend(wordpiece(vocab, word))
    return out


def encode(vocab: Vocab, text_a: str, text_b: str | None = None) -> EncodedInput:
    """[CLS] a [SEP] (b [SEP]), longest-first truncation, padded to max_seq_len."""
    limit = vocab.max_seq_len
    a = [vocab.token_to_id[t] for t in tokenize(vocab, text_a)]
    if text_b is None:
        a = a[: max(limit - 2, 0)]
        ids = [vocab.cls_id] + a + [vocab.sep_id]
        segs = [0] * len(ids)
    else:
        b = [vocab.token_to_id[t] for t in tokenize(vocab, text_b)]
        budget = max(limit - 3, 0)
        while len(a) + len(b) > budget:
            if len(a) > len(b):
                a.pop()
            else:
                b.pop()
        ids = [vocab.cls_id] + a + [vocab.sep_id] + b + [vocab.sep_id]
        segs = [0] * (len(a) + 2) + [1] * (len(b) + 1)
    length = len(ids)
    pad = limit - length
    ids = ids + [vocab.pad_id] * pad
    segs = segs + [segs[-1] if text_b is not None else 0] * pad
    return EncodedInput(ids, segs, length)


# ------------------------------------------------------------------ native batch encoder
def _native_tokenizer(vocab: Vocab):
    """The library's tokenizer for this vocab (built once per Vocab, freed with it)."""
    h = getattr(vocab, "_native", None)
    if h is not None:
        return h
    from . import _lib
    lib = _lib.load()
    toks = [vocab.id_to_token[i].encode("utf-8") for i in range(len(vocab))]
    arr = (ctypes.c_char_p * len(toks))(*toks)
    h = lib.samp_tokenizer_create(arr, len(toks), int(vocab.do_lower_case), vocab.max_seq_len, int(vocab.char_mode))
    if h:
        weakref.finalize(vocab, lib.samp_tokenizer_destroy, h)
    vocab._native = h or 0
    return vocab._native


def encode_batch(vocab: Vocab, texts_a, texts_b=None, threads: int | None = None):
    """encode() over many texts at once on the native multi-threaded tokenizer.

    Returns (ids, segs, att): int32 [n][max_seq_len], [n][max_seq_len], [n] — row i equals
    encode(vocab, texts_a[i], texts_b[i]).  Texts with non-ASCII characters are encoded by
    the Python path (Unicode normalisation), everything else natively.
    """
    texts_a = list(texts_a)
    n = len(texts_a)
    if texts_b is not None:
        texts_b = list(texts_b)
        if len(texts_b) != n:
            raise ConfigurationError("texts_a and texts_b differ in length")
    L = vocab.max_seq_len
    ids = np.empty((n, L), np.int32)
    segs = np.empty((n, L), np.int32)
    att = np.empty(n, np.int32)
    fb = np.ones(n, np.uint8)
    h = _native_tokenizer(vocab) if n else 0
    if h:
        from . import _lib
        def cstr(t):   # an embedded NUL would truncate the C string: route it to Python
            b = t.encode("utf-8")
            return b"\x80" if b"\x00" in b else b
        a_arr = (ctypes.c_char_p * n)(*[cstr(t) for t in texts_a])
        b_arr = None
        if texts_b is not None:
            b_arr = (ctypes.c_char_p * n)(*[None if t is None else cstr(t) for t in texts_b])
        nthreads = threads or min(16, os.cpu_count() or 1)
        _lib.load().samp_tokenize_batch(h, a_arr, b_arr, n, nthreads, ids.ctypes.data, segs.ctypes.data,
                                        att.ctypes.data, fb.ctypes.data)
    for i in np.nonzero(fb)[0]:
        enc = encode(vocab, texts_a[i], None if texts_b is None else texts_b[i])
        ids[i], segs[i], att[i] = enc.token_ids, enc.segment_ids, enc.attention_length
    return ids, segs, att
