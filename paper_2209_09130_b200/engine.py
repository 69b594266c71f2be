"""Engine: the drop-in for the reference's ``samp.encoder.Engine`` on a B200.

Same constructor, ``run``/``check_plan``/``quantized_layer``/``encode_text``
surface and the same exceptions as the reference
(reference: pkg/src/samp/encoder.py:421-530), backed by libsamp_b200.so.
``run_batch`` is the batched, padding-free entry the reference lacks (its
batches are Python loops over ``run``, cli.py:375-377): sequences are packed
back to back and every kernel walks the packed rows.

There is no CPU fallback: the device library must be present and the GPU an
sm_100 part, otherwise construction raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .archive import ModelArchive, layer_keys
from .errors import CalibrationError, ConfigurationError, InputError
from .plan import (EMBED_OUT_SITE, LAYER_CODE, LAYER_FP, PrecisionPlan, activation_sites)
from .quantization import CalibrationTable, CodeUsageReport, QuantScale, quantize, scale_edit_count
from .tokenization import EncodedInput, encode as encode_text
from . import trace as _trace

HEAD_NONE, HEAD_CLASSIFY, HEAD_TAG = 0, 1, 2
IO_HOST, IO_DEVICE = 0, 1

_LAYER_ORDER = ("qw", "qb", "kw", "kb", "vw", "vb", "ow", "ob", "attn_ln_g", "attn_ln_b",
                "w1", "b1", "w2", "b2", "ffn_ln_g", "ffn_ln_b")


@dataclass
class EncoderOutput:
    hidden_states: np.ndarray               # (seq, hidden) float32
    taps: dict | None = None
    head: dict | None = field(default=None, repr=False)   # device head results (logits/probs/labels)


@dataclass
class QuantizedLayerWeights:
    """INT8 weights + scales of one layer (reference encoder.py:197-225).

    Scales are the ones the device engine derived; codes use the same formula
    (per-tensor max|w| scale, half-away rounding) and are produced on request.
    """

    qkv_w_q: np.ndarray
    qkv_scales: tuple
    ow_q: np.ndarray
    ow_scale: QuantScale
    w1_q: np.ndarray
    w1_scale: QuantScale
    w2_q: np.ndarray
    w2_scale: QuantScale


@dataclass
class BatchOutput:
    """run_batch result: packed rows; ``seq_start`` gives each sequence's rows."""

    seq_start: np.ndarray
    hidden_states: np.ndarray | None
    logits: np.ndarray | None
    probs: np.ndarray | None
    labels: np.ndarray | None

    def sequence(self, s: int) -> np.ndarray:
        return self.hidden_states[self.seq_start[s]:self.seq_start[s + 1]]


class Engine:
    """Loaded model on one GPU; safe to share across threads (calls are serialised)."""

    def __init__(self, archive: ModelArchive, fp16_storage: bool = False, device: int = 0,
                 exact_fp32: bool = False):
        """``exact_fp32``: run the floating-point blocks (FP layers, FFN_ONLY's attention,
        MHA-only's FFN) on the FP32 pipe with the reference's k-ordered GEMM accumulation, so
        every plan is bit-exact with the reference (samp_set_exact_fp32); default: FP16
        tensor cores within tolerance."""
        self.archive = archive
        self.manifest = m = archive.manifest
        self.vocab = archive.vocab
        self.fp16_storage = bool(fp16_storage)
        self.device = int(device)
        self._lock = threading.RLock()   # re-entrant: forward_packed -> _push_calibration
        self._quantized: dict = {}
        self._lib = lib = _lib.load()
        desc = _lib.ModelDesc(m.num_layers, m.hidden, m.num_heads, m.intermediate, m.vocab_size,
                              m.max_position, m.type_vocab_size, m.num_labels, float(m.layernorm_eps),
                              int(self.fp16_storage))
        handle = ctypes.c_void_p()
        _lib.check(lib.samp_engine_create(ctypes.byref(desc), self.device, ctypes.byref(handle)))
        self._h = handle
        t = archive.tensors
        f32 = lambda k: np.ascontiguousarray(t[k], dtype=np.float32)  # noqa: E731
        emb = [f32(k) for k in ("embeddings.word.weight", "embeddings.position.weight",
                                "embeddings.token_type.weight", "embeddings.layernorm.gamma",
                                "embeddings.layernorm.beta")]
        _lib.check(lib.samp_load_embeddings(self._h, *[a.ctypes.data for a in emb]))
        for i in range(m.num_layers):
            keys = layer_keys(i)
            arrs = [f32(keys[n]) for n in _LAYER_ORDER]
            ptrs = (ctypes.c_void_p * 16)(*[a.ctypes.data for a in arrs])
            _lib.check(lib.samp_load_layer(self._h, i, ptrs))
        head = [f32(k) if k in t else None for k in ("pooler.weight", "pooler.bias", "head.weight", "head.bias")]
        _lib.check(lib.samp_load_heads(self._h, *[a.ctypes.data if a is not None else None for a in head]))
        self.exact_fp32 = bool(exact_fp32)
        if self.exact_fp32:
            _lib.check(lib.samp_set_exact_fp32(self._h, 1))
        self._pushed_calibration = None
        self._pushed_key = None
        self._push_calibration()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.samp_engine_destroy(h)
            self._h = None

    # ------------------------------------------------------------ calibration
    @property
    def calibration(self) -> CalibrationTable | None:
        return self.archive.calibration

    def _calibration_state(self):
        """Snapshot of the archive's table, read fresh on every call as the reference does
        (encoder.py:456-470): direct edits of ``table.entries`` (replaced or mutated
        QuantScale objects, deleted sites) are seen without relying on any version counter."""
        table = self.archive.calibration
        if table is None:
            return None
        # a plain list in the dict's order (a reordered but equal table only costs a re-push)
        return [(s, e.amax) for s, e in table.entries.items()]

    def _calibration_key(self):
        """Cheap fingerprint of the table as it stands: the table and dict objects, the sites,
        the QuantScale objects (C-level tuples, compared by identity first) and the
        process-wide count of QuantScale attribute writes.  Any edit the reference would see
        (an amax written, an entry added, replaced, deleted or re-keyed, the dict or the table
        swapped) changes it; an unchanged key means the full snapshot is unchanged too."""
        table = self.archive.calibration
        if table is None:
            return None
        d = table.entries
        return (id(table), id(d), tuple(d), tuple(d.values()), scale_edit_count())

    def _push_calibration(self) -> None:
        """Send the table's amax values to the device when they differ from what it holds.
        Per forward only the cheap key is compared; the full snapshot only when it moved."""
        with self._lock:
            key = self._calibration_key()
            if key is not None and key == self._pushed_key:
                return
            state = self._calibration_state()
            if state == self._pushed_calibration:
                self._pushed_key = key
                return
            _lib.check(self._lib.samp_clear_calibration(self._h))
            self._pushed_calibration = None
            self._pushed_key = None
            for site, amax in state or ():
                _lib.check(self._lib.samp_set_site_amax(self._h, site.encode(), float(amax)))
            self._pushed_calibration = state
            self._pushed_key = key

    def check_plan(self, plan: PrecisionPlan) -> CalibrationTable | None:
        """reference encoder.py:456-470 (same messages)."""
        table = self.calibration
        # a plan already checked against a table holding the same site names: nothing to redo
        key = (plan.layer_precisions, None if table is None else frozenset(table.entries))
        if key == getattr(self, "_checked_key", None):
            return table
        self._check_plan_uncached(plan)
        self._checked_key = key
        return table

    def _check_plan_uncached(self, plan: PrecisionPlan) -> CalibrationTable | None:
        if plan.num_layers != self.manifest.num_layers:
            raise ConfigurationError(f"plan covers {plan.num_layers} layers, model has {self.manifest.num_layers}")
        need = plan.required_sites()
        if not need:
            return self.calibration
        if self.calibration is None:
            raise CalibrationError("plan quantizes layers but the archive has no calibration table; "
                                   f"missing sites: {', '.join(sorted(need))}")
        self.calibration.require_all(need)
        return self.calibration

    def calibrate(self, encoded_inputs) -> CalibrationTable:
        from .calibrate import calibrate_engine
        return calibrate_engine(self, encoded_inputs)

    # ------------------------------------------------------------ weights
    def weight_scales(self, i: int) -> tuple:
        out = (ctypes.c_double * 6)()
        _lib.check(self._lib.samp_weight_scales(self._h, i, out))
        return tuple(out)

    def quantized_layer(self, i: int) -> QuantizedLayerWeights:
        with self._lock:
            if i not in self._quantized:
                keys = layer_keys(i)
                t = self.archive.tensors
                s = self.weight_scales(i)
                names = ("qw", "kw", "vw", "ow", "w1", "w2")
                qs = [QuantScale(keys[n], float(np.max(np.abs(t[keys[n]])))) for n in names]
                codes = [quantize(t[keys[n]], sc, site=keys[n]) for n, sc in zip(names, s)]
                self._quantized[i] = QuantizedLayerWeights(
                    np.ascontiguousarray(np.concatenate(codes[:3], axis=1)), tuple(qs[:3]),
                    codes[3], qs[3], codes[4], qs[4], codes[5], qs[5])
            return self._quantized[i]

    def encode_text(self, text_a: str, text_b: str | None = None) -> EncodedInput:
        return encode_text(self.vocab, text_a, text_b)

    # ------------------------------------------------------------ forward
    def _head_kind(self) -> int:
        return HEAD_TAG if self.manifest.task == "sequence_labeling" else HEAD_CLASSIFY

    @staticmethod
    def _validate(enc: EncodedInput, m) -> None:
        """reference embed_fused input checks (encoder.py:254-261), same messages."""
        ids = np.asarray(enc.token_ids)
        segs = np.asarray(enc.segment_ids)
        if ids.size == 0:
            raise InputError("empty token id sequence")
        if ids.min() < 0 or ids.max() >= m.vocab_size:
            raise InputError(f"token id out of range [0, {m.vocab_size})")
        if segs.size != ids.size:
            raise InputError("segment ids and token ids differ in length")
        if segs.min() < 0 or segs.max() >= m.type_vocab_size:
            raise InputError(f"segment id out of range [0, {m.type_vocab_size})")
        if len(ids) > m.max_position:
            raise InputError(f"sequence length {len(ids)} exceeds max_position {m.max_position}")

    def pack(self, encs):
        """Pack EncodedInputs back to back: (seq_start, att_len, ids, segs) int32 arrays."""
        lens = np.array([len(e.token_ids) for e in encs], dtype=np.int64)
        seq_start = np.zeros(len(encs) + 1, dtype=np.int32)
        seq_start[1:] = np.cumsum(lens)
        att = np.array([e.attention_length for e in encs], dtype=np.int32)
        ids = np.concatenate([np.asarray(e.token_ids, dtype=np.int32) for e in encs])
        segs = np.concatenate([np.asarray(e.segment_ids, dtype=np.int32) for e in encs])
        return seq_start, att, ids, segs

    def _trace(self, plan: PrecisionPlan, seq_start) -> None:
        tr = _trace.active()
        if tr is not None:
            m = self.manifest
            for s in range(len(seq_start) - 1):
                _trace.record_forward(tr, plan.layer_precisions, int(seq_start[s + 1] - seq_start[s]),
                                      m.hidden, m.num_heads, m.intermediate)

    def forward_packed(self, plan: PrecisionPlan, seq_start, att_len, ids, segs, *, hidden=True,
                       head: int | None = None) -> BatchOutput:
        """One samp_forward call over packed host arrays (validated by the library).  The
        plan check, the calibration push and the forward run under one lock, so another
        thread's table change cannot interleave with them."""
        with self._lock:
            return self._forward_packed_locked(plan, seq_start, att_len, ids, segs, hidden, head)

    def _forward_packed_locked(self, plan, seq_start, att_len, ids, segs, hidden, head) -> BatchOutput:
        self.check_plan(plan)
        self._trace(plan, seq_start)
        self._push_calibration()
        m = self.manifest
        nseq = len(seq_start) - 1
        T = int(seq_start[-1])
        head = self._head_kind() if head is None else head
        rows = nseq if head == HEAD_CLASSIFY else T
        hid = np.empty((T, m.hidden), np.float32) if hidden else None
        logits = probs = labels = None
        if head != HEAD_NONE:
            logits = np.empty((rows, m.num_labels), np.float32)
            probs = np.empty((rows, m.num_labels), np.float32)
            labels = np.empty(rows, np.int32)
        out = _lib.Outputs(hid.ctypes.data if hid is not None else None,
                           logits.ctypes.data if logits is not None else None,
                           probs.ctypes.data if probs is not None else None,
                           labels.ctypes.data if labels is not None else None, head)
        seq_start = np.ascontiguousarray(seq_start, dtype=np.int32)
        att_len = np.ascontiguousarray(att_len, dtype=np.int32)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        segs = np.ascontiguousarray(segs, dtype=np.int32)
        _lib.check(self._lib.samp_forward(self._h, plan.codes(), nseq, seq_start.ctypes.data,
                                          att_len.ctypes.data, ids.ctypes.data, segs.ctypes.data,
                                          IO_HOST, ctypes.byref(out), None))
        return BatchOutput(seq_start, hid, logits, probs, labels)

    def run(self, enc: EncodedInput, plan: PrecisionPlan, capture_taps: bool = False) -> EncoderOutput:
        """Run the full encoder stack under ``plan`` (reference encoder.py:472-530)."""
        self.check_plan(plan)
        self._validate(enc, self.manifest)
        if capture_taps:
            out = self.run_batch_taps([enc], plan)
            return EncoderOutput(hidden_states=out[0][0], taps=out[0][1], head=None)
        seq_start, att, ids, segs = self.pack([enc])
        res = self.forward_packed(plan, seq_start, att, ids, segs)
        head = None
        if res.logits is not None:
            head = {"logits": res.logits, "probs": res.probs, "labels": res.labels,
                    "kind": self._head_kind(), "archive": id(self.archive)}
        return EncoderOutput(hidden_states=res.hidden_states, taps=None, head=head)

    def encode_batch(self, texts_a, texts_b=None, threads: int | None = None):
        """Tokenize many texts at once on the native multi-threaded tokenizer (rows padded
        to the vocab's max_seq_len, as encode_text).  Returns packed (seq_start, att_len,
        ids, segs) for forward_packed."""
        from .tokenization import encode_batch
        ids, segs, att = encode_batch(self.vocab, texts_a, texts_b, threads)
        n, L = ids.shape
        seq_start = (np.arange(n + 1, dtype=np.int32) * L).astype(np.int32)
        return seq_start, att, ids.reshape(-1), segs.reshape(-1)

    def run_texts(self, plan: PrecisionPlan, texts_a, texts_b=None, hidden: bool = False,
                  head: int | None = None) -> BatchOutput:
        """Raw text -> device head results in one call: native tokenizer + one forward."""
        return self.forward_packed(plan, *self.encode_batch(texts_a, texts_b), hidden=hidden, head=head)

    def run_batch(self, encs, plan: PrecisionPlan, hidden: bool = True, head: int | None = None) -> BatchOutput:
        """Batched, padding-free Engine.run over many EncodedInputs (one device call)."""
        for e in encs:
            self._validate(e, self.manifest)
        return self.forward_packed(plan, *self.pack(encs), hidden=hidden, head=head)

    def run_batch_taps(self, encs, plan: PrecisionPlan) -> list:
        """[(hidden_states, taps)] per sequence: one device forward with every activation
        site's F32 value captured (reference Engine.run(..., capture_taps=True),
        encoder.py:472-530 / _tap :238-240).  Sites and shapes as the reference: [S, H]
        (ffn.mid [S, I]), softmax [heads, S, S].  INT8-chain sites are bit-exact; sites on
        the FP16 tensor-core path carry its tolerance."""
        for e in encs:
            self._validate(e, self.manifest)
        m = self.manifest
        seq_start, att, ids, segs = self.pack(encs)
        with self._lock:
            self.set_capture(2)
            try:
                res = self._forward_packed_locked(plan, seq_start, att, ids, segs, True, HEAD_NONE)
                got = {}
                for site in activation_sites(m.num_layers):
                    size = ctypes.c_size_t()
                    name = ("tap:" + site).encode()
                    if self._lib.samp_fetch_stage(self._h, name, -1, None, 0, ctypes.byref(size)) != 0:
                        continue
                    buf = np.empty(size.value // 4, np.float32)
                    _lib.check(self._lib.samp_fetch_stage(self._h, name, -1, buf.ctypes.data, buf.nbytes,
                                                          ctypes.byref(size)))
                    got[site] = buf
            finally:
                self.set_capture(0)
        out = []
        sq = 0
        for s, enc in enumerate(encs):
            r0, r1 = int(seq_start[s]), int(seq_start[s + 1])
            S = r1 - r0
            taps = {}
            for site, buf in got.items():
                if site.endswith(".softmax"):
                    n = m.num_heads * S * S
                    taps[site] = buf[sq:sq + n].reshape(m.num_heads, S, S).copy()
                else:
                    w = m.intermediate if site.endswith(".ffn.mid") else m.hidden
                    taps[site] = buf.reshape(-1, w)[r0:r1].copy()
            sq += m.num_heads * S * S
            out.append((res.hidden_states[r0:r1].copy(), taps))
        return out

    # ------------------------------------------------------------ analyze-quant
    def code_usage(self, encs, plan: PrecisionPlan) -> dict:
        """{site: CodeUsageReport} summed over ``encs`` for every site ``plan`` quantizes:
        one device forward with histogram taps on the INT8 codes the kernels write (the
        reference's tap -> quantize -> code_usage loop, cli.py:284-292)."""
        for e in encs:
            self._validate(e, self.manifest)
        seq_start, att, ids, segs = self.pack(encs)
        sites = activation_sites(self.manifest.num_layers)
        counts = np.zeros((len(sites), 256), np.uint64)
        with self._lock:
            self.check_plan(plan)
            self._push_calibration()
            _lib.check(self._lib.samp_code_usage(self._h, plan.codes(), len(encs), seq_start.ctypes.data,
                                                 att.ctypes.data, ids.ctypes.data, segs.ctypes.data,
                                                 counts.ctypes.data))
        need = plan.required_sites()
        return {s: CodeUsageReport(s, [int(c) for c in counts[k]])
                for k, s in enumerate(sites) if s in need}

    def analyze_quant(self, encs, plan: PrecisionPlan, sites: str = "*") -> dict:
        """reference cli.cmd_analyze_quant (cli.py:269-292) minus the CLI: per-site code
        usage over ``encs`` for the sites matching the fnmatch filter, in sorted order."""
        import fnmatch
        if plan.quantized_layer_count == 0:
            raise ConfigurationError("analyze-quant needs at least one quantized layer")
        self.check_plan(plan)
        names = sorted(plan.required_sites())
        selected = [s for s in names if fnmatch.fnmatch(s, sites)]
        if not selected:
            raise InputError(f"site filter {sites!r} matches nothing; valid sites: {', '.join(names)}")
        usage = self.code_usage(encs, plan)
        return {s: usage[s] for s in selected}

    # ------------------------------------------------------------ debug / parity
    def set_capture(self, on) -> None:
        """0 off, 1 (True) stage buffers for teacher-forced checks, 2 stages + F32 site taps."""
        _lib.check(self._lib.samp_set_capture(self._h, int(on)))

    def fetch_stage(self, name: str, layer: int, dtype, shape) -> np.ndarray:
        size = ctypes.c_size_t()
        _lib.check(self._lib.samp_fetch_stage(self._h, name.encode(), layer, None, 0, ctypes.byref(size)))
        buf = np.empty(size.value, np.uint8)
        _lib.check(self._lib.samp_fetch_stage(self._h, name.encode(), layer, buf.ctypes.data, buf.nbytes,
                                              ctypes.byref(size)))
        return buf.view(dtype).reshape(shape)

    def last_launch_count(self) -> int:
        return int(self._lib.samp_last_launch_count(self._h))

    @property
    def handle(self):
        return self._h
