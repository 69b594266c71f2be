/*
 * samp_b200 — C ABI of the B200-native SAMP mixed-precision encoder.
 *
 * The reference has no FFI: its hot path is the Python API
 *   Engine(archive, fp16_storage)            reference pkg/src/samp/encoder.py:424-431
 *   Engine.run(enc, plan, capture_taps)      reference pkg/src/samp/encoder.py:472-530
 *   Engine.quantized_layer / check_plan      reference pkg/src/samp/encoder.py:437-470
 *   classify / tag                           reference pkg/src/samp/tasks.py:28-55
 *   Engine.calibrate                         reference pkg/src/samp/encoder.py:446-454
 * Every entry point below is what that API binds to in paper_2209_09130_b200
 * (Python ctypes, _lib.py); INTEGRATION.md shows the binding a maintainer of
 * the reference would add.  Plain pointers and sizes only; no torch types.
 *
 * Errors: every call returns SAMP_OK or one SAMP_E_* code that maps 1:1 onto
 * the reference's exception classes (errors.py:4-41); the message is in
 * samp_last_error() (thread-local).  All validation happens before any
 * device work, as in the reference.
 *
 * Threading (reference: one Engine shared across threads, encoder.py:431,437-441;
 * results bitwise thread-independent, tests/test_encoder.py:340-350): every entry point
 * taking a samp_engine* holds that engine's (recursive) mutex for the whole call, so
 * calls on one engine are serialised — a calibration change can never interleave with
 * a forward that is reading scales or replaying a captured graph.  Different engines
 * run concurrently.  samp_engine_destroy must not race other calls on the same engine.
 */
#ifndef SAMP_B200_H
#define SAMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exception classes */
#define SAMP_OK              0
#define SAMP_E_DIMENSION     1  /* DimensionError      */
#define SAMP_E_CONFIGURATION 2  /* ConfigurationError  */
#define SAMP_E_CALIBRATION   3  /* CalibrationError    */
#define SAMP_E_INPUT         4  /* InputError          */
#define SAMP_E_DEVICE        5  /* (new) CUDA failure / no B200 */
#define SAMP_E_INTERNAL      6

/* per-layer precision codes (reference encoder.py:50-52 + MHA-only extension) */
#define SAMP_LAYER_FP        0  /* "FP"             */
#define SAMP_LAYER_FFN_INT8  1  /* "FFN_ONLY_INT8"  */
#define SAMP_LAYER_FULL_INT8 2  /* "FULL_INT8"      */
#define SAMP_LAYER_MHA_INT8  3  /* "MHA_ONLY_INT8"  (extension) */

/* heads (reference tasks.py) */
#define SAMP_HEAD_NONE     0
#define SAMP_HEAD_CLASSIFY 1    /* pooled [CLS] tanh pooler + classifier + softmax + argmax */
#define SAMP_HEAD_TAG      2    /* per-token classifier + softmax + argmax */

/* samp_forward io flags */
#define SAMP_IO_HOST   0        /* ids/segs/outputs are host pointers (copies inside the call) */
#define SAMP_IO_DEVICE 1        /* ids/segs/outputs are device pointers on the engine's GPU   */

typedef struct samp_engine samp_engine;

typedef struct samp_model_desc {
  int32_t num_layers, hidden, num_heads, intermediate;
  int32_t vocab_size, max_position, type_vocab_size, num_labels;
  double layernorm_eps;
  int32_t fp16_storage;     /* reference Engine(fp16_storage=...) */
} samp_model_desc;

typedef struct samp_outputs {
  float* hidden;    /* [T][hidden] final hidden states, or NULL */
  float* logits;    /* CLASSIFY: [nseq][num_labels]; TAG: [T][num_labels]; or NULL */
  float* probs;     /* same shape as logits, or NULL */
  int32_t* labels;  /* CLASSIFY: [nseq]; TAG: [T]; or NULL */
  int32_t head;     /* SAMP_HEAD_* */
} samp_outputs;

const char* samp_last_error(void);
int samp_device_check(int device);       /* SAMP_OK if `device` is an sm_100 GPU */

/* Engine(archive) — replaces reference encoder.py:424-431 */
int samp_engine_create(const samp_model_desc* desc, int device, samp_engine** out);
void samp_engine_destroy(samp_engine* e);

/* weight upload from the archive layout (F32, matrices (in, out) row-major,
 * reference archive.py:95-134); INT8 copies use quantize_weight (encoder.py:191-194) */
int samp_load_embeddings(samp_engine* e, const float* word, const float* position, const float* token_type,
                         const float* ln_gamma, const float* ln_beta);
/* t[16] = qw qb kw kb vw vb ow ob attn_ln_g attn_ln_b w1 b1 w2 b2 ffn_ln_g ffn_ln_b */
int samp_load_layer(samp_engine* e, int layer, const float* const* t);
int samp_load_heads(samp_engine* e, const float* pooler_w, const float* pooler_b,
                    const float* head_w, const float* head_b);
/* per-tensor INT8 weight scales the engine derived (encoder.py:191-225):
 * out[6] = s_qw, s_kw, s_vw, s_ow, s_w1, s_w2 */
int samp_weight_scales(samp_engine* e, int layer, double* out6);

/* calibration table -> site scales (quantization.py:72-80); site names as encoder.py:60-83 */
int samp_set_site_amax(samp_engine* e, const char* site, double amax);
int samp_clear_calibration(samp_engine* e);

/* Engine.run over a packed batch of nseq sequences.
 *   layer_prec[num_layers]: SAMP_LAYER_* (validated like PrecisionPlan + check_plan)
 *   seq_start[nseq+1] (host): packed row offsets; sequence s owns rows
 *       [seq_start[s], seq_start[s+1]) (its full, possibly padded, length)
 *   att_len[nseq] (host): non-pad prefix length (reference EncodedInput.attention_length)
 *   ids, segs [T]: token / segment ids (host or device per io)
 *   stream: cudaStream_t or NULL for the engine's stream */
int samp_forward(samp_engine* e, const uint8_t* layer_prec, int32_t nseq, const int32_t* seq_start,
                 const int32_t* att_len, const int32_t* ids, const int32_t* segs, int32_t io,
                 const samp_outputs* out, void* stream);

/* Engine.calibrate (encoder.py:446-454): all-FP forward of the packed batch (host arrays)
 * with max|x| taps at the 1 + 8L activation sites; amax_out[1 + 8L] in activation_sites
 * order (embed.out, then per layer attn.in q k v softmax out_in ffn.in ffn.mid).  FP16
 * tensor-core arithmetic: amax agree with the reference's FP32 calibration to ~1e-3. */
int samp_calibrate(samp_engine* e, int32_t nseq, const int32_t* seq_start, const int32_t* att_len,
                   const int32_t* ids, const int32_t* segs, double* amax_out);

/* analyze-quant code usage (replaces the tap + quantize + code_usage loop of
 * cli.py:284-292 / quantization.py:190-193): one forward of the packed batch (host arrays)
 * under layer_prec with histogram taps on the INT8 codes the kernels write;
 * counts[(1 + 8L) * 256] (activation_sites order, index code + 128) are overwritten.
 * Sites the plan keeps in floating point read zero.  Codes are bit-exact with the
 * reference's, so the histograms equal its per-site code_usage sums. */
int samp_code_usage(samp_engine* e, const uint8_t* layer_prec, int32_t nseq, const int32_t* seq_start,
                    const int32_t* att_len, const int32_t* ids, const int32_t* segs,
                    unsigned long long* counts);

/* Exact FP32 layers (Engine(exact_fp32=True)): the FP blocks (mha_fp / ffn_fp,
 * encoder.py:276-330 — FP plans, FFN_ONLY's attention, MHA-only's FFN) run the reference's
 * k-ordered FP32 GEMMs (kernels.py:48-71, 188-200) on the FP32 pipe instead of the FP16
 * tensor cores, so every plan's hidden states are bit-exact with the reference (and
 * Engine.calibrate equals its FP32 calibration).  Off by default (FP16 tensor cores). */
int samp_set_exact_fp32(samp_engine* e, int on);

/* CUDA-graph replay of the forward per (plan, batch geometry, head): on by default;
 * a key is captured on its second use and replayed afterwards */
int samp_set_graphs(samp_engine* e, int on);

/* synchronise the engine's stream */
int samp_sync(samp_engine* e);

/* Debug/parity: after samp_forward with samp_set_capture(e, 1), copy the named
 * stage buffer of `layer` (names in DESIGN.md: in_q, qkv_q, ctx_q, ffn_in_q, mid_q,
 * out_q, out_f32, embed_f32, ...) to host; *bytes receives the size.
 * samp_set_capture(e, 2) also records Engine.run(..., capture_taps=True)'s taps
 * (reference encoder.py:238-240 _tap; sites :294-311, :324-327, :360-379, :407-417):
 * stage "tap:<site>" at layer -1 holds the site's F32 values for the packed batch,
 * [T][H] ([T][I] for L.ffn.mid), and L.attn.softmax as each sequence's [heads][S][S]
 * in batch order.  INT8-chain sites are bit-exact with the reference. */
int samp_set_capture(samp_engine* e, int on);
int samp_fetch_stage(samp_engine* e, const char* name, int layer, void* dst, size_t capacity, size_t* bytes);

/* kernel-level parity entry points (host pointers; allocate + copy internally).
 * B is given in the reference layout [k][n] row-major (activation @ weight). */
int samp_debug_gemm_i8(const int8_t* a, const int8_t* b, int32_t* c, int m, int n, int k);
int samp_debug_gemm_f16(const uint16_t* a, const uint16_t* b, float* c, int m, int n, int k);
/* main-loop ceiling of the repo's tcgen05 GEMM (plain accumulator store, device-resident
 * operands): kind 0 = kind::i8, 1 = kind::f16; *ms = average of `iters` launches */
int samp_debug_gemm_peak(int kind, int m, int n, int k, int iters, float* ms);

/* Native multi-threaded host tokenizer (the paper's C++ tokenizer feeding the packed
 * varlen batch; replaces the reference's per-text tokenization.encode loop, cli.py:375-377,
 * SPEC.md:230-286).  tokens[i] is the UTF-8 token of id i.  Returns NULL when a special
 * token is missing or max_seq_len < 3 (callers use the Python encoder then). */
typedef struct samp_tokenizer samp_tokenizer;
samp_tokenizer* samp_tokenizer_create(const char* const* tokens, int ntokens, int do_lower_case, int max_seq_len,
                                      int char_mode);
void samp_tokenizer_destroy(samp_tokenizer* tok);
/* Encode n texts (text_b NULL or per-item NULL for single texts) into padded rows
 * ids/segs[n][max_seq_len], att[n] on nthreads threads.  Items with non-ASCII bytes are
 * flagged fallback[i] = 1 and left to the caller (Unicode normalisation); returns their
 * count. */
int samp_tokenize_batch(samp_tokenizer* tok, const char* const* text_a, const char* const* text_b, int n,
                        int nthreads, int32_t* ids, int32_t* segs, int32_t* att, uint8_t* fallback);

/* numerics validation: exhaustive (all 2^32 inputs) comparisons of the branch-free
 * quantize / divide / exp used by the kernels against their IEEE-divide formulations,
 * and device evaluation of fn 0 = numpy exp, 1 = numpy (SVML) tanh, 2 = reference GELU */
int samp_debug_quant_exhaustive(const float* scales, int n, unsigned long long* mismatches);
int samp_debug_div_exhaustive(const float* divisors, int n, unsigned long long* mismatches);
int samp_debug_exp_exhaustive(unsigned long long* mismatches);
/* gelu8_finite (FFN1 epilogue fast path) vs the general numpy-exact GELU, all |x| < 1e12 */
int samp_debug_gelu_finite_exhaustive(unsigned long long* mismatches);
/* softmax fast exp (FFMA2, exponent add) vs numpy exp over [-86.5, 0]: mismatches[0] unrefined, [1] refined reciprocal */
int samp_debug_exp2_fast_exhaustive(unsigned long long* mismatches);
/* FFN1 fast GELU epilogue admission check for one ffn.mid scale (every float |x| < 1e12):
 * counts[0] = unflagged elements whose fast code differs from the exact one (0 = admitted),
 * counts[1] = flagged elements (recomputed exactly by the kernel).  Replaces nothing in the
 * reference: it proves GELU_FAST equal to quantize(gelu(x), s) (encoder.py:406-410). */
int samp_debug_gelu_fast_check(float s, unsigned long long* counts);
int samp_debug_unary(int fn, const float* x, float* y, long n);

/* number of kernel launches issued by the last samp_forward (for bench gpu_launches) */
int samp_last_launch_count(samp_engine* e);

/* per-kernel device timing: with profiling on (1), every launch is bracketed by CUDA events
 * on the engine stream; samp_profile_report syncs and writes {"kernel": [total_ms, n], ...}.
 * 2: in-kernel phase stamps only (samp_debug_gemm_stamps), kernels launched back to back
 * with PDL as in a normal forward (no graph, no events): the cross-kernel timeline. */
int samp_set_profiling(samp_engine* e, int on);
/* GEMM phase stamps (profiling mode only): samp_debug_gemm_stamps(e, n) records, for the
 * next n GEMM launches, per CTA 8 u64 = {smid, t_start, t_first_slot_full, t_last_slot_full,
 * t_accumulator_done, t_epilogue_done, t_exit, 0} (%globaltimer ns), 1024 CTAs per launch;
 * _fetch copies them out with the launch names ('\n'-separated) and resets the list. */
int samp_debug_gemm_stamps(samp_engine* e, int max_launches);
int samp_debug_gemm_stamps_fetch(samp_engine* e, unsigned long long* out, int cap_launches, char* names,
                                 size_t names_cap, int* n_launches);
int samp_profile_report(samp_engine* e, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif
#endif /* SAMP_B200_H */
