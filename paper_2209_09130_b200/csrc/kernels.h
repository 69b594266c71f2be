// Launch wrappers implemented in separate translation units (parallel compile).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "attention.cuh"
#include "embed.cuh"
#include "gemm.cuh"
#include "heads.cuh"
#include "ln_rows.cuh"
#include "qkv_attention.cuh"

namespace samp {

// measurement switch: set and not empty / "0"
inline bool env_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && v[0] && !(v[0] == '0' && v[1] == 0);
}

struct Tiles {
  int bn_qkv, bn_ffn1, bn_ln, cluster_ln;
  int bn_ln_small;   // small batches: LN GEMMs as 8-CTA clusters of H/8 columns (0 = n/a)
};

// gemm_i8.cu
cudaError_t gemm_qkv_i8(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiQKV::Params& p, cudaStream_t st);
// finite: |acc*mult + bias| is bounded well below the GELU overflow (host check)
// exhaustive admission check of the FFN1 fast GELU epilogue for one scale (gemm_i8.cu)
cudaError_t gelu_fast_check(float s, float inv_s, unsigned long long* host_counts /*[2]*/, cudaStream_t st);
cudaError_t gemm_gelu_i8(int bn, int mode, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const EpiGeluQuant::Params& p, cudaStream_t st);
// gemm_ln.cu
// a_mc (optional): the same A with 32-row / 16-row boxes, for A multicast across 4- / 8-CTA
// clusters (SAMP_LN_MCAST)
cudaError_t gemm_ln_i8(const Tiles& t, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                       const EpiResLN::Params& p, cudaStream_t st, const CUtensorMap* a_mc = nullptr);
// small batches: split-K GEMM into an int32 workspace (64-wide tiles, grid z = ksplit)
cudaError_t gemm_splitk_i8(const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb, int ksplit,
                           const EpiSplitKAdd::Params& p, cudaStream_t st);
cudaError_t gemm_ln_f16(const Tiles& t, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiResLN::Params& p, cudaStream_t st);
// gemm_f16.cu
cudaError_t gemm_f16out(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiF16Out::Params& p, cudaStream_t st);
// attention.cu
cudaError_t launch_attention_i8(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                                cudaStream_t st);
cudaError_t launch_attention_f16(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                                 cudaStream_t st);
// qkv_attention.cu: fused INT8 QKV GEMM + attention (every tile S <= 128, H % 128 == 0)
int qa_tpr();   // threads per query row of the fused kernel (SAMP_QA_TPR=2: 2, else 4)
cudaError_t launch_qkv_attention(const CUtensorMap& a, const CUtensorMap& w64, const QAParams& q, int sms,
                                 cudaStream_t st);
// misc_kernels.cu
// L2 weight prefetch (side stream): the byte ranges are prefetched in list order in 32 KB
// chunks with cp.async.bulk.prefetch.L2 (no data reaches the SM)
constexpr int PREFETCH_MAX_RANGES = 128;
struct PrefetchList {
  const void* ptr[PREFETCH_MAX_RANGES];
  unsigned long long bytes[PREFETCH_MAX_RANGES];
  int n;
};
cudaError_t launch_l2_prefetch(const PrefetchList& l, int ctas, cudaStream_t st);
cudaError_t launch_embed(const EmbedParams& p, cudaStream_t st);
cudaError_t launch_ln_rows(const LnRowsParams& p, int hidden, cudaStream_t st);
bool ln_rows_supported(int hidden);
cudaError_t launch_classify(const HeadParams& p, cudaStream_t st);
cudaError_t launch_tag(const HeadParams& p, cudaStream_t st);
cudaError_t launch_pack_weight(const float* w, int K, int N, float scale, int8_t* out_i8, __half* out_f16,
                               int row_off, cudaStream_t st);
cudaError_t launch_transpose_f32(const float* w, int K, int N, float* out, cudaStream_t st);
// capture_taps (taps.cu): F32 site values re-derived next to the fused kernels
struct TapBiasParams {
  const void* acc;        // [M][ld_acc] int32 (kind::i8) or f32 (kind::f16) accumulators
  int acc_f32, ld_acc, M, N;
  const float* bias;      // [N]
  float mult0, mult1, mult2;   // per column block dequant multipliers (int32 accumulators)
  int block_cols;         // > 0: column blocks of this width are separate [M][block_cols] outputs
  int gelu, f16_round;
  float* out;
};
struct TapAttnParams {
  const void* qkv;        // [T][3H] int8 codes or f16 values (the fused QKV output)
  int f16, hidden;
  const int* seq_start;
  const int* att_len;
  float mult_scores, s_softmax, mult_ctx;
  int f16_round;
  float* probs;           // per sequence [heads][S][S] at prob_off[seq]
  const long long* prob_off;
  float* ctx;             // [T][H]
};
// exact FP32 layers (exact_fp32.cu): the reference's FP blocks bit for bit
struct ExactGemmParams {
  const float* a;         // [M][lda]
  int lda;
  const float* b;         // [K][ldb]  (archive (in, out) layout)
  int ldb, M, N, K;
  const float* bias;      // [N] or null
  int gelu, f16_round;
  float* out;             // [M][ldo]
  int ldo;
  float* amax;            // calibration (null = off): site + column block
  int site, block_cols;
};
struct ExactAttnParams {
  const float* qkv;       // [T][3H] f32
  int hidden;
  const int* seq_start;
  const int* att_len;
  float mult_scores;      // F32(1/sqrt(d))
  int f16_round;
  float* ctx;             // [T][H]
  float* probs;           // capture_taps: per sequence [heads][S][S] at prob_off[seq] (or null)
  const long long* prob_off;
  float* amax;
  int site_sm, site_ctx;
};
struct ExactLnParams {
  const float* acc;       // [M][H] projection (no bias)
  const float* bias;
  const float* res;       // [M][H] f32 residual
  const float* gamma;
  const float* beta;
  float eps;
  int M, f16_round;
  float* out_f32;         // or null
  int8_t* out_i8;         // or null: quantize(s_out) of the (rounded) output
  float s_out;
  float* amax;
  int site;
};
cudaError_t launch_exact_gemm(const ExactGemmParams& p, int sms, cudaStream_t st);
cudaError_t launch_exact_attention(const ExactAttnParams& p, int max_s, int heads, int nseq, cudaStream_t st);
cudaError_t launch_exact_ln(const ExactLnParams& p, int hidden, cudaStream_t st);
cudaError_t launch_tap_bias(const TapBiasParams& p, cudaStream_t st);
cudaError_t launch_tap_attention(const TapAttnParams& p, int max_s, int heads, int nseq, cudaStream_t st);
cudaError_t gemm_store_acc(int kind, int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                           void* out, int ldc, cudaStream_t st);
// code-usage tap: bins[256] += histogram of an int8 [rows][cols] matrix (row stride ld)
cudaError_t launch_code_hist(const int8_t* src, int rows, int cols, int ld, unsigned long long* bins,
                             cudaStream_t st);

}  // namespace samp
