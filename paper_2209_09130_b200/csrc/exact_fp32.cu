// Exact FP32 layers (Engine(exact_fp32=True)): the reference's floating-point blocks
// mha_fp / ffn_fp (pkg/src/samp/encoder.py:276-330) reproduced bit for bit.
//
// The reference's FP32 GEMM is deterministic by design: every output element accumulates
// its k products in k order, one F32 multiply then one F32 add per step, starting from +0
// (kernels.py:48-71, "bitwise equal to the scalar triple loop"); batched_gemm_f32 runs the
// same per head (:188-200).  So an FP32 SIMT kernel that keeps that per-element order — and
// never contracts the multiply-add into an FMA (-fmad=false, explicit __fmul_rn/__fadd_rn) —
// returns the reference's bits on any tiling, and together with the numpy-exact softmax,
// LayerNorm, GELU and f16 rounding of numerics.cuh the FP layers become bit-exact.  This is
// the parity mode: it runs on the FP32 pipe (one FMUL + one FADD per MAC), several times
// slower than the FP16 tensor-core path, which stays the default.
//
//   exact_gemm_kernel      C = A[M][K] x B[K][N] (+ bias) [-> GELU] [-> f16 round]
//   exact_attention_kernel scores (k-ordered dot), * F32(1/sqrt(d)) + mask, softmax,
//                          [f16 round], ctx = k-ordered P.V [f16 round]
//   exact_ln_kernel        LN((acc + b) + residual) [f16 round] -> f32 / int8 codes
// Each folds the calibration amax of the sites it produces (Engine.calibrate in this
// mode equals the reference's FP32 calibration).
#define SAMP_DEFINE_KERNELS
#include "kernels.h"

namespace samp {

// ---------------------------------------------------------------- GEMM
template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) exact_gemm_kernel(const ExactGemmParams p) {
  constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY, BK = 8;
  __shared__ float As[2][BK][BM];
  __shared__ float Bs[2][BK][BN];
  __shared__ TanhTable tt;
  pdl_trigger();
  if (p.gelu) load_tanh_table(&tt, threadIdx.x, NT);
  pdl_wait();
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  constexpr int AL = BM * BK / NT, BL = BK * BN / NT;   // per-thread tile loads
  static_assert(AL >= 1 && BL >= 1 && BM * BK % NT == 0 && BK * BN % NT == 0, "tile loads");
  float ra[AL], rb[BL];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < AL; ++u) {
      const int i = tid + u * NT, r = i / BK, c = i % BK;
      ra[u] = m0 + r < p.M ? p.a[size_t(m0 + r) * p.lda + k0 + c] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < BL; ++u) {
      const int i = tid + u * NT, r = i / BN, c = i % BN;
      rb[u] = p.b[size_t(k0 + r) * p.ldb + n0 + c];
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < AL; ++u) {
      const int i = tid + u * NT;
      As[buf][i % BK][i / BK] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < BL; ++u) {
      const int i = tid + u * NT;
      Bs[buf][i / BN][i % BN] = rb[u];
    }
  };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;   // numpy: out = zeros; out += a*b
  fetch(0);
  stash(0);
  __syncthreads();
  const int nk = p.K / BK;
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) fetch((kt + 1) * BK);   // next tile in flight during this tile's math
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty + i * TY];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
    }
    if (kt + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
  float amx = 0.0f;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = m0 + ty + i * TY;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = n0 + tx + j * TX;
      float x = acc[i][j];
      if (p.bias) x = __fadd_rn(x, p.bias[col]);
      if (p.gelu) x = gelu_ref(x, &tt);
      if (p.f16_round) x = __half2float(__float2half_rn(x));
      p.out[size_t(row) * p.ldo + col] = x;
      amx = fmaxf(amx, fabsf(x));
    }
  }
  // the launcher keeps a tile inside one q|k|v column block: one site per CTA
  if (p.amax) amax_commit(p.amax + p.site + (p.block_cols ? n0 / p.block_cols : 0), amx);
}

// ---------------------------------------------------------------- attention
// one CTA per (query row, head, sequence)
__global__ void __launch_bounds__(128) exact_attention_kernel(const ExactAttnParams p) {
  __shared__ float qs[64];
  __shared__ float xs[ATT_MAX_KEYS];
  __shared__ float es[ATT_MAX_KEYS];
  __shared__ float red[2];
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, head = blockIdx.y, seq = blockIdx.z;
  const int r0 = p.seq_start[seq];
  const int S = p.seq_start[seq + 1] - r0;
  if (row >= S) return;
  const int att = p.att_len[seq];
  const int H = p.hidden, ld = 3 * H, tid = threadIdx.x;
  if (tid < 64) qs[tid] = p.qkv[size_t(r0 + row) * ld + head * 64 + tid];
  __syncthreads();
  // scores = batched_gemm_f32(qh, kh^T): k-ordered over d, from +0
  for (int k = tid; k < S; k += blockDim.x) {
    const float* kr = p.qkv + size_t(r0 + k) * ld + H + head * 64;
    float acc = 0.0f;
#pragma unroll 8
    for (int d = 0; d < 64; ++d) acc = __fadd_rn(acc, __fmul_rn(qs[d], kr[d]));
    // scores * F32(1/sqrt(d)) + mask (encoder.py:299-300)
    xs[k] = __fadd_rn(__fmul_rn(acc, p.mult_scores), k < att ? 0.0f : -10000.0f);
  }
  __syncthreads();
  if (tid == 0) {
    float mx = xs[0];
    for (int k = 1; k < S; ++k) mx = fmaxf(mx, xs[k]);
    red[0] = mx;
  }
  __syncthreads();
  const float mx = red[0];
  for (int k = tid; k < S; k += blockDim.x) es[k] = np_expf(__fsub_rn(xs[k], mx));
  __syncthreads();
  if (tid == 0) {
    auto get8 = [&](int off, float (&v)[8]) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = off + j < S ? es[off + j] : 0.0f;
    };
    red[1] = __fadd_rn(0.0f, pairwise_sum(S, get8));
  }
  __syncthreads();
  const float den = red[1];
  float amx = 0.0f;
  float* prow = p.probs ? p.probs + p.prob_off[seq] + (size_t(head) * S + row) * S : nullptr;
  for (int k = tid; k < S; k += blockDim.x) {
    float v = __fdiv_rn(es[k], den);
    if (p.f16_round) v = __half2float(__float2half_rn(v));
    xs[k] = v;
    amx = fmaxf(amx, v);
    if (prow) prow[k] = v;
  }
  __syncthreads();
  if (p.amax) amax_commit(p.amax + p.site_sm, amx);   // every thread: warp-collective
  // ctx = batched_gemm_f32(probs, vh): k-ordered over the S keys, from +0
  if (tid < 64) {
    const float* v = p.qkv + size_t(r0) * ld + 2 * H + head * 64 + tid;
    float acc = 0.0f;
    for (int k = 0; k < S; ++k) acc = __fadd_rn(acc, __fmul_rn(xs[k], v[size_t(k) * ld]));
    if (p.f16_round) acc = __half2float(__float2half_rn(acc));
    p.ctx[size_t(r0 + row) * H + head * 64 + tid] = acc;
    amx = fabsf(acc);
  } else {
    amx = 0.0f;
  }
  if (p.amax && tid < 64) amax_commit(p.amax + p.site_ctx, amx);
}

// ---------------------------------------------------------------- residual + LayerNorm
constexpr int XLN_THREADS = 256;   // one warp per row

template <int H>
__global__ void __launch_bounds__(XLN_THREADS) exact_ln_kernel(const ExactLnParams p) {
  extern __shared__ float xrow[];   // [8][EmbLeaves<H>::ROW]
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * (XLN_THREADS / 32) + warp;
  if (t >= p.M) return;   // warp-uniform
  float* row = xrow + warp * EmbLeaves<H>::ROW;
  const size_t base = size_t(t) * H;
  for (int c = lane * 4; c < H; c += 128) {
    const float4 a = *reinterpret_cast<const float4*>(p.acc + base + c);
    const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + c));
    const float4 r = *reinterpret_cast<const float4*>(p.res + base + c);
    // add_bias_residual: (proj + b) + x  (encoder.py:308, :328)
    *reinterpret_cast<float4*>(row + emb_pad<H>(c)) =
        make_float4(__fadd_rn(__fadd_rn(a.x, b.x), r.x), __fadd_rn(__fadd_rn(a.y, b.y), r.y),
                    __fadd_rn(__fadd_rn(a.z, b.z), r.z), __fadd_rn(__fadd_rn(a.w, b.w), r.w));
  }
  __syncwarp();
  const float hf = float(H);
  float mean, var;
  if constexpr (EmbLeaves<H>::uniform) {
    auto at = [&](int i) { return row[emb_pad<H>(i)]; };
    auto vx = [&](int i) { return at(i); };
    mean = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp_uniform<H>(vx)), hf);
    auto vc = [&](int i) {
      const float d = __fsub_rn(at(i), mean);
      return __fmul_rn(d, d);
    };
    var = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp_uniform<H>(vc)), hf);
  } else {
    auto vx = [&](int i) { return row[i]; };
    mean = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp<H>(vx)), hf);
    auto vc = [&](int i) {
      const float d = __fsub_rn(row[i], mean);
      return __fmul_rn(d, d);
    };
    var = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp<H>(vc)), hf);
  }
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
  const Recip rq = make_recip(p.out_i8 ? p.s_out : 1.0f);
  float amx = 0.0f;
  for (int c = lane * 4; c < H; c += 128) {
    const float4 xv = *reinterpret_cast<const float4*>(row + emb_pad<H>(c));
    const float4 gv = __ldg(reinterpret_cast<const float4*>(p.gamma + c));
    const float4 bv = __ldg(reinterpret_cast<const float4*>(p.beta + c));
    const float xx[4] = {xv.x, xv.y, xv.z, xv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
    float y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      y[u] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xx[u], mean), inv), gg[u]), bb[u]);
      if (p.f16_round) y[u] = __half2float(__float2half_rn(y[u]));   // before any quantize
      amx = fmaxf(amx, fabsf(y[u]));
    }
    if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + base + c) = make_float4(y[0], y[1], y[2], y[3]);
    if (p.out_i8) {
      *reinterpret_cast<uint32_t*>(p.out_i8 + base + c) =
          trunc_pack4_s8(quant_pre_fast(y[0], rq), quant_pre_fast(y[1], rq), quant_pre_fast(y[2], rq),
                         quant_pre_fast(y[3], rq));
    }
  }
  if (p.amax) amax_commit(p.amax + p.site, amx);
}

// ---------------------------------------------------------------- launchers
template <int BM, int BN, int TM, int TN>
static cudaError_t exact_gemm_cfg(const ExactGemmParams& p, cudaStream_t st) {
  const dim3 grid(p.N / BN, (p.M + BM - 1) / BM);
  return launch_ex(exact_gemm_kernel<BM, BN, TM, TN>, grid, dim3((BM / TM) * (BN / TN)), 0, st, 1, p);
}

cudaError_t launch_exact_gemm(const ExactGemmParams& p, int sms, cudaStream_t st) {
  if (p.N % 64 || p.K % 8 || (p.block_cols && p.block_cols % 64)) return cudaErrorInvalidValue;
  // big tiles when they fill the GPU, small ones otherwise (batch 1: 128 rows)
  if (p.N % 128 == 0 && (!p.block_cols || p.block_cols % 128 == 0) &&
      long((p.M + 127) / 128) * (p.N / 128) >= sms)
    return exact_gemm_cfg<128, 128, 8, 8>(p, st);
  return exact_gemm_cfg<32, 64, 2, 4>(p, st);
}

cudaError_t launch_exact_attention(const ExactAttnParams& p, int max_s, int heads, int nseq, cudaStream_t st) {
  return launch_ex(exact_attention_kernel, dim3(max_s, heads, nseq), dim3(128), 0, st, 1, p);
}

template <int H>
static cudaError_t exact_ln_h(const ExactLnParams& p, cudaStream_t st) {
  constexpr int rows = XLN_THREADS / 32;
  return launch_ex(exact_ln_kernel<H>, dim3((p.M + rows - 1) / rows), dim3(XLN_THREADS),
                   size_t(rows) * EmbLeaves<H>::ROW * sizeof(float), st, 1, p);
}

cudaError_t launch_exact_ln(const ExactLnParams& p, int hidden, cudaStream_t st) {
  switch (hidden) {
    case 64: return exact_ln_h<64>(p, st);
    case 128: return exact_ln_h<128>(p, st);
    case 256: return exact_ln_h<256>(p, st);
    case 384: return exact_ln_h<384>(p, st);
    case 512: return exact_ln_h<512>(p, st);
    case 768: return exact_ln_h<768>(p, st);
    case 1024: return exact_ln_h<1024>(p, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
