// capture_taps on the device: the F32 value at every activation site, as the reference's
// Engine.run(..., capture_taps=True) records it (pkg/src/samp/encoder.py:238-240 _tap,
// taps at :294-311 mha_fp, :324-327 ffn_fp, :360-379 mha_int8, :407-417 ffn_int8, :492-516
// dispatch).  A debug / calibration-analysis path, not the hot path: it re-derives the
// tapped values next to the fused kernels (which emit only codes) from the same operands,
// with the reference's float32 arithmetic in the reference's order:
//   * q/k/v and ffn.mid: the tcgen05 GEMM with a plain accumulator store, then
//     tap_bias_kernel: F32(acc)*F32(s_a*s_b) + bias [-> numpy/SVML GELU] [-> f16 round];
//   * attn.softmax and attn.out_in: tap_attention_kernel recomputes one (sequence, head,
//     query) row per CTA from the q/k/v the fused QKV kernel wrote: integer scores,
//     masked row max, numpy exp, numpy pairwise denominator, IEEE divide, then the context
//     from the quantized probabilities (INT8) or the f32 probabilities (FP16 path);
//   * LayerNorm outputs (ffn.in, attn.in) come from the LN epilogue itself (tap_f32).
// INT8 sites are bit-exact with the reference; FP16-path sites carry the FP16 tensor-core
// tolerance of the values they are derived from.
#include "host_util.h"
#include "kernels.h"

namespace samp {

__global__ void tap_bias_kernel(TapBiasParams p) {
  __shared__ TanhTable tt;
  if (p.gelu) load_tanh_table(&tt, threadIdx.x, blockDim.x);
  __syncthreads();
  const long total = long(p.M) * p.N;
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
    const int row = int(i / p.N), col = int(i % p.N);
    const int blk = p.block_cols ? col / p.block_cols : 0;
    const float mult = blk == 0 ? p.mult0 : blk == 1 ? p.mult1 : p.mult2;
    const size_t a = size_t(row) * p.ld_acc + col;
    float x = p.acc_f32 ? static_cast<const float*>(p.acc)[a]
                        : __fmul_rn(__int2float_rn(static_cast<const int*>(p.acc)[a]), mult);
    x = __fadd_rn(x, p.bias[col]);
    if (p.gelu) x = gelu_ref(x, &tt);
    if (p.f16_round) x = __half2float(__float2half_rn(x));
    // block_cols: each column block (q | k | v site) is its own contiguous [M][block_cols]
    if (p.block_cols)
      p.out[size_t(blk) * p.M * p.block_cols + size_t(row) * p.block_cols + (col - blk * p.block_cols)] = x;
    else
      p.out[size_t(row) * p.N + col] = x;
  }
}

// one CTA per (query row, head, sequence); 128 threads
__global__ void __launch_bounds__(128) tap_attention_kernel(TapAttnParams p) {
  __shared__ float xs[ATT_MAX_KEYS];
  __shared__ float ps[ATT_MAX_KEYS];
  __shared__ int pq[ATT_MAX_KEYS];
  __shared__ float red[2];
  const int row = blockIdx.x, head = blockIdx.y, seq = blockIdx.z;
  const int r0 = p.seq_start[seq];
  const int S = p.seq_start[seq + 1] - r0;
  if (row >= S) return;
  const int att = p.att_len[seq];
  const int H = p.hidden, ld = 3 * H;
  const int tid = threadIdx.x;
  // scores: (Q.K^T)*m + mask  (INT8: exact int32 dot; FP16 path: f32 from the f16 q/k)
  for (int k = tid; k < S; k += blockDim.x) {
    float x;
    if (p.f16) {
      const __half* q = static_cast<const __half*>(p.qkv) + size_t(r0 + row) * ld + head * 64;
      const __half* kk = static_cast<const __half*>(p.qkv) + size_t(r0 + k) * ld + H + head * 64;
      float acc = 0.0f;
      for (int d = 0; d < 64; ++d) acc = __fadd_rn(acc, __fmul_rn(__half2float(q[d]), __half2float(kk[d])));
      x = __fmul_rn(acc, p.mult_scores);
    } else {
      const int8_t* q = static_cast<const int8_t*>(p.qkv) + size_t(r0 + row) * ld + head * 64;
      const int8_t* kk = static_cast<const int8_t*>(p.qkv) + size_t(r0 + k) * ld + H + head * 64;
      int acc = 0;
      for (int d = 0; d < 64; ++d) acc += int(q[d]) * int(kk[d]);
      x = __fmul_rn(__int2float_rn(acc), p.mult_scores);
    }
    xs[k] = __fadd_rn(x, k < att ? 0.0f : -10000.0f);
  }
  __syncthreads();
  if (tid == 0) {
    float mx = xs[0];
    for (int k = 1; k < S; ++k) mx = fmaxf(mx, xs[k]);
    red[0] = mx;
  }
  __syncthreads();
  const float mx = red[0];
  for (int k = tid; k < S; k += blockDim.x) ps[k] = np_expf(__fsub_rn(xs[k], mx));
  __syncthreads();
  if (tid == 0) {
    auto get8 = [&](int off, float (&v)[8]) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = off + j < S ? ps[off + j] : 0.0f;
    };
    red[1] = __fadd_rn(0.0f, pairwise_sum(S, get8));
  }
  __syncthreads();
  const float den = red[1];
  float* prow = p.probs + p.prob_off[seq] + (size_t(head) * S + row) * S;
  for (int k = tid; k < S; k += blockDim.x) {
    float v = __fdiv_rn(ps[k], den);
    if (p.f16_round) v = __half2float(__float2half_rn(v));
    prow[k] = v;
    ps[k] = v;
    if (!p.f16) pq[k] = quant_i8(v, p.s_softmax);
  }
  __syncthreads();
  // context: INT8 F32(sum P_q V_q) * F32(s_sm*s_v); FP16 path sum p * v (f32)
  if (tid < 64) {
    float c;
    if (p.f16) {
      const __half* v = static_cast<const __half*>(p.qkv) + size_t(r0) * ld + 2 * H + head * 64 + tid;
      float acc = 0.0f;
      for (int k = 0; k < S; ++k) acc = __fadd_rn(acc, __fmul_rn(ps[k], __half2float(v[size_t(k) * ld])));
      c = acc;
      if (p.f16_round) c = __half2float(__float2half_rn(c));
    } else {
      const int8_t* v = static_cast<const int8_t*>(p.qkv) + size_t(r0) * ld + 2 * H + head * 64 + tid;
      int acc = 0;
      for (int k = 0; k < S; ++k) acc += pq[k] * int(v[size_t(k) * ld]);
      c = __fmul_rn(__int2float_rn(acc), p.mult_ctx);
    }
    p.ctx[size_t(r0 + row) * H + head * 64 + tid] = c;
  }
}

cudaError_t launch_tap_bias(const TapBiasParams& p, cudaStream_t st) {
  const long total = long(p.M) * p.N;
  const int blocks = int(std::min<long>((total + 255) / 256, 148L * 16));
  tap_bias_kernel<<<blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tap_attention(const TapAttnParams& p, int max_s, int heads, int nseq, cudaStream_t st) {
  tap_attention_kernel<<<dim3(max_s, heads, nseq), 128, 0, st>>>(p);
  return cudaGetLastError();
}

// plain accumulator store GEMM over the engine's A / B tensor maps (B box rows = bn)
cudaError_t gemm_store_acc(int kind, int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                           void* out, int ldc, cudaStream_t st) {
  EpiStoreAcc::Params p{out, ldc};
  if (kind == KIND_I8) {
    switch (bn) {
      case 256: return launch_gemm<KIND_I8, 256, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
      case 128: return launch_gemm<KIND_I8, 128, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
      case 64: return launch_gemm<KIND_I8, 64, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
    }
  } else {
    switch (bn) {
      case 256: return launch_gemm<KIND_F16, 256, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
      case 128: return launch_gemm<KIND_F16, 128, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
      case 64: return launch_gemm<KIND_F16, 64, 4, 1, 4, EpiStoreAcc>(a, b, M, N, kb, p, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
