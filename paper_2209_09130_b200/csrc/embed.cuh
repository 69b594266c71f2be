// Fused embedding: word + position + token-type gather, LayerNorm, optional
// f16 storage rounding, optional INT8 quantize at embed.out.
// Reference: encoder.embed_fused (pkg/src/samp/encoder.py:249-273) and the first
// FULL_INT8 layer's quantize (encoder.py:505-510).
//
// One 8-lane group per token (4 tokens per warp, 32 per 256-thread block).
//   gather:  the group sums ((word + pos) + type) in reference order with float4 loads
//            (all rows of the block in flight at once) into a padded smem row;
//   LN:      numpy's pairwise tree over H, cooperatively: inside a leaf, lane j owns the
//            j-th of the 8 strided accumulators (exactly numpy's r[j] chains), the
//            ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) combine is an xor-butterfly (IEEE add is
//            commutative, the pairing is numpy's), tails and the tree above the leaves are
//            evaluated identically by all 8 lanes;
//   emit:    normalise + every requested output.
#pragma once
#include <cuda_fp16.h>

#include "numerics.cuh"

namespace samp {

constexpr int EMB_TOK = 32;        // tokens per block
constexpr int EMB_THREADS = 256;   // 8 lanes per token
constexpr int EMB_PAD = 8;         // row padding (floats): groups of a warp hit distinct banks

struct EmbedParams {
  const int* ids;
  const int* segs;
  const int* pos;           // position of each packed token within its sequence
  const float* word;        // [V][H]
  const float* position;    // [P][H]
  const float* token_type;  // [2][H]
  const float* gamma;
  const float* beta;
  float eps;
  int hidden;
  int T;
  int f16_round;            // reference Engine(fp16_storage=True): round the F32 output
  float* out_f32;           // [T][H] or null
  __half* out_f16;          // [T][H] or null
  int8_t* out_i8;           // [T][H] or null
  float s_out;              // F32(scale(embed.out)) for out_i8
};

// numpy pairwise sum of v(i), i in [0, n), evaluated by an 8-lane group (lane j = g)
template <class V>
__device__ __forceinline__ float pw_leaf_coop8(int lo, int n, int g, V& v) {
  if (n < 8) {
    float r = 0.0f;
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, v(lo + i));
    return r;
  }
  const int body = n - (n & 7);
  float acc = v(lo + g);
  for (int i = 8 + g; i < body; i += 8) acc = __fadd_rn(acc, v(lo + i));
  acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
  acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
  acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
  for (int i = body; i < n; ++i) acc = __fadd_rn(acc, v(lo + i));
  return acc;
}

template <class V>
__device__ __forceinline__ float pairwise_coop8(int n, int g, V& v) {
  if (n <= 128) return pw_leaf_coop8(0, n, g, v);
  int lo_s[12], n_s[12];
  float left[12];
  bool is_right[12];
  int d = 0;
  lo_s[0] = 0;
  n_s[0] = n;
  is_right[0] = false;
  for (;;) {
    while (n_s[d] > 128) {
      lo_s[d + 1] = lo_s[d];
      n_s[d + 1] = pw_split(n_s[d]);
      is_right[d + 1] = false;
      ++d;
    }
    float x = pw_leaf_coop8(lo_s[d], n_s[d], g, v);
    while (d > 0 && is_right[d]) {
      --d;
      x = __fadd_rn(left[d], x);
    }
    if (d == 0) return x;
    left[d - 1] = x;
    const int pp = d - 1, n2 = pw_split(n_s[pp]);
    lo_s[d] = lo_s[pp] + n2;
    n_s[d] = n_s[pp] - n2;
    is_right[d] = true;
  }
}

#ifdef SAMP_DEFINE_KERNELS  // kernel bodies live in misc_kernels.cu only
static __global__ void __launch_bounds__(EMB_THREADS) embed_kernel(const EmbedParams p) {
  extern __shared__ float xs[];              // [EMB_TOK][H + EMB_PAD]
  const int H = p.hidden, ld = H + EMB_PAD;
  const int tok = threadIdx.x >> 3, g = threadIdx.x & 7;
  const int t = blockIdx.x * EMB_TOK + tok;
  const bool live = t < p.T;
  float* row = xs + tok * ld;
  if (live) {
    const float* w = p.word + size_t(p.ids[t]) * H;
    const float* ps = p.position + size_t(p.pos[t]) * H;
    const float* ty = p.token_type + size_t(p.segs[t]) * H;
#pragma unroll 4
    for (int c = g * 4; c < H; c += 32) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(w + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(ps + c));
      const float4 d = __ldg(reinterpret_cast<const float4*>(ty + c));
      row[c] = __fadd_rn(__fadd_rn(a.x, b.x), d.x);
      row[c + 1] = __fadd_rn(__fadd_rn(a.y, b.y), d.y);
      row[c + 2] = __fadd_rn(__fadd_rn(a.z, b.z), d.z);
      row[c + 3] = __fadd_rn(__fadd_rn(a.w, b.w), d.w);
    }
  }
  __syncwarp();
  // every lane of the warp runs the (token-uniform) tree; dead tokens read zeros
  auto vx = [&](int i) { return live ? row[i] : 0.0f; };
  const float hf = float(H);
  const float mean = __fdiv_rn(__fadd_rn(0.0f, pairwise_coop8(H, g, vx)), hf);
  auto vc = [&](int i) {
    const float d = live ? __fsub_rn(row[i], mean) : 0.0f;
    return __fmul_rn(d, d);
  };
  const float var = __fdiv_rn(__fadd_rn(0.0f, pairwise_coop8(H, g, vc)), hf);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
  if (!live) return;
  const Recip rq = make_recip(p.out_i8 ? p.s_out : 1.0f);
  const size_t base = size_t(t) * H;
  for (int c = g * 4; c < H; c += 32) {
    float y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      y[u] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(row[c + u], mean), inv), __ldg(p.gamma + c + u)),
                       __ldg(p.beta + c + u));
      if (p.f16_round) y[u] = __half2float(__float2half_rn(y[u]));
    }
    if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + base + c) = make_float4(y[0], y[1], y[2], y[3]);
    if (p.out_f16) {
      __half2 h0 = __floats2half2_rn(y[0], y[1]), h1 = __floats2half2_rn(y[2], y[3]);
      *reinterpret_cast<uint2*>(p.out_f16 + base + c) =
          make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
    }
    if (p.out_i8) {
      const uint32_t w = (uint32_t(quant_fast(y[0], rq)) & 0xff) | ((uint32_t(quant_fast(y[1], rq)) & 0xff) << 8) |
                         ((uint32_t(quant_fast(y[2], rq)) & 0xff) << 16) | (uint32_t(quant_fast(y[3], rq)) << 24);
      *reinterpret_cast<uint32_t*>(p.out_i8 + base + c) = w;
    }
  }
}
#endif  // SAMP_DEFINE_KERNELS

}  // namespace samp
