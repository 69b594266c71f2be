// Fused embedding: word + position + token-type gather, LayerNorm, optional
// f16 storage rounding, optional INT8 quantize at embed.out.
// Reference: encoder.embed_fused (pkg/src/samp/encoder.py:249-273) and the first
// FULL_INT8 layer's quantize (encoder.py:505-510).
//
// One warp per token (8 tokens per 256-thread block).
//   gather:  lanes sum ((word + pos) + type) in reference order with float4 loads into a
//            smem row;
//   LN:      numpy's pairwise tree over H (pairwise_warp): the tree's leaves are shared
//            out to four 8-lane groups; inside a leaf lane j owns the j-th of numpy's 8
//            strided accumulators, the ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) combine is an
//            xor-butterfly (IEEE add is commutative, the pairing is numpy's), tails and
//            the tree above the leaves are evaluated identically by every lane;
//   emit:    normalise + every requested output.
#pragma once
#include <cuda_fp16.h>

#include "numerics.cuh"

namespace samp {

constexpr int EMB_THREADS = 256;   // one warp per token, 8 tokens per block

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
  float* amax;              // calibration: amax array (null = off); taps embed.out and L0.attn.in
  int site, site2;
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
// numpy pairwise sum over row[0, H) by a full warp, H compile-time: leaf l is reduced by
// the 8-lane group l % 4 (lane j of the group owns numpy's j-th strided accumulator, the
// xor-butterfly is numpy's ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), tails are added in order),
// then every lane combines the leaf sums up the (compile-time) tree.
template <int H, int LI, int PER, class V>
__device__ __forceinline__ void warp_leaves(float (&mine)[PER], int grp, int g, V& v) {
  if constexpr (LI < ct_leaves(H)) {
    constexpr int lo = ct_leaf_lo(H, LI), len = ct_leaf_n(H, LI);
    constexpr int body = len >= 8 ? len - (len & 7) : 0;
    if (grp == LI % 4) {
      const unsigned m = 0xffu << (8 * (LI % 4));
      float acc = 0.0f;
      if constexpr (len >= 8) {
        acc = v(lo + g);
#pragma unroll
        for (int i = 8; i < body; i += 8) acc = __fadd_rn(acc, v(lo + i + g));
        acc = __fadd_rn(acc, __shfl_xor_sync(m, acc, 1));
        acc = __fadd_rn(acc, __shfl_xor_sync(m, acc, 2));
        acc = __fadd_rn(acc, __shfl_xor_sync(m, acc, 4));
      }
#pragma unroll
      for (int i = body; i < len; ++i) acc = __fadd_rn(acc, v(lo + i));
      mine[LI / 4] = acc;
    }
    warp_leaves<H, LI + 1, PER>(mine, grp, g, v);
  }
}

template <int H, class V>
__device__ __forceinline__ float pairwise_warp(V& v) {
  constexpr int PER = (ct_leaves(H) + 3) / 4;
  const int lane = threadIdx.x & 31;
  float mine[PER];
#pragma unroll
  for (int t = 0; t < PER; ++t) mine[t] = 0.0f;
  warp_leaves<H, 0, PER>(mine, lane >> 3, lane & 7, v);
  auto leafval = [&](int li) { return __shfl_sync(0xffffffffu, mine[li >> 2], (li & 3) * 8); };
  return ct_combine<H, 0>(leafval);
}

// Uniform-leaf fast path: when numpy's tree over H ends in NL equal leaves of LEN (H = 768:
// 8 x 96, 1024: 8 x 128, 512: 4 x 128, 384: 4 x 96), the four 8-lane groups reduce four
// leaves at once (round rd: group q owns leaf 4*rd + q) instead of one group per leaf with
// the other 24 lanes masked off.  The row lives in smem with 8 pad floats after every leaf
// (emb_pad) so the four groups' reads fall in distinct banks.
template <int H>
struct EmbLeaves {
  static constexpr int NL = ct_leaves(H);
  static constexpr int LEN = H / NL;
  static constexpr bool uniform = NL >= 2 && NL <= 8 && H % NL == 0 && LEN % 8 == 0 && pw_splits_evenly(H, NL);
  static constexpr int ROW = uniform ? H + 8 * NL : H;   // smem floats per token row
};
template <int H>
__device__ __forceinline__ int emb_pad(int i) {
  if constexpr (EmbLeaves<H>::uniform) return i + (i / EmbLeaves<H>::LEN) * 8;
  else return i;
}

template <int H, class V>
__device__ __forceinline__ float pairwise_warp_uniform(V& v) {
  using EL = EmbLeaves<H>;
  constexpr int NL = EL::NL, LEN = EL::LEN, ROUNDS = (NL + 3) / 4;
  const int lane = threadIdx.x & 31, grp = lane >> 3, g = lane & 7;
  float mine[ROUNDS];
#pragma unroll
  for (int rd = 0; rd < ROUNDS; ++rd) {
    const int li = rd * 4 + grp;
    const int lo = (li < NL ? li : 0) * LEN;
    float acc = v(lo + g);
#pragma unroll
    for (int i = 8; i < LEN; i += 8) acc = __fadd_rn(acc, v(lo + i + g));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    mine[rd] = acc;
  }
  auto leafval = [&](int li) { return __shfl_sync(0xffffffffu, mine[li >> 2], (li & 3) * 8); };
  return ct_combine<H, 0>(leafval);
}

template <int H>
static __global__ void __launch_bounds__(EMB_THREADS) embed_kernel(const EmbedParams p) {
  extern __shared__ float xs[];              // [8 warps][EmbLeaves<H>::ROW]
  pdl_trigger();
  pdl_wait();                                 // xq / hidden buffers are still read by the previous forward
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * (EMB_THREADS / 32) + warp;
  if (t >= p.T) return;                       // warp-uniform
  float* row = xs + warp * EmbLeaves<H>::ROW;
  {
    const float* w = p.word + size_t(p.ids[t]) * H;
    const float* ps = p.position + size_t(p.pos[t]) * H;
    const float* ty = p.token_type + size_t(p.segs[t]) * H;
#pragma unroll 6
    for (int c = lane * 4; c < H; c += 128) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(w + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(ps + c));
      const float4 d = __ldg(reinterpret_cast<const float4*>(ty + c));
      *reinterpret_cast<float4*>(row + emb_pad<H>(c)) = make_float4(
          __fadd_rn(__fadd_rn(a.x, b.x), d.x), __fadd_rn(__fadd_rn(a.y, b.y), d.y),
          __fadd_rn(__fadd_rn(a.z, b.z), d.z), __fadd_rn(__fadd_rn(a.w, b.w), d.w));
    }
  }
  __syncwarp();
  const float hf = float(H);
  float mean, var;
  if constexpr (EmbLeaves<H>::uniform) {
    // leaf-local index i of leaf li sits at li*(LEN+8) + i: v(lo + i) with lo = li*LEN
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
  const size_t base = size_t(t) * H;
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
      if (p.f16_round) y[u] = __half2float(__float2half_rn(y[u]));
      amx = fmaxf(amx, fabsf(y[u]));
    }
    if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + base + c) = make_float4(y[0], y[1], y[2], y[3]);
    if (p.out_f16) {
      __half2 h0 = __floats2half2_rn(y[0], y[1]), h1 = __floats2half2_rn(y[2], y[3]);
      *reinterpret_cast<uint2*>(p.out_f16 + base + c) =
          make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
    }
    if (p.out_i8) {
      const uint32_t wv = trunc_pack4_s8(quant_pre_fast(y[0], rq), quant_pre_fast(y[1], rq),
                                         quant_pre_fast(y[2], rq), quant_pre_fast(y[3], rq));
      *reinterpret_cast<uint32_t*>(p.out_i8 + base + c) = wv;
    }
  }
  if (p.amax) {
    amax_commit(p.amax + p.site, amx);
    amax_commit(p.amax + p.site2, amx);
  }
}
#endif  // SAMP_DEFINE_KERNELS

}  // namespace samp
