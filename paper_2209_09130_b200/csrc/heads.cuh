// Downstream heads on the final F32 hidden states (reference pkg/src/samp/tasks.py:28-55).
//   classify: pooled = tanh(h[CLS] @ Wp + bp); logits = pooled @ Wh + bh;
//             probs = softmax_rows(logits); label = argmax (lowest index on ties)
//   tag:      logits = h[t] @ Wh + bh per token; softmax; argmax
// The reference's two small products are BLAS sgemm calls (order unspecified), so the
// dot products here are FP32 FMA chains: logits/probs agree within float rounding
// (tests use a tolerance); tanh, exp and the softmax normaliser are numpy-exact.
//
// classify = two launches: pooler_kernel spreads the [B,H]x[H,H] pooler over
// (32-column, 32-sequence, K-split) tiles with every weight load in flight at once;
// classifier_kernel is one CTA per sequence (tanh, label dot products, softmax/argmax).
#pragma once
#include "numerics.cuh"

namespace samp {

constexpr int HEAD_THREADS = 256;
constexpr int HEAD_MAX_LABELS = 64;
constexpr int POOL_COLS = 32;      // output columns per pooler CTA
constexpr int POOL_SEQS = 32;      // sequences per pooler CTA
constexpr int POOL_KSPLIT = 8;     // K splits (grid.z)
constexpr int POOL_MAX_KW = 16;    // K rows per warp: H / POOL_KSPLIT / 8 for H <= 1024

struct HeadParams {
  const float* hidden;     // [T][H]
  const int* seq_start;    // [nseq+1]
  const float* pool_w;     // [H][H] (in, out) — archive layout
  const float* pool_b;     // [H]
  const float* head_wt;    // [L][H] (out, in)
  const float* head_b;     // [L]
  float* pooled;           // [POOL_KSPLIT][nseq][H] scratch (partial pooler sums)
  int hidden_size, num_labels, nseq, T;
  float* logits;           // classify [nseq][L], tag [T][L]
  float* probs;
  int* labels;             // classify [nseq], tag [T]
};

#ifdef SAMP_DEFINE_KERNELS  // kernel bodies live in misc_kernels.cu only
__device__ __forceinline__ float warp_dot(const float* a, const float* b, int n) {
  float acc = 0.0f;
  for (int k = threadIdx.x % 32 * 4; k < n; k += 128) {
    const float4 x = *reinterpret_cast<const float4*>(a + k);
    const float4 y = __ldg(reinterpret_cast<const float4*>(b + k));
    acc = __fmaf_rn(x.x, y.x, acc);
    acc = __fmaf_rn(x.y, y.y, acc);
    acc = __fmaf_rn(x.z, y.z, acc);
    acc = __fmaf_rn(x.w, y.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  return acc;
}

// softmax over one short logit row + argmax (single thread)
__device__ __forceinline__ void softmax_argmax(const float* lg, float* pr, int* label, int L) {
  float mx = -INFINITY;
  for (int l = 0; l < L; ++l) mx = fmaxf(mx, lg[l]);
  float e[HEAD_MAX_LABELS];
  for (int l = 0; l < L; ++l) e[l] = np_expf(__fsub_rn(lg[l], mx));
  auto get = [&](int off, float (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = off + j < L ? e[off + j] : 0.0f;
  };
  const float s = __fadd_rn(0.0f, pairwise_sum(L, get));
  int best = 0;
  float bp = -INFINITY;
  for (int l = 0; l < L; ++l) {
    const float p = __fdiv_rn(e[l], s);
    pr[l] = p;
    if (p > bp) { bp = p; best = l; }
  }
  *label = best;
}

// pooler_kernel: CTA (x, y, z) = 32 output columns x up to 32 sequences x K-split z (of
// POOL_KSPLIT).  The CTA stages its [CLS] slices transposed in smem (hs[k][s]); warp w
// owns H/POOL_KSPLIT/8 K rows and issues all of its Wp loads (lane = column, one
// coalesced 128-byte row slice each) before any FMA, so the kernel is one memory round
// trip plus register FMAs; the 8 warp partials are summed in a fixed order into
// pooled[z][s][j].
static __global__ void __launch_bounds__(HEAD_THREADS) pooler_kernel(const HeadParams p) {
  extern __shared__ float sh[];           // hs [KQ][32] then partials [8][32 seqs][32 cols]
  pdl_trigger();
  const int H = p.hidden_size, KQ = H / POOL_KSPLIT, kw = KQ / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * POOL_COLS + lane;
  const int s0 = blockIdx.y * POOL_SEQS;
  const int k_base = blockIdx.z * KQ;
  const int ns = min(POOL_SEQS, p.nseq - s0);
  float* hs = sh;
  float* part = sh + KQ * POOL_SEQS;
  float wv[POOL_MAX_KW];
#pragma unroll
  for (int i = 0; i < POOL_MAX_KW; ++i)
    wv[i] = i < kw ? __ldg(p.pool_w + size_t(k_base + warp * kw + i) * H + j) : 0.0f;
  pdl_wait();   // weights above are constant: fetched while the last encoder kernel drains
  for (int idx = threadIdx.x; idx < POOL_SEQS * KQ; idx += HEAD_THREADS) {
    const int s = idx / KQ, k = idx - s * KQ;
    hs[k * POOL_SEQS + s] = s < ns ? p.hidden[size_t(p.seq_start[s0 + s]) * H + k_base + k] : 0.0f;
  }
  __syncthreads();
  float acc[POOL_SEQS];
#pragma unroll
  for (int s = 0; s < POOL_SEQS; ++s) acc[s] = 0.0f;
#pragma unroll
  for (int i = 0; i < POOL_MAX_KW; ++i) {
    if (i < kw) {
      const float4* h4 = reinterpret_cast<const float4*>(hs + (warp * kw + i) * POOL_SEQS);
#pragma unroll
      for (int q = 0; q < POOL_SEQS / 4; ++q) {
        const float4 hv = h4[q];
        acc[4 * q] = __fmaf_rn(hv.x, wv[i], acc[4 * q]);
        acc[4 * q + 1] = __fmaf_rn(hv.y, wv[i], acc[4 * q + 1]);
        acc[4 * q + 2] = __fmaf_rn(hv.z, wv[i], acc[4 * q + 2]);
        acc[4 * q + 3] = __fmaf_rn(hv.w, wv[i], acc[4 * q + 3]);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < POOL_SEQS; ++s) part[(warp * POOL_SEQS + s) * 32 + lane] = acc[s];
  __syncthreads();
  for (int s = warp; s < ns; s += HEAD_THREADS / 32) {
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < HEAD_THREADS / 32; ++w) v = __fadd_rn(v, part[(w * POOL_SEQS + s) * 32 + lane]);
    p.pooled[(size_t(blockIdx.z) * p.nseq + s0 + s) * H + j] = v;
  }
}

// classifier_kernel: one CTA per sequence.  Thread t owns columns t, t+256, ...: it adds
// the POOL_KSPLIT partials in order, + bias, numpy tanh -> smem; each label's dot product
// is a per-thread partial, a warp shuffle tree and a fixed-order sum of the 8 warp
// results; thread 0 runs the exact softmax / argmax.
static __global__ void __launch_bounds__(HEAD_THREADS) classifier_kernel(const HeadParams p) {
  extern __shared__ float pooled_s[];     // [H] then red [8][HEAD_MAX_LABELS] then lg [HEAD_MAX_LABELS]
  __shared__ TanhTable tt;
  const int H = p.hidden_size, L = p.num_labels;
  load_tanh_table(&tt, threadIdx.x, HEAD_THREADS);
  pdl_trigger();
  pdl_wait();
  const int s = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* x = pooled_s;
  float* red = pooled_s + H;
  float* lg = red + 8 * HEAD_MAX_LABELS;
  float v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = threadIdx.x + i * HEAD_THREADS;
    v[i] = 0.0f;
    if (k < H) {
      float parts[POOL_KSPLIT];
#pragma unroll
      for (int z = 0; z < POOL_KSPLIT; ++z) parts[z] = p.pooled[(size_t(z) * p.nseq + s) * H + k];
      float a = parts[0];
#pragma unroll
      for (int z = 1; z < POOL_KSPLIT; ++z) a = __fadd_rn(a, parts[z]);
      v[i] = a;
    }
  }
  __syncthreads();   // tanh table
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = threadIdx.x + i * HEAD_THREADS;
    if (k < H) {
      v[i] = np_tanhf(__fadd_rn(v[i], p.pool_b[k]), &tt);
      x[k] = v[i];
    }
  }
  for (int l = 0; l < L; ++l) {
    float a = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = threadIdx.x + i * HEAD_THREADS;
      if (k < H) a = __fmaf_rn(v[i], __ldg(p.head_wt + size_t(l) * H + k), a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) red[warp * HEAD_MAX_LABELS + l] = a;
  }
  __syncthreads();
  if (threadIdx.x < L) {
    float a = 0.0f;
#pragma unroll
    for (int w = 0; w < HEAD_THREADS / 32; ++w) a = __fadd_rn(a, red[w * HEAD_MAX_LABELS + threadIdx.x]);
    lg[threadIdx.x] = __fadd_rn(a, p.head_b[threadIdx.x]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float l2[HEAD_MAX_LABELS], pr[HEAD_MAX_LABELS];
    for (int l = 0; l < L; ++l) l2[l] = lg[l];
    int lab;
    softmax_argmax(l2, pr, &lab, L);
    for (int l = 0; l < L; ++l) {
      p.logits[size_t(s) * L + l] = l2[l];
      p.probs[size_t(s) * L + l] = pr[l];
    }
    p.labels[s] = lab;
  }
}

// one warp per token; the token's row is loaded into registers once (all of its loads in
// flight together) and reused for every label: the same per-lane FMA order as warp_dot
constexpr int TAG_MAX_V = 8;   // float4 per lane: H <= 1024
static __global__ void __launch_bounds__(HEAD_THREADS) tag_kernel(const HeadParams p) {
  pdl_trigger();
  pdl_wait();
  const int H = p.hidden_size, L = p.num_labels;
  const int t = blockIdx.x * (HEAD_THREADS / 32) + threadIdx.x / 32;
  if (t >= p.T) return;
  const int lane = threadIdx.x % 32;
  const float* h = p.hidden + size_t(t) * H;
  float4 hv[TAG_MAX_V];
#pragma unroll
  for (int i = 0; i < TAG_MAX_V; ++i) {
    const int k = lane * 4 + 128 * i;
    hv[i] = k < H ? __ldcs(reinterpret_cast<const float4*>(h + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float lg[HEAD_MAX_LABELS];
  for (int l = 0; l < L; ++l) {
    const float* w = p.head_wt + size_t(l) * H;
    float acc = 0.0f;
#pragma unroll
    for (int i = 0; i < TAG_MAX_V; ++i) {
      const int k = lane * 4 + 128 * i;
      if (k < H) {
        const float4 y = __ldg(reinterpret_cast<const float4*>(w + k));
        acc = __fmaf_rn(hv[i].x, y.x, acc);
        acc = __fmaf_rn(hv[i].y, y.y, acc);
        acc = __fmaf_rn(hv[i].z, y.z, acc);
        acc = __fmaf_rn(hv[i].w, y.w, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    lg[l] = __fadd_rn(acc, p.head_b[l]);
  }
  if (threadIdx.x % 32 == 0) {
    float pr[HEAD_MAX_LABELS];
    int lab;
    softmax_argmax(lg, pr, &lab, L);
    for (int l = 0; l < L; ++l) {
      p.logits[size_t(t) * L + l] = lg[l];
      p.probs[size_t(t) * L + l] = pr[l];
    }
    p.labels[t] = lab;
  }
}
#endif  // SAMP_DEFINE_KERNELS

}  // namespace samp
