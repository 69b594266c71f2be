// Downstream heads on the final F32 hidden states (reference pkg/src/samp/tasks.py:28-55).
//   classify: pooled = tanh(h[CLS] @ Wp + bp); logits = pooled @ Wh + bh;
//             probs = softmax_rows(logits); label = argmax (lowest index on ties)
//   tag:      logits = h[t] @ Wh + bh per token; softmax; argmax
// The reference's two small products are BLAS sgemm calls (order unspecified), so the
// dot products here are FP32 FMA chains: logits/probs agree within float rounding
// (tests use a tolerance); tanh, exp and the softmax normaliser are numpy-exact.
//
// classify = two launches: pooler_kernel spreads the [B,H]x[H,H] pooler over
// (32-column, 32-sequence) tiles — a warp owns 4 sequences, a lane one output column,
// so every Wp row slice is one coalesced 128-byte load; classifier_kernel is one warp
// per sequence (lanes over H, shuffle reduction) plus the exact softmax/argmax.
#pragma once
#include "numerics.cuh"

namespace samp {

constexpr int HEAD_THREADS = 256;
constexpr int HEAD_MAX_LABELS = 64;
constexpr int POOL_COLS = 32;      // output columns per pooler CTA
constexpr int POOL_SEQS = 32;      // sequences per pooler CTA
constexpr int POOL_KSPLIT = 4;     // K quarters (grid.z)

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

// pooler_kernel: CTA (x, y, z) = 32 output columns x up to 32 sequences x K-quarter z;
// warp w reduces K rows [z*H/4 + w*H/32, ...) for all its sequences (lane = column, 32
// independent accumulators); the 8 warp partials are added in a fixed order and written
// to pooled[z][s][j].  classifier_kernel (one warp per sequence) adds the 4 quarters in
// order, applies bias + numpy tanh, then the classifier dot products + exact softmax.
static __global__ void __launch_bounds__(HEAD_THREADS) pooler_kernel(const HeadParams p) {
  extern __shared__ float sh[];           // h [POOL_SEQS][H/4] then partials [8][POOL_SEQS][32]
  pdl_trigger();
  pdl_wait();
  const int H = p.hidden_size, KQ = H / POOL_KSPLIT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * POOL_COLS + lane;
  const int s0 = blockIdx.y * POOL_SEQS;
  const int k_base = blockIdx.z * KQ;
  const int ns = min(POOL_SEQS, p.nseq - s0);
  float* hs = sh;
  float* part = sh + POOL_SEQS * KQ;
  for (int s = warp; s < ns; s += HEAD_THREADS / 32) {      // [CLS] row slices
    const float* src = p.hidden + size_t(p.seq_start[s0 + s]) * H + k_base;
    for (int k = lane; k < KQ; k += 32) hs[s * KQ + k] = src[k];
  }
  __syncthreads();
  float acc[POOL_SEQS];
#pragma unroll
  for (int s = 0; s < POOL_SEQS; ++s) acc[s] = 0.0f;
  const int k_per = KQ / (HEAD_THREADS / 32);
  const int k0 = warp * k_per;
  if (j < H) {
#pragma unroll 4
    for (int k = k0; k < k0 + k_per; ++k) {
      const float wk = __ldg(p.pool_w + size_t(k_base + k) * H + j);
#pragma unroll
      for (int s = 0; s < POOL_SEQS; ++s) acc[s] = __fmaf_rn(hs[s * KQ + k], wk, acc[s]);
    }
  }
#pragma unroll
  for (int s = 0; s < POOL_SEQS; ++s) part[(warp * POOL_SEQS + s) * 32 + lane] = acc[s];
  __syncthreads();
  for (int s = warp; s < ns; s += HEAD_THREADS / 32) {
    if (j >= H) continue;
    float v = 0.0f;
    for (int w = 0; w < HEAD_THREADS / 32; ++w) v = __fadd_rn(v, part[(w * POOL_SEQS + s) * 32 + lane]);
    p.pooled[(size_t(blockIdx.z) * p.nseq + s0 + s) * H + j] = v;
  }
}

static __global__ void __launch_bounds__(HEAD_THREADS) classifier_kernel(const HeadParams p) {
  extern __shared__ float pooled_s[];     // [8 warps][H]
  __shared__ TanhTable tt;
  const int H = p.hidden_size, L = p.num_labels;
  load_tanh_table(&tt, threadIdx.x, HEAD_THREADS);
  pdl_trigger();
  pdl_wait();
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = blockIdx.x * (HEAD_THREADS / 32) + warp;
  if (s >= p.nseq) return;
  float* x = pooled_s + warp * H;
  for (int k = lane; k < H; k += 32) {
    float v = p.pooled[size_t(s) * H + k];
    for (int z = 1; z < POOL_KSPLIT; ++z) v = __fadd_rn(v, p.pooled[(size_t(z) * p.nseq + s) * H + k]);
    x[k] = np_tanhf(__fadd_rn(v, p.pool_b[k]), &tt);
  }
  __syncwarp();
  float lg[HEAD_MAX_LABELS];
  for (int l = 0; l < L; ++l) lg[l] = __fadd_rn(warp_dot(x, p.head_wt + size_t(l) * H, H), p.head_b[l]);
  if (lane == 0) {
    float pr[HEAD_MAX_LABELS];
    int lab;
    softmax_argmax(lg, pr, &lab, L);
    for (int l = 0; l < L; ++l) {
      p.logits[size_t(s) * L + l] = lg[l];
      p.probs[size_t(s) * L + l] = pr[l];
    }
    p.labels[s] = lab;
  }
}

// one warp per token
static __global__ void __launch_bounds__(HEAD_THREADS) tag_kernel(const HeadParams p) {
  pdl_trigger();
  pdl_wait();
  const int H = p.hidden_size, L = p.num_labels;
  const int t = blockIdx.x * (HEAD_THREADS / 32) + threadIdx.x / 32;
  if (t >= p.T) return;
  const float* h = p.hidden + size_t(t) * H;
  float lg[HEAD_MAX_LABELS];
  for (int l = 0; l < L; ++l) lg[l] = __fadd_rn(warp_dot(h, p.head_wt + size_t(l) * H, H), p.head_b[l]);
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
