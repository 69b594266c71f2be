// Embedding, heads, and load-time weight packing kernels.
#define SAMP_DEFINE_KERNELS
#include "kernels.h"

namespace samp {

// Weight ranges of the forward, in use order, pulled into L2 while the first layers run
// (the timed forward starts with a cold L2; small batches stream each weight tile through a
// handful of SMs, so their main loops wait on HBM latency).  Chunk c of the flattened list
// goes to CTA c % gridDim.x, so the early layers' chunks are issued first.
__global__ void l2_prefetch_kernel(const __grid_constant__ PrefetchList l) {
  constexpr unsigned long long CHUNK = 32768;
  if (threadIdx.x != 0) return;
  unsigned long long base = 0;   // first chunk index of range i
  for (int i = 0; i < l.n; ++i) {
    const unsigned long long nch = (l.bytes[i] + CHUNK - 1) / CHUNK;
    unsigned long long c = (blockIdx.x + gridDim.x - base % gridDim.x) % gridDim.x;   // my first chunk of range i
    for (; c < nch; c += gridDim.x) {
      const unsigned long long off = c * CHUNK;
      const unsigned long long sz = l.bytes[i] - off < CHUNK ? l.bytes[i] - off : CHUNK;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                   :: "l"(reinterpret_cast<const char*>(l.ptr[i]) + off), "r"(unsigned(sz & ~15ull)) : "memory");
    }
    base += nch;
  }
}

cudaError_t launch_l2_prefetch(const PrefetchList& l, int ctas, cudaStream_t st) {
  max_carveout_once(l2_prefetch_kernel);
  l2_prefetch_kernel<<<ctas, 32, 0, st>>>(l);
  return cudaGetLastError();
}

template <int H>
static cudaError_t embed_h(const EmbedParams& p, cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(embed_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  constexpr int tok = EMB_THREADS / 32;
  return launch_ex(embed_kernel<H>, dim3((p.T + tok - 1) / tok), dim3(EMB_THREADS),
                   size_t(tok) * EmbLeaves<H>::ROW * sizeof(float),
                   st, 1, p);
}

template <int H>
static cudaError_t ln_rows_h(const LnRowsParams& p, cudaStream_t st) {
  constexpr int rows = LNR_THREADS / 32;
  return launch_ex(ln_rows_kernel<H>, dim3((p.M + rows - 1) / rows), dim3(LNR_THREADS),
                   size_t(rows) * EmbLeaves<H>::ROW * sizeof(float), st, 1, p);
}

bool ln_rows_supported(int hidden) {
  return hidden == 768 || hidden == 1024 || hidden == 512 || hidden == 384;
}

cudaError_t launch_ln_rows(const LnRowsParams& p, int hidden, cudaStream_t st) {
  switch (hidden) {
    case 384: return ln_rows_h<384>(p, st);
    case 512: return ln_rows_h<512>(p, st);
    case 768: return ln_rows_h<768>(p, st);
    case 1024: return ln_rows_h<1024>(p, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_embed(const EmbedParams& p, cudaStream_t st) {
  switch (p.hidden) {
    case 64: return embed_h<64>(p, st);
    case 128: return embed_h<128>(p, st);
    case 256: return embed_h<256>(p, st);
    case 384: return embed_h<384>(p, st);
    case 512: return embed_h<512>(p, st);
    case 768: return embed_h<768>(p, st);
    case 1024: return embed_h<1024>(p, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_classify(const HeadParams& p, cudaStream_t st) {
  const dim3 grid((p.hidden_size + POOL_COLS - 1) / POOL_COLS, (p.nseq + POOL_SEQS - 1) / POOL_SEQS, POOL_KSPLIT);
  const size_t smem = (size_t(POOL_SEQS) * p.hidden_size / POOL_KSPLIT + 8 * POOL_SEQS * 32) * sizeof(float);
  cudaError_t e = launch_ex(pooler_kernel, grid, dim3(HEAD_THREADS), smem, st, 1, p);
  if (e != cudaSuccess) return e;
  return launch_ex(classifier_kernel, dim3(p.nseq), dim3(HEAD_THREADS),
                   (size_t(p.hidden_size) + 9 * HEAD_MAX_LABELS) * sizeof(float), st, 1, p);
}

cudaError_t launch_tag(const HeadParams& p, cudaStream_t st) {
  return launch_ex(tag_kernel, dim3((p.T + HEAD_THREADS / 32 - 1) / (HEAD_THREADS / 32)), dim3(HEAD_THREADS), 0, st,
                   1, p);
}

// W [K][N] F32 (archive layout) -> Wt int8 [N][K] (one per-tensor scale, reference
// quantize_weight encoder.py:191-194) and Wt f16 [N][K]; rows land at `row_off`.
__global__ void pack_weight_kernel(const float* __restrict__ w, int K, int N, float scale,
                                   int8_t* __restrict__ out_i8, __half* __restrict__ out_f16, int row_off) {
  __shared__ float tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx over N, by over K
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = by + i, n = bx + threadIdx.x;
    if (k < K && n < N) tile[i][threadIdx.x] = w[size_t(k) * N + n];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int n = bx + i, k = by + threadIdx.x;
    if (k < K && n < N) {
      const float v = tile[threadIdx.x][i];
      const size_t o = size_t(row_off + n) * K + k;
      out_i8[o] = int8_t(quant_i8(v, scale));
      out_f16[o] = __float2half_rn(v);
    }
  }
}

cudaError_t launch_pack_weight(const float* w, int K, int N, float scale, int8_t* out_i8, __half* out_f16,
                               int row_off, cudaStream_t st) {
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  pack_weight_kernel<<<grid, block, 0, st>>>(w, K, N, scale, out_i8, out_f16, row_off);
  return cudaGetLastError();
}

__global__ void transpose_f32_kernel(const float* __restrict__ w, int K, int N, float* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < size_t(K) * N) {
    const int k = int(i / N), n = int(i % N);
    out[size_t(n) * K + k] = w[i];
  }
}

cudaError_t launch_transpose_f32(const float* w, int K, int N, float* out, cudaStream_t st) {
  const size_t n = size_t(K) * N;
  transpose_f32_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(w, K, N, out);
  return cudaGetLastError();
}

// code-usage tap: bins[c + 128] += #{codes == c} over rows x cols of an int8 matrix with
// row stride ld (cols % 16 == 0, 16B-aligned rows).  Zeros are counted in registers (the
// dominant code at most sites), the rest through a shared histogram.
__global__ void __launch_bounds__(256) code_hist_kernel(const int8_t* __restrict__ src, int rows, int cols, int ld,
                                                        unsigned long long* __restrict__ bins) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int vpr = cols / 16;
  const size_t nvec = size_t(rows) * vpr;
  unsigned int zeros = 0;
  for (size_t v = blockIdx.x * size_t(blockDim.x) + threadIdx.x; v < nvec; v += size_t(gridDim.x) * blockDim.x) {
    const size_t row = v / vpr;
    const int c16 = int(v - row * vpr);
    const uint4 q = *reinterpret_cast<const uint4*>(src + row * ld + c16 * 16);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = int(int8_t(w[k] >> (8 * b)));
        if (c == 0) ++zeros;
        else atomicAdd(&h[c + 128], 1u);
      }
  }
  if (zeros) atomicAdd(&h[128], zeros);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&bins[i], (unsigned long long)h[i]);
}

cudaError_t launch_code_hist(const int8_t* src, int rows, int cols, int ld, unsigned long long* bins,
                             cudaStream_t st) {
  if (cols % 16 || ld % 16 || (reinterpret_cast<uintptr_t>(src) & 15)) return cudaErrorInvalidValue;
  const size_t nvec = size_t(rows) * (cols / 16);
  const unsigned blocks = unsigned(std::min<size_t>((nvec + 255) / 256, 4 * 148));
  if (blocks == 0) return cudaSuccess;
  code_hist_kernel<<<blocks, 256, 0, st>>>(src, rows, cols, ld, bins);
  return cudaGetLastError();
}

}  // namespace samp
