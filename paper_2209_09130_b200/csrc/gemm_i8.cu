#include "gemm_persistent.cuh"
#include "kernels.h"

namespace samp {

#ifndef SAMP_PERSIST_NE
#define SAMP_PERSIST_NE 8
#endif


// persistent (gemm_persistent.cuh) unless SAMP_NO_PERSISTENT is set (A/B measurements)
inline bool persistent_enabled() {
  static const bool on = !env_flag("SAMP_NO_PERSISTENT");
  return on;
}

static int sm_count() {
  static thread_local int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <class Epi>
static cudaError_t by_bn(int bn, bool persistent, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const typename Epi::Params& p, cudaStream_t st) {
  constexpr int NEP = SAMP_PERSIST_NE;
  if (persistent && persistent_enabled()) {
    // two persistent CTAs per SM where the ring fits twice (<= ~100 KB each)
    switch (bn) {
      case 256: return launch_gemm_persistent<KIND_I8, 256, 4, NEP, Epi>(a, b, M, N, kb, p, st);
      case 128: return launch_gemm_persistent<KIND_I8, 128, 3, NEP, Epi, 2>(a, b, M, N, kb, p, st);
      case 96: return launch_gemm_persistent<KIND_I8, 96, 3, 8, Epi, 2>(a, b, M, N, kb, p, st);
#ifdef SAMP_FFN1_64X3
      case 64: return launch_gemm_persistent<KIND_I8, 64, 2, 8, Epi, 3>(a, b, M, N, kb, p, st);
#else
      case 64:
        // at most one tile per SM (small batches): a deep ring instead of a second CTA —
        // the whole K of a BERT-base QKV/FFN1 tile in flight at once
        if (long((M + GEMM_BM - 1) / GEMM_BM) * (N / 64) <= sm_count() && !env_flag("SAMP_NO_DEEP64"))
          return launch_gemm_persistent<KIND_I8, 64, 6, 8, Epi, 1>(a, b, M, N, kb, p, st);
        return launch_gemm_persistent<KIND_I8, 64, 4, 8, Epi, 2>(a, b, M, N, kb, p, st);
#endif
    }
    return cudaErrorInvalidValue;
  }
  switch (bn) {
    case 256: return launch_gemm<KIND_I8, 256, 2, 1, 8, Epi>(a, b, M, N, kb, p, st);
    case 128: return launch_gemm<KIND_I8, 128, 3, 1, 8, Epi>(a, b, M, N, kb, p, st);
    case 64: return launch_gemm<KIND_I8, 64, 4, 1, 8, Epi>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t gemm_qkv_i8(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiQKV::Params& p, cudaStream_t st) {
  // bn < 0: persistent kernel with |bn|-wide tiles, two CTAs per SM (engine default, 128);
  // bn > 0: one tile per CTA (SAMP_QKV_ONETILE=1)
  if (bn < 0) return by_bn<EpiQKV>(-bn, true, a, b, M, N, kb, p, st);
  return by_bn<EpiQKV>(bn, false, a, b, M, N, kb, p, st);
}

cudaError_t gemm_gelu_i8(int bn, int mode, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const EpiGeluQuant::Params& p, cudaStream_t st) {
  if (mode == GELU_FAST) return by_bn<EpiGeluQuantFast>(bn, true, a, b, M, N, kb, p, st);
  if (mode == GELU_FINITE) return by_bn<EpiGeluQuantFinite>(bn, true, a, b, M, N, kb, p, st);
  return by_bn<EpiGeluQuant>(bn, true, a, b, M, N, kb, p, st);
}

// Exhaustive admission check of the GELU_FAST epilogue for one ffn.mid scale: every float x
// with |x| < 1e12 (the FINITE domain), each element's own near-flag; counts[0] = elements
// whose unflagged fast code differs from the exact code (must be 0), counts[1] = flagged.
__global__ void gelu_fast_exhaustive_kernel(float s, float inv_s, X2 k, unsigned long long* counts) {
  __shared__ TanhTable tt;
  load_tanh_table(&tt, threadIdx.x, blockDim.x);
  __syncthreads();
  const Recip rq = make_recip(s);
  unsigned long long bad = 0, flagged = 0;
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < (1ull << 29);
       g += uint64_t(gridDim.x) * blockDim.x) {
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x[u] = __uint_as_float(uint32_t(g * 8 + u));
      if (!(fabsf(x[u]) < 1e12f)) x[u] = 0.0f;
    }
    uint32_t e0, e1;
    EpiGeluQuantFast::exact8(x, &tt, rq, k, e0, e1);
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      bool near = false;
      const float2 t = gelu_q_fast2(f2(x[u], x[u + 1]), inv_s, k, near);
      const uint32_t fq = trunc_pack4_s8(t.x, t.y, 0.0f, 0.0f);
      const uint32_t ex = (u < 4 ? e0 : e1) >> (8 * (u & 3));
      flagged += near;
      bad += !near && ((fq ^ ex) & 0xffffu) != 0u;
    }
  }
  atomicAdd(counts, bad);
  atomicAdd(counts + 1, flagged);
}

cudaError_t gelu_fast_check(float s, float inv_s, unsigned long long* host_counts, cudaStream_t st) {
  unsigned long long* d = nullptr;
  cudaError_t err = cudaMallocAsync(&d, 2 * sizeof(unsigned long long), st);
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), st);
  gelu_fast_exhaustive_kernel<<<148 * 8, 256, 0, st>>>(s, inv_s, x2_consts(), d);
  cudaMemcpyAsync(host_counts, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  err = cudaStreamSynchronize(st);
  return err != cudaSuccess ? err : cudaGetLastError();
}

}  // namespace samp
