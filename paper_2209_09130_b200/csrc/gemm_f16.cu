#include "gemm_persistent.cuh"
#include "kernels.h"

namespace samp {

#ifndef SAMP_PERSIST_NE
#define SAMP_PERSIST_NE 8
#endif

static int sm_count_f16() {
  static thread_local int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

cudaError_t gemm_f16out(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiF16Out::Params& p, cudaStream_t st) {
  constexpr int NEP = SAMP_PERSIST_NE;
  if (!env_flag("SAMP_NO_PERSISTENT")) {
    switch (bn) {
      case 256: return launch_gemm_persistent<KIND_F16, 256, 4, NEP, EpiF16Out>(a, b, M, N, kb, p, st);
      case 128: return launch_gemm_persistent<KIND_F16, 128, 5, NEP, EpiF16Out>(a, b, M, N, kb, p, st);
      case 64:
        // at most one tile per SM (small batches): 8-stage ring, the whole K = 2 x 768 bytes
        // of a BERT-base tile in flight (batch-1 FP16 p50 0.693 -> 0.67 ms)
        if (long((M + GEMM_BM - 1) / GEMM_BM) * (N / 64) <= sm_count_f16())
          return launch_gemm_persistent<KIND_F16, 64, 8, 8, EpiF16Out>(a, b, M, N, kb, p, st);
        return launch_gemm_persistent<KIND_F16, 64, 6, 8, EpiF16Out>(a, b, M, N, kb, p, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (bn) {
    case 256: return launch_gemm<KIND_F16, 256, 2, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
    case 128: return launch_gemm<KIND_F16, 128, 3, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
    case 64: return launch_gemm<KIND_F16, 64, 4, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
