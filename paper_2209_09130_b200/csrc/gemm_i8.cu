#include "kernels.h"

namespace samp {

template <class Epi>
static cudaError_t by_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const typename Epi::Params& p, cudaStream_t st) {
  switch (bn) {
    case 256: return launch_gemm<KIND_I8, 256, 2, 1, 8, Epi>(a, b, M, N, kb, p, st);
    case 128: return launch_gemm<KIND_I8, 128, 3, 1, 8, Epi>(a, b, M, N, kb, p, st);
    case 64: return launch_gemm<KIND_I8, 64, 4, 1, 8, Epi>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t gemm_qkv_i8(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiQKV::Params& p, cudaStream_t st) {
  return by_bn<EpiQKV>(bn, a, b, M, N, kb, p, st);
}

cudaError_t gemm_gelu_i8(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const EpiGeluQuant::Params& p, cudaStream_t st) {
  return by_bn<EpiGeluQuant>(bn, a, b, M, N, kb, p, st);
}

}  // namespace samp
