#include "gemm_persistent.cuh"
#include "kernels.h"

namespace samp {

#ifndef SAMP_PERSIST_STAGES128
#define SAMP_PERSIST_STAGES128 5
#endif
#ifndef SAMP_PERSIST_NE
#define SAMP_PERSIST_NE 8
#endif

// persistent (gemm_persistent.cuh) unless SAMP_NO_PERSISTENT is set (A/B measurements)
inline bool persistent_enabled() {
  static const bool on = std::getenv("SAMP_NO_PERSISTENT") == nullptr;
  return on;
}

template <class Epi>
static cudaError_t by_bn(int bn, bool persistent, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const typename Epi::Params& p, cudaStream_t st) {
  constexpr int NEP = SAMP_PERSIST_NE;
  if (persistent && persistent_enabled()) {
    switch (bn) {
      case 256: return launch_gemm_persistent<KIND_I8, 256, 4, NEP, Epi>(a, b, M, N, kb, p, st);
      case 128: return launch_gemm_persistent<KIND_I8, 128, SAMP_PERSIST_STAGES128, NEP, Epi>(a, b, M, N, kb, p, st);
      case 96: return launch_gemm_persistent<KIND_I8, 96, 6, 8, Epi>(a, b, M, N, kb, p, st);
      case 64: return launch_gemm_persistent<KIND_I8, 64, 6, 8, Epi>(a, b, M, N, kb, p, st);
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
  // QKV's epilogue is light (dequant + quantize): two co-resident one-tile CTAs per SM
  // overlap each other better than one persistent CTA (18.3 vs 18.9 us at 4096 tokens)
  return by_bn<EpiQKV>(bn, false, a, b, M, N, kb, p, st);
}

cudaError_t gemm_gelu_i8(int bn, bool finite, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                         const EpiGeluQuant::Params& p, cudaStream_t st) {
  if (finite) return by_bn<EpiGeluQuantFinite>(bn, true, a, b, M, N, kb, p, st);
  return by_bn<EpiGeluQuant>(bn, true, a, b, M, N, kb, p, st);
}

}  // namespace samp
