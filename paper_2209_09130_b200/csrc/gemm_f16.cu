#include "kernels.h"

namespace samp {

cudaError_t gemm_f16out(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                        const EpiF16Out::Params& p, cudaStream_t st) {
  switch (bn) {
    case 256: return launch_gemm<KIND_F16, 256, 2, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
    case 128: return launch_gemm<KIND_F16, 128, 3, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
    case 64: return launch_gemm<KIND_F16, 64, 4, 1, 8, EpiF16Out>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
