#include "kernels.h"

namespace samp {

cudaError_t gemm_ln_i8(const Tiles& t, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                       const EpiResLN::Params& p, cudaStream_t st) {
  switch (t.bn_ln * 10 + t.cluster_ln) {
    case 1924: return launch_gemm<KIND_I8, 192, 4, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2564: return launch_gemm<KIND_I8, 256, 3, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2562: return launch_gemm<KIND_I8, 256, 3, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1922: return launch_gemm<KIND_I8, 192, 4, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2561: return launch_gemm<KIND_I8, 256, 3, 1, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1281: return launch_gemm<KIND_I8, 128, 3, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
    case 641: return launch_gemm<KIND_I8, 64, 4, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
