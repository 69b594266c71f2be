#include "gemm_ln_persistent.cuh"
#include "kernels.h"

namespace samp {

cudaError_t gemm_ln_f16(const Tiles& t, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                       const EpiResLN::Params& p, cudaStream_t st) {
  // same persistent rule as gemm_ln_i8 (kind::f16, f32 accumulators and residuals):
  // C5 out-proj 0.86 vs 1.22 ms per launch
  const int mtiles = (M + GEMM_BM - 1) / GEMM_BM;
  if (!env_flag("SAMP_NO_LN_PERSISTENT") && (mtiles >= 256 || env_flag("SAMP_LN_PERSISTENT"))) {
    switch (t.bn_ln * 10 + t.cluster_ln) {
      case 1924:
        if (mtiles >= 8 * ln_persistent_clusters<KIND_F16, 192, 4, 4>() || env_flag("SAMP_LN_PERSISTENT"))
          return launch_gemm_ln_persistent<KIND_F16, 192, 4, 4>(a, b, M, kb, p, st);
        break;
      case 2564:
        if (mtiles >= 8 * ln_persistent_clusters<KIND_F16, 256, 3, 4>() || env_flag("SAMP_LN_PERSISTENT"))
          return launch_gemm_ln_persistent<KIND_F16, 256, 3, 4>(a, b, M, kb, p, st);
        break;
    }
  }
  switch (t.bn_ln * 10 + t.cluster_ln) {
    case 1924: return launch_gemm<KIND_F16, 192, 4, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2564: return launch_gemm<KIND_F16, 256, 3, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2562: return launch_gemm<KIND_F16, 256, 3, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1922: return launch_gemm<KIND_F16, 192, 4, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2561: return launch_gemm<KIND_F16, 256, 3, 1, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1281: return launch_gemm<KIND_F16, 128, 3, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
    case 641: return launch_gemm<KIND_F16, 64, 4, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
    case 968: {   // small batches (the two-thread strided epilogue measured 0.681 -> 0.695 ms FP16 p50 here)
      // f32 (+ f16) outputs only: staged in smem and written by TMA stores (the per-row 16-byte
      // stores of 32 rows per warp instruction were half of this epilogue); SAMP_NO_LN_TMA_STORE=1: A/B
      EpiResLN::Params q = p;
      const bool plain = p.out_f32 && !p.out_i8 && !p.deq_outputs && !p.amax && !p.tap_f32;
      if (plain && !env_flag("SAMP_NO_LN_TMA_STORE")) q.tma_f = 1 | (p.out_f16 ? 2 : 0);
      // the f32 residual tile by TMA into the drained ring (instead of per-row global loads)
      if (p.res_f32 && !p.res_i8 && !env_flag("SAMP_NO_LN_TMA_RES")) q.tma_res = 1;
      // SAMP_LN96_STRIDED=1: two threads per row (run_strided, TMA residual and stores too):
      // bit-identical, measured slower (batch-1 FP16 p50 0.651 vs 0.618 ms)
      if (q.tma_f && q.tma_res && env_flag("SAMP_LN96_STRIDED"))
        return launch_gemm<KIND_F16, 96, 6, 8, 8, EpiResLN>(a, b, M, N, kb, q, st);
      // long K (FFN2): the two K halves on 16 SMs, partial tile through DSMEM (KS2)
      if (kb >= 4096 && env_flag("SAMP_LN_KS2"))
        return launch_gemm<KIND_F16, 96, 4, 8, 4, EpiResLNRegs96, false, true>(a, b, M, N, kb, q, st);
      return launch_gemm<KIND_F16, 96, 6, 8, 4, EpiResLNRegs96>(a, b, M, N, kb, q, st);
    }
    case 1288: return launch_gemm<KIND_F16, 128, 5, 8, 4, EpiResLN>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace samp
