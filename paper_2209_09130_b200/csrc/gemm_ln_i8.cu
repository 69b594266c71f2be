#include "gemm_ln_persistent.cuh"
#include "kernels.h"

namespace samp {

cudaError_t gemm_ln_i8(const Tiles& t, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb,
                       const EpiResLN::Params& p, cudaStream_t st, const CUtensorMap* a_mc) {
  const bool mc = a_mc && env_flag("SAMP_LN_MCAST");
  // Many more row tiles than co-resident clusters (probed, gemm_ln_persistent.cuh): persistent
  // clusters with double-buffered TMEM walk the row tiles (C5 FFN2 1.09 vs 1.51 ms at 262k
  // tokens).  With only a few tiles per cluster the fill/drain and the uneven split lose
  // (C4 out-proj 72 vs 57 us at 4 tiles/cluster), hence >= 8 tiles per cluster; otherwise
  // one tile per CTA.  SAMP_NO_LN_PERSISTENT=1 / SAMP_LN_PERSISTENT=1 force either.
  const int mtiles = (M + GEMM_BM - 1) / GEMM_BM;
  if (!env_flag("SAMP_NO_LN_PERSISTENT") && (mtiles >= 256 || env_flag("SAMP_LN_PERSISTENT"))) {
    switch (t.bn_ln * 10 + t.cluster_ln) {
      case 1924:
        if (mtiles >= 8 * ln_persistent_clusters<KIND_I8, 192, 4, 4>() || env_flag("SAMP_LN_PERSISTENT"))
          return launch_gemm_ln_persistent<KIND_I8, 192, 4, 4>(a, b, M, kb, p, st);
        break;
      case 2564:
        if (mtiles >= 8 * ln_persistent_clusters<KIND_I8, 256, 3, 4>() || env_flag("SAMP_LN_PERSISTENT"))
          return launch_gemm_ln_persistent<KIND_I8, 256, 3, 4>(a, b, M, kb, p, st);
        break;
    }
  }
  // the hot chain (int8 residual in, int8 codes out, nothing else): compact epilogue
  const bool i8_only = p.res_i8 && !p.acc_is_f32 && p.out_i8 && !p.deq_outputs && !p.f16_round && !p.amax &&
                       !p.out_f32 && !p.out_f16 && !p.tap_f32;
  if (i8_only) {
    // the code tile leaves through one TMA store per CTA (out_map: box bn_ln x 128) instead of
    // 16-byte row-strided stores (32 rows per warp instruction); SAMP_NO_LN_TMA_STORE=1: A/B
    EpiResLN::Params q = p;
    q.tma_store = env_flag("SAMP_NO_LN_TMA_STORE") ? 0 : 1;
    switch (t.bn_ln * 10 + t.cluster_ln) {
      case 1924:
        if (mc) return launch_gemm<KIND_I8, 192, 4, 4, 8, EpiResLNI8, true>(a_mc[0], b, M, N, kb, q, st);
        // 16 epilogue warps: four threads per row, two per 96-column numpy leaf (run_strided)
        if (env_flag("SAMP_LN_NE16")) return launch_gemm<KIND_I8, 192, 4, 4, 16, EpiResLNI8>(a, b, M, N, kb, q, st);
        return launch_gemm<KIND_I8, 192, 4, 4, 8, EpiResLNI8>(a, b, M, N, kb, q, st);
      case 2564: return launch_gemm<KIND_I8, 256, 3, 4, 8, EpiResLNI8>(a, b, M, N, kb, q, st);
    }
  }
  switch (t.bn_ln * 10 + t.cluster_ln) {
    case 1924:
      if (mc) return launch_gemm<KIND_I8, 192, 4, 4, 8, EpiResLN, true>(a_mc[0], b, M, N, kb, p, st);
      return launch_gemm<KIND_I8, 192, 4, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2564: return launch_gemm<KIND_I8, 256, 3, 4, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2562: return launch_gemm<KIND_I8, 256, 3, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1922: return launch_gemm<KIND_I8, 192, 4, 2, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 2561: return launch_gemm<KIND_I8, 256, 3, 1, 8, EpiResLN>(a, b, M, N, kb, p, st);
    case 1281: return launch_gemm<KIND_I8, 128, 3, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
    case 641: return launch_gemm<KIND_I8, 64, 4, 1, 4, EpiResLN>(a, b, M, N, kb, p, st);
    // small batches: 8-CTA clusters; each CTA streams K x 96 weights alone, so the ring
    // depth sets the bytes in flight (batch-1 fully-quant p50 0.474 vs 0.507 ms at 4 stages;
    // 7 stages no better)
    case 968: {
      // two epilogue threads per row, numpy's accumulators split by index (run_strided):
      // batch-1 fully-quant p50 0.469 -> 0.454 ms vs one thread per row
      if (mc) return launch_gemm<KIND_I8, 96, 6, 8, 4, EpiResLN, true>(a_mc[1], b, M, N, kb, p, st);
      if (env_flag("SAMP_NO_LN96_STRIDED")) return launch_gemm<KIND_I8, 96, 6, 8, 4, EpiResLN>(a, b, M, N, kb, p, st);
      if (i8_only) {   // int8-only chain: compact paired epilogue, codes out by one TMA store
        EpiResLN::Params q = p;
        q.tma_store = env_flag("SAMP_NO_LN_TMA_STORE") ? 0 : 1;
        // long K (FFN2): the two K halves on 16 SMs, partial tile through DSMEM (KS2)
        if (kb >= 2048 && env_flag("SAMP_LN_KS2"))
          return launch_gemm<KIND_I8, 96, 4, 8, 8, EpiResLNI8, false, true>(a, b, M, N, kb, q, st);
        return launch_gemm<KIND_I8, 96, 6, 8, 8, EpiResLNI8>(a, b, M, N, kb, q, st);
      }
      return launch_gemm<KIND_I8, 96, 6, 8, 8, EpiResLN>(a, b, M, N, kb, p, st);
    }
    case 1288: return launch_gemm<KIND_I8, 128, 5, 8, 4, EpiResLN>(a, b, M, N, kb, p, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t gemm_splitk_i8(const CUtensorMap& a, const CUtensorMap& b, int M, int N, int kb, int ksplit,
                           const EpiSplitKAdd::Params& p, cudaStream_t st) {
  return launch_gemm<KIND_I8, 64, 4, 1, 4, EpiSplitKAdd>(a, b, M, N, kb, p, st, ksplit);
}

}  // namespace samp
