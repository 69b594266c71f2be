#include <cstdlib>
#include "kernels.h"

namespace samp {

template <bool F16, int TPR, bool HIST = false>
static cudaError_t launch_tpr(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                              cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<F16, TPR, HIST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnLayout<F16>(ATT_MAX_KEYS).total);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  return launch_ex(attention_kernel<F16, TPR, HIST>, dim3(ntiles, heads), dim3(att_threads<TPR>()),
                   AttnLayout<F16>(keys_cap).total, st, 1, map, p, keys_cap);
}

// Two threads per row.  Four (SAMP_ATT_TPR=4; bit-identical) measured slower even where
// TMEM limits an SM to two CTAs (S = 256: 151 vs 142 us per BERT-large launch): the
// softmax passes are FMA-pipe bound, not thread-count bound.
template <bool F16>
static cudaError_t launch_att(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                              cudaStream_t st) {
  const char* f = std::getenv("SAMP_ATT_TPR");
  const int tpr = f ? std::atoi(f) : 2;
  if constexpr (!F16)
    if (p.hist) return launch_tpr<F16, 2, true>(map, p, ntiles, heads, keys_cap, st);   // analyze-quant
  if (tpr == 4) return launch_tpr<F16, 4>(map, p, ntiles, heads, keys_cap, st);
  return launch_tpr<F16, 2>(map, p, ntiles, heads, keys_cap, st);
}

cudaError_t launch_attention_i8(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                                cudaStream_t st) {
  return launch_att<false>(map, p, ntiles, heads, keys_cap, st);
}
cudaError_t launch_attention_f16(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                                 cudaStream_t st) {
  return launch_att<true>(map, p, ntiles, heads, keys_cap, st);
}

}  // namespace samp
