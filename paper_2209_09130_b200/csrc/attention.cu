#include "kernels.h"

namespace samp {

template <bool F16>
static cudaError_t launch_att(const CUtensorMap& map, const AttnParams& p, int ntiles, int heads, int keys_cap,
                              cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnLayout<F16>(ATT_MAX_KEYS).total);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  return launch_ex(attention_kernel<F16>, dim3(ntiles, heads), dim3(ATT_THREADS), AttnLayout<F16>(keys_cap).total,
                   st, 1, map, p, keys_cap);
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
