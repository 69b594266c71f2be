#include "kernels.h"
#include "qkv_attention.cuh"

namespace samp {

// One persistent CTA per SM (at most one per work item).  Four softmax threads per query
// row (16 softmax warps: the passes are latency-bound per warp); SAMP_QA_TPR=2 selects two
// (bit-identical).
template <int TPR>
static cudaError_t launch_qa_tpr(const CUtensorMap& a, const CUtensorMap& w, const QAParams& q, int sms,
                                 cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(qkv_attention_kernel<TPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         QALayout::TOTAL);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  const int items = q.ntiles * q.heads;
  const int grid = items < sms ? items : sms;
  QAParams qq = q;
  qq.att.stamps = g_gemm_stamps;   // profiling mode: phase stamps (tools/qa_phases.py)
  return launch_ex(qkv_attention_kernel<TPR>, dim3(grid), dim3(qa_threads<TPR>()), QALayout::TOTAL, st, 1, a, w, qq);
}

int qa_tpr() {
  const char* f = std::getenv("SAMP_QA_TPR");
  return f && std::atoi(f) == 2 ? 2 : 4;
}

cudaError_t launch_qkv_attention(const CUtensorMap& a, const CUtensorMap& w64, const QAParams& q, int sms,
                                 cudaStream_t st) {
  if (qa_tpr() == 2) return launch_qa_tpr<2>(a, w64, q, sms, st);
  return launch_qa_tpr<4>(a, w64, q, sms, st);
}

}  // namespace samp
