// Kernel-level parity entry points: the raw tcgen05 GEMM with an accumulator-store
// epilogue, driven from host buffers (tests compare against the reference's
// gemm_i8_i32, pkg/src/samp/kernels.py:112-127, which is exact).
#include <vector>

#include "gemm.cuh"
#include "host_util.h"

namespace samp {

template <class T>
__global__ void transpose_kernel(const T* __restrict__ src, T* __restrict__ dst, int rows, int cols) {
  // src [rows][cols] -> dst [cols][rows]
  __shared__ T tile[32][33];
  int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    int r = by + i, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[size_t(r) * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    int c = bx + i, r = by + threadIdx.x;
    if (r < rows && c < cols) dst[size_t(c) * rows + r] = tile[threadIdx.x][i];
  }
}

template <class T>
void transpose_device(const T* src, T* dst, int rows, int cols, cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  transpose_kernel<T><<<grid, block, 0, st>>>(src, dst, rows, cols);
}
template void transpose_device<int8_t>(const int8_t*, int8_t*, int, int, cudaStream_t);
template void transpose_device<__half>(const __half*, __half*, int, int, cudaStream_t);

template <int KIND>
static void debug_gemm(const void* a, const void* b, void* c, int m, int n, int k) {
  const int eb = KIND == KIND_I8 ? 1 : 2;
  SAMP_REQUIRE(m >= 1 && n >= 32 && n % 32 == 0 && k >= 1 && (k * eb) % 128 == 0, SAMP_E_DIMENSION,
               "debug gemm needs n % 32 == 0 and k*elt % 128 == 0");
  void *da, *db, *dbt, *dc;
  SAMP_CUDA(cudaMalloc(&da, size_t(m) * k * eb));
  SAMP_CUDA(cudaMalloc(&db, size_t(k) * n * eb));
  SAMP_CUDA(cudaMalloc(&dbt, size_t(k) * n * eb));
  SAMP_CUDA(cudaMalloc(&dc, size_t(m) * n * 4));
  SAMP_CUDA(cudaMemcpy(da, a, size_t(m) * k * eb, cudaMemcpyHostToDevice));
  SAMP_CUDA(cudaMemcpy(db, b, size_t(k) * n * eb, cudaMemcpyHostToDevice));
  if (KIND == KIND_I8)
    transpose_device(static_cast<int8_t*>(db), static_cast<int8_t*>(dbt), k, n, 0);
  else
    transpose_device(static_cast<__half*>(db), static_cast<__half*>(dbt), k, n, 0);
  const int box_k = 128 / eb;
  CUtensorMap ma, mb;
  int bn = n % 256 == 0 ? 256 : n % 128 == 0 ? 128 : n % 64 == 0 ? 64 : 32;
  if (KIND == KIND_I8) {
    ma = tmap_i8(da, m, k, k, box_k, 128);
    mb = tmap_i8(dbt, n, k, k, box_k, bn);
  } else {
    ma = tmap_f16(da, m, k, k, box_k, 128);
    mb = tmap_f16(dbt, n, k, k, box_k, bn);
  }
  EpiStoreAcc::Params p{dc, n};
  const int kb = k * eb;
  cudaError_t e;
  switch (bn) {
    case 256: e = launch_gemm<KIND, 256, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, kb, p, 0); break;
    case 128: e = launch_gemm<KIND, 128, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, kb, p, 0); break;
    case 64: e = launch_gemm<KIND, 64, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, kb, p, 0); break;
    default: e = launch_gemm<KIND, 32, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, kb, p, 0); break;
  }
  SAMP_CUDA(e);
  SAMP_CUDA(cudaDeviceSynchronize());
  SAMP_CUDA(cudaMemcpy(c, dc, size_t(m) * n * 4, cudaMemcpyDeviceToHost));
  cudaFree(da);
  cudaFree(db);
  cudaFree(dbt);
  cudaFree(dc);
}

}  // namespace samp

extern "C" int samp_debug_gemm_i8(const int8_t* a, const int8_t* b, int32_t* c, int m, int n, int k) {
  return samp::guarded([&] { samp::debug_gemm<samp::KIND_I8>(a, b, c, m, n, k); });
}

extern "C" int samp_debug_gemm_f16(const uint16_t* a, const uint16_t* b, float* c, int m, int n, int k) {
  return samp::guarded([&] { samp::debug_gemm<samp::KIND_F16>(a, b, c, m, n, k); });
}

// Tensor-pipe ceiling of this GEMM's main loop: an m x n x k product with the plain
// accumulator-store epilogue (BN = 256, 4-stage ring, one 128-row tile per CTA) on
// device-resident operands, `iters` launches back to back; *ms = average per launch.
// (tools/peak_gemm.py reports it next to the library INT8 / FP16 peaks.)
extern "C" int samp_debug_gemm_peak(int kind, int m, int n, int k, int iters, float* ms) {
  return samp::guarded([&] {
    using namespace samp;
    const int eb = kind == KIND_I8 ? 1 : 2;
    SAMP_REQUIRE(m % 128 == 0 && n % 256 == 0 && (k * eb) % 128 == 0 && iters >= 1, SAMP_E_DIMENSION,
                 "peak gemm needs m % 128, n % 256, k*elt % 128 == 0");
    void *da, *db, *dc;
    SAMP_CUDA(cudaMalloc(&da, size_t(m) * k * eb));
    SAMP_CUDA(cudaMalloc(&db, size_t(n) * k * eb));
    SAMP_CUDA(cudaMalloc(&dc, size_t(m) * n * 4));
    SAMP_CUDA(cudaMemset(da, 0x11, size_t(m) * k * eb));
    SAMP_CUDA(cudaMemset(db, 0x22, size_t(n) * k * eb));
    CUtensorMap ma, mb;
    if (kind == KIND_I8) {
      ma = tmap_i8(da, m, k, k, 128, 128);
      mb = tmap_i8(db, n, k, k, 128, 256);
    } else {
      ma = tmap_f16(da, m, k, k, 64, 128);
      mb = tmap_f16(db, n, k, k, 64, 256);
    }
    EpiStoreAcc::Params p{dc, n};
    auto launch = [&]() {
      return kind == KIND_I8 ? launch_gemm<KIND_I8, 256, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, k * eb, p, 0)
                             : launch_gemm<KIND_F16, 256, 4, 1, 4, EpiStoreAcc>(ma, mb, m, n, k * eb, p, 0);
    };
    SAMP_CUDA(launch());
    SAMP_CUDA(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, 0);
    for (int i = 0; i < iters; ++i) SAMP_CUDA(launch());
    cudaEventRecord(b, 0);
    SAMP_CUDA(cudaEventSynchronize(b));
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    *ms = t / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dc);
  });
}
