// Numerics validation entry points (tests only): the branch-free quantize / divide used
// by every epilogue against the IEEE-divide formulation, exhaustively over all 2^32
// float bit patterns, and device evaluation of exp / tanh / GELU for oracle comparison.
#include "host_util.h"
#include "numerics.cuh"

namespace samp {

__device__ __forceinline__ float np_expf_ieee(float x) {  // np_expf with __fdiv_rn
  if (!(x < 88.72283935546875f)) return x != x ? x : __int_as_float(0x7f800000);
  if (x <= -103.97208404541015625f) return 0.0f;
  const float magic = 12582912.0f;
  float k = __fmul_rn(x, 1.442695040888963407359924681001892137f);
  k = __fsub_rn(__fadd_rn(k, magic), magic);
  float r = __fmaf_rn(k, -6.93145752e-1f, x);
  r = __fmaf_rn(k, -1.42860677e-6f, r);
  r = __fmaf_rn(k, 0.0f, r);
  float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
  num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
  num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
  num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
  num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);
  float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
  den = __fmaf_rn(den, r, 1.0f);
  return scale_pow2(__fdiv_rn(num, den), static_cast<int>(k));
}

__global__ void quant_exhaustive_kernel(const float* scales, int n, unsigned long long* bad, const X2 k) {
  unsigned long long local = 0;
  for (int si = 0; si < n; ++si) {
    const float s = scales[si];
    const Recip r = make_recip(s);
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < (1ull << 32);
         u += uint64_t(gridDim.x) * blockDim.x) {
      const float x = __uint_as_float(uint32_t(u));
      if (x != x) continue;  // NaN codes are unspecified in the reference (clip keeps NaN)
      const int want = quant_i8(x, s);
      local += quant_fast(x, r) != want;
      const bool bounded = fabsf(x) < 1.1529215e18f;   // |x| < 2^60
      if (bounded) local += quant_bounded(x, r) != want;
      // packed path: byte 0 = x, byte 1 = -x, byte 2 = 0, byte 3 = x (bounded variant when legal)
      const uint32_t pk = trunc_pack4_s8(quant_pre_fast(x, r), quant_pre_fast(-x, r), 0.0f,
                                         bounded ? quant_pre_bounded(x, r) : quant_pre_fast(x, r));
      local += int(int8_t(pk & 0xffu)) != want;
      local += int(int8_t((pk >> 8) & 0xffu)) != quant_i8(-x, s);
      local += ((pk >> 16) & 0xffu) != 0u;
      local += int(int8_t(pk >> 24)) != want;
      if (bounded) {   // FFMA2 pair form (x, -x)
        const float2 q2 = quant_pre2(f2(x, -x), r, k);
        const uint32_t p2 = trunc_pack4_s8(q2.x, q2.y, 0.0f, 0.0f);
        local += (int(int8_t(p2 & 0xffu)) != want) + (int(int8_t((p2 >> 8) & 0xffu)) != quant_i8(-x, s));
      }
    }
  }
  atomicAdd(bad, local);
}

__global__ void div_exhaustive_kernel(const float* divisors, int n, unsigned long long* bad) {
  // quotient identity over the operand ranges the kernels use it for: x in [0, 1] (softmax
  // numerators) and any normal x with |x| in [2^-60, 2^60]
  unsigned long long local = 0;
  for (int si = 0; si < n; ++si) {
    const Recip r = make_recip(divisors[si]);
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < (1ull << 32);
         u += uint64_t(gridDim.x) * blockDim.x) {
      const float x = __uint_as_float(uint32_t(u));
      const float ax = fabsf(x);
      if (!(ax >= 8.6736174e-19f && ax <= 1.1529215e18f)) continue;
      const float a = div_fast(x, r), b = __fdiv_rn(x, divisors[si]);
      local += __float_as_uint(a) != __float_as_uint(b);
    }
  }
  atomicAdd(bad, local);
}

__global__ void exp_exhaustive_kernel(unsigned long long* bad) {
  unsigned long long local = 0;
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < (1ull << 32);
       u += uint64_t(gridDim.x) * blockDim.x) {
    const float x = __uint_as_float(uint32_t(u));
    const float a = np_expf(x), b = np_expf_ieee(x);
    local += (__float_as_uint(a) != __float_as_uint(b)) && !(a != a && b != b);
    if (x <= 0.0f) local += __float_as_uint(np_expf_nonpos(x)) != __float_as_uint(b);
  }
  atomicAdd(bad, local);
}

// np_exp2_fast (both reciprocal variants) against np_expf with the IEEE divide for every
// float in [NP_EXP2_FAST_MIN, 0] (both zeros included); bad[0] = unrefined, bad[1] = refined
__global__ void exp2_fast_exhaustive_kernel(unsigned long long* bad, const X2 k) {
  const uint32_t hi = __float_as_uint(NP_EXP2_FAST_MIN);
  unsigned long long l0 = 0, l1 = 0;
  for (uint64_t u = 0x80000000ull + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u <= hi + 1ull;
       u += uint64_t(gridDim.x) * blockDim.x) {
    const float x = u == hi + 1ull ? 0.0f : __uint_as_float(uint32_t(u));   // the extra slot = +0
    const float want = np_expf_ieee(x);
    const float2 a = np_exp2_fast<false>(f2(x, x), k), b = np_exp2_fast<true>(f2(x, x), k);
    l0 += (__float_as_uint(a.x) != __float_as_uint(want)) + (__float_as_uint(a.y) != __float_as_uint(want));
    l1 += (__float_as_uint(b.x) != __float_as_uint(want)) + (__float_as_uint(b.y) != __float_as_uint(want));
  }
  atomicAdd(bad, l0);
  atomicAdd(bad + 1, l1);
}

// gelu8_finite (and its FFMA2 form) against gelu_ref over every float with |x| < 1e12
// (the host-proven domain)
__global__ void gelu_finite_exhaustive_kernel(unsigned long long* bad, const X2 k) {
  __shared__ TanhTable tt;
  load_tanh_table(&tt, threadIdx.x, blockDim.x);
  __syncthreads();
  unsigned long long local = 0;
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < (1ull << 29);
       g += uint64_t(gridDim.x) * blockDim.x) {
    float v[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x[u] = __uint_as_float(uint32_t(g * 8 + u));
      if (!(fabsf(x[u]) < 1e12f)) x[u] = 0.0f;
      v[u] = x[u];
    }
    float v2[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v2[u] = v[u];
    gelu8_finite(v, &tt);
    gelu8_finite_x2(v2, &tt, k);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t want = __float_as_uint(gelu_ref(x[u], &tt));
      local += (__float_as_uint(v[u]) != want) + (__float_as_uint(v2[u]) != want);
    }
  }
  atomicAdd(bad, local);
}

__global__ void unary_kernel(int fn, const float* x, float* y, long n) {
  __shared__ TanhTable tt;
  load_tanh_table(&tt, threadIdx.x, blockDim.x);
  __syncthreads();
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    const float v = x[i];
    y[i] = fn == 0 ? np_expf(v) : fn == 1 ? np_tanhf(v, &tt) : gelu_ref(v, &tt);
  }
}

static unsigned long long run_count(void (*launch)(unsigned long long*)) {
  unsigned long long* d;
  SAMP_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  SAMP_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
  launch(d);
  SAMP_CUDA(cudaGetLastError());
  SAMP_CUDA(cudaDeviceSynchronize());
  unsigned long long h = 0;
  SAMP_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(d);
  return h;
}

static float* g_vals = nullptr;
static int g_n = 0;

}  // namespace samp

using namespace samp;

extern "C" int samp_debug_quant_exhaustive(const float* scales, int n, unsigned long long* mismatches) {
  return guarded([&] {
    SAMP_CUDA(cudaMalloc(&g_vals, n * sizeof(float)));
    SAMP_CUDA(cudaMemcpy(g_vals, scales, n * sizeof(float), cudaMemcpyHostToDevice));
    g_n = n;
    *mismatches = run_count([](unsigned long long* d) { quant_exhaustive_kernel<<<148 * 8, 256>>>(g_vals, g_n, d, x2_consts()); });
    cudaFree(g_vals);
  });
}

extern "C" int samp_debug_div_exhaustive(const float* divisors, int n, unsigned long long* mismatches) {
  return guarded([&] {
    SAMP_CUDA(cudaMalloc(&g_vals, n * sizeof(float)));
    SAMP_CUDA(cudaMemcpy(g_vals, divisors, n * sizeof(float), cudaMemcpyHostToDevice));
    g_n = n;
    *mismatches = run_count([](unsigned long long* d) { div_exhaustive_kernel<<<148 * 8, 256>>>(g_vals, g_n, d); });
    cudaFree(g_vals);
  });
}

extern "C" int samp_debug_exp_exhaustive(unsigned long long* mismatches) {
  return guarded([&] {
    *mismatches = run_count([](unsigned long long* d) { exp_exhaustive_kernel<<<148 * 8, 256>>>(d); });
  });
}

extern "C" int samp_debug_exp2_fast_exhaustive(unsigned long long* mismatches /* [2] */) {
  return guarded([&] {
    unsigned long long* d;
    SAMP_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
    SAMP_CUDA(cudaMemset(d, 0, 2 * sizeof(unsigned long long)));
    exp2_fast_exhaustive_kernel<<<148 * 8, 256>>>(d, x2_consts());
    SAMP_CUDA(cudaGetLastError());
    SAMP_CUDA(cudaDeviceSynchronize());
    SAMP_CUDA(cudaMemcpy(mismatches, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

extern "C" int samp_debug_gelu_finite_exhaustive(unsigned long long* mismatches) {
  return guarded([&] {
    *mismatches = run_count([](unsigned long long* d) { gelu_finite_exhaustive_kernel<<<148 * 8, 256>>>(d, x2_consts()); });
  });
}

extern "C" int samp_debug_unary(int fn, const float* x, float* y, long n) {
  return guarded([&] {
    float *dx, *dy;
    SAMP_CUDA(cudaMalloc(&dx, n * 4));
    SAMP_CUDA(cudaMalloc(&dy, n * 4));
    SAMP_CUDA(cudaMemcpy(dx, x, n * 4, cudaMemcpyHostToDevice));
    unary_kernel<<<148 * 4, 256>>>(fn, dx, dy, n);
    SAMP_CUDA(cudaGetLastError());
    SAMP_CUDA(cudaMemcpy(y, dy, n * 4, cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dy);
  });
}
