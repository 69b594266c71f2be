// Issue-rate microbenchmark for the epilogue instruction mix (B200, sm_100a).
// Each thread runs 8 independent chains of one op; 148*8 CTAs x 256 threads.
// Prints warp-instructions per cycle per SM for each op.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

constexpr int ITERS = 4096;

#define KERNEL(name, T, init, body)                                              \
  __global__ void name(T* out, float s) {                                        \
    T v[8];                                                                      \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) v[i] = init;                   \
    for (int it = 0; it < ITERS; ++it) {                                         \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) { body; }                    \
    }                                                                            \
    T acc = v[0];                                                                \
    _Pragma("unroll") for (int i = 1; i < 8; ++i) acc = acc + v[i];              \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                            \
  }

__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

KERNEL(k_ffma, float, s * (threadIdx.x + i), v[i] = __fmaf_rn(v[i], s, 0.5f * s))
KERNEL(k_ffma_reg, float, s * (threadIdx.x + i), v[i] = __fmaf_rn(v[i], v[(i + 1) & 7], s))
KERNEL(k_fmul, float, s * (threadIdx.x + i), v[i] = __fmul_rn(v[i], s))
KERNEL(k_fadd, float, s * (threadIdx.x + i), v[i] = __fadd_rn(v[i], s))
KERNEL(k_ffma2, float2, make_float2(s * threadIdx.x, s * i),
       v[i] = __ffma2_rn(v[i], make_float2(s, s), make_float2(0.5f * s, s)))
KERNEL(k_ffma2_reg, float2, make_float2(s * threadIdx.x, s * i),
       v[i] = __ffma2_rn(v[i], v[(i + 1) & 7], make_float2(s, s)))
KERNEL(k_ex2, float, s * (threadIdx.x + i), asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i])))
KERNEL(k_rcp, float, s * (threadIdx.x + i), asm("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[i])))
KERNEL(k_i2f, float, s * (threadIdx.x + i), v[i] = __int2float_rn(__float_as_int(v[i])))
KERNEL(k_f2i, float, s * (threadIdx.x + i), v[i] = __int_as_float(__float2int_rz(v[i])))
KERNEL(k_lop, float, s * (threadIdx.x + i), v[i] = __int_as_float(__float_as_int(v[i]) ^ (__float_as_int(s) | 3)))
KERNEL(k_iadd, float, s * (threadIdx.x + i), v[i] = __int_as_float(__float_as_int(v[i]) + __float_as_int(s)))
KERNEL(k_fmnmx, float, s * (threadIdx.x + i), v[i] = fminf(v[i], s))

template <class T>
void run(const char* name, void (*kern)(T*, float), int opsPerIter) {
  T* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<148 * 8, 256>>>(out, 1.0001f);
  cudaEventRecord(a);
  kern<<<148 * 8, 256>>>(out, 1.0001f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_instr = 148.0 * 8 * 256 / 32 * ITERS * 8 * opsPerIter;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-12s %7.3f ms  %6.2f warp-instr/clk/SM  (%5.2f per SMSP)\n", name, ms, warp_instr / cycles / 148,
         warp_instr / cycles / 148 / 4);
  cudaFree(out);
}

int main() {
  run("FFMA imm", k_ffma, 1);
  run("FFMA reg", k_ffma_reg, 1);
  run("FMUL", k_fmul, 1);
  run("FADD", k_fadd, 1);
  run("FFMA2 imm", k_ffma2, 1);
  run("FFMA2 reg", k_ffma2_reg, 1);
  run("MUFU.EX2", k_ex2, 1);
  run("MUFU.RCP", k_rcp, 1);
  run("I2F", k_i2f, 1);
  run("F2I", k_f2i, 1);
  run("LOP3", k_lop, 1);
  run("IADD", k_iadd, 1);
  run("FMNMX", k_fmnmx, 1);
  return 0;
}
