// Latency of a kernel-to-kernel dependency on B200: griddepcontrol.wait (PDL) vs a global
// release/acquire flag.  Kernel A (grid G) does a little work, records %globaltimer at its
// end; kernel B (launched with programmatic stream serialization, triggered at A's start)
// records the time its dependency wait returns.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long t_end[4096], t_wake[4096];
__device__ unsigned int flag;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void producer(int use_flag, int spin) {
  asm volatile("griddepcontrol.launch_dependents;");
  // some work
  float x = threadIdx.x;
  for (int i = 0; i < spin; ++i) x = x * 1.0001f + 0.5f;
  if (x == 12345.f) t_end[4095] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    t_end[blockIdx.x] = gt();
    if (use_flag) {
      __threadfence();
      atomicAdd(&flag, 1u);
    }
  }
}

__global__ void consumer(int use_flag, unsigned target) {
  if (use_flag) {
    if (threadIdx.x == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&flag));
      } while (v < target);
    }
    __syncthreads();
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 0) t_wake[blockIdx.x] = gt();
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int G : {8, 148}) {
    for (int use_flag = 0; use_flag < 2; ++use_flag) {
      double acc = 0, accmax = 0;
      const int reps = 20;
      for (int r = 0; r < reps; ++r) {
        unsigned zero = 0;
        cudaMemcpyToSymbol(flag, &zero, 4);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, producer, use_flag, 20000);
        cudaLaunchKernelEx(&cfg, consumer, use_flag, unsigned(G));
        cudaStreamSynchronize(st);
        unsigned long long e[4096], w[4096];
        cudaMemcpyFromSymbol(e, t_end, sizeof(e));
        cudaMemcpyFromSymbol(w, t_wake, sizeof(w));
        unsigned long long emax = 0, wmin = ~0ull, wmax = 0;
        for (int i = 0; i < G; ++i) { emax = e[i] > emax ? e[i] : emax; wmin = w[i] < wmin ? w[i] : wmin; wmax = w[i] > wmax ? w[i] : wmax; }
        if (r >= 5) { acc += double(wmin) - double(emax); accmax += double(wmax) - double(emax); }
      }
      printf("grid %3d %s: first consumer wakes %.2f us after the producer's last end (last wakes %.2f us)\n", G,
             use_flag ? "flag (release/acquire)" : "griddepcontrol.wait  ", acc / (reps - 5) / 1e3, accmax / (reps - 5) / 1e3);
    }
  }
  return 0;
}
