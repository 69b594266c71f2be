// Does a 320-thread CTA with ~96 / ~106 / ~114 KB of dynamic shared memory run two per SM on
// B200, and what does the occupancy API report?  Each CTA spins ~20 us and records its SM and
// start/end %globaltimer; the maximum number of CTAs overlapping on one SM is the residency.
// nvcc -gencode arch=compute_100a,code=sm_100a -o occ_probe occ_probe.cu && ./occ_probe
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(320, 2) spin(unsigned long long* rec) {
  extern __shared__ unsigned char sm[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  sm[threadIdx.x] = 1;
  unsigned long long t = t0;
  while (t - t0 < 20000) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  __syncthreads();
  if (threadIdx.x == 0) {
    rec[3 * blockIdx.x] = smid;
    rec[3 * blockIdx.x + 1] = t0;
    rec[3 * blockIdx.x + 2] = t;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 2 * sms;
  unsigned long long* d;
  cudaMalloc(&d, grid * 3 * 8);
  for (int carve = 0; carve < 2; ++carve) {
    if (carve) cudaFuncSetAttribute(spin, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (int smem : {96128, 100480, 108672, 116864}) {
      cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int occ = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spin, 320, smem);
      spin<<<grid, 320, smem>>>(d);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned long long> h(grid * 3);
      cudaMemcpy(h.data(), d, grid * 3 * 8, cudaMemcpyDeviceToHost);
      int maxc = 0;
      for (int i = 0; i < grid; ++i) {
        int c = 0;
        for (int j = 0; j < grid; ++j)
          if (h[3 * j] == h[3 * i] && h[3 * j + 1] < h[3 * i + 2] && h[3 * i + 1] < h[3 * j + 2]) ++c;
        maxc = std::max(maxc, c);
      }
      unsigned long long lo = ~0ull, hi = 0;
      for (int i = 0; i < grid; ++i) { lo = std::min(lo, h[3 * i + 1]); hi = std::max(hi, h[3 * i + 2]); }
      std::printf("carveout-attr %d smem %6d: occupancy API %d, max co-resident per SM %d, span %.1f us (%s)\n", carve,
                  smem, occ, maxc, (hi - lo) / 1e3, cudaGetErrorString(e));
    }
  }
  return 0;
}
