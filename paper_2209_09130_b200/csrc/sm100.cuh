// sm_100a primitives: mbarrier, TMA, tcgen05 (TMEM alloc / MMA / ld / st),
// UMMA shared-memory + instruction descriptors, cluster barriers and DSMEM.
// Inline PTX only (no CUTLASS); bit layouts follow the PTX ISA tcgen05
// "shared memory descriptor" and "instruction descriptor" tables.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

namespace samp {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() {
  return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 %%rx;\n .reg .pred %%px;\n"
      " elect.sync %%rx|%%px, %1;\n @%%px mov.s32 %0, 1;\n}\n"
      : "+r"(pred) : "r"(0xffffffffu));
  return pred != 0;
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_addr(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting thread is parked until the phase
// completes (or the hint expires) instead of re-issuing try_wait every few cycles,
// which would steal issue slots from the warps doing the work on the same SM sub-partition
#ifndef SAMP_MBAR_HINT_NS
#define SAMP_MBAR_HINT_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if defined(SAMP_MBAR_SPIN)   // measurement: test_wait spin
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n"
      :: "r"(smem_addr(bar)), "r"(parity) : "memory");
#elif SAMP_MBAR_HINT_NS > 0
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n}\n"
      :: "r"(smem_addr(bar)), "r"(parity), "r"(SAMP_MBAR_HINT_NS) : "memory");
#else
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n"
      :: "r"(smem_addr(bar)), "r"(parity) : "memory");
#endif
}

// one try_wait (returns whether the phase with `parity` has completed)
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P1;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      " selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// non-blocking probe (mbarrier.test_wait never suspends; try_wait may park the thread for a
// system-dependent time when the phase is incomplete, which an event loop polling several
// barriers cannot afford)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P1;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      " selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// Long waits (microseconds: a warp waiting for another role's whole phase) back off with
// __nanosleep so the spinning warp does not take issue slots from the warps doing the
// work on its SM sub-partition (ncu: 8.5% of the attention kernel's instructions were the
// MMA warp's try_wait loop).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ns = 64;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 512 ? 2 * ns : 512;
  }
}

// Long waits with a suspend-time hint: the waiting warp is parked by the hardware until the
// phase completes (or the hint expires) instead of re-issuing try_wait / nanosleep, so
// waiting warps take no issue slots from the warps sharing their SM sub-partition.
__device__ __forceinline__ void mbar_wait_park(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n}\n"
      :: "r"(smem_addr(bar)), "r"(parity), "r"(1000000) : "memory");
}

// ------------------------------------------------------------------ PDL
// Programmatic dependent launch.  Every kernel is launched with programmatic stream
// serialization, so it may start while its predecessor is still running:
//   pdl_trigger()  (one thread per CTA; in the tcgen05 kernels the MMA issuer once its
//                  last MMA is issued, measured better than triggering at kernel start:
//                  1.18 vs 1.22 ms per bench step, 0.69 vs 0.78 ms batch-1) lets the next
//                  kernel's CTAs launch once every CTA of this grid has triggered or exited;
//   pdl_wait()     blocks until the predecessor grid has completed and its writes are
//                  visible.  It precedes every global access that touches activations
//                  (reads of earlier kernels' outputs and all writes); only constant
//                  data (weights, tables, the geometry uploaded before the forward) and
//                  smem/TMEM set-up happen before it.
// A chain of triggered-but-waiting kernels can therefore be resident at once; TMEM is
// allocated before the trigger so an allocation never waits on a later grid.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ cross-grid row-tile flags
// A producer grid publishes finished row tiles (counter += 1 per finished piece, release at
// GPU scope after a CTA barrier, the CUTLASS semaphore pattern); a consumer grid launched
// early (PDL trigger at the producer's start) acquires the counters of the tiles it reads
// instead of waiting for the whole producer grid (griddepcontrol.wait).  The consumer reads
// the tiles by TMA (async proxy): proxy fence after the acquire.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// spin until cnt[t] >= target for t in [lo, hi]; a flag that never arrives (a producer that
// was not launched) traps after ~2 s instead of hanging the GPU
__device__ __forceinline__ void wait_tile_flags(const int* cnt, int lo, int hi, int target) {
  const unsigned long long t0 = globaltimer();
  for (int t = lo; t <= hi; ++t) {
    while (ld_acquire_gpu(cnt + t) < target) {
      __nanosleep(64);
      if (globaltimer() - t0 > 2000000000ull) __trap();
    }
  }
  fence_proxy_async_global();
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
         "r"(smem_addr(bar))
      : "memory");
}
// bulk (non-tensor) copy global -> this CTA's smem, completing `bytes` on an mbarrier
// (16-byte aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// TMA tile store smem -> global (bulk group): the whole box in one instruction, clipped at the
// tensor's bounds; the issuing thread waits for the smem reads before the buffer is reused
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(src)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// generic-proxy smem writes -> visible to the async proxy (UMMA operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_addr(slot)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

enum MmaKind { KIND_I8 = 0, KIND_F16 = 1 };

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major; issued by one thread.
template <int KIND>
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (KIND == KIND_I8) {
    asm volatile(
        "{\n .reg .pred P1;\n setp.ne.b32 P1, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, P1;\n}\n"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred P1;\n setp.ne.b32 P1, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, P1;\n}\n"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
  }
}
// mbarrier arrives once every previously issued tcgen05.mma of this thread completes
// TMA load multicast to the CTAs of `mask` (same smem offset / mbarrier offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      :: "r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
         "r"(smem_addr(bar)), "h"(mask)
      : "memory");
}
// MMA completion arrives on the mbarrier at this offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(smem_addr(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_addr(bar)) : "memory");
}

// Instruction descriptor (PTX ISA tcgen05 "Instruction descriptor", kind::f16 / kind::i8):
//  [4,6) D format (1=F32, 2=S32)  [7,10) A fmt  [10,13) B fmt  [15] A MN-major  [16] B MN-major
//  [17,23) N>>3  [24,29) M>>4
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n, bool b_mn_major = false) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool b_mn_major = false) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// Shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), layout [61,64) (2 = 128B swizzle, 4 = 64B, 6 = 32B, 0 = none).
enum SwizzleMode { SW_NONE = 0, SW_128B = 2, SW_64B = 4, SW_32B = 6 };
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                               uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFFu) >> 4);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7u) << 61;
  return d;
}
// K-major, 128B-swizzled tile: rows of 128 B, 8-row (1024 B) atoms stacked densely.
__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) { return make_sdesc(saddr, 16, 1024, SW_128B); }
// K-major, 64B-swizzled tile: rows of 64 B, 8-row (512 B) atoms.
__device__ __forceinline__ uint64_t sdesc_k_sw64(uint32_t saddr) { return make_sdesc(saddr, 16, 512, SW_64B); }
// MN-major, 64B-swizzled tile whose MN extent is exactly 64 B: K rows of 64 B, 8-row atoms.
__device__ __forceinline__ uint64_t sdesc_mn_sw64(uint32_t saddr) { return make_sdesc(saddr, 512, 512, SW_64B); }

// TMEM -> registers: warp reads its 32 lanes x N consecutive 32-bit columns.
#define SAMP_R8(b) "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), \
                   "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : SAMP_R8(0) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : SAMP_R8(0), SAMP_R8(8) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : SAMP_R8(0), SAMP_R8(8), SAMP_R8(16), SAMP_R8(24) : "r"(taddr));
}
#undef SAMP_R8
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

#define SAMP_W8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), \
                   "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(taddr), SAMP_W8(0), SAMP_W8(8), SAMP_W8(16), SAMP_W8(24) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), SAMP_W8(0) : "memory");
}
#undef SAMP_W8
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ clusters / DSMEM
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// read a float from the same smem offset in CTA `rank` of this cluster
__device__ __forceinline__ float dsmem_ld_f32(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t mapa_rank(const void* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(local)), "r"(rank));
  return remote;
}
// asynchronous remote store whose completion is a complete_tx on the destination CTA's
// mbarrier (data and barrier live in the same CTA: no cluster-scope fence, which would
// compile to MEMBAR.ALL.GPU + L1 invalidation and measured 1.5x slower per tile)
__device__ __forceinline__ void st_async_f32(uint32_t remote, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               :: "r"(remote), "r"(__float_as_uint(v)), "r"(remote_bar) : "memory");
}

// ------------------------------------------------------------------ host: launches
// SAMP_NO_PDL=1 disables the programmatic-serialization attribute (A/B measurements).
inline bool pdl_enabled() {
  static const bool on = std::getenv("SAMP_NO_PDL") == nullptr;
  return on;
}

// cudaLaunchKernelEx with programmatic stream serialization (+ optional cluster dims)
// Every hot-path kernel asks for the maximum shared-memory carveout: kernels that would
// otherwise get different L1/shared splits force the SMs to drain and reconfigure between
// consecutive launches (SAMP_NO_CARVEOUT=1 leaves the driver's choice, A/B only).
template <class K>
inline void max_carveout_once(K* kern) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured == dev) return;
  configured = dev;
  if (std::getenv("SAMP_NO_CARVEOUT") == nullptr)
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared));
}

template <class... KArgs, class... Args>
inline cudaError_t launch_ex_cl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                dim3 cluster, Args&&... args) {
  max_carveout_once(kern);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster.x * cluster.y * cluster.z > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster.x;
    attr[n].val.clusterDim.y = cluster.y;
    attr[n].val.clusterDim.z = cluster.z;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <class... KArgs, class... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             int cluster_x, Args&&... args) {
  return launch_ex_cl(kern, grid, block, smem, st, dim3(cluster_x, 1, 1), std::forward<Args>(args)...);
}

}  // namespace samp
