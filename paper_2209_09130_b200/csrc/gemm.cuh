// Warp-specialised tcgen05 GEMM for the encoder's four projections.
//
//   C[M, N] = A[M, K] * W[K, N]   A: activations, row-major [M][K] (K-major)
//                                 W: weights stored transposed Wt[N][K] (K-major)
//
// One CTA computes a 128 x BN tile (UMMA M=128, N=BN, cta_group::1); int32 (kind::i8)
// or f32 (kind::f16) accumulators live in TMEM.  Warp roles (64 + 32*NE threads):
//   warp 0     TMA producer: 128B-swizzled A/B k-blocks (128 bytes of K) into a
//              STAGES-deep smem ring, completion on full[] mbarriers
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (4 MMAs of 32 B of K
//              per k-block); tcgen05.commit frees ring slots and finally signals tmem_full
//   warps 2..  NE epilogue warps.  TMEM lane quarter q may only be read by warps with
//              warp%4 == q, so thread (warp, lane) owns accumulator row 32*(warp%4)+lane and
//              the column half (warp-2)/4 when NE == 8.  Owning a (half) row per thread is
//              what lets the fused LayerNorm epilogue reproduce numpy's pairwise tree
//              sequentially, bit-for-bit (numerics.cuh): NE == 8 is only used when the two
//              column halves are exact subtrees of that tree.
// The epilogues dominate (bit-exact GELU / quantize / LayerNorm cost far more than the
// MMAs at BERT shapes), so the ring is kept small enough (<= ~100 KB) for two CTAs per SM:
// one CTA's epilogue overlaps the other's TMA + MMA main loop.
// Row-complete epilogues (LayerNorm over N = hidden) run as a cluster of CLUSTER CTAs
// along N; each CTA reduces its BN columns (an exact numpy subtree) and partial sums
// are exchanged through DSMEM.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "numerics.cuh"
#include "sm100.cuh"

namespace samp {

constexpr int GEMM_BM = 128;
constexpr int GEMM_EPI_WARP0 = 2;

__host__ __device__ constexpr int tmem_cols_for(int n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}

template <int BN, int STAGES, int EPI_SMEM>
struct GemmLayout {
  static constexpr int A_BYTES = GEMM_BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = STAGES * A_BYTES;
  static constexpr int BAR_OFF = B_OFF + STAGES * B_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 8 * (2 * STAGES + 2) + 8;  // + tmem slot
  static constexpr int EPI_OFF_ALIGNED = (EPI_OFF + 127) & ~127;
  static constexpr int TOTAL = EPI_OFF_ALIGNED + EPI_SMEM + 1024;     // + alignment slack
};

// Shared epilogue context: where this thread's accumulator (half) row lives.
struct EpiCtx {
  uint32_t taddr;    // TMEM address of (this thread's lane, column c0)
  int row;           // global output row
  int tile_row;      // 0..127
  int n0;            // first output column of the tile
  int c0;            // first tile column this thread owns
  int ncols;         // columns this thread owns (BN or BN/2)
  int half;          // 0/1 (NE == 8) or 0
  int M;             // valid rows
  int ep_tid;        // 0 .. 32*NE-1
  int ne_threads;    // 32*NE
  unsigned long long* sub = nullptr;   // measurement: epilogue sub-phase stamps (thread 0 only)
  uint8_t* stage = nullptr;            // free smem (the drained operand ring) for a TMA-stored tile
  uint8_t* ring = nullptr;             // the operand ring's A slots (TMA-loaded residual boxes)
  int res_slot0 = 0, stages = 1;       // residual box k sits in A slot (res_slot0 + k) % stages
  const uint8_t* table = nullptr;      // persistent kernels: the shared read-only table (GELU
                                       // tanh); smem then holds only the tile's bias
  const uint32_t* kpart = nullptr;     // KS2: the other K half's accumulators [128][BN] (smem)
  uint64_t* kpart_bar = nullptr;       // ... complete when all of them landed
};

// epilogues that can take their f32 residual tile by TMA into the drained ring (EpiResLNT)
template <class E, class = void> struct has_res_tma : std::false_type {};
template <class E> struct has_res_tma<E, std::void_t<decltype(E::kResTma)>> : std::true_type {};
// epilogues whose Params carry row-tile flags (ResLNParams)
template <class E, class = void> struct has_dep : std::false_type {};
template <class E> struct has_dep<E, std::void_t<decltype(std::declval<typename E::Params>().dep_cnt)>> : std::true_type {};
template <class Epi>
__device__ __forceinline__ bool dep_set(const typename Epi::Params& ep) {
  if constexpr (has_dep<Epi>::value) return ep.dep_cnt != nullptr;
  else return false;
}

// named barrier among the epilogue warps only
__device__ __forceinline__ void epi_bar_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" :: "r"(nthreads) : "memory");
}

// Phase stamps (measurement only).  When a launch gets a non-null buffer, CTA b writes
// GEMM_STAMPS u64 at stamps[b * GEMM_STAMPS]: smid, then %globaltimer (ns) at kernel
// start, first ring slot full, last ring slot full, accumulator complete, epilogue done,
// exit.  The host sets g_gemm_stamps before a launch (profiling mode, no graphs).
constexpr int GEMM_STAMPS = 8, GEMM_STAMP_CTAS = 1024;
inline unsigned long long* g_gemm_stamps = nullptr;

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// rings <= ~110 KB run two CTAs per SM (register cap ~96); deeper rings one CTA per SM
template <int BN, int STAGES>
struct GemmOcc {
  static constexpr int value = STAGES * (GEMM_BM + BN) * 128 <= 110 * 1024 ? 2 : 1;
};

// MC (CLUSTER > 1): the cluster's CTAs share the A row tile; rank r loads rows
// [r*128/CLUSTER, (r+1)*128/CLUSTER) of every stage multicast to all ranks (map_a then has
// 128/CLUSTER-row boxes), and each MMA commit frees the stage in every rank
// KS2 (small batches, LayerNorm epilogues): the K range is split over the two z-halves of a
// (CLUSTER x 1 x 2) cluster; the z = 1 CTA pushes its accumulator tile into its z = 0
// partner's shared memory (st.async, completing on the partner's mbarrier) and the partner
// adds it before the epilogue — int32 adds are exact, so INT8 results are unchanged
template <int BN, bool KS2> __host__ __device__ constexpr int ks2_bytes() { return KS2 ? 128 * BN * 4 + 64 : 0; }

template <int KIND, int BN, int STAGES, int CLUSTER, int NE, class Epi, bool MC = false, bool KS2 = false>
__global__ void __launch_bounds__(64 + 32 * NE, GemmOcc<BN, STAGES>::value)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            int M, int k_bytes, const __grid_constant__ typename Epi::Params ep, unsigned long long* stamps) {
  constexpr int EPI_BYTES = (Epi::template smem_bytes<BN>() + 127) / 128 * 128;
  using Lay = GemmLayout<BN, STAGES, EPI_BYTES + ks2_bytes<BN, KS2>()>;
  constexpr int TMEM_COLS = tmem_cols_for(BN);
  constexpr uint32_t IDESC = KIND == KIND_I8 ? idesc_i8(GEMM_BM, BN) : idesc_f16(GEMM_BM, BN);
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  static_assert(NE == 4 || (NE == 8 && ((BN / 2) % 32 == 0 || BN == 96)) || (NE == 16 && BN == 192), "epilogue split");
  constexpr bool MCAST = MC && CLUSTER > 1;
  constexpr int A_ROWS = GEMM_BM / (MCAST ? CLUSTER : 1);   // rows of A this CTA loads
  constexpr uint16_t MASK = uint16_t((1u << CLUSTER) - 1);

  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array keeps the shared address space visible
  // to the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  uint8_t* epi_smem = smem + Lay::EPI_OFF_ALIGNED;

  const uint32_t warp = warp_id();
  const int m0 = blockIdx.y * GEMM_BM;
  const int n0 = blockIdx.x * BN;
  // split-K (gridDim.z > 1, host guarantees z | k-blocks): this CTA's k-block range
  const int nk = k_bytes / 128 / int(gridDim.z);
  const int kb0 = int(blockIdx.z) * nk;
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned long long* stamp = stamps && cta < GEMM_STAMP_CTAS ? stamps + size_t(cta) * GEMM_STAMPS : nullptr;
  if (stamp && threadIdx.x == 0) {
    stamp[0] = smid();
    stamp[1] = globaltimer();
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MCAST ? CLUSTER : 1);
    }
    mbar_init(tmem_full, 1);
    if constexpr (KS2) mbar_init(reinterpret_cast<uint64_t*>(epi_smem + EPI_BYTES + 128 * BN * 4), 1);
    if constexpr (CLUSTER > 1) Epi::template cluster_init<BN>(epi_smem);
    fence_barrier_init();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  if constexpr (CLUSTER > 1) cluster_sync_all();   // peers' exchange barriers are initialised
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (elect_one()) {
      // coordinates are in elements: 128 bytes of K = 128 int8 or 64 f16
      auto kcol = [kb0](int kb) { return KIND == KIND_I8 ? (kb0 + kb) * 128 : (kb0 + kb) * 64; };
      // weights (B) do not depend on the previous kernel: fill the ring's B halves
      // while it drains, then wait for it and stream A
      const int pre = nk < STAGES ? nk : STAGES;
      const int arow = MCAST ? int(cluster_rank()) * A_ROWS : 0;
      auto load_a = [&](int s, int kb) {
        uint8_t* dst = smem + Lay::A_OFF + s * Lay::A_BYTES + arow * 128;
        if constexpr (MCAST) tma_load_2d_mc(dst, &map_a, kcol(kb), m0 + arow, &full[s], MASK);
        else tma_load_2d(dst, &map_a, kcol(kb), m0, &full[s]);
      };
      for (int kb = 0; kb < pre; ++kb) {
        mbar_expect_tx(&full[kb], Lay::A_BYTES + Lay::B_BYTES);
        tma_load_2d(smem + Lay::B_OFF + kb * Lay::B_BYTES, &map_b, kcol(kb), n0, &full[kb]);
      }
      if constexpr (has_dep<Epi>::value) {
        if (ep.dep_cnt) {
          const int m = m0 / GEMM_BM;
          wait_tile_flags(ep.dep_cnt, ep.dep_rt[2 * m], ep.dep_rt[2 * m + 1], ep.dep_target);
        } else {
          pdl_wait();
        }
      } else {
        pdl_wait();
      }
      for (int kb = 0; kb < pre; ++kb) load_a(kb, kb);
      for (int kb = pre; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);   // MCAST: every rank consumed the stage
        mbar_expect_tx(&full[s], Lay::A_BYTES + Lay::B_BYTES);
        load_a(s, kb);
        tma_load_2d(smem + Lay::B_OFF + s * Lay::B_BYTES, &map_b, kcol(kb), n0, &full[s]);
      }
      if constexpr (has_res_tma<Epi>::value && !MCAST && CLUSTER > 1) {
        if (ep.tma_res && (!KS2 || blockIdx.z == 0)) {   // the f32 residual tile into the next A slots as the MMAs drain them
          static_assert(GEMM_BM * 128 == 128 * 32 * 4, "one 32-column f32 box per A slot");
          uint64_t* rb = Epi::template res_bar<BN>(smem + Lay::EPI_OFF_ALIGNED);
          mbar_expect_tx(rb, (BN / 32) * Lay::A_BYTES);
          for (int k = 0; k < BN / 32; ++k) {
            const int kb = nk + k, s = kb % STAGES;
            mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
            tma_load_2d(smem + Lay::A_OFF + s * Lay::A_BYTES, &ep.map_res, n0 + 32 * k, m0, rb);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        tc_fence_after();
        if (stamp && (kb == 0 || kb == nk - 1)) stamp[kb == 0 ? 2 : 3] = globaltimer();
        const uint32_t a_base = smem_addr(smem + Lay::A_OFF + s * Lay::A_BYTES);
        const uint32_t b_base = smem_addr(smem + Lay::B_OFF + s * Lay::B_BYTES);
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K per 128B swizzle row
          mma_ss<KIND>(tmem, sdesc_k_sw128(a_base + 32 * k), sdesc_k_sw128(b_base + 32 * k), IDESC,
                       (kb | k) != 0);
        }
        if constexpr (MCAST) mma_commit_mc(&empty[s], MASK);
        else mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
      pdl_trigger();   // last MMA issued: the next kernel's prologue overlaps our epilogue
    }
    __syncwarp();
  } else {
    const int ep_tid = threadIdx.x - GEMM_EPI_WARP0 * 32;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = NE >= 8 ? int(warp - GEMM_EPI_WARP0) / 4 : 0;   // NE = 16: quarter rows 0..3
    const int tile_row = quarter * 32 + lane_id();
    const int c0 = half * (BN / (NE / 4));
    if constexpr (KS2) {
      if (blockIdx.z == 1) {   // second K half: push the accumulator tile to the z = 0 partner
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const uint32_t partner = cluster_rank() - CLUSTER;
        const uint32_t dst = mapa_rank(epi_smem + EPI_BYTES + (tile_row * BN + c0) * 4, partner);
        const uint32_t bar = mapa_rank(epi_smem + EPI_BYTES + 128 * BN * 4, partner);
        const uint32_t ta = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(c0);
#pragma unroll 1
        for (int col = 0; col < BN / (NE / 4); col += 16) {
          uint32_t r[16];
          tmem_ld16(ta + col, r);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                         :: "r"(dst + (col + 4 * q) * 4), "r"(r[4 * q]), "r"(r[4 * q + 1]), "r"(r[4 * q + 2]),
                            "r"(r[4 * q + 3]), "r"(bar) : "memory");
        }
        goto epilogue_done;
      }
      if (ep_tid == 0) mbar_expect_tx(reinterpret_cast<uint64_t*>(epi_smem + EPI_BYTES + 128 * BN * 4), 128 * BN * 4);
    }
    if (!dep_set<Epi>(ep)) pdl_wait();   // residual tiles / outputs belong to earlier kernels
    // idle during the main loop: stage this tile's epilogue operands in smem
    Epi::template prefetch<BN>(ep, epi_smem, m0, n0, M, ep_tid, 32 * NE);
    epi_bar_sync(32 * NE);
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (stamp && ep_tid == 0) stamp[4] = globaltimer();
    EpiCtx c{tmem + (uint32_t(quarter * 32) << 16) + uint32_t(c0), m0 + tile_row, tile_row, n0, c0,
             BN / (NE / 4), half, M, ep_tid, 32 * NE};
    // sub-phase stamps of CTA b < 512 go to the unused CTA slots 512 + b (tools/ln_phases.py)
    if (stamps && cta < 512 && ep_tid == 0) c.sub = stamps + size_t(512 + cta) * GEMM_STAMPS;
    c.stage = smem + Lay::A_OFF;   // every MMA has completed (tmem_full): the ring is free
    c.ring = smem + Lay::A_OFF;
    c.res_slot0 = nk % STAGES;
    c.stages = STAGES;
    if constexpr (KS2) {
      c.kpart = reinterpret_cast<const uint32_t*>(epi_smem + EPI_BYTES);
      c.kpart_bar = reinterpret_cast<uint64_t*>(epi_smem + EPI_BYTES + 128 * BN * 4);
    }
    Epi::template run<BN, CLUSTER, NE>(ep, c, epi_smem);
    if (stamp && ep_tid == 0) stamp[5] = globaltimer();
  }
epilogue_done:
  // non-epilogue warps mirror the epilogue's cluster barriers
  if (warp < GEMM_EPI_WARP0) {
    for (int i = 0; i < Epi::template cluster_barriers<CLUSTER>(); ++i) cluster_sync_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
  // MCAST: peers' last MMA commits arrive on our empty barriers; nobody exits before all did
  if constexpr (MCAST) cluster_sync_all();
  if (stamp && threadIdx.x == 0) stamp[6] = globaltimer();
}

__device__ __forceinline__ uint32_t pack4_i8(int a, int b, int c, int d) {
  return (uint32_t(a) & 0xffu) | ((uint32_t(b) & 0xffu) << 8) | ((uint32_t(c) & 0xffu) << 16) |
         (uint32_t(d) << 24);
}

__device__ __forceinline__ void store32_i8(int8_t* dst, const int (&q)[32]) {
  uint32_t w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = pack4_i8(q[4 * j], q[4 * j + 1], q[4 * j + 2], q[4 * j + 3]);
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// 32 pre-rounded quantize values (quant_pre_*) -> 32 int8 codes at dst
__device__ __forceinline__ void store32_pre(int8_t* dst, const float (&v)[32]) {
  uint32_t w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = trunc_pack4_s8(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

__device__ __forceinline__ void load_bias32(const float* b, float (&out)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(b) + j);
    out[4 * j] = v.x; out[4 * j + 1] = v.y; out[4 * j + 2] = v.z; out[4 * j + 3] = v.w;
  }
}

__device__ __forceinline__ void load_smem32(const float* src, float (&out)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = reinterpret_cast<const float4*>(src)[j];
    out[4 * j] = v.x; out[4 * j + 1] = v.y; out[4 * j + 2] = v.z; out[4 * j + 3] = v.w;
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// copy n floats gmem -> smem cooperatively.  n % 4 == 0 and 16-byte aligned ends (every
// caller stages BN-column slices): 16-byte cp.async, all in flight at once, so the epilogue
// operands cost one L2 round trip instead of one per loop iteration (ncu: the scalar loop's
// dependent loads were the LN GEMMs' top stall).  The caller waits (cp_async_wait_all).
__device__ __forceinline__ void stage_floats_async(float* dst, const float* src, int n, int tid, int nthreads) {
  for (int i = tid; i < n / 4; i += nthreads) cp_async16(dst + 4 * i, src + 4 * i);
}
__device__ __forceinline__ void stage_floats(float* dst, const float* src, int n, int tid, int nthreads) {
#ifdef SAMP_EXP_SCALAR_STAGE
  for (int i = tid; i < n; i += nthreads) dst[i] = __ldg(src + i);
#else
  stage_floats_async(dst, src, n, tid, nthreads);
  cp_async_commit();
  cp_async_wait_all();
#endif
}

// ------------------------------------------------------------------ epilogues
// SAMP_BIAS_GLOBAL: the QKV / FFN1 epilogues read their bias row straight from global
// memory (L1-resident, a warp reads one 64-byte span) instead of a per-tile smem copy, so
// the persistent kernel needs no per-tile barrier among its epilogue warps to recycle the
// smem copy and the warps drift independently between tiles.
#ifndef SAMP_BIAS_GLOBAL
#define SAMP_BIAS_GLOBAL 0
#endif
// Interface: smem_bytes<BN>(); prefetch<BN>(params, smem, m0, n0, M, tid, nthreads) runs in
// the epilogue warps while the main loop is in flight; run<BN, CLUSTER, NE>(params, ctx, smem).

// raw int32 / f32 accumulator store (kernel tests, parity of the accumulators)
struct EpiStoreAcc {
  struct Params {
    void* out;   // int32 (kind::i8) or float (kind::f16), row-major
    int ldc;     // elements
  };
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return 0; }
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  template <int BN> __device__ static void prefetch(const Params&, uint8_t*, int, int, int, int, int) {}
  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t*) {
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += 32) {
      uint32_t r[32];
      tmem_ld32(c.taddr + col, r);
      tmem_wait_ld();
      if (c.row < c.M) {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<uint32_t*>(p.out) + size_t(c.row) * p.ldc + c.n0 + c.c0 + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) dst[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
      }
    }
  }
};

// Split-K partial: the int32 accumulator tile is added into an int32 workspace with
// coalesced red.global.add (the tile is transposed through smem so a warp's 32 lanes hit
// 32 consecutive columns).  Integer addition is exact and order-independent, so the
// workspace holds exactly the full-K accumulator whatever the CTA order.  The consumer
// (ln_rows_kernel) re-zeroes the workspace rows it reads.
struct EpiSplitKAdd {
  struct Params {
    int* ws;     // [M][ldw]
    int ldw;
  };
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return 128 * (BN + 1) * 4; }
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  template <int BN> __device__ static void prefetch(const Params&, uint8_t*, int, int, int, int, int) {}
  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t* smem) {
    int* tile = reinterpret_cast<int*>(smem);   // [128][BN + 1]
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += 32) {
      uint32_t r[32];
      tmem_ld32(c.taddr + col, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) tile[c.tile_row * (BN + 1) + c.c0 + col + j] = int(r[j]);
    }
    epi_bar_sync(c.ne_threads);
    const int lane = c.ep_tid & 31, w = c.ep_tid >> 5, nw = c.ne_threads >> 5;
    for (int row = w; row < 128; row += nw) {
      const int m0 = c.row - c.tile_row;
      if (m0 + row >= c.M) break;
      int* dst = p.ws + size_t(m0 + row) * p.ldw + c.n0;
      for (int cc = lane; cc < BN; cc += 32)
        asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" :: "l"(dst + cc), "r"(tile[row * (BN + 1) + cc]) : "memory");
    }
  }
};

// Fused QKV: per column block (q|k|v) dequant F32(acc)*F32(s_in*s_w) + bias, quantize
// at the block's site (reference encoder.py:355-366).
struct EpiQKV {
  static constexpr bool kStagedBias = !SAMP_BIAS_GLOBAL;   // tile bias copied to smem per tile
  struct Params {
    int8_t* out;          // [M][ldo]
    int ldo;
    const float* bias;    // [3H]
    int block_cols;       // H
    float mult0, mult1, mult2;     // F32(double(s_in) * double(s_w{q,k,v}))
    float sout0, sout1, sout2;     // F32(scale(L.attn.{q,k,v}))
  };
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return BN * 4; }
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  template <int BN>
  __device__ static void prefetch(const Params& p, uint8_t* smem, int, int n0, int, int tid, int nt) {
    stage_floats(reinterpret_cast<float*>(smem), p.bias + n0, BN, tid, nt);
  }
  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t* smem) {
    const float* sbias = reinterpret_cast<const float*>(smem);
    // a tile never straddles q|k|v blocks (block_cols % BN == 0)
    const int blk = c.n0 / p.block_cols;
    const float mult = blk == 0 ? p.mult0 : blk == 1 ? p.mult1 : p.mult2;
    const Recip rq = make_recip(blk == 0 ? p.sout0 : blk == 1 ? p.sout1 : p.sout2);
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += 32) {
      const int gcol = c.n0 + c.c0 + col;
      uint32_t r[32];
      tmem_ld32(c.taddr + col, r);
      float b[32];
      if constexpr (SAMP_BIAS_GLOBAL) load_bias32(p.bias + gcol, b);
      else load_smem32(sbias + c.c0 + col, b);
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        v[j] = quant_pre_bounded(__fadd_rn(__fmul_rn(__int2float_rn(int(r[j])), mult), b[j]), rq);
      if (c.row < c.M) store32_pre(p.out + size_t(c.row) * p.ldo + gcol, v);
    }
  }
};

// FFN1: F32(acc)*mult + b1 -> GELU (numpy/SVML-exact) -> quantize(ffn.mid)
// (reference encoder.py:406-410).  MODE 0: general gelu8 (inf/nan-capable); MODE 1
// (GELU_FINITE): the host proved the GELU argument finite for this launch (gelu8_finite);
// MODE 2 (GELU_FAST): additionally the scale passed the exhaustive fast-path check, so
// codes come from gelu_q_fast2 and only flagged elements take the exact path.
enum { GELU_GENERAL = 0, GELU_FINITE = 1, GELU_FAST = 2 };
struct GeluQuantParams {
  int8_t* out;
  int ldo;
  const float* bias;
  float mult;
  float s_out;
  float inv_s = 0.0f;   // ~1/s_out (GELU_FAST)
  X2 k = x2_consts();   // opaque FFMA2 constants (packed path)
  unsigned long long* flag_count = nullptr;   // measurement: flagged 8-groups (SAMP_GELU_FLAGS)
  int fixup_all = 0;    // test switch (SAMP_GELU_FIXUP_ALL): every 8-group through gelu_fixup
};
template <int MODE>
struct EpiGeluQuantT {
  static constexpr bool kStagedBias = !SAMP_BIAS_GLOBAL;
  using Params = GeluQuantParams;
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return sizeof(TanhTable) + BN * 4; }
  static constexpr int kTableBytes = sizeof(TanhTable);   // read-only: shared by persistent buffers
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  template <int BN>
  __device__ static void prefetch(const Params& p, uint8_t* smem, int, int n0, int, int tid, int nt) {
    load_tanh_table(reinterpret_cast<TanhTable*>(smem), tid, nt);
    stage_floats(reinterpret_cast<float*>(smem + sizeof(TanhTable)), p.bias + n0, BN, tid, nt);
  }
  // exact codes of 8 finite GELU arguments (packed FFMA2 arithmetic, see numerics.cuh)
  __device__ static void exact8(const float (&x)[8], const TanhTable* tt, const Recip& rq, const X2& k,
                                uint32_t& w0, uint32_t& w1) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = x[u];
    gelu8_finite_x2(v, tt, k);
    float2 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = quant_pre2(f2(v[2 * u], v[2 * u + 1]), rq, k);
    w0 = trunc_pack4_s8(q[0].x, q[0].y, q[1].x, q[1].y);
    w1 = trunc_pack4_s8(q[2].x, q[2].y, q[3].x, q[3].y);
  }
  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t* smem) {
    const TanhTable* tt = reinterpret_cast<const TanhTable*>(c.table ? c.table : smem);
    const float* sbias = reinterpret_cast<const float*>(c.table ? smem : smem + sizeof(TanhTable));
    const Recip rq = make_recip(p.s_out);
    // CH columns per TMEM load: 16 keeps the one-tile kernel under its 96-register cap
#ifndef SAMP_GELU_CHUNK
#define SAMP_GELU_CHUNK 16
#endif
    constexpr int COLS = BN / (NE / 4);
    constexpr int CH = COLS % SAMP_GELU_CHUNK == 0 ? SAMP_GELU_CHUNK : COLS % 16 == 0 ? 16 : 8;
    uint32_t fmask = 0;   // GELU_FAST: bit col/8 = that 8-group was flagged (exact codes after the loop)
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += CH) {
      const int gcol = c.n0 + c.c0 + col;
      uint32_t r[CH];
      if constexpr (CH == 32) tmem_ld32(c.taddr + col, r);
      else if constexpr (CH == 16) tmem_ld16(c.taddr + col, r);
      else tmem_ld8(c.taddr + col, r);
      float b[CH];
#pragma unroll
      for (int j = 0; j < CH / 4; ++j) {
        const float4 v = SAMP_BIAS_GLOBAL ? __ldg(reinterpret_cast<const float4*>(p.bias + gcol) + j)
                                          : reinterpret_cast<const float4*>(sbias + c.c0 + col)[j];
        b[4 * j] = v.x; b[4 * j + 1] = v.y; b[4 * j + 2] = v.z; b[4 * j + 3] = v.w;
      }
      tmem_wait_ld();
      uint32_t w[CH / 4];
#pragma unroll
      for (int g = 0; g < CH; g += 8) {
        float v[8];
        if constexpr (MODE != GELU_GENERAL) {   // packed (FFMA2) arithmetic, see numerics.cuh
          const X2 k = p.k;
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            const float2 d = add2(mul2(f2(__int2float_rn(int(r[g + u])), __int2float_rn(int(r[g + u + 1]))),
                                       f2(p.mult, p.mult), k),
                                  f2(b[g + u], b[g + u + 1]), k);
            v[u] = d.x;
            v[u + 1] = d.y;
          }
          if constexpr (MODE == GELU_FAST) {
            bool near = false;
            float2 t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = gelu_q_fast2(f2(v[2 * u], v[2 * u + 1]), p.inv_s, k, near);
#ifdef SAMP_GELU_FLAG_COUNT   // measurement build only (costs ~1 us per FFN1 launch)
            if (near && p.flag_count) atomicAdd(p.flag_count, 1ull);
#endif
#ifdef SAMP_GELU_INLINE_FALLBACK   // measurement: the exact path inside the loop (round-2 form)
            if (near) {
              exact8(v, tt, rq, k, w[g / 4], w[g / 4 + 1]);
            } else {
              w[g / 4] = trunc_pack4_s8(t[0].x, t[0].y, t[1].x, t[1].y);
              w[g / 4 + 1] = trunc_pack4_s8(t[2].x, t[2].y, t[3].x, t[3].y);
            }
#else
            // flagged groups get their exact codes after the loop (gelu_fixup), so the exact
            // path's code and registers stay out of the hot loop
            if (near || p.fixup_all) fmask |= 1u << ((col + g) >> 3);
            w[g / 4] = trunc_pack4_s8(t[0].x, t[0].y, t[1].x, t[1].y);
            w[g / 4 + 1] = trunc_pack4_s8(t[2].x, t[2].y, t[3].x, t[3].y);
#endif
          } else {
            exact8(v, tt, rq, k, w[g / 4], w[g / 4 + 1]);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __fadd_rn(__fmul_rn(__int2float_rn(int(r[g + u])), p.mult), b[g + u]);
          gelu8(v, tt);
          w[g / 4] = trunc_pack4_s8(quant_pre_bounded(v[0], rq), quant_pre_bounded(v[1], rq),
                                    quant_pre_bounded(v[2], rq), quant_pre_bounded(v[3], rq));
          w[g / 4 + 1] = trunc_pack4_s8(quant_pre_bounded(v[4], rq), quant_pre_bounded(v[5], rq),
                                        quant_pre_bounded(v[6], rq), quant_pre_bounded(v[7], rq));
        }
      }
#ifdef SAMP_EXP_GELU_NOSTORE   // measurement variant only: results garbage
      if (c.row < c.M && (w[0] ^ w[1]) == 0x12345678u) {
#else
      if (c.row < c.M) {
#endif
        if constexpr (CH == 8) {
          *reinterpret_cast<uint2*>(p.out + size_t(c.row) * p.ldo + gcol) = make_uint2(w[0], w[1]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(p.out + size_t(c.row) * p.ldo + gcol);
#pragma unroll
          for (int q = 0; q < CH / 16; ++q) dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      }
    }
    if constexpr (MODE == GELU_FAST) {
      const uint32_t any = __reduce_or_sync(0xffffffffu, fmask);   // warp-uniform: tcgen05.ld is .sync.aligned
      if (any)
        gelu_fixup(p.out + size_t(c.row) * p.ldo + c.n0 + c.c0, c.row < c.M,
                   SAMP_BIAS_GLOBAL ? p.bias + c.n0 + c.c0 : sbias + c.c0, p.mult, p.k, c.taddr, tt, rq, fmask, any);
    }
  }
  // Exact codes of the flagged 8-groups (~5e-4 of the groups on the bench batch): the warp
  // walks the union of its threads' flagged groups, re-reads those 8 accumulator columns
  // (still in TMEM: the buffer is released after run()), and each flagging thread recomputes
  // its group on the bit-exact numpy/SVML path and overwrites the 8 fast codes it stored.
  // (scalars only: a by-reference Params/EpiCtx would be copied to local memory per tile)
  __device__ static __noinline__ void gelu_fixup(int8_t* out, bool live, const float* bias, float mult, const X2 k,
                                                 uint32_t taddr, const TanhTable* tt, const Recip rq, uint32_t mine,
                                                 uint32_t any) {
    while (any) {
      const int gi = __ffs(int(any)) - 1;
      any &= any - 1;
      const int col = gi * 8;
      uint32_t r[8];
      tmem_ld8(taddr + col, r);
      tmem_wait_ld();
      if ((mine >> gi) & 1u) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const float2 d = add2(mul2(f2(__int2float_rn(int(r[u])), __int2float_rn(int(r[u + 1]))), f2(mult, mult), k),
                                f2(bias[col + u], bias[col + u + 1]), k);
          v[u] = d.x;
          v[u + 1] = d.y;
        }
        uint32_t w0, w1;
        exact8(v, tt, rq, k, w0, w1);
        if (live) *reinterpret_cast<uint2*>(out + col) = make_uint2(w0, w1);
      }
    }
  }
};

using EpiGeluQuant = EpiGeluQuantT<GELU_GENERAL>;
using EpiGeluQuantFinite = EpiGeluQuantT<GELU_FINITE>;
using EpiGeluQuantFast = EpiGeluQuantT<GELU_FAST>;

// FP16-path bias (+ optional GELU) epilogue: acc(F32) + bias [-> gelu] -> f16 storage.
// (reference mha_fp encoder.py:291-292 qkv = gemm + qkv_b; ffn_fp :325-326 gelu(mid))
struct EpiF16Out {
  static constexpr bool kStagedBias = true;
  struct Params {
    __half* out;
    int ldo;
    const float* bias;
    int gelu;
    float* amax;          // calibration: site amax array (null = off)
    int site0;            // site of column block 0
    int block_cols;       // columns per site (QKV: H -> q|k|v sites); 0 = one site
  };
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return sizeof(TanhTable) + BN * 4; }
  static constexpr int kTableBytes = sizeof(TanhTable);   // read-only: shared by persistent buffers
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  template <int BN>
  __device__ static void prefetch(const Params& p, uint8_t* smem, int, int n0, int, int tid, int nt) {
    load_tanh_table(reinterpret_cast<TanhTable*>(smem), tid, nt);
    stage_floats(reinterpret_cast<float*>(smem + sizeof(TanhTable)), p.bias + n0, BN, tid, nt);
  }
  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t* smem) {
    const TanhTable* tt = reinterpret_cast<const TanhTable*>(c.table ? c.table : smem);
    const float* sbias = reinterpret_cast<const float*>(c.table ? smem : smem + sizeof(TanhTable));
    float amx = 0.0f;
    // GELU and the calibration amax are per-launch switches: compiled into separate loop
    // bodies (a runtime test inside the loop would only be predicated)
    auto body = [&](auto gelu_tag, auto amax_tag) {
      constexpr bool GELU = decltype(gelu_tag)::value, AMAX = decltype(amax_tag)::value;
#pragma unroll 1
      for (int col = 0; col < c.ncols; col += 32) {
        const int gcol = c.n0 + c.c0 + col;
        uint32_t r[32];
        tmem_ld32(c.taddr + col, r);
        float b[32];
        load_smem32(sbias + c.c0 + col, b);
        tmem_wait_ld();
        uint32_t packed[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          float x0 = __fadd_rn(__uint_as_float(r[j]), b[j]);
          float x1 = __fadd_rn(__uint_as_float(r[j + 1]), b[j + 1]);
          if constexpr (GELU) {
            x0 = gelu_ref(x0, tt);
            x1 = gelu_ref(x1, tt);
          }
          if constexpr (AMAX)
            if (c.row < c.M) amx = fmaxf(amx, fmaxf(fabsf(x0), fabsf(x1)));
          __half2 h = __floats2half2_rn(x0, x1);
          packed[j / 2] = *reinterpret_cast<uint32_t*>(&h);
        }
        if (c.row < c.M) {
          uint4* dst = reinterpret_cast<uint4*>(p.out + size_t(c.row) * p.ldo + gcol);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
        }
      }
    };
    if (p.gelu) {
      if (p.amax) body(std::true_type{}, std::true_type{});
      else body(std::true_type{}, std::false_type{});
    } else {
      if (p.amax) body(std::false_type{}, std::true_type{});
      else body(std::false_type{}, std::false_type{});
    }
    if (p.amax) amax_commit(p.amax + p.site0 + (p.block_cols ? c.n0 / p.block_cols : 0), amx);
  }
};

// Row-complete residual + LayerNorm epilogue (the paper's "big kernel"):
//   x   = (F32(acc)*mult + bias) + residual      residual = F32(code)*s_in  or  f32
//   out = ((x - mean) * inv) * gamma + beta      mean/var: numpy pairwise over H
// then any of: int8 quantize(s_out), f32 store, f16 store.
// (reference encoder.py:381-385 out-proj, :412-418 FFN2; kernels.layernorm :138-154)
// Sum order: each thread reduces its (half) row = one numpy subtree; the two halves are
// added (NE == 8), then the CLUSTER CTAs' partials in tree order through DSMEM.
struct ResLNParams {
  const float* bias;
  const int8_t* res_i8;   // residual codes [M][H] (or null)
  const float* res_f32;   // residual values [M][H] (or null)
  float res_scale;
  const float* gamma;
  const float* beta;
  float mult;             // int32 accumulator dequant multiplier
  int acc_is_f32;         // kind::f16 GEMM: accumulator is already F32, no dequant
  float eps;
  int hidden;
  int8_t* out_i8;  float s_out;   // optional
  int deq_outputs;                // f32/f16 outputs carry F32(q)*s_out (MHA-only layers)
  int f16_round;                  // reference fp16 storage: round the f32 output through f16
  float* out_f32;                 // optional
  __half* out_f16;                // optional
  float* amax;                    // calibration: amax array (null = off)
  int site, site2;                // sites tapped with the emitted values (site2 < 0: none)
  float* tap_f32 = nullptr;       // capture_taps: [M][H] LayerNorm output before quantize
  X2 k = x2_consts();             // opaque FFMA2 constants (paired INT8 path, numerics.cuh)
  int tma_store = 0;              // I8_ONLY register path: the code tile leaves by one TMA store
  int noclamp = 0;                // host proved |LN output| < 1e18 (2 sqrt(H) max|g| + max|b|, eps > 0):
                                  // the +-2^64 clamp before the fast quotient is a no-op
  CUtensorMap out_map;            // ... over out_i8 [rows][hidden], box BN x 128, no swizzle
  // small-batch f32/f16 outputs (FP layers) by TMA: bit 0 out_f32 through map_f32 (box 32 x 128
  // f32, 128B swizzle), bit 1 out_f16 through map_f16 (box 32 x 128 f16, 64B swizzle)
  int tma_f = 0;
  CUtensorMap map_f32, map_f16;
  // small-batch f32 residual by TMA: boxes of 32 x 128 f32 (128B swizzle) loaded by the
  // producer into the first drained ring slots after the main loop (res_f32 rows)
  int tma_res = 0;
  CUtensorMap map_res;
  // row-tile flags (sm100.cuh): with dep_cnt set, the A rows of row tile m are read once
  // dep_cnt[t] >= dep_target for the producer tiles t in [dep_rt[2m], dep_rt[2m+1]], and the
  // kernel does not wait for its predecessor grid (it only reads the predecessor's A rows;
  // its other inputs are older, its outputs not read by a grid still running)
  const int* dep_cnt = nullptr;
  const int* dep_rt = nullptr;
  int dep_target = 0;
};
// I8_ONLY: the hot INT8 chain (int8 residual, int32 accumulator, only int8 codes out):
// the general variant's optional outputs are compiled out, shrinking the epilogue code
// ~3x (ncu showed 20% "no_instruction" stalls on the 80 KB general kernel).
template <bool I8_ONLY, bool REGS96 = false>
struct EpiResLNT {
  using Params = ResLNParams;

  // smem: [0,512) floats reduction scratch (per-half partials, 2 x CTA partials), then
  // bias / gamma / beta slices (BN floats each), then the int8 residual tile
  // [128][BN + 16] (16-byte row pad: conflict-free 16 B reads by consecutive rows)
  static constexpr int RED_FLOATS = 8 * 128;   // two reductions x up to 4 partials per row
  template <int BN> __host__ __device__ static constexpr int res_ld() { return BN + 16; }
  // cluster exchange (CLUSTER > 1): xpart [2 reductions][4][128] floats + xbar[2] mbarriers
  template <int BN> __host__ __device__ static constexpr int xp_off() { return (RED_FLOATS + 3 * BN) * 4 + 128 * res_ld<BN>(); }
  static constexpr int XP_MAX = 8;   // cluster ranks the exchange buffer holds
  template <int BN> __host__ __device__ static constexpr int smem_bytes() { return xp_off<BN>() + 2 * XP_MAX * 128 * 4 + 24; }
  static constexpr bool kResTma = true;
  // mbarrier of the TMA-loaded residual tile (after the two exchange barriers)
  template <int BN>
  __device__ static uint64_t* res_bar(uint8_t* smem) {
    return reinterpret_cast<uint64_t*>(smem + xp_off<BN>() + 2 * XP_MAX * 128 * 4) + 2;
  }
  template <int CLUSTER> __device__ static constexpr int cluster_barriers() { return 0; }
  // before the kernel's cluster-wide start barrier: the exchange barriers exist before any
  // peer's st.async can complete on them
  template <int BN>
  __device__ static void cluster_init(uint8_t* smem) {
    uint64_t* xb = reinterpret_cast<uint64_t*>(smem + xp_off<BN>() + 2 * XP_MAX * 128 * 4);
    mbar_init(&xb[0], 1);
    mbar_init(&xb[1], 1);
    mbar_init(&xb[2], 1);
  }
  template <int BN>
  __device__ static void prefetch(const Params& p, uint8_t* smem, int m0, int n0, int M, int tid, int nt) {
    float* f = reinterpret_cast<float*>(smem) + RED_FLOATS;
    stage_floats_async(f, p.bias + n0, BN, tid, nt);
    stage_floats_async(f + BN, p.gamma + n0, BN, tid, nt);
    stage_floats_async(f + 2 * BN, p.beta + n0, BN, tid, nt);
    if (p.res_i8) {   // the int8 residual tile, all 16-byte pieces in flight at once
      uint8_t* rt = smem + (RED_FLOATS + 3 * BN) * 4;
      constexpr int V = BN / 16;  // uint4 per row
      for (int i = tid; i < 128 * V; i += nt) {
        const int row = i / V, v = i % V;
        uint8_t* dst = rt + row * res_ld<BN>() + v * 16;
        if (m0 + row < M) cp_async16(dst, p.res_i8 + size_t(m0 + row) * p.hidden + n0 + 16 * v);
        else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
  }

  // Row total of reduction `red` (0: sum, 1: sum of squares): the two column halves inside
  // the CTA (NE == 8), then the CLUSTER CTAs' partials in rank order ((p0+p1)+(p2+p3)).
  // The cluster exchange is push-based: every CTA st.async's its 128 row partials into each
  // peer's xpart[red][rank][row], completing on the peer's xbar[red] (expect_tx of all
  // CLUSTER*128 floats); nobody reads remote smem, so no cluster barrier is needed after
  // the kernel's start (a CTA only exits after its own exchanges landed).
  template <int BN, int CLUSTER, int NE>
  __device__ static float reduce_row(float mine, const EpiCtx& c, float* halves, uint8_t* smem, int red) {
    float s = mine;
    if constexpr (NE == 8) {
      float* hv = halves + red * 256;   // one buffer per reduction: no reuse barrier
      hv[c.half * 128 + c.tile_row] = mine;
      epi_bar_sync(c.ne_threads);
      s = __fadd_rn(hv[c.tile_row], hv[128 + c.tile_row]);
    } else if constexpr (NE == 16) {    // two leaves x two accumulator halves (run_strided)
      float* hv = halves + red * 512;
      hv[c.half * 128 + c.tile_row] = mine;
      epi_bar_sync(c.ne_threads);
      s = __fadd_rn(__fadd_rn(hv[c.tile_row], hv[128 + c.tile_row]),
                    __fadd_rn(hv[256 + c.tile_row], hv[384 + c.tile_row]));
    }
    if constexpr (CLUSTER > 1) {
      float* xp = reinterpret_cast<float*>(smem + xp_off<BN>()) + red * XP_MAX * 128;
      uint64_t* xb = reinterpret_cast<uint64_t*>(smem + xp_off<BN>() + 2 * XP_MAX * 128 * 4) + red;
      if (c.ep_tid == 0) mbar_expect_tx(xb, CLUSTER * 128 * 4);
      if (c.half == 0) {
        const uint32_t me = cluster_rank();
#pragma unroll
        for (int rr = 0; rr < CLUSTER; ++rr)
          st_async_f32(mapa_rank(xp + me * 128 + c.tile_row, rr), s, mapa_rank(xb, rr));
      }
      mbar_wait(xb, 0);
      float p[CLUSTER];
#pragma unroll
      for (int r = 0; r < CLUSTER; ++r) p[r] = xp[r * 128 + c.tile_row];
      // numpy's tree above equal per-rank subtrees: pairs, then pairs of pairs, ...
      if constexpr (CLUSTER == 2) s = __fadd_rn(p[0], p[1]);
      else if constexpr (CLUSTER == 4) s = __fadd_rn(__fadd_rn(p[0], p[1]), __fadd_rn(p[2], p[3]));
      else s = __fadd_rn(__fadd_rn(__fadd_rn(p[0], p[1]), __fadd_rn(p[2], p[3])),
                         __fadd_rn(__fadd_rn(p[4], p[5]), __fadd_rn(p[6], p[7])));
    }
    return s;
  }

  // residual of 32 columns starting at tile column `col` (int8 tile in smem, or f32 global)
  template <int BN>
  __device__ static void residual32(const Params& p, const EpiCtx& c, const uint8_t* rtile, size_t rbase,
                                    int col, float (&res)[32]) {
    if (p.res_i8) {
      const uint4* src = reinterpret_cast<const uint4*>(rtile + col);
      const uint4 u0 = src[0], u1 = src[1];
      const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
      for (int j = 0; j < 32; ++j) res[j] = deq(int(int8_t((w[j / 4] >> (8 * (j % 4))) & 0xff)), p.res_scale);
    } else {
      const float4* src = reinterpret_cast<const float4*>(p.res_f32 + rbase + c.n0 + col);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = src[j];
        res[4 * j] = v.x; res[4 * j + 1] = v.y; res[4 * j + 2] = v.z; res[4 * j + 3] = v.w;
      }
    }
  }

  // emit 32 normalised values (quantize / deq / f16 round / amax / stores)
  __device__ static void emit32(const Params& p, size_t rbase, int gcol, const Recip& rq, float (&y)[32], float& amx) {
    // reference order: storage rounding (fp16 mode) happens before any quantize
    if (p.f16_round) {
#pragma unroll
      for (int j = 0; j < 32; ++j) y[j] = __half2float(__float2half_rn(y[j]));
    }
    if (p.tap_f32) {
      float4* dst = reinterpret_cast<float4*>(p.tap_f32 + rbase + gcol);
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
    }
    if (p.deq_outputs) {
      int q[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) q[j] = quant_fast(y[j], rq);
      if (p.out_i8) store32_i8(p.out_i8 + rbase + gcol, q);
#pragma unroll
      for (int j = 0; j < 32; ++j) y[j] = deq(q[j], p.s_out);
    } else if (p.out_i8) {
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = quant_pre_fast(y[j], rq);
      store32_pre(p.out_i8 + rbase + gcol, v);
    }
    if (p.amax) {
#pragma unroll
      for (int j = 0; j < 32; ++j) amx = fmaxf(amx, fabsf(y[j]));
    }
    if (p.out_f32) {
      float4* dst = reinterpret_cast<float4*>(p.out_f32 + rbase + gcol);
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
    }
    if (p.out_f16) {
      uint4* dst = reinterpret_cast<uint4*>(p.out_f16 + rbase + gcol);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __half2 h0 = __floats2half2_rn(y[8 * j], y[8 * j + 1]), h1 = __floats2half2_rn(y[8 * j + 2], y[8 * j + 3]);
        __half2 h2 = __floats2half2_rn(y[8 * j + 4], y[8 * j + 5]), h3 = __floats2half2_rn(y[8 * j + 6], y[8 * j + 7]);
        dst[j] = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                            *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
      }
    }
  }

  // Register-resident variant (1 CTA/SM tiles, NE == 8): the thread's whole (half) row is
  // pulled out of TMEM once; sums, normalisation and outputs all run from registers.
  template <int BN, int CLUSTER, int NE>
  __device__ static void run_regs(const Params& p, const EpiCtx& c, uint8_t* smem) {
    constexpr int NC = BN / (NE / 4);
    static_assert(NC % 32 == 0 && NC <= 128, "one numpy leaf per thread");
    float* halves = reinterpret_cast<float*>(smem);
    const float* sbias = halves + RED_FLOATS;
    const float* sgam = sbias + BN;
    const float* sbet = sgam + BN;
    const uint8_t* rtile = smem + (RED_FLOATS + 3 * BN) * 4 + c.tile_row * res_ld<BN>();
    const bool valid = c.row < c.M;
    const size_t rbase = size_t(valid ? c.row : 0) * p.hidden;
    float x[NC];
    {
      uint32_t r[NC];
#pragma unroll
      for (int k = 0; k < NC / 32; ++k)
        tmem_ld32(c.taddr + 32 * k, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * k));
      tmem_wait_ld();
      if (c.kpart) {   // KS2: add the other K half's accumulators (int32 exact; f32 for kind::f16)
        mbar_wait(c.kpart_bar, 0);
        const uint32_t* kp = c.kpart + c.tile_row * BN + c.c0;
#pragma unroll
        for (int j = 0; j < NC; ++j)
          r[j] = p.acc_is_f32 ? __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __uint_as_float(kp[j])))
                              : uint32_t(int(r[j]) + int(kp[j]));
      }
#pragma unroll
      for (int k = 0; k < NC / 32; ++k) {
        float res[32];
        if constexpr (I8_ONLY) {
          // x = (F32(acc)*mult + b) + F32(code)*s_in on FFMA2 pairs (same roundings as the
          // scalar form: mul2 = RN(a*b), add2 = RN(a+b), numerics.cuh), bias as float4
          const uint4* src = reinterpret_cast<const uint4*>(rtile + c.c0 + 32 * k);
          const uint4 u0 = src[0], u1 = src[1];
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
          const X2 kx = p.k;
          const float2 mm = f2(p.mult, p.mult), rs = f2(p.res_scale, p.res_scale);
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 b4 = *reinterpret_cast<const float4*>(sbias + c.c0 + 32 * k + 4 * g);
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = 4 * g + 2 * u;
              const float2 rv = mul2(f2(__int2float_rn(int(int8_t((w[g] >> (16 * u)) & 0xff))),
                                        __int2float_rn(int(int8_t((w[g] >> (16 * u + 8)) & 0xff)))), rs, kx);
              const float2 av = mul2(f2(__int2float_rn(int(r[32 * k + j])), __int2float_rn(int(r[32 * k + j + 1]))), mm,
                                     kx);
              const float2 xv = add2(add2(av, f2(bb[2 * u], bb[2 * u + 1]), kx), rv, kx);
              x[32 * k + j] = xv.x;
              x[32 * k + j + 1] = xv.y;
            }
          }
        } else {
          if (p.tma_res) {   // residual box k from its ring slot (128B swizzle: chunk ^ (row & 7))
            if (k == 0) {
              mbar_wait(res_bar<BN>(smem), 0);
            }
            int slot = c.res_slot0 + k;
            slot = slot >= c.stages ? slot - c.stages : slot;
            const uint8_t* rowp = c.ring + slot * (GEMM_BM * 128) + c.tile_row * 128;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 v = *reinterpret_cast<const float4*>(rowp + ((q ^ (c.tile_row & 7)) << 4));
              res[4 * q] = v.x; res[4 * q + 1] = v.y; res[4 * q + 2] = v.z; res[4 * q + 3] = v.w;
            }
          } else {
            residual32<BN>(p, c, rtile, rbase, c.c0 + 32 * k, res);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const uint32_t u = r[32 * k + j];
            const float acc = p.acc_is_f32 ? __uint_as_float(u) : __fmul_rn(__int2float_rn(int(u)), p.mult);
            x[32 * k + j] = __fadd_rn(__fadd_rn(acc, sbias[c.c0 + 32 * k + j]), res[j]);
          }
        }
      }
    }
    // one numpy leaf of NC elements: 8 strided accumulators, then ((0+1)+(2+3))+((4+5)+(6+7))
    auto leaf = [&](auto f) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = f(x[j]);
#pragma unroll
      for (int g = 1; g < NC / 8; ++g)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], f(x[8 * g + j]));
      return __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                       __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
    };
    // the same leaf with accumulator pairs (j, j+1) on FFMA2 lanes (per-lane order unchanged)
    auto leaf2 = [&](float msub, bool sq) {
      const X2 kx = p.k;
      const float2 nm = f2(-msub, -msub);
      auto term = [&](int i) {
        float2 v = f2(x[i], x[i + 1]);
        if (sq) {
          v = add2(v, nm, kx);
          v = mul2(v, v, kx);
        }
        return v;
      };
      float2 acc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = term(2 * j);
#pragma unroll
      for (int g = 1; g < NC / 8; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = add2(acc[j], term(8 * g + 2 * j), kx);
      return __fadd_rn(__fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)),
                       __fadd_rn(__fadd_rn(acc[2].x, acc[2].y), __fadd_rn(acc[3].x, acc[3].y)));
    };
    const float hf = float(p.hidden);
    if (c.sub) c.sub[0] = globaltimer();
    float lsum;
    if constexpr (I8_ONLY) lsum = leaf2(0.0f, false);
    else lsum = leaf([](float v) { return v; });
    if (c.sub) c.sub[1] = globaltimer();
    const float total = reduce_row<BN, CLUSTER, NE>(lsum, c, halves, smem, 0);
    const float mean = __fdiv_rn(__fadd_rn(0.0f, total), hf);
    if (c.sub) c.sub[2] = globaltimer();
    float lsum2;
    if constexpr (I8_ONLY) {
      lsum2 = leaf2(mean, true);
    } else {
      lsum2 = leaf([mean](float v) {
        const float d = __fsub_rn(v, mean);
        return __fmul_rn(d, d);
      });
    }
    if (c.sub) c.sub[3] = globaltimer();
    const float total2 = reduce_row<BN, CLUSTER, NE>(lsum2, c, halves, smem, 1);
    const float var = __fdiv_rn(__fadd_rn(0.0f, total2), hf);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
    const Recip rq = make_recip(p.out_i8 || p.deq_outputs ? p.s_out : 1.0f);
    if (c.sub) c.sub[4] = globaltimer();
    float amx = 0.0f;
    uint32_t tw[I8_ONLY ? NC / 4 : 1];   // TMA-store path: this thread's codes
    if (valid || (I8_ONLY && p.tma_store)) {
      // the +-2^64 clamp compiled out when the host proved it a no-op (p.noclamp): a runtime
      // test inside the loop was only predicated, not removed
      auto emit_rows = [&](auto clamp_tag) {
        constexpr bool CLAMP = decltype(clamp_tag)::value;
#pragma unroll
        for (int k = 0; k < NC / 32; ++k) {
          if constexpr (I8_ONLY) {
            // y = ((x - mean)*inv)*g + b and quantize on FFMA2 pairs, γ/β as float4
            const X2 kx = p.k;
            const float2 nm = f2(-mean, -mean), iv = f2(inv, inv);
            uint32_t w[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const int col = c.c0 + 32 * k + 4 * g;
              const float4 g4 = *reinterpret_cast<const float4*>(sgam + col);
              const float4 b4 = *reinterpret_cast<const float4*>(sbet + col);
              float2 q[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int j = 32 * k + 4 * g + 2 * u;
                float2 y = mul2(mul2(add2(f2(x[j], x[j + 1]), nm, kx), iv, kx),
                                u ? f2(g4.z, g4.w) : f2(g4.x, g4.y), kx);
                y = add2(y, u ? f2(b4.z, b4.w) : f2(b4.x, b4.y), kx);
                if constexpr (CLAMP)
                  y = f2(fminf(fmaxf(y.x, -1.8446744e19f), 1.8446744e19f), fminf(fmaxf(y.y, -1.8446744e19f), 1.8446744e19f));
                q[u] = quant_pre2(y, rq, kx);
              }
              w[g] = trunc_pack4_s8(q[0].x, q[0].y, q[1].x, q[1].y);
            }
            if (p.tma_store) {
#pragma unroll
              for (int u = 0; u < 8; ++u) tw[8 * k + u] = w[u];
              continue;
            }
            uint4* dst = reinterpret_cast<uint4*>(p.out_i8 + rbase + c.n0 + c.c0 + 32 * k);
#ifdef SAMP_EXP_LN_NOSTORE   // measurement variant only: results garbage
            if ((w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5] ^ w[6] ^ w[7]) == 0x12345678u)
#endif
            {
              dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
              dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
          } else {
            float y[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = c.c0 + 32 * k + j;
              y[j] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(x[32 * k + j], mean), inv), sgam[col]), sbet[col]);
            }
            if (p.tma_f) {
              // stage 32 columns: f32 box k (128 B rows, 128B swizzle: chunk ^ (row & 7)) and
              // f16 box k (64 B rows, 64B swizzle: chunk ^ ((row >> 1) & 3)); the XOR acts on
              // addresses, so the register indices stay compile-time
              if (p.f16_round) {
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = __half2float(__float2half_rn(y[j]));
              }
              if (p.tma_f & 1) {
                uint8_t* rowp = c.stage + k * (128 * 128) + c.tile_row * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  *reinterpret_cast<float4*>(rowp + ((q ^ (c.tile_row & 7)) << 4)) =
                      make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
              }
              if (p.tma_f & 2) {
                uint8_t* rowp = c.stage + 3 * (128 * 128) + k * (128 * 64) + c.tile_row * 64;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint32_t hw[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    __half2 h2 = __floats2half2_rn(y[8 * q + 2 * u], y[8 * q + 2 * u + 1]);
                    hw[u] = *reinterpret_cast<uint32_t*>(&h2);
                  }
                  *reinterpret_cast<uint4*>(rowp + ((q ^ ((c.tile_row >> 1) & 3)) << 4)) =
                      make_uint4(hw[0], hw[1], hw[2], hw[3]);
                }
              }
            } else {
              emit32(p, rbase, c.n0 + c.c0 + 32 * k, rq, y, amx);
            }
          }
        }
      };
#ifdef SAMP_LN_ALWAYS_CLAMP
      emit_rows(std::true_type{});
#else
      if (!I8_ONLY || !p.noclamp) emit_rows(std::true_type{});
      else emit_rows(std::false_type{});
#endif
    }
    if constexpr (!I8_ONLY) {
      if (p.tma_f) {   // three 32-column boxes of each staged output, one TMA store each
        fence_proxy_async_smem();
        epi_bar_sync(c.ne_threads);
        if (c.ep_tid == 0) {
          const int m0 = c.row - c.tile_row;
#pragma unroll
          for (int k = 0; k < NC / 32; ++k) {
            if (p.tma_f & 1) tma_store_2d(&p.map_f32, c.stage + k * (128 * 128), c.n0 + c.c0 + 32 * k, m0);
            if (p.tma_f & 2) tma_store_2d(&p.map_f16, c.stage + 3 * (128 * 128) + k * (128 * 64), c.n0 + c.c0 + 32 * k, m0);
          }
          bulk_commit();
          bulk_wait_read0();
        }
      }
    }
    if constexpr (I8_ONLY) {
      if (p.tma_store) {
        // stage the [128][BN] code tile row-major (the TMA box layout); the 16-byte chunks of a
        // row go out rotated by (row / 2) % NCH so a warp's 32 rows spread over the banks
        // (rows are BN bytes apart: without it 16 lanes hit the same bank group)
        constexpr int NCH = NC / 16;
        uint8_t* srow = c.stage + size_t(c.tile_row) * BN + c.c0;
        const int rot = (c.tile_row >> 1) % NCH;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          int ch = i + rot;
          ch = ch >= NCH ? ch - NCH : ch;
          uint4 v = make_uint4(tw[0], tw[1], tw[2], tw[3]);
#pragma unroll
          for (int q = 1; q < NCH; ++q)
            if (ch == q) v = make_uint4(tw[4 * q], tw[4 * q + 1], tw[4 * q + 2], tw[4 * q + 3]);
          *reinterpret_cast<uint4*>(srow + 16 * ch) = v;
        }
        fence_proxy_async_smem();
        epi_bar_sync(c.ne_threads);
        if (c.ep_tid == 0) {
          tma_store_2d(&p.out_map, c.stage, c.n0, c.row - c.tile_row);
          bulk_commit();
          bulk_wait_read0();
        }
      }
    }
    if (c.sub) c.sub[5] = globaltimer();
    if (!I8_ONLY && p.amax) {
      amax_commit(p.amax + p.site, amx);
      if (p.site2 >= 0) amax_commit(p.amax + p.site2, amx);
    }
  }

  // Two threads per row over one 96-column numpy leaf (BN = 96, NE = 8): numpy's 8 strided
  // accumulators split by index — half h owns r[4h .. 4h+3], i.e. columns 8g + 4h + u — so
  // half 0 forms (r0+r1)+(r2+r3), half 1 (r4+r5)+(r6+r7), and reduce_row's half combine is
  // numpy's final add.  Each thread reads the whole row from TMEM once and keeps its 48
  // values in registers; normalisation and outputs run on 4-column groups.
  template <int BN, int CLUSTER, int NE>
  __device__ static void run_strided(const Params& p, const EpiCtx& c, uint8_t* smem) {
    // NE = 16, BN = 192 (small hidden, 4-CTA clusters): two 96-column leaves per CTA, each
    // split the same way over two of the row's four threads (quarter q: leaf q >> 1, half q & 1)
    static_assert((BN == 96 && NE == 8) || (BN == 192 && NE == 16), "96-column leaves, two threads each");
    constexpr int LEAF = 96;
    float* halves = reinterpret_cast<float*>(smem);
    const float* sbias = halves + RED_FLOATS;
    const float* sgam = sbias + BN;
    const float* sbet = sgam + BN;
    const uint8_t* rtile = smem + (RED_FLOATS + 3 * BN) * 4 + c.tile_row * res_ld<BN>();
    const bool valid = c.row < c.M;
    const size_t rbase = size_t(valid ? c.row : 0) * p.hidden;
    const int hh = c.half & 1;                 // accumulator half within the leaf
    const int lbase = LEAF * (c.half >> 1);    // the leaf's first tile column
    const int jo = 4 * hh;
    const uint32_t tbase = c.taddr - uint32_t(c.c0) + uint32_t(lbase);
    float x[48];
    if (c.kpart) mbar_wait(c.kpart_bar, 0);    // KS2: the other K half's accumulators landed
    // the register index must be compile-time: one body per half; 32 TMEM columns at a time
    auto fill = [&](auto jo_c) {
      constexpr int JO = decltype(jo_c)::value;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
      uint32_t r[32];
      tmem_ld32(tbase + 32 * k, r);
      tmem_wait_ld();
      if (c.kpart) {   // KS2: add the other K half's accumulators (int32 exact; f32 for kind::f16)
        const uint32_t* kp = c.kpart + c.tile_row * BN + lbase + 32 * k;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 8 * gg + JO + u;
            r[j] = p.acc_is_f32 ? __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __uint_as_float(kp[j])))
                                : uint32_t(int(r[j]) + int(kp[j]));
          }
      }
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const int g = 4 * k + gg;
        const int col = lbase + 8 * g + JO;
        float res[4];
        if (p.res_i8) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(rtile + col);
#pragma unroll
          for (int u = 0; u < 4; ++u) res[u] = deq(int(int8_t((w >> (8 * u)) & 0xff)), p.res_scale);
        } else if (p.tma_res) {   // box col/32 in its ring slot, 16-byte chunk (col%32)/4 ^ (row & 7)
          int slot = c.res_slot0 + col / 32;
          slot = slot >= c.stages ? slot - c.stages : slot;
          const float4 v = *reinterpret_cast<const float4*>(c.ring + slot * (GEMM_BM * 128) + c.tile_row * 128 +
                                                            ((((col & 31) >> 2) ^ (c.tile_row & 7)) << 4));
          res[0] = v.x; res[1] = v.y; res[2] = v.z; res[3] = v.w;
        } else {
          const float4 v = *reinterpret_cast<const float4*>(p.res_f32 + rbase + c.n0 + col);
          res[0] = v.x; res[1] = v.y; res[2] = v.z; res[3] = v.w;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t a = r[8 * gg + JO + u];
          const float acc = p.acc_is_f32 ? __uint_as_float(a) : __fmul_rn(__int2float_rn(int(a)), p.mult);
          x[4 * g + u] = __fadd_rn(__fadd_rn(acc, sbias[col + u]), res[u]);
        }
      }
      }
    };
    if (p.tma_res) mbar_wait(res_bar<BN>(smem), 0);
    if (hh == 0) fill(std::integral_constant<int, 0>{});
    else fill(std::integral_constant<int, 4>{});
    auto half_leaf = [&](auto f) {
      float a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = f(x[u]);
#pragma unroll
      for (int g = 1; g < 12; ++g)
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = __fadd_rn(a[u], f(x[4 * g + u]));
      return __fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3]));
    };
    const float hf = float(p.hidden);
    if (c.sub) c.sub[0] = globaltimer();
    const float lsum = half_leaf([](float v) { return v; });
    if (c.sub) c.sub[1] = globaltimer();
    const float total = reduce_row<BN, CLUSTER, NE>(lsum, c, halves, smem, 0);
    const float mean = __fdiv_rn(__fadd_rn(0.0f, total), hf);
    if (c.sub) c.sub[2] = globaltimer();
    const float lsum2 = half_leaf([mean](float v) {
      const float d = __fsub_rn(v, mean);
      return __fmul_rn(d, d);
    });
    if (c.sub) c.sub[3] = globaltimer();
    const float total2 = reduce_row<BN, CLUSTER, NE>(lsum2, c, halves, smem, 1);
    const float var = __fdiv_rn(__fadd_rn(0.0f, total2), hf);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
    const Recip rq = make_recip(p.out_i8 || p.deq_outputs ? p.s_out : 1.0f);
    if (c.sub) c.sub[4] = globaltimer();
    float amx = 0.0f;
    if constexpr (I8_ONLY) {
      // int8-only chain: normalise + quantize on FFMA2 pairs, γ/β as float4 (same roundings)
      const X2 kx = p.k;
      const float2 nm = f2(-mean, -mean), iv = f2(inv, inv);
#pragma unroll
      for (int g = 0; g < 12; ++g) {
        const int col = lbase + 8 * g + jo;
        const float4 g4 = *reinterpret_cast<const float4*>(sgam + col);
        const float4 b4 = *reinterpret_cast<const float4*>(sbet + col);
        float2 q[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          float2 y = mul2(mul2(add2(f2(x[4 * g + 2 * u], x[4 * g + 2 * u + 1]), nm, kx), iv, kx),
                          u ? f2(g4.z, g4.w) : f2(g4.x, g4.y), kx);
          y = add2(y, u ? f2(b4.z, b4.w) : f2(b4.x, b4.y), kx);
          y = f2(fminf(fmaxf(y.x, -1.8446744e19f), 1.8446744e19f), fminf(fmaxf(y.y, -1.8446744e19f), 1.8446744e19f));
          q[u] = quant_pre2(y, rq, kx);
        }
        const uint32_t codes = trunc_pack4_s8(q[0].x, q[0].y, q[1].x, q[1].y);
        if (p.tma_store) *reinterpret_cast<uint32_t*>(c.stage + size_t(c.tile_row) * BN + col) = codes;
        else if (valid) *reinterpret_cast<uint32_t*>(p.out_i8 + rbase + c.n0 + col) = codes;
      }
    } else if (valid) {
#pragma unroll
      for (int g = 0; g < 12; ++g) {
        const int col = lbase + 8 * g + jo;
        const size_t o = rbase + c.n0 + col;
        float y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          y[u] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(x[4 * g + u], mean), inv), sgam[col + u]), sbet[col + u]);
        if (p.f16_round) {   // storage rounding precedes any quantize (reference order)
#pragma unroll
          for (int u = 0; u < 4; ++u) y[u] = __half2float(__float2half_rn(y[u]));
        }
        if (p.tap_f32) *reinterpret_cast<float4*>(p.tap_f32 + o) = make_float4(y[0], y[1], y[2], y[3]);
        if (p.deq_outputs) {
          int q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = quant_fast(y[u], rq);
          if (p.out_i8) *reinterpret_cast<uint32_t*>(p.out_i8 + o) = pack4_i8(q[0], q[1], q[2], q[3]);
#pragma unroll
          for (int u = 0; u < 4; ++u) y[u] = deq(q[u], p.s_out);
        } else if (p.out_i8) {
          const uint32_t codes = trunc_pack4_s8(quant_pre_fast(y[0], rq), quant_pre_fast(y[1], rq),
                                                quant_pre_fast(y[2], rq), quant_pre_fast(y[3], rq));
          if (p.tma_store) *reinterpret_cast<uint32_t*>(c.stage + size_t(c.tile_row) * BN + col) = codes;
          else *reinterpret_cast<uint32_t*>(p.out_i8 + o) = codes;
        }
        if (p.amax) {
#pragma unroll
          for (int u = 0; u < 4; ++u) amx = fmaxf(amx, fabsf(y[u]));
        }
        if (p.tma_f) {   // swizzled 32-column boxes (see run_regs): f32 16-byte, f16 8-byte pieces
          if (p.tma_f & 1)
            *reinterpret_cast<float4*>(c.stage + (col >> 5) * (128 * 128) + c.tile_row * 128 +
                                       ((((col & 31) >> 2) ^ (c.tile_row & 7)) << 4)) = make_float4(y[0], y[1], y[2], y[3]);
          if (p.tma_f & 2) {
            __half2 h0 = __floats2half2_rn(y[0], y[1]), h1 = __floats2half2_rn(y[2], y[3]);
            *reinterpret_cast<uint2*>(c.stage + 3 * (128 * 128) + (col >> 5) * (128 * 64) + c.tile_row * 64 +
                                      ((((col & 31) >> 3) ^ ((c.tile_row >> 1) & 3)) << 4) + (col & 4) * 2) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          }
          continue;
        }
        if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + o) = make_float4(y[0], y[1], y[2], y[3]);
        if (p.out_f16) {
          __half2 h0 = __floats2half2_rn(y[0], y[1]), h1 = __floats2half2_rn(y[2], y[3]);
          *reinterpret_cast<uint2*>(p.out_f16 + o) =
              make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        }
      }
    }
    if (p.tma_f) {   // three 32-column boxes per staged output, one TMA store each
      fence_proxy_async_smem();
      epi_bar_sync(c.ne_threads);
      if (c.ep_tid == 0) {
        const int m0 = c.row - c.tile_row;
#pragma unroll
        for (int k = 0; k < BN / 32; ++k) {
          if (p.tma_f & 1) tma_store_2d(&p.map_f32, c.stage + k * (128 * 128), c.n0 + 32 * k, m0);
          if (p.tma_f & 2) tma_store_2d(&p.map_f16, c.stage + 3 * (128 * 128) + k * (128 * 64), c.n0 + 32 * k, m0);
        }
        bulk_commit();
        bulk_wait_read0();
      }
    }
    if (p.tma_store) {   // int8-only chain: the [128][96] code tile leaves by one TMA store
      fence_proxy_async_smem();
      epi_bar_sync(c.ne_threads);
      if (c.ep_tid == 0) {
        tma_store_2d(&p.out_map, c.stage, c.n0, c.row - c.tile_row);
        bulk_commit();
        bulk_wait_read0();
      }
    }
    if (c.sub) c.sub[5] = globaltimer();
    if (p.amax) {
      amax_commit(p.amax + p.site, amx);
      if (p.site2 >= 0) amax_commit(p.amax + p.site2, amx);
    }
  }

  template <int BN, int CLUSTER, int NE>
  __device__ static void run(const Params& p, const EpiCtx& c, uint8_t* smem) {
    if constexpr ((NE == 8 && BN == 96) || (NE == 16 && BN == 192)) {
      run_strided<BN, CLUSTER, NE>(p, c, smem);
      return;
    }
    // register-resident: NE == 8 half rows, or (REGS96) the small-batch 8-CTA clusters'
    // 96-column rows, one numpy leaf per thread (f32-residual LN: batch-1 FP16 p50 0.712 ->
    // 0.69 ms; the int8-residual one measured 0.475 -> 0.488 ms and keeps the TMEM variant)
    else if constexpr ((NE == 8 && (BN / 2) % 32 == 0 && BN / 2 <= 128) || (REGS96 && NE == 4 && BN == 96)) {
      run_regs<BN, CLUSTER, NE>(p, c, smem);
    } else {
      run_tmem<BN, CLUSTER, NE>(p, c, smem);
    }
  }

  // TMEM-resident variant (generic shapes)
  template <int BN, int CLUSTER, int NE>
  __device__ static void run_tmem(const Params& p, const EpiCtx& c, uint8_t* smem) {
    float* halves = reinterpret_cast<float*>(smem);
    const float* sbias = halves + RED_FLOATS;
    const float* sgam = sbias + BN;
    const float* sbet = sgam + BN;
    const uint8_t* rtile = smem + (RED_FLOATS + 3 * BN) * 4 + c.tile_row * res_ld<BN>();
    const bool valid = c.row < c.M;
    const size_t rbase = size_t(valid ? c.row : 0) * p.hidden;
    const int gbase = c.n0 + c.c0;
    // pass 1: x = (acc*mult + b) + residual, written back into TMEM as f32 bits
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += 32) {
      const int gcol = gbase + col;
      uint32_t r[32];
      tmem_ld32(c.taddr + col, r);
      float res[32], b[32];
      load_smem32(sbias + c.c0 + col, b);
      if (p.res_i8) {
        const uint4* src = reinterpret_cast<const uint4*>(rtile + c.c0 + col);
        const uint4 u0 = src[0], u1 = src[1];
        const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int j = 0; j < 32; ++j) res[j] = deq(int(int8_t((w[j / 4] >> (8 * (j % 4))) & 0xff)), p.res_scale);
      } else {
        const float4* src = reinterpret_cast<const float4*>(p.res_f32 + rbase + gcol);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = src[j];
          res[4 * j] = v.x; res[4 * j + 1] = v.y; res[4 * j + 2] = v.z; res[4 * j + 3] = v.w;
        }
      }
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float acc = p.acc_is_f32 ? __uint_as_float(r[j]) : __fmul_rn(__int2float_rn(int(r[j])), p.mult);
        r[j] = __float_as_uint(__fadd_rn(__fadd_rn(acc, b[j]), res[j]));
      }
      tmem_st32(c.taddr + col, r);
    }
    tmem_wait_st();

    // numpy pairwise sum of f(x) over this thread's columns.  A single 32-aligned leaf
    // (96 / 128 columns for H = 768 / 1024) streams TMEM 32 columns per load; anything
    // else walks the generic tree 8 columns at a time.
    auto row_sum = [&](auto f) -> float {
      if (c.ncols <= 128 && (c.ncols & 31) == 0) {
        float acc[8];
#pragma unroll 1
        for (int col = 0; col < c.ncols; col += 32) {
          uint32_t u[32];
          tmem_ld32(c.taddr + col, u);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float v = f(__uint_as_float(u[8 * g + j]));
              acc[j] = (col == 0 && g == 0) ? v : __fadd_rn(acc[j], v);
            }
          }
        }
        return __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                         __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
      }
      auto get8 = [&](int off, float (&v)[8]) {
        uint32_t u[8];
        tmem_ld8(c.taddr + off, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = f(__uint_as_float(u[j]));
      };
      return pairwise_sum(c.ncols, get8);
    };
    const float total = reduce_row<BN, CLUSTER, NE>(row_sum([](float x) { return x; }), c, halves, smem, 0);
    const float hf = float(p.hidden);
    const float mean = __fdiv_rn(__fadd_rn(0.0f, total), hf);
    const float total2 = reduce_row<BN, CLUSTER, NE>(row_sum([mean](float x) {
                                                   const float d = __fsub_rn(x, mean);
                                                   return __fmul_rn(d, d);
                                                 }),
                                                 c, halves, smem, 1);
    const float var = __fdiv_rn(__fadd_rn(0.0f, total2), hf);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
    const Recip rq = make_recip(p.out_i8 || p.deq_outputs ? p.s_out : 1.0f);
    float amx = 0.0f;

    // pass 3: normalise, affine, emit
#pragma unroll 1
    for (int col = 0; col < c.ncols; col += 32) {
      const int gcol = gbase + col;
      uint32_t r[32];
      tmem_ld32(c.taddr + col, r);
      float g[32], be[32];
      load_smem32(sgam + c.c0 + col, g);
      load_smem32(sbet + c.c0 + col, be);
      tmem_wait_ld();
      float y[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        y[j] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(__uint_as_float(r[j]), mean), inv), g[j]), be[j]);
      if (!valid) continue;
      emit32(p, rbase, gcol, rq, y, amx);
    }
    if (p.amax) {
      amax_commit(p.amax + p.site, amx);
      if (p.site2 >= 0) amax_commit(p.amax + p.site2, amx);
    }
  }
};
using EpiResLN = EpiResLNT<false>;
using EpiResLNI8 = EpiResLNT<true>;
using EpiResLNRegs96 = EpiResLNT<false, true>;

// ------------------------------------------------------------------ host launcher
template <int KIND, int BN, int STAGES, int CLUSTER, int NE, class Epi, bool MC = false, bool KS2 = false>
inline cudaError_t launch_gemm(const CUtensorMap& map_a, const CUtensorMap& map_b, int M, int N, int k_bytes,
                               const typename Epi::Params& p, cudaStream_t stream, int ksplit = 1) {
  constexpr int EPI_BYTES = (Epi::template smem_bytes<BN>() + 127) / 128 * 128;
  using Lay = GemmLayout<BN, STAGES, EPI_BYTES + ks2_bytes<BN, KS2>()>;
  auto kern = gemm_kernel<KIND, BN, STAGES, CLUSTER, NE, Epi, MC, KS2>;
  static thread_local int configured_device = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_device != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL);
    if (e != cudaSuccess) return e;
    if (KS2 && 2 * CLUSTER > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    configured_device = dev;
  }
  unsigned long long* stamps = g_gemm_stamps;
  if constexpr (KS2)
    return launch_ex_cl(kern, dim3(N / BN, (M + GEMM_BM - 1) / GEMM_BM, 2), dim3(64 + 32 * NE, 1, 1), Lay::TOTAL,
                        stream, dim3(CLUSTER, 1, 2), map_a, map_b, M, k_bytes, p, stamps);
  return launch_ex(kern, dim3(N / BN, (M + GEMM_BM - 1) / GEMM_BM, ksplit), dim3(64 + 32 * NE, 1, 1), Lay::TOTAL, stream,
                   CLUSTER, map_a, map_b, M, k_bytes, p, stamps);
}

}  // namespace samp
