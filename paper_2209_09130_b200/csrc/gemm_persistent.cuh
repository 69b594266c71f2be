// Persistent warp-specialised tcgen05 GEMM for the row-local epilogues (QKV quantize,
// FFN1 GELU+quantize, f16 bias/GELU outputs).
//
// Why: the one-tile-per-CTA kernel (gemm.cuh) runs each CTA's epilogue strictly after its
// own main loop, and co-resident CTAs start in the same phase, so at 768 FFN1 tiles the
// SMs alternate between "everyone loads" and "everyone runs GELU" over 2.6 waves
// (tools/gemm_phases.py: 8.7 us per tile, 5.5 us of it epilogue).  Here one CTA per SM
// walks a static tile list with TWO TMEM accumulators: the MMA warp fills buffer j&1 for
// tile j while the epilogue warps drain tile j-1 from the other buffer, so per SM the
// time is ~max(sum of epilogues, sum of main loops) instead of their sum.
//
// Roles (64 + 32*NE threads, 1 CTA / SM):
//   warp 0      TMA producer over the flat (tile, k-block) sequence; the first tile's
//               weight (B) boxes are issued before griddepcontrol.wait (PDL)
//   warp 1      TMEM allocator (2*BN columns) + MMA issuer; acc_full[b] / acc_empty[b]
//   warps 2..   NE epilogue warps (NE = 8 or 16): warp w reads TMEM lane quarter w%4 and
//               column part (w-2)/4 of BN; per tile they stage the NEXT tile's bias with
//               cp.async into the other of two epilogue smem buffers (the read-only tanh
//               table is loaded once per buffer at start).
// The epilogue structs are the ones of gemm.cuh (same run(), bit-identical results); their
// smem layout ends with the BN bias floats, which is what the per-tile staging rewrites.
#pragma once
#include "gemm.cuh"

namespace samp {


// epilogues with a read-only table (the GELU tanh table, 8 KB): one copy shared by both
// epilogue buffers instead of one per buffer (two copies pushed the 128-wide FFN1 ring past
// half of the SM's shared memory: one CTA per SM, the persistent grid ran as two waves)
template <class E, class = void> struct epi_table_bytes { static constexpr int value = 0; };
template <class E> struct epi_table_bytes<E, std::void_t<decltype(E::kTableBytes)>> {
  static constexpr int value = E::kTableBytes;
};

template <int BN, int STAGES, int EPI_BYTES, int TABLE_BYTES = 0>
struct PersistLayout {
  static constexpr int A_BYTES = GEMM_BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = STAGES * A_BYTES;
  static constexpr int BAR_OFF = B_OFF + STAGES * B_BYTES;             // full, empty, acc_full[2], acc_empty[2]
  static constexpr int EPI_STRIDE = (EPI_BYTES - TABLE_BYTES + 127) & ~127;   // per-buffer part
  static constexpr int TBL_OFF = (BAR_OFF + 8 * (2 * STAGES + 6) + 8 + 127) & ~127;   // + bias_full[2]
  static constexpr int EPI_OFF = TBL_OFF + ((TABLE_BYTES + 127) & ~127);
  static constexpr int TOTAL = EPI_OFF + 2 * EPI_STRIDE + 1024;
};
template <int BN, int STAGES, class Epi>
using PersistLayoutFor = PersistLayout<BN, STAGES, Epi::template smem_bytes<BN>(), epi_table_bytes<Epi>::value>;

// CTAS: persistent CTAs per SM (2 for the epilogue-bound FFN1: two CTAs' epilogue warps
// hide each other's MUFU / TMEM latencies; measured 24.2 vs 26.5 us at 4096 tokens)
template <int KIND, int BN, int STAGES, int NE, class Epi, int CTAS = 1>
__global__ void __launch_bounds__(64 + 32 * NE, CTAS)
gemm_persistent_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       int M, int N, int k_bytes, const typename Epi::Params ep, unsigned long long* stamps,
                       int n_fastest) {
  using Lay = PersistLayoutFor<BN, STAGES, Epi>;
  constexpr int TBL = epi_table_bytes<Epi>::value;
  constexpr int TMEM_COLS = tmem_cols_for(2 * BN);
  constexpr int PARTS = NE / 4;
  constexpr int EPI_BIAS_OFF = Epi::template smem_bytes<BN>() - TBL - BN * 4;   // within a buffer
  constexpr uint32_t IDESC = KIND == KIND_I8 ? idesc_i8(GEMM_BM, BN) : idesc_f16(GEMM_BM, BN);
  static_assert(2 * BN <= 512 && BN % 16 == 0, "two accumulators must fit TMEM");
  static_assert(NE == 8 || NE == 16, "epilogue warps");
  static_assert((BN / PARTS) % 8 == 0, "epilogue column chunks");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bias_full = acc_empty + 2;   // [2] tile bias landed in epilogue buffer b (bulk copy)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bias_full + 2);
  uint8_t* epi_smem = smem + Lay::EPI_OFF;

  const uint32_t warp = warp_id();
  const int mtiles = (M + GEMM_BM - 1) / GEMM_BM;
  const int ntiles = mtiles * (N / BN);
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int nk = k_bytes / 128;
  // raster: row tiles fastest (the CTAs running together share a weight tile; small M), or,
  // when the activation rows do not stay in L2 (n_fastest), weight tiles fastest so every
  // row tile is read from HBM once and the weights (<= a few MB) are the L2-resident operand
  const int ntn = N / BN;
  auto tile_m0 = [&](int j) {
    const int t = int(blockIdx.x) + j * int(gridDim.x);
    return (n_fastest ? t / ntn : t % mtiles) * GEMM_BM;
  };
  auto tile_n0 = [&](int j) {
    const int t = int(blockIdx.x) + j * int(gridDim.x);
    return (n_fastest ? t % ntn : t / mtiles) * BN;
  };
  // phase stamps (measurement): CTA b < 64, tile j < 16 -> stamps[(b*16 + j)*8 + f]:
  // f0 epilogue starts waiting, f1 accumulator ready, f2 epilogue done, f3 MMA starts
  // (buffer free), f4 last MMA of the tile issued, f5 producer issues the tile's first box
  auto stamp = [&](int j, int f) {
    if (stamps && blockIdx.x < 64 && j < 16) stamps[(blockIdx.x * 16 + j) * 8 + f] = globaltimer();
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NE);
      mbar_init(&bias_full[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one() && my_tiles > 0) {
      auto kcol = [](int kb) { return KIND == KIND_I8 ? kb * 128 : kb * 64; };
      const int total = my_tiles * nk;
      const int pre = nk < STAGES ? nk : STAGES;   // first tile's weights before the PDL wait
      const int n00 = tile_n0(0);
      stamp(0, 5);
      for (int kb = 0; kb < pre; ++kb) {
        mbar_expect_tx(&full[kb], Lay::A_BYTES + Lay::B_BYTES);
        tma_load_2d(smem + Lay::B_OFF + kb * Lay::B_BYTES, &map_b, kcol(kb), n00, &full[kb]);
      }
      pdl_wait();
      const int m00 = tile_m0(0);
      for (int kb = 0; kb < pre; ++kb)
        tma_load_2d(smem + Lay::A_OFF + kb * Lay::A_BYTES, &map_a, kcol(kb), m00, &full[kb]);
      // counters instead of per-box divisions: the issuing thread sits on the MMA's critical
      // path each time a stage frees (runtime div/mod per box measured +12% on C4's FFN1)
      int j = 0, kb = pre, m0 = m00, n0 = n00;
      int s = pre == STAGES ? 0 : pre;
      uint32_t par = pre == STAGES ? 0u : 1u;   // ((it / STAGES) & 1) ^ 1
      for (int it = pre; it < total; ++it) {
        if (kb == nk) {
          kb = 0;
          ++j;
          m0 = tile_m0(j);
          n0 = tile_n0(j);
        }
        mbar_wait(&empty[s], par);
        if (kb == 0) stamp(j, 5);
        mbar_expect_tx(&full[s], Lay::A_BYTES + Lay::B_BYTES);
        tma_load_2d(smem + Lay::A_OFF + s * Lay::A_BYTES, &map_a, kcol(kb), m0, &full[s]);
        tma_load_2d(smem + Lay::B_OFF + s * Lay::B_BYTES, &map_b, kcol(kb), n0, &full[s]);
        ++kb;
        if (++s == STAGES) {
          s = 0;
          par ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      int it = 0;
      for (int j = 0; j < my_tiles; ++j) {
        const int b = j & 1;
        mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        stamp(j, 3);
        // the tile's bias into epilogue buffer b: its readers (tile j-2's epilogue) are done
        // once they released the accumulator buffer.  One bulk copy, completing bias_full[b]:
        // no per-tile staging or barrier among the epilogue warps.
        if constexpr (Epi::kStagedBias) {
          mbar_expect_tx(&bias_full[b], BN * 4);
          bulk_load(epi_smem + b * Lay::EPI_STRIDE + EPI_BIAS_OFF, ep.bias + tile_n0(j), BN * 4, &bias_full[b]);
        }
        const uint32_t d = tmem + uint32_t(b * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_addr(smem + Lay::A_OFF + s * Lay::A_BYTES);
          const uint32_t b_base = smem_addr(smem + Lay::B_OFF + s * Lay::B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss<KIND>(d, sdesc_k_sw128(a_base + 32 * k), sdesc_k_sw128(b_base + 32 * k), IDESC, (kb | k) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[b]);
        stamp(j, 4);
      }
      pdl_trigger();   // last MMA issued: the next kernel's prologue overlaps our epilogues
    }
    __syncwarp();
  } else {
    const int ep_tid = threadIdx.x - GEMM_EPI_WARP0 * 32;
    const int quarter = warp & 3;
    const int part = int(warp - GEMM_EPI_WARP0) / 4;
    const int tile_row = quarter * 32 + lane_id();
    const int c0 = part * (BN / PARTS);
    pdl_wait();
    // read-only tables once (the staged-bias epilogues get each tile's bias by the MMA
    // warp's bulk copy; others stage their per-buffer operands here)
    if constexpr (TBL > 0) {
      load_tanh_table(reinterpret_cast<TanhTable*>(smem + Lay::TBL_OFF), ep_tid, 32 * NE);
    } else if constexpr (!Epi::kStagedBias) {
      for (int b = 0; b < 2 && b < my_tiles; ++b)
        Epi::template prefetch<BN>(ep, epi_smem + b * Lay::EPI_STRIDE, tile_m0(b), tile_n0(b), M, ep_tid, 32 * NE);
    }
    epi_bar_sync(32 * NE);
    for (int j = 0; j < my_tiles; ++j) {
      const int b = j & 1;
      // the tile's coordinates (runtime div/mod) while the accumulator is still in flight
      const int m0 = tile_m0(j), n0 = tile_n0(j);
      if (ep_tid == 0) stamp(j, 0);
      mbar_wait(&acc_full[b], (j >> 1) & 1);
      tc_fence_after();
      if constexpr (Epi::kStagedBias) mbar_wait(&bias_full[b], (j >> 1) & 1);
      if (ep_tid == 0) stamp(j, 1);
      EpiCtx c{tmem + (uint32_t(quarter * 32) << 16) + uint32_t(b * BN + c0), m0 + tile_row, tile_row, n0, c0,
               BN / PARTS, part, M, ep_tid, 32 * NE};
      if constexpr (TBL > 0) c.table = smem + Lay::TBL_OFF;
      Epi::template run<BN, 1, NE>(ep, c, epi_smem + b * Lay::EPI_STRIDE);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&acc_empty[b]);
      if (ep_tid == 0) stamp(j, 2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

inline int device_sm_count() {
  static thread_local int dev = -1, count = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  return count;
}

template <int KIND, int BN, int STAGES, int NE, class Epi, int CTAS = 1>
inline cudaError_t launch_gemm_persistent(const CUtensorMap& map_a, const CUtensorMap& map_b, int M, int N,
                                          int k_bytes, const typename Epi::Params& p, cudaStream_t stream) {
  using Lay = PersistLayoutFor<BN, STAGES, Epi>;
  auto kern = gemm_persistent_kernel<KIND, BN, STAGES, NE, Epi, CTAS>;
  static thread_local int configured = -1, resident = CTAS;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL);
    if (e != cudaSuccess) return e;
    max_carveout_once(kern);
    // the grid must be resident at once (a persistent grid larger than the SMs can hold runs
    // as two waves: the 128-wide FFN1 did at 116.9 KB per CTA before its GELU table was
    // shared).  Shared memory is the binding limit here; the occupancy API reports one CTA
    // per SM even where two demonstrably co-reside (tools/ubench/occ_probe.cu), so count it.
    int per_sm = 0, reserved = 0;
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int fit = per_sm / (Lay::TOTAL + reserved);
    resident = fit < 1 ? 1 : fit < CTAS ? fit : CTAS;
    configured = dev;
    if (std::getenv("SAMP_DEBUG_OCC"))
      std::fprintf(stderr, "[persistent] BN %d stages %d NE %d CTAS %d smem %d -> %d resident per SM\n", BN, STAGES,
                   NE, CTAS, Lay::TOTAL, resident);
  }
  const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * (N / BN);
  const int slots = device_sm_count() * resident;
  const int grid = tiles < slots ? tiles : slots;
  unsigned long long* stamps = g_gemm_stamps;
  // activations past ~48 MB (C5: 262k tokens) would be streamed from HBM once per weight
  // tile with row tiles fastest (ncu: FFN1 read 6.3 GB for a 201 MB input)
#ifdef SAMP_EXP_NO_NFASTEST
  const int n_fastest = 0;
#else
  const int n_fastest = size_t(M) * size_t(k_bytes) > (48u << 20) ? 1 : 0;
#endif
  return launch_ex(kern, dim3(grid), dim3(64 + 32 * NE), Lay::TOTAL, stream, 1, map_a, map_b, M, N, k_bytes, p,
                   stamps, n_fastest);
}

}  // namespace samp
