// Persistent cluster GEMM with the fused residual + LayerNorm (+ quantize) epilogue, for
// the out-projection and FFN2 at large token counts (configs C4/C5).
//
// Why: the one-tile LN GEMM (gemm.cuh, EpiResLN) runs each CTA's main loop and its long
// LayerNorm epilogue back to back, one tile per CTA; with thousands of row tiles the SMs
// alternate between "everyone loads/MMAs" and "everyone normalises".  Here a cluster of
// CLUSTER CTAs (one N slice of BN columns each, CLUSTER*BN = H) walks row tiles
// m = cluster, cluster + nclusters, ... with TWO TMEM accumulators: the MMA warp fills
// buffer j&1 for tile j while the epilogue warps normalise tile j-1.
//
// Row statistics need all H columns, i.e. all CLUSTER CTAs.  The one-tile kernel exchanges
// them with cluster-wide barriers; here the producer and MMA warps are busy with later
// tiles, so the exchange is point-to-point through DSMEM: each CTA stores its per-row
// partial sums into every peer's xpart[slot][reduction][rank][row] (st.shared::cluster) and
// then arrives (release, cluster scope) on the peer's xbar[slot][reduction] (4 arrivals per
// phase); the consumer waits (acquire) on its own barrier and adds the partials in rank
// order, ((p0+p1)+(p2+p3)) — the numpy tree above the per-CTA subtrees, exactly as the
// one-tile kernel (reference kernels.layernorm :138-154).  Two slots by tile parity make
// reuse safe: a CTA writes tile j+2's partials only after it read every peer's tile j+1
// partials, which each peer wrote after finishing tile j.
//
// Arithmetic per element is EpiResLN::run_regs's (same operations, same order): bit-
// identical outputs.  Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps
// 2..9 epilogue (two threads per row, BN/2 columns each = one numpy subtree).
#pragma once
#include <algorithm>
#include <cstdio>
#include <vector>

#include "gemm_persistent.cuh"

namespace samp {

template <int BN, int STAGES, int CLUSTER>
struct LnPersistLayout {
  static constexpr int A_BYTES = GEMM_BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = STAGES * A_BYTES;
  // full[S], empty[S], acc_full[2], acc_empty[2], xbar[2 slots][2 reductions], tmem slot
  static constexpr int BAR_OFF = B_OFF + STAGES * B_BYTES;
  static constexpr int NBARS = 2 * STAGES + 4 + 4;
  static constexpr int PAR_OFF = (BAR_OFF + 8 * NBARS + 8 + 127) & ~127;      // bias/gamma/beta [3][BN]
  static constexpr int HALF_OFF = PAR_OFF + 3 * BN * 4;                          // halves [2 red][2][128]
  static constexpr int XP_OFF = HALF_OFF + 2 * 2 * 128 * 4;                      // xpart [2][2][CLUSTER][128]
  static constexpr int RES_OFF = XP_OFF + 2 * 2 * CLUSTER * 128 * 4;             // residual int8 [2][128][BN]
  static constexpr int TOTAL = RES_OFF + 2 * 128 * BN + 1024;
};

template <int KIND, int BN, int STAGES, int CLUSTER>
__global__ void __launch_bounds__(64 + 32 * 8, 1)
gemm_ln_persistent_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                          int M, int k_bytes, const EpiResLN::Params p) {
  using Lay = LnPersistLayout<BN, STAGES, CLUSTER>;
  constexpr int NE = 8;
  constexpr int NC = BN / 2;                  // columns per epilogue thread (one numpy subtree)
  constexpr int TMEM_COLS = tmem_cols_for(2 * BN);
  constexpr uint32_t IDESC = KIND == KIND_I8 ? idesc_i8(GEMM_BM, BN) : idesc_f16(GEMM_BM, BN);
  static_assert(2 * BN <= 512 && NC % 32 == 0 && NC <= 128, "tile shape");
  static_assert(CLUSTER == 2 || CLUSTER == 4, "cluster along N");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* xbar = acc_empty + 2;             // [slot][reduction]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 4);
  float* spar = reinterpret_cast<float*>(smem + Lay::PAR_OFF);
  float* halves = reinterpret_cast<float*>(smem + Lay::HALF_OFF);
  float* xpart = reinterpret_cast<float*>(smem + Lay::XP_OFF);

  const uint32_t warp = warp_id();
  const uint32_t rank = cluster_rank();
  const int ncl = int(gridDim.x) / CLUSTER, cid = int(blockIdx.x) / CLUSTER;
  const int mtiles = (M + GEMM_BM - 1) / GEMM_BM;
  const int my_tiles = cid < mtiles ? (mtiles - 1 - cid) / ncl + 1 : 0;   // same for every CTA of a cluster
  const int n0 = int(rank) * BN;
  const int nk = k_bytes / 128;
  auto tile_m0 = [&](int j) { return (cid + j * ncl) * GEMM_BM; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NE);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&xbar[i], 1);   // local expect_tx + remote complete_tx bytes
    fence_barrier_init();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  // constant per CTA: this N slice's bias / gamma / beta
  for (int i = threadIdx.x; i < BN; i += blockDim.x) {
    spar[i] = __ldg(p.bias + n0 + i);
    spar[BN + i] = __ldg(p.gamma + n0 + i);
    spar[2 * BN + i] = __ldg(p.beta + n0 + i);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                          // peers' barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one() && my_tiles > 0) {
      auto kcol = [](int kb) { return KIND == KIND_I8 ? kb * 128 : kb * 64; };
      const int total = my_tiles * nk;
      const int pre = nk < STAGES ? nk : STAGES;
      for (int kb = 0; kb < pre; ++kb) {
        mbar_expect_tx(&full[kb], Lay::A_BYTES + Lay::B_BYTES);
        tma_load_2d(smem + Lay::B_OFF + kb * Lay::B_BYTES, &map_b, kcol(kb), n0, &full[kb]);
      }
      pdl_wait();
      for (int kb = 0; kb < pre; ++kb)
        tma_load_2d(smem + Lay::A_OFF + kb * Lay::A_BYTES, &map_a, kcol(kb), tile_m0(0), &full[kb]);
      // counters, no per-box division (gemm_persistent.cuh)
      int kb = pre, m0 = tile_m0(0);
      int s = pre == STAGES ? 0 : pre;
      uint32_t par = pre == STAGES ? 0u : 1u;
      for (int it = pre; it < total; ++it) {
        if (kb == nk) {
          kb = 0;
          m0 += ncl * GEMM_BM;
        }
        mbar_wait(&empty[s], par);
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
      }
      pdl_trigger();
    }
    __syncwarp();
  } else {
    const int ep_tid = threadIdx.x - GEMM_EPI_WARP0 * 32;
    const int quarter = warp & 3;
    const int h = int(warp - GEMM_EPI_WARP0) / 4;      // column half
    const int tile_row = quarter * 32 + lane_id();
    const int c0 = h * NC;
    const float* sbias = spar;
    const float* sgam = spar + BN;
    const float* sbet = spar + 2 * BN;
    const float hf = float(p.hidden);
    const Recip rq = make_recip(p.out_i8 || p.deq_outputs ? p.s_out : 1.0f);
    pdl_wait();                                  // residuals / outputs belong to earlier kernels
    // residual codes: each thread copies its own row half of tile j+1 (cp.async) while it
    // works on tile j, so only its own wait_group is needed before reading them
    uint8_t* rbuf = smem + Lay::RES_OFF;
    auto stage_res = [&](int j) {
      const int row = tile_m0(j) + tile_row;
      if (p.res_i8 && row < M) {
        uint8_t* dst = rbuf + ((j & 1) * 128 + tile_row) * BN + c0;
        const int8_t* src = p.res_i8 + size_t(row) * p.hidden + n0 + c0;
#pragma unroll
        for (int q = 0; q < NC / 16; ++q) cp_async16(dst + 16 * q, src + 16 * q);
      }
      cp_async_commit();
    };
    if (my_tiles > 0) stage_res(0);
    for (int j = 0; j < my_tiles; ++j) {
      const int b = j & 1, slot = j & 1;
      const uint32_t xphase = (j >> 1) & 1;
      const int row = tile_m0(j) + tile_row;
      const bool valid = row < M;
      const size_t rbase = size_t(valid ? row : 0) * p.hidden;
      if (j + 1 < my_tiles) stage_res(j + 1);
      else cp_async_commit();
      cp_async_wait_group1();                    // tile j's residual group has landed
      uint4 rv[NC / 16];
      if (p.res_i8) {
#pragma unroll
        for (int q = 0; q < NC / 16; ++q)
          rv[q] = reinterpret_cast<const uint4*>(rbuf + (b * 128 + tile_row) * BN + c0)[q];
      }
      mbar_wait(&acc_full[b], (j >> 1) & 1);
      tc_fence_after();
      float x[NC];
      {
        uint32_t r[NC];
        const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(b * BN + c0);
#pragma unroll
        for (int kk = 0; kk < NC / 32; ++kk) tmem_ld32(taddr + 32 * kk, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * kk));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&acc_empty[b]);    // accumulator consumed: next MMA may start
#pragma unroll
        for (int kk = 0; kk < NC / 32; ++kk) {
          float rf[32];   // f32 residual (FP layers): 16-byte loads
          if (!p.res_i8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(p.res_f32 + rbase + n0 + c0 + 32 * kk) + q)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
              rf[4 * q] = v.x; rf[4 * q + 1] = v.y; rf[4 * q + 2] = v.z; rf[4 * q + 3] = v.w;
            }
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int cc = 32 * kk + jj;
            float res;
            if (p.res_i8) {
              const uint32_t w = reinterpret_cast<const uint32_t*>(&rv[cc / 16])[(cc % 16) / 4];
              res = deq(int(int8_t((w >> (8 * (cc % 4))) & 0xff)), p.res_scale);
            } else {
              res = rf[jj];
            }
            const uint32_t u = r[cc];
            const float acc = p.acc_is_f32 ? __uint_as_float(u) : __fmul_rn(__int2float_rn(int(u)), p.mult);
            x[cc] = __fadd_rn(__fadd_rn(acc, sbias[c0 + cc]), res);
          }
        }
      }
      // numpy leaf over NC: 8 strided accumulators, ((0+1)+(2+3))+((4+5)+(6+7))
      auto leaf = [&](auto f) {
        float a8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a8[q] = f(x[q]);
#pragma unroll
        for (int g = 1; g < NC / 8; ++g)
#pragma unroll
          for (int q = 0; q < 8; ++q) a8[q] = __fadd_rn(a8[q], f(x[8 * g + q]));
        return __fadd_rn(__fadd_rn(__fadd_rn(a8[0], a8[1]), __fadd_rn(a8[2], a8[3])),
                         __fadd_rn(__fadd_rn(a8[4], a8[5]), __fadd_rn(a8[6], a8[7])));
      };
      // (half0 + half1) inside the CTA, then the CLUSTER CTAs' partials in rank order
      auto reduce = [&](float mine, int red) {
        float* hv = halves + red * 256;
        hv[h * 128 + tile_row] = mine;
        epi_bar_sync(32 * NE);
        const float s = __fadd_rn(hv[tile_row], hv[128 + tile_row]);
        float* xp = xpart + ((slot * 2 + red) * CLUSTER + int(rank)) * 128 + tile_row;
        uint64_t* xb = &xbar[slot * 2 + red];
        if (ep_tid == 0) mbar_expect_tx(xb, CLUSTER * 128 * 4);   // this phase: every CTA's 128 partials
        if (h == 0) {
#pragma unroll
          for (int rr = 0; rr < CLUSTER; ++rr) st_async_f32(mapa_rank(xp, rr), s, mapa_rank(xb, rr));
        }
        mbar_wait(xb, xphase);
        const float* mine_xp = xpart + (slot * 2 + red) * CLUSTER * 128 + tile_row;
        float pr[CLUSTER];
#pragma unroll
        for (int rr = 0; rr < CLUSTER; ++rr) pr[rr] = mine_xp[rr * 128];
        if constexpr (CLUSTER == 2) return __fadd_rn(pr[0], pr[1]);
        else return __fadd_rn(__fadd_rn(pr[0], pr[1]), __fadd_rn(pr[2], pr[3]));
      };
      const float total = reduce(leaf([](float v) { return v; }), 0);
      const float mean = __fdiv_rn(__fadd_rn(0.0f, total), hf);
      const float total2 = reduce(leaf([mean](float v) {
                                    const float d = __fsub_rn(v, mean);
                                    return __fmul_rn(d, d);
                                  }),
                                  1);
      const float var = __fdiv_rn(__fadd_rn(0.0f, total2), hf);
      const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
      float amx = 0.0f;
      if (valid) {
#pragma unroll
        for (int kk = 0; kk < NC / 32; ++kk) {
          float y[32];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int col = c0 + 32 * kk + jj;
            y[jj] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(x[32 * kk + jj], mean), inv), sgam[col]), sbet[col]);
          }
          EpiResLN::emit32(p, rbase, n0 + c0 + 32 * kk, rq, y, amx);
        }
      }
      if (p.amax) {
        amax_commit(p.amax + p.site, amx);
        if (p.site2 >= 0) amax_commit(p.amax + p.site2, amx);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                          // no CTA leaves while peers may still address its smem
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// How many clusters of CLUSTER CTAs with `smem` bytes each are really co-resident.  The
// occupancy API reports 37 clusters of 4 at ~221 KB/CTA on a 148-SM B200, but GPC packing
// fits 33: a persistent grid of 34+ clusters leaves its last clusters waiting for others
// to finish and takes ~1.6x longer (measured).  The probe launches every candidate cluster
// holding its SMs for ~40 us and counts those that started together.
static __global__ void cluster_probe_kernel(unsigned long long* starts) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    starts[blockIdx.x] = t0;
    while (globaltimer() - t0 < 40000ull) {
    }
  }
}

static inline int probe_coresident_clusters(int cluster, size_t smem) {
  const int sms = device_sm_count();
  const int n = (sms / cluster) * cluster;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, n * sizeof(unsigned long long)) != cudaSuccess) return sms / cluster;
  cudaFuncSetAttribute(cluster_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(cluster_probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int together = sms / cluster;
  if (cudaLaunchKernelEx(&cfg, cluster_probe_kernel, d) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess) {
    std::vector<unsigned long long> h(n);
    cudaMemcpy(h.data(), d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const unsigned long long t_min = *std::min_element(h.begin(), h.end());
    int started = 0;
    for (unsigned long long t : h) started += t < t_min + 20000ull;
    together = std::max(1, started / cluster);
  }
  cudaGetLastError();
  cudaFree(d);
  return together;
}

template <int KIND, int BN, int STAGES, int CLUSTER>
inline int ln_persistent_clusters() {
  static thread_local int dev = -1, n = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    n = probe_coresident_clusters(CLUSTER, LnPersistLayout<BN, STAGES, CLUSTER>::TOTAL);
    dev = d;
    if (std::getenv("SAMP_VERBOSE")) std::fprintf(stderr, "ln_persistent: %d co-resident clusters of %d (BN %d)\n", n, CLUSTER, BN);
  }
  return n;
}

template <int KIND, int BN, int STAGES, int CLUSTER>
inline cudaError_t launch_gemm_ln_persistent(const CUtensorMap& map_a, const CUtensorMap& map_b, int M,
                                             int k_bytes, const EpiResLN::Params& p, cudaStream_t stream) {
  using Lay = LnPersistLayout<BN, STAGES, CLUSTER>;
  auto kern = gemm_ln_persistent_kernel<KIND, BN, STAGES, CLUSTER>;
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  const int mtiles = (M + GEMM_BM - 1) / GEMM_BM;
  int clusters = std::min(mtiles, ln_persistent_clusters<KIND, BN, STAGES, CLUSTER>());
  if (const char* f = std::getenv("SAMP_LNP_CLUSTERS")) clusters = std::min(mtiles, std::atoi(f));   // measurement
  return launch_ex(kern, dim3(clusters * CLUSTER), dim3(64 + 32 * 8), Lay::TOTAL, stream, CLUSTER, map_a, map_b, M,
                   k_bytes, p);
}

}  // namespace samp
