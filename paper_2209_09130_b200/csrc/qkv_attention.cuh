// Fused INT8 QKV projection + attention: one persistent CTA per SM walks (tile, head) work
// items; per item it computes the head's q|k|v GEMM columns (128 rows x 192 columns, K = H)
// on the tensor cores, quantizes them straight into shared memory, and runs the attention
// of the same tile (the sequences of the tile are the tile's own rows, S <= 128) on them.
//
// Reference semantics (pkg/src/samp/encoder.py:355-379): exactly those of the unfused pair
//   gemm_kernel<i8, EpiQKV>   q|k|v = quantize(F32(acc)*F32(s_in*s_w) + b, s_{q,k,v})
//   attention_kernel<i8>      scores, softmax, P codes, PV, ctx codes
// (same epilogue arithmetic, same att_softmax / att_ctx_out device code), so every code is
// bit-identical to the two-kernel path; only the q|k|v round trip through HBM/L2 and one
// launch boundary per layer disappear.
//
// Why: run separately, the QKV GEMM and the attention each fill and drain the whole GPU, and
// every attention CTA of a wave runs the same phase at the same time (load, MMA, then FMA-pipe
// softmax), so the tensor pipe idles during the softmax and the FMA pipe during the GEMM.
// Here the GEMM of item j+1 is issued while the softmax warps work on item j.
//
// Roles (64 + 128*TPR threads, one CTA per SM, all 512 TMEM columns):
//   warp 0      TMA producer: per item and k-block, the activation rows [128 x 128 B] and
//               the head's q, k and v weight rows [3 x 64 x 128 B] into a 3-stage ring
//   warp 1      TMEM owner + single-thread MMA issuer: an event loop over the GEMM k-blocks
//               (into two accumulators), MMA-1 (scores) and MMA-2 (P.V) of the items
//   warps 2..   TPR threads per query row: per item, the QKV epilogue of the NEXT item
//               (accumulator -> q|k|v codes in the 64B-swizzled K-major layout the MMAs read,
//               double-buffered in smem; it runs while MMA-2 of the current item computes),
//               then the softmax (att_softmax_rr) and the ctx codes (att_ctx_out)
// TMEM columns: q|k|v accumulator [0, 192), scores [256, 384), O [384, 448).
#pragma once
#include "attention.cuh"
#include "gemm.cuh"

namespace samp {

constexpr int QA_STAGES = 3;
constexpr int QA_SOFT_WARP0 = 2;
template <int TPR> constexpr int qa_threads() { return 32 * QA_SOFT_WARP0 + 128 * TPR; }

struct QALayout {
  static constexpr int A_BYTES = 128 * 128;              // activation rows x 128 B of K
  static constexpr int B_BYTES = 192 * 128;              // the head's q|k|v weight rows
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int QKV_OFF = QA_STAGES * STAGE;      // 2 x (Q, K, V: 128 rows x 64 B each)
  static constexpr int QKV_BYTES = 3 * 128 * 64;
  static constexpr int P_OFF = QKV_OFF + 2 * QKV_BYTES;  // P codes [128 rows][128 keys], 128B swizzle
  static constexpr int X_OFF = P_OFF + 128 * 128;
  static constexpr int X_BYTES = (3 * 4 + ATT_MAX_LEAVES + 1) * 128 * 4;
  static constexpr int BIAS_OFF = X_OFF + X_BYTES;       // q|k|v biases of every head (3H floats)
  static constexpr int BAR_OFF = BIAS_OFF + 3 * 1024 * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;     // + alignment slack
  static_assert(QKV_OFF % 1024 == 0 && P_OFF % 1024 == 0, "swizzle atoms need 1024-byte alignment");
};
// TMEM columns: the q|k|v accumulator, the scores and O = P.V each have their own columns,
// so MMA-1 of the next item (into the scores) never waits for this item's ctx (reading O)
constexpr uint32_t QA_TMEM_ACC = 0, QA_TMEM_S = 256, QA_TMEM_O = 384;

struct QAParams {
  AttnParams att;          // ctx output, tiles, sequence geometry, softmax / ctx scales
  const float* bias;       // [3H] q|k|v biases
  float mult0, mult1, mult2;   // F32(double(s_in) * double(s_w{q,k,v}))
  float sout0, sout1, sout2;   // F32(scale(L.attn.{q,k,v}))
  int8_t* qkv_out;         // optional [T][3H]: also store the q|k|v codes (stage capture)
  int heads, ntiles;
  // optional [ntiles] counters: +1 per softmax warp of a finished (tile, head) item once its
  // ctx rows are stored (release; 4 * TPR per item); the out-projection then starts on finished row tiles instead of
  // waiting for the whole grid, and this kernel triggers its dependents at its start
  int* tile_done;
  int late_trigger;        // measurement: keep the end-of-MMA trigger with tile_done set
};

// softmax warps' waits on the MMA results (s_full, o_full): a test_wait spin — one CTA per
// SM, so spinning only competes with this CTA's own warps, and the wake-up is immediate
// (C2 36.2-36.3k -> 36.9-37.1k sentences/s vs a parked try_wait, SAMP_QA_PARK=1 builds that)
#ifdef SAMP_QA_PARK
#define QA_SOFT_WAIT(bar, par) mbar_wait_park(bar, par)
#else
#define QA_SOFT_WAIT(bar, par) do { while (!mbar_test(bar, par)) {} } while (0)
#endif
#ifdef SAMP_QA_ACC_SPIN   // measurement: the epilogue's accumulator wait as a spin too
#define QA_ACC_WAIT(bar, par) do { while (!mbar_test(bar, par)) {} } while (0)
#else
#define QA_ACC_WAIT(bar, par) mbar_wait_park(bar, par)
#endif

template <int TPR>
__global__ void __launch_bounds__(qa_threads<TPR>(), 1)
qkv_attention_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_w,
                     const QAParams q) {
  using Lay = QALayout;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
  uint64_t* empty = full + QA_STAGES;
  uint64_t* acc_full = empty + QA_STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* qkv_full = acc_empty + 1;    // [2]
  uint64_t* s_full = qkv_full + 2;
  uint64_t* p_full = s_full + 1;
  uint64_t* o_full = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const AttnParams& p = q.att;
  const int H = p.hidden;
  const int nk = H / 128;                                // k-blocks of 128 bytes
  const int items = q.ntiles * q.heads;
  const int my = int(blockIdx.x) < items ? (items - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  // item order: tile-major, so the CTAs working at the same time share activation rows in L2
  auto item_tile = [&](int j) { return (int(blockIdx.x) + j * int(gridDim.x)) / q.heads; };
  auto item_head = [&](int j) { return (int(blockIdx.x) + j * int(gridDim.x)) % q.heads; };
  auto tile_keys = [&](int t) {   // padded keys of tile t
    const int seq = p.tile_seq[t];
    return ((p.seq_start[seq + 1] - p.seq_start[seq]) * p.tile_cnt[t] + 31) & ~31;
  };
  const uint32_t warp = warp_id();
  // phase stamps (measurement, tools/qa_phases.py): CTA b < 128, item j < 4 ->
  // p.stamps[(b*4 + j)*16 + f]: f0 epilogue waits, f1 accumulator ready, f2 codes written,
  // f3 softmax starts, f4-f7 pass 1 / pass 2 / sum / P written, f8 O ready, f9 ctx written,
  // f10 GEMM issue starts, f11 GEMM issued, f12 MMA-1 issued
  auto rec = [&](int j) -> unsigned long long* {
    return p.stamps && blockIdx.x < 128 && j < 4 ? p.stamps + (size_t(blockIdx.x) * 4 + j) * 16 : nullptr;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < QA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4 * TPR);
    for (int b = 0; b < 2; ++b) mbar_init(&qkv_full[b], 128 * TPR);
    mbar_init(s_full, 1);
    mbar_init(p_full, 128 * TPR);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_w);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one() && my > 0) {
      // weights do not depend on the previous kernel: the first item's weight boxes go out
      // before the PDL wait, its activation boxes after
      const int total = my * nk;
      const int pre = nk < QA_STAGES ? nk : QA_STAGES;
      auto load_w = [&](int s, int kb, int head) {
#pragma unroll
        for (int blk = 0; blk < 3; ++blk)
          tma_load_2d(smem + s * Lay::STAGE + Lay::A_BYTES + blk * 64 * 128, &map_w, kb * 128, blk * H + head * 64,
                      &full[s]);
      };
      const int head0 = item_head(0);
      for (int kb = 0; kb < pre; ++kb) {
        mbar_expect_tx(&full[kb], Lay::STAGE);
        load_w(kb, kb, head0);
      }
      pdl_wait();
      const int row00 = p.seq_start[p.tile_seq[item_tile(0)]];
      for (int kb = 0; kb < pre; ++kb) tma_load_2d(smem + kb * Lay::STAGE, &map_a, kb * 128, row00, &full[kb]);
      // per-item coordinates (two dependent global loads) once per item, not per box: the
      // issuing thread is on the MMA's critical path each time a ring slot frees
      int j = 0, kb = pre, head = head0, row0 = row00;
      int s = pre == QA_STAGES ? 0 : pre;
      uint32_t par = pre == QA_STAGES ? 0u : 1u;   // ((it / QA_STAGES) & 1) ^ 1
      for (int it = pre; it < total; ++it) {
        if (kb == nk) {
          kb = 0;
          ++j;
          head = item_head(j);
          row0 = p.seq_start[p.tile_seq[item_tile(j)]];
        }
        mbar_wait_park(&empty[s], par);
        mbar_expect_tx(&full[s], Lay::STAGE);
        load_w(s, kb, head);
        tma_load_2d(smem + s * Lay::STAGE, &map_a, kb * 128, row0, &full[s]);
        ++kb;
        if (++s == QA_STAGES) {
          s = 0;
          par ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one() && my > 0) {
      constexpr uint32_t IDESC_QKV = idesc_i8(128, 192);
      const uint32_t idesc_o = idesc_i8(128, 64, true);
      // Event loop over three in-order streams, most urgent first: MMA-2(m2) once P(m2) is
      // written (the softmax warps wait on O), MMA-1(m1) once the codes of m1 are in smem and
      // ctx(m1-1) has read O out of the score columns, and the GEMM k-blocks of item g as
      // soon as its accumulator is free and the ring slot has landed.  The GEMM of item j+1
      // thus runs while the epilogue drains item j and the softmax works on item j-1.
      int m1 = 0, m2 = 0, g = 0, gkb = 0, it = 0;
      // key counts of items m1 / m2 (dependent loads), refreshed as each advances, off the
      // path from a barrier flip to the MMA issue
      int nk1 = tile_keys(item_tile(0)), nk2 = nk1;
      while (m2 < my) {
        bool did = false;
        if (m2 < m1 && mbar_test(p_full, m2 & 1)) {
          tc_fence_after();
          const int b = m2 & 1;
          const int nkp = nk2;
          const uint32_t pa = smem_addr(smem + Lay::P_OFF);
          const uint32_t va = smem_addr(smem + Lay::QKV_OFF + b * Lay::QKV_BYTES + 2 * 128 * 64);
          for (int key = 0; key < nkp; key += 32)
            mma_ss<KIND_I8>(tmem + QA_TMEM_O, sdesc_k_sw128(pa + key), sdesc_mn_sw64(va + key * 64), idesc_o,
                            key != 0);
          mma_commit(o_full);
          if (rec(m2)) rec(m2)[15] = globaltimer();
          ++m2;
          if (m2 < my) nk2 = m2 == m1 ? nk1 : tile_keys(item_tile(m2));
          did = true;
        } else if (m1 == m2 && m1 < g && mbar_test(&qkv_full[m1 & 1], (m1 >> 1) & 1)) {
          tc_fence_after();
          const int b = m1 & 1;
          const int nkp = nk1;
          const uint32_t qa = smem_addr(smem + Lay::QKV_OFF + b * Lay::QKV_BYTES);
          const uint32_t ka = qa + 128 * 64;
          const uint32_t idesc_s = idesc_i8(128, nkp);
#pragma unroll
          for (int k = 0; k < 2; ++k)
            mma_ss<KIND_I8>(tmem + QA_TMEM_S, sdesc_k_sw64(qa + 32 * k), sdesc_k_sw64(ka + 32 * k), idesc_s, k);
          mma_commit(s_full);
          if (rec(m1)) rec(m1)[12] = globaltimer();
          ++m1;
          if (m1 < my) nk1 = tile_keys(item_tile(m1));
          did = true;
        } else if (g < my && g <= m1 &&   // GEMM(j+1) only after MMA-1(j): MMAs run in issue order,
                                            // so queued GEMM work would delay the scores the softmax waits for
                   (gkb > 0 || mbar_test(acc_empty, (g & 1) ^ 1)) &&
                   mbar_test(&full[it % QA_STAGES], (it / QA_STAGES) & 1)) {
          // one k-block of GEMM(g): acc[128 x 192] = A rows . [Wq | Wk | Wv] head slices
          tc_fence_after();
          if (gkb == 0 && rec(g)) rec(g)[10] = globaltimer();
          const int s = it % QA_STAGES;
          const uint32_t a_base = smem_addr(smem + s * Lay::STAGE);
          const uint32_t b_base = a_base + Lay::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss<KIND_I8>(tmem + QA_TMEM_ACC, sdesc_k_sw128(a_base + 32 * k), sdesc_k_sw128(b_base + 32 * k), IDESC_QKV,
                            (gkb | k) != 0);
          mma_commit(&empty[s]);
          ++it;
          if (++gkb == nk) {
            mma_commit(acc_full);
            if (rec(g)) rec(g)[11] = globaltimer();
            gkb = 0;
            ++g;
          }
          did = true;
        }
        if (!did) __nanosleep(20);   // one warp polling: keep the reaction time short
      }
      pdl_trigger();   // last MMA issued: the next kernel's prologue overlaps our tail
    }
    __syncwarp();
  } else {
    // ---------------- TPR threads per query row: QKV epilogue + softmax + ctx
    const int quarter = warp & 3;
    const int h = int(warp - QA_SOFT_WARP0) >> 2;
    const int r = quarter * 32 + lane_id();
    const int tid = int(threadIdx.x) - 32 * QA_SOFT_WARP0;
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    float* sbias = reinterpret_cast<float*>(smem + Lay::BIAS_OFF);
    for (int i = tid; i < 3 * H; i += 128 * TPR) sbias[i] = __ldg(q.bias + i);   // weights: before the PDL wait
    att_bar<TPR>();
    pdl_wait();   // ctx rows (and the capture copy) belong to the activation buffers of earlier kernels
    // every CTA of this persistent grid is resident: the out-projection's CTAs may launch
    // onto SMs as ours exit and start on the row tiles already published in tile_done
    if (q.tile_done && !q.late_trigger && tid == 0) pdl_trigger();
    // QKV epilogue of item jj: thread h converts columns [h*CW, h*CW + CW) of each of q, k, v
    // (EpiQKV's arithmetic on FFMA2 pairs: same roundings, gemm.cuh)
    constexpr int CW = 64 / TPR;
    auto epilogue = [&](int jj, unsigned long long* st) {
      const int b = jj & 1;
      const int head = item_head(jj);
      // the item's rows (two dependent global loads) only for the stage capture: on the
      // normal path nothing between the softmax and the accumulator wait touches memory
      int row0 = 0, rows = 0;
      if (q.qkv_out) {
        const int t = item_tile(jj), seq = p.tile_seq[t];
        row0 = p.seq_start[seq];
        rows = (p.seq_start[seq + 1] - row0) * p.tile_cnt[t];
      }
      if (st) st[0] = globaltimer();
      QA_ACC_WAIT(acc_full, jj & 1);
      tc_fence_after();
      if (st) st[1] = globaltimer();
      const uint32_t ta = tmem + QA_TMEM_ACC + lane_base + h * CW;
      uint32_t u[3][CW];
#pragma unroll
      for (int blk = 0; blk < 3; ++blk) {
        if constexpr (CW == 16) tmem_ld16(ta + blk * 64, u[blk]);
        else tmem_ld32(ta + blk * 64, u[blk]);
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(acc_empty);   // the accumulator is in registers
      uint8_t* buf = smem + Lay::QKV_OFF + b * Lay::QKV_BYTES + r * 64;
      const X2 kx = p.k;
#pragma unroll
      for (int blk = 0; blk < 3; ++blk) {
        const float mult = blk == 0 ? q.mult0 : blk == 1 ? q.mult1 : q.mult2;
        const Recip rq = make_recip(blk == 0 ? q.sout0 : blk == 1 ? q.sout1 : q.sout2);
        const float4* bias4 = reinterpret_cast<const float4*>(sbias + blk * H + head * 64 + h * CW);
        const float2 mm = f2(mult, mult);
        uint32_t wv[CW / 4];
#pragma unroll
        for (int g = 0; g < CW / 4; ++g) {
          const float4 bb = bias4[g];
          const float2 x0 = add2(mul2(f2(__int2float_rn(int(u[blk][4 * g])), __int2float_rn(int(u[blk][4 * g + 1]))), mm, kx),
                                 f2(bb.x, bb.y), kx);
          const float2 x1 = add2(mul2(f2(__int2float_rn(int(u[blk][4 * g + 2])), __int2float_rn(int(u[blk][4 * g + 3]))), mm, kx),
                                 f2(bb.z, bb.w), kx);
          const float2 q0 = quant_pre2(x0, rq, kx), q1 = quant_pre2(x1, rq, kx);
          wv[g] = trunc_pack4_s8(q0.x, q0.y, q1.x, q1.y);
        }
        // 64B swizzle: 16-byte chunk k of row r sits at chunk k ^ ((r >> 1) & 3)
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) {
          const int chunk = (h * CW / 16 + c) ^ ((r >> 1) & 3);
          *reinterpret_cast<uint4*>(buf + blk * 128 * 64 + chunk * 16) =
              make_uint4(wv[4 * c], wv[4 * c + 1], wv[4 * c + 2], wv[4 * c + 3]);
          if (q.qkv_out && r < rows)
            *reinterpret_cast<uint4*>(q.qkv_out + size_t(row0 + r) * 3 * H + blk * H + head * 64 + h * CW + 16 * c) =
                make_uint4(wv[4 * c], wv[4 * c + 1], wv[4 * c + 2], wv[4 * c + 3]);
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&qkv_full[b]);
      if (st) st[2] = globaltimer();
      if (lane_id() == 0 && rec(jj)) atomicMax(rec(jj) + 14, globaltimer());   // last warp's epilogue
    };
    // j = -1 only runs the first item's epilogue (one inlined copy of each phase: the
    // kernel's code must stay small for the instruction cache)
    // item geometry one item ahead (three levels of dependent global loads, ~1 us): the
    // tile's sequence before the next item's epilogue, the sequence's rows and attention
    // length before this item's ctx, the row geometry from registers at the loop top
    int tn = item_tile(0), seqn = p.tile_seq[tn], cntn = p.tile_cnt[tn];
    int k0n = p.seq_start[seqn], Sn = p.seq_start[seqn + 1] - k0n;
    int attn = p.att_len[seqn + att_sub(Sn, cntn, r)];
#pragma unroll 1
    for (int j = -1; j < my; ++j) {
      const int jc = j < 0 ? 0 : j;
      const int t = tn, head = item_head(jc);
      const AttRow w = att_row_of(Sn, attn, cntn, r, h);
      const size_t ctx_row = size_t(k0n + r);
      unsigned long long* st = threadIdx.x == 32 * QA_SOFT_WARP0 && j >= 0 ? rec(j) : nullptr;
      if (j >= 0) {
#ifdef SAMP_QA_STAMP_PRESOFT   // measurement: st[0] := reached the s_full wait (overwrites epi_wait)
        if (st) st[0] = globaltimer();
#endif
        QA_SOFT_WAIT(s_full, j & 1);
        tc_fence_after();
        if (st) st[3] = globaltimer();
        att_softmax_rr<TPR>(p, w, tmem + QA_TMEM_S + lane_base, smem + Lay::P_OFF, smem + Lay::X_OFF, p_full,
                            st ? st + 1 : nullptr);
      }
      if (j >= 0 && j + 1 < my) {   // next item: its tile's sequence
        tn = item_tile(j + 1);
        seqn = p.tile_seq[tn];
        cntn = p.tile_cnt[tn];
      }
      // the next item's codes while MMA-2 of this one runs (its MMA-1 then only waits for ctx)
      if (j + 1 < my) epilogue(j + 1, threadIdx.x == 32 * QA_SOFT_WARP0 ? rec(j + 1) : nullptr);
      if (j < 0) continue;
      if (j + 1 < my) {   // next item: the sequence's rows and attention length
        k0n = p.seq_start[seqn];
        Sn = p.seq_start[seqn + 1] - k0n;
        attn = p.att_len[seqn + att_sub(Sn, cntn, r)];
      }
      QA_SOFT_WAIT(o_full, j & 1);
      tc_fence_after();
      if (st) st[8] = globaltimer();
      att_ctx_out<false, TPR>(p, w, tmem + QA_TMEM_O + lane_base, ctx_row, head, 0.0f);
      if (q.tile_done) {   // publish: the warp's ctx stores, then one release add per warp
        __syncwarp();
        if (lane_id() == 0) red_release_gpu_add(q.tile_done + t, 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0 && rec(j)) atomicMax(rec(j) + 13, globaltimer());   // last warp's ctx
      if (st) st[9] = globaltimer();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace samp
