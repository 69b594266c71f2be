// Padding-free (varlen) multi-head attention, one CTA per (128-query tile, head),
// INT8 (kind::i8) or FP16 (kind::f16) operands.
//
// INT8 semantics (reference pkg/src/samp/encoder.py:368-379, kernels.py:130-135):
//   scores = F32(Q_q . K_q^T) * F32(s_q*s_k/sqrt(d)) + mask      mask = -10000 for keys >= att_len
//   probs  = softmax_rows(scores)   (row max, numpy exp, numpy pairwise sum, IEEE divide)
//   P_q    = quantize(probs, s_softmax)
//   ctx_q  = quantize(F32(P_q . V_q) * F32(s_softmax*s_v), s_out_in)
// FP semantics (encoder.py:298-305): scores = (Q.K^T)*F32(1/sqrt(d)) + mask, same softmax,
//   ctx = P . V, with Q/K/V/P/ctx held in f16 (the reference's fp16-storage points).
// Rows and keys of a sequence are its full (possibly padded) length S, so each sequence
// sees exactly the reference's per-sequence arithmetic; packing sequences back to back
// removes the reference's batch padding (cli.py:375-377 runs sequences one by one).
//
// Data path: TMA loads Q [128 x d], K and V [S x d] straight out of the fused QKV
// activation [T][3H] (64B swizzle for int8 rows of 64 B, 128B swizzle for f16 rows of
// 128 B).  tcgen05.mma #1: S_acc[128 x S] = Q K^T into TMEM (K-major A and B).  The four
// softmax warps own one query row per thread: they pull the row out of TMEM, write x and
// e back into TMEM, reduce e with numpy's pairwise tree and store P into smem in the
// 128B-swizzled K-major layout.  tcgen05.mma #2: O_acc[128 x 64] = P V, V consumed
// MN-major straight from its TMA image.  P is produced in chunks of up to 256 keys so the
// f16 path fits S = 512 in shared memory.
#pragma once
#include <cuda_fp16.h>

#include "numerics.cuh"
#include "sm100.cuh"

namespace samp {

constexpr int ATT_THREADS = 288;   // warp 0: TMA + MMA + TMEM owner; warps 1-8: softmax (2 per row)
constexpr int ATT_MAX_LEAVES = 8;  // numpy tree leaves for S <= 512
constexpr int ATT_MAX_KEYS = 512;
constexpr int ATT_P_CHUNK = 256;   // keys of P written per MMA-2 round

struct AttnParams {
  void* ctx_out;              // [T][H] int8 codes (INT8) or f16 values (FP16)
  const int* tile_seq;        // [ntiles] sequence of each 128-query tile
  const int* tile_q0;         // [ntiles] first query (within the sequence)
  const int* seq_start;       // [nseq+1] packed row offsets
  const int* att_len;         // [nseq]
  int hidden;                 // H
  float mult_scores;          // INT8: F32(s_q*s_k/sqrt(d))   FP16: F32(1/sqrt(d))
  float s_softmax;            // INT8: F32(scale(L.attn.softmax))
  float mult_ctx;             // INT8: F32(s_softmax*s_v)
  float s_ctx;                // INT8: F32(scale(L.attn.out_in))
  int tmem_cols;              // power of two >= max(64, padded keys in the batch)
  float* amax;                // FP16 calibration: site amax array (null = off)
  int site_sm, site_ctx;      // L.attn.softmax / L.attn.out_in
};

template <bool F16>
struct AttnCfg {
  static constexpr int ROW_BYTES = F16 ? 128 : 64;       // one head row (d = 64)
  static constexpr int KEY_STEP = F16 ? 16 : 32;         // keys per MMA-2 instruction
  static constexpr int KEYS_PER_PBLK = F16 ? 64 : 128;   // keys per 128B-swizzled P block
  static constexpr int P_ELT = F16 ? 2 : 1;
};

template <bool F16>
struct AttnLayout {
  int q_off, k_off, v_off, p_off, x_off, bar_off, total;
  __host__ __device__ AttnLayout(int keys_cap) {
    using C = AttnCfg<F16>;
    const int kv = ((keys_cap + 63) / 64) * 64 * C::ROW_BYTES;
    const int pchunk = keys_cap < ATT_P_CHUNK ? ((keys_cap + 127) / 128) * 128 : ATT_P_CHUNK;
    q_off = 0;
    k_off = q_off + 128 * C::ROW_BYTES;
    v_off = k_off + kv;
    p_off = ((v_off + kv + 1023) / 1024) * 1024;
    x_off = p_off + 128 * pchunk * C::P_ELT;
    bar_off = x_off + (2 + 2 * ATT_MAX_LEAVES) * 128 * 4;
    total = bar_off + 64 + 1024;
  }
};

// named barrier among the 256 softmax threads
__device__ __forceinline__ void att_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <bool F16>
__global__ void __launch_bounds__(ATT_THREADS, 3)
attention_kernel(const __grid_constant__ CUtensorMap map_qkv, const AttnParams p, int keys_cap) {
  using C = AttnCfg<F16>;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array keeps the shared address space visible
  // to the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const AttnLayout<F16> lay(keys_cap);
  uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* bar_s = bar_load + 1;       // MMA-1 done
  uint64_t* bar_p = bar_load + 2;       // P chunk written (128 arrivals per phase)
  uint64_t* bar_pf = bar_load + 3;      // MMA-2 round done (P buffer free / O ready)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_load + 4);

  const int tile = blockIdx.x, head = blockIdx.y;
  const int seq = p.tile_seq[tile];
  const int q0 = p.tile_q0[tile];
  const int row0 = p.seq_start[seq];
  const int S = p.seq_start[seq + 1] - row0;
  const int att = p.att_len[seq];
  const int nkp = (S + 31) & ~31;       // keys padded to the MMA K step (32 covers both kinds)
  const int nchunks = (nkp + ATT_P_CHUNK - 1) / ATT_P_CHUNK;
  const uint32_t warp = warp_id();

  if (threadIdx.x == 0) {
    mbar_init(bar_load, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_p, 256);
    mbar_init(bar_pf, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int KIND = F16 ? KIND_F16 : KIND_I8;
  if (warp == 0) {
    if (elect_one()) {
      pdl_wait();   // Q/K/V come from the QKV GEMM; every later access is ordered after this
      const int nblk = (nkp + 63) / 64;
      mbar_expect_tx(bar_load, 128 * C::ROW_BYTES + 2 * nblk * 64 * C::ROW_BYTES);
      const int H = p.hidden;
      // one tensor map (box = one head row x 64 rows) serves Q, K and V
      tma_load_2d(smem + lay.q_off, &map_qkv, head * 64, row0 + q0, bar_load);
      tma_load_2d(smem + lay.q_off + 64 * C::ROW_BYTES, &map_qkv, head * 64, row0 + q0 + 64, bar_load);
      for (int b = 0; b < nblk; ++b) {
        tma_load_2d(smem + lay.k_off + b * 64 * C::ROW_BYTES, &map_qkv, H + head * 64, row0 + b * 64, bar_load);
        tma_load_2d(smem + lay.v_off + b * 64 * C::ROW_BYTES, &map_qkv, 2 * H + head * 64, row0 + b * 64, bar_load);
      }
      mbar_wait(bar_load, 0);
      tc_fence_after();
      // MMA 1: S_acc[:, n0:n0+nn] = Q . K[n0:n0+nn]^T over d = 64 (K steps of 32 bytes)
      const uint32_t qa = smem_addr(smem + lay.q_off), ka = smem_addr(smem + lay.k_off);
      for (int n0 = 0; n0 < nkp; n0 += 256) {
        const int nn = min(256, nkp - n0);
        const uint32_t idesc = F16 ? idesc_f16(128, nn) : idesc_i8(128, nn);
#pragma unroll
        for (int k = 0; k < C::ROW_BYTES / 32; ++k) {
          const uint64_t ad = F16 ? sdesc_k_sw128(qa + 32 * k) : sdesc_k_sw64(qa + 32 * k);
          const uint64_t bd = F16 ? sdesc_k_sw128(ka + n0 * C::ROW_BYTES + 32 * k)
                                  : sdesc_k_sw64(ka + n0 * C::ROW_BYTES + 32 * k);
          mma_ss<KIND>(tmem + n0, ad, bd, idesc, k);
        }
      }
      mma_commit(bar_s);
      // MMA 2 rounds: O_acc += P[:, chunk] . V[chunk] (V MN-major), after each P chunk lands
      const uint32_t pa = smem_addr(smem + lay.p_off), va = smem_addr(smem + lay.v_off);
      const uint32_t idesc2 = F16 ? idesc_f16(128, 64, true) : idesc_i8(128, 64, true);
      for (int ch = 0; ch < nchunks; ++ch) {
        mbar_wait(bar_p, ch & 1);
        tc_fence_after();
        const int k_lo = ch * ATT_P_CHUNK, k_hi = min(nkp, k_lo + ATT_P_CHUNK);
        for (int key = k_lo; key < k_hi; key += C::KEY_STEP) {
          const int local = key - k_lo;
          const uint32_t a_addr = pa + (local / C::KEYS_PER_PBLK) * 16384 + (local % C::KEYS_PER_PBLK) * C::P_ELT;
          const uint32_t v_addr = va + key * C::ROW_BYTES;
          const uint64_t bd = F16 ? make_sdesc(v_addr, 1024, 1024, SW_128B) : sdesc_mn_sw64(v_addr);
          mma_ss<KIND>(tmem, sdesc_k_sw128(a_addr), bd, idesc2, key != 0);
        }
        mma_commit(bar_pf);
      }
      pdl_trigger();   // last MMA issued: the next kernel's prologue overlaps our epilogue
    }
    __syncwarp();
  } else {
    // two threads per query row: h = 0 (warps 1-4) and h = 1 (warps 5-8) of the same
    // TMEM lane quarter.  Element-wise passes split the 32-column chunks between them;
    // inside every numpy leaf h owns the strided accumulators r[4h..4h+3], and
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) is exactly numpy's combine.
    const int quarter = warp & 3;
    const int h = int(warp - 1) >> 2;
    const int r = quarter * 32 + lane_id();            // query row within the tile
    const uint32_t ta = tmem + (uint32_t(quarter * 32) << 16);
    float* xch = reinterpret_cast<float*>(smem + lay.x_off);   // [2][128] max / denom exchange
    float* part = xch + 2 * 128;                               // [2][ATT_MAX_LEAVES][128]
    mbar_wait(bar_s, 0);
    tc_fence_after();

    // pass 1: x = acc*mult + mask -> TMEM, row max over the S real keys
    // (chunks entirely inside [0, min(att, S)) skip the per-key mask / bounds checks)
    float mx = -INFINITY;
    const int clean = min(att, S);
    for (int c0 = 32 * h; c0 < nkp; c0 += 64) {
      uint32_t v[32];
      tmem_ld32(ta + c0, v);
      tmem_wait_ld();
      if (c0 + 32 <= clean) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float acc = F16 ? __uint_as_float(v[j]) : __int2float_rn(int(v[j]));
          const float x = __fadd_rn(__fmul_rn(acc, p.mult_scores), 0.0f);
          mx = fmaxf(mx, x);
          v[j] = __float_as_uint(x);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int key = c0 + j;
          const float acc = F16 ? __uint_as_float(v[j]) : __int2float_rn(int(v[j]));
          const float x = __fadd_rn(__fmul_rn(acc, p.mult_scores), key < att ? 0.0f : -10000.0f);
          if (key < S) mx = fmaxf(mx, x);
          v[j] = __float_as_uint(x);
        }
      }
      tmem_st32(ta + c0, v);
    }
    tmem_wait_st();
    xch[h * 128 + r] = mx;
    att_bar();
    mx = fmaxf(xch[r], xch[128 + r]);
    // pass 2: e = exp(x - max) -> TMEM (0 past S); x - max <= 0 (numpy exp on that domain)
    for (int c0 = 32 * h; c0 < nkp; c0 += 64) {
      uint32_t v[32];
      tmem_ld32(ta + c0, v);
      tmem_wait_ld();
      if (c0 + 32 <= S) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(np_expf_nonpos(__fsub_rn(__uint_as_float(v[j]), mx)));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = (c0 + j) < S ? np_expf_nonpos(__fsub_rn(__uint_as_float(v[j]), mx)) : 0.0f;
          v[j] = __float_as_uint(e);
        }
      }
      tmem_st32(ta + c0, v);
    }
    tmem_wait_st();
    tc_fence_before();
    att_bar();                                    // every e of the row is in TMEM
    tc_fence_after();
    // numpy pairwise sum over the S keys: half-leaf partials first ...
    auto half_leaf = [&](int lo, int n, int li) {
      if (n >= 8) {
        const int body = n - (n & 7);
        float acc[4];
        uint32_t u[8];
        tmem_ld8(ta + lo, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = __uint_as_float(u[4 * h + j]);
        for (int i = 8; i < body; i += 8) {
          tmem_ld8(ta + lo + i, u);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] = __fadd_rn(acc[j], __uint_as_float(u[4 * h + j]));
        }
        part[(h * ATT_MAX_LEAVES + li) * 128 + r] = __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
      }
      return 0.0f;
    };
    pw_tree_eval(S, half_leaf);
    att_bar();
    // ... then h = 0 combines leaves (+ sequential tails) up numpy's tree
    if (h == 0) {
      auto full_leaf = [&](int lo, int n, int li) {
        float res = 0.0f;
        int tail_lo = lo;
        if (n >= 8) {
          res = __fadd_rn(part[li * 128 + r], part[(ATT_MAX_LEAVES + li) * 128 + r]);
          tail_lo = lo + n - (n & 7);
        }
        uint32_t u[8];
        if (tail_lo < lo + n) {
          tmem_ld8(ta + tail_lo, u);
          tmem_wait_ld();
          for (int j = 0; j < lo + n - tail_lo; ++j) res = __fadd_rn(res, __uint_as_float(u[j]));
        }
        return res;
      };
      xch[r] = __fadd_rn(0.0f, pw_tree_eval(S, full_leaf));
    }
    att_bar();
    const float denom = xch[r];
    // denom in [1, S] and e in [0, 1]: the hoisted-reciprocal quotient is exact (numerics.cuh)
    const Recip rden = make_recip(denom), rsm = make_recip(F16 ? 1.0f : p.s_softmax);
    // pass 3: P = e / sum (quantized or f16) into the 128B-swizzled K-major A operand
    uint8_t* prow = smem + lay.p_off + r * 128;
    const bool row_live = q0 + r < S;
    float amx_sm = 0.0f;
    for (int ch = 0; ch < nchunks; ++ch) {
      if (ch > 0) mbar_wait(bar_pf, (ch - 1) & 1);    // previous round consumed the buffer
      const int k_lo = ch * ATT_P_CHUNK, k_hi = min(nkp, k_lo + ATT_P_CHUNK);
      for (int c0 = k_lo + 32 * h; c0 < k_hi; c0 += 64) {
        uint32_t v[32];
        tmem_ld32(ta + c0, v);
        tmem_wait_ld();
        uint32_t w[16];
        if constexpr (F16) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float a = (c0 + j) < S ? div_fast(__uint_as_float(v[j]), rden) : 0.0f;
            const float b = (c0 + j + 1) < S ? div_fast(__uint_as_float(v[j + 1]), rden) : 0.0f;
            if (row_live) amx_sm = fmaxf(amx_sm, fmaxf(a, b));
            __half2 hv = __floats2half2_rn(a, b);
            w[j / 2] = *reinterpret_cast<uint32_t*>(&hv);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              q[u] = (c0 + j + u) < S ? quant_pre_bounded(div_fast(__uint_as_float(v[j + u]), rden), rsm) : 0.0f;
            w[j / 4] = trunc_pack4_s8(q[0], q[1], q[2], q[3]);
          }
        }
        // 32 keys = 32 (int8) or 64 (f16) bytes: 2 or 4 swizzled 16-byte chunks
        const int local = c0 - k_lo;
        uint8_t* base = prow + (local / C::KEYS_PER_PBLK) * 16384;
        const int chunk0 = ((local % C::KEYS_PER_PBLK) * C::P_ELT) >> 4;
#pragma unroll
        for (int u = 0; u < 2 * C::P_ELT; ++u)
          *reinterpret_cast<uint4*>(base + (((chunk0 + u) ^ (r & 7)) << 4)) =
              make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar_p);
    }

    // context rows of this sequence: h writes output columns [32h, 32h+32)
    mbar_wait(bar_pf, (nchunks - 1) & 1);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld32(ta + 32 * h, o);
    tmem_wait_ld();
    const Recip rctx = make_recip(F16 ? 1.0f : p.s_ctx);
    float amx_ctx = 0.0f;
    if (q0 + r < S) {
      if constexpr (F16) {
        __half* dst = static_cast<__half*>(p.ctx_out) + size_t(row0 + q0 + r) * p.hidden + head * 64 + 32 * h;
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          __half2 hv = __floats2half2_rn(__uint_as_float(o[j]), __uint_as_float(o[j + 1]));
          w[j / 2] = *reinterpret_cast<uint32_t*>(&hv);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int u = 0; u < 4; ++u) d4[u] = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
        if (p.amax) {
#pragma unroll
          for (int j = 0; j < 32; ++j) amx_ctx = fmaxf(amx_ctx, fabsf(__uint_as_float(o[j])));
        }
      } else {
        int8_t* dst = static_cast<int8_t*>(p.ctx_out) + size_t(row0 + q0 + r) * p.hidden + head * 64 + 32 * h;
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = quant_pre_bounded(__fmul_rn(__int2float_rn(int(o[j + u])), p.mult_ctx), rctx);
          w[j / 4] = trunc_pack4_s8(q[0], q[1], q[2], q[3]);
        }
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    if (F16 && p.amax) {
      amax_commit(p.amax + p.site_sm, amx_sm);
      amax_commit(p.amax + p.site_ctx, amx_ctx);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
}

}  // namespace samp
