// Padding-free (varlen) multi-head attention, INT8 (kind::i8) or FP16 (kind::f16)
// operands.  One CTA per (tile, head); a tile is either 128 queries of one sequence, or
// several whole sequences of equal length S in {32, 64} packed block-diagonally (2 or 4
// sequences share the 128 MMA rows; keys of the other sequences get P = 0 exactly, so
// P.V over the packed keys equals each sequence's own product).
//
// INT8 semantics (reference pkg/src/samp/encoder.py:368-379, kernels.py:130-135):
//   scores = F32(Q_q . K_q^T) * F32(s_q*s_k/sqrt(d)) + mask      mask = -10000 for keys >= att_len
//   probs  = softmax_rows(scores)   (row max, numpy exp, numpy pairwise sum, IEEE divide)
//   P_q    = quantize(probs, s_softmax)
//   ctx_q  = quantize(F32(P_q . V_q) * F32(s_softmax*s_v), s_out_in)
// FP semantics (encoder.py:298-305): scores = (Q.K^T)*F32(1/sqrt(d)) + mask, same softmax,
//   ctx = P . V, with Q/K/V/P/ctx held in f16 (the reference's fp16-storage points).
// Rows and keys of a sequence are its full (possibly padded) length S, so each sequence
// sees exactly the reference's per-sequence arithmetic.
//
// Data path: TMA loads Q [128 x d], K and V [keys x d] straight out of the fused QKV
// activation [T][3H].  tcgen05.mma #1: S_acc[128 x keys] = Q K^T into TMEM.  Eight
// softmax warps, two threads per query row (h = 0/1 take alternate 32-key chunks):
//   pass 1  row max from the integer (INT8) / f32 (FP16) accumulators: x = RN(acc*m) is
//           monotone in acc, so max/min of acc over the unmasked and the masked keys give
//           the exact row max of x with one IMNMX per key;
//   pass 2  e = numpy exp(x - max) -> TMEM.  When the row's exp arguments provably lie in
//           [-86.5, 0] (checked per row from the pass-1 extremes; masked keys underflow to
//           0) the exp runs on FFMA2 pairs with an exact exponent add instead of numpy's
//           two-step scalef; otherwise the general scalar restatement runs;
//   sum     numpy's pairwise tree over the row's S values of e (TMEM reads in order);
//           S <= 128 is one leaf (h = 0), longer rows split at numpy's top-level split;
//   pass 3  P = e / sum (quantized or f16) into the 128B-swizzled K-major A operand.
// tcgen05.mma #2: O_acc[128 x 64] = P V, V consumed MN-major straight from its TMA image.
// P is produced in chunks of up to 256 keys so the f16 path fits S = 512 in smem.
#pragma once
#include <climits>
#include <type_traits>

#include <cuda_fp16.h>

#include "gemm.cuh"   // phase-stamp helpers (globaltimer, smid, GEMM_STAMPS)
#include "numerics.cuh"
#include "sm100.cuh"

namespace samp {

// warp 0: TMA + MMA + TMEM owner; warps 1..4*TPR: softmax, TPR threads per query row
// (TPR = 2 by default, 4 selectable: see attention.cu).
template <int TPR> constexpr int att_threads() { return 32 + 128 * TPR; }
constexpr int ATT_MAX_LEAVES = 8;  // numpy tree leaves for S <= 512
constexpr int ATT_MAX_KEYS = 512;
constexpr int ATT_P_CHUNK = 256;   // keys of P written per MMA-2 round

struct AttnParams {
  void* ctx_out;              // [T][H] int8 codes (INT8) or f16 values (FP16)
  const int* tile_seq;        // [ntiles] first sequence of each tile
  const int* tile_q0;         // [ntiles] first query (within the sequence); 0 for packed tiles
  const int* tile_cnt;        // [ntiles] sequences in the tile (> 1: equal S in {32, 64})
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
  X2 k = x2_consts();         // opaque FFMA2 constants (numerics.cuh)
  unsigned long long* stamps = nullptr;   // measurement only: 8 %globaltimer stamps per CTA
  unsigned long long* hist = nullptr;     // INT8 code-usage tap: [256] counts of the P codes
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
  int q_off, k_off, v_off, p_off, x_off, bar_off, hist_off, total;
  __host__ __device__ AttnLayout(int keys_cap) {
    using C = AttnCfg<F16>;
    const int kv = ((keys_cap + 63) / 64) * 64 * C::ROW_BYTES;
    const int pchunk = keys_cap < ATT_P_CHUNK ? ((keys_cap + 127) / 128) * 128 : ATT_P_CHUNK;
    q_off = 0;
    k_off = q_off + 128 * C::ROW_BYTES;
    v_off = k_off + kv;
    p_off = ((v_off + kv + 1023) / 1024) * 1024;
    x_off = p_off + 128 * pchunk * C::P_ELT;
    bar_off = x_off + (3 * 4 + ATT_MAX_LEAVES + 1) * 128 * 4;   // extremes [3][4][128], leaf sums, denom
    hist_off = bar_off + 64;                                    // [256] u32 code-usage bins
    total = hist_off + 1024 + 1024;
  }
};

// named barrier among the 128*TPR softmax threads
template <int TPR>
__device__ __forceinline__ void att_bar() { asm volatile("bar.sync 1, %0;" :: "n"(128 * TPR) : "memory"); }

constexpr float ATT_EXP_FAST_MIN = NP_EXP2_FAST_MIN;   // x - max >= this: np_exp2_fast is exact
constexpr float ATT_EXP_LO_CUT = -103.97208404541015625f;
constexpr float ATT_MASK = -10000.0f;

// accumulator -> float (INT8: I2FP on the ALU pipe, which has slack next to the FFMA2 chain)
template <bool F16>
__device__ __forceinline__ float2 acc_pair(uint32_t a, uint32_t b, const X2&) {
  if constexpr (F16) return f2(__uint_as_float(a), __uint_as_float(b));
  else return f2(__int2float_rn(int(a)), __int2float_rn(int(b)));
}

// numpy leaf (n <= 128) over e values in TMEM columns [col, col + n) of this thread's
// lane: 8 strided accumulators over the body, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the
// n % 8 tail sequentially; n < 8: 0 + sequential.  col is a multiple of 8 and uniform
// across the warp (tcgen05.ld is warp-collective).
__device__ __forceinline__ float att_leaf(uint32_t ta, int col, int n, const X2& k) {
  const int body = n - (n & 7);
  float res = 0.0f;
  if (body > 0) {
    float2 r[4];
    for (int g = 0; g < body; g += 32) {
      uint32_t u[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (g + 8 * i < body) tmem_ld8(ta + col + g + 8 * i, u[i]);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (g + 8 * i < body) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 v = f2(__uint_as_float(u[i][2 * j]), __uint_as_float(u[i][2 * j + 1]));
            r[j] = (g + i == 0) ? v : add2(r[j], v, k);
          }
        }
      }
    }
    res = __fadd_rn(__fadd_rn(__fadd_rn(r[0].x, r[0].y), __fadd_rn(r[1].x, r[1].y)),
                    __fadd_rn(__fadd_rn(r[2].x, r[2].y), __fadd_rn(r[3].x, r[3].y)));
  }
  if (n & 7) {
    uint32_t u[8];
    tmem_ld8(ta + col + body, u);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 7; ++j)
      if (j < (n & 7)) res = __fadd_rn(res, __uint_as_float(u[j]));
  }
  return res;
}

// Per-thread view of one attention tile for the softmax warps (two or four threads per
// query row; thread h of row r).  Shared by attention_kernel and the fused QKV+attention
// kernel (qkv_attention.cuh), so both run the same bit-exact arithmetic.
struct AttRow {
  int h, r;             // thread index within the row, query row within the tile
  int S, nk, nkp;       // sequence length, keys of the tile, keys padded to 32
  int nchunks;          // P chunks (MMA-2 rounds)
  int kbeg, att;        // this row's first key (packed tiles) and attention length
  bool live;            // the row is a real query
};

// the same row geometry from already-loaded sequence values (S = sequence length, att = the
// attention length of this row's sequence): arithmetic only
__device__ __forceinline__ AttRow att_row_of(int S, int att, int cnt, int r, int h) {
  AttRow w;
  w.h = h;
  w.r = r;
  w.S = S;
  w.nk = cnt * S;
  w.nkp = (w.nk + 31) & ~31;
  w.nchunks = (w.nkp + ATT_P_CHUNK - 1) / ATT_P_CHUNK;
  const int sub = cnt > 1 ? min(r / S, cnt - 1) : 0;
  w.kbeg = sub * S;
  w.att = att;
  w.live = cnt > 1 ? r < w.nk : r < S;
  return w;
}
// packed-tile row index of query row r (which sequence of the tile's cnt it belongs to)
__device__ __forceinline__ int att_sub(int S, int cnt, int r) { return cnt > 1 ? min(r / S, cnt - 1) : 0; }

template <int TPR>
__device__ __forceinline__ AttRow att_row(const AttnParams& p, int seq, int q0, int cnt, int r, int h) {
  AttRow w;
  w.h = h;
  w.r = r;
  const int krow0 = p.seq_start[seq];
  w.S = p.seq_start[seq + 1] - krow0;                 // every sequence of a packed tile has this length
  w.nk = cnt * w.S;
  w.nkp = (w.nk + 31) & ~31;                          // padded to the MMA K step (32 covers both kinds)
  w.nchunks = (w.nkp + ATT_P_CHUNK - 1) / ATT_P_CHUNK;
  // packed tiles hold whole sequences of S rows (S % 32 == 0, so a warp's 32 rows never
  // straddle two sequences: kbeg is warp-uniform)
  const int sub = cnt > 1 ? min(r / w.S, cnt - 1) : 0;
  w.kbeg = sub * w.S;
  w.att = p.att_len[seq + sub];
  w.live = cnt > 1 ? r < w.nk : q0 + r < w.S;
  return w;
}

// Softmax of the tile's score rows (TMEM, this thread's lane quarter at `ta`, column = key)
// into the 128B-swizzled K-major P operand at `pbuf`, chunk by chunk: before chunk ch > 0
// waits `bar_pf` phase (ch-1)&1 (MMA-2 consumed the buffer), after each chunk arrives on
// `bar_p`.  `xbuf` = [3][4][128] pass-1 extremes, [ATT_MAX_LEAVES][128] leaf sums, [128]
// denominators.  Barrier 1 (128*TPR threads) synchronises the softmax threads.  Returns
// the thread's max |P| (FP16 calibration).
template <bool F16, int TPR, bool HIST>
__device__ __forceinline__ float att_softmax(const AttnParams& p, const AttRow& w, uint32_t ta, uint8_t* pbuf,
                                             uint8_t* xbuf, unsigned int* hist_s, uint64_t* bar_p,
                                             uint64_t* bar_pf, unsigned long long* stamp) {
  using C = AttnCfg<F16>;
  const X2 kx = p.k;
  const int h = w.h, r = w.r, S = w.S, att = w.att, kbeg = w.kbeg, nkp = w.nkp;
  int* ixch = reinterpret_cast<int*>(xbuf);                                   // [3][4][128] pass-1 extremes
  float* leafs = reinterpret_cast<float*>(xbuf) + 3 * 4 * 128;                // [ATT_MAX_LEAVES][128]
  float* dsum = leafs + ATT_MAX_LEAVES * 128;                                 // [128] row denominators
  const int nrow = (S + 31) & ~31;                   // this row's key chunks: [kbeg, kbeg + nrow)
  const float m = p.mult_scores;

  // ---- pass 1: extremes of the accumulators over unmasked [0, att) and masked [att, S)
  // (INT8: int32 order == order of x = RN(F32(acc)*m), m > 0; FP16: f32 order likewise)
  using Acc = typename std::conditional<F16, float, int>::type;
  auto as_acc = [](uint32_t u) -> Acc {
    if constexpr (F16) return __uint_as_float(u); else return int(u);
  };
  Acc lowest, highest;
  if constexpr (F16) { lowest = -INFINITY; highest = INFINITY; } else { lowest = INT_MIN; highest = INT_MAX; }
  Acc umax = lowest, umin = highest, mmax = lowest;
  for (int c0 = 32 * h; c0 < nrow; c0 += 32 * TPR) {
    uint32_t v[32];
    tmem_ld32(ta + kbeg + c0, v);
    tmem_wait_ld();
    if (c0 + 32 <= att) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        umax = max(umax, as_acc(v[j]));
        umin = min(umin, as_acc(v[j]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int key = c0 + j;
        const Acc a = as_acc(v[j]);
        if (key < att) { umax = max(umax, a); umin = min(umin, a); }
        else if (key < S) mmax = max(mmax, a);
      }
    }
  }
  {
    Acc* ex = reinterpret_cast<Acc*>(ixch);
    ex[(0 * 4 + h) * 128 + r] = umax;
    ex[(1 * 4 + h) * 128 + r] = umin;
    ex[(2 * 4 + h) * 128 + r] = mmax;
    att_bar<TPR>();
#pragma unroll
    for (int q = 0; q < TPR; ++q) {
      umax = max(umax, ex[(0 * 4 + q) * 128 + r]);
      umin = min(umin, ex[(1 * 4 + q) * 128 + r]);
      mmax = max(mmax, ex[(2 * 4 + q) * 128 + r]);
    }
  }
  auto xval = [&](Acc a) -> float {
    if constexpr (F16) return __fmul_rn(a, m); else return __fmul_rn(__int2float_rn(a), m);
  };
  const bool has_u = att > 0, has_m = att < S;
  const float xm = has_m ? __fadd_rn(xval(mmax), ATT_MASK) : -INFINITY;
  const float mx = has_u ? fmaxf(xval(umax), xm) : xm;
  // fast exp for this row: every unmasked argument in [-86.5, 0], every masked one <= lo_cut
  const bool fast_row = !w.live || ((!has_u || __fsub_rn(xval(umin), mx) >= ATT_EXP_FAST_MIN) &&
                                    (!has_m || __fsub_rn(xm, mx) <= ATT_EXP_LO_CUT));
  const bool fast = __all_sync(0xffffffffu, fast_row);
  if (stamp) stamp[3] = globaltimer();
  const float2 negmx = f2(-mx, -mx), mm = f2(m, m);

  // ---- pass 2: e = exp(x - max) -> TMEM (0 past S).  The warp-uniform fast / exact choice
  // is made once, outside the chunk loop, so the fast loop body stays compact
#ifdef SAMP_ATT_PASS2_INLINE   // measurement: the round-2 form (choice inside the loop)
  for (int c0 = 32 * h; c0 < nrow; c0 += 32 * TPR) {
    uint32_t v[32];
    tmem_ld32(ta + kbeg + c0, v);
    tmem_wait_ld();
    if (fast) {
      const bool clean = c0 + 32 <= att;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 x = mul2(acc_pair<F16>(v[j], v[j + 1], kx), mm, kx);
        const float2 e = np_exp2_fast(add2(x, negmx, kx), kx);
        v[j] = __float_as_uint(clean || c0 + j < att ? e.x : 0.0f);
        v[j + 1] = __float_as_uint(clean || c0 + j + 1 < att ? e.y : 0.0f);
      }
    } else {
      // fully unrolled: a runtime index would put v[] in local memory for both paths
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int key = c0 + j;
        float x = xval(as_acc(v[j]));
        if (key >= att) x = __fadd_rn(x, ATT_MASK);
        v[j] = __float_as_uint(key < S ? np_expf_nonpos(__fsub_rn(x, mx)) : 0.0f);
      }
    }
    tmem_st32(ta + kbeg + c0, v);
  }
#else
  if (fast) {
    for (int c0 = 32 * h; c0 < nrow; c0 += 32 * TPR) {
      uint32_t v[32];
      tmem_ld32(ta + kbeg + c0, v);
      tmem_wait_ld();
#ifndef SAMP_ATT_CLEAN_SELECT
      if (c0 + 32 <= att) {   // every key of the chunk unmasked: no per-key select
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = mul2(acc_pair<F16>(v[j], v[j + 1], kx), mm, kx);
          const float2 e = np_exp2_fast(add2(x, negmx, kx), kx);
          v[j] = __float_as_uint(e.x);
          v[j + 1] = __float_as_uint(e.y);
        }
      } else
#endif
      {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = mul2(acc_pair<F16>(v[j], v[j + 1], kx), mm, kx);
          const float2 e = np_exp2_fast(add2(x, negmx, kx), kx);
          v[j] = __float_as_uint(c0 + j < att ? e.x : 0.0f);
          v[j + 1] = __float_as_uint(c0 + j + 1 < att ? e.y : 0.0f);
        }
      }
      tmem_st32(ta + kbeg + c0, v);
    }
  } else {
    for (int c0 = 32 * h; c0 < nrow; c0 += 32 * TPR) {
      uint32_t v[32];
      tmem_ld32(ta + kbeg + c0, v);
      tmem_wait_ld();
      // fully unrolled: a runtime index would put v[] in local memory
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int key = c0 + j;
        float x = xval(as_acc(v[j]));
        if (key >= att) x = __fadd_rn(x, ATT_MASK);
        v[j] = __float_as_uint(key < S ? np_expf_nonpos(__fsub_rn(x, mx)) : 0.0f);
      }
      tmem_st32(ta + kbeg + c0, v);
    }
  }
#endif
  tmem_wait_st();
  tc_fence_before();
  att_bar<TPR>();                               // every e of the row is in TMEM
  tc_fence_after();
  if (stamp) stamp[4] = globaltimer();

  // ---- numpy pairwise sum over the row's S values (np.sum = 0 + tree): the tree's
  // leaves (key order, <= 128 keys each) are summed from TMEM by thread h = leaf % TPR,
  // then thread 0 combines them up the tree
  if (S <= 128) {
    if (h == 0) dsum[r] = __fadd_rn(0.0f, att_leaf(ta, kbeg, S, kx));
  } else {                                      // single-sequence tile, kbeg = 0
    auto own = [&](int lo, int ln, int li) {
      if (li % TPR == h) leafs[li * 128 + r] = att_leaf(ta, lo, ln, kx);
      return 0.0f;
    };
    pw_tree_eval(S, own);
    att_bar<TPR>();
    if (h == 0) {
      auto read = [&](int, int, int li) { return leafs[li * 128 + r]; };
      dsum[r] = __fadd_rn(0.0f, pw_tree_eval(S, read));
    }
  }
  att_bar<TPR>();
  const float denom = dsum[r];
  if (stamp) stamp[5] = globaltimer();
  // denom in [1, S] and e in [0, 1]: the hoisted-reciprocal quotient is exact (numerics.cuh)
  const Recip rden = make_recip(denom), rsm = make_recip(F16 ? 1.0f : p.s_softmax);

  // ---- pass 3: P = e / sum (quantized or f16) into the 128B-swizzled K-major A operand
  uint8_t* prow = pbuf + r * 128;
  auto pstore = [&](int local, const uint32_t (&wv)[16]) {   // 32 keys at chunk-local column `local`
    uint8_t* base = prow + (local / C::KEYS_PER_PBLK) * 16384;
    const int chunk0 = ((local % C::KEYS_PER_PBLK) * C::P_ELT) >> 4;
#pragma unroll
    for (int u = 0; u < 2 * C::P_ELT; ++u)
      *reinterpret_cast<uint4*>(base + (((chunk0 + u) ^ (r & 7)) << 4)) =
          make_uint4(wv[4 * u], wv[4 * u + 1], wv[4 * u + 2], wv[4 * u + 3]);
  };
  float amx_sm = 0.0f;
  unsigned int zeros = 0;   // code-usage tap: zero codes counted in registers
  const float2 rden_r = f2(rden.r, rden.r), rden_ns = f2(-rden.s, -rden.s);
  const float2 rsm_r = f2(rsm.r, rsm.r), rsm_ns = f2(-rsm.s, -rsm.s);
  auto div_pair = [&](float2 x, float2 rr, float2 ns) {       // div_fast on a pair
    const float2 q = __ffma2_rn(x, rr, f2(kx.pzero, kx.pzero));
    return __ffma2_rn(rr, __ffma2_rn(ns, q, x), q);
  };
  for (int ch = 0; ch < w.nchunks; ++ch) {
    if (ch > 0) mbar_wait(bar_pf, (ch - 1) & 1);    // previous round consumed the buffer
    const int k_lo = ch * ATT_P_CHUNK, k_hi = min(nkp, k_lo + ATT_P_CHUNK);
    for (int c0 = k_lo + 32 * h; c0 < k_hi; c0 += 32 * TPR) {
      uint32_t wv[16] = {};
      const int key0 = c0 - kbeg;                   // sequence-local key of the chunk
      if (key0 >= 0 && key0 < nrow) {               // warp-uniform: the row's own keys
        uint32_t v[32];
        tmem_ld32(ta + c0, v);
        tmem_wait_ld();
        if constexpr (F16) {
#ifndef SAMP_ATT_F16_P3_SELECT
          if (key0 + 32 <= S && !p.amax) {   // all keys in the sequence, no calibration tap
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float2 pv = div_pair(f2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])), rden_r, rden_ns);
              __half2 hv = __floats2half2_rn(pv.x, pv.y);
              wv[j / 2] = *reinterpret_cast<uint32_t*>(&hv);
            }
          } else
#endif
          {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float2 pv = div_pair(f2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])), rden_r, rden_ns);
              const float a = key0 + j < S ? pv.x : 0.0f;
              const float b = key0 + j + 1 < S ? pv.y : 0.0f;
              if (w.live) amx_sm = fmaxf(amx_sm, fmaxf(a, b));
              __half2 hv = __floats2half2_rn(a, b);
              wv[j / 2] = *reinterpret_cast<uint32_t*>(&hv);
            }
          }
        } else {
          // probabilities are >= +0, so quantize's copysign(0.5, y) is +0.5.  Keys past S
          // hold e = +0 (pass 2), so their P = +0 / sum = +0 and t = 0.5 truncates to code
          // 0: no per-key select is needed
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float2 q[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float2 pv = div_pair(f2(__uint_as_float(v[j + 2 * u]), __uint_as_float(v[j + 2 * u + 1])),
                                         rden_r, rden_ns);
              q[u] = add2(div_pair(pv, rsm_r, rsm_ns), f2(0.5f, 0.5f), kx);
            }
            wv[j / 4] = trunc_pack4_s8(q[0].x, q[0].y, q[1].x, q[1].y);
            if (HIST && w.live) {   // code-usage tap over the row's S keys (masked ones included)
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int c = int(int8_t(wv[j / 4] >> (8 * b)));
                if (key0 + j + b >= S) continue;
                if (c == 0) ++zeros;
                else atomicAdd(&hist_s[c + 128], 1u);
              }
            }
          }
        }
      }
      pstore(c0 - k_lo, wv);                        // other sequences' keys: P = 0
    }
    fence_proxy_async_smem();
    tc_fence_before();
    mbar_arrive(bar_p);
  }
  if (HIST && zeros) atomicAdd(&hist_s[128], zeros);
  if (stamp) stamp[6] = globaltimer();
  return amx_sm;
}

// numpy leaf tail: res + e[8G] + ... + e[8G + n - 1] sequentially (n < 8) over a thread's
// register chunks v[CPT][32]; G is a template parameter so every register index is constant
template <int G, int CPT>
__device__ __forceinline__ float att_tail_g(float res, int n, const uint32_t (&v)[CPT][32]) {
  if constexpr (8 * G < 32 * CPT) {
#pragma unroll
    for (int t = 0; t < 7; ++t)
      if (t < n) res = __fadd_rn(res, __uint_as_float(v[(8 * G + t) >> 5][(8 * G + t) & 31]));
  }
  return res;
}
template <int CPT>
__device__ __forceinline__ float att_tail(float res, int start, int n, const uint32_t (&v)[CPT][32]) {
  switch (start >> 3) {
    case 0: return att_tail_g<0>(res, n, v);
    case 1: return att_tail_g<1>(res, n, v);
    case 2: return att_tail_g<2>(res, n, v);
    case 3: return att_tail_g<3>(res, n, v);
    case 4: return att_tail_g<4>(res, n, v);
    case 5: return att_tail_g<5>(res, n, v);
    case 6: return att_tail_g<6>(res, n, v);
    default: return att_tail_g<7>(res, n, v);
  }
}

// pass 1 of att_softmax_rr on one register chunk (sequence-local keys k0 .. k0+31)
__device__ __forceinline__ void att_extremes32(const uint32_t (&vc)[32], int k0, int att, int S, int& umax, int& umin,
                                               int& mmax) {
  if (k0 + 32 <= att) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      umax = max(umax, int(vc[j]));
      umin = min(umin, int(vc[j]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int a = int(vc[j]);
      if (k0 + j < att) { umax = max(umax, a); umin = min(umin, a); }
      else if (k0 + j < S) mmax = max(mmax, a);
    }
  }
}

// 32 P codes of a register chunk -> the row's 128B-swizzled P operand at tile column `local`
// (keys >= 128 live in the next 16 KB block of 128-key rows)
__device__ __forceinline__ void att_p_store32(uint8_t* prow, int local, int r, const uint32_t (&wv)[8]) {
  prow += (local >> 7) * 16384;
  const int chunk0 = (local & 127) >> 4;
  *reinterpret_cast<uint4*>(prow + ((chunk0 ^ (r & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  *reinterpret_cast<uint4*>(prow + (((chunk0 + 1) ^ (r & 7)) << 4)) = make_uint4(wv[4], wv[5], wv[6], wv[7]);
}

// pass 3 of att_softmax_rr: P = quantize(e / sum, s_softmax) for one register chunk
__device__ __forceinline__ void att_codes32(const uint32_t (&vc)[32], uint8_t* prow, int local, int r,
                                            const Recip& rden, const Recip& rsm, const X2& kx) {
  const float2 rden_r = f2(rden.r, rden.r), rden_ns = f2(-rden.s, -rden.s);
  const float2 rsm_r = f2(rsm.r, rsm.r), rsm_ns = f2(-rsm.s, -rsm.s);
  uint32_t wv[8];
#pragma unroll
  for (int j = 0; j < 32; j += 4) {
    float2 q[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float2 x = f2(__uint_as_float(vc[j + 2 * u]), __uint_as_float(vc[j + 2 * u + 1]));
      const float2 q1 = __ffma2_rn(x, rden_r, f2(kx.pzero, kx.pzero));
      const float2 pv = __ffma2_rn(rden_r, __ffma2_rn(rden_ns, q1, x), q1);
      const float2 q2 = __ffma2_rn(pv, rsm_r, f2(kx.pzero, kx.pzero));
      q[u] = add2(__ffma2_rn(rsm_r, __ffma2_rn(rsm_ns, q2, pv), q2), f2(0.5f, 0.5f), kx);
    }
    wv[j / 4] = trunc_pack4_s8(q[0].x, q[0].y, q[1].x, q[1].y);
  }
  att_p_store32(prow, local, r, wv);
}

// pass 2 of att_softmax_rr on one 32-key chunk held in registers (sequence-local keys
// k0 .. k0+31), fast rows: e = numpy exp(x - max) by np_exp2_fast, 0 past att
__device__ __forceinline__ void att_expo32_fast(uint32_t (&vc)[32], int k0, int att, float m, float mx, const X2& kx) {
  const float2 negmx = f2(-mx, -mx), mm = f2(m, m);
#ifndef SAMP_ATT_CLEAN_SELECT
  if (k0 + 32 <= att) {   // every key unmasked: no per-key select (as attention pass 2)
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float2 x = mul2(acc_pair<false>(vc[j], vc[j + 1], kx), mm, kx);
      const float2 e = np_exp2_fast(add2(x, negmx, kx), kx);
      vc[j] = __float_as_uint(e.x);
      vc[j + 1] = __float_as_uint(e.y);
    }
    return;
  }
#endif
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const float2 x = mul2(acc_pair<false>(vc[j], vc[j + 1], kx), mm, kx);
    const float2 e = np_exp2_fast(add2(x, negmx, kx), kx);
    vc[j] = __float_as_uint(k0 + j < att ? e.x : 0.0f);
    vc[j + 1] = __float_as_uint(k0 + j + 1 < att ? e.y : 0.0f);
  }
}

// pass 2 for rows outside the fast domain (rare): the general scalar numpy exp, 8 keys at a
// time straight from the scores still in TMEM (a rolled loop keeps the kernel's code small),
// written back to TMEM and reloaded into the chunk's registers
__device__ __forceinline__ void att_expo32_exact(uint32_t (&vc)[32], uint32_t taddr, int k0, int att, int S, float m,
                                                 float mx) {
#pragma unroll 1
  for (int g = 0; g < 4; ++g) {
    uint32_t u[8];
    tmem_ld8(taddr + 8 * g, u);
    tmem_wait_ld();
#pragma unroll 1   // rare path: one inlined copy of the scalar exp
    for (int t = 0; t < 8; ++t) {
      const int key = k0 + 8 * g + t;
      float x = __fmul_rn(__int2float_rn(int(u[t])), m);
      if (key >= att) x = __fadd_rn(x, ATT_MASK);
      u[t] = __float_as_uint(key < S ? np_expf_nonpos(__fsub_rn(x, mx)) : 0.0f);
    }
    tmem_st8(taddr + 8 * g, u);
  }
  tmem_wait_st();
  tmem_ld32(taddr, vc);
  tmem_wait_ld();
}

// Register-resident softmax for INT8 tiles whose keys fit one P chunk (S <= 128), used by
// the fused QKV+attention kernel (which has the registers).  Thread h of a row owns the
// row's 32-key chunks [h*CPT, h*CPT + CPT) (CPT = 4 / TPR).  The scores are read from TMEM
// once; the exp values stay in registers through the sum and pass 3.  numpy's leaf over the
// row (8 strided accumulators over the body, tree, sequential tail; S <= 128 is one leaf) is
// evaluated as ONE chain handed from thread to thread through shared memory in TPR
// barrier-separated rounds, so every add happens in numpy's order and the denominator (and
// every P code) equals att_softmax's bit for bit.
// MAXCH: 32-key chunks per row the caller's tiles can have (4: S <= 128, 8: S <= 256).
template <int TPR, int MAXCH = 4>
__device__ __forceinline__ void att_softmax_rr(const AttnParams& p, const AttRow& w, uint32_t ta, uint8_t* pbuf,
                                               uint8_t* xbuf, uint64_t* bar_p, unsigned long long* stamp) {
  constexpr int CPT = MAXCH / TPR;
  static_assert(CPT * 32 <= 64, "the leaf tail switch covers 64 register values per thread");
  const X2 kx = p.k;
  const int h = w.h, r = w.r, S = w.S, att = w.att, kbeg = w.kbeg;
  const int nch = (S + 31) >> 5;               // the row's key chunks (1..MAXCH)
  const int c_lo = h * CPT;
  const int cnt = max(0, min(CPT, nch - c_lo)); // my chunks, warp-uniform
  const int lo = 32 * c_lo;                    // sequence-local key of my first value
  const int hi = min(32 * (c_lo + cnt), S);    // end of my keys within the sequence
  int* ixch = reinterpret_cast<int*>(xbuf);                          // [3][4][128] extremes
  float* xr = reinterpret_cast<float*>(xbuf) + 3 * 4 * 128;          // [8][128] chain hand-off
  float* dsum = xr + ATT_MAX_LEAVES * 128;                           // [128] denominators
  const float m = p.mult_scores;

  uint32_t v[CPT][32];   // my chunks; indexed by constants only (register-resident)
#pragma unroll
  for (int c = 0; c < CPT; ++c)
    if (c < cnt) tmem_ld32(ta + kbeg + lo + 32 * c, v[c]);
  tmem_wait_ld();

  // ---- pass 1: integer extremes over unmasked [0, att) and masked [att, S) keys
  int umax = INT_MIN, umin = INT_MAX, mmax = INT_MIN;
#pragma unroll
  for (int c = 0; c < CPT; ++c)
    if (c < cnt) att_extremes32(v[c], lo + 32 * c, att, S, umax, umin, mmax);
  ixch[(0 * 4 + h) * 128 + r] = umax;
  ixch[(1 * 4 + h) * 128 + r] = umin;
  ixch[(2 * 4 + h) * 128 + r] = mmax;
  att_bar<TPR>();
#pragma unroll
  for (int q = 0; q < TPR; ++q) {
    umax = max(umax, ixch[(0 * 4 + q) * 128 + r]);
    umin = min(umin, ixch[(1 * 4 + q) * 128 + r]);
    mmax = max(mmax, ixch[(2 * 4 + q) * 128 + r]);
  }
  auto xval = [&](int a) { return __fmul_rn(__int2float_rn(a), m); };
  const bool has_u = att > 0, has_m = att < S;
  const float xm = has_m ? __fadd_rn(xval(mmax), ATT_MASK) : -INFINITY;
  const float mx = has_u ? fmaxf(xval(umax), xm) : xm;
  const bool fast_row = !w.live || ((!has_u || __fsub_rn(xval(umin), mx) >= ATT_EXP_FAST_MIN) &&
                                    (!has_m || __fsub_rn(xm, mx) <= ATT_EXP_LO_CUT));
  const bool fast = __all_sync(0xffffffffu, fast_row);
  if (stamp) stamp[3] = globaltimer();

  // ---- pass 2: e = exp(x - max) in registers (0 for keys past att when fast / past S)
#pragma unroll
  for (int c = 0; c < CPT; ++c)
    if (c < cnt) {
      if (fast) att_expo32_fast(v[c], lo + 32 * c, att, m, mx, kx);
      else att_expo32_exact(v[c], ta + kbeg + lo + 32 * c, lo + 32 * c, att, S, m, mx);
    }
  if (stamp) stamp[4] = globaltimer();

  // ---- numpy leaf over the row's S values as one chain, round q run by thread h = q:
  // the thread whose keys hold body groups continues the 8 strided accumulators (thread 0
  // starts them); the one holding the body's end combines them (tree) and adds the tail,
  // handing a partial result on when the tail starts in the next thread's keys
  const int body = S & ~7;
  float rr[8];
#pragma unroll
  for (int q = 0; q < TPR; ++q) {
    if (h == q && cnt > 0) {
      if (lo < body) {
        if (lo == 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) rr[k] = __uint_as_float(v[0][k]);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) rr[k] = xr[k * 128 + r];
        }
#pragma unroll
        for (int g = 0; g < 4 * CPT; ++g) {
          const int key = lo + 8 * g;
          if ((lo > 0 || g > 0) && key < body && key < hi) {
#pragma unroll
            for (int k = 0; k < 8; ++k) rr[k] = __fadd_rn(rr[k], __uint_as_float(v[(8 * g + k) >> 5][(8 * g + k) & 31]));
          }
        }
        if (body <= 32 * (c_lo + cnt)) {   // the body ends in my keys
          const float t = __fadd_rn(__fadd_rn(__fadd_rn(rr[0], rr[1]), __fadd_rn(rr[2], rr[3])),
                                    __fadd_rn(__fadd_rn(rr[4], rr[5]), __fadd_rn(rr[6], rr[7])));
          const float res = att_tail<CPT>(t, body - lo, min(S, hi) - body, v);
          if (S <= hi) dsum[r] = __fadd_rn(0.0f, res);
          else xr[r] = res;                  // the tail continues in the next thread's keys
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) xr[k * 128 + r] = rr[k];
        }
      } else if (lo < S) {                   // tail only (body ended at or before lo)
        const float start = body == 0 ? 0.0f : xr[r];   // S < 8: numpy's 0 + sequential
        dsum[r] = __fadd_rn(0.0f, att_tail<CPT>(start, 0, S - lo, v));
      }
    }
    att_bar<TPR>();
  }
  const float denom = dsum[r];
  if (stamp) stamp[5] = globaltimer();
  const Recip rden = make_recip(denom), rsm = make_recip(p.s_softmax);

  // ---- pass 3: P codes from the registers into the 128B-swizzled K-major A operand
  uint8_t* prow = pbuf + r * 128;
#pragma unroll
  for (int c = 0; c < CPT; ++c)
    if (c < cnt) att_codes32(v[c], prow, kbeg + lo + 32 * c, r, rden, rsm, kx);
  // keys of the tile outside this row's sequence (packed tiles): P = 0, chunk tc by thread tc % TPR
  const int tch = w.nkp >> 5, own0 = kbeg >> 5;
#pragma unroll
  for (int tc = 0; tc < MAXCH; ++tc)
    if (tc < tch && (tc < own0 || tc >= own0 + nch) && tc % TPR == h) {
      const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      att_p_store32(prow, 32 * tc, r, z);
    }
  fence_proxy_async_smem();
  tc_fence_before();
  mbar_arrive(bar_p);
  if (stamp) stamp[6] = globaltimer();
}

// Context rows: O (TMEM at `to`, this thread's lane quarter, 64 columns) -> ctx codes
// (INT8, quantize at attn.out_in) or f16 values; thread h writes columns [OC*h, OC*h + OC).
template <bool F16, int TPR>
__device__ __forceinline__ void att_ctx_out(const AttnParams& p, const AttRow& w, uint32_t to, size_t orow, int head,
                                            float amx_sm) {
  constexpr int OC = 64 / TPR;
  const int h = w.h;
  uint32_t o[OC];
  if constexpr (OC == 32) tmem_ld32(to + OC * h, o);
  else tmem_ld16(to + OC * h, o);
  tmem_wait_ld();
  const Recip rctx = make_recip(F16 ? 1.0f : p.s_ctx);
  float amx_ctx = 0.0f;
  if (w.live) {
    if constexpr (F16) {
      __half* dst = static_cast<__half*>(p.ctx_out) + orow * p.hidden + head * 64 + OC * h;
      uint32_t wv[OC / 2];
#pragma unroll
      for (int j = 0; j < OC; j += 2) {
        __half2 hv = __floats2half2_rn(__uint_as_float(o[j]), __uint_as_float(o[j + 1]));
        wv[j / 2] = *reinterpret_cast<uint32_t*>(&hv);
      }
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int u = 0; u < OC / 8; ++u) d4[u] = make_uint4(wv[4 * u], wv[4 * u + 1], wv[4 * u + 2], wv[4 * u + 3]);
      if (p.amax) {
#pragma unroll
        for (int j = 0; j < OC; ++j) amx_ctx = fmaxf(amx_ctx, fabsf(__uint_as_float(o[j])));
      }
    } else {
      int8_t* dst = static_cast<int8_t*>(p.ctx_out) + orow * p.hidden + head * 64 + OC * h;
      uint32_t wv[OC / 4];
#pragma unroll
      for (int j = 0; j < OC; j += 4) {
        float q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = quant_pre_bounded(__fmul_rn(__int2float_rn(int(o[j + u])), p.mult_ctx), rctx);
        wv[j / 4] = trunc_pack4_s8(q[0], q[1], q[2], q[3]);
      }
#pragma unroll
      for (int u = 0; u < OC / 16; ++u)
        reinterpret_cast<uint4*>(dst)[u] = make_uint4(wv[4 * u], wv[4 * u + 1], wv[4 * u + 2], wv[4 * u + 3]);
    }
  }
  if (F16 && p.amax) {
    amax_commit(p.amax + p.site_sm, amx_sm);
    amax_commit(p.amax + p.site_ctx, amx_ctx);
  }
}

template <bool F16, int TPR, bool HIST = false>   // HIST: code-usage tap (p.hist) compiled in
__global__ void __launch_bounds__(att_threads<TPR>(), TPR == 2 ? 3 : 2)
attention_kernel(const __grid_constant__ CUtensorMap map_qkv, const AttnParams p, int keys_cap) {
  using C = AttnCfg<F16>;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array keeps the shared address space visible
  // to the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const AttnLayout<F16> lay(keys_cap);
  uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* bar_s = bar_load + 1;       // MMA-1 done
  uint64_t* bar_p = bar_load + 2;       // P chunk written (256 arrivals per phase)
  uint64_t* bar_pf = bar_load + 3;      // MMA-2 round done (P buffer free / O ready)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_load + 4);

  const int tile = blockIdx.x, head = blockIdx.y;
  // phase stamps (tools/gemm_phases.py): smid, start, S in TMEM, pass 1, pass 2, sum, P written, exit
  const int cta_id = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned long long* stamp = p.stamps && cta_id < GEMM_STAMP_CTAS ? p.stamps + size_t(cta_id) * GEMM_STAMPS : nullptr;
  if (stamp && threadIdx.x == 0) {
    stamp[0] = smid();
    stamp[1] = globaltimer();
  }
  const int seq = p.tile_seq[tile];
  const int q0 = p.tile_q0[tile];
  const int cnt = p.tile_cnt[tile];
  const int krow0 = p.seq_start[seq];
  const int S = p.seq_start[seq + 1] - krow0;          // every sequence of a packed tile has this length
  const int nk = cnt * S;                               // keys of the tile
  const int nkp = (nk + 31) & ~31;                      // padded to the MMA K step (32 covers both kinds)
  const int nchunks = (nkp + ATT_P_CHUNK - 1) / ATT_P_CHUNK;
  const uint32_t warp = warp_id();

  if (threadIdx.x == 0) {
    mbar_init(bar_load, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_p, 128 * TPR);
    mbar_init(bar_pf, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, p.tmem_cols);
  unsigned int* hist_s = HIST ? reinterpret_cast<unsigned int*>(smem + lay.hist_off) : nullptr;
  if (hist_s)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist_s[i] = 0;
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
      tma_load_2d(smem + lay.q_off, &map_qkv, head * 64, krow0 + q0, bar_load);
      tma_load_2d(smem + lay.q_off + 64 * C::ROW_BYTES, &map_qkv, head * 64, krow0 + q0 + 64, bar_load);
      for (int b = 0; b < nblk; ++b) {
        tma_load_2d(smem + lay.k_off + b * 64 * C::ROW_BYTES, &map_qkv, H + head * 64, krow0 + b * 64, bar_load);
        tma_load_2d(smem + lay.v_off + b * 64 * C::ROW_BYTES, &map_qkv, 2 * H + head * 64, krow0 + b * 64, bar_load);
      }
      mbar_wait_park(bar_load, 0);
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
        mbar_wait_park(bar_p, ch & 1);   // the softmax passes take microseconds (parked: no issue slots)
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
    const int quarter = warp & 3;
    const int h = int(warp - 1) >> 2;                  // 0 .. TPR-1
    const int r = quarter * 32 + lane_id();            // query row within the tile
    const uint32_t ta = tmem + (uint32_t(quarter * 32) << 16);
    const AttRow w = att_row<TPR>(p, seq, q0, cnt, r, h);
    mbar_wait_park(bar_s, 0);             // Q/K/V loads + MMA 1 (after the PDL wait)
    tc_fence_after();
    const bool stamper = stamp && threadIdx.x == 32;
    if (stamper) stamp[2] = globaltimer();
    const float amx_sm = att_softmax<F16, TPR, HIST>(p, w, ta, smem + lay.p_off, smem + lay.x_off, hist_s, bar_p,
                                                     bar_pf, stamper ? stamp : nullptr);
    mbar_wait_park(bar_pf, (nchunks - 1) & 1);
    tc_fence_after();
    att_ctx_out<F16, TPR>(p, w, ta, size_t(krow0 + q0 + r), head, amx_sm);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
  if (hist_s)
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (hist_s[i]) atomicAdd(&p.hist[i], (unsigned long long)hist_s[i]);
  if (stamp && threadIdx.x == 0) stamp[7] = globaltimer();
}

}  // namespace samp
