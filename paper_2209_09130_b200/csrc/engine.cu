#include <cstdio>
// The samp_b200 engine: device weights, calibration scales, activation buffers and
// the per-layer mixed-precision forward (reference Engine, pkg/src/samp/encoder.py:421-530).
//
// Per-layer kernel sequence (5 launches per layer + embed + head):
//   FULL_INT8  QKV i8 GEMM [dequant+bias+quantize q|k|v] -> attention i8 ->
//              out-proj i8 GEMM [dequant+bias+residual+LN+quantize ffn.in] ->
//              FFN1 i8 GEMM [dequant+bias+GELU+quantize ffn.mid] ->
//              FFN2 i8 GEMM [dequant+bias+residual+LN (+quantize next attn.in | f32)]
//   FFN_ONLY   QKV f16 GEMM -> attention f16 -> out-proj f16 GEMM [+LN+quantize ffn.in] ->
//              FFN1 i8 -> FFN2 i8
//   FP         f16 GEMMs/attention, LN epilogues in F32 (f16 storage)
//   MHA_ONLY   (extension) INT8 attention block, FP16 FFN on dequantized ffn.in codes
// No standalone quantize / dequantize / LayerNorm kernel exists: every one is fused.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "host_util.h"
#include "kernels.h"

namespace samp {

// ------------------------------------------------------------------ helpers
static double site_scale(double amax) { return std::max(amax, 127 * 1e-8) / 127.0; }
static float f32(double x) { return static_cast<float>(x); }
static float mult_of(double a, double b) { return static_cast<float>(a * b); }

static double host_amax(const float* w, size_t n) {
  float m = 0.0f;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(w[i]));
  return double(m);
}

struct DevMem {
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    SAMP_CUDA(cudaMalloc(&p, count * sizeof(T)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~DevMem() {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

struct LayerDev {
  bool loaded = false;
  int8_t *qkv_i8 = nullptr, *wo_i8 = nullptr, *w1_i8 = nullptr, *w2_i8 = nullptr;    // K-major
  __half *qkv_f16 = nullptr, *wo_f16 = nullptr, *w1_f16 = nullptr, *w2_f16 = nullptr;
  float *qkv_b = nullptr, *ob = nullptr, *ln1_g = nullptr, *ln1_b = nullptr;
  float *qkv32 = nullptr, *wo32 = nullptr, *w132 = nullptr, *w232 = nullptr;   // exact FP32: (in, out)
  float *b1 = nullptr, *b2 = nullptr, *ln2_g = nullptr, *ln2_b = nullptr;
  double s_w[6] = {0, 0, 0, 0, 0, 0};  // qw kw vw ow w1 w2
  double b1_absmax = 0;                 // max|b1|: bounds the FFN1 GELU argument
  bool ln1_bounded = false, ln2_bounded = false;   // |LN output| < 1e18 proved (EpiResLN noclamp)
  CUtensorMap m_qkv_i8, m_wo_i8, m_w2_i8, m_qkv_f16, m_wo_f16, m_w2_f16;
  CUtensorMap m_wo_i8_64, m_w2_i8_64;    // 64-row boxes: split-K GEMMs for small batches
  CUtensorMap m_wo_i8_s, m_w2_i8_s, m_wo_f16_s, m_w2_f16_s;   // bn_ln_small-row boxes
  CUtensorMap m_qkv_i8_128, m_qkv_i8_64;   // persistent QKV tile widths
  CUtensorMap m_qkv_f16_64;                // small-batch f16 QKV
  CUtensorMap m_w1_i8[3], m_w1_f16[3];   // FFN1 B operand, box rows FFN1_BN[k]
};

static int pick_bn(int n) {
  for (int bn : {256, 128, 64})
    if (n % bn == 0) return bn;
  return 0;
}

// FFN1 runs persistent (walking tiles); its makespan is the per-CTA tile count times the
// tile width, so the width is picked per launch from these (costed per SM: with two INT8
// CTAs per SM the SM-level balance is what matters; measured 96-wide at 4096 tokens)
constexpr int FFN1_BN[3] = {64, 96, 128};
static int ffn1_bn_index(int T, int I, int slots, bool allow96 = true) {
  const int sms = slots;
  if (const char* f = std::getenv("SAMP_FFN1_BN")) {   // measurement override
    for (int k = 0; k < 3; ++k)
      if (FFN1_BN[k] == std::atoi(f) && I % FFN1_BN[k] == 0) return k;
  }
  const int mt = (T + GEMM_BM - 1) / GEMM_BM;
  int best = -1;
  long best_cost = 0;
  for (int k = 0; k < 3; ++k) {
    if (I % FFN1_BN[k] || (!allow96 && FFN1_BN[k] == 96)) continue;
    const long tiles = long(mt) * (I / FFN1_BN[k]);
    const long cost = (tiles + sms - 1) / sms * FFN1_BN[k];
    if (best < 0 || cost <= best_cost) best = k, best_cost = cost;   // ties: wider tile
  }
  return best;
}

static Tiles choose_tiles(int H, int I) {
  Tiles t{};
  t.bn_qkv = pick_bn(H);
  // FFN1 (N = I = 4H): 128-wide tiles give 2.6 waves of 2 CTAs/SM at 4096 tokens instead of
  // 1.3 waves of 256-wide ones (less tail), at the same MMA efficiency
  t.bn_ffn1 = I % 128 == 0 ? 128 : pick_bn(I);
  const int cand[][2] = {{192, 4}, {256, 4}, {256, 2}, {192, 2}, {256, 1}, {128, 1}, {64, 1}};
  for (auto& c : cand)
    if (c[0] * c[1] == H && pw_splits_evenly(H, c[1])) {
      t.bn_ln = c[0];
      t.cluster_ln = c[1];
      break;
    }
  // one numpy leaf per CTA: H = 8 leaves of 96 (768) or 128 (1024)
  t.bn_ln_small = (pw_splits_evenly(H, 8) && (H / 8 == 96 || H / 8 == 128)) ? H / 8 : 0;
  return t;
}

// ------------------------------------------------------------------ engine
struct Activations {
  int cap = 0;  // token rows
  float *hid_f32 = nullptr, *ln1_f32 = nullptr;
  __half *hid_f16 = nullptr, *qkv_f16 = nullptr, *ctx_f16 = nullptr, *ln1_f16 = nullptr, *mid_f16 = nullptr;
  int8_t *xq[2] = {nullptr, nullptr}, *qkv_i8 = nullptr, *ctx_i8 = nullptr, *ffn_in_i8 = nullptr, *mid_i8 = nullptr;
  int *ids = nullptr, *segs = nullptr, *pos = nullptr;
  float *logits = nullptr, *probs = nullptr, *pooled = nullptr;
  int* idseg = nullptr;       // [2][cap]: per forward ids = idseg, segs = idseg + T (one H2D)
  int* ws = nullptr;          // [cap][H] int32 split-K accumulators (zero between uses)
  float* headbuf = nullptr;   // per forward logits [rows][L] | probs [rows][L] | labels [rows] (one D2H)
  int* labels = nullptr;
  // A-operand tensor maps (box 128 B x 128 rows) and attention maps (box one head row x 64 rows)
  CUtensorMap a_xq[2], a_ctx_i8, a_ffn_in, a_mid_i8, a_hid_f16, a_ctx_f16, a_ln1_f16, a_mid_f16;
  CUtensorMap a_ctx_i8_mc[2], a_mid_i8_mc[2];   // 32- / 16-row boxes (A multicast in 4- / 8-CTA clusters)
  CUtensorMap att_qkv_i8, att_qkv_f16;
  // LN-GEMM outputs stored by TMA (one box of bn_ln columns x 128 rows, no swizzle)
  CUtensorMap st_ffn_in, st_xq[2];
  CUtensorMap st_small_ffn_in, st_small_xq[2];   // small batches: box bn_ln_small x 128
  // small-batch FP LN outputs by TMA (box 32 x 128; f32 128B swizzle, f16 64B swizzle)
  CUtensorMap st_ln1_f32, st_ln1_f16, st_hid_f32, st_hid_f16;
};

struct Geometry {
  std::vector<int> seq_start, att_len, tile_seq, tile_q0, tile_cnt;
  std::vector<int> rt;   // per 128-row tile m: the attention tiles [rt[2m], rt[2m+1]] holding its rows
  int nseq = 0, T = 0, ntiles = 0, max_nkp = 0, max_s = 0;
  int *d_seq_start = nullptr, *d_att_len = nullptr, *d_tile_seq = nullptr, *d_tile_q0 = nullptr, *d_tile_cnt = nullptr;
  int* d_tile_done = nullptr;   // [cap_tiles] fused-kernel (tile, head) counters (row-tile flags)
  int* d_rt = nullptr;          // [2 * cap_rt]
  int cap_seq = 0, cap_tiles = 0, cap_rt = 0;
};

}  // namespace samp

struct samp_engine {
  // every entry point that reads or writes engine state holds this (samp_b200.h threading
  // contract); recursive because samp_calibrate / samp_code_usage call samp_forward
  std::recursive_mutex mu;
  samp_model_desc d{};
  int device = 0;
  cudaStream_t stream = nullptr;          // the engine's own stream
  cudaStream_t stream_in_use = nullptr;   // stream of the current samp_forward
  samp::Tiles tiles{};
  samp::DevMem mem;
  // embeddings + heads (F32)
  float *word = nullptr, *position = nullptr, *token_type = nullptr, *emb_g = nullptr, *emb_b = nullptr;
  float *pool_w = nullptr, *pool_b = nullptr, *head_wt = nullptr, *head_b = nullptr;
  bool emb_loaded = false, heads_loaded = false;
  std::vector<samp::LayerDev> layers;
  std::map<std::string, double> amax;
  samp::Activations act;
  samp::Geometry geo;
  int launches = 0;
  // row-tile flags between the fused QKV+attention kernel and the out-projection (per forward)
  bool dep_on = false;
  int dep_count = 0;   // fused layers enqueued so far: the counters' target is dep_count * heads
  bool capture = false;
  bool stamp_only = false;   // samp_set_profiling(2): phase stamps without per-launch events
  std::map<std::string, std::vector<uint8_t>> stages;
  std::vector<int> h_pos;
  bool profiling = false;
  int sms = 148;                  // SM count of the engine's device
  cudaStream_t side = nullptr;    // L2 weight prefetch runs here, forked from the forward's stream
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // GEMM phase stamps (profiling mode): [stamp_cap launches][STAMP_CTAS][GEMM_STAMPS]
  unsigned long long* stamps = nullptr;
  int stamp_cap = 0;
  std::vector<std::pair<std::string, int>> stamp_launches;   // (name, CTAs) per GEMM launch
  float* calib_amax = nullptr;    // non-null while samp_calibrate runs: per-site amax taps
  unsigned long long* usage = nullptr;   // non-null while samp_code_usage runs: [1+8L][256] bins
  struct GraphEntry {
    cudaGraphExec_t exec;
    int launches;
  };
  bool graphs_enabled = true;
  std::map<std::string, GraphEntry> graphs;   // (plan, geometry, head) -> captured forward
  // ffn.mid scale (bits) -> GELU_FAST admitted (exhaustive check, gelu_fast_check)
  std::map<uint32_t, bool> gelu_fast_ok;
  std::set<std::string> seen;
  struct Pending { std::string name; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, std::pair<double, long>> prof;  // name -> (total ms, launches)
  // exact FP32 layers (samp_set_exact_fp32): FP blocks on the k-ordered FP32 SIMT path
  bool exact = false;
  int exact_cap = 0;
  float *x_qkv = nullptr, *x_ctx = nullptr, *x_proj = nullptr, *x_mid = nullptr;
  // capture_taps (samp_set_capture(e, 2)): F32 site values, recorded as stages "tap:<site>"
  bool taps = false;
  int tap_cap = 0;                 // token rows of the tap scratch buffers
  void* tap_acc = nullptr;         // [cap][max(3H, I)] int32 / f32 accumulators
  float *tap_out = nullptr, *tap_ctx = nullptr, *tap_ln = nullptr, *tap_probs = nullptr;
  size_t tap_probs_cap = 0;
  long long* tap_prob_off = nullptr;
  int tap_prob_off_cap = 0;
  size_t tap_probs_total = 0;      // floats of this forward's softmax tap
  int* pinned_ids = nullptr;   // staging for host inputs
  int pinned_cap = 0;
  float* pinned_out = nullptr;  // staging for the head outputs (one D2H)
  size_t pinned_out_cap = 0;
};

namespace samp {

using GraphEntry = samp_engine::GraphEntry;

// captured graphs bake buffer pointers, tensor maps and scales: drop them whenever any changes
static void clear_graphs(samp_engine* e) {
  for (auto& kv : e->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  e->graphs.clear();
  e->seen.clear();
}

static void ensure_activations(samp_engine* e, int T) {
  Activations& a = e->act;
  if (T <= a.cap) return;
  clear_graphs(e);
  int cap = std::max(T, 256);
  cap = (cap + 127) / 128 * 128;
  const int H = e->d.hidden, I = e->d.intermediate, L = std::max(1, e->d.num_labels);
  auto drop = [&](void* p) {
    if (p) e->mem.release(p);
  };
  drop(a.hid_f32); drop(a.ln1_f32); drop(a.hid_f16); drop(a.qkv_f16); drop(a.ctx_f16); drop(a.ln1_f16);
  drop(a.mid_f16); drop(a.xq[0]); drop(a.xq[1]); drop(a.qkv_i8); drop(a.ctx_i8); drop(a.ffn_in_i8);
  drop(a.mid_i8); drop(a.idseg); drop(a.pos); drop(a.headbuf); drop(a.pooled); drop(a.ws);
  a.hid_f32 = e->mem.alloc<float>(size_t(cap) * H);
  a.ln1_f32 = e->mem.alloc<float>(size_t(cap) * H);
  a.hid_f16 = e->mem.alloc<__half>(size_t(cap) * H);
  a.qkv_f16 = e->mem.alloc<__half>(size_t(cap) * 3 * H);
  a.ctx_f16 = e->mem.alloc<__half>(size_t(cap) * H);
  a.ln1_f16 = e->mem.alloc<__half>(size_t(cap) * H);
  a.mid_f16 = e->mem.alloc<__half>(size_t(cap) * I);
  a.xq[0] = e->mem.alloc<int8_t>(size_t(cap) * H);
  a.xq[1] = e->mem.alloc<int8_t>(size_t(cap) * H);
  a.qkv_i8 = e->mem.alloc<int8_t>(size_t(cap) * 3 * H);
  a.ctx_i8 = e->mem.alloc<int8_t>(size_t(cap) * H);
  a.ffn_in_i8 = e->mem.alloc<int8_t>(size_t(cap) * H);
  a.mid_i8 = e->mem.alloc<int8_t>(size_t(cap) * I);
  a.idseg = e->mem.alloc<int>(2 * size_t(cap));
  a.ws = e->mem.alloc<int>(size_t(cap) * H);
  SAMP_CUDA(cudaMemset(a.ws, 0, size_t(cap) * H * sizeof(int)));
  a.pos = e->mem.alloc<int>(cap);
  a.headbuf = e->mem.alloc<float>(size_t(cap) * (2 * L + 1));
  a.pooled = e->mem.alloc<float>(size_t(POOL_KSPLIT) * cap * H);
  a.cap = cap;
  // GEMM A operands: K-major rows, 128-byte boxes, 128 rows
  a.a_xq[0] = tmap_i8(a.xq[0], cap, H, H, 128, 128);
  a.a_xq[1] = tmap_i8(a.xq[1], cap, H, H, 128, 128);
  a.a_ctx_i8 = tmap_i8(a.ctx_i8, cap, H, H, 128, 128);
  a.a_ffn_in = tmap_i8(a.ffn_in_i8, cap, H, H, 128, 128);
  a.a_mid_i8 = tmap_i8(a.mid_i8, cap, I, I, 128, 128);
  for (int k = 0; k < 2; ++k) {
    a.a_ctx_i8_mc[k] = tmap_i8(a.ctx_i8, cap, H, H, 128, k ? 16 : 32);
    a.a_mid_i8_mc[k] = tmap_i8(a.mid_i8, cap, I, I, 128, k ? 16 : 32);
  }
  a.a_hid_f16 = tmap_f16(a.hid_f16, cap, H, H, 64, 128);
  a.a_ctx_f16 = tmap_f16(a.ctx_f16, cap, H, H, 64, 128);
  a.a_ln1_f16 = tmap_f16(a.ln1_f16, cap, H, H, 64, 128);
  a.a_mid_f16 = tmap_f16(a.mid_f16, cap, I, I, 64, 128);
  // attention: one head row (64 int8 / 64 f16) x 64 rows
  a.att_qkv_i8 = tmap_i8(a.qkv_i8, cap, 3 * H, 3 * H, 64, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  a.att_qkv_f16 = tmap_f16(a.qkv_f16, cap, 3 * H, 3 * H, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e->tiles.bn_ln && e->tiles.bn_ln <= 256) {
    a.st_ffn_in = tmap_i8(a.ffn_in_i8, cap, H, H, e->tiles.bn_ln, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
    a.st_xq[0] = tmap_i8(a.xq[0], cap, H, H, e->tiles.bn_ln, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
    a.st_xq[1] = tmap_i8(a.xq[1], cap, H, H, e->tiles.bn_ln, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  if (e->tiles.bn_ln_small && e->tiles.bn_ln_small <= 256) {
    const uint32_t bs = e->tiles.bn_ln_small;
    a.st_small_ffn_in = tmap_i8(a.ffn_in_i8, cap, H, H, bs, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
    a.st_small_xq[0] = tmap_i8(a.xq[0], cap, H, H, bs, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
    a.st_small_xq[1] = tmap_i8(a.xq[1], cap, H, H, bs, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  a.st_ln1_f32 = make_tmap_2d(a.ln1_f32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cap, H, size_t(H) * 4, 32, 128,
                              CU_TENSOR_MAP_SWIZZLE_128B);
  a.st_hid_f32 = make_tmap_2d(a.hid_f32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cap, H, size_t(H) * 4, 32, 128,
                              CU_TENSOR_MAP_SWIZZLE_128B);
  a.st_ln1_f16 = tmap_f16(a.ln1_f16, cap, H, H, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
  a.st_hid_f16 = tmap_f16(a.hid_f16, cap, H, H, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
}

static void set_geometry(samp_engine* e, int nseq, const int32_t* seq_start, const int32_t* att_len) {
  Geometry& g = e->geo;
  const bool same = g.nseq == nseq && std::equal(seq_start, seq_start + nseq + 1, g.seq_start.begin()) &&
                    std::equal(att_len, att_len + nseq, g.att_len.begin());
  if (same && g.nseq > 0) return;
  g.nseq = nseq;
  g.seq_start.assign(seq_start, seq_start + nseq + 1);
  g.att_len.resize(nseq);
  g.tile_seq.clear();
  g.tile_q0.clear();
  g.max_nkp = 0;
  e->h_pos.resize(seq_start[nseq]);
  g.tile_cnt.clear();
  g.max_s = 0;
  for (int s = 0; s < nseq; ++s) {
    const int S = seq_start[s + 1] - seq_start[s];
    g.max_s = std::max(g.max_s, S);
    g.att_len[s] = std::min(att_len[s], S);
    for (int t = 0; t < S; ++t) e->h_pos[seq_start[s] + t] = t;
  }
  // attention tiles: 128 queries of one sequence, or up to 128/S consecutive sequences of
  // equal length S in {32, 64} packed block-diagonally into one tile (attention.cuh)
  for (int s = 0; s < nseq;) {
    const int S = seq_start[s + 1] - seq_start[s];
    int cnt = 1;
    if (S == 32 || S == 64) {
      while (cnt < 128 / S && s + cnt < nseq && seq_start[s + cnt + 1] - seq_start[s + cnt] == S) ++cnt;
    }
    if (cnt > 1) {
      g.tile_seq.push_back(s);
      g.tile_q0.push_back(0);
      g.tile_cnt.push_back(cnt);
    } else {
      for (int q = 0; q < S; q += 128) {
        g.tile_seq.push_back(s);
        g.tile_q0.push_back(q);
        g.tile_cnt.push_back(1);
      }
    }
    g.max_nkp = std::max(g.max_nkp, (cnt * S + 31) & ~31);
    s += cnt;
  }
  g.T = seq_start[nseq];
  g.ntiles = int(g.tile_seq.size());
  // row tiles -> attention tiles (tiles are in row order; a tile holds whole sequences, or
  // 128 query rows of one)
  const int mt = (g.T + GEMM_BM - 1) / GEMM_BM;
  g.rt.assign(2 * std::max(mt, 1), 0);
  for (int m = 0, t = 0; m < mt; ++m) {
    const int r0 = m * GEMM_BM, r1 = std::min(g.T, r0 + GEMM_BM);
    auto tile_rows = [&](int k, int& a, int& b) {
      const int sq = g.tile_seq[k], S = seq_start[sq + 1] - seq_start[sq];
      a = seq_start[sq] + g.tile_q0[k];
      b = g.tile_cnt[k] > 1 ? seq_start[sq + g.tile_cnt[k]] : a + std::min(128, S - g.tile_q0[k]);
    };
    int a0, b0;
    tile_rows(t, a0, b0);
    while (b0 <= r0) tile_rows(++t, a0, b0);
    int hi = t, ah, bh;
    while (hi + 1 < g.ntiles && (tile_rows(hi + 1, ah, bh), ah < r1)) ++hi;
    g.rt[2 * m] = t;
    g.rt[2 * m + 1] = hi;
  }
  // captured graphs bake these device pointers into kernel arguments: a reallocation
  // invalidates every graph
  if (nseq + 1 > g.cap_seq || g.ntiles > g.cap_tiles || mt > g.cap_rt) clear_graphs(e);
  if (mt > g.cap_rt) {
    if (g.d_rt) e->mem.release(g.d_rt);
    g.cap_rt = std::max(mt, 64);
    g.d_rt = e->mem.alloc<int>(2 * g.cap_rt);
  }
  if (nseq + 1 > g.cap_seq) {
    if (g.d_seq_start) { e->mem.release(g.d_seq_start); e->mem.release(g.d_att_len); }
    g.cap_seq = std::max(nseq + 1, 64);
    g.d_seq_start = e->mem.alloc<int>(g.cap_seq);
    g.d_att_len = e->mem.alloc<int>(g.cap_seq);
  }
  if (g.ntiles > g.cap_tiles) {
    if (g.d_tile_seq) {
      e->mem.release(g.d_tile_seq); e->mem.release(g.d_tile_q0); e->mem.release(g.d_tile_cnt);
      e->mem.release(g.d_tile_done);
    }
    g.cap_tiles = std::max(g.ntiles, 64);
    g.d_tile_seq = e->mem.alloc<int>(g.cap_tiles);
    g.d_tile_q0 = e->mem.alloc<int>(g.cap_tiles);
    g.d_tile_cnt = e->mem.alloc<int>(g.cap_tiles);
    g.d_tile_done = e->mem.alloc<int>(g.cap_tiles);
  }
  ensure_activations(e, g.T);
  SAMP_CUDA(cudaMemcpyAsync(g.d_seq_start, g.seq_start.data(), (nseq + 1) * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(g.d_att_len, g.att_len.data(), nseq * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(g.d_tile_seq, g.tile_seq.data(), g.ntiles * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(g.d_tile_q0, g.tile_q0.data(), g.ntiles * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(g.d_tile_cnt, g.tile_cnt.data(), g.ntiles * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(g.d_rt, g.rt.data(), 2 * mt * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaMemcpyAsync(e->act.pos, e->h_pos.data(), g.T * sizeof(int), cudaMemcpyHostToDevice, e->stream_in_use));
  SAMP_CUDA(cudaStreamSynchronize(e->stream_in_use));  // host vectors may change on the next call
}

static double need_amax(samp_engine* e, const std::string& site) {
  auto it = e->amax.find(site);
  SAMP_REQUIRE(it != e->amax.end(), SAMP_E_CALIBRATION, "calibration table is missing site '" + site + "'");
  return it->second;
}
static double sc(samp_engine* e, const std::string& site) { return site_scale(need_amax(e, site)); }
static std::string lsite(int i, const char* blk, const char* name) {
  return "L" + std::to_string(i) + "." + blk + "." + name;
}
static std::string input_site(int i) { return i == 0 ? "embed.out" : lsite(i, "attn", "in"); }

// required sites for a plan, as PrecisionPlan.required_sites (encoder.py:126-136) + MHA-only
static std::set<std::string> required_sites(const uint8_t* prec, int L) {
  std::set<std::string> s;
  for (int i = 0; i < L; ++i) {
    if (prec[i] == SAMP_LAYER_FULL_INT8 || prec[i] == SAMP_LAYER_MHA_INT8) {
      s.insert(input_site(i));
      for (const char* n : {"q", "k", "v", "softmax", "out_in"}) s.insert(lsite(i, "attn", n));
      s.insert(lsite(i, "ffn", "in"));
      if (prec[i] == SAMP_LAYER_FULL_INT8) s.insert(lsite(i, "ffn", "mid"));
    } else if (prec[i] == SAMP_LAYER_FFN_INT8) {
      s.insert(lsite(i, "ffn", "in"));
      s.insert(lsite(i, "ffn", "mid"));
    }
  }
  return s;
}

static void record(samp_engine* e, const std::string& name, int layer, const void* dev, size_t bytes) {
  if (!e->capture) return;
  std::vector<uint8_t> host(bytes);
  SAMP_CUDA(cudaStreamSynchronize(e->stream_in_use));
  SAMP_CUDA(cudaMemcpy(host.data(), dev, bytes, cudaMemcpyDeviceToHost));
  e->stages[name + "@" + std::to_string(layer)] = std::move(host);
}

static void tap_record(samp_engine* e, const std::string& site, const void* dev, size_t bytes) {
  if (e->taps) record(e, "tap:" + site, -1, dev, bytes);
}

// grow the tap scratch buffers for this forward's geometry; per-sequence softmax offsets
static void ensure_taps(samp_engine* e) {
  const Geometry& g = e->geo;
  const int H = e->d.hidden, I = e->d.intermediate, A = e->d.num_heads;
  const int wide = std::max(3 * H, I);
  if (g.T > e->tap_cap) {
    for (void* q : {(void*)e->tap_acc, (void*)e->tap_out, (void*)e->tap_ctx, (void*)e->tap_ln})
      if (q) e->mem.release(q);
    e->tap_cap = std::max(g.T, 128);
    e->tap_acc = e->mem.alloc<int>(size_t(e->tap_cap) * wide);
    e->tap_out = e->mem.alloc<float>(size_t(e->tap_cap) * wide);
    e->tap_ctx = e->mem.alloc<float>(size_t(e->tap_cap) * H);
    e->tap_ln = e->mem.alloc<float>(size_t(e->tap_cap) * H);
  }
  std::vector<long long> off(g.nseq);
  size_t tot = 0;
  for (int s = 0; s < g.nseq; ++s) {
    const long long S = g.seq_start[s + 1] - g.seq_start[s];
    off[s] = (long long)tot;
    tot += size_t(A) * S * S;
  }
  if (tot > e->tap_probs_cap) {
    if (e->tap_probs) e->mem.release(e->tap_probs);
    e->tap_probs_cap = tot;
    e->tap_probs = e->mem.alloc<float>(tot);
  }
  if (g.nseq > e->tap_prob_off_cap) {
    if (e->tap_prob_off) e->mem.release(e->tap_prob_off);
    e->tap_prob_off_cap = g.nseq;
    e->tap_prob_off = e->mem.alloc<long long>(g.nseq);
  }
  e->tap_probs_total = tot;
  SAMP_CUDA(cudaMemcpy(e->tap_prob_off, off.data(), g.nseq * sizeof(long long), cudaMemcpyHostToDevice));
}

static void ensure_exact(samp_engine* e) {
  const int T = e->geo.T, H = e->d.hidden, I = e->d.intermediate;
  if (T <= e->exact_cap) return;
  clear_graphs(e);
  for (void* q : {(void*)e->x_qkv, (void*)e->x_ctx, (void*)e->x_proj, (void*)e->x_mid})
    if (q) e->mem.release(q);
  e->exact_cap = std::max(T, 128);
  e->x_qkv = e->mem.alloc<float>(size_t(e->exact_cap) * 3 * H);
  e->x_ctx = e->mem.alloc<float>(size_t(e->exact_cap) * H);
  e->x_proj = e->mem.alloc<float>(size_t(e->exact_cap) * H);
  e->x_mid = e->mem.alloc<float>(size_t(e->exact_cap) * I);
}

static cudaEvent_t take_event(samp_engine* e) {
  if (e->event_pool.empty()) {
    cudaEvent_t ev;
    SAMP_CUDA(cudaEventCreate(&ev));
    return ev;
  }
  cudaEvent_t ev = e->event_pool.back();
  e->event_pool.pop_back();
  return ev;
}

constexpr int STAMP_CTAS = GEMM_STAMP_CTAS;   // CTAs recorded per stamped GEMM launch

// launch through `fn` (returns cudaError_t); with profiling on, bracket it with CUDA
// events on the engine stream (the stream every kernel is launched on)
template <class F>
static void run_kernel(samp_engine* e, const char* what, F&& fn) {
  // measurement only: SAMP_SKIP=name[,name] drops those launches (results are garbage; the
  // step-time difference is the kernels' share of the pipelined critical path)
  static const std::string skip = std::getenv("SAMP_SKIP") ? "," + std::string(std::getenv("SAMP_SKIP")) + "," : "";
  if (!skip.empty() && skip.find("," + std::string(what) + ",") != std::string::npos) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (e->profiling) {
    a = take_event(e);
    b = take_event(e);
    SAMP_CUDA(cudaEventRecord(a, e->stream_in_use));
  }
  const bool stamped = (e->profiling || e->stamp_only) && e->stamps && int(e->stamp_launches.size()) < e->stamp_cap &&
                       std::strcmp(what, "embed") != 0 &&
                       std::strcmp(what, "head") != 0;
  if (stamped) {
    g_gemm_stamps = e->stamps + size_t(e->stamp_launches.size()) * STAMP_CTAS * GEMM_STAMPS;
    SAMP_CUDA(cudaMemsetAsync(g_gemm_stamps, 0, size_t(STAMP_CTAS) * GEMM_STAMPS * 8, e->stream_in_use));
  }
  cudaError_t err = fn();
  g_gemm_stamps = nullptr;
  if (stamped) e->stamp_launches.push_back({what, 0});
  if (err == cudaSuccess) err = cudaGetLastError();
  SAMP_REQUIRE(err == cudaSuccess, SAMP_E_DEVICE, std::string(what) + ": " + cudaGetErrorString(err));
  if (e->profiling) {
    SAMP_CUDA(cudaEventRecord(b, e->stream_in_use));
    e->pending.push_back({what, a, b});
  }
  e->launches++;
}
#define check_launch(E, CALL, NAME) run_kernel((E), (NAME), [&]() { return (CALL); })

// code-usage tap (analyze-quant): histogram of the int8 codes a stage just wrote at an
// activation site (activation_sites order), when samp_code_usage is running
static void usage_tap(samp_engine* e, int site, const int8_t* src, int rows, int cols, int ld) {
  if (!e->usage) return;
  check_launch(e, launch_code_hist(src, rows, cols, ld, e->usage + size_t(site) * 256, e->stream_in_use), "code_hist");
}

static void launch_attention(samp_engine* e, bool f16, const AttnParams& p) {
  const Geometry& g = e->geo;
  auto stamped = [&]() { AttnParams q = p; q.stamps = g_gemm_stamps; return q; };
  check_launch(e, f16 ? launch_attention_f16(e->act.att_qkv_f16, stamped(), g.ntiles, e->d.num_heads, g.max_nkp, e->stream_in_use)
                      : launch_attention_i8(e->act.att_qkv_i8, stamped(), g.ntiles, e->d.num_heads, g.max_nkp, e->stream_in_use),
               f16 ? "attention_f16" : "attention_i8");
}

static int tmem_cols_for_keys(int nkp) {
  int c = 64;
  while (c < nkp) c *= 2;
  return c;
}

static unsigned long long* g_gelu_flags = nullptr;   // SAMP_GELU_FLAGS measurement counter

static uint32_t bits_of(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
static float gelu_inv_s(float s) { return float(1.0 / double(s)); }

// Admit GELU_FAST for every INT8-FFN layer's ffn.mid scale of this plan (exhaustive device
// check per distinct scale, cached for the engine's lifetime).  SAMP_NO_GELU_FAST=1 keeps
// the exact epilogue everywhere (A/B measurements).
static void gelu_fast_prepare(samp_engine* e, const uint8_t* prec) {
  static const bool off = env_flag("SAMP_NO_GELU_FAST");
  if (off) return;
  for (int i = 0; i < e->d.num_layers; ++i) {
    if (prec[i] != SAMP_LAYER_FULL_INT8 && prec[i] != SAMP_LAYER_FFN_INT8) continue;
    const float s = f32(sc(e, lsite(i, "ffn", "mid")));
    if (e->gelu_fast_ok.count(bits_of(s))) continue;
    unsigned long long counts[2] = {1, 0};
    SAMP_CUDA(gelu_fast_check(s, gelu_inv_s(s), counts, e->stream));
    e->gelu_fast_ok[bits_of(s)] = counts[0] == 0;
  }
}

// Small batches: the out-projection / FFN2 as a split-K GEMM into the int32 workspace
// (64-wide tiles, grid z = ksplit k-block groups) + the row LayerNorm kernel, instead of
// a handful of 4-CTA clusters each streaming the whole K.  Returns false (caller runs the
// fused kernel) unless the launch is the hot int8 chain and the batch is small enough.
// Opt-in (SAMP_SPLITK=1): bit-exact, but the extra row-LayerNorm launch cancels the GEMM
// gain at batch 1 (fully-quant p50 0.595 vs 0.575 ms), so the fused cluster kernel stays
// the default.
static int splitk_factor(int T, int N, int kblocks, int sms) {
  if (!env_flag("SAMP_SPLITK")) return 0;
  const int tiles = ((T + GEMM_BM - 1) / GEMM_BM) * (N / 64);
  int best = 0;
  for (int d = 2; d <= kblocks; ++d)
    if (kblocks % d == 0 && tiles * d <= sms + sms / 4) best = d;
  return best;
}
// the out-projection launch gemm_ln_i8 picks reads its A rows by the row-tile flags (one tile
// per CTA, no A multicast); the persistent and split-K variants wait for the whole grid
static bool outproj_dep_ok(samp_engine* e) {
  const int T = e->geo.T, H = e->d.hidden, mtiles = (T + GEMM_BM - 1) / GEMM_BM;
  if (mtiles >= 256 || env_flag("SAMP_LN_PERSISTENT") || env_flag("SAMP_LN_MCAST")) return false;
  if (ln_rows_supported(H) && H % 64 == 0 && splitk_factor(T, H, H / 128, e->sms) >= 2) return false;
  return true;
}

static bool ln_gemm_splitk(samp_engine* e, const char* name, const CUtensorMap& a_map, const CUtensorMap& b64,
                           int K, const EpiResLN::Params& lp, cudaStream_t st) {
  const int T = e->geo.T, H = e->d.hidden;
  const bool i8_only = lp.res_i8 && !lp.acc_is_f32 && lp.out_i8 && !lp.deq_outputs && !lp.f16_round && !lp.amax && !lp.tap_f32 &&
                       !lp.out_f32 && !lp.out_f16;
  if (!i8_only || !ln_rows_supported(H) || H % 64) return false;
  const int ks = splitk_factor(T, H, K / 128, e->sms);
  if (ks < 2) return false;
  EpiSplitKAdd::Params sp{e->act.ws, H};
  check_launch(e, gemm_splitk_i8(a_map, b64, T, H, K, ks, sp, st), name);
  LnRowsParams rp{e->act.ws, lp.res_i8, lp.res_scale, lp.bias, lp.gamma, lp.beta, lp.mult, lp.eps, T,
                  lp.out_i8, lp.s_out};
  check_launch(e, launch_ln_rows(rp, H, st), "ln_rows");
  return true;
}

// capture_taps: q/k/v (per-block dequant + bias) from the QKV accumulators
static void taps_qkv(samp_engine* e, int i, bool f16, const CUtensorMap& a_map, const LayerDev& w, float m0,
                     float m1, float m2, int f16_round) {
  const int T = e->geo.T, H = e->d.hidden;
  cudaStream_t st = e->stream_in_use;
  check_launch(e, gemm_store_acc(f16 ? KIND_F16 : KIND_I8, e->tiles.bn_qkv, a_map, f16 ? w.m_qkv_f16 : w.m_qkv_i8,
                                 T, 3 * H, f16 ? 2 * H : H, e->tap_acc, 3 * H, st), "tap_gemm");
  TapBiasParams tb{e->tap_acc, int(f16), 3 * H, T, 3 * H, w.qkv_b, m0, m1, m2, H, 0, f16_round, e->tap_out};
  check_launch(e, launch_tap_bias(tb, st), "tap_bias");
  const char* nm[3] = {"q", "k", "v"};
  for (int k = 0; k < 3; ++k) tap_record(e, lsite(i, "attn", nm[k]), e->tap_out + size_t(k) * T * H, size_t(T) * H * 4);
}

// capture_taps: softmax probabilities and the context before its quantize
static void taps_attention(samp_engine* e, int i, bool f16, const AttnParams& ap, int f16_round) {
  const Geometry& g = e->geo;
  const int H = e->d.hidden;
  TapAttnParams ta{};
  ta.qkv = f16 ? static_cast<const void*>(e->act.qkv_f16) : static_cast<const void*>(e->act.qkv_i8);
  ta.f16 = f16;
  ta.hidden = H;
  ta.seq_start = g.d_seq_start;
  ta.att_len = g.d_att_len;
  ta.mult_scores = ap.mult_scores;
  ta.s_softmax = ap.s_softmax;
  ta.mult_ctx = ap.mult_ctx;
  ta.f16_round = f16_round;
  ta.probs = e->tap_probs;
  ta.prob_off = e->tap_prob_off;
  ta.ctx = e->tap_ctx;
  check_launch(e, launch_tap_attention(ta, g.max_s, e->d.num_heads, g.nseq, e->stream_in_use), "tap_attention");
  tap_record(e, lsite(i, "attn", "softmax"), e->tap_probs, e->tap_probs_total * 4);
  tap_record(e, lsite(i, "attn", "out_in"), e->tap_ctx, size_t(g.T) * H * 4);
}

// capture_taps: ffn.mid = GELU(dequant(acc) + b1) (int8) or GELU(acc + b1) (f16 path)
static void taps_ffn_mid(samp_engine* e, int i, bool f16, const CUtensorMap& a_map, const LayerDev& w, float mult,
                         int f16_round) {
  const int T = e->geo.T, H = e->d.hidden, I = e->d.intermediate;
  const int k1 = I % 128 == 0 ? 2 : 0;   // FFN1_BN[k1] = 128 or 64
  check_launch(e, gemm_store_acc(f16 ? KIND_F16 : KIND_I8, FFN1_BN[k1], a_map, f16 ? w.m_w1_f16[k1] : w.m_w1_i8[k1],
                                 T, I, f16 ? 2 * H : H, e->tap_acc, I, e->stream_in_use), "tap_gemm");
  TapBiasParams tb{e->tap_acc, int(f16), I, T, I, w.b1, mult, mult, mult, 0, 1, f16_round, e->tap_out};
  check_launch(e, launch_tap_bias(tb, e->stream_in_use), "tap_bias");
  tap_record(e, lsite(i, "ffn", "mid"), e->tap_out, size_t(T) * I * 4);
}

// capture_taps of q/k/v out of an interleaved [T][3H] f32 buffer
static void tap_qkv_f32(samp_engine* e, int i, const float* qkv) {
  if (!e->taps) return;
  const int T = e->geo.T, H = e->d.hidden;
  const char* nm[3] = {"q", "k", "v"};
  for (int k = 0; k < 3; ++k) {
    SAMP_CUDA(cudaMemcpy2DAsync(e->tap_out, size_t(H) * 4, qkv + size_t(k) * H, size_t(3) * H * 4, size_t(H) * 4, T,
                                cudaMemcpyDeviceToDevice, e->stream_in_use));
    tap_record(e, lsite(i, "attn", nm[k]), e->tap_out, size_t(T) * H * 4);
  }
}

// Exact FP32 MHA block (reference mha_fp, encoder.py:276-312): hid_f32 -> ln1_f32 (and the
// ffn.in codes when the FFN runs INT8).  rnd: fp16-storage rounding of this block's stored
// values (FP layers only; FFN_ONLY's MHA runs unrounded, encoder.py:495-497).
static void exact_mha(samp_engine* e, int i, const LayerDev& w, int rnd, bool int8_ffn) {
  const int T = e->geo.T, H = e->d.hidden;
  const Geometry& g = e->geo;
  Activations& a = e->act;
  cudaStream_t st = e->stream_in_use;
  float* cal = e->calib_amax;
  const int cbase = 1 + 8 * i;
  ExactGemmParams q{a.hid_f32, H, w.qkv32, 3 * H, T, 3 * H, H, w.qkv_b, 0, rnd, e->x_qkv, 3 * H, cal, cbase + 1, H};
  check_launch(e, launch_exact_gemm(q, e->sms, st), "qkv_f32");
  tap_qkv_f32(e, i, e->x_qkv);
  ExactAttnParams ap{e->x_qkv, H, g.d_seq_start, g.d_att_len, f32(1.0 / std::sqrt(double(H / e->d.num_heads))), rnd,
                     e->x_ctx, e->taps ? e->tap_probs : nullptr, e->tap_prob_off, cal, cbase + 4, cbase + 5};
  check_launch(e, launch_exact_attention(ap, g.max_s, e->d.num_heads, g.nseq, st), "attention_f32");
  tap_record(e, lsite(i, "attn", "softmax"), e->tap_probs, e->tap_probs_total * 4);
  tap_record(e, lsite(i, "attn", "out_in"), e->x_ctx, size_t(T) * H * 4);
  ExactGemmParams o{e->x_ctx, H, w.wo32, H, T, H, H, nullptr, 0, 0, e->x_proj, H, nullptr, 0, 0};
  check_launch(e, launch_exact_gemm(o, e->sms, st), "outproj_f32");
  ExactLnParams ln{e->x_proj, w.ob, a.hid_f32, w.ln1_g, w.ln1_b, f32(e->d.layernorm_eps), T, rnd, a.ln1_f32,
                   nullptr, 0.0f, cal, cbase + 6};
  if (int8_ffn) {   // x_q = quantize(mha_out, ffn.in) (encoder.py:497-499)
    ln.out_i8 = a.ffn_in_i8;
    ln.s_out = f32(sc(e, lsite(i, "ffn", "in")));
  }
  check_launch(e, launch_exact_ln(ln, H, st), "ln1_f32");
  tap_record(e, lsite(i, "ffn", "in"), a.ln1_f32, size_t(T) * H * 4);
}

// Exact FP32 FFN block (reference ffn_fp, encoder.py:315-330) on ln1_f32 (FP layers: the MHA
// output; MHA-only layers: dequantized ffn.in codes); the output is quantized for a next
// INT8-attention layer or stays F32 in hid_f32.
static void exact_ffn(samp_engine* e, int i, const LayerDev& w, int rnd, bool next_int8, int8_t* next_q) {
  const int T = e->geo.T, H = e->d.hidden, I = e->d.intermediate, L = e->d.num_layers;
  Activations& a = e->act;
  cudaStream_t st = e->stream_in_use;
  float* cal = e->calib_amax;
  ExactGemmParams g1{a.ln1_f32, H, w.w132, I, T, I, H, w.b1, 1, rnd, e->x_mid, I, cal, 1 + 8 * i + 7, 0};
  check_launch(e, launch_exact_gemm(g1, e->sms, st), "ffn1_f32");
  tap_record(e, lsite(i, "ffn", "mid"), e->x_mid, size_t(T) * I * 4);
  ExactGemmParams g2{e->x_mid, I, w.w232, H, T, H, I, nullptr, 0, 0, e->x_proj, H, nullptr, 0, 0};
  check_launch(e, launch_exact_gemm(g2, e->sms, st), "ffn2_f32");
  ExactLnParams ln{e->x_proj, w.b2, a.ln1_f32, w.ln2_g, w.ln2_b, f32(e->d.layernorm_eps), T, rnd, a.hid_f32,
                   nullptr, 0.0f, i + 1 < L ? cal : nullptr, 1 + 8 * (i + 1)};
  if (next_int8) {
    ln.out_f32 = e->taps ? e->tap_ln : nullptr;   // attn.in tap of the next layer
    ln.out_i8 = next_q;
    ln.s_out = f32(sc(e, input_site(i + 1)));
  }
  check_launch(e, launch_exact_ln(ln, H, st), "ln2_f32");
}

// one encoder layer; `in_q` = index of xq holding this layer's input codes (INT8 inputs)
static void run_layer(samp_engine* e, int i, const uint8_t* prec, int& cur) {
  const int L = e->d.num_layers, H = e->d.hidden, I = e->d.intermediate, T = e->geo.T;
  const uint8_t p = prec[i];
  const bool next_int8 = i + 1 < L && (prec[i + 1] == SAMP_LAYER_FULL_INT8 || prec[i + 1] == SAMP_LAYER_MHA_INT8);
  Activations& a = e->act;
  LayerDev& w = e->layers[i];
  // small batches: twice the LN-GEMM CTAs (8-CTA clusters, one numpy leaf each) so each
  // streams half the weights; SAMP_NO_LN_SMALL=1 keeps the 4-CTA clusters
  const int mtiles = (T + GEMM_BM - 1) / GEMM_BM;
  const bool ln_small = e->tiles.bn_ln_small && mtiles * 8 <= e->sms && !env_flag("SAMP_NO_LN_SMALL");
  Tiles tsm = e->tiles;
  if (ln_small) {
    tsm.bn_ln = tsm.bn_ln_small;
    tsm.cluster_ln = 8;
  }
  const Tiles& t = e->tiles;
  const Tiles& tln = tsm;
  // QKV tiles 64 wide when 128-wide ones would leave most SMs idle (batch 1: 36 CTAs, not 18)
  const bool qkv_narrow = mtiles * (3 * H / 128) * 2 <= e->sms && (3 * H) % 64 == 0 && !env_flag("SAMP_NO_QKV_NARROW");
  const float eps = f32(e->d.layernorm_eps);
  const int fp16_store = e->d.fp16_storage;
  const bool int8_attn = p == SAMP_LAYER_FULL_INT8 || p == SAMP_LAYER_MHA_INT8;
  cudaStream_t st = e->stream_in_use;

  // ---------------- attention block
  double s_in = 0;
  if (int8_attn) {
    s_in = sc(e, input_site(i));
    record(e, "in_q", i, a.xq[cur], size_t(T) * H);
    usage_tap(e, i == 0 ? 0 : 1 + 8 * i, a.xq[cur], T, H, H);
    EpiQKV::Params qp{};
    qp.out = a.qkv_i8;
    qp.ldo = 3 * H;
    qp.bias = w.qkv_b;
    qp.block_cols = H;
    qp.mult0 = mult_of(s_in, w.s_w[0]);
    qp.mult1 = mult_of(s_in, w.s_w[1]);
    qp.mult2 = mult_of(s_in, w.s_w[2]);
    qp.sout0 = f32(sc(e, lsite(i, "attn", "q")));
    qp.sout1 = f32(sc(e, lsite(i, "attn", "k")));
    qp.sout2 = f32(sc(e, lsite(i, "attn", "v")));
    AttnParams ap{};
    ap.ctx_out = a.ctx_i8;
    ap.tile_seq = e->geo.d_tile_seq;
    ap.tile_q0 = e->geo.d_tile_q0;
    ap.tile_cnt = e->geo.d_tile_cnt;
    ap.seq_start = e->geo.d_seq_start;
    ap.att_len = e->geo.d_att_len;
    ap.hidden = H;
    const double sq = sc(e, lsite(i, "attn", "q")), sk = sc(e, lsite(i, "attn", "k"));
    const double sv = sc(e, lsite(i, "attn", "v")), ssm = sc(e, lsite(i, "attn", "softmax"));
    ap.mult_scores = f32(sq * sk / std::sqrt(double(H / e->d.num_heads)));
    ap.s_softmax = f32(ssm);
    ap.mult_ctx = mult_of(ssm, sv);
    ap.s_ctx = f32(sc(e, lsite(i, "attn", "out_in")));
    ap.tmem_cols = tmem_cols_for_keys(e->geo.max_nkp);
    if (e->usage) ap.hist = e->usage + size_t(1 + 8 * i + 4) * 256;
    // fused QKV GEMM + attention (qkv_attention.cuh) when every tile's keys fit one 128-row
    // tile; the code-usage / capture_taps modes keep the two kernels (they tap q|k|v)
    const bool fused = e->geo.max_nkp <= 128 && H % 128 == 0 && !e->usage && !e->taps &&
                       !env_flag("SAMP_NO_QA_FUSED");
    if (fused) {
      QAParams fq{};
      fq.att = ap;
      fq.bias = w.qkv_b;
      fq.mult0 = qp.mult0;
      fq.mult1 = qp.mult1;
      fq.mult2 = qp.mult2;
      fq.sout0 = qp.sout0;
      fq.sout1 = qp.sout1;
      fq.sout2 = qp.sout2;
      fq.qkv_out = e->capture ? a.qkv_i8 : nullptr;
      fq.heads = e->d.num_heads;
      fq.ntiles = e->geo.ntiles;
      if (e->dep_on) {
        fq.tile_done = e->geo.d_tile_done;
        fq.late_trigger = env_flag("SAMP_QA_LATE_TRIGGER");
        ++e->dep_count;
      }
      check_launch(e, launch_qkv_attention(a.a_xq[cur], w.m_qkv_i8_64, fq, e->sms, st), "qkv_attention_i8");
      record(e, "qkv_q", i, a.qkv_i8, size_t(T) * 3 * H);
    } else {
    // persistent 128-wide tiles, two CTAs/SM: 35.9k vs 35.8k sentences/s at batch 32 and
    // batch-1 fully-quant p50 0.525 vs 0.55 ms (twice the CTAs at one row tile)
    if (!env_flag("SAMP_QKV_ONETILE") && (3 * H) % 128 == 0)
      check_launch(e, qkv_narrow ? gemm_qkv_i8(-64, a.a_xq[cur], w.m_qkv_i8_64, T, 3 * H, H, qp, st)
                                 : gemm_qkv_i8(-128, a.a_xq[cur], w.m_qkv_i8_128, T, 3 * H, H, qp, st), "qkv_i8");
    else
      check_launch(e, gemm_qkv_i8(t.bn_qkv, a.a_xq[cur], w.m_qkv_i8, T, 3 * H, H, qp, st), "qkv_i8");
    record(e, "qkv_q", i, a.qkv_i8, size_t(T) * 3 * H);
    if (e->taps) taps_qkv(e, i, false, a.a_xq[cur], w, qp.mult0, qp.mult1, qp.mult2, 0);
    for (int k = 0; k < 3; ++k) usage_tap(e, 1 + 8 * i + 1 + k, a.qkv_i8 + k * H, T, H, 3 * H);
    launch_attention(e, false, ap);
    }
    if (e->taps) taps_attention(e, i, false, ap, 0);
    record(e, "ctx_q", i, a.ctx_i8, size_t(T) * H);
    usage_tap(e, 1 + 8 * i + 5, a.ctx_i8, T, H, H);
    EpiResLN::Params lp{};
    lp.bias = w.ob;
    lp.res_i8 = a.xq[cur];
    lp.res_scale = f32(s_in);
    lp.gamma = w.ln1_g;
    lp.beta = w.ln1_b;
    lp.noclamp = w.ln1_bounded;
    lp.mult = mult_of(sc(e, lsite(i, "attn", "out_in")), w.s_w[3]);
    lp.eps = eps;
    lp.hidden = H;
    lp.out_i8 = a.ffn_in_i8;
    lp.out_map = ln_small ? a.st_small_ffn_in : a.st_ffn_in;   // TMA-store epilogue (gemm_ln_i8 decides)
    lp.s_out = f32(sc(e, lsite(i, "ffn", "in")));
    if (p == SAMP_LAYER_MHA_INT8) {  // FP FFN consumes dequant(ffn.in codes)
      lp.deq_outputs = 1;
      lp.out_f32 = a.ln1_f32;
      lp.out_f16 = a.ln1_f16;
    }
    if (e->taps) lp.tap_f32 = e->tap_ln;
    if (fused && e->dep_on) {
      lp.dep_cnt = e->geo.d_tile_done;
      lp.dep_rt = e->geo.d_rt;
      lp.dep_target = e->dep_count * e->d.num_heads * 4 * qa_tpr();
    }
    if (!ln_gemm_splitk(e, "outproj_i8", a.a_ctx_i8, w.m_wo_i8_64, H, lp, st))
      check_launch(e, gemm_ln_i8(tln, a.a_ctx_i8, ln_small ? w.m_wo_i8_s : w.m_wo_i8, T, H, H, lp, st, a.a_ctx_i8_mc), "outproj_i8");
    tap_record(e, lsite(i, "ffn", "in"), e->tap_ln, size_t(T) * H * 4);
    record(e, "ffn_in_q", i, a.ffn_in_i8, size_t(T) * H);
    usage_tap(e, 1 + 8 * i + 6, a.ffn_in_i8, T, H, H);
  } else {
    record(e, "in_f32", i, a.hid_f32, size_t(T) * H * 4);
    tap_record(e, lsite(i, "attn", "in"), a.hid_f32, size_t(T) * H * 4);
    // reference fp16 storage rounds the FP layers' stored values; FFN_ONLY's MHA runs
    // without it (encoder.py:493-497 passes round_fn None)
    const int rnd = p == SAMP_LAYER_FP ? fp16_store : 0;
    if (e->exact) {
      exact_mha(e, i, w, rnd, p == SAMP_LAYER_FFN_INT8);
      if (p == SAMP_LAYER_FFN_INT8) {
        record(e, "ffn_in_q", i, a.ffn_in_i8, size_t(T) * H);
        usage_tap(e, 1 + 8 * i + 6, a.ffn_in_i8, T, H, H);
      }
    }
    float* cal = e->calib_amax;
    const int cbase = 1 + 8 * i;   // activation_sites order: attn.in q k v softmax out_in ffn.in ffn.mid
    if (!e->exact) {
    EpiF16Out::Params qp{a.qkv_f16, 3 * H, w.qkv_b, 0, cal, cbase + 1, H};
    if (qkv_narrow)   // small batches: 64-wide tiles, 4x the CTAs of the 256-wide default
      check_launch(e, gemm_f16out(64, a.a_hid_f16, w.m_qkv_f16_64, T, 3 * H, 2 * H, qp, st), "qkv_f16");
    else
      check_launch(e, gemm_f16out(t.bn_qkv, a.a_hid_f16, w.m_qkv_f16, T, 3 * H, 2 * H, qp, st), "qkv_f16");
    if (e->taps) taps_qkv(e, i, true, a.a_hid_f16, w, 1.0f, 1.0f, 1.0f, rnd);
    AttnParams ap{};
    ap.ctx_out = a.ctx_f16;
    ap.tile_seq = e->geo.d_tile_seq;
    ap.tile_q0 = e->geo.d_tile_q0;
    ap.tile_cnt = e->geo.d_tile_cnt;
    ap.seq_start = e->geo.d_seq_start;
    ap.att_len = e->geo.d_att_len;
    ap.hidden = H;
    ap.mult_scores = f32(1.0 / std::sqrt(double(H / e->d.num_heads)));
    ap.tmem_cols = tmem_cols_for_keys(e->geo.max_nkp);
    ap.amax = cal;
    ap.site_sm = cbase + 4;
    ap.site_ctx = cbase + 5;
    launch_attention(e, true, ap);
    if (e->taps) taps_attention(e, i, true, ap, rnd);
    EpiResLN::Params lp{};
    lp.bias = w.ob;
    lp.res_f32 = a.hid_f32;
    lp.map_res = a.st_hid_f32;   // small-batch TMA-loaded residual (gemm_ln_f16 decides)
    lp.gamma = w.ln1_g;
    lp.beta = w.ln1_b;
    lp.acc_is_f32 = 1;
    lp.eps = eps;
    lp.hidden = H;
    if (p == SAMP_LAYER_FFN_INT8) {
      lp.out_i8 = a.ffn_in_i8;
      lp.s_out = f32(sc(e, lsite(i, "ffn", "in")));
    } else {
      lp.out_f32 = a.ln1_f32;
      lp.out_f16 = a.ln1_f16;
      lp.map_f32 = a.st_ln1_f32;   // small-batch TMA-store epilogue (gemm_ln_f16 decides)
      lp.map_f16 = a.st_ln1_f16;
      lp.f16_round = fp16_store;
      lp.amax = cal;
      lp.site = cbase + 6;
      lp.site2 = -1;
    }
    if (e->taps) lp.tap_f32 = e->tap_ln;
    check_launch(e, gemm_ln_f16(tln, a.a_ctx_f16, ln_small ? w.m_wo_f16_s : w.m_wo_f16, T, H, 2 * H, lp, st),
                 "outproj_f16");
    tap_record(e, lsite(i, "ffn", "in"), e->tap_ln, size_t(T) * H * 4);
    if (p == SAMP_LAYER_FFN_INT8) {
      record(e, "ffn_in_q", i, a.ffn_in_i8, size_t(T) * H);
      usage_tap(e, 1 + 8 * i + 6, a.ffn_in_i8, T, H, H);
    } else {
      record(e, "ln1_f32", i, a.ln1_f32, size_t(T) * H * 4);
    }
    }   // !e->exact
  }

  // ---------------- feed-forward block; output goes to xq[cur^1] (codes) or hid_f32/f16
  EpiResLN::Params lp{};
  lp.gamma = w.ln2_g;
  lp.beta = w.ln2_b;
  lp.noclamp = w.ln2_bounded;
  lp.eps = eps;
  lp.hidden = H;
  lp.bias = w.b2;
  if (next_int8) {
    lp.out_i8 = a.xq[cur ^ 1];
    lp.out_map = ln_small ? a.st_small_xq[cur ^ 1] : a.st_xq[cur ^ 1];
    lp.s_out = f32(sc(e, input_site(i + 1)));
    if (e->taps) lp.tap_f32 = e->tap_ln;   // attn.in of the next layer, before its quantize
  } else {
    lp.out_f32 = a.hid_f32;
    lp.out_f16 = i + 1 < L ? a.hid_f16 : nullptr;   // f16 copy only feeds a next FP layer
  }
  if (p == SAMP_LAYER_FULL_INT8 || p == SAMP_LAYER_FFN_INT8) {
    const double s_fin = sc(e, lsite(i, "ffn", "in")), s_mid = sc(e, lsite(i, "ffn", "mid"));
    EpiGeluQuant::Params gp{a.mid_i8, I, w.b1, mult_of(s_fin, w.s_w[4]), f32(s_mid)};
    // |x| <= K * 128^2 * |mult| + max|b1| far below where C*(x + K x^3) overflows: the
    // GELU's inf/nan path is unreachable (gelu8_finite)
    const bool finite = double(H) * 16384.0 * std::fabs(double(gp.mult)) + w.b1_absmax < 1e12;
    // codes from the MUFU GELU with exact fallback on flagged elements, when this scale
    // passed the exhaustive admission check (gelu_fast_prepare, before any capture)
    auto ok = e->gelu_fast_ok.find(bits_of(gp.s_out));
    const bool fast = finite && ok != e->gelu_fast_ok.end() && ok->second;
    gp.inv_s = gelu_inv_s(gp.s_out);
    gp.fixup_all = env_flag("SAMP_GELU_FIXUP_ALL");   // test: every 8-group through gelu_fixup
    if (env_flag("SAMP_GELU_FLAGS")) {   // measurement: count flagged 8-groups per forward
      if (!g_gelu_flags) cudaMallocManaged(&g_gelu_flags, sizeof(unsigned long long));
      gp.flag_count = g_gelu_flags;
    }
    const int k1 = ffn1_bn_index(T, I, e->sms);
    check_launch(e, gemm_gelu_i8(FFN1_BN[k1], fast ? GELU_FAST : finite ? GELU_FINITE : GELU_GENERAL, a.a_ffn_in,
                                 w.m_w1_i8[k1], T, I, H, gp, st), "ffn1_i8");
    record(e, "mid_q", i, a.mid_i8, size_t(T) * I);
    if (e->taps) taps_ffn_mid(e, i, false, a.a_ffn_in, w, gp.mult, 0);
    usage_tap(e, 1 + 8 * i + 7, a.mid_i8, T, I, I);
    lp.res_i8 = a.ffn_in_i8;
    lp.res_scale = f32(s_fin);
    lp.mult = mult_of(s_mid, w.s_w[5]);
    if (!ln_gemm_splitk(e, "ffn2_i8", a.a_mid_i8, w.m_w2_i8_64, I, lp, st))
      check_launch(e, gemm_ln_i8(tln, a.a_mid_i8, ln_small ? w.m_w2_i8_s : w.m_w2_i8, T, H, I, lp, st, a.a_mid_i8_mc), "ffn2_i8");
  } else if (e->exact) {
    exact_ffn(e, i, w, p == SAMP_LAYER_FP ? fp16_store : 0, next_int8, a.xq[cur ^ 1]);
  } else {
    EpiF16Out::Params gp{a.mid_f16, I, w.b1, 1, e->calib_amax, 1 + 8 * i + 7, 0};
    const int k1 = ffn1_bn_index(T, I, e->sms, false);   // EpiF16Out walks 32-column chunks
    check_launch(e, gemm_f16out(FFN1_BN[k1], a.a_ln1_f16, w.m_w1_f16[k1], T, I, 2 * H, gp, st), "ffn1_f16");
    if (e->taps) taps_ffn_mid(e, i, true, a.a_ln1_f16, w, 1.0f, p == SAMP_LAYER_FP ? fp16_store : 0);
    lp.res_f32 = a.ln1_f32;
    lp.acc_is_f32 = 1;
    lp.map_f32 = a.st_hid_f32;
    lp.map_f16 = a.st_hid_f16;
    lp.map_res = a.st_ln1_f32;
    lp.f16_round = (p == SAMP_LAYER_FP) ? fp16_store : 0;
    if (e->calib_amax && i + 1 < L) {   // tap L{i+1}.attn.in
      lp.amax = e->calib_amax;
      lp.site = 1 + 8 * (i + 1);
      lp.site2 = -1;
    }
    check_launch(e, gemm_ln_f16(tln, a.a_mid_f16, ln_small ? w.m_w2_f16_s : w.m_w2_f16, T, H, 2 * I, lp, st),
                 "ffn2_f16");
  }
  if (next_int8) {
    cur ^= 1;
    tap_record(e, input_site(i + 1), e->tap_ln, size_t(T) * H * 4);
    record(e, "out_q", i, a.xq[cur], size_t(T) * H);
  } else {
    record(e, "out_f32", i, a.hid_f32, size_t(T) * H * 4);
  }
}


// embed -> layers -> head for the current geometry, all launched on `st`
static void enqueue_kernels(samp_engine* e, const uint8_t* prec, int nseq, int head, cudaStream_t st) {
  // ---------------- embedding (+ quantize at embed.out when layer 0 is INT8-attention)
  const samp_model_desc& d = e->d;
  const int L = d.num_layers, H = d.hidden, T = e->geo.T;
  Activations& a = e->act;
  const bool first_int8 = prec[0] == SAMP_LAYER_FULL_INT8 || prec[0] == SAMP_LAYER_MHA_INT8;
  // SAMP_QA_FLAGS=1 (opt-in, measured slower): the out-projection of a fused layer starts on
  // row tiles the fused kernel has published instead of waiting for the whole grid (off in
  // the capture / tap / usage modes, exact mode, and when launches are dropped for measurement)
  e->dep_count = 0;
  e->dep_on = !e->exact && !e->taps && !e->usage && !e->capture && e->geo.max_nkp <= 128 && H % 128 == 0 &&
              !env_flag("SAMP_NO_QA_FUSED") && env_flag("SAMP_QA_FLAGS") && !std::getenv("SAMP_SKIP") &&
              outproj_dep_ok(e);
  if (e->dep_on) SAMP_CUDA(cudaMemsetAsync(e->geo.d_tile_done, 0, e->geo.ntiles * sizeof(int), st));
  EmbedParams ep{};
  ep.ids = a.ids;
  ep.segs = a.segs;
  ep.pos = a.pos;
  ep.word = e->word;
  ep.position = e->position;
  ep.token_type = e->token_type;
  ep.gamma = e->emb_g;
  ep.beta = e->emb_b;
  ep.eps = f32(d.layernorm_eps);
  ep.hidden = H;
  ep.T = T;
  ep.f16_round = d.fp16_storage;
  ep.out_f32 = a.hid_f32;
  ep.out_f16 = a.hid_f16;
  if (first_int8) {
    ep.out_i8 = a.xq[0];
    ep.s_out = f32(sc(e, "embed.out"));
    // layer 0 reads only the codes (its residual is dequant(codes)): the float copies are
    // written only for stage capture (7 B/element less HBM traffic)
    if (!e->capture) ep.out_f32 = nullptr;
    ep.out_f16 = nullptr;
  }
  ep.amax = e->calib_amax;   // taps embed.out and L0.attn.in (same tensor)
  ep.site = 0;
  ep.site2 = 1;
  check_launch(e, launch_embed(ep, st), "embed");
  record(e, "embed_f32", 0, a.hid_f32, size_t(T) * H * 4);
  tap_record(e, "embed.out", a.hid_f32, size_t(T) * H * 4);
  // SAMP_PREFETCH=1: the layers' weights (in use order) into L2 on a side stream while the
  // first layers run.  Opt-in: measured neutral (C2 and every batch-1 mode within noise,
  // DESIGN.md) — the small-batch kernels are not waiting on HBM.  Never in the per-kernel
  // profiling pass, which times kernels one by one.
  const bool prefetch = !e->exact && !e->profiling && env_flag("SAMP_PREFETCH");
  if (prefetch) {
    if (!e->side) {
      SAMP_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
      SAMP_CUDA(cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
      SAMP_CUDA(cudaEventCreateWithFlags(&e->join_ev, cudaEventDisableTiming));
    }
    PrefetchList pl{};
    const size_t HH = size_t(H) * H, HI = size_t(H) * d.intermediate;
    auto add = [&](const void* ptr, size_t bytes) {
      if (ptr && pl.n < PREFETCH_MAX_RANGES) {
        pl.ptr[pl.n] = ptr;
        pl.bytes[pl.n] = bytes;
        ++pl.n;
      }
    };
    for (int i = 0; i < L; ++i) {
      const LayerDev& w = e->layers[i];
      const bool mha8 = prec[i] == SAMP_LAYER_FULL_INT8 || prec[i] == SAMP_LAYER_MHA_INT8;
      const bool ffn8 = prec[i] == SAMP_LAYER_FULL_INT8 || prec[i] == SAMP_LAYER_FFN_INT8;
      if (mha8) { add(w.qkv_i8, 3 * HH); add(w.wo_i8, HH); }
      else { add(w.qkv_f16, 6 * HH); add(w.wo_f16, 2 * HH); }
      if (ffn8) { add(w.w1_i8, HI); add(w.w2_i8, HI); }
      else { add(w.w1_f16, 2 * HI); add(w.w2_f16, 2 * HI); }
    }
    SAMP_CUDA(cudaEventRecord(e->fork_ev, st));
    SAMP_CUDA(cudaStreamWaitEvent(e->side, e->fork_ev, 0));
    SAMP_REQUIRE(launch_l2_prefetch(pl, 32, e->side) == cudaSuccess, SAMP_E_DEVICE, "l2_prefetch launch failed");
    e->launches++;
    SAMP_CUDA(cudaEventRecord(e->join_ev, e->side));
  }
  int cur = 0;
  for (int i = 0; i < L; ++i) run_layer(e, i, prec, cur);
  if (prefetch) SAMP_CUDA(cudaStreamWaitEvent(st, e->join_ev, 0));
  // ---------------- heads + outputs (final hidden is always F32 in hid_f32)
  const int nl = d.num_labels;
  if (head != SAMP_HEAD_NONE) {
    HeadParams hp{};
    hp.hidden = a.hid_f32;
    hp.seq_start = e->geo.d_seq_start;
    hp.pool_w = e->pool_w;
    hp.pooled = a.pooled;
    hp.pool_b = e->pool_b;
    hp.head_wt = e->head_wt;
    hp.head_b = e->head_b;
    hp.hidden_size = H;
    hp.num_labels = nl;
    hp.nseq = nseq;
    hp.T = T;
    hp.logits = a.logits;
    hp.probs = a.probs;
    hp.labels = a.labels;
    check_launch(e, head == SAMP_HEAD_CLASSIFY ? launch_classify(hp, st) : launch_tag(hp, st), "head");
  }
}

}  // namespace samp

using namespace samp;

extern "C" int samp_engine_create(const samp_model_desc* desc, int device, samp_engine** out) {
  return guarded([&] {
    SAMP_REQUIRE(desc && out, SAMP_E_CONFIGURATION, "null argument");
    const samp_model_desc& d = *desc;
    SAMP_REQUIRE(d.num_layers >= 1 && d.hidden >= 1 && d.num_heads >= 1 && d.intermediate >= 1 &&
                     d.vocab_size >= 1 && d.max_position >= 1 && d.type_vocab_size >= 1 && d.num_labels >= 1,
                 SAMP_E_CONFIGURATION, "model sizes must be >= 1");
    SAMP_REQUIRE(d.hidden % d.num_heads == 0, SAMP_E_CONFIGURATION, "hidden not divisible by num_heads");
    SAMP_REQUIRE(d.hidden / d.num_heads == 64, SAMP_E_CONFIGURATION,
                 "the B200 kernels are built for head_dim = 64 (BERT-base/large); got " +
                     std::to_string(d.hidden / d.num_heads));
    SAMP_REQUIRE(d.max_position <= ATT_MAX_KEYS, SAMP_E_CONFIGURATION, "max_position > 512 is not supported");
    SAMP_REQUIRE(d.num_labels <= HEAD_MAX_LABELS, SAMP_E_CONFIGURATION, "num_labels > 64 is not supported");
    Tiles t = choose_tiles(d.hidden, d.intermediate);
    SAMP_REQUIRE(t.bn_qkv && t.bn_ffn1 && t.bn_ln, SAMP_E_CONFIGURATION,
                 "unsupported hidden/intermediate sizes for the tcgen05 tiles (need multiples of 64, hidden in "
                 "{64,128,256,384,512,768,1024})");
    int rc = samp_device_check(device);
    if (rc != SAMP_OK) throw SampError(rc, samp_last_error());
    SAMP_CUDA(cudaSetDevice(device));
    auto* e = new samp_engine();
    e->d = d;
    e->device = device;
    e->tiles = t;
    cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device);
    e->layers.resize(d.num_layers);
    if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete e;
      throw SampError(SAMP_E_DEVICE, "cudaStreamCreate failed");
    }
    e->stream_in_use = e->stream;
    *out = e;
  });
}

extern "C" void samp_engine_destroy(samp_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  clear_graphs(e);
  if (e->pinned_ids) cudaFreeHost(e->pinned_ids);
  if (e->pinned_out) cudaFreeHost(e->pinned_out);
  if (e->side) cudaStreamDestroy(e->side);
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->join_ev) cudaEventDestroy(e->join_ev);
  cudaStreamDestroy(e->stream);
  delete e;
}

extern "C" int samp_load_embeddings(samp_engine* e, const float* word, const float* position,
                                    const float* token_type, const float* g, const float* b) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_CUDA(cudaSetDevice(e->device));
    const size_t H = e->d.hidden;
    auto up = [&](const float* src, size_t n) {
      float* dst = e->mem.alloc<float>(n);
      SAMP_CUDA(cudaMemcpy(dst, src, n * 4, cudaMemcpyHostToDevice));
      return dst;
    };
    e->word = up(word, size_t(e->d.vocab_size) * H);
    e->position = up(position, size_t(e->d.max_position) * H);
    e->token_type = up(token_type, size_t(e->d.type_vocab_size) * H);
    e->emb_g = up(g, H);
    e->emb_b = up(b, H);
    e->emb_loaded = true;
  });
}

extern "C" int samp_load_layer(samp_engine* e, int layer, const float* const* t) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_REQUIRE(layer >= 0 && layer < e->d.num_layers, SAMP_E_CONFIGURATION, "layer index out of range");
    SAMP_CUDA(cudaSetDevice(e->device));
    const int H = e->d.hidden, I = e->d.intermediate;
    LayerDev& w = e->layers[layer];
    // per-tensor INT8 weight scales exactly as quantize_weight (encoder.py:191-194)
    const float* mats[6] = {t[0], t[2], t[4], t[6], t[10], t[12]};
    const size_t sizes[6] = {size_t(H) * H, size_t(H) * H, size_t(H) * H, size_t(H) * H, size_t(H) * I, size_t(I) * H};
    for (int k = 0; k < 6; ++k) w.s_w[k] = site_scale(host_amax(mats[k], sizes[k]));
    w.qkv_i8 = e->mem.alloc<int8_t>(size_t(3) * H * H);
    w.wo_i8 = e->mem.alloc<int8_t>(size_t(H) * H);
    w.w1_i8 = e->mem.alloc<int8_t>(size_t(I) * H);
    w.w2_i8 = e->mem.alloc<int8_t>(size_t(H) * I);
    w.qkv_f16 = e->mem.alloc<__half>(size_t(3) * H * H);
    w.wo_f16 = e->mem.alloc<__half>(size_t(H) * H);
    w.w1_f16 = e->mem.alloc<__half>(size_t(I) * H);
    w.w2_f16 = e->mem.alloc<__half>(size_t(H) * I);
    float* tmp = e->mem.alloc<float>(size_t(H) * std::max(H, I));
    auto pack = [&](const float* src, int K, int N, double scale, int8_t* oi8, __half* of16, int row_off) {
      SAMP_CUDA(cudaMemcpy(tmp, src, size_t(K) * N * 4, cudaMemcpyHostToDevice));
      SAMP_CUDA(launch_pack_weight(tmp, K, N, f32(scale), oi8, of16, row_off, 0));
      SAMP_CUDA(cudaDeviceSynchronize());
    };
    // exact FP32 copies in the archive's (in, out) layout; QKV concatenated along out
    w.qkv32 = e->mem.alloc<float>(size_t(H) * 3 * H);
    for (int k = 0; k < 3; ++k)
      SAMP_CUDA(cudaMemcpy2D(w.qkv32 + size_t(k) * H, size_t(3) * H * 4, t[2 * k], size_t(H) * 4, size_t(H) * 4, H,
                             cudaMemcpyHostToDevice));
    w.wo32 = e->mem.alloc<float>(size_t(H) * H);
    SAMP_CUDA(cudaMemcpy(w.wo32, t[6], size_t(H) * H * 4, cudaMemcpyHostToDevice));
    w.w132 = e->mem.alloc<float>(size_t(H) * I);
    SAMP_CUDA(cudaMemcpy(w.w132, t[10], size_t(H) * I * 4, cudaMemcpyHostToDevice));
    w.w232 = e->mem.alloc<float>(size_t(I) * H);
    SAMP_CUDA(cudaMemcpy(w.w232, t[12], size_t(I) * H * 4, cudaMemcpyHostToDevice));
    pack(t[0], H, H, w.s_w[0], w.qkv_i8, w.qkv_f16, 0);
    pack(t[2], H, H, w.s_w[1], w.qkv_i8, w.qkv_f16, H);
    pack(t[4], H, H, w.s_w[2], w.qkv_i8, w.qkv_f16, 2 * H);
    pack(t[6], H, H, w.s_w[3], w.wo_i8, w.wo_f16, 0);
    pack(t[10], H, I, w.s_w[4], w.w1_i8, w.w1_f16, 0);
    pack(t[12], I, H, w.s_w[5], w.w2_i8, w.w2_f16, 0);
    e->mem.release(tmp);
    auto up = [&](const float* src, size_t n) {
      float* dst = e->mem.alloc<float>(n);
      SAMP_CUDA(cudaMemcpy(dst, src, n * 4, cudaMemcpyHostToDevice));
      return dst;
    };
    w.qkv_b = e->mem.alloc<float>(size_t(3) * H);
    SAMP_CUDA(cudaMemcpy(w.qkv_b, t[1], H * 4, cudaMemcpyHostToDevice));
    SAMP_CUDA(cudaMemcpy(w.qkv_b + H, t[3], H * 4, cudaMemcpyHostToDevice));
    SAMP_CUDA(cudaMemcpy(w.qkv_b + 2 * H, t[5], H * 4, cudaMemcpyHostToDevice));
    w.ob = up(t[7], H);
    w.ln1_g = up(t[8], H);
    w.ln1_b = up(t[9], H);
    w.b1 = up(t[11], I);
    w.b1_absmax = 0;
    for (int j = 0; j < I; ++j) w.b1_absmax = std::max(w.b1_absmax, double(std::fabs(t[11][j])));
    w.b2 = up(t[13], H);
    w.ln2_g = up(t[14], H);
    w.ln2_b = up(t[15], H);
    // |((x - mean) * inv) * g + b| <= sqrt(H) max|g| + max|b| (each |x - mean| <= sqrt(H var),
    // inv = 1/sqrt(var + eps) with eps > 0), doubled for rounding: far below the 2^64 where
    // the LN epilogue's fast quotient needs its clamp
    auto ln_bounded = [&](const float* g, const float* b) {
      double mg = 0, mb = 0;
      for (int j = 0; j < H; ++j) {
        if (!std::isfinite(g[j]) || !std::isfinite(b[j])) return false;
        mg = std::max(mg, double(std::fabs(g[j])));
        mb = std::max(mb, double(std::fabs(b[j])));
      }
      return e->d.layernorm_eps > 0 && 2.0 * std::sqrt(double(H)) * mg + mb < 1e18;
    };
    w.ln1_bounded = ln_bounded(t[8], t[9]);
    w.ln2_bounded = ln_bounded(t[14], t[15]);
    const Tiles& tl = e->tiles;
    w.m_qkv_i8 = tmap_i8(w.qkv_i8, 3 * H, H, H, 128, tl.bn_qkv);
    w.m_qkv_i8_128 = tmap_i8(w.qkv_i8, 3 * H, H, H, 128, 128);
    w.m_qkv_i8_64 = tmap_i8(w.qkv_i8, 3 * H, H, H, 128, 64);
    w.m_wo_i8 = tmap_i8(w.wo_i8, H, H, H, 128, tl.bn_ln);
    w.m_wo_i8_64 = tmap_i8(w.wo_i8, H, H, H, 128, 64);
    for (int k = 0; k < 3; ++k)
      if (I % FFN1_BN[k] == 0) {
        w.m_w1_i8[k] = tmap_i8(w.w1_i8, I, H, H, 128, FFN1_BN[k]);
        w.m_w1_f16[k] = tmap_f16(w.w1_f16, I, H, H, 64, FFN1_BN[k]);
      }
    w.m_w2_i8 = tmap_i8(w.w2_i8, H, I, I, 128, tl.bn_ln);
    w.m_w2_i8_64 = tmap_i8(w.w2_i8, H, I, I, 128, 64);
    w.m_qkv_f16 = tmap_f16(w.qkv_f16, 3 * H, H, H, 64, tl.bn_qkv);
    w.m_qkv_f16_64 = tmap_f16(w.qkv_f16, 3 * H, H, H, 64, 64);
    w.m_wo_f16 = tmap_f16(w.wo_f16, H, H, H, 64, tl.bn_ln);
    w.m_w2_f16 = tmap_f16(w.w2_f16, H, I, I, 64, tl.bn_ln);
    if (tl.bn_ln_small) {
      w.m_wo_i8_s = tmap_i8(w.wo_i8, H, H, H, 128, tl.bn_ln_small);
      w.m_w2_i8_s = tmap_i8(w.w2_i8, H, I, I, 128, tl.bn_ln_small);
      w.m_wo_f16_s = tmap_f16(w.wo_f16, H, H, H, 64, tl.bn_ln_small);
      w.m_w2_f16_s = tmap_f16(w.w2_f16, H, I, I, 64, tl.bn_ln_small);
    }
    w.loaded = true;
  });
}

extern "C" int samp_load_heads(samp_engine* e, const float* pool_w, const float* pool_b, const float* head_w,
                               const float* head_b) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_CUDA(cudaSetDevice(e->device));
    const int H = e->d.hidden, L = e->d.num_labels;
    auto up_t = [&](const float* src, int K, int N) {  // (in,out) -> (out,in)
      float* raw = e->mem.alloc<float>(size_t(K) * N);
      float* dst = e->mem.alloc<float>(size_t(K) * N);
      SAMP_CUDA(cudaMemcpy(raw, src, size_t(K) * N * 4, cudaMemcpyHostToDevice));
      SAMP_CUDA(launch_transpose_f32(raw, K, N, dst, 0));
      SAMP_CUDA(cudaDeviceSynchronize());
      e->mem.release(raw);
      return dst;
    };
    if (pool_w) {
      e->pool_w = e->mem.alloc<float>(size_t(H) * H);
      SAMP_CUDA(cudaMemcpy(e->pool_w, pool_w, size_t(H) * H * 4, cudaMemcpyHostToDevice));
      e->pool_b = e->mem.alloc<float>(H);
      SAMP_CUDA(cudaMemcpy(e->pool_b, pool_b, H * 4, cudaMemcpyHostToDevice));
    }
    e->head_wt = up_t(head_w, H, L);
    e->head_b = e->mem.alloc<float>(L);
    SAMP_CUDA(cudaMemcpy(e->head_b, head_b, L * 4, cudaMemcpyHostToDevice));
    e->heads_loaded = true;
  });
}

extern "C" int samp_weight_scales(samp_engine* e, int layer, double* out6) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_REQUIRE(layer >= 0 && layer < e->d.num_layers && e->layers[layer].loaded, SAMP_E_CONFIGURATION,
                 "layer not loaded");
    for (int k = 0; k < 6; ++k) out6[k] = e->layers[layer].s_w[k];
  });
}

extern "C" int samp_set_site_amax(samp_engine* e, const char* site, double amax) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    clear_graphs(e);
    e->amax[site] = amax;
    // admit the FFN1 fast GELU for this ffn.mid scale now (exhaustive ~16 ms device check),
    // at calibration-load time instead of inside the first forward that needs it
    const std::string s(site);
    if (s.size() > 8 && s.compare(s.size() - 8, 8, ".ffn.mid") == 0 && !env_flag("SAMP_NO_GELU_FAST")) {
      SAMP_CUDA(cudaSetDevice(e->device));
      const float sm = f32(site_scale(amax));
      if (!e->gelu_fast_ok.count(bits_of(sm))) {
        unsigned long long counts[2] = {1, 0};
        SAMP_CUDA(gelu_fast_check(sm, gelu_inv_s(sm), counts, e->stream));
        e->gelu_fast_ok[bits_of(sm)] = counts[0] == 0;
      }
    }
  });
}

extern "C" int samp_clear_calibration(samp_engine* e) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    clear_graphs(e);
    e->amax.clear();
  });
}

extern "C" int samp_debug_gelu_fast_check(float s, unsigned long long* counts) {
  return guarded([&] { SAMP_CUDA(gelu_fast_check(s, gelu_inv_s(s), counts, nullptr)); });
}

extern "C" int samp_set_exact_fp32(samp_engine* e, int on) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    clear_graphs(e);
    e->exact = on != 0;
  });
}

extern "C" int samp_set_graphs(samp_engine* e, int on) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    clear_graphs(e);
    e->graphs_enabled = on != 0;
  });
}

extern "C" int samp_set_capture(samp_engine* e, int on) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    e->capture = on != 0;
    e->taps = on == 2;   // 2: also the F32 site taps (Engine.run capture_taps=True)
    if (e->capture) e->stages.clear();  // turning capture off keeps the last forward's stages
  });
}

extern "C" int samp_fetch_stage(samp_engine* e, const char* name, int layer, void* dst, size_t capacity,
                                size_t* bytes) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    auto it = e->stages.find(std::string(name) + "@" + std::to_string(layer));
    SAMP_REQUIRE(it != e->stages.end(), SAMP_E_CONFIGURATION,
                 std::string("no captured stage ") + name + " for layer " + std::to_string(layer));
    if (bytes) *bytes = it->second.size();
    if (dst) {
      SAMP_REQUIRE(capacity >= it->second.size(), SAMP_E_DIMENSION, "destination too small");
      std::memcpy(dst, it->second.data(), it->second.size());
    }
  });
}

// Engine.calibrate (reference encoder.py:446-454): FP forward (FP16 tensor-core path)
// with max|x| taps at all 1 + 8L activation sites, in activation_sites order.
extern "C" int samp_calibrate(samp_engine* e, int32_t nseq, const int32_t* seq_start, const int32_t* att_len,
                              const int32_t* ids, const int32_t* segs, double* amax_out) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  int rc = SAMP_OK;
  rc = guarded([&] {
    const int n = 1 + 8 * e->d.num_layers;
    SAMP_CUDA(cudaSetDevice(e->device));
    float* dev = e->mem.alloc<float>(n);
    SAMP_CUDA(cudaMemset(dev, 0, n * sizeof(float)));
    e->calib_amax = dev;
    std::vector<uint8_t> fp(e->d.num_layers, SAMP_LAYER_FP);
    samp_outputs none{};
    const int r = samp_forward(e, fp.data(), nseq, seq_start, att_len, ids, segs, SAMP_IO_HOST, &none, nullptr);
    e->calib_amax = nullptr;
    if (r != SAMP_OK) {
      e->mem.release(dev);
      throw SampError(r, samp_last_error());
    }
    std::vector<float> h(n);
    SAMP_CUDA(cudaMemcpy(h.data(), dev, n * sizeof(float), cudaMemcpyDeviceToHost));
    e->mem.release(dev);
    for (int k = 0; k < n; ++k) amax_out[k] = double(h[k]);
  });
  e->calib_amax = nullptr;
  return rc;
}

// analyze-quant (reference cli.py:269-292): one forward under `prec` with the code-usage
// taps on; counts[(site) * 256 + code + 128] += occurrences of each INT8 code the kernels
// wrote at every activation site the plan quantizes (activation_sites order, 1 + 8L sites;
// sites the plan keeps in floating point stay zero).
extern "C" int samp_code_usage(samp_engine* e, const uint8_t* prec, int32_t nseq, const int32_t* seq_start,
                               const int32_t* att_len, const int32_t* ids, const int32_t* segs,
                               unsigned long long* counts) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  int rc = SAMP_OK;
  rc = guarded([&] {
    const size_t n = size_t(1 + 8 * e->d.num_layers) * 256;
    SAMP_CUDA(cudaSetDevice(e->device));
    unsigned long long* dev = e->mem.alloc<unsigned long long>(n);
    SAMP_CUDA(cudaMemset(dev, 0, n * sizeof(unsigned long long)));
    e->usage = dev;
    samp_outputs none{};
    const int r = samp_forward(e, prec, nseq, seq_start, att_len, ids, segs, SAMP_IO_HOST, &none, nullptr);
    e->usage = nullptr;
    if (r != SAMP_OK) {
      e->mem.release(dev);
      throw SampError(r, samp_last_error());
    }
    SAMP_CUDA(cudaMemcpy(counts, dev, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    e->mem.release(dev);
  });
  e->usage = nullptr;
  return rc;
}

extern "C" int samp_sync(samp_engine* e) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] { SAMP_CUDA(cudaStreamSynchronize(e->stream_in_use)); });
}

extern "C" int samp_last_launch_count(samp_engine* e) { return e ? e->launches : 0; }

extern "C" int samp_debug_gemm_stamps(samp_engine* e, int max_launches) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    if (e->stamps) e->mem.release(e->stamps);
    e->stamps = nullptr;
    e->stamp_cap = 0;
    e->stamp_launches.clear();
    if (max_launches > 0) {
      e->stamps = e->mem.alloc<unsigned long long>(size_t(max_launches) * STAMP_CTAS * GEMM_STAMPS);
      e->stamp_cap = max_launches;
    }
  });
}

extern "C" int samp_debug_gemm_stamps_fetch(samp_engine* e, unsigned long long* out, int cap_launches,
                                            char* names, size_t names_cap, int* n_launches) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_REQUIRE(e->stamps, SAMP_E_CONFIGURATION, "GEMM stamps not enabled");
    SAMP_CUDA(cudaStreamSynchronize(e->stream_in_use));
    const int n = std::min<int>(cap_launches, int(e->stamp_launches.size()));
    SAMP_CUDA(cudaMemcpy(out, e->stamps, size_t(n) * STAMP_CTAS * GEMM_STAMPS * 8, cudaMemcpyDeviceToHost));
    std::string s;
    for (int i = 0; i < n; ++i) s += e->stamp_launches[i].first + "\n";
    SAMP_REQUIRE(s.size() < names_cap, SAMP_E_INPUT, "names buffer too small");
    std::memcpy(names, s.c_str(), s.size() + 1);
    *n_launches = n;
    e->stamp_launches.clear();
  });
}

extern "C" int samp_set_profiling(samp_engine* e, int on) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    // 1: per-launch CUDA events (+ stamps); 2: stamps only, kernels launched back to back
    // with PDL as in a normal forward (no graph) — the cross-kernel timeline (tools/timeline.py)
    e->profiling = on == 1;
    e->stamp_only = on == 2;
    e->prof.clear();
  });
}

// sync, fold pending event pairs into per-kernel totals, and write them as JSON
// {"name": [total_ms, launches], ...} into buf
extern "C" int samp_profile_report(samp_engine* e, char* buf, size_t cap) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    SAMP_CUDA(cudaStreamSynchronize(e->stream_in_use));
    for (auto& p : e->pending) {
      float ms = 0;
      SAMP_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      auto& slot = e->prof[p.name];
      slot.first += ms;
      slot.second += 1;
      e->event_pool.push_back(p.a);
      e->event_pool.push_back(p.b);
    }
    e->pending.clear();
    std::string js = "{";
    bool first = true;
    for (auto& kv : e->prof) {
      js += (first ? "\"" : ", \"") + kv.first + "\": [" + std::to_string(kv.second.first) + ", " +
            std::to_string(kv.second.second) + "]";
      first = false;
    }
    js += "}";
    SAMP_REQUIRE(buf && cap > js.size(), SAMP_E_DIMENSION, "profile buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
  });
}

extern "C" int samp_forward(samp_engine* e, const uint8_t* prec, int32_t nseq, const int32_t* seq_start,
                            const int32_t* att_len, const int32_t* ids, const int32_t* segs, int32_t io,
                            const samp_outputs* out, void* stream_arg) {
  std::lock_guard<std::recursive_mutex> lock(e->mu);   // threading contract (samp_b200.h)
  return guarded([&] {
    const samp_model_desc& d = e->d;
    const int L = d.num_layers, H = d.hidden;
    // ---------------- validation (before any device work, like the reference)
    SAMP_REQUIRE(e->emb_loaded, SAMP_E_CONFIGURATION, "embeddings not loaded");
    for (int i = 0; i < L; ++i) {
      SAMP_REQUIRE(prec[i] <= SAMP_LAYER_MHA_INT8, SAMP_E_CONFIGURATION, "bad layer precision code");
      SAMP_REQUIRE(e->layers[i].loaded, SAMP_E_CONFIGURATION, "layer " + std::to_string(i) + " not loaded");
    }
    {
      std::vector<std::string> missing;
      for (const auto& s : required_sites(prec, L))
        if (!e->amax.count(s)) missing.push_back(s);
      if (!missing.empty()) {
        std::string msg = "calibration table is missing sites: ";
        for (size_t k = 0; k < missing.size(); ++k) msg += (k ? ", " : "") + missing[k];
        throw SampError(SAMP_E_CALIBRATION, msg);
      }
    }
    SAMP_REQUIRE(nseq >= 1, SAMP_E_INPUT, "empty batch");
    SAMP_REQUIRE(seq_start[0] == 0, SAMP_E_INPUT, "seq_start[0] must be 0");
    for (int s = 0; s < nseq; ++s) {
      const int S = seq_start[s + 1] - seq_start[s];
      SAMP_REQUIRE(S >= 1, SAMP_E_INPUT, "empty token id sequence");
      SAMP_REQUIRE(S <= d.max_position, SAMP_E_INPUT,
                   "sequence length " + std::to_string(S) + " exceeds max_position " + std::to_string(d.max_position));
    }
    const int T = seq_start[nseq];
    if (io == SAMP_IO_HOST) {
      for (int k = 0; k < T; ++k) {
        SAMP_REQUIRE(ids[k] >= 0 && ids[k] < d.vocab_size, SAMP_E_INPUT,
                     "token id out of range [0, " + std::to_string(d.vocab_size) + ")");
        SAMP_REQUIRE(segs[k] >= 0 && segs[k] < d.type_vocab_size, SAMP_E_INPUT,
                     "segment id out of range [0, " + std::to_string(d.type_vocab_size) + ")");
      }
    }
    const int head = out ? out->head : SAMP_HEAD_NONE;
    if (head != SAMP_HEAD_NONE)
      SAMP_REQUIRE(e->heads_loaded && (head != SAMP_HEAD_CLASSIFY || e->pool_w), SAMP_E_CONFIGURATION,
                   "head weights not loaded");
    SAMP_CUDA(cudaSetDevice(e->device));
    // launch on the caller's stream when given (so its events / graphs see every kernel)
    e->stream_in_use = stream_arg ? static_cast<cudaStream_t>(stream_arg) : e->stream;
    set_geometry(e, nseq, seq_start, att_len);
    e->launches = 0;
    e->stages.clear();
    Activations& a = e->act;
    cudaStream_t st = e->stream_in_use;
    const int nl = d.num_labels;
    const size_t rows = head == SAMP_HEAD_CLASSIFY ? nseq : T;
    a.ids = a.idseg;
    a.segs = a.idseg + T;
    a.logits = a.headbuf;
    a.probs = a.headbuf + rows * nl;
    a.labels = reinterpret_cast<int*>(a.headbuf + 2 * rows * nl);
    // ---------------- inputs
    if (io == SAMP_IO_HOST) {
      if (e->pinned_cap < 2 * T) {
        if (e->pinned_ids) cudaFreeHost(e->pinned_ids);
        e->pinned_ids = nullptr;
        e->pinned_cap = 0;   // set only once the allocation succeeded
        const int cap = std::max(2 * T, 8192);
        SAMP_CUDA(cudaMallocHost(&e->pinned_ids, size_t(cap) * sizeof(int)));
        e->pinned_cap = cap;
      }
      SAMP_CUDA(cudaStreamSynchronize(st));  // staging buffer reuse
      std::memcpy(e->pinned_ids, ids, size_t(T) * 4);
      std::memcpy(e->pinned_ids + T, segs, size_t(T) * 4);
      SAMP_CUDA(cudaMemcpyAsync(a.ids, e->pinned_ids, size_t(T) * 8, cudaMemcpyHostToDevice, st));
    } else {
      SAMP_CUDA(cudaMemcpyAsync(a.ids, ids, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
      SAMP_CUDA(cudaMemcpyAsync(a.segs, segs, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
    }
    gelu_fast_prepare(e, prec);
    if (e->taps) ensure_taps(e);
    if (e->exact) ensure_exact(e);
    // ---------------- device work: replay a captured CUDA graph for this (plan, batch
    // geometry, head) when one exists; capture on the second sighting of a key (the first
    // run also configures every kernel's smem attributes outside of capture)
    const bool graphable = e->graphs_enabled && !e->capture && !e->profiling && !e->stamp_only && !e->calib_amax &&
                           !e->usage;
    std::string key;
    if (graphable) {
      key.assign(reinterpret_cast<const char*>(prec), L);
      key += char(head);
      key.append(reinterpret_cast<const char*>(seq_start), (nseq + 1) * sizeof(int32_t));
      key.append(reinterpret_cast<const char*>(att_len), nseq * sizeof(int32_t));
    }
    auto it = graphable ? e->graphs.find(key) : e->graphs.end();
    if (it != e->graphs.end() && it->second.exec) {
      SAMP_CUDA(cudaGraphLaunch(it->second.exec, st));
      e->launches = it->second.launches;
    } else if (graphable && e->seen.count(key)) {
      if (e->graphs.size() >= 64) clear_graphs(e);
      cudaGraph_t g = nullptr;
      SAMP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_kernels(e, prec, nseq, head, st);
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      SAMP_CUDA(cudaStreamEndCapture(st, &g));
      cudaGraphExec_t exec = nullptr;
      SAMP_CUDA(cudaGraphInstantiate(&exec, g, 0));
      cudaGraphDestroy(g);
      e->graphs[key] = GraphEntry{exec, e->launches};
      SAMP_CUDA(cudaGraphLaunch(exec, st));
    } else {
      enqueue_kernels(e, prec, nseq, head, st);
      if (graphable) {
        if (e->seen.size() >= 256) e->seen.clear();   // bounded: variable-shape servers
        e->seen.insert(key);
      }
    }
    const cudaMemcpyKind kind = io == SAMP_IO_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const size_t head_bytes = (2 * rows * nl + rows) * 4;
    const bool staged = io == SAMP_IO_HOST && out && head != SAMP_HEAD_NONE && (out->logits || out->probs || out->labels);
    if (out) {
      if (out->hidden) SAMP_CUDA(cudaMemcpyAsync(out->hidden, a.hid_f32, size_t(T) * H * 4, kind, st));
      if (staged) {   // the three head outputs are contiguous on the device: one D2H
        if (e->pinned_out_cap < head_bytes) {
          if (e->pinned_out) cudaFreeHost(e->pinned_out);
          e->pinned_out = nullptr;   // a failed allocation below must not leave a freed pointer
          e->pinned_out_cap = 0;
          const size_t cap = std::max<size_t>(head_bytes, 1 << 16);
          SAMP_CUDA(cudaMallocHost(&e->pinned_out, cap));
          e->pinned_out_cap = cap;
        }
        SAMP_CUDA(cudaMemcpyAsync(e->pinned_out, a.headbuf, head_bytes, cudaMemcpyDeviceToHost, st));
      } else if (head != SAMP_HEAD_NONE) {
        if (out->logits) SAMP_CUDA(cudaMemcpyAsync(out->logits, a.logits, rows * nl * 4, kind, st));
        if (out->probs) SAMP_CUDA(cudaMemcpyAsync(out->probs, a.probs, rows * nl * 4, kind, st));
        if (out->labels) SAMP_CUDA(cudaMemcpyAsync(out->labels, a.labels, rows * 4, kind, st));
      }
    }
    if (io == SAMP_IO_HOST) SAMP_CUDA(cudaStreamSynchronize(st));
    if (g_gelu_flags && env_flag("SAMP_GELU_FLAGS")) {
      SAMP_CUDA(cudaDeviceSynchronize());
      std::fprintf(stderr, "gelu_fast: %llu flagged 8-groups of %lld\n", *g_gelu_flags,
                   (long long)T * d.intermediate / 8 * d.num_layers);
      *g_gelu_flags = 0;
    }
    if (staged) {
      if (out->logits) std::memcpy(out->logits, e->pinned_out, rows * nl * 4);
      if (out->probs) std::memcpy(out->probs, e->pinned_out + rows * nl, rows * nl * 4);
      if (out->labels) std::memcpy(out->labels, e->pinned_out + 2 * rows * nl, rows * 4);
    }
  });
}
