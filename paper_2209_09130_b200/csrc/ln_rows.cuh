// Row LayerNorm over split-K int32 accumulators (small batches: the out-projection and
// FFN2 GEMMs run split-K into an int32 workspace, EpiSplitKAdd, then this kernel finishes
// each row).  Same arithmetic, in the same order, as the fused EpiResLN epilogue
// (reference encoder.py:381-385 / :412-418, kernels.layernorm :138-154):
//   x = (F32(acc)*mult + bias) + F32(res)*s_res
//   mean = (0 + pairwise(x)) / H;  var = (0 + pairwise((x - mean)^2)) / H
//   y = ((x - mean) * (1 / sqrt(var + eps))) * gamma + beta  ->  quantize(s_out)
// One warp per row; numpy's tree by embed.cuh's uniform-leaf warp reduction (the same tree
// EpiResLN evaluates per column half and cluster rank).  The workspace row is zeroed after
// it is read, ready for the next split-K accumulation.
#pragma once
#include "embed.cuh"

namespace samp {

struct LnRowsParams {
  int* ws;               // [M][H] int32 accumulators (zeroed after use)
  const int8_t* res_i8;  // [M][H] residual codes
  float res_scale;
  const float* bias;
  const float* gamma;
  const float* beta;
  float mult, eps;
  int M;
  int8_t* out_i8;        // [M][H]
  float s_out;
};

constexpr int LNR_THREADS = 256;   // 8 rows per block

#ifdef SAMP_DEFINE_KERNELS
template <int H>
static __global__ void __launch_bounds__(LNR_THREADS) ln_rows_kernel(const LnRowsParams p) {
  static_assert(EmbLeaves<H>::uniform, "uniform numpy leaves");
  extern __shared__ float lrow[];   // [8][EmbLeaves<H>::ROW]
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * (LNR_THREADS / 32) + warp;
  if (t >= p.M) return;
  float* row = lrow + warp * EmbLeaves<H>::ROW;
  const size_t base = size_t(t) * H;
  for (int c = lane * 4; c < H; c += 128) {
    int4* wsp = reinterpret_cast<int4*>(p.ws + base + c);
    const int4 a = *wsp;
    *wsp = make_int4(0, 0, 0, 0);
    const uint32_t rc = *reinterpret_cast<const uint32_t*>(p.res_i8 + base + c);
    const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + c));
    const int av[4] = {a.x, a.y, a.z, a.w};
    const float bv[4] = {b.x, b.y, b.z, b.w};
    float x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float res = deq(int(int8_t((rc >> (8 * u)) & 0xff)), p.res_scale);
      x[u] = __fadd_rn(__fadd_rn(__fmul_rn(__int2float_rn(av[u]), p.mult), bv[u]), res);
    }
    *reinterpret_cast<float4*>(row + emb_pad<H>(c)) = make_float4(x[0], x[1], x[2], x[3]);
  }
  __syncwarp();
  auto at = [&](int i) { return row[emb_pad<H>(i)]; };
  const float hf = float(H);
  auto vx = [&](int i) { return at(i); };
  const float mean = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp_uniform<H>(vx)), hf);
  auto vc = [&](int i) {
    const float d = __fsub_rn(at(i), mean);
    return __fmul_rn(d, d);
  };
  const float var = __fdiv_rn(__fadd_rn(0.0f, pairwise_warp_uniform<H>(vc)), hf);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
  const Recip rq = make_recip(p.s_out);
  for (int c = lane * 4; c < H; c += 128) {
    const float4 xv = *reinterpret_cast<const float4*>(row + emb_pad<H>(c));
    const float4 gv = __ldg(reinterpret_cast<const float4*>(p.gamma + c));
    const float4 bv = __ldg(reinterpret_cast<const float4*>(p.beta + c));
    const float xx[4] = {xv.x, xv.y, xv.z, xv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
    float q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      q[u] = quant_pre_fast(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xx[u], mean), inv), gg[u]), bb[u]), rq);
    *reinterpret_cast<uint32_t*>(p.out_i8 + base + c) = trunc_pack4_s8(q[0], q[1], q[2], q[3]);
  }
}
#endif  // SAMP_DEFINE_KERNELS

}  // namespace samp
