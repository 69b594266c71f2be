/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Linked by nothing in the product; loaded
 * by oracle/samp_oracle.py, which only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may import.
 *
 * CPU restatement of the two float32 transcendental kernels the reference's
 * arithmetic depends on, so the oracle is bit-identical to the reference's
 * numpy on any host CPU:
 *
 *   np.exp (float32)  — numpy's AVX512F/FMA3 "simd_exp_f32": clamp,
 *                        Cody-Waite reduction by ln2 (hi/lo), 5/2-degree
 *                        rational approximation, scalef by 2^k.
 *                        Used by softmax_rows (reference: pkg/src/samp/kernels.py:134).
 *   np.tanh (float32) — Intel SVML __svml_tanhf16 (numpy's AVX512_SKX dispatch):
 *                        32-interval table of degree-6 polynomials in |x|-b.
 *                        Used by gelu (reference: pkg/src/samp/kernels.py:160-161).
 *
 * Pinned: both functions equal np.exp / np.tanh bit-for-bit over all 2^32
 * float32 inputs on the build container (AVX512 Xeon, numpy 2.3.5); the
 * sweep is recorded in DESIGN.md and sampled by tests/test_oracle.py.
 * Compile WITHOUT fp contraction (-ffp-contract=off): every fmaf below is an
 * explicit fused op, everything else must round separately.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "svml_tanh_table.h"

static inline float bits_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t f_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

float npm_expf(float x) {
    const float hi_cut = 88.72283935546875f, lo_cut = -103.97208404541015625f;
    if (x != x) return x;
    if (x >= hi_cut) return INFINITY;
    if (x <= lo_cut) return 0.0f;
    const float magic = 0x1.800000p+23f;
    float k = x * 1.442695040888963407359924681001892137f;
    k = (k + magic) - magic;                       /* round to nearest int */
    float r = fmaf(k, -6.93145752e-1f, x);         /* Cody-Waite, ln2 high */
    r = fmaf(k, -1.42860677e-6f, r);               /* ln2 low */
    r = fmaf(k, 0.0f, r);
    float num = fmaf(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = fmaf(num, r, 5.114512081637298353406e-02f);
    num = fmaf(num, r, 2.473615434895520810817e-01f);
    num = fmaf(num, r, 7.257664613233124478488e-01f);
    num = fmaf(num, r, 9.999999999980870924916e-01f);
    float den = fmaf(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = fmaf(den, r, 1.0f);
    return ldexpf(num / den, (int)k);
}

float npm_tanhf(float x) {
    uint32_t u = f_bits(x);
    uint32_t sign = u & 0x80000000u;
    int32_t key = (int32_t)(u & 0x7fe00000u);
    if (key > 0x7f000000) {                        /* huge, inf or nan */
        if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return x + x;
        return sign ? -1.0f : 1.0f;
    }
    int32_t t = key - 0x3d400000;
    t = t < 0 ? 0 : (t > 0x03e00000 ? 0x03e00000 : t);
    int i = t >> 21;
    float r = bits_f(u & 0x7fffffffu) - bits_f(SVML_TANH_B[i]);
    float p = fmaf(bits_f(SVML_TANH_C6[i]), r, bits_f(SVML_TANH_C5[i]));
    p = fmaf(p, r, bits_f(SVML_TANH_C4[i]));
    p = fmaf(p, r, bits_f(SVML_TANH_C3[i]));
    p = fmaf(p, r, bits_f(SVML_TANH_C2[i]));
    p = fmaf(p, r, bits_f(SVML_TANH_C1[i]));
    p = fmaf(p, r, bits_f(SVML_TANH_C0[i]));
    return bits_f(f_bits(p) | sign);
}

void npm_exp_array(const float* x, float* y, long n) {
    for (long i = 0; i < n; ++i) y[i] = npm_expf(x[i]);
}

void npm_tanh_array(const float* x, float* y, long n) {
    for (long i = 0; i < n; ++i) y[i] = npm_tanhf(x[i]);
}
