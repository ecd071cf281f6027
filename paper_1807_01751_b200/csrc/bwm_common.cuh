// bwm_common.cuh — shared definitions of the BFAST-monitor kernels (sm_100a).
//
// Numerics: plain float32 accumulation of beta fails rtol 1e-4 on the
// MOSUM magnitude.  Three cheap changes fix it (emulated error <= 6e-6 relative):
//   * y is centred on the pixel's first finite value c (the intercept absorbs it, and the
//     leading back-fill becomes exactly 0);
//   * the trend regressor is centred/scaled on the host (M', X': a reparametrisation that
//     leaves fitted values unchanged in exact arithmetic);
//   * 32-date FFMA2 block partials are 2Sum-compensated into (hi, lo).
#pragma once
#include <cuda.h>
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bwm {

constexpr int kThreads = 128;
constexpr int kTile = 2 * kThreads;   // pixels per CTA tile
constexpr int kDepth = 16;            // LDG kernel: prefetch depth == compensation block (dates)
#ifndef BWM_COMP
#define BWM_COMP 32
#endif
constexpr int kComp = BWM_COMP;       // dates per 2Sum-compensated block partial (emulated 1e-5 at 32)

struct KParams {
    CUtensorMap tmap;           // TMA kernel: 2-D map of y (pixels x dates), box 64 px x 8 dates
    const float* y;             // this launch's pixel 0, row stride ld_y (elements)
    int64_t ld_y;
    int64_t n_pixels;
    int64_t pixel_offset;       // global index of pixel 0 (zero-sigma reporting)
    int N, n, h, sp;            // sp: padded row stride of the coefficient tables
    const float* xt;            // [N][sp]  Z^T = (R^-T X')^T (rows t < n: Q^T), the MMA kernel's table
    const float* rinv;          // [p][p]   R^-1 (row-major): beta' = R^-1 beta_Q (beta output)
    const float* bound;         // [N-n]
    float inv_dof;              // 1 / (n - p)
    float sqrt_n;
    int ring_rows;              // TMEM ring: L (multiple of 8, >= h); rows L..L+7 mirror 0..7
    int tmem_cols;              // TMEM columns allocated per CTA (power of 2 >= 32)
    float tc_ts;                // trend_center / trend_scale
    float inv_ts;               // 1 / trend_scale
    uint8_t* valid;
    int32_t* first_idx;
    float* max_abs;
    float* beta;
    float* mo_mean;
    float* mosum;
    float* sup;                 // [P] or nullptr: sup_j |MO_j| / bound_j (critical_value statistic)
    int64_t ld_out;
    unsigned long long* zero_sigma;   // atomicMin target (int64 bit pattern, non-negative)
    // masked-NaN mode (bwm_kernel_masked.cuh); xt then holds X'^T (the centred raw design)
    const float* xx;            // [n16][KP] x_t x_t^T lower triangles of the history dates, zero padded
    const double* gfull;        // [KK] sum of those rows over the whole history
    float* ring_g;              // per-CTA residual rings [grid][h][128] when they live in global memory
    float lambda;               // crit = bound[0]
    double gscale;              // exact-digit Gram complement: Gm = gscale * (D_hi + D_lo / 2048)
    // long monitoring horizons (LDG kernel): fitted values in float64 from this [N][sp] table
    // (Z^T in double) and the compensated beta_Q, so the trend extrapolation keeps 1e-4
    const double* xtd;          // nullptr: float32 fitted values (the default)
    // ill-conditioned pixels (||y-c||^2 > fix_ratio * RSS) are listed for the float64 fixup
    // (bwm_fixup.cu); list entries are pixel indices of the bwm_monitor call (launch + fix_base)
    int64_t* fix_list;          // nullptr: no fixup
    unsigned int* fix_count;
    unsigned int fix_cap;       // list capacity; pixels past it keep their float32 result
    float fix_ratio;
    int64_t fix_base;
    // tensor-core fitted values (bwm_kernel_mma.cuh): Z^T split into tf32 hi/lo B tables
    const float* zb_cur;        // current dates [w0, ...)
    const float* zb_lag;        // lag dates [t3 - h, ...)
    // window-sum formulation (TMA and LDG kernels): the MOSUM window sum of residuals is
    //   sum_{s in window(t)} r_s = sum_{s in window(t)} (y_s - c) - S_t^T beta_Q,
    //   S_t = sum_{s in window(t)} z_s  (host, float64),
    // linear in y, so the monitoring pass carries the window sum of the FILLED series and one
    // dot with S_t per date, and neither the lagged date nor window 0 needs a fitted value.
    // Design row 0 is the intercept, so z_t[0] = 1/R00 for every t and S_t[0] = s0 = h/R00:
    // that part enters the initial window sum once, in float64 (it also centres the running
    // sum on the history mean), and the per-date dot covers k >= 1.
    const float* wt;            // [N][sp] rows t < n: q_t (Q^T); rows t >= n: S_t (column 0 = 0)
    const double* wtd;          // the same table in float64 (precise mode), or nullptr
    double s0;                  // h * z[0]
    // TMA kernel: dynamic per-warp slice scheduler ([0] claim counter, [1] finished warps; the
    // last warp to finish resets both, so every launch starts from 0) — nullptr: static schedule
    unsigned int* sched;
    int sched_jit;              // 1: claim each slice when the cursor reaches it (long slices: no pre-claimed
                                // slice waits behind a busy warp at the end of the launch)
};

// append pixel `px` (launch-relative) to the fixup list when its history fit is ill-conditioned:
// ||y-c||^2 > ratio * RSS, or a one-pass RSS that cancelled to <= 0 (clamped to 0 by
// rss_onepass) on a history that is not constant — the worst-conditioned, near-noiseless
// pixels; the float64 fixup recomputes sigma with the reference's two-pass sum.
__device__ __forceinline__ void fix_flag(const KParams& prm, bool valid, double q, float rss, int64_t px) {
    if (prm.fix_list && valid && q > 0.0 && (rss == 0.f || q > (double)prm.fix_ratio * (double)rss)) {
        const unsigned int i = atomicAdd(prm.fix_count, 1u);
        if (i < prm.fix_cap) prm.fix_list[i] = prm.fix_base + px;
    }
}

// zero-sigma contract (engine.py:373-378): the reference raises when float64 gives sigma == 0
// exactly, i.e. for an identically zero filled history: ||y - c||^2 == 0 with c == 0.  A
// one-pass RSS that merely cancels to 0 on a varying history is not zero sigma (fix_flag).
__device__ __forceinline__ bool zero_history(bool valid, double q, float c) { return valid && q == 0.0 && c == 0.f; }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, f2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fma2s(float2 a, float s, float2 c) { return __ffma2_rn(a, f2(s, s), c); }
__device__ __forceinline__ bool finitef(float v) { return fabsf(v) < __int_as_float(0x7f800000); }

// One date of this thread's pixel pair.  Fast path: both pixels exist and the address is
// 8-byte aligned.  SAFE path (tail tile or odd row stride): scalar, bounds-checked loads.
template <bool SAFE>
__device__ __forceinline__ float2 ldp(const float* __restrict__ p, int npx) {
    if (!SAFE) return __ldg(reinterpret_cast<const float2*>(p));
    if (npx >= 2) return f2(__ldg(p), __ldg(p + 1));
    if (npx == 1) return f2(__ldg(p), 0.f);
    return f2(0.f, 0.f);
}

// Forward fill in the centred frame: missing -> previous filled value.  `last` starts
// at 0, i.e. at c, which is exactly the reference's leading back-fill (engine.py:316-317).
__device__ __forceinline__ float2 fill(float2 v, float2 negc, float2& last) {
    float2 vc = add2(v, negc);
    vc.x = finitef(v.x) ? vc.x : last.x;
    vc.y = finitef(v.y) ? vc.y : last.y;
    last = vc;
    return vc;
}

// hi + lo += b, error-free transformation (Knuth 2Sum).
__device__ __forceinline__ void two_sum(float2& hi, float2& lo, float2 b) {
    const float2 s = add2(hi, b);
    const float2 bb = sub2(s, hi);
    const float2 e = add2(sub2(hi, sub2(s, bb)), sub2(b, bb));
    hi = s;
    lo = add2(lo, e);
}

// r + sum_i nb_i * x_i   (x: one date's row of the design table in smem)
template <int NP, int SP>
__device__ __forceinline__ float2 dot_row(float2 r, const float* __restrict__ xrow, const float2 (&nb)[NP]) {
    const float4* x4 = reinterpret_cast<const float4*>(xrow);
#pragma unroll
    for (int q = 0; q < SP / 4; ++q) {
        const float4 x = x4[q];
        if (4 * q + 0 < NP) r = fma2s(nb[4 * q + 0], x.x, r);
        if (4 * q + 1 < NP) r = fma2s(nb[4 * q + 1], x.y, r);
        if (4 * q + 2 < NP) r = fma2s(nb[4 * q + 2], x.z, r);
        if (4 * q + 3 < NP) r = fma2s(nb[4 * q + 3], x.w, r);
    }
    return r;
}

// Numerator of MO_t in the window-sum formulation: acc + sum_{k >= 1} nb_k * S_t[k]
// (nb = -beta_Q; S_t[0] is folded into acc).  Same FFMA2 chain order as dot_row.
template <int NP, int SP>
__device__ __forceinline__ float2 wsum_row(float2 acc, const float* __restrict__ srow, const float2 (&nb)[NP]) {
    const float4* s4 = reinterpret_cast<const float4*>(srow);
#pragma unroll
    for (int q = 0; q < SP / 4; ++q) {
        const float4 s = s4[q];
        if (q > 0 && 4 * q + 0 < NP) acc = fma2s(nb[4 * q + 0], s.x, acc);
        if (4 * q + 1 < NP) acc = fma2s(nb[4 * q + 1], s.y, acc);
        if (4 * q + 2 < NP) acc = fma2s(nb[4 * q + 2], s.z, acc);
        if (4 * q + 3 < NP) acc = fma2s(nb[4 * q + 3], s.w, acc);
    }
    return acc;
}

// Initial window sum (window of date n minus its newest date: dates [n-h, n), h of them) minus
// the intercept part s0 * beta_Q[0], in float64 — the ỹ sum w and beta_Q[0] = hi + lo are
// large and nearly equal after a level shift, their difference is the residual window sum.
__device__ __forceinline__ float2 wsum_init(double w0, double w1, float2 hi0, float2 lo0, double s0) {
    return f2((float)(w0 - s0 * ((double)hi0.x + (double)lo0.x)), (float)(w1 - s0 * ((double)hi0.y + (double)lo0.y)));
}

// r = y_c - z^T beta_Q with z from the float64 table and beta_Q = hi + lo in float64 (precise mode)
template <int NP, int SP>
__device__ __forceinline__ float2 resid_f64(float2 vc, const double* __restrict__ zrow, const double (&b0)[NP],
                                            const double (&b1)[NP]) {
    double r0 = (double)vc.x, r1 = (double)vc.y;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const double z = __ldg(zrow + i);
        r0 = fma(-z, b0[i], r0);
        r1 = fma(-z, b1[i], r1);
    }
    return f2((float)r0, (float)r1);
}

// part_i += vc * m_i
template <int NP, int SP>
__device__ __forceinline__ void axpy_row(float2 (&part)[NP], float2 vc, const float* __restrict__ mrow) {
    const float4* m4 = reinterpret_cast<const float4*>(mrow);
#pragma unroll
    for (int q = 0; q < SP / 4; ++q) {
        const float4 m = m4[q];
        if (4 * q + 0 < NP) part[4 * q + 0] = fma2s(vc, m.x, part[4 * q + 0]);
        if (4 * q + 1 < NP) part[4 * q + 1] = fma2s(vc, m.y, part[4 * q + 1]);
        if (4 * q + 2 < NP) part[4 * q + 2] = fma2s(vc, m.z, part[4 * q + 2]);
        if (4 * q + 3 < NP) part[4 * q + 3] = fma2s(vc, m.w, part[4 * q + 3]);
    }
}

// Residual sum of squares of the history fit in the orthonormal basis (one pass):
// RSS = ||y_h - c||^2 - ||beta_Q||^2, accumulated in float64 (q from 32-date float32 block
// partials).  Clamped at 0: a (near-)exact fit is a zero-sigma pixel.
template <int NP>
__device__ __forceinline__ float2 rss_onepass(double q0, double q1, const float2 (&bq)[NP]) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        s0 = fma((double)bq[i].x, (double)bq[i].x, s0);
        s1 = fma((double)bq[i].y, (double)bq[i].y, s1);
    }
    return f2((float)fmax(q0 - s0, 0.0), (float)fmax(q1 - s1, 0.0));
}

// beta' = R^-1 beta_Q (centred basis), then the raw basis of the reference (bwm.h):
// b0 = c + b0' - b1' tc/ts, b1 = b1'/ts.  Invalid pixels report 0.
template <int NP>
__device__ __forceinline__ void store_beta(const KParams& prm, int64_t px0, float2 c, const float2 (&bq)[NP],
                                           bool v0, bool v1, int npx) {
    float2 bo[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        float2 a = f2(0.f, 0.f);
#pragma unroll
        for (int j = i; j < NP; ++j) a = fma2s(bq[j], __ldg(prm.rinv + i * NP + j), a);   // R^-1 upper triangular
        bo[i] = a;
    }
    const float2 b1 = bo[1];
    bo[0] = add2(c, sub2(bo[0], mul2(b1, f2(prm.tc_ts, prm.tc_ts))));
    bo[1] = mul2(b1, f2(prm.inv_ts, prm.inv_ts));
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        float* o = prm.beta + (int64_t)i * prm.ld_out + px0;
        if (npx >= 2 && (reinterpret_cast<uintptr_t>(o) & 7) == 0) {
            *reinterpret_cast<float2*>(o) = f2(v0 ? bo[i].x : 0.f, v1 ? bo[i].y : 0.f);
        } else {
            if (npx >= 1) o[0] = v0 ? bo[i].x : 0.f;
            if (npx >= 2) o[1] = v1 ? bo[i].y : 0.f;
        }
    }
}

// Finish a pixel pair after the monitoring pass, in the unscaled frame: the kernel tracks
// max |acc| and the window-sum total; MO = acc / (sigma sqrt n).  sigma == 0 (constant
// history) gives inv = 2^100: every non-zero window then crossed (b * 0 = 0), matching the
// reference's round-off-sigma behaviour, and the reported magnitude is huge.
__device__ __forceinline__ float2 sigma_scale(float2 ss, float inv_dof, float sqrt_n, bool v0, bool v1) {
    const float2 var = mul2(ss, f2(inv_dof, inv_dof));
    return f2(v0 ? sqrtf(var.x) * sqrt_n : 0.f, v1 ? sqrtf(var.y) * sqrt_n : 0.f);
}
__device__ __forceinline__ float2 inv_scale(float2 s) {
    return f2(s.x > 0.f ? 1.0f / s.x : 0x1p100f, s.y > 0.f ? 1.0f / s.y : 0x1p100f);
}

template <int NP>
struct Coefs {
    static constexpr int SP = (NP + 3) & ~3;
};

}  // namespace bwm
