// bwm_kernel_masked.cuh — masked-NaN BFAST-monitor kernel (nan_mode = mask).
//
// The reference fills gaps before fitting (engine.py:305-319).  In masked mode every pixel
// is instead fitted on its OWN valid history dates and monitored over its compacted valid
// series (the per-pixel restatement in oracle/bfast_oracle.py:monitor_masked):
//   beta   = (X_v X_v^T)^-1 X_v y_v over the valid history dates     (model.py:118-152 per pixel)
//   sigma  = sqrt(RSS / (n_v - p))                                     (engine.py:363-371, dof n_v - p)
//   MOSUM over the compacted residuals with n_v, h_v = floor(h n_v / n) (_kernels.py:21-34)
//   b_j    = lambda sqrt(log_plus((n_v + 1 + j) / n_v))                (mosum.py:68-79 with n = n_v)
//   first_break = original 1-based date of the first crossing window's last element.
// A pixel is invalid when n_v <= p, h_v < 1, it has no valid monitoring date or its valid
// history design is (numerically) singular.  On NaN-free input this is exactly fill mode.
//
// Layout: one pixel per thread (128-pixel tiles, 128 threads), predicated scalar loads, so
// tails and any row stride run the same code.  FFMA2 packs coefficient PAIRS of one pixel.
// Pass 1 (history): g = X' (y - c) with 2Sum-compensated 32-date blocks, and the Gram
//   complement Gm = sum over MISSING history dates of x_t x_t^T (x_t x_t^T from a table,
//   lower triangle); G_v = G_full - Gm is accurate because Gm has few terms, and whole
//   warps skip dates on which none of their 32 pixels is missing (clustered clouds).
// Solve: float64 Cholesky of G_v per pixel (in registers), beta' = G_v^-1 g.
// Pass 2 (history again, L2): two-pass RSS of the valid dates; the last h_v - 1 valid
//   residuals (and their dates) go to a per-pixel ring (slot 0 = 0: the element before
//   window 0).  The same sweep accumulates the normal-equation residual e = X_v r, and one
//   step of mixed-precision iterative refinement follows: dbeta = G_v^-1 e, RSS and the ring
//   residuals are corrected in place (RSS' = RSS - 2 dbeta.e + |L^T dbeta|^2).  This makes
//   the float32 Gram good to cond(G_v) ~ 1e5 (p = 18 on 23 valid dates: cond 3e4) at the cost
//   of p/2 FFMA2 per valid history date; realistic stacks have cond(G_v) < 10.
// Pass 3 (monitoring): per valid date r, old = ring[s], ring[s] = r, acc += r - old,
//   crossing |acc| > b_j sigma sqrt(n_v); invalid dates leave the state untouched.
// The ring is [h][128] floats + [h][128] dates (conflict-free: thread = bank); in shared
// memory, or in a per-CTA global scratch when h or the x x^T table is too large (BIG).
#pragma once

#include "bwm_common.cuh"

namespace bwm {

constexpr int kMaskThreads = 128;       // one pixel per thread
constexpr int kMaskTile = kMaskThreads;
constexpr int kMaskD = 16;              // dates per register block

template <int NP>
struct Gram {
    static constexpr int KK = NP * (NP + 1) / 2;          // lower triangle, (i, j<=i) at i(i+1)/2 + j
    static constexpr int K2 = (KK + 1) / 2;               // float2 accumulators
    static constexpr int KP = ((2 * K2 + 3) / 4) * 4;     // padded table row (floats)
};

// Shared-memory bytes of the masked kernel (host mirror in bwm_capi.cu).
__host__ __device__ inline int64_t masked_smem_bytes(int N, int n, int h, int p, bool big) {
    const int sp = (p + 3) & ~3;
    const int kk = p * (p + 1) / 2, kp = (((kk + 1) / 2 * 2 + 3) / 4) * 4;
    const int n16 = ((n + kMaskD - 1) / kMaskD) * kMaskD;
    int64_t bytes = (int64_t)(N + kMaskD) * sp * 4;       // X'^T, zero rows past N
    if (!big) bytes += (int64_t)n16 * kp * 4 + (int64_t)h * kMaskThreads * 8;
    return bytes;
}

template <int NP, bool BIG>
__global__ void __launch_bounds__(kMaskThreads, NP <= 8 ? 4 : 2)
    monitor_kernel_masked(const __grid_constant__ KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int KK = Gram<NP>::KK, K2 = Gram<NP>::K2, KP = Gram<NP>::KP;
    constexpr int D = kMaskD;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const int n16 = ((n + D - 1) / D) * D;
    float* s_x = reinterpret_cast<float*>(smem_raw);                   // [N + D][SP]   X'^T
    float* s_xx = s_x + (N + D) * SP;                                  // [n16][KP]     x x^T (!BIG)
    float* s_ring = s_xx + n16 * KP;                                   // [2][h][128]   (!BIG)
    for (int i = threadIdx.x; i < (N + D) * SP; i += kMaskThreads) s_x[i] = i < N * SP ? prm.xt[i] : 0.f;
    if (!BIG)
        for (int i = threadIdx.x; i < n16 * KP; i += kMaskThreads) s_xx[i] = i < n * KP ? prm.xx[i] : 0.f;
    __syncthreads();
    const float* xx = BIG ? prm.xx : s_xx;      // BIG: the padded table lives in global memory
    float* ring = (BIG ? prm.ring_g + (int64_t)blockIdx.x * 2 * h * kMaskThreads : s_ring) + threadIdx.x;
    int* ring_d = reinterpret_cast<int*>(ring + h * kMaskThreads);   // date of each ring entry

    const int tid = threadIdx.x;
    const int64_t ld = prm.ld_y;
    const float lam = prm.lambda;
    const float kE = 2.718281828459045f;
    const int64_t n_tiles = (prm.n_pixels + kMaskTile - 1) / kMaskTile;

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t px = tile * kMaskTile + tid;
        const bool act = px < prm.n_pixels;
        const float* yp = prm.y + (act ? px : 0);
        auto load = [&](int t, int end) -> float {
            return (act && t < end) ? __ldg(yp + (int64_t)t * ld) : __int_as_float(0x7fc00000);
        };

        // ---- pass 0: centre c = first finite value (any finite value would do numerically) -
        float c = 0.f;
        for (int t = 0; t < N && act; ++t) {
            const float v = __ldg(yp + (int64_t)t * ld);
            if (finitef(v)) { c = v; break; }
        }

        // ---- pass 1: g = X'(y - c) over valid dates; Gm over missing dates ---------------
        float2 gm[K2], gp[NP / 2], ghi[NP / 2], glo[NP / 2];
#pragma unroll
        for (int i = 0; i < K2; ++i) gm[i] = f2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) gp[i] = ghi[i] = glo[i] = f2(0.f, 0.f);
        int nv = 0;
        for (int t0 = 0; t0 < n; t0 += D) {
            float vb[D];
#pragma unroll
            for (int k = 0; k < D; ++k) vb[k] = load(t0 + k, n);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int t = t0 + k;
                const bool m = finitef(vb[k]);
                const float yc = m ? vb[k] - c : 0.f;
                nv += m ? 1 : 0;
                const float4* x4 = reinterpret_cast<const float4*>(s_x + t * SP);
#pragma unroll
                for (int q = 0; q < SP / 4; ++q) {
                    const float4 x = x4[q];
                    if (4 * q + 1 < NP) gp[2 * q] = fma2(f2(yc, yc), f2(x.x, x.y), gp[2 * q]);
                    if (4 * q + 3 < NP) gp[2 * q + 1] = fma2(f2(yc, yc), f2(x.z, x.w), gp[2 * q + 1]);
                }
                // rows t >= n carry NaN (missing) but their table rows are zero: no-ops
                if (__any_sync(0xffffffffu, !m)) {
                    const float w = m ? 0.f : 1.f;
                    const float4* r4 = reinterpret_cast<const float4*>(xx + (int64_t)t * KP);
#pragma unroll
                    for (int q = 0; q < KP / 4; ++q) {
                        const float4 a = BIG ? __ldg(r4 + q) : r4[q];
                        if (2 * q < K2) gm[2 * q] = fma2(f2(w, w), f2(a.x, a.y), gm[2 * q]);
                        if (2 * q + 1 < K2) gm[2 * q + 1] = fma2(f2(w, w), f2(a.z, a.w), gm[2 * q + 1]);
                    }
                }
            }
            if (((t0 + D) & (kComp - 1)) == 0 || t0 + D >= n) {
#pragma unroll
                for (int i = 0; i < NP / 2; ++i) { two_sum(ghi[i], glo[i], gp[i]); gp[i] = f2(0.f, 0.f); }
            }
        }

        // ---- solve G_v beta' = g in float64 (Cholesky, in registers) --------------------
        double L[KK];
#pragma unroll
        for (int i = 0; i < KK; ++i) {
            const float gmi = (i & 1) ? gm[i >> 1].y : gm[i >> 1].x;
            L[i] = __ldg(prm.gfull + i) - (double)gmi;
        }
        bool ok = nv > NP;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int jj = j * (j + 1) / 2 + j;
            double d = L[jj];
#pragma unroll
            for (int k = 0; k < j; ++k) d -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
            ok = ok && d > 1e-9 * fabs(L[jj]) && d > 0.0;
            const double inv = ok ? rsqrt(d) : 0.0;
            L[jj] = ok ? d * inv : 1.0;          // L_jj
#pragma unroll
            for (int i = j + 1; i < NP; ++i) {
                double s = L[i * (i + 1) / 2 + j];
#pragma unroll
                for (int k = 0; k < j; ++k) s -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
                L[i * (i + 1) / 2 + j] = s * inv;
            }
        }
        double z[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const float2 gg = ghi[i >> 1], gl = glo[i >> 1];
            double s = (i & 1) ? (double)gg.y + (double)gl.y : (double)gg.x + (double)gl.x;
#pragma unroll
            for (int k = 0; k < i; ++k) s -= L[i * (i + 1) / 2 + k] * z[k];
            z[i] = s / L[i * (i + 1) / 2 + i];
        }
#pragma unroll
        for (int i = NP - 1; i >= 0; --i) {
            double s = z[i];
#pragma unroll
            for (int k = i + 1; k < NP; ++k) s -= L[k * (k + 1) / 2 + i] * z[k];
            z[i] = s / L[i * (i + 1) / 2 + i];
        }
        float2 nb[NP / 2];    // -beta' in coefficient pairs
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) nb[i] = ok ? f2(-(float)z[2 * i], -(float)z[2 * i + 1]) : f2(0.f, 0.f);
        float Lf[KK];         // the factor, kept (float32) for the refinement step
#pragma unroll
        for (int i = 0; i < KK; ++i) Lf[i] = (float)L[i];
        auto resid = [&](float yc, int t) -> float {
            float2 r2 = f2(yc, 0.f);
            const float4* x4 = reinterpret_cast<const float4*>(s_x + t * SP);
#pragma unroll
            for (int q = 0; q < SP / 4; ++q) {
                const float4 x = x4[q];
                if (4 * q + 1 < NP) r2 = fma2(nb[2 * q], f2(x.x, x.y), r2);
                if (4 * q + 3 < NP) r2 = fma2(nb[2 * q + 1], f2(x.z, x.w), r2);
            }
            return r2.x + r2.y;
        };

        // ---- pass 2: RSS (two-pass) and the history part of window 0 -----------------------
        const int hv = (int)(((int64_t)h * nv) / n);
        const int wfirst = nv - hv + 1;          // 0-based compacted index of window 0's first element
        int seen = 0, slot = 1;
        double rss = 0.0;
        float2 e2[NP / 2];                       // X_v r (normal-equation residual)
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) e2[i] = f2(0.f, 0.f);
        if (hv >= 1) ring[0] = 0.f;              // the element before window 0
        for (int t0 = 0; t0 < n; t0 += D) {
            float vb[D];
#pragma unroll
            for (int k = 0; k < D; ++k) vb[k] = load(t0 + k, n);
            float part = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int t = t0 + k;
                const bool m = finitef(vb[k]);
                const float r = resid(m ? vb[k] - c : 0.f, t);
                const float rm = m ? r : 0.f;
                part = fmaf(rm, rm, part);
                const float4* x4 = reinterpret_cast<const float4*>(s_x + t * SP);
#pragma unroll
                for (int q = 0; q < SP / 4; ++q) {
                    const float4 x = x4[q];
                    if (4 * q + 1 < NP) e2[2 * q] = fma2(f2(rm, rm), f2(x.x, x.y), e2[2 * q]);
                    if (4 * q + 3 < NP) e2[2 * q + 1] = fma2(f2(rm, rm), f2(x.z, x.w), e2[2 * q + 1]);
                }
                if (m) {
                    if (seen >= wfirst) {
                        ring[slot * kMaskThreads] = r;
                        ring_d[slot * kMaskThreads] = t;
                        ++slot;
                    }
                    ++seen;
                }
            }
            rss += (double)part;
        }

        // ---- one refinement step: dbeta = G_v^-1 e; correct RSS and the window residuals ---
        float db[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            float sv = (i & 1) ? e2[i >> 1].y : e2[i >> 1].x;
#pragma unroll
            for (int k = 0; k < i; ++k) sv -= Lf[i * (i + 1) / 2 + k] * db[k];
            db[i] = sv / Lf[i * (i + 1) / 2 + i];            // L w = e
        }
        double quad = 0.0;                                  // |L^T dbeta|^2 = |w|^2
#pragma unroll
        for (int i = 0; i < NP; ++i) quad += (double)db[i] * (double)db[i];
#pragma unroll
        for (int i = NP - 1; i >= 0; --i) {
            float sv = db[i];
#pragma unroll
            for (int k = i + 1; k < NP; ++k) sv -= Lf[k * (k + 1) / 2 + i] * db[k];
            db[i] = sv / Lf[i * (i + 1) / 2 + i];            // L^T dbeta = w
        }
        double de = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) de += (double)db[i] * (double)((i & 1) ? e2[i >> 1].y : e2[i >> 1].x);
        if (ok) {
            rss = fmax(rss - 2.0 * de + quad, 0.0);
#pragma unroll
            for (int i = 0; i < NP / 2; ++i) nb[i] = sub2(nb[i], f2(db[2 * i], db[2 * i + 1]));
        }
        float acc = 0.f;
        for (int s2 = 1; s2 < slot; ++s2) {
            const int t = ring_d[s2 * kMaskThreads];
            const float* xr = s_x + t * SP;
            float r = ring[s2 * kMaskThreads];
#pragma unroll
            for (int i = 0; i < NP; ++i) r = fmaf(-db[i], xr[i], r);
            ring[s2 * kMaskThreads] = r;
            acc += r;
        }
        const float ss = ok ? (float)rss : 0.f;
        const bool fit_ok = ok && hv >= 1;
        const bool zero = fit_ok && ss == 0.f && c == 0.f;
        if (zero) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px));
        const float sc = fit_ok ? sqrtf(ss / (float)(nv - NP)) * sqrtf((float)nv) : 0.f;
        const float inv = sc > 0.f ? 1.0f / sc : 0x1p100f;
        const float lam_sc = lam * sc;
        const float inv_nv = fit_ok ? 1.0f / (float)nv : 0.f;

        // ---- pass 3: compacted MOSUM + per-pixel boundary ----------------------------------
        float mx = 0.f, msum = 0.f;
        int first = 0, j = 0;
        slot = 0;
        float* const mo_out = prm.mosum;
        for (int t0 = n; t0 < N; t0 += D) {
            float vb[D];
#pragma unroll
            for (int k = 0; k < D; ++k) vb[k] = load(t0 + k, N);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int t = t0 + k;
                const bool m = finitef(vb[k]) && fit_ok;
                const float r = resid(m ? vb[k] - c : 0.f, t);
                if (m) {
                    const float old = ring[slot * kMaskThreads];
                    ring[slot * kMaskThreads] = r;
                    slot = slot + 1 == hv ? 0 : slot + 1;
                    acc += r - old;
                    const float x = (float)(nv + 1 + j) * inv_nv;
                    const float b = lam_sc * sqrtf(__logf(fmaxf(x, kE)));
                    const float a = fabsf(acc);
                    mx = fmaxf(mx, a);
                    if (a > b && first == 0) first = t + 1 - n;
                    msum += acc;
                    ++j;
                }
                if (mo_out && act && t < N)
                    mo_out[(int64_t)(t - n) * prm.ld_out + px] = m ? acc * inv : __int_as_float(0x7fc00000);
            }
        }

        // ---- outputs ------------------------------------------------------------------------
        if (act) {
            const bool valid = fit_ok && j >= 1;
            prm.valid[px] = valid;
            prm.first_idx[px] = valid ? first : 0;
            prm.max_abs[px] = valid ? mx * inv : 0.f;
            if (prm.mo_mean) prm.mo_mean[px] = valid ? msum * inv / (float)j : 0.f;
            if (prm.beta) {
                // raw basis (bwm.h): b0 = c + b0' - b1' tc/ts, b1 = b1'/ts
                const float b0 = -nb[0].x, b1 = -nb[0].y;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    float b = (i & 1) ? -nb[i >> 1].y : -nb[i >> 1].x;
                    if (i == 0) b = (float)((double)c + (double)b0 - (double)b1 * (double)prm.tc_ts);
                    if (i == 1) b = b1 * prm.inv_ts;
                    prm.beta[(int64_t)i * prm.ld_out + px] = valid ? b : 0.f;
                }
            }
        }
    }
}

}  // namespace bwm
