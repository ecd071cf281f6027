// bwm_fixup.cu — float64 re-evaluation of ill-conditioned pixels (fill mode).
//
// The fused kernels compute in float32 (compensated).  Their one-pass residual sum of squares
// RSS = ||y - c||^2 - ||beta_Q||^2 and the fitted values lose digits in proportion to
// ||y - c||^2 / RSS: at realistic noise (C2: ~25-100) the error stays near 1e-5, but on
// near-noiseless series (sigma ~ 1e-3 of a 0.2 seasonal amplitude, ratio ~1e4) max |MO| can
// drift past the 1e-4 tolerance.  The fused kernels therefore append every valid pixel whose
// ratio exceeds `fix_ratio` to a device list, and this kernel recomputes those pixels exactly as
// the reference's fused backend does, in float64 (engine.py:305-411):
//   fill (engine.py:305-319), beta_Q = Q^T (y - c) with the float64 basis, residuals,
//   sigma^2 = sum_{t<n} r^2 / (n - p) (two-pass), the MOSUM recurrence (_kernels.py:21-34) with
//   r_{t-h} recomputed by a lagging cursor, and the strict boundary test (_kernels.py:37-48).
// One thread per listed pixel, grid-stride over the device-side count; columns are read with
// stride ld (uncoalesced, but the list is short on real data).  Outputs first_idx, max_abs and,
// when requested, the MOSUM mean and matrix are overwritten in place.
#include "bwm_common.cuh"

#include <algorithm>

namespace bwm {

constexpr int kFixMaxP = 18;

__global__ void __launch_bounds__(128) fixup_kernel(const KParams prm, int p, const int64_t* __restrict__ list,
                                                    const unsigned int* __restrict__ count) {
    const unsigned int cnt = min(*count, prm.fix_cap);
    const int N = prm.N, n = prm.n, h = prm.h, sp = prm.sp;
    const double* __restrict__ Z = prm.xtd;      // [N][sp] float64 Z^T (rows < n: Q^T)
    const double sqrt_n = sqrt((double)n);
    for (unsigned int w = blockIdx.x * blockDim.x + threadIdx.x; w < cnt; w += gridDim.x * blockDim.x) {
        const int64_t px = list[w];
        const float* y = prm.y + px;
        const int64_t ld = prm.ld_y;
        // centre and leading back-fill: the first finite value (the pixel is valid: one exists)
        double c = 0.0;
        for (int t = 0; t < N; ++t) {
            const float v = y[(int64_t)t * ld];
            if (finitef(v)) { c = (double)v; break; }
        }
        // pass 1: beta_Q over the filled history
        double beta[kFixMaxP];
        for (int i = 0; i < p; ++i) beta[i] = 0.0;
        double last = 0.0;
        for (int t = 0; t < n; ++t) {
            const float v = y[(int64_t)t * ld];
            const double yc = finitef(v) ? (double)v - c : last;
            last = yc;
            for (int i = 0; i < p; ++i) beta[i] = fma(Z[(int64_t)t * sp + i], yc, beta[i]);
        }
        auto resid = [&](double yc, int t) {
            double r = yc;
            for (int i = 0; i < p; ++i) r = fma(-Z[(int64_t)t * sp + i], beta[i], r);
            return r;
        };
        // pass 2: two-pass RSS and window 0 (dates [n-h+1, n-1] here; date n joins below)
        double rss = 0.0, acc = 0.0, lastw = 0.0;
        last = 0.0;
        for (int t = 0; t < n; ++t) {
            const float v = y[(int64_t)t * ld];
            const double yc = finitef(v) ? (double)v - c : last;
            last = yc;
            const double r = resid(yc, t);
            rss = fma(r, r, rss);
            if (t >= n - h + 1) acc += r;
            if (t == n - h) lastw = last;            // fill state of the lagging cursor at n-h
        }
        const double sigma = sqrt(rss / (double)(n - p));
        const double scale = sigma * sqrt_n;
        const double inv = scale > 0.0 ? 1.0 / scale : 0.0;
        // float64 two-pass sigma == 0 on a listed (valid, non-constant) pixel: the reference's
        // ZeroResidualError criterion (engine.py:373-378), decided here rather than from the
        // float32 one-pass RSS that flagged the pixel
        if (!(scale > 0.0)) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px));
        // pass 3: monitoring, r_{t-h} from a lagging cursor with its own fill state
        double mx = 0.0, msum = 0.0, lag_last = lastw, sr = 0.0;
        int first = 0;
        for (int t = n; t < N; ++t) {
            const float v = y[(int64_t)t * ld];
            const double yc = finitef(v) ? (double)v - c : last;
            last = yc;
            const double r = resid(yc, t);
            double old = 0.0;
            if (t > n) {                              // r_{n-h} is outside window 0
                const float lv = y[(int64_t)(t - h) * ld];
                const double lc = finitef(lv) ? (double)lv - c : lag_last;
                lag_last = lc;
                old = resid(lc, t - h);
            }
            acc += r - old;                           // _kernels.py:33 order
            const double mo = acc * inv;
            const double a = fabs(mo);
            mx = fmax(mx, a);
            const double b = (double)prm.bound[t - n];
            if (first == 0 && a > b) first = t - n + 1;   // strict crossing (_kernels.py:47)
            sr = fmax(sr, a / b);
            msum += mo;
            if (prm.mosum) prm.mosum[(int64_t)(t - n) * prm.ld_out + px] = (float)mo;
        }
        prm.first_idx[px] = first;
        prm.max_abs[px] = (float)mx;
        if (prm.mo_mean) prm.mo_mean[px] = (float)(msum / (double)(N - n));
        if (prm.sup) prm.sup[px] = (float)sr;
    }
}

cudaError_t launch_fixup(const KParams& prm, int p, const int64_t* list, const unsigned int* count, int sms,
                         cudaStream_t s) {
    fixup_kernel<<<(unsigned)(sms * 2), 128, 0, s>>>(prm, p, list, count);
    return cudaGetLastError();
}

// ---- masked mode, long monitoring horizons: every pixel in float64 ---------------------------
// The masked kernel (bwm_kernel_masked.cuh) fits in float32; like the fill kernels it keeps
// 1e-4 for horizons up to ~4x the history.  Plans that extrapolate further run this per-pixel
// float64 restatement of oracle/bfast_oracle.py:monitor_masked instead: Gram matrix and X'y over
// the valid history dates, Cholesky, two-pass sigma with n_v - p dof, the MOSUM over the
// compacted valid series with h_v = floor(h n_v / n) (the lagging cursor walks the valid dates,
// so no ring is needed), boundary lambda sqrt(log_plus((n_v + 1 + j) / n_v)), first break at the
// original date.  One thread per pixel.
__global__ void __launch_bounds__(128) masked_f64_kernel(const KParams prm, int p, double lambda) {
    const int N = prm.N, n = prm.n, h = prm.h, sp = prm.sp;
    const double* __restrict__ X = prm.xtd;       // [N][sp] float64 X'^T (centred design)
    const int KK = p * (p + 1) / 2;
    for (int64_t px = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; px < prm.n_pixels;
         px += (int64_t)gridDim.x * blockDim.x) {
        const float* y = prm.y + px;
        const int64_t ld = prm.ld_y;
        auto val = [&](int t) { return y[(int64_t)t * ld]; };
        double G[kFixMaxP * (kFixMaxP + 1) / 2], g[kFixMaxP], beta[kFixMaxP];
        for (int i = 0; i < KK; ++i) G[i] = 0.0;
        for (int i = 0; i < p; ++i) g[i] = 0.0;
        int nv = 0;
        bool all_zero = true;
        for (int t = 0; t < n; ++t) {
            const float v = val(t);
            if (!finitef(v)) continue;
            ++nv;
            all_zero = all_zero && v == 0.f;
            const double* x = X + (int64_t)t * sp;
            for (int i = 0; i < p; ++i) {
                g[i] = fma(x[i], (double)v, g[i]);
                for (int j = 0; j <= i; ++j) G[i * (i + 1) / 2 + j] = fma(x[i], x[j], G[i * (i + 1) / 2 + j]);
            }
        }
        int mv = 0;
        for (int t = n; t < N; ++t) mv += finitef(val(t)) ? 1 : 0;
        const int hv = (int)(((int64_t)h * nv) / n);
        bool ok = nv > p && hv >= 1 && mv >= 1;
        // Cholesky G = L L^T (in place); a pivot below 1e-10 of the largest diagonal entry marks
        // a (numerically) singular valid design — e.g. a harmonic aliased to zero by the gaps
        double gscale = 0.0;
        for (int j = 0; j < p; ++j) gscale = fmax(gscale, G[j * (j + 1) / 2 + j]);
        for (int j = 0; ok && j < p; ++j) {
            const int jr = j * (j + 1) / 2;
            double d = G[jr + j];
            for (int k = 0; k < j; ++k) d -= G[jr + k] * G[jr + k];
            if (!(d > 1e-10 * gscale)) { ok = false; break; }
            const double dj = sqrt(d);
            G[jr + j] = dj;
            for (int i = j + 1; i < p; ++i) {
                const int ir = i * (i + 1) / 2;
                double s = G[ir + j];
                for (int k = 0; k < j; ++k) s -= G[ir + k] * G[jr + k];
                G[ir + j] = s / dj;
            }
        }
        double sigma = 0.0;
        if (ok) {
            for (int i = 0; i < p; ++i) {                     // L w = g
                double s = g[i];
                for (int k = 0; k < i; ++k) s -= G[i * (i + 1) / 2 + k] * beta[k];
                beta[i] = s / G[i * (i + 1) / 2 + i];
            }
            for (int i = p - 1; i >= 0; --i) {                // L^T beta = w
                double s = beta[i];
                for (int k = i + 1; k < p; ++k) s -= G[k * (k + 1) / 2 + i] * beta[k];
                beta[i] = s / G[i * (i + 1) / 2 + i];
            }
            double rss = 0.0;
            for (int t = 0; t < n; ++t) {
                const float v = val(t);
                if (!finitef(v)) continue;
                double r = (double)v;
                for (int i = 0; i < p; ++i) r = fma(-X[(int64_t)t * sp + i], beta[i], r);
                rss = fma(r, r, rss);
            }
            sigma = sqrt(rss / (double)(nv - p));
            if (!(sigma > 0.0)) {
                if (all_zero) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px));
                ok = false;
            }
        }
        auto resid = [&](int t) {
            double r = (double)val(t);
            for (int i = 0; i < p; ++i) r = fma(-X[(int64_t)t * sp + i], beta[i], r);
            return r;
        };
        double mx = 0.0, msum = 0.0;
        int first = 0;
        if (ok) {
            const double inv = 1.0 / (sigma * sqrt((double)nv));
            // window 0: compacted indices [nv - hv + 1, nv] (1-based: the last hv - 1 history values
            // and the first monitoring value); the lagging cursor starts at compacted index nv - hv + 1
            double acc = 0.0;
            int seen = 0, lag = -1, lag_seen = 0;
            for (int t = 0; t < n; ++t) {
                if (!finitef(val(t))) continue;
                ++seen;                                   // 1-based compacted index of date t
                if (seen >= nv - hv + 2) acc += resid(t);
                if (seen == nv - hv + 1) { lag = t; lag_seen = seen; }
            }
            int j = 0;
            for (int t = n; t < N; ++t) {
                const float v = val(t);
                if (!finitef(v)) {
                    if (prm.mosum) prm.mosum[(int64_t)(t - n) * prm.ld_out + px] = __int_as_float(0x7fc00000);
                    continue;
                }
                const double r = resid(t);
                if (j == 0) {
                    acc += r;
                } else {
                    // advance the lagging cursor to the next valid date: compacted index lag_seen + 1
                    int tl = lag + 1;
                    while (!finitef(val(tl))) ++tl;
                    lag = tl;
                    ++lag_seen;
                    acc += r - resid(lag);
                }
                const double mo = acc * inv;
                const double a = fabs(mo);
                mx = fmax(mx, a);
                const double x = (double)(nv + 1 + j) / (double)nv;
                const double b = lambda * sqrt(x > 2.718281828459045 ? log(x) : 1.0);
                if (first == 0 && a > b) first = t + 1 - n;      // original date of the crossing
                msum += mo;
                if (prm.mosum) prm.mosum[(int64_t)(t - n) * prm.ld_out + px] = (float)mo;
                ++j;
            }
            msum /= (double)j;
        } else if (prm.mosum) {
            for (int t = n; t < N; ++t) prm.mosum[(int64_t)(t - n) * prm.ld_out + px] = __int_as_float(0x7fc00000);
        }
        prm.valid[px] = ok;
        prm.first_idx[px] = ok ? first : 0;
        prm.max_abs[px] = ok ? (float)mx : 0.f;
        if (prm.mo_mean) prm.mo_mean[px] = ok ? (float)msum : 0.f;
        if (prm.beta) {
            // raw basis (bwm.h): the fit is on the centred trend (t - tc)/ts
            for (int i = 0; i < p; ++i) {
                double b = ok ? beta[i] : 0.0;
                if (ok && i == 0) b = beta[0] - beta[1] * (double)prm.tc_ts;
                if (ok && i == 1) b = beta[1] * (double)prm.inv_ts;
                prm.beta[(int64_t)i * prm.ld_out + px] = (float)b;
            }
        }
    }
}

cudaError_t launch_masked_f64(const KParams& prm, int p, double lambda, int sms, cudaStream_t s) {
    const int64_t blocks = std::min<int64_t>((prm.n_pixels + 127) / 128, (int64_t)sms * 16);
    masked_f64_kernel<<<(unsigned)blocks, 128, 0, s>>>(prm, p, lambda);
    return cudaGetLastError();
}

}  // namespace bwm
