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

namespace bwm {

constexpr int kFixMaxP = 18;

__global__ void __launch_bounds__(128) fixup_kernel(const KParams prm, int p, const int64_t* __restrict__ list,
                                                    const unsigned int* __restrict__ count) {
    const unsigned int cnt = *count;
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
        // pass 3: monitoring, r_{t-h} from a lagging cursor with its own fill state
        double mx = 0.0, msum = 0.0, lag_last = lastw;
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
            msum += mo;
            if (prm.mosum) prm.mosum[(int64_t)(t - n) * prm.ld_out + px] = (float)mo;
        }
        prm.first_idx[px] = first;
        prm.max_abs[px] = (float)mx;
        if (prm.mo_mean) prm.mo_mean[px] = (float)(msum / (double)(N - n));
    }
}

cudaError_t launch_fixup(const KParams& prm, int p, const int64_t* list, const unsigned int* count, int sms,
                         cudaStream_t s) {
    fixup_kernel<<<(unsigned)(sms * 2), 128, 0, s>>>(prm, p, list, count);
    return cudaGetLastError();
}

}  // namespace bwm
