// bwm_kernel_ldg.cuh — fused BFAST-monitor kernel, register-prefetch variant (sm_100a).
//
// Used for the tail tile and for inputs whose rows are not 16-byte aligned (SAFE), and
// kept as the A/B baseline of the TMA-staged kernel (bwm_kernel_tma.cuh).
//
// One CTA = 128 threads = one tile of 256 pixels; one thread owns a pixel PAIR and
// runs the whole per-pixel pipeline of the reference's fused backend in registers:
//
//   reference phase (engine.py)                 here
//   ---------------------------------------     -------------------------------------------
//   ingest  _ingest_block  (305-319)            pass 0: first finite value c per pixel
//                                               fill on the fly: NaN/Inf -> last finite value,
//                                               leading gap -> c (exact float32 copies)
//   model   M @ values[:n]  (339-349)           pass 1: beta_Q = Q^T (y - c), FFMA2, 32-date
//                                               blocks 2Sum-compensated into (hi, lo); the
//                                               window sum of the filled dates [n-h, n)
//   predictions / residuals (351-385)           sigma from RSS = ||y-c||^2 - ||beta_Q||^2;
//                                               window-sum formulation (bwm_common.cuh): the
//                                               fitted values enter only as S_t^T beta_Q
//   mosum  _kernels.mosum_block (21-34)         pass 3: window recurrence acc += y~_new - y~_old
//   breaks _kernels.detect_block (37-48)                 |MO| max, first strict crossing
//
// Memory: the stack is time-major (row t = every pixel at date t), so a warp reading one
// date of its 64 pixels issues one coalesced 256-byte request (float2 per lane).  Rows are
// streamed through a 16-deep per-thread register ring (slot t mod 16 holds row t), in ONE
// sweep over the dates per tile; refills run across the pass boundary and into the next
// tile's first rows, so the load pipe never drains.  Every operation matches the TMA kernel's
// order, so both give bit-identical results (test_kernel_variants_bit_identical).
#pragma once

#include "bwm_common.cuh"

namespace bwm {

// RING = true : y~_{t-h} comes from a per-thread smem ring of h filled values (h*1 KB per CTA).
// RING = false: y~_{t-h} is refilled from y_{t-h} by a lagging cursor (an L2 hit: that row
//               was read h rows earlier) — used when the ring would not fit (large h, C4).
template <int NP, bool SAFE, bool RING>
__global__ void __launch_bounds__(kThreads, 2) monitor_kernel_ldg(const KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int D = kDepth;
    extern __shared__ __align__(16) float smem[];
    const int N = prm.N, n = prm.n, h = prm.h;
    // RING: the window-sum table (rows < n: Q^T, rows >= n: S_t) lives in smem.  !RING (large
    // h or long series): it stays in global memory, read through L1 (uniform addresses), so
    // any N fits; only the boundary is staged.
    float* s_tab = smem;
    const float* s_wt = RING ? s_tab : prm.wt;                                 // [N][SP]
    float* s_bd = s_tab + (RING ? N * SP : 0);                                 // [N-n] (padded to 4)
    float2* s_ring = reinterpret_cast<float2*>(s_bd + ((N - n + 3) & ~3));   // [h][kThreads]

    // --- constant tables -> smem (once per persistent CTA) -------------------------
    if (RING)
        for (int i = threadIdx.x; i < N * SP; i += kThreads) s_tab[i] = prm.wt[i];
    for (int i = threadIdx.x; i < N - n; i += kThreads) s_bd[i] = prm.bound[i];
    __syncthreads();

    const int tid = threadIdx.x;
    float2* ring = s_ring + tid;              // this thread's column of the MOSUM ring
    const int64_t n_tiles = (prm.n_pixels + kTile - 1) / kTile;
    const int64_t ld = prm.ld_y;
    const int64_t hld = (int64_t)h * ld;
    const int wst = n - h;                    // first date of the initial window [n-h, n)
    const double* const wtd = prm.wtd;        // precise mode: float64 table (long horizons)

    int64_t tile = blockIdx.x;
    if (tile >= n_tiles) return;
    int64_t px0 = tile * kTile + 2 * tid;
    int npx = SAFE ? (int)max((int64_t)0, min((int64_t)2, prm.n_pixels - px0)) : 2;
    const float* yp = prm.y + px0;

    float2 buf[D];                            // slot t mod D: row t
    float2 lbuf[RING ? 1 : D];                // !RING, slot t mod D: row t - h (t >= n)
#pragma unroll
    for (int k = 0; k < D; ++k) {
        if (k < N) buf[k] = ldp<SAFE>(yp + (int64_t)k * ld, npx);
        if (!RING && k >= n && k < N) lbuf[RING ? 0 : k] = ldp<SAFE>(yp + (int64_t)(k - h) * ld, npx);
    }

    for (;;) {
        const int64_t next_tile = tile + gridDim.x;
        const bool has_next = next_tile < n_tiles;
        const int64_t npx0 = has_next ? next_tile * kTile + 2 * tid : px0;
        const int nnpx = SAFE ? (has_next ? (int)max((int64_t)0, min((int64_t)2, prm.n_pixels - npx0)) : 0) : 2;
        const float* ynp = prm.y + npx0;

        // Consume row t (slot k = t mod D): refill the slot with row t + D of this tile, or,
        // past the last row, with row k of the next tile; the lag slot likewise with row
        // t + D - h (monitoring rows only).  pf points at row t + D.
        const float* pf = yp + (int64_t)D * ld;
        auto refill = [&](const int k, const int t) {
            if (t + D < N) {
                buf[k] = ldp<SAFE>(pf, npx);
                if (!RING && t + D >= n) lbuf[RING ? 0 : k] = ldp<SAFE>(pf - hld, npx);
            } else if (has_next && k < N) {
                buf[k] = ldp<SAFE>(ynp + (int64_t)k * ld, nnpx);
                if (!RING && k >= n) lbuf[RING ? 0 : k] = ldp<SAFE>(ynp + (int64_t)(k - h) * ld, nnpx);
            }
            pf += ld;
        };

        // ---- pass 0: first finite value per pixel (warp-cooperative early exit) -----
        float2 c = f2(0.f, 0.f);
        bool f0 = npx < 1, f1 = npx < 2;
        for (int t = 0; t < N; t += 4) {
            if (__all_sync(0xffffffffu, f0 && f1)) break;
            float2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v[k] = (t + k < N) ? ldp<SAFE>(yp + (int64_t)(t + k) * ld, npx)
                                   : f2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!f0 && finitef(v[k].x)) { c.x = v[k].x; f0 = true; }
                if (!f1 && finitef(v[k].y)) { c.y = v[k].y; f1 = true; }
            }
        }
        const bool valid0 = (npx >= 1) && f0;
        const bool valid1 = (npx >= 2) && f1;
        const float2 negc = f2(-c.x, -c.y);

        // ---- pass 1: beta_Q, ||y - c||^2, the initial window sum -----------------------
        float2 hi[NP], lo[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) { hi[i] = f2(0.f, 0.f); lo[i] = f2(0.f, 0.f); }
        double q0 = 0.0, q1 = 0.0;           // ||y - c||^2 (32-date float32 partials, float64 sum)
        double wd0 = 0.0, wd1 = 0.0;         // window sum of [n-h, n), same blocks
        float2 last = f2(0.f, 0.f), lag_last = f2(0.f, 0.f);
        float2 part[NP], qpart = f2(0.f, 0.f), wpart = f2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < NP; ++i) part[i] = f2(0.f, 0.f);
        int slot = RING ? wst % h : 0;       // RING: ring slot of date t is t mod h
        // precise mode (long horizons): beta_Q and ||y - c||^2 also accumulated in float64 — the
        // float32 block partials' rounding, multiplied by a far-extrapolated S_t, is what limits
        // the MOSUM there
        double pd0[NP], pd1[NP], qd0 = 0.0, qd1 = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) pd0[i] = pd1[i] = 0.0;
        auto hist_row = [&](const float2 v, const int t) {
            const float2 vc = fill(v, negc, last);
            axpy_row<NP, SP>(part, vc, s_wt + t * SP);
            qpart = fma2(vc, vc, qpart);
            if (t >= wst) {
                wpart = add2(wpart, vc);
                if (RING) {
                    ring[slot * kThreads] = vc;
                    slot = (slot + 1 == h) ? 0 : slot + 1;
                }
            }
            if (!RING && t == wst - 1) lag_last = vc;
            if (wtd) {
                const double a = (double)vc.x, b = (double)vc.y;
                const double* z = wtd + (int64_t)t * SP;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const double zz = __ldg(z + i);
                    pd0[i] = fma(a, zz, pd0[i]);
                    pd1[i] = fma(b, zz, pd1[i]);
                }
                qd0 = fma(a, a, qd0);
                qd1 = fma(b, b, qd1);
            }
        };
        for (int t0 = 0; t0 < n; t0 += D) {
            if (t0 + 2 * D <= n) {            // every refill row is a history row: no lag loads
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float2 v = buf[k];
                    buf[k] = ldp<SAFE>(pf, npx);
                    pf += ld;
                    hist_row(v, t0 + k);
                }
            } else {
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const int t = t0 + k;
                    if (t < n) {
                        const float2 v = buf[k];
                        refill(k, t);
                        hist_row(v, t);
                    }
                }
            }
            if ((t0 + D) % kComp == 0 || t0 + D >= n) {   // same blocks as the TMA kernel
#pragma unroll
                for (int i = 0; i < NP; ++i) { two_sum(hi[i], lo[i], part[i]); part[i] = f2(0.f, 0.f); }
                q0 += (double)qpart.x;
                q1 += (double)qpart.y;
                wd0 += (double)wpart.x;
                wd1 += (double)wpart.y;
                qpart = wpart = f2(0.f, 0.f);
            }
        }
        float2 bq[NP], nb[NP];    // beta_Q and -beta_Q
        double sd0 = 0.0, sd1 = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            bq[i] = add2(hi[i], lo[i]);
            nb[i] = f2(-bq[i].x, -bq[i].y);
            sd0 = fma(pd0[i], pd0[i], sd0);
            sd1 = fma(pd1[i], pd1[i], sd1);
        }
        const float2 ss = wtd ? f2((float)fmax(qd0 - sd0, 0.0), (float)fmax(qd1 - sd1, 0.0))
                              : rss_onepass<NP>(q0, q1, bq);
        if (!wtd) {
            fix_flag(prm, valid0, q0, ss.x, px0);
            fix_flag(prm, valid1, q1, ss.y, px0 + 1);
        }
        // initial window sum minus the intercept part of S^T beta_Q (float64)
        float2 acc = wtd ? f2((float)(wd0 - prm.s0 * pd0[0]), (float)(wd1 - prm.s0 * pd1[0]))
                         : wsum_init(wd0, wd1, hi[0], lo[0], prm.s0);
        // MOSUM numerator of date t: acc - S_t^T beta_Q (float64 for long horizons: uniform branch)
        auto numer = [&](const float2 a, const int t) -> float2 {
            if (wtd) {
                const double* s = wtd + (int64_t)t * SP;
                double r0 = (double)a.x, r1 = (double)a.y;
#pragma unroll
                for (int i = 1; i < NP; ++i) {
                    const double z = __ldg(s + i);
                    r0 = fma(-z, pd0[i], r0);
                    r1 = fma(-z, pd1[i], r1);
                }
                return f2((float)r0, (float)r1);
            }
            return wsum_row<NP, SP>(a, s_wt + t * SP, nb);
        };

        // sigma and the zero-sigma contract: see bwm_kernel_tma.cuh (identical arithmetic)
        const bool z0 = zero_history(valid0, wtd ? qd0 : q0, c.x), z1 = zero_history(valid1, wtd ? qd1 : q1, c.y);
        if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0 + (z0 ? 0 : 1)));
        const float2 sc = sigma_scale(ss, prm.inv_dof, prm.sqrt_n, valid0, valid1);
        const float2 inv = inv_scale(sc);

        // ---- pass 3: monitoring period, fused MOSUM + detect -------------------------
        float2 mx = f2(0.f, 0.f), msum = f2(0.f, 0.f), sr = f2(0.f, 0.f);
        int first0 = 0x7fffffff, first1 = 0x7fffffff;
        float* const mo_out = prm.mosum;
        const bool want_sup = prm.sup != nullptr;
        // one monitoring row; fast: no bounds checks, refill is the same tile's row t+D
        auto mon_row = [&](const int k, const int t, const bool fast) {
            const float2 v = buf[k];
            float2 lv = f2(0.f, 0.f);
            if (!RING) lv = lbuf[RING ? 0 : k];
            if (fast) {
                buf[k] = ldp<SAFE>(pf, npx);
                if (!RING) lbuf[RING ? 0 : k] = ldp<SAFE>(pf - hld, npx);
                pf += ld;
            } else {
                refill(k, t);
            }
            const float2 r = fill(v, negc, last);
            float2 old;
            if (RING) {
                old = ring[slot * kThreads];
                ring[slot * kThreads] = r;
                slot = (slot + 1 == h) ? 0 : slot + 1;
            } else {
                old = fill(lv, negc, lag_last);
            }
            acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
            const float2 num = numer(acc, t);
            const int j = t - n;
            const float bj = s_bd[j];
            const float2 bs = mul2(sc, f2(bj, bj));    // boundary in the unscaled frame
            const float a0 = fabsf(num.x), a1 = fabsf(num.y);
            mx.x = fmaxf(mx.x, a0);
            mx.y = fmaxf(mx.y, a1);
            if (a0 > bs.x) first0 = min(first0, j + 1);  // strict crossing (_kernels.py:47)
            if (a1 > bs.y) first1 = min(first1, j + 1);
            if (want_sup) {                              // max_j |num_j| / b_j (unscaled)
                sr.x = fmaxf(sr.x, __fdividef(a0, bj));
                sr.y = fmaxf(sr.y, __fdividef(a1, bj));
            }
            msum = add2(msum, num);
            if (mo_out) {
                const float2 mo = mul2(num, inv);
                float* o = mo_out + (int64_t)j * prm.ld_out + px0;
                if (npx >= 1) o[0] = mo.x;
                if (npx >= 2) o[1] = mo.y;
            }
        };
        for (int t0 = (n / D) * D; t0 < N; t0 += D) {
            if (t0 >= n && t0 + 2 * D <= N) {
#pragma unroll
                for (int k = 0; k < D; ++k) mon_row(k, t0 + k, true);
            } else {
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const int t = t0 + k;
                    if (t >= n && t < N) mon_row(k, t, false);
                }
            }
        }

        // ---- outputs --------------------------------------------------------------------
        if (npx >= 1) {
            const float inv_m = 1.0f / (float)(N - n);
            prm.valid[px0] = valid0;
            prm.first_idx[px0] = first0 == 0x7fffffff ? 0 : first0;
            const float2 mxs = mul2(mx, inv), mean = mul2(mul2(msum, inv), f2(inv_m, inv_m));
            prm.max_abs[px0] = mxs.x;
            if (prm.mo_mean) prm.mo_mean[px0] = mean.x;
            const float2 srs = mul2(sr, inv);
            if (want_sup) prm.sup[px0] = srs.x;
            if (npx >= 2) {
                prm.valid[px0 + 1] = valid1;
                prm.first_idx[px0 + 1] = first1 == 0x7fffffff ? 0 : first1;
                prm.max_abs[px0 + 1] = mxs.y;
                if (prm.mo_mean) prm.mo_mean[px0 + 1] = mean.y;
                if (want_sup) prm.sup[px0 + 1] = srs.y;
            }
            if (prm.beta) store_beta<NP>(prm, px0, c, bq, valid0, valid1, npx);
        }

        if (!has_next) break;
        tile = next_tile;
        px0 = npx0;
        npx = nnpx;
        yp = ynp;
    }
}

}  // namespace bwm
