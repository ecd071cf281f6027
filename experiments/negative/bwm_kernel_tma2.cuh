// bwm_kernel_tma2.cuh — the LEAN TMEM-ring kernel with TWO pixel pairs per lane.
//
// Same pipeline, arithmetic and order of operations per pixel as monitor_kernel_tma<NP,
// kRingTmem, true> (bwm_kernel_tma.cuh; results are bit-identical), restructured so that each
// lane owns two pixel pairs: a warp covers 128 pixels (8-date x 128-pixel TMA boxes, 512 B rows),
// a CTA a 512-pixel tile.  Per stage, the broadcast table rows (Q^T / Z^T), the mbarrier
// wait/probe, the TMA re-arm and the loop bookkeeping are paid once for four pixels instead
// of two, and every dependency chain (fill, FFMA2 accumulations, MOSUM recurrence) has a twin
// to interleave with.  Pair j of lane l in warp w: pixels 512 tile + 128 w + 64 j + 2 l, 2l+1;
// its TMEM ring occupies columns [2L j, 2L (j + 1)) of the lane.
#pragma once

#include "bwm_kernel_tma.cuh"

namespace bwm {

constexpr int kPP = 2;                              // pixel pairs per lane
constexpr int kWarpPx2 = 64 * kPP;                  // pixels per warp slice
constexpr int kTile2 = kWarpPx2 * kWarps;           // pixels per CTA tile
constexpr int kBox2Bytes = kStageRows * kWarpPx2 * 4;
#ifndef BWM_STAGES2
#define BWM_STAGES2 4
#endif
#ifndef BWM_TMA2_MINB
#define BWM_TMA2_MINB 3
#endif
constexpr int kStages2 = BWM_STAGES2;

// shared memory (host mirror in bwm_capi.cu)
__host__ __device__ inline int64_t tma2_smem_bytes(int N, int p) {
    const int sp = (p + 3) & ~3;
    const int64_t fl = (int64_t)N * sp + ((N + 3) & ~3);
    const int sched = 2 * ((N + kStageRows - 1) / kStageRows) + 4;
    return (int64_t)kWarps * kStages2 * kBox2Bytes + fl * 4 + kWarps * kStages2 * 8 + 16 + 4 * sched;
}

template <int NP>
__global__ void __launch_bounds__(kTmaThreads, BWM_TMA2_MINB)
    monitor_kernel_tma2(const __grid_constant__ KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int R = kStageRows;
    constexpr int S = kStages2;
    constexpr int SB = kBox2Bytes;
    constexpr int ROWF2 = kWarpPx2 / 2;          // float2 per staged row of a warp slice
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const int NA = (N + 3) & ~3;
    unsigned char* s_stage = smem_raw;                                   // [kWarps][S][SB]
    float* s_xt = reinterpret_cast<float*>(smem_raw + kWarps * S * SB);  // [N][SP] Z^T (rows < n: Q^T)
    const float* s_mt = s_xt;
    float* s_bd = s_xt + N * SP;                                         // [NA] bound by row t (t >= n)
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_bd + NA);           // [kWarps][S]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + kWarps * S);
    int* s_rows = reinterpret_cast<int*>(s_tmem + 4);                   // [tile_stages]

    for (int i = threadIdx.x; i < N * SP; i += kTmaThreads) s_xt[i] = prm.xt[i];
    for (int i = threadIdx.x; i < N - n; i += kTmaThreads) s_bd[n + i] = prm.bound[i];
    const int wstart = n - h + 1;                      // first row of MOSUM window 0 (mosum.py:59)
    const int w0 = (wstart / R) * R;                   // first parked row
    const int t3 = (n / R) * R;                        // first row of the (aligned) monitoring stream
    const int st1 = (n + R - 1) / R;
    const int tile_stages = st1 + (N - t3 + R - 1) / R;
    for (int i = threadIdx.x; i < tile_stages; i += kTmaThreads) s_rows[i] = i < st1 ? i * R : t3 + (i - st1) * R;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWarps * S; ++s) mbar_init(s_bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) tmem_alloc(s_tmem, (uint32_t)prm.tmem_cols);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    const int64_t n_tiles = prm.n_pixels / kTile2;     // host guarantees whole tiles
    const int64_t ld = prm.ld_y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wu = __shfl_sync(0xffffffffu, warp, 0);
    unsigned char* my_stage = s_stage + wu * S * SB;
    uint64_t* full = s_bar + wu * S;
    const uint32_t stage_u32 = smem_u32(my_stage), bar_u32 = smem_u32(full);

    int64_t itile = blockIdx.x;
    int istage = 0;
    int xw = (int)(itile * kTile2) + wu * kWarpPx2;
    auto issue_into = [&](int slot) {
        if (itile >= n_tiles) return;
        const int r0 = s_rows[istage];
        tma_box_elect(stage_u32 + (uint32_t)(slot * SB), &prm.tmap, xw, r0, bar_u32 + (uint32_t)(slot * 8), SB);
        if (++istage == tile_stages) {
            istage = 0;
            itile += gridDim.x;
            xw += (int)gridDim.x * kTile2;
        }
    };
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&prm.tmap)) : "memory");
    for (int s = 0; s < S; ++s) issue_into(s);

    const int L = prm.ring_rows;
    const uint32_t tbase = *s_tmem + ((uint32_t)(wu * 32) << 16);
    auto tcol = [&](int j, int row) -> uint32_t { return tbase + (uint32_t)(2 * row + 2 * L * j); };
    const int q_w0 = w0 % L, q_wstart = wstart % L, q_t3 = t3 % L, q_t3h = ((t3 - h) % L + L) % L;
    const int q_nh = (n - h) % L;
    auto ring_ld2 = [&](int j, int q, float2& v) {                        // no wait
        uint32_t a, b;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(tcol(j, q)) : "memory");
        v = f2(__uint_as_float(a), __uint_as_float(b));
    };
    auto ring_load = [&](int q0, float2 (&v)[kPP][R]) {                   // R rows from q0 < L, both pairs
        tmem_wait_st();
        if (q0 + R <= L) {
#pragma unroll
            for (int j = 0; j < kPP; ++j) tmem_ld16(tcol(j, q0), v[j]);
        } else {
#pragma unroll
            for (int j = 0; j < kPP; ++j)
#pragma unroll
                for (int k = 0; k < R; ++k) ring_ld2(j, q0 + k >= L ? q0 + k - L : q0 + k, v[j][k]);
            tmem_wait_ld();
        }
    };
    int cur = 0;
    uint32_t ph = 0;
    uint32_t next_ready = 0;
    auto acquire = [&]() -> const float2* {
        if (!next_ready) mbar_wait(full + cur, ph);
        const int nc = cur + 1 == S ? 0 : cur + 1;
        next_ready = mbar_test(full + nc, nc == 0 ? ph ^ 1 : ph);
        return reinterpret_cast<const float2*>(my_stage + cur * SB) + lane;
    };
    auto release = [&]() {
        __syncwarp();
        issue_into(cur);
        if (++cur == S) { cur = 0; ph ^= 1; }
    };

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int64_t px0[kPP];
#pragma unroll
        for (int j = 0; j < kPP; ++j) px0[j] = tile * kTile2 + wu * kWarpPx2 + 64 * j + 2 * lane;

        // ---- pass 1: beta_Q and ||y - c||^2 (+ pass 0 on the first stage) ---------------
        float2 hi[kPP][NP], lo[kPP][NP], part[kPP][NP];
#pragma unroll
        for (int j = 0; j < kPP; ++j)
#pragma unroll
            for (int i = 0; i < NP; ++i) { hi[j][i] = lo[j][i] = part[j][i] = f2(0.f, 0.f); }
        float2 qpart[kPP], c[kPP], last[kPP], negc[kPP];
        double qa[kPP], qb[kPP];
        bool fa[kPP], fb[kPP];
#pragma unroll
        for (int j = 0; j < kPP; ++j) {
            qpart[j] = c[j] = last[j] = negc[j] = f2(0.f, 0.f);
            qa[j] = qb[j] = 0.0;
            fa[j] = fb[j] = false;
        }
        int pr = q_w0;
        for (int t0 = 0; t0 < n; t0 += R) {
            const float2* st = acquire();
            if (t0 == 0) {
                const int rows = min(R, n);
#pragma unroll
                for (int j = 0; j < kPP; ++j) {
#pragma unroll 1
                    for (int k = rows - 1; k >= 0; --k) {
                        const float2 v = st[k * ROWF2 + 32 * j];
                        if (finitef(v.x)) { c[j].x = v.x; fa[j] = true; }
                        if (finitef(v.y)) { c[j].y = v.y; fb[j] = true; }
                    }
                    if (!(fa[j] && fb[j])) {   // rare: long leading gap or an all-missing pixel
                        const float* yp = prm.y + px0[j];
                        for (int t = rows; t < N && !(fa[j] && fb[j]); ++t) {
                            const float2 v = __ldg(reinterpret_cast<const float2*>(yp + (int64_t)t * ld));
                            if (!fa[j] && finitef(v.x)) { c[j].x = v.x; fa[j] = true; }
                            if (!fb[j] && finitef(v.y)) { c[j].y = v.y; fb[j] = true; }
                        }
                    }
                    negc[j] = f2(-c[j].x, -c[j].y);
                }
            }
            const bool park = t0 >= w0;
            if (t0 + R <= n) {
                const float* mrow = s_mt + t0 * SP;
                float2 yy[kPP][R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
#pragma unroll
                    for (int j = 0; j < kPP; ++j) {
                        const float2 vc = fill(st[k * ROWF2 + 32 * j], negc[j], last[j]);
                        yy[j][k] = vc;
                        axpy_row<NP, SP>(part[j], vc, mrow + k * SP);
                        qpart[j] = fma2(vc, vc, qpart[j]);
                    }
                }
                if (park)
#pragma unroll
                    for (int j = 0; j < kPP; ++j) tmem_st16(tcol(j, pr), yy[j]);
            } else {                                            // last stage: dates [t0, n) only
#pragma unroll 1
                for (int k = 0; k < n - t0; ++k) {
#pragma unroll
                    for (int j = 0; j < kPP; ++j) {
                        const float2 vc = fill(st[k * ROWF2 + 32 * j], negc[j], last[j]);
                        if (park) tmem_st2(tcol(j, pr + k >= L ? pr + k - L : pr + k), vc);
                        axpy_row<NP, SP>(part[j], vc, s_mt + (t0 + k) * SP);
                        qpart[j] = fma2(vc, vc, qpart[j]);
                    }
                }
            }
            release();
            if (park) { pr += R; if (pr >= L) pr -= L; }
            if (((t0 + R) & (kComp - 1)) == 0 || t0 + R >= n) {
#pragma unroll
                for (int j = 0; j < kPP; ++j) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) { two_sum(hi[j][i], lo[j][i], part[j][i]); part[j][i] = f2(0.f, 0.f); }
                    qa[j] += (double)qpart[j].x;
                    qb[j] += (double)qpart[j].y;
                    qpart[j] = f2(0.f, 0.f);
                }
            }
        }
        float2 nb[kPP][NP], sc[kPP];
        bool va[kPP], vb[kPP];
#pragma unroll
        for (int j = 0; j < kPP; ++j) {
            float2 bq[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) { bq[i] = add2(hi[j][i], lo[j][i]); nb[j][i] = f2(-bq[i].x, -bq[i].y); }
            va[j] = fa[j];
            vb[j] = fb[j];
            const float2 ss = rss_onepass<NP>(qa[j], qb[j], bq);
            const bool z0 = va[j] && ss.x == 0.f && c[j].x == 0.f, z1 = vb[j] && ss.y == 0.f && c[j].y == 0.f;
            if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0[j] + (z0 ? 0 : 1)));
            sc[j] = sigma_scale(ss, prm.inv_dof, prm.sqrt_n, va[j], vb[j]);
            if (prm.beta) store_beta<NP>(prm, px0[j], c[j], bq, va[j], vb[j], 2);
        }

        // ---- window 0: parked filled values -> residuals, in place, date order ----------
        float2 acc[kPP];
#pragma unroll
        for (int j = 0; j < kPP; ++j) acc[j] = f2(0.f, 0.f);
        tmem_wait_st();
        {
            int q = q_wstart;
#pragma unroll 1
            for (int t0 = wstart; t0 < n; t0 += R) {
                float2 v[kPP][R];
                int qk[R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    qk[k] = q + k >= L ? q + k - L : q + k;
#pragma unroll
                    for (int j = 0; j < kPP; ++j)
                        if (t0 + k < n) ring_ld2(j, qk[k], v[j][k]);
                }
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    if (t0 + k < n) {
#pragma unroll
                        for (int j = 0; j < kPP; ++j) {
                            const float2 r = dot_row<NP, SP>(v[j][k], s_xt + (t0 + k) * SP, nb[j]);
                            acc[j] = add2(acc[j], r);
                            tmem_st2(tcol(j, qk[k]), r);
                        }
                    }
                }
                q = q + R >= L ? q + R - L : q + R;
            }
        }
#pragma unroll
        for (int j = 0; j < kPP; ++j) tmem_st2(tcol(j, q_nh), f2(0.f, 0.f));   // r_{n-h} is not in window 0

        // ---- pass 3: monitoring period, fused MOSUM + detect (unscaled frame) ----------
        float2 mx[kPP], bsc[kPP];
        int fx[kPP], fy[kPP];
#pragma unroll
        for (int j = 0; j < kPP; ++j) {
            mx[j] = f2(0.f, 0.f);
            fx[j] = fy[j] = 0x7fffffff;
            bsc[j] = mul2(sc[j], f2(s_bd[n], s_bd[n]));
        }
        auto step = [&](int j, const float2 r, const float2 old, const int t) {
            acc[j] = add2(acc[j], sub2(r, old));       // _kernels.py:33 order
            const float a0 = fabsf(acc[j].x), a1 = fabsf(acc[j].y);
            mx[j].x = fmaxf(mx[j].x, a0);
            mx[j].y = fmaxf(mx[j].y, a1);
            const int j1 = t - n + 1;
            if (a0 > bsc[j].x) fx[j] = min(fx[j], j1);   // strict crossing (_kernels.py:47)
            if (a1 > bsc[j].y) fy[j] = min(fy[j], j1);
        };
        int wb = q_t3, rb = q_t3h;
        for (int t0 = t3; t0 < N; t0 += R) {
            const float2* st = acquire();
            if (t0 >= n && t0 + R <= N) {
                float2 oldv[kPP][R], newv[kPP][R];
                ring_load(rb, oldv);
                const float* xrow = s_xt + t0 * SP;
#pragma unroll
                for (int k = 0; k < R; ++k) {
#pragma unroll
                    for (int j = 0; j < kPP; ++j) {
                        const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2 + 32 * j], negc[j], last[j]), xrow + k * SP, nb[j]);
                        newv[j][k] = r;
                        step(j, r, oldv[j][k], t0 + k);
                    }
                }
#pragma unroll
                for (int j = 0; j < kPP; ++j) tmem_st16(tcol(j, wb), newv[j]);
            } else {
                // boundary stage: dates [max(t0, n), min(t0 + R, N)), one at a time
                tmem_wait_st();
                const int k0 = max(0, n - t0), k1 = min(R, N - t0);
#pragma unroll 1
                for (int k = k0; k < k1; ++k) {
                    const int qo = rb + k >= L ? rb + k - L : rb + k;
#pragma unroll
                    for (int j = 0; j < kPP; ++j) {
                        const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2 + 32 * j], negc[j], last[j]), s_xt + (t0 + k) * SP, nb[j]);
                        float2 old;
                        ring_ld2(j, qo, old);
                        tmem_wait_ld();
                        tmem_st2(tcol(j, wb + k), r);
                        step(j, r, old, t0 + k);
                    }
                }
            }
            release();
            wb += R; if (wb == L) wb = 0;
            rb += R; if (rb >= L) rb -= L;
        }

        // ---- outputs --------------------------------------------------------------------
#pragma unroll
        for (int j = 0; j < kPP; ++j) {
            const float2 inv = inv_scale(sc[j]);
            *reinterpret_cast<uchar2*>(prm.valid + px0[j]) = make_uchar2(va[j], vb[j]);
            *reinterpret_cast<int2*>(prm.first_idx + px0[j]) =
                make_int2(fx[j] == 0x7fffffff ? 0 : fx[j], fy[j] == 0x7fffffff ? 0 : fy[j]);
            *reinterpret_cast<float2*>(prm.max_abs + px0[j]) = mul2(mx[j], inv);
        }
    }

    tmem_wait_st();
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(*s_tmem, (uint32_t)prm.tmem_cols);
}

}  // namespace bwm
