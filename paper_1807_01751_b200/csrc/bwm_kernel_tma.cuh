// bwm_kernel_tma.cuh — fused BFAST-monitor kernel, TMA-staged variant (sm_100a, default).
//
// CTA = 4 consumer warps (128 threads, one pixel PAIR each -> a 256-pixel tile) + 1
// producer warp.  The producer streams the tile's rows (1 KB each: 256 float32 pixels of
// one date) from HBM/L2 into a ring of shared-memory stages with bulk asynchronous copies
// (cp.async.bulk -> the TMA engine, SASS UBLKCP), signalling an mbarrier per stage with
// complete_tx; consumers wait on the stage, read their float2 per row (LDS.64,
// conflict-free) and release the stage with one arrive per warp.  Registers therefore
// hold only the per-pixel pipeline state, and the number of bytes in flight per SM is set
// by the stage ring (kStages x kStageRows KB per CTA), not by register pressure.
//
// Row stream per tile (the producer runs ahead across passes and tiles):
//   pass 1 : rows [0, n)      beta' = M'(y - c)        (pass 0 scans the first stage for c)
//   pass 2 : rows [0, n)      residuals, sigma^2, MOSUM window 0   (re-read: L2 hit)
//   pass 3 : rows [n, N)      MOSUM recurrence + detect; with !RING each stage also carries
//                             rows t-h (the lagging cursor's input, L2 hit)
// Reference phases: see bwm_common.cuh / bwm_kernel_ldg.cuh (same arithmetic).
#pragma once

#include "bwm_common.cuh"

namespace bwm {

constexpr int kStageRows = 8;                   // dates per stage
constexpr int kStages = 4;                      // stage ring depth
constexpr int kRowBytes = kTile * 4;            // one date of one tile
constexpr int kConsumerWarps = kThreads / 32;
constexpr int kTmaThreads = kThreads + 32;      // + producer warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Shared-memory footprint of the TMA kernel (host mirror in bwm_capi.cu).
__host__ __device__ constexpr int64_t tma_stage_bytes(bool ring) {
    return (int64_t)kStageRows * kRowBytes * (ring ? 1 : 2);
}

template <int NP, bool RING>
__global__ void __launch_bounds__(kTmaThreads, 2) monitor_kernel_tma(const KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int R = kStageRows;
    constexpr int S = kStages;
    constexpr int64_t SB = tma_stage_bytes(RING);
    constexpr int ROWF2 = kTile / 2;             // float2 per staged row
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    unsigned char* s_stage = smem_raw;                                   // [S][SB]
    float* s_mt = reinterpret_cast<float*>(smem_raw + S * SB);           // [n][SP]
    float* s_xt = s_mt + n * SP;                                         // [N][SP]
    float* s_bd = s_xt + N * SP;                                         // [N-n] padded to 4
    float2* s_ring = reinterpret_cast<float2*>(s_bd + ((N - n + 3) & ~3));   // [h][kThreads] (RING)
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(
        reinterpret_cast<unsigned char*>(s_ring) + (RING ? (int64_t)h * kThreads * 8 : 0));
    uint64_t* full = s_bar;          // [S]
    uint64_t* empty = s_bar + S;     // [S]

    for (int i = threadIdx.x; i < n * SP; i += kTmaThreads) s_mt[i] = prm.mt[i];
    for (int i = threadIdx.x; i < N * SP; i += kTmaThreads) s_xt[i] = prm.xt[i];
    for (int i = threadIdx.x; i < N - n; i += kTmaThreads) s_bd[i] = prm.bound[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t n_tiles = prm.n_pixels / kTile;      // host guarantees whole tiles
    const int64_t ld = prm.ld_y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // =============================== producer ==========================================
    if (warp == kConsumerWarps) {
        if (lane != 0) return;
        uint32_t it = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const float* yt = prm.y + tile * kTile;
            for (int pass = 0; pass < 3; ++pass) {
                const int lo = pass == 2 ? n : 0, hi = pass == 2 ? N : n;
                const bool lag = !RING && pass == 2;
                for (int r0 = lo; r0 < hi; r0 += R) {
                    const int rows = min(R, hi - r0);
                    const int s = it % S;
                    mbar_wait(empty + s, ((it / S) & 1) ^ 1);
                    mbar_expect_tx(full + s, (uint32_t)(rows * kRowBytes * (lag ? 2 : 1)));
                    unsigned char* dst = s_stage + s * SB;
                    for (int r = 0; r < rows; ++r)
                        bulk_g2s(dst + r * kRowBytes, yt + (int64_t)(r0 + r) * ld, kRowBytes, full + s);
                    if (lag)
                        for (int r = 0; r < rows; ++r)
                            bulk_g2s(dst + (R + r) * kRowBytes, yt + (int64_t)(r0 + r - h) * ld, kRowBytes,
                                     full + s);
                    ++it;
                }
            }
        }
        return;
    }

    // =============================== consumers =========================================
    const int tid = threadIdx.x;
    float2* ring = s_ring + tid;
    const int wstart = n - h + 1;             // first row of MOSUM window 0 (mosum.py:59)
    uint32_t it = 0;
    int cur = 0;
    auto acquire = [&]() -> const float2* {
        cur = it % S;
        mbar_wait(full + cur, (it / S) & 1);
        return reinterpret_cast<const float2*>(s_stage + cur * SB) + tid;
    };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + cur);
        ++it;
    };

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t px0 = tile * kTile + 2 * tid;
        const float* yp = prm.y + px0;

        // ---- pass 1 (+ pass 0 on its first stage) ------------------------------------
        float2 hi[NP], lo[NP], part[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) { hi[i] = lo[i] = part[i] = f2(0.f, 0.f); }
        float2 c = f2(0.f, 0.f);
        bool f0 = false, f1 = false;
        float2 last = f2(0.f, 0.f);
        float2 negc = f2(0.f, 0.f);
        for (int t0 = 0; t0 < n; t0 += R) {
            const float2* st = acquire();
            const int rows = min(R, n - t0);
            if (t0 == 0) {
                // pass 0: first finite value (engine.py:316 first = finite.argmax)
#pragma unroll
                for (int k = R - 1; k >= 0; --k) {
                    if (k < rows) {
                        const float2 v = st[k * ROWF2];
                        if (finitef(v.x)) { c.x = v.x; f0 = true; }
                        if (finitef(v.y)) { c.y = v.y; f1 = true; }
                    }
                }
                if (!(f0 && f1)) {   // rare: long leading gap or an all-missing pixel
                    for (int t = rows; t < N && !(f0 && f1); ++t) {
                        const float2 v = __ldg(reinterpret_cast<const float2*>(yp + (int64_t)t * ld));
                        if (!f0 && finitef(v.x)) { c.x = v.x; f0 = true; }
                        if (!f1 && finitef(v.y)) { c.y = v.y; f1 = true; }
                    }
                }
                negc = f2(-c.x, -c.y);
            }
            if (rows == R) {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    axpy_row<NP, SP>(part, fill(st[k * ROWF2], negc, last), s_mt + (t0 + k) * SP);
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    if (k < rows) axpy_row<NP, SP>(part, fill(st[k * ROWF2], negc, last), s_mt + (t0 + k) * SP);
            }
            release();
            if ((t0 + R) % kComp == 0 || t0 + R >= n) {
#pragma unroll
                for (int i = 0; i < NP; ++i) { two_sum(hi[i], lo[i], part[i]); part[i] = f2(0.f, 0.f); }
            }
        }
        const bool valid0 = f0, valid1 = f1;
        float2 nb[NP];    // -beta'
#pragma unroll
        for (int i = 0; i < NP; ++i) { const float2 b = add2(hi[i], lo[i]); nb[i] = f2(-b.x, -b.y); }

        // ---- pass 2: history residuals, sigma^2, MOSUM window 0 ----------------------
        float2 ss = f2(0.f, 0.f), acc = f2(0.f, 0.f);
        last = f2(0.f, 0.f);
        float2 lag_last = f2(0.f, 0.f);          // !RING: fill state of the lagging cursor
        int slot = wstart % h;                   // ring slot of row t is t mod h
        for (int t0 = 0; t0 < n; t0 += R) {
            const float2* st = acquire();
            const int rows = min(R, n - t0);
            if (rows == R && t0 + R < wstart) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2], negc, last), s_xt + (t0 + k) * SP, nb);
                    ss = fma2(r, r, ss);
                }
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    if (k < rows) {
                        const int t = t0 + k;
                        const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2], negc, last), s_xt + t * SP, nb);
                        ss = fma2(r, r, ss);
                        if (t >= wstart) {
                            acc = add2(acc, r);
                            if (RING) {
                                ring[slot * kThreads] = r;
                                slot = (slot + 1 == h) ? 0 : slot + 1;
                            }
                        }
                        if (!RING && t == wstart - 1) lag_last = last;
                    }
                }
            }
            release();
        }
        if (RING) ring[slot * kThreads] = f2(0.f, 0.f);   // slot of r_{n-h}: not in window 0

        // sigma (engine.py:363-371) and the zero-sigma contract (engine.py:373-378)
        const bool z0 = valid0 && ss.x == 0.f, z1 = valid1 && ss.y == 0.f;
        if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0 + (z0 ? 0 : 1)));
        const float2 var = mul2(ss, f2(prm.inv_dof, prm.inv_dof));
        float2 inv;
        inv.x = (valid0 && ss.x > 0.f) ? 1.0f / (sqrtf(var.x) * prm.sqrt_n) : 0.f;
        inv.y = (valid1 && ss.y > 0.f) ? 1.0f / (sqrtf(var.y) * prm.sqrt_n) : 0.f;
        if (RING)
            for (int s = 0; s < h; ++s) ring[s * kThreads] = mul2(ring[s * kThreads], inv);
        acc = mul2(acc, inv);
        float2 nbs[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) nbs[i] = mul2(nb[i], inv);

        // ---- pass 3: monitoring period, fused MOSUM + detect -------------------------
        float2 mx = f2(0.f, 0.f), msum = f2(0.f, 0.f);
        int first0 = 0x7fffffff, first1 = 0x7fffffff;
        float* const mo_out = prm.mosum;
        auto mon_row = [&](const float2 v, const float2 lv, const int t, const bool past_n) {
            const float2 r = dot_row<NP, SP>(mul2(fill(v, negc, last), inv), s_xt + t * SP, nbs);
            float2 old = f2(0.f, 0.f);
            if (RING) {
                old = ring[slot * kThreads];
                ring[slot * kThreads] = r;
                slot = (slot + 1 == h) ? 0 : slot + 1;
            } else if (past_n || t > n) {   // r_{t-h}; at t == n, r_{n-h} is outside window 0
                old = dot_row<NP, SP>(mul2(fill(lv, negc, lag_last), inv), s_xt + (t - h) * SP, nbs);
            }
            acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
            const int j = t - n;
            const float b = s_bd[j];
            const float a0 = fabsf(acc.x), a1 = fabsf(acc.y);
            mx.x = fmaxf(mx.x, a0);
            mx.y = fmaxf(mx.y, a1);
            if (a0 > b) first0 = min(first0, j + 1);  // strict crossing (_kernels.py:47)
            if (a1 > b) first1 = min(first1, j + 1);
            msum = add2(msum, acc);
            if (mo_out) *reinterpret_cast<float2*>(mo_out + (int64_t)j * prm.ld_out + px0) = acc;
        };
        for (int t0 = n; t0 < N; t0 += R) {
            const float2* st = acquire();
            const float2* lst = st + R * ROWF2;          // lag rows (!RING)
            const int rows = min(R, N - t0);
            if (rows == R && t0 > n) {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    mon_row(st[k * ROWF2], RING ? f2(0.f, 0.f) : lst[k * ROWF2], t0 + k, true);
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    if (k < rows) mon_row(st[k * ROWF2], RING ? f2(0.f, 0.f) : lst[k * ROWF2], t0 + k, false);
            }
            release();
        }

        // ---- outputs --------------------------------------------------------------------
        {
            const float inv_m = 1.0f / (float)(N - n);
            *reinterpret_cast<uchar2*>(prm.valid + px0) = make_uchar2(valid0, valid1);
            *reinterpret_cast<int2*>(prm.first_idx + px0) =
                make_int2(first0 == 0x7fffffff ? 0 : first0, first1 == 0x7fffffff ? 0 : first1);
            *reinterpret_cast<float2*>(prm.max_abs + px0) = mx;
            if (prm.mo_mean) *reinterpret_cast<float2*>(prm.mo_mean + px0) = mul2(msum, f2(inv_m, inv_m));
            if (prm.beta) {
                // back to the raw basis (bwm.h): b0 = c + b0' - b1' tc/ts, b1 = b1'/ts
                float2 bo[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) bo[i] = f2(-nb[i].x, -nb[i].y);
                const float2 b1 = bo[1];
                bo[0] = add2(c, sub2(bo[0], mul2(b1, f2(prm.tc_ts, prm.tc_ts))));
                bo[1] = mul2(b1, f2(prm.inv_ts, prm.inv_ts));
#pragma unroll
                for (int i = 0; i < NP; ++i)
                    *reinterpret_cast<float2*>(prm.beta + (int64_t)i * prm.ld_out + px0) =
                        f2(valid0 ? bo[i].x : 0.f, valid1 ? bo[i].y : 0.f);
            }
        }
    }
}

}  // namespace bwm
