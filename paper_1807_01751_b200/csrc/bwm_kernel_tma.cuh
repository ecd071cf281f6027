// bwm_kernel_tma.cuh — fused BFAST-monitor kernel, TMA-staged variant (sm_100a, default).
//
// CTA = 4 consumer warps (128 threads, one pixel PAIR each -> a 256-pixel tile) + 1
// producer warp.  The producer streams the tile's rows (1 KB each: 256 float32 pixels of
// one date) from HBM/L2 into a ring of shared-memory stages with bulk asynchronous copies
// (cp.async.bulk -> the TMA engine, SASS UBLKCP), signalling an mbarrier per stage with
// complete_tx; consumers wait on the stage, read their float2 per row (LDS.64,
// conflict-free) and release the stage with one arrive per warp.  Registers hold only the
// per-pixel pipeline state; bytes in flight per SM are set by the stage ring.
//
// Row stream per tile (the producer runs ahead across passes and tiles):
//   pass 1 : rows [0, n)             beta' = M'(y - c)     (pass 0 scans the first stage for c)
//   pass 2 : rows [0, n)             residuals, sigma^2, MOSUM window 0   (re-read: L2 hit)
//   pass 3 : rows [8*floor(n/8), N)  MOSUM recurrence + detect (stages 8-row aligned);
//            LAG mode: each stage also carries rows t-h (the lagging cursor's input)
//
// MOSUM residual ring (r_{t-h} for the add-one/drop-one recurrence, _kernels.py:31-34):
//   MODE kRingTmem : in Tensor Memory.  Each thread owns its TMEM lane; ring row q of the
//                    pixel pair occupies columns 2q, 2q+1.  L = ring rows (multiple of 8,
//                    >= h) plus 8 mirror rows (L+k == k) so an 8-row window read
//                    starting anywhere in [0, L) never wraps: one tcgen05.ld.x16 and one
//                    tcgen05.st.x16 per stage instead of 8 shared loads/stores + index math.
//   MODE kRingSmem : per-thread shared-memory ring of h rows (small h < 8).
//   MODE kRingLag  : no ring; r_{t-h} recomputed from the staged row t-h (large h).
//
// The monitoring pass runs in the UNSCALED frame: acc = sum of window residuals, crossing
// test |acc| > b_j * sigma * sqrt(n) (== |MO_j| > b_j), MO = acc / (sigma sqrt n) applied to
// the max/mean at the end.
#pragma once

#include "bwm_common.cuh"

namespace bwm {

constexpr int kStageRows = 8;                   // dates per stage
constexpr int kStages = 7;                      // stage ring depth
constexpr int kRowBytes = kTile * 4;            // one date of one tile
constexpr int kConsumerWarps = kThreads / 32;
constexpr int kTmaThreads = kThreads + 32;      // + producer warp

enum RingMode { kRingSmem = 0, kRingTmem = 1, kRingLag = 2 };

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

// ---- Tensor Memory (tcgen05) helpers: the per-thread residual ring -------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 16 consecutive 32-bit columns of this thread's lane (8 ring rows of the pixel pair)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float2 (&v)[8]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = f2(__uint_as_float(r[2 * k]), __uint_as_float(r[2 * k + 1]));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float2 (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0].x)), "r"(__float_as_uint(v[0].y)), "r"(__float_as_uint(v[1].x)),
        "r"(__float_as_uint(v[1].y)), "r"(__float_as_uint(v[2].x)), "r"(__float_as_uint(v[2].y)),
        "r"(__float_as_uint(v[3].x)), "r"(__float_as_uint(v[3].y)), "r"(__float_as_uint(v[4].x)),
        "r"(__float_as_uint(v[4].y)), "r"(__float_as_uint(v[5].x)), "r"(__float_as_uint(v[5].y)),
        "r"(__float_as_uint(v[6].x)), "r"(__float_as_uint(v[6].y)), "r"(__float_as_uint(v[7].x)),
        "r"(__float_as_uint(v[7].y))
        : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(v.x)),
                 "r"(__float_as_uint(v.y))
                 : "memory");
}

// Shared-memory footprint of the TMA kernel (host mirror in bwm_capi.cu).
__host__ __device__ constexpr int64_t tma_stage_bytes(int mode) {
    return (int64_t)kStageRows * kRowBytes * (mode == kRingLag ? 2 : 1);
}

template <int NP, int MODE>
__global__ void __launch_bounds__(kTmaThreads, NP <= 10 ? 3 : 2) monitor_kernel_tma(const KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int R = kStageRows;
    constexpr int S = kStages;
    constexpr int64_t SB = tma_stage_bytes(MODE);
    constexpr int ROWF2 = kTile / 2;             // float2 per staged row
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const int NA = (N + 3) & ~3;
    unsigned char* s_stage = smem_raw;                                   // [S][SB]
    float* s_mt = reinterpret_cast<float*>(smem_raw + S * SB);           // [n][SP]
    float* s_xt = s_mt + n * SP;                                         // [N][SP]
    float* s_bd = s_xt + N * SP;                                         // [NA] bound by row t (t >= n)
    float2* s_ring = reinterpret_cast<float2*>(s_bd + NA);               // [h][kThreads] (kRingSmem)
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(
        reinterpret_cast<unsigned char*>(s_ring) + (MODE == kRingSmem ? (int64_t)h * kThreads * 8 : 0));
    uint64_t* full = s_bar;          // [S]
    uint64_t* empty = s_bar + S;     // [S]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 2 * S);

    for (int i = threadIdx.x; i < n * SP; i += kTmaThreads) s_mt[i] = prm.mt[i];
    for (int i = threadIdx.x; i < N * SP; i += kTmaThreads) s_xt[i] = prm.xt[i];
    for (int i = threadIdx.x; i < N - n; i += kTmaThreads) s_bd[n + i] = prm.bound[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (MODE == kRingTmem && threadIdx.x < 32) tmem_alloc(s_tmem, (uint32_t)prm.tmem_cols);
    if (MODE == kRingTmem) tmem_fence_before();
    __syncthreads();
    if (MODE == kRingTmem) tmem_fence_after();

    const int64_t n_tiles = prm.n_pixels / kTile;      // host guarantees whole tiles
    const int64_t ld = prm.ld_y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t3 = (n / R) * R;                        // first row of the aligned monitoring stream

    // =============================== producer ==========================================
    if (warp == kConsumerWarps) {
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const float* yt = prm.y + tile * kTile;
                for (int pass = 0; pass < 3; ++pass) {
                    const int lo = pass == 2 ? t3 : 0, hi = pass == 2 ? N : n;
                    const bool lag = MODE == kRingLag && pass == 2;
                    for (int r0 = lo; r0 < hi; r0 += R) {
                        const int rows = min(R, hi - r0);
                        const int s = it % S;
                        mbar_wait(empty + s, ((it / S) & 1) ^ 1);
                        // lag rows t-h < 0 only occur for skipped rows t < n: clamp their source
                        int lag_lo = 0;
                        if (lag) while (lag_lo < rows && r0 + lag_lo - h < 0) ++lag_lo;
                        mbar_expect_tx(full + s, (uint32_t)((rows + (lag ? rows - lag_lo : 0)) * kRowBytes));
                        unsigned char* dst = s_stage + s * SB;
                        for (int r = 0; r < rows; ++r)
                            bulk_g2s(dst + r * kRowBytes, yt + (int64_t)(r0 + r) * ld, kRowBytes, full + s);
                        if (lag)
                            for (int r = lag_lo; r < rows; ++r)
                                bulk_g2s(dst + (R + r) * kRowBytes, yt + (int64_t)(r0 + r - h) * ld, kRowBytes,
                                         full + s);
                        ++it;
                    }
                }
            }
        }
        return;
    }

    // =============================== consumers =========================================
    const int tid = threadIdx.x;
    float2* ring = s_ring + tid;
    const int wstart = n - h + 1;             // first row of MOSUM window 0 (mosum.py:59)
    const int L = prm.ring_rows;
    const uint32_t tbase = MODE == kRingTmem ? *s_tmem + ((uint32_t)(warp * 32) << 16) : 0u;
    auto tcol = [&](int row) -> uint32_t { return tbase + (uint32_t)(2 * row); };
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
        float2 lag_last = f2(0.f, 0.f);          // kRingLag: fill state of the lagging cursor
        int slot = wstart % h;                   // kRingSmem: slot of row t is t mod h
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
                float2 rr[R];
                if (MODE == kRingTmem && rows < R) {
                    tmem_wait_st();
                    tmem_ld16(tcol(t0 % L), rr);   // keep ring rows of t >= n (read-modify-write)
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    if (k < rows) {
                        const int t = t0 + k;
                        const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2], negc, last), s_xt + t * SP, nb);
                        ss = fma2(r, r, ss);
                        rr[k] = r;
                        if (t >= wstart) {
                            acc = add2(acc, r);
                            if (MODE == kRingSmem) {
                                ring[slot * kThreads] = r;
                                slot = (slot + 1 == h) ? 0 : slot + 1;
                            }
                        }
                        if (MODE == kRingLag && t == wstart - 1) lag_last = last;
                    }
                }
                if (MODE == kRingTmem) {
                    const int wb = t0 % L;
                    tmem_st16(tcol(wb), rr);
                    if (wb == 0) tmem_st16(tcol(L), rr);
                }
            }
            release();
        }
        // the ring slot of r_{n-h} must read as 0: window 0 does not contain it
        if (MODE == kRingSmem) ring[slot * kThreads] = f2(0.f, 0.f);
        if (MODE == kRingTmem) {
            const int z = (n - h) % L;
            tmem_st2(tcol(z), f2(0.f, 0.f));
            if (z < R) tmem_st2(tcol(L + z), f2(0.f, 0.f));
        }

        // sigma (engine.py:363-371) and the zero-sigma contract (engine.py:373-378): the
        // reference raises when float64 gives sigma == 0 exactly — an identically zero
        // history (c == 0).  A non-zero constant history has round-off sigma ~1e-17 there
        // (MO ~1e15): sigma_scale 0 reproduces its decisions (any non-zero window crosses).
        const bool z0 = valid0 && ss.x == 0.f && c.x == 0.f, z1 = valid1 && ss.y == 0.f && c.y == 0.f;
        if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0 + (z0 ? 0 : 1)));
        const float2 sc = sigma_scale(ss, prm.inv_dof, prm.sqrt_n, valid0, valid1);

        // ---- pass 3: monitoring period, fused MOSUM + detect (unscaled frame) ----------
        float2 mx = f2(0.f, 0.f), msum = f2(0.f, 0.f);
        int first0 = 0x7fffffff, first1 = 0x7fffffff;
        float* const mo_out = prm.mosum;
        const float2 inv = inv_scale(sc);
        for (int t0 = t3; t0 < N; t0 += R) {
            const float2* st = acquire();
            const float2* lst = st + R * ROWF2;          // lag rows (kRingLag)
            const bool full_stage = t0 > n && t0 + R <= N;
            float2 oldv[R], newv[R];
            if (MODE == kRingTmem) {
                tmem_wait_st();
                const int rb = ((t0 - h) % L + L) % L;
                tmem_ld16(tcol(rb), oldv);
                if (!full_stage) tmem_ld16(tcol(t0 % L), newv);   // preserve rows t < n
            }
            float4 b4[R / 4];
#pragma unroll
            for (int q = 0; q < R / 4; ++q) b4[q] = reinterpret_cast<const float4*>(s_bd + t0)[q];
            auto row = [&](const int k, const bool checked) {
                const int t = t0 + k;
                if (checked && (t < n || t >= N)) return;
                const float2 r = dot_row<NP, SP>(fill(st[k * ROWF2], negc, last), s_xt + t * SP, nb);
                float2 old = f2(0.f, 0.f);
                if (MODE == kRingTmem) {
                    old = oldv[k];
                    newv[k] = r;
                } else if (MODE == kRingSmem) {
                    old = ring[slot * kThreads];
                    ring[slot * kThreads] = r;
                    slot = (slot + 1 == h) ? 0 : slot + 1;
                } else if (!checked || t > n) {          // r_{t-h}; r_{n-h} is outside window 0
                    old = dot_row<NP, SP>(fill(lst[k * ROWF2], negc, lag_last), s_xt + (t - h) * SP, nb);
                }
                acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
                const float bj = (k & 3) == 0 ? b4[k >> 2].x : (k & 3) == 1 ? b4[k >> 2].y
                               : (k & 3) == 2 ? b4[k >> 2].z : b4[k >> 2].w;
                const float2 bs = mul2(sc, f2(bj, bj));   // boundary in the unscaled frame
                const float a0 = fabsf(acc.x), a1 = fabsf(acc.y);
                mx.x = fmaxf(mx.x, a0);
                mx.y = fmaxf(mx.y, a1);
                const int j1 = t - n + 1;
                if (a0 > bs.x) first0 = min(first0, j1);  // strict crossing (_kernels.py:47)
                if (a1 > bs.y) first1 = min(first1, j1);
                msum = add2(msum, acc);
                if (mo_out) *reinterpret_cast<float2*>(mo_out + (int64_t)(t - n) * prm.ld_out + px0) = mul2(acc, inv);
            };
            if (full_stage) {
#pragma unroll
                for (int k = 0; k < R; ++k) row(k, false);
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) row(k, true);
            }
            if (MODE == kRingTmem) {
                const int wb = t0 % L;
                tmem_st16(tcol(wb), newv);
                if (wb == 0) tmem_st16(tcol(L), newv);
            }
            release();
        }

        // ---- outputs --------------------------------------------------------------------
        {
            const float inv_m = 1.0f / (float)(N - n);
            *reinterpret_cast<uchar2*>(prm.valid + px0) = make_uchar2(valid0, valid1);
            *reinterpret_cast<int2*>(prm.first_idx + px0) =
                make_int2(first0 == 0x7fffffff ? 0 : first0, first1 == 0x7fffffff ? 0 : first1);
            *reinterpret_cast<float2*>(prm.max_abs + px0) = mul2(mx, inv);
            if (prm.mo_mean) *reinterpret_cast<float2*>(prm.mo_mean + px0) = mul2(mul2(msum, inv), f2(inv_m, inv_m));
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

    if (MODE == kRingTmem) {
        tmem_wait_st();
        tmem_fence_before();
        asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");   // consumer warps only
        tmem_fence_after();
        if (warp == 0) tmem_dealloc(*s_tmem, (uint32_t)prm.tmem_cols);
    }
}

}  // namespace bwm
