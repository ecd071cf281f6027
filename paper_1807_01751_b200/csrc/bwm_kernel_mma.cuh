// bwm_kernel_mma.cuh — fused BFAST-monitor kernel for long series with a large MOSUM bandwidth
// (the lagging-cursor mode, BASELINE config 4: N = 1000, p = 14, h = 250), with every fitted
// value on the TENSOR CORES (sm_100a tcgen05.mma.kind::tf32, 3xTF32).
//
// Why: in the lagging-cursor mode each monitoring date needs two fitted values, z_t^T beta_Q and
// z_{t-h}^T beta_Q (the residual leaving the window is recomputed from the re-staged date t-h,
// because an h = 250 residual ring does not fit on chip at full occupancy), plus one per
// window-0 date: 2p FFMA per pixel and date, 41% of the FFMA-kernel's instructions at C4
// (profiles/r02_C4_*).  Here they are one contraction per 16-date chunk and tile:
//   Yhat[pixel][date] = beta_Q[pixel][.] . Z^T[.][date]      (M = 128 pixels, N = 16 dates, K = p)
// A = beta_Q (per-pixel rows, written by each thread into its own TMEM lane: hi and lo tf32
// halves), B = Z^T rows (host-split tf32 hi/lo tables, staged in shared memory), D in TMEM;
// D = Ah.Bh + Ah.Bl + Al.Bh (3xTF32: ~2^-21 relative per product, float32 accumulation in the
// tensor core — the same error class as the FFMA path it replaces; the parity suite runs on it).
// beta_Q itself stays on FFMA2 with 2Sum-compensated 32-date blocks (pass 1).
//
// CTA = 8 warps = two independent 4-warp SETS; set s owns a 256-pixel tile (lane l of warp q
// owns pixels 64q + 2l, 64q + 2l + 1: MMA group 0 = even pixels, group 1 = odd) and 256 of the
// SM's 512 TMEM columns: A (2 groups x hi|lo x 8 KS) and NB chunk buffers, each holding the
// fitted values of 16 current dates and of their 16 lag dates for both groups.  One CTA per SM
// (the B tables: ~160 KB at C4, shared by both sets).
//
// Synchronisation (no producer warp): the LAST of a set's 4 warps to write its beta rows issues
// the first NB chunks' MMAs; the last warp to finish reading a chunk buffer issues the chunk NB
// ahead into it (acq_rel shared-memory tickets + tcgen05 fences); tcgen05.commit arrives on the
// buffer's mbarrier, which the warps wait on (parity = use count of the buffer).
//
// Per-warp y staging is the TMA kernel's: 8-date x 64-pixel tensor-TMA boxes, plus the lag box
// (dates t-h) in the monitoring pass (bwm_kernel_tma.cuh).
#pragma once

#include "bwm_common.cuh"
#include "bwm_kernel_tma.cuh"
#include "bwm_kernel_masked.cuh"   // smem_desc_kmajor, idesc_tf32, mma_tf32_ts, mma_commit

namespace bwm {

constexpr int kMmaSets = 2;
constexpr int kMmaWarps = 4 * kMmaSets;
constexpr int kMmaThreads = 32 * kMmaWarps;
constexpr int kMmaNB = 3;                      // D chunk buffers per set
constexpr int kMmaS = 2;                       // stages per warp (each: box t + box t-h)
constexpr int64_t kMmaStageBytes = 2 * kBoxBytes;

__host__ __device__ constexpr int mma_ks(int p) { return (p + 7) / 8; }          // K-steps of 8
__host__ __device__ constexpr int mma_a_cols(int p) { return 32 * mma_ks(p); }   // 2 groups x hi|lo x 8 KS
__host__ __device__ constexpr int mma_set_cols(int p) { return mma_a_cols(p) + kMmaNB * 64; }
// B table: [split hi|lo][K-step][8-date group][K chunk of 4][8 dates][4] floats: 256 B per
// (split, K-step, group) — K-major core matrices, LBO = 128 B (K chunk), SBO = 256 B (group)
__host__ __device__ constexpr int64_t mma_tab_bytes(int p, int groups) { return (int64_t)2 * mma_ks(p) * groups * 256; }

struct MmaGeom {
    int w0, t3;     // first date of the window-0 stream (pass 2) and of the monitoring stream (pass 3)
    int C2, C3;     // 16-date chunks of pass 2 / pass 3
    int gcur;       // 8-date groups of the current-date table: dates [w0, w0 + 8 gcur)
    int glag;       // 8-date groups of the lag table: dates [t3 - h, t3 - h + 8 glag)
};
__host__ __device__ inline MmaGeom mma_geom(int N, int n, int h) {
    MmaGeom g;
    g.w0 = ((n - h + 1) / 8) * 8;
    g.t3 = (n / 8) * 8;
    const int st2 = (n - g.w0 + 7) / 8, st3 = (N - g.t3 + 7) / 8;
    g.C2 = (st2 + 1) / 2;
    g.C3 = (st3 + 1) / 2;
    const int end = g.w0 + 16 * g.C2 > g.t3 + 16 * g.C3 ? g.w0 + 16 * g.C2 : g.t3 + 16 * g.C3;
    g.gcur = (end - g.w0) / 8;
    g.glag = 2 * g.C3;
    return g;
}
// shared-memory bytes of the MMA kernel (host mirror in bwm_capi.cu)
__host__ __device__ inline int64_t mma_smem_bytes(int N, int n, int h, int p) {
    const MmaGeom g = mma_geom(N, n, h);
    int64_t b = (int64_t)kMmaWarps * kMmaS * kMmaStageBytes;
    b += mma_tab_bytes(p, g.gcur) + mma_tab_bytes(p, g.glag);
    b += (int64_t)(((N - n) + 3) & ~3) * 4;                              // bound by monitoring date
    b += (int64_t)(kMmaWarps * kMmaS + kMmaSets * kMmaNB) * 8;          // mbarriers
    b += (int64_t)(kMmaSets * (kMmaNB + 1) + 4) * 4;                    // tickets + TMEM slot
    return b;
}

__device__ __forceinline__ uint32_t ticket(uint32_t* p) {
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(p)) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
// 8 consecutive 32-bit columns of this thread's lane (no wait)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

template <int NP, bool LEAN>
__global__ void __launch_bounds__(kMmaThreads, 1) monitor_kernel_mma(const __grid_constant__ KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int R = kStageRows;
    static_assert(R == 8 || NP < 0, "MMA kernel: 8-date stages (two per 16-date chunk)");
    constexpr int S = kMmaS;
    constexpr int64_t SB = kMmaStageBytes;
    constexpr int KS = mma_ks(NP), AC = mma_a_cols(NP), NB = kMmaNB;
    constexpr int ROWF2 = kWarpPx / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const MmaGeom G = mma_geom(N, n, h);
    const int NM = ((N - n) + 3) & ~3;
    unsigned char* s_stage = smem_raw;                                           // [8][S][SB]
    unsigned char* s_bc = s_stage + kMmaWarps * S * SB;                         // B table, current dates
    unsigned char* s_bl = s_bc + mma_tab_bytes(NP, G.gcur);                     // B table, lag dates
    float* s_bd = reinterpret_cast<float*>(s_bl + mma_tab_bytes(NP, G.glag));   // [N-n] bound by t - n
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_bd + NM);                   // [8][S] stage full
    uint64_t* s_dfull = s_bar + kMmaWarps * S;                                  // [2][NB] chunk ready
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_dfull + kMmaSets * NB);     // [2][NB] tickets
    uint32_t* s_bcnt = s_cnt + kMmaSets * NB;                                   // [2] beta tickets
    uint32_t* s_tmem = s_bcnt + kMmaSets;

    {   // stage the B tables (16-byte copies), the boundary and the per-tile stage schedule
        const uint4* src = reinterpret_cast<const uint4*>(prm.zb_cur);
        uint4* dst = reinterpret_cast<uint4*>(s_bc);
        const int nc = (int)(mma_tab_bytes(NP, G.gcur) / 16), nl = (int)(mma_tab_bytes(NP, G.glag) / 16);
        for (int i = threadIdx.x; i < nc; i += kMmaThreads) dst[i] = __ldg(src + i);
        src = reinterpret_cast<const uint4*>(prm.zb_lag);
        dst = reinterpret_cast<uint4*>(s_bl);
        for (int i = threadIdx.x; i < nl; i += kMmaThreads) dst[i] = __ldg(src + i);
        for (int i = threadIdx.x; i < N - n; i += kMmaThreads) s_bd[i] = prm.bound[i];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMmaWarps * S + kMmaSets * NB; ++s) mbar_init(s_bar + s, 1);
        for (int i = 0; i < kMmaSets * (NB + 1); ++i) s_cnt[i] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) tmem_alloc(s_tmem, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    const int tid = threadIdx.x, lane = tid & 31;
    const int wu = __shfl_sync(0xffffffffu, tid >> 5, 0);        // warp index (warp-uniform)
    const int set = wu >> 2, q = wu & 3;
    const int64_t n_tiles = prm.n_pixels / kTile;
    const int64_t tile_stride = (int64_t)gridDim.x * kMmaSets;
    const int64_t ld = prm.ld_y;
    const int wstart = n - h + 1;
    const int w0 = G.w0, t3 = G.t3;
    unsigned char* my_stage = s_stage + wu * S * SB;
    uint64_t* full = s_bar + wu * S;
    const uint32_t stage_u32 = smem_u32(my_stage), bar_u32 = smem_u32(full);
    const uint32_t tset = *s_tmem + (uint32_t)(set * 256);                     // this set's columns
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint64_t* dfull = s_dfull + set * NB;
    uint32_t* cnt = s_cnt + set * NB;
    const uint32_t bc_u32 = smem_u32(s_bc), bl_u32 = smem_u32(s_bl);
    const int NC = G.C2 + G.C3;                                                 // chunks per tile
    constexpr uint32_t kIdesc = idesc_tf32(16);

    // ---- MMA issue (one elected lane; the caller established the tcgen05 ordering) -------
    auto issue_chunk = [&](int j, int b) {
        const bool lagc = j >= G.C2;
        const int cdate = lagc ? t3 + 16 * (j - G.C2) : w0 + 16 * j;
        const int gc = (cdate - w0) / 8, gl = 2 * (j - G.C2);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const uint32_t ahi = tset + (uint32_t)(16 * KS * g), alo = ahi + 8 * KS;
            const uint32_t dcur = tset + AC + 64 * b + 32 * g, dlag = dcur + 16;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const uint64_t bh = smem_desc_kmajor(bc_u32 + (uint32_t)(((0 * KS + ks) * G.gcur + gc) * 256), 128, 256);
                const uint64_t bl = smem_desc_kmajor(bc_u32 + (uint32_t)(((1 * KS + ks) * G.gcur + gc) * 256), 128, 256);
                mma_tf32_ts(dcur, ahi + 8 * ks, bh, kIdesc, ks > 0 ? 1u : 0u);
                mma_tf32_ts(dcur, ahi + 8 * ks, bl, kIdesc, 1u);
                mma_tf32_ts(dcur, alo + 8 * ks, bh, kIdesc, 1u);
            }
            if (lagc) {
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const uint64_t bh = smem_desc_kmajor(bl_u32 + (uint32_t)(((0 * KS + ks) * G.glag + gl) * 256), 128, 256);
                    const uint64_t blo = smem_desc_kmajor(bl_u32 + (uint32_t)(((1 * KS + ks) * G.glag + gl) * 256), 128, 256);
                    mma_tf32_ts(dlag, ahi + 8 * ks, bh, kIdesc, ks > 0 ? 1u : 0u);
                    mma_tf32_ts(dlag, ahi + 8 * ks, blo, kIdesc, 1u);
                    mma_tf32_ts(dlag, alo + 8 * ks, bh, kIdesc, 1u);
                }
            }
        }
        mma_commit(smem_u32(dfull + b));
    };

    // ---- this warp's TMA issue cursor (as in bwm_kernel_tma.cuh, over its set's tiles) -----
    const int st1 = (n + R - 1) / R, st2 = (n - w0 + R - 1) / R;
    const int tile_stages = st1 + st2 + (N - t3 + R - 1) / R;
    int64_t itile = (int64_t)blockIdx.x * kMmaSets + set;
    int istage = 0;
    int xw = (int)(itile * kTile) + q * kWarpPx;
    auto issue_into = [&](int slot) {
        if (itile >= n_tiles) return;
        const int r0 = istage < st1 ? istage * R : istage < st1 + st2 ? w0 + (istage - st1) * R
                                                                       : t3 + (istage - st1 - st2) * R;
        const uint32_t dst = stage_u32 + (uint32_t)(slot * SB), bar = bar_u32 + (uint32_t)(slot * 8);
        if (istage >= st1 + st2)
            tma_box2_elect(dst, &prm.tmap, xw, r0, r0 - h, bar, 2 * kBoxBytes);   // + dates t-h
        else
            tma_box_elect(dst, &prm.tmap, xw, r0, bar, kBoxBytes);
        if (++istage == tile_stages) {
            istage = 0;
            itile += tile_stride;
            xw += (int)(tile_stride * kTile);
        }
    };
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&prm.tmap)) : "memory");
    for (int s = 0; s < S; ++s) issue_into(s);
    int cur = 0;
    uint32_t ph = 0, next_ready = 0;
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

    // fitted values of one stage (8 dates, both pixels) from chunk buffer b, half hf
    auto load_yhat = [&](int b, int hf, bool lagc, float2 (&yc)[R], float2 (&yl)[R]) {
        float a0[8], a1[8];
        const uint32_t base = tset + lane_off + AC + 64 * b + 8 * hf;
        tmem_ld8(base, a0);
        tmem_ld8(base + 32, a1);
        if (lagc) {
            float l0[8], l1[8];
            tmem_ld8(base + 16, l0);
            tmem_ld8(base + 48, l1);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < R; ++k) yl[k] = f2(l0[k], l1[k]);
        } else {
            tmem_wait_ld();
        }
#pragma unroll
        for (int k = 0; k < R; ++k) yc[k] = f2(a0[k], a1[k]);
    };
    int64_t gchunk = 0;                      // set-global chunk counter (parity of the buffers)
    // after the last stage of chunk j (buffer b): the last of the set's warps refills b
    auto chunk_done = [&](int j, int b) {
        tmem_fence_before();
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) last = (ticket(cnt + b) & 3u) == 3u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last && j + NB < NC) {
            tmem_fence_after();
            if (lane == 0) issue_chunk(j + NB, b);
            __syncwarp();
        }
    };

    for (int64_t tile = (int64_t)blockIdx.x * kMmaSets + set; tile < n_tiles; tile += tile_stride) {
        const int64_t px0 = tile * kTile + q * kWarpPx + 2 * lane;
        const float* yp = prm.y + px0;

        // ---- pass 1: beta_Q and ||y - c||^2 (FFMA2, 2Sum-compensated) — bwm_kernel_tma.cuh ----
        float2 hi[NP], lo[NP], part[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) { hi[i] = lo[i] = part[i] = f2(0.f, 0.f); }
        float2 qpart = f2(0.f, 0.f);
        double q0 = 0.0, q1 = 0.0;
        float2 c = f2(0.f, 0.f);
        bool f0 = false, f1 = false;
        float2 last = f2(0.f, 0.f), lastw = f2(0.f, 0.f);
        float2 negc = f2(0.f, 0.f);
        const float* s_mt = prm.xt;               // Q^T rows through L1 (uniform addresses)
        for (int t0 = 0; t0 < n; t0 += R) {
            const float2* st = acquire();
            if (t0 == 0) {
                const int rows = min(R, n);
#pragma unroll 1
                for (int k = rows - 1; k >= 0; --k) {
                    const float2 v = st[k * ROWF2];
                    if (finitef(v.x)) { c.x = v.x; f0 = true; }
                    if (finitef(v.y)) { c.y = v.y; f1 = true; }
                }
                if (!(f0 && f1)) {
                    for (int t = rows; t < N && !(f0 && f1); ++t) {
                        const float2 v = __ldg(reinterpret_cast<const float2*>(yp + (int64_t)t * ld));
                        if (!f0 && finitef(v.x)) { c.x = v.x; f0 = true; }
                        if (!f1 && finitef(v.y)) { c.y = v.y; f1 = true; }
                    }
                }
                negc = f2(-c.x, -c.y);
            }
            if (t0 + R <= n) {
                const float* mrow = s_mt + t0 * SP;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float2 vc = fill(st[k * ROWF2], negc, last);
                    axpy_row<NP, SP>(part, vc, mrow + k * SP);
                    qpart = fma2(vc, vc, qpart);
                }
            } else {
#pragma unroll 1
                for (int k = 0; k < n - t0; ++k) {
                    const float2 vc = fill(st[k * ROWF2], negc, last);
                    axpy_row<NP, SP>(part, vc, s_mt + (t0 + k) * SP);
                    qpart = fma2(vc, vc, qpart);
                }
            }
            release();
            if (t0 + R == w0) lastw = last;
            if (((t0 + R) & (kComp - 1)) == 0 || t0 + R >= n) {
#pragma unroll
                for (int i = 0; i < NP; ++i) { two_sum(hi[i], lo[i], part[i]); part[i] = f2(0.f, 0.f); }
                q0 += (double)qpart.x;
                q1 += (double)qpart.y;
                qpart = f2(0.f, 0.f);
            }
        }
        const bool valid0 = f0, valid1 = f1;
        float2 bq[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) bq[i] = add2(hi[i], lo[i]);
        const float2 ss = rss_onepass<NP>(q0, q1, bq);
        fix_flag(prm, valid0, q0, ss.x, px0);
        fix_flag(prm, valid1, q1, ss.y, px0 + 1);
        const bool z0 = zero_history(valid0, q0, c.x), z1 = zero_history(valid1, q1, c.y);
        if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0 + (z0 ? 0 : 1)));
        const float2 sc = sigma_scale(ss, prm.inv_dof, prm.sqrt_n, valid0, valid1);

        // ---- beta_Q -> the A operand: tf32 hi and lo halves, group g = pixel g of the pair -----
        {
            uint32_t ah[2][8 * KS], al[2][8 * KS];
#pragma unroll
            for (int i = 0; i < 8 * KS; ++i) {
                const float b0 = i < NP ? bq[i < NP ? i : 0].x : 0.f, b1 = i < NP ? bq[i < NP ? i : 0].y : 0.f;
                ah[0][i] = tf32_rna(b0);
                ah[1][i] = tf32_rna(b1);
                al[0][i] = tf32_rna(b0 - __uint_as_float(ah[0][i]));
                al[1][i] = tf32_rna(b1 - __uint_as_float(ah[1][i]));
            }
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    tmem_st8u(tset + lane_off + (uint32_t)(16 * KS * g + 8 * ks), *reinterpret_cast<const uint32_t(*)[8]>(&ah[g][8 * ks]));
                    tmem_st8u(tset + lane_off + (uint32_t)(16 * KS * g + 8 * KS + 8 * ks), *reinterpret_cast<const uint32_t(*)[8]>(&al[g][8 * ks]));
                }
            tmem_wait_st();
            tmem_fence_before();
            __syncwarp();
            uint32_t lastw_ = 0;
            if (lane == 0) lastw_ = (ticket(s_bcnt + set) & 3u) == 3u;
            lastw_ = __shfl_sync(0xffffffffu, lastw_, 0);
            if (lastw_) {                         // the set's beta rows are complete: first NB chunks
                tmem_fence_after();
                if (lane == 0)
                    for (int j = 0; j < NB && j < NC; ++j) issue_chunk(j, (int)((gchunk + j) % NB));
                __syncwarp();
            }
        }

        // ---- pass 2: window 0 (dates [w0, n), fitted values from the tensor cores) -----------
        float2 acc = f2(0.f, 0.f);
        float2 lag_last = w0 == wstart ? lastw : f2(0.f, 0.f);
        last = lastw;
        int sidx = 0;                              // stage index within the pass
        for (int t0 = w0; t0 < n; t0 += R, ++sidx) {
            const int j = sidx >> 1, hf = sidx & 1;
            const int b = (int)((gchunk + j) % NB);
            if (hf == 0) {
                mbar_wait(dfull + b, (uint32_t)(((gchunk + j) / NB) & 1));
                tmem_fence_after();
            }
            float2 yc[R], yl[R];
            load_yhat(b, hf, false, yc, yl);
            const float2* st = acquire();
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int t = t0 + k;
                if (t < n) {
                    const float2 r = sub2(fill(st[k * ROWF2], negc, last), yc[k]);
                    if (t >= wstart) acc = add2(acc, r);
                    if (t == wstart - 1) lag_last = last;
                }
            }
            release();
            if (hf == 1 || t0 + R >= n) chunk_done(j, b);
        }

        // ---- pass 3: monitoring period, fused MOSUM + detect (unscaled frame) --------------
        float2 mx = f2(0.f, 0.f), msum = f2(0.f, 0.f), sr = f2(0.f, 0.f);
        int first0 = 0x7fffffff, first1 = 0x7fffffff;
        float* const mo_out = prm.mosum;
        const bool want_sup = prm.sup != nullptr;
        const float2 inv = inv_scale(sc);
        const float2 bsc = mul2(sc, f2(s_bd[0], s_bd[0]));
        auto step = [&](const float2 r, const float2 old, const int t, const float bj) {
            acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
            const float2 bs = LEAN ? bsc : mul2(sc, f2(bj, bj));
            const float a0 = fabsf(acc.x), a1 = fabsf(acc.y);
            mx.x = fmaxf(mx.x, a0);
            mx.y = fmaxf(mx.y, a1);
            const int j1 = t - n + 1;
            if (a0 > bs.x) first0 = min(first0, j1);  // strict crossing (_kernels.py:47)
            if (a1 > bs.y) first1 = min(first1, j1);
            if (!LEAN) {
                if (want_sup) {
                    sr.x = fmaxf(sr.x, __fdividef(a0, bj));
                    sr.y = fmaxf(sr.y, __fdividef(a1, bj));
                }
                msum = add2(msum, acc);
                if (mo_out) *reinterpret_cast<float2*>(mo_out + (int64_t)(t - n) * prm.ld_out + px0) = mul2(acc, inv);
            }
        };
        sidx = 0;
        for (int t0 = t3; t0 < N; t0 += R, ++sidx) {
            const int j = G.C2 + (sidx >> 1), hf = sidx & 1;
            const int b = (int)((gchunk + j) % NB);
            if (hf == 0) {
                mbar_wait(dfull + b, (uint32_t)(((gchunk + j) / NB) & 1));
                tmem_fence_after();
            }
            float2 yc[R], yl[R];
            load_yhat(b, hf, true, yc, yl);
            const float2* st = acquire();
            const float2* lst = st + kBoxBytes / 8;      // lag dates: second box
            if (t0 >= n + 1 && t0 + R <= N) {
                float2 acck[R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const int t = t0 + k;
                    const float2 r = sub2(fill(st[k * ROWF2], negc, last), yc[k]);
                    const float2 old = sub2(fill(lst[k * ROWF2], negc, lag_last), yl[k]);
                    if (LEAN) {
                        acc = add2(acc, sub2(r, old));
                        acck[k] = acc;
                        mx.x = fmaxf(mx.x, fabsf(acc.x));
                        mx.y = fmaxf(mx.y, fabsf(acc.y));
                    } else {
                        step(r, old, t, s_bd[t - n]);
                    }
                }
                if (LEAN) {
                    if (first0 == 0x7fffffff && mx.x > bsc.x) {
#pragma unroll
                        for (int k = R - 1; k >= 0; --k)
                            if (fabsf(acck[k].x) > bsc.x) first0 = t0 + k - n + 1;
                    }
                    if (first1 == 0x7fffffff && mx.y > bsc.y) {
#pragma unroll
                        for (int k = R - 1; k >= 0; --k)
                            if (fabsf(acck[k].y) > bsc.y) first1 = t0 + k - n + 1;
                    }
                }
            } else {
                const int k0 = max(0, n - t0), k1 = min(R, N - t0);
#pragma unroll 1
                for (int k = k0; k < k1; ++k) {
                    const int t = t0 + k;
                    float2 yck = yc[0], ylk = yl[0];
#pragma unroll
                    for (int kk = 1; kk < R; ++kk)
                        if (kk == k) { yck = yc[kk]; ylk = yl[kk]; }
                    const float2 r = sub2(fill(st[k * ROWF2], negc, last), yck);
                    float2 old = f2(0.f, 0.f);
                    if (t > n) old = sub2(fill(lst[k * ROWF2], negc, lag_last), ylk);   // r_{n-h}: outside window 0
                    step(r, old, t, s_bd[t - n]);
                }
            }
            release();
            if (hf == 1 || t0 + R >= N) chunk_done(j, b);
        }
        gchunk += NC;

        // ---- outputs --------------------------------------------------------------------
        const float inv_m = 1.0f / (float)(N - n);
        *reinterpret_cast<uchar2*>(prm.valid + px0) = make_uchar2(valid0, valid1);
        *reinterpret_cast<int2*>(prm.first_idx + px0) =
            make_int2(first0 == 0x7fffffff ? 0 : first0, first1 == 0x7fffffff ? 0 : first1);
        *reinterpret_cast<float2*>(prm.max_abs + px0) = mul2(mx, inv);
        if (!LEAN && prm.mo_mean) *reinterpret_cast<float2*>(prm.mo_mean + px0) = mul2(mul2(msum, inv), f2(inv_m, inv_m));
        if (want_sup) {
            const float2 s = LEAN ? mul2(mul2(mx, inv), f2(1.0f / s_bd[0], 1.0f / s_bd[0])) : mul2(sr, inv);
            *reinterpret_cast<float2*>(prm.sup + px0) = s;
        }
        if (prm.beta) store_beta<NP>(prm, px0, c, bq, valid0, valid1, 2);
    }

    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (tid < 32) tmem_dealloc(*s_tmem, 512);
}

}  // namespace bwm
