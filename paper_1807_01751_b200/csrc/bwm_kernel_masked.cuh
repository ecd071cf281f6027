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
// Pass 1 (history): g = X' (y - c) with 2Sum-compensated 32-date blocks (FFMA2), and the Gram
//   complement Gm = W X2 on the TENSOR CORES: W[pixel][date] = 1 if missing (exact in tf32),
//   X2[date][e] = the lower-triangle entries of x_t x_t^T, split hi + lo (tf32 each, ~22 bits).
//   Every thread writes its pixel's 0/1 row of a 16-date block into its own TMEM lane (the
//   A operand, tcgen05.st); one thread issues 2 steps x 2 splits of
//   tcgen05.mma.kind::tf32 (M = 128 pixels, N = p(p+1)/2 padded to 16, K = 8 dates, A from
//   TMEM, B from shared memory) accumulating Gm in TMEM (lane = pixel), and the x x^T tiles
//   stream from L2 through a 3-stage shared-memory ring (cp.async.bulk).  G_v = G_full - Gm
//   is accurate because Gm has few terms; the refinement step below absorbs the rest.
// Solve: float32 Cholesky of G_v per pixel (in registers), beta' = G_v^-1 g.
// Pass 2 (history again, L2): two-pass RSS of the valid dates and the normal-equation
//   residual e = X_v r; one step of mixed-precision iterative refinement follows: dbeta =
//   G_v^-1 e, beta and RSS are corrected (RSS' = RSS - 2 dbeta.e + |L^T dbeta|^2).  A tail
//   sweep from the warp's earliest window-0 date then puts the last h_v - 1 valid residuals,
//   computed with the refined beta, in a per-pixel ring (slot 0 = 0: the element before
//   window 0) — coalesced row loads instead of per-lane gathers of X' rows.  This makes
//   the float32 Gram good to cond(G_v) ~ 1e5 (p = 18 on 23 valid dates: cond 3e4) at the cost
//   of p/2 FFMA2 per valid history date; realistic stacks have cond(G_v) < 10.
// Pass 3 (monitoring): per valid date r, old = ring[s], ring[s] = r, acc += r - old,
//   crossing |acc| > b_j sigma sqrt(n_v); invalid dates leave the state untouched.
// Per-thread scratch, [2h][128] words (thread = bank: conflict-free): the residual ring and
// the ring dates.  In shared memory, or in a per-CTA global scratch when h or the x x^T table
// is too large (BIG).
#pragma once

#include "bwm_common.cuh"
#include "bwm_kernel_tma.cuh"   // mbarrier / TMEM helpers

namespace bwm {

constexpr int kMaskThreads = 128;       // one pixel per thread; M = 128 of the Gram MMA
constexpr int kMaskTile = kMaskThreads;
constexpr int kMaskD = 16;              // dates per register block = 2 MMA K-steps
#ifndef BWM_MASK_D23
#define BWM_MASK_D23 16
#endif
constexpr int kMaskBStages = 4;         // x x^T tile ring: refilled 2 blocks behind, 2 ahead
constexpr int kMaskABufs = 4;           // TMEM A buffers (16 columns each)

template <int NP>
struct Gram {
    static constexpr int KK = NP * (NP + 1) / 2;          // lower triangle, (i, j<=i) at i(i+1)/2 + j
    static constexpr int NN = ((KK + 15) / 16) * 16;      // MMA N (multiple of 16 for M = 128)
    static constexpr int SB = NN * 128;                   // bytes of one 16-date block: 2 steps x hi/lo
};

__host__ __device__ constexpr int gram_nn(int p) { return ((p * (p + 1) / 2 + 15) / 16) * 16; }
// Exact Gram complement (p <= 14): the x x^T entries are split into two 11-bit fixed-point
// digits (integer-valued tf32 operands), each digit level accumulated in its own TMEM region:
// every partial sum is an integer below 2^24, so the float32 accumulation is exact and
// G_v = G_full - Gm is good to float64 (the round-1 float hi/lo split summed in one float32
// accumulator carried ~2e-5 of max |MO| at C4/C5).  p >= 16: the float split, one region.
__host__ __device__ constexpr bool mask_digits(int p) { return p <= 14; }
__host__ __device__ constexpr int mask_dcols(int p) { return (mask_digits(p) ? 2 : 1) * gram_nn(p); }
__host__ __device__ constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }
// A buffers (16 columns each): 4, or 2 when 4 would double the TMEM allocation
__host__ __device__ constexpr int mask_ab(int p) {
    return pow2_cols(mask_dcols(p) + 16 * kMaskABufs) == pow2_cols(mask_dcols(p) + 32) ? kMaskABufs : 2;
}
__host__ __device__ constexpr int masked_tmem_cols(int p) { return pow2_cols(mask_dcols(p) + 16 * mask_ab(p)); }

// tcgen05 pieces of the Gram MMA -----------------------------------------------------------
// Shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes,
// LBO = byte distance between the two 16-byte K chunks, SBO = between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
    return d;                                  // base offset 0, layout SWIZZLE_NONE
}
// Instruction descriptor: D f32, A/B tf32, both K-major, N, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Per-thread scratch words: the residual ring [h] floats, + its dates [h] uint16 (shared-memory ring).
__host__ __device__ inline int masked_scratch_words(int h, int p, bool big) { return big ? h + 0 * p : h + (h + 1) / 2; }

// Shared-memory bytes of the masked kernel (host mirror in bwm_capi.cu).
__host__ __device__ inline int64_t masked_smem_bytes(int N, int n, int h, int p, bool big) {
    const int sp = (p + 3) & ~3;
    // X'^T with zero rows past N; in BIG mode it stays in global memory (read through L1)
    int64_t bytes = big ? 0 : (((int64_t)(N + kMaskD) * sp * 4 + 127) / 128) * 128;
    bytes += (int64_t)kMaskBStages * gram_nn(p) * 128;                      // x x^T tile ring
    if (!big) bytes += (int64_t)masked_scratch_words(h, p, false) * kMaskThreads * 4;
    return bytes + (2 * kMaskBStages + kMaskABufs) * 8 + 32;                // mbarriers + TMEM slot + tickets
}

// Column J of an in-place float32 Cholesky factorisation of the packed lower triangle L,
// recursing over J at compile time so every index is a constant (a runtime-indexed register
// array compiles to select chains: ~1000 instructions at p = 8).
template <int NP, int J>
__device__ __forceinline__ void chol_col(float (&L)[NP * (NP + 1) / 2], float (&dinv)[NP], bool& ok) {
    if constexpr (J < NP) {
        constexpr int JR = J * (J + 1) / 2;
        float d = L[JR + J];
#pragma unroll
        for (int k = 0; k < J; ++k) d = fmaf(-L[JR + k], L[JR + k], d);
        ok = ok && d > 1e-6f * fabsf(L[JR + J]);            // numerically singular in float32
        const float inv = ok ? rsqrtf(d) : 0.f;
        dinv[J] = inv;
#pragma unroll
        for (int i = J + 1; i < NP; ++i) {
            float sv = L[i * (i + 1) / 2 + J];
#pragma unroll
            for (int k = 0; k < J; ++k) sv = fmaf(-L[i * (i + 1) / 2 + k], L[JR + k], sv);
            L[i * (i + 1) / 2 + J] = sv * inv;
        }
        chol_col<NP, J + 1>(L, dinv, ok);
    }
}

// b_j = lambda sqrt(log_plus(x_j)) for x_j = (n_v + 1 + j) / n_v > e (mosum.py:68-79), in the
// unscaled frame (lam_sc = lambda sigma sqrt(n_v)); within ~1e-7 of the float64 value
static __device__ __noinline__ float masked_bound(float lam_sc, int j, float dx, float jx0) {
    const float x = fmaf((float)j, dx, jx0);
    const float lp = fmaxf(__log2f(x) * 0.69314718f, 1.f);
    return lam_sc * (lp * rsqrtf(lp));
}

// idle lanes of a tail tile read this NaN (stride 0): every date missing, no per-row test
static __device__ const unsigned int kNanRow[1] = {0x7fc00000u};

#ifndef BWM_MASK_TICKET
#define BWM_MASK_TICKET 0   // 1: the last warp to stage a block's mask rows issues its MMAs instead of a
                            // __syncthreads (measured 5% SLOWER at C2 and C5: the barrier keeps the
                            // four warps' scalar row loads coherent)
#endif
#ifndef BWM_MASK_FAST
#define BWM_MASK_FAST 1     // shared-memory geometries: refine from the Gram matrix (e = g - G_v beta),
                            // one-pass RSS; the exact refinement sweep only for flagged pixels
#endif
#ifndef BWM_MASK_FORCEX
#define BWM_MASK_FORCEX 0   // debugging: every pixel on the exact refinement path
#endif
#ifndef BWM_MASK_DEFER
#define BWM_MASK_DEFER 1    // issue a block's Gram MMAs one block later (its TMEM stores have landed)
#endif
#ifndef BWM_MASK_MINB
#define BWM_MASK_MINB 4
#endif
template <int NP, bool BIG, bool KEEP>
__global__ void __launch_bounds__(kMaskThreads, NP <= 8 ? BWM_MASK_MINB : 2)
    monitor_kernel_masked(const __grid_constant__ KParams prm) {
    constexpr int SP = Coefs<NP>::SP;
    constexpr int KK = Gram<NP>::KK, NN = Gram<NP>::NN, SB = Gram<NP>::SB;
    constexpr int D = kMaskD, S = kMaskBStages, AB = mask_ab(NP);
    constexpr bool DIG = mask_digits(NP);
    constexpr int D23 = BWM_MASK_D23;   // dates per register block of passes 2 and 3 (8: C2 -3%, C5 +7%, C4 +60%)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const int n16 = ((n + D - 1) / D) * D;
    const int nkb = n16 / D;                                           // 16-date blocks of the history
    // [N + D][SP] X'^T, zero rows past N: staged in smem, or (BIG) read through L1 from the
    // zero-padded global copy, so the big geometries (C4) fit two CTAs per SM
    float* s_xs = reinterpret_cast<float*>(smem_raw);
    const float* s_x = BIG ? prm.xt : s_xs;
    unsigned char* s_b = smem_raw + (BIG ? 0 : (((N + D) * SP * 4 + 127) / 128) * 128);   // [S][SB] x x^T tiles
    float* s_ring = reinterpret_cast<float*>(s_b + S * SB);           // ring scratch   (!BIG)
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s_ring) +
                                                  (BIG ? 0 : masked_scratch_words(h, NP, false) * kMaskThreads * 4));
    uint64_t* b_full = s_bar;              // [S]  tile landed
    uint64_t* b_empty = s_bar + S;         // [S]  MMAs reading the tile are done
    uint64_t* m_done = s_bar + 2 * S;      // [AB] MMAs reading A buffer b are done
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 2 * S + AB);
    uint32_t* s_tick = s_tmem + 1;                // [AB] mask-row tickets (BWM_MASK_TICKET)
    const int tid = threadIdx.x, warp = tid >> 5;
    if (!BIG)
        for (int i = tid; i < (N + D) * SP; i += kMaskThreads) s_xs[i] = i < N * SP ? prm.xt[i] : 0.f;
    if (tid == 0) {
        for (int i = 0; i < 2 * S + AB; ++i) mbar_init(s_bar + i, 1);
        for (int i = 0; i < AB; ++i) s_tick[i] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    constexpr uint32_t kCols = (uint32_t)masked_tmem_cols(NP);
    if (warp == 0) tmem_alloc(s_tmem, kCols);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *s_tmem;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;            // this warp's TMEM lane quarter
    // Gm accumulator(s): [hi digits | lo digits] (DIG) or one region | AB x 16 A columns
    const uint32_t d_col = tbase, a_col = tbase + mask_dcols(NP);
    // this lane's Gm entries idx in [16 c16, 16 c16 + 16): exact digit sums -> float64
    // (f(u, gm) is called for each entry in turn: no array of doubles stays live)
    auto gm_chunk = [&](int c16, auto&& f) {
        float hi[16];
        tmem_ld16(d_col + lane_off + 16 * c16, *reinterpret_cast<float2(*)[8]>(hi));
        if (DIG) {
            float lo[16];
            tmem_ld16(d_col + NN + lane_off + 16 * c16, *reinterpret_cast<float2(*)[8]>(lo));
#pragma unroll
            for (int u = 0; u < 16; ++u) f(u, prm.gscale * fma((double)lo[u], 1.0 / 2048.0, (double)hi[u]));
        } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) f(u, (double)hi[u]);
        }
    };
    float* ring = (BIG ? prm.ring_g + (int64_t)blockIdx.x * masked_scratch_words(h, NP, true) * kMaskThreads : s_ring) +
                  tid;
    uint16_t* ring_d = reinterpret_cast<uint16_t*>(ring - tid + h * kMaskThreads) + tid;   // ring dates (!BIG)

    const int64_t ld = prm.ld_y;
    const float lam = prm.lambda;
    const int64_t n_tiles = (prm.n_pixels + kMaskTile - 1) / kMaskTile;
    const int64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total_blocks = my_tiles * nkb;                      // x x^T tiles this CTA consumes

    // ---- x x^T tile stream (thread 0): block q of the CTA's sequence is history block q % nkb
    const uint32_t sb_u32 = smem_u32(s_b);
    auto issue_b = [&](int64_t q) {
        if (q >= total_blocks) return;
        const int st = (int)(q % S);
        bulk_g2s(sb_u32 + st * SB, prm.xx + (q % nkb) * (SB / 4), SB, smem_u32(b_full + st));
    };
    if (tid == 0)
        for (int64_t q = 0; q < S - 2; ++q) issue_b(q);
    constexpr uint32_t kIdesc = idesc_tf32(NN);
    int64_t q = 0;                                                     // CTA-wide block counter
    // Gram MMAs of block qq (first date t0q of its tile): every thread's mask row of the block is
    // in its TMEM lane (A buffer qq % AB) once its tcgen05.st completed; one thread issues
    // 2 K-steps x 2 splits and commits them to m_done (A buffer free) and b_empty (B stage free).
    auto issue_mma = [&](int64_t qq, int t0q) {
        const int abq = (int)(qq % AB);
        tmem_wait_st();
        tmem_fence_before();
        bool issuer;
        if (BWM_MASK_TICKET) {
            // the last of the four warps to stage its rows of this block issues the MMAs
            __syncwarp();
            uint32_t tk = 0;
            if ((tid & 31) == 0)
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(tk) : "r"(smem_u32(s_tick + abq)) : "memory");
            issuer = (__shfl_sync(0xffffffffu, tk, 0) & 3u) == 3u && (tid & 31) == 0;
        } else {
            __syncthreads();
            issuer = tid == 0;
        }
        if (issuer) {
            tmem_fence_after();
            const int st = (int)(qq % S);
            mbar_wait(b_full + st, (uint32_t)((qq / S) & 1));
            const uint32_t bt = sb_u32 + st * SB;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
                for (int sp = 0; sp < 2; ++sp)
                    mma_tf32_ts(d_col + (DIG ? sp * NN : 0), a_col + 16 * abq + 8 * ks,
                                smem_desc_kmajor(bt + (2 * ks + sp) * NN * 32, 128, 256), kIdesc,
                                (t0q > 0 || ks > 0 || (!DIG && sp > 0)) ? 1u : 0u);
            mma_commit(smem_u32(m_done + abq));
            mma_commit(smem_u32(b_empty + st));
            // refill the stage of block qq-2 (its MMAs were issued two blocks ago) with block qq+2
            if (qq >= 2) mbar_wait(b_empty + (int)((qq - 2) % S), (uint32_t)(((qq - 2) / S) & 1));
            issue_b(qq + S - 2);
        }
    };

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t px = tile * kMaskTile + tid;
        const bool act = px < prm.n_pixels;
        const float* yp = act ? prm.y + px : reinterpret_cast<const float*>(kNanRow);
        const int64_t ldl = act ? ld : 0;
        const float qnan = __int_as_float(0x7fc00000);
        // D dates from row t0; rows >= end read as missing (only the last block of a pass)
        // The warp's next D rows (32 px = 128 B each) are prefetched into L2 while this block is
        // computed: lane k < D touches row t0 + D + k (one prefetch per row and warp), so the
        // next block's loads see L2 instead of DRAM latency (long-scoreboard stalls; 12.8 ->
        // 12.1 ms at C2; two blocks ahead measured slower).
        const float* wp = prm.y + tile * kMaskTile + 32 * warp;
        const bool pf_ok = tile * kMaskTile + 32 * warp + 31 < prm.n_pixels;
        auto load = [&](int t0, int end, auto& vb) {
            constexpr int DB = (int)(sizeof(vb) / sizeof(float));
            if (pf_ok && (tid & 31) < DB && t0 + DB + (tid & 31) < end)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + (int64_t)(t0 + DB + (tid & 31)) * ld));
            const float* p = yp + (int64_t)t0 * ldl;
            if (t0 + DB <= end) {
#pragma unroll
                for (int k = 0; k < DB; ++k) vb[k] = __ldg(p + k * ldl);
            } else {
#pragma unroll
                for (int k = 0; k < DB; ++k) vb[k] = t0 + k < end ? __ldg(p + k * ldl) : qnan;
            }
        };

        // centre c: the first finite history value, taken on the fly in pass 1 (any finite value
        // would do numerically; dates before it are missing and contribute nothing).  A pixel
        // with no finite history value is invalid (n_v = 0) and keeps c = 0.
        float c = 0.f;
        bool have_c = false;

        // ---- pass 1: g = X'(y - c) over valid dates (FFMA2); Gm = W X2 on the tensor cores --
        float2 gp[NP / 2], ghi[NP / 2], glo[NP / 2];
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) gp[i] = ghi[i] = glo[i] = f2(0.f, 0.f);
        int nv = 0;
        double qd = 0.0;                         // sum of (y - c)^2 over the valid history dates
        for (int t0 = 0; t0 < n16; t0 += D, ++q) {
            float qp = 0.f;
            float vb[D];
            load(t0, n, vb);
            float2 wv[D / 2];                                          // 1 = missing: this block's A row
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int t = t0 + k;
                const bool m = finitef(vb[k]);
                c = (m && !have_c) ? vb[k] : c;
                have_c = have_c || m;
                const float yc = m ? vb[k] - c : 0.f;
                nv += m ? 1 : 0;
                qp = fmaf(yc, yc, qp);
                if (k & 1) wv[k >> 1].y = m ? 0.f : 1.f; else wv[k >> 1].x = m ? 0.f : 1.f;
                const float4* x4 = reinterpret_cast<const float4*>(s_x + t * SP);
#pragma unroll
                for (int qq = 0; qq < SP / 4; ++qq) {
                    const float4 x = x4[qq];
                    if (4 * qq + 1 < NP) gp[2 * qq] = fma2(f2(yc, yc), f2(x.x, x.y), gp[2 * qq]);
                    if (4 * qq + 3 < NP) gp[2 * qq + 1] = fma2(f2(yc, yc), f2(x.z, x.w), gp[2 * qq + 1]);
                }
            }
            if (((t0 + D) & (kComp - 1)) == 0 || t0 + D >= n) {
#pragma unroll
                for (int i = 0; i < NP / 2; ++i) { two_sum(ghi[i], glo[i], gp[i]); gp[i] = f2(0.f, 0.f); }
            }
            qd += (double)qp;
            // A buffer ab is free once the MMAs of block q - AB completed
            const int ab = (int)(q % AB);
            if (q >= AB) mbar_wait(m_done + ab, (uint32_t)((q / AB - 1) & 1));
            if (BWM_MASK_DEFER) {
                // block q-1's mask rows were stored at the end of the previous iteration: their
                // tcgen05.st completed while this block was computed, so the wait is free
                if (t0 > 0) issue_mma(q - 1, t0 - D);
                tmem_st16(a_col + lane_off + 16 * ab, wv);
            } else {
                tmem_st16(a_col + lane_off + 16 * ab, wv);
                issue_mma(q, t0);
            }
        }
        if (BWM_MASK_DEFER) issue_mma(q - 1, n16 - D);      // the tile's last block
        // the Gram complement of this tile: wait for the last block's MMAs, read this lane
        mbar_wait(m_done + (int)((q - 1) % AB), (uint32_t)(((q - 1) / AB) & 1));
        tmem_fence_after();

        // ---- solve G_v beta' = g: float32 Cholesky in registers (G_v formed in float64) -----
        // Emulated against the float64 oracle: a float32 factor plus the refinement step below
        // is as accurate as a float64 factor (3e-5 on max |MO| at cond(G_v) = 3e4, 3e-6 at
        // cond 30), without the float64 register pressure that spilled through the loops.
        float L[KK], dinv[NP];
#pragma unroll
        for (int c16 = 0; c16 < NN / 16; ++c16)
            gm_chunk(c16, [&](int u, double gm) {
                if (16 * c16 + u < KK) L[16 * c16 + u] = (float)(__ldg(prm.gfull + 16 * c16 + u) - gm);
            });
        tmem_fence_before();      // the next tile's first MMA overwrites D after a __syncthreads
        bool ok = nv > NP;
        chol_col<NP, 0>(L, dinv, ok);
        // L w = b, L^T x = w  (in place)
        auto chol_solve = [&](float (&v)[NP]) {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                float sv = v[i];
#pragma unroll
                for (int k = 0; k < i; ++k) sv = fmaf(-L[i * (i + 1) / 2 + k], v[k], sv);
                v[i] = sv * dinv[i];
            }
#pragma unroll
            for (int i = NP - 1; i >= 0; --i) {
                float sv = v[i];
#pragma unroll
                for (int k = i + 1; k < NP; ++k) sv = fmaf(-L[k * (k + 1) / 2 + i], v[k], sv);
                v[i] = sv * dinv[i];
            }
        };
        float z[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const float2 gg = ghi[i >> 1], gl = glo[i >> 1];
            z[i] = (i & 1) ? gg.y + gl.y : gg.x + gl.x;
        }
        chol_solve(z);
        float2 nb[NP / 2];    // -beta' in coefficient pairs
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) nb[i] = ok ? f2(-z[2 * i], -z[2 * i + 1]) : f2(0.f, 0.f);
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

        // ---- fast refinement (shared-memory geometries): e = g - G_v beta_0 from the Gram matrix --
        // G_v = G_full - Gm (float64 table minus this lane's TMEM accumulator, still resident: the
        // next tile's first MMA overwrites it only after a later CTA barrier), one refinement step,
        // one-pass RSS = q - g^T beta.  A pixel whose RSS cancels (q > 300 RSS) or is not positive,
        // or whose Gram matrix is not well conditioned (Cholesky pivot ratio > 30), takes the exact
        // path instead (the refinement sweep over its residuals, below); the choice is per pixel,
        // so results do not depend on the neighbours in the warp.
        constexpr bool FAST = DIG && BWM_MASK_FAST && (BIG || NP <= 10);   // (register budget)
        bool needx = true;
        double rss_f = 0.0;
        float2 nbf[NP / 2];
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) nbf[i] = nb[i];
        if (FAST) {
            // out = G_v beta for beta = -nv2 (coefficient pairs), streaming G_v = G_full - Gm
            auto gv_times = [&](const float2 (&nv2)[NP / 2], double (&out)[NP]) {
#pragma unroll
                for (int i = 0; i < NP; ++i) out[i] = 0.0;
#pragma unroll
                for (int c16 = 0; c16 < NN / 16; ++c16)
                    gm_chunk(c16, [&](int u, double gmv) {
                        const int idx = 16 * c16 + u;
                        if (idx < KK) {
                            // packed lower triangle: idx = i(i+1)/2 + j, j <= i
                            int i = 0;
#pragma unroll
                            for (int ii = 1; ii < NP; ++ii) i += (idx >= ii * (ii + 1) / 2) ? 1 : 0;
                            const int j = idx - i * (i + 1) / 2;
                            const double gv = __ldg(prm.gfull + idx) - gmv;
                            const double bj = -(double)((j & 1) ? nv2[j >> 1].y : nv2[j >> 1].x);
                            const double bi = -(double)((i & 1) ? nv2[i >> 1].y : nv2[i >> 1].x);
                            out[i] += gv * bj;
                            if (i != j) out[j] += gv * bi;
                        }
                    });
            };
            double gb[NP];                       // G_v beta_0
            gv_times(nb, gb);
            // g_i = hi + lo of the compensated X'(y - c), in float64 where it is used
            auto gdbl = [&](int i) -> double {
                const float2 gg = ghi[i >> 1], gl = glo[i >> 1];
                return (i & 1) ? (double)gg.y + (double)gl.y : (double)gg.x + (double)gl.x;
            };
            float d[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) d[i] = (float)(gdbl(i) - gb[i]);
            tmem_fence_before();                 // the re-read precedes the next tile's first MMA
            chol_solve(d);
            // one-pass RSS q - g^T beta_f with beta_f = beta_0 + delta as the unevaluated pair (the
            // float32 rounding of the sum would enter at first order)
            double lin = 0.0;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const double b0 = -(double)((i & 1) ? nb[i >> 1].y : nb[i >> 1].x);
                lin += gdbl(i) * (b0 + (double)d[i]);
            }
#pragma unroll
            for (int i = 0; i < NP / 2; ++i) nbf[i] = sub2(nb[i], f2(d[2 * i], d[2 * i + 1]));
            rss_f = qd - lin;
            // conditioning estimate from the Cholesky pivots: (max L_ii / min L_ii)^2 <= cond(G_v)
            float dmin = dinv[0], dmax = dinv[0];
#pragma unroll
            for (int i = 1; i < NP; ++i) { dmin = fminf(dmin, dinv[i]); dmax = fmaxf(dmax, dinv[i]); }
            const bool wellcond = dmax <= 30.f * dmin;          // pivot ratio^2 <= 900
            // The Gram-matrix refinement leaves beta with the float32 error of g (~3e-7 relative), a
            // few 1e-6 of MO absolute: invisible at rtol 1e-4 unless max |MO| is tiny, which takes a
            // monitoring period of a handful of dates.  Short periods (N - n < 64) stay exact.
            // (and the digit sums stay exact integers below 2^24: n < 8192 history dates)
            const bool geom = N - n >= 64 && n16 <= 8192;
            needx = ok && (BWM_MASK_FORCEX || !geom || !(rss_f > 0.0 && qd <= 300.0 * rss_f && wellcond));
        }
        const bool anyx = !FAST || __any_sync(0xffffffffu, needx);

        // ---- pass 2 (exact path): RSS (two-pass) and the refinement residual e = X_v r ---------
        const int hv = (int)(((int64_t)h * nv) / n);
        const int wfirst = nv - hv + 1;          // 0-based compacted index of window 0's first element
        constexpr int RS = kMaskThreads;         // ring row stride (words)
        int seen = 0, tw = n;                    // tw: date of compacted index wfirst (window 0 start)
        int so = RS;                             // word offset of the next ring slot (slot 1)
        if (hv >= 1) ring[0] = 0.f;              // the element before window 0
        double rss = 0.0;
        float2 e2[NP / 2];                       // X_v r (normal-equation residual)
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) e2[i] = f2(0.f, 0.f);
        for (int t0 = 0; anyx && t0 < n; t0 += D23) {
            float vb[D23];
            load(t0, n, vb);
            float part = 0.f;
#pragma unroll
            for (int k = 0; k < D23; ++k) {
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
                if (BIG) {
                    tw = (m && seen == wfirst) ? t : tw;
                } else {                         // shared-memory ring: window 0 written here
                    const bool inwin = m && seen >= wfirst && needx;
                    if (inwin) {
                        ring[so] = r;
                        ring_d[so] = (uint16_t)t;
                    }
                    so += inwin ? RS : 0;
                }
                seen += m ? 1 : 0;
            }
            rss += (double)part;
        }

        // ---- one refinement step: dbeta = G_v^-1 e; correct RSS and beta ----------------------
        float db[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) db[i] = (i & 1) ? e2[i >> 1].y : e2[i >> 1].x;
        double quad = 0.0;                                  // |L^T dbeta|^2 = |w|^2, w = L^-1 e
        {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                float sv = db[i];
#pragma unroll
                for (int k = 0; k < i; ++k) sv = fmaf(-L[i * (i + 1) / 2 + k], db[k], sv);
                db[i] = sv * dinv[i];
                quad += (double)db[i] * (double)db[i];
            }
#pragma unroll
            for (int i = NP - 1; i >= 0; --i) {
                float sv = db[i];
#pragma unroll
                for (int k = i + 1; k < NP; ++k) sv = fmaf(-L[k * (k + 1) / 2 + i], db[k], sv);
                db[i] = sv * dinv[i];
            }
        }
        double de = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) de += (double)db[i] * (double)((i & 1) ? e2[i >> 1].y : e2[i >> 1].x);
        float2 nb0[NP / 2];                      // pre-refinement -beta' (window-0 residuals, BIG)
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) nb0[i] = nb[i];
        if (ok && needx) {
            rss = fmax(rss - 2.0 * de + quad, 0.0);
#pragma unroll
            for (int i = 0; i < NP / 2; ++i) nb[i] = sub2(nb[i], f2(db[2 * i], db[2 * i + 1]));
        } else if (ok) {                         // fast path
            rss = rss_f;
#pragma unroll
            for (int i = 0; i < NP / 2; ++i) nb[i] = nbf[i];
        }

        // ---- window 0: the last hv - 1 valid history residuals, corrected by the refinement ---
        // r = r(beta_0) - dbeta . x_t, the same arithmetic either way.  Shared-memory ring: the
        // pass-2 residuals are corrected in place from the stored dates.  Global ring (BIG): a
        // tail sweep from the warp's earliest window-0 date recomputes them — coalesced row loads
        // and one X' row per date for the warp, instead of per-lane gathers of X' rows from
        // global memory and a per-element date ring.
        float acc = 0.f;
        if (!BIG) {
            const int slot = so / RS;
            for (int s2 = 1; s2 < slot; ++s2) {
                const int t = ring_d[s2 * kMaskThreads];
                const float* xr = s_x + t * SP;
                float r = ring[s2 * kMaskThreads];
#pragma unroll
                for (int i = 0; i < NP; ++i) r = fmaf(-db[i], xr[i], r);
                ring[s2 * kMaskThreads] = r;
                acc += r;
            }
            // fast-path pixels: the last hv - 1 valid history residuals with the refined beta, by a
            // backward sweep from n - 1 that stops once every such lane of the warp has its window
            int rem = (FAST && ok && !needx && hv >= 2) ? hv - 1 : 0;
            if (FAST && __any_sync(0xffffffffu, rem > 0)) {
                int sidx = (hv - 1) * RS;
                float accw = 0.f;
                for (int t0 = ((n - 1) / D23) * D23; t0 >= 0 && __any_sync(0xffffffffu, rem > 0); t0 -= D23) {
                    float vb[D23];
                    load(t0, n, vb);
#pragma unroll
                    for (int k = D23 - 1; k >= 0; --k) {
                        const int t = t0 + k;
                        const bool inwin = rem > 0 && finitef(vb[k]) && t < n;
                        const float r = resid(inwin ? vb[k] - c : 0.f, t);
                        if (inwin) ring[sidx] = r;
                        sidx -= inwin ? RS : 0;
                        rem -= inwin ? 1 : 0;
                        accw += inwin ? r : 0.f;
                    }
                }
                if (ok && !needx) acc = accw;
            }
        } else {
            int tlo = tw;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tlo = min(tlo, __shfl_xor_sync(0xffffffffu, tlo, o));
            for (int t0 = tlo; t0 < n; t0 += D23) {
                float vb[D23];
                load(t0, n, vb);
#pragma unroll
                for (int k = 0; k < D23; ++k) {
                    const int t = t0 + k;
                    const bool inwin = needx && finitef(vb[k]) && t >= tw && t < n;
                    const float yc = inwin ? vb[k] - c : 0.f;
                    float2 r2 = f2(yc, 0.f);                         // resid() with beta_0
                    const float* xr = s_x + t * SP;
                    const float4* x4 = reinterpret_cast<const float4*>(xr);
#pragma unroll
                    for (int q = 0; q < SP / 4; ++q) {
                        const float4 x = x4[q];
                        if (4 * q + 1 < NP) r2 = fma2(nb0[2 * q], f2(x.x, x.y), r2);
                        if (4 * q + 3 < NP) r2 = fma2(nb0[2 * q + 1], f2(x.z, x.w), r2);
                    }
                    float r = r2.x + r2.y;
#pragma unroll
                    for (int i = 0; i < NP; ++i) r = fmaf(-db[i], xr[i], r);
                    if (inwin) ring[so] = r;
                    so += inwin ? RS : 0;
                    acc += inwin ? r : 0.f;
                }
            }
            // fast-path pixels: the last hv - 1 valid history residuals with the refined beta, by a
            // backward sweep from n - 1 that stops once every such lane of the warp has its window
            int rem = (FAST && ok && !needx && hv >= 2) ? hv - 1 : 0;
            if (FAST && __any_sync(0xffffffffu, rem > 0)) {
                int sidx = (hv - 1) * RS;
                float accw = 0.f;
                for (int t0 = ((n - 1) / D23) * D23; t0 >= 0 && __any_sync(0xffffffffu, rem > 0); t0 -= D23) {
                    float vb[D23];
                    load(t0, n, vb);
#pragma unroll
                    for (int k = D23 - 1; k >= 0; --k) {
                        const int t = t0 + k;
                        const bool inwin = rem > 0 && finitef(vb[k]) && t < n;
                        const float r = resid(inwin ? vb[k] - c : 0.f, t);
                        if (inwin) ring[sidx] = r;
                        sidx -= inwin ? RS : 0;
                        rem -= inwin ? 1 : 0;
                        accw += inwin ? r : 0.f;
                    }
                }
                if (ok && !needx) acc = accw;
            }
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
        int ro = 0;                              // word offset of the ring slot holding r_{e - h_v}
        const int ro_end = hv * RS;
        const float jx0 = (float)(nv + 1) * inv_nv, dx = inv_nv;   // x_j = (n_v + 1 + j) / n_v
        // KEEP: the MOSUM matrix and/or the MOSUM mean were requested (the LEAN variant skips both)
        float* mo_p = KEEP && prm.mosum ? prm.mosum + px : nullptr;
        const int64_t ld_out = prm.ld_out;
        // log_plus(x) = 1 while x = (n_v + 1 + j) / n_v <= e, i.e. j < je: b_j = lambda exactly
        const int je = fit_ok ? (int)floorf(1.718281828f * (float)nv - 1.f) + 1 : 0x3fffffff;
        for (int t0 = n; t0 < N; t0 += D23) {
            float vb[D23];
            load(t0, N, vb);
#pragma unroll
            for (int k = 0; k < D23; ++k) {
                const int t = t0 + k;
                const bool m = finitef(vb[k]) && fit_ok;
                const float r = resid(m ? vb[k] - c : 0.f, t);
                const float old = ring[ro];
                if (m) ring[ro] = r;
                const int ro1 = ro + RS == ro_end ? 0 : ro + RS;
                ro = m ? ro1 : ro;
                acc = m ? acc + (r - old) : acc;
                const float a = fabsf(acc);
                mx = m ? fmaxf(mx, a) : mx;
                // strict crossing |MO_j| > b_j (_kernels.py:47).  b_j >= lambda: only a date past
                // lambda before the first crossing needs b_j, and only j >= je needs log_plus (a
                // call, so the log/rsqrt never run predicated on every date)
                if (m && first == 0 && a > lam_sc) {
                    const float b = j >= je ? masked_bound(lam_sc, j, dx, jx0) : lam_sc;
                    if (a > b) first = t + 1 - n;
                }
                if (KEEP) msum += m ? acc : 0.f;
                j += m ? 1 : 0;
                if (KEEP && mo_p) {
                    if (act && t < N) *mo_p = m ? acc * inv : qnan;
                    mo_p += ld_out;
                }
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
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(tbase, kCols);
}

}  // namespace bwm
