// bwm_kernel_tma.cuh — fused BFAST-monitor kernel, TMA-pipelined variant (sm_100a, default).
//
// CTA = 4 warps, 128 threads, one pixel PAIR per thread -> a 256-pixel tile; warp w owns the
// 64-pixel slice [64w, 64w+64) of every tile.  Each warp runs its OWN asynchronous pipeline:
// lane 0 issues one 2-D tensor TMA per stage (cp.async.bulk.tensor.2d, SASS UTMALDG) that
// copies a box of 8 dates x 64 pixels (2 KB) of the time-major stack into the warp's stage
// ring in shared memory and completes an mbarrier with the byte count; the warp waits on
// it, each lane reads its float2 per date (LDS.64, conflict-free), and after the stage is
// consumed the same lane re-arms the slot with the stage kStages ahead.  No producer warp,
// no cross-warp barrier: warps never wait for each other.
//
// Row stream per tile (the issue cursor runs kStages ahead across passes and tiles):
//   pass 1 : rows [0, n)             beta_Q = Q^T (y - c) and ||y - c||^2 in ONE sweep
//                                    (pass 0 scans the first stage for c); sigma follows from
//                                    RSS = ||y-c||^2 - ||beta_Q||^2 (orthonormal basis Q).
//                                    Also the window sum of the filled dates [n-h, n) and (TMEM
//                                    mode) those dates parked in the ring.
//   pass 3 : rows [8*floor(n/8), N)  MOSUM recurrence + detect (stages 8-date aligned);
//            LAG mode: each stage also carries dates t-h (second box)
// Window-sum formulation (bwm_common.cuh, KParams::wt): the recurrence runs on the FILLED
// series, acc += y~_t - y~_{t-h} (_kernels.py:33 order), and the MOSUM numerator of date t is
// acc - S_t^T beta_Q, S_t the window sum of the fitted-value rows (host table).  So the
// history is read once (no window-0 re-read or conversion), and the lagged date needs no
// fitted value — at C4 (h = 250, p = 14) that halves the FMA work of the monitoring period.
// Measured (profiles/probe): SM-side ingest, DRAM or L2, saturates near 7 TB/s, so re-reading
// the whole history (342 rows/tile) cost ~1 ms at C2; the TMEM-mode stream is 232 rows/tile.
//
// MOSUM ring (y~_{t-h} for the add-one/drop-one recurrence, _kernels.py:31-34):
//   MODE kRingTmem : in Tensor Memory.  Each thread owns its TMEM lane; ring row q of the
//                    pixel pair occupies columns 2q, 2q+1; L = ring rows (multiple of the
//                    stage height R, >= h), plus R MIRROR rows L..L+R-1 that duplicate rows
//                    0..R-1 (every write of a row < R also writes row q + L), so the R lagged
//                    rows of a stage are always one contiguous run: R/8 tcgen05.st.x16 and R/8
//                    tcgen05.ld.x16 per stage, no wrap path.  2(L+R) columns: 128 at h <= 56.
//   MODE kRingLag  : no ring; y~_{t-h} refilled from the staged date t-h (large h) by a
//                    lagging fill cursor; tables read through L1 (any series length).
//                    kRingLagT: the same with the tables staged in shared memory (when they fit).
//   (h < R, where an R-row batch would read rows it has not written yet, runs the LDG kernel.)
//
// The monitoring pass runs in the UNSCALED frame: acc = sum of window residuals, crossing
// test |acc| > b_j * sigma * sqrt(n) (== |MO_j| > b_j), MO = acc / (sigma sqrt n) applied to
// the max/mean at the end.  Each pass is ONE unrolled R-date body; the partial stages at pass
// boundaries are handled by warp-uniform row predicates (and read-modify-write of ring rows),
// so the hot code stays small enough for the instruction cache.
#pragma once

#include "bwm_common.cuh"

namespace bwm {

#ifndef BWM_STAGE_ROWS
#define BWM_STAGE_ROWS 8
#endif
#ifndef BWM_TMA_ABL
#define BWM_TMA_ABL 0      // timing ablation: the stage pipeline without the arithmetic (results wrong)
#endif
#ifndef BWM_STAGES
#define BWM_STAGES 5
#endif
constexpr int kStageRows = BWM_STAGE_ROWS;      // dates per stage (multiple of 8)
#ifndef BWM_LAG_L2HINT
#define BWM_LAG_L2HINT 2   // L2 evict_last/evict_first hints on the lagging cursor's boxes (1: lead keep / lag drop;
#endif                     // 2: also pass-1 rows and never-re-read lead rows evict_first).  Static schedule: 2% slower;
                           // with the dynamic slice scheduler C4 is near DRAM-bound and mode 2 at keep 0.5 is 1% faster
#ifndef BWM_LAG_KEEP
#define BWM_LAG_KEEP 0.5   // fraction of a kept box's lines that get evict_last (createpolicy.fractional)
#endif
#define BWM_STR2(x) #x
#define BWM_STR(x) BWM_STR2(x)
#ifndef BWM_STAGES_LAG
#define BWM_STAGES_LAG 3
#endif
constexpr int kStages = BWM_STAGES;             // stage ring depth per warp (TMEM-ring mode)
#ifndef BWM_RING_MIRROR
#define BWM_RING_MIRROR 1  // TMEM ring with R mirror rows (no wrapped lag loads)
#endif
#ifndef BWM_LAZY_CROSS
#define BWM_LAZY_CROSS 1   // LEAN: first-crossing search once per stage from the running max
#endif
constexpr bool kMirror = BWM_RING_MIRROR != 0;
#ifndef BWM_LAGT_WARPS
#define BWM_LAGT_WARPS 16  // warps per CTA of the lagging-cursor kernel with smem tables (tables shared by all;
                           // C4: 16 warps x 2 stages at 1 CTA/SM 5.27 ms, 8 warps 5.87 (3 stages), 4 warps x 2 CTAs 6.09)
#endif
// the lagging-cursor mode moves two boxes per stage (dates t and t-h): 3 stages = 6 boxes
// (kRingLag: tables in global memory, 3 stages, 3 CTAs/SM; kRingLagT: tables in smem, 2 stages,
//  2 CTAs/SM — measured 8.85 vs 8.11 ms at C4, so kRingLagT whenever its tables fit)
#ifndef BWM_LAG_TMEMC
#define BWM_LAG_TMEMC 1    // kRingLagT: park pass 1's compensated beta_Q (hi, lo) in Tensor Memory (C4: 5.45 -> 5.23 ms, no spills)
#endif
#ifndef BWM_STAGES_LAGT
#define BWM_STAGES_LAGT 2
#endif
#ifndef BWM_STAGES_TALL
#define BWM_STAGES_TALL 2  // TALL variant (16-date stages, TMEM ring, LEAN): stages per warp (C2: 2 beat 3)
#endif
constexpr int kTallRows = 16;
__host__ __device__ constexpr int stages_for(int mode) {
    return mode == 2 /* kRingLag */ ? BWM_STAGES_LAG : mode == 3 /* kRingLagT */ ? BWM_STAGES_LAGT : kStages;
}
static_assert(kStageRows == 8 || kStageRows == 16, "stage height: 8 or 16 dates (compensation blocks are 16)");
constexpr int kWarpPx = 64;                     // pixels per warp slice (32 lanes x 2)
constexpr int kBoxBytes = kStageRows * kWarpPx * 4;
constexpr int kWarps = kThreads / 32;
constexpr int kTmaThreads = kThreads;

enum RingMode { kRingSmem = 0, kRingTmem = 1, kRingLag = 2, kRingLagT = 3 };

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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// Non-blocking probe: 1 if the phase with this parity has completed (acquire semantics).
__device__ __forceinline__ uint32_t mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok;
}
// 2-D tensor TMA: box (64 px, R dates) at (x, y) -> smem, completing `bar` with its bytes.
// Executed by the whole warp; one elected lane arms the barrier and issues the copy (no
// divergent branch, operands are warp-uniform).
__device__ __forceinline__ void tma_box_elect(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                              uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t"
        "}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "r"(bytes)
        : "memory");
}
// The same with an L2 eviction-priority hint (BWM_LAG_L2HINT == 2: pass-1 rows of the lagging
// cursor — dates re-read h dates later as lag rows are kept, the others marked evict_first).
__device__ __forceinline__ void tma_box_elect_hint(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                                   uint32_t bytes, bool keep) {
    asm volatile(
        "{\n\t.reg .pred p, k;\n\t.reg .b64 pol;\n\t"
        "setp.ne.b32 k, %6, 0;\n\t"
        "@k createpolicy.fractional.L2::evict_last.b64 pol, " BWM_STR(BWM_LAG_KEEP) ";\n\t"
        "@!k createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], pol;\n\t"
        "}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "r"(bytes), "r"((uint32_t)keep)
        : "memory");
}
__device__ __forceinline__ void tma_box2_elect(uint32_t dst, const CUtensorMap* map, int x, int y, int y2,
                                               uint32_t bar, uint32_t bytes, uint32_t box_bytes = kBoxBytes,
                                               bool keep_lead = true) {
    asm volatile(
        "{\n\t.reg .pred p, kl;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%5], %6;\n\t"
#if BWM_LAG_L2HINT
        // dates t: re-read h dates later as the lag box -> keep in L2; dates t-h: last use
        ".reg .b64 keep, drop, lead;\n\t"
        "setp.ne.b32 kl, %8, 0;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 keep, " BWM_STR(BWM_LAG_KEEP) ";\n\t"
        "createpolicy.fractional.L2::evict_first.b64 drop, 1.0;\n\t"
        "selp.b64 lead, keep, drop, kl;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%2, {%3, %4}], [%5], lead;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%1], [%2, {%3, %7}], [%5], drop;\n\t"
#else
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%2, {%3, %4}], [%5];\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%1], [%2, {%3, %7}], [%5];\n\t"
#endif
        "}" ::"r"(dst),
        "r"(dst + box_bytes), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y),
        "r"(bar), "r"(bytes), "r"(y2), "r"((uint32_t)keep_lead)
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
// the first NP float2 of a 32-column run of this thread's lane: .x16 pieces plus a tail
template <int NP>
__device__ __forceinline__ void tmem_ld_pairs(uint32_t taddr, float2 (&v)[NP]) {
    float2 a[8], b[8];                   // (callers use NP <= 16)
    tmem_ld16(taddr, a);                 // includes wait::ld
    if (NP > 8) tmem_ld16(taddr + 16, b);
#pragma unroll
    for (int i = 0; i < NP; ++i) v[i] = i < 8 ? a[i] : i < 16 ? b[i - 8] : f2(0.f, 0.f);
}
template <int NP>
__device__ __forceinline__ void tmem_st_pairs(uint32_t taddr, const float2 (&v)[NP]) {
    float2 a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = i < NP ? v[i] : f2(0.f, 0.f);
        b[i] = i + 8 < NP ? v[i + 8] : f2(0.f, 0.f);
    }
    tmem_st16(taddr, a);
    if (NP > 8) tmem_st16(taddr + 16, b);
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(v.x)),
                 "r"(__float_as_uint(v.y))
                 : "memory");
}

#ifndef BWM_TMA_MINB
#define BWM_TMA_MINB 4
#endif
#ifndef BWM_TMA_MINB_BIG
#define BWM_TMA_MINB_BIG 3
#endif
#ifndef BWM_RING_WARPS
#define BWM_RING_WARPS 4   // warps per CTA of the TMEM-ring kernel (multiple of 4: a warp per lane quarter
#endif                     // and TMEM column block)
// Warps per CTA: BWM_RING_WARPS (TMEM ring), 4 (lagging cursor through L1), or BWM_LAGT_WARPS
// for the lagging cursor with staged tables (C4: the 64 KB Z^T table is shared by more warps,
// so more warps fit per SM); the tile is 64 px per warp.
__host__ __device__ constexpr int tma_warps(int mode) {
    return mode == kRingLagT ? BWM_LAGT_WARPS : mode == kRingTmem ? BWM_RING_WARPS : kWarps;
}
__host__ __device__ constexpr int tma_threads(int mode) { return 32 * tma_warps(mode); }
__host__ __device__ constexpr int tma_tile(int mode) { return kWarpPx * tma_warps(mode); }
__host__ __device__ constexpr int tma_minb(int np, int mode) {
    return mode == kRingLagT ? (BWM_LAGT_WARPS > 4 ? 1 : 2)
                             : (np <= 10 ? BWM_TMA_MINB : BWM_TMA_MINB_BIG) * 4 / tma_warps(mode);
}

// Shared-memory footprint per warp stage (host mirror in bwm_capi.cu).
__host__ __device__ constexpr int64_t tma_stage_bytes(int mode) {
    return (int64_t)kBoxBytes * (mode == kRingLag || mode == kRingLagT ? 2 : 1);
}
__host__ __device__ constexpr int64_t tma_stage_region(int mode, int stages) {
    return (int64_t)tma_warps(mode) * stages * tma_stage_bytes(mode);
}
__host__ __device__ constexpr int tma_barriers(int mode, int stages) {
    return tma_warps(mode) * stages;
}

// LEAN: no MOSUM matrix / MOSUM mean outputs and a constant boundary over the monitoring
// period (b_j = lambda for every j: log_plus((n+1+j)/n) = 1 while (n+1+j)/n <= e, which holds
// for all BASELINE geometries, N/n = 2) — the per-date boundary product, mean accumulation
// and output branch drop out of the MOSUM loop.  Results are bit-identical to !LEAN.
// RR: dates per stage — kStageRows (8), or kTallRows (16) for the TALL variant of the TMEM-ring
// LEAN kernel (half the TMA boxes, barriers and stage bookkeeping per date; the host picks it
// when its ring needs no more Tensor Memory than the 8-date one, e.g. C2: 5% faster).
// MIR: R mirror rows after the TMEM ring (no wrapped lag loads); a TALL ring that would need more
// Tensor Memory with them (C5: 64 + 16 rows) runs without (MIR = false: a stage whose lagged run
// wraps loads it row by row).
template <int NP, int MODE, bool LEAN, int RR = kStageRows, bool MIR = kMirror>
__global__ void __launch_bounds__(tma_threads(MODE), tma_minb(NP, MODE))
    monitor_kernel_tma(const __grid_constant__ KParams prm) {
    static_assert(MODE == kRingTmem || MODE == kRingLag || MODE == kRingLagT, "TMA kernel: TMEM ring or lagging cursor");
    constexpr bool kLag = MODE == kRingLag || MODE == kRingLagT;
    constexpr int SP = Coefs<NP>::SP;
    constexpr int R = RR;
    static_assert(RR == kStageRows || (RR == kTallRows && MODE == kRingTmem), "TALL: TMEM ring only");
    constexpr int S = RR == kStageRows ? stages_for(MODE) : BWM_STAGES_TALL;
    constexpr int64_t SB = (int64_t)R * kWarpPx * 4 * (kLag ? 2 : 1);
    constexpr int NW = tma_warps(MODE), NT = tma_threads(MODE), TILE = tma_tile(MODE);
    constexpr int ROWF2 = kWarpPx / 2;                   // float2 per staged row
    static_assert(MODE != kRingTmem || NW % 4 == 0, "TMEM ring: warps in whole lane quarters");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = prm.N, n = prm.n, h = prm.h;
    const int NA = (N + 3) & ~3;
    unsigned char* s_stage = smem_raw;                                   // [NW][S][SB]
    // [N][SP] window-sum table: rows t < n are the rows of Q (pass 1), rows t >= n the window
    // sums S_t of the fitted-value rows (pass 3) — host: bwm_plan_create
    // kRingLag (long series): the table stays in global memory and is read through L1 (uniform
    // addresses, broadcast).
    constexpr bool kTblSmem = MODE != kRingLag;
    float* s_tbl = reinterpret_cast<float*>(smem_raw + (int64_t)NW * S * SB);
    const float* s_xt = kTblSmem ? s_tbl : prm.wt;
    const float* s_mt = s_xt;
    float* s_bd = s_tbl + (kTblSmem ? N * SP : 0);                       // [NA] bound by row t (t >= n)
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_bd + NA);           // [NW][S]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + tma_barriers(MODE, S));
    int* s_rows = reinterpret_cast<int*>(s_tmem + 4);                   // [tile_stages] stage -> first date

    if (kTblSmem)
        for (int i = threadIdx.x; i < N * SP; i += NT) s_tbl[i] = prm.wt[i];
    for (int i = threadIdx.x; i < N - n; i += NT) s_bd[n + i] = prm.bound[i];
    {
        // the per-tile stage schedule (identical for every tile): pass 1 [0, n), pass 3
        // [8 floor(n/8), N), R dates per stage
        const int t3_ = (n / R) * R;
        const int a = (n + R - 1) / R;
        const int c = a + (N - t3_ + R - 1) / R;
        for (int i = threadIdx.x; i < c; i += NT) s_rows[i] = i < a ? i * R : t3_ + (i - a) * R;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < tma_barriers(MODE, S); ++s) mbar_init(s_bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // kPark: pass 1's compensated beta_Q (hi, lo) lives in Tensor Memory (the lagging cursor has
    // no ring there), freeing 4 NP registers: 64 columns per warp (hi | lo, 32 each) in its lane
    // quarter; the 16+-warp CTA owns the SM, so it takes all 512 columns
    constexpr bool kPark = MODE == kRingLagT && BWM_LAG_TMEMC && NP <= 16 && BWM_LAGT_WARPS > 4;
    constexpr bool kTmem = MODE == kRingTmem || kPark;
    const uint32_t tmem_cols = MODE == kRingTmem ? (uint32_t)prm.tmem_cols * (NW / 4) : 512u;
    if (kTmem && threadIdx.x < 32) tmem_alloc(s_tmem, tmem_cols);
    if (kTmem) tmem_fence_before();
    __syncthreads();
    if (kTmem) tmem_fence_after();

    // host guarantees whole tiles (TILE = NW slices of 64 px)
    const int64_t ld = prm.ld_y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // initial window: dates [n-h, n) (window 0 of mosum.py:59 is [n-h+1, n]; the first
    // monitoring step adds date n and drops date n-h like every later one)
    const int wstart = n - h;
    const int w0 = (wstart / R) * R;                   // first parked row (TMEM ring)
    const int t3 = (n / R) * R;                        // first row of the (aligned) monitoring stream
    const int tid = threadIdx.x;
    const int wu = __shfl_sync(0xffffffffu, warp, 0);              // warp index, known warp-uniform
    unsigned char* my_stage = s_stage + wu * S * SB;
    uint64_t* full = s_bar + wu * S;
    const uint32_t stage_u32 = smem_u32(my_stage), bar_u32 = smem_u32(full);

    // ---- this warp's TMA issue cursor, kStages ahead of consumption ----------------------
    // The per-tile stage schedule (first date of each stage; pass 3 flagged) is a table, so
    // re-arming a slot is a lookup.  The slot being re-armed was read by this warp through
    // the generic proxy; __syncwarp() in release() orders those reads before lane 0 issues
    // the copy (the same release->acquire ordering an mbarrier handshake gives a producer).
    const int st1 = (n + R - 1) / R;
    const int tile_stages = st1 + (N - t3 + R - 1) / R;
    // The slot re-armed at a release is the one just consumed, so the issue cursor needs only
    // (slice, stage); the first date of a stage comes from the schedule table.
    // Work unit: a 64-px warp SLICE (warps are independent pipelines).  Static schedule: warp
    // w of CTA b takes slices b NW + w, then strides by the grid's warp count.  Dynamic
    // (prm.sched): the first slice is static, every later one is claimed from a global counter
    // one slice AHEAD (the atomic's latency hides behind a whole slice), so warps that run
    // ahead — free-running warps drift apart, and SMs differ — take more slices instead of
    // idling at the end of the kernel.  The cursor moves to the next slice S stages before
    // consumption does (host: tile_stages > S), so one `pending` register carries the slice
    // consumption takes next.
    const int64_t n_slices = prm.n_pixels / kWarpPx;
    const int64_t n_warps = (int64_t)gridDim.x * NW;
    const bool dyn = prm.sched != nullptr;
    int64_t islice = (int64_t)blockIdx.x * NW + wu;
    int64_t pending = islice;
    unsigned int pre = 0;                             // lane 0: the pre-claimed next slice (dynamic)
    const bool jit = dyn && prm.sched_jit;
    if (dyn && !jit && lane == 0) pre = atomicAdd(prm.sched, 1u);
    int istage = 0;
    int xw = (int)(islice * kWarpPx);                 // x of the cursor's slice
    constexpr uint32_t kBox = (uint32_t)(R * kWarpPx * 4);
    auto issue_into = [&](int slot) {
        if (islice >= n_slices) return;
        {
            const int r0 = s_rows[istage];
            const uint32_t dst = stage_u32 + (uint32_t)(slot * SB), bar = bar_u32 + (uint32_t)(slot * 8);
            if (kLag && istage >= st1)
                tma_box2_elect(dst, &prm.tmap, xw, r0, r0 - h, bar, 2 * kBox, kBox,    // + dates t-h
                               BWM_LAG_L2HINT < 2 || r0 + R <= N - h);                  // re-read as a lag row?
            else if (kLag && BWM_LAG_L2HINT == 2)
                tma_box_elect_hint(dst, &prm.tmap, xw, r0, bar, kBox, r0 + R > n - h);
            else
                tma_box_elect(dst, &prm.tmap, xw, r0, bar, kBox);
        }
        if (++istage == tile_stages) {
            istage = 0;
            if (dyn) {
                if (jit && lane == 0) pre = atomicAdd(prm.sched, 1u);
                islice = n_warps + (int64_t)__shfl_sync(0xffffffffu, pre, 0);
                if (islice < n_slices) {
                    if (!jit && lane == 0) pre = atomicAdd(prm.sched, 1u);
                } else if (lane == 0) {
                    // this warp's last claim; the last warp of the launch resets the scheduler
                    if (atomicAdd(prm.sched + 1, 1u) == (unsigned int)(n_warps - 1)) {
                        atomicExch(prm.sched, 0u);
                        atomicExch(prm.sched + 1, 0u);
                    }
                }
            } else {
                islice += n_warps;
            }
            pending = islice;
            xw = (int)(islice * kWarpPx);
        }
    };
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&prm.tmap)) : "memory");
    for (int s = 0; s < S; ++s) issue_into(s);

    const int L = prm.ring_rows;
    const uint32_t tbase = MODE == kRingTmem
                               ? *s_tmem + ((uint32_t)((wu & 3) * 32) << 16) + (uint32_t)((wu >> 2) * prm.tmem_cols)
                               : 0u;
    const uint32_t pbase = kPark ? *s_tmem + ((uint32_t)((wu & 3) * 32) << 16) + (uint32_t)((wu >> 2) * 64) : 0u;
    auto tcol = [&](int row) -> uint32_t { return tbase + (uint32_t)(2 * row); };
    // ring row q of time t is t mod L (2 columns per row: 2L columns, no mirror rows)
    // ring rows of the fixed dates of every tile (one modulo each, per CTA)
    const int q_w0 = MODE == kRingTmem ? w0 % L : 0;
    const int q_t3 = MODE == kRingTmem ? t3 % L : 0, q_t3h = MODE == kRingTmem ? ((t3 - h) % L + L) % L : 0;
    auto ring_put_row = [&](int q, float2 v) {                             // q < L (+ mirror)
        tmem_st2(tcol(q), v);
        if (MIR && q < R) tmem_st2(tcol(q + L), v);
    };
    auto ring_ld2 = [&](int q, float2& v) {                                // no wait
        uint32_t a, b;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(tcol(q)) : "memory");
        v = f2(__uint_as_float(a), __uint_as_float(b));
    };
    auto ring_get_row = [&](int q) -> float2 {                            // q < 2L: wraps once
        float2 v;
        ring_ld2(q >= L ? q - L : q, v);
        tmem_wait_ld();
        return v;
    };
    // R consecutive ring rows starting at row q0 < L: rows past L are the mirror rows, so the
    // run never wraps — R/8 tcgen05.ld.x16
    auto ring_load = [&](int q0, float2 (&v)[R]) {
        tmem_wait_st();
        if (MIR || q0 + R <= L) {
#pragma unroll
            for (int c8 = 0; c8 < R / 8; ++c8)
                tmem_ld16(tcol(q0 + 8 * c8), *reinterpret_cast<float2(*)[8]>(&v[8 * c8]));
        } else {                                             // no mirror: the run wraps
#pragma unroll
            for (int k = 0; k < R; ++k) ring_ld2(q0 + k >= L ? q0 + k - L : q0 + k, v[k]);
            tmem_wait_ld();
        }
    };
    auto ring_store = [&](int q0, const float2 (&v)[R]) {   // q0 multiple of R: never wraps
#pragma unroll
        for (int c8 = 0; c8 < R / 8; ++c8)
            tmem_st16(tcol(q0 + 8 * c8), *reinterpret_cast<const float2(*)[8]>(&v[8 * c8]));
        if (MIR && q0 == 0) {                                // rows 0..R-1: their mirror too
#pragma unroll
            for (int c8 = 0; c8 < R / 8; ++c8)
                tmem_st16(tcol(L + 8 * c8), *reinterpret_cast<const float2(*)[8]>(&v[8 * c8]));
        }
    };
    int cur = 0;
    uint32_t ph = 0;
    uint32_t next_ready = 0;     // result of the look-ahead probe of stage `cur`
    // Waiting on an mbarrier costs a round trip even when the stage has landed; the probe of
    // the following stage is issued here and consumed at the next acquire.
    auto acquire = [&]() -> const float2* {
        if (!next_ready) mbar_wait(full + cur, ph);
        const int nc = cur + 1 == S ? 0 : cur + 1;
        next_ready = mbar_test(full + nc, nc == 0 ? ph ^ 1 : ph);
        return reinterpret_cast<const float2*>(my_stage + cur * SB) + lane;
    };
    auto release = [&]() {
        __syncwarp();
        issue_into(cur);                             // re-arm this slot kStages ahead
        if (++cur == S) { cur = 0; ph ^= 1; }
    };

    for (int64_t slice = pending; slice < n_slices; slice = dyn ? pending : slice + n_warps) {
        const int64_t px0 = slice * kWarpPx + 2 * lane;
        const float* yp = prm.y + px0;

        // ---- pass 1: beta_Q and ||y - c||^2 (+ pass 0 on the first stage) ---------------
        float2 hi[NP], lo[NP], part[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) { hi[i] = lo[i] = part[i] = f2(0.f, 0.f); }
        if (kPark) {
            tmem_st_pairs<NP>(pbase, hi);
            tmem_st_pairs<NP>(pbase + 32, lo);
        }
        float2 qpart = f2(0.f, 0.f), wpart = f2(0.f, 0.f);
        double q0 = 0.0, q1 = 0.0, wd0 = 0.0, wd1 = 0.0;   // ||y-c||^2, window sum of [n-h, n)
        float2 c = f2(0.f, 0.f);
        bool f0 = false, f1 = false;
        float2 last = f2(0.f, 0.f);
        float2 lag_last = f2(0.f, 0.f);                   // LAG: fill state before date n-h
        float2 negc = f2(0.f, 0.f);
        int pr = q_w0;                                    // ring row of the next parked stage
        for (int t0 = 0; t0 < n; t0 += R) {
            const float2* st = acquire();
#if BWM_TMA_ABL
            {   // timing ablation (results wrong): consume the stage, no arithmetic
                float2 sacc = f2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < R; ++k) sacc = add2(sacc, st[k * ROWF2]);
                last = add2(last, sacc);
                release();
                continue;
            }
#endif
            if (t0 == 0) {
                // pass 0: first finite value (engine.py:316 first = finite.argmax)
                const int rows = min(R, n);
#pragma unroll 1
                for (int k = rows - 1; k >= 0; --k) {
                    const float2 v = st[k * ROWF2];
                    if (finitef(v.x)) { c.x = v.x; f0 = true; }
                    if (finitef(v.y)) { c.y = v.y; f1 = true; }
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
            // TMEM mode: the filled values of the dates [w0, n) also go to their ring rows
            // (t mod L) — the y~_{t-h} of the first monitoring dates (no re-read)
            const bool park = MODE == kRingTmem && t0 >= w0;
            if (t0 + R <= n) {
                const float* mrow = s_mt + t0 * SP;
                float2 yy[R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float2 vc = fill(st[k * ROWF2], negc, last);
                    yy[k] = vc;
                    axpy_row<NP, SP>(part, vc, mrow + k * SP);
                    qpart = fma2(vc, vc, qpart);
                }
                if (park) ring_store(pr, yy);
                if (t0 + R >= wstart) {                     // stages of the initial window (and the date before it)
#pragma unroll
                    for (int k = 0; k < R; ++k)
                        if (t0 + k >= wstart) wpart = add2(wpart, yy[k]);
                    if (kLag && t0 < wstart) {              // fill state before date n-h
#pragma unroll
                        for (int k = 0; k < R; ++k)
                            if (t0 + k == wstart - 1) lag_last = yy[k];
                    }
                }
            } else {                                            // last stage: dates [t0, n) only
#pragma unroll 1
                for (int k = 0; k < n - t0; ++k) {
                    const float2 vc = fill(st[k * ROWF2], negc, last);
                    if (park) ring_put_row(pr + k >= L ? pr + k - L : pr + k, vc);
                    axpy_row<NP, SP>(part, vc, s_mt + (t0 + k) * SP);
                    qpart = fma2(vc, vc, qpart);
                    if (t0 + k >= wstart) wpart = add2(wpart, vc);
                    if (kLag && t0 + k == wstart - 1) lag_last = vc;
                }
            }
            release();
            if (park) { pr += R; if (pr >= L) pr -= L; }
            if (((t0 + R) & (kComp - 1)) == 0 || t0 + R >= n) {
                if (kPark) {
                    float2 h2[NP], l2[NP];
                    tmem_wait_st();
                    tmem_ld_pairs<NP>(pbase, h2);
                    tmem_ld_pairs<NP>(pbase + 32, l2);
#pragma unroll
                    for (int i = 0; i < NP; ++i) { two_sum(h2[i], l2[i], part[i]); part[i] = f2(0.f, 0.f); }
                    tmem_st_pairs<NP>(pbase, h2);
                    tmem_st_pairs<NP>(pbase + 32, l2);
                } else {
#pragma unroll
                    for (int i = 0; i < NP; ++i) { two_sum(hi[i], lo[i], part[i]); part[i] = f2(0.f, 0.f); }
                }
                q0 += (double)qpart.x;
                q1 += (double)qpart.y;
                wd0 += (double)wpart.x;
                wd1 += (double)wpart.y;
                qpart = wpart = f2(0.f, 0.f);
            }
        }
        const bool valid0 = f0, valid1 = f1;
        if (kPark) {
            tmem_wait_st();
            tmem_ld_pairs<NP>(pbase, hi);
            tmem_ld_pairs<NP>(pbase + 32, lo);
        }
        float2 bq[NP], nb[NP];    // beta_Q and -beta_Q
#pragma unroll
        for (int i = 0; i < NP; ++i) { bq[i] = add2(hi[i], lo[i]); nb[i] = f2(-bq[i].x, -bq[i].y); }

        // sigma (engine.py:363-371) from the one-pass RSS and the zero-sigma contract
        // (engine.py:373-378): the reference raises when float64 gives sigma == 0 exactly —
        // an identically zero history (c == 0).  A non-zero constant history has round-off
        // sigma ~1e-17 there (MO ~1e15): scale 0 reproduces its decisions (any non-zero window
        // crosses).
        const float2 ss = rss_onepass<NP>(q0, q1, bq);
        fix_flag(prm, valid0, q0, ss.x, px0);
        fix_flag(prm, valid1, q1, ss.y, px0 + 1);
        const bool z0 = zero_history(valid0, q0, c.x), z1 = zero_history(valid1, q1, c.y);
        if (z0 || z1) atomicMin(prm.zero_sigma, (unsigned long long)(prm.pixel_offset + px0 + (z0 ? 0 : 1)));
        const float2 sc = sigma_scale(ss, prm.inv_dof, prm.sqrt_n, valid0, valid1);

        // initial window sum minus the intercept part of S^T beta_Q (float64, bwm_common.cuh)
        float2 acc = wsum_init(wd0, wd1, hi[0], lo[0], prm.s0);

        // ---- pass 3: monitoring period, fused MOSUM + detect (unscaled frame) ----------
        float2 mx = f2(0.f, 0.f), msum = f2(0.f, 0.f), sr = f2(0.f, 0.f);
        int first0 = 0x7fffffff, first1 = 0x7fffffff;
        float* const mo_out = prm.mosum;
        const bool want_sup = prm.sup != nullptr;
        const float2 inv = inv_scale(sc);
        const float2 bsc = mul2(sc, f2(s_bd[n], s_bd[n]));   // LEAN: the constant boundary, unscaled
        // one monitoring date: y~_t in, y~_{t-h} out, numerator acc - S_t^T beta_Q
        auto step = [&](const float2 r, const float2 old, const int t, const float bj) {
            acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
            const float2 num = wsum_row<NP, SP>(acc, s_xt + t * SP, nb);
            const float2 bs = LEAN ? bsc : mul2(sc, f2(bj, bj));   // boundary in the unscaled frame
            const float a0 = fabsf(num.x), a1 = fabsf(num.y);
            mx.x = fmaxf(mx.x, a0);
            mx.y = fmaxf(mx.y, a1);
            const int j1 = t - n + 1;
            if (a0 > bs.x) first0 = min(first0, j1);  // strict crossing (_kernels.py:47)
            if (a1 > bs.y) first1 = min(first1, j1);
            if (!LEAN) {
                if (want_sup) {                        // max_j |acc_j| / b_j (unscaled)
                    sr.x = fmaxf(sr.x, __fdividef(a0, bj));
                    sr.y = fmaxf(sr.y, __fdividef(a1, bj));
                }
                msum = add2(msum, num);
                if (mo_out) *reinterpret_cast<float2*>(mo_out + (int64_t)(t - n) * prm.ld_out + px0) = mul2(num, inv);
            }
        };
        int wb = q_t3;                                   // ring row of t0
        int rb = q_t3h;                                  // ring row of t0 - h
        for (int t0 = t3; t0 < N; t0 += R) {
            const float2* st = acquire();
#if BWM_TMA_ABL
            {   // timing ablation (results wrong): consume the stage, no arithmetic
                float2 sacc = f2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < R; ++k) sacc = add2(sacc, st[k * ROWF2]);
                mx = add2(mx, sacc);
                release();
                continue;
            }
#endif
            const float2* lst = st + kBox / 8;           // lag dates (kRingLag): second box
            if (t0 >= n && t0 + R <= N) {
                // the lagged and the new ring rows move in 8-row groups (one tcgen05.ld/st.x16 each),
                // so a 16-date stage keeps 8 of each live, not 16: group g reads rows rb + 8g (the
                // mirror rows cover runs past L) and writes rows wb + 8g; with h >= R no group writes
                // a row a later group of the same stage reads
                constexpr int G = R < 8 ? R : 8;
                float2 oldv[G], newv[G];
                float4 b4[R / 4];
#pragma unroll
                for (int q = 0; q < R / 4; ++q)
                    b4[q] = LEAN ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(s_bd + t0)[q];
                const float* xrow = s_xt + t0 * SP;
                // LEAN: MOSUM numerators of the current 8-date group (the first-crossing search
                // runs per group)
                float2 acck[G];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const int t = t0 + k;
                    if (MODE == kRingTmem && k % G == 0) {
                        int q = rb + k;
                        if (!MIR && q >= L) q -= L;
                        if (k == 0) tmem_wait_st();                  // the previous stage's rows landed
                        if (MIR || q + G <= L) {
                            tmem_ld16(tcol(q), *reinterpret_cast<float2(*)[8]>(&oldv[0]));
                        } else {                                     // no mirror: the run wraps
#pragma unroll
                            for (int g = 0; g < G; ++g) ring_ld2(q + g >= L ? q + g - L : q + g, oldv[g]);
                            tmem_wait_ld();
                        }
                    }
                    const float2 r = fill(st[k * ROWF2], negc, last);
                    float2 old;
                    if (MODE == kRingTmem) {
                        old = oldv[k % G];
                        newv[k % G] = r;
                    } else {
                        old = fill(lst[k * ROWF2], negc, lag_last);
                    }
                    if (LEAN && BWM_LAZY_CROSS) {
                        // constant boundary: the first crossing is the first date whose running max
                        // exceeds it, so the per-date test moves out of the loop (below)
                        acc = add2(acc, sub2(r, old));             // _kernels.py:33 order
                        const float2 num = wsum_row<NP, SP>(acc, xrow + k * SP, nb);
                        acck[k % G] = num;
                        mx.x = fmaxf(mx.x, fabsf(num.x));
                        mx.y = fmaxf(mx.y, fabsf(num.y));
                        if (k % G == G - 1) {
                            // strict crossing (_kernels.py:47) of the group's first date past the
                            // boundary; taken at most once per pixel
                            const int tg = t0 + k - (G - 1) - n + 1;
                            if (first0 == 0x7fffffff && mx.x > bsc.x) {
#pragma unroll
                                for (int g = G - 1; g >= 0; --g)
                                    if (fabsf(acck[g].x) > bsc.x) first0 = tg + g;
                            }
                            if (first1 == 0x7fffffff && mx.y > bsc.y) {
#pragma unroll
                                for (int g = G - 1; g >= 0; --g)
                                    if (fabsf(acck[g].y) > bsc.y) first1 = tg + g;
                            }
                        }
                    } else {
                        const float4 bq4 = b4[k >> 2];
                        step(r, old, t, (k & 3) == 0 ? bq4.x : (k & 3) == 1 ? bq4.y : (k & 3) == 2 ? bq4.z : bq4.w);
                    }
                    if (MODE == kRingTmem && k % G == G - 1) {
                        const int q = wb + k - (G - 1);              // multiple of 8, < L
                        tmem_st16(tcol(q), *reinterpret_cast<const float2(*)[8]>(&newv[0]));
                        if (MIR && q < R) tmem_st16(tcol(L + q), *reinterpret_cast<const float2(*)[8]>(&newv[0]));
                    }
                }
            } else {
                // boundary stage: dates [max(t0, n), min(t0 + R, N)), one at a time
                if (MODE == kRingTmem) tmem_wait_st();
                const int k0 = max(0, n - t0), k1 = min(R, N - t0);
#pragma unroll 1
                for (int k = k0; k < k1; ++k) {
                    const int t = t0 + k;
                    const float2 r = fill(st[k * ROWF2], negc, last);
                    float2 old;
                    if (MODE == kRingTmem) {
                        old = ring_get_row(rb + k);
                        ring_put_row(wb + k, r);
                    } else {
                        old = fill(lst[k * ROWF2], negc, lag_last);
                    }
                    step(r, old, t, s_bd[t]);
                }
            }
            release();
            if (MODE == kRingTmem) {
                wb += R; if (wb == L) wb = 0;
                rb += R; if (rb >= L) rb -= L;
            }
        }

        // ---- outputs --------------------------------------------------------------------
        const float inv_m = 1.0f / (float)(N - n);
        *reinterpret_cast<uchar2*>(prm.valid + px0) = make_uchar2(valid0, valid1);
        *reinterpret_cast<int2*>(prm.first_idx + px0) =
            make_int2(first0 == 0x7fffffff ? 0 : first0, first1 == 0x7fffffff ? 0 : first1);
        *reinterpret_cast<float2*>(prm.max_abs + px0) = mul2(mx, inv);
        if (!LEAN && prm.mo_mean) *reinterpret_cast<float2*>(prm.mo_mean + px0) = mul2(mul2(msum, inv), f2(inv_m, inv_m));
        if (want_sup) {        // LEAN: b_j == b_n for every j
            const float2 s = LEAN ? mul2(mul2(mx, inv), f2(1.0f / s_bd[n], 1.0f / s_bd[n])) : mul2(sr, inv);
            *reinterpret_cast<float2*>(prm.sup + px0) = s;
        }
        if (prm.beta) store_beta<NP>(prm, px0, c, bq, valid0, valid1, 2);
    }

    if (kTmem) {
        tmem_wait_st();
        tmem_fence_before();
        __syncthreads();
        tmem_fence_after();
        if (warp == 0) tmem_dealloc(*s_tmem, tmem_cols);
    }
}

}  // namespace bwm
