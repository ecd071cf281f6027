// bwm_capi.cu — C ABI of libbwm.so (declared in include/bwm.h).
//
// Owns: the device-resident constant tables (bwm_plan), kernel dispatch over the
// compiled (n_params, vectorised, ring) variants, persistent-grid sizing, and the
// host-buffer pipeline (bwm_monitor_host) that streams pixel chunks through the GPU
// with H2D / kernel / D2H overlapped on separate streams.
#include "../../include/bwm.h"
#include "bwm_io.h"
#include "bwm_variants.cuh"

#include <atomic>
#include <cudaTypedefs.h>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#define BWM_DECLARE_PICK(NP) bwm::KernelFn bwm_pick_p##NP(int kind, int mode);
// per-n_params kernel tables, one translation unit each (bwm_variants_p*.cu)
BWM_DECLARE_PICK(4)
BWM_DECLARE_PICK(6)
BWM_DECLARE_PICK(8)
BWM_DECLARE_PICK(10)
BWM_DECLARE_PICK(12)
BWM_DECLARE_PICK(14)
BWM_DECLARE_PICK(16)
BWM_DECLARE_PICK(18)
#define BWM_DECLARE_PICK_MMA(NP) bwm::KernelFn bwm_pick_mma_p##NP(int lean);
BWM_DECLARE_PICK_MMA(4)
BWM_DECLARE_PICK_MMA(6)
BWM_DECLARE_PICK_MMA(8)
BWM_DECLARE_PICK_MMA(10)
BWM_DECLARE_PICK_MMA(12)
BWM_DECLARE_PICK_MMA(14)
BWM_DECLARE_PICK_MMA(16)
BWM_DECLARE_PICK_MMA(18)
#define BWM_DECLARE_PICK_MASKED(NP) bwm::KernelFn bwm_pick_masked_p##NP(int big, int keep);
BWM_DECLARE_PICK_MASKED(4)
BWM_DECLARE_PICK_MASKED(6)
BWM_DECLARE_PICK_MASKED(8)
BWM_DECLARE_PICK_MASKED(10)
BWM_DECLARE_PICK_MASKED(12)
BWM_DECLARE_PICK_MASKED(14)
BWM_DECLARE_PICK_MASKED(16)
BWM_DECLARE_PICK_MASKED(18)

namespace bwm {
cudaError_t launch_fixup(const KParams& prm, int p, const int64_t* list, const unsigned int* count, int sms,
                         cudaStream_t s);
cudaError_t launch_masked_f64(const KParams& prm, int p, double lambda, int sms, cudaStream_t s);
cudaError_t launch_finalize(const int32_t* first_idx, const float* max_abs, int64_t P, int n, int64_t* first_break,
                            double* mx64, uint8_t* detected, cudaStream_t s);
}

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int set_err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

}  // namespace

namespace bwm {
int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace bwm

namespace {

#define BWM_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return set_err((int)e_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                        \
    } while (0)

constexpr int kRingMaxH = 64;   // ring in smem up to h = 64 (64 KB); above: lagging cursor

// shared memory of the LDG kernel: tables + MOSUM ring
int64_t smem_bytes_for(int N, int n, int h, int p, bool ring) {
    const int sp = (p + 3) & ~3;
    // ring variants stage the window-sum table; lagging-cursor variants read it from L1
    int64_t fl = (ring ? (int64_t)N * sp : 0) + (((N - n) + 3) & ~3);   // window-sum table + bound
    int64_t bytes = fl * 4;
    if (ring) bytes += (int64_t)h * bwm::kThreads * 8;
    return bytes;
}

// TMA kernel ring mode for a bandwidth h (bwm_kernel_tma.cuh): a TMEM ring of L rows (2
// columns each) when 8 <= h and it fits 256 columns; a shared-memory ring for
// h < 8; the lagging cursor above.
struct TmaRing {
    int mode, rows, cols;
};
// BWM_TMEM_COLS_MAX (power of two, 64..512): the largest TMEM ring a plan may allocate per CTA.
// 512 = the whole SM's Tensor Memory: one CTA per SM, but the h = 250 ring of C4 fits on chip.
int tmem_cols_max() {
    const char* e = std::getenv("BWM_TMEM_COLS_MAX");
    const int v = e ? std::atoi(e) : 256;
    return v >= 512 ? 512 : v >= 256 ? 256 : v >= 128 ? 128 : 64;
}
TmaRing tma_ring_for(int h) {
    constexpr int R = bwm::kStageRows;
    const int L = ((h + R - 1) / R) * R;
    const int need = 2 * (L + (bwm::kMirror ? R : 0));   // 2 columns per ring row; mirror rows L..L+R-1
    if (h >= R && need <= tmem_cols_max()) {
        int cols = 32;
        while (cols < need) cols *= 2;
        return {bwm::kRingTmem, L, cols};
    }
    return {h < R ? -1 : (int)bwm::kRingLag, 0, 0};   // -1: no TMA variant (LDG kernel)
}

// shared memory of the TMA kernel: per-warp stage rings + tables (Z^T, bound indexed by row) + the stage mbarriers + the TMEM address slot; 0 when no TMA variant applies
int64_t smem_bytes_tma(int N, int n, int h, int p, int mode) {
    (void)h;
    if (mode < 0) return 0;
    const int sp = (p + 3) & ~3;
    // Z^T (rows < n double as Q^T; global memory in the lagging-cursor mode) + bound
    int64_t fl = (mode == bwm::kRingLag ? 0 : (int64_t)N * sp) + ((N + 3) & ~3);
    const int S = bwm::stages_for(mode);
    int64_t bytes = bwm::tma_stage_region(mode, S) + fl * 4;
    const int sched = 2 * ((N + bwm::kStageRows - 1) / bwm::kStageRows) + 4;   // stage schedule table
    return bytes + bwm::tma_barriers(mode, S) * 8 + 16 + 4 * sched;  // + stage barriers, TMEM slot, schedule
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link needed).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D map of a time-major float32 block: dim0 = pixels (contiguous), dim1 = dates (stride ld)
int encode_map(CUtensorMap* map, const float* y, int64_t n_pixels, int n_obs, int64_t ld, int box_px = bwm::kWarpPx,
               int box_rows = bwm::kStageRows) {
    auto fn = encode_fn();
    if (!fn) return set_err((int)cudaErrorNotSupported, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)n_pixels, (cuuint64_t)n_obs};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_px, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    // L2 promotion of the box rows (A/B knob BWM_L2PROMO = 0 none, 1 64B, 2 128B, 3 256B; default 256B)
    static const int promo = [] {
        const char* e = std::getenv("BWM_L2PROMO");
        const int v = e ? std::atoi(e) : 3;
        return v < 0 || v > 3 ? 3 : v;
    }();
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(y), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err((int)cudaErrorInvalidValue, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return BWM_OK;
}

using bwm::Kind;
using bwm::kLdgFast;
using bwm::kLdgSafe;
using bwm::kTma;
using bwm::KernelFn;

struct DeviceRestore {
    int prev = -1;
    explicit DeviceRestore(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceRestore() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// (n_params, kind, mode) -> kernel.  kLdgSafe: tail tile / misaligned input (scalar loads).
KernelFn pick(int p, Kind kind, int mode) {
    switch (p) {
        case 4: return bwm_pick_p4(kind, mode);
        case 6: return bwm_pick_p6(kind, mode);
        case 8: return bwm_pick_p8(kind, mode);
        case 10: return bwm_pick_p10(kind, mode);
        case 12: return bwm_pick_p12(kind, mode);
        case 14: return bwm_pick_p14(kind, mode);
        case 16: return bwm_pick_p16(kind, mode);
        case 18: return bwm_pick_p18(kind, mode);
        default: return nullptr;
    }
}

KernelFn pick_masked(int p, bool big, bool keep) {
    switch (p) {
        case 4: return bwm_pick_masked_p4(big, keep);
        case 6: return bwm_pick_masked_p6(big, keep);
        case 8: return bwm_pick_masked_p8(big, keep);
        case 10: return bwm_pick_masked_p10(big, keep);
        case 12: return bwm_pick_masked_p12(big, keep);
        case 14: return bwm_pick_masked_p14(big, keep);
        case 16: return bwm_pick_masked_p16(big, keep);
        case 18: return bwm_pick_masked_p18(big, keep);
        default: return nullptr;
    }
}

KernelFn pick_mma(int p, bool lean) {
    switch (p) {
        case 4: return bwm_pick_mma_p4(lean);
        case 6: return bwm_pick_mma_p6(lean);
        case 8: return bwm_pick_mma_p8(lean);
        case 10: return bwm_pick_mma_p10(lean);
        case 12: return bwm_pick_mma_p12(lean);
        case 14: return bwm_pick_mma_p14(lean);
        case 16: return bwm_pick_mma_p16(lean);
        case 18: return bwm_pick_mma_p18(lean);
        default: return nullptr;
    }
}

// masked kernel: x x^T table and rings in shared memory up to this size, else global (BIG)
constexpr int64_t kMaskedSmemMax = 96 << 10;

int threads_of(Kind k, int tma_mode = bwm::kRingTmem) { return k == kTma ? bwm::tma_threads(tma_mode) : bwm::kThreads; }

}  // namespace

struct HostPipe {
    int64_t chunk = 0;                 // pixels per chunk
    int nbuf = 0;
    float* d_y[2] = {nullptr, nullptr};
    uint8_t* d_valid[2] = {nullptr, nullptr};
    int32_t* d_first[2] = {nullptr, nullptr};
    float* d_max[2] = {nullptr, nullptr};
    float* d_beta[2] = {nullptr, nullptr};
    float* d_mean[2] = {nullptr, nullptr};
    float* d_mosum[2] = {nullptr, nullptr};
    int64_t* d_fb[2] = {nullptr, nullptr};     // first_break (int64)
    double* d_mx64[2] = {nullptr, nullptr};    // max_abs (float64)
    uint8_t* d_det[2] = {nullptr, nullptr};    // detected
    int64_t* d_zero = nullptr;         // [2]
    size_t bytes = 0;                  // device memory held by the pipeline
    cudaStream_t s_h2d[2] = {nullptr, nullptr};
    cudaStream_t s_k[2] = {nullptr, nullptr};
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_k0[2] = {nullptr, nullptr}, ev_k1[2] = {nullptr, nullptr},
                ev_free[2] = {nullptr, nullptr};
    // pinned landing zone for result maps whose destination is pageable (plain numpy): the D2H
    // lands here at full rate and threads memcpy it out (grown on demand, kept across calls)
    char* h_stage = nullptr;
    size_t h_stage_bytes = 0;
    double last_kernel_ms = 0, last_total_ms = 0;
    int64_t last_h2d = 0, last_d2h = 0;
};

struct bwm_plan {
    bwm_dims dims{};
    int device = 0;
    int sp = 0;
    float* d_xt = nullptr;
    float* d_bound = nullptr;
    float* d_rinv = nullptr;
    float inv_dof = 0, sqrt_n = 0, tc_ts = 0, inv_ts = 0, lambda = 0;
    bool ring = true;                  // LDG kernels: smem ring (else lagging cursor)
    TmaRing tring{};                   // TMA kernel ring mode
    int64_t smem = 0;                  // LDG kernels
    int64_t smem_tma = 0;              // TMA kernel (0: does not fit -> LDG kernels only)
    int sms = 0;
    int blocks_per_sm[3] = {0, 0, 0};  // [Kind]
    int occ_raw[3] = {0, 0, 0};        // occupancy API result before the TMEM cap
    bool force_ldg = false;            // BWM_KERNEL=ldg (A/B against the TMA kernel)
    bool const_bound = false;          // b_j == b_0 for every j (LEAN TMA variant applies)
    bool precise = false;              // long horizon: float64 fitted values, LDG kernels only
    double* d_xtd = nullptr;           // [N][sp] Z^T in float64 (the fixup)
    float* d_wt = nullptr;             // [N][sp] window-sum table (rows < n: Q^T, rows >= n: S_t)
    double* d_wtd = nullptr;           // the same in float64 (precise mode)
    double s0 = 0.0;                   // h * z[0]: intercept part of every S_t
    // float64 fixup of ill-conditioned pixels (bwm_fixup.cu): device list + count, grown on use
    double lambda_d = 0.0;            // masked float64 kernel
    float fix_ratio = 300.f;     // ||y-c||^2 / RSS above which a pixel is recomputed in float64
    // Plan-owned scratch (the fixup list + count, the masked BIG rings) is shared by every
    // bwm_monitor call on the plan: calls that use it are ordered on the device through
    // scratch_ev (each waits for the previous user's last kernel, then records its own), so
    // concurrent calls on different streams — the chunked host pipeline, or callers — never
    // overlap on it.  scratch_mu makes the wait + record pair atomic across host threads.
    mutable std::mutex scratch_mu;
    cudaEvent_t scratch_ev = nullptr;
    mutable int64_t* d_fix_list = nullptr;
    mutable unsigned int* d_fix_count = nullptr;
    mutable int64_t fix_cap = 0;
    // TMA kernel: dynamic per-warp slice scheduler (two counters, zeroed here, reset by the
    // kernel's last warp); plan scratch like the fixup list (BWM_DYN=0: static schedule)
    unsigned int* d_sched = nullptr;
    bool dyn = true;
    // TALL variant of the LEAN TMEM-ring kernel (16-date stages, bwm_kernel_tma.cuh): used for
    // LEAN launches when its ring needs the same Tensor Memory and CTAs per SM (BWM_TALL=0: off)
    bool tall = false;
    bool tall_nomirror = false;        // the TALL ring without mirror rows (fits where 16 mirror rows would not)
    TmaRing tring_tall{};
    int64_t smem_tall = 0;
    int bpm_tall = 0;
    int bpm_tma_lean = 0;              // resident CTAs per SM of the LEAN TMA variant
    // lagging-cursor geometries: fitted values on the tensor cores (bwm_kernel_mma.cuh)
    bool use_mma = false;
    int64_t smem_mma = 0;
    float* d_zb_cur = nullptr;
    float* d_zb_lag = nullptr;
    // masked-NaN mode (bwm_kernel_masked.cuh)
    bool masked = false;
    bool mbig = false;                 // x x^T table + rings in global memory
    int64_t smem_masked = 0;
    int bpm_masked = 0;
    float* d_xx = nullptr;
    double* d_gfull = nullptr;
    float* d_ring = nullptr;           // [sms * bpm_masked][h][128] when mbig
    double gscale = 0.0;               // exact-digit Gram complement scale (bwm::mask_digits)
    HostPipe pipe;
    std::unique_ptr<bwm::StagedReader> freader;   // bwm_monitor_file: pinned slots + reader pool
    std::mutex mu;                     // serialises bwm_monitor_host on one plan
};

static int validate_dims(const bwm_dims* d) {
    if (!d) return set_err(BWM_E_NULL, "dims is NULL");
    if (d->n_params < 4 || d->n_params > 18 || (d->n_params & 1))
        return set_err(BWM_E_PARAMS, "n_params=%d not in {4,6,...,18} (harmonics 1..8)", d->n_params);
    if (!(d->n_hist > d->n_params))
        return set_err(BWM_E_DIMS, "history must exceed the coefficient count (n=%d, p=%d)",
                       d->n_hist, d->n_params);
    if (!(d->n_hist < d->n_obs))
        return set_err(BWM_E_DIMS, "history must end before the series does (n=%d, N=%d)",
                       d->n_hist, d->n_obs);
    if (d->nan_mode != BWM_NAN_FILL && d->nan_mode != BWM_NAN_MASK)
        return set_err(BWM_E_PARAMS, "nan_mode=%d is neither BWM_NAN_FILL nor BWM_NAN_MASK", d->nan_mode);
    if (d->bandwidth < 1 || d->bandwidth > d->n_hist)
        return set_err(BWM_E_DIMS, "bandwidth must satisfy 1 <= h <= n (h=%d, n=%d)", d->bandwidth,
                       d->n_hist);
    return BWM_OK;
}

static void plan_free_tables(bwm_plan* plan) {
    cudaFree(plan->d_xt);
    cudaFree(plan->d_bound);
    cudaFree(plan->d_rinv);
    cudaFree(plan->d_xtd);
    cudaFree(plan->d_wt);
    cudaFree(plan->d_wtd);
    cudaFree(plan->d_fix_list);
    cudaFree(plan->d_fix_count);
    cudaFree(plan->d_sched);
    plan->d_sched = nullptr;
    cudaFree(plan->d_xx);
    cudaFree(plan->d_gfull);
    cudaFree(plan->d_ring);
    cudaFree(plan->d_zb_cur);
    cudaFree(plan->d_zb_lag);
    if (plan->scratch_ev) cudaEventDestroy(plan->scratch_ev);
    plan->scratch_ev = nullptr;
}


// CTAs per SM for a kernel that allocates Tensor Memory dynamically: the occupancy API
// assumes such a kernel owns the SM's TMEM (reports 1), so bound residency by registers,
// shared memory, threads and our own column budget (512 columns / tmem_cols per CTA).
static int resident_ctas(const void* fn, int threads, int64_t smem, int tmem_cols, int device, cudaError_t* err) {
    cudaFuncAttributes fa{};
    if ((*err = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return 0;
    int regs_per_sm = 0, smem_per_sm = 0, reserved = 0, max_threads = 0;
    cudaDeviceGetAttribute(&regs_per_sm, cudaDevAttrMaxRegistersPerMultiprocessor, device);
    cudaDeviceGetAttribute(&smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
    cudaDeviceGetAttribute(&max_threads, cudaDevAttrMaxThreadsPerMultiProcessor, device);
    const int warps = (threads + 31) / 32;
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;     // per-warp allocation unit
    const int by_regs = regs_per_sm / (regs_warp * warps);
    const int by_smem = (int)(smem_per_sm / (smem + (int64_t)fa.sharedSizeBytes + reserved));
    const int by_thr = max_threads / threads;
    const int by_tmem = 512 / tmem_cols;
    return std::max(1, std::min(std::min(by_regs, by_smem), std::min(by_thr, by_tmem)));
}

// round to the nearest tf32 (10 explicit mantissa bits), as a float32 bit pattern
static float tf32_round(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    if ((b & 0x7f800000u) != 0x7f800000u) b = (b + 0xfffu + ((b >> 13) & 1u)) & 0xffffe000u;
    std::memcpy(&x, &b, 4);
    return x;
}

// Masked-NaN plan: float32 X'^T for residuals; the x_t x_t^T lower triangles of the history
// dates as tf32 hi + lo tiles in the tensor-core operand layout (bwm_kernel_masked.cuh: per
// 16-date block, [step][hi|lo][N/8 row groups][2 K chunks][8 rows][4 dates], zero padded);
// their float64 total G_full (summed from the same hi + lo values, so G_v = G_full - Gm is
// the Gram of exactly those rows); lambda.
static int plan_create_masked(bwm_plan* plan, const bwm_tables* tb, int max_optin, bwm_plan** out_plan) {
    const bwm_dims& d = plan->dims;
    const int N = d.n_obs, n = d.n_hist, p = d.n_params, h = d.bandwidth, sp = plan->sp;
    const int kk = p * (p + 1) / 2, nn = bwm::gram_nn(p);
    const int n16 = ((n + bwm::kMaskD - 1) / bwm::kMaskD) * bwm::kMaskD;
    plan->masked = true;
    const int64_t small = bwm::masked_smem_bytes(N, n, h, p, false);
    plan->mbig = small > kMaskedSmemMax;
    plan->smem_masked = bwm::masked_smem_bytes(N, n, h, p, plan->mbig);
    if (plan->smem_masked > max_optin) {
        const int64_t need = plan->smem_masked;
        plan_free_tables(plan);
        delete plan;
        return set_err(BWM_E_SMEM, "masked tables need %lld B of shared memory, device allows %d",
                       (long long)need, max_optin);
    }
    if (n16 > 65535 || N > 65535) {
        plan_free_tables(plan);
        delete plan;
        return set_err(BWM_E_DIMS, "masked mode supports at most 65535 dates");
    }
    // X'^T zero-padded by kMaskD rows (the BIG kernel reads it from global memory)
    std::vector<float> xt((size_t)(N + bwm::kMaskD) * sp, 0.f), tiles((size_t)(n16 / bwm::kMaskD) * nn * 32, 0.f);
    std::vector<double> gf((size_t)kk, 0.0);
    for (int t = 0; t < N; ++t)
        for (int i = 0; i < p; ++i) xt[(size_t)t * sp + i] = (float)tb->design[(size_t)i * N + t];
    // x_t x_t^T of the float32 design rows the kernel multiplies with (products of two floats are
    // exact in float64).  p <= 14 (bwm::mask_digits): two 11-bit fixed-point digits of x x^T / S
    // (S: a power of two >= max |x x^T|), integer-valued and exact in tf32, accumulated by the
    // kernel in separate TMEM regions (exact integer sums); Gm = S/2048 (D_hi + D_lo/2048).
    // p >= 16: tf32 hi + lo of the float32 product in one region.
    const bool digits = bwm::mask_digits(p);
    double smax = 0.0;
    for (int t = 0; t < n; ++t)
        for (int i = 0; i < p; ++i)
            for (int j = 0; j <= i; ++j)
                smax = std::max(smax, std::fabs((double)(float)tb->design[(size_t)i * N + t] *
                                                (double)(float)tb->design[(size_t)j * N + t]));
    double gsc = 1.0;
    while (gsc < smax) gsc *= 2.0;
    while (smax > 0.0 && gsc / 2.0 >= smax) gsc /= 2.0;
    plan->gscale = gsc / 2048.0;
    for (int t = 0; t < n; ++t) {
        const int kb = t / bwm::kMaskD, step = (t % bwm::kMaskD) / 8, k = t % 8;
        for (int i = 0; i < p; ++i)
            for (int j = 0; j <= i; ++j) {
                const int e = i * (i + 1) / 2 + j;
                const double pr = (double)(float)tb->design[(size_t)i * N + t] * (double)(float)tb->design[(size_t)j * N + t];
                float hi, lo;
                if (digits) {
                    const double u = pr / gsc * 2048.0;             // |u| <= 2048
                    hi = (float)std::nearbyint(u);
                    lo = (float)std::nearbyint((u - (double)hi) * 2048.0);
                    gf[e] += plan->gscale * ((double)hi + (double)lo / 2048.0);
                } else {
                    const float v = (float)pr;
                    hi = tf32_round(v);
                    lo = tf32_round(v - hi);
                    gf[e] += (double)hi + (double)lo;
                }
                const size_t in_region = (size_t)(e / 8) * 64 + (k / 4) * 32 + (e % 8) * 4 + (k % 4);
                const size_t base = (size_t)kb * nn * 32 + (size_t)(2 * step) * nn * 8;
                tiles[base + in_region] = hi;
                tiles[base + (size_t)nn * 8 + in_region] = lo;
            }
    }
    auto fail = [&](cudaError_t e, const char* what) {
        plan_free_tables(plan);
        delete plan;
        return set_err((int)e, "%s: %s", what, cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&plan->d_xt, xt.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&plan->d_xx, tiles.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&plan->d_gfull, gf.size() * 8)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMemcpy(plan->d_xt, xt.data(), xt.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    if ((e = cudaMemcpy(plan->d_xx, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    if ((e = cudaMemcpy(plan->d_gfull, gf.data(), gf.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    plan->lambda = (float)tb->bound[0];    // bound_0 = crit * sqrt(log_plus((n+1)/n)) = crit
    plan->lambda_d = tb->bound[0];
    {
        // long monitoring horizons: every pixel through the float64 masked kernel (bwm_fixup.cu)
        double s_max = 0.0;
        for (int t = n; t < N; ++t) s_max = std::max(s_max, std::fabs(tb->design[(size_t)1 * N + t]));
        const char* prec_env = getenv("BWM_PRECISE");
        plan->precise = prec_env ? std::strcmp(prec_env, "1") == 0 : s_max > 8.0;
        if (plan->precise) {
            std::vector<double> xd((size_t)N * sp, 0.0);
            for (int t = 0; t < N; ++t)
                for (int i = 0; i < p; ++i) xd[(size_t)t * sp + i] = tb->design[(size_t)i * N + t];
            cudaError_t e2 = cudaMalloc(&plan->d_xtd, xd.size() * 8);
            if (e2 == cudaSuccess) e2 = cudaMemcpy(plan->d_xtd, xd.data(), xd.size() * 8, cudaMemcpyHostToDevice);
            if (e2 != cudaSuccess) {
                plan_free_tables(plan);
                delete plan;
                return set_err((int)e2, "masked float64 table: %s", cudaGetErrorString(e2));
            }
        }
    }
    KernelFn fn = pick_masked(p, plan->mbig, false);
    for (int keep = 0; keep < 2; ++keep)
        if ((e = cudaFuncSetAttribute((const void*)pick_masked(p, plan->mbig, keep), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_optin)) != cudaSuccess)
            return fail(e, "cudaFuncSetAttribute");
    plan->bpm_masked = resident_ctas((const void*)fn, bwm::kMaskThreads, plan->smem_masked,
                                     bwm::masked_tmem_cols(p), plan->device, &e);
    if (e != cudaSuccess) return fail(e, "cudaFuncGetAttributes");
    if (plan->mbig) {
        const size_t rb = (size_t)plan->sms * plan->bpm_masked * bwm::masked_scratch_words(h, p, true) * bwm::kMaskThreads * 4;
        if ((e = cudaMalloc(&plan->d_ring, rb)) != cudaSuccess) return fail(e, "cudaMalloc(ring)");
    }
    *out_plan = plan;
    return BWM_OK;
}

extern "C" {

const char* bwm_last_error(void) { return g_err.c_str(); }
int bwm_abi_version(void) { return BWM_ABI_VERSION; }
int64_t bwm_launch_count(void) { return g_launches.load(); }

int bwm_zero_sigma_init(int64_t* z, void* stream) {
    if (!z) return set_err(BWM_E_NULL, "zero_sigma_pixel is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    // INT64_MAX little-endian: bytes 0-6 = 0xff, byte 7 = 0x7f
    BWM_CUDA(cudaMemsetAsync(z, 0xff, 7, st));
    BWM_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(z) + 7, 0x7f, 1, st));
    return BWM_OK;
}

int64_t bwm_smem_bytes(const bwm_dims* d) {
    int rc = validate_dims(d);
    if (rc) return rc;
    if (d->nan_mode == BWM_NAN_MASK) {
        const int64_t small = bwm::masked_smem_bytes(d->n_obs, d->n_hist, d->bandwidth, d->n_params, false);
        return small <= kMaskedSmemMax ? small
                                       : bwm::masked_smem_bytes(d->n_obs, d->n_hist, d->bandwidth, d->n_params, true);
    }
    constexpr int64_t kOptin = 232448;                 // sm_100 opt-in limit per CTA (no device here)
    bool ring = d->bandwidth <= kRingMaxH;
    int64_t ldg = smem_bytes_for(d->n_obs, d->n_hist, d->bandwidth, d->n_params, ring);
    if (ldg > kOptin && ring) ldg = smem_bytes_for(d->n_obs, d->n_hist, d->bandwidth, d->n_params, false);
    const int mode = tma_ring_for(d->bandwidth).mode;
    int64_t tma = smem_bytes_tma(d->n_obs, d->n_hist, d->bandwidth, d->n_params, mode);
    int tmode = mode;
    if (tma > kOptin && mode == (int)bwm::kRingTmem) tmode = bwm::kRingLag;
    if (tmode == (int)bwm::kRingLag &&
        smem_bytes_tma(d->n_obs, d->n_hist, d->bandwidth, d->n_params, bwm::kRingLagT) <= (BWM_LAGT_WARPS > 4 ? kOptin : (110 << 10)))
        tmode = bwm::kRingLagT;
    if (tmode != mode) tma = smem_bytes_tma(d->n_obs, d->n_hist, d->bandwidth, d->n_params, tmode);
    return tma > 0 ? tma : ldg;
}

int bwm_plan_create(const bwm_dims* dims, const bwm_tables* tb, int device, bwm_plan** out_plan) {
    if (!out_plan) return set_err(BWM_E_NULL, "out_plan is NULL");
    *out_plan = nullptr;
    int rc = validate_dims(dims);
    if (rc) return rc;
    if (!tb || !tb->design || !tb->bound)
        return set_err(BWM_E_NULL, "tables (design, bound) must be non-NULL");
    if (!(tb->trend_scale > 0) || !std::isfinite(tb->trend_center))
        return set_err(BWM_E_DIMS, "trend_scale must be positive and trend_center finite");

    DeviceRestore guard(device);
    BWM_CUDA(cudaSetDevice(device));
    const int N = dims->n_obs, n = dims->n_hist, p = dims->n_params, h = dims->bandwidth;
    const int sp = (p + 3) & ~3;

    auto* plan = new bwm_plan();
    plan->dims = *dims;
    plan->device = device;
    plan->sp = sp;
    plan->ring = h <= kRingMaxH;
    plan->smem = smem_bytes_for(N, n, h, p, plan->ring);
    plan->tring = tma_ring_for(h);
    plan->smem_tma = smem_bytes_tma(N, n, h, p, plan->tring.mode);
    {
        // long series: when the staged tables do not fit, run the lagging-cursor variants,
        // which read the tables through L1 (any N)
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        if (plan->smem > optin && plan->ring) {
            plan->ring = false;
            plan->smem = smem_bytes_for(N, n, h, p, false);
        }
        if (plan->smem_tma > optin && plan->tring.mode == (int)bwm::kRingTmem) {
            plan->tring = {(int)bwm::kRingLag, 0, 0};
            plan->smem_tma = smem_bytes_tma(N, n, h, p, plan->tring.mode);
        }
        // lagging cursor: tables staged in smem when they fit (kRingLagT), else through L1
        const char* l1_env = getenv("BWM_TMA_LAGL1");        // A/B: keep the L1-table variant
        if (plan->tring.mode == (int)bwm::kRingLag && !(l1_env && std::strcmp(l1_env, "1") == 0) &&
            smem_bytes_tma(N, n, h, p, bwm::kRingLagT) <= std::min<int64_t>(optin, BWM_LAGT_WARPS > 4 ? optin : (110 << 10))) {
            plan->tring = {(int)bwm::kRingLagT, 0, 0};
            plan->smem_tma = smem_bytes_tma(N, n, h, p, plan->tring.mode);
        }
    }
    const char* env = getenv("BWM_KERNEL");
    plan->force_ldg = env && strcmp(env, "ldg") == 0;
    plan->inv_dof = (float)(1.0 / (double)(n - p));
    plan->sqrt_n = (float)std::sqrt((double)n);
    plan->tc_ts = (float)(tb->trend_center / tb->trend_scale);
    plan->inv_ts = (float)(1.0 / tb->trend_scale);

    int max_optin = 0;
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&plan->sms, cudaDevAttrMultiProcessorCount, device);
    {
        cudaError_t e0 = cudaEventCreateWithFlags(&plan->scratch_ev, cudaEventDisableTiming);
        if (e0 != cudaSuccess) {
            delete plan;
            return set_err((int)e0, "cudaEventCreate: %s", cudaGetErrorString(e0));
        }
        const char* dyn_env = getenv("BWM_DYN");
        plan->dyn = !(dyn_env && std::strcmp(dyn_env, "0") == 0);
        if (plan->dyn && dims->nan_mode != BWM_NAN_MASK) {
            e0 = cudaMalloc(&plan->d_sched, 2 * sizeof(unsigned int));
            if (e0 == cudaSuccess) e0 = cudaMemset(plan->d_sched, 0, 2 * sizeof(unsigned int));
            if (e0 != cudaSuccess) {
                plan_free_tables(plan);
                delete plan;
                return set_err((int)e0, "scheduler counters: %s", cudaGetErrorString(e0));
            }
        }
    }
    if (dims->nan_mode == BWM_NAN_MASK) return plan_create_masked(plan, tb, max_optin, out_plan);
    if (plan->smem_tma > max_optin || plan->tring.mode < 0) plan->smem_tma = 0;
    if (plan->smem > max_optin) {
        int64_t need = plan->smem;
        plan_free_tables(plan);
        delete plan;
        return set_err(BWM_E_SMEM, "tables need %lld B of shared memory, device allows %d",
                       (long long)need, max_optin);
    }

    // History least squares, float64: thin QR of the centred history design X'_h^T = Q R
    // (modified Gram-Schmidt, two passes).  Q^T y_h are the coefficients in an orthonormal
    // basis (so RSS = ||y_h||^2 - ||Q^T y_h||^2 in one sweep), Z = R^-T X' maps them to fitted
    // values for every date, and R^-1 maps them back to beta' for the beta output.
    std::vector<double> Q((size_t)n * p), Rm((size_t)p * p, 0.0);
    for (int j = 0; j < p; ++j) {
        for (int t = 0; t < n; ++t) Q[(size_t)t * p + j] = tb->design[(size_t)j * N + t];
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i < j; ++i) {
                double d = 0.0;
                for (int t = 0; t < n; ++t) d += Q[(size_t)t * p + i] * Q[(size_t)t * p + j];
                Rm[(size_t)i * p + j] += d;
                for (int t = 0; t < n; ++t) Q[(size_t)t * p + j] -= d * Q[(size_t)t * p + i];
            }
        double nrm = 0.0;
        for (int t = 0; t < n; ++t) nrm += Q[(size_t)t * p + j] * Q[(size_t)t * p + j];
        nrm = std::sqrt(nrm);
        if (!(nrm > 1e-12)) {
            plan_free_tables(plan);
            delete plan;
            return set_err(BWM_E_DIMS, "history design is rank deficient (column %d)", j);
        }
        Rm[(size_t)j * p + j] = nrm;
        for (int t = 0; t < n; ++t) Q[(size_t)t * p + j] /= nrm;
    }
    std::vector<double> Rinv((size_t)p * p, 0.0);          // upper triangular
    for (int col = 0; col < p; ++col)
        for (int i = col; i >= 0; --i) {
            double v = (i == col) ? 1.0 : 0.0;
            for (int k = i + 1; k <= col; ++k) v -= Rm[(size_t)i * p + k] * Rinv[(size_t)k * p + col];
            Rinv[(size_t)i * p + col] = v / Rm[(size_t)i * p + i];
        }
    // float32 tables, transposed so one date's coefficients are contiguous (LDS.128)
    // (Z^T: the tensor-core fitted-value kernel, bwm_kernel_mma.cuh, reads its Q rows from it)
    std::vector<float> xt((size_t)N * sp, 0.f), bd((size_t)(N - n)), ri((size_t)p * p);
    for (int t = 0; t < N; ++t)
        for (int i = 0; i < p; ++i) {      // z_t = R^-T x_t  <=>  z_t,i = sum_k Rinv[k][i] x_k,t
            double z = 0.0;
            for (int k = 0; k <= i; ++k) z += Rinv[(size_t)k * p + i] * tb->design[(size_t)k * N + t];
            xt[(size_t)t * sp + i] = (float)(t < n ? Q[(size_t)t * p + i] : z);   // z_t == q_t for t < n
        }
    for (int j = 0; j < N - n; ++j) bd[j] = (float)tb->bound[j];
    for (size_t i = 0; i < ri.size(); ++i) ri[i] = (float)Rinv[i];
    // Long monitoring horizons: the fitted value of a far-extrapolated date carries the float32
    // error of (t - tc)/ts times the trend coefficient, which the MOSUM scale 1/(sigma sqrt n)
    // can amplify past 1e-4 (fuzz: N/n = 15).  Beyond |(t - tc)/ts| = 8 (N/n ~ 4.5 on a regular
    // axis) the fitted values are computed in float64 (LDG kernel, float64 Z^T).
    double s_max = 0.0;
    for (int t = n; t < N; ++t) s_max = std::max(s_max, std::fabs(tb->design[(size_t)1 * N + t]));
    const char* fix_env = getenv("BWM_FIX_RATIO");                   // 0 disables the fixup
    if (fix_env) plan->fix_ratio = (float)std::atof(fix_env);
    const char* prec_env = getenv("BWM_PRECISE");
    plan->precise = prec_env ? std::strcmp(prec_env, "1") == 0 : s_max > 8.0;
    std::vector<double> xtd;
    {
        xtd.assign((size_t)N * sp, 0.0);
        for (int t = 0; t < N; ++t)
            for (int i = 0; i < p; ++i) {
                double z = 0.0;
                for (int k = 0; k <= i; ++k) z += Rinv[(size_t)k * p + i] * tb->design[(size_t)k * N + t];
                xtd[(size_t)t * sp + i] = t < n ? Q[(size_t)t * p + i] : z;
            }
    }
    // Window-sum table (bwm_common.cuh, KParams::wt): rows t < n are q_t (pass 1), rows t >= n
    // S_t = sum of z_s over the MOSUM window of date t, [t-h+1, t] (mosum.py:59), in float64.
    // Design row 0 is the intercept (bwm_tables), so z_s[0] = 1/R00 for every s: S_t[0] is the
    // constant s0 = h/R00, applied once to the initial window sum, and column 0 is stored as 0.
    for (int t = 0; t < N; ++t)
        if (tb->design[t] != 1.0) {
            plan_free_tables(plan);
            delete plan;
            return set_err(BWM_E_DIMS, "design row 0 must be the intercept (1.0 at every date)");
        }
    std::vector<double> wtd((size_t)N * sp, 0.0);
    for (int t = 0; t < n; ++t)
        for (int i = 0; i < p; ++i) wtd[(size_t)t * sp + i] = Q[(size_t)t * p + i];
    for (int i = 1; i < p; ++i) {          // sliding window sum, O(N p) (long series)
        double s = 0.0;
        for (int u = n - h + 1; u <= n; ++u) s += xtd[(size_t)u * sp + i];
        wtd[(size_t)n * sp + i] = s;
        for (int t = n + 1; t < N; ++t) {
            s += xtd[(size_t)t * sp + i] - xtd[(size_t)(t - h) * sp + i];
            wtd[(size_t)t * sp + i] = s;
        }
    }
    plan->s0 = (double)h * Rinv[0];
    std::vector<float> wt(wtd.size());
    for (size_t i = 0; i < wt.size(); ++i) wt[i] = (float)wtd[i];

    auto fail = [&](cudaError_t e, const char* what) {
        plan_free_tables(plan);
        delete plan;
        return set_err((int)e, "%s: %s", what, cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&plan->d_xt, xt.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&plan->d_bound, std::max<size_t>(bd.size(), 1) * 4)) != cudaSuccess)
        return fail(e, "cudaMalloc");
    if ((e = cudaMemcpy(plan->d_xt, xt.data(), xt.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    if ((e = cudaMemcpy(plan->d_bound, bd.data(), bd.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    if ((e = cudaMalloc(&plan->d_rinv, ri.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMemcpy(plan->d_rinv, ri.data(), ri.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    {
        if ((e = cudaMalloc(&plan->d_xtd, xtd.size() * 8)) != cudaSuccess) return fail(e, "cudaMalloc");
        if ((e = cudaMemcpy(plan->d_xtd, xtd.data(), xtd.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(e, "cudaMemcpy");
    }
    if ((e = cudaMalloc(&plan->d_wt, wt.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMemcpy(plan->d_wt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy");
    if (plan->precise) {
        if ((e = cudaMalloc(&plan->d_wtd, wtd.size() * 8)) != cudaSuccess) return fail(e, "cudaMalloc");
        if ((e = cudaMemcpy(plan->d_wtd, wtd.data(), wtd.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(e, "cudaMemcpy");
    }

    // Lagging-cursor geometries (large h): the tensor-core fitted-value kernel (bwm_kernel_mma.cuh)
    // when BWM_MMA=1 and its tables fit shared memory.  Opt-in: measured SLOWER than the FFMA
    // kernel at C4 (10.2 vs 8.2 ms; profiles/r02_C4_mma_ncu_summary.txt), so not the default.
    if (plan->smem_tma > 0 && (plan->tring.mode == (int)bwm::kRingLag || plan->tring.mode == (int)bwm::kRingLagT)) {
        const char* mma_env = getenv("BWM_MMA");
        const bool want = mma_env && std::strcmp(mma_env, "1") == 0;
        const int64_t sm = bwm::mma_smem_bytes(N, n, h, p);
        if (want && sm <= max_optin && plan->d_xtd) {
            const bwm::MmaGeom g = bwm::mma_geom(N, n, h);
            const int KS = bwm::mma_ks(p);
            // [split][K-step][group][K chunk][8 rows][4]: z_t split into tf32 hi + lo
            auto build = [&](int date0, int groups, std::vector<float>& tab) {
                tab.assign((size_t)2 * KS * groups * 64, 0.f);
                for (int gi = 0; gi < groups; ++gi)
                    for (int r = 0; r < 8; ++r) {
                        const int t = date0 + 8 * gi + r;
                        if (t < 0 || t >= N) continue;
                        for (int k = 0; k < p; ++k) {
                            const float v = (float)xtd[(size_t)t * sp + k];
                            const float hi = tf32_round(v), lo = tf32_round(v - hi);
                            const int ks = k / 8, kc = (k % 8) / 4, e = k % 4;
                            const size_t in = (size_t)gi * 64 + kc * 32 + r * 4 + e;
                            tab[((size_t)(0 * KS + ks) * groups) * 64 + in] = hi;
                            tab[((size_t)(1 * KS + ks) * groups) * 64 + in] = lo;
                        }
                    }
            };
            std::vector<float> tc, tl;
            build(g.w0, g.gcur, tc);
            build(g.t3 - h, g.glag, tl);
            if ((e = cudaMalloc(&plan->d_zb_cur, tc.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
            if ((e = cudaMalloc(&plan->d_zb_lag, tl.size() * 4)) != cudaSuccess) return fail(e, "cudaMalloc");
            if ((e = cudaMemcpy(plan->d_zb_cur, tc.data(), tc.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(e, "cudaMemcpy");
            if ((e = cudaMemcpy(plan->d_zb_lag, tl.data(), tl.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(e, "cudaMemcpy");
            for (int lean = 0; lean < 2; ++lean)
                if ((e = cudaFuncSetAttribute((const void*)pick_mma(p, lean), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              max_optin)) != cudaSuccess)
                    return fail(e, "cudaFuncSetAttribute");
            plan->use_mma = true;
            plan->smem_mma = sm;
        }
    }

    // LEAN TMA variant: the boundary is one value over the whole monitoring period
    plan->const_bound = true;
    for (int j = 1; j < N - n; ++j) plan->const_bound = plan->const_bound && bd[(size_t)j] == bd[0];

    // per kernel: the dynamic shared-memory limit and the resident CTAs per SM
    auto setup = [&](KernelFn fn, Kind kind, int64_t sm, int* nb_out) -> cudaError_t {
        // the limit is per-kernel global state shared by every plan: set it to the device
        // maximum once, never lower it (a later plan must not shrink an earlier plan's launch)
        cudaError_t err = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
        if (err != cudaSuccess) return err;
        int nb = 0;
        if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn, threads_of(kind, plan->tring.mode), (size_t)sm)) !=
            cudaSuccess)
            return err;
        if (kind == kTma && plan->tring.mode == bwm::kRingTmem) {
            // The occupancy API assumes a kernel that allocates Tensor Memory owns the SM's
            // TMEM (reports 1).  Allocation is dynamic (tcgen05.alloc + relinquish_alloc_permit),
            // so residency is bounded by registers, shared memory, threads and our own column
            // budget: 512 columns per SM / tmem_cols per CTA.
            nb = resident_ctas((const void*)fn, threads_of(kind, plan->tring.mode), sm,
                               plan->tring.cols * (bwm::tma_warps(bwm::kRingTmem) / 4), device, &err);
            if (err != cudaSuccess) return err;
        }
        *nb_out = nb;
        return cudaSuccess;
    };
    for (int v = 0; v < 3; ++v) {
        const Kind kind = (Kind)v;
        const int64_t sm = kind == kTma ? plan->smem_tma : plan->smem;
        if (kind == kTma && sm == 0) continue;
        int nb = 0;
        if ((e = setup(pick(p, kind, kind == kTma ? plan->tring.mode : (plan->ring ? 0 : (int)bwm::kRingLag)), kind,
                       sm, &nb)) != cudaSuccess)
            return fail(e, "kernel setup");
        plan->occ_raw[v] = nb;
        plan->blocks_per_sm[v] = std::max(nb, 1);
        if (kind == kTma) {
            if ((e = setup(pick(p, kind, plan->tring.mode | bwm::kTmaLean), kind, sm, &nb)) != cudaSuccess)
                return fail(e, "kernel setup");
            plan->bpm_tma_lean = std::max(nb, 1);
        }
    }
    {
        const char* tall_env = getenv("BWM_TALL");
        const bool want = !(tall_env && std::strcmp(tall_env, "0") == 0);
        constexpr int RT = bwm::kTallRows;
        if (want && bwm::kStageRows == 8 && plan->tring.mode == (int)bwm::kRingTmem && plan->smem_tma > 0 &&
            plan->const_bound && h >= RT) {
            const int L = ((h + RT - 1) / RT) * RT;
            auto pow2 = [](int need) { int c = 32; while (c < need) c *= 2; return c; };
            const char* nm_env = getenv("BWM_TALL_NOMIRROR");       // A/B: 0 never, 1 whenever mirrors do not fit
            const bool nm_ok = !(nm_env && std::strcmp(nm_env, "0") == 0);
            const bool mir = pow2(2 * (L + RT)) == plan->tring.cols;
            const bool nomir = !mir && nm_ok && pow2(2 * L) == plan->tring.cols;
            const int need = 2 * (L + (mir ? RT : 0));
            const int cols = pow2(need);
            if ((mir || nomir) && need <= tmem_cols_max()) {
                const int64_t sm = plan->smem_tma - bwm::tma_stage_region(bwm::kRingTmem, bwm::kStages) +
                                   (int64_t)bwm::tma_warps(bwm::kRingTmem) * BWM_STAGES_TALL * RT * bwm::kWarpPx * 4;
                int nb = 0;
                const int tmode = bwm::kRingTmem | bwm::kTmaLean | bwm::kTmaTall | (nomir ? bwm::kTmaNoMirror : 0);
                if ((e = setup(pick(p, kTma, tmode), kTma, sm, &nb)) != cudaSuccess)
                    return fail(e, "kernel setup (tall)");
                if (nb >= plan->bpm_tma_lean) {
                    plan->tall = true;
                    plan->tall_nomirror = nomir;
                    plan->tring_tall = {(int)bwm::kRingTmem, L, cols};
                    plan->smem_tall = sm;
                    plan->bpm_tall = nb;
                }
            }
        }
    }
    *out_plan = plan;
    return BWM_OK;
}

static void pipe_free(HostPipe& hp) {
    for (int b = 0; b < 2; ++b) {
        cudaFree(hp.d_y[b]);
        cudaFree(hp.d_valid[b]);
        cudaFree(hp.d_first[b]);
        cudaFree(hp.d_max[b]);
        cudaFree(hp.d_beta[b]);
        cudaFree(hp.d_mean[b]);
        cudaFree(hp.d_mosum[b]);
        cudaFree(hp.d_fb[b]);
        cudaFree(hp.d_mx64[b]);
        cudaFree(hp.d_det[b]);
        if (hp.s_h2d[b]) cudaStreamDestroy(hp.s_h2d[b]);
        if (hp.s_k[b]) cudaStreamDestroy(hp.s_k[b]);
        for (cudaEvent_t ev : {hp.ev_in[b], hp.ev_k0[b], hp.ev_k1[b], hp.ev_free[b]})
            if (ev) cudaEventDestroy(ev);
    }
    cudaFree(hp.d_zero);
    if (hp.h_stage) cudaFreeHost(hp.h_stage);
    hp = HostPipe();
}

void bwm_plan_destroy(bwm_plan* plan) {
    if (!plan) return;
    DeviceRestore guard(plan->device);
    cudaSetDevice(plan->device);
    pipe_free(plan->pipe);
    plan_free_tables(plan);
    delete plan;
}

int bwm_monitor(const bwm_plan* plan, const float* y, int64_t ld_y, int64_t n_pixels,
                int64_t pixel_offset, const bwm_outputs* out, void* stream) {
    if (!plan) return set_err(BWM_E_NULL, "plan is NULL");
    if (!y || !out || !out->valid || !out->first_idx || !out->max_abs || !out->zero_sigma_pixel)
        return set_err(BWM_E_NULL, "y and outputs valid/first_idx/max_abs/zero_sigma_pixel are required");
    if (n_pixels < 1) return set_err(BWM_E_DIMS, "stack needs at least one pixel");
    if (ld_y < n_pixels) return set_err(BWM_E_DIMS, "ld_y (%lld) < n_pixels (%lld)", (long long)ld_y,
                                        (long long)n_pixels);
    if ((out->beta || out->mosum) && out->ld_out < n_pixels)
        return set_err(BWM_E_DIMS, "ld_out (%lld) < n_pixels (%lld)", (long long)out->ld_out,
                       (long long)n_pixels);
    if (pixel_offset < 0) return set_err(BWM_E_DIMS, "pixel_offset must be >= 0");
    if (out->sup_stat && plan->dims.nan_mode != BWM_NAN_FILL)
        return set_err(BWM_E_PARAMS, "sup_stat is a fill-mode output (critical_value)");
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != plan->device)
        return set_err(BWM_E_DEVICE, "plan lives on device %d, current device is %d", plan->device, cur);

    const bwm_dims& d = plan->dims;
    bwm::KParams k{};
    k.y = y;
    k.ld_y = ld_y;
    k.n_pixels = n_pixels;
    k.pixel_offset = pixel_offset;
    k.N = d.n_obs;
    k.n = d.n_hist;
    k.h = d.bandwidth;
    k.sp = plan->sp;
    k.xt = plan->d_xt;
    k.bound = plan->d_bound;
    k.rinv = plan->d_rinv;
    k.inv_dof = plan->inv_dof;
    k.sqrt_n = plan->sqrt_n;
    k.ring_rows = plan->tring.rows;
    k.tmem_cols = plan->tring.cols;
    k.tc_ts = plan->tc_ts;
    k.inv_ts = plan->inv_ts;
    k.valid = out->valid;
    k.first_idx = out->first_idx;
    k.max_abs = out->max_abs;
    k.beta = out->beta;
    k.mo_mean = out->mo_mean;
    k.mosum = out->mosum;
    k.sup = out->sup_stat;
    k.ld_out = out->ld_out;
    k.zero_sigma = reinterpret_cast<unsigned long long*>(out->zero_sigma_pixel);
    k.xtd = plan->precise ? plan->d_xtd : nullptr;
    k.wt = plan->d_wt;
    k.wtd = plan->precise ? plan->d_wtd : nullptr;
    k.s0 = plan->s0;
    cudaStream_t st = (cudaStream_t)stream;
    int launched = 0;
    // float64 fixup list for ill-conditioned pixels (fill mode, float32 kernels)
    const bool fixup = !plan->masked && !plan->precise && plan->fix_ratio > 0.f && plan->d_xtd;
    // dynamic slice scheduler of the TMA kernel: the cursor must enter a slice S stages before
    // consumption leaves the previous one (tile_stages > S, bwm_kernel_tma.cuh)
    auto dyn_for = [&](int R, int S) {
        if (plan->masked || !plan->d_sched || plan->use_mma || plan->tring.mode < 0) return false;
        const int n = d.n_hist, N = d.n_obs;
        const int t3 = (n / R) * R;
        const int tile_stages = (n + R - 1) / R + (N - t3 + R - 1) / R;
        return tile_stages > S;
    };
    const bool dyn = dyn_for(bwm::kStageRows, bwm::stages_for(plan->tring.mode));
    const bool dyn_tall = plan->tall && dyn_for(bwm::kTallRows, BWM_STAGES_TALL);
    const bool uses_scratch = fixup || dyn || dyn_tall || (plan->masked && !plan->precise && plan->mbig);
    std::unique_lock<std::mutex> scratch_lock(plan->scratch_mu, std::defer_lock);
    if (uses_scratch) {
        scratch_lock.lock();
        BWM_CUDA(cudaStreamWaitEvent(st, plan->scratch_ev, 0));
    }

    if (plan->masked && plan->precise) {
        bwm::KParams kf = k;
        kf.xtd = plan->d_xtd;
        cudaError_t e = bwm::launch_masked_f64(kf, d.n_params, plan->lambda_d, plan->sms, st);
        if (e != cudaSuccess) return set_err((int)e, "kernel launch failed: %s", cudaGetErrorString(e));
        ++launched;
    } else if (plan->masked) {
        // one launch, any alignment (scalar predicated loads and stores)
        k.xx = plan->d_xx;
        k.gfull = plan->d_gfull;
        k.ring_g = plan->d_ring;
        k.lambda = plan->lambda;
        k.gscale = plan->gscale;
        const int64_t tiles = (n_pixels + bwm::kMaskTile - 1) / bwm::kMaskTile;
        const int64_t grid = std::min<int64_t>(tiles, (int64_t)plan->sms * plan->bpm_masked);
        pick_masked(d.n_params, plan->mbig, out->mosum != nullptr || out->mo_mean != nullptr)<<<(unsigned)grid, bwm::kMaskThreads, (size_t)plan->smem_masked, st>>>(k);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_err((int)e, "kernel launch failed: %s", cudaGetErrorString(e));
        ++launched;
    }

    // Whole 256-pixel tiles go to the TMA kernel (rows 16-byte aligned, outputs 8-byte
    // aligned) or, with BWM_KERNEL=ldg / when its smem does not fit, the LDG fast kernel
    // (rows 8-byte aligned); the tail tile, or everything when misaligned, goes to the
    // scalar bounds-checked LDG kernel.
    auto al = [](const void* q, uintptr_t a) { return (reinterpret_cast<uintptr_t>(q) & (a - 1)) == 0; };
    const bool out_al = al(out->valid, 2) && al(out->first_idx, 8) && al(out->max_abs, 8) &&
                        (!out->mo_mean || al(out->mo_mean, 8)) && (!out->beta || al(out->beta, 8)) &&
                        (!out->mosum || al(out->mosum, 8)) && (!out->sup_stat || al(out->sup_stat, 8)) && (out->ld_out % 2 == 0 || (!out->beta && !out->mosum));
    const bool tma_ok = !plan->masked && !plan->force_ldg && !plan->precise && plan->smem_tma > 0 && al(y, 16) &&
                        (ld_y % 4 == 0) && out_al;
    const bool ldg_ok = al(y, 8) && (ld_y % 2 == 0);
    const Kind main_kind = tma_ok ? kTma : kLdgFast;
    // whole tiles of the main kernel (the TMA kernel's tile is 64 px per warp of its CTA)
    const int64_t main_tile = main_kind == kTma && !plan->use_mma ? bwm::tma_tile(plan->tring.mode) : bwm::kTile;
    const int64_t full = (tma_ok || ldg_ok) ? (n_pixels / main_tile) * main_tile : 0;
    if (fixup) {
        // capacity: every pixel of small calls, 4M entries (32 MB) at most — flagged pixels are
        // rare on real data, and a near-capacity stack must not run out of HBM for the list
        const int64_t want = std::min<int64_t>(n_pixels, 4ll << 20);
        if (plan->fix_cap < want) {
            cudaFree(plan->d_fix_list);
            plan->d_fix_list = nullptr;
            plan->fix_cap = 0;
            cudaError_t e = cudaMalloc(&plan->d_fix_list, (size_t)want * sizeof(int64_t));
            if (e != cudaSuccess) return set_err((int)e, "fixup list allocation failed: %s", cudaGetErrorString(e));
            plan->fix_cap = want;
            if (!plan->d_fix_count) {
                e = cudaMalloc(&plan->d_fix_count, sizeof(unsigned int));
                if (e != cudaSuccess) return set_err((int)e, "fixup count allocation failed: %s", cudaGetErrorString(e));
            }
        }
        cudaError_t e = cudaMemsetAsync(plan->d_fix_count, 0, sizeof(unsigned int), st);
        if (e != cudaSuccess) return set_err((int)e, "cudaMemsetAsync failed: %s", cudaGetErrorString(e));
        k.fix_list = plan->d_fix_list;
        k.fix_count = plan->d_fix_count;
        k.fix_cap = (unsigned int)plan->fix_cap;
        k.fix_ratio = plan->fix_ratio;
    }
    for (int part = 0; part < 2 && !plan->masked; ++part) {
        const Kind kind = part == 0 ? main_kind : kLdgSafe;
        const int64_t p0 = part == 0 ? 0 : full;
        const int64_t cnt = part == 0 ? full : n_pixels - full;
        if (cnt <= 0) continue;
        bwm::KParams kp = k;
        kp.fix_base = p0;
        kp.y = y + p0;
        kp.n_pixels = cnt;
        kp.pixel_offset = pixel_offset + p0;
        kp.valid = out->valid + p0;
        kp.first_idx = out->first_idx + p0;
        kp.max_abs = out->max_abs + p0;
        kp.beta = out->beta ? out->beta + p0 : nullptr;
        kp.mo_mean = out->mo_mean ? out->mo_mean + p0 : nullptr;
        kp.mosum = out->mosum ? out->mosum + p0 : nullptr;
        kp.sup = out->sup_stat ? out->sup_stat + p0 : nullptr;
        const bool lean = kind == kTma && plan->const_bound && !out->mosum && !out->mo_mean;
        if (kind == kTma && plan->use_mma) {
            // fitted values on the tensor cores: 1 CTA of two 4-warp sets per SM
            int rc = encode_map(&kp.tmap, kp.y, cnt, d.n_obs, ld_y);
            if (rc) return rc;
            kp.zb_cur = plan->d_zb_cur;
            kp.zb_lag = plan->d_zb_lag;
            const int64_t tiles = cnt / bwm::kTile;
            const int64_t grid = std::min<int64_t>((tiles + bwm::kMmaSets - 1) / bwm::kMmaSets, (int64_t)plan->sms);
            pick_mma(d.n_params, lean)<<<(unsigned)grid, bwm::kMmaThreads, (size_t)plan->smem_mma, st>>>(kp);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return set_err((int)e, "kernel launch failed: %s", cudaGetErrorString(e));
            ++launched;
            continue;
        }
        const bool tall = lean && plan->tall;
        KernelFn fn = pick(d.n_params, kind, kind == kTma ? plan->tring.mode | (lean ? bwm::kTmaLean : 0) | (tall ? bwm::kTmaTall : 0) |
                                                                (tall && plan->tall_nomirror ? bwm::kTmaNoMirror : 0)
                                                          : (plan->ring ? 0 : (int)bwm::kRingLag));
        const int64_t tile = kind == kTma ? bwm::tma_tile(plan->tring.mode) : bwm::kTile;
        const int64_t tiles = (cnt + tile - 1) / tile;
        const int bpm = tall ? plan->bpm_tall : lean ? plan->bpm_tma_lean : plan->blocks_per_sm[kind];
        const int64_t grid = std::min<int64_t>(tiles, (int64_t)plan->sms * bpm);
        const size_t sm = (size_t)(tall ? plan->smem_tall : kind == kTma ? plan->smem_tma : plan->smem);
        if (kind == kTma) {
            int rc = encode_map(&kp.tmap, kp.y, cnt, d.n_obs, ld_y, bwm::kWarpPx, tall ? bwm::kTallRows : bwm::kStageRows);
            if (rc) return rc;
            kp.sched = (tall ? dyn_tall : dyn) ? plan->d_sched : nullptr;
            {
                // long slices (C4: 126 stages, ~170 us each): claim just in time, so the launch's last
                // slices go to warps that are free, not to busy warps holding a pre-claimed one;
                // short slices pre-claim one ahead (the atomic's latency would not hide)
                const int R = tall ? bwm::kTallRows : bwm::kStageRows, n = d.n_hist, N = d.n_obs;
                const int t3 = (n / R) * R;
                const int ts = (n + R - 1) / R + (N - t3 + R - 1) / R;
                static const int jit_env = [] {
                    const char* e = std::getenv("BWM_SCHED_JIT");    // A/B: 0 never, 1 always
                    return e ? std::atoi(e) : -1;
                }();
                kp.sched_jit = jit_env >= 0 ? jit_env : (ts >= 64 ? 1 : 0);
            }
            if (tall) {
                kp.ring_rows = plan->tring_tall.rows;
                kp.tmem_cols = plan->tring_tall.cols;
            }
        }
        fn<<<(unsigned)grid, threads_of(kind, plan->tring.mode), sm, st>>>(kp);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_err((int)e, "kernel launch failed: %s", cudaGetErrorString(e));
        ++launched;
    }
    if (fixup) {
        bwm::KParams kf = k;
        kf.xtd = plan->d_xtd;
        cudaError_t e = bwm::launch_fixup(kf, d.n_params, plan->d_fix_list, plan->d_fix_count, plan->sms, st);
        if (e != cudaSuccess) return set_err((int)e, "fixup launch failed: %s", cudaGetErrorString(e));
        ++launched;
    }
    if (uses_scratch) BWM_CUDA(cudaEventRecord(plan->scratch_ev, st));
    if (out->first_break || out->max_abs_f64 || out->detected) {
        cudaError_t e = bwm::launch_finalize(out->first_idx, out->max_abs, n_pixels, d.n_hist, out->first_break,
                                             out->max_abs_f64, out->detected, st);
        if (e != cudaSuccess) return set_err((int)e, "finalize launch failed: %s", cudaGetErrorString(e));
        ++launched;
    }
    g_launches.fetch_add(launched);
    return BWM_OK;
}

struct PipeNeeds {
    bool beta, mean, mosum, fb, mx64, det;
};

static size_t pipe_bytes(const bwm_dims& d, int64_t chunk, int nbuf, const PipeNeeds& w) {
    size_t per = (size_t)d.n_obs * chunk * 4 + (size_t)chunk * (1 + 4 + 4);
    if (w.beta) per += (size_t)d.n_params * chunk * 4;
    if (w.mean) per += (size_t)chunk * 4;
    if (w.mosum) per += (size_t)(d.n_obs - d.n_hist) * chunk * 4;
    if (w.fb) per += (size_t)chunk * 8;
    if (w.mx64) per += (size_t)chunk * 8;
    if (w.det) per += (size_t)chunk;
    return per * nbuf;
}

static int pipe_ensure(bwm_plan* plan, int64_t chunk, int nbuf, const PipeNeeds& w) {
    HostPipe& hp = plan->pipe;
    const bwm_dims& d = plan->dims;
    const bool ok = hp.chunk == chunk && hp.nbuf == nbuf && (!w.beta || hp.d_beta[0]) && (!w.mean || hp.d_mean[0]) &&
                    (!w.mosum || hp.d_mosum[0]) && (!w.fb || hp.d_fb[0]) && (!w.mx64 || hp.d_mx64[0]) &&
                    (!w.det || hp.d_det[0]);
    if (ok) return BWM_OK;
    pipe_free(hp);
    // allocate into hp; any failure frees everything (no half-built pipe whose signature matches)
    const int rc = [&]() -> int {
    for (int b = 0; b < 2; ++b) {
        if (b < nbuf) {
            BWM_CUDA(cudaMalloc(&hp.d_y[b], (size_t)d.n_obs * chunk * 4));
            BWM_CUDA(cudaMalloc(&hp.d_valid[b], (size_t)chunk));
            BWM_CUDA(cudaMalloc(&hp.d_first[b], (size_t)chunk * 4));
            BWM_CUDA(cudaMalloc(&hp.d_max[b], (size_t)chunk * 4));
            if (w.beta) BWM_CUDA(cudaMalloc(&hp.d_beta[b], (size_t)d.n_params * chunk * 4));
            if (w.mean) BWM_CUDA(cudaMalloc(&hp.d_mean[b], (size_t)chunk * 4));
            if (w.mosum) BWM_CUDA(cudaMalloc(&hp.d_mosum[b], (size_t)(d.n_obs - d.n_hist) * chunk * 4));
            if (w.fb) BWM_CUDA(cudaMalloc(&hp.d_fb[b], (size_t)chunk * 8));
            if (w.mx64) BWM_CUDA(cudaMalloc(&hp.d_mx64[b], (size_t)chunk * 8));
            if (w.det) BWM_CUDA(cudaMalloc(&hp.d_det[b], (size_t)chunk));
        }
        BWM_CUDA(cudaStreamCreateWithFlags(&hp.s_h2d[b], cudaStreamNonBlocking));
        BWM_CUDA(cudaStreamCreateWithFlags(&hp.s_k[b], cudaStreamNonBlocking));
        BWM_CUDA(cudaEventCreateWithFlags(&hp.ev_in[b], cudaEventDisableTiming));
        BWM_CUDA(cudaEventCreate(&hp.ev_k0[b]));
        BWM_CUDA(cudaEventCreate(&hp.ev_k1[b]));
        BWM_CUDA(cudaEventCreateWithFlags(&hp.ev_free[b], cudaEventDisableTiming));
    }
    BWM_CUDA(cudaMalloc(&hp.d_zero, 2 * sizeof(int64_t)));
    return BWM_OK;
    }();
    if (rc != BWM_OK) {
        const std::string msg = g_err;
        pipe_free(hp);
        return set_err(rc, "%s", msg.c_str());
    }
    hp.chunk = chunk;
    hp.nbuf = nbuf;
    hp.bytes = pipe_bytes(d, chunk, nbuf, w);
    return BWM_OK;
}

// The host pipeline behind bwm_monitor_host (source: host memory y_host, row stride ld_y)
// and bwm_monitor_file (source: a time-major payload file; rectangles are read into pinned
// slots by a thread pool while earlier rectangles are copied to HBM).
static int monitor_pipeline(bwm_plan* plan, const float* y_host, int64_t ld_y, const bwm::PayloadFile* file,
                            int io_threads, int64_t n_pixels, int64_t pixel_offset, const bwm_outputs* out,
                            int64_t col_base = 0) {
    if (!plan) return set_err(BWM_E_NULL, "plan is NULL");
    if (!(y_host || file) || !out || !out->valid || !out->zero_sigma_pixel || !(out->first_idx || out->first_break) ||
        !(out->max_abs || out->max_abs_f64))
        return set_err(BWM_E_NULL,
                       "y, valid, zero_sigma_pixel, first_idx|first_break and max_abs|max_abs_f64 are required");
    if (n_pixels < 1) return set_err(BWM_E_DIMS, "stack needs at least one pixel");
    if (ld_y < n_pixels) return set_err(BWM_E_DIMS, "ld_y < n_pixels");
    if ((out->beta || out->mosum) && out->ld_out < n_pixels) return set_err(BWM_E_DIMS, "ld_out < n_pixels");
    if (out->sup_stat) return set_err(BWM_E_PARAMS, "sup_stat is a bwm_monitor (device) output");

    std::lock_guard<std::mutex> lock(plan->mu);
    DeviceRestore guard(plan->device);
    BWM_CUDA(cudaSetDevice(plan->device));
    const bwm_dims& d = plan->dims;
    const int N = d.n_obs, M = d.n_obs - d.n_hist, p = d.n_params;
    const PipeNeeds need{out->beta != nullptr, out->mo_mean != nullptr, out->mosum != nullptr,
                         out->first_break != nullptr, out->max_abs_f64 != nullptr, out->detected != nullptr};

    // Whole-stack mode when it fits (one contiguous H2D at full PCIe rate, one launch);
    // otherwise ~512 MB column chunks, double-buffered.
    size_t free_b = 0, total_b = 0;
    BWM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t avail = free_b + plan->pipe.bytes;
    const int64_t whole = ((n_pixels + bwm::kTile - 1) / bwm::kTile) * bwm::kTile;
    int64_t chunk;
    int nbuf;
    const char* force_chunk = std::getenv("BWM_HOST_CHUNK");       // tests: exercise the chunked pipeline
    const int64_t forced = force_chunk ? ((std::atoll(force_chunk) + bwm::kTile - 1) / bwm::kTile) * bwm::kTile : 0;
    if (forced > 0 && forced < whole) {
        chunk = forced;
        nbuf = 2;
    } else if (pipe_bytes(d, whole, 1, need) + (512ull << 20) <= avail) {
        chunk = whole;
        nbuf = 1;
    } else {
        chunk = (512ll << 20) / (4ll * N);
        chunk = std::max<int64_t>(bwm::kTile, (chunk / bwm::kTile) * bwm::kTile);
        nbuf = 2;
    }
    int rc = pipe_ensure(plan, chunk, nbuf, need);
    if (rc) return rc;
    HostPipe& hp = plan->pipe;

    const int64_t init[2] = {INT64_MAX, INT64_MAX};
    BWM_CUDA(cudaMemcpy(hp.d_zero, init, sizeof init, cudaMemcpyHostToDevice));

    cudaEvent_t t_start = nullptr, t_end = nullptr;
    std::vector<cudaEvent_t> kev;                      // per-chunk kernel timing
    struct EventGuard {                                 // destroys this call's events on every exit
        cudaEvent_t& a;
        cudaEvent_t& b;
        std::vector<cudaEvent_t>& v;
        ~EventGuard() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
            for (auto& e : v) if (e) cudaEventDestroy(e);
        }
    } event_guard{t_start, t_end, kev};
    BWM_CUDA(cudaEventCreate(&t_start));
    BWM_CUDA(cudaEventCreate(&t_end));
    BWM_CUDA(cudaEventRecord(t_start, hp.s_h2d[0]));
    BWM_CUDA(cudaStreamWaitEvent(hp.s_h2d[1], t_start, 0));

    const int64_t n_chunks = (n_pixels + chunk - 1) / chunk;
    std::vector<bwm::Rect> rects;
    std::vector<int64_t> rect_begin(1, 0);
    std::vector<cudaEvent_t> slot_ev;
    std::deque<int64_t> pending;
    int K = 0;
    if (!plan->freader) plan->freader.reset(new bwm::StagedReader());
    bwm::StagedReader& reader = *plan->freader;
    // A pageable host stack (a plain numpy array) is staged the same way as a file: threads
    // memcpy row blocks into pinned slots while earlier blocks are DMA'd (the driver's own
    // pageable path runs at ~11 GB/s on B200 hosts).  Pinned stacks are copied directly.
    bwm::HostSource hsrc{y_host, ld_y};
    bool staged = file != nullptr;
    if (!file) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, y_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();                                  // clear a possible "invalid value"
        const char* st_env = std::getenv("BWM_HOST_STAGED");
        staged = !pinned && !(st_env && std::strcmp(st_env, "0") == 0);
        if (staged && io_threads < 1)
            io_threads = (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    }
    if (staged) {
        const char* slot_env = std::getenv("BWM_IO_SLOT_BYTES");     // tests: small slots split rows
        const int64_t slot_bytes = slot_env ? std::max<int64_t>(256, std::atoll(slot_env)) : (32ll << 20);
        for (int64_t c = 0; c < n_chunks; ++c) {
            // file columns: this call's pixels start at column col_base of the payload
            bwm::plan_rects(N, col_base + c * chunk, col_base + std::min(n_pixels, (c + 1) * chunk), c, slot_bytes,
                            &rects);
            rect_begin.push_back((int64_t)rects.size());
        }
        const int threads = std::max(1, io_threads);
        K = std::max(4, std::min(threads + 4, 40));
        std::string err;
        if (int e = reader.ensure(K, slot_bytes, &err)) return set_err(e, "%s", err.c_str());
        slot_ev.resize((size_t)K, nullptr);
        for (auto& ev : slot_ev) BWM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        if (file)
            reader.start(file, &rects, threads);
        else
            reader.start(&hsrc, &rects, threads);
    }
    struct ReaderGuard {        // joins the reader threads and frees the slot events on every exit
        bwm::StagedReader& r;
        std::vector<cudaEvent_t>& ev;
        ~ReaderGuard() {
            r.stop();
            for (auto& e : ev) if (e) cudaEventDestroy(e);
        }
    } reader_guard{reader, slot_ev};
    int64_t h2d = 0, d2h = 0;
    // result maps: pinned destinations get the D2H directly, pageable ones through the landing zone
    struct MapDst {
        void* dst;
        int elem;
        size_t off;       // offset of this map in the landing zone (pageable destinations)
        bool pageable;
    };
    auto is_pageable = [](const void* q) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, q) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        return !pinned;
    };
    MapDst maps[7] = {{out->valid, 1, 0, false},       {out->first_idx, 4, 0, false}, {out->max_abs, 4, 0, false},
                      {out->first_break, 8, 0, false}, {out->max_abs_f64, 8, 0, false}, {out->detected, 1, 0, false},
                      {out->mo_mean, 4, 0, false}};
    size_t stage_need = 0;
    for (auto& m : maps) {
        if (!m.dst) continue;
        m.pageable = is_pageable(m.dst);
        if (m.pageable) {
            m.off = stage_need;
            stage_need += (((size_t)n_pixels * m.elem) + 255) & ~(size_t)255;
        }
    }
    if (stage_need > hp.h_stage_bytes) {
        if (hp.h_stage) cudaFreeHost(hp.h_stage);
        hp.h_stage = nullptr;
        hp.h_stage_bytes = 0;
        BWM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hp.h_stage), stage_need, cudaHostAllocPortable));
        hp.h_stage_bytes = stage_need;
    }
    kev.assign((size_t)(2 * n_chunks), nullptr);
    for (auto& ev : kev) BWM_CUDA(cudaEventCreate(&ev));
    for (int64_t c = 0; c < n_chunks; ++c) {
        const int b = nbuf == 1 ? 0 : (int)(c & 1);
        const int64_t p0 = c * chunk;
        const int64_t w = std::min(chunk, n_pixels - p0);
        cudaStream_t sh = hp.s_h2d[b], s = hp.s_k[b];
        // buffer b is free once chunk c-nbuf finished its D2H
        if (c >= nbuf) BWM_CUDA(cudaStreamWaitEvent(sh, hp.ev_free[b], 0));
        if (staged) {
            // rectangles of this chunk, alternating over the two copy engines in whole-stack mode
            for (int64_t g = rect_begin[(size_t)c]; g < rect_begin[(size_t)c + 1]; ++g) {
                const bwm::Rect& r = rects[(size_t)g];
                const float* src = reader.wait(g);
                if (!src) return set_err(BWM_E_IO, "%s", reader.error().c_str());
                cudaStream_t cs = nbuf == 1 ? hp.s_h2d[g & 1] : sh;
                const int64_t rw = r.c1 - r.c0;
                BWM_CUDA(cudaMemcpy2DAsync(hp.d_y[b] + r.r0 * w + (r.c0 - col_base - p0), (size_t)w * 4, src, (size_t)rw * 4,
                                           (size_t)rw * 4, (size_t)(r.r1 - r.r0), cudaMemcpyHostToDevice, cs));
                BWM_CUDA(cudaEventRecord(slot_ev[(size_t)(g % K)], cs));
                pending.push_back(g);
                while ((int)pending.size() > K / 2) {           // refill the oldest slots
                    const int64_t o = pending.front();
                    BWM_CUDA(cudaEventSynchronize(slot_ev[(size_t)(o % K)]));
                    reader.release(o);
                    pending.pop_front();
                }
            }
            if (nbuf == 1) {
                BWM_CUDA(cudaEventRecord(hp.ev_in[1], hp.s_h2d[1]));
                BWM_CUDA(cudaStreamWaitEvent(s, hp.ev_in[1], 0));
            }
        } else if (ld_y == w) {
            // contiguous block: split in two halves on both copy streams (one engine each)
            const size_t total = (size_t)w * 4 * N, half = (total / 2) & ~(size_t)255;
            BWM_CUDA(cudaMemcpyAsync(hp.d_y[b], y_host + p0, half, cudaMemcpyHostToDevice, sh));
            if (nbuf == 1) {
                BWM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(hp.d_y[b]) + half,
                                         reinterpret_cast<const char*>(y_host + p0) + half, total - half,
                                         cudaMemcpyHostToDevice, hp.s_h2d[1]));
                BWM_CUDA(cudaEventRecord(hp.ev_in[1], hp.s_h2d[1]));
                BWM_CUDA(cudaStreamWaitEvent(s, hp.ev_in[1], 0));
            } else {
                BWM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(hp.d_y[b]) + half,
                                         reinterpret_cast<const char*>(y_host + p0) + half, total - half,
                                         cudaMemcpyHostToDevice, sh));
            }
        } else {
            BWM_CUDA(cudaMemcpy2DAsync(hp.d_y[b], (size_t)w * 4, y_host + p0, (size_t)ld_y * 4, (size_t)w * 4,
                                       (size_t)N, cudaMemcpyHostToDevice, sh));
        }
        h2d += (int64_t)w * 4 * N;
        BWM_CUDA(cudaEventRecord(hp.ev_in[b], sh));
        BWM_CUDA(cudaStreamWaitEvent(s, hp.ev_in[b], 0));
        bwm_outputs o{};
        o.valid = hp.d_valid[b];
        o.first_idx = hp.d_first[b];
        o.max_abs = hp.d_max[b];
        o.beta = out->beta ? hp.d_beta[b] : nullptr;
        o.mo_mean = out->mo_mean ? hp.d_mean[b] : nullptr;
        o.mosum = out->mosum ? hp.d_mosum[b] : nullptr;
        o.ld_out = w;
        o.zero_sigma_pixel = hp.d_zero + b;
        o.first_break = out->first_break ? hp.d_fb[b] : nullptr;
        o.max_abs_f64 = out->max_abs_f64 ? hp.d_mx64[b] : nullptr;
        o.detected = out->detected ? hp.d_det[b] : nullptr;
        BWM_CUDA(cudaEventRecord(kev[2 * c], s));
        rc = bwm_monitor(plan, hp.d_y[b], w, w, pixel_offset + p0, &o, s);
        if (rc) return rc;
        BWM_CUDA(cudaEventRecord(kev[2 * c + 1], s));
        auto d2h_map = [&](int mi, const void* src) -> int {
            const MapDst& m = maps[mi];
            if (!m.dst) return BWM_OK;
            const size_t bytes = (size_t)w * m.elem;
            char* dst = m.pageable ? hp.h_stage + m.off + (size_t)p0 * m.elem
                                   : static_cast<char*>(m.dst) + (size_t)p0 * m.elem;
            BWM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
            d2h += (int64_t)bytes;
            return BWM_OK;
        };
        const void* srcs[7] = {hp.d_valid[b], hp.d_first[b], hp.d_max[b], hp.d_fb[b], hp.d_mx64[b], hp.d_det[b],
                               hp.d_mean[b]};
        for (int mi = 0; mi < 7; ++mi)
            if ((rc = d2h_map(mi, srcs[mi]))) return rc;
        if (out->beta) {
            BWM_CUDA(cudaMemcpy2DAsync(out->beta + p0, (size_t)out->ld_out * 4, hp.d_beta[b], (size_t)w * 4,
                                       (size_t)w * 4, (size_t)p, cudaMemcpyDeviceToHost, s));
            d2h += w * 4 * p;
        }
        if (out->mosum) {
            BWM_CUDA(cudaMemcpy2DAsync(out->mosum + p0, (size_t)out->ld_out * 4, hp.d_mosum[b], (size_t)w * 4,
                                       (size_t)w * 4, (size_t)M, cudaMemcpyDeviceToHost, s));
            d2h += w * 4 * M;
        }
        BWM_CUDA(cudaEventRecord(hp.ev_free[b], s));
    }
    // while the GPU transfers and computes: touch the pages of the pageable map destinations
    // (fresh numpy arrays fault on first write), so the copy-out below runs at memory speed
    {
        std::vector<std::pair<char*, size_t>> jobs;
        const size_t piece = 8u << 20;
        for (const auto& m : maps) {
            if (!m.dst || !m.pageable) continue;
            const size_t total = (size_t)n_pixels * m.elem;
            for (size_t a = 0; a < total; a += piece)
                jobs.emplace_back(static_cast<char*>(m.dst) + a, std::min(piece, total - a));
        }
        const int nt = (int)std::min<size_t>(jobs.size(), std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
        std::atomic<size_t> next{0};
        auto work = [&]() {
            for (size_t j; (j = next.fetch_add(1)) < jobs.size();) std::memset(jobs[j].first, 0, jobs[j].second);
        };
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(work);
        if (nt > 0) work();
        for (auto& t : th) t.join();
    }
    double kernel_ms = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        BWM_CUDA(cudaEventSynchronize(kev[2 * c + 1]));
        float ms = 0;
        BWM_CUDA(cudaEventElapsedTime(&ms, kev[2 * c], kev[2 * c + 1]));
        kernel_ms += ms;
    }
    for (int64_t g : pending) {
        BWM_CUDA(cudaEventSynchronize(slot_ev[(size_t)(g % K)]));
        reader.release(g);
    }
    for (int b = 0; b < 2; ++b) {
        BWM_CUDA(cudaStreamSynchronize(hp.s_k[b]));
        BWM_CUDA(cudaStreamSynchronize(hp.s_h2d[b]));
    }
    {
        // landing zone -> pageable destinations, split over threads
        std::vector<std::pair<char*, const char*>> jobs;
        std::vector<size_t> lens;
        const size_t piece = 16u << 20;
        for (const auto& m : maps) {
            if (!m.dst || !m.pageable) continue;
            const size_t total = (size_t)n_pixels * m.elem;
            for (size_t a = 0; a < total; a += piece) {
                jobs.emplace_back(static_cast<char*>(m.dst) + a, hp.h_stage + m.off + a);
                lens.push_back(std::min(piece, total - a));
            }
        }
        const int nt = (int)std::min<size_t>(jobs.size(), std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
        std::atomic<size_t> next{0};
        auto work = [&]() {
            for (size_t j; (j = next.fetch_add(1)) < jobs.size();) std::memcpy(jobs[j].first, jobs[j].second, lens[j]);
        };
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
    }
    int64_t z[2];
    BWM_CUDA(cudaMemcpy(z, hp.d_zero, sizeof z, cudaMemcpyDeviceToHost));
    d2h += sizeof z;
    const int64_t zmin = std::min(z[0], z[1]);
    if (zmin < *out->zero_sigma_pixel) *out->zero_sigma_pixel = zmin;
    BWM_CUDA(cudaEventRecord(t_end, hp.s_k[0]));
    BWM_CUDA(cudaEventSynchronize(t_end));
    float total = 0;
    cudaEventElapsedTime(&total, t_start, t_end);
    hp.last_kernel_ms = kernel_ms;
    hp.last_total_ms = total;
    hp.last_h2d = h2d;
    hp.last_d2h = d2h;
    return BWM_OK;
}

int bwm_monitor_host(bwm_plan* plan, const float* y_host, int64_t ld_y, int64_t n_pixels,
                     int64_t pixel_offset, const bwm_outputs* out_host) {
    return monitor_pipeline(plan, y_host, ld_y, nullptr, 0, n_pixels, pixel_offset, out_host);
}

int bwm_monitor_file_range(bwm_plan* plan, const char* path, int64_t payload_offset, int64_t file_pixels,
                           int64_t first_pixel, int64_t n_pixels, int io_threads, const bwm_outputs* out_host) {
    if (!plan) return set_err(BWM_E_NULL, "plan is NULL");
    if (!path) return set_err(BWM_E_NULL, "path is NULL");
    if (n_pixels < 1) return set_err(BWM_E_DIMS, "stack needs at least one pixel");
    if (first_pixel < 0 || first_pixel + n_pixels > file_pixels)
        return set_err(BWM_E_DIMS, "pixel range [%lld, %lld) outside the file's %lld pixels", (long long)first_pixel,
                       (long long)(first_pixel + n_pixels), (long long)file_pixels);
    bwm::PayloadFile f;
    std::string err;
    if (int rc = f.open(path, payload_offset, plan->dims.n_obs, file_pixels, &err)) return set_err(rc, "%s", err.c_str());
    if (io_threads < 1) io_threads = (int)std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
    return monitor_pipeline(plan, nullptr, n_pixels, &f, io_threads, n_pixels, first_pixel, out_host, first_pixel);
}

int bwm_monitor_file(bwm_plan* plan, const char* path, int64_t payload_offset, int64_t n_pixels,
                     int io_threads, const bwm_outputs* out_host) {
    return bwm_monitor_file_range(plan, path, payload_offset, n_pixels, 0, n_pixels, io_threads, out_host);
}

int bwm_plan_info(const bwm_plan* plan, bwm_plan_info_t* info) {
    if (!plan || !info) return set_err(BWM_E_NULL, "plan/info is NULL");
    info->ring_mode = plan->tring.mode;
    info->ring_rows = plan->tring.rows;
    info->tmem_cols = plan->tring.cols;
    info->smem_tma = plan->smem_tma;
    info->smem_ldg = plan->smem;
    info->ctas_per_sm_tma = plan->blocks_per_sm[kTma];
    info->ctas_per_sm_ldg = plan->blocks_per_sm[kLdgFast];
    info->occupancy_tma = plan->occ_raw[kTma];
    info->sms = plan->sms;
    info->force_ldg = plan->force_ldg ? 1 : 0;
    info->nan_mode = plan->dims.nan_mode;
    info->masked_global = plan->mbig ? 1 : 0;
    info->ctas_per_sm_masked = plan->bpm_masked;
    info->smem_masked = plan->smem_masked;
    info->const_bound = plan->const_bound ? 1 : 0;
    info->ctas_per_sm_tma_lean = plan->bpm_tma_lean;
    info->precise = plan->precise ? 1 : 0;
    info->mma = plan->use_mma ? 1 : 0;
    info->smem_mma = plan->smem_mma;
    info->dyn_sched = plan->d_sched ? 1 : 0;
    info->tall_stages = plan->tall ? (plan->tall_nomirror ? 2 : 1) : 0;
    return BWM_OK;
}

int bwm_last_host_stats(const bwm_plan* plan, double* kernel_ms, double* total_ms, int64_t* h2d_bytes,
                        int64_t* d2h_bytes) {
    if (!plan) return set_err(BWM_E_NULL, "plan is NULL");
    if (kernel_ms) *kernel_ms = plan->pipe.last_kernel_ms;
    if (total_ms) *total_ms = plan->pipe.last_total_ms;
    if (h2d_bytes) *h2d_bytes = plan->pipe.last_h2d;
    if (d2h_bytes) *d2h_bytes = plan->pipe.last_d2h;
    return BWM_OK;
}

}  // extern "C"
