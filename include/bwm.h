/*
 * bwm.h — C ABI of the B200-native BFAST-monitor hot path (libbwm.so).
 *
 * This is the drop-in boundary for the reference's fused batch backend:
 *   breakwatch.engine._fused_phases   (reference pkg/src/breakwatch/engine.py:322-411)
 * plus the two compiled kernels it calls,
 *   breakwatch._kernels.mosum_block   (reference pkg/src/breakwatch/_kernels.py:21-34)
 *   breakwatch._kernels.detect_block  (reference pkg/src/breakwatch/_kernels.py:37-48)
 * and the gap-fill ingest it runs first,
 *   breakwatch.engine._ingest_block   (reference pkg/src/breakwatch/engine.py:305-319).
 *
 * One call = one fused pass per pixel: forward/back gap fill -> beta = M . y_hist
 * -> residuals -> sigma -> sliding MOSUM -> strict boundary test -> first break,
 * max |MO| (and optionally beta, the MOSUM mean, the full MOSUM matrix).
 *
 * Conventions (mirroring the reference kernel seam, _kernels.py:21,37):
 *   - all arrays are caller-allocated; the hot call (bwm_monitor) never allocates;
 *   - data is time-major: y[t * ld_y + pixel], float32, NaN/+-Inf = missing;
 *   - outputs are per pixel, written at out[pixel] (beta/mosum: out[row * ld_out + pixel]);
 *   - return 0 on success, a negative BWM_E* code for invalid arguments, or a positive
 *     cudaError_t value for CUDA failures; bwm_last_error() holds the message (per thread).
 *
 * The constant tables (design, boundary) are host setup in float64 — the reference's
 * build_design_matrix / boundary_values (model.py:90-110, mosum.py:68-79) — handed over once
 * through bwm_plan_create.  The library solves the history least squares itself: a float64
 * QR of the history design gives an orthonormal basis Q (the role of fit_mapping's
 * M = (X_h X_h^T)^-1 X_h, model.py:118-152), so that beta_Q = Q^T y_h and the residual sum of
 * squares is ||y_h||^2 - ||beta_Q||^2 without a second sweep over the history.
 */
#ifndef BWM_H
#define BWM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BWM_ABI_VERSION 8

/* error codes (negative); positive returns are cudaError_t values */
#define BWM_OK 0
#define BWM_E_NULL (-1)        /* required pointer is NULL                      */
#define BWM_E_DIMS (-2)        /* inconsistent dimensions (n >= N, h > n, ...)  */
#define BWM_E_PARAMS (-3)      /* n_params outside the compiled set {4,...,18}  */
#define BWM_E_SMEM (-4)        /* tables + MOSUM ring exceed shared memory      */
#define BWM_E_DEVICE (-5)      /* plan used on a different device               */
#define BWM_E_ZERO_SIGMA (-6)  /* not returned by bwm_monitor; see zero_sigma   */
#define BWM_E_IO (-7)          /* file cannot be opened / read / written        */
#define BWM_E_FORMAT (-8)      /* file shorter than the payload it declares     */

/* Geometry shared by every pixel of a batch (reference MonitorConfig, engine.py:102-134). */
typedef struct bwm_dims {
    int32_t n_obs;      /* N : observations per series (rows of the stack)          */
    int32_t n_hist;     /* n : stable history length, p < n < N                     */
    int32_t bandwidth;  /* h : MOSUM window (integer count), 1 <= h <= n            */
    int32_t n_params;   /* p = 2 + 2k : intercept, trend, k sin/cos pairs           */
    int32_t nan_mode;   /* BWM_NAN_FILL (reference behaviour) or BWM_NAN_MASK        */
} bwm_dims;

/*
 * Missing-value handling.
 *   BWM_NAN_FILL: forward/back fill before fitting — the reference (engine.py:305-319).
 *   BWM_NAN_MASK: each pixel is fitted on its valid history dates only and monitored over
 *     its compacted valid series with n_v valid history dates, bandwidth h_v = floor(h n_v / n)
 *     and boundary lambda sqrt(log_plus((n_v+1+j)/n_v)), lambda = bound[0]; first_idx is the
 *     1-based offset (from n) of the ORIGINAL date that completes the first crossing window.
 *     Pixels with n_v <= p, h_v < 1, no valid monitoring date or a singular valid design are
 *     invalid.  With no missing values both modes give the same result.  (
 *     the reference has no such mode: oracle/bfast_oracle.py:monitor_masked defines it.)
 */
#define BWM_NAN_FILL 0
#define BWM_NAN_MASK 1

/*
 * Host-side float64 constants for one batch geometry.  The kernel runs in a
 * re-centred but equivalent basis: the trend regressor t is replaced by
 * (t - trend_center) / trend_scale, which leaves fitted values, residuals and
 * MOSUM unchanged in exact arithmetic and keeps the float32 contraction well
 * conditioned.  Beta is reported back in the reference's raw basis.
 */
typedef struct bwm_tables {
    const double* design;    /* [p][N]  X'  rows: 1, (t-tc)/ts, sin(2pi j t/f), cos(...)    */
    const double* bound;     /* [N-n]   crit * sqrt(log_plus((n+1+j)/n))  (mosum.py:68-79)  */
    double trend_center;     /* tc */
    double trend_scale;      /* ts */
} bwm_tables;

/* Per-pixel outputs.  Required: valid, first_idx, max_abs.  Optional: NULL to skip. */
typedef struct bwm_outputs {
    uint8_t* valid;          /* [P]  1 if the series has a finite sample (engine.py:308)          */
    int32_t* first_idx;      /* [P]  0 = no break, else 1-based offset into the monitor period    */
    float* max_abs;          /* [P]  max_j |MO_j|                                                  */
    float* beta;             /* [p][ld_out] or NULL: history coefficients, raw basis (model.py:90) */
    float* mo_mean;          /* [P] or NULL: mean_j MO_j                                           */
    float* mosum;            /* [N-n][ld_out] or NULL: the MOSUM process (keep_mosum); mask mode:  */
                             /*   row t-n holds the window ending at date t, NaN on missing dates */
    int64_t ld_out;          /* leading dimension of beta / mosum (>= P)                           */
    /* lowest global pixel index whose history fits exactly (sigma == 0); caller initialises
       to INT64_MAX (device pointer for bwm_monitor, host pointer for bwm_monitor_host).
       Mirrors ZeroResidualError (engine.py:373-378). */
    int64_t* zero_sigma_pixel;
    /* Optional maps in the reference BreakMap dtypes (engine.py:147-150, 297-299), produced on
       the device so the host does no conversion pass: NULL to skip. */
    int64_t* first_break;    /* [P]  n + first_idx, 0 = no break (1-based observation number)     */
    double* max_abs_f64;     /* [P]  max_abs widened to float64                                    */
    uint8_t* detected;       /* [P]  first_break > 0                                               */
    /* Optional: the Monte Carlo statistic of critical_value (reference mosum.py:166-227),
       sup_j |MO_j| / bound_j per pixel (with a unit-lambda plan: sup_j |MO_j| / sqrt(log_plus(
       (n+1+j)/n))), so lambda calibration needs no MOSUM matrix.  Fill mode only.  NULL to skip. */
    float* sup_stat;         /* [P] */
} bwm_outputs;

typedef struct bwm_plan bwm_plan;

/* Build the device-resident constant tables on `device` (cudaSetDevice is restored). */
int bwm_plan_create(const bwm_dims* dims, const bwm_tables* tables, int device,
                    bwm_plan** out_plan);
void bwm_plan_destroy(bwm_plan* plan);

/*
 * Hot call, device pointers, asynchronous on `stream` (a cudaStream_t; NULL = legacy).
 *   y        : device float32 [N][ld_y], pixel p of this shard at column p
 *   n_pixels : pixels in this shard (P)
 *   pixel_offset : global index of this shard's pixel 0 (for zero_sigma_pixel)
 * No synchronisation.  Allocation only on the first call of a plan (and when a larger call
 * grows it): the device list of the float64 fixup, at most 4M entries (32 MB) — valid pixels
 * whose ||y - c||^2 / RSS exceeds 300 (BWM_FIX_RATIO) are recomputed in float64 by a second
 * launch; plans whose monitoring horizon extrapolates the trend past |(t - tc)/ts| = 8 run
 * float64 kernels throughout (BWM_PRECISE).  Re-entrant across streams, host threads and
 * devices: calls that use the plan's device scratch (the fixup list; the TMA kernel's dynamic
 * slice-scheduler counters, which its last warp resets; the masked-mode rings of large
 * geometries) are ordered on the device through a plan-owned event, the rest overlap.
 * zero_sigma_pixel accumulates (atomicMin) across calls until the caller re-initialises it
 * (bwm_zero_sigma_init).
 */
int bwm_monitor(const bwm_plan* plan, const float* y, int64_t ld_y, int64_t n_pixels,
                int64_t pixel_offset, const bwm_outputs* out, void* stream);

/*
 * End-to-end call with HOST buffers (the reference-facing path: a numpy stack in,
 * numpy maps out).  When the stack fits in device memory it is copied as one contiguous
 * block (full PCIe rate) and monitored by one launch; otherwise pixels are processed in
 * column chunks with the H2D of chunk i+1 overlapping the kernel of chunk i and the D2H
 * of chunk i-1 on separate streams.  y_host may be pageable or pinned (pinned is faster).
 * Blocks until done.  Outputs are host pointers with the same layout as bwm_outputs;
 * first_idx / max_abs may be NULL here when first_break / max_abs_f64 are given.  Pageable
 * (unregistered) stacks are staged through pinned slots by memcpy threads; pageable result
 * maps receive their D2H through a plan-owned pinned landing zone.
 */
int bwm_monitor_host(bwm_plan* plan, const float* y_host, int64_t ld_y, int64_t n_pixels,
                     int64_t pixel_offset, const bwm_outputs* out_host);

/*
 * End-to-end call from a BTS1 stack FILE (reference dataio.read_stack, dataio.py:79-115,
 * followed by monitor_batch): the time-major float32 payload of n_pixels columns and
 * dims.n_obs rows starts at byte payload_offset (after the header and optional axis, which
 * the caller parsed — the plan's time axis comes from it).  io_threads threads pread row
 * blocks of the payload into pinned staging slots while earlier blocks are copied to HBM, so
 * the file read, the PCIe transfer and (for stacks larger than device memory) the kernel
 * overlap.  io_threads < 1: min(32, hardware threads).  Outputs as for bwm_monitor_host.
 * Returns BWM_E_IO / BWM_E_FORMAT for unreadable or truncated files.
 */
int bwm_monitor_file(bwm_plan* plan, const char* path, int64_t payload_offset, int64_t n_pixels,
                     int io_threads, const bwm_outputs* out_host);

/*
 * One rank's share of a BTS1 file: pixels [first_pixel, first_pixel + n_pixels) of a payload
 * with file_pixels columns (each row block is read as n_pixels-wide pieces).  Outputs are for
 * those pixels only (index 0 = first_pixel); zero_sigma_pixel reports file pixel indices.
 * bwm_monitor_file is the whole-file case.
 */
int bwm_monitor_file_range(bwm_plan* plan, const char* path, int64_t payload_offset, int64_t file_pixels,
                           int64_t first_pixel, int64_t n_pixels, int io_threads, const bwm_outputs* out_host);

/*
 * Parallel read of a time-major float32 payload [n_obs][n_pixels] at byte `offset` of a file
 * into dst (any host memory; pinned makes the later H2D faster).  The read half of
 * dataio.read_stack (dataio.py:110-114).  threads < 1: all hardware threads.
 */
int bwm_read_payload(const char* path, int64_t offset, int64_t n_obs, int64_t n_pixels, float* dst,
                     int threads);

/*
 * Break-map CSV (reference dataio.write_break_map, dataio.py:168-182), byte-identical:
 * header "pixel,valid,detected,first_break,max_abs_mo", one row per pixel in order,
 * first_break empty when 0, max_abs_mo at 9 significant digits.  Rows are formatted by
 * `threads` threads (< 1: all).  Returns the row count or a negative BWM_E_* code.
 */
int64_t bwm_write_break_map(const char* path, int64_t n_pixels, const uint8_t* valid, const uint8_t* detected,
                            const int64_t* first_break, const double* max_abs_mo, int threads);

/* Kernel time (ms) of the last bwm_monitor_host call, summed over chunks; and its
   H2D/D2H byte counts.  For PhaseTimings. */
int bwm_last_host_stats(const bwm_plan* plan, double* kernel_ms, double* total_ms,
                        int64_t* h2d_bytes, int64_t* d2h_bytes);

/* Launch configuration a plan chose (diagnostics; bench.py reports it). */
typedef struct bwm_plan_info_t {
    int32_t ring_mode;        /* TMA kernel residual ring: 0 smem, 1 tensor memory, 2 lagging cursor */
    int32_t ring_rows;        /* TMEM ring rows L (0 unless ring_mode == 1)                          */
    int32_t tmem_cols;        /* TMEM columns allocated per CTA                                      */
    int32_t sms;              /* streaming multiprocessors of the device                             */
    int64_t smem_tma;         /* dynamic shared memory per CTA, TMA kernel (0: not usable)           */
    int64_t smem_ldg;         /* dynamic shared memory per CTA, LDG kernels                          */
    int32_t ctas_per_sm_tma;  /* persistent CTAs per SM, TMA kernel                                  */
    int32_t ctas_per_sm_ldg;  /* persistent CTAs per SM, LDG kernel                                  */
    int32_t occupancy_tma;    /* occupancy-API result for the TMA kernel                             */
    int32_t force_ldg;        /* BWM_KERNEL=ldg was set at plan creation                             */
    int32_t nan_mode;         /* BWM_NAN_FILL / BWM_NAN_MASK                                         */
    int32_t masked_global;    /* mask mode: x x^T table and residual rings in global memory          */
    int32_t ctas_per_sm_masked;
    int64_t smem_masked;      /* dynamic shared memory per CTA, masked kernel                        */
    int32_t const_bound;      /* boundary constant over the monitoring period (LEAN TMA variant)     */
    int32_t ctas_per_sm_tma_lean; /* persistent CTAs per SM, LEAN TMA variant                        */
    int32_t precise;          /* long horizon: float64 fitted values (LDG kernels); BWM_PRECISE=0/1   */
    int32_t mma;              /* lagging-cursor geometry: fitted values on the tensor cores (BWM_MMA)  */
    int64_t smem_mma;         /* dynamic shared memory per CTA of that kernel                         */
    int32_t dyn_sched;        /* TMA kernel: dynamic per-warp slice scheduler (BWM_DYN=0: static)  (ABI 8) */
    int32_t tall_stages;      /* LEAN TMEM-ring launches use 16-date stages: 1 (2: ring without mirror rows); BWM_TALL=0: off (ABI 8) */
} bwm_plan_info_t;

int bwm_plan_info(const bwm_plan* plan, bwm_plan_info_t* info);

/* Stream-ordered reset of a device zero_sigma_pixel slot to INT64_MAX (two cudaMemsetAsync,
   no kernel, no allocation): lets a caller reuse one slot across bwm_monitor calls. */
int bwm_zero_sigma_init(int64_t* zero_sigma_pixel_device, void* stream);

/*
 * The null-hypothesis draws of critical_value on the device (reference mosum.py:195-198:
 * replication r draws np.random.Generator(np.random.Philox(key=seed, counter=r << 128))
 * .standard_normal(n_obs)).  numpy's Philox4x64-10 + ziggurat restated bit for bit; the draws of
 * replications [rep0, rep0 + reps) are written as float32 to out[t * ld + (r - rep0)]
 * (time-major, one column per replication: a stack bwm_monitor takes directly).  seed = seed_lo +
 * 2^64 seed_hi.  Asynchronous on `stream`.
 */
int bwm_null_draws(uint64_t seed_lo, uint64_t seed_hi, int64_t rep0, int64_t reps, int32_t n_obs,
                   float* out, int64_t ld, void* stream);

/* Number of bwm kernel launches issued by this process so far (all plans). */
int64_t bwm_launch_count(void);

/* Shared memory (bytes) a launch with these dims needs; <0 if unsupported. */
int64_t bwm_smem_bytes(const bwm_dims* dims);

const char* bwm_last_error(void);
int bwm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BWM_H */
