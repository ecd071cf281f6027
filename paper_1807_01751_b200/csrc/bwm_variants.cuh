// bwm_variants.cuh — kernel variant tables (one translation unit per n_params).
#pragma once
#include "bwm_kernel_ldg.cuh"
#include "bwm_kernel_tma.cuh"
#include "bwm_kernel_masked.cuh"
#include "bwm_kernel_mma.cuh"

namespace bwm {
enum Kind { kLdgFast = 0, kLdgSafe = 1, kTma = 2 };
using KernelFn = void (*)(const KParams);
constexpr int kTmaLean = 0x10;   // pick(): OR into the TMA ring mode for the LEAN variant
constexpr int kTmaTall = 0x20;   // pick(): with kRingTmem | kTmaLean, the 16-date-stage (TALL) variant
constexpr int kTmaNoMirror = 0x40;   // with kTmaTall: the ring without mirror rows
}  // namespace bwm

// Defines bwm::KernelFn bwm_pick_p<NP>(int kind, int mode) in the including TU.
// mode: bwm::RingMode of the TMA kernel (kRingTmem / kRingLag; < 0 = none), | kTmaLean for the
// LEAN variant (no MOSUM matrix/mean, constant boundary); the LDG kernels
// have a shared-memory ring (any mode but kRingLag) or the lagging cursor.
#define BWM_DEFINE_PICK(NP)                                                                      \
    bwm::KernelFn bwm_pick_p##NP(int kind, int mode) {                                           \
        const bool ring = mode != bwm::kRingLag;                                                 \
        switch (kind) {                                                                          \
            case bwm::kLdgFast:                                                                  \
                return ring ? bwm::monitor_kernel_ldg<NP, false, true> : bwm::monitor_kernel_ldg<NP, false, false>; \
            case bwm::kLdgSafe:                                                                  \
                return ring ? bwm::monitor_kernel_ldg<NP, true, true> : bwm::monitor_kernel_ldg<NP, true, false>;   \
            default:                                                                             \
                if ((mode & bwm::kTmaTall) && (mode & 0xF) == bwm::kRingTmem)                    \
                    return (mode & bwm::kTmaNoMirror)                                            \
                               ? bwm::monitor_kernel_tma<NP, bwm::kRingTmem, true, bwm::kTallRows, false> \
                               : bwm::monitor_kernel_tma<NP, bwm::kRingTmem, true, bwm::kTallRows, true>; \
                if (mode & bwm::kTmaLean)                                                        \
                    return (mode & 0xF) == bwm::kRingTmem  ? bwm::monitor_kernel_tma<NP, bwm::kRingTmem, true>  \
                           : (mode & 0xF) == bwm::kRingLagT ? bwm::monitor_kernel_tma<NP, bwm::kRingLagT, true> \
                                                           : bwm::monitor_kernel_tma<NP, bwm::kRingLag, true>;  \
                return (mode & 0xF) == bwm::kRingTmem  ? bwm::monitor_kernel_tma<NP, bwm::kRingTmem, false>      \
                       : (mode & 0xF) == bwm::kRingLagT ? bwm::monitor_kernel_tma<NP, bwm::kRingLagT, false>     \
                                                       : bwm::monitor_kernel_tma<NP, bwm::kRingLag, false>;      \
        }                                                                                        \
    }

// Defines bwm::KernelFn bwm_pick_mma_p<NP>(int lean): the lagging-cursor kernel with the
// fitted values on the tensor cores (bwm_kernel_mma.cuh).
#if BWM_STAGE_ROWS == 8
#define BWM_DEFINE_PICK_MMA(NP)                                                                  \
    bwm::KernelFn bwm_pick_mma_p##NP(int lean) {                                                 \
        return lean ? bwm::monitor_kernel_mma<NP, true> : bwm::monitor_kernel_mma<NP, false>;   \
    }
#else   // experimental 16-date stages: no tensor-core variant
#define BWM_DEFINE_PICK_MMA(NP) \
    bwm::KernelFn bwm_pick_mma_p##NP(int) { return nullptr; }
#endif

// Defines bwm::KernelFn bwm_pick_masked_p<NP>(int big, int keep): the masked-NaN kernel with
// its residual rings in shared memory (big = 0) or global memory (big = 1), writing the MOSUM
// matrix (keep = 1) or not.
#define BWM_DEFINE_PICK_MASKED(NP)                                                               \
    bwm::KernelFn bwm_pick_masked_p##NP(int big, int keep) {                                     \
        if (keep) return big ? bwm::monitor_kernel_masked<NP, true, true> : bwm::monitor_kernel_masked<NP, false, true>; \
        return big ? bwm::monitor_kernel_masked<NP, true, false> : bwm::monitor_kernel_masked<NP, false, false>;         \
    }
