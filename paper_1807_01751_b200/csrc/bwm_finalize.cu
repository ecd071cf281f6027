// bwm_finalize.cu — result maps in the reference BreakMap dtypes, produced on the device.
//
// The reference assembles first_break = where(first_idx > 0, n + first_idx, 0) as int64 and
// keeps max_abs_mo as float64 (engine.py:147-150, 297-299).  Doing that widening on the host
// for a 4096^2 stack costs ~0.4 s of numpy passes; here it is one memory-bound pass over
// 9 B/px in, 17 B/px out, before the D2H copy.
#include <cuda_runtime.h>
#include <stdint.h>

namespace bwm {

__global__ void __launch_bounds__(256) finalize_kernel(const int32_t* __restrict__ first_idx,
                                                       const float* __restrict__ max_abs, int64_t P, int n,
                                                       int64_t* __restrict__ first_break, double* __restrict__ mx64,
                                                       uint8_t* __restrict__ detected) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = first_idx[i];
        if (first_break) first_break[i] = f > 0 ? (int64_t)n + f : 0;
        if (detected) detected[i] = f > 0;
        if (mx64) mx64[i] = (double)max_abs[i];
    }
}

cudaError_t launch_finalize(const int32_t* first_idx, const float* max_abs, int64_t P, int n, int64_t* first_break,
                            double* mx64, uint8_t* detected, cudaStream_t s) {
    if (!first_break && !mx64 && !detected) return cudaSuccess;
    int64_t blocks = (P + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(first_idx, max_abs, P, n, first_break, mx64, detected);
    return cudaGetLastError();
}

}  // namespace bwm
