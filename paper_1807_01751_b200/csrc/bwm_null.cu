// bwm_null.cu — the null-hypothesis draws of critical_value, generated on the device.
//
// The reference calibrates lambda by Monte Carlo (mosum.py:166-227): replication r draws its
// N standard normals from np.random.Generator(np.random.Philox(key=seed, counter=r << 128))
// (mosum.py:195-198).  numpy implements that stream as Philox4x64-10 (Random123) feeding the
// 256-layer ziggurat of random_standard_normal (numpy/random/src/distributions/distributions.c);
// this file restates both, so every replication's series is bit-identical to the reference's
// (cast to float32 for the monitor kernel, as the host path did) — checked against numpy in
// tests/test_gpu_parity.py::test_null_draws_match_numpy.  One thread per replication walks its
// own counter-based substream; its N draws go down its column of the time-major stack, so a
// warp's stores of one date are one coalesced 128-byte row.  No host draws, no H2D.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bwm.h"
#include "bwm_ziggurat_tables.h"

namespace bwm {
int set_error(int code, const std::string& msg);   // bwm_capi.cu (thread-local last error)
namespace {

constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ull, kPhiloxM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ull, kPhiloxW1 = 0xBB67AE8584CAA73Bull;
constexpr double kNorR = 3.6541528853610087963519472518;      // ziggurat_nor_r
constexpr double kNorInvR = 0.27366123732975827203338247596;  // ziggurat_nor_inv_r

struct Philox {
    uint64_t c0, c1, c2, c3, k0, k1;
    uint64_t b[4];
    int pos;
    __device__ void block() {
        uint64_t x0 = c0, x1 = c1, x2 = c2, x3 = c3, a = k0, bb = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            if (r) { a += kPhiloxW0; bb += kPhiloxW1; }
            const uint64_t hi0 = __umul64hi(kPhiloxM0, x0), lo0 = kPhiloxM0 * x0;
            const uint64_t hi1 = __umul64hi(kPhiloxM1, x2), lo1 = kPhiloxM1 * x2;
            x0 = hi1 ^ x1 ^ a;
            x1 = lo1;
            x2 = hi0 ^ x3 ^ bb;
            x3 = lo0;
        }
        b[0] = x0; b[1] = x1; b[2] = x2; b[3] = x3;
    }
    // numpy philox_next64: increment the 256-bit counter, then encrypt it; 4 outputs per block
    __device__ uint64_t next64() {
        if (pos == 4) {
            if (++c0 == 0 && ++c1 == 0 && ++c2 == 0) ++c3;
            block();
            pos = 0;
        }
        return b[pos++];
    }
    __device__ double next_double() { return __dmul_rn((double)(next64() >> 11), 1.0 / 9007199254740992.0); }
};

// numpy random_standard_normal, operation for operation (no FMA contraction)
__device__ double standard_normal(Philox& s) {
    for (;;) {
        uint64_t r = s.next64();
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        double x = __dmul_rn(__ull2double_rn(rabs), kZigWi[idx]);
        if (sign) x = -x;
        if (rabs < kZigKi[idx]) return x;      // 99.3% of draws
        if (idx == 0) {
            for (;;) {
                const double xx = __dmul_rn(-kNorInvR, log1p(-s.next_double()));
                const double yy = -log1p(-s.next_double());
                if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
                    return ((rabs >> 8) & 1) ? -__dadd_rn(kNorR, xx) : __dadd_rn(kNorR, xx);
            }
        } else {
            const double u = s.next_double();
            if (__dadd_rn(__dmul_rn(__dadd_rn(kZigFi[idx - 1], -kZigFi[idx]), u), kZigFi[idx]) <
                exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
                return x;
        }
    }
}

__global__ void __launch_bounds__(128) null_draws_kernel(uint64_t seed_lo, uint64_t seed_hi, int64_t rep0,
                                                         int64_t reps, int n_obs, float* __restrict__ out,
                                                         int64_t ld) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= reps) return;
    const uint64_t rep = (uint64_t)(rep0 + j);
    Philox s;
    s.c0 = 0; s.c1 = 0; s.c2 = rep; s.c3 = 0;        // counter = rep << 128
    s.k0 = seed_lo; s.k1 = seed_hi;
    s.pos = 4;
    float* o = out + j;
    for (int t = 0; t < n_obs; ++t) o[(int64_t)t * ld] = (float)standard_normal(s);
}

}  // namespace
}  // namespace bwm

extern "C" int bwm_null_draws(uint64_t seed_lo, uint64_t seed_hi, int64_t rep0, int64_t reps, int32_t n_obs,
                              float* out, int64_t ld, void* stream) {
    if (!out) return bwm::set_error(BWM_E_NULL, "out is NULL");
    if (reps < 1 || n_obs < 1 || rep0 < 0 || ld < reps)
        return bwm::set_error(BWM_E_DIMS, "need reps >= 1, n_obs >= 1, rep0 >= 0, ld >= reps");
    const int64_t blocks = (reps + 127) / 128;
    bwm::null_draws_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(seed_lo, seed_hi, rep0, reps, n_obs,
                                                                                out, ld);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BWM_OK : bwm::set_error((int)e, std::string("null draws launch failed: ") + cudaGetErrorString(e));
}
