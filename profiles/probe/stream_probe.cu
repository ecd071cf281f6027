// stream_probe.cu — achievable read bandwidth for the access patterns the bfastmonitor
// kernel can use on a time-major [N][P] float32 stack (N=228, P=4096^2: 15.3 GB).
//
//   bulk<TILE>   : producer warp + 4 consumer warps; one cp.async.bulk per row of a TILE-px
//                  tile (TILE*4 bytes), 8 rows per stage, S stages; consumers sum the stage.
//   ldg          : every thread streams float4 of its pixels row by row (no smem).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t p) {
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}" ::"r"(su32(b)), "r"(p) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

template <int TILE, int S, int R>
__global__ void __launch_bounds__(160) k_bulk(const float* y, int64_t ld, int64_t P, int N, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int RB = TILE * 4;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * R * RB);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int64_t tiles = P / TILE;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 4) {
        if (lane) return;
        int cur = 0; uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
            for (int r0 = 0; r0 < N; r0 += R) {
                const int rows = min(R, N - r0);
                mb_wait(empty + cur, ph ^ 1);
                mb_tx(full + cur, rows * RB);
#pragma unroll 1
                for (int r = 0; r < rows; ++r) bulk(sm + (cur * R + r) * RB, y + (int64_t)(r0 + r) * ld + t * TILE, RB, full + cur);
                if (++cur == S) { cur = 0; ph ^= 1; }
            }
        return;
    }
    float acc = 0.f;
    int cur = 0; uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int r0 = 0; r0 < N; r0 += R) {
            mb_wait(full + cur, ph);
            const float* st = reinterpret_cast<const float*>(sm + cur * R * RB);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int q = 0; q < TILE / 128; ++q) acc += st[r * TILE + q * 128 + threadIdx.x];
            __syncwarp();
            if (lane == 0) mb_arrive(empty + cur);
            if (++cur == S) { cur = 0; ph ^= 1; }
        }
    if (acc == 12345.f) out[0] = acc;
}

// bulk3: the kernel's row stream (pass1 rows [0,n), pass2 rows [0,n), pass3 rows [t3,N)) with
// WORK dependent-chain FFMA2 per row per thread (emulating the fused per-row compute).
template <int TILE, int S, int R, int WORK>
__global__ void __launch_bounds__(160) k_bulk3(const float* y, int64_t ld, int64_t P, int N, int n, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int RB = TILE * 4;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * R * RB);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int64_t tiles = P / TILE;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int t3 = (n / R) * R;
    if (warp == 4) {
        if (lane) return;
        int cur = 0; uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
#pragma unroll 1
            for (int pass = 0; pass < 3; ++pass) {
                const int lo = pass == 2 ? t3 : 0, hi = pass == 2 ? N : n;
                for (int r0 = lo; r0 < hi; r0 += R) {
                    const int rows = min(R, hi - r0);
                    mb_wait(empty + cur, ph ^ 1);
                    mb_tx(full + cur, rows * RB);
#pragma unroll 1
                    for (int r = 0; r < rows; ++r) bulk(sm + (cur * R + r) * RB, y + (int64_t)(r0 + r) * ld + t * TILE, RB, full + cur);
                    if (++cur == S) { cur = 0; ph ^= 1; }
                }
            }
        return;
    }
    float2 acc = make_float2(0.f, 0.f), w = make_float2(1.0001f, 0.9999f);
    int cur = 0; uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int pass = 0; pass < 3; ++pass) {
            const int lo = pass == 2 ? t3 : 0, hi = pass == 2 ? N : n;
            for (int r0 = lo; r0 < hi; r0 += R) {
                mb_wait(full + cur, ph);
                const float2* st = reinterpret_cast<const float2*>(sm + cur * R * RB) + threadIdx.x;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 v = st[r * (TILE / 2)];
#pragma unroll
                    for (int q = 0; q < WORK; ++q) v = __ffma2_rn(v, w, acc);
                    acc = __fadd2_rn(acc, v);
                }
                __syncwarp();
                if (lane == 0) mb_arrive(empty + cur);
                if (++cur == S) { cur = 0; ph ^= 1; }
            }
        }
    if (acc.x == 12345.f) out[0] = acc.x;
}

template <int TILE, int S, int R, int WORK>
void run_bulk3(const float* y, int64_t P, int N, int n, float* out, int sms, int ctas) {
    auto k = k_bulk3<TILE, S, R, WORK>;
    const int smem = S * R * TILE * 4 + 2 * S * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float ms = timeit([&] { k<<<sms * ctas, 160, smem>>>(y, P, P, N, n, out); }, 5);
    cudaError_t e = cudaGetLastError();
    printf("bulk3 tile=%4d S=%2d R=%2d work=%2d ctas/sm=%d : %7.3f ms  %7.1f GB/s(alg) %s\n", TILE, S, R, WORK, ctas, ms,
           (double)P * N * 4 / ms / 1e6, e ? cudaGetErrorString(e) : "");
}

template <int PXT>   // pixels per thread (float PXT loads per row)
__global__ void __launch_bounds__(128) k_ldg(const float* y, int64_t ld, int64_t P, int N, float* out) {
    const int64_t tiles = P / (128 * PXT);
    float acc = 0.f;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const float* p = y + t * 128 * PXT + threadIdx.x * PXT;
#pragma unroll 8
        for (int r = 0; r < N; ++r) {
            if (PXT == 4) { float4 v = __ldg(reinterpret_cast<const float4*>(p + (int64_t)r * ld)); acc += v.x + v.y + v.z + v.w; }
            else { float2 v = __ldg(reinterpret_cast<const float2*>(p + (int64_t)r * ld)); acc += v.x + v.y; }
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

template <class F>
float timeit(F launch, int reps);
template <class F>
float timeit_impl(F launch, int reps) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

template <int TILE, int S, int R>
void run_bulk(const float* y, int64_t P, int N, float* out, int sms, int ctas) {
    auto k = k_bulk<TILE, S, R>;
    const int smem = S * R * TILE * 4 + 2 * S * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float ms = timeit([&] { k<<<sms * ctas, 160, smem>>>(y, P, P, N, out); }, 5);
    cudaError_t e = cudaGetLastError();
    printf("bulk tile=%4d S=%d R=%2d smem=%6d ctas/sm=%d : %7.3f ms  %7.1f GB/s %s\n", TILE, S, R, smem, ctas, ms,
           (double)P * N * 4 / ms / 1e6, e ? cudaGetErrorString(e) : "");
}

template <class F>
float timeit(F launch, int reps) { return timeit_impl(launch, reps); }

int main() {
    const int N = 228;
    const int64_t P = 4096LL * 4096;
    float *y, *out;
    CK(cudaMalloc(&y, (size_t)P * N * 4));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(y, 0, (size_t)P * N * 4));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 114;
    run_bulk3<256, 7, 8, 0>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 7, 8, 8>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 7, 8, 16>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 7, 8, 24>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 7, 8, 32>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 4, 8, 16>(y, P, N, n, out, sms, 3);
    run_bulk3<256, 12, 8, 16>(y, P, N, n, out, sms, 2);
    run_bulk3<256, 7, 8, 16>(y, P, N, n, out, sms, 2);
    if (getenv("PROBE_ALL") == nullptr) return 0;
    for (int c : {2, 4, 8}) {
        float ms = timeit([&] { k_ldg<4><<<sms * c, 128>>>(y, P, P, N, out); }, 5);
        printf("ldg float4 ctas/sm=%d : %7.3f ms %7.1f GB/s\n", c, ms, (double)P * N * 4 / ms / 1e6);
        ms = timeit([&] { k_ldg<2><<<sms * c, 128>>>(y, P, P, N, out); }, 5);
        printf("ldg float2 ctas/sm=%d : %7.3f ms %7.1f GB/s\n", c, ms, (double)P * N * 4 / ms / 1e6);
    }
    run_bulk<256, 7, 8>(y, P, N, out, sms, 3);
    run_bulk<256, 4, 8>(y, P, N, out, sms, 3);
    run_bulk<256, 8, 16>(y, P, N, out, sms, 1);
    run_bulk<256, 4, 16>(y, P, N, out, sms, 3);
    run_bulk<512, 4, 8>(y, P, N, out, sms, 3);
    run_bulk<512, 6, 8>(y, P, N, out, sms, 2);
    run_bulk<1024, 3, 8>(y, P, N, out, sms, 2);
    run_bulk<256, 12, 8>(y, P, N, out, sms, 2);
    run_bulk<256, 24, 8>(y, P, N, out, sms, 1);
    return 0;
}
