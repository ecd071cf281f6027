// tma_probe.cu — streaming bandwidth of the monitor kernel's exact access pattern with no
// compute: per-warp 2-D tensor TMA boxes of BOXW pixels x 8 dates into a warp-private stage
// ring (S stages), CTAs of 4 warps, persistent grid, the consumer only sums the box.
// Row schedule per tile: "full" = dates [0, N) once; "kernel" = the monitor kernel's 3-pass
// stream (history, window-0 re-read from L2, monitoring period).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu -lcuda
// Run:   ./tma_probe            (C2 geometry: 4096^2 px, N=228, n=114, h=28)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int BOXW, int S>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap map, int64_t P, int N, int n, int h,
                                             int sched, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int R = 8, SB = BOXW * R * 4, WPX = BOXW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* st = sm + warp * S * SB;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4 * S * SB) + warp * S;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const int64_t tiles = P / (4 * WPX);
    const int w0 = ((n - h + 1) / R) * R, t3 = (n / R) * R;
    const int st1 = (n + R - 1) / R, st2 = (n - w0 + R - 1) / R, st3 = (N - t3 + R - 1) / R;
    const int per_tile = sched ? st1 + st2 + st3 : (N + R - 1) / R;
    int64_t itile = blockIdx.x;
    int istage = 0;
    auto issue = [&](int slot) {
        if (itile >= tiles) return;
        int r0;
        if (!sched) r0 = istage * R;
        else r0 = istage < st1 ? istage * R : istage < st1 + st2 ? w0 + (istage - st1) * R : t3 + (istage - st1 - st2) * R;
        const int x = (int)(itile * 4 * WPX) + warp * WPX;
        const uint32_t dst = su32(st + slot * SB), b = su32(bar + slot);
        asm volatile(
            "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
            "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n\t"
            "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}"
            ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(r0), "r"(b), "r"(SB) : "memory");
        if (++istage == per_tile) { istage = 0; itile += gridDim.x; }
    };
    for (int s = 0; s < S; ++s) issue(s);
    float acc = 0.f;
    int cur = 0;
    uint32_t ph = 0;
    const int64_t my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    for (int64_t i = 0; i < my_tiles * per_tile; ++i) {
        asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}"
                     ::"r"(su32(bar + cur)), "r"(ph) : "memory");
        const float* f = reinterpret_cast<const float*>(st + cur * SB);
#pragma unroll
        for (int k = 0; k < R * WPX / 32; ++k) acc += f[k * 32 + lane];
        __syncwarp();
        issue(cur);
        if (++cur == S) { cur = 0; ph ^= 1; }
    }
    if (acc == 12345.f) out[0] = acc;
}


// CTA-synchronous variant: one thread issues NB boxes of 256/NB px covering the CTA's 256-px
// tile per stage; every warp consumes its 64 px; __syncthreads before a slot is re-armed.
// Same coupling for every NB, so only the box width changes.
template <int NB, int S>
__global__ void __launch_bounds__(128) k_sync(const __grid_constant__ CUtensorMap map, int64_t P, int N, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int R = 8, SB = 256 * R * 4, BW = 256 / NB;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S * SB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int64_t tiles = P / 256;
    const int per_tile = (N + R - 1) / R;
    int64_t itile = blockIdx.x;
    int istage = 0;
    auto issue = [&](int slot) {
        if (itile >= tiles) return;
        const uint32_t b = su32(bar + slot);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(SB) : "memory");
        for (int i = 0; i < NB; ++i) {
            // box i: pixels [i*BW, (i+1)*BW) of the tile, rows [r0, r0+8): smem rows of BW floats
            const uint32_t dst = su32(sm + slot * SB + i * BW * R * 4);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&map)), "r"((int)(itile * 256 + i * BW)), "r"(istage * R), "r"(b)
                : "memory");
        }
        if (++istage == per_tile) { istage = 0; itile += gridDim.x; }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) issue(s);
    float acc = 0.f;
    int cur = 0;
    uint32_t ph = 0;
    const int64_t my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    for (int64_t i = 0; i < my_tiles * per_tile; ++i) {
        asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}"
                     ::"r"(su32(bar + cur)), "r"(ph) : "memory");
        const float* f = reinterpret_cast<const float*>(sm + cur * SB) + warp * 64 * R;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += f[k * 32 + lane];
        __syncthreads();
        if (threadIdx.x == 0) issue(cur);
        if (++cur == S) { cur = 0; ph ^= 1; }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const int N = 228, n = 114, h = 28;
    const int64_t P = 4096ll * 4096;
    float* y = nullptr;
    CK(cudaMalloc(&y, (size_t)N * P * 4));
    CK(cudaMemset(y, 0, (size_t)N * P * 4));
    float* out = nullptr;
    CK(cudaMalloc(&out, 4));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](auto kern, int boxw, int S, int ctas, int sched, const char* name) -> int {
        CUtensorMap map;
        const cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)N};
        const cuuint64_t strides[1] = {(cuuint64_t)P * 4};
        const cuuint32_t box[2] = {(cuuint32_t)boxw, 8};
        const cuuint32_t es[2] = {1, 1};
        if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        const size_t smem = 4 * (size_t)S * boxw * 8 * 4 + 4 * S * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = sms * ctas;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int i = 0; i < 3; ++i) kern<<<grid, 128, smem>>>(map, P, N, n, h, sched, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        const int it = 10;
        for (int i = 0; i < it; ++i) kern<<<grid, 128, smem>>>(map, P, N, n, h, sched, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= it;
        const double rows = sched ? (double)(((n + 7) / 8) + ((n - ((n - h + 1) / 8) * 8 + 7) / 8) + ((N - (n / 8) * 8 + 7) / 8)) * 8 : N;
        printf("%-28s box %3d px, S=%d, %d CTA/SM: %.3f ms  DRAM-algorithmic %.0f GB/s  SM-ingest %.0f GB/s\n", name, boxw,
               S, ctas, ms, (double)N * P * 4 / ms / 1e6, rows * P * 4 / ms / 1e6);
        return 0;
    };
    auto run_sync = [&](auto kern, int boxw, int S, int ctas) -> int {
        CUtensorMap map;
        const cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)N};
        const cuuint64_t strides[1] = {(cuuint64_t)P * 4};
        const cuuint32_t box[2] = {(cuuint32_t)boxw, 8};
        const cuuint32_t es[2] = {1, 1};
        if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return 1;
        const size_t smem = (size_t)S * 256 * 8 * 4 + S * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = sms * ctas;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int i = 0; i < 3; ++i) kern<<<grid, 128, smem>>>(map, P, N, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) kern<<<grid, 128, smem>>>(map, P, N, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        printf("CTA-synchronous, %d boxes of %3d px per stage, S=%d, %d CTA/SM: %.3f ms  %.0f GB/s\n", 256 / boxw, boxw,
               S, ctas, ms, (double)N * P * 4 / ms / 1e6);
        return 0;
    };
    run_sync(k_sync<4, 5>, 64, 5, 4);
    run_sync(k_sync<2, 5>, 128, 5, 4);
    run_sync(k_sync<1, 5>, 256, 5, 4);
    run_sync(k_sync<4, 3>, 64, 3, 4);
    run_sync(k_sync<1, 3>, 256, 3, 4);
    for (int sched = 0; sched < 2; ++sched) {
        const char* nm = sched ? "kernel 3-pass schedule" : "dates [0,N) once";
        run(k_tma<64, 5>, 64, 5, 4, sched, nm);
        run(k_tma<64, 8>, 64, 8, 4, sched, nm);
        run(k_tma<128, 4>, 128, 4, 3, sched, nm);
        run(k_tma<256, 3>, 256, 3, 2, sched, nm);
    }
    return 0;
}
