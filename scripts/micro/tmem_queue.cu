// Micro-benchmark (development): a per-thread ring of float4 "planes" kept in TMEM instead of
// registers.  Each iteration stores one float4 (tcgen05.st 32x32b.x4) and reads the 2H others
// (tcgen05.ld 32x32b.x4 each, one wait), against the same pattern through shared memory.
#include <cstdio>
#include <cuda_runtime.h>
#define H 8
#define NQ (2 * H + 1)
__device__ __forceinline__ void tst4(unsigned addr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d) : "memory");
}
__device__ __forceinline__ float4 tld4(unsigned addr) {
    float4 v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
    return v;
}
__global__ void __launch_bounds__(512, 1) k_tmem(float* out, int iters, long long* cyc) {
    __shared__ unsigned base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane quadrant = warp % 4 (lanes 32q..32q+31); columns [128 * (warp / 4), +128) per warp
    const unsigned tb = base + ((unsigned)(32 * (warp & 3)) << 16) + 128u * (warp >> 2);
    float4 acc = make_float4(0, 0, 0, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int s = i % NQ;
        tst4(tb + 4 * s, i * 1.f, i * 2.f, i * 3.f, i * 4.f);
        float4 v[2 * H];
#pragma unroll
        for (int k = 1; k <= 2 * H; ++k) v[k - 1] = tld4(tb + 4 * ((s + k) % NQ));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 2 * H; ++k) {
            acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
        }
    }
    const long long t1 = clock64();
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
__device__ __forceinline__ void tld16(unsigned addr, float* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                   "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                 : "r"(addr) : "memory");
}
__global__ void __launch_bounds__(512, 1) k_tmem16(float* out, int iters, long long* cyc) {
    __shared__ unsigned base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tb = base + ((unsigned)(32 * (warp & 3)) << 16) + 128u * (warp >> 2);
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int s = i & 15;
        tst4(tb + 4 * (i % 32), i * 1.f, i * 2.f, i * 3.f, i * 4.f);
        float v[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q) tld16(tb + 16 * ((s + q) & 7), v[q]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] += v[q][j];
    }
    const long long t1 = clock64();
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    float r = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) r += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
__global__ void __launch_bounds__(512, 1) k_smem(float* out, int iters, long long* cyc) {
    extern __shared__ float4 ring[];  // [NQ][512]
    float4 acc = make_float4(0, 0, 0, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int s = i % NQ;
        ring[s * 512 + threadIdx.x] = make_float4(i * 1.f, i * 2.f, i * 3.f, i * 4.f);
        float4 v[2 * H];
#pragma unroll
        for (int k = 1; k <= 2 * H; ++k) v[k - 1] = ring[((s + k) % NQ) * 512 + threadIdx.x];
#pragma unroll
        for (int k = 0; k < 2 * H; ++k) {
            acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, NQ * 512 * 16);
    for (int rep = 0; rep < 2; ++rep) {
        long long c[148];
        k_tmem<<<148, 512>>>(out, iters, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        printf("tmem: %s  %.1f cycles/iter (16 warps/SM, 16 x4-loads + 1 x4-store per thread)\n", cudaGetErrorString(e), (double)c[0] / iters);
        k_smem<<<148, 512, NQ * 512 * 16>>>(out, iters, cyc);
        e = cudaDeviceSynchronize();
        cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        printf("smem: %s  %.1f cycles/iter (same pattern, LDS.128/STS.128)\n", cudaGetErrorString(e), (double)c[0] / iters);
        k_tmem16<<<148, 512>>>(out, iters, cyc);
        e = cudaDeviceSynchronize();
        cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        printf("tmem x16: %s  %.1f cycles/iter (4 x16-loads = 256 B/thread, 16 independent accumulators)\n", cudaGetErrorString(e), (double)c[0] / iters);
    }
    return 0;
}
