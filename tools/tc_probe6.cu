// Dev probe (not part of the product): TMEM read/write throughput for 32-lane x 32-column blocks
// by 1, 4, 8 warps; and a 4-chunk pipelined read-modify-write by one warp.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/tc_common.cuh"

using namespace qapsa;
constexpr int REPS = 64;

__device__ __forceinline__ long long clk(uint32_t dep) {
    long long c;
    asm volatile("{\n\t.reg .b32 d;\n\tmov.b32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(dep) : "memory");
    return c;
}

__global__ void k_probe6(long long* out, uint32_t* sink) {
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    long long acc[6] = {0};
    uint32_t x = 0;
    for (int rep = 0; rep < REPS; ++rep) {
        for (int mode = 0; mode < 3; ++mode) {
            const int nw = mode == 0 ? 1 : mode == 1 ? 4 : 8;
            __syncthreads();
            const long long c0 = clk(x);
            if (warp < nw) {
                uint32_t v[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tc::tmem_ld32(tm + 32 * c + 128 * (warp >> 2), v[c]);
                tc::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) x += v[c][i];
            }
            __syncthreads();
            acc[mode] += clk(x) - c0;
        }
        // 4-chunk pipelined RMW by one warp (load all, modify lane 5, store all, wait)
        __syncthreads();
        long long c0 = clk(x);
        if (warp == 0) {
            uint32_t v[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tmem_ld32(tm + 32 * c, v[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i) v[c][i] += (t == 5) ? 1u : 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tmem_st32(tm + 32 * c, v[c]);
            tc::tmem_wait_st();
        }
        __syncthreads();
        acc[3] += clk(x) - c0;
        // single chunk load+wait only
        c0 = clk(x);
        if (warp == 0) {
            uint32_t v[32];
            tc::tmem_ld32(tm, v);
            tc::tmem_wait_ld();
            x += v[3];
        }
        acc[4] += clk(x) - c0;
        __syncthreads();
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
    if (t == 0) for (int i = 0; i < 5; ++i) out[i] = acc[i] / REPS;
    sink[t] = x;
}

extern "C" int probe6_run(long long* host_out) {
    long long* d;
    uint32_t* s;
    cudaMalloc(&d, 8 * sizeof(long long));
    cudaMalloc(&s, 256 * 4);
    k_probe6<<<1, 256>>>(d, s);
    k_probe6<<<1, 256>>>(d, s);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(host_out, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    return 0;
}
