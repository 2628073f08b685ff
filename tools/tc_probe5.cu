// Dev probe (not part of the product): does issuing the 8 touching MMAs from 4 warps in
// parallel (2 each, separate accumulators, 4 commits) beat one thread issuing all 8?
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

__global__ void k_probe5(long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;               // 128 x 128
    uint8_t* sB = sm + 16384;       // 128 x 128
    uint8_t* sV = sm + 32768;       // 16 x 128
    uint8_t* sR = sm + 34816;       // 128 x 32
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar1, bar4;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 38912; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (t == 0) { tc::mbar_init(&bar1, 1); tc::mbar_init(&bar4, 4); }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    uint32_t ph1 = 0, ph4 = 0;
    long long acc[6] = {0};
    const uint32_t idt = tc::idesc_i8(128, 16, true), idr = tc::idesc_i8(128, 128, true);
    for (int rep = 0; rep < REPS; ++rep) {
        // (0) one thread: rank (SS) + 8 touching
        __syncthreads();
        long long c0 = clk(rep);
        if (t == 0) {
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::smem_desc(tc::smem_u32(sR), 128, 256), idr, true);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + 256, tc::smem_desc(tc::smem_u32(sA) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, kc > 0);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + 256, tc::smem_desc(tc::smem_u32(sB) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, true);
            tc::mma_commit(&bar1);
        }
        tc::mbar_wait(&bar1, ph1); ph1 ^= 1;
        acc[0] += clk(ph1) - c0;
        // (1) 4 warps: warp w issues kc = w for A and B' into accumulator 256 + 16 w; warp 0 also rank
        __syncthreads();
        c0 = clk(rep);
        if ((t & 31) == 0) {
            const int kc = warp;
            if (warp == 0)
                tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::smem_desc(tc::smem_u32(sR), 128, 256), idr, true);
            tc::mma_i8(tm + 256 + 16 * warp, tc::smem_desc(tc::smem_u32(sA) + 256 * kc, 128, 1024),
                       tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, false);
            tc::mma_i8(tm + 256 + 16 * warp, tc::smem_desc(tc::smem_u32(sB) + 256 * kc, 128, 1024),
                       tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, true);
            tc::mma_commit(&bar4);
        }
        tc::mbar_wait(&bar4, ph4); ph4 ^= 1;
        acc[1] += clk(ph4) - c0;
        // (2) issue-only cost in one thread: 9 MMAs without waiting (time to issue)
        __syncthreads();
        c0 = clk(rep);
        long long ci = 0;
        if (t == 0) {
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::smem_desc(tc::smem_u32(sR), 128, 256), idr, true);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + 256, tc::smem_desc(tc::smem_u32(sA) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, kc > 0);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + 256, tc::smem_desc(tc::smem_u32(sB) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(sV) + 256 * kc, 128, 1024), idt, true);
            ci = clk(rep) - c0;
            tc::mma_commit(&bar1);
        }
        tc::mbar_wait(&bar1, ph1); ph1 ^= 1;
        acc[2] += ci;
        acc[3] += clk(ph1) - c0;
        // (3) rank only (SS, N=128)
        __syncthreads();
        c0 = clk(rep);
        if (t == 0) {
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::smem_desc(tc::smem_u32(sR), 128, 256), idr, true);
            tc::mma_commit(&bar1);
        }
        tc::mbar_wait(&bar1, ph1); ph1 ^= 1;
        acc[4] += clk(ph1) - c0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 512);
    if (t == 0) for (int i = 0; i < 5; ++i) out[i] = acc[i] / REPS;
}

extern "C" int probe5_run(long long* host_out) {
    long long* d;
    cudaMalloc(&d, 8 * sizeof(long long));
    cudaFuncSetAttribute(k_probe5, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k_probe5<<<1, 128, 40000>>>(d);
    k_probe5<<<1, 128, 40000>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(host_out, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    return 0;
}
