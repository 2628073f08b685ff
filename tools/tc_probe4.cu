// Dev probe (not part of the product): warm costs of the synchronisation / fence primitives of
// the tensor-memory chain kernel, 128 threads, times by thread 0 (cycles per operation).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/tc_common.cuh"

using namespace qapsa;

__device__ __forceinline__ long long clk(uint32_t dep) {
    long long c;
    asm volatile("{\n\t.reg .b32 d;\n\tmov.b32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(dep) : "memory");
    return c;
}

constexpr int REPS = 256;

__global__ void k_probe4(long long* out, int* sink) {
    __shared__ __align__(16) uint8_t buf[128 * 32];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 256);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase + ((uint32_t)(32 * warp) << 16);
    long long acc[10] = {0};
    uint32_t x = t;
    for (int rep = 0; rep < REPS; ++rep) {
        __syncthreads();
        long long c0 = clk(x);
        buf[t] = (uint8_t)x;                                // (0) STS + fence.proxy.async
        tc::fence_proxy_async();
        long long c1 = clk(x);
        acc[0] += c1 - c0;
        __syncthreads();
        c0 = clk(x);
        tc::tmem_st4(tm + 144, x, x, x, x);                 // (1) STTM.x4 + wait::st
        tc::tmem_wait_st();
        c1 = clk(x);
        acc[1] += c1 - c0;
        __syncthreads();
        c0 = clk(x);
        tc::fence_before_sync();                            // (2) fence + bar + fence
        __syncthreads();
        tc::fence_after_sync();
        c1 = clk(buf[0]);
        acc[2] += c1 - c0;
        c0 = clk(x);
        __syncthreads();                                    // (3) plain bar
        c1 = clk(buf[1]);
        acc[3] += c1 - c0;
        c0 = clk(x);
        const int q = (int)(x * 37u) - 900;                 // (4) int division by 127
        const int g = q / 127;
        c1 = clk((uint32_t)g);
        acc[4] += c1 - c0;
        x += (uint32_t)g;
        __syncthreads();
        c0 = clk(x);                                        // (5) commit on an empty group + wait
        if (t == 0) tc::mma_commit(&bar);
        tc::mbar_wait(&bar, rep & 1);
        c1 = clk(x);
        acc[5] += c1 - c0;
        __syncthreads();
        c0 = clk(x);                                        // (6) all of the stage tail
        buf[t] = (uint8_t)x;
        tc::tmem_st4(tm + 144, x, x, x, x);
        tc::fence_proxy_async();
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncthreads();
        c1 = clk(buf[2]);
        acc[6] += c1 - c0;
        c0 = clk(x);                                        // (7) LDS.U8 x4 dependent on nothing
        const int a0 = buf[(t * 7) & 4095], a1 = buf[(t * 11 + 3) & 4095], a2 = buf[(t * 13 + 5) & 4095];
        c1 = clk((uint32_t)(a0 + a1 + a2));
        acc[7] += c1 - c0;
        x += a0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 256);
    if (t == 0)
        for (int i = 0; i < 8; ++i) out[i] = acc[i] / REPS;
    sink[t] = x;
}

extern "C" int probe4_run(long long* host_out) {
    long long* d;
    int* s;
    cudaMalloc(&d, 8 * sizeof(long long));
    cudaMalloc(&s, 128 * sizeof(int));
    k_probe4<<<1, 128>>>(d, s);
    k_probe4<<<1, 128>>>(d, s);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(host_out, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    return 0;
}
