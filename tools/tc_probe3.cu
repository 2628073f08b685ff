// Dev probe (not part of the product): A operand in TMEM (TS mode) for kind::i8.
// (1) correctness of D = A B^T with A (128 x 128 u8) in TMEM, B (16 x 128 u8) in smem;
// (2) warm timings of TS-mode MMAs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/tc_common.cuh"

using namespace qapsa;

__device__ __forceinline__ void st_x4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}

constexpr int REPS = 64;

__global__ void k_probe3(const uint8_t* Ag, const uint8_t* Bg, int* Dg, long long* out) {
    __shared__ __align__(1024) uint8_t sB[16 * 128];
    __shared__ __align__(1024) uint8_t sR[128 * 32];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t sboB = 8 * 128;
    for (int i = t; i < 16 * 128; i += blockDim.x) sB[tc::kmaj_off(i / 128, i % 128, sboB)] = Bg[i];
    for (int i = t; i < 128 * 32; i += blockDim.x) sR[i] = (uint8_t)(i * 5);
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    // A row t -> TMEM lane t, columns 160.. (4 bytes per column, little-endian K order)
    for (int c = 0; c < 32; c += 4) {
        uint32_t w[4];
        for (int i = 0; i < 4; ++i) {
            const uint8_t* a = Ag + t * 128 + 4 * (c + i);
            w[i] = a[0] | (a[1] << 8) | (a[2] << 16) | ((uint32_t)a[3] << 24);
        }
        st_x4(tm + lane_base + 160 + c, w[0], w[1], w[2], w[3]);
    }
    tc::tmem_wait_st();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    uint32_t phase = 0;
    if (t == 0) {
        for (int kb = 0; kb < 4; ++kb)
            tc::mma_i8_ts(tm + 128, tm + 160 + 8 * kb, tc::smem_desc(tc::smem_u32(sB) + kb * 256, 128, sboB),
                          tc::idesc_i8(128, 16, false), kb > 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    {
        uint32_t v[8];
        for (int c = 0; c < 16; c += 8) {
            tc::tmem_ld8(tm + lane_base + 128 + c, v);
            tc::tmem_wait_ld();
            for (int i = 0; i < 8; ++i) Dg[t * 16 + c + i] = (int)v[i];
        }
    }
    long long acc[8] = {0};
    for (int rep = 0; rep < REPS; ++rep) {
        __syncthreads();
        long long c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 4; ++kb)
                tc::mma_i8_ts(tm + 128, tm + 160 + 8 * kb, tc::smem_desc(tc::smem_u32(sB) + kb * 256, 128, sboB),
                              tc::idesc_i8(128, 16, false), kb > 0);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[0] += clock64() - c0;
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb)
                tc::mma_i8_ts(tm + 128 + 16 * (kb >> 2), tm + 160 + 8 * (kb & 3),
                              tc::smem_desc(tc::smem_u32(sB) + (kb & 3) * 256, 128, sboB),
                              tc::idesc_i8(128, 16, false), (kb & 3) > 0);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[1] += clock64() - c0;
        // rank-style: L in TMEM (8 cols), R (128 x 32) in smem, N = 128
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            tc::mma_i8_ts(tm, tm + 224, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::idesc_i8(128, 128), true);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[2] += clock64() - c0;
        // rank + 8 small, one commit
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            tc::mma_i8_ts(tm, tm + 224, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::idesc_i8(128, 128), true);
            for (int kb = 0; kb < 8; ++kb)
                tc::mma_i8_ts(tm + 128 + 16 * (kb >> 2), tm + 160 + 8 * (kb & 3),
                              tc::smem_desc(tc::smem_u32(sB) + (kb & 3) * 256, 128, sboB),
                              tc::idesc_i8(128, 16, false), (kb & 3) > 0);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[3] += clock64() - c0;
        // 8 independent TS N=16 (accumulators at 256 + 16 i)
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb)
                tc::mma_i8_ts(tm + 256 + 16 * kb, tm + 160 + 8 * (kb & 3),
                              tc::smem_desc(tc::smem_u32(sB) + (kb & 3) * 256, 128, sboB),
                              tc::idesc_i8(128, 16, false), false);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[4] += clock64() - c0;
        // 8 independent TS N=8
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb)
                tc::mma_i8_ts(tm + 256 + 8 * kb, tm + 160 + 8 * (kb & 3),
                              tc::smem_desc(tc::smem_u32(sB) + (kb & 3) * 256, 128, sboB),
                              tc::idesc_i8(128, 8, false), false);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[5] += clock64() - c0;
        // 1 TS N=16
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            tc::mma_i8_ts(tm + 256, tm + 160, tc::smem_desc(tc::smem_u32(sB), 128, sboB),
                          tc::idesc_i8(128, 16, false), false);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[6] += clock64() - c0;
        // rank + 8 independent
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            tc::mma_i8_ts(tm, tm + 224, tc::smem_desc(tc::smem_u32(sR), 128, 256), tc::idesc_i8(128, 128), true);
            for (int kb = 0; kb < 8; ++kb)
                tc::mma_i8_ts(tm + 256 + 16 * kb, tm + 160 + 8 * (kb & 3),
                              tc::smem_desc(tc::smem_u32(sB) + (kb & 3) * 256, 128, sboB),
                              tc::idesc_i8(128, 16, false), false);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        acc[7] += clock64() - c0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 512);
    if (t == 0)
        for (int i = 0; i < 8; ++i) out[i] = acc[i] / REPS;
}

extern "C" int probe3_run(const uint8_t* A, const uint8_t* B, int* D, long long* host_out) {
    uint8_t *dA, *dB;
    int* dD;
    long long* d;
    cudaMalloc(&dA, 128 * 128);
    cudaMalloc(&dB, 16 * 128);
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMalloc(&d, 8 * sizeof(long long));
    cudaMemcpy(dA, A, 128 * 128, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 16 * 128, cudaMemcpyHostToDevice);
    k_probe3<<<1, 128>>>(dA, dB, dD, d);
    k_probe3<<<1, 128>>>(dA, dB, dD, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D, dD, 128 * 16 * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(host_out, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    return 0;
}
