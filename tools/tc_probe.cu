// Dev probe (not part of the product): one int8 tcgen05 MMA D[128 x N] = A[128 x K] B[N x K]^T
// with operands in the K-major no-swizzle canonical layout, result read back with tcgen05.ld.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/tc_common.cuh"

using namespace qapsa;

constexpr int M = 128, N = 16, K = 128;   // K = 4 MMAs of 32

__global__ void k_probe(const int8_t* Ag, const int8_t* Bg, int* Dg, long long* cyc) {
    __shared__ __align__(1024) int8_t sA[M * K];
    __shared__ __align__(1024) int8_t sB[N * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x;
    const int sboA = (K / 16) * 128, sboB = (K / 16) * 128;
    for (int i = t; i < M * K; i += blockDim.x) {
        const int x = i / K, k = i % K;
        sA[tc::kmaj_off(x, k, sboA)] = Ag[i];
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        const int x = i / K, k = i % K;
        sB[tc::kmaj_off(x, k, sboB)] = Bg[i];
    }
    if (t < 32) tc::tmem_alloc(&tbase, 32);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tbase;
    long long c0 = clock64();
    if (t == 0) {
        const uint32_t id = tc::idesc_i8(M, N);
        for (int kb = 0; kb < K / 32; ++kb) {
            const uint64_t da = tc::smem_desc(tc::smem_u32(sA) + kb * 256, 128, sboA);
            const uint64_t db = tc::smem_desc(tc::smem_u32(sB) + kb * 256, 128, sboB);
            tc::mma_i8(tmem, da, db, id, kb > 0);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    long long c1 = clock64();
    const int warp = t >> 5, lane = t & 31;
    if (warp < 4) {
        uint32_t v[8];
        for (int c = 0; c < N; c += 8) {
            tc::tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
            tc::tmem_wait_ld();
            for (int i = 0; i < 8; ++i) Dg[(32 * warp + lane) * N + c + i] = (int)v[i];
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (t < 32) tc::tmem_dealloc(tmem, 32);
    if (t == 0) cyc[0] = c1 - c0;
}

extern "C" int probe_run(const int8_t* A, const int8_t* B, int* D, long long* cyc) {
    int8_t *dA, *dB;
    int* dD;
    long long* dc;
    cudaMalloc(&dA, M * K);
    cudaMalloc(&dB, N * K);
    cudaMalloc(&dD, M * N * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A, M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, N * K, cudaMemcpyHostToDevice);
    k_probe<<<1, 128>>>(dA, dB, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D, dD, M * N * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cyc, dc, 8, cudaMemcpyDeviceToHost);
    return 0;
}
