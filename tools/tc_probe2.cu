// Dev probe (not part of the product): warm latencies of the tcgen05 / TMEM operations a
// tensor-core chain step would use.  One CTA of 128 threads; times taken by thread 0.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/tc_common.cuh"

using namespace qapsa;

template <int NR>
__device__ __forceinline__ void ldx(uint32_t taddr, uint32_t (&v)[NR]);
template <>
__device__ __forceinline__ void ldx<32>(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                   "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                   "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                   "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void stx32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                 "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                 "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                 "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                 : "memory");
}

__device__ __forceinline__ long long clk(uint32_t dep) {
    long long c;
    asm volatile("{\n\t.reg .b32 d;\n\tmov.b32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(dep) : "memory");
    return c;
}

constexpr int REPS = 64;

__global__ void k_probe2(long long* out) {
    __shared__ __align__(1024) int8_t sA[128 * 128];   // 128 x K=128
    __shared__ __align__(1024) int8_t sB[128 * 128];   // N=128 x K=128
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 128 * 128; i += blockDim.x) { sA[i] = (int8_t)(i * 7); sB[i] = (int8_t)(i * 3); }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    uint32_t phase = 0;
    long long acc[12] = {0};
    const uint32_t sbo = 8 * 128;   // K=128 -> 8 core matrices along K, 1024 B per 8-row group
    for (int rep = 0; rep < REPS; ++rep) {
        // (0) one 128x128x32 MMA -> commit -> wait (all threads wait)
        __syncthreads();
        long long c0 = clock64();
        if (t == 0) {
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sA), 128, sbo), tc::smem_desc(tc::smem_u32(sB), 128, sbo),
                       tc::idesc_i8(128, 128), rep > 0);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        long long c1 = clock64();
        acc[0] += c1 - c0;
        // (1) 8 MMAs 128x16x32 (K = 256 total over two operand pairs) -> commit -> wait
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb) {
                const uint32_t o = (kb & 3) * 256;
                tc::mma_i8(tm + 256, tc::smem_desc(tc::smem_u32(kb < 4 ? sA : sB) + o, 128, sbo),
                           tc::smem_desc(tc::smem_u32(sB) + o, 128, sbo), tc::idesc_i8(128, 16), kb > 0);
            }
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        c1 = clock64();
        acc[1] += c1 - c0;
        // (2) ld x1 + wait (each warp its quadrant)
        __syncthreads();
        c0 = clock64();
        uint32_t v1;
        tc::tmem_ld1(tm + ((uint32_t)(32 * warp) << 16) + (rep & 63), v1);
        tc::tmem_wait_ld();
        c1 = clk(v1);
        acc[2] += c1 - c0;
        // (3) ld x32 + wait + st x32 + wait, warp 0 only (one 32-lane x 32-col chunk RMW)
        __syncthreads();
        c0 = clock64();
        if (warp == 0) {
            uint32_t v[32];
            ldx<32>(tm + 0, v);
            tc::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += (t == 5) ? 1u : 0u;
            stx32(tm + 0, v);
            tc::tmem_wait_st();
        }
        c1 = clock64();
        acc[3] += c1 - c0;
        // (4) same RMW over 128 columns (4 chunks), warp 0
        __syncthreads();
        c0 = clock64();
        if (warp == 0) {
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                ldx<32>(tm + 32 * ch, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += (t == 5) ? 1u : 0u;
                stx32(tm + 32 * ch, v);
            }
            tc::tmem_wait_st();
        }
        c1 = clock64();
        acc[4] += c1 - c0;
        // (5) same 128-col RMW, all 4 warps in parallel (each its quadrant)
        __syncthreads();
        c0 = clock64();
        {
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                ldx<32>(tm + ((uint32_t)(32 * warp) << 16) + 32 * ch, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += (t == 5) ? 1u : 0u;
                stx32(tm + ((uint32_t)(32 * warp) << 16) + 32 * ch, v);
            }
            tc::tmem_wait_st();
        }
        __syncthreads();
        c1 = clock64();
        acc[5] += c1 - c0;
        // (6) st x1 + wait, all warps
        __syncthreads();
        c0 = clock64();
        tc::tmem_st1(tm + ((uint32_t)(32 * warp) << 16) + 200, (uint32_t)rep);
        tc::tmem_wait_st();
        c1 = clock64();
        acc[6] += c1 - c0;
        // (7) named-barrier round (bar.sync 1, 128)
        c0 = clock64();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        c1 = clock64();
        acc[7] += c1 - c0;

        // (8) 8 MMAs 128x16x32 into 8 independent accumulators
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb) {
                const uint32_t o = (kb & 3) * 256;
                tc::mma_i8(tm + 256 + 16 * kb, tc::smem_desc(tc::smem_u32(kb < 4 ? sA : sB) + o, 128, sbo),
                           tc::smem_desc(tc::smem_u32(sB) + o, 128, sbo), tc::idesc_i8(128, 16), false);
            }
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        c1 = clock64();
        acc[8] += c1 - c0;
        // (9) two chains of 4
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb) {
                const uint32_t o = (kb >> 1) * 256;
                tc::mma_i8(tm + 256 + 16 * (kb & 1), tc::smem_desc(tc::smem_u32((kb & 1) ? sA : sB) + o, 128, sbo),
                           tc::smem_desc(tc::smem_u32(sB) + o, 128, sbo), tc::idesc_i8(128, 16), kb > 1);
            }
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        c1 = clock64();
        acc[9] += c1 - c0;
        // (10) rank MMA + 8 independent small MMAs, one commit
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sA), 128, sbo), tc::smem_desc(tc::smem_u32(sB), 128, sbo),
                       tc::idesc_i8(128, 128), true);
            for (int kb = 0; kb < 8; ++kb) {
                const uint32_t o = (kb & 3) * 256;
                tc::mma_i8(tm + 256 + 16 * kb, tc::smem_desc(tc::smem_u32(kb < 4 ? sA : sB) + o, 128, sbo),
                           tc::smem_desc(tc::smem_u32(sB) + o, 128, sbo), tc::idesc_i8(128, 16), false);
            }
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        c1 = clock64();
        acc[10] += c1 - c0;
        // (11) 8 small MMAs first, then rank, one commit
        __syncthreads();
        c0 = clock64();
        if (t == 0) {
            for (int kb = 0; kb < 8; ++kb) {
                const uint32_t o = (kb & 3) * 256;
                tc::mma_i8(tm + 256 + 16 * kb, tc::smem_desc(tc::smem_u32(kb < 4 ? sA : sB) + o, 128, sbo),
                           tc::smem_desc(tc::smem_u32(sB) + o, 128, sbo), tc::idesc_i8(128, 16), false);
            }
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(sA), 128, sbo), tc::smem_desc(tc::smem_u32(sB), 128, sbo),
                       tc::idesc_i8(128, 128), true);
            tc::mma_commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        c1 = clock64();
        acc[11] += c1 - c0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 512);
    if (t == 0)
        for (int i = 0; i < 12; ++i) out[i] = acc[i] / REPS;
}

extern "C" int probe2_run(long long* host_out) {
    long long* d;
    cudaMalloc(&d, 12 * sizeof(long long));
    k_probe2<<<1, 128>>>(d);
    k_probe2<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(host_out, d, 12 * sizeof(long long), cudaMemcpyDeviceToHost);
    return 0;
}
