// Dev microbenchmark (not part of the product): latency of the per-candidate
// preparation pieces on one warp, in SM cycles.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_1208_2675_b200/csrc/chain.cuh"

using namespace qapsa;

__global__ void k_micro(long long* out, Sched sch, int n, const int32_t* rowaddr_g, uint64_t k0) {
    __shared__ int32_t rowaddr[512];
    for (int i = threadIdx.x; i < n; i += blockDim.x) rowaddr[i] = rowaddr_g[i];
    __syncthreads();
    const int t = threadIdx.x;
    const int M = n * (n - 1) / 2;
    Prep pr;
    long long c0, c1, c2, c3, c4, c5;
    int sink = 0;
    c0 = clock_after(t);
    prepare_addr(pr, n, rowaddr, (t * 37) % M, k0 + t);
    c1 = clock_after(pr.addr);
    prepare_theta(pr, sch, 42ull, 0u);
    c2 = clock_after((int)pr.th);
    const U4 x = philox4x32_10((uint32_t)(k0 + t), 0u, 0u, 0u, 42u, 0u);
    c3 = clock_after((int)x.x);
    const float T = temp32(sch, k0 + t);
    c4 = clock_after((int)T);
    int r, s;
    tri_pair(n, (t * 53) % M, &r, &s);
    c5 = clock_after(r + s);
    sink = pr.addr + (int)pr.th + (int)x.y + (int)T + r;
    if (t == 0) {
        out[0] = c1 - c0;  // prepare_addr
        out[1] = c2 - c1;  // prepare_theta
        out[2] = c3 - c2;  // philox alone
        out[3] = c4 - c3;  // temp32 alone
        out[4] = c5 - c4;  // tri_pair alone
        out[5] = sink;
    }
}

extern "C" int micro_run(int n, long long* host_out) {
    long long* d_out;
    int32_t* d_row;
    int row[512];
    int NQ = (n + 3) / 4, g = 0;
    for (int u = 0; u + 1 < n; ++u) {
        const int j0 = (u + 1) / 4;
        row[u] = 4 * g - 4 * j0;
        g += NQ - j0;
    }
    cudaMalloc(&d_out, 8 * sizeof(long long));
    cudaMalloc(&d_row, 512 * 4);
    cudaMemcpy(d_row, row, 512 * 4, cudaMemcpyHostToDevice);
    Sched sch;
    sch.kind = 0; sch.t0 = 12500.2; sch.coef = -8.5e-8; sch.t0f = 12500.2f; sch.coeff = -8.5e-8f;
    for (int it = 0; it < 3; ++it) k_micro<<<1, 32>>>(d_out, sch, n, d_row, 123456789ull);
    cudaMemcpy(host_out, d_out, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d_out);
    cudaFree(d_row);
    return (int)cudaGetLastError();
}
