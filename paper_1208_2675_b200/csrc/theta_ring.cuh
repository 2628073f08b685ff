// theta_ring.cuh -- the thresholds θ_k = -T_k ln r_k of Eq.(2) (R1, R3) for a
// single chain, computed ahead on the SMs the chain does not use and streamed into the chain's
// shared memory by the tensor memory accelerator.
//
// A single chain runs on one SM (or one cluster); the other SMs of the B200 are idle.  θ_k depends
// only on the iteration index k (T_k by R1, r_k by R3), not on the state, so k_theta computes
// every θ of a call's iteration range [kb, kb + cnt) up front across the whole GPU (about
// 0.4 ms for 1e8 iterations) into an HBM buffer, and the chain kernel pulls 4 KB blocks of it
// into a ring of blocks with cp.async.bulk (one elected thread, completion on one mbarrier per
// slot; TH_SLOTS = 8 for the scratch phase's short windows, TH_SLOTS_TC = 32 for the Δ engine's
// whole-row windows of up to 7 blocks), as far ahead of the window as the ring allows.  The window then reads θ with one
// shared-memory load per candidate instead of a Philox4x32-10 block, a logf and an expf.
//
// Exactness is unchanged: θ is the float value prepare_theta computes (chain.cuh), the window
// brackets it with the margin m = 2e-4 θ + 2e-5 T (T = temp32 at the window's first iteration,
// >= T_k up to 2e-6 relative: T is non-increasing) and decides inside the margin with the exact
// double test (R16), so every decision equals the double-precision one.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <cstdint>

#include "chain.cuh"
#include "tc_common.cuh"

namespace qapsa {

constexpr int TH_BLK = 1024;                     // θ per ring block (4 KB, one bulk copy)
constexpr int TH_SLOTS = 8;                      // scratch phase: ring blocks (32 KB of shared memory)
constexpr int TH_RING = TH_BLK * TH_SLOTS;
constexpr int TH_RING_BYTES = TH_RING * 4;
constexpr int TH_SLOTS_TC = 32;                  // Δ engine (windows up to 7 blocks): 128 KB
constexpr unsigned long long TH_CHUNK = 1ull << 27;   // iterations per θ buffer fill (512 MB)

// θ_k for k = kb + i, i < cnt (cnt a multiple of TH_BLK); any grid
__global__ void k_theta(const Sched sch, unsigned long long seed, uint32_t chain, unsigned long long kb,
                        unsigned long long cnt, float* __restrict__ out) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        Prep pr;
        pr.k = kb + i;
        prepare_theta(pr, sch, seed, chain);
        out[i] = pr.th;
    }
}

namespace tc {
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy (TMA, non-tensor), completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
}  // namespace tc

// One chain's view of a ring of SLOTS blocks.  Every consumer thread keeps `ready` (blocks known
// complete, identical in all threads: they wait in the same order); the issuing thread also keeps
// `issued`.  A window of w iterations leaves SLOTS - ceil(w / TH_BLK) - 1 blocks of prefetch.
template <int SLOTS>
struct ThetaRing {
    static constexpr int RING = SLOTS * TH_BLK;
    float* ring;                 // shared memory, RING floats
    uint64_t* bars;              // shared memory, SLOTS mbarriers
    const float* src;            // θ of iterations [kb, kb + nblk TH_BLK)
    unsigned long long kb;
    long long nblk;
    long long ready;
    long long issued;

    // issuing thread: blocks [issued, min(nblk, b_lo + SLOTS)); the slot of block b held block
    // b - SLOTS < b_lo, whose iterations every consumer has passed (a CTA / group barrier
    // separates the last window that read it from this call)
    __device__ __forceinline__ void refill(unsigned long long k) {
        const long long b_lo = (long long)((k - kb) / TH_BLK);
        const long long hi = min(nblk, b_lo + SLOTS);
        for (; issued < hi; ++issued) {
            const int slot = (int)(issued & (SLOTS - 1));
            tc::mbar_expect_tx(bars + slot, TH_BLK * 4);
            tc::bulk_g2s(ring + slot * TH_BLK, src + issued * TH_BLK, TH_BLK * 4, bars + slot);
        }
    }
    // thread 0 of the chain before the kernel's first use: barriers, first SLOTS blocks
    // (the caller then synchronises the consumers)
    __device__ __forceinline__ void start(unsigned long long k) {
        for (int i = 0; i < SLOTS; ++i) tc::mbar_init(bars + i, 1);
        tc::fence_mbar_init();
        tc::fence_proxy_async();
        issued = 0;
        refill(k);
    }
    // every consumer: θ of iterations < k_hi resident (block b completes phase (b / SLOTS) & 1)
    __device__ __forceinline__ void ensure(unsigned long long k_hi) {
        const long long bh = (long long)((k_hi - 1 - kb) / TH_BLK);
        while (ready <= bh) {
            tc::mbar_wait(bars + (int)(ready & (SLOTS - 1)), (uint32_t)((ready / SLOTS) & 1));
            ++ready;
        }
    }
    __device__ __forceinline__ float at(unsigned long long kk) const {
        return ring[(int)((kk - kb) & (unsigned long long)(RING - 1))];
    }
    // issuing thread, before the CTA exits: no bulk copy may still be writing its shared memory
    __device__ __forceinline__ void drain() {
        for (long long b = ready; b < issued; ++b)
            tc::mbar_wait(bars + (int)(b & (SLOTS - 1)), (uint32_t)((b / SLOTS) & 1));
    }
};

template <int SLOTS>
__device__ __forceinline__ ThetaRing<SLOTS> theta_ring(float* ring, uint64_t* bars, const float* src,
                                                unsigned long long kb, unsigned long long cnt,
                                                unsigned long long k) {
    // blocks are counted from the one holding k (a kernel chained after the scratch phase starts
    // inside the buffer): every slot's first use is then phase 0 of its mbarrier
    const unsigned long long b0 = (k - kb) / TH_BLK;
    ThetaRing<SLOTS> R;
    R.ring = ring;
    R.bars = bars;
    R.src = src + b0 * TH_BLK;
    R.kb = kb + b0 * TH_BLK;
    R.nblk = (long long)((cnt + TH_BLK - 1) / TH_BLK) - (long long)b0;
    R.ready = 0;
    R.issued = 0;
    return R;
}

}  // namespace qapsa
