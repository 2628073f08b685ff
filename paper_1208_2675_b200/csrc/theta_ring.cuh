// theta_ring.cuh -- the acceptance thresholds of Eq.(2) (R1, R3, R16, R23) for a
// single chain, computed ahead on the SMs the chain does not use and streamed into the chain's
// shared memory by the tensor memory accelerator.
//
// A single chain runs on one SM (or one cluster); the other SMs of the B200 are idle.  The
// decision of Eq.(2) at iteration k depends on the state only through the integer δ, so k_theta
// reduces it, for every k of a call's iteration range, to ONE integer (R23):
//
//   thr_k = the largest δ accepted at iteration k, i.e. accept iff δ <= thr_k,
//
// evaluated with the very double-precision test the chain kernels apply (metropolis(): exp(-δ/T_k)
// > r_k, T_k by R1, r_k by R3) at the integers around θ_k = -T_k ln r_k; every integer at least
// one below (above) θ_k is accepted (rejected) by a relative margin of 1/T_k, far beyond the
// rounding of exp and log while T_k < 1e9.  Iterations whose test may hold a near tie (R16:
// |δ + T ln r| < 1e-9 T for an integer δ >= 1 next to θ_k; or T_k >= 1e9, or θ_k beyond int32) are
// flagged and stored as -1: a candidate at a flagged iteration takes the kernels' general test
// (float θ with a margin, exact double test inside it, near ties logged), so every decision and
// every near-tie record is the one the general test makes.
//
// Layout: blocks of TH_BLK iterations, thr as int32 (4 KB per block) plus a 16-byte header per
// block {any flagged iteration, max thr_k over the block (INT_MAX if flagged), 0, 0}.  The chain kernel pulls blocks
// into a ring of SLOTS blocks with cp.async.bulk (one elected thread, completion on one mbarrier
// per slot; TH_SLOTS = 8 for the scratch phase's short windows, TH_SLOTS_TC = 32 for the Δ
// engine's whole-row windows of up to 7 blocks), as far ahead of the window as the ring allows.
// The window then tests a candidate with one shared-memory load and one integer compare.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "chain.cuh"
#include "tc_common.cuh"

namespace qapsa {

constexpr int TH_BLK = 1024;                     // thresholds per ring block (4 KB, one bulk copy)
constexpr int TH_SLOTS = 8;                      // scratch phase: ring blocks (32 KB of shared memory)
constexpr int TH_RING = TH_BLK * TH_SLOTS;
constexpr int TH_RING_BYTES = TH_RING * 4;
constexpr int TH_SLOTS_TC = 32;                  // Δ engine (windows up to 7 blocks): 128 KB
constexpr unsigned long long TH_CHUNK = 1ull << 24;   // iterations per threshold buffer fill (64 MB)

// thr_k and its flag (R23): the decision of metropolis() at every integer next to θ_k
__device__ __forceinline__ int exact_threshold(const Sched& sch, uint64_t seed, uint32_t chain, uint64_t k,
                                               bool* flag) {
    const double T = temperature(sch, k);
    const double r = uniform_r(seed, k, chain);
    const double th = -__dmul_rn(T, log(r));     // θ_k = -T ln r_k >= 0
    if (!(T < 1e9) || !(th < 2.0e9)) {           // outside the margin argument: general path
        *flag = true;
        return th < 2.0e9 ? (int)th : INT_MAX;
    }
    const long long lo = (long long)floor(th) - 1;   // every δ < lo is accepted
    long long thr = lo - 1;
    bool fl = false, run = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {                // δ = lo .. lo + 3 (every δ > lo + 3 is rejected)
        const long long d = lo + i;
        // metropolis() with its log(r) hoisted: accept iff exp(-δ/T) > r, near iff |δ + T ln r| < 1e-9 T;
        // δ <= 0 is accepted without a test (R5)
        const double dd = (double)d;
        const bool acc = d <= 0 || exp(__ddiv_rn(-dd, T)) > r;
        fl |= d > 0 && fabs(__dadd_rn(dd, -th)) < __dmul_rn(1e-9, T);
        if (run && acc) thr = d;
        else run = false;
        fl |= acc && !run;                       // not monotone around θ (never expected): general path
    }
    *flag = fl;
    return (int)thr;
}

// thr_k for k = kb + i, i < cnt (cnt a multiple of TH_BLK), and the block headers; one CTA of
// 256 threads per block (grid-stride over blocks)
__global__ void __launch_bounds__(256) k_theta(const Sched sch, unsigned long long seed, uint32_t chain,
                                               unsigned long long kb, unsigned long long cnt,
                                               int* __restrict__ out, int4* __restrict__ hdr) {
    __shared__ int s_max, s_flag;
    const long long nblk = (long long)(cnt / TH_BLK);
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        if (threadIdx.x == 0) { s_max = INT_MIN; s_flag = 0; }
        __syncthreads();
        int mx = INT_MIN, fl = 0;
        for (int i = threadIdx.x; i < TH_BLK; i += blockDim.x) {
            const unsigned long long o = (unsigned long long)b * TH_BLK + i;
            bool f;
            const int t = exact_threshold(sch, seed, chain, kb + o, &f);
            out[o] = f ? -1 : t;                 // flagged: the candidate takes the general test
            mx = max(mx, f ? INT_MAX : t);
            fl |= f;
        }
        atomicMax(&s_max, mx);
        if (fl) atomicOr(&s_flag, 1);
        __syncthreads();
        if (threadIdx.x == 0) hdr[b] = make_int4(s_flag, s_max, 0, 0);
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

// One chain's view of a ring of SLOTS blocks of BS thresholds (BS divides TH_BLK; the block
// headers are copied only when BS == TH_BLK).  Every consumer thread keeps `ready` (blocks known
// complete, identical in all threads: they wait in the same order); the issuing thread also keeps
// `issued`.  A window of w iterations leaves SLOTS - ceil(w / BS) - 1 blocks of prefetch.
template <int SLOTS, int BS = TH_BLK>
struct ThetaRing {
    static_assert(TH_BLK % BS == 0 && BS % 4 == 0, "ring blocks split k_theta's blocks");
    static constexpr int RING = SLOTS * BS;
    static constexpr bool HDR = BS == TH_BLK;
    int* ring;                   // shared memory, RING thresholds
    int4* hring;                 // shared memory, SLOTS block headers (HDR)
    uint64_t* bars;              // shared memory, SLOTS mbarriers
    const int* src;              // thresholds of iterations [kb, kb + nblk BS)
    const int4* hsrc;            // their block headers (HDR)
    unsigned long long kb;
    long long nblk;
    long long ready;
    long long issued;

    // issuing thread: blocks [issued, min(nblk, b_lo + SLOTS)); the slot of block b held block
    // b - SLOTS < b_lo, whose iterations every consumer has passed (a CTA / group barrier
    // separates the last window that read it from this call)
    __device__ __forceinline__ void refill(unsigned long long k) {
        const long long b_lo = (long long)((k - kb) / BS);
        const long long hi = min(nblk, b_lo + SLOTS);
        for (; issued < hi; ++issued) {
            const int slot = (int)(issued & (SLOTS - 1));
            tc::mbar_expect_tx(bars + slot, BS * 4 + (HDR ? 16 : 0));
            tc::bulk_g2s(ring + slot * BS, src + issued * BS, BS * 4, bars + slot);
            if (HDR) tc::bulk_g2s(hring + slot, hsrc + issued, 16, bars + slot);
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
    // every consumer: thresholds of iterations < k_hi resident (block b completes phase
    // (b / SLOTS) & 1)
    __device__ __forceinline__ void ensure(unsigned long long k_hi) {
        const long long bh = (long long)((k_hi - 1 - kb) / BS);
        while (ready <= bh) {
            tc::mbar_wait(bars + (int)(ready & (SLOTS - 1)), (uint32_t)((ready / SLOTS) & 1));
            ++ready;
        }
    }
    // the same with 32-bit offsets from kb (a launch's range is far below 2^31)
    __device__ __forceinline__ void ensure_ofs(int ofs_hi) {
        while (ready * BS < (long long)ofs_hi) {
            tc::mbar_wait(bars + (int)(ready & (SLOTS - 1)), (uint32_t)((ready / SLOTS) & 1));
            ++ready;
        }
    }
    __device__ __forceinline__ int at_ofs(int ofs) const { return ring[ofs & (RING - 1)]; }
    __device__ __forceinline__ int at(unsigned long long kk) const {
        return ring[(int)((kk - kb) & (unsigned long long)(RING - 1))];
    }
    // iterations [k_lo, k_hi) (resident; HDR): {any flagged, max thr}
    __device__ __forceinline__ int2 span(unsigned long long k_lo, unsigned long long k_hi) const {
        int fl = 0, mx = INT_MIN;
        for (long long b = (long long)((k_lo - kb) / BS); b <= (long long)((k_hi - 1 - kb) / BS); ++b) {
            const int4 h = hring[(int)(b & (SLOTS - 1))];
            fl |= h.x;
            mx = max(mx, h.y);
        }
        return make_int2(fl, mx);
    }
    // issuing thread, before the CTA exits: no bulk copy may still be writing its shared memory
    __device__ __forceinline__ void drain() {
        for (long long b = ready; b < issued; ++b)
            tc::mbar_wait(bars + (int)(b & (SLOTS - 1)), (uint32_t)((b / SLOTS) & 1));
    }
};

template <int SLOTS, int BS = TH_BLK>
__device__ __forceinline__ ThetaRing<SLOTS, BS> theta_ring(int* ring, int4* hring, uint64_t* bars, const int* src,
                                                           const int4* hsrc, unsigned long long kb,
                                                           unsigned long long cnt, unsigned long long k) {
    // blocks are counted from the one holding k (a kernel chained after the scratch phase starts
    // inside the buffer): every slot's first use is then phase 0 of its mbarrier
    const unsigned long long b0 = (k - kb) / BS;
    ThetaRing<SLOTS, BS> R;
    R.ring = ring;
    R.hring = hring;
    R.bars = bars;
    R.src = src + b0 * BS;
    R.hsrc = hsrc + b0 * BS / TH_BLK;
    R.kb = kb + b0 * BS;
    R.nblk = (long long)((cnt + BS - 1) / BS) - (long long)b0;
    R.ready = 0;
    R.issued = 0;
    return R;
}

}  // namespace qapsa
