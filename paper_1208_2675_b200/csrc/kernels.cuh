// kernels.cuh -- the __global__ kernels of libqapsa (sm_100a).
//
//   k_reset          p <- source, best_p <- p, C <- Eq.(1), best <- C   (qap_reset / qap_create)
//   k_cost           Eq.(1) of a permutation (qap_cost)
//   k_delta_init     step (a), Δ for all pairs, one thread per pair  (qap_delta_init)
//   k_sa_chain       persistent single-chain kernel, 1 CTA           (qap_sa_run)
//   k_ensemble       persistent multi-chain kernel, G chains / CTA   (qap_ensemble_run)
//   k_ens_reduce     argmin over chains + summed statistics
//   k_delta_bounds   min nonzero |Δ|, max |Δ| for the schedule rule R2 (qap_schedule_bounds)
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <cstdint>

#include "chain.cuh"

namespace qapsa {

struct DevState {                 // single-chain scalars, device resident
    long long cost;
    long long best_cost;
    unsigned long long digest;
    unsigned long long accepted;  // cumulative since reset
    unsigned int near_count;      // cumulative since reset (= log entries, may exceed cap)
    unsigned int pad;
};

struct ChainResult {              // mirrors qap_chain_result
    long long cost, best_cost;
    unsigned long long accepted, near_ties, digest, iterations;
};

// ---------------- shared-memory layout of one chain group ----------------
struct GroupLayout {
    int bp, d, dab, dg, p, bestp, slots, flags, bytes;
};
__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }
// dab_bytes: 4 when A and B are both 8-bit (packed int16 pair), else 8
// nqt: number of Δ quads (quad layout, chain.cuh)
__host__ __device__ inline GroupLayout group_layout(int n, int ld, int nqt, int tb_bytes, int nw,
                                                    bool d_in_smem, int dab_bytes) {
    GroupLayout L;
    const int n4 = (n + 3) & ~3;
    int o = 0;
    L.bp = o;    o = align16(o + n * ld * tb_bytes);
    L.d = o;     o = align16(o + (d_in_smem ? nqt * 16 : 0));
    L.dab = o;   o = align16(o + n4 * dab_bytes);
    L.dg = o;    o = align16(o + n * 4);
    L.p = o;     o = align16(o + n * 2);
    L.bestp = o; o = align16(o + n * 2);
    L.slots = o; o = align16(o + 2 * nw * 16);
    L.flags = o; o = align16(o + 4 * 4);
    L.bytes = o;
    return L;
}

template <typename TA, typename TB>
__device__ inline ChainSmem<TA, TB> group_view(unsigned char* base, const GroupLayout& L,
                                               int32_t* d_global) {
    ChainSmem<TA, TB> cs;
    cs.Bp = reinterpret_cast<TB*>(base + L.bp);
    cs.D = d_global ? d_global : reinterpret_cast<int32_t*>(base + L.d);
    cs.dAB = reinterpret_cast<typename Dab<TA, TB>::T*>(base + L.dab);
    cs.Dg = reinterpret_cast<int32_t*>(base + L.dg);
    cs.p = reinterpret_cast<uint16_t*>(base + L.p);
    cs.best_p = reinterpret_cast<uint16_t*>(base + L.bestp);
    cs.slots = reinterpret_cast<int4*>(base + L.slots);
    cs.flags = reinterpret_cast<int*>(base + L.flags);
    return cs;
}

// per-CTA prefix: A (n x ld) | rowaddr (n int) | qdesc (nqt uint32)
__host__ __device__ inline int cta_prefix_bytes(int n, int ld, int ta_bytes, int nqt) {
    return align16(n * ld * ta_bytes) + align16(n * 4) + align16(nqt * 2);
}

// cooperative copy of bytes (16-byte aligned, size multiple of 4)
__device__ inline void copy_words(void* dst, const void* src, int bytes, int t, int nt) {
    const int n16 = bytes >> 4;
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    for (int i = t; i < n16; i += nt) d4[i] = s4[i];
    uint32_t* d1 = reinterpret_cast<uint32_t*>(dst);
    const uint32_t* s1 = reinterpret_cast<const uint32_t*>(src);
    for (int i = (n16 << 2) + t; i < (bytes >> 2); i += nt) d1[i] = s1[i];
}

// B'_ij = B_{p(i),p(j)} into shared memory; columns >= n zero.
template <typename TB>
__device__ inline void build_bprime(TB* Bp, const TB* __restrict__ B, const uint16_t* p, int n,
                                    int ld, int t, int nt) {
    for (int idx = t; idx < n * ld; idx += nt) {
        const int i = idx / ld, j = idx - i * ld;
        Bp[idx] = j < n ? B[p[i] * ld + p[j]] : (TB)0;
    }
}

// ---------------- small kernels ----------------

template <typename TA, typename TB>
__global__ void k_reset(const TA* __restrict__ A, const TB* __restrict__ B, const int32_t* src, int n,
                        int ld, int32_t* p, int32_t* best_p, DevState* st) {
    __shared__ long long part[32];
    const int t = threadIdx.x;
    src += (size_t)blockIdx.x * n;                // ensemble: CTA b resets chain b
    p += (size_t)blockIdx.x * n;
    best_p += (size_t)blockIdx.x * n;
    st += blockIdx.x;
    long long acc = 0;
    for (int idx = t; idx < n * n; idx += blockDim.x) {
        const int i = idx / n, j = idx - i * n;
        acc += (long long)A[i * ld + j] * (long long)B[src[i] * ld + src[j]];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((t & 31) == 0) part[t >> 5] = acc;
    __syncthreads();
    for (int i = t; i < n; i += blockDim.x) {
        const int32_t v = src[i];
        p[i] = v;
        best_p[i] = v;
    }
    if (t == 0) {
        long long c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += part[w];
        st->cost = c;
        st->best_cost = c;
        st->digest = kDigestSeed;
        st->accepted = 0;
        st->near_count = 0;
    }
}

template <typename TA, typename TB>
__global__ void k_cost(const TA* __restrict__ A, const TB* __restrict__ B, const int32_t* perm, int n,
                       int ld, long long* out) {
    __shared__ long long part[32];
    const int t = threadIdx.x;
    long long acc = 0;
    for (int idx = t; idx < n * n; idx += blockDim.x) {
        const int i = idx / n, j = idx - i * n;
        acc += (long long)A[i * ld + j] * (long long)B[perm[i] * ld + perm[j]];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((t & 31) == 0) part[t >> 5] = acc;
    __syncthreads();
    if (t == 0) {
        long long c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += part[w];
        *out = c;
    }
}

// Step (a): one thread per pair, B' read through p (gather from L2).
// δ(r,s) = 2 [ sum_all k (a_rk - a_sk)(B'_sk - B'_rk) + 2 a_rs B'_rs ]
template <typename TA, typename TB>
__global__ void k_delta_init(const TA* __restrict__ A, const TB* __restrict__ B,
                             const int32_t* __restrict__ p, const int32_t* __restrict__ rowaddr,
                             int n, int ld, int M, int32_t* D, int dstride = 0) {
    p += (size_t)blockIdx.y * n;                  // ensemble: grid row y = chain y
    D += (size_t)blockIdx.y * dstride;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < M; q += gridDim.x * blockDim.x) {
        int r, s;
        tri_pair(n, q, &r, &s);
        const TA* Ar = A + r * ld;
        const TA* As = A + s * ld;
        const TB* Br = B + p[r] * ld;
        const TB* Bs = B + p[s] * ld;
        int acc = 0;
        for (int k = 0; k < n; ++k) {
            const int pk = __ldg(p + k);
            acc += ((int)Ar[k] - (int)As[k]) * ((int)Bs[pk] - (int)Br[pk]);
        }
        D[rowaddr[r] + s] = 2 * (acc + 2 * (int)Ar[s] * (int)Br[p[s]]);
    }
}

// quad layout -> enumeration order (qap_get_state, qap_schedule_bounds)
__global__ void k_unpad(const int32_t* __restrict__ D, const int32_t* __restrict__ rowaddr, int n,
                        int M, int32_t* out) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < M; q += gridDim.x * blockDim.x) {
        int r, s;
        tri_pair(n, q, &r, &s);
        out[q] = D[rowaddr[r] + s];
    }
}

__global__ void k_delta_bounds(const int32_t* __restrict__ D, int M, int* out /* [0]=dmin, [1]=dmax */) {
    __shared__ int smin[32], smax[32];
    int mn = INT_MAX, mx = 0;
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
        const int a = abs(D[q]);
        mx = max(mx, a);
        if (a) mn = min(mn, a);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = mn; smax[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mn = min(mn, smin[w]); mx = max(mx, smax[w]); }
        out[0] = mn == INT_MAX ? 0 : mn;
        out[1] = mx;
    }
}

// ---------------- the persistent single-chain kernel (qap_sa_run) ----------------
struct ChainArgs {
    const void* A;           // n x ld compact
    const void* B;           // n x ld compact
    int32_t* p;              // n
    int32_t* best_p;         // n
    int32_t* D;              // quad layout (global copy; also the working Δ when !D_SMEM)
    const int32_t* rowaddr;  // n
    const uint16_t* qdesc;   // nqt
    int nqt;
    DevState* st;
    unsigned int* near_count;
    unsigned long long* near_k;
    unsigned char* near_dec;
    int near_cap;
    int n, ld, M, wmax;
    int wscan;               // Δ engine (k_sa_tc): window cap of its whole-row windows
    unsigned long long k0, k_end, seed;
    Sched sch;
    const unsigned long long* k0_dev;   // if set, k0 is read from device memory (chained launches)
    int proposal;            // 0 sequential enumeration (R4), 1 random pairs (R22)
    // ensemble launches of the tensor-memory kernels (ens = 1): CTA b runs chain chain + b on
    // p + b n, best_p + b n, st + b, D + b dstride, k0_dev + 2 b; near ties only counted
    int ens, dstride;
    uint32_t* near_chain;    // ensembles: chain id of every near-tie log entry (near_count = the
                             // launch-wide log counter, near_k / near_dec the log)
    uint32_t chain;          // Philox chain id (R3) of the chain (of CTA 0 when ens)
    unsigned long long switch_gap;   // scratch phase: switch to Δ after this many iterations
                                     // without an accept (0 = TCS_SWITCH_GAP)
    // single-chain launches of the tensor-memory kernels: integer thresholds of iterations
    // [theta_kb, theta_kb + theta_cnt) and their block headers precomputed by k_theta
    // (theta_ring.cuh, R23); ensemble launches compute θ in the kernel
    const int* theta;
    const int4* theta_hdr;
    unsigned long long theta_kb, theta_cnt;
};

// per-CTA chain state of a (possibly ensemble) launch of the tensor-memory kernels
struct ChainView {
    int32_t* p;
    int32_t* best_p;
    int32_t* D;
    DevState* st;
    const unsigned long long* k0_dev;
    NearSink sink;
    uint32_t chain;
};
// ENS = false (single-chain launches): the chain id is the constant 0, so the Philox rounds of
// the thresholds fold it as before
template <bool ENS>
__device__ __forceinline__ ChainView chain_view(const ChainArgs& a) {
    ChainView v;
    if (!ENS) {
        v.p = a.p; v.best_p = a.best_p; v.D = a.D; v.st = a.st; v.k0_dev = a.k0_dev;
        v.sink = NearSink{a.near_count, a.near_k, a.near_dec, a.near_cap, nullptr, nullptr, 0u};
        v.chain = 0u;
        return v;
    }
    const int b = (int)blockIdx.x;
    v.p = a.p + (size_t)b * a.n;
    v.best_p = a.best_p + (size_t)b * a.n;
    v.D = a.D + (size_t)b * a.dstride;
    v.st = a.st + b;
    v.k0_dev = a.k0_dev ? a.k0_dev + 2 * b : nullptr;
    v.chain = a.chain + (uint32_t)b;
    v.sink = NearSink{&v.st->near_count, a.near_k, a.near_dec, a.near_cap, a.near_count, a.near_chain, v.chain};
    return v;
}

// NFIX > 0: problem size fixed at compile time (layout offsets and loop bounds fold);
// NFIX == 0: any n.
template <typename TA, typename TB, int NT, bool D_SMEM, int NFIX>
__global__ void __launch_bounds__(NT, 1) k_sa_chain(const ChainArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = threadIdx.x;
    const int n = NFIX ? NFIX : a.n;
    const int ld = NFIX ? row_stride(NFIX, sizeof(TA) == 1 && sizeof(TB) == 1) : a.ld;
    const int M = NFIX ? NFIX * (NFIX - 1) / 2 : a.M;
    const int nqt = NFIX ? quad_count(NFIX) : a.nqt;
    const int a_bytes = align16(n * ld * (int)sizeof(TA));
    TA* As = reinterpret_cast<TA*>(smem);
    int32_t* rowaddr = reinterpret_cast<int32_t*>(smem + a_bytes);
    uint16_t* qdesc = reinterpret_cast<uint16_t*>(smem + a_bytes + align16(n * 4));
    const GroupLayout L = group_layout(n, ld, nqt, sizeof(TB), NT / 32, D_SMEM,
                                       sizeof(typename Dab<TA, TB>::T));
    ChainSmem<TA, TB> cs = group_view<TA, TB>(smem + cta_prefix_bytes(n, ld, sizeof(TA), nqt), L,
                                              D_SMEM ? nullptr : a.D);
    const ChainTables tb{rowaddr, qdesc};

    copy_words(As, a.A, n * ld * (int)sizeof(TA), t, NT);
    copy_words(rowaddr, a.rowaddr, n * 4, t, NT);
    copy_words(qdesc, a.qdesc, (nqt * 2 + 3) & ~3, t, NT);
    for (int i = t; i < n; i += NT) {
        cs.p[i] = (uint16_t)a.p[i];
        cs.best_p[i] = (uint16_t)a.best_p[i];
    }
    if (D_SMEM) copy_words(cs.D, a.D, nqt * 16, t, NT);
    if (t < 4) cs.flags[t] = 0;
    __syncthreads();
    build_bprime(cs.Bp, reinterpret_cast<const TB*>(a.B), cs.p, n, ld, t, NT);
    ChainScalars io{a.st->cost, a.st->best_cost, a.st->digest};
    __syncthreads();
    chain_diag_init<TA, TB, NT>(As, cs, n, ld, t);
    __syncthreads();

    const NearSink sink{a.near_count, a.near_k, a.near_dec, a.near_cap, nullptr, nullptr, 0u};
    constexpr int QPT = NFIX ? quads_per_thread(NT, NFIX) : 0;
    const uint64_t acc = chain_run<TA, TB, NT, QPT>(As, cs, tb, n, ld, M, nqt, a.k0, a.k_end, a.sch,
                                                    a.seed, 0u, 0, t, a.wmax, io, sink, a.proposal != 0);

    for (int i = t; i < n; i += NT) {
        a.p[i] = cs.p[i];
        a.best_p[i] = cs.best_p[i];
    }
    if (D_SMEM) copy_words(a.D, cs.D, nqt * 16, t, NT);
    if (t == scalar_tid(NT, n)) {
        a.st->cost = io.cost;
        a.st->best_cost = io.best;
        a.st->digest = io.digest;
        a.st->accepted += acc;
    }
}

// ---------------- the persistent ensemble kernel (qap_ensemble_run) ----------------
struct EnsArgs {
    const void* A;
    const void* B;
    const int32_t* p0s;          // count x n
    ChainResult* res;            // count
    uint16_t* best_perms;        // count x n
    unsigned int* next_chain;    // work counter
    const int32_t* rowaddr;      // n
    const uint16_t* qdesc;       // nqt
    int nqt;
    int count, n, ld, M, wmax;
    unsigned int chain_begin;
    unsigned long long iters, seed;
    Sched sch;
    int proposal;            // 0 sequential enumeration (R4), 1 random pairs (R22)
    unsigned int* near_count;    // launch-wide near-tie log (chain, k, decision), capacity near_cap
    unsigned long long* near_k;
    unsigned char* near_dec;
    uint32_t* near_chain;
    int near_cap;
};

template <typename TA, typename TB, int NT, int NFIX>
__global__ void __launch_bounds__(1024, 1) k_ensemble(const EnsArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = NFIX ? NFIX : a.n;
    const int ld = NFIX ? row_stride(NFIX, sizeof(TA) == 1 && sizeof(TB) == 1) : a.ld;
    const int M = NFIX ? NFIX * (NFIX - 1) / 2 : a.M;
    const int nqt = NFIX ? quad_count(NFIX) : a.nqt;
    const int a_bytes = align16(n * ld * (int)sizeof(TA));
    TA* As = reinterpret_cast<TA*>(smem);
    int32_t* rowaddr = reinterpret_cast<int32_t*>(smem + a_bytes);
    uint16_t* qdesc = reinterpret_cast<uint16_t*>(smem + a_bytes + align16(n * 4));
    const GroupLayout L = group_layout(n, ld, nqt, sizeof(TB), NT / 32, true,
                                       sizeof(typename Dab<TA, TB>::T));
    const int g = threadIdx.x / NT, t = threadIdx.x % NT, bar = 1 + 2 * g;  // +1: staging hand-off
    ChainSmem<TA, TB> cs =
        group_view<TA, TB>(smem + cta_prefix_bytes(n, ld, sizeof(TA), nqt) + g * L.bytes, L, nullptr);
    const ChainTables tb{rowaddr, qdesc};

    copy_words(As, a.A, n * ld * (int)sizeof(TA), threadIdx.x, blockDim.x);
    copy_words(rowaddr, a.rowaddr, n * 4, threadIdx.x, blockDim.x);
    copy_words(qdesc, a.qdesc, (nqt * 2 + 3) & ~3, threadIdx.x, blockDim.x);
    __syncthreads();

    for (;;) {
        if (t == 0) cs.flags[2] = (int)atomicAdd(a.next_chain, 1u);
        group_sync(bar, NT);
        const int ci = cs.flags[2];
        if (ci >= a.count) break;
        const int32_t* p0 = a.p0s + (size_t)ci * n;
        for (int i = t; i < n; i += NT) {
            cs.p[i] = (uint16_t)p0[i];
            cs.best_p[i] = (uint16_t)p0[i];
        }
        if (t < 2) cs.flags[t] = 0;
        group_sync(bar, NT);
        build_bprime(cs.Bp, reinterpret_cast<const TB*>(a.B), cs.p, n, ld, t, NT);
        group_sync(bar, NT);
        chain_delta_init<TA, TB, NT>(As, cs, tb, n, ld, M, t);
        chain_diag_init<TA, TB, NT>(As, cs, n, ld, t);
        // C = Eq.(1) = sum_ij A_ij B'_ij
        long long part = 0;
        for (int idx = t; idx < n * n; idx += NT) {
            const int i = idx / n, j = idx - i * n;
            part += (long long)As[i * ld + j] * (long long)cs.Bp[i * ld + j];
        }
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        long long* red = reinterpret_cast<long long*>(cs.slots);  // slots are free until the first window
        if ((t & 31) == 0) red[t >> 5] = part;
        group_sync(bar, NT);
        ChainScalars io{0, 0, kDigestSeed};
        for (int w = 0; w < NT / 32; ++w) io.cost += red[w];
        io.best = io.cost;
        group_sync(bar, NT);
        const NearSink sink{nullptr, a.near_k, a.near_dec, a.near_cap, a.near_count, a.near_chain,
                            a.chain_begin + (unsigned)ci};
        constexpr int QPT = NFIX ? quads_per_thread(NT, NFIX) : 0;
        const uint64_t acc = chain_run<TA, TB, NT, QPT>(As, cs, tb, n, ld, M, nqt, 0ull, a.iters, a.sch,
                                                   a.seed, a.chain_begin + (unsigned)ci, bar, t,
                                                   a.wmax, io, sink, a.proposal != 0);
        for (int i = t; i < n; i += NT) a.best_perms[(size_t)ci * n + i] = cs.best_p[i];
        if (t == scalar_tid(NT, n)) {
            ChainResult r;
            r.cost = io.cost;
            r.best_cost = io.best;
            r.accepted = acc;
            r.near_ties = (unsigned long long)cs.flags[1];
            r.digest = io.digest;
            r.iterations = a.iters;
            a.res[ci] = r;
        }
        group_sync(bar, NT);
    }
}

// Chain-keyed start permutations (R14b), one thread per chain:
// Fisher-Yates from the identity, for i = n-1 .. 1: j = floor(x (i+1) / 2^32) with
// x = Philox4x32-10(key = seed, ctr = (i, 0, chain, tag 1)).x, then swap p[i], p[j].
__global__ void k_start_perms(int n, unsigned long long seed, uint32_t chain_begin, int count, int32_t* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    int32_t* p = out + (size_t)c * n;
    for (int i = 0; i < n; ++i) p[i] = i;
    for (int i = n - 1; i >= 1; --i) {
        const U4 x = philox4x32_10((uint32_t)i, 0u, chain_begin + (uint32_t)c, 1u, (uint32_t)seed,
                                   (uint32_t)(seed >> 32));
        const int j = (int)(((uint64_t)x.x * (uint64_t)(i + 1)) >> 32);
        const int32_t t = p[i];
        p[i] = p[j];
        p[j] = t;
    }
}

// ChainResult / uint16 best permutation of every chain of a tensor-memory ensemble
__global__ void k_ens_collect(const DevState* __restrict__ st, const int32_t* __restrict__ best_p,
                              int count, int n, unsigned long long iters, ChainResult* res,
                              uint16_t* best_perms) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count * n; i += gridDim.x * blockDim.x)
        best_perms[i] = (uint16_t)best_p[i];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < count; c += gridDim.x * blockDim.x) {
        ChainResult r;
        r.cost = st[c].cost;
        r.best_cost = st[c].best_cost;
        r.accepted = st[c].accepted;
        r.near_ties = st[c].near_count;
        r.digest = st[c].digest;
        r.iterations = iters;
        res[c] = r;
    }
}

// argmin over chains of (best_cost, chain id) and summed statistics; 1 CTA.
__global__ void k_ens_reduce(const ChainResult* __restrict__ res, int count, long long* out /* 8 */) {
    __shared__ long long sbest[32];
    __shared__ int sidx[32];
    __shared__ unsigned long long sacc[32], snear[32], sdig[32];
    long long best = LLONG_MAX;
    int bi = INT_MAX;
    unsigned long long acc = 0, nr = 0, dg = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const ChainResult r = res[i];
        if (r.best_cost < best || (r.best_cost == best && i < bi)) { best = r.best_cost; bi = i; }
        acc += r.accepted;
        nr += r.near_ties;
        dg ^= r.digest;
    }
    for (int o = 16; o; o >>= 1) {
        const long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        nr += __shfl_xor_sync(0xffffffffu, nr, o);
        dg ^= __shfl_xor_sync(0xffffffffu, dg, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sbest[w] = best; sidx[w] = bi; sacc[w] = acc; snear[w] = nr; sdig[w] = dg; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            if (sbest[i] < best || (sbest[i] == best && sidx[i] < bi)) { best = sbest[i]; bi = sidx[i]; }
            acc += sacc[i];
            nr += snear[i];
            dg ^= sdig[i];
        }
        out[0] = best;
        out[1] = bi;
        out[2] = (long long)acc;
        out[3] = (long long)nr;
        out[4] = (long long)dg;
        out[5] = bi < count ? res[bi].cost : 0;
    }
}

}  // namespace qapsa
