// chain.cuh -- one Δ-matrix SA chain run by a group of NT threads that keeps
// its whole state in shared memory (Δ may instead live in global memory / L2).
//
// Per accepted swap (r,s) the group goes through two phases separated by
// named barriers ("a synchronization mechanism is needed"; the group is
// inside one CTA, so a hardware barrier suffices):
//   W  window: candidate k+o (o = window offset) is tested against Eq.(2)
//       by thread NT-1-o, with its Δ address and threshold
//      θ = -T ln r prepared off the critical path; a warp vote
//      (__ballot_sync) + cross-warp min picks the first accepted candidate
//      ("the swap which would have been found first").  Meanwhile the low
//      threads apply the previous accept's B' row/column exchange (Eq.(3),
//      P:90-94) and best_p copy.
//   SU stage+update (reads A and the PRE-swap B'; writes Δ):
//      touching entries: for every v != r,s the values δ''(r,v), δ''(s,v) of
//        the post-swap state from pre-swap rows (R10b), 4 lanes per v, 128-bit
//        loads and dp4a, written straight into Δ; diagonal D_v kept current;
//      disjoint entries: Δ_uv += 2(dA_u-dA_v)(dB_u-dB_v) (R10) in a padded quad
//        layout, one 128-bit load/store per 4 entries; every warp stages its own
//        copy of dA_x = a_xr - a_xs, dB_x = B'_xr - B'_xs;
//      p, C, best, digest; Δ_rs = -δ; next window's addresses and thresholds.
// A window without an accepted candidate costs one barrier.
//
// Δ quad layout: NQ = ceil(n/4); row u keeps the column quads
// j = floor((u+1)/4) .. NQ-1; quad g of the row-major sequence holds entries
// (u, 4j..4j+3) at D[4g..4g+3]; entry (u,v) is at rowaddr[u]+v.  Slots with
// v <= u or v >= n are dead (never read for a decision).  Rows of A and B'
// have stride ld (a multiple of 16 elements).
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "device_common.cuh"

namespace qapsa {

// staged (dA, dB): packed int16 pair when both matrices are 8-bit, else int2
template <typename TA, typename TB>
struct Dab {
    using T = int2;
    __device__ static T pack(int a, int b) { return make_int2(a, b); }
    __device__ static int rank(T pu, T pv) { return 2 * (pu.x - pv.x) * (pu.y - pv.y); }
    __device__ static void load4(const T* p, int v0, T out[4]) {
        const int4 x = *reinterpret_cast<const int4*>(p + v0);
        const int4 y = *reinterpret_cast<const int4*>(p + v0 + 2);
        out[0] = make_int2(x.x, x.y); out[1] = make_int2(x.z, x.w);
        out[2] = make_int2(y.x, y.y); out[3] = make_int2(y.z, y.w);
    }
};
template <>
struct Dab<uint8_t, uint8_t> {
    // value b * 2^16 + a as an integer (|a|, |b| < 2^15): the difference of two packed
    // values is the packed difference, so one IADD gives (au-av, bu-bv).
    using T = int;
    __device__ static T pack(int a, int b) { return (b << 16) + a; }
    __device__ static int rank(T pu, T pv) {       // 2 (au - av)(bu - bv)
        const int d = pu - pv;
        const int lo = (d << 16) >> 16;
        return lo * ((d - lo) >> 15);
    }
    __device__ static void load4(const T* p, int v0, T out[4]) {
        const int4 x = *reinterpret_cast<const int4*>(p + v0);
        out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
    }
};

template <typename TA, typename TB>
struct ChainSmem {
    TB* Bp;                            // n x ld, B'_ij = B_{p(i),p(j)}
    int32_t* D;                        // quad layout (shared or global memory)
    typename Dab<TA, TB>::T* dAB;      // n4: staged (dA_x, dB_x)
    int32_t* Dg;                       // n, diagonal D_x = sum_k A_xk B'_xk
    uint16_t* p;                       // n
    uint16_t* best_p;                  // n
    int4* slots;                       // 2 * NW window slots (double buffered)
    int* flags;                        // [0] improved, [1] near count, [2] chain id broadcast
};

struct ChainTables {                   // per instance, shared by all chains of a CTA
    const int32_t* rowaddr;            // n: address of entry (u,v) = rowaddr[u] + v
    const uint16_t* qdesc;             // nqt: u | (first column / 4) << 9   (n <= 512)
};

// number of Δ quads of the quad layout for problem size n
__host__ __device__ constexpr int quad_count(int n) {
    int c = 0;
    for (int u = 0; u + 1 < n; ++u) c += (n + 3) / 4 - (u + 1) / 4;
    return c;
}
// row stride: a multiple of 16 elements; for 8-bit rows an odd multiple when it fits, so
// that 8 rows read 16 bytes each at the same offset hit distinct banks (touching lanes).
__host__ __device__ constexpr int row_stride(int n, bool odd16) {
    const int m = (n + 15) / 16;
    return 16 * ((odd16 && !(m & 1)) ? m + 1 : m);
}
// Work split of a group of NT threads for problem size n: warps [0, TW) compute the
// touching entries (one lane per v); if the group has more warps, the others do the quads.
__host__ __device__ constexpr int touch_warps(int n) { return (n + 31) / 32; }
__host__ __device__ constexpr bool split_warps(int NT, int n) { return NT / 32 > touch_warps(n); }
__host__ __device__ constexpr int quad_lo(int NT, int n) { return split_warps(NT, n) ? 32 * touch_warps(n) : 0; }
__host__ __device__ constexpr int quads_per_thread(int NT, int n) {
    return (quad_count(n) + (NT - quad_lo(NT, n)) - 1) / (NT - quad_lo(NT, n));
}
// thread of a group that owns the scalar state (p swap, C, best, digest)
__host__ __device__ constexpr int scalar_tid(int NT, int n) {
    return split_warps(NT, n) ? quad_lo(NT, n) : NT / 2;
}

struct ChainScalars {  // meaningful in thread scalar_tid(NT, n) of the group
    int64_t cost;
    int64_t best;
    uint64_t digest;
};

// Near-tie sink (R16).  Single chain: count = the context's counter, log (ks, dec) indexed by it.
// Ensembles: count = the chain's own counter (or nullptr), lcount = the launch-wide log counter,
// and every entry also records the chain id, so a flagged chain can be followed by the oracle.
struct NearSink {
    unsigned int* count;
    unsigned long long* ks;
    unsigned char* dec;
    int cap;
    unsigned int* lcount;
    uint32_t* lchain;
    uint32_t chain;
};

// records near tie (k, decision) of a consumed iteration
__device__ __forceinline__ void near_record(const NearSink& s, uint64_t k, bool dec) {
    unsigned int e = 0;
    if (s.count) e = atomicAdd(s.count, 1u);
    if (s.lcount) e = atomicAdd(s.lcount, 1u);
    if (s.ks && (int)e < s.cap) {
        s.ks[e] = (unsigned long long)k;
        s.dec[e] = dec ? 1 : 0;
        if (s.lchain) s.lchain[e] = s.chain;
    }
}

__device__ __forceinline__ int round_up32(int x) { return (x + 31) & ~31; }

// (cur + step) mod M in 32-bit (step < 2^20)
__device__ __forceinline__ int advance_cursor(int cur, int step, int M) {
    int c = cur + step;
    if (c >= M) c = (c - M < M) ? c - M : c % M;
    return c;
}

// ---- touching dot products over 16-element blocks b = b0, b0+step, ... < nb
// X_r += B'_v . a_r, X_s += B'_v . a_s, Y_r += A_v . b'_r, Y_s += A_v . b'_s,
// Z_r += a_r . b'_s, Z_s += a_s . b'_r  (the last two do not depend on v)
template <typename TA, typename TB>
struct Dots {
    __device__ static void run(const TA* Av, const TB* Bv, const TA* Ar, const TA* As, const TB* Br,
                               const TB* Bs, int b0, int step, int nb, int& xr, int& xs, int& yr,
                               int& ys, int& zr, int& zs) {
        for (int b = b0; b < nb; b += step)
            for (int k = 16 * b; k < 16 * b + 16; ++k) {
                const int bv = Bv[k], av = Av[k];
                xr += bv * (int)Ar[k];
                xs += bv * (int)As[k];
                yr += av * (int)Br[k];
                ys += av * (int)Bs[k];
                zr += (int)Ar[k] * (int)Bs[k];
                zs += (int)As[k] * (int)Br[k];
            }
    }
    __device__ static int dot(const TA* X, const TB* Y, int b0, int step, int nb) {
        int acc = 0;
        for (int b = b0; b < nb; b += step)
            for (int k = 16 * b; k < 16 * b + 16; ++k) acc += (int)X[k] * (int)Y[k];
        return acc;
    }
};

__device__ __forceinline__ uint32_t dp16(const uint4 x, const uint4 y, uint32_t c) {
    return __dp4a(x.w, y.w, __dp4a(x.z, y.z, __dp4a(x.y, y.y, __dp4a(x.x, y.x, c))));
}

template <>
struct Dots<uint8_t, uint8_t> {
    __device__ static void run(const uint8_t* Av, const uint8_t* Bv, const uint8_t* Ar,
                               const uint8_t* As, const uint8_t* Br, const uint8_t* Bs, int b0,
                               int step, int nb, int& xr, int& xs, int& yr, int& ys, int& zr,
                               int& zs) {
        const uint4* av = reinterpret_cast<const uint4*>(Av);
        const uint4* bv = reinterpret_cast<const uint4*>(Bv);
        const uint4* ar = reinterpret_cast<const uint4*>(Ar);
        const uint4* as = reinterpret_cast<const uint4*>(As);
        const uint4* br = reinterpret_cast<const uint4*>(Br);
        const uint4* bs = reinterpret_cast<const uint4*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0, Zr = 0, Zs = 0;
#pragma unroll 2
        for (int b = b0; b < nb; b += step) {
            const uint4 a = av[b], bb = bv[b];
            const uint4 rA = ar[b], sA = as[b], rB = br[b], sB = bs[b];
            Xr = dp16(bb, rA, Xr);
            Xs = dp16(bb, sA, Xs);
            Yr = dp16(a, rB, Yr);
            Ys = dp16(a, sB, Ys);
            Zr = dp16(rA, sB, Zr);
            Zs = dp16(sA, rB, Zs);
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys; zr += (int)Zr; zs += (int)Zs;
    }
    __device__ static int dot(const uint8_t* X, const uint8_t* Y, int b0, int step, int nb) {
        const uint4* x = reinterpret_cast<const uint4*>(X);
        const uint4* y = reinterpret_cast<const uint4*>(Y);
        uint32_t acc = 0;
        for (int b = b0; b < nb; b += step) acc = dp16(x[b], y[b], acc);
        return (int)acc;
    }
};

// 16 bytes of 8-bit x (16 elements) against 32 bytes of 16-bit y
__device__ __forceinline__ uint32_t dp16w(const uint4 x, const uint4 y0, const uint4 y1, uint32_t c) {
    c = __dp2a_hi(y0.y, x.x, __dp2a_lo(y0.x, x.x, c));
    c = __dp2a_hi(y0.w, x.y, __dp2a_lo(y0.z, x.y, c));
    c = __dp2a_hi(y1.y, x.z, __dp2a_lo(y1.x, x.z, c));
    return __dp2a_hi(y1.w, x.w, __dp2a_lo(y1.z, x.w, c));
}

template <>
struct Dots<uint8_t, uint16_t> {
    __device__ static void run(const uint8_t* Av, const uint16_t* Bv, const uint8_t* Ar,
                               const uint8_t* As, const uint16_t* Br, const uint16_t* Bs, int b0,
                               int step, int nb, int& xr, int& xs, int& yr, int& ys, int& zr,
                               int& zs) {
        const uint4* av = reinterpret_cast<const uint4*>(Av);
        const uint4* bv = reinterpret_cast<const uint4*>(Bv);
        const uint4* ar = reinterpret_cast<const uint4*>(Ar);
        const uint4* as = reinterpret_cast<const uint4*>(As);
        const uint4* br = reinterpret_cast<const uint4*>(Br);
        const uint4* bs = reinterpret_cast<const uint4*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0, Zr = 0, Zs = 0;
        for (int b = b0; b < nb; b += step) {
            const uint4 a = av[b], b0w = bv[2 * b], b1w = bv[2 * b + 1];
            const uint4 r8 = ar[b], s8 = as[b];
            const uint4 R0 = br[2 * b], R1 = br[2 * b + 1], S0 = bs[2 * b], S1 = bs[2 * b + 1];
            Xr = dp16w(r8, b0w, b1w, Xr);
            Xs = dp16w(s8, b0w, b1w, Xs);
            Yr = dp16w(a, R0, R1, Yr);
            Ys = dp16w(a, S0, S1, Ys);
            Zr = dp16w(r8, S0, S1, Zr);
            Zs = dp16w(s8, R0, R1, Zs);
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys; zr += (int)Zr; zs += (int)Zs;
    }
    __device__ static int dot(const uint8_t* X, const uint16_t* Y, int b0, int step, int nb) {
        const uint4* x = reinterpret_cast<const uint4*>(X);
        const uint4* y = reinterpret_cast<const uint4*>(Y);
        uint32_t acc = 0;
        for (int b = b0; b < nb; b += step) acc = dp16w(x[b], y[2 * b], y[2 * b + 1], acc);
        return (int)acc;
    }
};

// producer/consumer hand-off of the staged dA/dB between touching and quad warps
__device__ __forceinline__ void stage_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void stage_wait(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Optional phase timers (debug build with -DQAPSA_PHASE_TIMERS, tools/phase_times.py):
// cycles spent by thread 0 of the group in W (accepting / non-accepting windows) and SU.
#ifdef QAPSA_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[128];
#define PT_COUNT(slot) atomicAdd(&g_phase_cycles[slot], 1ull)
// clock read that waits for `dep` (a shared-memory value read after a barrier): with
// BAR.SYNC.DEFER_BLOCKING a plain clock read would be issued before the barrier releases
__device__ __forceinline__ long long clock_after(int dep) {
    long long c;
    asm volatile("{\n\t.reg .b32 d;\n\tmov.b32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(dep) : "memory");
    return c;
}
#define PT_MARK(var) const long long var = clock64()
#define PT_MARKD(var, dep) const long long var = clock_after(dep)
#define PT_ADD(slot, a, b) if (t == 0) atomicAdd(&g_phase_cycles[slot], (unsigned long long)((b) - (a)))
#define PT_ADDT(tid, slot, a) if (t == (tid)) atomicAdd(&g_phase_cycles[slot], (unsigned long long)(clock64() - (a)))
#else
#define PT_ADDT(tid, slot, a)
#define PT_MARK(var)
#define PT_COUNT(slot)
#define PT_MARKD(var, dep)
#define PT_ADD(slot, a, b)
#endif

// A candidate prepared ahead of its window: where its δ lives and its threshold.
struct Prep {
    uint64_t k;       // iteration the preparation is for (~0 = none)
    int addr;         // Δ address of its pair
    int rs;           // r << 16 | s
    float th, m;      // θ = -T ln r (float) and the margin that brackets float error
};

// Address part of a preparation: candidate of iteration kk, pair index q.
__device__ __forceinline__ void prepare_addr(Prep& pr, int n, const int32_t* rowaddr, int q,
                                             uint64_t kk) {
    int r, s;
    tri_pair(n, q, &r, &s);
    pr.k = kk;
    pr.addr = rowaddr[r] + s;
    pr.rs = (r << 16) | s;
    pr.th = -1.0f;                                 // threshold not computed
}
// Threshold part: θ = -T_k ln r_k in float and its margin.
__device__ __forceinline__ void prepare_theta(Prep& pr, const Sched& sch, uint64_t seed,
                                              uint32_t chain) {
    const uint64_t kk = pr.k;
    const U4 x = philox4x32_10((uint32_t)kk, (uint32_t)(kk >> 32), chain, 0u, (uint32_t)seed,
                               (uint32_t)(seed >> 32));
    const uint64_t bits = ((uint64_t)x.y << 32) | (uint64_t)x.x;
    const float rf = (__ull2float_rn(bits >> 11) + 0.5f) * 0x1p-53f;   // r_k of R3 in float (> 0)
    const float T = temp32(sch, kk);
    pr.th = T * -__logf(rf);                                   // >= 0
    pr.m = 2e-4f * pr.th + 2e-5f * T;
}

// Pair index proposed at iteration kk: the sequential enumeration (R4: cursor + offset) or,
// with random proposals (R22), floor(x M / 2^32) with x = Philox(seed; kk, chain, tag 3).x
__device__ __forceinline__ int proposal_index(bool rnd, int cur, int off, int M, uint64_t kk,
                                              uint64_t seed, uint32_t chain) {
    if (!rnd) return advance_cursor(cur, off, M);
    const U4 x = philox4x32_10((uint32_t)kk, (uint32_t)(kk >> 32), chain, 3u, (uint32_t)seed,
                               (uint32_t)(seed >> 32));
    return (int)(((uint64_t)x.x * (uint64_t)M) >> 32);
}

// Runs iterations [k0, k_end) of one chain.  Returns the number of accepted
// swaps (identical in every thread of the group).  QPT > 0: the thread's quads
// are fixed at compile time (g = t - quad_lo + i * (NT - quad_lo), i < QPT).
template <typename TA, typename TB, int NT, int QPT>
__device__ __forceinline__ uint64_t chain_run(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                              const ChainTables tb, const int n, const int ld,
                                              const int M, const int nqt,
                                              const uint64_t k0, const uint64_t k_end,
                                              const Sched sch, const uint64_t seed,
                                              const uint32_t chain, const int bar_id, const int t,
                                              const int wmax, ChainScalars& io,
                                              const NearSink sink, const bool rnd = false) {
    using DB = Dab<TA, TB>;
    using DT = typename DB::T;
    constexpr int NW = NT / 32;
    const int lane = t & 31, warp = t >> 5;
    const int nb = ld >> 4;                        // 16-element blocks per row
    const int off = NT - 1 - t;                    // this thread's window offset (quad warps first)
    const int TW = touch_warps(n);
    const bool split = split_warps(NT, n);
    const int qlo = quad_lo(NT, n), QT = NT - qlo;
    const bool scalar_thread = t == scalar_tid(NT, n);
    const int stage_bar = bar_id + 1;              // named barrier of the staging hand-off

    // quads owned by this thread (compile-time count when QPT > 0)
    uint32_t qd[QPT > 0 ? QPT : 1];
#pragma unroll
    for (int i = 0; i < (QPT > 0 ? QPT : 0); ++i) {
        const int g = t - qlo + i * QT;
        qd[i] = (t >= qlo && g < nqt) ? tb.qdesc[g] : 0xFFFFFFFFu;
    }

    uint64_t k = k0, accepted = 0;
    int cur = (int)(k0 % (uint64_t)M);
    int W = wmax;
    int parity = 0;
    bool streak = false;                           // previous window accepted nothing
    float rejT = 38.5f * temp32(sch, k0);          // certain-reject bound of the current window
    int pend_r = -1, pend_s = -1;                  // B' exchange still to apply
    Prep pre;
    pre.k = ~0ull;
#ifdef QAPSA_PHASE_TIMERS
    long long su_start = 0;
#endif

    while (k < k_end) {
#ifdef QAPSA_PHASE_TIMERS
        PT_MARKD(pt0, cs.flags[3]);
        if (!streak && k != k0) PT_ADD(2, su_start, pt0);   // SU of the previous accept, barrier included
#endif
        const uint64_t remaining = k_end - k;
        const int Wl = (uint64_t)W < remaining ? W : (int)remaining;

        // ---------------- W: window of candidates (+ deferred B' exchange) ----------------
        if (pend_r >= 0) {
            const int r = pend_r, s = pend_s;
            for (int x = t; x < n; x += NT) {     // columns r,s of every other row (low threads)
                if (x == r || x == s) continue;
                TB* row = cs.Bp + x * ld;
                const TB br = row[r];
                row[r] = row[s];
                row[s] = br;
            }
            if (warp == 0) {                      // rows r,s, word-wise
                constexpr int EPW = 4 / sizeof(TB);
                constexpr uint32_t EMASK = sizeof(TB) == 1 ? 0xFFu : 0xFFFFu;
                uint32_t* Rw = reinterpret_cast<uint32_t*>(cs.Bp + r * ld);
                uint32_t* Sw = reinterpret_cast<uint32_t*>(cs.Bp + s * ld);
                for (int w = lane; w < ld / EPW; w += 32) {
                    uint32_t m = 0;
                    if (r / EPW == w) m |= EMASK << (8 * sizeof(TB) * (r % EPW));
                    if (s / EPW == w) m |= EMASK << (8 * sizeof(TB) * (s % EPW));
                    const uint32_t a = Rw[w], b = Sw[w];
                    Rw[w] = (b & ~m) | (a & m);   // rows exchange; (r,r),(r,s),(s,r),(s,s) keep
                    Sw[w] = (a & ~m) | (b & m);   // their values (B' symmetric, zero diagonal)
                }
            }
            if (cs.flags[0])
                for (int x = t; x < n; x += NT) cs.best_p[x] = cs.p[x];
            pend_r = -1;
#ifdef QAPSA_PHASE_TIMERS
            if (t == NT - 1) atomicAdd(&g_phase_cycles[7], (unsigned long long)(clock_after(cs.Bp[s]) - pt0));
#endif
        }
        bool acc = false, near = false;
        int d = 0;
        if (off < Wl) {
            const uint64_t kk = k + (uint64_t)off;
#ifdef QAPSA_PHASE_TIMERS
            if (t == 0 && !streak) atomicAdd(&g_phase_cycles[11], (unsigned long long)(clock_after((int)pre.k + Wl) - pt0));
#endif
            if (pre.k != kk) { PT_COUNT(8); prepare_addr(pre, n, tb.rowaddr, proposal_index(rnd, cur, off, M, kk, seed, chain), kk); }
            d = cs.D[pre.addr];
            if (d <= 0) {
                acc = true;                       // δ < 0, or δ = 0: exp(0) = 1 > r (R5)
            } else if ((float)d <= rejT) {
                // else certain reject: δ > 38.5 T32(k) >= 38.4 T_kk => exp(-δ/T) < 2^-54 <= r
                if (pre.th < 0.0f) { PT_COUNT(9); prepare_theta(pre, sch, seed, chain); }
                const float df = (float)d;
                if (df < pre.th - pre.m) {
                    acc = true;                   // clearly below θ
                } else if (!(df > pre.th + pre.m)) {   // inside the margin: exact double test (R16)
                    PT_COUNT(10);
                    acc = metropolis(d, temperature(sch, kk), uniform_r(seed, kk, chain), &near);
                }
            }
        }
#ifdef QAPSA_PHASE_TIMERS
        if (t == NT - 1 && !streak) atomicAdd(&g_phase_cycles[6], (unsigned long long)(clock_after(d + (int)acc) - pt0));
#endif
        int4* slots = cs.slots + parity * NW;
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        if (bal) {                                // smallest offset = highest accepting lane
            if (lane == 31 - __clz(bal)) slots[warp] = make_int4(off, d, pre.rs, 0);
        } else if (lane == 0) {
            slots[warp] = make_int4(INT_MAX, 0, 0, 0);
        }
        // in a run of windows without accepts, prepare the next window's addresses now
        const int Wn = min(2 * W, wmax);
        if (streak && off < Wn && (uint64_t)(Wl + off) < remaining)
            prepare_addr(pre, n, tb.rowaddr, proposal_index(rnd, cur, Wl + off, M, k + (uint64_t)(Wl + off), seed, chain),
                         k + (uint64_t)(Wl + off));
        group_sync(bar_id, NT);
        const int tv = lane < NW ? slots[lane].x : INT_MAX;
        PT_MARKD(pt1, tv);
        const int j = __reduce_min_sync(0xffffffffu, tv);
        parity ^= 1;
        const int consumed = (j == INT_MAX) ? Wl : j + 1;
        if (near && off < consumed) {             // R16: count / log near ties of consumed iterations
            atomicAdd(&cs.flags[1], 1);
            near_record(sink, k + (uint64_t)off, acc);
        }
        if (j == INT_MAX) {                       // no accepted swap in the window
            PT_ADD(1, pt0, pt1);
            PT_ADD(5, 0, 1);
            k += (uint64_t)consumed;
            cur = advance_cursor(cur, consumed, M);
            W = Wn;
            rejT = 38.5f * temp32(sch, k);
            streak = true;
            continue;
        }
        streak = false;
        const int4 win = slots[(NT - 1 - j) >> 5];   // (offset, δ, r<<16|s) of the first accept
        const int dw = win.y, r = win.z >> 16, s = win.z & 0xFFFF;
#ifdef QAPSA_PHASE_TIMERS

#endif
        const uint64_t kacc = k + (uint64_t)j;
        const int Wnext = max(64, min(wmax, round_up32(8 * (j + 1))));

        // ---------------- SU: touching values, disjoint quads, scalars (B' read-only) ----------------
        {
            const TA* Ar = A + r * ld;
            const TA* As = A + s * ld;
            const TB* Br = cs.Bp + r * ld;
            const TB* Bs = cs.Bp + s * ld;
            const int ars = Ar[s], brs = Br[s];
            // -- touching entries (rows / columns r and s): one lane per v --
            if (!split || warp < TW) {
                const int vmin = r != 0 ? 0 : (s != 1 ? 1 : 2);
                for (int vb = 0; vb < n; vb += 32 * (split ? TW : NW)) {
                    const int v = vb + 32 * warp + lane;
                    const bool act = v < n && v != r && v != s;
                    int arv = 0, asv = 0, brv = 0, bsv = 0, da = 0, db = 0;
                    if (act) {                        // staging, handed to the quad warps
                        arv = Ar[v]; asv = As[v]; brv = Br[v]; bsv = Bs[v];
                        da = arv - asv;               // dA_v = a_vr - a_vs
                        db = brv - bsv;               // dB_v = B'_vr - B'_vs (pre-swap)
                        cs.dAB[v] = DB::pack(da, db);
#ifdef QAPSA_PHASE_TIMERS

#endif
                    }
                    if (split && vb == 0) stage_arrive(stage_bar, NT);
                    if (act) {
                        int xr = 0, xs = 0, yr = 0, ys = 0, zr = 0, zs = 0;
                        Dots<TA, TB>::run(A + v * ld, cs.Bp + v * ld, Ar, As, Br, Bs, 0, 1, nb, xr, xs,
                                          yr, ys, zr, zs);
#ifdef QAPSA_PHASE_TIMERS
                        if (t == 0) atomicAdd(&g_phase_cycles[12], (unsigned long long)(clock_after(xr + ys + zr) - pt1));
#endif
                        const int Dr = zr + ars * brs;        // D''_r = a_r.b'_s + a_rs B'_rs
                        const int Ds = zs + ars * brs;        // D''_s = a_s.b'_r + a_rs B'_rs
                        const int dv = cs.Dg[v] - da * db;    // D''_v = D_v - dA_v dB_v
                        cs.Dg[v] = dv;
                        // R10b: δ''(r,v) and δ''(s,v) from pre-swap rows
                        cs.D[v > r ? tb.rowaddr[r] + v : tb.rowaddr[v] + r] =
                            2 * (xr + ars * db + ys - da * brs - Dr - dv + 2 * arv * bsv);
                        cs.D[v > s ? tb.rowaddr[s] + v : tb.rowaddr[v] + s] =
                            2 * (xs - ars * db + yr + da * brs - Ds - dv + 2 * asv * brv);
                        if (v == vmin) {
                            cs.Dg[r] = Dr;
                            cs.Dg[s] = Ds;
                        }
                    }
                }
            }
            // -- disjoint entries: every quad of a row u != r,s --
            if (!split || warp >= TW) {
                if (split) stage_wait(stage_bar, NT);
                else group_sync(stage_bar, NT);
#ifdef QAPSA_PHASE_TIMERS
                if (t == qlo) atomicAdd(&g_phase_cycles[3], (unsigned long long)(clock_after(cs.flags[3]) - pt1));
#endif
                const DT* stg = cs.dAB;
                auto quad = [&](const uint32_t desc, const int g) {
                    const int u = desc & 511, v0 = (desc >> 9) << 2;
                    if (u == r || u == s) return;     // rows r, s: touching lanes
                    const int4 d4 = *reinterpret_cast<const int4*>(cs.D + 4 * g);
                    const DT pu = stg[u];
                    DT pv[4];
                    DB::load4(stg, v0, pv);
                    const int4 nv = make_int4(d4.x + DB::rank(pu, pv[0]), d4.y + DB::rank(pu, pv[1]),
                                              d4.z + DB::rank(pu, pv[2]), d4.w + DB::rank(pu, pv[3]));
                    const unsigned er = (unsigned)(r - v0), es = (unsigned)(s - v0);
                    if (er < 4u || es < 4u) {         // columns r/s belong to the touching lanes
                        if (er != 0u && es != 0u) cs.D[4 * g + 0] = nv.x;
                        if (er != 1u && es != 1u) cs.D[4 * g + 1] = nv.y;
                        if (er != 2u && es != 2u) cs.D[4 * g + 2] = nv.z;
                        if (er != 3u && es != 3u) cs.D[4 * g + 3] = nv.w;
                    } else {
                        *reinterpret_cast<int4*>(cs.D + 4 * g) = nv;
                    }
                };
                if (QPT > 0) {
                    // all loads of this thread's quads first, then the arithmetic and stores
                    constexpr int QP = QPT > 0 ? QPT : 1;
                    int4 d4[QP];
                    DT pu[QP], pv[QP][4];
                    int gq[QP], v0q[QP];
                    bool stq[QP];
#pragma unroll
                    for (int i = 0; i < QP; ++i) {
                        const uint32_t desc = qd[i];
                        const bool valid = desc != 0xFFFFFFFFu;
                        const int u = valid ? (int)(desc & 511) : 0;
                        v0q[i] = valid ? (int)((desc >> 9) << 2) : 0;
                        gq[i] = valid ? t - qlo + i * QT : 0;
                        stq[i] = valid && u != r && u != s;        // rows r, s: touching lanes
                        d4[i] = *reinterpret_cast<const int4*>(cs.D + 4 * gq[i]);
                        pu[i] = stg[u];
                        DB::load4(stg, v0q[i], pv[i]);
                    }
#pragma unroll
                    for (int i = 0; i < QP; ++i) {
                        const int4 nv = make_int4(d4[i].x + DB::rank(pu[i], pv[i][0]),
                                                  d4[i].y + DB::rank(pu[i], pv[i][1]),
                                                  d4[i].z + DB::rank(pu[i], pv[i][2]),
                                                  d4[i].w + DB::rank(pu[i], pv[i][3]));
                        const unsigned er = (unsigned)(r - v0q[i]), es = (unsigned)(s - v0q[i]);
                        const int g = gq[i];
                        if (stq[i] && er >= 4u && es >= 4u) {
                            *reinterpret_cast<int4*>(cs.D + 4 * g) = nv;
                        } else if (stq[i]) {          // columns r/s belong to the touching lanes
                            if (er != 0u && es != 0u) cs.D[4 * g + 0] = nv.x;
                            if (er != 1u && es != 1u) cs.D[4 * g + 1] = nv.y;
                            if (er != 2u && es != 2u) cs.D[4 * g + 2] = nv.z;
                            if (er != 3u && es != 3u) cs.D[4 * g + 3] = nv.w;
                        }
                    }
                } else {
                    for (int g = t - qlo; g < nqt; g += QT) quad(tb.qdesc[g], g);
                }
            }
            // address and threshold of this thread's candidate in the next window
            // (the window lanes are the last warps: quad warps, after their quads)
            if (off < Wnext && kacc + 1 + (uint64_t)off < k_end) {
                prepare_addr(pre, n, tb.rowaddr,
                             proposal_index(rnd, cur, j + 1 + off, M, kacc + 1 + (uint64_t)off, seed, chain),
                             kacc + 1 + (uint64_t)off);
                prepare_theta(pre, sch, seed, chain);
            }
#ifdef QAPSA_PHASE_TIMERS
            if (t == 0) atomicAdd(&g_phase_cycles[13], (unsigned long long)(clock_after((int)pre.th) - pt1));
            if (t == qlo) atomicAdd(&g_phase_cycles[14], (unsigned long long)(clock_after(cs.D[4 * (t - qlo)]) - pt1));
            if (t == NT - 1) atomicAdd(&g_phase_cycles[15], (unsigned long long)(clock_after(cs.D[4 * (t - qlo)]) - pt1));
#endif
            if (scalar_thread) {                  // scalar state: p, C, best, digest, Δ_rs
                const uint16_t pr = cs.p[r];
                cs.p[r] = cs.p[s];
                cs.p[s] = pr;
                io.cost += dw;
                const int improved = io.cost < io.best;
                if (improved) io.best = io.cost;
                cs.flags[0] = improved;
                io.digest = digest_step(io.digest, kacc, r, s);
                cs.D[tb.rowaddr[r] + s] = -dw;    // swapping back restores C
                if (n < 3) {                      // no touching lane: diagonal of rows r,s here
                    cs.Dg[r] = Dots<TA, TB>::dot(Ar, Bs, 0, 1, nb) + ars * brs;
                    cs.Dg[s] = Dots<TA, TB>::dot(As, Br, 0, 1, nb) + ars * brs;
                }
            }
        }
        pend_r = r;
        pend_s = s;
        group_sync(bar_id, NT);
        PT_ADD(0, pt0, pt1);
        PT_ADD(4, 0, 1);
#ifdef QAPSA_PHASE_TIMERS
        su_start = pt1;
#endif

        ++accepted;
        k = kacc + 1;
        cur = advance_cursor(cur, j + 1, M);
        W = Wnext;
        rejT = 38.5f * temp32(sch, k);
    }
    // the B' exchange of the last accept is not needed (B' is rebuilt from p at the next
    // launch); its best_p copy is
    if (pend_r >= 0 && cs.flags[0])
        for (int x = t; x < n; x += NT) cs.best_p[x] = cs.p[x];
    return accepted;
}

// Δ for all pairs of the current (smem) B', by the group: step (a) of P:46.
// δ(r,s) = 2 [ sum_all k (a_rk - a_sk)(B'_sk - B'_rk) + 2 a_rs B'_rs ]
template <typename TA, typename TB, int NT>
__device__ __forceinline__ void chain_delta_init(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                                 const ChainTables tb, int n, int ld, int M, int t) {
    for (int q = t; q < M; q += NT) {
        int r, s;
        tri_pair(n, q, &r, &s);
        const TA* Ar = A + r * ld;
        const TA* As = A + s * ld;
        const TB* Br = cs.Bp + r * ld;
        const TB* Bs = cs.Bp + s * ld;
        int acc = 0;
        for (int k = 0; k < n; ++k) acc += ((int)Ar[k] - (int)As[k]) * ((int)Bs[k] - (int)Br[k]);
        cs.D[tb.rowaddr[r] + s] = 2 * (acc + 2 * (int)Ar[s] * (int)Br[s]);
    }
}

// D_x = sum_k A_xk B'_xk for all x (the diagonal of A B'^T)
template <typename TA, typename TB, int NT>
__device__ __forceinline__ void chain_diag_init(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                                int n, int ld, int t) {
    for (int x = t; x < n; x += NT) cs.Dg[x] = Dots<TA, TB>::dot(A + x * ld, cs.Bp + x * ld, 0, 1, ld >> 4);
}

}  // namespace qapsa
