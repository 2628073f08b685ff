// chain.cuh -- one Δ-matrix SA chain run by a group of NT threads that keeps
// its whole state in shared memory (Δ may instead live in global memory / L2).
//
// Per accepted swap (r,s) the group goes through three phases separated by
// named barriers ("a synchronization mechanism is needed"; the group is
// inside one CTA, so a hardware barrier suffices):
//   W  window: thread t tests candidate k+t against Eq.(2) with an
//      address and a threshold θ = -T ln r prepared off the critical path
//      (in U of the previous accept, or speculatively in the previous window);
//      warp vote (__ballot_sync/__ffs) + cross-warp min picks the first
//      accepted candidate ("the swap which would have been found first");
//   S  stage (reads A, B' only): for every v != r,s the touching values
//      δ'(r,v), δ'(s,v) of the POST-swap state from PRE-swap rows (R10b),
//      4 lanes per v, 128-bit loads, dp4a; dA_v = a_vr - a_vs,
//      dB_v = B'_vr - B'_vs; diagonal D_v = A_v . B'_v kept
//      current; p, C, best, digest;
//   U  update (writes Δ and B'): Δ in a padded "quad" layout so every thread
//      updates 4 entries with one 128-bit load/store: disjoint entries
//      Δ_uv += 2(dA_u-dA_v)(dB_u-dB_v) (R10), touching entries take the
//      staged values, Δ_rs = -δ; B' rows/columns r,s exchanged (Eq.(3),
//      P:90-94); the next window's addresses and thresholds are prepared.
// A window without an accepted candidate costs one barrier.
//
// Δ quad layout: NQ = ceil(n/4); row u keeps the
// column quads j = floor((u+1)/4) .. NQ-1; quad g of the row-major sequence
// holds entries (u, 4j..4j+3) at D[4g..4g+3]; entry (u,v) is at rowaddr[u]+v.
// Slots with v <= u or v >= n are dead (never read for a decision).
// Rows of A and B' have stride ld (a multiple of 16 elements).
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
    typename Dab<TA, TB>::T* dAB;      // n4, staged (dA_x, dB_x)
    int32_t* Dg;                       // n, diagonal D_x = sum_k A_xk B'_xk
    int32_t* Tr;                       // n4, staged δ'(r,v) + 2 D'_r
    int32_t* Ts;                       // n4, staged δ'(s,v) + 2 D'_s
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
// that 8 rows read 16 bytes each at the same offset hit distinct banks (phase S).
__host__ __device__ constexpr int row_stride(int n, bool odd16) {
    const int m = (n + 15) / 16;
    return 16 * ((odd16 && !(m & 1)) ? m + 1 : m);
}

// thread of a group that owns the scalar state (p swap, C, best, digest): lane 0 of
// the third-to-last warp (idle in phase S when the group has spare warps)
__host__ __device__ constexpr int scalar_tid(int NT) { return NT >= 96 ? NT - 96 : 0; }

struct ChainScalars {  // meaningful in thread scalar_tid(NT) of the group
    int64_t cost;
    int64_t best;
    uint64_t digest;
};

struct NearSink {      // global near-tie log (single chain) or nullptr
    unsigned int* count;
    unsigned long long* ks;
    unsigned char* dec;
    int cap;
};

__device__ __forceinline__ int round_up32(int x) { return (x + 31) & ~31; }

// (cur + step) mod M in 32-bit (step < 2^20)
__device__ __forceinline__ int advance_cursor(int cur, int step, int M) {
    int c = cur + step;
    if (c >= M) c = (c - M < M) ? c - M : c % M;
    return c;
}

// ---- touching dot products over 16-element blocks b = b0, b0+step, ... < nb
// X_r += B'_v . a_r, X_s += B'_v . a_s, Y_r += A_v . b'_r, Y_s += A_v . b'_s
template <typename TA, typename TB>
struct Dots {
    __device__ static void run(const TA* Av, const TB* Bv, const TA* Ar, const TA* As, const TB* Br,
                               const TB* Bs, int b0, int step, int nb, int& xr, int& xs, int& yr,
                               int& ys) {
        for (int b = b0; b < nb; b += step)
            for (int k = 16 * b; k < 16 * b + 16; ++k) {
                const int bv = Bv[k], av = Av[k];
                xr += bv * (int)Ar[k];
                xs += bv * (int)As[k];
                yr += av * (int)Br[k];
                ys += av * (int)Bs[k];
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
                               int step, int nb, int& xr, int& xs, int& yr, int& ys) {
        const uint4* av = reinterpret_cast<const uint4*>(Av);
        const uint4* bv = reinterpret_cast<const uint4*>(Bv);
        const uint4* ar = reinterpret_cast<const uint4*>(Ar);
        const uint4* as = reinterpret_cast<const uint4*>(As);
        const uint4* br = reinterpret_cast<const uint4*>(Br);
        const uint4* bs = reinterpret_cast<const uint4*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0;
#pragma unroll 2
        for (int b = b0; b < nb; b += step) {
            const uint4 a = av[b], bb = bv[b];
            Xr = dp16(bb, ar[b], Xr);
            Xs = dp16(bb, as[b], Xs);
            Yr = dp16(a, br[b], Yr);
            Ys = dp16(a, bs[b], Ys);
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys;
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
                               int step, int nb, int& xr, int& xs, int& yr, int& ys) {
        const uint4* av = reinterpret_cast<const uint4*>(Av);
        const uint4* bv = reinterpret_cast<const uint4*>(Bv);
        const uint4* ar = reinterpret_cast<const uint4*>(Ar);
        const uint4* as = reinterpret_cast<const uint4*>(As);
        const uint4* br = reinterpret_cast<const uint4*>(Br);
        const uint4* bs = reinterpret_cast<const uint4*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0;
        for (int b = b0; b < nb; b += step) {
            const uint4 a = av[b], b0w = bv[2 * b], b1w = bv[2 * b + 1];
            const uint4 r8 = ar[b], s8 = as[b];
            Xr = dp16w(r8, b0w, b1w, Xr);
            Xs = dp16w(s8, b0w, b1w, Xs);
            Yr = dp16w(a, br[2 * b], br[2 * b + 1], Yr);
            Ys = dp16w(a, bs[2 * b], bs[2 * b + 1], Ys);
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys;
    }
    __device__ static int dot(const uint8_t* X, const uint16_t* Y, int b0, int step, int nb) {
        const uint4* x = reinterpret_cast<const uint4*>(X);
        const uint4* y = reinterpret_cast<const uint4*>(Y);
        uint32_t acc = 0;
        for (int b = b0; b < nb; b += step) acc = dp16w(x[b], y[2 * b], y[2 * b + 1], acc);
        return (int)acc;
    }
};

constexpr int kTouchLanes = 4;   // lanes per touching v in phase S (lane = pl * 8 + v_local)

// Optional phase timers (debug build with -DQAPSA_PHASE_TIMERS, tools/phase_times.py):
// cycles spent by thread 0 of the group in W (accepting / non-accepting windows), S, U.
#ifdef QAPSA_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[8];
#define PT_MARK(var) const long long var = clock64()
#define PT_ADD(slot, a, b) if (t == 0) atomicAdd(&g_phase_cycles[slot], (unsigned long long)((b) - (a)))
#else
#define PT_MARK(var)
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
    const float rf = __ull2float_rn(bits >> 11) * 0x1p-53f;   // r_k in float (> 0)
    const float T = temp32(sch, kk);
    pr.th = T * -__logf(rf);                                   // >= 0
    pr.m = 2e-4f * pr.th + 2e-5f * T;
}

// Runs iterations [k0, k_end) of one chain.  Returns the number of accepted
// swaps (identical in every thread of the group).  QPT > 0: the thread's quads
// (g = t + i NT, i < QPT) are fixed at compile time.
template <typename TA, typename TB, int NT, int QPT>
__device__ __forceinline__ uint64_t chain_run(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                              const ChainTables tb, const int n, const int ld,
                                              const int M, const int nqt,
                                              const uint64_t k0, const uint64_t k_end,
                                              const Sched sch, const uint64_t seed,
                                              const uint32_t chain, const int bar_id, const int t,
                                              const int wmax, ChainScalars& io,
                                              const NearSink sink) {
    using DB = Dab<TA, TB>;
    using DT = typename DB::T;
    constexpr int NW = NT / 32;
    constexpr int TP = kTouchLanes;
    const int lane = t & 31, warp = t >> 5;
    const int nb = ld >> 4;                    // 16-element blocks per row
    // extra tasks of phase S go to the last warps (idle when NW > ceil(n/8) + 2)
    const int w_dr = NW - 1, w_ds = NW >= 2 ? NW - 2 : 0;
    const bool scalar_thread = t == scalar_tid(NT);

    // quads owned by this thread (compile-time count when QPT > 0)
    uint32_t qd[QPT > 0 ? QPT : 1];
#pragma unroll
    for (int i = 0; i < (QPT > 0 ? QPT : 0); ++i) {
        const int g = t + i * NT;
        qd[i] = g < nqt ? tb.qdesc[g] : 0xFFFFFFFFu;
    }

    uint64_t k = k0, accepted = 0;
    int cur = (int)(k0 % (uint64_t)M);
    int W = wmax;
    int parity = 0;
    bool streak = false;                       // previous window accepted nothing
    Prep pre;
    pre.k = ~0ull;

    while (k < k_end) {
        PT_MARK(pt0);
        const uint64_t remaining = k_end - k;
        const int Wl = (uint64_t)W < remaining ? W : (int)remaining;

        // ---------------- W: window of candidates ----------------
        bool acc = false, near = false;
        int d = 0;
        if (t < Wl) {
            const uint64_t kk = k + (uint64_t)t;
            if (pre.k != kk) prepare_addr(pre, n, tb.rowaddr, advance_cursor(cur, t, M), kk);
            d = cs.D[pre.addr];
            if (d <= 0) {
                acc = true;                       // δ < 0, or δ = 0: exp(0) = 1 > r (R5)
            } else if ((float)d <= 38.5f * temp32(sch, k)) {
                // else certain reject: δ > 38.5 T32(k) >= 38.4 T_kk => exp(-δ/T) < 2^-54 <= r
                if (pre.th < 0.0f) prepare_theta(pre, sch, seed, chain);
                const float df = (float)d;
                if (df < pre.th - pre.m) {
                    acc = true;                   // clearly below θ
                } else if (!(df > pre.th + pre.m)) {   // inside the margin: exact double test (R16)
                    acc = metropolis(d, temperature(sch, kk), uniform_r(seed, kk, chain), &near);
                }
            }
        }
        int4* slots = cs.slots + parity * NW;
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        if (bal) {
            if (lane == __ffs(bal) - 1) slots[warp] = make_int4(t, d, pre.rs, 0);
        } else if (lane == 0) {
            slots[warp] = make_int4(INT_MAX, 0, 0, 0);
        }
        // in a run of windows without accepts, prepare the next window's addresses now
        const int Wn = min(2 * W, wmax);
        if (streak && t < Wn && (uint64_t)(Wl + t) < remaining)
            prepare_addr(pre, n, tb.rowaddr, advance_cursor(cur, Wl + t, M), k + (uint64_t)(Wl + t));
        group_sync(bar_id, NT);
        PT_MARK(pt1);
        const int tv = lane < NW ? slots[lane].x : INT_MAX;
        const int j = __reduce_min_sync(0xffffffffu, tv);
        parity ^= 1;
        const int consumed = (j == INT_MAX) ? Wl : j + 1;
        if (near && t < consumed) {               // R16: count / log near ties of consumed iterations
            atomicAdd(&cs.flags[1], 1);
            if (sink.count) {
                const unsigned int i = atomicAdd(sink.count, 1u);
                if ((int)i < sink.cap) {
                    sink.ks[i] = (unsigned long long)(k + (uint64_t)t);
                    sink.dec[i] = acc ? 1 : 0;
                }
            }
        }
        if (j == INT_MAX) {                       // no accepted swap in the window
            PT_ADD(1, pt0, pt1);
            PT_ADD(5, 0, 1);
            k += (uint64_t)consumed;
            cur = advance_cursor(cur, consumed, M);
            W = Wn;
            streak = true;
            continue;
        }
        streak = false;
        const int4 win = slots[(j >> 5)];         // (t, δ, r<<16|s) of the first accepted candidate
        const int dw = win.y, r = win.z >> 16, s = win.z & 0xFFFF;
        const uint64_t kacc = k + (uint64_t)j;

        // ---------------- S: stage touching values, dA/dB, diagonal (reads A, B') ----------------
        {
            const TA* Ar = A + r * ld;
            const TA* As = A + s * ld;
            const TB* Br = cs.Bp + r * ld;
            const TB* Bs = cs.Bp + s * ld;
            const int ars = Ar[s], brs = Br[s];
            const int vl = lane & 7, pl = lane >> 3;
            for (int vb = 0; vb < n; vb += 8 * NW) {
                const int v = vb + 8 * warp + vl;
                const bool act = v < n && v != r && v != s;
                int arv = 0, asv = 0, brv = 0, bsv = 0, dgv = 0;
                if (act && pl == 0) {
                    arv = Ar[v]; asv = As[v]; brv = Br[v]; bsv = Bs[v]; dgv = cs.Dg[v];
                }
                int xr = 0, xs = 0, yr = 0, ys = 0;
                if (act)
                    Dots<TA, TB>::run(A + v * ld, cs.Bp + v * ld, Ar, As, Br, Bs, pl, TP, nb, xr, xs,
                                      yr, ys);
#pragma unroll
                for (int o = 8; o < 32; o <<= 1) {
                    xr += __shfl_xor_sync(0xffffffffu, xr, o);
                    xs += __shfl_xor_sync(0xffffffffu, xs, o);
                    yr += __shfl_xor_sync(0xffffffffu, yr, o);
                    ys += __shfl_xor_sync(0xffffffffu, ys, o);
                }
                if (act && pl == 0) {
                    const int da = arv - asv;             // dA_v = a_vr - a_vs
                    const int db = brv - bsv;             // dB_v = B'_vr - B'_vs (pre-swap)
                    cs.dAB[v] = DB::pack(da, db);
                    const int dv = dgv - da * db;         // D''_v = D_v - dA_v dB_v
                    cs.Dg[v] = dv;
                    // R10b: δ''(r,v) + 2D''_r and δ''(s,v) + 2D''_s from pre-swap rows
                    cs.Tr[v] = 2 * (xr + ars * db + ys - da * brs - dv + 2 * arv * bsv);
                    cs.Ts[v] = 2 * (xs - ars * db + yr + da * brs - dv + 2 * asv * brv);
                }
            }
            if (warp == w_dr || warp == w_ds) {
                // D''_r = sum_k a_rk B'_sk + a_rs B'_sr,  D''_s = sum_k a_sk B'_rk + a_sr B'_rs
                int dr = 0, ds = 0;
                if (warp == w_dr) dr = Dots<TA, TB>::dot(Ar, Bs, lane, 32, nb);
                if (warp == w_ds) ds = Dots<TA, TB>::dot(As, Br, lane, 32, nb);
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    dr += __shfl_xor_sync(0xffffffffu, dr, o);
                    ds += __shfl_xor_sync(0xffffffffu, ds, o);
                }
                if (lane == 0 && warp == w_dr) cs.Dg[r] = dr + ars * brs;
                if (lane == 0 && warp == w_ds) cs.Dg[s] = ds + ars * brs;
            }
            if (scalar_thread) {                  // scalar state: p, C, best, digest
                const uint16_t pr = cs.p[r];
                cs.p[r] = cs.p[s];
                cs.p[s] = pr;
                io.cost += dw;
                const int improved = io.cost < io.best;
                if (improved) io.best = io.cost;
                cs.flags[0] = improved;
                io.digest = digest_step(io.digest, kacc, r, s);
            }
        }
        group_sync(bar_id, NT);
        PT_MARK(pt2);

        // ---------------- U: Δ update (quads), B' exchange, next window ----------------
        const int Wnext = max(64, min(wmax, round_up32(8 * (j + 1))));
        {
            // address and threshold of this thread's candidate in the next window
            // (state independent; issued first so its latency overlaps the quad updates)
            if (t < Wnext && kacc + 1 + (uint64_t)t < k_end) {
                prepare_addr(pre, n, tb.rowaddr, advance_cursor(cur, j + 1 + t, M), kacc + 1 + (uint64_t)t);
                prepare_theta(pre, sch, seed, chain);
            }
            const int Dr2 = 2 * cs.Dg[r], Ds2 = 2 * cs.Dg[s];
            auto quad = [&](const uint32_t desc, const int g) {
                const int u = desc & 511, v0 = (desc >> 9) << 2;
                const int4 d4 = *reinterpret_cast<const int4*>(cs.D + 4 * g);
                const DT pu = cs.dAB[u];
                DT pv[4];
                DB::load4(cs.dAB, v0, pv);
                int4 nv = make_int4(d4.x + DB::rank(pu, pv[0]), d4.y + DB::rank(pu, pv[1]),
                                    d4.z + DB::rank(pu, pv[2]), d4.w + DB::rank(pu, pv[3]));
                const int er = r - v0, es = s - v0;
                const bool rowr = u == r, rows = u == s;
                if (rowr | rows) {                  // rows r, s: all touching
                    const int4 t4 = *reinterpret_cast<const int4*>((rowr ? cs.Tr : cs.Ts) + v0);
                    const int D2 = rowr ? Dr2 : Ds2;
                    nv = make_int4(t4.x - D2, t4.y - D2, t4.z - D2, t4.w - D2);
                }
                *reinterpret_cast<int4*>(cs.D + 4 * g) = nv;
                if (rowr && (unsigned)es < 4u) cs.D[4 * g + es] = -dw;   // swapping back restores C
                if (!(rowr | rows)) {
                    if ((unsigned)er < 4u) cs.D[4 * g + er] = cs.Tr[u] - Dr2;   // column r: δ''(u,r)
                    if ((unsigned)es < 4u) cs.D[4 * g + es] = cs.Ts[u] - Ds2;   // column s: δ''(u,s)
                }
            };
            if (QPT > 0) {
#pragma unroll
                for (int i = 0; i < (QPT > 0 ? QPT : 1); ++i)
                    if (qd[i] != 0xFFFFFFFFu) quad(qd[i], t + i * NT);
            } else {
                for (int g = t; g < nqt; g += NT) quad(tb.qdesc[g], g);
            }
            // B' exchange: columns r,s of every other row, then rows r,s (word-wise)
            for (int x = t; x < n; x += NT) {
                if (x == r || x == s) continue;
                TB* row = cs.Bp + x * ld;
                const TB br = row[r];
                row[r] = row[s];
                row[s] = br;
            }
            if (warp == w_dr) {
                constexpr int EPW = 4 / sizeof(TB);   // elements per 32-bit word
                constexpr uint32_t EMASK = sizeof(TB) == 1 ? 0xFFu : 0xFFFFu;
                const int nwords = ld / EPW;
                uint32_t* Rw = reinterpret_cast<uint32_t*>(cs.Bp + r * ld);
                uint32_t* Sw = reinterpret_cast<uint32_t*>(cs.Bp + s * ld);
                for (int w = lane; w < nwords; w += 32) {
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
        }
        group_sync(bar_id, NT);
        PT_MARK(pt3);
        PT_ADD(0, pt0, pt1);
        PT_ADD(2, pt1, pt2);
        PT_ADD(3, pt2, pt3);
        PT_ADD(4, 0, 1);

        ++accepted;
        k = kacc + 1;
        cur = advance_cursor(cur, j + 1, M);
        W = Wnext;
    }
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
