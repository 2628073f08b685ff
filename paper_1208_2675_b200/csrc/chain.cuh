// chain.cuh -- one Δ-matrix SA chain run by a group of NT threads that keeps
// its whole state in shared memory (Δ may instead live in global memory / L2).
//
// Per accepted swap the group goes through three phases separated by named
// barriers ("a synchronization mechanism is needed"; here the group
// is inside one CTA, so a hardware barrier suffices):
//   W  window: thread t tests candidate k+t against Eq.(2),
//      warp vote (__ballot_sync/__ffs) + cross-warp min picks the first
//      accepted candidate ("the swap which would have been found first");
//   S  swap: p(r)<->p(s), B' columns r,s exchanged per row and rows r,s
//      exchanged word-wise (Eq.(3)); staging dA_x = a_xr - a_xs and
//      dB_x = B'_xr - B'_xs (pre-swap); diagonal D_x = A_x . B'_x
//      kept current (D'_x = D_x - dA_x dB_x, R10 note);
//   U  update: disjoint pairs Δ_uv += 2(dA_u-dA_v)(dB_u-dB_v) (R10), touching
//      pairs recomputed on the post-swap B' with dp4a dot products,
//      Δ_rs = -δ.
// A window without an accepted candidate costs one barrier.
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
    __device__ static int a(T v) { return v.x; }
    __device__ static int b(T v) { return v.y; }
};
template <>
struct Dab<uint8_t, uint8_t> {
    using T = int;
    __device__ static T pack(int a, int b) { return (a & 0xFFFF) | (b << 16); }
    __device__ static int a(T v) { return (v << 16) >> 16; }
    __device__ static int b(T v) { return v >> 16; }
};

template <typename TA, typename TB>
struct ChainSmem {
    TB* Bp;                            // n x ld, B'_ij = B_{p(i),p(j)}
    int32_t* D;                        // M, Δ in enumeration order (shared or global memory)
    typename Dab<TA, TB>::T* dAB;      // n, staged (dA_x, dB_x)
    int32_t* Dg;                       // n, diagonal D_x = sum_k A_xk B'_xk
    uint16_t* p;                       // n
    uint16_t* best_p;                  // n
    int4* slots;                       // 2 * NW window slots (double buffered)
    int* flags;                        // [0] improved, [1] near count, [2] chain id broadcast
};

struct ChainScalars {  // meaningful in thread NT-1 of the group
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

// ---- dot products over 4-element chunks (rows zero-padded to ld, ld % 4 == 0)
// acc[0] += x.a1, acc[1] += x.a2 for x = row X (type TX), a = rows (type TY)
__device__ __forceinline__ uint32_t dot4(uint32_t x, uint32_t y, uint32_t c) { return __dp4a(x, y, c); }

template <typename TA, typename TB>
struct Dots {
    // X_r += B'_v . a_r, X_s += B'_v . a_s, Y_r += A_v . b'_r, Y_s += A_v . b'_s
    __device__ static void run(const TA* Av, const TB* Bv, const TA* Ar, const TA* As, const TB* Br,
                               const TB* Bs, int ld, int& xr, int& xs, int& yr, int& ys) {
        for (int k = 0; k < ld; ++k) {
            const int bv = Bv[k], av = Av[k];
            xr += bv * (int)Ar[k];
            xs += bv * (int)As[k];
            yr += av * (int)Br[k];
            ys += av * (int)Bs[k];
        }
    }
    // sum_k X_k Y_k over one row pair
    __device__ static int dot(const TA* X, const TB* Y, int lo, int hi) {
        int acc = 0;
        for (int k = lo; k < hi; ++k) acc += (int)X[k] * (int)Y[k];
        return acc;
    }
};

template <>
struct Dots<uint8_t, uint8_t> {
    __device__ static void run(const uint8_t* Av, const uint8_t* Bv, const uint8_t* Ar,
                               const uint8_t* As, const uint8_t* Br, const uint8_t* Bs, int ld,
                               int& xr, int& xs, int& yr, int& ys) {
        const uint32_t* av = reinterpret_cast<const uint32_t*>(Av);
        const uint32_t* bv = reinterpret_cast<const uint32_t*>(Bv);
        const uint32_t* ar = reinterpret_cast<const uint32_t*>(Ar);
        const uint32_t* as = reinterpret_cast<const uint32_t*>(As);
        const uint32_t* br = reinterpret_cast<const uint32_t*>(Br);
        const uint32_t* bs = reinterpret_cast<const uint32_t*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0;
        const int nch = ld >> 2;
#pragma unroll 5
        for (int c = 0; c < nch; ++c) {
            const uint32_t a = av[c], b = bv[c];
            Xr = dot4(b, ar[c], Xr);
            Xs = dot4(b, as[c], Xs);
            Yr = dot4(a, br[c], Yr);
            Ys = dot4(a, bs[c], Ys);
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys;
    }
    __device__ static int dot(const uint8_t* X, const uint8_t* Y, int lo, int hi) {
        // lo, hi multiples of 4
        const uint32_t* x = reinterpret_cast<const uint32_t*>(X);
        const uint32_t* y = reinterpret_cast<const uint32_t*>(Y);
        uint32_t acc = 0;
        for (int c = lo >> 2; c < (hi >> 2); ++c) acc = dot4(x[c], y[c], acc);
        return (int)acc;
    }
};

template <>
struct Dots<uint8_t, uint16_t> {
    __device__ static void run(const uint8_t* Av, const uint16_t* Bv, const uint8_t* Ar,
                               const uint8_t* As, const uint16_t* Br, const uint16_t* Bs, int ld,
                               int& xr, int& xs, int& yr, int& ys) {
        const uint32_t* av = reinterpret_cast<const uint32_t*>(Av);
        const uint2* bv = reinterpret_cast<const uint2*>(Bv);
        const uint32_t* ar = reinterpret_cast<const uint32_t*>(Ar);
        const uint32_t* as = reinterpret_cast<const uint32_t*>(As);
        const uint2* br = reinterpret_cast<const uint2*>(Br);
        const uint2* bs = reinterpret_cast<const uint2*>(Bs);
        uint32_t Xr = 0, Xs = 0, Yr = 0, Ys = 0;
        const int nch = ld >> 2;
#pragma unroll 4
        for (int c = 0; c < nch; ++c) {
            const uint32_t a = av[c];
            const uint2 b = bv[c];
            const uint32_t r8 = ar[c], s8 = as[c];
            Xr = __dp2a_hi(b.y, r8, __dp2a_lo(b.x, r8, Xr));
            Xs = __dp2a_hi(b.y, s8, __dp2a_lo(b.x, s8, Xs));
            const uint2 R = br[c], S = bs[c];
            Yr = __dp2a_hi(R.y, a, __dp2a_lo(R.x, a, Yr));
            Ys = __dp2a_hi(S.y, a, __dp2a_lo(S.x, a, Ys));
        }
        xr += (int)Xr; xs += (int)Xs; yr += (int)Yr; ys += (int)Ys;
    }
    __device__ static int dot(const uint8_t* X, const uint16_t* Y, int lo, int hi) {
        int acc = 0;
        for (int k = lo; k < hi; ++k) acc += (int)X[k] * (int)Y[k];
        return acc;
    }
};

// Runs iterations [k0, k_end) of one chain.  Returns the number of accepted
// swaps (identical in every thread of the group).
template <typename TA, typename TB, int NT>
__device__ __forceinline__ uint64_t chain_run(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                              const int n, const int ld, const int M,
                                              const uint64_t k0, const uint64_t k_end,
                                              const Sched sch, const uint64_t seed,
                                              const uint32_t chain, const int bar_id,
                                              const int t, const int wmax, ChainScalars& io,
                                              const NearSink sink) {
    using DB = Dab<TA, TB>;
    constexpr int NW = NT / 32;
    const int lane = t & 31, warp = t >> 5;

    // chunk ownership for the disjoint update: thread t owns q in [q0, q0+c),
    // c odd so that lanes' Δ accesses hit distinct banks.
    int c = (M + NT - 1) / NT;
    if (!(c & 1)) ++c;
    const int q0 = t * c;
    int u0 = 0, v0 = 1;
    if (q0 < M) tri_pair(n, q0, &u0, &v0);

    uint64_t k = k0, accepted = 0;
    int cur = (int)(k0 % (uint64_t)M);
    int W = wmax;
    int parity = 0;

    while (k < k_end) {
        const uint64_t remaining = k_end - k;
        const int Wl = (uint64_t)W < remaining ? W : (int)remaining;
        // certain reject: δ > 38.5 T32(k) >= 38.4 T_{k+t}  =>  exp(-δ/T) < 2^-54 <= r  (R16 note)
        const float rej = 38.5f * temp32(sch, k);

        // ---------------- W: window of candidates ----------------
        bool acc = false, near = false;
        int q = 0, d = 0;
        if (t < Wl) {
            q = cur + t;
            if (q >= M) q = (M >= NT) ? q - M : q % M;
            d = cs.D[q];
            if (d <= 0) {
                acc = true;                       // δ < 0, or δ = 0: exp(0) = 1 > r (R5)
            } else if ((float)d <= rej) {
                const uint64_t kk = k + (uint64_t)t;
                acc = metropolis_fast(d, sch, kk, seed, chain, &near);
            }
        }
        int4* slots = cs.slots + parity * NW;
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        if (bal) {
            if (lane == __ffs(bal) - 1) {
                int r, s;
                tri_pair(n, q, &r, &s);
                slots[warp] = make_int4(t, d, r, s);
            }
        } else if (lane == 0) {
            slots[warp] = make_int4(INT_MAX, 0, 0, 0);
        }
        group_sync(bar_id, NT);
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
            k += (uint64_t)consumed;
            cur = (int)(((uint64_t)cur + (uint64_t)consumed) % (uint64_t)M);
            W = min(2 * W, wmax);
            continue;
        }
        const int4 win = slots[(j >> 5)];         // (t, δ, r, s) of the first accepted candidate
        const int dw = win.y, r = win.z, s = win.w;
        const uint64_t kacc = k + (uint64_t)j;

        // ---------------- S: swap p and B', stage dA/dB, diagonal ----------------
        for (int x = t; x < n; x += NT) {
            if (x == r || x == s) continue;
            TB* row = cs.Bp + x * ld;
            const int br = row[r], bs = row[s];
            const int da = (int)A[r * ld + x] - (int)A[s * ld + x], db = br - bs;
            cs.dAB[x] = DB::pack(da, db);
            cs.Dg[x] -= da * db;                  // D'_x = D_x - dA_x dB_x
            row[r] = (TB)bs;
            row[s] = (TB)br;
        }
        if (warp == NW - 1) {
            // D'_r = sum_k a_rk B'_sk + a_rs B'_sr,  D'_s = sum_k a_sk B'_rk + a_sr B'_rs (pre-swap)
            const TA* Ar = A + r * ld;
            const TA* As = A + s * ld;
            TB* Br = cs.Bp + r * ld;
            TB* Bs = cs.Bp + s * ld;
            int dr = 0, ds = 0;
            for (int c4 = lane * 4; c4 < ld; c4 += 128) {
                dr += Dots<TA, TB>::dot(Ar, Bs, c4, c4 + 4);
                ds += Dots<TA, TB>::dot(As, Br, c4, c4 + 4);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                dr += __shfl_xor_sync(0xffffffffu, dr, o);
                ds += __shfl_xor_sync(0xffffffffu, ds, o);
            }
            const int ars = (int)Ar[s] * (int)Br[s];
            if (lane == 0) {
                cs.Dg[r] = dr + ars;
                cs.Dg[s] = ds + ars;
            }
            if (lane == 31) {                     // scalar state: p, C, best, digest
                const uint16_t pr = cs.p[r];
                cs.p[r] = cs.p[s];
                cs.p[s] = pr;
                io.cost += dw;
                const int improved = io.cost < io.best;
                if (improved) io.best = io.cost;
                cs.flags[0] = improved;
                io.digest = digest_step(io.digest, kacc, r, s);
            }
            __syncwarp();
            constexpr int EPW = 4 / sizeof(TB);   // elements per 32-bit word
            constexpr uint32_t EMASK = sizeof(TB) == 1 ? 0xFFu : 0xFFFFu;
            const int nwords = ld / EPW;
            uint32_t* Rw = reinterpret_cast<uint32_t*>(Br);
            uint32_t* Sw = reinterpret_cast<uint32_t*>(Bs);
            for (int w = lane; w < nwords; w += 32) {
                uint32_t m = 0;
                if (r / EPW == w) m |= EMASK << (8 * sizeof(TB) * (r % EPW));
                if (s / EPW == w) m |= EMASK << (8 * sizeof(TB) * (s % EPW));
                const uint32_t a = Rw[w], b = Sw[w];
                Rw[w] = (b & ~m) | (a & m);       // rows exchange; entries (r,r),(r,s),(s,r),(s,s) keep
                Sw[w] = (a & ~m) | (b & m);       // their values (B' symmetric, zero diagonal)
            }
        }
        group_sync(bar_id, NT);

        // ---------------- U: Δ update ----------------
        {                                         // touching pairs: lane <-> v, dot products over k
            const TA* Ar = A + r * ld;
            const TA* As = A + s * ld;
            const TB* Br = cs.Bp + r * ld;
            const TB* Bs = cs.Bp + s * ld;
            const int Dr = cs.Dg[r], Ds = cs.Dg[s];
            for (int v = t; v < n; v += NT) {
                if (v == r || v == s) continue;
                int xr = 0, xs = 0, yr = 0, ys = 0;
                Dots<TA, TB>::run(A + v * ld, cs.Bp + v * ld, Ar, As, Br, Bs, ld, xr, xs, yr, ys);
                const int Dv = cs.Dg[v];
                // δ(x,v) = 2 [ B'_v.a_x + A_v.b'_x - D_x - D_v + 2 a_xv B'_xv ]
                cs.D[v < r ? tri_index(n, v, r) : tri_index(n, r, v)] =
                    2 * (xr + yr - Dr - Dv + 2 * (int)Ar[v] * (int)Br[v]);
                cs.D[v < s ? tri_index(n, v, s) : tri_index(n, s, v)] =
                    2 * (xs + ys - Ds - Dv + 2 * (int)As[v] * (int)Bs[v]);
            }
        }
        if (q0 < M) {                             // disjoint pairs (rank form, R10)
            int u = u0, v = v0;
            typename DB::T au = cs.dAB[u];
            bool ut = (u == r) | (u == s);
            const int qe = min(q0 + c, M);
            for (int qq = q0; qq < qe; ++qq) {
                if (!ut && v != r && v != s) {
                    const typename DB::T av = cs.dAB[v];
                    cs.D[qq] += 2 * (DB::a(au) - DB::a(av)) * (DB::b(au) - DB::b(av));
                }
                if (++v == n) {
                    ++u;
                    v = u + 1;
                    if (u < n) {
                        au = cs.dAB[u];
                        ut = (u == r) | (u == s);
                    }
                }
            }
        }
        if (t == NT - 1) cs.D[tri_index(n, r, s)] = -dw;   // swapping back restores C
        if (cs.flags[0])
            for (int x = t; x < n; x += NT) cs.best_p[x] = cs.p[x];
        group_sync(bar_id, NT);

        ++accepted;
        k = kacc + 1;
        cur = (int)(((uint64_t)cur + (uint64_t)j + 1) % (uint64_t)M);
        W = max(64, min(wmax, round_up32(8 * (j + 1))));
    }
    return accepted;
}

// Δ for all pairs of the current (smem) B', by the group: step (a) of P:46.
template <typename TA, typename TB, int NT>
__device__ __forceinline__ void chain_delta_init(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                                 int n, int ld, int M, int t) {
    for (int q = t; q < M; q += NT) {
        int r, s;
        tri_pair(n, q, &r, &s);
        const TA* Ar = A + r * ld;
        const TA* As = A + s * ld;
        const TB* Br = cs.Bp + r * ld;
        const TB* Bs = cs.Bp + s * ld;
        int acc = 0;
        for (int k = 0; k < n; ++k) acc += ((int)Ar[k] - (int)As[k]) * ((int)Bs[k] - (int)Br[k]);
        cs.D[q] = 2 * (acc + 2 * (int)Ar[s] * (int)Br[s]);
    }
}

// D_x = sum_k A_xk B'_xk for all x (the diagonal of A B'^T)
template <typename TA, typename TB, int NT>
__device__ __forceinline__ void chain_diag_init(const TA* __restrict__ A, const ChainSmem<TA, TB>& cs,
                                                int n, int ld, int t) {
    for (int x = t; x < n; x += NT) cs.Dg[x] = Dots<TA, TB>::dot(A + x * ld, cs.Bp + x * ld, 0, ld);
}

}  // namespace qapsa
