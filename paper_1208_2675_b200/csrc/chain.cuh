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
//      dB_x = B'_xr - B'_xs (pre-swap);
//   U  update: disjoint pairs Δ_uv += 2(dA_u-dA_v)(dB_u-dB_v) (R10), touching
//      pairs recomputed on the post-swap B' by lane groups, Δ_rs = -δ.
// A window without an accepted candidate costs one barrier.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "device_common.cuh"

namespace qapsa {

template <typename TA, typename TB>
struct ChainSmem {
    TB* Bp;            // n x ld, B'_ij = B_{p(i),p(j)}
    int32_t* D;        // M, Δ in enumeration order (shared or global memory)
    int2* dAB;         // n, staged (dA_x, dB_x)
    uint16_t* p;       // n
    uint16_t* best_p;  // n
    int4* slots;       // 2 * NW window slots (double buffered)
    int* flags;        // [0] improved, [1] near count, [2] chain id broadcast
};

struct ChainScalars {  // meaningful in thread 0 of the group
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
        // certain-reject bound: δ > 38 T_k  =>  exp(-δ/T) < 2^-54 <= r  (R16 note)
        const double rej = __dmul_rn(38.0, temperature(sch, k));

        // ---------------- W: window of candidates ----------------
        bool acc = false, near = false;
        int q = 0, d = 0;
        if (t < Wl) {
            q = cur + t;
            if (q >= M) q = (M >= NT) ? q - M : q % M;
            d = cs.D[q];
            if (d <= 0) {
                acc = true;                       // δ < 0, or δ = 0: exp(0) = 1 > r (R5)
            } else if ((double)d <= rej) {
                const uint64_t kk = k + (uint64_t)t;
                acc = metropolis(d, temperature(sch, kk), uniform_r(seed, kk, chain), &near);
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

        // ---------------- S: swap p and B', stage dA/dB ----------------
        if (t == 0) {
            const uint16_t pr = cs.p[r];
            cs.p[r] = cs.p[s];
            cs.p[s] = pr;
            io.cost += dw;
            const int improved = io.cost < io.best;
            if (improved) io.best = io.cost;
            cs.flags[0] = improved;
            io.digest = digest_step(io.digest, kacc, r, s);
        }
        for (int x = t; x < n; x += NT) {
            if (x == r || x == s) continue;
            TB* row = cs.Bp + x * ld;
            const int br = row[r], bs = row[s];
            cs.dAB[x] = make_int2((int)A[r * ld + x] - (int)A[s * ld + x], br - bs);
            row[r] = (TB)bs;
            row[s] = (TB)br;
        }
        {
            constexpr int EPW = 4 / sizeof(TB);   // elements per 32-bit word
            constexpr uint32_t EMASK = sizeof(TB) == 1 ? 0xFFu : 0xFFFFu;
            const int nwords = ld / EPW;
            uint32_t* Rw = reinterpret_cast<uint32_t*>(cs.Bp + r * ld);
            uint32_t* Sw = reinterpret_cast<uint32_t*>(cs.Bp + s * ld);
            for (int w = t; w < nwords; w += NT) {
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
        if (q0 < M) {                             // disjoint pairs (rank form, R10)
            int u = u0, v = v0;
            int2 au = cs.dAB[u];
            bool ut = (u == r) | (u == s);
            const int qe = min(q0 + c, M);
            for (int qq = q0; qq < qe; ++qq) {
                if (!ut && v != r && v != s) {
                    const int2 av = cs.dAB[v];
                    cs.D[qq] += 2 * (au.x - av.x) * (au.y - av.y);
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
        {                                         // touching pairs: O(N) recompute, 8 lanes per v
            constexpr int L = 8, NG = NT / L;
            const int g = t / L, sub = t % L;
            const TA* Ar = A + r * ld;
            const TA* As = A + s * ld;
            const TB* Br = cs.Bp + r * ld;
            const TB* Bs = cs.Bp + s * ld;
            for (int vb = 0; vb < n; vb += NG) {
                const int v = vb + g;
                const bool act = v < n && v != r && v != s;
                int sr = 0, ss = 0;
                if (act) {
                    const TA* Av = A + v * ld;
                    const TB* Bv = cs.Bp + v * ld;
                    for (int kk = sub; kk < n; kk += L) {
                        const int av = Av[kk], bv = Bv[kk];
                        sr += ((int)Ar[kk] - av) * (bv - (int)Br[kk]);
                        ss += ((int)As[kk] - av) * (bv - (int)Bs[kk]);
                    }
                }
#pragma unroll
                for (int o = L / 2; o > 0; o >>= 1) {
                    sr += __shfl_xor_sync(0xffffffffu, sr, o);
                    ss += __shfl_xor_sync(0xffffffffu, ss, o);
                }
                if (act && sub == 0) {
                    // δ(x,v) = 2 [ sum_all k (a_xk - a_vk)(B'_vk - B'_xk) + 2 a_xv B'_xv ]
                    cs.D[v < r ? tri_index(n, v, r) : tri_index(n, r, v)] =
                        2 * (sr + 2 * (int)Ar[v] * (int)Br[v]);
                    cs.D[v < s ? tri_index(n, v, s) : tri_index(n, s, v)] =
                        2 * (ss + 2 * (int)As[v] * (int)Bs[v]);
                }
            }
        }
        if (t == 0) cs.D[tri_index(n, r, s)] = -dw;   // swapping back restores C
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

}  // namespace qapsa
