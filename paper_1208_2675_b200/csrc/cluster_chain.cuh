// cluster_chain.cuh -- one chain on a thread-block cluster of CLC = 8 CTAs for instances too
// large for one SM (N up to QAP_MAX_N = 512): SURVEY §8(f) row f1, "cluster-distributed single
// chain", the paper's multi-block decomposition of one chain with
// distributed shared memory and hardware cluster barriers instead of global memory and a
// software grid barrier.
//
// Ownership: CTA c of the cluster owns the locations x with x mod CLC = c (rows interleaved so
// that the upper-triangle rows of Δ spread evenly) and keeps, in its own shared memory, for each
// owned x: row x of A, row x of B' (B'_xy = B_{p(x) p(y)}, R9) and row x of Δ (entries (x, v),
// v > x).  Nothing is replicated but p (N x 2 B), the scalars and the staging vectors, so N = 512
// needs about 170 KB (8-bit B) or 200 KB (16-bit B) per CTA where one SM would need 1.3 MB.
//
// One window (R4, R6-R8): whole rows of the enumeration from the cursor; warp w of CTA
// c tests the w-th window row it owns, 32 columns at a time in order, against the exact integer
// thresholds of k_theta (theta_ring.cuh, R23; a flagged iteration takes the general test), and
// stops at its first accept; the CTA minimum goes to every CTA of the cluster (st.shared::cluster)
// and one cluster barrier later every CTA knows the window's first accept j.
//
// One accepted swap (r, s) (P:46-50 steps (c)-(d), R9, R10):
//   1. the owners of r and s copy the PRE-swap rows a_r, a_s, B'_r, B'_s to every CTA;
//      cluster barrier
//   2. every CTA: dA_x = a_rx - a_sx, dB_x = B'_rx - B'_sx (A, B' symmetric), then for its rows
//      u != r, s the disjoint entries Δ_uv += 2 (dA_u - dA_v)(dB_u - dB_v) (R10), the column swap
//      r <-> s of its B' rows and, if it owns r or s, the new row (post-swap row r = pre-swap row s
//      with columns r, s exchanged)
//   3. the touching entries δ''(r, v), δ''(s, v) of every owned v, recomputed from scratch on the
//      POST-swap rows (the oracle's definition) and stored into the owner of row min(r, v)
//      (a remote store when that is r); δ''(r, s) = -δ(r, s); cluster barrier
// Every quantity is an exact integer, so the trajectory is the oracle's.
//
// Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "kernels.cuh"
#include "relabel_chain.cuh"
#include "tc_chain.cuh"
#include "theta_ring.cuh"

namespace qapsa {

constexpr int CLC = 8;                   // CTAs per cluster (portable size)
constexpr int CLC_NT = 512;              // threads per CTA (16 warps)
constexpr int CLC_NW = CLC_NT / 32;
constexpr int CLC_WCAP = TH_RING - TH_BLK;   // window cap: the ring's reach (7168)

struct ClLayout {
    int arow, brow, drow, doff, ar, as, br, bs, dA, dB, p, bestp, wres, slots, ring, tbar, thdr, misc, bytes;
};
// R = ceil(n / CLC) owned rows; lda = row stride of the A / B' rows (elements, multiple of 16)
__host__ __device__ inline int clc_rows(int n) { return (n + CLC - 1) / CLC; }
__host__ __device__ inline int clc_lda(int n) { return (n + 15) & ~15; }
// Δ row x is kept quad-aligned: entries v in [b(x), n4), b(x) = 4 floor((x + 1) / 4), n4 = n
// rounded up to 4 (the cells v <= x and v >= n are padding, never read), so that the disjoint
// update runs on 16-byte quads like the single-SM engines' quad layout (§5)
__host__ __device__ inline int clc_n4(int n) { return (n + 3) & ~3; }
__host__ __device__ inline int clc_b(int x) { return (x + 1) & ~3; }
// owned Δ cells of CTA c (rows x = c, c + CLC, ...): sum of (n4 - b(x))
__host__ __device__ inline int clc_dcount(int n, int c) {
    int e = 0;
    for (int x = c; x < CLC * clc_rows(n); x += CLC) e += max(0, clc_n4(n) - clc_b(x));
    return e;
}
// offset of row x's first cell (column b(x)) in its owner's Δ rows: rows j CLC + c, j < x / CLC
// (CLC = 8: b(8 j + c) = 8 j + 4 floor((c + 1) / 4))
__host__ __device__ inline int clc_doff(int n, int x) {
    static_assert(CLC == 8, "closed form for clusters of 8");
    const int q = x / CLC, c = x % CLC;
    return q * (clc_n4(n) - 4 * ((c + 1) / 4)) - CLC * (q * (q - 1) / 2);
}
__host__ __device__ inline ClLayout cl_layout(int n, int tb) {
    ClLayout L;
    const int R = clc_rows(n), lda = clc_lda(n);
    int o = 0;
    L.arow = o;  o += align16(R * lda);                  // A rows (8-bit)
    L.brow = o;  o += align16(R * lda * tb);             // B' rows (8 or 16-bit)
    L.drow = o;  o += align16(clc_dcount(n, 0) * 4);     // Δ rows (CTA 0 owns the most entries)
    L.doff = o;  o += align16(R * 4);
    L.ar = o;    o += align16(lda);                      // PRE-swap rows a_r, a_s, B'_r, B'_s
    L.as = o;    o += align16(lda);
    L.br = o;    o += align16(lda * tb);
    L.bs = o;    o += align16(lda * tb);
    L.dA = o;    o += align16(n * 4);
    L.dB = o;    o += align16(n * 4);
    L.p = o;     o += align16(n * 2);
    L.bestp = o; o += align16(n * 2);
    L.wres = o;  o += CLC_NW * 16;                       // per-warp first accept (o, d, r|s, 0)
    L.slots = o; o += 2 * CLC * 16;                      // per-CTA first accept, by window parity
    L.ring = o;  o += TH_RING_BYTES;                     // threshold ring (theta_ring.cuh)
    L.tbar = o;  o += TH_SLOTS * 8;
    L.thdr = o;  o += TH_SLOTS * 16;
    L.misc = o;  o += 64;
    L.bytes = o;
    return L;
}

// remote (or local) 16-byte store into CTA `rank`'s copy of *local
__device__ __forceinline__ void cl_store4(int4* local, int rank, int4 v) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(local)), "r"(rank));
    asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void cl_sync() { cl_arrive(); cl_wait(); }

template <typename TB>
__global__ void __cluster_dims__(CLC, 1, 1) __launch_bounds__(CLC_NT, 1) k_sa_cluster(const ChainArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int c = cl_rank();
    const int n = a.n, M = a.M;
    const int R = clc_rows(n), lda = clc_lda(n);
    const ClLayout L = cl_layout(n, (int)sizeof(TB));
    uint8_t* Arow = smem + L.arow;
    TB* Brow = reinterpret_cast<TB*>(smem + L.brow);
    int32_t* Drow = reinterpret_cast<int32_t*>(smem + L.drow);
    int* doff = reinterpret_cast<int*>(smem + L.doff);
    uint8_t* ar = smem + L.ar;
    uint8_t* as = smem + L.as;
    TB* br = reinterpret_cast<TB*>(smem + L.br);
    TB* bs = reinterpret_cast<TB*>(smem + L.bs);
    int* dA = reinterpret_cast<int*>(smem + L.dA);
    int* dB = reinterpret_cast<int*>(smem + L.dB);
    uint16_t* p = reinterpret_cast<uint16_t*>(smem + L.p);
    uint16_t* best_p = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int4* wres = reinterpret_cast<int4*>(smem + L.wres);
    int4* slots = reinterpret_cast<int4*>(smem + L.slots);
    const TB* Bg = reinterpret_cast<const TB*>(a.B);
    const uint8_t* Ag = reinterpret_cast<const uint8_t*>(a.A);

    // ---------------- load: p, owned rows of A, B' and Δ ----------------
    for (int i = t; i < n; i += CLC_NT) {
        p[i] = (uint16_t)a.p[i];
        best_p[i] = (uint16_t)a.best_p[i];
    }
    for (int lx = t; lx < R; lx += CLC_NT) doff[lx] = clc_doff(n, lx * CLC + c);
    __syncthreads();
    for (int i = t; i < R * lda; i += CLC_NT) {
        const int lx = i / lda, y = i - lx * lda, x = lx * CLC + c;
        const bool in = x < n && y < n;
        Arow[i] = in ? Ag[(size_t)x * a.ld + y] : (uint8_t)0;
        Brow[i] = in ? Bg[(size_t)p[x] * a.ld + p[y]] : (TB)0;
    }
    for (int lx = warp; lx < R; lx += CLC_NW) {
        const int x = lx * CLC + c;
        const int b = clc_b(x), n4 = clc_n4(n);
        for (int v = b + lane; v < n4; v += 32)
            Drow[doff[lx] + v - b] = (v > x && v < n) ? a.D[a.rowaddr[x] + v] : 0;
    }
    ThetaRing<TH_SLOTS> TR = theta_ring<TH_SLOTS>(
        reinterpret_cast<int*>(smem + L.ring), reinterpret_cast<int4*>(smem + L.thdr),
        reinterpret_cast<uint64_t*>(smem + L.tbar), a.theta, a.theta_hdr, a.theta_kb, a.theta_cnt, a.k0);
    if (t == 0 && a.k0 < a.k_end) TR.start(a.k0);
    __syncthreads();
    cl_sync();                                   // every CTA of the cluster is resident and loaded

    const Sched sch = a.sch;
    const uint64_t seed = a.seed, k0 = a.k0;
    const uint32_t kr_end = (uint32_t)min((unsigned long long)(a.k_end - k0), 0x7FFFFFFFull);
    const NearSink sink{a.near_count, a.near_k, a.near_dec, a.near_cap, nullptr, nullptr, 0u};
    int64_t cost = a.st->cost, best = a.st->best_cost;
    uint64_t digest = a.st->digest, accepted = 0;
    uint32_t kr = 0;
    int u0, v0;
    tri_pair(n, (int)(k0 % (uint64_t)M), &u0, &v0);
    const int wcap = min(a.wscan, CLC_WCAP);
    int W = wcap;
    int parity = 0;
    const int kofs0 = (int)(k0 - TR.kb);
    int ring_blo = -1, ring_hi = 0;

    while (kr < kr_end) {
        // ---------------- window: whole rows u0 .. u0+Rw-1 ----------------
        const int L0 = n - v0, m1 = n - 1 - u0;
        // (at most CLC x CLC_NW rows: one per warp of the cluster; W <= 7168 keeps Rw below ~120)
        const int Rw = min(win_rows_whole(n, u0, L0, m1, W), CLC * CLC_NW);
        int Wl = win_f(Rw, L0, m1);
        if ((uint32_t)Wl > kr_end - kr) Wl = (int)(kr_end - kr);
        const int ko = kofs0 + (int)kr;
        if ((ko >> 10) != ring_blo) {     // a block passed (warp-uniform test; one thread refills)
            ring_blo = ko >> 10;
            if (t == 0) TR.refill(k0 + kr);
        }
        if (ko + Wl > ring_hi) {
            TR.ensure_ofs(ko + Wl);
            ring_hi = (int)(TR.ready * TH_BLK);
        }
        // this CTA's window rows: x = u0 + i with x mod CLC = c; warp w takes the w-th of them
        const int i_first = ((c - u0) % CLC + CLC) % CLC;
        const int i_row = i_first + CLC * warp;
        int best_o = INT_MAX, best_d = 0, best_rs = 0;
        int nt_o = INT_MAX, nt_d = 0;            // this thread's near tie (R16), if any
        if (i_row < Rw) {
            const int x = u0 + i_row, lx = x / CLC;
            const int first = i_row == 0 ? v0 : x + 1;
            const int f = i_row == 0 ? 0 : win_f(i_row, L0, m1);    // offset of (x, first)
            const int32_t* drow = Drow + doff[lx] - clc_b(x);       // drow[v] = Δ(x, v)
            for (int v = first + lane; v - lane < n; v += 32) {    // 32 columns at a time, in order
                const int o = f + v - first;
                const bool ex = v < n && o < Wl;
                const int d = ex ? drow[v] : 0;
                const int thr = ex ? TR.at_ofs(ko + o) : 0;
                // R23; δ <= 0 accepted (R5); a flagged iteration (thr = -1) with δ > 0 takes the
                // general test (branch-free in the common case: a warp vote guards the rare one)
                bool acc = ex & (d <= max(thr, 0));
                const bool need = ex & (thr < 0) & (d > 0);
                if (__any_sync(0xffffffffu, need)) {
                    if (need) {                  // flagged iteration: general test (R16)
                        float th, m;
                        theta_of(sch, seed, 0u, k0 + kr + (uint64_t)o, &th, &m);
                        const float df = (float)d;
                        acc = df < th - m;
                        if (!acc && !(df > th + m)) {
                            const int xx = tc_exact(d, k0 + kr + (uint64_t)o, sch, seed, 0u);
                            acc = xx & 1;
                            if ((xx & 2) && nt_o == INT_MAX) { nt_o = o; nt_d = acc; }
                        }
                    }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, acc);
                if (bal) {
                    const int l = __ffs(bal) - 1;
                    if (lane == l) {
                        best_o = o;
                        best_d = d;
                        best_rs = x | (v << 16);
                    }
                    break;
                }
            }
        }
        {
            const int wmin = __reduce_min_sync(0xffffffffu, best_o);
            if (lane == 0) wres[warp] = make_int4(INT_MAX, 0, 0, 0);
            __syncwarp();
            if (best_o == wmin && wmin != INT_MAX) wres[warp] = make_int4(best_o, best_d, best_rs, 0);
        }
        __syncthreads();
        if (warp == 0) {                         // the CTA's first accept, to every CTA of the cluster
            int4 w = lane < CLC_NW ? wres[lane] : make_int4(INT_MAX, 0, 0, 0);
            const int m = __reduce_min_sync(0xffffffffu, w.x);
            const unsigned bw = __ballot_sync(0xffffffffu, w.x == m);
            w = wres[__ffs(bw) - 1];
            if (lane < CLC) cl_store4(slots + parity * CLC + c, lane, w);
        }
        cl_sync();                               // window decision
        int4 win = make_int4(INT_MAX, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < CLC; ++q) {
            const int4 s4 = slots[parity * CLC + q];
            if (s4.x < win.x) win = s4;
        }
        parity ^= 1;
        const int j = win.x;
        if (nt_o != INT_MAX) {                   // R16: log a near tie of a consumed iteration
            const int consumed = (j == INT_MAX) ? Wl : j + 1;
            if (nt_o < consumed) near_record(sink, k0 + kr + (uint64_t)nt_o, nt_d != 0);
        }
        if (j == INT_MAX) {
            kr += (uint32_t)Wl;
            u0 += Rw;
            v0 = u0 + 1;
            if (u0 >= n - 1) { u0 = 0; v0 = 1; }
            W = min(2 * W, wcap);
            continue;
        }
        const int r = win.z & 0xFFFF, s = (win.z >> 16) & 0xFFFF;   // r < s
        const int dw = win.y;
        // ---------------- 1. the PRE-swap rows a_r, a_s, B'_r, B'_s to every CTA ----------------
        {
            const int cr = r % CLC, cs = s % CLC;
            const int wa = lda / 16;                               // 16-byte words of an A row
            const int wb = lda * (int)sizeof(TB) / 16;             // ... of a B' row
            const int per = 2 * wa + 2 * wb;                       // words per destination CTA
            for (int i = t; i < per * CLC; i += CLC_NT) {
                const int dst = i / per, q = i - dst * per;
                const int4* src;
                int4* to;
                if (q < wa) {
                    if (c != cr) continue;
                    src = reinterpret_cast<const int4*>(Arow + (r / CLC) * lda) + q;
                    to = reinterpret_cast<int4*>(ar) + q;
                } else if (q < 2 * wa) {
                    if (c != cs) continue;
                    src = reinterpret_cast<const int4*>(Arow + (s / CLC) * lda) + (q - wa);
                    to = reinterpret_cast<int4*>(as) + (q - wa);
                } else if (q < 2 * wa + wb) {
                    if (c != cr) continue;
                    src = reinterpret_cast<const int4*>(Brow + (size_t)(r / CLC) * lda) + (q - 2 * wa);
                    to = reinterpret_cast<int4*>(br) + (q - 2 * wa);
                } else {
                    if (c != cs) continue;
                    src = reinterpret_cast<const int4*>(Brow + (size_t)(s / CLC) * lda) + (q - 2 * wa - wb);
                    to = reinterpret_cast<int4*>(bs) + (q - 2 * wa - wb);
                }
                cl_store4(to, dst, *src);
            }
        }
        cl_sync();
        // ---------------- 2. staging vectors, disjoint entries, B' rows ----------------
        for (int x = t; x < clc_n4(n); x += CLC_NT) {   // (0 past n: the rows are zero-padded)
            dA[x] = (int)ar[x] - (int)as[x];     // a_xr - a_xs (A symmetric)
            dB[x] = (int)br[x] - (int)bs[x];     // B'_xr - B'_xs (PRE-swap, B' symmetric)
        }
        __syncthreads();
        for (int lx = warp; lx < R; lx += CLC_NW) {
            const int u = lx * CLC + c;
            if (u >= n) break;
            TB* brow = Brow + (size_t)lx * lda;
            if (u == r || u == s) {              // post-swap row r = pre-swap row s, columns r, s exchanged
                const TB* src = u == r ? bs : br;
                for (int y = lane; y < n; y += 32) brow[y] = src[y == r ? s : y == s ? r : y];
            } else {
                if (lane == 0) {                 // column swap r <-> s
                    const TB tr = brow[r];
                    brow[r] = brow[s];
                    brow[s] = tr;
                }
                // R10 on whole quads of the row: the cells of columns r, s are the touching entries,
                // overwritten in step 3 after the barrier; padding cells take anything
                const int dAu = dA[u], dBu = dB[u];
                const int b = clc_b(u), n4 = clc_n4(n);
                int4* drow4 = reinterpret_cast<int4*>(Drow + doff[lx]);
                for (int q4 = lane; 4 * q4 < n4 - b; q4 += 32) {
                    const int v0 = b + 4 * q4;
                    int4 o = drow4[q4];
                    const int4 xa = *reinterpret_cast<const int4*>(dA + v0);
                    const int4 xb = *reinterpret_cast<const int4*>(dB + v0);
                    o.x += 2 * (dAu - xa.x) * (dBu - xb.x);
                    o.y += 2 * (dAu - xa.y) * (dBu - xb.y);
                    o.z += 2 * (dAu - xa.z) * (dBu - xb.z);
                    o.w += 2 * (dAu - xa.w) * (dBu - xb.w);
                    drow4[q4] = o;
                }
            }
        }
        __syncthreads();
        // ---------------- 3. touching entries from the POST-swap rows ----------------
        // post-swap row r of B' is bs with r <-> s (likewise row s); a_r, a_s are unchanged
        for (int lx = warp; lx < R; lx += CLC_NW) {
            const int v = lx * CLC + c;
            if (v >= n || v == r || v == s) continue;
            const uint8_t* av = Arow + (size_t)lx * lda;
            const TB* bv = Brow + (size_t)lx * lda;   // post-swap row v
            int sr = 0, ss = 0;
            if constexpr (sizeof(TB) == 1) {
                // 8-bit rows: the sums over all k as byte dot products (dp4a, 16 k per lane; the
                // rows are zero past n), then the exchange of columns r, s in B'_r, B'_s and the
                // excluded terms k = r | s and k = v as exact scalar corrections (lane 0)
                unsigned P[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
                for (int k0 = 16 * lane; k0 < lda; k0 += 512) {
                    const uint4 Ar = *reinterpret_cast<const uint4*>(ar + k0);
                    const uint4 As_ = *reinterpret_cast<const uint4*>(as + k0);
                    const uint4 Av = *reinterpret_cast<const uint4*>(av + k0);
                    const uint4 Bv = *reinterpret_cast<const uint4*>(bv + k0);
                    const uint4 Bs_ = *reinterpret_cast<const uint4*>(bs + k0);
                    const uint4 Br_ = *reinterpret_cast<const uint4*>(br + k0);
                    auto dot = [](uint4 x, uint4 y, unsigned c) {
                        return __dp4a(x.x, y.x, __dp4a(x.y, y.y, __dp4a(x.z, y.z, __dp4a(x.w, y.w, c))));
                    };
                    P[0] = dot(Ar, Bv, P[0]);    // a_r . b'_v
                    P[1] = dot(Ar, Bs_, P[1]);   // a_r . (pre-swap row s)
                    P[2] = dot(Av, Bv, P[2]);    // a_v . b'_v
                    P[3] = dot(Av, Bs_, P[3]);   // a_v . (pre-swap row s)
                    P[4] = dot(As_, Bv, P[4]);   // a_s . b'_v
                    P[5] = dot(As_, Br_, P[5]);  // a_s . (pre-swap row r)
                    P[6] = dot(Av, Br_, P[6]);   // a_v . (pre-swap row r)
                }
#pragma unroll
                for (int e = 0; e < 7; ++e) P[e] = __reduce_add_sync(0xffffffffu, P[e]);
                if (lane == 0) {
                    auto g = [](const uint8_t* x, int k) { return (int)x[k]; };
                    const int arr = g(ar, r), ars_ = g(ar, s), asr = g(as, r), ass = g(as, s);
                    const int avr = g(av, r), avs = g(av, s), avv = g(av, v), arv = g(ar, v), asv = g(as, v);
                    const int bvr = (int)bv[r], bvs = (int)bv[s], bvv = (int)bv[v];
                    const int bsr = (int)bs[r], bss = (int)bs[s], bsv = (int)bs[v];
                    const int brr = (int)br[r], brs = (int)br[s], brv = (int)br[v];
                    // post-swap rows r, s of B': bs, br with columns r and s exchanged
                    const int P1 = (int)P[1] - arr * bsr - ars_ * bss + arr * bss + ars_ * bsr;
                    const int P3 = (int)P[3] - avr * bsr - avs * bss + avr * bss + avs * bsr;
                    const int P5 = (int)P[5] - asr * brr - ass * brs + asr * brs + ass * brr;
                    const int P6 = (int)P[6] - avr * brr - avs * brs + avr * brs + avs * brr;
                    // sum over every k, minus k = r and k = v (δ''(r, v)); k = s and k = v (δ''(s, v))
                    sr = (int)P[0] - P1 - (int)P[2] + P3 - (arr - avr) * (bvr - bss) - (arv - avv) * (bvv - bsv);
                    ss = (int)P[4] - P5 - (int)P[2] + P6 - (ass - avs) * (bvs - brr) - (asv - avv) * (bvv - brv);
                }
                ss = __shfl_sync(0xffffffffu, ss, 0);
                sr = __shfl_sync(0xffffffffu, sr, 0);
            } else {
                for (int k = lane; k < n; k += 32) {
                    const int kp = k == r ? s : k == s ? r : k;
                    const int bvk = (int)bv[k];
                    if (k != r && k != v) sr += ((int)ar[k] - (int)av[k]) * (bvk - (int)bs[kp]);
                    if (k != s && k != v) ss += ((int)as[k] - (int)av[k]) * (bvk - (int)br[kp]);
                }
#pragma unroll
                for (int sh = 16; sh > 0; sh >>= 1) {
                    sr += __shfl_xor_sync(0xffffffffu, sr, sh);
                    ss += __shfl_xor_sync(0xffffffffu, ss, sh);
                }
            }
            if (lane < 2) {                      // δ''(r, v) by lane 0, δ''(s, v) by lane 1
                const int x = lane == 0 ? r : s;
                const int val = 2 * (lane == 0 ? sr : ss);
                const int lo = min(x, v), hi = max(x, v);
                cl_store(Drow + clc_doff(n, lo) + hi - clc_b(lo), lo % CLC, val);   // same layout in every CTA
            }
        }
        if (t == 0) {                            // δ''(r, s) = -δ(r, s): swapping back restores the cost
            cl_store(Drow + clc_doff(n, r) + s - clc_b(r), r % CLC, -dw);
        }
        // p, the scalars (every CTA keeps them identically), best_p
        __syncthreads();
        if (t == 0) {
            const uint16_t pr = p[r];
            p[r] = p[s];
            p[s] = pr;
        }
        cost += dw;
        const uint64_t kacc = k0 + kr + (uint64_t)j;
        digest = digest_step(digest, kacc, r, s);
        ++accepted;
        __syncthreads();
        if (cost < best) {
            best = cost;
            for (int i = t; i < n; i += CLC_NT) best_p[i] = p[i];
        }
        int nu0, nv0;
        next_pair(n, r, s, &nu0, &nv0);
        u0 = nu0;
        v0 = nv0;
        W = max(64, min(wcap, round_up32(8 * (j + 1))));
        kr += (uint32_t)j + 1;
        cl_sync();                               // touching entries stored everywhere
    }
    if (t == 0) TR.drain();

    // ---------------- write back: Δ rows (every CTA), p, best_p, scalars (CTA 0) ----------------
    __syncthreads();
    for (int lx = warp; lx < R; lx += CLC_NW) {
        const int x = lx * CLC + c;
        if (x >= n - 1) break;
        for (int v = x + 1 + lane; v < n; v += 32) a.D[a.rowaddr[x] + v] = Drow[doff[lx] + v - clc_b(x)];
    }
    if (c == 0) {
        for (int i = t; i < n; i += CLC_NT) {
            a.p[i] = p[i];
            a.best_p[i] = best_p[i];
        }
        if (t == 0) {
            a.st->cost = cost;
            a.st->best_cost = best;
            a.st->digest = digest;
            a.st->accepted += accepted;
        }
    }
    cl_sync();                                   // no CTA exits while others may still store into it
}

}  // namespace qapsa
