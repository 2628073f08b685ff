// relabel_chain.cuh -- the single-chain engine for instances with 8-bit A and 16-bit B up to
// N = 256 (BASELINE config 4), with exact O(1) relabel swaps for twin locations
// (R21).
//
// Twins.  Locations x, y are twins when A_xz = A_yz for every z != x, y (A symmetric, zero
// diagonal).  Exchanging the facilities of two twins leaves Eq.(1) unchanged for every
// permutation (A is invariant under the transposition), so a twin candidate always has
// δ = 0 and is always accepted (R5).  The engine works in SLOT space: a map σ (location ->
// slot) that only ever exchanges twins, and the chain state of the slots: q = p∘σ⁻¹
// (facility in slot i), B~ = B[q][q], Δ~(σu, σv) = Δ(u, v), the diagonal D~.  Since σ
// preserves the twin classes, A in slot space is A itself.  A twin accept (r, s) then only
// exchanges σ(r), σ(s); a non-twin ("cross") accept (r, s) is the ordinary swap of the slots
// (σr, σs) with the ordinary Taillard update of Δ~ (R10, R10b).
//
// Windows never cross a row of the enumeration (candidates (r, s0 .. n-1)), so inside a window
// only σ(r) moves: at candidate (r, s) it is the slot σ held by the window's last twin column
// below s (table pt), or σ(r) if there is none.  The first accepted cross candidate ends the
// window; every twin before it is accepted, σ is rotated in one parallel step, and each twin
// thread adds its accept to a private count and digest (R18 is a sum).
//
// Per cross accept (slots a < b), 1024 threads:
//   stage   dA_x = A_ax - A_bx, dB_x = B~_ax - B~_bx; Z_a = A_a.B~_b, Z_b = A_b.B~_a (warps 8, 9)
//   touch   threads 0..511, 2 per v: X_a = B~_v.A_a, X_b, Y_a = A_v.B~_a, Y_b over half of the
//           row each, shuffle-reduced; δ''(a,v), δ''(b,v) (R10b) and D~_v written
//   quads   threads 512..1023, concurrently: Δ~ += 2(dA_u - dA_v)(dB_u - dB_v) for every pair
//           off rows / columns a, b (R10); Δ~ in global memory / L2 (quad layout)
//   next window: B~ rows / columns a, b exchanged, best_p = q∘σ if the cost improved
//
// Shared memory (N = 256): A 256 x 272 B (odd multiple of 16 B per row) and B~ 256 x 264 u16
// (528 B = 33 x 16 B per row): the 8 rows one warp reads at the same column offset fall on
// distinct 16-byte bank groups.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "kernels.cuh"

namespace qapsa {

constexpr int RLB_NT = 1024;
constexpr int RLB_MAXN = 256;
constexpr int RLB_MAXCLS = 4;   // twin classes (>= 2 members) the relabel path handles
constexpr int RLB_TOUCH = 512;  // threads [0, 512): touching entries (2 per v); the rest: quads
constexpr int RLB_QB = 4;       // quad loads in flight per thread

// row strides in shared memory: A an odd multiple of 16 elements (bytes), B~ 8 x odd elements
__host__ __device__ constexpr int rlb_lda(int n) { return row_stride(n, true); }
__host__ __device__ constexpr int rlb_ldb(int n) { return 16 * ((n + 15) / 16) + 8; }

struct RlbLayout {
    int a, b, rowaddr, qdesc, pt, cls, sig, q, bestp, dg, stg, slots, twm, zz, flags, red, bytes;
};
__host__ __device__ constexpr RlbLayout rlb_layout(int n) {
    RlbLayout L{};
    const int n4 = (n + 3) & ~3;
    int o = 0;
    L.a = o;       o = align16(o + n * rlb_lda(n));
    L.b = o;       o = align16(o + n * rlb_ldb(n) * 2);
    L.rowaddr = o; o = align16(o + n * 4);
    L.qdesc = o;   o = align16(o + quad_count(n) * 2);
    L.pt = o;      o = align16(o + RLB_MAXCLS * (n + 1) * 2);
    L.cls = o;     o = align16(o + n4);
    L.sig = o;     o = align16(o + n * 2);
    L.q = o;       o = align16(o + n * 2);
    L.bestp = o;   o = align16(o + n * 2);
    L.dg = o;      o = align16(o + n * 4);
    L.stg = o;     o = align16(o + n4 * 8);
    L.slots = o;   o = align16(o + 2 * 32 * 16);
    L.twm = o;     o = align16(o + 2 * 32 * 4);
    L.zz = o;      o = align16(o + 4 * 4);
    L.flags = o;   o = align16(o + 4 * 4);
    L.red = o;     o = align16(o + 2 * 8);
    L.bytes = o;
    return L;
}

struct RelabelArgs {
    ChainArgs c;               // A, B (global, stride c.ld), p, best_p, D (working Δ~), ...
    const uint8_t* cls;        // n: twin class of location x in [0, ncls), 0xFF = none
    const uint16_t* pt;        // ncls x (n+1): largest member of class c below x, 0xFFFF = none
    int ncls;
    int32_t* d_out;            // Δ in location space at exit (quad layout)
};

// X_a += B~_v.A_a, X_b += B~_v.A_b, Y_a += A_v.B~_a, Y_b += A_v.B~_b over blocks b0, b0+step, ..
__device__ __forceinline__ void rlb_dots(const uint8_t* Av, const uint16_t* Bv, const uint8_t* Aa,
                                         const uint8_t* Ab, const uint16_t* Ba, const uint16_t* Bb,
                                         int b0, int step, int nb, int& xa, int& xb, int& ya, int& yb) {
    const uint4* av = reinterpret_cast<const uint4*>(Av);
    const uint4* bv = reinterpret_cast<const uint4*>(Bv);
    const uint4* aa = reinterpret_cast<const uint4*>(Aa);
    const uint4* ab = reinterpret_cast<const uint4*>(Ab);
    const uint4* ba = reinterpret_cast<const uint4*>(Ba);
    const uint4* bb = reinterpret_cast<const uint4*>(Bb);
    uint32_t Xa = 0, Xb = 0, Ya = 0, Yb = 0;
#pragma unroll 2
    for (int b = b0; b < nb; b += step) {
        const uint4 a = av[b], v0 = bv[2 * b], v1 = bv[2 * b + 1];
        const uint4 a8 = aa[b], b8 = ab[b];
        const uint4 A0 = ba[2 * b], A1 = ba[2 * b + 1], B0 = bb[2 * b], B1 = bb[2 * b + 1];
        Xa = dp16w(a8, v0, v1, Xa);
        Xb = dp16w(b8, v0, v1, Xb);
        Ya = dp16w(a, A0, A1, Ya);
        Yb = dp16w(a, B0, B1, Yb);
    }
    xa += (int)Xa; xb += (int)Xb; ya += (int)Ya; yb += (int)Yb;
}

template <int NFIX>
__global__ void __launch_bounds__(RLB_NT, 1) k_sa_relabel(const RelabelArgs ra) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ChainArgs& a = ra.c;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = NFIX ? NFIX : a.n;
    const int lda = rlb_lda(n), ldb = rlb_ldb(n), ldg = a.ld;
    const int nb = (n + 15) >> 4;
    const int M = n * (n - 1) / 2;
    const int nqt = NFIX ? quad_count(NFIX) : a.nqt;
    const int ncls = ra.ncls;
    const RlbLayout L = rlb_layout(n);
    uint8_t* As = smem + L.a;
    uint16_t* Bt = reinterpret_cast<uint16_t*>(smem + L.b);
    int32_t* rowaddr = reinterpret_cast<int32_t*>(smem + L.rowaddr);
    uint16_t* qdesc = reinterpret_cast<uint16_t*>(smem + L.qdesc);
    uint16_t* pt = reinterpret_cast<uint16_t*>(smem + L.pt);
    uint8_t* cls = smem + L.cls;
    uint16_t* sig = reinterpret_cast<uint16_t*>(smem + L.sig);
    uint16_t* q = reinterpret_cast<uint16_t*>(smem + L.q);
    uint16_t* bestp = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int32_t* Dg = reinterpret_cast<int32_t*>(smem + L.dg);
    int2* stg = reinterpret_cast<int2*>(smem + L.stg);
    int4* slot_base = reinterpret_cast<int4*>(smem + L.slots);
    unsigned* twm_base = reinterpret_cast<unsigned*>(smem + L.twm);
    int* zz = reinterpret_cast<int*>(smem + L.zz);
    int* flags = reinterpret_cast<int*>(smem + L.flags);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(smem + L.red);
    int32_t* D = a.D;
    const uint8_t* Ag = reinterpret_cast<const uint8_t*>(a.A);
    const uint16_t* Bg = reinterpret_cast<const uint16_t*>(a.B);

    // ---- load: A (restrided), tables, σ = id, q = p, B~ = B[q][q], D~ diagonal
    for (int idx = t; idx < n * lda; idx += RLB_NT) {
        const int i = idx / lda, j = idx - i * lda;
        As[idx] = j < ldg ? Ag[i * ldg + j] : (uint8_t)0;
    }
    for (int i = t; i < n; i += RLB_NT) {
        rowaddr[i] = a.rowaddr[i];
        cls[i] = ra.cls[i];
        sig[i] = (uint16_t)i;
        q[i] = (uint16_t)a.p[i];
        bestp[i] = (uint16_t)a.best_p[i];
    }
    for (int i = t; i < ncls * (n + 1); i += RLB_NT) pt[i] = ra.pt[i];
    for (int i = t; i < nqt; i += RLB_NT) qdesc[i] = a.qdesc[i];
    if (t < 4) flags[t] = 0;
    if (t < 2) red[t] = 0ull;
    __syncthreads();
    for (int idx = t; idx < n * ldb; idx += RLB_NT) {
        const int i = idx / ldb, j = idx - i * ldb;
        Bt[idx] = j < n ? Bg[q[i] * ldg + q[j]] : (uint16_t)0;
    }
    __syncthreads();
    for (int x = t; x < n; x += RLB_NT) {
        const uint4* ax = reinterpret_cast<const uint4*>(As + x * lda);
        const uint4* bx = reinterpret_cast<const uint4*>(Bt + x * ldb);
        uint32_t acc = 0;
        for (int b = 0; b < nb; ++b) acc = dp16w(ax[b], bx[2 * b], bx[2 * b + 1], acc);
        Dg[x] = (int)acc;
    }
    __syncthreads();

    const NearSink sink{a.near_count, a.near_k, a.near_dec, a.near_cap};
    int64_t cost = a.st->cost, best = a.st->best_cost;   // scalar thread (t == 0)
    uint64_t my_dig = 0, my_cnt = 0;                     // this thread's accepts (digest is a sum)
    uint64_t k = a.k0;
    const uint64_t k_end = a.k_end;
    int r, s0;
    tri_pair(n, (int)(k % (uint64_t)M), &r, &s0);
    int parity = 0, pa = -1, pb = -1;
    float rejT = 38.5f * temp32(a.sch, k);

    while (k < k_end) {
        const uint64_t remaining = k_end - k;
        const int Wl = (uint64_t)(n - s0) < remaining ? n - s0 : (int)remaining;

        // ---- deferred B~ exchange of the last cross accept (slots pa, pb) and best_p
        if (pa >= 0) {
            for (int x = t; x < n; x += RLB_NT) {
                if (x == pa || x == pb) continue;
                uint16_t* row = Bt + x * ldb;
                const uint16_t v = row[pa];
                row[pa] = row[pb];
                row[pb] = v;
            }
            if (warp == 1) {                              // rows pa, pb, word-wise
                uint32_t* Rw = reinterpret_cast<uint32_t*>(Bt + pa * ldb);
                uint32_t* Sw = reinterpret_cast<uint32_t*>(Bt + pb * ldb);
                for (int w = lane; w < ldb / 2; w += 32) {
                    uint32_t m = 0;
                    if (pa / 2 == w) m |= 0xFFFFu << (16 * (pa & 1));
                    if (pb / 2 == w) m |= 0xFFFFu << (16 * (pb & 1));
                    const uint32_t x = Rw[w], y = Sw[w];
                    Rw[w] = (y & ~m) | (x & m);
                    Sw[w] = (x & ~m) | (y & m);
                }
            }
            if (flags[0])
                for (int x = t; x < n; x += RLB_NT) bestp[x] = q[sig[x]];
            pa = -1;
        }

        // ---- window: candidates (r, s0 + t), t < Wl
        const int cr = ncls ? cls[r] : 0xFF;
        bool acc = false, near = false, twin = false;
        int d = 0, sab = 0, s = s0 + t;
        uint16_t newsig = 0;
        if (t < Wl) {
            const int pv = cr != 0xFF ? pt[cr * (n + 1) + s] : 0xFFFF;
            const int sr = (pv != 0xFFFF && pv >= s0) ? sig[pv] : sig[r];   // σ(r) at this candidate
            twin = cr != 0xFF && cls[s] == cr;
            if (twin) {
                newsig = (uint16_t)sr;                    // σ(s) after the transposition (r s)
            } else {
                const int ss = sig[s];
                const int sa = min(sr, ss), sb = max(sr, ss);
                sab = (sa << 16) | sb;
                d = D[rowaddr[sa] + sb];
                if (d <= 0) {
                    acc = true;                           // δ < 0, or δ = 0: exp(0) = 1 > r (R5)
                } else if ((float)d <= rejT) {            // else certain reject (chain.cuh)
                    acc = metropolis_fast(d, a.sch, k + (uint64_t)t, a.seed, 0u, &near);
                }
            }
        }
        int4* slots = slot_base + parity * 32;
        unsigned* twm = twm_base + parity * 32;
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        const unsigned tw = __ballot_sync(0xffffffffu, twin);
        if (bal) {
            if (lane == __ffs(bal) - 1) slots[warp] = make_int4(t, d, sab, s);
        } else if (lane == 0) {
            slots[warp] = make_int4(INT_MAX, 0, 0, 0);
        }
        if (lane == 0) twm[warp] = tw;
        __syncthreads();
        const int j = __reduce_min_sync(0xffffffffu, slots[lane].x);
        parity ^= 1;
        const int cons = (j == INT_MAX) ? Wl : j + 1;
        // any twin among the consumed candidates (needs a barrier before σ is read again)
        const int lo = cons - 32 * lane;
        const unsigned below = lo >= 32 ? 0xffffffffu : (lo <= 0 ? 0u : ((1u << lo) - 1u));
        const bool any_twin = __reduce_or_sync(0xffffffffu, twm[lane] & below) != 0u;
        if (near && t < cons) {                           // R16: near ties of consumed iterations
            const unsigned int i = atomicAdd(sink.count, 1u);
            if ((int)i < sink.cap) {
                sink.ks[i] = (unsigned long long)(k + (uint64_t)t);
                sink.dec[i] = acc ? 1 : 0;
            }
        }
        if (twin && t < cons) {                           // relabel: σ rotated, accept counted
            const uint16_t old = sig[s];
            sig[s] = newsig;
            if (pt[cr * (n + 1) + s0 + cons] == s) sig[r] = old;   // last consumed twin
            ++my_cnt;
            my_dig += mix64(mix64(k + (uint64_t)t) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)s));
        }
        if (j == INT_MAX) {                               // no cross accept in the window
            k += (uint64_t)cons;
            s0 += cons;
            if (s0 >= n) { ++r; if (r >= n - 1) r = 0; s0 = r + 1; }
            rejT = 38.5f * temp32(a.sch, k);
            if (any_twin) __syncthreads();
            continue;
        }

        // ---- cross accept: slots (sa, sb), location pair (r, sl)
        const int4 win = slots[j >> 5];
        const int dw = win.y, sa = win.z >> 16, sb = win.z & 0xFFFF, sl = win.w;
        const uint64_t kacc = k + (uint64_t)j;
        const uint8_t* Aa = As + sa * lda;
        const uint8_t* Ab = As + sb * lda;
        const uint16_t* Ba = Bt + sa * ldb;
        const uint16_t* Bb = Bt + sb * ldb;
        // stage and Z (the new diagonal of slots a, b)
        if (t < n) stg[t] = make_int2((int)Aa[t] - (int)Ab[t], (int)Ba[t] - (int)Bb[t]);
        if (warp == 8 || warp == 9) {
            const uint8_t* X = warp == 8 ? Aa : Ab;
            const uint16_t* Y = warp == 8 ? Bb : Ba;
            int z = 0;
            for (int x = lane; x < n; x += 32) z += (int)X[x] * (int)Y[x];
            z = __reduce_add_sync(0xffffffffu, z);
            if (lane == 0) zz[warp - 8] = z;
        }
        __syncthreads();
        const int ars = Aa[sb], brs = Ba[sb];
        const int Da = zz[0] + ars * brs;                 // D''_a = A_a.B~_b + a_ab B~_ab
        const int Db = zz[1] + ars * brs;
        if (t < RLB_TOUCH) {
            // touching entries: 2 threads per v, half of the row blocks each
            const int v = t >> 1, part = t & 1;
            int xa = 0, xb = 0, ya = 0, yb = 0;
            if (v < n) rlb_dots(As + v * lda, Bt + v * ldb, Aa, Ab, Ba, Bb, part, 2, nb, xa, xb, ya, yb);
            xa += __shfl_xor_sync(0xffffffffu, xa, 1);
            xb += __shfl_xor_sync(0xffffffffu, xb, 1);
            ya += __shfl_xor_sync(0xffffffffu, ya, 1);
            yb += __shfl_xor_sync(0xffffffffu, yb, 1);
            if (part == 0 && v < n && v != sa && v != sb) {
                const int av = Aa[v], bv = Ab[v], abv = Ba[v], bbv = Bb[v];
                const int da = av - bv, db = abv - bbv;
                const int dv = Dg[v] - da * db;           // D''_v = D_v - dA_v dB_v
                Dg[v] = dv;
                // R10b: δ''(a,v) and δ''(b,v) from pre-swap rows
                D[v > sa ? rowaddr[sa] + v : rowaddr[v] + sa] =
                    2 * (xa + ars * db + yb - da * brs - Da - dv + 2 * av * bbv);
                D[v > sb ? rowaddr[sb] + v : rowaddr[v] + sb] =
                    2 * (xb - ars * db + ya + da * brs - Db - dv + 2 * bv * abv);
            }
        } else {
            // disjoint entries (R10): quads g = qt, qt + 512, ... (consecutive threads read
            // consecutive 16-byte quads of Δ~, which streams through L2); rows sa, sb skipped,
            // columns sa, sb left to the touching threads.  RLB_QB loads in flight per thread.
            const int qt = t - RLB_TOUCH;
            constexpr int QS = RLB_NT - RLB_TOUCH;
#pragma unroll 1
            for (int g0 = qt; g0 < nqt; g0 += RLB_QB * QS) {
                int4 d4[RLB_QB];
                uint32_t desc[RLB_QB];
#pragma unroll
                for (int i = 0; i < RLB_QB; ++i) {
                    const int g = g0 + i * QS;
                    desc[i] = g < nqt ? (uint32_t)qdesc[g] : 0xFFFFu;
                    const int u = desc[i] & 511;
                    if (desc[i] != 0xFFFFu && u != sa && u != sb)
                        d4[i] = *reinterpret_cast<const int4*>(D + 4 * g);
                }
#pragma unroll
                for (int i = 0; i < RLB_QB; ++i) {
                    const int u = desc[i] & 511, v0 = (desc[i] >> 9) << 2;
                    if (desc[i] == 0xFFFFu || u == sa || u == sb) continue;
                    const int g = g0 + i * QS;
                    const int2 pu = stg[u];
                    const int4 x = *reinterpret_cast<const int4*>(stg + v0);
                    const int4 y = *reinterpret_cast<const int4*>(stg + v0 + 2);
                    const int4 nv = make_int4(d4[i].x + 2 * (pu.x - x.x) * (pu.y - x.y),
                                              d4[i].y + 2 * (pu.x - x.z) * (pu.y - x.w),
                                              d4[i].z + 2 * (pu.x - y.x) * (pu.y - y.y),
                                              d4[i].w + 2 * (pu.x - y.z) * (pu.y - y.w));
                    const unsigned er = (unsigned)(sa - v0), es = (unsigned)(sb - v0);
                    if (__builtin_expect(er >= 4u && es >= 4u, 1)) {
                        *reinterpret_cast<int4*>(D + 4 * g) = nv;
                    } else {                              // column sa or sb in this quad
                        if (er != 0u && es != 0u) D[4 * g + 0] = nv.x;
                        if (er != 1u && es != 1u) D[4 * g + 1] = nv.y;
                        if (er != 2u && es != 2u) D[4 * g + 2] = nv.z;
                        if (er != 3u && es != 3u) D[4 * g + 3] = nv.w;
                    }
                }
            }
        }
        if (t == 0) {                                     // scalar state
            const uint16_t x = q[sa];
            q[sa] = q[sb];
            q[sb] = x;
            cost += dw;
            const int improved = cost < best;
            if (improved) best = cost;
            flags[0] = improved;
            my_dig += mix64(mix64(kacc) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)sl));
            ++my_cnt;
            D[rowaddr[sa] + sb] = -dw;                    // swapping back restores C
            Dg[sa] = Da;
            Dg[sb] = Db;
        }
        __syncthreads();
        pa = sa;
        pb = sb;
        k = kacc + 1;
        s0 += cons;
        if (s0 >= n) { ++r; if (r >= n - 1) r = 0; s0 = r + 1; }
        rejT = 38.5f * temp32(a.sch, k);
    }
    if (pa >= 0 && flags[0])
        for (int x = t; x < n; x += RLB_NT) bestp[x] = q[sig[x]];

    // ---- write back in location space: p = q∘σ, Δ(u,v) = Δ~(σu, σv)
    for (int o = 16; o; o >>= 1) {
        my_dig += __shfl_xor_sync(0xffffffffu, my_dig, o);
        my_cnt += __shfl_xor_sync(0xffffffffu, my_cnt, o);
    }
    if (lane == 0) {
        atomicAdd(&red[0], my_dig);
        atomicAdd(&red[1], my_cnt);
    }
    __syncthreads();
    for (int x = t; x < n; x += RLB_NT) {
        a.p[x] = q[sig[x]];
        a.best_p[x] = bestp[x];
    }
    for (int g = t; g < nqt; g += RLB_NT) {
        const uint32_t desc = a.qdesc[g];
        const int u = desc & 511, v0 = (desc >> 9) << 2;
        const int su = sig[u];
        int4 o4;
        int* o = &o4.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int v = v0 + e;
            int val = 0;
            if (v > u && v < n) {
                const int sv = sig[v];
                val = D[su < sv ? rowaddr[su] + sv : rowaddr[sv] + su];
            }
            o[e] = val;
        }
        *reinterpret_cast<int4*>(ra.d_out + 4 * g) = o4;
    }
    if (t == 0) {
        a.st->cost = cost;
        a.st->best_cost = best;
        a.st->digest = a.st->digest + red[0];
        a.st->accepted += red[1];
    }
}

}  // namespace qapsa
