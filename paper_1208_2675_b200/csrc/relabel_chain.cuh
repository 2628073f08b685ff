// relabel_chain.cuh -- the single-chain engine for instances with 8-bit A and 16-bit B up to
// N = 256 (BASELINE config 4; also 8-bit B when 128 < N <= 256), with exact O(1) relabel swaps
// for twin locations
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
// Per cross accept (slots a < b), 256 threads per CTA:
//   window  one candidate per thread, decided by one shared-memory load of the exact integer
//           threshold of its iteration (k_theta, theta_ring.cuh, R23; flagged iterations take the
//           general float-θ / exact-double test)
//   stage   dA_x = A_ax - A_bx, dB_x = B~_ax - B~_bx, D''_x = D_x - dA_x dB_x; Z_a = A_a.B~_b,
//           Z_b = A_b.B~_a (warps 8..15)
//   quads   all threads: Δ~ += 2(dA_u - dA_v)(dB_u - dB_v) for every pair off rows a, b (R10), one
//           16-byte quad at a time (on a cluster: the CTA's share, in its shared memory)
//   touch   the four dot products of every v, X_a = B~_v.A_a, X_b, Y_a = A_v.B~_a, Y_b, on the
//           CUDA cores (dp4a over the byte planes B~ = 256 Bh + Bl and A, one warp per v); on a
//           cluster each CTA computes N / 8 rows v and stores δ''(a,v), δ''(b,v) (R10b) into the
//           owner of the entry (distributed shared memory)
//   next window: B~ rows / columns a, b exchanged, best_p = q∘σ if the cost improved
//
// Shared memory (N = 256): [Bh | Bl | A] in the K-major canonical layout (tc_common.cuh), 192 KB,
// is the only copy of A and B~.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "theta_ring.cuh"

namespace qapsa {

constexpr int RLB_NT = 256;     // one thread per window candidate (a window is <= 255 candidates)
constexpr int RLB_NW = RLB_NT / 32;
constexpr int RLB_MAXN = 256;
constexpr int RLB_MAXCLS = 4;   // twin classes (>= 2 members) the relabel path handles
#ifndef RLB_QB_EXP
constexpr int RLB_QB = 4;       // quad loads in flight per thread
#else
constexpr int RLB_QB = RLB_QB_EXP;
#endif
constexpr int RLB_K = 768;      // K of the touching product: Bh | Bl | A
constexpr int RLB_SBO = RLB_K / 16 * 128;        // 8-row group stride of the canonical layout
constexpr int RLB_BL = 256, RLB_AOFF = 512;      // K offsets of the Bl and A parts

struct RlbLayout {
    int op1, dsh, rowaddr, qdesc, pt, cls, sig, q, bestp, dg, stg, slots, twm, ab, zz, flags, red,
        ring, tbar, bytes;
};
constexpr int RLB_RS = 4, RLB_RB = 256;          // threshold ring: 4 blocks of 256 (a window is <= 255)
// quads of Δ~ owned by each CTA of a cluster of CL (quad g belongs to CTA g % CL)
__host__ __device__ constexpr int rlb_share(int n, int CL) { return (quad_count(n) + CL - 1) / CL; }
// CL = 1: Δ~ in global memory, all quad descriptors in shared memory; CL > 1: this CTA's share of
// Δ~ and of the descriptors in shared memory
__host__ __device__ constexpr RlbLayout rlb_layout(int n, int CL = 1) {
    RlbLayout L{};
    const int n4 = (n + 3) & ~3;
    int o = 0;
    L.op1 = o;     o += RLB_MAXN / 8 * RLB_SBO;          // 256 rows x 768 B, canonical K-major
    L.dsh = o;     o += CL > 1 ? rlb_share(n, CL) * 16 : 0;
    L.rowaddr = o; o = align16(o + n * 4);
    L.qdesc = o;   o = align16(o + (CL > 1 ? rlb_share(n, CL) : quad_count(n)) * 2);
    L.pt = o;      o = align16(o + RLB_MAXCLS * (n + 1) * 2);
    L.cls = o;     o = align16(o + n4);
    L.sig = o;     o = align16(o + n * 2);
    L.q = o;       o = align16(o + n * 2);
    L.bestp = o;   o = align16(o + n * 2);
    L.dg = o;      o = align16(o + n * 4);
    L.stg = o;     o = align16(o + n4 * 4);
    L.slots = o;   o = align16(o + 2 * RLB_NW * 16);
    L.twm = o;     o = align16(o + 2 * RLB_NW * 4);
    L.ab = o;      o = align16(o + RLB_MAXN * 8);         // stage: (A_a | A_b << 16, B~_a | B~_b << 16) per x
    L.zz = o;      o = align16(o + 16 * 4);
    L.flags = o;   o = align16(o + 4 * 4);
    L.red = o;     o = align16(o + 2 * 8);
    L.ring = o;    o += RLB_RS * RLB_RB * 4;            // exact integer thresholds (theta_ring.cuh, R23)
    L.tbar = o;    o += RLB_RS * 8;
    L.bytes = o;
    return L;
}

struct RelabelArgs {
    ChainArgs c;               // A, B (global, stride c.ld), p, best_p, D (working Δ~), ...
    const uint8_t* cls;        // n: twin class of location x in [0, ncls), 0xFF = none
    const uint16_t* pt;        // ncls x (n+1): largest member of class c below x, 0xFFFF = none
    int ncls;
    int b8;                    // B stored as 8-bit (N > 128 instances with small entries)
    int32_t* d_out;            // Δ in location space at exit (quad layout)
};

// element accessors of the canonical operand (row x, K offset k)
__device__ __forceinline__ int rlb_off(int x, int k) { return tc::kmaj_off(x, k, RLB_SBO); }
__device__ __forceinline__ int rlb_A(const uint8_t* op1, int x, int k) { return op1[rlb_off(x, RLB_AOFF + k)]; }
__device__ __forceinline__ int rlb_B(const uint8_t* op1, int x, int k) {
    return ((int)op1[rlb_off(x, k)] << 8) | (int)op1[rlb_off(x, RLB_BL + k)];
}

// ---- thread-block cluster helpers (f1: Δ~ spread over the shared memory of CL CTAs)
__device__ __forceinline__ int cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_store(int32_t* local, int rank, int v) {  // *local in CTA `rank` = v
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(local)), "r"(rank));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ int cl_load(const int32_t* local, int rank) {   // *local in CTA `rank`
    uint32_t ra, v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(local)), "r"(rank));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
    return (int)v;
}

// CL = 1: one CTA, Δ~ in global memory / L2.  CL > 1 (launched as a cluster of CL CTAs): every
// CTA runs the same chain (same decisions, replicated σ, q, B~, stage and touching products) but
// owns only the quads g with g % CL == its rank, in shared memory; window reads of other CTAs'
// quads go through distributed shared memory; two split cluster barriers per non-twin accept
// (reads of the window done -> writes of the update; writes done -> next window's reads).
template <int NFIX, int CL>
__global__ void __launch_bounds__(RLB_NT, 1) k_sa_relabel(const RelabelArgs ra) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ChainArgs& a = ra.c;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = NFIX ? NFIX : a.n;
    const int ldg = a.ld;
    const int M = n * (n - 1) / 2;
    const int nqt = NFIX ? quad_count(NFIX) : a.nqt;
    const int ncls = ra.ncls;
    const RlbLayout L = rlb_layout(n, CL);
    const int crank = CL > 1 ? cl_rank() : 0;
    const int nql = CL > 1 ? (nqt - crank + CL - 1) / CL : nqt;   // quads this CTA owns
    int32_t* Ds = reinterpret_cast<int32_t*>(smem + L.dsh);       // CL > 1: local share of Δ~
    uint8_t* op1 = smem + L.op1;
    int32_t* rowaddr = reinterpret_cast<int32_t*>(smem + L.rowaddr);
    uint16_t* qdesc = reinterpret_cast<uint16_t*>(smem + L.qdesc);
    uint16_t* pt = reinterpret_cast<uint16_t*>(smem + L.pt);
    uint8_t* cls = smem + L.cls;
    uint16_t* sig = reinterpret_cast<uint16_t*>(smem + L.sig);
    uint16_t* q = reinterpret_cast<uint16_t*>(smem + L.q);
    uint16_t* bestp = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int32_t* Dg = reinterpret_cast<int32_t*>(smem + L.dg);
    int32_t* stg = reinterpret_cast<int32_t*>(smem + L.stg);   // 2 (1024 dB_x + dA_x)
    int4* slot_base = reinterpret_cast<int4*>(smem + L.slots);
    unsigned* twm_base = reinterpret_cast<unsigned*>(smem + L.twm);
    uint2* abx = reinterpret_cast<uint2*>(smem + L.ab);
    int* zz = reinterpret_cast<int*>(smem + L.zz);
    int* flags = reinterpret_cast<int*>(smem + L.flags);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(smem + L.red);
    int32_t* D = a.D;
    const uint8_t* Ag = reinterpret_cast<const uint8_t*>(a.A);
    const uint16_t* Bg = reinterpret_cast<const uint16_t*>(a.B);   // 16-bit B (ra.b8 == 0)
    const uint8_t* Bg8 = reinterpret_cast<const uint8_t*>(a.B);    // 8-bit B (ra.b8 == 1)

    // ---- load: tables, σ = id, q = p
    for (int i = t; i < n; i += RLB_NT) {
        rowaddr[i] = a.rowaddr[i];
        cls[i] = ra.cls[i];
        sig[i] = (uint16_t)i;
        q[i] = (uint16_t)a.p[i];
        bestp[i] = (uint16_t)a.best_p[i];
    }
    for (int i = t; i < ncls * (n + 1); i += RLB_NT) pt[i] = ra.pt[i];
    for (int i = t; i < nql; i += RLB_NT) qdesc[i] = a.qdesc[CL > 1 ? crank + CL * i : i];
    if (CL > 1)
        for (int i = t; i < nql; i += RLB_NT)
            reinterpret_cast<int4*>(Ds)[i] = reinterpret_cast<const int4*>(a.D)[crank + CL * i];
    if (t < 4) flags[t] = 0;
    if (t < 2) red[t] = 0ull;
    ThetaRing<RLB_RS, RLB_RB> TR = theta_ring<RLB_RS, RLB_RB>(
        reinterpret_cast<int*>(smem + L.ring), nullptr, reinterpret_cast<uint64_t*>(smem + L.tbar), a.theta,
        nullptr, a.theta_kb, a.theta_cnt, a.k0);
    if (t == 0 && a.k0 < a.k_end) TR.start(a.k0);
    __syncthreads();
    // op1 = [Bh | Bl | A] of the slots: B~ = B[q][q] split into bytes, A (zero beyond n)
    for (int idx = t; idx < RLB_MAXN * (RLB_K / 4); idx += RLB_NT) {
        const int x = idx / (RLB_K / 4), k = 4 * (idx - x * (RLB_K / 4));
        uint32_t w = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int kk = k + e;
            int v = 0;
            if (x < n) {
                if (kk >= RLB_AOFF) { if (kk - RLB_AOFF < n) v = Ag[x * ldg + kk - RLB_AOFF]; }
                else {
                    const int c = kk & 255;
                    if (c < n) {
                        const int b = ra.b8 ? (int)Bg8[q[x] * ldg + q[c]] : (int)Bg[q[x] * ldg + q[c]];
                        v = kk >= RLB_BL ? (b & 255) : (b >> 8);
                    }
                }
            }
            w |= (uint32_t)v << (8 * e);
        }
        *reinterpret_cast<uint32_t*>(op1 + rlb_off(x, k)) = w;
    }
    __syncthreads();
    for (int x = t; x < n; x += RLB_NT) {
        int acc = 0;
        for (int k = 0; k < n; ++k) acc += rlb_A(op1, x, k) * rlb_B(op1, x, k);
        Dg[x] = acc;
    }
    __syncthreads();
    if (CL > 1) { cl_arrive(); cl_wait(); }               // every CTA's share loaded

    // Δ~ entry e (int index of the quad layout; quad g lives in CTA g mod CL at slot g / CL):
    // write (owner only)
    auto dwr = [&](int e, int v) {                        // replicated value: owner stores
        if (CL == 1) { D[e] = v; return; }
        const int g = e >> 2;
        if (g % CL == crank) Ds[4 * (g / CL) + (e & 3)] = v;
    };
    auto dput = [&](int e, int v) {                       // value computed by this CTA only
        if (CL == 1) { D[e] = v; return; }
        const int g = e >> 2, own = g % CL;
        int32_t* loc = Ds + 4 * (g / CL) + (e & 3);
        cl_store(loc, own, v);                            // (own rank too: no divergent branch)
    };
    bool pend_wait = false;                               // CL > 1: writes of the last update
    const NearSink sink{a.near_count, a.near_k, a.near_dec, a.near_cap, nullptr, nullptr, 0u};
    int64_t cost = a.st->cost, best = a.st->best_cost;   // scalar thread (t == RLB_NT - 1)
    uint64_t my_dig = 0, my_cnt = 0;                     // this thread's accepts (digest is a sum)
    uint64_t k = a.k0;
    const uint64_t k_end = a.k_end;
    int r, s0;
    tri_pair(n, (int)(k % (uint64_t)M), &r, &s0);
    int parity = 0, pa = -1, pb = -1;
    float rejT = 38.5f * temp32(a.sch, k);
    int ring_blo = -1, ring_hi = 0;
    // touching rows of this CTA: [vlo, vhi) (a cluster splits the N rows into CL slices)
    const int vrows = (n + CL - 1) / CL, vlo = crank * vrows, vhi = min(n, vlo + vrows);

    while (k < k_end) {
        const uint64_t remaining = k_end - k;
        const int Wl = (uint64_t)(n - s0) < remaining ? n - s0 : (int)remaining;

        // ---- deferred B~ exchange of the last cross accept (slots pa, pb) and best_p
        if (pa >= 0) {
            for (int x = t; x < n; x += RLB_NT) {        // columns pa, pb of the other rows
                if (x == pa || x == pb) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint8_t* ra_ = op1 + rlb_off(x, h * RLB_BL + pa);
                    uint8_t* rb_ = op1 + rlb_off(x, h * RLB_BL + pb);
                    const uint8_t v = *ra_;
                    *ra_ = *rb_;
                    *rb_ = v;
                }
            }
            {                                             // rows pa, pb (Bh and Bl), word-wise
                for (int w = t; w < 2 * RLB_BL / 4; w += RLB_NT) {
                    const int kk = 4 * w, c = kk & 255;
                    uint32_t m = 0;
                    if ((unsigned)(pa - c) < 4u) m |= 0xFFu << (8 * (pa - c));
                    if ((unsigned)(pb - c) < 4u) m |= 0xFFu << (8 * (pb - c));
                    uint32_t* Rw = reinterpret_cast<uint32_t*>(op1 + rlb_off(pa, kk));
                    uint32_t* Sw = reinterpret_cast<uint32_t*>(op1 + rlb_off(pb, kk));
                    const uint32_t x = *Rw, y = *Sw;
                    *Rw = (y & ~m) | (x & m);             // (pa,pa), (pa,pb), (pb,pa), (pb,pb) keep
                    *Sw = (x & ~m) | (y & m);             // their values (B~ symmetric, zero diag)
                }
            }
            if (flags[0])
                for (int x = t; x < n; x += RLB_NT) bestp[x] = q[sig[x]];
            pa = -1;
        }

        {   // thresholds of the window's iterations resident (theta_ring.cuh)
            const int ko = (int)(k - TR.kb);
            if (((ko >> 8) != ring_blo) | (ko + Wl > ring_hi)) {   // one uniform branch for both rare cases
                if ((ko >> 8) != ring_blo) {      // a block passed (warp-uniform test; one thread refills)
                    ring_blo = ko >> 8;
                    if (t == 0) TR.refill(k);
                }
                if (ko + Wl > ring_hi) {
                    TR.ensure_ofs(ko + Wl);
                    ring_hi = (int)(TR.ready * RLB_RB);
                }
            }
        }
        if (CL > 1 && pend_wait) { cl_wait(); pend_wait = false; }   // other CTAs' updates visible
        // ---- window: candidates (r, s0 + t), t < Wl
        const int cr = ncls ? cls[r] : 0xFF;
        // (branch-free: every lane loads; a lane past the window reads location r + 1 <= n - 1)
        bool near = false;
        const int s = s0 + t;
        const bool live = t < Wl;
        const int sc = live ? s : r + 1;
        const int pv = cr != 0xFF ? pt[cr * (n + 1) + sc] : 0xFFFF;
        const int sr = (pv != 0xFFFF && pv >= s0) ? sig[pv] : sig[r];   // σ(r) at this candidate
        const bool twin = live & (cr != 0xFF) & (cls[sc] == cr);
        const uint16_t newsig = (uint16_t)sr;             // σ(s) after the transposition (r s), if twin
        const int ss = sig[sc];
        const int ca = min(sr, ss), cb = max(sr, ss);   // the candidate's slot pair
        const int sab = (ca << 16) | cb;
        const bool cross = live & !twin;
        int d = 0;
        if (cross) {                                      // Δ~(sa, sb) from its owner CTA
            const int e = rowaddr[ca] + cb;
            if (CL == 1) d = D[e];
            else d = cl_load(Ds + 4 * ((e >> 2) / CL) + (e & 3), (e >> 2) % CL);
        }
        // exact integer threshold (R23); δ <= 0 accepted (R5); a flagged iteration (thr = -1)
        // with δ > 0 takes the general test (float θ with a margin, exact inside it, near ties
        // flagged) unless δ is a certain reject (chain.cuh)
        const int thr = TR.at_ofs((int)(k - TR.kb) + t);
        bool acc = cross & (d <= max(thr, 0));
        const bool need = cross & (thr < 0) & (d > 0) & ((float)d <= rejT);
        if (__any_sync(0xffffffffu, need)) {
            if (need) acc = metropolis_fast(d, a.sch, k + (uint64_t)t, a.seed, 0u, &near);
        }
        int4* slots = slot_base + parity * RLB_NW;
        unsigned* twm = twm_base + parity * RLB_NW;
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        const unsigned tw = __ballot_sync(0xffffffffu, twin);
        if (bal) {
            if (lane == __ffs(bal) - 1) slots[warp] = make_int4(t, d, sab, s);
        } else if (lane == 0) {
            slots[warp] = make_int4(INT_MAX, 0, 0, 0);
        }
        if (lane == 0) twm[warp] = tw;
        __syncthreads();
        const int j = __reduce_min_sync(0xffffffffu, lane < RLB_NW ? slots[lane].x : INT_MAX);
        parity ^= 1;
        const int cons = (j == INT_MAX) ? Wl : j + 1;
        // any twin among the consumed candidates (needs a barrier before σ is read again)
        const int lo = cons - 32 * lane;
        const unsigned below = lo >= 32 ? 0xffffffffu : (lo <= 0 ? 0u : ((1u << lo) - 1u));
        const bool any_twin = __reduce_or_sync(0xffffffffu, lane < RLB_NW ? twm[lane] & below : 0u) != 0u;
        if (near && t < cons && crank == 0) {             // R16: near ties of consumed iterations
            near_record(sink, k + (uint64_t)t, acc);
        }
        if (twin && t < cons) {                           // relabel: σ rotated, accept counted
            const uint16_t old = sig[s];
            sig[s] = newsig;
            if (pt[cr * (n + 1) + s0 + cons] == s) sig[r] = old;   // last consumed twin
            if (crank == 0) {
                ++my_cnt;
                my_dig += mix64(mix64(k + (uint64_t)t) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)s));
            }
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
        if (CL > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // window reads done (nothing to publish)
        const int4 win = slots[j >> 5];
        const int dw = win.y, sa = win.z >> 16, sb = win.z & 0xFFFF, sl = win.w;
        const uint64_t kacc = k + (uint64_t)j;
        // stage, Z (the new diagonal of slots a, b), the MMA's B operand W
        // dA in [-255, 255], dB in [-65535, 65535] packed as 2 (1024 dB + dA): the difference of two
        // packed values is 2048 (dB_u - dB_v) + 2 (dA_u - dA_v) with |dA_u - dA_v| <= 510, so
        // hi = (d + 1024) >> 11 and lo2 = d - 2048 hi recover both and lo2 * hi is the rank term
        {                                                 // x = t: the rows a, b of A and B~ at x once
            int za = 0, zb = 0;                           // Z_a = A_a.B~_b, Z_b = A_b.B~_a (R10b)
            if (t < n) {
                const int aa = rlb_A(op1, sa, t), ab_ = rlb_A(op1, sb, t);
                const int ba = rlb_B(op1, sa, t), bb = rlb_B(op1, sb, t);
                const int da = aa - ab_, db = ba - bb;
                stg[t] = 2 * (1024 * db + da);
                if (t != sa && t != sb) Dg[t] -= da * db; // D''_v = D_v - dA_v dB_v (R10b)
                za = aa * bb;
                zb = ab_ * ba;
                abx[t] = make_uint2((uint32_t)aa | ((uint32_t)ab_ << 16), (uint32_t)ba | ((uint32_t)bb << 16));
            }
            za = __reduce_add_sync(0xffffffffu, za);
            zb = __reduce_add_sync(0xffffffffu, zb);
            if (lane == 0) { zz[2 * warp] = za; zz[2 * warp + 1] = zb; }
        }
        __syncthreads();
        const int ars = rlb_A(op1, sa, sb), brs = rlb_B(op1, sa, sb);
        int Da = ars * brs, Db = ars * brs;               // D''_a = A_a.B~_b + a_ab B~_ab, D''_b
#pragma unroll
        for (int w = 0; w < 8; ++w) { Da += zz[2 * w]; Db += zz[2 * w + 1]; }
        if (t == RLB_NT - 1) {                            // scalar state (row sa is off the quads)
            const uint16_t x = q[sa];
            q[sa] = q[sb];
            q[sb] = x;
            cost += dw;
            const int improved = cost < best;
            if (improved) best = cost;
            flags[0] = improved;
            if (crank == 0) {
                my_dig += mix64(mix64(kacc) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)sl));
                ++my_cnt;
            }
            Dg[sa] = Da;
            Dg[sb] = Db;
        }
        __syncwarp();
        if (CL > 1) cl_wait();                            // every CTA done reading this window
        if (CL > 1) {
            // disjoint entries (R10) of this CTA's share, in shared memory
            int4* D4 = reinterpret_cast<int4*>(Ds);
#pragma unroll 1
            for (int li = t; li < nql; li += RLB_NT) {
                const uint32_t dsc = qdesc[li];
                const int u = dsc & 511, v0 = (dsc >> 9) << 2;
                const bool skip = (u == sa) | (u == sb);   // rows sa, sb: recomputed (R10b)
                const int pu = stg[u];
                const int4 x = *reinterpret_cast<const int4*>(stg + v0);
                int4 o = D4[li];
                int dd = pu - x.x, hi = (dd + 1024) >> 11;
                o.x += (dd - (hi << 11)) * hi;
                dd = pu - x.y; hi = (dd + 1024) >> 11;
                o.y += (dd - (hi << 11)) * hi;
                dd = pu - x.z; hi = (dd + 1024) >> 11;
                o.z += (dd - (hi << 11)) * hi;
                dd = pu - x.w; hi = (dd + 1024) >> 11;
                o.w += (dd - (hi << 11)) * hi;
                // columns sa, sb are the touching entries, stored (possibly by another CTA,
                // unordered with this store) after the quads: leave them alone
                const unsigned er = (unsigned)(sa - v0), es = (unsigned)(sb - v0);
                if (!skip & (er >= 4u) & (es >= 4u)) {
                    D4[li] = o;
                } else if (!skip) {
                    int32_t* q1 = Ds + 4 * li;
                    if (er != 0u && es != 0u) q1[0] = o.x;
                    if (er != 1u && es != 1u) q1[1] = o.y;
                    if (er != 2u && es != 2u) q1[2] = o.z;
                    if (er != 3u && es != 3u) q1[3] = o.w;
                }
            }
        } else {
            // disjoint entries (R10), every thread: quads g = t, t + 1024, ... (consecutive threads read
            // consecutive 16-byte quads of Δ~, which streams through L2); rows sa, sb skipped; quads
            // holding columns sa, sb are written whole here and their two entries overwritten by the
            // touching stores after the barrier below.  RLB_QB loads in flight per thread.
    #pragma unroll 1
            for (int g0 = t; g0 < nqt; g0 += RLB_QB * RLB_NT) {
                int4 d4[RLB_QB];
                unsigned need = 0;
    #pragma unroll
                for (int i = 0; i < RLB_QB; ++i) {
                    const int g = g0 + i * RLB_NT;
                    const int u = g < nqt ? (qdesc[g] & 511) : sa;
                    if (u != sa && u != sb) {
                        need |= 1u << i;
                        d4[i] = *reinterpret_cast<const int4*>(D + 4 * g);
                    }
                }
    #pragma unroll
                for (int i = 0; i < RLB_QB; ++i) {
                    if (!(need & (1u << i))) continue;
                    const int g = g0 + i * RLB_NT;
                    const uint32_t dsc = qdesc[g];
                    const int u = dsc & 511, v0 = (dsc >> 9) << 2;
                    const int pu = stg[u];
                    const int4 x = *reinterpret_cast<const int4*>(stg + v0);
                    int4 o = d4[i];
                    int dd = pu - x.x, hi = (dd + 1024) >> 11;
                    o.x += (dd - (hi << 11)) * hi;
                    dd = pu - x.y; hi = (dd + 1024) >> 11;
                    o.y += (dd - (hi << 11)) * hi;
                    dd = pu - x.z; hi = (dd + 1024) >> 11;
                    o.z += (dd - (hi << 11)) * hi;
                    dd = pu - x.w; hi = (dd + 1024) >> 11;
                    o.w += (dd - (hi << 11)) * hi;
                    *reinterpret_cast<int4*>(D + 4 * g) = o;
                }
            }
        }
        // touching entries (R10b) of this CTA's rows v in [vlo, vhi) on the CUDA cores: the four
        // dot products X_a = B~_v.A_a, X_b, Y_a = A_v.B~_a, Y_b by dp4a over the byte planes
        // B~ = 256 Bh + Bl and A.  A warp takes 8 rows v = v8 .. v8 + 7 (one 8-row group of the
        // canonical layout, so the 8 lanes of a quarter warp read 128 contiguous bytes): lane l
        // handles row v8 + (l & 7) and the 16-byte K chunks l / 8, + 4, + 8, + 12; the 4 partial
        // sums of a row are added with two shuffles.  Lane l (l < 8) keeps row v8 + l's entries.
        // touching entries (R10b) of this CTA's rows v in [vlo, vhi) on the CUDA cores: the four
        // dot products X_a = B~_v.A_a, X_b, Y_a = A_v.B~_a, Y_b by dp4a over the byte planes
        // B~ = 256 Bh + Bl and A.  A warp pass takes 8 rows v8 .. v8 + 7 (one 8-row group of the
        // canonical layout, so the 8 lanes of a quarter warp read 128 contiguous bytes): lane l
        // handles row v8 + (l & 7) and the 16-byte K chunks l / 8, + 4, + 8, + 12; the 4 partial
        // sums of a row are added with two shuffles and lane l < 8 keeps row v8 + l's entries.
        constexpr int NPASS = (RLB_MAXN + 7 + 8 * RLB_NW - 1) / (8 * RLB_NW);   // 8-row groups per warp
        int wa[NPASS], wb[NPASS], va[NPASS], vb[NPASS];
#pragma unroll
        for (int ps_ = 0; ps_ < NPASS; ++ps_) { wa[ps_] = -1; wb[ps_] = -1; va[ps_] = 0; vb[ps_] = 0; }
        {
            const int rl = lane & 7, cq = lane >> 3;
#pragma unroll
            for (int pass = 0; pass < NPASS; ++pass) {
                const int v8 = (vlo & ~7) + 8 * warp + pass * 8 * RLB_NW;
                if (v8 >= vhi) break;
                const int v = v8 + rl;
                unsigned s8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};   // Xa h/l, Xb h/l, Ya h/l, Yb h/l
                // row bases of the canonical layout; K chunk c of row x is at base_x + 128 c
                const uint8_t* pv = op1 + rlb_off(v, 16 * cq);
                const uint8_t* pa_ = op1 + rlb_off(sa, 16 * cq);
                const uint8_t* pb_ = op1 + rlb_off(sb, 16 * cq);
                constexpr int CH = 128, CA = RLB_AOFF / 16 * 128, CL_ = RLB_BL / 16 * 128;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int o = 4 * i * CH;
                    const uint4 Av = *reinterpret_cast<const uint4*>(pv + CA + o);
                    const uint4 Hv = *reinterpret_cast<const uint4*>(pv + o);
                    const uint4 Lv = *reinterpret_cast<const uint4*>(pv + CL_ + o);
                    const uint4 Aa = *reinterpret_cast<const uint4*>(pa_ + CA + o);
                    const uint4 Ab = *reinterpret_cast<const uint4*>(pb_ + CA + o);
                    const uint4 Ha = *reinterpret_cast<const uint4*>(pa_ + o);
                    const uint4 La = *reinterpret_cast<const uint4*>(pa_ + CL_ + o);
                    const uint4 Hb = *reinterpret_cast<const uint4*>(pb_ + o);
                    const uint4 Lb = *reinterpret_cast<const uint4*>(pb_ + CL_ + o);
                    auto dot = [](uint4 x, uint4 y, unsigned c) {
                        return __dp4a(x.x, y.x, __dp4a(x.y, y.y, __dp4a(x.z, y.z, __dp4a(x.w, y.w, c))));
                    };
                    s8[0] = dot(Hv, Aa, s8[0]); s8[1] = dot(Lv, Aa, s8[1]);
                    s8[2] = dot(Hv, Ab, s8[2]); s8[3] = dot(Lv, Ab, s8[3]);
                    s8[4] = dot(Av, Ha, s8[4]); s8[5] = dot(Av, La, s8[5]);
                    s8[6] = dot(Av, Hb, s8[6]); s8[7] = dot(Av, Lb, s8[7]);
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    s8[e] += __shfl_xor_sync(0xffffffffu, s8[e], 8);
                    s8[e] += __shfl_xor_sync(0xffffffffu, s8[e], 16);
                }
                if (cq == 0 && v >= vlo && v < vhi && v != sa && v != sb) {
                    const int xa = (int)(s8[0] * 256u + s8[1]);    // X_a = B~_v.A_a
                    const int xb = (int)(s8[2] * 256u + s8[3]);    // X_b = B~_v.A_b
                    const int ya = (int)(s8[4] * 256u + s8[5]);    // Y_a = A_v.B~_a
                    const int yb = (int)(s8[6] * 256u + s8[7]);    // Y_b = A_v.B~_b
                    const uint2 abv_ = abx[v];                     // the stage's A_a, A_b, B~_a, B~_b at v
                    const int av = (int)(abv_.x & 0xFFFFu), bv = (int)(abv_.x >> 16);
                    const int abv = (int)(abv_.y & 0xFFFFu), bbv = (int)(abv_.y >> 16);
                    const int da = av - bv, db = abv - bbv;
                    const int dv = Dg[v];                 // D''_v (updated in the stage)
                    // R10b: δ''(a,v) and δ''(b,v) from pre-swap rows
                    wa[pass] = v > sa ? rowaddr[sa] + v : rowaddr[v] + sa;
                    va[pass] = 2 * (xa + ars * db + yb - da * brs - Da - dv + 2 * av * bbv);
                    wb[pass] = v > sb ? rowaddr[sb] + v : rowaddr[v] + sb;
                    vb[pass] = 2 * (xb - ars * db + ya + da * brs - Db - dv + 2 * bv * abv);
                }
            }
        }
        __syncthreads();                                  // quads written: columns sa, sb next
#pragma unroll
        for (int ps_ = 0; ps_ < NPASS; ++ps_) {
            if (wa[ps_] >= 0) {                           // this CTA computed them: store anywhere
                dput(wa[ps_], va[ps_]);
                dput(wb[ps_], vb[ps_]);
            }
        }
        if (t == RLB_NT - 1) dwr(rowaddr[sa] + sb, -dw);  // swapping back restores C
        // this CTA's update written: on a cluster the split barrier orders the stores before the
        // next window's reads (its wait comes first there); on one SM a CTA barrier does
        if (CL > 1) { cl_arrive(); pend_wait = true; }
        else __syncthreads();
        pa = sa;
        pb = sb;
        k = kacc + 1;
        s0 += cons;
        if (s0 >= n) { ++r; if (r >= n - 1) r = 0; s0 = r + 1; }
        rejT = 38.5f * temp32(a.sch, k);
    }
    if (pa >= 0 && flags[0])
        for (int x = t; x < n; x += RLB_NT) bestp[x] = q[sig[x]];
    if (CL > 1) {
        // every CTA's share back to global memory (slot space), visible to the whole cluster
        if (pend_wait) cl_wait();
        for (int li = t; li < nql; li += RLB_NT)
            reinterpret_cast<int4*>(D)[crank + CL * li] = reinterpret_cast<const int4*>(Ds)[li];
        __threadfence();
        cl_arrive();
        cl_wait();
    }

    // ---- write back in location space: p = q∘σ, Δ(u,v) = Δ~(σu, σv)
    for (int o = 16; o; o >>= 1) {
        my_dig += __shfl_xor_sync(0xffffffffu, my_dig, o);
        my_cnt += __shfl_xor_sync(0xffffffffu, my_cnt, o);
    }
    if (lane == 0) {
        atomicAdd(&red[0], my_dig);
        atomicAdd(&red[1], my_cnt);
    }
    if (t == 0) TR.drain();
    __syncthreads();
    if (crank == 0)
        for (int x = t; x < n; x += RLB_NT) {
            a.p[x] = q[sig[x]];
            a.best_p[x] = bestp[x];
        }
    for (int g = crank * RLB_NT + t; g < nqt; g += CL * RLB_NT) {
        const uint32_t desc = CL > 1 ? (uint32_t)a.qdesc[g] : (uint32_t)qdesc[g];
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
                val = __ldcg(D + (su < sv ? rowaddr[su] + sv : rowaddr[sv] + su));
            }
            o[e] = val;
        }
        *reinterpret_cast<int4*>(ra.d_out + 4 * g) = o4;
    }
    if (t == RLB_NT - 1 && crank == 0) {
        a.st->cost = cost;
        a.st->best_cost = best;
        a.st->digest = a.st->digest + red[0];
        a.st->accepted += red[1];
    }
}

}  // namespace qapsa
