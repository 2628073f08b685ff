// scratch_chain.cuh -- the high-acceptance phase of a single chain without Δ: SURVEY §8(f) row f2,
// "hybrid scratch / Δ mode with an acceptance-rate switch".
//
// While swaps are accepted every few iterations, maintaining all of Δ costs an O(N^2) update per
// accept but each δ is read once or twice before it changes again.  This kernel keeps instead
//   G[x][f] = sum_k a_xk B[f][p(k)]     (= (A B'^T)[x][p^-1(f)]),   H = G^T,
// in tensor memory (tensor-memory engine, tc_chain.cuh, reading R10c) and evaluates every
// candidate's δ from its definition in O(1) (P:46 / S:76 with the sums expanded, R10d):
//   δ(u,v) = 2 (G_uv + G_vu - D_u - D_v + 2 a_uv B'_uv),   G_uv = (A B'^T)_uv, D_x = G_xx,
// with G_uv = H[p(v)][u] and G_vu = G[v][p(u)].  An accepted swap changes G by the exact rank-1
// term -(a_xr - a_xs)(B[f][p(r)] - B[f][p(s)]) (one tcgen05 int8 MMA on [G | H]) and D by
// D''_v = D_v - dA_v dB_v, D''_r = G_r,p(s) + a_rs B'_rs, D''_s = G_s,p(r) + a_rs B'_rs.
//
// The kernel runs from k0 until k_end or until accepts become rare (no accept for
// TCS_SWITCH_GAP iterations); it then stores p, best_p and the scalars and reports the iteration
// reached, and qap_sa_run rebuilds Δ (k_delta_init) and continues with the Δ engine (k_sa_tc).
// Every quantity is an exact integer, so the trajectory is the same whatever the switch point.
//
// Threads: 4 lane warps (thread v = TMEM lane v = location v = facility v) and 4 helper warps
// (MMA issue, thresholds of the next window, digest).
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "tc_chain.cuh"
#include "theta_ring.cuh"

namespace qapsa {

constexpr int TCS_NT = 288;            // 8 row warps (two window rows each) + 1 helper warp (MMA, digest)
constexpr int TCS_RW = 8;              // row warps
// ensemble launches add a θ producer warp: thresholds of the chain's coming iterations into a
// shared-memory ring (each θ computed once, instead of per candidate and window)
constexpr int TCS_EB = 256;            // producer block (iterations)
constexpr int TCS_ERING = 2048;        // ring (iterations, 8 blocks; windows are <= 4 rows < 1792)
template <bool ENS> __host__ __device__ constexpr int tcs_nt() { return ENS ? TCS_NT + 32 : TCS_NT; }
constexpr uint32_t TCS_COL_G = 0;        // G: TMEM columns [0, 128)
constexpr uint32_t TCS_COL_H = 128;      // H: TMEM columns [128, 256)
constexpr uint32_t TCS_COL_L = 256;      // single chain: A operand of the update [dA, -dBf] (K = 32)
// TMEM columns: a single chain keeps the update's A operand in TMEM (512 columns); an ensemble
// launch keeps it in shared memory so that G and H (256 columns) let two chains share an SM
template <bool ENS> __host__ __device__ constexpr uint32_t tcs_cols() { return ENS ? 256u : 512u; }
constexpr uint64_t TCS_SWITCH_GAP = 4096;   // switch to the Δ engine after this many iterations without an accept

struct ScLayout {
    int a, b, rg, la, tmp, p, bestp, dg, xch, slots, rec, misc, tbar, thdr, ering, ebar, ectl, bytes;
};
__host__ __device__ inline ScLayout sc_layout(int ld) {
    ScLayout L;
    int o = 0;
    L.a = o;     o += 128 * ld;
    L.b = o;     o += 128 * ld;
    o = (o + 1023) & ~1023;
    L.rg = o;    o += 256 * 32;                 // [G | H] update B operand, K-major canonical (SBO 256)
    L.la = o;    o += 128 * 32;                 // its A operand [dA, -dBf], same layout
    L.tmp = o;   o += 2 * 128 * 128;            // init: A, C canonical (SBO 1024); then the θ ring
    L.p = o;     o += 128 * 2;
    L.bestp = o; o += 128 * 2;
    L.dg = o;    o += 128 * 4;                  // D_x
    L.xch = o;   o += 4 * 128 * 4;              // G[u_i][p(v)] by window row i and location v
    L.slots = o; o += 2 * TCS_RW * 16;
    L.rec = o;   o += 32;                       // the accept for the helpers, double-buffered
    L.misc = o;  o += 64;                       // mbarrier | TMEM base
    L.tbar = o;  o += TH_SLOTS * 8;             // threshold ring mbarriers
    L.thdr = o;  o += TH_SLOTS * 16;            // threshold ring block headers
    L.ering = o; o += TCS_ERING * 8;            // ensemble: integer (θ - m, θ + m) ring of the producer warp (int_bracket)
    L.ebar = o;  o += (TCS_ERING / TCS_EB) * 16; //   its block mbarriers: full[NB], empty[NB]
    L.ectl = o;  o += 16;                       //   stop flag
    L.bytes = o;
    return L;
}

// Window geometry of this row warp (rows h2, h2 + 1 of the window at cursor (u0, v0), at most W
// candidates and rem iterations): rf = first column of the row (n if the row is not in the window),
// rb = offset base (candidate (u0 + i, v) has offset rb + v), Wl = candidates in the window.
// Window geometry of this warp's rows i = h2 + e: row i's candidates are the locations
// v in [rf, n) at offsets o = rb + v; v takes part iff 0 <= v - rf < lim (lim = the row's
// candidates inside the window, 0 for rows past the window), one unsigned compare.
struct ScWin { int Wl; int rb[2]; int rf[2]; int lim[2]; };
__device__ __forceinline__ ScWin sc_win(int n, int u0, int v0, int W, uint32_t rem, int h2) {
    const int R = win_rows<4>(n, u0), L0 = n - v0, m1 = n - 1 - u0;
    ScWin w;
    w.Wl = min(win_f(R, L0, m1), W);
    if ((uint32_t)w.Wl > rem) w.Wl = (int)rem;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int i = h2 + e;
        const int f = i == 0 ? 0 : win_f(i, L0, m1);
        w.rf[e] = i >= R ? n : i == 0 ? v0 : u0 + i + 1;
        w.rb[e] = f - w.rf[e];
        w.lim[e] = i >= R ? 0 : max(0, min(w.Wl - f, n - w.rf[e]));
    }
    return w;
}

template <int NFIX, bool ENS = false>
__global__ void __launch_bounds__(tcs_nt<ENS>(), ENS ? 2 : 1) k_sa_scratch(const ChainArgs a, unsigned long long* k_out) {
    constexpr bool RING = !ENS;                  // single chain: precomputed θ (theta_ring.cuh)
    extern __shared__ __align__(16) unsigned char smem[];
    const ChainView cv = chain_view<ENS>(a);     // this CTA's chain (ensemble launches)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = NFIX ? NFIX : a.n;
    const int ld = NFIX ? row_stride(NFIX, true) : a.ld;
    const int M = n * (n - 1) / 2;
    const ScLayout L = sc_layout(ld);
    uint8_t* As = smem + L.a;
    uint8_t* Bs = smem + L.b;
    uint8_t* Rg = smem + L.rg;
    uint8_t* La = smem + L.la;
    uint16_t* p = reinterpret_cast<uint16_t*>(smem + L.p);
    uint16_t* best_p = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int* Dg = reinterpret_cast<int*>(smem + L.dg);
    int* xch = reinterpret_cast<int*>(smem + L.xch);
    int4* slots = reinterpret_cast<int4*>(smem + L.slots);
    int* rec = reinterpret_cast<int*>(smem + L.rec);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.misc);          // G|H update done
    int2* ering = reinterpret_cast<int2*>(smem + L.ering);                // ensemble θ bracket ring
    uint64_t* ebar = reinterpret_cast<uint64_t*>(smem + L.ebar);          // [0, NB) full, [NB, 2NB) empty
    volatile int* ectl = reinterpret_cast<volatile int*>(smem + L.ectl);  // [1] stop
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.misc + 8);
    const bool lanew = warp < 4;                 // lane warps: thread v owns TMEM lane v (one per v)
    const bool roww = warp < TCS_RW;             // row warps: window rows 2h, 2h + 1 (h = warp / 4)
    const int h2 = 2 * (warp >> 2);
    const uint32_t quad_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int v = t & 127;
    const bool vin = v < n;

    // ---------------- load the chain state; G and H on the tensor cores ----------------
    constexpr int NT = tcs_nt<ENS>();
    copy_words(As, a.A, n * ld, t, NT);
    copy_words(Bs, a.B, n * ld, t, NT);
    for (int i = t; i < n; i += NT) {
        p[i] = (uint16_t)cv.p[i];
        best_p[i] = (uint16_t)cv.best_p[i];
    }
    for (int i = t; i < (256 + 128) * 32 / 16; i += NT) reinterpret_cast<uint4*>(Rg)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tc::tmem_alloc(tmem_slot, tcs_cols<ENS>());
    if (t == 0) tc::mbar_init(mbar, 1);
    if (ENS && t == 0) {                         // θ producer ring: block barriers, consumer offset 0, no stop
        for (int b = 0; b < 2 * (TCS_ERING / TCS_EB); ++b) tc::mbar_init(reinterpret_cast<uint64_t*>(smem + L.ebar) + b, 1);
        reinterpret_cast<int*>(smem + L.ectl)[0] = 0;
        reinterpret_cast<int*>(smem + L.ectl)[1] = 0;
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tmem_slot;
    if (!ENS && lanew) {
        tc::tmem_st4(tm + quad_lane + TCS_COL_L, 0u, 0u, 0u, 0u);
        tc::tmem_st4(tm + quad_lane + TCS_COL_L + 4, 0u, 0u, 0u, 0u);
        tc::tmem_wait_st();
    }
    {
        uint8_t* Ac = smem + L.tmp;
        uint8_t* Cc = Ac + 128 * 128;
        for (int idx = t; idx < 128 * 128; idx += NT) {
            const int x = idx >> 7, kk = idx & 127;
            const bool in = x < n && kk < n;
            Ac[cofs(x, kk)] = in ? As[x * ld + kk] : (uint8_t)0;
            Cc[cofs(x, kk)] = in ? Bs[x * ld + p[kk]] : (uint8_t)0;
        }
        tc::fence_proxy_async();
        tc::fence_before_sync();
        __syncthreads();
        if (t == 0) {                            // G = A C^T, H = C A^T
            tc::fence_after_sync();
            const uint32_t id = tc::idesc_i8(128, 128, true);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + TCS_COL_G, tc::smem_desc(tc::smem_u32(Ac) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(Cc) + 256 * kc, 128, 1024), id, kc > 0);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + TCS_COL_H, tc::smem_desc(tc::smem_u32(Cc) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(Ac) + 256 * kc, 128, 1024), id, kc > 0);
            tc::mma_commit(mbar);
        }
    }
    int px = vin ? p[v] : 0;                     // p(v)
    int qv = 0;                                  // p^-1(v)
    for (int i = 0; i < n; ++i) qv = (p[i] == v) ? i : qv;
    if (lanew) {
        int dgv = 0;
        if (vin)
            for (int kk = 0; kk < n; ++kk) dgv += (int)As[v * ld + kk] * (int)Bs[px * ld + p[kk]];
        Dg[v] = dgv;
    }
    tc::mbar_wait(mbar, 0);
    uint32_t ph = 1;
    tc::fence_after_sync();
    // single chain: θ of the window from the precomputed ring (reuses the init operands' space)
    ThetaRing<TH_SLOTS> TR = theta_ring<TH_SLOTS>(
        reinterpret_cast<int*>(smem + L.tmp), reinterpret_cast<int4*>(smem + L.thdr),
        reinterpret_cast<uint64_t*>(smem + L.tbar), a.theta, a.theta_hdr, a.theta_kb, a.theta_cnt, a.k0);
    if (RING && t == 0 && a.k0 < a.k_end) TR.start(a.k0);
    __syncthreads();

    const Sched sch = a.sch;
    const uint64_t seed = a.seed, k_end = a.k_end;
    const NearSink sink = cv.sink;
    int64_t cost = cv.st->cost, best = cv.st->best_cost;
    uint64_t digest = cv.st->digest;
    // iterations relative to k0 in 32 bits: this launch runs at most 2^31 - 1 of them (the caller
    // continues from the iteration reached, so the trajectory does not depend on the split)
    const uint64_t k0 = a.k0;
    const uint32_t kr_end = (uint32_t)min((unsigned long long)(a.k_end - k0), 0x7FFFFFFFull);
    uint32_t kr = 0, kr_last = 0;
    uint64_t accepted = 0;
    int u0, v0;
    tri_pair(n, (int)(k0 % (uint64_t)M), &u0, &v0);
    const int wmax = a.wmax;
    int W = wmax;
    int parity = 0;
    const uint32_t id_gh = tc::idesc_i8(128, 256, true);
    const int kofs0 = RING ? (int)(k0 - TR.kb) : 0;   // ring offset of iteration k0
#ifdef QAPSA_PHASE_TIMERS
    long long tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

  if (roww) {
    const uint32_t gap = a.switch_gap ? (uint32_t)min(a.switch_gap, (unsigned long long)0x7FFFFFFF) : (uint32_t)TCS_SWITCH_GAP;
    // The window's rows u_i = u0 + i, i < 4; this warp's are i = h2 + e, e < 2: pu[e] = p(u_i),
    // gv[e] = G[v][p(u_i)] (registers) and xch[i][v] = G_{u_i, v} (shared memory).  After an
    // accept they are produced by the stage from the PRE-update tensor memory plus the exact rank-1
    // change of the accept, so the next window is tested while the tensor cores apply that change
    // (the MMA is waited for only before the next read or write of tensor memory); after a window
    // without accept they are read afresh.  The window's geometry (ScWin) is likewise computed by
    // the stage for the next window.
    bool fresh = true;
    bool mma_pending = false;
    int pu[2];
    uint32_t gv[2];
    ScWin wg = sc_win(n, u0, v0, W, kr_end - kr, h2);
    int ring_blo = -1, ring_hi = 0;              // ring: last block refilled from, offsets known resident
    int ering_ready = 0, ering_freed = 0;        // ensemble: producer blocks known complete / released
    static_assert(TH_BLK == 1024, "ring_blo counts 1024-iteration blocks");
    while ((kr < kr_end) & (kr - kr_last < gap)) {
        // ---------------- window: rows u0 .. u0+R-1 (R <= 4) ----------------
        TCT_MARK(pt0, u0 + v0);
        const int Wl = wg.Wl;
        // the loop top's rare cases behind one uniform branch: a threshold block passed or not yet
        // known resident, or the window's rows to be read afresh
        const int ko = kofs0 + (int)kr;
        const bool slow = RING ? (((ko >> 10) != ring_blo) | (ko + Wl > ring_hi) | fresh) : true;
      if (slow) {
        if (RING) {
            if ((ko >> 10) != ring_blo) {     // a block passed: its slot can be refilled (uniform test)
                ring_blo = ko >> 10;
                if (t == 0) TR.refill(k0 + kr);
            }
            if (ko + Wl > ring_hi) {             // blocks not yet known complete
                TR.ensure_ofs(ko + Wl);
                ring_hi = (int)(TR.ready * TH_BLK);
            }
        } else {                                 // ensemble: the producer warp's ring
            constexpr int NB = TCS_ERING / TCS_EB;
            if (t == 0) {                        // blocks wholly below kr are consumed: free their slots
                for (; ering_freed < (int)(kr / TCS_EB); ++ering_freed) tc::mbar_arrive(ebar + NB + (ering_freed % NB));
            }
            if ((int)kr + Wl > ring_hi) {
                while (ering_ready * TCS_EB < (int)kr + Wl) {
                    tc::mbar_wait(ebar + (ering_ready % NB), (uint32_t)((ering_ready / NB) & 1));
                    ++ering_ready;
                }
                ring_hi = ering_ready * TCS_EB;
            }
        }
        if (fresh) {
            if (mma_pending) {                   // G, H complete before they are read
                tc::mbar_wait(mbar, ph);
                ph ^= 1;
                tc::fence_after_sync();
                mma_pending = false;
            }
            uint32_t hf[2];                      // H[f][u_i] (facility lane f = v)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int u = min(u0 + h2 + e, n - 1);   // rows past n-1 are never used
                pu[e] = p[u];
                tc::tmem_ld1(tm + quad_lane + TCS_COL_G + (uint32_t)pu[e], gv[e]);
                tc::tmem_ld1(tm + quad_lane + TCS_COL_H + (uint32_t)u, hf[e]);
            }
            tc::tmem_wait_ld();
            if (vin) {
#pragma unroll
                for (int e = 0; e < 2; ++e) xch[(h2 + e) * 128 + qv] = (int)hf[e];   // G[u_i][v] to location p^-1(v)
            }
            group_sync(3, 32 * TCS_RW);          // exchange
        }
      }
        TCT_ACC(0, pt0, xch[v]);
        int4* sl = slots + parity * TCS_RW;
        unsigned acc_mask = 0, near_mask = 0;
        const int dv = Dg[v];
        unsigned need = 0, band = 0;
        int dd[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = h2 + e;
            const int u = u0 + i;                               // (rows past n - 1: in bounds, unused)
            const int guv = xch[i * 128 + v];                   // G_uv = (A B'^T)[u][v]
            const int auv = As[u * ld + v], buv = Bs[pu[e] * ld + px];
            dd[e] = 2 * (guv + (int)gv[e] - Dg[u] - dv + 2 * auv * buv);   // δ(u, v) (R10d)
            const int o = wg.rb[e] + v;
            const bool ex = (unsigned)(v - wg.rf[e]) < (unsigned)wg.lim[e];
            if (RING) {
                // exact integer threshold (R23): accept iff δ <= thr; a flagged iteration (thr = -1)
                // accepts δ <= 0 (R5) and takes the general test below for δ > 0: both are
                // δ <= max(thr, 0)
                const int thr = TR.at_ofs(kofs0 + (int)kr + o);
                const bool pass = dd[e] <= max(thr, 0);
                acc_mask |= (unsigned)(ex && pass) << e;
                need |= (unsigned)(ex && !pass && thr < 0) << e;
            } else {
                // ensemble: θ_k -+ its margin from the producer's ring (prepare_theta), decided
                // outside the bracket, exact double test inside it (R16); δ <= 0 accepted (R5)
                const int2 th = ering[((int)kr + o) & (TCS_ERING - 1)];
                const int lo = max(th.x, 0);
                acc_mask |= (unsigned)(ex & (dd[e] <= lo)) << e;
                band |= (unsigned)(ex & (dd[e] > lo) & (dd[e] <= th.y)) << e;
            }
        }
        if (__any_sync(0xffffffffu, (need | band) != 0)) {   // general test: float θ, exact inside its margin
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if ((band >> e) & 1u) {          // ensemble, inside the margin: exact double test (R16)
                    const int x = tc_exact(dd[e], k0 + kr + (uint64_t)(wg.rb[e] + v), sch, seed, cv.chain);
                    acc_mask |= (unsigned)(x & 1) << e;
                    near_mask |= (unsigned)((x >> 1) & 1) << e;
                }
                if ((need >> e) & 1u) {
                    const uint64_t kk = k0 + kr + (uint64_t)(wg.rb[e] + v);
                    float th, m;
                    theta_of(sch, seed, cv.chain, kk, &th, &m);
                    const float df = (float)dd[e];
                    bool ac = df < th - m;
                    if (!ac && !(df > th + m)) {  // inside the margin: exact double test (R16)
                        const int x = tc_exact(dd[e], kk, sch, seed, cv.chain);
                        ac = x & 1;
                        near_mask |= (unsigned)((x >> 1) & 1) << e;
                    }
                    acc_mask |= (unsigned)ac << e;
                }
            }
        }
        {   // this thread's first accepted candidate (row h2 before row h2 + 1; selects, no indexing)
            const bool a0 = acc_mask & 1u;
            const int best_o = a0 ? wg.rb[0] + v : (acc_mask ? wg.rb[1] + v : INT_MAX);
            const int bd = a0 ? dd[0] : dd[1];
            const int brs = (u0 + h2 + (a0 ? 0 : 1)) | (v << 8) | ((a0 ? pu[0] : pu[1]) << 16) | (px << 24);
            const int wmin = __reduce_min_sync(0xffffffffu, best_o);
            // slot key = offset << 3 | warp: the CTA minimum names its slot (no ballot afterwards)
            if (best_o == wmin && (wmin != INT_MAX || lane == 0))
                sl[warp] = make_int4(wmin == INT_MAX ? INT_MAX : (wmin << 3) | warp, bd, brs, 0);
        }
        TCT_ACC(1, pt0, acc_mask);
        // probe the previous update MMA now: the stage then waits only if it is still running
        const bool mma_done = !mma_pending || tc::mbar_test(mbar, ph);
        group_sync(4, 32 * TCS_RW);              // window decision
        const int jkey = __reduce_min_sync(0xffffffffu, lane < TCS_RW ? sl[lane].x : INT_MAX);
        const int j = jkey == INT_MAX ? INT_MAX : jkey >> 3;
        TCT_MARK(pt1, j);
        TCT_ACC(10, pt0, j);
        parity ^= 1;
        if (__any_sync(0xffffffffu, near_mask != 0)) {   // R16: log near ties of consumed iterations (uniform test)
            const int consumed = (j == INT_MAX) ? Wl : j + 1;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int o = wg.rb[e] + v;
                if (((near_mask >> e) & 1u) && o < consumed)
                    near_record(sink, k0 + kr + (uint64_t)o, (acc_mask >> e) & 1u);
            }
        }
        if (j == INT_MAX) {
            TCT_ACC(4, pt0, j);
            kr += (uint32_t)Wl;
            win_advance<4>(n, u0, v0, Wl, &u0, &v0);
            W = min(2 * W, wmax);
            wg = sc_win(n, u0, v0, W, kr_end - kr, h2);
            fresh = true;
            continue;
        }
        const int4 win = sl[jkey & 7];
        const int dw = win.y;
        const int r = win.z & 0xFF, s = (win.z >> 8) & 0xFF;
        const int pr = (win.z >> 16) & 0xFF, ps = (int)((unsigned)win.z >> 24);
        const uint32_t kracc = kr + (uint32_t)j;
        TCT_ACC(5, pt1, r + ps);
        // ---------------- stage: the G|H update operands, D'', the next window's rows ----------------
        // next window: cursor after (r, s) (next_pair as selects)
        const bool same_row = s + 1 < n, next_row = r + 1 < n - 1;
        const int nu0 = same_row ? r : next_row ? r + 1 : 0;
        const int nv0 = same_row ? s + 1 : next_row ? r + 2 : 1;
        int npu[2], nu[2];                       // this warp's next rows and their facilities after the swap
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            nu[e] = min(nu0 + h2 + e, n - 1);
            const int pn = p[nu[e]];             // unconditional load, then the swap's correction
            npu[e] = nu[e] == r ? ps : nu[e] == s ? pr : pn;
        }
        TCT_ACC(6, pt1, npu[0] + npu[1]);
        // shared-memory operands first (independent of the update MMA still in flight)
        // (v >= n reads padding or the next row: in bounds, and those lanes' values are never used)
        const int arv = As[r * ld + v], asv = As[s * ld + v];
        const int bfr = Bs[pr * ld + v], bfs = Bs[ps * ld + v];
        int dAu[2], dBfu[2];                     // dA of the next rows (locations), dBf of their facilities
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            dAu[e] = (int)As[nu[e] * ld + r] - (int)As[nu[e] * ld + s];
            dBfu[e] = (int)Bs[npu[e] * ld + pr] - (int)Bs[npu[e] * ld + ps];
        }
        // D'' below (stored by the h2 = 0 warps; loaded by all: no branch)
        // (v >= n reads padding or the next row: in bounds, never used)
        const int dB = (int)Bs[pr * ld + px] - (int)Bs[ps * ld + px];
        const int ars = As[r * ld + s], brs = Bs[pr * ld + ps];
        if (mma_pending & !mma_done) tc::mbar_wait(mbar, ph);
        ph ^= (uint32_t)mma_pending;
        tc::fence_after_sync();
        TCT_ACC(7, pt1, ph);
        uint32_t gps = 0, gpr = 0, g4[2], h4[2];   // PRE-update tensor memory
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            tc::tmem_ld1(tm + quad_lane + TCS_COL_G + (uint32_t)npu[e], g4[e]);
            tc::tmem_ld1(tm + quad_lane + TCS_COL_H + (uint32_t)nu[e], h4[e]);
        }
        // G[v][p(s)], G[v][p(r)]: needed by lanes r and s only (their new diagonal); loaded by
        // every warp (no branch)
        tc::tmem_ld1(tm + quad_lane + TCS_COL_G + (uint32_t)ps, gps);
        tc::tmem_ld1(tm + quad_lane + TCS_COL_G + (uint32_t)pr, gpr);
        const int dA = vin ? arv - asv : 0, dBf = vin ? bfr - bfs : 0;
        if (h2 != 0) {                           // the update's operands (one thread per v, the h2 = 1 warps)
            const int ro = (v >> 3) * 256 + (v & 7) * 16;
            if (ENS) *reinterpret_cast<uint16_t*>(La + ro) = (uint16_t)(b8(dA) | (b8(-dBf) << 8));   // A row v
            else tc::tmem_st1(tm + quad_lane + TCS_COL_L, b8(dA) | (b8(-dBf) << 8));
            *reinterpret_cast<uint32_t*>(Rg + ro) = b8(-dBf);               // G rows: facility v
            *reinterpret_cast<uint32_t*>(Rg + 4096 + ro) = b8(dA) << 8;    // H rows: location v
        }
        const int Wn = max(64, min(wmax, round_up32(8 * (j + 1))));
        const ScWin wn = sc_win(n, nu0, nv0, Wn, kr_end - kracc - 1, h2);   // next window's geometry
        if (t == 0) {                            // the accept, for the helper warp (buffer by accept parity:
            const uint64_t kacc = k0 + kracc;    // the helper is at most one accept behind)
            int* rc = rec + 4 * (int)(accepted & 1);
            rc[0] = r; rc[1] = s;
            rc[2] = (int)(uint32_t)kacc; rc[3] = (int)(uint32_t)(kacc >> 32);
        }
        TCT_ACC(9, pt1, dAu[1] + dBfu[1] + arv + bfs);
        tc::tmem_wait_ld();
        {                                        // D'' (one thread per v: the h2 = 0 warps store)
            const int dnew = ((v == r) | (v == s)) ? (int)(v == r ? gps : gpr) + ars * brs : dv - (vin ? dA * dB : 0);
            const bool own = (h2 == 0) & vin;
            if (own) Dg[v] = dnew;
            if (own & ((v == r) | (v == s))) p[v] = (uint16_t)(v == r ? ps : pr);
        }
        TCT_ACC(8, pt1, (int)(h4[1] + g4[1]));
        px = (v == r) ? ps : (v == s) ? pr : px;     // p(v), p^-1(v) after the swap
        qv = (v == pr) ? s : (v == ps) ? r : qv;
        const bool wrap = nu0 < r;               // cursor back at row 0: rows not staged
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            pu[e] = npu[e];
            gv[e] = (uint32_t)((int)g4[e] - dA * dBfu[e]);                 // G''[v][p''(u_i)]
            if (vin) xch[(h2 + e) * 128 + qv] = (int)h4[e] - dBf * dAu[e];  // H''[v][u_i] = G''_{u_i, p''^-1(v)}
        }
        TCT_ACC(2, pt1, gv[1]);
        if (h2 != 0) {                           // the update's operands visible to the tensor cores
            if (!ENS) tc::tmem_wait_st();
            tc::fence_proxy_async();
        }
        tc::fence_before_sync();
        group_sync(1, TCS_NT);                   // operands staged, next rows exchanged: MMA issue
        TCT_ACC(3, pt1, xch[v]);
        mma_pending = true;
        fresh = wrap;
        cost += dw;
        if (cost < best) {
            best = cost;
            if (h2 == 0 && vin) best_p[v] = (uint16_t)px;
        }
        u0 = nu0;
        v0 = nv0;
        W = Wn;
        wg = wn;
        ++accepted;
        kr = kracc + 1;
        kr_last = kr;
    }
    if (mma_pending) {                           // the last update complete before tensor memory is freed
        tc::mbar_wait(mbar, ph);
        ph ^= 1;
        tc::fence_after_sync();
    }
    if (RING && t == 0) TR.drain();
    if (ENS && t == 0) ectl[1] = 1;              // release the θ producer
    if (t == 0) rec[4 * (int)(accepted & 1)] = -1;
    group_sync(1, TCS_NT);                       // release the helper
  } else if (ENS && warp == TCS_RW + 1) {
    // ---------------- ensemble θ producer: θ_k of the coming iterations, block by block ----------------
    constexpr int NB = TCS_ERING / TCS_EB;
    for (uint32_t b = 0; (uint64_t)b * TCS_EB < (uint64_t)kr_end; ++b) {
        if (b >= (uint32_t)NB) {                 // the slot's previous block released by the consumers
            const uint64_t* eb = ebar + NB + (b % NB);
            const uint32_t par = ((b / NB) - 1) & 1;
            while (!tc::mbar_try(const_cast<uint64_t*>(eb), par))   // (suspends in hardware between probes)
                if (ectl[1] != 0) goto produced;
        }
        for (int i = lane; i < TCS_EB; i += 32) {
            Prep pr;
            pr.k = k0 + (uint64_t)b * TCS_EB + (uint64_t)i;
            prepare_theta(pr, sch, seed, cv.chain);
            ering[(b * TCS_EB + i) & (TCS_ERING - 1)] = int_bracket(pr.th, pr.m);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            tc::mbar_arrive(ebar + (b % NB));
        }
        if (ectl[1] != 0) break;
    }
  produced:;
  } else {
    // ---------------- helper warp: the update MMA of each accept, digest ----------------
    for (uint64_t na = 0;; ++na) {
        group_sync(1, TCS_NT);
        const int* rc = rec + 4 * (int)(na & 1);
        const int r = rc[0];
        if (r < 0) break;
        if (lane == 0) {
            tc::fence_after_sync();
            // [G | H] (256 columns) += [dA, -dBf] [[-dBf, 0]; [0, dA]]^T
            if (ENS)
                tc::mma_i8(tm + TCS_COL_G, tc::smem_desc(tc::smem_u32(La), 128, 256),
                           tc::smem_desc(tc::smem_u32(Rg), 128, 256), id_gh, true);
            else
                tc::mma_i8_ts(tm + TCS_COL_G, tm + TCS_COL_L, tc::smem_desc(tc::smem_u32(Rg), 128, 256), id_gh, true);
            tc::mma_commit(mbar);
            const int s = rc[1];
            const uint64_t kacc = (uint64_t)(uint32_t)rc[2] | ((uint64_t)(uint32_t)rc[3] << 32);
            digest = digest_step(digest, kacc, r, s);
        }
    }
  }

    // ---------------- write the chain state back (Δ is rebuilt by the caller) ----------------
#ifdef QAPSA_PHASE_TIMERS
    if (lane == 0)
        for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[16 * warp + i], (unsigned long long)tacc[i]);
    if (t == 0) { atomicAdd(&g_phase_cycles[127], accepted); }
#endif
    __syncthreads();
    for (int i = t; i < n; i += NT) {
        cv.p[i] = p[i];
        cv.best_p[i] = best_p[i];
    }
    if (t == 0) {
        cv.st->cost = cost;
        cv.st->best_cost = best;
        cv.st->accepted += accepted;
        unsigned long long* ko = k_out + (ENS ? 2 * blockIdx.x : 0);
        ko[0] = k0 + kr;                         // iteration reached (the Δ engine starts here)
        ko[1] = accepted;                        // swaps accepted in this phase
    }
    if (t == 32 * TCS_RW) cv.st->digest = digest;    // helper lane 0 holds the digest
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tm, tcs_cols<ENS>());
}

}  // namespace qapsa
