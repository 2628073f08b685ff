// tc_chain.cuh -- single-chain Δ-matrix SA with its O(N^2) state resident in tensor memory
// (TMEM) and every O(N^2) update of an accepted swap done by the 5th-generation tensor cores
// (tcgen05.mma kind::i8, exact s32 accumulation).
//
// Eligible instances (qapsa.cu, tc_eligible): 4 <= n <= 128 and 0 <= a_ij, b_ij <= 127, so
// that every operand is an exact signed 8-bit value.
//
// State (thread v of the 4 "lane warps" owns TMEM lane v; warp w reaches lanes 32(w%4)..+31):
//   Δ   TMEM columns [0,128):   Δ_uv (u < v) in cell (lane v, column u), the lower triangle.
//   G   TMEM columns [128,256): G[x][f] = sum_k a_xk B[f][p(k)] = (A B'^T)[x][p^-1(f)]
//       (location lanes x facility columns), the row sums of Taillard's update (R10b);
//   H   TMEM columns [256,384): H = G^T (facility lanes x location columns).
//   A, B row-major in shared memory (static), p and p^-1.
// With G and H the touching values need no dot products: for v != r,s (pre-swap)
//   X_r[v] = B'_v . a_r = H[p(v)][r],  X_s[v] = H[p(v)][s],
//   Y_r[v] = A_v . b'_r = G[v][p(r)],  Y_s[v] = G[v][p(s)],  Z_r = Y_s[r], Z_s = Y_r[s],
// each a column read of TMEM (H's values reach thread v through shared memory via p^-1).
//
// One accepted swap (r, s), r < s (P:40-46 step (d)), by the lane warps:
//   stage   thread x: dA_x = a_xr - a_xs, dB_x = B'_xr - B'_xs, and as facility f = x:
//           dBf_f = B[f][p(r)] - B[f][p(s)];  g_x = 2 dA_x dB_x = g0 + 127 (g1 + g2);
//             Δ:  L_x = [g0, g1, g2, 1, 127, 127, dA, dA, dB, dB, 0..]  (TMEM lane x)
//                 R_x = [1, 127, 127, g0, g1, g2, -dB, -dB, -dA, -dA, 0..] (smem row x)
//                 (L R^T)_uv = 2 (dA_u - dA_v)(dB_u - dB_v)           (R10)
//             G:  G += [dA] [-dBf]^T,   H += [-dBf] [dA]^T             (p(r) <-> p(s))
//           plus the touching reads of G and H above.
//   MMA     one thread issues the three updates (M = N = 128, K = 32 each).
//   epilog  thread v: δ''(r,v), δ''(s,v) (R10b), D''_v = D_v - dA_v dB_v; the cells
//           (lane v, column r|s) are column writes; the cells (lane r|s, column v < r|s) lie in
//           one TMEM lane and are patched by a read-modify-write of the 32-lane block (registers).  p, p^-1, best, digest.
// The 4 helper warps compute the thresholds θ of the next window meanwhile.
//
// Window of candidates ("the swap which would have been found first"): the
// next W iterations k+o are the pairs that follow the cursor in row-major triangle order (R4),
// i.e. rows u0..u0+3 at most (never wrapping); thread v tests (u0+i, v) reading its own cells
// Δ_{u0+i, v} (one tcgen05.ld of 4 columns).  Eq.(2) is decided exactly as in chain.cuh (θ =
// -T ln r in float with a margin, exact double test inside it, certain reject above 38.5 T);
// the smallest accepting offset over the CTA is the accepted swap.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "theta_ring.cuh"

namespace qapsa {

constexpr int TCK_NT = 256;              // 8 warps: 4 lane warps (thread v <-> TMEM lane v), 4 helpers
constexpr int TCK_NW = 8;                // warps: window slots
constexpr int TCK_WSCAN = 7168;          // window cap of the Δ engine (whole rows, cold phase): 7 θ blocks,
                                         // TH_SLOTS_TC - 8 blocks of prefetch
constexpr int TCK_TH = 256;              // thresholds prepared ahead per window (offsets < TCK_TH)
constexpr uint32_t TCK_COL_G = 128;      // G: TMEM columns [128, 256)
constexpr uint32_t TCK_COL_H = 256;      // H = G^T: TMEM columns [256, 384)
constexpr uint32_t TCK_COL_L = 384;      // L operands (A from TMEM): Δ [384,392), G|H [392,400)
constexpr uint32_t TCK_COLS = 512;       // TMEM columns allocated

__host__ __device__ constexpr bool tc_eligible(int n, int maxA, int maxB) {
    return n >= 4 && n <= 128 && maxA <= 127 && maxB <= 127;
}

// byte offset of element (x, k) of a 128-row x 128-K 8-bit operand in the K-major no-swizzle
// canonical layout: core matrix = 8 rows x 16 bytes; K-adjacent core matrices 128 B apart
// (LBO), 8-row groups 1024 B apart (SBO)
__host__ __device__ __forceinline__ int cofs(int x, int k) {
    return ((x >> 3) << 10) + ((k >> 4) << 7) + ((x & 7) << 4) + (k & 15);
}

struct TcLayout {
    int a, b, rd, rg, rh, tmp, p, pinv, bestp, rowr, rows, xbuf, zbuf, slots, thm, misc, tbar, thdr, rnd, bytes;
};
// ld: row stride of A and B (row_stride(n, true) <= 144)
__host__ __device__ inline TcLayout tc_layout(int ld) {
    TcLayout L;
    int o = 0;
    L.a = o;     o += 128 * ld;
    L.b = o;     o += 128 * ld;
    o = (o + 1023) & ~1023;
    L.rd = o;    o += 128 * 32;                 // B operands, K-major canonical (SBO 256, LBO 128)
    L.rg = o;    o += 256 * 32;                 // G|H update: rows 0..127 G (facility), 128..255 H (location)
    L.tmp = o;   o += TH_SLOTS_TC * TH_BLK * 4;  // init: A, C canonical (SBO 1024, LBO 128); then the θ ring
    static_assert(2 * 128 * 128 <= TH_SLOTS_TC * TH_BLK * 4, "the θ ring reuses the init operands");
    L.p = o;     o += 128 * 2;
    L.pinv = o;  o += 128 * 2;
    L.bestp = o; o += 128 * 2;
    L.rowr = o;  o += 128 * 4;
    L.rows = o;  o += 128 * 4 + 16;
    L.xbuf = o;  o += 128 * 8;
    L.zbuf = o;  o += 16;
    L.slots = o; o += 2 * TCK_NW * 16;
    L.thm = o;   o += TCK_TH * 8;               // (θ, margin) by window offset
    L.misc = o;  o += 64;                       // mbarriers (2 x 8 B) | TMEM base (4 B)
    L.tbar = o;  o += TH_SLOTS_TC * 8;          // threshold ring mbarriers
    L.thdr = o;  o += TH_SLOTS_TC * 16;         // threshold ring block headers
    L.rnd = o;   o += 64 + 2 * 4 * TCK_NT * 2 + TCK_NT * 8;   // random proposals: lists, pairs, gathered Δ
    L.bytes = o;
    return L;
}

__device__ __forceinline__ uint32_t b8(int v) { return (uint32_t)v & 0xFFu; }
__device__ __forceinline__ uint32_t pack8(int a, int b, int c, int d) {
    return b8(a) | (b8(b) << 8) | (b8(c) << 16) | (b8(d) << 24);
}

#ifdef QAPSA_PHASE_TIMERS
// register-accumulated phase timers (no memory traffic inside the loop); flushed at the end
#define TCT_MARK(var, dep) const long long var = clock_after((int)(dep))
#define TCT_ACC(slot, from, dep) tacc[slot] += clock_after((int)(dep)) - (from)
#else
#define TCT_MARK(var, dep)
#define TCT_ACC(slot, from, dep)
#endif

// Window geometry at cursor (u0, v0), in closed form: rows u0 .. u0+R-1 (R = min(8, n-1-u0), never
// past the last row, so a window never wraps).  Row i starts at offset f_i (f_0 = 0,
// f_1 = n - v0, f_{i+1} = f_i + m1 - i with m1 = n - 1 - u0) and column first_i (v0, then
// u0 + i + 1); candidate (u0+i, v) has offset f_i - first_i + v.
__device__ __forceinline__ int win_f(int i, int L0, int m1) {   // f_i for i >= 1
    return L0 + (i - 1) * m1 - (((i - 1) * i) >> 1);
}
template <int RMAX>
__device__ __forceinline__ int win_rows(int n, int u0) { return min(RMAX, n - 1 - u0); }
template <int RMAX>
__device__ __forceinline__ int win_total(int n, int u0, int v0) {
    return win_f(win_rows<RMAX>(n, u0), n - v0, n - 1 - u0);
}
// Δ engine: the number R >= 1 of whole rows from the cursor (the first from v0) whose candidates
// f_R fit in W (at least the first row); R <= n - 1 - u0 (the window never wraps).  The quadratic
// f_{x+1} = L0 + x m1 - x (x + 1) / 2 <= W is solved in float and corrected exactly.
__device__ __forceinline__ int win_rows_whole(int n, int u0, int L0, int m1, int W) {
    const int Rmax = n - 1 - u0;
    if (W <= L0 || Rmax <= 1) return 1;
    const float b = 2.0f * (float)m1 - 1.0f;
    const float disc = b * b - 8.0f * (float)(W - L0);
    int R = disc < 0.0f ? Rmax : min(Rmax, (int)(0.5f * (b - sqrtf(disc))) + 1);
    R = max(R, 1);
#pragma unroll 1
    while (R < Rmax && win_f(R + 1, L0, m1) <= W) ++R;
#pragma unroll 1
    while (R > 1 && win_f(R, L0, m1) > W) --R;
    return R;
}
// cursor after the first x candidates of the window (0 < x <= total)
template <int RMAX>
__device__ __forceinline__ void win_advance(int n, int u0, int v0, int x, int* nu, int* nv) {
    const int R = win_rows<RMAX>(n, u0), L0 = n - v0, m1 = n - 1 - u0;
    if (x >= win_f(R, L0, m1)) {
        const int u = u0 + R;
        if (u >= n - 1) { *nu = 0; *nv = 1; }
        else { *nu = u; *nv = u + 1; }
        return;
    }
    if (x < L0) { *nu = u0; *nv = v0 + x; return; }
    int i = 1, f = L0;                           // row i >= 1 holding offset x
#pragma unroll
    for (int e = 2; e < RMAX; ++e) {
        const int fe = win_f(e, L0, m1);
        if (e < R && x >= fe) { i = e; f = fe; }
    }
    *nu = u0 + i;
    *nv = u0 + i + 1 + (x - f);
}
// cursor after the accepted pair (r, s)
__device__ __forceinline__ void next_pair(int n, int r, int s, int* nu, int* nv) {
    if (s + 1 < n) { *nu = r; *nv = s + 1; }
    else if (r + 1 < n - 1) { *nu = r + 1; *nv = r + 2; }
    else { *nu = 0; *nv = 1; }
}

__device__ __forceinline__ int rej_of(float T32) { return __float2int_ru(fminf(38.5f * T32, 2.0e9f)); }
__device__ __forceinline__ int rej_bound(const Sched& sch, uint64_t k) { return rej_of(temp32(sch, k)); }

// θ = -T_k ln r_k in float and its margin (chain.cuh prepare_theta)
__device__ __forceinline__ void theta_of(const Sched& sch, uint64_t seed, uint32_t chain, uint64_t kk,
                                         float* th, float* m) {
    Prep pr;
    pr.k = kk;
    prepare_theta(pr, sch, seed, chain);
    *th = pr.th;
    *m = pr.m;
}
// The float bracket (θ - m, θ + m) as integers for δ: accepted outright iff δ <= max(lo, 0)
// (δ < θ - m, or δ <= 0 by R5), rejected outright iff δ > hi (δ > θ + m), the exact test in
// between.  Exact for |δ| < 2^24, where (float)δ is exact (tensor-memory instances: |δ| <=
// 4 n 127^2 < 2^24); brackets past 2^30 are clamped (every such δ is on the same side).
__device__ __forceinline__ int2 int_bracket(float th, float m) {
    return make_int2((int)ceilf(fminf(th - m, 1073741824.0f)) - 1, (int)floorf(fminf(th + m, 1073741824.0f)));
}
// exact double-precision Eq.(2) inside the float margin (rare; kept out of line):
// bit 0 = accept, bit 1 = near tie (R16)
__device__ __noinline__ int tc_exact(int d, uint64_t kk, Sched sch, uint64_t seed, uint32_t chain) {
    bool near = false;
    const bool acc = metropolis(d, temperature(sch, kk), uniform_r(seed, kk, chain), &near);
    return (acc ? 1 : 0) | (near ? 2 : 0);
}

// RND: random proposals (R22): iteration k proposes pair index floor(x M / 2^32),
// x = Philox(seed; k, chain, tag 3); a window is the next TCK_NT iterations, one candidate per
// thread, its Δ cells gathered from their TMEM lanes by the warps owning them
template <int NFIX, bool ENS = false, bool RND = false>
__global__ void __launch_bounds__(TCK_NT, 1) k_sa_tc(const ChainArgs a) {
    constexpr bool RING = !ENS;                  // single chain: precomputed θ (theta_ring.cuh)
    extern __shared__ __align__(16) unsigned char smem[];
    const ChainView cv = chain_view<ENS>(a);     // this CTA's chain (ensemble launches)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = NFIX ? NFIX : a.n;
    const int ld = NFIX ? row_stride(NFIX, true) : a.ld;
    const int M = n * (n - 1) / 2;
    const TcLayout L = tc_layout(ld);
    uint8_t* As = smem + L.a;
    uint8_t* Bs = smem + L.b;
    uint8_t* Rd = smem + L.rd;
    uint8_t* Rg = smem + L.rg;
    uint16_t* p = reinterpret_cast<uint16_t*>(smem + L.p);
    uint16_t* best_p = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int* rowR = reinterpret_cast<int*>(smem + L.rowr);
    int* rowS = reinterpret_cast<int*>(smem + L.rows);
    int2* xbuf = reinterpret_cast<int2*>(smem + L.xbuf);
    int* zbuf = reinterpret_cast<int*>(smem + L.zbuf);
    int4* slots = reinterpret_cast<int4*>(smem + L.slots);
    float2* thm = reinterpret_cast<float2*>(smem + L.thm);
    uint64_t* mbar_d = reinterpret_cast<uint64_t*>(smem + L.misc);        // Δ update done
    uint64_t* mbar_g = reinterpret_cast<uint64_t*>(smem + L.misc + 8);    // init only
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.misc + 16);
    const bool lanew = warp < 4;                 // lane warp (else helper)
    const uint32_t quad_lane = (uint32_t)(32 * (warp & 3)) << 16;   // this warp's TMEM lane quadrant
    const int v = t & 127;                       // TMEM lane v = location v = facility v

    // ---------------- load the chain state ----------------
    copy_words(As, a.A, n * ld, t, TCK_NT);
    copy_words(Bs, a.B, n * ld, t, TCK_NT);
    for (int i = t; i < n; i += TCK_NT) {
        p[i] = (uint16_t)cv.p[i];
        best_p[i] = (uint16_t)cv.best_p[i];
    }
    for (int i = t; i < 3 * 128 * 32 / 16; i += TCK_NT)    // Rd, Rg := 0
        reinterpret_cast<uint4*>(Rd)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tc::tmem_alloc(tmem_slot, TCK_COLS);
    if (t == 0) { tc::mbar_init(mbar_d, 1); tc::mbar_init(mbar_g, 1); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tmem_slot;
    {   // A and C[f][k] = B[f][p(k)] in canonical operand layout (init only)
        uint8_t* Ac = smem + L.tmp;
        uint8_t* Cc = Ac + 128 * 128;
        for (int idx = t; idx < 128 * 128; idx += TCK_NT) {
            const int x = idx >> 7, kk = idx & 127;
            const bool in = x < n && kk < n;
            Ac[cofs(x, kk)] = in ? As[x * ld + kk] : (uint8_t)0;
            Cc[cofs(x, kk)] = in ? Bs[x * ld + p[kk]] : (uint8_t)0;
        }
        tc::fence_proxy_async();
        __syncthreads();
        if (t == 0) {                            // G = A C^T, H = C A^T on the tensor cores
            const uint32_t id = tc::idesc_i8(128, 128, true);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + TCK_COL_G, tc::smem_desc(tc::smem_u32(Ac) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(Cc) + 256 * kc, 128, 1024), id, kc > 0);
            for (int kc = 0; kc < 4; ++kc)
                tc::mma_i8(tm + TCK_COL_H, tc::smem_desc(tc::smem_u32(Cc) + 256 * kc, 128, 1024),
                           tc::smem_desc(tc::smem_u32(Ac) + 256 * kc, 128, 1024), id, kc > 0);
            tc::mma_commit(mbar_g);
        }
    }
    if (lanew) {                                 // Δ -> TMEM (lane v, column u < v); L := 0
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t vals[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
                const int u = 32 * c + jj;
                vals[jj] = (u < v && v < n) ? (uint32_t)cv.D[a.rowaddr[u] + v] : 0u;
            }
            tc::tmem_st32(tm + quad_lane + 32 * c, vals);
        }
#pragma unroll
        for (int c = 0; c < 24; c += 4) tc::tmem_st4(tm + quad_lane + TCK_COL_L + c, 0u, 0u, 0u, 0u);
        tc::tmem_wait_st();
    }
    __syncthreads();
    const bool vin = v < n;
    int px = vin ? p[v] : 0;                     // p(v)
    int qv = 0;                                  // p^-1(v) (facility v's location)
    for (int i = 0; i < n; ++i) qv = (p[i] == v) ? i : qv;
    int Dgv = 0;                                 // D_v = sum_k a_vk B'_vk (lane v's diagonal)
    if (vin)
        for (int kk = 0; kk < n; ++kk) Dgv += (int)As[v * ld + kk] * (int)Bs[px * ld + p[kk]];
    tc::mbar_wait(mbar_g, 0);                    // G, H initialised
    uint32_t ph_d = 0;
    tc::fence_after_sync();
    uint64_t k = cv.k0_dev ? *cv.k0_dev : a.k0, accepted = 0;
    // single chain: θ of the window from the precomputed ring (reuses the init operands' space)
    ThetaRing<TH_SLOTS_TC> TR = theta_ring<TH_SLOTS_TC>(
        reinterpret_cast<int*>(smem + L.tmp), reinterpret_cast<int4*>(smem + L.thdr),
        reinterpret_cast<uint64_t*>(smem + L.tbar), a.theta, a.theta_hdr, a.theta_kb, a.theta_cnt, k);
    if (RING && t == 0 && k < a.k_end) TR.start(k);
    if (RND && t < 8) reinterpret_cast<int*>(smem + L.rnd)[t] = 0;   // random windows: list lengths
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();

    const Sched sch = a.sch;
    const uint64_t seed = a.seed, k_end = a.k_end;
    const NearSink sink = cv.sink;
    int64_t cost = cv.st->cost, best = cv.st->best_cost;
    uint64_t digest = cv.st->digest;
    int u0, v0;
    tri_pair(n, (int)(k % (uint64_t)M), &u0, &v0);
    // window cap: the ring (TH_SLOTS_TC blocks) keeps its prefetch ahead of a whole window
    const int wcap = RING ? min(a.wscan, TCK_WSCAN) : a.wscan;
    int W = RND ? 32 : wcap;
    int parity = 0;
    int ring_blo = -1, ring_hi = 0;              // ring: last block refilled from, offsets known resident
    // certain-reject bound: δ > 38.5 T32(k) >= 38.4 T_kk gives exp(-δ/T) < 2^-54 <= r (chain.cuh);
    // rounded up to an integer, so the exact test below also sees every δ <= 38.5 T32(k)
    int rejI = rej_bound(sch, k);
    uint64_t pk = ~0ull;                         // window whose thresholds are in thm
    int pn = 0;                                  // ... for offsets [0, pn)
    int pend_r = -1, pend_s = -1;                // rows r, s whose TMEM cells (lane r|s, column < r|s)
                                                 // the helpers are still patching (window reads rowR/rowS)
    const uint32_t id_rank = tc::idesc_i8(128, 128, true);
    const uint32_t id_gh = tc::idesc_i8(128, 256, true);
#ifdef QAPSA_PHASE_TIMERS
    long long tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

    while (k < k_end) {
        // ---------------- window: whole rows u0 .. u0+R-1 from the cursor (all warps) ----------------
        TCT_MARK(pt0, u0 + v0);
        const int L0 = n - v0, m1 = n - 1 - u0;
        const int R = win_rows_whole(n, u0, L0, m1, W);
        int Wl = RND ? min(W, TCK_NT) : win_f(R, L0, m1);   // random: W candidates (adaptive, <= one per thread)
        {
            const uint64_t remaining = k_end - k;
            if ((uint64_t)Wl > remaining) Wl = (int)remaining;
        }
        if (RING) {                              // thresholds of the window resident (theta_ring.cuh)
            const int ko = (int)(k - TR.kb);
            if ((ko >> 10) != ring_blo) {        // a block passed (warp-uniform test; one thread refills)
                ring_blo = ko >> 10;
                if (t == 0) TR.refill(k);
            }
            if (ko + Wl > ring_hi) {
                TR.ensure_ofs(ko + Wl);
                ring_hi = (int)(TR.ready * TH_BLK);
            }
        }
        int4* sl = slots + parity * TCK_NW;
        int best_o = INT_MAX, best_d = 0, best_rs = 0;
        int nt_o[2] = {INT_MAX, INT_MAX}, nt_d[2] = {0, 0};   // this thread's near ties (R16): offset, decision
        // groups of 8 rows u0 + 8g .. u0 + 8g + 7, g = warp / 4, + 2, ...: thread v reads its cells
        // Δ_{u, v} (columns u) with one tcgen05.ld; offsets grow with the row, so a warp stops after
        // its first group holding an accept (every later candidate comes after it)
        if (RND) {
            // ---------------- random window: candidate c = t at iteration k + c ----------------
            int* gcnt = reinterpret_cast<int*>(smem + L.rnd);                 // [2][4] list lengths
            uint16_t* glist = reinterpret_cast<uint16_t*>(smem + L.rnd + 64);  // [2][4][TCK_NT]
            uint16_t* cuv = glist + 2 * 4 * TCK_NT;                            // [TCK_NT] u | v << 8 ... as 2 x u16
            int* dval = reinterpret_cast<int*>(cuv + 2 * TCK_NT);               // [TCK_NT] gathered Δ_uv
            if (t < 4) gcnt[(parity ^ 1) * 4 + t] = 0;   // the next window's lists (this parity's were reset before)
            int cu = 0, cvv = 1;
            const bool cex = t < Wl;
            if (cex) {
                const int idx = proposal_index(true, 0, 0, M, k + (uint64_t)t, seed, cv.chain);
                tri_pair(n, idx, &cu, &cvv);
                cuv[2 * t] = (uint16_t)cu;
                cuv[2 * t + 1] = (uint16_t)cvv;
                const int qd = cvv >> 5;         // the lane quadrant holding cell (lane v, column u)
                const int pos = atomicAdd(&gcnt[parity * 4 + qd], 1);
                glist[(parity * 4 + qd) * TCK_NT + pos] = (uint16_t)t;
            }
            tc::fence_before_sync();
            __syncthreads();
            tc::fence_after_sync();
            {   // gather: warps q and q + 4 read their quadrant's cells, 8 columns per tcgen05.ld batch
                const int qd = warp & 3;
                const int cnt = gcnt[parity * 4 + qd];
                const uint16_t* gl = glist + (parity * 4 + qd) * TCK_NT;
                for (int e0 = 8 * (warp >> 2); e0 < cnt; e0 += 16) {
                    uint32_t vals[8];
                    int cs[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        cs[i] = e0 + i < cnt ? (int)gl[e0 + i] : -1;
                        const int col = cs[i] >= 0 ? (int)cuv[2 * cs[i]] : 0;
                        tc::tmem_ld1(tm + quad_lane + (uint32_t)col, vals[i]);
                    }
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (cs[i] < 0) continue;
                        const int u_ = cuv[2 * cs[i]], v_ = cuv[2 * cs[i] + 1];
                        if (lane == (v_ & 31)) {
                            int d = (int)vals[i];
                            if (v_ == pend_r) d = rowR[u_];      // cells still being patched
                            else if (v_ == pend_s) d = rowS[u_];
                            dval[cs[i]] = d;
                        }
                    }
                }
            }
            __syncthreads();
            if (cex) {
                const int d = dval[t];
                bool acc;
                const int thr = TR.at_ofs((int)(k - TR.kb) + t);
                if (thr >= 0 || d <= 0) {
                    acc = d <= thr || d <= 0;    // R23; δ <= 0 accepted (R5)
                } else {                         // flagged iteration: general test (R16)
                    float th, m;
                    theta_of(sch, seed, cv.chain, k + (uint64_t)t, &th, &m);
                    const float df = (float)d;
                    acc = df < th - m;
                    if (!acc && !(df > th + m)) {
                        const int x = tc_exact(d, k + (uint64_t)t, sch, seed, cv.chain);
                        acc = x & 1;
                        if (x & 2) { nt_o[0] = t; nt_d[0] = acc; }
                    }
                }
                if (acc) {
                    best_o = t;
                    best_d = d;
                    best_rs = cu | (cvv << 8) | ((int)p[cu] << 16) | ((int)p[cvv] << 24);
                }
            }
        } else {
            const int NG = (R + 7) >> 3;
            // exact integer thresholds (R23) unless a block of the window is flagged or the window is
            // cut short by the end of the call: the general path below
            const int2 sp = RING ? TR.span(k, k + (uint64_t)Wl) : make_int2(1, 0);
            if (!sp.x && Wl == win_f(R, L0, m1)) {
                // thread v's candidates: rows [ulo, uhi] (row u0 from column v0 on, u < v)
                const int ulo = v >= v0 ? u0 : u0 + 1;
                const int uhi = vin ? min(v - 1, u0 + R - 1) : -1;
                const int kofs = (int)(k - TR.kb);
                for (int g = warp >> 2; g < NG; g += 2) {
                    const int i0 = 8 * g;
                    int f = i0 == 0 ? 0 : win_f(i0, L0, m1);   // offset of row u0 + i0's first candidate
                    uint32_t dd[8];
                    tc::tmem_ld8(tm + quad_lane + (uint32_t)(u0 + i0), dd);
                    const int lo = ulo - u0 - i0, hi = uhi - u0 - i0;   // this thread's rows i in [lo, hi]
                    tc::tmem_wait_ld();
                    if (v == pend_r || v == pend_s) {    // cells still being patched: their new values
                        const int* row = v == pend_r ? rowR : rowS;
    #pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if (u0 + i0 + i < v) dd[i] = (uint32_t)row[u0 + i0 + i];
                    }
                    int mn = INT_MAX;                // smallest δ of the thread's candidates
                    // (lo <= 1, and lo > 0 only in the first group: the lower bound binds at i = 0 alone)
    #pragma unroll
                    for (int i = 0; i < 8; ++i) mn = min(mn, ((i > 0 || lo <= 0) && i <= hi) ? (int)dd[i] : INT_MAX);
                    unsigned am = 0;
                    int oo[8];
                    if (__any_sync(0xffffffffu, mn <= sp.y)) {   // else every candidate is above every threshold
    #pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int ii = i0 + i;
                            const int first = ii == 0 ? v0 : u0 + ii + 1;
                            oo[i] = f - first + v;
                            f += ii == 0 ? L0 : m1 - ii;
                            const int thr = TR.ring[(kofs + oo[i]) & (TR.RING - 1)];
                            am |= (unsigned)((i > 0 || lo <= 0) && i <= hi && (int)dd[i] <= thr) << i;
                        }
                    }
                    if (__any_sync(0xffffffffu, am != 0)) {
                        if (am) {                    // this thread's first accepted candidate
                            const int i = __ffs(am) - 1;
                            const int u = u0 + i0 + i;
                            best_o = oo[i];
                            best_d = (int)dd[i];
                            best_rs = u | (v << 8) | ((int)p[u] << 16) | (px << 24);
                        }
                        break;
                    }
                }
            } else {
            // the thread's candidate rows as in the fast path (a superset where the window is cut
            // short): a group whose candidates all lie above rejI holds no accept (prefilter)
            const int ulo = v >= v0 ? u0 : u0 + 1;
            const int uhi = vin ? min(v - 1, u0 + R - 1) : -1;
            for (int g = warp >> 2; g < NG; g += 2) {
                const int i0 = 8 * g;
                int f = i0 == 0 ? 0 : win_f(i0, L0, m1);   // offset of row u0 + i0's first candidate
                if (f >= Wl) break;                  // warp-uniform: the group starts past the window
                uint32_t dd[8];
                tc::tmem_ld8(tm + quad_lane + (uint32_t)(u0 + i0), dd);   // columns u0+i0 .. (< 140: inside G, unused)
                const int lo = ulo - u0 - i0, hi = uhi - u0 - i0;
                tc::tmem_wait_ld();
                if (v == pend_r || v == pend_s) {    // cells still being patched: their new values
                    const int* row = v == pend_r ? rowR : rowS;
    #pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (u0 + i0 + i < v) dd[i] = (uint32_t)row[u0 + i0 + i];
                }
                {
                    int mn = INT_MAX;
    #pragma unroll
                    for (int i = 0; i < 8; ++i) mn = min(mn, ((i > 0 || lo <= 0) && i <= hi) ? (int)dd[i] : INT_MAX);
                    if (!__any_sync(0xffffffffu, mn <= rejI)) continue;   // every candidate a certain reject
                }
                // per candidate: exists / accepted outright (δ <= 0, R5) / needs the threshold test
                unsigned need = 0, am = 0;
                int oo[8];
    #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int ii = i0 + i;
                    const int first = ii == 0 ? v0 : u0 + ii + 1;
                    oo[i] = f - first + v;
                    f += ii == 0 ? L0 : m1 - ii;
                    const int d = (int)dd[i];
                    const bool ex = ii < R && v >= first && vin && oo[i] < Wl;
                    am |= (unsigned)(ex && d <= 0) << i;
                    need |= (unsigned)(ex && d > 0 && d <= rejI) << i;   // above rejI: certain reject
                }
                if (__any_sync(0xffffffffu, need != 0)) {
                    const int pnk = pk == k ? pn : 0;
    #pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if ((need >> i) & 1u) {
                            const int o = oo[i];
                            const int d = (int)dd[i];
                            float th, m;
                            if (!RING && o < pnk) { const float2 q = thm[o]; th = q.x; m = q.y; }
                            else theta_of(sch, seed, cv.chain, k + (uint64_t)o, &th, &m);
                            const float df = (float)d;
                            bool ac = df < th - m;
                            if (!ac && !(df > th + m)) {  // inside the margin: exact double test (R16)
                                const int x = tc_exact(d, k + (uint64_t)o, sch, seed, cv.chain);
                                ac = x & 1;
                                if (x & 2) {          // near tie: logged after the decision if consumed
                                    const int e = nt_o[0] == INT_MAX ? 0 : 1;
                                    if (nt_o[e] == INT_MAX) { nt_o[e] = o; nt_d[e] = ac; }
                                    else near_record(sink, k + (uint64_t)o, ac);   // a third (never seen): logged eagerly
                                }
                            }
                            am |= (unsigned)ac << i;
                        }
                    }
                }
                if (__any_sync(0xffffffffu, am != 0)) {
                    if (am) {                        // this thread's first accepted candidate
                        const int i = __ffs(am) - 1;
                        const int u = u0 + i0 + i;
                        best_o = oo[i];
                        best_d = (int)dd[i];
                        best_rs = u | (v << 8) | ((int)p[u] << 16) | (px << 24);
                    }
                    break;
                }
            }
            }
        }
        {
            const int wmin = __reduce_min_sync(0xffffffffu, best_o);
            // slot key = offset << 3 | warp: the CTA minimum names its slot (no ballot afterwards)
            if (best_o == wmin && (wmin != INT_MAX || lane == 0))
                sl[warp] = make_int4(wmin == INT_MAX ? INT_MAX : (wmin << 3) | warp, best_d, best_rs, 0);
        }
        TCT_ACC(10, pt0, best_o);
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        pend_r = pend_s = -1;                    // the helpers' patch is complete
        const int jkey = __reduce_min_sync(0xffffffffu, lane < TCK_NW ? sl[lane].x : INT_MAX);
        const int j = jkey == INT_MAX ? INT_MAX : jkey >> 3;
        TCT_MARK(pt1, j);
        parity ^= 1;
        if (__any_sync(0xffffffffu, nt_o[0] != INT_MAX)) {   // R16: log near ties of consumed iterations
            const int consumed = (j == INT_MAX) ? Wl : j + 1;
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (nt_o[e] < consumed) near_record(sink, k + (uint64_t)nt_o[e], nt_d[e] != 0);
        }
        if (j == INT_MAX) {                      // no accepted swap in the window
            TCT_ACC(1, pt0, j);
            k += (uint64_t)Wl;
            if (!RND) {
                u0 += R;                         // whole rows: the cursor moves to the next row
                v0 = u0 + 1;
                if (u0 >= n - 1) { u0 = 0; v0 = 1; }
            }
            W = min(2 * W, wcap);
            rejI = rej_bound(sch, k);
            continue;
        }
        const int4 win = sl[jkey & 7];
        const int dw = win.y;
        const int r = win.z & 0xFF, s = (win.z >> 8) & 0xFF;    // r < s
        const int pr = (win.z >> 16) & 0xFF, ps = (int)((unsigned)win.z >> 24);
        const uint64_t kacc = k + (uint64_t)j;
        TCT_ACC(0, pt0, j);

        if (lanew) {
            // ---------------- stage (thread = location x = v and facility f = v) ----------------
            int arv = 0, asv = 0, brv = 0, bsv = 0, bfr = 0, bfs = 0;
            if (vin) {
                arv = As[r * ld + v]; asv = As[s * ld + v];
                brv = Bs[pr * ld + px]; bsv = Bs[ps * ld + px];
                bfr = Bs[pr * ld + v]; bfs = Bs[ps * ld + v];
            }
            const int ars = As[r * ld + s], brs = Bs[pr * ld + ps];
            uint32_t yr, ys, hr, hs;             // touching reads (pre-update)
            tc::tmem_ld1(tm + quad_lane + TCK_COL_G + (uint32_t)pr, yr);   // Y_r[v] = G[v][p(r)]
            tc::tmem_ld1(tm + quad_lane + TCK_COL_G + (uint32_t)ps, ys);   // Y_s[v] = G[v][p(s)]
            tc::tmem_ld1(tm + quad_lane + TCK_COL_H + (uint32_t)r, hr);    // X_r[p^-1(v)] = H[v][r]
            tc::tmem_ld1(tm + quad_lane + TCK_COL_H + (uint32_t)s, hs);    // X_s[p^-1(v)] = H[v][s]
            TCT_ACC(7, pt1, arv + bfs);
            const int dA = arv - asv, dB = brv - bsv;  // dA_v = a_vr - a_vs, dB_v = B'_vr - B'_vs (pre-swap)
            const int dBf = bfr - bfs;           // facility v: B[v][p(r)] - B[v][p(s)]
            {
                const int g = 2 * dA * dB;       // = g0 + 127 (g1 + g2): g0 in [0,127], g1, g2 in [-128,127]
                const int gq = (g * 66053) >> 23;    // floor(g / 127), or one less if 127 | g (|g| <= 32258)
                const int g0 = g - 127 * gq;
                const int g1 = gq >> 1;
                const int g2 = gq - g1;
                tc::tmem_st4(tm + quad_lane + TCK_COL_L, pack8(g0, g1, g2, 1), pack8(127, 127, dA, dA),
                             pack8(dB, dB, 0, 0), 0u);
                tc::tmem_st1(tm + quad_lane + TCK_COL_L + 8, b8(dA) | (b8(-dBf) << 8));
                const int ro = (v >> 3) * 256 + (v & 7) * 16;
                *reinterpret_cast<uint4*>(Rd + ro) =
                    make_uint4(pack8(1, 127, 127, g0), pack8(g1, g2, -dB, -dB), pack8(-dA, -dA, 0, 0), 0u);
                *reinterpret_cast<uint32_t*>(Rg + ro) = b8(-dBf);                 // G rows: facility v
                *reinterpret_cast<uint32_t*>(Rg + 4096 + ro) = b8(dA) << 8;      // H rows: location v
                TCT_ACC(8, pt1, g2);
            }
            tc::tmem_wait_ld();
            TCT_ACC(9, pt1, hs + yr);
            if (vin) xbuf[qv] = make_int2((int)hr, (int)hs);   // X_r, X_s of location p^-1(v)
            if (v == r) zbuf[0] = (int)ys;       // Z_r = a_r . b'_s
            if (v == s) zbuf[1] = (int)yr;       // Z_s = a_s . b'_r
            tc::fence_proxy_async();
            tc::tmem_wait_st();
            tc::fence_before_sync();
            TCT_ACC(11, pt1, ps);
            group_sync(1, 160);                  // operands staged; helper warp 7 issues the MMAs
            TCT_ACC(2, pt1, zbuf[0]);
            // ---------------- epilogue: touching values (R10b), column writes ----------------
            const int Dr = zbuf[0] + ars * brs;  // D''_r
            const int Ds = zbuf[1] + ars * brs;  // D''_s
            const int2 X = vin ? xbuf[v] : make_int2(0, 0);
            const int dv = Dgv - dA * dB;        // D''_v = D_v - dA_v dB_v
            int dr = 2 * (X.x + (int)ys + ars * dB - dA * brs - Dr - dv + 2 * arv * bsv);   // δ''(r,v)
            int ds = 2 * (X.y + (int)yr - ars * dB + dA * brs - Ds - dv + 2 * asv * brv);   // δ''(s,v)
            if (v == s) dr = -dw;                // Δ_rs after the swap: swapping back restores C
            if (v == r) ds = -dw;
            Dgv = (v == r) ? Dr : (v == s) ? Ds : dv;
            rowR[v] = dr;
            rowS[v] = ds;
            TCT_ACC(3, pt1, dr + ds);
            tc::mbar_wait(mbar_d, ph_d);         // Δ += L R^T complete
            tc::fence_after_sync();
            TCT_ACC(4, pt1, ph_d);
            tc::tmem_st1(tm + quad_lane + (uint32_t)r, (uint32_t)dr);
            tc::tmem_st1(tm + quad_lane + (uint32_t)s, (uint32_t)ds);
            // p after the swap (shared copy), best_p
            if (v == r) p[v] = (uint16_t)ps;
            if (v == s) p[v] = (uint16_t)pr;
            tc::tmem_wait_st();
            tc::fence_before_sync();
        } else {
            // ---------------- helpers: MMA issue (warp 7); thresholds of the next window; digest ----------------
            if (warp == 7) {
                group_sync(1, 160);
                if (t == 224) {
                    tc::fence_after_sync();
                    tc::mma_i8_ts(tm, tm + TCK_COL_L, tc::smem_desc(tc::smem_u32(Rd), 128, 256), id_rank, true);
                    // [G | H] (256 columns) += [dA, -dBf] [[-dBf, 0]; [0, dA]]^T
                    tc::mma_i8_ts(tm + TCK_COL_G, tm + TCK_COL_L + 8, tc::smem_desc(tc::smem_u32(Rg), 128, 256), id_gh, true);
                    tc::mma_commit(mbar_d);
                }
                __syncwarp();
            }
            int nu0, nv0;
            next_pair(n, r, s, &nu0, &nv0);
            const int Wln = (int)min((uint64_t)TCK_TH, k_end - kacc - 1);
            for (int o = v; !RING && o < Wln; o += 128) {
                float th, m;
                theta_of(sch, seed, cv.chain, kacc + 1 + (uint64_t)o, &th, &m);
                thm[o] = make_float2(th, m);
            }
            if (t == 128) digest = digest_step(digest, kacc, r, s);
            TCT_ACC(2, pt1, Wln);
        }
        group_sync(2, TCK_NT);                   // rowR / rowS, thresholds, p complete
        TCT_ACC(5, pt1, rowR[0]);
        px = (v == r) ? ps : (v == s) ? pr : px;     // p(v) and p^-1(v) after the swap
        qv = (v == pr) ? s : (v == ps) ? r : qv;
        cost += dw;
        const bool improved = cost < best;
        if (improved) best = cost;
        if (lanew) {
            if (improved && vin) best_p[v] = (uint16_t)px;
        } else {
            // ---------------- rows r, s: read-modify-write of the owning quadrant's lanes ----------------
            tc::fence_after_sync();
            const bool hr2 = (r >> 5) == (warp & 3), hs2 = (s >> 5) == (warp & 3);
            const int lim = hs2 ? s : (hr2 ? r : 0);   // columns [0, lim) hold row cells
            if (lim > 0) {                       // warp-uniform; chunks 32c .. 32c+31 for 32c < lim
                // Lane r (s) takes the whole chunk rows from rowR (rowS): its cells with column >= r
                // (>= s) are upper-triangle cells, never read, so overwriting them is harmless;
                // every other lane writes back what it read.
                uint32_t vv[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (32 * c < lim) tc::tmem_ld32(tm + quad_lane + 32 * c, vv[c]);
                tc::tmem_wait_ld();
                const int* src = (hr2 && lane == (r & 31)) ? rowR : (hs2 && lane == (s & 31)) ? rowS : nullptr;
                if (src) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (32 * c < lim) {
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const uint4 w4 = reinterpret_cast<const uint4*>(src + 32 * c)[i];
                                vv[c][4 * i] = w4.x; vv[c][4 * i + 1] = w4.y;
                                vv[c][4 * i + 2] = w4.z; vv[c][4 * i + 3] = w4.w;
                            }
                        }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (32 * c < lim) tc::tmem_st32(tm + quad_lane + 32 * c, vv[c]);
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            TCT_ACC(6, pt1, rowS[0]);
        }
        ph_d ^= 1;
        pend_r = r;
        pend_s = s;
        pk = kacc + 1;
        {
            int nu0, nv0;
            next_pair(n, r, s, &nu0, &nv0);
            pn = (int)min((uint64_t)TCK_TH, k_end - kacc - 1);   // thresholds the helpers prepared
            u0 = nu0;
            v0 = nv0;
            W = RND ? max(32, min(TCK_NT, round_up32(4 * (j + 1)))) : max(64, min(wcap, round_up32(8 * (j + 1))));
        }
        ++accepted;
        k = kacc + 1;
        rejI = rej_bound(sch, k);
    }
    if (RING && t == 0) TR.drain();

    // ---------------- write the chain state back ----------------
#ifdef QAPSA_PHASE_TIMERS
    if (lane == 0)
        for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[16 * warp + i], (unsigned long long)tacc[i]);
    if (t == 0) { atomicAdd(&g_phase_cycles[127], accepted); }
#endif
    __syncthreads();
    for (int i = t; i < n; i += TCK_NT) {
        cv.p[i] = p[i];
        cv.best_p[i] = best_p[i];
    }
    if (lanew) {
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t vals[32];
            tc::tmem_ld32(tm + quad_lane + 32 * c, vals);
            tc::tmem_wait_ld();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
                const int u = 32 * c + jj;
                if (u < v && v < n) cv.D[a.rowaddr[u] + v] = (int32_t)vals[jj];
            }
        }
    }
    if (t == 128) {                              // helper 0 holds the digest
        cv.st->cost = cost;
        cv.st->best_cost = best;
        cv.st->digest = digest;
        cv.st->accepted += accepted;
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tm, TCK_COLS);
}

}  // namespace qapsa
