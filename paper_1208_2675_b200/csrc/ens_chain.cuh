// ens_chain.cuh -- the scratch phase (R10d) of an ENSEMBLE of chains
// (BASELINE config 5; "run copies of the heuristic independently"), four chains per SM.
//
// Ensembles are throughput, not latency: the tensor-memory scratch phase of a single chain
// (scratch_chain.cuh) keeps G = A·B'^T and H = G^T in tensor memory (256 columns) so that each
// window costs no exchange of rows; that caps an SM at two chains (512 TMEM columns) and, at
// 320 threads per chain, its register file at two as well.  This kernel keeps only G (128 TMEM
// columns: G[x][f] = sum_k a_xk B[f][p(k)], location lanes x facility columns, R10c) and 160
// threads, so FOUR chains share an SM:
//   * the window's rows of G (G[u_i][f] for its <= 4 rows u_i) are read from the lanes u_i by the
//     warp owning them (tcgen05.ld of whole rows) into shared memory, after the update MMA;
//   * thread v (lane v) then has G_uv = G[u_i][p(v)] from shared memory and G_vu = G[v][p(u_i)]
//     from its own lane, so δ(u_i, v) = 2 (G_uv + G_vu - D_u - D_v + 2 a_uv B'_uv) costs O(1);
//   * an accept (r, s) is one SS-form int8 MMA, G += [dA] [-dBf]^T (M = N = 128, K = 32), with
//     dA_x = a_xr - a_xs, dBf_f = B[f][p(r)] - B[f][p(s)] (the exact change of G when p(r) and
//     p(s) exchange), plus D''_v = D_v - dA_v dB_v, D''_r = G[r][p(s)] + a_rs B'_rs,
//     D''_s = G[s][p(r)] + a_rs B'_rs (R10b);
//   * θ_k -+ its margin for the chain's coming iterations come from a producer warp (each θ once),
//     the window decides outside the bracket and takes the exact double test inside it (R16).
// Every quantity is an exact integer, so the trajectory is the single chain's (and the
// oracle's); the chain ends the phase after `switch_gap` iterations without an accept, and the
// caller rebuilds Δ and continues with the Δ engine (tc_chain.cuh), as for scratch_chain.cuh.
//
// Citation keys: P:n = PAPER.md line n, R# = DESIGN.md readings.
#pragma once
#include <climits>
#include <cstdint>

#include "scratch_chain.cuh"
#include "tc_chain.cuh"

namespace qapsa {

constexpr int E4_NT = 160;              // 4 row warps (thread v = TMEM lane v) + 1 θ producer warp
constexpr int E4_EB = 128;              // θ producer block (iterations)
constexpr int E4_ERING = 1024;          // θ ring (8 blocks; a window is <= 4 rows < 512 candidates)
constexpr uint32_t E4_COLS = 128;       // TMEM columns per chain: four chains per SM

struct E4Layout {
    int a, b, la, rg, p, bestp, dg, grow, slots, ering, ebar, ectl, misc, bytes;
};
__host__ __device__ inline E4Layout e4_layout(int n, int ld) {
    E4Layout L;
    int o = 0;
    L.a = o;     o += align16(n * ld);               // A, row-major (8-bit)
    L.b = o;     o += align16(n * ld);               // B, row-major (8-bit)
    o = (o + 1023) & ~1023;
    L.la = o;    o += 128 * 32;                      // update A operand [dA], K-major canonical (SBO 256)
    L.rg = o;    o += 128 * 32;                      // update B operand [-dBf]
    L.p = o;     o += 128 * 2;
    L.bestp = o; o += 128 * 2;
    L.dg = o;    o += 128 * 4;                       // D_x = G[x][p(x)]
    L.grow = o;  o += 4 * 128 * 4;                   // the window's rows of G: G[u_i][f]
    L.slots = o; o += 2 * 4 * 16;
    L.ering = o; o += E4_ERING * 8;                  // integer (θ - m, θ + m) ring of the producer warp (int_bracket)
    L.ebar = o;  o += 2 * (E4_ERING / E4_EB) * 8;    // full[NB], empty[NB]
    L.ectl = o;  o += 16;                            // stop flag
    L.misc = o;  o += 16;                            // mbarrier | TMEM base
    L.bytes = o;
    return L;
}
__host__ __device__ constexpr bool e4_eligible(int n) { return n >= 4 && n <= 128; }

// byte (x, k) of a [rows x 32] K-major canonical operand (core matrices 8 x 16 B, LBO 128, SBO 256)
__device__ __forceinline__ int e4_off(int x, int k) { return ((x >> 3) << 8) + ((k >> 4) << 7) + ((x & 7) << 4) + (k & 15); }

template <int NFIX>
__global__ void __launch_bounds__(E4_NT, 4) k_ens_scratch(const ChainArgs a, unsigned long long* k_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ChainView cv = chain_view<true>(a);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = NFIX ? NFIX : a.n;
    const int ld = NFIX ? row_stride(NFIX, true) : a.ld;
    const int M = n * (n - 1) / 2;
    const E4Layout L = e4_layout(n, ld);
    uint8_t* As = smem + L.a;
    uint8_t* Bs = smem + L.b;
    uint8_t* La = smem + L.la;
    uint8_t* Rg = smem + L.rg;
    uint16_t* p = reinterpret_cast<uint16_t*>(smem + L.p);
    uint16_t* best_p = reinterpret_cast<uint16_t*>(smem + L.bestp);
    int* Dg = reinterpret_cast<int*>(smem + L.dg);
    int* grow = reinterpret_cast<int*>(smem + L.grow);
    int4* slots = reinterpret_cast<int4*>(smem + L.slots);
    int2* ering = reinterpret_cast<int2*>(smem + L.ering);
    uint64_t* ebar = reinterpret_cast<uint64_t*>(smem + L.ebar);
    volatile int* ectl = reinterpret_cast<volatile int*>(smem + L.ectl);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.misc);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.misc + 8);
    constexpr int NB = E4_ERING / E4_EB;
    const bool roww = warp < 4;
    const uint32_t quad_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int v = t & 127;
    const bool vin = v < n;

    // ---------------- load the chain state; G = A C^T on the tensor cores ----------------
    copy_words(As, a.A, n * ld, t, E4_NT);
    copy_words(Bs, a.B, n * ld, t, E4_NT);
    for (int i = t; i < n; i += E4_NT) {
        p[i] = (uint16_t)cv.p[i];
        best_p[i] = (uint16_t)cv.best_p[i];
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, E4_COLS);
    if (t == 0) {
        tc::mbar_init(mbar, 1);
        for (int b = 0; b < 2 * NB; ++b) tc::mbar_init(ebar + b, 1);
        ectl[1] = 0;
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tmem_slot;
    uint32_t ph = 0;
    const uint32_t id_g = tc::idesc_i8(128, 128, true);
    for (int c = 0; c < 4; ++c) {                // K = 128 in four chunks of 32 (La, Rg as staging)
        if (32 * c >= n) break;
        for (int idx = t; idx < 128 * 32; idx += E4_NT) {
            const int x = idx >> 5, kk = idx & 31, k = 32 * c + kk;
            const bool in = x < n && k < n;
            La[e4_off(x, kk)] = in ? As[x * ld + k] : (uint8_t)0;
            Rg[e4_off(x, kk)] = in ? Bs[x * ld + p[k]] : (uint8_t)0;   // C[f][k] = B[f][p(k)]
        }
        tc::fence_proxy_async();
        tc::fence_before_sync();
        __syncthreads();
        if (t == 0) {
            tc::fence_after_sync();
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(La), 128, 256), tc::smem_desc(tc::smem_u32(Rg), 128, 256),
                       id_g, c > 0);
            tc::mma_commit(mbar);
        }
        tc::mbar_wait(mbar, ph);
        ph ^= 1;
        tc::fence_after_sync();
        __syncthreads();                         // La / Rg free for the next chunk
    }
    // operands of the update MMA: only K element 0 is ever non-zero
    for (int i = t; i < 2 * 128 * 32 / 16; i += E4_NT) reinterpret_cast<uint4*>(La)[i] = make_uint4(0, 0, 0, 0);
    int px = vin ? p[v] : 0;                     // p(v)
    if (roww) {
        int dgv = 0;
        if (vin)
            for (int kk = 0; kk < n; ++kk) dgv += (int)As[v * ld + kk] * (int)Bs[px * ld + p[kk]];
        Dg[v] = dgv;
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();

    const Sched sch = a.sch;
    const uint64_t seed = a.seed, k0 = a.k0;
    const uint32_t kr_end = (uint32_t)min((unsigned long long)(a.k_end - k0), 0x7FFFFFFFull);

  if (roww) {
    const NearSink sink = cv.sink;
    int64_t cost = cv.st->cost, best = cv.st->best_cost;
    uint64_t digest = cv.st->digest, accepted = 0;
    uint32_t kr = 0, kr_last = 0;
    int u0, v0;
    tri_pair(n, (int)(k0 % (uint64_t)M), &u0, &v0);
    const int wmax = a.wmax;
    int W = wmax;
    int parity = 0;
    const uint32_t gap = a.switch_gap ? (uint32_t)min(a.switch_gap, 0x7FFFFFFFull) : (uint32_t)TCS_SWITCH_GAP;
    int ering_ready = 0, ering_freed = 0, ring_hi = 0;
    const int q = warp;                          // this warp's lane quadrant: locations 32q .. 32q + 31
    while (kr < kr_end && kr - kr_last < gap) {
        // ---------------- window: rows u0 .. u0+R-1 (R <= 4) ----------------
        const int R = win_rows<4>(n, u0), L0 = n - v0, m1 = n - 1 - u0;
        int Wl = win_f(R, L0, m1);
        if (W < Wl) Wl = W;
        if ((uint32_t)Wl > kr_end - kr) Wl = (int)(kr_end - kr);
        // the ring's rare cases behind one uniform branch (every thread counts the freed blocks)
        if ((ering_freed < (int)(kr / E4_EB)) | ((int)kr + Wl > ring_hi)) {
            for (; ering_freed < (int)(kr / E4_EB); ++ering_freed)   // blocks wholly below kr are consumed
                if (t == 0) tc::mbar_arrive(ebar + NB + (ering_freed % NB));
            if ((int)kr + Wl > ring_hi) {
                while (ering_ready * E4_EB < (int)kr + Wl) {
                    tc::mbar_wait(ebar + (ering_ready % NB), (uint32_t)((ering_ready / NB) & 1));
                    ++ering_ready;
                }
                ring_hi = ering_ready * E4_EB;
            }
        }
        // the window's rows of G to shared memory: the warp owning lane u_i reads whole lanes
        int pu[4];
        uint32_t gv[4];                          // G[v][p(u_i)] (this lane)
#pragma unroll
        for (int i = 0; i < 4; ++i) pu[i] = p[min(u0 + i, n - 1)];
        {
            const int rlo = u0, rhi = u0 + R - 1;    // rows [rlo, rhi]
            if (rhi >= 32 * q && rlo < 32 * q + 32) {   // warp-uniform
                const int li = lane + 32 * q - u0;   // this lane's window row, if in [0, R)
#pragma unroll 1
                for (int c = 0; 32 * c < n; ++c) {
                    uint32_t vals[32];
                    tc::tmem_ld32(tm + quad_lane + 32 * c, vals);
                    tc::tmem_wait_ld();
                    if (li >= 0 && li < R) {
                        int4* dst = reinterpret_cast<int4*>(grow + li * 128 + 32 * c);
#pragma unroll
                        for (int w4 = 0; w4 < 8; ++w4)
                            dst[w4] = make_int4((int)vals[4 * w4], (int)vals[4 * w4 + 1], (int)vals[4 * w4 + 2],
                                                (int)vals[4 * w4 + 3]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) tc::tmem_ld1(tm + quad_lane + (uint32_t)pu[i], gv[i]);
            tc::tmem_wait_ld();
        }
        group_sync(3, 128);                      // the window's rows of G exchanged
        int rb[4], rf[4], lim[4];                // row i: locations [rf, n) at offsets rb + v, lim of them in the window
        {
            int f = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rf[i] = i >= R ? n : i == 0 ? v0 : u0 + i + 1;
                rb[i] = f - rf[i];
                lim[i] = i >= R ? 0 : max(0, min(Wl - f, n - rf[i]));
                f += i == 0 ? L0 : m1 - i;
            }
        }
        int4* sl = slots + parity * 4;
        unsigned acc_mask = 0, near_mask = 0, band = 0;
        const int dv = Dg[v];
        int dd[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int u = min(u0 + i, n - 1);
            const int guv = grow[i * 128 + px];                 // G_uv = G[u][p(v)]
            const int auv = As[u * ld + v], buv = Bs[pu[i] * ld + px];
            dd[i] = 2 * (guv + (int)gv[i] - Dg[u] - dv + 2 * auv * buv);   // δ(u, v) (R10d)
            const int o = rb[i] + v;
            const bool ex = (unsigned)(v - rf[i]) < (unsigned)lim[i];
            // θ_k -+ its margin from the producer as integers (int_bracket); δ <= 0 accepted (R5)
            const int2 th = ering[((int)kr + o) & (E4_ERING - 1)];
            const int lo = max(th.x, 0);
            acc_mask |= (unsigned)(ex & (dd[i] <= lo)) << i;
            band |= (unsigned)(ex & (dd[i] > lo) & (dd[i] <= th.y)) << i;
        }
        if (__any_sync(0xffffffffu, band != 0)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if ((band >> i) & 1u) {          // inside the margin: exact double test (R16)
                    const int x = tc_exact(dd[i], k0 + kr + (uint64_t)(rb[i] + v), sch, seed, cv.chain);
                    acc_mask |= (unsigned)(x & 1) << i;
                    near_mask |= (unsigned)((x >> 1) & 1) << i;
                }
            }
        }
        {   // this thread's first accepted candidate (rows in order)
            int best_o = INT_MAX, best_d = 0, best_rs = 0;
#pragma unroll
            for (int i = 3; i >= 0; --i) {
                const bool ac = (acc_mask >> i) & 1u;
                best_o = ac ? rb[i] + v : best_o;
                best_d = ac ? dd[i] : best_d;
                best_rs = ac ? ((u0 + i) | (v << 8) | (pu[i] << 16) | (px << 24)) : best_rs;
            }
            const int wmin = __reduce_min_sync(0xffffffffu, best_o);
            // slot key = offset << 2 | warp: the CTA minimum names its slot (no ballot afterwards)
            if (best_o == wmin && (wmin != INT_MAX || lane == 0))
                sl[warp] = make_int4(wmin == INT_MAX ? INT_MAX : (wmin << 2) | warp, best_d, best_rs, 0);
        }
        group_sync(4, 128);                      // window decision
        const int jkey = __reduce_min_sync(0xffffffffu, lane < 4 ? sl[lane].x : INT_MAX);
        const int j = jkey == INT_MAX ? INT_MAX : jkey >> 2;
        parity ^= 1;
        if (__any_sync(0xffffffffu, near_mask != 0)) {   // R16: log near ties of consumed iterations (uniform test)
            const int consumed = (j == INT_MAX) ? Wl : j + 1;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int o = rb[i] + v;
                if (((near_mask >> i) & 1u) && o < consumed) near_record(sink, k0 + kr + (uint64_t)o, (acc_mask >> i) & 1u);
            }
        }
        if (j == INT_MAX) {
            kr += (uint32_t)Wl;
            win_advance<4>(n, u0, v0, Wl, &u0, &v0);
            W = min(2 * W, wmax);
            continue;
        }
        const int4 win = sl[jkey & 3];
        const int dw = win.y;
        const int r = win.z & 0xFF, s = (win.z >> 8) & 0xFF;
        const int pr = (win.z >> 16) & 0xFF, ps = (int)((unsigned)win.z >> 24);
        // ---------------- stage: the update's operands, D'' (thread v = location v = facility v) ----------------
        const int arv = As[r * ld + v], asv = As[s * ld + v];
        const int bfr = Bs[pr * ld + v], bfs = Bs[ps * ld + v];
        const int dA = vin ? arv - asv : 0, dBf = vin ? bfr - bfs : 0;
        const int dB = vin ? (int)Bs[pr * ld + px] - (int)Bs[ps * ld + px] : 0;
        const int ro = e4_off(v, 0);
        La[ro] = (uint8_t)b8(dA);                // A operand row x = v: [dA_x, 0, ...]
        Rg[ro] = (uint8_t)b8(-dBf);              // B operand row f = v: [-dBf_f, 0, ...]
        // the new diagonal of r and s (R10b) needs G[r][p(s)] and G[s][p(r)] (pre-update): row r
        // is a window row (its copy in grow); row s is one only if s < u0 + R, else lane s reads
        // column p(r) of its own TMEM lane (a warp-uniform load by the warp holding lane s)
        int dnew = dv - dA * dB;
        const int ars = As[r * ld + s], brs = Bs[pr * ld + ps];
        const bool s_row = s - u0 < R;
        if (v == r) dnew = grow[(r - u0) * 128 + ps] + ars * brs;
        if (v == s && s_row) dnew = grow[(s - u0) * 128 + pr] + ars * brs;
        if (!s_row && (s >> 5) == q) {
            uint32_t gs;
            tc::tmem_ld1(tm + quad_lane + (uint32_t)pr, gs);
            tc::tmem_wait_ld();
            if (v == s) dnew = (int)gs + ars * brs;
        }
        if (vin) Dg[v] = dnew;
        if (v == r) p[v] = (uint16_t)ps;
        if (v == s) p[v] = (uint16_t)pr;
        px = (v == r) ? ps : (v == s) ? pr : px;
        cost += dw;
        if (cost < best) {
            best = cost;
            if (vin) best_p[v] = (uint16_t)px;
        }
        tc::fence_proxy_async();                 // operands visible to the tensor cores
        tc::fence_before_sync();
        group_sync(1, 128);                      // operands staged
        if (t == 0) {
            tc::fence_after_sync();
            tc::mma_i8(tm, tc::smem_desc(tc::smem_u32(La), 128, 256), tc::smem_desc(tc::smem_u32(Rg), 128, 256),
                       id_g, true);              // G += [dA] [-dBf]^T
            tc::mma_commit(mbar);
            digest = digest_step(digest, k0 + kr + (uint64_t)j, r, s);
        }
        int nu0, nv0;
        next_pair(n, r, s, &nu0, &nv0);
        W = max(64, min(wmax, round_up32(8 * (j + 1))));
        ++accepted;
        kr += (uint32_t)j + 1;
        kr_last = kr;
        u0 = nu0;
        v0 = nv0;
        tc::mbar_wait(mbar, ph);                 // G updated before the next window reads it
        ph ^= 1;
        tc::fence_after_sync();
    }
    if (t == 0) ectl[1] = 1;                     // release the θ producer
    // ---------------- write the chain state back (Δ is rebuilt by the caller) ----------------
    group_sync(1, 128);
    for (int i = t; i < n; i += 128) {
        cv.p[i] = p[i];
        cv.best_p[i] = best_p[i];
    }
    if (t == 0) {
        cv.st->cost = cost;
        cv.st->best_cost = best;
        cv.st->accepted += accepted;
        cv.st->digest = digest;
        unsigned long long* ko = k_out + 2 * blockIdx.x;
        ko[0] = k0 + kr;                         // iteration reached (the Δ engine starts here)
        ko[1] = accepted;
    }
  } else {
    // ---------------- θ producer: θ_k -+ its margin of the coming iterations, block by block ----------------
    for (uint32_t b = 0; (uint64_t)b * E4_EB < (uint64_t)kr_end; ++b) {
        if (b >= (uint32_t)NB) {                 // the slot's previous block released by the consumers
            const uint32_t par = ((b / NB) - 1) & 1;
            while (!tc::mbar_try(ebar + NB + (b % NB), par))
                if (ectl[1] != 0) goto produced;
        }
        for (int i = lane; i < E4_EB; i += 32) {
            Prep pr;
            pr.k = k0 + (uint64_t)b * E4_EB + (uint64_t)i;
            prepare_theta(pr, sch, seed, cv.chain);
            ering[(b * E4_EB + i) & (E4_ERING - 1)] = int_bracket(pr.th, pr.m);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            tc::mbar_arrive(ebar + (b % NB));
        }
        if (ectl[1] != 0) break;
    }
  produced:;
  }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tm, E4_COLS);
}

}  // namespace qapsa
