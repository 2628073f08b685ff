// device_common.cuh -- per-iteration arithmetic of the Δ-matrix SA hot path
// on sm_100a: the counter-based uniform r_k, the cooling schedule T_k, the
// candidate enumeration and the trajectory digest.
//
// Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, R# = DESIGN.md
// "Readings of the paper".  This file shares no code with oracle/: both
// implement DESIGN.md's definitions independently and the parity tests
// compare them.
#pragma once
#include <cstdint>

namespace qapsa {

// ---- Philox4x32-10 (R3): key = (seed lo, seed hi), ctr = (k lo, k hi, chain, tag)
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return U4{c0, c1, c2, c3};
}

// r_k of Eq.(2): ((x1:x0 >> 11) + 0.5) * 2^-53, in [2^-54, 1 - 2^-54].
__device__ __forceinline__ double uniform_r(uint64_t seed, uint64_t k, uint32_t chain) {
    const U4 x = philox4x32_10((uint32_t)k, (uint32_t)(k >> 32), chain, 0u,
                               (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t bits = ((uint64_t)x.y << 32) | (uint64_t)x.x;
    return __dmul_rn(__dadd_rn((double)(bits >> 11), 0.5), 0x1p-53);
}

// ---- cooling schedule (R1); coef = lambda (geometric) or beta (Lundy-Mees),
// computed once on the host in double.
struct Sched {
    int kind;      // 0 geometric, 1 Lundy-Mees
    double t0;
    double coef;
    float t0f;     // (float)t0
    float coeff;   // (float)coef
};

__device__ __forceinline__ double temperature(const Sched& s, uint64_t k) {
    if (s.kind == 1)
        return __ddiv_rn(s.t0, __dadd_rn(1.0, __dmul_rn(__dmul_rn((double)k, s.coef), s.t0)));
    return __dmul_rn(s.t0, exp(__dmul_rn(s.coef, (double)k)));
}

// T_k in float, relative error < 2e-6: only brackets decisions (never decides alone).
// Float only (no FP64 on the fast path): coef and k each rounded to float, so the
// exponent carries a relative error ~2e-7; with __expf T32 is within ~2e-6 of T_k.
__device__ __forceinline__ float temp32(const Sched& s, uint64_t k) {
    const float x = s.coeff * __ull2float_rn(k);
    if (s.kind == 1) return __fdividef(s.t0f, 1.0f + x * s.t0f);
    return s.t0f * __expf(x);
}

// ---- Eq.(2) acceptance for one candidate in the "live band" (0 < delta <= 38 T):
// accept iff exp(-delta/T) > r;  near tie iff |delta + T ln r| < 1e-9 T (R16).
__device__ __forceinline__ bool metropolis(int32_t delta, double T, double r, bool* near) {
    const double d = (double)delta;
    const bool acc = exp(__ddiv_rn(-d, T)) > r;
    *near = fabs(__dadd_rn(d, __dmul_rn(T, log(r)))) < __dmul_rn(1e-9, T);
    return acc;
}

// Fast path: θ = -T ln r in float with a margin far wider than its error; the
// exact double test decides (and flags near ties) only inside the margin, so
// the decision equals the double-precision one everywhere.
__device__ __forceinline__ bool metropolis_fast(int32_t delta, const Sched& s, uint64_t k,
                                                uint64_t seed, uint32_t chain, bool* near) {
    const double r = uniform_r(seed, k, chain);
    const float T = temp32(s, k);
    const float th = T * -__logf((float)r);
    const float m = 2e-4f * th + 2e-5f * T;
    const float df = (float)delta;
    if (df < th - m) return true;
    if (df > th + m) return false;
    return metropolis(delta, temperature(s, k), r, near);
}

// ---- candidate enumeration: row-major upper triangle (R4, R11)
__host__ __device__ __forceinline__ int tri_base(int n, int r) { return r * n - (r * (r + 1)) / 2; }
__host__ __device__ __forceinline__ int tri_index(int n, int r, int s) {
    return tri_base(n, r) + (s - r - 1);
}
// q -> (r, s); closed form guess corrected by integer checks.
// The closed form r = floor((b - sqrt(b^2 - 8q)) / 2), b = 2n-1, with the approximate
// MUFU square root (error << 1e-3 for b^2 - 8q < 2^24), is off by at most one;
// one branch-free correction each way makes it exact.
__device__ __forceinline__ void tri_pair(int n, int q, int* r, int* s) {
    const int b = 2 * n - 1;
    float sq;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"((float)(b * b - 8 * q)));
    int rr = (int)(((float)b - sq) * 0.5f);
    rr = max(0, min(rr, n - 2));
    rr = (rr > 0 && tri_base(n, rr) > q) ? rr - 1 : rr;
    rr = (rr < n - 2 && tri_base(n, rr + 1) <= q) ? rr + 1 : rr;
    *r = rr;
    *s = q - tri_base(n, rr) + rr + 1;
}

// ---- trajectory digest (R18): wrapping sum over the accepted (k, r, s) of
// mix(mix(k) ^ (r << 32 | s)), mix = splitmix64 finaliser.  The sum does not depend
// on the order in which accepts are added, so batches of accepts hash in parallel.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t digest_step(uint64_t d, uint64_t k, int r, int s) {
    return d + mix64(mix64(k) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)s));
}
constexpr uint64_t kDigestSeed = 0x9E3779B97F4A7C15ull;

// ---- named barrier over the threads of one chain group
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace qapsa
