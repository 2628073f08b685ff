/*
 * qap_oracle.h -- plain, slow, obviously-correct CPU oracle for the
 * Δ-matrix simulated-annealing hot path of G. Paul, arXiv 1208.2675.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1208_2675_b200/, include/qapsa.h) never links,
 * imports or calls it, and shares no code, header, table or constant
 * generator with it.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * DESIGN.md R# = the numbered reading in DESIGN.md "Readings of the paper".
 *
 * Pins (see tests/test_oracle_*.py): SPEC worked examples, Random123 Philox
 * KATs, brute force over all permutations, numpy matmul identity for Δ-init,
 * Eq.(1) cost differences for δ, Δ == scratch after every accept, EQ1 ==
 * SCRATCH == DELTA trajectories, schedule end points.  Parity unpinned:
 * nothing beyond what DESIGN.md "Parity pins" lists as unpinned (the
 * exact bit stream of the uniform map is pinned only through the Philox KATs).
 */
#ifndef QAP_ORACLE_H
#define QAP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MODE_EQ1 = 0, ORC_MODE_SCRATCH = 1, ORC_MODE_DELTA = 2 };
enum { ORC_COOL_GEOMETRIC = 0, ORC_COOL_LUNDY_MEES = 1 };

/* Philox4x32-10 (Salmon et al. 2011), R3. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* r of Eq.(2): U(Philox(key=seed; ctr=(k lo, k hi, chain, tag))), R3. */
double orc_uniform(uint64_t seed, uint64_t k, uint32_t chain, uint32_t tag);
/* T_k of the cooling schedule, R1. */
double orc_temperature(int kind, double t0, double tf, uint64_t total_iters, uint64_t k);

/* Eq.(1): C = sum_i sum_j A_ij B_{p(i),p(j)}. */
int64_t orc_cost(int n, const int32_t* A, const int32_t* B, const int32_t* p);
/* B'_ij = B_{p(i),p(j)} (Eq.(3) read as the invariant, R9). */
void orc_bprime(int n, const int32_t* B, const int32_t* p, int32_t* Bp);
/* δ by definition: Eq.(1) after swapping p(r),p(s) minus Eq.(1) before. */
int64_t orc_delta_eq1(int n, const int32_t* A, const int32_t* B, const int32_t* p, int r, int s);
/* δ by the O(N) scratch formula on symmetric zero-diagonal instances. */
int64_t orc_delta_scratch(int n, const int32_t* A, const int32_t* Bp, int r, int s);
/* Step (a): Δ for every pair r<s, row-major upper triangle. */
void orc_delta_init(int n, const int32_t* A, const int32_t* Bp, int64_t* D);
/* Row-major upper-triangle enumeration: q -> (r,s) and back. */
void orc_pair(int n, int64_t q, int32_t* r, int32_t* s);
int64_t orc_index(int n, int r, int s);
/* Step (d): swap p(r),p(s); exchange B' rows r,s and columns r,s. */
void orc_apply_swap(int n, int32_t* p, int32_t* Bp, int r, int s);
/* Step (d) Δ update (R10): disjoint pairs by the rank
 * form with PRE-swap B' (Bp_pre), touching pairs recomputed by the scratch
 * formula on POST-swap B' (Bp_post). */
void orc_update_delta(int n, const int32_t* A, const int32_t* Bp_pre, const int32_t* Bp_post,
                      int r, int s, int64_t* D);
/* SPEC S:190 bench rule over all pairs (R2). */
void orc_temperature_bounds(int n, const int64_t* D, double* t0, double* tf);
/* min over all n! permutations of Eq.(1) (Heap's algorithm), n <= 10. */
int64_t orc_bruteforce(int n, const int32_t* A, const int32_t* B, int32_t* best_p);

typedef struct {
    int32_t n;
    int32_t mode;          /* ORC_MODE_* */
    const int32_t* A;      /* n*n */
    const int32_t* B;      /* n*n */
    int32_t* p;            /* n    current permutation */
    int32_t* best_p;       /* n */
    int32_t* Bp;           /* n*n  B' = B[p][p] */
    int64_t* D;            /* n(n-1)/2 (DELTA mode; may be NULL otherwise) */
    int64_t cost, best_cost;
    uint64_t digest, accepted, near_ties, iterations;
    int32_t proposal;      /* 0: sequential enumeration (R4); 1: random pairs (R22) */
    int32_t pad;
} orc_state;

/* Set p = p0, B' = B[p0][p0], C = Eq.(1), best = C, digest = seed value,
 * counters 0, and (DELTA mode) Δ by step (a). */
void orc_state_reset(orc_state* st, const int32_t* p0);

/* Sequential SA, iterations k in [k0, k0+iters) of a schedule of
 * total_iters iterations (R1-R8, R16).
 * follow_k/follow_d: near-tie decisions to adopt (R16), may be NULL.
 * near_k/near_d: out log of near ties (k, decision taken), capacity near_cap.
 * check_every > 0: after every check_every-th accept verify B' == B[p][p],
 * C == Eq.(1) and (DELTA) Δ == scratch for all pairs; returns -1 on mismatch.
 * Returns number of near ties logged (<= near_cap) or -1. */
int orc_sa_run(orc_state* st, uint64_t k0, uint64_t iters, int kind, double t0, double tf,
               uint64_t total_iters, uint64_t seed, uint32_t chain,
               const uint64_t* follow_k, const uint8_t* follow_d, int n_follow,
               uint64_t* near_k, uint8_t* near_d, int near_cap, int64_t check_every);

/* Start permutation of chain `chain` (R14b): Fisher-Yates from the
 * identity, j = floor(x (i+1) / 2^32), x = Philox(key = seed; ctr = (i, 0, chain, tag 1)).x. */
void orc_start_perm(int n, uint64_t seed, uint32_t chain, int32_t* p);

/* Independent chains chain_base..chain_base+count-1 (BASELINE config 5)
 * on `threads` host threads, δ source `mode`, each chain its own full schedule of
 * iters iterations; p0s (count*n) or NULL = orc_start_perm(seed, chain).
 * out: count*6 int64 = (cost, best_cost, accepted, near_ties, digest bits,
 * iterations) per chain; near_k/near_d (nullable, count*near_cap): per-chain
 * near-tie log (k, decision). */
int orc_ensemble_run(int n, const int32_t* A, const int32_t* B, const int32_t* p0s, int64_t count,
                     uint32_t chain_base, uint64_t iters, int kind, double t0, double tf,
                     uint64_t seed, int threads, int mode, int64_t* out, uint64_t* near_k,
                     uint8_t* near_d, int near_cap);

#ifdef __cplusplus
}
#endif
#endif
