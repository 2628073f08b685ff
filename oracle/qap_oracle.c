/*
 * qap_oracle.c -- CPU oracle for the Δ-matrix SA hot path (arXiv 1208.2675).
 *
 * TEST INFRASTRUCTURE ONLY (see qap_oracle.h).  Plain loops in the paper's
 * order and notation; int64 for every integer quantity, IEEE double for
 * Eq.(2).  Built with -ffp-contract=off so no FMA changes a rounding.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n,
 * R# = DESIGN.md "Readings of the paper" item #.
 */
#include "qap_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (R3).  Constants of Salmon, Moraes, Dror, Shaw (SC'11). */
/* ------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k[0] += PHILOX_W0; k[1] += PHILOX_W1; }
        philox_round(c, k);
    }
    memcpy(out, c, sizeof c);
}

/* r of Eq.(2): "a uniformly distributed random variable between 0 and 1".
 * R3: 53 bits of (x1:x0), centred: ((bits >> 11) + 0.5) * 2^-53, in (0,1). */
double orc_uniform(uint64_t seed, uint64_t k, uint32_t chain, uint32_t tag) {
    uint32_t ctr[4] = {(uint32_t)k, (uint32_t)(k >> 32), chain, tag};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    uint64_t bits = ((uint64_t)x[1] << 32) | (uint64_t)x[0];
    return ((double)(bits >> 11) + 0.5) * 0x1p-53;
}

/* "T ... is slowly decreased according to a specified cooling schedule after
 * each iteration".  R1: closed forms in k. */
double orc_temperature(int kind, double t0, double tf, uint64_t total_iters, uint64_t k) {
    if (kind == ORC_COOL_LUNDY_MEES) {
        double beta = total_iters > 1 ? (t0 - tf) / (((double)(total_iters - 1) * t0) * tf) : 0.0;
        return t0 / (1.0 + ((double)k * beta) * t0);
    }
    double lambda = total_iters > 1 ? log(tf / t0) / (double)(total_iters - 1) : 0.0;
    return t0 * exp(lambda * (double)k);
}

/* ------------------------------------------------------------------ */
/* qap-core                                                            */
/* ------------------------------------------------------------------ */

/* Eq.(1): C = sum_{i,j} A_ij B_{p(i),p(j)}. */
int64_t orc_cost(int n, const int32_t* A, const int32_t* B, const int32_t* p) {
    int64_t c = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            c += (int64_t)A[i * n + j] * (int64_t)B[p[i] * n + p[j]];
    return c;
}

/* "we maintain a matrix B', the elements of which reflect swaps which
 * have been performed"; invariant B'_ij = B_{p(i),p(j)} (R9). */
void orc_bprime(int n, const int32_t* B, const int32_t* p, int32_t* Bp) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            Bp[i * n + j] = B[p[i] * n + p[j]];
}

/* δ by definition ("the change in cost, δ, for the potential swap"). */
int64_t orc_delta_eq1(int n, const int32_t* A, const int32_t* B, const int32_t* p, int r, int s) {
    int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(q, p, sizeof(int32_t) * (size_t)n);
    int32_t t = q[r]; q[r] = q[s]; q[s] = t;
    int64_t d = orc_cost(n, A, B, q) - orc_cost(n, A, B, p);
    free(q);
    return d;
}

/* δ = 2 sum_{k != r,s} (a_rk - a_sk)(B'_sk - B'_rk), symmetric zero-diagonal. */
int64_t orc_delta_scratch(int n, const int32_t* A, const int32_t* Bp, int r, int s) {
    int64_t acc = 0;
    for (int k = 0; k < n; ++k) {
        if (k == r || k == s) continue;
        acc += ((int64_t)A[r * n + k] - A[s * n + k]) * ((int64_t)Bp[s * n + k] - Bp[r * n + k]);
    }
    return 2 * acc;
}

/* row-major upper triangle (0,1),(0,2),...,(0,n-1),(1,2),... */
int64_t orc_index(int n, int r, int s) {
    return (int64_t)r * n - (int64_t)r * (r + 1) / 2 + (s - r - 1);
}

void orc_pair(int n, int64_t q, int32_t* r, int32_t* s) {
    int row = 0;
    while (q >= (int64_t)(n - 1 - row)) {
        q -= n - 1 - row;
        ++row;
    }
    *r = row;
    *s = row + 1 + (int32_t)q;
}

/* Step (a): "a matrix Δ_ij containing the cost of swapping i and j for
 * all i and j, given a current assignment p". */
void orc_delta_init(int n, const int32_t* A, const int32_t* Bp, int64_t* D) {
    for (int r = 0; r < n; ++r)
        for (int s = r + 1; s < n; ++s)
            D[orc_index(n, r, s)] = orc_delta_scratch(n, A, Bp, r, s);
}

/* Step (d), "update p to reflect the swap" and Eq.(3)/"equivalent to
 * swapping rows r and s and swapping columns r and s". */
void orc_apply_swap(int n, int32_t* p, int32_t* Bp, int r, int s) {
    int32_t t = p[r]; p[r] = p[s]; p[s] = t;
    for (int k = 0; k < n; ++k) {                 /* rows r <-> s */
        t = Bp[r * n + k]; Bp[r * n + k] = Bp[s * n + k]; Bp[s * n + k] = t;
    }
    for (int k = 0; k < n; ++k) {                 /* columns r <-> s */
        t = Bp[k * n + r]; Bp[k * n + r] = Bp[k * n + s]; Bp[k * n + s] = t;
    }
}

/* Δ update after an accepted swap (r,s) (P:44 Taillard-style, P:98 staging).
 * dA_x = a_xr - a_xs and dB_x = B'_xr - B'_xs are the staged PRE-swap rows.
 * Disjoint {u,v} ∩ {r,s} = ∅:  Δ'_uv = Δ_uv + 2 (dA_u - dA_v)(dB_u - dB_v)   (R10)
 * Touching pairs: recomputed from scratch on the POST-swap B'.       */
static void update_delta_staged(int n, const int32_t* A, const int64_t* dA, const int64_t* dB,
                                const int32_t* Bp_post, int r, int s, int64_t* D) {
    for (int u = 0; u < n; ++u) {
        for (int v = u + 1; v < n; ++v) {
            int64_t q = orc_index(n, u, v);
            if (u == r || u == s || v == r || v == s)
                D[q] = orc_delta_scratch(n, A, Bp_post, u, v);
            else
                D[q] += 2 * (dA[u] - dA[v]) * (dB[u] - dB[v]);
        }
    }
}

void orc_update_delta(int n, const int32_t* A, const int32_t* Bp_pre, const int32_t* Bp_post,
                      int r, int s, int64_t* D) {
    int64_t* dA = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* dB = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int x = 0; x < n; ++x) {
        dA[x] = (int64_t)A[x * n + r] - A[x * n + s];
        dB[x] = (int64_t)Bp_pre[x * n + r] - Bp_pre[x * n + s];
    }
    update_delta_staged(n, A, dA, dB, Bp_post, r, s, D);
    free(dA);
    free(dB);
}

/* R2 (S:190 without the random sample): over all pairs of Δ at p0,
 * dmin = smallest nonzero |δ|, dmax = largest |δ|; t0 = dmin + (dmax-dmin)/10,
 * tf = dmin; all zero -> (1.0, 0.1). */
void orc_temperature_bounds(int n, const int64_t* D, double* t0, double* tf) {
    int64_t M = (int64_t)n * (n - 1) / 2, dmin = 0, dmax = 0;
    for (int64_t q = 0; q < M; ++q) {
        int64_t a = D[q] < 0 ? -D[q] : D[q];
        if (a > dmax) dmax = a;
        if (a != 0 && (dmin == 0 || a < dmin)) dmin = a;
    }
    if (dmax == 0) { *t0 = 1.0; *tf = 0.1; return; }
    *t0 = (double)dmin + ((double)dmax - (double)dmin) / 10.0;
    *tf = (double)dmin;
}

/* Exhaustive minimum of Eq.(1) over all permutations (Heap's algorithm). */
int64_t orc_bruteforce(int n, const int32_t* A, const int32_t* B, int32_t* best_p) {
    int32_t p[16] = {0}, c[16] = {0};
    if (n < 1 || n > 12) return -1;
    for (int i = 0; i < n; ++i) { p[i] = i; c[i] = 0; }
    int64_t best = orc_cost(n, A, B, p);
    memcpy(best_p, p, sizeof(int32_t) * (size_t)n);
    int i = 1;
    while (i < n) {
        if (c[i] < i) {
            int j = (i % 2 == 0) ? 0 : c[i];
            int32_t t = p[j]; p[j] = p[i]; p[i] = t;
            int64_t v = orc_cost(n, A, B, p);
            if (v < best) { best = v; memcpy(best_p, p, sizeof(int32_t) * (size_t)n); }
            c[i] += 1;
            i = 1;
        } else {
            c[i] = 0;
            ++i;
        }
    }
    return best;
}

/* ------------------------------------------------------------------ */
/* annealer                                                            */
/* ------------------------------------------------------------------ */
#define DIGEST_SEED 0x9E3779B97F4A7C15ull

/* splitmix64 finaliser (R-digest in DESIGN.md). */
static uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void orc_state_reset(orc_state* st, const int32_t* p0) {
    int n = st->n;
    memcpy(st->p, p0, sizeof(int32_t) * (size_t)n);
    memcpy(st->best_p, p0, sizeof(int32_t) * (size_t)n);
    orc_bprime(n, st->B, st->p, st->Bp);
    st->cost = orc_cost(n, st->A, st->B, st->p);
    st->best_cost = st->cost;
    st->digest = DIGEST_SEED;
    st->accepted = st->near_ties = st->iterations = 0;
    if (st->mode == ORC_MODE_DELTA && st->D) orc_delta_init(n, st->A, st->Bp, st->D);
}

static int check_state(const orc_state* st) {
    int n = st->n;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (st->Bp[i * n + j] != st->B[st->p[i] * n + st->p[j]]) return -1;
    if (st->cost != orc_cost(n, st->A, st->B, st->p)) return -1;
    if (st->mode == ORC_MODE_DELTA)
        for (int r = 0; r < n; ++r)
            for (int s = r + 1; s < n; ++s)
                if (st->D[orc_index(n, r, s)] != orc_delta_scratch(n, st->A, st->Bp, r, s)) return -1;
    return 0;
}

/* R22, random proposals ("the swaps may be chosen randomly"): iteration k proposes pair
 * index q = floor(x * M / 2^32), x the first word of Philox4x32-10(key = seed, ctr = (k lo,
 * k hi, chain, tag 3)), i.e. (r, s) = pair(q). */
static void random_pair(int n, int64_t M, uint64_t seed, uint64_t k, uint32_t chain, int32_t* r,
                        int32_t* s) {
    const uint32_t ctr[4] = {(uint32_t)k, (uint32_t)(k >> 32), chain, 3u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    orc_pair(n, (int64_t)(((uint64_t)x[0] * (uint64_t)M) >> 32), r, s);
}

/* Steps (b)-(e) of P:46-50 for iterations k0 .. k0+iters-1.
 * (b) "Increment the iteration number. Retrieve the cost Δ_rs of the next
 *     possible swap (r,s)" -- sequential cyclic enumeration (R4).
 * (c) Eq.(2): accept iff δ < 0 or exp(-δ/T) > r  (R5: δ = 0 accepts).
 * (d) on accept: update p, B', Δ; C += δ; best; digest.
 * (e) stop after the iteration budget.                                        */
int orc_sa_run(orc_state* st, uint64_t k0, uint64_t iters, int kind, double t0, double tf,
               uint64_t total_iters, uint64_t seed, uint32_t chain,
               const uint64_t* follow_k, const uint8_t* follow_d, int n_follow,
               uint64_t* near_k, uint8_t* near_d, int near_cap, int64_t check_every) {
    const int n = st->n;
    const int32_t* A = st->A;
    const int64_t M = (int64_t)n * (n - 1) / 2;
    int32_t r, s;
    orc_pair(n, (int64_t)(k0 % (uint64_t)M), &r, &s);
    int64_t* dA = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* dB = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int n_logged = 0, status = 0;

    for (uint64_t it = 0; it < iters; ++it) {
        const uint64_t k = k0 + it;
        if (st->proposal) random_pair(n, M, seed, k, chain, &r, &s);
        int64_t delta;
        if (st->mode == ORC_MODE_EQ1)
            delta = orc_delta_eq1(n, A, st->B, st->p, r, s);
        else if (st->mode == ORC_MODE_SCRATCH)
            delta = orc_delta_scratch(n, A, st->Bp, r, s);
        else
            delta = st->D[orc_index(n, r, s)];

        const double T = orc_temperature(kind, t0, tf, total_iters, k);
        const double u = orc_uniform(seed, k, chain, 0);
        const double d = (double)delta;
        int accept = (delta < 0) || (exp(-d / T) > u);
        /* R16: near tie |δ + T ln r| < 1e-9 T (only δ > 0 can be one). */
        if (delta > 0 && fabs(d + T * log(u)) < 1e-9 * T) {
            for (int f = 0; f < n_follow; ++f)
                if (follow_k[f] == k) { accept = follow_d[f] ? 1 : 0; break; }
            if (n_logged < near_cap) {
                if (near_k) near_k[n_logged] = k;
                if (near_d) near_d[n_logged] = (uint8_t)accept;
            }
            ++n_logged;
            st->near_ties += 1;
        }

        if (accept) {
            if (st->mode == ORC_MODE_DELTA) {
                /* stage A_r., A_s., B'_r., B'_s. before the update. */
                for (int x = 0; x < n; ++x) {
                    dA[x] = (int64_t)A[x * n + r] - A[x * n + s];
                    dB[x] = (int64_t)st->Bp[x * n + r] - st->Bp[x * n + s];
                }
            }
            orc_apply_swap(n, st->p, st->Bp, r, s);
            if (st->mode == ORC_MODE_DELTA) update_delta_staged(n, A, dA, dB, st->Bp, r, s, st->D);
            st->cost += delta;
            st->accepted += 1;
            if (st->cost < st->best_cost) {
                st->best_cost = st->cost;
                memcpy(st->best_p, st->p, sizeof(int32_t) * (size_t)n);
            }
            /* R18: wrapping sum of one hash per accepted (k, r, s) */
            st->digest += mix64(mix64(k) ^ (((uint64_t)(uint32_t)r << 32) | (uint32_t)s));
            if (check_every > 0 && (int64_t)(st->accepted % (uint64_t)check_every) == 0) {
                if (check_state(st) != 0) { status = -1; st->iterations += it + 1; goto done; }
            }
        }
        /* next possible swap: cursor + 1, cyclic (F2 / R4) */
        if (!st->proposal && ++s == n) {
            ++r;
            if (r == n - 1) r = 0;
            s = r + 1;
        }
    }
    st->iterations += iters;
done:
    free(dA);
    free(dB);
    return status < 0 ? -1 : (n_logged < near_cap ? n_logged : near_cap);
}

/* ------------------------------------------------------------------ */
/* Start permutation of a chain (R14b).  */
/* ------------------------------------------------------------------ */
/* Fisher-Yates from the identity (Knuth, TAOCP vol. 2, Algorithm 3.4.2 P): for i = n-1 down to 1,
 * j = floor(x (i+1) / 2^32) with x the first word of Philox4x32-10(key = seed, ctr = (i, 0, chain,
 * tag 1)), then swap p[i] and p[j].  j is uniform on 0..i up to the 2^-32 granularity of x. */
void orc_start_perm(int n, uint64_t seed, uint32_t chain, int32_t* p) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int i = 0; i < n; ++i) p[i] = i;
    for (int i = n - 1; i >= 1; --i) {
        const uint32_t ctr[4] = {(uint32_t)i, 0u, chain, 1u};
        uint32_t x[4];
        orc_philox4x32_10(ctr, key, x);
        const int j = (int)(((uint64_t)x[0] * (uint64_t)(i + 1)) >> 32);
        const int32_t t = p[i]; p[i] = p[j]; p[j] = t;
    }
}

/* ------------------------------------------------------------------ */
/* Independent chains (BASELINE config 5) on host threads.       */
/* ------------------------------------------------------------------ */
typedef struct {
    int n; const int32_t* A; const int32_t* B; const int32_t* p0s;
    int64_t begin, end; uint64_t iters; int kind; double t0, tf; uint64_t seed;
    uint32_t chain_base; int mode; int64_t* out; uint64_t* near_k; uint8_t* near_d; int near_cap;
    int64_t* next; pthread_mutex_t* lock;
} ens_job;

static void* ens_worker(void* arg) {
    ens_job* j = (ens_job*)arg;
    int n = j->n;
    int32_t* p = malloc(sizeof(int32_t) * n);
    int32_t* bp = malloc(sizeof(int32_t) * n);
    int32_t* p0 = malloc(sizeof(int32_t) * n);
    int32_t* Bp = malloc(sizeof(int32_t) * n * n);
    int64_t* D = malloc(sizeof(int64_t) * (size_t)(n * (n - 1) / 2 + 1));
    for (;;) {
        pthread_mutex_lock(j->lock);
        int64_t c = (*j->next)++;
        pthread_mutex_unlock(j->lock);
        if (c >= j->end) break;
        const uint32_t chain = j->chain_base + (uint32_t)(c - j->begin);
        if (j->p0s) memcpy(p0, j->p0s + (size_t)(c - j->begin) * n, sizeof(int32_t) * (size_t)n);
        else orc_start_perm(n, j->seed, chain, p0);
        orc_state st = {n, j->mode, j->A, j->B, p, bp, Bp, D, 0, 0, 0, 0, 0, 0, 0, 0};
        orc_state_reset(&st, p0);
        const size_t lo = (size_t)(c - j->begin) * (size_t)j->near_cap;
        orc_sa_run(&st, 0, j->iters, j->kind, j->t0, j->tf, j->iters, j->seed, chain, NULL, NULL, 0,
                   j->near_k ? j->near_k + lo : NULL, j->near_d ? j->near_d + lo : NULL, j->near_cap, 0);
        int64_t* o = j->out + (size_t)(c - j->begin) * 6;
        o[0] = st.cost; o[1] = st.best_cost; o[2] = (int64_t)st.accepted;
        o[3] = (int64_t)st.near_ties; o[4] = (int64_t)st.digest; o[5] = (int64_t)st.iterations;
    }
    free(p); free(bp); free(p0); free(Bp); free(D);
    return NULL;
}

/* Runs chains chain_base .. chain_base+count-1, each for iters iterations of its own schedule,
 * with δ taken from `mode` (ORC_MODE_*; all three give the same trajectory).  Start permutations:
 * p0s (count*n) or, if p0s is NULL, orc_start_perm(seed, chain).  out: count*6 int64 (cost,
 * best_cost, accepted, near_ties, digest, iterations); near_k/near_d (nullable, count*near_cap):
 * each chain's first near_cap near ties (k, decision). */
int orc_ensemble_run(int n, const int32_t* A, const int32_t* B, const int32_t* p0s, int64_t count,
                     uint32_t chain_base, uint64_t iters, int kind, double t0, double tf,
                     uint64_t seed, int threads, int mode, int64_t* out, uint64_t* near_k,
                     uint8_t* near_d, int near_cap) {
    if (threads < 1) threads = 1;
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    pthread_mutex_t lock = PTHREAD_MUTEX_INITIALIZER;
    int64_t next = 0;
    ens_job job = {n, A, B, p0s, 0, count, iters, kind, t0, tf, seed, chain_base, mode, out,
                   near_k, near_d, near_cap, &next, &lock};
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, ens_worker, &job);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return 0;
}
