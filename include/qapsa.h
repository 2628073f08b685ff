/*
 * qapsa.h -- C ABI of the B200-native Δ-matrix simulated annealing library
 * for the Quadratic Assignment Problem (G. Paul, arXiv 1208.2675).
 *
 * Citation keys: P:n = reference PAPER.md line n, S:n = SPEC.md line n,
 * R# = DESIGN.md "Readings of the paper" item #.
 *
 * Problem: N facilities, flow matrix A (N x N), distance matrix B
 * (N x N); find the permutation p (facility i -> location p(i)) minimising
 * Eq.(1)  C = sum_i sum_j A_ij B_{p(i),p(j)}.
 * Method: Δ-matrix simulated annealing -- Δ_rs = change of
 * C if p(r),p(s) are swapped, kept for every pair; candidate swaps are taken in
 * a fixed sequential order (R4), each tested against Eq.(2) with its
 * own temperature T_k (R1) and uniform r_k (R3); after an accepted swap Δ is
 * updated in O(N^2) (R10) and B' = B[p][p] by exchanging two rows and two
 * columns.
 *
 * Conventions (all entry points):
 *  - Host arrays are row-major int32, read during the call only; the caller
 *    keeps ownership.  Outputs go to caller-allocated host buffers of the
 *    stated length (n for permutations, M = n(n-1)/2 for Δ).
 *  - Δ layout: upper triangle r < s in row-major enumeration order,
 *    index k(r,s) = r*n - r(r+1)/2 + (s - r - 1)  (R11).  This is also
 *    the candidate order: iteration k proposes the pair with index k mod M.
 *  - All device memory is owned by the context and comes from a per-device
 *    stream-ordered pool of the library (allocated and released on the
 *    context's stream, so the stream must outlive the context); released
 *    buffers are kept for the next context on the device (qap_trim_memory).
 *    Work is issued on the context's stream; every call returns after that
 *    stream is synchronised.
 *  - A validation failure returns an error and leaves the context unchanged.
 *    A CUDA failure is sticky: the call returns QAP_E_CUDA and so do all
 *    later calls on that context (qap_last_error() has the CUDA message).
 *  - One context per host thread at a time.
 *  - There is no CPU fallback: without a usable sm_100 device every call
 *    that needs one returns QAP_E_CUDA.
 */
#ifndef QAPSA_H
#define QAPSA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QAPSA_VERSION 1

typedef struct qap_ctx qap_ctx; /* opaque */

typedef enum {
    QAP_OK = 0,
    QAP_E_INVALID_ARG = 1, /* NULL pointer, n < 2, n > QAP_MAX_N, iters == 0, chains == 0, cap < 0 */
    QAP_E_DIMENSION = 2,   /* a permutation that is not a bijection on 0..n-1 */
    QAP_E_UNSUPPORTED = 3, /* A or B asymmetric, nonzero diagonal, negative or > 65535 entries (R12) */
    QAP_E_OVERFLOW = 4,    /* 4 n maxA maxB >= 2^31 (int32 Δ and dot products, R13) */
    QAP_E_SCHEDULE = 5,    /* kind unknown, !(t0 >= tf > 0), non-finite, total_iters == 0,
                              or the iteration range exceeds total_iters */
    QAP_E_STATE = 6,       /* Δ not initialised for the current p (call qap_delta_init) */
    QAP_E_CUDA = 7,        /* CUDA error or no usable device (sticky) */
    QAP_E_NOMEM = 9        /* device or host allocation failed */
} qap_status;

#define QAP_MAX_N 512   /* and A, B' must fit in one SM's shared memory, or the chain in a cluster's (cluster
                           engine, 8-bit A); else QAP_E_UNSUPPORTED */

typedef enum { QAP_COOL_GEOMETRIC = 0, QAP_COOL_LUNDY_MEES = 1 } qap_cooling;

/* Cooling schedule ("slowly decreased according to a specified cooling
 * schedule after each iteration"), a closed form in the global iteration k
 * (R1).  total_iters = I, the length of the whole run; t0 = T_0, tf = T_{I-1}.
 *   GEOMETRIC:   T_k = t0 * exp(lambda * k),     lambda = ln(tf/t0) / (I-1)
 *   LUNDY_MEES:  T_k = t0 / (1 + (k beta) t0),   beta = (t0-tf) / (((I-1) t0) tf)
 * (lambda = beta = 0 when I = 1), evaluated in IEEE double without FMA. */
typedef struct {
    int32_t kind;          /* qap_cooling */
    int32_t reserved;      /* must be 0 */
    double t0;
    double tf;
    uint64_t total_iters;
} qap_schedule;

/* Statistics of one qap_sa_run call (counts cover that call only; cost,
 * best_cost and digest are the context's running values). */
typedef struct {
    uint64_t iterations;   /* proposals evaluated (= iters) */
    uint64_t accepted;     /* accepted swaps; a(I) = accepted / iterations */
    uint64_t near_ties;    /* proposals with delta > 0 and |delta + T ln r| < 1e-9 T (R16) */
    int64_t cost;          /* current C (Eq.(1)) */
    int64_t best_cost;     /* min C since qap_reset / qap_create (R17) */
    uint64_t digest;       /* running trajectory digest over accepted (k, r, s) (R18) */
} qap_stats;

/* Per-chain result of qap_ensemble_run. */
typedef struct {
    int64_t cost;
    int64_t best_cost;
    uint64_t accepted;
    uint64_t near_ties;
    uint64_t digest;
    uint64_t iterations;
} qap_chain_result;

/* qap_create -- problem statement of P:20-24.
 *  n:      problem size N, 2 <= n <= QAP_MAX_N.
 *  A, B:   n*n row-major int32 host arrays: flows A (facilities) and distances
 *          B (locations); symmetric, zero diagonal, entries in [0, 65535]
 *          (the family of P:105); otherwise QAP_E_UNSUPPORTED.
 *  p0:     n int32 host array, start permutation, p0[i] = location of facility i.
 *  device: CUDA device ordinal.
 *  stream: cudaStream_t to issue work on (NULL = the legacy default stream).
 *          PyTorch passes torch.cuda.current_stream().cuda_stream.
 *  out:    receives the new context.
 * Sets p = p0, B' = B[p0][p0], C = Eq.(1)(p0), best = C, digest = its seed
 * value; Δ is NOT yet valid (qap_delta_init). */
qap_status qap_create(int32_t n, const int32_t* A, const int32_t* B, const int32_t* p0,
                      int32_t device, void* stream, qap_ctx** out);

/* Releases all device memory of ctx to the library's device pool (stream-
 * ordered on the context's stream) and frees ctx (NULL is a no-op). */
void qap_destroy(qap_ctx* ctx);

/* qap_trim_memory -- returns the unused part of the library's pool on
 * `device` to the driver (after synchronising the device).  Not on the hot
 * path: the pool exists so that repeated create / run / destroy cycles (the
 * end-to-end path) allocate nothing in steady state.
 * Errors: QAP_E_INVALID_ARG for a bad ordinal, QAP_E_CUDA. */
qap_status qap_trim_memory(int32_t device);

/* qap_reset -- restart the chain from an assignment: "an initial assignment
 * p" (step (a)) and B' = B[p][p] (R9).  p = perm (n int32 host
 * array) or, if perm is NULL, the p0 of qap_create, kept on the device (no
 * host transfer).  Recomputes B', C = Eq.(1), best = C, best_p = p
 * (R17), digest seed (R18), clears the near-tie log; Δ becomes invalid until
 * qap_delta_init.  Errors: QAP_E_DIMENSION if perm is not a permutation. */
qap_status qap_reset(qap_ctx* ctx, const int32_t* perm);

/* qap_delta_init -- step (a) of P:46: Δ_rs for every pair r < s at the
 * current p, O(N^3) on the device (exact int32). */
qap_status qap_delta_init(qap_ctx* ctx);

/* qap_sa_run -- steps (b)-(e) of P:46-50 for global iterations
 * k = k0 .. k0+iters-1 of the schedule *s (k0 + iters <= s->total_iters),
 * one persistent kernel, no host round trip per iteration.
 * Iteration k proposes pair index k mod M (R4), draws
 * r_k = U(Philox4x32-10(key = seed, ctr = (k, chain 0, tag 0))) (R3) and
 * accepts iff delta < 0 or exp(-delta/T_k) > r_k (Eq.(2)).
 * Requires a valid Δ (QAP_E_STATE otherwise) and leaves it valid, so calls
 * over consecutive ranges continue one chain bit-exactly (resume).
 * out (nullable) receives the call's statistics. */
qap_status qap_sa_run(qap_ctx* ctx, uint64_t k0, uint64_t iters, const qap_schedule* s,
                      uint64_t seed, qap_stats* out);

/* qap_cost -- Eq.(1) of perm (n int32 host array, must be a
 * permutation) or, if perm is NULL, of the context's current p, computed on
 * the device in int64. */
qap_status qap_cost(qap_ctx* ctx, const int32_t* perm, int64_t* out);

/* qap_get_state -- the outputs of step (e) ("end after I iterations"):
 * copies the current assignment p, the best assignment best_p (R17; n int32
 * each) and the swap-cost matrix Δ (M int32, layout above) to
 * caller-owned host buffers; any of them may be NULL.
 * delta != NULL requires a valid Δ (QAP_E_STATE otherwise). */
qap_status qap_get_state(qap_ctx* ctx, int32_t* perm, int32_t* best_perm, int32_t* delta);

/* qap_get_near_ties -- Eq.(2) evaluated in double precision can be
 * decided differently by two correct implementations only when
 * |delta + T ln r| is within rounding of 0 (R16, BASELINE north_star): those
 * iterations k (delta > 0, |delta + T ln r| < 1e-9 T) flagged since the last
 * reset, with the decision the device took (1 = accepted), in the order they
 * were logged, up to cap entries (ks: cap uint64, decisions: cap uint8, host);
 * *count receives the total number flagged (may exceed cap; only the first
 * QAP_NEAR_LOG_CAP are kept). */
#define QAP_NEAR_LOG_CAP 1024
qap_status qap_get_near_ties(qap_ctx* ctx, uint64_t* ks, uint8_t* decisions, int32_t cap,
                             int32_t* count);

/* qap_schedule_bounds -- the T0/Tf rule of R2 (SPEC S:190 over all pairs):
 * dmin = smallest nonzero |Δ|, dmax = largest |Δ| at the current p;
 * t0 = dmin + (dmax - dmin)/10, tf = dmin; (1.0, 0.1) if Δ == 0.
 * Requires a valid Δ. */
qap_status qap_schedule_bounds(qap_ctx* ctx, double* t0, double* tf);

/* qap_ensemble_run -- independent chains ("run copies of the heuristic
 * independently"; BASELINE config 5) on the context's instance: chains with
 * GLOBAL ids chain_begin .. chain_begin + chain_count - 1, each running
 * iterations 0 .. iters-1 of *s with r_k keyed by (seed, k, c) (R3, R19).
 * Chain c starts from p0s[(c - chain_begin) * n ...] (chain_count*n int32,
 * host) or, if p0s is NULL, from the chain-keyed Fisher-Yates permutation
 * generated on the device (qap_start_perms(seed, c), R14b): no host array.
 * The context's single-chain state is not touched.
 *  best_cost/best_chain/best_perm (n int32): argmin over these chains of
 *      best_cost, ties to the lowest chain id;
 *  sum_stats (nullable): summed iterations/accepted/near_ties, digest =
 *      XOR of chain digests, cost/best_cost = those of best_chain;
 *  per_chain (nullable): chain_count results in chain order.
 * Engine: on instances the tensor-memory engine takes (and QAP_OPT_TENSOR_CORE = 1,
 * QAP_OPT_PROPOSAL = 0) the single-chain tensor-memory kernels run over all chains, one CTA
 * per chain (two per SM in the scratch phase); otherwise the shared-memory kernel runs several
 * chains per CTA (QAP_OPT_ENSEMBLE_GROUP threads each).  Same results either way. */
qap_status qap_ensemble_run(qap_ctx* ctx, uint32_t chain_begin, uint32_t chain_count,
                            const int32_t* p0s, uint64_t iters, const qap_schedule* s,
                            uint64_t seed, int64_t* best_cost, uint32_t* best_chain,
                            int32_t* best_perm, qap_stats* sum_stats,
                            qap_chain_result* per_chain);

/* qap_ensemble_near_ties -- the near ties (R16, see qap_get_near_ties) of the
 * last qap_ensemble_run, every entry with its GLOBAL chain id, so that each
 * flagged chain can be replayed with the device's decisions.  chains (uint32),
 * ks (uint64), decisions (uint8): cap entries each, host; *count = the total
 * flagged in that run (only the first QAP_ENS_NEAR_LOG_CAP are kept). */
#define QAP_ENS_NEAR_LOG_CAP 65536
qap_status qap_ensemble_near_ties(qap_ctx* ctx, uint32_t* chains, uint64_t* ks, uint8_t* decisions,
                                  int32_t cap, int32_t* count);

/* qap_start_perms -- initial assignments of independent chains (P:46 step (a)
 * "an initial assignment p"): chain c = chain_begin .. chain_begin +
 * count - 1 gets the Fisher-Yates shuffle of the identity with, for
 * i = n-1 .. 1, j = floor(x (i+1) / 2^32), x = Philox4x32-10(key = seed,
 * ctr = (i, 0, c, tag 1)).x, swap p[i], p[j] (R14b), computed on
 * the device.  out: count*n int32 host buffer, row c - chain_begin = p of c. */
qap_status qap_start_perms(qap_ctx* ctx, uint64_t seed, uint32_t chain_begin, uint32_t count,
                           int32_t* out);

/* Tuning knobs.  Results never depend on them (window / CTA shape
 * invariance); they exist for the invariance tests and benchmarks. */
typedef enum {
    QAP_OPT_WINDOW_MAX = 1,      /* max candidates per window, multiple of 32 in 32..8192 (default:
                                    1024; the tensor-memory Δ engine scans whole rows, up to 7168) */
    QAP_OPT_THREADS = 2,         /* single-chain CTA threads: 0 = auto (default), 64..1024 */
    QAP_OPT_FORCE_GLOBAL_DELTA = 3, /* 1: keep Δ in global memory/L2 even if it fits on chip */
    QAP_OPT_ENSEMBLE_GROUP = 4,  /* threads per chain in qap_ensemble_run: 64, 128 or 256 */
    QAP_OPT_TENSOR_CORE = 5,     /* qap_sa_run engine: 1 (default) = Δ in tensor memory with the
                                    rank update on the tensor cores when the instance allows it
                                    (4 <= n <= 128, all entries <= 127) and proposals are
                                    sequential, else the shared-memory kernel; 2 = also for random
                                    proposals (R22; slower than the shared-memory kernel); 0 =
                                    always the shared-memory kernel */
    QAP_OPT_SCRATCH_PHASE = 6,   /* tensor-memory engine only: 1 (default) = run the high-acceptance
                                    start of each qap_sa_run without Δ (δ from G = A B'^T, SURVEY
                                    f2) until no swap is accepted for 4096 iterations, then rebuild
                                    Δ and continue with Δ; 0 = Δ throughout.  Same trajectory. */
    QAP_OPT_RELABEL = 7,         /* instances with 8-bit A, 4 <= n <= 256, and either 16-bit B
                                    (config 4) or 8-bit B whose Δ would not fit the shared-memory
                                    kernel (n = 256): 1 (default) = relabel engine: swaps of twin
                                    locations (equal rows of A off the pair, R21) are
                                    exact O(1) index relabels, other swaps the ordinary update
                                    (SURVEY f3); 2 = the same engine with the relabels off; 3 =
                                    the relabel engine for every 8-bit-A instance with
                                    4 <= n <= 256 not on the tensor-memory engine; 0 = the
                                    shared-memory kernel.  Same trajectory in every case. */
    QAP_OPT_RELABEL_CLUSTER = 8, /* relabel engine: 8 (default) = one chain on a thread-block
                                    cluster of 8 SMs, Δ spread over their shared memory (SURVEY
                                    f1); 1 = one SM, Δ in L2 */
    QAP_OPT_PROPOSAL = 9,        /* candidate order: 0 (default) = the sequential cyclic
                                    enumeration (R4); 1 = random pairs, iteration k proposes pair
                                    index floor(x M / 2^32), x = Philox(seed; k, chain, tag 3)
                                    (R22); the shared-memory kernel (single chain and
                                    qap_ensemble_run), or with QAP_OPT_TENSOR_CORE = 2 the
                                    tensor-memory Δ engine (windows of up to 256 random candidates
                                    whose Δ cells are gathered from their TMEM lanes) */
    QAP_OPT_CLUSTER_ENGINE = 10, /* cluster engine (f1; one chain spread over the
                                    shared memory of a thread-block cluster of 8 SMs, rows of A,
                                    B' and Δ distributed, N up to QAP_MAX_N): 1 (default) = only
                                    for chains no single SM holds (N > 256, 8-bit A); 2 = always
                                    (8-bit A, n >= 4); 0 = never.  Same trajectory either way. */
    QAP_OPT_ENSEMBLE_SCRATCH4 = 11, /* tensor-memory ensembles: 1 (default) = the scratch phase of four
                                    chains per SM (G only in tensor memory, 128 columns; the window's
                                    rows of G exchanged through shared memory); 0 = two chains per
                                    SM (G and H).  Same results either way. */
    QAP_OPT_SWITCH_GAP = 12      /* tensor-memory engine: the scratch phase hands over to the Δ engine
                                    after this many iterations without an accept; 0 (default) =
                                    4096 for single chains, 65536 for ensembles.  Same results. */
} qap_option;
qap_status qap_set_option(qap_ctx* ctx, int32_t key, int64_t value);
/* 1 if the next qap_sa_run uses the tensor-memory engine (QAP_OPT_TENSOR_CORE), else 0. */
int32_t qap_uses_tensor_core(const qap_ctx* ctx);
/* The engine the next qap_sa_run uses (QAP_ENGINE_*), -1 if ctx is NULL. */
enum { QAP_ENGINE_SHARED_MEMORY = 0, QAP_ENGINE_TENSOR_MEMORY = 1, QAP_ENGINE_RELABEL = 2, QAP_ENGINE_CLUSTER = 3 };
int32_t qap_engine(const qap_ctx* ctx);

/* Device time in milliseconds of the last qap_sa_run kernel (CUDA events
 * on the context stream), and the number of kernels the last call launched. */
qap_status qap_last_kernel_time(qap_ctx* ctx, float* ms, int32_t* launches);
/* The last qap_sa_run's scratch phase (QAP_OPT_SCRATCH_PHASE): device time in milliseconds
 * (CUDA events around its kernel; the rest of qap_last_kernel_time is the Δ rebuild and the Δ
 * engine), the iteration it reached (where the Δ engine took over) and the swaps it accepted.
 * All zero if it did not run.  Any argument may be NULL. */
qap_status qap_last_scratch_time(qap_ctx* ctx, float* ms, uint64_t* k_reached, uint64_t* accepted);

const char* qap_status_str(qap_status st);
/* Last error message on ctx ("" if none); static string if ctx is NULL. */
const char* qap_last_error(const qap_ctx* ctx);
int32_t qap_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QAPSA_H */
