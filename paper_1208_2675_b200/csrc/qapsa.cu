// qapsa.cu -- C ABI (include/qapsa.h): validation, device memory, launches.
//
// Every step of the hot path runs in the kernels of kernels.cuh; this file
// only validates arguments, converts the int32 host matrices to their compact
// device form (uint8 or uint16, rows padded to a multiple of 4 elements),
// chooses the kernel instance and moves results back.  There is no CPU
// fallback: without an sm_100 device the calls fail with QAP_E_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qapsa.h"
#include "kernels.cuh"
#include "tc_chain.cuh"
#include "scratch_chain.cuh"
#include "relabel_chain.cuh"
#include "cluster_chain.cuh"
#include "ens_chain.cuh"

using namespace qapsa;

// Device memory: one stream-ordered pool per device, owned by the library.  A freed buffer stays in
// the pool (release threshold = max) and serves the next context on that device, so the
// create / run / destroy cycle of the end-to-end path allocates nothing from the driver in steady
// state (a plain cudaMalloc / cudaFree pair costs milliseconds and, measured on the B200, stalls
// for up to 100 ms at times).  qap_trim_memory() hands the unused part back.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[128];

static cudaMemPool_t dev_pool(int dev) {
    if (dev < 0 || dev >= 128) return nullptr;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        g_pool[dev] = pool;
    }
    return g_pool[dev];
}

struct qap_ctx {
    int n = 0, ld = 0, M = 0, dev = 0;
    cudaStream_t stream = nullptr;
    int ta = 1, tb = 1;                 // bytes per A / B element on the device
    void* dA = nullptr;
    void* dB = nullptr;
    int32_t *dp0 = nullptr, *dp = nullptr, *dbest = nullptr, *dD = nullptr, *dperm = nullptr;
    int32_t* dDlin = nullptr;           // M, enumeration-order copy of Δ
    int32_t* drowaddr = nullptr;        // n, quad layout row addresses
    uint16_t* dqdesc = nullptr;         // nqt, quad descriptors
    int nqt = 0;
    DevState* dst = nullptr;
    unsigned int* dnear_count = nullptr;
    unsigned long long* dnear_k = nullptr;
    unsigned char* dnear_dec = nullptr;
    long long* dscratch = nullptr;      // 8 x int64
    // ensemble buffers (grown on demand)
    int32_t* ens_p0 = nullptr;
    ChainResult* ens_res = nullptr;
    uint16_t* ens_best = nullptr;
    unsigned int* ens_counter = nullptr;
    size_t ens_cap = 0;
    bool delta_valid = false;
    bool sticky = false;
    std::string err;
    long long switch_gap = 0;            // QAP_OPT_SWITCH_GAP (0 = engine default)
    int ens4 = 1;                        // QAP_OPT_ENSEMBLE_SCRATCH4: ensemble scratch phase 4 chains per SM
    int use_cluster = 1;                 // QAP_OPT_CLUSTER_ENGINE: 0 never, 1 when needed (default), 2 always
    int wmax = 0 /* auto */, threads = 0 /* auto */, force_global = 0, ens_group = 128;
    int smem_optin = 0, num_sms = 0;
    bool tc_ok = false;                 // instance fits the tensor-memory engine (tc_chain.cuh)
    int use_tc = 1;
    int use_scratch = 1;                // high-acceptance phase without Δ (scratch_chain.cuh)
    unsigned long long* dkout = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evm = nullptr;   // evm: after the scratch phase
    float last_scratch_ms = 0.f;
    unsigned long long last_scratch[2] = {0, 0};   // iteration reached, accepted swaps
    float last_ms = 0.f;
    int last_launches = 0;
    // relabel engine (relabel_chain.cuh): twin classes of A, second Δ buffer for the write-back
    int use_relabel = 1;                // QAP_OPT_RELABEL
    int rlb_cluster = 8;                // QAP_OPT_RELABEL_CLUSTER: CTAs sharing Δ~ (1 = Δ~ in L2)
    int proposal = 0;                   // QAP_OPT_PROPOSAL: 0 sequential (R4), 1 random (R22)
    // tensor-memory ensemble (per-chain state of k_sa_scratch / k_sa_tc ensemble launches)
    int32_t *tp = nullptr, *tbp = nullptr, *tD = nullptr;
    DevState* tst = nullptr;
    unsigned long long* tkout = nullptr;
    size_t tcap = 0;
    int ncls = 0;
    uint8_t* dcls = nullptr;            // n
    uint16_t* dpt = nullptr;            // ncls x (n+1)
    int32_t* dD2 = nullptr;             // quad layout, same size as dD
    // integer thresholds of a single-chain call's iterations and their block headers (k_theta,
    // theta_ring.cuh), grown on demand
    int* dtheta = nullptr;
    int4* dtheta_hdr = nullptr;
    size_t theta_cap = 0;
    // near-tie log of the last qap_ensemble_run: (chain, k, decision), R16
    unsigned int* ens_near_count = nullptr;
    unsigned long long* ens_near_k = nullptr;
    unsigned char* ens_near_dec = nullptr;
    uint32_t* ens_near_chain = nullptr;
};

static thread_local std::string g_static_err;

static qap_status fail(qap_ctx* c, qap_status st, const std::string& msg) {
    if (c) c->err = msg;
    else g_static_err = msg;
    return st;
}

#define CU(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            if (c) c->sticky = true;                                                         \
            return fail(c, QAP_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
        }                                                                                    \
    } while (0)

#define CHECK_CTX(c)                                                        \
    do {                                                                    \
        if (!(c)) return fail(nullptr, QAP_E_INVALID_ARG, "ctx is NULL");  \
        if ((c)->sticky) return QAP_E_CUDA;                                 \
    } while (0)

static bool is_perm(int n, const int32_t* p) {
    std::vector<char> seen(n, 0);
    for (int i = 0; i < n; ++i) {
        if (p[i] < 0 || p[i] >= n || seen[p[i]]) return false;
        seen[p[i]] = 1;
    }
    return true;
}

// A or B: symmetric, zero diagonal, 0 <= x <= 65535 (R12).
static bool instance_ok(int n, const int32_t* X, int32_t* maxv, std::string* why, const char* name) {
    int32_t mx = 0;
    for (int i = 0; i < n; ++i) {
        if (X[(size_t)i * n + i] != 0) { *why = std::string(name) + " has a nonzero diagonal"; return false; }
        for (int j = 0; j < n; ++j) {
            const int32_t v = X[(size_t)i * n + j];
            if (v < 0 || v > 65535) { *why = std::string(name) + " entry outside [0, 65535]"; return false; }
            if (v != X[(size_t)j * n + i]) { *why = std::string(name) + " is not symmetric"; return false; }
            if (v > mx) mx = v;
        }
    }
    *maxv = mx;
    return true;
}

template <typename T>
static std::vector<unsigned char> compact(int n, int ld, const int32_t* X) {
    std::vector<unsigned char> out((size_t)n * ld * sizeof(T), 0);
    T* o = reinterpret_cast<T*>(out.data());
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) o[(size_t)i * ld + j] = (T)X[(size_t)i * n + j];
    return out;
}

// single chains: sequential proposals (R4); random ones (R22) only when forced
// (QAP_OPT_TENSOR_CORE = 2: measured slower than the shared-memory engine, config 3: 2.0e7 vs
// 6.0e7 it/s); ensembles: sequential only
static bool use_tc_engine(const qap_ctx* c) {
    return c->tc_ok && c->use_tc && !c->force_global && (c->proposal == 0 || c->use_tc == 2);
}
static bool use_tc_ensemble(const qap_ctx* c) { return use_tc_engine(c) && c->proposal == 0; }

static int dab_bytes(const qap_ctx* c) { return (c->ta == 1 && c->tb == 1) ? 4 : 8; }

static int chain_smem_bytes(const qap_ctx* c, int threads, bool d_smem) {
    const GroupLayout L = group_layout(c->n, c->ld, c->nqt, c->tb, threads / 32, d_smem, dab_bytes(c));
    return cta_prefix_bytes(c->n, c->ld, c->ta, c->nqt) + L.bytes;
}

// Quad layout of Δ (chain.cuh): row u keeps column quads floor((u+1)/4) .. ceil(n/4)-1.
static void quad_tables(int n, std::vector<int32_t>* rowaddr, std::vector<uint16_t>* qdesc) {
    const int NQ = (n + 3) / 4;
    rowaddr->assign(n, 0);
    qdesc->clear();
    for (int u = 0; u + 1 < n; ++u) {
        const int j0 = (u + 1) / 4;
        (*rowaddr)[u] = 4 * (int)qdesc->size() - 4 * j0;
        for (int j = j0; j < NQ; ++j) qdesc->push_back((uint16_t)(u | (j << 9)));
    }
}

// Twin classes of A (R21): x ~ y iff A_xz == A_yz for every z != x, y.  A class is kept only if
// all its members are pairwise twins; the RLB_MAXCLS largest classes with >= 2 members get
// indices, every other location 0xFF (its swaps take the ordinary update, which is exact for
// any pair).  pt[c][x] = largest member of class c below x, 0xFFFF if none.
static void twin_classes(int n, const int32_t* A, std::vector<uint8_t>* cls, std::vector<uint16_t>* pt,
                         int* ncls) {
    auto twin = [&](int x, int y) {
        for (int z = 0; z < n; ++z)
            if (z != x && z != y && A[(size_t)x * n + z] != A[(size_t)y * n + z]) return false;
        return true;
    };
    std::vector<std::vector<int>> classes;
    for (int x = 0; x < n; ++x) {
        bool placed = false;
        for (auto& cl : classes) {
            if (!twin(cl[0], x)) continue;
            bool all = true;
            for (int y : cl) all = all && twin(y, x);
            if (all) { cl.push_back(x); placed = true; break; }
        }
        if (!placed) classes.push_back({x});
    }
    std::vector<int> order;
    for (int i = 0; i < (int)classes.size(); ++i)
        if (classes[i].size() >= 2) order.push_back(i);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return classes[a].size() > classes[b].size(); });
    if ((int)order.size() > RLB_MAXCLS) order.resize(RLB_MAXCLS);
    cls->assign(n, 0xFF);
    *ncls = (int)order.size();
    pt->assign((size_t)(*ncls) * (n + 1), 0xFFFF);
    for (int c = 0; c < *ncls; ++c) {
        for (int x : classes[order[c]]) (*cls)[x] = (uint8_t)c;
        int last = 0xFFFF;
        for (int x = 0; x <= n; ++x) {
            (*pt)[(size_t)c * (n + 1) + x] = (uint16_t)last;
            if (x < n && (*cls)[x] == c) last = x;
        }
    }
}

// The relabel engine runs 16-bit-B instances (config 4) and 8-bit ones whose Δ no longer fits
// the shared-memory engine's CTA (N = 256): measured, the shared-memory engine is faster while
// its Δ stays on chip (N = 150: 0.26 s vs 0.51 s, N = 200: 0.51 s vs 0.65 s for 1e7 iterations)
// and slower once Δ spills to L2 (N = 256: 0.64 s vs 0.46 s).
static bool use_relabel_engine(const qap_ctx* c) {
    const bool spills = c->n > 128 && chain_smem_bytes(c, 1024, true) > c->smem_optin;
    return c->use_relabel && c->proposal == 0 && c->ta == 1 && (c->tb == 2 || spills || c->use_relabel == 3) &&
           c->n >= 4 &&
           c->n <= RLB_MAXN &&
           rlb_layout(c->n, c->rlb_cluster).bytes <= c->smem_optin;
}

// The cluster engine (cluster_chain.cuh, f1) runs the chains that fit no single SM: N > 256, or
// whatever the other engines cannot hold on chip; QAP_OPT_CLUSTER_ENGINE = 2 forces it (tests).
static bool cluster_fits(const qap_ctx* c) {
    return c->ta == 1 && c->proposal == 0 && c->n >= 4 && cl_layout(c->n, c->tb).bytes <= c->smem_optin;
}
static bool use_cluster_engine(const qap_ctx* c) {
    if (!c->use_cluster || !cluster_fits(c)) return false;
    if (c->use_cluster == 2) return true;
    return c->n > RLB_MAXN || chain_smem_bytes(c, 256, false) > c->smem_optin;
}

static qap_status validate_schedule(qap_ctx* c, const qap_schedule* s, uint64_t k0, uint64_t iters,
                                    Sched* out) {
    if (!s) return fail(c, QAP_E_INVALID_ARG, "schedule is NULL");
    if (s->kind != QAP_COOL_GEOMETRIC && s->kind != QAP_COOL_LUNDY_MEES)
        return fail(c, QAP_E_SCHEDULE, "unknown cooling kind");
    if (s->reserved != 0) return fail(c, QAP_E_SCHEDULE, "reserved field must be 0");
    if (!std::isfinite(s->t0) || !std::isfinite(s->tf) || !(s->tf > 0.0) || !(s->t0 >= s->tf))
        return fail(c, QAP_E_SCHEDULE, "need finite t0 >= tf > 0");
    if (s->total_iters == 0) return fail(c, QAP_E_SCHEDULE, "total_iters == 0");
    if (k0 > s->total_iters || iters > s->total_iters - k0)
        return fail(c, QAP_E_SCHEDULE, "iteration range exceeds total_iters");
    // R1: coefficients once on the host, in double.
    const double I1 = (double)(s->total_iters - 1);
    out->kind = s->kind;
    out->t0 = s->t0;
    out->t0f = (float)s->t0;
    if (s->kind == QAP_COOL_GEOMETRIC)
        out->coef = s->total_iters > 1 ? std::log(s->tf / s->t0) / I1 : 0.0;
    else
        out->coef = s->total_iters > 1 ? (s->t0 - s->tf) / ((I1 * s->t0) * s->tf) : 0.0;
    out->coeff = (float)out->coef;
    return QAP_OK;
}

extern "C" {

int32_t qap_version(void) { return QAPSA_VERSION; }

const char* qap_status_str(qap_status st) {
    switch (st) {
        case QAP_OK: return "QAP_OK";
        case QAP_E_INVALID_ARG: return "QAP_E_INVALID_ARG";
        case QAP_E_DIMENSION: return "QAP_E_DIMENSION";
        case QAP_E_UNSUPPORTED: return "QAP_E_UNSUPPORTED";
        case QAP_E_OVERFLOW: return "QAP_E_OVERFLOW";
        case QAP_E_SCHEDULE: return "QAP_E_SCHEDULE";
        case QAP_E_STATE: return "QAP_E_STATE";
        case QAP_E_CUDA: return "QAP_E_CUDA";
        case QAP_E_NOMEM: return "QAP_E_NOMEM";
    }
    return "QAP_E_UNKNOWN";
}

const char* qap_last_error(const qap_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_static_err.c_str();
}

// stream-ordered allocation / release on the context's stream from the device pool
static cudaError_t dalloc(qap_ctx* c, void* p, size_t bytes) {
    cudaMemPool_t pool = dev_pool(c->dev);
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync((void**)p, bytes, pool, c->stream);
}
static void dfree(qap_ctx* c, void* p) {
    if (p) cudaFreeAsync(p, c->stream);
}

qap_status qap_trim_memory(int32_t device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(nullptr, QAP_E_INVALID_ARG, "bad device ordinal");
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (device < 128) pool = g_pool[device];
    }
    if (pool && (cudaSetDevice(device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
                 cudaMemPoolTrimTo(pool, 0) != cudaSuccess))
        return fail(nullptr, QAP_E_CUDA, "cudaMemPoolTrimTo failed");
    return QAP_OK;
}

void qap_destroy(qap_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    void* ptrs[] = {c->dA, c->dB, c->dp0, c->dp, c->dbest, c->dD, c->dperm, c->dDlin, c->drowaddr,
                    c->dqdesc, c->dst, c->dnear_count,
                    c->dnear_k, c->dnear_dec, c->dscratch, c->ens_p0, c->ens_res, c->ens_best,
                    c->ens_counter, c->dkout, c->dcls, c->dpt, c->dD2, c->tp, c->tbp, c->tD,
                    c->tst, c->tkout, c->ens_near_count, c->ens_near_k, c->ens_near_dec,
                    c->ens_near_chain, c->dtheta, c->dtheta_hdr};
    for (void* p : ptrs) dfree(c, p);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->evm) cudaEventDestroy(c->evm);
    delete c;
}

static qap_status launch_reset(qap_ctx* c, const int32_t* src) {
    if (c->ta == 1 && c->tb == 1)
        k_reset<uint8_t, uint8_t><<<1, 512, 0, c->stream>>>((const uint8_t*)c->dA, (const uint8_t*)c->dB, src, c->n, c->ld, c->dp, c->dbest, c->dst);
    else if (c->ta == 1)
        k_reset<uint8_t, uint16_t><<<1, 512, 0, c->stream>>>((const uint8_t*)c->dA, (const uint16_t*)c->dB, src, c->n, c->ld, c->dp, c->dbest, c->dst);
    else if (c->tb == 1)
        k_reset<uint16_t, uint8_t><<<1, 512, 0, c->stream>>>((const uint16_t*)c->dA, (const uint8_t*)c->dB, src, c->n, c->ld, c->dp, c->dbest, c->dst);
    else
        k_reset<uint16_t, uint16_t><<<1, 512, 0, c->stream>>>((const uint16_t*)c->dA, (const uint16_t*)c->dB, src, c->n, c->ld, c->dp, c->dbest, c->dst);
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(c->dnear_count, 0, sizeof(unsigned int), c->stream));
    c->delta_valid = false;
    return QAP_OK;
}

qap_status qap_create(int32_t n, const int32_t* A, const int32_t* B, const int32_t* p0, int32_t device,
                      void* stream, qap_ctx** out) {
    qap_ctx* c = nullptr;
    if (!out || !A || !B || !p0) return fail(nullptr, QAP_E_INVALID_ARG, "NULL argument");
    *out = nullptr;
    if (n < 2 || n > QAP_MAX_N) return fail(nullptr, QAP_E_INVALID_ARG, "n out of range");
    std::string why;
    int32_t maxA = 0, maxB = 0;
    if (!instance_ok(n, A, &maxA, &why, "A") || !instance_ok(n, B, &maxB, &why, "B"))
        return fail(nullptr, QAP_E_UNSUPPORTED, why);
    // R13: every partial dot product and Δ entry stays below 2^31.
    if (4.0 * (double)n * (double)maxA * (double)maxB >= 2147483648.0)
        return fail(nullptr, QAP_E_OVERFLOW, "4 n maxA maxB >= 2^31");
    if (!is_perm(n, p0)) return fail(nullptr, QAP_E_DIMENSION, "p0 is not a permutation");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, QAP_E_CUDA, "no CUDA device (libqapsa has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(nullptr, QAP_E_INVALID_ARG, "bad device ordinal");
    // three attributes (cudaGetDeviceProperties queries them all and costs milliseconds per call)
    int major = 0, smem_optin = 0, num_sms = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess || major < 10 ||
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess ||
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return fail(nullptr, QAP_E_CUDA, "device is not sm_100 (Blackwell)");

    c = new qap_ctx();
    c->n = n;
    c->ld = row_stride(n, maxA <= 255 && maxB <= 255);
    c->M = n * (n - 1) / 2;
    c->dev = device;
    c->stream = (cudaStream_t)stream;
    c->ta = maxA <= 255 ? 1 : 2;
    c->tb = maxB <= 255 ? 1 : 2;
    c->tc_ok = tc_eligible(n, maxA, maxB);
    c->smem_optin = smem_optin;
    std::vector<int32_t> hrow;
    std::vector<uint16_t> hq;
    quad_tables(n, &hrow, &hq);
    c->nqt = (int)hq.size();
    c->num_sms = num_sms;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return fail(nullptr, QAP_E_CUDA, "cudaSetDevice failed");
    }
    // A and B' must fit on one SM (Δ may spill to global memory / L2), or the chain must fit the
    // shared memory of a cluster (cluster engine, f1)
    if (chain_smem_bytes(c, 256, false) > c->smem_optin && !cluster_fits(c)) {
        delete c;
        return fail(nullptr, QAP_E_UNSUPPORTED, "the chain fits neither one SM nor a cluster's shared memory");
    }
    const size_t nA = (size_t)n * c->ld * c->ta, nB = (size_t)n * c->ld * c->tb;
    auto hA = c->ta == 1 ? compact<uint8_t>(n, c->ld, A) : compact<uint16_t>(n, c->ld, A);
    auto hB = c->tb == 1 ? compact<uint8_t>(n, c->ld, B) : compact<uint16_t>(n, c->ld, B);
    qap_status st = QAP_OK;
    auto alloc = [&](void** p, size_t bytes) {
        if (st != QAP_OK) return;
        if (dalloc(c, p, bytes) != cudaSuccess) st = fail(nullptr, QAP_E_NOMEM, "device allocation failed");
    };
    alloc(&c->dA, nA);
    alloc(&c->dB, nB);
    alloc((void**)&c->dp0, n * 4);
    alloc((void**)&c->dp, n * 4);
    alloc((void**)&c->dbest, n * 4);
    alloc((void**)&c->dperm, n * 4);
    alloc((void**)&c->dD, (size_t)c->nqt * 16 + 16);
    alloc((void**)&c->dDlin, (size_t)c->M * 4);
    alloc((void**)&c->drowaddr, (size_t)n * 4);
    alloc((void**)&c->dqdesc, (size_t)c->nqt * 4 + 4);
    alloc((void**)&c->dst, sizeof(DevState));
    alloc((void**)&c->dnear_count, sizeof(unsigned int));
    alloc((void**)&c->dnear_k, QAP_NEAR_LOG_CAP * sizeof(unsigned long long));
    alloc((void**)&c->dnear_dec, QAP_NEAR_LOG_CAP);
    alloc((void**)&c->dscratch, 8 * sizeof(long long));
    alloc((void**)&c->dkout, 2 * sizeof(unsigned long long));
    alloc((void**)&c->dD2, (size_t)c->nqt * 16 + 16);
    alloc((void**)&c->ens_near_count, sizeof(unsigned int));
    alloc((void**)&c->ens_near_k, QAP_ENS_NEAR_LOG_CAP * sizeof(unsigned long long));
    alloc((void**)&c->ens_near_dec, QAP_ENS_NEAR_LOG_CAP);
    alloc((void**)&c->ens_near_chain, QAP_ENS_NEAR_LOG_CAP * sizeof(uint32_t));
    std::vector<uint8_t> hcls;
    std::vector<uint16_t> hpt;
    twin_classes(n, A, &hcls, &hpt, &c->ncls);
    alloc((void**)&c->dcls, (size_t)n + 16);
    alloc((void**)&c->dpt, hpt.size() * 2 + 16);
    if (st != QAP_OK) {
        qap_destroy(c);
        return st;
    }
    if (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
        cudaEventCreate(&c->evm) != cudaSuccess) {
        qap_destroy(c);
        return fail(nullptr, QAP_E_CUDA, "cudaEventCreate failed");
    }
    cudaError_t e = cudaMemcpyAsync(c->dA, hA.data(), nA, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->dB, hB.data(), nB, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->dp0, p0, n * 4, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->drowaddr, hrow.data(), n * 4, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->dqdesc, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->dcls, hcls.data(), n, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess && !hpt.empty()) e = cudaMemcpyAsync(c->dpt, hpt.data(), hpt.size() * 2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->dD2, 0, (size_t)c->nqt * 16 + 16, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->ens_near_count, 0, sizeof(unsigned int), c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);   // host tables go out of scope
    if (e != cudaSuccess) {
        std::string m = cudaGetErrorString(e);
        qap_destroy(c);
        return fail(nullptr, QAP_E_CUDA, m);
    }
    st = launch_reset(c, c->dp0);
    if (st == QAP_OK && cudaStreamSynchronize(c->stream) != cudaSuccess)
        st = fail(c, QAP_E_CUDA, "create: stream synchronize failed");
    if (st != QAP_OK) {
        g_static_err = c->err;
        qap_destroy(c);
        return st;
    }
    c->last_launches = 1;
    *out = c;
    return QAP_OK;
}

qap_status qap_reset(qap_ctx* c, const int32_t* perm) {
    CHECK_CTX(c);
    if (perm && !is_perm(c->n, perm)) return fail(c, QAP_E_DIMENSION, "perm is not a permutation");
    CU(cudaSetDevice(c->dev));
    const int32_t* src = c->dp0;
    if (perm) {
        CU(cudaMemcpyAsync(c->dperm, perm, c->n * 4, cudaMemcpyHostToDevice, c->stream));
        src = c->dperm;
    }
    qap_status st = launch_reset(c, src);
    if (st != QAP_OK) return st;
    CU(cudaStreamSynchronize(c->stream));
    c->last_launches = 1;
    return QAP_OK;
}

qap_status qap_delta_init(qap_ctx* c) {
    CHECK_CTX(c);
    CU(cudaSetDevice(c->dev));
    const int threads = 256, blocks = (c->M + threads - 1) / threads;
    CU(cudaMemsetAsync(c->dD, 0, (size_t)c->nqt * 16, c->stream));   // dead slots of the quad layout
    if (c->ta == 1 && c->tb == 1)
        k_delta_init<uint8_t, uint8_t><<<blocks, threads, 0, c->stream>>>((const uint8_t*)c->dA, (const uint8_t*)c->dB, c->dp, c->drowaddr, c->n, c->ld, c->M, c->dD);
    else if (c->ta == 1)
        k_delta_init<uint8_t, uint16_t><<<blocks, threads, 0, c->stream>>>((const uint8_t*)c->dA, (const uint16_t*)c->dB, c->dp, c->drowaddr, c->n, c->ld, c->M, c->dD);
    else if (c->tb == 1)
        k_delta_init<uint16_t, uint8_t><<<blocks, threads, 0, c->stream>>>((const uint16_t*)c->dA, (const uint8_t*)c->dB, c->dp, c->drowaddr, c->n, c->ld, c->M, c->dD);
    else
        k_delta_init<uint16_t, uint16_t><<<blocks, threads, 0, c->stream>>>((const uint16_t*)c->dA, (const uint16_t*)c->dB, c->dp, c->drowaddr, c->n, c->ld, c->M, c->dD);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(c->stream));
    c->delta_valid = true;
    c->last_launches = 1;
    return QAP_OK;
}

}  // extern "C"

template <typename TA, typename TB, int NT, bool DS, int NFIX>
static cudaError_t launch_chain_t(qap_ctx* c, const ChainArgs& a, int smem) {
    auto kern = k_sa_chain<TA, TB, NT, DS, NFIX>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<1, NT, smem, c->stream>>>(a);
    return cudaGetLastError();
}

template <typename TA, typename TB, int NT>
static cudaError_t launch_generic(qap_ctx* c, const ChainArgs& a, bool ds, int smem) {
    return ds ? launch_chain_t<TA, TB, NT, true, 0>(c, a, smem)
              : launch_chain_t<TA, TB, NT, false, 0>(c, a, smem);
}

// Threads of the single-chain CTA: touching warps (8 v each) plus quad warps with
// <= 4 quads per thread, rounded to a power of two.
static int auto_threads(const qap_ctx* c) {
    const int need = 32 * touch_warps(c->n) + (c->nqt + 3) / 4;
    int nt = 64;
    while (nt < 1024 && nt < need) nt *= 2;
    return nt;
}

// Specialised instances (problem size fixed at compile time) for the BASELINE
// configurations; everything else runs the generic instance of the same code.
static cudaError_t launch_chain(qap_ctx* c, const ChainArgs& a, int threads, bool explicit_threads,
                                bool ds, int smem) {
    (void)explicit_threads;
    {
        if (c->ta == 1 && c->tb == 1 && ds) {
            if (c->n == 12 && threads == 64) return launch_chain_t<uint8_t, uint8_t, 64, true, 12>(c, a, smem);
            if (c->n == 50 && threads == 256) return launch_chain_t<uint8_t, uint8_t, 256, true, 50>(c, a, smem);
            if (c->n == 100 && threads == 512) return launch_chain_t<uint8_t, uint8_t, 512, true, 100>(c, a, smem);
            if (c->n == 100 && threads == 1024) return launch_chain_t<uint8_t, uint8_t, 1024, true, 100>(c, a, smem);
        }
        if (c->ta == 1 && c->tb == 2 && !ds && c->n == 256 && threads == 1024)
            return launch_chain_t<uint8_t, uint16_t, 1024, false, 256>(c, a, smem);
    }
    if (c->ta == 1 && c->tb == 1) {
        switch (threads) {
            case 64: return launch_generic<uint8_t, uint8_t, 64>(c, a, ds, smem);
            case 128: return launch_generic<uint8_t, uint8_t, 128>(c, a, ds, smem);
            case 256: return launch_generic<uint8_t, uint8_t, 256>(c, a, ds, smem);
            case 512: return launch_generic<uint8_t, uint8_t, 512>(c, a, ds, smem);
            default: return launch_generic<uint8_t, uint8_t, 1024>(c, a, ds, smem);
        }
    }
    if (c->ta == 1) return threads == 256 ? launch_generic<uint8_t, uint16_t, 256>(c, a, ds, smem)
                                          : launch_generic<uint8_t, uint16_t, 1024>(c, a, ds, smem);
    if (c->tb == 1) return launch_generic<uint16_t, uint8_t, 1024>(c, a, ds, smem);
    return launch_generic<uint16_t, uint16_t, 1024>(c, a, ds, smem);
}

// the instance launch_chain will actually run (for the shared-memory size)
static int effective_threads(const qap_ctx* c, int threads) {
    if (c->ta == 1 && c->tb == 1) return threads;
    if (c->ta == 1) return threads == 256 ? 256 : 1024;
    return 1024;
}

extern "C" {

qap_status qap_sa_run(qap_ctx* c, uint64_t k0, uint64_t iters, const qap_schedule* s, uint64_t seed,
                      qap_stats* out) {
    CHECK_CTX(c);
    if (iters == 0) return fail(c, QAP_E_INVALID_ARG, "iters == 0");
    Sched sch;
    qap_status vs = validate_schedule(c, s, k0, iters, &sch);
    if (vs != QAP_OK) return vs;
    if (!c->delta_valid) return fail(c, QAP_E_STATE, "Δ not initialised: call qap_delta_init");
    CU(cudaSetDevice(c->dev));
    DevState before;
    unsigned int near_before = 0;
    CU(cudaMemcpyAsync(&before, c->dst, sizeof before, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(&near_before, c->dnear_count, sizeof near_before, cudaMemcpyDeviceToHost, c->stream));

    const bool clu = use_cluster_engine(c);
    const bool tc = !clu && use_tc_engine(c);
    const bool rlb = !clu && !tc && use_relabel_engine(c);
    const bool explicit_threads = c->threads != 0;
    const int threads = tc ? TCK_NT : clu ? CLC_NT : effective_threads(c, explicit_threads ? c->threads : auto_threads(c));
    bool ds = !c->force_global && chain_smem_bytes(c, threads, true) <= c->smem_optin;
    const int smem = clu ? cl_layout(c->n, c->tb).bytes
                   : tc ? tc_layout(c->ld).bytes
                        : rlb ? rlb_layout(c->n, c->rlb_cluster).bytes
                              : chain_smem_bytes(c, threads, ds);
    if (smem > c->smem_optin) return fail(c, QAP_E_UNSUPPORTED, "chain state does not fit on chip");

    ChainArgs a;
    a.A = c->dA; a.B = c->dB; a.p = c->dp; a.best_p = c->dbest; a.D = c->dD; a.st = c->dst;
    a.rowaddr = c->drowaddr; a.qdesc = c->dqdesc; a.nqt = c->nqt;
    a.near_count = c->dnear_count; a.near_k = c->dnear_k; a.near_dec = c->dnear_dec;
    a.near_cap = QAP_NEAR_LOG_CAP;
    a.near_chain = nullptr;
    a.n = c->n; a.ld = c->ld; a.M = c->M; a.wmax = std::min(c->wmax ? c->wmax : 1024, threads);
    a.wscan = c->wmax ? c->wmax : TCK_WSCAN;
    a.k0 = k0; a.k_end = k0 + iters; a.seed = seed; a.sch = sch;

    a.theta = nullptr; a.theta_hdr = nullptr;
    a.theta_kb = a.theta_cnt = 0;
    if (tc || clu || rlb) {   // threshold buffer of one chunk of the call (theta_ring.cuh)
        const size_t need = (size_t)((std::min<uint64_t>(iters, TH_CHUNK) + TH_BLK - 1) / TH_BLK) * TH_BLK;
        if (c->theta_cap < need) {
            dfree(c, c->dtheta);
            dfree(c, c->dtheta_hdr);
            c->dtheta = nullptr;
            c->dtheta_hdr = nullptr;
            c->theta_cap = 0;
            if (dalloc(c, &c->dtheta, need * 4) != cudaSuccess ||
                dalloc(c, &c->dtheta_hdr, need / TH_BLK * sizeof(int4)) != cudaSuccess)
                return fail(c, QAP_E_NOMEM, "threshold buffer");
            c->theta_cap = need;
        }
    }
    CU(cudaEventRecord(c->ev0, c->stream));
    a.k0_dev = nullptr;
    a.proposal = c->proposal;
    a.ens = 0;
    a.dstride = 0;
    a.chain = 0u;
    a.switch_gap = (unsigned long long)c->switch_gap;
    int launches = 0;
    if (tc) {
        a.wmax = c->wmax ? c->wmax : 1024;
        // compile-time problem size for the BASELINE configurations, generic otherwise
        // random proposals (R22): the Δ engine with gathered windows, no scratch phase
        auto kern = c->proposal ? k_sa_tc<0, false, true>
                  : c->n == 100 ? k_sa_tc<100> : c->n == 50 ? k_sa_tc<50> : c->n == 12 ? k_sa_tc<12> : k_sa_tc<0>;
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        auto ks = c->n == 100 ? k_sa_scratch<100> : c->n == 50 ? k_sa_scratch<50>
                : c->n == 12 ? k_sa_scratch<12> : k_sa_scratch<0>;
        const int ssm = sc_layout(c->ld).bytes;
        CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
        bool scratch = c->use_scratch != 0 && c->proposal == 0;
        // chunks of TH_CHUNK iterations: θ of the chunk on the whole GPU, then the chain kernels
        for (uint64_t kc = k0; kc < k0 + iters; kc += TH_CHUNK) {
            const uint64_t ke = std::min<uint64_t>(k0 + iters, kc + TH_CHUNK);
            const uint64_t cnt = (ke - kc + TH_BLK - 1) / TH_BLK * TH_BLK;
            k_theta<<<c->num_sms * 8, 256, 0, c->stream>>>(sch, seed, 0u, kc, cnt, c->dtheta, c->dtheta_hdr);
            CU(cudaGetLastError());
            a.k0 = kc;
            a.k_end = ke;
            a.theta = c->dtheta;
            a.theta_hdr = c->dtheta_hdr;
            a.theta_kb = kc;
            a.theta_cnt = cnt;
            a.k0_dev = nullptr;
            launches += 2;
            if (scratch) {
                // f2: the high-acceptance phase without Δ, then Δ rebuilt at the iteration reached and
                // the Δ engine from there (device-side chaining, no host round trip)
                ks<<<1, TCS_NT, ssm, c->stream>>>(a, c->dkout);
                CU(cudaGetLastError());
                if (kc == k0) CU(cudaEventRecord(c->evm, c->stream));
                const int dt = 256, db = (c->M + dt - 1) / dt;
                k_delta_init<uint8_t, uint8_t><<<db, dt, 0, c->stream>>>((const uint8_t*)c->dA, (const uint8_t*)c->dB,
                                                                         c->dp, c->drowaddr, c->n, c->ld, c->M, c->dD);
                CU(cudaGetLastError());
                a.k0_dev = c->dkout;
                launches += 2;
            }
            kern<<<1, TCK_NT, smem, c->stream>>>(a);
            CU(cudaGetLastError());
            if (scratch && ke < k0 + iters) {    // did the scratch phase end inside this chunk?
                unsigned long long kr = 0;
                CU(cudaMemcpyAsync(&kr, c->dkout, sizeof kr, cudaMemcpyDeviceToHost, c->stream));
                CU(cudaStreamSynchronize(c->stream));
                scratch = kr >= ke;
            }
        }
    } else if (clu) {
        // chunks of TH_CHUNK iterations: thresholds of the chunk on the whole GPU, then the cluster
        auto kern = c->tb == 1 ? k_sa_cluster<uint8_t> : k_sa_cluster<uint16_t>;
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (uint64_t kc = k0; kc < k0 + iters; kc += TH_CHUNK) {
            const uint64_t ke = std::min<uint64_t>(k0 + iters, kc + TH_CHUNK);
            const uint64_t cnt = (ke - kc + TH_BLK - 1) / TH_BLK * TH_BLK;
            k_theta<<<c->num_sms * 8, 256, 0, c->stream>>>(sch, seed, 0u, kc, cnt, c->dtheta, c->dtheta_hdr);
            CU(cudaGetLastError());
            a.k0 = kc;
            a.k_end = ke;
            a.theta = c->dtheta;
            a.theta_hdr = c->dtheta_hdr;
            a.theta_kb = kc;
            a.theta_cnt = cnt;
            a.k0_dev = nullptr;
            kern<<<CLC, CLC_NT, smem, c->stream>>>(a);   // one cluster (__cluster_dims__)
            CU(cudaGetLastError());
            launches += 2;
        }
    } else if (rlb) {
        RelabelArgs ra;
        ra.c = a;
        ra.cls = c->dcls;
        ra.pt = c->dpt;
        ra.ncls = c->use_relabel == 2 ? 0 : c->ncls;
        ra.b8 = c->tb == 1;
        ra.d_out = c->dD2;
        const int CL = c->rlb_cluster;
        auto kern = CL == 8 ? (c->n == 256 ? k_sa_relabel<256, 8> : k_sa_relabel<0, 8>)
                            : (c->n == 256 ? k_sa_relabel<256, 1> : k_sa_relabel<0, 1>);
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        // exact integer thresholds of the call (theta_ring.cuh, R23), then the chain: one launch
        // per chunk of TH_CHUNK iterations, Δ~ handed over in location space between launches
        for (uint64_t kc = k0; kc < k0 + iters; kc += TH_CHUNK) {
        const uint64_t ke = std::min<uint64_t>(k0 + iters, kc + TH_CHUNK);
        const uint64_t cnt = (ke - kc + TH_BLK - 1) / TH_BLK * TH_BLK;
        k_theta<<<c->num_sms * 8, 256, 0, c->stream>>>(sch, seed, 0u, kc, cnt, c->dtheta, c->dtheta_hdr);
        CU(cudaGetLastError());
        ra.c.k0 = kc;
        ra.c.k_end = ke;
        ra.c.theta = c->dtheta;
        ra.c.theta_hdr = c->dtheta_hdr;
        ra.c.theta_kb = kc;
        ra.c.theta_cnt = cnt;
        ra.c.D = c->dD;
        ra.d_out = c->dD2;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(CL, 1, 1);
        lc.blockDim = dim3(RLB_NT, 1, 1);
        lc.dynamicSmemBytes = smem;
        lc.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        CU(cudaLaunchKernelEx(&lc, kern, ra));
        std::swap(c->dD, c->dD2);              // Δ in location space is in the second buffer
        launches += 2;
        }
    } else {
        CU(launch_chain(c, a, threads, explicit_threads, ds, smem));
    }
    CU(cudaEventRecord(c->ev1, c->stream));
    DevState after;
    unsigned int near_after = 0;
    CU(cudaMemcpyAsync(&after, c->dst, sizeof after, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(&near_after, c->dnear_count, sizeof near_after, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    c->last_scratch_ms = 0.f;
    c->last_scratch[0] = c->last_scratch[1] = 0;
    if (tc && c->use_scratch && c->proposal == 0) {
        CU(cudaEventElapsedTime(&c->last_scratch_ms, c->ev0, c->evm));
        CU(cudaMemcpy(c->last_scratch, c->dkout, sizeof c->last_scratch, cudaMemcpyDeviceToHost));
    }
    c->last_launches = (tc || clu || rlb) ? launches : 1;
    if (out) {
        out->iterations = iters;
        out->accepted = after.accepted - before.accepted;
        out->near_ties = near_after - near_before;
        out->cost = after.cost;
        out->best_cost = after.best_cost;
        out->digest = after.digest;
    }
    return QAP_OK;
}

qap_status qap_cost(qap_ctx* c, const int32_t* perm, int64_t* out) {
    CHECK_CTX(c);
    if (!out) return fail(c, QAP_E_INVALID_ARG, "out is NULL");
    if (perm && !is_perm(c->n, perm)) return fail(c, QAP_E_DIMENSION, "perm is not a permutation");
    CU(cudaSetDevice(c->dev));
    const int32_t* src = c->dp;
    if (perm) {
        CU(cudaMemcpyAsync(c->dperm, perm, c->n * 4, cudaMemcpyHostToDevice, c->stream));
        src = c->dperm;
    }
    if (c->ta == 1 && c->tb == 1)
        k_cost<uint8_t, uint8_t><<<1, 512, 0, c->stream>>>((const uint8_t*)c->dA, (const uint8_t*)c->dB, src, c->n, c->ld, c->dscratch);
    else if (c->ta == 1)
        k_cost<uint8_t, uint16_t><<<1, 512, 0, c->stream>>>((const uint8_t*)c->dA, (const uint16_t*)c->dB, src, c->n, c->ld, c->dscratch);
    else if (c->tb == 1)
        k_cost<uint16_t, uint8_t><<<1, 512, 0, c->stream>>>((const uint16_t*)c->dA, (const uint8_t*)c->dB, src, c->n, c->ld, c->dscratch);
    else
        k_cost<uint16_t, uint16_t><<<1, 512, 0, c->stream>>>((const uint16_t*)c->dA, (const uint16_t*)c->dB, src, c->n, c->ld, c->dscratch);
    CU(cudaGetLastError());
    long long v = 0;
    CU(cudaMemcpyAsync(&v, c->dscratch, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *out = v;
    c->last_launches = 1;
    return QAP_OK;
}

qap_status qap_get_state(qap_ctx* c, int32_t* perm, int32_t* best_perm, int32_t* delta) {
    CHECK_CTX(c);
    if (delta && !c->delta_valid) return fail(c, QAP_E_STATE, "Δ not initialised");
    CU(cudaSetDevice(c->dev));
    if (perm) CU(cudaMemcpyAsync(perm, c->dp, c->n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (best_perm) CU(cudaMemcpyAsync(best_perm, c->dbest, c->n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (delta) {
        k_unpad<<<(c->M + 255) / 256, 256, 0, c->stream>>>(c->dD, c->drowaddr, c->n, c->M, c->dDlin);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(delta, c->dDlin, (size_t)c->M * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CU(cudaStreamSynchronize(c->stream));
    c->last_launches = 0;
    return QAP_OK;
}

qap_status qap_get_near_ties(qap_ctx* c, uint64_t* ks, uint8_t* decisions, int32_t cap, int32_t* count) {
    CHECK_CTX(c);
    if (cap < 0 || !count || (cap > 0 && (!ks || !decisions)))
        return fail(c, QAP_E_INVALID_ARG, "bad near-tie buffers");
    CU(cudaSetDevice(c->dev));
    unsigned int cnt = 0;
    CU(cudaMemcpyAsync(&cnt, c->dnear_count, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    int m = std::min<int>(std::min<unsigned>(cnt, QAP_NEAR_LOG_CAP), cap);
    if (m > 0) {
        CU(cudaMemcpyAsync(ks, c->dnear_k, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(decisions, c->dnear_dec, m, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    *count = (int32_t)cnt;
    return QAP_OK;
}

qap_status qap_schedule_bounds(qap_ctx* c, double* t0, double* tf) {
    CHECK_CTX(c);
    if (!t0 || !tf) return fail(c, QAP_E_INVALID_ARG, "NULL output");
    if (!c->delta_valid) return fail(c, QAP_E_STATE, "Δ not initialised");
    CU(cudaSetDevice(c->dev));
    k_unpad<<<(c->M + 255) / 256, 256, 0, c->stream>>>(c->dD, c->drowaddr, c->n, c->M, c->dDlin);
    k_delta_bounds<<<1, 1024, 0, c->stream>>>(c->dDlin, c->M, reinterpret_cast<int*>(c->dscratch));
    CU(cudaGetLastError());
    int mm[2];
    CU(cudaMemcpyAsync(mm, c->dscratch, sizeof mm, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (mm[1] == 0) {
        *t0 = 1.0;
        *tf = 0.1;
    } else {  // R2
        *t0 = (double)mm[0] + ((double)mm[1] - (double)mm[0]) / 10.0;
        *tf = (double)mm[0];
    }
    c->last_launches = 1;
    return QAP_OK;
}

}  // extern "C"

template <typename TA, typename TB, int NT, int NFIX>
static cudaError_t launch_ens_t(qap_ctx* c, const EnsArgs& a, int groups, int smem) {
    auto kern = k_ensemble<TA, TB, NT, NFIX>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int blocks = std::min(c->num_sms, (a.count + groups - 1) / groups);
    kern<<<blocks, NT * groups, smem, c->stream>>>(a);
    return cudaGetLastError();
}

static cudaError_t launch_ens(qap_ctx* c, const EnsArgs& a, int nt, int groups, int smem) {
    if (c->ta == 1 && c->tb == 1) {
        if (nt == 128 && c->n == 100) return launch_ens_t<uint8_t, uint8_t, 128, 100>(c, a, groups, smem);
        if (nt == 256) return launch_ens_t<uint8_t, uint8_t, 256, 0>(c, a, groups, smem);
        if (nt == 64) return launch_ens_t<uint8_t, uint8_t, 64, 0>(c, a, groups, smem);
        return launch_ens_t<uint8_t, uint8_t, 128, 0>(c, a, groups, smem);
    }
    if (c->ta == 1) return launch_ens_t<uint8_t, uint16_t, 128, 0>(c, a, groups, smem);
    if (c->tb == 1) return launch_ens_t<uint16_t, uint8_t, 128, 0>(c, a, groups, smem);
    return launch_ens_t<uint16_t, uint16_t, 128, 0>(c, a, groups, smem);
}

// Ensemble on the tensor-memory engine: one CTA per chain, the single-chain kernels launched over
// all chains at once -- the scratch phase (two chains per SM: 256 TMEM columns each), the Δ
// rebuild of every chain, the Δ engine (one chain per SM) -- then the per-chain results and the
// argmin.
static qap_status ensemble_tc(qap_ctx* c, uint32_t chain_begin, uint32_t chain_count, const int32_t* p0s,
                              uint64_t iters, const Sched& sch, uint64_t seed, int64_t* best_cost,
                              uint32_t* best_chain, int32_t* best_perm, qap_stats* sum_stats,
                              qap_chain_result* per_chain) {
    const int n = c->n;
    const int dstride = c->nqt * 4 + 4;
    CU(cudaSetDevice(c->dev));
    if (c->ens_cap < chain_count) {
        dfree(c, c->ens_p0);
        dfree(c, c->ens_res);
        dfree(c, c->ens_best);
        c->ens_p0 = nullptr; c->ens_res = nullptr; c->ens_best = nullptr; c->ens_cap = 0;
        if (dalloc(c, &c->ens_p0, (size_t)chain_count * n * 4) != cudaSuccess ||
            dalloc(c, &c->ens_res, (size_t)chain_count * sizeof(ChainResult)) != cudaSuccess ||
            dalloc(c, &c->ens_best, (size_t)chain_count * n * 2) != cudaSuccess)
            return fail(c, QAP_E_NOMEM, "ensemble buffers");
        c->ens_cap = chain_count;
    }
    if (c->tcap < chain_count) {
        void* ptrs[] = {c->tp, c->tbp, c->tD, c->tst, c->tkout};
        for (void* q : ptrs) dfree(c, q);
        c->tp = c->tbp = c->tD = nullptr; c->tst = nullptr; c->tkout = nullptr; c->tcap = 0;
        if (dalloc(c, &c->tp, (size_t)chain_count * n * 4) != cudaSuccess ||
            dalloc(c, &c->tbp, (size_t)chain_count * n * 4) != cudaSuccess ||
            dalloc(c, &c->tD, (size_t)chain_count * dstride * 4) != cudaSuccess ||
            dalloc(c, &c->tst, (size_t)chain_count * sizeof(DevState)) != cudaSuccess ||
            dalloc(c, &c->tkout, (size_t)chain_count * 2 * sizeof(unsigned long long)) != cudaSuccess)
            return fail(c, QAP_E_NOMEM, "tensor-memory ensemble buffers");
        c->tcap = chain_count;
    }
    if (p0s) CU(cudaMemcpyAsync(c->ens_p0, p0s, (size_t)chain_count * n * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemsetAsync(c->ens_near_count, 0, sizeof(unsigned int), c->stream));
    ChainArgs a;
    a.A = c->dA; a.B = c->dB; a.p = c->tp; a.best_p = c->tbp; a.D = c->tD; a.st = c->tst;
    a.rowaddr = c->drowaddr; a.qdesc = c->dqdesc; a.nqt = c->nqt;
    a.near_count = c->ens_near_count; a.near_k = c->ens_near_k; a.near_dec = c->ens_near_dec;
    a.near_chain = c->ens_near_chain; a.near_cap = QAP_ENS_NEAR_LOG_CAP;
    a.n = n; a.ld = c->ld; a.M = c->M; a.wmax = c->wmax ? c->wmax : 1024;
    a.wscan = c->wmax ? c->wmax : TCK_WSCAN;
    a.k0 = 0; a.k_end = iters; a.seed = seed; a.sch = sch;
    a.k0_dev = nullptr; a.proposal = 0;
    a.ens = 1; a.dstride = dstride; a.chain = chain_begin;
    a.theta = nullptr; a.theta_hdr = nullptr; a.theta_kb = a.theta_cnt = 0;
    // two scratch-phase chains share an SM but the Δ engine holds one: stay longer in the scratch
    // phase (config 5: gap 4096 / 16384 / 65536 / never = 3.67 / 3.64 / 3.62 / 3.66 s)
    a.switch_gap = c->switch_gap ? (unsigned long long)c->switch_gap : 65536ull;
    CU(cudaEventRecord(c->ev0, c->stream));
    if (!p0s) {                                  // chain-keyed start permutations on the device (R14b)
        k_start_perms<<<(chain_count + 127) / 128, 128, 0, c->stream>>>(n, seed, chain_begin, (int)chain_count, c->ens_p0);
        CU(cudaGetLastError());
    }
    k_reset<uint8_t, uint8_t><<<chain_count, 512, 0, c->stream>>>((const uint8_t*)c->dA, (const uint8_t*)c->dB,
                                                                   c->ens_p0, n, c->ld, c->tp, c->tbp, c->tst);
    CU(cudaGetLastError());
    if (c->ens4 && e4_eligible(n)) {
        // scratch phase four chains per SM (ens_chain.cuh): 128 TMEM columns and 160 threads per
        // chain; more than a fifth of the shared memory per CTA caps an SM at the four chains
        // whose 4 x 128 TMEM columns fill its 512
        auto ks = n == 100 ? k_ens_scratch<100> : n == 50 ? k_ens_scratch<50> : n == 12 ? k_ens_scratch<12>
                                                                                           : k_ens_scratch<0>;
        const int ssm = std::max(e4_layout(n, c->ld).bytes, c->smem_optin / 5 + 1024);
        CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
        ks<<<chain_count, E4_NT, ssm, c->stream>>>(a, c->tkout);
    } else {
    auto ks = n == 100 ? k_sa_scratch<100, true> : n == 50 ? k_sa_scratch<50, true>
            : n == 12 ? k_sa_scratch<12, true> : k_sa_scratch<0, true>;
    // more than a third of the shared memory: at most two chains' CTAs per SM, whose 2 x 256 TMEM
    // columns fill the SM's 512
    const int ssm = std::max(sc_layout(c->ld).bytes, c->smem_optin / 3 + 1024);
    CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    ks<<<chain_count, tcs_nt<true>(), ssm, c->stream>>>(a, c->tkout);
    }
    CU(cudaGetLastError());
    const int dt = 256, db = (c->M + dt - 1) / dt;
    for (uint32_t c0 = 0; c0 < chain_count; c0 += 65535u) {   // gridDim.y <= 65535: slices of chains
        const uint32_t cs = std::min<uint32_t>(65535u, chain_count - c0);
        k_delta_init<uint8_t, uint8_t><<<dim3(db, cs), dt, 0, c->stream>>>(
            (const uint8_t*)c->dA, (const uint8_t*)c->dB, c->tp + (size_t)c0 * n, c->drowaddr, n, c->ld, c->M,
            c->tD + (size_t)c0 * dstride, dstride);
        CU(cudaGetLastError());
    }
    a.k0_dev = c->tkout;
    auto kern = n == 100 ? k_sa_tc<100, true> : n == 50 ? k_sa_tc<50, true> : n == 12 ? k_sa_tc<12, true>
              : k_sa_tc<0, true>;
    const int tsm = tc_layout(c->ld).bytes;
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm));
    kern<<<chain_count, TCK_NT, tsm, c->stream>>>(a);
    CU(cudaGetLastError());
    CU(cudaEventRecord(c->ev1, c->stream));
    k_ens_collect<<<std::min<int>(1024, (chain_count * n + 255) / 256), 256, 0, c->stream>>>(
        c->tst, c->tbp, (int)chain_count, n, iters, c->ens_res, c->ens_best);
    CU(cudaGetLastError());
    k_ens_reduce<<<1, 1024, 0, c->stream>>>(c->ens_res, (int)chain_count, c->dscratch);
    CU(cudaGetLastError());
    long long red[8];
    CU(cudaMemcpyAsync(red, c->dscratch, sizeof red, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const int bi = (int)red[1];
    std::vector<uint16_t> bp(n);
    CU(cudaMemcpy(bp.data(), c->ens_best + (size_t)bi * n, n * 2, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) best_perm[i] = bp[i];
    *best_cost = red[0];
    *best_chain = chain_begin + (uint32_t)bi;
    if (sum_stats) {
        sum_stats->iterations = iters * (uint64_t)chain_count;
        sum_stats->accepted = (uint64_t)red[2];
        sum_stats->near_ties = (uint64_t)red[3];
        sum_stats->digest = (uint64_t)red[4];
        sum_stats->cost = red[5];
        sum_stats->best_cost = red[0];
    }
    if (per_chain)
        CU(cudaMemcpy(per_chain, c->ens_res, (size_t)chain_count * sizeof(ChainResult), cudaMemcpyDeviceToHost));
    CU(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    c->last_launches = 4 + (p0s ? 0 : 1) + (int)((chain_count - 1) / 65535u);
    return QAP_OK;
}

extern "C" {

qap_status qap_ensemble_run(qap_ctx* c, uint32_t chain_begin, uint32_t chain_count, const int32_t* p0s,
                            uint64_t iters, const qap_schedule* s, uint64_t seed, int64_t* best_cost,
                            uint32_t* best_chain, int32_t* best_perm, qap_stats* sum_stats,
                            qap_chain_result* per_chain) {
    CHECK_CTX(c);
    if (!best_cost || !best_chain || !best_perm) return fail(c, QAP_E_INVALID_ARG, "NULL argument");
    if (chain_count == 0 || iters == 0) return fail(c, QAP_E_INVALID_ARG, "chain_count or iters is 0");
    Sched sch;
    qap_status vs = validate_schedule(c, s, 0, iters, &sch);
    if (vs != QAP_OK) return vs;
    const int n = c->n;
    if (p0s)
        for (uint32_t i = 0; i < chain_count; ++i)
            if (!is_perm(n, p0s + (size_t)i * n)) return fail(c, QAP_E_DIMENSION, "a start permutation is invalid");
    if (use_tc_ensemble(c))
        return ensemble_tc(c, chain_begin, chain_count, p0s, iters, sch, seed, best_cost, best_chain,
                           best_perm, sum_stats, per_chain);
    const int nt = (c->ta == 1 && c->tb == 1) ? c->ens_group : 128;
    const GroupLayout L = group_layout(n, c->ld, c->nqt, c->tb, nt / 32, true, dab_bytes(c));
    const int a_bytes = cta_prefix_bytes(n, c->ld, c->ta, c->nqt);
    // each group uses 2 of the 16 hardware named barriers (ids 1+2g, 2+2g; id 0 is the CTA's)
    int groups = std::min(std::min((c->smem_optin - a_bytes) / L.bytes, 1024 / nt), 7);
    if (groups < 1) return fail(c, QAP_E_UNSUPPORTED, "one ensemble chain does not fit on chip");
    const int smem = a_bytes + groups * L.bytes;
    CU(cudaSetDevice(c->dev));
    if (c->ens_cap < chain_count) {
        dfree(c, c->ens_p0);
        dfree(c, c->ens_res);
        dfree(c, c->ens_best);
        c->ens_p0 = nullptr; c->ens_res = nullptr; c->ens_best = nullptr; c->ens_cap = 0;
        if (dalloc(c, &c->ens_p0, (size_t)chain_count * n * 4) != cudaSuccess ||
            dalloc(c, &c->ens_res, (size_t)chain_count * sizeof(ChainResult)) != cudaSuccess ||
            dalloc(c, &c->ens_best, (size_t)chain_count * n * 2) != cudaSuccess)
            return fail(c, QAP_E_NOMEM, "ensemble buffers");
        c->ens_cap = chain_count;
    }
    if (!c->ens_counter) CU(dalloc(c, &c->ens_counter, sizeof(unsigned int)));
    if (p0s) CU(cudaMemcpyAsync(c->ens_p0, p0s, (size_t)chain_count * n * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemsetAsync(c->ens_counter, 0, sizeof(unsigned int), c->stream));
    CU(cudaMemsetAsync(c->ens_near_count, 0, sizeof(unsigned int), c->stream));
    EnsArgs a;
    a.A = c->dA; a.B = c->dB; a.p0s = c->ens_p0; a.res = c->ens_res; a.best_perms = c->ens_best;
    a.next_chain = c->ens_counter; a.count = (int)chain_count; a.n = n; a.ld = c->ld; a.M = c->M;
    a.rowaddr = c->drowaddr; a.qdesc = c->dqdesc; a.nqt = c->nqt;
    a.proposal = c->proposal;
    a.wmax = std::min(c->wmax ? c->wmax : 1024, nt); a.chain_begin = chain_begin; a.iters = iters; a.seed = seed; a.sch = sch;
    a.near_count = c->ens_near_count; a.near_k = c->ens_near_k; a.near_dec = c->ens_near_dec;
    a.near_chain = c->ens_near_chain; a.near_cap = QAP_ENS_NEAR_LOG_CAP;
    CU(cudaEventRecord(c->ev0, c->stream));
    if (!p0s) {                                  // chain-keyed start permutations on the device (R14b)
        k_start_perms<<<(chain_count + 127) / 128, 128, 0, c->stream>>>(n, seed, chain_begin, (int)chain_count, c->ens_p0);
        CU(cudaGetLastError());
    }
    CU(launch_ens(c, a, nt, groups, smem));
    CU(cudaEventRecord(c->ev1, c->stream));
    k_ens_reduce<<<1, 1024, 0, c->stream>>>(c->ens_res, (int)chain_count, c->dscratch);
    CU(cudaGetLastError());
    long long red[8];
    CU(cudaMemcpyAsync(red, c->dscratch, sizeof red, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const int bi = (int)red[1];
    std::vector<uint16_t> bp(n);
    CU(cudaMemcpy(bp.data(), c->ens_best + (size_t)bi * n, n * 2, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) best_perm[i] = bp[i];
    *best_cost = red[0];
    *best_chain = chain_begin + (uint32_t)bi;
    if (sum_stats) {
        sum_stats->iterations = iters * (uint64_t)chain_count;
        sum_stats->accepted = (uint64_t)red[2];
        sum_stats->near_ties = (uint64_t)red[3];
        sum_stats->digest = (uint64_t)red[4];
        sum_stats->cost = red[5];
        sum_stats->best_cost = red[0];
    }
    if (per_chain) {
        static_assert(sizeof(ChainResult) == sizeof(qap_chain_result), "layout");
        CU(cudaMemcpy(per_chain, c->ens_res, (size_t)chain_count * sizeof(ChainResult), cudaMemcpyDeviceToHost));
    }
    CU(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    c->last_launches = 2 + (p0s ? 0 : 1);
    return QAP_OK;
}

qap_status qap_ensemble_near_ties(qap_ctx* c, uint32_t* chains, uint64_t* ks, uint8_t* decisions, int32_t cap,
                                  int32_t* count) {
    CHECK_CTX(c);
    if (cap < 0 || !count || (cap > 0 && (!chains || !ks || !decisions)))
        return fail(c, QAP_E_INVALID_ARG, "bad near-tie buffers");
    CU(cudaSetDevice(c->dev));
    unsigned int cnt = 0;
    CU(cudaMemcpyAsync(&cnt, c->ens_near_count, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const int m = std::min<int>(std::min<unsigned>(cnt, QAP_ENS_NEAR_LOG_CAP), cap);
    if (m > 0) {
        CU(cudaMemcpyAsync(chains, c->ens_near_chain, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(ks, c->ens_near_k, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(decisions, c->ens_near_dec, m, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    *count = (int32_t)cnt;
    return QAP_OK;
}

qap_status qap_start_perms(qap_ctx* c, uint64_t seed, uint32_t chain_begin, uint32_t count, int32_t* out) {
    CHECK_CTX(c);
    if (!out || count == 0) return fail(c, QAP_E_INVALID_ARG, "out is NULL or count is 0");
    CU(cudaSetDevice(c->dev));
    int32_t* d = nullptr;
    CU(dalloc(c, &d, (size_t)count * c->n * 4));
    k_start_perms<<<(count + 127) / 128, 128, 0, c->stream>>>(c->n, seed, chain_begin, (int)count, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, (size_t)count * c->n * 4, cudaMemcpyDeviceToHost, c->stream);
    dfree(c, d);
    CU(e);
    CU(cudaStreamSynchronize(c->stream));
    c->last_launches = 1;
    return QAP_OK;
}

#ifdef QAPSA_PHASE_TIMERS
// debug build only (not part of include/qapsa.h): read-and-clear the phase cycle counters
int qapsa_debug_phase_cycles(unsigned long long* out8) {
    if (cudaMemcpyFromSymbol(out8, g_phase_cycles, 128 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    unsigned long long z[128] = {0};
    return cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z) != cudaSuccess;
}
#endif

qap_status qap_set_option(qap_ctx* c, int32_t key, int64_t value) {
    CHECK_CTX(c);
    switch (key) {
        case QAP_OPT_WINDOW_MAX:
            if (value < 32 || value > 8192 || (value & 31)) return fail(c, QAP_E_INVALID_ARG, "window must be a multiple of 32 in [32,8192]");
            c->wmax = (int)value;
            return QAP_OK;
        case QAP_OPT_THREADS:
            if (value != 0 && value != 64 && value != 128 && value != 256 && value != 512 && value != 1024)
                return fail(c, QAP_E_INVALID_ARG, "threads must be 0 (auto), 64, 128, 256, 512 or 1024");
            c->threads = (int)value;
            return QAP_OK;
        case QAP_OPT_FORCE_GLOBAL_DELTA:
            c->force_global = value ? 1 : 0;
            return QAP_OK;
        case QAP_OPT_TENSOR_CORE:
            if (value < 0 || value > 2) return fail(c, QAP_E_INVALID_ARG, "tensor core must be 0, 1 or 2");
            c->use_tc = (int)value;
            return QAP_OK;
        case QAP_OPT_SCRATCH_PHASE:
            c->use_scratch = value ? 1 : 0;
            return QAP_OK;
        case QAP_OPT_RELABEL:
            if (value < 0 || value > 3) return fail(c, QAP_E_INVALID_ARG, "relabel must be 0, 1, 2 or 3");
            c->use_relabel = (int)value;
            return QAP_OK;
        case QAP_OPT_PROPOSAL:
            if (value != 0 && value != 1) return fail(c, QAP_E_INVALID_ARG, "proposal must be 0 or 1");
            c->proposal = (int)value;
            return QAP_OK;
        case QAP_OPT_SWITCH_GAP:
            if (value < 0 || value > 0x7FFFFFFFll) return fail(c, QAP_E_INVALID_ARG, "switch gap must be in [0, 2^31)");
            c->switch_gap = value;
            return QAP_OK;
        case QAP_OPT_ENSEMBLE_SCRATCH4:
            if (value != 0 && value != 1) return fail(c, QAP_E_INVALID_ARG, "value must be 0 or 1");
            c->ens4 = (int)value;
            return QAP_OK;
        case QAP_OPT_CLUSTER_ENGINE:
            if (value < 0 || value > 2) return fail(c, QAP_E_INVALID_ARG, "cluster engine must be 0, 1 or 2");
            c->use_cluster = (int)value;
            return QAP_OK;
        case QAP_OPT_RELABEL_CLUSTER:
            if (value != 1 && value != 8) return fail(c, QAP_E_INVALID_ARG, "relabel cluster must be 1 or 8");
            c->rlb_cluster = (int)value;
            return QAP_OK;
        case QAP_OPT_ENSEMBLE_GROUP:
            if (value != 64 && value != 128 && value != 256) return fail(c, QAP_E_INVALID_ARG, "group must be 64, 128 or 256");
            c->ens_group = (int)value;
            return QAP_OK;
    }
    return fail(c, QAP_E_INVALID_ARG, "unknown option");
}

int32_t qap_uses_tensor_core(const qap_ctx* c) { return (c && use_tc_engine(c)) ? 1 : 0; }

int32_t qap_engine(const qap_ctx* c) {
    if (!c) return -1;
    if (use_cluster_engine(c)) return QAP_ENGINE_CLUSTER;
    if (use_tc_engine(c)) return QAP_ENGINE_TENSOR_MEMORY;
    if (use_relabel_engine(c)) return QAP_ENGINE_RELABEL;
    return QAP_ENGINE_SHARED_MEMORY;
}

qap_status qap_last_scratch_time(qap_ctx* c, float* ms, uint64_t* k_reached, uint64_t* accepted) {
    CHECK_CTX(c);
    if (ms) *ms = c->last_scratch_ms;
    if (k_reached) *k_reached = c->last_scratch[0];
    if (accepted) *accepted = c->last_scratch[1];
    return QAP_OK;
}

qap_status qap_last_kernel_time(qap_ctx* c, float* ms, int32_t* launches) {
    CHECK_CTX(c);
    if (ms) *ms = c->last_ms;
    if (launches) *launches = c->last_launches;
    return QAP_OK;
}

}  // extern "C"
