// engine.cu -- traversal state, level driver, bfs_full / adaptive loops and
// the C ABI of include/abfs.h (except graph construction, see graph.cu).
//
// Per level: [optional prepare from caller depths] ->
// [optional queue<->bitmap conversion] -> one strategy kernel (two for
// push-warp: warp pass + CTA heavy pass) -> one 64-byte counter readback.
// Host decides the next (kernel, variant) from the reference's float64
// features and the FlatTree (adaptive.py:101-129).

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "launch.cuh"
#include "megakernel.cuh"

namespace abfs {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

static uint64_t host_ns() {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace abfs

using namespace abfs;

struct abfs_traversal {
    // per-handle lock: calls on one traversal are serialised,
    // distinct traversals of one graph run concurrently;
    // recursive because entry points call each other (run_level -> load/read)
    mutable std::recursive_mutex mu;
    abfs_graph *g = nullptr;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int32_t *depth = nullptr;
    uint32_t *visited = nullptr;
    uint32_t *noin = nullptr;  // in-degree-0 bitmap (static)
    uint32_t *fbm[2] = {nullptr, nullptr};
    uint32_t *q[2] = {nullptr, nullptr};
    uint2 *units = nullptr;
    Ctr *dctr = nullptr;
    Ctr *hctr = nullptr;       // pinned
    Mailbox *mb = nullptr;     // host-mapped level results
    Mailbox *dmb = nullptr;    // device view of mb
    uint64_t words = 0;
    int cur = 0;
    bool has_q = false, has_bm = false;
    uint64_t F = 0;            // current frontier size (host-known)
    int64_t expect_level = -1; // level whose frontier the state holds; -1 = rebuild
    uint64_t call = 0;
    bool inconsistent = false;
    std::vector<cudaEvent_t> ev;  // 2 per level of the current traversal
    cudaEvent_t et0 = nullptr;
    uint64_t last_trav_ns = 0;
    uint64_t launches = 0;     // kernels launched by this traversal
    unsigned long long *des = nullptr;   // pull scanned-edge counter (instrumented)
    bool instrument = false;
    std::vector<uint64_t> es_log;        // per level (instrumented runs)
    // device-resident loop (megakernel)
    bool use_mega = true;
    MegaRecord *mrecs = nullptr;         // host-mapped level records (written by the kernel)
    MegaRecord *drecs = nullptr;         // device view of mrecs
    std::vector<MegaRecord> hrecs;
    unsigned long long *mnlev = nullptr, *dnlev = nullptr;   // host-mapped level counts (per root)
    uint32_t *hroots = nullptr, *droots = nullptr;            // batch roots (pinned / device)
    unsigned long long *dsums = nullptr;                     // per-root depth checksums (device)
    uint32_t *acc = nullptr;                                 // RED-mode candidate bits [words], all-zero between levels
    uint32_t *pl = nullptr;                                  // list-based pull: 3 x [n] candidate lists
    std::vector<unsigned char> last_blob;                    // tree blob resident on the device
    std::vector<unsigned long long> batch_levels;            // per-root level counts, last launch
    size_t batch_recs = 0;                                   // records kept in mrecs, last launch
    unsigned char *dtree = nullptr, *htree = nullptr;   // device / pinned staging blob
    size_t tree_cap = 0;
    uint64_t max_out_degree = 0;   // decides the megakernel's cluster solo mode
    uint64_t n_noin = 0;           // vertices of in-degree 0 (sparse-pull estimate)
    int mega_grid = 0;
    int mega_cluster = 0;       // cluster size of the megakernel launch (0: plain cooperative)
    int solo_req = 0;           // cluster size asked for when mega_grid was sized (ABFS_SOLO_CLUSTER)
    int grid_div = 1;           // batch sub-traversal: 1/grid_div of the co-resident grid
    int batch_ways_req = 0;     // abfs_traversal_set_batch_ways (0: automatic)
    bool is_sub = false;        // owned by a parent's split batch (the parent holds the device lock)
    abfs_traversal *sub[kMaxSplit] = {};   // split batch: concurrent half-grid traversals
    SoloState *dsolo = nullptr; // solo-mode hand-off (device)
    int mega_minb = kMegaMinB;  // resident CTAs per SM the megakernel is compiled for
    void *mega_kfn = nullptr;   // the megakernel instantiation mega_grid was sized for
    char *stage = nullptr;                     // pinned D2H staging (2 chunks)
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
};

#define ABFS_LOCK(t) std::lock_guard<std::recursive_mutex> _abfs_guard((t)->mu)

// Cooperative megakernels of one device run one at a time: two persistent
// grids sharing the SMs could each be partly resident and wait at a grid
// barrier for blocks that never get scheduled.
static std::mutex g_mega_mu[64];
namespace abfs {
std::mutex &mega_mutex(int device) { return g_mega_mu[device & 63]; }
}  // namespace abfs

extern "C" const char *abfs_last_error(void) { return g_err.c_str(); }
extern "C" int abfs_version(void) { return 1; }

// Pull phase-A depth (tunable for experiments via ABFS_PULL_LIGHT).
static uint32_t pull_light() {
    static uint32_t v = 0;
    if (!v) {
        const char *e = getenv("ABFS_PULL_LIGHT");
        v = e ? (uint32_t)atoi(e) : kPullLight;
        if (v < 1) v = 1;
    }
    return v;
}

// Unsigned tuning knob from the environment (read per call: tests toggle it).
static uint64_t env_u64(const char *name, uint64_t dflt) {
    const char *e = getenv(name);
    return (e && *e) ? (uint64_t)strtoull(e, nullptr, 10) : dflt;
}

// Push-warp's virtual-warp width.  The reference's chunk size is a schedule
// parameter (depths and counts do not depend on it, kernels.py:303-322), so
// the width is fitted to the degree distribution: on a graph without a
// heavy tail (max out-degree <= 4 x mean: uniform-random, meshes) a vertex's
// adjacency is covered by 4 strides of mean/8 lanes (ER-32M: 4-lane warps,
// its 18.6 M-discovery level 724 -> 617 us; mesh: 1 lane, as push); skewed
// graphs keep warps of min(chunk, 32, max degree) lanes (Kronecker-24 is
// 1-8 % slower with narrower warps).  ABFS_VW_MAX caps it for experiments.
static int64_t vw_chunk(const abfs_traversal *t, int64_t chunk) {
    const uint64_t n = t->g->d.n ? t->g->d.n : 1, mean = t->g->d.m / n;
    int64_t w = 1;
    if (t->max_out_degree <= 4 * (mean ? mean : 1)) {
        while (w * 2 <= (int64_t)(mean / 8) && w < 32) w <<= 1;
    } else {
        while (w < (int64_t)t->max_out_degree && w < 32) w <<= 1;
    }
    const int64_t cap = (int64_t)env_u64("ABFS_VW_MAX", 32);
    if (w > cap) w = cap;
    if (const uint64_t f = env_u64("ABFS_VW_FORCE", 0)) w = (int64_t)f;   // A/B experiments
    return chunk < w ? chunk : w;
}

// One level's strategy launch over a StratArgs view (launch.cuh).
template <int VAR>
static void launch_strategy(abfs_traversal *t, const LevelCtx &c, int kernel, int64_t chunk) {
    const DevGraph &g = t->g->d;
    StratArgs a;
    a.out_off = g.out_off;
    a.dst = g.dst;
    a.org = g.org;
    a.m_fwd = g.m;
    a.in_off = g.in_off;
    a.src = g.src;
    a.rev_owner = g.rev_owner;
    a.m_rev = g.m;
    a.first_src = g.first_src;
    a.noin = t->noin;
    a.fbm_next = t->fbm[t->cur ^ 1];
    a.word0 = 0;
    a.word_end = t->words;
    a.q = t->q[t->cur];
    a.F = (uint32_t)t->F;
    t->launches += launch_strategy_args<VAR>(c, a, kernel, vw_chunk(t, chunk), t->stream);
}

static int ensure_events(abfs_traversal *t, size_t n) {
    while (t->ev.size() < n) {
        cudaEvent_t e;
        ABFS_CUDA(cudaEventCreate(&e));
        t->ev.push_back(e);
    }
    return ABFS_OK;
}

// Wait for the level's mailbox stamp; poll the stream for faults.
static int wait_mailbox(abfs_traversal *t, unsigned long long seq) {
    volatile Mailbox *mb = t->mb;
    for (uint64_t spin = 1;; ++spin) {
        if (mb->seq == seq) return ABFS_OK;
        if ((spin & 4095) == 0) {
            cudaError_t e = cudaStreamQuery(t->stream);
            if (e == cudaSuccess) {
                if (mb->seq == seq) return ABFS_OK;
                return fail(ABFS_ECUDA, "level completed without publishing its count");
            }
            if (e != cudaErrorNotReady)
                return fail(ABFS_ECUDA, std::string("level kernel failed: ") + cudaGetErrorString(e));
        }
    }
}

// One level on the device-resident state.  ev_slot selects the event pair
// bracketing the level; elapsed_ns is filled only when `timed_now` (else the
// caller reads the events after the traversal).
static int level_impl(abfs_traversal *t, int64_t level, int kernel, int variant, int64_t chunk,
                      uint64_t *new_count, size_t ev_slot, bool timed_now, uint64_t *elapsed_ns,
                      int *converted) {
    ABFS_TRY(level_params_ok(level, kernel, variant, chunk));
    ABFS_CUDA(cudaSetDevice(t->device));
    ABFS_TRY(ensure_events(t, 2 * ev_slot + 2));
    const DevGraph &g = t->g->d;
    cudaStream_t s = t->stream;
    int conv = 0;
    ABFS_CUDA(cudaEventRecord(t->ev[2 * ev_slot], s));
    if (t->expect_level != level) {
        // Frontier unknown for this level: rebuild from the depth array.
        ABFS_CUDA(cudaMemsetAsync(&t->dctr->inconsistent, 0, sizeof(unsigned), s));
        ABFS_CUDA(cudaMemsetAsync(&t->dctr->fcount, 0, sizeof(unsigned long long), s));
        k_prepare<<<grid_for(t->words, kBlock / 32, 148 * 512), kBlock, 0, s>>>(
            t->depth, g.n, t->words, (int32_t)level, t->fbm[t->cur], t->visited, t->dctr);
        t->launches += 1;
        ABFS_CUDA(cudaGetLastError());
        ABFS_CUDA(cudaMemcpyAsync(t->hctr, t->dctr, sizeof(Ctr), cudaMemcpyDeviceToHost, s));
        ABFS_CUDA(cudaStreamSynchronize(s));
        t->F = t->hctr->fcount;
        t->inconsistent = t->hctr->inconsistent != 0;
        t->has_bm = true;
        t->has_q = false;
        t->expect_level = level;
        conv = 1;
    }
    const bool need_queue = (kernel == ABFS_VERTEX_PUSH || kernel == ABFS_VERTEX_PUSH_WARP);
    if (need_queue && !t->has_q) {
        k_bitmap_to_queue<<<grid_for(t->words, kBlock, 1ull << 31), kBlock, 0, s>>>(
            t->fbm[t->cur], t->words, t->q[t->cur], &t->dctr->cq);
        t->launches += 1;
        t->has_q = true;
        conv = 1;
    } else if (!need_queue && !t->has_bm) {
        ABFS_CUDA(cudaMemsetAsync(t->fbm[t->cur], 0, t->words * 4, s));
        if (t->F) {
            k_queue_to_bitmap<<<grid_for(t->F, kBlock, 148 * 16), kBlock, 0, s>>>(
                t->q[t->cur], (uint32_t)t->F, t->fbm[t->cur]);
            t->launches += 1;
        }
        t->has_bm = true;
        conv = 1;
    }
    const int out = (int)(t->call % 3);
    const unsigned long long seq = ++t->call;
    LevelCtx c;
    c.acc = nullptr;
    c.depth = t->depth;
    c.visited = t->visited;
    c.fbm = t->fbm[t->cur];
    c.q_next = t->q[t->cur ^ 1];
    c.q_tail = &t->dctr->qlen[out];
    c.count = &t->dctr->count[out];
    c.units_tail = &t->dctr->units[out];
    c.units = t->units;
    c.inconsistent = &t->dctr->inconsistent;
    c.ctr = t->dctr;
    c.mb = t->dmb;
    c.es = nullptr;
    c.work = &t->dctr->work[out];
    c.pull_light = pull_light();
    c.direct_claim = 0;
    if (t->instrument) {
        ABFS_CUDA(cudaMemsetAsync(t->des, 0, sizeof(unsigned long long), s));
        c.es = t->des;
    }
    c.seq = seq;
    c.zero_slot = (int)(seq % 3);
    c.level = (int32_t)level;
    c.lvl1 = (int32_t)(level + 1);
    switch (variant) {
    case 0: launch_strategy<0>(t, c, kernel, chunk); break;
    case 1: launch_strategy<1>(t, c, kernel, chunk); break;
    default: launch_strategy<2>(t, c, kernel, chunk); break;
    }
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaEventRecord(t->ev[2 * ev_slot + 1], s));
    ABFS_TRY(wait_mailbox(t, seq));
    const bool topdown = kernel != ABFS_VERTEX_PULL;
    const uint64_t cnt = topdown ? (uint64_t)t->mb->qlen : (uint64_t)t->mb->count;
    t->cur ^= 1;
    t->has_q = topdown;
    t->has_bm = !topdown;
    t->F = cnt;
    // After an inconsistent level, lowered (non-counted) vertices also sit at
    // depth level+1: the next level must rebuild its frontier from depths.
    t->expect_level = t->inconsistent ? -1 : level + 1;
    *new_count = cnt;
    if (t->instrument) {
        unsigned long long es = 0;
        ABFS_CUDA(cudaMemcpyAsync(&es, t->des, sizeof(es), cudaMemcpyDeviceToHost, s));
        ABFS_CUDA(cudaStreamSynchronize(s));
        if (t->es_log.size() <= ev_slot) t->es_log.resize(ev_slot + 1);
        t->es_log[ev_slot] = es;
    }
    if (timed_now) {
        ABFS_CUDA(cudaEventSynchronize(t->ev[2 * ev_slot + 1]));
        float ms = 0.f;
        ABFS_CUDA(cudaEventElapsedTime(&ms, t->ev[2 * ev_slot], t->ev[2 * ev_slot + 1]));
        const uint64_t ns = (uint64_t)llround((double)ms * 1e6);
        *elapsed_ns = ns ? ns : 1;
    }
    if (converted) *converted = conv;
    return ABFS_OK;
}

static int event_ns(abfs_traversal *t, size_t slot, uint64_t *ns) {
    float ms = 0.f;
    ABFS_CUDA(cudaEventElapsedTime(&ms, t->ev[2 * slot], t->ev[2 * slot + 1]));
    const uint64_t v = (uint64_t)llround((double)ms * 1e6);
    *ns = v ? v : 1;
    return ABFS_OK;
}

extern "C" int abfs_traversal_create(abfs_graph *g, abfs_traversal **out) {
    if (!g || !out) return fail(ABFS_EINVAL, "null argument");
    ABFS_CUDA(cudaSetDevice(g->device));
    abfs_traversal *t = new abfs_traversal();
    t->g = g;
    t->device = g->device;
    const uint64_t n = g->d.n, m = g->d.m;
    t->words = (n + 31) / 32;
    const uint64_t wpad = t->words + 4;
    const uint64_t qcap = n + 4;
    // CTA work units of one level: a vertex-push hub (degree > kPushHub)
    // yields ceil(deg / kUnit) <= deg / kPushHub units, a push-warp hub or a
    // pull remainder (> kHeavy / kPullHeavy) fewer -- m / kPushHub bounds all
    const uint64_t ucap = m / kPushHub + 64;
    static_assert(kPushHub <= kHeavy && kPushHub <= kPullHeavy && kPushHub <= kUnit, "unit bound");
    cudaError_t e = cudaSuccess;
    auto A = [&](void **p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(p, bytes);
    };
    A((void **)&t->depth, (n + 4) * sizeof(int32_t));
    A((void **)&t->visited, wpad * 4);
    A((void **)&t->noin, wpad * 4);
    A((void **)&t->fbm[0], wpad * 4);
    A((void **)&t->fbm[1], wpad * 4);
    A((void **)&t->q[0], qcap * 4);
    A((void **)&t->q[1], qcap * 4);
    A((void **)&t->units, ucap * sizeof(uint2));
    A((void **)&t->dctr, sizeof(Ctr));
    A((void **)&t->des, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost((void **)&t->hctr, sizeof(Ctr));
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&t->mb, sizeof(Mailbox), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void **)&t->dmb, t->mb, 0);
    if (e == cudaSuccess) std::memset(t->mb, 0, sizeof(Mailbox));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) t->own_stream = true;
    if (e == cudaSuccess) e = cudaEventCreate(&t->et0);
    if (e == cudaSuccess) e = cudaMemset(t->dctr, 0, sizeof(Ctr));
    if (e == cudaSuccess) e = cudaMemset(t->depth, 0xff, (n + 4) * sizeof(int32_t));
    if (e == cudaSuccess && t->words) {
        k_noin<<<grid_for(t->words, kBlock, 1ull << 31), kBlock>>>(g->d.in_off, n, t->words, t->noin);
        e = cudaDeviceSynchronize();
        if (e == cudaSuccess) {
            unsigned int *dmax = nullptr;
            e = cudaMalloc(&dmax, sizeof(unsigned int));
            if (e == cudaSuccess) e = cudaMemset(dmax, 0, sizeof(unsigned int));
            if (e == cudaSuccess) {
                k_max_degree<<<grid_for(n, kBlock, 148 * 16), kBlock>>>(g->d.out_off, n, dmax);
                unsigned int h = 0;
                e = cudaMemcpy(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost);
                t->max_out_degree = h;
            }
            cudaFree(dmax);
        }
        if (e == cudaSuccess) {
            unsigned long long *dcnt = nullptr, hc = 0;
            e = cudaMalloc(&dcnt, sizeof(unsigned long long));
            if (e == cudaSuccess) e = cudaMemset(dcnt, 0, sizeof(unsigned long long));
            if (e == cudaSuccess) {
                k_count_bits<<<grid_for(t->words, kBlock, 148 * 16), kBlock>>>(t->noin, t->words, dcnt);
                e = cudaMemcpy(&hc, dcnt, sizeof(hc), cudaMemcpyDeviceToHost);
            }
            cudaFree(dcnt);
            t->n_noin = hc - (t->words * 32 - n);   // padding bits are set
        }
    }
    if (e != cudaSuccess) {
        set_error(std::string("traversal_create: ") + cudaGetErrorString(e));
        abfs_traversal_destroy(t);
        return e == cudaErrorMemoryAllocation ? ABFS_ENOMEM : ABFS_ECUDA;
    }
    *out = t;
    return ABFS_OK;
}

extern "C" void abfs_traversal_destroy(abfs_traversal *t) {
    if (!t) return;
    { ABFS_LOCK(t); }   // no call on this handle is in flight any more
    for (abfs_traversal *u : t->sub) abfs_traversal_destroy(u);
    cudaSetDevice(t->device);
    if (t->stream) cudaStreamSynchronize(t->stream);
    cudaFree(t->depth);
    cudaFree(t->visited);
    cudaFree(t->noin);
    cudaFree(t->fbm[0]);
    cudaFree(t->fbm[1]);
    cudaFree(t->q[0]);
    cudaFree(t->q[1]);
    cudaFree(t->units);
    cudaFree(t->dctr);
    cudaFree(t->des);
    cudaFree(t->dsolo);
    if (t->mrecs) cudaFreeHost(t->mrecs);
    if (t->mnlev) cudaFreeHost(t->mnlev);
    if (t->hroots) cudaFreeHost(t->hroots);
    cudaFree(t->droots);
    cudaFree(t->dsums);
    cudaFree(t->acc);
    cudaFree(t->pl);
    cudaFree(t->dtree);
    if (t->htree) cudaFreeHost(t->htree);
    if (t->stage) cudaFreeHost(t->stage);
    for (cudaEvent_t e : t->stage_ev)
        if (e) cudaEventDestroy(e);
    if (t->hctr) cudaFreeHost(t->hctr);
    if (t->mb) cudaFreeHost(t->mb);
    for (cudaEvent_t e : t->ev) cudaEventDestroy(e);
    if (t->et0) cudaEventDestroy(t->et0);
    if (t->own_stream && t->stream) cudaStreamDestroy(t->stream);
    delete t;
}

extern "C" int abfs_traversal_set_stream(abfs_traversal *t, void *stream) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    ABFS_LOCK(t);
    ABFS_CUDA(cudaSetDevice(t->device));
    ABFS_CUDA(cudaStreamSynchronize(t->stream));
    if (t->own_stream) cudaStreamDestroy(t->stream);
    if (stream) {
        t->stream = (cudaStream_t)stream;
        t->own_stream = false;
    } else {
        ABFS_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
        t->own_stream = true;
    }
    return ABFS_OK;
}

static int init_impl(abfs_traversal *t, int64_t root) {
    const uint64_t n = t->g->d.n;
    if (root < 0 || (uint64_t)root >= n)
        return fail(ABFS_EINVAL, "root " + std::to_string(root) + " out of range for |V|=" +
                                     std::to_string(n));
    ABFS_CUDA(cudaSetDevice(t->device));
    t->cur = 0;
    k_init<<<grid_for(t->words, kBlock, 1ull << 31), kBlock, 0, t->stream>>>(
        t->depth, t->visited, t->fbm[0], t->q[0], n, t->words, (uint32_t)root);
    t->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaMemsetAsync(&t->dctr->inconsistent, 0, sizeof(unsigned), t->stream));
    t->has_q = true;
    t->has_bm = true;
    t->F = 1;
    t->expect_level = 0;
    t->inconsistent = false;
    return ABFS_OK;
}

extern "C" int abfs_init_depths(abfs_traversal *t, int64_t root) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    ABFS_LOCK(t);
    ABFS_TRY(init_impl(t, root));
    ABFS_CUDA(cudaStreamSynchronize(t->stream));
    return ABFS_OK;
}

extern "C" int abfs_load_depths(abfs_traversal *t, const int32_t *host) {
    if (!t || !host) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_CUDA(cudaSetDevice(t->device));
    ABFS_CUDA(cudaMemcpyAsync(t->depth, host, t->g->d.n * sizeof(int32_t),
                              cudaMemcpyHostToDevice, t->stream));
    ABFS_CUDA(cudaStreamSynchronize(t->stream));
    t->expect_level = -1;
    return ABFS_OK;
}

// Depths to a caller (pageable) buffer: large arrays go through two pinned
// staging chunks, the D2H of chunk k+1 overlapping the multi-threaded host
// copy of chunk k (pageable cudaMemcpy alone is several times slower).
constexpr size_t kStageChunk = 8u << 20;   // bytes

extern "C" int abfs_read_depths(abfs_traversal *t, int32_t *host) {
    if (!t || !host) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_CUDA(cudaSetDevice(t->device));
    const size_t bytes = t->g->d.n * sizeof(int32_t);
    cudaPointerAttributes pa;
    const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    if (!pinned) cudaGetLastError();   // clear a sticky-free lookup error
    if (pinned || bytes < 2 * kStageChunk) {
        ABFS_CUDA(cudaMemcpyAsync(host, t->depth, bytes, cudaMemcpyDeviceToHost, t->stream));
        ABFS_CUDA(cudaStreamSynchronize(t->stream));
        return ABFS_OK;
    }
    if (!t->stage) {
        ABFS_CUDA(cudaMallocHost(&t->stage, 2 * kStageChunk));
        for (int i = 0; i < 2; ++i) ABFS_CUDA(cudaEventCreateWithFlags(&t->stage_ev[i], cudaEventDisableTiming));
    }
    const char *dsrc = reinterpret_cast<const char *>(t->depth);
    char *dst = reinterpret_cast<char *>(host);
    const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
    auto issue = [&](size_t k) -> cudaError_t {
        const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
        cudaError_t e = cudaMemcpyAsync(t->stage + (k & 1) * kStageChunk, dsrc + off, len,
                                        cudaMemcpyDeviceToHost, t->stream);
        if (e == cudaSuccess) e = cudaEventRecord(t->stage_ev[k & 1], t->stream);
        return e;
    };
    ABFS_CUDA(issue(0));
    for (size_t k = 0; k < nchunks; ++k) {
        if (k + 1 < nchunks) ABFS_CUDA(issue(k + 1));
        ABFS_CUDA(cudaEventSynchronize(t->stage_ev[k & 1]));
        const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
        const char *from = t->stage + (k & 1) * kStageChunk;
        const int parts = 8;
#pragma omp parallel for num_threads(parts) schedule(static)
        for (int p = 0; p < parts; ++p) {
            const size_t a = len * p / parts, b = len * (p + 1) / parts;
            std::memcpy(dst + off + a, from + a, b - a);
        }
    }
    return ABFS_OK;
}

extern "C" int abfs_level(abfs_traversal *t, int64_t level, int kernel, int variant,
                          int64_t chunk, uint64_t *new_count, uint64_t *elapsed_ns) {
    if (!t || !new_count || !elapsed_ns) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    return level_impl(t, level, kernel, variant, chunk, new_count, 0, true, elapsed_ns, nullptr);
}

extern "C" int abfs_run_level(abfs_traversal *t, int32_t *host, int64_t level, int kernel,
                              int variant, int64_t chunk, uint64_t *new_count,
                              uint64_t *elapsed_ns) {
    if (!t || !host || !new_count || !elapsed_ns) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_TRY(level_params_ok(level, kernel, variant, chunk));
    ABFS_TRY(abfs_load_depths(t, host));
    ABFS_TRY(level_impl(t, level, kernel, variant, chunk, new_count, 0, true, elapsed_ns, nullptr));
    return abfs_read_depths(t, host);
}

static int finish_traversal(abfs_traversal *t, size_t n_levels, int32_t *depths_out) {
    ABFS_CUDA(cudaEventSynchronize(t->ev[2 * (n_levels - 1) + 1]));
    float ms = 0.f;
    ABFS_CUDA(cudaEventElapsedTime(&ms, t->et0, t->ev[2 * (n_levels - 1) + 1]));
    t->last_trav_ns = (uint64_t)llround((double)ms * 1e6);
    if (depths_out) ABFS_TRY(abfs_read_depths(t, depths_out));
    return ABFS_OK;
}

constexpr uint32_t kMegaCap = 1u << 16;   // level records kept by the megakernel

// Run a whole traversal in the persistent cooperative kernel.  fixed_pair
// >= 0 runs bfs_full with that pair; otherwise the tree picks per level.
constexpr size_t kMaxBatch = 4096;         // roots per batched megakernel launch

// The tree with every node that tests a STATIC feature (vertex / edge count,
// degree summaries) resolved for this graph: those comparisons have the same
// outcome at every level, so the device walk only visits nodes on the four
// per-level features.  Leaf reached for any feature vector is unchanged.
struct PrunedTree {
    std::vector<uint16_t> feat;
    std::vector<double> thr;
    std::vector<uint32_t> left, right;
    std::vector<uint8_t> cls;
};

static bool dynamic_feature(int canon) { return canon >= 2 && canon <= 5; }

static uint32_t prune_node(const abfs_tree *tr, const double *st, uint32_t node, PrunedTree &out) {
    while (tr->leaf_classes[node] == ABFS_NOT_A_LEAF) {
        const int canon = tr->selection[tr->features[node]];
        if (dynamic_feature(canon)) break;
        node = (st[canon] < tr->thresholds[node]) ? tr->lefts[node] : tr->rights[node];
    }
    const uint32_t idx = (uint32_t)out.cls.size();
    out.feat.push_back(tr->features[node]);
    out.thr.push_back(tr->thresholds[node]);
    out.left.push_back(0);
    out.right.push_back(0);
    out.cls.push_back(tr->leaf_classes[node]);
    if (tr->leaf_classes[node] == ABFS_NOT_A_LEAF) {
        const uint32_t l = prune_node(tr, st, tr->lefts[node], out);
        const uint32_t r = prune_node(tr, st, tr->rights[node], out);
        out.left[idx] = l;
        out.right[idx] = r;
    }
    return idx;
}

// roots: nroots >= 1 traversals run back to back in one launch; with
// host_init the host ran init_depths for the single root, otherwise every
// root's init runs inside the kernel.  n_levels = the last root's level count.
namespace abfs {
// The device tree of the megakernel for a graph with n vertices (CutNode
// array; one zero node when there is no tree).
void stage_cut_tree(const abfs_tree *tr, const double *static24, uint64_t n,
                    std::vector<unsigned char> &blob, uint32_t &nn) {
    PrunedTree pt;
    if (tr && static24) prune_node(tr, static24, 0, pt);
    nn = (uint32_t)pt.cls.size();
    blob.assign((nn ? nn : 1) * sizeof(CutNode), 0);
    if (!nn) return;
    const double nv = (double)(unsigned long long)static24[0];
    CutNode *cn = reinterpret_cast<CutNode *>(blob.data());
    for (uint32_t k = 0; k < nn; ++k) {
        cn[k].cls = pt.cls[k];
        cn[k].left = pt.left[k];
        cn[k].right = pt.right[k];
        if (pt.cls[k] != ABFS_NOT_A_LEAF) continue;
        const int canon = tr->selection[pt.feat[k]];
        const double thr = pt.thr[k];
        const bool pct = canon == 3 || canon == 5;
        cn[k].on_disc = (canon == 4 || canon == 5) ? 1 : 0;
        // smallest k in [0, n] failing "x(k) < thr" (n + 1 if none does)
        auto holds = [&](uint64_t x) { return pct ? ((double)x / nv < thr) : ((double)x < thr); };
        uint64_t lo = 0, hi = n + 1;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (holds(mid)) lo = mid + 1;
            else hi = mid;
        }
        cn[k].cutoff = lo;
    }
}

// Plain cooperative launch of the default megakernel variant (partitions).
int mega_launch_plain(const MegaParams &P, cudaStream_t s, int device) {
    // co-resident grid per device (processes may drive GPUs of different
    // occupancy); written once per device, same value from any thread
    static int grids[64] = {0};
    if (device < 0 || device >= 64) return fail(ABFS_EINVAL, "device ordinal out of range");
    int &grid = grids[device];
    void *kfn = (void *)k_mega<kMegaMinB, true>;
    if (!grid) {
        int per = 0, sms = 0;
        ABFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, kBlock, 0));
        ABFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        if (per < 1) return fail(ABFS_ECUDA, "megakernel cannot be resident");
        grid = per * sms;
    }
    MegaParams Q = P;
    void *args[] = {&Q};
    ABFS_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kBlock), args, 0, s));
    return ABFS_OK;
}
}  // namespace abfs

static int mega_run(abfs_traversal *t, const uint32_t *roots, size_t nroots, bool host_init,
                    int fixed_pair, const abfs_tree *tr, const double *static24, int64_t chunk,
                    size_t *n_levels, uint64_t *checksums = nullptr) {
    const DevGraph &g = t->g->d;
    cudaStream_t s = t->stream;
    ABFS_CUDA(cudaSetDevice(t->device));
    if (!t->mrecs) {
        // level records go straight to host-mapped memory (one 64-byte posted
        // write per level), so a traversal needs a single stream sync
        ABFS_CUDA(cudaHostAlloc((void **)&t->mrecs, kMegaCap * sizeof(MegaRecord), cudaHostAllocMapped));
        ABFS_CUDA(cudaHostGetDevicePointer((void **)&t->drecs, t->mrecs, 0));
        ABFS_CUDA(cudaHostAlloc((void **)&t->mnlev, kMaxBatch * sizeof(unsigned long long),
                                cudaHostAllocMapped));
        ABFS_CUDA(cudaHostGetDevicePointer((void **)&t->dnlev, t->mnlev, 0));
        ABFS_CUDA(cudaMallocHost((void **)&t->hroots, kMaxBatch * sizeof(uint32_t)));
        ABFS_CUDA(cudaMalloc((void **)&t->droots, kMaxBatch * sizeof(uint32_t)));
        ABFS_CUDA(cudaMalloc((void **)&t->dsums, kMaxBatch * sizeof(unsigned long long)));
    }
    if (nroots < 1 || nroots > kMaxBatch) return fail(ABFS_EINVAL, "bad root count");
    // cluster solo mode only on graphs without hubs (max out-degree <=
    // kPushHub): there no small level ever needs CTA units, so solo levels
    // never hand back; on skewed graphs the cluster-constrained grid and hub
    // hand-backs cost more than the solo levels save (measured on
    // Kronecker-24).  The kernel without solo code spills less (224 / 340 B
    // instead of 260 / 504 B).
    const char *solo_env = getenv("ABFS_SOLO");
    const bool want_solo = solo_env ? atoi(solo_env) != 0 : t->max_out_degree <= kSoloMaxDegree;
#ifdef ABFS_MEGA_VARIANTS   // occupancy experiments (set_mode 2 / 3)
    void *kfn = t->mega_minb == 4   ? (void *)k_mega<4, false>
                : t->mega_minb == 6 ? (void *)k_mega<6, false>
                                    : (void *)k_mega<kMegaMinB, false>;
#else
    void *kfn = want_solo ? (void *)k_mega<kMegaMinB, false, true>
                          : (void *)k_mega<kMegaMinB, false, false>;
#endif
    // solo cluster size: 16 CTAs (non-portable; 4096 lanes, one pass over a
    // mesh-4096 level where 8 CTAs need two: mesh 4096^2 -23 % time) on
    // low-degree graphs, whose long diameters are runs of small levels; 8
    // elsewhere (16-CTA clusters fit fewer CTAs per grid: 608 vs 740 on B200,
    // which big levels pay)
    const int solo_cl = (int)env_u64("ABFS_SOLO_CLUSTER", t->max_out_degree <= 8 ? 16 : 8);
    if (t->mega_kfn != kfn || t->solo_req != solo_cl) {   // e.g. ABFS_SOLO toggled: re-size the grid
        t->mega_kfn = kfn;
        t->solo_req = solo_cl;
        t->mega_grid = 0;
    }
    if (!t->mega_grid) {
        int per = 0, sms = 0;
        ABFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, kBlock, 0));
        ABFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device));
        if (per < 1) return fail(ABFS_ECUDA, "megakernel cannot be resident");
        t->mega_grid = std::max(1, per * sms / t->grid_div);
        t->mega_cluster = 0;
        // cluster launch for solo mode: the grid must be whole clusters that
        // are all co-resident (cooperative)
        if (want_solo) {
            // (a refused 16-CTA cluster falls back to 8)
            for (int cl = solo_cl; cl >= 2 && !t->mega_cluster; cl = cl > 8 ? cl / 2 : 0) {
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                if (cl > 8) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                at[0].val.clusterDim.x = cl;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3((unsigned)(t->mega_grid / cl * cl));
                cfg.blockDim = dim3(kBlock);
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int nclusters = 0;
                if (cudaOccupancyMaxActiveClusters(&nclusters, kfn, &cfg) == cudaSuccess &&
                    nclusters / t->grid_div > 0) {
                    t->mega_grid = std::min(t->mega_grid / cl, nclusters / t->grid_div) * cl;
                    t->mega_cluster = cl;
                }
                cudaGetLastError();
            }
        }
    }
    if (!t->dsolo) ABFS_CUDA(cudaMalloc(&t->dsolo, sizeof(SoloState)));
    // stage the device tree: static-feature nodes resolved, float64 tests on
    // the per-level features turned into exact integer cutoffs (CutNode)
    std::vector<unsigned char> blob;
    uint32_t nn = 0;
    stage_cut_tree(tr, static24, g.n, blob, nn);
    const size_t bytes = blob.size();
    if (bytes > t->tree_cap) {
        cudaFree(t->dtree);
        if (t->htree) cudaFreeHost(t->htree);
        t->dtree = nullptr;
        t->htree = nullptr;
        t->last_blob.clear();
        ABFS_CUDA(cudaMalloc(&t->dtree, bytes * 2));
        ABFS_CUDA(cudaMallocHost(&t->htree, bytes * 2));
        t->tree_cap = bytes * 2;
    }
    if (blob != t->last_blob) {
        // every mega_run ends with a stream sync, so the pinned staging copy
        // is never in flight here; an unchanged tree is not re-uploaded
        std::memcpy(t->htree, blob.data(), bytes);
        ABFS_CUDA(cudaMemcpyAsync(t->dtree, t->htree, bytes, cudaMemcpyHostToDevice, s));
        t->last_blob.swap(blob);
    }
    if (host_init) {
        ABFS_TRY(init_impl(t, roots[0]));
        ABFS_CUDA(cudaMemsetAsync(t->dctr, 0, offsetof(Ctr, cq), s));
        // every megakernel slot array from cq3 on (cq3, es3, work, ps, pc)
        ABFS_CUDA(cudaMemsetAsync(&t->dctr->cq3[0], 0, sizeof(Ctr) - offsetof(Ctr, cq3), s));
    } else {
        std::memcpy(t->hroots, roots, nroots * sizeof(uint32_t));
        ABFS_CUDA(cudaMemcpyAsync(t->droots, t->hroots, nroots * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, s));
    }
    ABFS_TRY(ensure_events(t, 2));
    MegaParams P{};   // value-initialised: every optional pointer starts null
    P.depth = t->depth;
    P.visited = t->visited;
    P.noin = t->noin;
    P.fbm0 = t->fbm[0];
    P.fbm1 = t->fbm[1];
    P.q0 = t->q[0];
    P.q1 = t->q[1];
    P.units = t->units;
    P.ctr = t->dctr;
    P.out_off = g.out_off;
    P.dst = g.dst;
    P.org = g.org;
    P.in_off = g.in_off;
    P.src = g.src;
    P.rev_owner = g.rev_owner;
    P.first_src = g.first_src;
    P.n = g.n;
    P.m = g.m;
    P.words = t->words;
    P.tree = t->dtree;
    P.tree_nodes = nn;
    P.fixed_pair = fixed_pair;
    {
        const int64_t vc = vw_chunk(t, chunk);
        P.vw_log2 = vc >= 32 ? 5 : vc >= 16 ? 4 : vc >= 8 ? 3 : vc >= 4 ? 2 : vc >= 2 ? 1 : 0;
        const int64_t wc = chunk < 32 ? chunk : 32;
        P.vw_wide_log2 = wc >= 32 ? 5 : wc >= 16 ? 4 : wc >= 8 ? 3 : wc >= 4 ? 2 : wc >= 2 ? 1 : 0;
        if (env_u64("ABFS_VW_FORCE", 0)) P.vw_wide_log2 = P.vw_log2;   // A/B: one width for all levels
        // ER-32M, F <= 28 K levels: 21.8 -> 10.5 us (F = 877), 49 -> 39 us (F = 28 K)
        P.vw_wide_f = env_u64("ABFS_VW_WIDE_F", 1ull << 16);
    }
    P.instrument = t->instrument ? 1 : 0;
    P.pull_light = pull_light();
    P.cap = kMegaCap;
    P.recs = t->drecs;
    P.n_levels = t->dnlev;
    P.roots = t->droots;
    P.nroots = (uint32_t)nroots;
    P.init_in_kernel = host_init ? 0 : 1;
    P.solo_ctas = t->mega_cluster ? (uint32_t)t->mega_cluster : 0u;
    P.solo = t->dsolo;
    P.solo_passes = (uint32_t)env_u64("ABFS_SOLO_PASSES", 2);   // mesh 4096^2: 2 passes -9 % vs 1
    // claims without the visited-word filter load: every solo level (mesh
    // 4096^2 -8.5 %: the filter load is one more L2 round trip on a level's
    // chain) and grid levels of at most direct_f frontier vertices
    P.solo_direct = (uint32_t)env_u64("ABFS_SOLO_DIRECT", 1);
    P.direct_f = env_u64("ABFS_DIRECT_F", 0);
    // RED levels reduce every candidate without the visited-word filter load
    // on graphs without a heavy tail (max out-degree <= 4 x mean; ER-32M BFS
    // -8.6 %: its 883 K-vertex push level reaches mostly unvisited vertices,
    // so the filter only lengthened the chain).  Hub frontiers keep the
    // filter: their neighbourhoods overlap, and the unfiltered duplicates
    // cost fixed-push K24 runs 1.5x.
    {
        const uint64_t mean = g.n ? g.m / g.n : 0;
        P.red_direct = (uint32_t)env_u64("ABFS_RED_DIRECT", t->max_out_degree <= 4 * (mean ? mean : 1));
    }
    P.part = 0;
    P.m_rev = g.m;
    P.lo = 0;
    P.hi = g.n;
    P.wlo = 0;
    P.wend = t->words;
    P.vprev = nullptr;
    P.fnext = nullptr;
    P.peer_fbm = nullptr;
    P.peer_box = nullptr;
    P.box = nullptr;
    P.nranks = 0;
    P.rank = 0;
    P.xseq0 = 0;
    P.checksums = nullptr;
    if (checksums) {
        ABFS_CUDA(cudaMemsetAsync(t->dsums, 0, nroots * sizeof(unsigned long long), s));
        P.checksums = t->dsums;
    }
    // RED-mode top-down levels (ABFS_RED=0 disables; ABFS_RED_F / ABFS_RED_UNITS
    // override the thresholds, e.g. 1 / 1 forces every top-down level).
    // Measured on B200 (tools/level_ab.py): a full RED level is about as fast
    // as per-edge atomic claims (the random-address L2 reductions bound both)
    // but hands the next level a ready frontier bitmap -- ER-32M's pull after
    // its 18.6 M-discovery push level drops 437 -> 289 us (the queue -> bitmap
    // conversion it saves scatters one atomic per frontier vertex).  RED on a
    // hub's CTA units alone is slower (K24 hub level 61 -> 95 us: duplicate
    // candidates are not filtered by claims made earlier in the level), so
    // units stay on atomic claims by default.
    P.acc = nullptr;
    P.red_frontier = env_u64("ABFS_RED_F", g.n >> 7 > 4096 ? g.n >> 7 : 4096);
    P.red_units = (uint32_t)env_u64("ABFS_RED_UNITS", 0xffffffffull);
    P.n_noin = t->n_noin;
    // list-based pull levels (pull2.cuh), opt-in with ABFS_PULL2=1: measured
    // slower than the sub-tile pull on B200 (K24 8 roots: 2967 vs 2233 us;
    // the grid-wide probe-0 sweep moves no more loads per warp round trip
    // than the sub-tile chain, and the survivors' scans lose the L1 reuse of
    // the offsets their probe just loaded), kept tested for the carried-list
    // tail levels it does speed up
    P.pl_s = P.pl_c0 = P.pl_c1 = nullptr;
    if (ABFS_PULL2_CODE && env_u64("ABFS_PULL2", 0) && g.n < (1ull << 31)) {
        if (!t->pl) ABFS_CUDA(cudaMalloc((void **)&t->pl, 3 * (g.n + 4) * sizeof(uint32_t)));
        P.pl_s = t->pl;
        P.pl_c0 = t->pl + (g.n + 4);
        P.pl_c1 = t->pl + 2 * (g.n + 4);
    }
    P.pull_wide_max = env_u64("ABFS_PULL_WIDE", g.n >> 5);
    if (env_u64("ABFS_RED", 1)) {
        if (!t->acc) {
            ABFS_CUDA(cudaMalloc((void **)&t->acc, (t->words + 4) * 4));
            ABFS_CUDA(cudaMemsetAsync(t->acc, 0, (t->words + 4) * 4, s));
        }
        P.acc = t->acc;
    }
    for (size_t i = 0; i < nroots; ++i) ((volatile unsigned long long *)t->mnlev)[i] = 0;
    // one megakernel per device at a time (co-residency), except a split
    // batch's sub-traversals: their parent holds the lock for all of them and
    // their grids add up to one co-resident grid
    std::unique_lock<std::mutex> mega_guard(g_mega_mu[t->device & 63], std::defer_lock);
    if (!t->is_sub) mega_guard.lock();
    ABFS_CUDA(cudaEventRecord(t->et0, s));
    void *args[] = {&P};
    if (t->mega_cluster) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = (unsigned)t->mega_cluster;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)t->mega_grid);
        cfg.blockDim = dim3(kBlock);
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        if (cudaLaunchKernelExC(&cfg, kfn, args) != cudaSuccess) {
            // cluster + cooperative launch refused: plain cooperative launch
            // without solo mode (same results, one grid barrier per level)
            cudaGetLastError();
            int per = 0, sms = 0;
            ABFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, kBlock, 0));
            ABFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device));
            t->mega_grid = std::max(1, per * sms / t->grid_div);
            t->mega_cluster = 0;
            P.solo_ctas = 0;
            ABFS_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(t->mega_grid), dim3(kBlock), args, 0, s));
        }
    } else {
        ABFS_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(t->mega_grid), dim3(kBlock), args, 0, s));
    }
    t->launches += 1;
    ABFS_CUDA(cudaEventRecord(t->ev[1], s));
    ABFS_CUDA(cudaStreamSynchronize(s));
    if (checksums)
        ABFS_CUDA(cudaMemcpy(checksums, t->dsums, nroots * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost));
    unsigned long long tot = 0;
    for (size_t i = 0; i < nroots; ++i) tot += ((volatile unsigned long long *)t->mnlev)[i];
    const unsigned long long nl = ((volatile unsigned long long *)t->mnlev)[nroots - 1];
    // records of the last root (the batch keeps all roots' records in mrecs)
    const size_t keep_all = tot < kMegaCap ? tot : kMegaCap;
    const size_t first = (size_t)(tot - nl) < keep_all ? (size_t)(tot - nl) : keep_all;
    t->hrecs.assign(t->mrecs + first, t->mrecs + keep_all);
    const size_t keep = t->hrecs.size();
    t->batch_levels.assign(t->mnlev, t->mnlev + nroots);
    t->batch_recs = keep_all;
    float ms = 0.f;
    ABFS_CUDA(cudaEventElapsedTime(&ms, t->et0, t->ev[1]));
    t->last_trav_ns = (uint64_t)llround((double)ms * 1e6);
    // final state: depths + frontier of the terminating level are resident
    const MegaRecord *last = keep ? &t->hrecs[keep - 1] : nullptr;
    t->cur = (int)((nl - 1 + 1) & 1);
    t->has_q = last && last->kernel != ABFS_VERTEX_PULL;
    t->has_bm = !t->has_q;
    t->F = 0;
    t->expect_level = -1;
    // the per-level path needs its counter slots zeroed again (all three, so
    // any starting slot works; t->call keeps growing for mailbox stamps)
    ABFS_CUDA(cudaMemsetAsync(t->dctr, 0, offsetof(Ctr, cq) + sizeof(unsigned), s));
    ABFS_CUDA(cudaMemsetAsync(&t->dctr->work[0], 0, 8 * 3, s));
    if (t->instrument) {
        t->es_log.resize(keep);
        for (size_t l = 0; l < keep; ++l) t->es_log[l] = t->hrecs[l].scanned;
    }
    *n_levels = (size_t)nl;
    return ABFS_OK;
}

static uint64_t rec_ns(const MegaRecord &r) {
    const uint64_t d = r.t_end > r.t_start ? r.t_end - r.t_start : 0;
    return d ? d : 1;
}

extern "C" int abfs_traversal_set_mode(abfs_traversal *t, int device_loop) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    ABFS_LOCK(t);
    t->use_mega = device_loop != 0;
    const int minb = device_loop == 3 ? 4 : device_loop == 2 ? 6 : kMegaMinB;
    if (minb != t->mega_minb) {
        t->mega_minb = minb;
        t->mega_grid = 0;
    }
    return ABFS_OK;
}

extern "C" int abfs_bfs_full(abfs_traversal *t, int64_t root, int kernel, int variant,
                             int64_t chunk, int32_t *depths_out, uint64_t *counts,
                             uint64_t *elapsed, size_t cap, size_t *n_levels) {
    if (!t || !n_levels) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_TRY(level_params_ok(0, kernel, variant, chunk));
    if (t->use_mega) {
        if (root < 0 || (uint64_t)root >= t->g->d.n)
            return fail(ABFS_EINVAL, "root " + std::to_string(root) + " out of range for |V|=" +
                                         std::to_string(t->g->d.n));
        size_t nl = 0;
        const uint32_t r32 = (uint32_t)root;
        ABFS_TRY(mega_run(t, &r32, 1, true, kernel * 3 + variant, nullptr, nullptr, chunk, &nl));
        // more levels than the megakernel keeps records for (> kMegaCap): the
        // launch-path driver below reports every level (the reference returns
        // them all, kernels.py:356-371)
        if (!((counts || elapsed) && nl > t->hrecs.size() && cap > t->hrecs.size())) {
            *n_levels = nl;
            for (size_t l = 0; l < nl && l < cap && l < t->hrecs.size(); ++l) {
                if (counts) counts[l] = t->hrecs[l].new_count;
                if (elapsed) elapsed[l] = rec_ns(t->hrecs[l]);
            }
            if (depths_out) ABFS_TRY(abfs_read_depths(t, depths_out));
            return ABFS_OK;
        }
    }
    ABFS_TRY(init_impl(t, root));
    ABFS_CUDA(cudaEventRecord(t->et0, t->stream));
    size_t nl = 0;
    for (int64_t level = 0;; ++level) {
        uint64_t c = 0;
        ABFS_TRY(level_impl(t, level, kernel, variant, chunk, &c, (size_t)level, false, nullptr,
                            nullptr));
        if ((size_t)level < cap && counts) counts[level] = c;
        if (c == 0) {
            nl = (size_t)level + 1;
            break;
        }
    }
    *n_levels = nl;
    ABFS_TRY(finish_traversal(t, nl, depths_out));
    if (elapsed)
        for (size_t l = 0; l < nl && l < cap; ++l) ABFS_TRY(event_ns(t, l, &elapsed[l]));
    return ABFS_OK;
}

extern "C" int abfs_features(const double *static24, uint64_t frontier, uint64_t discovered,
                             double *out24) {
    // extract_runtime_features (features.py:98-121): float64 true divisions.
    if (!static24 || !out24) return fail(ABFS_EINVAL, "null argument");
    const double nd = static24[0];
    const uint64_t n = (uint64_t)nd;
    if (n < 1) return fail(ABFS_EFEATURE, "stats must describe a non-empty graph");
    if (discovered < frontier)
        return fail(ABFS_EFEATURE, "need 0 <= frontier_abs <= discovered_abs, got " +
                                       std::to_string(frontier) + " and " + std::to_string(discovered));
    if (discovered > n)
        return fail(ABFS_EFEATURE, "discovered_abs " + std::to_string(discovered) +
                                       " exceeds |V|=" + std::to_string(n));
    std::memcpy(out24, static24, 24 * sizeof(double));
    out24[2] = (double)frontier;
    out24[3] = (double)frontier / (double)n;
    out24[4] = (double)discovered;
    out24[5] = (double)discovered / (double)n;
    return ABFS_OK;
}

static int tree_leaf(const abfs_tree *tr, const double *canonical24) {
    // FlatTree.predict_one (tree.py:332-339): strict < goes left.
    uint32_t node = 0;
    while (tr->leaf_classes[node] == ABFS_NOT_A_LEAF) {
        const double x = canonical24[tr->selection[tr->features[node]]];
        node = (x < tr->thresholds[node]) ? tr->lefts[node] : tr->rights[node];
    }
    return tr->leaf_classes[node];
}

static int tree_ok(const abfs_tree *tr) {
    if (!tr || tr->node_count == 0 || !tr->selection || !tr->features || !tr->thresholds ||
        !tr->lefts || !tr->rights || !tr->leaf_classes)
        return fail(ABFS_EINVAL, "invalid tree");
    for (uint32_t i = 0; i < tr->n_selection; ++i)
        if (tr->selection[i] >= ABFS_N_FEATURES) return fail(ABFS_EINVAL, "bad selection index");
    for (uint32_t k = 0; k < tr->node_count; ++k) {
        const uint8_t c = tr->leaf_classes[k];
        if (c == ABFS_NOT_A_LEAF) {
            if (tr->features[k] >= tr->n_selection || tr->lefts[k] >= tr->node_count ||
                tr->rights[k] >= tr->node_count || tr->lefts[k] <= k || tr->rights[k] <= k)
                return fail(ABFS_EINVAL, "malformed tree node " + std::to_string(k));
        } else if (c >= 15 && c != ABFS_LEAF_UNKNOWN) {
            return fail(ABFS_EINVAL, "bad leaf class " + std::to_string(c));
        }
    }
    return ABFS_OK;
}

extern "C" int abfs_tree_predict(const abfs_tree *tr, const double *projected, int *leaf) {
    if (!projected || !leaf) return fail(ABFS_EINVAL, "null argument");
    ABFS_TRY(tree_ok(tr));
    uint32_t node = 0;
    while (tr->leaf_classes[node] == ABFS_NOT_A_LEAF) {
        const double x = projected[tr->features[node]];
        node = (x < tr->thresholds[node]) ? tr->lefts[node] : tr->rights[node];
    }
    *leaf = tr->leaf_classes[node];
    return ABFS_OK;
}

extern "C" int abfs_adaptive_bfs(abfs_traversal *t, int64_t root, const abfs_tree *tr,
                                 const double *static24, int64_t chunk, int32_t *depths_out,
                                 abfs_level_record *recs, size_t cap, size_t *n_levels) {
    if (!t || !static24 || !n_levels) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_TRY(tree_ok(tr));
    if (t->use_mega) {
        if (root < 0 || (uint64_t)root >= t->g->d.n)
            return fail(ABFS_EINVAL, "root " + std::to_string(root) + " out of range for |V|=" +
                                         std::to_string(t->g->d.n));
        size_t nl = 0;
        const uint32_t r32 = (uint32_t)root;
        ABFS_TRY(mega_run(t, &r32, 1, true, -1, tr, static24, chunk, &nl));
        if (recs && nl > t->hrecs.size() && cap > t->hrecs.size())
            goto launch_path;   // > kMegaCap levels: the launch path records them all
        *n_levels = nl;
        uint64_t disc = 1;
        if (recs)
            for (size_t l = 0; l < nl && l < cap && l < t->hrecs.size(); ++l) {
                const MegaRecord &m = t->hrecs[l];
                abfs_level_record &r = recs[l];
                disc += m.new_count;
                r.unvisited = t->g->d.n - disc;
                r.next_out_edges = t->instrument ? m.next_out_edges : ~0ull;
                r.level = (int64_t)l;
                r.kernel = m.kernel;
                r.variant = m.variant;
                r.fallback = m.fallback;
                r.converted = m.converted;
                r.frontier_size = m.frontier;
                r.new_count = m.new_count;
                r.elapsed_ns = rec_ns(m);
                const uint64_t pn = m.t_pred > m.t_start ? m.t_pred - m.t_start : 0;
                r.prediction_ns = pn ? pn : 1;
            }
        if (depths_out) ABFS_TRY(abfs_read_depths(t, depths_out));
        return ABFS_OK;
    }
launch_path:
    ABFS_TRY(init_impl(t, root));
    ABFS_CUDA(cudaEventRecord(t->et0, t->stream));
    uint64_t frontier = 1, discovered = 1;
    int pk = ABFS_EDGE_LIST, pv = ABFS_DIRECT_ATOMIC;  // DEFAULT_KERNEL adaptive.py:36-38
    double vec[24];
    for (int64_t level = 0;; ++level) {
        const uint64_t t0 = host_ns();
        ABFS_TRY(abfs_features(static24, frontier, discovered, vec));
        const int cls = tree_leaf(tr, vec);
        const uint64_t pred = host_ns() - t0;
        const int fallback = cls == ABFS_LEAF_UNKNOWN;
        if (!fallback) {
            pk = cls / 3;
            pv = cls % 3;
        }
        uint64_t c = 0;
        int conv = 0;
        ABFS_TRY(level_impl(t, level, pk, pv, chunk, &c, (size_t)level, false, nullptr, &conv));
        if (recs && (size_t)level < cap) {
            abfs_level_record &r = recs[level];
            r.level = level;
            r.kernel = pk;
            r.variant = pv;
            r.fallback = fallback;
            r.converted = conv;
            r.frontier_size = frontier;
            r.new_count = c;
            r.elapsed_ns = 0;   // filled from the level's events after the traversal
            r.prediction_ns = pred ? pred : 1;
            r.unvisited = t->g->d.n - (discovered + c);
            r.next_out_edges = ~0ull;   // instrumented runs: filled below
        }
        if (c == 0) {
            *n_levels = (size_t)level + 1;
            break;
        }
        frontier = c;
        discovered += c;
    }
    ABFS_TRY(finish_traversal(t, *n_levels, depths_out));
    if (recs)
        for (size_t l = 0; l < *n_levels && l < cap; ++l) ABFS_TRY(event_ns(t, l, &recs[l].elapsed_ns));
    if (recs && t->instrument) {
        // launch path: the discoveries of level l are the depth-(l+1)
        // vertices; one device histogram of the final depths gives every
        // level's next-frontier out-edges
        const size_t nl = *n_levels;
        std::vector<uint64_t> cnt(nl + 2), od(nl + 2), idg(nl + 2);
        ABFS_TRY(abfs_traversal_level_stats(t, nl + 1, cnt.data(), od.data(), idg.data(), nullptr));
        for (size_t l = 0; l < nl && l < cap; ++l) recs[l].next_out_edges = od[l + 1];
    }
    return ABFS_OK;
}

static int batch_ways(const abfs_traversal *t, size_t nroots);

extern "C" int abfs_traversal_set_batch_ways(abfs_traversal *t, int ways) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    if (ways < 0) return fail(ABFS_EINVAL, "ways must be >= 0 (0 = automatic)");
    ABFS_LOCK(t);
    t->batch_ways_req = ways;
    return ABFS_OK;
}

extern "C" int abfs_traversal_batch_ways(const abfs_traversal *t, size_t nroots, int *ways) {
    if (!t || !ways) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    *ways = batch_ways(t, nroots);
    return ABFS_OK;
}

extern "C" int abfs_traversal_launches(const abfs_traversal *t, uint64_t *launches) {
    if (!t || !launches) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    *launches = t->launches;
    return ABFS_OK;
}

extern "C" int abfs_last_traversal_ns(const abfs_traversal *t, uint64_t *ns) {
    if (!t || !ns) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    *ns = t->last_trav_ns;
    return ABFS_OK;
}

extern "C" int abfs_reached_edges(abfs_traversal *t, uint64_t *edges, uint64_t *vertices) {
    if (!t || !edges || !vertices) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_CUDA(cudaSetDevice(t->device));
    ABFS_CUDA(cudaMemsetAsync(&t->dctr->reached_edges, 0, 16, t->stream));
    k_reached<<<148 * 8, kBlock, 0, t->stream>>>(t->depth, t->g->d.out_off, t->g->d.n, t->dctr);
    t->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaMemcpyAsync(t->hctr, t->dctr, sizeof(Ctr), cudaMemcpyDeviceToHost, t->stream));
    ABFS_CUDA(cudaStreamSynchronize(t->stream));
    *edges = t->hctr->reached_edges;
    *vertices = t->hctr->reached_vertices;
    return ABFS_OK;
}

extern "C" int abfs_aggregate_count(int device, const int64_t *host_counts, size_t n,
                                    int variant, int64_t *total) {
    if (!total || (n && !host_counts)) return fail(ABFS_EINVAL, "null argument");
    if (variant < 0 || variant > 2)
        return fail(ABFS_EINVAL, "unknown count variant " + std::to_string(variant));
    ABFS_CUDA(cudaSetDevice(device));
    long long *d = nullptr;
    unsigned long long *dt = nullptr;
    ABFS_CUDA(cudaMalloc(&d, (n ? n : 1) * sizeof(long long)));
    cudaError_t e = cudaMalloc(&dt, sizeof(unsigned long long));
    if (e == cudaSuccess && n) e = cudaMemcpy(d, host_counts, n * sizeof(long long), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dt, 0, sizeof(unsigned long long));
    if (e == cudaSuccess && n) {
        const unsigned grid = grid_for(n, kBlock, 1ull << 31);
        if (variant == 0) k_aggregate<0><<<grid, kBlock>>>(d, n, dt);
        else if (variant == 1) k_aggregate<1><<<grid, kBlock>>>(d, n, dt);
        else k_aggregate<2><<<grid, kBlock>>>(d, n, dt);
        e = cudaGetLastError();
    }
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&h, dt, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(dt);
    if (e != cudaSuccess) return fail(ABFS_ECUDA, std::string("aggregate_count: ") + cudaGetErrorString(e));
    *total = (int64_t)h;
    return ABFS_OK;
}

extern "C" int abfs_traversal_instrument(abfs_traversal *t, int on) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    ABFS_LOCK(t);
    t->instrument = on != 0;
    t->es_log.clear();
    return ABFS_OK;
}

extern "C" int abfs_traversal_level_stats(abfs_traversal *t, size_t nlev, uint64_t *count,
                                          uint64_t *out_deg, uint64_t *in_deg, uint64_t *scanned) {
    if (!t || !count || !out_deg || !in_deg) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    ABFS_CUDA(cudaSetDevice(t->device));
    unsigned long long *h = nullptr;
    const size_t cells = 3 * (nlev + 1);
    ABFS_CUDA(cudaMalloc(&h, cells * sizeof(unsigned long long)));
    cudaError_t e = cudaMemsetAsync(h, 0, cells * sizeof(unsigned long long), t->stream);
    if (e == cudaSuccess) {
        k_level_hist<<<148 * 8, kBlock, 0, t->stream>>>(t->depth, t->g->d.out_off, t->g->d.in_off,
                                                       t->g->d.n, (uint32_t)nlev, h);
        e = cudaGetLastError();
    }
    std::vector<unsigned long long> hv(cells);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hv.data(), h, cells * 8, cudaMemcpyDeviceToHost, t->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(t->stream);
    cudaFree(h);
    if (e != cudaSuccess) return fail(ABFS_ECUDA, std::string("level_stats: ") + cudaGetErrorString(e));
    for (size_t i = 0; i <= nlev; ++i) {
        count[i] = hv[i];
        out_deg[i] = hv[(nlev + 1) + i];
        in_deg[i] = hv[2 * (nlev + 1) + i];
    }
    if (scanned)
        for (size_t i = 0; i < nlev; ++i) scanned[i] = i < t->es_log.size() ? t->es_log[i] : 0;
    return ABFS_OK;
}

extern "C" int abfs_host_register(void *ptr, size_t bytes) {
    if (!ptr || !bytes) return fail(ABFS_EINVAL, "null argument");
    ABFS_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
    return ABFS_OK;
}

extern "C" int abfs_host_unregister(void *ptr) {
    if (!ptr) return fail(ABFS_EINVAL, "null argument");
    ABFS_CUDA(cudaHostUnregister(ptr));
    return ABFS_OK;
}

// ---- split batch --------------------------------------------------------------
// A multi-root batch runs as S concurrent megakernels (S sub-traversals with
// their own scratch and stream, each 1/S of the co-resident grid, roots dealt
// round-robin).  Every level of a BFS is a grid-wide dependent chain; the
// small top-down levels (a handful of vertices, ~5-30 us of barriers and
// L2 round trips each) leave the GPU idle, and a big pull level on half the
// grid runs only ~1.3x longer (latency-bound), so two traversals side by side
// overlap one's small levels with the other's work.  Throughput, not
// latency: each BFS takes longer on its share of the grid (the per-root
// t_bfs grows), the batch finishes sooner.  Same per-root results: each root
// is one unchanged single-traversal run.  ABFS_BATCH_SPLIT=S sets the ways
// (1 disables).
static int batch_ways(const abfs_traversal *t, size_t nroots) {
    if (t->is_sub || t->instrument || nroots < 2) return 1;
    if (t->batch_ways_req > 0) return std::min({t->batch_ways_req, kMaxSplit, (int)nroots});
    // measured on B200, 8-root batches: K24 1 / 2 / 4 / 8 ways 906 / 1069 / 1136 /
    // 1022 GTEPS, ER-32M (2^25 vertices) 986 / 1103 / 1105-1178, K26 (2^26)
    // 1251 / 1289 / 1187 (bigger levels, less to overlap), mesh 4096^2 (pure
    // latency: every level is a cluster-solo chain) 0.91 / 1.78 / 3.4 / 6.8
    const int def = t->max_out_degree <= 8 ? 8 : t->g->d.n > (1ull << 25) ? 2 : 4;
    const int s = (int)env_u64("ABFS_BATCH_SPLIT", def);
    return std::max(1, std::min({s, kMaxSplit, (int)nroots}));
}

static int batch_split(abfs_traversal *t, const std::vector<uint32_t> &r32, int S,
                       const abfs_tree *tr, const double *static24, int64_t chunk,
                       uint64_t *levels, uint64_t *bfs_ns, uint64_t *total_ns,
                       uint64_t *checksums, uint64_t *new_counts, size_t counts_cap,
                       size_t *n_counts) {
    const size_t nroots = r32.size();
    for (int k = 0; k < S; ++k) {
        abfs_traversal *&u = t->sub[k];
        if (u && u->grid_div != S) {
            abfs_traversal_destroy(u);
            u = nullptr;
        }
        if (!u) {
            ABFS_TRY(abfs_traversal_create(t->g, &u));
            u->is_sub = true;
            u->grid_div = S;
        }
        u->mega_minb = t->mega_minb;
    }
    std::vector<std::vector<uint32_t>> rk(S);
    for (size_t i = 0; i < nroots; ++i) rk[i % S].push_back(r32[i]);
    std::vector<std::vector<uint64_t>> ck(S);
    for (int k = 0; k < S; ++k) ck[k].assign(rk[k].size(), 0);
    const cudaStream_t s = t->stream;
    ABFS_CUDA(cudaSetDevice(t->device));
    ABFS_TRY(ensure_events(t, 2));
    uint64_t launches0 = 0;
    for (int k = 0; k < S; ++k) launches0 += t->sub[k]->launches;
    std::lock_guard<std::mutex> mega_guard(g_mega_mu[t->device & 63]);
    // fork: the sub streams start after the caller's stream's prior work
    ABFS_CUDA(cudaEventRecord(t->et0, s));
    for (int k = 0; k < S; ++k) ABFS_CUDA(cudaStreamWaitEvent(t->sub[k]->stream, t->et0, 0));
    std::vector<int> rc(S, ABFS_OK);
    std::vector<std::string> err(S);
    std::vector<size_t> nl(S, 0);
    auto go = [&](int k) {
        rc[k] = mega_run(t->sub[k], rk[k].data(), rk[k].size(), false, -1, tr, static24, chunk,
                         &nl[k], checksums ? ck[k].data() : nullptr);
        if (rc[k] != ABFS_OK) err[k] = abfs_last_error();
    };
    std::vector<std::thread> th;
    for (int k = 1; k < S; ++k) th.emplace_back(go, k);
    go(0);
    for (auto &x : th) x.join();
    for (int k = 0; k < S; ++k)
        if (rc[k] != ABFS_OK) return fail(rc[k], err[k]);
    // join: the caller's stream continues after every sub-traversal
    for (int k = 0; k < S; ++k) ABFS_CUDA(cudaStreamWaitEvent(s, t->sub[k]->ev[1], 0));
    ABFS_CUDA(cudaEventRecord(t->ev[1], s));
    // the batch's final state on the parent: the last root's depths
    const abfs_traversal *last = t->sub[(nroots - 1) % S];
    ABFS_CUDA(cudaMemcpyAsync(t->depth, last->depth, t->g->d.n * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, s));
    ABFS_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    ABFS_CUDA(cudaEventElapsedTime(&ms, t->et0, t->ev[1]));
    t->last_trav_ns = (uint64_t)llround((double)ms * 1e6);
    uint64_t launches1 = 0;
    for (int k = 0; k < S; ++k) launches1 += t->sub[k]->launches;
    t->launches += launches1 - launches0;
    if (total_ns) *total_ns = t->last_trav_ns;
    // per-root outputs in the caller's root order
    std::vector<size_t> off(S, 0);
    t->batch_levels.assign(nroots, 0);
    size_t nc = 0;
    bool counts_whole = true;
    for (size_t i = 0; i < nroots; ++i) {
        const abfs_traversal *u = t->sub[i % S];
        const size_t j = i / S, li = (size_t)u->batch_levels[j], o = off[i % S];
        off[i % S] += li;
        t->batch_levels[i] = li;
        if (levels) levels[i] = li;
        if (checksums) checksums[i] = ck[i % S][j];
        const bool kept = li && o + li <= u->batch_recs;
        if (bfs_ns) {
            uint64_t ns = 0;
            if (kept) {
                const MegaRecord &a = u->mrecs[o], &b = u->mrecs[o + li - 1];
                ns = b.t_end > a.t_start ? b.t_end - a.t_start : 1;
            }
            bfs_ns[i] = ns;
        }
        // every root's per-level new counts, concatenated in root order, up
        // to the first root whose records were not kept
        counts_whole = counts_whole && kept;
        for (size_t l = 0; counts_whole && l < li; ++l, ++nc)
            if (new_counts && nc < counts_cap) new_counts[nc] = u->mrecs[o + l].new_count;
    }
    if (n_counts) *n_counts = nc;
    t->batch_recs = 0;   // (the records live in the sub-traversals)
    t->hrecs.clear();
    t->F = 0;
    t->expect_level = -1;
    t->has_q = t->has_bm = false;
    return ABFS_OK;
}

static int batch_impl(abfs_traversal *t, const int64_t *roots, size_t nroots,
                      const abfs_tree *tr, const double *static24, int64_t chunk,
                      uint64_t *levels, uint64_t *bfs_ns, uint64_t *total_ns,
                      uint64_t *checksums, uint64_t *new_counts, size_t counts_cap,
                      size_t *n_counts) {
    if (!t || !roots || !static24) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    if (nroots < 1 || nroots > kMaxBatch)
        return fail(ABFS_EINVAL, "need 1.." + std::to_string(kMaxBatch) + " roots per batch");
    ABFS_TRY(tree_ok(tr));
    ABFS_TRY(level_params_ok(0, 0, 0, chunk));
    std::vector<uint32_t> r32(nroots);
    for (size_t i = 0; i < nroots; ++i) {
        if (roots[i] < 0 || (uint64_t)roots[i] >= t->g->d.n)
            return fail(ABFS_EINVAL, "root " + std::to_string(roots[i]) + " out of range for |V|=" +
                                         std::to_string(t->g->d.n));
        r32[i] = (uint32_t)roots[i];
    }
    const int S = batch_ways(t, nroots);
    if (S > 1)
        return batch_split(t, r32, S, tr, static24, chunk, levels, bfs_ns, total_ns, checksums,
                           new_counts, counts_cap, n_counts);
    size_t nl = 0;
    ABFS_TRY(mega_run(t, r32.data(), nroots, false, -1, tr, static24, chunk, &nl, checksums));
    if (total_ns) *total_ns = t->last_trav_ns;
    size_t off = 0;
    for (size_t i = 0; i < nroots; ++i) {
        const size_t li = (size_t)t->batch_levels[i];
        if (levels) levels[i] = li;
        if (bfs_ns) {
            // t_bfs of root i: first level's start to last level's end
            uint64_t ns = 0;
            if (li && off + li <= t->batch_recs) {
                const MegaRecord &a = t->mrecs[off], &b = t->mrecs[off + li - 1];
                ns = b.t_end > a.t_start ? b.t_end - a.t_start : 1;
            }
            bfs_ns[i] = ns;
        }
        off += li;
    }
    if (n_counts) {
        // every root's per-level new counts, concatenated (records kept: the
        // first kMegaCap levels of the launch)
        const size_t k = std::min(t->batch_recs, counts_cap);
        for (size_t l = 0; new_counts && l < k; ++l) new_counts[l] = t->mrecs[l].new_count;
        *n_counts = t->batch_recs;
    }
    return ABFS_OK;
}

extern "C" int abfs_adaptive_bfs_batch(abfs_traversal *t, const int64_t *roots, size_t nroots,
                                       const abfs_tree *tr, const double *static24,
                                       int64_t chunk, uint64_t *levels, uint64_t *bfs_ns,
                                       uint64_t *total_ns) {
    if (!t) return fail(ABFS_EINVAL, "null traversal");
    ABFS_LOCK(t);
    return batch_impl(t, roots, nroots, tr, static24, chunk, levels, bfs_ns, total_ns, nullptr,
                      nullptr, 0, nullptr);
}

extern "C" int abfs_adaptive_bfs_batch_check(abfs_traversal *t, const int64_t *roots,
                                             size_t nroots, const abfs_tree *tr,
                                             const double *static24, int64_t chunk,
                                             uint64_t *levels, uint64_t *checksums,
                                             uint64_t *new_counts, size_t counts_cap,
                                             size_t *n_counts) {
    if (!t || !checksums) return fail(ABFS_EINVAL, "null argument");
    ABFS_LOCK(t);
    return batch_impl(t, roots, nroots, tr, static24, chunk, levels, nullptr, nullptr, checksums,
                      new_counts, counts_cap, n_counts);
}

#ifdef ABFS_DIAG_CTA
// diagnostic build only (tools/diag_cta.py): copy g_diag_cta out
extern "C" __attribute__((visibility("default"))) int abfs_debug_diag_cta(unsigned long long *out) {
    ABFS_CUDA(cudaMemcpyFromSymbol(out, abfs::g_diag_cta, sizeof(abfs::g_diag_cta)));
    static unsigned long long zeros[128 * 1024];
    ABFS_CUDA(cudaMemcpyToSymbol(abfs::g_diag_cta, zeros, sizeof(zeros)));   // clear for the next run
    return ABFS_OK;
}
#endif
