// partition.cu -- 1-D vertex-partitioned level-synchronous BFS.
//
// Rank p owns the contiguous destination range [lo, hi) (lo a multiple of
// 32, so its bitmap words [lo/32, ceil(hi/32)) are whole words) and holds:
//   * the destination-filtered out-CSR over ALL sources: for every u the
//     out-edges u -> v with v in [lo, hi) (a contiguous sub-range of u's sorted
//     adjacency, found by two binary searches) -- push / push-warp / edge-list;
//   * the in-CSR rows and reverse slots of its owned vertices -- pull /
//     rev-edge-list;
//   * owned depths, owned visited bitmap, and a REPLICATED global frontier
//     bitmap (V/8 bytes) plus a global frontier queue built from it.
// Per level: [bitmap -> queue if the strategy is top-down] -> the strategy
// kernels on the local slice (the same device functions as the single-GPU
// engine; depth/visited/bitmap pointers are rebased so they index by global
// id) -> a pack kernel writes the rank's next-frontier slice (visited bits
// gained this level) into the caller's send buffer.  The caller all-gathers
// the send buffers (NCCL over NVLink, or a device concat for partitions
// sharing one GPU) and abfs_part_exchange unpacks the padded slices into
// the global next-frontier bitmap, counting it with popc: every rank gets
// the same global count, hence the same features and the same tree choice.
//
// Semantics equal the single-GPU engine from init_depths (consistent state):
// each owned vertex is claimed by its owner only, exactly once.

#include <cub/cub.cuh>

#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "launch.cuh"
#include "megakernel.cuh"

using namespace abfs;


struct abfs_part {
    mutable std::recursive_mutex mu;   // per-handle lock
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t n = 0, lo = 0, hi = 0, wlo = 0, whi = 0, W = 0, nv = 0, nwl = 0, mf = 0, mr = 0;
    uint32_t *fo_off = nullptr, *fo_dst = nullptr, *fo_org = nullptr;   // filtered forward
    uint32_t *r_off = nullptr, *r_src = nullptr, *r_own = nullptr;      // owned reverse rows
    uint32_t *r_first = nullptr;                                         // first_src[lo, hi)
    int32_t *depth = nullptr;                                            // [nv]
    uint32_t *visited = nullptr, *vprev = nullptr, *noin = nullptr, *fnext = nullptr;  // [nwl]
    uint32_t *fbm[2] = {nullptr, nullptr};                               // global [W]
    uint32_t *q = nullptr;                                               // global frontier queue
    uint32_t *qn = nullptr;                                              // local discoveries
    uint2 *units = nullptr;
    Ctr *dctr = nullptr;
    Mailbox *dmb = nullptr;
    unsigned long long *dres = nullptr, *hres = nullptr;   // {global count, local count}
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int cur = 0;
    bool has_q = false;
    uint64_t F = 0;
    uint64_t call = 0;
    uint64_t launches = 0;
    int last_kernel = -1;
    int last_out = 0;
    // fused peer exchange (abfs_part_set_peers / abfs_part_ipc_open)
    PeerBox *box = nullptr;                      // this rank's mailbox (peers write it)
    uint32_t nranks = 0, rank = 0;
    uint32_t **peer_fbm = nullptr;               // device [2][nranks] bitmap pointers
    PeerBox **peer_box = nullptr;                // device [nranks] mailbox pointers
    unsigned int *pack_ticket = nullptr;         // last-CTA ticket of the push kernel
    unsigned long long p2p_seq = 0;              // launch-path exchanges done (every rank agrees)
    unsigned long long mk_seq = 0;               // megakernel exchanges done (PeerBox::mk_*)
    int x_sys = 1;                               // a peer buffer lives on another device
    std::vector<void *> ipc_opened;              // peer allocations mapped by IPC
    // persistent per-rank level loop (abfs_part_mega_*)
    uint32_t *q2 = nullptr;                      // second global-size queue
    MegaRecord *mrecs = nullptr, *drecs = nullptr;   // host staging / device records
    unsigned long long *mnlev = nullptr, *dnlev = nullptr;
    uint32_t *droots = nullptr;
    unsigned char *dtree = nullptr;
    size_t tree_cap = 0;
};

namespace {

constexpr int kMaxRanks = 64;

struct Bounds {
    uint64_t w[kMaxRanks + 1];   // global word bounds of the ranks' slices
    uint32_t P;
};

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *__restrict__ a, uint32_t b,
                                                    uint32_t e, uint32_t key) {
    while (b < e) {
        const uint32_t mid = b + ((e - b) >> 1);
        if (__ldg(a + mid) < key) b = mid + 1;
        else e = mid;
    }
    return b;
}

// Per source u: the filtered adjacency is dst[start[u] .. start[u]+cnt[u]).
__global__ void k_part_fcount(const uint32_t *__restrict__ out_off, const uint32_t *__restrict__ dst,
                              uint64_t n, uint32_t lo, uint32_t hi, uint32_t *cnt, uint32_t *start) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = __ldg(out_off + u), e = __ldg(out_off + u + 1);
        const uint32_t j0 = lower_bound_u32(dst, b, e, lo);
        const uint32_t j1 = lower_bound_u32(dst, j0, e, hi);
        cnt[u] = j1 - j0;
        start[u] = j0;
    }
}

// Edge-parallel copy of the filtered forward slots (keeps (origin, dest) order).
__global__ void k_part_fcopy(const uint32_t *__restrict__ org, const uint32_t *__restrict__ dst,
                             uint64_t m, const uint32_t *__restrict__ start,
                             const uint32_t *__restrict__ fo_off, uint32_t lo, uint32_t hi,
                             uint32_t *fo_dst, uint32_t *fo_org) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldg(dst + e);
        if (v < lo || v >= hi) continue;
        const uint32_t u = __ldg(org + e);
        const uint32_t pos = __ldg(fo_off + u) + (uint32_t)(e - __ldg(start + u));
        fo_dst[pos] = v;
        fo_org[pos] = u;
    }
}

__global__ void k_part_roff(const uint32_t *__restrict__ in_off, uint64_t lo, uint64_t nv,
                            uint32_t base, uint32_t *r_off) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nv;
         i += (uint64_t)gridDim.x * blockDim.x)
        r_off[i] = __ldg(in_off + lo + i) - base;
}

// Local in-degree-0 bitmap; padding bits (local index >= nv) set.
__global__ void k_part_noin(const uint32_t *__restrict__ r_off, uint64_t nv, uint64_t nwl,
                            uint32_t *noin) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nwl;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            const uint64_t i = k * 32 + b;
            if (i >= nv || r_off[i + 1] == r_off[i]) bits |= 1u << b;
        }
        noin[k] = bits;
    }
}

// init_depths (kernels.py:134-140) on the owned slice + global frontier {root}.
__global__ void k_part_init(int32_t *depth, uint64_t nv, uint32_t *visited, uint32_t *vprev,
                            uint64_t nwl, uint32_t *fbm, uint64_t W, uint32_t *q, uint64_t lo,
                            uint64_t hi, uint32_t root) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const bool owned = root >= lo && root < hi;
    for (uint64_t i = tid; i < nv; i += nt) depth[i] = (owned && i == root - lo) ? 0 : kInf;
    for (uint64_t k = tid; k < nwl; k += nt) {
        const uint32_t bits = (owned && k == (root - lo) >> 5) ? 1u << ((root - lo) & 31) : 0u;
        visited[k] = bits;
        vprev[k] = bits;
    }
    for (uint64_t w = tid; w < W; w += nt) fbm[w] = (w == (root >> 5)) ? 1u << (root & 31) : 0u;
    if (tid == 0) q[0] = root;
}

// Next-frontier slice = visited bits gained this level; padded to stride.
__global__ void k_part_pack(const uint32_t *__restrict__ visited, uint32_t *vprev, uint64_t nwl,
                            uint32_t *send, uint64_t stride) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < stride;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = 0;
        if (k < nwl) {
            const uint32_t v = visited[k];
            x = v & ~vprev[k];
            vprev[k] = v;
        }
        send[k] = x;
    }
}

// Gathered padded slices -> global next-frontier bitmap, popc -> count.
__global__ void __launch_bounds__(kBlock)
k_part_unpack(const uint32_t *__restrict__ gathered, Bounds b, uint64_t stride, uint32_t *fbm,
              uint64_t W, unsigned long long *res, const unsigned *qlen,
              const unsigned long long *count) {
    unsigned long long c = 0;
    uint32_t r = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W;
         w += (uint64_t)gridDim.x * blockDim.x) {
        while (r + 1 < b.P && w >= b.w[r + 1]) ++r;   // w only grows per thread
        const uint32_t x = __ldg(gathered + (uint64_t)r * stride + (w - b.w[r]));
        fbm[w] = x;
        c += __popc(x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(res, c);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        res[1] = qlen ? (unsigned long long)*qlen : *count;
}

// Fused exchange, sending side: the rank's next-frontier slice (visited bits
// gained this level) is stored straight into EVERY rank's global
// next-frontier bitmap over NVLink peer memory (own GPU included) -- no
// send buffer, no collective, no unpack.  The last CTA publishes the slice
// count into every rank's mailbox and signals arrival (system-scope atomics
// after a system fence, so the peers see the bitmap stores first).
__global__ void __launch_bounds__(kBlock)
k_part_push_peers(const uint32_t *__restrict__ visited, uint32_t *vprev, uint64_t nwl,
                  uint64_t wlo, uint32_t *const *peer_fbm, PeerBox *const *peer_box,
                  uint32_t nranks, uint32_t rank, int parity, PeerBox *mine,
                  unsigned int *ticket) {
    __shared__ unsigned long long part[kWarps];
    unsigned long long c = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nwl;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = visited[k];
        const uint32_t x = v & ~vprev[k];
        vprev[k] = v;
        for (uint32_t q = 0; q < nranks; ++q) peer_fbm[q][wlo + k] = x;
        c += __popc(x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < kWarps; ++w) s += part[w];
        if (s) atomicAdd(&mine->local, s);
        __threadfence_system();   // this CTA's peer stores before its ticket
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
            *ticket = 0;
            __threadfence_system();
            const unsigned long long tot = *(volatile unsigned long long *)&mine->local;
            mine->local = 0;
            for (uint32_t q = 0; q < nranks; ++q)
                *(volatile unsigned long long *)&peer_box[q]->counts[parity][rank] = tot;
            __threadfence_system();
            for (uint32_t q = 0; q < nranks; ++q) atomicAdd_system(&peer_box[q]->arrive, 1ull);
        }
    }
}

// Fused exchange, receiving side: wait until all ranks signalled this level
// (bounded: a rank that never arrives sets `timeout` instead of hanging the
// GPU), then sum the per-rank counts -> res = {global, this rank's}.
__global__ void k_part_p2p_wait(PeerBox *box, unsigned long long expect, uint32_t nranks,
                                uint32_t rank, int parity, unsigned long long *res) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long t0 = [] {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    }();
    for (;;) {
        if (*(volatile unsigned long long *)&box->arrive >= expect) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {   // 20 s
            box->timeout = 1;
            res[0] = ~0ull;
            return;
        }
        __nanosleep(200);
    }
    __threadfence_system();
    unsigned long long g = 0;
    for (uint32_t q = 0; q < nranks; ++q) g += *(volatile unsigned long long *)&box->counts[parity][q];
    res[0] = g;
    res[1] = *(volatile unsigned long long *)&box->counts[parity][rank];
}

}  // namespace

extern "C" void abfs_part_destroy(abfs_part *p) {
    if (!p) return;
    cudaSetDevice(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    void *dev[] = {p->fo_off, p->fo_dst, p->fo_org, p->r_off, p->r_src, p->r_own, p->r_first, p->depth,
                   p->visited, p->vprev, p->noin, p->fnext, p->fbm[0], p->fbm[1], p->q,
                   p->qn, p->units, p->dctr, p->dmb, p->dres};
    for (void *x : dev) cudaFree(x);
    for (void *x : p->ipc_opened) cudaIpcCloseMemHandle(x);
    cudaFree(p->box);
    cudaFree(p->q2);
    if (p->mrecs) cudaFreeHost(p->mrecs);
    cudaFree(p->drecs);
    if (p->mnlev) cudaFreeHost(p->mnlev);
    cudaFree(p->droots);
    cudaFree(p->dtree);
    cudaFree(p->peer_fbm);
    cudaFree(p->peer_box);
    cudaFree(p->pack_ticket);
    if (p->hres) cudaFreeHost(p->hres);
    if (p->e0) cudaEventDestroy(p->e0);
    if (p->e1) cudaEventDestroy(p->e1);
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
    delete p;
}

// Traversal state of a partition whose slice arrays are in place: owned
// depths / visited / in-degree-0 bitmaps, global frontier bitmaps and queue,
// counters and the peer mailbox.
static int part_alloc_state(abfs_part *p) {
    cudaStream_t s = p->stream;
    cudaError_t e = cudaSuccess;
    auto A = [&](void **ptr, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(ptr, bytes ? bytes : 4);
    };
    const uint64_t wpad = p->nwl + 4;
    A((void **)&p->depth, (p->nv + 4) * 4);
    A((void **)&p->visited, wpad * 4);
    A((void **)&p->vprev, wpad * 4);
    A((void **)&p->noin, wpad * 4);
    A((void **)&p->fnext, wpad * 4);
    A((void **)&p->fbm[0], (p->W + 4) * 4);
    A((void **)&p->fbm[1], (p->W + 4) * 4);
    A((void **)&p->q, (p->n + 4) * 4);
    A((void **)&p->qn, (p->nv + 4) * 4);
    const uint64_t mx = p->mf > p->mr ? p->mf : p->mr;
    A((void **)&p->units, (mx / kPushHub + 64) * sizeof(uint2));   // see traversal ucap
    A((void **)&p->dctr, sizeof(Ctr));
    A((void **)&p->dmb, sizeof(Mailbox));
    A((void **)&p->dres, 2 * sizeof(unsigned long long));
    static_assert(sizeof(PeerBox) <= kLLOffset, "LL planes overlap the mailbox");
    const size_t box_bytes = kLLOffset + 2 * (p->W + 4) * sizeof(unsigned long long);
    A((void **)&p->box, box_bytes);
    A((void **)&p->pack_ticket, sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemsetAsync(p->box, 0, box_bytes, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->pack_ticket, 0, sizeof(unsigned int), s);
    if (e == cudaSuccess) e = cudaMallocHost((void **)&p->hres, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(p->dctr, 0, sizeof(Ctr), s);
    if (e == cudaSuccess && p->nwl) {
        k_part_noin<<<grid_for(p->nwl, kBlock, 148 * 64), kBlock, 0, s>>>(p->r_off, p->nv, p->nwl, p->noin);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventCreate(&p->e0);
    if (e == cudaSuccess) e = cudaEventCreate(&p->e1);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error(std::string("part_create: ") + cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? ABFS_ENOMEM : ABFS_ECUDA;
    }
    return ABFS_OK;
}

static int part_new(int device, uint64_t n, uint64_t lo, uint64_t hi, abfs_part **out) {
    if (lo > hi || hi > n) return fail(ABFS_EINVAL, "partition range out of bounds");
    if (lo % 32) return fail(ABFS_EINVAL, "partition start must be a multiple of 32");
    if (hi % 32 && hi != n) return fail(ABFS_EINVAL, "partition end must be a multiple of 32 or |V|");
    ABFS_CUDA(cudaSetDevice(device));
    abfs_part *p = new abfs_part();
    p->device = device;
    p->n = n;
    p->lo = lo;
    p->hi = hi;
    p->nv = hi - lo;
    p->wlo = lo / 32;
    p->whi = (hi + 31) / 32;
    p->nwl = p->whi - p->wlo;
    p->W = (n + 31) / 32;
    const cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete p;
        return fail(ABFS_ECUDA, std::string("part_create: ") + cudaGetErrorString(e));
    }
    p->own_stream = true;
    *out = p;
    return ABFS_OK;
}

extern "C" int abfs_part_create(abfs_graph *g, uint64_t lo, uint64_t hi, abfs_part **out) {
    if (!g || !out) return fail(ABFS_EINVAL, "null argument");
    const uint64_t n = g->d.n, m = g->d.m;
    abfs_part *p = nullptr;
    ABFS_TRY(part_new(g->device, n, lo, hi, &p));
    cudaError_t e = cudaSuccess;
    cudaStream_t s = p->stream;
    auto A = [&](void **ptr, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(ptr, bytes ? bytes : 4);
    };
    // ---- forward slice: counts, offsets, copy ----------------------------
    uint32_t *cnt = nullptr, *start = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    A((void **)&cnt, (n + 1) * 4);
    A((void **)&start, (n + 1) * 4);
    A((void **)&p->fo_off, (n + 1) * 4);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt + n, 0, 4, s);
    if (e == cudaSuccess && n) {
        k_part_fcount<<<grid_for(n, kBlock, 148 * 64), kBlock, 0, s>>>(g->d.out_off, g->d.dst, n,
                                                                       (uint32_t)lo, (uint32_t)hi, cnt, start);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, p->fo_off, (int64_t)(n + 1), s);
    A(&tmp, tmp_bytes);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, p->fo_off, (int64_t)(n + 1), s);
    uint32_t mf = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&mf, p->fo_off + n, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    p->mf = mf;
    // +16 on every stream array: the edge kernels' bulk copies move whole
    // 16-byte groups (chunk_bytes rounds the last chunk up)
    A((void **)&p->fo_dst, (uint64_t)mf * 4 + 16);
    A((void **)&p->fo_org, (uint64_t)mf * 4 + 16);
    if (e == cudaSuccess && m) {
        k_part_fcopy<<<148 * 16, kBlock, 0, s>>>(g->d.org, g->d.dst, m, start, p->fo_off, (uint32_t)lo,
                                                 (uint32_t)hi, p->fo_dst, p->fo_org);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(cnt);
    cudaFree(start);
    cudaFree(tmp);
    // ---- reverse rows of the owned vertices (contiguous) -----------------
    uint32_t rb = 0, re = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&rb, g->d.in_off + lo, 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&re, g->d.in_off + hi, 4, cudaMemcpyDeviceToHost);
    p->mr = (uint64_t)re - rb;
    A((void **)&p->r_off, (p->nv + 1) * 4);
    A((void **)&p->r_src, p->mr * 4 + 16);   // +16: aligned 16-byte reads in pull
    A((void **)&p->r_own, p->mr * 4 + 16);
    A((void **)&p->r_first, p->nv * 4 + 16);
    if (e == cudaSuccess && p->nv)
        e = cudaMemcpyAsync(p->r_first, g->d.first_src + lo, p->nv * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && p->mr)
        e = cudaMemcpyAsync(p->r_src, g->d.src + rb, p->mr * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && p->mr)
        e = cudaMemcpyAsync(p->r_own, g->d.rev_owner + rb, p->mr * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) {
        k_part_roff<<<grid_for(p->nv + 1, kBlock, 148 * 64), kBlock, 0, s>>>(g->d.in_off, lo, p->nv, rb,
                                                                             p->r_off);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        set_error(std::string("part_create: ") + cudaGetErrorString(e));
        abfs_part_destroy(p);
        return e == cudaErrorMemoryAllocation ? ABFS_ENOMEM : ABFS_ECUDA;
    }
    const int rc = part_alloc_state(p);
    if (rc != ABFS_OK) {
        abfs_part_destroy(p);
        return rc;
    }
    *out = p;
    return ABFS_OK;
}

extern "C" int abfs_part_create_generated(int device, const abfs_gen_spec *spec, uint64_t lo,
                                          uint64_t hi, abfs_part **out) {
    if (!spec || !out) return fail(ABFS_EINVAL, "null argument");
    uint64_t n = 0;
    ABFS_TRY(abfs_gen_size(spec, &n, nullptr));
    abfs_part *p = nullptr;
    ABFS_TRY(part_new(device, n, lo, hi, &p));
    Slice sl;
    int rc = gen_slice(device, spec, lo, hi, sl, &n, p->stream);
    p->fo_off = sl.fo_off;
    p->fo_dst = sl.fo_dst;
    p->fo_org = sl.fo_org;
    p->r_off = sl.r_off;
    p->r_src = sl.r_src;
    p->r_own = sl.r_own;
    p->r_first = sl.r_first;
    p->mf = sl.mf;
    p->mr = sl.mr;
    if (rc == ABFS_OK) rc = part_alloc_state(p);
    if (rc != ABFS_OK) {
        abfs_part_destroy(p);
        return rc;
    }
    *out = p;
    return ABFS_OK;
}

extern "C" int abfs_part_download(const abfs_part *p, uint32_t *fo_off, uint32_t *fo_dst,
                                  uint32_t *fo_org, uint32_t *r_off, uint32_t *r_src,
                                  uint32_t *r_own, uint32_t *r_first) {
    if (!p) return fail(ABFS_EINVAL, "null partition");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    ABFS_CUDA(cudaSetDevice(p->device));
    ABFS_CUDA(cudaStreamSynchronize(p->stream));
    auto down = [&](uint32_t *h, const uint32_t *d, uint64_t cnt) -> cudaError_t {
        if (!h || !cnt) return cudaSuccess;
        return cudaMemcpy(h, d, cnt * 4, cudaMemcpyDeviceToHost);
    };
    ABFS_CUDA(down(fo_off, p->fo_off, p->n + 1));
    ABFS_CUDA(down(fo_dst, p->fo_dst, p->mf));
    ABFS_CUDA(down(fo_org, p->fo_org, p->mf));
    ABFS_CUDA(down(r_off, p->r_off, p->nv + 1));
    ABFS_CUDA(down(r_src, p->r_src, p->mr));
    ABFS_CUDA(down(r_own, p->r_own, p->mr));
    ABFS_CUDA(down(r_first, p->r_first, p->nv));
    return ABFS_OK;
}

extern "C" int abfs_part_info(const abfs_part *p, uint64_t *lo, uint64_t *hi, uint64_t *m_fwd,
                              uint64_t *m_rev) {
    if (!p) return fail(ABFS_EINVAL, "null partition");
    if (lo) *lo = p->lo;
    if (hi) *hi = p->hi;
    if (m_fwd) *m_fwd = p->mf;
    if (m_rev) *m_rev = p->mr;
    return ABFS_OK;
}

extern "C" int abfs_part_set_stream(abfs_part *p, void *stream) {
    if (!p) return fail(ABFS_EINVAL, "null partition");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    ABFS_CUDA(cudaSetDevice(p->device));
    ABFS_CUDA(cudaStreamSynchronize(p->stream));
    if (p->own_stream) cudaStreamDestroy(p->stream);
    // taken as given, NULL included (= the legacy default stream, which is
    // torch's default stream: the exchange must be ordered with torch ops)
    p->stream = (cudaStream_t)stream;
    p->own_stream = false;
    return ABFS_OK;
}

extern "C" int abfs_part_init(abfs_part *p, int64_t root) {
    if (!p) return fail(ABFS_EINVAL, "null partition");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (root < 0 || (uint64_t)root >= p->n)
        return fail(ABFS_EINVAL, "root " + std::to_string(root) + " out of range for |V|=" +
                                     std::to_string(p->n));
    ABFS_CUDA(cudaSetDevice(p->device));
    const uint64_t items = p->W > p->nv ? p->W : p->nv;
    k_part_init<<<grid_for(items, kBlock, 148 * 32), kBlock, 0, p->stream>>>(
        p->depth, p->nv, p->visited, p->vprev, p->nwl, p->fbm[0], p->W, p->q, p->lo, p->hi,
        (uint32_t)root);
    p->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaMemsetAsync(p->dctr, 0, sizeof(Ctr), p->stream));
    p->cur = 0;
    p->has_q = true;
    p->F = 1;
    return ABFS_OK;
}

static int part_strategy(abfs_part *p, int64_t level, int kernel, int variant, int64_t chunk) {
    ABFS_TRY(level_params_ok(level, kernel, variant, chunk));
    ABFS_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    ABFS_CUDA(cudaEventRecord(p->e0, s));
    const bool need_queue = (kernel == ABFS_VERTEX_PUSH || kernel == ABFS_VERTEX_PUSH_WARP);
    if (need_queue && !p->has_q) {
        k_bitmap_to_queue<<<grid_for(p->W, kBlock, 1ull << 31), kBlock, 0, s>>>(p->fbm[p->cur], p->W,
                                                                                p->q, &p->dctr->cq);
        p->launches += 1;
        p->has_q = true;
    }
    const int out = (int)(p->call % 3);
    const unsigned long long seq = ++p->call;
    LevelCtx c;
    c.acc = nullptr;
    c.depth = p->depth - p->lo;          // rebased: indexed by global id in [lo, hi)
    c.visited = p->visited - p->wlo;
    c.fbm = p->fbm[p->cur];
    c.q_next = p->qn;
    c.q_tail = &p->dctr->qlen[out];
    c.count = &p->dctr->count[out];
    c.units_tail = &p->dctr->units[out];
    c.units = p->units;
    c.inconsistent = &p->dctr->inconsistent;
    c.ctr = p->dctr;
    c.mb = p->dmb;
    c.es = nullptr;
    c.work = &p->dctr->work[out];
    c.pull_light = kPullLight;
    c.direct_claim = 0;
    c.seq = seq;
    c.zero_slot = (int)(seq % 3);
    c.level = (int32_t)level;
    c.lvl1 = (int32_t)(level + 1);
    StratArgs a;
    a.out_off = p->fo_off;
    a.dst = p->fo_dst;
    a.org = p->fo_org;
    a.m_fwd = p->mf;
    a.in_off = p->r_off - p->lo;
    a.src = p->r_src;
    a.rev_owner = p->r_own;
    a.m_rev = p->mr;
    a.first_src = p->r_first - p->lo;
    a.noin = p->noin - p->wlo;
    a.fbm_next = p->fnext - p->wlo;
    a.word0 = p->wlo;
    a.word_end = p->whi;
    a.q = p->q;
    a.F = (uint32_t)p->F;
    switch (variant) {
    case 0: p->launches += launch_strategy_args<0>(c, a, kernel, chunk, s); break;
    case 1: p->launches += launch_strategy_args<1>(c, a, kernel, chunk, s); break;
    default: p->launches += launch_strategy_args<2>(c, a, kernel, chunk, s); break;
    }
    ABFS_CUDA(cudaGetLastError());
    p->last_kernel = kernel;
    p->last_out = out;
    return ABFS_OK;
}

extern "C" int abfs_part_level(abfs_part *p, int64_t level, int kernel, int variant,
                               int64_t chunk, uint32_t *send, uint64_t stride) {
    if (!p || !send) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (stride < p->nwl) return fail(ABFS_EINVAL, "send stride smaller than the owned slice");
    ABFS_TRY(part_strategy(p, level, kernel, variant, chunk));
    k_part_pack<<<grid_for(stride, kBlock, 148 * 16), kBlock, 0, p->stream>>>(
        p->visited, p->vprev, p->nwl, send, stride);
    p->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    return ABFS_OK;
}

extern "C" int abfs_part_exchange(abfs_part *p, const uint32_t *gathered, const uint64_t *word_bounds,
                                  uint32_t nranks, uint64_t stride, uint64_t *global_count,
                                  uint64_t *local_count, uint64_t *elapsed_ns) {
    if (!p || !gathered || !word_bounds || !global_count) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (p->last_kernel < 0) return fail(ABFS_EINVAL, "exchange without a level");
    if (nranks < 1 || nranks > kMaxRanks) return fail(ABFS_EINVAL, "bad rank count");
    Bounds b;
    std::memset(&b, 0, sizeof(b));
    b.P = nranks;
    bool mine = false;
    for (uint32_t r = 0; r <= nranks; ++r) b.w[r] = word_bounds[r];
    for (uint32_t r = 0; r < nranks; ++r) {
        if (b.w[r] > b.w[r + 1] || b.w[r + 1] - b.w[r] > stride)
            return fail(ABFS_EINVAL, "bad word bounds / stride");
        mine |= b.w[r] == p->wlo && b.w[r + 1] == p->whi;
    }
    if (b.w[0] != 0 || b.w[nranks] != p->W || !mine)
        return fail(ABFS_EINVAL, "word bounds do not tile the bitmap around this partition");
    ABFS_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    ABFS_CUDA(cudaMemsetAsync(p->dres, 0, 2 * sizeof(unsigned long long), s));
    const bool topdown = p->last_kernel != ABFS_VERTEX_PULL;
    k_part_unpack<<<grid_for(p->W, kBlock, 148 * 8), kBlock, 0, s>>>(
        gathered, b, stride, p->fbm[p->cur ^ 1], p->W, p->dres,
        topdown ? &p->dctr->qlen[p->last_out] : nullptr, topdown ? nullptr : &p->dctr->count[p->last_out]);
    p->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaEventRecord(p->e1, s));
    ABFS_CUDA(cudaMemcpyAsync(p->hres, p->dres, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    ABFS_CUDA(cudaStreamSynchronize(s));
    *global_count = p->hres[0];
    if (local_count) *local_count = p->hres[1];
    if (elapsed_ns) {
        float ms = 0.f;
        ABFS_CUDA(cudaEventElapsedTime(&ms, p->e0, p->e1));
        const uint64_t ns = (uint64_t)((double)ms * 1e6 + 0.5);
        *elapsed_ns = ns ? ns : 1;
    }
    p->cur ^= 1;
    p->F = p->hres[0];
    p->has_q = false;
    p->last_kernel = -1;
    return ABFS_OK;
}

extern "C" int abfs_part_read_depths(abfs_part *p, int32_t *host_owned) {
    if (!p || !host_owned) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    ABFS_CUDA(cudaSetDevice(p->device));
    ABFS_CUDA(cudaMemcpyAsync(host_owned, p->depth, p->nv * 4, cudaMemcpyDeviceToHost, p->stream));
    ABFS_CUDA(cudaStreamSynchronize(p->stream));
    return ABFS_OK;
}

extern "C" int abfs_part_depths_device(abfs_part *p, int32_t *dev_out) {
    if (!p || !dev_out) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    ABFS_CUDA(cudaSetDevice(p->device));
    ABFS_CUDA(cudaMemcpyAsync(dev_out, p->depth, p->nv * 4, cudaMemcpyDeviceToDevice, p->stream));
    return ABFS_OK;
}

extern "C" int abfs_part_launches(const abfs_part *p, uint64_t *launches) {
    if (!p || !launches) return fail(ABFS_EINVAL, "null argument");
    *launches = p->launches;
    return ABFS_OK;
}

// ---- fused peer exchange ----------------------------------------------------

static int part_peers_common(abfs_part *p, uint32_t nranks, uint32_t rank,
                             const std::vector<uint32_t *> &f0, const std::vector<uint32_t *> &f1,
                             const std::vector<PeerBox *> &bx) {
    ABFS_CUDA(cudaSetDevice(p->device));
    std::vector<uint32_t *> tab(2 * (size_t)nranks);
    for (uint32_t q = 0; q < nranks; ++q) {
        tab[q] = f0[q];
        tab[nranks + q] = f1[q];
    }
    cudaFree(p->peer_fbm);
    cudaFree(p->peer_box);
    p->peer_fbm = nullptr;
    p->peer_box = nullptr;
    ABFS_CUDA(cudaMalloc((void **)&p->peer_fbm, tab.size() * sizeof(uint32_t *)));
    ABFS_CUDA(cudaMalloc((void **)&p->peer_box, nranks * sizeof(PeerBox *)));
    ABFS_CUDA(cudaMemcpy(p->peer_fbm, tab.data(), tab.size() * sizeof(uint32_t *), cudaMemcpyHostToDevice));
    ABFS_CUDA(cudaMemcpy(p->peer_box, bx.data(), nranks * sizeof(PeerBox *), cudaMemcpyHostToDevice));
    p->nranks = nranks;
    p->rank = rank;
    // every peer bitmap on this device (one process, or ranks sharing a GPU
    // through IPC): the exchange can synchronise at GPU scope
    int same = 1;
    for (uint32_t q = 0; q < nranks && same; ++q) {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, f0[q]) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
            pa.device != p->device)
            same = 0;
    }
    cudaGetLastError();
    p->x_sys = same ? 0 : 1;
    return ABFS_OK;
}

extern "C" int abfs_part_peer_buffers(abfs_part *p, void **fbm0, void **fbm1, void **mailbox) {
    if (!p || !fbm0 || !fbm1 || !mailbox) return fail(ABFS_EINVAL, "null argument");
    *fbm0 = p->fbm[0];
    *fbm1 = p->fbm[1];
    *mailbox = p->box;
    return ABFS_OK;
}

extern "C" int abfs_part_set_peers(abfs_part *p, void *const *fbm0, void *const *fbm1,
                                   void *const *mailboxes, uint32_t nranks, uint32_t rank) {
    if (!p || !fbm0 || !fbm1 || !mailboxes) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (nranks < 1 || nranks > kMaxRanks || rank >= nranks) return fail(ABFS_EINVAL, "bad rank count");
    if (fbm0[rank] != p->fbm[0] || fbm1[rank] != p->fbm[1] || mailboxes[rank] != p->box)
        return fail(ABFS_EINVAL, "own buffers must sit at this rank's slot");
    std::vector<uint32_t *> f0(nranks), f1(nranks);
    std::vector<PeerBox *> bx(nranks);
    for (uint32_t q = 0; q < nranks; ++q) {
        f0[q] = (uint32_t *)fbm0[q];
        f1[q] = (uint32_t *)fbm1[q];
        bx[q] = (PeerBox *)mailboxes[q];
    }
    return part_peers_common(p, nranks, rank, f0, f1, bx);
}

extern "C" int abfs_part_ipc_export(abfs_part *p, unsigned char *handles) {
    if (!p || !handles) return fail(ABFS_EINVAL, "null argument");
    ABFS_CUDA(cudaSetDevice(p->device));
    cudaIpcMemHandle_t h[3];
    ABFS_CUDA(cudaIpcGetMemHandle(&h[0], p->fbm[0]));
    ABFS_CUDA(cudaIpcGetMemHandle(&h[1], p->fbm[1]));
    ABFS_CUDA(cudaIpcGetMemHandle(&h[2], p->box));
    std::memcpy(handles, h, sizeof(h));
    return ABFS_OK;
}

extern "C" int abfs_part_ipc_open(abfs_part *p, const unsigned char *all_handles, uint32_t nranks,
                                  uint32_t rank) {
    if (!p || !all_handles) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (nranks < 1 || nranks > kMaxRanks || rank >= nranks) return fail(ABFS_EINVAL, "bad rank count");
    ABFS_CUDA(cudaSetDevice(p->device));
    std::vector<uint32_t *> f0(nranks), f1(nranks);
    std::vector<PeerBox *> bx(nranks);
    for (uint32_t q = 0; q < nranks; ++q) {
        if (q == rank) {
            f0[q] = p->fbm[0];
            f1[q] = p->fbm[1];
            bx[q] = p->box;
            continue;
        }
        cudaIpcMemHandle_t h[3];
        std::memcpy(h, all_handles + (size_t)q * 3 * sizeof(cudaIpcMemHandle_t), sizeof(h));
        void *ptr[3];
        for (int k = 0; k < 3; ++k) {
            ABFS_CUDA(cudaIpcOpenMemHandle(&ptr[k], h[k], cudaIpcMemLazyEnablePeerAccess));
            p->ipc_opened.push_back(ptr[k]);
        }
        f0[q] = (uint32_t *)ptr[0];
        f1[q] = (uint32_t *)ptr[1];
        bx[q] = (PeerBox *)ptr[2];
    }
    return part_peers_common(p, nranks, rank, f0, f1, bx);
}

extern "C" int abfs_part_level_p2p(abfs_part *p, int64_t level, int kernel, int variant,
                                   int64_t chunk) {
    if (!p) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (!p->nranks) return fail(ABFS_EINVAL, "peers not set (abfs_part_set_peers / abfs_part_ipc_open)");
    ABFS_TRY(part_strategy(p, level, kernel, variant, chunk));
    const int parity = (int)(p->p2p_seq & 1);
    uint32_t *const *fbm_next = p->peer_fbm + (size_t)(p->cur ^ 1) * p->nranks;
    k_part_push_peers<<<grid_for(p->nwl, kBlock, 148 * 4), kBlock, 0, p->stream>>>(
        p->visited, p->vprev, p->nwl, p->wlo, fbm_next, p->peer_box, p->nranks, p->rank, parity,
        p->box, p->pack_ticket);
    p->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    return ABFS_OK;
}

extern "C" int abfs_part_p2p_finish(abfs_part *p, uint64_t *global_count, uint64_t *local_count,
                                    uint64_t *elapsed_ns) {
    if (!p || !global_count) return fail(ABFS_EINVAL, "null argument");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (p->last_kernel < 0) return fail(ABFS_EINVAL, "finish without a level");
    ABFS_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const int parity = (int)(p->p2p_seq & 1);
    ++p->p2p_seq;
    k_part_p2p_wait<<<1, 32, 0, s>>>(p->box, p->p2p_seq * p->nranks, p->nranks, p->rank, parity,
                                     p->dres);
    p->launches += 1;
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaEventRecord(p->e1, s));
    ABFS_CUDA(cudaMemcpyAsync(p->hres, p->dres, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    ABFS_CUDA(cudaStreamSynchronize(s));
    if (p->hres[0] == ~0ull)
        return fail(ABFS_ENCCL, "peer exchange timed out (a rank never signalled this level)");
    *global_count = p->hres[0];
    if (local_count) *local_count = p->hres[1];
    if (elapsed_ns) {
        float ms = 0.f;
        ABFS_CUDA(cudaEventElapsedTime(&ms, p->e0, p->e1));
        const uint64_t ns = (uint64_t)((double)ms * 1e6 + 0.5);
        *elapsed_ns = ns ? ns : 1;
    }
    p->cur ^= 1;
    p->F = p->hres[0];
    p->has_q = false;
    p->last_kernel = -1;
    return ABFS_OK;
}

// ---- whole traversals over fused-exchange partitions (no host per level) --

// adaptive_bfs (adaptive.py:83-129) / bfs_full (kernels.py:356-371) driven in
// C over the partitions this process owns: per level every partition's
// strategy + peer push is enqueued, then every partition's device wait; the
// tree is evaluated on the reference's float64 features between levels.
static int parts_traverse(abfs_part *const *parts, uint32_t nparts, int64_t root,
                          const abfs_tree *tr, const double *static24, int fixed_pair,
                          int64_t chunk, abfs_level_record *recs, uint64_t *local_counts,
                          size_t cap, size_t *n_levels) {
    if (!parts || !nparts || !n_levels) return fail(ABFS_EINVAL, "null argument");
    for (uint32_t i = 0; i < nparts; ++i) {
        if (!parts[i]) return fail(ABFS_EINVAL, "null partition");
        if (!parts[i]->nranks)
            return fail(ABFS_EINVAL, "peers not set (abfs_part_set_peers / abfs_part_ipc_open)");
        ABFS_TRY(abfs_part_init(parts[i], root));
    }
    uint64_t frontier = 1, discovered = 1;
    int pk = ABFS_EDGE_LIST, pv = ABFS_DIRECT_ATOMIC;   // DEFAULT_KERNEL adaptive.py:36-38
    std::vector<double> canon(ABFS_N_FEATURES), proj(tr ? tr->n_selection : 0);
    for (int64_t level = 0;; ++level) {
        int fallback = 0;
        if (fixed_pair >= 0) {
            pk = fixed_pair / 3;
            pv = fixed_pair % 3;
        } else {
            ABFS_TRY(abfs_features(static24, frontier, discovered, canon.data()));
            for (uint32_t k = 0; k < tr->n_selection; ++k) proj[k] = canon[tr->selection[k]];
            int cls = 0;
            ABFS_TRY(abfs_tree_predict(tr, proj.data(), &cls));
            fallback = cls == ABFS_LEAF_UNKNOWN;
            if (!fallback) {
                pk = cls / 3;
                pv = cls % 3;
            }
        }
        for (uint32_t i = 0; i < nparts; ++i) ABFS_TRY(abfs_part_level_p2p(parts[i], level, pk, pv, chunk));
        uint64_t g = 0, ns = 0;
        for (uint32_t i = 0; i < nparts; ++i) {
            uint64_t gi = 0, li = 0, nsi = 0;
            ABFS_TRY(abfs_part_p2p_finish(parts[i], &gi, &li, &nsi));
            if (i && gi != g) return fail(ABFS_ENCCL, "partitions disagree on the level count");
            g = gi;
            if (local_counts && (size_t)level < cap) local_counts[(size_t)level * nparts + i] = li;
            ns = nsi > ns ? nsi : ns;
        }
        if (recs && (size_t)level < cap) {
            abfs_level_record &r = recs[level];
            r.level = level;
            r.kernel = pk;
            r.variant = pv;
            r.fallback = fallback;
            r.converted = 0;
            r.frontier_size = frontier;
            r.new_count = g;
            r.elapsed_ns = ns;
            r.prediction_ns = 1;
            r.unvisited = parts[0]->n - (discovered + g);
            r.next_out_edges = ~0ull;
        }
        if (g == 0) {
            *n_levels = (size_t)level + 1;
            return ABFS_OK;
        }
        frontier = g;
        discovered += g;
    }
}

extern "C" int abfs_parts_adaptive_bfs(abfs_part *const *parts, uint32_t nparts, int64_t root,
                                       const abfs_tree *tree, const double *static24,
                                       int64_t chunk_size, abfs_level_record *records,
                                       uint64_t *local_counts, size_t cap, size_t *n_levels) {
    if (!tree || !static24) return fail(ABFS_EINVAL, "null argument");
    return parts_traverse(parts, nparts, root, tree, static24, -1, chunk_size, records,
                          local_counts, cap, n_levels);
}

extern "C" int abfs_parts_bfs_full(abfs_part *const *parts, uint32_t nparts, int64_t root,
                                   int kernel, int variant, int64_t chunk_size,
                                   abfs_level_record *records, uint64_t *local_counts, size_t cap,
                                   size_t *n_levels) {
    ABFS_TRY(level_params_ok(0, kernel, variant, chunk_size));
    return parts_traverse(parts, nparts, root, nullptr, nullptr, kernel * 3 + variant, chunk_size,
                          records, local_counts, cap, n_levels);
}

// ---- persistent per-rank level loop ------------------------------------------

// One whole traversal of this rank inside the persistent megakernel
// (megakernel.cuh, part = 1): levels, tree decisions and the fused exchange
// (peer stores + mailbox wait) all on the device; one launch, one sync.
static int part_mega(abfs_part *p, int64_t root, const abfs_tree *tr, const double *static24,
                     int fixed_pair, int64_t chunk, abfs_level_record *recs,
                     uint64_t *local_counts, size_t cap, size_t *n_levels) {
    if (!p || !n_levels) return fail(ABFS_EINVAL, "null argument");
    if (!p->nranks) return fail(ABFS_EINVAL, "peers not set (abfs_part_set_peers / abfs_part_ipc_open)");
    std::lock_guard<std::recursive_mutex> _abfs_guard(p->mu);
    if (root < 0 || (uint64_t)root >= p->n)
        return fail(ABFS_EINVAL, "root " + std::to_string(root) + " out of range for |V|=" +
                                     std::to_string(p->n));
    ABFS_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    if (!p->mrecs) {
        ABFS_CUDA(cudaMalloc(&p->q2, (p->n + 4) * 4));
        // records in device memory, copied back after the launch: a level's
        // system-scope exchange release would otherwise wait on the lead's
        // PCIe record writes to mapped host memory
        ABFS_CUDA(cudaMallocHost((void **)&p->mrecs, kMegaCapPart * sizeof(MegaRecord)));
        ABFS_CUDA(cudaMalloc((void **)&p->drecs, kMegaCapPart * sizeof(MegaRecord)));
        ABFS_CUDA(cudaHostAlloc((void **)&p->mnlev, sizeof(unsigned long long), cudaHostAllocMapped));
        ABFS_CUDA(cudaHostGetDevicePointer((void **)&p->dnlev, p->mnlev, 0));
        ABFS_CUDA(cudaMalloc(&p->droots, 16));
    }
    std::vector<unsigned char> blob;
    uint32_t nn = 0;
    stage_cut_tree(tr, static24, p->n, blob, nn);
    if (blob.size() > p->tree_cap) {
        cudaFree(p->dtree);
        p->dtree = nullptr;
        ABFS_CUDA(cudaMalloc(&p->dtree, blob.size()));
        p->tree_cap = blob.size();
    }
    ABFS_CUDA(cudaMemcpy(p->dtree, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    const uint32_t r32 = (uint32_t)root;
    ABFS_CUDA(cudaMemcpy(p->droots, &r32, 4, cudaMemcpyHostToDevice));
    ABFS_CUDA(cudaMemsetAsync(p->dctr, 0, sizeof(Ctr), s));
    ABFS_CUDA(cudaMemsetAsync(&p->box->timeout, 0, sizeof(unsigned int), s));
    MegaParams P{};   // value-initialised: every optional pointer starts null
    std::memset(&P, 0, sizeof(P));
    P.depth = p->depth - p->lo;
    P.visited = p->visited - p->wlo;
    P.noin = p->noin - p->wlo;
    P.fbm0 = p->fbm[0];
    P.fbm1 = p->fbm[1];
    P.q0 = p->q;
    P.q1 = p->q2;
    P.units = p->units;
    P.ctr = p->dctr;
    P.out_off = p->fo_off;
    P.dst = p->fo_dst;
    P.org = p->fo_org;
    P.in_off = p->r_off - p->lo;
    P.src = p->r_src;
    P.rev_owner = p->r_own;
    P.first_src = p->r_first - p->lo;
    P.n = p->n;
    P.m = p->mf;
    P.words = p->W;
    P.tree = p->dtree;
    P.tree_nodes = nn;
    P.fixed_pair = fixed_pair;
    P.vw_log2 = chunk >= 32 ? 5 : chunk >= 16 ? 4 : chunk >= 8 ? 3 : chunk >= 4 ? 2 : chunk >= 2 ? 1 : 0;
    P.vw_wide_log2 = P.vw_log2;
    P.vw_wide_f = 0;
    P.instrument = 0;
    P.pull_light = kPullLight;
    P.cap = kMegaCapPart;
    P.recs = p->drecs;
    P.n_levels = p->dnlev;
    P.roots = p->droots;
    P.nroots = 1;
    P.init_in_kernel = 1;
    P.solo_ctas = 0;
    P.solo = nullptr;
    P.part = 1;
    P.m_rev = p->mr;
    P.lo = p->lo;
    P.hi = p->hi;
    P.wlo = p->wlo;
    P.wend = p->whi;
    P.vprev = p->vprev;
    P.fnext = p->fnext - p->wlo;
    P.peer_fbm = p->peer_fbm;
    P.peer_box = p->peer_box;
    P.box = p->box;
    P.nranks = p->nranks;
    P.rank = p->rank;
    P.xseq0 = p->mk_seq;
    {
        // cross-device ranks: LL exchange (no system-scope fence per level);
        // same device: GPU-scoped release / acquire.  ABFS_XSYS=0/1/2 forces
        // GPU scope / system scope / LL (tests)
        const char *xs = getenv("ABFS_XSYS");
        P.xsys = xs ? atoi(xs) : (p->x_sys ? 2 : 0);
    }
    P.checksums = nullptr;
    P.acc = nullptr;   // RED-mode levels are single-graph only
    *(volatile unsigned long long *)p->mnlev = 0;
    {
        std::lock_guard<std::mutex> mega_guard(mega_mutex(p->device));
        ABFS_CUDA(cudaEventRecord(p->e0, s));
        ABFS_TRY(mega_launch_plain(P, s, p->device));
        p->launches += 1;
        ABFS_CUDA(cudaEventRecord(p->e1, s));
        ABFS_CUDA(cudaStreamSynchronize(s));
    }
    const unsigned long long nl = *(volatile unsigned long long *)p->mnlev;
    p->mk_seq += nl;
    ABFS_CUDA(cudaMemcpy(p->mrecs, p->drecs,
                         (size_t)std::min<unsigned long long>(nl, kMegaCapPart) * sizeof(MegaRecord),
                         cudaMemcpyDeviceToHost));
    p->last_kernel = -1;
    p->has_q = false;
    int timed_out = 0;
    ABFS_CUDA(cudaMemcpy(&timed_out, &p->box->timeout, sizeof(int), cudaMemcpyDeviceToHost));
    if (timed_out) return fail(ABFS_ENCCL, "peer exchange timed out (a rank never signalled a level)");
    const size_t keep = nl < kMegaCapPart ? (size_t)nl : kMegaCapPart;
    if ((recs || local_counts) && nl > keep && cap > keep) {
        // more levels than the persistent loop keeps records for: redo the
        // traversal with the host-driven fused-exchange loop, which records
        // every level (nl is global, so every rank takes this branch)
        abfs_part *const one[1] = {p};
        return parts_traverse(one, 1, root, tr, static24, fixed_pair, chunk, recs, local_counts,
                              cap, n_levels);
    }
    uint64_t disc = 1;
    for (size_t l = 0; recs && l < keep && l < cap; ++l) {
        const MegaRecord &m = p->mrecs[l];
        abfs_level_record &r = recs[l];
        disc += m.new_count;
        r.unvisited = p->n - disc;
        r.next_out_edges = ~0ull;
        r.level = (int64_t)l;
        r.kernel = m.kernel;
        r.variant = m.variant;
        r.fallback = m.fallback;
        r.converted = m.converted;
        r.frontier_size = m.frontier;
        r.new_count = m.new_count;
        const uint64_t d = m.t_end > m.t_start ? m.t_end - m.t_start : 0;
        r.elapsed_ns = d ? d : 1;
        const uint64_t pn = m.t_pred > m.t_start ? m.t_pred - m.t_start : 0;
        r.prediction_ns = pn ? pn : 1;
    }
    if (local_counts)
        for (size_t l = 0; l < keep && l < cap; ++l) local_counts[l] = p->mrecs[l].scanned;
    *n_levels = (size_t)nl;
    return ABFS_OK;
}

extern "C" int abfs_part_mega_adaptive_bfs(abfs_part *p, int64_t root, const abfs_tree *tree,
                                           const double *static24, int64_t chunk_size,
                                           abfs_level_record *records, uint64_t *local_counts,
                                           size_t cap, size_t *n_levels) {
    if (!tree || !static24) return fail(ABFS_EINVAL, "null argument");
    ABFS_TRY(level_params_ok(0, 0, 0, chunk_size));
    return part_mega(p, root, tree, static24, -1, chunk_size, records, local_counts, cap, n_levels);
}

extern "C" int abfs_part_mega_bfs_full(abfs_part *p, int64_t root, int kernel, int variant,
                                       int64_t chunk_size, abfs_level_record *records,
                                       uint64_t *local_counts, size_t cap, size_t *n_levels) {
    ABFS_TRY(level_params_ok(0, kernel, variant, chunk_size));
    return part_mega(p, root, nullptr, nullptr, kernel * 3 + variant, chunk_size, records,
                     local_counts, cap, n_levels);
}
