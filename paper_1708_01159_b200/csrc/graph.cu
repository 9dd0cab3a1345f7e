// graph.cu -- device-resident combined representation: upload, device
// build_combined (graph.py:93-134) and bit-exact device generators
// (generate_graph, graph.py:211-252) for the K24/K26/ER/mesh configs.
//
// build_combined on the device: pack each edge as a 64-bit key
// (src << 32 | dst) and radix-sort it (CUB) -> forward CSR order
// (lexsort by (src, dst)); pack (dst << 32 | src) and sort -> reverse order
// (lexsort by (dst, src)) whose high words are rev_owner for free.  Offsets
// come from a boundary pass over the sorted high words.
//
// Generators reproduce numpy's PCG64 stream (state = state*M + inc, XSL-RR
// output) with jump-ahead, so a thread can start anywhere in the stream:
//   rmat-like:  draw index bit*m + i for edge i at bit level `bit`,
//               random() = (x >> 11) * 2^-53 compared against the cumulative
//               quadrant probabilities (compared exactly as integers
//               k >= ceil(t * 2^53));
//   uniform:    u32 half-words low-then-high, src = u32[0:m],
//               dst = u32[m:2m], value = u32 * n >> 32 (n a power of two:
//               Lemire's rejection never fires).

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"

using namespace abfs;

namespace {

typedef unsigned __int128 u128;

__host__ __device__ inline u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64 - r) & 63));
}

// Affine map of `delta` LCG steps: s -> A*s + C.
__host__ __device__ inline void pcg_jump(u128 inc, u128 delta, u128 &A, u128 &C) {
    u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    A = am;
    C = ap;
}

struct RmatParams {
    u128 s0, inc;
    uint64_t m;
    uint64_t t1, t2, t3;   // integer thresholds ceil(a*2^53), ceil((a+b)*2^53), ...
    uint32_t scale;
    u128 bitA[64], bitC[64];  // jump from stream position i to bit*m + i
    int symmetrize;
};

constexpr int kGenChunk = 16;

// The scale-bit draws of edges [i0, i0 + cnt) (cnt <= kGenChunk).
__device__ __forceinline__ void rmat_pairs(const RmatParams &p, uint64_t i0, int cnt,
                                           uint32_t (&src)[kGenChunk], uint32_t (&dst)[kGenChunk]) {
    u128 A, C;
    pcg_jump(p.inc, (u128)i0, A, C);
    const u128 base = A * p.s0 + C;  // state before draw i0 at bit 0
#pragma unroll
    for (int k = 0; k < kGenChunk; ++k) src[k] = dst[k] = 0;
    const u128 M = pcg_mult();
    for (uint32_t bit = 0; bit < p.scale; ++bit) {
        u128 s = p.bitA[bit] * base + p.bitC[bit];
#pragma unroll
        for (int k = 0; k < kGenChunk; ++k) {
            if (k < cnt) {
                s = s * M + p.inc;
                const uint64_t r = pcg_out(s) >> 11;
                const uint32_t sb = r >= p.t2;
                const uint32_t db = (r >= p.t1 && r < p.t2) || r >= p.t3;
                src[k] = (src[k] << 1) | sb;
                dst[k] = (dst[k] << 1) | db;
            }
        }
    }
}

__global__ void k_gen_rmat(const RmatParams *__restrict__ P, uint64_t *keys_fwd) {
    const RmatParams &p = *P;
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kGenChunk;
    if (i0 >= p.m) return;
    const int cnt = (int)min((uint64_t)kGenChunk, p.m - i0);
    uint32_t src[kGenChunk], dst[kGenChunk];
    rmat_pairs(p, i0, cnt, src, dst);
    if (p.symmetrize & 2) {
        // Graph500-style relabelling: an odd-multiplier affine map is a
        // bijection of [0, 2^scale), so hubs no longer sit at low ids
        const uint32_t mask = (uint32_t)((1ull << p.scale) - 1);
        for (int k = 0; k < cnt; ++k) {
            src[k] = (src[k] * 0x9E3779B1u + 0x7F4A7C15u) & mask;
            dst[k] = (dst[k] * 0x9E3779B1u + 0x7F4A7C15u) & mask;
        }
    }
    for (int k = 0; k < cnt; ++k) {
        keys_fwd[i0 + k] = ((uint64_t)src[k] << 32) | dst[k];
        if (p.symmetrize & 1) keys_fwd[p.m + i0 + k] = ((uint64_t)dst[k] << 32) | src[k];
    }
}

struct UniParams {
    u128 s0, inc;
    uint64_t n_log2, m;
};

// u64 draw k yields u32 stream positions 2k (low) and 2k+1 (high).
__global__ void k_gen_uniform(UniParams p, uint64_t *keys) {
    const uint64_t k0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kGenChunk;
    const uint64_t draws = p.m;  // 2m half-words
    if (k0 >= draws) return;
    u128 A, C;
    pcg_jump(p.inc, (u128)k0, A, C);
    u128 s = A * p.s0 + C;
    const u128 M = pcg_mult();
    const uint64_t cnt = min((uint64_t)kGenChunk, draws - k0);
    uint32_t *key32 = reinterpret_cast<uint32_t *>(keys);  // little-endian: [2i]=lo(dst), [2i+1]=hi(src)
    for (uint64_t k = 0; k < cnt; ++k) {
        s = s * M + p.inc;
        const uint64_t o = pcg_out(s);
        const uint64_t j0 = 2 * (k0 + k);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint64_t j = j0 + h;
            const uint64_t u = h ? (o >> 32) : (o & 0xffffffffull);
            const uint32_t val = (uint32_t)((u << p.n_log2) >> 32);
            if (j < p.m) key32[2 * j + 1] = val;           // src -> high word
            else key32[2 * (j - p.m)] = val;               // dst -> low word
        }
    }
}

__global__ void k_gen_mesh(uint32_t rows, uint32_t cols, uint64_t *keys, unsigned long long *cursor) {
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t n = (uint64_t)rows * cols;
    if (v >= n) return;
    const uint32_t r = (uint32_t)(v / cols), c = (uint32_t)(v % cols);
    uint64_t nb[4];
    int k = 0;
    if (r > 0) nb[k++] = v - cols;
    if (c > 0) nb[k++] = v - 1;
    if (c + 1 < cols) nb[k++] = v + 1;
    if (r + 1 < rows) nb[k++] = v + cols;
    if (!k) return;
    const unsigned long long p = atomicAdd(cursor, (unsigned long long)k);
    for (int i = 0; i < k; ++i) keys[p + i] = (v << 32) | nb[i];
}

__global__ void k_pack_pairs(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                             uint64_t m, uint64_t *keys) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = ((uint64_t)a[i] << 32) | b[i];
}

// Split sorted keys into (hi, lo) arrays and write CSR offsets: off[v] is the
// first index whose hi >= v (boundary pass, O(m + n)).
__global__ void k_split_offsets(const uint64_t *__restrict__ keys, uint64_t m, uint64_t n,
                                uint32_t *hi_out, uint32_t *lo_out, uint32_t *off) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t cur = i < m ? (keys[i] >> 32) : n;
        const int64_t prev = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
        if (i < m) {
            if (hi_out) hi_out[i] = (uint32_t)(keys[i] >> 32);
            lo_out[i] = (uint32_t)keys[i];
        }
        for (int64_t v = prev + 1; v <= (int64_t)cur && v <= (int64_t)n; ++v) off[v] = (uint32_t)i;
    }
}

// rev_owner from in_offsets (upload path): binary search per slot.
__global__ void k_rev_owner(const uint32_t *__restrict__ in_off, uint64_t n, uint64_t m,
                            uint32_t *owner) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n;  // last v with in_off[v] <= e
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (in_off[mid] <= e) lo = mid;
            else hi = mid;
        }
        owner[e] = (uint32_t)lo;
    }
}

inline unsigned grid_cap(uint64_t items, unsigned block, uint64_t cap = 148ull * 64) {
    uint64_t b = (items + block - 1) / block;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

int bits_for(uint64_t n) {
    int b = 0;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

// Sort `keys` (m entries, significant bits: 32 + vbits) with CUB; result in
// *keys_io (may swap with alt).
int sort_keys(uint64_t *&keys, uint64_t *&alt, uint64_t m, int vbits, cudaStream_t s) {
    if (m == 0) return ABFS_OK;
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t tmp = 0;
    ABFS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)m, 0, 32 + vbits, s));
    void *dtmp = nullptr;
    ABFS_CUDA(cudaMallocAsync(&dtmp, tmp, s));
    // Low word holds the minor key; sort all of it plus the used high bits.
    cudaError_t e = cub::DeviceRadixSort::SortKeys(dtmp, tmp, db, (int64_t)m, 0, 32 + vbits, s);
    cudaFreeAsync(dtmp, s);
    if (e != cudaSuccess) return fail(ABFS_ECUDA, std::string("radix sort: ") + cudaGetErrorString(e));
    if (db.Current() != keys) std::swap(keys, alt);
    return ABFS_OK;
}

// keys: forward-packed (src<<32|dst), m entries, device; consumed.
int build_from_keys(abfs_graph *g, uint64_t *keys, uint64_t *alt, cudaStream_t s) {
    DevGraph &d = g->d;
    const uint64_t n = d.n, m = d.m;
    const int vb = bits_for(n);
    ABFS_TRY(sort_keys(keys, alt, m, vb, s));
    k_split_offsets<<<grid_cap(m + 1, 256), 256, 0, s>>>(keys, m, n, d.org, d.dst, d.out_off);
    ABFS_CUDA(cudaGetLastError());
    // reverse: (dst << 32 | src) from the forward arrays
    k_pack_pairs<<<grid_cap(m, 256), 256, 0, s>>>(d.dst, d.org, m, keys);
    ABFS_CUDA(cudaGetLastError());
    ABFS_TRY(sort_keys(keys, alt, m, vb, s));
    k_split_offsets<<<grid_cap(m + 1, 256), 256, 0, s>>>(keys, m, n, d.rev_owner, d.src, d.in_off);
    ABFS_CUDA(cudaGetLastError());
    ABFS_CUDA(cudaStreamSynchronize(s));
    return ABFS_OK;
}

struct KeyBufs {
    uint64_t *a = nullptr, *b = nullptr;
    ~KeyBufs() {
        cudaFree(a);
        cudaFree(b);
    }
};

int new_graph(int device, uint64_t n, uint64_t m, abfs_graph **out) {
    if (!out) return fail(ABFS_EINVAL, "null output");
    if (n >= (1ull << 32)) return fail(ABFS_EINVAL, "vertex_count must be < 2^32");
    if (m >= (1ull << 32)) return fail(ABFS_EINVAL, "edge_count must be < 2^32 (u32 offsets)");
    ABFS_CUDA(cudaSetDevice(device));
    abfs_graph *g = new abfs_graph();
    g->device = device;
    int rc = graph_alloc(g, n, m);
    if (rc) {
        delete g;
        return rc;
    }
    *out = g;
    return ABFS_OK;
}

__global__ void k_first_src(const uint32_t *__restrict__ in_off, const uint32_t *__restrict__ src,
                            uint64_t n, uint32_t *first_src) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = in_off[v], e = in_off[v + 1];
        first_src[v] = b < e ? src[b] : 0u;
    }
}

int finish_build(int rc, abfs_graph *g, abfs_graph **out) {
    if (rc == ABFS_OK && g->d.n) {
        k_first_src<<<grid_cap(g->d.n, 256), 256>>>(g->d.in_off, g->d.src, g->d.n, g->d.first_src);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("first_src: ") + cudaGetErrorString(e));
    }
    if (rc != ABFS_OK) {
        abfs_graph_destroy(g);
        *out = nullptr;
    }
    return rc;
}

}  // namespace

namespace abfs {

int graph_alloc(abfs_graph *g, uint64_t n, uint64_t m) {
    DevGraph &d = g->d;
    d.n = n;
    d.m = m;
    const size_t mb = (m ? m : 1) * 4 + 16;
    cudaError_t e = cudaSuccess;
    auto A = [&](uint32_t **p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc((void **)p, bytes);
    };
    A(&d.out_off, (n + 1) * 4 + 16);
    A(&d.in_off, (n + 1) * 4 + 16);
    A(&d.dst, mb);
    A(&d.org, mb);
    A(&d.src, mb);
    A(&d.rev_owner, mb);
    A(&d.first_src, (n ? n : 1) * 4 + 16);
    if (e != cudaSuccess) {
        graph_free(g);
        return fail(e == cudaErrorMemoryAllocation ? ABFS_ENOMEM : ABFS_ECUDA,
                    std::string("graph alloc: ") + cudaGetErrorString(e));
    }
    return ABFS_OK;
}

void graph_free(abfs_graph *g) {
    DevGraph &d = g->d;
    cudaFree(d.out_off);
    cudaFree(d.in_off);
    cudaFree(d.dst);
    cudaFree(d.org);
    cudaFree(d.src);
    cudaFree(d.rev_owner);
    cudaFree(d.first_src);
    d = DevGraph();
}

}  // namespace abfs

extern "C" void abfs_graph_destroy(abfs_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    graph_free(g);
    delete g;
}

extern "C" int abfs_graph_info(const abfs_graph *g, uint64_t *n, uint64_t *m, int *device) {
    if (!g) return fail(ABFS_EINVAL, "null graph");
    if (n) *n = g->d.n;
    if (m) *m = g->d.m;
    if (device) *device = g->device;
    return ABFS_OK;
}

extern "C" int abfs_graph_upload(int device, uint64_t n, uint64_t m, const uint32_t *out_offsets,
                                 const uint32_t *destinations, const uint32_t *origins,
                                 const uint32_t *in_offsets, const uint32_t *sources,
                                 abfs_graph **out) {
    if (!out_offsets || !in_offsets || (m && (!destinations || !origins || !sources)))
        return fail(ABFS_EINVAL, "null array");
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, m, &g));
    DevGraph &d = g->d;
    int rc = ABFS_OK;
    auto up = [&](uint32_t *dptr, const uint32_t *h, uint64_t cnt) {
        if (rc == ABFS_OK && cnt) {
            cudaError_t e = cudaMemcpy(dptr, h, cnt * 4, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("upload: ") + cudaGetErrorString(e));
        }
    };
    up(d.out_off, out_offsets, n + 1);
    up(d.in_off, in_offsets, n + 1);
    up(d.dst, destinations, m);
    up(d.org, origins, m);
    up(d.src, sources, m);
    if (rc == ABFS_OK && m) {
        k_rev_owner<<<grid_cap(m, 256), 256>>>(d.in_off, n, m, d.rev_owner);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("rev_owner: ") + cudaGetErrorString(e));
    }
    *out = g;
    return finish_build(rc, g, out);
}

extern "C" int abfs_graph_download(const abfs_graph *g, uint32_t *out_offsets,
                                   uint32_t *destinations, uint32_t *origins,
                                   uint32_t *in_offsets, uint32_t *sources, uint32_t *rev_owner) {
    if (!g) return fail(ABFS_EINVAL, "null graph");
    ABFS_CUDA(cudaSetDevice(g->device));
    const DevGraph &d = g->d;
    auto down = [&](uint32_t *h, const uint32_t *dp, uint64_t cnt) -> cudaError_t {
        if (!h || !cnt) return cudaSuccess;
        return cudaMemcpy(h, dp, cnt * 4, cudaMemcpyDeviceToHost);
    };
    ABFS_CUDA(down(out_offsets, d.out_off, d.n + 1));
    ABFS_CUDA(down(in_offsets, d.in_off, d.n + 1));
    ABFS_CUDA(down(destinations, d.dst, d.m));
    ABFS_CUDA(down(origins, d.org, d.m));
    ABFS_CUDA(down(sources, d.src, d.m));
    ABFS_CUDA(down(rev_owner, d.rev_owner, d.m));
    return ABFS_OK;
}

extern "C" int abfs_graph_build(int device, uint64_t n, uint64_t m, const uint32_t *src,
                                const uint32_t *dst, abfs_graph **out) {
    if (m && (!src || !dst)) return fail(ABFS_EINVAL, "null array");
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, m, &g));
    KeyBufs kb;
    int rc = ABFS_OK;
    cudaError_t e = cudaMalloc(&kb.a, (m ? m : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kb.b, (m ? m : 1) * 8);
    // stage pairs through the (not yet filled) dst/org arrays
    if (e == cudaSuccess && m) e = cudaMemcpy(g->d.org, src, m * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(g->d.dst, dst, m * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("build: ") + cudaGetErrorString(e));
    if (rc == ABFS_OK && m) {
        k_pack_pairs<<<grid_cap(m, 256), 256>>>(g->d.org, g->d.dst, m, kb.a);
        if ((e = cudaGetLastError()) != cudaSuccess) rc = fail(ABFS_ECUDA, cudaGetErrorString(e));
    }
    if (rc == ABFS_OK) rc = build_from_keys(g, kb.a, kb.b, 0);
    *out = g;
    return finish_build(rc, g, out);
}

static u128 words_to_u128(const uint64_t w[2]) { return ((u128)w[0] << 64) | (u128)w[1]; }

static uint64_t thr53(double t) {
    // r >= t  <=>  k >= ceil(t * 2^53) for r = k * 2^-53, 0 <= k < 2^53
    if (t <= 0.0) return 0;
    const double x = std::ceil(t * 9007199254740992.0);
    if (x >= 18446744073709551615.0) return ~0ull;
    return (uint64_t)x;
}

extern "C" int abfs_graph_generate_rmat(int device, uint32_t scale, uint64_t edges, double a,
                                        double b, double c, const uint64_t pcg_state[2],
                                        const uint64_t pcg_inc[2], int symmetrize,
                                        abfs_graph **out) {
    if (!pcg_state || !pcg_inc) return fail(ABFS_EINVAL, "null pcg state");
    if (scale < 1 || scale > 31) return fail(ABFS_EINVAL, "scale must be in [1, 31]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0 + 1e-9)
        return fail(ABFS_EINVAL, "rmat probabilities must be non-negative and sum to <= 1");
    const uint64_t n = 1ull << scale;
    const uint64_t m = (symmetrize & 1) ? 2 * edges : edges;
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, m, &g));
    RmatParams hp;
    hp.s0 = words_to_u128(pcg_state);
    hp.inc = words_to_u128(pcg_inc);
    hp.m = edges;
    hp.scale = scale;
    hp.symmetrize = symmetrize & 3;
    // Same float64 operations as graph.py:247-248: a+b and (a+b)+c.
    hp.t1 = thr53(a);
    hp.t2 = thr53(a + b);
    hp.t3 = thr53(a + b + c);
    for (uint32_t bit = 0; bit < scale; ++bit) pcg_jump(hp.inc, (u128)bit * edges, hp.bitA[bit], hp.bitC[bit]);
    KeyBufs kb;
    RmatParams *dp = nullptr;
    int rc = ABFS_OK;
    cudaError_t e = cudaMalloc(&kb.a, (m ? m : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kb.b, (m ? m : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dp, sizeof(RmatParams));
    if (e == cudaSuccess) e = cudaMemcpy(dp, &hp, sizeof(RmatParams), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && edges) {
        const uint64_t threads = (edges + kGenChunk - 1) / kGenChunk;
        k_gen_rmat<<<(unsigned)((threads + 255) / 256), 256>>>(dp, kb.a);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("generate_rmat: ") + cudaGetErrorString(e));
    if (rc == ABFS_OK) rc = build_from_keys(g, kb.a, kb.b, 0);
    cudaFree(dp);
    *out = g;
    return finish_build(rc, g, out);
}

extern "C" int abfs_graph_generate_uniform(int device, uint64_t n, uint64_t edges,
                                           const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                                           abfs_graph **out) {
    if (!pcg_state || !pcg_inc) return fail(ABFS_EINVAL, "null pcg state");
    if (n == 0 || (n & (n - 1)) || n > (1ull << 31))
        return fail(ABFS_EINVAL, "device uniform-random needs a power-of-two n <= 2^31");
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, edges, &g));
    UniParams p;
    p.s0 = words_to_u128(pcg_state);
    p.inc = words_to_u128(pcg_inc);
    p.n_log2 = (uint64_t)bits_for(n);
    p.m = edges;
    KeyBufs kb;
    int rc = ABFS_OK;
    cudaError_t e = cudaMalloc(&kb.a, (edges ? edges : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kb.b, (edges ? edges : 1) * 8);
    if (e == cudaSuccess && edges) {
        const uint64_t threads = (edges + kGenChunk - 1) / kGenChunk;
        k_gen_uniform<<<(unsigned)((threads + 255) / 256), 256>>>(p, kb.a);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("generate_uniform: ") + cudaGetErrorString(e));
    if (rc == ABFS_OK) rc = build_from_keys(g, kb.a, kb.b, 0);
    *out = g;
    return finish_build(rc, g, out);
}

extern "C" int abfs_graph_generate_mesh(int device, uint32_t rows, uint32_t cols, abfs_graph **out) {
    if (rows < 1 || cols < 1) return fail(ABFS_EINVAL, "mesh needs rows, cols >= 1");
    const uint64_t n = (uint64_t)rows * cols;
    const uint64_t m = 2 * ((uint64_t)rows * (cols - 1) + (uint64_t)(rows - 1) * cols);
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, m, &g));
    KeyBufs kb;
    unsigned long long *cur = nullptr;
    int rc = ABFS_OK;
    cudaError_t e = cudaMalloc(&kb.a, (m ? m : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kb.b, (m ? m : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cur, 8);
    if (e == cudaSuccess) e = cudaMemset(cur, 0, 8);
    if (e == cudaSuccess) {
        k_gen_mesh<<<(unsigned)((n + 255) / 256), 256>>>(rows, cols, kb.a, cur);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("generate_mesh: ") + cudaGetErrorString(e));
    if (rc == ABFS_OK) rc = build_from_keys(g, kb.a, kb.b, 0);
    cudaFree(cur);
    *out = g;
    return finish_build(rc, g, out);
}

// ---- streaming generation: degrees and destination-filtered slices -----------
//
// The generators above materialise the whole key stream (8 bytes per slot)
// and sort it.  A rank of a 1-D partition needs only the edges whose
// destination it owns, and compute_stats / the edge-balanced bounds need only
// the degrees, so these kernels regenerate the same stream (same draws, same
// pairs) and either count degrees or keep the owned pairs.

namespace {

struct GenArgs {
    int kind;                     // ABFS_GEN_RMAT / ABFS_GEN_UNIFORM
    const RmatParams *rp;         // rmat (device copy)
    UniParams up;                 // uniform
    uint64_t pairs;               // generated pairs
    int sym;                      // rmat: each pair also yields (dst, src)
    // degree mode
    uint32_t *out_deg, *in_deg;   // in_deg NULL: symmetric (one array)
    // filter mode: keep (s, d) with lo <= d < hi; keys NULL = count only
    uint64_t *keys;
    unsigned long long *cursor;
    uint32_t lo, hi;
};

// uniform: the pairs of edges [i0, i0 + cnt): src = u32 stream positions
// i0.., dst = positions m + i0..; u64 draw k yields positions 2k (low half)
// and 2k + 1 (high half), as in k_gen_uniform.
__device__ __forceinline__ void uniform_pairs(const UniParams &p, uint64_t i0,
                                              uint32_t (&src)[kGenChunk], uint32_t (&dst)[kGenChunk]) {
    const u128 M = pcg_mult();
    auto val = [&](uint64_t u32) { return (uint32_t)((u32 << p.n_log2) >> 32); };
    u128 A, C;
    pcg_jump(p.inc, (u128)(i0 >> 1), A, C);   // i0 is a multiple of kGenChunk: even
    u128 s = A * p.s0 + C;
#pragma unroll
    for (int k = 0; k < kGenChunk / 2; ++k) {
        s = s * M + p.inc;
        const uint64_t o = pcg_out(s);
        src[2 * k] = val(o & 0xffffffffull);
        src[2 * k + 1] = val(o >> 32);
    }
    const uint64_t j = p.m + i0;
    pcg_jump(p.inc, (u128)(j >> 1), A, C);
    s = A * p.s0 + C;
    const int off = (int)(j & 1);
    uint32_t hw[kGenChunk + 2];
#pragma unroll
    for (int k = 0; k < kGenChunk / 2 + 1; ++k) {
        s = s * M + p.inc;
        const uint64_t o = pcg_out(s);
        hw[2 * k] = val(o & 0xffffffffull);
        hw[2 * k + 1] = val(o >> 32);
    }
#pragma unroll
    for (int k = 0; k < kGenChunk; ++k) dst[k] = off ? hw[k + 1] : hw[k];
}

// Warp-aggregated append of this thread's kept pairs (all lanes call).
__device__ __forceinline__ void append_kept(const GenArgs &a, int nkeep, const uint64_t *kept) {
    const unsigned lane = threadIdx.x & 31u;
    unsigned incl = (unsigned)nkeep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(kFull, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    const unsigned tot = __shfl_sync(kFull, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(a.cursor, (unsigned long long)tot);
    base = __shfl_sync(kFull, base, 31);
    if (a.keys) {
        const unsigned long long at = base + incl - (unsigned)nkeep;
        for (int k = 0; k < nkeep; ++k) a.keys[at + k] = kept[k];
    }
}

template <bool DEGREES>
__global__ void __launch_bounds__(256) k_gen_stream(GenArgs a) {
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kGenChunk;
    const int cnt = i0 < a.pairs ? (int)min((uint64_t)kGenChunk, a.pairs - i0) : 0;
    uint32_t src[kGenChunk], dst[kGenChunk];
    if (cnt) {
        if (a.kind == ABFS_GEN_RMAT) rmat_pairs(*a.rp, i0, cnt, src, dst);
        else uniform_pairs(a.up, i0, src, dst);
    }
    if (DEGREES) {
        for (int k = 0; k < cnt; ++k) {
            atomicAdd(a.out_deg + src[k], 1u);
            if (a.in_deg) atomicAdd(a.in_deg + dst[k], 1u);
            else if (a.sym) atomicAdd(a.out_deg + dst[k], 1u);   // (dst, src) slot
            if (a.sym && a.in_deg) {
                atomicAdd(a.out_deg + dst[k], 1u);
                atomicAdd(a.in_deg + src[k], 1u);
            }
        }
        return;
    }
    uint64_t kept[2 * kGenChunk];
    int nk = 0;
    for (int k = 0; k < cnt; ++k) {
        if (dst[k] >= a.lo && dst[k] < a.hi) kept[nk++] = ((uint64_t)src[k] << 32) | dst[k];
        if (a.sym && src[k] >= a.lo && src[k] < a.hi) kept[nk++] = ((uint64_t)dst[k] << 32) | src[k];
    }
    append_kept(a, nk, kept);
}

// mesh: vertex v's pairs (v, neighbour) as k_gen_mesh emits them.
template <bool DEGREES>
__global__ void __launch_bounds__(256) k_mesh_stream(uint32_t rows, uint32_t cols, GenArgs a) {
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t n = (uint64_t)rows * cols;
    uint64_t nb[4];
    int k = 0;
    if (v < n) {
        const uint32_t r = (uint32_t)(v / cols), c = (uint32_t)(v % cols);
        if (r > 0) nb[k++] = v - cols;
        if (c > 0) nb[k++] = v - 1;
        if (c + 1 < cols) nb[k++] = v + 1;
        if (r + 1 < rows) nb[k++] = v + cols;
    }
    if (DEGREES) {
        if (v < n) {
            a.out_deg[v] = (uint32_t)k;
            if (a.in_deg) a.in_deg[v] = (uint32_t)k;   // the grid is symmetric
        }
        return;
    }
    uint64_t kept[4];
    int nk = 0;
    for (int i = 0; i < k; ++i)
        if (nb[i] >= a.lo && nb[i] < a.hi) kept[nk++] = (v << 32) | nb[i];
    append_kept(a, nk, kept);
}

__global__ void k_pack_rev_local(const uint32_t *__restrict__ dst, const uint32_t *__restrict__ org,
                                 uint64_t m, uint32_t lo, uint64_t *keys) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = ((uint64_t)(dst[i] - lo) << 32) | org[i];
}

__global__ void k_add_u32(uint32_t *x, uint64_t m, uint32_t add) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        x[i] += add;
}

// Host side of a spec: sizes and the kernel arguments (rmat params on the device).
struct GenPlan {
    uint64_t n = 0, m = 0;
    GenArgs a{};
    RmatParams *dp = nullptr;
    ~GenPlan() { cudaFree(dp); }
};

int gen_plan(const abfs_gen_spec *spec, GenPlan &g, bool upload) {
    if (!spec) return fail(ABFS_EINVAL, "null generator spec");
    g.a.kind = spec->kind;
    switch (spec->kind) {
    case ABFS_GEN_RMAT: {
        if (spec->scale < 1 || spec->scale > 31) return fail(ABFS_EINVAL, "scale must be in [1, 31]");
        if (spec->a < 0 || spec->b < 0 || spec->c < 0 || spec->a + spec->b + spec->c > 1.0 + 1e-9)
            return fail(ABFS_EINVAL, "rmat probabilities must be non-negative and sum to <= 1");
        g.n = 1ull << spec->scale;
        g.m = spec->symmetrize ? 2 * spec->edges : spec->edges;
        g.a.pairs = spec->edges;
        g.a.sym = spec->symmetrize ? 1 : 0;
        if (upload) {
            RmatParams hp;
            hp.s0 = words_to_u128(spec->pcg_state);
            hp.inc = words_to_u128(spec->pcg_inc);
            hp.m = spec->edges;
            hp.scale = spec->scale;
            hp.symmetrize = g.a.sym;
            hp.t1 = thr53(spec->a);
            hp.t2 = thr53(spec->a + spec->b);
            hp.t3 = thr53(spec->a + spec->b + spec->c);
            for (uint32_t bit = 0; bit < spec->scale; ++bit)
                pcg_jump(hp.inc, (u128)bit * spec->edges, hp.bitA[bit], hp.bitC[bit]);
            ABFS_CUDA(cudaMalloc(&g.dp, sizeof(RmatParams)));
            ABFS_CUDA(cudaMemcpy(g.dp, &hp, sizeof(RmatParams), cudaMemcpyHostToDevice));
            g.a.rp = g.dp;
        }
        break;
    }
    case ABFS_GEN_UNIFORM:
        if (spec->n == 0 || (spec->n & (spec->n - 1)) || spec->n > (1ull << 31))
            return fail(ABFS_EINVAL, "device uniform-random needs a power-of-two n <= 2^31");
        g.n = spec->n;
        g.m = spec->edges;
        g.a.pairs = spec->edges;
        g.a.up.s0 = words_to_u128(spec->pcg_state);
        g.a.up.inc = words_to_u128(spec->pcg_inc);
        g.a.up.n_log2 = (uint64_t)bits_for(spec->n);
        g.a.up.m = spec->edges;
        break;
    case ABFS_GEN_MESH:
        if (spec->rows < 1 || spec->cols < 1) return fail(ABFS_EINVAL, "mesh needs rows, cols >= 1");
        g.n = (uint64_t)spec->rows * spec->cols;
        g.m = 2 * ((uint64_t)spec->rows * (spec->cols - 1) + (uint64_t)(spec->rows - 1) * spec->cols);
        break;
    default:
        return fail(ABFS_EINVAL, "unknown generator kind " + std::to_string(spec->kind));
    }
    if (g.n >= (1ull << 32)) return fail(ABFS_EINVAL, "vertex_count must be < 2^32");
    if (g.m >= (1ull << 32)) return fail(ABFS_EINVAL, "edge_count must be < 2^32 (u32 offsets)");
    return ABFS_OK;
}

template <bool DEGREES>
cudaError_t gen_launch(const abfs_gen_spec *spec, const GenPlan &g, const GenArgs &a, cudaStream_t s) {
    if (spec->kind == ABFS_GEN_MESH) {
        if (g.n) k_mesh_stream<DEGREES><<<(unsigned)((g.n + 255) / 256), 256, 0, s>>>(spec->rows, spec->cols, a);
    } else if (a.pairs) {
        const uint64_t threads = (a.pairs + kGenChunk - 1) / kGenChunk;
        k_gen_stream<DEGREES><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

extern "C" int abfs_gen_size(const abfs_gen_spec *spec, uint64_t *n, uint64_t *m) {
    GenPlan g;
    ABFS_TRY(gen_plan(spec, g, false));
    if (n) *n = g.n;
    if (m) *m = g.m;
    return ABFS_OK;
}

extern "C" int abfs_gen_degrees(int device, const abfs_gen_spec *spec, uint32_t *out_deg,
                                uint32_t *in_deg) {
    if (!out_deg) return fail(ABFS_EINVAL, "null output");
    GenPlan g;
    ABFS_CUDA(cudaSetDevice(device));
    ABFS_TRY(gen_plan(spec, g, true));
    uint32_t *dd = nullptr;
    const uint64_t n = g.n;
    ABFS_CUDA(cudaMalloc(&dd, 2 * (n ? n : 1) * 4));
    GenArgs a = g.a;
    a.out_deg = dd;
    // symmetric specs (symmetrised rmat, mesh) have in == out: one array
    const bool sym = spec->kind == ABFS_GEN_MESH || (spec->kind == ABFS_GEN_RMAT && spec->symmetrize);
    a.in_deg = sym ? nullptr : dd + n;
    cudaError_t e = cudaMemset(dd, 0, 2 * (n ? n : 1) * 4);
    if (e == cudaSuccess) e = gen_launch<true>(spec, g, a, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out_deg, dd, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && in_deg) e = cudaMemcpy(in_deg, sym ? dd : dd + n, n * 4, cudaMemcpyDeviceToHost);
    cudaFree(dd);
    if (e != cudaSuccess) return fail(ABFS_ECUDA, std::string("gen_degrees: ") + cudaGetErrorString(e));
    return ABFS_OK;
}

namespace abfs {

int gen_slice(int device, const abfs_gen_spec *spec, uint64_t lo, uint64_t hi, Slice &out,
              uint64_t *n_out, cudaStream_t s) {
    GenPlan g;
    ABFS_CUDA(cudaSetDevice(device));
    ABFS_TRY(gen_plan(spec, g, true));
    const uint64_t n = g.n;
    if (lo > hi || hi > n) return fail(ABFS_EINVAL, "partition range out of bounds");
    *n_out = n;
    const uint64_t nv = hi - lo;
    GenArgs a = g.a;
    a.lo = (uint32_t)lo;
    a.hi = (uint32_t)hi;
    unsigned long long *cur = nullptr, mk = 0;
    ABFS_CUDA(cudaMalloc(&cur, 8));
    cudaError_t e = cudaMemsetAsync(cur, 0, 8, s);
    a.cursor = cur;
    a.keys = nullptr;   // pass 1: count the owned in-edges
    if (e == cudaSuccess) e = gen_launch<false>(spec, g, a, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&mk, cur, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    KeyBufs kb;
    if (e == cudaSuccess) e = cudaMalloc(&kb.a, (mk ? mk : 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kb.b, (mk ? mk : 1) * 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(cur, 0, 8, s);
    a.keys = kb.a;      // pass 2: keep them (any order; sorted below)
    if (e == cudaSuccess) e = gen_launch<false>(spec, g, a, s);
    cudaFree(cur);
    auto A = [&](uint32_t **p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc((void **)p, bytes ? bytes : 4);
    };
    out.mf = out.mr = mk;
    // +16 on every stream array: the edge kernels' bulk copies and pull's
    // aligned 16-byte reads round the last chunk up
    A(&out.fo_off, (n + 1) * 4);
    A(&out.fo_dst, mk * 4 + 16);
    A(&out.fo_org, mk * 4 + 16);
    A(&out.r_off, (nv + 1) * 4);
    A(&out.r_src, mk * 4 + 16);
    A(&out.r_own, mk * 4 + 16);
    A(&out.r_first, nv * 4 + 16);
    if (e != cudaSuccess) return fail(ABFS_ECUDA, std::string("gen_slice: ") + cudaGetErrorString(e));
    // forward slice: (src, dst) order over all sources
    ABFS_TRY(sort_keys(kb.a, kb.b, mk, bits_for(n), s));
    k_split_offsets<<<grid_cap(mk + 1, 256), 256, 0, s>>>(kb.a, mk, n, out.fo_org, out.fo_dst, out.fo_off);
    ABFS_CUDA(cudaGetLastError());
    // owned in-rows: (dst - lo, src) order
    if (mk) {
        k_pack_rev_local<<<grid_cap(mk, 256), 256, 0, s>>>(out.fo_dst, out.fo_org, mk, (uint32_t)lo, kb.a);
        ABFS_CUDA(cudaGetLastError());
    }
    ABFS_TRY(sort_keys(kb.a, kb.b, mk, bits_for(nv ? nv : 1), s));
    k_split_offsets<<<grid_cap(mk + 1, 256), 256, 0, s>>>(kb.a, mk, nv, out.r_own, out.r_src, out.r_off);
    ABFS_CUDA(cudaGetLastError());
    if (mk) {
        k_add_u32<<<grid_cap(mk, 256), 256, 0, s>>>(out.r_own, mk, (uint32_t)lo);
        ABFS_CUDA(cudaGetLastError());
    }
    if (nv) {
        k_first_src<<<grid_cap(nv, 256), 256, 0, s>>>(out.r_off, out.r_src, nv, out.r_first);
        ABFS_CUDA(cudaGetLastError());
    }
    ABFS_CUDA(cudaStreamSynchronize(s));
    return ABFS_OK;
}

}  // namespace abfs

// ---- ADGR files on the engine side ---------------------------

namespace {

// Python's repr() of a bytes object (the reference's error texts quote the
// magic with {magic!r}).
std::string bytes_repr(const unsigned char *b, size_t n) {
    bool sq = false, dq = false;
    for (size_t i = 0; i < n; ++i) {
        sq |= b[i] == '\'';
        dq |= b[i] == '"';
    }
    const char q = (sq && !dq) ? '"' : '\'';
    std::string s = "b";
    s += q;
    static const char *hex = "0123456789abcdef";
    for (size_t i = 0; i < n; ++i) {
        const unsigned char c = b[i];
        if (c == (unsigned char)q || c == '\\') {
            s += '\\';
            s += (char)c;
        } else if (c == '\t') {
            s += "\\t";
        } else if (c == '\n') {
            s += "\\n";
        } else if (c == '\r') {
            s += "\\r";
        } else if (c < 0x20 || c >= 0x7f) {
            s += "\\x";
            s += hex[c >> 4];
            s += hex[c & 15];
        } else {
            s += (char)c;
        }
    }
    s += q;
    return s;
}

struct File {
    FILE *f = nullptr;
    ~File() {
        if (f) fclose(f);
    }
};

}  // namespace

extern "C" int abfs_graph_read(int device, const char *path, abfs_graph **out) {
    // read_graph (graph.py:304-324): "ADGR", <IQQ> (version 1, |V|, |E|),
    // five little-endian u32 arrays; the arrays are streamed through a pinned
    // buffer straight into HBM (no host copy of the graph).
    if (!path || !out) return fail(ABFS_EINVAL, "null argument");
    File fh;
    fh.f = fopen(path, "rb");
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot open graph file ") + path);
    unsigned char magic[4];
    const size_t got = fread(magic, 1, 4, fh.f);
    if (got != 4 || std::memcmp(magic, "ADGR", 4) != 0)
        return fail(ABFS_EINVAL, "bad magic " + bytes_repr(magic, got) + " in graph file " + path);
    unsigned char hdr[20];
    if (fread(hdr, 1, 20, fh.f) != 20) return fail(ABFS_EINVAL, std::string("truncated graph header in ") + path);
    uint32_t version;
    uint64_t n, m;
    std::memcpy(&version, hdr, 4);
    std::memcpy(&n, hdr + 4, 8);
    std::memcpy(&m, hdr + 12, 8);
    if (version != 1) return fail(ABFS_EINVAL, "unsupported graph format version " + std::to_string(version));
    abfs_graph *g = nullptr;
    ABFS_TRY(new_graph(device, n, m, &g));
    DevGraph &d = g->d;
    const size_t chunk = 16u << 20;
    char *stage = nullptr;
    int rc = ABFS_OK;
    if (cudaMallocHost(&stage, chunk) != cudaSuccess) rc = fail(ABFS_ENOMEM, "pinned staging buffer");
    uint32_t *dst_of[5] = {d.out_off, d.dst, d.org, d.in_off, d.src};
    const uint64_t cnt_of[5] = {n + 1, m, m, n + 1, m};
    for (int a = 0; a < 5 && rc == ABFS_OK; ++a) {
        const uint64_t bytes = cnt_of[a] * 4;
        for (uint64_t off = 0; off < bytes && rc == ABFS_OK; off += chunk) {
            const size_t len = (size_t)std::min<uint64_t>(chunk, bytes - off);
            if (fread(stage, 1, len, fh.f) != len) {
                rc = fail(ABFS_EINVAL, std::string("truncated graph file ") + path);
                break;
            }
            const cudaError_t e = cudaMemcpy(reinterpret_cast<char *>(dst_of[a]) + off, stage, len,
                                             cudaMemcpyHostToDevice);
            if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("graph_read: ") + cudaGetErrorString(e));
        }
    }
    if (rc == ABFS_OK && fgetc(fh.f) != EOF) rc = fail(ABFS_EINVAL, std::string("trailing bytes in graph file ") + path);
    if (stage) cudaFreeHost(stage);
    if (rc == ABFS_OK && m) {
        k_rev_owner<<<grid_cap(m, 256), 256>>>(d.in_off, n, m, d.rev_owner);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("rev_owner: ") + cudaGetErrorString(e));
    }
    *out = g;
    return finish_build(rc, g, out);
}

extern "C" int abfs_graph_write(const abfs_graph *g, const char *path) {
    // write_graph (graph.py:292-301): same bytes as the reference writer.
    if (!g || !path) return fail(ABFS_EINVAL, "null argument");
    ABFS_CUDA(cudaSetDevice(g->device));
    File fh;
    fh.f = fopen(path, "wb");
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot create graph file ") + path);
    const DevGraph &d = g->d;
    unsigned char hdr[24];
    const uint32_t version = 1;
    std::memcpy(hdr, "ADGR", 4);
    std::memcpy(hdr + 4, &version, 4);
    std::memcpy(hdr + 8, &d.n, 8);
    std::memcpy(hdr + 16, &d.m, 8);
    if (fwrite(hdr, 1, 24, fh.f) != 24) return fail(ABFS_EINVAL, std::string("write failed: ") + path);
    const size_t chunk = 16u << 20;
    char *stage = nullptr;
    ABFS_CUDA(cudaMallocHost(&stage, chunk));
    const uint32_t *src_of[5] = {d.out_off, d.dst, d.org, d.in_off, d.src};
    const uint64_t cnt_of[5] = {d.n + 1, d.m, d.m, d.n + 1, d.m};
    int rc = ABFS_OK;
    for (int a = 0; a < 5 && rc == ABFS_OK; ++a) {
        const uint64_t bytes = cnt_of[a] * 4;
        for (uint64_t off = 0; off < bytes && rc == ABFS_OK; off += chunk) {
            const size_t len = (size_t)std::min<uint64_t>(chunk, bytes - off);
            const cudaError_t e = cudaMemcpy(stage, reinterpret_cast<const char *>(src_of[a]) + off, len,
                                             cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) rc = fail(ABFS_ECUDA, std::string("graph_write: ") + cudaGetErrorString(e));
            else if (fwrite(stage, 1, len, fh.f) != len) rc = fail(ABFS_EINVAL, std::string("write failed: ") + path);
        }
    }
    cudaFreeHost(stage);
    return rc;
}
