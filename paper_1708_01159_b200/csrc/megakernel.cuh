// megakernel.cuh -- device-resident tree-switched level loop.
//
// One cooperative, persistent kernel runs the whole traversal: every CTA
// evaluates the FlatTree on the reference's float64 features (identical
// arithmetic, so all CTAs pick the same pair), runs the chosen strategy body
// over the grid, and meets the others at a grid barrier; the new count is
// read from the rotating counter slot after the barrier.  No host round trip
// and no kernel launch between levels: the per-level fixed cost drops from a
// launch + readback (~10 us) to one or two grid barriers.
//
// The strategy bodies are the same device functions the per-level kernels
// use (bfs_kernels.cuh), so results are identical by construction; the
// megakernel always starts from init_depths, hence runs in consistent mode.
#pragma once

#include <cooperative_groups.h>

#include <mutex>
#include <vector>

#include "bfs_kernels.cuh"
#ifndef ABFS_PULL2_CODE
#define ABFS_PULL2_CODE 0   // the list-based pull (pull2.cuh) in the megakernel: opt-in build,
                            // it costs the default path registers even when unused
#endif
#include "pull2.cuh"

namespace abfs {

namespace cg = cooperative_groups;

struct MegaRecord {
    int32_t kernel, variant, fallback, converted;
    unsigned long long frontier, new_count;
    unsigned long long t_start, t_pred, t_end;   // %globaltimer (ns)
    unsigned long long scanned;                  // pull ES (instrumented)
    unsigned long long next_out_edges;           // N2: sum out-degree of the discoveries (instrumented)
};

struct MegaParams {
    int32_t *depth;
    uint32_t *visited;
    const uint32_t *noin;
    uint32_t *fbm0, *fbm1;
    uint32_t *q0, *q1;
    uint2 *units;
    Ctr *ctr;
    const uint32_t *out_off, *dst, *org, *in_off, *src, *rev_owner, *first_src;
    uint64_t n, m, words;
    // device tree: CutNode array (see below), staged into shared memory
    const void *tree;
    uint32_t tree_nodes;
    int fixed_pair;      // >= 0: bfs_full with this pair ordinal, no tree
    int vw_log2;
    // push-warp levels with at most vw_wide_f frontier vertices run at width
    // 2^vw_wide_log2 (= min(chunk, 32)) instead of the degree-fitted one: a
    // small level's chain is shorter with more lanes per vertex
    int vw_wide_log2;
    unsigned long long vw_wide_f;
    int instrument;
    uint32_t pull_light;
    uint32_t cap;
    MegaRecord *recs;
    unsigned long long *n_levels;   // per root
    // roots of this launch, traversed one after the other; with init_in_kernel
    // every root's init_depths runs inside the kernel (else the host did it
    // for the single root)
    const uint32_t *roots;
    uint32_t nroots;
    int init_in_kernel;
    // cluster solo mode (0 = off): with a cluster launch, runs of small
    // top-down levels execute on cluster 0 alone (solo_ctas CTAs, cluster
    // barriers) while the other CTAs wait at one grid barrier
    uint32_t solo_ctas;
    uint32_t solo_passes;       // frontier passes of the cluster's threads a solo level may take
    uint32_t solo_direct;       // solo levels claim without the visited-word filter load
    unsigned long long direct_f; // grid top-down levels of at most this many frontier vertices too
    uint32_t red_direct;         // RED-mode levels reduce every candidate (no filter load)
    struct SoloState *solo;
    // ---- vertex partition (part = 1; partition.cu): this rank owns
    // destinations [lo, hi); depth / visited / noin / in_off / first_src are
    // rebased to global ids, out_off / dst / org are the destination-filtered
    // forward slice (m slots), in_off / src / rev_owner the owned reverse
    // rows (m_rev slots); the frontier bitmaps fbm0/1 are global (words).
    // After every level the visited bits gained are stored into every rank's
    // next-frontier bitmap (peer memory) and the global count is summed from
    // the ranks' mailboxes.  Single graph: lo = 0, hi = n, m_rev = m,
    // wlo = 0, wend = words, part = 0.
    int part;
    uint64_t m_rev, lo, hi, wlo, wend;
    uint32_t *vprev;            // [wend - wlo] visited words at the previous exchange
    uint32_t *fnext;            // pull's next-frontier words (rebased); single: unused
    uint32_t *const *peer_fbm;  // [2][nranks]
    PeerBox *const *peer_box;   // [nranks]
    PeerBox *box;
    uint32_t nranks, rank;
    unsigned long long xseq0;   // megakernel exchanges completed before this launch (PeerBox::mk_*)
    int xsys;                   // exchange signalling: 0 GPU-scope release/acquire (same device),
                                // 1 system-scope release/acquire, 2 LL words (cross-device)
    // optional [nroots]: per-root depth checksum (depth_mix) of the final
    // depth array of each traversal, for batch parity checks
    unsigned long long *checksums;
    // RED-mode top-down levels (single graph only; acc = nullptr disables):
    // acc [words] all-zero between levels; a push / push-warp level with
    // frontier >= red_frontier runs its edge phase with fire-and-forget OR
    // reductions into acc and settles them in one bitmap pass (which also
    // yields the next frontier bitmap); a level whose light pass queued >=
    // red_units CTA units runs just the unit pass that way
    uint32_t *acc;
    uint64_t red_frontier;
    uint32_t red_units;
    // sparse pull levels: when at most pull_wide_max candidates can remain
    // (|V| - discovered - n_noin, n_noin = vertices of in-degree 0) the pull
    // sweeps 4 sub-tiles per warp fetch (0 disables)
    uint64_t pull_wide_max;
    uint64_t n_noin;
    // list-based pull (pull2.cuh; single graph): survivor list + two
    // carried candidate lists, each [n] (pl_s = nullptr: sub-tile pull)
    uint32_t *pl_s, *pl_c0, *pl_c1;
};

// Order-sensitive checksum term of one vertex's depth (numpy restatement in
// tests: sum over v of (uint64(uint32(d)) + 1) * ((v + 1) * 0x9E3779B97F4A7C15),
// all mod 2^64).
__device__ __forceinline__ unsigned long long depth_mix(uint64_t v, int32_t d) {
    return ((unsigned long long)(uint32_t)d + 1ull) * ((v + 1ull) * 0x9E3779B97F4A7C15ull);
}

// Hand-off from cluster 0 back to the grid after a solo run.
struct SoloState {
    unsigned long long frontier, discovered;
    uint32_t level;
    int32_t pk, pv, cur, has_q, has_bm, done;
    uint32_t pad;
};

// Host helpers (engine.cu).
void stage_cut_tree(const abfs_tree *tr, const double *static24, uint64_t n,
                    std::vector<unsigned char> &blob, uint32_t &nn);
int mega_launch_plain(const MegaParams &P, cudaStream_t s, int device);
std::mutex &mega_mutex(int device);   // held from a megakernel launch to its completion

constexpr uint32_t kMegaCapPart = 1u << 16;   // level records of a partition's loop
constexpr int kMaxSplit = 8;          // batch: concurrent sub-traversals at most
constexpr uint32_t kSoloUnits = 16;   // more CTA units than this: hand the level to the grid


__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The tree as the device walks it.  The host (engine.cu, mega_run) resolves
// every node on a static feature for this graph and turns each remaining
// float64 test on a per-level feature into an exact integer cutoff:
//   frontier_abs / discovered_abs:  (double)k < thr
//   frontier_pct / discovered_pct:  (double)k / (double)|V| < thr
// are monotone in the integer k (IEEE conversion and division are correctly
// rounded), so each is "k < cutoff" with cutoff = the smallest k failing the
// test, found on the host with the very same float64 arithmetic.  The walk is
// then integer compares on shared memory: same leaf as tree.py:332-339 for
// every reachable (frontier, discovered).
struct CutNode {
    unsigned long long cutoff;
    uint32_t left, right;
    uint8_t cls;       // 255 = internal
    uint8_t on_disc;   // 0: compare frontier, 1: compare discovered
    uint8_t pad[14];
};
static_assert(sizeof(CutNode) == 32, "CutNode layout");

constexpr uint32_t kMegaTreeNodes = 512;   // 16 KB of shared memory

// The pruned tree is a pure function of (frontier, discovered): each leaf
// owns a box [flo,fhi) x [dlo,dhi).  Thread 0 of a CTA keeps the box of its
// last leaf (in shared memory: registers are the megakernel's scarcest
// resource) and re-walks only when the counts leave it -- a mesh BFS stays in
// one leaf for hundreds of levels, and a walk is a chain of dependent shared
// loads (~0.5 us at depth 12).
struct TreeCache {
    unsigned long long flo, fhi, dlo, dhi;
    int cls;
};

__device__ __forceinline__ int mega_tree_class(const CutNode *T, unsigned long long frontier,
                                               unsigned long long discovered, TreeCache *tc) {
    if (frontier >= tc->flo && frontier < tc->fhi && discovered >= tc->dlo && discovered < tc->dhi)
        return tc->cls;
    unsigned long long flo = 0, fhi = ~0ull, dlo = 0, dhi = ~0ull;
    uint32_t node = 0;
    while (T[node].cls == 255) {
        const CutNode &n = T[node];
        const unsigned long long x = n.on_disc ? discovered : frontier;
        const unsigned long long cut = n.cutoff;
        if (x < cut) {
            node = n.left;
            if (n.on_disc) dhi = min(dhi, cut);
            else fhi = min(fhi, cut);
        } else {
            node = n.right;
            if (n.on_disc) dlo = max(dlo, cut);
            else flo = max(flo, cut);
        }
    }
    tc->flo = flo;
    tc->fhi = fhi;
    tc->dlo = dlo;
    tc->dhi = dhi;
    tc->cls = T[node].cls;
    return tc->cls;
}

#ifdef ABFS_DIAG_CTA
// diagnostic build only: per level, per CTA, the %globaltimer at the end of
// the light pass [2*level] and of the CTA-unit pass [2*level+1]
__device__ unsigned long long g_diag_cta[128 * 1024];
#define ABFS_DIAG_MARK(slot)                                                                \
    do {                                                                                    \
        if (threadIdx.x == 0 && c.level < 64 && blockIdx.x < 1024)                          \
            g_diag_cta[(2 * c.level + (slot)) * 1024 + blockIdx.x] = globaltimer();         \
    } while (0)
#else
#define ABFS_DIAG_MARK(slot) \
    do {                     \
    } while (0)
#endif

// Returns kStratBitmap if the level also wrote a complete next-frontier
// bitmap (full RED-mode top-down level).
constexpr int kStratBitmap = 1;

template <int VAR>
__device__ __forceinline__ int mega_strategy(const MegaParams &P, const LevelCtx &c, int kernel,
                                             uint32_t F, const uint32_t *q, uint32_t *fbm_next,
                                             SmemQ *sq, unsigned *sn, int *s_done,
                                             uint32_t *pfound, unsigned int *sfetch,
                                             unsigned *warp_tot, unsigned *s_base, bool wide,
                                             const PullLists *PL, uint32_t pl_n,
                                             cg::grid_group &grid) {
    // Two-phase strategies (light pass, then CTA work units) need a second
    // barrier only if the light pass created units: after the first barrier
    // every CTA reads the same unit count, and with none the level's count
    // is already final (saves a grid barrier on most small levels).
    const auto units = [&]() { return *(volatile unsigned *)c.units_tail; };
    switch (kernel) {
    case 0:
        edge_body<VAR, false, 1>(c, sq, P.org, P.dst, P.m);
        break;
    case 1:
        edge_body<VAR, true, 1>(c, sq, P.rev_owner, P.src, P.m_rev);
        break;
    case 2:
    case 4: {
        if (kernel == 2) push_body<VAR>(c, sq, q, F, P.out_off, P.dst, blockIdx.x, gridDim.x);
        else push_warp_body<VAR>(c, sq, q, F, P.out_off, P.dst,
                                 F <= P.vw_wide_f && P.vw_wide_log2 > P.vw_log2 ? P.vw_wide_log2 : P.vw_log2,
                                 blockIdx.x, gridDim.x);
        ABFS_DIAG_MARK(0);
        grid.sync();
        const unsigned nu = units();
        if (!c.acc && !nu) return 0;
        // a heavy unit pass goes RED too once it is big enough
        LevelCtx cu = c;
        if (!cu.acc && P.acc && nu >= P.red_units) cu.acc = P.acc;
        if (nu) {
            heavy_body<VAR>(cu, sq, P.out_off, P.dst, blockIdx.x, gridDim.x);
            ABFS_DIAG_MARK(1);
            grid.sync();
        }
        if (!cu.acc) return 0;
        red_compact_body<VAR>(c, cu.acc, c.acc ? fbm_next : nullptr, P.words, warp_tot, s_base);
        grid.sync();
        return c.acc ? kStratBitmap : 0;
    }
    case 3:
#if ABFS_PULL2_CODE
        if (PL) {
            // list-based pull: probe 0 grid-wide, then the survivors' scans
            CEmit<VAR> em(sn, c.count);
            unsigned long long scanned = 0;
            if (PL->c_in)
                pull2_list_probe(c, PL->c_in, pl_n, P.first_src, fbm_next, P.wlo, P.wend, scanned);
            else
                pull2_sweep<VAR>(c, em, P.noin, P.first_src, fbm_next, P.wlo, P.wend, *PL, warp_tot,
                                 s_base, scanned);
            ABFS_DIAG_MARK(1);   // diagnostic builds: phase-1 end in the unit-pass slot
            grid.sync();
            const uint32_t *lst = PL->c_in ? PL->c_in : PL->s;
            const uint32_t nl = PL->c_in ? pl_n : *(volatile unsigned *)PL->s_tail;
            pull2_scan<VAR>(c, em, lst, nl, P.in_off, P.src, fbm_next, *PL, warp_tot, s_base, scanned);
            em.finish();
            ABFS_DIAG_MARK(0);
            if (c.es) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) scanned += __shfl_down_sync(kFull, scanned, o);
                if ((threadIdx.x & 31) == 0 && scanned) atomicAdd(c.es, scanned);
            }
            grid.sync();
            if (!units()) return 0;
            pull_heavy_body(c, s_done, P.in_off, P.src, fbm_next);
            break;
        }
#endif
        {
            // the pull scratch lists alias the (idle) CTA queue buffer
            static_assert(sizeof(uint32_t) * kWarps * kPullList <= sizeof(sq->buf), "pull list");
            const unsigned w = threadIdx.x >> 5;
            if (wide)
                pull_body<VAR, 4>(c, sn, P.in_off, P.src, P.first_src, P.noin, fbm_next, P.wlo,
                                  P.wend, sq->buf + w * kPullList, pfound + w * kPullSub, sfetch);
            else
                pull_body<VAR, 1>(c, sn, P.in_off, P.src, P.first_src, P.noin, fbm_next, P.wlo,
                                  P.wend, sq->buf + w * kPullList, pfound + w * kPullSub, sfetch);
        }
        ABFS_DIAG_MARK(0);
        grid.sync();
        if (!units()) return 0;
        pull_heavy_body(c, s_done, P.in_off, P.src, fbm_next);
        break;
    }
    ABFS_DIAG_MARK(1);
    grid.sync();
    return 0;
}

// One top-down level's light pass on cluster 0 (solo mode).
template <int VAR>
__device__ __forceinline__ void solo_light(const MegaParams &P, const LevelCtx &c, int kernel,
                                           uint32_t F, const uint32_t *q, SmemQ *sq) {
    if (kernel == 2) push_body<VAR>(c, sq, q, F, P.out_off, P.dst, blockIdx.x, P.solo_ctas);
    else push_warp_body<VAR>(c, sq, q, F, P.out_off, P.dst, P.vw_log2, blockIdx.x, P.solo_ctas);
}

__device__ __forceinline__ bool solo_fits(const MegaParams &P, int kernel,
                                          unsigned long long frontier) {
    // one pass of the cluster's threads (two for virtual warps)
    const unsigned long long lanes = (unsigned long long)P.solo_ctas * kBlock * P.solo_passes;
    if (kernel == 2) return frontier <= lanes;
    // virtual warps: two passes pay off for wide warps (few vertices per
    // pass); narrow ones (a degree-fitted width of 1-2 lanes) are push-like
    if (kernel == 4) return (frontier << P.vw_log2) <= (P.vw_log2 >= 2 ? 2 : 1) * lanes;
    return false;
}

#ifndef ABFS_SOLO_DSMEM
#define ABFS_SOLO_DSMEM 1
#endif

#ifndef ABFS_MEGA_MINB
#define ABFS_MEGA_MINB 5
#endif
constexpr int kMegaMinB = ABFS_MEGA_MINB;   // default variant (set_mode 1)

// MINB = resident CTAs per SM the register budget is sized for (6 -> 40
// registers, 4 -> 64); latency-bound pull levels want the higher occupancy.
// PART: the partition (one rank's slice, fused exchange) instantiation; the
// single-graph one carries none of the partition code (fewer live registers)
template <int MINB, bool PART, bool SOLO = true>
__global__ void __launch_bounds__(kBlock, MINB) k_mega(MegaParams P) {
    __shared__ SmemQ sq;
    __shared__ uint32_t pfound[kWarps * kPullSub];
    __shared__ unsigned int s_fetch[2];
    __shared__ unsigned sn;
    __shared__ int s_done;
    __shared__ int s_cls;
    __shared__ unsigned warp_tot[kWarps];
    __shared__ unsigned s_base;
    __shared__ unsigned long long s_nw;   // partition mode: the exchanged level count
    __shared__ unsigned s_incons;         // ctr->inconsistent, constant for a traversal
    __shared__ unsigned s_solo_cnt[3][2]; // solo mode: cluster 0's queue / unit tails
                                          // (CTA 0's copy, reached over DSMEM), rotating slots
    __shared__ __align__(16) CutNode s_tree[kMegaTreeNodes];
    cg::grid_group grid = cg::this_grid();
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    // stage the tree into shared memory (global fallback if it is too big)
    const CutNode *T = reinterpret_cast<const CutNode *>(P.tree);
    if (P.tree_nodes <= kMegaTreeNodes) {
        const uint4 *src4 = reinterpret_cast<const uint4 *>(P.tree);
        uint4 *dst4 = reinterpret_cast<uint4 *>(s_tree);
        for (uint32_t i = threadIdx.x; i < P.tree_nodes * 2; i += kBlock)
            dst4[i] = src4[i];
        T = s_tree;
    }
    __syncthreads();
    __shared__ TreeCache tcache;   // thread 0's last leaf box
    if (threadIdx.x == 0) tcache = TreeCache{1, 0, 1, 0, 0};   // empty box
    unsigned long long rec_off = 0;
    unsigned long long xseq = P.xseq0;   // fused exchanges so far (partition mode)
    for (uint32_t ri = 0; ri < P.nroots; ++ri) {
    if (P.init_in_kernel) {
        // init_depths (kernels.py:134-140) + frontier {root}, as k_init
        const uint32_t root = P.roots[ri];
        const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
        const uint64_t nt = (uint64_t)gridDim.x * kBlock;
        const bool owned = root >= P.lo && root < P.hi;
        if (!PART) {
            const uint64_t n4 = P.n / 4;
            const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
            for (uint64_t i = tid; i < n4; i += nt) reinterpret_cast<int4 *>(P.depth)[i] = inf4;
            for (uint64_t i = n4 * 4 + tid; i < P.n; i += nt) P.depth[i] = kInf;
        } else {
            for (uint64_t i = P.lo + tid; i < P.hi; i += nt) P.depth[i] = kInf;
        }
        for (uint64_t w = P.wlo + tid; w < P.wend; w += nt) {
            const uint32_t bits = (owned && w == (root >> 5)) ? 1u << (root & 31) : 0u;
            P.visited[w] = bits;
            if (PART) P.vprev[w - P.wlo] = bits;
        }
        for (uint64_t w = tid; w < P.words; w += nt) P.fbm0[w] = (w == (root >> 5)) ? 1u << (root & 31) : 0u;
        grid.sync();
        if (lead) {
            if (owned) P.depth[root] = 0;
            P.q0[0] = root;
            for (int s = 0; s < 3; ++s) {
                P.ctr->qlen[s] = 0;
                P.ctr->units[s] = 0;
                P.ctr->count[s] = 0;
                P.ctr->cq3[s] = 0;
                P.ctr->es3[s] = 0;
                P.ctr->work[s] = 0;
                P.ctr->ps[s] = 0;
                P.ctr->pc[s] = 0;
                P.ctr->oe3[s] = 0;
            }
            P.ctr->cq = 0;
            P.ctr->inconsistent = 0;
        }
        grid.sync();
    }
    // the run_level-contract flag is fixed for the whole traversal (set by the
    // host's prepare or by the init above): every level's claims read a
    // shared-memory copy instead of an L2 round trip
    if (threadIdx.x == 0) s_incons = *(volatile unsigned *)&P.ctr->inconsistent;
    __syncthreads();
    unsigned long long frontier = 1, discovered = 1;
    int pk = 0, pv = 0;   // DEFAULT_KERNEL (adaptive.py:36-38)
    int cur = 0;
    bool has_q = true, has_bm = true;
    int pl_have = -1;      // carried pull candidate list: -1 none, 0 / 1 = pl_c0 / pl_c1
    uint32_t pl_n = 0;
    uint32_t solo_skip = 0xffffffffu;
    for (uint32_t level = 0;; ++level) {
        const unsigned long long t0 = lead ? globaltimer() : 0ull;
        if (threadIdx.x == 0)
            s_cls = P.fixed_pair >= 0 ? P.fixed_pair : mega_tree_class(T, frontier, discovered, &tcache);
        __syncthreads();
        const int cls = s_cls;
        const int fallback = cls == 254;
        if (!fallback) {
            pk = cls / 3;
            pv = cls % 3;
        }
        const unsigned long long tp = lead ? globaltimer() : 0ull;
        const int out = (int)(level % 3), zero = (int)((level + 1) % 3);
        if (lead) {
            P.ctr->qlen[zero] = 0;
            P.ctr->units[zero] = 0;
            P.ctr->count[zero] = 0;
            P.ctr->cq3[zero] = 0;
            P.ctr->es3[zero] = 0;
            P.ctr->work[zero] = 0;
            P.ctr->ps[zero] = 0;
            P.ctr->pc[zero] = 0;
            P.ctr->oe3[zero] = 0;
        }
        // (instrumented work-model runs take the grid path: it records N2 features)
        if (SOLO && P.solo_ctas && !P.instrument && has_q && level != solo_skip &&
            solo_fits(P, pk, frontier)) {
            // ---- cluster solo mode: cluster 0 runs this level and the
            // following small top-down levels alone (cluster barriers,
            // ~0.3 us) while every other CTA waits at ONE grid barrier
            if (blockIdx.x < P.solo_ctas) {
                cg::cluster_group cl = cg::this_cluster();
                // the level counters live in CTA 0's shared memory: the
                // cluster's tail atomics and the count readback are DSMEM
                // round trips instead of L2 ones
                unsigned *const cnt0 = ABFS_SOLO_DSMEM ? cl.map_shared_rank(&s_solo_cnt[0][0], 0) : nullptr;
                if (ABFS_SOLO_DSMEM) {
                    if (lead)
                        for (int s = 0; s < 3; ++s) s_solo_cnt[s][0] = s_solo_cnt[s][1] = 0;
                    cl.sync();
                }
                uint32_t L = level;
                int fb = fallback;
                unsigned long long ts = t0, tq = tp;
                int ppk = pk, ppv = pv;   // pair of the last executed level
                for (;;) {
                    const int o = (int)(L % 3), z = (int)((L + 1) % 3);
                    if (ABFS_SOLO_DSMEM && lead) s_solo_cnt[z][0] = s_solo_cnt[z][1] = 0;
                    if (lead && L != level) {
                        P.ctr->qlen[z] = 0;
                        P.ctr->units[z] = 0;
                        P.ctr->count[z] = 0;
                        P.ctr->cq3[z] = 0;
                        P.ctr->es3[z] = 0;
                        P.ctr->work[z] = 0;
                        P.ctr->ps[z] = 0;
                        P.ctr->pc[z] = 0;
                        P.ctr->oe3[z] = 0;
                    }
                    LevelCtx sc;
                    sc.acc = nullptr;
                    sc.depth = P.depth;
                    sc.visited = P.visited;
                    sc.fbm = cur ? P.fbm1 : P.fbm0;
                    sc.q_next = cur ? P.q0 : P.q1;
                    sc.q_tail = ABFS_SOLO_DSMEM ? cnt0 + 2 * o : &P.ctr->qlen[o];
                    sc.count = &P.ctr->count[o];
                    sc.units_tail = ABFS_SOLO_DSMEM ? cnt0 + 2 * o + 1 : &P.ctr->units[o];
                    sc.units = P.units;
                    sc.inconsistent = &s_incons;
                    sc.ctr = P.ctr;
                    sc.mb = nullptr;
                    sc.es = nullptr;
                    sc.work = &P.ctr->work[o];
                    sc.pull_light = P.pull_light;
                    sc.direct_claim = P.solo_direct;
                    sc.seq = 0;
                    sc.zero_slot = z;
                    sc.level = (int32_t)L;
                    sc.lvl1 = (int32_t)L + 1;
                    const uint32_t *qc = cur ? P.q1 : P.q0;
                    switch (pv) {
                    case 0: solo_light<0>(P, sc, pk, (uint32_t)frontier, qc, &sq); break;
                    case 1: solo_light<1>(P, sc, pk, (uint32_t)frontier, qc, &sq); break;
                    default: solo_light<2>(P, sc, pk, (uint32_t)frontier, qc, &sq); break;
                    }
                    cl.sync();
                    const unsigned nu = *(volatile unsigned *)sc.units_tail;
                    if (nu > kSoloUnits) {
                        // hubs in the frontier: the grid redoes this level (its
                        // claims so far stay counted in qlen[o]; units are rebuilt)
                        if (lead) {
                            P.ctr->units[o] = 0;
                            // the claims taken so far stay counted (the grid
                            // continues the global tail)
                            if (ABFS_SOLO_DSMEM) P.ctr->qlen[o] = s_solo_cnt[o][0];
                            P.solo->level = L;
                            P.solo->frontier = frontier;
                            P.solo->discovered = discovered;
                            P.solo->pk = ppk;
                            P.solo->pv = ppv;
                            P.solo->cur = cur;
                            P.solo->has_q = 1;
                            P.solo->has_bm = has_bm ? 1 : 0;
                            P.solo->done = 0;
                        }
                        break;
                    }
                    if (nu) {
                        switch (pv) {
                        case 0: heavy_body<0>(sc, &sq, P.out_off, P.dst, blockIdx.x, P.solo_ctas); break;
                        case 1: heavy_body<1>(sc, &sq, P.out_off, P.dst, blockIdx.x, P.solo_ctas); break;
                        default: heavy_body<2>(sc, &sq, P.out_off, P.dst, blockIdx.x, P.solo_ctas); break;
                        }
                        cl.sync();
                    }
                    const unsigned long long nw2 = *(volatile unsigned *)sc.q_tail;
                    if (lead && rec_off + L < P.cap) {
                        MegaRecord &r = P.recs[rec_off + L];
                        r.kernel = pk;
                        r.variant = pv;
                        r.fallback = fb;
                        r.converted = 0;
                        r.frontier = frontier;
                        r.new_count = nw2;
                        r.t_start = ts;
                        r.t_pred = tq;
                        r.t_end = globaltimer();
                        r.scanned = 0;
                    }
                    ppk = pk;
                    ppv = pv;
                    if (nw2 == 0) {
                        if (lead) {
                            P.solo->level = L;
                            P.solo->done = 1;
                        }
                        break;
                    }
                    frontier = nw2;
                    discovered += nw2;
                    cur ^= 1;
                    has_bm = false;
                    ++L;
                    // next level's decision (every cluster CTA, same result)
                    ts = lead ? globaltimer() : 0ull;
                    if (threadIdx.x == 0)
                        s_cls = P.fixed_pair >= 0 ? P.fixed_pair
                                                  : mega_tree_class(T, frontier, discovered, &tcache);
                    __syncthreads();
                    const int ncls = s_cls;
                    fb = ncls == 254;
                    const int npk = fb ? pk : ncls / 3, npv = fb ? pv : ncls % 3;
                    if (!solo_fits(P, npk, frontier)) {
                        if (lead) {
                            P.solo->level = L;
                            P.solo->frontier = frontier;
                            P.solo->discovered = discovered;
                            P.solo->pk = ppk;
                            P.solo->pv = ppv;
                            P.solo->cur = cur;
                            P.solo->has_q = 1;
                            P.solo->has_bm = 0;
                            P.solo->done = 0;
                        }
                        break;
                    }
                    pk = npk;
                    pv = npv;
                    tq = lead ? globaltimer() : 0ull;
                }
            }
            grid.sync();
            {
                volatile SoloState *st = P.solo;
                const uint32_t L = st->level;
                if (st->done) {
                    if (lead) P.n_levels[ri] = (unsigned long long)L + 1;
                    rec_off += L + 1;
                    break;
                }
                frontier = st->frontier;
                discovered = st->discovered;
                pk = st->pk;
                pv = st->pv;
                cur = st->cur;
                has_q = st->has_q != 0;
                has_bm = st->has_bm != 0;
                solo_skip = L;   // the grid runs level L (never solo again)
                pl_have = -1;    // solo levels are top-down
                level = L - 1;   // ++level
            }
            grid.sync();         // everyone has read the hand-off before it is reused
            continue;
        }
        uint32_t *fbm_cur = cur ? P.fbm1 : P.fbm0, *fbm_nxt = cur ? P.fbm0 : P.fbm1;
        uint32_t *q_cur = cur ? P.q1 : P.q0, *q_nxt = cur ? P.q0 : P.q1;
        const bool need_queue = (pk == 2 || pk == 4);
        int conv = 0;
        if (need_queue && !has_q) {          // bitmap -> queue (switch cost)
            bitmap_to_queue_grid(fbm_cur, P.words, q_cur, &P.ctr->cq3[out], warp_tot, &s_base);
            grid.sync();
            has_q = true;
            conv = 1;
        } else if (!need_queue && !has_bm) { // queue -> bitmap (switch cost)
            for (uint64_t w = (uint64_t)blockIdx.x * kBlock + threadIdx.x; w < P.words;
                 w += (uint64_t)gridDim.x * kBlock)
                fbm_cur[w] = 0u;
            grid.sync();
            for (uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x; i < frontier;
                 i += (uint64_t)gridDim.x * kBlock) {
                const uint32_t v = q_cur[i];
                atomicOr(fbm_cur + (v >> 5), 1u << (v & 31));
            }
            grid.sync();
            has_bm = true;
            conv = 1;
        }
        LevelCtx c;
        c.depth = P.depth;
        c.visited = P.visited;
        c.fbm = fbm_cur;
        c.q_next = q_nxt;
        c.q_tail = &P.ctr->qlen[out];
        c.count = &P.ctr->count[out];
        c.units_tail = &P.ctr->units[out];
        c.units = P.units;
        c.inconsistent = &s_incons;
        c.ctr = P.ctr;
        c.mb = nullptr;
        c.es = P.instrument ? &P.ctr->es3[out] : nullptr;
        c.work = &P.ctr->work[out];
        c.pull_light = P.pull_light;
        c.direct_claim = frontier <= P.direct_f ? 1u : 0u;
        // RED-mode top-down level (single graph, big frontier): the same for
        // every CTA (depends on the level's pair and frontier only)
        c.acc = (need_queue && P.acc && frontier >= P.red_frontier) ? P.acc : nullptr;
        // unfiltered RED only while most vertices are unvisited (the filter
        // load would mostly pass); late top-down levels keep it
        if (c.acc && P.red_direct && (P.n - discovered) * 2 > P.n) c.direct_claim = 1u;
        c.seq = 0;
        c.zero_slot = zero;
        c.level = (int32_t)level;
        c.lvl1 = (int32_t)level + 1;
        uint32_t *pull_next = PART ? P.fnext : fbm_nxt;
        // list-based pull (single graph): sweep after a top-down level, the
        // carried candidate list after a pull level
        PullLists pl;
        const bool use_pl = pk == 3 && P.pl_s && !PART;
        if (use_pl) {
            pl.s = P.pl_s;
            pl.c_in = pl_have >= 0 ? (pl_have ? P.pl_c1 : P.pl_c0) : nullptr;
            pl.c_out = pl_have == 0 ? P.pl_c1 : P.pl_c0;
            pl.s_tail = &P.ctr->ps[out];
            pl.c_tail = &P.ctr->pc[out];
        }
        const unsigned long long settled = discovered + P.n_noin;
        const bool wide = P.pull_wide_max && (settled >= P.n || P.n - settled <= P.pull_wide_max);
        int sflags;
        switch (pv) {
        case 0: sflags = mega_strategy<0>(P, c, pk, (uint32_t)frontier, q_cur, pull_next, &sq, &sn, &s_done, pfound, s_fetch, warp_tot, &s_base, wide, use_pl ? &pl : nullptr, pl_n, grid); break;
        case 1: sflags = mega_strategy<1>(P, c, pk, (uint32_t)frontier, q_cur, pull_next, &sq, &sn, &s_done, pfound, s_fetch, warp_tot, &s_base, wide, use_pl ? &pl : nullptr, pl_n, grid); break;
        default: sflags = mega_strategy<2>(P, c, pk, (uint32_t)frontier, q_cur, pull_next, &sq, &sn, &s_done, pfound, s_fetch, warp_tot, &s_base, wide, use_pl ? &pl : nullptr, pl_n, grid); break;
        }
        const bool topdown = pk != 3;
        if (use_pl) {   // the candidates this pull leaves for the next one
            pl_have = pl_have == 0 ? 1 : 0;
            pl_n = *(volatile unsigned *)&P.ctr->pc[out];
        } else {
            pl_have = -1;
        }
        unsigned long long nw;
        if (PART) {
            // fused frontier exchange: the visited bits this rank gained are
            // stored into every rank's next-frontier bitmap over peer memory,
            // then the ranks' counts are summed through the mailboxes
            const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
            const uint64_t nt = (uint64_t)gridDim.x * kBlock;
            uint32_t *const *nxt_tab = P.peer_fbm + (size_t)(cur ^ 1) * P.nranks;
            if (P.xsys == 2) {
                // LL exchange: each word goes to every rank's receive plane as
                // one 8-byte (epoch | word) store; every rank then rebuilds
                // its global next bitmap from its plane, spinning per word on
                // the epoch, and counts the level from it (popc) -- no fence,
                // one grid barrier.  Planes alternate by exchange parity: a
                // rank writes plane x%2 again only after every rank consumed
                // it (it waited on their exchange-(x+1) words first).
                const unsigned long long ep = (xseq + 1) & 0xffffffffull;
                const size_t plane = (size_t)(xseq & 1) * (P.words + 4);
                for (uint64_t w = P.wlo + tid; w < P.wend; w += nt) {
                    const uint32_t v = P.visited[w];
                    const uint32_t x = v & ~P.vprev[w - P.wlo];
                    P.vprev[w - P.wlo] = v;
                    const unsigned long long word = (ep << 32) | x;
                    for (uint32_t r = 0; r < P.nranks; ++r) {
                        unsigned long long *ll = reinterpret_cast<unsigned long long *>(
                            reinterpret_cast<char *>(P.peer_box[r]) + kLLOffset) + plane;
                        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(ll + w), "l"(word) : "memory");
                    }
                }
                const unsigned long long *mine = reinterpret_cast<const unsigned long long *>(
                    reinterpret_cast<const char *>(P.box) + kLLOffset) + plane;
                uint32_t *const fn = cur ? P.fbm0 : P.fbm1;   // this rank's next bitmap
                unsigned long long cnt = 0;
                const unsigned long long tw = globaltimer();
                bool ok = true;
                for (uint64_t w = tid; w < P.words && ok; w += nt) {
                    unsigned long long word;
                    for (;;) {
                        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(word) : "l"(mine + w) : "memory");
                        if ((word >> 32) == ep) break;
                        if (globaltimer() - tw > 20000000000ull) {   // a rank never sent
                            P.box->timeout = 1;
                            ok = false;
                            break;
                        }
                    }
                    fn[w] = (uint32_t)word;
                    cnt += __popc((uint32_t)word);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(kFull, cnt, o);
                if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&P.ctr->oe3[out], cnt);
                (void)ok;   // a timed-out CTA set box->timeout; every CTA reads it below
                ++xseq;
                grid.sync();
                nw = *(volatile unsigned *)&P.box->timeout
                         ? 0ull : *(volatile unsigned long long *)&P.ctr->oe3[out];
            } else {
                unsigned long long cnt = 0;
                for (uint64_t w = P.wlo + tid; w < P.wend; w += nt) {
                    const uint32_t v = P.visited[w];
                    const uint32_t x = v & ~P.vprev[w - P.wlo];
                    P.vprev[w - P.wlo] = v;
                    for (uint32_t r = 0; r < P.nranks; ++r) nxt_tab[r][w] = x;
                    cnt += __popc(x);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(kFull, cnt, o);
                if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = (unsigned)cnt;
                __syncthreads();
                // one cross-rank round per level, per CTA (no grid barrier, no
                // lead-only phase): each CTA adds its slice count into every
                // rank's mailbox sum and releases its arrival at system scope
                // (cumulative over the CTA's peer stores through the CTA
                // barrier), then waits for every CTA of every rank.  A rank's CTAs
                // add weights summing to exactly 2^32 per exchange, whatever its
                // grid size.  GPU-scoped when every rank shares this device
                // (P = 1, ranks sharing a GPU: ~1 us); system-scoped only when
                // forced (ABFS_XSYS=1: ~6 us per level on B200, which is why
                // cross-device ranks take the LL branch above).  Sums rotate over 3 slots: slot (x+1)%3 is cleared
                // by this rank before it signals exchange x, and no peer adds to
                // it before seeing that signal.
                if (threadIdx.x == 0) {
                    unsigned long long s = 0;
                    for (int w = 0; w < kWarps; ++w) s += warp_tot[w];
                    const uint32_t slot = (uint32_t)(xseq % 3);
                    if (lead) P.box->mk_sum[(xseq + 1) % 3] = 0;
                    const unsigned long long b = blockIdx.x, G = gridDim.x;
                    const unsigned long long wgt = ((b + 1) << 32) / G - (b << 32) / G;
                    for (uint32_t r = 0; r < P.nranks; ++r) {
                        if (s) atomicAdd_system(&P.peer_box[r]->mk_sum[slot], s);
                        if (P.xsys)
                            asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(&P.peer_box[r]->mk_arrive),
                                         "l"(wgt) : "memory");
                        else
                            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&P.peer_box[r]->mk_arrive),
                                         "l"(wgt) : "memory");
                    }
                    const unsigned long long expect = ((xseq + 1) * P.nranks) << 32, tw = globaltimer();
                    bool ok = true;
                    for (;;) {
                        unsigned long long a;
                        if (P.xsys)
                            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(&P.box->mk_arrive) : "memory");
                        else
                            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(&P.box->mk_arrive) : "memory");
                        if (a >= expect) break;
                        if (globaltimer() - tw > 20000000000ull) {   // a rank never arrived
                            P.box->timeout = 1;
                            ok = false;
                            break;
                        }
                        __nanosleep(32);
                    }
                    unsigned long long g = 0;
                    if (ok) g = *(volatile unsigned long long *)&P.box->mk_sum[slot];
                    s_nw = g;   // 0 ends the traversal
                }
                ++xseq;
                __syncthreads();
                nw = s_nw;
            }
        } else {
            nw = topdown ? (unsigned long long)*(volatile unsigned *)&P.ctr->qlen[out]
                         : *(volatile unsigned long long *)&P.ctr->count[out];
        }
        // N2 (instrumented runs only): sum of the out-degrees of this level's
        // discoveries -- the next frontier's out-edges -- reduced on the device
        unsigned long long next_oe = ~0ull;
        if (P.instrument && !PART) {
            const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
            const uint64_t nt = (uint64_t)gridDim.x * kBlock;
            unsigned long long acc = 0;
            if (topdown) {
                for (uint64_t i = tid; i < nw; i += nt) {
                    const uint32_t v = q_nxt[i];
                    acc += P.out_off[v + 1] - P.out_off[v];
                }
            } else {
                for (uint64_t w = tid; w < P.words; w += nt) {
                    uint32_t x = pull_next[w];
                    while (x) {
                        const uint64_t v = w * 32 + (__ffs(x) - 1);
                        acc += P.out_off[v + 1] - P.out_off[v];
                        x &= x - 1;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
            if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&P.ctr->oe3[out], acc);
            grid.sync();
            next_oe = *(volatile unsigned long long *)&P.ctr->oe3[out];
        }
#ifdef ABFS_NO_RECORDS   // overhead experiment only
        if (false) {
#else
        if (lead && rec_off + level < P.cap) {
#endif
            MegaRecord &r = P.recs[rec_off + level];
            r.kernel = pk;
            r.variant = pv;
            r.fallback = fallback;
            r.converted = conv;
            r.frontier = frontier;
            r.new_count = nw;
            r.t_start = t0;
            r.t_pred = tp;
            r.t_end = globaltimer();
            // partitions: this rank's count through the level's count variant
            r.next_out_edges = next_oe;
            r.scanned = PART ? (topdown ? (unsigned long long)*(volatile unsigned *)&P.ctr->qlen[out]
                                          : *(volatile unsigned long long *)&P.ctr->count[out])
                      : P.instrument ? *(volatile unsigned long long *)&P.ctr->es3[out] : 0ull;
        }
        if (nw == 0) {
            if (lead) P.n_levels[ri] = (unsigned long long)level + 1;
            rec_off += level + 1;
            break;
        }
        frontier = nw;
        discovered += nw;
        cur ^= 1;
        has_q = PART ? false : topdown;   // a partition's next frontier is the gathered bitmap
        has_bm = PART ? true : (!topdown || (sflags & kStratBitmap));
    }
    if (P.checksums) {
        // the traversal's last level ended at a grid barrier: every depth is final
        const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
        const uint64_t nt = (uint64_t)gridDim.x * kBlock;
        unsigned long long acc = 0;
        for (uint64_t v = P.lo + tid; v < P.hi; v += nt) acc += depth_mix(v, P.depth[v]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(P.checksums + ri, acc);
        grid.sync();   // before the next root's init overwrites the depths
    }
    }   // roots
}

}  // namespace abfs
