// bfs_kernels.cuh -- the 5 level strategies x 3 count epilogues, the
// queue<->bitmap frontier conversions and the state kernels (sm_100a).
//
// Semantics (all strategies; kernels.py:177-193):
//   * a level may only lower a depth to level+1;
//   * new_count = number of INF -> level+1 transitions (exactly once each);
//   * top-down strategies (edge, rev-edge, push, push-warp) lower any depth
//     > level+1 reached from a frontier vertex; pull only touches INF vertices.
//
// Frontier state on the device (the reference's implicit `depth == level`):
//   visited  u32 bitmap   bit v <=> depth[v] != INF (maintained exactly)
//   fbm      u32 bitmap   current frontier (depth == level)   [bitmap form]
//   q        u32 queue    current frontier vertex ids           [queue form]
//   noin     u32 bitmap   in-degree 0 (static per graph; pull never scans them)
// Top-down kernels emit the next frontier as a queue, pull emits a bitmap;
// the engine converts between forms only when the next kernel needs the
// other one (that conversion is the switching overhead).
//
// "Consistent" state (every finite depth <= level+1, which a BFS from
// init_depths always satisfies) lets a claim be a single atomicOr on the
// L2-resident visited bitmap followed by a plain depth store.  Arbitrary
// caller depth arrays (run_level contract) set ctr->inconsistent and claims
// fall back to atomicMin on the depth array, which reproduces _claim's
// "lower to level+1, count only INF transitions" rule exactly.
//
// Level completion: the last CTA of a level's final kernel publishes the
// counts into a host-mapped mailbox (seq-stamped), so the host learns the
// level result without a memcpy or an event synchronisation.
#pragma once

#include "common.cuh"

namespace abfs {

// Receiving side of the fused frontier exchange of a vertex partition
// (partition.cu, megakernel.cuh): every rank adds 1 to `arrive` per level
// (after its bitmap stores are visible system-wide) and writes its level
// count into counts[parity][rank].
// A rank's mailbox allocation also holds its LL receive planes (2 parities
// x words x 8 bytes) at kLLOffset: a peer stores (epoch << 32 | word) there
// with one 8-byte store (single-copy atomic), so the receiver needs no fence.
constexpr size_t kLLOffset = 4096;
struct PeerBox {
    unsigned long long arrive;
    unsigned long long mk_arrive;     // megakernel exchanges: 2^32 per rank per exchange
    unsigned long long mk_sum[3];     // megakernel exchanges: level count, rotating slots
    unsigned long long pad[3];
    unsigned long long counts[2][64];
    unsigned long long local;      // this rank's own count (accumulator)
    unsigned int timeout;          // set if a wait gave up
};

// Device counters.  Slots rotate per level call so that no separate zeroing
// launch is needed: call c appends into slot c%3 and zeroes slot (c+1)%3.
struct Ctr {
    unsigned int qlen[3];
    unsigned int units[3];
    unsigned long long count[3];
    unsigned int cq;             // bitmap->queue compaction cursor
    unsigned int inconsistent;   // 1 if some finite depth > level+1 (prepare)
    unsigned long long fcount;   // frontier size found by prepare
    unsigned long long reached_edges;
    unsigned long long reached_vertices;
    unsigned int done;           // finished-CTA ticket of the publishing kernel
    unsigned int pad;
    unsigned int cq3[3];         // megakernel: per-level compaction cursors
    unsigned int pad2;
    unsigned long long es3[3];   // megakernel: per-level pull scanned edges
    unsigned long long work[3];  // per-level dynamic work cursors
    unsigned int ps[3];          // megakernel pull: survivor-list tails
    unsigned int pc[3];          // megakernel pull: carried-candidate-list tails
    unsigned long long oe3[3];   // megakernel: N2 next-frontier out-edges (instrumented)
};

// Host-mapped result of the last level (written by the device).
struct Mailbox {
    unsigned long long seq;
    unsigned long long qlen;
    unsigned long long count;
    unsigned long long pad;
};

struct LevelCtx {
    int32_t *depth;
    uint32_t *visited;
    const uint32_t *fbm;         // current frontier bitmap (read-only here)
    uint32_t *q_next;            // next frontier queue (top-down)
    unsigned int *q_tail;        // = &ctr->qlen[out]
    unsigned long long *count;   // = &ctr->count[out] (pull)
    unsigned int *units_tail;    // = &ctr->units[out] (heavy work units)
    uint2 *units;
    const unsigned int *inconsistent;
    Ctr *ctr;
    Mailbox *mb;                 // device view of the host mailbox
    unsigned long long *es;      // optional: in-edges scanned by pull (instrumented runs)
    unsigned long long *work;    // dynamic work cursor of this level (= &ctr->work[out])
    uint32_t pull_light;         // pull phase A: entries each lane scans alone
    uint32_t direct_claim;       // claim4: no visited-word filter load before the atomic
    uint32_t *acc;               // non-null: RED-mode top-down claims (candidate bits are
                                 // OR-ed here fire-and-forget; red_compact_body settles them)
    unsigned long long seq;
    int zero_slot;
    int32_t level;
    int32_t lvl1;
};

#ifndef ABFS_RED_FILTER
#define ABFS_RED_FILTER 0   // RED-mode claim filter (A/B on B200, K24 / ER-32M switched GTEPS):
                            // 0 = visited check only (811 / 889), 1 = + skip bits already pending
                            // in acc (831 / 816), 2 = warp word dedupe (729 / 564), 3 = both (774 / 615)
#endif

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
#ifndef ABFS_QBUF
#define ABFS_QBUF 2048
#endif
constexpr int kQBuf = ABFS_QBUF;      // TWO_LEVEL CTA-local queue buffer (also the megakernel's pull lists)
constexpr int kEdgeTileMax = kBlock * 4 * 4;  // edge slots per CTA iteration (4 x uint4 / thread)
constexpr uint32_t kHeavy = 256;      // push-warp: degree above -> CTA units
constexpr uint32_t kUnit = 1024;      // edges per CTA work unit (4 steps of 256)
#ifndef ABFS_PUSH_HUB
#define ABFS_PUSH_HUB 64
#endif
constexpr uint32_t kPushHub = ABFS_PUSH_HUB;   // vertex push: degree above -> CTA units
constexpr uint64_t kSoloMaxDegree = 64;        // cluster solo mode: graphs of max out-degree <= this
constexpr uint32_t kPullLight = 32;   // pull phase A default (ABFS_PULL_LIGHT overrides)
#ifndef ABFS_PULL_HEAVY
#define ABFS_PULL_HEAVY 256
#endif
constexpr uint32_t kPullHeavy = ABFS_PULL_HEAVY;  // pull: warp scan up to this, CTA units above

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ void zero_slot(const LevelCtx &c) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c.ctr->qlen[c.zero_slot] = 0;
        c.ctr->units[c.zero_slot] = 0;
        c.ctr->count[c.zero_slot] = 0;
        c.ctr->work[c.zero_slot] = 0;
        c.ctr->cq = 0;
    }
}

// Last CTA to finish publishes (qlen, count) to the mapped mailbox.  Must be
// reached by every thread of every CTA of the level's final kernel.
__device__ __forceinline__ void publish(const LevelCtx &c) {
    // the CTA barrier orders every thread's counter atomics before thread
    // 0's (cumulative) gpu-scope fence, so one fence per CTA suffices
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(&c.ctr->done, 1u);
        if (ticket == gridDim.x - 1) {
            __threadfence();
            const unsigned long long q = atomicAdd(c.q_tail, 0u);
            const unsigned long long n = atomicAdd(c.count, 0ull);
            c.ctr->done = 0;
            volatile Mailbox *mb = c.mb;
            mb->qlen = q;
            mb->count = n;
            __threadfence_system();
            mb->seq = c.seq;
            __threadfence_system();
        }
    }
}

__device__ __forceinline__ bool in_bitmap(const uint32_t *bm, uint32_t v) {
    return (__ldg(bm + (v >> 5)) >> (v & 31)) & 1u;
}

// Could claiming v change anything?  (cheap filter before the atomic)
__device__ __forceinline__ bool claim_possible(const LevelCtx &c, uint32_t v, bool consistent) {
    if (consistent) return !((c.visited[v >> 5] >> (v & 31)) & 1u);
    return c.depth[v] > c.lvl1;
}

// _claim (kernels.py:177-193) for one candidate; true iff this thread won
// the INF -> level+1 transition of v.
__device__ __forceinline__ bool claim(const LevelCtx &c, uint32_t v, bool consistent) {
    const uint32_t bit = 1u << (v & 31);
    uint32_t *w = c.visited + (v >> 5);
    if (consistent) {
        if (*w & bit) return false;
        const uint32_t old = atomicOr(w, bit);
        if (old & bit) return false;
        c.depth[v] = c.lvl1;
        return true;
    }
    if (c.depth[v] <= c.lvl1) return false;
    const int32_t old = atomicMin(c.depth + v, c.lvl1);
    if (old != kInf) return false;
    atomicOr(w, bit);
    return true;
}

// Four candidates at once: the visited-word loads, then the atomics, are
// issued back to back (4 independent L2 round trips in flight instead of a
// chain of 4).  Same outcome as four claim() calls in order: a vertex
// repeated within the batch is won at most once.
__device__ __forceinline__ void claim4(const LevelCtx &c, const uint32_t (&v)[4],
                                       const bool (&act)[4], bool (&won)[4], bool consistent) {
    if (!consistent) {
#pragma unroll
        for (int k = 0; k < 4; ++k) won[k] = act[k] && claim(c, v[k], false);
        return;
    }
    uint32_t wv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        wv[k] = !act[k] ? 0xffffffffu : c.direct_claim ? 0u : c.visited[v[k] >> 5];
    if (c.acc) {
        // RED mode: no returning atomic, no depth write, no emission here --
        // the unvisited candidates' bits go to acc with fire-and-forget
        // reductions and red_compact_body claims them word by word
#if ABFS_RED_FILTER & 1
        // skip candidates whose bit is already pending (hub adjacency:
        // many frontier vertices share neighbours; a RED per duplicate
        // serialises on the word in L2)
        uint32_t av[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            av[k] = (act[k] && !(wv[k] & (1u << (v[k] & 31)))) ? __ldcg(c.acc + (v[k] >> 5)) : 0xffffffffu;
#endif
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t bit = 1u << (v[k] & 31);
#if ABFS_RED_FILTER & 1
            bool need = !(av[k] & bit);
#else
            bool need = act[k] && !(wv[k] & bit);
#endif
#if ABFS_RED_FILTER & 2
            // one RED per distinct word of the warp instruction
            const unsigned peers = __match_any_sync(kFull, need ? (v[k] >> 5) : 0xffffffffu);
            const uint32_t all = __reduce_or_sync(peers, need ? bit : 0u);
            need = need && lane_id() == (unsigned)(__ffs(peers) - 1);
#else
            const uint32_t all = bit;
#endif
            if (need)
                asm volatile("red.global.or.b32 [%0], %1;" ::"l"(c.acc + (v[k] >> 5)), "r"(all)
                             : "memory");
            won[k] = false;
        }
        return;
    }
    uint32_t old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t bit = 1u << (v[k] & 31);
        old[k] = (wv[k] & bit) ? bit : atomicOr(c.visited + (v[k] >> 5), bit);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        won[k] = act[k] && !(old[k] & (1u << (v[k] & 31)));
        if (won[k]) c.depth[v[k]] = c.lvl1;
    }
}

// ---------------------------------------------------------------------------
// Count epilogues (aggregate_count kernels.py:143-170).
// QEmit: winners append to the next queue; the append cursor IS the count.
//   VAR 0 DIRECT_ATOMIC    one global atomic per discovery
//   VAR 1 GROUP_REDUCE     warp ballot/popc, one global atomic per warp
//   VAR 2 TWO_LEVEL_REDUCE warp ballot -> CTA shared-memory queue, one
//                          global atomic per CTA flush (coalesced copy-out)
// emit() must be called by all 32 lanes of a warp together; tile_end() and
// finish() by all threads of the CTA.
// ---------------------------------------------------------------------------
// Single-lane atomics without the compiler's warp-aggregation wrapper.
__device__ __forceinline__ unsigned atom_add_shared(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                 : "=r"(old) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned atom_add_global(unsigned *p, unsigned v) {   // generic address
    unsigned old;
    asm volatile("atom.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

struct SmemQ {
    unsigned int n;
    unsigned int fail;
    unsigned int base;
    uint32_t buf[kQBuf];
};

template <int VAR>
struct QEmit {
    SmemQ *s;
    uint32_t *q;
    unsigned int *tail;

    __device__ __forceinline__ QEmit(SmemQ *sm, uint32_t *qq, unsigned int *t)
        : s(sm), q(qq), tail(t) {
        if (VAR == 2) {
            if (threadIdx.x == 0) { s->n = 0; s->fail = 0xffffffffu; }
            __syncthreads();
        }
    }

    __device__ __forceinline__ void emit(bool won, uint32_t v) {
        if (VAR == 0) {
            if (won) q[atomicAdd(tail, 1u)] = v;
            return;
        }
        const unsigned mask = __ballot_sync(kFull, won);
        if (!mask) return;
        const unsigned lane = lane_id();
        const int leader = __ffs(mask) - 1;
        const unsigned cnt = __popc(mask);
        const unsigned rank = __popc(mask & ((1u << lane) - 1u));
        if (VAR == 1) {
            unsigned b = 0;
            if (lane == (unsigned)leader) b = atom_add_global(tail, cnt);
            b = __shfl_sync(kFull, b, leader);
            if (won) q[b + rank] = v;
            return;
        }
        unsigned sb = 0;
        if (lane == (unsigned)leader) sb = atom_add_shared(&s->n, cnt);
        sb = __shfl_sync(kFull, sb, leader);
        if (sb + cnt <= (unsigned)kQBuf) {
            if (won) s->buf[sb + rank] = v;
        } else {  // CTA buffer full: this warp batch goes straight to global
            unsigned b = 0;
            if (lane == (unsigned)leader) {
                atomicMin(&s->fail, sb);
                b = atom_add_global(tail, cnt);
            }
            b = __shfl_sync(kFull, b, leader);
            if (won) q[b + rank] = v;
        }
    }

    // Four candidates per lane (a claim4 step) with ONE reservation for all
    // of the warp's winners: one atomic per step instead of up to four, and
    // the reservation is issued by lane 0 as a plain atom (the compiler's own
    // warp-aggregation wrapper around a leader-lane atomicAdd costs ~15
    // single-thread instructions per call).
    __device__ __forceinline__ void emit4(const bool (&won)[4], const uint32_t (&v)[4]) {
        if (VAR == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) emit(won[k], v[k]);
            return;
        }
        unsigned m[4], tot = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            m[k] = __ballot_sync(kFull, won[k]);
            tot += __popc(m[k]);
        }
        if (!tot) return;
        const unsigned lane = lane_id(), lt = (1u << lane) - 1u;
        unsigned base = 0;
        bool to_global = VAR == 1;
        if (VAR == 2) {
            if (lane == 0) base = atom_add_shared(&s->n, tot);
            base = __shfl_sync(kFull, base, 0);
            if (base + tot <= (unsigned)kQBuf) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (won[k]) s->buf[base + __popc(m[k] & lt)] = v[k];
                    base += __popc(m[k]);
                }
                return;
            }
            if (lane == 0) atomicMin(&s->fail, base);   // CTA buffer full: straight to global
            to_global = true;
        }
        if (to_global) {
            if (lane == 0) base = atom_add_global(tail, tot);
            base = __shfl_sync(kFull, base, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (won[k]) q[base + __popc(m[k] & lt)] = v[k];
                base += __popc(m[k]);
            }
        }
    }

    __device__ __forceinline__ void flush() {
        const unsigned n = min(s->n, s->fail);
        if (threadIdx.x == 0) s->base = n ? atomicAdd(tail, n) : 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) q[s->base + i] = s->buf[i];
        __syncthreads();
        if (threadIdx.x == 0) { s->n = 0; s->fail = 0xffffffffu; }
        __syncthreads();
    }

    // Between block-uniform loop iterations: flush once half full.
    __device__ __forceinline__ void tile_end() {
        if (VAR != 2) return;
        __syncthreads();
        if (s->n >= (unsigned)kQBuf / 2) flush();
    }

    __device__ __forceinline__ void finish() {
        if (VAR != 2) return;
        __syncthreads();
        flush();
    }
};

// Count-only epilogue (pull): same three shapes over a warp's found mask.
//   DIRECT    one global atomic per discovery
//   GROUP     warp popc; the warp's sum goes out in one global atomic per
//             sub-tile of work (tile())
//   TWO_LEVEL warp popc -> CTA shared counter (one shared atomic per warp
//             sub-tile), one global atomic per CTA
template <int VAR>
struct CEmit {
    unsigned int *sn;
    unsigned long long *count;
    unsigned acc = 0;   // GROUP / TWO_LEVEL: this warp's open sum

    __device__ __forceinline__ CEmit(unsigned int *smem_n, unsigned long long *c)
        : sn(smem_n), count(c) {
        if (VAR == 2) {
            if (threadIdx.x == 0) *sn = 0;
            __syncthreads();
        }
    }

    __device__ __forceinline__ void add(unsigned mask) {  // warp-uniform mask
        if (VAR == 0) {
            if ((mask >> lane_id()) & 1u) atomicAdd(count, 1ull);
        } else {
            acc += __popc(mask);
        }
    }

    // per-lane discovery counts (all lanes call)
    __device__ __forceinline__ void add_n(unsigned n) {
        if (VAR == 0) {
            if (n) atomicAdd(count, (unsigned long long)n);
        } else {
            acc += __reduce_add_sync(kFull, n);
        }
    }

    __device__ __forceinline__ void tile() {   // warp-uniform
        if (VAR != 0 && acc) {
            if (lane_id() == 0) {
                if (VAR == 1) atomicAdd(count, (unsigned long long)acc);
                else atom_add_shared(sn, acc);
            }
            acc = 0;
        }
    }

    __device__ __forceinline__ void finish() {
        tile();
        if (VAR != 2) return;
        __syncthreads();
        if (threadIdx.x == 0 && *sn) atomicAdd(count, (unsigned long long)*sn);
    }
};

// ---------------------------------------------------------------------------
// EDGE_LIST (run_level_edge_list + _relax_from_edges, kernels.py:196-219):
// one item per forward slot e; active iff origins[e] is in the frontier;
// relax destinations[e].  Persistent CTAs stream origins with four 128-bit
// evict-first loads in flight per thread; destinations are gathered only
// for active slots.
// REV_EDGE_LIST (kernels.py:222-231): item per reverse slot f, head
// sources[f], tail rev_owner[f].  The sorted tail stream is read first so
// that sources[f] is gathered only when the claim could have an effect.
// ---------------------------------------------------------------------------
template <int VAR, bool REV, int kEdgeVec = 4>
__device__ __forceinline__ void edge_body(const LevelCtx &c, SmemQ *sq,
                                          const uint32_t *__restrict__ stream_arr,
                                          const uint32_t *__restrict__ gather_arr, uint64_t m) {
    QEmit<VAR> em(sq, c.q_next, c.q_tail);
    const bool consistent = (*c.inconsistent == 0);
    constexpr uint64_t kEdgeTile = kBlock * 4 * kEdgeVec;  // slots per CTA iteration
    for (uint64_t tile = (uint64_t)blockIdx.x * kEdgeTile; tile < m;
         tile += (uint64_t)gridDim.x * kEdgeTile) {
        uint4 t4[kEdgeVec];
#pragma unroll
        for (int h = 0; h < kEdgeVec; ++h) {
            const uint64_t e = tile + (uint64_t)h * (kBlock * 4) + threadIdx.x * 4u;
            if (e + 4 <= m) {
                t4[h] = __ldcs(reinterpret_cast<const uint4 *>(stream_arr + e));
            } else {
                t4[h].x = e + 0 < m ? stream_arr[e + 0] : 0u;
                t4[h].y = e + 1 < m ? stream_arr[e + 1] : 0u;
                t4[h].z = e + 2 < m ? stream_arr[e + 2] : 0u;
                t4[h].w = e + 3 < m ? stream_arr[e + 3] : 0u;
            }
        }
        bool act[kEdgeVec][4];
        bool any = false;
#pragma unroll
        for (int h = 0; h < kEdgeVec; ++h) {
            const uint64_t e = tile + (uint64_t)h * (kBlock * 4) + threadIdx.x * 4u;
            const uint32_t s4[4] = {t4[h].x, t4[h].y, t4[h].z, t4[h].w};
            if (!REV) {
                // origins are sorted: one frontier word usually covers all four
                const uint32_t w0 = s4[0] >> 5, w3 = s4[3] >> 5;
                if (w0 == w3) {
                    const uint32_t fw = __ldg(c.fbm + w0);
#pragma unroll
                    for (int k = 0; k < 4; ++k) act[h][k] = (e + k < m) && ((fw >> (s4[k] & 31)) & 1u);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) act[h][k] = (e + k < m) && in_bitmap(c.fbm, s4[k]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    act[h][k] = (e + k < m) && claim_possible(c, s4[k], consistent);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) any |= act[h][k];
        }
        if (__any_sync(kFull, any)) {  // idle warps skip the claim/emit stage
#pragma unroll
            for (int h = 0; h < kEdgeVec; ++h) {
                const uint64_t e = tile + (uint64_t)h * (kBlock * 4) + threadIdx.x * 4u;
                const uint32_t s4[4] = {t4[h].x, t4[h].y, t4[h].z, t4[h].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    bool won = false;
                    uint32_t v = 0;
                    if (act[h][k]) {
                        if (!REV) {
                            v = __ldg(gather_arr + e + k);
                            won = claim(c, v, consistent);
                        } else {
                            v = s4[k];
                            if (in_bitmap(c.fbm, __ldg(gather_arr + e + k))) won = claim(c, v, consistent);
                        }
                    }
                    em.emit(won, v);
                }
            }
        }
        em.tile_end();
    }
    em.finish();
}

// ---------------------------------------------------------------------------
// TMA-streamed edge list.  The head stream (origins / reverse owners, 4 bytes
// per slot, read exactly once per level) is moved by the copy engine: one
// thread arms an mbarrier and issues a 1-D bulk copy (cp.async.bulk) of the
// CTA's next chunk into a shared-memory stage while the CTA processes the
// previous one, so the stream's DRAM latency leaves the threads' critical
// path and registers hold no in-flight stream data.  The per-slot logic is
// edge_body's (frontier test on sorted origins, dst/src gathered only for
// active slots, claim + count epilogue).
// ---------------------------------------------------------------------------
constexpr int kStreamStages = 2;

// Two-stage ring of CH-slot chunks.  full[s]: armed by the producer with the
// chunk's byte count, completed by the copy engine.  empty[s]: one arrival
// per warp once it holds its slots in registers; the producer (thread 0)
// waits on it before re-filling the stage, so no warp ever waits for another
// warp's claim work (no CTA-wide barrier per chunk).  Barriers are set up once
// per kernel; the parity of every stage's next phase is carried in `uses`.
template <uint32_t CH>
struct SmemStreamT {
    uint32_t buf[kStreamStages][CH];
    unsigned long long full[kStreamStages], empty[kStreamStages];
    uint32_t uses[kStreamStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait(const unsigned long long *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

template <uint32_t CH>
__device__ __forceinline__ void stream_init(SmemStreamT<CH> *ss) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStreamStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&ss->full[s])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                         :: "r"(smem_u32(&ss->empty[s])), "r"(kWarps) : "memory");
            ss->uses[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

template <uint32_t CH>
__device__ __forceinline__ void stream_issue(SmemStreamT<CH> *ss, int stage, const uint32_t *src,
                                             uint32_t bytes) {
    // generic-proxy reads of this stage (ordered by the empty barrier) before
    // the async-proxy write
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(&ss->full[stage])), "r"(bytes) : "memory");
    // evict-first: the 2-4 GB stream must not push the L2-resident bitmaps
    // (visited / frontier, probed by every claim) out of L2
    unsigned long long policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(ss->buf[stage])), "l"(src), "r"(bytes),
                    "r"(smem_u32(&ss->full[stage])), "l"(policy) : "memory");
}

template <int VAR, bool REV, uint32_t CH>
__device__ __forceinline__ void edge_stream_body(const LevelCtx &c, SmemQ *sq, SmemStreamT<CH> *ss,
                                                 const uint32_t *__restrict__ stream_arr,
                                                 const uint32_t *__restrict__ gather_arr,
                                                 uint64_t m) {
    static_assert(CH % (kBlock * 4) == 0, "chunk = whole uint4 groups");
    QEmit<VAR> em(sq, c.q_next, c.q_tail);
    const bool consistent = (*c.inconsistent == 0);
    const uint64_t nchunks = (m + CH - 1) / CH;
    auto chunk_bytes = [&](uint64_t ch) -> uint32_t {
        const uint64_t slots = min((uint64_t)CH, m - ch * CH);
        return (uint32_t)((slots * 4 + 15) & ~15ull);   // arrays are padded by 16 bytes
    };
    uint32_t u[kStreamStages];
#pragma unroll
    for (int s = 0; s < kStreamStages; ++s) u[s] = ss->uses[s];
    __syncthreads();   // every thread has read `uses` before thread 0 advances it
    if (threadIdx.x == 0)
        for (int s = 0; s < kStreamStages; ++s) {
            const uint64_t ch = blockIdx.x + (uint64_t)s * gridDim.x;
            if (ch < nchunks) stream_issue(ss, s, stream_arr + ch * CH, chunk_bytes(ch));
        }
    uint32_t k = 0;
    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++k) {
        const int stage = (int)(k % kStreamStages);
        const uint32_t par = (u[stage] + k / kStreamStages) & 1u;
        mbar_wait(&ss->full[stage], par);
        const uint64_t tile = ch * CH;
        constexpr int kGroups = CH / (kBlock * 4);
        uint4 t4[kGroups];
#pragma unroll
        for (int h = 0; h < kGroups; ++h)
            t4[h] = reinterpret_cast<const uint4 *>(ss->buf[stage])[h * kBlock + threadIdx.x];
        __syncwarp();
        if (lane_id() == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                         :: "r"(smem_u32(&ss->empty[stage])) : "memory");
        if (threadIdx.x == 0) {
            const uint64_t nxt = ch + (uint64_t)kStreamStages * gridDim.x;
            if (nxt < nchunks) {
                mbar_wait(&ss->empty[stage], par);   // all warps hold this chunk
                stream_issue(ss, stage, stream_arr + nxt * CH, chunk_bytes(nxt));
            }
        }
        bool act[kGroups][4];
        bool any = false;
#pragma unroll
        for (int h = 0; h < kGroups; ++h) {
            const uint64_t e = tile + (uint64_t)h * (kBlock * 4) + threadIdx.x * 4u;
            const uint32_t s4[4] = {t4[h].x, t4[h].y, t4[h].z, t4[h].w};
            if (!REV) {
                const uint32_t w0 = s4[0] >> 5, w3 = s4[3] >> 5;
                if (w0 == w3 && e + 3 < m) {
                    const uint32_t fw = __ldg(c.fbm + w0);
#pragma unroll
                    for (int q = 0; q < 4; ++q) act[h][q] = (fw >> (s4[q] & 31)) & 1u;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) act[h][q] = (e + q < m) && in_bitmap(c.fbm, s4[q]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    act[h][q] = (e + q < m) && claim_possible(c, s4[q], consistent);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) any |= act[h][q];
        }
        if (__any_sync(kFull, any)) {  // idle warps skip the claim/emit stage
#pragma unroll
            for (int h = 0; h < kGroups; ++h) {
                const uint64_t e = tile + (uint64_t)h * (kBlock * 4) + threadIdx.x * 4u;
                const uint32_t s4[4] = {t4[h].x, t4[h].y, t4[h].z, t4[h].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    bool won = false;
                    uint32_t v = 0;
                    if (act[h][q]) {
                        if (!REV) {
                            v = __ldg(gather_arr + e + q);
                            won = claim(c, v, consistent);
                        } else {
                            v = s4[q];
                            if (in_bitmap(c.fbm, __ldg(gather_arr + e + q))) won = claim(c, v, consistent);
                        }
                    }
                    em.emit(won, v);
                }
            }
        }
        em.tile_end();
    }
    __syncthreads();   // every wait of this call is done before `uses` advances
    if (threadIdx.x == 0)
        for (int s = 0; s < kStreamStages; ++s)
            ss->uses[s] = u[s] + (k + kStreamStages - 1 - s) / kStreamStages;   // chunks on stage s
    __syncthreads();
    em.finish();
}

// 4 KB stages: the unified L1 / shared memory must keep most of its capacity
// as L1 (frontier and visited probes of every claim hit there)
constexpr uint32_t kStreamChunk = 1024;
using SmemStream = SmemStreamT<kStreamChunk>;

template <int VAR, bool REV>
__global__ void __launch_bounds__(kBlock)
k_edge(LevelCtx c, const uint32_t *__restrict__ stream_arr,
       const uint32_t *__restrict__ gather_arr, uint64_t m) {
    __shared__ SmemQ sq;
    __shared__ __align__(16) SmemStream ss;
    zero_slot(c);
    stream_init(&ss);
    edge_stream_body<VAR, REV, kStreamChunk>(c, &sq, &ss, stream_arr, gather_arr, m);
    publish(c);
}

// ---------------------------------------------------------------------------
// VERTEX_PUSH (run_level_vertex_push + _push_block, kernels.py:234-267):
// one thread per frontier vertex walks its out-adjacency in order.  A
// vertex of degree > kPushHub is not walked by one thread (a Kronecker hub
// has ~10^5-10^6 edges: one thread would serialise the whole level); its
// adjacency is queued as kUnit-edge CTA work units for k_heavy, exactly as
// in push-warp.  Semantics are unchanged (same claims, same counts).
// ---------------------------------------------------------------------------
template <int VAR>
__device__ __forceinline__ void push_body(const LevelCtx &c, SmemQ *sq,
                                          const uint32_t *__restrict__ q, uint32_t F,
                                          const uint32_t *__restrict__ out_off,
                                          const uint32_t *__restrict__ dst, uint32_t bid,
                                          uint32_t nblk) {
    QEmit<VAR> em(sq, c.q_next, c.q_tail);
    const bool consistent = (*c.inconsistent == 0);
    for (uint32_t base = bid * kBlock; base < F; base += nblk * kBlock) {
        const uint32_t i = base + threadIdx.x;
        uint32_t j = 0, e = 0;
        if (i < F) {
            const uint32_t u = __ldg(q + i);
            j = __ldg(out_off + u);
            e = __ldg(out_off + u + 1);
            if (e - j > kPushHub) {
                const uint32_t nu = (e - j + kUnit - 1) / kUnit;
                const uint32_t s = atomicAdd(c.units_tail, nu);
                for (uint32_t k = 0; k < nu; ++k)
                    c.units[s + k] = make_uint2(j + k * kUnit, min(e, j + (k + 1) * kUnit));
                j = e;
            }
        }
        while (__any_sync(kFull, j < e)) {
            uint32_t v[4];
            bool act[4], won[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                act[k] = j + k < e;
                v[k] = act[k] ? __ldg(dst + j + k) : 0u;
            }
            j = min(e, j + 4);
            claim4(c, v, act, won, consistent);
            em.emit4(won, v);
        }
        em.tile_end();
    }
    em.finish();
}

template <int VAR>
__global__ void __launch_bounds__(kBlock)
k_push(LevelCtx c, const uint32_t *__restrict__ q, uint32_t F,
       const uint32_t *__restrict__ out_off, const uint32_t *__restrict__ dst) {
    __shared__ SmemQ sq;
    zero_slot(c);
    push_body<VAR>(c, &sq, q, F, out_off, dst, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// VERTEX_PUSH_WARP (run_level_push_warp, kernels.py:303-322; virtual-warp
// method PAPER.md:414-432): a virtual warp of VW lanes owns one frontier
// vertex at a time and strides its adjacency in VW-wide coalesced chunks.
// Vertices with degree > kHeavy are split into kUnit-edge CTA work units
// processed by k_heavy (CTA-centric push), so hubs never serialise a warp.
// ---------------------------------------------------------------------------
template <int VAR>
__device__ __forceinline__ void push_warp_body(const LevelCtx &c, SmemQ *sq,
                                               const uint32_t *__restrict__ q, uint32_t F,
                                               const uint32_t *__restrict__ out_off,
                                               const uint32_t *__restrict__ dst, int vw_log2,
                                               uint32_t bid, uint32_t nblk) {
    QEmit<VAR> em(sq, c.q_next, c.q_tail);
    const bool consistent = (*c.inconsistent == 0);
    const uint32_t VW = 1u << vw_log2;
    const uint32_t per = 32u >> vw_log2;            // frontier entries per warp step
    const uint32_t per_block = per * kWarps;
    const unsigned lane = lane_id();
    const uint32_t sub = lane >> vw_log2, sl = lane & (VW - 1);
    const uint32_t wib = threadIdx.x >> 5;
    for (uint32_t bb = bid * per_block; bb < F; bb += nblk * per_block) {
        const uint32_t i = bb + wib * per + sub;
        uint32_t j = 0, e = 0;
        if (i < F) {
            const uint32_t u = __ldg(q + i);
            const uint32_t b = __ldg(out_off + u), en = __ldg(out_off + u + 1);
            if (en - b > kHeavy) {
                if (sl == 0) {
                    const uint32_t nu = (en - b + kUnit - 1) / kUnit;
                    const uint32_t s = atomicAdd(c.units_tail, nu);
                    for (uint32_t k = 0; k < nu; ++k)
                        c.units[s + k] = make_uint2(b + k * kUnit, min(en, b + (k + 1) * kUnit));
                }
            } else {
                j = b + sl;
                e = en;
            }
        }
        while (__any_sync(kFull, j < e)) {
            uint32_t v[4];
            bool act[4], won[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                act[k] = j + k * VW < e;
                v[k] = act[k] ? __ldg(dst + j + k * VW) : 0u;
            }
            j += 4 * VW;
            claim4(c, v, act, won, consistent);
            em.emit4(won, v);
        }
        em.tile_end();
    }
    em.finish();
}

template <int VAR, int VWL>
__global__ void __launch_bounds__(kBlock)
k_push_warp(LevelCtx c, const uint32_t *__restrict__ q, uint32_t F,
            const uint32_t *__restrict__ out_off, const uint32_t *__restrict__ dst) {
    __shared__ SmemQ sq;
    zero_slot(c);
    push_warp_body<VAR>(c, &sq, q, F, out_off, dst, VWL, blockIdx.x, gridDim.x);
}

template <int VAR>
__device__ __forceinline__ void heavy_body(const LevelCtx &c, SmemQ *sq,
                                           const uint32_t *__restrict__ out_off,
                                           const uint32_t *__restrict__ dst, uint32_t bid,
                                           uint32_t nblk) {
    QEmit<VAR> em(sq, c.q_next, c.q_tail);
    const bool consistent = (*c.inconsistent == 0);
    const unsigned nunits = *(volatile unsigned *)c.units_tail;
    // push units carry their adjacency slice [x, y) directly (no offset
    // lookup); the next unit's descriptor is loaded while this one runs
    uint2 nxt = bid < nunits ? c.units[bid] : make_uint2(0, 0);
    for (unsigned w = bid; w < nunits; w += nblk) {
        const uint2 un = nxt;
        if (w + nblk < nunits) nxt = c.units[w + nblk];
        const uint32_t b = un.x, e = un.y;
        for (uint32_t jb = b; jb < e; jb += kBlock * 4) {
            uint32_t v[4];
            bool act[4], won[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t j = jb + k * kBlock + threadIdx.x;
                act[k] = j < e;
                v[k] = act[k] ? __ldg(dst + j) : 0u;
            }
            claim4(c, v, act, won, consistent);
            em.emit4(won, v);
        }
        em.tile_end();
    }
    em.finish();
}

template <int VAR>
__global__ void __launch_bounds__(kBlock)
k_heavy(LevelCtx c, const uint32_t *__restrict__ out_off, const uint32_t *__restrict__ dst) {
    __shared__ SmemQ sq;
    heavy_body<VAR>(c, &sq, out_off, dst, blockIdx.x, gridDim.x);
    publish(c);
}

// ---------------------------------------------------------------------------
// RED-mode epilogue of a top-down level (megakernel).  The edge phase OR-ed
// the bits of unvisited candidates into `acc` with fire-and-forget
// reductions (claim4 with c.acc set); here every bitmap word is settled by
// exactly one thread: new = acc & ~visited, visited |= new, depth[new] =
// level + 1, the new vertices are appended to the next queue (the count
// variant shapes the reservations: DIRECT one global atomic per discovery,
// GROUP one per warp, TWO_LEVEL one per CTA tile), acc is cleared (it is
// all-zero between levels), and fbm_out (if given) receives the next
// frontier bitmap.  The set of discoveries is the same as with per-edge
// atomic claims: every unvisited vertex with a frontier in-neighbour.
// ---------------------------------------------------------------------------
template <int VAR>
__device__ __forceinline__ void red_compact_body(const LevelCtx &c, uint32_t *acc,
                                                 uint32_t *fbm_out, uint64_t words,
                                                 unsigned *warp_tot, unsigned *s_base) {
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
    for (uint64_t w0 = (uint64_t)blockIdx.x * kBlock; w0 < words; w0 += (uint64_t)gridDim.x * kBlock) {
        const uint64_t w = w0 + threadIdx.x;
        uint32_t nw = 0;
        if (w < words) {
            const uint32_t a = acc[w];
            if (a) {
                acc[w] = 0u;
                const uint32_t vis = c.visited[w];
                nw = a & ~vis;
                if (nw) c.visited[w] = vis | nw;
            }
            if (fbm_out) fbm_out[w] = nw;
        }
        const unsigned cnt = __popc(nw);
        unsigned pos = 0;
        if (VAR == 0) {
            uint32_t x = nw;
            while (x) {
                const uint32_t v = (uint32_t)(w * 32 + (__ffs(x) - 1));
                c.depth[v] = c.lvl1;
                c.q_next[atomicAdd(c.q_tail, 1u)] = v;
                x &= x - 1;
            }
            continue;
        }
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        if (VAR == 1) {
            const unsigned tot = __shfl_sync(kFull, incl, 31);
            unsigned b = 0;
            if (lane == 31 && tot) b = atom_add_global(c.q_tail, tot);
            pos = __shfl_sync(kFull, b, 31) + incl - cnt;
        } else {
            if (lane == 31) warp_tot[wid] = incl;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned acc_ = 0;
                for (int i = 0; i < kWarps; ++i) {
                    const unsigned t = warp_tot[i];
                    warp_tot[i] = acc_;
                    acc_ += t;
                }
                *s_base = acc_ ? atomicAdd(c.q_tail, acc_) : 0u;
            }
            __syncthreads();
            pos = *s_base + warp_tot[wid] + incl - cnt;
            __syncthreads();   // warp_tot / s_base are reused by the next tile
        }
        uint32_t x = nw;
        while (x) {
            const uint32_t v = (uint32_t)(w * 32 + (__ffs(x) - 1));
            c.depth[v] = c.lvl1;
            c.q_next[pos++] = v;
            x &= x - 1;
        }
    }
}

// ---------------------------------------------------------------------------
// VERTEX_PULL (run_level_vertex_pull, kernels.py:270-300): unvisited
// vertices scan their in-neighbours and stop at the first frontier vertex.
// The CTA takes chunks of 8 sub-tiles (one global atomic), its warps take
// sub-tiles of 8 words (256 vertices) from a shared cursor.  Fully settled
// words (visited or in-degree 0) cost one load and one store.  The
// candidates of a sub-tile (unvisited, in-degree > 0) are compacted into a
// per-warp shared-memory list, so every lane carries a real vertex (a word
// with 3 candidates no longer idles 29 lanes through a chain of dependent
// loads):
//   probe 0                   two candidates per lane, first in-neighbour
//                             from the dense first_src array
//   survivors, compacted again in place, 32 per step:
//   first pull_light entries  each lane scans its own list, 16-byte loads
//   rest <= kPullHeavy        the warp scans the pending remainders together,
//                             128 entries per step (load balanced)
//   rest larger               kUnit-edge CTA units (k_pull_heavy)
// with early exit on the first frontier in-neighbour in every case.  Found
// bits gather in a per-warp shared word array; the warp owns its visited /
// next-frontier words, so they are written without global atomics, and every
// next-frontier word is written (no clearing pass).
// ---------------------------------------------------------------------------
#ifndef ABFS_PULL_SUB
#define ABFS_PULL_SUB 8
#endif
constexpr int kPullSub = ABFS_PULL_SUB;      // words per sub-tile
constexpr int kPullList = kPullSub * 32;     // candidate list entries per warp
#ifndef ABFS_PROBE_BATCH
#define ABFS_PROBE_BATCH 2
#endif
constexpr int kProbeBatch = ABFS_PROBE_BATCH;  // candidates per lane whose first probes are in flight together
#ifndef ABFS_PULL_CHUNK
#define ABFS_PULL_CHUNK 8
#endif
constexpr int kPullChunkSubs = ABFS_PULL_CHUNK;  // sub-tiles per CTA chunk fetch
// CTA chunk cursor: one 32-bit shared word (chunk id << 8 | next sub-tile),
// so the fetch is a native shared atomic (a 64-bit one is a CAS loop)
constexpr uint32_t kFetchInit = 0xfffffeu, kFetchDone = 0xffffffu;

template <int VAR, int G = 1>
__device__ __forceinline__ void pull_body(const LevelCtx &c, unsigned int *sn,
                                          const uint32_t *__restrict__ in_off,
                                          const uint32_t *__restrict__ src,
                                          const uint32_t *__restrict__ first_src,
                                          const uint32_t *__restrict__ noin,
                                          uint32_t *__restrict__ fbm_next, uint64_t word0,
                                          uint64_t words, uint32_t *wbuf, uint32_t *wfound,
                                          unsigned int *sfetch /* [2] */) {
    // words [word0, words) of the bitmaps (a vertex partition passes its
    // owned range; bitmap/offset pointers are indexed by global ids);
    // wbuf = kPullList entries, wfound = kPullSub words, both per warp
    // Work distribution: the CTA fetches chunks of kPullChunkSubs sub-tiles
    // with one global atomic; its warps take single sub-tiles from the
    // chunk through a shared-memory cursor (packed chunk id : next index).
    // The warp that overflows the cursor refills it; the others wait for the
    // new chunk id.  Few global atomics (sparse levels stay cheap) and an
    // 8-word grain at the end of the level (dense levels balance).
    CEmit<VAR> em(sn, c.count);
    const unsigned lane = lane_id();
    // word indices fit 32 bits (|V| < 2^32): 32-bit bookkeeping keeps the
    // megakernel's register pressure down
    const uint32_t w0 = (uint32_t)word0, wend = (uint32_t)words;
    // G sub-tiles per warp fetch ("unit"): G = 1 on dense levels (fine
    // grain balances the level's end); G = 4 on sparse levels, where the
    // sweep is latency-bound -- all 32 lanes load visited / in-degree-0 words
    // at once (4x the loads in flight) and sub-tiles without candidates cost
    // nothing more
    static_assert(G * kPullSub <= 32 && (kPullSub & (kPullSub - 1)) == 0, "pull unit");
    const uint32_t nsub = (wend - w0 + kPullSub - 1) / kPullSub;
    const uint32_t nunit = (nsub + G - 1) / G;
    const uint32_t nchunks = (nunit + kPullChunkSubs - 1) / kPullChunkSubs;
    // sfetch[0] = cursor (chunk id << 8 | next sub-tile), sfetch[1] = the
    // CTA's NEXT chunk, fetched one chunk ahead: the global atomic's round
    // trip is paid by the warp that installs a chunk while the other warps
    // work on it (a refill on demand stalled all 8 warps once per chunk --
    // most of a sparse pull level's sweep time).  CTA b starts on chunk b;
    // dynamic chunks are numbered from gridDim on.
    const uint32_t nblk = gridDim.x;
    if (threadIdx.x == 0) {
        sfetch[0] = blockIdx.x < nchunks ? (blockIdx.x << 8) : (kFetchDone << 8);
        sfetch[1] = kFetchInit;
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < nchunks) {
        const uint32_t g = nblk + (uint32_t)atomicAdd(c.work, 1ull);
        *(volatile unsigned int *)(sfetch + 1) = g < nchunks ? g : kFetchDone;
    }
    unsigned long long scanned = 0;
    for (;;) {
        uint32_t st = 0;
        if (lane == 0) st = atom_add_shared(sfetch, 1u);
        st = __shfl_sync(kFull, st, 0);
        uint32_t cid = st >> 8, sidx = st & 0xffu;
        if (cid == kFetchDone) break;
        if (sidx > (uint32_t)kPullChunkSubs) {   // another warp is installing the next chunk
            if (lane == 0)
                while ((*(volatile unsigned int *)sfetch >> 8) == cid) {
                }
            __syncwarp();
            continue;
        }
        if (sidx == (uint32_t)kPullChunkSubs) {  // this warp installs the prefetched chunk
            uint32_t g = 0;
            if (lane == 0) {
                while ((g = *(volatile unsigned int *)(sfetch + 1)) == kFetchInit) {
                }
                *(volatile unsigned int *)(sfetch + 1) = kFetchInit;
                atomicExch(sfetch, g != kFetchDone ? (g << 8) | 1u : kFetchDone << 8);
                if (g != kFetchDone) {   // and fetches the one after it
                    const uint32_t g2 = nblk + (uint32_t)atomicAdd(c.work, 1ull);
                    *(volatile unsigned int *)(sfetch + 1) = g2 < nchunks ? g2 : kFetchDone;
                }
            }
            g = __shfl_sync(kFull, g, 0);
            if (g == kFetchDone) break;
            cid = g;
            sidx = 0;
        }
        const uint32_t ug = cid * kPullChunkSubs + sidx;
        if (ug >= nunit) continue;
        const uint32_t ubase = w0 + ug * (G * kPullSub);
        const uint32_t myw = ubase + lane;
        const bool mine = lane < (unsigned)(G * kPullSub) && myw < wend;
        uint32_t vis = 0xffffffffu, cand = 0;
        if (mine) {
            vis = c.visited[myw];
            cand = ~(vis | __ldg(noin + myw));   // padding bits are set in noin
            if (!cand) fbm_next[myw] = 0u;
        }
        if (G > 1 && !__any_sync(kFull, cand != 0u)) continue;
        // candidate counts, scanned within each sub-tile's kPullSub lanes
        const uint32_t cnt = __popc(cand);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < kPullSub; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o, kPullSub);
            if ((lane & (kPullSub - 1)) >= (unsigned)o) incl += t;
        }
#pragma unroll 1
        for (int s = 0; s < G; ++s) {
            const uint32_t total = __shfl_sync(kFull, incl, s * kPullSub + kPullSub - 1);
            if (!total) continue;
            const uint32_t wbase = ubase + s * kPullSub;
            if (lane < (unsigned)kPullSub) wfound[lane] = 0u;
            {
                // compact the candidates of the sub-tile into wbuf (vertex
                // order): all 32 lanes scatter one word at a time (lane l
                // places bit l of word w), no serial per-bit loop
                const uint32_t excl = incl - cnt;
                const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                for (int w = 0; w < kPullSub; ++w) {
                    const uint32_t cw = __shfl_sync(kFull, cand, s * kPullSub + w);
                    const uint32_t ow = __shfl_sync(kFull, excl, s * kPullSub + w);
                    if ((cw >> lane) & 1u) wbuf[ow + __popc(cw & lt)] = (wbase + w) * 32 + lane;
                }
            }
            __syncwarp();
            // probe 0 for every candidate (two per lane at once): the offsets
            // and the first in-neighbour (dense array, coalesced over
            // consecutive candidates), then the frontier bits -- the smallest
            // in-neighbour is a hub on skewed graphs, so most candidates stop
            // here without touching src.  The rest are compacted in place to
            // the front of wbuf, so the scans below run on full warps (a
            // scan over the probe-0 survivors of a raw batch kept ~3 of 32
            // lanes busy).
            uint32_t npend = 0;
            for (uint32_t base = 0; base < total; base += 32 * kProbeBatch) {
                uint32_t vv[kProbeBatch], jj[kProbeBatch], ee[kProbeBatch], ff0[kProbeBatch];
#pragma unroll
                for (int h = 0; h < kProbeBatch; ++h) {
                    const bool has = base + h * 32 + lane < total;
                    vv[h] = has ? wbuf[base + h * 32 + lane] : 0u;
                    jj[h] = has ? __ldg(in_off + vv[h]) : 0u;
                    ee[h] = has ? __ldg(in_off + vv[h] + 1) : 0u;
                    ff0[h] = has ? __ldg(first_src + vv[h]) : 0u;
                }
                __syncwarp();   // every lane has read its entries before the in-place writes
#pragma unroll
                for (int h = 0; h < kProbeBatch; ++h) {
                    bool found = false;
                    if (jj[h] < ee[h]) {
                        ++scanned;
                        found = in_bitmap(c.fbm, ff0[h]);
                    }
                    if (found) {
                        c.depth[vv[h]] = c.lvl1;
                        atomicOr(wfound + ((vv[h] >> 5) - wbase), 1u << (vv[h] & 31));
                    }
                    em.add(__ballot_sync(kFull, found));
                    const bool pend = !found && jj[h] + 1 < ee[h];
                    const unsigned pm = __ballot_sync(kFull, pend);
                    if (pend) wbuf[npend + __popc(pm & ((1u << lane) - 1u))] = vv[h];
                    npend += __popc(pm);
                }
            }
            __syncwarp();
            for (uint32_t base = 0; base < npend; base += 32) {
                const bool has = base + lane < npend;
                const uint32_t v = has ? wbuf[base + lane] : 0u;
                uint32_t j = has ? __ldg(in_off + v) + 1 : 0u;   // L1 hits: just probed
                const uint32_t e = has ? __ldg(in_off + v + 1) : 0u;
                bool found = false;
                // phase A: each candidate scans up to pull_light more of its
                // in-neighbours, one aligned 16-byte load per step (one L1
                // wavefront per lane instead of four), early exit
                const uint32_t ja = min(e, j + c.pull_light);
                while (__any_sync(kFull, j < ja)) {
                    if (j < ja) {
                        const uint32_t b4 = j & ~3u;
                        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(src + b4));
                        const uint32_t jb = min(ja, b4 + 4);
                        scanned += jb - j;
                        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
                        bool hit = false;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (b4 + k >= j && b4 + k < jb) hit |= in_bitmap(c.fbm, xs[k]);
                        if (hit) {
                            found = true;
                            j = e;
                        } else {
                            j = jb;
                        }
                    }
                }
                // super-heavy remainders go to CTA units (k_pull_heavy)
                bool pend = !found && j < e;
                if (pend && e - j > kPullHeavy) {
                    const uint32_t nu = (e - j + kUnit - 1) / kUnit;
                    const uint32_t s = atomicAdd(c.units_tail, nu);
                    // a unit carries its absolute start slot: the units cover
                    // exactly the unscanned remainder [j, e)
                    for (uint32_t k = 0; k < nu; ++k) c.units[s + k] = make_uint2(v, j + k * kUnit);
                    pend = false;
                }
                // phase B: the warp walks the concatenation of all pending
                // remainders 128 entries per step, skipping owners already
                // found, until every pending owner is found or exhausted
                const unsigned pmask = __ballot_sync(kFull, pend);
                if (pmask) {
                    const uint32_t rem = pend ? e - j : 0u;
                    uint32_t inc2 = rem;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(kFull, inc2, o);
                        if (lane >= (unsigned)o) inc2 += t;
                    }
                    const uint32_t excl = inc2 - rem;
                    const uint32_t tot2 = __shfl_sync(kFull, inc2, 31);
                    unsigned fmask = 0;
                    for (uint32_t b2 = 0; b2 < tot2; b2 += 128) {
                        unsigned hit_bits = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t p = b2 + k * 32 + lane;
                            // owner = last lane whose exclusive offset <= p
                            int owner = 0;
#pragma unroll
                            for (int step = 16; step > 0; step >>= 1) {
                                const uint32_t ex = __shfl_sync(kFull, excl, owner + step);
                                if (ex <= p) owner += step;
                            }
                            const uint32_t oj = __shfl_sync(kFull, j, owner);
                            const uint32_t oex = __shfl_sync(kFull, excl, owner);
                            if (p < tot2 && !((fmask >> owner) & 1u)) {
                                ++scanned;
                                if (in_bitmap(c.fbm, __ldg(src + oj + (p - oex)))) hit_bits |= 1u << owner;
                            }
                        }
                        fmask |= __reduce_or_sync(kFull, hit_bits);
                        if ((fmask & pmask) == pmask) break;
                    }
                    found |= (fmask >> lane) & 1u;
                }
                if (found) {
                    c.depth[v] = c.lvl1;
                    atomicOr(wfound + ((v >> 5) - wbase), 1u << (v & 31));
                }
                em.add(__ballot_sync(kFull, found));
            }
            em.tile();
            __syncwarp();
            if (mine && cand && (lane / kPullSub) == (unsigned)s) {
                const uint32_t fm = wfound[lane & (kPullSub - 1)];
                fbm_next[myw] = fm;
                if (fm) c.visited[myw] = vis | fm;
            }
            __syncwarp();
        }
    }
    em.finish();
    if (c.es) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) scanned += __shfl_down_sync(kFull, scanned, o);
        if (lane == 0 && scanned) atomicAdd(c.es, scanned);
    }
}

// Per-warp scratch of pull_body inside one CTA.
struct SmemPull {
    uint32_t list[kWarps][kPullList];
    uint32_t found[kWarps][kPullSub];
};

template <int VAR>
__global__ void __launch_bounds__(kBlock)
k_pull(LevelCtx c, const uint32_t *__restrict__ in_off, const uint32_t *__restrict__ src,
       const uint32_t *__restrict__ first_src, const uint32_t *__restrict__ noin,
       uint32_t *__restrict__ fbm_next, uint64_t word0, uint64_t words) {
    __shared__ unsigned int sn;
    __shared__ SmemPull sp;
    __shared__ unsigned int sfetch[2];
    zero_slot(c);
    const unsigned w = threadIdx.x >> 5;
    pull_body<VAR>(c, &sn, in_off, src, first_src, noin, fbm_next, word0, words, sp.list[w],
                   sp.found[w], sfetch);
}

// CTA-centric pull for in-degree > kPullHeavy: each CTA scans one kUnit
// segment [un.y, un.y + kUnit) of one vertex's unscanned in-list remainder
// with early exit; the first unit to find a
// frontier in-neighbour claims the vertex (atomicOr on its visited bit).
__device__ __forceinline__ void pull_heavy_body(const LevelCtx &c, int *s_done_p,
                                                const uint32_t *__restrict__ in_off,
                                                const uint32_t *__restrict__ src,
                                                uint32_t *fbm_next) {
    int &s_done = *s_done_p;
    const unsigned nunits = *(volatile unsigned *)c.units_tail;
    for (unsigned w = blockIdx.x; w < nunits; w += gridDim.x) {
        const uint2 un = c.units[w];
        const uint32_t v = un.x, bit = 1u << (v & 31);
        const uint32_t b = un.y;   // absolute start slot of this unit
        const uint32_t e = min(__ldg(in_off + v + 1), b + kUnit);
        if (threadIdx.x == 0) s_done = (*(volatile uint32_t *)(c.visited + (v >> 5)) & bit) ? 1 : 0;
        __syncthreads();
        bool hit = false;
        if (!s_done) {
            for (uint32_t jb = b; jb < e; jb += kBlock * 4) {
                if (c.es && threadIdx.x == 0) atomicAdd(c.es, (unsigned long long)min(kBlock * 4u, e - jb));
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t x = jb + k * kBlock + threadIdx.x;
                    if (x < e) hit |= in_bitmap(c.fbm, __ldg(src + x));
                }
                if (__syncthreads_or(hit)) {
                    hit = true;
                    break;
                }
            }
        }
        if (threadIdx.x == 0 && hit) {
            const uint32_t old = atomicOr(c.visited + (v >> 5), bit);
            if (!(old & bit)) {
                c.depth[v] = c.lvl1;
                atomicOr(fbm_next + (v >> 5), bit);
                atomicAdd(c.count, 1ull);
            }
        }
        __syncthreads();
    }
}

static __global__ void __launch_bounds__(kBlock)
k_pull_heavy(LevelCtx c, const uint32_t *__restrict__ in_off, const uint32_t *__restrict__ src,
             uint32_t *fbm_next) {
    __shared__ int s_done;
    pull_heavy_body(c, &s_done, in_off, src, fbm_next);
    publish(c);
}

// ---------------------------------------------------------------------------
// Frontier conversions (switching overhead).
// ---------------------------------------------------------------------------

// bitmap -> queue: per-word popc, warp + CTA scan, one atomic per CTA.
// One call covers the kBlock words starting at word0 (CTA-uniform).
__device__ __forceinline__ void bitmap_to_queue_tile(const uint32_t *__restrict__ fbm,
                                                     uint64_t words, uint64_t word0, uint32_t *q,
                                                     unsigned int *cursor, unsigned *warp_tot,
                                                     unsigned *base) {
    const uint64_t word = word0 + threadIdx.x;
    uint32_t w = word < words ? fbm[word] : 0u;
    const unsigned cnt = __popc(w);
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(kFull, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int i = 0; i < kWarps; ++i) {
            const unsigned t = warp_tot[i];
            warp_tot[i] = acc;
            acc += t;
        }
        *base = acc ? atomicAdd(cursor, acc) : 0u;
    }
    __syncthreads();
    unsigned pos = *base + warp_tot[wid] + incl - cnt;
    __syncthreads();   // warp_tot / base are reused by the next tile
    while (w) {
        const int b = __ffs(w) - 1;
        q[pos++] = (uint32_t)(word * 32 + b);
        w &= w - 1;
    }
}

// bitmap -> queue for a persistent grid: CTA b converts the contiguous word
// range [b*per, (b+1)*per), each thread a contiguous run of its words (loads
// issued back to back), one CTA scan and ONE queue reservation per CTA (the
// tile version above makes every CTA walk several 256-word tiles, each with
// its own barriers and global atomic).
__device__ __forceinline__ void bitmap_to_queue_grid(const uint32_t *__restrict__ fbm, uint64_t words,
                                                     uint32_t *q, unsigned int *cursor,
                                                     unsigned *warp_tot, unsigned *base) {
    const uint64_t per = (words + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = min(words, (uint64_t)blockIdx.x * per), b1 = min(words, b0 + per);
    const uint64_t K = (per + kBlock - 1) / kBlock;
    const uint64_t t0 = min(b1, b0 + threadIdx.x * K), t1 = min(b1, t0 + K);
    unsigned cnt = 0;
    for (uint64_t w = t0; w < t1; ++w) cnt += __popc(fbm[w]);
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(kFull, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int i = 0; i < kWarps; ++i) {
            const unsigned t = warp_tot[i];
            warp_tot[i] = acc;
            acc += t;
        }
        *base = acc ? atomicAdd(cursor, acc) : 0u;
    }
    __syncthreads();
    unsigned pos = *base + warp_tot[wid] + incl - cnt;
    __syncthreads();   // warp_tot / base are reused by the caller's next use
    if (!cnt) return;
    for (uint64_t w = t0; w < t1; ++w) {
        uint32_t x = fbm[w];
        while (x) {
            q[pos++] = (uint32_t)(w * 32 + (__ffs(x) - 1));
            x &= x - 1;
        }
    }
}

static __global__ void __launch_bounds__(kBlock)
k_bitmap_to_queue(const uint32_t *__restrict__ fbm, uint64_t words, uint32_t *q,
                  unsigned int *cursor) {
    __shared__ unsigned warp_tot[kWarps];
    __shared__ unsigned base;
    bitmap_to_queue_tile(fbm, words, (uint64_t)blockIdx.x * kBlock, q, cursor, warp_tot, &base);
}

// queue -> bitmap (bitmap cleared by the caller).
static __global__ void k_queue_to_bitmap(const uint32_t *__restrict__ q, uint32_t F, uint32_t *fbm) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
        const uint32_t v = q[i];
        atomicOr(fbm + (v >> 5), 1u << (v & 31));
    }
}

// init_depths (kernels.py:134-140) + frontier {root} in both forms.
static __global__ void k_init(int32_t *depth, uint32_t *visited, uint32_t *fbm, uint32_t *q,
                       uint64_t n, uint64_t words, uint32_t root) {
    const uint64_t word = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (word >= words) return;
    const uint64_t v0 = word * 32;
    if (v0 + 32 <= n) {
        int4 *d4 = reinterpret_cast<int4 *>(depth + v0);
        const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
#pragma unroll
        for (int k = 0; k < 8; ++k) d4[k] = inf4;
    } else {
        for (uint64_t v = v0; v < n; ++v) depth[v] = kInf;
    }
    uint32_t bits = 0;
    if ((root >> 5) == word) {
        bits = 1u << (root & 31);
        depth[root] = 0;
        q[0] = root;
    }
    visited[word] = bits;
    fbm[word] = bits;
}

// noin: bit v set iff in-degree(v) == 0 or v >= n (padding).
static __global__ void k_noin(const uint32_t *__restrict__ in_off, uint64_t n, uint64_t words,
                       uint32_t *noin) {
    const uint64_t word = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (word >= words) return;
    uint32_t bits = 0;
    for (int k = 0; k < 32; ++k) {
        const uint64_t v = word * 32 + k;
        if (v >= n || in_off[v + 1] == in_off[v]) bits |= 1u << k;
    }
    noin[word] = bits;
}

// Largest out-degree (decides the megakernel's solo mode).
static __global__ void __launch_bounds__(kBlock)
k_count_bits(const uint32_t *__restrict__ bm, uint64_t words, unsigned long long *out) {
    unsigned long long c = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        c += __popc(bm[w]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

static __global__ void k_max_degree(const uint32_t *__restrict__ out_off, uint64_t n,
                                    unsigned int *out) {
    unsigned int mx = 0;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        mx = max(mx, out_off[v + 1] - out_off[v]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_down_sync(kFull, mx, o));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// Rebuild frontier bitmap + visited bitmap from an arbitrary depth array.
static __global__ void __launch_bounds__(kBlock)
k_prepare(const int32_t *__restrict__ depth, uint64_t n, uint64_t words, int32_t level,
          uint32_t *fbm, uint32_t *visited, Ctr *ctr) {
    const unsigned lane = lane_id();
    const uint64_t warp = ((uint64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * kBlock) >> 5;
    const int64_t lvl1 = (int64_t)level + 1;
    for (uint64_t word = warp; word < words; word += nwarps) {
        const uint64_t v = word * 32 + lane;
        const int32_t d = v < n ? depth[v] : kInf;
        const unsigned fm = __ballot_sync(kFull, v < n && d == level);
        const unsigned vm = __ballot_sync(kFull, d != kInf);
        const bool bad = __any_sync(kFull, d != kInf && (int64_t)d > lvl1);
        if (lane == 0) {
            fbm[word] = fm;
            visited[word] = vm;
            if (fm) atomicAdd(&ctr->fcount, (unsigned long long)__popc(fm));
            if (bad) ctr->inconsistent = 1;
        }
    }
}

// Σ out-degree over reached vertices (GTEPS numerator) + reached count.
static __global__ void __launch_bounds__(kBlock)
k_reached(const int32_t *__restrict__ depth, const uint32_t *__restrict__ out_off,
          uint64_t n, Ctr *ctr) {
    unsigned long long e = 0, r = 0;
    for (uint64_t v = (uint64_t)blockIdx.x * kBlock + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * kBlock) {
        if (depth[v] != kInf) {
            e += out_off[v + 1] - out_off[v];
            ++r;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_down_sync(kFull, e, o);
        r += __shfl_down_sync(kFull, r, o);
    }
    if (lane_id() == 0 && (e || r)) {
        atomicAdd(&ctr->reached_edges, e);
        atomicAdd(&ctr->reached_vertices, r);
    }
}

// Per-depth histograms for the work model (bench roofline): for each depth
// d < nlev: vertex count, Σ out-degree, Σ in-degree; slot nlev = unreached.
static __global__ void __launch_bounds__(kBlock)
k_level_hist(const int32_t *__restrict__ depth, const uint32_t *__restrict__ out_off,
             const uint32_t *__restrict__ in_off, uint64_t n, uint32_t nlev,
             unsigned long long *hist /* 3 * (nlev + 1) */) {
    __shared__ unsigned long long sh[3 * 65];
    const bool local = nlev < 64;
    for (int i = threadIdx.x; i < 3 * 65; i += kBlock) sh[i] = 0;
    __syncthreads();
    for (uint64_t v = (uint64_t)blockIdx.x * kBlock + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * kBlock) {
        const int32_t d = depth[v];
        const uint32_t slot = (d == kInf || d < 0 || (uint32_t)d >= nlev) ? nlev : (uint32_t)d;
        const unsigned long long od = out_off[v + 1] - out_off[v], id = in_off[v + 1] - in_off[v];
        if (local) {
            atomicAdd(&sh[slot], 1ull);
            atomicAdd(&sh[65 + slot], od);
            atomicAdd(&sh[130 + slot], id);
        } else {
            atomicAdd(&hist[slot], 1ull);
            atomicAdd(&hist[(nlev + 1) + slot], od);
            atomicAdd(&hist[2 * (nlev + 1) + slot], id);
        }
    }
    __syncthreads();
    if (local)
        for (uint32_t i = threadIdx.x; i <= nlev; i += kBlock) {
            if (sh[i]) atomicAdd(&hist[i], sh[i]);
            if (sh[65 + i]) atomicAdd(&hist[(nlev + 1) + i], sh[65 + i]);
            if (sh[130 + i]) atomicAdd(&hist[2 * (nlev + 1) + i], sh[130 + i]);
        }
}

// aggregate_count on the device with the three reduction shapes.
template <int VAR>
__global__ void __launch_bounds__(kBlock)
k_aggregate(const long long *__restrict__ counts, uint64_t n, unsigned long long *total) {
    __shared__ unsigned long long part[kWarps];
    const uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    unsigned long long x = i < n ? (unsigned long long)counts[i] : 0ull;
    if constexpr (VAR == 0) {
        if (i < n) atomicAdd(total, x);
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(kFull, x, o);
        if constexpr (VAR == 1) {
            if (lane_id() == 0) atomicAdd(total, x);
        } else {
            if (lane_id() == 0) part[threadIdx.x >> 5] = x;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long s = 0;
                for (int k = 0; k < kWarps; ++k) s += part[k];
                atomicAdd(total, s);
            }
        }
    }
}

}  // namespace abfs
