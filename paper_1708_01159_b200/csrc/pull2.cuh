// pull2.cuh -- VERTEX_PULL (run_level_vertex_pull, kernels.py:270-300) for the
// device-resident level loop, split into two grid-wide phases joined by
// candidate lists instead of one per-warp chain per sub-tile.
//
// The per-sub-tile pull (bfs_kernels.cuh pull_body) walks every candidate
// through a chain of dependent round trips (visited word -> offsets and
// first in-neighbour -> frontier bit -> in-list -> frontier bits) inside one
// warp, so a level costs (sub-tiles per warp) x (chain latency) however few
// bytes it moves.  Here the chain is cut at its natural seams:
//
//   phase 1, probe 0  every candidate tests its first in-neighbour
//                     (first_src, the smallest one: a hub on skewed graphs)
//                     against the frontier bitmap.  SWEEP form (after a
//                     top-down level): a warp owns 32 bitmap words, each lane
//                     one word -- one visited/in-degree-0 load, one 128-byte
//                     run of first_src, probes of its candidates; found bits
//                     are written straight into visited / next frontier /
//                     depth (the lane owns the word), the rest are appended
//                     to the survivor list S.  LIST form (after a pull
//                     level): the candidates are exactly the previous pull's
//                     carried list C_in (every unvisited vertex with
//                     in-degree > 0 that it did not find); each entry is
//                     probed and tagged in place, and the next-frontier
//                     bitmap is cleared in the same pass.
//   grid barrier
//   phase 2, scans    survivors (S, or the untagged C_in entries) scan the
//                     rest of their in-lists with early exit: per lane up to
//                     pull_light entries with 16-byte loads, then the warp
//                     walks all pending remainders load-balanced, remainders
//                     > kPullHeavy become CTA units (pull_heavy_body).  Found
//                     vertices are claimed with atomicOr on visited / next
//                     frontier; the others are appended to C_out, the next
//                     pull level's candidate list (a vertex handed to CTA
//                     units is appended too: if a unit finds it, the next
//                     list pass drops it on its visited bit).
//
// Every list holds each vertex at most once per level and every claim is
// arbitrated by the visited bit, so the level's discoveries, count and depth
// writes are exactly the reference's (all unvisited vertices with a
// frontier in-neighbour).
#pragma once

#include "bfs_kernels.cuh"

namespace abfs {

constexpr uint32_t kFoundTag = 0x80000000u;   // list entry found by phase 1 (|V| <= 2^31)
constexpr uint32_t kDropped = 0xffffffffu;    // list entry already visited

struct PullLists {
    uint32_t *s;            // survivors of a sweep phase 1 [V]
    uint32_t *c_in;         // this level's carried candidates (list form) [V]
    uint32_t *c_out;        // candidates the level leaves for the next pull [V]
    unsigned int *s_tail;   // = &ctr->ps[out]
    unsigned int *c_tail;   // = &ctr->pc[out]
};

// CTA-aggregated reservation of each thread's n list slots: one global
// atomic per CTA call (a reservation per warp put ~20 K same-address atomics
// on the list tail per level -- the largest stall of the first version).
// All threads of the CTA call; warp_tot [kWarps] / s_base are shared scratch.
__device__ __forceinline__ uint32_t cta_reserve(unsigned int *tail, uint32_t n, unsigned *warp_tot,
                                                unsigned *s_base) {
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
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
        *s_base = acc ? atomicAdd(tail, acc) : 0u;
    }
    __syncthreads();
    const uint32_t pos = *s_base + warp_tot[wid] + incl - n;
    __syncthreads();   // warp_tot / s_base are reused by the next call
    return pos;
}

// Phase 1, sweep form: a warp owns 32 consecutive bitmap words (lane r loads
// word r's visited / in-degree-0 bits) and walks them one word per round
// with lane = vertex, so the first_src loads and the depth stores of a round
// are single coalesced 128-byte accesses; found bits gather in lane r.
template <int VAR>
__device__ __forceinline__ void pull2_sweep(const LevelCtx &c, CEmit<VAR> &em,
                                            const uint32_t *__restrict__ noin,
                                            const uint32_t *__restrict__ first_src,
                                            uint32_t *__restrict__ fbm_next, uint64_t w0,
                                            uint64_t wend, const PullLists &L,
                                            unsigned *warp_tot, unsigned *s_base,
                                            unsigned long long &scanned) {
    const unsigned lane = lane_id();
    // CTA-uniform iterations (cta_reserve has barriers): 8 warps x 32 words
    for (uint64_t cb = w0 + (uint64_t)blockIdx.x * (kWarps * 32); cb < wend;
         cb += (uint64_t)gridDim.x * (kWarps * 32)) {
        const uint64_t base = cb + (threadIdx.x >> 5) * 32;
        const uint64_t w = base + lane;
        uint32_t cand = 0, vis = 0;
        if (w < wend) {
            vis = c.visited[w];
            cand = ~(vis | __ldg(noin + w));   // padding bits are set in noin
        }
        uint32_t found = 0;   // lane r: found bits of word r
        unsigned rounds = __ballot_sync(kFull, cand != 0u);
        while (rounds) {
            // up to 4 words per step: their first_src rows are loaded together
            int rr[4];
            uint32_t cw[4], ff[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                rr[k] = rounds ? __ffs(rounds) - 1 : -1;
                if (rounds) rounds &= rounds - 1;
                cw[k] = __shfl_sync(kFull, cand, rr[k] < 0 ? 0 : rr[k]);
                if (rr[k] < 0) cw[k] = 0u;
                const bool mine = (cw[k] >> lane) & 1u;
                ff[k] = mine ? __ldg(first_src + (base + rr[k]) * 32 + lane) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool mine = (cw[k] >> lane) & 1u;
                const bool hit = mine && in_bitmap(c.fbm, ff[k]);
                const unsigned fm = __ballot_sync(kFull, hit);
                if (hit) c.depth[(base + rr[k]) * 32 + lane] = c.lvl1;
                if (rr[k] >= 0 && lane == (unsigned)rr[k]) found = fm;
                scanned += mine;
            }
        }
        if (w < wend) {
            fbm_next[w] = found;
            if (found) c.visited[w] = vis | found;
        }
        em.add_n(__popc(found));
        // survivors -> S (vertex order within a word)
        uint32_t sv = cand & ~found;
        uint32_t pos = cta_reserve(L.s_tail, __popc(sv), warp_tot, s_base);
        while (sv) {
            L.s[pos++] = (uint32_t)(w * 32 + (__ffs(sv) - 1));
            sv &= sv - 1;
        }
        em.tile();
    }
}

// Phase 1, list form: probe and tag the carried candidates in place; clear
// the next-frontier bitmap (written again in phase 2 only by atomics).
__device__ __forceinline__ void pull2_list_probe(const LevelCtx &c, uint32_t *list, uint32_t n,
                                                 const uint32_t *__restrict__ first_src,
                                                 uint32_t *__restrict__ fbm_next, uint64_t w0,
                                                 uint64_t wend, unsigned long long &scanned) {
    const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    const uint64_t nt = (uint64_t)gridDim.x * kBlock;
    for (uint64_t w = w0 + tid; w < wend; w += nt) fbm_next[w] = 0u;
    for (uint64_t i = tid; i < n; i += nt) {
        const uint32_t v = list[i];
        if ((c.visited[v >> 5] >> (v & 31)) & 1u) {   // found by a CTA unit last level
            list[i] = kDropped;
            continue;
        }
        ++scanned;
        if (in_bitmap(c.fbm, __ldg(first_src + v))) list[i] = v | kFoundTag;
    }
}

// Phase 2: the survivors' in-list scans.  `list` entries: vertex ids,
// optionally tagged kFoundTag (claim without scanning) or kDropped.
template <int VAR>
__device__ __forceinline__ void pull2_scan(const LevelCtx &c, CEmit<VAR> &em, const uint32_t *list,
                                           uint32_t n, const uint32_t *__restrict__ in_off,
                                           const uint32_t *__restrict__ src, uint32_t *fbm_next,
                                           const PullLists &L, unsigned *warp_tot, unsigned *s_base,
                                           unsigned long long &scanned) {
    const unsigned lane = lane_id();
    // CTA-uniform iterations (cta_reserve has barriers): 8 warps x 32 entries
    for (uint32_t cb = blockIdx.x * kBlock; cb < n; cb += gridDim.x * kBlock) {
        const uint32_t i = cb + threadIdx.x;
        uint32_t v = i < n ? list[i] : kDropped;
        bool found = false, keep = false, scan = false;
        uint32_t j = 0, e = 0;
        if (v != kDropped) {
            if (v & kFoundTag) {
                v &= ~kFoundTag;
                found = true;
            } else {
                j = __ldg(in_off + v) + 1;   // probe 0 (first_src) failed
                e = __ldg(in_off + v + 1);
                scan = true;
            }
        }
        // phase A: each lane scans up to pull_light more entries alone,
        // one aligned 16-byte load per step, early exit
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
        bool pend = scan && !found && j < e;
        if (pend && e - j > kPullHeavy) {
            // super-heavy remainder: CTA units over [j, e); v stays a candidate
            // for the next level unless a unit finds it
            const uint32_t nu = (e - j + kUnit - 1) / kUnit;
            const uint32_t s = atomicAdd(c.units_tail, nu);
            for (uint32_t k = 0; k < nu; ++k) c.units[s + k] = make_uint2(v, j + k * kUnit);
            pend = false;
            keep = true;
        }
        // phase B: the warp walks the concatenation of the pending
        // remainders 128 entries per step, skipping owners already found
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
        {
            // one atomicOr per distinct word of the warp's found vertices (list
            // order keeps neighbours in the same words); listed once and
            // unvisited: every found vertex is new
            const unsigned peers = __match_any_sync(kFull, found ? (v >> 5) : 0xffffffffu);
            const uint32_t bits = __reduce_or_sync(peers, found ? 1u << (v & 31) : 0u);
            if (found) {
                if (lane == (unsigned)(__ffs(peers) - 1)) {
                    atomicOr(c.visited + (v >> 5), bits);
                    atomicOr(fbm_next + (v >> 5), bits);
                }
                c.depth[v] = c.lvl1;
            }
        }
        em.add(__ballot_sync(kFull, found));
        keep = keep || (scan && !found);
        const uint32_t pos = cta_reserve(L.c_tail, keep ? 1u : 0u, warp_tot, s_base);
        if (keep) L.c_out[pos] = v;
        em.tile();
    }
}

}  // namespace abfs
