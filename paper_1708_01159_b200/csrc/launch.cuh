// launch.cuh -- host-side launch of one level's strategy kernels over a view
// of the graph (StratArgs).  The single-GPU traversal passes the whole
// combined representation; a vertex partition (partition.cu) passes its
// destination-filtered forward slice and its owned reverse rows, with the
// bitmap / depth pointers rebased so the kernels index by global vertex id.
#pragma once

#include "bfs_kernels.cuh"

namespace abfs {

static inline unsigned grid_for(uint64_t items, uint64_t per_block, uint64_t cap) {
    uint64_t b = (items + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

// One full wave of resident CTAs for a persistent kernel (cached per kernel).
template <typename K>
static uint64_t persist_grid(K kernel) {
    static uint64_t grid = 0;
    if (!grid) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kBlock, 0);
        grid = (uint64_t)sms * (uint64_t)(per > 0 ? per : 1);
    }
    return grid;
}

// run_level argument checks (kernels.py:312-313, :353, :161).
static inline int level_params_ok(int64_t level, int kernel, int variant, int64_t chunk) {
    if (kernel < 0 || kernel > 4) return fail(ABFS_EINVAL, "unknown kernel " + std::to_string(kernel));
    if (variant < 0 || variant > 2)
        return fail(ABFS_EINVAL, "unknown count variant " + std::to_string(variant));
    if (kernel == ABFS_VERTEX_PUSH_WARP && chunk < 1)
        return fail(ABFS_EINVAL, "chunk_size must be >= 1");
    if (level < INT32_MIN || level > (int64_t)kInf - 2)
        return fail(ABFS_EINVAL, "level out of range");
    return ABFS_OK;
}

struct StratArgs {
    // forward slots (sorted by origin): out-CSR + origins, m_fwd slots
    const uint32_t *out_off, *dst, *org;
    uint64_t m_fwd;
    // reverse slots (sorted by owner): in-CSR + owners, m_rev slots
    const uint32_t *in_off, *src, *rev_owner;
    uint64_t m_rev;
    const uint32_t *first_src;   // src[in_off[v]] by global id
    // pull: in-degree-0 bitmap, next-frontier bitmap, word range scanned
    const uint32_t *noin;
    uint32_t *fbm_next;
    uint64_t word0, word_end;
    // top-down: current frontier queue
    const uint32_t *q;
    uint32_t F;
};

// Launches the chosen strategy; returns the number of kernels launched.
template <int VAR>
static int launch_strategy_args(const LevelCtx &c, const StratArgs &a, int kernel, int64_t chunk,
                                cudaStream_t s) {
    switch (kernel) {
    case ABFS_EDGE_LIST:
        k_edge<VAR, false><<<grid_for(a.m_fwd, kEdgeTileMax, persist_grid(k_edge<VAR, false>)), kBlock,
                             0, s>>>(c, a.org, a.dst, a.m_fwd);
        return 1;
    case ABFS_REV_EDGE_LIST:
        k_edge<VAR, true><<<grid_for(a.m_rev, kEdgeTileMax, persist_grid(k_edge<VAR, true>)), kBlock,
                            0, s>>>(c, a.rev_owner, a.src, a.m_rev);
        return 1;
    case ABFS_VERTEX_PUSH:
        k_push<VAR><<<grid_for(a.F, kBlock, 148 * 64), kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst);
        k_heavy<VAR><<<148 * 8, kBlock, 0, s>>>(c, a.out_off, a.dst);
        return 2;
    case ABFS_VERTEX_PULL:
        k_pull<VAR><<<grid_for(a.word_end - a.word0, kBlock, 148 * 64), kBlock, 0, s>>>(
            c, a.in_off, a.src, a.first_src, a.noin, a.fbm_next, a.word0, a.word_end);
        k_pull_heavy<<<148 * 8, kBlock, 0, s>>>(c, a.in_off, a.src, a.fbm_next);
        return 2;
    default: {  // VERTEX_PUSH_WARP: nearest legal virtual-warp width <= chunk
        const int vw = chunk >= 32 ? 32 : chunk >= 16 ? 16 : chunk >= 8 ? 8 : chunk >= 4 ? 4 : chunk >= 2 ? 2 : 1;
        const unsigned grid = grid_for((uint64_t)a.F * vw, kBlock, 148 * 32);
        switch (vw) {
        case 32: k_push_warp<VAR, 5><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        case 16: k_push_warp<VAR, 4><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        case 8: k_push_warp<VAR, 3><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        case 4: k_push_warp<VAR, 2><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        case 2: k_push_warp<VAR, 1><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        default: k_push_warp<VAR, 0><<<grid, kBlock, 0, s>>>(c, a.q, a.F, a.out_off, a.dst); break;
        }
        k_heavy<VAR><<<148 * 8, kBlock, 0, s>>>(c, a.out_off, a.dst);
        return 2;
    }
    }
}

}  // namespace abfs
