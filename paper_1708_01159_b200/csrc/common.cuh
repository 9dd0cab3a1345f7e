// common.cuh -- shared definitions of the libabfs engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/abfs.h"

namespace abfs {

constexpr int32_t kInf = 0x7fffffff;
constexpr unsigned kFull = 0xffffffffu;

// Thread-local error message (abfs_last_error).
void set_error(const std::string &msg);

#define ABFS_CUDA(call)                                                        \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) {                                               \
            ::abfs::set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
            return _e == cudaErrorMemoryAllocation ? ABFS_ENOMEM : ABFS_ECUDA; \
        }                                                                      \
    } while (0)

#define ABFS_TRY(call)                                                         \
    do {                                                                       \
        int _rc = (call);                                                      \
        if (_rc != ABFS_OK) return _rc;                                        \
    } while (0)

inline int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

// Device-resident combined representation (graph.py:27-69).  Edge indices
// fit u32 offsets (m < 2^32), vertex ids are u32.
struct DevGraph {
    uint64_t n = 0, m = 0;
    uint32_t *out_off = nullptr;   // [n+1]
    uint32_t *dst = nullptr;       // [m] destinations, sorted by (origin, dest)
    uint32_t *org = nullptr;       // [m] origins
    uint32_t *in_off = nullptr;    // [n+1]
    uint32_t *src = nullptr;       // [m] sources, sorted by (dest, origin)
    uint32_t *rev_owner = nullptr; // [m] owning destination of reverse slot
    uint32_t *first_src = nullptr; // [n] src[in_off[v]]: pull's first probe as a dense,
                                   //     coalesced read (derived, like rev_owner)
};

}  // namespace abfs

struct abfs_graph {
    int device = 0;
    abfs::DevGraph d;
};

namespace abfs {
int graph_alloc(abfs_graph *g, uint64_t n, uint64_t m);
void graph_free(abfs_graph *g);

// One rank's slice of a 1-D partition (partition.cu): the destination-
// filtered out-CSR over all n sources and the in-CSR rows of the owned range
// [lo, hi).  gen_slice (graph.cu) builds it from a generator stream; the
// caller owns the arrays.
struct Slice {
    uint64_t mf = 0, mr = 0;
    uint32_t *fo_off = nullptr, *fo_dst = nullptr, *fo_org = nullptr;
    uint32_t *r_off = nullptr, *r_src = nullptr, *r_own = nullptr, *r_first = nullptr;
};
int gen_slice(int device, const abfs_gen_spec *spec, uint64_t lo, uint64_t hi, Slice &out,
              uint64_t *n_out, cudaStream_t s);
}  // namespace abfs
