/*
 * abfs.h -- C ABI of the B200-native tree-switched level-synchronous BFS
 * engine (libabfs.so, built from paper_1708_01159_b200/csrc/).
 *
 * The reference (/root/reference/pkg/src/adaptive_bfs/, pure Python + numpy)
 * has no FFI: its operator API is the Python callables listed beside each
 * entry point below ("replaces ...").  The Python package
 * paper_1708_01159_b200 binds this header with ctypes and re-exposes the
 * reference names and signatures; INTEGRATION.md shows the binding a
 * reference maintainer would add.
 *
 * Conventions
 *   - every call returns an abfs_status; abfs_last_error() gives the
 *     thread-local message of the last failure (mapped to ValueError with the
 *     reference's text by the Python layer);
 *   - plain pointers + sizes only; "host" pointers are ordinary CPU memory,
 *     the engine owns all device memory;
 *   - one CUDA stream per traversal (settable), calls on one traversal are not
 *     reentrant (same rule as bfs_full on one depth array);
 *   - depths are int32 with INF = 2^31-1 (kernels.py:30-31).
 */
#ifndef ABFS_H
#define ABFS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ABFS_API __attribute__((visibility("default")))
#else
#define ABFS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ABFS_OK = 0,
    ABFS_EINVAL = 1,    /* invalid argument (root/chunk/kernel/variant/...)   */
    ABFS_ECUDA = 2,     /* CUDA runtime error                                 */
    ABFS_ENCCL = 3,     /* reserved: multi-GPU exchange error                 */
    ABFS_ENOMEM = 4,    /* device or host allocation failed                   */
    ABFS_EFEATURE = 5   /* invalid runtime feature state (features.py:103-110)*/
} abfs_status;

#define ABFS_INF_DEPTH 2147483647
#define ABFS_LEAF_UNKNOWN 254   /* tree.py:25 */
#define ABFS_NOT_A_LEAF 255     /* tree.py:26 */
#define ABFS_N_FEATURES 24      /* features.py:25-35 canonical order */

/* KernelId (kernels.py:40-47) and CountVariant (kernels.py:50-55). */
enum { ABFS_EDGE_LIST = 0, ABFS_REV_EDGE_LIST = 1, ABFS_VERTEX_PUSH = 2,
       ABFS_VERTEX_PULL = 3, ABFS_VERTEX_PUSH_WARP = 4 };
enum { ABFS_DIRECT_ATOMIC = 0, ABFS_GROUP_REDUCE = 1, ABFS_TWO_LEVEL_REDUCE = 2 };

typedef struct abfs_graph abfs_graph;          /* device-resident Graph      */
typedef struct abfs_traversal abfs_traversal;  /* device depth/frontier state */

/* FlatTree (tree.py:303-359) in array form.  selection[i] is the canonical
 * FEATURE_NAMES index of the tree's i-th selected feature; features[node]
 * indexes into the selection (tree.py:332-339). */
typedef struct {
    uint32_t node_count;
    uint32_t n_selection;
    const uint16_t *selection;
    const uint16_t *features;
    const double *thresholds;
    const uint32_t *lefts;
    const uint32_t *rights;
    const uint8_t *leaf_classes;
} abfs_tree;

/* One LevelTrace (adaptive.py:51-60) plus engine diagnostics. */
typedef struct {
    int64_t level;
    int32_t kernel;
    int32_t variant;
    int32_t fallback;
    int32_t converted;        /* 1 if a queue<->bitmap conversion ran (switch cost) */
    uint64_t frontier_size;
    uint64_t new_count;
    uint64_t elapsed_ns;      /* CUDA-event time of the level incl. conversion */
    uint64_t prediction_ns;   /* host feature extraction + tree descent        */
    /* SURVEY §8a N2, per-level integer features from the device: */
    uint64_t unvisited;       /* |V| - discovered after this level (exact)           */
    uint64_t next_out_edges;  /* sum of out-degrees of this level's discoveries (the
                                 next frontier's out-edges); measured in instrumented
                                 runs (abfs_traversal_instrument), else UINT64_MAX */
} abfs_level_record;

ABFS_API const char *abfs_last_error(void);
ABFS_API int abfs_version(void);

/* ---- graph (graph.py) --------------------------------------------------- */

/* Upload a host combined representation (replaces Graph, graph.py:27-69;
 * rev_owner (graph.py:57-65) is derived on the device). */
ABFS_API int abfs_graph_upload(int device, uint64_t n, uint64_t m,
                      const uint32_t *out_offsets, const uint32_t *destinations,
                      const uint32_t *origins, const uint32_t *in_offsets,
                      const uint32_t *sources, abfs_graph **out);

/* Device build_combined from host (src, dst) pairs (replaces
 * build_combined, graph.py:93-134; pairs must be range-checked). */
ABFS_API int abfs_graph_build(int device, uint64_t n, uint64_t m, const uint32_t *src,
                     const uint32_t *dst, abfs_graph **out);

/* Device generators, bit-exact to generate_graph (graph.py:211-252):
 * pcg_state/pcg_inc are numpy default_rng(seed)'s PCG64 words (hi, lo).
 * symmetrize bit 0 appends the reversed pairs; bit 1
 * (rmat only, no reference counterpart) relabels ids with the bijection
 * v -> (v * 0x9E3779B1 + 0x7F4A7C15) mod 2^scale, Graph500-style, so hubs are
 * not clustered at low ids (robustness runs, bench.py --permute). */
ABFS_API int abfs_graph_generate_rmat(int device, uint32_t scale, uint64_t edges,
                             double a, double b, double c,
                             const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                             int symmetrize, abfs_graph **out);
/* uniform-random (graph.py:226-231); n must be a power of two <= 2^32. */
ABFS_API int abfs_graph_generate_uniform(int device, uint64_t n, uint64_t edges,
                                const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                                abfs_graph **out);
/* rows x cols 4-neighbour grid, both directions. */
ABFS_API int abfs_graph_generate_mesh(int device, uint32_t rows, uint32_t cols,
                             abfs_graph **out);

ABFS_API int abfs_graph_info(const abfs_graph *g, uint64_t *n, uint64_t *m, int *device);
/* Copy arrays back to host; any pointer may be NULL (skipped). */
ABFS_API int abfs_graph_download(const abfs_graph *g, uint32_t *out_offsets,
                        uint32_t *destinations, uint32_t *origins,
                        uint32_t *in_offsets, uint32_t *sources, uint32_t *rev_owner);
ABFS_API void abfs_graph_destroy(abfs_graph *g);

/* ---- traversal state ---------------------------------------------------- */

ABFS_API int abfs_traversal_create(abfs_graph *g, abfs_traversal **out);
ABFS_API void abfs_traversal_destroy(abfs_traversal *t);
/* Use an external cudaStream_t (NULL = engine-owned stream). */
ABFS_API int abfs_traversal_set_stream(abfs_traversal *t, void *cuda_stream);

/* init_depths on the device (replaces init_depths, kernels.py:134-140). */
ABFS_API int abfs_init_depths(abfs_traversal *t, int64_t root);
/* Arbitrary caller depths (run_level contract, tests/test_kernels.py:209-236);
 * the next level rebuilds its frontier from the depth array. */
ABFS_API int abfs_load_depths(abfs_traversal *t, const int32_t *host_depths);
ABFS_API int abfs_read_depths(abfs_traversal *t, int32_t *host_depths);

/* One level on the device-resident state (replaces run_level,
 * kernels.py:340-353): kernel/variant/chunk as in the reference; one small
 * readback.  new_count = INF->level+1 transitions. */
ABFS_API int abfs_level(abfs_traversal *t, int64_t level, int kernel, int variant,
               int64_t chunk_size, uint64_t *new_count, uint64_t *elapsed_ns);

/* run_level on a caller-owned HOST depth array, mutated in place
 * (H2D, level, D2H). */
ABFS_API int abfs_run_level(abfs_traversal *t, int32_t *host_depths, int64_t level,
                   int kernel, int variant, int64_t chunk_size,
                   uint64_t *new_count, uint64_t *elapsed_ns);

/* bfs_full (kernels.py:356-371).  counts/elapsed receive one entry per
 * executed level (terminating zero level included) up to cap; depths_out may
 * be NULL (depths stay on the device). */
ABFS_API int abfs_bfs_full(abfs_traversal *t, int64_t root, int kernel, int variant,
                  int64_t chunk_size, int32_t *depths_out, uint64_t *counts,
                  uint64_t *elapsed, size_t cap, size_t *n_levels);

/* adaptive_bfs with a FlatTree model (adaptive.py:83-129): per level the
 * device produces the new count, the host evaluates the tree on the
 * reference's float64 features (features.py:98-121; static24 holds the 24
 * canonical features, slots 2..5 ignored), then launches the chosen pair. */
ABFS_API int abfs_adaptive_bfs(abfs_traversal *t, int64_t root, const abfs_tree *tree,
                      const double *static24, int64_t chunk_size,
                      int32_t *depths_out, abfs_level_record *records,
                      size_t cap, size_t *n_levels);

/* Multi-source throughput form of adaptive_bfs (no reference counterpart;
 * each traversal has adaptive.py:83-129 semantics): nroots (<= 4096)
 * tree-switched BFSs run inside persistent launches, each root's
 * init_depths inside the kernel, no host round trip between them: the
 * roots are dealt round-robin to S concurrent launches of 1/S of the
 * co-resident grid (private scratch and stream each, forked from and joined
 * back into the traversal's stream; S = abfs_traversal_batch_ways), each
 * running its roots back to back.  levels[i] / bfs_ns[i] (optional) = level
 * calls and device time (first level start .. last level end) of root i;
 * total_ns = fork to join.  The depth array afterwards holds the last
 * root's traversal. */
ABFS_API int abfs_adaptive_bfs_batch(abfs_traversal *t, const int64_t *roots, size_t nroots,
                                     const abfs_tree *tree, const double *static24,
                                     int64_t chunk_size, uint64_t *levels, uint64_t *bfs_ns,
                                     uint64_t *total_ns);
/* The same batch with per-root parity evidence (tests; not on the timed
 * path): checksums[i] = sum over v of (uint64(uint32(depth_i[v])) + 1) *
 * ((v + 1) * 0x9E3779B97F4A7C15) mod 2^64 of root i's final depth array,
 * computed in the kernel after each traversal; new_counts = every root's
 * per-level new counts concatenated (root order, levels[i] each; the first
 * counts_cap are written, *n_counts = how many the launch recorded). */
ABFS_API int abfs_adaptive_bfs_batch_check(abfs_traversal *t, const int64_t *roots,
                                           size_t nroots, const abfs_tree *tree,
                                           const double *static24, int64_t chunk_size,
                                           uint64_t *levels, uint64_t *checksums,
                                           uint64_t *new_counts, size_t counts_cap,
                                           size_t *n_counts);

/* Total device time (ns) of the last abfs_bfs_full/abfs_adaptive_bfs call,
 * from after init_depths to the final count readback. */
ABFS_API int abfs_last_traversal_ns(const abfs_traversal *t, uint64_t *ns);

/* 1 (default): bfs_full / adaptive_bfs run the whole level loop inside one
 * persistent cooperative kernel (device-side FlatTree, grid barriers between
 * levels; 5 CTAs x 256 threads per SM, 48 registers); 2 = the same with
 * 6 CTAs / 40 registers, 3 = 4 CTAs / 64 registers; 0: one launch chain +
 * one host round trip per level.  On graphs with max out-degree <= 64 the
 * megakernel also runs small levels on one 8-CTA cluster ("solo mode";
 * environment ABFS_SOLO=0/1 forces it off/on). */
ABFS_API int abfs_traversal_set_mode(abfs_traversal *t, int device_loop);

/* Concurrent launches a batch of nroots roots is split into (1 = one
 * launch): abfs_traversal_set_batch_ways, else ABFS_BATCH_SPLIT, else 8 on graphs of max out-degree <= 8, 2 on
 * graphs of more than 2^25 vertices, 4 otherwise; at most nroots. */
ABFS_API int abfs_traversal_batch_ways(const abfs_traversal *t, size_t nroots, int *ways);
/* Fix the split (ways >= 1; 1 = every batch in one full-grid launch, each
 * BFS with the whole GPU: per-BFS t_bfs semantics) or 0 = automatic. */
ABFS_API int abfs_traversal_set_batch_ways(abfs_traversal *t, int ways);

/* Number of kernels this traversal has launched (bench gpu_launches). */
ABFS_API int abfs_traversal_launches(const abfs_traversal *t, uint64_t *launches);

/* Work-model instrumentation (bench roofline, not on the timed path):
 * when on, pull levels count the in-edges they scan (ES). */
ABFS_API int abfs_traversal_instrument(abfs_traversal *t, int on);
/* Per-depth histograms of the current depth array: count, Σ out-degree,
 * Σ in-degree for depths 0..nlev-1 and slot nlev = unreached (each array
 * nlev+1 long); scanned[l] = ES of level l from the last instrumented run. */
ABFS_API int abfs_traversal_level_stats(abfs_traversal *t, size_t nlev, uint64_t *count,
                                        uint64_t *out_deg, uint64_t *in_deg, uint64_t *scanned);

/* Sum over reached vertices of out-degree (GTEPS numerator basis). */
ABFS_API int abfs_reached_edges(abfs_traversal *t, uint64_t *edges, uint64_t *vertices);

/* ---- 1-D vertex partition ---------------------------------- */

/* One rank's share of a vertex-partitioned BFS: the destination range
 * [lo, hi) (lo a multiple of 32; hi a multiple of 32 or |V|) of graph g,
 * i.e. the destination-filtered out-CSR over all sources plus the owned
 * in-CSR rows, owned depths/visited bits and a replicated global frontier
 * bitmap.  There is no reference counterpart (the reference is one process,
 * kernels.py:82-127); the per-level semantics are run_level's
 * (kernels.py:340-353) restricted to owned destinations. */
typedef struct abfs_part abfs_part;
ABFS_API int abfs_part_create(abfs_graph *g, uint64_t lo, uint64_t hi, abfs_part **out);

/* A generator description (the device generators above as data), so a rank
 * can build its slice without the whole graph ever being on its GPU. */
enum { ABFS_GEN_RMAT = 0, ABFS_GEN_UNIFORM = 1, ABFS_GEN_MESH = 2 };
typedef struct abfs_gen_spec {
    int32_t kind;            /* ABFS_GEN_* */
    int32_t symmetrize;      /* rmat: append the reversed pairs */
    uint32_t scale;          /* rmat: |V| = 2^scale */
    uint32_t rows, cols;     /* mesh */
    uint64_t n;              /* uniform: |V| (power of two) */
    uint64_t edges;          /* rmat / uniform: generated pairs */
    double a, b, c;          /* rmat quadrant probabilities */
    uint64_t pcg_state[2], pcg_inc[2];
} abfs_gen_spec;
/* |V| and |E| (directed slots) of the graph the spec generates. */
ABFS_API int abfs_gen_size(const abfs_gen_spec *spec, uint64_t *n, uint64_t *m);
/* Out-/in-degree of every vertex of the generated graph (host arrays of
 * |V| u32; in_deg may be NULL for a symmetrised spec) from one streaming
 * pass of the generator on `device` (O(|V|) device memory, no edge arrays):
 * the inputs of compute_stats (graph.py:180-208) and of the edge-balanced
 * partition bounds. */
ABFS_API int abfs_gen_degrees(int device, const abfs_gen_spec *spec, uint32_t *out_deg,
                              uint32_t *in_deg);
/* abfs_part_create for the graph `spec` generates, built on `device` from
 * the generator stream filtered to destinations in [lo, hi): peak device
 * memory ~ 2 x 8 bytes per owned in-edge plus the slice itself, never the
 * whole graph.  The slice's arrays equal abfs_part_create's on the full
 * graph (tests compare them with abfs_part_download). */
ABFS_API int abfs_part_create_generated(int device, const abfs_gen_spec *spec, uint64_t lo,
                                        uint64_t hi, abfs_part **out);
/* Copy a slice's arrays back (tests): fo_off [|V|+1], fo_dst/fo_org [m_fwd],
 * r_off [hi-lo+1], r_src/r_own [m_rev], r_first [hi-lo]; NULL skips one. */
ABFS_API int abfs_part_download(const abfs_part *p, uint32_t *fo_off, uint32_t *fo_dst,
                                uint32_t *fo_org, uint32_t *r_off, uint32_t *r_src,
                                uint32_t *r_own, uint32_t *r_first);
ABFS_API void abfs_part_destroy(abfs_part *p);
ABFS_API int abfs_part_info(const abfs_part *p, uint64_t *lo, uint64_t *hi, uint64_t *m_fwd,
                            uint64_t *m_rev);
/* The stream the partition enqueues on, used as given: NULL is the legacy
 * default stream (a new partition owns a private stream). */
ABFS_API int abfs_part_set_stream(abfs_part *p, void *cuda_stream);
/* init_depths (kernels.py:134-140) on the owned slice; frontier = {root}. */
ABFS_API int abfs_part_init(abfs_part *p, int64_t root);
/* One level on the local slice; writes this rank's next-frontier bitmap
 * slice into the DEVICE buffer send[0..stride) (zero padded).  Enqueued on
 * the partition's stream, no host sync: the caller all-gathers `send`
 * (rank-major, stride words each) on the same stream, then calls
 * abfs_part_exchange. */
ABFS_API int abfs_part_level(abfs_part *p, int64_t level, int kernel, int variant,
                             int64_t chunk_size, uint32_t *send, uint64_t stride);
/* Unpack the gathered slices (DEVICE, nranks x stride words; word_bounds =
 * host array of nranks+1 global word offsets) into the global frontier;
 * global_count = popc of it (identical on every rank), local_count = this
 * rank's count through the level's count variant, elapsed_ns = device time
 * from the level's start to here (exchange included).  One host sync. */
ABFS_API int abfs_part_exchange(abfs_part *p, const uint32_t *gathered,
                                const uint64_t *word_bounds, uint32_t nranks, uint64_t stride,
                                uint64_t *global_count, uint64_t *local_count,
                                uint64_t *elapsed_ns);
/* Fused exchange (no collective): each rank's level ends with a kernel that
 * stores its next-frontier slice straight into every rank's global bitmap
 * over NVLink peer memory and signals each rank's mailbox with system-scope
 * atomics; abfs_part_p2p_finish waits (bounded, ABFS_ENCCL on timeout) for
 * all ranks' signals and sums their counts.  Peers are given either as
 * device pointers (partitions of one process, abfs_part_peer_buffers) or
 * by CUDA IPC handles (one process per GPU: abfs_part_ipc_export fills 192
 * bytes per rank; abfs_part_ipc_open takes all ranks' handles in rank
 * order). */
ABFS_API int abfs_part_peer_buffers(abfs_part *p, void **fbm0, void **fbm1, void **mailbox);
ABFS_API int abfs_part_set_peers(abfs_part *p, void *const *fbm0, void *const *fbm1,
                                 void *const *mailboxes, uint32_t nranks, uint32_t rank);
ABFS_API int abfs_part_ipc_export(abfs_part *p, unsigned char *handles /* 192 bytes */);
ABFS_API int abfs_part_ipc_open(abfs_part *p, const unsigned char *all_handles, uint32_t nranks,
                                uint32_t rank);
ABFS_API int abfs_part_level_p2p(abfs_part *p, int64_t level, int kernel, int variant,
                                 int64_t chunk_size);
ABFS_API int abfs_part_p2p_finish(abfs_part *p, uint64_t *global_count, uint64_t *local_count,
                                  uint64_t *elapsed_ns);

/* Whole traversals over fused-exchange partitions of this process (peers
 * set), driven in C with no Python per level: adaptive_bfs
 * (adaptive.py:83-129, tree on the reference's float64 features) and
 * bfs_full (kernels.py:356-371).  records[l] as abfs_adaptive_bfs
 * (elapsed_ns = slowest partition's level time incl. the exchange);
 * local_counts (optional, cap x nparts) = each partition's count of each
 * level through its count variant. */
ABFS_API int abfs_parts_adaptive_bfs(abfs_part *const *parts, uint32_t nparts, int64_t root,
                                     const abfs_tree *tree, const double *static24,
                                     int64_t chunk_size, abfs_level_record *records,
                                     uint64_t *local_counts, size_t cap, size_t *n_levels);
ABFS_API int abfs_parts_bfs_full(abfs_part *const *parts, uint32_t nparts, int64_t root,
                                 int kernel, int variant, int64_t chunk_size,
                                 abfs_level_record *records, uint64_t *local_counts, size_t cap,
                                 size_t *n_levels);

/* The same traversals for ONE partition per process (one GPU) inside the
 * persistent megakernel: levels, tree decisions and the fused exchange (peer
 * stores, device-side mailbox wait) all on the device, one launch per
 * traversal.  Every rank calls it with the same root and tree. */
ABFS_API int abfs_part_mega_adaptive_bfs(abfs_part *p, int64_t root, const abfs_tree *tree,
                                         const double *static24, int64_t chunk_size,
                                         abfs_level_record *records, uint64_t *local_counts,
                                         size_t cap, size_t *n_levels);
ABFS_API int abfs_part_mega_bfs_full(abfs_part *p, int64_t root, int kernel, int variant,
                                     int64_t chunk_size, abfs_level_record *records,
                                     uint64_t *local_counts, size_t cap, size_t *n_levels);

/* Owned depths (hi - lo entries) to host / to a device buffer (async). */
ABFS_API int abfs_part_read_depths(abfs_part *p, int32_t *host_owned);
ABFS_API int abfs_part_depths_device(abfs_part *p, int32_t *dev_out);
ABFS_API int abfs_part_launches(const abfs_part *p, uint64_t *launches);

/* ---- reference artefacts on the engine side -------------- */
/* With these a C/C++ host runs a tree-switched BFS from the reference's own
 * files without Python: abfs_graph_read -> abfs_traversal_create ->
 * abfs_tree_read -> abfs_adaptive_bfs -> abfs_trace_write. */

/* read_graph (graph.py:304-324): ADGR file streamed straight into HBM;
 * ABFS_EINVAL with the reference's ValueError texts (bad magic / truncated
 * header / unsupported version / truncated file / trailing bytes). */
ABFS_API int abfs_graph_read(int device, const char *path, abfs_graph **out);
/* write_graph (graph.py:292-301): byte-identical ADGR file. */
ABFS_API int abfs_graph_write(const abfs_graph *g, const char *path);

/* deserialize (tree.py:409-447): an ADBT model; the selection names are
 * resolved to canonical feature indices (validate_selection,
 * features.py:53-63).  abfs_tree_file_view gives the abfs_tree the traversal
 * calls take; valid until abfs_tree_file_free. */
typedef struct abfs_tree_file abfs_tree_file;
ABFS_API int abfs_tree_read(const char *path, abfs_tree_file **out);
ABFS_API const abfs_tree *abfs_tree_file_view(const abfs_tree_file *t);
ABFS_API void abfs_tree_file_free(abfs_tree_file *t);
/* serialize (tree.py:389-406): byte-identical ADBT file (selection written
 * as the canonical names of tree->selection). */
ABFS_API int abfs_tree_write(const abfs_tree *tree, const char *path);

/* write_trace / read_trace (adaptive.py:225-254): the trace CSV, byte-
 * identical to Python's csv writer ("\r\n" line ends).  read: up to cap
 * records into recs (NULL to count), *n = rows in the file; new_count and
 * converted are not CSV columns and read back as 0. */
ABFS_API int abfs_trace_write(const char *path, const abfs_level_record *records, size_t n);
ABFS_API int abfs_trace_read(const char *path, abfs_level_record *records, size_t cap,
                             size_t *n);

/* ---- helpers ------------------------------------------------------------ */

/* Page-lock caller memory so depth read-backs into it are direct DMA (the
 * Python layer's recycled output arrays; no reference counterpart). */
ABFS_API int abfs_host_register(void *ptr, size_t bytes);
ABFS_API int abfs_host_unregister(void *ptr);

/* aggregate_count (kernels.py:143-170) on the device with the three
 * reduction shapes: DIRECT = 1 atomic/item, GROUP = warp reduce + 1
 * atomic/warp, TWO_LEVEL = warp + CTA reduce + 1 atomic/CTA. */
ABFS_API int abfs_aggregate_count(int device, const int64_t *host_counts, size_t n,
                         int variant, int64_t *total);

/* FlatTree.predict_one (tree.py:332-339) on a projected vector. */
ABFS_API int abfs_tree_predict(const abfs_tree *tree, const double *projected, int *leaf_class);

/* extract_runtime_features (features.py:98-121) into out24 (canonical). */
ABFS_API int abfs_features(const double *static24, uint64_t frontier_abs,
                  uint64_t discovered_abs, double *out24);

#ifdef __cplusplus
}
#endif
#endif /* ABFS_H */
