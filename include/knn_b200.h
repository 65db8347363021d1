/*
 * knn_b200.h -- C ABI of the B200-native brute-force kNN engine.
 *
 * This is the drop-in boundary for the reference's single hot-path entry point
 *
 *   knn::NeighborTable knn::bf_knn(const PointSet& queries,
 *                                  const PointSet& references, std::size_t k,
 *                                  const Metric& metric,
 *                                  const BfConfig& config = {},
 *                                  SearchStats* stats = nullptr);
 *   (/root/reference/proj/include/knn/bruteforce.hpp:31-33,
 *    implementation src/bruteforce.cpp:42-100)
 *
 * The reference has no FFI; its "operator API" is that C++ function.  The
 * C++ mirror in include/knn_b200/bruteforce.hpp (knn_b200::bf_knn, same
 * signature and exception text) and the reference-side drop-in shown in
 * INTEGRATION.md both call the entry points below.  Plain pointers and sizes
 * only; no exceptions cross this boundary (status codes + a thread-local
 * message instead).
 *
 * Layouts (match bruteforce.cpp / neighbor_table.hpp):
 *   queries     n x d float32, row-major, contiguous
 *   references  m x d float32, row-major, contiguous
 *   out_dist    n x k float32, row-major by query, ascending distance
 *   out_idx     n x k int64,   same order; ties broken by ascending
 *               reference index (topk.cpp:11-13)
 * Distances are finalized like bf_knn reports them: sqrt of the squared key
 * for euclidean / mahalanobis (bruteforce.cpp:67-69,89-93), the raw key for
 * manhattan / chebyshev.  Keys are exact FP32 (sequential-order fmaf SSD), so
 * results agree with the double reference to ~1e-7 relative.
 */
#ifndef KNN_B200_H
#define KNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNN_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define KNN_B200_API __attribute__((visibility("default")))
#else
#define KNN_B200_API
#endif

typedef enum knn_b200_status {
    KNN_B200_OK = 0,
    /* The conditions under which bf_knn throws std::invalid_argument
     * (bruteforce.cpp:44-56, metric.hpp:90-96, point_set.hpp:18-31). */
    KNN_B200_EINVAL = 1,
    KNN_B200_ENOMEM = 2,    /* device or pinned-host allocation failed */
    KNN_B200_ECUDA = 3,     /* CUDA runtime / driver error */
    KNN_B200_ENCCL = 4,     /* collective failure (sharded search) */
    KNN_B200_EINTERNAL = 5  /* engine invariant violated (a bug) */
} knn_b200_status;

typedef enum knn_b200_metric {
    KNN_B200_EUCLIDEAN = 0,   /* metric.hpp:22-29 */
    KNN_B200_MANHATTAN = 1,   /* metric.hpp:31-35 */
    KNN_B200_CHEBYSHEV = 2,   /* metric.hpp:37-44 */
    KNN_B200_MAHALANOBIS = 3  /* metric.hpp:52-106, metric.cpp:20-82 */
} knn_b200_metric;

/* Which device path computes the keys.  Results are identical for every
 * choice (the tensor path re-ranks its candidates with the exact kernel's
 * arithmetic); the choice only affects speed. */
typedef enum knn_b200_path {
    KNN_B200_PATH_AUTO = 0,    /* tensor path where it applies, else exact */
    KNN_B200_PATH_EXACT = 1,   /* FP32 SIMT kernel with fused top-k */
    KNN_B200_PATH_TENSOR = 2   /* tcgen05 fp16 candidates + exact re-rank (L2 only) */
} knn_b200_path;

typedef struct knn_b200_options {
    uint32_t struct_size;          /* = sizeof(knn_b200_options) */
    int32_t device;                /* CUDA ordinal; -1 = current device */
    int32_t path;                  /* knn_b200_path */
    int32_t count_distance_evals;  /* BfConfig::count_distance_evals (bruteforce.hpp:19) */
    uint64_t chunk_size;           /* BfConfig::chunk_size; must be >= 1, never changes results */
    uint32_t worker_count;         /* BfConfig::worker_count; accepted, ignored */
    int32_t raw_keys;              /* 1: out_dist holds the un-finalized keys (for shard merges) */
    const double *mahalanobis;     /* d x d row-major inverse covariance (metric 3) */
    int64_t mahalanobis_dim;       /* its dimension (Metric::pinned_dim, metric.hpp:64) */
    void *stream;                  /* cudaStream_t for *_device calls; NULL = engine stream */
} knn_b200_options;

/* Fills defaults (device -1, AUTO, chunk_size 1024 as BfConfig does). */
KNN_B200_API void knn_b200_options_init(knn_b200_options *opt);

/* Message of the last failing call on this thread ("" if none). */
KNN_B200_API const char *knn_b200_last_error(void);
KNN_B200_API const char *knn_b200_version(void);

/* One-shot search on HOST buffers: the bf_knn drop-in.  Validation order and
 * messages follow bruteforce.cpp:44-56.  dq/dr are the two point sets'
 * dimensions (a mismatch is EINVAL, bruteforce.cpp:44-48).  distance_evals
 * (nullable) receives n*m when opt->count_distance_evals, else 0
 * (bruteforce.cpp:76,94,98). */
KNN_B200_API knn_b200_status knn_b200_search(const float *queries, int64_t n, int32_t dq,
                                const float *references, int64_t m, int32_t dr,
                                int32_t k, int32_t metric, const knn_b200_options *opt,
                                float *out_dist, int64_t *out_idx,
                                uint64_t *distance_evals);

/* Same search on DEVICE buffers (inputs already resident in HBM).  Runs on
 * opt->stream (or the engine stream) and returns without synchronizing when
 * a stream is given.  Mahalanobis (opt->mahalanobis, d <= 8192): the inputs
 * are whitened on the device into engine scratch copies (the caller's buffers
 * are not modified), bitwise as the host path does. */
KNN_B200_API knn_b200_status knn_b200_search_device(const float *d_queries, int64_t n,
                                       const float *d_references, int64_t m, int32_t d,
                                       int32_t k, int32_t metric,
                                       const knn_b200_options *opt,
                                       float *d_out_dist, int64_t *d_out_idx);

/* ---- device-resident reference set (mirrors the
 *      KdTree build/search split, kdtree.hpp:21,70-72) --------------------- */
typedef struct knn_b200_index knn_b200_index;

/* Upload (host pointer) or adopt (device pointer, not copied, must outlive
 * the index) an m x d reference set.  index_base is added to every returned
 * index: the global offset of this shard in a reference-sharded search. */
KNN_B200_API knn_b200_status knn_b200_index_create(const float *references, int64_t m, int32_t d,
                                      int64_t index_base, const knn_b200_options *opt,
                                      knn_b200_index **out);
KNN_B200_API knn_b200_status knn_b200_index_create_device(const float *d_references, int64_t m,
                                             int32_t d, int64_t index_base,
                                             const knn_b200_options *opt,
                                             knn_b200_index **out);
/* Host queries in, host results out (H2D + D2H inside). */
KNN_B200_API knn_b200_status knn_b200_index_search(knn_b200_index *index, const float *queries,
                                      int64_t n, int32_t k, int32_t metric,
                                      const knn_b200_options *opt, float *out_dist,
                                      int64_t *out_idx);
/* Device queries in, device results out. */
KNN_B200_API knn_b200_status knn_b200_index_search_device(knn_b200_index *index,
                                             const float *d_queries, int64_t n, int32_t k,
                                             int32_t metric, const knn_b200_options *opt,
                                             float *d_out_dist, int64_t *d_out_idx);
KNN_B200_API void knn_b200_index_destroy(knn_b200_index *index);

/* ---- shard merge ---------------------------------------
 * parts x n x k RAW keys + global indices (each part sorted ascending, as
 * produced with opt.raw_keys = 1), merged into the n x k best under the
 * (key, index) order and finalized for `metric`.  Device pointers. */
KNN_B200_API knn_b200_status knn_b200_merge_device(const float *d_part_keys, const int64_t *d_part_idx,
                                      int32_t parts, int64_t n, int32_t k, int32_t metric,
                                      void *stream, float *d_out_dist, int64_t *d_out_idx);

/* ---- multi-GPU (north star (4)) --------------------------
 * The reference scans all m references per query in one process
 * (bruteforce.cpp:24-29,81-96); here the m axis (or the query axis) is split
 * over GPUs.  Reference-sharded: device g holds the contiguous rows
 * [g m / G, (g+1) m / G) and all queries, the per-device n x k lists are
 * all-gathered over NCCL and merged on the device -- bitwise one search over
 * all of R.  Query-sharded: every device holds R and searches its rows of Q;
 * no collective.  NCCL (libnccl.so.2) is loaded at first use; its failures
 * are KNN_B200_ENCCL. */
typedef enum knn_b200_shard_mode {
    KNN_B200_SHARD_REFERENCES = 0,
    KNN_B200_SHARD_QUERIES = 1
} knn_b200_shard_mode;

/* One process driving G devices (devices NULL = 0..G-1): host R is uploaded
 * shard by shard (each shard prepared once, like knn_b200_index_create). */
typedef struct knn_b200_sharded knn_b200_sharded;
KNN_B200_API knn_b200_status knn_b200_sharded_create(const float *references, int64_t m,
                                                     int32_t d, int32_t num_devices,
                                                     const int32_t *devices, int32_t shard_mode,
                                                     const knn_b200_options *opt,
                                                     knn_b200_sharded **out);
/* Host queries in, host n x k table out (bf_knn layout). */
KNN_B200_API knn_b200_status knn_b200_sharded_search(knn_b200_sharded *h, const float *queries,
                                                     int64_t n, int32_t k, int32_t metric,
                                                     const knn_b200_options *opt,
                                                     float *out_dist, int64_t *out_idx);
KNN_B200_API void knn_b200_sharded_destroy(knn_b200_sharded *h);

/* One process per GPU (e.g. torchrun): rank 0 creates the NCCL unique id
 * (len >= 128 bytes), the caller broadcasts it, every rank creates its
 * communicator, builds an index over its own shard (index_base = its first
 * global row) and calls knn_b200_dist_search_device with the same queries:
 * local search, NCCL all-gather of the raw-key lists, device merge -- every
 * rank receives the final n x k table in its device buffers. */
typedef struct knn_b200_comm knn_b200_comm;
KNN_B200_API knn_b200_status knn_b200_nccl_unique_id(void *out, size_t len);
KNN_B200_API int knn_b200_nccl_version(void);
KNN_B200_API knn_b200_status knn_b200_comm_create(const void *unique_id, size_t len,
                                                  int32_t nranks, int32_t rank, int32_t device,
                                                  knn_b200_comm **out);
KNN_B200_API void knn_b200_comm_destroy(knn_b200_comm *comm);
KNN_B200_API knn_b200_status knn_b200_dist_search_device(knn_b200_comm *comm,
                                                         knn_b200_index *local_shard,
                                                         const float *d_queries, int64_t n,
                                                         int32_t k, int32_t metric,
                                                         const knn_b200_options *opt,
                                                         float *d_out_dist, int64_t *d_out_idx);

/* ---- the hot path's next consumers, on the device
 * One engine search + an epilogue kernel over the table in HBM. */

/* entropy.cpp:75-89 rho_k_all: for every point, the Euclidean distance to its
 * k-th nearest OTHER point (self excluded by index; coincident points count
 * at distance 0).  Error text as the reference ("rho_k_all: k = K needs at
 * least k + 1 points, set has N"). */
KNN_B200_API knn_b200_status knn_b200_rho_k_all(const float *points, int64_t n, int32_t d,
                                                int32_t k, const knn_b200_options *opt,
                                                double *out_rho);
KNN_B200_API knn_b200_status knn_b200_rho_k_all_device(const float *d_points, int64_t n,
                                                       int32_t d, int32_t k,
                                                       const knn_b200_options *opt,
                                                       double *d_out_rho);
/* applications.cpp:36-63 knn_classify: majority label of the k nearest training
 * points; vote ties by the smaller summed distance, then the smaller label. */
KNN_B200_API knn_b200_status knn_b200_knn_classify(const float *train, int64_t m, int32_t d,
                                                   const int64_t *labels, const float *queries,
                                                   int64_t n, int32_t dq, int32_t k,
                                                   int32_t metric, const knn_b200_options *opt,
                                                   int64_t *out_labels);
/* applications.cpp:65-86 retrieve_vote: every query descriptor's k nearest
 * database descriptors vote for their owning image; scores[image_count] and
 * the ranking (descending score, ties by ascending id).  DescriptorDatabase
 * validation and messages as applications.cpp:9-34. */
KNN_B200_API knn_b200_status knn_b200_retrieve_vote(const float *descriptors, int64_t m,
                                                    int32_t d, const int64_t *image_of,
                                                    int64_t image_count, const float *queries,
                                                    int64_t n, int32_t dq, int32_t k,
                                                    int32_t metric, const knn_b200_options *opt,
                                                    uint64_t *out_scores, int64_t *out_ranking);

/* Number of CUDA kernels this library launched on the calling thread since
 * the last reset (for bench.py's gpu_launches accounting). */
KNN_B200_API uint64_t knn_b200_launch_count(void);
KNN_B200_API void knn_b200_reset_launch_count(void);

/* ---- measurement support (bench.py) -------------------------------------
 * Per-kernel CUDA-event timing on the launch stream, per calling thread.
 * collect() synchronizes, writes newline-separated kernel names, total ms and
 * launch counts per kernel, resets, and returns the number of kernels. */
KNN_B200_API void knn_b200_profile_enable(int on);
/* Restrict the events to launches whose name starts with `prefix` (NULL or ""
 * = every launch): fewer events, less perturbation of the timed region. */
KNN_B200_API void knn_b200_profile_only(const char *prefix);
KNN_B200_API int knn_b200_profile_collect(char *names, size_t names_len, double *ms,
                                          uint64_t *counts, int max_kernels);

/* Tensor path diagnostics: how many queries of the last search on `device`
 * (-1 = current) failed the candidate certificate and were recomputed by the
 * exact kernel (results are identical either way). */
KNN_B200_API int knn_b200_last_fallback_count(int device);

/* Test hook: D[128x128] fp32 = A[128xK] * B[128xK]^T for fp16 device
 * matrices through the engine's TMA / tcgen05 / TMEM primitives. */
KNN_B200_API knn_b200_status knn_b200_debug_mma_probe(const void *d_a, const void *d_b, int32_t K,
                                                      float *d_out);

/* Synthetic uniform [0,1) FP32 on the device: element i of the stream is
 * splitmix64(seed + offset + i) >> 40 scaled by 2^-24 (host-reproducible). */
KNN_B200_API knn_b200_status knn_b200_fill_uniform_device(float *d_out, int64_t count,
                                                          uint64_t seed, int64_t offset,
                                                          void *stream);

#ifdef __cplusplus
}
#endif

#endif /* KNN_B200_H */
