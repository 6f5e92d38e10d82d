/* gk_bdl.h — C ABI of the B200-native BDL-tree hot path (kNN_L + BuildvEB_S).
 *
 * This is the drop-in boundary.  The reference (arxiv 2207.01834 "ParGeo",
 * /root/reference) declares no batch interface in code; the
 * entry points below reconstruct the one SPEC.md's `bdltree` module specifies
 * and the shipped headers' conventions imply:
 *
 *   gk_bdl_create   <- BDLTree type, X = 1024, leaf 16
 *   gk_bdl_insert   <- bdl_build / bdl_insert (Insert_L)     SPEC.md:563-580, PAPER.md:1178-1195 (Alg. 3)
 *   gk_bdl_erase    <- bdl_erase (Erase_L)                   SPEC.md:581-589, PAPER.md:1203-1216 (Alg. 4)
 *   gk_bdl_knn      <- bdl_knn (kNN_L) over knn_batch/kNN_S
 *                      rows = KnnBuffer::extract() order     geokit/kdtree/knn_buffer.hpp:42-46 (sorted by (d2, id))
 *   gk_bdl_range    <- kd-tree range search (ball / box)     PAPER.md:188-190, 204, 230 (
 *                      SPEC.md:628 leaves it out of geokit's scope)
 *   gk_bdl_knn_graph <- k-NN graph generator over kNN
 *   point layout    <- Point<D>/PointSet<D>: D doubles, AoS  geokit/core/point.hpp:11-16
 *   ids             <- PointId = uint32, kNoPoint = ~0u       geokit/core/point.hpp:18-19
 *   dim range 2..8  <- dispatch_dim (invalid_argument else)  geokit/core/point.hpp:22-35
 *   errors          <- std::invalid_argument / logic_error   point.hpp:33, seb/orthant.hpp:143
 *                      mapped to GK_ERR_INVALID / GK_ERR_LOGIC + gk_last_error()
 *
 * Conventions: pointers are plain host pointers unless the function name ends
 * in _device (then they are device pointers on the handle's GPU).  Points are
 * row-major n x d fp64 (byte-identical to std::vector<Eigen::Matrix<double,D,1>>).
 * A point's id is its global insertion ordinal (0,1,2,... over all inserts);
 * points reinserted by Erase_L keep their ids.  kNN output is row-major nq x k,
 * each row sorted by (squared distance, id), padded with (GK_NO_POINT, +inf)
 * when fewer than k points are live.  All calls are synchronous with respect
 * to the host; one handle must be used by one host thread at a time; kNN may
 * not run concurrently with insert/erase.
 */
#ifndef GK_BDL_H
#define GK_BDL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_NO_POINT 0xffffffffu /* geokit::core::kNoPoint */

enum gk_status {
  GK_OK = 0,
  GK_ERR_INVALID = 1,     /* std::invalid_argument in the reference */
  GK_ERR_CUDA = 2,        /* CUDA runtime failure (message in gk_last_error) */
  GK_ERR_UNSUPPORTED = 3, /* e.g. k > GK_MAX_K */
  GK_ERR_LOGIC = 4,       /* std::logic_error: id space exhausted, bad handle state */
  GK_ERR_CAPACITY = 5     /* range search: more rows than `capacity`; offsets were written, call again */
};

enum gk_heuristic { GK_SPATIAL_MEDIAN = 0, GK_OBJECT_MEDIAN = 1 };

#define GK_MAX_K 65536 /* k <= 256: k-buffers in shared memory; above: a global scratch heap */
#define GK_MAX_LEAF 32

typedef struct gk_bdl gk_bdl; /* opaque handle: owns all device arenas + one CUDA stream */

/* Canonical static-tree node record, exported for parity
 * checks; identical to the oracle's gko::Node.  168 bytes. */
typedef struct gk_canon_node {
  int32_t kind;  /* 0 internal, 1 leaf */
  int32_t dim;   /* split dimension, -1 for a leaf */
  int32_t mode;  /* 0 spatial median, 1 object median */
  int32_t depth;
  double split;  /* split value (internal) */
  int32_t left, right;   /* child slots in vEB order, -1 for a leaf */
  uint32_t start, count; /* the node's point range in the tree's leaf order */
  double lo[8], hi[8];   /* bounding box (first `dim` entries used) */
} gk_canon_node;

typedef struct gk_bdl_info {
  uint64_t F;            /* fullness bitmask (bit i <=> static tree i exists) */
  uint64_t buffer;       /* points in the buffer tree */
  uint64_t live;         /* total live points */
  uint64_t next_id;      /* next insertion ordinal */
  uint64_t build_size[64];
  uint64_t live_per_tree[64];
  uint64_t nodes_per_tree[64];
  int32_t height_per_tree[64];
  int32_t root_per_tree[64]; /* root slot after Erase_S collapses (-1: emptied) */
} gk_bdl_info;

typedef struct gk_knn_counters {
  uint64_t node_bytes;   /* sum over queries of traversal-node bytes the query itself needed */
  uint64_t leaf_bytes;   /* sum over queries of leaf point bytes (8D + 4 per point) it needed */
  uint64_t nodes;        /* node visits needed (all queries) */
  uint64_t leaves;       /* leaf visits needed */
  uint64_t dists;        /* distance evaluations needed */
  uint64_t warp_nodes;   /* node loads actually issued (one per warp tile) */
  uint64_t warp_leaves;  /* leaf loads actually issued (one per warp tile) */
  uint64_t inserts;      /* points accepted into a k-buffer (all queries) */
  uint64_t warp_leaf_points; /* points of the leaves actually loaded (summed over warp leaf loads) */
  uint64_t warp_inserts;     /* warp-level k-buffer update events (a warp executing an insert) */
} gk_knn_counters;

const char* gk_last_error(void);
const char* gk_version(void);

int gk_bdl_create(int dim, uint32_t buffer_size_X, uint32_t leaf_size, int heuristic, int device, gk_bdl** out);
int gk_bdl_destroy(gk_bdl* h);

/* Insert_L of n points (host / device row-major n x dim). */
int gk_bdl_insert(gk_bdl* h, const double* pts, uint64_t n);
int gk_bdl_insert_device(gk_bdl* h, const double* pts_dev, uint64_t n);

/* Erase_L: tombstone every live point coordinate-equal to some batch point. */
int gk_bdl_erase(gk_bdl* h, const double* pts, uint64_t n, uint64_t* n_erased);
int gk_bdl_erase_device(gk_bdl* h, const double* pts_dev, uint64_t n, uint64_t* n_erased);

/* kNN_L: exact k nearest live points of every query, 1 <= k <= GK_MAX_K. */
int gk_bdl_knn(gk_bdl* h, const double* q, uint64_t nq, int k, uint32_t* ids, double* d2);
int gk_bdl_knn_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, uint32_t* ids_dev, double* d2_dev);
/* Radius-bounded kNN_L: the k nearest live points with d2 <= r2_dev[i] (r2 >= 0, +inf allowed) of
 * every query, rows as gk_bdl_knn; slots beyond the points within the radius are (GK_NO_POINT, +inf).
 * With r2 = +inf this is gk_bdl_knn. */
int gk_bdl_knn_bounded_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, const double* r2_dev,
                              uint32_t* ids_dev, double* d2_dev);
/* Instrumented kNN_L (same results) that also counts the work of §8(d). */
int gk_bdl_knn_counted_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, uint32_t* ids_dev, double* d2_dev,
                              gk_knn_counters* counters);

/* Range search (ball; the kd-tree range search of ParGeo): for every
 * query, every live point p with canonical squared distance d2(q, p) <= r2 (r2 >= 0, +inf allowed).
 * gk_bdl_range_count: counts[i] = number of rows of query i.
 * gk_bdl_range: offsets[nq + 1] = exclusive prefix sums of the counts (offsets[nq] = total), rows of
 * query i at [offsets[i], offsets[i+1]) of ids / d2, sorted by (d2, id).  ids and d2 hold `capacity`
 * rows; a larger result fails with GK_ERR_CAPACITY after writing offsets (call again with room);
 * any other failure (GK_ERR_INVALID for a NaN / negative r2, ...) leaves offsets unwritten.
 * The _device variant takes device pointers and reports the total in *total. */
int gk_bdl_range_count(gk_bdl* h, const double* q, uint64_t nq, double r2, uint64_t* counts);
int gk_bdl_range(gk_bdl* h, const double* q, uint64_t nq, double r2, uint64_t* offsets, uint32_t* ids, double* d2,
                 uint64_t capacity);
int gk_bdl_range_device(gk_bdl* h, const double* q_dev, uint64_t nq, double r2, uint64_t* offsets_dev, uint32_t* ids_dev,
                        double* d2_dev, uint64_t capacity, uint64_t* total);
/* Ball range search with one squared radius per query (r2[i] >= 0, +inf allowed; ParGeo calls its
 * range search per query point with that point's radius); results as above. */
int gk_bdl_range_radii_count(gk_bdl* h, const double* q, uint64_t nq, const double* r2, uint64_t* counts);
int gk_bdl_range_radii(gk_bdl* h, const double* q, uint64_t nq, const double* r2, uint64_t* offsets, uint32_t* ids,
                       double* d2, uint64_t capacity);
int gk_bdl_range_radii_device(gk_bdl* h, const double* q_dev, uint64_t nq, const double* r2_dev, uint64_t* offsets_dev,
                              uint32_t* ids_dev, double* d2_dev, uint64_t capacity, uint64_t* total);

/* Orthogonal (box) range search: for every query box [lo_i, hi_i] (row-major nq x dim each), the
 * ids of the live points p with lo_i[j] <= p[j] <= hi_i[j] for all j, ascending; offsets / capacity
 * as for gk_bdl_range (an empty box, lo > hi in some j, has no rows). */
int gk_bdl_range_box_count(gk_bdl* h, const double* lo, const double* hi, uint64_t nq, uint64_t* counts);
int gk_bdl_range_box(gk_bdl* h, const double* lo, const double* hi, uint64_t nq, uint64_t* offsets, uint32_t* ids,
                     uint64_t capacity);
int gk_bdl_range_box_device(gk_bdl* h, const double* lo_dev, const double* hi_dev, uint64_t nq, uint64_t* offsets_dev,
                            uint32_t* ids_dev, uint64_t capacity, uint64_t* total);

/* k-NN graph (ParGeo's generator over kd-tree kNN): one row per live point in
 * ascending id order (row_ids[r] = its id; gk_bdl_info.live rows), holding its k nearest live
 * points other than itself, sorted by (d2, id), padded with (GK_NO_POINT, +inf).  1 <= k < GK_MAX_K. */
int gk_bdl_knn_graph(gk_bdl* h, int k, uint32_t* row_ids, uint32_t* ids, double* d2);
int gk_bdl_knn_graph_device(gk_bdl* h, int k, uint32_t* row_ids_dev, uint32_t* ids_dev, double* d2_dev);

int gk_bdl_info_get(gk_bdl* h, gk_bdl_info* info);
/* Export static tree `tree` (0..63) or the buffer tree (-1): canonical nodes in
 * vEB slot order, ids and AoS points in leaf order.  Pass NULL to query sizes. */
int gk_bdl_tree_export(gk_bdl* h, int tree, gk_canon_node* nodes, uint32_t* ids, double* pts,
                       uint64_t* n_nodes, uint64_t* n_pts);
/* Bloom prefilter of static tree `tree` (built lazily, 10 bits/key, 7 probes;
 * PAPER.md:1468-1475): may_contain[i] = 0 means point i is
 * definitely not in the tree.  Erase_L uses the same filters internally. */
int gk_bdl_bloom_query(gk_bdl* h, int tree, const double* pts, uint64_t n, uint8_t* may_contain);
/* Stream the handle runs on (cudaStream_t), e.g. to time with events. */
void* gk_bdl_stream(gk_bdl* h);
int gk_bdl_sync(gk_bdl* h);
/* Device time (ms) of the last kNN_L traversal kernel (K1) and of the whole
 * kNN_L device pipeline, recorded with CUDA events on the handle's stream. */
int gk_bdl_last_knn_ms(gk_bdl* h, float* traversal_ms, float* total_ms);
/* Device time (ms) of the last insert's BuildvEB_S work and #points built. */
int gk_bdl_last_build_ms(gk_bdl* h, float* build_ms, uint64_t* points_built);

/* Diagnostics: L2 read bandwidth (GB/s) of `device`, streaming 16-byte L2-only loads over an
 * L2-resident buffer of `bytes` (the ceiling bench.py reports warp-requested bytes against). */
int gk_diag_l2_read_gbs(int device, uint64_t bytes, double* gbs);

/* Seeded input generators (host, OpenMP), restating geokit/generators.hpp:56-63
 * with side 1 and the BASELINE.json config recipes. */
int gk_gen_uniform(uint64_t n, int d, uint64_t seed, double* out);
int gk_gen_mixture(uint64_t n, int d, uint64_t seed, int centres, double sigma, double* out);
int gk_gen_walk(uint64_t clusters, uint64_t steps, uint64_t seed, double* out);
int gk_sample_without_replacement(uint64_t n, uint64_t m, uint64_t seed, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* GK_BDL_H */
