// gk_common.cuh — shared device types of the B200 BDL-tree (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gk_bdl.h"

namespace gk {

constexpr int kMaxDim = 8;
constexpr int kDepthCap = 40;     // depth >= 40 -> object-median split (frozen decision)
constexpr int kStack = 72;        // traversal stack bound: max depth <= 40 + 28 (n < 2^32)
constexpr int kChunk = 1024;      // points per warp work item in the build passes
constexpr std::uint64_t kLeafFlag = 1ULL << 63;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GK_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::gk::Error(GK_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) +      \
                                          " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define GK_CHECK_LAUNCH() GK_CUDA(cudaGetLastError())

// Kernel attributes and occupancy-derived grid sizes are cached per (instantiation, device): a
// process may drive handles on several GPUs, and the dynamic-shared-memory opt-in is per device.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  GK_CUDA(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) throw Error(GK_ERR_UNSUPPORTED, "device index >= 64");
  return d;
}

// Traversal node (query-optimised mirror of one internal canonical node):
// both children's boxes, rounded outward to fp32 (conservative, so pruning
// stays exact), interleaved per dimension (lo[j] = {child0, child1}) so one
// packed f32x2 instruction tests both children, and the two child references.  A child reference is either an
// internal-node index (rank among internal nodes in vEB order) or, with bit 63
// set, a leaf: bits [8,56) = first point, bits [0,8) = point count.
template <int D>
struct alignas(16) TNode {
  float lo[D][2];
  float hi[D][2];
  std::uint64_t ref[2];
};

__host__ __device__ inline bool is_leaf_ref(std::uint64_t r) { return (r & kLeafFlag) != 0; }
__host__ __device__ inline std::uint32_t leaf_count(std::uint64_t r) { return static_cast<std::uint32_t>(r & 0xffu); }
__host__ __device__ inline std::uint64_t leaf_start(std::uint64_t r) { return (r >> 8) & ((1ULL << 48) - 1); }
__host__ __device__ inline std::uint64_t make_leaf_ref(std::uint64_t start, std::uint32_t count) {
  return kLeafFlag | (start << 8) | count;
}

// order-preserving fp64 <-> uint64 map (for atomicMin/Max on doubles)
__device__ __forceinline__ std::uint64_t dkey(double x) {
  std::uint64_t b = static_cast<std::uint64_t>(__double_as_longlong(x));
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(std::uint64_t k) {
  std::uint64_t b = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// One static tree on the device.
struct DevTree {
  int d = 0;
  std::uint64_t n = 0;            // points (stride of the SoA arrays)
  double* coords = nullptr;       // SoA [d][n] in leaf order; tombstone = NaN in coordinate 0
  std::uint32_t* ids = nullptr;
  void* tnodes = nullptr;         // TNode<D>[n_internal]
  std::uint64_t n_internal = 0;
  std::uint64_t root_ref = 0;
  gk_canon_node* canon = nullptr; // canonical nodes, vEB slot order
  std::uint64_t n_nodes = 0;
  std::int32_t* orig = nullptr;   // build-time topology per slot: [left | right | parent] (3 x n_nodes)
  std::uint32_t* irank = nullptr; // slot -> internal rank (TNode index), n_nodes + 1
  std::int32_t root_slot = 0;     // -1 once Erase_S removed every point
  std::uint64_t* bloom = nullptr; // lazily built erase prefilter, bloom_bits bits
  std::uint64_t bloom_bits = 0;
  int height = 0;
  std::uint64_t build_size = 0, live = 0;
};

// Kernel-side tree descriptor (passed by value in a launch parameter).
struct TreeRef {
  const void* tnodes;
  const double* coords;
  const std::uint32_t* ids;
  std::uint64_t stride;
  std::uint64_t root;
  const std::uint64_t* bloom = nullptr;  // erase only; nullptr = no prefilter
  std::uint64_t bloom_bits = 0;
};

// Bloom filter over points (10 bits/key, 7 probes; SPEC.md:599-606 parameters):
// the key hashes all d coordinates with -0 canonicalised to +0 (erase matches by
// value, so -0 and +0 must probe the same bits).
constexpr int kBloomHashes = 7;
constexpr int kBloomBitsPerKey = 10;
__host__ __device__ inline std::uint64_t bloom_mix(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ inline std::uint64_t bloom_key(const double* x, int d, std::uint64_t stride) {
  std::uint64_t z = 0x243f6a8885a308d3ULL;
  for (int j = 0; j < d; ++j) {
    const double v = x[j * stride] == 0.0 ? 0.0 : x[j * stride];
    z = bloom_mix(z ^ static_cast<std::uint64_t>(__double_as_longlong(v)));
  }
  return z;
}
template <int D>
__device__ inline std::uint64_t bloom_key_reg(const double (&x)[D]) {
  std::uint64_t z = 0x243f6a8885a308d3ULL;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double v = x[j] == 0.0 ? 0.0 : x[j];
    z = bloom_mix(z ^ static_cast<std::uint64_t>(__double_as_longlong(v)));
  }
  return z;
}
// probe i of a key: bit floor(h_i m / 2^64) of the m-bit filter, h_i = h1 + i h2 (multiply-shift range
// reduction: one 64 x 64 -> high-64 multiply; a 64-bit `% m` costs ~100 instructions per probe on the GPU)
__device__ __forceinline__ std::uint64_t bloom_bit(std::uint64_t h1, std::uint64_t h2, int i, std::uint64_t m) {
  return __umul64hi(h1 + static_cast<std::uint64_t>(i) * h2, m);
}
// two probes first (their loads in flight together; an absent key leaves after them three times out of
// four), then the other five together
__device__ inline bool bloom_test(const std::uint64_t* __restrict__ bits, std::uint64_t m, std::uint64_t key) {
  const std::uint64_t h1 = key, h2 = bloom_mix(key ^ 0x5851f42d4c957f2dULL) | 1ULL;
  const std::uint64_t b0 = bloom_bit(h1, h2, 0, m), b1 = bloom_bit(h1, h2, 1, m);
  const std::uint64_t w0 = bits[b0 >> 6], w1 = bits[b1 >> 6];
  if (!((w0 >> (b0 & 63)) & (w1 >> (b1 & 63)) & 1ULL)) return false;
  std::uint64_t all = 1ULL;
#pragma unroll
  for (int i = 2; i < kBloomHashes; ++i) {
    const std::uint64_t b = bloom_bit(h1, h2, i, m);
    all &= bits[b >> 6] >> (b & 63);
  }
  return (all & 1ULL) != 0;
}
constexpr int kMaxTrees = 66;
struct TreeSet {
  TreeRef t[kMaxTrees];
  int count;
};

// build.cu
// Grow-only device scratch for BuildvEB_S plus a pinned control-word readback
// buffer.  One build can be in flight per scratch: build_begin launches the
// cooperative build kernel on `st` (asynchronously), build_finish waits for it,
// sizes the node arrays and emits them.  Builds of distinct trees on distinct
// (stream, scratch) pairs run concurrently (PAPER.md:1185 builds new trees in parallel).
struct BuildScratch {
  void* base = nullptr;
  std::size_t size = 0;
  std::uint32_t* host_ctrl = nullptr;
  alignas(16) unsigned char args[1024];  // the in-flight build's kernel arguments
  int d = 0, grid = 0;
  std::uint64_t n = 0;
  DevTree* out = nullptr;
  cudaStream_t st = nullptr;
  bool pending = false;
  ~BuildScratch();
  char* reserve(std::size_t bytes, cudaStream_t st);
};
// max_grid > 0 caps the cooperative grid (concurrent builds share the co-resident capacity)
void build_begin(BuildScratch& sc, int d, int leaf, int heuristic, const double* src, std::uint64_t src_stride,
                 const std::uint32_t* src_ids, std::uint64_t n, DevTree& out, cudaStream_t st, int max_grid = 0,
                 std::uint64_t wave_max_n = 0);  // the largest tree built concurrently with this one
// co-resident blocks of the BuildvEB_S kernel for dimension d (its largest cooperative grid)
int build_capacity(int d);
// upper bound of the device bytes one build of n points allocates (scratch + the resulting tree)
std::size_t build_bytes(int d, std::uint64_t n);
// the grid a build of n points asks for when it runs alone
int build_grid_wanted(int d, std::uint64_t n);
void build_finish(BuildScratch& sc);
inline void build_tree(BuildScratch& sc, int d, int leaf, int heuristic, const double* src, std::uint64_t src_stride,
                       const std::uint32_t* src_ids, std::uint64_t n, DevTree& out, cudaStream_t st) {
  build_begin(sc, d, leaf, heuristic, src, src_stride, src_ids, n, out, st);
  build_finish(sc);
}
void free_tree(DevTree& t, cudaStream_t st);
// Erase_S collapse (Alg. 2): after tombstoning, drop emptied leaves
// and splice out internal nodes left with one child; relinks the canonical
// nodes and the traversal nodes and updates root_slot / root_ref.
void collapse_tree(int d, DevTree& t, cudaStream_t st);
// the same for several trees, one host round-trip for all their new roots
// The trees' collapses are independent.  With side streams every tree's kernels run on one of them, forked
// from st by an event, so that st stays free for the caller's own work (Erase_L compacts and rebuilds the
// buffer meanwhile); collapse_trees_finish joins them into st, reads the new roots back (one host
// round-trip) and releases the temporaries.
struct CollapseJob {
  std::vector<DevTree*> ts;
  std::uint32_t* info = nullptr;
  std::vector<std::int32_t*> repl;
  std::vector<std::uint32_t*> arrive;
  std::vector<cudaEvent_t> ev;  // [0]: fork; [1 + i]: tree i done
  cudaStream_t st = nullptr;
};
void collapse_trees_begin(CollapseJob& job, int d, const std::vector<DevTree*>& trees, cudaStream_t st,
                          cudaStream_t* side = nullptr, int nside = 0);
void collapse_trees_finish(CollapseJob& job);
void collapse_trees(int d, const std::vector<DevTree*>& trees, cudaStream_t st, cudaStream_t* side = nullptr,
                    int nside = 0);

// knn.cu
void knn_launch(int d, int k, const TreeSet& trees, const double* q_dev, std::uint64_t nq,
                std::uint32_t* ids_dev, double* d2_dev, gk_knn_counters* counters, cudaStream_t st,
                cudaEvent_t ev_k0, cudaEvent_t ev_k1, const double* bound = nullptr);
void knn_traverse(int d, int k, const TreeSet& trees, const double* q_dev, const std::uint32_t* perm, std::uint64_t nq,
                  std::uint32_t* ids_dev, double* d2_dev, cudaStream_t st);
// range search (ball, d2 <= r2): K2 order, count / fill passes over the same order, per-query sort
void range_order(int d, const double* q_dev, std::uint64_t nq, std::uint32_t* perm, cudaStream_t st);
// mode 0: counts; 1: rows at offs; 2: the first capq rows of query i at ids/d2 + i * capq, and counts
void range_launch(int d, const TreeSet& trees, const double* q_dev, std::uint64_t nq, double r2, const double* r2q,
                  const std::uint32_t* perm,
                  unsigned long long* counts, const unsigned long long* offs, std::uint32_t* ids, double* d2, int mode,
                  unsigned capq, cudaStream_t st);
// slot rows into CSR; returns the number of overflowing queries, listed in K2 order in ovf
std::uint64_t range_slots_compact(std::uint64_t nq, unsigned capq, const std::uint32_t* perm,
                                  const unsigned long long* counts, const unsigned long long* offs, const std::uint32_t* ti,
                                  const double* td, std::uint32_t* ids, double* d2, std::uint32_t* ovf, cudaStream_t st);
void range_sort(std::uint32_t* ids, double* d2, std::uint64_t total, const unsigned long long* offs, std::uint64_t nq,
                cudaStream_t st);
void range_sort_ovf(std::uint32_t* ids, double* d2, std::uint64_t total, const unsigned long long* offs,
                    const std::uint32_t* ovf, std::uint64_t no, cudaStream_t st);
// orthogonal (box) range search: ids of live points in [lo, hi] per query, ascending
void range_box_order(int d, const double* lo, const double* hi, std::uint64_t nq, std::uint32_t* perm, cudaStream_t st);
void range_box_launch(int d, const TreeSet& trees, const double* lo, const double* hi, std::uint64_t nq,
                      const std::uint32_t* perm, unsigned long long* counts, const unsigned long long* offs,
                      std::uint32_t* ids, bool fill, cudaStream_t st);
void range_box_sort(std::uint32_t* ids, std::uint64_t total, const unsigned long long* offs, std::uint64_t nq,
                    cudaStream_t st);
// kNN graph over the n live points of `trees`: rows in ascending id order (row_ids), k neighbours each
void knn_graph_launch(int d, int k, const TreeSet& trees, std::uint64_t n, std::uint32_t* row_ids, std::uint32_t* ids,
                      double* d2, cudaStream_t st);

}  // namespace gk
