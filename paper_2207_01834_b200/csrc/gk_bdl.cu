// gk_bdl.cu — the BDL-tree log structure on the device and the C ABI
// (include/gk_bdl.h).  Host C++ orchestration, device-resident arenas.
//
// Reference semantics (restated; the reference ships no code for it):
//   BDLTree type        SPEC.md:549-555 (buffer tree, statics[i] of X*2^i, bitmask F)
//   Insert_L (Alg. 3)
//   Erase_L  (Alg. 4)
//   Erase_S  (Alg. 2)
//   kNN_L
// Frozen decisions (identical in oracle/gk_oracle.cpp):
//   * ids are global insertion ordinals; Erase_L reinsertions keep their ids
//   * Insert_L: the LAST |P| mod X points go to the buffer; on overflow the X
//     oldest buffer points drain; pool = live points of destroyed trees
//     (ascending tree index, leaf order) ++ drained ++ the first |P| - |P| mod X
//     points of P; new trees are filled largest-first from contiguous slices
//     (short/empty with tombstoned sources: an empty one clears its bit)
//   * Erase: coordinate-exact match, every duplicate; a tombstone is a NaN
//     written into coordinate 0 (never matches, never enters a k-buffer);
//     boxes are not tightened; trees with 2*live < build size are gathered
//     (ascending index, leaf order) and reinserted; buffer excluded from that rule
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "gk_common.cuh"
#include "gk_host.h"

using namespace gk;

namespace {

thread_local std::string g_last_error;

template <class T>
T* dalloc(std::size_t count, cudaStream_t st) {
  void* p = nullptr;
  if (count == 0) count = 1;
  GK_CUDA(cudaMallocAsync(&p, count * sizeof(T), st));
  return static_cast<T*>(p);
}
template <class T>
void dfree(T*& p, cudaStream_t st) {
  if (p) GK_CUDA(cudaFreeAsync(p, st));
  p = nullptr;
}
inline unsigned blocks_for(std::uint64_t n, unsigned t = 256) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, (n + t - 1) / t));
}

// ---------------------------------------------------------------- kernels --
// AoS rows (n x d) -> SoA [d][stride] + ids = base + i; flags non-finite input
__global__ void k_ingest(const double* __restrict__ aos, int d, std::uint64_t n, double* __restrict__ soa,
                         std::uint64_t stride, std::uint32_t* __restrict__ ids, std::uint64_t id_base, int* bad) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < d; ++j) {
    double x = aos[i * d + j];
    if (!isfinite(x)) *bad = 1;
    soa[j * stride + i] = x;
  }
  if (ids) ids[i] = static_cast<std::uint32_t>(id_base + i);
}

// flags a squared radius that is NaN or negative (per-query range search on device pointers)
__global__ void k_check_radii(const double* __restrict__ r2, std::uint64_t n, int* bad) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && !(r2[i] >= 0.0)) *bad = 1;
}

// copy SoA rows [0, n) from (src, sstride) to (dst, dstride)
__global__ void k_copy_soa(const double* __restrict__ src, std::uint64_t sstride, const std::uint32_t* __restrict__ sids,
                           double* __restrict__ dst, std::uint64_t dstride, std::uint32_t* __restrict__ dids, int d,
                           std::uint64_t n) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < d; ++j) dst[j * dstride + i] = src[j * sstride + i];
  dids[i] = sids[i];
}

__global__ void k_live_flags(const double* __restrict__ c0, std::uint64_t n, std::uint32_t* flags) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) flags[i] = isnan(c0[i]) ? 0u : 1u;
  else if (i == n) flags[i] = 0u;
}

__global__ void k_compact(const double* __restrict__ src, std::uint64_t sstride, const std::uint32_t* __restrict__ sids,
                          const std::uint32_t* __restrict__ flags, const std::uint32_t* __restrict__ pos, int d,
                          std::uint64_t n, double* __restrict__ dst, std::uint64_t dstride, std::uint32_t* __restrict__ dids) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !flags[i]) return;
  const std::uint32_t o = pos[i];
  for (int j = 0; j < d; ++j) dst[j * dstride + o] = src[j * sstride + i];
  dids[o] = sids[i];
}

// src[i] = arrival index of tree id ids[i]: binary search in the (id, arrival) pairs sorted by id
__global__ void k_map_src(const std::uint32_t* __restrict__ ids, std::uint64_t n, const std::uint32_t* __restrict__ skeys,
                          const std::uint32_t* __restrict__ svals, std::uint32_t* __restrict__ src) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const std::uint32_t x = ids[i];
  std::uint64_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const std::uint64_t mid = (lo + hi) / 2;
    if (skeys[mid] <= x) lo = mid;
    else hi = mid;
  }
  src[i] = svals[lo];
}

__global__ void k_iota(std::uint32_t* out, std::uint64_t n) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = static_cast<std::uint32_t>(i);
}

// buffer arrival-order live flags from the buffer tree's tombstones
__global__ void k_buffer_dead(const double* __restrict__ tree_c0, const std::uint32_t* __restrict__ src_idx, std::uint64_t n,
                              std::uint32_t* flags) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && isnan(tree_c0[i])) flags[src_idx[i]] = 0u;
}

// lazy bloom construction over a tree's live points (parallel over the point range)
__global__ void k_bloom_build(const double* __restrict__ coords, std::uint64_t n, int d, std::uint64_t* bits,
                              std::uint64_t m) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || isnan(coords[i])) return;
  const std::uint64_t key = bloom_key(coords + i, d, n);
  const std::uint64_t h1 = key, h2 = bloom_mix(key ^ 0x5851f42d4c957f2dULL) | 1ULL;
  for (int k = 0; k < kBloomHashes; ++k) {
    const std::uint64_t b = bloom_bit(h1, h2, k, m);
    atomicOr(reinterpret_cast<unsigned long long*>(&bits[b >> 6]), 1ULL << (b & 63));
  }
}

__global__ void k_bloom_query(const std::uint64_t* __restrict__ bits, std::uint64_t m, const double* __restrict__ P, int d,
                              std::uint64_t n, std::uint8_t* out) {
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  out[i] = bloom_test(bits, m, bloom_key(P + i * d, d, 1)) ? 1 : 0;
}

// Erase_S for every tree at once: one thread per erase point walks each tree
// along the children whose (conservative) box contains the point and
// tombstones coordinate-exact matches with a CAS on coordinate 0 (so every
// tombstone is counted once even with duplicate batch points).
template <int D>
__global__ void __launch_bounds__(128) k_erase(const TreeSet ts, const double* __restrict__ P,
                                               const std::uint32_t* __restrict__ perm, std::uint64_t n,
                                               unsigned long long* killed) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const std::uint64_t src = perm ? perm[i] : i;  // K2 (Hilbert) order: neighbouring threads walk neighbouring paths
  double p[D];
  float pf_lo[D], pf_hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    p[j] = P[src * D + j];
    pf_lo[j] = __double2float_rd(p[j]);
    pf_hi[j] = __double2float_ru(p[j]);
  }
  std::uint64_t stk[kStack];
  const std::uint64_t key = bloom_key_reg<D>(p);
  // candidate trees of this point: every bloom filter is tested up front (independent loads), then the
  // lane walks its candidates one after another without waiting for the warp at tree boundaries.  (A
  // loop over the trees with the warp reconverging per tree made every lane wait for each false
  // positive's walk: at 1-2 % per lane and tree, about half of the warps walked every tree.)
  unsigned long long cand = 0;
  unsigned cand_hi = 0;  // trees 64.. (kMaxTrees = 66)
  for (int t = 0; t < ts.count; ++t)
    if (!ts.t[t].bloom || bloom_test(ts.t[t].bloom, ts.t[t].bloom_bits, key)) {  // else definitely absent
      if (t < 64) cand |= 1ULL << t;
      else cand_hi |= 1u << (t - 64);
    }
  while (cand | cand_hi) {
    int t;
    if (cand) {
      t = __ffsll(static_cast<long long>(cand)) - 1;
      cand &= cand - 1;
    } else {
      t = 64 + __ffs(static_cast<int>(cand_hi)) - 1;
      cand_hi &= cand_hi - 1;
    }
    const TNode<D>* nodes = static_cast<const TNode<D>*>(ts.t[t].tnodes);
    double* coords = const_cast<double*>(ts.t[t].coords);
    const std::uint64_t stride = ts.t[t].stride;
    // the walk follows one child in a register; the stack (local memory) only takes the second child of a
    // node whose two boxes both contain the point (boundary points, duplicates)
    int sp = 0;
    std::uint64_t ref = ts.t[t].root;
    unsigned long long local = 0;
    while (true) {
      if (is_leaf_ref(ref)) {
        const std::uint32_t c = leaf_count(ref);
        const std::uint64_t s = leaf_start(ref);
        // coordinate 0 of four points at a time (independent loads; the CAS below keeps the compiler from
        // moving later loads above it, so one point per trip was one dependent round trip per point)
        for (std::uint32_t k0 = 0; k0 < c; k0 += 4) {
          double c0[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) c0[u] = k0 + u < c ? coords[s + k0 + u] : __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // compare by value (so -0 == +0 as in the oracle), then swap exactly the bits that matched
            bool eq = (c0[u] == p[0]);
            if (!eq) continue;
            const std::uint32_t k = k0 + u;
#pragma unroll
            for (int j = 1; j < D; ++j) eq = eq && (coords[j * stride + s + k] == p[j]);
            if (eq) {
              unsigned long long* a = reinterpret_cast<unsigned long long*>(&coords[s + k]);
              const unsigned long long old = static_cast<unsigned long long>(__double_as_longlong(c0[u]));
              if (atomicCAS(a, old, 0x7ff8000000000000ULL) == old) ++local;
            }
          }
        }
        if (sp == 0) break;
        ref = stk[--sp];
        continue;
      }
      // the node in D + 1 16-byte loads: (lo0, lo1) and (hi0, hi1) per dimension pair, then the child refs
      const float4* nd4 = reinterpret_cast<const float4*>(nodes + ref);
      float4 w[D + 1];
#pragma unroll
      for (int v = 0; v <= D; ++v) w[v] = __ldg(nd4 + v);
      const float* wf = reinterpret_cast<const float*>(w);  // lo[D][2], hi[D][2], ref[2]
      const std::uint64_t* wr = reinterpret_cast<const std::uint64_t*>(w + D);
      bool in[2];
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        in[sd] = true;
#pragma unroll
        for (int j = 0; j < D; ++j) in[sd] = in[sd] && (pf_hi[j] >= wf[2 * j + sd]) && (pf_lo[j] <= wf[2 * D + 2 * j + sd]);
      }
      if (in[0] && in[1]) {
        if (sp >= kStack) __trap();  // unreachable: tree depth <= kDepthCap + 31 < kStack
        stk[sp++] = wr[1];
        ref = wr[0];
      } else if (in[0]) {
        ref = wr[0];
      } else if (in[1]) {
        ref = wr[1];
      } else {
        if (sp == 0) break;
        ref = stk[--sp];
      }
    }
    if (local) atomicAdd(&killed[t], local);
  }
}

// L2 read bandwidth probe (the ceiling for traffic that hits in L2): every thread streams
// 16-byte L2-only loads (ld.global.cg, L1 bypassed) over a buffer that fits in L2
__global__ void k_l2_read(const ulonglong2* __restrict__ a, std::uint64_t n, int reps, unsigned long long* sink) {
  unsigned long long acc = 0;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
      const ulonglong2 v = __ldcg(a + i);
      acc ^= v.x ^ (v.y + static_cast<unsigned long long>(r));
    }
  if (acc == 0x9e3779b97f4a7c15ULL) *sink = acc;  // keeps the loads alive
}

}  // namespace

// GK_TRACE=1: host-side phase timestamps of Insert_L on stderr (diagnostics only)
struct PhaseTrace {
  bool on = std::getenv("GK_TRACE") != nullptr;
  bool nosync = on && std::getenv("GK_TRACE")[0] == '2';  // GK_TRACE=2: host stamps only, no stream syncs
  cudaStream_t st = nullptr;  // synchronised before each stamp when tracing
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void operator()(const char* what, long long arg = -1) const {
    if (!on) return;
    if (st && !nosync) GK_CUDA(cudaStreamSynchronize(st));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[gk] %8.3f ms  %s %lld\n", ms, what, arg);
  }
};

// ================================================================= handle ==
struct gk_bdl {
  int d = 0;
  std::uint32_t X = 1024, leaf = 16;
  int heuristic = 0, device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t pst[2] = {nullptr, nullptr};  // pipelined host-API kNN: [0] H2D, [1] D2H (compute on st)
  std::vector<cudaEvent_t> pev;               // pipeline events, grown on demand
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<DevTree> statics = std::vector<DevTree>(64);
  std::uint64_t F = 0;
  double* buf_coords = nullptr;  // arrival order, SoA stride 2X
  std::uint32_t* buf_ids = nullptr;
  std::uint64_t buf_n = 0;
  DevTree buf_tree;
  std::uint64_t next_id = 0;
  float knn_ms = 0.f, knn_total_ms = 0.f, build_ms = 0.f;
  double knn_ns_q = 0.0;  // device ns per query of the last one-shot kNN_L (k = knn_ns_k): e2e chunk planning
  int knn_ns_k = 0;
  std::uint64_t built_pts = 0;
  void* cub_tmp = nullptr;
  std::size_t cub_bytes = 0;
  BuildScratch scratch;                 // buffer-tree rebuilds (on st)
  static constexpr int kBuildSlots = 16;  // concurrent builds of distinct new trees (<= 14 per Insert_L at 2^24 points)
  BuildScratch bscratch[kBuildSlots];
  cudaStream_t bst[kBuildSlots] = {};
  cudaEvent_t ev_pool = nullptr;
  // pinned staging ring of the pageable-host kNN_L pipeline (allocated on first use)
  static constexpr int kStageSlots = 4;
  static constexpr std::size_t kStageBytes = 16u << 20;
  void* stage[kStageSlots] = {};
  cudaEvent_t stage_ev[kStageSlots] = {};

  std::uint64_t bstride() const { return 2ULL * X; }

  // The memory pool (release threshold: never) only grows, and growing it maps new physical memory
  // inside whichever cudaMallocAsync finds it short -- milliseconds each, erratic, on the host.  Before
  // an operation that allocates `bytes`, grow it once, in one piece, to have that much free.
  void ensure_pool(std::size_t bytes) {
    cudaMemPool_t pool;
    GK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    std::uint64_t reserved = 0, used = 0;
    GK_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    GK_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
    const std::uint64_t free_b = reserved > used ? reserved - used : 0;
    if (free_b >= bytes) return;
    const std::size_t grow = bytes + bytes / 4;
    void* p = nullptr;
    if (cudaMallocAsync(&p, grow, st) != cudaSuccess) {  // out of memory here is not an error yet: the
      cudaGetLastError();                                // operation itself may still fit
      return;
    }
    GK_CUDA(cudaFreeAsync(p, st));
    GK_CUDA(cudaStreamSynchronize(st));  // the free completed: every stream may reuse the block
  }

  void ensure_stage() {
    if (stage[0]) return;
    for (int i = 0; i < kStageSlots; ++i) {
      GK_CUDA(cudaMallocHost(&stage[i], kStageBytes));
      GK_CUDA(cudaEventCreateWithFlags(&stage_ev[i], cudaEventDisableTiming));
    }
  }

  void scan(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n) {
    std::size_t need = 0;
    GK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, static_cast<int>(n), st));
    if (need > cub_bytes) {
      if (cub_tmp) GK_CUDA(cudaFreeAsync(cub_tmp, st));
      cub_bytes = std::max(need, 2 * cub_bytes);
      GK_CUDA(cudaMallocAsync(&cub_tmp, cub_bytes, st));
    }
    GK_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, need, in, out, static_cast<int>(n), st));
  }

  // order-preserving copy of the live points of tree T to (dst + off, dstride)
  std::uint64_t gather_live(const DevTree& T, double* dst, std::uint64_t dstride, std::uint32_t* dids, std::uint64_t off) {
    if (T.n == 0) return 0;
    std::uint32_t* flags = dalloc<std::uint32_t>(T.n + 1, st);
    std::uint32_t* pos = dalloc<std::uint32_t>(T.n + 1, st);
    k_live_flags<<<blocks_for(T.n + 1), 256, 0, st>>>(T.coords, T.n, flags);
    scan(flags, pos, T.n + 1);
    k_compact<<<blocks_for(T.n), 256, 0, st>>>(T.coords, T.n, T.ids, flags, pos, d, T.n, dst + off, dstride, dids + off);
    GK_CHECK_LAUNCH();
    dfree(flags, st);
    dfree(pos, st);
    return T.live;
  }

  void rebuild_buffer_tree() {
    PhaseTrace tr;
    tr.st = st;
    free_tree(buf_tree, st);
    if (buf_n == 0) return;
    // Build_S over the buffer with its real ids (object-median ties break by id, as in every static tree)
    build_begin(scratch, d, static_cast<int>(leaf), heuristic, buf_coords, bstride(), buf_ids, buf_n, buf_tree, st);
    tr("  buffer: k_build done");
    build_finish(scratch);
    tr("  buffer: emitted");
  }

  // src[pos] = arrival index of the buffer point at buffer-tree position pos (erase compaction only):
  // ids are unique, so sort (id, arrival) by id and binary-search each tree id
  std::uint32_t* buffer_src_map() {
    std::uint32_t* iota = dalloc<std::uint32_t>(buf_n, st);
    std::uint32_t* skeys = dalloc<std::uint32_t>(buf_n, st);
    std::uint32_t* svals = dalloc<std::uint32_t>(buf_n, st);
    k_iota<<<blocks_for(buf_n), 256, 0, st>>>(iota, buf_n);
    std::size_t tb = 0;
    GK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, buf_ids, skeys, iota, svals, static_cast<int>(buf_n), 0, 32, st));
    void* tmp = dalloc<char>(tb, st);
    GK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, buf_ids, skeys, iota, svals, static_cast<int>(buf_n), 0, 32, st));
    std::uint32_t* src = dalloc<std::uint32_t>(buf_n, st);
    k_map_src<<<blocks_for(buf_n), 256, 0, st>>>(buf_tree.ids, buf_n, skeys, svals, src);
    GK_CHECK_LAUNCH();
    dfree(tmp, st);
    dfree(iota, st);
    dfree(skeys, st);
    dfree(svals, st);
    return src;
  }

  // Insert_L of device SoA points (stride sp) with their ids.
  void insert_l(const double* P, std::uint64_t sp, const std::uint32_t* ids, std::uint64_t n) {
    if (n == 0) return;
    PhaseTrace tr;
    tr.st = st;
    const std::uint64_t r = n % X, bulk = n - r;
    tr("insert_l start");
    if (r) {
      k_copy_soa<<<blocks_for(r), 256, 0, st>>>(P + bulk, sp, ids + bulk, buf_coords + buf_n, bstride(), buf_ids + buf_n, d, r);
      GK_CHECK_LAUNCH();
      buf_n += r;
    }
    tr("buffer append", static_cast<long long>(r));
    const std::uint64_t drained = (buf_n >= X) ? X : 0;
    const std::uint64_t add = (bulk + drained) / X;
    if (add == 0) {
      if (r) rebuild_buffer_tree();
      return;
    }
    const std::uint64_t Fn = F + add;
    const std::uint64_t destroyed = F & ~Fn, built = Fn & ~F;
    std::uint64_t pool_n = drained + bulk;
    for (int i = 0; i < 64; ++i)
      if (destroyed >> i & 1ULL) pool_n += statics[i].live;
    {
      std::size_t need = pool_n * (8 * d + 4) + build_bytes(d, buf_n + X);
      std::uint64_t left = pool_n;
      for (int i = 63; i >= 0; --i)
        if (built >> i & 1ULL) {
          const std::uint64_t c = std::min<std::uint64_t>(static_cast<std::uint64_t>(X) << i, left);
          need += build_bytes(d, c);
          left -= c;
        }
      ensure_pool(need);
    }
    double* pool = dalloc<double>(pool_n * d, st);
    std::uint32_t* pool_ids = dalloc<std::uint32_t>(pool_n, st);
    tr("pool allocated", static_cast<long long>(pool_n));
    std::uint64_t off = 0;
    for (int i = 0; i < 64; ++i)
      if (destroyed >> i & 1ULL) {
        off += gather_live(statics[i], pool, pool_n, pool_ids, off);
        free_tree(statics[i], st);
      }
    if (drained) {
      k_copy_soa<<<blocks_for(X), 256, 0, st>>>(buf_coords, bstride(), buf_ids, pool + off, pool_n, pool_ids + off, d, X);
      off += X;
      // shift the remaining buffer points to the front (arrival order kept)
      const std::uint64_t rest = buf_n - X;
      if (rest) {
        double* tmpc = dalloc<double>(rest * d, st);
        std::uint32_t* tmpi = dalloc<std::uint32_t>(rest, st);
        k_copy_soa<<<blocks_for(rest), 256, 0, st>>>(buf_coords + X, bstride(), buf_ids + X, tmpc, rest, tmpi, d, rest);
        k_copy_soa<<<blocks_for(rest), 256, 0, st>>>(tmpc, rest, tmpi, buf_coords, bstride(), buf_ids, d, rest);
        dfree(tmpc, st);
        dfree(tmpi, st);
      }
      buf_n = rest;
    }
    if (bulk) {
      k_copy_soa<<<blocks_for(bulk), 256, 0, st>>>(P, sp, ids, pool + off, pool_n, pool_ids + off, d, bulk);
      off += bulk;
    }
    GK_CHECK_LAUNCH();
    tr("pool staged (launches)", static_cast<long long>(pool_n));
    // build the new trees, largest first, from contiguous pool slices; distinct trees
    // build concurrently on their own streams
    F = Fn;
    std::vector<int> order;
    std::vector<std::uint64_t> offs, cnts;
    std::uint64_t o = 0;
    for (int i = 63; i >= 0; --i) {
      if (!(built >> i & 1ULL)) continue;
      const std::uint64_t cap = static_cast<std::uint64_t>(X) << i;
      const std::uint64_t c = std::min(cap, pool_n - o);
      if (c == 0) {
        F &= ~(1ULL << i);
        continue;
      }
      order.push_back(i);
      offs.push_back(o);
      cnts.push_back(c);
      o += c;
    }
    const auto t0 = std::chrono::steady_clock::now();
    GK_CUDA(cudaEventRecord(ev_pool, st));
    const bool rebuild_buf = r || drained;
    for (std::size_t w0 = 0; w0 < order.size(); w0 += kBuildSlots) {
      const std::size_t w1 = std::min(order.size(), w0 + kBuildSlots);
      // the wave's cooperative grids share the co-resident capacity (one block kept for the
      // buffer tree), in proportion to their points, so every build of the wave runs at once
      // instead of the small trees queueing behind the largest one's full-GPU grid
      const int cap = build_capacity(d) - (rebuild_buf && w0 == 0 ? 1 : 0);
      std::vector<int> grid(w1 - w0);
      long long want = 0;
      for (std::size_t t = w0; t < w1; ++t) {
        want += grid[t - w0] = build_grid_wanted(d, cnts[t]);
      }
      if (want > cap) {
        // shares in proportion to points^p (GK_GRID_POW, experiments; p > 1 favours the largest tree)
        static const double gp = std::getenv("GK_GRID_POW") ? std::atof(std::getenv("GK_GRID_POW")) : 1.0;
        double wsum = 0.0;
        for (std::size_t t = w0; t < w1; ++t) wsum += std::pow(static_cast<double>(cnts[t]), gp);
        const int spare = cap - static_cast<int>(w1 - w0);
        for (std::size_t t = w0; t < w1; ++t)
          grid[t - w0] = std::min(grid[t - w0], 1 + static_cast<int>(static_cast<double>(spare) *
                                                                     std::pow(static_cast<double>(cnts[t]), gp) / wsum));
      }
      for (std::size_t t = w0; t < w1; ++t) {
        const int slot = static_cast<int>(t - w0);
        GK_CUDA(cudaStreamWaitEvent(bst[slot], ev_pool, 0));
        build_begin(bscratch[slot], d, static_cast<int>(leaf), heuristic, pool + offs[t], pool_n, pool_ids + offs[t],
                    cnts[t], statics[order[t]], bst[slot], grid[slot], cnts[w0]);
        tr("  build launched, points", static_cast<long long>(cnts[t]));
      }
      if (w0 == 0 && rebuild_buf) {  // the buffer tree builds on st, alongside the static trees
        rebuild_buffer_tree();
        tr("buffer tree rebuilt", static_cast<long long>(buf_n));
      }
      for (std::size_t t = w0; t < w1; ++t) {
        build_finish(bscratch[t - w0]);
        tr("  build finished, points", static_cast<long long>(cnts[t]));
      }
    }
    if (order.empty() && rebuild_buf) rebuild_buffer_tree();
    for (auto& bs : bst) GK_CUDA(cudaStreamSynchronize(bs));
    build_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    tr("all builds done");
    built_pts = o;
    dfree(pool, st);
    dfree(pool_ids, st);
    GK_CUDA(cudaStreamSynchronize(st));
    tr("insert_l done");
  }

  // bloom filters are built lazily, on the first erase that touches the tree
  void ensure_bloom(DevTree& T) {
    if (T.bloom || T.n == 0) return;
    const std::uint64_t m = std::max<std::uint64_t>(64, ((T.n * kBloomBitsPerKey + 63) / 64) * 64);
    T.bloom = dalloc<std::uint64_t>(m / 64, st);
    T.bloom_bits = m;
    GK_CUDA(cudaMemsetAsync(T.bloom, 0, m / 8, st));
    k_bloom_build<<<blocks_for(T.n), 256, 0, st>>>(T.coords, T.n, d, T.bloom, m);
    GK_CHECK_LAUNCH();
  }

  TreeSet trees(bool include_buffer = true) const {
    TreeSet ts{};
    ts.count = 0;
    for (int i = 63; i >= 0; --i)
      if ((F >> i & 1ULL) && statics[i].live > 0) {
        const DevTree& T = statics[i];
        ts.t[ts.count++] = TreeRef{T.tnodes, T.coords, T.ids, T.n, T.root_ref};
      }
    if (include_buffer && buf_n > 0)
      ts.t[ts.count++] = TreeRef{buf_tree.tnodes, buf_tree.coords, buf_tree.ids, buf_tree.n, buf_tree.root_ref};
    return ts;
  }

  std::uint64_t erase_l(const double* P_aos, std::uint64_t n) {
    if (n == 0) return 0;
    // all trees (largest first) + buffer tree, one kernel
    std::vector<int> which;
    TreeSet ts{};
    for (int i = 63; i >= 0; --i)
      if ((F >> i & 1ULL) && statics[i].live > 0) {
        DevTree& T = statics[i];
        ensure_bloom(T);
        ts.t[ts.count++] = TreeRef{T.tnodes, T.coords, T.ids, T.n, T.root_ref, T.bloom, T.bloom_bits};
        which.push_back(i);
      }
    if (buf_n > 0) {
      ts.t[ts.count++] = TreeRef{buf_tree.tnodes, buf_tree.coords, buf_tree.ids, buf_tree.n, buf_tree.root_ref};
      which.push_back(-1);
    }
    if (ts.count == 0) return 0;
    unsigned long long* killed = dalloc<unsigned long long>(kMaxTrees, st);
    GK_CUDA(cudaMemsetAsync(killed, 0, kMaxTrees * 8, st));
    std::uint32_t* perm = nullptr;
    if (n >= 4096 && n < 0xffffffffULL) {
      perm = dalloc<std::uint32_t>(n, st);
      range_order(d, P_aos, n, perm, st);
    }
    switch (d) {
#define GK_D(DD) case DD: k_erase<DD><<<blocks_for(n, 128), 128, 0, st>>>(ts, P_aos, perm, n, killed); break;
      GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    }
    GK_CHECK_LAUNCH();
    if (perm) dfree(perm, st);
    std::vector<unsigned long long> hk(kMaxTrees);
    GK_CUDA(cudaMemcpyAsync(hk.data(), killed, kMaxTrees * 8, cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    dfree(killed, st);
    std::uint64_t total = 0;
    std::vector<DevTree*> hit;
    for (std::size_t t = 0; t < which.size(); ++t)
      if (which[t] >= 0 && hk[t]) hit.push_back(&statics[which[t]]);
    for (std::size_t t = 0; t < which.size(); ++t)
      if (which[t] >= 0) statics[which[t]].live -= hk[t];
    // the static trees' collapses run side by side on the build streams while st compacts and rebuilds the buffer
    CollapseJob cjob;
    collapse_trees_begin(cjob, d, hit, st, bst, kBuildSlots);
    for (std::size_t t = 0; t < which.size(); ++t) {
      total += hk[t];
      if (which[t] >= 0) {
        continue;
      } else if (hk[t]) {
        // drop the dead buffer points, keeping arrival order, and rebuild the buffer tree
        std::uint32_t* flags = dalloc<std::uint32_t>(buf_n + 1, st);
        std::uint32_t* pos = dalloc<std::uint32_t>(buf_n + 1, st);
        std::vector<std::uint32_t> ones(buf_n + 1, 1u);
        ones[buf_n] = 0;
        GK_CUDA(cudaMemcpyAsync(flags, ones.data(), (buf_n + 1) * 4, cudaMemcpyHostToDevice, st));
        std::uint32_t* src = buffer_src_map();
        k_buffer_dead<<<blocks_for(buf_n), 256, 0, st>>>(buf_tree.coords, src, buf_n, flags);
        dfree(src, st);
        scan(flags, pos, buf_n + 1);
        double* nc = dalloc<double>(bstride() * d, st);
        std::uint32_t* ni = dalloc<std::uint32_t>(bstride(), st);
        k_compact<<<blocks_for(buf_n), 256, 0, st>>>(buf_coords, bstride(), buf_ids, flags, pos, d, buf_n, nc, bstride(), ni);
        GK_CHECK_LAUNCH();
        dfree(buf_coords, st);
        dfree(buf_ids, st);
        buf_coords = nc;
        buf_ids = ni;
        buf_n -= hk[t];
        dfree(flags, st);
        dfree(pos, st);
        rebuild_buffer_tree();
      }
    }
    collapse_trees_finish(cjob);
    // trees below half of their build size are gathered into R and reinserted
    std::uint64_t rn = 0;
    for (int i = 0; i < 64; ++i)
      if ((F >> i & 1ULL) && 2 * statics[i].live < statics[i].build_size) rn += statics[i].live;
    std::vector<int> gone;
    for (int i = 0; i < 64; ++i)
      if ((F >> i & 1ULL) && 2 * statics[i].live < statics[i].build_size) gone.push_back(i);
    if (!gone.empty()) {
      double* R = dalloc<double>(rn * d, st);
      std::uint32_t* Rid = dalloc<std::uint32_t>(rn, st);
      std::uint64_t off = 0;
      for (int i : gone) {
        off += gather_live(statics[i], R, rn, Rid, off);
        free_tree(statics[i], st);
        F &= ~(1ULL << i);
      }
      insert_l(R, rn, Rid, rn);
      dfree(R, st);
      dfree(Rid, st);
    }
    GK_CUDA(cudaStreamSynchronize(st));
    return total;
  }

  std::uint64_t live_total() const {
    std::uint64_t s = buf_n;
    for (int i = 0; i < 64; ++i)
      if (F >> i & 1ULL) s += statics[i].live;
    return s;
  }
};

// ==================================================================== C ABI ==
namespace {
int fail(int code, const std::string& m) {
  g_last_error = m;
  return code;
}
template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return GK_OK;
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::exception& e) {
    return fail(GK_ERR_LOGIC, e.what());
  }
}
void need(bool c, const std::string& m) {
  if (!c) throw Error(GK_ERR_INVALID, m);
}
struct DevScope {  // make the handle's GPU current for the call
  int prev = 0;
  explicit DevScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) GK_CUDA(cudaSetDevice(dev));
  }
  ~DevScope() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};
// frees the stream-ordered temporaries of a call on every exit path (no throw from the destructor)
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* take(std::size_t count) {
    T* p = dalloc<T>(count, st);
    ptrs.push_back(p);
    return p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
};

}  // namespace

extern "C" {

const char* gk_last_error(void) { return g_last_error.c_str(); }
const char* gk_version(void) { return "gk_bdl 0.1 (sm_100a)"; }

int gk_bdl_create(int dim, uint32_t X, uint32_t leaf, int heuristic, int device, gk_bdl** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    need(dim >= 2 && dim <= 8, "unsupported dimension " + std::to_string(dim));
    need(X >= 1, "buffer size X must be >= 1");
    need(leaf >= 1 && leaf <= GK_MAX_LEAF, "leaf size must be in [1, 32]");
    need(heuristic == GK_SPATIAL_MEDIAN || heuristic == GK_OBJECT_MEDIAN, "unknown splitting heuristic");
    int ndev = 0;
    GK_CUDA(cudaGetDeviceCount(&ndev));
    need(device >= 0 && device < ndev, "no such CUDA device");
    DevScope ds(device);
    auto* h = new gk_bdl();
    h->d = dim;
    h->X = X;
    h->leaf = leaf;
    h->heuristic = heuristic;
    h->device = device;
    try {
      GK_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
      for (auto& ps : h->pst) GK_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
      for (auto& bs : h->bst) GK_CUDA(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
      GK_CUDA(cudaEventCreateWithFlags(&h->ev_pool, cudaEventDisableTiming));
      // pinned control words of every build slot, allocated here rather than inside a timed Insert_L
      GK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->scratch.host_ctrl), 64));
      for (auto& bs : h->bscratch) GK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&bs.host_ctrl), 64));
      for (auto& e : h->ev) GK_CUDA(cudaEventCreate(&e));
      cudaMemPool_t pool;
      GK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      std::uint64_t thr = ~0ULL;  // keep freed blocks cached in the pool
      GK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      h->buf_coords = dalloc<double>(h->bstride() * dim, h->st);
      h->buf_ids = dalloc<std::uint32_t>(h->bstride(), h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int gk_bdl_destroy(gk_bdl* h) {
  if (!h) return GK_OK;
  return guard([&] {
    DevScope ds(h->device);
    for (auto& t : h->statics) free_tree(t, h->st);
    free_tree(h->buf_tree, h->st);
    dfree(h->buf_coords, h->st);
    dfree(h->buf_ids, h->st);
    if (h->cub_tmp) cudaFreeAsync(h->cub_tmp, h->st);
    cudaStreamSynchronize(h->st);
    for (auto& e : h->ev) cudaEventDestroy(e);
    for (auto& ps : h->pst) cudaStreamDestroy(ps);
    for (auto& e : h->pev) cudaEventDestroy(e);
    for (auto& bs : h->bst) cudaStreamDestroy(bs);
    cudaEventDestroy(h->ev_pool);
    for (int i = 0; i < gk_bdl::kStageSlots; ++i)
      if (h->stage[i]) {
        cudaFreeHost(h->stage[i]);
        cudaEventDestroy(h->stage_ev[i]);
      }
    cudaStreamDestroy(h->st);
    delete h;
  });
}

static void insert_device_impl(gk_bdl* h, const double* pts_dev, std::uint64_t n) {
  if (n == 0) return;
  if (h->next_id + n > 0xffffffffULL) throw Error(GK_ERR_LOGIC, "id space exhausted (uint32 PointId)");
  double* soa = dalloc<double>(n * h->d, h->st);
  std::uint32_t* ids = dalloc<std::uint32_t>(n, h->st);
  int* bad = dalloc<int>(1, h->st);
  GK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), h->st));
  k_ingest<<<blocks_for(n), 256, 0, h->st>>>(pts_dev, h->d, n, soa, n, ids, h->next_id, bad);
  GK_CHECK_LAUNCH();
  int hb = 0;
  GK_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  GK_CUDA(cudaStreamSynchronize(h->st));
  if (hb) {
    dfree(soa, h->st);
    dfree(ids, h->st);
    dfree(bad, h->st);
    throw Error(GK_ERR_INVALID, "non-finite coordinate in insert batch");
  }
  h->next_id += n;
  h->insert_l(soa, n, ids, n);
  dfree(soa, h->st);
  dfree(ids, h->st);
  dfree(bad, h->st);
  GK_CUDA(cudaStreamSynchronize(h->st));
}

int gk_bdl_insert_device(gk_bdl* h, const double* pts_dev, uint64_t n) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(n == 0 || pts_dev != nullptr, "null points");
    DevScope ds(h->device);
    insert_device_impl(h, pts_dev, n);
  });
}

int gk_bdl_insert(gk_bdl* h, const double* pts, uint64_t n) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(n == 0 || pts != nullptr, "null points");
    if (n == 0) return;
    DevScope ds(h->device);
    double* d = dalloc<double>(n * h->d, h->st);
    GK_CUDA(cudaMemcpyAsync(d, pts, n * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    insert_device_impl(h, d, n);
    dfree(d, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_erase_device(gk_bdl* h, const double* pts_dev, uint64_t n, uint64_t* n_erased) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(n == 0 || pts_dev != nullptr, "null points");
    DevScope ds(h->device);
    std::uint64_t k = h->erase_l(pts_dev, n);
    if (n_erased) *n_erased = k;
  });
}

int gk_bdl_erase(gk_bdl* h, const double* pts, uint64_t n, uint64_t* n_erased) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(n == 0 || pts != nullptr, "null points");
    DevScope ds(h->device);
    std::uint64_t k = 0;
    if (n) {
      double* d = dalloc<double>(n * h->d, h->st);
      GK_CUDA(cudaMemcpyAsync(d, pts, n * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
      k = h->erase_l(d, n);
      dfree(d, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
    }
    if (n_erased) *n_erased = k;
  });
}

static void knn_device_impl(gk_bdl* h, const double* q_dev, std::uint64_t nq, int k, std::uint32_t* ids_dev,
                            double* d2_dev, gk_knn_counters* ctr, const double* bound = nullptr) {
  need(k >= 1, "k must be >= 1");
  if (k > GK_MAX_K) throw Error(GK_ERR_UNSUPPORTED, "k > " + std::to_string(GK_MAX_K) + " is not supported");
  if (nq == 0) return;
  TreeSet ts = h->trees();
  GK_CUDA(cudaEventRecord(h->ev[0], h->st));
  if (ts.count == 0) {
    // empty structure: every row is (kNoPoint, +inf)
    GK_CUDA(cudaMemsetAsync(ids_dev, 0xff, nq * k * sizeof(std::uint32_t), h->st));
    std::vector<double> inf(nq * k, INFINITY);
    GK_CUDA(cudaMemcpyAsync(d2_dev, inf.data(), nq * k * sizeof(double), cudaMemcpyHostToDevice, h->st));
    GK_CUDA(cudaStreamSynchronize(h->st));
    return;
  }
  knn_launch(h->d, k, ts, q_dev, nq, ids_dev, d2_dev, ctr, h->st, h->ev[2], h->ev[3], bound);
  GK_CUDA(cudaEventRecord(h->ev[1], h->st));
  GK_CUDA(cudaStreamSynchronize(h->st));
  GK_CUDA(cudaEventElapsedTime(&h->knn_ms, h->ev[2], h->ev[3]));
  GK_CUDA(cudaEventElapsedTime(&h->knn_total_ms, h->ev[0], h->ev[1]));
  if (nq >= (1u << 16) && !ctr && !bound) {
    h->knn_ns_q = 1e6 * h->knn_total_ms / static_cast<double>(nq);
    h->knn_ns_k = k;
  }
}

int gk_bdl_knn_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, uint32_t* ids_dev, double* d2_dev) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (q_dev && ids_dev && d2_dev), "null buffer");
    DevScope ds(h->device);
    knn_device_impl(h, q_dev, nq, k, ids_dev, d2_dev, nullptr);
  });
}

int gk_diag_l2_read_gbs(int device, uint64_t bytes, double* gbs) {
  return guard([&] {
    need(gbs != nullptr, "null output");
    need(bytes >= (1u << 20) && bytes % 16 == 0, "bytes must be >= 1 MiB and a multiple of 16");
    DevScope ds(device);
    cudaStream_t st = nullptr;
    GK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ulonglong2* a = dalloc<ulonglong2>(bytes / 16, st);
    unsigned long long* sink = dalloc<unsigned long long>(1, st);
    GK_CUDA(cudaMemsetAsync(a, 1, bytes, st));
    int sms = 0, per = 0;
    GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_l2_read, 512, 0));
    const unsigned grid = static_cast<unsigned>(std::max(1, per) * sms);
    const int reps = 20;
    cudaEvent_t e0, e1;
    GK_CUDA(cudaEventCreate(&e0));
    GK_CUDA(cudaEventCreate(&e1));
    k_l2_read<<<grid, 512, 0, st>>>(a, bytes / 16, 2, sink);  // warm: the buffer L2-resident
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
      GK_CUDA(cudaEventRecord(e0, st));
      k_l2_read<<<grid, 512, 0, st>>>(a, bytes / 16, reps, sink);
      GK_CUDA(cudaEventRecord(e1, st));
      GK_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      GK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    GK_CHECK_LAUNCH();
    *gbs = static_cast<double>(bytes) * reps / (best * 1e-3) / 1e9;
    dfree(a, st);
    dfree(sink, st);
    GK_CUDA(cudaStreamSynchronize(st));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

int gk_bdl_knn_bounded_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, const double* r2_dev,
                              uint32_t* ids_dev, double* d2_dev) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (q_dev && r2_dev && ids_dev && d2_dev), "null buffer");
    DevScope ds(h->device);
    if (nq > 0) {
      int* bad = dalloc<int>(1, h->st);
      int hb = 0;
      GK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), h->st));
      k_check_radii<<<blocks_for(nq), 256, 0, h->st>>>(r2_dev, nq, bad);
      GK_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st));
      dfree(bad, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
      need(hb == 0, "every r2 must be a non-negative squared radius");
    }
    knn_device_impl(h, q_dev, nq, k, ids_dev, d2_dev, nullptr, r2_dev);
  });
}

int gk_bdl_knn_counted_device(gk_bdl* h, const double* q_dev, uint64_t nq, int k, uint32_t* ids_dev, double* d2_dev,
                              gk_knn_counters* counters) {
  return guard([&] {
    need(h != nullptr && counters != nullptr, "null handle/counters");
    need(nq == 0 || (q_dev && ids_dev && d2_dev), "null buffer");
    DevScope ds(h->device);
    std::memset(counters, 0, sizeof(*counters));
    knn_device_impl(h, q_dev, nq, k, ids_dev, d2_dev, counters);
  });
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int gk_bdl_knn(gk_bdl* h, const double* q, uint64_t nq, int k, uint32_t* ids, double* d2) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (q && ids && d2), "null buffer");
    need(k >= 1, "k must be >= 1");
    if (k > GK_MAX_K) throw Error(GK_ERR_UNSUPPORTED, "k > " + std::to_string(GK_MAX_K) + " is not supported");
    if (nq == 0) return;
    DevScope ds(h->device);
    const TreeSet ts = h->trees();
    // chunk schedule (weights below); experiments: GK_PIPE_FRACS="w1,w2,..." or a geometric
    // schedule of GK_PIPE_CHUNKS chunks growing by GK_PIPE_RATIO.
    int nchunk = 4;
    double ratio = 1.0;
    if (const char* e = std::getenv("GK_PIPE_CHUNKS")) nchunk = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("GK_PIPE_RATIO")) ratio = std::max(0.1, std::atof(e));
    std::vector<double> wts;  // chunk weights: geometric, or an explicit list (GK_PIPE_FRACS="1,8,7,4,4")
    if (const char* e = std::getenv("GK_PIPE_FRACS")) {
      for (const char* p = e; *p;) {
        char* end = nullptr;
        const double v = std::strtod(p, &end);
        if (end == p) break;
        if (v > 0) wts.push_back(v);
        p = (*end == ',') ? end + 1 : end;
      }
    }
    if (wts.empty() && (std::getenv("GK_PIPE_CHUNKS") || std::getenv("GK_PIPE_RATIO")))
      for (int c = 0; c < nchunk; ++c) wts.push_back(std::pow(ratio, c));
    // default: two large chunks first (their packets stay compact: K1 of a 1/4 chunk costs 1.6x its
    // share of the one-piece kernel), then shrinking ones so the last D2H after the last kNN_L is short.
    // C2 sweep (profiles/e2e_sweep.py): 7,7,5,3,2 -> 29.9 ms; 4 equal chunks 31.1; 3 equal 30.6.
    if (wts.empty()) {
      // Chunking overlaps the PCIe copies with kNN_L but makes each chunk's query packets sparser
      // (C2: a quarter of the queries costs 1.6x its share).  Plan from the device cost per query
      // of the last one-shot kNN_L with this k (or a guess by dimension) against the PCIe cost:
      //   compute-bound (C3, 7D: 25 ns vs 2.2 ns)  -> one coherent chunk (5 chunks were 1.6x slower);
      //   transfer-bound, small batch (C1, 1M)     -> two chunks;
      //   transfer-bound, large batch (C2, 10M)    -> 7,7,5,3,2 (two large chunks, short D2H tail).
      const double tx = static_cast<double>(h->d * 8 + k * 12) / 55.0;  // ns per query at ~55 GB/s
      const double tc = (h->knn_ns_k == k && h->knn_ns_q > 0.0) ? h->knn_ns_q : (h->d >= 5 ? 10.0 * tx : 0.5 * tx);
      if (tc > 1.2 * tx) wts = {1};
      else if (nq < (4ULL << 20)) wts = {1, 1};
      else wts = {7, 7, 5, 3, 2};
    }
    nchunk = static_cast<int>(wts.size());
    std::vector<std::uint64_t> bounds{0};
    {
      double wsum = 0.0;
      for (double w : wts) wsum += w;
      double acc = 0.0;
      for (int c = 0; c < nchunk; ++c) {
        const double w = wts[c];
        acc += w;
        const std::uint64_t e = c + 1 == nchunk ? nq : static_cast<std::uint64_t>(static_cast<double>(nq) * acc / wsum);
        if (e - bounds.back() >= (1u << 16) || (c + 1 == nchunk && e > bounds.back())) bounds.push_back(e);
      }
      if (bounds.back() != nq) bounds.back() = nq;
    }
    const std::uint64_t nck = bounds.size() - 1;
    if (ts.count > 0 && nck > 1 && is_pinned(q) && is_pinned(ids) && is_pinned(d2)) {
      // pinned host buffers: three-stage pipeline over full-size device buffers, chained by events --
      // H2D of every chunk on pst[0], kNN_L of chunk i on st once its queries landed, D2H of chunk i on
      // pst[1] once its rows are final.  Each chunk is Hilbert-ordered on its own; results are
      // bit-identical to the one-shot path.
      // The K2 order of chunk c + 1 runs on a side stream (the first build stream) as soon as its queries
      // landed: its kernels fill the SMs that chunk c's persistent K1 blocks leave at its tail, instead of
      // starting after it (5 x ~0.25 ms on the compute stream's chain).
      while (h->pev.size() < 3 * nck + 2) {
        cudaEvent_t e;
        GK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->pev.push_back(e);
      }
      cudaEvent_t ev_alloc = h->pev[0], ev_done = h->pev[1];
      cudaEvent_t* ev_ord = h->pev.data() + 2 + 2 * nck;
      cudaStream_t ost = h->bst[0];
      double* dq = dalloc<double>(nq * h->d, h->st);
      std::uint32_t* di = dalloc<std::uint32_t>(nq * k, h->st);
      double* dd = dalloc<double>(nq * k, h->st);
      std::uint32_t* dperm = dalloc<std::uint32_t>(nq, h->st);
      GK_CUDA(cudaEventRecord(ev_alloc, h->st));
      GK_CUDA(cudaStreamWaitEvent(h->pst[0], ev_alloc, 0));
      GK_CUDA(cudaStreamWaitEvent(h->pst[1], ev_alloc, 0));
      GK_CUDA(cudaStreamWaitEvent(ost, ev_alloc, 0));
      for (std::uint64_t c = 0; c < nck; ++c) {
        const std::uint64_t off = bounds[c], m = bounds[c + 1] - off;
        GK_CUDA(cudaMemcpyAsync(dq + off * h->d, q + off * h->d, m * h->d * sizeof(double), cudaMemcpyHostToDevice,
                                h->pst[0]));
        GK_CUDA(cudaEventRecord(h->pev[2 + 2 * c], h->pst[0]));
        GK_CUDA(cudaStreamWaitEvent(ost, h->pev[2 + 2 * c], 0));
        range_order(h->d, dq + off * h->d, m, dperm + off, ost);
        GK_CUDA(cudaEventRecord(ev_ord[c], ost));
      }
      for (std::uint64_t c = 0; c < nck; ++c) {
        const std::uint64_t off = bounds[c], m = bounds[c + 1] - off;
        GK_CUDA(cudaStreamWaitEvent(h->st, ev_ord[c], 0));
        knn_traverse(h->d, k, ts, dq + off * h->d, dperm + off, m, di + off * k, dd + off * k, h->st);
        GK_CUDA(cudaEventRecord(h->pev[3 + 2 * c], h->st));
        GK_CUDA(cudaStreamWaitEvent(h->pst[1], h->pev[3 + 2 * c], 0));
        GK_CUDA(cudaMemcpyAsync(ids + off * k, di + off * k, m * k * sizeof(std::uint32_t), cudaMemcpyDeviceToHost,
                                h->pst[1]));
        GK_CUDA(cudaMemcpyAsync(d2 + off * k, dd + off * k, m * k * sizeof(double), cudaMemcpyDeviceToHost, h->pst[1]));
      }
      GK_CUDA(cudaEventRecord(ev_done, h->pst[1]));
      GK_CUDA(cudaStreamWaitEvent(h->st, ev_done, 0));
      dfree(dq, h->st);
      dfree(di, h->st);
      dfree(dd, h->st);
      dfree(dperm, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
      return;
    }
    if (ts.count > 0 && nck > 1) {
      // pageable host buffers (a std::vector caller): the same three-stage pipeline through a pinned
      // staging ring -- host threads copy each 16 MiB block of queries into a ring slot that PCIe then
      // reads, and copy each block of result rows out of the slot PCIe wrote, while the GPU works on the
      // other slots and chunks.  Buffers that are already pinned are copied directly.
      h->ensure_stage();
      while (h->pev.size() < 3 * nck + 2) {
        cudaEvent_t e;
        GK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->pev.push_back(e);
      }
      const int nth = std::max(1, std::min(16, host_threads()));
      const bool pq = is_pinned(q), pi = is_pinned(ids), pd = is_pinned(d2);
      cudaEvent_t ev_alloc = h->pev[0], ev_done = h->pev[1];
      cudaEvent_t* ev_ord = h->pev.data() + 2 + 2 * nck;  // chunk c K2-ordered (on the side stream, as above)
      cudaStream_t ost = h->bst[0];
      double* dq = dalloc<double>(nq * h->d, h->st);
      std::uint32_t* di = dalloc<std::uint32_t>(nq * k, h->st);
      double* dd = dalloc<double>(nq * k, h->st);
      std::uint32_t* dperm = dalloc<std::uint32_t>(nq, h->st);
      GK_CUDA(cudaEventRecord(ev_alloc, h->st));
      GK_CUDA(cudaStreamWaitEvent(h->pst[0], ev_alloc, 0));
      GK_CUDA(cudaStreamWaitEvent(h->pst[1], ev_alloc, 0));
      GK_CUDA(cudaStreamWaitEvent(ost, ev_alloc, 0));
      int slot = 0;
      bool used[gk_bdl::kStageSlots] = {};
      // ring slot for the next transfer: wait until its previous transfer (and copy-out) finished
      struct Out { int slot; void* dst; std::size_t n; };
      std::vector<Out> pending;  // D2H blocks whose rows still have to reach the caller's memory
      auto drain_one = [&] {
        const Out o = pending.front();
        pending.erase(pending.begin());
        GK_CUDA(cudaEventSynchronize(h->stage_ev[o.slot]));
        host_copy(o.dst, h->stage[o.slot], o.n, nth);
      };
      auto take_slot = [&]() {
        const int s0 = slot;
        slot = (slot + 1) % gk_bdl::kStageSlots;
        for (std::size_t i = 0; i < pending.size(); ++i)
          if (pending[i].slot == s0) {  // its rows must leave the slot first (in order)
            while (!pending.empty() && pending.front().slot != s0) drain_one();
            drain_one();
            break;
          }
        if (used[s0]) GK_CUDA(cudaEventSynchronize(h->stage_ev[s0]));
        used[s0] = true;
        return s0;
      };
      auto h2d = [&](void* dst, const void* src, std::size_t n, bool pinned) {
        if (pinned) {
          GK_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, h->pst[0]));
          return;
        }
        for (std::size_t off = 0; off < n; off += gk_bdl::kStageBytes) {
          const std::size_t m = std::min(gk_bdl::kStageBytes, n - off);
          const int sl = take_slot();
          host_copy(h->stage[sl], static_cast<const char*>(src) + off, m, nth);
          GK_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, h->stage[sl], m, cudaMemcpyHostToDevice, h->pst[0]));
          GK_CUDA(cudaEventRecord(h->stage_ev[sl], h->pst[0]));
        }
      };
      auto d2h = [&](void* dst, const void* src, std::size_t n, bool pinned) {
        if (pinned) {
          GK_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, h->pst[1]));
          return;
        }
        for (std::size_t off = 0; off < n; off += gk_bdl::kStageBytes) {
          const std::size_t m = std::min(gk_bdl::kStageBytes, n - off);
          const int sl = take_slot();
          GK_CUDA(cudaMemcpyAsync(h->stage[sl], static_cast<const char*>(src) + off, m, cudaMemcpyDeviceToHost, h->pst[1]));
          GK_CUDA(cudaEventRecord(h->stage_ev[sl], h->pst[1]));
          pending.push_back({sl, static_cast<char*>(dst) + off, m});
          if (pending.size() >= gk_bdl::kStageSlots - 1) drain_one();
        }
      };
      // queries in, kNN_L of each chunk as soon as its queries landed
      for (std::uint64_t c = 0; c < nck; ++c) {
        const std::uint64_t off = bounds[c], m = bounds[c + 1] - off;
        h2d(dq + off * h->d, q + off * h->d, m * h->d * sizeof(double), pq);
        GK_CUDA(cudaEventRecord(h->pev[2 + 2 * c], h->pst[0]));
        GK_CUDA(cudaStreamWaitEvent(ost, h->pev[2 + 2 * c], 0));
        range_order(h->d, dq + off * h->d, m, dperm + off, ost);
        GK_CUDA(cudaEventRecord(ev_ord[c], ost));
        GK_CUDA(cudaStreamWaitEvent(h->st, ev_ord[c], 0));
        knn_traverse(h->d, k, ts, dq + off * h->d, dperm + off, m, di + off * k, dd + off * k, h->st);
        GK_CUDA(cudaEventRecord(h->pev[3 + 2 * c], h->st));
      }
      // rows out, chunk by chunk as they become final
      for (std::uint64_t c = 0; c < nck; ++c) {
        const std::uint64_t off = bounds[c], m = bounds[c + 1] - off;
        GK_CUDA(cudaStreamWaitEvent(h->pst[1], h->pev[3 + 2 * c], 0));
        d2h(ids + off * k, di + off * k, m * k * sizeof(std::uint32_t), pi);
        d2h(d2 + off * k, dd + off * k, m * k * sizeof(double), pd);
      }
      while (!pending.empty()) drain_one();
      GK_CUDA(cudaEventRecord(ev_done, h->pst[1]));
      GK_CUDA(cudaStreamWaitEvent(h->st, ev_done, 0));
      dfree(dq, h->st);
      dfree(di, h->st);
      dfree(dd, h->st);
      dfree(dperm, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
      return;
    }
    double* dq = dalloc<double>(nq * h->d, h->st);
    std::uint32_t* di = dalloc<std::uint32_t>(nq * k, h->st);
    double* dd = dalloc<double>(nq * k, h->st);
    GK_CUDA(cudaMemcpyAsync(dq, q, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    knn_device_impl(h, dq, nq, k, di, dd, nullptr);
    GK_CUDA(cudaMemcpyAsync(ids, di, nq * k * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, h->st));
    GK_CUDA(cudaMemcpyAsync(d2, dd, nq * k * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    dfree(dq, h->st);
    dfree(di, h->st);
    dfree(dd, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

// ------------------------------------------------------------ range search --
// Ball range search over the log structure.  Rows requested: one
// traversal writes each query's first kRangeSlots rows into fixed slots and counts them all;
// after the offset scan the slots are compacted into the CSR rows and only the queries with
// more rows than slots are traversed again (their rows straight to their offsets).  Counts
// only (or a slot buffer that would exceed kRangeSlotBytes): a count traversal.
constexpr unsigned kRangeSlots = 32;
constexpr std::uint64_t kRangeSlotBytes = 4ULL << 30;
static std::uint64_t range_device_impl(gk_bdl* h, const double* q_dev, std::uint64_t nq, double r2,
                                       unsigned long long* counts_dev, unsigned long long* offs_dev, std::uint32_t* ids_dev,
                                       double* d2_dev, std::uint64_t capacity, const double* r2q_dev = nullptr) {
  if (!r2q_dev) need(!std::isnan(r2) && r2 >= 0.0, "r2 must be a non-negative squared radius");
  if (nq >= 0x7fffffffULL) throw Error(GK_ERR_INVALID, "range batch larger than 2^31-1 queries");
  if (nq == 0) {
    if (offs_dev) GK_CUDA(cudaMemsetAsync(offs_dev, 0, 8, h->st));
    GK_CUDA(cudaStreamSynchronize(h->st));
    return 0;
  }
  const bool rows = offs_dev && (ids_dev || d2_dev);
  if (rows) need(ids_dev && d2_dev, "range rows need both ids and d2");
  const TreeSet ts = h->trees();
  Scratch tmp(h->st);
  unsigned long long* cnt = counts_dev ? counts_dev : tmp.take<unsigned long long>(nq + 1);
  GK_CUDA(cudaMemsetAsync(cnt, 0, (nq + (counts_dev ? 0 : 1)) * 8, h->st));
  std::uint32_t* perm = nullptr;
  std::uint32_t* ti = nullptr;
  double* td = nullptr;
  const bool slots = rows && nq * kRangeSlots * 12 <= kRangeSlotBytes;
  std::uint64_t total = 0;
  if (ts.count > 0) {
    perm = tmp.take<std::uint32_t>(nq);
    range_order(h->d, q_dev, nq, perm, h->st);
    if (slots) {
      ti = tmp.take<std::uint32_t>(nq * kRangeSlots);
      td = tmp.take<double>(nq * kRangeSlots);
      range_launch(h->d, ts, q_dev, nq, r2, r2q_dev, perm, cnt, nullptr, ti, td, 2, kRangeSlots, h->st);
    } else {
      range_launch(h->d, ts, q_dev, nq, r2, r2q_dev, perm, cnt, nullptr, nullptr, nullptr, 0, 0, h->st);
    }
  }
  if (offs_dev) {
    std::size_t tb = 0;
    GK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs_dev, nq + 1, h->st));
    GK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.take<char>(tb), tb, cnt, offs_dev, nq + 1, h->st));
    unsigned long long t = 0;
    GK_CUDA(cudaMemcpyAsync(&t, offs_dev + nq, 8, cudaMemcpyDeviceToHost, h->st));
    GK_CUDA(cudaStreamSynchronize(h->st));
    total = t;
    if (rows) {
      if (total > capacity)  // offsets are valid: the caller may size its buffers and call again
        throw Error(GK_ERR_CAPACITY, "range result (" + std::to_string(total) + " rows) exceeds the capacity (" +
                                         std::to_string(capacity) + ")");
      if (total > 0x7fffffffULL)  // the per-query row sort's limit, checked before any row is written
        throw Error(GK_ERR_UNSUPPORTED, "range result larger than 2^31-1 rows");
      if (total > 0) {
        if (slots) {
          std::uint32_t* ovf = tmp.take<std::uint32_t>(nq);
          const std::uint64_t no =
              range_slots_compact(nq, kRangeSlots, perm, cnt, offs_dev, ti, td, ids_dev, d2_dev, ovf, h->st);
          if (no) {  // the overflowing queries again (in K2 order), rows straight to their offsets, then sorted
            range_launch(h->d, ts, q_dev, no, r2, r2q_dev, ovf, nullptr, offs_dev, ids_dev, d2_dev, 1, 0, h->st);
            range_sort_ovf(ids_dev, d2_dev, total, offs_dev, ovf, no, h->st);
          }
        } else {
          range_launch(h->d, ts, q_dev, nq, r2, r2q_dev, perm, nullptr, offs_dev, ids_dev, d2_dev, 1, 0, h->st);
          range_sort(ids_dev, d2_dev, total, offs_dev, nq, h->st);
        }
      }
    }
  }
  GK_CUDA(cudaStreamSynchronize(h->st));
  return total;
}

int gk_bdl_range_count(gk_bdl* h, const double* q, uint64_t nq, double r2, uint64_t* counts) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (q && counts), "null buffer");
    need(!std::isnan(r2) && r2 >= 0.0, "r2 must be a non-negative squared radius");
    DevScope ds(h->device);
    if (nq == 0) return;
    double* dq = dalloc<double>(nq * h->d, h->st);
    unsigned long long* dc = dalloc<unsigned long long>(nq, h->st);
    GK_CUDA(cudaMemcpyAsync(dq, q, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    range_device_impl(h, dq, nq, r2, dc, nullptr, nullptr, nullptr, 0);
    GK_CUDA(cudaMemcpyAsync(counts, dc, nq * 8, cudaMemcpyDeviceToHost, h->st));
    dfree(dq, h->st);
    dfree(dc, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_range(gk_bdl* h, const double* q, uint64_t nq, double r2, uint64_t* offsets, uint32_t* ids, double* d2,
                 uint64_t capacity) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(offsets != nullptr && (nq == 0 || q), "null buffer");
    need(capacity == 0 || (ids && d2), "null row buffers");
    need(!std::isnan(r2) && r2 >= 0.0, "r2 must be a non-negative squared radius");
    DevScope ds(h->device);
    if (nq == 0) {
      offsets[0] = 0;
      return;
    }
    double* dq = dalloc<double>(nq * h->d, h->st);
    unsigned long long* doff = dalloc<unsigned long long>(nq + 1, h->st);
    std::uint32_t* di = dalloc<std::uint32_t>(std::max<std::uint64_t>(capacity, 1), h->st);
    double* dd = dalloc<double>(std::max<std::uint64_t>(capacity, 1), h->st);
    GK_CUDA(cudaMemcpyAsync(dq, q, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    auto release = [&] {
      dfree(dq, h->st);
      dfree(doff, h->st);
      dfree(di, h->st);
      dfree(dd, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
    };
    std::uint64_t total = 0;
    try {  // one count pass, one fill pass into the caller-sized row buffers
      total = range_device_impl(h, dq, nq, r2, nullptr, doff, di, dd, capacity);
    } catch (const Error& e) {
      if (e.code == GK_ERR_CAPACITY)  // offsets are final even when the rows do not fit
        cudaMemcpy(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost);
      release();
      throw;
    } catch (...) {
      release();
      throw;
    }
    GK_CUDA(cudaMemcpyAsync(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost, h->st));
    if (total) {
      GK_CUDA(cudaMemcpyAsync(ids, di, total * 4, cudaMemcpyDeviceToHost, h->st));
      GK_CUDA(cudaMemcpyAsync(d2, dd, total * 8, cudaMemcpyDeviceToHost, h->st));
    }
    release();
  });
}

int gk_bdl_range_device(gk_bdl* h, const double* q_dev, uint64_t nq, double r2, uint64_t* offsets_dev, uint32_t* ids_dev,
                        double* d2_dev, uint64_t capacity, uint64_t* total) {
  return guard([&] {
    need(h != nullptr && offsets_dev != nullptr, "null handle/offsets");
    need(nq == 0 || q_dev, "null queries");
    DevScope ds(h->device);
    const std::uint64_t t = range_device_impl(h, q_dev, nq, r2, nullptr, reinterpret_cast<unsigned long long*>(offsets_dev),
                                              ids_dev, d2_dev, capacity);
    if (total) *total = t;
  });
}

// Ball range search with one squared radius per query (ParGeo's range search is called per query point with
// its own radius): the same traversal, each lane's threshold read from r2[query].
static void check_radii(const double* r2, std::uint64_t nq) {
  for (std::uint64_t i = 0; i < nq; ++i)
    need(!std::isnan(r2[i]) && r2[i] >= 0.0, "r2[" + std::to_string(i) + "] must be a non-negative squared radius");
}

int gk_bdl_range_radii_count(gk_bdl* h, const double* q, uint64_t nq, const double* r2, uint64_t* counts) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (q && r2 && counts), "null buffer");
    check_radii(r2, nq);
    DevScope ds(h->device);
    if (nq == 0) return;
    double* dq = dalloc<double>(nq * h->d, h->st);
    double* dr = dalloc<double>(nq, h->st);
    unsigned long long* dc = dalloc<unsigned long long>(nq, h->st);
    GK_CUDA(cudaMemcpyAsync(dq, q, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    GK_CUDA(cudaMemcpyAsync(dr, r2, nq * sizeof(double), cudaMemcpyHostToDevice, h->st));
    range_device_impl(h, dq, nq, 0.0, dc, nullptr, nullptr, nullptr, 0, dr);
    GK_CUDA(cudaMemcpyAsync(counts, dc, nq * 8, cudaMemcpyDeviceToHost, h->st));
    dfree(dq, h->st);
    dfree(dr, h->st);
    dfree(dc, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_range_radii(gk_bdl* h, const double* q, uint64_t nq, const double* r2, uint64_t* offsets, uint32_t* ids,
                       double* d2, uint64_t capacity) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(offsets != nullptr && (nq == 0 || (q && r2)), "null buffer");
    need(capacity == 0 || (ids && d2), "null row buffers");
    check_radii(r2, nq);
    DevScope ds(h->device);
    if (nq == 0) {
      offsets[0] = 0;
      return;
    }
    double* dq = dalloc<double>(nq * h->d, h->st);
    double* dr = dalloc<double>(nq, h->st);
    unsigned long long* doff = dalloc<unsigned long long>(nq + 1, h->st);
    std::uint32_t* di = dalloc<std::uint32_t>(std::max<std::uint64_t>(capacity, 1), h->st);
    double* dd = dalloc<double>(std::max<std::uint64_t>(capacity, 1), h->st);
    GK_CUDA(cudaMemcpyAsync(dq, q, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    GK_CUDA(cudaMemcpyAsync(dr, r2, nq * sizeof(double), cudaMemcpyHostToDevice, h->st));
    auto release = [&] {
      dfree(dq, h->st);
      dfree(dr, h->st);
      dfree(doff, h->st);
      dfree(di, h->st);
      dfree(dd, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
    };
    std::uint64_t total = 0;
    try {
      total = range_device_impl(h, dq, nq, 0.0, nullptr, doff, di, dd, capacity, dr);
    } catch (const Error& e) {
      if (e.code == GK_ERR_CAPACITY)  // offsets are final even when the rows do not fit
        cudaMemcpy(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost);
      release();
      throw;
    } catch (...) {
      release();
      throw;
    }
    GK_CUDA(cudaMemcpyAsync(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost, h->st));
    if (total) {
      GK_CUDA(cudaMemcpyAsync(ids, di, total * 4, cudaMemcpyDeviceToHost, h->st));
      GK_CUDA(cudaMemcpyAsync(d2, dd, total * 8, cudaMemcpyDeviceToHost, h->st));
    }
    release();
  });
}

int gk_bdl_range_radii_device(gk_bdl* h, const double* q_dev, uint64_t nq, const double* r2_dev, uint64_t* offsets_dev,
                              uint32_t* ids_dev, double* d2_dev, uint64_t capacity, uint64_t* total) {
  return guard([&] {
    need(h != nullptr && offsets_dev != nullptr, "null handle/offsets");
    need(nq == 0 || (q_dev && r2_dev), "null queries/radii");
    DevScope ds(h->device);
    if (nq > 0) {
      int* bad = dalloc<int>(1, h->st);
      int hb = 0;
      GK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), h->st));
      k_check_radii<<<blocks_for(nq), 256, 0, h->st>>>(r2_dev, nq, bad);
      GK_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st));
      dfree(bad, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
      need(hb == 0, "every r2 must be a non-negative squared radius");
    }
    const std::uint64_t t = range_device_impl(h, q_dev, nq, 0.0, nullptr, reinterpret_cast<unsigned long long*>(offsets_dev),
                                              ids_dev, d2_dev, capacity, r2_dev);
    if (total) *total = t;
  });
}

// Orthogonal (box) range search: ids of the live points in the closed box [lo, hi], ascending.
static std::uint64_t range_box_device_impl(gk_bdl* h, const double* lo, const double* hi, std::uint64_t nq,
                                           unsigned long long* counts_dev, unsigned long long* offs_dev,
                                           std::uint32_t* ids_dev, std::uint64_t capacity) {
  if (nq >= 0x7fffffffULL) throw Error(GK_ERR_INVALID, "range batch larger than 2^31-1 queries");
  if (nq == 0) {
    if (offs_dev) GK_CUDA(cudaMemsetAsync(offs_dev, 0, 8, h->st));
    GK_CUDA(cudaStreamSynchronize(h->st));
    return 0;
  }
  const TreeSet ts = h->trees();
  unsigned long long* cnt = counts_dev ? counts_dev : dalloc<unsigned long long>(nq + 1, h->st);
  GK_CUDA(cudaMemsetAsync(cnt, 0, (nq + (counts_dev ? 0 : 1)) * 8, h->st));
  std::uint32_t* perm = nullptr;
  std::uint64_t total = 0;
  if (ts.count > 0) {
    perm = dalloc<std::uint32_t>(nq, h->st);
    range_box_order(h->d, lo, hi, nq, perm, h->st);
    range_box_launch(h->d, ts, lo, hi, nq, perm, cnt, nullptr, nullptr, false, h->st);
  }
  bool too_small = false;
  if (offs_dev) {
    std::size_t tb = 0;
    GK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs_dev, nq + 1, h->st));
    void* tmp = dalloc<char>(tb, h->st);
    GK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, offs_dev, nq + 1, h->st));
    dfree(tmp, h->st);
    unsigned long long t = 0;
    GK_CUDA(cudaMemcpyAsync(&t, offs_dev + nq, 8, cudaMemcpyDeviceToHost, h->st));
    GK_CUDA(cudaStreamSynchronize(h->st));
    total = t;
    if (ids_dev) {
      if (total > capacity) too_small = true;
      else if (total > 0) {
        range_box_launch(h->d, ts, lo, hi, nq, perm, nullptr, offs_dev, ids_dev, true, h->st);
        range_box_sort(ids_dev, total, offs_dev, nq, h->st);
      }
    }
  }
  if (perm) dfree(perm, h->st);
  if (!counts_dev) dfree(cnt, h->st);
  GK_CUDA(cudaStreamSynchronize(h->st));
  if (too_small)
    throw Error(GK_ERR_CAPACITY, "range result (" + std::to_string(total) + " rows) exceeds the capacity (" +
                                    std::to_string(capacity) + ")");
  return total;
}

int gk_bdl_range_box_count(gk_bdl* h, const double* lo, const double* hi, uint64_t nq, uint64_t* counts) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(nq == 0 || (lo && hi && counts), "null buffer");
    DevScope ds(h->device);
    if (nq == 0) return;
    double* dl = dalloc<double>(2 * nq * h->d, h->st);
    double* dh = dl + nq * h->d;
    unsigned long long* dc = dalloc<unsigned long long>(nq, h->st);
    GK_CUDA(cudaMemcpyAsync(dl, lo, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    GK_CUDA(cudaMemcpyAsync(dh, hi, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    range_box_device_impl(h, dl, dh, nq, dc, nullptr, nullptr, 0);
    GK_CUDA(cudaMemcpyAsync(counts, dc, nq * 8, cudaMemcpyDeviceToHost, h->st));
    dfree(dl, h->st);
    dfree(dc, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_range_box(gk_bdl* h, const double* lo, const double* hi, uint64_t nq, uint64_t* offsets, uint32_t* ids,
                     uint64_t capacity) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(offsets != nullptr && (nq == 0 || (lo && hi)), "null buffer");
    need(capacity == 0 || ids, "null row buffer");
    DevScope ds(h->device);
    if (nq == 0) {
      offsets[0] = 0;
      return;
    }
    double* dl = dalloc<double>(2 * nq * h->d, h->st);
    double* dh = dl + nq * h->d;
    unsigned long long* doff = dalloc<unsigned long long>(nq + 1, h->st);
    std::uint32_t* di = dalloc<std::uint32_t>(std::max<std::uint64_t>(capacity, 1), h->st);
    GK_CUDA(cudaMemcpyAsync(dl, lo, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    GK_CUDA(cudaMemcpyAsync(dh, hi, nq * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    auto release = [&] {
      dfree(dl, h->st);
      dfree(doff, h->st);
      dfree(di, h->st);
      GK_CUDA(cudaStreamSynchronize(h->st));
    };
    std::uint64_t total = 0;
    try {  // one count pass, one fill pass into the caller-sized row buffer
      total = range_box_device_impl(h, dl, dh, nq, nullptr, doff, di, capacity);
    } catch (const Error& e) {
      if (e.code == GK_ERR_CAPACITY)  // offsets are final even when the rows do not fit
        cudaMemcpy(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost);
      release();
      throw;
    } catch (...) {
      release();
      throw;
    }
    GK_CUDA(cudaMemcpyAsync(offsets, doff, (nq + 1) * 8, cudaMemcpyDeviceToHost, h->st));
    if (total) GK_CUDA(cudaMemcpyAsync(ids, di, total * 4, cudaMemcpyDeviceToHost, h->st));
    release();
  });
}

int gk_bdl_range_box_device(gk_bdl* h, const double* lo_dev, const double* hi_dev, uint64_t nq, uint64_t* offsets_dev,
                            uint32_t* ids_dev, uint64_t capacity, uint64_t* total) {
  return guard([&] {
    need(h != nullptr && offsets_dev != nullptr, "null handle/offsets");
    need(nq == 0 || (lo_dev && hi_dev), "null boxes");
    DevScope ds(h->device);
    const std::uint64_t t = range_box_device_impl(h, lo_dev, hi_dev, nq, nullptr,
                                                  reinterpret_cast<unsigned long long*>(offsets_dev), ids_dev, capacity);
    if (total) *total = t;
  });
}

// ---------------------------------------------------------------- kNN graph --
static void knn_graph_impl(gk_bdl* h, int k, std::uint32_t* row_ids_dev, std::uint32_t* ids_dev, double* d2_dev) {
  need(k >= 1, "k must be >= 1");
  if (k + 1 > GK_MAX_K) throw Error(GK_ERR_UNSUPPORTED, "kNN graph needs k + 1 <= " + std::to_string(GK_MAX_K));
  const std::uint64_t n = h->live_total();
  if (n == 0) return;
  const TreeSet ts = h->trees();
  knn_graph_launch(h->d, k, ts, n, row_ids_dev, ids_dev, d2_dev, h->st);
  GK_CUDA(cudaStreamSynchronize(h->st));
}

int gk_bdl_knn_graph_device(gk_bdl* h, int k, uint32_t* row_ids_dev, uint32_t* ids_dev, double* d2_dev) {
  return guard([&] {
    need(h != nullptr, "null handle");
    DevScope ds(h->device);
    need(h->live_total() == 0 || (row_ids_dev && ids_dev && d2_dev), "null buffer");
    knn_graph_impl(h, k, row_ids_dev, ids_dev, d2_dev);
  });
}

int gk_bdl_knn_graph(gk_bdl* h, int k, uint32_t* row_ids, uint32_t* ids, double* d2) {
  return guard([&] {
    need(h != nullptr, "null handle");
    DevScope ds(h->device);
    const std::uint64_t n = h->live_total();
    if (n == 0) return;
    need(row_ids && ids && d2, "null buffer");
    need(k >= 1, "k must be >= 1");
    std::uint32_t* dr = dalloc<std::uint32_t>(n, h->st);
    std::uint32_t* di = dalloc<std::uint32_t>(n * k, h->st);
    double* dd = dalloc<double>(n * k, h->st);
    knn_graph_impl(h, k, dr, di, dd);
    GK_CUDA(cudaMemcpyAsync(row_ids, dr, n * 4, cudaMemcpyDeviceToHost, h->st));
    GK_CUDA(cudaMemcpyAsync(ids, di, n * k * 4, cudaMemcpyDeviceToHost, h->st));
    GK_CUDA(cudaMemcpyAsync(d2, dd, n * k * 8, cudaMemcpyDeviceToHost, h->st));
    dfree(dr, h->st);
    dfree(di, h->st);
    dfree(dd, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_info_get(gk_bdl* h, gk_bdl_info* info) {
  return guard([&] {
    need(h != nullptr && info != nullptr, "null handle/info");
    std::memset(info, 0, sizeof(*info));
    info->F = h->F;
    info->buffer = h->buf_n;
    info->live = h->live_total();
    info->next_id = h->next_id;
    for (int i = 0; i < 64; ++i)
      if (h->F >> i & 1ULL) {
        info->build_size[i] = h->statics[i].build_size;
        info->live_per_tree[i] = h->statics[i].live;
        info->nodes_per_tree[i] = h->statics[i].n_nodes;
        info->height_per_tree[i] = h->statics[i].height;
        info->root_per_tree[i] = h->statics[i].root_slot;
      }
  });
}

int gk_bdl_tree_export(gk_bdl* h, int tree, gk_canon_node* nodes, uint32_t* ids, double* pts, uint64_t* n_nodes,
                       uint64_t* n_pts) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(tree >= -1 && tree < 64, "tree index out of range");
    DevScope ds(h->device);
    const DevTree* T = nullptr;
    if (tree < 0) T = &h->buf_tree;
    else {
      need(h->F >> tree & 1ULL, "static tree " + std::to_string(tree) + " does not exist");
      T = &h->statics[tree];
    }
    if (n_nodes) *n_nodes = T->n_nodes;
    if (n_pts) *n_pts = T->n;
    if (nodes && T->n_nodes)
      GK_CUDA(cudaMemcpyAsync(nodes, T->canon, T->n_nodes * sizeof(gk_canon_node), cudaMemcpyDeviceToHost, h->st));
    if (ids && T->n) GK_CUDA(cudaMemcpyAsync(ids, T->ids, T->n * 4, cudaMemcpyDeviceToHost, h->st));
    std::vector<double> soa;
    if (pts && T->n) {
      soa.resize(T->n * h->d);
      GK_CUDA(cudaMemcpyAsync(soa.data(), T->coords, soa.size() * 8, cudaMemcpyDeviceToHost, h->st));
    }
    GK_CUDA(cudaStreamSynchronize(h->st));
    if (pts)
      for (std::uint64_t i = 0; i < T->n; ++i)
        for (int j = 0; j < h->d; ++j) pts[i * h->d + j] = soa[j * T->n + i];
  });
}

int gk_bdl_bloom_query(gk_bdl* h, int tree, const double* pts, uint64_t n, uint8_t* may_contain) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(tree >= 0 && tree < 64 && (h->F >> tree & 1ULL), "static tree does not exist");
    need(n == 0 || (pts && may_contain), "null buffer");
    if (n == 0) return;
    DevScope ds(h->device);
    DevTree& T = h->statics[tree];
    h->ensure_bloom(T);
    double* dp = dalloc<double>(n * h->d, h->st);
    std::uint8_t* dm = dalloc<std::uint8_t>(n, h->st);
    GK_CUDA(cudaMemcpyAsync(dp, pts, n * h->d * sizeof(double), cudaMemcpyHostToDevice, h->st));
    k_bloom_query<<<blocks_for(n), 256, 0, h->st>>>(T.bloom, T.bloom_bits, dp, h->d, n, dm);
    GK_CHECK_LAUNCH();
    GK_CUDA(cudaMemcpyAsync(may_contain, dm, n, cudaMemcpyDeviceToHost, h->st));
    dfree(dp, h->st);
    dfree(dm, h->st);
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

void* gk_bdl_stream(gk_bdl* h) { return h ? static_cast<void*>(h->st) : nullptr; }

int gk_bdl_sync(gk_bdl* h) {
  return guard([&] {
    need(h != nullptr, "null handle");
    GK_CUDA(cudaStreamSynchronize(h->st));
  });
}

int gk_bdl_last_knn_ms(gk_bdl* h, float* traversal_ms, float* total_ms) {
  return guard([&] {
    need(h != nullptr, "null handle");
    if (traversal_ms) *traversal_ms = h->knn_ms;
    if (total_ms) *total_ms = h->knn_total_ms;
  });
}

int gk_bdl_last_build_ms(gk_bdl* h, float* build_ms, uint64_t* points_built) {
  return guard([&] {
    need(h != nullptr, "null handle");
    if (build_ms) *build_ms = h->build_ms;
    if (points_built) *points_built = h->built_pts;
  });
}

}  // extern "C"
