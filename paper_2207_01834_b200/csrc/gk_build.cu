// gk_build.cu — BuildvEB_S on the B200 (sm_100a): one persistent cooperative
// kernel per tree; every level of the build runs inside it, separated by
// grid-wide barriers, so no level ever returns to the host.
//
// Reference semantics (restated; the reference ships no code for it):
//   PAPER.md:1056-1093 Alg. 1 BuildvEB_S, 1110-1113 recursion, 1484-1487 spatial
//   median = (min+max)/2, 1491 leaf 16.
// Frozen decisions (mirrored by oracle/gk_oracle.cpp):
//   split dim = depth mod D; spatial split s = (lo+hi)/2, left x_c < s <= right;
//   stable partition; degenerate side or depth >= 40 or heuristic = object ->
//   object median by (x_c, id), left = the floor(n/2) smallest keys; leaf when
//   n <= leaf; vEB layout topology-driven (complete-tree vEB order restricted
//   to the nodes that exist).
//
// k_build<D> (cooperative, grid = co-resident blocks, sized to n) runs, for
// every level L (all nodes of the level at once):
//   A  per node:  chunk counts (<=1024-point chunks), bbox accumulators reset
//   -  grid scan: chunk offsets
//   B  per chunk (one warp): chunk->node, coalesced fp64 loads, warp min/max, one atomic per chunk
//   C  per node:  node record, leaf / spatial split / object flag
//   D  per chunk: left counts (ballot + popc) + per-node totals
//   E  per node:  degenerate spatial splits -> object median; internal flags
//   O  (object nodes only) 12 x 8-bit MSD radix select of the (x_c, id) median
//   -  grid scans: internal ranks (BFS child slots) and chunk left-count offsets
//   F  per node:  child records in left-to-right (BFS) order
//   G  per chunk: stable partition into the ping-pong buffer; finished leaves written in place
// then, per depth top-down, each node's vEB slot (cut frame of its depth,
// range propagation over the level arrays).  A second small kernel (after the
// host learns the exact node count) writes the canonical nodes and the
// traversal nodes (TNode) in vEB order.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "gk_common.cuh"

namespace cg = cooperative_groups;

#ifndef GK_BUILD_TIMELINE
#define GK_BUILD_TIMELINE 0  // 1: per-level device timestamps via printf (diagnostics)
#endif
#if GK_BUILD_TIMELINE
// stamps kept in thread 0's local memory and printed once at the end (printf inside the
// level loop would delay block 0 and inflate every later phase)
#define GK_PHASE_STAMP(id)                                                                     \
  do {                                                                                         \
    if (gtid == 0 && level < 32) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_st[level][id])); \
  } while (0)
#define GK_TL_PRINT(L0)                                                                                      \
  do {                                                                                                       \
    if (gtid == 0)                                                                                           \
      for (int L = (L0); L + 1 <= level && L < 32; ++L)                                                      \
        printf("[tl] n=%u grid=%u level %2d S=%7u: scan %6.1f  C+D %6.1f  E %6.1f  scan2 %6.1f  G %6.1f  total %6.1f us\n", \
               n, gridDim.x, L, tl_S[L], (tl_st[L][1] - tl_st[L][0]) * 1e-3, (tl_st[L][2] - tl_st[L][1]) * 1e-3,   \
               (tl_st[L][3] - tl_st[L][2]) * 1e-3, (tl_st[L][4] - tl_st[L][3]) * 1e-3,                        \
               (tl_st[L + 1][0] - tl_st[L][4]) * 1e-3, (tl_st[L + 1][0] - tl_st[L][0]) * 1e-3);              \
  } while (0)
#else
#define GK_PHASE_STAMP(name) do {} while (0)
#define GK_TL_PRINT(L0) do {} while (0)
#endif

namespace gk {
namespace {

// F_SMALL: a node of at most a.Tsmall points (more than a leaf) whose whole subtree the bottom phase
// (k_subtree) builds inside one block; the level loop treats it like a leaf
constexpr std::uint8_t F_LEAF = 1, F_OBJECT = 2, F_SMALL = 4;
constexpr int kThreads = 256;
constexpr int kSelCap = 4096;  // object nodes per radix-select batch
constexpr int kMaxLevels = 256;
#ifndef GK_CHUNKS_PER_WARP
#define GK_CHUNKS_PER_WARP 4
#endif
constexpr std::uint64_t kChunksPerWarp = GK_CHUNKS_PER_WARP;
// partition lane groups at sparse levels: 16-lane groups from this many chunks per warp, 8-lane from
#ifndef GK_GROUP16_CHUNKS
#define GK_GROUP16_CHUNKS 20
#endif
#ifndef GK_GROUP8_CHUNKS
#define GK_GROUP8_CHUNKS 40
#endif
#ifndef GK_GROUP4_CHUNKS
#define GK_GROUP4_CHUNKS 80
#endif
constexpr std::uint32_t kGroup16Chunks = GK_GROUP16_CHUNKS, kGroup8Chunks = GK_GROUP8_CHUNKS,
                        kGroup4Chunks = GK_GROUP4_CHUNKS;

__host__ __device__ inline std::uint64_t hyperceiling_u(std::uint64_t x) {
  std::uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct NodeArrays {
  std::uint32_t *start, *count, *parent, *cbase, *nleft, *pos, *thr_id;
  std::uint8_t *flags, *level;
  double *split, *lo, *hi;
};

struct SelState {
  unsigned long long hi;  // known high digits of dkey(x_c)
  std::uint32_t lo;       // known digits of the id
  std::uint32_t rank;     // rank still to skip inside the current prefix bucket
};

// control words (device)
enum Ctrl { C_S = 0, C_NOBJ = 1, C_H = 2, C_N = 3, C_LEVEL = 4, C_NSMALL = 5, C_SUBCTR = 6, C_WORK = 7, C_NCHUNKS = 8, C_COUNT = 9 };
constexpr int kSubLevels = 64;  // local levels of a bottom-phase subtree (<= kDepthCap + 12 + 1)
constexpr int kVLevels = 160;
// trees up to this size use the bottom phase by default: every tree at D <= 4 (measured on the B200, bottom
// phase on / off: C1 Insert_L 1.23 / 1.51 ms, C4's ten Insert_L 20.0 / 20.4 ms, C2 5.64 / 5.93 ms once k_subtree's
// warp min/max went through REDUX, C5 Insert_L 1.86 / 1.82 G points/s); at D >= 5 (subtrees of <= 256 points) it
// lost 5 % on C3; GK_SMALL_MAX_N overrides
template <int D>
constexpr std::uint64_t small_max_n() { return D <= 4 ? (1ull << 32) : 0; }   // absolute levels a merge spans (small roots at depths <= ~72, + kSubLevels)

struct BuildArgs {
  int leaf, heuristic;
  std::uint32_t n;
  std::uint32_t kc;  // points per chunk
  const double* src;
  std::uint64_t src_stride;
  const std::uint32_t* src_ids;
  double *bufA, *bufB;
  std::uint32_t *idsA, *idsB;
  double* out;
  std::uint32_t* out_ids;
  NodeArrays na;
  std::uint32_t* lvl_off;   // [kMaxLevels + 2]
  std::uint32_t* ctrl;      // [C_COUNT]
  // chunk_off / chunk_node: a level's chunk offsets per node and chunk -> node map, ping-pong by level parity
  // (the parent level's F writes them while its G still reads its own); ccnt / coff: chunks of a node's
  // children and their exclusive scan
  std::uint32_t *chunk_off[2], *chunk_node[2], *ccnt, *coff, *chunk_left, *left_scan, *is_int, *irank, *obj_list;
  unsigned long long* keys;
  SelState* sel;
  std::uint32_t* hist;      // [kSelCap * 256]
  std::uint32_t* bsum;      // [3 * gridDim + 2]
  std::uint32_t* int_by_slot;  // [cap + 1]
  std::uint32_t* irank_slot;   // [cap + 1] slot -> internal rank (k_emit copies it into the tree)
  // bottom phase (k_subtree + k_merge): subtrees of nodes with leaf < count <= Tsmall, one block each
  std::uint32_t Tsmall;        // 0: off (object-median heuristic, leaf < 4, or a tree that fits no block)
  std::uint32_t rmax;          // capacity of the small-root arrays
  std::uint32_t* small_list;   // [rmax] level-array index of every small root (unordered)
  std::uint32_t* sub_base;     // [rmax] first record of the subtree's node region
  std::uint32_t* sub_cnt;      // [rmax * kSubLevels] nodes per local level (level 0 = the root)
  std::uint32_t* sub_nlev;     // [rmax] local levels
  std::uint32_t *s_start, *s_count, *s_child;  // sub-node records, [2n] (a region of 2 * count per subtree);
                                               // s_child: an internal record's first child record
  std::uint8_t* s_flags;
  double *s_split, *s_lo, *s_hi;
  std::uint32_t *marks, *mscan;  // [n + 1] small-root starts marked / scanned (roots in start order)
  std::uint32_t* order;          // [rmax] small roots in start order
  std::uint32_t* V;              // [vcap + 1] per (level, root) node counts, scanned in place
  std::uint32_t vcap;
  std::uint32_t* new_off;        // [kMaxLevels + 2] merged level offsets
  NodeArrays na2;                // merged level arrays (copied back into na)
};

// ------------------------------------------------------------ block helpers --
__device__ __forceinline__ std::uint32_t block_sum(std::uint32_t v, std::uint32_t* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  std::uint32_t t = 0;
  for (int i = 0; i < (kThreads >> 5); ++i) t += sh[i];
  return t;
}

__device__ __forceinline__ void sync_all(cg::grid_group& grid) {
  if (gridDim.x == 1) {  // small trees build in one block: a block barrier is enough
    __syncthreads();
    return;
  }
  grid.sync();  // gpu-scope ordering; every cross-block read below goes through L2 (__ldcg), never a stale L1 line
}

// Grid-wide exclusive scans, split in two halves around one grid barrier: every block
// sums its segment (scan_partial -> bsum[b]), then every block scans its segment from
// the prefix of the other blocks' sums (scan_finish).  Several arrays share one barrier.
__device__ void scan_partial(const std::uint32_t* in, std::uint32_t n, std::uint32_t* bsum, std::uint32_t* sh) {
  const std::uint32_t G = gridDim.x, b = blockIdx.x;
  const std::uint32_t seg = (n + G - 1) / G;
  const std::uint32_t lo = min(n, b * seg), hi = min(n, lo + seg);
  std::uint32_t s = 0;
  for (std::uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += __ldcg(&in[i]);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) bsum[b] = s;
}

// map != nullptr: also writes map[c] = i for c in [out[i], out[i] + in[i]) (chunk -> node)
__device__ void scan_finish(const std::uint32_t* in, std::uint32_t* out, std::uint32_t n, const std::uint32_t* bsum,
                            std::uint32_t* sh, std::uint32_t* map = nullptr) {
  const std::uint32_t G = gridDim.x, b = blockIdx.x;
  const std::uint32_t seg = (n + G - 1) / G;
  const std::uint32_t lo = min(n, b * seg), hi = min(n, lo + seg);
  std::uint32_t o = 0;
  for (std::uint32_t i = threadIdx.x; i < b; i += blockDim.x) o += __ldcg(&bsum[i]);
  o = block_sum(o, sh);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  std::uint32_t carry = o;
  for (std::uint32_t base = lo; base < hi; base += blockDim.x) {
    const std::uint32_t i = base + threadIdx.x;
    const std::uint32_t v = i < hi ? __ldcg(&in[i]) : 0u;
    std::uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    __syncthreads();
    if (lane == 31) sh[w] = x;
    __syncthreads();
    std::uint32_t wpre = 0, tot = 0;
    for (int j = 0; j < (kThreads >> 5); ++j) {
      const std::uint32_t t = sh[j];
      if (j < w) wpre += t;
      tot += t;
    }
    if (i < hi) {
      const std::uint32_t e = carry + wpre + x - v;
      out[i] = e;
      if (map)
        for (std::uint32_t c = e; c < e + v; ++c) map[c] = i;
    }
    carry += tot;
  }
}

// exclusive scan of in[0, n) into out, all blocks of the grid (one grid barrier inside)
__device__ void grid_scan(cg::grid_group& grid, const std::uint32_t* in, std::uint32_t* out, std::uint32_t n,
                          std::uint32_t* bsum, std::uint32_t* sh, std::uint32_t* map = nullptr) {
  scan_partial(in, n, bsum, sh);
  sync_all(grid);
  scan_finish(in, out, n, bsum, sh, map);
}

// ---- vEB slots, top-down, over complete level arrays (lvl_off[0..H]).  Depth d is the cut depth of
// exactly one frame (d0, l) of the recursion; its root r is d's ancestor at depth d0, and
// pos(v) = pos(r) + |top part of the frame| + sizes of the bottom subtrees left of v's, all
// restricted to the frame's levels (range propagation).  Writes ctrl[C_H] / ctrl[C_N] and the
// slot -> internal flags, scanned into TNode indices (a.irank_slot) at the end.
__device__ void veb_phase(cg::grid_group& grid, const BuildArgs& a, const NodeArrays& na, std::uint32_t* lvl_off, int H,
                          std::uint32_t* sh) {
  const std::uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const std::uint32_t gthreads = gridDim.x * blockDim.x;
  const std::uint32_t N = __ldcg(&lvl_off[H]);
  if (gtid == 0) {
    lvl_off[H + 1] = N;
    a.ctrl[C_H] = static_cast<std::uint32_t>(H);
    a.ctrl[C_N] = N;
    na.pos[0] = 0;
  }
  sync_all(grid);
  for (int d = 1; d < H; ++d) {
    int d0 = 0, l = H;  // locate the frame whose cut is at depth d
    while (true) {
      const int lb = static_cast<int>(hyperceiling_u(static_cast<std::uint64_t>((l + 1) / 2)));
      const int lt = l - lb;
      if (d == d0 + lt) break;
      if (d < d0 + lt) l = lt;
      else { d0 += lt; l = lb; }
    }
    const std::uint32_t off = __ldcg(&lvl_off[d]), S = __ldcg(&lvl_off[d + 1]) - off;
    for (std::uint32_t v = gtid; v < S; v += gthreads) {
      const std::uint32_t g = off + v;
      std::uint32_t r = g;
      for (int e = d; e > d0; --e) r = __ldcg(&na.parent[r]);
      auto child_idx = [&](std::uint32_t x, int e) -> std::uint32_t {
        return (x < __ldcg(&lvl_off[e + 1])) ? __ldcg(&na.cbase[x]) : __ldcg(&lvl_off[e + 2]);
      };
      std::uint32_t lo = r, hi = r + 1, top = 0;
      for (int e = d0; e < d; ++e) {
        top += hi - lo;
        lo = child_idx(lo, e);
        hi = child_idx(hi, e);
      }
      std::uint32_t x = g, y = lo, left = 0;
      for (int e = d; e < d0 + l; ++e) {
        left += x - y;
        if (e + 1 < d0 + l) {
          x = child_idx(x, e);
          y = child_idx(y, e);
        }
      }
      na.pos[g] = __ldcg(&na.pos[r]) + top + left;
    }
    sync_all(grid);
  }
  // slot -> internal flag
  for (std::uint32_t g = gtid; g <= N; g += gthreads) {
    if (g == N) a.int_by_slot[N] = 0;
    else a.int_by_slot[__ldcg(&na.pos[g])] = (__ldcg(&na.flags[g]) & F_LEAF) ? 0u : 1u;
  }
  // ... scanned into internal ranks (= TNode indices) here, in the same launch (a cooperative k_slot_rank
  // launch after the host learned N used to do it: ~25 us on every tree's critical path)
  sync_all(grid);
  grid_scan(grid, a.int_by_slot, a.irank_slot, N + 1, a.bsum, sh);
}

// -------------------------------------------------------------- the build --
#ifndef GK_BUILD_MINB
#define GK_BUILD_MINB 4  // D <= 4: 64 registers, 4 blocks per SM (C2 build -4 % vs 80 registers)
#endif
// PH = 0: the dense top levels; the kernel hands over to PH = 1 (same grid, next launch on the
// stream) at the first sparse level, so that the lane-group partition of the sparse levels does
// not cost the dense levels registers.  PH = 1 resumes at ctrl[C_LEVEL] (or returns at once when
// PH = 0 finished the whole build) and runs the remaining levels and the vEB phase.
template <int D, int PH>
#ifndef GK_BUILD_MINB_HI
#define GK_BUILD_MINB_HI 0  // D >= 5: min blocks per SM for ptxas (0: none)
#endif
__global__ void __launch_bounds__(kThreads, (D <= 4 ? GK_BUILD_MINB : GK_BUILD_MINB_HI)) k_build(const BuildArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ std::uint32_t sh[32];
  const NodeArrays& na = a.na;
  const std::uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const std::uint32_t gthreads = gridDim.x * blockDim.x;
  const std::uint32_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const std::uint32_t n = a.n;
  const std::uint32_t kc = a.kc;  // points per chunk (the warp work item), sized to the grid
  // D <= 4: children's boxes accumulate during the parent's partition (G), so only the root
  // level runs the box pass B.  At D >= 5 the 4D extra accumulators cost more occupancy than
  // the saved pass (C3 build +13 %).
  constexpr bool kChildBoxes = D <= 4;
  // lane-group partition at sparse levels (PH = 1) for D <= 4 (C2 build -8 %); at D >= 5 it lost (C3 +4 %)
  constexpr bool kGroupedSparse = D <= 4;
  // partition rounds per loop trip whose loads are in flight together: 2 at D >= 5 (C3 build
  // -20 %), 1 at D <= 4, where the 64-register budget has no room for a second round
#ifdef GK_PART_UNROLL
  constexpr int kPartUnroll = GK_PART_UNROLL;
#else
  constexpr int kPartUnroll = D >= 5 ? 2 : 1;
#endif

  const double* cur = a.src;
  const std::uint32_t* cur_ids = a.src_ids;
  std::uint64_t cur_stride = a.src_stride;
  double* nxt = a.bufA;
  std::uint32_t* nxt_ids = a.idsA;
  int level = 0;

  if (PH == 1) {
    const std::uint32_t l0 = __ldcg(&a.ctrl[C_LEVEL]);
    if (l0 == 0xffffffffu) return;  // PH = 0 built the whole tree
    level = static_cast<int>(l0);
    if (level > 0) {  // ping-pong state at the start of `level` (level 1 reads bufA)
      const bool odd = (level & 1) != 0;
      cur = odd ? a.bufA : a.bufB;
      cur_ids = odd ? a.idsA : a.idsB;
      cur_stride = n;
      nxt = odd ? a.bufB : a.bufA;
      nxt_ids = odd ? a.idsB : a.idsA;
    }
  } else if (gtid == 0) {
    na.start[0] = 0; na.count[0] = n; na.parent[0] = 0xffffffffu;
    na.nleft[0] = 0;
    a.lvl_off[0] = 0;
    a.ctrl[C_S] = 1;
    a.ctrl[C_NOBJ] = 0;
    a.chunk_off[0][0] = 0;  // the root's chunks (deeper levels' offsets and maps are written by the parent level's F)
    a.chunk_off[0][1] = (n + kc - 1) / kc;
    a.ctrl[C_NCHUNKS] = (n + kc - 1) / kc;
    a.ctrl[C_LEVEL] = 0xffffffffu;
    a.ctrl[C_NSMALL] = 0;
    a.ctrl[C_SUBCTR] = 0;
    a.ctrl[C_WORK] = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      a.keys[j * 2] = ~0ULL;
      a.keys[j * 2 + 1] = 0ULL;
    }
  }
  if (PH == 0) {
    for (std::uint32_t c = gtid; c < (n + kc - 1) / kc; c += gthreads) a.chunk_node[0][c] = 0;
    sync_all(grid);
  }
  [[maybe_unused]] const int level0 = level;
#if GK_BUILD_TIMELINE
  unsigned long long tl_st[33][5];
  std::uint32_t tl_S[33];
#endif
  for (;; ++level) {
    const std::uint32_t S = __ldcg(&a.ctrl[C_S]);
#if GK_BUILD_TIMELINE
    if (gtid == 0 && level < 33) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_st[level][0]));
      tl_S[level] = S;
    }
#endif
    if (S == 0 || level >= kMaxLevels) break;
    const std::uint32_t off = __ldcg(&a.lvl_off[level]);
    const int cdim = level % D;
    const bool box_pass = level == 0 || !kChildBoxes;  // else the parent's G accumulated the boxes
    const bool spatial_level = a.heuristic != GK_OBJECT_MEDIAN && level < kDepthCap;

    // this level's chunk offsets and chunk -> node map: written by the parent level's F (level 0: at
    // the start), so a level costs four grid barriers: C+D | E + scan partials | scan finish | F+G
    const std::uint32_t* chunk_off = a.chunk_off[level & 1];
    const std::uint32_t* chunk_node = a.chunk_node[level & 1];
    std::uint32_t* chunk_off_nx = a.chunk_off[(level & 1) ^ 1];
    std::uint32_t* chunk_node_nx = a.chunk_node[(level & 1) ^ 1];
    GK_PHASE_STAMP(1);
    const std::uint32_t nchunks = __ldcg(&a.ctrl[C_NCHUNKS]);
    // Sparse levels (many small chunks per warp): the partition runs in lane groups (PH = 1)
    const std::uint32_t cpw = nchunks / nwarps;
    if (PH == 0 && kGroupedSparse && cpw >= kGroup16Chunks) {
      if (gtid == 0) a.ctrl[C_LEVEL] = static_cast<std::uint32_t>(level);  // PH = 1 resumes here
      GK_TL_PRINT(level0);
      return;
    }
    // A warp takes a contiguous run of chunks: consecutive chunks mostly belong to one node, so the per-node
    // accumulators (left counts, bounding boxes) stay in registers across them and reach the node's words with
    // one atomic per run instead of one per chunk (at the top levels every chunk of the grid hit the same few
    // addresses: 4096 same-address atomics cost ~12 us of a 25 us partition phase on a 512K-point tree)
    // (runs only where chunks are even -- few partial chunks, i.e. large nodes: with nodes of mixed sizes a
    // run of full chunks next to a run of tiny ones would unbalance the warps, C5 Insert_L -8 %; there the
    // chunks go round-robin as before)
    const std::uint32_t cq = (nchunks + nwarps - 1) / nwarps;
    const bool runs = nchunks <= n / kc + n / kc / 4 + 8;
    const std::uint32_t cfirst = runs ? min(nchunks, gwarp * cq) : gwarp;
    const std::uint32_t cstep = runs ? 1u : nwarps;
    const std::uint32_t cend = runs ? min(nchunks, cfirst + cq) : nchunks;

    // C: node records and split decisions (needs the final boxes)
    auto node_records = [&]() {
      for (std::uint32_t v = gtid; v < S; v += gthreads) {
        const std::uint32_t g = off + v;
        double lo[D], hi[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          lo[j] = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + j) * 2]));
          hi[j] = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + j) * 2 + 1]));
          na.lo[static_cast<std::uint64_t>(g) * D + j] = lo[j];
          na.hi[static_cast<std::uint64_t>(g) * D + j] = hi[j];
        }
        na.level[g] = static_cast<std::uint8_t>(level);
        const std::uint32_t cnt_g = __ldcg(&na.count[g]);
        if (cnt_g <= static_cast<std::uint32_t>(a.leaf)) {
          na.flags[g] = F_LEAF;
          na.split[g] = 0.0;
        } else if (cnt_g <= a.Tsmall) {
          na.flags[g] = F_SMALL;
          na.split[g] = 0.0;
        } else if (!spatial_level) {
          na.flags[g] = F_OBJECT;
          na.split[g] = 0.0;
        } else {
          na.flags[g] = 0;
          double l = lo[0], h = hi[0];
#pragma unroll
          for (int j = 1; j < D; ++j)
            if (cdim == j) { l = lo[j]; h = hi[j]; }
          na.split[g] = __dmul_rn(__dadd_rn(l, h), 0.5);  // (lo + hi) / 2 exactly
        }
      }
    };

    if (box_pass) {
      // B: per run of chunks of one node: bounding box
      {
        double mn[D], mx[D];
        std::uint32_t acc_v = 0xffffffffu;
        auto reset = [&]() {
#pragma unroll
          for (int j = 0; j < D; ++j) { mn[j] = __longlong_as_double(0x7ff0000000000000LL); mx[j] = -mn[j]; }
        };
        auto flush = [&]() {
          if (acc_v == 0xffffffffu) return;
#pragma unroll
          for (int j = 0; j < D; ++j) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              mn[j] = fmin(mn[j], __shfl_xor_sync(0xffffffffu, mn[j], o));
              mx[j] = fmax(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], o));
            }
          }
          if (lane < D) {
            double l = mn[0], h = mx[0];
#pragma unroll
            for (int j = 1; j < D; ++j)
              if (lane == j) { l = mn[j]; h = mx[j]; }
            unsigned long long* kk = a.keys + (static_cast<std::uint64_t>(acc_v) * D + lane) * 2;
            atomicMin(kk, dkey(l));
            atomicMax(kk + 1, dkey(h));
          }
        };
        reset();
        std::uint32_t vn = cfirst < cend ? __ldcg(&chunk_node[cfirst]) : 0u, s0 = 0, cnt = 0, coff_v = 0;
        for (std::uint32_t c = cfirst; c < cend; c += cstep) {
          const std::uint32_t v = vn;
          if (c + cstep < cend) vn = __ldcg(&chunk_node[c + cstep]);
          if (v != acc_v) {  // the node's words once per run of its chunks
            flush();
            reset();
            acc_v = v;
            s0 = __ldcg(&na.start[off + v]);
            cnt = __ldcg(&na.count[off + v]);
            coff_v = __ldcg(&chunk_off[v]);
          }
          const std::uint32_t first = s0 + (c - coff_v) * kc;
          const std::uint32_t end = min(first + kc, s0 + cnt);
          constexpr int UB = 2;  // rounds whose loads are in flight together (the pass is latency-bound)
          for (std::uint32_t i0 = first + lane; i0 < end; i0 += 32 * UB) {
            double x[UB][D];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              const std::uint32_t i = i0 + 32 * u;
#pragma unroll
              for (int j = 0; j < D; ++j)  // NaN past the end: fmin / fmax keep the other operand
                x[u][j] = i < end ? __ldcg(&cur[j * cur_stride + i]) : __longlong_as_double(0x7ff8000000000000LL);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u)
#pragma unroll
              for (int j = 0; j < D; ++j) {
                mn[j] = fmin(mn[j], x[u][j]);
                mx[j] = fmax(mx[j], x[u][j]);
              }
          }
        }
        flush();
      }
      sync_all(grid);
      node_records();
    } else {
      node_records();
    }

    // Sparse levels (>= 64 chunks per warp, chunks of a few dozen points): the count pass runs
    // one lane per chunk, 32 chunks of a warp side by side, instead of a warp walking them one
    // after another (the partition keeps a warp per chunk: lane-private stores do not coalesce)
    const bool lane_mode = nchunks >= 64u * nwarps;

    // D: spatial left counts per chunk (x_c < s); the split is re-derived from the box exactly as C does
    if (lane_mode) {
      for (std::uint32_t c = gwarp * 32 + lane; c < ((nchunks + 31) & ~31u); c += nwarps * 32) {
        if (c >= nchunks) continue;
        const std::uint32_t v = __ldcg(&chunk_node[c]), g = off + v;
        const std::uint32_t s0 = __ldcg(&na.start[g]), nn = __ldcg(&na.count[g]);
        std::uint32_t cnt = 0;
        if (spatial_level && nn > static_cast<std::uint32_t>(a.leaf) && nn > a.Tsmall) {
          const std::uint32_t first = s0 + (c - __ldcg(&chunk_off[v])) * kc;
          const std::uint32_t end = min(first + kc, s0 + nn);
          const double l = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + cdim) * 2]));
          const double h = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + cdim) * 2 + 1]));
          const double s = __dmul_rn(__dadd_rn(l, h), 0.5);
          const double* xc = cur + cdim * cur_stride;
#pragma unroll 4
          for (std::uint32_t i = first; i < end; ++i) cnt += __ldcg(&xc[i]) < s ? 1u : 0u;
          if (cnt) atomicAdd(&na.nleft[g], cnt);
        }
        a.chunk_left[c] = cnt;
      }
    } else {
    std::uint32_t acc = 0, acc_g = 0;  // left count of the run's current node
    std::uint32_t vn = cfirst < cend ? __ldcg(&chunk_node[cfirst]) : 0u, cur_v = 0xffffffffu;
    std::uint32_t g = 0, s0 = 0, nn = 0, coff_v = 0;
    bool counted = false;
    double s = 0.0;
    for (std::uint32_t c = cfirst; c < cend; c += cstep) {
      const std::uint32_t v = vn;
      if (c + cstep < cend) vn = __ldcg(&chunk_node[c + cstep]);
      if (v != cur_v) {  // the node's words once per run of its chunks
        cur_v = v;
        g = off + v;
        s0 = __ldcg(&na.start[g]);
        nn = __ldcg(&na.count[g]);
        coff_v = __ldcg(&chunk_off[v]);
        counted = spatial_level && nn > static_cast<std::uint32_t>(a.leaf) && nn > a.Tsmall;
        if (counted) {
          const double l = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + cdim) * 2]));
          const double h = dkey_inv(__ldcg(&a.keys[(static_cast<std::uint64_t>(v) * D + cdim) * 2 + 1]));
          s = __dmul_rn(__dadd_rn(l, h), 0.5);
        }
      }
      std::uint32_t cnt = 0;
      if (counted) {
        const std::uint32_t first = s0 + (c - coff_v) * kc;
        const std::uint32_t end = min(first + kc, s0 + nn);
        const double* xc = cur + cdim * cur_stride;
        constexpr int U = 4;  // loads of U rounds in flight before their ballots (memory-level parallelism)
        for (std::uint32_t i0 = first; i0 < end; i0 += 32 * U) {
          double x[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const std::uint32_t i = i0 + 32 * u + lane;
            x[u] = i < end ? __ldcg(&xc[i]) : s;  // s: never counted
          }
#pragma unroll
          for (int u = 0; u < U; ++u) cnt += __popc(__ballot_sync(0xffffffffu, x[u] < s));
        }
      }
      if (g != acc_g) {
        if (lane == 0 && acc) atomicAdd(&na.nleft[acc_g], acc);
        acc = 0;
        acc_g = g;
      }
      acc += cnt;
      if (lane == 0) a.chunk_left[c] = cnt;
    }
    if (lane == 0 && acc) atomicAdd(&na.nleft[acc_g], acc);
    }
    if (gtid == 0) a.chunk_left[nchunks] = 0;
    sync_all(grid);
    GK_PHASE_STAMP(2);

    // E: degenerate spatial splits -> object median; internal flags; reset the next
    // level's box accumulators (this level's were consumed by C and D)
    // (each block on its own scan segment of [0, S], so that the scans' block sums follow after a block barrier)
    const std::uint32_t e_seg = (S + 1 + gridDim.x - 1) / gridDim.x;
    const std::uint32_t e_lo = min(S + 1, blockIdx.x * e_seg), e_hi = min(S + 1, e_lo + e_seg);
    for (std::uint32_t v = e_lo + threadIdx.x; v < e_hi; v += blockDim.x) {
      a.ccnt[v] = 0;
      if (v == S) { a.is_int[S] = 0; continue; }
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const std::uint64_t u = 2ULL * v + cc;
        if (u < n) {
#pragma unroll
          for (int j = 0; j < D; ++j) {
            a.keys[(u * D + j) * 2] = ~0ULL;
            a.keys[(u * D + j) * 2 + 1] = 0ULL;
          }
        }
      }
      const std::uint32_t g = off + v;
      std::uint8_t fl = __ldcg(&na.flags[g]);
      if (fl & (F_LEAF | F_SMALL)) {
        a.is_int[v] = 0;
        if (fl & F_SMALL) a.small_list[atomicAdd(&a.ctrl[C_NSMALL], 1u)] = g;  // the bottom phase builds it
        continue;
      }
      a.is_int[v] = 1;
      const std::uint32_t cnt = __ldcg(&na.count[g]);
      std::uint32_t nl = __ldcg(&na.nleft[g]);
      if (!(fl & F_OBJECT)) {
        if (nl == 0 || nl == cnt) { fl |= F_OBJECT; na.flags[g] = fl; }
      }
      if (fl & F_OBJECT) {
        const std::uint32_t o = atomicAdd(&a.ctrl[C_NOBJ], 1u);
        a.obj_list[o] = g;
        nl = cnt / 2;
        na.nleft[g] = nl;
        na.pos[g] = o;  // temporary: object index (pos is recomputed by the vEB phase)
      }
      a.ccnt[v] = (nl + kc - 1) / kc + (cnt - nl + kc - 1) / kc;  // the children's chunks
    }
    __syncthreads();
    // block sums of the three scans: BFS child slots, the children's chunk offsets, chunk left counts
    scan_partial(a.is_int, S + 1, a.bsum, sh);
    scan_partial(a.ccnt, S + 1, a.bsum + 2 * gridDim.x, sh);
    scan_partial(a.chunk_left, nchunks + 1, a.bsum + gridDim.x, sh);
    sync_all(grid);
    GK_PHASE_STAMP(3);

    // O: object-median radix select (batches of kSelCap object nodes)
    const std::uint32_t nobj = __ldcg(&a.ctrl[C_NOBJ]);
    for (std::uint32_t b0 = 0; b0 < nobj; b0 += kSelCap) {
      const std::uint32_t nb = min(static_cast<std::uint32_t>(kSelCap), nobj - b0);
      for (std::uint32_t o = gtid; o < nb * 256; o += gthreads) a.hist[o] = 0;
      for (std::uint32_t o = gtid; o < nb; o += gthreads) {
        a.sel[o].hi = 0;
        a.sel[o].lo = 0;
        a.sel[o].rank = __ldcg(&na.count[__ldcg(&a.obj_list[b0 + o])]) / 2;
      }
      sync_all(grid);
      for (int p = 0; p < 12; ++p) {
        for (std::uint32_t c = gwarp; c < nchunks; c += nwarps) {
          const std::uint32_t v = __ldcg(&chunk_node[c]), g = off + v;
          if ((__ldcg(&na.flags[g]) & (F_LEAF | F_OBJECT)) != F_OBJECT) continue;
          const std::uint32_t o = __ldcg(&na.pos[g]);
          if (o < b0 || o >= b0 + nb) continue;
          SelState s;
          s.hi = __ldcg(&a.sel[o - b0].hi);
          s.lo = __ldcg(&a.sel[o - b0].lo);
          const std::uint32_t s0 = __ldcg(&na.start[g]), nn = __ldcg(&na.count[g]);
          const std::uint32_t first = s0 + (c - __ldcg(&chunk_off[v])) * kc;
          const std::uint32_t end = min(first + kc, s0 + nn);
          for (std::uint32_t i0 = first; i0 < end; i0 += 32) {
            const std::uint32_t i = i0 + lane;
            int digit = -1;
            if (i < end) {
              const unsigned long long k = dkey(__dadd_rn(__ldcg(&cur[cdim * cur_stride + i]), 0.0));  // -0 == +0
              const std::uint32_t id = __ldcg(&cur_ids[i]);
              bool match;
              if (p < 8) {
                const int sh8 = 8 * (8 - p);
                match = (sh8 >= 64) ? true : ((k >> sh8) == (s.hi >> sh8));
                digit = static_cast<int>((k >> (8 * (7 - p))) & 0xff);
              } else {
                const int q = p - 8, sh8 = 8 * (4 - q);
                match = (k == s.hi) && ((sh8 >= 32) ? true : ((id >> sh8) == (s.lo >> sh8)));
                digit = static_cast<int>((id >> (8 * (3 - q))) & 0xff);
              }
              if (!match) digit = -1;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, digit);
            if (digit >= 0 && lane == __ffs(peers) - 1) atomicAdd(&a.hist[(o - b0) * 256 + digit], __popc(peers));
          }
        }
        sync_all(grid);
        for (std::uint32_t o = gtid; o < nb; o += gthreads) {
          SelState s;
          s.hi = __ldcg(&a.sel[o].hi);
          s.lo = __ldcg(&a.sel[o].lo);
          s.rank = __ldcg(&a.sel[o].rank);
          std::uint32_t* h = a.hist + o * 256;
          std::uint32_t acc = 0;
          int dsel = 255;
          for (int dg = 0; dg < 256; ++dg) {
            const std::uint32_t c = __ldcg(&h[dg]);
            if (s.rank < acc + c) { dsel = dg; break; }
            acc += c;
          }
          s.rank -= acc;
          if (p < 8) s.hi |= static_cast<unsigned long long>(dsel) << (8 * (7 - p));
          else s.lo |= static_cast<std::uint32_t>(dsel) << (8 * (3 - (p - 8)));
          a.sel[o] = s;
          for (int dg = 0; dg < 256; ++dg) h[dg] = 0;
          if (p == 11) {
            const std::uint32_t g = __ldcg(&a.obj_list[b0 + o]);
            na.split[g] = dkey_inv(s.hi);  // canonical +0 for a zero median
            na.thr_id[g] = s.lo;
          }
        }
        sync_all(grid);
      }
    }
    if (nobj) {  // left counts of object nodes ((x_c, id) < threshold)
      for (std::uint32_t c = gwarp; c < nchunks; c += nwarps) {
        const std::uint32_t v = __ldcg(&chunk_node[c]), g = off + v;
        if ((__ldcg(&na.flags[g]) & (F_LEAF | F_OBJECT)) != F_OBJECT) continue;
        const std::uint32_t s0 = __ldcg(&na.start[g]), nn = __ldcg(&na.count[g]);
        const std::uint32_t first = s0 + (c - __ldcg(&chunk_off[v])) * kc;
        const std::uint32_t end = min(first + kc, s0 + nn);
        const double s = __ldcg(&na.split[g]);
        const std::uint32_t tid = __ldcg(&na.thr_id[g]);
        std::uint32_t cnt = 0;
        for (std::uint32_t i0 = first; i0 < end; i0 += 32) {
          const std::uint32_t i = i0 + lane;
          bool pr = false;
          if (i < end) {
            const double x = __ldcg(&cur[cdim * cur_stride + i]);
            pr = x < s || (x == s && __ldcg(&cur_ids[i]) < tid);
          }
          cnt += __popc(__ballot_sync(0xffffffffu, pr));
        }
        if (lane == 0) a.chunk_left[c] = cnt;
      }
      sync_all(grid);
      scan_partial(a.chunk_left, nchunks + 1, a.bsum + gridDim.x, sh);  // again, with the object nodes' counts
      sync_all(grid);
    }

    scan_finish(a.is_int, a.irank, S + 1, a.bsum, sh);
    scan_finish(a.ccnt, a.coff, S + 1, a.bsum + 2 * gridDim.x, sh);
    scan_finish(a.chunk_left, a.left_scan, nchunks + 1, a.bsum + gridDim.x, sh);
    sync_all(grid);
    GK_PHASE_STAMP(4);
    const std::uint32_t nint = __ldcg(&a.irank[S]);
    const std::uint32_t nchunks_nx = __ldcg(&a.coff[S]);
    const std::uint32_t next_off = off + S;

    // F: child node records, the next level's chunk offsets and chunk -> node map (a node's few entries by
    // its own thread, a node of many chunks by its whole warp); G: stable partition
    for (std::uint32_t vb = gwarp * 32; vb < S; vb += nwarps * 32) {
      const std::uint32_t v = vb + lane, g = off + v;
      std::uint32_t u = 0, c0 = 0, c1 = 0, c2 = 0;
      if (v < S) {
        const std::uint32_t cb = next_off + 2 * __ldcg(&a.irank[v]);
        na.cbase[g] = cb;
        if (!(__ldcg(&na.flags[g]) & (F_LEAF | F_SMALL))) {
          const std::uint32_t s0 = __ldcg(&na.start[g]), nn = __ldcg(&na.count[g]), nl = __ldcg(&na.nleft[g]);
          na.start[cb] = s0; na.count[cb] = nl; na.parent[cb] = g;
          na.start[cb + 1] = s0 + nl; na.count[cb + 1] = nn - nl; na.parent[cb + 1] = g;
          na.nleft[cb] = 0;
          na.nleft[cb + 1] = 0;
          u = cb - next_off;
          c0 = __ldcg(&a.coff[v]);
          c1 = c0 + (nl + kc - 1) / kc;
          c2 = c1 + (nn - nl + kc - 1) / kc;
          chunk_off_nx[u] = c0;
          chunk_off_nx[u + 1] = c1;
        }
      }
      const bool wide = c2 - c0 > 8;
      if (!wide) {
        for (std::uint32_t c = c0; c < c2; ++c) chunk_node_nx[c] = c < c1 ? u : u + 1;
      }
      unsigned wm = __ballot_sync(0xffffffffu, wide);
      while (wm) {
        const int src = __ffs(wm) - 1;
        wm &= wm - 1;
        const std::uint32_t bu = __shfl_sync(0xffffffffu, u, src), b0 = __shfl_sync(0xffffffffu, c0, src),
                            b1 = __shfl_sync(0xffffffffu, c1, src), b2 = __shfl_sync(0xffffffffu, c2, src);
        for (std::uint32_t c = b0 + lane; c < b2; c += 32) chunk_node_nx[c] = c < b1 ? bu : bu + 1;
      }
    }
    if (gtid == 0) {
      chunk_off_nx[2 * nint] = nchunks_nx;
      a.ctrl[C_NCHUNKS] = nchunks_nx;
      a.ctrl[C_NOBJ] = 0;
    }
    // Sparse levels (many small chunks per warp): the warp splits into 32/gl lane groups that
    // partition as many chunks side by side, so the chunks' dependent metadata loads and their
    // point loads overlap instead of running one chunk after another
    const std::uint32_t gl =
        cpw >= kGroup4Chunks ? 4u : (cpw >= kGroup8Chunks ? 8u : (cpw >= kGroup16Chunks ? 16u : 32u));
    if (PH == 1 && gl < 32) {
      const std::uint32_t ngr = 32 / gl, grp = lane / gl, gla = lane % gl;
      const unsigned gmask = ((1u << gl) - 1u) << (grp * gl);
      const unsigned below = lt_mask & gmask;
      const std::uint32_t ncg = (nchunks + ngr - 1) / ngr;
      for (std::uint32_t cgi = gwarp; cgi < ncg; cgi += nwarps) {
        const std::uint32_t c = cgi * ngr + grp;
        std::uint32_t v = 0, g = 0, s0 = 0, first = 0, end = 0;
        std::uint8_t fl = F_LEAF;
        if (c < nchunks) {
          v = __ldcg(&chunk_node[c]);
          g = off + v;
          fl = __ldcg(&na.flags[g]);
          s0 = __ldcg(&na.start[g]);
          const std::uint32_t nn = __ldcg(&na.count[g]);
          first = s0 + (c - __ldcg(&chunk_off[v])) * kc;
          end = min(first + kc, s0 + nn);
        }
        const bool part = !(fl & (F_LEAF | F_SMALL));
        if (!part) {  // finished leaf or small subtree root (or no chunk): positions are final for this loop
          for (std::uint32_t i = first + gla; i < end; i += gl) {
#pragma unroll
            for (int j = 0; j < D; ++j) a.out[j * static_cast<std::uint64_t>(n) + i] = __ldcg(&cur[j * cur_stride + i]);
            a.out_ids[i] = __ldcg(&cur_ids[i]);
          }
        }
        const bool obj = (fl & F_OBJECT) != 0;
        double s = 0.0;
        std::uint32_t tid = 0, nl = 0, lbefore = 0;
        if (part) {
          s = __ldcg(&na.split[g]);
          tid = obj ? __ldcg(&na.thr_id[g]) : 0u;
          nl = __ldcg(&na.nleft[g]);
          lbefore = __ldcg(&a.left_scan[c]) - __ldcg(&a.left_scan[__ldcg(&chunk_off[v])]);
        }
        const std::uint32_t lb0 = lbefore;
        double mnl[D], mxl[D], mnr[D], mxr[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          mnl[j] = mnr[j] = __longlong_as_double(0x7ff0000000000000LL);
          mxl[j] = mxr[j] = -mnl[j];
        }
        const std::uint32_t rounds = part ? (end - first + gl - 1) / gl : 0u;
        const std::uint32_t maxr = __reduce_max_sync(0xffffffffu, rounds);
        for (std::uint32_t r = 0; r < maxr; ++r) {
          const std::uint32_t i = first + r * gl + gla;
          const bool valid = part && i < end;
          double x[D];
          std::uint32_t id = 0;
          bool pr = false;
          if (valid) {
#pragma unroll
            for (int j = 0; j < D; ++j) x[j] = __ldcg(&cur[j * cur_stride + i]);
            id = __ldcg(&cur_ids[i]);
            double xc = x[0];
#pragma unroll
            for (int j = 1; j < D; ++j)
              if (cdim == j) xc = x[j];
            pr = obj ? (xc < s || (xc == s && id < tid)) : (xc < s);
          }
          const unsigned bal = __ballot_sync(0xffffffffu, pr);
          if (valid) {
            const std::uint32_t lrank = lbefore + __popc(bal & below);
            const std::uint32_t np = pr ? s0 + lrank : s0 + nl + (i - s0 - lrank);
#pragma unroll
            for (int j = 0; j < D; ++j) {
              nxt[j * static_cast<std::uint64_t>(n) + np] = x[j];
              if (!kChildBoxes) continue;
              if (pr) { mnl[j] = fmin(mnl[j], x[j]); mxl[j] = fmax(mxl[j], x[j]); }
              else { mnr[j] = fmin(mnr[j], x[j]); mxr[j] = fmax(mxr[j], x[j]); }
            }
            nxt_ids[np] = id;
          }
          lbefore += __popc(bal & gmask);
        }
        if (!kChildBoxes) continue;
        const std::uint32_t nleft_chunk = lbefore - lb0, nright_chunk = end - first - nleft_chunk;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          for (std::uint32_t o = gl >> 1; o > 0; o >>= 1) {  // within the lane group
            mnl[j] = fmin(mnl[j], __shfl_xor_sync(0xffffffffu, mnl[j], o));
            mxl[j] = fmax(mxl[j], __shfl_xor_sync(0xffffffffu, mxl[j], o));
            mnr[j] = fmin(mnr[j], __shfl_xor_sync(0xffffffffu, mnr[j], o));
            mxr[j] = fmax(mxr[j], __shfl_xor_sync(0xffffffffu, mxr[j], o));
          }
        }
        if (part)
          for (int t = static_cast<int>(gla); t < 2 * D; t += static_cast<int>(gl)) {  // (side, dim) per lane
            const int j = t % D, side = t / D;
            double l = side ? mnr[0] : mnl[0], h = side ? mxr[0] : mxl[0];
#pragma unroll
            for (int jj = 1; jj < D; ++jj)
              if (j == jj) { l = side ? mnr[jj] : mnl[jj]; h = side ? mxr[jj] : mxl[jj]; }
            if (side ? nright_chunk : nleft_chunk) {
              const std::uint64_t u = 2ULL * __ldcg(&a.irank[v]) + side;
              unsigned long long* kk = a.keys + (u * D + j) * 2;
              atomicMin(kk, dkey(l));
              atomicMax(kk + 1, dkey(h));
            }
          }
      }
    } else {
    // the children's bounding boxes, accumulated while partitioning (the next level needs no box pass):
    // lane-private over the run's chunks of one node, reduced over the warp and sent to the children's
    // words when the node changes
    double mnl[D], mxl[D], mnr[D], mxr[D];
    std::uint32_t acc_v = 0xffffffffu, acc_nl = 0, acc_nr = 0;
    auto box_reset = [&]() {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        mnl[j] = mnr[j] = __longlong_as_double(0x7ff0000000000000LL);
        mxl[j] = mxr[j] = -mnl[j];
      }
      acc_nl = acc_nr = 0;
    };
    auto box_flush = [&]() {
      if constexpr (kChildBoxes) {
      if (acc_v == 0xffffffffu || (acc_nl | acc_nr) == 0) return;
#pragma unroll
      for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mnl[j] = fmin(mnl[j], __shfl_xor_sync(0xffffffffu, mnl[j], o));
          mxl[j] = fmax(mxl[j], __shfl_xor_sync(0xffffffffu, mxl[j], o));
          mnr[j] = fmin(mnr[j], __shfl_xor_sync(0xffffffffu, mnr[j], o));
          mxr[j] = fmax(mxr[j], __shfl_xor_sync(0xffffffffu, mxr[j], o));
        }
      }
      if (lane < 2 * D) {
        const int j = lane % D, side = lane / D;  // lanes [0, D): left child, [D, 2D): right child
        double l = side ? mnr[0] : mnl[0], h = side ? mxr[0] : mxl[0];
#pragma unroll
        for (int jj = 1; jj < D; ++jj)
          if (j == jj) { l = side ? mnr[jj] : mnl[jj]; h = side ? mxr[jj] : mxl[jj]; }
        if (side ? acc_nr : acc_nl) {
          const std::uint64_t u = 2ULL * __ldcg(&a.irank[acc_v]) + side;  // the child's index in the next level
          unsigned long long* kk = a.keys + (u * D + j) * 2;
          atomicMin(kk, dkey(l));
          atomicMax(kk + 1, dkey(h));
        }
      }
      }
    };
    box_reset();
    // the node's words are loaded once per run of its chunks (the chain chunk -> node -> split / counts ->
    // scan offsets is four dependent L2 round trips; a chunk of the same node as the last one needs none:
    // its left rank continues where the last chunk's ended), the next chunk's node one chunk ahead
    std::uint32_t vn = cfirst < cend ? __ldcg(&chunk_node[cfirst]) : 0u;
    std::uint8_t fl = 0;
    std::uint32_t s0 = 0, nn = 0, coff_v = 0, tid = 0, nl = 0, lbefore = 0, ls0 = 0;
    double s = 0.0;
    for (std::uint32_t c = cfirst; c < cend; c += cstep) {
      const std::uint32_t v = vn;
      if (c + cstep < cend) vn = __ldcg(&chunk_node[c + cstep]);
      if (v == acc_v && !runs && !(fl & (F_LEAF | F_SMALL)))  // same node, but not the next chunk: its own left rank
        lbefore = __ldcg(&a.left_scan[c]) - ls0;
      if (v != acc_v) {
        box_flush();
        box_reset();
        acc_v = v;
        const std::uint32_t g = off + v;
        fl = __ldcg(&na.flags[g]);
        s0 = __ldcg(&na.start[g]);
        nn = __ldcg(&na.count[g]);
        coff_v = __ldcg(&chunk_off[v]);
        if (!(fl & (F_LEAF | F_SMALL))) {
          s = __ldcg(&na.split[g]);
          tid = (fl & F_OBJECT) ? __ldcg(&na.thr_id[g]) : 0u;
          nl = __ldcg(&na.nleft[g]);
          ls0 = __ldcg(&a.left_scan[coff_v]);
          lbefore = __ldcg(&a.left_scan[c]) - ls0;
        }
      }
      const std::uint32_t first = s0 + (c - coff_v) * kc;
      const std::uint32_t end = min(first + kc, s0 + nn);
      if (fl & (F_LEAF | F_SMALL)) {  // finished (a small root's subtree is built by the bottom phase)
        for (std::uint32_t i = first + lane; i < end; i += 32) {
#pragma unroll
          for (int j = 0; j < D; ++j) a.out[j * static_cast<std::uint64_t>(n) + i] = __ldcg(&cur[j * cur_stride + i]);
          a.out_ids[i] = __ldcg(&cur_ids[i]);
        }
        continue;
      }
      const bool obj = (fl & F_OBJECT) != 0;
      const std::uint32_t lb0 = lbefore;
      constexpr int U = kPartUnroll;  // rounds whose loads are in flight together
      for (std::uint32_t i0 = first; i0 < end; i0 += 32 * U) {
        double x[U][D];
        std::uint32_t id[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const std::uint32_t i = i0 + 32 * u + lane;
          if (i < end) {
#pragma unroll
            for (int j = 0; j < D; ++j) x[u][j] = __ldcg(&cur[j * cur_stride + i]);
            id[u] = __ldcg(&cur_ids[i]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const std::uint32_t i = i0 + 32 * u + lane;
          const bool valid = i < end;
          bool pr = false;
          if (valid) {
            double xc = x[u][0];
#pragma unroll
            for (int j = 1; j < D; ++j)
              if (cdim == j) xc = x[u][j];
            pr = obj ? (xc < s || (xc == s && id[u] < tid)) : (xc < s);
          }
          const unsigned bal = __ballot_sync(0xffffffffu, pr);
          if (valid) {
            const std::uint32_t lrank = lbefore + __popc(bal & lt_mask);
            const std::uint32_t np = pr ? s0 + lrank : s0 + nl + (i - s0 - lrank);
#pragma unroll
            for (int j = 0; j < D; ++j) {
              nxt[j * static_cast<std::uint64_t>(n) + np] = x[u][j];
              if (!kChildBoxes) continue;
              if (pr) { mnl[j] = fmin(mnl[j], x[u][j]); mxl[j] = fmax(mxl[j], x[u][j]); }
              else { mnr[j] = fmin(mnr[j], x[u][j]); mxr[j] = fmax(mxr[j], x[u][j]); }
            }
            nxt_ids[np] = id[u];
          }
          lbefore += __popc(bal);
        }
      }
      acc_nl += lbefore - lb0;
      acc_nr += end - first - (lbefore - lb0);
    }
    box_flush();
    }
    if (gtid == 0) {
      a.lvl_off[level + 1] = next_off;
      a.ctrl[C_S] = 2 * nint;
    }
    // ping-pong: the partitioned points now live in nxt (stride n)
    cur = nxt;
    cur_ids = nxt_ids;
    cur_stride = n;
    nxt = (nxt == a.bufA) ? a.bufB : a.bufA;
    nxt_ids = (nxt_ids == a.idsA) ? a.idsB : a.idsA;
    sync_all(grid);
  }

  GK_TL_PRINT(level0);
#if GK_BUILD_TIMELINE
  unsigned long long tv_a = 0, tv_b = 0;
  if (gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tv_a));
#endif
  if (__ldcg(&a.ctrl[C_NSMALL]) > 0) {  // small subtrees pending: k_subtree + k_merge finish the tree
    if (gtid == 0) a.ctrl[C_H] = static_cast<std::uint32_t>(level);  // the level loop's levels
    GK_TL_PRINT(level0);
    return;
  }
  veb_phase(grid, a, na, a.lvl_off, level, sh);
#if GK_BUILD_TIMELINE
  if (gtid == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tv_b));
    printf("[tlveb] n=%u grid=%u H=%d N=%u vEB %.1f us\n", n, gridDim.x, level, a.ctrl[C_N], (tv_b - tv_a) * 1e-3);
  }
#endif
}

// ============================================================ bottom phase --
// Nodes of at most a.Tsmall points (F_SMALL, registered by phase E of the level loop) have their
// whole subtree built by k_subtree, one block per subtree, entirely in shared memory: the points are
// read once and written once, and the subtree's levels cost block barriers instead of grid barriers
// (the sparse bottom levels of the level loop were bound by per-chunk metadata latency).  Same split
// rules as the level loop and the oracle (Alg. 1; frozen decisions 3-6): split
// dim = depth mod D, spatial s = (lo + hi) / 2 with left x_c < s, degenerate side / depth >= 40 ->
// object median by (x_c, id) with left = the floor(n/2) smallest keys, stable partitions.  k_merge
// then interleaves the subtrees' nodes with the level loop's into complete level arrays (left-to-right
// = start order at every level) and runs the vEB slot phase over them.
constexpr int kSubThreads = 256;
#ifdef GK_DBG
#include <cassert>
#define GK_ASSERT(c) assert(c)
#else
#define GK_ASSERT(c) do {} while (0)
#endif
#ifndef GK_SMALL_T
#define GK_SMALL_T 1024
#endif
template <int D>
__host__ __device__ constexpr int small_cap() {
  return D <= 3 ? GK_SMALL_T : (D <= 5 ? GK_SMALL_T / 2 : GK_SMALL_T / 4);
}
template <int D>
__host__ __device__ constexpr int small_nmax() {  // nodes per level of a subtree (leaf >= 4: internal nodes >= 5 points)
  return 2 * small_cap<D>() / 5 + 2;
}
template <int D>
__host__ __device__ constexpr std::size_t small_smem() {
  constexpr int T = small_cap<D>(), NM = small_nmax<D>();
  return static_cast<std::size_t>(T) * D * 8 + static_cast<std::size_t>(NM) * 2 * 2 * 8 + 32 * 4 * 8 + T * 4 +
         32 * 4 + 16 + 2 * (kSubLevels + 1) * 4 + T * 2 * 2 + (T + 1) * 2 + NM * 2 * 4 + (NM + 1) * 2 +
         (T / 128 + 2) * 2 + 64;
}

// in-place exclusive scan of a[0, n) (a[n] = total) by the whole block; wsum: 32 words of shared memory
__device__ void block_exscan_u16(std::uint16_t* a, int n, std::uint32_t* wsum) {
  constexpr int nth = kSubThreads, nw = nth >> 5;  // compile-time: no integer division for the segment size
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + nth - 1) / nth;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  std::uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  std::uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    std::uint32_t v = lane < nw ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) wsum[lane] = v;
  }
  __syncthreads();
  std::uint32_t base = (wid ? wsum[wid - 1] : 0u) + x - s;
  for (int i = lo; i < hi; ++i) {
    const std::uint32_t t = a[i];
    a[i] = static_cast<std::uint16_t>(base);
    base += t;
  }
  if (tid == 0) a[n] = static_cast<std::uint16_t>(wsum[nw - 1]);
  __syncthreads();
}

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return b < a ? b : a; }
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return b > a ? b : a; }
// warp-wide min / max of 64-bit keys with the 32-bit redux unit (REDUX): the high words first, then
// the low words among the lanes that hold the extreme high word -- 4 reductions instead of 10 64-bit
// shuffle steps
__device__ __forceinline__ void warp_minmax(unsigned long long& mn, unsigned long long& mx) {
  const unsigned mh = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(mn >> 32));
  const unsigned ml = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(mn >> 32) == mh ? static_cast<unsigned>(mn) : 0xffffffffu);
  const unsigned xh = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(mx >> 32));
  const unsigned xl = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(mx >> 32) == xh ? static_cast<unsigned>(mx) : 0u);
  mn = (static_cast<unsigned long long>(mh) << 32) | ml;
  mx = (static_cast<unsigned long long>(xh) << 32) | xl;
}

// One subtree per block.  Per local level, nodes of at most kSubBig points are handled by one warp each
// (their positions in <= 4 rounds of 32, predicates and ranks by ballots), larger ones by the whole
// block one after another (block scan).  The split-dimension box of every node comes from its parent's
// partition (the children's min/max in the next level's dimension accumulate while it partitions);
// leaves reduce their full box; internal nodes' full boxes are the unions of their children's,
// bottom-up after the last level.
// nodes of up to this many points are split by one warp (1, 2, 4 or 8 rounds of 32 points), larger ones by the
// whole block one after another: 256 instead of 128 moves a 1024-point subtree's four 256-point nodes from the
// block path (~8 block barriers per node) to four warps side by side (C2 Insert_L 5.13 -> 5.00 ms, C1 -3.5 %)
#ifndef GK_SUB_BIG
#define GK_SUB_BIG 256
#endif
constexpr int kSubBig = GK_SUB_BIG;
template <int D>
__global__ void __launch_bounds__(kSubThreads) k_subtree(const BuildArgs a) {
  constexpr int T = small_cap<D>(), NM = small_nmax<D>();
  static_assert(kSubBig <= 256, "warp-mode nodes take at most 8 rounds of 32 points");
  extern __shared__ __align__(16) unsigned char smem[];
  double* X = reinterpret_cast<double*>(smem);                                        // [D][T]
  unsigned long long* nbl = reinterpret_cast<unsigned long long*>(X + D * T);          // [2][NM] split-dim lo key
  unsigned long long* nbh = nbl + 2 * NM;                                              // [2][NM] split-dim hi key
  unsigned long long* red = nbh + 2 * NM;                                              // [32][4] block reductions
  std::uint32_t* ID = reinterpret_cast<std::uint32_t*>(red + 32 * 4);                  // [T]
  std::uint32_t* wsum = ID + T;                                                        // [32]
  std::uint32_t* misc = wsum + 32;                                                     // [4]
  std::uint32_t* lvo = misc + 4;                                                       // [kSubLevels + 1]
  std::uint32_t* lvc = lvo + kSubLevels + 1;                                           // [kSubLevels + 1]
  std::uint16_t* permA = reinterpret_cast<std::uint16_t*>(lvc + kSubLevels + 1);       // [T]
  std::uint16_t* permB = permA + T;                                                    // [T]
  std::uint16_t* Lsc = permB + T;                                                      // [T + 1]
  std::uint16_t* nst = Lsc + T + 1;                                                    // [2][NM]
  std::uint16_t* ncn = nst + 2 * NM;                                                   // [2][NM]
  std::uint16_t* nscan = ncn + 2 * NM;                                                 // [NM + 1]
  std::uint16_t* bigl = nscan + NM + 1;                                                // [T / kSubBig + 1]

  const NodeArrays& na = a.na;
  constexpr int nth = kSubThreads, nwarps = nth >> 5;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const std::uint64_t N = a.n;  // SoA stride of the output
  const bool spatial_heur = a.heuristic != GK_OBJECT_MEDIAN;
  const int leaf = a.leaf;
  while (true) {
    if (tid == 0) misc[0] = atomicAdd(&a.ctrl[C_WORK], 1u);
    __syncthreads();
    const std::uint32_t r = misc[0];
    if (r >= __ldcg(&a.ctrl[C_NSMALL])) return;
    const std::uint32_t g = __ldcg(&a.small_list[r]);
    const std::uint32_t s0 = __ldcg(&na.start[g]);
    const int n = static_cast<int>(__ldcg(&na.count[g]));
    const int L = __ldcg(&na.level[g]);
    if (tid == 0) {
      misc[1] = atomicAdd(&a.ctrl[C_SUBCTR], 2u * static_cast<std::uint32_t>(n));
      nst[0] = 0;
      ncn[0] = static_cast<std::uint16_t>(n);
      const int c0 = L % D;  // the root's box in its split dimension (the level loop computed it)
      nbl[0] = dkey(__ldcg(&na.lo[static_cast<std::uint64_t>(g) * D + c0]));
      nbh[0] = dkey(__ldcg(&na.hi[static_cast<std::uint64_t>(g) * D + c0]));
    }
    for (int i = tid; i < n; i += nth) {
#pragma unroll
      for (int j = 0; j < D; ++j) X[j * T + i] = __ldcg(&a.out[j * N + s0 + i]);
      ID[i] = __ldcg(&a.out_ids[s0 + i]);
      permA[i] = static_cast<std::uint16_t>(i);
    }
    __syncthreads();
    const std::uint32_t base = misc[1];
    GK_ASSERT(base + 2u * n <= 2u * a.n && n <= T && r < a.rmax);
    std::uint32_t rec = base;  // this level's first record (local levels >= 1, level-major)
    std::uint16_t* perm = permA;
    std::uint16_t* perm2 = permB;
    int cb = 0, nc = 1, lv = 0;
    for (;; ++lv) {
      if (lv >= kSubLevels) __trap();  // unreachable: depth cap 40 + log2(T) + 1 levels
      const int depth = L + lv, c = depth % D, c1 = (depth + 1) % D;
      const bool spatial = spatial_heur && depth < kDepthCap;
      const std::uint16_t* cst = nst + cb * NM;
      const std::uint16_t* ccn = ncn + cb * NM;
      const unsigned long long* cbl = nbl + cb * NM;
      const unsigned long long* cbh = nbh + cb * NM;
      std::uint16_t* xst = nst + (cb ^ 1) * NM;
      std::uint16_t* xcn = ncn + (cb ^ 1) * NM;
      unsigned long long* xbl = nbl + (cb ^ 1) * NM;
      unsigned long long* xbh = nbh + (cb ^ 1) * NM;
      if (tid == 0) misc[3] = 0;
      __syncthreads();
      for (int i = tid; i < nc; i += nth) {
        nscan[i] = ccn[i] > leaf ? 1 : 0;  // internal -> child slots
        if (ccn[i] > kSubBig) bigl[atomicAdd(&misc[3], 1u)] = static_cast<std::uint16_t>(i);  // block-mode nodes
      }
      __syncthreads();
      const int nbig = static_cast<int>(misc[3]);
      block_exscan_u16(nscan, nc, wsum);
      const int nint = nscan[nc];
      // the node's record (this level), its children's slots and split-dim boxes (next level)
      auto finish = [&](int i, int st, int cnt, std::uint8_t fl, double sp, std::uint32_t thr, int nl,
                        unsigned long long mnl, unsigned long long mxl, unsigned long long mnr, unsigned long long mxr) {
        const int k2 = 2 * nscan[i];
        xst[k2] = static_cast<std::uint16_t>(st);
        xcn[k2] = static_cast<std::uint16_t>(nl);
        xst[k2 + 1] = static_cast<std::uint16_t>(st + nl);
        xcn[k2 + 1] = static_cast<std::uint16_t>(cnt - nl);
        xbl[k2] = mnl;
        xbh[k2] = mxl;
        xbl[k2 + 1] = mnr;
        xbh[k2 + 1] = mxr;
        if (lv == 0) {  // the subtree root is the level loop's node g: finish its record
          na.flags[g] = fl;
          na.split[g] = sp;
          na.thr_id[g] = thr;
        } else {
          const std::uint32_t ri = rec + i;
          GK_ASSERT(ri < base + 2u * n);
          a.s_start[ri] = s0 + st;
          a.s_count[ri] = cnt;
          a.s_flags[ri] = fl;
          a.s_split[ri] = sp;
          a.s_child[ri] = rec + nc + k2;  // the next level's records follow this level's
        }
      };
      // ---- warp mode: leaves and nodes of <= kSubBig points, one warp each
      for (int i = wid; i < nc; i += nwarps) {
        const int st = cst[i], cnt = ccn[i];
        if (cnt > kSubBig) continue;
        if (cnt <= leaf) {  // a leaf (<= 32 points): positions final (both buffers), full box
          const bool v = lane < cnt;
          const int ip = v ? perm[st + lane] : 0;
          if (v) perm2[st + lane] = static_cast<std::uint16_t>(ip);
          if (lv > 0) {
            const std::uint32_t ri = rec + i;
#pragma unroll
            for (int j = 0; j < D; ++j) {
              unsigned long long mn = v ? dkey(X[j * T + ip]) : ~0ULL, mx = v ? mn : 0ULL;
              warp_minmax(mn, mx);
              if (lane == 0) {
                a.s_lo[static_cast<std::uint64_t>(ri) * D + j] = dkey_inv(mn);
                a.s_hi[static_cast<std::uint64_t>(ri) * D + j] = dkey_inv(mx);
              }
            }
            if (lane == 0) {
              a.s_start[ri] = s0 + st;
              a.s_count[ri] = cnt;
              a.s_flags[ri] = F_LEAF;
              a.s_split[ri] = 0.0;
            }
          }
          continue;
        }
        // rounds of 32 points, compiled for 1, 2 and 4 rounds (most nodes of the bottom levels hold <= 64 points)
        auto split_node = [&](auto nit_c) {
          constexpr int NIT = decltype(nit_c)::value;
          bool v[NIT];
          int ip[NIT];
          double x[NIT];
          unsigned b[NIT];
#pragma unroll
          for (int it = 0; it < NIT; ++it) {
            const int q = 32 * it + lane;
            v[it] = q < cnt;
            ip[it] = v[it] ? perm[st + q] : 0;
            x[it] = v[it] ? X[c * T + ip[it]] : 0.0;
            b[it] = 0;
          }
          std::uint8_t fl = F_OBJECT;
          double sp = 0.0;
          std::uint32_t thr = 0;
          int nl = 0;
          if (spatial) {
            sp = __dmul_rn(__dadd_rn(dkey_inv(cbl[i]), dkey_inv(cbh[i])), 0.5);  // (lo + hi) / 2 exactly
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
              b[it] = __ballot_sync(0xffffffffu, v[it] && x[it] < sp);
              nl += __popc(b[it]);
            }
            if (nl > 0 && nl < cnt) fl = 0;
          }
          if (fl == F_OBJECT) {  // object median: the key of rank floor(cnt/2) in (x_c, id) order (-0 == +0)
            const int m = cnt / 2;
            std::uint32_t idv[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
              idv[it] = v[it] ? ID[ip[it]] : 0u;
              int rank = -1;
              if (v[it]) {
                rank = 0;
                for (int q = st; q < st + cnt; ++q) {
                  const int iq = perm[q];
                  const double xq = X[c * T + iq];
                  rank += (xq < x[it] || (xq == x[it] && ID[iq] < idv[it])) ? 1 : 0;
                }
              }
              const unsigned hit = __ballot_sync(0xffffffffu, rank == m);
              if (hit) {
                const int src = __ffs(hit) - 1;
                sp = __dadd_rn(__shfl_sync(0xffffffffu, x[it], src), 0.0);  // canonical +0, as the level loop
                thr = __shfl_sync(0xffffffffu, idv[it], src);
              }
            }
            nl = 0;
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
              b[it] = __ballot_sync(0xffffffffu, v[it] && (x[it] < sp || (x[it] == sp && idv[it] < thr)));
              nl += __popc(b[it]);
            }
          }
          // stable partition + the children's boxes in the next level's split dimension
          unsigned long long mnl = ~0ULL, mxl = 0ULL, mnr = ~0ULL, mxr = 0ULL;
          int before = 0;
#pragma unroll
          for (int it = 0; it < NIT; ++it) {
            const bool pr = (b[it] >> lane) & 1u;
            if (v[it]) {
              const int q = 32 * it + lane;
              const int rk = before + __popc(b[it] & lt_mask);
              const int np = pr ? st + rk : st + nl + (q - rk);
              perm2[np] = static_cast<std::uint16_t>(ip[it]);
              const unsigned long long k = dkey(X[c1 * T + ip[it]]);
              if (pr) { mnl = umin64(mnl, k); mxl = umax64(mxl, k); }
              else { mnr = umin64(mnr, k); mxr = umax64(mxr, k); }
            }
            before += __popc(b[it]);
          }
          warp_minmax(mnl, mxl);
          warp_minmax(mnr, mxr);
          if (lane == 0) finish(i, st, cnt, fl, sp, thr, nl, mnl, mxl, mnr, mxr);
        };
        if (cnt <= 32) split_node(std::integral_constant<int, 1>{});
        else if (cnt <= 64) split_node(std::integral_constant<int, 2>{});
        else if (kSubBig <= 128 || cnt <= 128) split_node(std::integral_constant<int, 4>{});
        else split_node(std::integral_constant<int, 8>{});
      }
      // ---- block mode: nodes of more than kSubBig points, the whole block on one node at a time
      for (int bi = 0; bi < nbig; ++bi) {
        const int i = bigl[bi];
        const int st = cst[i], cnt = ccn[i];
        std::uint8_t fl = F_OBJECT;
        double sp = 0.0;
        std::uint32_t thr = 0;
        int nl = 0;
        if (spatial) {
          sp = __dmul_rn(__dadd_rn(dkey_inv(cbl[i]), dkey_inv(cbh[i])), 0.5);
          int cntl = 0;
          for (int q = tid; q < cnt; q += nth) cntl += X[c * T + perm[st + q]] < sp ? 1 : 0;
          nl = 0;
          for (int o = 16; o > 0; o >>= 1) cntl += __shfl_xor_sync(0xffffffffu, cntl, o);
          if (lane == 0) wsum[wid] = static_cast<std::uint32_t>(cntl);
          __syncthreads();
          for (int w = 0; w < nwarps; ++w) nl += static_cast<int>(wsum[w]);
          __syncthreads();
          if (nl > 0 && nl < cnt) fl = 0;
        }
        if (fl == F_OBJECT) {
          const int m = cnt / 2;
          for (int q = tid; q < cnt; q += nth) {
            const int ipq = perm[st + q];
            const double xp = X[c * T + ipq];
            const std::uint32_t idp = ID[ipq];
            int rank = 0;
            for (int u = st; u < st + cnt; ++u) {
              const int iu = perm[u];
              const double xu = X[c * T + iu];
              rank += (xu < xp || (xu == xp && ID[iu] < idp)) ? 1 : 0;
            }
            if (rank == m) {  // unique
              reinterpret_cast<double*>(red)[0] = __dadd_rn(xp, 0.0);
              misc[2] = idp;
            }
          }
          __syncthreads();
          sp = reinterpret_cast<double*>(red)[0];
          thr = misc[2];
          nl = m;
          __syncthreads();
        }
        // predicates, block scan, stable partition, children's split-dim boxes
        for (int q = tid; q < cnt; q += nth) {
          const int ipq = perm[st + q];
          const double xq = X[c * T + ipq];
          const bool pr = (fl == F_OBJECT) ? (xq < sp || (xq == sp && ID[ipq] < thr)) : (xq < sp);
          Lsc[q] = pr ? 1 : 0;
        }
        __syncthreads();
        block_exscan_u16(Lsc, cnt, wsum);
        unsigned long long mnl = ~0ULL, mxl = 0ULL, mnr = ~0ULL, mxr = 0ULL;
        for (int q = tid; q < cnt; q += nth) {
          const int ipq = perm[st + q];
          const bool pr = Lsc[q + 1] != Lsc[q];
          const int np = pr ? st + Lsc[q] : st + nl + (q - Lsc[q]);
          perm2[np] = static_cast<std::uint16_t>(ipq);
          const unsigned long long k = dkey(X[c1 * T + ipq]);
          if (pr) { mnl = umin64(mnl, k); mxl = umax64(mxl, k); }
          else { mnr = umin64(mnr, k); mxr = umax64(mxr, k); }
        }
        warp_minmax(mnl, mxl);
        warp_minmax(mnr, mxr);
        if (lane == 0) {
          red[wid * 4 + 0] = mnl;
          red[wid * 4 + 1] = mxl;
          red[wid * 4 + 2] = mnr;
          red[wid * 4 + 3] = mxr;
        }
        __syncthreads();
        if (tid == 0) {
          for (int w = 1; w < nwarps; ++w) {
            mnl = umin64(mnl, red[w * 4 + 0]);
            mxl = umax64(mxl, red[w * 4 + 1]);
            mnr = umin64(mnr, red[w * 4 + 2]);
            mxr = umax64(mxr, red[w * 4 + 3]);
          }
          finish(i, st, cnt, fl, sp, thr, nl, mnl, mxl, mnr, mxr);
        }
        __syncthreads();
      }
      if (tid == 0) {
        a.sub_cnt[static_cast<std::uint64_t>(r) * kSubLevels + lv] = static_cast<std::uint32_t>(nc);
        lvo[lv] = rec;
        lvc[lv] = static_cast<std::uint32_t>(nc);
      }
      if (lv > 0) rec += nc;
      __syncthreads();
      {
        std::uint16_t* t = perm;
        perm = perm2;
        perm2 = t;
      }
      if (nint == 0) break;
      cb ^= 1;
      nc = 2 * nint;
      if (nc > NM) __trap();  // unreachable for leaf >= 4
    }
    // internal nodes' boxes, bottom-up: the union of their children's (dkey order, as the level loop's
    // atomics; the root's box came from the level loop)
    for (int l2 = lv - 1; l2 >= 1; --l2) {
      const std::uint32_t r0 = lvo[l2], rc = lvc[l2];
      for (std::uint32_t i = tid; i < rc; i += nth) {
        const std::uint32_t ri = r0 + i;
        if (a.s_flags[ri] & F_LEAF) continue;
        const std::uint64_t c0 = a.s_child[ri];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double l0 = a.s_lo[c0 * D + j], l1 = a.s_lo[(c0 + 1) * D + j];
          const double h0 = a.s_hi[c0 * D + j], h1 = a.s_hi[(c0 + 1) * D + j];
          a.s_lo[static_cast<std::uint64_t>(ri) * D + j] = dkey(l1) < dkey(l0) ? l1 : l0;
          a.s_hi[static_cast<std::uint64_t>(ri) * D + j] = dkey(h1) > dkey(h0) ? h1 : h0;
        }
      }
      __syncthreads();
    }
    // the subtree's points in their final (leaf) order
    for (int p = tid; p < n; p += nth) {
      const int ip = perm[p];
#pragma unroll
      for (int j = 0; j < D; ++j) a.out[j * N + s0 + p] = X[j * T + ip];
      a.out_ids[s0 + p] = ID[ip];
    }
    if (tid == 0) {
      a.sub_base[r] = base;
      a.sub_nlev[r] = static_cast<std::uint32_t>(lv + 1);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ std::uint32_t lower_bound_u32(const std::uint32_t* a, std::uint32_t lo, std::uint32_t hi,
                                                         std::uint32_t x) {  // first i in [lo, hi) with a[i] >= x
  while (lo < hi) {
    const std::uint32_t mid = (lo + hi) >> 1;
    if (__ldcg(&a[mid]) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Interleaves the subtrees' nodes with the level loop's ones.  At every level the left-to-right order
// is the order of the nodes' first points (disjoint ranges), so: small roots in start order, per
// (level, root) node counts scanned into positions, each node's merged index = level offset +
// (level-loop nodes left of it) + (subtree nodes left of it), then parent and first-child indices by
// binary search over each level's starts, then the vEB phase.  The merged arrays are a.na2 (parent,
// cbase and pos shared with a.na); k_emit reads a.na2 when the bottom phase ran.
template <int D>
__global__ void __launch_bounds__(kThreads) k_merge(const BuildArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ std::uint32_t sh[32];
  const NodeArrays& na = a.na;
  const NodeArrays& nb = a.na2;
  const std::uint32_t R = __ldcg(&a.ctrl[C_NSMALL]);
  if (R == 0) return;
  const std::uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  const std::uint32_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const int lane = threadIdx.x & 31;
  const std::uint32_t n = a.n;
#if GK_BUILD_TIMELINE
  unsigned long long mst[12];
  int nm = 0;
#define GK_MSTAMP() do { if (gtid == 0 && nm < 12) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(mst[nm++])); } while (0)
#else
#define GK_MSTAMP() do {} while (0)
#endif
  GK_MSTAMP();
  const int HA = static_cast<int>(__ldcg(&a.ctrl[C_H]));  // level-loop levels
  const std::uint32_t NA = __ldcg(&a.lvl_off[HA]);
  // small roots' first points marked over the points and scanned: rank(x) = # roots starting before x
  for (std::uint32_t i = gtid; i <= n; i += gthreads) a.marks[i] = 0;
  if (gtid == 0) {
    a.ctrl[C_S] = static_cast<std::uint32_t>(HA);  // max level + 1
    a.ctrl[C_NOBJ] = 0xffffffffu;                  // min root level
  }
  sync_all(grid);
  GK_MSTAMP();
  for (std::uint32_t r = gtid; r < R; r += gthreads) {
    const std::uint32_t g = __ldcg(&a.small_list[r]);
    a.marks[__ldcg(&na.start[g])] = 1;
    const std::uint32_t L = __ldcg(&na.level[g]);
    atomicMax(&a.ctrl[C_S], L + __ldcg(&a.sub_nlev[r]));
    atomicMin(&a.ctrl[C_NOBJ], L);
  }
  sync_all(grid);
  GK_MSTAMP();
  grid_scan(grid, a.marks, a.mscan, n + 1, a.bsum, sh);
  sync_all(grid);
  GK_MSTAMP();
  const int H = static_cast<int>(__ldcg(&a.ctrl[C_S]));
  const int Lmin = static_cast<int>(__ldcg(&a.ctrl[C_NOBJ]));
  // # small roots whose first point precedes position x
  auto root_rank = [&](std::uint32_t x) -> std::uint32_t { return __ldcg(&a.mscan[x]); };
  for (std::uint32_t r = gtid; r < R; r += gthreads) {
    const std::uint32_t k = root_rank(__ldcg(&na.start[__ldcg(&a.small_list[r])]));
    GK_ASSERT(k < R);
    a.order[k] = r;
  }
  const std::uint32_t span = static_cast<std::uint32_t>(H - Lmin - 1);  // levels Lmin + 1 .. H - 1 hold subtree nodes
  if (static_cast<std::uint64_t>(span) * R + 1 > a.vcap) __trap();       // unreachable: vcap = rmax x 160 levels
  sync_all(grid);
  GK_MSTAMP();
  // V[(l - Lmin - 1) * R + k] = nodes of root order[k] at level l, scanned in place
  const std::uint32_t VN = span * R;
  for (std::uint32_t i = gtid; i <= VN; i += gthreads) {
    std::uint32_t v = 0;
    if (i < VN) {
      const int l = Lmin + 1 + static_cast<int>(i / R);
      const std::uint32_t r = __ldcg(&a.order[i % R]);
      const int lam = l - static_cast<int>(__ldcg(&na.level[__ldcg(&a.small_list[r])]));
      if (lam >= 1 && lam < static_cast<int>(__ldcg(&a.sub_nlev[r])))
        v = __ldcg(&a.sub_cnt[static_cast<std::uint64_t>(r) * kSubLevels + lam]);
    }
    a.V[i] = v;
  }
  sync_all(grid);
  GK_MSTAMP();
  grid_scan(grid, a.V, a.V, VN + 1, a.bsum, sh);
  sync_all(grid);
  GK_MSTAMP();
  if (gtid == 0) {
    std::uint32_t acc = 0;
    for (int l = 0; l < H; ++l) {
      a.new_off[l] = acc;
      const std::uint32_t A = l < HA ? __ldcg(&a.lvl_off[l + 1]) - __ldcg(&a.lvl_off[l]) : 0u;
      std::uint32_t S = 0;
      if (l > Lmin) S = __ldcg(&a.V[(l - Lmin) * R]) - __ldcg(&a.V[(l - Lmin - 1) * R]);
      acc += A + S;
    }
    a.new_off[H] = acc;
    a.new_off[H + 1] = acc;
  }
  sync_all(grid);
  GK_MSTAMP();
  // scatter the level loop's nodes
  for (std::uint32_t x = gtid; x < NA; x += gthreads) {
    const int l = __ldcg(&na.level[x]);
    const std::uint32_t st = __ldcg(&na.start[x]);
    std::uint32_t y = __ldcg(&a.new_off[l]) + (x - __ldcg(&a.lvl_off[l]));
    if (l > Lmin) {
      const std::uint32_t row = (l - Lmin - 1) * R;
      y += __ldcg(&a.V[row + root_rank(st)]) - __ldcg(&a.V[row]);
    }
    GK_ASSERT(y < 2 * n - 1);
    nb.start[y] = st;
    nb.count[y] = __ldcg(&na.count[x]);
    nb.flags[y] = __ldcg(&na.flags[x]);
    nb.level[y] = static_cast<std::uint8_t>(l);
    nb.split[y] = __ldcg(&na.split[x]);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      nb.lo[static_cast<std::uint64_t>(y) * D + j] = __ldcg(&na.lo[static_cast<std::uint64_t>(x) * D + j]);
      nb.hi[static_cast<std::uint64_t>(y) * D + j] = __ldcg(&na.hi[static_cast<std::uint64_t>(x) * D + j]);
    }
  }
  // scatter the subtrees' nodes: one warp per subtree, level by level.  Their parent / first-child links
  // follow from the subtree's own level-major layout (an internal node's children are records 2 p, 2 p + 1
  // of the subtree's next level, p = internal nodes before it in its level; a leaf's insertion point among
  // the next level is the same 2 p), so only the level loop's nodes need the binary searches below
  // (1.4M nodes x two ~17-step searches were ~40 % of k_merge on C2's largest tree)
  const unsigned lt_mask = (1u << lane) - 1u;
  // merged index of the first node of subtree (rs = first point, k = root rank) at level l (or, where it
  // has none, of the position its nodes would take): level offset + subtree nodes of roots left of it +
  // level-loop nodes left of it
  auto sub_level_base = [&](int l, std::uint32_t rs, std::uint32_t k) -> std::uint32_t {
    if (l >= H) return __ldcg(&a.new_off[H]);
    std::uint32_t y = __ldcg(&a.new_off[l]);
    if (l > Lmin) {
      const std::uint32_t row = (l - Lmin - 1) * R;
      y += __ldcg(&a.V[row + k]) - __ldcg(&a.V[row]);
    }
    if (l < HA) y += lower_bound_u32(na.start, __ldcg(&a.lvl_off[l]), __ldcg(&a.lvl_off[l + 1]), rs) - __ldcg(&a.lvl_off[l]);
    return y;
  };
  for (std::uint32_t r = gwarp; r < R; r += nwarps) {
    const std::uint32_t g = __ldcg(&a.small_list[r]);
    const std::uint32_t rs = __ldcg(&na.start[g]);
    const int L = __ldcg(&na.level[g]);
    const int nlev = static_cast<int>(__ldcg(&a.sub_nlev[r]));
    const std::uint32_t k = root_rank(rs);
    std::uint32_t src = __ldcg(&a.sub_base[r]);
    // the root is the level loop's node g: its merged index (as in the scatter above)
    std::uint32_t yg = __ldcg(&a.new_off[L]) + (g - __ldcg(&a.lvl_off[L]));
    if (L > Lmin) {
      const std::uint32_t row = (L - Lmin - 1) * R;
      yg += __ldcg(&a.V[row + k]) - __ldcg(&a.V[row]);
    }
    std::uint32_t y0 = nlev > 1 ? sub_level_base(L + 1, rs, k) : 0u;
    for (int lam = 1; lam < nlev; ++lam) {
      const int l = L + lam;
      const std::uint32_t cnt = __ldcg(&a.sub_cnt[static_cast<std::uint64_t>(r) * kSubLevels + lam]);
      const std::uint32_t y0n = sub_level_base(l + 1, rs, k);
      if (lam == 1 && lane < static_cast<int>(cnt)) nb.parent[y0 + lane] = yg;  // the root's two children
      std::uint32_t carry = 0;  // internal nodes of this level before the current round
      for (std::uint32_t jb = 0; jb < cnt; jb += 32) {
        const std::uint32_t j = jb + lane;
        const bool valid = j < cnt;
        const std::uint32_t xs = src + j, y = y0 + j;
        GK_ASSERT(!valid || (y < 2 * n - 1 && xs < 2 * n));
        const std::uint8_t fl = valid ? __ldcg(&a.s_flags[xs]) : F_LEAF;
        const bool internal = valid && !(fl & F_LEAF);
        const unsigned bal = __ballot_sync(0xffffffffu, internal);
        const std::uint32_t cb = y0n + 2 * (carry + __popc(bal & lt_mask));
        carry += __popc(bal);
        if (!valid) continue;
        nb.cbase[y] = cb;
        if (internal) {
          nb.parent[cb] = y;
          nb.parent[cb + 1] = y;
        }
        nb.start[y] = __ldcg(&a.s_start[xs]);
        nb.count[y] = __ldcg(&a.s_count[xs]);
        nb.flags[y] = fl;
        nb.level[y] = static_cast<std::uint8_t>(l);
        nb.split[y] = __ldcg(&a.s_split[xs]);
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
          nb.lo[static_cast<std::uint64_t>(y) * D + jj] = __ldcg(&a.s_lo[static_cast<std::uint64_t>(xs) * D + jj]);
          nb.hi[static_cast<std::uint64_t>(y) * D + jj] = __ldcg(&a.s_hi[static_cast<std::uint64_t>(xs) * D + jj]);
        }
      }
      src += cnt;
      y0 = y0n;
    }
  }
  sync_all(grid);
  GK_MSTAMP();
  // parent / first child (or, for a leaf, the insertion point among the next level) of the level loop's
  // nodes, by start
  for (std::uint32_t x0 = gtid; x0 < NA; x0 += gthreads) {
    const int l = __ldcg(&na.level[x0]);
    const std::uint32_t st = __ldcg(&na.start[x0]);
    std::uint32_t x = __ldcg(&a.new_off[l]) + (x0 - __ldcg(&a.lvl_off[l]));  // its merged index (as scattered)
    if (l > Lmin) {
      const std::uint32_t row = (l - Lmin - 1) * R;
      x += __ldcg(&a.V[row + root_rank(st)]) - __ldcg(&a.V[row]);
    }
    GK_ASSERT(l < H && st < n);
    const std::uint32_t o1 = __ldcg(&a.new_off[l + 1]), o2 = __ldcg(&a.new_off[l + 2 <= H ? l + 2 : H]);
    nb.cbase[x] = (l + 1 < H) ? lower_bound_u32(nb.start, o1, o2, st) : o1;
    if (l == 0) {
      nb.parent[x] = 0xffffffffu;
    } else {
      const std::uint32_t p0 = __ldcg(&a.new_off[l - 1]);
      nb.parent[x] = lower_bound_u32(nb.start, p0, __ldcg(&a.new_off[l]), st + 1) - 1;  // last start <= st
    }
  }
  sync_all(grid);
  GK_MSTAMP();
  veb_phase(grid, a, nb, a.new_off, H, sh);
  GK_MSTAMP();
#if GK_BUILD_TIMELINE
  if (gtid == 0) {
    printf("[tlmerge] n=%u grid=%u R=%u H=%d:", n, gridDim.x, R, H);
    for (int q = 1; q < nm; ++q) printf(" %.1f", (mst[q] - mst[q - 1]) * 1e-3);
    printf(" us\n");
  }
#endif
#undef GK_MSTAMP
}


// One thread per node (level-array order, so the node-array reads coalesce); the canonical record and
// the traversal node are staged in shared memory and written by the whole warp, 8 / 16 bytes per lane
// over consecutive words of consecutive records (a record per thread was ~21 scattered stores, each
// touching 32 sectors: k_emit took 337 us on C2's largest tree)
constexpr int kEmitThreads = 128;
template <int D>
__global__ void __launch_bounds__(kEmitThreads) k_emit(const BuildArgs a, std::uint32_t N, std::uint32_t* __restrict__ irank_out,
                                                      gk_canon_node* canon, TNode<D>* tn, std::int32_t* orig) {
  const std::uint32_t* __restrict__ irank_by_slot = a.irank_slot;  // scanned at the end of the vEB phase
  static_assert(sizeof(gk_canon_node) % 8 == 0 && sizeof(TNode<D>) % 16 == 0, "record sizes");
  __shared__ gk_canon_node s_c[kEmitThreads];
  __shared__ TNode<D> s_t[kEmitThreads];
  __shared__ std::uint32_t s_slot[kEmitThreads], s_ti[kEmitThreads];
  const NodeArrays& na = a.na;
  const std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g <= N) irank_out[g] = irank_by_slot[g];  // the tree's own copy (erase collapse relinks through it)
  if (g < N) {
    const std::uint32_t slot = na.pos[g];
    const std::uint8_t fl = na.flags[g];
    const bool leaf = (fl & F_LEAF) != 0;
    gk_canon_node c;
    c.kind = leaf ? 1 : 0;
    c.depth = na.level[g];
    c.dim = leaf ? -1 : (c.depth % D);
    c.mode = (!leaf && (fl & F_OBJECT)) ? 1 : 0;
    c.split = na.split[g];
    c.start = na.start[g];
    c.count = na.count[g];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c.lo[j] = j < D ? na.lo[static_cast<std::uint64_t>(g) * D + j] : 0.0;
      c.hi[j] = j < D ? na.hi[static_cast<std::uint64_t>(g) * D + j] : 0.0;
    }
    std::uint32_t ti = 0xffffffffu;
    if (leaf) {
      c.left = c.right = -1;
      orig[slot] = -1;
      orig[N + slot] = -1;
    } else {
      const std::uint32_t cb = na.cbase[g];
      c.left = static_cast<int32_t>(na.pos[cb]);
      c.right = static_cast<int32_t>(na.pos[cb + 1]);
      orig[slot] = c.left;
      orig[N + slot] = c.right;
      orig[2 * N + c.left] = static_cast<std::int32_t>(slot);
      orig[2 * N + c.right] = static_cast<std::int32_t>(slot);
      TNode<D> t;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const std::uint32_t ch = cb + s;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          t.lo[j][s] = __double2float_rd(na.lo[static_cast<std::uint64_t>(ch) * D + j]);
          t.hi[j][s] = __double2float_ru(na.hi[static_cast<std::uint64_t>(ch) * D + j]);
        }
        t.ref[s] = (na.flags[ch] & F_LEAF) ? make_leaf_ref(na.start[ch], na.count[ch])
                                           : static_cast<std::uint64_t>(irank_by_slot[na.pos[ch]]);
      }
      s_t[threadIdx.x] = t;
      ti = irank_by_slot[slot];
    }
    s_c[threadIdx.x] = c;
    s_slot[threadIdx.x] = slot;
    s_ti[threadIdx.x] = ti;
  }
  __syncwarp();
  // the warp's 32 records, word by word: consecutive lanes write consecutive words of one record
  const int lane = threadIdx.x & 31, w0 = threadIdx.x & ~31;
  const std::uint32_t gw = blockIdx.x * blockDim.x + w0;
  const int nrec = gw >= N ? 0 : static_cast<int>(min(32u, N - gw));
  constexpr int kCW = sizeof(gk_canon_node) / 8, kTW = sizeof(TNode<D>) / 16;
  const unsigned long long* cs = reinterpret_cast<const unsigned long long*>(&s_c[w0]);
  for (int t = lane; t < nrec * kCW; t += 32) {
    const int r = t / kCW, wd = t - r * kCW;
    reinterpret_cast<unsigned long long*>(canon + s_slot[w0 + r])[wd] = cs[t];
  }
  const uint4* ts = reinterpret_cast<const uint4*>(&s_t[w0]);
  for (int t = lane; t < nrec * kTW; t += 32) {
    const int r = t / kTW, wd = t - r * kTW;
    const std::uint32_t ti = s_ti[w0 + r];
    if (ti != 0xffffffffu) reinterpret_cast<uint4*>(tn + ti)[wd] = ts[t];
  }
}

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

// ------------------------------------------------------------ Erase_S collapse --
// Bottom-up over the build-time topology (LBVH-refit style: the second child to
// arrive at a parent computes it).  repl[v] = v if both children survive, the
// surviving child's replacement if one does, -1 if none; a leaf survives while
// any of its points is live (tombstone = NaN in coordinate 0).
__global__ void k_collapse_up(std::uint32_t N, const gk_canon_node* __restrict__ canon, const double* __restrict__ c0,
                              const std::int32_t* __restrict__ orig, std::int32_t* repl, std::uint32_t* arrive) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N || canon[v].kind != 1) return;
  bool alive = false;
  for (std::uint32_t i = canon[v].start; i < canon[v].start + canon[v].count; ++i) alive = alive || !isnan(c0[i]);
  std::int32_t cur = static_cast<std::int32_t>(v);
  __stcg(&repl[cur], alive ? cur : -1);
  while (true) {
    __threadfence();
    const std::int32_t p = orig[2 * N + cur];
    if (p < 0) break;
    if (atomicAdd(&arrive[p], 1u) == 0) break;  // the sibling's thread finishes the parent
    __threadfence();
    const std::int32_t x = __ldcg(&repl[orig[p]]), y = __ldcg(&repl[orig[N + p]]);
    __stcg(&repl[p], (x >= 0 && y >= 0) ? p : (x >= 0 ? x : y));
    cur = p;
  }
}

template <int D>
__global__ void k_relink(std::uint32_t N, gk_canon_node* canon, TNode<D>* tn, const std::uint32_t* __restrict__ irank,
                         const std::int32_t* __restrict__ orig, const std::int32_t* __restrict__ repl) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N || canon[v].kind != 0) return;
  const std::int32_t x = repl[orig[v]], y = repl[orig[N + v]];
  if (x < 0 || y < 0) return;  // v itself is spliced out or removed
  canon[v].left = x;
  canon[v].right = y;
  TNode<D> t = tn[irank[v]];
  const std::int32_t ch[2] = {x, y};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const gk_canon_node& c = canon[ch[s]];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      t.lo[j][s] = __double2float_rd(c.lo[j]);
      t.hi[j][s] = __double2float_ru(c.hi[j]);
    }
    t.ref[s] = c.kind == 1 ? make_leaf_ref(c.start, c.count) : static_cast<std::uint64_t>(irank[ch[s]]);
  }
  tn[irank[v]] = t;
}

template <int D>
void collapse_d(DevTree& T, cudaStream_t st) {
  const std::uint32_t N = static_cast<std::uint32_t>(T.n_nodes);
  if (N == 0) return;
  std::int32_t* repl = dalloc<std::int32_t>(N, st);
  std::uint32_t* arrive = dalloc<std::uint32_t>(N, st);
  GK_CUDA(cudaMemsetAsync(arrive, 0, static_cast<std::size_t>(N) * 4, st));
  k_collapse_up<<<blocks_for(N), 256, 0, st>>>(N, T.canon, T.coords, T.orig, repl, arrive);
  k_relink<D><<<blocks_for(N), 256, 0, st>>>(N, T.canon, static_cast<TNode<D>*>(T.tnodes), T.irank, T.orig, repl);
  GK_CHECK_LAUNCH();
  std::int32_t root = -1;
  gk_canon_node rc;
  GK_CUDA(cudaMemcpyAsync(&root, repl, 4, cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  T.root_slot = root;
  if (root >= 0) {
    std::uint32_t ir = 0;
    GK_CUDA(cudaMemcpyAsync(&rc, T.canon + root, sizeof(rc), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaMemcpyAsync(&ir, T.irank + root, 4, cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    T.root_ref = rc.kind == 1 ? make_leaf_ref(rc.start, rc.count) : ir;
  }
  dfree(repl, st);
  dfree(arrive, st);
}

// the surviving root of a collapsed tree: {root slot, leaf?, start, count, internal rank}
__global__ void k_root_info(const std::int32_t* __restrict__ repl, const gk_canon_node* __restrict__ canon,
                            const std::uint32_t* __restrict__ irank, std::uint32_t* out) {
  const std::int32_t r = repl[0];
  out[0] = static_cast<std::uint32_t>(r);
  if (r >= 0) {
    out[1] = static_cast<std::uint32_t>(canon[r].kind);
    out[2] = canon[r].start;
    out[3] = canon[r].count;
    out[4] = irank[r];
  }
}

template <int D>
void collapse_launch(DevTree& T, std::int32_t* repl, std::uint32_t* arrive, std::uint32_t* info, cudaStream_t st) {
  const std::uint32_t N = static_cast<std::uint32_t>(T.n_nodes);
  GK_CUDA(cudaMemsetAsync(arrive, 0, static_cast<std::size_t>(N) * 4, st));
  k_collapse_up<<<blocks_for(N), 256, 0, st>>>(N, T.canon, T.coords, T.orig, repl, arrive);
  k_relink<D><<<blocks_for(N), 256, 0, st>>>(N, T.canon, static_cast<TNode<D>*>(T.tnodes), T.irank, T.orig, repl);
  k_root_info<<<1, 1, 0, st>>>(repl, T.canon, T.irank, info);
  GK_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ driver --
int coresident_blocks(const void* fn) {
  int dev = 0, sms = 0, per = 0;
  GK_CUDA(cudaGetDevice(&dev));
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, 0));
  return std::max(1, per) * sms;
}

template <int D>
int capacity_d() {
  static int maxb[kMaxDevices] = {};  // per D and device
  const int dev = current_device();
  if (!maxb[dev])
    maxb[dev] = std::min(std::min(coresident_blocks(reinterpret_cast<const void*>(k_build<D, 0>)),
                                  coresident_blocks(reinterpret_cast<const void*>(k_build<D, 1>))),
                         coresident_blocks(reinterpret_cast<const void*>(k_merge<D>)));
  return maxb[dev];
}

// grid of a build running alone: co-resident blocks, fewer for small trees (barriers are
// cheaper with fewer blocks)
template <int D>
int grid_wanted_d(std::uint64_t n) {
  // one block per 2048 points (GK_GRID_DIV overrides): 4096 was the optimum while every chunk sent its
  // atomics to the node's words; with a warp's run of chunks accumulated in registers C1 Insert_L gains 4 %
  static const std::uint64_t div = std::getenv("GK_GRID_DIV") ? std::strtoull(std::getenv("GK_GRID_DIV"), nullptr, 10) : 2048;
  return static_cast<int>(std::min<std::uint64_t>(capacity_d<D>(), std::max<std::uint64_t>(1, n / div)));
}

// device scratch of one build (every array build_begin_d carves out of it, 256-byte aligned)
template <int D>
std::size_t scratch_bytes(std::uint64_t n, std::uint64_t cap_chunks, int G) {
  const std::uint64_t cap = 2 * n - 1, cap_level = std::min<std::uint64_t>(cap, n);
  return 2 * n * D * 8 + 2 * n * 4 + cap * (7 * 4 + 2 + 8 + 2 * D * 8) + 4 * (cap + 1) + (cap_level + 1) * 4 * 7 +
         cap_chunks * 4 * 4 + cap_level * D * 2 * 8 + (kMaxLevels + 2) * 4 + C_COUNT * 4 + kSelCap * sizeof(SelState) +
         kSelCap * 256 * 4 + (3 * G + 2) * 4 + 8 * (cap + 1) + 46 * 256;
}

// the bottom phase's arrays (small roots, subtree node records, merge scratch, merged level arrays)
template <int D>
std::size_t bottom_bytes(std::uint64_t n, int leaf) {
  const std::uint64_t cap = 2 * n - 1, rmax = n / (leaf + 1) + 1;
  return rmax * 4 * 4 + rmax * kSubLevels * 4 + 2 * n * (4 + 4 + 4 + 1 + 8 + 16 * D) + 2 * (n + 1) * 4 +
         (rmax * kVLevels + 1) * 4 + (kMaxLevels + 2) * 4 + cap * (4 + 4 + 1 + 1 + 8 + 16 * D) + 16 * 256;
}

// upper bound of the device memory one build allocates: its scratch (at the smallest chunk size) plus
// the tree it leaves behind (coordinates, ids, canonical + traversal nodes, topology, ranks)
template <int D>
std::size_t build_bytes_d(std::uint64_t n) {
  if (n == 0) return 0;
  const std::uint64_t cap = 2 * n - 1;
  const std::size_t tree = n * (8 * D + 4) + cap * (sizeof(gk_canon_node) + 12 + 4) + (cap / 2 + 1) * sizeof(TNode<D>);
  return scratch_bytes<D>(n, n / 32 + std::min<std::uint64_t>(cap, n) + 2, capacity_d<D>()) + bottom_bytes<D>(n, 4) +
         tree + 8 * 4096;
}

template <int D>
void build_begin_d(BuildScratch& sc, int leaf, int heuristic, const double* src, std::uint64_t src_stride,
                   const std::uint32_t* src_ids, std::uint64_t n, DevTree& T, cudaStream_t st, int max_grid,
                   std::uint64_t wave_max_n) {
  static_assert(sizeof(BuildArgs) <= sizeof(sc.args), "BuildScratch::args too small");
  sc.pending = false;
  T = DevTree();
  T.d = D;
  T.n = n;
  T.build_size = n;
  T.live = n;
  if (n == 0) return;
  if (n >= 0x7fffffffULL) throw Error(GK_ERR_INVALID, "static tree larger than 2^31-2 points");
  const std::uint64_t cap = 2 * n - 1;
  const std::uint64_t cap_level = std::min<std::uint64_t>(cap, n);

  T.coords = dalloc<double>(n * D, st);
  T.ids = dalloc<std::uint32_t>(n, st);

  const int G = max_grid > 0 ? std::min(max_grid, grid_wanted_d<D>(n)) : grid_wanted_d<D>(n);
  // chunk size: about kChunksPerWarp chunks per warp at the top levels, so the last round of
  // chunks is not a mostly idle one (8192 chunks of 1024 points over 3928 warps left 30 % idle)
  const std::uint64_t warps = static_cast<std::uint64_t>(G) * (kThreads / 32);
  const std::uint32_t kc = static_cast<std::uint32_t>(
      std::max<std::uint64_t>(32, ((n + kChunksPerWarp * warps - 1) / (kChunksPerWarp * warps) + 31) & ~std::uint64_t(31)));

  BuildArgs& a = *reinterpret_cast<BuildArgs*>(sc.args);
  a = BuildArgs();
  a.leaf = leaf;
  a.heuristic = heuristic;
  a.n = static_cast<std::uint32_t>(n);
  a.kc = kc;
  const std::uint64_t cap_chunks = n / kc + cap_level + 2;
  a.src = src;
  a.src_stride = src_stride;
  a.src_ids = src_ids;
  // bottom phase: both heuristics, leaves of >= 4 points (the per-level node arrays of a subtree are
  // sized for internal nodes of >= 5 points); GK_NO_SMALL=1 turns it off (A/B experiments)
  static const bool no_small = std::getenv("GK_NO_SMALL") != nullptr;
  static const std::uint64_t max_n = std::getenv("GK_SMALL_MAX_N") ? std::strtoull(std::getenv("GK_SMALL_MAX_N"), nullptr, 10)
                                                                   : small_max_n<D>();
  // (a wave of concurrent builds that contains a larger tree skips it for all its trees: the large tree's
  // level loop is the critical path and the small trees' subtree blocks only contend with it -- C2
  // Insert_L 6.3 ms with, 5.85 ms without)
  const bool bottom = !no_small && leaf >= 4 && leaf < small_cap<D>() && std::max(n, wave_max_n) <= max_n;
  const std::size_t need = scratch_bytes<D>(n, cap_chunks, G) + (bottom ? bottom_bytes<D>(n, leaf) : 0);
  char* base = sc.reserve(need, st);
  std::size_t used = 0;
  auto take = [&](std::size_t bytes) -> char* {
    used = (used + 255) & ~std::size_t(255);
    char* p = base + used;
    used += bytes;
    return p;
  };
  a.bufA = reinterpret_cast<double*>(take(n * D * 8));
  a.bufB = reinterpret_cast<double*>(take(n * D * 8));
  a.idsA = reinterpret_cast<std::uint32_t*>(take(n * 4));
  a.idsB = reinterpret_cast<std::uint32_t*>(take(n * 4));
  a.out = T.coords;
  a.out_ids = T.ids;
  NodeArrays& na = a.na;
  na.start = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.count = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.parent = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.cbase = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.nleft = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.pos = reinterpret_cast<std::uint32_t*>(take((cap + 1) * 4));
  na.thr_id = reinterpret_cast<std::uint32_t*>(take(cap * 4));
  na.flags = reinterpret_cast<std::uint8_t*>(take(cap));
  na.level = reinterpret_cast<std::uint8_t*>(take(cap));
  na.split = reinterpret_cast<double*>(take(cap * 8));
  na.lo = reinterpret_cast<double*>(take(cap * D * 8));
  na.hi = reinterpret_cast<double*>(take(cap * D * 8));
  a.lvl_off = reinterpret_cast<std::uint32_t*>(take((kMaxLevels + 2) * 4));
  a.ctrl = reinterpret_cast<std::uint32_t*>(take(C_COUNT * 4));
  a.chunk_off[0] = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.chunk_off[1] = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.ccnt = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.coff = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.is_int = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.irank = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.obj_list = reinterpret_cast<std::uint32_t*>(take((cap_level + 1) * 4));
  a.chunk_node[0] = reinterpret_cast<std::uint32_t*>(take(cap_chunks * 4));
  a.chunk_node[1] = reinterpret_cast<std::uint32_t*>(take(cap_chunks * 4));
  a.chunk_left = reinterpret_cast<std::uint32_t*>(take(cap_chunks * 4));
  a.left_scan = reinterpret_cast<std::uint32_t*>(take(cap_chunks * 4));
  a.keys = reinterpret_cast<unsigned long long*>(take(cap_level * D * 2 * 8));
  a.sel = reinterpret_cast<SelState*>(take(kSelCap * sizeof(SelState)));
  a.hist = reinterpret_cast<std::uint32_t*>(take(kSelCap * 256 * 4));
  a.bsum = reinterpret_cast<std::uint32_t*>(take((3 * G + 2) * 4));
  a.int_by_slot = reinterpret_cast<std::uint32_t*>(take((cap + 1) * 4));
  a.irank_slot = reinterpret_cast<std::uint32_t*>(take((cap + 1) * 4));
  a.Tsmall = bottom ? static_cast<std::uint32_t>(small_cap<D>()) : 0u;
  if (bottom) {
    const std::uint64_t rmax = n / (leaf + 1) + 1;
    a.rmax = static_cast<std::uint32_t>(rmax);
    a.small_list = reinterpret_cast<std::uint32_t*>(take(rmax * 4));
    a.sub_base = reinterpret_cast<std::uint32_t*>(take(rmax * 4));
    a.sub_nlev = reinterpret_cast<std::uint32_t*>(take(rmax * 4));
    a.order = reinterpret_cast<std::uint32_t*>(take(rmax * 4));
    a.sub_cnt = reinterpret_cast<std::uint32_t*>(take(rmax * kSubLevels * 4));
    a.s_start = reinterpret_cast<std::uint32_t*>(take(2 * n * 4));
    a.s_count = reinterpret_cast<std::uint32_t*>(take(2 * n * 4));
    a.s_child = reinterpret_cast<std::uint32_t*>(take(2 * n * 4));
    a.s_flags = reinterpret_cast<std::uint8_t*>(take(2 * n));
    a.s_split = reinterpret_cast<double*>(take(2 * n * 8));
    a.s_lo = reinterpret_cast<double*>(take(2 * n * D * 8));
    a.s_hi = reinterpret_cast<double*>(take(2 * n * D * 8));
    a.marks = reinterpret_cast<std::uint32_t*>(take((n + 1) * 4));
    a.mscan = reinterpret_cast<std::uint32_t*>(take((n + 1) * 4));
    a.vcap = static_cast<std::uint32_t>(std::min<std::uint64_t>(rmax * kVLevels, 0xfffffff0ULL));
    a.V = reinterpret_cast<std::uint32_t*>(take((static_cast<std::uint64_t>(a.vcap) + 1) * 4));
    a.new_off = reinterpret_cast<std::uint32_t*>(take((kMaxLevels + 2) * 4));
    NodeArrays& nb = a.na2;
    nb.start = reinterpret_cast<std::uint32_t*>(take(cap * 4));
    nb.count = reinterpret_cast<std::uint32_t*>(take(cap * 4));
    nb.flags = reinterpret_cast<std::uint8_t*>(take(cap));
    nb.level = reinterpret_cast<std::uint8_t*>(take(cap));
    nb.split = reinterpret_cast<double*>(take(cap * 8));
    nb.lo = reinterpret_cast<double*>(take(cap * D * 8));
    nb.hi = reinterpret_cast<double*>(take(cap * D * 8));
    nb.parent = na.parent;  // recomputed by k_merge; the level loop's values are dead by then
    nb.cbase = na.cbase;
    nb.pos = na.pos;
    nb.nleft = na.nleft;
    nb.thr_id = na.thr_id;
  }
  if (used > need) throw Error(GK_ERR_LOGIC, "BuildvEB_S scratch accounting");

  void* args[] = {&a};
  GK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_build<D, 0>), dim3(G), dim3(kThreads), args, 0, st));
  GK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_build<D, 1>), dim3(G), dim3(kThreads), args, 0, st));
  if (bottom) {  // the subtrees of the small nodes (one block each), then the merge + vEB phase
    static std::once_flag once[kMaxDevices];
    static int sub_resident[kMaxDevices] = {};
    const int dev = current_device();
    std::call_once(once[dev], [&] {
      GK_CUDA(cudaFuncSetAttribute(k_subtree<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(small_smem<D>())));
      int sms = 0, per = 0;
      GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_subtree<D>, kSubThreads, small_smem<D>()));
      sub_resident[dev] = std::max(1, per) * sms;
    });
    const unsigned sg = static_cast<unsigned>(std::min<std::uint64_t>(sub_resident[dev], n / (leaf + 1) + 1));
    k_subtree<D><<<sg, kSubThreads, small_smem<D>(), st>>>(a);
    GK_CHECK_LAUNCH();
    GK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_merge<D>), dim3(G), dim3(kThreads), args, 0, st));
  }
  GK_CUDA(cudaMemcpyAsync(sc.host_ctrl, a.ctrl, C_COUNT * 4, cudaMemcpyDeviceToHost, st));
  sc.d = D;
  sc.grid = G;
  sc.n = n;
  sc.out = &T;
  sc.st = st;
  sc.pending = true;
}

template <int D>
void build_finish_d(BuildScratch& sc) {
  sc.pending = false;
  BuildArgs& a = *reinterpret_cast<BuildArgs*>(sc.args);
  DevTree& T = *sc.out;
  cudaStream_t st = sc.st;
  const std::uint64_t n = sc.n;
  GK_CUDA(cudaStreamSynchronize(st));
  const int H = static_cast<int>(sc.host_ctrl[C_H]);
  const std::uint32_t N = sc.host_ctrl[C_N];
  if (H >= kMaxLevels) throw Error(GK_ERR_LOGIC, "BuildvEB_S: tree deeper than 256 levels");
  T.height = H;
  T.n_nodes = N;
  T.n_internal = (N - 1) / 2;
  T.irank = dalloc<std::uint32_t>(static_cast<std::uint64_t>(N) + 1, st);
  T.canon = dalloc<gk_canon_node>(N, st);
  T.tnodes = dalloc<TNode<D>>(T.n_internal, st);
  T.orig = dalloc<std::int32_t>(3 * static_cast<std::uint64_t>(N), st);
  GK_CUDA(cudaMemsetAsync(T.orig + 2 * static_cast<std::uint64_t>(N), 0xff, 4, st));  // parent(root) = -1
  BuildArgs ea = a;  // after the bottom phase the merged level arrays are a.na2
  if (sc.host_ctrl[C_NSMALL] > 0) ea.na = a.na2;
  k_emit<D><<<(N + 1 + kEmitThreads - 1) / kEmitThreads, kEmitThreads, 0, st>>>(ea, N, T.irank, T.canon, static_cast<TNode<D>*>(T.tnodes), T.orig);
  GK_CHECK_LAUNCH();
  T.root_ref = (N == 1) ? make_leaf_ref(0, static_cast<std::uint32_t>(n)) : 0;
  T.root_slot = 0;
  GK_CUDA(cudaFreeAsync(sc.base, st));
  sc.base = nullptr;
}

}  // namespace

BuildScratch::~BuildScratch() {
  if (host_ctrl) cudaFreeHost(host_ctrl);
}

// stream-ordered scratch from the device memory pool (cached across builds and handles)
char* BuildScratch::reserve(std::size_t bytes, cudaStream_t st) {
  if (!host_ctrl) GK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&host_ctrl), 64));
  GK_CUDA(cudaMallocAsync(&base, bytes, st));
  size = bytes;
  return static_cast<char*>(base);
}

void build_begin(BuildScratch& sc, int d, int leaf, int heuristic, const double* src, std::uint64_t src_stride,
                 const std::uint32_t* src_ids, std::uint64_t n, DevTree& out, cudaStream_t st, int max_grid,
                 std::uint64_t wave_max_n) {
  switch (d) {
    case 2: build_begin_d<2>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 3: build_begin_d<3>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 4: build_begin_d<4>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 5: build_begin_d<5>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 6: build_begin_d<6>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 7: build_begin_d<7>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    case 8: build_begin_d<8>(sc, leaf, heuristic, src, src_stride, src_ids, n, out, st, max_grid, wave_max_n); break;
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

int build_capacity(int d) {
  switch (d) {
    case 2: return capacity_d<2>();
    case 3: return capacity_d<3>();
    case 4: return capacity_d<4>();
    case 5: return capacity_d<5>();
    case 6: return capacity_d<6>();
    case 7: return capacity_d<7>();
    case 8: return capacity_d<8>();
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

std::size_t build_bytes(int d, std::uint64_t n) {
  switch (d) {
    case 2: return build_bytes_d<2>(n);
    case 3: return build_bytes_d<3>(n);
    case 4: return build_bytes_d<4>(n);
    case 5: return build_bytes_d<5>(n);
    case 6: return build_bytes_d<6>(n);
    case 7: return build_bytes_d<7>(n);
    case 8: return build_bytes_d<8>(n);
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

int build_grid_wanted(int d, std::uint64_t n) {
  switch (d) {
    case 2: return grid_wanted_d<2>(n);
    case 3: return grid_wanted_d<3>(n);
    case 4: return grid_wanted_d<4>(n);
    case 5: return grid_wanted_d<5>(n);
    case 6: return grid_wanted_d<6>(n);
    case 7: return grid_wanted_d<7>(n);
    case 8: return grid_wanted_d<8>(n);
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

void build_finish(BuildScratch& sc) {
  if (!sc.pending) return;
  switch (sc.d) {
    case 2: build_finish_d<2>(sc); break;
    case 3: build_finish_d<3>(sc); break;
    case 4: build_finish_d<4>(sc); break;
    case 5: build_finish_d<5>(sc); break;
    case 6: build_finish_d<6>(sc); break;
    case 7: build_finish_d<7>(sc); break;
    case 8: build_finish_d<8>(sc); break;
    default: throw Error(GK_ERR_INVALID, "unsupported dimension");
  }
}

void collapse_tree(int d, DevTree& t, cudaStream_t st) {
  switch (d) {
    case 2: collapse_d<2>(t, st); break;
    case 3: collapse_d<3>(t, st); break;
    case 4: collapse_d<4>(t, st); break;
    case 5: collapse_d<5>(t, st); break;
    case 6: collapse_d<6>(t, st); break;
    case 7: collapse_d<7>(t, st); break;
    case 8: collapse_d<8>(t, st); break;
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

// Erase_S collapses of several trees with one host round-trip for all their new roots
void collapse_trees_begin(CollapseJob& job, int d, const std::vector<DevTree*>& trees, cudaStream_t st,
                          cudaStream_t* side, int nside) {
  job = CollapseJob();
  job.st = st;
  for (DevTree* t : trees)
    if (t->n_nodes) job.ts.push_back(t);
  if (job.ts.empty()) return;
  const std::size_t m = job.ts.size();
  job.info = dalloc<std::uint32_t>(5 * m, st);
  job.repl.resize(m);
  job.arrive.resize(m);
  for (std::size_t i = 0; i < m; ++i) {  // stream-ordered on st; the side streams start after the fork event
    job.repl[i] = dalloc<std::int32_t>(job.ts[i]->n_nodes, st);
    job.arrive[i] = dalloc<std::uint32_t>(job.ts[i]->n_nodes, st);
  }
  const bool fork = side && nside > 0;
  if (fork) {
    job.ev.resize(m + 1);
    for (auto& e : job.ev) GK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    GK_CUDA(cudaEventRecord(job.ev[0], st));
  }
  for (std::size_t i = 0; i < m; ++i) {
    cudaStream_t s = st;
    if (fork) {
      s = side[i % static_cast<std::size_t>(nside)];
      GK_CUDA(cudaStreamWaitEvent(s, job.ev[0], 0));
    }
    switch (d) {
#define GK_D(DD) case DD: collapse_launch<DD>(*job.ts[i], job.repl[i], job.arrive[i], job.info + 5 * i, s); break;
      GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
      default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
    }
    if (fork) GK_CUDA(cudaEventRecord(job.ev[1 + i], s));
  }
}

void collapse_trees_finish(CollapseJob& job) {
  if (job.ts.empty()) return;
  cudaStream_t st = job.st;
  const std::size_t m = job.ts.size();
  for (std::size_t i = 1; i < job.ev.size(); ++i) GK_CUDA(cudaStreamWaitEvent(st, job.ev[i], 0));
  for (auto& e : job.ev) GK_CUDA(cudaEventDestroy(e));
  job.ev.clear();
  std::vector<std::uint32_t> h(5 * m);
  GK_CUDA(cudaMemcpyAsync(h.data(), job.info, 5 * m * 4, cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  for (std::size_t i = 0; i < m; ++i) {
    DevTree& T = *job.ts[i];
    const std::int32_t root = static_cast<std::int32_t>(h[5 * i]);
    T.root_slot = root;
    if (root >= 0) T.root_ref = h[5 * i + 1] == 1 ? make_leaf_ref(h[5 * i + 2], h[5 * i + 3]) : h[5 * i + 4];
    dfree(job.repl[i], st);
    dfree(job.arrive[i], st);
  }
  dfree(job.info, st);
  job.ts.clear();
}

void collapse_trees(int d, const std::vector<DevTree*>& trees, cudaStream_t st, cudaStream_t* side, int nside) {
  CollapseJob job;
  collapse_trees_begin(job, d, trees, st, side, nside);
  collapse_trees_finish(job);
}

void free_tree(DevTree& t, cudaStream_t st) {
  dfree(t.coords, st);
  dfree(t.ids, st);
  if (t.tnodes) GK_CUDA(cudaFreeAsync(t.tnodes, st));
  t.tnodes = nullptr;
  dfree(t.canon, st);
  dfree(t.orig, st);
  dfree(t.irank, st);
  dfree(t.bloom, st);
  t = DevTree();
}

}  // namespace gk
