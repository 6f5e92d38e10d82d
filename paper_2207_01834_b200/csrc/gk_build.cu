// gk_build.cu — BuildvEB_S on the B200 (sm_100a): a level-synchronous pipeline.
//
// Reference semantics (restated; the reference ships no code for it):
//   PAPER.md:1110-1127 Alg. 1 BuildvEB_S, 1141-1146 recursion, 1484-1487 spatial
//   median = (min+max)/2, 1491 leaf 16.
// Frozen decisions (mirrored by oracle/gk_oracle.cpp):
//   split dim = depth mod D; spatial split s = (lo+hi)/2, left x_c < s <= right;
//   stable partition; degenerate side or depth >= 40 or heuristic = object ->
//   object median by (x_c, id), left = the floor(n/2) smallest keys; leaf when
//   n <= leaf; vEB layout topology-driven (complete-tree vEB order restricted
//   to the nodes that exist).
//
// Device pipeline per level L (all nodes of the level at once, any number of trees' worth of segments):
//   chunking   -> each node's point range is cut into <=1024-point chunks, one warp per chunk
//   k_bbox     -> per-node bounding box: coalesced fp64 loads, warp min/max, one atomic per chunk
//   k_split    -> node record: leaf / spatial split / object-median flag
//   k_count    -> per-chunk left counts (ballot+popc) + per-node totals
//   k_check    -> degenerate spatial splits fall back to object median
//   radix      -> (object nodes only) 12 x 8-bit MSD radix select of the (x_c, id) median
//   scan       -> CUB exclusive scan of the chunk left counts
//   k_children -> child node records in left-to-right (BFS) order
//   k_scatter  -> stable partition into the ping-pong buffer; finished leaves written in place
// then k_veb (per level, top-down) computes each node's vEB slot and k_emit writes
// the canonical node array and the traversal nodes (TNode) in vEB order.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gk_common.cuh"

namespace gk {
namespace {

constexpr std::uint8_t F_LEAF = 1, F_OBJECT = 2;

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

// ------------------------------------------------------------------ chunks --
__global__ void k_chunk_counts(const std::uint32_t* __restrict__ count, std::uint32_t S, std::uint32_t* out) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < S) out[v] = (count[v] + kChunk - 1) / kChunk;
  else if (v == S) out[v] = 0;
}

__global__ void k_chunk_node(const std::uint32_t* __restrict__ chunk_off, std::uint32_t S, std::uint32_t* chunk_node) {
  const std::uint32_t total = chunk_off[S];
  for (std::uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    std::uint32_t lo = 0, hi = S;  // largest v with chunk_off[v] <= c
    while (hi - lo > 1) {
      std::uint32_t mid = (lo + hi) >> 1;
      if (chunk_off[mid] <= c) lo = mid; else hi = mid;
    }
    chunk_node[c] = lo;
  }
}

struct ChunkIt {
  std::uint32_t v, first, len;
};
__device__ __forceinline__ ChunkIt chunk_at(std::uint32_t c, const std::uint32_t* chunk_off, const std::uint32_t* chunk_node,
                                            const std::uint32_t* start, const std::uint32_t* count, std::uint32_t off) {
  ChunkIt it;
  it.v = chunk_node[c];
  std::uint32_t g = off + it.v;
  std::uint32_t s = start[g], n = count[g];
  it.first = s + (c - chunk_off[it.v]) * kChunk;
  it.len = min(static_cast<std::uint32_t>(kChunk), s + n - it.first);
  return it;
}

// -------------------------------------------------------------------- bbox --
__global__ void k_bbox_init(unsigned long long* keys, std::uint32_t n_keys_half) {
  std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_keys_half) { keys[2 * i] = ~0ULL; keys[2 * i + 1] = 0ULL; }
}

template <int D>
__global__ void __launch_bounds__(256) k_bbox(const double* __restrict__ cur, std::uint64_t stride,
                                              const std::uint32_t* __restrict__ chunk_off,
                                              const std::uint32_t* __restrict__ chunk_node, std::uint32_t S,
                                              std::uint32_t off, NodeArrays na, unsigned long long* keys) {
  const std::uint32_t total = chunk_off[S];
  const int lane = threadIdx.x & 31;
  const std::uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (std::uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < total; c += nw) {
    ChunkIt it = chunk_at(c, chunk_off, chunk_node, na.start, na.count, off);
    double lo[D], hi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { lo[j] = __longlong_as_double(0x7ff0000000000000LL); hi[j] = -lo[j]; }
    for (std::uint32_t i = it.first + lane; i < it.first + it.len; i += 32) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double x = cur[j * stride + i];
        lo[j] = fmin(lo[j], x);
        hi[j] = fmax(hi[j], x);
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo[j] = fmin(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], o));
        hi[j] = fmax(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], o));
      }
    }
    if (lane < D) {
      double l = lo[0], h = hi[0];
#pragma unroll
      for (int j = 1; j < D; ++j)
        if (lane == j) { l = lo[j]; h = hi[j]; }
      unsigned long long* kk = keys + (static_cast<std::uint64_t>(it.v) * D + lane) * 2;
      atomicMin(kk, dkey(l));
      atomicMax(kk + 1, dkey(h));
    }
  }
}

// ------------------------------------------------------------------- split --
template <int D>
__global__ void k_split(std::uint32_t S, std::uint32_t off, int level, int leaf, int heuristic,
                        const unsigned long long* __restrict__ keys, NodeArrays na) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= S) return;
  const std::uint32_t g = off + v;
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = dkey_inv(keys[(static_cast<std::uint64_t>(v) * D + j) * 2]);
    hi[j] = dkey_inv(keys[(static_cast<std::uint64_t>(v) * D + j) * 2 + 1]);
    na.lo[static_cast<std::uint64_t>(g) * D + j] = lo[j];
    na.hi[static_cast<std::uint64_t>(g) * D + j] = hi[j];
  }
  na.nleft[g] = 0;
  na.level[g] = static_cast<std::uint8_t>(level);
  if (na.count[g] <= static_cast<std::uint32_t>(leaf)) {
    na.flags[g] = F_LEAF;
    na.split[g] = 0.0;
    return;
  }
  const int c = level % D;
  if (heuristic == GK_OBJECT_MEDIAN || level >= kDepthCap) {
    na.flags[g] = F_OBJECT;
    na.split[g] = 0.0;
  } else {
    na.flags[g] = 0;
    double l = lo[0], h = hi[0];
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (c == j) { l = lo[j]; h = hi[j]; }
    na.split[g] = __dmul_rn(__dadd_rn(l, h), 0.5);  // (lo + hi) / 2 exactly
  }
}

// ------------------------------------------------------------------- count --
// pass 0: spatial nodes (x_c < s); pass 1: object nodes ((x_c, id) < threshold)
template <int D>
__global__ void __launch_bounds__(256) k_count(const double* __restrict__ cur, const std::uint32_t* __restrict__ cur_ids,
                                               std::uint64_t stride, const std::uint32_t* __restrict__ chunk_off,
                                               const std::uint32_t* __restrict__ chunk_node, std::uint32_t S,
                                               std::uint32_t off, int level, int pass, NodeArrays na,
                                               std::uint32_t* chunk_left) {
  const std::uint32_t total = chunk_off[S];
  const int lane = threadIdx.x & 31;
  const std::uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const int cdim = level % D;
  for (std::uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < total; c += nw) {
    ChunkIt it = chunk_at(c, chunk_off, chunk_node, na.start, na.count, off);
    const std::uint32_t g = off + it.v;
    const std::uint8_t fl = na.flags[g];
    if (fl & F_LEAF) { if (pass == 0 && lane == 0) chunk_left[c] = 0; continue; }
    const bool obj = (fl & F_OBJECT) != 0;
    if (pass == 0 && obj) { if (lane == 0) chunk_left[c] = 0; continue; }
    if (pass == 1 && !obj) continue;
    const double s = na.split[g];
    const std::uint32_t tid = na.thr_id[g];
    const double* xc = cur + cdim * stride;
    std::uint32_t cnt = 0;
    for (std::uint32_t i0 = it.first; i0 < it.first + it.len; i0 += 32) {
      const std::uint32_t i = i0 + lane;
      bool p = false;
      if (i < it.first + it.len) {
        double x = xc[i];
        p = obj ? (x < s || (x == s && cur_ids[i] < tid)) : (x < s);
      }
      cnt += __popc(__ballot_sync(0xffffffffu, p));
    }
    if (lane == 0) {
      chunk_left[c] = cnt;
      if (pass == 0) atomicAdd(&na.nleft[g], cnt);
    }
  }
}

// degenerate spatial splits -> object median; internal flags for the BFS scan
__global__ void k_check(std::uint32_t S, std::uint32_t off, NodeArrays na, std::uint32_t* is_int,
                        std::uint32_t* obj_list, std::uint32_t* counters) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v == S) is_int[S] = 0;
  if (v >= S) return;
  const std::uint32_t g = off + v;
  std::uint8_t fl = na.flags[g];
  if (fl & F_LEAF) { is_int[v] = 0; return; }
  is_int[v] = 1;
  if (!(fl & F_OBJECT)) {
    std::uint32_t nl = na.nleft[g];
    if (nl == 0 || nl == na.count[g]) { fl |= F_OBJECT; na.flags[g] = fl; }
  }
  if (fl & F_OBJECT) {
    std::uint32_t o = atomicAdd(&counters[0], 1u);
    obj_list[o] = g;
    na.nleft[g] = na.count[g] / 2;
    na.pos[g] = o;  // temporary: object index (pos is recomputed by k_veb)
  }
}

// ------------------------------------------------------- object median select --
struct SelState {
  unsigned long long hi;  // known high digits of dkey(x_c)
  std::uint32_t lo;       // known digits of the id
  std::uint32_t rank;     // rank still to skip inside the current prefix bucket
};

__global__ void k_sel_init(std::uint32_t nobj, const std::uint32_t* obj_list, NodeArrays na, SelState* st) {
  std::uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nobj) return;
  st[o].hi = 0; st[o].lo = 0; st[o].rank = na.count[obj_list[o]] / 2;
}

// digit p in 0..11: p < 8 -> byte (7-p) of the 64-bit key, else byte (11-p) of the id
template <int D>
__global__ void __launch_bounds__(256) k_sel_hist(const double* __restrict__ cur, const std::uint32_t* __restrict__ cur_ids,
                                                  std::uint64_t stride, const std::uint32_t* __restrict__ chunk_off,
                                                  const std::uint32_t* __restrict__ chunk_node, std::uint32_t S,
                                                  std::uint32_t off, int level, int p, NodeArrays na,
                                                  const SelState* __restrict__ st, std::uint32_t* hist) {
  const std::uint32_t total = chunk_off[S];
  const int lane = threadIdx.x & 31;
  const std::uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const int cdim = level % D;
  for (std::uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < total; c += nw) {
    ChunkIt it = chunk_at(c, chunk_off, chunk_node, na.start, na.count, off);
    const std::uint32_t g = off + it.v;
    if ((na.flags[g] & (F_LEAF | F_OBJECT)) != F_OBJECT) continue;
    const std::uint32_t o = na.pos[g];
    const SelState s = st[o];
    for (std::uint32_t i0 = it.first; i0 < it.first + it.len; i0 += 32) {
      const std::uint32_t i = i0 + lane;
      int digit = -1;
      if (i < it.first + it.len) {
        unsigned long long k = dkey(__dadd_rn(cur[cdim * stride + i], 0.0));  // -0 == +0 as in the oracle
        std::uint32_t id = cur_ids[i];
        bool match;
        if (p < 8) {
          const int sh = 8 * (8 - p);  // bits above the current digit
          match = (sh >= 64) ? true : ((k >> sh) == (s.hi >> sh));
          digit = static_cast<int>((k >> (8 * (7 - p))) & 0xff);
        } else {
          const int q = p - 8;
          const int sh = 8 * (4 - q);
          match = (k == s.hi) && ((sh >= 32) ? true : ((id >> sh) == (s.lo >> sh)));
          digit = static_cast<int>((id >> (8 * (3 - q))) & 0xff);
        }
        if (!match) digit = -1;
      }
      unsigned peers = __match_any_sync(0xffffffffu, digit);
      int leader = __ffs(peers) - 1;
      if (digit >= 0 && lane == leader) atomicAdd(&hist[o * 256 + digit], __popc(peers));
    }
  }
}

__global__ void k_sel_pick(std::uint32_t nobj, int p, SelState* st, std::uint32_t* hist) {
  std::uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nobj) return;
  SelState s = st[o];
  std::uint32_t* h = hist + o * 256;
  std::uint32_t acc = 0;
  int dsel = 255;
  for (int dgt = 0; dgt < 256; ++dgt) {
    std::uint32_t c = h[dgt];
    if (s.rank < acc + c) { dsel = dgt; break; }
    acc += c;
  }
  s.rank -= acc;
  if (p < 8) s.hi |= static_cast<unsigned long long>(dsel) << (8 * (7 - p));
  else s.lo |= static_cast<std::uint32_t>(dsel) << (8 * (3 - (p - 8)));
  st[o] = s;
  for (int dgt = 0; dgt < 256; ++dgt) h[dgt] = 0;
}

__global__ void k_sel_finish(std::uint32_t nobj, const std::uint32_t* obj_list, const SelState* st, NodeArrays na) {
  std::uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nobj) return;
  const std::uint32_t g = obj_list[o];
  na.split[g] = dkey_inv(st[o].hi);  // canonical +0 for a zero median
  na.thr_id[g] = st[o].lo;
}

// ---------------------------------------------------------------- children --
__global__ void k_children(std::uint32_t S, std::uint32_t off, std::uint32_t next_off, const std::uint32_t* __restrict__ irank,
                           NodeArrays na) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= S) return;
  const std::uint32_t g = off + v;
  const std::uint32_t cb = next_off + 2 * irank[v];
  na.cbase[g] = cb;
  if (na.flags[g] & F_LEAF) return;
  const std::uint32_t s = na.start[g], n = na.count[g], nl = na.nleft[g];
  na.start[cb] = s; na.count[cb] = nl; na.parent[cb] = g;
  na.start[cb + 1] = s + nl; na.count[cb + 1] = n - nl; na.parent[cb + 1] = g;
}

// ----------------------------------------------------------------- scatter --
template <int D>
__global__ void __launch_bounds__(256) k_scatter(const double* __restrict__ cur, const std::uint32_t* __restrict__ cur_ids,
                                                 std::uint64_t stride, double* __restrict__ nxt,
                                                 std::uint32_t* __restrict__ nxt_ids, double* __restrict__ out,
                                                 std::uint32_t* __restrict__ out_ids, std::uint64_t n,
                                                 const std::uint32_t* __restrict__ chunk_off,
                                                 const std::uint32_t* __restrict__ chunk_node,
                                                 const std::uint32_t* __restrict__ left_scan, std::uint32_t S,
                                                 std::uint32_t off, int level, NodeArrays na) {
  const std::uint32_t total = chunk_off[S];
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const std::uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const int cdim = level % D;
  for (std::uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < total; c += nw) {
    ChunkIt it = chunk_at(c, chunk_off, chunk_node, na.start, na.count, off);
    const std::uint32_t g = off + it.v;
    const std::uint8_t fl = na.flags[g];
    const std::uint32_t end = it.first + it.len;
    if (fl & F_LEAF) {  // finished: positions are final
      for (std::uint32_t i = it.first + lane; i < end; i += 32) {
#pragma unroll
        for (int j = 0; j < D; ++j) out[j * n + i] = cur[j * stride + i];
        out_ids[i] = cur_ids[i];
      }
      continue;
    }
    const bool obj = (fl & F_OBJECT) != 0;
    const double s = na.split[g];
    const std::uint32_t tid = na.thr_id[g];
    const std::uint32_t nstart = na.start[g], nl = na.nleft[g];
    std::uint32_t lbefore = left_scan[c] - left_scan[chunk_off[it.v]];
    for (std::uint32_t i0 = it.first; i0 < end; i0 += 32) {
      const std::uint32_t i = i0 + lane;
      bool valid = i < end;
      bool p = false;
      double x[D];
      std::uint32_t id = 0;
      if (valid) {
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = cur[j * stride + i];
        id = cur_ids[i];
        double xc = x[0];
#pragma unroll
        for (int j = 1; j < D; ++j)
          if (cdim == j) xc = x[j];
        p = obj ? (xc < s || (xc == s && id < tid)) : (xc < s);
      }
      unsigned b = __ballot_sync(0xffffffffu, p);
      if (valid) {
        std::uint32_t lrank = lbefore + __popc(b & lt_mask);
        std::uint32_t np = p ? nstart + lrank : nstart + nl + (i - nstart - lrank);
#pragma unroll
        for (int j = 0; j < D; ++j) nxt[j * n + np] = x[j];
        nxt_ids[np] = id;
      }
      lbefore += __popc(b);
    }
  }
}

// -------------------------------------------------------------------- vEB --
__device__ __forceinline__ std::uint32_t child_idx(std::uint32_t x, int e, const std::uint32_t* lvl_off,
                                                   const std::uint32_t* cbase) {
  return (x < lvl_off[e + 1]) ? cbase[x] : lvl_off[e + 2];
}

// vEB slot of every node at depth d: d is the cut depth of frame (d0, l) whose
// root r is d's ancestor at depth d0; pos = pos(r) + |top part| + sizes of the
// bottom subtrees left of v's (all sizes restricted to the frame's levels).
__global__ void k_veb(int d, int d0, int l, const std::uint32_t* __restrict__ lvl_off, NodeArrays na) {
  const std::uint32_t off = lvl_off[d];
  const std::uint32_t S = lvl_off[d + 1] - off;
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= S) return;
  const std::uint32_t g = off + v;
  std::uint32_t r = g;
  for (int e = d; e > d0; --e) r = na.parent[r];
  std::uint32_t lo = r, hi = r + 1, top = 0;
  for (int e = d0; e < d; ++e) {
    top += hi - lo;
    lo = child_idx(lo, e, lvl_off, na.cbase);
    hi = child_idx(hi, e, lvl_off, na.cbase);
  }
  std::uint32_t a = g, b = lo, left = 0;
  for (int e = d; e < d0 + l; ++e) {
    left += a - b;
    if (e + 1 < d0 + l) {
      a = child_idx(a, e, lvl_off, na.cbase);
      b = child_idx(b, e, lvl_off, na.cbase);
    }
  }
  na.pos[g] = na.pos[r] + top + left;
}

__global__ void k_slot_flags(std::uint32_t N, NodeArrays na, std::uint32_t* int_by_slot) {
  std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g == N) int_by_slot[N] = 0;
  if (g >= N) return;
  int_by_slot[na.pos[g]] = (na.flags[g] & F_LEAF) ? 0u : 1u;
}

template <int D>
__global__ void k_emit(std::uint32_t N, NodeArrays na, const std::uint32_t* __restrict__ irank_by_slot,
                       gk_canon_node* canon, TNode<D>* tn, std::int32_t* orig) {
  std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= N) return;
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
  for (int j = 0; j < 8; ++j) {
    c.lo[j] = j < D ? na.lo[static_cast<std::uint64_t>(g) * D + j] : 0.0;
    c.hi[j] = j < D ? na.hi[static_cast<std::uint64_t>(g) * D + j] : 0.0;
  }
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
        t.lo[s][j] = __double2float_rd(na.lo[static_cast<std::uint64_t>(ch) * D + j]);
        t.hi[s][j] = __double2float_ru(na.hi[static_cast<std::uint64_t>(ch) * D + j]);
      }
      t.ref[s] = (na.flags[ch] & F_LEAF) ? make_leaf_ref(na.start[ch], na.count[ch])
                                         : static_cast<std::uint64_t>(irank_by_slot[na.pos[ch]]);
    }
    tn[irank_by_slot[slot]] = t;
  }
  canon[slot] = c;
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

struct Scratch {
  void* cub = nullptr;
  std::size_t cub_bytes = 0;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() { if (cub) cudaFreeAsync(cub, st); }
  void scan(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n) {
    std::size_t need = 0;
    GK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, static_cast<int>(n), st));
    if (need > cub_bytes) {
      if (cub) GK_CUDA(cudaFreeAsync(cub, st));
      cub_bytes = std::max(need, cub_bytes * 2);
      GK_CUDA(cudaMallocAsync(&cub, cub_bytes, st));
    }
    GK_CUDA(cub::DeviceScan::ExclusiveSum(cub, need, in, out, static_cast<int>(n), st));
  }
};

inline unsigned blocks_for(std::uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// cut frame (d0, l) for every depth 1..H-1 of the vEB recursion over H levels
void veb_cuts(int d0, int l, std::vector<std::pair<int, int>>& cut) {
  if (l <= 1) return;
  int lb = static_cast<int>(hyperceiling_u(static_cast<std::uint64_t>((l + 1) / 2)));
  int lt = l - lb;
  cut[d0 + lt] = {d0, l};
  veb_cuts(d0, lt, cut);
  veb_cuts(d0 + lt, lb, cut);
}

template <int D>
void build_tree_d(int leaf, int heuristic, const double* src, std::uint64_t src_stride, const std::uint32_t* src_ids,
                  std::uint64_t n, DevTree& T, cudaStream_t st) {
  T = DevTree();
  T.d = D;
  T.n = n;
  T.build_size = n;
  T.live = n;
  if (n == 0) return;
  if (n >= 0xffffffffULL) throw Error(GK_ERR_INVALID, "static tree larger than 2^32-2 points");
  const std::uint64_t cap = 2 * n - 1;
  const int grid_w = 148 * 16;  // persistent-style grid for the chunk passes (8 warps x 16 blocks per SM)

  T.coords = dalloc<double>(n * D, st);
  T.ids = dalloc<std::uint32_t>(n, st);
  double* bufA = dalloc<double>(n * D, st);
  double* bufB = dalloc<double>(n * D, st);
  std::uint32_t* idsA = dalloc<std::uint32_t>(n, st);
  std::uint32_t* idsB = dalloc<std::uint32_t>(n, st);

  NodeArrays na;
  na.start = dalloc<std::uint32_t>(cap, st);
  na.count = dalloc<std::uint32_t>(cap, st);
  na.parent = dalloc<std::uint32_t>(cap, st);
  na.cbase = dalloc<std::uint32_t>(cap, st);
  na.nleft = dalloc<std::uint32_t>(cap, st);
  na.pos = dalloc<std::uint32_t>(cap + 1, st);
  na.thr_id = dalloc<std::uint32_t>(cap, st);
  na.flags = dalloc<std::uint8_t>(cap, st);
  na.level = dalloc<std::uint8_t>(cap, st);
  na.split = dalloc<double>(cap, st);
  na.lo = dalloc<double>(cap * D, st);
  na.hi = dalloc<double>(cap * D, st);

  const std::uint64_t cap_level = std::min<std::uint64_t>(cap, n);  // nodes in one level <= n
  const std::uint64_t cap_chunks = n / kChunk + cap_level + 2;
  std::uint32_t* chunk_cnt = dalloc<std::uint32_t>(cap_level + 1, st);
  std::uint32_t* chunk_off = dalloc<std::uint32_t>(cap_level + 1, st);
  std::uint32_t* chunk_node = dalloc<std::uint32_t>(cap_chunks, st);
  std::uint32_t* chunk_left = dalloc<std::uint32_t>(cap_chunks + 1, st);
  std::uint32_t* left_scan = dalloc<std::uint32_t>(cap_chunks + 1, st);
  std::uint32_t* is_int = dalloc<std::uint32_t>(cap_level + 1, st);
  std::uint32_t* irank = dalloc<std::uint32_t>(cap_level + 1, st);
  std::uint32_t* obj_list = dalloc<std::uint32_t>(cap_level, st);
  unsigned long long* keys = dalloc<unsigned long long>(cap_level * D * 2, st);
  std::uint32_t* counters = dalloc<std::uint32_t>(4, st);
  std::uint32_t* h_counters = nullptr;
  GK_CUDA(cudaMallocHost(&h_counters, 4 * sizeof(std::uint32_t)));
  SelState* sel = nullptr;
  std::uint32_t* hist = nullptr;
  std::uint64_t sel_cap = 0;
  Scratch scratch(st);

  // root
  std::uint32_t zero = 0, n32 = static_cast<std::uint32_t>(n), none = 0xffffffffu;
  GK_CUDA(cudaMemcpyAsync(na.start, &zero, 4, cudaMemcpyHostToDevice, st));
  GK_CUDA(cudaMemcpyAsync(na.count, &n32, 4, cudaMemcpyHostToDevice, st));
  GK_CUDA(cudaMemcpyAsync(na.parent, &none, 4, cudaMemcpyHostToDevice, st));

  std::vector<std::uint32_t> lvl_off{0};
  std::uint32_t S = 1;
  const double* cur = src;
  const std::uint32_t* cur_ids = src_ids;
  std::uint64_t cur_stride = src_stride;
  double* nxt = bufA;
  std::uint32_t* nxt_ids = idsA;
  int level = 0;
  while (S > 0) {
    if (level > 250) throw Error(GK_ERR_LOGIC, "BuildvEB_S: tree deeper than 250 levels");
    const std::uint32_t off = lvl_off.back();
    k_chunk_counts<<<blocks_for(S + 1), 256, 0, st>>>(na.count + off, S, chunk_cnt);
    scratch.scan(chunk_cnt, chunk_off, S + 1);
    k_chunk_node<<<std::min<unsigned>(blocks_for(n / kChunk + S), 4096), 256, 0, st>>>(chunk_off, S, chunk_node);
    k_bbox_init<<<blocks_for(static_cast<std::uint64_t>(S) * D), 256, 0, st>>>(keys, S * D);
    k_bbox<D><<<grid_w, 256, 0, st>>>(cur, cur_stride, chunk_off, chunk_node, S, off, na, keys);
    k_split<D><<<blocks_for(S), 256, 0, st>>>(S, off, level, leaf, heuristic, keys, na);
    k_count<D><<<grid_w, 256, 0, st>>>(cur, cur_ids, cur_stride, chunk_off, chunk_node, S, off, level, 0, na, chunk_left);
    GK_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(std::uint32_t), st));
    k_check<<<blocks_for(S + 1), 256, 0, st>>>(S, off, na, is_int, obj_list, counters);
    scratch.scan(is_int, irank, S + 1);
    GK_CUDA(cudaMemcpyAsync(counters + 1, irank + S, 4, cudaMemcpyDeviceToDevice, st));
    GK_CUDA(cudaMemcpyAsync(counters + 2, chunk_off + S, 4, cudaMemcpyDeviceToDevice, st));
    GK_CUDA(cudaMemcpyAsync(h_counters, counters, 3 * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    const std::uint32_t nobj = h_counters[0], nint = h_counters[1], nchunks = h_counters[2];
    if (nobj > 0) {
      if (nobj > sel_cap) {
        dfree(sel, st);
        dfree(hist, st);
        sel_cap = std::max<std::uint64_t>(nobj, 2 * sel_cap);
        sel = dalloc<SelState>(sel_cap, st);
        hist = dalloc<std::uint32_t>(sel_cap * 256, st);
      }
      GK_CUDA(cudaMemsetAsync(hist, 0, static_cast<std::size_t>(nobj) * 256 * 4, st));
      k_sel_init<<<blocks_for(nobj), 256, 0, st>>>(nobj, obj_list, na, sel);
      for (int p = 0; p < 12; ++p) {
        k_sel_hist<D><<<grid_w, 256, 0, st>>>(cur, cur_ids, cur_stride, chunk_off, chunk_node, S, off, level, p, na, sel,
                                              hist);
        k_sel_pick<<<blocks_for(nobj), 256, 0, st>>>(nobj, p, sel, hist);
      }
      k_sel_finish<<<blocks_for(nobj), 256, 0, st>>>(nobj, obj_list, sel, na);
      k_count<D><<<grid_w, 256, 0, st>>>(cur, cur_ids, cur_stride, chunk_off, chunk_node, S, off, level, 1, na,
                                         chunk_left);
    }
    scratch.scan(chunk_left, left_scan, static_cast<std::uint64_t>(nchunks) + 1);
    const std::uint32_t next_off = off + S;
    k_children<<<blocks_for(S), 256, 0, st>>>(S, off, next_off, irank, na);
    k_scatter<D><<<grid_w, 256, 0, st>>>(cur, cur_ids, cur_stride, nxt, nxt_ids, T.coords, T.ids, n, chunk_off,
                                         chunk_node, left_scan, S, off, level, na);
    GK_CHECK_LAUNCH();
    lvl_off.push_back(next_off);
    S = 2 * nint;
    ++level;
    // ping-pong: the partitioned points now live in nxt (stride n)
    cur = nxt;
    cur_ids = nxt_ids;
    cur_stride = n;
    nxt = (nxt == bufA) ? bufB : bufA;
    nxt_ids = (nxt_ids == idsA) ? idsB : idsA;
  }
  const int H = level;
  const std::uint32_t N = lvl_off.back();
  lvl_off.push_back(N);  // lvl_off[H+1] = N (so child_idx of an end position at level H-1 is defined)
  T.height = H;
  T.n_nodes = N;

  // vEB slots, top-down
  std::uint32_t* d_lvl_off = dalloc<std::uint32_t>(lvl_off.size(), st);
  GK_CUDA(cudaMemcpyAsync(d_lvl_off, lvl_off.data(), lvl_off.size() * 4, cudaMemcpyHostToDevice, st));
  GK_CUDA(cudaMemsetAsync(na.pos, 0, 4, st));
  std::vector<std::pair<int, int>> cut(H + 1, {0, 0});
  veb_cuts(0, H, cut);
  for (int d = 1; d < H; ++d) {
    const std::uint32_t Sd = lvl_off[d + 1] - lvl_off[d];
    k_veb<<<blocks_for(Sd), 256, 0, st>>>(d, cut[d].first, cut[d].second, d_lvl_off, na);
  }
  std::uint32_t* int_by_slot = dalloc<std::uint32_t>(N + 1, st);
  T.irank = dalloc<std::uint32_t>(N + 1, st);
  k_slot_flags<<<blocks_for(N + 1), 256, 0, st>>>(N, na, int_by_slot);
  scratch.scan(int_by_slot, T.irank, static_cast<std::uint64_t>(N) + 1);
  T.n_internal = (N - 1) / 2;
  T.canon = dalloc<gk_canon_node>(N, st);
  T.tnodes = dalloc<TNode<D>>(T.n_internal, st);
  T.orig = dalloc<std::int32_t>(3 * static_cast<std::uint64_t>(N), st);
  GK_CUDA(cudaMemsetAsync(T.orig + 2 * static_cast<std::uint64_t>(N), 0xff, 4, st));  // parent(root) = -1
  k_emit<D><<<blocks_for(N), 256, 0, st>>>(N, na, T.irank, T.canon, static_cast<TNode<D>*>(T.tnodes), T.orig);
  GK_CHECK_LAUNCH();
  T.root_ref = (N == 1) ? make_leaf_ref(0, static_cast<std::uint32_t>(n)) : 0;
  T.root_slot = 0;

  dfree(int_by_slot, st);
  dfree(d_lvl_off, st);
  dfree(bufA, st); dfree(bufB, st); dfree(idsA, st); dfree(idsB, st);
  dfree(na.start, st); dfree(na.count, st); dfree(na.parent, st); dfree(na.cbase, st); dfree(na.nleft, st);
  dfree(na.pos, st); dfree(na.thr_id, st); dfree(na.flags, st); dfree(na.level, st); dfree(na.split, st);
  dfree(na.lo, st); dfree(na.hi, st);
  dfree(chunk_cnt, st); dfree(chunk_off, st); dfree(chunk_node, st); dfree(chunk_left, st); dfree(left_scan, st);
  dfree(is_int, st); dfree(irank, st); dfree(obj_list, st); dfree(keys, st); dfree(counters, st);
  dfree(sel, st); dfree(hist, st);
  GK_CUDA(cudaFreeHost(h_counters));
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
    const std::int32_t a = __ldcg(&repl[orig[p]]), b = __ldcg(&repl[orig[N + p]]);
    __stcg(&repl[p], (a >= 0 && b >= 0) ? p : (a >= 0 ? a : b));
    cur = p;
  }
}

template <int D>
__global__ void k_relink(std::uint32_t N, gk_canon_node* canon, TNode<D>* tn, const std::uint32_t* __restrict__ irank,
                         const std::int32_t* __restrict__ orig, const std::int32_t* __restrict__ repl) {
  std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N || canon[v].kind != 0) return;
  const std::int32_t a = repl[orig[v]], b = repl[orig[N + v]];
  if (a < 0 || b < 0) return;  // v itself is spliced out or removed
  canon[v].left = a;
  canon[v].right = b;
  TNode<D> t = tn[irank[v]];
  const std::int32_t ch[2] = {a, b};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const gk_canon_node& c = canon[ch[s]];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      t.lo[s][j] = __double2float_rd(c.lo[j]);
      t.hi[s][j] = __double2float_ru(c.hi[j]);
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

}  // namespace

void build_tree(int d, int leaf, int heuristic, const double* src, std::uint64_t src_stride, const std::uint32_t* src_ids,
                std::uint64_t n, DevTree& out, cudaStream_t st) {
  switch (d) {
    case 2: build_tree_d<2>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 3: build_tree_d<3>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 4: build_tree_d<4>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 5: build_tree_d<5>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 6: build_tree_d<6>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 7: build_tree_d<7>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    case 8: build_tree_d<8>(leaf, heuristic, src, src_stride, src_ids, n, out, st); break;
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
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

void free_tree(DevTree& t, cudaStream_t st) {
  dfree(t.coords, st);
  dfree(t.ids, st);
  if (t.tnodes) GK_CUDA(cudaFreeAsync(t.tnodes, st));
  t.tnodes = nullptr;
  dfree(t.canon, st);
  dfree(t.orig, st);
  dfree(t.irank, st);
  t = DevTree();
}

}  // namespace gk
