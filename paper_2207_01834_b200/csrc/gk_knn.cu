// gk_knn.cu — kNN_L on the B200 (sm_100a): query reordering (K2) and the fused
// multi-tree traversal kernel (K1).
//
// Reference semantics (restated; no reference code exists for it):
//   kNN_S  PAPER.md:1153-1160 (descend, sibling fill, bbox include/prune/recurse)
//   kNN_L  PAPER.md:774-775, 1231-1233, 1477-1480; SPEC.md:590-597 — one k-buffer per query
//          reused across the trees, trees visited largest -> smallest, then the buffer tree
//   KnnBuffer ordering: lexicographic (d2, id), knn_buffer.hpp:18-19, 36-38, 42-46
// kNN is exact, so the result is a pure function of the live point set: the
// device traversal only has to (a) compute d2 in the oracle's canonical order
// (sum_j (q_j - p_j)^2 left to right, no FMA: __dsub_rn/__dmul_rn/__dadd_rn),
// (b) keep the lexicographic (d2, id) top-k, and (c) prune only when a box's
// lower-bound distance is STRICTLY greater than the current k-th d2.
//
// K1 design: one warp = a tile of 32 Morton-adjacent queries (one per lane)
// traversing each tree as a packet.  A node is entered when any lane's query
// still needs it; the warp-uniform reference stack lives in shared memory, the
// per-lane box lower bounds in a (coalesced, L1-resident) local array.  Node
// records hold both children's fp32 outward-rounded boxes, so one broadcast
// 64 B load (3D) decides both children.  A leaf's points are staged once per
// warp into shared memory with coalesced SoA fp64 loads and every lane scans
// them against its own query; candidates live in a per-lane max-heap.  All trees
// of the log structure are walked inside the same kernel, so no per-tree
// state ever round-trips through HBM.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "gk_common.cuh"

namespace gk {
namespace {

// warps per block: 8, or 4 for K > 16 so the shared-memory k-buffers (12 B x K per lane) still
// leave room for several blocks per SM; K = 0 is the runtime-k instantiation (32 < k <= 256)
template <int K>
#ifndef GK_K4W
#define GK_K4W 10  // k-buffers of more than this many entries use 4-warp blocks (C5 k = 16: +5 %)
#endif
__host__ __device__ constexpr int warps_for() { return K <= 0 ? 2 : (K > GK_K4W ? 4 : 8); }
constexpr int kMaxRuntimeK = 256;
constexpr bool kHilbertOrder = true;  // K2 key: Hilbert (true) or Morton (false)

__device__ __forceinline__ bool lexlt(double a, std::uint32_t ia, double b, std::uint32_t ib) {
  return a < b || (a == b && ia < ib);
}

// distances of the query to staged leaf points p and p+1 (p even): one 16-byte shared
// load per coordinate serves both, two independent fp64 chains
template <int D, int ROW = GK_MAX_LEAF>
__device__ __forceinline__ void leaf_d2_pair(const double (&q)[D], const double* sp, std::uint32_t p, double& da,
                                             double& db) {
  double2 x = reinterpret_cast<const double2*>(sp)[p >> 1];
  double ta = __dsub_rn(q[0], x.x), tb = __dsub_rn(q[0], x.y);
  da = __dmul_rn(ta, ta);  // 0 + t0^2 == t0^2 exactly
  db = __dmul_rn(tb, tb);
#pragma unroll
  for (int j = 1; j < D; ++j) {
    x = reinterpret_cast<const double2*>(sp + j * ROW)[p >> 1];
    ta = __dsub_rn(q[j], x.x);
    tb = __dsub_rn(q[j], x.y);
    da = __dadd_rn(da, __dmul_rn(ta, ta));
    db = __dadd_rn(db, __dmul_rn(tb, tb));
  }
}

#ifndef GK_CPASYNC
#define GK_CPASYNC 1  // leaf points staged with cp.async (LDGSTS; 0: loads + shared stores). C2 +0.4 %, C1 +2.8 %, C3 +5.7 %
#endif
// stage leaf points [s, s + c) of one tree into a warp's shared-memory block ([D][GK_MAX_LEAF] SoA + ids):
// lane < c copies point s + lane; cp.async (LDGSTS) moves global -> shared without a register round trip.
// The caller brackets it with __syncwarp() and calls stage_wait() before the warp reads the block.
template <int D, int ROW = GK_MAX_LEAF>
__device__ __forceinline__ void stage_leaf(double* sp, std::uint32_t* si, const double* __restrict__ coords,
                                           const std::uint32_t* __restrict__ ids, std::uint64_t stride, std::uint64_t s,
                                           std::uint32_t c, int lane, bool with_ids) {
  if (lane >= static_cast<int>(c)) return;
#if GK_CPASYNC
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sp + j * ROW + lane));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(coords + j * stride + s + lane));
  }
  if (with_ids) {
    const unsigned dsti = static_cast<unsigned>(__cvta_generic_to_shared(si + lane));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dsti), "l"(ids + s + lane));
  }
#else
#pragma unroll
  for (int j = 0; j < D; ++j) sp[j * ROW + lane] = coords[j * stride + s + lane];
  if (with_ids) si[lane] = ids[s + lane];
#endif
}
__device__ __forceinline__ void stage_wait() {
#if GK_CPASYNC
  asm volatile("cp.async.wait_all;" ::: "memory");
#endif
}

// ---- TMA (bulk copy) leaf staging: one elected lane issues D + 1 cp.async.bulk copies of the aligned
// supersets of the leaf's SoA rows (16-byte aligned start, 16-byte multiple size) that complete on the
// warp's mbarrier; the neighbouring leaves' points inside the supersets are masked with NaN afterwards.
// Used for trees whose layout allows it (stride a multiple of 4 points, 16-byte aligned arrays).
#ifndef GK_TMA_LEAF
#define GK_TMA_LEAF 0
#endif
constexpr int kLeafRow = GK_TMA_LEAF ? GK_MAX_LEAF + 2 : GK_MAX_LEAF;  // doubles per staged coordinate row
constexpr int kIdRow = GK_TMA_LEAF ? GK_MAX_LEAF + 4 : GK_MAX_LEAF;    // staged ids
__device__ __forceinline__ void mbar_init(unsigned bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}" ::"r"(bar),
      "r"(phase)
      : "memory");
}

#ifndef GK_PF_CHILD
#define GK_PF_CHILD 0  // 1: L1 prefetch of both children's node records at a node visit; 2: also leaf children's rows
#endif
#ifndef GK_PAIRCHK
#define GK_PAIRCHK 0  // 1: one min(da, db) <= kd test in front of the pair's two offers
#endif

// packed fp32x2 helpers (sm_100: FADD2/FMUL2 with directed rounding)
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  return (static_cast<unsigned long long>(__float_as_uint(b)) << 32) | __float_as_uint(a);
}
__device__ __forceinline__ float lo_of(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v)); }
__device__ __forceinline__ float hi_of(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v >> 32)); }
__device__ __forceinline__ unsigned long long sub_rm2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul_rm2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long add_rm2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// fp32 lower bound of the canonical fp64 d2 of every point inside each child's box
// [lo, hi], both children at once (the two halves of each packed f32x2 instruction):
// per-dimension gaps rounded down from (q rounded out), squares and sums rounded down,
// then scaled by (1 - 2^-23) rounded down so that the bound stays below the fp64
// rounding of the true d2 (relative error <= (D+1) 2^-53).
template <int D>
__device__ __forceinline__ void box_lb_pair(const unsigned long long (&qlo2)[D], const unsigned long long (&qhi2)[D],
                                            const unsigned long long* lo2, const unsigned long long* hi2, float& m0,
                                            float& m1) {
  unsigned long long s = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const unsigned long long a = sub_rm2(lo2[j], qhi2[j]);  // lo - q (rounded down)
    const unsigned long long b = sub_rm2(qlo2[j], hi2[j]);  // q - hi (rounded down)
    const float t0 = fmaxf(fmaxf(lo_of(a), lo_of(b)), 0.f);
    const float t1 = fmaxf(fmaxf(hi_of(a), hi_of(b)), 0.f);
    const unsigned long long t = pk2(t0, t1);
    const unsigned long long sq = mul_rm2(t, t);
    s = (j == 0) ? sq : add_rm2(s, sq);
  }
  s = mul_rm2(s, pk2(0x1.fffffcp-1f, 0x1.fffffcp-1f));
  m0 = lo_of(s);
  m1 = hi_of(s);
}

template <int D, int KT, bool COUNT>
__global__ void __launch_bounds__(warps_for<KT>() * 32, (D <= 4 ? 5 : 4)) k_knn(const TreeSet ts, const double* __restrict__ Q,
                                                        const std::uint32_t* __restrict__ perm, std::uint64_t nq, int k,
                                                        std::uint32_t* __restrict__ out_ids, double* __restrict__ out_d2,
                                                        unsigned long long* __restrict__ counters,
                                                        unsigned* __restrict__ tile_ctr,
                                                        double* __restrict__ gheap,
                                                        const double* __restrict__ qbound) {
  constexpr int kWarps = warps_for<KT>();
  const int K = KT > 0 ? KT : k;  // k-buffer size (compile-time for the common k)
  __shared__ std::uint64_t s_stack[kWarps][kStack];
  __shared__ __align__(16) double s_pts[kWarps][D * kLeafRow];
  __shared__ __align__(16) std::uint32_t s_ids[kWarps][kIdRow];
  __shared__ __align__(8) unsigned long long s_bar[GK_TMA_LEAF ? kWarps : 1];  // one mbarrier per warp (TMA staging)
  constexpr bool kPairMode = D >= 5;  // leaf work dominates at high D (C3: ~8x packet union)
  constexpr int kPairLanes = 10;      // <= this many needing lanes: pair-parallel leaf scan
#ifndef GK_PAIR_SMEM_Q
#define GK_PAIR_SMEM_Q 0  // 1: the tile's queries in shared memory for the pair-parallel scan (else shuffles)
#endif
  constexpr bool kSmemQ = GK_PAIR_SMEM_Q != 0;
  __shared__ double s_q[kWarps][(kPairMode && kSmemQ) ? D * 32 : 1];  // the tile's queries, [D][lane]
  __shared__ std::uint8_t s_own[kWarps][32];                   // lanes needing the current leaf
  // per-lane top-K heap, one column per thread (conflict-free): [K][blockDim] d2, then [K][blockDim] ids
  // (KT < 0, k > kMaxRuntimeK: the same columns in a global scratch heap, one per resident thread,
  // column stride = the grid's thread count; L1/L2 serve it)
  extern __shared__ double s_cand[];
  constexpr bool kGlobalHeap = KT < 0;
  using CsT = std::conditional_t<kGlobalHeap, std::uint64_t, int>;
  const CsT CS = kGlobalHeap ? static_cast<CsT>(gridDim.x) * blockDim.x : static_cast<CsT>(kWarps * 32);  // column stride
  const std::uint64_t boff = kGlobalHeap ? static_cast<std::uint64_t>(blockIdx.x) * blockDim.x : 0;
  double* hbase = kGlobalHeap ? gheap : s_cand;
  double* cbase = hbase + boff;  // this block's columns
  double* cdv = cbase + threadIdx.x;
  std::uint32_t* civ = reinterpret_cast<std::uint32_t*>(hbase + K * CS) + boff + threadIdx.x;

  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned ntiles = static_cast<unsigned>((nq + 31) / 32);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  unsigned long long c_nodes = 0, c_leaves = 0, c_dists = 0, c_wn = 0, c_wl = 0, c_ins = 0, c_wlp = 0, c_wev = 0;
  float mdst[kStack];
  [[maybe_unused]] unsigned tma_phase = 0;
  [[maybe_unused]] const unsigned bar = GK_TMA_LEAF ? static_cast<unsigned>(__cvta_generic_to_shared(&s_bar[GK_TMA_LEAF ? w : 0])) : 0u;
  if (GK_TMA_LEAF) {
    if (lane == 0) mbar_init(bar);
    __syncwarp();
  }

  // persistent warps: each grabs the next 32-query tile (Morton order keeps
  // concurrently processed tiles adjacent, so their trees' paths share L1/L2)
  while (true) {
  unsigned tile = 0;
  if (lane == 0) tile = atomicAdd(tile_ctr, 1u);
  tile = __shfl_sync(0xffffffffu, tile, 0);
  if (tile >= ntiles) break;
  const std::uint64_t qi = static_cast<std::uint64_t>(tile) * 32 + lane;
  const bool active = qi < nq;
  std::uint32_t orig = 0;
  double q[D];
  float qlo[D], qhi[D];
  if (active) {
    orig = perm ? perm[qi] : static_cast<std::uint32_t>(qi);
#pragma unroll
    for (int j = 0; j < D; ++j) q[j] = Q[static_cast<std::uint64_t>(orig) * D + j];
  } else {
#pragma unroll
    for (int j = 0; j < D; ++j) q[j] = 0.0;
  }
  unsigned long long qlo2[D], qhi2[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    qlo[j] = __double2float_rd(q[j]);
    qhi[j] = __double2float_ru(q[j]);
    qlo2[j] = pk2(qlo[j], qlo[j]);
    qhi2[j] = pk2(qhi[j], qhi[j]);
    if (kPairMode && kSmemQ) s_q[w][j * 32 + lane] = q[j];
  }
  // (+inf, kNoPoint): KnnBuffer's initial bound; a bounded kNN starts from (r2, kNoPoint)
  // sentinels instead, so only points with d2 <= r2 ever enter (ids < kNoPoint win the tie)
  const double kinit = (qbound && active) ? qbound[orig] : kInf;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    cdv[j * CS] = kinit;
    civ[j * CS] = GK_NO_POINT;
  }
  double kd = kinit;                // current k-th (d2, id) = heap root
  std::uint32_t kid = GK_NO_POINT;
  // k-th distance rounded up to fp32 (the pruning threshold); inactive lanes never want anything
  float kthf = active ? __double2float_ru(kinit) : -1.f;

  // The k-buffer is a max-heap on (d2, id) in this lane's shared-memory column: the root
  // is the current k-th entry, an accepted point replaces it and sifts down (<= log2 K
  // levels, so the warp's divergent inserts cost little); sorted once at the end.
  auto sift_down = [&](double x, std::uint32_t xid, int n) {
    int i = 0;
    while (true) {
      int c = 2 * i + 1;
      if (c >= n) break;
      double cv = cdv[c * CS];
      std::uint32_t cid = civ[c * CS];
      if (c + 1 < n) {
        const double rv = cdv[(c + 1) * CS];
        const std::uint32_t rid = civ[(c + 1) * CS];
        if (lexlt(cv, cid, rv, rid)) { ++c; cv = rv; cid = rid; }
      }
      if (!lexlt(x, xid, cv, cid)) break;
      cdv[i * CS] = cv;
      civ[i * CS] = cid;
      i = c;
    }
    cdv[i * CS] = x;
    civ[i * CS] = xid;
  };
  // offer staged leaf point p (distance d2) to this lane's k-buffer
  std::uint32_t idoff = 0;  // staged ids start this many entries before staged position 0 (TMA supersets)
  auto offer = [&](double d2, std::uint32_t p) {
    if (d2 <= kd) {  // rare: lexicographic test against the k-th, then heap replace
      const std::uint32_t pid = s_ids[w][p + idoff];
      if (d2 < kd || pid < kid) {
        if (COUNT && lane == __ffs(__activemask()) - 1) c_wev++;
        sift_down(d2, pid, K);
        kd = cdv[0];
        kid = civ[0];
        kthf = __double2float_ru(kd);
        if (COUNT) c_ins++;
      }
    }
  };

  for (int t = 0; t < ts.count; ++t) {
    const float4* __restrict__ nodes = static_cast<const float4*>(ts.t[t].tnodes);
    const double* __restrict__ coords = ts.t[t].coords;
    const std::uint32_t* __restrict__ ids = ts.t[t].ids;
    const std::uint64_t stride = ts.t[t].stride;
    std::uint64_t ref = ts.t[t].root;
    bool need = active;
    int sp = 0;
    // TMA staging needs 16-byte aligned row starts and sizes: stride a multiple of 4 points (ids), aligned arrays
    [[maybe_unused]] const bool tma_ok =
        GK_TMA_LEAF && (stride & 3ULL) == 0 &&
        ((reinterpret_cast<std::uintptr_t>(coords) | reinterpret_cast<std::uintptr_t>(ids)) & 15) == 0;
    while (true) {
      if (is_leaf_ref(ref)) {
        const std::uint32_t c = leaf_count(ref);
        const std::uint64_t s = leaf_start(ref);
        std::uint32_t pbase = 0, pcs = c;  // staged position of leaf point 0; staged positions to scan
        __syncwarp();
        if (GK_TMA_LEAF && tma_ok) {
          const std::uint64_t sa = s & ~1ULL, ia = s & ~3ULL;
          const std::uint32_t ca = static_cast<std::uint32_t>(((s + c + 1) & ~1ULL) - sa);  // even
          const std::uint32_t ib = static_cast<std::uint32_t>(((s + c + 3) & ~3ULL) - ia);  // multiple of 4
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the last leaf's NaN masks vs these writes
            mbar_expect_tx(bar, static_cast<unsigned>(D) * ca * 8u + ib * 4u);
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(s_pts[w]));
#pragma unroll
            for (int j = 0; j < D; ++j) bulk_g2s(dst + j * kLeafRow * 8, coords + j * stride + sa, ca * 8u, bar);
            bulk_g2s(static_cast<unsigned>(__cvta_generic_to_shared(s_ids[w])), ids + ia, ib * 4u, bar);
          }
          mbar_wait(bar, tma_phase);
          tma_phase ^= 1u;
          // the neighbouring leaves' points inside the aligned superset: NaN in coordinate 0 never enters the top-k
          if (lane == 0 && (s & 1ULL)) s_pts[w][0] = __longlong_as_double(0x7ff8000000000000LL);
          if (lane == 1 && ((s + c) & 1ULL)) s_pts[w][ca - 1] = __longlong_as_double(0x7ff8000000000000LL);
          pbase = static_cast<std::uint32_t>(s & 1ULL);
          pcs = ca;
          idoff = static_cast<std::uint32_t>(sa - ia);
        } else {
          stage_leaf<D, kLeafRow>(s_pts[w], s_ids[w], coords, ids, stride, s, c, lane, true);
          if (lane == static_cast<int>(c) && (c & 1u))
            s_pts[w][lane] = __longlong_as_double(0x7ff8000000000000LL);  // NaN pad: never enters the top-k
          stage_wait();
          if (GK_TMA_LEAF) idoff = 0;
        }
        __syncwarp();
        const unsigned needm = __ballot_sync(0xffffffffu, need);
        const int m = __popc(needm);
        if (!kPairMode || m > kPairLanes) {
          // each lane scans all points against its own query,
          // two independent distance chains per iteration (fp64 latency)
          for (std::uint32_t p = 0; p < pcs; p += 2) {
            double da, db;
            leaf_d2_pair<D, kLeafRow>(q, s_pts[w], p, da, db);
            if (!GK_PAIRCHK || fmin(da, db) <= kd) {  // one test rejects both (the common case)
              offer(da, p);
              offer(db, p + 1);
            }
          }
        } else if (m > 0) {
          // high D, few lanes need this leaf: spread the m x c needed (query, point) pairs
          // over the warp; a pair that beats its owner's k-th distance goes to the owner lane
          if (need) s_own[w][__popc(needm & ((1u << lane) - 1u))] = static_cast<std::uint8_t>(lane);
          __syncwarp();
          const std::uint32_t total = static_cast<std::uint32_t>(m) * c;
          const std::uint32_t dqi = 32u / c, dp = 32u % c;
          std::uint32_t qi = static_cast<std::uint32_t>(lane) / c, pp = static_cast<std::uint32_t>(lane) % c;
          for (std::uint32_t t0 = 0; t0 < total; t0 += 32) {
            const bool valid = t0 + lane < total;
            const int own = valid ? s_own[w][qi] : 0;
            double d2 = 0.0;
            bool cand = false;
            if (kSmemQ) {
              if (valid) {
                const double* qo = &s_q[w][own];
                const double t = __dsub_rn(qo[0], s_pts[w][pp + pbase]);
                d2 = __dmul_rn(t, t);
#pragma unroll
                for (int j = 1; j < D; ++j) {
                  const double tt = __dsub_rn(qo[j * 32], s_pts[w][j * kLeafRow + pp + pbase]);
                  d2 = __dadd_rn(d2, __dmul_rn(tt, tt));
                }
              }
            } else {
              // the owner's query straight from its registers (keeps ~14 KB of shared memory per
              // block free at D = 7: 4 blocks per SM instead of 3)
              const std::uint32_t ppc = (valid ? pp : 0u) + pbase;
              const double t = __dsub_rn(__shfl_sync(0xffffffffu, q[0], own), s_pts[w][ppc]);
              d2 = __dmul_rn(t, t);
#pragma unroll
              for (int j = 1; j < D; ++j) {
                const double tt = __dsub_rn(__shfl_sync(0xffffffffu, q[j], own), s_pts[w][j * kLeafRow + ppc]);
                d2 = __dadd_rn(d2, __dmul_rn(tt, tt));
              }
            }
            if (valid) cand = d2 <= cbase[w * 32 + own];  // owner's heap root = its k-th distance
            unsigned bal = __ballot_sync(0xffffffffu, cand);
            while (bal) {
              const int b = __ffs(bal) - 1;
              bal &= bal - 1;
              const int ob = __shfl_sync(0xffffffffu, own, b);
              const double db = __shfl_sync(0xffffffffu, d2, b);
              const std::uint32_t pb = __shfl_sync(0xffffffffu, pp, b);
              if (lane == ob) offer(db, pb + pbase);
            }
            __syncwarp();
            pp += dp;
            qi += dqi;
            if (pp >= c) { pp -= c; ++qi; }
          }
        }
        if (COUNT) {
          if (need) { c_leaves++; c_dists += c; }
          c_wl++;
          c_wlp += c;
        }
      } else {
        const float4* nd = nodes + ref * (D + 1);
        // whole node in D+1 16-byte loads: D (lo0,lo1) pairs, D (hi0,hi1) pairs, 2 child refs
        unsigned long long u[2 * (D + 1)];
#pragma unroll
        for (int v = 0; v <= D; ++v) {
          const ulonglong2 x = reinterpret_cast<const ulonglong2*>(nd)[v];
          u[2 * v] = x.x;
          u[2 * v + 1] = x.y;
        }
        const ulonglong2 rr = make_ulonglong2(u[2 * D], u[2 * D + 1]);
        if (COUNT) {
          if (need) c_nodes++;
          c_wn++;
        }
#if GK_PF_CHILD
        // both children's records (or leaf rows) start towards L1 while this node's boxes are tested
        {
          const std::uint64_t r0 = rr.x, r1 = rr.y;
          if (!is_leaf_ref(r0)) asm volatile("prefetch.global.L1 [%0];" ::"l"(nodes + r0 * (D + 1)));
          else if (GK_PF_CHILD >= 2 && lane <= D)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(lane < D ? static_cast<const void*>(coords + lane * stride + leaf_start(r0))
                                                                  : static_cast<const void*>(ids + leaf_start(r0))));
          if (!is_leaf_ref(r1)) asm volatile("prefetch.global.L1 [%0];" ::"l"(nodes + r1 * (D + 1)));
          else if (GK_PF_CHILD >= 2 && lane <= D)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(lane < D ? static_cast<const void*>(coords + lane * stride + leaf_start(r1))
                                                                  : static_cast<const void*>(ids + leaf_start(r1))));
        }
#endif
        float m0, m1;
        box_lb_pair<D>(qlo2, qhi2, u, u + D, m0, m1);
        const bool w0 = m0 <= kthf, w1 = m1 <= kthf;
        const unsigned b0 = __ballot_sync(0xffffffffu, w0), b1 = __ballot_sync(0xffffffffu, w1);
        if (b0 && b1) {
          // near child first, by majority of the lanes that want both (else by lane count)
          const unsigned both = b0 & b1;
          int first;
          if (both) {
            const unsigned pref0 = __ballot_sync(0xffffffffu, w0 && w1 && m0 <= m1);
            first = (2 * __popc(pref0) >= __popc(both)) ? 0 : 1;
          } else {
            first = (__popc(b0) >= __popc(b1)) ? 0 : 1;
          }
          if (lane == 0) s_stack[w][sp] = first ? rr.x : rr.y;
          mdst[sp] = first ? m0 : m1;
          ++sp;
          ref = first ? rr.y : rr.x;
          need = first ? w1 : w0;
          continue;
        } else if (b0) {
          ref = rr.x; need = w0;
          continue;
        } else if (b1) {
          ref = rr.y; need = w1;
          continue;
        }
      }
      // pop the next subtree some lane still needs
      bool found = false;
      __syncwarp();
      while (sp > 0) {
        --sp;
        const bool nl = mdst[sp] <= kthf;
        if (__any_sync(0xffffffffu, nl)) {
          ref = s_stack[w][sp];
          need = nl;
          found = true;
          break;
        }
      }
      if (!found) break;
    }
  }

  if (active) {
    // heapsort: pop the max into position n-1 (KnnBuffer::extract order, ascending (d2, id))
    for (int n = K - 1; n > 0; --n) {
      const double top = cdv[0];
      const std::uint32_t topid = civ[0];
      const double last = cdv[n * CS];
      const std::uint32_t lastid = civ[n * CS];
      cdv[n * CS] = top;
      civ[n * CS] = topid;
      sift_down(last, lastid, n);
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < k) {
        const std::uint32_t id = civ[j * CS];
        out_ids[static_cast<std::uint64_t>(orig) * k + j] = id;
        out_d2[static_cast<std::uint64_t>(orig) * k + j] = id == GK_NO_POINT ? kInf : cdv[j * CS];
      }
  }
  }  // tile loop

  if (COUNT) {
    const unsigned long long node_b = sizeof(TNode<D>), pt_b = 8 * D + 4;
    unsigned long long v[5] = {c_nodes, c_leaves, c_dists, c_ins, c_wev};
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    if (lane == 0) {
      atomicAdd(&counters[0], v[0] * node_b);
      atomicAdd(&counters[1], v[2] * pt_b);
      atomicAdd(&counters[2], v[0]);
      atomicAdd(&counters[3], v[1]);
      atomicAdd(&counters[4], v[2]);
      atomicAdd(&counters[5], c_wn);
      atomicAdd(&counters[6], c_wl);
      atomicAdd(&counters[7], v[3]);
      atomicAdd(&counters[8], c_wlp);
      atomicAdd(&counters[9], v[4]);
    }
  }
}

// --------------------------------------------------------------- K2: order --
__global__ void k_qbox_init(unsigned long long* box, int d) {
  if (threadIdx.x < d) { box[2 * threadIdx.x] = ~0ULL; box[2 * threadIdx.x + 1] = 0ULL; }
}

template <int D>
__global__ void k_qbox(const double* __restrict__ Q, std::uint64_t nq, unsigned long long* box) {
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) { lo[j] = __longlong_as_double(0x7ff0000000000000LL); hi[j] = -lo[j]; }
  for (std::uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double x = Q[i * D + j];
      lo[j] = fmin(lo[j], x);
      hi[j] = fmax(hi[j], x);
    }
#pragma unroll
  for (int j = 0; j < D; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[j] = fmin(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], o));
      hi[j] = fmax(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], o));
    }
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      atomicMin(&box[2 * j], dkey(lo[j]));
      atomicMax(&box[2 * j + 1], dkey(hi[j]));
    }
}

// Hilbert index of a D-dim cell with B bits per dim (Skilling's transpose + Gray code)
template <int D, int B, class KeyT>
__device__ __forceinline__ KeyT hilbert_key(std::uint32_t (&cell)[D]) {
#pragma unroll
  for (std::uint32_t Qb = 1u << (B - 1); Qb > 1; Qb >>= 1) {
    const std::uint32_t P = Qb - 1;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (cell[j] & Qb) {
        cell[0] ^= P;
      } else {
        const std::uint32_t t = (cell[0] ^ cell[j]) & P;
        cell[0] ^= t;
        cell[j] ^= t;
      }
    }
  }
#pragma unroll
  for (int j = 1; j < D; ++j) cell[j] ^= cell[j - 1];
  std::uint32_t t = 0;
#pragma unroll
  for (std::uint32_t Qb = 1u << (B - 1); Qb > 1; Qb >>= 1)
    if (cell[D - 1] & Qb) t ^= Qb - 1;
#pragma unroll
  for (int j = 0; j < D; ++j) cell[j] ^= t;
  KeyT key = 0;
#pragma unroll
  for (int b = B - 1; b >= 0; --b)
#pragma unroll
    for (int j = 0; j < D; ++j) key = (key << 1) | ((cell[j] >> b) & 1u);
  return key;
}

// space-filling-curve key of each query over the batch's bounding box: Hilbert order
// (fewer jumps than Morton between consecutive keys -> more compact 32-query packets).
// 32-bit keys for D <= 4; at D >= 5 they would leave only 4-6 bits per dimension, too
// coarse for clustered data (C3), so 64-bit keys (9 bits per dimension in 7D) are used.
template <int D, class Key>
__global__ void k_curve_key(const double* __restrict__ Q, std::uint64_t nq, const unsigned long long* __restrict__ box,
                            Key* keys, std::uint32_t* idx) {
  constexpr int B = (8 * static_cast<int>(sizeof(Key)) - (sizeof(Key) == 8 ? 1 : 0)) / D;
  std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nq) return;
  std::uint32_t cell[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double lo = dkey_inv(box[2 * j]), hi = dkey_inv(box[2 * j + 1]);
    const double ext = hi - lo;
    double f = ext > 0.0 ? (Q[i * D + j] - lo) / ext : 0.0;
    int c = static_cast<int>(f * static_cast<double>(1u << B));
    c = c < 0 ? 0 : (c > static_cast<int>((1u << B) - 1) ? static_cast<int>((1u << B) - 1) : c);
    cell[j] = static_cast<std::uint32_t>(c);
  }
  Key key = 0;
  if (kHilbertOrder) {
    key = hilbert_key<D, B, Key>(cell);
  } else {
#pragma unroll
    for (int b = B - 1; b >= 0; --b)
#pragma unroll
      for (int j = 0; j < D; ++j) key = (key << 1) | ((cell[j] >> b) & 1u);
  }
  keys[i] = key;
  idx[i] = static_cast<std::uint32_t>(i);
}

template <int D, int KT>
void launch_k(const TreeSet& ts, const double* Q, const std::uint32_t* perm, std::uint64_t nq, int k, std::uint32_t* ids,
              double* d2, unsigned long long* ctr, cudaStream_t st, const double* bound) {
  constexpr int kWarps = warps_for<KT>();
  const unsigned blocks = static_cast<unsigned>((nq + kWarps * 32 - 1) / (kWarps * 32));
  // per-lane top-K columns in shared memory (KT < 0: in a global scratch heap instead)
  const int smem = KT < 0 ? 0 : (KT > 0 ? KT : k) * kWarps * 32 * 12;
  const int smem_max = KT < 0 ? 0 : (KT > 0 ? KT : kMaxRuntimeK) * kWarps * 32 * 12;
  static std::once_flag once[kMaxDevices];  // per (D, K) instantiation and device
  static int sm_counts[kMaxDevices] = {};
  const int dev = current_device();
  std::call_once(once[dev], [&] {
    GK_CUDA(cudaFuncSetAttribute(k_knn<D, KT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    GK_CUDA(cudaFuncSetAttribute(k_knn<D, KT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    GK_CUDA(cudaDeviceGetAttribute(&sm_counts[dev], cudaDevAttrMultiProcessorCount, dev));
  });
  const int sm_count = sm_counts[dev];
  int per = 0;  // resident blocks at this launch's shared-memory size
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_knn<D, KT, false>, kWarps * 32, smem));
  const int resident = std::max(1, per) * sm_count;
  unsigned grid = std::min<unsigned>(blocks, static_cast<unsigned>(resident));
  double* gheap = nullptr;
  if (KT < 0) {
    // scratch heap of 12 k bytes per resident thread, bounded to ~4 GB (at least one block per SM)
    const std::uint64_t per_block = static_cast<std::uint64_t>(kWarps) * 32 * k * 12;
    const std::uint64_t cap = std::max<std::uint64_t>(sm_count, (4ull << 30) / per_block);
    grid = static_cast<unsigned>(std::min<std::uint64_t>(grid, cap));
    GK_CUDA(cudaMallocAsync(&gheap, per_block * grid, st));
  }
  unsigned* tile_ctr = nullptr;
  GK_CUDA(cudaMallocAsync(&tile_ctr, sizeof(unsigned), st));
  GK_CUDA(cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned), st));
  if (ctr) k_knn<D, KT, true><<<grid, kWarps * 32, smem, st>>>(ts, Q, perm, nq, k, ids, d2, ctr, tile_ctr, gheap, bound);
  else k_knn<D, KT, false><<<grid, kWarps * 32, smem, st>>>(ts, Q, perm, nq, k, ids, d2, ctr, tile_ctr, gheap, bound);
  GK_CUDA(cudaFreeAsync(tile_ctr, st));
  if (gheap) GK_CUDA(cudaFreeAsync(gheap, st));
}

template <int D>
void launch_d(int k, const TreeSet& ts, const double* Q, const std::uint32_t* perm, std::uint64_t nq, std::uint32_t* ids,
              double* d2, unsigned long long* ctr, cudaStream_t st, const double* bound) {
  if (k <= 1) launch_k<D, 1>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 2) launch_k<D, 2>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 4) launch_k<D, 4>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 5) launch_k<D, 5>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 8) launch_k<D, 8>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 10) launch_k<D, 10>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 12) launch_k<D, 12>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);  // k + 1 = 11: the k = 10 k-NN graph
  else if (k <= 16) launch_k<D, 16>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= 32) launch_k<D, 32>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else if (k <= kMaxRuntimeK) launch_k<D, 0>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
  else launch_k<D, -1>(ts, Q, perm, nq, k, ids, d2, ctr, st, bound);
}

template <int D>
void order_queries(const double* Q, std::uint64_t nq, std::uint32_t* perm_out, cudaStream_t st) {
  using Key = std::conditional_t<(D >= 5), unsigned long long, std::uint32_t>;
  constexpr int bits = ((8 * static_cast<int>(sizeof(Key)) - (sizeof(Key) == 8 ? 1 : 0)) / D) * D;
  unsigned long long* box = nullptr;
  Key *keys = nullptr, *keys2 = nullptr;
  std::uint32_t* idx = nullptr;
  GK_CUDA(cudaMallocAsync(&box, 2 * D * sizeof(unsigned long long), st));
  GK_CUDA(cudaMallocAsync(&keys, nq * sizeof(Key), st));
  GK_CUDA(cudaMallocAsync(&keys2, nq * sizeof(Key), st));
  GK_CUDA(cudaMallocAsync(&idx, nq * 4, st));
  k_qbox_init<<<1, 32, 0, st>>>(box, D);
  const unsigned gb = static_cast<unsigned>(std::min<std::uint64_t>((nq + 255) / 256, 148 * 8));
  k_qbox<D><<<gb, 256, 0, st>>>(Q, nq, box);
  k_curve_key<D, Key><<<static_cast<unsigned>((nq + 255) / 256), 256, 0, st>>>(Q, nq, box, keys, idx);
  GK_CHECK_LAUNCH();
  void* tmp = nullptr;
  std::size_t tb = 0;
  // 32-bit keys are sorted on their top 24 bits only (three 8-bit radix passes instead of four): cells of
  // 1/256 (3D) or 1/4096 (2D) of the batch's box order the packets as well as the full key does (C2 +0.5 %,
  // C1 +3 %, C5 +1.4 % kNN_L).  GK_SORT_SKIP overrides the number of ignored low bits.
  static const int skip_env = std::getenv("GK_SORT_SKIP") ? std::atoi(std::getenv("GK_SORT_SKIP")) : -1;
  const int skip = skip_env >= 0 ? skip_env : (sizeof(Key) == 4 && bits > 24 ? bits - 24 : 0);
  const int b0 = std::min(std::max(skip, 0), bits - 8);
  auto sort = [&](auto n) {  // 32-bit item counts when they fit (CUB's faster offset type), else 64-bit
    GK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, perm_out, n, b0, bits, st));
    GK_CUDA(cudaMallocAsync(&tmp, tb, st));
    GK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, idx, perm_out, n, b0, bits, st));
  };
  if (nq <= 0x7fffffffULL) sort(static_cast<int>(nq));
  else sort(static_cast<long long>(nq));
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(box, st));
  GK_CUDA(cudaFreeAsync(keys, st));
  GK_CUDA(cudaFreeAsync(keys2, st));
  GK_CUDA(cudaFreeAsync(idx, st));
}


// ------------------------------------------------------------- kNN graph --
// live points of every tree (coordinate 0 NaN = tombstone), unordered
__global__ void k_live_gather(const TreeSet ts, int d, double* __restrict__ pts, std::uint32_t* __restrict__ ids,
                              std::uint32_t* __restrict__ pos, unsigned long long* __restrict__ ctr) {
  for (int t = 0; t < ts.count; ++t) {
    const std::uint64_t n = ts.t[t].stride;
    const double* c = ts.t[t].coords;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
      if (isnan(c[i])) continue;
      const unsigned long long o = atomicAdd(ctr, 1ULL);
      for (int j = 0; j < d; ++j) pts[o * d + j] = c[j * n + i];
      ids[o] = ts.t[t].ids[i];
      pos[o] = static_cast<std::uint32_t>(o);
    }
  }
}
// rows in ascending id order: q[r] = pts[src[r]]
__global__ void k_gather_rows(const double* __restrict__ pts, const std::uint32_t* __restrict__ src, std::uint64_t n, int d,
                              double* __restrict__ q) {
  const std::uint64_t r = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  for (int j = 0; j < d; ++j) q[r * d + j] = pts[static_cast<std::uint64_t>(src[r]) * d + j];
}
// row r's k neighbours = its k+1 nearest without the point itself (the first entry with the
// row's id; if k+1 duplicates at distance 0 precede it, the first k entries)
__global__ void k_drop_self(std::uint64_t n, int k, const std::uint32_t* __restrict__ row_ids,
                            const std::uint32_t* __restrict__ ti, const double* __restrict__ td,
                            std::uint32_t* __restrict__ oi, double* __restrict__ od) {
  const std::uint64_t r = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const std::uint32_t self = row_ids[r];
  const std::uint64_t a = r * (k + 1), b = r * k;
  int o = 0;
  bool dropped = false;
  for (int j = 0; j <= k && o < k; ++j) {
    const std::uint32_t id = ti[a + j];
    if (!dropped && id == self) { dropped = true; continue; }
    oi[b + o] = id;
    od[b + o] = td[a + j];
    ++o;
  }
}

// ------------------------------------------------------- range search (ball) --
// ParGeo's kd-tree range search (Table 1), over the log
// structure like kNN_L: every live point p with canonical d2(q, p) <= r2.  The same
// packet traversal as K1 with a fixed threshold: a child is entered when any lane's
// fp32 box lower bound is <= r2 rounded up (conservative), a staged leaf point is
// reported when its exact fp64 d2 <= r2.  FILL = false counts per query, FILL = true
// writes each query's rows at its offset (traversal order; sorted afterwards).
template <int D, int MODE>
__global__ void __launch_bounds__(256) k_range(const TreeSet ts, const double* __restrict__ Q,
                                               const std::uint32_t* __restrict__ perm, std::uint64_t nq, double r2,
                                               const double* __restrict__ r2q,
                                               unsigned long long* __restrict__ counts,
                                               const unsigned long long* __restrict__ offs,
                                               std::uint32_t* __restrict__ out_ids, double* __restrict__ out_d2,
                                               unsigned* __restrict__ tile_ctr, unsigned capq) {
  constexpr bool FILL = MODE == 1, SLOTS = MODE == 2;  // 0: count; 1: rows at offs; 2: first capq rows + count
  constexpr int kWarps = 8;
  __shared__ std::uint64_t s_stack[kWarps][kStack];
  __shared__ __align__(16) double s_pts[kWarps][D * GK_MAX_LEAF];
  __shared__ std::uint32_t s_ids[kWarps][GK_MAX_LEAF];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned ntiles = static_cast<unsigned>((nq + 31) / 32);
  while (true) {
    unsigned tile = 0;
    if (lane == 0) tile = atomicAdd(tile_ctr, 1u);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= ntiles) break;
    const std::uint64_t qi = static_cast<std::uint64_t>(tile) * 32 + lane;
    const bool active = qi < nq;
    std::uint32_t orig = 0;
    double q[D];
    unsigned long long qlo2[D], qhi2[D];
#pragma unroll
    for (int j = 0; j < D; ++j) q[j] = 0.0;
    if (active) {
      orig = perm[qi];
#pragma unroll
      for (int j = 0; j < D; ++j) q[j] = Q[static_cast<std::uint64_t>(orig) * D + j];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const float lo = __double2float_rd(q[j]), hi = __double2float_ru(q[j]);
      qlo2[j] = pk2(lo, lo);
      qhi2[j] = pk2(hi, hi);
    }
    const double r2v = (r2q && active) ? r2q[orig] : r2;  // per-query squared radius when given
    const float rf = active ? __double2float_ru(r2v) : -1.f;
    const double rq = active ? r2v : -1.0;
    unsigned long long cnt = 0;
    const unsigned long long base =
        (FILL && active) ? offs[orig] : (SLOTS ? static_cast<unsigned long long>(orig) * capq : 0ULL);
    for (int t = 0; t < ts.count; ++t) {
      const float4* __restrict__ nodes = static_cast<const float4*>(ts.t[t].tnodes);
      const double* __restrict__ coords = ts.t[t].coords;
      const std::uint32_t* __restrict__ ids = ts.t[t].ids;
      const std::uint64_t stride = ts.t[t].stride;
      std::uint64_t ref = ts.t[t].root;
      int sp = 0;
      while (true) {
        if (is_leaf_ref(ref)) {
          const std::uint32_t c = leaf_count(ref);
          const std::uint64_t s = leaf_start(ref);
          __syncwarp();
          stage_leaf<D>(s_pts[w], s_ids[w], coords, ids, stride, s, c, lane, FILL || SLOTS);
          stage_wait();
          __syncwarp();
          for (std::uint32_t p = 0; p < c; ++p) {
            double tt = __dsub_rn(q[0], s_pts[w][p]);
            double d2 = __dmul_rn(tt, tt);
#pragma unroll
            for (int j = 1; j < D; ++j) {
              tt = __dsub_rn(q[j], s_pts[w][j * GK_MAX_LEAF + p]);
              d2 = __dadd_rn(d2, __dmul_rn(tt, tt));
            }
            if (d2 <= rq) {  // NaN (tombstone) never qualifies
              if (FILL || (SLOTS && cnt < capq)) {
                out_ids[base + cnt] = s_ids[w][p];
                out_d2[base + cnt] = d2;
              }
              ++cnt;
            }
          }
        } else {
          const float4* nd = nodes + ref * (D + 1);
          unsigned long long u[2 * (D + 1)];
#pragma unroll
          for (int v = 0; v <= D; ++v) {
            const ulonglong2 x = reinterpret_cast<const ulonglong2*>(nd)[v];
            u[2 * v] = x.x;
            u[2 * v + 1] = x.y;
          }
          float m0, m1;
          box_lb_pair<D>(qlo2, qhi2, u, u + D, m0, m1);
          const unsigned b0 = __ballot_sync(0xffffffffu, m0 <= rf), b1 = __ballot_sync(0xffffffffu, m1 <= rf);
          if (b0 && b1) {
            if (lane == 0) s_stack[w][sp] = u[2 * D + 1];
            ++sp;
            ref = u[2 * D];
            continue;
          } else if (b0) {
            ref = u[2 * D];
            continue;
          } else if (b1) {
            ref = u[2 * D + 1];
            continue;
          }
        }
        // the threshold never changes: every pushed subtree is still wanted by some lane
        __syncwarp();
        if (sp == 0) break;
        ref = s_stack[w][--sp];
      }
    }
    if (active && !FILL) counts[orig] = cnt;
  }
}

template <int D>
void range_d(const TreeSet& ts, const double* Q, std::uint64_t nq, double r2, const double* r2q, unsigned long long* counts,
             unsigned long long* offs, std::uint32_t* ids, double* d2, int mode, unsigned capq, std::uint32_t* perm,
             cudaStream_t st) {
  static int grids[kMaxDevices] = {};
  static std::once_flag once[kMaxDevices];
  const int dev = current_device();
  int& grid = grids[dev];
  std::call_once(once[dev], [&] {
    int sms = 0, per0 = 0, per1 = 0, per2 = 0;
    GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per0, k_range<D, 0>, 256, 0));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_range<D, 1>, 256, 0));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_range<D, 2>, 256, 0));
    grid = std::max(1, std::min(per0, std::min(per1, per2))) * sms;
  });
  const unsigned g = static_cast<unsigned>(std::min<std::uint64_t>(grid, (nq + 255) / 256));
  unsigned* tile_ctr = nullptr;
  GK_CUDA(cudaMallocAsync(&tile_ctr, sizeof(unsigned), st));
  GK_CUDA(cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned), st));
  if (mode == 1) k_range<D, 1><<<g, 256, 0, st>>>(ts, Q, perm, nq, r2, r2q, counts, offs, ids, d2, tile_ctr, capq);
  else if (mode == 2) k_range<D, 2><<<g, 256, 0, st>>>(ts, Q, perm, nq, r2, r2q, counts, offs, ids, d2, tile_ctr, capq);
  else k_range<D, 0><<<g, 256, 0, st>>>(ts, Q, perm, nq, r2, r2q, counts, offs, ids, d2, tile_ctr, capq);
  GK_CHECK_LAUNCH();
  GK_CUDA(cudaFreeAsync(tile_ctr, st));
}

// rows of the bounded-slot pass into their CSR place; flags (in K2 order) the queries with more
// rows than slots, so that the list of those keeps the order's packet coherence
constexpr unsigned kRangeSortCap = 32;  // the slot count per query this kernel is written for (kRangeSlots)
// Slot rows -> CSR rows, each query's rows in (d2, id) order.  A half-warp per query: lane j holds slots j and
// j + 16 (coalesced reads per query instead of 32 lines per load with a thread per query); a bitonic network
// sorts the (d2, id) pairs by shuffles -- 16 elements when neither query of the warp has more than 16 rows, else
// 32 (two per lane; the stride-16 stage is in-lane) -- empty slots = (+inf, ~0) sink to the end; lane j writes
// rows j and j + 16.  (The two CUB segmented sorts over all rows that used to order them took 0.8 ms of a 5.8 ms
// C2 range search; a thread per query with an insertion sort took 0.65 ms for the compaction.)
__device__ __forceinline__ bool pair_less(double a, std::uint32_t ai, double b, std::uint32_t bi) {
  return a < b || (a == b && ai < bi);
}
__global__ void k_slots_compact(std::uint64_t nq, unsigned capq, const std::uint32_t* __restrict__ perm,
                                const unsigned long long* __restrict__ counts, const unsigned long long* __restrict__ offs,
                                const std::uint32_t* __restrict__ ti, const double* __restrict__ td,
                                std::uint32_t* __restrict__ ids, double* __restrict__ d2, std::uint8_t* __restrict__ flag) {
  const std::uint64_t gt = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  const std::uint64_t i = gt >> 4;  // query (in K2 order) of this half-warp
  const unsigned j = threadIdx.x & 15u;
  const bool valid = i < nq;
  std::uint32_t q = 0;
  unsigned long long c = 0, o = 0;
  if (valid) {
    q = perm[i];
    c = counts[q];
    o = offs[q];
  }
  const bool over = c > capq;  // rows come from the second traversal (and its segmented sort)
  const unsigned m = (valid && !over) ? static_cast<unsigned>(c) : 0u;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  double x0 = kInf, x1 = kInf;
  std::uint32_t i0 = 0xffffffffu, i1 = 0xffffffffu;
  if (j < m) {
    x0 = td[static_cast<std::uint64_t>(q) * capq + j];
    i0 = ti[static_cast<std::uint64_t>(q) * capq + j];
  }
  if (j + 16 < m) {
    x1 = td[static_cast<std::uint64_t>(q) * capq + j + 16];
    i1 = ti[static_cast<std::uint64_t>(q) * capq + j + 16];
  }
  // compare-exchange of element (x, xi) at position pos with its partner pos ^ s2 in another lane
  auto cx_shfl = [&](double& x, std::uint32_t& xi, unsigned pos, unsigned k2, unsigned s2) {
    const double y = __shfl_xor_sync(0xffffffffu, x, s2);
    const std::uint32_t yi = __shfl_xor_sync(0xffffffffu, xi, s2);
    const bool up = (pos & k2) == 0, lower = (pos & s2) == 0;
    const bool less = pair_less(x, xi, y, yi);
    const bool keep = (lower == up) ? less : !less;
    if (!keep && !(x == y && xi == yi)) { x = y; xi = yi; }
  };
  if (__any_sync(0xffffffffu, m > 16)) {
    // 32 elements: position p = j (x0) or j + 16 (x1)
#pragma unroll
    for (unsigned k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
      for (unsigned s2 = k2 >> 1; s2 > 0; s2 >>= 1) {
        if (s2 == 16) {  // partners are the lane's own two elements (positions j and j + 16; k2 = 32: ascending)
          if (pair_less(x1, i1, x0, i0)) {
            const double t = x0; x0 = x1; x1 = t;
            const std::uint32_t u = i0; i0 = i1; i1 = u;
          }
        } else {
          cx_shfl(x0, i0, j, k2, s2);
          cx_shfl(x1, i1, j + 16, k2, s2);
        }
      }
    }
  } else {
#pragma unroll
    for (unsigned k2 = 2; k2 <= 16; k2 <<= 1) {
#pragma unroll
      for (unsigned s2 = k2 >> 1; s2 > 0; s2 >>= 1) cx_shfl(x0, i0, j, k2, s2);
    }
  }
  if (j < m) {
    ids[o + j] = i0;
    d2[o + j] = x0;
  }
  if (j + 16 < m) {
    ids[o + j + 16] = i1;
    d2[o + j + 16] = x1;
  }
  if (valid && j == 0) flag[i] = over ? 1 : 0;
}


// ------------------------------------------------- range search (box) --
// Orthogonal range search: every live point p with lo_j <= p_j <= hi_j for all j (closed
// box).  Same packet traversal; a child is entered when any lane's query box meets the
// child's fp32 box (both rounded outward: conservative), a staged point is reported when
// it lies in the box in exact fp64 (NaN tombstones never do).  Queries ordered by the K2
// key of their box centres.
template <int D, bool FILL>
__global__ void __launch_bounds__(256) k_range_box(const TreeSet ts, const double* __restrict__ LO,
                                                   const double* __restrict__ HI, const std::uint32_t* __restrict__ perm,
                                                   std::uint64_t nq, unsigned long long* __restrict__ counts,
                                                   const unsigned long long* __restrict__ offs,
                                                   std::uint32_t* __restrict__ out_ids, unsigned* __restrict__ tile_ctr) {
  constexpr int kWarps = 8;
  __shared__ std::uint64_t s_stack[kWarps][kStack];
  __shared__ __align__(16) double s_pts[kWarps][D * GK_MAX_LEAF];
  __shared__ std::uint32_t s_ids[kWarps][GK_MAX_LEAF];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned ntiles = static_cast<unsigned>((nq + 31) / 32);
  while (true) {
    unsigned tile = 0;
    if (lane == 0) tile = atomicAdd(tile_ctr, 1u);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= ntiles) break;
    const std::uint64_t qi = static_cast<std::uint64_t>(tile) * 32 + lane;
    const bool active = qi < nq;
    std::uint32_t orig = 0;
    double lo[D], hi[D];
    float flo[D], fhi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { lo[j] = 1.0; hi[j] = -1.0; }  // inactive lanes: empty box
    if (active) {
      orig = perm[qi];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        lo[j] = LO[static_cast<std::uint64_t>(orig) * D + j];
        hi[j] = HI[static_cast<std::uint64_t>(orig) * D + j];
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      flo[j] = __double2float_rd(lo[j]);
      fhi[j] = __double2float_ru(hi[j]);
    }
    unsigned long long cnt = 0;
    const unsigned long long base = (FILL && active) ? offs[orig] : 0ULL;
    for (int t = 0; t < ts.count; ++t) {
      const float* __restrict__ nodes = static_cast<const float*>(ts.t[t].tnodes);
      const double* __restrict__ coords = ts.t[t].coords;
      const std::uint32_t* __restrict__ ids = ts.t[t].ids;
      const std::uint64_t stride = ts.t[t].stride;
      std::uint64_t ref = ts.t[t].root;
      int sp = 0;
      while (true) {
        if (is_leaf_ref(ref)) {
          const std::uint32_t c = leaf_count(ref);
          const std::uint64_t s = leaf_start(ref);
          __syncwarp();
          stage_leaf<D>(s_pts[w], s_ids[w], coords, ids, stride, s, c, lane, FILL);
          stage_wait();
          __syncwarp();
          for (std::uint32_t p = 0; p < c; ++p) {
            bool in = true;
#pragma unroll
            for (int j = 0; j < D; ++j) {
              const double x = s_pts[w][j * GK_MAX_LEAF + p];
              in = in && (lo[j] <= x) && (x <= hi[j]);
            }
            if (in) {
              if (FILL) out_ids[base + cnt] = s_ids[w][p];
              ++cnt;
            }
          }
        } else {
          const TNode<D>* nd = reinterpret_cast<const TNode<D>*>(nodes) + ref;
          bool w0 = true, w1 = true;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const float2 l = *reinterpret_cast<const float2*>(nd->lo[j]);
            const float2 h = *reinterpret_cast<const float2*>(nd->hi[j]);
            w0 = w0 && l.x <= fhi[j] && h.x >= flo[j];
            w1 = w1 && l.y <= fhi[j] && h.y >= flo[j];
          }
          w0 = w0 && active;
          w1 = w1 && active;
          const std::uint64_t r0 = nd->ref[0], r1 = nd->ref[1];
          const unsigned b0 = __ballot_sync(0xffffffffu, w0), b1 = __ballot_sync(0xffffffffu, w1);
          if (b0 && b1) {
            if (lane == 0) s_stack[w][sp] = r1;
            ++sp;
            ref = r0;
            continue;
          } else if (b0) {
            ref = r0;
            continue;
          } else if (b1) {
            ref = r1;
            continue;
          }
        }
        __syncwarp();
        if (sp == 0) break;
        ref = s_stack[w][--sp];
      }
    }
    if (active && !FILL) counts[orig] = cnt;
  }
}

__global__ void k_box_centre(const double* __restrict__ lo, const double* __restrict__ hi, std::uint64_t n,
                             double* __restrict__ c) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) c[i] = 0.5 * lo[i] + 0.5 * hi[i];  // finite for any finite box
}

template <int D>
void range_box_d(const TreeSet& ts, const double* lo, const double* hi, std::uint64_t nq, unsigned long long* counts,
                 const unsigned long long* offs, std::uint32_t* ids, bool fill, const std::uint32_t* perm, cudaStream_t st) {
  static int grids[kMaxDevices] = {};
  static std::once_flag once[kMaxDevices];
  const int dev = current_device();
  int& grid = grids[dev];
  std::call_once(once[dev], [&] {
    int sms = 0, per0 = 0, per1 = 0;
    GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per0, k_range_box<D, false>, 256, 0));
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_range_box<D, true>, 256, 0));
    grid = std::max(1, std::min(per0, per1)) * sms;
  });
  const unsigned g = static_cast<unsigned>(std::min<std::uint64_t>(grid, (nq + 255) / 256));
  unsigned* tile_ctr = nullptr;
  GK_CUDA(cudaMallocAsync(&tile_ctr, sizeof(unsigned), st));
  GK_CUDA(cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned), st));
  if (fill) k_range_box<D, true><<<g, 256, 0, st>>>(ts, lo, hi, perm, nq, counts, offs, ids, tile_ctr);
  else k_range_box<D, false><<<g, 256, 0, st>>>(ts, lo, hi, perm, nq, counts, offs, ids, tile_ctr);
  GK_CHECK_LAUNCH();
  GK_CUDA(cudaFreeAsync(tile_ctr, st));
}

}  // namespace

void knn_launch(int d, int k, const TreeSet& trees, const double* q_dev, std::uint64_t nq, std::uint32_t* ids_dev,
                double* d2_dev, gk_knn_counters* counters, cudaStream_t st, cudaEvent_t ev_k0, cudaEvent_t ev_k1,
                const double* bound) {
  if (nq == 0) return;
  if (nq >= 0xffffffffULL) throw Error(GK_ERR_INVALID, "kNN batch larger than 2^32-1 queries");
  std::uint32_t* perm = nullptr;
  GK_CUDA(cudaMallocAsync(&perm, nq * 4, st));
  unsigned long long* ctr = nullptr;
  if (counters) {
    GK_CUDA(cudaMallocAsync(&ctr, 10 * sizeof(unsigned long long), st));
    GK_CUDA(cudaMemsetAsync(ctr, 0, 10 * sizeof(unsigned long long), st));
  }
  switch (d) {
#define GK_D(DD)                                                   \
  case DD:                                                         \
    order_queries<DD>(q_dev, nq, perm, st);                        \
    if (ev_k0) GK_CUDA(cudaEventRecord(ev_k0, st));                \
    launch_d<DD>(k, trees, q_dev, perm, nq, ids_dev, d2_dev, ctr, st, bound); \
    if (ev_k1) GK_CUDA(cudaEventRecord(ev_k1, st));                \
    break;
    GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
  GK_CHECK_LAUNCH();
  if (counters) {
    unsigned long long h[10];
    GK_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    counters->node_bytes = h[0];
    counters->leaf_bytes = h[1];
    counters->nodes = h[2];
    counters->leaves = h[3];
    counters->dists = h[4];
    counters->warp_nodes = h[5];
    counters->warp_leaves = h[6];
    counters->inserts = h[7];
    counters->warp_leaf_points = h[8];
    counters->warp_inserts = h[9];
    GK_CUDA(cudaFreeAsync(ctr, st));
  }
  GK_CUDA(cudaFreeAsync(perm, st));
}

// K1 alone over queries already ordered by range_order (the pinned host pipeline orders chunk c + 1 on a
// side stream while chunk c is traversed)
void knn_traverse(int d, int k, const TreeSet& trees, const double* q_dev, const std::uint32_t* perm, std::uint64_t nq,
                  std::uint32_t* ids_dev, double* d2_dev, cudaStream_t st) {
  if (nq == 0) return;
  if (nq >= 0xffffffffULL) throw Error(GK_ERR_INVALID, "kNN batch larger than 2^32-1 queries");
  switch (d) {
#define GK_D(DD) case DD: launch_d<DD>(k, trees, q_dev, perm, nq, ids_dev, d2_dev, nullptr, st, nullptr); break;
    GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
  GK_CHECK_LAUNCH();
}

void range_order(int d, const double* q_dev, std::uint64_t nq, std::uint32_t* perm, cudaStream_t st) {
  switch (d) {
#define GK_D(DD) case DD: order_queries<DD>(q_dev, nq, perm, st); break;
    GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

void range_launch(int d, const TreeSet& trees, const double* q_dev, std::uint64_t nq, double r2, const double* r2q,
                  const std::uint32_t* perm,
                  unsigned long long* counts, const unsigned long long* offs, std::uint32_t* ids, double* d2, int mode,
                  unsigned capq, cudaStream_t st) {
  if (nq == 0) return;
  switch (d) {
#define GK_D(DD)                                                                                                \
  case DD:                                                                                                      \
    range_d<DD>(trees, q_dev, nq, r2, r2q, counts, const_cast<unsigned long long*>(offs), ids, d2, mode, capq,      \
                const_cast<std::uint32_t*>(perm), st);                                                          \
    break;
    GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

std::uint64_t range_slots_compact(std::uint64_t nq, unsigned capq, const std::uint32_t* perm,
                                  const unsigned long long* counts, const unsigned long long* offs, const std::uint32_t* ti,
                                  const double* td, std::uint32_t* ids, double* d2, std::uint32_t* ovf, cudaStream_t st) {
  if (capq != kRangeSortCap) throw Error(GK_ERR_LOGIC, "k_slots_compact is written for 32 slots per query");
  std::uint8_t* flag = nullptr;
  unsigned long long* nsel = nullptr;
  GK_CUDA(cudaMallocAsync(&flag, nq, st));
  GK_CUDA(cudaMallocAsync(&nsel, 8, st));
  k_slots_compact<<<static_cast<unsigned>((nq * 16 + 255) / 256), 256, 0, st>>>(nq, capq, perm, counts, offs, ti, td, ids,
                                                                              d2, flag);
  GK_CHECK_LAUNCH();
  std::size_t tb = 0;
  void* tmp = nullptr;
  GK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, perm, flag, ovf, nsel, static_cast<long long>(nq), st));
  GK_CUDA(cudaMallocAsync(&tmp, tb, st));
  GK_CUDA(cub::DeviceSelect::Flagged(tmp, tb, perm, flag, ovf, nsel, static_cast<long long>(nq), st));
  unsigned long long h = 0;
  GK_CUDA(cudaMemcpyAsync(&h, nsel, 8, cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(flag, st));
  GK_CUDA(cudaFreeAsync(nsel, st));
  return h;
}

// Each query's rows sorted by (d2, id): an id sort, then a stable d2 sort, per segment.
void range_sort(std::uint32_t* ids, double* d2, std::uint64_t total, const unsigned long long* offs, std::uint64_t nq,
                cudaStream_t st) {
  if (total == 0) return;
  if (total > 0x7fffffffULL || nq > 0x7fffffffULL)
    throw Error(GK_ERR_UNSUPPORTED, "range result larger than 2^31-1 rows");
  std::uint32_t* ids2 = nullptr;
  double* d22 = nullptr;
  GK_CUDA(cudaMallocAsync(&ids2, total * 4, st));
  GK_CUDA(cudaMallocAsync(&d22, total * 8, st));
  const int ni = static_cast<int>(total), ns = static_cast<int>(nq);
  std::size_t b1 = 0, b2 = 0;
  GK_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, b1, ids, ids2, d2, d22, ni, ns, offs, offs + 1, st));
  GK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, b2, d22, d2, ids2, ids, ni, ns, offs, offs + 1, st));
  void* tmp = nullptr;
  GK_CUDA(cudaMallocAsync(&tmp, std::max(b1, b2), st));
  std::size_t tb = std::max(b1, b2);
  GK_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp, tb, ids, ids2, d2, d22, ni, ns, offs, offs + 1, st));
  tb = std::max(b1, b2);
  GK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, d22, d2, ids2, ids, ni, ns, offs, offs + 1, st));
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(ids2, st));
  GK_CUDA(cudaFreeAsync(d22, st));
}

__global__ void k_ovf_segments(const std::uint32_t* __restrict__ ovf, std::uint64_t no,
                               const unsigned long long* __restrict__ offs, unsigned long long* beg,
                               unsigned long long* end) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= no) return;
  beg[i] = offs[ovf[i]];
  end[i] = offs[ovf[i] + 1];
}

// The slot path sorted every query's rows while compacting them; only the `no` overflowing queries (ovf),
// whose rows the second traversal wrote in arbitrary order, still need the segmented (id, then stable d2) sort.
void range_sort_ovf(std::uint32_t* ids, double* d2, std::uint64_t total, const unsigned long long* offs,
                    const std::uint32_t* ovf, std::uint64_t no, cudaStream_t st) {
  if (total == 0 || no == 0) return;
  if (total > 0x7fffffffULL || no > 0x7fffffffULL)
    throw Error(GK_ERR_UNSUPPORTED, "range result larger than 2^31-1 rows");
  std::uint32_t* ids2 = nullptr;
  double* d22 = nullptr;
  unsigned long long *beg = nullptr, *end = nullptr;
  GK_CUDA(cudaMallocAsync(&ids2, total * 4, st));
  GK_CUDA(cudaMallocAsync(&d22, total * 8, st));
  GK_CUDA(cudaMallocAsync(&beg, no * 8, st));
  GK_CUDA(cudaMallocAsync(&end, no * 8, st));
  k_ovf_segments<<<static_cast<unsigned>((no + 255) / 256), 256, 0, st>>>(ovf, no, offs, beg, end);
  GK_CHECK_LAUNCH();
  const int ni = static_cast<int>(total), ns = static_cast<int>(no);
  std::size_t b1 = 0, b2 = 0;
  GK_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, b1, ids, ids2, d2, d22, ni, ns, beg, end, st));
  GK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, b2, d22, d2, ids2, ids, ni, ns, beg, end, st));
  void* tmp = nullptr;
  GK_CUDA(cudaMallocAsync(&tmp, std::max(b1, b2), st));
  std::size_t tb = std::max(b1, b2);
  GK_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp, tb, ids, ids2, d2, d22, ni, ns, beg, end, st));
  tb = std::max(b1, b2);
  GK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, d22, d2, ids2, ids, ni, ns, beg, end, st));
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(ids2, st));
  GK_CUDA(cudaFreeAsync(d22, st));
  GK_CUDA(cudaFreeAsync(beg, st));
  GK_CUDA(cudaFreeAsync(end, st));
}

// kNN graph (ParGeo's k-NN graph generator over kd-tree kNN): every live point
// as a query (rows in ascending id order), kNN_L with k + 1, the point itself dropped.
void knn_graph_launch(int d, int k, const TreeSet& ts, std::uint64_t n, std::uint32_t* row_ids, std::uint32_t* ids,
                      double* d2, cudaStream_t st) {
  if (n == 0) return;
  if (n > 0x7fffffffULL) throw Error(GK_ERR_UNSUPPORTED, "kNN graph over more than 2^31-1 points");
  double *pts = nullptr, *q = nullptr, *td = nullptr;
  std::uint32_t *uid = nullptr, *pos = nullptr, *src = nullptr, *ti = nullptr;
  unsigned long long* ctr = nullptr;
  GK_CUDA(cudaMallocAsync(&pts, n * d * 8, st));
  GK_CUDA(cudaMallocAsync(&q, n * d * 8, st));
  GK_CUDA(cudaMallocAsync(&uid, n * 4, st));
  GK_CUDA(cudaMallocAsync(&pos, n * 4, st));
  GK_CUDA(cudaMallocAsync(&src, n * 4, st));
  GK_CUDA(cudaMallocAsync(&ctr, 8, st));
  GK_CUDA(cudaMemsetAsync(ctr, 0, 8, st));
  k_live_gather<<<static_cast<unsigned>(std::min<std::uint64_t>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(ts, d, pts, uid,
                                                                                                          pos, ctr);
  GK_CHECK_LAUNCH();
  unsigned long long got = 0;
  GK_CUDA(cudaMemcpyAsync(&got, ctr, 8, cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  if (got != n) throw Error(GK_ERR_LOGIC, "kNN graph: live point count mismatch");
  void* tmp = nullptr;
  std::size_t tb = 0;
  GK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, uid, row_ids, pos, src, static_cast<int>(n), 0, 32, st));
  GK_CUDA(cudaMallocAsync(&tmp, tb, st));
  GK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, uid, row_ids, pos, src, static_cast<int>(n), 0, 32, st));
  k_gather_rows<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pts, src, n, d, q);
  GK_CHECK_LAUNCH();
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(pts, st));
  GK_CUDA(cudaFreeAsync(uid, st));
  GK_CUDA(cudaFreeAsync(pos, st));
  GK_CUDA(cudaFreeAsync(src, st));
  GK_CUDA(cudaFreeAsync(ctr, st));
  GK_CUDA(cudaMallocAsync(&ti, n * (k + 1) * 4, st));
  GK_CUDA(cudaMallocAsync(&td, n * (k + 1) * 8, st));
  knn_launch(d, k + 1, ts, q, n, ti, td, nullptr, st, nullptr, nullptr);
  k_drop_self<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, k, row_ids, ti, td, ids, d2);
  GK_CHECK_LAUNCH();
  GK_CUDA(cudaFreeAsync(q, st));
  GK_CUDA(cudaFreeAsync(ti, st));
  GK_CUDA(cudaFreeAsync(td, st));
}

void range_box_order(int d, const double* lo, const double* hi, std::uint64_t nq, std::uint32_t* perm, cudaStream_t st) {
  double* c = nullptr;
  GK_CUDA(cudaMallocAsync(&c, nq * d * 8, st));
  k_box_centre<<<static_cast<unsigned>((nq * d + 255) / 256), 256, 0, st>>>(lo, hi, nq * d, c);
  GK_CHECK_LAUNCH();
  range_order(d, c, nq, perm, st);
  GK_CUDA(cudaFreeAsync(c, st));
}

void range_box_launch(int d, const TreeSet& trees, const double* lo, const double* hi, std::uint64_t nq,
                      const std::uint32_t* perm, unsigned long long* counts, const unsigned long long* offs,
                      std::uint32_t* ids, bool fill, cudaStream_t st) {
  if (nq == 0) return;
  switch (d) {
#define GK_D(DD) case DD: range_box_d<DD>(trees, lo, hi, nq, counts, offs, ids, fill, perm, st); break;
    GK_D(2) GK_D(3) GK_D(4) GK_D(5) GK_D(6) GK_D(7) GK_D(8)
#undef GK_D
    default: throw Error(GK_ERR_INVALID, "unsupported dimension " + std::to_string(d));
  }
}

// each query's rows in ascending id order
void range_box_sort(std::uint32_t* ids, std::uint64_t total, const unsigned long long* offs, std::uint64_t nq,
                    cudaStream_t st) {
  if (total == 0) return;
  if (total > 0x7fffffffULL || nq > 0x7fffffffULL)
    throw Error(GK_ERR_UNSUPPORTED, "range result larger than 2^31-1 rows");
  std::uint32_t* ids2 = nullptr;
  GK_CUDA(cudaMallocAsync(&ids2, total * 4, st));
  const int ni = static_cast<int>(total), ns = static_cast<int>(nq);
  std::size_t tb = 0;
  GK_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, ids, ids2, ni, ns, offs, offs + 1, st));
  void* tmp = nullptr;
  GK_CUDA(cudaMallocAsync(&tmp, tb, st));
  GK_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, tb, ids, ids2, ni, ns, offs, offs + 1, st));
  GK_CUDA(cudaMemcpyAsync(ids, ids2, total * 4, cudaMemcpyDeviceToDevice, st));
  GK_CUDA(cudaFreeAsync(tmp, st));
  GK_CUDA(cudaFreeAsync(ids2, st));
}

}  // namespace gk
