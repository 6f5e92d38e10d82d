// gk_oracle.cpp — CPU ORACLE for the BDL-tree kNN_L / BuildvEB_S hot path.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2207_01834_b200/)
// links, loads or calls this file; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may.  It is the checker the
// CUDA path is compared against, and the "reference CPU path" timed beside it.
//
// It is a restatement, in plain C++17 + OpenMP (TBB/Eigen are absent here), of
//   * PAPER.md Alg. 1 BuildvEB_S
//   * PAPER.md Alg. 2 Erase_S
//   * PAPER.md kNN_S / data-parallel kNN
//   * PAPER.md Alg. 3 Insert_L, Alg. 4 Erase_L
//   * PAPER.md implementation details            (leaf 16, X=1024,
//                                                  spatial median, largest->smallest trees)
//   * SPEC.md kdtree / bdltree contracts
//   * geokit/kdtree/knn_buffer.hpp:20-67 (KnnBuffer, restated below as KnnBuf)
//   * geokit/core/rng.hpp:10-66 (SplitMix64 counter Rng, restated below)
//   * geokit/generators.hpp:44-63 (per-point split streams, Box-Muller)
// The reference ships no implementation of the tree itself;
// every ambiguity is frozen here and listed in DESIGN.md "Frozen decisions".
//
// Parity pins: KnnBuf and Rng are checked bit-for-bit against the reference's
// own headers compiled into oracle/_ref (tests/test_oracle_pins.py).  The tree
// algorithms have no reference implementation to run: they are
// pinned only by the SPEC known-answer examples and an exact brute-force scan
// (tests/test_oracle.py) — beyond those, tree-level parity is unpinned.
// Floating point: compile with -ffp-contract=off; squared distance is
// sum_{j=0..D-1} (q_j - p_j)^2 accumulated left-to-right, no FMA.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#include <omp.h>

namespace gko {

using Id = std::uint32_t;
constexpr Id kNoPoint = 0xffffffffu;  // geokit/core/point.hpp:18-19
constexpr int kMaxDim = 8;            // dispatch_dim covers 2..8 (point.hpp:22-35)
constexpr int kDepthCap = 40;         // frozen: depth >= 40 -> object-median split

// ---------------------------------------------------------------- Rng ------
// SplitMix64 finalizer + counter stream (rng.hpp:10-48).
static inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) { return mix64(mix64(a) ^ b); }
static inline double unit_double(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

struct Rng {
  std::uint64_t seed_, ctr_ = 0;
  explicit Rng(std::uint64_t seed) : seed_(mix64(seed)) {}
  std::uint64_t next_u64() { return mix64(seed_, ctr_++); }
  double next_double() { return unit_double(next_u64()); }
  std::uint64_t next_below(std::uint64_t n) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
  }
  Rng split(std::uint64_t stream) const { return Rng(mix64(seed_, ~stream)); }
};

// Box-Muller normal (generators.hpp:44-50).
static inline double gaussian(Rng& r) {
  double u1 = unit_double(r.next_u64());
  double u2 = r.next_double();
  u1 = 1.0 - u1;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// ----------------------------------------------------------- KnnBuf --------
// Restatement of geokit::kdtree::KnnBuffer (knn_buffer.hpp:20-67): 2k slots of
// (sqdist, id), lexicographic order, compaction = nth_element at k-1.
struct KnnBuf {
  using Entry = std::pair<double, Id>;
  std::size_t k;
  std::vector<Entry> e;
  Entry bound{std::numeric_limits<double>::infinity(), kNoPoint};
  std::size_t compactions = 0;
  explicit KnnBuf(std::size_t kk) : k(kk) { e.reserve(2 * kk); }
  void insert(Id id, double d) {
    Entry x{d, id};
    if (!(x < bound)) return;  // (knn_buffer.hpp:36) e >= bound_  (pair order)
    if (e.size() == 2 * k) compact();
    if (x < bound) e.push_back(x);
  }
  void compact() {
    std::nth_element(e.begin(), e.begin() + (k - 1), e.end());
    bound = e[k - 1];
    e.resize(k);
    ++compactions;
  }
  std::vector<Entry> extract() {
    std::sort(e.begin(), e.end());
    if (e.size() > k) e.resize(k);
    return e;
  }
};

// Canonical squared distance (frozen decision 1).
static inline double sqdist(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int j = 0; j < d; ++j) {
    double t = a[j] - b[j];
    double t2 = t * t;
    s = s + t2;
  }
  return s;
}

static inline std::uint64_t hyperceiling(std::uint64_t x) {
  std::uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ------------------------------------------------------------- Tree --------
// Canonical node record.  Exported verbatim for the GPU
// parity check (same struct as gk_canon_node in include/gk_bdl.h).
struct Node {
  std::int32_t kind;   // 0 internal, 1 leaf
  std::int32_t dim;    // split dim (internal), -1 for leaf
  std::int32_t mode;   // 0 spatial median, 1 object median (internal)
  std::int32_t depth;
  double split;        // split value (internal)
  std::int32_t left, right;  // child slots (internal), -1 for leaf
  std::uint32_t start, count;  // point range (contiguous, leaf order)
  double lo[kMaxDim], hi[kMaxDim];
};
static_assert(sizeof(Node) == 168, "canonical node layout");

struct TmpNode {
  Node n{};
  std::unique_ptr<TmpNode> l, r;
  int32_t slot = -1;
};

struct Tree {
  int d = 0;
  std::size_t n = 0;
  std::vector<double> pts;   // AoS in leaf order
  std::vector<Id> ids;
  std::vector<std::uint8_t> dead;
  std::vector<Node> nodes;   // vEB slots
  std::int32_t root = -1;
  int height = 0;
  std::size_t build_size = 0, live = 0;
};

struct BuildCtx {
  int d, leaf, heuristic;
  double* pts;
  Id* ids;
  std::vector<double> tmp_pts;
  std::vector<Id> tmp_ids;
};

// Stable partition of [s, s+c) by predicate pred(i) (frozen decision 3).
template <class Pred>
static std::size_t stable_partition_range(BuildCtx& B, std::size_t s, std::size_t c, Pred pred) {
  const int d = B.d;
  std::size_t nl = 0;
  for (std::size_t i = s; i < s + c; ++i) nl += pred(i) ? 1 : 0;
  std::size_t il = s, ir = s + nl;
  for (std::size_t i = s; i < s + c; ++i) {
    std::size_t o = pred(i) ? il++ : ir++;
    std::memcpy(&B.tmp_pts[o * d], &B.pts[i * d], sizeof(double) * d);
    B.tmp_ids[o] = B.ids[i];
  }
  std::memcpy(&B.pts[s * d], &B.tmp_pts[s * d], sizeof(double) * d * c);
  std::memcpy(&B.ids[s], &B.tmp_ids[s], sizeof(Id) * c);
  return nl;
}

// Topology build (Alg. 1 split rule).
static std::unique_ptr<TmpNode> build_rec(BuildCtx& B, std::size_t s, std::size_t c, int depth) {
  auto t = std::make_unique<TmpNode>();
  Node& nd = t->n;
  const int d = B.d;
  nd.depth = depth;
  nd.start = static_cast<std::uint32_t>(s);
  nd.count = static_cast<std::uint32_t>(c);
  for (int j = 0; j < kMaxDim; ++j) { nd.lo[j] = 0.0; nd.hi[j] = 0.0; }
  for (int j = 0; j < d; ++j) { nd.lo[j] = B.pts[s * d + j]; nd.hi[j] = B.pts[s * d + j]; }
  for (std::size_t i = s + 1; i < s + c; ++i)
    for (int j = 0; j < d; ++j) {
      double x = B.pts[i * d + j];
      nd.lo[j] = std::min(nd.lo[j], x);
      nd.hi[j] = std::max(nd.hi[j], x);
    }
  if (c <= static_cast<std::size_t>(B.leaf)) {
    nd.kind = 1; nd.dim = -1; nd.mode = 0; nd.split = 0.0; nd.left = nd.right = -1;
    return t;
  }
  nd.kind = 0;
  const int cd = depth % d;
  nd.dim = cd;
  std::size_t nl = 0;
  bool object = (B.heuristic == 1) || depth >= kDepthCap;
  if (!object) {
    // spatial median: s = (lo + hi) / 2, left x_c < s <= right (frozen decision 4)
    double sp = (nd.lo[cd] + nd.hi[cd]) / 2.0;
    std::size_t cnt = 0;
    for (std::size_t i = s; i < s + c; ++i) cnt += (B.pts[i * d + cd] < sp) ? 1 : 0;
    if (cnt == 0 || cnt == c) {
      object = true;  // degenerate: fall back to object median
    } else {
      nl = stable_partition_range(B, s, c, [&](std::size_t i) { return B.pts[i * d + cd] < sp; });
      nd.mode = 0;
      nd.split = sp;
    }
  }
  if (object) {
    // object median by (x_c, id): left = the floor(c/2) smallest keys (frozen decision 5)
    std::vector<std::pair<double, Id>> keys(c);
    for (std::size_t i = 0; i < c; ++i) keys[i] = {B.pts[(s + i) * d + cd], B.ids[s + i]};
    std::size_t m = c / 2;
    std::nth_element(keys.begin(), keys.begin() + m, keys.end());
    const auto thr = keys[m];
    nl = stable_partition_range(B, s, c, [&](std::size_t i) {
      return std::make_pair(B.pts[i * d + cd], B.ids[i]) < thr;
    });
    nd.mode = 1;
    nd.split = thr.first;
  }
  if (c >= 1000) {  // serial base case below 1000 points
#pragma omp task shared(B, t)
    t->l = build_rec(B, s, nl, depth + 1);
#pragma omp task shared(B, t)
    t->r = build_rec(B, s + nl, c - nl, depth + 1);
#pragma omp taskwait
  } else {
    t->l = build_rec(B, s, nl, depth + 1);
    t->r = build_rec(B, s + nl, c - nl, depth + 1);
  }
  return t;
}

static int tree_height(const TmpNode* t) {
  if (!t) return 0;
  return 1 + std::max(tree_height(t->l.get()), tree_height(t->r.get()));
}

static void collect_at_depth(TmpNode* t, int rel, std::vector<TmpNode*>& out) {
  if (!t) return;
  if (rel == 0) { out.push_back(t); return; }
  collect_at_depth(t->l.get(), rel - 1, out);
  collect_at_depth(t->r.get(), rel - 1, out);
}

// Topology-driven vEB layout (Alg. 1 lines 6-9, frozen decision 6): place the
// nodes of depth < l under r starting at slot `base`; returns #nodes placed.
// l_b = hyperceiling(floor((l+1)/2)), l_t = l - l_b (Fig. vebconstruct).
static std::size_t veb_layout(TmpNode* r, int l, std::size_t base) {
  if (!r) return 0;
  if (l == 1) { r->slot = static_cast<int32_t>(base); return 1; }
  int lb = static_cast<int>(hyperceiling(static_cast<std::uint64_t>((l + 1) / 2)));
  int lt = l - lb;
  std::size_t top = veb_layout(r, lt, base);
  std::vector<TmpNode*> bottoms;
  collect_at_depth(r, lt, bottoms);
  std::size_t off = base + top;
  for (TmpNode* b : bottoms) off += veb_layout(b, lb, off);
  return off - base;
}

static void emit_nodes(TmpNode* t, std::vector<Node>& nodes) {
  if (!t) return;
  Node nd = t->n;
  if (nd.kind == 0) {
    nd.left = t->l->slot;
    nd.right = t->r->slot;
  }
  nodes[t->slot] = nd;
  emit_nodes(t->l.get(), nodes);
  emit_nodes(t->r.get(), nodes);
}

// BuildvEB_S over (pts AoS, ids) in the given (pool) order.
static void build_tree(Tree& T, int d, const double* pts, const Id* ids, std::size_t n, int leaf, int heuristic) {
  T = Tree();
  T.d = d;
  T.n = n;
  T.pts.assign(pts, pts + n * d);
  T.ids.assign(ids, ids + n);
  T.dead.assign(n, 0);
  T.build_size = n;
  T.live = n;
  if (n == 0) return;
  BuildCtx B{d, leaf, heuristic, T.pts.data(), T.ids.data(), std::vector<double>(n * d), std::vector<Id>(n)};
  std::unique_ptr<TmpNode> root;
  if (n >= 1000 && omp_get_max_threads() > 1 && !omp_in_parallel()) {
#pragma omp parallel
#pragma omp single
    root = build_rec(B, 0, n, 0);
  } else {
    root = build_rec(B, 0, n, 0);
  }
  T.height = tree_height(root.get());
  std::size_t total = veb_layout(root.get(), T.height, 0);
  T.nodes.assign(total, Node{});
  emit_nodes(root.get(), T.nodes);
  T.root = 0;
  // free the pointer tree iteratively-ish (recursion depth bounded by height)
}

// --------------------------------------------------------------- kNN_S -----
static inline double mindist2(const double* q, const Node& nd, int d) {
  double s = 0.0;
  for (int j = 0; j < d; ++j) {
    double t = 0.0;
    if (q[j] < nd.lo[j]) t = nd.lo[j] - q[j];
    else if (q[j] > nd.hi[j]) t = q[j] - nd.hi[j];
    double t2 = t * t;
    s = s + t2;
  }
  return s;
}
static inline double maxdist2(const double* q, const Node& nd, int d) {
  double s = 0.0;
  for (int j = 0; j < d; ++j) {
    double t = std::max(std::fabs(q[j] - nd.lo[j]), std::fabs(nd.hi[j] - q[j]));
    double t2 = t * t;
    s = s + t2;
  }
  return s;
}

struct KnnStats { std::uint64_t nodes = 0, leaves = 0, dists = 0; };

static void insert_range(const Tree& T, const double* q, std::uint32_t s, std::uint32_t c, KnnBuf& buf, KnnStats* st) {
  const int d = T.d;
  for (std::uint32_t i = s; i < s + c; ++i) {
    if (T.dead[i]) continue;
    buf.insert(T.ids[i], sqdist(q, &T.pts[static_cast<std::size_t>(i) * d], d));
    if (st) st->dists++;
  }
}

// kNN_S: descend to q's leaf, then while unwinding:
// sibling-fill while the buffer holds fewer than k entries; otherwise
// include-all / prune / recurse against the buffer's k-th bound (strict prune,
// frozen decision 2).
static void knn_rec(const Tree& T, std::int32_t slot, const double* q, KnnBuf& buf, KnnStats* st) {
  const Node& nd = T.nodes[slot];
  if (st) st->nodes++;
  if (nd.kind == 1) {
    if (st) st->leaves++;
    insert_range(T, q, nd.start, nd.count, buf, st);
    return;
  }
  const bool goleft = q[nd.dim] < nd.split;
  const std::int32_t near = goleft ? nd.left : nd.right;
  const std::int32_t far = goleft ? nd.right : nd.left;
  knn_rec(T, near, q, buf, st);
  const Node& f = T.nodes[far];
  if (buf.e.size() < buf.k) {
    if (st) st->nodes++;
    insert_range(T, q, f.start, f.count, buf, st);
    return;
  }
  const double bd = buf.bound.first;
  if (mindist2(q, f, T.d) > bd) return;
  if (maxdist2(q, f, T.d) < bd) {
    if (st) st->nodes++;
    insert_range(T, q, f.start, f.count, buf, st);
    return;
  }
  knn_rec(T, far, q, buf, st);
}

static void knn_single(const Tree& T, const double* q, KnnBuf& buf, KnnStats* st) {
  if (T.root < 0 || T.live == 0) return;
  knn_rec(T, T.root, q, buf, st);
}

// ------------------------------------------------------------ Erase_S -----
static inline bool in_box(const double* p, const Node& nd, int d) {
  for (int j = 0; j < d; ++j)
    if (p[j] < nd.lo[j] || p[j] > nd.hi[j]) return false;
  return true;
}

// Alg. 2: route the batch down by the children's boxes
// (frozen decision 9), tombstone coordinate-exact matches in leaves, collapse
// single-child nodes.  Returns the surviving slot or -1.
static std::int32_t erase_rec(Tree& T, std::int32_t slot, const std::vector<const double*>& Q, std::size_t& killed) {
  Node& nd = T.nodes[slot];
  const int d = T.d;
  if (nd.kind == 1) {
    bool any_live = false;
    for (std::uint32_t i = nd.start; i < nd.start + nd.count; ++i) {
      if (T.dead[i]) continue;
      const double* p = &T.pts[static_cast<std::size_t>(i) * d];
      for (const double* x : Q) {
        bool eq = true;
        for (int j = 0; j < d; ++j) eq = eq && (x[j] == p[j]);
        if (eq) { T.dead[i] = 1; ++killed; break; }
      }
      if (!T.dead[i]) any_live = true;
    }
    return any_live ? slot : -1;
  }
  std::vector<const double*> QL, QR;
  const Node& L = T.nodes[nd.left];
  const Node& R = T.nodes[nd.right];
  for (const double* x : Q) {
    if (in_box(x, L, d)) QL.push_back(x);
    if (in_box(x, R, d)) QR.push_back(x);
  }
  std::int32_t nl = QL.empty() ? nd.left : erase_rec(T, nd.left, QL, killed);
  std::int32_t nr = QR.empty() ? nd.right : erase_rec(T, nd.right, QR, killed);
  if (nl >= 0 && nr >= 0) { nd.left = nl; nd.right = nr; return slot; }
  if (nl < 0 && nr < 0) return -1;
  return nl >= 0 ? nl : nr;
}

static std::size_t erase_static(Tree& T, const double* P, std::size_t np) {
  if (T.root < 0 || T.live == 0 || np == 0) return 0;
  std::vector<const double*> Q;
  Q.reserve(np);
  const Node& r = T.nodes[T.root];
  for (std::size_t i = 0; i < np; ++i)
    if (in_box(P + i * T.d, r, T.d)) Q.push_back(P + i * T.d);
  if (Q.empty()) return 0;
  std::size_t killed = 0;
  T.root = erase_rec(T, T.root, Q, killed);
  T.live -= killed;
  return killed;
}

// --------------------------------------------------------------- BDL ------
struct Bdl {
  int d;
  std::uint64_t X;
  int leaf, heuristic;
  std::vector<double> buf_pts;   // buffer points, arrival order (AoS)
  std::vector<Id> buf_ids;
  Tree buf_tree;
  std::vector<Tree> statics;     // statics[i] capacity X * 2^i
  std::uint64_t F = 0;
  std::uint64_t next_id = 0;
  int nthreads = 0;
};

static void rebuild_buffer(Bdl& b) {
  build_tree(b.buf_tree, b.d, b.buf_pts.data(), b.buf_ids.data(), b.buf_ids.size(), b.leaf, b.heuristic);
}

static void gather_live(const Tree& T, std::vector<double>& pts, std::vector<Id>& ids) {
  for (std::size_t i = 0; i < T.n; ++i) {
    if (T.dead[i]) continue;
    pts.insert(pts.end(), T.pts.begin() + i * T.d, T.pts.begin() + (i + 1) * T.d);
    ids.push_back(T.ids[i]);
  }
}

// Insert_L (Alg. 3; frozen decisions 7-8).
static void insert_l(Bdl& b, const double* P, const Id* ids, std::size_t n) {
  const int d = b.d;
  const std::uint64_t X = b.X;
  const std::size_t r = n % X;
  const std::size_t bulk = n - r;
  // |P| mod X points (the LAST r of P) go to the buffer
  b.buf_pts.insert(b.buf_pts.end(), P + bulk * d, P + n * d);
  b.buf_ids.insert(b.buf_ids.end(), ids + bulk, ids + n);
  std::vector<double> drained_pts;
  std::vector<Id> drained_ids;
  if (b.buf_ids.size() >= X) {  // buffer full: the X oldest drain into P
    drained_pts.assign(b.buf_pts.begin(), b.buf_pts.begin() + X * d);
    drained_ids.assign(b.buf_ids.begin(), b.buf_ids.begin() + X);
    b.buf_pts.erase(b.buf_pts.begin(), b.buf_pts.begin() + X * d);
    b.buf_ids.erase(b.buf_ids.begin(), b.buf_ids.begin() + X);
  }
  if (r > 0 || !drained_ids.empty()) rebuild_buffer(b);
  const std::uint64_t add = (bulk + drained_ids.size()) / X;
  if (add == 0) return;
  const std::uint64_t Fn = b.F + add;
  const std::uint64_t destroyed = b.F & ~Fn;
  const std::uint64_t built = Fn & ~b.F;
  // pool = live points of destroyed trees (ascending index, leaf order) ++ drained ++ bulk
  std::vector<double> pool_pts;
  std::vector<Id> pool_ids;
  for (int i = 0; i < 64; ++i)
    if (destroyed >> i & 1ULL) {
      gather_live(b.statics[i], pool_pts, pool_ids);
      b.statics[i] = Tree();
    }
  pool_pts.insert(pool_pts.end(), drained_pts.begin(), drained_pts.end());
  pool_ids.insert(pool_ids.end(), drained_ids.begin(), drained_ids.end());
  pool_pts.insert(pool_pts.end(), P, P + bulk * d);
  pool_ids.insert(pool_ids.end(), ids, ids + bulk);
  // new trees filled largest-first from contiguous pool slices; with tombstoned
  // sources the pool may be short and the smallest new trees come up short/empty
  std::vector<int> order;
  for (int i = 63; i >= 0; --i)
    if (built >> i & 1ULL) order.push_back(i);
  std::vector<std::size_t> offs(order.size()), cnts(order.size());
  std::size_t off = 0;
  for (std::size_t t = 0; t < order.size(); ++t) {
    std::size_t cap = static_cast<std::size_t>(X) << order[t];
    std::size_t c = std::min(cap, pool_ids.size() - off);
    offs[t] = off; cnts[t] = c; off += c;
  }
  b.F = Fn;
  if (b.statics.size() < 64) b.statics.resize(64);
  for (std::size_t t = 0; t < order.size(); ++t) {  // builds of distinct new trees
    const int i = order[t];
    if (cnts[t] == 0) { b.F &= ~(1ULL << i); b.statics[i] = Tree(); continue; }
    build_tree(b.statics[i], d, pool_pts.data() + offs[t] * d, pool_ids.data() + offs[t], cnts[t], b.leaf, b.heuristic);
  }
}

// Erase_L (Alg. 4).
static std::size_t erase_l(Bdl& b, const double* P, std::size_t n) {
  const int d = b.d;
  std::size_t killed = 0;
  for (int i = 0; i < 64; ++i)
    if (b.F >> i & 1ULL) killed += erase_static(b.statics[i], P, n);
  // buffer: remove every coordinate-exact match, keep arrival order
  {
    std::vector<double> np;
    std::vector<Id> ni;
    bool changed = false;
    for (std::size_t i = 0; i < b.buf_ids.size(); ++i) {
      const double* p = &b.buf_pts[i * d];
      bool hit = false;
      for (std::size_t k = 0; k < n && !hit; ++k) {
        bool eq = true;
        for (int j = 0; j < d; ++j) eq = eq && (P[k * d + j] == p[j]);
        hit = eq;
      }
      if (hit) { changed = true; ++killed; continue; }
      np.insert(np.end(), p, p + d);
      ni.push_back(b.buf_ids[i]);
    }
    if (changed) {
      b.buf_pts.swap(np);
      b.buf_ids.swap(ni);
      rebuild_buffer(b);
    }
  }
  // trees below half of their build size are gathered into R (buffer excluded)
  std::vector<double> R;
  std::vector<Id> Rid;
  for (int i = 0; i < 64; ++i)
    if ((b.F >> i & 1ULL) && 2 * b.statics[i].live < b.statics[i].build_size) {
      gather_live(b.statics[i], R, Rid);
      b.statics[i] = Tree();
      b.F &= ~(1ULL << i);
    }
  if (!Rid.empty()) insert_l(b, R.data(), Rid.data(), Rid.size());
  return killed;
}

// kNN_L: one buffer per query; trees serially
// largest -> smallest, then the buffer tree; queries in parallel.
static void knn_l(const Bdl& b, const double* Q, std::size_t nq, int k, Id* out_ids, double* out_d2,
                  KnnStats* stats) {
  std::vector<const Tree*> trees;
  for (int i = 63; i >= 0; --i)
    if ((b.F >> i & 1ULL) && b.statics[i].live > 0) trees.push_back(&b.statics[i]);
  if (b.buf_tree.live > 0) trees.push_back(&b.buf_tree);
  const int d = b.d;
  std::vector<KnnBuf> bufs;
  bufs.reserve(nq);
  for (std::size_t i = 0; i < nq; ++i) bufs.emplace_back(static_cast<std::size_t>(k));
  std::uint64_t sn = 0, sl = 0, sd = 0;
  for (const Tree* T : trees) {
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : sn, sl, sd)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
      KnnStats st;
      knn_single(*T, Q + i * d, bufs[i], stats ? &st : nullptr);
      sn += st.nodes; sl += st.leaves; sd += st.dists;
    }
  }
  if (stats) { stats->nodes = sn; stats->leaves = sl; stats->dists = sd; }
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
    auto res = bufs[i].extract();
    for (int j = 0; j < k; ++j) {
      if (j < static_cast<int>(res.size())) {
        out_ids[i * k + j] = res[j].second;
        out_d2[i * k + j] = res[j].first;
      } else {
        out_ids[i * k + j] = kNoPoint;
        out_d2[i * k + j] = std::numeric_limits<double>::infinity();
      }
    }
  }
}

// Range search (ball) over one tree (the kd-tree range search of PAPER.md:188-190, 204):
// prune a subtree iff its box's mindist2 > r2; report live leaf points with d2 <= r2.
static void range_rec(const Tree& T, std::int32_t slot, const double* q, double r2,
                      std::vector<std::pair<double, Id>>& out) {
  const Node& nd = T.nodes[slot];
  if (mindist2(q, nd, T.d) > r2) return;
  if (nd.kind == 1) {
    for (std::uint32_t i = nd.start; i < nd.start + nd.count; ++i) {
      if (T.dead[i]) continue;
      const double d2 = sqdist(q, &T.pts[static_cast<std::size_t>(i) * T.d], T.d);
      if (d2 <= r2) out.push_back({d2, T.ids[i]});
    }
    return;
  }
  range_rec(T, nd.left, q, r2, out);
  range_rec(T, nd.right, q, r2, out);
}

// Orthogonal range search over one tree: prune a subtree whose box misses [lo, hi]; report
// live leaf points inside the closed box.
static void range_box_rec(const Tree& T, std::int32_t slot, const double* lo, const double* hi, std::vector<Id>& out) {
  const Node& nd = T.nodes[slot];
  for (int j = 0; j < T.d; ++j)
    if (nd.hi[j] < lo[j] || nd.lo[j] > hi[j]) return;
  if (nd.kind == 1) {
    for (std::uint32_t i = nd.start; i < nd.start + nd.count; ++i) {
      if (T.dead[i]) continue;
      const double* p = &T.pts[static_cast<std::size_t>(i) * T.d];
      bool in = true;
      for (int j = 0; j < T.d; ++j) in = in && lo[j] <= p[j] && p[j] <= hi[j];
      if (in) out.push_back(T.ids[i]);
    }
    return;
  }
  range_box_rec(T, nd.left, lo, hi, out);
  range_box_rec(T, nd.right, lo, hi, out);
}

// every live tree of the structure (order irrelevant: rows sorted by (d2, id))
static void range_l(const Bdl& b, const double* Q, std::size_t nq, double r2,
                    std::vector<std::vector<std::pair<double, Id>>>& res) {
  std::vector<const Tree*> trees;
  for (int i = 63; i >= 0; --i)
    if ((b.F >> i & 1ULL) && b.statics[i].live > 0) trees.push_back(&b.statics[i]);
  if (b.buf_tree.live > 0) trees.push_back(&b.buf_tree);
  res.assign(nq, {});
#pragma omp parallel for schedule(dynamic, 256)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
    for (const Tree* T : trees)
      if (T->root >= 0 && T->live > 0) range_rec(*T, T->root, Q + i * b.d, r2, res[i]);
    std::sort(res[i].begin(), res[i].end());
  }
}

}  // namespace gko

// ===================================================================== C ABI
using namespace gko;

extern "C" {

const char* gko_version() { return "gk_oracle 1"; }
int gko_node_size() { return static_cast<int>(sizeof(Node)); }
std::uint64_t gko_hyperceiling(std::uint64_t x) { return hyperceiling(x); }
void gko_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
int gko_max_threads() { return omp_get_max_threads(); }

// ---- Rng / generators (seeded inputs, generators.hpp:56-63 with side 1)
std::uint64_t gko_mix64(std::uint64_t z) { return mix64(z); }
void gko_rng_u64(std::uint64_t seed, std::uint64_t stream, int use_split, std::uint64_t n, std::uint64_t* out) {
  Rng r(seed);
  if (use_split) r = r.split(stream);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void gko_rng_below(std::uint64_t seed, std::uint64_t bound, std::uint64_t n, std::uint64_t* out) {
  Rng r(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_below(bound);
}
void gko_random_permutation(std::uint64_t n, std::uint64_t seed, std::uint32_t* out) {
  Rng r(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = static_cast<std::uint32_t>(i);
  for (std::uint64_t i = n; i > 1; --i) std::swap(out[i - 1], out[r.next_below(i)]);
}
void gko_gen_uniform(std::uint64_t n, int d, std::uint64_t seed, double* out) {
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(i));
    for (int j = 0; j < d; ++j) out[i * d + j] = r.next_double();
  }
}
// Gaussian mixture (BASELINE.json config 3): centres c from Rng(seed ^ 0x6d69787475726573).split(c),
// point i from Rng(seed).split(i): centre = next_below(nc), coords N(centre, sigma) clipped to [0,1].
void gko_gen_mixture(std::uint64_t n, int d, std::uint64_t seed, int nc, double sigma, double* out) {
  std::vector<double> C(static_cast<std::size_t>(nc) * d);
  for (int c = 0; c < nc; ++c) {
    Rng r = Rng(seed ^ 0x6d69787475726573ULL).split(static_cast<std::uint64_t>(c));
    for (int j = 0; j < d; ++j) C[c * d + j] = r.next_double();
  }
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(i));
    std::uint64_t c = r.next_below(static_cast<std::uint64_t>(nc));
    for (int j = 0; j < d; ++j) {
      double v = C[c * d + j] + sigma * gaussian(r);
      out[i * d + j] = std::min(1.0, std::max(0.0, v));
    }
  }
}
// Random-walk clusters (BASELINE.json config 5), 2D: cluster c uses Rng(seed).split(c):
// start (u, u); then per step len = 0.001*u, ang = 2*pi*u, p += (len cos ang, len sin ang).
// Point (c, t) = position after t steps, t = 0..steps-1; id = c*steps + t.  No clipping.
void gko_gen_walk(std::uint64_t clusters, std::uint64_t steps, std::uint64_t seed, double* out) {
#pragma omp parallel for schedule(static)
  for (std::int64_t c = 0; c < static_cast<std::int64_t>(clusters); ++c) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(c));
    double x = r.next_double(), y = r.next_double();
    for (std::uint64_t t = 0; t < steps; ++t) {
      std::size_t o = (static_cast<std::size_t>(c) * steps + t) * 2;
      out[o] = x; out[o + 1] = y;
      double len = 0.001 * r.next_double();
      double ang = 2.0 * M_PI * r.next_double();
      x = x + len * std::cos(ang);
      y = y + len * std::sin(ang);
    }
  }
}
// Partial Fisher-Yates (rng.hpp:58-66): the last m entries of the n-step shuffle of 0..n-1
// (identical to random_permutation(n)[n-m..n)); out[0..m) in shuffle order from the end.
void gko_sample_without_replacement(std::uint64_t n, std::uint64_t m, std::uint64_t seed, std::uint32_t* out) {
  std::vector<std::uint32_t> perm(n);
  for (std::uint64_t i = 0; i < n; ++i) perm[i] = static_cast<std::uint32_t>(i);
  Rng r(seed);
  for (std::uint64_t i = n, t = 0; i > 1 && t < m; --i, ++t) std::swap(perm[i - 1], perm[r.next_below(i)]);
  for (std::uint64_t t = 0; t < m; ++t) out[t] = perm[n - 1 - t];
}

// ---- KnnBuf known-answer harness (knn_buffer.hpp:34-46)
int gko_knnbuf_run(int k, const double* d2, const std::uint32_t* ids, std::uint64_t n, double* out_d2,
                   std::uint32_t* out_ids, std::uint64_t* compactions, double* bound) {
  KnnBuf b(static_cast<std::size_t>(k));
  for (std::uint64_t i = 0; i < n; ++i) b.insert(ids[i], d2[i]);
  if (compactions) *compactions = b.compactions;
  if (bound) *bound = b.bound.first;
  auto r = b.extract();
  for (std::size_t i = 0; i < r.size(); ++i) { out_d2[i] = r[i].first; out_ids[i] = r[i].second; }
  return static_cast<int>(r.size());
}

// ---- single static tree (BuildvEB_S)
void* gko_tree_build(int d, const double* pts, const std::uint32_t* ids, std::uint64_t n, int leaf, int heuristic) {
  auto* t = new Tree();
  build_tree(*t, d, pts, ids, n, leaf, heuristic);
  return t;
}
void gko_tree_free(void* h) { delete static_cast<Tree*>(h); }
void gko_tree_info(void* h, std::uint64_t* n_nodes, int* height, int* root, std::uint64_t* live) {
  auto* t = static_cast<Tree*>(h);
  *n_nodes = t->nodes.size(); *height = t->height; *root = t->root; *live = t->live;
}
void gko_tree_export(void* h, void* nodes_out, std::uint32_t* ids_out, double* pts_out) {
  auto* t = static_cast<Tree*>(h);
  if (nodes_out) std::memcpy(nodes_out, t->nodes.data(), t->nodes.size() * sizeof(Node));
  if (ids_out) std::memcpy(ids_out, t->ids.data(), t->n * sizeof(Id));
  if (pts_out) std::memcpy(pts_out, t->pts.data(), t->n * t->d * sizeof(double));
}
void gko_tree_dead(void* h, std::uint8_t* out) {
  auto* t = static_cast<Tree*>(h);
  if (out && t->n) std::memcpy(out, t->dead.data(), t->n);
}
std::uint64_t gko_tree_erase(void* h, const double* P, std::uint64_t n) {
  return erase_static(*static_cast<Tree*>(h), P, n);
}
void gko_tree_knn(void* h, const double* Q, std::uint64_t nq, int k, std::uint32_t* ids, double* d2) {
  auto* t = static_cast<Tree*>(h);
#pragma omp parallel for schedule(dynamic, 256)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
    KnnBuf b(static_cast<std::size_t>(k));
    knn_single(*t, Q + i * t->d, b, nullptr);
    auto r = b.extract();
    for (int j = 0; j < k; ++j) {
      bool ok = j < static_cast<int>(r.size());
      ids[i * k + j] = ok ? r[j].second : kNoPoint;
      d2[i * k + j] = ok ? r[j].first : std::numeric_limits<double>::infinity();
    }
  }
}

// ---- BDL-tree
void* gko_bdl_create(int d, std::uint64_t X, int leaf, int heuristic) {
  auto* b = new Bdl();
  b->d = d; b->X = X; b->leaf = leaf; b->heuristic = heuristic;
  b->statics.resize(64);
  return b;
}
void gko_bdl_free(void* h) { delete static_cast<Bdl*>(h); }
void gko_bdl_insert(void* h, const double* P, std::uint64_t n) {
  auto* b = static_cast<Bdl*>(h);
  std::vector<Id> ids(n);
  for (std::uint64_t i = 0; i < n; ++i) ids[i] = static_cast<Id>(b->next_id + i);
  b->next_id += n;
  insert_l(*b, P, ids.data(), n);
}
std::uint64_t gko_bdl_erase(void* h, const double* P, std::uint64_t n) {
  return erase_l(*static_cast<Bdl*>(h), P, n);
}
void gko_bdl_knn(void* h, const double* Q, std::uint64_t nq, int k, std::uint32_t* ids, double* d2,
                 std::uint64_t* stats3) {
  KnnStats st;
  knn_l(*static_cast<Bdl*>(h), Q, nq, k, ids, d2, stats3 ? &st : nullptr);
  if (stats3) { stats3[0] = st.nodes; stats3[1] = st.leaves; stats3[2] = st.dists; }
}
// F, buffer count, then per tree i (0..63): build_size, live
void gko_bdl_stats(void* h, std::uint64_t* F, std::uint64_t* buffer, std::uint64_t* build64, std::uint64_t* live64) {
  auto* b = static_cast<Bdl*>(h);
  *F = b->F;
  *buffer = b->buf_ids.size();
  for (int i = 0; i < 64; ++i) {
    bool on = b->F >> i & 1ULL;
    build64[i] = on ? b->statics[i].build_size : 0;
    live64[i] = on ? b->statics[i].live : 0;
  }
}
// tree i (0..63) or the buffer tree (i = -1)
void* gko_bdl_tree(void* h, int i) {
  auto* b = static_cast<Bdl*>(h);
  return i < 0 ? static_cast<void*>(&b->buf_tree) : static_cast<void*>(&b->statics[i]);
}
// all live (id, coords) in the structure, ascending id
std::uint64_t gko_bdl_live(void* h, std::uint32_t* ids, double* pts) {
  auto* b = static_cast<Bdl*>(h);
  std::vector<std::pair<Id, std::size_t>> idx;  // (id, global offset)
  std::vector<const double*> src;
  for (int i = 0; i < 64; ++i)
    if (b->F >> i & 1ULL) {
      const Tree& T = b->statics[i];
      for (std::size_t p = 0; p < T.n; ++p)
        if (!T.dead[p]) { idx.push_back({T.ids[p], src.size()}); src.push_back(&T.pts[p * T.d]); }
    }
  for (std::size_t p = 0; p < b->buf_ids.size(); ++p) {
    idx.push_back({b->buf_ids[p], src.size()});
    src.push_back(&b->buf_pts[p * b->d]);
  }
  std::sort(idx.begin(), idx.end());
  if (ids)
    for (std::size_t i = 0; i < idx.size(); ++i) {
      ids[i] = idx[i].first;
      if (pts) std::memcpy(pts + i * b->d, src[idx[i].second], sizeof(double) * b->d);
    }
  return idx.size();
}

// range search: counts (always) and, when ids/d2 are given, the rows (concatenated, sorted by (d2, id))
std::uint64_t gko_bdl_range(void* h, const double* Q, std::uint64_t nq, double r2, std::uint64_t* counts,
                            std::uint32_t* ids, double* d2) {
  std::vector<std::vector<std::pair<double, Id>>> res;
  range_l(*static_cast<Bdl*>(h), Q, nq, r2, res);
  std::uint64_t o = 0;
  for (std::size_t i = 0; i < nq; ++i) {
    if (counts) counts[i] = res[i].size();
    for (const auto& e : res[i]) {
      if (ids) ids[o] = e.second;
      if (d2) d2[o] = e.first;
      ++o;
    }
  }
  return o;
}

// orthogonal range search: counts (always) and, when ids is given, the rows (ascending ids)
std::uint64_t gko_bdl_range_box(void* h, const double* LO, const double* HI, std::uint64_t nq, std::uint64_t* counts,
                                std::uint32_t* ids) {
  const Bdl& b = *static_cast<Bdl*>(h);
  std::vector<const Tree*> trees;
  for (int i = 63; i >= 0; --i)
    if ((b.F >> i & 1ULL) && b.statics[i].live > 0) trees.push_back(&b.statics[i]);
  if (b.buf_tree.live > 0) trees.push_back(&b.buf_tree);
  std::vector<std::vector<Id>> res(nq);
#pragma omp parallel for schedule(dynamic, 256)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
    for (const Tree* T : trees)
      if (T->root >= 0 && T->live > 0) range_box_rec(*T, T->root, LO + i * b.d, HI + i * b.d, res[i]);
    std::sort(res[i].begin(), res[i].end());
  }
  std::uint64_t o = 0;
  for (std::size_t i = 0; i < nq; ++i) {
    if (counts) counts[i] = res[i].size();
    for (Id id : res[i]) {
      if (ids) ids[o] = id;
      ++o;
    }
  }
  return o;
}

// k-NN graph: every live point (ascending id) as a query, kNN_L with k + 1,
// the point itself dropped (the first entry carrying its id, else the (k+1)-th)
std::uint64_t gko_bdl_knn_graph(void* h, int k, std::uint32_t* row_ids, std::uint32_t* ids, double* d2) {
  auto* b = static_cast<Bdl*>(h);
  const std::uint64_t n = gko_bdl_live(h, nullptr, nullptr);
  std::vector<Id> rid(n);
  std::vector<double> pts(n * b->d);
  gko_bdl_live(h, rid.data(), pts.data());
  std::vector<Id> ti(n * (k + 1));
  std::vector<double> td(n * (k + 1));
  knn_l(*b, pts.data(), n, k + 1, ti.data(), td.data(), nullptr);
  for (std::uint64_t r = 0; r < n; ++r) {
    row_ids[r] = rid[r];
    int o = 0;
    bool dropped = false;
    for (int j = 0; j <= k && o < k; ++j) {
      const Id id = ti[r * (k + 1) + j];
      if (!dropped && id == rid[r]) { dropped = true; continue; }
      ids[r * k + o] = id;
      d2[r * k + o] = td[r * (k + 1) + j];
      ++o;
    }
  }
  return n;
}

// ---- brute-force linear-scan oracle: exact (d2, id) top-k
void gko_brute_knn(int d, const double* P, const std::uint32_t* ids, std::uint64_t n, const double* Q,
                   std::uint64_t nq, int k, std::uint32_t* out_ids, double* out_d2) {
#pragma omp parallel for schedule(dynamic, 16)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(nq); ++i) {
    KnnBuf b(static_cast<std::size_t>(k));
    for (std::uint64_t p = 0; p < n; ++p) b.insert(ids[p], sqdist(Q + i * d, P + p * d, d));
    auto r = b.extract();
    for (int j = 0; j < k; ++j) {
      bool ok = j < static_cast<int>(r.size());
      out_ids[i * k + j] = ok ? r[j].second : kNoPoint;
      out_d2[i * k + j] = ok ? r[j].first : std::numeric_limits<double>::infinity();
    }
  }
}

}  // extern "C"
