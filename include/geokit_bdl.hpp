// geokit_bdl.hpp — the reference-side C++ binding of the B200 BDL-tree C ABI.
//
// Drop-in for the batch interface SPEC.md's `bdltree` module specifies
// (bdl_build / bdl_insert / bdl_erase / bdl_knn) in the
// conventions of the shipped headers: namespace geokit::<module>, template<int D>,
// PointSet<D> inputs (geokit/core/point.hpp:11-16), results returned by value
// as KnnBuffer::Entry pairs (geokit/kdtree/knn_buffer.hpp:22, 42-46), errors as
// std::invalid_argument / std::logic_error (point.hpp:33, seb/orthant.hpp:143).
//
// Header-only and dependency-free apart from include/gk_bdl.h; it accepts any
// contiguous range of D-double points, so it works with the reference's
// std::vector<Eigen::Matrix<double,D,1>> (whose storage is D packed doubles per
// point) and with plain std::vector<std::array<double,D>>.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gk_bdl.h"

namespace geokit::bdltree {

using PointId = std::uint32_t;                               // geokit/core/point.hpp:18
inline constexpr PointId kNoPoint = GK_NO_POINT;              // geokit/core/point.hpp:19
using Entry = std::pair<double, PointId>;                     // (squared distance, id), knn_buffer.hpp:22

namespace detail {
inline void check(int rc) {
  if (rc == GK_OK) return;
  const std::string msg = gk_last_error();
  if (rc == GK_ERR_INVALID || rc == GK_ERR_CAPACITY) throw std::invalid_argument(msg);
  if (rc == GK_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
  if (rc == GK_ERR_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}
template <class Range>
const double* data_of(const Range& r) {
  return r.empty() ? nullptr : reinterpret_cast<const double*>(r.data());
}
}  // namespace detail

enum class Heuristic { SpatialMedian = GK_SPATIAL_MEDIAN, ObjectMedian = GK_OBJECT_MEDIAN };

/// BDL-tree of D-dimensional points, device resident on one B200.
template <int D>
class BDLTree {
 public:
  static_assert(D >= 2 && D <= 8, "dispatch_dim covers 2..8");

  explicit BDLTree(std::uint32_t buffer_size = 1024, std::uint32_t leaf_size = 16,
                   Heuristic h = Heuristic::SpatialMedian, int device = 0) {
    detail::check(gk_bdl_create(D, buffer_size, leaf_size, static_cast<int>(h), device, &h_));
  }
  ~BDLTree() { gk_bdl_destroy(h_); }
  BDLTree(const BDLTree&) = delete;
  BDLTree& operator=(const BDLTree&) = delete;
  BDLTree(BDLTree&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  BDLTree& operator=(BDLTree&& o) noexcept {
    if (this != &o) {
      gk_bdl_destroy(h_);
      h_ = o.h_;
      o.h_ = nullptr;
    }
    return *this;
  }

  /// bdl_insert (Insert_L, Alg. 3); on an empty tree this is bdl_build.
  template <class PointSet>
  void insert(const PointSet& P) {
    detail::check(gk_bdl_insert(h_, detail::data_of(P), static_cast<std::uint64_t>(P.size())));
  }

  /// bdl_erase (Erase_L, Alg. 4); returns the number of points removed.
  template <class PointSet>
  std::uint64_t erase(const PointSet& P) {
    std::uint64_t n = 0;
    detail::check(gk_bdl_erase(h_, detail::data_of(P), static_cast<std::uint64_t>(P.size()), &n));
    return n;
  }

  /// bdl_knn (kNN_L): per query the k nearest live points as KnnBuffer::extract()
  /// would return them (sorted by (sqdist, id); fewer than k when fewer are live).
  template <class PointSet>
  std::vector<std::vector<Entry>> knn(const PointSet& S, int k) {
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    const std::uint64_t nq = S.size();
    std::vector<PointId> ids(nq * k);
    std::vector<double> d2(nq * k);
    detail::check(gk_bdl_knn(h_, detail::data_of(S), nq, k, ids.data(), d2.data()));
    std::vector<std::vector<Entry>> out(nq);
    for (std::uint64_t i = 0; i < nq; ++i) {
      out[i].reserve(k);
      for (int j = 0; j < k; ++j)
        if (ids[i * k + j] != kNoPoint) out[i].emplace_back(d2[i * k + j], ids[i * k + j]);
    }
    return out;
  }

  /// Flat variant: row-major nq x k ids / squared distances, padded with (kNoPoint, +inf).
  void knn(const double* queries, std::uint64_t nq, int k, PointId* ids, double* d2) {
    detail::check(gk_bdl_knn(h_, queries, nq, k, ids, d2));
  }

  /// Range search (ball): per query every live point with squared distance <= r2, sorted by
  /// (sqdist, id) (the kd-tree range search of PAPER.md:188-190, 204).
  template <class PointSet>
  std::vector<std::vector<Entry>> range(const PointSet& S, double r2) {
    const std::uint64_t nq = S.size();
    std::vector<std::uint64_t> counts(nq), offs(nq + 1);
    detail::check(gk_bdl_range_count(h_, detail::data_of(S), nq, r2, counts.data()));
    std::uint64_t total = 0;
    for (auto c : counts) total += c;
    std::vector<PointId> ids(total ? total : 1);
    std::vector<double> d2(total ? total : 1);
    detail::check(gk_bdl_range(h_, detail::data_of(S), nq, r2, offs.data(), ids.data(), d2.data(), total));
    std::vector<std::vector<Entry>> out(nq);
    for (std::uint64_t i = 0; i < nq; ++i)
      for (std::uint64_t j = offs[i]; j < offs[i + 1]; ++j) out[i].emplace_back(d2[j], ids[j]);
    return out;
  }

  /// Range search (ball) with one squared radius per query: r2[i] applies to S[i].
  template <class PointSet>
  std::vector<std::vector<Entry>> range(const PointSet& S, const std::vector<double>& r2) {
    const std::uint64_t nq = S.size();
    if (r2.size() != nq) throw std::invalid_argument("range: one squared radius per query expected");
    std::vector<std::uint64_t> counts(nq), offs(nq + 1);
    detail::check(gk_bdl_range_radii_count(h_, detail::data_of(S), nq, r2.data(), counts.data()));
    std::uint64_t total = 0;
    for (auto c : counts) total += c;
    std::vector<PointId> ids(total ? total : 1);
    std::vector<double> d2(total ? total : 1);
    detail::check(gk_bdl_range_radii(h_, detail::data_of(S), nq, r2.data(), offs.data(), ids.data(), d2.data(), total));
    std::vector<std::vector<Entry>> out(nq);
    for (std::uint64_t i = 0; i < nq; ++i)
      for (std::uint64_t j = offs[i]; j < offs[i + 1]; ++j) out[i].emplace_back(d2[j], ids[j]);
    return out;
  }

  /// Orthogonal range search: per query box [lo_i, hi_i] the ids of the live points inside, ascending.
  template <class PointSet>
  std::vector<std::vector<PointId>> range_box(const PointSet& lo, const PointSet& hi) {
    if (lo.size() != hi.size()) throw std::invalid_argument("lo and hi must hold the same number of boxes");
    const std::uint64_t nq = lo.size();
    std::vector<std::uint64_t> counts(nq), offs(nq + 1);
    detail::check(gk_bdl_range_box_count(h_, detail::data_of(lo), detail::data_of(hi), nq, counts.data()));
    std::uint64_t total = 0;
    for (auto c : counts) total += c;
    std::vector<PointId> ids(total ? total : 1);
    detail::check(gk_bdl_range_box(h_, detail::data_of(lo), detail::data_of(hi), nq, offs.data(), ids.data(), total));
    std::vector<std::vector<PointId>> out(nq);
    for (std::uint64_t i = 0; i < nq; ++i) out[i].assign(ids.begin() + offs[i], ids.begin() + offs[i + 1]);
    return out;
  }

  /// k-NN graph: for every live point (ascending id) its k nearest other
  /// live points, sorted by (sqdist, id); returns (point id, neighbours) rows.
  std::vector<std::pair<PointId, std::vector<Entry>>> knn_graph(int k) {
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    const std::uint64_t n = size();
    std::vector<PointId> rows(n), ids(n * k);
    std::vector<double> d2(n * k);
    detail::check(gk_bdl_knn_graph(h_, k, rows.data(), ids.data(), d2.data()));
    std::vector<std::pair<PointId, std::vector<Entry>>> out(n);
    for (std::uint64_t r = 0; r < n; ++r) {
      out[r].first = rows[r];
      for (int j = 0; j < k; ++j)
        if (ids[r * k + j] != kNoPoint) out[r].second.emplace_back(d2[r * k + j], ids[r * k + j]);
    }
    return out;
  }

  gk_bdl_info info() const {
    gk_bdl_info i;
    detail::check(gk_bdl_info_get(h_, &i));
    return i;
  }
  std::uint64_t size() const { return info().live; }
  gk_bdl* handle() const { return h_; }

 private:
  gk_bdl* h_ = nullptr;
};

// ---- SPEC.md's free-function interface of the bdltree module, over the class above.

/// bdl_build(P) -> BDLTree: bdl_insert(P) on an empty structure.
template <int D, class PointSet>
BDLTree<D> bdl_build(const PointSet& P, std::uint32_t buffer_size = 1024, std::uint32_t leaf_size = 16,
                     Heuristic h = Heuristic::SpatialMedian, int device = 0) {
  BDLTree<D> t(buffer_size, leaf_size, h, device);
  t.insert(P);
  return t;
}

/// bdl_insert(tree, P) (Algorithm 3).
template <int D, class PointSet>
void bdl_insert(BDLTree<D>& tree, const PointSet& P) {
  tree.insert(P);
}

/// bdl_erase(tree, P) (Algorithm 4); also returns the number of points removed.
template <int D, class PointSet>
std::uint64_t bdl_erase(BDLTree<D>& tree, const PointSet& P) {
  return tree.erase(P);
}

/// bdl_knn(tree, S, k) -> per-query k nearest, each row as KnnBuffer::extract().
template <int D, class PointSet>
std::vector<std::vector<Entry>> bdl_knn(BDLTree<D>& tree, const PointSet& S, int k) {
  return tree.knn(S, k);
}

}  // namespace geokit::bdltree
