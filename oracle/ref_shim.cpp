// ref_shim.cpp — compiles the REFERENCE's own headers (read in place from
// /root/reference/proj/include, never copied) into oracle/_ref/libgkref.so so
// the oracle's restatements can be pinned against them (TEST INFRASTRUCTURE).
//   * geokit/core/rng.hpp:10-66         (mix64, Rng, random_permutation)
//   * geokit/kdtree/knn_buffer.hpp:20-67 (KnnBuffer)
// knn_buffer.hpp:50 uses an unqualified kNoPoint that is not in scope in
// geokit::kdtree (latent compile error); the using-declaration
// below is the one-line shim that makes the shipped header compile.
#include <string>
#include "geokit/core/point.hpp"
#include "geokit/core/rng.hpp"
namespace geokit::kdtree { using geokit::core::kNoPoint; }
#include "geokit/kdtree/knn_buffer.hpp"

#include <cstdint>

extern "C" {

std::uint64_t gkref_mix64(std::uint64_t z) { return geokit::core::mix64(z); }

void gkref_rng_u64(std::uint64_t seed, std::uint64_t stream, int use_split, std::uint64_t n, std::uint64_t* out) {
  geokit::core::Rng r(seed);
  if (use_split) r = r.split(stream);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void gkref_rng_double(std::uint64_t seed, std::uint64_t stream, int use_split, std::uint64_t n, double* out) {
  geokit::core::Rng r(seed);
  if (use_split) r = r.split(stream);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_double();
}

void gkref_rng_below(std::uint64_t seed, std::uint64_t bound, std::uint64_t n, std::uint64_t* out) {
  geokit::core::Rng r(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_below(bound);
}

void gkref_random_permutation(std::uint64_t n, std::uint64_t seed, std::uint32_t* out) {
  auto p = geokit::core::random_permutation(n, geokit::core::Rng(seed));
  for (std::uint64_t i = 0; i < n; ++i) out[i] = p[i];
}

int gkref_knnbuf_run(int k, const double* d2, const std::uint32_t* ids, std::uint64_t n, double* out_d2,
                     std::uint32_t* out_ids, std::uint64_t* compactions, double* bound) {
  geokit::kdtree::KnnBuffer b(static_cast<std::size_t>(k));
  for (std::uint64_t i = 0; i < n; ++i) b.insert(ids[i], d2[i]);
  if (compactions) *compactions = b.compactions();
  if (bound) *bound = b.bound();
  auto r = b.extract();
  for (std::size_t i = 0; i < r.size(); ++i) { out_d2[i] = r[i].first; out_ids[i] = r[i].second; }
  return static_cast<int>(r.size());
}

}  // extern "C"
