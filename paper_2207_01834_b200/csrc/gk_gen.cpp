// gk_gen.cpp — seeded input generators of the bench harness (host, OpenMP).
//
// Restates geokit/core/rng.hpp:10-66 (SplitMix64 counter Rng, split streams,
// Fisher-Yates via next_below) and geokit/generators.hpp:44-63 (one split
// stream per point; Box-Muller normals) with the BASELINE.json config recipes
// (DESIGN.md "Inputs").  The oracle carries its own independent restatement;
// tests/test_inputs.py checks the two agree bit for bit and that both match
// the reference's own rng.hpp compiled into oracle/_ref.
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/gk_bdl.h"

namespace {

inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) { return mix64(mix64(a) ^ b); }
inline double unit_double(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : seed_(mix64(seed)) {}
  std::uint64_t next_u64() { return mix64(seed_, ctr_++); }
  double next_double() { return unit_double(next_u64()); }
  std::uint64_t next_below(std::uint64_t n) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
  }
  Rng split(std::uint64_t stream) const { return Rng(mix64(seed_, ~stream)); }

 private:
  std::uint64_t seed_;
  std::uint64_t ctr_ = 0;
};

inline double normal(Rng& r) {
  double u1 = unit_double(r.next_u64());
  double u2 = r.next_double();
  u1 = 1.0 - u1;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

}  // namespace

extern "C" {

int gk_gen_uniform(uint64_t n, int d, uint64_t seed, double* out) {
  if (!out || d < 1) return GK_ERR_INVALID;
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(i));
    for (int j = 0; j < d; ++j) out[i * d + j] = r.next_double();
  }
  return GK_OK;
}

int gk_gen_mixture(uint64_t n, int d, uint64_t seed, int centres, double sigma, double* out) {
  if (!out || d < 1 || centres < 1) return GK_ERR_INVALID;
  std::vector<double> C(static_cast<std::size_t>(centres) * d);
  for (int c = 0; c < centres; ++c) {
    Rng r = Rng(seed ^ 0x6d69787475726573ULL).split(static_cast<std::uint64_t>(c));
    for (int j = 0; j < d; ++j) C[static_cast<std::size_t>(c) * d + j] = r.next_double();
  }
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(i));
    const std::uint64_t c = r.next_below(static_cast<std::uint64_t>(centres));
    for (int j = 0; j < d; ++j) {
      double v = C[c * d + j] + sigma * normal(r);
      out[i * d + j] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
  }
  return GK_OK;
}

int gk_gen_walk(uint64_t clusters, uint64_t steps, uint64_t seed, double* out) {
  if (!out) return GK_ERR_INVALID;
#pragma omp parallel for schedule(static)
  for (std::int64_t c = 0; c < static_cast<std::int64_t>(clusters); ++c) {
    Rng r = Rng(seed).split(static_cast<std::uint64_t>(c));
    double x = r.next_double(), y = r.next_double();
    for (std::uint64_t t = 0; t < steps; ++t) {
      const std::size_t o = (static_cast<std::size_t>(c) * steps + t) * 2;
      out[o] = x;
      out[o + 1] = y;
      const double len = 0.001 * r.next_double();
      const double ang = 2.0 * M_PI * r.next_double();
      x = x + len * std::cos(ang);
      y = y + len * std::sin(ang);
    }
  }
  return GK_OK;
}

int gk_sample_without_replacement(uint64_t n, uint64_t m, uint64_t seed, uint32_t* out) {
  if (!out || m > n) return GK_ERR_INVALID;
  std::vector<std::uint32_t> perm(n);
  for (std::uint64_t i = 0; i < n; ++i) perm[i] = static_cast<std::uint32_t>(i);
  Rng r(seed);
  for (std::uint64_t i = n, t = 0; i > 1 && t < m; --i, ++t) {
    const std::uint64_t j = r.next_below(i);
    const std::uint32_t tmp = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = tmp;
  }
  for (std::uint64_t t = 0; t < m; ++t) out[t] = perm[n - 1 - t];
  return GK_OK;
}

}  // extern "C"
