// gk_host.cpp — host-side helpers of the C ABI that want OpenMP (compiled by g++ -fopenmp;
// the CUDA translation units call them through gk_host.h).
#include "gk_host.h"

#include <omp.h>

#include <algorithm>
#include <cstring>

namespace gk {

// memcpy split over up to `threads` OpenMP threads in >= 1 MiB pieces: the pageable-host
// side of the staged kNN_L pipeline (one thread moves ~10 GB/s, the copy of a 1.2 GB result
// must keep up with PCIe).
void host_copy(void* dst, const void* src, std::size_t n, int threads) {
  constexpr std::size_t kPiece = 1u << 20;
  const long pieces = static_cast<long>((n + kPiece - 1) / kPiece);
  if (pieces <= 1 || threads <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const int t = std::min<long>(threads, pieces);
#pragma omp parallel for num_threads(t) schedule(static)
  for (long i = 0; i < pieces; ++i) {
    const std::size_t off = static_cast<std::size_t>(i) * kPiece;
    std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(kPiece, n - off));
  }
}

int host_threads() { return omp_get_max_threads(); }

}  // namespace gk
