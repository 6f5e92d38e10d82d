// gk_host.h — host helpers (gk_host.cpp, OpenMP) used by the CUDA translation units.
#pragma once
#include <cstddef>

namespace gk {
void host_copy(void* dst, const void* src, std::size_t n, int threads);
int host_threads();
}  // namespace gk
