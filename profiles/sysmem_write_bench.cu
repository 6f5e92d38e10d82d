// Micro-benchmark (experiment, not product): how fast can a kernel write kNN result rows
// (k = 10: 40 B of ids + 80 B of d^2 per query) straight into mapped pinned host memory,
// for row-contiguous and for permuted (Hilbert-order) row positions?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/swb profiles/sysmem_write_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e_)); std::exit(1); } } while (0)

constexpr int K = 10;

// pattern 1: flat coalesced 16 B stores
__global__ void k_flat(uint4* out, std::uint64_t n16) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n16; i += (std::uint64_t)gridDim.x * blockDim.x)
    out[i] = make_uint4((unsigned)i, 1, 2, 3);
}

// pattern 2: thread per row, row = perm[i], per-lane scalar stores (what K1's epilogue does)
__global__ void k_row_thread(const std::uint32_t* perm, std::uint64_t nq, std::uint32_t* ids, double* d2) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < nq; i += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t r = perm[i];
#pragma unroll
    for (int j = 0; j < K; ++j) ids[r * K + j] = (std::uint32_t)(i + j);
#pragma unroll
    for (int j = 0; j < K; ++j) d2[r * K + j] = (double)(i + j);
  }
}

// pattern 3: warp-cooperative -- one row per (group of K lanes), 3 rows per store instruction
__global__ void k_row_warp(const std::uint32_t* perm, std::uint64_t nq, std::uint32_t* ids, double* d2) {
  const int lane = threadIdx.x & 31;
  const int g = lane / K, j = lane % K;
  const std::uint64_t warp = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) >> 5;
  const std::uint64_t nwarps = ((std::uint64_t)gridDim.x * blockDim.x) >> 5;
  for (std::uint64_t base = warp * 3; base < nq; base += nwarps * 3) {
    const std::uint64_t i = base + g;
    if (g < 3 && i < nq) {
      const std::uint64_t r = perm[i];
      ids[r * K + j] = (std::uint32_t)(i + j);
      d2[r * K + j] = (double)(i + j);
    }
  }
}

int main(int argc, char** argv) {
  const std::uint64_t nq = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 10000000ULL;
  const std::uint64_t bytes = nq * K * 12;
  std::uint32_t *h_ids, *d_ids;
  double *h_d2, *d_d2;
  CK(cudaHostAlloc(&h_ids, nq * K * 4, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_d2, nq * K * 8, cudaHostAllocMapped));
  CK(cudaMalloc(&d_ids, nq * K * 4));
  CK(cudaMalloc(&d_d2, nq * K * 8));
  std::uint32_t *m_ids, *m_d2raw;
  CK(cudaHostGetDevicePointer((void**)&m_ids, h_ids, 0));
  CK(cudaHostGetDevicePointer((void**)&m_d2raw, h_d2, 0));
  double* m_d2 = (double*)m_d2raw;
  // permutations: identity, random, and "blocked random" (random within windows of 32 rows... no:
  // Hilbert order of random queries is a random permutation of rows)
  std::vector<std::uint32_t> perm(nq);
  for (std::uint64_t i = 0; i < nq; ++i) perm[i] = (std::uint32_t)i;
  std::uint32_t *p_id, *p_rnd;
  CK(cudaMalloc(&p_id, nq * 4));
  CK(cudaMalloc(&p_rnd, nq * 4));
  CK(cudaMemcpy(p_id, perm.data(), nq * 4, cudaMemcpyHostToDevice));
  std::mt19937_64 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  CK(cudaMemcpy(p_rnd, perm.data(), nq * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto run = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    std::printf("%-44s %8.2f ms  %7.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  const int G = 148 * 8, T = 256;
  run("host: flat 16B coalesced", [&] { k_flat<<<G, T>>>((uint4*)m_ids, nq * K * 4 / 16); k_flat<<<G, T>>>((uint4*)m_d2, nq * K * 8 / 16); });
  run("host: thread-per-row, identity rows", [&] { k_row_thread<<<G, T>>>(p_id, nq, m_ids, m_d2); });
  run("host: thread-per-row, random rows", [&] { k_row_thread<<<G, T>>>(p_rnd, nq, m_ids, m_d2); });
  run("host: warp-coop rows, identity", [&] { k_row_warp<<<G, T>>>(p_id, nq, m_ids, m_d2); });
  run("host: warp-coop rows, random", [&] { k_row_warp<<<G, T>>>(p_rnd, nq, m_ids, m_d2); });
  run("dev:  thread-per-row, random rows", [&] { k_row_thread<<<G, T>>>(p_rnd, nq, d_ids, d_d2); });
  run("dev:  warp-coop rows, random", [&] { k_row_warp<<<G, T>>>(p_rnd, nq, d_ids, d_d2); });
  // check content of one random row
  std::uint64_t i = nq / 3;
  std::printf("check row %u: id0=%u d0=%g (expect %llu)\n", perm[i], h_ids[(std::uint64_t)perm[i] * K], h_d2[(std::uint64_t)perm[i] * K],
              (unsigned long long)i);
  return 0;
}
