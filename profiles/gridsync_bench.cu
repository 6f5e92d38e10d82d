// Micro-benchmark (experiment): cost of one cooperative-groups grid barrier vs grid shape,
// and of a hand-rolled barrier (one atomic per block + spin on a generation word).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/_gsb profiles/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) { x += threadIdx.x; g.sync(); }
  if (x == 12345) *sink = x;
}

__device__ __forceinline__ void my_sync(unsigned* count, volatile unsigned* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) {}
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_my(int iters, unsigned* count, unsigned* gen, unsigned* sink) {
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) { x += threadIdx.x; my_sync(count, gen, gridDim.x); }
  if (x == 12345) *sink = x;
}

int main() {
  unsigned *sink, *cnt, *gen;
  cudaMalloc(&sink, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int shapes[][2] = {{148, 256}, {296, 256}, {444, 256}, {592, 256}, {148, 512}, {148, 1024}, {296, 512}, {74, 256}, {1, 256}};
  for (auto& sh : shapes) {
    int iters = 2000;
    for (int which = 0; which < 2; ++which) {
      void* args_cg[] = {&iters, &sink};
      void* args_my[] = {&iters, &cnt, &gen, &sink};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaError_t e = which == 0 ? cudaLaunchCooperativeKernel((void*)k_cg, sh[0], sh[1], args_cg, 0, 0)
                                   : cudaLaunchCooperativeKernel((void*)k_my, sh[0], sh[1], args_my, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("%-3s grid %4d x %4d: %.2f us per barrier (%s)\n", which ? "own" : "cg", sh[0], sh[1], ms * 1e3 / iters, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
