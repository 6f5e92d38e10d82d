// Minimal C++ client of include/geokit_bdl.hpp (what a reference-side caller,
// e.g. the absent `knn` CLI subcommand of SPEC.md:660-663, would write).
//   g++ -std=c++20 -Iinclude examples/cpp_client.cpp -Lpaper_2207_01834_b200/_lib -lgkbdl
//       -Wl,-rpath,$PWD/paper_2207_01834_b200/_lib -o /tmp/cpp_client && /tmp/cpp_client
#include <array>
#include <cstdio>
#include <vector>

#include "geokit_bdl.hpp"

int main() {
  std::vector<std::array<double, 3>> P(100000);
  if (gk_gen_uniform(P.size(), 3, 2, P[0].data()) != GK_OK) return 1;
  namespace bdl = geokit::bdltree;
  // SPEC.md's free functions: bdl_build / bdl_insert / bdl_erase / bdl_knn (X = 1024, leaf 16, spatial median)
  auto tree = bdl::bdl_build<3>(std::vector<std::array<double, 3>>(P.begin(), P.begin() + 60000));
  bdl::bdl_insert(tree, std::vector<std::array<double, 3>>(P.begin() + 60000, P.end()));
  auto nn = bdl::bdl_knn(tree, std::vector<std::array<double, 3>>(P.begin(), P.begin() + 4), 3);
  for (auto& row : nn) {
    for (auto& [d2, id] : row) std::printf("(%u, %.3g) ", id, d2);
    std::printf("\n");
  }
  auto ball = tree.range(std::vector<std::array<double, 3>>(P.begin(), P.begin() + 2), 1e-4);  // range search
  std::printf("range rows %zu %zu\n", ball[0].size(), ball[1].size());
  auto ball2 = tree.range(std::vector<std::array<double, 3>>(P.begin(), P.begin() + 2),
                          std::vector<double>{1e-4, 4e-4});  // one squared radius per query
  std::printf("per-query range rows %zu %zu\n", ball2[0].size(), ball2[1].size());
  std::vector<std::array<double, 3>> lo{{0.4, 0.4, 0.4}}, hi{{0.45, 0.45, 0.45}};
  std::printf("box rows %zu\n", tree.range_box(lo, hi)[0].size());  // orthogonal range search
  const unsigned long long erased = bdl::bdl_erase(tree, std::vector<std::array<double, 3>>(P.begin(), P.begin() + 10));
  auto graph = tree.knn_graph(2);  // k-NN graph over the live points
  std::printf("graph rows %zu, first row of id %u\n", graph.size(), graph[0].first);
  std::printf("erased %llu, live %llu\n", erased, (unsigned long long)tree.size());
  return 0;
}
