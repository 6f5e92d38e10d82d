// gk_bdl_cli.cpp — the path's slice of the reference's (absent) CLI harness,
// SPEC.md:635-696 (`cli` module): text point files, the `knn` and `bdl-script`
// tasks and BenchRecord CSV rows, driving the BDL-tree through the C ABI.
//
//   gk_bdl_cli knn <points> <queries> -k K [-o result] [--check] [--leaf L] [-X X]
//   gk_bdl_cli bdl-script <script> [-o result] [--check] [--leaf L] [-X X]
//
// PointFile: optional header line "pargeo <d>", then one point per
// line, d whitespace-separated decimal floats.  Script lines:
// `insert <file>` / `erase <file>` / `knn <file> <k>`, executed in order; file
// names are relative to the script's directory.  Result file: per query one
// line of k ids (kNoPoint as -1).  BenchRecord CSV row per task or
// script op on stdout: algorithm,dataset,n,d,threads,seconds,summary, with
// summary = FNV-1a-64 checksum of the result ids.  --check re-derives a
// sample of kNN rows (every nq/1000-th) by exact linear scan over the live points (this
// tool's own code, not the test oracle) and exits 2 on any mismatch.
// Exit codes: 0 ok, 1 usage, 2 check failure, 3 I/O.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/gk_bdl.h"

namespace {

struct PointFile {
  int d = 0;
  std::vector<double> xs;  // row-major
  std::size_t n() const { return d ? xs.size() / d : 0; }
};

[[noreturn]] void die(int code, const std::string& m) {
  std::fprintf(stderr, "gk_bdl_cli: %s\n", m.c_str());
  std::exit(code);
}

PointFile read_points(const std::string& path, int want_d) {
  std::ifstream f(path);
  if (!f) die(3, "cannot read " + path);
  PointFile pf;
  pf.d = want_d;
  std::string line;
  bool first = true;
  while (std::getline(f, line)) {
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream is(line);
    if (first && line.rfind("pargeo", 0) == 0) {
      std::string tag;
      int d = 0;
      is >> tag >> d;
      if (d < 2 || d > 8) die(3, path + ": bad header");
      if (pf.d && pf.d != d) die(3, path + ": dimension " + std::to_string(d) + " != " + std::to_string(pf.d));
      pf.d = d;
      first = false;
      continue;
    }
    first = false;
    std::vector<double> row;
    double v;
    while (is >> v) row.push_back(v);
    if (!is.eof()) die(3, path + ": unparsable row: " + line);
    if (!pf.d) pf.d = static_cast<int>(row.size());
    if (static_cast<int>(row.size()) != pf.d) die(3, path + ": row with " + std::to_string(row.size()) + " fields");
    for (double x : row)
      if (!std::isfinite(x)) die(3, path + ": non-finite coordinate");
    pf.xs.insert(pf.xs.end(), row.begin(), row.end());
  }
  if (pf.d < 2 || pf.d > 8) die(3, path + ": dimension must be 2..8");
  return pf;
}

std::string dir_of(const std::string& p) {
  const auto s = p.find_last_of('/');
  return s == std::string::npos ? std::string() : p.substr(0, s + 1);
}
std::string base_of(const std::string& p) {
  const auto s = p.find_last_of('/');
  return s == std::string::npos ? p : p.substr(s + 1);
}

std::uint64_t fnv1a(const std::vector<std::uint32_t>& v) {
  std::uint64_t h = 1469598103934665603ULL;
  for (std::uint32_t x : v)
    for (int b = 0; b < 4; ++b) {
      h ^= (x >> (8 * b)) & 0xffu;
      h *= 1099511628211ULL;
    }
  return h;
}

void check(int rc) {
  if (rc != GK_OK) die(rc == GK_ERR_INVALID ? 1 : 3, gk_last_error());
}

// live point multiset mirror (id, coords) for --check; ids follow the ABI rule
// (global insertion ordinals), erase removes every coordinate-equal point
struct Mirror {
  int d = 0;
  std::uint32_t next = 0;
  std::vector<std::uint32_t> ids;
  std::vector<double> xs;
  void insert(const PointFile& p) {
    for (std::size_t i = 0; i < p.n(); ++i) ids.push_back(next++);
    xs.insert(xs.end(), p.xs.begin(), p.xs.end());
  }
  void erase(const PointFile& p) {
    std::vector<std::uint32_t> ni;
    std::vector<double> nx;
    for (std::size_t i = 0; i < ids.size(); ++i) {
      bool hit = false;
      for (std::size_t e = 0; e < p.n() && !hit; ++e) {
        bool eq = true;
        for (int j = 0; j < d; ++j) eq = eq && xs[i * d + j] == p.xs[e * d + j];
        hit = eq;
      }
      if (hit) continue;
      ni.push_back(ids[i]);
      nx.insert(nx.end(), xs.begin() + i * d, xs.begin() + (i + 1) * d);
    }
    ids.swap(ni);
    xs.swap(nx);
  }
  // exact (d2, id) top-k of query q by linear scan; d2 in the ABI's canonical order
  void knn(const double* q, int k, std::vector<std::uint32_t>& oi, std::vector<double>& od) const {
    std::vector<std::pair<double, std::uint32_t>> all;
    all.reserve(ids.size());
    for (std::size_t i = 0; i < ids.size(); ++i) {
      double s = 0.0;  // left to right, no FMA (built with -ffp-contract=off)
      for (int j = 0; j < d; ++j) {
        const double t = q[j] - xs[i * d + j];
        s = s + t * t;
      }
      all.push_back({s, ids[i]});
    }
    const std::size_t m = std::min<std::size_t>(k, all.size());
    std::partial_sort(all.begin(), all.begin() + m, all.end());
    oi.assign(k, GK_NO_POINT);
    od.assign(k, std::numeric_limits<double>::infinity());
    for (std::size_t j = 0; j < m; ++j) {
      oi[j] = all[j].second;
      od[j] = all[j].first;
    }
  }
};

struct Opts {
  std::string out;
  bool check = false;
  int k = 0;
  std::uint32_t X = 1024, leaf = 16;
  std::vector<std::string> pos;
};

Opts parse(int argc, char** argv) {
  Opts o;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) die(1, "missing value for " + a);
      return argv[++i];
    };
    if (a == "-o") o.out = next();
    else if (a == "-k") o.k = std::atoi(next().c_str());
    else if (a == "-X") o.X = static_cast<std::uint32_t>(std::atoi(next().c_str()));
    else if (a == "--leaf") o.leaf = static_cast<std::uint32_t>(std::atoi(next().c_str()));
    else if (a == "--check") o.check = true;
    else if (!a.empty() && a[0] == '-') die(1, "unknown flag " + a);
    else o.pos.push_back(a);
  }
  return o;
}

struct Runner {
  Opts o;
  gk_bdl* h = nullptr;
  int d = 0;
  Mirror mirror;
  std::ofstream result;
  bool failed = false;

  explicit Runner(const Opts& opts) : o(opts) {
    if (!o.out.empty()) {
      result.open(o.out);
      if (!result) die(3, "cannot write " + o.out);
    }
  }
  ~Runner() { gk_bdl_destroy(h); }

  void ensure(int dim) {
    if (h) {
      if (dim != d) die(3, "dimension changes inside one run");
      return;
    }
    d = dim;
    mirror.d = dim;
    check(gk_bdl_create(dim, o.X, o.leaf, GK_SPATIAL_MEDIAN, 0, &h));
  }

  void record(const char* algo, const std::string& tag, std::size_t n, double secs, const std::string& summary) {
    std::printf("%s,%s,%zu,%d,1,%.6f,%s\n", algo, tag.c_str(), n, d, secs, summary.c_str());
  }

  void insert(const std::string& path) {
    PointFile p = read_points(path, d);
    ensure(p.d);
    const auto t0 = std::chrono::steady_clock::now();
    check(gk_bdl_insert(h, p.xs.data(), p.n()));
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (o.check) mirror.insert(p);
    gk_bdl_info info;
    check(gk_bdl_info_get(h, &info));
    record("bdl-insert", base_of(path), p.n(), s, "live=" + std::to_string(info.live));
  }

  void erase(const std::string& path) {
    PointFile p = read_points(path, d);
    ensure(p.d);
    std::uint64_t killed = 0;
    const auto t0 = std::chrono::steady_clock::now();
    check(gk_bdl_erase(h, p.xs.data(), p.n(), &killed));
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (o.check) mirror.erase(p);
    record("bdl-erase", base_of(path), p.n(), s, "erased=" + std::to_string(killed));
  }

  void knn(const std::string& path, int k) {
    if (k < 1 || k > GK_MAX_K) die(1, "k must be in [1, " + std::to_string(GK_MAX_K) + "]");
    PointFile q = read_points(path, d);
    ensure(q.d);
    const std::size_t nq = q.n();
    std::vector<std::uint32_t> ids(nq * k);
    std::vector<double> d2(nq * k);
    const auto t0 = std::chrono::steady_clock::now();
    check(gk_bdl_knn(h, q.xs.data(), nq, k, ids.data(), d2.data()));
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    char sum[32];
    std::snprintf(sum, sizeof(sum), "%016llx", static_cast<unsigned long long>(fnv1a(ids)));
    record("bdl-knn", base_of(path), nq, s, sum);
    if (result.is_open())
      for (std::size_t i = 0; i < nq; ++i) {
        for (int j = 0; j < k; ++j) {
          const std::uint32_t v = ids[i * k + j];
          result << (j ? " " : "") << (v == GK_NO_POINT ? -1LL : static_cast<long long>(v));
        }
        result << "\n";
      }
    if (o.check) {
      std::vector<std::uint32_t> oi;
      std::vector<double> od;
      const std::size_t stride = std::max<std::size_t>(1, nq / 1000);  // <= ~1000 sampled rows
      for (std::size_t i = 0; i < nq; i += stride) {
        mirror.knn(&q.xs[i * d], k, oi, od);
        for (int j = 0; j < k; ++j)
          if (oi[j] != ids[i * k + j] || !(od[j] == d2[i * k + j] || (std::isinf(od[j]) && std::isinf(d2[i * k + j])))) {
            std::fprintf(stderr, "gk_bdl_cli: --check mismatch at query %zu slot %d\n", i, j);
            failed = true;
            return;
          }
      }
    }
  }
};

void usage() {
  std::fprintf(stderr,
               "usage: gk_bdl_cli knn <points> <queries> -k K [-o result] [--check] [-X X] [--leaf L]\n"
               "       gk_bdl_cli bdl-script <script> [-o result] [--check] [-X X] [--leaf L]\n");
  std::exit(1);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage();
  const std::string task = argv[1];
  Opts o = parse(argc, argv);
  std::printf("algorithm,dataset,n,d,threads,seconds,summary\n");
  Runner r(o);
  if (task == "knn") {
    if (o.pos.size() != 2 || o.k < 1) usage();
    r.insert(o.pos[0]);
    r.knn(o.pos[1], o.k);
  } else if (task == "bdl-script") {
    if (o.pos.size() != 1) usage();
    std::ifstream f(o.pos[0]);
    if (!f) die(3, "cannot read " + o.pos[0]);
    const std::string dir = dir_of(o.pos[0]);
    std::string line;
    int lineno = 0;
    while (std::getline(f, line)) {
      ++lineno;
      std::istringstream is(line);
      std::string op, file;
      if (!(is >> op) || op[0] == '#') continue;
      if (!(is >> file)) die(1, "script line " + std::to_string(lineno) + ": missing file");
      const std::string path = (file[0] == '/') ? file : dir + file;
      if (op == "insert") r.insert(path);
      else if (op == "erase") r.erase(path);
      else if (op == "knn") {
        int k = 0;
        if (!(is >> k)) die(1, "script line " + std::to_string(lineno) + ": knn needs k");
        r.knn(path, k);
      } else die(1, "script line " + std::to_string(lineno) + ": unknown op " + op);
      if (r.failed) break;
    }
  } else {
    usage();
  }
  std::fflush(stdout);
  return r.failed ? 2 : 0;
}
