// host_graph.cpp -- graph builders of include/sssp_graph_gen.h.
//
// The generators restate generate.hpp:15-83 on top of std::mt19937_64 (whose
// output the standard fixes, generate.hpp:17-20) and write straight into a
// column block of the uint64 adjacency matrix instead of materialising an
// EdgeList (24 B/edge: 12.9 GB at n = 32768).  Draw order is
// the reference's, so the matrices are bit-identical to
// graph_from_edges(generate_*(n, seed), directed); tests/test_graph_gen.py
// checks that against the reference compiled from its own headers.
#include <cstdint>
#include <cstring>
#include <random>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/sssp_cuda.h"
#include "../../include/sssp_graph_gen.h"

namespace {

constexpr uint64_t kInf = ~0ull;

// generate.hpp:21-29
uint64_t uniform_below(std::mt19937_64& rng, uint64_t bound) {
  const uint64_t span = ~0ull;
  const uint64_t limit = span - span % bound;
  uint64_t x;
  do {
    x = rng();
  } while (x >= limit);
  return x % bound;
}

uint64_t random_weight(std::mt19937_64& rng) { return 1 + uniform_below(rng, 100); }

struct Block {
  uint64_t n, cb, cc, ld;
  uint64_t* out;
  // graph.hpp:37-44 restricted to the block
  void init() const {
    for (uint64_t u = 0; u < n; ++u) {
      uint64_t* row = out + u * ld;
      for (uint64_t j = 0; j < cc; ++j) row[j] = (cb + j == u) ? 0 : kInf;
    }
  }
  bool has(uint64_t v) const { return v >= cb && v < cb + cc; }
  // graph.hpp:80-86: keep the minimum, mirror when undirected
  void put(uint64_t u, uint64_t v, uint64_t w, bool directed) const {
    if (has(v)) {
      uint64_t& c = out[u * ld + (v - cb)];
      if (w < c) c = w;
    }
    if (!directed && has(u)) {
      uint64_t& m = out[v * ld + (u - cb)];
      if (w < m) m = w;
    }
  }
};

bool block_ok(uint64_t n, uint64_t cb, uint64_t cc, uint64_t ld, const uint64_t* out) {
  return out && cb <= n && cc <= n - cb && ld >= cc;
}

}  // namespace

extern "C" {

int sssp_gen_dense(uint64_t n, uint64_t seed, int directed, uint64_t col_begin,
                   uint64_t col_count, uint64_t ld, uint64_t* out) {
  if (n < 2 || !block_ok(n, col_begin, col_count, ld, out)) return SSSP_ERR_BAD_ARG;
  const Block b{n, col_begin, col_count, ld, out};
  b.init();
  std::mt19937_64 rng(seed);
  // generate.hpp:44-46: u < v row-major, one weight draw per pair
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = u + 1; v < n; ++v) b.put(u, v, random_weight(rng), directed != 0);
  return SSSP_OK;
}

int sssp_gen_sparse(uint64_t n, uint64_t seed, int directed, uint64_t col_begin,
                    uint64_t col_count, uint64_t ld, uint64_t* out) {
  if (n < 7 || !block_ok(n, col_begin, col_count, ld, out)) return SSSP_ERR_BAD_ARG;
  const Block b{n, col_begin, col_count, ld, out};
  b.init();
  std::mt19937_64 rng(seed);
  // generate.hpp:61-66 Fisher-Yates
  std::vector<uint64_t> order(n);
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  for (uint64_t i = n - 1; i > 0; --i) std::swap(order[i], order[uniform_below(rng, i + 1)]);
  std::unordered_set<uint64_t> seen;
  seen.reserve(6 * n);
  auto canon = [](uint64_t a, uint64_t c) { return a < c ? (a << 32 | c) : (c << 32 | a); };
  uint64_t m = 0;
  // generate.hpp:72-75 connecting chain
  for (uint64_t i = 0; i + 1 < n; ++i, ++m) {
    seen.insert(canon(order[i], order[i + 1]));
    b.put(order[i], order[i + 1], random_weight(rng), directed != 0);
  }
  // generate.hpp:76-81 distinct random extras up to 3n edges
  while (m < 3 * n) {
    const uint64_t u = uniform_below(rng, n);
    const uint64_t v = uniform_below(rng, n);
    if (u == v || !seen.insert(canon(u, v)).second) continue;
    b.put(u, v, random_weight(rng), directed != 0);
    ++m;
  }
  return SSSP_OK;
}

int sssp_gen_bernoulli(uint64_t n, uint64_t p_q53, uint64_t seed, int directed,
                       uint64_t col_begin, uint64_t col_count, uint64_t ld, uint64_t* out) {
  if (n < 1 || !block_ok(n, col_begin, col_count, ld, out)) return SSSP_ERR_BAD_ARG;
  const Block b{n, col_begin, col_count, ld, out};
  b.init();
  std::mt19937_64 rng(seed);
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = directed ? 0 : u + 1; v < n; ++v) {
      if (u == v) continue;
      if ((rng() >> 11) >= p_q53) continue;
      b.put(u, v, random_weight(rng), directed != 0);
    }
  return SSSP_OK;
}

int sssp_graph_from_edges(uint64_t n, const uint64_t* edges, uint64_t m, int directed,
                          uint64_t col_begin, uint64_t col_count, uint64_t ld, uint64_t* out) {
  if (!block_ok(n, col_begin, col_count, ld, out)) return SSSP_ERR_BAD_ARG;
  const Block b{n, col_begin, col_count, ld, out};
  b.init();
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t u = edges[3 * i], v = edges[3 * i + 1], w = edges[3 * i + 2];
    if (u >= n || v >= n || u == v || w > 0xFFFFFFFFull) return SSSP_ERR_BAD_ARG;
    b.put(u, v, w, directed != 0);
  }
  return SSSP_OK;
}

}  // extern "C"
