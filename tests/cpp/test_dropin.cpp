// test_dropin.cpp -- the C++ drop-in (include/sssp/cuda.hpp) against the
// reference's own dijkstra_serial / dijkstra_partitioned /
// dijkstra_dataparallel, compiled from the
// unmodified reference headers (oracle/Makefile -> oracle/_ref/test_dropin).
// Exit code 0 = every ShortestPathResult compares equal (result.hpp:18).
#include <cstdio>
#include <random>
#include <sstream>

#include "sssp/cuda.hpp"
#include "sssp/sssp.hpp"

using namespace sssp;

static int failures = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                   \
    }                                                               \
  } while (0)

int main() {
  // test_serial.cpp:11-19 / 69-75
  EdgeList el;
  el.n = 4;
  el.edges = {{0, 1, 2}, {0, 2, 4}, {1, 2, 1}, {1, 3, 3}, {2, 3, 5}};
  const Graph four = graph_from_edges(el, false);
  std::vector<VertexId> order;
  const ShortestPathResult r = cuda::dijkstra(four, 0, &order);
  EXPECT(r == dijkstra_serial(four, 0));
  EXPECT((r.dist == std::vector<Weight>{0, 2, 3, 5}));
  EXPECT((r.pred == std::vector<VertexId>{kNoVertex, 0, 1, 1}));
  EXPECT((order == std::vector<VertexId>{0, 1, 2, 3}));
  // test_serial.cpp:35-38
  bool threw = false;
  try {
    cuda::dijkstra(four, 4);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  // acceptance.cpp:42-80 style sweep, full-result equality
  std::mt19937_64 rng(20240601);
  int graphs = 0;
  for (bool dense : {false, true})
    for (bool directed : {false, true})
      for (int i = 0; i < 25; ++i) {
        const std::size_t n = 7 + rng() % 194;
        const EdgeList e = dense ? generate_dense(n, rng()) : generate_sparse(n, rng());
        const Graph g = graph_from_edges(e, directed);
        const VertexId s = rng() % n;
        const ShortestPathResult want = dijkstra_serial(g, s);
        EXPECT(cuda::dijkstra(g, s) == want);
        EXPECT(cuda::dijkstra_partitioned(g, s, {0, 0, 0}) == want);
        EXPECT(dijkstra_partitioned(g, s, 3).result == want);
        // the paper's data-parallel engine: result AND round count
        const DataParallelRun dp = dijkstra_dataparallel(g, s);
        const cuda::DataParallelRun cdp = cuda::dijkstra_dataparallel(g, s);
        EXPECT(cdp.result == dp.result);
        EXPECT(cdp.rounds == dp.rounds);
        EXPECT(cdp.cells_in == dp.cells_in && cdp.cells_out == dp.cells_out);
        ++graphs;
      }
  // test_dataparallel.cpp:144-154: zero-weight ties, reconstructed pred
  {
    EdgeList z;
    z.n = 4;
    z.edges = {{2, 0, 5}, {2, 1, 5}, {0, 1, 0}, {1, 3, 2}};
    const Graph zg = graph_from_edges(z, false);
    const cuda::DataParallelRun c = cuda::dijkstra_dataparallel(zg, 2);
    EXPECT(c.result == dijkstra_dataparallel(zg, 2).result);
    EXPECT((c.result.dist == std::vector<Weight>{5, 5, 0, 7}));
    EXPECT(validate_result(zg, c.result).empty());
    bool t2 = false;
    try {
      cuda::dijkstra_dataparallel(zg, 4);
    } catch (const std::invalid_argument&) {
      t2 = true;
    }
    EXPECT(t2);
  }
  // the multi-threaded parser: same EdgeList, same ParseError as graph.hpp:126-170
  {
    const char* texts[] = {"# c\n4 2\r\n0 1 5\r\n\n2 3 7 \n", "3 1\n0 1 1\n1 2 1\n", "3 2\n0 1 1\n",
                           "3 1\n1 1 4\n", "3 1\n0 x 4\n", "5 6\n0 1 4\n1 2 1\n0 2 9\n2 3 2\n3 4 1\n0 1 3\n"};
    for (const char* t : texts) {
      std::istringstream in(t);
      std::string want_err, got_err;
      EdgeList want, got;
      try { want = parse_edge_list_text(in); } catch (const ParseError& e) { want_err = e.what(); }
      try { got = cuda::parse_edge_list_text(t); } catch (const ParseError& e) { got_err = e.what(); }
      EXPECT(want_err == got_err);
      EXPECT(want.n == got.n && want.edges.size() == got.edges.size());
      for (std::size_t i = 0; i < want.edges.size() && i < got.edges.size(); ++i)
        EXPECT(want.edges[i].u == got.edges[i].u && want.edges[i].v == got.edges[i].v &&
               want.edges[i].w == got.edges[i].w);
    }
  }
  // device-side build from the reference's own parsed EdgeList (-w off and on)
  {
    std::istringstream in("5 6\n0 1 4\n1 2 1\n0 2 9\n2 3 2\n3 4 1\n0 1 3\n");
    const EdgeList pel = parse_edge_list_text(in);
    for (bool directed : {false, true}) {
      cuda::DeviceGraph eg(pel, directed);
      const Graph hg = graph_from_edges(pel, directed);
      for (VertexId s = 0; s < 5; ++s) EXPECT(eg.solve(s) == dijkstra_serial(hg, s));
    }
  }
  // repeated solves + batch on one resident graph
  const Graph big = graph_from_edges(generate_dense(3000, 99), false);
  cuda::DeviceGraph dg(big);
  const std::vector<VertexId> srcs = {0, 17, 2999, 1500};
  const auto batch = dg.solve_batch(srcs);
  for (std::size_t i = 0; i < srcs.size(); ++i) {
    const ShortestPathResult want = dijkstra_serial(big, srcs[i]);
    EXPECT(batch[i] == want);
    EXPECT(dg.solve(srcs[i]) == want);
  }
  const cuda::CudaRun run = cuda::dijkstra_run(big, 5);
  EXPECT(run.iterations == 3000);
  EXPECT(run.phases.rounds_s > 0);
  std::printf("%s: %d graphs, %d failures\n", failures ? "FAIL" : "PASS", graphs, failures);
  return failures ? 1 : 0;
}
