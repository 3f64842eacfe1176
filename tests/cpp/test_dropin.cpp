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
  // test_serial.cpp:11-19: OpCounters land on n*n; the counters overload
  {
    OpCounters c, cr;
    std::vector<VertexId> vo, vr;
    EXPECT(cuda::dijkstra(four, 0, c, &vo) == dijkstra_serial(four, 0, cr, &vr));
    EXPECT(c.extract_min_scans == 16 && c.relax_checks == 16);
    EXPECT(c.extract_min_scans == cr.extract_min_scans && c.relax_checks == cr.relax_checks);
    EXPECT(vo == vr);
    // test_serial.cpp:21-26: directed, source 3 reaches nothing -- the visit
    // order still lists all n rounds (unreachable ones lowest id first)
    const Graph dg4 = graph_from_edges(el, true);
    EXPECT(cuda::dijkstra(dg4, 3, c, &vo) == dijkstra_serial(dg4, 3, cr, &vr));
    EXPECT(vo == vr && vo.size() == 4);
  }
  // partitioned.hpp:184-225: the reference's PartitionedRun, any p (also p > 8)
  {
    const Graph g = graph_from_edges(generate_sparse(61, 7), false);
    for (std::size_t p : {1, 2, 3, 8, 12}) {
      const PartitionedRun want = dijkstra_partitioned(g, 5, p);
      const PartitionedRun got = cuda::dijkstra_partitioned(g, 5, p, WorkerMode::sequential);
      EXPECT(got.result == want.result);
      EXPECT(got.stats.allreduce_count == want.stats.allreduce_count);
      EXPECT(got.stats.scatter_bytes == want.stats.scatter_bytes);
      EXPECT(got.stats.gather_bytes == want.stats.gather_bytes);
      EXPECT(got.phases.rounds_s > 0);
    }
    bool t3 = false;
    try {
      cuda::dijkstra_partitioned(g, 0, std::size_t{0});
    } catch (const std::invalid_argument&) {
      t3 = true;
    }
    EXPECT(t3);
  }
  // the reference's full value domain (weight.hpp:18, graph.hpp:79): a weight of
  // kMaxWeight = 2^32-1, and n * max_weight >= 2^32 -- 64-bit distances
  {
    EdgeList w;
    w.n = 6;
    w.edges = {{0, 1, kMaxWeight}, {1, 2, kMaxWeight}, {0, 2, 7}, {2, 3, kMaxWeight - 1},
               {3, 4, 1}, {1, 4, 0}};
    for (bool directed : {false, true}) {
      const Graph wg = graph_from_edges(w, directed);
      for (VertexId s = 0; s < 6; ++s) {
        EXPECT(cuda::dijkstra(wg, s) == dijkstra_serial(wg, s));
        EXPECT(cuda::dijkstra_partitioned(wg, s, 2).result == dijkstra_serial(wg, s));
      }
      cuda::DeviceGraph edg(w, directed);
      EXPECT(edg.solve(0) == dijkstra_serial(wg, 0));
    }
    std::mt19937_64 wr(4242);
    for (int i = 0; i < 6; ++i) {
      const std::size_t n = 20 + wr() % 300;
      EdgeList big;
      big.n = n;
      for (std::size_t u = 0; u + 1 < n; ++u) big.edges.push_back({u, u + 1, 3000000000ull + wr() % 1000});
      for (int k = 0; k < 3 * (int)n; ++k) {
        const std::size_t a = wr() % n, b = wr() % n;
        if (a != b) big.edges.push_back({a, b, 4000000000ull + wr() % 294967295ull});
      }
      const Graph bg = graph_from_edges(big, i % 2 == 1);
      const VertexId s = wr() % n;
      EXPECT(cuda::dijkstra(bg, s) == dijkstra_serial(bg, s));
    }
  }
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
