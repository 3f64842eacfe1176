// ref_shim.cpp -- C-ABI shim around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see sssp_oracle.c header).  Built by
// oracle/Makefile into oracle/_ref/libref_sssp.so with
//   -I/root/reference/proj/include
// so the reference's own dijkstra_serial / dijkstra_partitioned /
// generate_* / graph_from_edges / parse_edge_list / timed_run run exactly as
// shipped.  Nothing here re-implements reference logic: every entry point
// copies plain arrays into the reference types, calls the reference, and
// copies the result out.  It is the "reference" CPU arm of bench.py and the
// generator of tests/golden/.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>

#include "sssp/sssp.hpp"

namespace {

enum { RS_OK = 0, RS_BAD_SOURCE = 1, RS_BAD_ARG = 2, RS_ERR = 3 };

sssp::Graph make_graph(const std::uint64_t* adj, std::uint64_t n, int directed) {
  sssp::Graph g;
  g.n = n;
  g.directed = directed != 0;
  g.adj.assign(adj, adj + n * n);
  return g;
}

void copy_out(const sssp::ShortestPathResult& r, std::uint64_t* dist, std::uint64_t* pred) {
  for (std::size_t v = 0; v < r.dist.size(); ++v) {
    dist[v] = r.dist[v];
    pred[v] = static_cast<std::uint64_t>(r.pred[v]);
  }
}

thread_local std::string g_last_error;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// generate.hpp:38-48 + graph.hpp:73-88
int ref_generate_dense(std::uint64_t n, std::uint64_t seed, int directed, std::uint64_t* adj) {
  try {
    const sssp::Graph g = sssp::graph_from_edges(sssp::generate_dense(n, seed), directed != 0);
    std::memcpy(adj, g.adj.data(), n * n * sizeof(std::uint64_t));
    return RS_OK;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_BAD_ARG;
  }
}

// generate.hpp:53-83 -> edges (3n triples)
int ref_generate_sparse_edges(std::uint64_t n, std::uint64_t seed, std::uint64_t* edges) {
  try {
    const sssp::EdgeList el = sssp::generate_sparse(n, seed);
    for (std::size_t i = 0; i < el.edges.size(); ++i) {
      edges[3 * i] = el.edges[i].u;
      edges[3 * i + 1] = el.edges[i].v;
      edges[3 * i + 2] = el.edges[i].w;
    }
    return RS_OK;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_BAD_ARG;
  }
}

// graph.hpp:73-88 (graph_from_edges) over m (u, v, w) triples
int ref_graph_from_edges(std::uint64_t n, const std::uint64_t* edges, std::uint64_t m,
                         int directed, std::uint64_t* adj) {
  try {
    sssp::EdgeList el;
    el.n = n;
    for (std::uint64_t i = 0; i < m; ++i)
      el.edges.push_back({edges[3 * i], edges[3 * i + 1], edges[3 * i + 2]});
    const sssp::Graph g = sssp::graph_from_edges(el, directed != 0);
    std::memcpy(adj, g.adj.data(), n * n * sizeof(std::uint64_t));
    return RS_OK;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_BAD_ARG;
  }
}

// graph.hpp:172-174 (parse_edge_list, the '-w' switch is `directed`).
// On success *n_out is set and adj (capacity adj_cap cells) is filled when
// n*n <= adj_cap; returns RS_ERR with *line_out set on ParseError.
int ref_parse_edge_list(const char* text, int directed, std::uint64_t* n_out,
                        std::uint64_t* adj, std::uint64_t adj_cap, std::uint64_t* line_out) {
  try {
    std::istringstream in(text);
    const sssp::Graph g = sssp::parse_edge_list(in, directed != 0);
    *n_out = g.n;
    if (g.n * g.n <= adj_cap) std::memcpy(adj, g.adj.data(), g.n * g.n * sizeof(std::uint64_t));
    return RS_OK;
  } catch (const sssp::ParseError& e) {
    g_last_error = e.what();
    *line_out = e.line();
    return RS_ERR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    *line_out = 0;
    return RS_BAD_ARG;
  }
}

// serial.hpp:26-63
int ref_dijkstra_serial(const std::uint64_t* adj, std::uint64_t n, std::uint64_t source,
                        std::uint64_t* dist, std::uint64_t* pred, std::uint64_t* visit_order,
                        std::uint64_t* counters) {
  try {
    const sssp::Graph g = make_graph(adj, n, 1);
    sssp::OpCounters c;
    std::vector<sssp::VertexId> order;
    const sssp::ShortestPathResult r =
        sssp::dijkstra_serial(g, source, c, visit_order ? &order : nullptr);
    copy_out(r, dist, pred);
    if (visit_order)
      for (std::size_t i = 0; i < order.size(); ++i) visit_order[i] = order[i];
    if (counters) {
      counters[0] = c.extract_min_scans;
      counters[1] = c.relax_checks;
    }
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_ERR;
  }
}

// partitioned.hpp:184-225; phases (optional) = {scatter_s, rounds_s, gather_s}
int ref_dijkstra_partitioned(const std::uint64_t* adj, std::uint64_t n, std::uint64_t source,
                             std::uint64_t p, int threaded, std::uint64_t* dist,
                             std::uint64_t* pred, double* phases) {
  try {
    const sssp::Graph g = make_graph(adj, n, 1);
    const sssp::PartitionedRun run = sssp::dijkstra_partitioned(
        g, source, p, threaded ? sssp::WorkerMode::threaded : sssp::WorkerMode::sequential);
    copy_out(run.result, dist, pred);
    if (phases) {
      phases[0] = run.phases.scatter_s;
      phases[1] = run.phases.rounds_s;
      phases[2] = run.phases.gather_s;
    }
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_ERR;
  }
}

// dataparallel.hpp:302-327 with the given lane schedule (0 threaded,
// 1 sequential, 2 shuffled with seed 7); *rounds = DataParallelRun::rounds.
int ref_dijkstra_dataparallel(const std::uint64_t* adj, std::uint64_t n, std::uint64_t source,
                              int schedule, std::uint64_t* dist, std::uint64_t* pred,
                              std::uint64_t* rounds) {
  try {
    const sssp::Graph g = make_graph(adj, n, 1);
    sssp::LaneConfig cfg;
    cfg.schedule = schedule == 1   ? sssp::LaneSchedule::sequential
                   : schedule == 2 ? sssp::LaneSchedule::shuffled
                                   : sssp::LaneSchedule::threaded;
    cfg.shuffle_seed = 7;
    const sssp::DataParallelRun run = sssp::dijkstra_dataparallel(g, source, cfg);
    copy_out(run.result, dist, pred);
    if (rounds) *rounds = run.rounds;
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_ERR;
  }
}

// bench.hpp:114-180 (detail::timed_run): min-of-reps, validated.  engine:
// 0 serial, 1 partitioned.  Returns the scoped total seconds in *total_s
// and the result of the best repetition.  The Graph is built once from adj
// (untimed, as the reference harness does).
int ref_timed_run(int engine, const std::uint64_t* adj, std::uint64_t n, int directed,
                  std::uint64_t source, std::uint64_t workers, std::uint64_t reps,
                  std::uint64_t* dist, std::uint64_t* pred, double* total_s) {
  try {
    const sssp::Graph g = make_graph(adj, n, directed);
    const sssp::EngineKind kind =
        engine == 0 ? sssp::EngineKind::serial : sssp::EngineKind::partitioned;
    const sssp::detail::TimedRun tr = sssp::detail::timed_run(kind, g, source, workers, reps);
    if (dist && pred) copy_out(tr.result, dist, pred);
    *total_s = tr.record.total_s;
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RS_ERR;
  }
}

// Serial solve over a Graph that the caller keeps alive between calls, so a
// benchmark can time repeated solves without re-copying the matrix.
void* ref_graph_new(const std::uint64_t* adj, std::uint64_t n, int directed) {
  try {
    return new sssp::Graph(make_graph(adj, n, directed));
  } catch (...) {
    return nullptr;
  }
}

void ref_graph_free(void* g) { delete static_cast<sssp::Graph*>(g); }

int ref_graph_serial(void* gp, std::uint64_t source, std::uint64_t* dist, std::uint64_t* pred) {
  try {
    const sssp::ShortestPathResult r =
        sssp::dijkstra_serial(*static_cast<sssp::Graph*>(gp), source);
    if (dist && pred) copy_out(r, dist, pred);
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  }
}

int ref_graph_partitioned(void* gp, std::uint64_t source, std::uint64_t p, std::uint64_t* dist,
                          std::uint64_t* pred, double* phases) {
  try {
    const sssp::PartitionedRun run =
        sssp::dijkstra_partitioned(*static_cast<sssp::Graph*>(gp), source, p);
    if (dist && pred) copy_out(run.result, dist, pred);
    if (phases) {
      phases[0] = run.phases.scatter_s;
      phases[1] = run.phases.rounds_s;
      phases[2] = run.phases.gather_s;
    }
    return RS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RS_BAD_SOURCE;
  }
}

}  // extern "C"
