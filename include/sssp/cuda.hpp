// sssp/cuda.hpp -- C++ drop-in for the reference's solve entry points.
//
// Add this header next to the reference's proj/include/sssp/*.hpp and link
// libsssp_cuda.so.  It keeps the reference's own types (sssp::Graph,
// graph.hpp:33-58; sssp::ShortestPathResult, result.hpp:13-19; VertexId,
// weight.hpp:9-21) and its error behaviour:
//
//   reference                                        drop-in (B200)
//   dijkstra_serial(g, s)            serial.hpp:65   sssp::cuda::dijkstra(g, s)
//   dijkstra_serial(g, s, c, &vo)    serial.hpp:26   sssp::cuda::dijkstra(g, s, c, &vo)
//   dijkstra_partitioned(g, s, p, m) partitioned:184 sssp::cuda::dijkstra_partitioned(g, s, p, m)
//                                                    (the reference's PartitionedRun: result,
//                                                    CollectiveStats, PartitionedPhases), or
//                                                    sssp::cuda::dijkstra_partitioned(g, s, devices)
//   dijkstra_dataparallel(g, s)      dataparallel:302 sssp::cuda::dijkstra_dataparallel(g, s)
//   parse_edge_list_text(in)         graph.hpp:126   sssp::cuda::parse_edge_list_text(text)
//   (repeated solves on one graph)                   sssp::cuda::DeviceGraph
//
// Results are bit-identical to dijkstra_serial (dist AND pred), so
// `sssp::cuda::dijkstra(g, s) == sssp::dijkstra_serial(g, s)` holds; the
// data-parallel drop-in equals dijkstra_dataparallel (result and rounds).
// source >= n throws std::invalid_argument (serial.hpp:30); every other
// failure throws std::runtime_error -- there is no CPU fallback.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "sssp/graph.hpp"
#include "sssp/partitioned.hpp"
#include "sssp/result.hpp"
#include "sssp/serial.hpp"
#include "sssp/weight.hpp"
#include "sssp_cuda.h"
#include "sssp_graph_gen.h"

namespace sssp::cuda {

// Mirrors DataParallelRun's timing scope {transfer_in, rounds, transfer_out}
// (dataparallel.hpp:284-296, bench.hpp:50-51).
struct Phases {
  double transfer_in_s = 0;
  double rounds_s = 0;
  double transfer_out_s = 0;
};

struct CudaRun {
  ShortestPathResult result;
  Phases phases;
  std::size_t iterations = 0;  // elections executed (vertices reached)
  sssp_solve_stats stats{};
};

inline void check(int rc, const char* where) {
  if (rc == SSSP_OK) return;
  const std::string msg = std::string(where) + ": " + sssp_status_string(rc) + " (" +
                          sssp_last_error() + ")";
  if (rc == SSSP_ERR_BAD_SOURCE) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// A Graph resident in HBM; one GPU, or several column shards (one per entry of
// `devices`, partition.hpp:31-41).  Not safe for concurrent solves.
class DeviceGraph {
 public:
  explicit DeviceGraph(const Graph& g, std::vector<int> devices = {0},
                       const sssp_options* opt = nullptr)
      : n_(g.n) {
    static_assert(sizeof(Weight) == sizeof(std::uint64_t), "Weight is uint64 (weight.hpp:9)");
    check(sssp_graph_create(g.adj.data(), g.n, g.directed ? 1 : 0, devices.data(),
                            static_cast<int>(devices.size()), opt, &h_),
          "sssp_graph_create");
  }
  // Built on the device from the reference's EdgeList (graph.hpp:20-26) with
  // graph_from_edges semantics (graph.hpp:73-88); `directed` is the -w switch.
  DeviceGraph(const EdgeList& el, bool directed, std::vector<int> devices = {0},
              const sssp_options* opt = nullptr)
      : n_(el.n) {
    std::vector<std::uint64_t> e;
    e.reserve(el.edges.size() * 3);
    for (const Edge& x : el.edges) {
      e.push_back(x.u);
      e.push_back(x.v);
      e.push_back(x.w);
    }
    const int rc = sssp_graph_create_from_edges(el.n, e.data(), el.edges.size(), directed ? 1 : 0,
                                                devices.data(), static_cast<int>(devices.size()),
                                                opt, &h_);
    if (rc == SSSP_ERR_BAD_ARG) throw std::invalid_argument("graph_from_edges: bad edge");
    check(rc, "sssp_graph_create_from_edges");
  }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
  DeviceGraph(DeviceGraph&& o) noexcept : h_(std::exchange(o.h_, nullptr)), n_(o.n_) {}
  ~DeviceGraph() {
    if (h_) sssp_graph_destroy(h_);
  }

  CudaRun run(VertexId source, std::vector<VertexId>* visit_order = nullptr) {
    if (source >= n_) throw std::invalid_argument("dijkstra: source out of range");
    CudaRun r;
    r.result.source = source;
    r.result.dist.resize(n_);
    r.result.pred.resize(n_);
    std::vector<std::uint64_t> vo(visit_order ? n_ : 0);
    static_assert(sizeof(VertexId) == sizeof(std::uint64_t), "VertexId is 64-bit (LP64)");
    check(sssp_solve(h_, source, r.result.dist.data(),
                     reinterpret_cast<std::uint64_t*>(r.result.pred.data()),
                     visit_order ? vo.data() : nullptr, &r.stats),
          "sssp_solve");
    r.phases = {r.stats.transfer_in_s, r.stats.rounds_s, r.stats.transfer_out_s};
    r.iterations = r.stats.iterations;
    // all n rounds: the reachable vertices in election order, then the
    // unreachable ones in ascending id (serial.hpp:41-48)
    if (visit_order) visit_order->assign(vo.begin(), vo.end());
    return r;
  }

  ShortestPathResult solve(VertexId source) { return run(source).result; }

  std::vector<ShortestPathResult> solve_batch(const std::vector<VertexId>& sources) {
    for (VertexId s : sources)
      if (s >= n_) throw std::invalid_argument("dijkstra: source out of range");
    std::vector<std::uint64_t> src(sources.begin(), sources.end());
    std::vector<std::uint64_t> dist(src.size() * n_), pred(src.size() * n_);
    check(sssp_solve_batch(h_, src.data(), static_cast<std::uint32_t>(src.size()), dist.data(),
                           pred.data(), nullptr),
          "sssp_solve_batch");
    std::vector<ShortestPathResult> out(src.size());
    for (std::size_t i = 0; i < src.size(); ++i) {
      out[i].source = sources[i];
      out[i].dist.assign(dist.begin() + i * n_, dist.begin() + (i + 1) * n_);
      out[i].pred.assign(pred.begin() + i * n_, pred.begin() + (i + 1) * n_);
    }
    return out;
  }

  // The paper's data-parallel engine (dataparallel.hpp:302-327): result and
  // round count equal dijkstra_dataparallel's.
  CudaRun run_dataparallel(VertexId source, std::size_t* rounds = nullptr) {
    if (source >= n_) throw std::invalid_argument("dijkstra_dataparallel: source out of range");
    CudaRun r;
    r.result.source = source;
    r.result.dist.resize(n_);
    r.result.pred.resize(n_);
    std::uint64_t nr = 0;
    check(sssp_solve_dataparallel(h_, source, r.result.dist.data(),
                                  reinterpret_cast<std::uint64_t*>(r.result.pred.data()), &nr,
                                  &r.stats),
          "sssp_solve_dataparallel");
    r.phases = {r.stats.transfer_in_s, r.stats.rounds_s, r.stats.transfer_out_s};
    r.iterations = nr;
    if (rounds) *rounds = nr;
    return r;
  }

  sssp_graph* handle() const { return h_; }

 private:
  sssp_graph* h_ = nullptr;
  std::size_t n_ = 0;
};

// parse_edge_list_text (graph.hpp:126-170) on all host threads: same EdgeList,
// same ParseError (line and message) for input the reference rejects.
inline EdgeList parse_edge_list_text(std::string_view text) {
  std::uint64_t n = 0, m = 0, line = 0;
  char err[512] = {};
  int rc = sssp_parse_edge_list(text.data(), text.size(), &n, &m, nullptr, 0, &line, err, sizeof(err));
  std::vector<std::uint64_t> e;
  if (rc == SSSP_OK) {
    e.resize(3 * m);
    rc = sssp_parse_edge_list(text.data(), text.size(), &n, &m, e.data(), m, &line, err, sizeof(err));
  }
  if (rc != SSSP_OK) {
    if (line) {
      const std::string msg(err);
      const std::size_t k = msg.find(": ");
      throw ParseError(line, k == std::string::npos ? msg : msg.substr(k + 2));
    }
    check(rc, "sssp_parse_edge_list");
  }
  EdgeList el;
  el.n = n;
  el.edges.resize(m);
  for (std::uint64_t i = 0; i < m; ++i) el.edges[i] = {e[3 * i], e[3 * i + 1], e[3 * i + 2]};
  return el;
}

// Drop-in for dijkstra_serial(g, source) (serial.hpp:65-68).
inline ShortestPathResult dijkstra(const Graph& g, VertexId source,
                                   std::vector<VertexId>* visit_order = nullptr) {
  if (source >= g.n) throw std::invalid_argument("dijkstra: source out of range");
  sssp_options opt{};
  opt.flags = SSSP_FLAGS_DEFAULT;
  opt.record_visit_order = visit_order ? 1 : 0;
  DeviceGraph dg(g, {0}, &opt);
  return dg.run(source, visit_order).result;
}

// Drop-in for dijkstra_serial(g, source, counters, visit_order) (serial.hpp:26-28):
// the counters are the reference's own definition of the work, n*n each
// (serial.hpp:13-19); the device's actual work is in CudaRun::stats.
inline ShortestPathResult dijkstra(const Graph& g, VertexId source, OpCounters& counters,
                                   std::vector<VertexId>* visit_order = nullptr) {
  if (source >= g.n) throw std::invalid_argument("dijkstra_serial: source out of range");
  sssp_options opt{};
  opt.flags = SSSP_FLAGS_DEFAULT;
  opt.record_visit_order = visit_order ? 1 : 0;
  DeviceGraph dg(g, {0}, &opt);
  CudaRun r = dg.run(source, visit_order);
  counters.extract_min_scans = r.stats.extract_min_scans;
  counters.relax_checks = r.stats.ref_relax_checks;
  return std::move(r.result);
}

// The same solve with the phase timings of the data-parallel scope.
inline CudaRun dijkstra_run(const Graph& g, VertexId source) {
  if (source >= g.n) throw std::invalid_argument("dijkstra: source out of range");
  DeviceGraph dg(g);
  return dg.run(source);
}

// Drop-in for dijkstra_partitioned(g, source, p, mode) (partitioned.hpp:184-225),
// returning the reference's own PartitionedRun.  The p column shards are dealt
// round-robin over the visible GPUs, at most SSSP_MAX_SHARDS of them (dist and
// pred do not depend on p: partitioned == serial, test_partitioned.cpp:135-165);
// the shards of one GPU run as one launch, the analogue of WorkerMode::sequential
// (partitioned.hpp:142-154), so `mode` changes nothing.  stats are the
// reference's CollectiveStats for THIS p (allreduce_count = padded_n, scatter /
// gather bytes of workers 1..p-1); phases = {upload, kernel, download}.  A graph
// that needs 64-bit distances runs on one shard (same result).
inline PartitionedRun dijkstra_partitioned(const Graph& g, VertexId source, std::size_t p,
                                           WorkerMode mode = WorkerMode::threaded) {
  (void)mode;
  if (p < 1) throw std::invalid_argument("dijkstra_partitioned: p >= 1");
  if (source >= g.n) throw std::invalid_argument("dijkstra_partitioned: source out of range");
  int ndev = 0;
  check(sssp_device_count(&ndev), "sssp_device_count");
  const std::size_t shards = std::min<std::size_t>({p, (std::size_t)SSSP_MAX_SHARDS,
                                                    std::max<std::size_t>(g.n, 1)});
  std::vector<int> devices(shards);
  for (std::size_t i = 0; i < shards; ++i) devices[i] = static_cast<int>(i % std::max(ndev, 1));
  sssp_graph* h = nullptr;
  int rc = sssp_graph_create(g.adj.data(), g.n, g.directed ? 1 : 0, devices.data(),
                             static_cast<int>(devices.size()), nullptr, &h);
  if (rc == SSSP_ERR_UNSUPPORTED && shards > 1)  // 64-bit distances: one shard
    rc = sssp_graph_create(g.adj.data(), g.n, g.directed ? 1 : 0, devices.data(), 1, nullptr, &h);
  check(rc, "sssp_graph_create");
  PartitionedRun run;
  run.result.source = source;
  run.result.dist.resize(g.n);
  run.result.pred.resize(g.n);
  sssp_solve_stats st{};
  rc = sssp_solve(h, source, run.result.dist.data(),
                  reinterpret_cast<std::uint64_t*>(run.result.pred.data()), nullptr, &st);
  sssp_graph_destroy(h);
  check(rc, "sssp_solve");
  const PartitionPlan plan = make_partition_plan(g.n, p);
  run.stats.allreduce_count = plan.padded_n;
  for (std::size_t k = 1; k < p; ++k) {
    const std::size_t loc = plan.ranges[k].second - plan.ranges[k].first;
    run.stats.scatter_bytes += plan.padded_n * loc * sizeof(Weight);
    run.stats.gather_bytes += loc * (sizeof(Weight) + sizeof(VertexId));
  }
  run.phases.scatter_s = st.transfer_in_s;
  run.phases.rounds_s = st.rounds_s;
  run.phases.gather_s = st.transfer_out_s;
  return run;
}

// Column-partitioned over one shard per device (partitioned.hpp:184-225);
// repeat a device id to run several shards on one GPU.
inline ShortestPathResult dijkstra_partitioned(const Graph& g, VertexId source,
                                               std::vector<int> devices) {
  if (devices.empty()) throw std::invalid_argument("dijkstra_partitioned: p >= 1");
  if (source >= g.n) throw std::invalid_argument("dijkstra_partitioned: source out of range");
  DeviceGraph dg(g, std::move(devices));
  return dg.solve(source);
}

// Mirrors DataParallelRun (dataparallel.hpp:284-296): result, rounds, phases.
struct DataParallelRun {
  ShortestPathResult result;
  std::size_t rounds = 0;
  Phases phases;
  std::size_t cells_in = 0;   // n*n, as transfer_in reports (:269-276)
  std::size_t cells_out = 0;  // 2n (:279-282)
};

// Drop-in for dijkstra_dataparallel(g, source) (dataparallel.hpp:302-327).
inline DataParallelRun dijkstra_dataparallel(const Graph& g, VertexId source) {
  if (source >= g.n) throw std::invalid_argument("dijkstra_dataparallel: source out of range");
  DeviceGraph dg(g);
  DataParallelRun out;
  CudaRun r = dg.run_dataparallel(source, &out.rounds);
  out.result = std::move(r.result);
  out.phases = r.phases;
  out.cells_in = g.n * g.n;
  out.cells_out = 2 * g.n;
  return out;
}

}  // namespace sssp::cuda
