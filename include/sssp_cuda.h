/*
 * sssp_cuda.h -- C ABI of the B200-native matrix-scan Dijkstra.
 *
 * Drop-in boundary for the reference's solve path:
 *   reference  sssp::dijkstra_serial(const Graph&, VertexId)      serial.hpp:65-68
 *              sssp::dijkstra_serial(g, s, OpCounters&, visit*)  serial.hpp:26-28
 *              sssp::dijkstra_partitioned(g, s, p, mode)         partitioned.hpp:184-186
 *   replaced by  sssp_graph_create + sssp_solve (+ sssp_graph_destroy); the C++
 *   wrapper include/sssp/cuda.hpp restores the reference's exact signature and
 *   return type (ShortestPathResult, result.hpp:13-19).
 *
 * Plain pointers and sizes only; no exceptions cross this boundary.  The
 * input is the reference's own Graph::adj layout: row-major n*n uint64
 * weights, UINT64_MAX = no edge (weight.hpp:13, graph.hpp:30-45).  Outputs
 * use the reference encoding: dist UINT64_MAX = unreachable, pred
 * UINT64_MAX = kNoVertex (weight.hpp:13, :21).
 *
 * Threading: a handle is not safe for concurrent solves (its exchange
 * buffers and scratch are per handle); distinct handles are independent.
 * Every solve is synchronous unless the *_enqueue entry points are used.
 * There is no CPU fallback: without a usable CUDA device every entry point
 * returns SSSP_ERR_CUDA.
 */
#ifndef SSSP_CUDA_H
#define SSSP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSSP_ABI_VERSION 3 /* 2: sssp_options.record_round_times, sssp_solve_dataparallel, sssp_round_times
                              3: SSSP_ENGINE_WIDE (64-bit distances), the reference's OpCounters /
                                 CollectiveStats and device exchange counts in sssp_solve_stats */
#define SSSP_IPC_HANDLE_BYTES 64 /* sizeof(cudaIpcMemHandle_t) */
#define SSSP_MAX_SHARDS 8

typedef enum {
  SSSP_OK = 0,
  SSSP_ERR_BAD_SOURCE = 1,   /* source >= n: std::invalid_argument at serial.hpp:30 */
  SSSP_ERR_BAD_ARG = 2,      /* p < 1 (partitioned.hpp:187), n == 0, bad shard ids ... */
  SSSP_ERR_WEIGHT_RANGE = 3, /* (ABI < 3) a weight/distance the 32-bit encoding cannot hold;
                                since ABI 3 such graphs run on SSSP_ENGINE_WIDE */
  SSSP_ERR_OOM = 4,          /* device or pinned-host allocation failed */
  SSSP_ERR_CUDA = 5,         /* CUDA runtime error (no device, launch failure ...) */
  SSSP_ERR_NO_PEER = 6,      /* peer access / IPC import failed between shards */
  SSSP_ERR_TIMEOUT = 7,      /* the persistent kernel's exchange watchdog fired */
  SSSP_ERR_UNSUPPORTED = 8   /* configuration not supported on this device */
} sssp_status;

/* Solve engines -- all bit-identical to dijkstra_serial.
 * GRID / CLUSTER run the reference's n rounds in one persistent kernel and
 * differ in how a round's election is exchanged.  BUCKET settles a whole
 * distance class per step and is exact only when every finite off-diagonal
 * weight is >= 1.  AUTO: WIDE when distances need 64 bits; else BUCKET when
 * it is exact (any number of shards), else CLUSTER.  In one process an AUTO
 * bucket solve that needs more than n/12 distance classes stops and reruns on
 * CLUSTER inside the same call (classes cost ~12 scan rounds each), and the
 * handle keeps CLUSTER for its later solves. */
typedef enum {
  SSSP_ENGINE_AUTO = 0,
  SSSP_ENGINE_GRID = 1,    /* single-warp CTAs across the GPU, exchange through L2 */
  SSSP_ENGINE_CLUSTER = 2, /* one thread-block cluster per solve, exchange through DSMEM */
  SSSP_ENGINE_BUCKET = 3,  /* distance-class steps, push/pull over B200 HBM */
  SSSP_ENGINE_DATAPARALLEL = 4, /* reported by sssp_solve_dataparallel only */
  SSSP_ENGINE_WIDE = 5     /* 64-bit distances (a weight of 2^32-1, or n*max_weight >= 2^32-1):
                              n-round cluster kernel, one shard; AUTO/CLUSTER select it */
} sssp_engine;

typedef struct {
  int engine;             /* sssp_engine */
  uint32_t ctas_per_shard;/* 0 = auto; CTAs of one solve on one shard (cluster engine:
                             the cluster size, <= 16; grid engine: <= SM count) */
  uint32_t flags;         /* bit0: runner-up row prefetch, bit1: owner L2 row prefetch;
                             SSSP_FLAGS_DEFAULT when the options pointer is NULL */
  uint32_t max_batch;     /* concurrent solves a batch launch may run (0 = auto) */
  uint64_t timeout_ms;    /* exchange watchdog (0 = 60000) */
  int record_visit_order; /* 1: keep the elected vertex of every round */
  uint32_t replicas;      /* grid engine: copies of the L2 exchange array (0 = 1) */
  uint32_t warps_per_cta; /* cluster engine: 4, 8 or 16 (0 = 4) */
  int64_t global_min_weight; /* shard mode: smallest finite off-diagonal weight of the WHOLE
                                graph (sssp_block_weight_range + an allreduce), -1 = unknown;
                                the bucket engine needs it >= 1 on every rank */
  int record_round_times; /* cluster engine: %globaltimer at the end of every round of the
                             last solve (sssp_round_times; SURVEY §8d latency histogram);
                             runs a traced kernel instance, the untraced one is unchanged */
} sssp_options;

#define SSSP_FLAGS_DEFAULT 3u /* bit2 (4): speculative relax, off by default */

/* Per-solve statistics; phases mirror the reference's data-parallel timing
 * scope {transfer_in, rounds, transfer_out} (bench.hpp:50-51). */
typedef struct {
  double transfer_in_s;   /* graph upload (narrow + permute + H2D) of the handle */
  double rounds_s;        /* kernel time, CUDA events on the launch stream */
  double transfer_out_s;  /* D2H of dist/pred */
  uint64_t iterations;    /* vertices settled (= elections executed / vertices reached) */
  uint64_t relax_checks;  /* iterations * columns scanned (OpCounters analogue) */
  uint64_t mispredicts;   /* rounds whose row was not prefetched */
  uint64_t matrix_bytes;  /* device bytes of the stored matrix (all local shards) */
  uint32_t weight_bytes;  /* device weight encoding: 1, 2 or 4 bytes */
  uint32_t ctas;          /* CTAs per solve per shard */
  uint32_t shards;        /* P */
  uint32_t packed_key;    /* 1 if the single-redux packed local key is in use */
  uint32_t engine;        /* sssp_engine that ran */
  uint32_t classes;       /* BUCKET: distance classes (steps) */
  uint64_t rows_read;     /* matrix rows streamed (scan: = iterations) */
  /* ABI 3.  The reference's own instrumentation, as it defines it for this
   * input (so a caller of the drop-in reads the numbers the reference would):
   *   OpCounters (serial.hpp:16-19): both counters are n*n for every solve;
   *   CollectiveStats (partitioned.hpp:28-32) of dijkstra_partitioned with
   *   p = shards: allreduce_count = padded_n (:205), scatter_bytes = uint64
   *   bytes of the column blocks of workers 1..p-1 (:196-198), gather_bytes =
   *   dist + pred bytes of workers 1..p-1 (:219-221); 0 for p = 1.
   * And what the device actually executed: */
  uint64_t extract_min_scans; /* OpCounters::extract_min_scans = n*n */
  uint64_t ref_relax_checks;  /* OpCounters::relax_checks = n*n */
  uint64_t allreduce_count;   /* CollectiveStats::allreduce_count = padded_n */
  uint64_t scatter_bytes;     /* CollectiveStats::scatter_bytes */
  uint64_t gather_bytes;      /* CollectiveStats::gather_bytes */
  uint64_t exchanges;         /* device global-argmin exchanges executed per solve (mean over
                                 a batch): scan / wide engines one per election (rounds until
                                 the first INF election), bucket one per distance class */
  uint64_t barriers;          /* device-wide barriers per solve (bucket: grid barriers incl.
                                 pull-combine barriers; scan / wide: = exchanges) */
  uint64_t upload_bytes;      /* host->device bytes of the graph upload (all local shards) */
  uint64_t download_bytes;    /* device->host bytes of one solve's dist + pred */
  uint64_t bytes_read;        /* matrix bytes the solve kernel loaded per solve, all local shards
                                 (bucket: counted by every CTA; scan / wide: rows x row bytes) */
} sssp_solve_stats;

typedef struct sssp_graph sssp_graph;

const char* sssp_status_string(int status);
const char* sssp_last_error(void); /* thread-local detail of the last failure */
int sssp_abi_version(void);
int sssp_device_count(int* count);

/* Single-GPU (devices == NULL or ndev == 1) or single-process multi-GPU
 * column-partitioned graph: shard k of P = ndev owns columns
 * [k*loc_n, (k+1)*loc_n) with loc_n = pad_vertex_count(n, P)/P
 * (partition.hpp:25-41).  Repeating a device id runs several shards on one
 * GPU (the "P logical shards" simulation of the multi-GPU protocol).
 * `directed` is recorded only; the matrix is taken as given. */
int sssp_graph_create(const uint64_t* adj, uint64_t n, int directed, const int* devices,
                      int ndev, const sssp_options* opt, sssp_graph** out);

/* Same, built on the device from an edge list instead of the n*n matrix:
 * `edges` = m (u, v, w) uint64 triples, exactly what graph_from_edges
 * (graph.hpp:73-88) consumes -- minimum over duplicates, mirrored unless
 * `directed` (the '-w' switch).  Rejects endpoint >= n, self-loops and
 * w > 2^32-1 with SSSP_ERR_BAD_ARG like the reference's invalid_argument.
 * Only O(m) bytes cross PCIe (config 4: 100 MB instead of a 32 GiB matrix). */
int sssp_graph_create_from_edges(uint64_t n, const uint64_t* edges, uint64_t m, int directed,
                                 const int* devices, int ndev, const sssp_options* opt,
                                 sssp_graph** out);

/* One process per GPU: this process owns shard `rank` of `world`.
 * `block` holds rows 0..n-1 of the shard's real columns
 * [rank*loc_n, min(n, (rank+1)*loc_n)) with leading dimension `ld` (pass the
 * full matrix with ld = n and block = adj + rank*loc_n, or a column block).
 * `max_weight` = largest finite weight of the WHOLE graph (0 = derive it from
 * the block, exact only when world == 1).  After every rank has called
 * sssp_shard_export, pass the world * SSSP_IPC_HANDLE_BYTES handles gathered
 * in rank order to sssp_shard_connect. */
int sssp_shard_create(const uint64_t* block, uint64_t ld, uint64_t n, uint32_t world,
                      uint32_t rank, uint64_t max_weight, int device, const sssp_options* opt,
                      sssp_graph** out);
int sssp_shard_export(sssp_graph* g, void* handle_out);
int sssp_shard_connect(sssp_graph* g, const void* handles);
/* Columns [*col_begin, *col_begin + *col_count) are this process's slice. */
int sssp_shard_range(const sssp_graph* g, uint64_t* col_begin, uint64_t* col_count);
/* Finite weight range of a column block (rows 0..n-1, global column offset
 * col_begin, leading dimension ld): *min_offdiag excludes the diagonal
 * (UINT64_MAX if there is no edge), *max_finite includes it.  Host only. */
int sssp_block_weight_range(const uint64_t* block, uint64_t ld, uint64_t n, uint64_t col_begin,
                            uint64_t col_count, uint64_t* min_offdiag, uint64_t* max_finite);

int sssp_graph_destroy(sssp_graph* g);
int sssp_graph_info(const sssp_graph* g, sssp_solve_stats* st);

/* Synchronous solve.  dist_out/pred_out: n entries (single process), or the
 * shard's col_count entries in shard mode.  visit_order_out (optional, n
 * entries; needs record_visit_order): the vertex elected in every round of
 * dijkstra_serial -- the stats.iterations reachable ones in election order,
 * then the unreachable ones in ascending id, as the reference's later rounds
 * elect them (serial.hpp:41-48). */
int sssp_solve(sssp_graph* g, uint64_t source, uint64_t* dist_out, uint64_t* pred_out,
               uint64_t* visit_order_out, sssp_solve_stats* st);

/* k independent sources; outputs are k consecutive n-entry rows. */
int sssp_solve_batch(sssp_graph* g, const uint64_t* sources, uint32_t k, uint64_t* dist_out,
                     uint64_t* pred_out, sssp_solve_stats* st);

/* Asynchronous form for device-side timing: enqueue k solves on the handle's
 * stream (results stay on the device); several enqueues queue up in stream
 * order and reuse the output slots.  sssp_finish waits, checks the watchdog
 * and reports the last launch (rounds_s = mean kernel time per launch).  sssp_stream returns the cudaStream_t of shard `local` as a
 * pointer so a caller can record its own CUDA events around the launches. */
int sssp_enqueue(sssp_graph* g, const uint64_t* sources, uint32_t k);
int sssp_finish(sssp_graph* g, sssp_solve_stats* st);
void* sssp_stream(sssp_graph* g, int local);

/* validate_result (oracle.hpp:51-120) on the device against the stored matrix:
 * *violations = number of failed checks (0 = a valid shortest-path tree with
 * fixpoint distances).  dist/pred: n entries, reference encoding.  The
 * reference harness refuses to time invalid results (bench.hpp:167-173). */
int sssp_validate(sssp_graph* g, uint64_t source, const uint64_t* dist, const uint64_t* pred,
                  uint64_t* violations);

/* The paper's data-parallel engine: dijkstra_dataparallel(g, s)
 * (dataparallel.hpp:302-327; Alg. 3-4) -- synchronous relaxation
 * rounds to the fixpoint, then reconstruct_predecessors (:221-264).  dist
 * equals dijkstra_serial's; pred follows the reference's reconstruction (it
 * differs from serial's on tie-heavy graphs, exactly as the reference's
 * does); *rounds_out = DataParallelRun::rounds (relax rounds executed,
 * including the final one that changes nothing).  Bad source:
 * SSSP_ERR_BAD_SOURCE (std::invalid_argument at :305).  One shard only.
 * stats.classes = pass-number sweeps needed by zero-weight ties (0: none). */
int sssp_solve_dataparallel(sssp_graph* g, uint64_t source, uint64_t* dist_out,
                            uint64_t* pred_out, uint64_t* rounds_out, sssp_solve_stats* st);

/* Per-round %globaltimer stamps (ns) of the last scan-engine solve (needs
 * record_round_times; source's shard 0): *count = rounds recorded, at most
 * cap written.  Differences of consecutive stamps = per-round latency. */
int sssp_round_times(sssp_graph* g, uint64_t* ns_out, uint64_t cap, uint64_t* count);

/* t_sync_min microbenchmark (the roofline's sync term): runs
 * `rounds` exchange rounds with the solve's launch shape and exchange code
 * but no relaxation; *seconds_per_round = max over shards of elapsed/rounds
 * (device %globaltimer).  Collective in shard mode: every rank must call. */
int sssp_probe_sync(sssp_graph* g, uint32_t rounds, double* seconds_per_round);

/* Host-driven comparison path: the reference's partitioned
 * round (partitioned.hpp:142-154) with the allreduce done by the HOST between
 * two launches -- begin(source) once, then every round
 *   sssp_nccl_local_min(g, key)   local_min (:81-90) -> 8-byte key on the device
 *   <caller: ncclAllReduce(key, int64, MIN) across the shards' ranks>
 *   sssp_nccl_relax(g, key)       relax_owned (:106-119) with the winner
 * for n rounds, then end() copies this shard's dist/pred (col_count entries;
 * n for one process).  Key = (dist << 32 | vertex) ^ 2^63: signed MIN orders it
 * as the (dist, vertex) MinLocPair.  Kernels run on sssp_stream(g, 0).  One
 * local shard, 32-bit distances; results bit-identical to dijkstra_serial. */
int sssp_nccl_begin(sssp_graph* g, uint64_t source);
int sssp_nccl_local_min(sssp_graph* g, uint64_t* d_key);
int sssp_nccl_relax(sssp_graph* g, const uint64_t* d_key);
int sssp_nccl_end(sssp_graph* g, uint64_t* dist_out, uint64_t* pred_out);

/* The bucket engine's synchronisation floor (SURVEY.md §8d roofline, sync
 * term): `launches` back-to-back cooperative launches of an empty kernel with
 * the solve's grid, block and shared memory doing `barriers` grid barriers;
 * *seconds_per_launch = CUDA-event time / launches.  Single-shard bucket
 * graphs only (SSSP_ERR_UNSUPPORTED otherwise). */
int sssp_probe_skeleton(sssp_graph* g, uint32_t barriers, uint32_t launches,
                        double* seconds_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* SSSP_CUDA_H */
