// sssp_host.cu -- the C-ABI host side (include/sssp_cuda.h).
//
// Owns: choosing the device encoding of the reference's uint64 matrix
// (weight.hpp:9-26), the column partition (partition.hpp:25-41), the
// narrow -> H2D -> permute upload pipeline, the exchange buffers of the
// persistent kernel (scan_kernel.cuh), and the launch / finish / D2H of a
// solve.  No CPU solve path exists: every error surfaces as a status code.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sssp_cuda.h"
#include "bucket_kernel.cuh"
#include "dataparallel_kernel.cuh"
#include "validate_kernel.cuh"
#include "wide_kernel.cuh"
#include "nccl_kernel.cuh"
#include "dispatch.h"
#include "host_narrow.h"

using namespace sssp_b200;
namespace sssp_b200 {  // kernels_bucket_u*.cu: variant 0 one shard, 1 slots, 2 sharded
void* bucket_fn_u8(int variant);
void* bucket_fn_u16(int variant);
void* bucket_fn_u32(int variant);
}  // namespace sssp_b200

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? SSSP_ERR_OOM : SSSP_ERR_CUDA,    \
                  std::string(#call) + ": " + cudaGetErrorString(e_));               \
    }                                                                                \
  } while (0)

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

uint32_t bitlen(uint64_t x) {
  uint32_t b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// partition.hpp:25-29
uint64_t pad_vertex_count(uint64_t n, uint64_t p) {
  if (p > n) return p;
  return n + (p - n % p) % p;
}

// Rearranges a chunk of staged rows (natural column order) into the
// cyclic-by-CTA layout of scan_kernel.cuh.  Padding columns get INF.
template <typename W>
__global__ void permute_rows_kernel(const W* __restrict__ stage, uint32_t cols,
                                    W* __restrict__ dst, uint64_t row_stride, uint64_t row0,
                                    uint32_t rows, uint32_t G, uint32_t L) {
  const uint64_t total = (uint64_t)rows * row_stride;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = idx / row_stride;
    const uint32_t q = (uint32_t)(idx - r * row_stride);
    const uint32_t c = q / L, s = q - c * L;
    const uint32_t vl = s * G + c;
    dst[(row0 + r) * row_stride + q] =
        vl < cols ? stage[r * cols + vl] : (W)WInf<W>::v;
  }
}

// ---- device-side graph_from_edges (graph.hpp:73-88) into the permuted layout

// Rows u < n: INF everywhere, 0 on the diagonal (graph.hpp:37-44).
template <typename W>
__global__ void init_matrix_kernel(W* __restrict__ a, uint64_t n, uint64_t row_stride,
                                   uint64_t col_base, uint64_t cols, uint32_t G, uint32_t L) {
  const uint64_t total = n * row_stride;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = idx / row_stride;
    const uint32_t q = (uint32_t)(idx - u * row_stride);
    const uint32_t c = q / L, sl = q - c * L;
    const uint64_t vl = (uint64_t)sl * G + c;
    a[idx] = (vl < cols && col_base + vl == u) ? (W)0 : (W)WInf<W>::v;
  }
}

// Keep-the-minimum store of w into cell (u, position of local column vl);
// sub-word weights use a CAS on the containing 32-bit word.
template <typename W>
__device__ __forceinline__ void min_cell(W* a, uint64_t row_stride, uint64_t u, uint64_t vl,
                                         uint32_t G, uint32_t L, uint32_t w) {
  const uint64_t pos = (vl % G) * L + vl / G;
  W* cell = a + u * row_stride + pos;
  if constexpr (sizeof(W) == 8) {
    atomicMin(reinterpret_cast<unsigned long long*>(cell), (unsigned long long)w);
  } else if constexpr (sizeof(W) == 4) {
    atomicMin(reinterpret_cast<unsigned int*>(cell), w);
  } else {
    unsigned int* word = reinterpret_cast<unsigned int*>(reinterpret_cast<uintptr_t>(cell) & ~(uintptr_t)3);
    const uint32_t sh = (uint32_t)((reinterpret_cast<uintptr_t>(cell) & 3) * 8);
    const uint32_t mask = (uint32_t)WInf<W>::v << sh;
    unsigned int old = *word, assumed;
    do {
      assumed = old;
      if (((assumed & mask) >> sh) <= w) break;
      old = atomicCAS(word, assumed, (assumed & ~mask) | (w << sh));
    } while (old != assumed);
  }
}

template <typename W>
__global__ void scatter_edges_kernel(const uint64_t* __restrict__ e, uint64_t m, W* __restrict__ a,
                                     uint64_t row_stride, uint64_t col_base, uint64_t cols,
                                     uint32_t G, uint32_t L, int directed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e[3 * i], v = e[3 * i + 1];
    const uint32_t w = (uint32_t)e[3 * i + 2];
    if (v >= col_base && v < col_base + cols) min_cell<W>(a, row_stride, u, v - col_base, G, L, w);
    if (!directed && u >= col_base && u < col_base + cols)
      min_cell<W>(a, row_stride, v, u - col_base, G, L, w);
  }
}

template <typename F>
void parallel_for(uint64_t begin, uint64_t end, unsigned nthreads, F&& f) {
  if (end <= begin) return;
  nthreads = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nthreads, end - begin));
  if (nthreads == 1) {
    f(begin, end, 0u);
    return;
  }
  std::vector<std::thread> ts;
  const uint64_t span = end - begin;
  for (unsigned t = 0; t < nthreads; ++t) {
    const uint64_t a = begin + span * t / nthreads, b = begin + span * (t + 1) / nthreads;
    ts.emplace_back([&f, a, b, t] { f(a, b, t); });
  }
  for (auto& th : ts) th.join();
}

unsigned host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(h ? h : 1u, 32u));
}

}  // namespace

struct Shard {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* d_adj = nullptr;
  uint64_t row_stride = 0;  // G*L
  uint32_t G = 0, EPL = 0, L = 0, NP = 0;  // G = participants (warps) per solve
  uint32_t C = 1, NW = 1;                   // cluster engine: CTAs per cluster, warps per CTA
  bool hier = false;                        // cluster engine: hierarchical (CTA pre-reduction)
  uint32_t k = 0;           // shard index
  uint64_t col_base = 0, loc_n = 0, cols = 0;  // cols = real columns held
  uint64_t* d_slots = nullptr;
  uint64_t* d_dist = nullptr;
  uint64_t* d_pred = nullptr;
  uint64_t* d_info = nullptr;
  uint32_t* d_sources = nullptr;
  uint32_t* d_visit = nullptr;
  uint64_t* d_round_ns = nullptr;  // [n] per-round stamps (record_round_times, shard 0)
  bool slots_pooled = false;       // d_slots from the stream-ordered pool (not IPC-exported)
  uint32_t* h_sources = nullptr;  // pinned
  uint64_t* h_info = nullptr;     // pinned
  uint64_t* peer[kMaxShards] = {};
  // bucket engine (bucket_kernel.cuh)
  void* d_adjT = nullptr;        // transpose in position order (nullptr: symmetric or absent)
  uint4* d_rsum = nullptr;       // bucket, one shard: per-row class-1 summaries [n][2] (row_summary_kernel)
  uint32_t* d_rlist = nullptr;   //   ... and the rows' class-1 id lists (row_list_kernel)
  uint32_t* d_spoff = nullptr;   // bucket, one shard, sparse matrix: tile-list offsets [n*G+1]
  uint32_t* d_spent = nullptr;   //   ... and entries (tile_list_kernel); sp_T = their tile
  uint32_t sp_T = 0;
  const void* pull_src = nullptr;// d_adjT, or d_adj when the matrix is symmetric
  uint64_t* d_info2 = nullptr;   // bucket: [B][2] barriers used, watchdog
  uint64_t* d_ctab = nullptr;    // bucket: [B][ctab] matrix bytes loaded per CTA
  uint64_t* d_trace = nullptr;   // debug (SSSP_BUCKET_TRACE)
  unsigned long long* d_spans = nullptr;  // debug (SSSP_BUCKET_SPANS): [64][2] launch spans
  bool peer_ipc[kMaxShards] = {};
  bool own_stream = true;        // false: shares the stream of the device's first shard
  KernelFn fn = nullptr;
};

struct sssp_graph {
  uint64_t n = 0;
  int directed = 0;
  uint32_t P = 1;
  bool multiproc = false;
  bool connected = false;
  std::vector<Shard> sh;
  sssp_options opt{};
  uint32_t wbytes = 0;
  uint64_t max_w = 0, min_w = ~0ull;
  uint32_t vbits = 0, sbits = 0, packed = 0;
  uint32_t max_batch = 1;
  uint64_t slot_stride = 0, bstride = 0;
  uint32_t nrep = 1;
  bool cluster = true;  // scan engine: cluster (DSMEM exchange) or grid (L2 exchange)
  bool bucket = false;  // distance-class engine available and selected (min weight >= 1)
  bool wide = false;    // 64-bit distances (wide_kernel.cuh): a weight of 2^32-1 or n*max_w >= 2^32-1
  uint32_t wPC = 0;     // wide engine: positions per CTA
  // bucket engine layout (identical on every shard)
  uint32_t bT = 0, bG = 0;               // positions per CTA, CTAs per shard
  uint64_t bseq = 0;                     // bucket launch tags (watchdog reports)
  uint32_t bslots = 1;                   // bucket: independent solves per launch (one shard)
  uint32_t bTb = 0, bGb = 0, bslots_b = 0;  // batch tiling: wider tiles, more slots per launch
  uint32_t ctab = 0;                     // bucket: CTAs per solve slot in d_ctab (max tiling)
  uint64_t done_off = 0;                 // bucket: per-slot done flags (after the slot regions)
  uint64_t slots_bytes = 0;              // scan-engine exchange region (start of d_slots)
  uint64_t bar_off = 0, arrive_off = 0, epoch_off = 0, release_off = 0, ctrl_off = 0, bm_off = 0, ubm_off = 0, pkey_off = 0,
           region_bytes = 0;
  uint64_t exch_base = 0;
  double transfer_in_s = 0;
  uint32_t pending = 0;  // solves of the last enqueued launch (0: nothing pending)
  std::vector<uint64_t> last_sources;  // of the last enqueue (AUTO reruns a bailed bucket solve)
  uint32_t queued = 0;   // launches enqueued since the last finish
  uint64_t matrix_bytes = 0;
  uint64_t upload_bytes = 0;  // host->device bytes of the graph upload (stats)
  // host-driven NCCL comparison path (nccl_kernel.cuh): per-position state
  uint32_t* nc_dist = nullptr;
  uint32_t* nc_pred = nullptr;
  uint8_t* nc_vis = nullptr;
};

namespace {

sssp_options default_options(const sssp_options* o) {
  sssp_options d{};
  if (o) d = *o;
  else d.flags = SSSP_FLAGS_DEFAULT;
  if (d.timeout_ms == 0) d.timeout_ms = 60000;
  if (!o) d.global_min_weight = -1;
  return d;
}

// Grid engine: EPL/G for a shard of loc_n columns with at most gmax CTAs.
int plan_layout(Shard& s, uint64_t loc_n, uint32_t gmax) {
  static const uint32_t epls[] = {4, 8, 16, 32, 64};
  for (uint32_t epl : epls) {
    const uint64_t L = 32ull * epl;
    const uint64_t G = (loc_n + L - 1) / L;
    if (G <= gmax || epl == 64) {
      if (G > gmax) return fail(SSSP_ERR_UNSUPPORTED, "graph too large for one shard");
      s.EPL = epl;
      s.L = (uint32_t)L;
      s.G = (uint32_t)std::max<uint64_t>(1, G);
      s.C = s.G;
      s.NW = 1;
      s.row_stride = (uint64_t)s.G * s.L;
      return SSSP_OK;
    }
  }
  return SSSP_ERR_UNSUPPORTED;
}

// Cluster engine: C CTAs (<= cmax) of NW warps, EPL columns per lane; the
// smallest EPL whose cluster of at most cmax CTAs covers loc_n.
int plan_cluster_layout(Shard& s, uint64_t loc_n, uint32_t cmax, uint32_t nw) {
  static const uint32_t epls[] = {4, 8, 16, 32};
  for (uint32_t epl : epls) {
    const uint64_t per_cta = (uint64_t)nw * 32 * epl;
    uint64_t C = std::max<uint64_t>(1, (loc_n + per_cta - 1) / per_cta);
    while (C & (C - 1)) ++C;  // participants Q = C*NW must be a power of two
    if (C <= cmax) {
      s.EPL = epl;
      s.L = 32 * epl;
      s.NW = nw;
      s.C = (uint32_t)C;
      s.G = s.C * nw;
      s.row_stride = (uint64_t)s.G * s.L;
      return SSSP_OK;
    }
  }
  return fail(SSSP_ERR_UNSUPPORTED, "graph too large for one cluster; use more shards or the grid engine");
}

// Process-wide pinned staging buffers for uploads (two, double-buffered).
struct PinnedStaging {
  std::mutex m;
  void* buf[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  void* get(int b, size_t bytes) {
    if (cap[b] < bytes) {
      if (buf[b]) cudaFreeHost(buf[b]);
      buf[b] = nullptr;
      cap[b] = 0;
      if (cudaHostAlloc(&buf[b], bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
      cap[b] = bytes;
    }
    return buf[b];
  }
};
PinnedStaging g_staging;
std::mutex g_pinned_m;
std::multimap<size_t, void*> g_pinned;  // cached small pinned blocks (pinned_get)

int pool_alloc(struct Shard& s, void** p, size_t bytes);

struct ScanResult {
  std::atomic<bool> overflow{false};
  uint64_t max_w = 0, min_w = ~0ull;
};

// Narrows the caller's uint64 block (rows 0..n-1, `cols` columns, leading
// dimension ld, global column offset col_base) to W and uploads it in the
// permuted layout.  Sets res.overflow if some finite weight exceeds W's
// finite range (the caller then retries with a wider W).
template <typename W>
int upload_block(Shard& s, const uint64_t* src, uint64_t ld, uint64_t n, ScanResult& res) {
  double t_narrow = 0, t_wait = 0;
  const double t_all = now_s();
  const uint64_t WINF64 = WInf<W>::v;
  const uint64_t fmax = WINF64 - 1;  // largest finite weight W can carry
  const uint64_t cols = s.cols;
  const uint64_t row_in_bytes = std::max<uint64_t>(1, cols) * 8;
  const uint64_t R = std::max<uint64_t>(1, std::min<uint64_t>(n, (32ull << 20) / row_in_bytes));
  const uint64_t stage_elems = R * std::max<uint64_t>(1, cols);
  // pinned staging is process-wide and grow-only (pinning / unpinning on every
  // graph creation measured 0.2-0.8 s of jitter); device staging comes from the
  // stream-ordered pool (no cudaFree device synchronisation)
  std::lock_guard<std::mutex> staging_lock(g_staging.m);
  W* pin[2] = {nullptr, nullptr};
  W* dst[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  int rc = SSSP_OK;

  auto cleanup = [&]() {
    cudaStreamSynchronize(s.stream);
    for (int b = 0; b < 2; ++b) {
      if (dst[b]) cudaFreeAsync(dst[b], s.stream);
      if (done[b]) cudaEventDestroy(done[b]);
    }
  };
  for (int b = 0; b < 2; ++b) {
    void* d = nullptr;
    if (!(pin[b] = static_cast<W*>(g_staging.get(b, stage_elems * sizeof(W)))) ||
        pool_alloc(s, &d, stage_elems * sizeof(W)) != SSSP_OK ||
        cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) {
      dst[b] = static_cast<W*>(d);
      cleanup();
      return fail(SSSP_ERR_OOM, "upload staging allocation failed");
    }
    dst[b] = static_cast<W*>(d);
  }
  uint64_t chunk = 0;
  for (uint64_t r0 = 0; r0 < n && rc == SSSP_OK; r0 += R, ++chunk) {
    const int b = (int)(chunk & 1);
    const uint64_t rows = std::min<uint64_t>(R, n - r0);
    const double tw0 = now_s();
    if (used[b]) cudaEventSynchronize(done[b]);
    t_wait += now_s() - tw0;
    W* out = pin[b];
    const double tn0 = now_s();
    const NarrowStats ns = narrow_rows<W>(src, ld, r0, rows, cols, s.col_base, out);
    t_narrow += now_s() - tn0;
    res.max_w = std::max(res.max_w, ns.max_w);
    res.min_w = std::min(res.min_w, ns.min_w);
    if (ns.overflow) res.overflow = true;
    if (res.overflow) break;
    if (cols) {
      cudaError_t e = cudaMemcpyAsync(dst[b], out, rows * cols * sizeof(W),
                                      cudaMemcpyHostToDevice, s.stream);
      if (e != cudaSuccess) {
        rc = fail(SSSP_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e));
        break;
      }
    }
    const uint64_t total = rows * s.row_stride;
    const unsigned blocks = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    permute_rows_kernel<W><<<blocks, 256, 0, s.stream>>>(dst[b], (uint32_t)cols,
                                                        static_cast<W*>(s.d_adj), s.row_stride,
                                                        r0, (uint32_t)rows, s.G, s.L);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      rc = fail(SSSP_ERR_CUDA, std::string("permute launch: ") + cudaGetErrorString(e));
      break;
    }
    cudaEventRecord(done[b], s.stream);
    used[b] = true;
  }
  cleanup();
  if (rc == SSSP_OK) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(SSSP_ERR_CUDA, cudaGetErrorString(e));
  }
  if (getenv("SSSP_UPLOAD_TRACE"))
    fprintf(stderr, "upload: total %.1f ms, host narrow %.1f ms, waiting on device %.1f ms\n",
            (now_s() - t_all) * 1e3, t_narrow * 1e3, t_wait * 1e3);
  return rc;
}

// Matrices come from the device's stream-ordered pool with an unbounded
// release threshold, so re-creating a graph of the same size (every drop-in
// dijkstra(G, s) call) reuses the memory instead of cudaMalloc/cudaFree.
int pool_alloc(Shard& s, void** p, size_t bytes) {
  static bool configured[64] = {};
  if (s.device >= 0 && s.device < 64 && !configured[s.device]) {
    cudaMemPool_t mp;
    CK(cudaDeviceGetDefaultMemPool(&mp, s.device));
    uint64_t thr = ~0ull;
    CK(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
    configured[s.device] = true;
  }
  CK(cudaMallocAsync(p, bytes, s.stream));
  return SSSP_OK;
}

void pool_free(Shard& s, void* p) {
  if (p) cudaFreeAsync(p, s.stream);
}

int alloc_matrix(Shard& s, uint64_t n, uint32_t wbytes) {
  if (s.d_adj) {
    pool_free(s, s.d_adj);
    s.d_adj = nullptr;
  }
  return pool_alloc(s, &s.d_adj, n * s.row_stride * wbytes);
}

// Uploads with the narrowest encoding that holds every finite weight.
int upload_shard(Shard& s, const uint64_t* src, uint64_t ld, uint64_t n, uint64_t hint_max_w,
                 uint32_t* wbytes_out, uint64_t* max_w, uint64_t* min_w) {
  CK(cudaSetDevice(s.device));
  uint32_t wb = hint_max_w == 0 ? 1 : hint_max_w <= 0xFEull ? 1 : hint_max_w <= 0xFFFEull ? 2
               : hint_max_w <= 0xFFFFFFFEull ? 4 : 8;
  while (true) {
    int rc = alloc_matrix(s, n, wb);
    if (rc) return rc;
    ScanResult res;
    rc = wb == 1 ? upload_block<uint8_t>(s, src, ld, n, res)
         : wb == 2 ? upload_block<uint16_t>(s, src, ld, n, res)
         : wb == 4 ? upload_block<uint32_t>(s, src, ld, n, res)
                   : upload_block<uint64_t>(s, src, ld, n, res);  // a weight of 2^32-1: wide
    if (rc) return rc;
    if (!res.overflow) {
      *wbytes_out = wb;
      *max_w = res.max_w;
      *min_w = res.min_w;
      return SSSP_OK;
    }
    if (wb == 8) return fail(SSSP_ERR_WEIGHT_RANGE, "weight outside uint64");  // unreachable
    wb *= 2;
  }
}

// Small pinned host blocks (launch sources, solve info) cached process-wide:
// cudaHostAlloc / cudaFreeHost per graph cost milliseconds, sometimes hundreds.
void* pinned_get(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_pinned_m);
  auto it = g_pinned.find(bytes);
  if (it != g_pinned.end()) {
    void* p = it->second;
    g_pinned.erase(it);
    return p;
  }
  void* p = nullptr;
  return cudaHostAlloc(&p, bytes, cudaHostAllocDefault) == cudaSuccess ? p : nullptr;
}
void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_m);
  g_pinned.emplace(bytes, p);
}

// Per-graph device state comes from the stream-ordered pool (cached across
// graphs: cudaMalloc / cudaFree per graph cost 10-500 ms on the box), except
// the exchange region of a one-process-per-GPU shard, which is exported by
// CUDA IPC and so needs a plain cudaMalloc.
int alloc_state(sssp_graph* g, Shard& s) {
  CK(cudaSetDevice(s.device));
  const uint64_t B = g->max_batch;
  g->slots_bytes = (B * g->slot_stride * sizeof(uint64_t) + 255) & ~255ull;
  const uint64_t bytes =
      g->slots_bytes + (g->bucket ? g->region_bytes * std::max(g->bslots, g->bslots_b) + 256 : 0);
  s.slots_pooled = !g->multiproc;
  if (s.slots_pooled) {
    if (pool_alloc(s, (void**)&s.d_slots, bytes)) return SSSP_ERR_OOM;
  } else {
    CK(cudaMalloc(&s.d_slots, bytes));
  }
  CK(cudaMemsetAsync(s.d_slots, 0, bytes, s.stream));
  void** bufs[] = {(void**)&s.d_info2, (void**)&s.d_dist, (void**)&s.d_pred, (void**)&s.d_info,
                   (void**)&s.d_sources};
  const uint64_t cols = std::max<uint64_t>(1, s.loc_n);
  const uint64_t sizes[] = {B * 2 * sizeof(uint64_t), B * cols * sizeof(uint64_t),
                            B * cols * sizeof(uint64_t), B * 4 * sizeof(uint64_t), B * sizeof(uint32_t)};
  for (int i = 0; i < 5; ++i)
    if (pool_alloc(s, bufs[i], sizes[i])) return SSSP_ERR_OOM;
  CK(cudaMemsetAsync(s.d_info2, 0, B * 2 * sizeof(uint64_t), s.stream));
  if (g->bucket) {
    g->ctab = std::max(g->bG, g->bGb);
    if (pool_alloc(s, (void**)&s.d_ctab, B * g->ctab * sizeof(uint64_t))) return SSSP_ERR_OOM;
    CK(cudaMemsetAsync(s.d_ctab, 0, B * g->ctab * sizeof(uint64_t), s.stream));
  }
  s.h_sources = static_cast<uint32_t*>(pinned_get(B * sizeof(uint32_t)));
  s.h_info = static_cast<uint64_t*>(pinned_get(B * 4 * sizeof(uint64_t)));
  if (!s.h_sources || !s.h_info) return fail(SSSP_ERR_OOM, "pinned host allocation failed");
  if (g->opt.record_visit_order && s.k == 0)
    if (pool_alloc(s, (void**)&s.d_visit, B * g->n * sizeof(uint32_t))) return SSSP_ERR_OOM;
  if (g->opt.record_round_times && s.k == 0) {
    if (pool_alloc(s, (void**)&s.d_round_ns, g->n * sizeof(uint64_t))) return SSSP_ERR_OOM;
    CK(cudaMemsetAsync(s.d_round_ns, 0, g->n * sizeof(uint64_t), s.stream));
  }
  CK(cudaStreamSynchronize(s.stream));
  return SSSP_OK;
}

// Shards of this process on `device` (they share one launch).
uint32_t shards_on_device(const sssp_graph* g, int device) {
  uint32_t c = 0;
  for (const auto& t : g->sh) c += t.device == device ? 1u : 0u;
  return c;
}

// Encoding-dependent constants shared by every shard; requires max_w.
int finalize_encoding(sssp_graph* g) {
  const uint64_t n = g->n;
  const Shard& s0 = g->sh[0];
  // u32 distances need every candidate du + w <= n*max_w below INF; otherwise
  // (or with a weight of exactly 2^32-1, which only uint64 storage keeps apart
  // from INF) the solve runs on 64-bit distances (wide_kernel.cuh).
  g->wide = g->wbytes == 8 || (g->max_w != 0 && n > 0xFFFFFFFEull / g->max_w);
  if (g->wide) {
    if (g->P > 1 || g->multiproc)
      return fail(SSSP_ERR_UNSUPPORTED, "64-bit distances run on one shard (the result does not depend on p)");
    if (!g->cluster || g->opt.engine == SSSP_ENGINE_BUCKET)
      return fail(SSSP_ERR_UNSUPPORTED, "64-bit distances run on the wide n-round engine (engine AUTO or CLUSTER)");
    g->wPC = (uint32_t)(s0.row_stride / s0.C);
    if (wide_smem_bytes(g->wPC) > 200 * 1024)
      return fail(SSSP_ERR_UNSUPPORTED, "graph too large for the 64-bit distance engine");
    return SSSP_OK;
  }
  g->sbits = bitlen(s0.L) - 1;
  const uint64_t dmax = n * g->max_w;
  g->packed = (dmax + 1) < (1ull << (32 - g->sbits)) ? 1u : 0u;
  const uint64_t total_cols = (uint64_t)g->P * s0.loc_n;
  g->vbits = std::max<uint32_t>(1, bitlen(total_cols));
  if (g->vbits > 29) return fail(SSSP_ERR_UNSUPPORTED, "vertex count exceeds the 29-bit key field");
  if (g->cluster) {
    // exchange lives in shared memory; global memory holds only the P-slot
    // cross-shard mailbox [2][bstride] per solve
    g->bstride = ((uint64_t)g->P + 15) & ~15ull;
    g->nrep = 1;
    g->slot_stride = 2ull * g->bstride;
    for (auto& s : g->sh) {
      s.NP = s.NW / 4;
      s.hier = g->packed && (g->opt.flags & kFlagHier) && s.C <= 16;
      const bool ms = shards_on_device(g, s.device) > 1;
      s.fn = s.hier ? get_cluster_hier_kernel((int)g->wbytes, (int)s.EPL, (int)s.NW, ms)
                    : get_cluster_kernel((int)g->wbytes, (int)s.EPL, (int)s.NW, g->packed != 0,
                                         g->opt.record_round_times != 0, ms);
      if (!s.fn) return fail(SSSP_ERR_UNSUPPORTED, "no cluster kernel instance for this layout");
    }
    return SSSP_OK;
  }
  g->bstride = ((uint64_t)g->P * s0.G + 15) & ~15ull;
  uint32_t rep = g->opt.replicas ? g->opt.replicas : 1u;
  rep = std::max<uint32_t>(1, std::min<uint32_t>(rep, s0.G));
  while ((uint64_t)rep * g->P > 64) rep = std::max<uint32_t>(1, rep / 2);
  g->nrep = rep;
  g->slot_stride = 2ull * g->nrep * g->bstride;
  const uint64_t nslot = (uint64_t)g->P * s0.G;
  const uint32_t np = nslot <= 128 ? 2 : nslot <= 256 ? 4 : nslot <= 1024 ? 16 : 0;
  if (!np) return fail(SSSP_ERR_UNSUPPORTED, "too many exchange participants");
  for (auto& s : g->sh) {
    s.NP = np;
    s.fn = get_grid_kernel((int)g->wbytes, (int)s.EPL, (int)np, shards_on_device(g, s.device) > 1);
    if (!s.fn) return fail(SSSP_ERR_UNSUPPORTED, "no kernel instance for this layout");
  }
  return SSSP_OK;
}

// Concurrent solves one launch may hold while keeping every CTA resident
// (the persistent kernel spins, so all CTAs must be co-resident).
// Raises (never lowers) a kernel's dynamic shared-memory limit on the current
// device.  The limit is per function and process-wide: lowering it for one
// graph would break launches of another graph that needs more
// (tests/test_gpu_parity.py::test_interleaved_graphs_of_different_sizes).
cudaError_t raise_smem(const void* fn, size_t bytes) {
  static std::mutex m;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(m);
  size_t& c = cur[{dev, fn}];
  if (bytes <= c) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) c = bytes;
  return e;
}

void* wide_fn(uint32_t wbytes) {
  return wbytes == 1 ? (void*)wide_kernel<uint8_t>
         : wbytes == 2 ? (void*)wide_kernel<uint16_t>
         : wbytes == 4 ? (void*)wide_kernel<uint32_t> : (void*)wide_kernel<uint64_t>;
}

int compute_max_batch(sssp_graph* g) {
  if (g->wide) {  // independent clusters: no co-residency needed
    const Shard& s = g->sh[0];
    CK(cudaSetDevice(s.device));
    void* fn = wide_fn(g->wbytes);
    if (s.C > 8) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(raise_smem(fn, wide_smem_bytes(g->wPC)));
    g->max_batch = g->opt.max_batch ? g->opt.max_batch : 64;
    return SSSP_OK;
  }
  uint32_t cap = ~0u;
  for (auto& s : g->sh) {
    CK(cudaSetDevice(s.device));
    uint32_t same = 0;
    for (auto& t : g->sh) same += (t.device == s.device) ? 1 : 0;
    if (g->cluster) {
      if (s.C > 8) CK(cudaFuncSetAttribute(s.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg{};
      const size_t dsm = (size_t)s.NW * s.L * 4;
      CK(raise_smem((const void*)s.fn, dsm));
      cfg.gridDim = dim3(s.C);
      cfg.blockDim = dim3(s.NW * 32);
      cfg.dynamicSmemBytes = dsm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = s.C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int clusters = 0;
      CK(cudaOccupancyMaxActiveClusters(&clusters, (void*)s.fn, &cfg));
      if (clusters < 1) return fail(SSSP_ERR_UNSUPPORTED, "cluster shape not schedulable");
      // Independent single-shard solves need no co-residency (clusters never
      // wait on each other).  Shards of one solve do: keep every launch resident.
      if (g->P > 1) {
        if ((uint32_t)clusters < same) return fail(SSSP_ERR_UNSUPPORTED, "shards do not fit co-resident");
        cap = std::min<uint32_t>(cap, (uint32_t)clusters / same);
      }
      continue;
    }
    int per_sm = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, s.fn, 32, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
    const uint64_t blocks = (uint64_t)per_sm * sms;
    const uint64_t need = (uint64_t)s.G * same;
    if (need > blocks) return fail(SSSP_ERR_UNSUPPORTED, "shards do not fit co-resident");
    cap = std::min<uint32_t>(cap, (uint32_t)(blocks / need));
  }
  uint32_t want = g->opt.max_batch ? g->opt.max_batch : 64;
  g->max_batch = std::max<uint32_t>(1, std::min(cap, want));
  return SSSP_OK;
}

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = getenv(name);
  return e && *e ? strtoull(e, nullptr, 10) : dflt;
}

// multi: several solves share the launch; one: a single shard (nshards == 1)
void* bucket_fn(uint32_t wbytes, bool multi = false, bool one = true, bool sparse = false) {
  (void)one;  // no one-shard instance (kernels_bucket_u8.cu)
  const int v = multi ? 1 : sparse && wbytes <= 2 ? 3 : 2;
  return wbytes == 1 ? sssp_b200::bucket_fn_u8(v) : wbytes == 2 ? sssp_b200::bucket_fn_u16(v)
                                                   : sssp_b200::bucket_fn_u32(v);
}

size_t bucket_smem(const sssp_graph* g, bool batch_tiles = false) {
  const uint64_t rs = g->sh[0].row_stride;
  return batch_tiles ? bucket_smem_bytes(g->bTb, g->bGb * g->P, (uint32_t)(rs / 32 * g->P), g->wbytes)
                     : bucket_smem_bytes(g->bT, g->bG * g->P, (uint32_t)(rs / 32 * g->P), g->wbytes);
}

// The distance-class engine is exact iff every finite off-diagonal weight is
// >= 1 (bucket_kernel.cuh); it needs the cluster layout (power-of-two
// participant count) and no visit-order recording.  Chooses the tile T (128 B
// of each row per CTA, widened until every shard's grid is co-resident) and
// the exchange-region layout; allocation happens in alloc_state.
int plan_bucket(sssp_graph* g) {
  g->bucket = false;
  const int want = g->opt.engine;
  if (want == SSSP_ENGINE_GRID || want == SSSP_ENGINE_CLUSTER) return SSSP_OK;
  const bool exact = g->min_w >= 1 && !g->wide;
  const Shard& s0 = g->sh[0];
  const bool shape = g->cluster && g->n > 1 && !g->opt.record_visit_order &&
                     !g->opt.record_round_times &&
                     !(s0.G & (s0.G - 1)) && !(s0.L & (s0.L - 1));
  if (want == SSSP_ENGINE_BUCKET && !(exact && shape))
    return fail(SSSP_ERR_UNSUPPORTED, exact ? "bucket engine needs the cluster layout"
                                            : "bucket engine needs min weight >= 1");
  if (!(exact && shape)) return SSSP_OK;
  void* fn = bucket_fn(g->wbytes, false, g->P == 1);
  uint32_t T = 128 / g->wbytes;
  if (const char* e = getenv("SSSP_BUCKET_TILE_BYTES"))  // tuning experiments: bytes of each row per CTA
    T = std::max<uint32_t>(32, (uint32_t)atoi(e) / g->wbytes);
  while (true) {
    if (T > s0.row_stride) T = (uint32_t)s0.row_stride;
    g->bT = T;
    g->bG = (uint32_t)(s0.row_stride / T);
    const size_t smem = bucket_smem(g);
    bool fits = T * g->wbytes / 16 <= kBucketThreads && smem <= 200 * 1024 &&
                (uint64_t)g->bG * g->P <= 4ull * kBucketThreads;  // kernel: 4 tiles per thread
    uint64_t capacity = 0;  // co-resident CTAs of this kernel on one device
    for (const auto& s : g->sh) {
      if (!fits) break;
      CK(cudaSetDevice(s.device));
      CK(raise_smem(fn, smem));
      CK(raise_smem(bucket_fn(g->wbytes, true), smem));
      CK(raise_smem(bucket_fn(g->wbytes, false, false), smem));
      if (g->wbytes <= 2) CK(raise_smem(bucket_fn(g->wbytes, false, false, true), smem));
      uint32_t same = 0;
      for (const auto& t : g->sh) same += t.device == s.device ? 1 : 0;
      int per_sm = 0, sms = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBucketThreads, smem));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
      fits = per_sm > 0 && (uint64_t)g->bG * same <= (uint64_t)per_sm * sms;
      capacity = (uint64_t)per_sm * sms;
    }
    if (fits) {
      // batches on one shard: as many independent solves per launch as fit
      // co-resident (config 5: n=16384 -> 128 CTAs per solve, 2 per launch)
      g->bslots = g->P == 1 ? (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(
                                  {capacity / g->bG, (uint64_t)kBucketMaxSlots, g->max_batch}))
                            : 1u;
      // Batch tiling: 4x wider tiles (<= 512 B of each row per CTA) give 4x
      // fewer CTAs per solve and so more concurrent solves per launch; slower
      // per solve, faster per batch (config 5: 2.6 -> 1.75 ms for 64 sources,
      // profiles/r01_bucket_tile_sweep.txt).  Same exchange-region layout
      // (sized for the larger single-solve grid).
      g->bslots_b = 0;
      if (g->P == 1 && g->max_batch > g->bslots) {
        const uint32_t Tb = std::min<uint32_t>(std::min<uint32_t>(T * 4, 512 / g->wbytes),
                                               (uint32_t)s0.row_stride);
        g->bTb = Tb;
        g->bGb = (uint32_t)(s0.row_stride / Tb);
        const size_t smb = bucket_smem(g, true);
        int per_sm = 0;
        void* fm = bucket_fn(g->wbytes, true);
        CK(raise_smem(fm, std::max(smem, smb)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fm, kBucketThreads, smb));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s0.device));
        const uint64_t slots = std::min<uint64_t>(
            {(uint64_t)per_sm * sms / g->bGb, (uint64_t)kBucketMaxSlots, g->max_batch});
        if (Tb > T && Tb * g->wbytes / 16 <= kBucketThreads && smb <= 200 * 1024 && slots > g->bslots)
          g->bslots_b = (uint32_t)slots;
      }
      break;
    }
    if (T * g->wbytes >= 1024 || T >= s0.row_stride) {  // pull: (T + 2) keys + ids fit the combine region
      if (want == SSSP_ENGINE_BUCKET) return fail(SSSP_ERR_UNSUPPORTED, "bucket grid does not fit");
      return SSSP_OK;  // AUTO: stay on the scan engine
    }
    T *= 2;
  }
  // exchange region: [barrier counter | epoch | ctrl [2][4][P*G] | bitmap [2][P*row_stride/32]
  //                   | local: unsettled bitmap [2][row_stride/32] | pull keys [row_stride] u64]
  const uint64_t GT = (uint64_t)g->bG * g->P;
  const uint64_t words = s0.row_stride / 32 * g->P;
  g->bar_off = 0;
  g->arrive_off = 64;
  g->epoch_off = 128;
  g->release_off = 192;
  g->ctrl_off = 256;
  g->bm_off = (g->ctrl_off + 2 * 4 * GT * 4 + 255) & ~255ull;
  g->ubm_off = (g->bm_off + 2 * words * 4 + 255) & ~255ull;
  g->pkey_off = (g->ubm_off + 2 * (s0.row_stride / 32) * 4 + 255) & ~255ull;
  g->region_bytes = (g->pkey_off + s0.row_stride * 8 + 255) & ~255ull;
  g->done_off = g->region_bytes * std::max(g->bslots, g->bslots_b);  // [kBucketMaxSlots] u32 after
  g->bucket = true;
  return SSSP_OK;
}

// Builds the PULL source of every local shard.  One shard: the matrix itself
// when symmetric (row v = column v), else its transpose in position order.
// Several shards: AT_k[p][g] = A_k[vertex(g)][p] over global positions g
// (a shard holds every row of its columns, so a column is local but strided).
int prepare_bucket_impl(sssp_graph* g);
int prepare_bucket(sssp_graph* g) {
  const double t0 = now_s();
  const int rc = prepare_bucket_impl(g);
  if (getenv("SSSP_UPLOAD_TRACE")) fprintf(stderr, "prepare_bucket: %.1f ms\n", (now_s() - t0) * 1e3);
  return rc;
}
int prepare_bucket_impl(sssp_graph* g) {
  if (!g->bucket) return SSSP_OK;
  for (auto& s : g->sh) {
    CK(cudaSetDevice(s.device));
    const uint32_t Q = s.G, L = s.L, qb = bitlen(Q) - 1, lb = bitlen(L) - 1;
    const uint64_t rs = s.row_stride;
    s.pull_src = nullptr;
    if (g->P == 1) {  // class-1 row summaries: one CTA per row, once per upload
      if (!s.d_rsum && pool_alloc(s, (void**)&s.d_rsum, g->n * 2 * sizeof(uint4)) != SSSP_OK) return SSSP_ERR_OOM;
      const uint32_t fb0 = (uint32_t)std::min<uint64_t>(1 + g->min_w, 0xFFFFFFFEull);
      const unsigned nb = (unsigned)g->n;
      if (g->wbytes == 1)
        row_summary_kernel<uint8_t><<<nb, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, fb0, s.d_rsum);
      else if (g->wbytes == 2)
        row_summary_kernel<uint16_t><<<nb, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, fb0, s.d_rsum);
      else
        row_summary_kernel<uint32_t><<<nb, 256, 0, s.stream>>>((const uint32_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, fb0, s.d_rsum);
      CK(cudaGetLastError());
      // class-1 id lists: rows whose class 1 fits one push pass, within a
      // memory budget (a quarter of the matrix); the rest scan their row
      std::vector<uint4> hs(2 * g->n);
      CK(cudaMemcpyAsync(hs.data(), s.d_rsum, hs.size() * sizeof(uint4), cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      uint64_t total = 0;
      const uint64_t budget = std::max<uint64_t>(1ull << 20, g->n * rs * g->wbytes / 4) / 4;
      for (uint64_t u = 0; u < g->n; ++u) {
        const uint4 r = hs[2 * u];
        const bool listed = r.x != 0xFFFFFFFFu && r.y > 0 && r.y <= kIdCap && total + r.y <= budget;
        hs[2 * u + 1] = make_uint4(listed ? (uint32_t)total : 0xFFFFFFFFu, 0, 0, 0);
        if (listed) total += r.y;
      }
      CK(cudaMemcpyAsync(s.d_rsum, hs.data(), hs.size() * sizeof(uint4), cudaMemcpyHostToDevice, s.stream));
      if (s.d_rlist) pool_free(s, s.d_rlist);
      s.d_rlist = nullptr;
      if (total && pool_alloc(s, (void**)&s.d_rlist, total * sizeof(uint32_t)) != SSSP_OK) return SSSP_ERR_OOM;
      if (total) {
        const uint32_t* rsw = reinterpret_cast<const uint32_t*>(s.d_rsum);
        if (g->wbytes == 1)
          row_list_kernel<uint8_t><<<nb, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, rsw, s.d_rlist);
        else if (g->wbytes == 2)
          row_list_kernel<uint16_t><<<nb, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, rsw, s.d_rlist);
        else
          row_list_kernel<uint32_t><<<nb, 256, 0, s.stream>>>((const uint32_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, rsw, s.d_rlist);
        CK(cudaGetLastError());
      }
      // Sparse tile lists: when the finite entries take at most 1/8 of the
      // matrix bytes as 4 B list entries, the push reads each class row's
      // entries in its tile instead of the dense 128 B slice (config 4:
      // 0.1 % density -> ~0.13 entries per row and tile).  u8/u16 only (the
      // entry packs w in 16 bits).
      uint64_t finite = 0;
      for (uint64_t u = 0; u < g->n; ++u) finite += hs[2 * u].w;
      pool_free(s, s.d_spoff);
      pool_free(s, s.d_spent);
      s.d_spoff = s.d_spent = nullptr;
      s.sp_T = 0;
      const uint32_t T = g->bT, G = g->bG;
      static const bool k_sparse = env_u64("SSSP_BUCKET_SPARSE", 1) != 0;  // A/B: dense push
      if (k_sparse && g->wbytes <= 2 && G <= 1024 && rs <= (g->wbytes == 1 ? (1ull << 24) : (1ull << 16)) &&
          finite * 4 * 8 <= g->n * rs * g->wbytes &&
          (uint64_t)G * g->n + 1 < (1ull << 31)) {
        const double tl0 = now_s();
        const size_t ncnt = (size_t)G * g->n + 1;
        uint32_t* d_cnt = nullptr;
        if (pool_alloc(s, (void**)&d_cnt, ncnt * 4) != SSSP_OK ||
            pool_alloc(s, (void**)&s.d_spoff, ncnt * 4) != SSSP_OK)
          return SSSP_ERR_OOM;
        if (g->wbytes == 1)
          tile_list_kernel<uint8_t, false><<<nb, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, T, G, d_cnt, nullptr);
        else
          tile_list_kernel<uint16_t, false><<<nb, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, T, G, d_cnt, nullptr);
        CK(cudaGetLastError());
        size_t tmp_bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt, s.d_spoff, (int)ncnt, s.stream));
        void* d_tmp = nullptr;
        if (pool_alloc(s, &d_tmp, std::max<size_t>(tmp_bytes, 16)) != SSSP_OK) return SSSP_ERR_OOM;
        CK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_cnt, s.d_spoff, (int)ncnt, s.stream));
        pool_free(s, d_tmp);
        pool_free(s, d_cnt);
        // the list total = the terminator's offset (its count is 0)
        uint32_t total_ent = 0;
        CK(cudaMemcpyAsync(&total_ent, s.d_spoff + ncnt - 1, 4, cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        if (pool_alloc(s, (void**)&s.d_spent, std::max<uint64_t>(total_ent, 1) * 4) != SSSP_OK) return SSSP_ERR_OOM;
        if (g->wbytes == 1)
          tile_list_kernel<uint8_t, true><<<nb, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, T, G, s.d_spoff, s.d_spent);
        else
          tile_list_kernel<uint16_t, true><<<nb, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, T, G, s.d_spoff, s.d_spent);
        CK(cudaGetLastError());
        s.sp_T = T;
        if (getenv("SSSP_UPLOAD_TRACE")) {
          CK(cudaStreamSynchronize(s.stream));
          fprintf(stderr, "tile lists: %u entries, %u tiles, %.2f ms\n", total_ent, G, (now_s() - tl0) * 1e3);
        }
      }
      CK(cudaStreamSynchronize(s.stream));  // hs is freed on return
    }
    // sparse tile lists: every step pushes, so no pull source (symmetry check,
    // transpose) is needed
    if (s.d_spoff) continue;
    if (rs % 64) continue;
    const uint64_t mbytes = g->n * rs * g->wbytes;
    if (g->P == 1) {
      uint32_t* d_flag = nullptr;
      CK(cudaMallocAsync((void**)&d_flag, 4, s.stream));
      CK(cudaMemsetAsync(d_flag, 0, 4, s.stream));
      const uint64_t tl = 128 / g->wbytes;  // 128 B row segments (symmetric_check_wide_kernel)
      const dim3 gridw((unsigned)(rs / tl), (unsigned)(rs / tl));
      const dim3 grid((unsigned)(rs / 64), (unsigned)(rs / 64));
      if (rs % tl == 0) {
        if (g->wbytes == 1)
          symmetric_check_wide_kernel<uint8_t><<<gridw, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
        else if (g->wbytes == 2)
          symmetric_check_wide_kernel<uint16_t><<<gridw, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
        else
          symmetric_check_wide_kernel<uint32_t><<<gridw, 256, 0, s.stream>>>((const uint32_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
      } else if (g->wbytes == 1)
        symmetric_check_kernel<uint8_t><<<grid, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
      else if (g->wbytes == 2)
        symmetric_check_kernel<uint16_t><<<grid, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
      else
        symmetric_check_kernel<uint32_t><<<grid, 256, 0, s.stream>>>((const uint32_t*)s.d_adj, rs, (uint32_t)g->n, Q, qb, lb, d_flag);
      CK(cudaGetLastError());
      uint32_t asym = 1;
      CK(cudaMemcpyAsync(&asym, d_flag, 4, cudaMemcpyDeviceToHost, s.stream));
      CK(cudaFreeAsync(d_flag, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      if (!asym) {
        s.pull_src = s.d_adj;
        continue;
      }
    }
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t tbytes = (uint64_t)rs * rs * g->P * g->wbytes;  // loc positions x global positions
    if (tbytes + (256ull << 20) >= free_b || pool_alloc(s, &s.d_adjT, tbytes) != SSSP_OK) continue;
    const dim3 grid((unsigned)(rs / 64), (unsigned)(rs * g->P / 64));
    const uint32_t P = g->P, loc = (uint32_t)s.loc_n;
    if (g->wbytes == 1)
      transpose_global_kernel<uint8_t><<<grid, 256, 0, s.stream>>>((const uint8_t*)s.d_adj, (uint8_t*)s.d_adjT, rs, (uint32_t)g->n, Q, qb, lb, P, loc);
    else if (g->wbytes == 2)
      transpose_global_kernel<uint16_t><<<grid, 256, 0, s.stream>>>((const uint16_t*)s.d_adj, (uint16_t*)s.d_adjT, rs, (uint32_t)g->n, Q, qb, lb, P, loc);
    else
      transpose_global_kernel<uint32_t><<<grid, 256, 0, s.stream>>>((const uint32_t*)s.d_adj, (uint32_t*)s.d_adjT, rs, (uint32_t)g->n, Q, qb, lb, P, loc);
    CK(cudaGetLastError());
    s.pull_src = s.d_adjT;
    g->matrix_bytes += tbytes;
    (void)mbytes;
  }
  return SSSP_OK;
}

int setup_common(sssp_graph* g) {
  int rc = finalize_encoding(g);
  if (rc) return rc;
  rc = compute_max_batch(g);
  if (rc) return rc;
  rc = plan_bucket(g);
  if (rc) return rc;
  g->matrix_bytes = 0;
  for (auto& s : g->sh) {
    rc = alloc_state(g, s);
    if (rc) return rc;
    g->matrix_bytes += g->n * s.row_stride * g->wbytes;
  }
  return prepare_bucket(g);
}

int create_shard_objects(sssp_graph* g, uint32_t P, const int* devices, uint32_t nlocal,
                         uint32_t first_k) {
  const uint64_t padded = pad_vertex_count(g->n, P);
  const uint64_t loc_n = padded / P;
  uint32_t gmax = g->opt.ctas_per_shard;
  g->cluster = g->opt.engine != SSSP_ENGINE_GRID;
  g->sh.resize(nlocal);
  for (uint32_t i = 0; i < nlocal; ++i) {
    Shard& s = g->sh[i];
    s.device = devices[i];
    s.k = first_k + i;
    s.col_base = (uint64_t)s.k * loc_n;
    s.loc_n = loc_n;
    s.cols = s.col_base >= g->n ? 0 : std::min<uint64_t>(loc_n, g->n - s.col_base);
    int sms = 148;
    CK(cudaSetDevice(s.device));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
    int rc;
    if (g->cluster) {
      const uint32_t nw = g->opt.warps_per_cta ? g->opt.warps_per_cta : 4;
      if (nw != 4 && nw != 8 && nw != 16) return fail(SSSP_ERR_BAD_ARG, "warps_per_cta: 4, 8 or 16");
      rc = plan_cluster_layout(s, loc_n, gmax ? std::min<uint32_t>(gmax, 16) : 16, nw);
    } else {
      uint32_t gm = gmax;
      if (!gm) gm = P == 1 ? (uint32_t)sms : std::max<uint32_t>(4, std::min<uint32_t>(sms, 256 / P));
      rc = plan_layout(s, loc_n, gm);
    }
    if (rc) return rc;
    // shards on one device share one stream (and one cooperative launch)
    s.own_stream = true;
    for (uint32_t j = 0; j < i; ++j)
      if (g->sh[j].device == s.device) {
        s.stream = g->sh[j].stream;
        s.own_stream = false;
        break;
      }
    if (s.own_stream) CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s.ev0));
    CK(cudaEventCreate(&s.ev1));
  }
  return SSSP_OK;
}

void destroy_graph(sssp_graph* g) {
  if (g->nc_dist && !g->sh.empty()) {
    cudaSetDevice(g->sh[0].device);
    for (void* p : {(void*)g->nc_dist, (void*)g->nc_pred, (void*)g->nc_vis}) pool_free(g->sh[0], p);
  }
  for (auto& s : g->sh) {
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (int j = 0; j < kMaxShards; ++j)
      if (s.peer_ipc[j] && s.peer[j]) cudaIpcCloseMemHandle(s.peer[j]);
    pool_free(s, s.d_adj);
    if (s.slots_pooled) pool_free(s, s.d_slots);
    else cudaFree(s.d_slots);
    for (void* p : {(void*)s.d_dist, (void*)s.d_pred, (void*)s.d_info, (void*)s.d_sources,
                    (void*)s.d_visit, (void*)s.d_round_ns, (void*)s.d_info2, s.d_adjT, (void*)s.d_ctab,
                    (void*)s.d_rsum, (void*)s.d_rlist, (void*)s.d_spoff, (void*)s.d_spent})
      pool_free(s, p);
    if (s.stream) cudaStreamSynchronize(s.stream);
    cudaFree(s.d_trace);
    cudaFree(s.d_spans);
    const uint64_t B = g->max_batch;
    pinned_put(s.h_sources, B * sizeof(uint32_t));
    pinned_put(s.h_info, B * 4 * sizeof(uint64_t));
    if (s.ev0) cudaEventDestroy(s.ev0);
    if (s.ev1) cudaEventDestroy(s.ev1);
  }
  for (auto& s : g->sh)  // after every shard's frees were queued (shared streams)
    if (s.stream && s.own_stream) {
      cudaSetDevice(s.device);
      cudaStreamDestroy(s.stream);
    }
  delete g;
}

// Shards grouped by device, in order of first appearance: every group is ONE
// launch (shards as block ranges), so shards on one device never depend on
// CUDA co-scheduling two kernels.
std::vector<std::vector<uint32_t>> device_groups(const sssp_graph* g) {
  std::vector<std::vector<uint32_t>> groups;
  for (uint32_t a = 0; a < g->sh.size(); ++a) {
    bool placed = false;
    for (auto& gr : groups)
      if (!placed && g->sh[gr[0]].device == g->sh[a].device) {
        gr.push_back(a);
        placed = true;
      }
    if (!placed) groups.push_back({a});
  }
  return groups;
}

// Launches k solves of `fn` for every shard of a device group (cluster
// engine: k clusters of C CTAs x NW warps per shard; grid engine: k*G
// single-warp CTAs per shard).  Probe kernels pass rounds/out_ns.  Several
// shards in one launch spin on each other's mailboxes, so that launch is
// cooperative (co-residency guaranteed or the launch fails loudly).
cudaError_t launch_kernel(sssp_graph* g, const std::vector<uint32_t>& grp, void* fn, uint32_t k,
                          const std::vector<ScanParams>& ps, const uint32_t* rounds, int is_probe,
                          uint64_t* out_ns) {
  const Shard& s = g->sh[grp[0]];
  ScanLaunch la{};
  la.nlocal = (uint32_t)grp.size();
  for (uint32_t i = 0; i < la.nlocal; ++i) la.sh[i] = ps[i];
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[2];
  int na = 0;
  cfg.stream = s.stream;
  if (g->cluster) {
    la.bps = k * s.C;
    cfg.gridDim = dim3(la.bps * la.nlocal);
    cfg.blockDim = dim3(s.NW * 32);
    cfg.dynamicSmemBytes = is_probe ? 0 : (size_t)s.NW * s.L * 4;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = s.C;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  } else {
    la.bps = k * s.G;
    cfg.gridDim = dim3(la.bps * la.nlocal);
    cfg.blockDim = dim3(32);
  }
  // independent single-shard clusters never wait on each other; everything
  // else spins on other blocks of the launch
  const bool coop = !g->cluster || la.nlocal > 1;
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (is_probe) {
    uint32_t r = *rounds;
    void* args[] = {(void*)&la, (void*)&r, (void*)&out_ns};
    return cudaLaunchKernelExC(&cfg, fn, args);
  }
  void* args[] = {(void*)&la};
  return cudaLaunchKernelExC(&cfg, fn, args);
}


// Enqueues one launch of k solves on every local shard.
int launch(sssp_graph* g, const uint64_t* sources, uint32_t k) {
  if (g->multiproc && !g->connected)
    return fail(SSSP_ERR_BAD_ARG, "shard not connected: call sssp_shard_connect first");
  if (k == 0 || k > g->max_batch) return fail(SSSP_ERR_BAD_ARG, "bad batch size");
  for (uint32_t i = 0; i < k; ++i)
    if (sources[i] >= g->n) return fail(SSSP_ERR_BAD_SOURCE, "dijkstra: source out of range");
  g->last_sources.assign(sources, sources + k);
  if (g->wide) {  // k independent clusters, 64-bit distances (wide_kernel.cuh)
    Shard& s = g->sh[0];
    CK(cudaSetDevice(s.device));
    for (uint32_t i = 0; i < k; ++i) s.h_sources[i] = (uint32_t)sources[i];
    CK(cudaMemcpyAsync(s.d_sources, s.h_sources, k * sizeof(uint32_t), cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemsetAsync(s.d_info, 0, (uint64_t)k * 4 * sizeof(uint64_t), s.stream));
    WideParams wp{};
    wp.adj = s.d_adj;
    wp.row_stride = s.row_stride;
    wp.n = (uint32_t)g->n;
    wp.Q = s.G;
    wp.qbits = bitlen(s.G) - 1;
    wp.lbits = bitlen(s.L) - 1;
    wp.C = s.C;
    wp.PC = g->wPC;
    wp.sources = s.d_sources;
    wp.dist_out = s.d_dist;
    wp.pred_out = s.d_pred;
    wp.visit_order = s.d_visit;
    wp.info = s.d_info;
    if (!g->pending) CK(cudaEventRecord(s.ev0, s.stream));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = s.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(k * s.C);
    cfg.blockDim = dim3(kWideThreads);
    cfg.dynamicSmemBytes = wide_smem_bytes(g->wPC);
    cfg.stream = s.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&wp};
    CK(cudaLaunchKernelExC(&cfg, wide_fn(g->wbytes), args));
    // the end event is recorded by finish(): an event record between two
    // back-to-back launches costs ~3 us of GPU time (tools/ubench_launch2.cu)
    g->pending = k;
    g->queued += 1;
    return SSSP_OK;
  }
  if (g->bucket) {
    void* fn = bucket_fn(g->wbytes, false, g->P == 1);
    const size_t smem = bucket_smem(g);
    for (auto& s : g->sh) {
      CK(cudaSetDevice(s.device));
      if (!g->pending) CK(cudaEventRecord(s.ev0, s.stream));
    }
    const size_t smem_b = g->bslots_b ? bucket_smem(g, true) : 0;
    // shards on one device share one cooperative launch (grid = nlocal x tiles)
    const auto groups = device_groups(g);
    for (uint32_t i = 0; i < k;) {  // solves i .. i+ns-1 share a launch
      // more solves left than the single-solve grid can pair: batch tiling
      const bool wide = g->bslots_b > 0 && k - i > g->bslots;
      const uint32_t ns = std::min<uint32_t>(wide ? g->bslots_b : g->bslots, k - i);
      const uint32_t tiles = wide ? g->bGb : g->bG;
      for (const auto& gr : groups) {
        Shard& s0 = g->sh[gr[0]];
        CK(cudaSetDevice(s0.device));
        BucketParams bp{};
        bp.nslots = ns;
        for (uint32_t j = 0; j < ns; ++j) bp.slot_src[j] = (uint32_t)sources[i + j];
        bp.slot_bytes = g->region_bytes;
        bp.out_stride = s0.loc_n;
        bp.nlocal = (uint32_t)gr.size();
        for (uint32_t li = 0; li < gr.size(); ++li) {
          Shard& s = g->sh[gr[li]];
          BucketLocal& L = bp.loc[li];
          char* own = reinterpret_cast<char*>(s.d_slots) + g->slots_bytes;
          L.adj = s.d_adj;
          L.adjT = s.pull_src;
          L.ubm = reinterpret_cast<uint32_t*>(own + g->ubm_off);
          L.pkey = own + g->pkey_off;
          L.dist_out = s.d_dist + (uint64_t)i * s.loc_n;
          L.pred_out = s.d_pred + (uint64_t)i * s.loc_n;
          L.info = s.d_info + (uint64_t)i * 4;
          L.info2 = s.d_info2 + (uint64_t)i * 2;
          L.cta_bytes = s.d_ctab + (uint64_t)i * g->ctab;
          L.shard = s.k;
        }
        bp.adjT_by_pos = s0.pull_src == s0.d_adj ? 0u : 1u;  // transpose rows: local positions
        bp.adjT_stride = s0.pull_src == s0.d_adj ? s0.row_stride : s0.row_stride * g->P;
        bp.row_stride = s0.row_stride;
        bp.n = (uint32_t)g->n;
        bp.Q = s0.G;
        bp.L = s0.L;
        bp.qbits = bitlen(s0.G) - 1;
        bp.lbits = bitlen(s0.L) - 1;
        bp.T = wide ? g->bTb : g->bT;
        bp.nshards = g->P;
        bp.loc_n = (uint32_t)s0.loc_n;
        bp.wmin = (uint32_t)std::min<uint64_t>(g->min_w, 0xFFFFFFFFull);
        // AUTO picks the engine per call: a class step costs ~12 scan rounds
        // (profiles/r01_configs_1gpu.jsonl: ~5.7 us vs ~0.45 us), so a solve
        // that needs more than n/12 classes stops and reruns on the n-round
        // engine (finish()).  One process only: every shard stops together.
        bp.max_classes = g->opt.engine == SSSP_ENGINE_AUTO && !g->multiproc
                             ? (uint32_t)std::max<uint64_t>(16, g->n / 12) : 0u;
        // A/B switches (read once per process): bulk-copy push,
        // 16-deep register push, owner-pull limit (0 = balanced pulls only)
        static const uint32_t k_push_ldg = env_u64("SSSP_PUSH_BULK", 0) ? 0u : 1u;
        static const uint32_t k_depth16 = env_u64("SSSP_PUSH_DEPTH16", 0) ? 1u : 0u;
        static const uint32_t k_owner = (uint32_t)env_u64("SSSP_OWNER_PULL_COLS", 4);
        bp.push_ldg = k_push_ldg;
        bp.push_depth16 = k_depth16;
        bp.owner_cols = k_owner;
        for (uint32_t j = 0; j < g->P; ++j) {
          char* base = reinterpret_cast<char*>(g->multiproc ? (void*)s0.peer[j] : (void*)g->sh[j].d_slots) +
                       g->slots_bytes;
          bp.peer_ctrl[j] = reinterpret_cast<uint32_t*>(base + g->ctrl_off);
          bp.peer_bitmap[j] = reinterpret_cast<uint32_t*>(base + g->bm_off);
          bp.peer_bar[j] = reinterpret_cast<unsigned long long*>(base + g->bar_off);
        }
        char* own0 = reinterpret_cast<char*>(s0.d_slots) + g->slots_bytes;
        bp.bar_epoch = reinterpret_cast<uint64_t*>(own0 + g->epoch_off);
        bp.arrive = reinterpret_cast<unsigned long long*>(own0 + g->arrive_off);
        bp.release = reinterpret_cast<unsigned long long*>(own0 + g->release_off);
        bp.done = reinterpret_cast<uint32_t*>(own0 + g->done_off);
        bp.ctab_stride = g->ctab;
        bp.timeout_ns = g->opt.timeout_ms * 1000000ull;
        if (getenv("SSSP_BUCKET_TRACE") && s0.k == 0) {  // debug: per-barrier timestamps
          if (!s0.d_trace) CK(cudaMalloc(&s0.d_trace, (512 + 4096) * 8));
          CK(cudaMemsetAsync(s0.d_trace, 0, (512 + 4096) * 8, s0.stream));
          bp.trace = s0.d_trace;
        }
        bp.seq = g->bseq + 1 + i;
        if (getenv("SSSP_BUCKET_SPANS") && !s0.d_spans) {
          CK(cudaMalloc(&s0.d_spans, 128 * 8));
          CK(cudaMemset(s0.d_spans, 0, 128 * 8));
        }
        bp.spans = s0.d_spans;
        static const uint32_t k_reps = (uint32_t)std::max<uint64_t>(1, env_u64("SSSP_BUCKET_REPS", 1));
        bp.dbg_reps = k_reps;
        // exchange-free class 1 (one shard; A/B: SSSP_BUCKET_LOCAL1=0)
        static const bool k_local1 = env_u64("SSSP_BUCKET_LOCAL1", 1) != 0;
        bp.rsum = k_local1 && g->P == 1 ? reinterpret_cast<const uint32_t*>(s0.d_rsum) : nullptr;
        static const bool k_lists = env_u64("SSSP_BUCKET_LISTS", 1) != 0;  // A/B: scan row s instead
        bp.rlist = k_lists ? s0.d_rlist : nullptr;
        const bool sp = g->P == 1 && ns <= 1 && s0.d_spoff && s0.sp_T == bp.T;  // lists of this tiling (single solves)
        bp.sp_off = sp ? s0.d_spoff : nullptr;
        bp.sp_ent = sp ? s0.d_spent : nullptr;
        static const uint32_t k_split = (uint32_t)env_u64("SSSP_SPLIT_ROWS", 512);  // 0: never row-split
        bp.sp_split = k_split;
        void* args[] = {&bp};
        const uint32_t grid = tiles * (ns > 1 ? ns : bp.nlocal);
        // local shards other than the first wait for the launch on the
        // group's stream (their own streams record the completion below)
        // cooperative + programmatic stream serialisation: a solve queued
        // behind another is launched while its predecessor drains (the kernel
        // waits on griddepcontrol.wait before any memory access); A/B:
        // SSSP_BUCKET_PDL=0
        static const bool k_pdl = env_u64("SSSP_BUCKET_PDL", 1) != 0;
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute la[2];
        la[0].id = cudaLaunchAttributeCooperative;
        la[0].val.cooperative = 1;
        la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        la[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kBucketThreads);
        cfg.dynamicSmemBytes = wide ? smem_b : smem;
        cfg.stream = s0.stream;
        cfg.attrs = la;
        cfg.numAttrs = k_pdl ? 2 : 1;
        CK(cudaLaunchKernelExC(&cfg, ns > 1 ? bucket_fn(g->wbytes, true) : sp ? bucket_fn(g->wbytes, false, false, true) : fn, args));
      }
      i += ns;
    }
    for (const auto& gr : groups)  // group leaders record their end event in finish()
      for (size_t li = 1; li < gr.size(); ++li) {
        Shard& s = g->sh[gr[li]];
        CK(cudaSetDevice(s.device));
        CK(cudaEventRecord(s.ev1, s.stream));
      }
    g->bseq += k;
    g->pending = k;
    g->queued += 1;
    return SSSP_OK;
  }
  // Single process: reset the exchange buffers of every shard first, and make
  // every launch wait for all resets (a peer may publish into our buffers as
  // soon as its kernel starts).
  std::vector<cudaEvent_t> reset_ev;
  if (!g->multiproc) {
    g->exch_base = 0;
    for (auto& s : g->sh) {
      CK(cudaSetDevice(s.device));
      CK(cudaMemsetAsync(s.d_slots, 0, (uint64_t)k * g->slot_stride * sizeof(uint64_t), s.stream));
      if (g->sh.size() > 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, s.stream));
        reset_ev.push_back(e);
      }
    }
  }
  for (const auto& grp : device_groups(g)) {
    std::vector<ScanParams> ps;
    for (uint32_t li : grp) {
      Shard& s = g->sh[li];
      CK(cudaSetDevice(s.device));
      for (cudaEvent_t e : reset_ev) CK(cudaStreamWaitEvent(s.stream, e, 0));
      for (uint32_t i = 0; i < k; ++i) s.h_sources[i] = (uint32_t)sources[i];
      CK(cudaMemcpyAsync(s.d_sources, s.h_sources, k * sizeof(uint32_t), cudaMemcpyHostToDevice,
                         s.stream));
      CK(cudaMemsetAsync(s.d_info, 0, (uint64_t)k * 4 * sizeof(uint64_t), s.stream));
      ScanParams p{};
      p.adj = s.d_adj;
      p.row_stride = s.row_stride;
      p.n = (uint32_t)g->n;
      p.G = s.G;
      p.col_base = (uint32_t)s.col_base;
      p.loc_n = (uint32_t)s.loc_n;
      p.vbits = g->vbits;
      p.shard = s.k;
      p.nshards = g->P;
      p.packed = g->packed;
      p.sbits = g->sbits;
      p.flags = g->opt.flags;
      p.slots = s.d_slots;
      for (uint32_t j = 0; j < g->P && j < (uint32_t)kMaxShards; ++j)
        p.peer_slots[j] = g->multiproc ? s.peer[j] : g->sh[j].d_slots;
      p.slot_stride = g->slot_stride;
      p.bstride = (uint32_t)g->bstride;
      p.nrep = g->nrep;
      p.exch_base = g->exch_base;
      p.sources = s.d_sources;
      p.nsolve = k;
      p.dist_out = s.d_dist;
      p.pred_out = s.d_pred;
      p.visit_order = s.d_visit;
      p.round_ns = s.d_round_ns;
      p.info = s.d_info;
      p.timeout_ns = g->opt.timeout_ms * 1000000ull;
      if (!g->pending) CK(cudaEventRecord(s.ev0, s.stream));
      ps.push_back(p);
    }
    Shard& s0 = g->sh[grp[0]];
    CK(cudaSetDevice(s0.device));
    CK(launch_kernel(g, grp, (void*)s0.fn, k, ps, nullptr, 0, nullptr));
    for (size_t li = 1; li < grp.size(); ++li)  // the leader records its end event in finish()
      CK(cudaEventRecord(g->sh[grp[li]].ev1, g->sh[grp[li]].stream));
  }
  for (cudaEvent_t e : reset_ev) cudaEventDestroy(e);
  g->pending = k;
  g->queued += 1;
  return SSSP_OK;
}

// Waits for the pending launch, checks the watchdog, fills stats.
// The reference's OpCounters (serial.hpp:16-19) and the CollectiveStats of
// dijkstra_partitioned with p = shards (partitioned.hpp:196-221), as the
// reference defines them for this input, plus the upload / output bytes.
void fill_reference_stats(const sssp_graph* g, sssp_solve_stats* st) {
  const uint64_t n = g->n, p = g->P;
  const uint64_t padded = pad_vertex_count(n, p), loc_n = padded / p;
  st->extract_min_scans = n * n;
  st->ref_relax_checks = n * n;
  st->allreduce_count = padded;
  st->scatter_bytes = (p - 1) * padded * loc_n * sizeof(uint64_t);
  st->gather_bytes = (p - 1) * loc_n * (sizeof(uint64_t) + sizeof(uint64_t));
  st->upload_bytes = g->upload_bytes;
  uint64_t cols = 0;
  for (const auto& s : g->sh) cols += s.cols;
  st->download_bytes = cols * 16;
}

int finish(sssp_graph* g, sssp_solve_stats* st) {
  const uint32_t k = g->pending, nqueued = g->queued;
  if (k == 0) return fail(SSSP_ERR_BAD_ARG, "nothing enqueued");
  // end events of the launching streams (deferred by launch(): one record
  // after the last queued launch instead of one between every two launches)
  for (const auto& gr : device_groups(g)) {
    Shard& s = g->sh[gr[0]];
    CK(cudaSetDevice(s.device));
    CK(cudaEventRecord(s.ev1, s.stream));
  }
  double rounds = 0;
  uint64_t iters = 0, last = 0, mis = 0, classes = 0, rows = 0, nbars = 0, nbytes = 0;
  bool timeout = false, bailed = false;
  for (auto& s : g->sh) {
    CK(cudaSetDevice(s.device));
    CK(cudaMemcpyAsync(s.h_info, s.d_info, (uint64_t)k * 4 * sizeof(uint64_t),
                       cudaMemcpyDeviceToHost, s.stream));
    if (g->bucket) {
      uint64_t i2[2 * 64] = {};
      CK(cudaMemcpyAsync(i2, s.d_info2, std::min<uint64_t>(k, 64) * 2 * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      // launch i of the last enqueue carried tag bseq - k + 1 + i
      for (uint32_t i = 0; i < std::min<uint32_t>(k, 64); ++i) {
        timeout |= i2[2 * i + 1] == g->bseq - k + 1 + i;
        if (s.k == g->sh[0].k) nbars += i2[2 * i];
      }
      std::vector<uint64_t> cb((uint64_t)k * g->ctab);
      CK(cudaMemcpyAsync(cb.data(), s.d_ctab, cb.size() * 8, cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      for (uint64_t x : cb) nbytes += x;
    }
    CK(cudaStreamSynchronize(s.stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
    rounds = std::max(rounds, ms * 1e-3 / std::max(1u, g->queued));
    for (uint32_t i = 0; i < k; ++i) {
      if (g->bucket) {
        if (s.k == g->sh[0].k) {
          iters += s.h_info[4 * i];
          bailed |= (s.h_info[4 * i + 1] >> 63) != 0;
          classes += s.h_info[4 * i + 1] & ~(1ull << 63);
          rows += s.h_info[4 * i + 2] + s.h_info[4 * i + 3];
        }
        continue;
      }
      iters += s.k == g->sh[0].k ? s.h_info[4 * i] : 0;
      last = std::max(last, s.h_info[4 * i + 1]);
      timeout |= s.h_info[4 * i + 2] != 0;
      mis += s.k == g->sh[0].k ? s.h_info[4 * i + 3] : 0;
    }
  }
  g->pending = 0;
  g->queued = 0;
  if (bailed && !timeout) {
    // AUTO's class budget ran out (bucket_kernel.cuh): this graph is one for
    // the n-round engine -- rerun these solves there, and keep it for the
    // handle's later solves
    g->bucket = false;
    const std::vector<uint64_t> src = g->last_sources;
    const float spent_ms = [&] {
      float ms = 0;
      cudaEventElapsedTime(&ms, g->sh[0].ev0, g->sh[0].ev1);
      return ms;
    }();
    int rc = launch(g, src.data(), (uint32_t)src.size());
    if (rc) return rc;
    rc = finish(g, st);
    if (rc == SSSP_OK && st) st->rounds_s += spent_ms * 1e-3;  // both launches count
    return rc;
  }
  // AUTO re-plan: a distance class costs ~10x a scan round (measured: ~5 us vs
  // ~0.5 us), so a graph whose solves need more than n/8 classes (long sparse
  // paths: config 1 sparse has 154 classes at n=1000) runs faster on the
  // n-round cluster engine from the next solve on.  Deterministic, hence
  // identical on every shard/rank.
  if (g->bucket && g->opt.engine == SSSP_ENGINE_AUTO && k > 0 && classes / k > g->n / 8)
    g->bucket = false;
  if (g->multiproc) g->exch_base = last + 1;
  if (g->bucket && g->sh[0].d_spans && k == 1 && nqueued > 1) {  // debug: gaps between launches
    std::vector<unsigned long long> sp(128);
    CK(cudaMemcpy(sp.data(), g->sh[0].d_spans, 128 * 8, cudaMemcpyDeviceToHost));
    double sum_span = 0, sum_gap = 0;
    int ns = 0, ng = 0;
    const uint64_t last = g->bseq, first = g->bseq + 1 - std::min<uint64_t>(nqueued, 64);
    for (uint64_t q = first; q <= last; ++q) {
      const unsigned long long st0 = ~sp[(q % 64) * 2], en = sp[(q % 64) * 2 + 1];
      if (!sp[(q % 64) * 2] || !en) continue;
      sum_span += (en - st0) * 1e-3;
      ++ns;
      if (q > first && sp[((q - 1) % 64) * 2 + 1]) {
        sum_gap += (st0 - sp[((q - 1) % 64) * 2 + 1]) * 1e-3;
        ++ng;
      }
    }
    fprintf(stderr, "launch spans: %d launches, mean span %.2f us, mean gap %.2f us\n", ns, ns ? sum_span / ns : 0.0,
            ng ? sum_gap / ng : 0.0);
    CK(cudaMemset(g->sh[0].d_spans, 0, 128 * 8));
  }
  if (g->bucket && g->sh[0].d_trace) {
    std::vector<uint64_t> tr(512 + 4096);
    CK(cudaMemcpy(tr.data(), g->sh[0].d_trace, tr.size() * 8, cudaMemcpyDeviceToHost));
    // entries: phase code << 56 | %globaltimer (bucket_kernel.cuh stamp())
    static const char* names[] = {"start", "bar", "detld", "det", "enum", "pushld", "push",
                                  "pullset", "pull", "pub0", "pub1", "wb", "row0", "owner", "x14", "local1", "rsum", "scan"};
    const uint64_t tmask = (1ull << 56) - 1;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, g->sh[0].device);
    fprintf(stderr, "bucket trace (us since kernel start at %d MHz; phase:end):", khz / 1000);
    for (int i = 1; i < 512 && tr[i < 64 ? i : 4096 + i]; ++i) {
      const uint64_t t = tr[i < 64 ? i : 4096 + i];
      const uint32_t c = (uint32_t)(t >> 56);
      fprintf(stderr, " %s:%.2f", c < 18 ? names[c] : "?", ((t & tmask) - (tr[0] & tmask)) * 1e3 / khz);
    }
    fprintf(stderr, "\n");
    // per-CTA span of the last pull step (start, end relative to kernel start)
    double smin = 1e30, smax = 0, emin = 1e30, emax = 0, dsum = 0;
    int nc = 0;
    for (int c = 0; c < 1024 && tr[64 + 2 * c]; ++c, ++nc) {
      const double a = (tr[64 + 2 * c] - tr[0]) * 1e-3, b = (tr[64 + 2 * c + 1] - tr[0]) * 1e-3;
      smin = std::min(smin, a); smax = std::max(smax, a);
      emin = std::min(emin, b); emax = std::max(emax, b);
      dsum += b - a;
    }
    if (nc) fprintf(stderr, "pull per CTA (%d): start %.2f..%.2f end %.2f..%.2f mean %.2f us\n", nc, smin,
                    smax, emin, emax, dsum / nc);
    {  // every CTA's start / end (%globaltimer) relative to the earliest start
      uint64_t s0t = ~0ull, s1t = 0, e0t = ~0ull, e1t = 0;
      int m = 0;
      for (int c = 0; c < 1024 && tr[64 + 2048 + 2 * c]; ++c, ++m) {
        s0t = std::min(s0t, tr[64 + 2048 + 2 * c]);
        s1t = std::max(s1t, tr[64 + 2048 + 2 * c]);
        e0t = std::min(e0t, tr[64 + 2048 + 2 * c + 1]);
        e1t = std::max(e1t, tr[64 + 2048 + 2 * c + 1]);
      }
      if (m)
        fprintf(stderr, "CTA spans (%d): start 0..%.2f end %.2f..%.2f us (CTA 0 starts at %.2f)\n", m,
                (s1t - s0t) * 1e-3, (e0t - s0t) * 1e-3, (e1t - s0t) * 1e-3, (tr[64 + 2048] - s0t) * 1e-3);
    }
  }
  if (st) {
    st->transfer_in_s = g->transfer_in_s;
    st->rounds_s = rounds;
    st->iterations = iters;
    st->relax_checks = (g->bucket ? rows : iters) * g->sh[0].row_stride * g->P;
    st->mispredicts = mis;
    st->engine = g->wide ? SSSP_ENGINE_WIDE : g->bucket ? SSSP_ENGINE_BUCKET
                 : g->cluster ? SSSP_ENGINE_CLUSTER : SSSP_ENGINE_GRID;
    st->classes = (uint32_t)classes;
    st->rows_read = g->bucket ? rows : iters;
    fill_reference_stats(g, st);
    st->exchanges = (g->bucket ? classes : iters) / k;
    st->barriers = g->bucket ? nbars / std::min<uint32_t>(k, 64) : st->exchanges;
    st->bytes_read = g->bucket ? nbytes / k
                               : iters / k * g->sh[0].row_stride * g->wbytes * g->P;
    st->matrix_bytes = g->matrix_bytes;
    st->weight_bytes = g->wbytes;
    st->ctas = g->cluster ? g->sh[0].C : g->sh[0].G;
    st->shards = g->P;
    st->packed_key = g->packed;
  }
  if (timeout && g->bucket && g->P > 1 && !g->multiproc)  // barrier counters out of step: restart
    for (auto& s : g->sh) {
      CK(cudaSetDevice(s.device));
      CK(cudaMemset(reinterpret_cast<char*>(s.d_slots) + g->slots_bytes, 0, g->ctrl_off));
    }
  if (timeout) return fail(SSSP_ERR_TIMEOUT, "exchange watchdog fired (a peer never published)");
  return SSSP_OK;
}

// Copies solve i's owned columns of every local shard into the caller rows.
int copy_out(sssp_graph* g, uint32_t k, uint64_t* dist_out, uint64_t* pred_out,
             uint64_t row_len) {
  for (auto& s : g->sh) {
    if (s.cols == 0) continue;
    CK(cudaSetDevice(s.device));
    const uint64_t off = g->multiproc ? 0 : s.col_base;
    if (dist_out)
      CK(cudaMemcpy2DAsync(dist_out + off, row_len * 8, s.d_dist, s.loc_n * 8, s.cols * 8, k,
                           cudaMemcpyDeviceToHost, s.stream));
    if (pred_out)
      CK(cudaMemcpy2DAsync(pred_out + off, row_len * 8, s.d_pred, s.loc_n * 8, s.cols * 8, k,
                           cudaMemcpyDeviceToHost, s.stream));
  }
  for (auto& s : g->sh) {
    CK(cudaSetDevice(s.device));
    CK(cudaStreamSynchronize(s.stream));
  }
  return SSSP_OK;
}

}  // namespace

namespace {

// Uploads an edge list into every shard's matrix: H2D of the (u, v, w)
// triples in pinned chunks, then init + keep-minimum scatter on the device.
template <typename W>
int build_from_edges(sssp_graph* g, Shard& s, const uint64_t* edges, uint64_t m) {
  CK(cudaSetDevice(s.device));
  int rc = alloc_matrix(s, g->n, sizeof(W));
  if (rc) return rc;
  const uint64_t total = g->n * s.row_stride;
  init_matrix_kernel<W><<<(unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 32), 256, 0,
                          s.stream>>>(static_cast<W*>(s.d_adj), g->n, s.row_stride, s.col_base,
                                      s.cols, s.G, s.L);
  CK(cudaGetLastError());
  if (m == 0) return SSSP_OK;
  std::lock_guard<std::mutex> staging_lock(g_staging.m);
  const uint64_t chunk = std::min<uint64_t>(m, 1ull << 20);  // edges per chunk (24 MB)
  void* dbuf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    if (!g_staging.get(b, chunk * 24) || pool_alloc(s, &dbuf[b], chunk * 24) != SSSP_OK)
      return fail(SSSP_ERR_OOM, "edge staging");
    CK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
  }
  bool used[2] = {false, false};
  for (uint64_t e0 = 0, k = 0; e0 < m; e0 += chunk, ++k) {
    const int b = (int)(k & 1);
    const uint64_t cnt = std::min(chunk, m - e0);
    if (used[b]) CK(cudaEventSynchronize(done[b]));
    std::memcpy(g_staging.buf[b], edges + 3 * e0, cnt * 24);
    CK(cudaMemcpyAsync(dbuf[b], g_staging.buf[b], cnt * 24, cudaMemcpyHostToDevice, s.stream));
    scatter_edges_kernel<W><<<(unsigned)std::min<uint64_t>((cnt + 255) / 256, 148ull * 16), 256, 0,
                              s.stream>>>(static_cast<const uint64_t*>(dbuf[b]), cnt,
                                          static_cast<W*>(s.d_adj), s.row_stride, s.col_base,
                                          s.cols, s.G, s.L, g->directed);
    CK(cudaGetLastError());
    CK(cudaEventRecord(done[b], s.stream));
    used[b] = true;
  }
  CK(cudaStreamSynchronize(s.stream));
  for (int b = 0; b < 2; ++b) {
    cudaFreeAsync(dbuf[b], s.stream);
    cudaEventDestroy(done[b]);
  }
  return SSSP_OK;
}

int enable_peers(const int* devices, int ndev) {
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < ndev; ++j) {
      if (devices[i] == devices[j]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
      if (!can) return fail(SSSP_ERR_NO_PEER, "no peer access between devices");
      cudaSetDevice(devices[i]);
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(SSSP_ERR_NO_PEER, cudaGetErrorString(e));
      cudaGetLastError();
    }
  return SSSP_OK;
}

}  // namespace

extern "C" {

const char* sssp_status_string(int status) {
  switch (status) {
    case SSSP_OK: return "ok";
    case SSSP_ERR_BAD_SOURCE: return "source out of range";
    case SSSP_ERR_BAD_ARG: return "bad argument";
    case SSSP_ERR_WEIGHT_RANGE: return "weight outside the device encoding";
    case SSSP_ERR_OOM: return "out of memory";
    case SSSP_ERR_CUDA: return "CUDA error";
    case SSSP_ERR_NO_PEER: return "peer access unavailable";
    case SSSP_ERR_TIMEOUT: return "exchange watchdog timeout";
    case SSSP_ERR_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* sssp_last_error(void) { return g_err.c_str(); }

int sssp_abi_version(void) { return SSSP_ABI_VERSION; }

int sssp_device_count(int* count) {
  *count = 0;
  CK(cudaGetDeviceCount(count));
  return SSSP_OK;
}

int sssp_graph_create_from_edges(uint64_t n, const uint64_t* edges, uint64_t m, int directed,
                                 const int* devices, int ndev, const sssp_options* opt,
                                 sssp_graph** out) {
  *out = nullptr;
  if (n == 0 || (m && !edges)) return fail(SSSP_ERR_BAD_ARG, "empty graph");
  if (n > 0x1FFFFFFFull) return fail(SSSP_ERR_UNSUPPORTED, "n exceeds 2^29");
  if (ndev < 0 || ndev > SSSP_MAX_SHARDS) return fail(SSSP_ERR_BAD_ARG, "1..8 shards");
  const int dev0 = 0;
  if (!devices || ndev == 0) {
    devices = &dev0;
    ndev = 1;
  }
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count) return fail(SSSP_ERR_BAD_ARG, "bad device id");
  // graph.hpp:80-83: the inputs graph_from_edges rejects; and the weight range
  const double t0 = now_s();
  const unsigned nt = narrow_threads();
  std::vector<uint64_t> tmx(nt, 0), tmn(nt, ~0ull);
  std::vector<char> bad(nt, 0);
  parallel_run([&](unsigned t) {
    uint64_t mx = 0, mn = ~0ull;
    for (uint64_t i = m * t / nt; i < m * (t + 1) / nt; ++i) {
      const uint64_t u = edges[3 * i], v = edges[3 * i + 1], w = edges[3 * i + 2];
      if (u >= n || v >= n || u == v || w > 0xFFFFFFFFull) bad[t] = 1;
      mx = std::max(mx, w);
      mn = std::min(mn, w);
    }
    tmx[t] = mx;
    tmn[t] = mn;
  });
  for (unsigned t = 0; t < nt; ++t)
    if (bad[t]) return fail(SSSP_ERR_BAD_ARG, "edge endpoint out of range, self-loop or weight > 2^32-1");
  const uint64_t max_w = *std::max_element(tmx.begin(), tmx.end());
  const uint64_t min_w = *std::min_element(tmn.begin(), tmn.end());
  sssp_graph* g = new sssp_graph();
  g->n = n;
  g->directed = directed;
  g->P = (uint32_t)ndev;
  g->opt = default_options(opt);
  g->max_w = max_w;
  g->min_w = min_w;
  g->wbytes = max_w <= 0xFE ? 1 : max_w <= 0xFFFE ? 2 : max_w <= 0xFFFFFFFEull ? 4 : 8;
  int rc = create_shard_objects(g, g->P, devices, g->P, 0);
  if (rc == SSSP_OK) rc = enable_peers(devices, ndev);
  for (uint32_t i = 0; rc == SSSP_OK && i < g->P; ++i)
    rc = g->wbytes == 1 ? build_from_edges<uint8_t>(g, g->sh[i], edges, m)
         : g->wbytes == 2 ? build_from_edges<uint16_t>(g, g->sh[i], edges, m)
         : g->wbytes == 4 ? build_from_edges<uint32_t>(g, g->sh[i], edges, m)
                          : build_from_edges<uint64_t>(g, g->sh[i], edges, m);
  if (rc == SSSP_OK) rc = setup_common(g);
  if (rc) {
    destroy_graph(g);
    return rc;
  }
  g->upload_bytes = m * 24 * g->P;  // the (u, v, w) triples, to every shard
  g->transfer_in_s = now_s() - t0;
  *out = g;
  return SSSP_OK;
}

int sssp_graph_create(const uint64_t* adj, uint64_t n, int directed, const int* devices,
                      int ndev, const sssp_options* opt, sssp_graph** out) {
  *out = nullptr;
  if (n == 0 || !adj) return fail(SSSP_ERR_BAD_ARG, "empty graph");
  if (n > 0x1FFFFFFFull) return fail(SSSP_ERR_UNSUPPORTED, "n exceeds 2^29");
  if (ndev < 0 || ndev > SSSP_MAX_SHARDS) return fail(SSSP_ERR_BAD_ARG, "1..8 shards");
  const int dev0 = 0;
  if (!devices || ndev == 0) {
    devices = &dev0;
    ndev = 1;
  }
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count) return fail(SSSP_ERR_BAD_ARG, "bad device id");
  const double t0 = now_s();
  sssp_graph* g = new sssp_graph();
  g->n = n;
  g->directed = directed;
  g->P = (uint32_t)ndev;
  g->opt = default_options(opt);
  int rc = create_shard_objects(g, g->P, devices, g->P, 0);
  if (rc == SSSP_OK) rc = enable_peers(devices, ndev);
  // Several shards must agree on one encoding: take it from a scan of the
  // whole matrix.  A single shard widens optimistically inside the upload.
  uint64_t hint = 0;
  if (rc == SSSP_OK && g->P > 1) {
    const unsigned nt = narrow_threads();
    std::vector<uint64_t> tm(nt, 0);
    parallel_run([&](unsigned t) {
      const uint64_t a = n * t / nt, e = n * (t + 1) / nt;
      uint64_t mx = 0;
      for (uint64_t i = a * n; i < e * n; ++i) {
        const uint64_t x = adj[i];
        if (x != ~0ull && x > mx) mx = x;
      }
      tm[t] = mx;
    });
    for (uint64_t x : tm) hint = std::max(hint, x);
  }
  for (uint32_t i = 0; rc == SSSP_OK && i < g->P; ++i) {
    Shard& s = g->sh[i];
    uint32_t wb = 0;
    uint64_t mx = 0, mn = ~0ull;
    rc = upload_shard(s, adj + s.col_base, n, n, hint, &wb, &mx, &mn);
    g->wbytes = std::max(g->wbytes, wb);
    g->max_w = std::max(g->max_w, mx);
    g->min_w = std::min(g->min_w, mn);
  }
  if (rc == SSSP_OK) rc = setup_common(g);
  if (rc) {
    destroy_graph(g);
    return rc;
  }
  for (const auto& sh : g->sh) g->upload_bytes += g->n * sh.cols * g->wbytes;  // narrowed H2D
  g->transfer_in_s = now_s() - t0;
  *out = g;
  return SSSP_OK;
}

int sssp_shard_create(const uint64_t* block, uint64_t ld, uint64_t n, uint32_t world,
                      uint32_t rank, uint64_t max_weight, int device, const sssp_options* opt,
                      sssp_graph** out) {
  *out = nullptr;
  if (n == 0 || !block) return fail(SSSP_ERR_BAD_ARG, "empty graph");
  if (world < 1 || world > SSSP_MAX_SHARDS || rank >= world)
    return fail(SSSP_ERR_BAD_ARG, "bad rank/world");
  const double t0 = now_s();
  sssp_graph* g = new sssp_graph();
  g->n = n;
  g->P = world;
  g->multiproc = world > 1;
  g->connected = world == 1;
  g->opt = default_options(opt);
  int rc = create_shard_objects(g, world, &device, 1, rank);
  if (rc == SSSP_OK) {
    uint32_t wb = 0;
    uint64_t mx = 0, mn = ~0ull;
    rc = upload_shard(g->sh[0], block, ld, n, max_weight, &wb, &mx, &mn);
    g->wbytes = wb;
    g->max_w = std::max(mx, max_weight);
    // the bucket engine must be chosen identically on every rank: with several
    // ranks only the caller-supplied global minimum counts
    g->min_w = world == 1 ? mn
               : g->opt.global_min_weight >= 0 ? (uint64_t)g->opt.global_min_weight : 0;
    // all ranks must agree on the encoding: derive it from the global bound
    if (rc == SSSP_OK && max_weight) {
      const uint32_t want = max_weight <= 0xFE ? 1 : max_weight <= 0xFFFE ? 2 : 4;
      if (want != wb) rc = fail(SSSP_ERR_WEIGHT_RANGE, "max_weight hint below the block's weights");
    }
  }
  if (rc == SSSP_OK) rc = setup_common(g);
  if (rc == SSSP_OK && world == 1) g->sh[0].peer[0] = g->sh[0].d_slots;
  if (rc) {
    destroy_graph(g);
    return rc;
  }
  for (const auto& sh : g->sh) g->upload_bytes += g->n * sh.cols * g->wbytes;  // narrowed H2D
  g->transfer_in_s = now_s() - t0;
  *out = g;
  return SSSP_OK;
}

int sssp_block_weight_range(const uint64_t* block, uint64_t ld, uint64_t n, uint64_t col_begin,
                            uint64_t col_count, uint64_t* min_offdiag, uint64_t* max_finite) {
  if (!block || !min_offdiag || !max_finite || ld < col_count)
    return fail(SSSP_ERR_BAD_ARG, "bad block");
  const unsigned nt = narrow_threads();
  std::vector<uint64_t> mn(nt, ~0ull), mx(nt, 0);
  parallel_run([&](unsigned t) {
    uint64_t lo = ~0ull, hi = 0;
    for (uint64_t r = n * t / nt; r < n * (t + 1) / nt; ++r) {
      const uint64_t* row = block + r * ld;
      for (uint64_t j = 0; j < col_count; ++j) {
        const uint64_t x = row[j];
        if (x == ~0ull) continue;
        hi = std::max(hi, x);
        if (col_begin + j != r) lo = std::min(lo, x);
      }
    }
    mn[t] = lo;
    mx[t] = hi;
  });
  *min_offdiag = *std::min_element(mn.begin(), mn.end());
  *max_finite = *std::max_element(mx.begin(), mx.end());
  return SSSP_OK;
}

int sssp_shard_export(sssp_graph* g, void* handle_out) {
  if (!g || g->sh.size() != 1) return fail(SSSP_ERR_BAD_ARG, "not a shard handle");
  CK(cudaSetDevice(g->sh[0].device));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, g->sh[0].d_slots));
  std::memcpy(handle_out, &h, sizeof(h));
  return SSSP_OK;
}

int sssp_shard_connect(sssp_graph* g, const void* handles) {
  if (!g || g->sh.size() != 1) return fail(SSSP_ERR_BAD_ARG, "not a shard handle");
  Shard& s = g->sh[0];
  CK(cudaSetDevice(s.device));
  for (uint32_t j = 0; j < g->P; ++j) {
    if (j == s.k) {
      s.peer[j] = s.d_slots;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)j * SSSP_IPC_HANDLE_BYTES,
                sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(SSSP_ERR_NO_PEER, cudaGetErrorString(e));
    s.peer[j] = static_cast<uint64_t*>(p);
    s.peer_ipc[j] = true;
  }
  g->connected = true;
  return SSSP_OK;
}

int sssp_shard_range(const sssp_graph* g, uint64_t* col_begin, uint64_t* col_count) {
  if (!g || g->sh.empty()) return fail(SSSP_ERR_BAD_ARG, "null handle");
  *col_begin = g->sh[0].col_base;
  *col_count = g->multiproc ? g->sh[0].cols : g->n;
  if (!g->multiproc) *col_begin = 0;
  return SSSP_OK;
}

int sssp_graph_destroy(sssp_graph* g) {
  if (g) destroy_graph(g);
  return SSSP_OK;
}

int sssp_graph_info(const sssp_graph* g, sssp_solve_stats* st) {
  if (!g || !st) return fail(SSSP_ERR_BAD_ARG, "null");
  std::memset(st, 0, sizeof(*st));
  st->transfer_in_s = g->transfer_in_s;
  st->matrix_bytes = g->matrix_bytes;
  st->weight_bytes = g->wbytes;
  st->ctas = g->cluster ? g->sh[0].C : g->sh[0].G;
  st->shards = g->P;
  st->packed_key = g->packed;
  st->engine = g->wide ? SSSP_ENGINE_WIDE : g->bucket ? SSSP_ENGINE_BUCKET
               : g->cluster ? SSSP_ENGINE_CLUSTER : SSSP_ENGINE_GRID;
  fill_reference_stats(g, st);
  st->iterations = g->max_batch;  // reused: concurrent solve capacity
  st->relax_checks = g->min_w;    // reused: min finite off-diagonal weight
  st->mispredicts = g->max_w;     // reused: max finite weight
  return SSSP_OK;
}

int sssp_solve(sssp_graph* g, uint64_t source, uint64_t* dist_out, uint64_t* pred_out,
               uint64_t* visit_order_out, sssp_solve_stats* st) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  int rc = launch(g, &source, 1);
  if (rc) return rc;
  sssp_solve_stats local{};
  rc = finish(g, &local);
  if (rc) return rc;
  const double t0 = now_s();
  rc = copy_out(g, 1, dist_out, pred_out, g->multiproc ? g->sh[0].cols : g->n);
  if (rc) return rc;
  if (visit_order_out) {
    if (!g->sh[0].d_visit) return fail(SSSP_ERR_BAD_ARG, "record_visit_order was not set");
    std::vector<uint32_t> tmp(local.iterations);
    CK(cudaSetDevice(g->sh[0].device));
    CK(cudaMemcpy(tmp.data(), g->sh[0].d_visit, local.iterations * 4, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < local.iterations; ++i) visit_order_out[i] = tmp[i];
    // the reference keeps electing after the last reachable vertex: the
    // unreachable ones, lowest id first (serial.hpp:41-48, INF ties), relaxing
    // nothing -- the order is completed here (n entries, as visit_order gets)
    if (!g->multiproc) {
      std::vector<char> seen(g->n, 0);
      for (uint64_t i = 0; i < local.iterations; ++i) seen[tmp[i]] = 1;
      uint64_t k = local.iterations;
      for (uint64_t v = 0; v < g->n; ++v)
        if (!seen[v]) visit_order_out[k++] = v;
    }
  }
  local.transfer_out_s = now_s() - t0;
  if (st) *st = local;
  return SSSP_OK;
}

int sssp_solve_batch(sssp_graph* g, const uint64_t* sources, uint32_t k, uint64_t* dist_out,
                     uint64_t* pred_out, sssp_solve_stats* st) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  sssp_solve_stats total{};
  const uint64_t row_len = g->multiproc ? g->sh[0].cols : g->n;
  for (uint32_t i0 = 0; i0 < k; i0 += g->max_batch) {
    const uint32_t kk = std::min<uint32_t>(g->max_batch, k - i0);
    int rc = launch(g, sources + i0, kk);
    if (rc) return rc;
    sssp_solve_stats part{};
    rc = finish(g, &part);
    if (rc) return rc;
    const double t0 = now_s();
    rc = copy_out(g, kk, dist_out ? dist_out + (uint64_t)i0 * row_len : nullptr,
                  pred_out ? pred_out + (uint64_t)i0 * row_len : nullptr, row_len);
    if (rc) return rc;
    total.transfer_out_s += now_s() - t0;
    total.rounds_s += part.rounds_s;
    total.iterations += part.iterations;
    total.relax_checks += part.relax_checks;
    total.mispredicts += part.mispredicts;
    total.transfer_in_s = part.transfer_in_s;
    total.matrix_bytes = part.matrix_bytes;
    total.weight_bytes = part.weight_bytes;
    total.ctas = part.ctas;
    total.shards = part.shards;
    total.packed_key = part.packed_key;
  }
  if (st) *st = total;
  return SSSP_OK;
}

int sssp_enqueue(sssp_graph* g, const uint64_t* sources, uint32_t k) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  // Launches queue up in stream order; each one reuses the handle's output
  // slots, so sssp_finish reports (and the buffers hold) the last one.
  return launch(g, sources, k);
}

int sssp_finish(sssp_graph* g, sssp_solve_stats* st) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  return finish(g, st);
}

int sssp_probe_sync(sssp_graph* g, uint32_t rounds, double* seconds_per_round) {
  if (!g || rounds == 0) return fail(SSSP_ERR_BAD_ARG, "bad probe arguments");
  if (g->multiproc && !g->connected) return fail(SSSP_ERR_BAD_ARG, "shard not connected");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  const uint32_t np = g->sh[0].NP;
  if (g->wide) return fail(SSSP_ERR_UNSUPPORTED, "not available with 64-bit distances (wide engine)");
  auto probe_fn = [&](int device) -> ProbeFn {  // a launch with several shards: the MS instance
    const bool ms = shards_on_device(g, device) > 1;
    return g->cluster ? get_cluster_probe((int)g->sh[0].NW, g->sh[0].hier, ms)
                      : get_grid_probe((int)np, ms);
  };
  std::vector<cudaEvent_t> reset_ev;
  if (!g->multiproc) {
    g->exch_base = 0;
    for (auto& s : g->sh) {
      CK(cudaSetDevice(s.device));
      CK(cudaMemsetAsync(s.d_slots, 0, g->slot_stride * sizeof(uint64_t), s.stream));
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, s.stream));
      reset_ev.push_back(e);
    }
  }
  const auto groups = device_groups(g);
  std::vector<uint64_t*> d_ns(groups.size(), nullptr);
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    std::vector<ScanParams> ps;
    for (uint32_t li : groups[gi]) {
      Shard& s = g->sh[li];
      CK(cudaSetDevice(s.device));
      for (cudaEvent_t e : reset_ev) CK(cudaStreamWaitEvent(s.stream, e, 0));
      CK(cudaMemsetAsync(s.d_info, 0, 4 * sizeof(uint64_t), s.stream));
      ScanParams p{};
      p.G = s.G;
      p.vbits = g->vbits;
      p.shard = s.k;
      p.nshards = g->P;
      p.slots = s.d_slots;
      for (uint32_t j = 0; j < g->P && j < (uint32_t)kMaxShards; ++j)
        p.peer_slots[j] = g->multiproc ? s.peer[j] : g->sh[j].d_slots;
      p.slot_stride = g->slot_stride;
      p.bstride = (uint32_t)g->bstride;
      p.nrep = g->nrep;
      p.exch_base = g->exch_base;
      p.info = s.d_info;
      p.timeout_ns = g->opt.timeout_ms * 1000000ull;
      ps.push_back(p);
    }
    CK(cudaSetDevice(g->sh[groups[gi][0]].device));
    ProbeFn fn = probe_fn(g->sh[groups[gi][0]].device);
    if (!fn) return fail(SSSP_ERR_UNSUPPORTED, "no probe instance");
    if (g->cluster && g->sh[0].C > 8)
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaMalloc(&d_ns[gi], groups[gi].size() * sizeof(uint64_t)));  // [local shard]
    CK(launch_kernel(g, groups[gi], (void*)fn, 1, ps, &rounds, 1, d_ns[gi]));
  }
  double worst = 0;
  uint64_t last = 0;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    for (size_t li = 0; li < groups[gi].size(); ++li) {
      Shard& s = g->sh[groups[gi][li]];
      CK(cudaSetDevice(s.device));
      CK(cudaStreamSynchronize(s.stream));
      uint64_t ns = 0, info[4];
      CK(cudaMemcpy(&ns, d_ns[gi] + li, sizeof(ns), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(info, s.d_info, sizeof(info), cudaMemcpyDeviceToHost));
      if (ns == ~0ull) return fail(SSSP_ERR_TIMEOUT, "probe watchdog fired");
      worst = std::max(worst, ns * 1e-9 / rounds);
      last = std::max(last, info[1]);
    }
    cudaFree(d_ns[gi]);
  }
  for (cudaEvent_t e : reset_ev) cudaEventDestroy(e);
  if (g->multiproc) g->exch_base = last + 1;
  *seconds_per_round = worst;
  return SSSP_OK;
}

int sssp_probe_skeleton(sssp_graph* g, uint32_t barriers, uint32_t launches,
                        double* seconds_per_launch) {
  if (!g || !seconds_per_launch || launches == 0) return fail(SSSP_ERR_BAD_ARG, "bad probe arguments");
  if (!g->bucket || g->P != 1 || g->multiproc)
    return fail(SSSP_ERR_UNSUPPORTED, "skeleton probe: single-shard bucket engine only");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  Shard& s = g->sh[0];
  CK(cudaSetDevice(s.device));
  const size_t smem = bucket_smem(g);
  CK(raise_smem((const void*)bucket_skeleton_kernel, smem));
  uint32_t* sink = nullptr;
  CK(pool_alloc(s, (void**)&sink, 64) == SSSP_OK ? cudaSuccess : cudaErrorMemoryAllocation);
  void* args[] = {(void*)&barriers, (void*)&sink};
  // launched exactly as the solves are: cooperative + programmatic stream
  // serialisation (SSSP_BUCKET_PDL)
  static const bool k_pdl = env_u64("SSSP_BUCKET_PDL", 1) != 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeCooperative;
  la[0].val.cooperative = 1;
  la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(g->bG);
  cfg.blockDim = dim3(kBucketThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s.stream;
  cfg.attrs = la;
  cfg.numAttrs = k_pdl ? 2 : 1;
  for (int w = 0; w < 3; ++w) CK(cudaLaunchKernelExC(&cfg, (void*)bucket_skeleton_kernel, args));
  CK(cudaEventRecord(s.ev0, s.stream));
  for (uint32_t i = 0; i < launches; ++i) CK(cudaLaunchKernelExC(&cfg, (void*)bucket_skeleton_kernel, args));
  CK(cudaEventRecord(s.ev1, s.stream));
  CK(cudaEventSynchronize(s.ev1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
  pool_free(s, sink);
  CK(cudaStreamSynchronize(s.stream));
  *seconds_per_launch = ms * 1e-3 / launches;
  return SSSP_OK;
}

// ---- host-driven NCCL comparison path (nccl_kernel.cuh)
namespace {
int nccl_params(sssp_graph* g, NcclRoundParams* p) {
  if (g->sh.size() != 1 || g->wide || !g->cluster)
    return fail(SSSP_ERR_UNSUPPORTED, "NCCL comparison path: one local shard, cluster layout, 32-bit distances");
  if (g->multiproc && !g->connected) return fail(SSSP_ERR_BAD_ARG, "shard not connected");
  const Shard& s = g->sh[0];
  p->adj = s.d_adj;
  p->row_stride = s.row_stride;
  p->npos = (uint32_t)s.row_stride;
  p->Q = s.G;
  p->qbits = bitlen(s.G) - 1;
  p->lbits = bitlen(s.L) - 1;
  p->loc_n = (uint32_t)s.loc_n;
  p->col_base = (uint32_t)s.col_base;
  p->n = (uint32_t)g->n;
  p->dist = g->nc_dist;
  p->pred = g->nc_pred;
  p->visited = g->nc_vis;
  return SSSP_OK;
}
unsigned nccl_grid(uint32_t npos) { return (unsigned)std::min<uint64_t>((npos + 255) / 256, 148ull * 8); }
}  // namespace

int sssp_nccl_begin(sssp_graph* g, uint64_t source) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  if (source >= g->n) return fail(SSSP_ERR_BAD_SOURCE, "dijkstra_partitioned: source out of range");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  NcclRoundParams p{};
  int rc = nccl_params(g, &p);
  if (rc) return rc;
  Shard& s = g->sh[0];
  CK(cudaSetDevice(s.device));
  if (!g->nc_dist) {
    if (pool_alloc(s, (void**)&g->nc_dist, s.row_stride * 4) || pool_alloc(s, (void**)&g->nc_pred, s.row_stride * 4) ||
        pool_alloc(s, (void**)&g->nc_vis, s.row_stride))
      return fail(SSSP_ERR_OOM, "NCCL path state");
    nccl_params(g, &p);
  }
  nccl_init_kernel<<<nccl_grid(p.npos), 256, 0, s.stream>>>(p, (uint32_t)source);
  CK(cudaGetLastError());
  return SSSP_OK;
}

int sssp_nccl_local_min(sssp_graph* g, uint64_t* d_key) {
  if (!g || !d_key) return fail(SSSP_ERR_BAD_ARG, "null argument");
  NcclRoundParams p{};
  int rc = nccl_params(g, &p);
  if (rc) return rc;
  if (!g->nc_dist) return fail(SSSP_ERR_BAD_ARG, "sssp_nccl_begin first");
  nccl_local_min_kernel<<<1, kNcclMinThreads, 0, g->sh[0].stream>>>(p, d_key);
  CK(cudaGetLastError());
  return SSSP_OK;
}

int sssp_nccl_relax(sssp_graph* g, const uint64_t* d_key) {
  if (!g || !d_key) return fail(SSSP_ERR_BAD_ARG, "null argument");
  NcclRoundParams p{};
  int rc = nccl_params(g, &p);
  if (rc) return rc;
  if (!g->nc_dist) return fail(SSSP_ERR_BAD_ARG, "sssp_nccl_begin first");
  const unsigned grid = nccl_grid(p.npos);
  cudaStream_t st = g->sh[0].stream;
  if (g->wbytes == 1) nccl_relax_kernel<uint8_t><<<grid, 256, 0, st>>>(p, d_key);
  else if (g->wbytes == 2) nccl_relax_kernel<uint16_t><<<grid, 256, 0, st>>>(p, d_key);
  else nccl_relax_kernel<uint32_t><<<grid, 256, 0, st>>>(p, d_key);
  CK(cudaGetLastError());
  return SSSP_OK;
}

int sssp_nccl_end(sssp_graph* g, uint64_t* dist_out, uint64_t* pred_out) {
  if (!g || !dist_out || !pred_out) return fail(SSSP_ERR_BAD_ARG, "null argument");
  NcclRoundParams p{};
  int rc = nccl_params(g, &p);
  if (rc) return rc;
  if (!g->nc_dist) return fail(SSSP_ERR_BAD_ARG, "sssp_nccl_begin first");
  Shard& s = g->sh[0];
  CK(cudaSetDevice(s.device));
  nccl_out_kernel<<<nccl_grid(p.npos), 256, 0, s.stream>>>(p, s.d_dist, s.d_pred);
  CK(cudaGetLastError());
  if (s.cols) {
    CK(cudaMemcpyAsync(dist_out, s.d_dist, s.cols * 8, cudaMemcpyDeviceToHost, s.stream));
    CK(cudaMemcpyAsync(pred_out, s.d_pred, s.cols * 8, cudaMemcpyDeviceToHost, s.stream));
  }
  CK(cudaStreamSynchronize(s.stream));
  return SSSP_OK;
}

int sssp_validate(sssp_graph* g, uint64_t source, const uint64_t* dist, const uint64_t* pred,
                  uint64_t* violations) {
  if (!g || !dist || !pred || !violations) return fail(SSSP_ERR_BAD_ARG, "null argument");
  if (source >= g->n) return fail(SSSP_ERR_BAD_SOURCE, "validate: source out of range");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  if (g->wide) return fail(SSSP_ERR_UNSUPPORTED, "not available with 64-bit distances (wide engine)");
  uint64_t total = 0;
  const uint64_t n = g->n;
  for (auto& s : g->sh) {
    CK(cudaSetDevice(s.device));
    void *dd = nullptr, *dp = nullptr, *dj = nullptr, *dj2 = nullptr, *db = nullptr;
    int rc = pool_alloc(s, &dd, n * 8);
    if (!rc) rc = pool_alloc(s, &dp, n * 8);
    if (!rc) rc = pool_alloc(s, &db, 8);
    if (!rc && s.k == 0) rc = pool_alloc(s, &dj, n * 8);
    if (!rc && s.k == 0) rc = pool_alloc(s, &dj2, n * 8);
    if (rc) return rc;
    CK(cudaMemcpyAsync(dd, dist, n * 8, cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemcpyAsync(dp, pred, n * 8, cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemsetAsync(db, 0, 8, s.stream));
    const uint64_t* D = static_cast<const uint64_t*>(dd);
    const uint64_t* Pp = static_cast<const uint64_t*>(dp);
    auto* B = static_cast<unsigned long long*>(db);
    const unsigned grid = 148 * 8;
#define SSSP_VALIDATE(W)                                                                        \
  validate_edges_kernel<W><<<grid, 256, 0, s.stream>>>(static_cast<const W*>(s.d_adj), n,        \
                                                       s.row_stride, s.col_base, s.cols, s.G,    \
                                                       s.L, D, B);                               \
  validate_pred_kernel<W><<<grid, 256, 0, s.stream>>>(static_cast<const W*>(s.d_adj), n,         \
                                                      s.row_stride, s.col_base, s.cols, s.G, s.L, \
                                                      source, D, Pp, B)
    if (g->wbytes == 1) { SSSP_VALIDATE(uint8_t); }
    else if (g->wbytes == 2) { SSSP_VALIDATE(uint16_t); }
    else { SSSP_VALIDATE(uint32_t); }
#undef SSSP_VALIDATE
    if (s.k == 0) {
      uint64_t* j0 = static_cast<uint64_t*>(dj);
      uint64_t* j1 = static_cast<uint64_t*>(dj2);
      chain_init_kernel<<<grid, 256, 0, s.stream>>>(D, Pp, n, source, j0);
      for (uint64_t r = 1; r < 2 * n; r <<= 1) {  // ceil(log2 n) + 1 doublings
        chain_jump_kernel<<<grid, 256, 0, s.stream>>>(j0, j1, n);
        std::swap(j0, j1);
      }
      chain_check_kernel<<<grid, 256, 0, s.stream>>>(D, j0, n, source, B);
    }
    CK(cudaGetLastError());
    uint64_t bad = 0;
    CK(cudaMemcpyAsync(&bad, db, 8, cudaMemcpyDeviceToHost, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    total += bad;
    for (void* x : {dd, dp, dj, dj2, db}) pool_free(s, x);
  }
  *violations = total;
  return SSSP_OK;
}

// The paper's data-parallel engine (dataparallel_kernel.cuh): relaxation
// rounds to a fixpoint, then reconstruct_predecessors, bit-identical to
// dijkstra_dataparallel (dataparallel.hpp:302-327).  One shard.
int sssp_solve_dataparallel(sssp_graph* g, uint64_t source, uint64_t* dist_out, uint64_t* pred_out,
                            uint64_t* rounds_out, sssp_solve_stats* st) {
  if (!g) return fail(SSSP_ERR_BAD_ARG, "null handle");
  if (source >= g->n) return fail(SSSP_ERR_BAD_SOURCE, "dijkstra_dataparallel: source out of range");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  if (g->wide) return fail(SSSP_ERR_UNSUPPORTED, "not available with 64-bit distances (wide engine)");
  if (g->P != 1 || g->multiproc) return fail(SSSP_ERR_UNSUPPORTED, "dataparallel engine: one shard");
  Shard& s = g->sh[0];
  if (!g->cluster || (s.G & (s.G - 1)) || (s.L & (s.L - 1)))
    return fail(SSSP_ERR_UNSUPPORTED, "dataparallel engine needs the cluster layout");
  CK(cudaSetDevice(s.device));
  const uint32_t wb = g->wbytes, n = (uint32_t)g->n;
  const uint64_t rs = s.row_stride, words = rs / 32;
  void* frelax = wb == 1 ? (void*)dp_relax_kernel<uint8_t>
                 : wb == 2 ? (void*)dp_relax_kernel<uint16_t> : (void*)dp_relax_kernel<uint32_t>;
  void* ftree = wb == 1 ? (void*)dp_tree_kernel<uint8_t, false, false>
                : wb == 2 ? (void*)dp_tree_kernel<uint16_t, false, false>
                          : (void*)dp_tree_kernel<uint32_t, false, false>;
  void* ffast = wb == 1 ? (void*)dp_tree_kernel<uint8_t, false, true>
                : wb == 2 ? (void*)dp_tree_kernel<uint16_t, false, true>
                          : (void*)dp_tree_kernel<uint32_t, false, true>;
  void* fsweep = wb == 1 ? (void*)dp_tree_kernel<uint8_t, true, false>
                 : wb == 2 ? (void*)dp_tree_kernel<uint16_t, true, false>
                           : (void*)dp_tree_kernel<uint32_t, true, false>;
  // tile: 128 B of every row per CTA, widened until the grid is co-resident
  uint32_t T = 128 / wb;
  size_t sm_relax = 0, sm_tree = 0;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
  while (true) {
    if (T > rs) T = (uint32_t)rs;
    const uint64_t G = rs / T;
    sm_relax = dp_relax_smem_bytes(T, (uint32_t)words, wb);
    sm_tree = dp_pred_smem_bytes(T, wb);
    bool fits = T * wb / 16 <= (uint32_t)kBucketThreads && sm_relax <= 200 * 1024;
    for (void* f : {frelax, fsweep}) {
      if (!fits) break;
      const size_t sm = f == frelax ? sm_relax : sm_tree;
      CK(raise_smem(f, sm));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kBucketThreads, sm));
      fits = per_sm > 0 && G <= (uint64_t)per_sm * sms;
    }
    if (fits) break;
    if (T * wb >= 4096 || T >= rs) return fail(SSSP_ERR_UNSUPPORTED, "dataparallel grid does not fit");
    T *= 2;
  }
  CK(raise_smem(ftree, sm_tree));
  CK(raise_smem(ffast, sm_tree));
  const uint32_t G = (uint32_t)(rs / T);
  const uint32_t max_sweeps = n + 2;
  // scratch: front [2][words] | cnt [2][G] | snap [2][rs] | dist_v [n] | pass_v [n] |
  //          sweep_chg [max_sweeps] | flag | info [4] u64
  const uint64_t o_front = 0, o_cnt = o_front + 2 * words * 4, o_snap = (o_cnt + 2ull * G * 4 + 15) & ~15ull;
  const uint64_t o_dv = o_snap + 2 * rs * 4, o_pv = o_dv + (uint64_t)n * 4, o_chg = o_pv + (uint64_t)n * 4;
  const uint64_t o_flag = o_chg + (uint64_t)max_sweeps * 4, o_info = (o_flag + 4 + 15) & ~15ull;
  const uint64_t bytes = o_info + 4 * 8;
  void* scratch = nullptr;
  int rc = pool_alloc(s, &scratch, bytes);
  if (rc) return rc;
  char* b = static_cast<char*>(scratch);
  DpParams p{};
  p.adj = s.d_adj;
  p.row_stride = rs;
  p.n = n;
  p.Q = s.G;
  p.qbits = bitlen(s.G) - 1;
  p.lbits = bitlen(s.L) - 1;
  p.T = T;
  p.source = (uint32_t)source;
  p.gfront = reinterpret_cast<uint32_t*>(b + o_front);
  p.gcnt = reinterpret_cast<uint32_t*>(b + o_cnt);
  p.gsnap = reinterpret_cast<uint32_t*>(b + o_snap);
  p.dist_v = reinterpret_cast<uint32_t*>(b + o_dv);
  p.pass_v = nullptr;
  p.sweep_chg = reinterpret_cast<uint32_t*>(b + o_chg);
  p.max_sweeps = max_sweeps;
  p.flag = reinterpret_cast<uint32_t*>(b + o_flag);
  p.dist_out = s.d_dist;
  p.pred_out = s.d_pred;
  p.info = reinterpret_cast<uint64_t*>(b + o_info);
  CK(cudaMemsetAsync(b + o_flag, 0, o_info + 32 - o_flag, s.stream));
  CK(cudaEventRecord(s.ev0, s.stream));
  void* args[] = {&p};
  CK(cudaLaunchCooperativeKernel(frelax, dim3(G), dim3(kBucketThreads), args, sm_relax, s.stream));
  // FAST tree pass when no weight is 0 (no zero-weight tie can exist) and no
  // finite dist reaches WINF: with u8/u16 weights an INF weight or an
  // unreachable column (dv = 2^32-1) can then never look tight (not u32)
  uint64_t dmax = 0;
  CK(cudaMemcpyAsync(&dmax, p.info + 3, 8, cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  const uint64_t winf = wb == 1 ? 0xFFull : wb == 2 ? 0xFFFFull : 0xFFFFFFFFull;
  const bool fast = wb <= 2 && g->min_w >= 1 && dmax < winf;
  CK(cudaLaunchKernel(fast ? ffast : ftree, dim3(G), dim3(kBucketThreads), args, sm_tree, s.stream));
  uint32_t flag = 0;
  CK(cudaMemcpyAsync(&flag, p.flag, 4, cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  uint64_t tree_passes = 1;
  if (flag) {  // zero-weight tight edges: solve the pass numbers, then rebuild pred with them
    p.pass_v = reinterpret_cast<uint32_t*>(b + o_pv);
    CK(cudaMemsetAsync(p.pass_v, 0xFF, (uint64_t)n * 4, s.stream));
    const uint32_t one = 1;
    CK(cudaMemcpyAsync(p.pass_v + source, &one, 4, cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemsetAsync(p.sweep_chg, 0, (uint64_t)max_sweeps * 4, s.stream));
    CK(cudaLaunchCooperativeKernel(fsweep, dim3(G), dim3(kBucketThreads), args, sm_tree, s.stream));
    CK(cudaLaunchKernel(ftree, dim3(G), dim3(kBucketThreads), args, sm_tree, s.stream));
    tree_passes = 2;
  }
  CK(cudaEventRecord(s.ev1, s.stream));
  uint64_t info[4] = {};
  CK(cudaMemcpyAsync(info, p.info, sizeof(info), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
  if (flag && info[2] >= max_sweeps) {
    pool_free(s, scratch);
    return fail(SSSP_ERR_CUDA, "dataparallel: pass numbers did not converge");
  }
  const double t0 = now_s();
  if (dist_out) CK(cudaMemcpyAsync(dist_out, s.d_dist, g->n * 8, cudaMemcpyDeviceToHost, s.stream));
  if (pred_out) CK(cudaMemcpyAsync(pred_out, s.d_pred, g->n * 8, cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  pool_free(s, scratch);
  if (rounds_out) *rounds_out = info[0];
  if (st) {
    *st = sssp_solve_stats{};
    st->transfer_in_s = g->transfer_in_s;
    st->rounds_s = ms * 1e-3;
    st->transfer_out_s = now_s() - t0;
    st->iterations = info[0];
    st->rows_read = info[1] + g->n * (tree_passes + (flag ? info[2] : 0));
    st->relax_checks = st->rows_read * rs;
    st->bytes_read = st->rows_read * rs * wb;
    st->matrix_bytes = g->matrix_bytes;
    st->weight_bytes = wb;
    st->ctas = G;
    st->shards = 1;
    st->engine = SSSP_ENGINE_DATAPARALLEL;
    fill_reference_stats(g, st);
    st->classes = (uint32_t)(flag ? info[2] : 0);  // pass-number sweeps (0: none needed)
  }
  return SSSP_OK;
}

int sssp_round_times(sssp_graph* g, uint64_t* ns_out, uint64_t cap, uint64_t* count) {
  if (!g || !count) return fail(SSSP_ERR_BAD_ARG, "null argument");
  if (g->pending) return fail(SSSP_ERR_BAD_ARG, "a launch is pending");
  if (g->wide) return fail(SSSP_ERR_UNSUPPORTED, "not available with 64-bit distances (wide engine)");
  Shard* s0 = nullptr;
  for (auto& s : g->sh)
    if (s.d_round_ns) s0 = &s;
  if (!s0) return fail(SSSP_ERR_BAD_ARG, "record_round_times was not set (or not shard 0)");
  CK(cudaSetDevice(s0->device));
  std::vector<uint64_t> t(g->n);
  CK(cudaMemcpy(t.data(), s0->d_round_ns, g->n * 8, cudaMemcpyDeviceToHost));
  uint64_t k = 0;
  while (k < g->n && t[k] != 0) ++k;
  *count = k;
  if (ns_out) std::copy(t.begin(), t.begin() + std::min(k, cap), ns_out);
  CK(cudaMemset(s0->d_round_ns, 0, g->n * 8));  // the next solve records afresh
  return SSSP_OK;
}

void* sssp_stream(sssp_graph* g, int local) {
  if (!g || local < 0 || (size_t)local >= g->sh.size()) return nullptr;
  return g->sh[(size_t)local].stream;
}

}  // extern "C"
