// nccl_kernel.cuh -- the host-driven comparison path of SURVEY.md §8e.
//
// The reference's partitioned round (partitioned.hpp:142-154): local_min
// (:81-90) -> allreduce_minloc (:94-101) -> relax_owned (:106-119), with the
// allreduce done the conventional way: one ncclAllReduce(MIN) of an 8-byte
// key per round issued by the host between two kernel launches.  The
// product path does the same exchange with device-initiated P2P stores inside
// one persistent kernel; this path exists to put a number on that choice.
//
// Key: (dist << 32 | global vertex) with the sign bit flipped, so that the
// signed int64 MIN that NCCL / torch.distributed offer orders it exactly like
// the unsigned (dist, vertex) pair: lowest dist, then lowest id
// (MinLocPair, partitioned.hpp:21-26).  INF = dist field 0xFFFFFFFF; a shard
// with no unvisited column contributes the all-ones key (the reference's
// (INF, padded_n) sentinel, :82).
#pragma once

#include <cstdint>

#include "scan_kernel.cuh"

namespace sssp_b200 {

constexpr uint64_t kNcclSign = 1ull << 63;
constexpr int kNcclMinThreads = 1024;

struct NcclRoundParams {
  const void* adj;      // this shard's matrix, cyclic position layout (scan_kernel.cuh)
  uint64_t row_stride;  // positions per row
  uint32_t npos;        // positions of the shard (= row_stride)
  uint32_t Q, lbits, qbits;
  uint32_t loc_n, col_base, n;
  uint32_t* dist;       // [npos] u32, INF = 0xFFFFFFFF
  uint32_t* pred;       // [npos]
  uint8_t* visited;     // [npos]
};

__device__ __forceinline__ uint32_t nccl_vid(const NcclRoundParams& p, uint32_t pos) {
  return ((pos & ((1u << p.lbits) - 1u)) << p.qbits) | (pos >> p.lbits);
}

// state init (serial.hpp:32-36): dist INF, pred NONE, padding visited
__global__ void nccl_init_kernel(const NcclRoundParams p, uint32_t source) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.npos; i += gridDim.x * blockDim.x) {
    const uint32_t v = nccl_vid(p, i);
    const bool real = v < p.loc_n && p.col_base + v < p.n;
    p.dist[i] = real && p.col_base + v == source ? 0u : 0xFFFFFFFFu;
    p.pred[i] = 0xFFFFFFFFu;
    p.visited[i] = real ? 0 : 1;
  }
}

// local_min (partitioned.hpp:81-90): one CTA scans the shard's unvisited
// columns and writes the sign-flipped packed key.
__global__ void __launch_bounds__(kNcclMinThreads) nccl_local_min_kernel(const NcclRoundParams p,
                                                                        uint64_t* key_out) {
  __shared__ uint64_t s_k[kNcclMinThreads / 32];
  uint64_t best = ~0ull;
  for (uint32_t i = threadIdx.x; i < p.npos; i += kNcclMinThreads) {
    if (p.visited[i]) continue;
    const uint64_t k = ((uint64_t)p.dist[i] << 32) | (p.col_base + nccl_vid(p, i));
    best = k < best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t x = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    best = x < best ? x : best;
  }
  if ((threadIdx.x & 31) == 0) s_k[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kNcclMinThreads / 32; ++w) best = s_k[w] < best ? s_k[w] : best;
    *key_out = best ^ kNcclSign;
  }
}

// relax_owned (partitioned.hpp:106-119) with the allreduced winner: mark it
// visited if owned, relax its row over the shard's columns (strict '<').
template <typename W>
__global__ void nccl_relax_kernel(const NcclRoundParams p, const uint64_t* key) {
  const uint64_t k = *key ^ kNcclSign;
  const uint32_t du = (uint32_t)(k >> 32), u = (uint32_t)k;
  if (k == ~0ull) return;  // every shard exhausted
  const W* row = static_cast<const W*>(p.adj) + (size_t)u * p.row_stride;
  constexpr uint32_t WINF = WInf<W>::v;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.npos; i += gridDim.x * blockDim.x) {
    const uint32_t v = p.col_base + nccl_vid(p, i);
    if (v == u) p.visited[i] = 1;
    if (p.visited[i] || du == 0xFFFFFFFFu) continue;
    const uint32_t w = row[i];
    if (w == WINF) continue;
    const uint32_t c = du + w;  // < 2^32 - 1: n * max_w fits the narrow encoding
    if (c < p.dist[i]) {
      p.dist[i] = c;
      p.pred[i] = u;
    }
  }
}

// positions -> the shard's vertex order, reference encoding
__global__ void nccl_out_kernel(const NcclRoundParams p, uint64_t* dist_out, uint64_t* pred_out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.npos; i += gridDim.x * blockDim.x) {
    const uint32_t v = nccl_vid(p, i);
    if (v < p.loc_n && p.col_base + v < p.n) {
      dist_out[v] = p.dist[i] == 0xFFFFFFFFu ? ~0ull : p.dist[i];
      pred_out[v] = p.pred[i] == 0xFFFFFFFFu ? ~0ull : p.pred[i];
    }
  }
}

}  // namespace sssp_b200
