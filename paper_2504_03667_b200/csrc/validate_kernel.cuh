// validate_kernel.cuh -- validate_result (oracle.hpp:51-120) on the device.
//
// The reference's harness refuses to time a result that fails validation
// (bench.hpp:167-173).  These kernels run the same checks against the
// device-resident matrix, so a drop-in harness can validate without a CPU
// O(n^2) pass:
//   * source has dist 0 and no predecessor,
//   * relaxation fixpoint over every finite edge (no dist[u] + w < dist[v]),
//   * every reachable vertex's predecessor edge exists and is tight,
//   * unreachable vertices have no predecessor,
//   * predecessor chains reach the source (pointer jumping, log2(n) rounds).
// Distances/preds are the reference encoding (uint64, UINT64_MAX = INF/NONE),
// indexed by global vertex id.
#pragma once

#include <cstdint>

#include "scan_kernel.cuh"

namespace sssp_b200 {

// One CTA-stride over (row u, local position p) cells of this shard.
template <typename W>
__global__ void validate_edges_kernel(const W* __restrict__ a, uint64_t n, uint64_t row_stride,
                                      uint64_t col_base, uint64_t cols, uint32_t G, uint32_t L,
                                      const uint64_t* __restrict__ dist,
                                      unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  const uint64_t total = n * row_stride;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = idx / row_stride;
    const uint32_t q = (uint32_t)(idx - u * row_stride);
    const uint32_t c = q / L, sl = q - c * L;
    const uint64_t vl = (uint64_t)sl * G + c;
    if (vl >= cols) continue;
    const uint32_t w = a[idx];
    const uint64_t du = dist[u];
    if (w == WInf<W>::v || du == ~0ull) continue;
    if (du + w < dist[col_base + vl]) ++local;  // not a fixpoint (oracle.hpp:71-80)
  }
  if (local) atomicAdd(bad, local);
}

// Per owned vertex: source checks, predecessor existence and tightness
// (oracle.hpp:65-104).
template <typename W>
__global__ void validate_pred_kernel(const W* __restrict__ a, uint64_t n, uint64_t row_stride,
                                     uint64_t col_base, uint64_t cols, uint32_t G, uint32_t L,
                                     uint64_t source, const uint64_t* __restrict__ dist,
                                     const uint64_t* __restrict__ pred,
                                     unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  for (uint64_t vl = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; vl < cols;
       vl += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = col_base + vl;
    const uint64_t dv = dist[v], pv = pred[v];
    if (v == source) {
      local += (dv != 0) + (pv != ~0ull);
      continue;
    }
    if (dv == ~0ull) {
      local += pv != ~0ull;
      continue;
    }
    if (pv >= n) {
      ++local;
      continue;
    }
    const uint64_t pos = (vl % G) * L + vl / G;
    const uint32_t w = a[pv * row_stride + pos];
    if (w == WInf<W>::v || dist[pv] == ~0ull || dist[pv] + w != dv) ++local;
  }
  if (local) atomicAdd(bad, local);
}

// Pointer jumping: jump[v] = pred[v] for reachable non-source v, else v.
__global__ void chain_init_kernel(const uint64_t* __restrict__ dist,
                                  const uint64_t* __restrict__ pred, uint64_t n, uint64_t source,
                                  uint64_t* __restrict__ jump) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    jump[v] = (v == source || dist[v] == ~0ull || pred[v] >= n) ? v : pred[v];
}

__global__ void chain_jump_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                  uint64_t n) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = in[in[v]];
}

// A reachable vertex whose chain does not end at the source (oracle.hpp:106-118).
__global__ void chain_check_kernel(const uint64_t* __restrict__ dist,
                                   const uint64_t* __restrict__ jump, uint64_t n, uint64_t source,
                                   unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    if (v != source && dist[v] != ~0ull && jump[v] != source) ++local;
  if (local) atomicAdd(bad, local);
}

}  // namespace sssp_b200
