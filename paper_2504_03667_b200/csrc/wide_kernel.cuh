// wide_kernel.cuh -- the reference's full value domain: 64-bit distances.
//
// The narrow engines hold distances in 32 bits, which covers every graph whose
// n * max_weight stays below 2^32 - 1 (all BASELINE configs).  The reference
// accepts any finite weight up to kMaxWeight = 2^32 - 1 (weight.hpp:18,
// graph.hpp:79) and sums them in uint64 (add_weight, weight.hpp:23-26), so a
// graph with a weight of exactly 2^32 - 1, or with n * max_weight >= 2^32 - 1,
// runs here: weights stay in the narrowest type that holds them (uint64 when a
// weight equals 2^32 - 1, since INF must stay distinct), distances are uint64
// with INF = UINT64_MAX exactly as in the reference.
//
// One thread-block cluster of C CTAs per solve runs the serial engine's n
// rounds (serial.hpp:41-61) in one launch:
//  * CTA r owns the C-th share of the row positions [r*PC, (r+1)*PC) of the
//    cyclic layout (position p = q*L + s <-> vertex s*Q + q); dist (u64), pred
//    and visited live in its shared memory, each position owned by one thread
//    for the whole solve (no intra-CTA hazards on the state);
//  * election (serial.hpp:42-48): lexicographic (dist, vertex) minimum per
//    CTA, written into every cluster CTA's exchange slot through DSMEM, one
//    cluster barrier, every CTA reduces the C candidates itself (the redundant
//    allreduce of partitioned.hpp:94-101); ties go to the lowest vertex id;
//  * relaxation (serial.hpp:51-60): strict '<', pred = the elected vertex.
// The loop stops at the first INF election: every later round of the
// reference elects an unreachable vertex and relaxes nothing.
#pragma once

#include <cstdint>

#include "scan_kernel.cuh"

namespace sssp_b200 {

template <>
struct WInf<uint64_t> {
  static constexpr uint64_t v = ~0ull;
};

constexpr int kWideThreads = 256;

struct WideParams {
  const void* adj;       // n rows x row_stride positions (cyclic layout), W elements
  uint64_t row_stride;   // Q * L positions
  uint32_t n;
  uint32_t Q, lbits, qbits;  // position p <-> vertex ((p & (L-1)) << qbits) | (p >> lbits)
  uint32_t C;            // CTAs per cluster (= per solve)
  uint32_t PC;           // positions per CTA (row_stride / C)
  const uint32_t* sources;  // [nsolve]
  uint64_t* dist_out;    // [nsolve][n]
  uint64_t* pred_out;    // [nsolve][n]
  uint32_t* visit_order; // optional [nsolve][n]
  uint64_t* info;        // [nsolve][4]: iterations (elections of finite vertices)
};

__host__ __device__ constexpr size_t wide_smem_bytes(uint32_t PC) {
  return (size_t)PC * (8 + 4 + 1);
}

__device__ __forceinline__ uint32_t wide_vid(uint32_t pos, uint32_t lbits, uint32_t qbits) {
  return ((pos & ((1u << lbits) - 1u)) << qbits) | (pos >> lbits);
}

// lexicographic (dist, vertex) minimum
__device__ __forceinline__ void wide_lexmin(uint64_t& d, uint32_t& v, uint64_t d2, uint32_t v2) {
  if (d2 < d || (d2 == d && v2 < v)) {
    d = d2;
    v = v2;
  }
}

template <typename W>
__global__ void __launch_bounds__(kWideThreads) wide_kernel(const WideParams p) {
  constexpr uint64_t DINF = ~0ull;
  constexpr uint64_t WINF = (uint64_t)WInf<W>::v;
  extern __shared__ __align__(16) uint8_t wsm[];
  uint64_t* sdist = reinterpret_cast<uint64_t*>(wsm);
  uint32_t* spred = reinterpret_cast<uint32_t*>(sdist + p.PC);
  uint8_t* svis = reinterpret_cast<uint8_t*>(spred + p.PC);
  __shared__ uint64_t s_xd[2][16];  // exchange slots, written by every cluster CTA (DSMEM)
  __shared__ uint32_t s_xv[2][16];
  __shared__ uint64_t s_wd[kWideThreads / 32];
  __shared__ uint32_t s_wv[kWideThreads / 32];

  uint32_t rank, solve_idx;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  solve_idx = blockIdx.x / p.C;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t p0 = rank * p.PC;
  const uint32_t source = p.sources[solve_idx];
  const W* adj = static_cast<const W*>(p.adj);

  // init (serial.hpp:32-36); padding positions are visited from the start
  for (uint32_t i = tid; i < p.PC; i += kWideThreads) {
    const uint32_t v = wide_vid(p0 + i, p.lbits, p.qbits);
    sdist[i] = v == source ? 0ull : DINF;
    spred[i] = 0xFFFFFFFFu;
    svis[i] = v >= p.n ? 1 : 0;
  }
  // every CTA of the cluster has started (DSMEM targets exist) and initialised
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  uint32_t iters = 0;
  for (uint32_t round = 0; round < p.n; ++round) {
    const uint32_t par = round & 1u;
    // ---- local (dist, vertex) minimum over unvisited owned positions
    uint64_t bd = DINF;
    uint32_t bv = 0xFFFFFFFFu;
    for (uint32_t i = tid; i < p.PC; i += kWideThreads)
      if (!svis[i]) wide_lexmin(bd, bv, sdist[i], wide_vid(p0 + i, p.lbits, p.qbits));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t d2 = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
      const uint32_t v2 = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
      wide_lexmin(bd, bv, d2, v2);
    }
    if (lane == 0) {
      s_wd[warp] = bd;
      s_wv[warp] = bv;
    }
    __syncthreads();
    if (warp == 0) {
      bd = lane < kWideThreads / 32 ? s_wd[lane] : DINF;
      bv = lane < kWideThreads / 32 ? s_wv[lane] : 0xFFFFFFFFu;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        const uint64_t d2 = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
        const uint32_t v2 = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
        wide_lexmin(bd, bv, d2, v2);
      }
      // publish this CTA's candidate into slot [par][rank] of every cluster CTA
      if (lane < p.C) {
        const uint32_t a_d = (uint32_t)__cvta_generic_to_shared(&s_xd[par][rank]);
        const uint32_t a_v = (uint32_t)__cvta_generic_to_shared(&s_xv[par][rank]);
        uint32_t r_d, r_v;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_d) : "r"(a_d), "r"(lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_v) : "r"(a_v), "r"(lane));
        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(r_d), "l"(bd) : "memory");
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(r_v), "r"(bv) : "memory");
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // ---- the winner (allreduce_minloc): every thread reduces the C slots
    uint64_t du = DINF;
    uint32_t u = 0xFFFFFFFFu;
    for (uint32_t c = 0; c < p.C; ++c) wide_lexmin(du, u, s_xd[par][c], s_xv[par][c]);
    if (du == DINF) break;  // the rest is unreachable: later rounds relax nothing
    ++iters;
    if (p.visit_order && rank == 0 && tid == 0) p.visit_order[(size_t)solve_idx * p.n + round] = u;
    // ---- relax row u over the owned positions (strict '<', serial.hpp:56)
    const uint32_t upos = (u % p.Q) << p.lbits | (u / p.Q);  // inverse of wide_vid
    const W* row = adj + (size_t)u * p.row_stride + p0;
    for (uint32_t i = tid; i < p.PC; i += kWideThreads) {
      if (p0 + i == upos) svis[i] = 1;  // the elected vertex is mine
      const uint64_t w = (uint64_t)row[i];
      if (!svis[i] && w != WINF) {
        const uint64_t c = du + w;  // du <= (n-1)(2^32-1), no uint64 overflow
        if (c < sdist[i]) {
          sdist[i] = c;
          spred[i] = u;
        }
      }
    }
  }
  // ---- write back (positions -> vertex ids)
  for (uint32_t i = tid; i < p.PC; i += kWideThreads) {
    const uint32_t v = wide_vid(p0 + i, p.lbits, p.qbits);
    if (v < p.n) {
      p.dist_out[(size_t)solve_idx * p.n + v] = sdist[i];
      p.pred_out[(size_t)solve_idx * p.n + v] = spred[i] == 0xFFFFFFFFu ? ~0ull : (uint64_t)spred[i];
    }
  }
  if (rank == 0 && tid == 0) p.info[(size_t)solve_idx * 4] = iters;
  // no CTA may exit while a peer can still write into its exchange slots
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace sssp_b200
