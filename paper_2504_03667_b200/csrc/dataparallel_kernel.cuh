// dataparallel_kernel.cuh -- the paper's data-parallel engine (PAPER.md
// Alg. 3-4), restated for B200: synchronous relaxation rounds to a fixpoint,
// then the deterministic predecessor rebuild.  Bit-identical to the
// reference's dijkstra_dataparallel (dataparallel.hpp:302-327): same dist,
// same pred (reconstruct_predecessors, :221-264), same round count.
//
// Rounds (relax_round, dataparallel.hpp:184-217).  Every round relaxes every
// edge against the round-start snapshot; the reference's atomic minimum makes
// the round's outcome schedule-independent:
//   dist_{r+1}[v] = min(dist_r[v], min_u snapshot_r[u] + w(u,v)).
// A row u whose snapshot did not change since the previous round cannot lower
// anything (its candidates were applied then), so only the FRONTIER -- the
// vertices lowered in the previous round, {source} in round 1 -- is pushed.
// That gives the same dist after every round and the same round count
// (rounds_executed counts the final round that changes nothing).  One
// cooperative launch runs all rounds: a CTA owns T matrix positions (dist in
// shared memory), pushes its slice of every frontier row, and publishes its
// lowered columns (bitmap + snapshot values) before one grid barrier per
// round.
//
// Predecessors (reconstruct_predecessors).  Vertices are attached in
// ascending (dist, id) order, each to its smallest already-attached tight
// parent, in passes until nothing changes.  Writing pass(v) for the pass in
// which v attaches, with the source attached before pass 1, v attaches in the
// first pass p in which some tight parent u (u != v, du + w(u,v) == dv) is
// attached when v is visited:  u == source, or pass(u) < p, or pass(u) == p
// and u precedes v in the order.  Hence
//   pass(v) = min over tight u of f(u),  f(source) = 1,
//             f(u) = pass(u) + [(du, u) > (dv, v)]  otherwise,
//   pred(v) = the smallest tight u with f(u) <= pass(v).
// A tight edge with w >= 1 always runs forward in the order, so without a
// zero-weight tight edge every pass is 1 and pred(v) is simply the smallest
// tight parent: one pass over the matrix (dp_tree_kernel).  Only when that
// pass finds a zero-weight tight edge between distinct vertices are the pass
// numbers solved -- a min-plus fixpoint over the tight edges, iterated to
// convergence by dp_tree_kernel<SWEEP> -- and the predecessors recomputed.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

#include "bucket_kernel.cuh"

namespace sssp_b200 {

struct DpParams {
  const void* adj;      // [n rows][row_stride] positions (the permuted matrix)
  uint64_t row_stride;  // positions per row (= Q*L)
  uint32_t n, Q, qbits, lbits, T, source;
  uint32_t* gfront;     // [2][row_stride/32] frontier bitmap by position, per round parity
  uint32_t* gcnt;       // [2][G] frontier vertices per tile
  uint32_t* gsnap;      // [2][row_stride] snapshot dist of frontier positions
  uint32_t* dist_v;     // [n] final dist by vertex id (u32, all-ones = INF)
  uint32_t* pass_v;     // [n] pass numbers (dp_pass_kernel); nullptr: every pass is 1
  uint32_t* sweep_chg;  // [max_sweeps] CTAs that changed a pass number in sweep i (zeroed)
  uint32_t max_sweeps;
  uint32_t* flag;       // [1] dp_pred_kernel: 1 if a zero-weight tight edge u != v exists
  uint64_t* dist_out;   // [n] reference encoding
  uint64_t* pred_out;   // [n]
  uint64_t* info;       // [4]: rounds, frontier rows pushed, sweeps, max finite dist (zeroed)
};

constexpr uint32_t kDpInf = 0xFFFFFFFFu;

// weight j of a 16 B chunk word (u8: one PRMT, zero-extended)
template <typename W>
__device__ __forceinline__ uint32_t dp_weight(uint32_t word, int j) {
  if constexpr (sizeof(W) == 1) return __byte_perm(word, 0u, 0x4440u + (uint32_t)(j % 4));
  else if constexpr (sizeof(W) == 2) return __byte_perm(word, 0u, (j % 2) ? 0x4432u : 0x4410u);
  else return word;
}

constexpr int kDpBatch = 8;  // rows per thread per cp.async pipeline stage
constexpr int kDpChunk = kBucketThreads * 32;  // frontier ids enumerated per pass (1 word/thread)

// Dynamic smem of dp_relax_kernel: stage[2][kDpBatch][threads] uint4 (aliased by
// the per-thread column minima once the rows are consumed) | dist[T] |
// lowered[T/32] | frontier bitmap [row_stride/32] | ids [kDpChunk].
__host__ __device__ constexpr size_t dp_relax_smem_bytes(uint32_t T, uint32_t words, uint32_t wbytes) {
  return 16ull * 2 * kDpBatch * kBucketThreads +
         4ull * (T + bucket_round4(T / 32) + bucket_round4(words) + kDpChunk) + 0 * wbytes;
}

template <typename W>
__global__ void __launch_bounds__(kBucketThreads, 2) dp_relax_kernel(const DpParams p) {
  namespace cg = cooperative_groups;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr int CPT = 16 / (int)sizeof(W);
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t T = p.T, G = gridDim.x, TW = T / 32;
  const uint32_t words = (uint32_t)(p.row_stride / 32);
  uint4* sstage = reinterpret_cast<uint4*>(smem);  // [2][kDpBatch][threads], thread-private
  uint32_t* scomb = smem;                           // aliases the stage after the rows
  uint32_t* sdist = smem + 4 * 2 * kDpBatch * kBucketThreads;
  uint32_t* slow = sdist + T;  // columns lowered this round
  uint32_t* sbm = slow + bucket_round4(TW);
  uint32_t* schunk = sbm + bucket_round4(words);
  __shared__ uint32_t s_red[kBucketThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t p0 = blockIdx.x * T;
  const W* adj = static_cast<const W*>(p.adj);
  const uint32_t TPR = T * sizeof(W) / 16, RG = kBucketThreads / TPR;
  auto vid = [&](uint32_t pos) { return pos_to_vid(pos, p.Q, p.lbits, p.qbits); };

  // ---- init (RelaxState, dataparallel.hpp:44-52): dist = INF, dist[s] = 0;
  // round 1's frontier is {source} with snapshot 0.
  for (uint32_t i = tid; i < T; i += kBucketThreads) sdist[i] = vid(p0 + i) == p.source ? 0u : kDpInf;
  __shared__ uint32_t s_src;
  if (tid == 0) s_src = 0;
  __syncthreads();
  for (uint32_t i = warp; i < TW; i += kBucketThreads / 32) {
    const uint32_t pos = p0 + i * 32 + lane;
    const uint32_t b = __ballot_sync(0xFFFFFFFFu, vid(pos) == p.source);
    if (lane == 0) p.gfront[i + blockIdx.x * TW] = b;
    if (b && lane == __ffs(b) - 1) {
      p.gsnap[pos] = 0;
      s_src = 1;
    }
  }
  __syncthreads();
  if (tid == 0) p.gcnt[blockIdx.x] = s_src;
  cg::this_grid().sync();

  uint64_t rounds = 0, pushed = 0;
  uint32_t par = 0;
  while (true) {
    // frontier of this round (published before the last barrier)
    const uint32_t* fb = p.gfront + par * words;
    for (uint32_t i = tid; i < words; i += kBucketThreads) sbm[i] = __ldcg(&fb[i]);
    uint32_t f = 0;
    for (uint32_t c = tid; c < G; c += kBucketThreads) f += __ldcg(&p.gcnt[par * G + c]);
    f = __reduce_add_sync(0xFFFFFFFFu, f);
    if (lane == 0) s_red[warp] = f;
    for (uint32_t i = tid; i < TW; i += kBucketThreads) slow[i] = 0u;
    __syncthreads();
    f = 0;
    for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) f += s_red[w2];
    if (f == 0) break;  // the previous round lowered nothing: fixpoint (uniform)
    ++rounds;
    pushed += f;
    // ---- push the frontier rows: per column min of snapshot[u] + w(u, v)
    const uint32_t rg = tid / TPR, ct = tid - rg * TPR;
    uint32_t best[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) best[j] = kDpInf;
    // u8 rows whose snapshot distance is below 0xFF00: candidates fit 16 bits,
    // two columns per VIADDMNMX.U16x2 (lanes j = 2k, 2k + 1; 0xFFFF = none)
    uint32_t best16[CPT / 2];
#pragma unroll
    for (int k = 0; k < CPT / 2; ++k) best16[k] = 0xFFFFFFFFu;
    constexpr uint32_t WPT = 1;
    for (uint32_t wbase = 0; wbase < words; wbase += kBucketThreads * WPT) {
      const uint32_t w0 = wbase + tid * WPT;
      uint32_t bw[WPT];
      uint32_t c = 0;
#pragma unroll
      for (uint32_t k2 = 0; k2 < WPT; ++k2) {
        bw[k2] = w0 + k2 < words ? sbm[w0 + k2] : 0u;
        c += __popc(bw[k2]);
      }
      if (!__syncthreads_or(c != 0)) continue;
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      if (lane == 31) s_red[warp] = incl;
      __syncthreads();
      uint32_t wofs = 0, tot = 0;
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) {
        if (w2 < warp) wofs += s_red[w2];
        tot += s_red[w2];
      }
      uint32_t o = wofs + incl - c;
#pragma unroll
      for (uint32_t k2 = 0; k2 < WPT; ++k2)
        for (uint32_t m = bw[k2]; m; m &= m - 1) schunk[o++] = (w0 + k2) * 32 + (__ffs(m) - 1);
      __syncthreads();
      const uint32_t* snap = p.gsnap + par * p.row_stride;
      // two-stage cp.async pipeline over this pass's rows: batch b+1's slices
      // stream into the thread's shared-memory slots while batch b is relaxed
      const uint32_t per_batch = kDpBatch * RG;
      const uint32_t nbatch = (tot + per_batch - 1) / per_batch;
      uint32_t du_c[kDpBatch], du_n[kDpBatch];
      auto issue = [&](uint32_t b, uint32_t* du) {
        uint4* st = sstage + (size_t)(b & 1u) * kDpBatch * kBucketThreads;
#pragma unroll
        for (int m = 0; m < kDpBatch; ++m) {
          const uint32_t r = b * per_batch + rg + m * RG;
          du[m] = kDpInf;
          if (r < tot) {
            const uint32_t pos = schunk[r];
            du[m] = __ldcg(&snap[pos]);
            cp_async16(&st[m * kBucketThreads + tid],
                       reinterpret_cast<const uint8_t*>(adj + (size_t)vid(pos) * p.row_stride + p0) +
                           ct * 16);
          }
        }
        cp_async_commit();
      };
      if (nbatch) issue(0, du_c);
      for (uint32_t b = 0; b < nbatch; ++b) {
        if (b + 1 < nbatch) issue(b + 1, du_n);
        else cp_async_commit();
        cp_async_wait<1>();
        const uint4* st = sstage + (size_t)(b & 1u) * kDpBatch * kBucketThreads;
#pragma unroll
        for (int m = 0; m < kDpBatch; ++m) {
          const uint32_t dum = du_c[m];
          du_c[m] = du_n[m];
          if (b * per_batch + rg + m * RG >= tot) break;
          const uint4 v4 = st[m * kBucketThreads + tid];
          const uint32_t wd[4] = {v4.x, v4.y, v4.z, v4.w};
          // u8 chunks without an INF byte (every chunk of a complete graph):
          // min(du + w, best) is one PRMT + one VIADDMNMX per weight
          bool inf_free = false;
          if constexpr (sizeof(W) == 1) {
            uint32_t z = 0;
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) z |= (~wd[k2] - 0x01010101u) & wd[k2] & 0x80808080u;
            inf_free = z == 0;  // no byte == 0xFF (haszero(~x))
          }
          if (sizeof(W) == 1 && inf_free && dum < 0xFF00u) {
            const uint32_t d2 = dum * 0x10001u;  // du + w <= 0xFEFF + 0xFE < 0xFFFF
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              best16[2 * q] = __viaddmin_u16x2(d2, __byte_perm(wd[q], 0u, 0x4140u), best16[2 * q]);
              best16[2 * q + 1] = __viaddmin_u16x2(d2, __byte_perm(wd[q], 0u, 0x4342u), best16[2 * q + 1]);
            }
          } else if (sizeof(W) == 1 && dum < 0xFF00u) {
            // INF bytes (0xFF): that lane's addend becomes 0xFF00, so its
            // candidate is exactly 0xFFFF ("none"); finite ones stay <= 0xFFFD
            const uint32_t d2 = dum * 0x10001u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t y = ~wd[q];
              const uint32_t ff = ~(((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y) & 0x80808080u;  // byte == 0xFF
              const uint32_t m0 = (__byte_perm(ff, 0u, 0x4140u) >> 7) * 0xFFFFu;  // lane -> 0xFFFF
              const uint32_t m1 = (__byte_perm(ff, 0u, 0x4342u) >> 7) * 0xFFFFu;
              const uint32_t a0 = (d2 & ~m0) | (0xFF00FF00u & m0), a1 = (d2 & ~m1) | (0xFF00FF00u & m1);
              best16[2 * q] = __viaddmin_u16x2(a0, __byte_perm(wd[q], 0u, 0x4140u), best16[2 * q]);
              best16[2 * q + 1] = __viaddmin_u16x2(a1, __byte_perm(wd[q], 0u, 0x4342u), best16[2 * q + 1]);
            }
          } else if (inf_free) {
#pragma unroll
            for (int j = 0; j < CPT; ++j)
              best[j] = __viaddmin_u32(dum, dp_weight<W>(wd[(j * sizeof(W)) / 4], j), best[j]);
          } else {
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
              const uint32_t w = dp_weight<W>(wd[(j * sizeof(W)) / 4], j);
              // min(du + w, best) in one VIADDMNMX; an INF weight gets the base
              // INF - WINF so its candidate is exactly INF (du + w < 2^32 - 1
              // for finite operands: host-checked n * max_w)
              const uint32_t base = w == WINF ? kDpInf - WINF : dum;
              best[j] = __viaddmin_u32(base, w, best[j]);
            }
          }
        }
      }
      cp_async_wait<0>();
      __syncthreads();
    }
    if constexpr (sizeof(W) == 1) {
#pragma unroll
      for (int k = 0; k < CPT / 2; ++k) {
        const uint32_t lo = best16[k] & 0xFFFFu, hi = best16[k] >> 16;
        if (lo != 0xFFFFu) best[2 * k] = min(best[2 * k], lo);
        if (hi != 0xFFFFu) best[2 * k + 1] = min(best[2 * k + 1], hi);
      }
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) scomb[tid * CPT + j] = best[j];
    __syncthreads();
    // ---- apply (strict '<', relax_cell :74) and publish the lowered columns
    const uint32_t nxt = par ^ 1u;
    for (uint32_t col = tid; col < T; col += kBucketThreads) {
      const uint32_t cth = col / CPT, j = col % CPT;
      uint32_t k = kDpInf;
      for (uint32_t g2 = 0; g2 < RG; ++g2) k = min(k, scomb[(g2 * TPR + cth) * CPT + j]);
      if (k < sdist[col]) {
        sdist[col] = k;
        atomicOr(&slow[col >> 5], 1u << (col & 31));
        p.gsnap[nxt * p.row_stride + p0 + col] = k;
      }
    }
    __syncthreads();
    uint32_t cnt = 0;
    for (uint32_t i = tid; i < TW; i += kBucketThreads) {
      p.gfront[nxt * words + blockIdx.x * TW + i] = slow[i];
      cnt += __popc(slow[i]);
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (lane == 0) s_red[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
      uint32_t c = 0;
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) c += s_red[w2];
      p.gcnt[nxt * G + blockIdx.x] = c;
    }
    cg::this_grid().sync();
    par = nxt;
  }
  uint32_t dmax = 0;
  for (uint32_t i = tid; i < T; i += kBucketThreads) {
    const uint32_t v = vid(p0 + i);
    if (v < p.n) {
      p.dist_v[v] = sdist[i];
      p.dist_out[v] = sdist[i] == kDpInf ? ~0ull : (uint64_t)sdist[i];
      if (sdist[i] != kDpInf) dmax = max(dmax, sdist[i]);
    }
  }
  dmax = __reduce_max_sync(0xFFFFFFFFu, dmax);
  if (lane == 0 && dmax) atomicMax(reinterpret_cast<unsigned long long*>(&p.info[3]), (unsigned long long)dmax);
  if (blockIdx.x == 0 && tid == 0) {
    p.info[0] = rounds;
    p.info[1] = pushed;
  }
}


// Dynamic smem of dp_tree_kernel: stage[2][kDpBatch][threads] uint4 | dv[T] |
// passv[T] | combine.
__host__ __device__ constexpr size_t dp_pred_smem_bytes(uint32_t T, uint32_t wbytes) {
  return 16ull * 2 * kDpBatch * kBucketThreads + 4ull * 2 * T + 4ull * kBucketThreads * (16 / wbytes);
}

// One pass over every row: pred(v) = the smallest tight u != v with
// f(u) <= pass(v) (pass_v == nullptr: every pass is 1, so every tight parent
// qualifies); flags a zero-weight tight edge between distinct vertices.
// SWEEP = true instead iterates pass(v) = min over tight u of f(u) to its
// fixpoint (cooperative launch; one grid barrier per sweep).
// FAST (non-SWEEP, u8/u16 weights, no zero weight anywhere and every finite
// dist < WINF): tight <=> w == dv - du, and an INF weight or an unreachable
// column (dv - du > WINF) can never satisfy it, so the per-weight work is one compare and a predicated
// min; only the diagonal (w(v,v) = 0 == dv - dv) needs excluding, once per
// row.  Branch-free straight-line code in the inner loops (a data-dependent
// skip there measured slower).
template <typename W, bool SWEEP, bool FAST>
__global__ void __launch_bounds__(kBucketThreads, 2) dp_tree_kernel(const DpParams p) {
  namespace cg = cooperative_groups;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr int CPT = 16 / (int)sizeof(W);
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t T = p.T;
  uint4* sstage = reinterpret_cast<uint4*>(smem);  // [2][kDpBatch][threads], thread-private slots
  uint32_t* sdv = smem + 4 * 2 * kDpBatch * kBucketThreads;
  uint32_t* spv = sdv + T;
  uint32_t* scomb = spv + T;
  const uint32_t tid = threadIdx.x;
  const uint32_t p0 = blockIdx.x * T;
  const W* adj = static_cast<const W*>(p.adj);
  const uint32_t TPR = T * sizeof(W) / 16, RG = kBucketThreads / TPR;
  const uint32_t rg = tid / TPR, ct = tid - rg * TPR;
  auto vid = [&](uint32_t pos) { return pos_to_vid(pos, p.Q, p.lbits, p.qbits); };
  for (uint32_t i = tid; i < T; i += kBucketThreads) {
    const uint32_t v = vid(p0 + i);
    sdv[i] = v < p.n ? p.dist_v[v] : kDpInf;
    spv[i] = v < p.n && p.pass_v ? p.pass_v[v] : 1u;
  }
  __syncthreads();
  // my CPT columns: consecutive positions of one participant, ids step by Q
  uint32_t cd[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) cd[j] = sdv[ct * CPT + j];
  const uint32_t cv0 = vid(p0 + ct * CPT);
  // u8 FAST: my columns' distances as 16-bit lanes (j = 2k, 2k + 1) for a
  // per-row filter; a row passes it only if some lane has w == (dv - du) mod
  // 2^16 (no false negatives), and only those rows run the exact test
  uint32_t cd2[CPT / 2];
  bool small16 = true;
#pragma unroll
  for (int k = 0; k < CPT / 2; ++k) {
    cd2[k] = (cd[2 * k] & 0xFFFFu) | (cd[2 * k + 1] << 16);
    small16 &= cd[2 * k] <= 0xFFFFu && cd[2 * k + 1] <= 0xFFFFu;
  }
  bool zero_tight = false;
  for (uint32_t sweep = 0;; ++sweep) {
    uint32_t best[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) best[j] = kDpInf;
    // two-stage pipeline: batch b+1's row slices stream into shared memory
    // (cp.async) while batch b is processed
    const uint32_t per_batch = kDpBatch * RG;
    const uint32_t nbatch = (p.n + per_batch - 1) / per_batch;
    uint32_t du_c[kDpBatch], pu_c[kDpBatch], du_n[kDpBatch], pu_n[kDpBatch];
    auto issue = [&](uint32_t b, uint32_t* du, uint32_t* pu) {
      uint4* st = sstage + (size_t)(b & 1u) * kDpBatch * kBucketThreads;
#pragma unroll
      for (int m = 0; m < kDpBatch; ++m) {
        const uint32_t u = b * per_batch + rg + m * RG;
        du[m] = u < p.n ? __ldcg(&p.dist_v[u]) : kDpInf;
        pu[m] = (!FAST && u < p.n && p.pass_v) ? __ldcg(&p.pass_v[u]) : 1u;
        if (u < p.n)
          cp_async16(&st[m * kBucketThreads + tid],
                     reinterpret_cast<const uint8_t*>(adj + (size_t)u * p.row_stride + p0) + ct * 16);
      }
      cp_async_commit();
    };
    issue(0, du_c, pu_c);
    for (uint32_t b = 0; b < nbatch; ++b) {
      if (b + 1 < nbatch) issue(b + 1, du_n, pu_n);
      else cp_async_commit();  // empty group: the wait below always leaves one group pending
      cp_async_wait<1>();
      const uint4* st = sstage + (size_t)(b & 1u) * kDpBatch * kBucketThreads;
#pragma unroll
      for (int m = 0; m < kDpBatch; ++m) {
        const uint32_t u = b * per_batch + rg + m * RG;
        const uint32_t dum = du_c[m], pum = pu_c[m];
        du_c[m] = du_n[m];
        pu_c[m] = pu_n[m];
        if (dum == kDpInf || pum == kDpInf) continue;  // unreachable, or not attached yet
        const uint4 v4 = st[m * kBucketThreads + tid];
        const uint32_t wd[4] = {v4.x, v4.y, v4.z, v4.w};
        if constexpr (FAST) {
          if constexpr (sizeof(W) == 1) {
            if (small16 && dum <= 0xFFFFu) {
              const uint32_t du2 = dum * 0x10001u;
              uint32_t any = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t x0 = __vsub2(cd2[2 * q], du2) ^ __byte_perm(wd[q], 0u, 0x4140u);
                const uint32_t x1 = __vsub2(cd2[2 * q + 1], du2) ^ __byte_perm(wd[q], 0u, 0x4342u);
                any |= ((x0 - 0x00010001u) & ~x0) | ((x1 - 0x00010001u) & ~x1);  // a zero lane
              }
              if (!(any & 0x80008000u)) continue;
            }
          }
          const uint32_t dj = u - cv0;  // row u is my column j's own vertex iff dj == j*Q
          const uint32_t jd = ((dj & (p.Q - 1)) == 0 && (dj >> p.qbits) < (uint32_t)CPT)
                                  ? (dj >> p.qbits) : (uint32_t)CPT;
#pragma unroll
          for (int j = 0; j < CPT; ++j) {
            const uint32_t w = dp_weight<W>(wd[(j * (int)sizeof(W)) / 4], j);
            if (w == cd[j] - dum && (uint32_t)j != jd) best[j] = min(best[j], u);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CPT; ++j) {
            const uint32_t w = dp_weight<W>(wd[(j * (int)sizeof(W)) / 4], j);
            const uint32_t v = cv0 + j * p.Q;
            const bool tight = w != WINF && u != v && cd[j] != kDpInf && dum + w == cd[j];
            // f(u): the pass in which v may attach to u (source: pass 1)
            const uint32_t after = (dum > cd[j] || (dum == cd[j] && u > v)) ? 1u : 0u;
            const uint32_t f = u == p.source ? 1u : pum + after;
            if (!SWEEP) {
              zero_tight |= tight && w == 0;
              if (tight && f <= spv[ct * CPT + j]) best[j] = min(best[j], u);  // smallest qualifying parent
            } else {
              if (tight) best[j] = min(best[j], f);
            }
          }
        }
      }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < CPT; ++j) scomb[tid * CPT + j] = best[j];
    __syncthreads();
    if (!SWEEP) {
      for (uint32_t col = tid; col < T; col += kBucketThreads) {
        const uint32_t cth = col / CPT, j = col % CPT;
        uint32_t k = kDpInf;
        for (uint32_t g2 = 0; g2 < RG; ++g2) k = min(k, scomb[(g2 * TPR + cth) * CPT + j]);
        const uint32_t v = vid(p0 + col);
        if (v < p.n) p.pred_out[v] = (k == kDpInf || v == p.source) ? ~0ull : (uint64_t)k;
      }
      if (__syncthreads_or(zero_tight) && tid == 0) atomicOr(p.flag, 1u);
      return;
    }
    // SWEEP: lower pass(v); count the CTAs that changed anything this sweep
    bool changed = false;
    for (uint32_t col = tid; col < T; col += kBucketThreads) {
      const uint32_t cth = col / CPT, j = col % CPT;
      uint32_t k = kDpInf;
      for (uint32_t g2 = 0; g2 < RG; ++g2) k = min(k, scomb[(g2 * TPR + cth) * CPT + j]);
      const uint32_t v = vid(p0 + col);
      if (v < p.n && v != p.source && k < spv[col]) {
        spv[col] = k;
        p.pass_v[v] = k;  // read by other CTAs this or next sweep (monotone: any order converges)
        changed = true;
      }
    }
    if (__syncthreads_or(changed) && tid == 0) atomicAdd(&p.sweep_chg[sweep], 1u);
    cg::this_grid().sync();
    if (__ldcg(&p.sweep_chg[sweep]) == 0 || sweep + 1 >= p.max_sweeps) {
      if (blockIdx.x == 0 && tid == 0) p.info[2] = sweep + 1;
      return;
    }
  }
}

}  // namespace sssp_b200
