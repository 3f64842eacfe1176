// cluster_kernel.cuh -- the cluster-resident persistent Dijkstra kernel.
//
// Same algorithm, layout and key protocol as scan_kernel.cuh (read that
// header first), but one solve lives in ONE thread-block cluster of C CTAs
// x NW warps (C <= 16, non-portable size) and the per-round election is
// exchanged through distributed shared memory instead of L2:
//
//  * participant q = cta_rank*NW + warp owns local columns {s*Q + q}, Q = C*NW
//    (the cyclic layout of scan_kernel.cuh with G = Q);
//  * every warp reduces its (dist, vertex) key with redux.sync and stores the
//    tagged key into slot q of EVERY CTA's shared-memory exchange array
//    (mapa + st.shared::cluster: one DSMEM store per destination CTA);
//  * every warp polls its own CTA's array with ld.shared (no L2 round trip)
//    until all Q keys carry this round's tag, and reduces them itself.
//
// A DSMEM store + local poll costs a few hundred cycles where the grid-wide
// L2 exchange of scan_kernel.cuh measured ~1 us per round (profiles/), so a
// 16-SM cluster beats the 128-SM grid on every configured size, and
// independent solves (batched sources) simply occupy more clusters without
// any inter-cluster synchronisation.
//
// With P > 1 shards (one per GPU) the cluster minimum of the local columns
// is published to every shard's global mailbox by P2P store (NVLink), and the
// global winner is the minimum over the P mailbox keys: the allreduce_minloc
// of partitioned.hpp:94-101.
#pragma once

#include "scan_kernel.cuh"

namespace sssp_b200 {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void st_dsmem(uint32_t local_addr, uint32_t cta, uint64_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(cta));
  asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(remote), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_smem_pair(uint32_t addr, uint64_t& hi) {
  uint64_t lo;
  asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];"
               : "=l"(lo), "=l"(hi)
               : "r"(addr)
               : "memory");
  return lo;
}

// Per-lane column state.  PACKED (the common case, chosen on the host when
// (n*max_w + 1) < 2^(32-SB)) keeps ONE 32-bit register per column:
//   ek = ((dist << SB) | slot) + 1   unvisited, finite dist
//   ek = 0xFFFFFFFF                  unvisited, dist = INF
//   ek = 0                           visited (elected)
// so that  relax    : improve iff  w != INF  and  cand + 1 < ek   (a visited
//                     column can never improve: 0 is the minimum), and
//          election : min over (ek - 1) puts visited columns (0 - 1 = MAX)
//                     last and orders the rest by (dist, slot) = (dist, vertex).
// The +1 keeps the encoding monotone; finite keys stay below 2^32 - 2^SB.
// Without PACKED, dist and a visited mask are kept apart and the election is
// a 2-stage redux (dist, then slot).
// TRACE: record %globaltimer at every round end (record_round_times); a
// separate instance because even an untaken trace branch in the round loop
// cost ~4 % of the solve (18.6 vs 17.85 ms at n=32768)
template <typename W, int EPL, int NW, bool PACKED, bool TRACE = false, bool MS = false>
__global__ void __launch_bounds__(NW * 32, 1) cluster_scan_kernel(const __grid_constant__ ScanLaunch LA) {
  SSSP_LAUNCH_SHARD(MS, LA, p, bid);
  using Row = RowSlice<W, EPL>;
  constexpr int NP = NW / 4;  // key pairs per lane: Q <= 16*NW = 64*NP
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t DINF = 0xFFFFFFFFu;
  constexpr uint32_t L = 32u * EPL;
  constexpr uint32_t SB = (L == 128 ? 7 : L == 256 ? 8 : L == 512 ? 9 : 10);
  constexpr uint32_t QMAX = 16u * NW;
  static_assert(NW >= 4 && NW % 4 == 0, "NW must be a multiple of 4");
  static_assert((1u << SB) == L, "L must be a power of two");

  extern __shared__ uint32_t s_pred[];  // [NW][L], dynamic (up to 64 KB)
  __shared__ __align__(16) uint64_t s_keys[2][QMAX];

  const int lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t cr = cluster_ctarank();
  const uint32_t csize = cluster_nctarank();
  const uint32_t Q = p.G;             // = csize * NW, a power of two
  const uint32_t qbits = 31u - __clz(Q);
  const uint32_t solve = bid / csize;
  const uint32_t q = cr * NW + warp;
  const uint32_t tb = 32u - p.vbits;
  const uint64_t tagmask = (1ull << tb) - 1ull;
  const uint32_t vmask_all = (p.vbits >= 32) ? 0xFFFFFFFFu : ((1u << p.vbits) - 1u);
  const bool multi = p.nshards > 1;
  const W* const adj = static_cast<const W*>(p.adj) + (size_t)q * L;
  const bool pf_reg = (p.flags & kFlagPrefetchReg) != 0;
  const bool pf_l2 = (p.flags & kFlagPrefetchL2) != 0;
  uint32_t* const pred = s_pred + warp * L;
  uint64_t* const dout = p.dist_out + (size_t)solve * p.loc_n;
  uint64_t* const pout = p.pred_out + (size_t)solve * p.loc_n;
  // lane's slot of element e is  ebase(e) | lbase  (disjoint bit fields)
  const uint32_t lbase = (uint32_t)lane * Row::VEC;

  // ---- init (serial.hpp:32-36)
  const uint32_t source = p.sources[solve];
  uint32_t ek[EPL];  // PACKED state
  uint32_t d[EPL];   // !PACKED state
  uint64_t vis = 0;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t s = Row::slot(e, lane);
    const uint32_t vl = (s << qbits) | q;
    const bool pad = vl >= p.loc_n || p.col_base + vl >= p.n;
    const bool src = !pad && p.col_base + vl == source;
    if constexpr (PACKED) {
      ek[e] = pad ? 0u : src ? s + 1u : DINF;
    } else {
      d[e] = src ? 0u : DINF;
      if (pad) vis |= (1ull << e);
    }
  }
  for (uint32_t i = lane; i < L; i += 32) pred[i] = 0xFFFFFFFFu;
  for (uint32_t i = threadIdx.x; i < 2 * QMAX; i += NW * 32) (&s_keys[0][0])[i] = 0;
  cluster_sync_all();  // every exchange array is zeroed before anyone publishes

  uint32_t u = source, du = 0;
  uint64_t E = p.exch_base;
  uint64_t iters = 0, mispredicts = 0;
  uint32_t pred_u = 0xFFFFFFFFu;
  Row cur, nxt;
  cur.load(adj + (size_t)u * p.row_stride, lane);
  uint64_t ks[2 * NP];
#pragma unroll
  for (int j = 0; j < 2 * NP; ++j) ks[j] = ~0ull;
  uint64_t best_key = 0;
  const uint64_t t_start = globaltimer();
  bool failed = false;
  const uint32_t keys_base = (uint32_t)__cvta_generic_to_shared(&s_keys[0][0]);

  // Polls round E's keys (own smem), then with P > 1 exchanges the cluster
  // minimum through the P2P mailbox.  Returns false if the watchdog fired.
  auto gather = [&](uint32_t buf, uint64_t want) -> bool {
    const uint32_t arr = keys_base + buf * QMAX * 8u;
    const uint32_t want32 = (uint32_t)want;
    const uint32_t tm32 = (uint32_t)tagmask;
    uint32_t polls = 0;
    while (true) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const uint32_t i = 2u * lane + 64u * j;
        if (i < Q) {  // Q is even (NW >= 4)
          uint64_t hi;
          const uint64_t lo = ld_smem_pair(arr + i * 8u, hi);
          ks[2 * j] = lo;
          ks[2 * j + 1] = hi;
          ok &= (((uint32_t)lo & tm32) == want32) & (((uint32_t)hi & tm32) == want32);
        } else {
          ks[2 * j] = ks[2 * j + 1] = ~0ull;
        }
      }
      if (__all_sync(0xFFFFFFFFu, ok)) break;
      if ((++polls & 1023u) == 0 && globaltimer() - t_start > p.timeout_ns) return false;
    }
    best_key = min_key<NP>(ks);
    if (multi) {
      if (q == 0 && (uint32_t)lane < p.nshards)
        st_slot(p.peer_slots[lane] + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride +
                    p.shard,
                best_key, true);
      const uint64_t* mb = p.slots + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride;
      uint64_t mk = ~0ull;
      uint32_t polls2 = 0;
      while (true) {
        mk = (uint32_t)lane < p.nshards ? ld_slot(mb + lane, true) : ~0ull;
        const bool ok = (uint32_t)lane >= p.nshards || (mk & tagmask) == want;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
        if ((++polls2 & 1023u) == 0 && globaltimer() - t_start > p.timeout_ns) return false;
      }
      uint32_t a = (uint32_t)(mk >> 32), b = (uint32_t)mk;
      warp_lexmin(a, b);
      best_key = ((uint64_t)a << 32) | b;
    }
    return true;
  };

  // smallest gathered key strictly greater than `after` (keys are unique)
  auto next_key = [&](uint64_t after) -> uint64_t {
    uint64_t r = ~0ull;
#pragma unroll
    for (int j = 0; j < 2 * NP; ++j) r = (ks[j] > after && ks[j] < r) ? ks[j] : r;
    uint32_t a = (uint32_t)(r >> 32), b = (uint32_t)r;
    warp_lexmin(a, b);
    return ((uint64_t)a << 32) | b;
  };
  // L2-prefetch this warp's slice of a row that is needed two rounds ahead
  auto prefetch_slice = [&](uint32_t v) {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(adj + (size_t)v * p.row_stride);
#pragma unroll
    for (int k = 0; k < Row::NCH; ++k)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(b + (size_t)(k * 32 + lane) * Row::CB));
  };

  if (PACKED && (p.flags & kFlagSpeculate)) {
    // Speculative loop.  While round E's exchange is in flight, each warp
    // already relaxes the row of the PREDICTED winner of round E (the
    // runner-up of round E-1) into a shadow state eks[] and
    // elects from it.  When round E resolves to exactly that (vertex, dist),
    // the shadow state is committed and the precomputed key is published at
    // once, so the relax + election cost hides behind the exchange latency;
    // otherwise the round is recomputed from the committed state.  Results
    // are identical either way.
    uint32_t eks[EPL];
    uint32_t spec_u = 0xFFFFFFFFu, spec_du = 0, spec_bd = DINF, spec_bv = vmask_all;
    uint64_t spec_pm = 0;  // columns the speculative relax improved
    // two-slot row ring: the row for this round's speculation, and the row of
    // the vertex predicted two rounds ahead (third-best key), in flight
    Row ra = cur, rb;
    uint32_t ra_u = u, rb_u = 0xFFFFFFFFu;

    auto owner_of = [&](uint32_t v, uint32_t& ul) -> bool {
      ul = v - p.col_base;
      return v >= p.col_base && ul < p.loc_n && (ul & (Q - 1)) == q;
    };
    // zero the element of `arr` holding local column ul (owner warp only)
    auto mark = [&](uint32_t (&arr)[EPL], uint32_t ul) -> bool {
      const uint32_t su = ul >> qbits;
      if ((uint32_t)lane != ((su / Row::VEC) & 31u)) return false;
      const uint32_t eu = (su / (32u * Row::VEC)) * Row::VEC + su % Row::VEC;
#pragma unroll
      for (int e = 0; e < EPL; ++e)
        if ((uint32_t)e == eu) arr[e] = 0u;
      return true;
    };
    auto elect = [&](const uint32_t (&arr)[EPL], uint32_t& bd, uint32_t& bv) {
      uint32_t k = 0xFFFFFFFFu;
#pragma unroll
      for (int e = 0; e < EPL; ++e) k = min(k, arr[e] - 1u);
      k = __reduce_min_sync(0xFFFFFFFFu, k);
      const bool none = k >= 0xFFFFFFFEu || (k >> SB) == (DINF >> SB);
      bd = none ? DINF : (k >> SB);
      bv = none ? vmask_all : (p.col_base + (((k & (L - 1u)) << qbits) | q));
    };

    // One round.  A = the slot holding the row predicted for this round's
    // speculation (loaded one round ago), B = the slot this round loads the
    // two-rounds-ahead row into.  The loop alternates the roles, so every
    // load targets a fixed register set (a runtime-selected load target would
    // force the compiler to wait for the load right away).
    // Returns 0 = continue, 1 = solve finished, 2 = watchdog fired.
    auto step = [&](Row& A, uint32_t& A_u, Row& B, uint32_t& B_u) -> int {
      uint32_t bd, bv;
      const bool hit = (u == spec_u) && (du == spec_du);
      if (hit) {
        bd = spec_bd;
        bv = spec_bv;
      } else {
        // ---- recompute this round from the committed state
        if (u == B_u) {
          cur = B;
        } else if (u == A_u) {
          cur = A;
        } else {
          if (iters > 0) ++mispredicts;
          cur.load(adj + (size_t)u * p.row_stride, lane);
        }
        uint32_t ul;
        if (owner_of(u, ul) && mark(ek, ul)) dout[ul] = du;
        const uint32_t dus1 = (du << SB) + 1u + lbase;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const uint32_t w = cur.elem(e);
          const uint32_t nk = w * L + dus1 + (Row::slot(e, 0));
          if (w != WINF && nk < ek[e]) {
            ek[e] = nk;
            pred[Row::slot(e, 0) | lbase] = u;
          }
        }
        elect(ek, bd, bv);
      }

      // ---- publish (DSMEM) -- the only work between gather and publish on a hit
      ++E;
      const uint32_t buf = (uint32_t)(E & 1ull);
      const uint64_t want = E & tagmask;
      const uint64_t key = ((uint64_t)bd << 32) | ((uint64_t)(bv & vmask_all) << tb) | want;
      if ((uint32_t)lane < csize) st_dsmem(keys_base + (buf * QMAX + q) * 8u, (uint32_t)lane, key);

      // ---- commit the speculation's side effects
      if (hit) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) ek[e] = eks[e];
#pragma unroll
        for (int e = 0; e < EPL; ++e)
          if ((spec_pm >> e) & 1ull) pred[Row::slot(e, 0) | lbase] = u;
        uint32_t ul;
        if (owner_of(u, ul)) {
          const uint32_t su = ul >> qbits;
          if ((uint32_t)lane == ((su / Row::VEC) & 31u)) dout[ul] = du;
        }
      }
      ++iters;
      if (p.visit_order != nullptr && p.shard == 0 && q == 0 && lane == 0)
        p.visit_order[(size_t)solve * p.n + (iters - 1)] = u;
      if constexpr (TRACE)
        if (p.round_ns != nullptr && solve == 0 && p.shard == 0 && q == 0 && lane == 0)
          p.round_ns[iters - 1] = globaltimer();  // per-round latency trace
      // ---- speculate on the next round: runner-up of the last exchange
      spec_u = 0xFFFFFFFFu;
      const uint64_t r2 = next_key(best_key);
      if (pf_reg && iters > 1 && (uint32_t)(r2 >> 32) != DINF) {
        spec_u = (uint32_t)(r2 & 0xFFFFFFFFull) >> tb;
        spec_du = (uint32_t)(r2 >> 32);
        if (spec_u != A_u && spec_u != B_u) {
          ++mispredicts;
          A.load(adj + (size_t)spec_u * p.row_stride, lane);
          A_u = spec_u;
        }
        const Row sr = (spec_u == B_u) ? B : A;
#pragma unroll
        for (int e = 0; e < EPL; ++e) eks[e] = ek[e];
        uint32_t ul;
        if (owner_of(spec_u, ul)) mark(eks, ul);
        const uint32_t dus1 = (spec_du << SB) + 1u + lbase;
        uint64_t pm = 0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const uint32_t w = sr.elem(e);
          const uint32_t nk = w * L + dus1 + (Row::slot(e, 0));
          if (w != WINF && nk < eks[e]) {
            eks[e] = nk;
            pm |= 1ull << e;
          }
        }
        spec_pm = pm;
        elect(eks, spec_bd, spec_bv);
        // two rounds ahead: the third-best key's row into slot B
        const uint64_t r3 = next_key(r2);
        if ((uint32_t)(r3 >> 32) != DINF) {
          const uint32_t v3 = (uint32_t)(r3 & 0xFFFFFFFFull) >> tb;
          if (v3 != A_u && v3 != B_u && spec_u != B_u) {
            B.load(adj + (size_t)v3 * p.row_stride, lane);
            B_u = v3;
          }
        }
      }

      // ---- gather round E
      if (!gather(buf, want)) return 2;
      du = (uint32_t)(best_key >> 32);
      if (du == DINF) return 1;
      u = (uint32_t)(best_key & 0xFFFFFFFFull) >> tb;
      return 0;
    };

    int st = 0;
    while (st == 0) {
      st = step(rb, rb_u, ra, ra_u);
      if (st == 0) st = step(ra, ra_u, rb, rb_u);
    }
    failed = st == 2;
  } else {
    while (true) {
      // ---- the owner of u marks it visited and records its final distance
      {
        const uint32_t ul = u - p.col_base;
        if (u >= p.col_base && ul < p.loc_n && (ul & (Q - 1)) == q) {
          const uint32_t su = ul >> qbits;
          if ((uint32_t)lane == ((su / Row::VEC) & 31u)) {
            const uint32_t eu = (su / (32u * Row::VEC)) * Row::VEC + su % Row::VEC;
  #pragma unroll
            for (int e = 0; e < EPL; ++e)
              if ((uint32_t)e == eu) {
                if constexpr (PACKED) ek[e] = 0u;
                else vis |= (1ull << e);
              }
            dout[ul] = du;
          }
        }
      }
      // ---- relax row u (serial.hpp:51-60; strict '<' keeps the earliest parent)
      if constexpr (PACKED) {
        const uint32_t dus1 = (du << SB) + 1u + lbase;
  #pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const uint32_t w = cur.elem(e);
          const uint32_t nk = w * L + dus1 + (Row::slot(e, 0));
          if (w != WINF && nk < ek[e]) {
            ek[e] = nk;
            pred[Row::slot(e, 0) | lbase] = u;
          }
        }
      } else {
  #pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const uint32_t w = cur.elem(e);
          const uint32_t nd = du + w;
          if (w != WINF && nd < d[e] && !((vis >> e) & 1ull)) {
            d[e] = nd;
            pred[Row::slot(e, 0) | lbase] = u;
          }
        }
      }
      ++iters;
      if (p.visit_order != nullptr && p.shard == 0 && q == 0 && lane == 0)
        p.visit_order[(size_t)solve * p.n + (iters - 1)] = u;
      if constexpr (TRACE)
        if (p.round_ns != nullptr && solve == 0 && p.shard == 0 && q == 0 && lane == 0)
          p.round_ns[iters - 1] = globaltimer();  // per-round latency trace

      // ---- warp election (serial.hpp:42-48)
      uint32_t bd, bs;
      if constexpr (PACKED) {
        uint32_t k = 0xFFFFFFFFu;
  #pragma unroll
        for (int e = 0; e < EPL; ++e) k = min(k, ek[e] - 1u);
        k = __reduce_min_sync(0xFFFFFFFFu, k);
        const bool none = k >= 0xFFFFFFFEu || (k >> SB) == (DINF >> SB);
        bd = none ? DINF : (k >> SB);
        bs = k & (L - 1u);
      } else {
        bd = DINF;
        bs = 0xFFFFFFFFu;
  #pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const bool live = !((vis >> e) & 1ull) && d[e] != DINF;
          if (live && d[e] < bd) {
            bd = d[e];
            bs = Row::slot(e, lane);
          }
        }
        warp_lexmin(bd, bs);
      }
      const uint32_t bv = (bd == DINF) ? vmask_all : (p.col_base + ((bs << qbits) | q));

      // ---- publish into every CTA's exchange array (DSMEM)
      ++E;
      const uint32_t buf = (uint32_t)(E & 1ull);
      const uint64_t want = E & tagmask;
      const uint64_t key = ((uint64_t)bd << 32) | ((uint64_t)(bv & vmask_all) << tb) | want;
      const uint32_t my_slot_addr = keys_base + (buf * QMAX + q) * 8u;
      if ((uint32_t)lane < csize) st_dsmem(my_slot_addr, (uint32_t)lane, key);

      // ---- off the critical path, while the exchange is in flight: the
      // runner-up of the last exchange (the likely next winner, SURVEY.md
      // §8d) into registers, the third-best row's slice into L2.
      if (pf_reg) {
        const uint64_t r2 = next_key(best_key);
        if ((uint32_t)(r2 >> 32) != DINF && iters > 1) {
          pred_u = (uint32_t)(r2 & 0xFFFFFFFFull) >> tb;
          nxt.load(adj + (size_t)pred_u * p.row_stride, lane);
          if (pf_l2) {
            const uint64_t r3 = next_key(r2);
            if ((uint32_t)(r3 >> 32) != DINF) prefetch_slice((uint32_t)(r3 & 0xFFFFFFFFull) >> tb);
          }
        } else {
          pred_u = 0xFFFFFFFFu;
        }
      }

      if (!gather(buf, want)) {
        failed = true;
        break;
      }

      du = (uint32_t)(best_key >> 32);
      if (du == DINF) break;
      u = (uint32_t)(best_key & 0xFFFFFFFFull) >> tb;
      if (pf_reg && u == pred_u) {
        cur = nxt;
      } else {
        if (pf_reg) ++mispredicts;
        cur.load(adj + (size_t)u * p.row_stride, lane);
      }
    }
  }

  // ---- write back: unvisited columns are unreachable; pred from smem
  __syncwarp();
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t s = Row::slot(e, lane);
    const uint32_t vl = (s << qbits) | q;
    if (vl < p.loc_n && p.col_base + vl < p.n) {
      bool visited;
      if constexpr (PACKED) visited = ek[e] == 0u;
      else visited = (vis >> e) & 1ull;
      if (!visited) dout[vl] = ~0ull;
      const uint32_t pr = pred[s];
      pout[vl] = pr == 0xFFFFFFFFu ? ~0ull : (uint64_t)pr;
    }
  }
  uint64_t* inf = p.info + (size_t)solve * 4;
  if (failed && lane == 0) atomicOr((unsigned long long*)(inf + 2), 1ull);
  if (q == 0 && lane == 0) {
    inf[0] = iters;
    inf[1] = E;
    inf[3] = mispredicts;
  }
  cluster_sync_all();  // no CTA leaves while a peer could still address its smem
}

// Hierarchical variant (flag kFlagHier): each CTA first reduces its NW warp
// keys through shared memory (one named barrier), and only the C CTA minima
// are all-gathered over DSMEM -- C stores per CTA per round instead of C*NW,
// and C keys to poll (ubench: a 16-participant DSMEM all-gather costs ~380
// cycles vs ~590 for 64).  Participant q = warp*C + cta_rank, so consecutive
// vertex ids fall on consecutive CTAs and the runner-up CTA minimum is still
// the likely next winner.  PACKED state only (the host falls back otherwise).
template <typename W, int EPL, int NW, bool MS = false>
__global__ void __launch_bounds__(NW * 32, 1) cluster_hier_kernel(const __grid_constant__ ScanLaunch LA) {
  SSSP_LAUNCH_SHARD(MS, LA, p, bid);
  using Row = RowSlice<W, EPL>;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t DINF = 0xFFFFFFFFu;
  constexpr uint32_t L = 32u * EPL;
  constexpr uint32_t SB = (L == 128 ? 7 : L == 256 ? 8 : L == 512 ? 9 : 10);
  static_assert((1u << SB) == L, "L must be a power of two");

  extern __shared__ uint32_t s_pred[];  // [NW][L]
  __shared__ __align__(16) uint64_t s_keys[2][16];   // CTA minima of the round, by CTA rank
  __shared__ __align__(16) uint64_t s_wk[2][NW];     // warp keys of this CTA

  const int lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t cr = cluster_ctarank();
  const uint32_t csize = cluster_nctarank();
  const uint32_t Q = p.G;  // = csize * NW, a power of two
  const uint32_t qbits = 31u - __clz(Q);
  const uint32_t solve = bid / csize;
  const uint32_t q = warp * csize + cr;
  const uint32_t tb = 32u - p.vbits;
  const uint64_t tagmask = (1ull << tb) - 1ull;
  const uint32_t vmask_all = (p.vbits >= 32) ? 0xFFFFFFFFu : ((1u << p.vbits) - 1u);
  const bool multi = p.nshards > 1;
  const W* const adj = static_cast<const W*>(p.adj) + (size_t)q * L;
  const bool pf_reg = (p.flags & kFlagPrefetchReg) != 0;
  const bool pf_l2 = (p.flags & kFlagPrefetchL2) != 0;
  uint32_t* const pred = s_pred + warp * L;
  uint64_t* const dout = p.dist_out + (size_t)solve * p.loc_n;
  uint64_t* const pout = p.pred_out + (size_t)solve * p.loc_n;
  const uint32_t lbase = (uint32_t)lane * Row::VEC;

  const uint32_t source = p.sources[solve];
  uint32_t ek[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t s = Row::slot(e, lane);
    const uint32_t vl = (s << qbits) | q;
    const bool pad = vl >= p.loc_n || p.col_base + vl >= p.n;
    ek[e] = pad ? 0u : (p.col_base + vl == source) ? s + 1u : DINF;
  }
  for (uint32_t i = lane; i < L; i += 32) pred[i] = 0xFFFFFFFFu;
  for (uint32_t i = threadIdx.x; i < 2 * 16; i += NW * 32) (&s_keys[0][0])[i] = 0;
  cluster_sync_all();

  uint32_t u = source, du = 0;
  uint64_t E = p.exch_base, iters = 0, mispredicts = 0;
  uint32_t pred_u = 0xFFFFFFFFu;
  Row cur, nxt;
  cur.load(adj + (size_t)u * p.row_stride, lane);
  uint64_t ck = ~0ull;  // this lane's gathered CTA key (lanes < csize)
  uint64_t best_key = 0;
  const uint64_t t_start = globaltimer();
  bool failed = false;
  const uint32_t keys_base = (uint32_t)__cvta_generic_to_shared(&s_keys[0][0]);

  auto next_key = [&](uint64_t after) -> uint64_t {
    const uint64_t r = (ck > after) ? ck : ~0ull;
    uint32_t a = (uint32_t)(r >> 32), b = (uint32_t)r;
    warp_lexmin(a, b);
    return ((uint64_t)a << 32) | b;
  };

  while (true) {
    // ---- owner marks u visited, records its final distance
    {
      const uint32_t ul = u - p.col_base;
      if (u >= p.col_base && ul < p.loc_n && (ul & (Q - 1)) == q) {
        const uint32_t su = ul >> qbits;
        if ((uint32_t)lane == ((su / Row::VEC) & 31u)) {
          const uint32_t eu = (su / (32u * Row::VEC)) * Row::VEC + su % Row::VEC;
#pragma unroll
          for (int e = 0; e < EPL; ++e)
            if ((uint32_t)e == eu) ek[e] = 0u;
          dout[ul] = du;
        }
      }
    }
    // ---- relax (serial.hpp:51-60)
    {
      const uint32_t dus1 = (du << SB) + 1u + lbase;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const uint32_t w = cur.elem(e);
        const uint32_t nk = w * L + dus1 + (Row::slot(e, 0));
        if (w != WINF && nk < ek[e]) {
          ek[e] = nk;
          pred[Row::slot(e, 0) | lbase] = u;
        }
      }
    }
    ++iters;
    if (p.visit_order != nullptr && p.shard == 0 && q == 0 && lane == 0)
      p.visit_order[(size_t)solve * p.n + (iters - 1)] = u;

    // ---- warp election, then the CTA minimum through shared memory
    ++E;
    const uint32_t buf = (uint32_t)(E & 1ull);
    const uint64_t want = E & tagmask;
    {
      uint32_t k = 0xFFFFFFFFu;
#pragma unroll
      for (int e = 0; e < EPL; ++e) k = min(k, ek[e] - 1u);
      k = __reduce_min_sync(0xFFFFFFFFu, k);
      const bool none = k >= 0xFFFFFFFEu || (k >> SB) == (DINF >> SB);
      const uint32_t bd = none ? DINF : (k >> SB);
      const uint32_t bv = none ? vmask_all : (p.col_base + (((k & (L - 1u)) << qbits) | q));
      if (lane == 0) s_wk[buf][warp] = ((uint64_t)bd << 32) | ((uint64_t)(bv & vmask_all) << tb);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    if (warp == 0) {
      uint64_t m = (uint32_t)lane < NW ? s_wk[buf][lane] : ~0ull;
      uint32_t a = (uint32_t)(m >> 32), b = (uint32_t)m;
      warp_lexmin(a, b);
      const uint64_t key = ((uint64_t)a << 32) | b | want;
      // ---- publish the CTA minimum into every CTA's exchange array (DSMEM)
      if ((uint32_t)lane < csize) st_dsmem(keys_base + (buf * 16 + cr) * 8u, (uint32_t)lane, key);
    }

    // ---- off the critical path: runner-up row into registers, third into L2
    if (pf_reg) {
      const uint64_t r2 = next_key(best_key);
      if ((uint32_t)(r2 >> 32) != DINF && iters > 1) {
        pred_u = (uint32_t)(r2 & 0xFFFFFFFFull) >> tb;
        nxt.load(adj + (size_t)pred_u * p.row_stride, lane);
        if (pf_l2) {
          const uint64_t r3 = next_key(r2);
          if ((uint32_t)(r3 >> 32) != DINF) {
            const uint32_t v3 = (uint32_t)(r3 & 0xFFFFFFFFull) >> tb;
            const uint8_t* b3 = reinterpret_cast<const uint8_t*>(adj + (size_t)v3 * p.row_stride);
#pragma unroll
            for (int k2 = 0; k2 < Row::NCH; ++k2)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(b3 + (size_t)(k2 * 32 + lane) * Row::CB));
          }
        }
      } else {
        pred_u = 0xFFFFFFFFu;
      }
    }

    // ---- gather the C CTA minima from my own shared memory
    {
      const uint32_t addr = keys_base + (buf * 16 + (uint32_t)lane) * 8u;
      const uint32_t want32 = (uint32_t)want, tm32 = (uint32_t)tagmask;
      uint32_t polls = 0;
      while (true) {
        uint64_t v = ~0ull;
        if ((uint32_t)lane < csize)
          asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
        const bool ok = (uint32_t)lane >= csize || (((uint32_t)v & tm32) == want32);
        if (__all_sync(0xFFFFFFFFu, ok)) {
          ck = (uint32_t)lane < csize ? (v & ~tagmask) : ~0ull;
          break;
        }
        if ((++polls & 1023u) == 0 && globaltimer() - t_start > p.timeout_ns) {
          failed = true;
          break;
        }
      }
    }
    if (failed) break;
    {
      uint32_t a = (uint32_t)(ck >> 32), b = (uint32_t)ck;
      warp_lexmin(a, b);
      best_key = ((uint64_t)a << 32) | b;
    }
    if (multi) {
      const uint64_t tagged = best_key | want;
      if (q == 0 && (uint32_t)lane < p.nshards)
        st_slot(p.peer_slots[lane] + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride +
                    p.shard,
                tagged, true);
      const uint64_t* mb = p.slots + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride;
      uint64_t mk = ~0ull;
      uint32_t polls = 0;
      while (true) {
        mk = (uint32_t)lane < p.nshards ? ld_slot(mb + lane, true) : ~0ull;
        const bool ok = (uint32_t)lane >= p.nshards || (mk & tagmask) == want;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
        if ((++polls & 1023u) == 0 && globaltimer() - t_start > p.timeout_ns) {
          failed = true;
          break;
        }
      }
      if (failed) break;
      mk = (uint32_t)lane < p.nshards ? (mk & ~tagmask) : ~0ull;
      uint32_t a = (uint32_t)(mk >> 32), b = (uint32_t)mk;
      warp_lexmin(a, b);
      best_key = ((uint64_t)a << 32) | b;
    }
    du = (uint32_t)(best_key >> 32);
    if (du == DINF) break;
    u = (uint32_t)(best_key & 0xFFFFFFFFull) >> tb;
    if (pf_reg && u == pred_u) {
      cur = nxt;
    } else {
      if (pf_reg) ++mispredicts;
      cur.load(adj + (size_t)u * p.row_stride, lane);
    }
  }

  __syncwarp();
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t s = Row::slot(e, lane);
    const uint32_t vl = (s << qbits) | q;
    if (vl < p.loc_n && p.col_base + vl < p.n) {
      if (ek[e] != 0u) dout[vl] = ~0ull;
      const uint32_t pr = pred[s];
      pout[vl] = pr == 0xFFFFFFFFu ? ~0ull : (uint64_t)pr;
    }
  }
  uint64_t* inf = p.info + (size_t)solve * 4;
  if (failed && lane == 0) atomicOr((unsigned long long*)(inf + 2), 1ull);
  if (q == 0 && lane == 0) {
    inf[0] = iters;
    inf[1] = E;
    inf[3] = mispredicts;
  }
  cluster_sync_all();
}

// t_sync microbenchmark for the cluster exchange (same code, no relax).
// HIER = the hierarchical variant: named barrier, warp 0 publishes the CTA
// key, every warp polls the C CTA keys.
template <int NW, bool HIER = false, bool MS = false>
__global__ void __launch_bounds__(NW * 32, 1) cluster_probe_kernel(const __grid_constant__ ScanLaunch LA,
                                                                  uint32_t rounds,
                                                                  uint64_t* out_ns) {
  SSSP_LAUNCH_SHARD(MS, LA, p, bid);
  constexpr int NP = NW / 4;
  constexpr uint32_t QMAX = 16u * NW;
  __shared__ __align__(16) uint64_t s_keys[2][QMAX];
  __shared__ __align__(16) uint64_t s_wk[2][NW];
  const int lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t cr = cluster_ctarank();
  const uint32_t csize = cluster_nctarank();
  const uint32_t Q = HIER ? csize : p.G;  // participants of the DSMEM exchange
  const uint32_t solve = bid / csize;
  const uint32_t q = HIER ? cr : cr * NW + warp;
  const uint32_t tb = 32u - p.vbits;
  const uint64_t tagmask = (1ull << tb) - 1ull;
  const bool multi = p.nshards > 1;
  for (uint32_t i = threadIdx.x; i < 2 * QMAX; i += NW * 32) (&s_keys[0][0])[i] = 0;
  cluster_sync_all();
  const uint32_t keys_base = (uint32_t)__cvta_generic_to_shared(&s_keys[0][0]);
  uint64_t ks[2 * NP];
  uint64_t E = p.exch_base, acc = 0;
  const uint64_t t0 = globaltimer();
  bool failed = false;
  for (uint32_t r = 0; r < rounds && !failed; ++r) {
    ++E;
    const uint32_t buf = (uint32_t)(E & 1ull);
    const uint64_t want = E & tagmask;
    const uint32_t dist = (r * 2654435761u + (cr * NW + warp) * 40503u) >> 20;
    uint64_t key = ((uint64_t)dist << 32) | ((uint64_t)(p.shard * p.G + cr * NW + warp) << tb);
    if (HIER) {
      if (lane == 0) s_wk[buf][warp] = key;
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
      if (warp == 0) {
        uint64_t m = (uint32_t)lane < NW ? s_wk[buf][lane] : ~0ull;
        uint32_t a = (uint32_t)(m >> 32), b = (uint32_t)m;
        warp_lexmin(a, b);
        key = ((uint64_t)a << 32) | b | want;
        if ((uint32_t)lane < csize) st_dsmem(keys_base + (buf * QMAX + q) * 8u, (uint32_t)lane, key);
      }
    } else {
      key |= want;
      if ((uint32_t)lane < csize) st_dsmem(keys_base + (buf * QMAX + q) * 8u, (uint32_t)lane, key);
    }
    const uint32_t arr = keys_base + buf * QMAX * 8u;
    uint32_t polls = 0;
    while (true) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const uint32_t i = 2u * lane + 64u * j;
        if (i < Q) {
          uint64_t hi;
          const uint64_t lo = ld_smem_pair(arr + i * 8u, hi);
          ks[2 * j] = lo;
          ok &= (lo & tagmask) == want;
          ks[2 * j + 1] = i + 1 < Q ? hi : ~0ull;
          if (i + 1 < Q) ok &= (hi & tagmask) == want;
        } else {
          ks[2 * j] = ks[2 * j + 1] = ~0ull;
        }
      }
      if (__all_sync(0xFFFFFFFFu, ok)) break;
      if ((++polls & 1023u) == 0 && globaltimer() - t0 > p.timeout_ns) {
        failed = true;
        break;
      }
    }
    if (failed) break;
    uint64_t best = min_key<NP>(ks);
    if (multi) {
      if (cr == 0 && warp == 0 && (uint32_t)lane < p.nshards)
        st_slot(p.peer_slots[lane] + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride +
                    p.shard,
                best, true);
      const uint64_t* mb = p.slots + (uint64_t)solve * p.slot_stride + (uint64_t)buf * p.bstride;
      uint32_t polls2 = 0;
      uint64_t mk;
      while (true) {
        mk = (uint32_t)lane < p.nshards ? ld_slot(mb + lane, true) : ~0ull;
        const bool ok = (uint32_t)lane >= p.nshards || (mk & tagmask) == want;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
        if ((++polls2 & 1023u) == 0 && globaltimer() - t0 > p.timeout_ns) {
          failed = true;
          break;
        }
      }
      uint32_t a = (uint32_t)(mk >> 32), b = (uint32_t)mk;
      warp_lexmin(a, b);
      best = ((uint64_t)a << 32) | b;
    }
    acc += best >> 32;
  }
  if (cr == 0 && warp == 0 && lane == 0) {
    out_ns[lsh_ + solve] = failed ? ~0ull : globaltimer() - t0;
    p.info[solve * 4 + 1] = E;
    p.info[solve * 4 + 0] = acc;
  }
  cluster_sync_all();
}

}  // namespace sssp_b200
