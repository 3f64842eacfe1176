// scan_kernel.cuh -- the persistent sm_100a matrix-scan Dijkstra kernel.
//
// One launch runs a whole solve (or a batch of independent solves): the
// reference's n-round loop (serial.hpp:41-61; partitioned.hpp:147-153)
// becomes a loop inside the kernel.  Layout and protocol:
//
//  * A shard owns loc_n consecutive global columns [col_base, col_base+loc_n)
//    (partition.hpp:31-41).  Inside a shard the columns are dealt CYCLICALLY
//    to G single-warp CTAs: CTA c owns local columns {s*G + c : s < L}, and
//    the matrix row is stored permuted so that CTA c's L columns are one
//    contiguous, 16B-aligned run: row u, CTA c, slot s -> adj[u*stride + c*L + s].
//    Consecutive vertex ids therefore land on different CTAs, which is what
//    makes the next few elections predictable from other CTAs' candidates.
//  * dist lives in registers (EPL per lane), pred in shared memory, visited
//    in a per-lane bitmask.  Nothing but the matrix row touches HBM.
//  * Election (serial.hpp:42-48, MinLocPair partitioned.hpp:21-26): every CTA
//    reduces its (dist, vertex) minimum with redux.sync, then publishes one
//    tagged 64-bit key  [dist:32 | vertex:VB | tag:32-VB]  into a slot of every
//    shard's exchange array (flag-in-data: no atomics, no barrier, no reset).
//    Every CTA polls the whole array of P*G keys until all carry this
//    exchange's tag and reduces them itself (the redundant allreduce of
//    partitioned.hpp:168).  Keys order by (dist, vertex) because all valid
//    keys share the tag bits, so ties go to the lowest vertex id exactly as
//    the serial scan's strict '<' does.
//  * Relaxation (serial.hpp:51-60, relax_owned partitioned.hpp:106-119):
//    strict '<', pred = elected vertex.
//  * The elected row slice is normally already in registers: after
//    publishing, each CTA computes the runner-up key of the previous exchange
//    and loads that row while it waits (the runner-up is the
//    next winner in >99.9% of rounds), and the owner of each local minimum
//    prefetches that vertex's full row into L2 with cp.async.bulk.prefetch.
#pragma once

#include <cstdint>

namespace sssp_b200 {

constexpr int kMaxShards = 8;

struct ScanParams {
  const void* adj;          // shard matrix (W elements), permuted layout
  uint64_t row_stride;      // elements per stored row (= G*L)
  uint32_t n;               // global vertex count (real)
  uint32_t G;               // CTAs per solve on this shard
  uint32_t col_base;        // global id of this shard's first column
  uint32_t loc_n;           // columns owned by this shard (partition plan)
  uint32_t vbits;           // vertex bits in the exchange key
  uint32_t shard;           // this shard's index k
  uint32_t nshards;         // P
  uint32_t packed;          // 1: (dist << sbits | slot) fits 32 bits
  uint32_t sbits;           // log2(L)
  uint32_t flags;           // kFlag* below
  uint64_t* slots;          // local exchange array, [nsolve][2][P*G]
  uint64_t* peer_slots[kMaxShards];  // every shard's exchange array (self included)
  uint64_t slot_stride;     // words per solve in an exchange array (= 2*nrep*bstride)
  uint32_t bstride;         // words per replica (P*G rounded up to 16 = one 128 B line)
  uint32_t nrep;            // replicas of every buffer; CTA c polls replica c % nrep
  uint64_t exch_base;       // first exchange index of this launch
  const uint32_t* sources;  // [nsolve] global source ids
  uint32_t nsolve;
  uint64_t* dist_out;       // [nsolve][loc_n]
  uint64_t* pred_out;       // [nsolve][loc_n]
  uint32_t* visit_order;    // optional [nsolve][n], shard 0 only
  uint64_t* round_ns;       // optional [n]: %globaltimer at every round end (cluster engine, TRACE instances)
  uint64_t* info;           // [nsolve][4]: iterations, last exchange, error, mispredicts
                            // (error word is OR-ed by any CTA that times out)
  uint64_t timeout_ns;
};

// One launch carries every shard that lives on the launching device: blocks
// [i*bps, (i+1)*bps) run local shard i.  Shards of one device therefore never
// wait on a separate kernel that CUDA is free not to co-schedule (ncu replay,
// CUDA_LAUNCH_BLOCKING, MPS); only shards on other devices / processes are
// separate launches.
struct ScanLaunch {
  ScanParams sh[kMaxShards];
  uint32_t nlocal;  // shards in this launch
  uint32_t bps;     // blocks per shard (solves x CTAs per solve)
};

// Kernel preamble: this block's shard parameters and its block index within
// the shard (`bid` replaces blockIdx.x in the kernels).  MS (a template
// constant) = the launch may carry several shards; the single-shard instances
// index sh[0] statically, so every parameter stays an immediate constant-bank
// operand in the round loop (a runtime index costs an LDC per use: the n-round
// kernel measured 18.8 vs 17.9 ms at n=32768).
#define SSSP_LAUNCH_SHARD(MS, LA, p, bid)                       \
  const uint32_t lsh_ = (MS) ? blockIdx.x / (LA).bps : 0u;     \
  const ScanParams& p = (LA).sh[(MS) ? lsh_ : 0u];             \
  const uint32_t bid = blockIdx.x - lsh_ * (LA).bps

constexpr uint32_t kFlagPrefetchReg = 1u;  // runner-up row into registers
constexpr uint32_t kFlagPrefetchL2 = 2u;   // owner L2 prefetch of local-best rows
constexpr uint32_t kFlagSpeculate = 4u;    // cluster engine: speculative relax of the runner-up
constexpr uint32_t kFlagHier = 8u;         // cluster engine: CTA pre-reduction, C-key exchange

template <typename W>
struct WInf;
template <>
struct WInf<uint8_t> {
  static constexpr uint32_t v = 0xFFu;
};
template <>
struct WInf<uint16_t> {
  static constexpr uint32_t v = 0xFFFFu;
};
template <>
struct WInf<uint32_t> {
  static constexpr uint32_t v = 0xFFFFFFFFu;
};

__device__ __forceinline__ uint64_t ld_slot_pair(const uint64_t* p, uint64_t& hi, bool sys) {
  uint64_t lo;
  if (sys)
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
  return lo;
}

__device__ __forceinline__ uint64_t ld_slot(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_slot(uint64_t* p, uint64_t v, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Lexicographic warp minimum of (a, b): redux.sync on a, then on b among the
// lanes holding the minimal a.
__device__ __forceinline__ void warp_lexmin(uint32_t& a, uint32_t& b) {
  const uint32_t ma = __reduce_min_sync(0xFFFFFFFFu, a);
  const uint32_t mb = __reduce_min_sync(0xFFFFFFFFu, a == ma ? b : 0xFFFFFFFFu);
  a = ma;
  b = mb;
}

// Loads one lane's share of a row slice: NCH chunks of CB bytes each.
template <int CB>
struct Chunk;
template <>
struct Chunk<16> {
  uint4 v;
  __device__ __forceinline__ void load(const uint8_t* p) {
    v = __ldg(reinterpret_cast<const uint4*>(p));
  }
  __device__ __forceinline__ uint32_t word(int i) const {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
};
template <>
struct Chunk<8> {
  uint2 v;
  __device__ __forceinline__ void load(const uint8_t* p) {
    v = __ldg(reinterpret_cast<const uint2*>(p));
  }
  __device__ __forceinline__ uint32_t word(int i) const { return i == 0 ? v.x : v.y; }
};
template <>
struct Chunk<4> {
  uint32_t v;
  __device__ __forceinline__ void load(const uint8_t* p) {
    v = __ldg(reinterpret_cast<const uint32_t*>(p));
  }
  __device__ __forceinline__ uint32_t word(int) const { return v; }
};

template <typename W, int EPL>
struct RowSlice {
  static constexpr int kBytes = EPL * (int)sizeof(W);         // per lane
  static constexpr int CB = kBytes >= 16 ? 16 : kBytes;        // chunk bytes
  static constexpr int VEC = CB / (int)sizeof(W);              // elements per chunk
  static constexpr int NCH = EPL / VEC;
  Chunk<CB> ch[NCH];

  // rowp = start of this CTA's L-element slice of the row
  __device__ __forceinline__ void load(const W* rowp, int lane) {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(rowp);
#pragma unroll
    for (int k = 0; k < NCH; ++k) ch[k].load(b + (size_t)(k * 32 + lane) * CB);
  }
  __device__ __forceinline__ uint32_t elem(int e) const {
    const int k = e / VEC, j = e % VEC;
    const uint32_t w = ch[k].word((j * (int)sizeof(W)) / 4);
    if (sizeof(W) == 4) return w;
    const int sh = ((j * (int)sizeof(W)) % 4) * 8;
    return (w >> sh) & WInf<W>::v;
  }
  // slot index of element e for this lane (ascending in e)
  __device__ __forceinline__ static uint32_t slot(int e, int lane) {
    return (uint32_t)((e / VEC) * 32 * VEC + lane * VEC + (e % VEC));
  }
};



// Flag-in-data publish: lane j stores the key into replica j % nrep of shard
// j / nrep's exchange array (an NVLink P2P store for a remote shard).
__device__ __forceinline__ void publish_key(const ScanParams& p, uint64_t* my_slots,
                                            uint32_t solve, uint32_t c, int lane, uint32_t buf,
                                            uint64_t key, bool multi) {
  // Every buffer is replicated nrep times so that at most ceil(G/nrep)
  // pollers share an L2 line (one line hammered by all G pollers serialises
  // in its L2 slice and was the dominant cost of a round).
  const uint64_t slot_off = (uint64_t)buf * p.nrep * p.bstride + (uint64_t)p.shard * p.G + c;
  const uint32_t fan = p.nshards * p.nrep;
  for (uint32_t j = lane; j < fan; j += 32) {
    const uint32_t dst = j / p.nrep, rep = j - dst * p.nrep;
    uint64_t* base = multi ? p.peer_slots[dst] + (uint64_t)solve * p.slot_stride : my_slots;
    st_slot(base + slot_off + (uint64_t)rep * p.bstride, key, multi);
  }
}

// Polls the nslot keys of one exchange buffer until all carry tag `want`
// (relaxed loads: each 8-byte key is single-copy atomic and is the only
// payload).  Returns false if the watchdog fired.
template <int NP>
__device__ __forceinline__ bool gather_keys(const ScanParams& p, const uint64_t* arr,
                                            uint32_t nslot, int lane, uint64_t want,
                                            uint64_t tagmask, bool multi, uint64_t t_start,
                                            uint64_t (&ks)[2 * NP]) {
  uint32_t polls = 0;
  while (true) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const uint32_t i = 2u * lane + 64u * j;
      if (i < nslot) {
        uint64_t hi;
        const uint64_t lo = ld_slot_pair(arr + i, hi, multi);
        ks[2 * j] = lo;
        ok &= (lo & tagmask) == want;
        if (i + 1 < nslot) {
          ks[2 * j + 1] = hi;
          ok &= (hi & tagmask) == want;
        } else {
          ks[2 * j + 1] = ~0ull;
        }
      } else {
        ks[2 * j] = ks[2 * j + 1] = ~0ull;
      }
    }
    if (__all_sync(0xFFFFFFFFu, ok)) return true;
    if ((++polls & 255u) == 0 && globaltimer() - t_start > p.timeout_ns) return false;
  }
}

// Warp-wide minimum of the gathered keys: (dist, vertex) lexicographic.
template <int NP>
__device__ __forceinline__ uint64_t min_key(const uint64_t (&ks)[2 * NP]) {
  uint64_t kmin = ~0ull;
#pragma unroll
  for (int j = 0; j < 2 * NP; ++j) kmin = ks[j] < kmin ? ks[j] : kmin;
  uint32_t a = (uint32_t)(kmin >> 32), b = (uint32_t)kmin;
  warp_lexmin(a, b);
  return ((uint64_t)a << 32) | b;
}

// t_sync microbenchmark: the same launch shape and the same publish/gather
// code as the solve, with the relaxation and local election removed.  Each
// CTA publishes a synthetic key per round; out_ns[solve] = elapsed ns.
template <int NP, bool MS = false>
__global__ void __launch_bounds__(32, 1) exchange_probe_kernel(const __grid_constant__ ScanLaunch LA,
                                                               uint32_t rounds,
                                                               uint64_t* out_ns) {
  SSSP_LAUNCH_SHARD(MS, LA, p, bid);
  const int lane = threadIdx.x;
  const uint32_t solve = bid / p.G;
  const uint32_t c = bid - solve * p.G;
  const uint32_t nslot = p.nshards * p.G;
  const uint32_t tb = 32u - p.vbits;
  const uint64_t tagmask = (1ull << tb) - 1ull;
  const bool multi = p.nshards > 1;
  uint64_t* const my_slots = p.slots + (uint64_t)solve * p.slot_stride;
  uint64_t ks[2 * NP];
  uint64_t E = p.exch_base;
  const uint64_t t0 = globaltimer();
  uint64_t acc = 0;
  bool failed = false;
  for (uint32_t r = 0; r < rounds; ++r) {
    ++E;
    const uint32_t buf = (uint32_t)(E & 1ull);
    const uint64_t want = E & tagmask;
    const uint32_t dist = (r * 2654435761u + c * 40503u) >> 20;
    const uint64_t key = ((uint64_t)dist << 32) | ((uint64_t)(p.shard * p.G + c) << tb) | want;
    publish_key(p, my_slots, solve, c, lane, buf, key, multi);
    if (!gather_keys<NP>(p, my_slots + ((uint64_t)buf * p.nrep + c % p.nrep) * p.bstride, nslot,
                         lane, want, tagmask, multi, t0, ks)) {
      failed = true;
      break;
    }
    acc += min_key<NP>(ks) >> 32;
  }
  if (c == 0 && lane == 0) {
    out_ns[lsh_ + solve] = failed ? ~0ull : globaltimer() - t0;
    p.info[solve * 4 + 1] = E;
    p.info[solve * 4 + 0] = acc;  // keeps the reduction live
  }
}

// NP = pairs of exchange slots each lane reads (P*G <= 64*NP).
template <typename W, int EPL, int NP, bool MS = false>
__global__ void __launch_bounds__(32, 1) scan_dijkstra_kernel(const __grid_constant__ ScanLaunch LA) {
  SSSP_LAUNCH_SHARD(MS, LA, p, bid);
  using Row = RowSlice<W, EPL>;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t DINF = 0xFFFFFFFFu;
  constexpr uint32_t L = 32u * EPL;
  static_assert(EPL <= 64, "visited mask is 64 bits");

  __shared__ uint32_t s_pred[L];

  const int lane = threadIdx.x;
  const uint32_t G = p.G;
  const uint32_t solve = bid / G;
  const uint32_t c = bid - solve * G;
  const uint32_t nslot = p.nshards * G;
  const uint32_t tb = 32u - p.vbits;
  const uint64_t tagmask = (1ull << tb) - 1ull;
  const uint32_t vmask_all = (p.vbits >= 32) ? 0xFFFFFFFFu : ((1u << p.vbits) - 1u);
  const bool multi = p.nshards > 1;
  uint64_t* const my_slots = p.slots + (uint64_t)solve * p.slot_stride;
  const W* const adj = static_cast<const W*>(p.adj) + (size_t)c * L;
  const uint32_t row_bytes = (uint32_t)(p.row_stride * sizeof(W));
  const bool pf_reg = (p.flags & kFlagPrefetchReg) != 0;
  const bool pf_l2 = (p.flags & kFlagPrefetchL2) != 0;

  // ---- init (serial.hpp:32-36): dist = INF, pred = NONE, padding visited.
  const uint32_t source = p.sources[solve];
  uint32_t d[EPL];
  uint64_t vis = 0;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t vl = Row::slot(e, lane) * G + c;
    d[e] = (p.col_base + vl == source && vl < p.loc_n) ? 0u : DINF;  // serial.hpp:35
    if (vl >= p.loc_n || p.col_base + vl >= p.n) vis |= (1ull << e);
  }
  for (uint32_t i = lane; i < L; i += 32) s_pred[i] = 0xFFFFFFFFu;
  __syncwarp();

  // Round 0 elects the source: its dist 0 is the unique minimum.
  uint32_t u = source;
  uint32_t du = 0;
  uint64_t E = p.exch_base;
  uint64_t iters = 0, mispredicts = 0;
  uint32_t pred_u = 0xFFFFFFFFu;  // vertex whose row slice sits in `nxt`
  uint32_t last_l2 = 0xFFFFFFFFu;
  Row cur, nxt;
  cur.load(adj + (size_t)u * p.row_stride, lane);
  uint64_t ks[2 * NP];  // keys of the latest exchange (for the runner-up)
  uint64_t best_key = 0;
#pragma unroll
  for (int j = 0; j < 2 * NP; ++j) ks[j] = ~0ull;

  const uint64_t t_start = globaltimer();
  bool failed = false;

  while (true) {
    // ---- relax row u (serial.hpp:51-60); mark u visited where owned.
    {
      const uint32_t ul = u - p.col_base;
      if (u >= p.col_base && ul < p.loc_n && (ul % G) == c) {
        const uint32_t su = ul / G;
#pragma unroll
        for (int e = 0; e < EPL; ++e)
          if (Row::slot(e, lane) == su) vis |= (1ull << e);
      }
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t w = cur.elem(e);
      const uint32_t nd = du + w;
      if (w != WINF && nd < d[e]) {
        d[e] = nd;
        s_pred[Row::slot(e, lane)] = u;
      }
    }
    ++iters;
    if (p.visit_order != nullptr && p.shard == 0 && c == 0 && lane == 0)
      p.visit_order[(size_t)solve * p.n + (iters - 1)] = u;

    // ---- local election over unvisited owned columns (serial.hpp:42-48).
    uint32_t bd, bs;
    if (p.packed) {
      uint32_t k = 0xFFFFFFFFu;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const uint32_t ke = (((vis >> e) & 1ull) || d[e] == DINF)
                                ? 0xFFFFFFFFu
                                : ((d[e] << p.sbits) | Row::slot(e, lane));
        k = ke < k ? ke : k;
      }
      k = __reduce_min_sync(0xFFFFFFFFu, k);
      bd = k == 0xFFFFFFFFu ? DINF : (k >> p.sbits);
      bs = k & ((1u << p.sbits) - 1u);
    } else {
      bd = DINF;
      bs = 0xFFFFFFFFu;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const bool live = !((vis >> e) & 1ull) && d[e] != DINF;
        if (live && d[e] < bd) {  // ascending slots: strict '<' keeps the lowest
          bd = d[e];
          bs = Row::slot(e, lane);
        }
      }
      warp_lexmin(bd, bs);
    }
    const uint32_t bv = (bd == DINF) ? vmask_all : (p.col_base + bs * G + c);

    // ---- publish (flag-in-data) into every shard's exchange array.
    ++E;
    const uint32_t buf = (uint32_t)(E & 1ull);
    const uint64_t want = E & tagmask;
    const uint64_t key = ((uint64_t)bd << 32) | ((uint64_t)(bv & vmask_all) << tb) | want;
    publish_key(p, my_slots, solve, c, lane, buf, key, multi);

    // ---- off the critical path, while the exchange is in flight:
    // (a) the owner of a new local best pulls that vertex's full row into L2;
    if (pf_l2 && bd != DINF && bv != last_l2) {
      if (lane == 0)
        prefetch_l2_bulk(static_cast<const W*>(p.adj) + (size_t)bv * p.row_stride, row_bytes);
      last_l2 = bv;
    }
    // (b) the runner-up of the previous exchange predicts this exchange's
    //     winner: load its row slice into registers now.
    if (pf_reg) {
      uint64_t r = ~0ull;
#pragma unroll
      for (int j = 0; j < 2 * NP; ++j) r = (ks[j] != best_key && ks[j] < r) ? ks[j] : r;
      uint32_t a = (uint32_t)(r >> 32), b = (uint32_t)r;
      warp_lexmin(a, b);
      if (a != DINF && iters > 1) {
        pred_u = b >> tb;
        nxt.load(adj + (size_t)pred_u * p.row_stride, lane);
      } else {
        pred_u = 0xFFFFFFFFu;
      }
    }

    // ---- gather: poll until every participant's key carries tag E.
    failed = !gather_keys<NP>(p, my_slots + ((uint64_t)buf * p.nrep + c % p.nrep) * p.bstride,
                              nslot, lane, want, tagmask, multi, t_start, ks);
    if (failed) break;
    best_key = min_key<NP>(ks);
    du = (uint32_t)(best_key >> 32);
    if (du == DINF) break;  // no finite unvisited vertex remains on any shard
    u = (uint32_t)(best_key & 0xFFFFFFFFull) >> tb;
    if (pf_reg && u == pred_u) {
      cur = nxt;
    } else {
      if (pf_reg) ++mispredicts;
      cur.load(adj + (size_t)u * p.row_stride, lane);
    }
  }

  // ---- write back owned columns (the gather of partitioned.hpp:208-223).
  __syncwarp();
  uint64_t* dout = p.dist_out + (size_t)solve * p.loc_n;
  uint64_t* pout = p.pred_out + (size_t)solve * p.loc_n;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t s = Row::slot(e, lane);
    const uint32_t vl = s * G + c;
    if (vl < p.loc_n && p.col_base + vl < p.n) {
      dout[vl] = d[e] == DINF ? ~0ull : (uint64_t)d[e];
      const uint32_t pr = s_pred[s];
      pout[vl] = pr == 0xFFFFFFFFu ? ~0ull : (uint64_t)pr;
    }
  }
  uint64_t* inf = p.info + (size_t)solve * 4;
  if (failed && lane == 0) atomicOr((unsigned long long*)(inf + 2), 1ull);
  if (c == 0 && lane == 0) {
    inf[0] = iters;
    inf[1] = E;
    inf[3] = mispredicts;
  }
}

}  // namespace sssp_b200
