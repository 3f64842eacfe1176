// bucket_kernel.cuh -- exact distance-class ("bucket") Dijkstra, one
// cooperative persistent launch per solve.
//
// When every finite off-diagonal weight is >= 1 (checked at upload), the
// serial engine's n rounds (serial.hpp:41-61) decompose into distance classes:
//
//  * when the first vertex of class d is elected, EVERY vertex whose final
//    distance is d already holds dist == d (its tight parent has dist <= d-1
//    and was relaxed earlier), and no class-d vertex changes during the class
//    (w >= 1), so the class's elections are exactly B_d = {unsettled v :
//    dist[v] == d} in increasing vertex id (the lowest-id tie rule,
//    serial.hpp:46);
//  * relaxing B_d in that order with a strict '<' (serial.hpp:56) gives each
//    unsettled column v:  cand = d + min_{u in B_d} w(u,v),  pred = the LOWEST
//    u attaining that min (later equal candidates never win a strict '<'),
//    applied iff cand < dist[v].
//
// So one step = one class: find d (grid min), settle B_d, relax.  With zero
// weights the decomposition is wrong (3092/4000 mismatches),
// so the host only selects this engine when min weight >= 1; otherwise the
// n-round scan engines run.  Results are bit-identical to dijkstra_serial.
//
// Each step relaxes by PUSH (stream the rows of B_d, per-column min of the
// packed key (w, u)) or by PULL (for every still-unsettled column v, stream
// column v -- row v of the stored transpose, or of the matrix itself when it
// is symmetric -- masked by the B_d bitmap), whichever reads fewer rows:
// min(|B_d|, |unsettled|) rows per step (direction-optimising, as in BFS).
// A CTA owns a fixed tile of T matrix positions for the whole solve; its
// dist / pred / settled state lives in shared memory.  Two grid barriers per
// class.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

#include "scan_kernel.cuh"

namespace sssp_b200 {

// Global positions: shard j's local position p is global position
// g = j*row_stride + p, i.e. vertex j*loc_n + vid(p).  Tiles are numbered
// globally (shard j, CTA c) -> j*G + c.  With one shard this is the plain
// position order.
constexpr int kBucketMaxSlots = 8;

// One shard of the launch.  Every shard that lives on the launching device
// runs in the SAME cooperative launch (CTA range [i*G, (i+1)*G) = local shard
// i), so shards never wait on a kernel that CUDA is free not to co-schedule
// (ncu replay, CUDA_LAUNCH_BLOCKING, MPS).  Only shards on other devices /
// processes sit behind the cross-launch barrier.
struct BucketLocal {
  const void* adj;      // [n rows][row_stride]: this shard's columns, positions
  const void* adjT;     // PULL source (nullptr: push only); row r, global positions
  uint32_t* ubm;        // [2][row_stride/32]: published unsettled bitmap per tile
  void* pkey;           // [row_stride] K: per-column pull minimum (balanced pull)
  uint64_t* dist_out;   // [loc_n] (local vertex ids)
  uint64_t* pred_out;   // [loc_n]
  uint64_t* info;       // [4]: settled vertices, classes, rows pushed, rows pulled
  uint64_t* info2;      // [2]: barriers used, error
  uint32_t shard;       // global shard index
};

struct BucketParams {
  BucketLocal loc[kMaxShards];  // the shards of this launch (nlocal)
  uint32_t nlocal;
  uint64_t adjT_stride; // elements per adjT row (= nshards * row_stride)
  uint32_t adjT_by_pos; // 1: adjT row of column p is the local position p (sharded
                        //    transpose); 0: the vertex id vid(p) (one shard)
  uint64_t row_stride;  // positions per row (= Q*L)
  uint32_t n;           // vertices (global)
  uint32_t Q, L;        // layout: position p = q*L + s  <->  local vertex s*Q + q
  uint32_t qbits, lbits;
  uint32_t T;           // positions per CTA
  uint32_t nshards, loc_n;
  uint32_t* peer_bitmap[kMaxShards];  // every shard's [2][nshards*row_stride/32] (self incl.)
  uint32_t* peer_ctrl[kMaxShards];    // every shard's [2][3][nshards*G]: tile lmin, cand, uns
  // Cross-launch barrier (nlocal < nshards): launch counters, by global shard.
  // The leader of every launch adds nlocal to EVERY shard's counter once per
  // barrier; a launch waits on the counter of its first shard.
  unsigned long long* peer_bar[kMaxShards];
  unsigned long long* arrive;  // this launch's CTA arrival counter (monotonic)
  unsigned long long* release; // this launch's release word (barrier count)
  uint64_t* bar_epoch;  // cross-launch barriers completed by earlier launches (read at
                        // start, advanced at exit; the same value on every launch)
  uint64_t timeout_ns;
  uint64_t* trace;      // optional [64]: %globaltimer after every barrier (CTA 0 of shard 0)
  uint64_t seq;         // launch tag: a watchdog failure writes it to info2[1] (no reset needed)
  // Independent solves sharing one launch (one shard only): the grid is
  // nslots x tiles CTAs, slot s solves from slot_src[s] with its own exchange
  // region (slot_bytes apart) and its own outputs (out_stride / info strides).
  uint32_t nslots;
  uint32_t slot_src[kBucketMaxSlots];
  uint64_t slot_bytes;
  uint64_t out_stride;
  uint32_t* done;       // [kBucketMaxSlots] per-slot done flags (nslots > 1)
};

__device__ __forceinline__ uint32_t pos_to_vid(uint32_t pos, uint32_t Q, uint32_t lbits,
                                              uint32_t qbits) {
  return ((pos & ((1u << lbits) - 1u)) << qbits) | (pos >> lbits);
}

template <typename W>
struct BucketKey;  // per-column running minimum of (w, u): packed, smaller = better
template <>
struct BucketKey<uint8_t> {
  using T = uint32_t;  // w:8 | u:24
  static constexpr T kNone = 0xFFFFFFFFu;
  __device__ static T make(uint32_t w, uint32_t u) { return (w << 24) | u; }
  __device__ static uint32_t w(T k) { return k >> 24; }
  __device__ static uint32_t u(T k) { return k & 0xFFFFFFu; }
};
template <>
struct BucketKey<uint16_t> {
  using T = uint64_t;
  static constexpr T kNone = ~0ull;
  __device__ static T make(uint32_t w, uint32_t u) { return ((uint64_t)w << 32) | u; }
  __device__ static uint32_t w(T k) { return (uint32_t)(k >> 32); }
  __device__ static uint32_t u(T k) { return (uint32_t)k; }
};
template <>
struct BucketKey<uint32_t> : BucketKey<uint16_t> {};

// Packed key of weight j of a 16 B chunk word and vertex u.  u8: one PRMT
// builds (w << 24) | u (u < 2^24).
template <typename W>
__device__ __forceinline__ typename BucketKey<W>::T chunk_key(uint32_t word, int j, uint32_t u) {
  if constexpr (sizeof(W) == 1) {
    return __byte_perm(word, u, 0x0654u | ((uint32_t)(j % 4) << 12));
  } else {
    const uint32_t w = sizeof(W) == 4 ? word : (word >> ((j % 2) * 16)) & 0xFFFFu;
    return BucketKey<W>::make(w, u);
  }
}

// Asynchronous 16 B global -> shared copies (LDGSTS, L2 only): a thread
// streams row slices into its own shared-memory slots so the next batch's
// loads are in flight while the current batch is processed.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// shared- or global-memory atomic minimum of a packed key
__device__ __forceinline__ void smem_min(uint32_t* a, uint32_t v) { atomicMin(a, v); }
__device__ __forceinline__ void smem_min(uint64_t* a, uint64_t v) {
  atomicMin(reinterpret_cast<unsigned long long*>(a), (unsigned long long)v);
}
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* a) { return __ldcg(a); }
__device__ __forceinline__ uint64_t ld_cg(const uint64_t* a) {
  return (uint64_t)__ldcg(reinterpret_cast<const unsigned long long*>(a));
}

template <typename K>
__device__ __forceinline__ K warp_min_key(K k) {
  if constexpr (sizeof(K) == 4) {
    return __reduce_min_sync(0xFFFFFFFFu, k);
  } else {
    uint32_t a = (uint32_t)(k >> 32), b = (uint32_t)k;
    warp_lexmin(a, b);
    return ((uint64_t)a << 32) | b;
  }
}

constexpr int kBucketThreads = 256;

__host__ __device__ constexpr uint32_t bucket_round4(uint32_t x) { return (x + 3u) & ~3u; }

// dynamic shared memory of bucket_kernel (keeps every region 16 B aligned)
__host__ __device__ constexpr size_t bucket_smem_bytes(uint32_t T, uint32_t G, uint32_t words,
                                                       uint32_t wbytes);
constexpr int kBucketChunk = kBucketThreads * 32 * 2;  // ids of one pass over 512 bitmap words

// Dynamic smem: dist[T] u32 | pred[T] u32 | settled[T/32] u32 | lmin[GT] u32 |
//               bitmap[nshards*row_stride/32] u32 | unsettled[same] u32 | chunk[kBucketChunk] u32 |
//               combine[kBucketThreads * CPT] keys
//
// One grid barrier per class.  Before the barrier that ends step s every CTA
// publishes, for its own tile: its minimum unsettled dist (lmin), the bitmap
// of its unsettled columns at that minimum (the class candidates), and its
// counts.  After the barrier every CTA derives d = min(lmin); the candidates
// of the tiles with lmin == d form B_d -- no second barrier is needed to
// build the class.
// MULTI: several independent solves (slots) share the launch; the single-solve
// instance compiles the slot bookkeeping away.
template <typename W, bool MULTI>
__global__ void __launch_bounds__(kBucketThreads, 2) bucket_kernel(const BucketParams p) {
  namespace cg = cooperative_groups;
  using KT = BucketKey<W>;
  using K = typename KT::T;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t DINF = 0xFFFFFFFFu;
  constexpr int CPT = 16 / (int)sizeof(W);  // columns per thread (one 16 B load)

  extern __shared__ __align__(16) uint32_t smem[];
  // slot (independent solve; MULTI) or local shard of this CTA, and its tile
  const uint32_t Gs = MULTI ? gridDim.x / p.nslots : gridDim.x / p.nlocal;
  const uint32_t grp = blockIdx.x / Gs, bx = blockIdx.x - grp * Gs;
  const uint32_t slot = MULTI ? grp : 0u;
  const BucketLocal& S = p.loc[MULTI ? 0u : grp];
  const uint32_t shard = S.shard;
  auto at = [&](auto* ptr) {  // this slot's copy of an exchange-region array
    return reinterpret_cast<decltype(ptr)>(reinterpret_cast<char*>(const_cast<void*>(
                                               static_cast<const void*>(ptr))) + slot * p.slot_bytes);
  };
  const uint32_t source = p.slot_src[slot];
  uint32_t* const ubm = at(S.ubm);
  const uint32_t T = p.T, G = Gs * p.nshards;  // G = tiles of ALL shards
  const uint32_t TW = T / 32;  // bitmap words per tile
  const uint32_t lwords = (uint32_t)(p.row_stride / 32);
  const uint32_t words = lwords * p.nshards;  // global bitmap words
  uint32_t* sdist = smem;
  uint32_t* spred = sdist + T;
  uint32_t* ssettled = spred + T;
  uint32_t* slmin = ssettled + bucket_round4(TW);
  uint32_t* sbm = slmin + bucket_round4(G);  // B_d bitmap (all positions), staged per class
  uint32_t* sub = sbm + bucket_round4(words);  // this shard's unsettled bitmap (pull steps)
  uint32_t* schunk = sub + bucket_round4(words);
  K* scomb = reinterpret_cast<K*>(schunk + kBucketChunk);
  __shared__ uint32_t s_red[kBucketThreads / 32];
  __shared__ uint32_t s_red2[kBucketThreads / 32], s_red3[kBucketThreads / 32];
  __shared__ uint32_t s_cnt[2];

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t me = shard * Gs + bx;    // global tile id
  const uint32_t p0 = bx * T;             // first LOCAL position of the tile
  const uint32_t tbits = 31u - __clz(T);  // T is a power of two
  const W* adj = static_cast<const W*>(S.adj);
  const W* adjT = static_cast<const W*>(S.adjT);
  const uint32_t TPR = T * sizeof(W) / 16;  // threads per row slice
  const uint32_t RG = kBucketThreads / TPR; // row groups
  // global per-step arrays: ctrl = [2][3][G] (lmin, candidates, unsettled)
  uint32_t* const glob = at(p.peer_ctrl[shard]);
  const uint32_t* const gbm = at(p.peer_bitmap[shard]);
  K* const pkey = at(static_cast<K*>(S.pkey));
  // global position -> global vertex id
  auto gvid = [&](uint32_t g) -> uint32_t {
    const uint32_t j = g >> (p.qbits + p.lbits);  // row_stride = Q*L = 2^(qbits+lbits)
    return j * p.loc_n + pos_to_vid(g & ((1u << (p.qbits + p.lbits)) - 1u), p.Q, p.lbits, p.qbits);
  };

  uint32_t ntr = 0;
  auto stamp = [&]() {
    if (p.trace && me == 0 && slot == 0 && tid == 0 && ntr < 64) p.trace[ntr++] = globaltimer();
  };
  // One barrier over every CTA of every shard.  All shards in this launch:
  // the cooperative grid barrier (1.29 us at 256 CTAs, the fastest measured
  // variant: profiles/r01_ubench_barrier.jsonl).  Shards in other launches
  // (other GPUs / processes): hierarchical -- CTAs arrive on this launch's
  // counter, the launch leader adds nlocal to every shard's counter with one
  // system-scope atomic each (an NVLink write for a remote shard), waits for
  // all nshards arrivals on its own, then releases its CTAs: nshards NVLink
  // atomics per launch per barrier, not one per CTA.  Every counter continues
  // across launches (bar_epoch), so nothing is reset between solves.
  __shared__ uint32_t s_fail;
  if (tid == 0) s_fail = 0;
  uint64_t nbar = 0;
  bool failed = false;
  const uint64_t t_start = globaltimer();
  const bool cross = p.nlocal < p.nshards;
  const uint64_t bar_base = cross ? *(volatile uint64_t*)p.bar_epoch : 0;
  stamp();  // trace[0]: kernel start
  auto spin_until = [&](const unsigned long long* a, unsigned long long target, bool sys) -> bool {
    unsigned long long v;
    uint32_t polls = 0;
    while (true) {
      if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
      else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
      if (v >= target) return (v >> 63) == 0;  // bit 63: the leader's watchdog fired
      if ((++polls & 1023u) == 0 && globaltimer() - t_start > p.timeout_ns) return false;
    }
  };
  auto barrier = [&]() {
    if (!cross) {
      cg::this_grid().sync();
    } else {
      __syncthreads();
      if (tid == 0) {
        const unsigned long long b = bar_base + nbar + 1;  // global barrier number
        bool ok = true;
        __threadfence();
        atomicAdd(p.arrive, 1ull);
        if (blockIdx.x == 0) {
          ok = spin_until(p.arrive, b * gridDim.x, false);
          __threadfence_system();
          for (uint32_t j = 0; j < p.nshards; ++j) atomicAdd_system(p.peer_bar[j], (unsigned long long)p.nlocal);
          ok = ok && spin_until(p.peer_bar[p.loc[0].shard], b * p.nshards, true);
          const unsigned long long rel = ok ? b : (b | (1ull << 63));
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.release), "l"(rel) : "memory");
        } else {
          ok = spin_until(p.release, b, false);
        }
        if (!ok) {
          s_fail = 1;
          S.info2[slot * 2 + 1] = p.seq + slot;
        }
      }
      __syncthreads();
      failed = s_fail != 0;
    }
    ++nbar;
  };

  // Publishes this tile's minimum, candidate bitmap and counts for step `s`.
  auto publish = [&](uint32_t par) {
    uint32_t m = DINF, uns = 0;
    for (uint32_t col = tid; col < T; col += kBucketThreads)
      if (!((ssettled[col >> 5] >> (col & 31)) & 1u)) {
        m = min(m, sdist[col]);
        ++uns;
      }
    m = __reduce_min_sync(0xFFFFFFFFu, m);
    uns = __reduce_add_sync(0xFFFFFFFFu, uns);
    if (lane == 0) s_red[warp] = m;
    if (tid < 2) s_cnt[tid] = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&s_cnt[1], uns);
    for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) m = min(m, s_red[w2]);
    // candidate bitmap word i (columns 32i..32i+31) = one ballot of warp i % 8
    for (uint32_t i = warp; i < TW; i += kBucketThreads / 32) {
      const uint32_t sm = ssettled[i];
      const uint32_t cm =
          __ballot_sync(0xFFFFFFFFu, m != DINF && !((sm >> lane) & 1u) && sdist[i * 32 + lane] == m);
      if (lane < p.nshards)  // remote shards: P2P stores
        at(p.peer_bitmap[lane])[par * words + me * TW + i] = cm;
      if (lane == 31) {
        ubm[par * lwords + bx * TW + i] = ~sm;  // local only (pull work list)
        if (cm) atomicAdd(&s_cnt[0], __popc(cm));
      }
    }
    for (uint32_t col = tid; col < T; col += kBucketThreads) pkey[p0 + col] = KT::kNone;
    __syncthreads();
    if (tid < p.nshards) {
      uint32_t* c = at(p.peer_ctrl[tid]);
      c[(par * 3 + 0) * G + me] = m;
      c[(par * 3 + 1) * G + me] = s_cnt[0];
      c[(par * 3 + 2) * G + me] = s_cnt[1];
    }
  };

  // ---- init: dist = INF, pred = NONE, padding settled (serial.hpp:32-36),
  // then class 0 = {source} -- with every weight >= 1 the only vertex at
  // distance 0 -- settled and its row pushed by every CTA over its own tile
  // without a barrier (every CTA knows the source): dist = w(s,v), pred = s
  // for each finite w, exactly the serial engine's first round.
  const uint32_t vbase = shard * p.loc_n;
  for (uint32_t i = warp; i < TW; i += kBucketThreads / 32) {  // one ballot per bitmap word
    const uint32_t vl = pos_to_vid(p0 + i * 32 + lane, p.Q, p.lbits, p.qbits);
    const uint32_t m =
        __ballot_sync(0xFFFFFFFFu, vl >= p.loc_n || vbase + vl >= p.n || vbase + vl == source);
    if (lane == 0) ssettled[i] = m;
  }
  for (uint32_t i = tid; i < T; i += kBucketThreads) {
    const uint32_t vl = pos_to_vid(p0 + i, p.Q, p.lbits, p.qbits);
    const bool real = vl < p.loc_n && vbase + vl < p.n;
    const uint32_t w = real ? (uint32_t)adj[(size_t)source * p.row_stride + p0 + i] : WINF;
    const bool src = real && vbase + vl == source;
    sdist[i] = src ? 0u : (w != WINF ? w : DINF);
    spred[i] = (!src && w != WINF) ? source : 0xFFFFFFFFu;
  }
  __syncthreads();
  // Buffer parity = parity of the barrier that follows the publish, counted
  // GLOBALLY (the count continues across launches): a fast shard's next
  // launch then publishes into the buffer the slow shard is NOT reading after
  // its final barrier, and a step's extra (pull) barrier never lets a publish
  // overwrite a buffer some CTA may still read.
  if (MULTI && bx == 0 && tid == 0) p.done[slot] = 0;  // read after the first barrier
  publish((uint32_t)(bar_base & 1ull));
  barrier();
  stamp();

  bool done = false;  // this slot's solve has settled every reachable vertex
  uint64_t pushed = 1, pulled = 0, settled = 1;
  uint32_t step = 1;
  while (!failed) {
    const uint32_t par = (uint32_t)((bar_base + nbar - 1) & 1ull);
    bool relax = false, pull = false;
    uint32_t dk = 0, bcount = 0, ucount = 0;
    if (!done) {
      // ---- the class: d = min over tiles, B_d = candidates of the tiles at d.
      // One memory round trip: every tile's (lmin, candidates, unsettled) and
      // the whole candidate bitmap are loaded together, then reduced in smem.
      {
        const uint32_t* bm = gbm + par * words;
        for (uint32_t i = tid; i < words; i += kBucketThreads) sbm[i] = __ldcg(&bm[i]);
        // this shard's published unsettled bitmap, staged for a pull step
        const uint32_t* ub = ubm + par * lwords;
        for (uint32_t i = tid; i < lwords; i += kBucketThreads) sub[i] = __ldcg(&ub[i]);
      }
      uint32_t lm_r[4], cc_r[4], uu_r[4];  // G <= 4 * kBucketThreads tiles (host-checked)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        const uint32_t c = tid + k2 * kBucketThreads;
        lm_r[k2] = c < G ? __ldcg(&glob[(par * 3 + 0) * G + c]) : DINF;
        cc_r[k2] = c < G ? __ldcg(&glob[(par * 3 + 1) * G + c]) : 0u;
        uu_r[k2] = c < G ? __ldcg(&glob[(par * 3 + 2) * G + c]) : 0u;
      }
      uint32_t d = DINF;
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        const uint32_t c = tid + k2 * kBucketThreads;
        if (c < G) slmin[c] = lm_r[k2];
        d = min(d, lm_r[k2]);
      }
      d = __reduce_min_sync(0xFFFFFFFFu, d);
      if (lane == 0) s_red[warp] = d;
      __syncthreads();
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) d = min(d, s_red[w2]);
      if (d == DINF) {  // uniform within the slot: every CTA reads the same values
        done = true;
      } else {
        uint32_t uns = 0;
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
          bcount += lm_r[k2] == d ? cc_r[k2] : 0u;
          uns += uu_r[k2];
        }
        bcount = __reduce_add_sync(0xFFFFFFFFu, bcount);
        uns = __reduce_add_sync(0xFFFFFFFFu, uns);
        if (lane == 0) {
          s_red2[warp] = bcount;
          s_red3[warp] = uns;
        }
        // mask the staged bitmap to the tiles at d
        for (uint32_t i = tid; i < words; i += kBucketThreads)
          if (slmin[i >> (tbits - 5)] != d) sbm[i] = 0u;  // TW = T/32 words per tile
        __syncthreads();
        bcount = 0;
        uns = 0;
        for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) {
          bcount += s_red2[w2];
          uns += s_red3[w2];
        }
        ucount = uns - bcount;  // unsettled after settling B_d
        // settle my candidates if my tile is in the class
        for (uint32_t i = tid; i < TW; i += kBucketThreads) ssettled[i] |= sbm[me * TW + i];
        __syncthreads();
        stamp();
        ++step;
        settled += bcount;
        if (ucount == 0) {
          done = true;  // nothing left to relax (the last class needs no rows)
        } else {
          relax = true;
          pull = adjT != nullptr && ucount < bcount;
          dk = d;
        }
      }
    }
    if (!MULTI && done) break;

    if (relax && !pull) {
      // ---- PUSH: stream the rows of B_d (ascending ids), per-column min key
      pushed += bcount;
      const uint32_t rg = tid / TPR, ct = tid - rg * TPR;  // row group, column thread
      K best[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) best[j] = KT::kNone;
      // enumerate B_d in ascending order with one block scan per pass: a
      // class that fits the id chunk takes a single pass over all words (up
      // to 8 per thread), otherwise passes of 2 words per thread (<=
      // kBucketChunk ids each)
      constexpr uint32_t WMAX = 8;
      const uint32_t wpt = (bcount <= (uint32_t)kBucketChunk && words <= WMAX * kBucketThreads)
                               ? (words + kBucketThreads - 1) / kBucketThreads
                               : 2u;
      for (uint32_t wbase = 0; wbase < words; wbase += kBucketThreads * wpt) {
        const uint32_t w0 = wbase + tid * wpt;
        uint32_t bw[WMAX];
        uint32_t c = 0;
#pragma unroll
        for (uint32_t k2 = 0; k2 < WMAX; ++k2) {
          bw[k2] = k2 < wpt && w0 + k2 < words ? sbm[w0 + k2] : 0u;
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
        for (uint32_t k2 = 0; k2 < WMAX; ++k2)
          for (uint32_t m = bw[k2]; m; m &= m - 1)
            schunk[o++] = gvid((w0 + k2) * 32 + (__ffs(m) - 1));
        __syncthreads();
        // batches of 8 rows: all 8 loads are issued before any is consumed
        for (uint32_t r0 = rg; r0 < tot; r0 += 8 * RG) {
          uint32_t ub[8];
          uint4 vb[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const uint32_t r = r0 + m * RG;
            ub[m] = r < tot ? schunk[r] : 0xFFFFFFFFu;
            if (r < tot)
              vb[m] = __ldg(reinterpret_cast<const uint4*>(
                  reinterpret_cast<const uint8_t*>(adj + (size_t)ub[m] * p.row_stride + p0) + ct * 16));
          }
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            if (ub[m] == 0xFFFFFFFFu) break;
            const uint32_t wd[4] = {vb[m].x, vb[m].y, vb[m].z, vb[m].w};
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
              // INF weights make keys above every finite one
              const K k = chunk_key<W>(wd[(j * sizeof(W)) / 4], j, ub[m]);
              best[j] = k < best[j] ? k : best[j];
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int j = 0; j < CPT; ++j) scomb[tid * CPT + j] = best[j];
      __syncthreads();
      for (uint32_t col = tid; col < T; col += kBucketThreads) {
        const uint32_t cth = col / CPT, j = col % CPT;
        K k = KT::kNone;
        for (uint32_t g2 = 0; g2 < RG; ++g2) {
          const K x = scomb[(g2 * TPR + cth) * CPT + j];
          k = x < k ? x : k;
        }
        if (KT::w(k) != WINF && k != KT::kNone) {
          const uint32_t cand = dk + KT::w(k);
          if (cand < sdist[col]) {  // settled columns hold dist <= d < cand
            sdist[col] = cand;
            spred[col] = KT::u(k);
          }
        }
      }
      __syncthreads();
    } else if (relax && pull) {
      // ---- PULL, balanced over the whole shard: U = this shard's unsettled
      // columns after B_d (the published unsettled bitmaps minus the class).
      // The (column of U, 16 B chunk of its transposed row) items are split
      // evenly over the shard's CTAs -- a CTA no longer waits on the columns
      // of its own tile, whose count varies from tile to tile -- each CTA
      // folds its partial (w, u) minima into pkey[column] with one global
      // atomicMin per column it touched, and after an extra barrier every
      // owner applies its columns' minima.
      pulled += ucount;
      // the combine region holds the touched columns' running keys and local
      // positions (ncols <= T + 2, host-checked); the id chunk region becomes
      // the cp.async stage [2][kPullDepth][threads] of 16 B slots
      K* sk = scomb;
      uint32_t* scol = reinterpret_cast<uint32_t*>(scomb + (T + 2));
      const uint32_t* bml = sbm + shard * lwords;
      const uint32_t wpt = (lwords + kBucketThreads - 1) / kBucketThreads;
      const uint32_t w0 = tid * wpt;
      auto uword = [&](uint32_t k2) -> uint32_t {  // unsettled-after-B_d word w0 + k2
        return sub[w0 + k2] & ~bml[w0 + k2];
      };
      uint32_t c = 0;
      for (uint32_t k2 = 0; k2 < wpt && w0 + k2 < lwords; ++k2) c += __popc(uword(k2));
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      if (lane == 31) s_red[warp] = incl;
      __syncthreads();
      uint32_t base = 0, nuL = 0;
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) {
        if (w2 < warp) base += s_red[w2];
        nuL += s_red[w2];
      }
      base += incl - c;  // rank of this thread's first unsettled column
      // chunks per transposed row (nshards * row_stride: not a power of two for P = 3, 5, 6, 7)
      const uint32_t cpr = (uint32_t)(p.adjT_stride * sizeof(W) / 16);
      const bool cpow2 = (cpr & (cpr - 1u)) == 0;  // uniform: shifts instead of divisions
      const uint32_t cbits = 31u - __clz(cpr);
      const uint32_t total = nuL * cpr;
      const uint32_t per = (total + Gs - 1) / Gs;
      const uint32_t lo = min(total, bx * per), hi = min(total, lo + per);
      const uint32_t r0 = cpow2 ? lo >> cbits : lo / cpr;
      const uint32_t ncols = lo < hi ? (cpow2 ? (hi - 1) >> cbits : (hi - 1) / cpr) - r0 + 1 : 0;
      if (ncols && base < r0 + ncols && base + c > r0) {
        uint32_t r = base;
        for (uint32_t k2 = 0; k2 < wpt && w0 + k2 < lwords && r < r0 + ncols; ++k2)
          for (uint32_t m = uword(k2); m; m &= m - 1, ++r)
            if (r >= r0 && r < r0 + ncols) scol[r - r0] = (w0 + k2) * 32 + (__ffs(m) - 1);
      }
      for (uint32_t i = tid; i < ncols; i += kBucketThreads) sk[i] = KT::kNone;
      __syncthreads();
      stamp();
      if (p.trace && tid == 0 && shard == 0 && slot == 0 && bx < 1024)  // per-CTA pull span (debug)
        p.trace[64 + 2 * bx] = globaltimer();
      // Two-stage cp.async pipeline: a thread's items are lo + tid + k*256;
      // batch b+1's 16 B chunks stream into the thread's stage slots while
      // batch b is consumed.  (column rank, chunk) pairs are walked
      // incrementally (one division per thread, none per item).
      constexpr int kPullDepth = 8;
      uint4* sstage = reinterpret_cast<uint4*>(schunk);
      auto row_of = [&](uint32_t rk) -> const uint8_t* {
        const uint32_t col = scol[rk - r0];
        const uint32_t v = p.adjT_by_pos ? col : pos_to_vid(col, p.Q, p.lbits, p.qbits);
        return reinterpret_cast<const uint8_t*>(adjT + (size_t)v * p.adjT_stride);
      };
      auto advance = [&](uint32_t& rk, uint32_t& ch) {
        ch += kBucketThreads;
        while (ch >= cpr) {
          ch -= cpr;
          ++rk;
        }
      };
      uint32_t rk_t = 0, ch_t = 0;  // consume walk: this thread's next item
      if (lo + tid < hi) {
        rk_t = cpow2 ? (lo + tid) >> cbits : (lo + tid) / cpr;
        ch_t = lo + tid - rk_t * cpr;
      }
      uint32_t rk_i = rk_t, ch_i = ch_t;  // issue walk, one batch ahead
      const uint32_t nbatch = lo + tid < hi ? (hi - (lo + tid) + kBucketThreads * kPullDepth - 1) /
                                                  (kBucketThreads * kPullDepth) : 0u;
      auto issue = [&](uint32_t b) {
        uint4* st = sstage + (size_t)(b & 1u) * kPullDepth * kBucketThreads;
        const uint32_t it0 = lo + tid + b * kBucketThreads * kPullDepth;
        uint32_t rrow = rk_i;
        const uint8_t* row = row_of(rk_i);
#pragma unroll
        for (int m = 0; m < kPullDepth; ++m) {
          if (it0 + m * kBucketThreads < hi) {
            if (rk_i != rrow) {
              rrow = rk_i;
              row = row_of(rk_i);
            }
            cp_async16(&st[m * kBucketThreads + tid], row + ch_i * 16);
          }
          advance(rk_i, ch_i);
        }
        cp_async_commit();
      };
      uint32_t cur = 0xFFFFFFFFu;
      K run = KT::kNone;
      if (nbatch) issue(0);
      for (uint32_t b = 0; b < nbatch; ++b) {
        if (b + 1 < nbatch) issue(b + 1);
        else cp_async_commit();  // empty group: the wait below leaves one group pending
        cp_async_wait<1>();
        const uint4* st = sstage + (size_t)(b & 1u) * kPullDepth * kBucketThreads;
        const uint32_t it0 = lo + tid + b * kBucketThreads * kPullDepth;
#pragma unroll
        for (int m = 0; m < kPullDepth; ++m) {
          const uint32_t item = it0 + m * kBucketThreads;
          if (item >= hi) break;
          const uint32_t rk = rk_t, ch = ch_t;
          advance(rk_t, ch_t);
          const uint32_t ci = rk - r0;
          if (ci != cur) {
            if (cur != 0xFFFFFFFFu && run != KT::kNone) smem_min(&sk[cur], run);
            cur = ci;
            run = KT::kNone;
          }
          const uint32_t pos0 = ch * CPT;
          const uint32_t bits = (sbm[pos0 >> 5] >> (pos0 & 31)) & ((1u << CPT) - 1u);
          if (!bits) continue;
          // consecutive positions of one participant: vertex ids step by Q
          const uint32_t vid0 = gvid(pos0);
          const uint4 v4m = st[m * kBucketThreads + tid];
          const uint32_t wd[4] = {v4m.x, v4m.y, v4m.z, v4m.w};
          if constexpr (sizeof(W) == 1) {
            // u8, branch-free: the chunk's minimum (w, position) pair on the
            // native 16x2 min.  Non-class bytes -> 0xFF (INF); one PRMT packs
            // two bytes with their in-chunk index as (w << 8 | cc) lanes; the
            // min lane gives the smallest w at the lowest cc = lowest vertex id
            // (ids rise with cc).  (A data-dependent skip here measured slower.)
            uint32_t lanes[8];
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              const uint32_t b4 = (bits >> (4 * k2)) & 0xFu;
              const uint32_t mw = wd[k2] | ~(((b4 * 0x00204081u) & 0x01010101u) * 0xFFu);
              const uint32_t ccs = 0x03020100u + 0x04040404u * (uint32_t)k2;
              lanes[2 * k2] = __byte_perm(mw, ccs, 0x1504u);
              lanes[2 * k2 + 1] = __byte_perm(mw, ccs, 0x3726u);
            }
            uint32_t mv = __vminu2(__vminu2(__vminu2(lanes[0], lanes[1]), __vminu2(lanes[2], lanes[3])),
                                   __vminu2(__vminu2(lanes[4], lanes[5]), __vminu2(lanes[6], lanes[7])));
            mv = min(mv & 0xFFFFu, mv >> 16);
            const K kk = ((mv >> 8) << 24) | (vid0 + (mv & 0xFFu) * p.Q);
            run = kk < run ? kk : run;
          } else {
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
              const K kk = ((bits >> cc) & 1u) ? chunk_key<W>(wd[(cc * sizeof(W)) / 4], cc, vid0 + cc * p.Q)
                                                : KT::kNone;
              run = kk < run ? kk : run;
            }
          }
        }
      }
      cp_async_wait<0>();
      if (cur != 0xFFFFFFFFu && run != KT::kNone) smem_min(&sk[cur], run);
      __syncthreads();
      for (uint32_t i = tid; i < ncols; i += kBucketThreads)
        if (sk[i] != KT::kNone) smem_min(&pkey[scol[i]], sk[i]);
      if (p.trace && tid == 0 && shard == 0 && slot == 0 && bx < 1024)
        p.trace[64 + 2 * bx + 1] = globaltimer();
    }
    // the pull's extra barrier (every partial minimum is in pkey); with
    // several slots every step has it, so all CTAs count the same barriers
    if (pull || MULTI) {
      stamp();
      barrier();
      stamp();
    }
    if (relax && pull) {
      for (uint32_t col = tid; col < T; col += kBucketThreads) {
        if ((ssettled[col >> 5] >> (col & 31)) & 1u) continue;
        const K k = ld_cg(&pkey[p0 + col]);
        if (k != KT::kNone && KT::w(k) != WINF) {
          const uint32_t cand = dk + KT::w(k);
          if (cand < sdist[col]) {
            sdist[col] = cand;
            spred[col] = KT::u(k);
          }
        }
      }
      __syncthreads();
    }
    // ---- publish the next class's candidates, one barrier per class
    if (!done) {
      stamp();
      publish((uint32_t)((bar_base + nbar) & 1ull));
    } else if (MULTI && bx == 0 && tid == 0) {
      p.done[slot] = 1;  // read by every slot after the barrier
    }
    barrier();
    stamp();
    if (MULTI) {  // all slots done: leave together (uniform)
      bool all = true;
      for (uint32_t s2 = 0; s2 < p.nslots; ++s2) all &= __ldcg(&p.done[s2]) != 0;
      if (all) break;
    }
  }

  // ---- write back (positions -> local vertex ids)
  for (uint32_t i = tid; i < T; i += kBucketThreads) {
    const uint32_t v = pos_to_vid(p0 + i, p.Q, p.lbits, p.qbits);
    if (v < p.loc_n && vbase + v < p.n) {
      S.dist_out[slot * p.out_stride + v] = sdist[i] == DINF ? ~0ull : (uint64_t)sdist[i];
      S.pred_out[slot * p.out_stride + v] = spred[i] == 0xFFFFFFFFu ? ~0ull : (uint64_t)spred[i];
    }
  }
  stamp();
  if (bx == 0 && tid == 0) {
    uint64_t* const info = S.info + slot * 4;
    info[0] = settled;
    info[1] = step;
    info[2] = pushed;
    info[3] = pulled;
    S.info2[slot * 2] = nbar;
    if (cross && blockIdx.x == 0) *p.bar_epoch = bar_base + nbar;  // every CTA read it before barrier 1
  }
}

__host__ __device__ constexpr size_t bucket_smem_bytes(uint32_t T, uint32_t G, uint32_t words,
                                                       uint32_t wbytes) {
  return 4ull * (2ull * T + bucket_round4(T / 32) + bucket_round4(G) + 2ull * bucket_round4(words) +
                 kBucketChunk) +
         (size_t)kBucketThreads * (16 / wbytes) * (wbytes == 1 ? 4 : 8);
}

}  // namespace sssp_b200

namespace sssp_b200 {

// AT[v][p'] = A[vid(p')][pos(v)]: row v of the transpose in the same cyclic
// position order.  64x64 tiles staged through shared memory; both the reads
// (64 consecutive positions of row vid(p')) and the writes (64 consecutive
// positions of row vid(p)) are contiguous.
template <typename W>
__global__ void __launch_bounds__(256) transpose_positions_kernel(const W* __restrict__ a,
                                                                  W* __restrict__ at,
                                                                  uint64_t row_stride, uint32_t n,
                                                                  uint32_t Q, uint32_t qbits,
                                                                  uint32_t lbits) {
  __shared__ W tile[64][65];
  const uint32_t pb = blockIdx.x * 64;   // columns of A (positions p -> rows v of AT)
  const uint32_t ppb = blockIdx.y * 64;  // rows of A (positions p' -> vertex u = vid(p'))
  const uint32_t tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (uint32_t r = ty; r < 64; r += 4) {
    const uint32_t u = pos_to_vid(ppb + r, Q, lbits, qbits);
    tile[r][tx] = u < n ? a[(size_t)u * row_stride + pb + tx] : (W)WInf<W>::v;
  }
  __syncthreads();
  for (uint32_t r = ty; r < 64; r += 4) {
    const uint32_t v = pos_to_vid(pb + r, Q, lbits, qbits);
    if (v < n) at[(size_t)v * row_stride + ppb + tx] = tile[tx][r];
  }
}

// Sharded transpose: AT_k[p][g] = A_k[vertex(g)][p] for this shard's local
// positions p and all global positions g (shard j, local position q ->
// g = j*rs + q, vertex j*loc_n + vid(q)); padding / absent rows give INF.
template <typename W>
__global__ void __launch_bounds__(256) transpose_global_kernel(const W* __restrict__ a,
                                                               W* __restrict__ at, uint64_t rs,
                                                               uint32_t n, uint32_t Q,
                                                               uint32_t qbits, uint32_t lbits,
                                                               uint32_t P, uint32_t loc_n) {
  __shared__ W tile[64][65];
  const uint32_t pb = blockIdx.x * 64;  // local positions (rows of AT)
  const uint32_t gb = blockIdx.y * 64;  // global positions (columns of AT)
  const uint32_t tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  for (uint32_t r = ty; r < 64; r += 4) {
    const uint32_t g = gb + r;
    const uint32_t j = (uint32_t)(g / rs), vl = pos_to_vid((uint32_t)(g - j * rs), Q, lbits, qbits);
    const uint32_t u = j * loc_n + vl;
    tile[r][tx] = (vl < loc_n && u < n) ? a[(size_t)u * rs + pb + tx] : (W)WInf<W>::v;
  }
  __syncthreads();
  const uint64_t ats = rs * P;
  for (uint32_t r = ty; r < 64; r += 4) at[(size_t)(pb + r) * ats + gb + tx] = tile[tx][r];
}

// flag = 1 if the stored matrix is not symmetric: compares every element
// A[vid(p')][p] with its mirror A[vid(p)][p'] (same 64x64 tiling as the
// transpose, no transpose buffer needed; each tile pair once).
template <typename W>
__global__ void __launch_bounds__(256) symmetric_check_kernel(const W* __restrict__ a,
                                                              uint64_t row_stride, uint32_t n,
                                                              uint32_t Q, uint32_t qbits,
                                                              uint32_t lbits, uint32_t* flag) {
  // block (x, y) compares the (y, x) tile with the transpose of the (x, y)
  // tile, so (y, x) would repeat the comparison: half the blocks exit
  if (blockIdx.y < blockIdx.x) return;
  __shared__ W tile[64][65];
  const uint32_t pb = blockIdx.x * 64, ppb = blockIdx.y * 64;
  const uint32_t tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  for (uint32_t r = ty; r < 64; r += 4) {
    const uint32_t u = pos_to_vid(ppb + r, Q, lbits, qbits);
    tile[r][tx] = u < n ? a[(size_t)u * row_stride + pb + tx] : (W)WInf<W>::v;
  }
  __syncthreads();
  bool diff = false;
  for (uint32_t r = ty; r < 64; r += 4) {
    const uint32_t v = pos_to_vid(pb + r, Q, lbits, qbits);
    if (v < n) {
      const uint32_t u = pos_to_vid(ppb + tx, Q, lbits, qbits);
      if (u < n) diff |= a[(size_t)v * row_stride + ppb + tx] != tile[tx][r];
    }
  }
  if (__any_sync(0xFFFFFFFFu, diff) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// flag = 1 if A and AT differ anywhere (i.e. the matrix is not symmetric)
template <typename W>
__global__ void compare_rows_kernel(const W* __restrict__ a, const W* __restrict__ b,
                                    uint64_t elems, uint32_t* flag) {
  bool diff = false;
  const uint64_t n16 = elems * sizeof(W) / 16;
  const uint4* a4 = reinterpret_cast<const uint4*>(a);
  const uint4* b4 = reinterpret_cast<const uint4*>(b);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 x = a4[i], y = b4[i];
    diff |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (__any_sync(0xFFFFFFFFu, diff) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace sssp_b200
