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
#include <type_traits>

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
  uint64_t* cta_bytes;  // [slots][ctab_stride]: matrix bytes each CTA of the solve loaded
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
  uint32_t* peer_ctrl[kMaxShards];    // every shard's [2][4][nshards*G]: tile lmin, cand, open, finite
  uint32_t wmin;        // smallest finite off-diagonal weight of the whole graph (>= 1)
  uint32_t max_classes; // AUTO: stop after this many classes (0 = no limit; single solves)
  uint32_t push_ldg;    // 1: push rows through registers (LDG) instead of bulk copies (A/B)
  uint32_t push_depth16;  // LDG push: one 16-deep batch for classes of <= 16 rows per row group
  uint32_t owner_cols;   // pull steps with <= this many open columns in every tile run
                         // on the column owners (no combine barrier); 0 = never
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
  uint32_t dbg_reps;    // debug (SSSP_BUCKET_REPS): repeat the class-1 row scan
  unsigned long long* spans;  // debug (SSSP_BUCKET_SPANS): [64][2] per launch: max ~start, max end
  const uint32_t* rsum; // [n][8] row summaries (row_summary_kernel; one shard only) or nullptr
  const uint32_t* rlist;  // class-1 id lists: row u's B_1 at rlist[rsum[u][4]] (~0u: none)
  uint32_t ctab_stride; // CTAs per slot in cta_bytes
  // Sparse tile lists (tile_list_kernel; one shard, u8/u16, built at upload
  // for sparse matrices): the finite entries of row u inside tile t are
  // sp_ent[sp_off[u*G+t] .. sp_off[u*G+t+1]), each (position << 8*sizeof(W) | w);
  // row-major, so row u's entries are sp_ent[sp_off[u*G] .. sp_off[(u+1)*G]).
  // nullptr: the push streams the dense row slices.
  const uint32_t* sp_off;
  const uint32_t* sp_ent;
  uint32_t sp_split;    // classes of >= this many rows push row-split (0: never)
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
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Bulk (TMA-engine) global -> shared copies completing on an mbarrier
// (cp.async.bulk -> UBLKCP, expect_tx -> SYNCS.ARRIVE.TRANS64): a row slice
// is one copy instruction, so every row of a class is in flight at once
// instead of the 8 16 B loads a thread can keep outstanding.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// generic-proxy accesses of a shared buffer before async-proxy (bulk) writes to it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

constexpr int kBucketThreads = 256;
// Registers per thread: 2 CTAs x 256 threads per SM at <= 128.  (A full
// register file costs ~2.3 us per back-to-back launch -- tools/ubench_launch2.cu,
// 5.1 vs 2.8 us -- but capping this kernel at 120 or fewer registers spills and
// loses more than that: config 2 50.6 -> 53.3 us, config 4 1.42 -> 1.47 ms.)
#ifndef SSSP_BUCKET_MAXREG
#define SSSP_BUCKET_MAXREG 128
#endif

// A/B variants measured and rejected: the bulk-copy push and
// the 16-deep register push.  Compiled only with -DSSSP_BUCKET_AB=1 so the
// default instance keeps its code (and instruction-cache footprint) small.
#ifndef SSSP_BUCKET_AB
#define SSSP_BUCKET_AB 0
#endif
constexpr bool kBucketAB = SSSP_BUCKET_AB != 0;

__host__ __device__ constexpr uint32_t bucket_round4(uint32_t x) { return (x + 3u) & ~3u; }

// dynamic shared memory of bucket_kernel (keeps every region 16 B aligned)
__host__ __device__ constexpr size_t bucket_smem_bytes(uint32_t T, uint32_t G, uint32_t words,
                                                       uint32_t wbytes);
constexpr int kBucketChunk = kBucketThreads * 32 * 2;  // ids of one pass over 512 bitmap words
constexpr uint32_t kIdCap = kBucketChunk / 2;           // ids of one push pass (the rest stages rows)

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
// ONE: one shard in the launch and no peer launches (nshards == nlocal == 1):
// the shard / cross-launch bookkeeping folds away, which keeps the code a solve
// executes small (the instruction cache behind L0 is 32 KB; a miss is an L2
// round trip).
// SP: the sparse-list instance (p.sp_off set); the dense instances compile
// without any of its code.
template <typename W, bool MULTI, bool ONE, bool SP = false>
__global__ void __maxnreg__(SSSP_BUCKET_MAXREG) bucket_kernel(const BucketParams p) {
  namespace cg = cooperative_groups;
  using KT = BucketKey<W>;
  using K = typename KT::T;
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t DINF = 0xFFFFFFFFu;
  constexpr int CPT = 16 / (int)sizeof(W);  // columns per thread (one 16 B load)

  // Programmatic dependent launch: the next solve's grid may be launched at
  // once (its CTAs become resident only as this grid's CTAs exit), and this
  // grid waits for its predecessor's completion and memory before touching
  // anything -- back-to-back solves then pay no launch-processing gap
  // (tools/ubench_launch2.cu: 5.2 -> 2.9 us per cooperative launch).  Both
  // are no-ops when the launch carries no programmatic dependency.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t nsh = ONE ? 1u : p.nshards, nloc = ONE ? 1u : p.nlocal;
  // slot (independent solve; MULTI) or local shard of this CTA, and its tile
  const uint32_t Gs = MULTI ? gridDim.x / p.nslots : gridDim.x / nloc;
  const uint32_t grp = blockIdx.x / Gs, bx = blockIdx.x - grp * Gs;
  const uint32_t slot = MULTI ? grp : 0u;
  const BucketLocal& S = p.loc[MULTI ? 0u : grp];
  const uint32_t shard = ONE ? 0u : S.shard;
  auto at = [&](auto* ptr) {  // this slot's copy of an exchange-region array
    return reinterpret_cast<decltype(ptr)>(reinterpret_cast<char*>(const_cast<void*>(
                                               static_cast<const void*>(ptr))) + slot * p.slot_bytes);
  };
  const uint32_t source = p.slot_src[slot];
  uint32_t* const ubm = at(S.ubm);
  const uint32_t T = p.T, G = Gs * nsh;  // G = tiles of ALL shards
  const uint32_t TW = T / 32;  // bitmap words per tile
  const uint32_t lwords = (uint32_t)(p.row_stride / 32);
  const uint32_t words = lwords * nsh;  // global bitmap words
  uint32_t* sdist = smem;
  uint32_t* spred = sdist + T;
  uint32_t* ssettled = spred + T;
  uint32_t* slmin = ssettled + bucket_round4(TW);
  uint32_t* sbm = slmin + bucket_round4(G);  // B_d bitmap (all positions), staged per class
  uint32_t* sub = sbm + bucket_round4(words);  // this shard's unsettled bitmap (pull steps)
  uint32_t* schunk = sub + bucket_round4(words);
  K* scomb = reinterpret_cast<K*>(schunk + kBucketChunk);
  __shared__ uint32_t s_red[kBucketThreads / 32];
  __shared__ uint32_t s_red2[kBucketThreads / 32], s_red3[kBucketThreads / 32], s_red4[kBucketThreads / 32], s_red5[kBucketThreads / 32];
  __shared__ uint32_t s_cnt[3];

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t me = shard * Gs + bx;    // global tile id
  const uint32_t p0 = bx * T;             // first LOCAL position of the tile
  const uint32_t tbits = 31u - __clz(T);  // T is a power of two
  const W* adj = static_cast<const W*>(S.adj);
  const W* adjT = static_cast<const W*>(S.adjT);
  const uint32_t TPR = T * sizeof(W) / 16;  // threads per row slice
  const uint32_t RG = kBucketThreads / TPR; // row groups
  // global per-step arrays: ctrl = [2][4][G] (lmin, candidates, open, finite)
  uint32_t* const glob = at(p.peer_ctrl[shard]);
  const uint32_t* const gbm = at(p.peer_bitmap[shard]);
  K* const pkey = at(static_cast<K*>(S.pkey));
  // global position -> global vertex id
  auto gvid = [&](uint32_t g) -> uint32_t {
    if (ONE) return pos_to_vid(g, p.Q, p.lbits, p.qbits);
    const uint32_t j = g >> (p.qbits + p.lbits);  // row_stride = Q*L = 2^(qbits+lbits)
    return j * p.loc_n + pos_to_vid(g & ((1u << (p.qbits + p.lbits)) - 1u), p.Q, p.lbits, p.qbits);
  };

  // Minimum (w, u) key over the class members of one 16 B chunk of a
  // transposed row: `bits` = the B_d bits of its CPT positions, vid0 = the
  // vertex of its first position (consecutive positions of one participant:
  // vertex ids step by Q).
  auto chunk_min = [&](const uint4 v4m, uint32_t bits, uint32_t vid0) -> K {
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
      return (K)(((mv >> 8) << 24) | (vid0 + (mv & 0xFFu) * p.Q));
    } else {
      K run = KT::kNone;
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        const K kk = ((bits >> cc) & 1u) ? chunk_key<W>(wd[(cc * sizeof(W)) / 4], cc, vid0 + cc * p.Q)
                                          : KT::kNone;
        run = kk < run ? kk : run;
      }
      return run;
    }
  };

  uint32_t ntr = 0;
  // trace entry = phase code << 56 | %globaltimer (CTA 0 of shard 0, debug)
  const bool tr_on = p.trace != nullptr && me == 0 && slot == 0 && tid == 0;
  auto stamp = [&](uint32_t code) {
    if (tr_on && ntr < 512) {  // stamps 64..511 live after the per-CTA spans (4096 words)
      p.trace[ntr < 64 ? ntr : 4096 + ntr] = ((uint64_t)code << 56) | ((uint64_t)clock64() & ((1ull << 56) - 1));
      ++ntr;
    }
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
  __shared__ __align__(8) uint64_t s_mbar[2];  // bulk-copy completion (stage buffers 0/1)
  uint32_t mph = 0;                             // their phase parities (bit per buffer)
  if (tid == 0) {
    mbar_init(&s_mbar[0], 1);
    mbar_init(&s_mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __shared__ uint32_t s_fail;
  __shared__ unsigned long long s_spb;  // sparse-list bytes this CTA loaded
  if (tid == 0) s_fail = 0;
  if (SP && tid == 0) s_spb = 0;
  uint64_t nbar = 0;
  bool failed = false;
  const uint64_t t_start = globaltimer();
  const bool cross = !ONE && nloc < nsh;
  const uint64_t bar_base = cross ? *(volatile uint64_t*)p.bar_epoch : 0;
  stamp(0);  // trace[0]: kernel start
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
          for (uint32_t j = 0; j < nsh; ++j) atomicAdd_system(p.peer_bar[j], (unsigned long long)nloc);
          ok = ok && spin_until(p.peer_bar[p.loc[0].shard], b * nsh, true);
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
  // A column whose dist is <= fb = (lowest possible next class) + wmin is
  // FINAL: every later class d' relaxes it with d' + w >= fb, which never
  // beats it under the strict '<' (serial.hpp:56), so neither dist nor pred
  // can change.  Only the other ("open") unsettled columns are published for
  // pull steps and counted for the push/pull choice and the end test.
  auto publish = [&](uint32_t par, uint32_t fb) {
    uint32_t m = DINF, nopen = 0, nfin = 0;
    for (uint32_t col = tid; col < T; col += kBucketThreads)
      if (!((ssettled[col >> 5] >> (col & 31)) & 1u)) {
        const uint32_t dv = sdist[col];
        m = min(m, dv);
        nopen += dv > fb ? 1u : 0u;
        nfin += dv != DINF ? 1u : 0u;
      }
    m = __reduce_min_sync(0xFFFFFFFFu, m);
    nopen = __reduce_add_sync(0xFFFFFFFFu, nopen);
    nfin = __reduce_add_sync(0xFFFFFFFFu, nfin);
    if (lane == 0) s_red[warp] = m;
    if (tid < 3) s_cnt[tid] = 0;
    __syncthreads();
    if (lane == 0) {
      atomicAdd(&s_cnt[1], nopen);
      atomicAdd(&s_cnt[2], nfin);
    }
    for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) m = min(m, s_red[w2]);
    // candidate bitmap word i (columns 32i..32i+31) = one ballot of warp i % 8
    for (uint32_t i = warp; i < TW; i += kBucketThreads / 32) {
      const uint32_t sm = ssettled[i];
      const bool live = !((sm >> lane) & 1u);
      const uint32_t dv = sdist[i * 32 + lane];
      const uint32_t cm = __ballot_sync(0xFFFFFFFFu, m != DINF && live && dv == m);
      const uint32_t om = __ballot_sync(0xFFFFFFFFu, live && dv > fb);
      if (lane < nsh)  // remote shards: P2P stores
        at(p.peer_bitmap[lane])[par * words + me * TW + i] = cm;
      if (lane == 31) {
        ubm[par * lwords + bx * TW + i] = om;  // local only (pull work list)
        if (cm) atomicAdd(&s_cnt[0], __popc(cm));
      }
    }
    for (uint32_t col = tid; col < T; col += kBucketThreads) pkey[p0 + col] = KT::kNone;
    __syncthreads();
    if (tid < nsh) {
      uint32_t* c = at(p.peer_ctrl[tid]);
      c[(par * 4 + 0) * G + me] = m;
      c[(par * 4 + 1) * G + me] = s_cnt[0];
      c[(par * 4 + 2) * G + me] = s_cnt[1];
      c[(par * 4 + 3) * G + me] = s_cnt[2];
    }
    stamp(10);
  };
  // lowest possible next class + wmin (64-bit: no wrap), capped below INF
  auto final_bound = [&](uint32_t dlast) -> uint32_t {
    return (uint32_t)umin64((uint64_t)dlast + 1u + p.wmin, (uint64_t)DINF - 1u);
  };

  // Row-split ("spread") sparse push for large classes: the class rows are
  // divided over every warp of the slot, each row's whole entry list goes to
  // the per-column global key array pkey by atomicMin, and every tile applies
  // its columns after one extra barrier -- instead of every CTA walking every
  // class row for its own tile.  Uniform: depends on the class size only.
  // Only after a determination (every tile's publish reset its pkey words).
  auto spread_ok = [&](uint32_t bc) -> bool {
    return SP && sizeof(W) <= 2 && p.sp_off != nullptr && p.sp_split != 0 && bc >= p.sp_split;
  };
  bool local1 = false;
  uint32_t l_d1 = DINF, l_bc = 0, l_uc = 0, l_fin = 0;
  const uint32_t l_off = p.rsum && p.rlist ? __ldg(p.rsum + (size_t)source * 8 + 4) : 0xFFFFFFFFu;
  if (p.rsum) {
    local1 = true;
    for (uint32_t s2 = 0; s2 < (MULTI ? p.nslots : 1u); ++s2) {
      const uint32_t src2 = MULTI ? p.slot_src[s2] : source;
      const uint4 r4 = __ldg(reinterpret_cast<const uint4*>(p.rsum + (size_t)src2 * 8));
      const bool pull1 = r4.x != DINF && r4.z != 0 && adjT != nullptr && r4.z < r4.y && !(SP && p.sp_off != nullptr);
      local1 = local1 && !pull1 && r4.y <= kIdCap;
      if (src2 == source) {
        l_d1 = r4.x;
        l_bc = r4.y;
        l_uc = r4.z;
        l_fin = r4.w;
      }
    }
  }
  // The class-1 id list (an upload product, read-only) is copied into the id
  // chunk asynchronously here, so its round trip overlaps the class-0 row
  // slice below instead of following it; visible after the init barrier.
  const bool pre_ids = local1 && l_d1 != DINF && l_uc != 0 && l_off != 0xFFFFFFFFu;
  if (pre_ids) {
    for (uint32_t i = tid; i < l_bc; i += kBucketThreads) cp_async4(&schunk[i], p.rlist + l_off + i);
    cp_async_commit();
  }
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
  if (pre_ids) cp_async_wait<0>();
  __syncthreads();
  // Buffer parity = parity of the barrier that follows the publish, counted
  // GLOBALLY (the count continues across launches): a fast shard's next
  // launch then publishes into the buffer the slow shard is NOT reading after
  // its final barrier, and a step's extra (pull) barrier never lets a publish
  // overwrite a buffer some CTA may still read.
  if (MULTI && bx == 0 && tid == 0) p.done[slot] = 0;  // read after the first barrier
  stamp(12);  // class-0 row slice loaded
  uint32_t fb = final_bound(0);  // class 0 = {source} at distance 0

  bool done = false;  // this slot's solve has settled every reachable vertex
  bool bailed = false;  // class budget exceeded (results invalid; host reruns)
  uint64_t pushed = 1, pulled = 0, settled = 1;
  uint64_t my_bytes = (uint64_t)T * sizeof(W);  // matrix bytes this CTA loaded (class 0: one slice)
  uint32_t step = 1;
  uint32_t ids_n = 0xFFFFFFFFu;  // B_d ids already staged in schunk (class 1 from the row summary)

  // ---- class 1 without an exchange (one shard).  rsum[source] holds what the
  // exchange after class 0 would produce -- d1 = min_v w(source, v), |B_1|,
  // the open-column count left after B_1, the finite count (row_summary_kernel)
  // -- so every CTA knows the first class; B_1 itself is found by scanning row
  // `source` (one row, L2-resident after the first CTA's miss).  A class-1
  // PULL, or a class too large for one id pass, takes the exchange as before.
  // With several slots the choice is made for all of them together, so every
  // slot counts the same barriers.
  stamp(16);
  bool pre = false;  // the first loop step's class decisions are already made
  __shared__ uint32_t s_pre[4];  // its d, |B_d|, open count, relax (smem: not live across the loop)
  if (local1) {
    if (l_d1 == DINF) {  // no finite edge out of the source
      done = true;
    } else if (l_uc == 0) {  // nothing any class could lower (see the determination)
      settled += l_fin;
      done = true;
    } else {
      // B_1 = the positions of row `source` holding d1 (not the source, not padding):
      // the list built at upload (row_list_kernel), else a scan of the row
      if (pre_ids) {  // ids already in schunk (copied at kernel start)
        if (tid == 0) s_cnt[0] = l_bc;
      } else
      for (uint32_t rr = 0; rr < p.dbg_reps; ++rr) {
      if (tid == 0) s_cnt[0] = 0;
      __syncthreads();
      const uint4* row4 = reinterpret_cast<const uint4*>(adj + (size_t)source * p.row_stride);
      const uint32_t pos_src = ((source & (p.Q - 1u)) << p.lbits) | (source >> p.qbits);
      const uint32_t nch = (uint32_t)(p.row_stride * sizeof(W) / 16);
      for (uint32_t c0 = 0; c0 < nch; c0 += kBucketThreads * 8) {
        // each lane: a 16-bit mask of its chunk's d1 positions per 16 B chunk;
        // one warp prefix + one shared atomic per warp place the ids (a
        // per-lane branch on a match diverges in almost every warp)
        uint32_t mk[8], cnt = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t j = c0 + tid + k * kBucketThreads;
          mk[k] = 0;
          if (j < nch) {
            const uint4 v = __ldcg(row4 + j);
            const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if constexpr (sizeof(W) == 1) {  // exact zero-byte mask of w ^ d1x4 -> 4 bits
                const uint32_t t = wd[e] ^ (l_d1 * 0x01010101u);
                const uint32_t z = ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t | 0x7F7F7F7Fu);
                mk[k] |= ((((z >> 7) * 0x00204081u) >> 21) & 0xFu) << (4 * e);
              } else {
#pragma unroll
                for (int b = 0; b < 4 / (int)sizeof(W); ++b) {
                  const uint32_t w = sizeof(W) == 4 ? wd[e] : (wd[e] >> (8 * sizeof(W) * b)) & WINF;
                  if (w == l_d1) mk[k] |= 1u << (e * (4 / sizeof(W)) + b);
                }
              }
            }
            // not class members: the source's own entry and padding positions
            if (j == pos_src / CPT) mk[k] &= ~(1u << (pos_src % CPT));
            if (p.n < p.row_stride) {  // chunk = CPT positions of one run: ids vid0, vid0 + Q, ...
              const uint32_t vid0 = pos_to_vid(j * CPT, p.Q, p.lbits, p.qbits);
              const uint32_t nv = vid0 >= p.n ? 0u : min((uint32_t)CPT, (p.n - vid0 + p.Q - 1) >> p.qbits);
              mk[k] &= nv >= 32 ? 0xFFFFFFFFu : (1u << nv) - 1u;
            }
          }
          cnt += __popc(mk[k]);
        }
        if (!__any_sync(0xFFFFFFFFu, cnt != 0)) continue;
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += t;
        }
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(&s_cnt[0], incl);
        base = __shfl_sync(0xFFFFFFFFu, base, 31) + incl - cnt;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          for (uint32_t m = mk[k]; m; m &= m - 1) {
            const uint32_t pos = (c0 + tid + k * kBucketThreads) * CPT + (__ffs(m) - 1);
            schunk[base++] = pos_to_vid(pos, p.Q, p.lbits, p.qbits);
          }
      }
      __syncthreads();
      stamp(17);
      }
      // my tile's class-1 columns are settled now
      for (uint32_t i = warp; i < TW; i += kBucketThreads / 32) {
        const uint32_t bits = __ballot_sync(
            0xFFFFFFFFu, !((ssettled[i] >> lane) & 1u) && sdist[i * 32 + lane] == l_d1);
        if (lane == 0) ssettled[i] |= bits;
      }
      __syncthreads();
      ids_n = s_cnt[0];  // == l_bc
      settled += l_bc;
      step = 2;
      fb = final_bound(l_d1);
      // push: a tile none of whose columns is open after B_1 skips the rows
      const uint32_t lim = (uint32_t)umin64((uint64_t)l_d1 + p.wmin, (uint64_t)DINF - 1u);
      bool open = false;
      for (uint32_t col = tid; col < T; col += kBucketThreads)
        open |= !((ssettled[col >> 5] >> (col & 31)) & 1u) && sdist[col] > lim;
      const bool relax0 = __syncthreads_or(open);
      if (!relax0) ids_n = 0xFFFFFFFFu;  // nothing to push into this tile
      if (tid == 0) {
        s_pre[0] = l_d1;
        s_pre[1] = l_bc;
        s_pre[2] = l_uc;
        s_pre[3] = relax0;
      }
      __syncthreads();
      pre = true;
    }
    stamp(15);
  } else {
    publish((uint32_t)(bar_base & 1ull), fb);
    barrier();
    stamp(1);
  }
  while (!failed) {
    const uint32_t par = (uint32_t)((bar_base + nbar - 1) & 1ull);
    bool relax = false, pull = false, owner = false, spread = false;
    uint32_t dk = 0, bcount = 0, ucount = 0;
    if (pre) {
      pre = false;
      dk = s_pre[0];
      bcount = s_pre[1];
      ucount = s_pre[2];
      relax = s_pre[3] != 0;  // class 1 never spreads: pkey is reset by the first publish
    } else if (!done) {
      // ---- the class: d = min over tiles, B_d = candidates of the tiles at d.
      // One memory round trip: every tile's (lmin, candidates, unsettled) and
      // the whole candidate bitmap are loaded together, then reduced in smem.
      {
        const uint32_t* bm = gbm + par * words;
        for (uint32_t i = tid; i < words; i += kBucketThreads) sbm[i] = __ldcg(&bm[i]);
      }
      uint32_t lm_r[4], cc_r[4], uu_r[4], ff_r[4];  // G <= 4 * kBucketThreads tiles (host-checked)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        const uint32_t c = tid + k2 * kBucketThreads;
        lm_r[k2] = c < G ? __ldcg(&glob[(par * 4 + 0) * G + c]) : DINF;
        cc_r[k2] = c < G ? __ldcg(&glob[(par * 4 + 1) * G + c]) : 0u;
        uu_r[k2] = c < G ? __ldcg(&glob[(par * 4 + 2) * G + c]) : 0u;
        ff_r[k2] = c < G ? __ldcg(&glob[(par * 4 + 3) * G + c]) : 0u;
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
      stamp(2);
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) d = min(d, s_red[w2]);
      if (d == DINF) {  // uniform within the slot: every CTA reads the same values
        done = true;
      } else {
        uint32_t uns = 0, fin = 0, mopen = 0;  // mopen: most open columns left in one tile
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
          const uint32_t cls = lm_r[k2] == d ? cc_r[k2] : 0u;
          bcount += cls;
          uns += uu_r[k2];
          fin += ff_r[k2];
          mopen = max(mopen, uu_r[k2] - (d > fb ? cls : 0u));
        }
        bcount = __reduce_add_sync(0xFFFFFFFFu, bcount);
        uns = __reduce_add_sync(0xFFFFFFFFu, uns);
        fin = __reduce_add_sync(0xFFFFFFFFu, fin);
        mopen = __reduce_max_sync(0xFFFFFFFFu, mopen);
        if (lane == 0) {
          s_red2[warp] = bcount;
          s_red3[warp] = uns;
          s_red4[warp] = fin;
          s_red5[warp] = mopen;
        }
        // mask the staged bitmap to the tiles at d
        for (uint32_t i = tid; i < words; i += kBucketThreads)
          if (slmin[i >> (tbits - 5)] != d) sbm[i] = 0u;  // TW = T/32 words per tile
        __syncthreads();
        bcount = 0;
        uns = 0;
        fin = 0;
        mopen = 0;
        for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) {
          bcount += s_red2[w2];
          uns += s_red3[w2];
          fin += s_red4[w2];
          mopen = max(mopen, s_red5[w2]);
        }
        // open columns left after settling B_d (B_d is open iff d > fb: all
        // its members hold dist d)
        ucount = uns - (d > fb ? bcount : 0u);
        // settle my candidates if my tile is in the class
        for (uint32_t i = tid; i < TW; i += kBucketThreads) ssettled[i] |= sbm[me * TW + i];
        __syncthreads();
        stamp(3);
        ++step;
        if (!MULTI && p.max_classes && step > p.max_classes) {
          // AUTO's class budget is spent: this graph has too many distance
          // classes for class steps to beat n scan rounds -- stop; the host
          // reruns the solve on the n-round engine (uniform: step is)
          bailed = true;
          done = true;
        } else if (ucount == 0) {
          // nothing left any class could lower: every remaining finite column
          // is final (it would be elected later without relaxing anything)
          settled += fin;
          done = true;
        } else {
          settled += bcount;
          relax = true;
          pull = adjT != nullptr && ucount < bcount && !(SP && p.sp_off != nullptr);  // sparse: push
          // small pulls run on the column owners: no partial minima to
          // combine, so no extra barrier (uniform: every CTA read the same counts)
          // (a column read in id order stops at its first w == wmin hit; a
          // row of <= 32 KB bounds the no-hit case at 32 rounds of 4 KB)
          owner = pull && mopen <= p.owner_cols && p.adjT_stride * sizeof(W) <= 32768;
          dk = d;
          fb = final_bound(d);
          // push: a tile none of whose columns is open after B_d skips the rows
          if (!pull) {
            const uint32_t lim = (uint32_t)umin64((uint64_t)d + p.wmin, (uint64_t)DINF - 1u);
            bool open = false;
            for (uint32_t col = tid; col < T; col += kBucketThreads)
              open |= !((ssettled[col >> 5] >> (col & 31)) & 1u) && sdist[col] > lim;
            relax = __syncthreads_or(open);
            spread = spread_ok(bcount);
          }
        }
      }
    }
    if (!MULTI && done) break;

    if ((relax || spread) && !pull) {
      // ---- PUSH: stream the rows of B_d (ascending ids), per-column min key
      pushed += bcount;
      // sparse lists: per class row its tile's (column, w) entries, folded
      // into one per-column key array by shared atomicMin (the minimum of
      // (w, u) keys does not depend on the order); dense: every class row's
      // slice of this tile
      const bool sparse = SP && sizeof(W) <= 2 && p.sp_off != nullptr;
      constexpr uint32_t WB = sizeof(W) <= 2 ? 8u * (uint32_t)sizeof(W) : 16u, WM = (1u << WB) - 1u;
      if (spread) {
        // warp gw of the slot walks B_d bitmap words gw, gw + GW, ...: lane l
        // loads the extent of the row at bit l, then the warp walks each set
        // bit's entry list (no id enumeration; row loads overlap across bits)
        const uint32_t GW = Gs * (kBucketThreads / 32), gw = bx * (kBucketThreads / 32) + warp;
        uint32_t nb = 0;
        for (uint32_t wi = gw; wi < words; wi += GW) {
          const uint32_t bits = sbm[wi];
          if (!bits) continue;  // warp-uniform
          const bool mine = (bits >> lane) & 1u;
          const uint32_t u = mine ? gvid(wi * 32 + lane) : 0u;
          const uint32_t b = mine ? __ldg(p.sp_off + (size_t)u * G) : 0u;
          const uint32_t e = mine ? __ldg(p.sp_off + (size_t)(u + 1) * G) : 0u;
          nb += mine ? 8u + 4u * (e - b) : 0u;
          for (uint32_t mm = bits; mm; mm &= mm - 1) {
            const uint32_t j = (uint32_t)(__ffs(mm) - 1);
            const uint32_t uj = __shfl_sync(0xFFFFFFFFu, u, j);
            const uint32_t bj = __shfl_sync(0xFFFFFFFFu, b, j), ej = __shfl_sync(0xFFFFFFFFu, e, j);
            for (uint32_t i = bj + lane; i < ej; i += 32) {
              const uint32_t ent = __ldg(p.sp_ent + i);
              smem_min(&pkey[ent >> WB], KT::make(ent & WM, uj));
            }
          }
        }
        nb = __reduce_add_sync(0xFFFFFFFFu, nb);
        if (lane == 0) atomicAdd(&s_spb, (unsigned long long)nb);
      } else if (sparse) {
        for (uint32_t col = tid; col < T; col += kBucketThreads) scomb[col] = KT::kNone;
      } else {
        my_bytes += (uint64_t)bcount * T * sizeof(W);
      }
      const uint32_t rg = tid / TPR, ct = tid - rg * TPR;  // row group, column thread
      K best[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) best[j] = KT::kNone;
      // enumerate B_d in ascending order with one block scan per pass: a
      // class of <= kIdCap ids takes a single pass over all words (up to 8
      // per thread), otherwise passes of one word per thread (<= kIdCap ids
      // each); the rest of the chunk region stages the row slices
      constexpr uint32_t WMAX = 8;
      const uint32_t wpt = (bcount <= kIdCap && words <= WMAX * kBucketThreads)
                               ? (words + kBucketThreads - 1) / kBucketThreads
                               : 1u;
      for (uint32_t wbase = spread ? words : 0u; wbase < words; wbase += kBucketThreads * wpt) {
        uint32_t tot;
        if (ids_n != 0xFFFFFFFFu) {  // class 1 from the row summary: ids already in schunk
          tot = ids_n;
          ids_n = 0xFFFFFFFFu;
          wbase = words;  // one pass
        } else {
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
        uint32_t wofs = 0;
        tot = 0;
        for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) {
          if (w2 < warp) wofs += s_red[w2];
          tot += s_red[w2];
        }
        uint32_t o = wofs + incl - c;
#pragma unroll
        for (uint32_t k2 = 0; k2 < WMAX; ++k2)
          for (uint32_t m = bw[k2]; m; m &= m - 1)
            schunk[o++] = gvid((w0 + k2) * 32 + (__ffs(m) - 1));
        }
        stamp(4);
        if (kBucketAB && !p.push_ldg) {
          // Row slices staged by bulk copies: thread t issues the copies of
          // rows t, t+256, ... of a batch (one UBLKCP per row slice); a batch
          // is every row of the pass when it fits the stage, else the stage
          // is split in two and batch b+2 is issued while b+1 is in flight.
          const uint32_t TB = T * (uint32_t)sizeof(W);
          uint8_t* const stage = reinterpret_cast<uint8_t*>(schunk + bucket_round4(tot));
          const uint32_t SB = (kBucketChunk - bucket_round4(tot)) * 4u;
          const uint32_t RB = tot * TB <= SB ? tot : (SB / 2u) / TB;  // rows per batch
          const uint32_t nbt = (tot + RB - 1u) / RB;
          auto buf = [&](uint32_t b) { return stage + (size_t)(b & 1u) * RB * TB; };
          auto issue = [&](uint32_t b) {
            const uint32_t r0 = b * RB, nr = min(RB, tot - r0);
            if (tid == 0) mbar_arrive_expect_tx(&s_mbar[b & 1u], nr * TB);
            for (uint32_t r = tid; r < nr; r += kBucketThreads)
              bulk_g2s(buf(b) + r * TB,
                       reinterpret_cast<const uint8_t*>(adj + (size_t)schunk[r0 + r] * p.row_stride + p0),
                       TB, &s_mbar[b & 1u]);
          };
          fence_proxy_async();  // earlier generic accesses of the stage bytes
          __syncthreads();
          issue(0);
          if (nbt > 1) issue(1);
          for (uint32_t b = 0; b < nbt; ++b) {
            mbar_wait(&s_mbar[b & 1u], (mph >> (b & 1u)) & 1u);
            mph ^= 1u << (b & 1u);
            const uint8_t* sb = buf(b);
            const uint32_t r0 = b * RB, nr = min(RB, tot - r0);
#pragma unroll 4
            for (uint32_t r = rg; r < nr; r += RG) {
              const uint4 v = *reinterpret_cast<const uint4*>(sb + r * TB + ct * 16);
              const uint32_t u = schunk[r0 + r];
              const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < CPT; ++j) {
                const K k = chunk_key<W>(wd[(j * sizeof(W)) / 4], j, u);
                best[j] = k < best[j] ? k : best[j];
              }
            }
            if (b + 2 < nbt) {
              fence_proxy_async();
              __syncthreads();  // batch b's buffer is free
              issue(b + 2);
            }
          }
          __syncthreads();
          continue;
        }
        __syncthreads();
        // batches of DEPTH rows per thread: all loads of a batch are issued
        // before any is consumed; a class of <= 16 rows per row group takes
        // one 16-deep batch (one memory round trip), larger ones 8-deep batches
        auto batches = [&](auto depth_c) {
          constexpr int DEPTH = decltype(depth_c)::value;
          for (uint32_t r0 = rg; r0 < tot; r0 += DEPTH * RG) {
            uint32_t ub[DEPTH];
            uint4 vb[DEPTH];
#pragma unroll
            for (int m = 0; m < DEPTH; ++m) {
              const uint32_t r = r0 + m * RG;
              ub[m] = r < tot ? schunk[r] : 0xFFFFFFFFu;
              if (r < tot)
                vb[m] = __ldg(reinterpret_cast<const uint4*>(
                    reinterpret_cast<const uint8_t*>(adj + (size_t)ub[m] * p.row_stride + p0) + ct * 16));
            }
            if constexpr (sizeof(W) == 1) {
              // u8: rows in pairs through the 3-input minimum (VIMNMX3): one
              // PRMT per key + half a min instead of a whole one; an odd last
              // row of the class takes the 2-input minimum.
#pragma unroll
              for (int m = 0; m < DEPTH; m += 2) {
                if (ub[m] == 0xFFFFFFFFu) break;
                const uint32_t w0[4] = {vb[m].x, vb[m].y, vb[m].z, vb[m].w};
                if (ub[m + 1] != 0xFFFFFFFFu) {
                  const uint32_t w1[4] = {vb[m + 1].x, vb[m + 1].y, vb[m + 1].z, vb[m + 1].w};
#pragma unroll
                  for (int j = 0; j < CPT; ++j)
                    best[j] = __vimin3_u32(best[j], chunk_key<W>(w0[j / 4], j, ub[m]),
                                           chunk_key<W>(w1[j / 4], j, ub[m + 1]));
                } else {
#pragma unroll
                  for (int j = 0; j < CPT; ++j) best[j] = min(best[j], chunk_key<W>(w0[j / 4], j, ub[m]));
                }
              }
            } else {
#pragma unroll
            for (int m = 0; m < DEPTH; ++m) {
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
          }
        };
        if (sparse) {
          // 4 rows per thread in flight: the extents of all four, then the
          // first entry of each (most rows hold 0 or 1 entries in a tile), then
          // the rare remainder
          const uint32_t* const off = p.sp_off + me;  // + u * G
          uint32_t nb = 0;
          for (uint32_t r0 = tid; r0 < tot; r0 += 4 * kBucketThreads) {
            uint32_t ub[4], b[4], e[4], f[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const uint32_t r = r0 + m * kBucketThreads;
              ub[m] = r < tot ? schunk[r] : 0u;
              b[m] = r < tot ? __ldg(off + (size_t)ub[m] * G) : 0u;
              e[m] = r < tot ? __ldg(off + (size_t)ub[m] * G + 1) : 0u;
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) f[m] = b[m] < e[m] ? __ldg(p.sp_ent + b[m]) : 0u;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              nb += 8u + 4u * (e[m] - b[m]);
              if (b[m] < e[m]) smem_min(&scomb[(f[m] >> WB) - p0], KT::make(f[m] & WM, ub[m]));
              for (uint32_t i = b[m] + 1; i < e[m]; ++i) {
                const uint32_t ent = __ldg(p.sp_ent + i);
                smem_min(&scomb[(ent >> WB) - p0], KT::make(ent & WM, ub[m]));
              }
            }
          }
          nb = __reduce_add_sync(0xFFFFFFFFu, nb);
          if (lane == 0) atomicAdd(&s_spb, (unsigned long long)nb);
        } else if (kBucketAB && p.push_depth16 && tot > 8 * RG && tot <= 16 * RG)
          batches(std::integral_constant<int, 16>{});
        else
          batches(std::integral_constant<int, 8>{});
        __syncthreads();
        stamp(5);
      }
      // fold the row groups that share a warp with shuffles first (TPR < 32:
      // 32/TPR groups per warp), so the cross-warp combine reads one partial
      // per warp instead of one per row group
      const uint32_t gpw = TPR < 32 ? 32u / TPR : 1u;  // row groups per warp
      if (!spread) {
      for (uint32_t o = TPR; !sparse && o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const K x = __shfl_xor_sync(0xFFFFFFFFu, best[j], o);
          best[j] = x < best[j] ? x : best[j];
        }
      }
      if (!sparse && (gpw == 1 || lane < TPR)) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) scomb[((rg / gpw) * TPR + ct) * CPT + j] = best[j];
      }
      __syncthreads();
      const uint32_t ngrp = sparse ? 1u : RG / gpw;  // sparse: group 0's slots = scomb[col]
      for (uint32_t col = tid; col < T; col += kBucketThreads) {
        const uint32_t cth = col / CPT, j = col % CPT;
        K k = KT::kNone;
        for (uint32_t g2 = 0; g2 < ngrp; ++g2) {
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
      }
      stamp(6);
    } else if (relax && owner) {
      // ---- PULL on the column owners (small pulls), in ascending vertex id.
      // An open column's transposed row is read id-block by id-block: a round
      // is 256 16 B chunks = chunk b of every participant run (ids
      // [b*CPT*Q, (b+1)*CPT*Q) of a shard, since position q*L + s holds vertex
      // s*Q + q), and the column is final as soon as its minimum so far has
      // w == wmin -- no later (larger) id can beat it: a smaller w does not
      // exist and an equal w loses the lowest-id tie (serial.hpp:46, 56).
      // Dense classes hit in the first round (~4 KB instead of the row).  Up
      // to 4 columns share a round; nothing is combined across CTAs, so the
      // step needs no extra barrier.
      pulled += ucount;
      const uint32_t lim = (uint32_t)umin64((uint64_t)dk + p.wmin, (uint64_t)DINF - 1u);
      uint32_t* ocol = reinterpret_cast<uint32_t*>(scomb);      // open columns of the tile
      K* skey = reinterpret_cast<K*>(ocol + ((T + 3u) & ~3u));  // [4][8] warp minima + [4] result
      __shared__ uint32_t s_odone[4];
      if (tid == 0) s_cnt[0] = 0;
      __syncthreads();
      for (uint32_t col = tid; col < T; col += kBucketThreads)
        if (!((ssettled[col >> 5] >> (col & 31)) & 1u) && sdist[col] > lim)
          ocol[atomicAdd(&s_cnt[0], 1u)] = col;
      __syncthreads();
      const uint32_t no = s_cnt[0];
      uint32_t nld = 0;  // 16 B chunks this thread loaded
      const uint32_t nbits = p.lbits - (31u - __clz((uint32_t)CPT));  // log2(L / CPT)
      const uint32_t total = nsh << (nbits + p.qbits);           // chunks per row
      for (uint32_t c0 = 0; c0 < no; c0 += 4) {
        const uint32_t nc = min(4u, no - c0);
        const uint8_t* rows[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          const uint32_t pos = p0 + ocol[c0 + min(k, nc - 1)];
          const uint32_t v = p.adjT_by_pos ? pos : pos_to_vid(pos, p.Q, p.lbits, p.qbits);
          rows[k] = reinterpret_cast<const uint8_t*>(adjT + (size_t)v * p.adjT_stride);
        }
        K best[4] = {KT::kNone, KT::kNone, KT::kNone, KT::kNone};
        if (tid < 4) s_odone[tid] = tid >= nc ? 1u : 0u;
        __syncthreads();
        for (uint32_t base = 0; base < total; base += kBucketThreads) {
          const uint32_t it = base + tid;
          uint32_t bits = 0, g = 0;
          uint4 v4[4];
          if (it < total) {
            const uint32_t q = it & (p.Q - 1u), t2 = it >> p.qbits;
            const uint32_t b = t2 & ((1u << nbits) - 1u), j = t2 >> nbits;
            g = j * (uint32_t)p.row_stride + (q << p.lbits) + b * CPT;
            bits = (sbm[g >> 5] >> (g & 31)) & ((1u << CPT) - 1u);
            if (bits) {
#pragma unroll
              for (uint32_t k = 0; k < 4; ++k)
                if (!s_odone[k]) {
                  v4[k] = __ldg(reinterpret_cast<const uint4*>(rows[k] + (size_t)g * sizeof(W)));
                  ++nld;
                }
            }
          }
          if (bits) {
            const uint32_t vid0 = gvid(g);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
              if (!s_odone[k]) {
                const K kk = chunk_min(v4[k], bits, vid0);
                best[k] = kk < best[k] ? kk : best[k];
              }
          }
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k) {
            const K kk = warp_min_key(best[k]);
            if (lane == 0) skey[k * 8 + warp] = kk;
          }
          __syncthreads();
          if (tid < nc && !s_odone[tid]) {
            K m = skey[tid * 8];
            for (uint32_t w2 = 1; w2 < kBucketThreads / 32; ++w2) {
              const K x = skey[tid * 8 + w2];
              m = x < m ? x : m;
            }
            skey[32 + tid] = m;
            if (m != KT::kNone && KT::w(m) == p.wmin) s_odone[tid] = 1u;  // final
          }
          __syncthreads();
          if (s_odone[0] & s_odone[1] & s_odone[2] & s_odone[3]) break;  // uniform
        }
        if (tid < nc) {  // apply (strict '<': serial.hpp:56)
          const K m = skey[32 + tid];
          const uint32_t col = ocol[c0 + tid];
          if (m != KT::kNone && KT::w(m) != WINF) {
            const uint32_t cand = dk + KT::w(m);
            if (cand < sdist[col]) {
              sdist[col] = cand;
              spred[col] = KT::u(m);
            }
          }
        }
        __syncthreads();
      }
      nld = __reduce_add_sync(0xFFFFFFFFu, nld);
      if (lane == 0) s_red[warp] = nld;
      __syncthreads();
      for (uint32_t w2 = 0; w2 < kBucketThreads / 32; ++w2) my_bytes += 16ull * s_red[w2];
      __syncthreads();
      stamp(13);
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
      {  // this shard's published open-column bitmap (the pull work list)
        const uint32_t* ub = ubm + par * lwords;
        for (uint32_t i = tid; i < lwords; i += kBucketThreads) sub[i] = __ldcg(&ub[i]);
        __syncthreads();
      }
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
      my_bytes += 16ull * (hi - lo);  // every item of the range is streamed
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
      stamp(7);
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
          const K kk = chunk_min(st[m * kBucketThreads + tid], bits, gvid(pos0));
          run = kk < run ? kk : run;
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
    if ((pull && !owner) || spread || MULTI) {
      stamp(8);
      barrier();
      stamp(1);
    }
    if ((relax && pull && !owner) || spread) {
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
      stamp(9);
      publish((uint32_t)((bar_base + nbar) & 1ull), fb);
    } else if (MULTI && bx == 0 && tid == 0) {
      p.done[slot] = 1;  // read by every slot after the barrier
    }
    barrier();
    stamp(1);
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
  stamp(11);
  if (p.spans && tid == 0) {  // debug: launch span = (min CTA start, max CTA end), %globaltimer
    atomicMax(&p.spans[(p.seq % 64) * 2], ~(unsigned long long)t_start);
    atomicMax(&p.spans[(p.seq % 64) * 2 + 1], (unsigned long long)globaltimer());
  }
  if (p.trace && tid == 0 && slot == 0 && me < 1024) {  // debug: every CTA's start / end
    p.trace[64 + 2048 + 2 * me] = t_start;
    p.trace[64 + 2048 + 2 * me + 1] = globaltimer();
  }
  if (bx == 0 && tid == 0) {
    uint64_t* const info = S.info + slot * 4;
    info[0] = settled;
    info[1] = step | (bailed ? 1ull << 63 : 0ull);
    info[2] = pushed;
    info[3] = pulled;
    S.info2[slot * 2] = nbar;
  }
  if (S.cta_bytes) {
    if (tid == 0) S.cta_bytes[slot * p.ctab_stride + bx] = my_bytes + (SP ? s_spb : 0ull);
    if (bx == 0)  // entries of a wider tiling's CTAs (not in this launch) read as 0
      for (uint32_t i = Gs + tid; i < p.ctab_stride; i += kBucketThreads) S.cta_bytes[slot * p.ctab_stride + i] = 0;
  }
  if (bx == 0 && tid == 0) {
    if (cross && blockIdx.x == 0) *p.bar_epoch = bar_base + nbar;  // every CTA read it before barrier 1
  }
}

// ---- upload-time row scans (one shard).  Rows are read as 16 B chunks: a
// chunk is CPT consecutive positions of one participant run, i.e. vertices
// vid0, vid0 + Q, ... (L >= CPT, so a chunk never straddles runs).  A chunk
// that holds the row's own vertex or padding positions takes the per-element
// path; every other chunk is folded with byte-SIMD (u8) or per element.

// exact count of zero bytes of x
__device__ __forceinline__ uint32_t zero_bytes(uint32_t x) {
  return __popc(~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu));
}
// 4-bit mask of the zero bytes of x (bit k = byte k)
__device__ __forceinline__ uint32_t zero_byte_mask(uint32_t x) {
  const uint32_t z = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
  return (((z >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// vertices of chunk j that are real columns of row u: a CPT-bit mask
template <typename W>
__device__ __forceinline__ uint32_t chunk_valid_mask(uint32_t j, uint32_t u, uint32_t n, uint32_t Q,
                                                     uint32_t qbits, uint32_t lbits, uint32_t& vid0) {
  constexpr uint32_t CPT = 16 / sizeof(W);
  vid0 = pos_to_vid(j * CPT, Q, lbits, qbits);
  uint32_t mask = 0;
#pragma unroll
  for (uint32_t k = 0; k < CPT; ++k) {
    const uint32_t v = vid0 + k * Q;
    mask |= (v < n && v != u) ? 1u << k : 0u;
  }
  return mask;
}

// Row summaries for class 1 (bucket_kernel's exchange-free first class, one
// shard): for source u, exactly the values the exchange after class 0 yields
// (dist after class 0 = row u, source and padding settled):
//   [0] d1 = min finite w(u, v) over v != u (DINF: none)   [1] |B_1| = #{v : w == d1}
//   [2] open columns after B_1: #{v : dist > fb0} minus B_1 when d1 > fb0
//       (fb0 = 1 + wmin, final_bound(0); INF counts as open)
//   [3] finite columns #{v : w != INF}
// One CTA per row, ONE pass of 16 B loads: every thread keeps a running
// (min, count at min) pair, combined across the CTA at the end.  Run once at
// upload.
template <typename W>
__global__ void __launch_bounds__(256) row_summary_kernel(const W* __restrict__ adj, uint64_t row_stride,
                                                          uint32_t n, uint32_t Q, uint32_t qbits,
                                                          uint32_t lbits, uint32_t fb0, uint4* out) {
  // out: [n][2] uint4 (second: list offset, written by the host)
  constexpr uint32_t WINF = WInf<W>::v, DINF = 0xFFFFFFFFu;
  constexpr uint32_t CPT = 16 / sizeof(W);
  __shared__ uint32_t s_r[5][8];
  const uint32_t u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint4* row4 = reinterpret_cast<const uint4*>(adj + (size_t)u * row_stride);
  const uint32_t nch = (uint32_t)(row_stride / CPT);
  const uint32_t pos_src = ((u & (Q - 1u)) << lbits) | (u >> qbits);
  const bool padded = n < row_stride;
  uint32_t m = DINF, c = 0, fin = 0, gt = 0;
  auto fold = [&](uint32_t d, uint32_t k) {  // one candidate distance d with multiplicity k
    c = d < m ? k : (d == m ? c + k : c);
    m = min(m, d);
  };
  auto chunk = [&](uint32_t j, const uint4 v) {
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
    uint32_t vid0 = 0;
    const uint32_t valid = (padded || j == pos_src / CPT)
                               ? chunk_valid_mask<W>(j, u, n, Q, qbits, lbits, vid0)
                               : (1u << CPT) - 1u;
    if (sizeof(W) == 1 && valid == 0xFFFFu) {
      // byte-SIMD: chunk minimum on 16x2 lanes, then counts of its bytes
      uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mn = __vminu2(mn, __vminu2(wd[k] & 0x00FF00FFu, __byte_perm(wd[k], 0u, 0x4341u)));
      const uint32_t cm = min(mn & 0xFFFFu, mn >> 16);
      const uint32_t cmx = cm * 0x01010101u;
      const uint32_t K = (0x7FFFu - min(fb0, 0xFEu)) * 0x00010001u;  // lane > fb0 <=> bit 15 of lane + K
      uint32_t ninf = 0, neq = 0, ngt = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ninf += zero_bytes(~wd[k]);
        neq += zero_bytes(wd[k] ^ cmx);
        ngt += __popc(((wd[k] & 0x00FF00FFu) + K) & 0x80008000u) +
               __popc((__byte_perm(wd[k], 0u, 0x4341u) + K) & 0x80008000u);
      }
      fin += 16u - ninf;
      gt += fb0 >= 0xFFu ? ninf : ngt;  // fb0 >= INF byte: only INF columns are open
      if (cm != 0xFFu) fold(cm, neq);
      return;
    }
#pragma unroll
    for (uint32_t k = 0; k < CPT; ++k) {
      if (!((valid >> k) & 1u)) continue;
      const uint32_t w = sizeof(W) == 4 ? wd[k] : (wd[(k * sizeof(W)) / 4] >> (8 * sizeof(W) * (k % (4 / sizeof(W))))) & WINF;
      const uint32_t d = w != WINF ? w : DINF;
      fin += d != DINF ? 1u : 0u;
      gt += d > fb0 ? 1u : 0u;
      if (d != DINF) fold(d, 1u);
    }
  };
  uint32_t j = tid;
  for (; j + 3 * 256 < nch; j += 4 * 256) {  // four loads in flight per thread
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(row4 + j + k * 256);
#pragma unroll
    for (int k = 0; k < 4; ++k) chunk(j + k * 256, v[k]);
  }
  for (; j < nch; j += 256) chunk(j, __ldcs(row4 + j));
  // CTA combine of the (min, count) pairs and the counts
  const uint32_t wm = __reduce_min_sync(0xFFFFFFFFu, m);
  const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, m == wm ? c : 0u);
  fin = __reduce_add_sync(0xFFFFFFFFu, fin);
  gt = __reduce_add_sync(0xFFFFFFFFu, gt);
  if (lane == 0) {
    s_r[0][warp] = wm;
    s_r[1][warp] = wc;
    s_r[2][warp] = gt;
    s_r[3][warp] = fin;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t mm = DINF;
    for (int w2 = 0; w2 < 8; ++w2) mm = min(mm, s_r[0][w2]);
    uint4 r = make_uint4(mm, 0, 0, 0);
    for (int w2 = 0; w2 < 8; ++w2) {
      r.y += s_r[0][w2] == mm ? s_r[1][w2] : 0u;
      r.z += s_r[2][w2];
      r.w += s_r[3][w2];
    }
    if (mm == DINF) r.y = 0;
    else if (mm > fb0) r.z -= r.y;  // B_1 itself is settled, not open
    out[2 * u] = r;
  }
}

// Class-1 id list of row u (rsum[u][4] != ~0u): the vertices v != u with
// w(u, v) == d1, in any order (the class-1 push takes a per-column minimum of
// (w, u) keys, which does not depend on the order).  One CTA per row, 16 B
// loads; ids are placed by one shared atomic per warp and pass.
template <typename W>
__global__ void __launch_bounds__(256) row_list_kernel(const W* __restrict__ adj, uint64_t row_stride,
                                                       uint32_t n, uint32_t Q, uint32_t qbits, uint32_t lbits,
                                                       const uint32_t* __restrict__ rsum, uint32_t* list) {
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t CPT = 16 / sizeof(W);
  const uint32_t u = blockIdx.x, lane = threadIdx.x & 31;
  const uint32_t off = rsum[(size_t)u * 8 + 4], d1 = rsum[(size_t)u * 8];
  if (off == 0xFFFFFFFFu) return;
  __shared__ uint32_t s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const uint4* row4 = reinterpret_cast<const uint4*>(adj + (size_t)u * row_stride);
  const uint32_t nch = (uint32_t)(row_stride / CPT);
  const uint32_t pos_src = ((u & (Q - 1u)) << lbits) | (u >> qbits);
  const bool padded = n < row_stride;
  const uint32_t nrounds = (nch + 255u) / 256u;  // warp-uniform trip count
  for (uint32_t rd = 0; rd < nrounds; ++rd) {
    const uint32_t j = rd * 256u + threadIdx.x;
    uint32_t mask = 0, vid0 = pos_to_vid(j * CPT, Q, lbits, qbits);
    if (j < nch) {
      const uint4 v = __ldcs(row4 + j);
      const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
      if constexpr (sizeof(W) == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) mask |= zero_byte_mask(wd[k] ^ (d1 * 0x01010101u)) << (4 * k);
      } else {
#pragma unroll
        for (uint32_t k = 0; k < CPT; ++k) {
          const uint32_t w = sizeof(W) == 4 ? wd[k] : (wd[k / 2] >> (16 * (k % 2))) & WINF;
          mask |= w == d1 ? 1u << k : 0u;
        }
      }
      if (mask && (padded || j == pos_src / CPT)) mask &= chunk_valid_mask<W>(j, u, n, Q, qbits, lbits, vid0);
    }
    const uint32_t cnt = __popc(mask);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    const uint32_t wtot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (wtot == 0) continue;
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(&s_n, wtot);
    base = __shfl_sync(0xFFFFFFFFu, base, 31) + incl - cnt;
    for (uint32_t mm = mask; mm; mm &= mm - 1) list[off + base++] = vid0 + (uint32_t)(__ffs(mm) - 1) * Q;
  }
}

// Sparse tile lists (BucketParams::sp_off / sp_ent), two passes over the
// matrix, one CTA per row u: COUNT writes cnt[u*G+t] = the finite real
// entries of row u in tile t (positions [t*T, (t+1)*T)), cnt[n*G] = 0; an
// exclusive scan turns cnt into offsets (lists in (row, tile) order); FILL places each entry (position - t*T) << 16 | w
// (position << 8*sizeof(W) | w) behind its tile's cursor (order inside a list
// is free: the push takes a per-column minimum).  Per-tile counters live in shared memory (G <= 1024).
template <typename W, bool FILL>
__global__ void __launch_bounds__(256) tile_list_kernel(const W* __restrict__ adj, uint64_t row_stride,
                                                        uint32_t n, uint32_t Q, uint32_t qbits, uint32_t lbits,
                                                        uint32_t T, uint32_t G, uint32_t* cnt_off,
                                                        uint32_t* ent) {
  constexpr uint32_t WINF = WInf<W>::v;
  constexpr uint32_t CPT = 16 / sizeof(W);
  const uint32_t u = blockIdx.x;
  __shared__ uint32_t sc[1024];
  for (uint32_t t = threadIdx.x; t < G; t += 256)
    sc[t] = FILL ? cnt_off[(size_t)u * G + t] : 0u;
  __syncthreads();
  const uint4* row4 = reinterpret_cast<const uint4*>(adj + (size_t)u * row_stride);
  const uint32_t nch = (uint32_t)(row_stride / CPT);
  const uint32_t pos_src = ((u & (Q - 1u)) << lbits) | (u >> qbits);
  const bool padded = n < row_stride;
  for (uint32_t j = threadIdx.x; j < nch; j += 256) {
    const uint4 v = __ldcs(row4 + j);
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
    uint32_t mask = 0, vid0;
    if constexpr (sizeof(W) == 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mask |= (zero_byte_mask(~wd[k]) ^ 0xFu) << (4 * k);
    } else {
#pragma unroll
      for (uint32_t k = 0; k < CPT; ++k) {
        const uint32_t w = sizeof(W) == 4 ? wd[k] : (wd[k / 2] >> (16 * (k % 2))) & WINF;
        mask |= w != WINF ? 1u << k : 0u;
      }
    }
    if (mask && (padded || j == pos_src / CPT)) mask &= chunk_valid_mask<W>(j, u, n, Q, qbits, lbits, vid0);
    if (!mask) continue;
    const uint32_t t = (j * CPT) / T;
    if (!FILL) {
      atomicAdd(&sc[t], (uint32_t)__popc(mask));
    } else {
      for (uint32_t mm = mask; mm; mm &= mm - 1) {
        const uint32_t k = (uint32_t)(__ffs(mm) - 1);
        const uint32_t w = sizeof(W) == 1 ? (wd[k / 4] >> (8 * (k % 4))) & 0xFFu
                                          : (wd[k / 2] >> (16 * (k % 2))) & 0xFFFFu;
        ent[atomicAdd(&sc[t], 1u)] = ((j * CPT + k) << (8 * sizeof(W))) | w;
      }
    }
  }
  if (!FILL) {
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < G; t += 256) cnt_off[(size_t)u * G + t] = sc[t];
    if (u == 0 && threadIdx.x == 0) cnt_off[(size_t)n * G] = 0u;  // terminator: the end of the last list
  }
}

#ifndef SSSP_BUCKET_INSTANCES_ONLY
// The bucket engine's synchronisation skeleton (bench roofline): the same
// cooperative launch shape and shared memory, `nbar` grid barriers, no data.
// Its time per launch is the floor under a solve with that many barriers.
__global__ void __launch_bounds__(kBucketThreads, 2) bucket_skeleton_kernel(uint32_t nbar,
                                                                             uint32_t* sink) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // as bucket_kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) uint32_t smem[];
  if (threadIdx.x == 0) smem[0] = blockIdx.x;
  for (uint32_t i = 0; i < nbar; ++i) cooperative_groups::this_grid().sync();
  if (threadIdx.x == 0 && smem[0] == 0xFFFFFFFFu) sink[0] = 1;
}
#endif

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

// The same check on 128 B row segments: a tile is TL = 128 / sizeof(W)
// positions square, read with 16 B loads (one full line per tile row), the
// first tile staged in shared memory, the mirror tile compared from registers
// against its transpose there.  Needs row_stride % TL == 0 (else the kernel
// above).
template <typename W>
__global__ void __launch_bounds__(256) symmetric_check_wide_kernel(const W* __restrict__ a,
                                                                   uint64_t row_stride, uint32_t n,
                                                                   uint32_t Q, uint32_t qbits,
                                                                   uint32_t lbits, uint32_t* flag) {
  constexpr uint32_t TL = 128 / sizeof(W), CPT = 16 / sizeof(W), CPR = 8;  // chunks per tile row
  constexpr uint32_t NCH = TL * CPR / 256;                                 // chunks per thread
  if (blockIdx.y < blockIdx.x) return;
  __shared__ W tile[TL][TL + 1];
  const uint32_t pb = blockIdx.x * TL, ppb = blockIdx.y * TL;
  uint4 v[NCH];
#pragma unroll
  for (uint32_t k = 0; k < NCH; ++k) {  // tile (rows vid(ppb + r), positions pb + ...)
    const uint32_t i = threadIdx.x + k * 256, r = i / CPR, ch = i % CPR;
    const uint32_t uu = pos_to_vid(ppb + r, Q, lbits, qbits);
    v[k] = uu < n ? __ldcs(reinterpret_cast<const uint4*>(a + (size_t)uu * row_stride + pb) + ch)
                  : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  }
  uint4 m4[NCH];
#pragma unroll
  for (uint32_t k = 0; k < NCH; ++k) {  // mirror tile (rows vid(pb + r), positions ppb + ...)
    const uint32_t i = threadIdx.x + k * 256, r = i / CPR, ch = i % CPR;
    const uint32_t vv = pos_to_vid(pb + r, Q, lbits, qbits);
    m4[k] = vv < n ? __ldcs(reinterpret_cast<const uint4*>(a + (size_t)vv * row_stride + ppb) + ch)
                   : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (uint32_t k = 0; k < NCH; ++k) {
    const uint32_t i = threadIdx.x + k * 256, r = i / CPR, ch = i % CPR;
    const W* e = reinterpret_cast<const W*>(&v[k]);
#pragma unroll
    for (uint32_t x = 0; x < CPT; ++x) tile[r][ch * CPT + x] = e[x];
  }
  __syncthreads();
  bool diff = false;
#pragma unroll
  for (uint32_t k = 0; k < NCH; ++k) {
    const uint32_t i = threadIdx.x + k * 256, r = i / CPR, ch = i % CPR;
    if (pos_to_vid(pb + r, Q, lbits, qbits) >= n) continue;
    const W* e = reinterpret_cast<const W*>(&m4[k]);
#pragma unroll
    for (uint32_t x = 0; x < CPT; ++x) {
      const uint32_t c = ch * CPT + x;
      if (pos_to_vid(ppb + c, Q, lbits, qbits) < n) diff |= e[x] != tile[c][r];
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
