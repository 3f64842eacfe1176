// Bucket-engine kernel instances for uint16_t weights (bucket_kernel.cuh), in their
// own translation unit so the three weight types compile in parallel.
#define SSSP_BUCKET_INSTANCES_ONLY
#include "bucket_kernel.cuh"

namespace sssp_b200 {
// variant 1: several solves (slots) of one shard; otherwise the general
// instance (any shard layout).  A one-shard single-solve instance (ONE) measured
// slower than the general one at config 3 (26.4 vs 24.7 us: register spills at
// the 128-register bound), so none is built.
void* bucket_fn_u16(int variant) {
  // variant 3: the sparse-list instance (one shard, single solves)
  if (variant == 3) return (void*)bucket_kernel<uint16_t, false, false, true>;
  return variant == 1 ? (void*)bucket_kernel<uint16_t, true, true> : (void*)bucket_kernel<uint16_t, false, false>;
}
}  // namespace sssp_b200
