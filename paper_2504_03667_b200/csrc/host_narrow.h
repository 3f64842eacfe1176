// host_narrow.h -- host worker pool and uint64 -> W row narrowing (upload).
#pragma once

#include <cstdint>
#include <functional>

namespace sssp_b200 {

struct NarrowStats {
  uint64_t max_w = 0;      // largest finite weight seen (diagonal included)
  uint64_t min_w = ~0ull;  // smallest finite OFF-diagonal weight seen
  uint64_t overflow = 0;   // nonzero: a finite weight does not fit W
};

unsigned narrow_threads();
// fn(t) for t in [0, narrow_threads()), on a persistent pool; t = 0 is the caller
void parallel_run(const std::function<void(unsigned)>& fn);

// Narrows rows [r0, r0+rows) x `cols` columns of src (leading dimension ld,
// global column offset col_base) into out (row-major, cols per row).
template <typename W>
NarrowStats narrow_rows(const uint64_t* src, uint64_t ld, uint64_t r0, uint64_t rows,
                        uint64_t cols, uint64_t col_base, W* out);

}  // namespace sssp_b200
