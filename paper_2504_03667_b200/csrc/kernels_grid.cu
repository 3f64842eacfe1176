// kernels_grid.cu -- instances of the grid engine (scan_kernel.cuh).
#include "dispatch.h"

namespace sssp_b200 {
namespace {

template <typename W, int EPL, bool MS>
KernelFn pick_np(int np) {
  switch (np) {
    case 2: return scan_dijkstra_kernel<W, EPL, 2, MS>;
    case 4: return scan_dijkstra_kernel<W, EPL, 4, MS>;
    case 16: return scan_dijkstra_kernel<W, EPL, 16, MS>;
  }
  return nullptr;
}

template <typename W, bool MS>
KernelFn pick_epl(int epl, int np) {
  switch (epl) {
    case 4: return pick_np<W, 4, MS>(np);
    case 8: return pick_np<W, 8, MS>(np);
    case 16: return pick_np<W, 16, MS>(np);
    case 32: return pick_np<W, 32, MS>(np);
    case 64: return pick_np<W, 64, MS>(np);
  }
  return nullptr;
}

template <bool MS>
KernelFn pick_w(int wbytes, int epl, int np) {
  switch (wbytes) {
    case 1: return pick_epl<uint8_t, MS>(epl, np);
    case 2: return pick_epl<uint16_t, MS>(epl, np);
    case 4: return pick_epl<uint32_t, MS>(epl, np);
  }
  return nullptr;
}

template <bool MS>
ProbeFn probe(int np) {
  switch (np) {
    case 2: return exchange_probe_kernel<2, MS>;
    case 4: return exchange_probe_kernel<4, MS>;
    case 16: return exchange_probe_kernel<16, MS>;
  }
  return nullptr;
}

}  // namespace

KernelFn get_grid_kernel(int wbytes, int epl, int np, bool ms) {
  return ms ? pick_w<true>(wbytes, epl, np) : pick_w<false>(wbytes, epl, np);
}

ProbeFn get_grid_probe(int np, bool ms) { return ms ? probe<true>(np) : probe<false>(np); }

}  // namespace sssp_b200
