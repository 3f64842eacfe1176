// kernels_grid.cu -- instances of the grid engine (scan_kernel.cuh).
#include "dispatch.h"

namespace sssp_b200 {
namespace {

template <typename W, int EPL>
KernelFn pick_np(int np) {
  switch (np) {
    case 2: return scan_dijkstra_kernel<W, EPL, 2>;
    case 4: return scan_dijkstra_kernel<W, EPL, 4>;
    case 16: return scan_dijkstra_kernel<W, EPL, 16>;
  }
  return nullptr;
}

template <typename W>
KernelFn pick_epl(int epl, int np) {
  switch (epl) {
    case 4: return pick_np<W, 4>(np);
    case 8: return pick_np<W, 8>(np);
    case 16: return pick_np<W, 16>(np);
    case 32: return pick_np<W, 32>(np);
    case 64: return pick_np<W, 64>(np);
  }
  return nullptr;
}

}  // namespace

KernelFn get_grid_kernel(int wbytes, int epl, int np) {
  switch (wbytes) {
    case 1: return pick_epl<uint8_t>(epl, np);
    case 2: return pick_epl<uint16_t>(epl, np);
    case 4: return pick_epl<uint32_t>(epl, np);
  }
  return nullptr;
}

ProbeFn get_grid_probe(int np) {
  switch (np) {
    case 2: return exchange_probe_kernel<2>;
    case 4: return exchange_probe_kernel<4>;
    case 16: return exchange_probe_kernel<16>;
  }
  return nullptr;
}

}  // namespace sssp_b200
