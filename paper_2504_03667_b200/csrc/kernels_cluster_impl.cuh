// kernels_cluster_impl.cuh -- instance tables of the cluster engine
// (cluster_kernel.cuh) for one value of MS (several shards per launch).
// Included by kernels_cluster.cu (MS = false) and kernels_cluster_ms.cu
// (MS = true), compiled in parallel.
#pragma once

#include "cluster_kernel.cuh"
#include "dispatch.h"

namespace sssp_b200 {
namespace cluster_tables {

template <typename W, int EPL, bool PK, bool TR, bool MS>
KernelFn pick_nw(int nw) {
  switch (nw) {
    case 4: return cluster_scan_kernel<W, EPL, 4, PK, TR, MS>;
    case 8: return cluster_scan_kernel<W, EPL, 8, PK, TR, MS>;
    case 16: return cluster_scan_kernel<W, EPL, 16, PK, TR, MS>;
  }
  return nullptr;
}

template <typename W, bool PK, bool TR, bool MS>
KernelFn pick_epl(int epl, int nw) {
  switch (epl) {
    case 4: return pick_nw<W, 4, PK, TR, MS>(nw);
    case 8: return pick_nw<W, 8, PK, TR, MS>(nw);
    case 16: return pick_nw<W, 16, PK, TR, MS>(nw);
    case 32: return pick_nw<W, 32, PK, TR, MS>(nw);
  }
  return nullptr;
}

template <bool PK, bool TR, bool MS>
KernelFn pick_w(int wbytes, int epl, int nw) {
  switch (wbytes) {
    case 1: return pick_epl<uint8_t, PK, TR, MS>(epl, nw);
    case 2: return pick_epl<uint16_t, PK, TR, MS>(epl, nw);
    case 4: return pick_epl<uint32_t, PK, TR, MS>(epl, nw);
  }
  return nullptr;
}

template <bool MS>
ProbeFn probe(int nw, bool hier) {
  switch (nw) {
    case 4: return hier ? cluster_probe_kernel<4, true, MS> : cluster_probe_kernel<4, false, MS>;
    case 8: return hier ? cluster_probe_kernel<8, true, MS> : cluster_probe_kernel<8, false, MS>;
    case 16: return hier ? cluster_probe_kernel<16, true, MS> : cluster_probe_kernel<16, false, MS>;
  }
  return nullptr;
}

template <typename W, int EPL, bool MS>
KernelFn pick_hier_nw(int nw) {
  switch (nw) {
    case 4: return cluster_hier_kernel<W, EPL, 4, MS>;
    case 8: return cluster_hier_kernel<W, EPL, 8, MS>;
    case 16: return cluster_hier_kernel<W, EPL, 16, MS>;
  }
  return nullptr;
}
template <typename W, bool MS>
KernelFn pick_hier_epl(int epl, int nw) {
  switch (epl) {
    case 4: return pick_hier_nw<W, 4, MS>(nw);
    case 8: return pick_hier_nw<W, 8, MS>(nw);
    case 16: return pick_hier_nw<W, 16, MS>(nw);
    case 32: return pick_hier_nw<W, 32, MS>(nw);
  }
  return nullptr;
}
template <bool MS>
KernelFn hier(int wbytes, int epl, int nw) {
  switch (wbytes) {
    case 1: return pick_hier_epl<uint8_t, MS>(epl, nw);
    case 2: return pick_hier_epl<uint16_t, MS>(epl, nw);
    case 4: return pick_hier_epl<uint32_t, MS>(epl, nw);
  }
  return nullptr;
}

}  // namespace cluster_tables
}  // namespace sssp_b200
