// kernels_cluster.cu -- instances of the cluster engine (cluster_kernel.cuh).
#include "cluster_kernel.cuh"
#include "dispatch.h"

namespace sssp_b200 {
namespace {

template <typename W, int EPL, bool PK, bool TR>
KernelFn pick_nw(int nw) {
  switch (nw) {
    case 4: return cluster_scan_kernel<W, EPL, 4, PK, TR>;
    case 8: return cluster_scan_kernel<W, EPL, 8, PK, TR>;
    case 16: return cluster_scan_kernel<W, EPL, 16, PK, TR>;
  }
  return nullptr;
}

template <typename W, bool PK, bool TR>
KernelFn pick_epl(int epl, int nw) {
  switch (epl) {
    case 4: return pick_nw<W, 4, PK, TR>(nw);
    case 8: return pick_nw<W, 8, PK, TR>(nw);
    case 16: return pick_nw<W, 16, PK, TR>(nw);
    case 32: return pick_nw<W, 32, PK, TR>(nw);
  }
  return nullptr;
}

template <bool PK, bool TR>
KernelFn pick_w(int wbytes, int epl, int nw) {
  switch (wbytes) {
    case 1: return pick_epl<uint8_t, PK, TR>(epl, nw);
    case 2: return pick_epl<uint16_t, PK, TR>(epl, nw);
    case 4: return pick_epl<uint32_t, PK, TR>(epl, nw);
  }
  return nullptr;
}

}  // namespace

KernelFn get_cluster_kernel(int wbytes, int epl, int nw, bool packed, bool trace) {
  if (trace) return packed ? pick_w<true, true>(wbytes, epl, nw) : pick_w<false, true>(wbytes, epl, nw);
  return packed ? pick_w<true, false>(wbytes, epl, nw) : pick_w<false, false>(wbytes, epl, nw);
}

ProbeFn get_cluster_probe(int nw, bool hier) {
  switch (nw) {
    case 4: return hier ? cluster_probe_kernel<4, true> : cluster_probe_kernel<4, false>;
    case 8: return hier ? cluster_probe_kernel<8, true> : cluster_probe_kernel<8, false>;
    case 16: return hier ? cluster_probe_kernel<16, true> : cluster_probe_kernel<16, false>;
  }
  return nullptr;
}

namespace {
template <typename W, int EPL>
KernelFn pick_hier_nw(int nw) {
  switch (nw) {
    case 4: return cluster_hier_kernel<W, EPL, 4>;
    case 8: return cluster_hier_kernel<W, EPL, 8>;
    case 16: return cluster_hier_kernel<W, EPL, 16>;
  }
  return nullptr;
}
template <typename W>
KernelFn pick_hier_epl(int epl, int nw) {
  switch (epl) {
    case 4: return pick_hier_nw<W, 4>(nw);
    case 8: return pick_hier_nw<W, 8>(nw);
    case 16: return pick_hier_nw<W, 16>(nw);
    case 32: return pick_hier_nw<W, 32>(nw);
  }
  return nullptr;
}
}  // namespace

KernelFn get_cluster_hier_kernel(int wbytes, int epl, int nw) {
  switch (wbytes) {
    case 1: return pick_hier_epl<uint8_t>(epl, nw);
    case 2: return pick_hier_epl<uint16_t>(epl, nw);
    case 4: return pick_hier_epl<uint32_t>(epl, nw);
  }
  return nullptr;
}

}  // namespace sssp_b200
