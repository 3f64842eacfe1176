// kernels_cluster_ms.cu -- cluster-engine instances whose launch carries
// several shards of one device (MS = true; no round-time TRACE variant).
#include "kernels_cluster_impl.cuh"

namespace sssp_b200 {

KernelFn get_cluster_kernel_ms(int wbytes, int epl, int nw, bool packed) {
  using namespace cluster_tables;
  return packed ? pick_w<true, false, true>(wbytes, epl, nw) : pick_w<false, false, true>(wbytes, epl, nw);
}

ProbeFn get_cluster_probe_ms(int nw, bool hier) { return cluster_tables::probe<true>(nw, hier); }

KernelFn get_cluster_hier_kernel_ms(int wbytes, int epl, int nw) {
  return cluster_tables::hier<true>(wbytes, epl, nw);
}

}  // namespace sssp_b200
