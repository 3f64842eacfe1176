// kernels_cluster.cu -- single-shard-per-launch instances of the cluster
// engine (cluster_kernel.cuh) and the dispatch entry points.
#include "kernels_cluster_impl.cuh"

namespace sssp_b200 {

KernelFn get_cluster_kernel(int wbytes, int epl, int nw, bool packed, bool trace, bool ms) {
  using namespace cluster_tables;
  if (ms) return get_cluster_kernel_ms(wbytes, epl, nw, packed);
  if (trace) return packed ? pick_w<true, true, false>(wbytes, epl, nw) : pick_w<false, true, false>(wbytes, epl, nw);
  return packed ? pick_w<true, false, false>(wbytes, epl, nw) : pick_w<false, false, false>(wbytes, epl, nw);
}

ProbeFn get_cluster_probe(int nw, bool hier, bool ms) {
  return ms ? get_cluster_probe_ms(nw, hier) : cluster_tables::probe<false>(nw, hier);
}

KernelFn get_cluster_hier_kernel(int wbytes, int epl, int nw, bool ms) {
  return ms ? get_cluster_hier_kernel_ms(wbytes, epl, nw) : cluster_tables::hier<false>(wbytes, epl, nw);
}

}  // namespace sssp_b200
