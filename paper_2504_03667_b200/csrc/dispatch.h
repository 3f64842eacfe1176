// dispatch.h -- kernel-instance lookup shared by the host code and the
// separately compiled kernel translation units.  `ms`: the launch carries
// several shards of one device (ScanLaunch.nlocal > 1).
#pragma once

#include "scan_kernel.cuh"

namespace sssp_b200 {

using KernelFn = void (*)(const ScanLaunch);
using ProbeFn = void (*)(const ScanLaunch, uint32_t, uint64_t*);

// grid engine (scan_kernel.cuh): one single-warp CTA per participant, L2 exchange
KernelFn get_grid_kernel(int wbytes, int epl, int np, bool ms = false);
ProbeFn get_grid_probe(int np, bool ms = false);

// cluster engine (cluster_kernel.cuh): one cluster per solve, DSMEM exchange
// (trace: the round-time instance; single-shard launches only)
KernelFn get_cluster_kernel(int wbytes, int epl, int nw, bool packed, bool trace = false,
                            bool ms = false);
ProbeFn get_cluster_probe(int nw, bool hier, bool ms = false);
// hierarchical cluster variant (CTA pre-reduction, PACKED state only)
KernelFn get_cluster_hier_kernel(int wbytes, int epl, int nw, bool ms = false);

// kernels_cluster_ms.cu
KernelFn get_cluster_kernel_ms(int wbytes, int epl, int nw, bool packed);
ProbeFn get_cluster_probe_ms(int nw, bool hier);
KernelFn get_cluster_hier_kernel_ms(int wbytes, int epl, int nw);

}  // namespace sssp_b200
