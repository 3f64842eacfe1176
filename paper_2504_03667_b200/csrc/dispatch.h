// dispatch.h -- kernel-instance lookup shared by the host code and the
// separately compiled kernel translation units.
#pragma once

#include "scan_kernel.cuh"

namespace sssp_b200 {

using KernelFn = void (*)(const ScanParams);
using ProbeFn = void (*)(const ScanParams, uint32_t, uint64_t*);

// grid engine (scan_kernel.cuh): one single-warp CTA per participant, L2 exchange
KernelFn get_grid_kernel(int wbytes, int epl, int np);
ProbeFn get_grid_probe(int np);

// cluster engine (cluster_kernel.cuh): one cluster per solve, DSMEM exchange
KernelFn get_cluster_kernel(int wbytes, int epl, int nw, bool packed, bool trace = false);
ProbeFn get_cluster_probe(int nw, bool hier);
// hierarchical cluster variant (CTA pre-reduction, PACKED state only)
KernelFn get_cluster_hier_kernel(int wbytes, int epl, int nw);

}  // namespace sssp_b200
