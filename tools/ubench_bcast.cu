// ubench_bcast.cu -- cost of a broadcast read: every CTA of the bucket
// kernel's launch shape (256 CTAs x 256 threads, 2 per SM) loads the same X
// bytes from L2 (the class data after an exchange, the source row of class 1).
//  same      : every CTA reads the one copy
//  repl-R    : R copies at different addresses, CTA c reads copy c % R
//  distinct  : every CTA reads its own X bytes (no sharing; the reference rate)
//  dsmem-C   : clusters of C CTAs: each CTA loads X/C bytes and stores them into
//              every cluster peer's shared memory, then one cluster barrier
//  mcast-C   : clusters of C CTAs: rank 0 issues cp.async.bulk ...multicast::cluster
//              copies of X bytes into every peer; each CTA waits on its mbarrier
// Reported: the in-kernel span of the load phase (max CTA end - min CTA start,
// %globaltimer) and event time per launch; data warm in L2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bcast tools/ubench_bcast.cu
#include <cuda_runtime.h>

#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr uint32_t NT = 256, G = 256;

// mode 0: plain loads (same / repl / distinct via `stride_cta`), 1: dsmem, 2: mcast
__global__ void __launch_bounds__(NT, 2) bcast_kernel(int mode, const uint4* __restrict__ src, uint32_t X,
                                                      uint32_t R, uint32_t* out, uint64_t* span) {
  extern __shared__ __align__(128) uint4 sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x, bx = blockIdx.x;
  const uint32_t nv = X / 16;
  if (mode == 2 && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (mode != 0) cg::this_cluster().sync();
  else __syncthreads();
  const uint64_t t0 = gtimer();
  uint32_t acc = 0;
  if (mode == 0) {
    const uint4* s = src + (size_t)(bx % R) * nv;
    for (uint32_t i0 = 0; i0 < nv; i0 += NT * 8) {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + tid + k * NT < nv) v[k] = __ldcg(s + i0 + tid + k * NT);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + tid + k * NT < nv) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
  } else if (mode == 1) {
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t C = cl.num_blocks(), rk = cl.block_rank();
    const uint32_t per = nv / C;
    for (uint32_t i = tid; i < per; i += NT) {
      const uint4 v = __ldcg(src + rk * per + i);
      for (uint32_t c = 0; c < C; ++c) {
        uint4* dst = cl.map_shared_rank(sm, c);
        dst[rk * per + i] = v;
      }
    }
    cl.sync();
    for (uint32_t i = tid; i < nv; i += NT) acc ^= sm[i].x ^ sm[i].w;
  } else {
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t C = cl.num_blocks(), rk = cl.block_rank();
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(X) : "memory");
    cl.sync();  // every peer armed before the multicast lands
    if (rk == 0 && tid == 0) {
      const uint16_t mask = (uint16_t)((1u << C) - 1u);
      for (uint32_t o = 0; o < X; o += 16384) {
        const uint32_t b = X - o < 16384 ? X - o : 16384;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
            ::"r"(su32(reinterpret_cast<char*>(sm) + o)), "l"(reinterpret_cast<const char*>(src) + o), "r"(b),
            "r"(su32(&bar)), "h"(mask) : "memory");
      }
    }
    asm volatile("{\n .reg .pred P1;\n W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n"
                 ::"r"(su32(&bar)) : "memory");
    for (uint32_t i = tid; i < nv; i += NT) acc ^= sm[i].x ^ sm[i].w;
  }
  __syncthreads();
  const uint64_t t1 = gtimer();
  if (tid == 0) {
    span[2 * bx] = t0;
    span[2 * bx + 1] = t1;
  }
  if (acc == 0x12345678u) out[bx] = acc;
}

int main() {
  const uint32_t maxX = 32768, maxR = 256;
  uint4* d_src;
  CK(cudaMalloc(&d_src, (size_t)maxX * maxR));
  CK(cudaMemset(d_src, 1, (size_t)maxX * maxR));
  uint32_t* d_out;
  uint64_t* d_span;
  CK(cudaMalloc(&d_out, G * 4));
  CK(cudaMalloc(&d_span, G * 16));
  CK(cudaFuncSetAttribute(bcast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
  CK(cudaFuncSetAttribute(bcast_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<uint64_t> sp(2 * G);
  auto run = [&](const char* name, int mode, uint32_t X, uint32_t R, uint32_t C) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = mode == 0 ? 0 : X;
    cfg.stream = 0;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = mode == 0 ? 0 : 1;
    double span_sum = 0;
    const int reps = 50;
    for (int it = 0; it < 5; ++it) CK(cudaLaunchKernelEx(&cfg, bcast_kernel, mode, (const uint4*)d_src, X, R, d_out, d_span));
    CK(cudaEventRecord(e0));
    for (int it = 0; it < reps; ++it) CK(cudaLaunchKernelEx(&cfg, bcast_kernel, mode, (const uint4*)d_src, X, R, d_out, d_span));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    for (int it = 0; it < 10; ++it) {
      CK(cudaLaunchKernelEx(&cfg, bcast_kernel, mode, (const uint4*)d_src, X, R, d_out, d_span));
      CK(cudaMemcpy(sp.data(), d_span, sp.size() * 8, cudaMemcpyDeviceToHost));
      uint64_t a = ~0ull, b = 0;
      for (uint32_t c = 0; c < G; ++c) {
        a = std::min(a, sp[2 * c]);
        b = std::max(b, sp[2 * c + 1]);
      }
      span_sum += (b - a) * 1e-3;
    }
    printf("{\"bench\": \"bcast\", \"variant\": \"%s\", \"bytes\": %u, \"R\": %u, \"C\": %u, \"span_us\": %.2f, \"event_us\": %.2f}\n",
           name, X, R, C, span_sum / 10, ms * 1e3 / reps);
  };
  for (uint32_t X : {1024u, 4096u, 8192u, 32768u}) {
    run("same", 0, X, 1, 1);
    run("repl", 0, X, 8, 1);
    run("repl", 0, X, 32, 1);
    run("distinct", 0, X, 256, 1);
    run("dsmem", 1, X, 1, 8);
    run("mcast", 2, X, 1, 8);
    run("mcast", 2, X, 1, 16);
  }
  return 0;
}
