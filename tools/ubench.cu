// ubench.cu -- latency microbenchmarks behind the kernel design choices
// (DESIGN.md §4).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
// Each test prints cycles (clock64) per operation / per round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// 1. dependent chains: CREDUX (__reduce_min_sync), SHFL butterfly min, LDS
__global__ void chain_kernel(uint64_t* out, uint32_t seed) {
  uint32_t x = threadIdx.x ^ seed;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = __reduce_min_sync(0xFFFFFFFFu, x + threadIdx.x) ^ i;
  long long t1 = clock64();
  for (int i = 0; i < 1024; ++i) {
    uint32_t y = x + threadIdx.x;
#pragma unroll
    for (int o = 16; o; o >>= 1) y = min(y, __shfl_xor_sync(0xFFFFFFFFu, y, o));
    x = y ^ i;
  }
  long long t2 = clock64();
  __shared__ uint32_t sm[64];
  sm[threadIdx.x] = x;
  __syncwarp();
  uint32_t a = threadIdx.x;
  for (int i = 0; i < 1024; ++i) a = sm[(a + i) & 31];
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 1024;
    out[1] = (t2 - t1) / 1024;
    out[2] = (t3 - t2) / 1024;
    out[3] = x + a;
  }
}

// 2. DSMEM ping-pong: CTA 0 lane 0 stores a tagged word into CTA k's smem,
//    CTA k polls its own smem and answers into CTA 0's smem.  Round trip / 2.
__global__ void dsmem_pingpong(uint64_t* out, int rounds) {
  __shared__ volatile uint64_t box;
  box = 0;
  csync();
  const uint32_t r = ctarank();
  uint32_t la = (uint32_t)__cvta_generic_to_shared((const void*)&box);
  uint32_t peer = r == 0 ? 1 : 0;
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(peer));
  long long t0 = clock64();
  if (threadIdx.x == 0 && r < 2) {
    for (int i = 1; i <= rounds; ++i) {
      if (r == 0) {
        asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"((uint64_t)i) : "memory");
        uint64_t v;
        do { asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(la) : "memory"); } while (v != (uint64_t)i);
      } else {
        uint64_t v;
        do { asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(la) : "memory"); } while (v != (uint64_t)i);
        asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"((uint64_t)i) : "memory");
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[0] = (t1 - t0) / rounds;
  csync();
}

// 3. same ping-pong through global memory (L2): relaxed.gpu store / load
__global__ void l2_pingpong(uint64_t* out, uint64_t* flags, int rounds) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0 || b > 1) return;
  uint64_t* mine = flags + 32 * b;          // separate 256 B lines
  uint64_t* theirs = flags + 32 * (1 - b);
  long long t0 = clock64();
  for (int i = 1; i <= rounds; ++i) {
    if (b == 0) {
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(theirs), "l"((uint64_t)i) : "memory");
      uint64_t v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v != (uint64_t)i);
    } else {
      uint64_t v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v != (uint64_t)i);
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(theirs), "l"((uint64_t)i) : "memory");
    }
  }
  long long t1 = clock64();
  if (b == 0) out[0] = (t1 - t0) / rounds;
}

// 4. DSMEM all-gather round with C CTAs x NW warps (what the solve does per
//    round, minus compute): measures cycles per round.
template <int NW>
__global__ void allgather_round(uint64_t* out, int rounds) {
  __shared__ __align__(16) uint64_t keys[2][16 * NW];
  uint32_t cs;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const uint32_t r = ctarank(), warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Q = cs * NW, q = r * NW + warp;
  for (uint32_t i = threadIdx.x; i < 2 * 16 * NW; i += blockDim.x) (&keys[0][0])[i] = 0;
  csync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(&keys[0][0]);
  long long t0 = clock64();
  for (int it = 1; it <= rounds; ++it) {
    const uint32_t buf = it & 1;
    const uint64_t key = ((uint64_t)(it * 7 + q) << 32) | (uint32_t)it;
    if (lane < cs) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + (buf * 16 * NW + q) * 8), "r"(lane));
      asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(key) : "memory");
    }
    while (true) {
      bool ok = true;
      for (uint32_t i = 2 * lane; i < Q; i += 64) {
        uint64_t lo, hi;
        asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(base + (buf * 16 * NW + i) * 8) : "memory");
        ok &= ((uint32_t)lo == (uint32_t)it) & ((uint32_t)hi == (uint32_t)it);
      }
      if (__all_sync(0xFFFFFFFFu, ok)) break;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[0] = (t1 - t0) / rounds;
  csync();
}

template <int NW>
int run_allgather(int C, uint64_t* d_out, uint64_t* h) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(NW * 32);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  CK(cudaFuncSetAttribute(allgather_round<NW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int rounds = 20000;
  CK(cudaLaunchKernelEx(&cfg, allgather_round<NW>, d_out, rounds));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
  printf("{\"test\": \"dsmem_allgather\", \"C\": %d, \"NW\": %d, \"Q\": %d, \"cycles_per_round\": %llu}\n", C, NW, C * NW, (unsigned long long)h[0]);
  return 0;
}

int main() {
  uint64_t *d_out, *d_flags, h[8];
  CK(cudaMalloc(&d_out, 64));
  CK(cudaMalloc(&d_flags, 4096));
  CK(cudaMemset(d_flags, 0, 4096));
  chain_kernel<<<1, 32>>>(d_out, 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_out, 32, cudaMemcpyDeviceToHost));
  printf("{\"test\": \"chains\", \"credux_cycles\": %llu, \"shfl_min_5level_cycles\": %llu, \"lds_cycles\": %llu}\n",
         (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)h[2]);
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(32);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaFuncSetAttribute(dsmem_pingpong, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaLaunchKernelEx(&cfg, dsmem_pingpong, d_out, 20000));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
    printf("{\"test\": \"dsmem_pingpong_roundtrip\", \"C\": %d, \"cycles\": %llu}\n", C, (unsigned long long)h[0]);
  }
  l2_pingpong<<<148, 32>>>(d_out, d_flags, 20000);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
  printf("{\"test\": \"l2_pingpong_roundtrip\", \"cycles\": %llu}\n", (unsigned long long)h[0]);
  for (int C : {2, 4, 8, 16}) {
    if (run_allgather<4>(C, d_out, h)) return 1;
    if (run_allgather<8>(C, d_out, h)) return 1;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"test\": \"clock\", \"khz\": %d}\n", clk);
  return 0;
}
