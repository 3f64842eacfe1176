// ubench_launch.cu -- per-launch cost of back-to-back launches in the bucket
// kernel's shape (256 CTAs x 256 threads, dynamic smem), cooperative vs plain
// vs plain + one in-kernel grid barrier, and the in-kernel span of one barrier
// launch.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_launch tools/ubench_launch.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Big { uint64_t w[48]; };  // ~ BucketParams size

__global__ void __launch_bounds__(256, 2) empty_kernel(const Big p) {
  extern __shared__ uint32_t dyn[];
  if (threadIdx.x == 0 && p.w[0] == 12345) dyn[0] = 1;
}
__global__ void __launch_bounds__(256, 2) coop_kernel(const Big p, int nbar) {
  extern __shared__ uint32_t dyn[];
  for (int i = 0; i < nbar; ++i) cooperative_groups::this_grid().sync();
  if (threadIdx.x == 0 && p.w[0] == 12345) dyn[0] = 1;
}

// spins ~`ns` nanoseconds (every CTA), then exits: per-launch time minus ns =
// the GPU-side launch + drain overhead of this grid shape
__global__ void __launch_bounds__(256, 2) spin_kernel(const Big p, unsigned long long ns) {
  extern __shared__ uint32_t dyn[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
  if (threadIdx.x == 0 && p.w[0] == 12345) dyn[0] = 1;
}

int main() {
  Big b{};
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t smems[] = {0, 48 * 1024, 92 * 1024};
  CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  const int K = 200;
  for (size_t smem : smems)
    for (int variant = 0; variant < 4; ++variant) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaStreamSynchronize(st));
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < K; ++i) {
          int nb = variant == 3 ? 4 : 0;
          void* args[] = {&b, &nb};
          if (variant == 0) {
            empty_kernel<<<256, 256, smem, st>>>(b);
          } else if (variant == 1) {
            void* a1[] = {&b};
            CK(cudaLaunchCooperativeKernel((void*)empty_kernel, dim3(256), dim3(256), a1, smem, st));
          } else {
            CK(cudaLaunchCooperativeKernel((void*)coop_kernel, dim3(256), dim3(256), args, smem, st));
          }
        }
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      const char* names[] = {"plain empty", "coop empty", "coop 0 barriers", "coop 4 grid.sync"};
      printf("{\"bench\": \"launch\", \"variant\": \"%s\", \"smem_kb\": %zu, \"us_per_launch\": %.2f}\n",
             names[variant], smem / 1024, best * 1e3 / K);
    }
  CK(cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  for (size_t smem : smems)
    for (int coop = 0; coop < 2; ++coop) {
      unsigned long long ns = 30000;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaStreamSynchronize(st));
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < 100; ++i) {
          void* a2[] = {&b, &ns};
          if (coop) CK(cudaLaunchCooperativeKernel((void*)spin_kernel, dim3(256), dim3(256), a2, smem, st));
          else spin_kernel<<<256, 256, smem, st>>>(b, ns);
        }
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      printf("{\"bench\": \"launch_overhead\", \"coop\": %d, \"smem_kb\": %zu, \"spin_us\": 30, \"us_per_launch\": %.2f, \"overhead_us\": %.2f}\n",
             coop, smem / 1024, best * 10.0, best * 10.0 - 30.0);
    }
  return 0;
}
