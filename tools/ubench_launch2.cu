// ubench_launch2.cu -- per-launch cost of back-to-back cooperative launches in
// the bucket kernel's shape (256 CTAs x 256 threads, 92 KB smem) as a function
// of the kernel-parameter size and of an event record between launches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_launch2 tools/ubench_launch2.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int W> struct Big { uint64_t w[W]; };

template <int W>
__global__ void __launch_bounds__(256, 2) k_empty(const Big<W> p) {
  extern __shared__ uint32_t dyn[];
  if (threadIdx.x == 0 && p.w[W - 1] == 12345) dyn[0] = 1;
}
// the same empty launch, but the kernel holds 128 registers and ~40 KB of code
// (a never-taken branch): does register / code footprint change launch cost?
#define FAT_BODY \
  extern __shared__ uint32_t dyn[]; \
  if (p.w[0] == 777) { \
    uint32_t r[100]; \
    _Pragma("unroll") for (int i = 0; i < 100; ++i) r[i] = (uint32_t)p.w[i % 192] * (i + 3); \
    _Pragma("unroll 1") for (int it = 0; it < (int)p.w[1]; ++it) { \
      _Pragma("unroll") for (int i = 0; i < 100; ++i) r[i] = __byte_perm(r[i], r[(i + 7) % 100], 0x5140) + r[(i * 13) % 100]; \
    } \
    uint32_t acc = 0; \
    _Pragma("unroll") for (int i = 0; i < 100; ++i) acc ^= r[i]; \
    dyn[threadIdx.x] = acc; \
  } \
  if (threadIdx.x == 0 && p.w[191] == 12345) dyn[0] = 1;
template <int MAXR>
__global__ void __launch_bounds__(256, 1) __maxnreg__(MAXR) k_fatr(const Big<192> p) { FAT_BODY }
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_fat(const Big<192> p) {
  extern __shared__ uint32_t dyn[];
  if (p.w[0] == 777) {
    uint32_t r[100];
#pragma unroll
    for (int i = 0; i < 100; ++i) r[i] = (uint32_t)p.w[i % 192] * (i + 3);
#pragma unroll 1
    for (int it = 0; it < (int)p.w[1]; ++it) {
#pragma unroll
      for (int i = 0; i < 100; ++i) r[i] = __byte_perm(r[i], r[(i + 7) % 100], 0x5140) + r[(i * 13) % 100];
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 100; ++i) acc ^= r[i];
    dyn[threadIdx.x] = acc;
  }
  if (threadIdx.x == 0 && p.w[191] == 12345) dyn[0] = 1;
}
// the same, with programmatic dependent launch: the grid lets its dependent
// launch start at once and waits for its predecessor before any memory work
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_fat_pdl(const Big<192> p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ uint32_t dyn[];
  if (p.w[0] == 777) {
    uint32_t r[100];
#pragma unroll
    for (int i = 0; i < 100; ++i) r[i] = (uint32_t)p.w[i % 192] * (i + 3);
#pragma unroll 1
    for (int it = 0; it < (int)p.w[1]; ++it) {
#pragma unroll
      for (int i = 0; i < 100; ++i) r[i] = __byte_perm(r[i], r[(i + 7) % 100], 0x5140) + r[(i * 13) % 100];
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 100; ++i) acc ^= r[i];
    dyn[threadIdx.x] = acc;
  }
  if (threadIdx.x == 0 && p.w[191] == 12345) dyn[0] = 1;
}
__global__ void __launch_bounds__(256, 2) k_ptr(const uint64_t* p) {
  extern __shared__ uint32_t dyn[];
  if (threadIdx.x == 0 && p[0] == 12345) dyn[0] = 1;
}

template <int W>
int run(cudaStream_t st, int ev_between, const char* name) {
  Big<W> b{};
  cudaEvent_t e0, e1, em;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&em));
  const size_t smem = 92 * 1024;
  CK(cudaFuncSetAttribute(k_empty<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  const int K = 200;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < K; ++i) {
      void* a1[] = {&b};
      CK(cudaLaunchCooperativeKernel((void*)k_empty<W>, dim3(256), dim3(256), a1, smem, st));
      if (ev_between) CK(cudaEventRecord(em, st));
    }
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  printf("{\"bench\": \"launch2\", \"variant\": \"%s\", \"param_bytes\": %d, \"event_between\": %d, \"us_per_launch\": %.2f}\n",
         name, (int)sizeof(Big<W>), ev_between, best * 1e3 / K);
  return 0;
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto fat = [&](void* fn, const char* name, int grid = 256, int threads = 256, int pdl = 0, int coop = 1) -> int {
    Big<192> b{};
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, fn));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      for (int i = 0; i < 200; ++i) {
        void* a1[] = {&b};
        if (!pdl && !coop) {
          fn == nullptr ? (void)0 : (void)0;
          CK(cudaLaunchKernel(fn, dim3(grid), dim3(threads), a1, 92 * 1024, st));
        } else if (!pdl) {
          CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), a1, 92 * 1024, st));
        } else {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(threads);
          cfg.dynamicSmemBytes = 92 * 1024;
          cfg.stream = st;
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          at[1].id = cudaLaunchAttributeCooperative;
          at[1].val.cooperative = 1;
          cfg.attrs = at;
          cfg.numAttrs = coop ? 2 : 1;
          CK(cudaLaunchKernelExC(&cfg, fn, a1));
        }
      }
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf("{\"bench\": \"launch2\", \"variant\": \"%s\", \"regs\": %d, \"code_bytes\": %d, \"param_bytes\": 1536, \"grid\": %d, \"threads\": %d, \"us_per_launch\": %.2f}\n",
           name, fa.numRegs, 0, grid, threads, best * 1e3 / 200);
    return 0;
  };
  fat((void*)k_fat<2>, "coop fat code, 2 CTAs/SM regs");
  fat((void*)k_fat_pdl<2>, "coop fat code, 2 CTAs/SM regs, PDL", 256, 256, 1);
  fat((void*)k_fat_pdl<2>, "non-coop fat code, 2 CTAs/SM regs, PDL", 256, 256, 1, 0);
  fat((void*)k_fat<2>, "non-coop fat code, 2 CTAs/SM regs", 256, 256, 0, 0);
  fat((void*)k_fatr<120>, "coop fat code, maxnreg 120 (again)");
  fat((void*)k_fat<2>, "coop fat code, 1 CTA/SM", 148);
  fat((void*)k_fatr<120>, "coop fat code, maxnreg 120");
  fat((void*)k_fatr<112>, "coop fat code, maxnreg 112");
  fat((void*)k_fatr<96>, "coop fat code, maxnreg 96");
  fat((void*)k_fat<2>, "coop fat code, 128 CTAs", 128);
  fat((void*)k_fat<2>, "coop fat code, 128 threads", 256, 128);
  fat((void*)k_fat<4>, "coop fat code, <=64 regs");
  fat((void*)k_fat<8>, "coop fat code, <=32 regs");
  for (int ev = 0; ev < 2; ++ev) {
    run<8>(st, ev, "coop empty");
    run<48>(st, ev, "coop empty");
    run<192>(st, ev, "coop empty");
    run<512>(st, ev, "coop empty");
  }
  return 0;
}
