// ubench_barrier.cu -- grid-barrier and streaming-read microbenchmarks in the
// bucket kernel's launch shape (256 CTAs x 256 threads, 2 CTAs per SM), used
// to choose the bucket engine's barrier and pull-load design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_barrier tools/ubench_barrier.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t csize() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }

// mode 0: cooperative grid.sync
// mode 1: flat: every CTA red.release.gpu + ld.acquire.gpu poll
// mode 2: flat: __threadfence + atomicAdd + volatile poll
// mode 3: cluster hierarchical (release/acquire), one arrival per cluster
// mode 4: cluster hierarchical, fence.acq_rel + relaxed red + relaxed poll, fence after
// store: every thread writes one word to global before each barrier (publish-like traffic)
__global__ void barrier_kernel(int mode, int rounds, int store, unsigned long long* ctr,
                               uint32_t* scratch, uint64_t* out) {
  extern __shared__ uint32_t dyn[];
  namespace cg = cooperative_groups;
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x;
  const uint64_t ncl = G / csize();
  const uint32_t cr = crank();
  if (tid == 0) dyn[0] = 0;
  __syncthreads();
  const uint64_t t0 = gtimer();
  for (int r = 0; r < rounds; ++r) {
    if (store) scratch[(size_t)blockIdx.x * blockDim.x + tid] = r;
    if (mode == 0) {
      cg::this_grid().sync();
    } else if (mode == 1 || mode == 2) {
      __syncthreads();
      if (tid == 0) {
        const unsigned long long target = (unsigned long long)(r + 1) * G;
        unsigned long long v;
        if (mode == 1) {
          asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
          do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory"); } while (v < target);
        } else {
          __threadfence();
          atomicAdd(ctr, 1ull);
          do { v = *(volatile unsigned long long*)ctr; } while (v < target);
          __threadfence();
        }
      }
      __syncthreads();
    } else {
      csync();
      if (cr == 0 && tid == 0) {
        const unsigned long long target = (unsigned long long)(r + 1) * ncl;
        unsigned long long v;
        if (mode == 3) {
          asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
          do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory"); } while (v < target);
        } else {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
          do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory"); } while (v < target);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
      }
      csync();
    }
  }
  const uint64_t t1 = gtimer();
  if (blockIdx.x == 0 && tid == 0) out[0] = (t1 - t0) / rounds;
}

// Streaming read of `bytes` split evenly over the grid; each thread keeps DEPTH
// 16 B loads in flight.  cg: ld.global.cg (L2 only) instead of ld.global.nc.
__device__ unsigned long long g_t[2];
template <int DEPTH, bool CG>
__global__ void __launch_bounds__(256, 2) stream_kernel(const uint4* __restrict__ src, uint64_t n16, uint32_t* out) {
  extern __shared__ uint32_t dyn[];
  if (threadIdx.x == 0) atomicMin(&g_t[0], (unsigned long long)gtimer());
  const uint64_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * per, hi = min(n16, lo + per);
  uint32_t acc = 0;
  for (uint64_t i0 = lo + threadIdx.x; i0 < hi; i0 += 256 * DEPTH) {
    uint4 v[DEPTH];
#pragma unroll
    for (int m = 0; m < DEPTH; ++m) {
      const uint64_t i = i0 + m * 256;
      if (i < hi) v[m] = CG ? __ldcg(&src[i]) : __ldg(&src[i]);
      else v[m] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int m = 0; m < DEPTH; ++m) acc = min(acc ^ v[m].x, v[m].y ^ v[m].z ^ v[m].w);
  }
  if (acc == 0x12345678u) out[0] = acc + dyn[0];
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t[1], (unsigned long long)gtimer());
}

// Same with cp.async.bulk (TMA bulk copy) into a ring of NBUF smem slots of
// SLOT bytes, mbarrier-completed; one elected thread issues, all consume.
template <int NBUF, int SLOT>
__global__ void __launch_bounds__(256, 2) bulk_kernel(const uint8_t* __restrict__ src, uint64_t bytes, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t full[NBUF];
  const uint64_t per = ((bytes / 16 + gridDim.x - 1) / gridDim.x) * 16;
  const uint64_t lo = blockIdx.x * per, hi = min(bytes, lo + per);
  const uint32_t nslots = (uint32_t)((hi > lo ? hi - lo : 0) + SLOT - 1) / SLOT;
  if (threadIdx.x == 0)
    for (int b = 0; b < NBUF; ++b) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&full[b]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](uint32_t s) {
    const int b = s % NBUF;
    const uint64_t off = lo + (uint64_t)s * SLOT;
    const uint64_t rem = hi - off;
    const uint32_t len = (uint32_t)(rem < (uint64_t)SLOT ? rem : (uint64_t)SLOT);
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&full[b]);
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(sbuf + (size_t)b * SLOT);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src + off), "r"(len), "r"(mb) : "memory");
  };
  if (threadIdx.x == 0)
    for (uint32_t s = 0; s < nslots && s < NBUF; ++s) issue(s);
  uint32_t acc = 0;
  for (uint32_t s = 0; s < nslots; ++s) {
    const int b = s % NBUF;
    const uint32_t phase = (s / NBUF) & 1;
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&full[b]);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(phase) : "memory");
    const uint4* v = reinterpret_cast<const uint4*>(sbuf + (size_t)b * SLOT);
    for (int i = threadIdx.x; i < SLOT / 16; i += 256) acc = min(acc ^ v[i].x, v[i].y ^ v[i].z ^ v[i].w);
    __syncthreads();
    if (threadIdx.x == 0 && s + NBUF < nslots) issue(s + NBUF);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Matrix-slice streaming: a [rows x rowbytes] matrix read by 256 CTAs, CTA c
// taking column block c % nb (width rowbytes/nb) over row block c / nb;
// 16 B per thread, 8 rows in flight.  nb = 256 is the bucket/dataparallel
// tile layout (128 B of every row per CTA).
__global__ void __launch_bounds__(256, 2) slice_kernel(const uint8_t* __restrict__ m, uint32_t rows,
                                                       uint32_t rowbytes, uint32_t nb, uint32_t* out) {
  const uint32_t cb = blockIdx.x % nb, rb = blockIdx.x / nb, nrb = gridDim.x / nb;
  const uint32_t width = rowbytes / nb, tpr = width / 16, rg = 256 / tpr;
  const uint32_t r_lo = rb * (rows / nrb), r_hi = r_lo + rows / nrb;
  const uint32_t t = threadIdx.x % tpr, g = threadIdx.x / tpr;
  uint32_t acc = 0;
  for (uint32_t r0 = r_lo + g; r0 < r_hi; r0 += 8 * rg) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t r = r0 + k * rg;
      v[k] = r < r_hi ? __ldg(reinterpret_cast<const uint4*>(m + (size_t)r * rowbytes + cb * width) + t)
                      : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = min(acc ^ v[k].x, v[k].y ^ v[k].z ^ v[k].w);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// The bucket pull's access pattern: `nrows` rows of `rowbytes` each, at the
// given row indices of a large matrix, split as one contiguous item range per
// CTA (16 B items, 8 in flight per thread); in-kernel span like stream_kernel.
__global__ void __launch_bounds__(256, 2) rows_kernel(const uint8_t* __restrict__ m, const uint32_t* rows,
                                                      uint32_t nrows, uint32_t rowbytes, uint32_t* out) {
  if (threadIdx.x == 0) atomicMin(&g_t[0], (unsigned long long)gtimer());
  const uint32_t cpr = rowbytes / 16, total = nrows * cpr;
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = min(total, blockIdx.x * per), hi = min(total, lo + per);
  uint32_t acc = 0;
  for (uint32_t i0 = lo + threadIdx.x; i0 < hi; i0 += 256 * 8) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = i0 + k * 256;
      v[k] = i < hi ? __ldg(reinterpret_cast<const uint4*>(m + (size_t)rows[i / cpr] * rowbytes) + i % cpr)
                    : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = min(acc ^ v[k].x, v[k].y ^ v[k].z ^ v[k].w);
  }
  if (acc == 0x12345678u) out[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t[1], (unsigned long long)gtimer());
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int G = 256, rounds = 2000;
  unsigned long long* ctr;
  uint32_t* scratch;
  uint64_t* out;
  CK(cudaMalloc(&ctr, 8));
  CK(cudaMalloc(&scratch, (size_t)G * 256 * 4));
  CK(cudaMalloc(&out, 64));
  const size_t smems[] = {92 * 1024, 40 * 1024};
  CK(cudaFuncSetAttribute(barrier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  for (size_t smem : smems)
    for (int store = 0; store < (smem > 50000 ? 2 : 0); ++store)
      for (int mode = 0; mode < 5; ++mode) {
        const int cls[] = {1, 8, 4};
        for (int C : cls) {
          if (mode < 3 && C != 1) continue;
          if (mode >= 3 && C == 1) continue;
          CK(cudaMemset(ctr, 0, 8));
          int mode_ = mode, rounds_ = rounds, store_ = store;
          void* args[] = {&mode_, &rounds_, &store_, &ctr, &scratch, &out};
          cudaLaunchConfig_t cfg{};
          cudaLaunchAttribute at[2];
          cfg.gridDim = dim3(G);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = smem;
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = C;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          at[1].id = cudaLaunchAttributeCooperative;
          at[1].val.cooperative = mode == 0 ? 1 : 0;
          cfg.attrs = at;
          cfg.numAttrs = 2;
          cudaError_t e = cudaLaunchKernelExC(&cfg, (void*)barrier_kernel, args);
          if (e == cudaSuccess) e = cudaDeviceSynchronize();
          uint64_t ns = 0;
          if (e == cudaSuccess) CK(cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost));
          printf("{\"bench\": \"barrier\", \"mode\": %d, \"cluster\": %d, \"smem_kb\": %zu, \"store\": %d, \"ns_per_barrier\": %llu, \"err\": \"%s\"}\n",
                 mode, C, smem / 1024, store, (unsigned long long)ns, e == cudaSuccess ? "" : cudaGetErrorString(e));
          cudaGetLastError();
        }
      }
  // streaming: in-kernel span (min start .. max end, %globaltimer) of a read of
  // `bytes` over `grid` CTAs, L2 holding clean unrelated lines (no dirty flush)
  uint8_t* buf;
  CK(cudaMalloc(&buf, 1024ull << 20));  // >= the 1 GiB slice matrix
  CK(cudaMemset(buf, 1, 1024ull << 20));
  CK(cudaDeviceSynchronize());
  const uint64_t sizes[] = {1073ull * 32768, 128ull << 20, 512ull << 20};
  const int grids[] = {148, 256, 296};
  for (uint64_t bytes : sizes)
    for (int grid : grids) {
      for (int variant = 0; variant < 2; ++variant) {
        uint64_t best = ~0ull;
        for (int it = 0; it < 8; ++it) {
          // touch a different 512 MB region to evict the target from L2 (clean lines)
          stream_kernel<8, false><<<296, 256, 0>>>((const uint4*)(buf + (512ull << 20)), (512ull << 20) / 16, (uint32_t*)out);
          unsigned long long init[2] = {~0ull, 0ull};
          CK(cudaMemcpyToSymbol(g_t, init, 16));
          if (variant == 0) stream_kernel<8, false><<<grid, 256, 0>>>((const uint4*)buf, bytes / 16, (uint32_t*)out);
          else stream_kernel<16, false><<<grid, 256, 0>>>((const uint4*)buf, bytes / 16, (uint32_t*)out);
          CK(cudaDeviceSynchronize());
          unsigned long long t[2];
          CK(cudaMemcpyFromSymbol(t, g_t, 16));
          if (t[1] - t[0] < best) best = t[1] - t[0];
        }
        printf("{\"bench\": \"stream_span\", \"depth\": %d, \"grid\": %d, \"bytes\": %llu, \"us\": %.2f, \"GBps\": %.0f}\n",
               variant ? 16 : 8, grid, (unsigned long long)bytes, best * 1e-3, bytes / (best * 1e-9) / 1e9);
      }
    }
  {
    const uint32_t rows = 32768, rowbytes = 32768;
    const uint32_t nbs[] = {256, 64, 16, 8};
    for (uint32_t nb : nbs) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        stream_kernel<8, false><<<296, 256, 0>>>((const uint4*)(buf + (512ull << 20)), (256ull << 20) / 16, (uint32_t*)out);
        cudaEvent_t a, b2;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b2));
        CK(cudaEventRecord(a));
        slice_kernel<<<256, 256>>>(buf, rows, rowbytes, nb, (uint32_t*)out);
        CK(cudaEventRecord(b2));
        CK(cudaEventSynchronize(b2));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b2));
        if (ms < best) best = ms;
      }
      const double bytes = (double)rows * rowbytes;
      printf("{\"bench\": \"slice\", \"col_blocks\": %u, \"slice_bytes\": %u, \"us\": %.1f, \"GBps\": %.0f}\n",
             nb, rowbytes / nb, best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  }
  {
    // bare 35 MB stream, 256 CTAs, with the bucket kernel's 92 KB of dynamic
    // smem per CTA (L1 left for in-flight loads) vs none; in-kernel span
    CK(cudaFuncSetAttribute(stream_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    CK(cudaFuncSetAttribute(stream_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    const uint64_t bytes = 1073ull * 32768;
    for (int cgv = 0; cgv < 2; ++cgv)
      for (size_t smem : {(size_t)0, (size_t)92 * 1024}) {
        uint64_t best = ~0ull;
        for (int it = 0; it < 8; ++it) {
          stream_kernel<8, false><<<296, 256, 0>>>((const uint4*)(buf + (512ull << 20)), (256ull << 20) / 16, (uint32_t*)out);
          unsigned long long init[2] = {~0ull, 0ull};
          CK(cudaMemcpyToSymbol(g_t, init, 16));
          if (cgv) stream_kernel<8, true><<<256, 256, smem>>>((const uint4*)buf, bytes / 16, (uint32_t*)out);
          else stream_kernel<8, false><<<256, 256, smem>>>((const uint4*)buf, bytes / 16, (uint32_t*)out);
          CK(cudaDeviceSynchronize());
          unsigned long long t[2];
          CK(cudaMemcpyFromSymbol(t, g_t, 16));
          if (t[1] - t[0] < best) best = t[1] - t[0];
        }
        printf("{\"bench\": \"stream_smem\", \"load\": \"%s\", \"smem_kb\": %zu, \"us\": %.2f, \"GBps\": %.0f}\n",
               cgv ? "ld.cg" : "ld.nc", smem / 1024, best * 1e-3, bytes / (best * 1e-9) / 1e9);
      }
  }
  {
    // 1073 rows of 32 KB: contiguous block vs random rows of a 1 GiB matrix
    const uint32_t nrows = 1073, rowbytes = 32768;
    uint32_t h[1073];
    uint32_t* drows;
    CK(cudaMalloc(&drows, sizeof(h)));
    for (int variant = 0; variant < 2; ++variant) {
      uint64_t x = 88172645463325252ull;
      for (uint32_t i = 0; i < nrows; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = variant ? (uint32_t)(x % 32768) : i;
      }
      CK(cudaMemcpy(drows, h, sizeof(h), cudaMemcpyHostToDevice));
      uint64_t best = ~0ull;
      for (int it = 0; it < 8; ++it) {
        stream_kernel<8, false><<<296, 256, 0>>>((const uint4*)(buf + (512ull << 20)), (256ull << 20) / 16, (uint32_t*)out);
        unsigned long long init[2] = {~0ull, 0ull};
        CK(cudaMemcpyToSymbol(g_t, init, 16));
        rows_kernel<<<256, 256>>>(buf, drows, nrows, rowbytes, (uint32_t*)out);
        CK(cudaDeviceSynchronize());
        unsigned long long t[2];
        CK(cudaMemcpyFromSymbol(t, g_t, 16));
        if (t[1] - t[0] < best) best = t[1] - t[0];
      }
      printf("{\"bench\": \"rows\", \"rows\": \"%s\", \"bytes\": %u, \"us\": %.2f, \"GBps\": %.0f}\n",
             variant ? "random of 32768 (1 GiB)" : "contiguous", nrows * rowbytes, best * 1e-3,
             (double)nrows * rowbytes / (best * 1e-9) / 1e9);
    }
  }
  printf("{\"bench\": \"info\", \"sms\": %d}\n", sms);
  return 0;
}
