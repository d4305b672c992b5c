// Microbenchmark: tcgen05.mma throughput from SMEM for the operand layouts the
// NMFA kernels use (no-swizzle interleaved vs 128B swizzle), 1-CTA and 2-CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_1806_08422_b200/csrc/common.cuh"

using namespace nmfa;

__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                      // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32; // SBO = 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CG, int SW, int N>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  uint8_t* sA = smem;                 // 128 rows x 64 k x 2 B = 16 KB
  uint8_t* sB = smem + 16384;         // up to 128/256 rows x 64 k
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) {
    if (CG == 1) tmem_alloc(&slot, 256);
    else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t M = CG == 2 ? 256 : 128;
  const uint32_t idesc = make_idesc_f16(M, N);
  const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
  if (threadIdx.x == 0 && (CG == 1 || cluster_rank() == 0)) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 4; ++ks) {
        uint64_t ad, bd;
        if (SW) { ad = make_desc_sw128(a0 + ks * 32); bd = make_desc_sw128(b0 + ks * 32); }
        else { ad = make_desc_noswizzle(a0 + ks * 256, 128, 1024); bd = make_desc_noswizzle(b0 + ks * 256, 128, 1024); }
        if (CG == 1) mma_f16_ss(tbase, ad, bd, idesc, 1u);
        else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(1u) : "memory");
      }
    }
    if (CG == 1) mma_commit(&bar);
    else asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (CG == 2 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 1) tmem_dealloc(tbase, 256);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
  }
}

template <int CG, int SW, int N>
void run(const char* name, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * grid);
  const int iters = 2000;
  auto k = mma_bench<CG, SW, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 49152 + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double M = CG == 2 ? 256 : 128;
  const double mmas = iters * 4.0;
  const double cyc = (double)h[0];
  const double flop_per_cyc_per_sm = 2.0 * M * N * 16 * mmas / cyc / CG;
  const double tflops = 2.0 * M * N * 16 * mmas * (grid / CG) / (ms * 1e-3) / 1e12;
  printf("%-28s grid=%3d err=%d cycles/mma=%7.1f  FLOP/cyc/SM=%7.0f (peak 8192)  chip=%7.1f TFLOP/s\n",
         name, grid, (int)err, cyc / mmas, flop_per_cyc_per_sm, tflops);
  cudaFree(d);
}

int main() {
  run<1, 0, 256>("1cta M128 N256 noswz", 1);
  run<1, 1, 256>("1cta M128 N256 sw128", 1);
  run<1, 0, 128>("1cta M128 N128 noswz", 1);
  run<1, 1, 128>("1cta M128 N128 sw128", 1);
  run<2, 0, 224>("2cta M256 N224 noswz", 2);
  run<2, 1, 224>("2cta M256 N224 sw128", 2);
  run<2, 0, 256>("2cta M256 N256 noswz", 2);
  run<2, 1, 256>("2cta M256 N256 sw128", 2);
  run<2, 0, 256>("2cta M256 N256 noswz full", 148);
  run<2, 1, 256>("2cta M256 N256 sw128 full", 148);
  run<1, 1, 256>("1cta M128 N256 sw128 full", 148);
  return 0;
}
