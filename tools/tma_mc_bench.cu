// Microbenchmark: does TMA multicast shorten the per-SM operand feed of the
// dense kernel?  Each CTA of a 2-CTA cluster needs, per pipeline stage, its
// own 32 KB A box plus a 28 KB B tile that both CTAs of the cluster share
// (the J rows of one spin tile).  3 stages of 60 KB, as in the kernel.
//   U : A and B unicast by each CTA (60 KB through each SM's TMA unit)
//   M : A unicast, B split: each CTA loads 14 KB and multicasts it to both
//   A : A only (32 KB), B skipped (the feed bound without B)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_mc_bench tools/tma_mc_bench.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#include "../paper_1806_08422_b200/csrc/common.cuh"

using namespace nmfa;

constexpr int kStages = 3;
constexpr int kA = 32768, kB = 28672, kStage = kA + kB;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    bench(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmBh, int iters, long long a_lines, long long b_lines,
          unsigned long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == 1 ? 2 : 1);
    }
    fence_mbar_init();
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  const long long cl = blockIdx.x / 2;
  const unsigned bytes = MODE == 2 ? kA : kStage;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      // A: this CTA's 128 replica rows of the k-slice (each CTA its own lines)
      const long long al = ((cl * 2 + rank) * 7919 + it) * 256 % (a_lines - 256);
      // B: the spin tile both CTAs share
      const long long bl = ((cl * 131 + it) * 224) % (b_lines - 224);
      uint8_t* st = smem + s * kStage;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(st)),
          "l"(&tmA), "r"(0), "r"((int)al), "r"(smem_u32(&full[s]))
          : "memory");
      if (MODE == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(st + kA)),
            "l"(&tmB), "r"(0), "r"((int)bl), "r"(smem_u32(&full[s]))
            : "memory");
      } else if (MODE == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                smem_u32(st + kA + rank * (kB / 2))),
            "l"(&tmBh), "r"(0), "r"((int)(bl + rank * 112)), "r"(smem_u32(&full[s])), "h"((uint16_t)3)
            : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      if (MODE != 1) {
        mbar_arrive(&empty[s]);
      } else {
        for (uint32_t r = 0; r < 2; ++r) {
          uint32_t a;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(&empty[s])), "r"(r));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
        }
      }
    }
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;

static CUtensorMap lines_map(void* base, long long lines, int box) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)lines};
  cuuint64_t strides[1] = {128};
  cuuint32_t b[2] = {64, (cuuint32_t)box}, estr[2] = {1, 1};
  encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims, strides, b, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return tm;
}

template <int MODE>
void run(const char* name, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& bh, long long al,
         long long bl, unsigned long long* clk) {
  const int iters = 6000, grid = 148;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<MODE><<<grid, 64, kStages * kStage>>>(a, b, bh, iters, al, bl, clk);
  cudaEventRecord(e0);
  bench<MODE><<<grid, 64, kStages * kStage>>>(a, b, bh, iters, al, bl, clk);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
  const double per_stage = mean / iters;
  const double delivered = (MODE == 2 ? kA : kStage);
  printf("%-34s err=%d  %7.1f clk/stage  %6.1f B/clk/SM delivered  %.2f us total\n", name, (int)err, per_stage,
         delivered / per_stage, ms * 1e3);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long abytes = 32LL << 20, bbytes = 8LL << 20;  // state image slice, J image (L2-resident)
  void *abuf, *bbuf;
  cudaMalloc(&abuf, abytes);
  cudaMalloc(&bbuf, bbytes);
  cudaMemset(abuf, 1, abytes);
  cudaMemset(bbuf, 1, bbytes);
  unsigned long long* clk;
  cudaMalloc(&clk, 148 * 8);
  const long long al = abytes / 128, bl = bbytes / 128;
  CUtensorMap ta = lines_map(abuf, al, 256), tb = lines_map(bbuf, bl, 224), tbh = lines_map(bbuf, bl, 112);
  run<2>("A only (32 KB/stage)", ta, tb, tbh, al, bl, clk);
  run<0>("U: A + B unicast (60 KB/stage)", ta, tb, tbh, al, bl, clk);
  run<1>("M: A + B-half multicast (60 KB)", ta, tb, tbh, al, bl, clk);
  run<0>("U again", ta, tb, tbh, al, bl, clk);
  run<1>("M again", ta, tb, tbh, al, bl, clk);
  return 0;
}
