// Microbenchmark 2: TMA multicast delivery rate on B200, B-operand only.
// Each CTA needs a tile of `tile` bytes per stage that all `CS` CTAs of its
// cluster share.  Unicast: every CTA loads the whole tile.  Multicast: each
// CTA loads tile/CS and multicasts it to the whole cluster (ctaMask = all).
// 4 stages.  Prints clocks per stage per CTA and bytes delivered per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_mc_bench2 tools/tma_mc_bench2.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#include "../paper_1806_08422_b200/csrc/common.cuh"

using namespace nmfa;

#ifndef STAGES
#define STAGES 4
#endif
constexpr int kStages = STAGES;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CS, bool MC>
__global__ void __launch_bounds__(64, 1)
    bench(const __grid_constant__ CUtensorMap tm, int iters, long long lines_total, int tile_lines,
          unsigned long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int tile = tile_lines * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? CS : 1);
    }
    fence_mbar_init();
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  const long long cl = blockIdx.x / CS;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], tile);
      const long long line = ((cl * 131 + it) * tile_lines) % (lines_total - tile_lines);
      uint8_t* st = smem + s * tile;
      if (!MC) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(st)),
            "l"(&tm), "r"(0), "r"((int)line), "r"(smem_u32(&full[s]))
            : "memory");
      } else {
        const int part = tile_lines / CS;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                smem_u32(st + rank * part * 128)),
            "l"(&tm), "r"(0), "r"((int)(line + rank * part)), "r"(smem_u32(&full[s])),
            "h"((uint16_t)((1 << CS) - 1))
            : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      if (!MC) {
        mbar_arrive(&empty[s]);
      } else {
        for (uint32_t r = 0; r < CS; ++r) {
          uint32_t a;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(&empty[s])), "r"(r));
#ifdef RELAXED_ARRIVE  // the consumer frees the slot with relaxed remote arrives (no cluster release)
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
#else
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
#endif
        }
      }
    }
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;

template <int CS, bool MC>
void run(void* buf, long long lines, int tile_lines, unsigned long long* clk) {
  CUtensorMap tm;
  const int box = MC ? tile_lines / CS : tile_lines;
  cuuint64_t dims[2] = {64, (cuuint64_t)lines};
  cuuint64_t strides[1] = {128};
  cuuint32_t b[2] = {64, (cuuint32_t)box}, estr[2] = {1, 1};
  encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, dims, strides, b, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int iters = 4000, grid = 144;  // a multiple of 2 and 4 within 148 SMs
  const size_t smem = (size_t)kStages * tile_lines * 128;
  cudaFuncSetAttribute(bench<CS, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bench<CS, MC>, tm, iters, lines, tile_lines, clk);
  cudaError_t err = cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, bench<CS, MC>, tm, iters, lines, tile_lines, clk);
  err = cudaDeviceSynchronize();
  unsigned long long h[144];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
  const double per = mean / iters;
  printf("%s stages %d cluster %d %-9s tile %3d KB (box %2d KB)  err=%d  %7.1f clk/stage  %6.1f B/clk/SM delivered, %6.1f B/clk/SM issued\n",
#ifdef RELAXED_ARRIVE
         "relaxed",
#else
         "release",
#endif
         kStages, CS, MC ? "multicast" : "unicast", tile_lines / 8, box / 8, (int)err, per, tile_lines * 128 / per,
         box * 128 / per);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long bytes = 16LL << 20, lines = bytes / 128;  // J-sized, L2-resident
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* clk;
  cudaMalloc(&clk, 148 * 8);
  for (int tl : {128, 224}) {
    run<1, false>(buf, lines, tl, clk);
    run<2, false>(buf, lines, tl, clk);
    run<2, true>(buf, lines, tl, clk);
    run<4, false>(buf, lines, tl, clk);
    run<4, true>(buf, lines, tl, clk);
  }
  return 0;
}
