// Microbenchmark: TMA (cp.async.bulk.tensor) L2 -> SMEM bandwidth with the
// line-tensor maps the dense kernel uses; unicast vs cluster multicast.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_bench tools/tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>

#include "../paper_1806_08422_b200/csrc/common.cuh"

using namespace nmfa;

constexpr int kStages = 6;
constexpr int kTile = 32768;  // 256 lines x 128 B per stage

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CS, int MODE>
__global__ void __launch_bounds__(64, 1) tma_bench(const __grid_constant__ CUtensorMap tm, int iters,
                                                   long long lines_total, int box_lines) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MODE == 1 ? 1 : CS); }
    fence_mbar_init();
  }
  if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  const long long cl = blockIdx.x / CS;
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], kTile);
      long long line = ((cl * 7919 + it) * 256) % (lines_total - 256);
      if (CS == 1 || MODE == 1) {   // MODE 1: unicast in a cluster (protocol cost only)
        for (int o = 0; o < kTile / 128; o += box_lines)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(smem + s * kTile + o * 128)), "l"(&tm), "r"(0), "r"((int)line + o), "r"(smem_u32(&full[s])) : "memory");
      } else if (MODE == 2) {       // MODE 2: rank 0 multicasts the whole stage
        if (rank == 0)
          for (int o = 0; o < kTile / 128; o += box_lines)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;"
                         ::"r"(smem_u32(smem + s * kTile + o * 128)), "l"(&tm), "r"(0), "r"((int)(line + o)),
                           "r"(smem_u32(&full[s])), "h"((uint16_t)((1 << CS) - 1)) : "memory");
      } else {
        // each CTA loads 1/CS of the stage (box_lines each) and multicasts it to every CTA
        const int part = (kTile / 128) / CS;
        for (int o = 0; o < part; o += box_lines)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;"
                       ::"r"(smem_u32(smem + s * kTile + (rank * part + o) * 128)), "l"(&tm), "r"(0),
                         "r"((int)(line + rank * part + o)), "r"(smem_u32(&full[s])),
                         "h"((uint16_t)((1 << CS) - 1)) : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      if (CS == 1 || MODE == 1) mbar_arrive(&empty[s]);
      else {
        for (int r = 0; r < CS; ++r) {
          uint32_t a;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(&empty[s])), "r"(r));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
        }
      }
    }
  }
  if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
}

template <int CS, int MODE = 0>
void run(const CUtensorMap& tm, long long lines, const char* name, int box_lines = 128, int grid = 148) {
  const int iters = 4000;
  auto k = tma_bench<CS, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kTile);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid / CS * CS);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = kStages * kTile;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, tm, iters, lines, box_lines);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, tm, iters, lines, box_lines);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const double delivered = (double)(grid / CS * CS) * iters * kTile;
  printf("%-32s grid=%3d err=%d  delivered to SMEM: %8.2f TB/s  (%6.1f B/clk/SM @1.9GHz)  L2 reads: %8.2f TB/s\n", name, grid, (int)err,
         delivered / (ms * 1e-3) / 1e12, delivered / (ms * 1e-3) / (grid / CS * CS) / 1.9e9, delivered / CS / (ms * 1e-3) / 1e12);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long bytes = 64LL << 20, lines = bytes / 128;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  CUtensorMap tm128, tm256;
  cuuint64_t dims[2] = {64, (cuuint64_t)lines};
  cuuint64_t strides[1] = {128};
  cuuint32_t b128[2] = {64, 128}, b256[2] = {64, 256}, estr[2] = {1, 1};
  encode(&tm128, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, dims, strides, b128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  encode(&tm256, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, dims, strides, b256, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<1, 0>(tm256, lines, "unicast box=256", 256, 148);
  run<2, 1>(tm256, lines, "cluster2 unicast box=256", 256, 148);
  run<2, 2>(tm256, lines, "cluster2 rank0-multicast 256", 256, 148);
  run<2, 0>(tm128, lines, "cluster2 split-multicast 128", 128, 148);
  return 0;
}
