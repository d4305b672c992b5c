// Is the per-SM limit the TMA engine or the SM<->L2 port?  TMA unicast stream
// (one 32 KB box per stage) + W extra warps streaming LDG.128 from L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/port_bench tools/port_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1806_08422_b200/csrc/common.cuh"
using namespace nmfa;
constexpr int kStages = 6, kTile = 32768;

__global__ void __launch_bounds__(512, 1) port_bench(const __grid_constant__ CUtensorMap tm, int iters, long long lines_total,
                                                      const uint4* __restrict__ ld_buf, long long ld_elems, int ld_warps,
                                                      unsigned long long* out, int use_tma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ unsigned long long t_tma;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  if (warp == 0 && lane == 0 && use_tma) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], kTile);
      long long line = (((long long)blockIdx.x * 7919 + it) * 256) % (lines_total - 256);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(smem + s * kTile)), "l"(&tm), "r"(0), "r"((int)line), "r"(smem_u32(&full[s])) : "memory");
    }
    t_tma = clock64() - t0;
  } else if (warp == 1 && lane == 0 && use_tma) {
    for (int it = 0; it < iters; ++it) { const int s = it % kStages; mbar_wait(&full[s], (it / kStages) & 1); mbar_arrive(&empty[s]); }
  } else if (warp >= 2 && warp < 2 + ld_warps) {
    // streaming L2 reads: each warp reads 512 B per iteration, 4 in flight
    uint4 acc = make_uint4(0, 0, 0, 0);
    long long base = ((long long)(blockIdx.x * 16 + warp) * 4096) % (ld_elems - 32 * 4 * 2048);
    unsigned long long t0 = clock64();
    const int n_it = 2048;
    for (int it = 0; it < n_it; ++it) {
      const uint4* p = ld_buf + base + ((long long)it * 128) % (32 * 4 * 2000) + lane;
      uint4 v0 = __ldcg(p), v1 = __ldcg(p + 32), v2 = __ldcg(p + 64), v3 = __ldcg(p + 96);
      acc.x ^= v0.x ^ v1.y ^ v2.z ^ v3.w;
    }
    unsigned long long dt = clock64() - t0;
    if (acc.x == 0xdeadbeef) out[1000] = 1;
    if (lane == 0) atomicAdd(&out[blockIdx.x * 4 + 1], dt), atomicAdd(&out[blockIdx.x * 4 + 2], (unsigned long long)n_it * 512 * 4);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x * 4 + 0] = use_tma ? t_tma : 0;
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long bytes = 48LL << 20, lines = bytes / 128;
  void *buf, *buf2; cudaMalloc(&buf, bytes); cudaMalloc(&buf2, bytes); cudaMemset(buf, 1, bytes); cudaMemset(buf2, 2, bytes);
  CUtensorMap tm; cuuint64_t dims[2] = {64, (cuuint64_t)lines}; cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 256}, estr[2] = {1, 1};
  encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* out; cudaMalloc(&out, 8 * 2048);
  cudaFuncSetAttribute(port_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kTile);
  for (int use_tma : {1, 0}) for (int w : {0, 2, 4, 8, 14}) {
    if (!use_tma && w == 0) continue;
    cudaMemset(out, 0, 8 * 2048);
    const int iters = 3000;
    port_bench<<<148, 512, kStages * kTile>>>(tm, iters, lines, (const uint4*)buf2, bytes / 16, w, out, use_tma);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[4]; cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    double tma_bpc = use_tma ? (double)iters * kTile / h[0] : 0;
    double ld_bpc = w ? (double)h[2] / ((double)h[1] / w) : 0;  // bytes per cycle while LD warps ran
    printf("tma=%d ld_warps=%2d err=%d  TMA %.1f B/clk/SM  LDG %.1f B/clk/SM  (sum %.1f)\n", use_tma, w, (int)e, tma_bpc, ld_bpc, tma_bpc + ld_bpc);
  }
  return 0;
}
