// Microbenchmark: throughput of the fused NMFA update (update16: Philox + Box-Muller
// + odd tanh + damping) in isolation, vs warps per SM.  Elements/cycle/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/epi_bench tools/epi_bench.cu
#include <cstdio>

#include "../paper_1806_08422_b200/csrc/common.cuh"

using namespace nmfa;

template <int kMinBlocks>
__global__ void __launch_bounds__(512, kMinBlocks) epi_bench(int chunks, const float* invn, const float* hn,
                                                             float* out, unsigned long long* cyc) {
  const int tid = threadIdx.x;
  const unsigned long long key = 12345ull + blockIdx.x * blockDim.x + tid;
  const PhiloxKey K = philox_schedule((uint32_t)key, (uint32_t)(key >> 32));
  float ms[16], acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) { ms[c] = 0.01f * c; acc[c] = 0.3f * (c - 7); }
  const float4* invn4 = reinterpret_cast<const float4*>(invn);
  const float4* hn4 = reinterpret_cast<const float4*>(hn);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int k = 0; k < chunks; ++k) {
    update16<false>(acc, ms, invn4 + (k & 7) * 4, hn4 + (k & 7) * 4, nullptr, 16, K, (uint32_t)k,
                    7u, 0.15f, 1.3f, 0.15f, 0.85f);
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = ms[(c + 1) & 15] * 31.f;
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += ms[c];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float *invn, *hn, *out;
  unsigned long long* cyc;
  cudaError_t e0r = cudaMalloc(&invn, 512 * 4); printf("init: %s\n", cudaGetErrorString(e0r)); cudaMalloc(&hn, 512 * 4);
  cudaMemset(invn, 0, 512 * 4); cudaMemset(hn, 0, 512 * 4);
  cudaMalloc(&out, 148 * 4 * 512 * 4); cudaMalloc(&cyc, 148 * 4 * 8);
  const int chunks = 200;
  for (int warps : {4, 8, 16, 32}) {
    for (int bps : {1, 2}) {
      const int threads = warps * 32 / bps;
      if (threads > 512) continue;
      if (bps == 1) epi_bench<1><<<148 * bps, threads>>>(chunks, invn, hn, out, cyc);
      else epi_bench<2><<<148 * bps, threads>>>(chunks, invn, hn, out, cyc);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (bps == 1) epi_bench<1><<<148 * bps, threads>>>(chunks, invn, hn, out, cyc);
      else epi_bench<2><<<148 * bps, threads>>>(chunks, invn, hn, out, cyc);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double elems_per_sm = (double)warps * 32 * chunks * 16;
      printf("warps/SM=%2d (%d CTA x %3d thr) err=%s  cycles=%llu  elem/cycle/SM=%.2f  chip=%.3e elem/s\n",
             warps, bps, threads, cudaGetErrorString(err), h, elems_per_sm / h, elems_per_sm * 148 / (ms * 1e-3));
    }
  }
  return 0;
}
