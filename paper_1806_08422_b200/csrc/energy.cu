// Exact Ising energy of +-1 configurations, best-of-reads, sign extraction.
//
// energy(c) = sum_(i<j) w_ij c_i c_j + sum_i h_i c_i   (problem.py:150-154)
//
// Configs are bit-packed 32 replicas per word (bits[i][word], bit set for
// c = -1), so every canonical edge (i, j, w) is one warp-uniform broadcast
// and each lane adds +w or -w for its replica from (b_i ^ b_j).  Partial sums
// over edge chunks are float64 and reduced in a fixed order (deterministic);
// for integer weights every partial is an exact integer, so the result is
// bit-identical to the reference's float64 dot for any summation order.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace nmfa {

// bits[i * W + wd] bit l  <=>  cfg[(32*wd + l) * n + i] < 0
__global__ void pack_bits_kernel(const int8_t* __restrict__ cfg, long long R, int n, long long W,
                                 uint32_t* __restrict__ bits) {
  // word index on grid.x (R * t_f configurations can exceed 65535 * 32), 128-spin
  // blocks on grid.y, strided when n / 128 exceeds the grid
  __shared__ int8_t tile[32][129];
  const long long wd = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long i0 = (long long)blockIdx.y * 128; i0 < n; i0 += (long long)gridDim.y * 128) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 128; e += blockDim.x) {
      const int rr = e >> 7, ii = e & 127;
      const long long r = wd * 32 + rr;
      tile[rr][ii] = (r < R && i0 + ii < n) ? cfg[r * n + i0 + ii] : (int8_t)1;
    }
    __syncthreads();
    for (int ii = warp; ii < 128; ii += blockDim.x >> 5) {
      const uint32_t b = __ballot_sync(0xffffffffu, tile[lane][ii] < 0);
      if (lane == 0 && i0 + ii < n) bits[(i0 + ii) * W + wd] = b;
    }
  }
}

// part[c][r]: rows c < e_chunks are chunks of the canonical edge list, rows
// e_chunks <= c < e_chunks + f_chunks chunks of the spins for the field term
// (no field rows when h = 0).  Each row is one grid row of warps, 32 replicas
// per warp.
__global__ void __launch_bounds__(128) energy_partial_kernel(
    const uint32_t* __restrict__ bits, long long R, long long W, int n, long long n_edges,
    const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
    const double* __restrict__ ew, const double* __restrict__ h, long long e_chunks,
    long long f_chunks, double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const long long wd = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (wd >= W) return;
  const long long r = wd * 32 + lane;
  const long long c = blockIdx.y;
  double acc = 0.0;
  if (c < e_chunks) {
    const long long k0 = n_edges * c / e_chunks, k1 = n_edges * (c + 1) / e_chunks;
    for (long long k = k0; k < k1; ++k) {
      const uint32_t x = __ldg(bits + (long long)__ldg(ei + k) * W + wd) ^
                         __ldg(bits + (long long)__ldg(ej + k) * W + wd);
      const double w = __ldg(ew + k);
      acc += ((x >> lane) & 1u) ? -w : w;
    }
  } else {
    const long long f = c - e_chunks;
    const int i0 = (int)(n * f / f_chunks), i1 = (int)(n * (f + 1) / f_chunks);
    for (int i = i0; i < i1; ++i) {
      const double hv = __ldg(h + i);
      const uint32_t b = __ldg(bits + (long long)i * W + wd);
      acc += ((b >> lane) & 1u) ? -hv : hv;
    }
  }
  if (r < R) part[c * R + r] = acc;
}

__global__ void energy_reduce_kernel(const double* __restrict__ part, long long R,
                                     long long e_chunks, long long f_chunks,
                                     double* __restrict__ e) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double pair = 0.0, field = 0.0;
  for (long long c = 0; c < e_chunks; ++c) pair += part[c * R + r];
  for (long long c = e_chunks; c < e_chunks + f_chunks; ++c) field += part[c * R + r];
  e[r] = pair + field;  // pair + field, like problem.py:153-154
}

// Edge chunks: enough warps for ~8 per SM, >= 512 edges each.  Field chunks:
// 2048 spins each (a single serial row cost 14 ms at n = 131072), none when
// h = 0 (the field term is then +0.0 exactly, as before).
static int64_t edge_chunks_for(const nmfa_problem* p, int64_t n_cfg) {
  const int64_t W = (n_cfg + 31) / 32;
  const int64_t nblk = (W + 3) / 4;
  int64_t want = (148 * 8 + nblk - 1) / nblk;
  int64_t cap = p->n_edges / 512;
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return want;
}

static int64_t field_chunks_for(const nmfa_problem* p) {
  return p->has_field ? std::max<int64_t>(1, (p->n + 2047) / 2048) : 0;
}

// Scratch rows minus one (callers allocate (chunks + 1) * n_cfg doubles).
int64_t energy_chunks_for(const nmfa_problem* p, int64_t n_cfg) {
  return edge_chunks_for(p, n_cfg) + field_chunks_for(p) - 1;
}

int launch_energy(const nmfa_problem* p, const int8_t* cfg, int64_t R, double* energy,
                  uint32_t* bits, double* part, int64_t chunks, cudaStream_t st) {
  const long long W = (R + 31) / 32;
  dim3 g1((unsigned)W, (unsigned)std::min<long long>((p->n + 127) / 128, 65535));
  pack_bits_kernel<<<g1, 256, 0, st>>>(cfg, R, (int)p->n, W, bits);
  NMFA_LAUNCH_CHECK();
  // `part` holds chunks + 1 rows (energy_chunks_for): field rows first claimed
  const long long f_chunks = field_chunks_for(p);
  const long long e_chunks = chunks + 1 - f_chunks;
  if (e_chunks < 1) {
    set_error("energy scratch too small");
    return NMFA_ERR_ARG;
  }
  dim3 g2((unsigned)((W + 3) / 4), (unsigned)(e_chunks + f_chunks));
  energy_partial_kernel<<<g2, 128, 0, st>>>(bits, R, W, (int)p->n, p->n_edges, p->d_e_i,
                                            p->d_e_j, p->d_e_w, p->d_h, e_chunks, f_chunks, part);
  NMFA_LAUNCH_CHECK();
  energy_reduce_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(part, R, e_chunks, f_chunks,
                                                                   energy);
  NMFA_LAUNCH_CHECK();
  add_launches(3);
  return NMFA_OK;
}

__global__ void sign_kernel(const float* __restrict__ s, long long count, int8_t* __restrict__ c) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < count) c[k] = s[k] < 0.f ? (int8_t)-1 : (int8_t)1;  // problem.py:181-183
}

int launch_sign(const float* s, int64_t count, int8_t* cfg, cudaStream_t st) {
  sign_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(s, count, cfg);
  NMFA_LAUNCH_CHECK();
  add_launches(1);
  return NMFA_OK;
}

// min energy, lowest index among ties (cli.py:236 `np.min`; argmin semantics)
__global__ void __launch_bounds__(1024) best_of_kernel(const double* __restrict__ e, long long n,
                                                      double* best_e, long long* best_i) {
  __shared__ double se[32];
  __shared__ long long si[32];
  double v = DBL_MAX;
  long long vi = LLONG_MAX;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    const double x = e[k];
    if (x < v || (x == v && k < vi)) {
      v = x;
      vi = k;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, vi, o);
    if (ov < v || (ov == v && oi < vi)) {
      v = ov;
      vi = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    se[warp] = v;
    si[warp] = vi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    v = lane < nw ? se[lane] : DBL_MAX;
    vi = lane < nw ? si[lane] : LLONG_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, vi, o);
      if (ov < v || (ov == v && oi < vi)) {
        v = ov;
        vi = oi;
      }
    }
    if (lane == 0) {
      *best_e = v;
      *best_i = vi;
    }
  }
}

int launch_best_of(const double* e, int64_t n, double* best_e, int64_t* best_i,
                   cudaStream_t st) {
  best_of_kernel<<<1, 1024, 0, st>>>(e, n, best_e, reinterpret_cast<long long*>(best_i));
  NMFA_LAUNCH_CHECK();
  add_launches(1);
  return NMFA_OK;
}

}  // namespace nmfa
