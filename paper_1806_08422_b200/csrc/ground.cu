// Exact ground state by exhaustive enumeration (brute_force_ground,
// metrics.py:53-67; kernel gray_ground, _kernels_numba.py:83-114).
//
// Every thread owns a prefix of the high spins and walks the 2^b low-spin
// configurations in Gray-code order, one single-spin flip per step with an
// incremental energy update dE = -2 s_v (h_v + sum_j J_vj s_j).
//  * Integer path (every J_ij in {-1, 0, +1}, integer h, bounded energies):
//    the field of spin v is rowsum_v - 2 (popc(P_v & b) - popc(N_v & b)) with
//    bitmasks of its positive / negative neighbours -- O(1), exact int64.
//  * General path: f64 field from the dense J row in shared memory (the
//    reference's arithmetic class); ties within TIE_TOL = 1e-9 as in the
//    reference (_kernels_numba.py:21, 108-112).
// With h = 0 the energy is invariant under a global flip, so the top spin is
// fixed to -1 and every count doubles.
// Blocks reduce (min energy, count, one argmin configuration); the host
// combines the block results.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace nmfa {

constexpr int kGroundMaxN = 40;
constexpr int kGroundThreads = 256;
constexpr double kTieTol = 1e-9;

struct GroundArgs {
  int n, b;                    // spins, walked (suffix) bits
  int fix_top;                 // h == 0: top spin fixed to -1 (bit 0)
  long long n_prefix;          // prefixes (threads)
  // integer path
  const unsigned long long* pmask;  // [n] positive-neighbour masks
  const unsigned long long* nmask;  // [n] negative-neighbour masks
  const long long* hint;            // [n] integer fields
  const long long* rowsum;          // [n] sum_j J_vj
  // general path
  const double* J;             // [n][n] dense, zero diagonal
  const double* h;             // [n]
  // per-block results
  double* blk_e;
  long long* blk_c;
  unsigned long long* blk_cfg;
};

// bit i of a configuration index = 1 means s_i = +1; the walk starts from
// s = -1 everywhere, like the reference (_kernels_numba.py:86).
template <bool kInt>
__global__ void __launch_bounds__(kGroundThreads) ground_kernel(const GroundArgs a) {
  __shared__ double sJ[kGroundMaxN * kGroundMaxN];
  __shared__ double sh[kGroundMaxN];
  __shared__ unsigned long long sP[kGroundMaxN], sN[kGroundMaxN];
  __shared__ long long sH[kGroundMaxN], sR[kGroundMaxN];
  const int n = a.n;
  if (kInt) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      sP[k] = a.pmask[k];
      sN[k] = a.nmask[k];
      sH[k] = a.hint[k];
      sR[k] = a.rowsum[k];
    }
  } else {
    for (int k = threadIdx.x; k < n * n; k += blockDim.x) sJ[k] = a.J[k];
    for (int k = threadIdx.x; k < n; k += blockDim.x) sh[k] = a.h[k];
  }
  __syncthreads();

  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double best_e = 1e300;
  long long best_c = 0;
  unsigned long long best_cfg = 0;
  if (tid < a.n_prefix) {
    // prefix bits occupy positions [b, n); the walk covers [0, b)
    unsigned long long bits = (unsigned long long)tid << a.b;
    // energy of the starting configuration (suffix all -1)
    if (kInt) {
      long long e2 = 0;  // 2E = sum_i s_i (2 h_i + sum_j J_ij s_j)
      for (int i = 0; i < n; ++i) {
        const long long si = ((bits >> i) & 1ULL) ? 1 : -1;
        const long long f = 2LL * ((long long)__popcll(sP[i] & bits) - (long long)__popcll(sN[i] & bits)) - sR[i];
        e2 += si * (2 * sH[i] + f);
      }
      long long e = e2 / 2, emin = e, cnt = 1;
      unsigned long long cfg = bits;
      const long long steps = 1LL << a.b;
      for (long long step = 1; step < steps; ++step) {
        const int v = __ffsll(step) - 1;  // trailing zeros
        const long long sv = ((bits >> v) & 1ULL) ? 1 : -1;
        const long long f = sH[v] + 2LL * ((long long)__popcll(sP[v] & bits) - (long long)__popcll(sN[v] & bits)) - sR[v];
        e -= 2 * sv * f;
        bits ^= 1ULL << v;
        if (e < emin) {
          emin = e;
          cnt = 1;
          cfg = bits;
        } else if (e == emin) {
          ++cnt;
        }
      }
      best_e = (double)emin;
      best_c = cnt;
      best_cfg = cfg;
    } else {
      double e = 0.0;
      for (int i = 0; i < n; ++i) {
        const double si = ((bits >> i) & 1ULL) ? 1.0 : -1.0;
        double f = 0.0;
        for (int j = i + 1; j < n; ++j) f += sJ[i * n + j] * (((bits >> j) & 1ULL) ? 1.0 : -1.0);
        e += si * (f + sh[i]);
      }
      double emin = e;
      long long cnt = 1;
      unsigned long long cfg = bits;
      const long long steps = 1LL << a.b;
      for (long long step = 1; step < steps; ++step) {
        const int v = __ffsll(step) - 1;
        const double sv = ((bits >> v) & 1ULL) ? 1.0 : -1.0;
        double f = sh[v];
        for (int j = 0; j < n; ++j) f += sJ[v * n + j] * (((bits >> j) & 1ULL) ? 1.0 : -1.0);
        e -= 2.0 * sv * f;
        bits ^= 1ULL << v;
        if (e < emin - kTieTol) {
          emin = e;
          cnt = 1;
          cfg = bits;
        } else if (e <= emin + kTieTol) {
          ++cnt;
        }
      }
      best_e = emin;
      best_c = cnt;
      best_cfg = cfg;
    }
    if (a.fix_top) best_c *= 2;  // E(s) == E(-s) exactly when h == 0
  }
  // block reduction: minimum energy (ties within tolerance add counts; the
  // argmin kept is the smallest configuration index among exact minima)
  __shared__ double re[kGroundThreads];
  __shared__ long long rc[kGroundThreads];
  __shared__ unsigned long long rg[kGroundThreads];
  re[threadIdx.x] = best_e;
  rc[threadIdx.x] = best_c;
  rg[threadIdx.x] = best_cfg;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double e1 = re[threadIdx.x], e2 = re[threadIdx.x + s];
      const long long c1 = rc[threadIdx.x], c2 = rc[threadIdx.x + s];
      const double tol = kInt ? 0.0 : kTieTol;
      if (e2 < e1 - tol) {
        re[threadIdx.x] = e2;
        rc[threadIdx.x] = c2;
        rg[threadIdx.x] = rg[threadIdx.x + s];
      } else if (e2 <= e1 + tol) {
        rc[threadIdx.x] = c1 + c2;
        if (e2 < e1 || (e2 == e1 && rg[threadIdx.x + s] < rg[threadIdx.x])) {
          re[threadIdx.x] = e2;
          rg[threadIdx.x] = rg[threadIdx.x + s];
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.blk_e[blockIdx.x] = re[0];
    a.blk_c[blockIdx.x] = rc[0];
    a.blk_cfg[blockIdx.x] = rg[0];
  }
}

int ground_state(const nmfa_problem* p, int max_n, double* energy, int64_t* degeneracy,
                 int8_t* config) {
  const int n = (int)p->n;
  if (n > max_n || n > kGroundMaxN) {
    set_error("exhaustive enumeration is limited to n <= " + std::to_string(std::min(max_n, kGroundMaxN)) +
              ", got n = " + std::to_string(n));
    return NMFA_ERR_ARG;
  }
  if (p->device_generated) {
    set_error("exhaustive enumeration needs the host edge list (device-generated problem)");
    return NMFA_ERR_STATE;
  }
  // dense J and h from the canonical edge list (host copies)
  std::vector<double> J((size_t)n * n, 0.0), h(p->h.begin(), p->h.end());
  std::vector<int32_t> ei(p->n_edges), ej(p->n_edges);
  std::vector<double> ew(p->n_edges);
  if (p->n_edges) {
    NMFA_CUDA_TRY(cudaMemcpy(ei.data(), p->d_e_i, 4 * p->n_edges, cudaMemcpyDeviceToHost));
    NMFA_CUDA_TRY(cudaMemcpy(ej.data(), p->d_e_j, 4 * p->n_edges, cudaMemcpyDeviceToHost));
    NMFA_CUDA_TRY(cudaMemcpy(ew.data(), p->d_e_w, 8 * p->n_edges, cudaMemcpyDeviceToHost));
  }
  bool pm1 = true;
  for (int64_t k = 0; k < p->n_edges; ++k) {
    J[(size_t)ei[k] * n + ej[k]] += ew[k];
    J[(size_t)ej[k] * n + ei[k]] += ew[k];
  }
  for (double v : J) pm1 = pm1 && (v == 0.0 || v == 1.0 || v == -1.0);
  double hsum = 0.0;
  bool hint_ok = true, hzero = true;
  for (double v : h) {
    hint_ok = hint_ok && v == std::floor(v) && std::fabs(v) < 1e12;
    hzero = hzero && v == 0.0;
    hsum += std::fabs(v);
  }
  const bool use_int = pm1 && hint_ok && hsum < 1e15;
  if (n == 0) {
    *energy = 0.0;
    *degeneracy = 1;
    return NMFA_OK;
  }

  GroundArgs a{};
  a.n = n;
  a.fix_top = hzero && n >= 1;
  const int free_bits = n - (a.fix_top ? 1 : 0);
  // walk length 2^b: at most 2^12 steps, shortened (down to 2^6) so that at
  // least 2^16 threads enumerate in parallel when the problem allows it
  a.b = std::min(free_bits, std::max(6, std::min(12, free_bits - 16)));
  a.n_prefix = 1LL << (free_bits - a.b);
  const long long blocks = (a.n_prefix + kGroundThreads - 1) / kGroundThreads;

  std::vector<unsigned long long> pm(n, 0), nm(n, 0);
  std::vector<long long> hi(n, 0), rs(n, 0);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      const double v = J[(size_t)i * n + j];
      if (v == 1.0) pm[i] |= 1ULL << j;
      if (v == -1.0) nm[i] |= 1ULL << j;
      rs[i] += (long long)v;
    }
    hi[i] = use_int ? (long long)h[i] : 0;
  }
  void* dbuf = nullptr;
  const size_t bytes = (size_t)n * n * 8 + (size_t)n * 8 * 5 + (size_t)blocks * 24;
  NMFA_CUDA_TRY(cudaMalloc(&dbuf, bytes));
  uint8_t* b8 = static_cast<uint8_t*>(dbuf);
  double* dJ = reinterpret_cast<double*>(b8);
  double* dh = dJ + (size_t)n * n;
  auto* dP = reinterpret_cast<unsigned long long*>(dh + n);
  auto* dN = dP + n;
  auto* dHi = reinterpret_cast<long long*>(dN + n);
  auto* dRs = dHi + n;
  double* dBe = reinterpret_cast<double*>(dRs + n);
  auto* dBc = reinterpret_cast<long long*>(dBe + blocks);
  auto* dBg = reinterpret_cast<unsigned long long*>(dBc + blocks);
  int err = NMFA_OK;
  do {
    if (cudaMemcpy(dJ, J.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(dh, h.data(), (size_t)n * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(dP, pm.data(), (size_t)n * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(dN, nm.data(), (size_t)n * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(dHi, hi.data(), (size_t)n * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(dRs, rs.data(), (size_t)n * 8, cudaMemcpyHostToDevice)) {
      set_error("cudaMemcpy failed in ground_state");
      err = NMFA_ERR_CUDA;
      break;
    }
    a.pmask = dP;
    a.nmask = dN;
    a.hint = dHi;
    a.rowsum = dRs;
    a.J = dJ;
    a.h = dh;
    a.blk_e = dBe;
    a.blk_c = dBc;
    a.blk_cfg = dBg;
    if (use_int)
      ground_kernel<true><<<(unsigned)blocks, kGroundThreads>>>(a);
    else
      ground_kernel<false><<<(unsigned)blocks, kGroundThreads>>>(a);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("ground_kernel failed");
      err = NMFA_ERR_CUDA;
      break;
    }
    add_launches(1);
    std::vector<double> be(blocks);
    std::vector<long long> bc(blocks);
    std::vector<unsigned long long> bg(blocks);
    if (cudaMemcpy(be.data(), dBe, blocks * 8, cudaMemcpyDeviceToHost) ||
        cudaMemcpy(bc.data(), dBc, blocks * 8, cudaMemcpyDeviceToHost) ||
        cudaMemcpy(bg.data(), dBg, blocks * 8, cudaMemcpyDeviceToHost)) {
      set_error("cudaMemcpy failed in ground_state");
      err = NMFA_ERR_CUDA;
      break;
    }
    const double tol = use_int ? 0.0 : kTieTol;
    double emin = be[0];
    long long cnt = bc[0];
    unsigned long long g = bg[0];
    for (long long k = 1; k < blocks; ++k) {
      if (be[k] < emin - tol) {
        emin = be[k];
        cnt = bc[k];
        g = bg[k];
      } else if (be[k] <= emin + tol) {
        cnt += bc[k];
        if (be[k] < emin || (be[k] == emin && bg[k] < g)) {
          emin = be[k];
          g = bg[k];
        }
      }
    }
    *energy = emin;
    *degeneracy = cnt;
    if (config)
      for (int i = 0; i < n; ++i) config[i] = ((g >> i) & 1ULL) ? (int8_t)1 : (int8_t)-1;
  } while (0);
  cudaFree(dbuf);
  return err;
}

}  // namespace nmfa
