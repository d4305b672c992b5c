// Sparse NMFA step (CSR gather), one launch per step.
// State layout: S[i][r] fp32, replicas contiguous (Rp = R rounded up to 32),
// ping-pong between two buffers (synchronous update, SPEC: all mean fields
// from the incoming S).  One warp owns a group of 8 consecutive spins for 32
// consecutive replicas: every CSR entry (j, w) is a warp-uniform broadcast
// and the gather S[j][r..r+31] is one coalesced 128-byte load.  The group
// matches the Philox counter granularity, so one Philox call per thread
// feeds its eight spins (common.cuh noise identity).
// Reference: _kernels_numba.py:48-56 (row accumulate, then tanh/mix).
#include "common.cuh"
#include "internal.h"

#ifndef NMFA_SPARSE_MINB
#define NMFA_SPARSE_MINB 4  // blocks per SM the register budget targets
#endif

namespace nmfa {

struct SparseStepArgs {
  const int32_t* ptr;
  const int32_t* idx;
  const float* w;
  const float* invn;
  const float* hn;
  const float* s_old;
  float* s_new;
  int n, t, t_f;
  long long R, Rp;
  float inv_t, alpha, oma, sigma;
  unsigned long long key_base;
  const float* noise;  // [R][t_f][n] or null
  int8_t* cfg;         // written at the last step
  float* s_out;
  float* s_hist;
  int last;
};

__global__ void __launch_bounds__(256, NMFA_SPARSE_MINB) sparse_step_kernel(const SparseStepArgs a) {
  // grid (replica-group blocks, spin groups): warp w of block x owns replicas
  // [32 (8x + w), +32) of spin group y, so consecutive blocks read the same
  // state rows (no index division; 32-bit element offsets, n * Rp < 2^31)
  const int lane = threadIdx.x & 31;
  const int rb = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int Rp = (int)a.Rp, n = a.n;
  if (rb * 32 >= Rp) return;
  const int q = blockIdx.y;
  const int r = rb * 32 + lane;
  const float* __restrict__ so = a.s_old + r;
  const int* __restrict__ idx = a.idx;
  const float* __restrict__ wts = a.w;

  // Memory-level parallelism: the group's 9 row pointers come from one
  // cooperative load; then every gather of the 8 spins is issued before the
  // first use (degree <= kFast unrolled, longer rows in a general loop).
  constexpr int kFast = 3;  // unrolled row length (cubic / Moebius ladder); longer rows loop
  const int i_base = 8 * q;
  const int pl = lane <= 8 ? __ldg(a.ptr + min(i_base + lane, n)) : 0;
  int k0[8], deg[8];
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    k0[qq] = __shfl_sync(0xffffffffu, pl, qq);
    deg[qq] = __shfl_sync(0xffffffffu, pl, qq + 1) - k0[qq];
  }
  float sold[8];
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) sold[qq] = (i_base + qq < n) ? so[(i_base + qq) * Rp] : 0.f;
  float v[8][kFast];
  float acc[8];
  const int K0 = k0[0], seg = k0[7] + deg[7] - K0;  // the group's CSR entries [K0, K0 + seg)
  bool fast = seg <= 32;
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) fast = fast && deg[qq] <= kFast;
  if (fast) {
    // lanes hold the segment's element offsets (idx * Rp) and weights; every
    // gather broadcasts its entry by shuffle (no per-lane index arithmetic)
    const int off_l = lane < seg ? __ldg(idx + K0 + lane) * Rp : 0;
    const float w_l = lane < seg ? __ldg(wts + K0 + lane) : 0.f;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        const int off = __shfl_sync(0xffffffffu, off_l, (k0[qq] - K0 + u) & 31);
        v[qq][u] = u < deg[qq] ? so[off] : 0.f;
      }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2 = 0.f;
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        const float wv = __shfl_sync(0xffffffffu, w_l, (k0[qq] - K0 + u) & 31);
        if (u < deg[qq]) s2 = fmaf(wv, v[qq][u], s2);  // CSR order, like the general path
      }
      acc[qq] = s2;
    }
  } else {
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
#pragma unroll
      for (int u = 0; u < kFast; ++u)
        v[qq][u] = u < deg[qq] ? so[__ldg(idx + k0[qq] + u) * Rp] : 0.f;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2 = 0.f;
#pragma unroll
      for (int u = 0; u < kFast; ++u)
        if (u < deg[qq]) s2 = fmaf(__ldg(wts + k0[qq] + u), v[qq][u], s2);  // uniform: L1 broadcast
      for (int k = k0[qq] + kFast; k < k0[qq] + deg[qq]; ++k)  // rows longer than kFast
        s2 = fmaf(__ldg(wts + k), so[__ldg(idx + k) * Rp], s2);
      acc[qq] = s2;
    }
  }
  const bool valid = r < a.R;
  float z[8];
  if (a.noise) {
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      const int i = i_base + qq;
      z[qq] = (valid && i < n) ? a.noise[((long long)r * a.t_f + a.t) * n + i] : 0.f;
    }
  } else {
    const unsigned long long key = a.key_base + (unsigned long long)r;
    normal8(philox_schedule((uint32_t)key, (uint32_t)(key >> 32)), (uint32_t)q, (uint32_t)a.t,
            bm_scale(a.sigma), z);
  }
  float* __restrict__ sn = a.s_new + r;
  const float inv_t = a.inv_t, alpha = a.alpha, oma = a.oma;
  const bool extra = valid && (a.s_hist != nullptr || a.last);
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    const int i = i_base + qq;
    if (i >= n) break;
    const float s = nmfa_update(acc[qq], __ldg(a.invn + i), __ldg(a.hn + i), z[qq], inv_t, alpha,
                                oma, sold[qq]);
    sn[i * Rp] = s;
    if (extra) {
      if (a.s_hist) a.s_hist[((long long)r * a.t_f + a.t) * n + i] = s;
      if (a.last) {
        a.cfg[(long long)r * n + i] = s < 0.f ? (int8_t)-1 : (int8_t)1;
        if (a.s_out) a.s_out[(long long)r * n + i] = s;
      }
    }
  }
}

// S[i][r] <- s0[r][i] (or 0) for the padded state.
__global__ void sparse_init_kernel(float* s, const float* s0, int n, long long R, long long Rp) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * Rp) return;
  const long long i = e / Rp, r = e - i * Rp;
  s[e] = (s0 && r < R) ? s0[r * n + i] : 0.f;
}

int launch_sparse_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                         const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                         cudaStream_t st) {
  const nmfa_problem* p = pl->p;
  const long long tot = (long long)p->n * pl->Rp;
  sparse_init_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->d_sa, s0, (int)p->n,
                                                                     pl->R, pl->Rp);
  NMFA_LAUNCH_CHECK();
  const std::vector<float>& inv_t = pl->h_inv_temp;
  SparseStepArgs a{};
  a.ptr = p->d_csr_ptr;
  a.idx = p->d_csr_idx;
  a.w = p->d_csr_w;
  a.invn = p->d_invn;
  a.hn = p->d_hn;
  a.n = (int)p->n;
  a.t_f = pl->t_f;
  a.R = pl->R;
  a.Rp = pl->Rp;
  a.alpha = pl->alpha;
  a.oma = pl->oma;
  a.sigma = pl->sigma;
  a.key_base = key_base;
  a.noise = noise;
  a.cfg = cfg;
  a.s_out = s_out;
  a.s_hist = s_hist;
  if ((long long)p->n * pl->Rp >= (1LL << 31) || (p->n + 7) / 8 > 65535) {
    set_error("sparse path: needs n <= 524280 and n x padded replicas < 2^31 per plan");
    return NMFA_ERR_ARG;
  }
  const dim3 grid((unsigned)((pl->Rp / 32 + 7) / 8), (unsigned)((p->n + 7) / 8));
  float* cur = pl->d_sa;
  float* nxt = pl->d_sb;
  for (int t = 0; t < pl->t_f; ++t) {
    a.t = t;
    a.inv_t = inv_t[t];
    a.last = (t == pl->t_f - 1);
    a.s_old = cur;
    a.s_new = nxt;
    sparse_step_kernel<<<grid, 256, 0, st>>>(a);
    NMFA_LAUNCH_CHECK();
    std::swap(cur, nxt);
  }
  add_launches(1 + pl->t_f);
  return NMFA_OK;
}

}  // namespace nmfa
