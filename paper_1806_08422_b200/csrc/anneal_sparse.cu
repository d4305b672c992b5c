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

__global__ void __launch_bounds__(256) sparse_step_kernel(const SparseStepArgs a) {
  const int lane = threadIdx.x & 31;
  const long long wg = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nrb = a.Rp / 32;
  const long long q = wg / nrb;
  const long long rb = wg - q * nrb;
  if (8 * q >= a.n) return;
  const long long r = rb * 32 + lane;

  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    const int i = (int)(8 * q) + qq;
    if (i < a.n) {
      const int k1 = __ldg(a.ptr + i + 1);
      float s = 0.f;
      for (int k = __ldg(a.ptr + i); k < k1; ++k)
        s = fmaf(__ldg(a.w + k), a.s_old[(long long)__ldg(a.idx + k) * a.Rp + r], s);
      acc[qq] = s;
    }
  }
  const bool valid = r < a.R;
  float z[8];
  if (a.noise) {
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      const int i = (int)(8 * q) + qq;
      z[qq] = (valid && i < a.n) ? a.noise[((long long)r * a.t_f + a.t) * a.n + i] : 0.f;
    }
  } else {
    const unsigned long long key = a.key_base + (unsigned long long)r;
    normal8(philox_schedule((uint32_t)key, (uint32_t)(key >> 32)), (uint32_t)q, (uint32_t)a.t,
            bm_scale(a.sigma), z);
  }
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    const int i = (int)(8 * q) + qq;
    if (i >= a.n) break;
    const long long o = (long long)i * a.Rp + r;
    const float s = nmfa_update(acc[qq], __ldg(a.invn + i), __ldg(a.hn + i), z[qq], a.inv_t,
                                a.alpha, a.oma, a.s_old[o]);
    a.s_new[o] = s;
    if (valid) {
      if (a.s_hist) a.s_hist[((long long)r * a.t_f + a.t) * a.n + i] = s;
      if (a.last) {
        a.cfg[r * a.n + i] = s < 0.f ? (int8_t)-1 : (int8_t)1;
        if (a.s_out) a.s_out[r * a.n + i] = s;
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
  const long long warps = ((p->n + 7) / 8) * (pl->Rp / 32);
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  float* cur = pl->d_sa;
  float* nxt = pl->d_sb;
  for (int t = 0; t < pl->t_f; ++t) {
    a.t = t;
    a.inv_t = inv_t[t];
    a.last = (t == pl->t_f - 1);
    a.s_old = cur;
    a.s_new = nxt;
    sparse_step_kernel<<<blocks, 256, 0, st>>>(a);
    NMFA_LAUNCH_CHECK();
    std::swap(cur, nxt);
  }
  add_launches(1 + pl->t_f);
  return NMFA_OK;
}

}  // namespace nmfa
