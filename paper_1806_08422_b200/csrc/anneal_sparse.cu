// Sparse NMFA step, one launch per step: ELL gather (max degree <= 4) or
// CSR gather (any degree).
// State layout: S[i][r] fp32, replicas contiguous (Rp = R rounded up to 32),
// ping-pong between two buffers (synchronous update, SPEC: all mean fields
// from the incoming S).  One warp owns a group of 8 consecutive spins for
// 32V consecutive replicas (V = 2: one float2 per lane): every row entry
// (j, w) is a warp-uniform broadcast and the gather S[j][r..r+32V) is one
// coalesced load.  The group matches the Philox counter granularity, so one
// Philox call per replica feeds its eight spins (common.cuh noise identity).
// Both kernels sum each row in CSR order from +0, so they agree bit for bit.
// The CSR kernel stages a group's segment (<= 64 or <= 96 entries) in lane
// registers and broadcasts offsets by shuffle; its three instances (64-entry
// staging, 96-entry staging, 96 + 3 entries per row per round beyond) are
// chosen per problem from the segment-size histogram (capi.cu csr_variant).
// Measured design steps: profiles/r01/ell_notes.log, profiles/r02/
// csr_staged_segments.log, DESIGN.md section 6.
// Reference: _kernels_numba.py:48-56 (row accumulate, then tanh/mix).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

#ifndef NMFA_CSR_ROUNDS
#define NMFA_CSR_ROUNDS 2
#endif
#ifndef NMFA_CSR_ROUNDS_LONG
#define NMFA_CSR_ROUNDS_LONG 2  // the default instances; 3 in the long-segment instance
#endif
#ifndef NMFA_FULL_GROUP_STORES
#define NMFA_FULL_GROUP_STORES 1  // unpredicated state stores for interior groups (+1%)
#endif
#ifndef NMFA_ELL_FULL_GROUPS
#define NMFA_ELL_FULL_GROUPS 1  // unpredicated state loads for interior groups (+1-1.5%, no spill)
#endif
#ifndef NMFA_ELL4_MINB
#define NMFA_ELL4_MINB 2  // the degree-4 ELL variant (A/B knob)
#endif
#ifndef NMFA_ELL_MINB
#define NMFA_ELL_MINB 2  // ELL kernel blocks per SM (128 registers, no spill at V = 2)
#endif
#ifdef NMFA_CSR_UNSTAGED  // A/B: no staged-segment path in the CSR kernel
constexpr bool kDisableStaged = true;
#else
constexpr bool kDisableStaged = false;
#endif

#ifndef NMFA_SPARSE_MINB
#define NMFA_SPARSE_MINB 4  // blocks per SM the register budget targets
#endif

namespace nmfa {

struct SparseStepArgs {
  const int32_t* ptr;
  const int32_t* idx;
  const float* w;
  const int32_t* ell_idx;  // ELL rows (problem ell_k > 0), else null
  const float* ell_w;
  int groups_per_warp;     // ELL kernel: consecutive spin groups per warp
  uint32_t elem_bytes;     // sizeof(float), passed at run time (see elem_addr)
  int slices_per_block;    // ELL kernel: replica slices per block (1, 2, 4, 8)
  const float* invn;
  const float* hn;
  const float* s_old;
  float* s_new;
  int n, t, t_f;
  long long R, Rp;
  float inv_t, alpha, oma, sigma;
  const unsigned long long* key_base;  // device word, written per run (graph-stable args)
  const float* noise;  // [R][t_f][n] or null
  int8_t* cfg;         // written at the last step
  float* s_out;
  float* s_hist;
  int last;
};

// p + off elements in ONE instruction (IMAD.WIDE.U32).  Written as plain C++
// the compiler re-associates (s_old + r) + off into 64-bit sign-extended
// arithmetic, four instructions per gather (profiles/r01/ell_notes.log).
// Element offsets are < 2^31 (n x Rp bound checked at launch).  The result is
// a generic pointer: accesses through it use __ldg / st.global (global space).
// kImad: the multiplier is a kernel argument (4), so the address is one
// IMAD.WIDE.U32; otherwise the immediate 4 gives a LEA / LEA.HI.X pair on the
// ALU pipe.  The ELL kernel's FMA-pipe-heavy mix prefers the LEA pair (4.19e11
// vs 4.0e11 spin-updates/s), the CSR kernel the IMAD (2.75e11 vs 2.49e11)
// (profiles/r01/ell_notes.log).
template <bool kImad, typename T>
__device__ __forceinline__ T* elem_addr(T* p, int off, uint32_t elem_bytes) {
  uint64_t a;
  if constexpr (kImad)
    asm("mad.wide.u32 %0, %1, %2, %3;"
        : "=l"(a)
        : "r"((uint32_t)off), "r"(elem_bytes), "l"(reinterpret_cast<uint64_t>(p)));
  else
    asm("mad.wide.u32 %0, %1, 4, %2;"
        : "=l"(a)
        : "r"((uint32_t)off), "l"(reinterpret_cast<uint64_t>(p)));
  return reinterpret_cast<T*>(a);
}

__device__ __forceinline__ void st_global(float* p, float x) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(x) : "memory");
}
__device__ __forceinline__ void st_global_v2(float* p, float x, float y) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(x), "f"(y) : "memory");
}

// The N(0, sigma^2) noise of one warp's 8 spins (group q) x V replicas per
// lane: injected (`a.noise`) or in-kernel Philox.  Independent of the state,
// so the ELL kernel computes it while the group's gathers are in flight.
template <int V>
__device__ __forceinline__ void sparse_noise(const SparseStepArgs& a, int q, int r,
                                             float (&z)[V][8]) {
  const int n = a.n, i_base = 8 * q;
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const int rc = r + c;
    if (a.noise) {
      const bool valid = rc < a.R;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const int i = i_base + qq;
        z[c][qq] = (valid && i < n) ? a.noise[((long long)rc * a.t_f + a.t) * n + i] : 0.f;
      }
    } else {
      const unsigned long long key = __ldg(a.key_base) + (unsigned long long)rc;
      normal8(philox_schedule((uint32_t)key, (uint32_t)(key >> 32)), (uint32_t)q, (uint32_t)a.t,
              bm_scale(a.sigma), z[c]);
    }
  }
}

// Update and stores for group q x V replicas per lane; acc = the row sums.
// The per-spin constants are read once per group (two float4 each; the
// arrays are zero-padded to a multiple of 16 spins).
template <int V, bool kImad>
__device__ __forceinline__ void sparse_update(const SparseStepArgs& a, int q, int r,
                                              float (&acc)[8][V], const float (&sold)[8][V],
                                              const float (&z)[V][8]) {
  const int n = a.n, i_base = 8 * q;
  const int Rp = (int)a.Rp;
  const float inv_t = a.inv_t, alpha = a.alpha, oma = a.oma;
  float* __restrict__ sn = a.s_new + r;
  const float4* iv4 = reinterpret_cast<const float4*>(a.invn + i_base);
  const float4* hv4 = reinterpret_cast<const float4*>(a.hn + i_base);
  const float4 iv0 = __ldg(iv4), iv1 = __ldg(iv4 + 1), hv0 = __ldg(hv4), hv1 = __ldg(hv4 + 1);
  const float invn[8] = {iv0.x, iv0.y, iv0.z, iv0.w, iv1.x, iv1.y, iv1.z, iv1.w};
  const float hn[8] = {hv0.x, hv0.y, hv0.z, hv0.w, hv1.x, hv1.y, hv1.z, hv1.w};
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const int rc = r + c;
    const bool valid = rc < a.R;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
      acc[qq][c] = nmfa_update(acc[qq][c], invn[qq], hn[qq], z[c][qq], inv_t, alpha, oma,
                               sold[qq][c]);
    const bool extra = valid && (a.s_hist != nullptr || a.last);
    if (extra) {
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const int i = i_base + qq;
        if (i >= n) break;
        const float sv = acc[qq][c];
        if (a.s_hist) a.s_hist[((long long)rc * a.t_f + a.t) * n + i] = sv;
        if (a.last) {
          a.cfg[(long long)rc * n + i] = sv < 0.f ? (int8_t)-1 : (int8_t)1;
          if (a.s_out) a.s_out[(long long)rc * n + i] = sv;
        }
      }
    }
  }
  auto store = [&](int qq) {
    const int i = i_base + qq;
    if constexpr (V == 2)
      st_global_v2(elem_addr<kImad>(sn, i * Rp, a.elem_bytes), acc[qq][0], acc[qq][1]);
    else
      st_global(elem_addr<kImad>(sn, i * Rp, a.elem_bytes), acc[qq][0]);
  };
#if NMFA_FULL_GROUP_STORES
  if (i_base + 8 <= n) {  // interior group: no per-spin bounds checks
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) store(qq);
    return;
  }
#endif
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    if (i_base + qq >= n) break;
    store(qq);
  }
}

// V replicas per lane (1 or 2): with V = 2 every state access is one float2,
// halving the per-update address arithmetic and the uniform CSR overhead of
// the V = 1 layout (the CSR path is issue-bound; profiles/r01/korder_ab.log).
// Per replica the arithmetic and summation order are the same for any V.
template <int V, bool k96 = false, int kRL = NMFA_CSR_ROUNDS_LONG>
__global__ void __launch_bounds__(256, V == 2 ? 2 : NMFA_SPARSE_MINB)
    sparse_step_kernel(const SparseStepArgs a) {
  using Vec = typename std::conditional<V == 2, float2, float>::type;
  // grid (replica-group blocks, spin groups): warp w of block x owns replicas
  // [32V (8x + w), +32V) of spin group y, so consecutive blocks read the same
  // state rows (no index division; 32-bit element offsets, n * Rp < 2^31)
  const int lane = threadIdx.x & 31;
  const int rb = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int Rp = (int)a.Rp, n = a.n;
  if (rb * 32 * V >= Rp) return;
  const int q = blockIdx.y;
  const int r = (rb * 32 + lane) * V;  // this lane's first replica
  const float* __restrict__ so = a.s_old + r;
  const int* __restrict__ idx = a.idx;
  const float* __restrict__ wts = a.w;
  auto ld = [&](int off, float* out) {  // V consecutive replicas of one state row
    const Vec x = __ldg(reinterpret_cast<const Vec*>(elem_addr<true>(so, off, a.elem_bytes)));  // global, read-only
    if constexpr (V == 2) {
      out[0] = x.x;
      out[1] = x.y;
    } else {
      out[0] = x;
    }
  };

  // Memory-level parallelism: the group's 9 row pointers come from one
  // cooperative load; then every gather of the 8 spins is issued before the
  // first use (degree <= kFast unrolled, longer rows in a general loop).
  constexpr int kFast = 3;  // unrolled row length (cubic / Moebius ladder); longer rows loop
  constexpr int kRounds = NMFA_CSR_ROUNDS;  // entries per row gathered per round beyond kFast
  // segments beyond the staged size (mean degree > 8); 3 entries per row per round trip
  // measured +10% at degree 10 but cost the staged path 7% (register allocation), so 2
  constexpr int kRoundsLong = V == 2 ? kRL : NMFA_CSR_ROUNDS;  // V = 1 would spill
  const int i_base = 8 * q;
  const int pl = lane <= 8 ? __ldg(a.ptr + min(i_base + lane, n)) : 0;
  int k0[8], deg[8];
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    k0[qq] = __shfl_sync(0xffffffffu, pl, qq);
    deg[qq] = __shfl_sync(0xffffffffu, pl, qq + 1) - k0[qq];
  }
  float sold[8][V];
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    if (i_base + qq < n) {
      ld((i_base + qq) * Rp, sold[qq]);
    } else {
#pragma unroll
      for (int c = 0; c < V; ++c) sold[qq][c] = 0.f;
    }
  }
  float v[8][kFast][V];
  float acc[8][V];
  float z[V][8];
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
        if (u < deg[qq]) {
          ld(off, v[qq][u]);
        } else {
#pragma unroll
          for (int c = 0; c < V; ++c) v[qq][u][c] = 0.f;
        }
      }
    sparse_noise<V>(a, q, r, z);  // overlaps the gathers' latency
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2[V];
#pragma unroll
      for (int c = 0; c < V; ++c) s2[c] = 0.f;
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        const float wv = __shfl_sync(0xffffffffu, w_l, (k0[qq] - K0 + u) & 31);
        if (u < deg[qq])
#pragma unroll
          for (int c = 0; c < V; ++c) s2[c] = fmaf(wv, v[qq][u][c], s2[c]);  // CSR order
      }
#pragma unroll
      for (int c = 0; c < V; ++c) acc[qq][c] = s2[c];
    }
  } else if (seg <= (k96 ? 96 : 64) && !kDisableStaged) {
    // Staged segment (rows longer than kFast, up to 64 entries per group:
    // G-set-class random graphs of mean degree 2-8): every lane holds two
    // entries of the segment, offsets pre-multiplied, loaded with ONE coalesced
    // round trip; each gather then takes its offset and weight by shuffle
    // instead of a dependent global index load (one L2 round trip per round
    // instead of two).  Same entries, same per-row CSR order from +0: bitwise
    // the unstaged path.  Measured (tools/csr_probe.py): +20-25% at mean degree
    // 5, +12% at degree 2.  Not better: staging in shared memory with broadcast
    // loads (= unstaged), 3-4 registers per lane for 96-128 entries (local
    // memory; slower than unstaged).
    const int offA = lane < seg ? __ldg(idx + K0 + lane) * Rp : 0;
    const int offB = lane + 32 < seg ? __ldg(idx + K0 + 32 + lane) * Rp : 0;
    const float wA = lane < seg ? __ldg(wts + K0 + lane) : 0.f;
    const float wB = lane + 32 < seg ? __ldg(wts + K0 + 32 + lane) : 0.f;
    // k96: a third register for segments up to 96 entries (its own kernel, so the
    // nested select does not cost the 64-entry kernel)
    const int offC = k96 && lane + 64 < seg ? __ldg(idx + K0 + 64 + lane) * Rp : 0;
    const float wC = k96 && lane + 64 < seg ? __ldg(wts + K0 + 64 + lane) : 0.f;
    auto off_of = [&](int e) {
      return __shfl_sync(0xffffffffu, e < 32 ? offA : (!k96 || e < 64 ? offB : offC), e & 31);
    };
    auto w_of = [&](int e) {
      return __shfl_sync(0xffffffffu, e < 32 ? wA : (!k96 || e < 64 ? wB : wC), e & 31);
    };
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        const int off = off_of(k0[qq] - K0 + u);  // unconditional: no branch around the shuffle
        if (u < deg[qq]) {
          ld(off, v[qq][u]);
        } else {
#pragma unroll
          for (int c = 0; c < V; ++c) v[qq][u][c] = 0.f;
        }
      }
    sparse_noise<V>(a, q, r, z);  // overlaps the gathers' latency
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2[V];
#pragma unroll
      for (int c = 0; c < V; ++c) s2[c] = 0.f;
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        const float wv = w_of(k0[qq] - K0 + u);
        if (u < deg[qq])
#pragma unroll
          for (int c = 0; c < V; ++c) s2[c] = fmaf(wv, v[qq][u][c], s2[c]);  // CSR order
      }
#pragma unroll
      for (int c = 0; c < V; ++c) acc[qq][c] = s2[c];
    }
    int dmax = 0;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) dmax = max(dmax, deg[qq]);
    for (int u = kFast; u < dmax; u += kRounds) {
      float x[kRounds][8][V], wv[kRounds][8];
#pragma unroll
      for (int j = 0; j < kRounds; ++j)
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          if (u + j < deg[qq]) {  // warp-uniform
            const int e = k0[qq] - K0 + u + j;
            ld(off_of(e), x[j][qq]);
            wv[j][qq] = w_of(e);
          }
        }
#pragma unroll
      for (int j = 0; j < kRounds; ++j)
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          if (u + j < deg[qq])
#pragma unroll
            for (int c = 0; c < V; ++c) acc[qq][c] = fmaf(wv[j][qq], x[j][qq][c], acc[qq][c]);
    }
  } else {
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
#pragma unroll
      for (int u = 0; u < kFast; ++u) {
        if (u < deg[qq]) {
          ld(__ldg(idx + k0[qq] + u) * Rp, v[qq][u]);
        } else {
#pragma unroll
          for (int c = 0; c < V; ++c) v[qq][u][c] = 0.f;
        }
      }
    sparse_noise<V>(a, q, r, z);
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2[V];
#pragma unroll
      for (int c = 0; c < V; ++c) s2[c] = 0.f;
#pragma unroll
      for (int u = 0; u < kFast; ++u)
        if (u < deg[qq]) {
          const float wv = __ldg(wts + k0[qq] + u);  // uniform: L1 broadcast
#pragma unroll
          for (int c = 0; c < V; ++c) s2[c] = fmaf(wv, v[qq][u][c], s2[c]);
        }
#pragma unroll
      for (int c = 0; c < V; ++c) acc[qq][c] = s2[c];
    }
    // entries beyond kFast: round u gathers entry u of all 8 rows at once (8
    // loads in flight instead of one), then adds them in each row's CSR order
    int dmax = 0;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) dmax = max(dmax, deg[qq]);
    for (int u = kFast; u < dmax; u += kRoundsLong) {
      float x[kRoundsLong][8][V], wv[kRoundsLong][8];
#pragma unroll
      for (int j = 0; j < kRoundsLong; ++j)
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          if (u + j < deg[qq]) {
            ld(__ldg(idx + k0[qq] + u + j) * Rp, x[j][qq]);
            wv[j][qq] = __ldg(wts + k0[qq] + u + j);
          }
        }
#pragma unroll
      for (int j = 0; j < kRoundsLong; ++j)
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          if (u + j < deg[qq])
#pragma unroll
            for (int c = 0; c < V; ++c) acc[qq][c] = fmaf(wv[j][qq], x[j][qq][c], acc[qq][c]);
    }
  }
  sparse_update<V, true>(a, q, r, acc, sold, z);
}

// ELL step for graphs of max degree <= K (K = 3: cubic, Moebius ladder; 4:
// toroidal grids).  Same warp tiling, summation order and tail as the CSR
// kernel; the fixed row length removes the row-pointer round trip, and each
// warp walks `groups_per_warp` consecutive spin groups with the next group's
// 8K (index, weight) slots loaded while the current group's gathers are in
// flight, so one memory round trip per group remains on the critical path.
template <int V, int K>
__global__ void __launch_bounds__(256, K == 4 ? NMFA_ELL4_MINB : NMFA_ELL_MINB)
    sparse_ell_kernel(const SparseStepArgs a) {
  using Vec = typename std::conditional<V == 2, float2, float>::type;
  static_assert(8 * K <= 32, "one slot per lane");
  // grid (spin strips, replica slices), strips fastest.  A block's 8 warps
  // cover `slices_per_block` (RS) replica slices of 32V x 8/RS strips of G
  // groups.  Small RS keeps the resident blocks on few replica slices, so the
  // gathered rows (n x 32V x 4 B per slice) stay in L2 (random graphs); larger
  // RS reads wider contiguous row segments (local graphs).  profiles/r01/ell_ab*.log
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Rp = (int)a.Rp, n = a.n;
  const int RS = a.slices_per_block;
  const int slice = blockIdx.y * RS + warp % RS;
  if (slice * 32 * V >= Rp) return;
  const int r = (slice * 32 + lane) * V;
  const float* __restrict__ so = a.s_old + r;
  auto ld = [&](int off, float* out) {
    const Vec x = __ldg(reinterpret_cast<const Vec*>(elem_addr<false>(so, off, a.elem_bytes)));  // global, read-only
    if constexpr (V == 2) {
      out[0] = x.x;
      out[1] = x.y;
    } else {
      out[0] = x;
    }
  };
  const int n_groups = (n + 7) / 8;
  const int q_begin = (blockIdx.x * (8 / RS) + warp / RS) * a.groups_per_warp;
  if (q_begin >= n_groups) return;
  const int q_end = min(q_begin + a.groups_per_warp, n_groups);
  const bool slot = lane < 8 * K;
  auto issue = [&](int q, int off_l, float (&sold)[8][V], float (&v)[8][K][V]) {
    const int i_base = 8 * q;
#if NMFA_ELL_FULL_GROUPS
    if (i_base + 8 <= n) {  // interior group: no per-spin bounds checks
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) ld((i_base + qq) * Rp, sold[qq]);
    } else
#endif
    {
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        if (i_base + qq < n) {
          ld((i_base + qq) * Rp, sold[qq]);
        } else {
#pragma unroll
          for (int c = 0; c < V; ++c) sold[qq][c] = 0.f;
        }
      }
    }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
#pragma unroll
      for (int u = 0; u < K; ++u) ld(__shfl_sync(0xffffffffu, off_l, qq * K + u), v[qq][u]);
  };
  auto sums = [&](float w_l, const float (&v)[8][K][V], float (&acc)[8][V]) {
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      float s2[V];
#pragma unroll
      for (int c = 0; c < V; ++c) s2[c] = 0.f;
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const float wv = __shfl_sync(0xffffffffu, w_l, qq * K + u);
#pragma unroll
        for (int c = 0; c < V; ++c) s2[c] = fmaf(wv, v[qq][u][c], s2[c]);  // CSR order, pads last
      }
#pragma unroll
      for (int c = 0; c < V; ++c) acc[qq][c] = s2[c];
    }
  };
  int nx_idx = slot ? __ldg(a.ell_idx + q_begin * 8 * K + lane) : 0;
  float nx_w = slot ? __ldg(a.ell_w + q_begin * 8 * K + lane) : 0.f;
  for (int q = q_begin; q < q_end; ++q) {
    const int off_l = nx_idx * Rp;
    const float w_l = nx_w;
    if (q + 1 < q_end && slot) {
      nx_idx = __ldg(a.ell_idx + (q + 1) * 8 * K + lane);
      nx_w = __ldg(a.ell_w + (q + 1) * 8 * K + lane);
    }
    float sold[8][V], v[8][K][V], acc[8][V];
    issue(q, off_l, sold, v);
    float z[V][8];
    sparse_noise<V>(a, q, r, z);  // independent of the loads above: overlaps their latency
    sums(w_l, v, acc);
    sparse_update<V, false>(a, q, r, acc, sold, z);
  }
}

// S[i][r] <- s0[r][i] (or 0) for the padded state.
__global__ void sparse_init_kernel(float* s, const float* s0, int n, long long R, long long Rp) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * Rp) return;
  const long long i = e / Rp, r = e - i * Rp;
  s[e] = (s0 && r < R) ? s0[r * n + i] : 0.f;
}

constexpr int kEllSlicesPerBlock = 1;

// NMFA_SPARSE_CSR=1 forces the CSR kernel on ELL-eligible graphs (A/B and tests)
static bool ell_disabled() {
  const char* e = getenv("NMFA_SPARSE_CSR");
  return e && e[0] == '1';
}

// Per-plan launch state.  The t_f step launches of a run differ from run to
// run only in the Philox key base (a device word, written by a one-thread
// kernel), the initial state s0 (init node) and the outputs written at the
// last step (last node).  So the init + t_f steps are built once as a CUDA
// graph and replayed: about 2.7 us less per step than stream launches
// (cubic n = 512: 6.35 -> 3.62 us/step; profiles/r01/ell_notes.log).  Runs
// with injected noise or a trajectory record, runs on a stream that is itself
// being captured, and NMFA_SPARSE_GRAPH=0 launch the same kernels directly.
struct SparseGraph {
  unsigned long long* d_key = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t init_node = nullptr, last_node = nullptr;
  std::string signature;  // kernel variant + launch geometry the graph holds
  const float* s0 = nullptr;
  int8_t* cfg = nullptr;
  float* s_out = nullptr;
};

void sparse_plan_free(nmfa_plan* pl) {
  auto* g = static_cast<SparseGraph*>(pl->sparse);
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  if (g->d_key) cudaFree(g->d_key);
  delete g;
  pl->sparse = nullptr;
}

__global__ void sparse_set_key_kernel(unsigned long long* d, unsigned long long v) { *d = v; }

int launch_sparse_anneal(nmfa_plan* pl, uint64_t key_base, const float* noise,
                         const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                         cudaStream_t st) {
  const nmfa_problem* p = pl->p;
  if ((long long)p->n * pl->Rp >= (1LL << 31) || (p->n + 7) / 8 > 65535) {
    set_error("sparse path: needs n <= 524280 and n x padded replicas < 2^31 per plan");
    return NMFA_ERR_ARG;
  }
  if (!pl->sparse) {
    auto* g = new SparseGraph();
    if (cudaMalloc(&g->d_key, sizeof(unsigned long long)) != cudaSuccess) {
      delete g;
      set_error("out of device memory for the sparse plan");
      return NMFA_ERR_CUDA;
    }
    pl->sparse = g;
  }
  auto* G = static_cast<SparseGraph*>(pl->sparse);
  sparse_set_key_kernel<<<1, 1, 0, st>>>(G->d_key, (unsigned long long)key_base);
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
  a.key_base = G->d_key;
  a.elem_bytes = (uint32_t)sizeof(float);
  a.noise = noise;
  a.cfg = cfg;
  a.s_out = s_out;
  a.s_hist = s_hist;
  // two replicas per lane whenever the padded replica count allows (Rp % 64 == 0)
  const char* v_env = getenv("NMFA_SPARSE_V");  // A/B: "1" forces one replica per lane
  const bool v2 = pl->Rp % 64 == 0 && !(v_env && v_env[0] == '1');
  const dim3 grid((unsigned)((pl->Rp / (v2 ? 64 : 32) + 7) / 8), (unsigned)((p->n + 7) / 8));
  // ELL kernel: G consecutive groups per warp amortise the slot prefetch; G
  // is capped so that the resident blocks (2 per SM) still span few replica
  // slices (the L2-resident working set)
  const int ell_k = ell_disabled() ? 0 : p->ell_k;
  const long long n_groups = (p->n + 7) / 8;
  const long long n_slices = pl->Rp / (v2 ? 64 : 32);
  int sm_count = 148;
  cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, p->device);
  a.ell_idx = p->d_ell_idx;
  a.ell_w = p->d_ell_w;
  a.slices_per_block = kEllSlicesPerBlock;
  if (const char* e = getenv("NMFA_ELL_RS")) a.slices_per_block = atoi(e);
  if (a.slices_per_block != 1 && a.slices_per_block != 2 && a.slices_per_block != 4 &&
      a.slices_per_block != 8)
    a.slices_per_block = kEllSlicesPerBlock;
  const int strips_per_block = 8 / a.slices_per_block;
  a.groups_per_warp = (int)std::max(
      1LL, std::min(8LL, n_groups * a.slices_per_block / (8LL * 2 * sm_count)));
  if (const char* e = getenv("NMFA_ELL_G")) a.groups_per_warp = std::max(1, atoi(e));
  const long long strips = (n_groups + a.groups_per_warp - 1) / a.groups_per_warp;
  const dim3 grid_ell((unsigned)((strips + strips_per_block - 1) / strips_per_block),
                      (unsigned)((n_slices + a.slices_per_block - 1) / a.slices_per_block));
  void* kern;
  dim3 kgrid = grid_ell;
  if (ell_k == 3 && v2)
    kern = (void*)sparse_ell_kernel<2, 3>;
  else if (ell_k == 3)
    kern = (void*)sparse_ell_kernel<1, 3>;
  else if (ell_k == 4 && v2)
    kern = (void*)sparse_ell_kernel<2, 4>;
  else if (ell_k == 4)
    kern = (void*)sparse_ell_kernel<1, 4>;
  else {
    // kernel instance by the graph's segment sizes (capi.cu csr_variant): 64-entry staging;
    // 96-entry staging; 96-entry staging + 3 entries per row per round for longer segments
    static const char* cv_env = getenv("NMFA_CSR_VARIANT");  // A/B override
    const int cv = cv_env ? atoi(cv_env) : p->csr_variant;
    kern = !v2      ? (void*)sparse_step_kernel<1>
           : cv == 2 ? (void*)sparse_step_kernel<2, true, 3>
           : cv == 1 ? (void*)sparse_step_kernel<2, true>
                     : (void*)sparse_step_kernel<2>;
    kgrid = grid;
  }
  const long long tot = (long long)p->n * pl->Rp;
  const dim3 init_grid((unsigned)((tot + 255) / 256));
  int n_i = (int)p->n;
  long long R = pl->R, Rp = pl->Rp;
  float* d_sa = pl->d_sa;
  add_launches(2 + pl->t_f);

  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  const char* g_env = getenv("NMFA_SPARSE_GRAPH");
  const bool direct = noise || s_hist || cap != cudaStreamCaptureStatusNone ||
                      (g_env && g_env[0] == '0');
  if (direct) {
    sparse_init_kernel<<<init_grid, 256, 0, st>>>(d_sa, s0, n_i, R, Rp);
    NMFA_LAUNCH_CHECK();
    float* cur = pl->d_sa;
    float* nxt = pl->d_sb;
    for (int t = 0; t < pl->t_f; ++t) {
      a.t = t;
      a.inv_t = inv_t[t];
      a.last = (t == pl->t_f - 1);
      a.s_old = cur;
      a.s_new = nxt;
      void* args[] = {&a};
      NMFA_CUDA_TRY(cudaLaunchKernel(kern, kgrid, dim3(256), args, 0, st));
      std::swap(cur, nxt);
    }
    return NMFA_OK;
  }

  char sig[256];
  snprintf(sig, sizeof(sig), "%p %u %u %d %d %d", kern, kgrid.x, kgrid.y, a.groups_per_warp,
           a.slices_per_block, pl->t_f);
  if (!G->exec || G->signature != sig) {
    if (G->exec) cudaGraphExecDestroy(G->exec);
    if (G->graph) cudaGraphDestroy(G->graph);
    G->exec = nullptr;
    G->graph = nullptr;
    NMFA_CUDA_TRY(cudaGraphCreate(&G->graph, 0));
    cudaKernelNodeParams kp{};
    void* init_args[] = {&d_sa, (void*)&s0, &n_i, &R, &Rp};
    kp.func = (void*)sparse_init_kernel;
    kp.gridDim = init_grid;
    kp.blockDim = dim3(256);
    kp.kernelParams = init_args;
    NMFA_CUDA_TRY(cudaGraphAddKernelNode(&G->init_node, G->graph, nullptr, 0, &kp));
    cudaGraphNode_t prev_node = G->init_node;
    float* cur = pl->d_sa;
    float* nxt = pl->d_sb;
    for (int t = 0; t < pl->t_f; ++t) {
      a.t = t;
      a.inv_t = inv_t[t];
      a.last = (t == pl->t_f - 1);
      a.s_old = cur;
      a.s_new = nxt;
      void* args[] = {&a};
      kp.func = kern;
      kp.gridDim = kgrid;
      kp.kernelParams = args;
      cudaGraphNode_t node;
      NMFA_CUDA_TRY(cudaGraphAddKernelNode(&node, G->graph, &prev_node, 1, &kp));
      prev_node = node;
      std::swap(cur, nxt);
    }
    G->last_node = prev_node;
    NMFA_CUDA_TRY(cudaGraphInstantiate(&G->exec, G->graph, 0));
    G->signature = sig;
    G->s0 = s0;
    G->cfg = cfg;
    G->s_out = s_out;
  }
  if (G->s0 != s0) {  // re-point the init node
    cudaKernelNodeParams kp{};
    void* init_args[] = {&d_sa, (void*)&s0, &n_i, &R, &Rp};
    kp.func = (void*)sparse_init_kernel;
    kp.gridDim = init_grid;
    kp.blockDim = dim3(256);
    kp.kernelParams = init_args;
    NMFA_CUDA_TRY(cudaGraphExecKernelNodeSetParams(G->exec, G->init_node, &kp));
    G->s0 = s0;
  }
  if (G->cfg != cfg || G->s_out != s_out) {  // re-point the last step's outputs
    a.t = pl->t_f - 1;
    a.inv_t = inv_t[pl->t_f - 1];
    a.last = 1;
    a.s_old = (pl->t_f - 1) % 2 == 0 ? pl->d_sa : pl->d_sb;
    a.s_new = (pl->t_f - 1) % 2 == 0 ? pl->d_sb : pl->d_sa;
    void* args[] = {&a};
    cudaKernelNodeParams kp{};
    kp.func = kern;
    kp.gridDim = kgrid;
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    NMFA_CUDA_TRY(cudaGraphExecKernelNodeSetParams(G->exec, G->last_node, &kp));
    G->cfg = cfg;
    G->s_out = s_out;
  }
  NMFA_CUDA_TRY(cudaGraphLaunch(G->exec, st));
  return NMFA_OK;
}

}  // namespace nmfa
