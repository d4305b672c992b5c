// Persistent small-N NMFA kernel (n <= 256, any density): the whole anneal in
// one launch.  One CTA owns 128 replicas for all t_f steps:
//   J (B operand, fp16, K-major)      -> SMEM, loaded once
//   S (A operand, fp16, K-major)      -> SMEM, rewritten by the epilogue
//   Phi accumulator  D = S J^T        -> TMEM columns [0, np)
//   fp32 master S                     -> TMEM columns [np, 2np)
// Per step: one thread issues np/16 tcgen05.mma (M=128, N=np, K=16), commits
// to an mbarrier; every warp then drains its TMEM lane quarter, applies the
// fused update (reference _kernels_numba.py:71-75) and writes the new fp16
// operand back into SMEM.  No HBM traffic inside the anneal.
// HILO field (NMFA_FIELD_HILO): the operand is hi = fp16(s) plus a second SMEM
// image lo = fp16(s - hi), and every K step issues one MMA per part into the
// same accumulator, so the field sees ~22 bits of the fp32 master (np <= 224:
// J + two operand images fit in SMEM).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace nmfa {

// One instance of a grouped launch (nmfa_anneal_many): every instance has the
// same padded size np and replica count R; blockIdx.y selects the instance.
struct SmallInstance {
  const uint4* j_img;
  const float* invn;
  const float* hn;
  unsigned long long key_base;
  int8_t* cfg;  // [R][n]
};

struct SmallArgs {
  const SmallInstance* inst;  // grouped launch table, or null (single problem below)
  const uint4* j_img;
  uint32_t j_bytes;
  const float* invn;
  const float* hn;
  const float* inv_temp;
  int n, np, t_f;
  uint32_t tmem_cols;
  float alpha, oma, sigma;
  unsigned long long key_base;
  long long R;
  const float* noise;  // [R][t_f][n] or null
  const float* s0;     // [R][n] or null
  int8_t* cfg;         // [R][n]
  float* s_out;        // [R][n] or null
  float* s_hist;       // [R][t_f][n] or null
  int cs;              // warps per TMEM lane quarter (column split)
  int hilo;            // HILO field: second operand image (lo), two MMAs per K step
};

constexpr uint32_t kRowsPerCta = 128;
constexpr uint32_t kLboA = (kRowsPerCta / 8) * 128;  // A: K core matrices 2048 B apart

#ifndef NMFA_SMALL_MINB
#define NMFA_SMALL_MINB 1  // blocks per SM the register budget targets (A/B knob)
#endif

// 16 spins of replica row rl into the operand image (fp16 hi) and, for the
// HILO field, the residual image (fp16 lo = s - hi)
__device__ __forceinline__ void store_operand(uint8_t* sA, uint8_t* sL, int hilo, int rl, int c0,
                                              const float v[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint4 hv, lv;
    if (hilo) {
      split_hilo8<true>(v + 8 * h, hv, lv, false);
      *reinterpret_cast<uint4*>(sL + kmajor_off(rl, c0 + 8 * h, kLboA)) = lv;
    } else {
      hv = make_uint4(pack_half2(v[8 * h + 0], v[8 * h + 1]), pack_half2(v[8 * h + 2], v[8 * h + 3]),
                      pack_half2(v[8 * h + 4], v[8 * h + 5]), pack_half2(v[8 * h + 6], v[8 * h + 7]));
    }
    *reinterpret_cast<uint4*>(sA + kmajor_off(rl, c0 + 8 * h, kLboA)) = hv;
  }
}

// kTab: the Box-Muller (sin, cos) of the 4096 noise angles come from a 32 KB
// shared-memory table built at launch with the same MUFU instructions (bitwise
// the same normals, two XU operations fewer per pair); used when it fits.
template <bool kInjected, bool kTab>
__global__ void __launch_bounds__(512, NMFA_SMALL_MINB) small_anneal_kernel(const SmallArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int np = a.np;
  uint8_t* sJ = smem;
  uint8_t* sA = smem + (size_t)np * np * 2;
  uint8_t* sL = sA + (size_t)kRowsPerCta * np * 2;  // HILO: lo image (else zero bytes)
  float2* sTab = reinterpret_cast<float2*>(sL + (a.hilo ? (size_t)kRowsPerCta * np * 2 : 0));
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sTab) + (kTab ? 4096 * 8 : 0));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, cpart = warp >> 2;
  const int rl = 32 * quarter + lane;
  const long long rrel = (long long)blockIdx.x * kRowsPerCta + rl;
  const bool valid = rrel < a.R;
  const int nchunks = np / 16;
  const SmallInstance* I = a.inst ? a.inst + blockIdx.y : nullptr;
  const uint4* j_img = I ? I->j_img : a.j_img;
  const float* invn = I ? I->invn : a.invn;
  const float* hn = I ? I->hn : a.hn;
  int8_t* cfg = I ? I->cfg : a.cfg;

  for (uint32_t i = tid; i < a.j_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sJ)[i] = j_img[i];
  if (kTab) sincos_table_fill(sTab, tid, blockDim.x);  // visible after the __syncthreads below
  if (warp == 0) tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t t_acc = tbase + ((uint32_t)(32 * quarter) << 16);
  const uint32_t t_mst = t_acc + (uint32_t)np;

  const unsigned long long key = (I ? I->key_base : a.key_base) + (unsigned long long)rrel;
  const PhiloxKey K = philox_schedule((uint32_t)key, (uint32_t)(key >> 32));

  // initial state: s0 or zeros, into the TMEM master and the SMEM operand
  for (int j = cpart; j < nchunks; j += a.cs) {
    const int c0 = 16 * j;
    float v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      int i = c0 + c;
      v[c] = (a.s0 && valid && i < a.n) ? a.s0[rrel * a.n + i] : 0.f;
    }
    tmem_st16(t_mst + c0, v);
    store_operand(sA, sL, a.hilo, rl, c0, v);
  }
  tmem_wait_st();
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();

  const uint32_t idesc = make_idesc_f16(kRowsPerCta, (uint32_t)np);
  const uint32_t a_addr = smem_u32(sA), l_addr = smem_u32(sL), b_addr = smem_u32(sJ);
  const uint32_t lboB = (uint32_t)np * 16u;

  for (int t = 0; t < a.t_f; ++t) {
    if (tid == 0) {
      tc_fence_after();
      for (int ks = 0; ks < nchunks; ++ks) {
        uint64_t ad = make_desc_noswizzle(a_addr + ks * 2 * kLboA, kLboA, 128);
        uint64_t bd = make_desc_noswizzle(b_addr + ks * 2 * lboB, lboB, 128);
        mma_f16_ss(tbase, ad, bd, idesc, ks > 0 ? 1u : 0u);
        if (a.hilo)
          mma_f16_ss(tbase, make_desc_noswizzle(l_addr + ks * 2 * kLboA, kLboA, 128), bd, idesc, 1u);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, (uint32_t)(t & 1));
    tc_fence_after();
    const float inv_t = a.inv_temp[t];
    const bool last = (t == a.t_f - 1);

    const float4* invn4 = reinterpret_cast<const float4*>(invn);
    const float4* hn4 = reinterpret_cast<const float4*>(hn);
    const bool extra = (a.s_hist != nullptr) || last;
    for (int j = cpart; j < nchunks; j += a.cs) {
      const int c0 = 16 * j;
      float acc[16], ms[16];
      tmem_ld16(t_acc + c0, acc);
      tmem_ld16(t_mst + c0, ms);
      tmem_wait_ld();
      const int nvalid = valid ? min(16, a.n - c0) : 0;
      const float* nz = kInjected ? a.noise + ((long long)rrel * a.t_f + t) * a.n + c0 : nullptr;
      if (a.n - c0 <= 8)  // the padded tail chunk: columns >= n only meet zero J columns
        update_chunk<kInjected, 8, kTab>(acc, ms, invn4 + c0 / 4, hn4 + c0 / 4, nz, nvalid, K,
                                         (uint32_t)(c0 / 8), (uint32_t)t, a.sigma, inv_t, a.alpha,
                                         a.oma, sTab);
      else
        update16<kInjected, kTab>(acc, ms, invn4 + c0 / 4, hn4 + c0 / 4, nz, nvalid, K,
                                  (uint32_t)(c0 / 8), (uint32_t)t, a.sigma, inv_t, a.alpha, a.oma,
                                  sTab);
      tmem_st16(t_mst + c0, ms);
      store_operand(sA, sL, a.hilo, rl, c0, ms);
      if (extra && nvalid > 0) {
        if (a.s_hist) {
          float* hrow = a.s_hist + ((long long)rrel * a.t_f + t) * a.n + c0;
          #pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < nvalid) hrow[c] = ms[c];
        }
        if (last) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c < nvalid) {
              cfg[rrel * a.n + c0 + c] = ms[c] < 0.f ? (int8_t)-1 : (int8_t)1;  // problem.py:181-183
              if (a.s_out) a.s_out[rrel * a.n + c0 + c] = ms[c];
            }
          }
        }
      }
    }
    NMFA_JITTER(threadIdx.x + 977 * blockIdx.x, t);  // checked build only
    tmem_wait_st();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, a.tmem_cols);
  }
}

constexpr size_t kTabBytes = 4096 * sizeof(float2);
// the sincos table is used when it fits beside J and the operand image(s), at
// two CTAs per SM while the image alone allowed two (NMFA_SMALL_TABLE=0: never)
static bool small_table_fits(size_t smem, int device) {
  static const char* env = getenv("NMFA_SMALL_TABLE");
  if (env && env[0] == '0') return false;
  int sm_bytes = 228 * 1024, cta_bytes = 227 * 1024;
  cudaDeviceGetAttribute(&sm_bytes, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&cta_bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const size_t per_sm = (size_t)sm_bytes, per_cta = (size_t)cta_bytes;
  const int ctas_before = (int)std::min<size_t>(2, per_sm / (smem + 1024));
  const int ctas_after = (int)std::min<size_t>(2, per_sm / (smem + kTabBytes + 1024));
  return smem + kTabBytes <= per_cta && ctas_after >= ctas_before;
}

static uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

int launch_small_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                        const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                        cudaStream_t st) {
  const nmfa_problem* p = pl->p;
  SmallArgs a{};
  a.j_img = reinterpret_cast<const uint4*>(p->d_j_small);
  a.j_bytes = (uint32_t)p->np * p->np * 2;
  a.invn = p->d_invn;
  a.hn = p->d_hn;
  a.inv_temp = pl->d_inv_temp;
  a.n = (int)p->n;
  a.np = p->np;
  a.t_f = pl->t_f;
  a.tmem_cols = pow2_cols(2u * p->np);
  a.alpha = pl->alpha;
  a.oma = pl->oma;
  a.sigma = pl->sigma;
  a.key_base = key_base;
  a.R = pl->R;
  a.noise = noise;
  a.s0 = s0;
  a.cfg = cfg;
  a.s_out = s_out;
  a.s_hist = s_hist;
  a.hilo = pl->field == NMFA_FIELD_HILO ? 1 : 0;
  const long long ctas = (pl->R + kRowsPerCta - 1) / kRowsPerCta;
  // Spread columns over more warps when the grid cannot fill the GPU.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  a.cs = ctas >= sms ? 2 : 4;
  if (const char* e = getenv("NMFA_SMALL_CS")) a.cs = atoi(e);  // tuning override
  if (a.cs > p->np / 16) a.cs = p->np / 16;
  size_t smem = (size_t)p->np * p->np * 2 + (size_t)kRowsPerCta * p->np * 2 * (1 + a.hilo) + 16;
  const bool tab = !noise && small_table_fits(smem, p->device);
  if (tab) smem += kTabBytes;
  auto kern = noise ? small_anneal_kernel<true, false>
                    : (tab ? small_anneal_kernel<false, true> : small_anneal_kernel<false, false>);
  NMFA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)ctas, 128 * a.cs, smem, st>>>(a);
  NMFA_LAUNCH_CHECK();
  add_launches(1);
  return NMFA_OK;
}

// Grouped launch: `count` small problems of the same padded size, R replicas
// each, in ONE persistent launch (grid = CTAs per instance x count), so many
// small instances fill the GPU (Fig. 4-style sweeps, cli.py:280-347).
int launch_small_anneal_many(const nmfa_problem* const* ps, int count, int64_t R, int t_f,
                             const float* d_inv_temp, float alpha, float sigma,
                             const uint64_t* key_bases, int8_t* cfg, cudaStream_t st) {
  const nmfa_problem* p0 = ps[0];
  std::vector<SmallInstance> h(count);
  for (int k = 0; k < count; ++k) {
    h[k].j_img = reinterpret_cast<const uint4*>(ps[k]->d_j_small);
    h[k].invn = ps[k]->d_invn;
    h[k].hn = ps[k]->d_hn;
    h[k].key_base = key_bases[k];
    h[k].cfg = cfg + (size_t)k * R * p0->n;
  }
  SmallInstance* d_inst = nullptr;
  NMFA_CUDA_TRY(cudaMallocAsync(&d_inst, sizeof(SmallInstance) * count, st));
  NMFA_CUDA_TRY(cudaMemcpyAsync(d_inst, h.data(), sizeof(SmallInstance) * count,
                                cudaMemcpyHostToDevice, st));
  SmallArgs a{};
  a.inst = d_inst;
  a.j_bytes = (uint32_t)p0->np * p0->np * 2;
  a.inv_temp = d_inv_temp;
  a.n = (int)p0->n;
  a.np = p0->np;
  a.t_f = t_f;
  a.tmem_cols = pow2_cols(2u * p0->np);
  a.alpha = alpha;
  a.oma = 1.0f - alpha;
  a.sigma = sigma;
  a.R = R;
  a.hilo = 1;  // the HILO field when every instance asks for it
  for (int k = 0; k < count; ++k) a.hilo &= ps[k]->field == NMFA_FIELD_HILO ? 1 : 0;
  const long long ctas = (R + kRowsPerCta - 1) / kRowsPerCta;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p0->device);
  a.cs = ctas * count >= sms ? 2 : 4;
  if (a.cs > p0->np / 16) a.cs = p0->np / 16;
  size_t smem = (size_t)p0->np * p0->np * 2 + (size_t)kRowsPerCta * p0->np * 2 * (1 + a.hilo) + 16;
  const bool tab = small_table_fits(smem, p0->device);
  if (tab) smem += kTabBytes;
  auto kern = tab ? small_anneal_kernel<false, true> : small_anneal_kernel<false, false>;
  NMFA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3((unsigned)ctas, (unsigned)count), 128 * a.cs, smem, st>>>(a);
  NMFA_LAUNCH_CHECK();
  add_launches(1);
  NMFA_CUDA_TRY(cudaFreeAsync(d_inst, st));
  return NMFA_OK;
}

}  // namespace nmfa
