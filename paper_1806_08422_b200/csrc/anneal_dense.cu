// Dense large-N NMFA step: a 2-CTA (cta_group::2) tcgen05 GEMM with the NMFA
// update fused into its epilogue.  Reference: _kernels_numba.py:71-75
// (mv = J s; phi = (h + mv)/norm + noise; s = a*(-tanh(phi/T)) + (1-a)*s),
// batched over replicas.
//
// GEMM orientation: D[r, i] = sum_k S[r, k] J[i, k]
//   M = replicas (256 per CTA pair, 128 per CTA), N = spins (tile of <= 256),
//   K = spins.  A = S (fp16, K-major), B = J (fp16, K-major; J symmetric).
// Operand images in HBM are pre-tiled so a (128 rows x 128 k) tile is 32 KB of
// contiguous bytes in the UMMA canonical no-swizzle K-major layout:
//   byte(row, k) = (k/128)*Rows*256 + (row/8)*2048 + ((k%128)/8)*128 + (row%8)*16 + (k%8)*2
// (measured: the per-SM TMA engine costs ~100 cycles per box + ~11 cycles/KB,
// so operands move in one 32 KB box each per stage; see profiles/).
// TMA moves them as a 2-D tensor of 128-byte lines.  The epilogue writes the
// next step's A image directly in that layout (two 16-B stores per 16
// spins, a warp covers four full 128-B lines), so no transpose pass exists.
//
// Roles per CTA (640 threads): warps 0-15 epilogue (lane quarter x column
// part; 4 warps per scheduler to hide the Philox/MUFU latency chains),
// warp 16 TMA producer, warp 17 MMA issuer (leader CTA only), warp 18 TMEM
// allocator and then readiness prefetcher (polls the readiness counters of the
// producer's upcoming tiles and posts them to a shared-memory mailbox, so a
// switch to a new replica block does not stall the TMA ring on L2 polls and
// fences).  The control roles take the HIGHEST warp ids on purpose: the
// warp scheduler favours high ids, and with low ids the producer and MMA
// issuer starved behind the epilogue warps (measured: 3x longer k-block
// intervals, see profiles/).  3-stage smem ring (A: one 32 KB box; B: one box
// of exactly the tile half, <= 32 KB), 2 TMEM accumulator slots of 256
// columns so the epilogue of tile j overlaps the MMAs of tile j+1.
//
// Field precision (NMFA_FIELD_*): FP16 multiplies the hi part of the state
// (one MMA per k-slice).  HILO multiplies hi and then lo for every k-slice into
// the same fp32 accumulator (two ring stages per k-slice, B loaded for each),
// so the field sees the full ~22-bit state; lo then ping-pongs between two
// images like hi, because other tiles' GEMMs read it while its owner rewrites
// it.  The energy pass multiplies the +-1 configuration (hi) alone.
//
// Persistence: one cooperative launch runs every sweep of the anneal (plus the
// exact energy pass).  Each pair owns 3-4 (replica block, spin range) tiles
// per sweep in a skewed order: the replica blocks are split into an early and
// a late class, every pair runs its early-class tiles first, so the tiles
// that start a sweep consume blocks finished a tile-time before the boundary
// (profiles/r02/dense_schedule.log; widths from a cost model of the MMA and
// TMA time per k-slice).  Instead of a kernel boundary between
// sweeps, every warp publishes the k-slices it wrote in per-(replica block,
// k-slice) readiness counters, and producers wait only for the slices they
// are about to load; the K order is natural so results do not depend on the
// schedule, the replica count or the row sharding.
//
// Experiment switches (measurements in profiles/r01/ and profiles/r02/, none
// changes results unless noted):
//   env NMFA_TILE_ORDER = skew (default) | mmajor | sorted | spin | block | alt | rev
//   env NMFA_KORDER = rotate | rotm | rotmn  (rotated K orders; timing only)
//   env NMFA_SLICE_PAD = lines  (pad between image k-slices; layout only)
//   env NMFA_KORDER = early    (earliest-published-slice-first K order; results
//                               then depend on the schedule)
//   env NMFA_TILE_W = 1..16    (force the tile width in 16-spin units)
//   env NMFA_TRACE / NMFA_TRACE2 / NMFA_TRACE3 = <file>  (clock64/globaltimer traces)
//   -DNMFA_DBG_NOEPI / NOMEM / NOLOAD / NOLO / NOMATH / NOTMEM / NOMUFU / SPREAD /
//    PLAINMEM / LOKEEP  (epilogue ablations for timing; results are wrong)
//   -DNMFA_EPI_PREFETCH, -DNMFA_EPI_WARPS=n, -DNMFA_DSTAGES=n, -DNMFA_DMAXW=n,
//   -DNMFA_ROLES_FIRST, -DNMFA_EPI_SPIN / NMFA_EPI_BACKOFF=ns, -DNMFA_EPI_FENCE_FIRST,
//   -DNMFA_EPI_NOALLOC, -DNMFA_EPI_STCS, -DNMFA_L2_PREFETCH=k
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstdlib>
#include <numeric>

#include "common.cuh"
#include "internal.h"

namespace nmfa {

#ifndef NMFA_DSTAGES
#define NMFA_DSTAGES 3
#endif
#ifndef NMFA_PF_SLEEP_NS
#define NMFA_PF_SLEEP_NS 20  // producer's back-off while its next slice is not yet known ready
#endif
#ifndef NMFA_POLL_SLEEP_NS
#define NMFA_POLL_SLEEP_NS 32  // prefetch thread's back-off between readiness polls
#endif
constexpr int kDStages = NMFA_DSTAGES;
constexpr int kBK = 128;  // K per pipeline stage: one 32 KB TMA box per operand
#ifndef NMFA_EPI_WARPS
#define NMFA_EPI_WARPS 16
#endif
constexpr int kDEpiWarps = NMFA_EPI_WARPS;
constexpr int kParts = kDEpiWarps / 4;  // column parts per TMEM lane quarter
constexpr int kDThreads = 32 * kDEpiWarps + 128;
// Warp roles: epilogue warps first, control warps on the highest ids (the
// scheduler favours high ids; see the header).  Warp w reads TMEM lane quarter
// w % 4.  NMFA_ROLES_FIRST (experiment) puts producer/MMA/alloc on warps 0-2.
#ifdef NMFA_ROLES_FIRST
constexpr int kEpiBase = 4;
constexpr int kWarpProducer = 0, kWarpMma = 1, kWarpAlloc = 2;
#else
constexpr int kEpiBase = 0;
constexpr int kWarpProducer = kDEpiWarps, kWarpMma = kDEpiWarps + 1, kWarpAlloc = kDEpiWarps + 2;
#endif
constexpr uint32_t kATile = 128 * kBK * 2;     // 128 rows x 128 k fp16 = 32 KB
#ifndef NMFA_DMAXW
#define NMFA_DMAXW 16  // widest tile in 16-spin units (experiment: 12 makes room for a 4th stage)
#endif
constexpr int kMaxW = NMFA_DMAXW;
constexpr uint32_t kBTileMax = 8 * kMaxW * kBK * 2;  // <= 8 * kMaxW rows (N/2) x 128 k
constexpr uint32_t kDStageBytes = kATile + kBTileMax;
constexpr uint32_t kAccCols = 256;
// Box-Muller (sin, cos) table of the 4096 noise angles after the ring (common.cuh
// sincos_table_fill: bitwise the inline MUFU values), when it fits
constexpr size_t kDRingBytes = (size_t)kDStages * kDStageBytes;
#ifndef NMFA_DENSE_TABLE
#define NMFA_DENSE_TABLE 0  // measured neutral at K2000, -8% at small N (the 32 KB it takes from L1)
#endif
constexpr bool kDTab = NMFA_DENSE_TABLE && kDRingBytes + 4096 * 8 + 2048 <= 227 * 1024;
constexpr size_t kDSmemBytes = kDRingBytes + 1024;  // the table is static shared memory

struct DenseTile {
  int m_blk, n0, nlen, pad;
};

constexpr int kMaxPeers = 7;  // other shards of a fused-exchange plan (8 GPUs)

struct DenseState {
  int np = 0, kp = 0, kblocks = 0, k_last_sub = 0, pairs = 0;
  int slice_lo = 0, slice_hi = 0;  // k-slices of the image this device writes
  long long Rp = 0;
  long long slice_b = 0;           // bytes per k-slice of an operand image (Rp * 256 + pad)
  uint8_t* lo_img = nullptr;
  uint8_t* lo_img2 = nullptr;      // HILO field: second lo image (lo ping-pongs like hi)
  bool hilo = false;               // NMFA_FIELD_HILO: hi and lo both enter the GEMM
  uint8_t* a_img[2] = {nullptr, nullptr};
  DenseTile* d_tiles = nullptr;
  int* d_tile_off = nullptr;
  unsigned* d_kneed = nullptr;    // per (block, k-slice): spins published per sweep (x2 CTAs)
  unsigned* d_ready = nullptr;    // per (block, k-slice): spins published this launch
  int n_mblk = 0;
  int n_tiles = 0;
  std::vector<int> grp_off_base;  // per replica group: start of its tile offsets in d_tile_off
  std::vector<int> grp_pairs;     // per replica group: CTA pairs of its launch
  int16_t* d_korder = nullptr;     // [tile][kblocks] K order (null: natural)
  CUtensorMap tmA[2];
  CUtensorMap tmL[2];  // lo images as A operands (HILO field; copies of tmA otherwise)
  CUtensorMap tmB[2];  // B boxes of exactly one tile half (2 x rows lines), the two widths
  int bhalf[2] = {0, 0};
  uint32_t stage_bytes = kDStageBytes;  // sized for the plan's tile widths (leaves L1 the rest)
  // fused exchange (row-sharded J): the operand images are peer-accessible
  // buffers owned by the caller, and the epilogue also stores every new hi
  // line into the other shards' images at the same offset
  bool external_images = false;
  int n_peers = 0;
  uint8_t* peer_img[2][kMaxPeers] = {};
};

struct DenseStepArgs {
  const DenseTile* tiles;
  const int* tile_off;
  const unsigned* kneed;   // [m][kblocks] spins a sweep publishes into the slice (both CTAs)
  unsigned* ready;         // [m][kblocks] spins published so far this launch
  int kblocks, k_last_sub;
  int n, brows, row_lo;    // B image rows (row shard of J) and the shard's first spin
  long long R, Rp;
  long long slice_b;       // bytes per k-slice of an image (a multiple of 128)
  int t_begin, t_end, t_f;  // sweeps [t_begin, t_end) of t_f; energy pass after t_f-1
  int energy_pass;
  float alpha, oma, sigma;
  const float* inv_temp;
  const float* invn;
  const float* hn;
  uint8_t* img0;           // operand images (hi part of the state), ping-pong by parity
  uint8_t* img1;
  uint8_t* lo;             // residual image, same layout (HILO: lo of even sweeps)
  uint8_t* lo1;            // HILO: lo of odd sweeps (the GEMM reads lo, so it ping-pongs)
  int hilo;                // HILO field: A = hi then lo per k-slice, one fp32 accumulator
  uint32_t stage_bytes;    // ring stage: A box + this plan's widest B half (multiple of 1 KB)
  unsigned long long key_base;
  const float* noise;
  int8_t* cfg;
  float* s_out;
  float* s_hist;
  double* energy;          // energy pass: E[r] accumulator (zeroed)
  const double* h;         // raw fields (energy pass)
  double half_scale;       // 0.5 * j_scale (energy pass)
  unsigned long long* trace;  // debug timeline (NMFA_TRACE), CTA 0 only
  unsigned long long* tl2;    // debug: globaltimer per (pair, tile) (NMFA_TRACE2)
  const int16_t* korder;      // [tile][kblocks] K order, or null for natural order
  int bhalf0, bhalf1;         // rows per CTA of the two tile widths (B box sizes)
  int n_peers;                // fused exchange: other shards' images (same layout)
  uint8_t* peer0[kMaxPeers];
  uint8_t* peer1[kMaxPeers];
  unsigned long long* tl3;    // debug: per k-slice clock64 of CTA 0 (NMFA_TRACE3)
};

// ---------------------------------------------------------------------------
// cluster / 2-CTA PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* tm, int c0, int c1,
                                           uint32_t mbar_cluster, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(mbar_cluster), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive(uint32_t mbar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mbar_cluster)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// 2-CTA MMA from descriptor words: the high word (SBO, version) is constant and
// the low word is (LBO << 16) | (smem address >> 4), so stepping K by 16 is one
// add (keeps the single issuing thread lean while 16 epilogue warps compete).
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo,
                                         uint32_t desc_hi, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "mov.b64 da, {%1, %3};\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %4, p;\n\t}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(desc_hi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_pair_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_release_gpu() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive_relaxed(uint32_t mbar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mbar_cluster)
               : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// L2 residency: operand images and J are re-read by every pair of a replica
// block (TMA, evict_last); the lo residual is touched once per sweep per element
// (evict_first) so it does not push the operands out of L2.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
#ifdef NMFA_DBG_PLAINMEM  // experiment: no L2 cache-policy hints on state loads/stores
__device__ __forceinline__ uint4 ld_hint(const void* ptr, uint64_t) {
  return *reinterpret_cast<const uint4*>(ptr);
}
__device__ __forceinline__ void st_hint(void* ptr, uint4 v, uint64_t) {
  *reinterpret_cast<uint4*>(ptr) = v;
}
#else
__device__ __forceinline__ uint4 ld_hint(const void* ptr, uint64_t pol) {
  uint4 v;
#ifdef NMFA_EPI_NOALLOC  // experiment: state loads do not allocate in L1 (the SMEM/L1 SRAM)
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
#else
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
#endif
  return v;
}
__device__ __forceinline__ void st_hint(void* ptr, uint4 v, uint64_t pol) {
#ifdef NMFA_EPI_STCS  // experiment: streaming (.cs) stores, no L2 policy
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
#else
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
#endif
}
#endif

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// readiness mailbox between the prefetch thread and the TMA producer of a CTA
__device__ __forceinline__ unsigned long long ld_acquire_cta_smem(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_smem(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}

// Persistent multi-sweep kernel.  Every pair walks its static tile list once
// per sweep t in [t_begin, t_end) and then (energy_pass) once more in energy
// mode: the A operand is then the +-1 configuration written by the last sweep
// and the epilogue reduces E_r = 1/2 c_r.(J c_r) + h.c_r exactly (integer J,
// |J c| < 2^24).  Sweep t+1 of replica block m may start once every (CTA, tile)
// epilogue of block m for sweep t has published its rows, tracked per
// 128-spin k-slice (`ready[m][kb]`, counted in spins): the next sweep's MMAs
// start on the slices that finished first (a static, deterministic order per
// block, so results do not depend on timing) while the previous sweep's last
// epilogues are still running.  Replica blocks are independent.
template <bool kInjected>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kDThreads, 1)
    dense_anneal_kernel(const __grid_constant__ CUtensorMap tmA0,
                        const __grid_constant__ CUtensorMap tmA1,
                        const __grid_constant__ CUtensorMap tmB0,
                        const __grid_constant__ CUtensorMap tmB1,
                        const __grid_constant__ CUtensorMap tmL0,
                        const __grid_constant__ CUtensorMap tmL1, const DenseStepArgs a) {
  extern __shared__ __align__(1024) uint8_t dsmem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[kDStages], empty_bar[kDStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_slot;
  // readiness mailbox: (tile step << 16) | k-order slices of that step known ready
  __shared__ __align__(8) unsigned long long pf_ready;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_rank();
  const int pair = blockIdx.x >> 1;
  const int j0 = a.tile_off[pair], j1 = a.tile_off[pair + 1];
  const int n_phases = (a.t_end - a.t_begin) + (a.energy_pass ? 1 : 0);

  if (warp == kWarpProducer && lane == 0) {
    const CUtensorMap* maps[6] = {&tmA0, &tmA1, &tmB0, &tmB1, &tmL0, &tmL1};
#pragma unroll
    for (int m = 0; m < (a.hilo ? 6 : 4); ++m)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(maps[m])) : "memory");
    for (int s = 0; s < kDStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * kDEpiWarps);
    }
    fence_mbar_init();
    pf_ready = 0;
  }
  // static, so its address is an immediate (no register in the 96-register epilogue)
  __shared__ float2 sTab[kDTab ? 4096 : 1];
  if (kDTab) sincos_table_fill(sTab, threadIdx.x, blockDim.x);
  if (warp == kWarpAlloc) tmem_alloc_pair(&tmem_slot, 2 * kAccCols);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;

  if (warp == kWarpProducer) {
    // ------------------------- TMA producer -------------------------
    if (lane == 0) {
      int it = 0;
      unsigned long long seen = 0;  // last pf_ready value observed
      const uint64_t pol_keep = policy_evict_last();
      for (int ph = 0; ph < n_phases; ++ph) {
        const int t = a.t_begin + ph;
        const CUtensorMap* tmA = (t & 1) ? &tmA1 : &tmA0;
        const CUtensorMap* tmL = (t & 1) ? &tmL1 : &tmL0;
        // HILO field: every k-slice is two stages, A = hi then A = lo (same B);
        // the energy pass multiplies the +-1 configuration (hi) only
        const int subs = (a.hilo && t < a.t_end) ? 2 : 1;
        for (int j = j0; j < j1; ++j) {
          const DenseTile tl = a.tiles[j];
          const int half = tl.nlen >> 1;
          const int arow = tl.m_blk * 256 + (int)cta * 128;
          const int brow = tl.n0 - a.row_lo + (int)cta * half;  // row within this shard of J
          const int jglob = ph * (j1 - j0) + (j - j0);
          const int16_t* kord = a.korder ? a.korder + (size_t)j * a.kblocks : nullptr;
          if (a.trace && blockIdx.x == 0 && jglob < 512) a.trace[jglob * 8 + 0] = clock64();
          unsigned long long* t2 = (a.tl2 && cta == 0 && jglob < 64) ? a.tl2 + ((blockIdx.x >> 1) * 64 + jglob) * 8 : nullptr;
          if (t2) t2[0] = gtimer();
          long long wempty = 0;
          const unsigned long long step = (unsigned long long)jglob << 16;
          for (int ki = 0; ki < a.kblocks; ++ki) {
            const int kb = kord ? kord[ki] : ki;
            if (seen < step + (unsigned long long)(ki + 1)) {
              // the slices of block m for sweep t were written by sweep t-1: the
              // prefetch thread (alloc warp) polls the readiness counters ahead of
              // this thread and posts progress in pf_ready, so a block switch costs
              // one shared-memory load instead of a round of L2 polls and fences
              do {
                seen = ld_acquire_cta_smem(&pf_ready);
                if (seen < step + (unsigned long long)(ki + 1)) __nanosleep(NMFA_PF_SLEEP_NS);
              } while (seen < step + (unsigned long long)(ki + 1));
              fence_proxy_async_global();
            }
            if (ki == a.kblocks - 1 && a.trace && blockIdx.x == 0 && jglob < 512)
              a.trace[jglob * 8 + 1] = clock64();  // producer reached the last slice
            if (t2 && ki == 0) t2[5] = gtimer();
            if (t2 && ki == a.kblocks - 1) t2[1] = gtimer();
            for (int sub = 0; sub < subs; ++sub, ++it) {
              const int s = it % kDStages;
              NMFA_JITTER(blockIdx.x, it);  // checked build only
              if (a.trace) {
                const long long c0 = clock64();
                mbar_wait(&empty_bar[s], ((it / kDStages) & 1) ^ 1);
                wempty += clock64() - c0;
              } else {
                mbar_wait(&empty_bar[s], ((it / kDStages) & 1) ^ 1);
              }
              if (a.tl3 && blockIdx.x == 0 && it >= 256 && it < 320) a.tl3[(it - 256) * 4 + 0] = clock64();
              const uint32_t fb = map_to_rank(smem_u32(&full_bar[s]), 0);
              if (cta == 0)
#ifdef NMFA_DBG_NOB  // timing bound only: no J bytes through TMA (results are wrong)
                mbar_arrive_expect_tx(&full_bar[s], 2u * kATile);
#else
                mbar_arrive_expect_tx(&full_bar[s], 2u * (kATile + (uint32_t)half * (kBK * 2)));
#endif
              uint8_t* st = smem + (size_t)s * a.stage_bytes;
              tma2d_pair(smem_u32(st), sub ? tmL : tmA, 0, (int)(kb * (a.slice_b >> 7) + arow * 2), fb,
                         pol_keep);
#ifndef NMFA_DBG_NOB
              // J rows of this CTA's half of the tile: ONE box (the per-box TMA cost is
              // ~100 cycles, so the half is never split into power-of-two boxes)
              tma2d_pair(smem_u32(st + kATile), half == a.bhalf1 ? &tmB1 : &tmB0, 0,
                         (kb * a.brows + brow) * 2, fb, pol_keep);
#endif
#ifdef NMFA_L2_PREFETCH  // experiment: pull the A box NMFA_L2_PREFETCH k-slices ahead into L2
              if (ki + NMFA_L2_PREFETCH < a.kblocks) {
                const int kb2 = kord ? kord[ki + NMFA_L2_PREFETCH] : ki + NMFA_L2_PREFETCH;
                asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                                 reinterpret_cast<uint64_t>(tmA)),
                             "r"(0), "r"((int)(kb2 * (a.slice_b >> 7) + arow * 2))
                             : "memory");
              }
#endif
            }  // sub
          }
          if (a.trace && blockIdx.x == 0 && jglob < 512)
            a.trace[jglob * 8 + 7] = wempty;  // cycles the producer waited for a free stage
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ------------------------- MMA issuer (leader CTA) -------------------------
    if (cta == 0 && lane == 0) {
      int it = 0, jj = 0;
      const uint64_t desc0 = make_desc_noswizzle(smem_u32(smem), 128, 2048);
      const uint32_t desc_lo0 = (uint32_t)desc0, desc_hi = (uint32_t)(desc0 >> 32);
      for (int ph = 0; ph < n_phases; ++ph) {
        const int subs = (a.hilo && a.t_begin + ph < a.t_end) ? 2 : 1;  // as the producer
        for (int j = j0; j < j1; ++j, ++jj) {
          const DenseTile tl = a.tiles[j];
          const int slot = jj & 1, use = jj >> 1;
          mbar_wait(&tempty_bar[slot], (use & 1) ^ 1);
          if (a.trace && blockIdx.x == 0 && jj < 512) a.trace[jj * 8 + 2] = clock64();
          if (a.tl2 && jj < 64) a.tl2[((blockIdx.x >> 1) * 64 + jj) * 8 + 2] = gtimer();
          tc_fence_after();
          const uint32_t idesc = make_idesc_f16(256, (uint32_t)tl.nlen);
          const uint32_t d = tbase + (uint32_t)slot * kAccCols;
          long long wfull = 0;
          for (int ki = 0; ki < a.kblocks; ++ki)
          for (int sub = 0; sub < subs; ++sub, ++it) {
            const int s = it % kDStages;
            NMFA_JITTER(blockIdx.x + 7919, it);  // checked build only
            if (a.trace) {
              const long long c0 = clock64();
              mbar_wait(&full_bar[s], (it / kDStages) & 1);
              wfull += clock64() - c0;
            } else {
              mbar_wait(&full_bar[s], (it / kDStages) & 1);
            }
            tc_fence_after();
            if (a.tl3 && blockIdx.x == 0 && it >= 256 && it < 320) a.tl3[(it - 256) * 4 + 1] = clock64();
            const uint32_t a_lo = desc_lo0 + (uint32_t)s * (a.stage_bytes >> 4);
            const uint32_t b_lo = a_lo + (kATile >> 4);
            if (ki != tl.pad) {
#pragma unroll
              for (int ks = 0; ks < kBK / 16; ++ks)
                mma_pair(d, a_lo + ks * 16, b_lo + ks * 16, desc_hi, idesc, (ki | sub | ks) ? 1u : 0u);
            } else {
              for (int ks = 0; ks < a.k_last_sub; ++ks)
                mma_pair(d, a_lo + ks * 16, b_lo + ks * 16, desc_hi, idesc, (ki | sub | ks) ? 1u : 0u);
            }
            commit_pair_mc(&empty_bar[s]);
            if (a.tl3 && blockIdx.x == 0 && it >= 256 && it < 320) a.tl3[(it - 256) * 4 + 2] = clock64();
          }
          commit_pair_mc(&tfull_bar[slot]);
          if (a.tl2 && jj < 64) a.tl2[((blockIdx.x >> 1) * 64 + jj) * 8 + 3] = gtimer();
          if (a.trace && blockIdx.x == 0 && jj < 512) {
            a.trace[jj * 8 + 3] = clock64();
            a.trace[jj * 8 + 6] = wfull;  // cycles the MMA issuer waited for TMA data
          }
        }
      }
    }
  } else if (warp == kWarpAlloc) {
    // ------------------------- readiness prefetch -------------------------
    // Walks the producer's tile sequence ahead of it.  For sweep t > t_begin a
    // tile needs every k-slice of its replica block from sweep t-1, tracked
    // per (block, slice) in `ready` (spins published, summed over the epilogue
    // warps of all pairs).  Progress is posted as (step << 16) | slices known,
    // in the tile's K order; a later step's value implies all earlier ones.
    if (lane == 0) {
      unsigned long long step = 0;
      for (int ph = 0; ph < n_phases; ++ph) {
        int done_m = -1;  // block whose slices are all known ready in this sweep
        for (int j = j0; j < j1; ++j, ++step) {
          const DenseTile tl = a.tiles[j];
          if (ph == 0 || tl.m_blk == done_m) {
            st_release_cta_smem(&pf_ready, (step << 16) | (unsigned long long)a.kblocks);
            continue;
          }
          const int16_t* kord = a.korder ? a.korder + (size_t)j * a.kblocks : nullptr;
          const int qb = tl.m_blk * a.kblocks;
          int known = 0;
          while (known < a.kblocks) {
            unsigned v[8];
            const int cnt = min(8, a.kblocks - known);
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (x < cnt) v[x] = ld_relaxed_gpu(a.ready + qb + (kord ? kord[known + x] : known + x));
            int adv = 0;
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (x < cnt && adv == x &&
                  v[x] >= (unsigned)ph * a.kneed[qb + (kord ? kord[known + x] : known + x)])
                ++adv;
            if (adv) {
              known += adv;
              fence_acq_rel_gpu();  // acquire the published slices for this CTA
              st_release_cta_smem(&pf_ready, (step << 16) | (unsigned long long)known);
            } else {
              __nanosleep(NMFA_POLL_SLEEP_NS);
            }
          }
          done_m = tl.m_blk;
        }
      }
    }
  } else if (warp >= kEpiBase && warp < kEpiBase + kDEpiWarps) {
    // ------------------------- fused NMFA epilogue -------------------------
    // State per (replica r, spin i): hi = fp16(s) lives in the operand image
    // the TMA reads this sweep, lo = fp16(s - hi) in a second image of the same
    // layout, so s = hi + lo carries ~22 bits and the per-sweep working set
    // (2 images + lo + J) is ~104 MB at K2000 / 8192 reads.
    const int e = warp - kEpiBase, quarter = e & 3, hpart = e >> 2;  // lane quarter x column part
    const int row = 32 * quarter + lane;
    const uint32_t leader_tempty0 = map_to_rank(smem_u32(&tempty_bar[0]), 0);
    const uint32_t leader_tempty1 = map_to_rank(smem_u32(&tempty_bar[1]), 0);
    const float4* invn4 = reinterpret_cast<const float4*>(a.invn);
    const float4* hn4 = reinterpret_cast<const float4*>(a.hn);
    #ifdef NMFA_DBG_LOKEEP  // experiment: keep the lo residual in L2 too
    const uint64_t pol_keep = policy_evict_last(), pol_stream0 = policy_evict_last();
#else
    const uint64_t pol_keep = policy_evict_last(), pol_stream0 = policy_evict_first();
#endif
    // HILO: lo is a GEMM operand re-read by every pair of its block, like hi
    const uint64_t pol_stream = a.hilo ? pol_keep : pol_stream0;
    int jj = 0;
    for (int ph = 0; ph < n_phases; ++ph) {
      const int t = a.t_begin + ph;
      const bool energy_phase = t >= a.t_end;
      const bool last = (t == a.t_f - 1);
      const float inv_t = energy_phase ? 0.f : __ldg(a.inv_temp + t);
      const uint8_t* a_cur = (t & 1) ? a.img1 : a.img0;
      uint8_t* a_next = (t & 1) ? a.img0 : a.img1;
      // lo is read and rewritten in place by its owning tile alone, unless the
      // GEMM reads it too (HILO): then it ping-pongs with the sweep parity
      const uint8_t* lo_cur = (a.hilo && (t & 1)) ? a.lo1 : a.lo;
      uint8_t* lo_next = (a.hilo && !(t & 1)) ? a.lo1 : a.lo;
      for (int j = j0; j < j1; ++j, ++jj) {
        const DenseTile tl = a.tiles[j];
        const int slot = jj & 1, use = jj >> 1;
        const long long r = (long long)tl.m_blk * 256 + (long long)cta * 128 + row;
        const bool valid = r < a.R;
        const unsigned long long key = a.key_base + (unsigned long long)r;
        const PhiloxKey K = philox_schedule((uint32_t)key, (uint32_t)(key >> 32));
        const long long row_off = (r >> 3) * 2048 + (r & 7) * 16;
#if defined(NMFA_EPI_SPIN)  // experiment: plain spinning wait
        mbar_wait(&tfull_bar[slot], use & 1);
#elif defined(NMFA_EPI_BACKOFF)  // experiment: test_wait + nanosleep(NMFA_EPI_BACKOFF) ns
        mbar_wait_backoff(&tfull_bar[slot], use & 1, NMFA_EPI_BACKOFF);
#else
        mbar_wait_sleep(&tfull_bar[slot], use & 1, 100000u);
#endif
        if (a.trace && blockIdx.x == 0 && e == 0 && lane == 0 && jj < 512) a.trace[jj * 8 + 4] = clock64();
        tc_fence_after();
        const uint32_t tacc = tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)slot * kAccCols;
        // this warp's columns: a contiguous, 8-aligned quarter of the tile (balanced to 8 spins)
        const int n8 = tl.nlen >> 3;
        const int c_lo = (n8 * hpart / kParts) * 8, c_hi = (n8 * (hpart + 1) / kParts) * 8;
        // byte offset of spins i..i+7 of replica r in an operand image: 32-bit
        // (plans keep each image below 4 GiB), k-slice stride slice_b bytes
        const uint32_t slice_bytes = (uint32_t)a.slice_b, row_off32 = (uint32_t)row_off;
        auto img_off = [&](int i) {
          return (uint32_t)(i >> 7) * slice_bytes + row_off32 + (uint32_t)((i & 127) >> 3) * 128u;
        };
        if (energy_phase) {
          // a_cur holds the +-1 configuration written by the last sweep
          double e_pair = 0.0, e_field = 0.0;
          for (int c = c_lo; c < c_hi; c += 8) {
            const int i0 = tl.n0 + c;
            float acc[8], cs[8];
            tmem_ld8(tacc + c, acc);
            unpack_half8(*reinterpret_cast<const uint4*>(a_cur + img_off(i0)), cs);
            tmem_wait_ld();
            const int nvalid = valid ? min(8, a.n - i0) : 0;
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              if (cc < nvalid) {
                e_pair += (double)(cs[cc] * acc[cc]);        // c_i (J c)_i, exact integers
                const double hv = __ldg(a.h + i0 + cc);
                e_field += cs[cc] < 0.f ? -hv : hv;
              }
            }
          }
          if (valid) atomicAdd(a.energy + r, a.half_scale * e_pair + e_field);  // exact: integers
        } else {
          const bool extra = valid && (a.s_hist != nullptr || (last && a.cfg != nullptr));
          // L1 prefetch of a chunk's state lines (no registers): the loads of chunk
          // c + 16 are in flight while chunk c is computed
          auto prefetch_chunk = [&](int c) {
#ifdef NMFA_EPI_PREFETCH
            if (c < c_hi) {
              const long long off = img_off(tl.n0 + c);
              asm volatile("prefetch.global.L1 [%0];" ::"l"(a_cur + off));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(lo_cur + off));
              if (c + 8 < c_hi) {
                const long long off2 = img_off(tl.n0 + c + 8);
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a_cur + off2));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(lo_cur + off2));
              }
            }
#endif
          };
          auto do_chunk = [&](auto wtag, int c) {
            constexpr int W = decltype(wtag)::value;
            const int i0 = tl.n0 + c;
            prefetch_chunk(c + 16);
            float acc[W], ms[W], lo[W];
#ifdef NMFA_DBG_NOTMEM  // experiment: no accumulator reads (fake fields)
#pragma unroll
            for (int cc = 0; cc < W; ++cc) acc[cc] = 0.001f * (float)(cc + c);
#else
            if constexpr (W == 16) tmem_ld16(tacc + c, acc);
            else tmem_ld8(tacc + c, acc);
#endif
#ifdef NMFA_DBG_NOEPI
            tmem_wait_ld();
#ifdef NMFA_DBG_SPREAD  // experiment: accumulator reads spread over the tile, no math
            __nanosleep(NMFA_DBG_SPREAD);
#endif
            if (acc[0] == 12345.f) a.lo[0] = 1;
            return;
#endif
#pragma unroll
            for (int h = 0; h < W / 8; ++h) {
              const uint32_t off = img_off(i0 + 8 * h);
#if defined(NMFA_DBG_NOLOAD)
#pragma unroll
              for (int q = 0; q < 8; ++q) { ms[8 * h + q] = 0.01f * q; lo[8 * h + q] = 0.f; }
#elif defined(NMFA_DBG_NOLO)
              unpack_half8(ld_hint(a_cur + off, pol_keep), ms + 8 * h);
#pragma unroll
              for (int q = 0; q < 8; ++q) lo[8 * h + q] = 0.f;
#elif !defined(NMFA_DBG_NOMEM) && defined(NMFA_HILO_PLAIN)  // A/B: two converts + FADD
              unpack_half8(ld_hint(a_cur + off, pol_keep), ms + 8 * h);
              unpack_half8(ld_hint(lo_cur + off, pol_stream), lo + 8 * h);
#elif !defined(NMFA_DBG_NOMEM)
              hilo_sum8(ld_hint(a_cur + off, pol_keep), ld_hint(lo_cur + off, pol_stream), ms + 8 * h);
#pragma unroll
              for (int q = 0; q < 8; ++q) lo[8 * h + q] = -0.f;  // x + (-0) == x for every x
#else
#pragma unroll
              for (int q = 0; q < 8; ++q) { ms[8 * h + q] = 0.01f * q; lo[8 * h + q] = 0.f; }
#endif
            }
#pragma unroll
            for (int cc = 0; cc < W; ++cc) ms[cc] += lo[cc];
            tmem_wait_ld();
            const int nvalid = valid ? min(W, a.n - i0) : 0;
            const float* nz = kInjected ? a.noise + ((long long)r * a.t_f + t) * a.n + i0 : nullptr;
#ifdef NMFA_DBG_NOMATH
#pragma unroll
            for (int cc = 0; cc < W; ++cc) ms[cc] = fmaf(acc[cc], 1e-6f, ms[cc]);
#else
            update_chunk<kInjected, W, kDTab>(acc, ms, invn4 + i0 / 4, hn4 + i0 / 4, nz, nvalid, K,
                                              (uint32_t)(i0 / 8), (uint32_t)t, a.sigma, inv_t,
                                              a.alpha, a.oma, sTab);
#endif
            // split s -> (hi, lo); the last sweep writes the +-1 configuration for the energy pass
#pragma unroll
            for (int h = 0; h < W / 8; ++h) {
              const uint32_t off = img_off(i0 + 8 * h);
              uint4 hv, lv;
              if (last)  // uniform: only the final sweep writes the +-1 configuration
                split_hilo8(ms + 8 * h, hv, lv, true);
              else
                split_hilo8(ms + 8 * h, hv, lv, false);
#if defined(NMFA_DBG_NOLO)
              st_hint(a_next + off, hv, pol_keep);
              if (lv.x == 0x12345u && lv.y == 7u) a.lo[0] = 1;
#elif !defined(NMFA_DBG_NOMEM)
              st_hint(a_next + off, hv, pol_keep);
              st_hint(lo_next + off, lv, pol_stream);
              // fused exchange: the same 16 bytes into every other shard's image
              // (NVLink peer stores, overlapped with the GEMM of the next tile)
              for (int pk = 0; pk < a.n_peers; ++pk)
                *reinterpret_cast<uint4*>(((t & 1) ? a.peer0[pk] : a.peer1[pk]) + off) = hv;
#else
              if (hv.x == 0x12345u && lv.y == 7u) a.lo[0] = 1;
#endif
            }
            if (extra) {
              if (a.s_hist) {
                float* hrow = a.s_hist + ((long long)r * a.t_f + t) * a.n + i0;
#pragma unroll
                for (int cc = 0; cc < W; ++cc)
                  if (cc < nvalid) hrow[cc] = ms[cc];
              }
              if (last && a.cfg) {
                int8_t* crow = a.cfg + r * a.n + i0;
#pragma unroll
                for (int cc = 0; cc < W; ++cc)  // sign_round: s < 0 -> -1 else +1 (problem.py:181)
                  if (cc < nvalid) crow[cc] = ms[cc] < 0.f ? (int8_t)-1 : (int8_t)1;
                if (a.s_out) {
#pragma unroll
                  for (int cc = 0; cc < W; ++cc)
                    if (cc < nvalid) a.s_out[r * a.n + i0 + cc] = ms[cc];
                }
              }
            }
          };
          int c = c_lo;
          prefetch_chunk(c);
          for (; c + 16 <= c_hi; c += 16) do_chunk(std::integral_constant<int, 16>{}, c);
          if (c < c_hi) do_chunk(std::integral_constant<int, 8>{}, c);
        }
        NMFA_JITTER(threadIdx.x + 641 * blockIdx.x, jj);  // checked build only
        tc_fence_before();
        __syncwarp();
        if (a.trace && blockIdx.x == 0 && lane == 0 && jj < 512) atomicMax(&a.trace[jj * 8 + 5], clock64());
        if (a.tl2 && lane == 0 && jj < 64) atomicMax(&a.tl2[((blockIdx.x >> 1) * 64 + jj) * 8 + 4], gtimer());
        if (lane == 0) {
#ifdef NMFA_EPI_FENCE_FIRST  // round-1 order: the accumulator-free arrive waits for the stores
          fence_release_gpu();
          mbar_remote_arrive_relaxed(slot ? leader_tempty1 : leader_tempty0);
#else
          // The accumulator slot is free once this warp's TMEM reads are done
          // (tcgen05.wait::ld, tcgen05 fence + __syncwarp above): the arrive does not
          // wait for the state stores.  Only the readiness counters need them, so the
          // gpu-scope release fence (which waits for the stores to be acknowledged)
          // now sits on that path alone and no longer delays the MMA of tile j+2.
          mbar_remote_arrive_relaxed(slot ? leader_tempty1 : leader_tempty0);
#endif
          if (!energy_phase && c_hi > c_lo) {
            // publish this warp's rows x columns for the next sweep (spin-quarters):
            // release its state stores (all lanes', ordered by the __syncwarp) first;
            // the consumers acquire and fence the async proxy
#ifndef NMFA_EPI_FENCE_FIRST
            fence_release_gpu();
#endif
            fence_proxy_async_global();
            const int s_lo = tl.n0 + c_lo, s_hi = tl.n0 + c_hi;
            for (int kb = s_lo >> 7; kb <= (s_hi - 1) >> 7; ++kb)
              red_relaxed_gpu(a.ready + tl.m_blk * a.kblocks + kb,
                              (unsigned)(min(s_hi, kb * 128 + 128) - max(s_lo, kb * 128)));
          }
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 2 * kAccCols);
  }
}

// A image 0 (hi) and the lo image from s0: one thread per (replica, 8-spin
// core row) writes one 16-byte chunk of each image (padding stays zero).
__global__ void dense_init_kernel(uint8_t* a_img, uint8_t* lo_img, const float* s0, int n, int kp,
                                  long long R, long long Rp, long long slice_b) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)(kp / 8) * Rp) return;
  const long long r = e % Rp;
  const int i0 = (int)(e / Rp) * 8;
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = (r < R && i0 + k < n) ? s0[r * n + i0 + k] : 0.f;
  uint4 hv, lv;
  split_hilo8<true>(v, hv, lv, false);
  const long long off = (long long)(i0 >> 7) * slice_b + (r >> 3) * 2048 + ((i0 & 127) >> 3) * 128 +
                        (r & 7) * 16;
  *reinterpret_cast<uint4*>(a_img + off) = hv;
  *reinterpret_cast<uint4*>(lo_img + off) = lv;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_line_map(CUtensorMap* tm, void* base, uint64_t lines, uint32_t box_lines) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return NMFA_ERR_CUDA;
  }
  cuuint64_t dims[2] = {64, lines};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, box_lines};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return NMFA_ERR_CUDA;
  }
  return NMFA_OK;
}

static inline size_t img_off(uint32_t row, uint32_t k, uint32_t rows) {
  return (size_t)(k >> 7) * rows * 256 + (row >> 3) * 2048 + ((k & 127) >> 3) * 128 +
         (row & 7) * 16 + (k & 7) * 2;
}

int dense_problem_upload(nmfa_problem* p, const std::vector<float>& jd) {
  const uint32_t n = (uint32_t)p->n;
  const uint32_t np = (n + 15) / 16 * 16, kp = (n + kBK - 1) / kBK * kBK;
  std::vector<__half> img((size_t)kp * np, __float2half(0.f));
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t k = 0; k < n; ++k) {
      const float v = jd[(size_t)i * n + k];
      if (v != 0.f) img[img_off(i, k, np) / 2] = __float2half(v);
    }
  p->j_dense_bytes = img.size() * 2;
  NMFA_CUDA_TRY(cudaMalloc(&p->d_j_dense, p->j_dense_bytes));
  NMFA_CUDA_TRY(cudaMemcpy(p->d_j_dense, img.data(), p->j_dense_bytes, cudaMemcpyHostToDevice));
  p->row_lo = 0;
  p->row_hi = p->n;
  p->brows = (int32_t)np;
  return NMFA_OK;
}

// J image rows [row_lo, row_lo + brows) of the synthetic SK instance (see
// nmfa_problem_create_sk_device): one thread per (row, 8 consecutive k).
__global__ void sk_image_kernel(uint8_t* img, long long n, int brows, long long row_lo, int kp,
                                unsigned long long seed) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_row = kp / 8;
  if (e >= (long long)brows * per_row) return;
  const int lrow = (int)(e / per_row);
  const int k0 = (int)(e - (long long)lrow * per_row) * 8;
  const long long i = row_lo + lrow;
  const PhiloxKey K = philox_schedule((uint32_t)seed, (uint32_t)(seed >> 32));
  float v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const long long k = k0 + c;
    v[c] = 0.f;
    if (i < n && k < n && k != i) {
      const uint32_t a = (uint32_t)(i < k ? i : k), b = (uint32_t)(i < k ? k : i);
      const uint4_ w = philox4x32_10(b >> 7, a, 0x534B4A31u, 0u, K);
      const uint32_t word = ((b & 127u) >> 5) == 0 ? w.x : ((b & 127u) >> 5) == 1 ? w.y
                          : ((b & 127u) >> 5) == 2 ? w.z : w.w;
      v[c] = ((word >> (b & 31u)) & 1u) ? 1.f : -1.f;
    }
  }
  const long long off = (long long)(k0 >> 7) * brows * 256 + (lrow >> 3) * 2048 +
                        ((k0 & 127) >> 3) * 128 + (lrow & 7) * 16;
  *reinterpret_cast<uint4*>(img + off) =
      make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                 pack_half2(v[6], v[7]));
}

// J image rows [row_lo, row_lo + brows) of a complete +-1 instance given as
// packed sign bits (the bit-packed device format): bit
// a * n + b (a < b, row-major over the n x n matrix, 32 per uint32 word,
// LSB first) set means J_ab = +1, clear means -1.  One thread per (row,
// 8 consecutive k); J is symmetric, so (i, k) reads bit (min, max).
__global__ void bits_image_kernel(uint8_t* img, const uint32_t* __restrict__ bits, long long n,
                                  int brows, long long row_lo, int kp) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_row = kp / 8;
  if (e >= (long long)brows * per_row) return;
  const int lrow = (int)(e / per_row);
  const int k0 = (int)(e - (long long)lrow * per_row) * 8;
  const long long i = row_lo + lrow;
  float v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const long long k = k0 + c;
    v[c] = 0.f;
    if (i < n && k < n && k != i) {
      const unsigned long long b = (unsigned long long)(i < k ? i : k) * (unsigned long long)n +
                                   (unsigned long long)(i < k ? k : i);
      v[c] = ((__ldg(bits + (b >> 5)) >> (b & 31)) & 1u) ? 1.f : -1.f;
    }
  }
  const long long off = (long long)(k0 >> 7) * brows * 256 + (lrow >> 3) * 2048 +
                        ((k0 & 127) >> 3) * 128 + (lrow & 7) * 16;
  *reinterpret_cast<uint4*>(img + off) =
      make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                 pack_half2(v[6], v[7]));
}

int dense_problem_from_bits(nmfa_problem* p, const uint32_t* d_bits) {
  const int kp = (int)((p->n + kBK - 1) / kBK * kBK);
  const size_t bytes = (size_t)kp * p->brows * 2;
  p->j_dense_bytes = bytes;
  NMFA_CUDA_TRY(cudaMalloc(&p->d_j_dense, bytes));
  NMFA_CUDA_TRY(cudaMemset(p->d_j_dense, 0, bytes));
  const long long tot = (long long)p->brows * (kp / 8);
  bits_image_kernel<<<(unsigned)((tot + 255) / 256), 256>>>(
      reinterpret_cast<uint8_t*>(p->d_j_dense), d_bits, p->n, p->brows, p->row_lo, kp);
  NMFA_LAUNCH_CHECK();
  NMFA_CUDA_TRY(cudaDeviceSynchronize());
  return NMFA_OK;
}

// Exact energies of arbitrary +-1 configurations through the dense kernel's
// tensor-core energy pass alone (t_begin = t_end = 0): the configurations are
// written as the A image (hi = +-1, lo = 0) and E = 1/2 j_scale c.(J c) + h.c
// is reduced in the epilogue.  For device-built problems, which have no edge
// list.  cfg: int8 [R][n] of +-1 (R = the plan's replica count).
__global__ void cfg_to_float_kernel(const int8_t* __restrict__ cfg, long long count,
                                    float* __restrict__ s) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < count) s[k] = cfg[k] < 0 ? -1.f : 1.f;
}

int dense_energy_only(const nmfa_plan* pl, const int8_t* cfg, double* energy, cudaStream_t st) {
  const long long count = pl->p->n * pl->R;
  float* s0 = nullptr;
  NMFA_CUDA_TRY(cudaMallocAsync(&s0, (size_t)count * sizeof(float), st));
  cfg_to_float_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(cfg, count, s0);
  int err = cudaGetLastError() == cudaSuccess ? NMFA_OK : NMFA_ERR_CUDA;
  if (!err)
    err = dense_run_sweeps(pl, 0, nullptr, s0, nullptr, nullptr, nullptr, energy, 0, 0, true, st);
  cudaFreeAsync(s0, st);
  if (!err) add_launches(1);
  return err;
}

int dense_problem_generate_sk(nmfa_problem* p, uint64_t seed) {
  const int kp = (int)((p->n + kBK - 1) / kBK * kBK);
  const size_t bytes = (size_t)kp * p->brows * 2;
  p->j_dense_bytes = bytes;
  NMFA_CUDA_TRY(cudaMalloc(&p->d_j_dense, bytes));
  NMFA_CUDA_TRY(cudaMemset(p->d_j_dense, 0, bytes));
  const long long tot = (long long)p->brows * (kp / 8);
  sk_image_kernel<<<(unsigned)((tot + 255) / 256), 256>>>(
      reinterpret_cast<uint8_t*>(p->d_j_dense), p->n, p->brows, p->row_lo, kp, seed);
  NMFA_LAUNCH_CHECK();
  NMFA_CUDA_TRY(cudaDeviceSynchronize());
  return NMFA_OK;
}

void dense_plan_free(nmfa_plan* pl) {
  auto* ds = static_cast<DenseState*>(pl->dense);
  if (!ds) return;
  if (ds->lo_img) cudaFree(ds->lo_img);
  if (ds->lo_img2) cudaFree(ds->lo_img2);
  if (!ds->external_images) {
    if (ds->a_img[0]) cudaFree(ds->a_img[0]);
    if (ds->a_img[1]) cudaFree(ds->a_img[1]);
  }
  if (ds->d_tiles) cudaFree(ds->d_tiles);
  if (ds->d_tile_off) cudaFree(ds->d_tile_off);
  if (ds->d_kneed) cudaFree(ds->d_kneed);
  if (ds->d_korder) cudaFree(ds->d_korder);
  if (ds->d_ready) cudaFree(ds->d_ready);
  delete ds;
  pl->dense = nullptr;
}

int dense_plan_alloc(nmfa_plan* pl) {
  const nmfa_problem* p = pl->p;
  auto* ds = new DenseState();
  pl->dense = ds;
  const int n = (int)p->n;
  ds->np = (n + 15) / 16 * 16;
  ds->kp = (n + kBK - 1) / kBK * kBK;
  ds->kblocks = ds->kp / kBK;
  ds->k_last_sub = (n - (ds->kblocks - 1) * kBK + 15) / 16;
  ds->Rp = (pl->R + 255) / 256 * 256;
  // experiment knob NMFA_SLICE_PAD: extra 128-byte lines between k-slices, so
  // the slices of one replica block are not a power-of-two stride apart
  static const char* pad_env = getenv("NMFA_SLICE_PAD");
  ds->slice_b = ds->Rp * 256 + 128LL * (pad_env ? std::max(0, atoi(pad_env)) : 0);
  const size_t img_bytes = (size_t)ds->kblocks * ds->slice_b;
  if (img_bytes >= (1ULL << 32)) {  // the epilogue addresses images with 32-bit offsets
    set_error("dense plan: n x replicas too large for one plan (state image >= 4 GiB); "
              "split the replicas over several calls (r0)");
    return NMFA_ERR_ARG;
  }
  NMFA_CUDA_TRY(cudaMalloc(&ds->lo_img, img_bytes));
  NMFA_CUDA_TRY(cudaMalloc(&ds->a_img[0], img_bytes));
  NMFA_CUDA_TRY(cudaMalloc(&ds->a_img[1], img_bytes));
  NMFA_CUDA_TRY(cudaMemset(ds->a_img[0], 0, img_bytes));
  NMFA_CUDA_TRY(cudaMemset(ds->a_img[1], 0, img_bytes));
  ds->hilo = pl->field == NMFA_FIELD_HILO;
  if (ds->hilo) {
    if (dense_is_sharded(p)) {
      set_error("field precision HILO is not available on a row shard");
      return NMFA_ERR_ARG;
    }
    // the GEMM reads lo over the whole padded k range: zero it once (the
    // epilogue never writes spins >= the padded n, and J is zero there)
    NMFA_CUDA_TRY(cudaMalloc(&ds->lo_img2, img_bytes));
    NMFA_CUDA_TRY(cudaMemset(ds->lo_img2, 0, img_bytes));
  }

  // Static schedule.  A tile is (replica block of 256, w x 16 spins); per
  // k-slice of 128 it costs max(MMA = 64 w, TMA = 563 + 22.6 w) cycles
  // (profiles/r01/tma_bench2.log: ~100 cycles per box + ~11.3 cycles/KB, one
  // 32 KB A box + one w*2 KB B box per CTA).  Pick the width minimising the
  // makespan ceil(tiles / pairs) * cost(w); then give every pair a contiguous
  // run of whole tiles (counts differ by at most one), so no pair gets a narrow,
  // TMA-bound remainder tile.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  // tiles cover this device's spins [row_lo, row_lo + brows) only
  ds->slice_lo = (int)(p->row_lo / kBK);
  ds->slice_hi = (int)((p->row_hi + kBK - 1) / kBK);
  const long long upm = p->brows / 16, mb = ds->Rp / 256;
  // Tile width for a group of `blocks` replica blocks: minimise the makespan
  // ceil(tiles / pairs) * cost(w) of the cost model above.
  auto width_for = [&](long long blocks) {
    int bw = kMaxW;
    double bc = 1e300;
    for (int w = 1; w <= kMaxW; ++w) {
      const long long tpm = (upm + w - 1) / w, T = tpm * blocks;
      const long long pairs_used = std::min<long long>(sms / 2, T);
      const double per_slice = std::max(64.0 * w, 563.0 + 22.6 * w);
      const double makespan = (double)((T + pairs_used - 1) / pairs_used) * per_slice;
      if (makespan < bc - 1e-9) {
        bc = makespan;
        bw = w;
      }
    }
    return bw;
  };
  // L2-aware replica groups: replica blocks never interact, so when the
  // working set of one sweep (two hi images + lo + J) outgrows L2 the blocks
  // are split into groups annealed one after another (one persistent launch
  // each, all t_f sweeps), as long as every group still deals >= 3.75 tiles
  // per pair: below that a sweep is bound by its dependency chain (a tile's
  // MMA, then its epilogue, then the next sweep's wait), not by L2, and the
  // split lost up to 14% at N = 1000-1500 (profiles/r02/dense_groups.log).
  // Results are unchanged (natural K order, global replica keys).  N x R
  // beyond L2 fell to 0.65-0.70 of the sustained peak as one group.
  // Row-sharded plans advance sweep by sweep across devices and stay one
  // group.  NMFA_DENSE_GROUPS=k forces k groups, NMFA_L2_BUDGET_MB sets the
  // budget.
  const double j_bytes = (double)ds->kp * p->brows * 2.0;
  const double images = ds->hilo ? 4.0 : 3.0;  // two hi images + lo (+ the second lo of HILO)
  auto footprint = [&](long long blocks) { return images * 2.0 * ds->kp * 256.0 * blocks + j_bytes; };
  static const char* budget_env = getenv("NMFA_L2_BUDGET_MB");
  const double budget = (budget_env ? atof(budget_env) : 120.0) * 1e6;
  auto tiles_for = [&](long long blocks) {
    const int w = width_for(blocks);
    return (upm + w - 1) / w * blocks;
  };
  long long n_groups = 1;
  if (!dense_is_sharded(p)) {
    while (footprint((mb + n_groups - 1) / n_groups) > budget) {
      const long long g2 = n_groups * 2;
      if (g2 > mb || 4 * tiles_for(mb / g2) < 15LL * (sms / 2)) break;  // >= 3.75 per pair
      n_groups = g2;
    }
  }
  static const char* groups_env = getenv("NMFA_DENSE_GROUPS");
  if (groups_env && atoi(groups_env) >= 1) n_groups = std::min<long long>(mb, atoi(groups_env));
  const long long mb_g = (mb + n_groups - 1) / n_groups;  // largest group
  int best_w = width_for(mb_g);
  static const char* w_env = getenv("NMFA_TILE_W");  // experiment: force the tile width
  if (w_env && atoi(w_env) >= 1 && atoi(w_env) <= kMaxW) best_w = atoi(w_env);
  const long long tpm = (upm + best_w - 1) / best_w;
  static const char* order_env = getenv("NMFA_TILE_ORDER");
  const std::string order = order_env ? order_env : "skew";
  std::vector<DenseTile> tiles;            // every group's list, concatenated
  std::vector<int> off;                    // per group: pairs_g + 1 absolute offsets
  ds->grp_off_base.clear();
  ds->grp_pairs.clear();
  for (long long g = 0; g < n_groups; ++g) {
    const long long gm0 = mb * g / n_groups, gm1 = mb * (g + 1) / n_groups;
    const long long T = tpm * (gm1 - gm0);
    const int pairs = (int)std::min<long long>(sms / 2, T);
    ds->grp_off_base.push_back((int)off.size());
    ds->grp_pairs.push_back(pairs);
    // Spin-major dealing: sort tiles by (spin tile k, replica block m) and give
    // position j of pair q the tile q + j*pairs.  Every pair works on the
    // lowest spins first, so in sweep t the k-slices become ready in the order
    // the sweep-(t+1) k-loops consume them (natural K order), and the first tile
    // of a sweep does not wait for the end of the previous one.
    // debug knob NMFA_TILE_ORDER: mmajor (contiguous m-major runs), sorted (the
    // same runs ordered by spin within each pair), spin (spin-major dealing)
    std::vector<DenseTile> mmaj;
    mmaj.reserve(T);
    for (long long m = gm0; m < gm1; ++m)
      for (long long k = 0; k < tpm; ++k) {  // balanced widths within the block
        const long long a0 = upm * k / tpm, a1 = upm * (k + 1) / tpm;
        mmaj.push_back({(int)m, (int)(p->row_lo + a0 * 16), (int)((a1 - a0) * 16), 0});
      }
    std::vector<int> goff(pairs + 1, 0);
    // Skewed dealing (default): replica blocks split into an early class E and a
    // late class L.  Every pair runs its E tiles first and its L tiles last, at
    // least one of each, so an E block's tiles sit in positions [0, S-2] and an
    // L block's in [1, S-1] (S = tiles per pair).  Position 0 of sweep t+1 then
    // consumes only E blocks, finished at least one tile-time before the sweep
    // boundary, and no pair waits for another pair's last tile (m-major runs made
    // every sweep start wait ~20 us for the previous sweep's last epilogues,
    // profiles/r02/dense_schedule.log).  Within a class the tiles are m-major
    // runs, as before.  K order and results are unchanged.
    const long long mbk = gm1 - gm0;  // blocks in this group
    std::vector<long long> cnt(pairs), ecnt(pairs, 0);
    for (int q = 0; q < pairs; ++q) cnt[q] = T * (q + 1) / pairs - T * q / pairs;
    bool skew = order == "skew" || order_env == nullptr;
    long long mbE = 0;
    if (skew) {
      // E = the first mbE blocks; find a split the per-pair bounds can realise
      long long lo_sum = 0, hi_sum = 0;
      for (int q = 0; q < pairs; ++q) {
        lo_sum += cnt[q] >= 2 ? 1 : 0;
        hi_sum += cnt[q] >= 2 ? cnt[q] - 1 : cnt[q];
      }
      skew = false;
      for (long long dm = 0; dm <= mbk && !skew; ++dm)
        for (long long cand : {mbk / 2 - dm, (mbk + 1) / 2 + dm})
          if (!skew && cand >= 1 && cand < mbk && cand * tpm >= lo_sum && cand * tpm <= hi_sum) {
            mbE = cand;
            skew = true;
          }
      if (skew) {
        long long need = mbE * tpm, sum = 0;
        for (int q = 0; q < pairs; ++q) {
          ecnt[q] = cnt[q] >= 2 ? std::max(1LL, cnt[q] / 2) : 0;
          sum += ecnt[q];
        }
        for (int q = 0; sum < need && q < 4 * pairs; ++q) {  // raise E counts up to cnt - 1
          const int i = q % pairs;
          const long long cap = cnt[i] >= 2 ? cnt[i] - 1 : cnt[i];
          if (ecnt[i] < cap) ++ecnt[i], ++sum;
        }
        for (int q = 0; sum > need && q < 4 * pairs; ++q) {  // lower them down to 1 (0 for single tiles)
          const int i = pairs - 1 - q % pairs;
          const long long floor_ = cnt[i] >= 2 ? 1 : 0;
          if (ecnt[i] > floor_) --ecnt[i], --sum;
        }
        skew = sum == need;
      }
    }
    if (skew) {
      long long je = 0, jl = mbE * tpm;  // cursors into the m-major list (E blocks first)
      for (int q = 0; q < pairs; ++q) {
        goff[q] = (int)tiles.size();
        for (long long k = 0; k < ecnt[q]; ++k) tiles.push_back(mmaj[je++]);
        for (long long k = ecnt[q]; k < cnt[q]; ++k) tiles.push_back(mmaj[jl++]);
      }
    } else if (order == "block") {
      // m-major list dealt round-robin: at position j the pairs hold whole replica
      // blocks (~pairs / tiles-per-block of them), so block m's sweep-t tiles all
      // finish at one position and its sweep-(t+1) tiles run a full sweep later
      for (int q = 0; q < pairs; ++q) {
        goff[q] = (int)tiles.size();
        for (long long j = q; j < T; j += pairs) tiles.push_back(mmaj[j]);
      }
    } else if (order == "spin") {
      std::vector<DenseTile> sorted(mmaj);
      std::stable_sort(sorted.begin(), sorted.end(),
                       [](const DenseTile& x, const DenseTile& y) { return x.n0 < y.n0; });
      for (int q = 0; q < pairs; ++q) {
        goff[q] = (int)tiles.size();
        for (long long j = q; j < T; j += pairs) tiles.push_back(sorted[j]);
      }
    } else {
      for (int q = 0; q < pairs; ++q) {
        goff[q] = (int)tiles.size();
        const long long j0 = T * q / pairs, j1 = T * (q + 1) / pairs;
        std::vector<DenseTile> run(mmaj.begin() + j0, mmaj.begin() + j1);
        if (order == "sorted")
          std::stable_sort(run.begin(), run.end(),
                           [](const DenseTile& x, const DenseTile& y) { return x.n0 < y.n0; });
        if ((order == "alt" && (q & 1)) || order == "rev") std::reverse(run.begin(), run.end());
        tiles.insert(tiles.end(), run.begin(), run.end());
      }
    }
    goff[pairs] = (int)tiles.size();
    off.insert(off.end(), goff.begin(), goff.end());
  }  // groups
  if (getenv("NMFA_DENSE_VERBOSE"))
    fprintf(stderr, "dense plan: Rp=%d groups=%lld w=%d tiles=%zu footprint/group=%.1f MB\n",
            ds->Rp, n_groups, best_w, tiles.size(), footprint(mb_g) / 1e6);
  // widest launch (sizes the debug traces; NMFA_TRACE2 decodes group 0 only)
  ds->pairs = *std::max_element(ds->grp_pairs.begin(), ds->grp_pairs.end());
  const long long T = (long long)tiles.size();
  // K order per tile: natural (slice 0 first), so a spin's fp32 field is summed
  // in the same order for every schedule, replica count and row sharding.  The
  // debug knob NMFA_KORDER=early consumes slices earliest-published first
  // (slice (m, kb) is published when the last tile covering it ends, estimated
  // by that tile's position in its pair's list); results then depend on the
  // schedule.  Measured: no gain at K2000 (profiles/r01/korder_ab.log).
  const int kbn = ds->kblocks;
  static const char* korder_env = getenv("NMFA_KORDER");
  const bool early = korder_env && std::string(korder_env) == "early";
  // debug knob NMFA_KORDER=rotate: tile j starts at its own spin range's k-slice
  // (spreads the concurrent reads of tiles that share A/J lines; timing only)
  // rotm: by the replica block (pairs sharing a J tile start apart); rotmn: by both
  const std::string kord_s = korder_env ? korder_env : "";
  const bool rotate = kord_s == "rotate" || kord_s == "rotm" || kord_s == "rotmn";
  std::vector<int> avail((size_t)mb * kbn, 0);
  for (size_t g = 0; g < ds->grp_pairs.size(); ++g) {
    const int* go = off.data() + ds->grp_off_base[g];
    for (int q = 0; q < ds->grp_pairs[g]; ++q)
      for (int j = go[q]; j < go[q + 1]; ++j) {
        const DenseTile& t = tiles[j];
        for (int kb = t.n0 >> 7; kb <= (t.n0 + t.nlen - 1) >> 7; ++kb)
          avail[(size_t)t.m_blk * kbn + kb] = std::max(avail[(size_t)t.m_blk * kbn + kb], j - go[q]);
      }
  }
  std::vector<int16_t> korder;
  if (early || rotate) korder.resize((size_t)T * kbn);
  for (long long j = 0; j < T; ++j) {
    DenseTile& t = tiles[j];
    t.pad = kbn - 1;  // position of the short last k-slice in the tile's K order
    if (rotate) {
      int16_t* ko = &korder[(size_t)j * kbn];
      const int sn = (t.n0 - (int)p->row_lo) >> 7;
      const int s0 = (kord_s == "rotm" ? 3 * t.m_blk : kord_s == "rotmn" ? sn + 3 * t.m_blk : sn) % kbn;
      for (int k = 0; k < kbn; ++k) ko[k] = (int16_t)((k + s0) % kbn);
      t.pad = (kbn - 1 - s0 + kbn) % kbn;
      continue;
    }
    if (!early) continue;
    int16_t* ko = &korder[(size_t)j * kbn];
    for (int k = 0; k < kbn; ++k) ko[k] = (int16_t)k;
    std::stable_sort(ko, ko + kbn, [&](int16_t x, int16_t y) {
      return avail[(size_t)t.m_blk * kbn + x] < avail[(size_t)t.m_blk * kbn + y];
    });
    for (int k = 0; k < kbn; ++k)
      if (ko[k] == kbn - 1) t.pad = k;
  }
  if (early || rotate) {
    NMFA_CUDA_TRY(cudaMalloc(&ds->d_korder, korder.size() * sizeof(int16_t)));
    NMFA_CUDA_TRY(cudaMemcpy(ds->d_korder, korder.data(), korder.size() * sizeof(int16_t),
                             cudaMemcpyHostToDevice));
  }
  NMFA_CUDA_TRY(cudaMalloc(&ds->d_tiles, tiles.size() * sizeof(DenseTile)));
  NMFA_CUDA_TRY(cudaMemcpy(ds->d_tiles, tiles.data(), tiles.size() * sizeof(DenseTile),
                           cudaMemcpyHostToDevice));
  NMFA_CUDA_TRY(cudaMalloc(&ds->d_tile_off, off.size() * sizeof(int)));
  NMFA_CUDA_TRY(
      cudaMemcpy(ds->d_tile_off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
  ds->n_mblk = (int)mb;
  ds->n_tiles = (int)T;
  // Readiness is counted per (replica block, k-slice) in spin-quarters; slices
  // of other shards need 0.
  std::vector<unsigned> kneed((size_t)mb * kbn, 0);
  for (const DenseTile& t : tiles)
    for (int kb = t.n0 >> 7; kb <= (t.n0 + t.nlen - 1) >> 7; ++kb) {
      const int lo_s = std::max(t.n0, kb * 128), hi_s = std::min(t.n0 + t.nlen, kb * 128 + 128);
      kneed[(size_t)t.m_blk * kbn + kb] += 8u * (unsigned)(hi_s - lo_s);  // 2 CTAs x 4 quarters
    }
  NMFA_CUDA_TRY(cudaMalloc(&ds->d_kneed, kneed.size() * sizeof(unsigned)));
  NMFA_CUDA_TRY(cudaMemcpy(ds->d_kneed, kneed.data(), kneed.size() * sizeof(unsigned),
                           cudaMemcpyHostToDevice));
  NMFA_CUDA_TRY(cudaMalloc(&ds->d_ready, kneed.size() * sizeof(unsigned)));

  int err;
  for (int b = 0; b < 2; ++b) {
    if ((err = make_line_map(&ds->tmA[b], ds->a_img[b], (uint64_t)ds->kblocks * (ds->slice_b >> 7), 256)))
      return err;
    ds->tmL[b] = ds->tmA[b];
    if (ds->hilo && (err = make_line_map(&ds->tmL[b], b ? ds->lo_img2 : ds->lo_img,
                                         (uint64_t)ds->kblocks * (ds->slice_b >> 7), 256)))
      return err;
  }
  // one B tensor map per distinct tile width (balanced widths: at most two)
  {
    int hs[2] = {-1, -1}, nh = 0;
    for (const DenseTile& t : tiles) {
      const int h = t.nlen / 2;
      if (h == hs[0] || h == hs[1]) continue;
      if (nh == 2 || h > 128 || h % 8) {
        set_error("dense schedule: unsupported tile width " + std::to_string(t.nlen));
        return NMFA_ERR_STATE;
      }
      hs[nh++] = h;
    }
    if (nh == 1) hs[1] = hs[0];
    // ring stages sized for this plan's widest B half (the unused shared memory
    // stays L1); NMFA_STAGE_FULL=1 keeps the kMaxW-sized stages (A/B)
    static const char* full_env = getenv("NMFA_STAGE_FULL");
    const uint32_t bmax = (uint32_t)std::max(hs[0], hs[1]) * (kBK * 2);
    ds->stage_bytes = (full_env && full_env[0] == '1') ? kDStageBytes
                                                      : (kATile + bmax + 1023u) / 1024u * 1024u;
    for (int b = 0; b < 2; ++b) {
      ds->bhalf[b] = hs[b];
      if ((err = make_line_map(&ds->tmB[b], p->d_j_dense, (uint64_t)ds->kblocks * p->brows * 2,
                               2u * (uint32_t)hs[b])))
        return err;
    }
  }
  NMFA_CUDA_TRY(cudaFuncSetAttribute(dense_anneal_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDSmemBytes));
  NMFA_CUDA_TRY(cudaFuncSetAttribute(dense_anneal_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDSmemBytes));
  return NMFA_OK;
}

// Sweeps [t_begin, t_end) (+ the energy pass) in ONE persistent launch.
// t_begin == 0 initialises the state from s0 (or zeros).
int dense_run_sweeps(const nmfa_plan* pl, uint64_t key_base, const float* noise, const float* s0,
                     int8_t* cfg, float* s_out, float* s_hist, double* energy, int t_begin,
                     int t_end, bool energy_pass, cudaStream_t st) {
  const nmfa_problem* p = pl->p;
  auto* ds = static_cast<DenseState*>(pl->dense);
  if (!ds) {
    set_error("dense plan state missing");
    return NMFA_ERR_STATE;
  }
  int64_t launches = 1;
  const size_t img_bytes = (size_t)ds->kblocks * ds->slice_b;
  if (t_begin == 0) {
    if (s0) {
      const long long tot = (long long)(ds->kp / 8) * ds->Rp;
      dense_init_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          ds->a_img[0], ds->lo_img, s0, (int)p->n, ds->kp, pl->R, ds->Rp, ds->slice_b);
      NMFA_LAUNCH_CHECK();
      ++launches;
    } else {  // S(0) = 0 (solver.py:200-201)
      NMFA_CUDA_TRY(cudaMemsetAsync(ds->a_img[0], 0, img_bytes, st));
      NMFA_CUDA_TRY(cudaMemsetAsync(ds->lo_img, 0, img_bytes, st));
    }
  }
  if (energy_pass) NMFA_CUDA_TRY(cudaMemsetAsync(energy, 0, sizeof(double) * pl->R, st));
  NMFA_CUDA_TRY(cudaMemsetAsync(ds->d_ready, 0, sizeof(unsigned) * ds->n_mblk * ds->kblocks, st));
  DenseStepArgs a{};
  a.tiles = ds->d_tiles;
  a.tile_off = ds->d_tile_off;
  a.kneed = ds->d_kneed;
  a.korder = ds->d_korder;
  a.ready = ds->d_ready;
  a.kblocks = ds->kblocks;
  a.k_last_sub = ds->k_last_sub;
  a.n = (int)p->n;
  a.brows = p->brows;
  a.row_lo = (int)p->row_lo;
  a.R = pl->R;
  a.Rp = ds->Rp;
  a.slice_b = ds->slice_b;
  a.t_begin = t_begin;
  a.t_end = t_end;
  a.t_f = pl->t_f;
  a.energy_pass = energy_pass ? 1 : 0;
  a.alpha = pl->alpha;
  a.oma = pl->oma;
  a.sigma = pl->sigma;
  a.inv_temp = pl->d_inv_temp;
  a.invn = p->d_invn;
  a.hn = p->d_hn;
  a.img0 = ds->a_img[0];
  a.img1 = ds->a_img[1];
  a.lo = ds->lo_img;
  a.lo1 = ds->lo_img2;
  a.hilo = ds->hilo ? 1 : 0;
  a.stage_bytes = ds->stage_bytes;
  a.key_base = key_base;
  a.noise = noise;
  a.cfg = cfg;
  a.s_out = s_out;
  a.s_hist = s_hist;
  a.energy = energy;
  a.h = p->d_h;
  a.half_scale = 0.5 * p->j_scale;
  // one persistent launch for every sweep; all clusters must be co-resident
  // (the readiness spin-waits cross CTAs), which the cooperative attribute asserts
  cudaLaunchConfig_t cfgl{};
  cfgl.gridDim = dim3(2 * ds->pairs);
  cfgl.blockDim = dim3(kDThreads);
  cfgl.dynamicSmemBytes = (size_t)kDStages * ds->stage_bytes + 1024;
  cfgl.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfgl.attrs = attr;
  cfgl.numAttrs = 1;
  static const char* trace_path = getenv("NMFA_TRACE");
  static unsigned long long* trace = nullptr;
  if (trace_path) {
    if (!trace) cudaMallocManaged(&trace, 512 * 8 * 8);
    cudaMemset(trace, 0, 512 * 8 * 8);
    a.trace = trace;
  }
  static const char* tl2_path = getenv("NMFA_TRACE2");
  static unsigned long long* tl2 = nullptr;
  if (tl2_path) {
    if (!tl2) cudaMallocManaged(&tl2, (size_t)ds->pairs * 64 * 8 * 8);
    cudaMemset(tl2, 0, (size_t)ds->pairs * 64 * 8 * 8);
    a.tl2 = tl2;
  }
  static const char* tl3_path = getenv("NMFA_TRACE3");
  static unsigned long long* tl3 = nullptr;
  if (tl3_path) {
    if (!tl3) cudaMallocManaged(&tl3, 64 * 4 * 8);
    cudaMemset(tl3, 0, 64 * 4 * 8);
    a.tl3 = tl3;
  }
  auto kern = noise ? dense_anneal_kernel<true> : dense_anneal_kernel<false>;
  a.bhalf0 = ds->bhalf[0];
  a.bhalf1 = ds->bhalf[1];
  a.n_peers = ds->n_peers;
  for (int k = 0; k < kMaxPeers; ++k) {
    a.peer0[k] = ds->peer_img[0][k];
    a.peer1[k] = ds->peer_img[1][k];
  }
  // one persistent launch per replica group (L2-aware split, dense_plan_alloc)
  for (size_t g = 0; g < ds->grp_pairs.size(); ++g) {
    a.tile_off = ds->d_tile_off + ds->grp_off_base[g];
    cfgl.gridDim = dim3(2 * ds->grp_pairs[g]);
    NMFA_CUDA_TRY(
        cudaLaunchKernelEx(&cfgl, kern, ds->tmA[0], ds->tmA[1], ds->tmB[0], ds->tmB[1],
                           ds->tmL[0], ds->tmL[1], a));
  }
  launches += (int64_t)ds->grp_pairs.size() - 1;
  add_launches(launches);
  if (tl3_path) {
    cudaStreamSynchronize(st);
    FILE* f = fopen(tl3_path, "w");
    if (f) {
      for (int k = 0; k < 64; ++k) fprintf(f, "%llu %llu %llu\n", tl3[k * 4], tl3[k * 4 + 1], tl3[k * 4 + 2]);
      fclose(f);
    }
  }
  if (tl2_path) {
    cudaStreamSynchronize(st);
    std::vector<DenseTile> ht(ds->n_tiles);
    std::vector<int> hoff(ds->pairs + 1);
    cudaMemcpy(ht.data(), ds->d_tiles, ht.size() * sizeof(DenseTile), cudaMemcpyDeviceToHost);
    cudaMemcpy(hoff.data(), ds->d_tile_off, hoff.size() * sizeof(int), cudaMemcpyDeviceToHost);
    FILE* f = fopen(tl2_path, "w");
    if (f) {
      // pair jglob m n0 nlen | prod_start last_slice_ready mma_start mma_end epi_end first_slice_ready
      for (int q = 0; q < ds->pairs; ++q) {
        const int nt = hoff[q + 1] - hoff[q];
        for (int j = 0; j < 64; ++j) {
          const unsigned long long* r = tl2 + ((size_t)q * 64 + j) * 8;
          if (!r[2]) continue;
          const DenseTile& t = ht[hoff[q] + j % nt];
          fprintf(f, "%d %d %d %d %d %llu %llu %llu %llu %llu %llu\n", q, j, t.m_blk, t.n0, t.nlen,
                  r[0], r[1], r[2], r[3], r[4], r[5]);
        }
      }
      fclose(f);
    }
  }
  if (trace_path) {
    cudaStreamSynchronize(st);
    FILE* f = fopen(trace_path, "w");
    if (f) {
      for (int j = 0; j < 512; ++j) {
        for (int k = 0; k < 8; ++k) fprintf(f, "%llu ", trace[j * 8 + k]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  return NMFA_OK;
}

// Fused exchange for a row-sharded plan: adopt the caller's peer-accessible
// buffers as this shard's operand images (images[p][rank]) and record the
// other shards' images as store targets.  The caller synchronises the shards
// between sweeps (every shard's stores must land before the next sweep reads).
int dense_set_exchange(nmfa_plan* pl, void* const* img0, void* const* img1, int world, int rank,
                       int64_t bytes) {
  auto* ds = static_cast<DenseState*>(pl->dense);
  if (!ds) {
    set_error("not a dense plan");
    return NMFA_ERR_STATE;
  }
  const size_t img_bytes = (size_t)ds->kblocks * ds->slice_b;
  if (world < 1 || world > kMaxPeers + 1 || rank < 0 || rank >= world) {
    set_error("fused exchange needs 1 <= world <= 8 and 0 <= rank < world");
    return NMFA_ERR_ARG;
  }
  if (bytes < (int64_t)img_bytes) {
    set_error("exchange buffers smaller than the plan's operand image (" +
              std::to_string(img_bytes) + " bytes)");
    return NMFA_ERR_ARG;
  }
  for (int g = 0; g < world; ++g)
    if (!img0[g] || !img1[g]) {
      set_error("NULL exchange buffer");
      return NMFA_ERR_ARG;
    }
  if (ds->hilo) {
    set_error("the fused exchange carries the hi image only; use an FP16-field plan");
    return NMFA_ERR_ARG;
  }
  const bool own = img0[rank] == ds->a_img[0] && img1[rank] == ds->a_img[1];
  if (!own) {  // adopt the caller's buffers (not freed by the plan)
    if (!ds->external_images) {
      cudaFree(ds->a_img[0]);
      cudaFree(ds->a_img[1]);
    }
    ds->external_images = true;
    ds->a_img[0] = static_cast<uint8_t*>(img0[rank]);
    ds->a_img[1] = static_cast<uint8_t*>(img1[rank]);
  }
  int err;
  for (int b = 0; b < 2; ++b) {
    if ((err = make_line_map(&ds->tmA[b], ds->a_img[b], (uint64_t)ds->kblocks * (ds->slice_b >> 7), 256)))
      return err;
    ds->tmL[b] = ds->tmA[b];  // unused: exchange plans are FP16-field plans
  }
  ds->n_peers = 0;
  for (int g = 0; g < world; ++g) {
    if (g == rank) continue;
    ds->peer_img[0][ds->n_peers] = static_cast<uint8_t*>(img0[g]);
    ds->peer_img[1][ds->n_peers] = static_cast<uint8_t*>(img1[g]);
    ++ds->n_peers;
  }
  return NMFA_OK;
}

bool dense_is_sharded(const nmfa_problem* p) { return p->row_lo != 0 || p->row_hi != p->n; }

int launch_dense_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                        const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                        double* energy, bool* energy_done, cudaStream_t st) {
  if (dense_is_sharded(pl->p)) {
    set_error("a row-sharded problem runs one sweep per nmfa_plan_run_sweeps call "
              "with an all-gather of the operand image in between");
    return NMFA_ERR_STATE;
  }
  *energy_done = energy && dense_energy_exact(pl->p);
  return dense_run_sweeps(pl, key_base, noise, s0, cfg, s_out, s_hist, energy, 0, pl->t_f,
                          *energy_done, st);
}

int dense_image_info(const nmfa_plan* pl, void** img0, void** img1, int64_t* slice_bytes,
                     int32_t* n_slices, int32_t* slice_lo, int32_t* slice_hi) {
  auto* ds = static_cast<DenseState*>(pl->dense);
  if (!ds) {
    set_error("not a dense plan");
    return NMFA_ERR_STATE;
  }
  *img0 = ds->a_img[0];
  *img1 = ds->a_img[1];
  *slice_bytes = ds->slice_b;
  *n_slices = ds->kblocks;
  *slice_lo = ds->slice_lo;
  *slice_hi = ds->slice_hi;
  return NMFA_OK;
}

// cfg[r][i] = sign of the fp16 +-1 sign image
__global__ void read_config_kernel(const uint8_t* img, int8_t* cfg, int n, long long R,
                                   long long slice_b) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * R) return;
  const long long r = e / n;
  const int i = (int)(e - r * n);
  const long long off = (long long)(i >> 7) * slice_b + (r >> 3) * 2048 + ((i & 127) >> 3) * 128 +
                        (r & 7) * 16 + (i & 7) * 2;
  const __half h = *reinterpret_cast<const __half*>(img + off);
  cfg[e] = __half2float(h) < 0.f ? (int8_t)-1 : (int8_t)1;
}

int dense_read_config(const nmfa_plan* pl, int8_t* cfg, cudaStream_t st) {
  auto* ds = static_cast<DenseState*>(pl->dense);
  if (!ds) {
    set_error("not a dense plan");
    return NMFA_ERR_STATE;
  }
  const long long tot = pl->p->n * pl->R;
  read_config_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      ds->a_img[pl->t_f & 1], cfg, (int)pl->p->n, pl->R, ds->slice_b);
  NMFA_LAUNCH_CHECK();
  add_launches(1);
  return NMFA_OK;
}

bool dense_energy_exact(const nmfa_problem* p) {
  // integer weights stored as J / j_scale lie on a 1/j_scale grid (j_scale a
  // power of two); every fp32 partial row sum k / j_scale is exact while the
  // integer |k| <= max_row_abs stays below 2^24
  return p->int_weights && p->j_exact && p->max_row_abs < 16777216.0;
}

}  // namespace nmfa
