// The reference's own noise streams on the device: run k
// of a seeded batch draws noise_stream(seed + k).standard_normal((t_f, n)) *
// sigma (solver.py:182-185, 236-241), i.e. numpy's Philox4x64-10 bit
// generator keyed [seed + k, RUN_STREAM_TAG = 2] with counter 0 and a
// four-word output buffer, fed to numpy's 256-layer ziggurat
// (Generator.standard_normal; tables in numpy_normal_tables.h, extracted and
// checked bit for bit by tools/gen_numpy_normal_tables.py).
//
// The default generator is warp-parallel (ref_noise_warp_kernel below); the
// original one-thread-per-run walk (NMFA_REFNOISE_SEQ=1) is kept as its
// reference: ziggurat rejection makes the stream position data-dependent, so
// the parallel form finds the start positions instead of skipping ahead.  The fast
// path (99.3% of draws) is integer work plus one multiply and is bitwise
// numpy's; the wedge test compares against exp() and the tail uses log1p(),
// where CUDA's double functions may differ from the host libm in the last
// ulp: the tail draws can then differ by an ulp in float64 (never observed
// in float32, the precision the anneal kernels consume).
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "numpy_normal_tables.h"

namespace nmfa {
namespace {

constexpr uint64_t kPM0 = 0xD2E7470EE14C6C93ull, kPM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPW0 = 0x9E3779B97F4A7C15ull, kPW1 = 0xBB67AE8584CAA73Bull;

struct NpPhilox {
  uint64_t c0, c1, c2, c3;  // 256-bit counter
  uint64_t k0, k1;          // key
  uint64_t b0, b1, b2, b3;  // output buffer
  int pos;                  // next buffer word (4 = empty)
};

__device__ __forceinline__ uint64_t np_next(NpPhilox& s) {
  if (s.pos < 4) {
    const uint64_t v = s.pos == 1 ? s.b1 : s.pos == 2 ? s.b2 : s.b3;
    ++s.pos;
    return v;
  }
  // increment the counter (carry through all four words), then 10 rounds
  if (++s.c0 == 0 && ++s.c1 == 0 && ++s.c2 == 0) ++s.c3;
  uint64_t x0 = s.c0, x1 = s.c1, x2 = s.c2, x3 = s.c3, k0 = s.k0, k1 = s.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPM0 * x0, hi0 = __umul64hi(kPM0, x0);
    const uint64_t lo1 = kPM1 * x2, hi1 = __umul64hi(kPM1, x2);
    x0 = hi1 ^ x1 ^ k0;
    x1 = lo1;
    x2 = hi0 ^ x3 ^ k1;
    x3 = lo0;
    k0 += kPW0;
    k1 += kPW1;
  }
  s.b0 = x0, s.b1 = x1, s.b2 = x2, s.b3 = x3;
  s.pos = 1;
  return x0;
}

__device__ __forceinline__ double np_double(NpPhilox& s) {
  return (double)(np_next(s) >> 11) * (1.0 / 9007199254740992.0);
}

__device__ double np_standard_normal(NpPhilox& s) {
  for (;;) {
    uint64_t r = np_next(s);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const uint64_t sign = r & 1;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZigWi[idx];
    if (sign) x = -x;
    if (rabs < kZigKi[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -kZigInvR * log1p(-np_double(s));
        const double yy = -log1p(-np_double(s));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
      }
    }
    if ((kZigFi[idx - 1] - kZigFi[idx]) * np_double(s) + kZigFi[idx] < exp(-0.5 * x * x)) return x;
  }
}

// ---------------------------------------------------------------------------
// Warp-parallel form (the default): one warp per run.  The stream is counter
// based, so word p of run r is Philox4x64-10(key, counter = p / 4 + 1)[p % 4]
// (numpy's counter is incremented before each block).  Each lane evaluates the
// ziggurat starting at position pos + lane of a 32-position window (the rare
// rejection loops read further positions), giving a value and the number of
// words it consumed; the normals of the stream start at pos, and at s + c(s)
// after each start s, so the lanes of a window that start normals are found
// with ballots (every lane up to the next multi-word lane starts one).  Same
// words, same arithmetic: bitwise the sequential walk.
__device__ __forceinline__ uint64_t np_word(uint64_t k0, uint64_t k1, uint64_t p) {
  const uint64_t blk = (p >> 2) + 1;  // counter words c1..c3 stay 0 below 2^64 blocks
  uint64_t x0 = blk, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPM0 * x0, hi0 = __umul64hi(kPM0, x0);
    const uint64_t lo1 = kPM1 * x2, hi1 = __umul64hi(kPM1, x2);
    x0 = hi1 ^ x1 ^ k0;
    x1 = lo1;
    x2 = hi0 ^ x3 ^ k1;
    x3 = lo0;
    k0 += kPW0;
    k1 += kPW1;
  }
  const int w = (int)(p & 3);
  return w == 0 ? x0 : w == 1 ? x1 : w == 2 ? x2 : x3;
}

// The ziggurat draw starting at word p (np_standard_normal's loop); *used =
// words consumed.
__device__ double np_normal_at(uint64_t k0, uint64_t k1, uint64_t p, int* used) {
  const uint64_t p0 = p;
  auto next = [&]() { return np_word(k0, k1, p++); };
  auto next_double = [&]() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); };
  for (;;) {
    uint64_t r = next();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const uint64_t sign = r & 1;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZigWi[idx];
    if (sign) x = -x;
    if (rabs < kZigKi[idx]) {
      *used = (int)(p - p0);
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = -kZigInvR * log1p(-next_double());
        const double yy = -log1p(-next_double());
        if (yy + yy > xx * xx) {
          *used = (int)(p - p0);
          return ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
        }
      }
    }
    if ((kZigFi[idx - 1] - kZigFi[idx]) * next_double() + kZigFi[idx] < exp(-0.5 * x * x)) {
      *used = (int)(p - p0);
      return x;
    }
  }
}

__global__ void ref_noise_warp_kernel(uint64_t seed, int64_t r0, int64_t R, int64_t count,
                                      double sigma, int scale, float* out32, double* out64) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= R) return;  // warp-uniform
  const uint64_t k0 = seed + (uint64_t)(r0 + r), k1 = 2ull;
  float* o32 = out32 ? out32 + r * count : nullptr;
  double* o64 = out64 ? out64 + r * count : nullptr;
  uint64_t pos = 0;
  int64_t k = 0;
  while (k < count) {
    int c;
    double z = np_normal_at(k0, k1, pos + (uint64_t)lane, &c);
    const unsigned multi = __ballot_sync(0xffffffffu, c != 1);
    // starts: from lane `cur`, every lane up to and including the next multi-word
    // lane starts a normal; that lane's consumption gives the next start
    unsigned starts = 0;
    int cur = 0;
    uint64_t next_pos = pos + 32;
    while (cur < 32) {
      const unsigned ahead = multi & (0xffffffffu << cur);
      if (!ahead) {
        starts |= 0xffffffffu << cur;
        break;
      }
      const int f = __ffs(ahead) - 1;
      starts |= (f == 31 ? 0xffffffffu : ((2u << f) - 1u)) & (0xffffffffu << cur);
      const int cf = __shfl_sync(0xffffffffu, c, f);
      cur = f + cf;
      if (cur >= 32) next_pos = pos + (uint64_t)cur;
    }
    const int rank = __popc(starts & ((1u << lane) - 1u));
    if (((starts >> lane) & 1u) && k + rank < count) {
      if (scale) z *= sigma;
      if (o32) o32[k + rank] = (float)z;
      if (o64) o64[k + rank] = z;
    }
    k += __popc(starts);
    pos = next_pos;
  }
}

// Run r (global index r0 + r) writes `count` = t_f * n draws, scaled by sigma
// in float64 exactly as _run does (skipped when sigma == 1, solver.py:240).
__global__ void ref_noise_kernel(uint64_t seed, int64_t r0, int64_t R, int64_t count, double sigma,
                                 int scale, float* out32, double* out64) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  NpPhilox s{0, 0, 0, 0, seed + (uint64_t)(r0 + r), 2ull, 0, 0, 0, 0, 4};
  float* o32 = out32 ? out32 + r * count : nullptr;
  double* o64 = out64 ? out64 + r * count : nullptr;
  for (int64_t i = 0; i < count; ++i) {
    double z = np_standard_normal(s);
    if (scale) z *= sigma;
    if (o32) o32[i] = (float)z;
    if (o64) o64[i] = z;
  }
}

}  // namespace

int launch_reference_noise(uint64_t seed, int64_t r0, int64_t R, int64_t count, double sigma,
                           float* out32, double* out64, cudaStream_t st) {
  static const char* seq_env = getenv("NMFA_REFNOISE_SEQ");  // A/B: one thread per run
  if (seq_env && seq_env[0] == '1') {
    const int threads = 64;
    ref_noise_kernel<<<(unsigned)((R + threads - 1) / threads), threads, 0, st>>>(
        seed, r0, R, count, sigma, sigma != 1.0, out32, out64);
  } else {
    const int threads = 256;  // 8 runs per block, one warp each
    ref_noise_warp_kernel<<<(unsigned)((R * 32 + threads - 1) / threads), threads, 0, st>>>(
        seed, r0, R, count, sigma, sigma != 1.0, out32, out64);
  }
  NMFA_LAUNCH_CHECK();
  return NMFA_OK;
}

}  // namespace nmfa

using namespace nmfa;

extern "C" int nmfa_reference_noise(uint64_t seed, int64_t r0, int64_t n_reads, int64_t count,
                                    double sigma, float* noise_dev, double* noise64_dev,
                                    void* stream) {
  try {
    if (n_reads < 1 || count < 1) {
      set_error("reference noise: n_reads and count must be positive");
      return NMFA_ERR_ARG;
    }
    if (!noise_dev && !noise64_dev) {
      set_error("reference noise: no output buffer");
      return NMFA_ERR_ARG;
    }
    if (!(sigma >= 0.0)) {
      set_error("sigma must be non-negative");
      return NMFA_ERR_ARG;
    }
    return launch_reference_noise(seed, r0, n_reads, count, sigma, noise_dev, noise64_dev,
                                  (cudaStream_t)stream);
  } catch (...) {
    set_error("internal error");
    return NMFA_ERR_STATE;
  }
}
