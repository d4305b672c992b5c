// Checked build (compiled with -DNMFA_GUARD into libnmfa_b200_guard.so): the
// memcheck / racecheck substitute on pools where compute-sanitizer is closed.
//
// * Every device allocation the library makes (cudaMalloc / cudaMallocAsync in
//   the sources, redirected by internal.h) gets a 4 KB redzone on each side
//   filled with kGuardByte; the body is poisoned with 0xFF bytes (NaN in fp16
//   and fp32) so a kernel that reads memory nobody wrote changes its results.
// * Redzones are verified when the allocation is freed and on demand through
//   nmfa_debug_guard_check(), which returns the number of corrupted bytes seen.
// * common.cuh's NMFA_JITTER sleeps a pseudo-random time at the protocol points
//   of the persistent kernels (producer before each TMA, MMA issuer before each
//   k-slice, epilogue before publishing), so a missing fence or readiness
//   check shows up as a result that differs from the unchecked library.
// The unchecked library exports the same symbol and returns -1 from it.
#include <map>

#include "internal.h"

#ifdef NMFA_GUARD
namespace nmfa {
namespace {
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5, kPoisonByte = 0xFF;
std::mutex g_mu;
std::map<uintptr_t, size_t> g_live;  // user pointer -> user bytes
int64_t g_bad = 0;                   // corrupted redzone bytes found so far
std::string g_first;                 // description of the first violation

int64_t check_locked(uintptr_t p, size_t n) {
  std::vector<unsigned char> lo(kGuard), hi(kGuard);
  const char* base = reinterpret_cast<const char*>(p);
  if ((cudaMemcpy)(lo.data(), base - kGuard, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
      (cudaMemcpy)(hi.data(), base + n, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  int64_t bad = 0;
  for (size_t k = 0; k < kGuard; ++k) {
    if (lo[k] != kGuardByte) {
      if (!bad && g_first.empty())
        g_first = "write " + std::to_string(kGuard - k) + " bytes before a " + std::to_string(n) +
                  "-byte allocation";
      ++bad;
    }
    if (hi[k] != kGuardByte) {
      if (!bad && g_first.empty())
        g_first = "write " + std::to_string(k) + " bytes past the end of a " + std::to_string(n) +
                  "-byte allocation";
      ++bad;
    }
  }
  return bad;
}
}  // namespace

cudaError_t guard_malloc(void** p, size_t n) {
  void* raw = nullptr;
  cudaError_t e = (cudaMalloc)(&raw, n + 2 * kGuard);
  if (e != cudaSuccess) return e;
  char* b = static_cast<char*>(raw);
  (cudaMemset)(b, kGuardByte, kGuard);
  (cudaMemset)(b + kGuard, kPoisonByte, n);
  (cudaMemset)(b + kGuard + n, kGuardByte, kGuard);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  *p = b + kGuard;
  std::lock_guard<std::mutex> lk(g_mu);
  g_live[reinterpret_cast<uintptr_t>(*p)] = n;
  return cudaSuccess;
}

cudaError_t guard_free(void* p) {
  if (!p) return cudaSuccess;
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_live.find(reinterpret_cast<uintptr_t>(p));
  if (it == g_live.end()) return (cudaFree)(p);  // not ours (never happens in-library)
  g_bad += check_locked(it->first, it->second);
  g_live.erase(it);
  return (cudaFree)(static_cast<char*>(p) - kGuard);
}

cudaError_t guard_malloc_async(void** p, size_t n, cudaStream_t st) {
  cudaStreamSynchronize(st);
  return guard_malloc(p, n);
}

cudaError_t guard_free_async(void* p, cudaStream_t st) {
  cudaStreamSynchronize(st);
  return guard_free(p);
}
}  // namespace nmfa

extern "C" int64_t nmfa_debug_guard_check(void) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(nmfa::g_mu);
  int64_t bad = nmfa::g_bad;
  for (const auto& kv : nmfa::g_live) bad += nmfa::check_locked(kv.first, kv.second);
  if (bad) nmfa::set_error("redzone corrupted: " + nmfa::g_first);
  return bad;
}
#else
extern "C" int64_t nmfa_debug_guard_check(void) { return -1; }
#endif
