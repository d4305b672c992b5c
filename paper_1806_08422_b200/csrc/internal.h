// Internal (non-ABI) declarations shared by the C-ABI layer and the kernels.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nmfa_b200.h"

namespace nmfa {

void set_error(const std::string& msg);
void add_launches(int64_t k);

#define NMFA_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::nmfa::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                        __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");  \
      return NMFA_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define NMFA_LAUNCH_CHECK() NMFA_CUDA_TRY(cudaGetLastError())

constexpr int kSmallMaxN = 256;  // persistent path keeps J (<=128 KB fp16) in SMEM
// nmfa_problem_create_dense_bits builds the host edge list up to this many
// spins; larger complete +-1 instances are expanded on the device
constexpr int64_t kBitsHostMaxN = 4096;

}  // namespace nmfa

// Device-resident immutable problem (mirrors IsingProblem, problem.py:16-138).
struct nmfa_problem {
  int32_t device = 0;
  int64_t n = 0, n_edges = 0;
  double density = 0.0;
  bool is_dense = false;   // reference dispatch bit (problem.py:99)
  int32_t path = NMFA_PATH_SPARSE;
  int32_t field = NMFA_FIELD_FP16;  // dense-path GEMM operand precision (nmfa_problem_set_field_precision)
  bool j_exact = true;
  bool int_weights = true;
  bool has_field = false;  // some h_i != 0 (the energy's field term is skipped otherwise)
  double j_scale = 1.0;    // J_dev = J / j_scale (power of two); inv_norm carries j_scale
  double max_row_abs = 0.0; // max_i sum_j |J_ij| (exactness bound of tensor-core energies)
  int32_t np = 0;          // n padded to a multiple of 16 (tensor-core paths)
  // Row shard held on this device (dense path): spins [row_lo, row_hi) are the
  // rows of J stored here and the spins this device updates; the B image has
  // `brows` rows.  The whole problem is row_lo = 0, row_hi = n, brows = np.
  int64_t row_lo = 0, row_hi = 0;
  int32_t brows = 0;
  bool device_generated = false;  // on-device SK couplings: no edge list / CSR
  uint64_t sk_seed = 0;

  std::vector<double> h, norm_safe;  // host copies (float64)

  // per-spin epilogue constants, padded to np (zeros beyond n)
  float* d_invn = nullptr;  // j_scale / norm_safe
  float* d_hn = nullptr;    // h / norm_safe
  // small path: B-operand image of J (K-major, no swizzle), np x np fp16
  __half* d_j_small = nullptr;
  // dense path: J tiles (see anneal_dense.cu for the layout)
  __half* d_j_dense = nullptr;
  size_t j_dense_bytes = 0;
  // symmetric CSR, rows sorted by column (problem.py:78-88), J / j_scale in f32
  int32_t* d_csr_ptr = nullptr;
  int32_t* d_csr_idx = nullptr;
  float* d_csr_w = nullptr;
  // the same rows as ELL (max degree <= 4): ell_k slots per spin, rows padded
  // to a multiple of 8 spins, short rows padded with (own index, weight 0)
  int32_t ell_k = 0;
  // CSR kernel instance by the segment sizes of the 8-spin groups
  // (anneal_sparse.cu): 0 = up to 64 entries staged; 1 = mostly 65-96 (3
  // staged registers); 2 = mostly longer (3 registers + 3 entries per row per
  // round beyond the staged size)
  int32_t csr_variant = 0;
  int32_t* d_ell_idx = nullptr;
  float* d_ell_w = nullptr;
  // canonical upper edge list for the exact energy (problem.py:150-154)
  int32_t* d_e_i = nullptr;
  int32_t* d_e_j = nullptr;
  double* d_e_w = nullptr;
  double* d_h = nullptr;
  // one-shot entry points (nmfa_anneal / nmfa_anneal_host) reuse one cached
  // plan; the mutex serialises them (they are synchronous).
  std::mutex cache_mu;
  std::mutex host_mu;  // serialises nmfa_anneal_host calls (they share the cached buffers)
  nmfa_plan* cached_plan = nullptr;
  std::vector<double> cached_temps;
  double cached_alpha = -1.0, cached_sigma = -1.0;
  // nmfa_anneal_host: device result buffers + stream
  cudaStream_t host_stream = nullptr;
  int8_t* host_cfg = nullptr;
  double* host_e = nullptr;
  int64_t host_cap = 0;
};

struct nmfa_plan {
  const nmfa_problem* p = nullptr;
  int64_t R = 0;
  int32_t t_f = 0;
  int32_t path = 0;             // the problem's path when the plan was built
  int32_t field = 0;            // the problem's field precision when the plan was built
  float alpha = 0.f, oma = 0.f, sigma = 0.f;
  float* d_inv_temp = nullptr;  // [t_f]
  std::vector<float> h_inv_temp; // host copy (per-step launches read it)
  // sparse / dense per-step state
  int64_t Rp = 0;               // replica count padded for the state layout
  float* d_sa = nullptr;        // master state ping
  float* d_sb = nullptr;        // master state pong
  __half* d_h16a = nullptr;     // dense path operand ping
  __half* d_h16b = nullptr;     // dense path operand pong
  uint32_t* d_bits = nullptr;   // energy: packed config bits
  double* d_epart = nullptr;    // energy: partial sums
  int64_t energy_chunks = 0;
  int8_t* d_hist_cfg = nullptr; // trajectory energies: signs of s_hist
  int64_t bits_words = 0;       // capacity of d_bits in uint32
  void* dense = nullptr;        // DenseState (anneal_dense.cu)
  void* sparse = nullptr;       // SparseGraph (anneal_sparse.cu): captured step graph
};

namespace nmfa {
constexpr int kSmallHiloMaxNp = 224;  // small path + HILO field: J + 2 operand images in SMEM
// kernels (launchers return NMFA_OK or an error code)
int launch_small_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                        const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                        cudaStream_t st);
int launch_sparse_anneal(nmfa_plan* pl, uint64_t key_base, const float* noise,
                         const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                         cudaStream_t st);
void sparse_plan_free(nmfa_plan* pl);
int launch_dense_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                        const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                        double* energy, bool* energy_done, cudaStream_t st);
bool dense_energy_exact(const nmfa_problem* p);
int launch_small_anneal_many(const nmfa_problem* const* ps, int count, int64_t R, int t_f,
                             const float* d_inv_temp, float alpha, float sigma,
                             const uint64_t* key_bases, int8_t* cfg, cudaStream_t st);
int gset_parse(const char* text, int64_t len, int64_t* n_out, int64_t* m_out, int64_t* ei,
               int64_t* ej, double* w, int64_t cap);
int dense_set_exchange(nmfa_plan* pl, void* const* img0, void* const* img1, int world, int rank,
                       int64_t bytes);
int ground_state(const nmfa_problem* p, int max_n, double* energy, int64_t* degeneracy,
                 int8_t* config);
bool dense_is_sharded(const nmfa_problem* p);
int dense_run_sweeps(const nmfa_plan* pl, uint64_t key_base, const float* noise, const float* s0,
                     int8_t* cfg, float* s_out, float* s_hist, double* energy, int t_begin,
                     int t_end, bool energy_pass, cudaStream_t st);
int dense_image_info(const nmfa_plan* pl, void** img0, void** img1, int64_t* slice_bytes,
                     int32_t* n_slices, int32_t* slice_lo, int32_t* slice_hi);
int dense_read_config(const nmfa_plan* pl, int8_t* cfg, cudaStream_t st);
int dense_problem_generate_sk(nmfa_problem* p, uint64_t seed);
int dense_problem_from_bits(nmfa_problem* p, const uint32_t* d_bits);
int dense_energy_only(const nmfa_plan* pl, const int8_t* cfg, double* energy, cudaStream_t st);
int dense_plan_alloc(nmfa_plan* pl);
void dense_plan_free(nmfa_plan* pl);
int dense_problem_upload(nmfa_problem* p, const std::vector<float>& jdense_rowmajor);
int launch_energy(const nmfa_problem* p, const int8_t* cfg, int64_t n_cfg, double* energy,
                  uint32_t* bits_scratch, double* part_scratch, int64_t chunks,
                  cudaStream_t st);
int64_t energy_chunks_for(const nmfa_problem* p, int64_t n_cfg);
int launch_sign(const float* s, int64_t count, int8_t* cfg, cudaStream_t st);
int launch_best_of(const double* e, int64_t n, double* best_e, int64_t* best_i,
                   cudaStream_t st);
}  // namespace nmfa

#ifdef NMFA_GUARD
// Checked build: every device allocation goes through the redzone allocator
// (guard.cu).  Defined last, after the CUDA runtime declarations, so only the
// library's own call sites are redirected.
namespace nmfa {
cudaError_t guard_malloc(void** p, size_t n);
cudaError_t guard_free(void* p);
cudaError_t guard_malloc_async(void** p, size_t n, cudaStream_t st);
cudaError_t guard_free_async(void* p, cudaStream_t st);
}  // namespace nmfa
#define cudaMalloc(p, n) ::nmfa::guard_malloc(reinterpret_cast<void**>(p), (size_t)(n))
#define cudaFree(p) ::nmfa::guard_free((void*)(p))
#define cudaMallocAsync(p, n, st) ::nmfa::guard_malloc_async(reinterpret_cast<void**>(p), (size_t)(n), (st))
#define cudaFreeAsync(p, st) ::nmfa::guard_free_async((void*)(p), (st))
#endif
