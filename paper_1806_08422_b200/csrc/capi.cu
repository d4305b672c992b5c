// C-ABI layer: problem construction (problem.py:25-116 restated in C++),
// plans, dispatch to the kernel paths, errors.  See include/nmfa_b200.h.
#include <algorithm>
#include <new>
#include <stdexcept>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "internal.h"

namespace nmfa {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
void add_launches(int64_t k) { g_launches += k; }

static int arg_error(const std::string& msg) {
  set_error(msg);
  return NMFA_ERR_ARG;
}

static int state_error(const std::string& msg) {
  set_error(msg);
  return NMFA_ERR_STATE;
}

template <class T>
static int upload(T** dst, const T* src, size_t count) {
  if (count == 0) count = 1;  // keep a valid pointer for empty arrays
  NMFA_CUDA_TRY(cudaMalloc(dst, count * sizeof(T)));
  if (src) NMFA_CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
  return NMFA_OK;
}

// Path choice is internal (the reference picks dense vs CSR by density alone,
// problem.py:97-99).  Measured on B200, R = 1024 (profiles/r01/path_crossover.log):
// * graphs of max degree <= 4 (ELL kernel) beat the tensor-core path at every
//   n >= 512 (1.4x at n = 512, 6.5x at n = 16384);
// * otherwise the tcgen05 path costs ~n^2 R / 5.5e14 s per sweep and the CSR
//   gather ~nnz R / 9e11 s, so dense wins while n^2 < 611 nnz (er_d10: dense
//   at n = 4096, CSR from n = 8192; er_d20: CSR from n = 16384); the fp16 J
//   image is capped at 1 GiB.
static bool prefer_dense(int64_t n, int64_t n_edges, int32_t ell_k) {
  if (ell_k > 0) return false;
  const double dense_cost = (double)n * (double)n / 5.5e14;
  const double sparse_cost = 2.0 * (double)n_edges / 9e11;
  return (double)n * (double)n * 2.0 <= 1073741824.0 && dense_cost < sparse_cost;
}

static bool exact_in_half(double v) {
  __half h = __double2half(v);
  return (double)__half2float(h) == v;
}

}  // namespace nmfa

using namespace nmfa;

extern "C" {

// Every entry point converts C++ exceptions (host allocation failures above
// all) into status codes: nothing may unwind across the C ABI.
#define NMFA_API_BEGIN try {
#define NMFA_API_END                                                          \
  }                                                                           \
  catch (const std::bad_alloc&) {                                             \
    nmfa::set_error("host out of memory");                                    \
    return NMFA_ERR_STATE;                                                    \
  }                                                                           \
  catch (const std::exception& ex) {                                          \
    nmfa::set_error(std::string("internal error: ") + ex.what());             \
    return NMFA_ERR_STATE;                                                    \
  }                                                                           \
  catch (...) {                                                               \
    nmfa::set_error("internal error");                                        \
    return NMFA_ERR_STATE;                                                    \
  }

const char* nmfa_last_error(void) { return g_err.c_str(); }
const char* nmfa_version(void) { return "nmfa_b200 0.1.0 (sm_100a)"; }
int64_t nmfa_last_launch_count(void) { return g_launches; }

int nmfa_problem_destroy(nmfa_problem_t* p) {
  NMFA_API_BEGIN
  if (!p) return NMFA_OK;
  if (p->cached_plan) nmfa_plan_destroy(p->cached_plan);
  if (p->host_cfg) cudaFree(p->host_cfg);
  if (p->host_e) cudaFree(p->host_e);
  if (p->host_stream) cudaStreamDestroy(p->host_stream);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  void* bufs[] = {p->d_invn, p->d_hn,    p->d_j_small, p->d_j_dense, p->d_csr_ptr, p->d_csr_idx,
                  p->d_csr_w, p->d_e_i, p->d_e_j,     p->d_e_w,     p->d_h,
                  p->d_ell_idx, p->d_ell_w};
  for (void* b : bufs)
    if (b) cudaFree(b);
  cudaSetDevice(prev);
  delete p;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_create(int64_t n, int64_t n_edges, const int64_t* ei_in, const int64_t* ej_in,
                        const double* w_in, const double* h_in, int32_t device,
                        nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out) return arg_error("out pointer is NULL");
  *out = nullptr;
  // ---- validation, problem.py:25-62 ----
  if (n < 1) return arg_error("spin count must be positive, got " + std::to_string(n));
  if (n > (int64_t)1 << 30) return arg_error("spin count too large");
  if (n_edges < 0) return arg_error("couplers must be a sequence of (i, j, w) triples");
  if (n_edges > 0 && (!ei_in || !ej_in || !w_in))
    return arg_error("coupler arrays are NULL");
  std::vector<double> h(n, 0.0);
  if (h_in) {
    for (int64_t i = 0; i < n; ++i) {
      if (!std::isfinite(h_in[i])) return arg_error("h contains non-finite entries");
      h[i] = h_in[i];
    }
  }
  std::vector<int64_t> lo(n_edges), hi(n_edges);
  std::vector<double> w(n_edges);
  bool sorted = true;
  for (int64_t k = 0; k < n_edges; ++k) {
    int64_t a = ei_in[k], b = ej_in[k];
    if (a < 0 || a >= n || b < 0 || b >= n)
      return arg_error("coupler index out of range [0, " + std::to_string(n) + ")");
    if (a == b) return arg_error("self-couplings are not allowed");
    if (!std::isfinite(w_in[k])) return arg_error("coupler weights must be finite");
    if (w_in[k] == 0.0) return arg_error("coupler weights must be nonzero");
    lo[k] = std::min(a, b);
    hi[k] = std::max(a, b);
    w[k] = w_in[k];
    if (k > 0 && (lo[k] < lo[k - 1] || (lo[k] == lo[k - 1] && hi[k] <= hi[k - 1])))
      sorted = false;
  }
  if (!sorted) {  // canonical order: lexicographic (lo, hi), problem.py:63-66
    std::vector<int64_t> perm(n_edges);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) {
      return lo[x] != lo[y] ? lo[x] < lo[y] : hi[x] < hi[y];
    });
    std::vector<int64_t> lo2(n_edges), hi2(n_edges);
    std::vector<double> w2(n_edges);
    for (int64_t k = 0; k < n_edges; ++k) {
      lo2[k] = lo[perm[k]];
      hi2[k] = hi[perm[k]];
      w2[k] = w[perm[k]];
    }
    lo.swap(lo2);
    hi.swap(hi2);
    w.swap(w2);
  }
  for (int64_t k = 1; k < n_edges; ++k)
    if (lo[k] == lo[k - 1] && hi[k] == hi[k - 1])
      return arg_error("duplicate coupler (" + std::to_string(lo[k]) + ", " +
                       std::to_string(hi[k]) + ")");

  auto* p = new nmfa_problem();
  p->device = device;
  p->n = n;
  p->n_edges = n_edges;
  int64_t pairs = n * (n - 1) / 2;
  p->density = pairs == 0 ? 0.0 : (double)n_edges / (double)pairs;
  p->is_dense = p->density > 0.5;
  p->h = h;

  // ---- symmetric CSR, rows sorted by column (problem.py:78-88) ----
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t k = 0; k < n_edges; ++k) {
    cnt[lo[k] + 1]++;
    cnt[hi[k] + 1]++;
  }
  std::vector<int64_t> ptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + cnt[i + 1];
  if (ptr[n] > INT32_MAX) {
    delete p;
    return arg_error("too many couplers for the int32 CSR");
  }
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  std::vector<int32_t> cidx(ptr[n]);
  std::vector<double> cw(ptr[n]);
  // columns below the row first (edges with hi == row, increasing lo) ...
  for (int64_t k = 0; k < n_edges; ++k) {
    int64_t r = hi[k];
    cidx[fill[r]] = (int32_t)lo[k];
    cw[fill[r]++] = w[k];
  }
  // ... then columns above it (edges with lo == row, increasing hi)
  for (int64_t k = 0; k < n_edges; ++k) {
    int64_t r = lo[k];
    cidx[fill[r]] = (int32_t)hi[k];
    cw[fill[r]++] = w[k];
  }
  // ---- normalizers: np.bincount order (lo pass, then hi pass), problem.py:90-95 ----
  std::vector<double> sq(n, 0.0);
  for (int64_t k = 0; k < n_edges; ++k) sq[lo[k]] += w[k] * w[k];
  for (int64_t k = 0; k < n_edges; ++k) sq[hi[k]] += w[k] * w[k];
  p->norm_safe.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    double nr = std::sqrt(h[i] * h[i] + sq[i]);
    p->norm_safe[i] = nr == 0.0 ? 1.0 : nr;
  }

  // ---- operand precision: J / 2^e exact in fp16? ----
  double wmax = 0.0;
  bool ints = true;
  for (int64_t k = 0; k < n_edges; ++k) {
    wmax = std::max(wmax, std::fabs(w[k]));
    if (w[k] != std::floor(w[k])) ints = false;
  }
  for (int64_t i = 0; i < n; ++i)
    if (h[i] != std::floor(h[i])) ints = false;
  p->int_weights = ints;
  for (int64_t i = 0; i < n && !p->has_field; ++i) p->has_field = h[i] != 0.0;
  double scale = 1.0;
  if (wmax > 0.0) {
    bool exact1 = wmax <= 2048.0;
    for (int64_t k = 0; k < n_edges && exact1; ++k) exact1 = exact_in_half(w[k]);
    if (!exact1) scale = std::ldexp(1.0, (int)std::ceil(std::log2(wmax)));  // |J/scale| <= 1
  }
  p->j_scale = scale;
  {
    std::vector<double> rs(n, 0.0);
    for (int64_t k = 0; k < n_edges; ++k) {
      rs[lo[k]] += std::fabs(w[k]);
      rs[hi[k]] += std::fabs(w[k]);
    }
    for (int64_t i = 0; i < n; ++i) p->max_row_abs = std::max(p->max_row_abs, rs[i]);
  }
  bool jex = true;
  for (int64_t k = 0; k < n_edges && jex; ++k) jex = exact_in_half(w[k] / scale);
  p->j_exact = jex;

  int err = NMFA_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    delete p;
    return arg_error("invalid CUDA device " + std::to_string(device));
  }
  do {
    p->np = (int32_t)((n + 15) / 16 * 16);
    std::vector<float> invn(p->np, 0.f), hn(p->np, 0.f);
    for (int64_t i = 0; i < n; ++i) {
      invn[i] = (float)(scale / p->norm_safe[i]);
      hn[i] = (float)(h[i] / p->norm_safe[i]);
    }
    if ((err = upload(&p->d_invn, invn.data(), invn.size()))) break;
    if ((err = upload(&p->d_hn, hn.data(), hn.size()))) break;

    std::vector<int32_t> ptr32(n + 1);
    for (int64_t i = 0; i <= n; ++i) ptr32[i] = (int32_t)ptr[i];
    std::vector<float> cw32(cw.size());
    for (size_t k = 0; k < cw.size(); ++k) cw32[k] = (float)(cw[k] / scale);
    if ((err = upload(&p->d_csr_ptr, ptr32.data(), ptr32.size()))) break;
    if ((err = upload(&p->d_csr_idx, cidx.data(), cidx.size()))) break;
    if ((err = upload(&p->d_csr_w, cw32.data(), cw32.size()))) break;
    {
      // CSR kernel variant by segment size per 8-spin group (anneal_sparse.cu):
      // the 3-register staged kernel when more groups need 65-96 entries than
      // fit the 2-register one (33-64): measured +18% at degree 10, -5..9% at 5;
      // mostly longer segments: also 3 entries per row per round
      int64_t mid = 0, big = 0, huge = 0;
      for (int64_t g = 0; g * 8 < n; ++g) {
        const int64_t seg = ptr[std::min(n, g * 8 + 8)] - ptr[g * 8];
        mid += seg > 32 && seg <= 64;
        big += seg > 64 && seg <= 96;
        huge += seg > 96;
      }
      p->csr_variant = huge > std::max(mid, big) ? 2 : big > mid ? 1 : 0;
    }
    {
      // ELL copy of the CSR rows for low-degree graphs (anneal_sparse.cu). A
      // zero-weight pad slot leaves the row sum bit-identical: the sum starts
      // at +0 and fmaf(0, v, s) == s for every s that can occur (never -0).
      int64_t max_deg = 0;
      for (int64_t i = 0; i < n; ++i) max_deg = std::max(max_deg, ptr[i + 1] - ptr[i]);
      const int64_t n8 = (n + 7) / 8 * 8;
      if (n > 0 && max_deg <= 4 && n8 * 4 <= INT32_MAX) {
        const int k = max_deg <= 3 ? 3 : 4;
        std::vector<int32_t> ei((size_t)(n8 * k));
        std::vector<float> ew((size_t)(n8 * k), 0.f);
        for (int64_t i = 0; i < n8; ++i)
          for (int u = 0; u < k; ++u) {
            const int64_t e = ptr[std::min(i, n - 1)] + u;
            const bool real = i < n && e < ptr[i + 1];
            ei[i * k + u] = real ? cidx[e] : (int32_t)std::min(i, n - 1);
            ew[i * k + u] = real ? cw32[e] : 0.f;
          }
        if ((err = upload(&p->d_ell_idx, ei.data(), ei.size()))) break;
        if ((err = upload(&p->d_ell_w, ew.data(), ew.size()))) break;
        p->ell_k = k;
      }
    }

    std::vector<int32_t> e_i(n_edges), e_j(n_edges);
    for (int64_t k = 0; k < n_edges; ++k) {
      e_i[k] = (int32_t)lo[k];
      e_j[k] = (int32_t)hi[k];
    }
    if ((err = upload(&p->d_e_i, e_i.data(), e_i.size()))) break;
    if ((err = upload(&p->d_e_j, e_j.data(), e_j.size()))) break;
    if ((err = upload(&p->d_e_w, w.data(), w.size()))) break;
    if ((err = upload(&p->d_h, h.data(), h.size()))) break;

    if (n <= kSmallMaxN) {
      // B operand image for the persistent kernel: B[row=i][k=j] = J_ij / scale
      const uint32_t np = (uint32_t)p->np, lbo = np * 16u;
      std::vector<__half> img((size_t)np * np, __float2half(0.f));
      for (int64_t k = 0; k < n_edges; ++k) {
        __half v = __double2half(w[k] / scale);
        img[kmajor_off((uint32_t)lo[k], (uint32_t)hi[k], lbo) / 2] = v;
        img[kmajor_off((uint32_t)hi[k], (uint32_t)lo[k], lbo) / 2] = v;
      }
      if ((err = upload(&p->d_j_small, img.data(), img.size()))) break;
      p->path = NMFA_PATH_SMALL;
    } else if (prefer_dense(n, n_edges, p->ell_k)) {
      std::vector<float> jd((size_t)n * n, 0.f);
      for (int64_t k = 0; k < n_edges; ++k) {
        float v = (float)(w[k] / scale);
        jd[(size_t)lo[k] * n + hi[k]] = v;
        jd[(size_t)hi[k] * n + lo[k]] = v;
      }
      if ((err = dense_problem_upload(p, jd))) break;
      p->path = NMFA_PATH_DENSE;
    } else {
      p->path = NMFA_PATH_SPARSE;
    }
  } while (0);
  cudaSetDevice(prev);
  if (err) {
    nmfa_problem_destroy(p);
    return err;
  }
  *out = p;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_create_dense(int64_t n, const double* J, const double* h, int32_t device,
                              nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out || !J) return arg_error("NULL argument");
  *out = nullptr;
  if (n < 1) return arg_error("spin count must be positive, got " + std::to_string(n));
  if (n > (int64_t)1 << 20) return arg_error("spin count too large for a dense matrix");
  std::vector<int64_t> ei, ej;
  std::vector<double> w;
  for (int64_t i = 0; i < n; ++i) {
    if (J[i * n + i] != 0.0) return arg_error("self-couplings are not allowed");
    for (int64_t j = i + 1; j < n; ++j) {
      const double a = J[i * n + j];
      if (a != J[j * n + i]) return arg_error("J must be symmetric");
      if (a != 0.0) {
        ei.push_back(i);
        ej.push_back(j);
        w.push_back(a);
      }
    }
  }
  return nmfa_problem_create(n, (int64_t)w.size(), ei.data(), ej.data(), w.data(), h, device, out);
  NMFA_API_END
}

int nmfa_problem_create_csr(int64_t n, const int64_t* indptr, const int64_t* indices,
                            const double* weights, const double* h, int32_t device,
                            nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out || !indptr || !indices || !weights) return arg_error("NULL argument");
  *out = nullptr;
  if (n < 1) return arg_error("spin count must be positive, got " + std::to_string(n));
  if (indptr[0] != 0) return arg_error("indptr must start at 0");
  std::vector<int64_t> ei, ej;
  std::vector<double> w;
  int64_t lower = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (indptr[i + 1] < indptr[i]) return arg_error("indptr must be nondecreasing");
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int64_t j = indices[k];
      if (j < 0 || j >= n) return arg_error("coupler index out of range [0, " + std::to_string(n) + ")");
      if (j > i) {
        ei.push_back(i);
        ej.push_back(j);
        w.push_back(weights[k]);
      } else if (j < i) {
        ++lower;
      } else {
        return arg_error("self-couplings are not allowed");
      }
    }
  }
  if (lower != (int64_t)w.size()) return arg_error("the CSR must be symmetric (problem.py:78-88)");
  return nmfa_problem_create(n, (int64_t)w.size(), ei.data(), ej.data(), w.data(), h, device, out);
  NMFA_API_END
}

int nmfa_problem_create_dense_bits(int64_t n, const uint32_t* sign_bits, const double* h,
                                   int32_t device, nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out || !sign_bits) return arg_error("NULL argument");
  *out = nullptr;
  if (n < 2) return arg_error("a complete +-1 graph needs n >= 2, got " + std::to_string(n));
  // beyond kBitsHostMaxN spins the n(n-1)/2-entry host edge list is not built:
  // the bits go to the device and are expanded there (dense path only)
  if (n > kBitsHostMaxN) return nmfa_problem_create_bits_device(n, sign_bits, h, 0, n, device, out);
  const int64_t m = n * (n - 1) / 2;
  std::vector<int64_t> ei((size_t)m), ej((size_t)m);
  std::vector<double> w((size_t)m);
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j, ++k) {
      const uint64_t b = (uint64_t)i * (uint64_t)n + (uint64_t)j;  // row-major bit (i, j), i < j
      ei[k] = i;
      ej[k] = j;
      w[k] = ((sign_bits[b >> 5] >> (b & 31)) & 1u) ? 1.0 : -1.0;
    }
  return nmfa_problem_create(n, m, ei.data(), ej.data(), w.data(), h, device, out);
  NMFA_API_END
}

int nmfa_problem_create_bits_device(int64_t n, const uint32_t* sign_bits, const double* h,
                                    int64_t row_lo, int64_t row_hi, int32_t device,
                                    nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out || !sign_bits) return arg_error("NULL argument");
  *out = nullptr;
  if (n < 2) return arg_error("a complete +-1 graph needs n >= 2, got " + std::to_string(n));
  if (n > (int64_t)1 << 20) return arg_error("spin count too large for the dense path");
  if (row_lo < 0 || row_hi > n || row_lo >= row_hi)
    return arg_error("row shard must satisfy 0 <= row_lo < row_hi <= n");
  if (row_lo % 128 != 0 || (row_hi % 128 != 0 && row_hi != n))
    return arg_error("row shard boundaries must be multiples of 128 (or n)");
  auto* p = new nmfa_problem();
  p->device = device;
  p->n = n;
  p->n_edges = n * (n - 1) / 2;
  p->density = 1.0;
  p->is_dense = true;
  p->path = NMFA_PATH_DENSE;
  p->int_weights = true;
  p->j_exact = true;
  p->j_scale = 1.0;
  p->device_generated = true;
  p->h.assign(n, 0.0);
  if (h)
    for (int64_t i = 0; i < n; ++i) {
      if (!std::isfinite(h[i])) {
        delete p;
        return arg_error("fields must be finite");
      }
      p->h[i] = h[i];
      p->has_field = p->has_field || h[i] != 0.0;
    }
  // normalizers_safe = sqrt(h^2 + sum_j J_ij^2) (problem.py:90-95): n - 1 unit couplers per row
  p->norm_safe.resize(n);
  double max_h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    p->norm_safe[i] = std::sqrt(p->h[i] * p->h[i] + (double)(n - 1));
    max_h = std::max(max_h, std::fabs(p->h[i]));
  }
  p->max_row_abs = (double)(n - 1);
  p->row_lo = row_lo;
  p->row_hi = row_hi;
  p->brows = (int32_t)((row_hi - row_lo + 15) / 16 * 16);
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    delete p;
    return arg_error("invalid CUDA device " + std::to_string(device));
  }
  int err = NMFA_OK;
  uint32_t* d_bits = nullptr;
  do {
    p->np = (int32_t)((n + 15) / 16 * 16);
    std::vector<float> invn(p->np, 0.f), hn(p->np, 0.f);
    for (int64_t i = 0; i < n; ++i) {
      invn[i] = (float)(1.0 / p->norm_safe[i]);
      hn[i] = (float)(p->h[i] / p->norm_safe[i]);
    }
    if ((err = upload(&p->d_invn, invn.data(), invn.size()))) break;
    if ((err = upload(&p->d_hn, hn.data(), hn.size()))) break;
    if ((err = upload(&p->d_h, p->h.data(), p->h.size()))) break;
    const size_t words = (size_t)(((unsigned long long)n * (unsigned long long)n + 31) / 32);
    if ((err = upload(&d_bits, sign_bits, words))) break;
    err = dense_problem_from_bits(p, d_bits);
  } while (0);
  if (d_bits) cudaFree(d_bits);
  cudaSetDevice(prev);
  if (err) {
    nmfa_problem_destroy(p);
    return err;
  }
  *out = p;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_create_sk_device(int64_t n, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                  int32_t device, nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!out) return arg_error("out pointer is NULL");
  *out = nullptr;
  if (n < 2) return arg_error("sk generator needs n >= 2, got " + std::to_string(n));
  if (n > (int64_t)1 << 20) return arg_error("spin count too large for the dense path");
  if (row_lo < 0 || row_hi > n || row_lo >= row_hi)
    return arg_error("row shard must satisfy 0 <= row_lo < row_hi <= n");
  if (row_lo % 128 != 0 || (row_hi % 128 != 0 && row_hi != n))
    return arg_error("row shard boundaries must be multiples of 128 (or n)");
  auto* p = new nmfa_problem();
  p->device = device;
  p->n = n;
  p->n_edges = n * (n - 1) / 2;
  p->density = 1.0;
  p->is_dense = true;
  p->path = NMFA_PATH_DENSE;
  p->int_weights = true;
  p->j_exact = true;
  p->j_scale = 1.0;
  p->max_row_abs = (double)(n - 1);
  p->device_generated = true;
  p->sk_seed = seed;
  p->h.assign(n, 0.0);
  p->norm_safe.assign(n, std::sqrt((double)(n - 1)));  // every row holds n-1 couplings of |w| = 1
  p->row_lo = row_lo;
  p->row_hi = row_hi;
  p->brows = (int32_t)((row_hi - row_lo + 15) / 16 * 16);
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    delete p;
    return arg_error("invalid CUDA device " + std::to_string(device));
  }
  int err = NMFA_OK;
  do {
    p->np = (int32_t)((n + 15) / 16 * 16);
    std::vector<float> invn(p->np, 0.f), hn(p->np, 0.f);
    for (int64_t i = 0; i < n; ++i) invn[i] = (float)(1.0 / p->norm_safe[i]);
    if ((err = upload(&p->d_invn, invn.data(), invn.size()))) break;
    if ((err = upload(&p->d_hn, hn.data(), hn.size()))) break;
    if ((err = upload(&p->d_h, p->h.data(), p->h.size()))) break;
    err = dense_problem_generate_sk(p, seed);
  } while (0);
  cudaSetDevice(prev);
  if (err) {
    nmfa_problem_destroy(p);
    return err;
  }
  *out = p;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_get_info(const nmfa_problem_t* p, nmfa_problem_info_t* info) {
  NMFA_API_BEGIN
  if (!p || !info) return arg_error("NULL argument");
  info->n = p->n;
  info->n_edges = p->n_edges;
  info->density = p->density;
  info->is_dense = p->is_dense;
  info->path = p->path;
  info->j_exact = p->j_exact;
  info->int_weights = p->int_weights;
  info->j_scale = p->j_scale;
  info->ell_slots = p->ell_k;
  info->field = p->field;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_set_field_precision(nmfa_problem_t* p, int32_t field) {
  NMFA_API_BEGIN
  if (!p) return arg_error("NULL problem");
  if (field != NMFA_FIELD_FP16 && field != NMFA_FIELD_HILO)
    return arg_error("unknown field precision " + std::to_string(field));
  std::lock_guard<std::mutex> lock(p->cache_mu);
  if (field == NMFA_FIELD_HILO && p->path == NMFA_PATH_SMALL && p->np > kSmallHiloMaxNp)
    return arg_error("field precision HILO on the small path needs n <= 224 (J and two operand "
                     "images in shared memory); set_path('dense') first");
  if (field == NMFA_FIELD_HILO && p->d_j_dense && (p->row_lo != 0 || p->row_hi != p->n))
    return arg_error("field precision HILO is not available on a row shard");
  if (p->cached_plan) {  // the cached plan was built with the old precision
    nmfa_plan_destroy(p->cached_plan);
    p->cached_plan = nullptr;
  }
  p->field = field;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_problem_set_path(nmfa_problem_t* p, int32_t path) {
  NMFA_API_BEGIN
  if (!p) return arg_error("NULL problem");
  if (path < 0 || path > 2) return arg_error("unknown path");
  std::lock_guard<std::mutex> lock(p->cache_mu);
  if (p->cached_plan) {  // a cached plan holds the old path's buffers
    nmfa_plan_destroy(p->cached_plan);
    p->cached_plan = nullptr;
  }
  if (p->device_generated && path != NMFA_PATH_DENSE)
    return arg_error("a device-generated problem only runs the dense path");
  if (path == NMFA_PATH_SMALL && !p->d_j_small)
    return arg_error("small path needs n <= 256");
  if (path == NMFA_PATH_SMALL && p->field == NMFA_FIELD_HILO && p->np > kSmallHiloMaxNp)
    return arg_error("field precision HILO on the small path needs n <= 224; set the field "
                     "precision to FP16 first");
  if (path == NMFA_PATH_DENSE && !p->d_j_dense) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    std::vector<float> jd((size_t)p->n * p->n, 0.f);
    std::vector<int32_t> e_i(p->n_edges), e_j(p->n_edges);
    std::vector<double> w(p->n_edges);
    int err = NMFA_OK;
    if (p->n_edges) {
      if (cudaMemcpy(e_i.data(), p->d_e_i, 4 * p->n_edges, cudaMemcpyDeviceToHost) ||
          cudaMemcpy(e_j.data(), p->d_e_j, 4 * p->n_edges, cudaMemcpyDeviceToHost) ||
          cudaMemcpy(w.data(), p->d_e_w, 8 * p->n_edges, cudaMemcpyDeviceToHost))
        err = NMFA_ERR_CUDA;
    }
    if (!err) {
      for (int64_t k = 0; k < p->n_edges; ++k) {
        float v = (float)(w[k] / p->j_scale);
        jd[(size_t)e_i[k] * p->n + e_j[k]] = v;
        jd[(size_t)e_j[k] * p->n + e_i[k]] = v;
      }
      err = dense_problem_upload(p, jd);
    }
    cudaSetDevice(prev);
    if (err) {
      if (err == NMFA_ERR_CUDA && g_err.empty()) set_error("dense upload failed");
      return err;
    }
  }
  p->path = path;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_plan_destroy(nmfa_plan_t* pl) {
  NMFA_API_BEGIN
  if (!pl) return NMFA_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->p->device);
  void* bufs[] = {pl->d_inv_temp, pl->d_sa,    pl->d_sb,       pl->d_h16a,
                  pl->d_h16b,     pl->d_bits,  pl->d_epart,    pl->d_hist_cfg};
  for (void* b : bufs)
    if (b) cudaFree(b);
  dense_plan_free(pl);
  sparse_plan_free(pl);
  cudaSetDevice(prev);
  delete pl;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_plan_create(const nmfa_problem_t* p, int64_t R, int32_t t_f, const double* temps,
                     double alpha, double sigma, nmfa_plan_t** out) {
  NMFA_API_BEGIN
  if (!p || !out) return arg_error("NULL argument");
  *out = nullptr;
  if (R < 1) return arg_error("n_runs must be at least 1, got " + std::to_string(R));
  if (t_f < 1) return arg_error("t_f must be at least 1, got " + std::to_string(t_f));
  if (!(alpha >= 0.0 && alpha <= 1.0))
    return arg_error("alpha must be in [0, 1], got " + std::to_string(alpha));
  if (!(sigma >= 0.0)) return arg_error("sigma must be nonnegative, got " + std::to_string(sigma));
  if (!temps) return arg_error("temps is NULL");
  std::vector<float> inv_t(t_f);
  for (int32_t t = 0; t < t_f; ++t) {
    if (!(temps[t] > 0.0) || !std::isfinite(temps[t]))
      return arg_error("temperature must be positive, got " + std::to_string(temps[t]));
    inv_t[t] = (float)(1.0 / temps[t]);
  }
  auto* pl = new nmfa_plan();
  pl->p = p;
  pl->R = R;
  pl->t_f = t_f;
  pl->path = p->path;
  pl->field = p->path != NMFA_PATH_SPARSE ? p->field : NMFA_FIELD_FP16;
  pl->alpha = (float)alpha;
  pl->oma = (float)(1.0 - alpha);
  pl->sigma = (float)sigma;
  pl->h_inv_temp = inv_t;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  int err = NMFA_OK;
  do {
    if ((err = upload(&pl->d_inv_temp, inv_t.data(), inv_t.size()))) break;
    if (p->path == NMFA_PATH_SPARSE) {
      pl->Rp = (R + 31) / 32 * 32;
      size_t bytes = (size_t)p->n * pl->Rp * sizeof(float);
      if (cudaMalloc(&pl->d_sa, bytes) != cudaSuccess || cudaMalloc(&pl->d_sb, bytes) != cudaSuccess) {
        set_error("out of device memory for sparse state");
        err = NMFA_ERR_CUDA;
        break;
      }
    } else if (p->path == NMFA_PATH_DENSE) {
      if ((err = dense_plan_alloc(pl))) break;
    }
    int64_t chunks = energy_chunks_for(p, R);
    pl->energy_chunks = chunks;
    pl->bits_words = p->n * ((R + 31) / 32);
    if (cudaMalloc(&pl->d_bits, pl->bits_words * 4) != cudaSuccess ||
        cudaMalloc(&pl->d_epart, (size_t)(chunks + 1) * R * 8) != cudaSuccess) {
      set_error("out of device memory for energy scratch");
      err = NMFA_ERR_CUDA;
      break;
    }
  } while (0);
  cudaSetDevice(prev);
  if (err) {
    nmfa_plan_destroy(pl);
    return err;
  }
  *out = pl;
  return NMFA_OK;
  NMFA_API_END
}

int nmfa_plan_run(nmfa_plan_t* pl, uint64_t seed, int64_t r0, const float* noise,
                  const float* s0, int8_t* cfg, double* energy, float* s_out, float* s_hist,
                  double* e_hist, void* stream) {
  NMFA_API_BEGIN
  if (!pl) return arg_error("NULL plan");
  if (!cfg) return arg_error("config output is NULL");
  if (e_hist && !s_hist) return arg_error("e_hist requires s_hist");
  g_launches = 0;
  const nmfa_problem* p = pl->p;
  if (pl->path != p->path)
    return state_error("plan was built for another path; create a new plan after set_path");
  cudaStream_t st = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  uint64_t key_base = seed + (uint64_t)r0;
  int err = NMFA_OK;
  bool energy_done = false;
  switch (p->path) {
    case NMFA_PATH_SMALL:
      err = launch_small_anneal(pl, key_base, noise, s0, cfg, s_out, s_hist, st);
      break;
    case NMFA_PATH_DENSE:
      err = launch_dense_anneal(pl, key_base, noise, s0, cfg, s_out, s_hist, energy, &energy_done,
                                st);
      break;
    default:
      err = launch_sparse_anneal(pl, key_base, noise, s0, cfg, s_out, s_hist, st);
  }
  if (!err && energy && !energy_done && p->device_generated) {
    set_error("energies of a device-generated problem need the tensor-core pass");
    err = NMFA_ERR_STATE;
  }
  if (!err && energy && !energy_done)
    err = launch_energy(p, cfg, pl->R, energy, pl->d_bits, pl->d_epart, pl->energy_chunks, st);
  if (!err && e_hist) {
    // energies of sign(s_t) for every recorded step (_kernels_numba.py:57-60)
    int64_t cnt = pl->R * (int64_t)pl->t_f;
    int8_t* hc = nullptr;
    uint32_t* hb = nullptr;
    double* hp = nullptr;
    int64_t ch = energy_chunks_for(p, cnt);
    if (cudaMallocAsync(&hc, (size_t)cnt * p->n, st) != cudaSuccess ||
        cudaMallocAsync(&hb, (size_t)p->n * ((cnt + 31) / 32) * 4, st) != cudaSuccess ||
        cudaMallocAsync(&hp, (size_t)(ch + 1) * cnt * 8, st) != cudaSuccess) {
      set_error("out of device memory for trajectory energies");
      err = NMFA_ERR_CUDA;
    } else {
      err = launch_sign(s_hist, cnt * p->n, hc, st);
      if (!err) err = launch_energy(p, hc, cnt, e_hist, hb, hp, ch, st);
      cudaFreeAsync(hc, st);
      cudaFreeAsync(hb, st);
      cudaFreeAsync(hp, st);
    }
  }
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_plan_run_sweeps(nmfa_plan_t* pl, uint64_t seed, int64_t r0, int32_t t_begin,
                         int32_t t_end, int32_t energy_pass, int8_t* cfg, double* energy,
                         void* stream) {
  NMFA_API_BEGIN
  if (!pl) return arg_error("NULL plan");
  const nmfa_problem* p = pl->p;
  if (p->path != NMFA_PATH_DENSE) return arg_error("sweep ranges are a dense-path feature");
  if (t_begin < 0 || t_end < t_begin || t_end > pl->t_f)
    return arg_error("sweep range must satisfy 0 <= t_begin <= t_end <= t_f");
  if (dense_is_sharded(p) && t_end - t_begin > 1)
    return arg_error("a row-sharded problem runs one sweep per call (all-gather in between)");
  if (energy_pass && !energy) return arg_error("energy pass needs an energy buffer");
  if (energy_pass && !dense_energy_exact(p))
    return arg_error("the tensor-core energy pass needs integer couplings with |J c| < 2^24");
  if (energy_pass && t_end != pl->t_f)
    return arg_error("the energy pass follows the last sweep (t_end == t_f)");
  g_launches = 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  const int err = dense_run_sweeps(pl, seed + (uint64_t)r0, nullptr, nullptr, cfg, nullptr,
                                   nullptr, energy, t_begin, t_end, energy_pass != 0,
                                   (cudaStream_t)stream);
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_gset_parse(const char* text, int64_t len, int64_t* n_out, int64_t* m_out,
                    int64_t* edges_i, int64_t* edges_j, double* weights, int64_t cap) {
  NMFA_API_BEGIN
  if (!text || len < 0 || !n_out || !m_out) return arg_error("NULL argument");
  if ((edges_i || edges_j || weights) && !(edges_i && edges_j && weights))
    return arg_error("edge arrays must be all NULL (header query) or all set");
  return gset_parse(text, len, n_out, m_out, edges_i, edges_j, weights, cap);
  NMFA_API_END
}

int nmfa_problem_create_gset(const char* text, int64_t len, int32_t device,
                             nmfa_problem_t** out) {
  NMFA_API_BEGIN
  if (!text || len < 0 || !out) return arg_error("NULL argument");
  *out = nullptr;
  int64_t n = 0, m = 0;
  int err = gset_parse(text, len, &n, &m, nullptr, nullptr, nullptr, 0);
  if (err) return err;
  std::vector<int64_t> ei((size_t)m), ej((size_t)m);
  std::vector<double> w((size_t)m);
  if ((err = gset_parse(text, len, &n, &m, ei.data(), ej.data(), w.data(), m))) return err;
  std::vector<double> h((size_t)n, 0.0);  // the instance format has no field column (gset.py:99-109)
  return nmfa_problem_create(n, m, ei.data(), ej.data(), w.data(), h.data(), device, out);
  NMFA_API_END
}

int nmfa_ground_state(const nmfa_problem_t* p, int32_t max_n, double* energy,
                      int64_t* degeneracy, int8_t* config) {
  NMFA_API_BEGIN
  if (!p || !energy || !degeneracy) return arg_error("NULL argument");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  g_launches = 0;
  const int err = ground_state(p, max_n, energy, degeneracy, config);
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_plan_image_info(const nmfa_plan_t* pl, void** img0, void** img1, int64_t* slice_bytes,
                         int32_t* n_slices, int32_t* slice_lo, int32_t* slice_hi) {
  NMFA_API_BEGIN
  if (!pl || !img0 || !img1 || !slice_bytes || !n_slices || !slice_lo || !slice_hi)
    return arg_error("NULL argument");
  return dense_image_info(pl, img0, img1, slice_bytes, n_slices, slice_lo, slice_hi);
  NMFA_API_END
}

int nmfa_plan_set_exchange(nmfa_plan_t* pl, void* const* image0_ptrs, void* const* image1_ptrs,
                           int32_t world, int32_t rank, int64_t bytes) {
  NMFA_API_BEGIN
  if (!pl || !image0_ptrs || !image1_ptrs) return arg_error("NULL argument");
  if (pl->p->path != NMFA_PATH_DENSE) return arg_error("the fused exchange is a dense-path feature");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->p->device);
  const int err = dense_set_exchange(pl, image0_ptrs, image1_ptrs, world, rank, bytes);
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_plan_read_config(const nmfa_plan_t* pl, int8_t* cfg, void* stream) {
  NMFA_API_BEGIN
  if (!pl || !cfg) return arg_error("NULL argument");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->p->device);
  const int err = dense_read_config(pl, cfg, (cudaStream_t)stream);
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_anneal(const nmfa_problem_t* cp, int64_t R, int32_t t_f, const double* temps,
                double alpha, double sigma, uint64_t seed, int64_t r0, const float* noise,
                const float* s0, int8_t* cfg, double* energy, float* s_out, float* s_hist,
                double* e_hist, void* stream) {
  NMFA_API_BEGIN
  if (!cp) return arg_error("NULL problem");
  if (!temps || t_f < 1) return arg_error("t_f must be at least 1, got " + std::to_string(t_f));
  auto* p = const_cast<nmfa_problem*>(cp);  // only the plan cache is mutated
  std::lock_guard<std::mutex> lock(p->cache_mu);
  nmfa_plan_t* pl = p->cached_plan;
  const bool hit = pl && pl->R == R && pl->t_f == t_f && p->cached_alpha == alpha &&
                   p->cached_sigma == sigma &&
                   std::equal(temps, temps + t_f, p->cached_temps.begin(), p->cached_temps.end());
  if (!hit) {
    if (pl) nmfa_plan_destroy(pl);
    p->cached_plan = nullptr;
    int err = nmfa_plan_create(p, R, t_f, temps, alpha, sigma, &pl);
    if (err) return err;
    p->cached_plan = pl;
    p->cached_temps.assign(temps, temps + t_f);
    p->cached_alpha = alpha;
    p->cached_sigma = sigma;
  }
  static const bool timing = getenv("NMFA_TIMING") != nullptr;
  const auto ta = std::chrono::steady_clock::now();
  int err = nmfa_plan_run(pl, seed, r0, noise, s0, cfg, energy, s_out, s_hist, e_hist, stream);
  const auto tb = std::chrono::steady_clock::now();
  if (timing)
    fprintf(stderr, "nmfa_anneal: cache %s, enqueue %.3f ms\n", hit ? "hit" : "miss",
            std::chrono::duration<double, std::milli>(tb - ta).count());
  if (!err && cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
    set_error(std::string("CUDA error: ") + cudaGetErrorString(cudaGetLastError()));
    err = NMFA_ERR_CUDA;
  }
  return err;
  NMFA_API_END
}

int nmfa_anneal_many(const nmfa_problem_t* const* ps, int32_t count, int64_t R, int32_t t_f,
                     const double* temps, double alpha, double sigma, const uint64_t* seeds,
                     int8_t* cfg, double* energy, void* stream) {
  NMFA_API_BEGIN
  if (!ps || !seeds || !cfg || count < 1) return arg_error("NULL argument or empty instance list");
  if (R < 1) return arg_error("n_runs must be at least 1, got " + std::to_string(R));
  if (!temps || t_f < 1) return arg_error("t_f must be at least 1, got " + std::to_string(t_f));
  if (!(alpha >= 0.0 && alpha <= 1.0))
    return arg_error("alpha must be in [0, 1], got " + std::to_string(alpha));
  if (!(sigma >= 0.0)) return arg_error("sigma must be nonnegative, got " + std::to_string(sigma));
  const int64_t n = ps[0] ? ps[0]->n : 0;
  bool grouped = true;
  for (int32_t k = 0; k < count; ++k) {
    if (!ps[k]) return arg_error("NULL problem in the instance list");
    if (ps[k]->n != n) return arg_error("every instance of a group must have the same n");
    if (ps[k]->device != ps[0]->device) return arg_error("instances must live on one device");
    grouped = grouped && ps[k]->path == NMFA_PATH_SMALL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!grouped) {  // larger instances: one (cached-plan) anneal per instance
    for (int32_t k = 0; k < count; ++k) {
      const int err = nmfa_anneal(ps[k], R, t_f, temps, alpha, sigma, seeds[k], 0, nullptr,
                                  nullptr, cfg + (size_t)k * R * n,
                                  energy ? energy + (size_t)k * R : nullptr, nullptr, nullptr,
                                  nullptr, stream);
      if (err) return err;
    }
    return NMFA_OK;
  }
  std::vector<float> inv_t(t_f);
  for (int32_t t = 0; t < t_f; ++t) {
    if (!(temps[t] > 0.0) || !std::isfinite(temps[t]))
      return arg_error("temperature must be positive, got " + std::to_string(temps[t]));
    inv_t[t] = (float)(1.0 / temps[t]);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ps[0]->device);
  g_launches = 0;
  int err = NMFA_OK;
  float* d_inv = nullptr;
  uint32_t* bits = nullptr;
  double* part = nullptr;
  do {
    if (cudaMallocAsync(&d_inv, 4 * t_f, st) != cudaSuccess ||
        cudaMemcpyAsync(d_inv, inv_t.data(), 4 * t_f, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      set_error("out of device memory for the schedule");
      err = NMFA_ERR_CUDA;
      break;
    }
    std::vector<uint64_t> keys(seeds, seeds + count);
    err = launch_small_anneal_many(ps, count, R, t_f, d_inv, (float)alpha, (float)sigma,
                                   keys.data(), cfg, st);
    if (err || !energy) break;
    int64_t chunks = 1;
    for (int32_t k = 0; k < count; ++k) chunks = std::max(chunks, energy_chunks_for(ps[k], R));
    if (cudaMallocAsync(&bits, (size_t)n * ((R + 31) / 32) * 4, st) != cudaSuccess ||
        cudaMallocAsync(&part, (size_t)(chunks + 1) * R * 8, st) != cudaSuccess) {
      set_error("out of device memory for energy scratch");
      err = NMFA_ERR_CUDA;
      break;
    }
    for (int32_t k = 0; k < count && !err; ++k)
      err = launch_energy(ps[k], cfg + (size_t)k * R * n, R, energy + (size_t)k * R, bits, part,
                          energy_chunks_for(ps[k], R), st);
  } while (0);
  if (d_inv) cudaFreeAsync(d_inv, st);
  if (bits) cudaFreeAsync(bits, st);
  if (part) cudaFreeAsync(part, st);
  if (!err && cudaStreamSynchronize(st) != cudaSuccess) {
    set_error(std::string("CUDA error: ") + cudaGetErrorString(cudaGetLastError()));
    err = NMFA_ERR_CUDA;
  }
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_anneal_host(const nmfa_problem_t* p, int64_t R, int32_t t_f, const double* temps,
                     double alpha, double sigma, uint64_t seed, int64_t r0, int8_t* cfg_host,
                     double* energy_host) {
  NMFA_API_BEGIN
  if (!p || !cfg_host) return arg_error("NULL argument");
  if (R < 1) return arg_error("n_runs must be at least 1, got " + std::to_string(R));
  static const bool timing = getenv("NMFA_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  auto* mp = const_cast<nmfa_problem*>(p);
  // the cached stream and result buffers are shared by every host-entry call
  // on this problem: hold them for the whole call
  std::lock_guard<std::mutex> host_lock(mp->host_mu);
  int err = NMFA_OK;
  {
    // device result buffers and the stream are cached on the problem handle
    std::lock_guard<std::mutex> lock(mp->cache_mu);
    if (!mp->host_stream && cudaStreamCreateWithFlags(&mp->host_stream, cudaStreamNonBlocking))
      err = NMFA_ERR_CUDA;
    if (!err && mp->host_cap < R) {
      if (mp->host_cfg) cudaFree(mp->host_cfg);
      if (mp->host_e) cudaFree(mp->host_e);
      mp->host_cfg = nullptr;
      mp->host_e = nullptr;
      if (cudaMalloc(&mp->host_cfg, (size_t)R * p->n) || cudaMalloc(&mp->host_e, (size_t)R * 8))
        err = NMFA_ERR_CUDA;
      else
        mp->host_cap = R;
    }
  }
  if (err) {
    set_error("out of device memory / stream creation failed");
    cudaSetDevice(prev);
    return err;
  }
  cudaStream_t st = mp->host_stream;
  const auto t1 = now();
  err = nmfa_anneal(p, R, t_f, temps, alpha, sigma, seed, r0, nullptr, nullptr, mp->host_cfg,
                    energy_host ? mp->host_e : nullptr, nullptr, nullptr, nullptr, st);
  const auto t2 = now();
  if (!err && (cudaMemcpyAsync(cfg_host, mp->host_cfg, (size_t)R * p->n, cudaMemcpyDeviceToHost, st) ||
               (energy_host && cudaMemcpyAsync(energy_host, mp->host_e, (size_t)R * 8,
                                               cudaMemcpyDeviceToHost, st)) ||
               cudaStreamSynchronize(st))) {
    set_error("device to host copy failed");
    err = NMFA_ERR_CUDA;
  }
  const auto t3 = now();
  if (timing)
    fprintf(stderr, "nmfa_anneal_host: setup %.3f ms, anneal %.3f ms, d2h %.3f ms\n", ms(t0, t1),
            ms(t1, t2), ms(t2, t3));
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_energy(const nmfa_problem_t* p, const int8_t* cfg, int64_t n_cfg, double* energy,
                void* stream) {
  NMFA_API_BEGIN
  if (!p || !cfg || !energy) return arg_error("NULL argument");
  if (n_cfg < 1) return arg_error("need at least one configuration");
  if (p->device_generated) {
    // no edge list on the device: the dense kernel's exact tensor-core energy
    // pass on the given configurations (integer J, |J c| < 2^24)
    if (dense_is_sharded(p))
      return arg_error("a row-sharded problem holds only its rows of J; its energies come from "
                       "the sharded protocol (sharded.py)");
    if (!dense_energy_exact(p)) return state_error("tensor-core energies are not exact here");
    const double one = 1.0;
    nmfa_plan_t* pl = nullptr;
    int err = nmfa_plan_create(p, n_cfg, 1, &one, 0.15, 0.15, &pl);
    if (err) return err;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    err = dense_energy_only(pl, cfg, energy, (cudaStream_t)stream);
    if (!err && cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
      set_error("CUDA error in the tensor-core energy pass");
      err = NMFA_ERR_CUDA;
    }
    cudaSetDevice(prev);
    nmfa_plan_destroy(pl);
    return err;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  int64_t ch = energy_chunks_for(p, n_cfg);
  uint32_t* bits = nullptr;
  double* part = nullptr;
  int err = NMFA_OK;
  if (cudaMallocAsync(&bits, (size_t)p->n * ((n_cfg + 31) / 32) * 4, st) != cudaSuccess ||
      cudaMallocAsync(&part, (size_t)(ch + 1) * n_cfg * 8, st) != cudaSuccess) {
    set_error("out of device memory");
    err = NMFA_ERR_CUDA;
  } else {
    err = launch_energy(p, cfg, n_cfg, energy, bits, part, ch, st);
  }
  if (bits) cudaFreeAsync(bits, st);
  if (part) cudaFreeAsync(part, st);
  cudaSetDevice(prev);
  return err;
  NMFA_API_END
}

int nmfa_best_of(const double* e, int64_t n, double* best_e, int64_t* best_i, void* stream) {
  NMFA_API_BEGIN
  if (!e || !best_e || !best_i) return arg_error("NULL argument");
  if (n < 1) return arg_error("best-of needs at least one energy");
  return launch_best_of(e, n, best_e, best_i, (cudaStream_t)stream);
  NMFA_API_END
}

}  // extern "C"
