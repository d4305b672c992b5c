/*
 * nmfa_b200.h -- C ABI of the B200-native noisy mean-field annealing sampler.
 *
 * The reference package (`nmfa`, pure Python) has no native FFI; its operator
 * boundary is the per-run kernel pair bound in kernels.py:30-31 and its
 * sampling entry point is nmfa_batch (solver.py:262-280).  This header is the
 * native boundary the Python mirror in `paper_1806_08422_b200` binds through
 * ctypes (see INTEGRATION.md for the binding a maintainer of the reference
 * would add).  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Every function returns 0 on success and a nonzero NMFA_ERR_* code on
 *    failure; nmfa_last_error() then holds a thread-local message.  Argument
 *    errors mirror the reference's ValueError messages (solver.py:196-205,
 *    problem.py:25-62); CUDA failures return NMFA_ERR_CUDA.
 *  - "dev" pointers are CUDA device pointers on the problem's device; "host"
 *    pointers are ordinary host memory.  `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  Device entry points are asynchronous.
 *  - Replica r of a call with first global index r0 uses noise key seed+r0+r,
 *    so results do not depend on how replicas are split over calls or GPUs.
 */
#ifndef NMFA_B200_H_
#define NMFA_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMFA_OK 0
#define NMFA_ERR_ARG 1   /* invalid argument (reference: ValueError) */
#define NMFA_ERR_CUDA 2  /* CUDA runtime / launch failure (RuntimeError) */
#define NMFA_ERR_STATE 3 /* wrong object state / unsupported request */

/* Kernel path chosen for a problem (internal detail, reported for tests). */
#define NMFA_PATH_SMALL 0  /* n <= 256: persistent tcgen05 kernel, J in SMEM */
#define NMFA_PATH_DENSE 1  /* dense n > 256: tcgen05 GEMM step, J streamed */
#define NMFA_PATH_SPARSE 2 /* sparse n > 256: ELL (max degree <= 4) or CSR gather step */

/* Precision of the dense path's GEMM operand (the field J.s; the state itself is
 * always fp16 hi + fp16 lo, ~22 bits).  FP16: the hi part only (one tcgen05 MMA
 * per k-slice; the throughput mode, trajectories within 2e-3 of float64).  HILO:
 * hi and lo both enter the GEMM (two MMAs per k-slice into one fp32
 * accumulator, a second lo image; about half the throughput), so the field
 * carries the full state and trajectories follow the float64 reference like
 * the fp32 sparse path (the fidelity mode).  The small path
 * (n <= 256) supports HILO up to n = 224 (a second operand image in shared
 * memory; the MMA is a small part of its step); the sparse path is fp32
 * either way. */
#define NMFA_FIELD_FP16 0
#define NMFA_FIELD_HILO 1

typedef struct nmfa_problem nmfa_problem_t;
typedef struct nmfa_plan nmfa_plan_t;

typedef struct {
  int64_t n;
  int64_t n_edges;
  double density;      /* edges / (n(n-1)/2), problem.py:96-99 */
  int32_t is_dense;    /* density > 0.5, the reference's dispatch bit */
  int32_t path;        /* NMFA_PATH_* */
  int32_t j_exact;     /* 1 if every coupler is exact in the fp16 operand */
  int32_t int_weights; /* 1 if all weights and fields are integers */
  double j_scale;      /* power-of-two scale applied to J on device */
  int32_t ell_slots;   /* sparse path: ELL row length (3 or 4) when the max
                          degree is <= 4, 0 when rows use the CSR kernel */
  int32_t field;       /* NMFA_FIELD_* (nmfa_problem_set_field_precision) */
} nmfa_problem_info_t;

/* Build an immutable device-resident problem from the canonical coupler
 * list (IsingProblem(n, couplers, h), problem.py:25-116).  Edges may come in
 * any order and orientation; they are canonicalised to i<j.  Validation and
 * error text follow problem.py:25-62.  h_host may be NULL (zero fields).
 * Replaces: IsingProblem construction + the dense/CSR arrays handed to
 * kernels.anneal_dense / kernels.anneal_sparse (solver.py:206-216). */
int nmfa_problem_create(int64_t n, int64_t n_edges, const int64_t* edges_i_host,
                        const int64_t* edges_j_host, const double* weights_host,
                        const double* h_host, int32_t device, nmfa_problem_t** out);
/* The same problem from a dense row-major n x n coupling matrix (symmetric,
 * zero diagonal; the `J` that kernels.anneal_dense receives, solver.py:206-210,
 * problem.py:100-104); h_host may be NULL. */
int nmfa_problem_create_dense(int64_t n, const double* J_host, const double* h_host,
                              int32_t device, nmfa_problem_t** out);
/* ... or from the symmetric CSR that kernels.anneal_sparse receives
 * (problem.py:78-88; indptr[n+1], indices/weights[indptr[n]]): entries with
 * j > i define the couplers, and their mirror entries must be present. */
int nmfa_problem_create_csr(int64_t n, const int64_t* indptr, const int64_t* indices,
                            const double* weights, const double* h_host, int32_t device,
                            nmfa_problem_t** out);
/* A complete +-1 graph (SK) from packed sign bits: bit (i*n + j) of the
 * row-major bitmap (word b>>5, bit b&31) set -> J_ij = +1, clear -> -1, read
 * for i < j (1/64 of a float64 J).  Up to 4096 spins the host builds the
 * edge list (every path and the edge-list energy); beyond that this is
 * nmfa_problem_create_bits_device(n, bits, h, 0, n, ...). */
int nmfa_problem_create_dense_bits(int64_t n, const uint32_t* sign_bits_host, const double* h_host,
                                   int32_t device, nmfa_problem_t** out);

/* The bit-packed +-1 device format: the same bitmap is
 * uploaded (n^2/8 bytes; 512 MiB at n = 65,536) and expanded ON THE DEVICE
 * into the dense path's fp16 J image of rows [row_lo, row_hi) -- no
 * n(n-1)/2-entry host edge list, so user instances reach the row-sharded
 * sizes of BASELINE config 5 (problem.py:25-116 otherwise needs ~50 GB of
 * host arrays there).  normalizers_safe_i = sqrt(h_i^2 + n - 1)
 * (problem.py:90-95).  Dense path only; energies come from the tensor-core
 * energy pass (nmfa_energy included, exact).  Row shards as in
 * nmfa_problem_create_sk_device. */
int nmfa_problem_create_bits_device(int64_t n, const uint32_t* sign_bits_host, const double* h_host,
                                    int64_t row_lo, int64_t row_hi, int32_t device,
                                    nmfa_problem_t** out);
int nmfa_problem_destroy(nmfa_problem_t* p);
int nmfa_problem_get_info(const nmfa_problem_t* p, nmfa_problem_info_t* info);
/* Synthetic Sherrington-Kirkpatrick instance generated ON DEVICE (BASELINE
 * config 5, SK N = 65,536: the reference cannot build it, problem.py:41-104
 * would need >150 GB of host arrays).  J_ij = +-1 for every pair i != j from a
 * counter-based hash: bit (b mod 128) of Philox4x32-10(key = seed, counter =
 * (b >> 7, a, 0x534B4A31 'SKJ1', 0)) with a = min(i,j), b = max(i,j), set bit
 * -> +1; h = 0 (same distribution as gen_sk, generators.py:27-35, not the same
 * stream).  Only rows [row_lo, row_hi) of J are materialised (row sharding:
 * row_lo a multiple of 128, row_hi a multiple of 128 or n).  Energies come
 * from the tensor-core energy pass; nmfa_energy is not available. */
int nmfa_problem_create_sk_device(int64_t n, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                  int32_t device, nmfa_problem_t** out);

/* Force a kernel path (tests / crossover studies); NMFA_ERR_ARG if the path
 * cannot run this problem (e.g. SMALL with n > 256). */
int nmfa_problem_set_path(nmfa_problem_t* p, int32_t path);

/* Operand precision of the tensor-core paths for plans created from now on
 * (NMFA_FIELD_*; default FP16).  Drops the problem's cached plan; existing
 * explicit plans keep the precision they were built with.  NMFA_ERR_ARG for
 * HILO on a small-path problem with n > 224, and for a row shard (its
 * exchange carries the hi image only).
 * No reference counterpart: the reference computes the field in float64
 * (_kernels_numba.py:72); HILO is the closest this path gets to it. */
int nmfa_problem_set_field_precision(nmfa_problem_t* p, int32_t field);

/* A plan owns the device state for `n_reads` replicas and `t_f` steps so
 * repeated runs allocate nothing and can be captured in a CUDA graph.  A plan
 * runs one batch at a time (use one plan per concurrent stream); problems are
 * immutable and shareable, and nmfa_anneal / nmfa_anneal_host serialise their
 * per-problem caches internally.
 * temps_host: t_f temperatures (Schedule.temperatures, solver.py:70-84),
 * each > 0.  alpha in [0,1], sigma >= 0 (NmfaParams, solver.py:141-162). */
int nmfa_plan_create(const nmfa_problem_t* p, int64_t n_reads, int32_t t_f,
                     const double* temps_host, double alpha, double sigma,
                     nmfa_plan_t** out);
int nmfa_plan_destroy(nmfa_plan_t* plan);

/* Run one batch of `n_reads` anneals from the plan.  Replaces
 * nmfa_batch (solver.py:262-280) / _run (236-253) for all replicas at once.
 *   noise_dev   [n_reads][t_f][n] f32 pre-scaled additive noise, or NULL to
 *               draw in-kernel Philox noise (run_with_noise seam, 188-218)
 *   s0_dev      [n_reads][n] f32 initial analog spins, or NULL for zeros
 *   config_dev  [n_reads][n] i8 out: sign_round(s) in {-1,+1} (181-183)
 *   energy_dev  [n_reads] f64 out: energy(config) (150-154), or NULL
 *   s_final_dev [n_reads][n] f32 out, or NULL
 *   s_hist_dev  [n_reads][t_f][n] f32 out (record_trajectory), or NULL
 *   e_hist_dev  [n_reads][t_f] f64 out, requires s_hist_dev, or NULL */
int nmfa_plan_run(nmfa_plan_t* plan, uint64_t seed, int64_t r0, const float* noise_dev,
                  const float* s0_dev, int8_t* config_dev, double* energy_dev,
                  float* s_final_dev, float* s_hist_dev, double* e_hist_dev, void* stream);

/* Run sweeps [t_begin, t_end) of the plan's schedule (dense path), then, if
 * energy_pass, the exact tensor-core energy pass into energy_dev (partial over
 * the device's row shard for a row-sharded problem).  t_begin == 0
 * (re)initialises the state from s0_dev / zeros.  A row-sharded problem must
 * run one sweep per call: between calls the host all-gathers every shard's
 * k-slices of the next operand image (nmfa_plan_image_info).  config_dev, if
 * not NULL, receives the configuration of this device's spins at the last
 * sweep (use nmfa_plan_read_config for the all-gathered one). */
int nmfa_plan_run_sweeps(nmfa_plan_t* plan, uint64_t seed, int64_t r0, int32_t t_begin,
                         int32_t t_end, int32_t energy_pass, int8_t* config_dev,
                         double* energy_dev, void* stream);

/* Operand images of a dense plan (the hi part of the replica state, fp16,
 * tiled): image[p] for sweep parity p.  Spins [128k, 128k+128) of all replicas
 * occupy bytes [k * slice_bytes, (k+1) * slice_bytes); this device writes
 * slices [slice_lo, slice_hi). */
int nmfa_plan_image_info(const nmfa_plan_t* plan, void** image0, void** image1,
                         int64_t* slice_bytes, int32_t* n_slices, int32_t* slice_lo,
                         int32_t* slice_hi);

/* Fused exchange for a row-sharded plan (replaces the per-sweep all-gather):
 * image0_ptrs / image1_ptrs hold, for every shard g < world, a device pointer
 * to shard g's operand image of each sweep parity (peer-accessible memory, e.g.
 * CUDA IPC / symmetric-memory buffers of >= bytes each; the plan adopts
 * entries [rank] as its own images and does not free them).  Each sweep's
 * epilogue then stores every new hi line into all shards' images directly, so
 * the exchange overlaps the GEMM.  Between nmfa_plan_run_sweeps calls the
 * caller must synchronise the shards (a device-side barrier after each
 * sweep).  world <= 8. */
int nmfa_plan_set_exchange(nmfa_plan_t* plan, void* const* image0_ptrs, void* const* image1_ptrs,
                           int32_t world, int32_t rank, int64_t bytes);

/* +-1 configurations [n_reads][n] from the (all-gathered) sign image that the
 * last sweep t_f-1 wrote (parity t_f & 1). */
int nmfa_plan_read_config(const nmfa_plan_t* plan, int8_t* config_dev, void* stream);

/* One-shot convenience over plan_create/plan_run/plan_destroy. */
int nmfa_anneal(const nmfa_problem_t* p, int64_t n_reads, int32_t t_f,
                const double* temps_host, double alpha, double sigma, uint64_t seed,
                int64_t r0, const float* noise_dev, const float* s0_dev, int8_t* config_dev,
                double* energy_dev, float* s_final_dev, float* s_hist_dev,
                double* e_hist_dev, void* stream);

/* Many instances, one call (the Fig. 4-style sweep of cli.py:280-347, where
 * the reference runs nmfa_batch once per instance).  Instance k runs n_reads
 * replicas with keys seeds[k] + r (its nmfa_batch seed, cli.py:319-321);
 * config_dev [count][n_reads][n] i8, energy_dev [count][n_reads] f64 (or NULL).
 * Every instance must have the same n.  Small instances (n <= 256) run in ONE
 * persistent launch (grid = replica blocks x instances); larger ones fall back
 * to one anneal per instance.  Synchronous on `stream`. */
int nmfa_anneal_many(const nmfa_problem_t* const* problems, int32_t count, int64_t n_reads,
                     int32_t t_f, const double* temps_host, double alpha, double sigma,
                     const uint64_t* seeds_host, int8_t* config_dev, double* energy_dev,
                     void* stream);

/* Same batch with HOST buffers (H2D of inputs, D2H of results inside the
 * call; synchronous).  This is the end-to-end entry a non-CUDA host binds. */
int nmfa_anneal_host(const nmfa_problem_t* p, int64_t n_reads, int32_t t_f,
                     const double* temps_host, double alpha, double sigma, uint64_t seed,
                     int64_t r0, int8_t* config_host, double* energy_host);

/* energy(problem, config) for a batch of +-1 configs (problem.py:150-154).
 * Bit-exact for integer weights/fields (f64 accumulation of integers),
 * within ~1e-15 relative otherwise. */
int nmfa_energy(const nmfa_problem_t* p, const int8_t* config_dev, int64_t n_configs,
                double* energy_dev, void* stream);

/* best-of-reads: minimum energy and the lowest index attaining it
 * (cli.py:236 min; metrics.py:105). */
int nmfa_best_of(const double* energy_dev, int64_t n, double* best_energy_dev,
                 int64_t* best_index_dev, void* stream);

/* Parse edge-list / G-set instance text (parse_gset, gset.py:35-89): header
 * "n m", then m lines "u v w" (1-based), '#'/'c' comment lines.  Call once
 * with edges_i == NULL to read n and m, then with arrays of capacity >= m to
 * receive the 0-based edges in file order.  Errors follow the reference
 * (GsetParseError): NMFA_ERR_ARG with "line N: <message>" in nmfa_last_error. */
int nmfa_gset_parse(const char* text, int64_t len, int64_t* n_out, int64_t* m_out,
                    int64_t* edges_i, int64_t* edges_j, double* weights, int64_t cap);

/* Instance text straight to a device problem, no host-language layer: the
 * native parse above (same errors and messages), then nmfa_problem_create on
 * the parsed couplers (load_gset + IsingProblem, gset.py:35-96 and
 * problem.py:25-116, in one call for a non-Python host). */
int nmfa_problem_create_gset(const char* text, int64_t len, int32_t device,
                             nmfa_problem_t** out);

/* Exact ground state by exhaustive enumeration: minimum energy over all 2^n
 * configurations and its degeneracy (brute_force_ground, metrics.py:53-67;
 * gray_ground, _kernels_numba.py:83-114: Gray-code single-flip walk, ties
 * within 1e-9).  Exact integer arithmetic when every coupler is in {-1,0,+1}
 * and h is integer, else float64.  NMFA_ERR_ARG if n > max_n (the reference's
 * MAX_EXACT_N = 26; this implementation allows up to 40).  config_host, if not
 * NULL, receives one minimising configuration (+-1).  Synchronous. */
int nmfa_ground_state(const nmfa_problem_t* p, int32_t max_n, double* energy_host,
                      int64_t* degeneracy_host, int8_t* config_host);

/* The reference's own per-run noise on the device (the
 * replay mode of nmfa_batch): run r (global index r0 + r) gets
 * noise_stream(seed + r0 + r).standard_normal(count) * sigma (solver.py:
 * 182-185, 236-241: numpy Philox4x64-10 keyed [seed + r0 + r, 2], numpy's
 * ziggurat), count = t_f * n in C order, into noise_dev [n_reads][count] f32
 * and/or noise64_dev (f64).  Bitwise numpy's draws in f32; f64 tail draws may
 * differ by an ulp (device log1p).  Asynchronous on `stream`. */
int nmfa_reference_noise(uint64_t seed, int64_t r0, int64_t n_reads, int64_t count, double sigma,
                         float* noise_dev, double* noise64_dev, void* stream);

const char* nmfa_last_error(void);
const char* nmfa_version(void);
/* Number of kernels the last nmfa_plan_run on this thread enqueued. */
int64_t nmfa_last_launch_count(void);

/* Checked build only (libnmfa_b200_guard.so, -DNMFA_GUARD; the memcheck
 * substitute where compute-sanitizer is unavailable): synchronises the device
 * and returns the number of redzone bytes found corrupted around the
 * library's own device allocations (live ones now, freed ones when they were
 * freed); nmfa_last_error() names the first.  Returns -1 in normal builds. */
int64_t nmfa_debug_guard_check(void);

#ifdef __cplusplus
}
#endif
#endif /* NMFA_B200_H_ */
