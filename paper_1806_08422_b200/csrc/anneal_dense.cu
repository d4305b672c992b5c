// Dense large-N NMFA step (tcgen05 GEMM with fused update epilogue).
#include "common.cuh"
#include "internal.h"

namespace nmfa {

int dense_problem_upload(nmfa_problem* p, const std::vector<float>& jd) {
  (void)jd;
  p->d_j_dense = nullptr;
  return NMFA_OK;
}

int dense_plan_alloc(nmfa_plan* pl) {
  (void)pl;
  return NMFA_OK;
}

int launch_dense_anneal(const nmfa_plan* pl, uint64_t key_base, const float* noise,
                        const float* s0, int8_t* cfg, float* s_out, float* s_hist,
                        cudaStream_t st) {
  // Until the tcgen05 dense kernel lands, dense problems run the CSR path.
  return launch_sparse_anneal(pl, key_base, noise, s0, cfg, s_out, s_hist, st);
}

}  // namespace nmfa
