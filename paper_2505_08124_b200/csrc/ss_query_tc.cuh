// Tensor-core query path (ss_query_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ss {

// |coarse - exact| bound for unit vectors: fp16 input rounding (2u + u^2,
// u = 2^-11), fp32 tensor-core accumulation over K <= 1024 terms, fp16
// rounding of the coarse score, and the exact scorer's own fp32 rounding.
constexpr float kCoarseEps = 2.0e-3f;

size_t tc_scores_smem();
cudaError_t launch_to_half(const float* in, uint64_t n, void* out, cudaStream_t s);
cudaError_t launch_coarse_scores(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                 uint32_t k_dim, void* scores, uint64_t ld, int num_sms, cudaStream_t s);
cudaError_t launch_select_candidates(const void* scores, uint64_t ld, uint32_t n_rows, uint32_t nq, uint32_t k,
                                     float eps2, uint32_t* cand, uint32_t cand_cap, uint32_t* cand_count,
                                     cudaStream_t s);
cudaError_t launch_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn, uint32_t nq,
                           const uint32_t* cand, uint32_t cand_cap, const uint32_t* cand_count, uint32_t k,
                           float* cand_sim, uint32_t* out_ids, float* out_sims, cudaStream_t s);

} // namespace ss
