// Tensor-core query path (ss_query_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ss {

// |coarse - exact| bound for unit vectors: fp16 input rounding (2u + u^2,
// u = 2^-11), fp32 tensor-core accumulation over K <= 1024 terms, fp16
// rounding of the coarse score, and the exact scorer's own fp32 rounding.
constexpr float kCoarseEps = 2.0e-3f;

// Pilot: row tiles sampled with a uniform stride, at most this many (256 rows each).
constexpr uint32_t kPilotTiles = 512;

cudaError_t launch_to_half(const float* in, uint64_t n, void* out, cudaStream_t s);
uint32_t pilot_tiles(uint32_t n_rows);
uint64_t pilot_cols(uint32_t n_rows);
// fp16 coarse scores of the pilot sample, [nq][pilot_cols(n_rows)]
cudaError_t launch_coarse_pilot(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                uint32_t k_dim, void* scores, int num_sms, cudaStream_t s);
// per-query candidate threshold from the pilot scores
cudaError_t launch_pilot_threshold(const void* scores, uint32_t n_rows, uint32_t nq, uint32_t k, float eps2,
                                   float* thr, cudaStream_t s);
// full pass: rows with coarse >= thr[q] appended to cand[q * cap ...], cand_count[q] (zeroed by the caller)
cudaError_t launch_coarse_candidates(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                     uint32_t k_dim, const float* thr, uint32_t* cand, float* cand_val,
                                     uint32_t cand_cap, uint32_t* cand_count, int num_sms, cudaStream_t s);
// exact top-k among the candidates within 2*eps of the k-th coarse score;
// sets cand_count[q] = ~0 when a query's finalists overflow
cudaError_t launch_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn, uint32_t nq,
                           const uint32_t* cand, const float* cand_val, uint32_t cand_cap, uint32_t* cand_count,
                           uint32_t k, float eps2, uint32_t* out_ids, float* out_sims, cudaStream_t s);
// query_threshold: exact rescoring of the tau - eps candidates of one query
cudaError_t launch_threshold_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn,
                                     const uint32_t* cand, uint32_t cand_cap, const uint32_t* cand_count, float tau,
                                     uint32_t* out_ids, float* out_sims, uint64_t out_cap, uint32_t* out_count,
                                     cudaStream_t s);

} // namespace ss
