// Launchers of the non-exact kernels (ss_kernels.cu).
#pragma once
#include <type_traits>

#include "ss_internal.cuh"

namespace ss {

// One view of a contraction group: its compositor outputs and CLIP rows.
struct ContractMember {
    const uint32_t* touched_list;        // Gaussians touched in the view
    const unsigned long long* touched_count;
    const uint32_t* touched;             // generation stamps
    uint32_t gen;                        // the view's stamp
    void* acc;                           // [N x n_masks] float (or acc_t if fix), consumed and cleared
    uint32_t fix;                        // scalars in fixed point (SS_OPT_DETERMINISTIC)
    uint32_t n_masks;
    const float* clip;                   // [n_masks x dim]
};

// One Gaussian's row of a member's scalars, in either representation.
struct AccRow {
    void* p;
    bool fix;
    __device__ __forceinline__ float get(uint32_t i) const {
        return fix ? acc_val(static_cast<const acc_t*>(p)[i]) : static_cast<const float*>(p)[i];
    }
    __device__ __forceinline__ void clear(uint32_t i) const {
        if (fix) static_cast<acc_t*>(p)[i] = 0ull;
        else static_cast<float*>(p)[i] = 0.0f;
    }
};
__device__ __forceinline__ AccRow acc_row(const ContractMember& m, uint64_t gid) {
    const size_t off = (size_t)gid * m.n_masks;
    return AccRow{m.fix ? (void*)(static_cast<acc_t*>(m.acc) + off) : (void*)(static_cast<float*>(m.acc) + off),
                  m.fix != 0};
}

// The same with the representation fixed at compile time (the hot group kernels).
template <bool FIX>
struct AccRowT {
    using T = typename std::conditional<FIX, acc_t, float>::type;
    T* p;
    __device__ __forceinline__ float get(uint32_t i) const {
        if constexpr (FIX) return acc_val(p[i]);
        else return p[i];
    }
    __device__ __forceinline__ void clear(uint32_t i) const { p[i] = T(0); }
};
template <bool FIX>
__device__ __forceinline__ AccRowT<FIX> acc_row_t(const ContractMember& m, uint64_t gid) {
    return AccRowT<FIX>{static_cast<typename AccRowT<FIX>::T*>(m.acc) + (size_t)gid * m.n_masks};
}

constexpr uint32_t kMaxGroup = 4;

// Contraction of a group of consecutive views (view order = member order).
struct ContractParams {
    ContractMember m[kMaxGroup];
    uint32_t n_members;
    uint32_t dim;
    float* sums;           // [N x dim]
    float* totals;         // [N]
    int count_pairs;
    unsigned long long* cum; // running totals: [0] G_v, [1] K_v (summed over views), [2] rows read+written
    uint2* union_list;       // group scratch: (gid, member mask), sum of the members' lists
    unsigned int* union_count;
    void* tc_scratch;        // contract_tc_scratch_bytes(): prepared CLIP operands of the tensor-core path
    int use_tc;              // SS_OPT_CONTRACT_TC: groups on the tensor cores (ss_contract_tc.cu)
};

// Tensor-core group contraction (ss_contract_tc.cu): 2-3 members, D = 512,
// <= 64 masks each, union list required.
size_t contract_tc_scratch_bytes();
bool contract_tc_eligible(const ContractParams& p);
cudaError_t launch_contract_tc(const ContractParams& p, void* scratch, int ctas, cudaStream_t s);

cudaError_t launch_rle_to_bits(const uint32_t* runs, const uint64_t* run_offsets, uint32_t n_masks, uint32_t words,
                               uint32_t* bits, uint4* spans, unsigned int* n_spans, cudaStream_t s);
cudaError_t launch_resample_bits(const uint32_t* src, uint32_t sw, uint32_t sh, uint32_t* dst, uint32_t tw,
                                 uint32_t th, uint32_t words, cudaStream_t s);
cudaError_t launch_narrow_keys(const unsigned long long* keys, uint64_t n, const ViewInfo* info, uint32_t* k32,
                               cudaStream_t s);
cudaError_t launch_tie_fixup(const uint32_t* k32s, uint64_t n, const unsigned long long* keys, uint32_t* order,
                             cudaStream_t s);
cudaError_t launch_gather_boxes(const uint2* boxes, const uint32_t* k32s, const uint32_t* order, uint64_t n,
                                uint2* rbox, uint32_t* cnt, cudaStream_t s);
cudaError_t launch_instance_offsets(const uint32_t* cnt, uint64_t n, uint32_t* offsets, void* tmp, size_t* tmp_bytes,
                                    cudaStream_t s);
cudaError_t launch_emit_instances(const uint2* rbox, const uint32_t* order, uint64_t n, const uint32_t* offsets,
                                  uint32_t tiles_x, uint64_t cap, void* keys, bool k16, uint32_t* vals, ViewInfo* info,
                                  cudaStream_t s);
cudaError_t launch_tile_ranges(const void* keys, bool k16, const uint32_t* offsets, uint64_t n, uint64_t cap,
                               uint32_t* start, uint32_t* end, ViewInfo* info, cudaStream_t s);

// Direct box binning (count / scan / scatter; ss_kernels.cu): tile lists and
// ranges straight from the depth order, bit-identical to the sort path.
struct BinParams {
    const uint2* boxes;    // per Gaussian (projection)
    const uint32_t* order; // depth order, survivors first
    uint64_t n;            // Gaussians (grid size; survivors come from info)
    uint32_t tiles, tiles_x;
    uint2* rbox;           // [n] boxes in rank order (scratch)
    uint32_t* counts;      // [bin_counts_entries] per-chunk tile counts / prefixes
    uint32_t* slice;       // [32 x tiles] slice bases
    uint32_t* tot;         // [tiles] tile totals
    uint32_t* done;        // CTA counter, zero between launches
    uint32_t* start;       // [tiles] tile ranges
    uint32_t* end;
    uint32_t* list;        // [cap] splat ids
    uint64_t cap;
    ViewInfo* info;
};
// Tile-sort binning (ss_kernels.cu): each Gaussian's tile instances are
// scattered, unordered, into fixed-capacity per-tile slots (chunk histograms in
// shared memory reserve each tile's range with one global atomic per chunk),
// then one CTA per tile orders its slots by (depth, id) with a shared-memory
// bucket sort on the narrowed key plus an exact fix-up of shared buckets.  No
// global depth sort is needed for the fused pass.
struct TileSortParams {
    const uint2* boxes;              // by gid (projection; culled: all ones)
    const unsigned long long* keys;  // by gid: depth bits (~0 culled)
    uint64_t n;                      // Gaussians
    uint32_t tiles, tiles_x;
    uint32_t cap;                    // slots per tile
    uint32_t* fill;                  // [tiles], zero before the scatter
    uint2* slab;                     // [tiles * cap] (narrowed key, gid), unordered
    uint32_t* list;                  // [tiles * cap] gids in (depth, id) order
    uint32_t* start;                 // [tiles] list ranges
    uint32_t* end;
    ViewInfo* info;
    // prefix mode (fused pass): a tile of n > prefix_min instances is ranked
    // only over its first max(prefix_min, n / 4) instances (whole buckets),
    // end = start + that prefix; blocks that exhaust it with live pixels are
    // resumed after the fixup sort (fix_tiles, fix_count[1]) completes the tile
    uint32_t prefix_min;             // 0: full sort
    const uint32_t* fix_tiles;       // fixup launch: tiles to sort in full
    const uint32_t* fix_count;       // [1] = number of fix_tiles
    uint32_t* need;                  // [tiles] tile queued for the fixup (cleared by it)
};
constexpr uint32_t kTileSortMax = 8192; // instances one CTA orders in shared memory
// slot capacity for a view whose largest tile holds max_fill instances: 4096, 6144 or 8192
inline uint32_t tile_sort_capacity(uint32_t max_fill) {
    return max_fill <= kTileSortMax / 2 ? kTileSortMax / 2 : (max_fill <= kTileSortMax * 3 / 4 ? kTileSortMax * 3 / 4 : kTileSortMax);
}
uint32_t tile_sort_max_tiles();         // views with more tiles use the other paths
cudaError_t launch_tile_sort_bin(const TileSortParams& p, cudaStream_t s);
// covered rows of a normalised slice packed (ids, coverage, rows; count atomically)
cudaError_t launch_compact_covered(const float* rows, const float* cov, uint64_t n, uint32_t dim, uint32_t* ids,
                                   float* pcov, float* prow, unsigned long long* count, cudaStream_t s);
// the full sort of the tiles the resumed compositor needs (prefix mode)
cudaError_t launch_tile_sort_fixup(const TileSortParams& p, cudaStream_t s);

// warps per scatter CTA for a tile count (0: too many tiles, use the sort path)
uint32_t bin_scatter_warps(uint32_t tiles);
size_t bin_counts_entries(uint64_t n, uint32_t tiles);
cudaError_t launch_bin(const BinParams& p, cudaStream_t s);
cudaError_t launch_contract(const ContractParams& p, uint64_t max_touched, cudaStream_t s);
// covered (optional): += rows with total > 1e-8 (their sums are read; the rest are only written)
cudaError_t launch_normalize(const float* sums, const float* totals, uint64_t n, uint32_t dim, float* rows,
                             float* coverage, unsigned long long* covered, cudaStream_t s);
cudaError_t launch_normalize_rows(const float* in, const uint32_t* select, uint64_t n, uint32_t dim, float* out,
                                  int* zero_flag, cudaStream_t s);
// eval.hpp:122-158 (labels [n_labels][dim]; labels_t, label_norms: scratch)
cudaError_t launch_assign_classes(const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                                  const int32_t* label_ids, const float* labels, uint32_t n_labels, float* labels_t,
                                  double* label_norms, int32_t* out, cudaStream_t s);
cudaError_t launch_flag_covered(const float* coverage, uint64_t n, uint8_t* flags, cudaStream_t s);
int score_query_tile();
cudaError_t launch_score(const float* rows, uint64_t count, uint32_t dim, const float* queries, uint32_t nq,
                         uint32_t q0, float* scores, cudaStream_t s);
cudaError_t launch_topk(const float* scores, const uint32_t* ids, uint64_t count, uint32_t k, uint32_t nq_tile,
                        uint32_t q0, uint32_t* out_ids, float* out_sims, cudaStream_t s);
cudaError_t launch_threshold_keys(const float* scores, const uint32_t* ids, uint64_t count, float tau,
                                  unsigned long long* keys, uint8_t* flags, cudaStream_t s);
// list (count starts at 0) <- every g < n with touched[g] == gen (the compositor's stamps)
cudaError_t launch_touched_compact(const uint32_t* touched, uint64_t n, uint32_t gen, uint32_t* list,
                                  unsigned long long* count, cudaStream_t s);
// partition_store (vecstore.hpp:169-213) scratch, n records
struct PartitionScratch {
    unsigned long long* mn3;        // [3] bbox.min as ordered keys
    unsigned long long *yz, *yz_s;  // [n] (y << 32 | z) by record; sorted scratch, then in cell order
    uint32_t *kx, *kx_p, *kx_s;     // [n] x by record, permuted, sorted
    uint32_t *idx, *perm1, *perm2;  // [n] iota, after the (y, z) pass, final record order
    uint8_t* head;                  // [n]
    uint32_t* heads;                // [n] first position of every cell
    int* n_heads;                   // cells
    int32_t* cells;                 // [3 n] (x, y, z) per cell
    uint64_t* offsets;              // [n + 1] first position per cell, then n
    float* out_rows;                // [n x dim] rows in cell order
    uint32_t* out_ids;              // [n]
    void* tmp;
    size_t tmp_bytes;
};
size_t partition_tmp_bytes(uint64_t n);
cudaError_t launch_store_partition(const float* means, const float* rows, const uint32_t* ids, uint64_t n,
                                   uint32_t dim, double cell, const PartitionScratch& w, cudaStream_t s);
// covered-row combine (ss_encode_combine with SS_OPT_COMBINE_SPARSE)
cudaError_t launch_covered_flags(const float* totals, uint64_t n, uint8_t* flags, cudaStream_t s);
// pos[0..n] exclusive prefix of flags (tmp == nullptr: *tmp_bytes <- scratch size)
cudaError_t launch_flag_positions(const uint8_t* flags, uint64_t n, uint32_t* pos, void* tmp, size_t* tmp_bytes,
                                  cudaStream_t s);
cudaError_t launch_sparse_pack(const float* sums, const float* totals, uint64_t n, uint32_t dim, uint64_t block,
                               const uint8_t* flags, const uint32_t* pos, uint64_t P, float* send_sums,
                               float* send_tot, cudaStream_t s);
cudaError_t launch_sparse_unpack(const float* recv_sums, const float* recv_tot, uint64_t block, uint64_t own0,
                                 const uint8_t* flags, const uint32_t* pos, uint32_t dim, float* rows, float* coverage,
                                 unsigned long long* covered, cudaStream_t s);
// first `take` sorted threshold keys -> (id, sim) result row, on the device
cudaError_t launch_decode_keys(const unsigned long long* keys, uint64_t take, uint32_t* ids, float* sims,
                               cudaStream_t s);
// *max_bits = max(*max_bits, bits of an upper bound of every row's L2 norm); +inf bits for non-finite rows
cudaError_t launch_row_norm_max(const float* rows, uint64_t n, uint32_t dim, unsigned int* max_bits, cudaStream_t s);

} // namespace ss
