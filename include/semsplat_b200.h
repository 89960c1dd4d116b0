/* semsplat_b200.h -- C ABI of libsemsplat_b200.so, the B200-native
 * implementation of SLAG's per-Gaussian language-embedding pass and cosine
 * top-k query (reference: /root/reference/proj/include/semsplat/, a
 * header-only C++20 CPU library with no C ABI of its own).
 *
 * Every entry point below replaces the reference function cited beside it;
 * the C++ drop-in layer (include/semsplat_b200/semsplat_b200.hpp) and the
 * Python host mirror (paper_2505_08124_b200/semsplat.py) bind these symbols
 * and re-raise the reference's exception classes from ss_last_error_kind().
 *
 * Conventions: plain C types; int return = ss_status (0 = ok); per-thread
 * ss_last_error() text; one ss_ctx per device, used from one host thread at a
 * time; host pointers unless a parameter is named d_* (device pointer).
 * All kernels are sm_100a; there is no CPU fallback -- ss_create() fails with
 * SS_ERR_CUDA when no sm_100 device is present.
 */
#ifndef SEMSPLAT_B200_H
#define SEMSPLAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error kinds, mapped onto the reference's exception taxonomy
 * (core.hpp:14-57). */
enum ss_status {
    SS_OK = 0,
    SS_ERR_CONTRACT = 1, /* ContractError  (core.hpp:27) */
    SS_ERR_DATA = 2,     /* DataError      (core.hpp:21) */
    SS_ERR_NUMERIC = 3,  /* NumericError   (core.hpp:33) */
    SS_ERR_FORMAT = 4,   /* FormatError    (core.hpp:15) */
    SS_ERR_IO = 5,       /* IoError        (core.hpp:39) */
    SS_ERR_PIPELINE = 6, /* PipelineError  (core.hpp:51) */
    SS_ERR_CUDA = 7      /* device / driver failure (no reference analogue) */
};

/* WeightMode (rasterizer.hpp:33-36) */
enum ss_weight_mode { SS_ALPHA_COMPOSITED = 0, SS_FALLOFF_ONLY = 1 };

/* CameraPose (scene.hpp:79-85) at raster resolution, i.e. after
 * camera_scaled_to (pipeline.hpp:196-207).  R is row-major world-to-camera. */
typedef struct ss_camera {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    uint32_t width, height, image_id, pad;
} ss_camera;

/* Projected2D (projection.hpp:24-31) */
typedef struct ss_projected {
    uint32_t gaussian_id;
    uint32_t visible;
    double mu_x, mu_y, cov_xx, cov_xy, cov_yy, depth;
} ss_projected;

/* WeightEntry (rasterizer.hpp:38-43) */
typedef struct ss_weight_entry {
    uint32_t gaussian_id;
    uint32_t pixel;
    float weight;
} ss_weight_entry;

/* One view's SAM masks in their on-disk encoding (providers.hpp:77-127:
 * alternating run lengths over row-major bits, zeros first) plus the mask
 * CLIP vectors (providers.hpp:156-204).  Masks are resampled to the raster
 * resolution on the device (providers.hpp:359-373). */
#define SS_MASKS_ON_DEVICE 1u /* ss_view_masks.flags: runs/run_offsets/clip are device pointers */
typedef struct ss_view_masks {
    uint32_t n_masks;
    uint32_t mask_width, mask_height;
    uint32_t flags;              /* SS_MASKS_ON_DEVICE or 0 (host pointers) */
    const uint32_t* runs;        /* all masks' runs, concatenated */
    const uint64_t* run_offsets; /* n_masks + 1 prefix offsets into runs (device: absolute) */
    const float* clip;           /* n_masks x dim, row-major */
    uint64_t n_runs;             /* total runs of the view (required with SS_MASKS_ON_DEVICE) */
} ss_view_masks;

typedef struct ss_ctx ss_ctx;

/* ---- context ---------------------------------------------------------- */
int ss_create(int device, ss_ctx** out);
void ss_destroy(ss_ctx* ctx);
const char* ss_last_error(void);
int ss_last_error_kind(void);
/* Run subsequent work on this CUDA stream (cudaStream_t as uintptr; 0 = the
 * context's own stream).  Lets a host framework order our kernels with its
 * own collectives. */
int ss_set_stream(ss_ctx* ctx, uintptr_t stream);
int ss_synchronize(ss_ctx* ctx);
/* Tuning options.  SS_OPT_LANES: per-view pipeline lanes (1..6, default 5);
 * 1 serialises views, which the bench uses for exclusive per-kernel timing.
 * SS_OPT_QUERY_PATH: 0 = auto (tensor-core coarse scoring + exact rescoring
 * for stores of >= 16384 rows with dim % 64 == 0 and dim <= 512), 1 = exact
 * scan only,
 * 2 = tensor-core path whenever dim allows.  Results are identical.
 * SS_OPT_CONTRACT_GROUP: views contracted together (1..4; default 0 = auto:
 * three consecutive views with D = 512 and <= 64 masks each, other views
 * alone): each touched Gaussian's row is read and written once per group; the
 * fp32 operation order per row is the same for every group size.
 * SS_OPT_BIN_PATH: tile lists from 0 = auto (default: direct count/scan/
 * scatter binning for views of <= 5734 16x16 tiles, else the key sort),
 * 1 = stable key sort, 2 = direct binning (up to 18000 tiles; error above).
 * The tile lists are identical.

 * SS_OPT_COMBINE_ROWS: rows per block of the block-cyclic combine (see the
 * multi-GPU section; 0 = contiguous shards).  Set before ss_encode_begin.
 * SS_OPT_RASTER: compositor schedule, 2 = one splat per step for all pixels
 * of a warp's 8x4 block, warps taking (tile, block) items from a work counter
 * on a grid of 4 CTAs per SM (default); 1 = the same per-step compositor with
 * one CTA per tile; 0 = staged evaluation (per staged chunk the box test and
 * Mahalanobis distance per splat, then exp and alpha dense over the surviving
 * pairs, then the front-to-back transmittance walk; measured slower on c4,
 * 510 vs 382 us/view).  Identical bits.
 * SS_OPT_COMBINE_SPARSE: how ss_encode_combine moves the partials: 1 =
 * only the rows some rank touched (default with a communicator of more than
 * one rank: an all-reduce of covered flags, then a reduce-scatter of the
 * covered rows packed per owner -- c4 touches ~6 % of the rows, so ~16x fewer
 * bytes than the dense reduce-scatter), 0 = every row, 2 = the covered-row
 * path even for a one-rank communicator (tests).  Same output rows.
 * SS_OPT_CONTRACT_TC: 1 = contract groups of 2-3 views (D = 512, <= 64 masks
 * each) on the tensor cores (tcgen05 kind::f16, fp16 hi/lo split, fp32 TMEM
 * accumulation; within the path's tolerance, not bit-identical to the CUDA-
 * core order); 0 = the shared-memory CUDA-core passes (default: faster on
 * c4 so far, 65 vs 82 us/view of SM time).
 * SS_OPT_DETERMINISTIC: 1 = the per-(Gaussian, mask) scalars are u64 fixed
 * point (2^-32 units) added with integer atomics: every added group sum is an
 * f32 >= 1/255, a multiple of 2^-31, so the additions are exact in any
 * order and the table is bitwise identical run to run and for every lane
 * count and contraction grouping (pipeline.hpp:272-279); 0 = f32 atomics
 * (default: 4-5 % faster on c4; results differ run to run in the last bits,
 * well inside the path's tolerance).  Set before ss_encode_begin.
 * SS_OPT_SORT_PREFIX: in the fused pass (alpha-composited, <= 128 masks) a
 * tile of n > P instances is put in (depth, id) order only over its first
 * max(P, n / 4) instances (whole key buckets, exactly the head of the full
 * order); a compositor block that reaches the end of that prefix with pixels
 * still compositing saves its transmittances, the tile is then sorted in full
 * and the block resumes where it stopped -- the same per-pixel sequence, the
 * same bits.  0 = full sorts; default 1024. */
enum ss_option {
    SS_OPT_LANES = 1,
    SS_OPT_QUERY_PATH = 2,
    SS_OPT_CONTRACT_GROUP = 3,
    SS_OPT_BIN_PATH = 4,
    SS_OPT_RASTER = 5,
    SS_OPT_COMBINE_ROWS = 6,
    SS_OPT_CONTRACT_TC = 7,
    SS_OPT_COMBINE_SPARSE = 8,
    SS_OPT_DETERMINISTIC = 9,
    SS_OPT_SORT_PREFIX = 10
};
int ss_set_option(ss_ctx* ctx, int option, int64_t value);

/* ---- scene (GaussianScene, scene.hpp:54-76) --------------------------- */
/* mean/scale: n x 3; quat_xyzw: n x 4 in Eigen coeffs() order; opacity: n.
 * Stored on the device as three float4 SoA streams. */
int ss_scene_set(ss_ctx* ctx, const float* mean, const float* scale, const float* quat_xyzw, const float* opacity,
                 uint64_t n);

/* ---- projection / rasterizer (parity entry points) -------------------- */
/* project_gaussian (projection.hpp:33-55) for every Gaussian. */
int ss_project(ss_ctx* ctx, const ss_camera* cam, ss_projected* out);
/* rasterize_weights_only (rasterizer.hpp:268-271): runs projection, depth
 * sort, tile binning and the capture-mode compositor; results stay on the
 * device until ss_raster_fetch. */
int ss_raster_capture(ss_ctx* ctx, const ss_camera* cam, int mode, uint64_t* n_entries, uint64_t* n_splats,
                      uint64_t* n_tile_instances);
/* Copies the last capture to host.  Any pointer may be NULL.
 * entries: n_entries, (pixel, front-to-back rank) order (rasterizer.hpp:250)
 * per_pixel_total / alpha: width*height (rasterizer.hpp:48-53, :231-232)
 * splat_gid: n_splats, the depth-sorted, box-culled splat list
 * tile_offsets: tiles+1; tile_splats: n_tile_instances splat indices
 * (rasterizer.hpp:183-194 tile_bins, flattened). */
/* rasterizer.hpp:261-264 rasterize: the capture above plus the rendered
 * image.  Colors (scene.hpp:28, n x 3 RGB) are uploaded once per scene with
 * ss_scene_set_color.  The WeightMap and alpha come from ss_raster_fetch; the
 * image (row-major, 3 floats per pixel; black where the total weight is
 * <= kRenderTotalEps) from ss_render_fetch_image. */
int ss_scene_set_color(ss_ctx* ctx, const float* rgb, uint64_t n);
int ss_render(ss_ctx* ctx, const ss_camera* raster_cam, int mode, uint64_t* n_entries, uint64_t* n_splats,
              uint64_t* n_tile_instances);
int ss_render_fetch_image(ss_ctx* ctx, float* rgb);
int ss_raster_fetch(ss_ctx* ctx, ss_weight_entry* entries, float* per_pixel_total, float* alpha,
                    uint32_t* splat_gid, uint32_t* tile_offsets, uint32_t* tile_splats);

/* ---- embedding pass (encode_scene, pipeline.hpp:280-470) -------------- */
/* Zeroes the per-Gaussian accumulators (N x dim fp32 sums + N fp32 totals).
 * d_sums / d_totals may be caller-owned device buffers (e.g. torch tensors
 * that a collective will reduce-scatter) or NULL for context-owned ones. */
int ss_encode_begin(ss_ctx* ctx, uint32_t dim, float* d_sums, float* d_totals);
/* One view: device RLE decode + resample to a per-pixel mask bitset, project,
 * depth sort, tile binning, fused mask-gated compositing into per-(Gaussian,
 * mask) scalars, then the sparse 512-d contraction into the sums.  Replaces
 * worker_body's per-image loop (pipeline.hpp:306-356) plus accumulate
 * (pipeline.hpp:70-86). */
int ss_encode_view(ss_ctx* ctx, const ss_camera* raster_cam, const ss_view_masks* masks, int mode);
/* Batch form: nviews cameras and mask sets, processed in order. */
int ss_encode_views(ss_ctx* ctx, uint32_t nviews, const ss_camera* raster_cams, const ss_view_masks* masks,
                    int mode);
/* finalize_into (pipeline.hpp:120-135) for rows [row_lo, row_hi) of the
 * context's accumulators: rows_out (row_hi-row_lo) x dim and coverage_out
 * (row_hi-row_lo).  out_on_device != 0: the outputs are device pointers. */
int ss_encode_finalize(ss_ctx* ctx, uint64_t row_lo, uint64_t row_hi, float* rows_out, float* coverage_out,
                       int out_on_device);
/* finalize_into (pipeline.hpp:120-135) into a host table whose rows are
 * already zero (the reference's EmbeddingTable constructor zero-fills):
 * only covered rows are normalised into rows_out / coverage_out (host
 * pointers to row row_lo), the uncovered ones are left untouched -- the
 * reference writes zeros there.  The covered rows are packed on the device
 * and scattered by id on the host, so the readout moves ~6 % of the c4
 * table.  covered_out (optional): rows written. */
int ss_encode_finalize_sparse(ss_ctx* ctx, uint64_t row_lo, uint64_t row_hi, float* rows_out, float* coverage_out,
                              uint64_t* covered_out);
/* finalize over caller-provided device buffers (a reduce-scattered shard):
 * rows d_sums[n x dim] / d_totals[n] -> d_rows_out, d_coverage_out. */
int ss_normalize_device(ss_ctx* ctx, const float* d_sums, const float* d_totals, uint64_t n, uint32_t dim,
                        float* d_rows_out, float* d_coverage_out);

/* ---- multi-GPU combine (pipeline.hpp:90-100 combine_partials + :120-141) -
 * Views shard across devices like the reference's workers
 * (pipeline.hpp:306-316); every device accumulates a full N x dim fp32
 * partial.  One NCCL reduce-scatter (sums and totals in one NCCL group) over
 * NVLink combines them, and every rank normalises the rows it receives.
 * Row ownership is block-cyclic with block B = SS_OPT_COMBINE_ROWS rows
 * (0 = one contiguous shard of ceil(N / nranks) rows per rank; otherwise
 * chunk_rows of encode_scene, pipeline.hpp:396-402): round q reduce-scatters
 * rows [q*nranks*B, (q+1)*nranks*B) and rank r receives rows
 * [q*nranks*B + r*B, q*nranks*B + (r+1)*B); the next round's collective
 * overlaps this round's normalisation.  NCCL is loaded at run time (the copy
 * already in the process, e.g. torch's, else libnccl.so.2). */
#define SS_NCCL_UNIQUE_ID_BYTES 128
/* A new NCCL unique id (rank 0 creates it; the caller ships it to the others). */
int ss_comm_unique_id(unsigned char id[SS_NCCL_UNIQUE_ID_BYTES]);
/* Join the communicator as `rank` of `nranks` (one process per device). */
int ss_comm_init(ss_ctx* ctx, int nranks, int rank, const unsigned char id[SS_NCCL_UNIQUE_ID_BYTES]);
/* One process driving several devices: ctxs[i] becomes rank i (ncclCommInitAll). */
int ss_comm_init_all(ss_ctx* const* ctxs, int n);
/* Accumulator rows to allocate (N padded to whole rounds), block rows B,
 * rounds, and the rows this rank receives (rounds * B, padding included). */
int ss_combine_layout(ss_ctx* ctx, uint64_t* rows_alloc, uint64_t* block_rows, uint64_t* rounds,
                      uint64_t* rank_rows);
/* The same layout for n rows over nranks ranks with SS_OPT_COMBINE_ROWS =
 * combine_rows (no context or device needed). */
int ss_combine_layout_for(uint64_t n, int nranks, uint64_t combine_rows, uint64_t* rows_alloc, uint64_t* block_rows,
                          uint64_t* rounds);
/* Reduce-scatter the accumulators of ss_encode_begin/ss_encode_views over the
 * communicator (a plain pass-through without one) and finalize_into the
 * received rows: rows_out (rank_rows x dim) and coverage_out (rank_rows), in
 * round order; rows past N come out zero.  out_on_device: device pointers.
 * With several ranks every rank must call it (collective). */
int ss_encode_combine(ss_ctx* ctx, float* rows_out, float* coverage_out, int out_on_device);
/* Number of CUDA devices visible to the library. */
int ss_device_count(int* n);

/* ---- vector store + query (vecstore.hpp:21-146) ----------------------- */
/* build_store (vecstore.hpp:88-103): covered rows of a table -> unit rows
 * (normalized_copy, vecstore.hpp:34-42, f64 norm).  Keeps the store on the
 * device; returns the number of covered rows. */
int ss_store_build(ss_ctx* ctx, const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                   uint64_t* count_out);
/* Upload an already-normalized store (ids + unit rows). */
int ss_store_set(ss_ctx* ctx, const uint32_t* ids, const float* unit_rows, uint64_t count, uint32_t dim);
/* Fetch the device store (ids: count; unit_rows: count x dim). */
int ss_store_fetch(ss_ctx* ctx, uint32_t* ids, float* unit_rows);
/* partition_store (vecstore.hpp:169-213) of the device store: records grouped
 * by the uniform grid cell floor((mean - bbox.min) / cell_size) of their
 * payload means (means_xyz: 3 floats per record, store order, host memory;
 * bbox.min over the means widened to f64, NaN skipped), cells in (x, y, z)
 * order, records in store order within a cell, out-of-range cell indices
 * INT_MIN (x86 conversion).  ContractError unless cell_size > 0.  The result
 * stays on the device until ss_store_partition_fetch. */
int ss_store_partition(ss_ctx* ctx, const float* means_xyz, double cell_size, uint64_t* n_cells);
/* Results of the last ss_store_partition (any pointer may be NULL):
 * cells 3 x n_cells int32 (x, y, z); offsets n_cells + 1 (first record
 * position of each cell, then count); order count (store record index at
 * each position); ids count and rows count x dim in cell order; bbox_min 3. */
int ss_store_partition_fetch(ss_ctx* ctx, int32_t* cells, uint64_t* offsets, uint32_t* order, uint32_t* ids,
                             float* rows, double* bbox_min);
/* query_topk (vecstore.hpp:121-132) for nq queries (raw, un-normalized):
 * out_ids/out_sims nq x k; out_counts[q] = min(k, count). */
int ss_query_topk(ss_ctx* ctx, const float* queries, uint32_t nq, uint32_t k, uint32_t* out_ids, float* out_sims,
                  uint64_t* out_counts);
/* query_threshold (vecstore.hpp:135-146) for one query: all sims >= tau,
 * (sim desc, id asc).  capacity = size of out arrays. */
int ss_query_threshold(ss_ctx* ctx, const float* query, float tau, uint32_t* out_ids, float* out_sims,
                       uint64_t capacity, uint64_t* out_count);

/* ---- instrumentation --------------------------------------------------- */
/* Per-kernel-class device time (CUDA events on the launching stream) and
 * algorithmic byte/flop counts, accumulated while enabled. */
enum ss_kernel_class {
    SS_K_MASKS = 0,    /* RLE decode + resample into per-pixel bitsets */
    SS_K_PROJECT = 1,  /* project (+ ordered compaction) */
    SS_K_SORT = 2,     /* depth sort + tile-key sort */
    SS_K_BIN = 3,      /* record gather, tile counts, key emission, ranges */
    SS_K_RASTER = 4,   /* fused mask-gated compositor */
    SS_K_CONTRACT = 5, /* sparse 512-d contraction */
    SS_K_NORMALIZE = 6,
    SS_K_QUERY = 7,
    SS_K_H2D = 8,
    SS_K_QUERY_GEMM = 9,    /* tcgen05 coarse scores (inside SS_K_QUERY) */
    SS_K_QUERY_SELECT = 10, /* candidate selection + exact rescoring (inside SS_K_QUERY) */
    SS_K_COMBINE = 11,      /* NCCL reduce-scatter of the partials (bytes: sent per rank) */
    SS_K_COUNT = 12
};
int ss_profile_enable(ss_ctx* ctx, int on);
int ss_profile_reset(ss_ctx* ctx);
/* ms[SS_K_COUNT], launches[SS_K_COUNT], bytes[SS_K_COUNT] (algorithmic). */
int ss_profile_read(ss_ctx* ctx, double* ms, uint64_t* launches, double* bytes);
/* Running totals of the geometry counters (SURVEY.md 8 notation), summed over
 * views since ss_profile_reset: [0]=N_vis [1]=I_v [2]=G_v [3]=K_v [4]=views. */
int ss_counters_read(ss_ctx* ctx, uint64_t* out5);
/* eval.hpp:122-158 assign_classes: arg-max cosine class per covered row of an
 * EmbeddingTable (uncovered rows -1 = kUnlabeled, ties to the lowest class
 * id), bit-identical to the reference (sequential f64 dots).  rows (n x dim)
 * and coverage (n) are host arrays, or device pointers with
 * SS_ROWS_ON_DEVICE; label_vecs is n_labels x dim, label_ids n_labels. */
#define SS_ROWS_ON_DEVICE 1
int ss_assign_classes(ss_ctx* ctx, const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                      const int32_t* label_ids, const float* label_vecs, uint32_t n_labels, int32_t* out, int flags);
/* Tensor-core query statistics since reset: queries answered on that path,
 * total and maximum candidates per query, batches answered by the exact scan
 * after a candidate overflow. */
int ss_query_stats(ss_ctx* ctx, uint64_t* out4);
/* Measurement helper: the device's fp64 pipe rate in DFMA lane-operations
 * per second (eight independent chains per thread on every SM), the
 * denominator of the compositor's fp64 roofline in bench.py. */
int ss_probe_fp64_rate(ss_ctx* ctx, double* lane_ops_per_s);
/* Number of kernels this library launched (own + CUB) since reset. */
int ss_launch_count(ss_ctx* ctx, uint64_t* own, uint64_t* cub);

#ifdef __cplusplus
}
#endif
#endif /* SEMSPLAT_B200_H */
