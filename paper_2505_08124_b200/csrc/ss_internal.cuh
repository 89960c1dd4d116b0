// Internal declarations shared by the libsemsplat_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/semsplat_b200.h"

namespace ss {

constexpr uint32_t kTile = 16;          // rasterizer.hpp:30 kTileSize
constexpr int kRasterThreads = 256;     // pixels of a 16x16 tile
constexpr int kMaxMaskWords = 4;        // masks per compositor pass: views with more run 128-mask windows

// Per-splat record staged through shared memory by the compositor: exactly
// the six doubles it reads (48 B, three 16 B vectors; a batch of 256 is 12 KB).
// Fields are the reference's SplatRecord (rasterizer.hpp:99-106) minus color,
// id and box (the box is the separate `boxes` array, the id comes from the
// tile list).
struct __align__(16) SplatRec {
    double mu_x, mu_y; // rasterizer.hpp:101
    double a, b2;      // conic (rasterizer.hpp:66-71); b2 = 2*b (exact)
    double c;
    double opacity;    // SplatRecord::opacity: the f32 opacity widened once
};
static_assert(sizeof(SplatRec) == 48, "SplatRec must stay 48 B");

// Per-(Gaussian, mask) weight scalars (mask_weights, pipeline.hpp:25-49):
// f32 by default; with SS_OPT_DETERMINISTIC u64 fixed point in units of
// 2^-32.  Every value the compositor adds is an f32 sum of emitted weights,
// each >= 1/255 > 2^-8, hence a multiple of 2^-31: the integer atomics add it
// exactly and in any order, so the scalars -- and everything contracted from
// them -- are bitwise identical run to run and for any lane count (the
// reference's determinism contract, pipeline.hpp:272-279), where f32 atomics
// round in arrival order.  (Measured on c4: 4-5 % slower, the 64-bit
// atomics and the doubled scalar reads.)
typedef unsigned long long acc_t;
__device__ __forceinline__ acc_t acc_fix(float v) { return __float2ull_rn(v * 4294967296.0f); }
__device__ __forceinline__ float acc_val(acc_t a) { return __ull2float_rn(a) * 2.3283064365386963e-10f; }

// Per-view scalars kept on the device; the host reads them only at batch
// boundaries (copied into a per-view status array), never per view.
struct ViewInfo {
    unsigned long long n_surv;       // visible, box-non-empty splats
    unsigned long long min_key;      // min / max depth bit patterns over them
    unsigned long long max_key;
    unsigned long long n_instances;  // tile instances I_v (total of tile_count)
    unsigned int err_count;          // singular screen covariances
    unsigned int err_gid;            // smallest gid with one
    unsigned long long n_touched;    // G_v (Gaussians with any masked weight)
    unsigned int overflow;           // tile lists unusable: compositor skips, the host re-runs the view
    unsigned int bin_fallback;       // tile-sort binning: 1 = a tile outgrew its slot capacity (grow it),
                                     // 2 = beyond the in-CTA sort (re-run with the global depth sort)
    unsigned int max_fill;           // tile-sort binning: largest tile list
    unsigned int pad;
};

struct ProjectParams {
    const float4* mean_op; // x, y, z, opacity
    const float4* scale;   // sx, sy, sz, -
    const float4* quat;    // x, y, z, w (Eigen coeffs order)
    const double* cov3;    // [9][n] 3-D covariances (cov3d_kernel, per scene)
    uint64_t n;
    ss_camera cam;
    SplatRec* rec;        // [n] by gid
    uint2* boxes;         // [n] by gid: (x0 | x1 << 16, y0 | y1 << 16), L2-resident copy of the records' boxes
                          // (0xffffffff, 0xffffffff) for Gaussians that do not survive
    unsigned long long* keys; // [n] depth bits (~0 when culled)
    uint32_t* tile_count; // [tiles] instances per tile (atomic), or null
    uint32_t tiles_x;
    ViewInfo* info;
    ss_projected* dbg;    // optional Projected2D dump (parity entry point)
};

struct RasterParams {
    const SplatRec* rec;        // by Gaussian id
    const uint2* boxes;         // by Gaussian id (compact copy of rec[].x0..y1)
    const uint32_t* tile_list;  // per tile: Gaussian ids in (depth, id) order
    const uint32_t* tile_start; // tile t is tile_list[start[t], end[t])
    const uint32_t* tile_end;
    uint32_t width, height, tiles_x;
    uint32_t algo;                 // compositor (SS_OPT_RASTER): 1 = per-step, CTA per tile; 2 = per-step,
                                   // work-stealing warps (needs work); 0 = staged evaluation
    uint32_t* work;                // [2] zero-initialised counters of the work-stealing grid (one pair per stream)
    uint32_t n_tiles;              // set by the launcher
    // capture mode
    uint32_t* pix_count;           // pass 0 output [P]
    const uint32_t* pix_offset;    // pass 1 input  [P]
    ss_weight_entry* entries;      // pass 1 output
    float* per_pixel_total;        // pass 1 output [P]
    float* alpha;                  // pass 1 output [P]
    const float4* color;           // render: Gaussian colors (r, g, b, -) by id
    float* image;                  // render output [P * 3], zero where no weight
    // fused mode
    const uint32_t* pix_bits;      // [P * bits_stride]
    uint32_t mask_words, n_masks;  // words of this pass's window (1, 2 or 4); masks of the view
    uint32_t bits_stride;          // words per pixel in pix_bits (= mask_words unless windowed)
    uint32_t mask_base;            // first mask of the window (multiple of 128; word offset mask_base / 32)
    void* acc;                     // [N * n_masks] per-(Gaussian, mask) scalars: float, or acc_t (KIND 4)
    uint32_t acc_fix;              // scalars are acc_t (SS_OPT_DETERMINISTIC): the compositor runs KIND 4
    uint32_t* touched;             // [N] generation stamp of the last view that touched the Gaussian
    uint32_t* touched_list;        // [N] Gaussian ids touched in this view
    unsigned long long* touched_count; // entries of touched_list
    uint32_t gen;                  // this view's stamp (never 0)
    ViewInfo* info;
    // prefix-sorted tile lists (fused pass, SS_OPT_SORT_PREFIX): tile t's list
    // holds the first end - start of tile_full[t] instances; a block that
    // exhausts it with live pixels saves its state and is resumed after the
    // fixup sort (raster_resume_kernel)
    const uint32_t* tile_full;     // [tiles] instances per tile, or null (full lists)
    double* rs_T;                  // [tiles * 8 * 32] saved transmittance per pixel
    uint2* rs_state;               // [tiles * 8] (live lanes, list position reached)
    uint32_t* rs_items;            // [tiles * 8] (tile << 3 | block) to resume
    uint32_t* rs_count;            // [2]: items, tiles queued for the fixup sort
    uint32_t* rs_tiles;            // [tiles] tiles queued for the fixup sort
    uint32_t* rs_need;             // [tiles] tile queued (the fixup clears it)
};

// Kernel launchers (return cudaError_t of the launch).
cudaError_t launch_project(const ProjectParams& p, cudaStream_t s);
cudaError_t probe_fp64_rate(double* lane_ops_per_s); // DFMA lane-operations per second, whole device
cudaError_t launch_cov3d(const float4* scale, const float4* quat, uint64_t n, double* cov3, cudaStream_t s);
cudaError_t launch_raster_count(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s);
cudaError_t launch_raster_capture(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s);
cudaError_t launch_raster_render(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s);
cudaError_t launch_raster_fused(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s);
// the blocks a prefix-sorted fused pass left unfinished, after the fixup sort
cudaError_t launch_raster_resume(const RasterParams& p, int mode, cudaStream_t s);

} // namespace ss
