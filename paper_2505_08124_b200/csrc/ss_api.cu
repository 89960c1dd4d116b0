// libsemsplat_b200 host runtime: the C ABI of include/semsplat_b200.h.
//
// One ss_ctx per device.  It owns the resident scene (float4 SoA), the
// capacity-managed per-view scratch, the per-(rank, mask) scalar buffer and
// the N x D fp32 accumulators, and drives the per-view pipeline
//   RLE -> bitset -> project -> ordered compaction -> depth radix sort ->
//   record gather + tile counts -> scan -> key emission -> tile radix sort ->
//   tile ranges -> fused compositor -> sparse contraction
// on one CUDA stream.  Replaces encode_scene's phase 1/phase 2 loops
// (pipeline.hpp:280-470) for the views handed to it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h> // types only: the library is resolved at run time (nccl_api)

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <thrust/iterator/counting_iterator.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "ss_kernels.cuh"

// SS_OPT_SORT_PREFIX default: tiles of more than this many instances are
// ranked over their first max(this, n / 4) instances in the fused pass
#ifndef SS_SORT_PREFIX_DEFAULT
#define SS_SORT_PREFIX_DEFAULT 1024
#endif
#include "ss_query_tc.cuh"

namespace ss {
namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

struct Error : std::runtime_error {
    int kind;
    Error(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

#define SS_CUDA(expr)                                                                                       \
    do {                                                                                                    \
        cudaError_t _e = (expr);                                                                            \
        if (_e != cudaSuccess)                                                                              \
            throw Error(SS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" __FILE__ ":" + \
                                         std::to_string(__LINE__) + ")");                                   \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        g_kind = 0;
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        g_kind = e.kind;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        g_kind = SS_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = SS_ERR_CUDA;
    }
    return g_kind;
}

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* ensure(size_t want) {
        if (want <= bytes && p) return p;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t cap = std::max<size_t>(want, 256);
        cap = (cap + cap / 8 + 255) & ~(size_t)255; // slack so slowly growing sizes do not thrash; 256-B granules
        SS_CUDA(cudaMalloc(&p, cap));
        bytes = cap;
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct ProfState {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double ms[SS_K_COUNT] = {};
    uint64_t launches[SS_K_COUNT] = {};
    double bytes[SS_K_COUNT] = {};
    cudaEvent_t get() {
        if (pool.empty()) {
            cudaEvent_t e;
            SS_CUDA(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
};

// Per-view scratch + stream of one pipeline lane.  Consecutive views
// alternate between two lanes so one view's sorts and host handshakes overlap
// the previous view's compositor; the contraction into the shared N x D sums
// stays in view order through an event chain.
// What a view leaves for the group contraction: per-(Gaussian, mask) scalars,
// the touched list/stamps/count and its CLIP rows.  Two per lane, alternating
// by group, so a lane's next view never waits for the previous group's
// contraction.
struct ContractSet {
    DevBuf acc, touched, touched_list, clip, tcount;
    uint64_t acc_elems = 0;        // zero-initialised elements of acc
    bool acc_fix = false;          // acc holds acc_t (fixed point) rather than float
    uint32_t gen = 0;              // last stamp handed out
    cudaEvent_t free_ev = nullptr; // recorded after the contraction that consumed this set
    bool pending = false;          // a contraction reading this set has been issued
    bool in_group = false;         // part of the group being formed
    bool dirty = false;            // rasterized into but never contracted (error path): acc must be zeroed
    void release() {
        DevBuf* b[] = {&acc, &touched, &touched_list, &clip, &tcount};
        for (auto* x : b) x->release();
        if (free_ev) cudaEventDestroy(free_ev);
        free_ev = nullptr;
        acc_elems = 0;
        gen = 0;
        pending = false;
        in_group = false;
        dirty = false;
    }
};

struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t contract_done = nullptr, done = nullptr, raster_done = nullptr;
#ifndef SS_LANE_SETS
#define SS_LANE_SETS 2
#endif
    ContractSet sets[SS_LANE_SETS]; // per-(Gaussian, mask) scalars in flight per lane (views awaiting contraction)
    uint32_t set_next = 0;
    DevBuf rec, boxes, rbox, rcnt, keys, k32, k32s, order, iota, offsets, tkeys, tkeys_sorted, tvals, tile_start, tile_end, list;
    DevBuf bin_counts, bin_slice, bin_tot, bin_done; // direct binning scratch
    DevBuf ts_fill, ts_slab;       // tile-sort binning: per-tile fill counters, unordered (key, gid) slots
    DevBuf raster_work;            // work-stealing compositor counters (zero between launches)
    // prefix-sorted tile lists (SS_OPT_SORT_PREFIX): saved block state of the
    // fused pass, queued blocks / tiles, the fixup sort's parameters
    DevBuf rs_T, rs_state, rs_items, rs_tiles, rs_need, rs_count;
    uint32_t rs_tiles_cap = 0;     // tiles the rs_* buffers hold
    TileSortParams ts_params{};    // the view's tile-sort binning (for the fixup sort)
    uint32_t ts_cap = kTileSortMax / 2; // tile-sort slots per tile: grows to kTileSortMax when a tile
                                        // outgrows it (larger tiles take the global path)
    uint64_t iota_n = 0;           // entries of the 0..n-1 sequence in `iota`
    uint64_t list_cap = 0;         // entries of `list`
    DevBuf cub_tmp, info;
    DevBuf pix_bits, mask_bits, runs, run_offsets, spans;
    ViewInfo* h_info = nullptr;    // pinned
    uint32_t* h_u32 = nullptr;     // pinned scratch
    void release_all() {
        DevBuf* b[] = {&rec, &boxes, &rbox, &rcnt, &keys, &k32, &k32s, &order, &iota, &offsets, &tkeys, &tkeys_sorted, &tvals, &tile_start,
                       &tile_end, &list, &cub_tmp, &info, &raster_work, &pix_bits, &mask_bits, &bin_counts, &bin_slice, &bin_tot, &bin_done,
                       &runs, &run_offsets, &spans, &ts_fill, &ts_slab, &rs_T, &rs_state, &rs_items, &rs_tiles,
                       &rs_need, &rs_count};
        for (auto* x : b) x->release();
        for (auto& cs : sets) cs.release();
        if (raster_done) cudaEventDestroy(raster_done);
        raster_done = nullptr;
        if (h_info) cudaFreeHost(h_info);
        if (h_u32) cudaFreeHost(h_u32);
        if (contract_done) cudaEventDestroy(contract_done);
        if (done) cudaEventDestroy(done);
        if (stream) cudaStreamDestroy(stream);
        h_info = nullptr;
        h_u32 = nullptr;
        contract_done = done = nullptr;
        stream = nullptr;
    }
};

struct GroupMember {
    Lane* lane;
    ContractSet* set;
    uint32_t n_masks;
    const float* clip;
};

} // namespace
} // namespace ss

struct ss_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;

    // scene
    uint64_t n = 0;
    ss::DevBuf mean_op, scale, quat, cov3; // cov3: [9][n] f64 3-D covariances (per scene)

    // per-view pipeline lanes (scratch + stream each)
    static constexpr uint32_t kMaxLanes = 6;
    ss::Lane lanes[kMaxLanes];
    uint32_t next_lane = 0;
    uint32_t n_lanes = 5;
    cudaEvent_t ev_user = nullptr;
    // contraction group: consecutive views whose contraction is issued together
    std::vector<ss::GroupMember> group;
    cudaStream_t cstream = nullptr;      // group contractions (keeps lanes free)
    uint32_t group_max = 0;              // SS_OPT_CONTRACT_GROUP (0 = auto)
    cudaEvent_t group_done = nullptr;
    bool group_done_valid = false;
    ss::DevBuf cub_tmp, num_sel, info; // store / query scratch
    ss::DevBuf vstat; // per-view status of the last batch
    ss::DevBuf union_list, union_count; // group contraction scratch
    ss::DevBuf tc_scratch;              // tensor-core contraction: prepared CLIP operands
    uint64_t cap_n_surv = 0;
    ss::ViewInfo* h_init = nullptr;    // pinned
    uint32_t* h_u32 = nullptr;         // pinned scratch
    char* h_stage = nullptr;           // pinned staging for readouts into pageable memory (kStageBytes x 2)
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};

    // capture / render
    ss::DevBuf pix_count, pix_offset, entries, per_pixel_total, alpha, color, image;
    bool color_ok = false;     // colors uploaded for the current scene
    bool cap_image = false;    // the last capture rendered an image
    uint64_t cap_entries = 0, cap_splats = 0, cap_instances = 0;
    bool cap_tile_sort = false; // the last capture's lists are per-tile slot ranges
    uint32_t cap_width = 0, cap_height = 0, cap_tiles = 0;
    ss::DevBuf counters; // [0] G_v sum, [1] K_v sum, [2] contraction rows RMW, [3] covered rows normalised
    // accumulators
    uint32_t dim = 0;
    float* sums = nullptr;
    float* totals = nullptr;
    bool own_acc = false;
    ss::DevBuf sums_buf, totals_buf;
    ss::DevBuf sparse_out; // ss_encode_finalize_sparse: packed covered rows
    // store + query
    ss::DevBuf store_rows, store_ids, qbuf, qnorm, scores, topk_ids, topk_sims, sel_flags, thr_keys, thr_keys_sorted,
        thr_ids, thr_ids_sorted, zero_flag;
    uint64_t store_count = 0;
    uint32_t store_dim = 0;
    // tensor-core query path: fp16 copy of the store, coarse scores, candidates
    ss::DevBuf store_half, qhalf, tc_scores, tc_thr, cand, cand_count, cand_sim;
    ss::DevBuf part_buf, part_means; // partition_store scratch + the records' means
    ss::PartitionScratch part{};
    uint64_t part_cells = 0;         // cells of the last ss_store_partition
    double part_min[3] = {0, 0, 0};  // its bbox.min
    bool store_half_ok = false;
    // upper bound of the store's row norms (1 for build_store's unit rows):
    // the tensor-core query's error margin scales with it
    float store_norm = 1.0f;
    int query_path = 0; // SS_OPT_QUERY_PATH
    int bin_path = 0;   // SS_OPT_BIN_PATH
    int contract_tc = 0; // SS_OPT_CONTRACT_TC
    uint32_t sort_prefix = SS_SORT_PREFIX_DEFAULT; // SS_OPT_SORT_PREFIX (0: full tile sorts)
    bool deterministic = false; // SS_OPT_DETERMINISTIC: fixed-point per-(Gaussian, mask) scalars
    int raster_algo = 2; // SS_OPT_RASTER (2 = per-step compositor on work-stealing warps, the fastest on c4)
    int num_sms = 0;

    // multi-GPU combine (ss_comm_*, ss_encode_combine)
    ncclComm_t comm = nullptr;
    bool own_comm = false;
    int nranks = 1, rank = 0;
    uint64_t combine_rows = 0;            // SS_OPT_COMBINE_ROWS
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_acc = nullptr, ev_rs[2] = {nullptr, nullptr}, ev_norm[2] = {nullptr, nullptr};
    ss::DevBuf rs_sum[2], rs_tot[2], rs_stage;
    int combine_sparse = 1;             // SS_OPT_COMBINE_SPARSE: 0 dense, 1 covered rows (with a communicator), 2 forced
    ss::DevBuf sp_flags, sp_pos, sp_tmp, sp_send, sp_bounds;
    uint64_t acc_rows = 0;                // accumulator rows (N padded to whole combine rounds)

    // instrumentation
    ss::ProfState prof;
    uint64_t launches_own = 0, launches_cub = 0;
    uint64_t cnt_vis = 0, cnt_inst = 0, cnt_views = 0;
    uint64_t qstat[4] = {}; // tensor-core queries, candidates, max candidates, exact fallbacks
};

namespace ss {
namespace {

struct Scope {
    ss_ctx* c;
    cudaStream_t st;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    Scope(ss_ctx* ctx, cudaStream_t stream, int k) : c(ctx), st(stream), cls(k) {
        if (c->prof.on) {
            a = c->prof.get();
            b = c->prof.get();
            SS_CUDA(cudaEventRecord(a, st));
        }
    }
    ~Scope() {
        if (c->prof.on && a) {
            cudaEventRecord(b, st);
            c->prof.pending.push_back({cls, {a, b}});
        }
    }
};

inline void own_launch(ss_ctx* c, cudaError_t e, int cls, uint64_t count = 1) {
    if (e != cudaSuccess) throw Error(SS_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
    c->launches_own += count;
    c->prof.launches[cls] += count;
}

void set_device(ss_ctx* c) { SS_CUDA(cudaSetDevice(c->device)); }

void reset_info(ss_ctx* c, Lane& L, cudaStream_t s) {
    SS_CUDA(cudaMemcpyAsync(L.info.p, c->h_init, sizeof(ViewInfo), cudaMemcpyHostToDevice, s));
}

uint32_t bits_for(uint64_t v) { // number of bits to represent v (v >= 1 -> >= 1)
    uint32_t b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b ? b : 1;
}

void check_camera(const ss_camera* cam) {
    if (!cam) throw Error(SS_ERR_CONTRACT, "camera is null");
    if (cam->width == 0 || cam->height == 0) throw Error(SS_ERR_DATA, "camera has zero raster resolution");
    if (cam->width > 65535 || cam->height > 65535)
        throw Error(SS_ERR_CONTRACT, "raster resolution above 65535 is not supported");
}

// rasterizer.hpp:66-70,187-191: conic_of throws for the first singular
// projection in depth order (it runs over the depth-sorted visible list before
// any box cull).  The kernels only count singular covariances; on that (rare)
// error path the view is projected again with the Projected2D dump and the
// host picks the first (depth, id) one, so the error names the same Gaussian.
uint32_t first_singular_gid(ss_ctx* c, const ss_camera& cam) {
    const uint64_t N = c->n;
    std::vector<ss_projected> h(N);
    if (ss_project(c, &cam, h.data()) != SS_OK) throw Error(SS_ERR_CUDA, "re-projection failed: " + g_err);
    uint64_t best = N;
    for (uint64_t k = 0; k < N; ++k) {
        const ss_projected& q = h[k];
        if (!q.visible) continue;
        const double det = q.cov_xx * q.cov_yy - q.cov_xy * q.cov_xy; // conic_of, no FMA (x86-64 baseline)
        if (!(det < 1e-12)) continue;
        if (best == N || q.depth < h[best].depth) best = k; // ids ascend: ties keep the lower id
    }
    return best == N ? 0xffffffffu : (uint32_t)best;
}

struct Geometry {
    uint32_t tiles_x = 0, tiles_y = 0, tiles = 0;
    bool k16 = true; // 16-bit tile keys
    bool tile_sort = false; // lists from the tile-sort binning (no global depth order)
    bool prefix = false;    // tile lists sorted only over a prefix (fused pass resumes the rest)
};

// The fused pass bins by tile sort (SS_OPT_BIN_PATH 0 or 3) unless the view
// needs the global depth order (captures report it) or was sent back to the
// global path (bin_fallback 2).
bool use_tile_sort(const ss_ctx* c, uint32_t tiles, bool force_global) {
    if (force_global) return false;
    return (c->bin_path == 0 || c->bin_path == 3) && tiles <= tile_sort_max_tiles();
}

// project (+ per-tile instance counts) -> scan -> scatter ids into tile
// slices -> per-tile (depth, id) sort.  No host synchronisation: sizes,
// offsets and key ranges stay on the device; a view whose tile lists would
// overflow the list buffer raises info->overflow and its compositor skips.
Geometry run_geometry(ss_ctx* c, Lane& L, cudaStream_t s, const ss_camera& cam, bool force_global = false,
                      bool need_order = false, uint32_t prefix_min = 0) {
    Geometry g;
    const uint64_t N = c->n;
    g.tiles_x = (cam.width + kTile - 1) / kTile;
    g.tiles_y = (cam.height + kTile - 1) / kTile;
    g.tiles = g.tiles_x * g.tiles_y;

    auto* rec = static_cast<SplatRec*>(L.rec.ensure(std::max<uint64_t>(N, 1) * sizeof(SplatRec)));
    auto* boxes = static_cast<uint2*>(L.boxes.ensure(std::max<uint64_t>(N, 1) * sizeof(uint2)));
    auto* keys = static_cast<unsigned long long*>(L.keys.ensure(std::max<uint64_t>(N, 1) * 8));
    if (g.tiles > 50000u) throw Error(SS_ERR_CONTRACT, "raster resolution too large (more than 50000 16x16 tiles)");
    auto* tstart = static_cast<uint32_t*>(L.tile_start.ensure((g.tiles + 1ull) * 4));
    auto* tend = static_cast<uint32_t*>(L.tile_end.ensure((g.tiles + 1ull) * 4));
    g.k16 = g.tiles <= 65535u;
    if (L.list_cap == 0) L.list_cap = std::max<uint64_t>(4 * N, 1u << 20);
    auto* list = static_cast<uint32_t*>(L.list.ensure(L.list_cap * 4));
    const uint32_t bin_warps = bin_scatter_warps(g.tiles);
    if (c->bin_path == 2 && !bin_warps)
        throw Error(SS_ERR_CONTRACT, "SS_OPT_BIN_PATH=2: too many tiles for the direct binning path");
    // auto: the direct path where its scatter runs 8-warp CTAs (<= 5734 tiles);
    // with 4-warp CTAs (larger views) the key sort is faster (c3: 1029 vs 989 views/s)
    const bool direct = c->bin_path == 2 || (c->bin_path != 1 && bin_warps == 8);
    if (c->bin_path == 3 && g.tiles > tile_sort_max_tiles())
        throw Error(SS_ERR_CONTRACT, "SS_OPT_BIN_PATH=3: too many tiles for the tile-sort binning");
    if (!direct && !use_tile_sort(c, g.tiles, force_global)) {
        L.tkeys.ensure(L.list_cap * (g.k16 ? 2 : 4));
        L.tkeys_sorted.ensure(L.list_cap * (g.k16 ? 2 : 4));
        L.tvals.ensure(L.list_cap * 4);
    }
    ViewInfo* info = L.info.as<ViewInfo>();

    reset_info(c, L, s);
    {
        Scope sc(c, s, SS_K_PROJECT);
        ProjectParams p;
        p.mean_op = c->mean_op.as<float4>();
        p.scale = c->scale.as<float4>();
        p.quat = c->quat.as<float4>();
        p.cov3 = c->cov3.as<double>();
        p.n = N;
        p.cam = cam;
        p.rec = rec;
        p.boxes = boxes;
        p.keys = keys;
        p.tile_count = nullptr;
        p.tiles_x = g.tiles_x;
        p.info = info;
        p.dbg = nullptr;
        own_launch(c, launch_project(p, s), SS_K_PROJECT);
        c->prof.bytes[SS_K_PROJECT] += 44.0 * (double)N;
    }
    g.tile_sort = use_tile_sort(c, g.tiles, force_global);
    if (g.tile_sort) {
        // tile-sort binning: unordered per-tile slots, then an exact per-tile sort
        Scope sc(c, s, SS_K_BIN);
        TileSortParams tp;
        tp.boxes = boxes;
        tp.keys = keys;
        tp.n = N;
        tp.tiles = g.tiles;
        tp.tiles_x = g.tiles_x;
        tp.cap = L.ts_cap;
        const uint64_t slots = (uint64_t)g.tiles * L.ts_cap;
        tp.fill = static_cast<uint32_t*>(L.ts_fill.ensure((g.tiles + 1ull) * 4));
        tp.slab = static_cast<uint2*>(L.ts_slab.ensure(slots * 8));
        if (L.list_cap < slots) {
            L.list_cap = slots;
            list = static_cast<uint32_t*>(L.list.ensure(L.list_cap * 4));
        }
        tp.list = list;
        tp.start = tstart;
        tp.end = tend;
        tp.info = info;
        tp.prefix_min = 0;
        tp.fix_tiles = nullptr;
        tp.fix_count = nullptr;
        tp.need = nullptr;
        if (prefix_min && !need_order) {
            // prefix mode: per-block resume state, zero / NaN between views
            // (the resume and fixup kernels reset what they consume)
            if (L.rs_tiles_cap < g.tiles) {
                const uint64_t items = (uint64_t)g.tiles * 8u;
                L.rs_T.release();
                L.rs_state.release();
                L.rs_need.release();
                SS_CUDA(cudaMemsetAsync(L.rs_T.ensure(items * 32u * 8u), 0xff, items * 32u * 8u, s));
                SS_CUDA(cudaMemsetAsync(L.rs_state.ensure(items * 8u), 0, items * 8u, s));
                L.rs_items.ensure(items * 4u);
                L.rs_tiles.ensure((uint64_t)g.tiles * 4u);
                SS_CUDA(cudaMemsetAsync(L.rs_need.ensure((uint64_t)g.tiles * 4u), 0, (uint64_t)g.tiles * 4u, s));
                L.rs_count.ensure(16);
                L.rs_tiles_cap = g.tiles;
            }
            SS_CUDA(cudaMemsetAsync(L.rs_count.p, 0, 8, s));
            tp.prefix_min = prefix_min;
            tp.fix_tiles = L.rs_tiles.as<uint32_t>();
            tp.fix_count = L.rs_count.as<uint32_t>();
            tp.need = L.rs_need.as<uint32_t>();
            g.prefix = true;
        }
        L.ts_params = tp;
        own_launch(c, launch_tile_sort_bin(tp, s), SS_K_BIN, 2);
        if (!need_order) return g;
    }
    auto* k32 = static_cast<uint32_t*>(L.k32.ensure(std::max<uint64_t>(N, 1) * 4));
    auto* k32s = static_cast<uint32_t*>(L.k32s.ensure(std::max<uint64_t>(N, 1) * 4));
    auto* order = static_cast<uint32_t*>(L.order.ensure(std::max<uint64_t>(N, 1) * 4));
    {
        // depth order of all Gaussians (culled ones last), no host round trip
        Scope sc(c, s, SS_K_SORT);
        own_launch(c, launch_narrow_keys(keys, N, info, k32, s), SS_K_SORT);
        if (L.iota_n < N) {
            std::vector<uint32_t> h(N);
            for (uint64_t i = 0; i < N; ++i) h[i] = (uint32_t)i;
            SS_CUDA(cudaMemcpy(L.iota.ensure(N * 4), h.data(), N * 4, cudaMemcpyHostToDevice));
            L.iota_n = N;
        }
        const uint32_t* iota = L.iota.as<uint32_t>();
        size_t tb = 0;
        SS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k32, k32s, iota, order, (int)N, 0, 32, s));
        void* tmp = L.cub_tmp.ensure(tb);
        tb = L.cub_tmp.bytes;
        SS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k32, k32s, iota, order, (int)N, 0, 32, s));
        c->launches_cub += 1;
        c->prof.launches[SS_K_SORT] += 1;
        own_launch(c, launch_tie_fixup(k32s, N, keys, order, s), SS_K_SORT);
    }
    if (g.tile_sort) return g; // the depth order was only wanted for reporting (captures)
    if (direct) {
        // count / scan / scatter straight into the tile slices (no key sort)
        Scope sc(c, s, SS_K_BIN);
        if (!L.bin_done.p) {
            L.bin_done.ensure(4);
            SS_CUDA(cudaMemset(L.bin_done.p, 0, 4));
        }
        BinParams bp;
        bp.boxes = boxes;
        bp.order = order;
        bp.n = N;
        bp.tiles = g.tiles;
        bp.tiles_x = g.tiles_x;
        bp.rbox = static_cast<uint2*>(L.rbox.ensure(std::max<uint64_t>(N, 1) * sizeof(uint2)));
        bp.counts = static_cast<uint32_t*>(L.bin_counts.ensure(std::max<size_t>(bin_counts_entries(N, g.tiles), 1) * 4));
        bp.slice = static_cast<uint32_t*>(L.bin_slice.ensure(32ull * g.tiles * 4));
        bp.tot = static_cast<uint32_t*>(L.bin_tot.ensure((g.tiles + 1ull) * 4));
        bp.done = L.bin_done.as<uint32_t>();
        bp.start = tstart;
        bp.end = tend;
        bp.list = list;
        bp.cap = L.list_cap;
        bp.info = info;
        own_launch(c, launch_bin(bp, s), SS_K_BIN, 3);
        return g;
    }
    {
        Scope sc(c, s, SS_K_BIN);
        auto* offsets = static_cast<uint32_t*>(L.offsets.ensure((N + 1) * 4));
        auto* rbox = static_cast<uint2*>(L.rbox.ensure(std::max<uint64_t>(N, 1) * sizeof(uint2)));
        auto* rcnt = static_cast<uint32_t*>(L.rcnt.ensure((N + 1) * 4));
        own_launch(c, launch_gather_boxes(boxes, k32s, order, N, rbox, rcnt, s), SS_K_BIN);
        size_t tb = 0;
        SS_CUDA(launch_instance_offsets(rcnt, N, offsets, nullptr, &tb, s));
        void* tmp = L.cub_tmp.ensure(tb);
        tb = L.cub_tmp.bytes;
        SS_CUDA(launch_instance_offsets(rcnt, N, offsets, tmp, &tb, s));
        c->launches_cub += 1;
        c->prof.launches[SS_K_BIN] += 1;
        own_launch(c,
                   launch_emit_instances(rbox, order, N, offsets, g.tiles_x, L.list_cap, L.tkeys.p, g.k16,
                                         L.tvals.as<uint32_t>(), info, s),
                   SS_K_BIN, 2);
    }
    {
        // stable sort by tile: slices come out in depth order
        Scope sc(c, s, SS_K_SORT);
        const uint32_t tbits = bits_for(g.tiles - 1);
        size_t tb = 0;
        const int cap = (int)L.list_cap;
        auto* vin = L.tvals.as<uint32_t>();
        if (g.k16) {
            auto* kin = L.tkeys.as<uint16_t>();
            auto* kout = L.tkeys_sorted.as<uint16_t>();
            SS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, list, cap, 0, (int)tbits, s));
            void* tmp = L.cub_tmp.ensure(tb);
            tb = L.cub_tmp.bytes;
            SS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, list, cap, 0, (int)tbits, s));
        } else {
            auto* kin = L.tkeys.as<uint32_t>();
            auto* kout = L.tkeys_sorted.as<uint32_t>();
            SS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, list, cap, 0, (int)tbits, s));
            void* tmp = L.cub_tmp.ensure(tb);
            tb = L.cub_tmp.bytes;
            SS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, list, cap, 0, (int)tbits, s));
        }
        c->launches_cub += 1;
        c->prof.launches[SS_K_SORT] += 1;
    }
    {
        Scope sc(c, s, SS_K_BIN);
        SS_CUDA(cudaMemsetAsync(tstart, 0, (g.tiles + 1ull) * 4, s));
        SS_CUDA(cudaMemsetAsync(tend, 0, (g.tiles + 1ull) * 4, s));
        own_launch(c,
                   launch_tile_ranges(L.tkeys_sorted.p, g.k16, L.offsets.as<uint32_t>(), N, L.list_cap, tstart, tend,
                                      info, s),
                   SS_K_BIN);
    }
    return g;
}

RasterParams raster_params(ss_ctx* c, Lane& L, const ss_camera& cam, const Geometry& g) {
    RasterParams p;
    std::memset(&p, 0, sizeof(p));
    p.rec = L.rec.as<SplatRec>();
    p.boxes = L.boxes.as<uint2>();
    p.tile_list = L.list.as<uint32_t>();
    p.tile_start = L.tile_start.as<uint32_t>();
    p.tile_end = L.tile_end.as<uint32_t>();
    p.width = cam.width;
    p.height = cam.height;
    p.tiles_x = g.tiles_x;
    p.info = L.info.as<ViewInfo>();
    p.algo = (uint32_t)c->raster_algo;
    if (!L.raster_work.p) {
        L.raster_work.ensure(16);
        SS_CUDA(cudaMemset(L.raster_work.p, 0, 16));
    }
    p.work = L.raster_work.as<uint32_t>();
    return p;
}

// words per pixel of a view's mask bitsets: 1, 2 or 4 (one compositor pass),
// or whole 128-mask windows of 4 words for views with more than 128 masks
uint32_t mask_words_for(uint32_t m) {
    if (m <= 128) return m <= 32 ? 1 : (m <= 64 ? 2 : 4);
    return (m + 127) / 128 * 4;
}

// Upload one view's RLE masks + CLIP and build the raster-resolution bitsets.
void build_mask_bits(ss_ctx* c, Lane& L, cudaStream_t s, const ss_camera& cam, const ss_view_masks* vm,
                     uint32_t words, uint32_t image_id) {
    const uint32_t M = vm->n_masks;
    const uint64_t P = (uint64_t)cam.width * cam.height;
    auto* pb = static_cast<uint32_t*>(L.pix_bits.ensure(P * words * 4));
    Scope sc(c, s, SS_K_MASKS);
    SS_CUDA(cudaMemsetAsync(pb, 0, P * words * 4, s));
    if (M == 0) return;
    const uint64_t mw = vm->mask_width, mh = vm->mask_height;
    if (mw == 0 || mh == 0) throw Error(SS_ERR_CONTRACT, "resample_mask: zero mask resolution");
    const uint32_t* d_runs;
    const uint64_t* d_off;
    uint64_t nr;
    if (vm->flags & SS_MASKS_ON_DEVICE) {
        // device-resident encodings: absolute offsets, validated by the caller
        d_runs = vm->runs;
        d_off = vm->run_offsets;
        nr = 0;
    } else {
        // validate run streams against the mask area (providers.hpp:97-107)
        nr = vm->run_offsets[M] - vm->run_offsets[0];
        for (uint32_t m = 0; m < M; ++m) {
            uint64_t tot = 0;
            for (uint64_t r = vm->run_offsets[m]; r < vm->run_offsets[m + 1]; ++r) tot += vm->runs[r];
            if (tot != mw * mh)
                throw Error(SS_ERR_FORMAT, "image " + std::to_string(image_id) +
                                               ": mask RLE length mismatch: runs cover " + std::to_string(tot) +
                                               " of " + std::to_string(mw * mh) + " pixels");
        }
        auto* hr = static_cast<uint32_t*>(L.runs.ensure(std::max<uint64_t>(nr, 1) * 4));
        auto* ho = static_cast<uint64_t*>(L.run_offsets.ensure((M + 1) * 8ull));
        std::vector<uint64_t> rel(M + 1);
        for (uint32_t m = 0; m <= M; ++m) rel[m] = vm->run_offsets[m] - vm->run_offsets[0];
        Scope h(c, s, SS_K_H2D);
        SS_CUDA(cudaMemcpyAsync(hr, vm->runs + vm->run_offsets[0], nr * 4, cudaMemcpyHostToDevice, s));
        // pageable source: staged synchronously, so `rel` may go out of scope after the call
        SS_CUDA(cudaMemcpyAsync(ho, rel.data(), (M + 1) * 8ull, cudaMemcpyHostToDevice, s));
        c->prof.bytes[SS_K_H2D] += nr * 4.0 + (M + 1) * 8.0;
        d_runs = hr;
        d_off = ho;
    }
    const bool same = mw == cam.width && mh == cam.height;
    uint32_t* target = pb;
    if (!same) {
        target = static_cast<uint32_t*>(L.mask_bits.ensure(mw * mh * words * 4));
        SS_CUDA(cudaMemsetAsync(target, 0, mw * mh * words * 4, s));
    }
    // spans: at most one per run; the run count is bounded by the RLE stream length
    const uint64_t max_spans = ((vm->flags & SS_MASKS_ON_DEVICE) ? vm->n_runs : nr) / 2 + M;
    auto* spans = static_cast<uint4*>(L.spans.ensure(std::max<uint64_t>(max_spans, 1) * 16 + 16));
    auto* n_spans = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(L.spans.p) + L.spans.bytes - 16);
    own_launch(c, launch_rle_to_bits(d_runs, d_off, M, words, target, spans, n_spans, s), SS_K_MASKS, 2);
    if (!same)
        own_launch(c, launch_resample_bits(target, (uint32_t)mw, (uint32_t)mh, pb, cam.width, cam.height, words, s),
                   SS_K_MASKS);
    c->prof.bytes[SS_K_MASKS] += nr * 4.0 + (double)P * ((M + 7) / 8);
}

// Issues the contraction of the views gathered in c->group on the stream of
// the last one: after every member's compositor and after the previous
// group's contraction (the shared sums are updated in view order).
constexpr uint32_t kAutoGroup = 3; // views per group under SS_OPT_CONTRACT_GROUP = 0

void flush_group(ss_ctx* c) {
    if (c->group.empty()) return;
    // in order: groups contract one after another on their own stream; with a
    // single lane everything stays on that lane (serialised attribution pass)
    cudaStream_t st = c->n_lanes > 1 ? c->cstream : c->group.back().lane->stream;
    for (auto& g : c->group) SS_CUDA(cudaStreamWaitEvent(st, g.lane->raster_done, 0));
    if (c->n_lanes == 1 && c->group_done_valid) SS_CUDA(cudaStreamWaitEvent(st, c->group_done, 0));
    ContractParams q;
    std::memset(&q, 0, sizeof(q));
    q.n_members = (uint32_t)c->group.size();
    for (uint32_t i = 0; i < q.n_members; ++i) {
        const GroupMember& g = c->group[i];
        q.m[i].touched_list = g.set->touched_list.as<uint32_t>();
        q.m[i].touched_count = g.set->tcount.as<unsigned long long>();
        q.m[i].touched = g.set->touched.as<uint32_t>();
        q.m[i].gen = g.set->gen;
        q.m[i].acc = g.set->acc.p;
        q.m[i].fix = g.set->acc_fix ? 1u : 0u;
        q.m[i].n_masks = g.n_masks;
        q.m[i].clip = g.clip;
        c->prof.bytes[SS_K_CONTRACT] += (double)g.n_masks * c->dim * 4;
    }
    q.dim = c->dim;
    q.sums = c->sums;
    q.totals = c->totals;
    q.count_pairs = 1;
    q.cum = c->counters.as<unsigned long long>();
    if (q.n_members > 1) {
        q.union_list = static_cast<uint2*>(c->union_list.ensure(std::max<uint64_t>(c->n * q.n_members, 1) * 8));
        q.union_count = static_cast<unsigned int*>(c->union_count.ensure(16));
        if (c->contract_tc) q.tc_scratch = c->tc_scratch.ensure(contract_tc_scratch_bytes());
        q.use_tc = c->contract_tc;
    }
    {
        Scope sc(c, st, SS_K_CONTRACT);
        own_launch(c, launch_contract(q, c->n * q.n_members, st), SS_K_CONTRACT);
    }
    SS_CUDA(cudaEventRecord(c->group_done, st));
    c->group_done_valid = true;
    for (auto& g : c->group) {
        SS_CUDA(cudaEventRecord(g.set->free_ev, st));
        g.set->pending = true;
        g.set->in_group = false;
    }
    c->group.clear();
}

bool encode_one(ss_ctx* c, Lane& L, const ss_camera& cam, const ss_view_masks* vm, int mode,
                ViewInfo* vstat_slot, bool force_global) {
    check_camera(&cam);
    const uint32_t M = vm ? vm->n_masks : 0;
    const uint32_t words = mask_words_for(M);
    cudaStream_t s = L.stream;
    ContractSet* S = nullptr;
    if (M) {
        S = &L.sets[L.set_next];
        L.set_next = (L.set_next + 1u) % SS_LANE_SETS;
        if (S->in_group) flush_group(c); // the set is needed again before its group closed
        if (S->pending) {                // its last contraction must be done before we overwrite it
            SS_CUDA(cudaStreamWaitEvent(s, S->free_ev, 0));
            S->pending = false;
        }
        if (S->dirty) { // a view of an abandoned group left its per-(Gaussian, mask) scalars behind
            if (S->acc.p) SS_CUDA(cudaMemsetAsync(S->acc.p, 0, S->acc.bytes, s));
            S->dirty = false;
        }
        build_mask_bits(c, L, s, cam, vm, words, cam.image_id);
    }
    const float* d_clip = vm && (vm->flags & SS_MASKS_ON_DEVICE) ? vm->clip : nullptr;
    if (M && !d_clip) {
        auto* dc = static_cast<float*>(S->clip.ensure(std::max<uint64_t>((uint64_t)M * c->dim, 1) * 4));
        d_clip = dc;
        Scope h(c, s, SS_K_H2D);
        SS_CUDA(cudaMemcpyAsync(dc, vm->clip, (size_t)M * c->dim * 4, cudaMemcpyHostToDevice, s));
        c->prof.bytes[SS_K_H2D] += (double)M * c->dim * 4;
    }
    // prefix-sorted tile lists for the fused pass: one per-step compositor pass
    // (<= 128 masks) in alpha-composited mode (falloff pixels never terminate;
    // the staged-evaluation compositor has no resume path)
    const bool staged = c->raster_algo == 0 && !c->deterministic;
    const uint32_t prefix = M && c->sort_prefix && words <= (uint32_t)kMaxMaskWords && mode == SS_ALPHA_COMPOSITED &&
                                    !staged
                                ? c->sort_prefix
                                : 0u;
    const Geometry g = run_geometry(c, L, s, cam, force_global, false, prefix);
    if (M) {
        // per-(Gaussian, mask) scalars: grow-only and kept zero by consume-and-clear
        // (zero is all-zero bytes in both representations, so a set switches
        // representation by size alone)
        const uint64_t need = c->n * (uint64_t)M;
        const uint64_t esz = c->deterministic ? sizeof(acc_t) : sizeof(float);
        if (need * esz > S->acc.bytes) {
            S->acc.release();
            S->acc.ensure(need * esz);
            SS_CUDA(cudaMemsetAsync(S->acc.p, 0, S->acc.bytes, s));
        }
        S->acc_fix = c->deterministic;
        S->acc_elems = S->acc.bytes / esz;
        if (S->touched.bytes < c->n * 4 || S->gen == 0xffffffffu) {
            S->touched.release();
            S->touched.ensure(c->n * 4);
            SS_CUDA(cudaMemsetAsync(S->touched.p, 0, S->touched.bytes, s));
            S->gen = 0;
        }
        S->gen += 1;
        auto* tlist = static_cast<uint32_t*>(S->touched_list.ensure(c->n * 4));
        auto* tcount = static_cast<unsigned long long*>(S->tcount.ensure(16));
        SS_CUDA(cudaMemsetAsync(tcount, 0, 8, s));
        {
            Scope sc(c, s, SS_K_RASTER);
            RasterParams p = raster_params(c, L, cam, g);
            p.pix_bits = L.pix_bits.as<uint32_t>();
            p.n_masks = M;
            p.bits_stride = words;
            p.acc = S->acc.p;
            p.acc_fix = S->acc_fix ? 1u : 0u;
            p.touched = S->touched.as<uint32_t>();
            p.touched_list = tlist;
            p.touched_count = tcount;
            p.gen = S->gen;
            if (g.prefix) {
                p.tile_full = L.ts_params.fill;
                p.rs_T = L.rs_T.as<double>();
                p.rs_state = L.rs_state.as<uint2>();
                p.rs_items = L.rs_items.as<uint32_t>();
                p.rs_count = L.rs_count.as<uint32_t>();
                p.rs_tiles = L.rs_tiles.as<uint32_t>();
                p.rs_need = L.rs_need.as<uint32_t>();
            }
            // one pass per 128-mask window (a single pass for M <= 128)
            for (uint32_t w0 = 0; w0 < words; w0 += kMaxMaskWords) {
                p.mask_words = std::min<uint32_t>(words - w0, kMaxMaskWords);
                p.mask_base = 32u * w0;
                own_launch(c, launch_raster_fused(p, mode, g.tiles, s), SS_K_RASTER);
            }
        }
        if (g.prefix) {
            // the tiles whose prefix some block exhausted: sorted in full (bin
            // time), then those blocks continue where they stopped (raster
            // time; the raster class counts the main pass as its launch, so
            // per-launch figures stay those of the compositor pass)
            {
                Scope sc(c, s, SS_K_BIN);
                own_launch(c, launch_tile_sort_fixup(L.ts_params, s), SS_K_BIN, 0);
                c->launches_own += 1;
            }
            Scope sc(c, s, SS_K_RASTER);
            RasterParams p = raster_params(c, L, cam, g);
            p.pix_bits = L.pix_bits.as<uint32_t>();
            p.n_masks = M;
            p.bits_stride = words;
            p.mask_words = words;
            p.mask_base = 0;
            p.acc = S->acc.p;
            p.acc_fix = S->acc_fix ? 1u : 0u;
            p.touched = S->touched.as<uint32_t>();
            p.gen = S->gen;
            p.rs_T = L.rs_T.as<double>();
            p.rs_state = L.rs_state.as<uint2>();
            p.rs_items = L.rs_items.as<uint32_t>();
            p.rs_count = L.rs_count.as<uint32_t>();
            own_launch(c, launch_raster_resume(p, mode, s), SS_K_RASTER, 0);
            c->launches_own += 1;
        }
        {
            // the view's touched Gaussians, compacted from the compositor's stamps
            Scope sc(c, s, SS_K_CONTRACT);
            own_launch(c, launch_touched_compact(S->touched.as<uint32_t>(), c->n, S->gen, tlist, tcount, s),
                       SS_K_CONTRACT);
            c->prof.bytes[SS_K_CONTRACT] += 4.0 * (double)c->n;
        }
        SS_CUDA(cudaEventRecord(L.raster_done, s));
        // auto grouping: only views the shared-memory group kernel takes
        // (D = 512, <= 64 masks) are contracted three at a time
        if (c->group_max == 0 && !(c->dim == 512 && M <= 64)) flush_group(c);
        S->in_group = true;
        c->group.push_back(GroupMember{&L, S, M, d_clip});
    }
    SS_CUDA(cudaMemcpyAsync(vstat_slot, L.info.p, sizeof(ViewInfo), cudaMemcpyDeviceToDevice, s));
    const uint32_t cap = c->group_max ? std::min<uint32_t>(c->group_max, kMaxGroup)
                                      : (c->dim == 512 && M <= 64 ? kAutoGroup : 1u);
    if (c->group.size() >= cap) flush_group(c);
    return g.tile_sort;
}

// Encodes a batch of views with no per-view host synchronisation; the host
// looks at the per-view status once at the end: views whose tile lists
// overflowed the list buffer contributed nothing and are re-run with a larger
// buffer; singular covariances surface as the reference's per-image error.
void encode_batch(ss_ctx* c, uint32_t nviews, const ss_camera* cams, const ss_view_masks* masks, int mode) {
    if (!c->sums) throw Error(SS_ERR_CONTRACT, "ss_encode_view before ss_encode_begin");
    if (nviews == 0 || c->n == 0) return;
    auto* vstat = static_cast<ViewInfo*>(c->vstat.ensure((uint64_t)nviews * sizeof(ViewInfo)));
    std::vector<ViewInfo> hstat(nviews);
    std::vector<uint32_t> todo(nviews);
    for (uint32_t v = 0; v < nviews; ++v) todo[v] = v;
    std::vector<uint8_t> force_global(nviews, 0), tile_sorted(nviews, 0);
    uint64_t max_inst = 0; // largest tile-instance count of the views that fit
    uint64_t ts_slots = 0; // list entries the tile-sort binning needs
    for (int attempt = 0; attempt < 4 && !todo.empty(); ++attempt) {
        // lanes start after everything already queued on the user stream
        SS_CUDA(cudaEventRecord(c->ev_user, c->stream));
        for (auto& L : c->lanes) SS_CUDA(cudaStreamWaitEvent(L.stream, c->ev_user, 0));
        SS_CUDA(cudaStreamWaitEvent(c->cstream, c->ev_user, 0));
        {
            struct Join {
                ss_ctx* c;
                ~Join() {
                    // the user stream resumes after all lanes drain (also on errors;
                    // a group left open by an error contributes nothing, and its
                    // members' scalars are zeroed before the sets are used again)
                    for (auto& g : c->group) {
                        g.set->in_group = false;
                        g.set->dirty = true;
                    }
                    c->group.clear();
                    for (auto& L : c->lanes) {
                        cudaEventRecord(L.done, L.stream);
                        cudaStreamWaitEvent(c->stream, L.done, 0);
                    }
                    cudaEventRecord(c->group_done, c->cstream);
                    cudaStreamWaitEvent(c->stream, c->group_done, 0);
                }
            } join{c};
            for (uint32_t v : todo) {
                // view v runs on lane v mod n; contractions run per group of
                // consecutive views, groups in view order
                const uint32_t li = c->next_lane % c->n_lanes;
                Lane& L = c->lanes[li];
                c->next_lane = (li + 1) % c->n_lanes;
                tile_sorted[v] = encode_one(c, L, cams[v], masks ? &masks[v] : nullptr, mode, vstat + v,
                                            force_global[v] != 0);
                if (tile_sorted[v]) {
                    const uint64_t tiles = (uint64_t)((cams[v].width + kTile - 1) / kTile) *
                                           ((cams[v].height + kTile - 1) / kTile);
                    ts_slots = std::max<uint64_t>(ts_slots, tiles * L.ts_cap);
                }
            }
            flush_group(c);
        }
        SS_CUDA(cudaMemcpyAsync(hstat.data(), vstat, (uint64_t)nviews * sizeof(ViewInfo), cudaMemcpyDeviceToHost,
                                c->stream));
        SS_CUDA(cudaStreamSynchronize(c->stream));
        std::vector<uint32_t> again;
        uint64_t need = 0;
        for (uint32_t v : todo) {
            const ViewInfo& st = hstat[v];
            if (st.err_count)
                throw Error(SS_ERR_DATA, "image " + std::to_string(cams[v].image_id) +
                                             ": singular screen covariance for gaussian " +
                                             std::to_string(first_singular_gid(c, cams[v])));
            if (st.overflow) {
                again.push_back(v);
                if (st.bin_fallback == 1 && st.max_fill <= kTileSortMax) {
                    // a tile outgrew its slots: every lane's capacity grows to the largest tile seen
                    const uint32_t cap = tile_sort_capacity(st.max_fill);
                    for (auto& L : c->lanes) L.ts_cap = std::max(L.ts_cap, cap);
                } else if (st.bin_fallback) {
                    force_global[v] = 1; // beyond the in-CTA tile sort: the global depth sort path
                } else {
                    need = std::max<uint64_t>(need, st.n_instances);
                }
                continue;
            }
            max_inst = std::max<uint64_t>(max_inst, st.n_instances);
            const double P = (double)cams[v].width * cams[v].height;
            const uint32_t M = masks ? masks[v].n_masks : 0;
            c->cnt_vis += st.n_surv;
            c->cnt_inst += st.n_instances;
            c->cnt_views += 1;
            c->prof.bytes[SS_K_PROJECT] += 76.0 * (double)st.n_surv;
            if (tile_sorted[v]) {
                // boxes by gid, survivors' depth keys; (key, gid) slots written and read; the list written
                c->prof.bytes[SS_K_BIN] += 8.0 * (double)c->n + 8.0 * (double)st.n_surv + 20.0 * (double)st.n_instances;
            } else {
                c->prof.bytes[SS_K_BIN] += 8.0 * (double)st.n_surv + 4.0 * (double)st.n_instances;
                c->prof.bytes[SS_K_SORT] += 16.0 * (double)st.n_instances;
            }
            if (M) c->prof.bytes[SS_K_RASTER] += 64.0 * (double)st.n_instances + P * ((M + 7) / 8);
        }
        for (auto& L : c->lanes)
            if (need > L.list_cap) {
                L.list_cap = need + need / 16;
            }
        todo.swap(again);
    }
    if (!todo.empty()) throw Error(SS_ERR_CUDA, "tile-list buffer kept overflowing");
    // the tile sort runs over the whole list capacity: track the views' actual
    // sizes (+1/16; a view that overflows is re-run with a larger capacity)
    if (max_inst) {
        const uint64_t want = std::max<uint64_t>((max_inst + max_inst / 16 + 1023) / 1024 * 1024, ts_slots);
        for (auto& L : c->lanes)
            if (L.list_cap > want + want / 8) L.list_cap = want;
    }
}

void profile_drain(ss_ctx* c) {
    if (c->prof.pending.empty()) return;
    SS_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& L : c->lanes) SS_CUDA(cudaStreamSynchronize(L.stream));
    SS_CUDA(cudaStreamSynchronize(c->cstream));
    if (c->comm_stream) SS_CUDA(cudaStreamSynchronize(c->comm_stream));
    for (auto& pe : c->prof.pending) {
        float ms = 0;
        SS_CUDA(cudaEventElapsedTime(&ms, pe.second.first, pe.second.second));
        c->prof.ms[pe.first] += ms;
        c->prof.pool.push_back(pe.second.first);
        c->prof.pool.push_back(pe.second.second);
    }
    c->prof.pending.clear();
}

// ---------------------------------------------------------------- NCCL
// Resolved at run time so the library never pins a second NCCL into a process
// that already has one (torch's): the copy already loaded wins, then
// $SS_NCCL_LIB, then libnccl.so.2 on the loader path.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = getenv("SS_NCCL_LIB");
            if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
            return a;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(sym("ncclReduceScatter"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        if (!a.GetUniqueId || !a.CommInitRank || !a.CommInitAll || !a.CommDestroy || !a.ReduceScatter || !a.AllReduce ||
            !a.GroupStart || !a.GroupEnd || !a.GetErrorString)
            a.error = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    if (!api.error.empty()) throw Error(SS_ERR_CUDA, api.error);
    return api;
}

#define SS_NCCL(expr)                                                                                      \
    do {                                                                                                   \
        const NcclApi& _a = nccl_api();                                                                    \
        ncclResult_t _r = (_a.expr);                                                                       \
        if (_r != ncclSuccess)                                                                             \
            throw Error(SS_ERR_CUDA, std::string("nccl") + #expr + ": " + _a.GetErrorString(_r));          \
    } while (0)

// Block-cyclic combine layout (include/semsplat_b200.h, multi-GPU section).
struct CombineLayout {
    uint64_t block = 0, rounds = 0, rows_alloc = 0;
};
CombineLayout combine_layout(uint64_t n, int nranks, uint64_t combine_rows) {
    CombineLayout L;
    const uint64_t W = (uint64_t)std::max(nranks, 1);
    const uint64_t shard = std::max<uint64_t>((n + W - 1) / W, 1);
    L.block = combine_rows ? std::min<uint64_t>(combine_rows, shard) : shard;
    L.rounds = (n + W * L.block - 1) / (W * L.block);
    if (L.rounds == 0) L.rounds = 1;
    L.rows_alloc = L.rounds * W * L.block;
    return L;
}

void comm_setup(ss_ctx* c) {
    if (!c->comm_stream) SS_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    cudaEvent_t* evs[] = {&c->ev_acc, &c->ev_rs[0], &c->ev_rs[1], &c->ev_norm[0], &c->ev_norm[1]};
    for (auto* e : evs)
        if (!*e) SS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void comm_release(ss_ctx* c) {
    if (c->comm && c->own_comm) nccl_api().CommDestroy(c->comm);
    c->comm = nullptr;
    c->own_comm = false;
    c->nranks = 1;
    c->rank = 0;
}

} // namespace
} // namespace ss

using namespace ss;

namespace {
// Device -> pageable host copy of `bytes` (the reference's host containers are
// plain std::vectors): chunks of kStageBytes DMA into two pinned staging
// buffers while host threads move the previous chunk out, so the readout runs
// at pinned-DMA speed instead of the driver's pageable path (~4x slower).
constexpr size_t kStageBytes = 64u << 20;

void copy_d2h_pageable(ss_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, dst) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError(); // unregistered pointers may set an error on older drivers
    if (pinned || bytes < (4u << 20)) { // pinned destination, or small: the plain copy
        SS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        return;
    }
    if (!c->h_stage) {
        SS_CUDA(cudaMallocHost(&c->h_stage, 2 * kStageBytes));
        for (auto& e : c->stage_ev) SS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
    auto host_copy = [&](char* d, const char* sp, size_t n) {
        const size_t per = (n + hw - 1) / hw;
        std::vector<std::thread> th;
        for (unsigned t = 1; t < hw && t * per < n; ++t)
            th.emplace_back([=] { std::memcpy(d + t * per, sp + t * per, std::min(per, n - t * per)); });
        std::memcpy(d, sp, std::min(per, n));
        for (auto& x : th) x.join();
    };
    const size_t chunks = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t k) {
        const size_t off = k * kStageBytes, n = std::min(kStageBytes, bytes - off);
        SS_CUDA(cudaMemcpyAsync(c->h_stage + (k & 1) * kStageBytes, static_cast<const char*>(src) + off, n,
                                cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaEventRecord(c->stage_ev[k & 1], s));
    };
    issue(0);
    for (size_t k = 0; k < chunks; ++k) {
        if (k + 1 < chunks) issue(k + 1); // its buffer was drained in iteration k - 1
        SS_CUDA(cudaEventSynchronize(c->stage_ev[k & 1]));
        const size_t off = k * kStageBytes, n = std::min(kStageBytes, bytes - off);
        host_copy(static_cast<char*>(dst) + off, c->h_stage + (k & 1) * kStageBytes, n);
    }
}
} // namespace

extern "C" {

const char* ss_last_error(void) { return ss::g_err.c_str(); }
int ss_last_error_kind(void) { return ss::g_kind; }

int ss_create(int device, ss_ctx** out) {
    return guarded([&] {
        if (!out) throw Error(SS_ERR_CONTRACT, "out is null");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0)
            throw Error(SS_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
        if (device < 0 || device >= ndev) throw Error(SS_ERR_CONTRACT, "device index out of range");
        cudaDeviceProp prop;
        SS_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw Error(SS_ERR_CUDA, std::string("libsemsplat_b200 is built for sm_100a; device is ") + prop.name);
        auto* c = new ss_ctx();
        c->device = device;
        SS_CUDA(cudaSetDevice(device));
        SS_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        SS_CUDA(cudaMallocHost(&c->h_init, sizeof(ViewInfo)));
        SS_CUDA(cudaMallocHost(&c->h_u32, 64));
        SS_CUDA(cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming));
        SS_CUDA(cudaEventCreateWithFlags(&c->group_done, cudaEventDisableTiming));
        SS_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (auto& L : c->lanes) {
            SS_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
            SS_CUDA(cudaEventCreateWithFlags(&L.contract_done, cudaEventDisableTiming));
            SS_CUDA(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
            SS_CUDA(cudaEventCreateWithFlags(&L.raster_done, cudaEventDisableTiming));
            for (auto& cs : L.sets) SS_CUDA(cudaEventCreateWithFlags(&cs.free_ev, cudaEventDisableTiming));
            SS_CUDA(cudaMallocHost(&L.h_info, sizeof(ViewInfo)));
            SS_CUDA(cudaMallocHost(&L.h_u32, 64));
            L.info.ensure(sizeof(ViewInfo));
        }
        std::memset(c->h_init, 0, sizeof(ViewInfo));
        c->h_init->min_key = ~0ull;
        c->h_init->err_gid = ~0u;
        c->info.ensure(sizeof(ViewInfo));
        c->counters.ensure(32);
        SS_CUDA(cudaMemset(c->counters.p, 0, c->counters.bytes));
        *out = c;
    });
}

void ss_destroy(ss_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& L : c->lanes) cudaStreamSynchronize(L.stream);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    ss::DevBuf* bufs[] = {&c->mean_op, &c->scale, &c->quat, &c->cov3, &c->cub_tmp, &c->num_sel, &c->info, &c->vstat, &c->union_list, &c->union_count, &c->tc_scratch, &c->pix_count,
                          &c->pix_offset, &c->entries, &c->per_pixel_total, &c->alpha, &c->color, &c->image, &c->counters, &c->sums_buf,
                          &c->totals_buf, &c->store_rows, &c->store_ids, &c->part_buf, &c->part_means, &c->qbuf, &c->qnorm, &c->scores,
                          &c->topk_ids, &c->topk_sims, &c->sel_flags, &c->thr_keys, &c->thr_keys_sorted, &c->thr_ids,
                          &c->thr_ids_sorted, &c->zero_flag, &c->store_half, &c->qhalf, &c->tc_scores, &c->tc_thr,
                          &c->cand, &c->cand_count, &c->cand_sim};
    for (auto* b : bufs) b->release();
    for (auto e : c->prof.pool) cudaEventDestroy(e);
    for (auto& pe : c->prof.pending) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    for (auto& L : c->lanes) L.release_all();
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    try {
        comm_release(c);
    } catch (...) {
    }
    for (int i = 0; i < 2; ++i) {
        c->rs_sum[i].release();
        c->rs_tot[i].release();
        if (c->ev_rs[i]) cudaEventDestroy(c->ev_rs[i]);
        if (c->ev_norm[i]) cudaEventDestroy(c->ev_norm[i]);
    }
    c->rs_stage.release();
    for (ss::DevBuf* b : {&c->sp_flags, &c->sp_pos, &c->sp_tmp, &c->sp_send, &c->sp_bounds}) b->release();
    if (c->ev_acc) cudaEventDestroy(c->ev_acc);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->ev_user) cudaEventDestroy(c->ev_user);
    if (c->group_done) cudaEventDestroy(c->group_done);
    if (c->cstream) {
        cudaStreamSynchronize(c->cstream);
        cudaStreamDestroy(c->cstream);
    }
    if (c->h_init) cudaFreeHost(c->h_init);
    if (c->h_u32) cudaFreeHost(c->h_u32);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    for (cudaEvent_t e : c->stage_ev)
        if (e) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

int ss_set_stream(ss_ctx* c, uintptr_t stream) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        c->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : c->own_stream;
    });
}

int ss_set_option(ss_ctx* c, int option, int64_t value) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (option == SS_OPT_LANES) {
            if (value < 1 || value > (int64_t)ss_ctx::kMaxLanes)
                throw Error(SS_ERR_CONTRACT, "SS_OPT_LANES must be between 1 and 6");
            c->n_lanes = (uint32_t)value;
        } else if (option == SS_OPT_CONTRACT_GROUP) {
            if (value < 0 || value > (int64_t)kMaxGroup)
                throw Error(SS_ERR_CONTRACT, "SS_OPT_CONTRACT_GROUP must be between 0 (auto) and 4");
            c->group_max = (uint32_t)value;
        } else if (option == SS_OPT_QUERY_PATH) {
            if (value < 0 || value > 2) throw Error(SS_ERR_CONTRACT, "SS_OPT_QUERY_PATH must be 0, 1 or 2");
            c->query_path = (int)value;
        } else if (option == SS_OPT_COMBINE_ROWS) {
            if (value < 0) throw Error(SS_ERR_CONTRACT, "SS_OPT_COMBINE_ROWS must be >= 0");
            c->combine_rows = (uint64_t)value;
        } else if (option == SS_OPT_RASTER) {
            if (value < 0 || value > 2) throw Error(SS_ERR_CONTRACT, "SS_OPT_RASTER must be 0, 1 or 2");
            c->raster_algo = (int)value;
        } else if (option == SS_OPT_COMBINE_SPARSE) {
            if (value < 0 || value > 2) throw Error(SS_ERR_CONTRACT, "SS_OPT_COMBINE_SPARSE must be 0, 1 or 2");
            c->combine_sparse = (int)value;
        } else if (option == SS_OPT_SORT_PREFIX) {
            if (value < 0 || value > 65536) throw Error(SS_ERR_CONTRACT, "SS_OPT_SORT_PREFIX must be 0..65536");
            c->sort_prefix = (uint32_t)value;
        } else if (option == SS_OPT_DETERMINISTIC) {
            if (value < 0 || value > 1) throw Error(SS_ERR_CONTRACT, "SS_OPT_DETERMINISTIC must be 0 or 1");
            c->deterministic = value != 0;
        } else if (option == SS_OPT_CONTRACT_TC) {
            if (value < 0 || value > 1) throw Error(SS_ERR_CONTRACT, "SS_OPT_CONTRACT_TC must be 0 or 1");
            c->contract_tc = (int)value;
        } else if (option == SS_OPT_BIN_PATH) {
            if (value < 0 || value > 3) throw Error(SS_ERR_CONTRACT, "SS_OPT_BIN_PATH must be 0, 1, 2 or 3");
            c->bin_path = (int)value;
        } else {
            throw Error(SS_ERR_CONTRACT, "unknown option");
        }
    });
}

int ss_synchronize(ss_ctx* c) {
    return guarded([&] {
        set_device(c);
        SS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ss_scene_set(ss_ctx* c, const float* mean, const float* scale, const float* quat_xyzw, const float* opacity,
                 uint64_t n) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (n >= (1ull << 32)) throw Error(SS_ERR_CONTRACT, "gaussian ids are u32 (scene.hpp:23)");
        set_device(c);
        std::vector<float> a(std::max<uint64_t>(n, 1) * 4), b(std::max<uint64_t>(n, 1) * 4),
            q(std::max<uint64_t>(n, 1) * 4);
        for (uint64_t k = 0; k < n; ++k) {
            a[4 * k] = mean[3 * k];
            a[4 * k + 1] = mean[3 * k + 1];
            a[4 * k + 2] = mean[3 * k + 2];
            a[4 * k + 3] = opacity[k];
            b[4 * k] = scale[3 * k];
            b[4 * k + 1] = scale[3 * k + 1];
            b[4 * k + 2] = scale[3 * k + 2];
            b[4 * k + 3] = 0.0f;
            for (int i = 0; i < 4; ++i) q[4 * k + i] = quat_xyzw[4 * k + i];
        }
        c->n = n;
        c->color_ok = false;
        const size_t bytes = std::max<uint64_t>(n, 1) * 16;
        SS_CUDA(cudaMemcpyAsync(c->mean_op.ensure(bytes), a.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
        SS_CUDA(cudaMemcpyAsync(c->scale.ensure(bytes), b.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
        SS_CUDA(cudaMemcpyAsync(c->quat.ensure(bytes), q.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
        auto* cov = static_cast<double*>(c->cov3.ensure(std::max<uint64_t>(n, 1) * 72));
        own_launch(c, launch_cov3d(c->scale.as<float4>(), c->quat.as<float4>(), n, cov, c->stream), SS_K_PROJECT);
        SS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ss_project(ss_ctx* c, const ss_camera* cam, ss_projected* out) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        check_camera(cam);
        set_device(c);
        const uint64_t N = c->n;
        if (N == 0) return;
        cudaStream_t s = c->stream;
        auto* dbg = static_cast<ss_projected*>(c->scores.ensure(N * sizeof(ss_projected)));
        ss::Lane& L = c->lanes[0];
        reset_info(c, L, s);
        ProjectParams p;
        p.mean_op = c->mean_op.as<float4>();
        p.scale = c->scale.as<float4>();
        p.quat = c->quat.as<float4>();
        p.cov3 = c->cov3.as<double>();
        p.n = N;
        p.cam = *cam;
        p.rec = static_cast<SplatRec*>(L.rec.ensure(N * sizeof(SplatRec)));
        p.boxes = static_cast<uint2*>(L.boxes.ensure(N * sizeof(uint2)));
        p.keys = static_cast<unsigned long long*>(L.keys.ensure(N * 8));
        p.tile_count = nullptr;
        p.tiles_x = 0;
        p.info = L.info.as<ViewInfo>();
        p.dbg = dbg;
        own_launch(c, launch_project(p, s), SS_K_PROJECT);
        SS_CUDA(cudaMemcpyAsync(out, dbg, N * sizeof(ss_projected), cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
    });
}

namespace {
// rasterize_weights_only (rasterizer.hpp:268-271) or, with color, rasterize
// (rasterizer.hpp:261-264): tile lists, then the counting and capture passes
// of the compositor (the capture pass also forms the normalised pixel colors).
void capture_view(ss_ctx* c, const ss_camera* cam, int mode, bool color, uint64_t* n_entries, uint64_t* n_splats,
                  uint64_t* n_tile_instances) {
    check_camera(cam);
    set_device(c);
    cudaStream_t s = c->stream;
    const uint64_t P = (uint64_t)cam->width * cam->height;
    ss::Lane& L = c->lanes[0];
    Geometry g;
    bool force_global = false;
    for (int attempt = 0;; ++attempt) {
        g = run_geometry(c, L, s, *cam, force_global, true);
        SS_CUDA(cudaMemcpyAsync(L.h_info, L.info.p, sizeof(ViewInfo), cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        if (!L.h_info->overflow) break;
        if (attempt > 3) throw Error(SS_ERR_CUDA, "tile-list buffer kept overflowing");
        if (L.h_info->bin_fallback == 1 && L.h_info->max_fill <= kTileSortMax) {
            L.ts_cap = std::max(L.ts_cap, tile_sort_capacity(L.h_info->max_fill));
        } else if (L.h_info->bin_fallback) {
            force_global = true;
        } else {
            L.list_cap = L.h_info->n_instances + L.h_info->n_instances / 16;
        }
    }
    c->cap_tile_sort = g.tile_sort;
    if (L.h_info->err_count)
        throw Error(SS_ERR_NUMERIC, "singular screen covariance for gaussian " +
                                        std::to_string(first_singular_gid(c, *cam)));
    const uint64_t n_surv = L.h_info->n_surv, n_inst = L.h_info->n_instances;
    auto* cnt = static_cast<uint32_t*>(c->pix_count.ensure((P + 1) * 4));
    auto* off = static_cast<uint32_t*>(c->pix_offset.ensure((P + 1) * 4));
    auto* ppt = static_cast<float*>(c->per_pixel_total.ensure(P * 4));
    auto* alp = static_cast<float*>(c->alpha.ensure(P * 4));
    SS_CUDA(cudaMemsetAsync(cnt, 0, (P + 1) * 4, s));
    SS_CUDA(cudaMemsetAsync(ppt, 0, P * 4, s));
    SS_CUDA(cudaMemsetAsync(alp, 0, P * 4, s));
    RasterParams p = raster_params(c, L, *cam, g);
    if (n_surv) {
        p.pix_count = cnt;
        own_launch(c, launch_raster_count(p, mode, g.tiles, s), SS_K_RASTER);
    }
    size_t tb = 0;
    SS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(P + 1), s));
    void* tmp = c->cub_tmp.ensure(tb);
    tb = c->cub_tmp.bytes;
    SS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(P + 1), s));
    c->launches_cub += 1;
    SS_CUDA(cudaMemcpyAsync(c->h_u32, off + P, 4, cudaMemcpyDeviceToHost, s));
    SS_CUDA(cudaStreamSynchronize(s));
    const uint64_t E = c->h_u32[0];
    auto* ent = static_cast<ss_weight_entry*>(c->entries.ensure(std::max<uint64_t>(E, 1) * sizeof(ss_weight_entry)));
    if (color) {
        auto* img = static_cast<float*>(c->image.ensure(std::max<uint64_t>(P, 1) * 12));
        SS_CUDA(cudaMemsetAsync(img, 0, P * 12, s));
        p.color = c->color.as<float4>();
        p.image = img;
    }
    if (n_surv) {
        p.pix_offset = off;
        p.entries = ent;
        p.per_pixel_total = ppt;
        p.alpha = alp;
        own_launch(c, color ? launch_raster_render(p, mode, g.tiles, s) : launch_raster_capture(p, mode, g.tiles, s),
                   SS_K_RASTER);
    }
    SS_CUDA(cudaStreamSynchronize(s));
    c->cap_entries = E;
    c->cap_splats = n_surv;
    c->cap_instances = n_inst;
    c->cap_width = cam->width;
    c->cap_height = cam->height;
    c->cap_tiles = g.tiles;
    c->cap_image = color;
    if (n_entries) *n_entries = E;
    if (n_splats) *n_splats = n_surv;
    if (n_tile_instances) *n_tile_instances = n_inst;
}
} // namespace

int ss_raster_capture(ss_ctx* c, const ss_camera* cam, int mode, uint64_t* n_entries, uint64_t* n_splats,
                      uint64_t* n_tile_instances) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        capture_view(c, cam, mode, false, n_entries, n_splats, n_tile_instances);
    });
}

int ss_scene_set_color(ss_ctx* c, const float* rgb, uint64_t n) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (n != c->n) throw Error(SS_ERR_CONTRACT, "ss_scene_set_color: count differs from the scene");
        set_device(c);
        std::vector<float> a(std::max<uint64_t>(n, 1) * 4, 0.0f);
        for (uint64_t k = 0; k < n; ++k)
            for (int i = 0; i < 3; ++i) a[4 * k + i] = rgb[3 * k + i];
        SS_CUDA(cudaMemcpyAsync(c->color.ensure(std::max<uint64_t>(n, 1) * 16), a.data(), n * 16,
                                cudaMemcpyHostToDevice, c->stream));
        SS_CUDA(cudaStreamSynchronize(c->stream));
        c->color_ok = true;
    });
}

int ss_render(ss_ctx* c, const ss_camera* cam, int mode, uint64_t* n_entries, uint64_t* n_splats,
              uint64_t* n_tile_instances) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!c->color_ok && c->n) throw Error(SS_ERR_CONTRACT, "ss_render: scene colors not set (ss_scene_set_color)");
        capture_view(c, cam, mode, true, n_entries, n_splats, n_tile_instances);
    });
}

int ss_render_fetch_image(ss_ctx* c, float* rgb) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!c->cap_image) throw Error(SS_ERR_CONTRACT, "ss_render_fetch_image: the last capture was not a render");
        set_device(c);
        const uint64_t P = (uint64_t)c->cap_width * c->cap_height;
        if (P) SS_CUDA(cudaMemcpy(rgb, c->image.p, P * 12, cudaMemcpyDeviceToHost));
    });
}

int ss_raster_fetch(ss_ctx* c, ss_weight_entry* entries, float* per_pixel_total, float* alpha, uint32_t* splat_gid,
                    uint32_t* tile_offsets, uint32_t* tile_splats) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        const uint64_t P = (uint64_t)c->cap_width * c->cap_height;
        if (entries && c->cap_entries)
            SS_CUDA(cudaMemcpy(entries, c->entries.p, c->cap_entries * sizeof(ss_weight_entry), cudaMemcpyDeviceToHost));
        if (per_pixel_total && P) SS_CUDA(cudaMemcpy(per_pixel_total, c->per_pixel_total.p, P * 4, cudaMemcpyDeviceToHost));
        if (alpha && P) SS_CUDA(cudaMemcpy(alpha, c->alpha.p, P * 4, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> order(c->cap_splats);
        if (c->cap_splats)
            SS_CUDA(cudaMemcpy(order.data(), c->lanes[0].order.p, c->cap_splats * 4, cudaMemcpyDeviceToHost));
        if (splat_gid) std::copy(order.begin(), order.end(), splat_gid);
        if (tile_offsets && c->cap_tiles) {
            // tiles are contiguous in key order: tile t starts after all instances of tiles < t
            std::vector<uint32_t> st(c->cap_tiles), en(c->cap_tiles);
            SS_CUDA(cudaMemcpy(st.data(), c->lanes[0].tile_start.p, c->cap_tiles * 4, cudaMemcpyDeviceToHost));
            SS_CUDA(cudaMemcpy(en.data(), c->lanes[0].tile_end.p, c->cap_tiles * 4, cudaMemcpyDeviceToHost));
            uint32_t run = 0;
            for (uint32_t t = 0; t < c->cap_tiles; ++t) {
                tile_offsets[t] = run;
                run += en[t] - st[t];
            }
            tile_offsets[c->cap_tiles] = run;
        }
        if (tile_splats && c->cap_instances) {
            // tile lists hold Gaussian ids; report them as indices into the
            // depth-sorted splat list, as the reference's tile_bins do
            std::vector<uint32_t> ids(c->cap_instances);
            if (c->cap_tile_sort) {
                // per-tile slot ranges: gather them in tile order
                std::vector<uint32_t> st(c->cap_tiles), en(c->cap_tiles);
                SS_CUDA(cudaMemcpy(st.data(), c->lanes[0].tile_start.p, c->cap_tiles * 4, cudaMemcpyDeviceToHost));
                SS_CUDA(cudaMemcpy(en.data(), c->lanes[0].tile_end.p, c->cap_tiles * 4, cudaMemcpyDeviceToHost));
                const uint64_t span = en.empty() ? 0 : *std::max_element(en.begin(), en.end());
                std::vector<uint32_t> all(span);
                if (span) SS_CUDA(cudaMemcpy(all.data(), c->lanes[0].list.p, span * 4, cudaMemcpyDeviceToHost));
                uint64_t k = 0;
                for (uint32_t t = 0; t < c->cap_tiles; ++t)
                    for (uint32_t i = st[t]; i < en[t]; ++i) ids[k++] = all[i];
            } else {
                SS_CUDA(cudaMemcpy(ids.data(), c->lanes[0].list.p, c->cap_instances * 4, cudaMemcpyDeviceToHost));
            }
            std::vector<uint32_t> rank_of(c->n, 0xffffffffu);
            for (uint64_t r = 0; r < order.size(); ++r) rank_of[order[r]] = (uint32_t)r;
            for (uint64_t i = 0; i < ids.size(); ++i) tile_splats[i] = rank_of[ids[i]];
        }
    });
}

int ss_encode_begin(ss_ctx* c, uint32_t dim, float* d_sums, float* d_totals) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (dim == 0) throw Error(SS_ERR_CONTRACT, "embedding dimension must be positive");
        if ((d_sums == nullptr) != (d_totals == nullptr))
            throw Error(SS_ERR_CONTRACT, "pass both external accumulators or neither");
        set_device(c);
        c->dim = dim;
        // rows padded to whole combine rounds (= N on one device without blocks);
        // external buffers must hold ss_combine_layout's rows_alloc rows
        const uint64_t N = std::max<uint64_t>(combine_layout(c->n, c->nranks, c->combine_rows).rows_alloc, 1);
        c->acc_rows = N;
        if (d_sums) {
            c->sums = d_sums;
            c->totals = d_totals;
            c->own_acc = false;
        } else {
            c->sums = static_cast<float*>(c->sums_buf.ensure(N * dim * 4));
            c->totals = static_cast<float*>(c->totals_buf.ensure(N * 4));
            c->own_acc = true;
        }
        SS_CUDA(cudaMemsetAsync(c->sums, 0, N * dim * 4, c->stream));
        SS_CUDA(cudaMemsetAsync(c->totals, 0, N * 4, c->stream));
    });
}

int ss_encode_view(ss_ctx* c, const ss_camera* cam, const ss_view_masks* masks, int mode) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        encode_batch(c, 1, cam, masks, mode);
    });
}

int ss_encode_views(ss_ctx* c, uint32_t nviews, const ss_camera* cams, const ss_view_masks* masks, int mode) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        encode_batch(c, nviews, cams, masks, mode);
    });
}

int ss_encode_finalize(ss_ctx* c, uint64_t row_lo, uint64_t row_hi, float* rows_out, float* coverage_out,
                       int out_on_device) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!c->sums) throw Error(SS_ERR_CONTRACT, "finalize before ss_encode_begin");
        if (row_lo > row_hi || row_hi > c->n) throw Error(SS_ERR_CONTRACT, "finalize_into: rows do not fit the table");
        set_device(c);
        const uint64_t n = row_hi - row_lo;
        if (n == 0) return;
        cudaStream_t s = c->stream;
        float* d_rows = rows_out;
        float* d_cov = coverage_out;
        if (!out_on_device) {
            d_rows = static_cast<float*>(c->scores.ensure(n * c->dim * 4 + n * 4));
            d_cov = d_rows + n * c->dim;
        }
        {
            Scope sc(c, s, SS_K_NORMALIZE);
            own_launch(c,
                       launch_normalize(c->sums + row_lo * c->dim, c->totals + row_lo, n, c->dim, d_rows, d_cov,
                                        c->counters.as<unsigned long long>() + 3, s),
                       SS_K_NORMALIZE);
            // totals read + rows and coverage written; covered rows' sums (read) are added at readout
            c->prof.bytes[SS_K_NORMALIZE] += (double)n * (4.0 * c->dim + 8.0);
        }
        if (!out_on_device) {
            copy_d2h_pageable(c, rows_out, d_rows, n * c->dim * 4, s);
            copy_d2h_pageable(c, coverage_out, d_cov, n * 4, s);
        }
    });
}

int ss_encode_finalize_sparse(ss_ctx* c, uint64_t row_lo, uint64_t row_hi, float* rows_out, float* coverage_out,
                              uint64_t* covered_out) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!c->sums) throw Error(SS_ERR_CONTRACT, "finalize before ss_encode_begin");
        if (row_lo > row_hi || row_hi > c->n) throw Error(SS_ERR_CONTRACT, "finalize_into: rows do not fit the table");
        set_device(c);
        const uint64_t n = row_hi - row_lo;
        if (covered_out) *covered_out = 0;
        if (n == 0) return;
        cudaStream_t s = c->stream;
        const uint32_t D = c->dim;
        auto* d_rows = static_cast<float*>(c->scores.ensure(n * D * 4 + n * 4));
        float* d_cov = d_rows + n * D;
        {
            Scope sc(c, s, SS_K_NORMALIZE);
            own_launch(c,
                       launch_normalize(c->sums + row_lo * D, c->totals + row_lo, n, D, d_rows, d_cov,
                                        c->counters.as<unsigned long long>() + 3, s),
                       SS_K_NORMALIZE);
            c->prof.bytes[SS_K_NORMALIZE] += (double)n * (4.0 * D + 8.0);
        }
        // covered rows packed on the device: ids, coverage, rows
        auto* pk = static_cast<char*>(c->sparse_out.ensure(n * 4 + n * 4 + n * (uint64_t)D * 4 + 16));
        auto* d_cnt = reinterpret_cast<unsigned long long*>(pk);
        auto* d_ids = reinterpret_cast<uint32_t*>(pk + 16);
        float* d_pcov = reinterpret_cast<float*>(pk + 16 + n * 4);
        float* d_prow = reinterpret_cast<float*>(pk + 16 + n * 8);
        SS_CUDA(cudaMemsetAsync(d_cnt, 0, 8, s));
        own_launch(c, launch_compact_covered(d_rows, d_cov, n, D, d_ids, d_pcov, d_prow, d_cnt, s), SS_K_NORMALIZE);
        unsigned long long cnt = 0;
        SS_CUDA(cudaMemcpyAsync(&cnt, d_cnt, 8, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        if (covered_out) *covered_out = cnt;
        if (cnt == 0) return;
        std::vector<uint32_t> ids(cnt);
        std::vector<float> pcov(cnt);
        SS_CUDA(cudaMemcpyAsync(ids.data(), d_ids, cnt * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaMemcpyAsync(pcov.data(), d_pcov, cnt * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        for (uint64_t k = 0; k < cnt; ++k) coverage_out[ids[k]] = pcov[k];
        // the packed rows through the pinned staging buffers, scattered by id
        // into the caller's (zero) table while the next chunk is in flight
        if (!c->h_stage) {
            SS_CUDA(cudaMallocHost(&c->h_stage, 2 * kStageBytes));
            for (auto& e : c->stage_ev) SS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const uint64_t row_bytes = (uint64_t)D * 4, per_chunk = std::max<uint64_t>(1, kStageBytes / row_bytes);
        const uint64_t chunks = (cnt + per_chunk - 1) / per_chunk;
        auto issue = [&](uint64_t k) {
            const uint64_t r0 = k * per_chunk, nr = std::min<uint64_t>(per_chunk, cnt - r0);
            SS_CUDA(cudaMemcpyAsync(c->h_stage + (k & 1) * kStageBytes, d_prow + r0 * D, nr * row_bytes,
                                    cudaMemcpyDeviceToHost, s));
            SS_CUDA(cudaEventRecord(c->stage_ev[k & 1], s));
        };
        const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
        issue(0);
        for (uint64_t k = 0; k < chunks; ++k) {
            if (k + 1 < chunks) issue(k + 1);
            SS_CUDA(cudaEventSynchronize(c->stage_ev[k & 1]));
            const uint64_t r0 = k * per_chunk, nr = std::min<uint64_t>(per_chunk, cnt - r0);
            const float* src = reinterpret_cast<const float*>(c->h_stage + (k & 1) * kStageBytes);
            auto scatter = [&](uint64_t a, uint64_t b) {
                for (uint64_t j = a; j < b; ++j) std::memcpy(rows_out + (uint64_t)ids[r0 + j] * D, src + j * D, row_bytes);
            };
            const uint64_t per = (nr + hw - 1) / hw;
            std::vector<std::thread> th;
            for (unsigned t = 1; t < hw && t * per < nr; ++t)
                th.emplace_back([=] { scatter(t * per, std::min<uint64_t>(nr, (t + 1) * per)); });
            scatter(0, std::min<uint64_t>(nr, per));
            for (auto& x : th) x.join();
        }
    });
}

int ss_normalize_device(ss_ctx* c, const float* d_sums, const float* d_totals, uint64_t n, uint32_t dim,
                        float* d_rows_out, float* d_coverage_out) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        Scope sc(c, c->stream, SS_K_NORMALIZE);
        own_launch(c,
                   launch_normalize(d_sums, d_totals, n, dim, d_rows_out, d_coverage_out,
                                    c->counters.as<unsigned long long>() + 3, c->stream),
                   SS_K_NORMALIZE);
        c->prof.bytes[SS_K_NORMALIZE] += (double)n * (4.0 * dim + 8.0);
    });
}

// ------------------------------------------------------------------ store
int ss_store_set(ss_ctx* c, const uint32_t* ids, const float* unit_rows, uint64_t count, uint32_t dim) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        c->store_count = count;
        c->store_dim = dim;
        c->store_half_ok = false;
        SS_CUDA(cudaMemcpy(c->store_ids.ensure(std::max<uint64_t>(count, 1) * 4), ids, count * 4,
                           cudaMemcpyHostToDevice));
        SS_CUDA(cudaMemcpy(c->store_rows.ensure(std::max<uint64_t>(count, 1) * dim * 4), unit_rows,
                           count * dim * 4, cudaMemcpyHostToDevice));
        // the reference's VectorStore does not enforce unit rows (vecstore.hpp:61):
        // bound the norms so the tensor-core margin stays a proof
        auto* nb = static_cast<unsigned int*>(c->zero_flag.ensure(16));
        SS_CUDA(cudaMemsetAsync(nb, 0, 4, c->stream));
        own_launch(c, launch_row_norm_max(c->store_rows.as<float>(), count, dim, nb, c->stream), SS_K_QUERY);
        SS_CUDA(cudaMemcpyAsync(c->h_u32, nb, 4, cudaMemcpyDeviceToHost, c->stream));
        SS_CUDA(cudaStreamSynchronize(c->stream));
        float nm;
        std::memcpy(&nm, c->h_u32, 4);
        c->store_norm = nm;
    });
}

int ss_store_build(ss_ctx* c, const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                   uint64_t* count_out) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        cudaStream_t s = c->stream;
        auto* d_in = static_cast<float*>(c->scores.ensure(std::max<uint64_t>(n, 1) * (dim + 1) * 4));
        float* d_cov = d_in + n * dim;
        SS_CUDA(cudaMemcpyAsync(d_in, rows, n * dim * 4, cudaMemcpyHostToDevice, s));
        SS_CUDA(cudaMemcpyAsync(d_cov, coverage, n * 4, cudaMemcpyHostToDevice, s));
        auto* flags = static_cast<uint8_t*>(c->sel_flags.ensure(std::max<uint64_t>(n, 1)));
        auto* ids = static_cast<uint32_t*>(c->store_ids.ensure(std::max<uint64_t>(n, 1) * 4));
        auto* num = static_cast<int*>(c->num_sel.ensure(16));
        own_launch(c, launch_flag_covered(d_cov, n, flags, s), SS_K_QUERY);
        size_t tb = 0;
        thrust::counting_iterator<uint32_t> it(0);
        SS_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flags, ids, num, (int)n, s));
        void* tmp = c->cub_tmp.ensure(tb);
        tb = c->cub_tmp.bytes;
        SS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, it, flags, ids, num, (int)n, s));
        c->launches_cub += 1;
        SS_CUDA(cudaMemcpyAsync(c->h_u32, num, 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        const uint64_t count = c->h_u32[0];
        auto* out = static_cast<float*>(c->store_rows.ensure(std::max<uint64_t>(count, 1) * dim * 4));
        auto* zf = static_cast<int*>(c->zero_flag.ensure(16));
        SS_CUDA(cudaMemsetAsync(zf, 0, 4, s));
        own_launch(c, launch_normalize_rows(d_in, ids, count, dim, out, zf, s), SS_K_QUERY);
        SS_CUDA(cudaMemcpyAsync(c->h_u32, zf, 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        if (c->h_u32[0]) throw Error(SS_ERR_DATA, "build_store: a covered gaussian has a zero embedding row");
        c->store_count = count;
        c->store_dim = dim;
        c->store_half_ok = false;
        c->store_norm = 1.0f; // normalized_copy rows
        if (count_out) *count_out = count;
    });
}

// eval.hpp:122-158 assign_classes.  rows/coverage: host arrays, or device
// pointers with SS_ROWS_ON_DEVICE (e.g. the shard ss_encode_finalize left on
// the device); labels and out are host arrays.
int ss_assign_classes(ss_ctx* c, const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                      const int32_t* label_ids, const float* label_vecs, uint32_t n_labels, int32_t* out, int flags) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (n_labels == 0) throw Error(SS_ERR_CONTRACT, "assign_classes: empty label set");
        if (dim == 0) throw Error(SS_ERR_CONTRACT, "assign_classes: label vector dimension mismatch");
        set_device(c);
        cudaStream_t s = c->stream;
        const float* d_rows = rows;
        const float* d_cov = coverage;
        if (!(flags & SS_ROWS_ON_DEVICE)) {
            auto* buf = static_cast<float*>(c->scores.ensure(std::max<uint64_t>(n, 1) * (dim + 1) * 4));
            SS_CUDA(cudaMemcpyAsync(buf, rows, n * dim * 4, cudaMemcpyHostToDevice, s));
            SS_CUDA(cudaMemcpyAsync(buf + n * dim, coverage, n * 4, cudaMemcpyHostToDevice, s));
            d_rows = buf;
            d_cov = buf + n * dim;
        }
        auto* lab = static_cast<char*>(c->qbuf.ensure((uint64_t)n_labels * (2ull * dim * 4 + 8 + 4) + 256));
        float* d_lv = reinterpret_cast<float*>(lab);
        float* d_lt = d_lv + (size_t)n_labels * dim;
        double* d_ln = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(d_lt + (size_t)n_labels * dim) + 15) & ~uintptr_t(15));
        int32_t* d_lid = reinterpret_cast<int32_t*>(d_ln + n_labels);
        SS_CUDA(cudaMemcpyAsync(d_lv, label_vecs, (size_t)n_labels * dim * 4, cudaMemcpyHostToDevice, s));
        SS_CUDA(cudaMemcpyAsync(d_lid, label_ids, (size_t)n_labels * 4, cudaMemcpyHostToDevice, s));
        auto* d_out = static_cast<int32_t*>(c->topk_ids.ensure(std::max<uint64_t>(n, 1) * 4));
        own_launch(c, launch_assign_classes(d_rows, d_cov, n, dim, d_lid, d_lv, n_labels, d_lt, d_ln, d_out, s),
                   SS_K_QUERY, 2);
        if (n) SS_CUDA(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
    });
}

int ss_store_fetch(ss_ctx* c, uint32_t* ids, float* unit_rows) {
    return guarded([&] {
        set_device(c);
        if (ids && c->store_count)
            SS_CUDA(cudaMemcpy(ids, c->store_ids.p, c->store_count * 4, cudaMemcpyDeviceToHost));
        if (unit_rows && c->store_count)
            SS_CUDA(cudaMemcpy(unit_rows, c->store_rows.p, c->store_count * c->store_dim * 4, cudaMemcpyDeviceToHost));
    });
}

// vecstore.hpp:169-213 partition_store of the device store
int ss_store_partition(ss_ctx* c, const float* means_xyz, double cell_size, uint64_t* n_cells) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!(cell_size > 0)) throw Error(SS_ERR_CONTRACT, "partition_store: cell_size must be positive");
        set_device(c);
        const uint64_t n = c->store_count;
        c->part_cells = 0;
        if (n_cells) *n_cells = 0;
        if (n == 0) return;
        if (n >= (1ull << 31)) throw Error(SS_ERR_CONTRACT, "partition_store: more than 2^31 records");
        cudaStream_t s = c->stream;
        const uint32_t dim = c->store_dim;
        auto* means = static_cast<float*>(c->part_means.ensure(n * 12));
        SS_CUDA(cudaMemcpyAsync(means, means_xyz, n * 12, cudaMemcpyHostToDevice, s));
        // carve the scratch out of one allocation (256-byte aligned pieces)
        const size_t tmp = ss::partition_tmp_bytes(n);
        const size_t sizes[] = {24, n * 8, n * 8, n * 4, n * 4, n * 4, n * 4, n * 4, n * 4, n, n * 4, 16, n * 12,
                                (n + 1) * 8, n * dim * 4ull, n * 4, tmp};
        size_t total = 0;
        for (size_t z : sizes) total += (z + 255) / 256 * 256;
        char* b = static_cast<char*>(c->part_buf.ensure(total));
        void* piece[17];
        for (int i = 0; i < 17; ++i) {
            piece[i] = b;
            b += (sizes[i] + 255) / 256 * 256;
        }
        ss::PartitionScratch& w = c->part;
        w.mn3 = static_cast<unsigned long long*>(piece[0]);
        w.yz = static_cast<unsigned long long*>(piece[1]);
        w.yz_s = static_cast<unsigned long long*>(piece[2]);
        w.kx = static_cast<uint32_t*>(piece[3]);
        w.kx_p = static_cast<uint32_t*>(piece[4]);
        w.kx_s = static_cast<uint32_t*>(piece[5]);
        w.idx = static_cast<uint32_t*>(piece[6]);
        w.perm1 = static_cast<uint32_t*>(piece[7]);
        w.perm2 = static_cast<uint32_t*>(piece[8]);
        w.head = static_cast<uint8_t*>(piece[9]);
        w.heads = static_cast<uint32_t*>(piece[10]);
        w.n_heads = static_cast<int*>(piece[11]);
        w.cells = static_cast<int32_t*>(piece[12]);
        w.offsets = static_cast<uint64_t*>(piece[13]);
        w.out_rows = static_cast<float*>(piece[14]);
        w.out_ids = static_cast<uint32_t*>(piece[15]);
        w.tmp = piece[16];
        w.tmp_bytes = tmp;
        own_launch(c,
                   ss::launch_store_partition(means, c->store_rows.as<float>(), c->store_ids.as<uint32_t>(), n, dim,
                                              cell_size, w, s),
                   SS_K_QUERY, 9);
        c->launches_cub += 3;
        unsigned long long mn[3];
        int nh = 0;
        SS_CUDA(cudaMemcpyAsync(mn, w.mn3, 24, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaMemcpyAsync(&nh, w.n_heads, 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        for (int a = 0; a < 3; ++a) {
            // inverse of the ordered-key map; all-NaN axes keep Aabb's initial DBL_MAX
            const unsigned long long k = mn[a];
            const unsigned long long bits = k == ~0ull ? 0x7fefffffffffffffull
                                                       : ((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
            std::memcpy(&c->part_min[a], &bits, 8);
        }
        c->part_cells = (uint64_t)nh;
        if (n_cells) *n_cells = (uint64_t)nh;
    });
}

int ss_store_partition_fetch(ss_ctx* c, int32_t* cells, uint64_t* offsets, uint32_t* order, uint32_t* ids,
                             float* rows, double* bbox_min) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        const uint64_t n = c->store_count, nc = c->part_cells;
        if (bbox_min) std::memcpy(bbox_min, c->part_min, 24);
        if (!nc) return;
        const ss::PartitionScratch& w = c->part;
        if (cells) SS_CUDA(cudaMemcpy(cells, w.cells, nc * 12, cudaMemcpyDeviceToHost));
        if (offsets) SS_CUDA(cudaMemcpy(offsets, w.offsets, (nc + 1) * 8, cudaMemcpyDeviceToHost));
        if (order) SS_CUDA(cudaMemcpy(order, w.perm2, n * 4, cudaMemcpyDeviceToHost));
        if (ids) SS_CUDA(cudaMemcpy(ids, w.out_ids, n * 4, cudaMemcpyDeviceToHost));
        if (rows) SS_CUDA(cudaMemcpy(rows, w.out_rows, n * c->store_dim * 4ull, cudaMemcpyDeviceToHost));
    });
}

namespace {
// vecstore.hpp:112-115 prepare_query for nq raw queries -> device unit queries
float* prepare_queries(ss_ctx* c, const float* queries, uint32_t nq) {
    cudaStream_t s = c->stream;
    const uint32_t dim = c->store_dim;
    auto* d_q = static_cast<float*>(c->qbuf.ensure(std::max<uint64_t>(nq, 1) * dim * 4));
    auto* d_qn = static_cast<float*>(c->qnorm.ensure(std::max<uint64_t>(nq, 1) * dim * 4));
    SS_CUDA(cudaMemcpyAsync(d_q, queries, (size_t)nq * dim * 4, cudaMemcpyHostToDevice, s));
    auto* zf = static_cast<int*>(c->zero_flag.ensure(16));
    SS_CUDA(cudaMemsetAsync(zf, 0, 4, s));
    own_launch(c, launch_normalize_rows(d_q, nullptr, nq, dim, d_qn, zf, s), SS_K_QUERY);
    // the zero-norm flag is read back with the results (no round trip here);
    // check_query_norm() raises prepare_query's NumericError after the next sync
    c->h_u32[1] = 0;
    SS_CUDA(cudaMemcpyAsync(c->h_u32 + 1, zf, 4, cudaMemcpyDeviceToHost, s));
    return d_qn;
}

// vecstore.hpp:37 -- after a stream sync that followed prepare_queries
void check_query_norm(ss_ctx* c) {
    if (c->h_u32[1]) throw Error(SS_ERR_NUMERIC, "cannot normalize a zero vector");
}
} // namespace

namespace {
// Exact scan: every (query, row) score with the exact dot_lanes, per-query
// top-k by (sim desc, id asc).  Rows of out are [q][k].
void topk_exact(ss_ctx* c, const float* d_qn, uint32_t nq, uint32_t k, uint32_t* oid, float* osim) {
    cudaStream_t s = c->stream;
    const uint64_t count = c->store_count;
    const uint32_t qt = (uint32_t)score_query_tile();
    const uint32_t tile = std::max<uint32_t>(qt, 64);
    auto* sc_buf = static_cast<float*>(c->scores.ensure((size_t)tile * count * 4));
    for (uint32_t q0 = 0; q0 < nq; q0 += tile) {
        const uint32_t nt = std::min(tile, nq - q0);
        for (uint32_t t = 0; t < nt; t += qt)
            own_launch(c, launch_score(c->store_rows.as<float>(), count, c->store_dim, d_qn, q0 + std::min(nt, t + qt),
                                       q0 + t, sc_buf + (size_t)t * count, s),
                       SS_K_QUERY);
        own_launch(c, launch_topk(sc_buf, c->store_ids.as<uint32_t>(), count, k, nt, q0, oid, osim, s), SS_K_QUERY);
    }
}

// k beyond the top-k kernels' 64: every record's exact score, a full radix
// sort of the (sim desc, id asc) keys, the first k (vecstore.hpp:121-132).
void topk_sorted(ss_ctx* c, const float* d_qn, uint32_t nq, uint32_t k, uint32_t* oid, float* osim) {
    cudaStream_t s = c->stream;
    const uint64_t count = c->store_count;
    const uint64_t take = std::min<uint64_t>(k, count);
    auto* sc_buf = static_cast<float*>(c->scores.ensure(count * 4));
    auto* keys = static_cast<unsigned long long*>(c->thr_keys.ensure(count * 8));
    auto* ksorted = static_cast<unsigned long long*>(c->thr_keys_sorted.ensure(count * 8));
    auto* flags = static_cast<uint8_t*>(c->sel_flags.ensure(count));
    size_t tb = 0;
    SS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, ksorted, (int)count, 0, 64, s));
    void* tmp = c->cub_tmp.ensure(tb);
    tb = c->cub_tmp.bytes;
    // queries back to back on the stream; each query's first k keys are decoded
    // into its result row on the device
    for (uint32_t q = 0; q < nq; ++q) {
        own_launch(c, launch_score(c->store_rows.as<float>(), count, c->store_dim, d_qn, q + 1, q, sc_buf, s),
                   SS_K_QUERY);
        own_launch(c, launch_threshold_keys(sc_buf, c->store_ids.as<uint32_t>(), count, -INFINITY, keys, flags, s),
                   SS_K_QUERY);
        SS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, ksorted, (int)count, 0, 64, s));
        c->launches_cub += 1;
        own_launch(c, launch_decode_keys(ksorted, take, oid + (uint64_t)q * k, osim + (uint64_t)q * k, s),
                   SS_K_QUERY);
    }
}

// |coarse - exact| <= kCoarseEps for unit rows and unit queries; every term
// of the bound (fp16 operand rounding, fp32 accumulation, fp16 pilot scores,
// the exact scorer's rounding) scales with the row norm
float coarse_eps(const ss_ctx* c) { return ss::kCoarseEps * std::max(1.0f, c->store_norm); }

constexpr uint32_t kQueryChunk = 1024; // queries per coarse-score pass
constexpr uint32_t kCandCap = 4096;    // candidates kept per query

// Tensor-core path: fp16 coarse scores (tcgen05), candidate selection with a
// proven margin, exact rescoring.  Returns false when some query's candidate
// set is unusable (overflow, or fewer than k finite candidates); the caller
// then answers with the exact scan.
bool topk_tensor(ss_ctx* c, const float* d_qn, uint32_t nq, uint32_t k, uint32_t* oid, float* osim) {
    cudaStream_t s = c->stream;
    const uint64_t count = c->store_count;
    const uint32_t dim = c->store_dim;
    if (!c->num_sms) SS_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (!c->store_half_ok) {
        void* h = c->store_half.ensure(count * dim * 2);
        own_launch(c, ss::launch_to_half(c->store_rows.as<float>(), count * dim, h, s), SS_K_QUERY);
        c->store_half_ok = true;
    }
    void* qh = c->qhalf.ensure((uint64_t)nq * dim * 2);
    own_launch(c, ss::launch_to_half(d_qn, (uint64_t)nq * dim, qh, s), SS_K_QUERY);
    const uint32_t chunk = std::min(nq, kQueryChunk);
    const uint64_t pcols = ss::pilot_cols((uint32_t)count);
    void* pscores = c->tc_scores.ensure((uint64_t)chunk * pcols * 2);
    auto* thr = static_cast<float*>(c->tc_thr.ensure((uint64_t)nq * 4));
    auto* cand = static_cast<uint32_t*>(c->cand.ensure((uint64_t)nq * kCandCap * 4));
    auto* ccount = static_cast<uint32_t*>(c->cand_count.ensure((uint64_t)nq * 4));
    auto* cval = static_cast<float*>(c->cand_sim.ensure((uint64_t)nq * kCandCap * 4));
    SS_CUDA(cudaMemsetAsync(ccount, 0, (size_t)nq * 4, s));
    for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
        const uint32_t nt = std::min(chunk, nq - q0);
        const void* qc = static_cast<const char*>(qh) + (uint64_t)q0 * dim * 2;
        {
            // pilot over a strided sample of row tiles -> per-query threshold
            Scope sp(c, s, SS_K_QUERY_SELECT);
            own_launch(c, ss::launch_coarse_pilot(c->store_half.p, (uint32_t)count, qc, nt, dim, pscores, c->num_sms, s),
                       SS_K_QUERY);
            own_launch(c,
                       ss::launch_pilot_threshold(pscores, (uint32_t)count, nt, k, 2.0f * coarse_eps(c), thr + q0, s),
                       SS_K_QUERY);
            c->prof.bytes[SS_K_QUERY_SELECT] += 2.0 * nt * (double)pcols * dim;
        }
        {
            Scope sg(c, s, SS_K_QUERY_GEMM);
            own_launch(c,
                       ss::launch_coarse_candidates(c->store_half.p, (uint32_t)count, qc, nt, dim, thr + q0,
                                                    cand + (uint64_t)q0 * kCandCap, cval + (uint64_t)q0 * kCandCap,
                                                    kCandCap, ccount + q0, c->num_sms, s),
                       SS_K_QUERY);
            c->prof.bytes[SS_K_QUERY_GEMM] += 2.0 * nt * (double)count * dim; // flops
        }
    }
    {
        Scope sr(c, s, SS_K_QUERY_SELECT);
        own_launch(c,
                   ss::launch_rescore(c->store_rows.as<float>(), c->store_ids.as<uint32_t>(), dim, d_qn, nq, cand,
                                      cval, kCandCap, ccount, k, 2.0f * coarse_eps(c), oid, osim, s),
                   SS_K_QUERY);
    }
    std::vector<uint32_t> hc(nq);
    SS_CUDA(cudaMemcpyAsync(hc.data(), ccount, (size_t)nq * 4, cudaMemcpyDeviceToHost, s));
    SS_CUDA(cudaStreamSynchronize(s));
    const uint64_t take = std::min<uint64_t>(k, count);
    bool ok = true;
    for (uint32_t q = 0; q < nq; ++q) {
        if (hc[q] <= kCandCap) {
            c->qstat[1] += hc[q];
            c->qstat[2] = std::max<uint64_t>(c->qstat[2], hc[q]);
        }
        if (hc[q] > kCandCap || hc[q] < take) ok = false;
    }
    c->qstat[0] += nq;
    if (!ok) c->qstat[3] += 1;
    return ok;
}
} // namespace

namespace {
bool tc_eligible(const ss_ctx* c) {
    // rows beyond norm 1e4 (or non-finite) could overflow the fp16 operands and scores
    return c->store_norm <= 1.0e4f && c->store_dim % 64 == 0 && c->store_dim <= 512 && c->store_count < (1ull << 31) &&
           (c->query_path == 2 || (c->query_path == 0 && c->store_count >= 16384));
}

// query_threshold on the tensor cores: candidates with coarse >= tau - eps
// (a superset of {exact >= tau}), exact rescoring, (sim desc, id asc) order.
// False when the candidates overflow; the caller then runs the exact scan.
bool threshold_tensor(ss_ctx* c, const float* d_qn, float tau, uint32_t* out_ids, float* out_sims, uint64_t capacity,
                      uint64_t* out_count) {
    cudaStream_t s = c->stream;
    const uint64_t count = c->store_count;
    const uint32_t dim = c->store_dim;
    if (!c->num_sms) SS_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (!c->store_half_ok) {
        void* h = c->store_half.ensure(count * dim * 2);
        own_launch(c, ss::launch_to_half(c->store_rows.as<float>(), count * dim, h, s), SS_K_QUERY);
        c->store_half_ok = true;
    }
    void* qh = c->qhalf.ensure((uint64_t)dim * 2);
    own_launch(c, ss::launch_to_half(d_qn, dim, qh, s), SS_K_QUERY);
    auto* thr = static_cast<float*>(c->tc_thr.ensure(64));
    auto* cand = static_cast<uint32_t*>(c->cand.ensure((uint64_t)kCandCap * 4));
    auto* cval = static_cast<float*>(c->cand_sim.ensure((uint64_t)kCandCap * 4));
    auto* ccount = static_cast<uint32_t*>(c->cand_count.ensure(64));
    auto* oid = static_cast<uint32_t*>(c->topk_ids.ensure((uint64_t)kCandCap * 4));
    auto* osim = static_cast<float*>(c->topk_sims.ensure((uint64_t)kCandCap * 4));
    c->h_u32[0] = 0;
    float h_thr = tau - coarse_eps(c);
    SS_CUDA(cudaMemcpyAsync(thr, &h_thr, 4, cudaMemcpyHostToDevice, s));
    SS_CUDA(cudaMemsetAsync(ccount, 0, 8, s));
    {
        Scope sg(c, s, SS_K_QUERY_GEMM);
        own_launch(c,
                   ss::launch_coarse_candidates(c->store_half.p, (uint32_t)count, qh, 1, dim, thr, cand, cval,
                                                kCandCap, ccount, c->num_sms, s),
                   SS_K_QUERY);
    }
    {
        Scope sr(c, s, SS_K_QUERY_SELECT);
        own_launch(c,
                   ss::launch_threshold_rescore(c->store_rows.as<float>(), c->store_ids.as<uint32_t>(), dim, d_qn,
                                                cand, kCandCap, ccount, tau, oid, osim, kCandCap, ccount + 1, s),
                   SS_K_QUERY);
    }
    uint32_t hc[2];
    SS_CUDA(cudaMemcpyAsync(hc, ccount, 8, cudaMemcpyDeviceToHost, s));
    SS_CUDA(cudaStreamSynchronize(s));
    check_query_norm(c);
    if (hc[0] > kCandCap) {
        c->qstat[3] += 1;
        return false;
    }
    const uint64_t m = hc[1], out = std::min<uint64_t>(m, capacity);
    if (out) {
        SS_CUDA(cudaMemcpyAsync(out_ids, oid, out * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaMemcpyAsync(out_sims, osim, out * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
    }
    c->qstat[0] += 1;
    c->qstat[1] += hc[0];
    c->qstat[2] = std::max<uint64_t>(c->qstat[2], hc[0]);
    *out_count = m;
    return true;
}
} // namespace

int ss_query_topk(ss_ctx* c, const float* queries, uint32_t nq, uint32_t k, uint32_t* out_ids, float* out_sims,
                  uint64_t* out_counts) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        set_device(c);
        const uint64_t count = c->store_count;
        const uint64_t take = std::min<uint64_t>(k, count);
        for (uint32_t q = 0; q < nq; ++q) out_counts[q] = (k == 0 || count == 0) ? 0 : take;
        if (k == 0 || count == 0 || nq == 0) return; // vecstore.hpp:122

        cudaStream_t s = c->stream;
        Scope sc(c, s, SS_K_QUERY);
        const float* d_qn = prepare_queries(c, queries, nq);
        auto* oid = static_cast<uint32_t*>(c->topk_ids.ensure((size_t)nq * k * 4));
        auto* osim = static_cast<float*>(c->topk_sims.ensure((size_t)nq * k * 4));
        if (k > 64)
            topk_sorted(c, d_qn, nq, k, oid, osim);
        else if (!(tc_eligible(c) && topk_tensor(c, d_qn, nq, k, oid, osim)))
            topk_exact(c, d_qn, nq, k, oid, osim);
        // rows written are [q][k] with k stride; take <= k
        std::vector<uint32_t> hid((size_t)nq * k);
        std::vector<float> hsim((size_t)nq * k);
        SS_CUDA(cudaMemcpyAsync(hid.data(), oid, hid.size() * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaMemcpyAsync(hsim.data(), osim, hsim.size() * 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        check_query_norm(c);
        std::memcpy(out_ids, hid.data(), hid.size() * 4);
        std::memcpy(out_sims, hsim.data(), hsim.size() * 4);
        c->prof.bytes[SS_K_QUERY] += 2.0 * nq * (double)count * c->store_dim; // flops
    });
}

int ss_query_threshold(ss_ctx* c, const float* query, float tau, uint32_t* out_ids, float* out_sims,
                       uint64_t capacity, uint64_t* out_count) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!(tau >= -1.0f && tau <= 1.0f)) throw Error(SS_ERR_CONTRACT, "cosine threshold must lie in [-1, 1]");
        set_device(c);
        *out_count = 0;
        const uint64_t count = c->store_count;
        if (count == 0) return;
        cudaStream_t s = c->stream;
        const float* d_qn = prepare_queries(c, query, 1);
        if (tc_eligible(c) && threshold_tensor(c, d_qn, tau, out_ids, out_sims, capacity, out_count)) return;
        auto* sc_buf = static_cast<float*>(c->scores.ensure(count * 4));
        own_launch(c, launch_score(c->store_rows.as<float>(), count, c->store_dim, d_qn, 1, 0, sc_buf, s), SS_K_QUERY);
        auto* keys = static_cast<unsigned long long*>(c->thr_keys.ensure(count * 8));
        auto* flags = static_cast<uint8_t*>(c->sel_flags.ensure(count));
        own_launch(c, launch_threshold_keys(sc_buf, c->store_ids.as<uint32_t>(), count, tau, keys, flags, s), SS_K_QUERY);
        auto* ksel = static_cast<unsigned long long*>(c->thr_ids.ensure(count * 8));
        auto* ksorted = static_cast<unsigned long long*>(c->thr_keys_sorted.ensure(count * 8));
        auto* num = static_cast<int*>(c->num_sel.ensure(16));
        size_t tb = 0;
        SS_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, keys, flags, ksel, num, (int)count, s));
        size_t tb2 = 0;
        SS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, ksel, ksorted, (int)count, 0, 64, s));
        void* tmp = c->cub_tmp.ensure(std::max(tb, tb2));
        tb = c->cub_tmp.bytes;
        SS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, keys, flags, ksel, num, (int)count, s));
        SS_CUDA(cudaMemcpyAsync(c->h_u32, num, 4, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        check_query_norm(c);
        const uint64_t m = c->h_u32[0];
        tb = c->cub_tmp.bytes;
        SS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, ksel, ksorted, (int)m, 0, 64, s));
        c->launches_cub += 2;
        std::vector<unsigned long long> hk(m);
        SS_CUDA(cudaMemcpyAsync(hk.data(), ksorted, m * 8, cudaMemcpyDeviceToHost, s));
        SS_CUDA(cudaStreamSynchronize(s));
        const uint64_t out = std::min<uint64_t>(m, capacity);
        for (uint64_t i = 0; i < out; ++i) {
            out_ids[i] = (uint32_t)(hk[i] & 0xffffffffu);
            uint32_t b = ~(uint32_t)(hk[i] >> 32);
            b = (b & 0x80000000u) ? (b & 0x7fffffffu) : ~b;
            float f;
            std::memcpy(&f, &b, 4);
            out_sims[i] = f;
        }
        *out_count = m;
    });
}

// ------------------------------------------------------------ multi-GPU
int ss_device_count(int* n) {
    return guarded([&] {
        if (!n) throw Error(SS_ERR_CONTRACT, "output is null");
        *n = 0;
        cudaError_t e = cudaGetDeviceCount(n);
        if (e != cudaSuccess) {
            *n = 0;
            cudaGetLastError();
        }
    });
}

int ss_comm_unique_id(unsigned char id[SS_NCCL_UNIQUE_ID_BYTES]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == SS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
        if (!id) throw Error(SS_ERR_CONTRACT, "id is null");
        ncclUniqueId u;
        SS_NCCL(GetUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

int ss_comm_init(ss_ctx* c, int nranks, int rank, const unsigned char id[SS_NCCL_UNIQUE_ID_BYTES]) {
    return guarded([&] {
        if (!c || !id) throw Error(SS_ERR_CONTRACT, "ctx or id is null");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(SS_ERR_CONTRACT, "rank out of range");
        set_device(c);
        comm_release(c);
        comm_setup(c);
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        ncclComm_t comm = nullptr;
        SS_NCCL(CommInitRank(&comm, nranks, u, rank));
        c->comm = comm;
        c->own_comm = true;
        c->nranks = nranks;
        c->rank = rank;
    });
}

int ss_comm_init_all(ss_ctx* const* ctxs, int n) {
    return guarded([&] {
        if (!ctxs || n < 1) throw Error(SS_ERR_CONTRACT, "need at least one context");
        std::vector<int> devs(n);
        for (int i = 0; i < n; ++i) {
            if (!ctxs[i]) throw Error(SS_ERR_CONTRACT, "ctx is null");
            devs[i] = ctxs[i]->device;
            for (int j = 0; j < i; ++j)
                if (devs[j] == devs[i]) throw Error(SS_ERR_CONTRACT, "ss_comm_init_all: one context per device");
        }
        std::vector<ncclComm_t> comms(n, nullptr);
        for (int i = 0; i < n; ++i) {
            set_device(ctxs[i]);
            comm_release(ctxs[i]);
            comm_setup(ctxs[i]);
        }
        SS_NCCL(CommInitAll(comms.data(), n, devs.data()));
        for (int i = 0; i < n; ++i) {
            ctxs[i]->comm = comms[i];
            ctxs[i]->own_comm = true;
            ctxs[i]->nranks = n;
            ctxs[i]->rank = i;
        }
    });
}

int ss_combine_layout(ss_ctx* c, uint64_t* rows_alloc, uint64_t* block_rows, uint64_t* rounds, uint64_t* rank_rows) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        const CombineLayout L = combine_layout(c->n, c->nranks, c->combine_rows);
        if (rows_alloc) *rows_alloc = L.rows_alloc;
        if (block_rows) *block_rows = L.block;
        if (rounds) *rounds = L.rounds;
        if (rank_rows) *rank_rows = L.rounds * L.block;
    });
}

int ss_combine_layout_for(uint64_t n, int nranks, uint64_t combine_rows, uint64_t* rows_alloc, uint64_t* block_rows,
                          uint64_t* rounds) {
    return guarded([&] {
        if (nranks < 1) throw Error(SS_ERR_CONTRACT, "nranks must be >= 1");
        const CombineLayout L = combine_layout(n, nranks, combine_rows);
        if (rows_alloc) *rows_alloc = L.rows_alloc;
        if (block_rows) *block_rows = L.block;
        if (rounds) *rounds = L.rounds;
    });
}

// combine_partials (pipeline.hpp:90-100: the partials' elementwise sum) as a
// reduce-scatter per round on the communicator's stream, then finalize_into
// (pipeline.hpp:120-135) of the received rows on the context's stream; round
// q + 1's collective overlaps round q's normalisation (double-buffered).
namespace {
// ss_encode_combine over the covered rows only (SS_OPT_COMBINE_SPARSE): per
// round, an all-reduce (max) of every rank's covered flags, positions by a
// scan, the covered rows of each owner block packed into equal P-row segments
// (P = the largest owner's count), one grouped reduce-scatter of [sums |
// totals] segments, and the owner unpacks and normalises its block.  The
// rank's output block is the dense path's, row for row (uncovered rows zero).
void combine_sparse_rounds(ss_ctx* c, const CombineLayout& L, float* rows_out, float* coverage_out,
                           bool out_on_device) {
    const uint64_t D = c->dim, W = (uint64_t)c->nranks, B = L.block, RB = W * B;
    const uint64_t r = (uint64_t)c->rank;
    cudaStream_t s = c->stream;
    auto* flags = static_cast<uint8_t*>(c->sp_flags.ensure(RB + 1));
    auto* pos = static_cast<uint32_t*>(c->sp_pos.ensure((RB + 1) * 4));
    auto* bounds = static_cast<uint32_t*>(c->sp_bounds.ensure((W + 1) * 4));
    size_t tb = 0;
    SS_CUDA(launch_flag_positions(flags, RB, pos, nullptr, &tb, s));
    void* tmp = c->sp_tmp.ensure(std::max<size_t>(tb, 1));
    std::vector<uint32_t> hb(W + 1);
    for (uint64_t q = 0; q < L.rounds; ++q) {
        const uint64_t row0 = q * RB;
        {
            Scope sc(c, s, SS_K_COMBINE);
            own_launch(c, launch_covered_flags(c->totals + row0, RB, flags, s), SS_K_COMBINE);
            if (W > 1) SS_NCCL(AllReduce(flags, flags, RB, ncclUint8, ncclMax, c->comm, s));
            size_t tb2 = tb;
            SS_CUDA(launch_flag_positions(flags, RB, pos, tmp, &tb2, s));
            c->launches_cub += 1;
            for (uint64_t k = 0; k <= W; ++k)
                SS_CUDA(cudaMemcpyAsync(hb.data() + k, pos + k * B, 4, cudaMemcpyDeviceToHost, s));
            SS_CUDA(cudaStreamSynchronize(s));
        }
        uint64_t P = 0;
        for (uint64_t k = 0; k < W; ++k) P = std::max<uint64_t>(P, hb[k + 1] - hb[k]);
        const float* recv_s = nullptr;
        const float* recv_t = nullptr;
        if (P) {
            Scope sc(c, s, SS_K_COMBINE);
            auto* send = static_cast<float*>(c->sp_send.ensure((W * P * (D + 1) + P * (D + 1)) * 4));
            float* send_s = send;
            float* send_t = send + W * P * D;
            float* rs = send_t + W * P;
            float* rt = rs + P * D;
            SS_CUDA(cudaMemsetAsync(send, 0, W * P * (D + 1) * 4, s)); // padding rows stay zero
            own_launch(c,
                       launch_sparse_pack(c->sums + row0 * D, c->totals + row0, RB, (uint32_t)D, B, flags, pos, P,
                                          send_s, send_t, s),
                       SS_K_COMBINE);
            if (W > 1) {
                SS_NCCL(GroupStart());
                SS_NCCL(ReduceScatter(send_s, rs, P * D, ncclFloat32, ncclSum, c->comm, s));
                SS_NCCL(ReduceScatter(send_t, rt, P, ncclFloat32, ncclSum, c->comm, s));
                SS_NCCL(GroupEnd());
                recv_s = rs;
                recv_t = rt;
            } else {
                recv_s = send_s; // one rank: its packed rows are the combined ones
                recv_t = send_t;
            }
            c->prof.launches[SS_K_COMBINE] += 1;
            c->prof.bytes[SS_K_COMBINE] += (double)(W - 1) * P * (D + 1) * 4; // sent per rank
        }
        float* dr = out_on_device ? rows_out + q * B * D : c->rs_stage.as<float>();
        float* dc = out_on_device ? coverage_out + q * B : c->rs_stage.as<float>() + B * D;
        {
            Scope sc(c, s, SS_K_NORMALIZE);
            // P == 0: no covered row anywhere in the round; the unpack writes zeros
            own_launch(c,
                       launch_sparse_unpack(recv_s ? recv_s : c->sums, recv_t ? recv_t : c->totals, B, r * B, flags,
                                            pos, (uint32_t)D, dr, dc, c->counters.as<unsigned long long>() + 3, s),
                       SS_K_NORMALIZE);
            c->prof.bytes[SS_K_NORMALIZE] += (double)B * (4.0 * D + 8.0);
        }
        if (!out_on_device) {
            copy_d2h_pageable(c, rows_out + q * B * D, dr, B * D * 4, s);
            copy_d2h_pageable(c, coverage_out + q * B, dc, B * 4, s);
        } else if (q + 1 < L.rounds) {
            SS_CUDA(cudaStreamSynchronize(s)); // flags / pos / send are reused next round
        }
    }
}
} // namespace

int ss_encode_combine(ss_ctx* c, float* rows_out, float* coverage_out, int out_on_device) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        if (!c->sums) throw Error(SS_ERR_CONTRACT, "combine before ss_encode_begin");
        set_device(c);
        const CombineLayout L = combine_layout(c->n, c->nranks, c->combine_rows);
        if (L.rows_alloc != c->acc_rows)
            throw Error(SS_ERR_CONTRACT, "ss_encode_combine: communicator or SS_OPT_COMBINE_ROWS changed after ss_encode_begin");
        const uint64_t D = c->dim, W = (uint64_t)c->nranks, B = L.block;
        cudaStream_t s = c->stream;
        const bool collective = c->comm && W > 1;
        if (!out_on_device) c->rs_stage.ensure(B * (D + 1) * 4);
        const bool sparse = c->comm && (c->combine_sparse == 2 || (c->combine_sparse == 1 && W > 1));
        if (sparse) {
            combine_sparse_rounds(c, L, rows_out, coverage_out, out_on_device != 0);
            return;
        }
        if (collective) SS_CUDA(cudaEventRecord(c->ev_acc, s));
        for (uint64_t q = 0; q < L.rounds; ++q) {
            const int buf = (int)(q & 1);
            const float* src_s;
            const float* src_t;
            if (collective) {
                float* rs = static_cast<float*>(c->rs_sum[buf].ensure(B * D * 4));
                float* rt = static_cast<float*>(c->rs_tot[buf].ensure(B * 4));
                if (q == 0) SS_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_acc, 0));
                if (q >= 2) SS_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_norm[buf], 0));
                Scope sc(c, c->comm_stream, SS_K_COMBINE);
                SS_NCCL(GroupStart());
                SS_NCCL(ReduceScatter(c->sums + q * W * B * D, rs, B * D, ncclFloat32, ncclSum, c->comm,
                                      c->comm_stream));
                SS_NCCL(ReduceScatter(c->totals + q * W * B, rt, B, ncclFloat32, ncclSum, c->comm, c->comm_stream));
                SS_NCCL(GroupEnd());
                c->prof.launches[SS_K_COMBINE] += 1;
                c->prof.bytes[SS_K_COMBINE] += (double)(W - 1) * B * (D + 1) * 4; // sent per rank
                SS_CUDA(cudaEventRecord(c->ev_rs[buf], c->comm_stream));
                SS_CUDA(cudaStreamWaitEvent(s, c->ev_rs[buf], 0));
                src_s = rs;
                src_t = rt;
            } else {
                src_s = c->sums + q * B * D; // one rank: its own partial is the combined one
                src_t = c->totals + q * B;
            }
            float* dr = out_on_device ? rows_out + q * B * D : c->rs_stage.as<float>();
            float* dc = out_on_device ? coverage_out + q * B : c->rs_stage.as<float>() + B * D;
            {
                Scope sc(c, s, SS_K_NORMALIZE);
                own_launch(c, launch_normalize(src_s, src_t, B, (uint32_t)D, dr, dc,
                                               c->counters.as<unsigned long long>() + 3, s),
                           SS_K_NORMALIZE);
                c->prof.bytes[SS_K_NORMALIZE] += (double)B * (4.0 * D + 8.0);
            }
            if (!out_on_device) { // synchronous: the staging buffer is reused next round
                copy_d2h_pageable(c, rows_out + q * B * D, dr, B * D * 4, s);
                copy_d2h_pageable(c, coverage_out + q * B, dc, B * 4, s);
            }
            if (collective) SS_CUDA(cudaEventRecord(c->ev_norm[buf], s));
        }
    });
}

// ---------------------------------------------------------- instrumentation
int ss_profile_enable(ss_ctx* c, int on) {
    return guarded([&] {
        set_device(c);
        if (!on) profile_drain(c);
        c->prof.on = on != 0;
    });
}

int ss_profile_reset(ss_ctx* c) {
    return guarded([&] {
        set_device(c);
        profile_drain(c);
        for (int i = 0; i < SS_K_COUNT; ++i) {
            c->prof.ms[i] = 0;
            c->prof.launches[i] = 0;
            c->prof.bytes[i] = 0;
        }
        c->launches_own = c->launches_cub = 0;
        c->cnt_vis = c->cnt_inst = c->cnt_views = 0;
        for (auto& v : c->qstat) v = 0;
        SS_CUDA(cudaMemsetAsync(c->counters.p, 0, c->counters.bytes, c->stream));
    });
}

int ss_profile_read(ss_ctx* c, double* ms, uint64_t* launches, double* bytes) {
    return guarded([&] {
        set_device(c);
        profile_drain(c);
        // fold the device-side counters into raster / contract / normalize bytes:
        // K_v pairs (one 4 B scalar each, written by the compositor, read and
        // cleared by the contraction; fixed-point scalars are 8 B), rows read and written by the
        // contraction (once per group: the union of the members' touched
        // sets), covered rows whose sums normalize reads
        unsigned long long h[4];
        SS_CUDA(cudaMemcpy(h, c->counters.p, 32, cudaMemcpyDeviceToHost));
        const double kv = (double)h[1], rows = (double)h[2], covered = (double)h[3];
        for (int i = 0; i < SS_K_COUNT; ++i) {
            if (ms) ms[i] = c->prof.ms[i];
            if (launches) launches[i] = c->prof.launches[i];
            if (bytes) bytes[i] = c->prof.bytes[i];
        }
        if (bytes) {
            const double D = c->dim ? c->dim : 512;
            const double sb = c->deterministic ? 8.0 : 4.0;
            bytes[SS_K_RASTER] += 2.0 * sb * kv;
            bytes[SS_K_CONTRACT] += 2.0 * sb * kv + rows * (8.0 * D + 8.0);
            bytes[SS_K_NORMALIZE] += covered * 4.0 * D;
        }
    });
}

int ss_counters_read(ss_ctx* c, uint64_t* out5) {
    return guarded([&] {
        set_device(c);
        SS_CUDA(cudaStreamSynchronize(c->stream));
        unsigned long long h[4];
        SS_CUDA(cudaMemcpy(h, c->counters.p, 32, cudaMemcpyDeviceToHost));
        const uint64_t gv = h[0], kv = h[1];
        out5[0] = c->cnt_vis;
        out5[1] = c->cnt_inst;
        out5[2] = gv;
        out5[3] = kv;
        out5[4] = c->cnt_views;
    });
}

int ss_query_stats(ss_ctx* c, uint64_t* out4) {
    return guarded([&] {
        if (!c) throw Error(SS_ERR_CONTRACT, "ctx is null");
        for (int i = 0; i < 4; ++i) out4[i] = c->qstat[i];
    });
}

int ss_probe_fp64_rate(ss_ctx* c, double* lane_ops_per_s) {
    return guarded([&] {
        if (!c || !lane_ops_per_s) throw Error(SS_ERR_CONTRACT, "ctx or output is null");
        set_device(c);
        SS_CUDA(ss::probe_fp64_rate(lane_ops_per_s));
    });
}

int ss_launch_count(ss_ctx* c, uint64_t* own, uint64_t* cub) {
    if (own) *own = c->launches_own;
    if (cub) *cub = c->launches_cub;
    return 0;
}

} // extern "C"
