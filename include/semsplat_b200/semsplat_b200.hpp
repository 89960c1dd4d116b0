// semsplat_b200.hpp -- C++ drop-in for the reference's embedding path.
//
// Include AFTER the reference's own headers (semsplat/pipeline.hpp,
// semsplat/vecstore.hpp); link libsemsplat_b200.so.  Every function keeps the
// reference's signature, argument meaning and exception behaviour, so a caller
// switches by qualifying the call with semsplat::b200:::
//
//   semsplat::encode_scene(...)            pipeline.hpp:280   -> b200::encode_scene
//   semsplat::rasterize_weights_only(...)  rasterizer.hpp:268 -> b200::rasterize_weights_only
//   semsplat::rasterize(...)               rasterizer.hpp:261 -> b200::rasterize
//   semsplat::project_gaussian(...)        projection.hpp:33  -> b200::project_all (batch)
//   semsplat::build_store(...)             vecstore.hpp:88    -> b200::build_store
//   semsplat::query_topk(...)              vecstore.hpp:121   -> b200::query_topk
//   semsplat::query_threshold(...)         vecstore.hpp:135   -> b200::query_threshold
//   semsplat::run_query(...)               query.hpp:102     -> b200::run_query
//   semsplat::partition_store(...)        vecstore.hpp:169   -> b200::partition_store (device grouping)
//   (device store -> host VectorStore for snapshots / select_partitions: b200::fetch_store)
//
// All compute runs in the sm_100a kernels behind the C ABI
// (include/semsplat_b200.h); this header only marshals the reference's types.
#pragma once

#include <atomic>
#include <cstring>
#include <future>
#include <memory>
#include <optional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>
#ifdef __linux__
#include <sys/mman.h>
#endif

#include "../semsplat_b200.h"
#include "semsplat/pipeline.hpp"
#include "semsplat/providers.hpp"
#include "semsplat/query.hpp"
#include "semsplat/vecstore.hpp"

namespace semsplat {
namespace b200 {

// ss_status -> the reference's exception taxonomy (core.hpp:14-57)
[[noreturn]] inline void raise_status(int st) {
    const std::string msg = ss_last_error();
    switch (st) {
    case SS_ERR_CONTRACT: throw ContractError(msg);
    case SS_ERR_DATA: throw DataError(msg);
    case SS_ERR_NUMERIC: throw NumericError(msg);
    case SS_ERR_FORMAT: throw FormatError(msg);
    case SS_ERR_IO: throw IoError(msg);
    case SS_ERR_PIPELINE: throw PipelineError(msg, {msg}, false);
    default: throw std::runtime_error("libsemsplat_b200: " + msg);
    }
}
inline void check(int st) {
    if (st != SS_OK) raise_status(st);
}

// One context per device for the process (the reference is stateless; the
// device keeps the scene resident between calls).
class Device {
public:
    static Device& get(int device = 0) {
        static std::mutex mu;
        static std::vector<std::unique_ptr<Device>> devs;
        std::lock_guard<std::mutex> lock(mu);
        if (devs.size() <= static_cast<size_t>(device)) devs.resize(device + 1);
        if (!devs[device]) devs[device].reset(new Device(device));
        return *devs[device];
    }
    ss_ctx* ctx() { return ctx_; }
    int device() const { return device_; }
    std::mutex& mutex() { return mu_; }
    // Content key of a scene: size plus a 64-bit mix of every Gaussian's
    // fields (a caller may reuse the same storage for another scene, so the
    // address alone is not a key).
    static uint64_t scene_key(const GaussianScene& scene) {
        uint64_t h = 0x9e3779b97f4a7c15ull ^ scene.size();
        for (size_t k = 0; k < scene.size(); ++k) {
            const Gaussian3D& g = scene[k];
            const float f[11] = {g.mean[0], g.mean[1], g.mean[2], g.scale[0], g.scale[1], g.scale[2],
                                 g.rotation.x(), g.rotation.y(), g.rotation.z(), g.rotation.w(), g.opacity};
            for (float v : f) {
                uint32_t b;
                std::memcpy(&b, &v, 4);
                h = (h ^ b) * 0x100000001b3ull;
                h ^= h >> 29;
            }
        }
        return h;
    }
    // Upload the scene unless this device already holds it (same content
    // key): per-view calls (eval.hpp:94, fixture.hpp:157) do not re-upload
    // and re-derive the 3-D covariances of an unchanged scene.
    void bind(const GaussianScene& scene) {
        const uint64_t key = scene_key(scene);
        if (bound_ && key == key_) return;
        upload(scene);
        bound_ = true;
        key_ = key;
        color_bound_ = false;
    }
    void upload(const GaussianScene& scene) {
        const size_t n = scene.size();
        std::vector<float> mean(3 * n), scale(3 * n), quat(4 * n), op(n);
        for (size_t k = 0; k < n; ++k) {
            const Gaussian3D& g = scene[k];
            for (int i = 0; i < 3; ++i) {
                mean[3 * k + i] = g.mean[i];
                scale[3 * k + i] = g.scale[i];
            }
            quat[4 * k + 0] = g.rotation.x();
            quat[4 * k + 1] = g.rotation.y();
            quat[4 * k + 2] = g.rotation.z();
            quat[4 * k + 3] = g.rotation.w();
            op[k] = g.opacity;
        }
        check(ss_scene_set(ctx_, mean.data(), scale.data(), quat.data(), op.data(), n));
    }
    // Colors for rasterize (scene.hpp:28), after bind().
    void bind_color(const GaussianScene& scene) {
        if (color_bound_) return;
        const size_t n = scene.size();
        std::vector<float> rgb(3 * n);
        for (size_t k = 0; k < n; ++k)
            for (int i = 0; i < 3; ++i) rgb[3 * k + i] = scene[k].color[i];
        check(ss_scene_set_color(ctx_, rgb.data(), n));
        color_bound_ = true;
    }
    ~Device() { ss_destroy(ctx_); }

private:
    explicit Device(int device) : device_(device) { check(ss_create(device, &ctx_)); }
    int device_ = 0;
    ss_ctx* ctx_ = nullptr;
    std::mutex mu_;
    bool bound_ = false, color_bound_ = false;
    uint64_t key_ = 0;
};

// Binds a scene to a device ahead of per-view calls (optional: every call
// binds, but a bound scene with an unchanged content key is not re-uploaded).
inline void bind_scene(const GaussianScene& scene, int device = 0) {
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    d.bind(scene);
}

inline int device_count() {
    int n = 0;
    check(ss_device_count(&n));
    return n;
}

// Devices 0..n-1 joined in one NCCL communicator (ss_comm_init_all), created
// once per device count and kept for the process.
inline void ensure_group(int n) {
    static std::mutex mu;
    static int joined = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (joined == n) return;
    std::vector<ss_ctx*> ctxs;
    for (int d = 0; d < n; ++d) ctxs.push_back(Device::get(d).ctx());
    check(ss_comm_init_all(ctxs.data(), n));
    joined = n;
}

inline ss_camera to_c(const CameraPose& cam) {
    ss_camera c{};
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.R[3 * i + j] = cam.rotation(i, j);
    for (int i = 0; i < 3; ++i) c.t[i] = cam.translation[i];
    c.width = cam.width;
    c.height = cam.height;
    c.image_id = cam.image_id;
    return c;
}

// rasterizer.hpp:268-271
inline WeightMap rasterize_weights_only(const GaussianScene& scene, const CameraPose& cam,
                                        WeightMode mode = WeightMode::kAlphaComposited, int device = 0) {
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    d.bind(scene);
    const ss_camera c = to_c(cam);
    uint64_t ne = 0, ns = 0, ni = 0;
    check(ss_raster_capture(d.ctx(), &c, mode == WeightMode::kFalloffOnly ? SS_FALLOFF_ONLY : SS_ALPHA_COMPOSITED, &ne,
                            &ns, &ni));
    WeightMap wm;
    wm.image_id = cam.image_id;
    wm.width = cam.width;
    wm.height = cam.height;
    std::vector<ss_weight_entry> e(ne);
    wm.per_pixel_total.assign(static_cast<size_t>(cam.width) * cam.height, 0.0f);
    check(ss_raster_fetch(d.ctx(), e.data(), wm.per_pixel_total.data(), nullptr, nullptr, nullptr, nullptr));
    wm.entries.resize(ne);
    for (size_t i = 0; i < ne; ++i) wm.entries[i] = {e[i].gaussian_id, e[i].pixel, e[i].weight};
    return wm;
}

// rasterizer.hpp:261-264: image, WeightMap and alpha, bit-identical to the
// reference's RenderResult
inline RenderResult rasterize(const GaussianScene& scene, const CameraPose& cam,
                              WeightMode mode = WeightMode::kAlphaComposited, int device = 0) {
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    d.bind(scene);
    d.bind_color(scene);
    const ss_camera c = to_c(cam);
    uint64_t ne = 0, ns = 0, ni = 0;
    check(ss_render(d.ctx(), &c, mode == WeightMode::kFalloffOnly ? SS_FALLOFF_ONLY : SS_ALPHA_COMPOSITED, &ne, &ns,
                    &ni));
    RenderResult out;
    out.image = ImageRGB(cam.image_id, cam.width, cam.height);
    out.weights.image_id = cam.image_id;
    out.weights.width = cam.width;
    out.weights.height = cam.height;
    const size_t P = static_cast<size_t>(cam.width) * cam.height;
    out.weights.per_pixel_total.assign(P, 0.0f);
    out.alpha.assign(P, 0.0f);
    std::vector<ss_weight_entry> e(ne);
    check(ss_raster_fetch(d.ctx(), e.data(), out.weights.per_pixel_total.data(), out.alpha.data(), nullptr, nullptr,
                          nullptr));
    check(ss_render_fetch_image(d.ctx(), out.image.pixels.data()));
    out.weights.entries.resize(ne);
    for (size_t i = 0; i < ne; ++i) out.weights.entries[i] = {e[i].gaussian_id, e[i].pixel, e[i].weight};
    return out;
}

// projection.hpp:33-55 for every Gaussian of the scene
inline std::vector<Projected2D> project_all(const GaussianScene& scene, const CameraPose& cam, int device = 0) {
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    d.bind(scene);
    const ss_camera c = to_c(cam);
    std::vector<ss_projected> raw(scene.size());
    check(ss_project(d.ctx(), &c, raw.data()));
    std::vector<Projected2D> out(raw.size());
    for (size_t k = 0; k < raw.size(); ++k) {
        out[k].gaussian_id = raw[k].gaussian_id;
        out[k].visible = raw[k].visible != 0;
        out[k].mu2d = Eigen::Vector2d(raw[k].mu_x, raw[k].mu_y);
        out[k].cov_xx = raw[k].cov_xx;
        out[k].cov_xy = raw[k].cov_xy;
        out[k].cov_yy = raw[k].cov_yy;
        out[k].depth = raw[k].depth;
    }
    return out;
}

namespace detail {
// EmbeddingTable(n, dim) with its row storage on 2 MB pages where the kernel
// allows it (THP "madvise" mode): the 4 GB c4 table is then zero-filled at
// memset speed instead of taking a million 4 KB page faults (1.7 s measured).
// Same object as the reference's constructor builds.
inline EmbeddingTable make_table(uint64_t n, uint32_t dim) {
    EmbeddingTable t;
    t.gaussian_count = n;
    t.dim = dim;
    t.embeddings.reserve(n * dim);
#ifdef __linux__
    constexpr uintptr_t kHuge = uintptr_t(2) << 20;
    const uintptr_t b = reinterpret_cast<uintptr_t>(t.embeddings.data()), e = b + n * dim * sizeof(float);
    const uintptr_t a = (b + kHuge - 1) & ~(kHuge - 1);
    if (e > a + kHuge) madvise(reinterpret_cast<void*>(a), (e - a) & ~(kHuge - 1), MADV_HUGEPAGE);
#endif
    t.embeddings.resize(n * dim, 0.0f);
    t.coverage.assign(n, 0.0f);
    return t;
}

// One view's masks in their on-disk encoding (RLE runs, no bitmap decode on
// the host) and CLIP vectors, read as load_maskset / load_mask_embeddings do.
struct ViewData {
    std::vector<uint32_t> runs;
    std::vector<uint64_t> offs;
    std::vector<float> clip;
};

inline ViewData read_view(const DatasetManifest& manifest, const ImageEntry& entry) {
    const std::string path = manifest.resolve(entry.mask_path);
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open mask file: " + path);
    if (semsplat::detail::read_le<uint32_t>(is) != kMaskFileMagic) throw FormatError("bad mask file magic: " + path);
    const uint32_t mw = semsplat::detail::read_le<uint32_t>(is), mh = semsplat::detail::read_le<uint32_t>(is);
    const uint32_t count = semsplat::detail::read_le<uint32_t>(is);
    if (mw != manifest.mask_width || mh != manifest.mask_height)
        throw DataError("mask of image " + std::to_string(entry.image_id) +
                        " does not match the manifest mask resolution");
    std::vector<std::pair<uint32_t, std::vector<uint32_t>>> masks(count);
    for (auto& m : masks) {
        m.first = semsplat::detail::read_le<uint32_t>(is);
        const uint64_t nr = semsplat::detail::read_le<uint64_t>(is);
        m.second.resize(nr);
        for (auto& r : m.second) r = semsplat::detail::read_le<uint32_t>(is);
    }
    std::sort(masks.begin(), masks.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    ViewData vd;
    vd.offs.push_back(0);
    for (auto& m : masks) {
        vd.runs.insert(vd.runs.end(), m.second.begin(), m.second.end());
        vd.offs.push_back(vd.runs.size());
    }
    const std::vector<MaskEmbedding> emb = load_mask_embeddings(manifest, entry.image_id, count);
    vd.clip.resize(static_cast<size_t>(count) * manifest.embedding_dim);
    for (uint32_t j = 0; j < count; ++j)
        std::memcpy(vd.clip.data() + static_cast<size_t>(j) * manifest.embedding_dim, emb[j].vector.data(),
                    manifest.embedding_dim * sizeof(float));
    return vd;
}
} // namespace detail

// SS_OPT_DETERMINISTIC for encode_scene: fixed-point per-(Gaussian, mask)
// scalars, so the table is bitwise identical run to run (the reference's
// contract for a fixed worker count, pipeline.hpp:272-279) at ~4-5 % of c4
// throughput.  Off by default (f32 atomics: last-bit differences between
// runs, inside the path's tolerance).
inline std::atomic<bool>& deterministic_flag() {
    static std::atomic<bool> f{false};
    return f;
}
inline void set_deterministic(bool on) { deterministic_flag() = on; }

// pipeline.hpp:280-470.  Workers map to GPUs: with G = min(workers, visible
// devices) devices, worker w (the reference's view-to-worker assignment,
// round-robin or contiguous) runs on device w mod G, each device on its own
// host thread with its own fp32 partial; for G > 1 the partials are combined
// by one NCCL reduce-scatter per chunk of chunk_rows rows per device
// (SS_OPT_COMBINE_ROWS; the reference's phase-2 chunks, pipeline.hpp:396-402)
// and each device normalises the rows it receives (ss_encode_combine).  Per-
// image failures stop their worker (pipeline.hpp:350-351); with several
// workers they surface as PipelineError with one status line per worker,
// naming its GPU.  `device` is the device of a single-GPU run.
inline EmbeddingTable encode_scene(const GaussianScene& scene, const DatasetManifest& manifest, uint32_t workers,
                                   uint64_t chunk_rows, const EncodeOptions& options = {},
                                   EncodeStats* stats_out = nullptr, int device = 0) {
    if (workers < 1) throw ContractError("encode_scene: workers must be >= 1");
    if (manifest.raster_width == 0 || manifest.raster_height == 0)
        throw DataError("encode_scene: manifest has no raster resolution");
    const std::vector<CameraPose> cameras = load_cameras(manifest.resolve(manifest.camera_file));
    std::unordered_map<uint32_t, const CameraPose*> camera_by_id;
    for (const CameraPose& c : cameras) camera_by_id[c.image_id] = &c;
    for (const ImageEntry& e : manifest.images)
        if (!camera_by_id.count(e.camera_id))
            throw DataError("image " + std::to_string(e.image_id) + ": no camera with id " +
                            std::to_string(e.camera_id));

    // the host table (4.1 GB at c4, zero-filled by its constructor) is built
    // while the devices run phase 1
    const uint64_t n = scene.size();
    std::optional<EmbeddingTable> table_slot;
    std::thread table_thread([&] { table_slot.emplace(detail::make_table(n, manifest.embedding_dim)); });
    struct JoinTable {
        std::thread& t;
        ~JoinTable() {
            if (t.joinable()) t.join();
        }
    } join_table{table_thread};
    const int G = workers > 1 ? std::max(1, std::min<int>((int)workers, device_count())) : 1;
    std::vector<Device*> devs;
    for (int g = 0; g < G; ++g) devs.push_back(&Device::get(G == 1 ? device : g));
    std::vector<std::unique_lock<std::mutex>> locks;
    for (Device* d : devs) locks.emplace_back(d->mutex());
    if (G > 1) ensure_group(G);
    for (Device* d : devs) {
        d->bind(scene);
        check(ss_set_option(d->ctx(), SS_OPT_COMBINE_ROWS, G > 1 ? (int64_t)chunk_rows : 0));
        check(ss_set_option(d->ctx(), SS_OPT_DETERMINISTIC, deterministic_flag() ? 1 : 0));
        check(ss_encode_begin(d->ctx(), manifest.embedding_dim, nullptr, nullptr));
    }
    const auto t0 = std::chrono::steady_clock::now();
    const size_t n_img = manifest.images.size();
    const size_t block = (n_img + workers - 1) / workers;
    std::vector<std::string> failures(workers);
    std::vector<size_t> worker_images(workers, 0);
    std::vector<double> worker_seconds(workers, 0.0);
    std::vector<size_t> worker_entries(workers, 0);
    const ss_weight_mode wmode = options.mode == WeightMode::kFalloffOnly ? SS_FALLOFF_ONLY : SS_ALPHA_COMPOSITED;

    // one batch of a worker's views read from disk (camera scaled to the raster
    // resolution, RLE runs, CLIP rows); `failure` names the image that stopped it
    struct Batch {
        std::vector<detail::ViewData> data;
        std::vector<ss_camera> cams;
        std::string failure;
        size_t next = 0; // manifest index to continue from
    };
    constexpr size_t kBatchViews = 48;
    auto read_batch = [&](uint32_t rank, size_t from) {
        Batch b;
        size_t idx = from;
        for (; idx < n_img && b.cams.size() < kBatchViews; ++idx) {
            const bool mine = options.contiguous_batching ? (idx / block == rank) : (idx % workers == rank);
            if (!mine) continue;
            const ImageEntry& entry = manifest.images[idx];
            try {
                const CameraPose raster_cam = camera_scaled_to(*camera_by_id.at(entry.camera_id),
                                                               manifest.raster_width, manifest.raster_height);
                b.data.push_back(detail::read_view(manifest, entry));
                ss_camera c = to_c(raster_cam);
                c.image_id = entry.image_id;
                b.cams.push_back(c);
            } catch (const std::exception& ex) {
                std::string m = ex.what();
                const std::string pre = "image " + std::to_string(entry.image_id) + ":";
                if (m.rfind(pre, 0) != 0) m = "image " + std::to_string(entry.image_id) + ": " + m;
                b.failure = m;
                break;
            }
        }
        b.next = idx;
        return b;
    };
    auto run_worker = [&](uint32_t rank, ss_ctx* ctx) {
        const auto ts = std::chrono::steady_clock::now();
        // the worker's views go to its device batch by batch (views overlap in
        // the device's pipeline lanes) while the next batch is read from disk;
        // host-side decoding errors stop the worker at that image, as the
        // reference's worker_body does
        uint64_t before[5] = {}, after[5] = {};
        check(ss_counters_read(ctx, before));
        size_t images = 0;
        std::future<Batch> next = std::async(std::launch::async, read_batch, rank, size_t(0));
        for (;;) {
            Batch cur = next.get();
            const bool more = cur.failure.empty() && cur.next < n_img;
            if (more) next = std::async(std::launch::async, read_batch, rank, cur.next);
            std::vector<ss_view_masks> vms(cur.data.size());
            for (size_t v = 0; v < cur.data.size(); ++v) {
                vms[v] = ss_view_masks{};
                vms[v].n_masks = static_cast<uint32_t>(cur.data[v].offs.size() - 1);
                vms[v].mask_width = manifest.mask_width;
                vms[v].mask_height = manifest.mask_height;
                vms[v].flags = 0;
                vms[v].runs = cur.data[v].runs.data();
                vms[v].run_offsets = cur.data[v].offs.data();
                vms[v].clip = cur.data[v].clip.data();
                vms[v].n_runs = cur.data[v].runs.size();
            }
            if (!cur.cams.empty()) {
                const int st = ss_encode_views(ctx, static_cast<uint32_t>(cur.cams.size()), cur.cams.data(), vms.data(),
                                               wmode);
                if (st != SS_OK) {
                    if (failures[rank].empty()) failures[rank] = ss_last_error(); // names the image
                    if (more) next.wait();
                    break;
                }
            }
            images += cur.cams.size();
            if (!cur.failure.empty()) {
                failures[rank] = cur.failure;
                break;
            }
            if (!more) break;
        }
        check(ss_counters_read(ctx, after));
        worker_images[rank] = images;
        worker_entries[rank] = static_cast<size_t>(after[3] - before[3]); // masked-weight (gid, mask) entries
        worker_seconds[rank] = std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
    };
    // one host thread per device, its workers in rank order
    std::vector<std::string> device_errors(G);
    auto run_device = [&](int g) {
        try {
            for (uint32_t w = (uint32_t)g; w < workers; w += (uint32_t)G) run_worker(w, devs[g]->ctx());
        } catch (const std::exception& ex) {
            device_errors[g] = ex.what();
        }
    };
    if (G == 1) {
        run_device(0);
    } else {
        std::vector<std::thread> threads;
        for (int g = 0; g < G; ++g) threads.emplace_back(run_device, g);
        for (auto& t : threads) t.join();
    }
    for (int g = 0; g < G; ++g)
        if (!device_errors[g].empty()) throw std::runtime_error("libsemsplat_b200: gpu " + std::to_string(g) + ": " +
                                                                device_errors[g]);
    bool failed = false;
    for (const auto& f : failures) failed |= !f.empty();
    if (failed) {
        if (workers == 1) throw DataError(failures[0]);
        std::vector<std::string> status;
        for (uint32_t r = 0; r < workers; ++r)
            status.push_back("worker " + std::to_string(r) + " (gpu " + std::to_string(G == 1 ? device : (int)(r % G)) +
                             "): " + (failures[r].empty() ? "ok" : failures[r]));
        throw PipelineError("scene encoding failed", std::move(status), true);
    }
    for (Device* d : devs) check(ss_synchronize(d->ctx()));
    const auto t1 = std::chrono::steady_clock::now();
    table_thread.join();
    EmbeddingTable& table = *table_slot;
    if (G == 1) {
        const uint64_t step = (chunk_rows == 0 || chunk_rows > n) ? std::max<uint64_t>(n, 1) : chunk_rows;
        for (uint64_t lo = 0; lo < n; lo += step) {
            const uint64_t hi = std::min<uint64_t>(n, lo + step);
            // the table is freshly zero-filled: only covered rows move
            check(ss_encode_finalize_sparse(devs[0]->ctx(), lo, hi, table.row(lo), table.coverage.data() + lo,
                                            nullptr));
        }
    } else {
        // combine_partials + finalize_into: every device reduce-scatters its
        // partial and normalises the rows it receives (block-cyclic rounds)
        std::vector<std::string> errs(G);
        std::vector<std::thread> threads;
        for (int g = 0; g < G; ++g)
            threads.emplace_back([&, g] {
                ss_ctx* ctx = devs[g]->ctx();
                uint64_t rows_alloc = 0, blk = 0, rounds = 0, rank_rows = 0;
                if (ss_combine_layout(ctx, &rows_alloc, &blk, &rounds, &rank_rows) != SS_OK) {
                    errs[g] = ss_last_error();
                    return;
                }
                std::vector<float> rows(rank_rows * manifest.embedding_dim), cov(rank_rows);
                if (ss_encode_combine(ctx, rows.data(), cov.data(), 0) != SS_OK) {
                    errs[g] = ss_last_error();
                    return;
                }
                for (uint64_t q = 0; q < rounds; ++q)
                    for (uint64_t i = 0; i < blk; ++i) {
                        const uint64_t row = q * (uint64_t)G * blk + (uint64_t)g * blk + i, at = q * blk + i;
                        if (row >= n) break;
                        std::memcpy(table.row(row), rows.data() + at * manifest.embedding_dim,
                                    manifest.embedding_dim * sizeof(float));
                        table.coverage[row] = cov[at];
                    }
            });
        for (auto& t : threads) t.join();
        for (int g = 0; g < G; ++g)
            if (!errs[g].empty()) throw std::runtime_error("libsemsplat_b200: gpu " + std::to_string(g) + ": " + errs[g]);
    }
    if (stats_out) {
        stats_out->phase1_seconds = std::chrono::duration<double>(t1 - t0).count();
        stats_out->phase2_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        stats_out->worker_seconds = worker_seconds;
        stats_out->worker_images = worker_images;
        stats_out->worker_entries = worker_entries;
    }
    return std::move(table);
}

// A device-resident VectorStore: ids + unit rows on the device; the records'
// payloads (the scene's Gaussians, in the store's record order) on the host.
struct DeviceStore {
    int device = 0;
    uint64_t count = 0;
    uint32_t dim = 0;
    std::vector<uint32_t> ids;          // record order (= device order)
    std::vector<Gaussian3D> payloads;   // record order
};

// vecstore.hpp:88-103
inline DeviceStore build_store(const EmbeddingTable& table, const GaussianScene& scene, int device = 0) {
    if (table.gaussian_count != scene.size()) throw ContractError("build_store: table rows and scene size differ");
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    uint64_t cnt = 0;
    check(ss_store_build(d.ctx(), table.embeddings.data(), table.coverage.data(), table.gaussian_count, table.dim,
                         &cnt));
    DeviceStore st{device, cnt, table.dim, {}, {}};
    st.ids.resize(cnt);
    if (cnt) check(ss_store_fetch(d.ctx(), st.ids.data(), nullptr));
    st.payloads.reserve(cnt);
    for (uint32_t id : st.ids) st.payloads.push_back(scene[id]);
    return st;
}

inline DeviceStore upload_store(const VectorStore& store, int device = 0) {
    Device& d = Device::get(device);
    std::lock_guard<std::mutex> lock(d.mutex());
    std::vector<float> rows(store.count() * store.dim());
    for (size_t i = 0; i < store.count(); ++i)
        std::memcpy(rows.data() + i * store.dim(), store.vector_at(i), store.dim() * sizeof(float));
    check(ss_store_set(d.ctx(), store.ids().data(), rows.data(), store.count(), store.dim()));
    DeviceStore st{device, store.count(), store.dim(), store.ids(), {}};
    st.payloads.reserve(store.count());
    for (size_t i = 0; i < store.count(); ++i) st.payloads.push_back(store.payload_at(i));
    return st;
}

// The device store as the reference's host VectorStore (ids, unit rows,
// payloads in record order), e.g. for partition_store / save_snapshot
// (vecstore.hpp:160-328), which run on the host in the reference too.
inline VectorStore fetch_store(const DeviceStore& store) {
    Device& d = Device::get(store.device);
    std::lock_guard<std::mutex> lock(d.mutex());
    std::vector<uint32_t> ids(store.count);
    std::vector<float> rows(store.count * store.dim);
    if (store.count) check(ss_store_fetch(d.ctx(), ids.data(), rows.data()));
    VectorStore out(store.dim);
    out.reserve(store.count);
    for (size_t i = 0; i < store.count; ++i)
        out.add_record(ids[i], std::vector<float>(rows.begin() + i * store.dim, rows.begin() + (i + 1) * store.dim),
                       store.payloads.size() == store.count ? store.payloads[i] : Gaussian3D{});
    return out;
}

// vecstore.hpp:169-213: cell keys, the (x, y, z)-ordered grouping and the
// row gather run on the device; the snapshots are the reference's own types
// (bounds from the reference's f64 expressions on the device bbox.min).
inline std::vector<PartitionSnapshot> partition_store(const DeviceStore& store, double cell_size) {
    if (!(cell_size > 0)) throw ContractError("partition_store: cell_size must be positive");
    if (store.count == 0) return {};
    if (store.payloads.size() != store.count) throw ContractError("partition_store: the store has no payloads");
    std::vector<float> means(3 * store.count);
    for (size_t i = 0; i < store.count; ++i)
        for (int a = 0; a < 3; ++a) means[3 * i + a] = store.payloads[i].mean[a];
    Device& d = Device::get(store.device);
    std::lock_guard<std::mutex> lock(d.mutex());
    uint64_t nc = 0;
    check(ss_store_partition(d.ctx(), means.data(), cell_size, &nc));
    std::vector<int32_t> cells(3 * nc);
    std::vector<uint64_t> offs(nc + 1);
    std::vector<uint32_t> order(store.count), ids(store.count);
    std::vector<float> rows(store.count * store.dim);
    double bmin[3];
    check(ss_store_partition_fetch(d.ctx(), cells.data(), offs.data(), order.data(), ids.data(), rows.data(), bmin));
    Aabb bbox;
    bbox.min = Eigen::Vector3d(bmin[0], bmin[1], bmin[2]);
    std::vector<PartitionSnapshot> snapshots;
    snapshots.reserve(nc);
    for (uint64_t c = 0; c < nc; ++c) {
        PartitionSnapshot snap;
        const int32_t kx = cells[3 * c], ky = cells[3 * c + 1], kz = cells[3 * c + 2];
        snap.cell = {kx, ky, kz};
        snap.bounds.min = bbox.min + cell_size * Eigen::Vector3d(kx, ky, kz);
        snap.bounds.max = bbox.min + cell_size * Eigen::Vector3d(kx + 1, ky + 1, kz + 1);
        snap.store = VectorStore(store.dim);
        snap.store.reserve(offs[c + 1] - offs[c]);
        for (uint64_t j = offs[c]; j < offs[c + 1]; ++j)
            snap.store.add_record(ids[j],
                                  std::vector<float>(rows.begin() + j * store.dim, rows.begin() + (j + 1) * store.dim),
                                  store.payloads[order[j]]);
        snapshots.push_back(std::move(snap));
    }
    return snapshots;
}

// vecstore.hpp:121-132
inline std::vector<ScoredId> query_topk(const DeviceStore& store, const std::vector<float>& q, size_t k) {
    if (k == 0 || store.count == 0) return {};
    if (q.size() != store.dim) throw ContractError("query dimension differs from store dimension");
    Device& d = Device::get(store.device);
    std::lock_guard<std::mutex> lock(d.mutex());
    std::vector<uint32_t> ids(k);
    std::vector<float> sims(k);
    uint64_t cnt = 0;
    check(ss_query_topk(d.ctx(), q.data(), 1, static_cast<uint32_t>(k), ids.data(), sims.data(), &cnt));
    std::vector<ScoredId> out(cnt);
    for (size_t i = 0; i < cnt; ++i) out[i] = {ids[i], sims[i]};
    return out;
}

// vecstore.hpp:135-146
inline std::vector<ScoredId> query_threshold(const DeviceStore& store, const std::vector<float>& q, float tau) {
    if (!(tau >= -1.0f && tau <= 1.0f)) throw ContractError("cosine threshold must lie in [-1, 1]");
    if (store.count == 0) return {};
    if (q.size() != store.dim) throw ContractError("query dimension differs from store dimension");
    Device& d = Device::get(store.device);
    std::lock_guard<std::mutex> lock(d.mutex());
    std::vector<uint32_t> ids(store.count);
    std::vector<float> sims(store.count);
    uint64_t cnt = 0;
    check(ss_query_threshold(d.ctx(), q.data(), tau, ids.data(), sims.data(), store.count, &cnt));
    std::vector<ScoredId> out(cnt);
    for (size_t i = 0; i < cnt; ++i) out[i] = {ids[i], sims[i]};
    return out;
}

// Batched query_topk: row q of the result is query_topk(store, queries[q], k)
// (the device answers the whole batch in one pass).
inline std::vector<std::vector<ScoredId>> query_topk_batch(const DeviceStore& store,
                                                           const std::vector<std::vector<float>>& queries, size_t k) {
    std::vector<std::vector<ScoredId>> out(queries.size());
    if (k == 0 || store.count == 0 || queries.empty()) return out;
    std::vector<float> q(queries.size() * store.dim);
    for (size_t i = 0; i < queries.size(); ++i) {
        if (queries[i].size() != store.dim) throw ContractError("query dimension differs from store dimension");
        std::memcpy(q.data() + i * store.dim, queries[i].data(), store.dim * sizeof(float));
    }
    Device& d = Device::get(store.device);
    std::lock_guard<std::mutex> lock(d.mutex());
    std::vector<uint32_t> ids(queries.size() * k);
    std::vector<float> sims(queries.size() * k);
    std::vector<uint64_t> cnt(queries.size());
    check(ss_query_topk(d.ctx(), q.data(), static_cast<uint32_t>(queries.size()), static_cast<uint32_t>(k), ids.data(),
                        sims.data(), cnt.data()));
    for (size_t i = 0; i < queries.size(); ++i) {
        out[i].resize(cnt[i]);
        for (size_t j = 0; j < cnt[i]; ++j) out[i][j] = {ids[i * k + j], sims[i * k + j]};
    }
    return out;
}

// query.hpp:102-122: encode_text + store search + payload assembly.
inline QueryResult run_query(const DeviceStore& store, const std::string& text, const QueryMode& mode,
                             const TextProvider& provider) {
    QueryResult result;
    result.text = text;
    result.mode = mode;
    result.query_vector = encode_text(text, provider);
    std::vector<ScoredId> scored;
    if (store.count > 0)
        scored = (mode.kind == QueryMode::Kind::kTopK) ? query_topk(store, result.query_vector, mode.k)
                                                       : query_threshold(store, result.query_vector, mode.tau);
    std::unordered_map<uint32_t, size_t> index_by_id;
    index_by_id.reserve(store.ids.size());
    for (size_t i = 0; i < store.ids.size(); ++i) index_by_id[store.ids[i]] = i;
    result.matches.reserve(scored.size());
    for (const ScoredId& sc : scored)
        result.matches.push_back({sc.gaussian_id, sc.similarity, store.payloads.at(index_by_id.at(sc.gaussian_id))});
    return result;
}

} // namespace b200
} // namespace semsplat
