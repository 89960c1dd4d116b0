// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference headers
// (/root/reference/proj/include/semsplat/*.hpp, compiled against
// oracle/eigen_shim).  Built by oracle/build_oracle.py into
// oracle/_ref/libssref.so; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, as the checker
// and as the reference CPU arm.  It contains no algorithm of its own: every
// entry point forwards to the reference function named beside it.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "semsplat/core.hpp"
#include "semsplat/eval.hpp"
#include "semsplat/fixture.hpp"
#include "semsplat/pipeline.hpp"
#include "semsplat/projection.hpp"
#include "semsplat/providers.hpp"
#include "semsplat/rasterizer.hpp"
#include "semsplat/scene.hpp"
#include "semsplat/scene_io.hpp"
#include "semsplat/vecstore.hpp"

using namespace semsplat;

extern "C" {

struct ssref_camera {
    double fx, fy, cx, cy;
    double R[9]; // row-major world-to-camera
    double t[3];
    uint32_t width, height, image_id, pad;
};

struct ssref_projected {
    uint32_t gaussian_id;
    uint32_t visible;
    double mu_x, mu_y, cov_xx, cov_xy, cov_yy, depth;
};

struct ssref_entry {
    uint32_t gaussian_id;
    uint32_t pixel;
    float weight;
};
}

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        g_kind = 0;
        return 0;
    } catch (const ContractError& e) {
        g_err = e.what();
        g_kind = 1;
    } catch (const DataError& e) {
        g_err = e.what();
        g_kind = 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        g_kind = 3;
    } catch (const FormatError& e) {
        g_err = e.what();
        g_kind = 4;
    } catch (const IoError& e) {
        g_err = e.what();
        g_kind = 5;
    } catch (const PipelineError& e) {
        g_err = e.what();
        for (const auto& s : e.worker_status) g_err += "\n" + s;
        g_kind = 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = 7;
    }
    return g_kind;
}

GaussianScene make_scene(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity,
                         const float* color, uint64_t n) {
    std::vector<Gaussian3D> gs(n);
    for (uint64_t k = 0; k < n; ++k) {
        Gaussian3D& g = gs[k];
        g.mean = Eigen::Vector3f(mean[3 * k], mean[3 * k + 1], mean[3 * k + 2]);
        g.scale = Eigen::Vector3f(scale[3 * k], scale[3 * k + 1], scale[3 * k + 2]);
        g.rotation = Eigen::Quaternionf(quat_xyzw[4 * k + 3], quat_xyzw[4 * k], quat_xyzw[4 * k + 1],
                                        quat_xyzw[4 * k + 2]);
        g.opacity = opacity[k];
        if (color) g.color = Eigen::Vector3f(color[3 * k], color[3 * k + 1], color[3 * k + 2]);
    }
    return GaussianScene(std::move(gs));
}

CameraPose make_cam(const ssref_camera& c) {
    CameraPose cam;
    cam.image_id = c.image_id;
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.rotation << c.R[0], c.R[1], c.R[2], c.R[3], c.R[4], c.R[5], c.R[6], c.R[7], c.R[8];
    cam.translation = Eigen::Vector3d(c.t[0], c.t[1], c.t[2]);
    cam.width = c.width;
    cam.height = c.height;
    return cam;
}

void put_cam(const CameraPose& cam, ssref_camera* c) {
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->cx = cam.cx;
    c->cy = cam.cy;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c->R[3 * i + j] = cam.rotation(i, j);
    for (int i = 0; i < 3; ++i) c->t[i] = cam.translation[i];
    c->width = cam.width;
    c->height = cam.height;
    c->image_id = cam.image_id;
    c->pad = 0;
}

struct WeightMapHandle {
    WeightMap wm;
    std::vector<float> alpha;
    std::vector<float> image; // RenderResult::image.pixels (full_render)
};

} // namespace

extern "C" {

const char* ssref_last_error() { return g_err.c_str(); }
int ssref_last_error_kind() { return g_kind; }

// projection.hpp:33 project_gaussian (+ scene.hpp:33 covariance3d)
int ssref_project(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity, uint64_t n,
                  const ssref_camera* cam, ssref_projected* out) {
    return guarded([&] {
        const GaussianScene scene = make_scene(mean, scale, quat_xyzw, opacity, nullptr, n);
        const CameraPose c = make_cam(*cam);
        for (uint64_t k = 0; k < n; ++k) {
            const Projected2D p = project_gaussian(scene[k], c);
            out[k] = {p.gaussian_id, p.visible ? 1u : 0u, p.mu2d.x(), p.mu2d.y(), p.cov_xx, p.cov_xy, p.cov_yy,
                      p.depth};
        }
    });
}

// projection.hpp:59 depth_sort over the visible projections; returns ids in order.
int ssref_depth_order(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity, uint64_t n,
                      const ssref_camera* cam, uint32_t* ids_out, uint64_t* n_visible) {
    return guarded([&] {
        const GaussianScene scene = make_scene(mean, scale, quat_xyzw, opacity, nullptr, n);
        const CameraPose c = make_cam(*cam);
        std::vector<Projected2D> projected;
        for (const Gaussian3D& g : scene.gaussians()) {
            Projected2D p = project_gaussian(g, c);
            if (p.visible) projected.push_back(p);
        }
        depth_sort(projected);
        for (size_t i = 0; i < projected.size(); ++i) ids_out[i] = projected[i].gaussian_id;
        *n_visible = projected.size();
    });
}

// rasterizer.hpp:268 rasterize_weights_only (mode 0 = alpha-composited, 1 = falloff)
// or rasterizer.hpp:261 rasterize (want_alpha) -> handle
int ssref_rasterize(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity,
                    const float* color, uint64_t n, const ssref_camera* cam, int mode, int full_render,
                    void** handle, uint64_t* n_entries) {
    return guarded([&] {
        const GaussianScene scene = make_scene(mean, scale, quat_xyzw, opacity, color, n);
        const CameraPose c = make_cam(*cam);
        const WeightMode wmode = mode ? WeightMode::kFalloffOnly : WeightMode::kAlphaComposited;
        auto* h = new WeightMapHandle();
        if (full_render) {
            RenderResult r = rasterize(scene, c, wmode);
            h->wm = std::move(r.weights);
            h->alpha = std::move(r.alpha);
            h->image = std::move(r.image.pixels);
        } else {
            h->wm = rasterize_weights_only(scene, c, wmode);
        }
        *n_entries = h->wm.entries.size();
        *handle = h;
    });
}

void ssref_weightmap_fetch(void* handle, ssref_entry* entries, float* per_pixel_total, float* alpha) {
    auto* h = static_cast<WeightMapHandle*>(handle);
    for (size_t i = 0; i < h->wm.entries.size(); ++i)
        entries[i] = {h->wm.entries[i].gaussian_id, h->wm.entries[i].pixel, h->wm.entries[i].weight};
    if (per_pixel_total)
        std::memcpy(per_pixel_total, h->wm.per_pixel_total.data(), h->wm.per_pixel_total.size() * sizeof(float));
    if (alpha && !h->alpha.empty()) std::memcpy(alpha, h->alpha.data(), h->alpha.size() * sizeof(float));
}

// RenderResult::image pixels (3 x width x height floats) of a full_render handle
void ssref_image_fetch(void* handle, float* rgb) {
    auto* h = static_cast<WeightMapHandle*>(handle);
    if (rgb && !h->image.empty()) std::memcpy(rgb, h->image.data(), h->image.size() * sizeof(float));
}

void ssref_weightmap_free(void* handle) { delete static_cast<WeightMapHandle*>(handle); }

// eval.hpp:122-158 assign_classes on an EmbeddingTable (rows n x dim, coverage n)
int ssref_assign_classes(const float* rows, const float* coverage, uint64_t n, uint32_t dim, const int32_t* label_ids,
                         const float* label_vecs, uint32_t n_labels, int32_t* out) {
    return guarded([&] {
        EmbeddingTable table(n, dim);
        std::memcpy(table.embeddings.data(), rows, n * dim * sizeof(float));
        std::memcpy(table.coverage.data(), coverage, n * sizeof(float));
        std::vector<std::pair<int32_t, std::vector<float>>> labels;
        for (uint32_t c = 0; c < n_labels; ++c)
            labels.push_back({label_ids[c], std::vector<float>(label_vecs + (size_t)c * dim,
                                                               label_vecs + (size_t)(c + 1) * dim)});
        const std::vector<int32_t> cls = assign_classes(table, labels);
        std::memcpy(out, cls.data(), cls.size() * sizeof(int32_t));
    });
}

// pipeline.hpp:35 mask_weights on a WeightMap handle and a raster-resolution u8 bitmap.
// Outputs (gid, sum) pairs sorted by gid; caller provides capacity >= n_entries.
int ssref_mask_weights(void* handle, const uint8_t* bits, uint32_t width, uint32_t height, uint32_t* gids,
                       double* sums, uint64_t* count) {
    return guarded([&] {
        auto* h = static_cast<WeightMapHandle*>(handle);
        MaskBitmap bm(width, height);
        std::memcpy(bm.bits.data(), bits, static_cast<size_t>(width) * height);
        const MaskedWeights mw = mask_weights(h->wm, bm, 0, 0);
        for (size_t i = 0; i < mw.entries.size(); ++i) {
            gids[i] = mw.entries[i].first;
            sums[i] = mw.entries[i].second;
        }
        *count = mw.entries.size();
    });
}

// providers.hpp:359 resample_mask
int ssref_resample_mask(const uint8_t* bits, uint32_t w, uint32_t h, uint32_t tw, uint32_t th, uint8_t* out) {
    return guarded([&] {
        MaskBitmap bm(w, h);
        std::memcpy(bm.bits.data(), bits, static_cast<size_t>(w) * h);
        const MaskBitmap r = resample_mask(bm, tw, th);
        std::memcpy(out, r.bits.data(), static_cast<size_t>(tw) * th);
    });
}

// pipeline.hpp:280 encode_scene over a dataset on disk (manifest) with the
// scene given as arrays (the loaded scene both paths consume).
int ssref_encode(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity, uint64_t n,
                 const char* manifest_path, uint32_t workers, uint64_t chunk_rows, int mode, int contiguous,
                 float* embeddings_out, float* coverage_out, double* stats_out) {
    return guarded([&] {
        const GaussianScene scene = make_scene(mean, scale, quat_xyzw, opacity, nullptr, n);
        const DatasetManifest manifest = load_manifest(manifest_path);
        EncodeOptions opt;
        opt.mode = mode ? WeightMode::kFalloffOnly : WeightMode::kAlphaComposited;
        opt.contiguous_batching = contiguous != 0;
        EncodeStats stats;
        const EmbeddingTable table = encode_scene(scene, manifest, workers, chunk_rows, opt, &stats);
        std::memcpy(embeddings_out, table.embeddings.data(), table.embeddings.size() * sizeof(float));
        std::memcpy(coverage_out, table.coverage.data(), table.coverage.size() * sizeof(float));
        if (stats_out) {
            stats_out[0] = stats.phase1_seconds;
            stats_out[1] = stats.phase2_seconds;
            size_t entries = 0;
            for (size_t e : stats.worker_entries) entries += e;
            stats_out[2] = static_cast<double>(entries);
        }
    });
}

// scene_io.hpp:132 load_scene -> arrays (quat as x,y,z,w)
int ssref_load_scene_count(const char* path, uint64_t* n) {
    return guarded([&] { *n = load_scene(path).size(); });
}
int ssref_load_scene(const char* path, float* mean, float* scale, float* quat_xyzw, float* opacity, float* color) {
    return guarded([&] {
        const GaussianScene s = load_scene(path);
        for (size_t k = 0; k < s.size(); ++k) {
            const Gaussian3D& g = s[k];
            for (int i = 0; i < 3; ++i) {
                mean[3 * k + i] = g.mean[i];
                scale[3 * k + i] = g.scale[i];
                if (color) color[3 * k + i] = g.color[i];
            }
            quat_xyzw[4 * k + 0] = g.rotation.x();
            quat_xyzw[4 * k + 1] = g.rotation.y();
            quat_xyzw[4 * k + 2] = g.rotation.z();
            quat_xyzw[4 * k + 3] = g.rotation.w();
            opacity[k] = g.opacity;
        }
    });
}

// scene_io.hpp:203 save_scene from arrays
int ssref_save_scene(const char* path, const float* mean, const float* scale, const float* quat_xyzw,
                     const float* opacity, const float* color, uint64_t n) {
    return guarded([&] { save_scene(make_scene(mean, scale, quat_xyzw, opacity, color, n), path); });
}

// scene_io.hpp:217 load_cameras
int ssref_load_cameras(const char* path, ssref_camera* out, uint64_t capacity, uint64_t* n) {
    return guarded([&] {
        const std::vector<CameraPose> cams = load_cameras(path);
        *n = cams.size();
        for (size_t i = 0; i < cams.size() && i < capacity; ++i) put_cam(cams[i], &out[i]);
    });
}

// pipeline.hpp:196 camera_scaled_to
void ssref_camera_scaled_to(const ssref_camera* in, uint32_t w, uint32_t h, ssref_camera* out) {
    put_cam(camera_scaled_to(make_cam(*in), w, h), out);
}

// fixture.hpp:65 look_at
void ssref_look_at(const double* eye, const double* target, uint32_t w, uint32_t h, double focal,
                   ssref_camera* out) {
    put_cam(detail::look_at(Eigen::Vector3d(eye[0], eye[1], eye[2]), Eigen::Vector3d(target[0], target[1], target[2]),
                            w, h, focal),
            out);
}

// fixture.hpp:88/202 generate_fixture + write_fixture -> manifest path
int ssref_write_fixture(uint32_t objects, uint32_t per_object, uint32_t views, uint32_t resolution,
                        uint32_t mask_scale, uint32_t dim, uint64_t seed, const char* dir, char* manifest_out,
                        uint64_t cap) {
    return guarded([&] {
        FixtureSpec spec;
        spec.object_count = objects;
        spec.gaussians_per_object = per_object;
        spec.view_count = views;
        spec.resolution = resolution;
        spec.mask_scale = mask_scale;
        spec.embedding_dim = dim;
        spec.seed = seed;
        const SyntheticFixture fx = generate_fixture(spec);
        const std::string path = write_fixture(fx, dir);
        std::snprintf(manifest_out, cap, "%s", path.c_str());
    });
}

// providers.hpp:381 synth_embedding
int ssref_synth_embedding(const char* label, uint32_t dim, float* out) {
    return guarded([&] {
        const std::vector<float> v = synth_embedding(label, dim);
        std::memcpy(out, v.data(), dim * sizeof(float));
    });
}

// vecstore.hpp:21 dot_lanes
float ssref_dot_lanes(const float* a, const float* b, uint64_t n) { return dot_lanes(a, b, n); }

// vecstore.hpp:34 normalized_copy
int ssref_normalized_copy(const float* v, uint64_t n, float* out) {
    return guarded([&] {
        const std::vector<float> r = normalized_copy(v, n);
        std::memcpy(out, r.data(), n * sizeof(float));
    });
}

// vecstore.hpp:88 build_store -> (ids, unit rows) of the covered rows
int ssref_build_store(const float* embeddings, const float* coverage, uint64_t n, uint32_t dim, uint32_t* ids,
                      float* rows, uint64_t* count) {
    return guarded([&] {
        EmbeddingTable table(n, dim);
        std::memcpy(table.embeddings.data(), embeddings, n * dim * sizeof(float));
        std::memcpy(table.coverage.data(), coverage, n * sizeof(float));
        std::vector<Gaussian3D> gs(n);
        const VectorStore store = build_store(table, GaussianScene(std::move(gs)));
        *count = store.count();
        for (size_t i = 0; i < store.count(); ++i) {
            ids[i] = store.id_at(i);
            std::memcpy(rows + i * dim, store.vector_at(i), dim * sizeof(float));
        }
    });
}

namespace {
VectorStore make_store(const uint32_t* ids, const float* unit_rows, uint64_t count, uint32_t dim) {
    VectorStore store(dim);
    store.reserve(count);
    const Gaussian3D g;
    std::vector<float> v(dim);
    for (uint64_t i = 0; i < count; ++i) {
        std::memcpy(v.data(), unit_rows + i * dim, dim * sizeof(float));
        store.add_record(ids[i], v, g);
    }
    return store;
}
} // namespace

// vecstore.hpp:121 query_topk for nq queries; threads > 1 splits queries across std::threads.
int ssref_query_topk(const uint32_t* ids, const float* unit_rows, uint64_t count, uint32_t dim, const float* queries,
                     uint32_t nq, uint64_t k, uint32_t threads, uint32_t* out_ids, float* out_sims,
                     uint64_t* out_counts) {
    return guarded([&] {
        const VectorStore store = make_store(ids, unit_rows, count, dim);
        std::vector<std::string> errors(threads ? threads : 1);
        auto run = [&](uint32_t t, uint32_t nt) {
            try {
                for (uint32_t q = t; q < nq; q += nt) {
                    std::vector<float> qv(queries + static_cast<size_t>(q) * dim,
                                          queries + static_cast<size_t>(q + 1) * dim);
                    const std::vector<ScoredId> res = query_topk(store, qv, k);
                    out_counts[q] = res.size();
                    for (size_t i = 0; i < res.size(); ++i) {
                        out_ids[q * k + i] = res[i].gaussian_id;
                        out_sims[q * k + i] = res[i].similarity;
                    }
                }
            } catch (const std::exception& e) {
                errors[t] = e.what();
            }
        };
        const uint32_t nt = threads ? threads : 1;
        if (nt == 1) {
            run(0, 1);
        } else {
            std::vector<std::thread> pool;
            for (uint32_t t = 0; t < nt; ++t) pool.emplace_back(run, t, nt);
            for (auto& th : pool) th.join();
        }
        for (const auto& e : errors)
            if (!e.empty()) {
                // re-run the first failing query serially to surface the typed exception
                for (uint32_t q = 0; q < nq; ++q) {
                    std::vector<float> qv(queries + static_cast<size_t>(q) * dim,
                                          queries + static_cast<size_t>(q + 1) * dim);
                    query_topk(store, qv, k);
                }
            }
    });
}

// vecstore.hpp:135 query_threshold for one query; caller provides capacity = count.
int ssref_query_threshold(const uint32_t* ids, const float* unit_rows, uint64_t count, uint32_t dim, const float* q,
                          float tau, uint32_t* out_ids, float* out_sims, uint64_t* out_count) {
    return guarded([&] {
        const VectorStore store = make_store(ids, unit_rows, count, dim);
        const std::vector<ScoredId> res = query_threshold(store, std::vector<float>(q, q + dim), tau);
        *out_count = res.size();
        for (size_t i = 0; i < res.size(); ++i) {
            out_ids[i] = res[i].gaussian_id;
            out_sims[i] = res[i].similarity;
        }
    });
}

// vecstore.hpp:169-213 partition_store over records with payload means
// (means: 3 floats per record).  Outputs sized for count cells/records:
// cells 3 x n_cells, bounds 6 x n_cells (min xyz, max xyz), offsets
// n_cells + 1, ids / rows in cell order.
int ssref_partition_store(const uint32_t* ids, const float* rows, const float* means, uint64_t count, uint32_t dim,
                          double cell_size, uint64_t* n_cells, int32_t* cells, double* bounds, uint64_t* offsets,
                          uint32_t* out_ids, float* out_rows) {
    return guarded([&] {
        VectorStore store(dim);
        store.reserve(count);
        std::vector<float> v(dim);
        for (uint64_t i = 0; i < count; ++i) {
            std::memcpy(v.data(), rows + i * dim, dim * sizeof(float));
            Gaussian3D g;
            g.id = ids[i];
            g.mean = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
            store.add_record(ids[i], v, g);
        }
        const std::vector<PartitionSnapshot> snaps = partition_store(store, cell_size);
        *n_cells = snaps.size();
        uint64_t pos = 0;
        for (size_t c = 0; c < snaps.size(); ++c) {
            const PartitionSnapshot& sn = snaps[c];
            for (int a = 0; a < 3; ++a) {
                cells[3 * c + a] = sn.cell[a];
                bounds[6 * c + a] = sn.bounds.min[a];
                bounds[6 * c + 3 + a] = sn.bounds.max[a];
            }
            offsets[c] = pos;
            for (size_t i = 0; i < sn.store.count(); ++i, ++pos) {
                out_ids[pos] = sn.store.id_at(i);
                std::memcpy(out_rows + pos * dim, sn.store.vector_at(i), dim * sizeof(float));
            }
        }
        offsets[snaps.size()] = pos;
    });
}

uint32_t ssref_hardware_threads() { return std::thread::hardware_concurrency(); }

} // extern "C"
