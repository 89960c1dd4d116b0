// Drop-in check of include/semsplat_b200/semsplat_b200.hpp: the reference's
// own API types and scenarios (tests/test_pipeline.cpp, test_rasterizer.cpp,
// test_vecstore.cpp), once through the reference CPU implementation and once
// through semsplat::b200:: on the GPU.  Built by tests/cpp/build_dropin.py in
// the build container (needs /root/reference headers + oracle/eigen_shim);
// run by tests/test_gpu_dropin.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <random>
#include <string>

#include "semsplat/fixture.hpp"
#include "semsplat/pipeline.hpp"
#include "semsplat/vecstore.hpp"
#include "semsplat_b200/semsplat_b200.hpp"

using namespace semsplat;
namespace fs = std::filesystem;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        if (cond) {                                                                   \
            ++g_pass;                                                                 \
        } else {                                                                      \
            ++g_fail;                                                                 \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
        }                                                                             \
    } while (0)

static double urand(std::mt19937_64& rng, double lo, double hi) {
    return lo + (hi - lo) * ((static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53);
}

static GaussianScene random_scene(size_t n, uint64_t seed) { // helpers.hpp:16-37
    std::mt19937_64 rng(seed);
    std::vector<Gaussian3D> gs(n);
    for (auto& g : gs) {
        const double mx = urand(rng, -2, 2), my = urand(rng, -2, 2), mz = urand(rng, -2, 2);
        g.mean = Eigen::Vector3f(float(mx), float(my), float(mz));
        const double a = urand(rng, 0.05, 0.4), b = urand(rng, 0.05, 0.4), c = urand(rng, 0.05, 0.4);
        g.scale = Eigen::Vector3f(float(a), float(b), float(c));
        const double qw = urand(rng, -1, 1), qx = urand(rng, -1, 1), qy = urand(rng, -1, 1), qz = urand(rng, -1, 1);
        g.rotation = Eigen::Quaterniond(qw, qx, qy, qz).normalized().cast<float>();
        g.opacity = float(urand(rng, 0.05, 0.95));
    }
    return GaussianScene(std::move(gs));
}

static double max_row_rel_diff(const EmbeddingTable& a, const EmbeddingTable& b) { // oracles.hpp:147-160
    double worst = 0.0;
    for (uint64_t k = 0; k < a.gaussian_count; ++k) {
        double ref = 0, err = 0;
        for (uint32_t d = 0; d < a.dim; ++d) {
            const double x = a.row(k)[d], y = b.row(k)[d];
            ref += x * x;
            err += (x - y) * (x - y);
        }
        worst = std::max(worst, ref > 0 ? std::sqrt(err / ref) : std::sqrt(err));
    }
    return worst;
}

int main() {
    const fs::path tmp = fs::temp_directory_path() / "semsplat_b200_dropin";
    fs::remove_all(tmp);

    // --- rasterize_weights_only: bit-identical WeightMap (test_rasterizer.cpp:254-270 style)
    for (uint64_t seed : {101ull, 202ull, 303ull}) {
        const GaussianScene scene = random_scene(50, seed);
        const CameraPose cam = detail::look_at(Eigen::Vector3d(0, 0, -7), Eigen::Vector3d::Zero(), 32, 32, 28.8);
        const WeightMap a = rasterize_weights_only(scene, cam);
        const WeightMap b = b200::rasterize_weights_only(scene, cam);
        bool same = a.entries.size() == b.entries.size();
        for (size_t i = 0; same && i < a.entries.size(); ++i)
            same = a.entries[i].gaussian_id == b.entries[i].gaussian_id && a.entries[i].pixel == b.entries[i].pixel &&
                   a.entries[i].weight == b.entries[i].weight;
        CHECK(same);
        CHECK(a.per_pixel_total == b.per_pixel_total);
        const std::vector<Projected2D> pa = b200::project_all(scene, cam);
        bool pok = true;
        for (size_t k = 0; k < scene.size(); ++k) {
            const Projected2D r = project_gaussian(scene[k], cam);
            pok = pok && r.visible == pa[k].visible;
            if (r.visible)
                pok = pok && r.mu2d.x() == pa[k].mu2d.x() && r.mu2d.y() == pa[k].mu2d.y() && r.cov_xx == pa[k].cov_xx &&
                      r.cov_xy == pa[k].cov_xy && r.cov_yy == pa[k].cov_yy && r.depth == pa[k].depth;
        }
        CHECK(pok);
        // rasterize (rasterizer.hpp:261): RenderResult image, alpha and WeightMap bit-identical
        const RenderResult ra = rasterize(scene, cam);
        const RenderResult rb = b200::rasterize(scene, cam);
        CHECK(ra.image.pixels == rb.image.pixels);
        CHECK(ra.alpha == rb.alpha);
        CHECK(ra.weights.entries.size() == rb.weights.entries.size());
        CHECK(ra.weights.per_pixel_total == rb.weights.per_pixel_total);
    }

    // --- encode_scene vs the reference on its own fixtures (test_pipeline.cpp:283-354)
    for (uint32_t mask_scale : {1u, 2u}) {
        FixtureSpec spec;
        spec.object_count = 3;
        spec.gaussians_per_object = 12;
        spec.view_count = 4;
        spec.resolution = 32;
        spec.mask_scale = mask_scale;
        spec.embedding_dim = 16;
        spec.seed = 5;
        const std::string dir = (tmp / ("fx" + std::to_string(mask_scale))).string();
        const DatasetManifest manifest = load_manifest(write_fixture(generate_fixture(spec), dir));
        const GaussianScene scene = load_scene(manifest.resolve("scene.ply"));
        const EmbeddingTable ref = encode_scene(scene, manifest, 1, 0);
        for (uint32_t workers : {1u, 3u}) {
            EncodeStats stats, ref_stats;
            const EmbeddingTable got = b200::encode_scene(scene, manifest, workers, 7, {}, &stats);
            encode_scene(scene, manifest, workers, 7, {}, &ref_stats);
            CHECK(max_row_rel_diff(ref, got) <= 1e-4);
            bool cov = true;
            for (uint64_t k = 0; k < scene.size(); ++k) cov = cov && ref.covered(k) == got.covered(k);
            CHECK(cov);
            CHECK(stats.worker_images == ref_stats.worker_images);
            CHECK(stats.worker_entries == ref_stats.worker_entries); // (gid, mask) entries per worker
        }
        // pipeline.hpp:272-279: with SS_OPT_DETERMINISTIC the table is bitwise
        // identical run to run
        b200::set_deterministic(true);
        const EmbeddingTable d1 = b200::encode_scene(scene, manifest, 1, 0);
        const EmbeddingTable d2 = b200::encode_scene(scene, manifest, 1, 0);
        b200::set_deterministic(false);
        CHECK(max_row_rel_diff(ref, d1) <= 1e-4);
        CHECK(d1.embeddings.size() == d2.embeddings.size() && d1.coverage.size() == d2.coverage.size() &&
              std::memcmp(d1.embeddings.data(), d2.embeddings.data(), d1.embeddings.size() * sizeof(float)) == 0 &&
              std::memcmp(d1.coverage.data(), d2.coverage.data(), d1.coverage.size() * sizeof(float)) == 0);
    }

    // --- failure paths (test_pipeline.cpp:356-393)
    {
        FixtureSpec spec;
        spec.object_count = 2;
        spec.gaussians_per_object = 8;
        spec.view_count = 3;
        spec.resolution = 24;
        spec.embedding_dim = 8;
        spec.seed = 33;
        const std::string dir = (tmp / "fail").string();
        const DatasetManifest manifest = load_manifest(write_fixture(generate_fixture(spec), dir));
        const GaussianScene scene = load_scene(manifest.resolve("scene.ply"));
        bool contract = false;
        try {
            b200::encode_scene(scene, manifest, 0, 0);
        } catch (const ContractError&) {
            contract = true;
        }
        CHECK(contract);
        fs::remove(manifest.resolve("masks/view_1.rle"));
        bool named = false;
        try {
            b200::encode_scene(scene, manifest, 1, 0);
        } catch (const DataError& e) {
            named = std::string(e.what()).find("image 1") != std::string::npos;
        }
        CHECK(named);
        bool pipeline = false;
        try {
            b200::encode_scene(scene, manifest, 2, 0);
        } catch (const PipelineError& e) {
            pipeline = e.worker_status.size() == 2;
        }
        CHECK(pipeline);
    }

    // --- query_topk / query_threshold vs the reference (test_vecstore.cpp:144-183)
    {
        std::mt19937_64 rng(1234);
        const uint32_t dim = 64;
        VectorStore store(dim);
        for (uint32_t i = 0; i < 5000; ++i) {
            std::vector<float> v(dim);
            for (auto& x : v) x = float(urand(rng, -1, 1));
            store.add_record(i, normalized_copy(v.data(), dim), Gaussian3D{});
        }
        const b200::DeviceStore ds = b200::upload_store(store);
        bool ok = true;
        for (int t = 0; t < 10; ++t) {
            std::vector<float> q(dim);
            for (auto& x : q) x = float(urand(rng, -1, 1));
            const auto a = query_topk(store, q, 37);
            const auto b = b200::query_topk(ds, q, 37);
            ok = ok && a.size() == b.size();
            for (size_t i = 0; ok && i < a.size(); ++i)
                ok = a[i].gaussian_id == b[i].gaussian_id && a[i].similarity == b[i].similarity;
            const auto c = query_threshold(store, q, 0.05f);
            const auto d = b200::query_threshold(ds, q, 0.05f);
            ok = ok && c.size() == d.size();
            for (size_t i = 0; ok && i < c.size(); ++i)
                ok = c[i].gaussian_id == d[i].gaussian_id && c[i].similarity == d[i].similarity;
        }
        CHECK(ok);
        bool numeric = false;
        try {
            b200::query_topk(ds, std::vector<float>(dim, 0.0f), 3);
        } catch (const NumericError&) {
            numeric = true;
        }
        CHECK(numeric);

        // k beyond 64, batched queries, run_query payloads, fetch_store round trip
        std::vector<std::vector<float>> qs;
        bool big = true;
        for (int t = 0; t < 5; ++t) {
            std::vector<float> q(dim);
            for (auto& x : q) x = float(urand(rng, -1, 1));
            qs.push_back(q);
            const auto a = query_topk(store, q, 300);
            const auto b = b200::query_topk(ds, q, 300);
            big = big && a.size() == b.size();
            for (size_t i = 0; big && i < a.size(); ++i)
                big = a[i].gaussian_id == b[i].gaussian_id && a[i].similarity == b[i].similarity;
        }
        CHECK(big);
        const auto batch = b200::query_topk_batch(ds, qs, 20);
        bool bok = batch.size() == qs.size();
        for (size_t t = 0; bok && t < qs.size(); ++t) {
            const auto a = query_topk(store, qs[t], 20);
            bok = a.size() == batch[t].size();
            for (size_t i = 0; bok && i < a.size(); ++i)
                bok = a[i].gaussian_id == batch[t][i].gaussian_id && a[i].similarity == batch[t][i].similarity;
        }
        CHECK(bok);
        const VectorStore back = b200::fetch_store(ds);
        bool fok = back.count() == store.count() && back.dim() == store.dim();
        for (size_t i = 0; fok && i < store.count(); ++i)
            fok = back.id_at(i) == store.id_at(i) &&
                  std::memcmp(back.vector_at(i), store.vector_at(i), dim * sizeof(float)) == 0;
        CHECK(fok);
    }

    // --- run_query (query.hpp:102-122) on a store built from an encoded fixture
    {
        const uint32_t dim = 32;
        std::mt19937_64 rng(77);
        GaussianScene scene = random_scene(400, 9);
        EmbeddingTable table(scene.size(), dim);
        for (uint64_t k = 0; k < scene.size(); ++k) {
            if (k % 3 == 0) continue; // uncovered rows stay out of the store
            for (uint32_t d = 0; d < dim; ++d) table.embeddings[k * dim + d] = float(urand(rng, -1, 1));
            table.coverage[k] = 1.0f;
        }
        const VectorStore hs = build_store(table, scene);
        const b200::DeviceStore ds = b200::build_store(table, scene);
        const TextProvider prov = TextProvider::synthetic(dim);
        bool rq = true;
        for (const QueryMode& mode : {QueryMode::topk(7), QueryMode::threshold(0.1f)}) {
            const QueryResult a = run_query(hs, "a chair", mode, prov);
            const QueryResult b = b200::run_query(ds, "a chair", mode, prov);
            rq = rq && a.query_vector == b.query_vector && a.matches.size() == b.matches.size();
            for (size_t i = 0; rq && i < a.matches.size(); ++i)
                rq = a.matches[i].gaussian_id == b.matches[i].gaussian_id &&
                     a.matches[i].similarity == b.matches[i].similarity &&
                     a.matches[i].payload.mean == b.matches[i].payload.mean &&
                     a.matches[i].payload.opacity == b.matches[i].payload.opacity;
        }
        CHECK(rq);
    }

    // --- partition_store (vecstore.hpp:169-213): device grouping vs the reference, incl. boundary means
    {
        const uint32_t dim = 16;
        std::mt19937_64 rng(91);
        VectorStore store(dim);
        for (uint32_t i = 0; i < 3000; ++i) {
            std::vector<float> v(dim);
            for (auto& x : v) x = float(urand(rng, -1, 1));
            Gaussian3D g;
            g.id = 5000 - i;
            // means on a 0.25 lattice land exactly on cell boundaries for cell sizes 0.5 / 1.0
            g.mean = {float(std::floor(urand(rng, -12, 12)) * 0.25), float(urand(rng, -3, 3)),
                      float(i % 7 == 0 ? 1.0 : urand(rng, 0, 2))};
            store.add_record(g.id, normalized_copy(v.data(), dim), g);
        }
        const b200::DeviceStore ds = b200::upload_store(store);
        bool pok = true;
        for (double cell : {0.5, 1.0, 0.37, 1e-9}) {
            const auto a = partition_store(store, cell);
            const auto b = b200::partition_store(ds, cell);
            pok = pok && a.size() == b.size();
            for (size_t c = 0; pok && c < a.size(); ++c) {
                pok = a[c].cell == b[c].cell && a[c].bounds.min == b[c].bounds.min &&
                      a[c].bounds.max == b[c].bounds.max && a[c].store.count() == b[c].store.count();
                for (size_t i = 0; pok && i < a[c].store.count(); ++i)
                    pok = a[c].store.id_at(i) == b[c].store.id_at(i) &&
                          std::memcmp(a[c].store.vector_at(i), b[c].store.vector_at(i), dim * sizeof(float)) == 0 &&
                          a[c].store.payload_at(i).mean == b[c].store.payload_at(i).mean;
            }
        }
        CHECK(pok);
        bool contract = false;
        try {
            b200::partition_store(ds, 0.0);
        } catch (const ContractError&) {
            contract = true;
        }
        CHECK(contract);
    }

    fs::remove_all(tmp);
    std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
