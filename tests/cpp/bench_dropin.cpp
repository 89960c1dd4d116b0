// bench_dropin (MEASUREMENT INFRASTRUCTURE): the end-to-end embedding pass
// through the C++ drop-in, b200::encode_scene (include/semsplat_b200/
// semsplat_b200.hpp), on a dataset in the reference's on-disk formats --
// the call a reference user makes after switching (pipeline.hpp:280-282).
// Each repetition parses the scene PLY and the manifest (load_scene,
// load_manifest: the reference's own loaders), then encode_scene reads every
// view's RLE masks and CLIP vectors from disk, runs the pass on the GPU(s) and
// returns the EmbeddingTable in host memory.  Prints one JSON line.
//   bench_dropin <scene.ply> <manifest.txt> <workers> <chunk_rows> <reps>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "semsplat/pipeline.hpp"
#include "semsplat/scene_io.hpp"
#include "semsplat_b200/semsplat_b200.hpp"

using namespace semsplat;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s scene.ply manifest.txt workers chunk_rows reps\n", argv[0]);
        return 2;
    }
    const std::string scene_path = argv[1], manifest_path = argv[2];
    const uint32_t workers = (uint32_t)std::atoi(argv[3]);
    const uint64_t chunk = (uint64_t)std::atoll(argv[4]);
    const int reps = std::atoi(argv[5]);
    double best_total = 1e30, best_parse = 0, best_encode = 0, best_p1 = 0, best_p2 = 0, first_total = 0;
    size_t views = 0, covered = 0, n = 0;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = clk::now();
        const GaussianScene scene = load_scene(scene_path);
        const DatasetManifest manifest = load_manifest(manifest_path);
        const auto t1 = clk::now();
        EncodeStats st;
        const EmbeddingTable table = b200::encode_scene(scene, manifest, workers, chunk, {}, &st);
        const auto t2 = clk::now();
        const double parse = std::chrono::duration<double>(t1 - t0).count();
        const double enc = std::chrono::duration<double>(t2 - t1).count();
        if (r == 0) first_total = parse + enc;
        if (parse + enc < best_total) {
            best_total = parse + enc;
            best_parse = parse;
            best_encode = enc;
            best_p1 = st.phase1_seconds;
            best_p2 = st.phase2_seconds;
        }
        views = manifest.images.size();
        n = table.gaussian_count;
        covered = 0;
        for (size_t k = 0; k < n; ++k) covered += table.covered(k) ? 1 : 0;
    }
    std::printf("{\"views\": %zu, \"gaussians\": %zu, \"covered\": %zu, \"workers\": %u, \"reps\": %d, "
                "\"seconds\": %.6f, \"parse_seconds\": %.6f, \"encode_seconds\": %.6f, \"phase1_seconds\": %.6f, "
                "\"phase2_seconds\": %.6f, \"first_rep_seconds\": %.6f}\n",
                views, n, covered, workers, reps, best_total, best_parse, best_encode, best_p1, best_p2, first_total);
    return 0;
}
