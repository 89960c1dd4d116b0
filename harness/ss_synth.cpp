// Synthetic workload generator: the B200 framework's counterpart of the
// reference CLI's `bench` dataset writer (main.cpp:334-410) and of
// synth_embedding (providers.hpp:381-400) / look_at (fixture.hpp:65-84).
// BENCH/TEST HARNESS, not linked into libsemsplat_b200.so: host code that
// produces the inputs the bench and the tests feed to BOTH the device path
// and the CPU oracle (built as harness/libss_synth.so and oracle/libssgen.so).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "ss_synth.h"

namespace {

uint64_t fnv1a64(const std::string& s) { // core.hpp:94-101
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

struct Uniform { // main.cpp:335-338
    std::mt19937_64 rng;
    explicit Uniform(uint64_t seed) : rng(seed) {}
    double operator()(double lo, double hi) {
        return lo + (hi - lo) * ((static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53);
    }
};

// Vector helpers with the evaluation order of the oracle's Eigen shim
// (oracle/eigen_shim/Eigen/Dense): 3-vector squaredNorm = (x*x + y*y) + z*z.
void normalize3(double v[3]) {
    const double n = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
    if (!(n > 0)) return;
    const double s = std::sqrt(n);
    for (int i = 0; i < 3; ++i) v[i] = v[i] / s;
}
void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

} // namespace

extern "C" {

int ss_synth_scene(uint64_t seed, uint64_t n, double xy_extent, double z_extent, float* mean, float* scale,
                   float* quat_xyzw, float* opacity, float* color) {
    Uniform u(seed);
    for (uint64_t k = 0; k < n; ++k) {
        // main.cpp:341-351, draws taken in source order
        const double mx = u(-xy_extent, xy_extent), my = u(-xy_extent, xy_extent), mz = u(-z_extent, z_extent);
        mean[3 * k] = static_cast<float>(mx);
        mean[3 * k + 1] = static_cast<float>(my);
        mean[3 * k + 2] = static_cast<float>(mz);
        for (int i = 0; i < 3; ++i) scale[3 * k + i] = static_cast<float>(u(0.02, 0.05));
        double qw = u(-1, 1), qx = u(-1, 1), qy = u(-1, 1), qz = u(-1, 1);
        // Quaterniond::normalized: (x*x + z*z) + (y*y + w*w)
        const double n2 = (qx * qx + qz * qz) + (qy * qy + qw * qw);
        if (n2 > 0) {
            const double s = std::sqrt(n2);
            qx /= s;
            qy /= s;
            qz /= s;
            qw /= s;
        }
        quat_xyzw[4 * k] = static_cast<float>(qx);
        quat_xyzw[4 * k + 1] = static_cast<float>(qy);
        quat_xyzw[4 * k + 2] = static_cast<float>(qz);
        quat_xyzw[4 * k + 3] = static_cast<float>(qw);
        opacity[k] = static_cast<float>(u(0.3, 0.9));
        for (int i = 0; i < 3; ++i) {
            const float cv = static_cast<float>(u(0, 1));
            if (color) color[3 * k + i] = cv;
        }
    }
    return 0;
}

int ss_synth_look_at(const double* eye, const double* target, uint32_t width, uint32_t height, double focal,
                     ss_synth_camera* out) {
    double fwd[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
    normalize3(fwd);
    double up[3] = {0, 1, 0};
    if (std::abs((fwd[0] * up[0] + fwd[1] * up[1]) + fwd[2] * up[2]) > 0.99) {
        up[0] = 1;
        up[1] = 0;
        up[2] = 0;
    }
    double right[3], down[3];
    cross3(fwd, up, right);
    normalize3(right);
    cross3(fwd, right, down);
    std::memset(out, 0, sizeof(*out));
    for (int j = 0; j < 3; ++j) {
        out->R[j] = right[j];
        out->R[3 + j] = down[j];
        out->R[6 + j] = fwd[j];
    }
    // translation = -(R * eye), product order a0 + (a1 + a2)
    for (int i = 0; i < 3; ++i)
        out->t[i] = -(out->R[3 * i] * eye[0] + (out->R[3 * i + 1] * eye[1] + out->R[3 * i + 2] * eye[2]));
    out->fx = out->fy = focal;
    out->cx = width / 2.0;
    out->cy = height / 2.0;
    out->width = width;
    out->height = height;
    return 0;
}

int ss_synth_embedding(const char* label, uint32_t dim, float* out) {
    if (dim < 2) return 1; // ContractError
    std::mt19937_64 rng(fnv1a64(label) ^ 0x9e3779b97f4a7c15ull);
    auto uniform01 = [&rng]() { return (static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53; };
    std::vector<double> values(dim);
    for (uint32_t i = 0; i < dim; i += 2) {
        const double u1 = uniform01();
        const double u2 = uniform01();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        values[i] = radius * std::cos(2.0 * M_PI * u2);
        if (i + 1 < dim) values[i + 1] = radius * std::sin(2.0 * M_PI * u2);
    }
    double norm_sq = 0.0;
    for (double v : values) norm_sq += v * v;
    const double inv_norm = 1.0 / std::sqrt(norm_sq);
    for (uint32_t i = 0; i < dim; ++i) out[i] = static_cast<float>(values[i] * inv_norm);
    return 0;
}

int ss_synth_rect_masks(uint64_t seed, uint32_t width, uint32_t height, uint32_t n_masks, uint32_t* runs,
                        uint64_t* run_offsets) {
    Uniform u(seed);
    uint64_t w = 0;
    run_offsets[0] = 0;
    for (uint32_t j = 0; j < n_masks; ++j) {
        // main.cpp:390-395
        const uint32_t x0 = static_cast<uint32_t>(u(0, width / 2)), y0 = static_cast<uint32_t>(u(0, height / 2));
        const uint32_t x1 = x0 + static_cast<uint32_t>(u(4, width / 2)),
                       y1 = y0 + static_cast<uint32_t>(u(4, height / 2));
        const uint32_t xe = x1 < width - 1 ? x1 : width - 1, ye = y1 < height - 1 ? y1 : height - 1;
        // rle_encode (providers.hpp:77-93): alternating runs, zeros first, no
        // empty runs except a leading zero run
        uint64_t pos = 0;
        uint8_t cur = 0;
        uint64_t run = 0;
        const uint64_t total = static_cast<uint64_t>(width) * height;
        auto push = [&](uint8_t v, uint64_t len) {
            if (len == 0) return;
            if (v == cur) {
                run += len;
            } else {
                runs[w++] = static_cast<uint32_t>(run);
                cur = v;
                run = len;
            }
        };
        for (uint32_t y = y0; y <= ye && x0 <= xe; ++y) {
            const uint64_t s = static_cast<uint64_t>(y) * width + x0, e = static_cast<uint64_t>(y) * width + xe + 1;
            push(0, s - pos);
            push(1, e - s);
            pos = e;
        }
        push(0, total - pos);
        runs[w++] = static_cast<uint32_t>(run);
        run_offsets[j + 1] = w;
    }
    return 0;
}

// main.cpp:440-450 (cmd_bench query store): x = f32((rng() >> 11) + 0.5) * 2^-53 - 0.5)
// for every element, store rows first, then the query vectors, from
// std::mt19937_64(seed) -- the caller passes cfg.seed ^ 0xbe9c.
int ss_synth_uniform(uint64_t seed, uint64_t count, float* out) {
    std::mt19937_64 rng(seed);
    for (uint64_t i = 0; i < count; ++i)
        out[i] = static_cast<float>((static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53 - 0.5);
    return 0;
}

} // extern "C"
