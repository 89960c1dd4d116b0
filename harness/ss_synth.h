/* ss_synth.h -- synthetic workload generator of the bench and the tests
 * (BENCH/TEST HARNESS, not part of libsemsplat_b200.so).
 *
 * The counterpart of the reference CLI's `bench` dataset writer
 * (main.cpp:334-410 write_bench_dataset), synth_embedding
 * (providers.hpp:381-400) and look_at (fixture.hpp:65-84).  Built twice from
 * the same source: harness/libss_synth.so feeds the B200 arm and the tests,
 * oracle/libssgen.so feeds the reference arm of bench.py, so the reference
 * process never maps the product library.  Both produce identical bytes.
 */
#ifndef SS_SYNTH_H
#define SS_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as ss_camera (include/semsplat_b200.h). */
typedef struct ss_synth_camera {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    uint32_t width, height, image_id, pad;
} ss_synth_camera;

/* Bench-style uniform scene (main.cpp:340-352) from std::mt19937_64(seed). */
int ss_synth_scene(uint64_t seed, uint64_t n, double xy_extent, double z_extent, float* mean, float* scale,
                   float* quat_xyzw, float* opacity, float* color);
/* fixture.hpp:65-84 look_at */
int ss_synth_look_at(const double* eye, const double* target, uint32_t width, uint32_t height, double focal,
                     ss_synth_camera* out);
/* providers.hpp:381-400 synth_embedding */
int ss_synth_embedding(const char* label, uint32_t dim, float* out);
/* main.cpp:440-450: the bench query store/queries, U(-0.5, 0.5) per element
 * from std::mt19937_64(seed) (cmd_bench seeds it with seed ^ 0xbe9c). */
int ss_synth_uniform(uint64_t seed, uint64_t count, float* out);
/* Random-rectangle masks for one view (main.cpp:386-396) from the rng state
 * seeded by seed; writes RLE runs (capacity >= n_masks*(2*height+2)) and
 * run_offsets (n_masks+1). */
int ss_synth_rect_masks(uint64_t seed, uint32_t width, uint32_t height, uint32_t n_masks, uint32_t* runs,
                        uint64_t* run_offsets);

#ifdef __cplusplus
}
#endif
#endif /* SS_SYNTH_H */
