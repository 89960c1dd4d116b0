// Bit-exact fp64 kernels: projection and the tile compositor.
//
// Compiled with -fmad=false AND written with explicit __dmul_rn/__dadd_rn/
// __ddiv_rn/__dsqrt_rn so no FMA contraction can creep in: the reference is
// built for baseline x86-64 (no FMA, proj/CMakeLists.txt:11), and its bits
// -- depth order, per-tile lists, per-pixel contributor lists and f32
// weights -- must be reproduced exactly (BASELINE.json north_star).
// Evaluation order: SURVEY.md Appendix A.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <stdint.h>

#include "glibc_exp.cuh"
#include "ss_internal.cuh"

namespace ss {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

// x86 cvttsd2si semantics (rasterizer.hpp:173-176): NaN / out of range -> INT_MIN
__device__ __forceinline__ int32_t cvt_i32_x86(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
    return (int32_t)v;
}

constexpr double kNearPlane = 0.01;        // projection.hpp:15
constexpr double kCovDilation = 0.3;       // projection.hpp:17
constexpr double kWeightCutoff = 1.0 / 255.0; // rasterizer.hpp:17
constexpr double kAlphaMax = 0.99;         // rasterizer.hpp:19
constexpr double kAlphaSkip = 1.0 / 255.0; // rasterizer.hpp:21
constexpr double kTransmittanceFloor = 1e-4; // rasterizer.hpp:23
constexpr double kMahalanobisSqCutoff = 9.0; // rasterizer.hpp:26
// kAlphaMax, kAlphaSkip, kWeightCutoff, kTransmittanceFloor for the compositor's
// inner loop (non-const so they stay constant-bank operands)
__device__ __constant__ double kCompositeConst[4] = {kAlphaMax, kAlphaSkip, kWeightCutoff, kTransmittanceFloor};

// ------------------------------------------------------- 3-D covariance
// scene.hpp:33-37 covariance3d: Eigen quaternion normalize (2-wide redux) +
// toRotationMatrix, then R * diag(s^2) * R^T.  It does not depend on the
// camera, so it is evaluated once per scene (same operation order as the
// reference) and projection reads the nine doubles (SoA, [9][n]).
__global__ void __launch_bounds__(256) cov3d_kernel(const float4* __restrict__ scale, const float4* __restrict__ quat,
                                                    uint64_t n, double* __restrict__ cov3) {
    const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const float4 q = quat[id];
    double qx = q.x, qy = q.y, qz = q.z, qw = q.w;
    const double n2 = da(da(dm(qx, qx), dm(qz, qz)), da(dm(qy, qy), dm(qw, qw)));
    if (n2 > 0.0) {
        const double nn = __dsqrt_rn(n2);
        qx = dd(qx, nn);
        qy = dd(qy, nn);
        qz = dd(qz, nn);
        qw = dd(qw, nn);
    }
    const double tx = dm(2.0, qx), ty = dm(2.0, qy), tz = dm(2.0, qz);
    const double twx = dm(tx, qw), twy = dm(ty, qw), twz = dm(tz, qw);
    const double txx = dm(tx, qx), txy = dm(ty, qx), txz = dm(tz, qx);
    const double tyy = dm(ty, qy), tyz = dm(tz, qy), tzz = dm(tz, qz);
    double R[9];
    R[0] = ds(1.0, da(tyy, tzz));
    R[1] = ds(txy, twz);
    R[2] = da(txz, twy);
    R[3] = da(txy, twz);
    R[4] = ds(1.0, da(txx, tzz));
    R[5] = ds(tyz, twx);
    R[6] = ds(txz, twy);
    R[7] = da(tyz, twx);
    R[8] = ds(1.0, da(txx, tyy));
    const float4 sc = scale[id];
    const double s0 = sc.x, s1 = sc.y, s2c = sc.z;
    const double s2[3] = {dm(s0, s0), dm(s1, s1), dm(s2c, s2c)};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            cov3[(size_t)(3 * i + j) * n + id] = da(dm(dm(R[3 * i], s2[0]), R[3 * j]),
                                                    da(dm(dm(R[3 * i + 1], s2[1]), R[3 * j + 1]),
                                                       dm(dm(R[3 * i + 2], s2[2]), R[3 * j + 2])));
}

// ---------------------------------------------------------------- project
// One thread per Gaussian (id order).  scene.hpp:33-37 covariance3d +
// projection.hpp:33-55 project_gaussian + rasterizer.hpp:66-71 conic_of +
// the padded 3-sigma box and cull (rasterizer.hpp:160-179).  Survivors get
// their depth bit pattern as sort key (positive f64 => monotone as u64).
#ifndef SS_PROJECT_THREADS
#define SS_PROJECT_THREADS 128
#endif
__global__ void __launch_bounds__(SS_PROJECT_THREADS) project_kernel(ProjectParams p) {
    const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool survive = false;
    unsigned long long key = ~0ull;
    if (id < p.n) {
        const float4 mo = p.mean_op[id];
        const ss_camera& cam = p.cam;
        const double m0 = mo.x, m1 = mo.y, m2 = mo.z;
        const double* Rc = cam.R;
        double xc[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            xc[i] = da(da(dm(Rc[3 * i], m0), da(dm(Rc[3 * i + 1], m1), dm(Rc[3 * i + 2], m2))), cam.t[i]);
        if (p.dbg) p.dbg[id] = ss_projected{(uint32_t)id, 0u, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (xc[2] > kNearPlane) {
            const double z = xc[2];
            const double mu_x = da(dd(dm(cam.fx, xc[0]), z), cam.cx);
            const double mu_y = da(dd(dm(cam.fy, xc[1]), z), cam.cy);

            // scene.hpp:33-37 covariance3d, cached per scene (cov3d_kernel)
            double S[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) S[k] = __ldg(p.cov3 + (size_t)k * p.n + id);
            const double zz = dm(z, z);
            const double J00 = dd(cam.fx, z), J02 = dd(dm(-cam.fx, xc[0]), zz);
            const double J11 = dd(cam.fy, z), J12 = dd(dm(-cam.fy, xc[1]), zz);
            double M[6];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                M[j] = da(da(dm(J00, Rc[j]), dm(0.0, Rc[3 + j])), dm(J02, Rc[6 + j]));
                M[3 + j] = da(da(dm(0.0, Rc[j]), dm(J11, Rc[3 + j])), dm(J12, Rc[6 + j]));
            }
            double T[6];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    T[3 * i + j] = da(da(dm(M[3 * i], S[j]), dm(M[3 * i + 1], S[3 + j])), dm(M[3 * i + 2], S[6 + j]));
            double C[4];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    C[2 * i + j] =
                        da(da(dm(T[3 * i], M[3 * j]), dm(T[3 * i + 1], M[3 * j + 1])), dm(T[3 * i + 2], M[3 * j + 2]));
            const double cxx = da(C[0], kCovDilation);
            const double cxy = dm(0.5, da(C[1], C[2]));
            const double cyy = da(C[3], kCovDilation);
            if (p.dbg) p.dbg[id] = ss_projected{(uint32_t)id, 1u, mu_x, mu_y, cxx, cxy, cyy, z};

            // conic_of
            const double det = ds(dm(cxx, cyy), dm(cxy, cxy));
            if (det < 1e-12) {
                atomicAdd(&p.info->err_count, 1u);
                atomicMin(&p.info->err_gid, (unsigned int)id);
            } else {
                SplatRec r;
                r.mu_x = mu_x;
                r.mu_y = mu_y;
                r.a = dd(cyy, det);
                r.b2 = dm(2.0, dd(-cxy, det));
                r.c = dd(cxx, det);
                r.opacity = (double)mo.w;
                const double rx = da(dm(3.0, __dsqrt_rn(cxx)), 1.0);
                const double ry = da(dm(3.0, __dsqrt_rn(cyy)), 1.0);
                const int32_t W = (int32_t)cam.width, H = (int32_t)cam.height;
                int32_t v;
                v = cvt_i32_x86(ceil(ds(mu_x, rx)));
                const int32_t x0 = v > 0 ? v : 0;
                v = cvt_i32_x86(floor(da(mu_x, rx)));
                const int32_t x1 = v < W - 1 ? v : W - 1;
                v = cvt_i32_x86(ceil(ds(mu_y, ry)));
                const int32_t y0 = v > 0 ? v : 0;
                v = cvt_i32_x86(floor(da(mu_y, ry)));
                const int32_t y1 = v < H - 1 ? v : H - 1;
                if (!(x0 > x1 || y0 > y1)) {
                    if (p.tile_count) {
                        // rasterizer.hpp:185-194: the splat joins every tile its box covers
                        for (uint32_t ty = (uint32_t)y0 / kTile; ty <= (uint32_t)y1 / kTile; ++ty)
                            for (uint32_t tx = (uint32_t)x0 / kTile; tx <= (uint32_t)x1 / kTile; ++tx)
                                atomicAdd(p.tile_count + ty * p.tiles_x + tx, 1u);
                    }
                    p.rec[id] = r;
                    p.boxes[id] = make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
                    survive = true;
                    key = (unsigned long long)__double_as_longlong(z);
                }
            }
        }
        p.keys[id] = key;
        if (!survive) p.boxes[id] = make_uint2(0xffffffffu, 0xffffffffu); // no tile instances
    }
    // block-reduce survivors' count and key range, one atomic per block
    const unsigned long long kmin = survive ? key : ~0ull;
    const unsigned long long kmax = survive ? key : 0ull;
    __shared__ unsigned long long s_min[8], s_max[8];
    __shared__ unsigned int s_cnt[8];
    unsigned long long wmin = kmin, wmax = kmax;
    unsigned int wcnt = __popc(__ballot_sync(0xffffffffu, survive));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, wmin, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, wmax, o);
        wmin = a < wmin ? a : wmin;
        wmax = b > wmax ? b : wmax;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_min[warp] = wmin;
        s_max[warp] = wmax;
        s_cnt[warp] = wcnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bmin = ~0ull, bmax = 0;
        unsigned int bcnt = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            bmin = s_min[w] < bmin ? s_min[w] : bmin;
            bmax = s_max[w] > bmax ? s_max[w] : bmax;
            bcnt += s_cnt[w];
        }
        if (bcnt) {
            atomicAdd(&p.info->n_surv, (unsigned long long)bcnt);
            atomicMin(&p.info->min_key, bmin);
            atomicMax(&p.info->max_key, bmax);
        }
    }
}

// ------------------------------------------------------------- compositor
#ifndef SS_PIX_SMEM
#define SS_PIX_SMEM 1
#endif

// Per-pixel compositing state (rasterizer.hpp:112-133).
struct PixelState {
    double T;
    double total;
    uint32_t count, out, pixel;
    uint32_t px, py;
    double dpx, dpy;
    bool inside, done;
    uint32_t lbit; // per-step compositor: the lane's bit while compositing, 0 once done
};

// Evaluate one splat at one pixel: the reference's box test, Mahalanobis
// cutoff, alpha clamp, skip rule, weight cutoff and transmittance floor, in
// its exact fp64 operation order.  Returns whether an entry is emitted.
template <bool FALLOFF, typename Rec>
__device__ __forceinline__ bool composite_one(PixelState& ps, double dpx, double dpy, const Rec& s, uint32_t stab_addr,
                                              float& wf) {
    const double dx = ds(dpx, s.mu_x), dy = ds(dpy, s.mu_y);
    const double d2 = da(da(dm(dm(s.a, dx), dx), dm(dm(s.b2, dx), dy)), dm(dm(s.c, dy), dy));
    if (d2 > kMahalanobisSqCutoff) return false;
    const double g = glibc_exp_small(dm(-0.5, d2), stab_addr);
    if constexpr (FALLOFF) {
        if (g >= kWeightCutoff) {
            wf = __double2float_rn(g);
            return true;
        }
        return false;
    } else {
        const double og = dm(s.opacity, g);
        // std::min(kAlphaMax, og) (rasterizer.hpp:124): (og < max) ? og : max, NaN -> max.
        // The thresholds come from the constant bank (kCompositeConst) so the
        // loop does not re-materialise 64-bit literals.
        const double amax = kCompositeConst[0];
        const double alpha = og < amax ? og : amax;
        if (alpha < kCompositeConst[1]) return false;
        const double w = dm(alpha, ps.T);
        const bool emit = w >= kCompositeConst[2];
        if (emit) wf = __double2float_rn(w);
        ps.T = dm(ps.T, ds(1.0, alpha));
        if (ps.T < kCompositeConst[3]) {
            ps.done = true;
            ps.lbit = 0u;
        }
        return emit;
    }
}

// The six doubles of a staged SplatRec (its first 48 bytes), read from a
// 32-bit shared-window address.
struct StagedSplat {
    double mu_x, mu_y, a, b2, c, opacity;
};
__device__ __forceinline__ StagedSplat lds_splat(uint32_t addr) {
    StagedSplat r;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.mu_x), "=d"(r.mu_y) : "r"(addr));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(r.a), "=d"(r.b2) : "r"(addr));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+32];" : "=d"(r.c), "=d"(r.opacity) : "r"(addr));
    return r;
}

// Bits of a warp's 8x4 block (lane l = column l&7, row l>>3) inside the
// splat's padded box: the reference's per-pixel box test (rasterizer.hpp:115)
// evaluated once per (splat, block).
__device__ __forceinline__ uint32_t block_box_mask(uint32_t sx0, uint32_t sx1, uint32_t sy0, uint32_t sy1, uint32_t bx0,
                                                   uint32_t by0) {
    const int c0 = max((int)sx0 - (int)bx0, 0), c1 = min((int)sx1 - (int)bx0, 7);
    const int r0 = max((int)sy0 - (int)by0, 0), r1 = min((int)sy1 - (int)by0, 3);
    if (c0 > c1 || r0 > r1) return 0u;
    const uint32_t row = (0xffu >> (7 - c1)) & (0xffu << c0);           // columns c0..c1 of one row
    const uint32_t rows = (0xffffffffu >> (8 * (3 - r1))) & (0xffffffffu << (8 * r0)); // bytes r0..r1
    return (row * 0x01010101u) & rows;                                   // row replicated, rows kept
}

// Fused-mode gating of one pixel slot's contribution: lanes with identical
// mask bitsets are summed with an xor butterfly (bit-identical in every lane),
// then lane m adds the group sum to mask 32w+m when the group has that bit.
// FIX: the scalars are u64 fixed point (KIND 4, SS_OPT_DETERMINISTIC): the
// group sum is added exactly by an integer atomic.
template <int MW, bool FIX>
__device__ __forceinline__ void gate_and_accumulate(const RasterParams& p, bool contrib, float wf, uint32_t grp,
                                                    const uint32_t (&bits)[MW], uint32_t gid, uint32_t lane) {
    const uint32_t em = __ballot_sync(0xffffffffu, contrib);
    if (!em) return;
    uint32_t rem = em;
    using Acc = typename std::conditional<FIX, acc_t, float>::type;
    Acc* row = static_cast<Acc*>(p.acc) + ((size_t)gid * p.n_masks + p.mask_base + lane);
    while (rem) {
        const int leader = __ffs(rem) - 1;
        const uint32_t gm = __shfl_sync(0xffffffffu, grp, leader);
        float v = (contrib && ((gm >> lane) & 1u)) ? wf : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
#pragma unroll
        for (int w = 0; w < MW; ++w) {
            const uint32_t gb = __shfl_sync(0xffffffffu, bits[w], leader);
            if ((gb >> lane) & 1u) {
                if constexpr (FIX) atomicAdd(row + w * 32, acc_fix(v));
                else atomicAdd(row + w * 32, v);
            }
        }
        rem &= ~gm;
    }
    // stamp the Gaussian as touched in this view (fire-and-forget; stamps are
    // never cleared, the next view uses gen + 1); the contraction list is
    // compacted from the stamps after the compositor (touched_compact_kernel)
    if ((int)lane == __ffs(em) - 1) p.touched[gid] = p.gen;
}

template <int MW>
__device__ __forceinline__ uint32_t match_bits(const uint32_t (&bits)[MW]) {
    if constexpr (MW == 1) {
        return __match_any_sync(0xffffffffu, bits[0]);
    } else if constexpr (MW == 2) {
        return __match_any_sync(0xffffffffu, ((unsigned long long)bits[1] << 32) | bits[0]);
    } else {
        return __match_any_sync(0xffffffffu, ((unsigned long long)bits[1] << 32) | bits[0]) &
               __match_any_sync(0xffffffffu, ((unsigned long long)bits[3] << 32) | bits[2]);
    }
}

// One CTA (8 warps) per 16x16 tile, one thread per pixel.  Warp w owns the
// 8x4 block at (8*(w&1), 4*(w>>1)).  Each warp walks the tile's depth-ordered
// splat list independently, 32 entries at a time: one ballot culls the splats
// whose padded box misses the block, the hits are staged in the warp's
// shared-memory slice, and every lane composites its pixel against them front
// to back; the warp stops when all 32 of its pixels have terminated.  This
// shaping changes nothing in the arithmetic: every pixel still visits exactly
// the splats whose box contains it, in depth order.
//
// KIND 0: count contributions per pixel (sizes the capture).
// KIND 1: capture -- write WeightEntry records at per-pixel offsets, in depth
//         order (= the reference's stable_sort by pixel), per_pixel_total and
//         alpha = 1 - T_final.
// KIND 2: fused -- gate each contribution by the pixel's SAM-mask bitset and
//         add w into per-(Gaussian, mask) fp32 scalars (never a 512-d scatter).
//         One pass covers up to 128 masks (MW words); views with more masks
//         (providers.hpp:135 allows any count) run one pass per 128-mask
//         window [mask_base, mask_base + 128), each recompositing the tile.
// KIND 4: KIND 2 with u64 fixed-point scalars (SS_OPT_DETERMINISTIC).
// One warp composites one 8x4 block (bx0, by0) of a tile against the tile's
// list: the body of raster_kernel / raster_persist_kernel.
// RESUME: continue a block the prefix-sorted pass left unfinished, from its
// saved list position and per-pixel transmittance (raster_resume_kernel).
template <int KIND, bool FALLOFF, int MW, bool RESUME = false>
__device__ __forceinline__ void composite_block(const RasterParams& p, uint32_t tile, uint32_t wb, uint32_t lane,
                                                SplatRec* wrec, uint2* wmg, uint32_t srec_addr,
                                                uint32_t stab_addr, uint32_t spix_addr) {
    const uint32_t tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const uint32_t bx0 = tx * kTile + 8u * (wb & 1u), by0 = ty * kTile + 4u * (wb >> 1);
    const uint32_t bx1 = bx0 + 7u, by1 = by0 + 3u;
    const uint32_t start = p.tile_start[tile], end = p.tile_end[tile];

    PixelState ps;
    ps.px = bx0 + (lane & 7u);
    ps.py = by0 + (lane >> 3);
    ps.inside = ps.px < p.width && ps.py < p.height;
    ps.pixel = ps.py * p.width + ps.px;
    ps.dpx = (double)(int32_t)ps.px;
    ps.dpy = (double)(int32_t)ps.py;
#if SS_PIX_SMEM
    // the pixel's fp64 coordinates wait in the lane's shared-memory slot: one
    // LDS per evaluated step instead of re-deriving and converting them (the
    // 40-register budget cannot keep two doubles live across the loop)
    uint32_t pix_addr = spix_addr + lane * 16u;
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(pix_addr), "d"(ps.dpx), "d"(ps.dpy) : "memory");
#endif
    ps.T = 1.0;
    ps.total = 0.0;
    ps.count = 0;
    ps.out = 0;
    ps.done = !ps.inside;
    double csum[3] = {0.0, 0.0, 0.0}; // render (KIND 3): color_sum, rasterizer.hpp:224
    if constexpr (KIND == 1 || KIND == 3) {
        if (ps.inside) ps.out = p.pix_offset[ps.pixel];
    }
    uint32_t bits[MW];
    uint32_t grp = 0;
    if constexpr (KIND == 2 || KIND == 4) {
        bool any = false;
#pragma unroll
        for (int w = 0; w < MW; ++w) {
            bits[w] = ps.inside ? p.pix_bits[(size_t)ps.pixel * p.bits_stride + (p.mask_base >> 5) + w] : 0u;
            any |= bits[w] != 0;
        }
        grp = match_bits<MW>(bits);
        ps.done = ps.done || !any; // unmasked pixels contribute nothing
    }
    // the loop tests "still compositing" as the lane's bit (one LOP3 against
    // the staged splat's pixel mask); ps.done is not read below
    ps.lbit = ps.done ? 0u : 1u << lane;
    uint32_t first = start;
    if constexpr (RESUME) {
        // the saved list position and transmittance; pixels that were not
        // compositing at the end of the prefix saved nothing (NaN).  The slots
        // are reset for the next view (T back to NaN, the block's flag to 0).
        const uint32_t item = tile * 8u + wb;
        first = p.rs_state[item].y;
        double* tslot = p.rs_T + (size_t)item * 32u + lane;
        ps.T = *tslot;
        *tslot = __longlong_as_double(-1ll); // NaN
        if (!(ps.T >= 0.0)) ps.lbit = 0u;
        __syncwarp();
        if (lane == 0) p.rs_state[item].x = 0u;
    }

    // prefetch the first chunk's ranks and boxes
    uint32_t nr = 0;
    uint2 nbox = make_uint2(0u, 0u);
    if (first + lane < end) {
        nr = __ldg(p.tile_list + first + lane);
        nbox = __ldg(p.boxes + nr);
    }
    const uint32_t lane_bit = 1u << lane;
    uint32_t mg_addr = (uint32_t)__cvta_generic_to_shared(wmg);
    for (uint32_t base = first; base < end; base += 32u) {
        const uint32_t live = __ballot_sync(0xffffffffu, ps.lbit != 0u);
        if (live == 0u) break;
        const uint32_t i = base + lane;
        const uint32_t r = nr;
        const uint2 box = nbox;
        if (i + 32u < end) { // software prefetch of the next chunk
            nr = __ldg(p.tile_list + i + 32u);
            nbox = __ldg(p.boxes + nr);
        }
        const uint32_t sx0 = box.x & 0xffffu, sx1 = box.x >> 16, sy0 = box.y & 0xffffu, sy1 = box.y >> 16;
        // pixels of the block inside the box that are still compositing
        uint32_t m = 0u;
        if (i < end && !(sx1 < bx0 || sx0 > bx1 || sy1 < by0 || sy0 > by1))
            m = block_box_mask(sx0, sx1, sy0, sy1, bx0, by0) & live;
        const uint32_t cand = __ballot_sync(0xffffffffu, m != 0u);
        if (m) {
            const uint32_t slot = __popc(cand & (lane_bit - 1u));
            const uint4* src = reinterpret_cast<const uint4*>(p.rec + r);
            uint4* dst = reinterpret_cast<uint4*>(wrec + slot);
            dst[0] = __ldg(src);
            dst[1] = __ldg(src + 1);
            dst[2] = __ldg(src + 2);
            wmg[slot] = make_uint2(m, r);
        }
        __syncwarp();
        const uint32_t nh = __popc(cand);
        // running shared addresses of staged splat j's record and (mask, id);
        // the steps go in unrolled groups of 8 (constant offsets, one bound
        // test per step, the all-terminated vote once per group)
        uint32_t ra = srec_addr, ma = mg_addr;
        for (uint32_t j0 = 0; j0 < nh; j0 += 8u, ra += 8u * (uint32_t)sizeof(SplatRec), ma += 64u) {
            // keep the staging and exp-table addresses live instead of re-deriving
            // the shared window base for every splat
            asm volatile("" : "+r"(ra), "+r"(stab_addr), "+r"(ma));
#if SS_PIX_SMEM
            asm volatile("" : "+r"(pix_addr));
#endif
#pragma unroll
            for (uint32_t k = 0; k < 8u; ++k) {
                if (j0 + k >= nh) break;
                const StagedSplat s = lds_splat(ra + k * (uint32_t)sizeof(SplatRec));
                // staged splat j's pixel mask and id: one broadcast shared load
                uint32_t mj, gj;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(mj), "=r"(gj) : "r"(ma + 8u * k));
                float wf; // read only when c
                bool c = false;
                if (mj & ps.lbit) {
#if SS_PIX_SMEM
                    double dpx, dpy;
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(dpx), "=d"(dpy) : "r"(pix_addr));
                    c = composite_one<FALLOFF>(ps, dpx, dpy, s, stab_addr, wf);
#else
                    c = composite_one<FALLOFF>(ps, ps.dpx, ps.dpy, s, stab_addr, wf);
#endif
                }
                if constexpr (KIND == 0) {
                    ps.count += c ? 1u : 0u;
                } else if constexpr (KIND == 1 || KIND == 3) {
                    if (c) {
                        p.entries[ps.out++] = ss_weight_entry{gj, ps.pixel, wf};
                        ps.total = da(ps.total, (double)wf);
                        if constexpr (KIND == 3) {
                            // color_sum += double(wf) * color (rasterizer.hpp:231), per component
                            const float4 col = __ldg(p.color + gj);
                            csum[0] = da(csum[0], dm((double)wf, (double)col.x));
                            csum[1] = da(csum[1], dm((double)wf, (double)col.y));
                            csum[2] = da(csum[2], dm((double)wf, (double)col.z));
                        }
                    }
                } else {
                    gate_and_accumulate<MW, KIND == 4>(p, c, wf, grp, bits, gj, lane);
                }
            }
            if (__all_sync(0xffffffffu, ps.lbit == 0u)) break;
        }
        if constexpr ((KIND == 2 || KIND == 4) && !RESUME) {
            if (base + 32u >= end && p.tile_full && ps.lbit) {
                // this pixel is still compositing at the end of the list.  The
                // block is re-derived from the pixel; if the tile's list is only
                // a prefix, save the pixel's transmittance and queue the block
                // (first such lane) and its tile: it resumes after the fixup
                // sort completes the tile (raster_resume_kernel)
                double dpx, dpy;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(dpx), "=d"(dpy) : "r"(pix_addr));
                const uint32_t px = (uint32_t)dpx, py = (uint32_t)dpy;
                const uint32_t rt = (py / kTile) * p.tiles_x + px / kTile;
                const uint32_t item = rt * 8u + ((py % kTile) >> 2) * 2u + ((px % kTile) >> 3);
                if (end - p.tile_start[rt] < p.tile_full[rt]) {
                    p.rs_T[(size_t)item * 32u + (px & 7u) + 8u * (py & 3u)] = ps.T;
                    if (atomicExch(&p.rs_state[item].x, 1u) == 0u) {
                        p.rs_state[item].y = end;
                        p.rs_items[atomicAdd(p.rs_count, 1u)] = item;
                        if (atomicExch(p.rs_need + rt, 1u) == 0u) p.rs_tiles[atomicAdd(p.rs_count + 1, 1u)] = rt;
                    }
                }
            }
        }
        __syncwarp();
    }
    if (ps.inside) {
        if constexpr (KIND == 0) {
            p.pix_count[ps.pixel] = ps.count;
        } else if constexpr (KIND == 1 || KIND == 3) {
            p.per_pixel_total[ps.pixel] = __double2float_rn(ps.total);
            p.alpha[ps.pixel] = __double2float_rn(ds(1.0, ps.T));
            if constexpr (KIND == 3) {
                // rasterizer.hpp:236-243: normalised color, background kept below kRenderTotalEps
                if (ps.total > 1e-6) {
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        p.image[3ull * ps.pixel + k] = __double2float_rn(dd(csum[k], ps.total));
                }
            }
        }
    }
}

// One CTA (8 warps) per 16x16 tile, one thread per pixel.  Warp w owns the
// 8x4 block at (8*(w&1), 4*(w>>1)).  Each warp walks the tile's depth-ordered
// splat list independently, 32 entries at a time: one ballot culls the splats
// whose padded box misses the block, the hits are staged in the warp's
// shared-memory slice, and every lane composites its pixel against them front
// to back; the warp stops when all 32 of its pixels have terminated.  This
// shaping changes nothing in the arithmetic: every pixel still visits exactly
// the splats whose box contains it, in depth order.
//
// KIND 0: count contributions per pixel (sizes the capture).
// KIND 1: capture -- write WeightEntry records at per-pixel offsets, in depth
//         order (= the reference's stable_sort by pixel), per_pixel_total and
//         alpha = 1 - T_final.
// KIND 2: fused -- gate each contribution by the pixel's SAM-mask bitset and
//         add w into per-(Gaussian, mask) fp32 scalars (never a 512-d scatter).
//         One pass covers up to 128 masks (MW words); views with more masks
//         (providers.hpp:135 allows any count) run one pass per 128-mask
//         window [mask_base, mask_base + 128), each recompositing the tile.
template <int KIND, bool FALLOFF, int MW>
__global__ void __launch_bounds__(kRasterThreads, 6) raster_kernel(RasterParams p) {
    __shared__ SplatRec srec[kRasterThreads]; // warp w stages its hits in srec[32w, 32w+32)
    __shared__ uint2 smg[kRasterThreads];
    __shared__ unsigned long long stab[256];
    __shared__ double2 spix[SS_PIX_SMEM ? kRasterThreads : 1];
    stab[threadIdx.x] = kExpTab[threadIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    if (p.info->overflow) return; // tile lists incomplete: the view is re-run by the host
    __syncthreads();              // exp table staged
    composite_block<KIND, FALLOFF, MW>(p, blockIdx.x, warp, lane, srec + 32u * warp, smg + 32u * warp,
                                       (uint32_t)__cvta_generic_to_shared(srec + 32u * warp),
                                       (uint32_t)__cvta_generic_to_shared(stab),
                                       (uint32_t)__cvta_generic_to_shared(spix + (SS_PIX_SMEM ? 32u * warp : 0u)));
}

// Work-stealing form: a grid sized to the resident CTAs, each warp taking
// (tile, block) items from a counter until all tiles * 8 are done, so no warp
// idles while its CTA's other blocks finish and no CTA waits for a tail wave.
// Items go tile-major (the eight blocks of a tile run side by side and share
// the tile's list in L2).  work[0] is the item counter, work[1] counts warps
// out; the last warp resets both, so the next launch on the lane starts at 0.
template <int KIND, bool FALLOFF, int MW>
__global__ void __launch_bounds__(kRasterThreads, 6) raster_persist_kernel(RasterParams p) {
    __shared__ SplatRec srec[kRasterThreads];
    __shared__ uint2 smg[kRasterThreads];
    __shared__ unsigned long long stab[256];
    __shared__ double2 spix[SS_PIX_SMEM ? kRasterThreads : 1];
    stab[threadIdx.x] = kExpTab[threadIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    __syncthreads(); // exp table staged
    const uint32_t items = p.n_tiles * 8u;
    if (!p.info->overflow) { // else: tile lists incomplete, the view is re-run by the host
        for (;;) {
            uint32_t item = 0;
            if (lane == 0) item = atomicAdd(p.work, 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= items) break;
            composite_block<KIND, FALLOFF, MW>(p, item >> 3, item & 7u, lane, srec + 32u * warp, smg + 32u * warp,
                                               (uint32_t)__cvta_generic_to_shared(srec + 32u * warp),
                                               (uint32_t)__cvta_generic_to_shared(stab),
                                               (uint32_t)__cvta_generic_to_shared(spix + (SS_PIX_SMEM ? 32u * warp : 0u)));
        }
    }
    if (lane == 0 && atomicAdd(p.work + 1, 1u) == gridDim.x * (kRasterThreads / 32u) - 1u) {
        p.work[0] = 0u;
        p.work[1] = 0u;
    }
}

// The blocks a prefix-sorted fused pass saved (rs_items), after the fixup
// sort completed their tiles' lists: each warp takes items in turn and
// continues from the saved list position with the saved transmittance --
// the same front-to-back sequence per pixel as one uninterrupted walk.
template <int KIND, bool FALLOFF, int MW>
__global__ void __launch_bounds__(kRasterThreads, 6) raster_resume_kernel(RasterParams p) {
    __shared__ SplatRec srec[kRasterThreads];
    __shared__ uint2 smg[kRasterThreads];
    __shared__ unsigned long long stab[256];
    __shared__ double2 spix[SS_PIX_SMEM ? kRasterThreads : 1];
    stab[threadIdx.x] = kExpTab[threadIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    __syncthreads(); // exp table staged
    if (p.info->overflow) return;
    const uint32_t n_items = p.rs_count[0];
    for (uint32_t k = blockIdx.x * (kRasterThreads / 32u) + warp; k < n_items; k += gridDim.x * (kRasterThreads / 32u)) {
        const uint32_t item = p.rs_items[k];
        composite_block<KIND, FALLOFF, MW, true>(p, item >> 3, item & 7u, lane, srec + 32u * warp, smg + 32u * warp,
                                                 (uint32_t)__cvta_generic_to_shared(srec + 32u * warp),
                                                 (uint32_t)__cvta_generic_to_shared(stab),
                                                 (uint32_t)__cvta_generic_to_shared(spix + (SS_PIX_SMEM ? 32u * warp : 0u)));
    }
}

// ------------------------------------------------- staged-evaluation compositor
// Same tile / warp / block shaping and the same staging of 32 list entries as
// raster_kernel, but the per-(splat, pixel) work of a staged chunk is split by
// what depends on the transmittance:
//   A1  for each staged splat j (SIMT over the block's pixels): the box test
//       and d2 (rasterizer.hpp:115-121, fp64, reference order); the pairs with
//       d2 <= 9 are appended, j-major, to the warp's compact list (d2, j);
//   A2  dense over that list, all 32 lanes busy: g = exp(-d2/2) (glibc
//       restated) and alpha = min(0.99, o*g) (rasterizer.hpp:120-124) -- none
//       of it depends on T;
//   B   front to back over the staged splats with at least one such pair:
//       each pixel reads its alpha at off_j + rank, applies the skip rule,
//       w = alpha*T, the emission cutoff, T *= 1 - alpha and the floor
//       (rasterizer.hpp:125-131), then counts / captures / gates exactly as
//       raster_kernel.
// Every pixel still sees exactly its box's splats in depth order with the
// same operations, so the bits are raster_kernel's; the exp -- most of the
// fp64 work -- runs on full warps instead of the ~40 % of lanes a (splat,
// block) step keeps busy.  A list round holds <= kEvalCap pairs; a chunk with
// more is split into rounds (A1 stops before a splat could overflow it).
constexpr uint32_t kEvalCap = 256; // compacted (splat, pixel) evaluations per warp round

template <int KIND, bool FALLOFF, int MW>
__global__ void __launch_bounds__(kRasterThreads) raster_staged_kernel(RasterParams p) {
    __shared__ SplatRec srec[kRasterThreads]; // warp w stages its hits in srec[32w, 32w+32)
    __shared__ uint32_t sgid[kRasterThreads];
    __shared__ uint32_t smask[kRasterThreads];
    __shared__ double sval[kRasterThreads / 32][kEvalCap]; // d2, then alpha (or g: falloff)
    __shared__ uint8_t sjj[kRasterThreads / 32][kEvalCap];  // staged splat of each list entry
    __shared__ unsigned long long stab[256];
    stab[threadIdx.x] = kExpTab[threadIdx.x];

    const uint32_t tile = blockIdx.x;
    const uint32_t tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t bx0 = tx * kTile + 8u * (warp & 1u), by0 = ty * kTile + 4u * (warp >> 1);
    const uint32_t bx1 = bx0 + 7u, by1 = by0 + 3u;
    const uint32_t start = p.tile_start[tile], end = p.tile_end[tile];
    if (p.info->overflow) return; // tile lists incomplete: the view is re-run by the host
    const uint32_t wbase = 32u * warp;
    SplatRec* wrec = srec + wbase;
    const uint32_t srec_addr = (uint32_t)__cvta_generic_to_shared(wrec);
    uint32_t stab_addr = (uint32_t)__cvta_generic_to_shared(stab);
    uint32_t* wgid = sgid + wbase;
    uint32_t* wmask = smask + wbase;
    double* wval = sval[warp];
    uint8_t* wjj = sjj[warp];

    PixelState ps;
    ps.px = bx0 + (lane & 7u);
    ps.py = by0 + (lane >> 3);
    ps.inside = ps.px < p.width && ps.py < p.height;
    ps.pixel = ps.py * p.width + ps.px;
    ps.dpx = (double)(int32_t)ps.px;
    ps.dpy = (double)(int32_t)ps.py;
    ps.T = 1.0;
    ps.total = 0.0;
    ps.count = 0;
    ps.out = 0;
    ps.done = !ps.inside;
    double csum[3] = {0.0, 0.0, 0.0}; // render (KIND 3): color_sum, rasterizer.hpp:224
    if constexpr (KIND == 1 || KIND == 3) {
        if (ps.inside) ps.out = p.pix_offset[ps.pixel];
    }
    uint32_t bits[MW];
    uint32_t grp = 0;
    if constexpr (KIND == 2) {
        bool any = false;
#pragma unroll
        for (int w = 0; w < MW; ++w) {
            bits[w] = ps.inside ? p.pix_bits[(size_t)ps.pixel * p.bits_stride + (p.mask_base >> 5) + w] : 0u;
            any |= bits[w] != 0;
        }
        grp = match_bits<MW>(bits);
        ps.done = ps.done || !any; // unmasked pixels contribute nothing
    }
    __syncthreads(); // exp table staged

    uint32_t nr = 0;
    uint2 nbox = make_uint2(0u, 0u);
    if (start + lane < end) {
        nr = __ldg(p.tile_list + start + lane);
        nbox = __ldg(p.boxes + nr);
    }
    const uint32_t lane_bit = 1u << lane, below = lane_bit - 1u;
    bool finished = false;
    for (uint32_t base = start; base < end && !finished; base += 32u) {
        const uint32_t live = ~__ballot_sync(0xffffffffu, ps.done);
        if (live == 0u) break;
        const uint32_t i = base + lane;
        const uint32_t r = nr;
        const uint2 box = nbox;
        if (i + 32u < end) { // software prefetch of the next chunk
            nr = __ldg(p.tile_list + i + 32u);
            nbox = __ldg(p.boxes + nr);
        }
        const uint32_t sx0 = box.x & 0xffffu, sx1 = box.x >> 16, sy0 = box.y & 0xffffu, sy1 = box.y >> 16;
        uint32_t m = 0u;
        if (i < end && !(sx1 < bx0 || sx0 > bx1 || sy1 < by0 || sy0 > by1))
            m = block_box_mask(sx0, sx1, sy0, sy1, bx0, by0) & live;
        const uint32_t cand = __ballot_sync(0xffffffffu, m != 0u);
        if (m) {
            const uint32_t slot = __popc(cand & below);
            const uint4* src = reinterpret_cast<const uint4*>(p.rec + r);
            uint4* dst = reinterpret_cast<uint4*>(wrec + slot);
            dst[0] = __ldg(src);
            dst[1] = __ldg(src + 1);
            dst[2] = __ldg(src + 2);
            wgid[slot] = r;
            wmask[slot] = m;
        }
        __syncwarp();
        const uint32_t nh = __popc(cand);
        // staged splat j's pixel mask and id live in lane j's registers
        const uint32_t smk = lane < nh ? wmask[lane] : 0u;
        const uint32_t sgd = lane < nh ? wgid[lane] : 0u;
        for (uint32_t j0 = 0; j0 < nh && !finished;) {
            // ---- A1: box test + d2 for the staged splats j0.., compacted
            uint32_t ne = 0, e_reg = 0, off_reg = 0, j = j0;
            for (; j < nh && ne + 32u <= kEvalCap; ++j) {
                asm volatile("" : "+r"(stab_addr));
                const uint32_t mj = __shfl_sync(0xffffffffu, smk, j);
                bool pass = false;
                double d2 = 0.0;
                if ((mj & lane_bit) && !ps.done) {
                    const uint32_t a = srec_addr + j * (uint32_t)sizeof(SplatRec);
                    double mu_x, mu_y, ca, cb2, cc;
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(mu_x), "=d"(mu_y) : "r"(a));
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(ca), "=d"(cb2) : "r"(a));
                    asm volatile("ld.shared.f64 %0, [%1+32];" : "=d"(cc) : "r"(a));
                    const double dx = ds(ps.dpx, mu_x), dy = ds(ps.dpy, mu_y);
                    d2 = da(da(dm(dm(ca, dx), dx), dm(dm(cb2, dx), dy)), dm(dm(cc, dy), dy));
                    pass = !(d2 > kMahalanobisSqCutoff); // NaN continues, as in the reference
                }
                const uint32_t e = __ballot_sync(0xffffffffu, pass);
                if (pass) {
                    const uint32_t slot = ne + __popc(e & below);
                    wval[slot] = d2;
                    wjj[slot] = (uint8_t)j;
                }
                if (lane == j) {
                    e_reg = e;
                    off_reg = ne;
                }
                ne += __popc(e);
            }
            const uint32_t j1 = j;
            __syncwarp();
            // ---- A2: exp and alpha, dense over the list
            for (uint32_t k = lane; k < ne; k += 32u) {
                const double d2 = wval[k];
                const double g = glibc_exp_small(dm(-0.5, d2), stab_addr);
                if constexpr (FALLOFF) {
                    wval[k] = g;
                } else {
                    double o;
                    asm volatile("ld.shared.f64 %0, [%1+40];"
                                 : "=d"(o)
                                 : "r"(srec_addr + (uint32_t)wjj[k] * (uint32_t)sizeof(SplatRec)));
                    const double og = dm(o, g);
                    // std::min(kAlphaMax, og) (rasterizer.hpp:124): (og < max) ? og : max, NaN -> max
                    const double amax = kCompositeConst[0];
                    wval[k] = og < amax ? og : amax;
                }
            }
            __syncwarp();
            // ---- B: front to back over the splats with an evaluated pair
            uint32_t todo = __ballot_sync(0xffffffffu, e_reg != 0u);
            uint32_t steps = 0;
            while (todo) {
                const uint32_t jb = __ffs(todo) - 1u;
                todo &= todo - 1u;
                const uint32_t ej = __shfl_sync(0xffffffffu, e_reg, jb);
                const uint32_t oj = __shfl_sync(0xffffffffu, off_reg, jb);
                const uint32_t gj = __shfl_sync(0xffffffffu, sgd, jb);
                float wf = 0.0f;
                bool c = false;
                if ((ej & lane_bit) && !ps.done) {
                    const double v = wval[oj + __popc(ej & below)];
                    if constexpr (FALLOFF) {
                        if (v >= kWeightCutoff) {
                            wf = __double2float_rn(v);
                            c = true;
                        }
                    } else if (v >= kCompositeConst[1]) { // else: alpha < 1/255 skips, T untouched
                        const double w = dm(v, ps.T);
                        c = w >= kCompositeConst[2];
                        if (c) wf = __double2float_rn(w);
                        ps.T = dm(ps.T, ds(1.0, v));
                        if (ps.T < kCompositeConst[3]) ps.done = true;
                    }
                }
                if constexpr (KIND == 0) {
                    ps.count += c ? 1u : 0u;
                } else if constexpr (KIND == 1 || KIND == 3) {
                    if (c) {
                        p.entries[ps.out++] = ss_weight_entry{gj, ps.pixel, wf};
                        ps.total = da(ps.total, (double)wf);
                        if constexpr (KIND == 3) {
                            const float4 col = __ldg(p.color + gj);
                            csum[0] = da(csum[0], dm((double)wf, (double)col.x));
                            csum[1] = da(csum[1], dm((double)wf, (double)col.y));
                            csum[2] = da(csum[2], dm((double)wf, (double)col.z));
                        }
                    }
                } else {
                    gate_and_accumulate<MW, false>(p, c, wf, grp, bits, gj, lane);
                }
                if ((++steps & 7u) == 0u && __all_sync(0xffffffffu, ps.done)) {
                    finished = true;
                    break;
                }
            }
            if (__all_sync(0xffffffffu, ps.done)) finished = true;
            j0 = j1;
            __syncwarp();
        }
        __syncwarp();
    }
    if (ps.inside) {
        if constexpr (KIND == 0) {
            p.pix_count[ps.pixel] = ps.count;
        } else if constexpr (KIND == 1 || KIND == 3) {
            p.per_pixel_total[ps.pixel] = __double2float_rn(ps.total);
            p.alpha[ps.pixel] = __double2float_rn(ds(1.0, ps.T));
            if constexpr (KIND == 3) {
                if (ps.total > 1e-6) {
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        p.image[3ull * ps.pixel + k] = __double2float_rn(dd(csum[k], ps.total));
                }
            }
        }
    }
}

// CTAs of the work-stealing grid: 4 per SM (of the 6 that fit) leaves room for
// the other lanes' kernels; measured on 300 c4 views, 5 lanes: 3 per SM 1571,
// 4 per SM 1573-1580, 5 per SM 1552-1558, 6 per SM 1521-1529 views/s, against
// 1536 for the CTA-per-tile grid.  SS_RASTER_CTAS_PER_SM overrides (timing).
uint32_t persist_grid(uint32_t tiles) {
    static uint32_t per_sm = [] {
        const char* e = getenv("SS_RASTER_CTAS_PER_SM");
        const int v = e ? atoi(e) : 4;
        return (uint32_t)(v >= 1 && v <= 6 ? v : 4);
    }();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return std::min<uint32_t>(tiles, (uint32_t)sms * per_sm);
}

template <int KIND, bool FO, int MW>
void launch_per_step(const RasterParams& p, uint32_t tiles, cudaStream_t s) {
    if (p.algo == 2 && p.work) {
        RasterParams q = p;
        q.n_tiles = tiles;
        raster_persist_kernel<KIND, FO, MW><<<persist_grid(tiles), kRasterThreads, 0, s>>>(q);
    } else {
        raster_kernel<KIND, FO, MW><<<tiles, kRasterThreads, 0, s>>>(p);
    }
}

template <int KIND>
cudaError_t launch_raster(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s) {
    if (tiles == 0) return cudaSuccess;
    const bool fo = mode == SS_FALLOFF_ONLY;
    if (p.algo != 0) {
        if (fo) launch_per_step<KIND, true, 1>(p, tiles, s);
        else launch_per_step<KIND, false, 1>(p, tiles, s);
    } else {
        if (fo) raster_staged_kernel<KIND, true, 1><<<tiles, kRasterThreads, 0, s>>>(p);
        else raster_staged_kernel<KIND, false, 1><<<tiles, kRasterThreads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

} // namespace

namespace {
// fp64 pipe probe (the compositor's roofline denominator):
// eight independent DFMA chains per thread, every SM full.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, uint32_t iters) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (double)(threadIdx.x + 8 * k);
    const double m = 0.9999999, c = 1e-7;
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], m, c);
    }
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += a[k];
    if (sum == -1.0) out[0] = sum; // keeps the chains live
}
} // namespace

cudaError_t probe_fp64_rate(double* lane_ops_per_s) {
    int dev = 0, sms = 148;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t iters = 8192, blocks = (uint32_t)sms * 8u;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) { // first launch warms up
        cudaEventRecord(a);
        fp64_probe_kernel<<<blocks, 256>>>(nullptr, iters);
        cudaEventRecord(b);
        if ((e = cudaEventSynchronize(b)) != cudaSuccess) break;
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        const double rate = (double)blocks * 256.0 * 8.0 * iters / (ms * 1e-3);
        if (rep > 0 && rate > best) best = rate;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (e == cudaSuccess) e = cudaGetLastError();
    *lane_ops_per_s = best;
    return e;
}

cudaError_t launch_cov3d(const float4* scale, const float4* quat, uint64_t n, double* cov3, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cov3d_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scale, quat, n, cov3);
    return cudaGetLastError();
}

cudaError_t launch_project(const ProjectParams& p, cudaStream_t s) {
    if (p.n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((p.n + SS_PROJECT_THREADS - 1) / SS_PROJECT_THREADS);
    project_kernel<<<blocks, SS_PROJECT_THREADS, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_raster_count(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s) {
    return launch_raster<0>(p, mode, tiles, s);
}
cudaError_t launch_raster_capture(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s) {
    return launch_raster<1>(p, mode, tiles, s);
}
cudaError_t launch_raster_render(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s) {
    return launch_raster<3>(p, mode, tiles, s);
}

cudaError_t launch_raster_resume(const RasterParams& p, int mode, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool fo = mode == SS_FALLOFF_ONLY;
#define SS_RESUME(K, MWV)                                                         \
    do {                                                                          \
        if (fo) raster_resume_kernel<K, true, MWV><<<sms, kRasterThreads, 0, s>>>(p); \
        else raster_resume_kernel<K, false, MWV><<<sms, kRasterThreads, 0, s>>>(p);   \
    } while (0)
#define SS_RESUME_MW(MWV)                   \
    do {                                    \
        if (p.acc_fix) SS_RESUME(4, MWV);   \
        else SS_RESUME(2, MWV);             \
    } while (0)
    switch (p.mask_words) {
    case 1: SS_RESUME_MW(1); break;
    case 2: SS_RESUME_MW(2); break;
    case 3:
    case 4: SS_RESUME_MW(4); break;
    default: return cudaErrorInvalidValue;
    }
#undef SS_RESUME_MW
#undef SS_RESUME
    return cudaGetLastError();
}

cudaError_t launch_raster_fused(const RasterParams& p, int mode, uint32_t tiles, cudaStream_t s) {
    if (tiles == 0) return cudaSuccess;
    const bool fo = mode == SS_FALLOFF_ONLY;
#define SS_FUSED(MWV)                                                                       \
    do {                                                                                    \
        if (p.acc_fix) { /* fixed-point scalars: the per-step compositor, KIND 4 */         \
            if (fo) launch_per_step<4, true, MWV>(p, tiles, s);                             \
            else launch_per_step<4, false, MWV>(p, tiles, s);                               \
        } else if (p.algo != 0) {                                                           \
            if (fo) launch_per_step<2, true, MWV>(p, tiles, s);                             \
            else launch_per_step<2, false, MWV>(p, tiles, s);                               \
        } else {                                                                            \
            if (fo) raster_staged_kernel<2, true, MWV><<<tiles, kRasterThreads, 0, s>>>(p); \
            else raster_staged_kernel<2, false, MWV><<<tiles, kRasterThreads, 0, s>>>(p);   \
        }                                                                                   \
    } while (0)
    switch (p.mask_words) {
    case 1: SS_FUSED(1); break;
    case 2: SS_FUSED(2); break;
    case 3:
    case 4: SS_FUSED(4); break;
    default: return cudaErrorInvalidValue;
    }
#undef SS_FUSED
    return cudaGetLastError();
}

} // namespace ss
