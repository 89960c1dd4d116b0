/* oracle/ssoracle.c -- TEST INFRASTRUCTURE ONLY: the CPU restatement of the
 * reference's language-embedding path, used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Never linked
 * into, or called by, the product path (paper_2505_08124_b200/).
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/include/semsplat/...).  Arithmetic follows SURVEY.md
 * Appendix A with no FMA contraction (built with -ffp-contract=off), exactly
 * as the reference builds with plain -O3 for baseline x86-64.
 *
 * Parity pinning: this restatement is checked bit-for-bit against the
 * reference code itself compiled here (oracle/_ref/libssref.so, built from
 * the unmodified headers + oracle/eigen_shim) and against the golden vectors
 * in tests/golden/ generated from it.  At the Eigen boundary (covariance3d,
 * projection products) the bits are those of the shim's documented
 * evaluation order, since real Eigen is not available offline.
 *
 * exp(): the reference calls glibc's std::exp (rasterizer.hpp:85,120), an
 * ifunc that resolves to __exp_fma on FMA-capable x86.  sso_exp() restates
 * that routine (table-driven, 5-term polynomial, explicit fma()) -- verified
 * bit-identical to glibc 2.39 exp() on 2e8 inputs in [-4.5, 0].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef struct {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    uint32_t width, height, image_id, pad;
} sso_camera;

typedef struct {
    uint32_t gaussian_id;
    uint32_t visible;
    double mu_x, mu_y, cov_xx, cov_xy, cov_yy, depth;
} sso_projected;

typedef struct {
    uint32_t gaussian_id;
    uint32_t pixel;
    float weight;
} sso_entry;

/* constants: projection.hpp:15,17; rasterizer.hpp:17-30; pipeline.hpp:23 */
#define K_NEAR 0.01
#define K_DILATION 0.3
#define K_WEIGHT_CUTOFF (1.0 / 255.0)
#define K_ALPHA_MAX 0.99
#define K_ALPHA_SKIP (1.0 / 255.0)
#define K_T_FLOOR 1e-4
#define K_MAHA_CUTOFF 9.0
#define K_TILE 16u
#define K_COVERAGE_EPS 1e-8

/* ------------------------------------------------------------------ exp */
/* glibc sysdeps/ieee754/dbl-64/e_exp_data.c __exp_data.tab (N = 128):
   2^(k/N) ~= H[k]*(1+T[k]); tab[2k] = bits(T[k]), tab[2k+1] = bits(H[k]) - (k<<45).
   Values computed with 80-digit decimal arithmetic (tests/golden/make_golden.py
   re-derives them) and found byte-identical in this container's libm.so.6. */
static const uint64_t g_exp_tab[256] = {
    0x0000000000000000ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull, 0x3feff63da9fb3335ull,
    0xbc7160139cd8dc5dull, 0x3fefec9a3e778061ull, 0xbc905e7a108766d1ull, 0x3fefe315e86e7f85ull,
    0x3c8cd2523567f613ull, 0x3fefd9b0d3158574ull, 0xbc8bce8023f98efaull, 0x3fefd06b29ddf6deull,
    0x3c60f74e61e6c861ull, 0x3fefc74518759bc8ull, 0x3c90a3e45b33d399ull, 0x3fefbe3ecac6f383ull,
    0x3c979aa65d837b6dull, 0x3fefb5586cf9890full, 0x3c8eb51a92fdeffcull, 0x3fefac922b7247f7ull,
    0x3c3ebe3d702f9cd1ull, 0x3fefa3ec32d3d1a2ull, 0xbc6a033489906e0bull, 0x3fef9b66affed31bull,
    0xbc9556522a2fbd0eull, 0x3fef9301d0125b51ull, 0xbc5080ef8c4eea55ull, 0x3fef8abdc06c31ccull,
    0xbc91c923b9d5f416ull, 0x3fef829aaea92de0ull, 0x3c80d3e3e95c55afull, 0x3fef7a98c8a58e51ull,
    0xbc801b15eaa59348ull, 0x3fef72b83c7d517bull, 0xbc8f1ff055de323dull, 0x3fef6af9388c8deaull,
    0x3c8b898c3f1353bfull, 0x3fef635beb6fcb75ull, 0xbc96d99c7611eb26ull, 0x3fef5be084045cd4ull,
    0x3c9aecf73e3a2f60ull, 0x3fef54873168b9aaull, 0xbc8fe782cb86389dull, 0x3fef4d5022fcd91dull,
    0x3c8a6f4144a6c38dull, 0x3fef463b88628cd6ull, 0x3c807a05b0e4047dull, 0x3fef3f49917ddc96ull,
    0x3c968efde3a8a894ull, 0x3fef387a6e756238ull, 0x3c875e18f274487dull, 0x3fef31ce4fb2a63full,
    0x3c80472b981fe7f2ull, 0x3fef2b4565e27cddull, 0xbc96b87b3f71085eull, 0x3fef24dfe1f56381ull,
    0x3c82f7e16d09ab31ull, 0x3fef1e9df51fdee1ull, 0xbc3d219b1a6fbffaull, 0x3fef187fd0dad990ull,
    0x3c8b3782720c0ab4ull, 0x3fef1285a6e4030bull, 0x3c6e149289cecb8full, 0x3fef0cafa93e2f56ull,
    0x3c834d754db0abb6ull, 0x3fef06fe0a31b715ull, 0x3c864201e2ac744cull, 0x3fef0170fc4cd831ull,
    0x3c8fdd395dd3f84aull, 0x3feefc08b26416ffull, 0xbc86a3803b8e5b04ull, 0x3feef6c55f929ff1ull,
    0xbc924aedcc4b5068ull, 0x3feef1a7373aa9cbull, 0xbc9907f81b512d8eull, 0x3feeecae6d05d866ull,
    0xbc71d1e83e9436d2ull, 0x3feee7db34e59ff7ull, 0xbc991919b3ce1b15ull, 0x3feee32dc313a8e5ull,
    0x3c859f48a72a4c6dull, 0x3feedea64c123422ull, 0xbc9312607a28698aull, 0x3feeda4504ac801cull,
    0xbc58a78f4817895bull, 0x3feed60a21f72e2aull, 0xbc7c2c9b67499a1bull, 0x3feed1f5d950a897ull,
    0x3c4363ed60c2ac11ull, 0x3feece086061892dull, 0x3c9666093b0664efull, 0x3feeca41ed1d0057ull,
    0x3c6ecce1daa10379ull, 0x3feec6a2b5c13cd0ull, 0x3c93ff8e3f0f1230ull, 0x3feec32af0d7d3deull,
    0x3c7690cebb7aafb0ull, 0x3feebfdad5362a27ull, 0x3c931dbdeb54e077ull, 0x3feebcb299fddd0dull,
    0xbc8f94340071a38eull, 0x3feeb9b2769d2ca7ull, 0xbc87deccdc93a349ull, 0x3feeb6daa2cf6642ull,
    0xbc78dec6bd0f385full, 0x3feeb42b569d4f82ull, 0xbc861246ec7b5cf6ull, 0x3feeb1a4ca5d920full,
    0x3c93350518fdd78eull, 0x3feeaf4736b527daull, 0x3c7b98b72f8a9b05ull, 0x3feead12d497c7fdull,
    0x3c9063e1e21c5409ull, 0x3feeab07dd485429ull, 0x3c34c7855019c6eaull, 0x3feea9268a5946b7ull,
    0x3c9432e62b64c035ull, 0x3feea76f15ad2148ull, 0xbc8ce44a6199769full, 0x3feea5e1b976dc09ull,
    0xbc8c33c53bef4da8ull, 0x3feea47eb03a5585ull, 0xbc845378892be9aeull, 0x3feea34634ccc320ull,
    0xbc93cedd78565858ull, 0x3feea23882552225ull, 0x3c5710aa807e1964ull, 0x3feea155d44ca973ull,
    0xbc93b3efbf5e2228ull, 0x3feea09e667f3bcdull, 0xbc6a12ad8734b982ull, 0x3feea012750bdabfull,
    0xbc6367efb86da9eeull, 0x3fee9fb23c651a2full, 0xbc80dc3d54e08851ull, 0x3fee9f7df9519484ull,
    0xbc781f647e5a3ecfull, 0x3fee9f75e8ec5f74ull, 0xbc86ee4ac08b7db0ull, 0x3fee9f9a48a58174ull,
    0xbc8619321e55e68aull, 0x3fee9feb564267c9ull, 0x3c909ccb5e09d4d3ull, 0x3feea0694fde5d3full,
    0xbc7b32dcb94da51dull, 0x3feea11473eb0187ull, 0x3c94ecfd5467c06bull, 0x3feea1ed0130c132ull,
    0x3c65ebe1abd66c55ull, 0x3feea2f336cf4e62ull, 0xbc88a1c52fb3cf42ull, 0x3feea427543e1a12ull,
    0xbc9369b6f13b3734ull, 0x3feea589994cce13ull, 0xbc805e843a19ff1eull, 0x3feea71a4623c7adull,
    0xbc94d450d872576eull, 0x3feea8d99b4492edull, 0x3c90ad675b0e8a00ull, 0x3feeaac7d98a6699ull,
    0x3c8db72fc1f0eab4ull, 0x3feeace5422aa0dbull, 0xbc65b6609cc5e7ffull, 0x3feeaf3216b5448cull,
    0x3c7bf68359f35f44ull, 0x3feeb1ae99157736ull, 0xbc93091fa71e3d83ull, 0x3feeb45b0b91ffc6ull,
    0xbc5da9b88b6c1e29ull, 0x3feeb737b0cdc5e5ull, 0xbc6c23f97c90b959ull, 0x3feeba44cbc8520full,
    0xbc92434322f4f9aaull, 0x3feebd829fde4e50ull, 0xbc85ca6cd7668e4bull, 0x3feec0f170ca07baull,
    0x3c71affc2b91ce27ull, 0x3feec49182a3f090ull, 0x3c6dd235e10a73bbull, 0x3feec86319e32323ull,
    0xbc87c50422622263ull, 0x3feecc667b5de565ull, 0x3c8b1c86e3e231d5ull, 0x3feed09bec4a2d33ull,
    0xbc91bbd1d3bcbb15ull, 0x3feed503b23e255dull, 0x3c90cc319cee31d2ull, 0x3feed99e1330b358ull,
    0x3c8469846e735ab3ull, 0x3feede6b5579fdbfull, 0xbc82dfcd978e9db4ull, 0x3feee36bbfd3f37aull,
    0x3c8c1a7792cb3387ull, 0x3feee89f995ad3adull, 0xbc907b8f4ad1d9faull, 0x3feeee07298db666ull,
    0xbc55c3d956dcaebaull, 0x3feef3a2b84f15fbull, 0xbc90a40e3da6f640ull, 0x3feef9728de5593aull,
    0xbc68d6f438ad9334ull, 0x3feeff76f2fb5e47ull, 0xbc91eee26b588a35ull, 0x3fef05b030a1064aull,
    0x3c74ffd70a5fddcdull, 0x3fef0c1e904bc1d2ull, 0xbc91bdfbfa9298acull, 0x3fef12c25bd71e09ull,
    0x3c736eae30af0cb3ull, 0x3fef199bdd85529cull, 0x3c8ee3325c9ffd94ull, 0x3fef20ab5fffd07aull,
    0x3c84e08fd10959acull, 0x3fef27f12e57d14bull, 0x3c63cdaf384e1a67ull, 0x3fef2f6d9406e7b5ull,
    0x3c676b2c6c921968ull, 0x3fef3720dcef9069ull, 0xbc808a1883ccb5d2ull, 0x3fef3f0b555dc3faull,
    0xbc8fad5d3ffffa6full, 0x3fef472d4a07897cull, 0xbc900dae3875a949ull, 0x3fef4f87080d89f2ull,
    0x3c74a385a63d07a7ull, 0x3fef5818dcfba487ull, 0xbc82919e2040220full, 0x3fef60e316c98398ull,
    0x3c8e5a50d5c192acull, 0x3fef69e603db3285ull, 0x3c843a59ac016b4bull, 0x3fef7321f301b460ull,
    0xbc82d52107b43e1full, 0x3fef7c97337b9b5full, 0xbc892ab93b470dc9ull, 0x3fef864614f5a129ull,
    0x3c74b604603a88d3ull, 0x3fef902ee78b3ff6ull, 0x3c83c5ec519d7271ull, 0x3fef9a51fbc74c83ull,
    0xbc8ff7128fd391f0ull, 0x3fefa4afa2a490daull, 0xbc8dae98e223747dull, 0x3fefaf482d8e67f1ull,
    0x3c8ec3bc41aa2008ull, 0x3fefba1bee615a27ull, 0x3c842b94c3a9eb32ull, 0x3fefc52b376bba97ull,
    0x3c8a64a931d185eeull, 0x3fefd0765b6e4540ull, 0xbc8e37bae43be3edull, 0x3fefdbfdad9cbe14ull,
    0x3c77893b4d91cd9dull, 0x3fefe7c1819e90d8ull, 0x3c5305c14160cc89ull, 0x3feff3c22b8f71f1ull,
};
void sso_exp_table(uint64_t* out) { memcpy(out, g_exp_tab, sizeof(g_exp_tab)); }

static inline double asd(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}
static inline uint64_t asu(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}

/* glibc sysdeps/ieee754/dbl-64/e_exp.c as compiled into __exp_fma */
double sso_exp(double x) {
    static const double InvLn2N = 0x1.71547652b82fep0 * 128, Shift = 0x1.8p52,
                        NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47,
                        C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3, C4 = 0x1.55555cf172b91p-5,
                        C5 = 0x1.1111167a4d017p-7;
    const uint32_t abstop = (uint32_t)(asu(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x; /* |x| < 2^-54 */
        return exp(x);                                     /* |x| >= 512: not on this path */
    }
    double kd = fma(x, InvLn2N, Shift);
    const uint64_t ki = asu(kd);
    kd = kd - Shift;
    double r = fma(kd, NegLn2hiN, x);
    r = fma(kd, NegLn2loN, r);
    const uint64_t idx = 2 * (ki & 127), top = ki << 45;
    const double tail = asd(g_exp_tab[idx]);
    const uint64_t sbits = g_exp_tab[idx + 1] + top;
    const double r2 = r * r;
    const double tmp = fma(r2 * r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, tail + r));
    const double scale = asd(sbits);
    return fma(scale, tmp, scale);
}

/* ----------------------------------------------------------- projection */
/* scene.hpp:33-37 covariance3d + projection.hpp:33-55 project_gaussian,
   in SURVEY.md Appendix A order (steps 2-7). */
static void project_one(const float* mean, const float* scale, const float* q_xyzw, const sso_camera* cam,
                        uint32_t id, sso_projected* out) {
    memset(out, 0, sizeof(*out));
    out->gaussian_id = id;
    const double* Rc = cam->R;
    const double m0 = mean[0], m1 = mean[1], m2 = mean[2];
    double xc[3];
    for (int i = 0; i < 3; ++i) xc[i] = (Rc[3 * i] * m0 + (Rc[3 * i + 1] * m1 + Rc[3 * i + 2] * m2)) + cam->t[i];
    if (xc[2] <= K_NEAR) return;
    const double z = xc[2];
    out->mu_x = ((cam->fx * xc[0]) / z) + cam->cx;
    out->mu_y = ((cam->fy * xc[1]) / z) + cam->cy;
    out->depth = z;

    /* quaternion normalize: (x*x + z*z) + (y*y + w*w) */
    double qx = q_xyzw[0], qy = q_xyzw[1], qz = q_xyzw[2], qw = q_xyzw[3];
    const double n2 = (qx * qx + qz * qz) + (qy * qy + qw * qw);
    if (n2 > 0.0) {
        const double n = sqrt(n2);
        qx = qx / n;
        qy = qy / n;
        qz = qz / n;
        qw = qw / n;
    }
    const double tx = 2.0 * qx, ty = 2.0 * qy, tz = 2.0 * qz;
    const double twx = tx * qw, twy = ty * qw, twz = tz * qw;
    const double txx = tx * qx, txy = ty * qx, txz = tz * qx;
    const double tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
    double R[9];
    R[0] = 1.0 - (tyy + tzz);
    R[1] = txy - twz;
    R[2] = txz + twy;
    R[3] = txy + twz;
    R[4] = 1.0 - (txx + tzz);
    R[5] = tyz - twx;
    R[6] = txz - twy;
    R[7] = tyz + twx;
    R[8] = 1.0 - (txx + tyy);
    const double s0 = scale[0], s1 = scale[1], s2c = scale[2];
    const double s2[3] = {s0 * s0, s1 * s1, s2c * s2c};
    double S[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            S[3 * i + j] = (R[3 * i] * s2[0]) * R[3 * j] +
                           ((R[3 * i + 1] * s2[1]) * R[3 * j + 1] + (R[3 * i + 2] * s2[2]) * R[3 * j + 2]);

    const double J00 = cam->fx / z, J02 = ((-cam->fx) * xc[0]) / (z * z);
    const double J11 = cam->fy / z, J12 = ((-cam->fy) * xc[1]) / (z * z);
    double M[6];
    for (int j = 0; j < 3; ++j) {
        M[j] = (J00 * Rc[j] + 0.0 * Rc[3 + j]) + J02 * Rc[6 + j];
        M[3 + j] = (0.0 * Rc[j] + J11 * Rc[3 + j]) + J12 * Rc[6 + j];
    }
    double T[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            T[3 * i + j] = (M[3 * i] * S[j] + M[3 * i + 1] * S[3 + j]) + M[3 * i + 2] * S[6 + j];
    double C[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            C[2 * i + j] = (T[3 * i] * M[3 * j] + T[3 * i + 1] * M[3 * j + 1]) + T[3 * i + 2] * M[3 * j + 2];
    out->cov_xx = C[0] + K_DILATION;
    out->cov_xy = 0.5 * (C[1] + C[2]);
    out->cov_yy = C[3] + K_DILATION;
    out->visible = 1;
}

int sso_project(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity, uint64_t n,
                const sso_camera* cam, sso_projected* out) {
    (void)opacity;
    for (uint64_t k = 0; k < n; ++k)
        project_one(mean + 3 * k, scale + 3 * k, quat_xyzw + 4 * k, cam, (uint32_t)k, &out[k]);
    return 0;
}

/* projection.hpp:59-64 depth_sort: (depth asc, id asc) */
static int cmp_depth(const void* a, const void* b) {
    const sso_projected* p = (const sso_projected*)a;
    const sso_projected* q = (const sso_projected*)b;
    if (p->depth != q->depth) return p->depth < q->depth ? -1 : 1;
    return p->gaussian_id < q->gaussian_id ? -1 : (p->gaussian_id > q->gaussian_id);
}

/* x86 cvttsd2si: out of range or NaN -> INT32_MIN (rasterizer.hpp:173-176) */
static inline int32_t cvt_i32(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
    return (int32_t)v;
}

typedef struct {
    double a, b, c; /* conic */
    double mu_x, mu_y;
    double opacity;
    uint32_t gid;
    int32_t x0, x1, y0, y1;
} splat_t;

typedef struct {
    uint64_t n_entries;
    sso_entry* entries;
    float* per_pixel_total;
    float* alpha;
    /* binning products for tile-range parity */
    uint64_t n_splats;
    uint32_t* splat_gid;       /* depth-ordered, box-culled (the reference's `splats`) */
    uint32_t tiles;
    uint32_t* tile_offsets;    /* tiles + 1 */
    uint32_t* tile_splats;     /* concatenated splat indices per tile */
    int status;                /* 3 = NumericError */
    uint32_t bad_gid;
} sso_raster;

/* rasterizer.hpp:139-253 rasterize_impl (weights + alpha; color path unused
   on the embedding pass), emitting directly in (pixel, rank) order -- the
   order the reference reaches via stable_sort by pixel (:250-251). */
sso_raster* sso_rasterize(const float* mean, const float* scale, const float* quat_xyzw, const float* opacity,
                          uint64_t n, const sso_camera* cam, int mode) {
    sso_raster* r = (sso_raster*)calloc(1, sizeof(sso_raster));
    const uint32_t W = cam->width, H = cam->height;
    const uint64_t P = (uint64_t)W * H;
    r->per_pixel_total = (float*)calloc(P ? P : 1, sizeof(float));
    r->alpha = (float*)calloc(P ? P : 1, sizeof(float));

    sso_projected* proj = (sso_projected*)malloc((n ? n : 1) * sizeof(sso_projected));
    uint64_t nv = 0;
    for (uint64_t k = 0; k < n; ++k) {
        sso_projected p;
        project_one(mean + 3 * k, scale + 3 * k, quat_xyzw + 4 * k, cam, (uint32_t)k, &p);
        if (p.visible) proj[nv++] = p;
    }
    qsort(proj, nv, sizeof(sso_projected), cmp_depth);

    splat_t* splats = (splat_t*)malloc((nv ? nv : 1) * sizeof(splat_t));
    uint64_t ns = 0;
    for (uint64_t i = 0; i < nv; ++i) {
        const sso_projected* p = &proj[i];
        /* rasterizer.hpp:66-71 conic_of */
        const double det = p->cov_xx * p->cov_yy - p->cov_xy * p->cov_xy;
        if (det < 1e-12) {
            r->status = 3;
            r->bad_gid = p->gaussian_id;
            free(proj);
            free(splats);
            return r;
        }
        splat_t s;
        s.a = p->cov_yy / det;
        s.b = (-p->cov_xy) / det;
        s.c = p->cov_xx / det;
        s.mu_x = p->mu_x;
        s.mu_y = p->mu_y;
        s.opacity = (double)opacity[p->gaussian_id];
        s.gid = p->gaussian_id;
        const double rx = 3.0 * sqrt(p->cov_xx) + 1.0;
        const double ry = 3.0 * sqrt(p->cov_yy) + 1.0;
        int32_t v;
        v = cvt_i32(ceil(s.mu_x - rx));
        s.x0 = v > 0 ? v : 0;
        v = cvt_i32(floor(s.mu_x + rx));
        s.x1 = v < (int32_t)W - 1 ? v : (int32_t)W - 1;
        v = cvt_i32(ceil(s.mu_y - ry));
        s.y0 = v > 0 ? v : 0;
        v = cvt_i32(floor(s.mu_y + ry));
        s.y1 = v < (int32_t)H - 1 ? v : (int32_t)H - 1;
        if (s.x0 > s.x1 || s.y0 > s.y1) continue;
        splats[ns++] = s;
    }
    free(proj);
    r->n_splats = ns;
    r->splat_gid = (uint32_t*)malloc((ns ? ns : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < ns; ++i) r->splat_gid[i] = splats[i].gid;

    /* rasterizer.hpp:181-194 tile binning (counting pass + fill, same order) */
    const uint32_t tiles_x = (W + K_TILE - 1) / K_TILE, tiles_y = (H + K_TILE - 1) / K_TILE;
    const uint32_t tiles = tiles_x * tiles_y;
    r->tiles = tiles;
    r->tile_offsets = (uint32_t*)calloc(tiles + 1, sizeof(uint32_t));
    for (uint64_t i = 0; i < ns; ++i) {
        const splat_t* s = &splats[i];
        for (uint32_t ty = (uint32_t)s->y0 / K_TILE; ty <= (uint32_t)s->y1 / K_TILE; ++ty)
            for (uint32_t tx = (uint32_t)s->x0 / K_TILE; tx <= (uint32_t)s->x1 / K_TILE; ++tx)
                r->tile_offsets[ty * tiles_x + tx + 1]++;
    }
    for (uint32_t t = 0; t < tiles; ++t) r->tile_offsets[t + 1] += r->tile_offsets[t];
    const uint64_t inst = r->tile_offsets[tiles];
    r->tile_splats = (uint32_t*)malloc((inst ? inst : 1) * sizeof(uint32_t));
    uint32_t* fill = (uint32_t*)malloc((tiles ? tiles : 1) * sizeof(uint32_t));
    memcpy(fill, r->tile_offsets, tiles * sizeof(uint32_t));
    for (uint64_t i = 0; i < ns; ++i) {
        const splat_t* s = &splats[i];
        for (uint32_t ty = (uint32_t)s->y0 / K_TILE; ty <= (uint32_t)s->y1 / K_TILE; ++ty)
            for (uint32_t tx = (uint32_t)s->x0 / K_TILE; tx <= (uint32_t)s->x1 / K_TILE; ++tx)
                r->tile_splats[fill[ty * tiles_x + tx]++] = (uint32_t)i;
    }
    free(fill);

    /* rasterizer.hpp:112-133 composite_pixel per pixel, row-major pixel order */
    uint64_t cap = 1024, cnt = 0;
    sso_entry* ent = (sso_entry*)malloc(cap * sizeof(sso_entry));
    for (uint32_t y = 0; y < H; ++y) {
        for (uint32_t x = 0; x < W; ++x) {
            const uint32_t tile = (y / K_TILE) * tiles_x + x / K_TILE;
            const uint32_t pixel = y * W + x;
            double T = 1.0, total = 0.0;
            for (uint32_t b = r->tile_offsets[tile]; b < r->tile_offsets[tile + 1]; ++b) {
                const splat_t* s = &splats[r->tile_splats[b]];
                const int32_t px = (int32_t)x, py = (int32_t)y;
                if (px < s->x0 || px > s->x1 || py < s->y0 || py > s->y1) continue;
                const double dx = (double)px - s->mu_x, dy = (double)py - s->mu_y;
                const double d2 = ((s->a * dx) * dx + ((2.0 * s->b) * dx) * dy) + (s->c * dy) * dy;
                if (d2 > K_MAHA_CUTOFF) continue;
                const double g = sso_exp(-0.5 * d2);
                double w;
                int emit;
                if (mode == 0) {
                    const double og = s->opacity * g;
                    const double alpha = og < K_ALPHA_MAX ? og : K_ALPHA_MAX;
                    if (alpha < K_ALPHA_SKIP) continue;
                    w = alpha * T;
                    emit = w >= K_WEIGHT_CUTOFF;
                    if (emit) {
                        if (cnt == cap) {
                            cap *= 2;
                            ent = (sso_entry*)realloc(ent, cap * sizeof(sso_entry));
                        }
                        const float wf = (float)w;
                        ent[cnt].gaussian_id = s->gid;
                        ent[cnt].pixel = pixel;
                        ent[cnt].weight = wf;
                        ++cnt;
                        total += (double)wf;
                    }
                    T *= 1.0 - alpha;
                    if (T < K_T_FLOOR) break;
                } else {
                    if (g >= K_WEIGHT_CUTOFF) {
                        if (cnt == cap) {
                            cap *= 2;
                            ent = (sso_entry*)realloc(ent, cap * sizeof(sso_entry));
                        }
                        const float wf = (float)g;
                        ent[cnt].gaussian_id = s->gid;
                        ent[cnt].pixel = pixel;
                        ent[cnt].weight = wf;
                        ++cnt;
                        total += (double)wf;
                    }
                }
            }
            r->per_pixel_total[pixel] = (float)total;
            r->alpha[pixel] = (float)(1.0 - T);
        }
    }
    free(splats);
    r->entries = ent;
    r->n_entries = cnt;
    return r;
}

void sso_raster_free(sso_raster* r) {
    if (!r) return;
    free(r->entries);
    free(r->per_pixel_total);
    free(r->alpha);
    free(r->splat_gid);
    free(r->tile_offsets);
    free(r->tile_splats);
    free(r);
}

/* --------------------------------------------------------------- masks */
/* providers.hpp:95-109 rle_decode (zeros first); returns 0 ok, 4 FormatError */
int sso_rle_decode(const uint32_t* runs, uint64_t nruns, uint32_t w, uint32_t h, uint8_t* out) {
    const uint64_t total = (uint64_t)w * h;
    uint64_t pos = 0;
    uint8_t cur = 0;
    for (uint64_t i = 0; i < nruns; ++i) {
        if (pos + runs[i] > total) return 4;
        memset(out + pos, cur, runs[i]);
        pos += runs[i];
        cur ^= 1;
    }
    return pos == total ? 0 : 4;
}

/* providers.hpp:359-373 resample_mask (nearest neighbour, u64 index math) */
void sso_resample_mask(const uint8_t* in, uint32_t w, uint32_t h, uint32_t tw, uint32_t th, uint8_t* out) {
    if (w == tw && h == th) {
        memcpy(out, in, (size_t)w * h);
        return;
    }
    for (uint32_t y = 0; y < th; ++y) {
        uint32_t sy = (uint32_t)((2ull * y + 1) * h / (2ull * th));
        if (sy > h - 1) sy = h - 1;
        for (uint32_t x = 0; x < tw; ++x) {
            uint32_t sx = (uint32_t)((2ull * x + 1) * w / (2ull * tw));
            if (sx > w - 1) sx = w - 1;
            out[(size_t)y * tw + x] = in[(size_t)sy * w + sx];
        }
    }
}

/* pipeline.hpp:35-49 mask_weights: per-gid f64 sums over entries in entry
   order; dense scratch instead of unordered_map (same summation order per
   gid).  Outputs (gid, sum) sorted by gid (pipeline.hpp:46-47). */
static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}
uint64_t sso_mask_weights(const sso_entry* entries, uint64_t n_entries, const uint8_t* bits,
                          double* scratch /* n_gauss, zeroed; left zeroed */, uint8_t* seen /* n_gauss, zeroed */,
                          uint32_t* gids_out, double* sums_out) {
    uint64_t touched = 0;
    for (uint64_t i = 0; i < n_entries; ++i) {
        const sso_entry* e = &entries[i];
        if (!bits[e->pixel]) continue;
        if (!seen[e->gaussian_id]) {
            seen[e->gaussian_id] = 1;
            gids_out[touched++] = e->gaussian_id;
        }
        scratch[e->gaussian_id] += (double)e->weight;
    }
    qsort(gids_out, touched, sizeof(uint32_t), cmp_u32);
    for (uint64_t m = 0; m < touched; ++m) {
        const uint32_t g = gids_out[m];
        sums_out[m] = scratch[g];
        scratch[g] = 0.0;
        seen[g] = 0;
    }
    return touched;
}

/* ---------------------------------------------------------------- encode */
typedef struct {
    const float* mean;
    const float* scale;
    const float* quat;
    const float* opacity;
    uint64_t n;
    const sso_camera* cams; /* raster cameras (already camera_scaled_to) */
    uint32_t nviews;
    uint32_t mask_w, mask_h;
    const uint32_t* masks_per_view;    /* nviews */
    const uint64_t* view_mask_offset;  /* nviews+1, index into mask arrays */
    const uint32_t* runs;              /* all RLE runs */
    const uint64_t* run_offsets;       /* total_masks+1 */
    const float* clip;                 /* total_masks x dim */
    uint32_t dim;
    int mode;
} sso_encode_args;

/* pipeline.hpp:280-470 encode_scene with workers = 1 semantics: views in
   manifest order, masks in id order; accumulate (pipeline.hpp:70-80) in f64;
   finalize_into (pipeline.hpp:120-135).  Views [v_lo, v_hi) only when the
   caller wants a prefix; out_sum/out_total are the f64 PartialAccumulator. */
int sso_encode_partial(const sso_encode_args* a, uint32_t v_lo, uint32_t v_hi, double* sum, double* total) {
    const uint64_t n = a->n;
    const uint32_t D = a->dim;
    double* scratch = (double*)calloc(n ? n : 1, sizeof(double));
    uint8_t* seen = (uint8_t*)calloc(n ? n : 1, 1);
    uint32_t* gids = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    double* sums = (double*)malloc((n ? n : 1) * sizeof(double));
    const uint32_t mw = a->mask_w, mh = a->mask_h;
    uint8_t* mbits = (uint8_t*)malloc((size_t)mw * mh + 1);
    int status = 0;
    for (uint32_t v = v_lo; v < v_hi && status == 0; ++v) {
        const sso_camera* cam = &a->cams[v];
        const uint32_t W = cam->width, H = cam->height;
        uint8_t* rbits = (uint8_t*)malloc((size_t)W * H + 1);
        sso_raster* r = sso_rasterize(a->mean, a->scale, a->quat, a->opacity, n, cam, a->mode);
        if (r->status) {
            status = r->status;
            sso_raster_free(r);
            free(rbits);
            break;
        }
        const uint64_t m0 = a->view_mask_offset[v];
        for (uint32_t j = 0; j < a->masks_per_view[v]; ++j) {
            const uint64_t mi = m0 + j;
            const uint64_t r0 = a->run_offsets[mi], r1 = a->run_offsets[mi + 1];
            if (sso_rle_decode(a->runs + r0, r1 - r0, mw, mh, mbits)) {
                status = 4;
                break;
            }
            sso_resample_mask(mbits, mw, mh, W, H, rbits);
            const uint64_t k = sso_mask_weights(r->entries, r->n_entries, rbits, scratch, seen, gids, sums);
            const float* e = a->clip + mi * D;
            for (uint64_t t = 0; t < k; ++t) {
                double* row = sum + (uint64_t)gids[t] * D;
                const double w = sums[t];
                for (uint32_t d = 0; d < D; ++d) row[d] += w * (double)e[d];
                total[gids[t]] += w;
            }
        }
        sso_raster_free(r);
        free(rbits);
    }
    free(scratch);
    free(seen);
    free(gids);
    free(sums);
    free(mbits);
    return status;
}

/* pipeline.hpp:120-135 finalize_into */
void sso_finalize(const double* sum, const double* total, uint64_t n, uint32_t D, float* rows, float* coverage) {
    for (uint64_t k = 0; k < n; ++k) {
        if (total[k] > K_COVERAGE_EPS) {
            for (uint32_t d = 0; d < D; ++d) rows[k * D + d] = (float)(sum[k * D + d] / total[k]);
            coverage[k] = (float)total[k];
        } else {
            for (uint32_t d = 0; d < D; ++d) rows[k * D + d] = 0.0f;
            coverage[k] = 0.0f;
        }
    }
}

int sso_encode(const sso_encode_args* a, float* rows, float* coverage) {
    double* sum = (double*)calloc((a->n ? a->n : 1) * a->dim, sizeof(double));
    double* total = (double*)calloc(a->n ? a->n : 1, sizeof(double));
    if (!sum || !total) return 7;
    const int st = sso_encode_partial(a, 0, a->nviews, sum, total);
    if (st == 0) sso_finalize(sum, total, a->n, a->dim, rows, coverage);
    free(sum);
    free(total);
    return st;
}

/* ----------------------------------------------------------------- query */
/* vecstore.hpp:21-31 dot_lanes */
float sso_dot_lanes(const float* a, const float* b, uint64_t n) {
    float lanes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int l = 0; l < 8; ++l) lanes[l] += a[i + l] * b[i + l];
    float tail = 0.0f;
    for (; i < n; ++i) tail += a[i] * b[i];
    const float s01 = lanes[0] + lanes[1], s23 = lanes[2] + lanes[3];
    const float s45 = lanes[4] + lanes[5], s67 = lanes[6] + lanes[7];
    return ((s01 + s23) + (s45 + s67)) + tail;
}

/* vecstore.hpp:34-42 normalized_copy; returns 3 (NumericError) on zero norm */
int sso_normalized_copy(const float* v, uint64_t n, float* out) {
    double ns = 0.0;
    for (uint64_t i = 0; i < n; ++i) ns += (double)v[i] * v[i];
    if (!(ns > 0.0)) return 3;
    const double inv = 1.0 / sqrt(ns);
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)(v[i] * inv);
    return 0;
}

typedef struct {
    uint32_t id;
    float sim;
} scored_t;

/* vecstore.hpp:107-110 scored_before */
static inline int before(scored_t a, scored_t b) {
    if (a.sim != b.sim) return a.sim > b.sim;
    return a.id < b.id;
}

typedef struct {
    const uint32_t* ids;
    const float* rows;
    uint64_t count;
    uint32_t dim;
    const float* queries;
    uint32_t nq;
    uint64_t k;
    uint32_t* out_ids;
    float* out_sims;
    uint64_t* out_counts;
    uint32_t t, nt;
    int status;
} topk_job;

static void* topk_worker(void* arg) {
    topk_job* j = (topk_job*)arg;
    const uint64_t take = j->k < j->count ? j->k : j->count;
    scored_t* heap = (scored_t*)malloc((take + 1) * sizeof(scored_t));
    float* qn = (float*)malloc(j->dim * sizeof(float));
    for (uint32_t q = j->t; q < j->nq; q += j->nt) {
        if (j->k == 0 || j->count == 0) {
            j->out_counts[q] = 0;
            continue;
        }
        if (sso_normalized_copy(j->queries + (uint64_t)q * j->dim, j->dim, qn)) {
            j->status = 3;
            break;
        }
        /* keep the best `take` in a sorted array (insertion; take is small) */
        uint64_t have = 0;
        for (uint64_t i = 0; i < j->count; ++i) {
            scored_t s = {j->ids[i], sso_dot_lanes(j->rows + i * j->dim, qn, j->dim)};
            if (have == take && !before(s, heap[take - 1])) continue;
            uint64_t pos = have < take ? have : take - 1;
            while (pos > 0 && before(s, heap[pos - 1])) {
                heap[pos] = heap[pos - 1];
                --pos;
            }
            heap[pos] = s;
            if (have < take) ++have;
        }
        j->out_counts[q] = have;
        for (uint64_t i = 0; i < have; ++i) {
            j->out_ids[q * j->k + i] = heap[i].id;
            j->out_sims[q * j->k + i] = heap[i].sim;
        }
    }
    free(heap);
    free(qn);
    return NULL;
}

/* vecstore.hpp:121-132 query_topk, nq queries over `threads` pthreads */
int sso_query_topk(const uint32_t* ids, const float* rows, uint64_t count, uint32_t dim, const float* queries,
                   uint32_t nq, uint64_t k, uint32_t threads, uint32_t* out_ids, float* out_sims,
                   uint64_t* out_counts) {
    if (threads < 1) threads = 1;
    topk_job* jobs = (topk_job*)calloc(threads, sizeof(topk_job));
    pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
    for (uint32_t t = 0; t < threads; ++t) {
        jobs[t] = (topk_job){ids, rows, count, dim, queries, nq, k, out_ids, out_sims, out_counts, t, threads, 0};
        if (threads == 1) topk_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, topk_worker, &jobs[t]);
    }
    int st = 0;
    for (uint32_t t = 0; t < threads; ++t) {
        if (threads > 1) pthread_join(th[t], NULL);
        if (jobs[t].status) st = jobs[t].status;
    }
    free(jobs);
    free(th);
    return st;
}

static int cmp_scored(const void* a, const void* b) {
    const scored_t x = *(const scored_t*)a, y = *(const scored_t*)b;
    if (before(x, y)) return -1;
    if (before(y, x)) return 1;
    return 0;
}

/* vecstore.hpp:135-146 query_threshold: tau in [-1, 1] (ContractError = 1
 * otherwise), q normalised (NumericError = 3 on zero norm), every record with
 * sim >= tau, ordered by scored_before.  Writes min(n, capacity) records and
 * returns n in *out_count. */
int sso_query_threshold(const uint32_t* ids, const float* rows, uint64_t count, uint32_t dim, const float* query,
                        float tau, uint32_t* out_ids, float* out_sims, uint64_t capacity, uint64_t* out_count) {
    *out_count = 0;
    if (!(tau >= -1.0f && tau <= 1.0f)) return 1;
    if (count == 0) return 0; /* before prepare_query, as the reference */
    float* qn = (float*)malloc((dim ? dim : 1) * sizeof(float));
    if (sso_normalized_copy(query, dim, qn)) {
        free(qn);
        return 3;
    }
    scored_t* all = (scored_t*)malloc((count ? count : 1) * sizeof(scored_t));
    uint64_t n = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const float sim = sso_dot_lanes(rows + i * dim, qn, dim);
        if (sim >= tau) all[n++] = (scored_t){ids[i], sim};
    }
    qsort(all, n, sizeof(scored_t), cmp_scored);
    for (uint64_t i = 0; i < n && i < capacity; ++i) {
        out_ids[i] = all[i].id;
        out_sims[i] = all[i].sim;
    }
    *out_count = n;
    free(all);
    free(qn);
    return 0;
}

