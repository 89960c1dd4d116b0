// Group contraction on the 5th-generation tensor cores (pipeline.hpp:70-86
// accumulate, for a group of 2-3 consecutive views with D = 512 and <= 64
// masks each):
//
//   sums[g][n] += sum_j sum_m w_j[g][m] * CLIP_j[m][n]      (union rows g)
//   totals[g] += sum_j sum_m w_j[g][m]
//
// as one dense GEMM per 128-row tile of the group's union list: A = the
// members' per-(Gaussian, mask) scalars [128 x 64*members] (gathered from the
// acc rows, consumed and cleared), B = the members' CLIP rows [64*members x
// 512].  fp32 operands are carried as fp16 hi + lo pairs with power-of-two
// scales (rows of A per Gaussian, rows of B per mask) and multiplied as
// A_hi*B_hi + A_hi*B_lo + A_lo*B_hi with fp32 accumulation in TMEM: the
// dropped A_lo*B_lo and the split residuals are below 2^-21 of each product,
// far inside the path's 1e-4 tolerance.  The epilogue reads
// the accumulator back with tcgen05.ld and adds it, unscaled, into the rows.
//
// One persistent CTA per SM, warp-specialised:
//   warps 0-7  epilogue   (TMEM lane quarter w & 3, 128-column slice w >> 2 of each half)
//   warp  8    producer   (cp.async.bulk of the prepared B tiles from L2)
//   warp  9    MMA issuer (one thread, tcgen05.mma.cta_group::1.kind::f16)
//   warps 10-17 A builders (gather, split, swizzle; totals; acc cleared;
//               L2 prefetch of the next tile's scalars and this tile's rows)
// TMEM: 2 x 256 fp32 columns -- the output's two 256-wide halves, so the
// epilogue of one half overlaps the MMAs of the other.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "ss_kernels.cuh"

namespace ss {
namespace ctc {

constexpr uint32_t BM = 128;       // union rows per tile
constexpr uint32_t KB = 64;        // K per member (masks, zero-padded)
constexpr uint32_t NC = 128;       // N per MMA (one B tile)
constexpr uint32_t NCHUNKS = 4;    // 512 / NC
constexpr uint32_t UK = 16;        // UMMA K for kind::f16
constexpr uint32_t MAXM = 3;       // members
constexpr uint32_t TILE = BM * KB * 2;          // 16 KB: one 128 x 64 fp16 operand tile (= one B tile)
constexpr uint32_t A_BYTES = MAXM * 2 * TILE;   // hi + lo per member: 96 KB
constexpr uint32_t STAGE = 2 * TILE;            // B hi + lo of one (member, n-chunk): 32 KB
constexpr uint32_t STAGES = 3;
constexpr uint32_t EPI_WARPS = 8, BUILD_WARPS = 8;
constexpr uint32_t PROD_WARP = EPI_WARPS, MMA_WARP = EPI_WARPS + 1, BUILD0 = EPI_WARPS + 2;
constexpr uint32_t THREADS = 32 * (EPI_WARPS + 2 + BUILD_WARPS);
constexpr uint32_t META_BYTES = 2 * BM * 8;     // row gid + row 1/scale, double-buffered
constexpr uint32_t BAR_BYTES = 128;
constexpr size_t SMEM_BYTES = 1024 + A_BYTES + STAGES * STAGE + META_BYTES + MAXM * KB * 4 + BAR_BYTES;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t kNoRow = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled operand tile: 8-row atoms of 128 B, atoms 1024 B apart
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fffu);
    d |= (uint64_t)(16u >> 4) << 16;
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}
// byte offset of element (row r, k) in such a tile (fp16 elements, k < 64)
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t k) {
    return (r >> 3) * 1024u + (r & 7u) * 128u + ((((k >> 3) ^ (r & 7u)) & 7u) << 4) + (k & 7u) * 2u;
}
// kind::f16: D fp32, A/B fp16 K-major, M = 128, N = 128
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | ((NC >> 3) << 17) | ((BM >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(instr_desc()), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

#define CTC_TMEM_LD16(taddr, r)                                                                                      \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                                           \
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"                                   \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15])                                                                                     \
                 : "r"(taddr))

// power of two s with m * s in [2^14, 2^15) (1 for m == 0): keeps the fp16
// hi/lo split of every value of a row normal, far from overflow
__device__ __forceinline__ float pow2_scale(float m) {
    if (!(m > 0.0f)) return 1.0f;
    const int e = (int)((__float_as_uint(m) >> 23) & 0xffu); // biased exponent (0: subnormal)
    const int se = min(254, max(1, 268 - max(e, 1)));
    return __uint_as_float((uint32_t)se << 23);
}

// B for a group: per member j and n-chunk c, a 32 KB block [hi tile | lo tile]
// of CLIP_j^T * t_j (K-major: row n, k = mask), t_{j,m} = pow2_scale(max_n
// |CLIP_j[m][n]|); inv_t[j][m] = 1 / t_{j,m} (0 for padded masks).
__global__ void __launch_bounds__(128) prep_b_kernel(ContractParams p, unsigned char* bglob, float* inv_t) {
    const uint32_t j = blockIdx.y, m = blockIdx.x; // member, mask (< 64)
    const uint32_t M = j < p.n_members ? p.m[j].n_masks : 0u;
    const bool live = m < M;
    const float* row = live ? p.m[j].clip + (size_t)m * 512u : nullptr;
    float v[4];
    float mx = 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        v[q] = live ? row[threadIdx.x + 128u * q] : 0.0f;
        mx = fmaxf(mx, fabsf(v[q]));
    }
    __shared__ float wmax[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31u) == 0) wmax[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]));
    const float t = pow2_scale(mx);
    if (threadIdx.x == 0) inv_t[j * KB + m] = live ? 1.0f / t : 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t n = threadIdx.x + 128u * q;
        const float x = v[q] * t;
        const __half hi = __float2half_rn(x);
        const __half lo = __float2half_rn(x - __half2float(hi));
        unsigned char* blk = bglob + ((size_t)j * NCHUNKS + (n >> 7)) * STAGE;
        const uint32_t off = sw128_off(n & 127u, m);
        *reinterpret_cast<__half*>(blk + off) = hi;
        *reinterpret_cast<__half*>(blk + TILE + off) = lo;
    }
}

__global__ void __launch_bounds__(THREADS, 1) contract_tc_kernel(ContractParams p, const uint2* ulist,
                                                                 const unsigned int* ucount,
                                                                 const unsigned char* bglob, const float* inv_t_g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* a_tiles = smem;                       // [member][hi, lo] 16 KB tiles
    unsigned char* b_stages = smem + A_BYTES;            // [stage] hi | lo
    uint32_t* meta_gid = reinterpret_cast<uint32_t*>(b_stages + STAGES * STAGE); // [2][BM]
    float* meta_inv = reinterpret_cast<float*>(meta_gid + 2 * BM);                // [2][BM]
    float* inv_t = meta_inv + 2 * BM;                                             // [MAXM][KB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(inv_t + MAXM * KB);
    uint64_t* full = bars;              // [STAGES] B stage landed
    uint64_t* empty = bars + 3;         // [STAGES] MMAs done with the stage
    uint64_t* a_full = bars + 6;        // builders: A of the tile written
    uint64_t* a_empty = bars + 7;       // MMAs done with A
    uint64_t* tfull = bars + 8;         // [2] output half in TMEM
    uint64_t* tempty = bars + 10;       // [2] epilogue drained the half
    uint64_t* meta_free = bars + 12;    // [2] epilogue read the tile's row metadata
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t nm = p.n_members;
    const uint32_t total = *ucount;
    const uint32_t n_tiles = (total + BM - 1) / BM;

    for (uint32_t i = threadIdx.x; i < MAXM * KB; i += THREADS) inv_t[i] = inv_t_g[i];
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(a_full, BUILD_WARPS);
        mbar_init(a_empty, 1);
        for (uint32_t h = 0; h < 2; ++h) {
            mbar_init(tfull + h, 1);
            mbar_init(tempty + h, EPI_WARPS);
            mbar_init(meta_free + h, EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == PROD_WARP) {
        // ===== B stages: per tile, per output half, per member, per n-chunk of the half
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
                for (uint32_t h = 0; h < 2; ++h)
                    for (uint32_t j = 0; j < nm; ++j)
                        for (uint32_t c = 0; c < 2; ++c) {
                            mbar_wait(empty + s, ph ^ 1u);
                            mbar_expect_tx(full + s, STAGE);
                            bulk_g2s(b_stages + s * STAGE, bglob + ((size_t)j * NCHUNKS + 2 * h + c) * STAGE, STAGE,
                                     full + s);
                            if (++s == STAGES) {
                                s = 0;
                                ph ^= 1u;
                            }
                        }
        }
    } else if (warp == MMA_WARP) {
        // ===== MMA issuer
        if (lane == 0) {
            uint32_t s = 0, ph = 0, it = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
                mbar_wait(a_full, it & 1u);
                fence_after();
                for (uint32_t h = 0; h < 2; ++h) {
                    mbar_wait(tempty + h, (it & 1u) ^ 1u);
                    fence_after();
                    for (uint32_t j = 0; j < nm; ++j) {
                        const uint32_t ahi = smem_u32(a_tiles + (2 * j) * TILE), alo = ahi + TILE;
                        for (uint32_t c = 0; c < 2; ++c) {
                            mbar_wait(full + s, ph);
                            fence_after();
                            const uint32_t bhi = smem_u32(b_stages + s * STAGE), blo = bhi + TILE;
                            const uint32_t d = tmem_base + h * 256u + c * NC;
#pragma unroll
                            for (uint32_t k = 0; k < KB / UK; ++k) {
                                const uint32_t o = k * UK * 2u;
                                mma_f16(d, smem_desc(ahi + o), smem_desc(bhi + o), (j | k) != 0);
                                mma_f16(d, smem_desc(ahi + o), smem_desc(blo + o), 1u);
                                mma_f16(d, smem_desc(alo + o), smem_desc(bhi + o), 1u);
                            }
                            mma_commit(empty + s);
                            if (++s == STAGES) {
                                s = 0;
                                ph ^= 1u;
                            }
                        }
                    }
                    mma_commit(tfull + h);
                }
                mma_commit(a_empty);
            }
        }
    } else if (warp >= BUILD0) {
        // ===== A builders: warp b owns rows [16b, 16b + 16) of every tile, eight at a time
        constexpr uint32_t ROWS = BM / BUILD_WARPS, GR = 8;
        const uint32_t b = warp - BUILD0;
        unsigned long long pairs = 0;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
            const uint32_t buf = it & 1u;
            // lane l: the entry of row 32b + l of this tile; warm L2 with the next
            // tile's scalars (the next iteration's loads)
            const uint32_t e_mine = t * BM + b * ROWS + lane;
            const uint2 ent = lane < ROWS && e_mine < total ? ulist[e_mine] : make_uint2(kNoRow, 0u);
            {
                const uint32_t e_next = (t + gridDim.x) * BM + b * ROWS + lane;
                if (lane < ROWS && e_next < total) {
                    const uint2 nx = ulist[e_next];
                    for (uint32_t j = 0; j < nm; ++j)
                        if ((nx.y >> j) & 1u) {
                            const char* a = static_cast<const char*>(acc_row(p.m[j], nx.x).p);
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(a + 128));
                        }
                }
            }
            // this row's running total (read once per tile, written back after the tile)
            float tot_mine = ent.x != kNoRow ? p.totals[ent.x] : 0.0f, wsum_mine = 0.0f;
            mbar_wait(a_empty, (it & 1u) ^ 1u);
            mbar_wait(meta_free + buf, ((it >> 1) & 1u) ^ 1u);
            for (uint32_t rr = 0; rr < ROWS; rr += GR) {
                uint32_t gid[GR], mask[GR];
                float v[GR][MAXM][2];
#pragma unroll
                for (uint32_t q = 0; q < GR; ++q) {
                    gid[q] = __shfl_sync(0xffffffffu, ent.x, rr + q);
                    mask[q] = __shfl_sync(0xffffffffu, ent.y, rr + q);
#pragma unroll
                    for (uint32_t j = 0; j < MAXM; ++j) {
                        v[q][j][0] = v[q][j][1] = 0.0f;
                        if (j < nm && ((mask[q] >> j) & 1u)) {
                            const uint32_t M = p.m[j].n_masks;
                            const AccRow accrow = acc_row(p.m[j], gid[q]);
                            if (2u * lane < M) v[q][j][0] = accrow.get(2u * lane);
                            if (2u * lane + 1u < M) v[q][j][1] = accrow.get(2u * lane + 1u);
                        }
                    }
                }
#pragma unroll
                for (uint32_t q = 0; q < GR; ++q) {
                    const uint32_t r = b * ROWS + rr + q;
                    float wsum = 0.0f, mx = 0.0f;
#pragma unroll
                    for (uint32_t j = 0; j < MAXM; ++j) {
                        if (j < nm && ((mask[q] >> j) & 1u)) {
                            // consume and clear the member's scalars; totals in member order
                            const AccRow accrow = acc_row(p.m[j], gid[q]);
                            if (v[q][j][0] != 0.0f) accrow.clear(2u * lane);
                            if (v[q][j][1] != 0.0f) accrow.clear(2u * lane + 1u);
                            pairs += __popc(__ballot_sync(0xffffffffu, v[q][j][0] != 0.0f)) +
                                     __popc(__ballot_sync(0xffffffffu, v[q][j][1] != 0.0f));
                            float vs = v[q][j][0] + v[q][j][1];
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) vs += __shfl_xor_sync(0xffffffffu, vs, o);
                            wsum += vs;
                        }
                        v[q][j][0] *= inv_t[j * KB + 2u * lane];
                        v[q][j][1] *= inv_t[j * KB + 2u * lane + 1u];
                        mx = fmaxf(mx, fmaxf(fabsf(v[q][j][0]), fabsf(v[q][j][1])));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    const float sc = pow2_scale(mx);
                    const uint32_t off = sw128_off(r, 2u * lane);
#pragma unroll
                    for (uint32_t j = 0; j < MAXM; ++j) {
                        if (j >= nm) break;
                        const float x0 = v[q][j][0] * sc, x1 = v[q][j][1] * sc;
                        const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
                        const __half l0 = __float2half_rn(x0 - __half2float(h0));
                        const __half l1 = __float2half_rn(x1 - __half2float(h1));
                        *reinterpret_cast<__half2*>(a_tiles + (2 * j) * TILE + off) = __halves2half2(h0, h1);
                        *reinterpret_cast<__half2*>(a_tiles + (2 * j + 1) * TILE + off) = __halves2half2(l0, l1);
                    }
                    if (lane == 0) {
                        meta_gid[buf * BM + r] = gid[q];
                        meta_inv[buf * BM + r] = 1.0f / sc;
                    }
                    if (lane == rr + q) wsum_mine = wsum;
                }
            }
            if (ent.x != kNoRow) p.totals[ent.x] = tot_mine + wsum_mine;
            // generic-proxy smem writes -> visible to the tensor core's async proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full);
        }
        if (p.count_pairs && lane == 0) {
            // K_v pairs (warp-uniform ballot counts); G_v and the union rows once per group
            if (pairs) atomicAdd(p.cum + 1, pairs);
            if (blockIdx.x == 0 && b == 0) {
                unsigned long long all = 0;
                for (uint32_t i = 0; i < nm; ++i) all += *p.m[i].touched_count;
                atomicAdd(p.cum, all);
                atomicAdd(p.cum + 2, (unsigned long long)total);
            }
        }
    } else {
        // ===== epilogue: row 32*(w&3) + lane of the tile, columns [128*(w>>2), +128) of each half
        const uint32_t quarter = warp & 3u, cols = (warp >> 2) * 128u;
        const uint32_t r = quarter * 32u + lane;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
            const uint32_t buf = it & 1u;
            uint32_t gid = kNoRow;
            float inv = 1.0f;
            for (uint32_t h = 0; h < 2; ++h) {
                mbar_wait(tfull + h, it & 1u);
                fence_after();
                if (h == 0) {
                    gid = meta_gid[buf * BM + r];
                    inv = meta_inv[buf * BM + r];
                    __syncwarp();
                    if (lane == 0) mbar_arrive(meta_free + buf);
                }
                float* row = gid != kNoRow ? p.sums + (size_t)gid * 512u + h * 256u + cols : nullptr;
#pragma unroll 2
                for (uint32_t c = 0; c < 128u; c += 32u) {
                    uint32_t a[16], bq[16];
                    float4 cur[8];
                    const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + h * 256u + cols + c;
                    CTC_TMEM_LD16(taddr, a);
                    CTC_TMEM_LD16(taddr + 16u, bq);
                    if (row) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) cur[q] = reinterpret_cast<const float4*>(row + c)[q];
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (row) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            cur[q].x += __uint_as_float(a[4 * q]) * inv;
                            cur[q].y += __uint_as_float(a[4 * q + 1]) * inv;
                            cur[q].z += __uint_as_float(a[4 * q + 2]) * inv;
                            cur[q].w += __uint_as_float(a[4 * q + 3]) * inv;
                            cur[q + 4].x += __uint_as_float(bq[4 * q]) * inv;
                            cur[q + 4].y += __uint_as_float(bq[4 * q + 1]) * inv;
                            cur[q + 4].z += __uint_as_float(bq[4 * q + 2]) * inv;
                            cur[q + 4].w += __uint_as_float(bq[4 * q + 3]) * inv;
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) reinterpret_cast<float4*>(row + c)[q] = cur[q];
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + h);
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
}

} // namespace ctc

size_t contract_tc_scratch_bytes() { return (size_t)ctc::MAXM * ctc::NCHUNKS * ctc::STAGE + ctc::MAXM * ctc::KB * 4; }

bool contract_tc_eligible(const ContractParams& p) {
    if (p.n_members < 2 || p.n_members > ctc::MAXM || p.dim != 512 || !p.union_list) return false;
    for (uint32_t i = 0; i < p.n_members; ++i)
        if (p.m[i].n_masks == 0 || p.m[i].n_masks > ctc::KB) return false;
    return true;
}

// The union list (group_union_kernel) must be built; scratch holds the
// prepared B tiles and the per-mask scales (contract_tc_scratch_bytes()).
cudaError_t launch_contract_tc(const ContractParams& p, void* scratch, int ctas, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<int> configured[64] = {};
    if (dev >= 0 && dev < 64 && !configured[dev].load()) {
        cudaError_t e = cudaFuncSetAttribute(ctc::contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)ctc::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured[dev].store(1);
    }
    unsigned char* bglob = static_cast<unsigned char*>(scratch);
    float* inv_t = reinterpret_cast<float*>(bglob + (size_t)ctc::MAXM * ctc::NCHUNKS * ctc::STAGE);
    ctc::prep_b_kernel<<<dim3(ctc::KB, p.n_members), 128, 0, s>>>(p, bglob, inv_t);
    ctc::contract_tc_kernel<<<ctas, ctc::THREADS, ctc::SMEM_BYTES, s>>>(p, p.union_list, p.union_count, bglob, inv_t);
    return cudaGetLastError();
}

} // namespace ss
