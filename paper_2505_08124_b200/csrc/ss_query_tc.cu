// Cosine top-k over the vector store with the 5th-generation tensor cores
// (vecstore.hpp:121-132 query_topk, batched).
//
//   1. coarse scores  C[q][r] = fp16( sum_k fp16(Q[q][k]) * fp16(V[r][k]) )
//      tcgen05.mma kind::f16 (fp32 accumulation in TMEM), operands staged by
//      TMA in 128B-swizzled K-major tiles, persistent warp-specialised kernel:
//      warp 0 = TMA producer, warp 1 = single-thread MMA issuer, warps 2..5 =
//      epilogue (tcgen05.ld TMEM -> registers -> fp16 -> global).
//   2. per query: k-th largest coarse score c_k by a 4096-bin histogram of the
//      orderable fp16 key; candidates are all rows with c >= c_k - 2*eps
//      (eps bounds |coarse - exact|, see kCoarseEps) -- a superset of the
//      exact top-k, proven in DESIGN.md;
//   3. candidates are rescored with the exact 8-lane fp32 dot_lanes
//      (vecstore.hpp:21-31) and ordered by (sim desc, id asc)
//      (vecstore.hpp:107-110).  Ids and similarities are therefore exact.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "ss_query_tc.cuh"

namespace ss {
namespace tc {

// CTA pair (cta_group::2): the pair computes a 256-row x 256-query tile with
// M=256 MMAs issued by the leader.  Each CTA stages its own 128 store rows
// (A, streamed) and keeps its 128-query half of B resident in shared memory,
// so per 64-wide k-block a CTA receives 16 KB from L2 and the tensor core
// reads 64 B/clk of operands from each SM's shared memory -- half of what a
// single-CTA M=128 tile needs, which is what bounds the single-CTA kernel.
constexpr uint32_t BM = 128;        // store rows per CTA (pair: 256)
constexpr uint32_t BN = 256;        // queries per pair tile (UMMA N)
constexpr uint32_t BN_HALF = 128;   // resident B rows per CTA
constexpr uint32_t BK = 64;         // fp16 per 128-byte swizzle row
constexpr uint32_t UK = 16;         // UMMA K for kind::f16
constexpr uint32_t MAX_K = 512;     // resident B half: 128 queries x 512 fp16 = 128 KB
constexpr uint32_t STAGES = 5;
constexpr uint32_t A_BYTES = BM * BK * 2;         // 16 KB
constexpr uint32_t BKB_BYTES = BN_HALF * BK * 2;  // 16 KB per resident k-block of B
constexpr uint32_t B_RES_BYTES = (MAX_K / BK) * BKB_BYTES;
constexpr uint32_t ACC_STAGES = 2;
constexpr uint32_t TMEM_COLS = 512; // 2 x 256 fp32 accumulator columns
#ifndef SS_QTC_EPI_WARPS
#define SS_QTC_EPI_WARPS 8
#endif
constexpr uint32_t EPI_WARPS = SS_QTC_EPI_WARPS; // 4, 8 or 16: 1, 2 or 4 per TMEM lane quarter
constexpr uint32_t EPI_COLS = BN / (EPI_WARPS / 4);
#ifndef SS_QTC_EPI_ROUND
#define SS_QTC_EPI_ROUND 16
#endif
// TMEM columns per tcgen05.ld round (8, 16, 32 or 64).  Measured on B200 for
// the c5 query (GEMM only): 8 warps x16 1.63 ms, x8 1.70, x32 1.72, x64 1.90;
// 4 warps x16 2.00, 16 warps x16 1.75; no TMEM reads at all 1.48.
constexpr uint32_t EPI_ROUND = SS_QTC_EPI_ROUND;
static_assert(EPI_ROUND == 8 || EPI_ROUND == 16 || EPI_ROUND == 32, "SS_QTC_EPI_ROUND must be 8, 16 or 32");
constexpr uint32_t THREADS = 32 * (2 + EPI_WARPS);
constexpr uint32_t BAR_BYTES = 256;
constexpr uint32_t THR_SMEM = EPI_WARPS * EPI_COLS * 4; // per-warp copy of its thresholds
constexpr size_t SMEM_BYTES = 1024 + STAGES * A_BYTES + B_RES_BYTES + BAR_BYTES + THR_SMEM;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of this CTA's variable at `local` in CTA `rank`
__device__ __forceinline__ uint32_t map_to_rank(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// Arrive on the leader's barrier from either CTA.  Only tcgen05.ld results
// are being handed over (ordered by tcgen05.wait::ld + fence::before_thread_sync),
// so no cluster-scope release -- which would cost a GPU-wide MEMBAR per tile.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// pair TMA: data into this CTA's shared memory, completion to the leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int32_t x,
                                                 int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}

// K-major, 128B-swizzled operand tile: 8-row atoms of 128 B, atoms 1024 B apart
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fffu);      // start address
    d |= (uint64_t)(16u >> 4) << 16;             // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024u >> 4) << 32;           // stride byte offset: next 8-row atom
    d |= (uint64_t)1u << 46;                     // descriptor version (sm_100)
    d |= (uint64_t)2u << 61;                     // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: D fp32, A/B fp16, both K-major, M=256 (pair), N=256
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4)            // c_format = F32
           | (0u << 7)          // a_format = F16
           | (0u << 10)         // b_format = F16
           | ((BN >> 3) << 17)  // N >> 3
           | (((2 * BM) >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrives on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}

#define SS_TMEM_LD32(taddr, r)                                                                                       \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                           \
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                         \
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),      \
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),      \
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                           \
                 : "r"(taddr))

#define SS_TMEM_LD16(taddr, r)                                                                                       \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                                           \
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"                                   \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15])                                                                                     \
                 : "r"(taddr))

#define SS_TMEM_LD8(taddr, r)                                                                                        \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                           \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])  \
                 : "r"(taddr))

// ------------------------------------------------------------ coarse GEMM
// Tiles are (row tile, query tile) pairs, query tile fastest, so the
// q_tiles passes over one store tile run on neighbouring CTAs and share it
// through L2.  Row tiles visited: rt = i * rt_stride, i < row_tiles_iter.
//   PILOT: scores[q * ld + i*BM + r] = fp16 coarse score (rows past the store
//          are written as -inf so they never rank);
//   main:  rows with coarse >= thr[q] are appended to query q's candidates.
struct CoarseParams {
    uint32_t n_rows, n_queries, k_dim;
    uint32_t row_tiles_iter, rt_stride;
    __half* scores;
    uint64_t ld;
    const float* thr;
    uint32_t* cand;
    float* cand_val;
    uint32_t cand_cap;
    uint32_t* cand_count;
};

// Pair tile t (qt-major: t = qt * row_tiles_iter + it) covers store rows
// [rt*2BM, rt*2BM + 2BM) with rt = it * rt_stride (CTA r of the pair owns
// rows rt*2BM + r*BM + [0, BM)) and queries [qt*BN, qt*BN + BN) (CTA r keeps
// queries qt*BN + r*BN_HALF + [0, BN_HALF) resident).  With at most as many
// query tiles as pairs, each pair owns one query tile and a contiguous range
// of row tiles shared with the other query tiles' pairs; otherwise pair c of G
// runs the contiguous tile range [c*T/G, (c+1)*T/G).  TMEM of CTA r holds its BM rows x BN
// queries of the accumulator.
template <bool PILOT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    coarse_scores_kernel(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_q,
                         const CoarseParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stage_a = smem;
    unsigned char* b_res = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(b_res + B_RES_BYTES);
    uint64_t* full = bars;                       // [STAGES]   leader: both CTAs' A landed
    uint64_t* empty = bars + STAGES;             // [STAGES]   MMAs done with the slot (both CTAs)
    uint64_t* tfull = bars + 2 * STAGES;         // [ACC_STAGES] accumulator ready (both CTAs)
    uint64_t* tempty = tfull + ACC_STAGES;       // [ACC_STAGES] leader: both epilogues drained it
    uint64_t* bfull = tempty + ACC_STAGES;       // leader: both resident B halves loaded
    uint64_t* bempty = bfull + 1;                // MMAs done with the resident B (both CTAs)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 1);
    float* thr_smem = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bars) + BAR_BYTES);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t rank = cluster_rank();
    const uint32_t pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const uint32_t q_tiles = (p.n_queries + BN - 1) / BN;
    uint32_t t_begin, t_end;
    if (q_tiles <= n_pairs) {
        // pair -> (query tile, row group): the q_tiles pairs of a group walk the
        // same store rows side by side, so each store tile comes from HBM once
        // and from L2 for the other query tiles
        const uint32_t groups = n_pairs / q_tiles, qt = pair % q_tiles, grp = pair / q_tiles;
        const uint32_t rt_lo = grp < groups ? (uint32_t)((uint64_t)p.row_tiles_iter * grp / groups) : 0u;
        const uint32_t rt_hi = grp < groups ? (uint32_t)((uint64_t)p.row_tiles_iter * (grp + 1) / groups) : 0u;
        t_begin = qt * p.row_tiles_iter + rt_lo;
        t_end = qt * p.row_tiles_iter + rt_hi;
    } else {
        const uint64_t n_tiles = (uint64_t)p.row_tiles_iter * q_tiles;
        t_begin = (uint32_t)(n_tiles * pair / n_pairs);
        t_end = (uint32_t)(n_tiles * (pair + 1) / n_pairs);
    }
    const uint32_t k_blocks = p.k_dim / BK;

    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (uint32_t a = 0; a < ACC_STAGES; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 2 * EPI_WARPS); // one arrival per epilogue warp of either CTA
        }
        mbar_init(bfull, 1);
        mbar_init(bempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_v) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_q) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all(); // barriers of both CTAs initialised, TMEM allocated
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer (both CTAs; completions land on the leader's barriers)
        if (lane == 0) {
            const uint32_t full0 = map_to_rank(smem_u32(full), 0), bfull0 = map_to_rank(smem_u32(bfull), 0);
            uint32_t stage = 0, phase = 0, cur_qt = 0xffffffffu, be_phase = 0;
            for (uint32_t t = t_begin; t < t_end; ++t) {
                const uint32_t qt = t / p.row_tiles_iter, rt = (t % p.row_tiles_iter) * p.rt_stride;
                if (qt != cur_qt) {
                    if (cur_qt != 0xffffffffu) {
                        mbar_wait(bempty, be_phase);
                        be_phase ^= 1u;
                    }
                    if (rank == 0) mbar_expect_tx(bfull, 2 * k_blocks * BKB_BYTES);
                    for (uint32_t kb = 0; kb < k_blocks; ++kb)
                        tma_load_2d_pair(b_res + kb * BKB_BYTES, &map_q, bfull0, (int32_t)(kb * BK),
                                         (int32_t)(qt * BN + rank * BN_HALF));
                    cur_qt = qt;
                }
                for (uint32_t kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1u);
                    if (rank == 0) mbar_expect_tx(full + stage, 2 * A_BYTES);
                    tma_load_2d_pair(stage_a + stage * A_BYTES, &map_v, full0 + stage * 8, (int32_t)(kb * BK),
                                     (int32_t)((rt * 2 + rank) * BM));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA, one thread)
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = instr_desc();
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, cur_qt = 0xffffffffu, bf_phase = 0;
            for (uint32_t t = t_begin; t < t_end; ++t) {
                const uint32_t qt = t / p.row_tiles_iter;
                if (qt != cur_qt) {
                    if (cur_qt != 0xffffffffu) mma_commit(bempty); // fires once the old B's MMAs retire
                    mbar_wait(bfull, bf_phase);
                    bf_phase ^= 1u;
                    fence_after();
                    cur_qt = qt;
                }
                mbar_wait(tempty + acc, acc_phase ^ 1u);
                fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (uint32_t kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(full + stage, phase);
                    fence_after();
                    const uint32_t a0 = smem_u32(stage_a + stage * A_BYTES), b0 = smem_u32(b_res + kb * BKB_BYTES);
#pragma unroll
                    for (uint32_t k = 0; k < BK / UK; ++k)
                        mma_f16(d, smem_desc(a0 + k * UK * 2), smem_desc(b0 + k * UK * 2), idesc, (kb | k) != 0);
                    mma_commit(empty + stage); // frees the slot in both CTAs once these MMAs retire
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                mma_commit(tfull + acc); // accumulator ready for both epilogues
                if (++acc == ACC_STAGES) {
                    acc = 0;
                    acc_phase ^= 1u;
                }
            }
        }
    } else {
        // ===== epilogue: TMEM lane (= store row) per thread; warp w reads TMEM
        // lanes 32*(w%4) (the hardware's lane-quarter rule) and half of the
        // tile's query columns
        const uint32_t ew = warp - 2;
        const uint32_t quarter = warp & 3u;
        const uint32_t half = ew >> 2; // column slice [EPI_COLS*half, EPI_COLS*half + EPI_COLS)
        const uint32_t row_in_tile = rank * BM + quarter * 32u + lane;
        const uint32_t tempty0 = map_to_rank(smem_u32(tempty), 0);
        float* my_thr = thr_smem + ew * EPI_COLS;
        uint32_t acc = 0, acc_phase = 0, cur_qt = 0xffffffffu;
        for (uint32_t t = t_begin; t < t_end; ++t) {
            const uint32_t qt = t / p.row_tiles_iter, it = t % p.row_tiles_iter;
            const uint32_t row = it * p.rt_stride * (2 * BM) + row_in_tile;
            const uint32_t qbase = qt * BN + half * EPI_COLS;
            const bool row_ok = row < p.n_rows;
            if constexpr (!PILOT) {
                if (qt != cur_qt) {
                    __syncwarp();
#pragma unroll
                    for (uint32_t j = 0; j < EPI_COLS / 32; ++j) {
                        const uint32_t q = qbase + lane + 32u * j;
                        my_thr[lane + 32u * j] = q < p.n_queries ? __ldg(p.thr + q) : INFINITY;
                    }
                    __syncwarp();
                    cur_qt = qt;
                }
            }
            mbar_wait(tfull + acc, acc_phase);
            fence_after();
            // ROUND columns at a time; the accumulator goes back to the MMA warp
            // right after the last tcgen05.ld.  (tcgen05.ld shares TMEM
            // bandwidth with the MMAs accumulating the other stage: more
            // loads in flight slow the MMAs down more than they gain.)
#pragma unroll 1
            for (uint32_t c = 0; c < EPI_COLS; c += EPI_ROUND) {
                uint32_t r[EPI_ROUND];
                const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN + half * EPI_COLS + c;
                if constexpr (EPI_ROUND == 8) {
                    SS_TMEM_LD8(taddr, r);
                } else if constexpr (EPI_ROUND == 16) {
                    SS_TMEM_LD16(taddr, r);
                } else {
                    SS_TMEM_LD32(taddr, r);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c + EPI_ROUND >= EPI_COLS) {
                    fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (rank == 0) mbar_arrive(tempty + acc);
                        else mbar_arrive_remote(tempty0 + acc * 8);
                    }
                }
                if constexpr (PILOT) {
                    const uint64_t col = (uint64_t)it * (2 * BM) + row_in_tile;
#pragma unroll
                    for (uint32_t j = 0; j < EPI_ROUND; ++j) {
                        const uint32_t q = qbase + c + j;
                        if (q < p.n_queries)
                            p.scores[(uint64_t)q * p.ld + col] =
                                row_ok ? __float2half_rn(__uint_as_float(r[j])) : __ushort_as_half(0xfc00u);
                    }
                } else {
                    // branch-free screen: any column at or above its threshold?
                    const float4* t4 = reinterpret_cast<const float4*>(my_thr + c);
                    float mx = -INFINITY;
#pragma unroll
                    for (uint32_t j = 0; j < EPI_ROUND / 4; ++j) {
                        const float4 tv = t4[j];
                        mx = fmaxf(mx, fmaxf(fmaxf(__uint_as_float(r[4 * j]) - tv.x, __uint_as_float(r[4 * j + 1]) - tv.y),
                                             fmaxf(__uint_as_float(r[4 * j + 2]) - tv.z,
                                                   __uint_as_float(r[4 * j + 3]) - tv.w)));
                    }
                    if (row_ok && mx >= 0.0f) {
#pragma unroll
                        for (uint32_t j = 0; j < EPI_ROUND; ++j) {
                            const float v = __uint_as_float(r[j]);
                            if (v >= my_thr[c + j]) {
                                const uint32_t q = qbase + c + j;
                                const uint32_t slot = atomicAdd(p.cand_count + q, 1u);
                                if (slot < p.cand_cap) {
                                    p.cand[(uint64_t)q * p.cand_cap + slot] = row;
                                    p.cand_val[(uint64_t)q * p.cand_cap + slot] = v;
                                }
                            }
                        }
                    }
                }
            }
            if (++acc == ACC_STAGES) {
                acc = 0;
                acc_phase ^= 1u;
            }
        }
    }
    fence_before();
    cluster_sync_all(); // the pair's MMAs and remote arrivals are done
    fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
}

// ---------------------------------------------------------- selection
// fp16 -> u16 key increasing with the value
__device__ __forceinline__ uint32_t half_key(__half h) {
    const uint32_t b = __half_as_ushort(h);
    return (b & 0x8000u) ? (~b & 0xffffu) : (b | 0x8000u);
}
__device__ __forceinline__ float key_half(uint32_t key) {
    const uint32_t b = (key & 0x8000u) ? (key & 0x7fffu) : (~key & 0xffffu);
    return __half2float(__ushort_as_half((unsigned short)b));
}

// One CTA per query over the pilot's fp16 scores: a 4096-bin histogram of
// the top 12 bits of the orderable key finds the bin holding the sample's
// k-th largest coarse score c_k^S; thr = (that bin's lower edge) - 2*eps.
// The sample is a subset of the store, so the store's k-th largest coarse
// score c_k >= c_k^S, and every row of the exact top-k has
// coarse >= c_k - 2*eps >= thr ("query").
constexpr uint32_t SEL_THREADS = 1024;
constexpr uint32_t SEL_BINS = 4096;
__global__ void __launch_bounds__(SEL_THREADS) pilot_threshold_kernel(const __half* scores, uint64_t ld,
                                                                      uint32_t n_cols, uint32_t k, float eps2,
                                                                      float* thr) {
    __shared__ uint32_t hist[SEL_BINS];
    const uint32_t q = blockIdx.x;
    const __half* sc = scores + (uint64_t)q * ld;
    for (uint32_t i = threadIdx.x; i < SEL_BINS; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t nvec = n_cols / 8;
    const uint4* sv = reinterpret_cast<const uint4*>(sc);
    for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
        const uint4 pk = __ldg(sv + v);
        const __half* h = reinterpret_cast<const __half*>(&pk);
#pragma unroll
        for (int j = 0; j < 8; ++j) atomicAdd(hist + (half_key(h[j]) >> 4), 1u);
    }
    for (uint32_t r = nvec * 8 + threadIdx.x; r < n_cols; r += blockDim.x) atomicAdd(hist + (half_key(sc[r]) >> 4), 1u);
    __syncthreads();
    // bin of the k-th largest: warp 0 scans the bins from the top, 32 at a time
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint32_t above = 0, found = 0xffffffffu;
        for (int b0 = (int)SEL_BINS - 32; b0 >= 0 && found == 0xffffffffu; b0 -= 32) {
            const uint32_t b = (uint32_t)b0 + 31u - lane; // lane 0 = highest bin of the group
            uint32_t incl = hist[b];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            const uint32_t hit = __ballot_sync(0xffffffffu, above + incl >= k);
            if (hit) found = (uint32_t)b0 + 31u - (uint32_t)(__ffs(hit) - 1);
            above += __shfl_sync(0xffffffffu, incl, 31);
        }
        // NaN (or fewer than k sample rows) leaves no usable bound: every row is a candidate
        float t = -INFINITY;
        if (found != 0xffffffffu) {
            const float lo = key_half(found << 4);
            if (lo == lo) t = lo - eps2;
        }
        if (lane == 0) thr[q] = t;
    }
}

__device__ __forceinline__ bool scored_before(float sa, uint32_t ia, float sb, uint32_t ib) {
    if (sa != sb) return sa > sb; // vecstore.hpp:107-110
    return ia < ib;
}

// dot_lanes (vecstore.hpp:21-31) of store row `row` with the query held in
// shared memory, by a pair of threads (h = threadIdx.x & 1): thread h owns
// accumulators 4h..4h+3 and streams the row as float4 at 8i + 4h, 16 loads in
// flight; the pair combines ((l0+l1)+(l2+l3)) + ((l4+l5)+(l6+l7)), then adds
// the tail -- the literal 0.0f here, dim % 8 == 0.  Both threads return the sum.
__device__ __forceinline__ float pair_dot_lanes(const float* rows, uint32_t row, uint32_t dim, const float4* qs4,
                                                bool live) {
    const uint32_t h = threadIdx.x & 1u;
    const float4* a4 = reinterpret_cast<const float4*>(rows + (uint64_t)row * dim) + h;
    float l0 = 0.0f, l1 = 0.0f, l2 = 0.0f, l3 = 0.0f;
    if (live) {
        const uint32_t steps = dim / 8;
        for (uint32_t i0 = 0; i0 < steps; i0 += 16) {
            float4 av[16];
#pragma unroll
            for (uint32_t u = 0; u < 16; ++u)
                if (i0 + u < steps) av[u] = __ldg(a4 + 2 * (i0 + u));
#pragma unroll
            for (uint32_t u = 0; u < 16; ++u) {
                if (i0 + u < steps) {
                    const float4 bv = qs4[2 * (i0 + u) + h];
                    l0 = __fadd_rn(l0, __fmul_rn(av[u].x, bv.x));
                    l1 = __fadd_rn(l1, __fmul_rn(av[u].y, bv.y));
                    l2 = __fadd_rn(l2, __fmul_rn(av[u].z, bv.z));
                    l3 = __fadd_rn(l3, __fmul_rn(av[u].w, bv.w));
                }
            }
        }
    }
    const float half_sum = __fadd_rn(__fadd_rn(l0, l1), __fadd_rn(l2, l3)); // (s01+s23) or (s45+s67)
    const float other = __shfl_xor_sync(0xffffffffu, half_sum, 1);
    const float lo = h ? other : half_sum, hi = h ? half_sum : other;
    return __fadd_rn(__fadd_rn(lo, hi), 0.0f);
}

// One CTA per query.
//  1. c_k = the k-th largest fp32 coarse score among the candidates.  Every
//     row with coarse >= thr is a candidate and c_k >= thr, so this is the
//     store's exact k-th largest coarse score; the exact top-k lies in
//     {coarse >= c_k - 2*eps} ("query"), typically ~k rows.
//  2. those rows are rescored with the exact dot_lanes (vecstore.hpp:21-31:
//     eight fp32 lanes accumulated in index order with separately rounded
//     multiply and add, combined ((l0+l1)+(l2+l3)) + ((l4+l5)+(l6+l7)), then
//     the tail; dim % 8 == 0 here, so the tail is the literal 0.0f the
//     reference adds).  Two threads per row: thread h owns accumulators
//     4h..4h+3 and streams the row as float4 at 8i + 4h;
//  3. ranks under (sim desc, id asc) (vecstore.hpp:107-110) by counting in
//     shared memory; ranks < k are written.  Rows with equal (sim, id) --
//     duplicate ids in a user store -- are ordered by slot; their output
//     records are identical either way.
constexpr uint32_t RS_THREADS = 512;
__global__ void __launch_bounds__(RS_THREADS) rescore_kernel(const float* rows, const uint32_t* ids, uint32_t dim,
                                                             const float* qn, const uint32_t* cand,
                                                             const float* cand_val, uint32_t cand_cap,
                                                             uint32_t* cand_count, uint32_t k, float eps2,
                                                             uint32_t* out_ids, float* out_sims) {
    extern __shared__ float4 smem4[];
    float4* qs4 = smem4;                                           // dim / 4
    float* sval = reinterpret_cast<float*>(smem4 + dim / 4);       // cand_cap coarse scores
    uint32_t* srow = reinterpret_cast<uint32_t*>(sval + cand_cap); // cand_cap rows
    __shared__ uint32_t s_n;
    __shared__ float fsim[RS_THREADS / 2];
    __shared__ uint32_t fid[RS_THREADS / 2];
    const uint32_t q = blockIdx.x;
    const uint32_t nc = cand_count[q];
    if (nc > cand_cap) return; // overflow: the host answers this batch with the exact scan
    const float4* qv = reinterpret_cast<const float4*>(qn + (uint64_t)q * dim);
    for (uint32_t i = threadIdx.x; i < dim / 4; i += blockDim.x) qs4[i] = qv[i];
    const float* cv = cand_val + (uint64_t)q * cand_cap;
    const uint32_t* cq = cand + (uint64_t)q * cand_cap;
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
        sval[i] = cv[i];
        srow[i] = cq[i];
    }
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    // 1. k-th largest coarse score: min (as orderable key) over candidates
    //    with fewer than k strictly larger coarse scores
    const uint32_t kk = min(k, nc);
    __shared__ uint32_t s_key;
    if (threadIdx.x == 0) s_key = 0xffffffffu;
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
        const float v = sval[c];
        uint32_t gt = 0;
        for (uint32_t o = 0; o < nc; ++o) gt += sval[o] > v ? 1u : 0u;
        if (gt < kk) {
            const uint32_t b = __float_as_uint(v);
            atomicMin(&s_key, (b & 0x80000000u) ? ~b : (b | 0x80000000u));
        }
    }
    __syncthreads();
    const uint32_t kb = s_key;
    const float ck = __uint_as_float((kb & 0x80000000u) ? (kb & 0x7fffffffu) : ~kb);
    const float lim = ck - eps2;
    // 2. exact rescoring of the rows with coarse >= c_k - 2 eps, two threads per row
    uint32_t n_done = 0;
    for (uint32_t base = 0; base < nc; base += RS_THREADS / 2) {
        const uint32_t ci = base + (threadIdx.x >> 1);
        const bool live = ci < nc && sval[ci] >= lim;
        const uint32_t row = live ? srow[ci] : 0u;
        const float sim = pair_dot_lanes(rows, row, dim, qs4, live);
        if (live && (threadIdx.x & 1u) == 0) {
            const uint32_t slot = atomicAdd(&s_n, 1u);
            if (slot < RS_THREADS / 2) {
                fsim[slot] = isnan(sim) ? -INFINITY : sim;
                fid[slot] = __ldg(ids + row);
            }
        }
        __syncthreads();
        n_done = s_n;
        __syncthreads();
        if (n_done > RS_THREADS / 2) break;
    }
    if (n_done > RS_THREADS / 2) { // more finalists than slots: the host re-answers with the exact scan
        if (threadIdx.x == 0) cand_count[q] = 0xffffffffu;
        return;
    }
    // 3. ranks
    const uint32_t nf = n_done;
    const uint32_t take = min(k, nf);
    for (uint32_t c = threadIdx.x; c < nf; c += blockDim.x) {
        const float sc = fsim[c];
        const uint32_t ic = fid[c];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < nf; ++o) {
            const float so = fsim[o];
            const uint32_t io = fid[o];
            rank += (so > sc || (so == sc && (io < ic || (io == ic && o < c)))) ? 1u : 0u;
        }
        if (rank < take) {
            out_ids[(uint64_t)q * k + rank] = ic;
            out_sims[(uint64_t)q * k + rank] = sc;
        }
    }
}

// query_threshold (vecstore.hpp:135-146) for one query: every candidate of
// the coarse pass with thr = tau - eps (a superset of {exact >= tau}) is
// rescored with the exact dot_lanes; those with sim >= tau are ranked by
// (sim desc, id asc) in shared memory.  out_count gets the full count; at
// most out_cap records are written.
__global__ void __launch_bounds__(RS_THREADS) threshold_rescore_kernel(const float* rows, const uint32_t* ids,
                                                                       uint32_t dim, const float* qn,
                                                                       const uint32_t* cand, uint32_t cand_cap,
                                                                       const uint32_t* cand_count, float tau,
                                                                       uint32_t* out_ids, float* out_sims,
                                                                       uint64_t out_cap, uint32_t* out_count) {
    extern __shared__ float4 smem4[];
    float4* qs4 = smem4;                                          // dim / 4
    float* ksim = reinterpret_cast<float*>(smem4 + dim / 4);      // cand_cap
    uint32_t* kid = reinterpret_cast<uint32_t*>(ksim + cand_cap); // cand_cap
    __shared__ uint32_t s_n;
    const uint32_t nc = cand_count[0];
    if (nc > cand_cap) return; // overflow: the host answers with the exact scan
    const float4* qv = reinterpret_cast<const float4*>(qn);
    for (uint32_t i = threadIdx.x; i < dim / 4; i += blockDim.x) qs4[i] = qv[i];
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nc; base += RS_THREADS / 2) {
        const uint32_t ci = base + (threadIdx.x >> 1);
        const bool live = ci < nc;
        const uint32_t row = live ? __ldg(cand + ci) : 0u;
        const float sim = pair_dot_lanes(rows, row, dim, qs4, live);
        if (live && (threadIdx.x & 1u) == 0 && sim >= tau) {
            const uint32_t slot = atomicAdd(&s_n, 1u);
            ksim[slot] = sim;
            kid[slot] = __ldg(ids + row);
        }
    }
    __syncthreads();
    const uint32_t n = s_n;
    for (uint32_t c = threadIdx.x; c < n; c += blockDim.x) {
        const float sc = ksim[c];
        const uint32_t ic = kid[c];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < n; ++o) {
            const float so = ksim[o];
            const uint32_t io = kid[o];
            rank += (so > sc || (so == sc && (io < ic || (io == ic && o < c)))) ? 1u : 0u;
        }
        if (rank < out_cap) {
            out_ids[rank] = ic;
            out_sims[rank] = sc;
        }
    }
    if (threadIdx.x == 0) *out_count = n;
}

__global__ void to_half_kernel(const float* in, uint64_t n, __half* out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = __float2half_rn(in[i]);
}

} // namespace tc

// ------------------------------------------------------------------- host
namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t k, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {k, rows};
    const cuuint64_t strides[1] = {(cuuint64_t)k * 2};
    const cuuint32_t box[2] = {tc::BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
} // namespace

cudaError_t launch_to_half(const float* in, uint64_t n, void* out, cudaStream_t s) {
    if (!n) return cudaSuccess;
    tc::to_half_kernel<<<148 * 8, 256, 0, s>>>(in, n, static_cast<__half*>(out));
    return cudaGetLastError();
}

namespace {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember the
// largest size set for each (kernel, device) pair.  `done` is one array per
// kernel (kernels of the same function type must not share it).
using SmemDone = std::atomic<size_t>[64];
template <typename K>
cudaError_t ensure_smem(K kernel, size_t bytes, SmemDone& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (done[dev].load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[dev].store(bytes, std::memory_order_relaxed);
    return e;
}
} // namespace

namespace {
template <bool PILOT>
cudaError_t coarse_launch(const CUtensorMap& mv, const CUtensorMap& mq, const tc::CoarseParams& p, int num_sms,
                          cudaStream_t s) {
    static SmemDone done = {};
    cudaError_t e = ensure_smem(tc::coarse_scores_kernel<PILOT>, tc::SMEM_BYTES, done);
    if (e != cudaSuccess) return e;
    if (p.k_dim > tc::MAX_K) return cudaErrorInvalidValue;
    const uint64_t tiles = (uint64_t)p.row_tiles_iter * ((p.n_queries + tc::BN - 1) / tc::BN);
    const uint32_t grid = 2u * (uint32_t)std::min<uint64_t>(tiles, (uint64_t)(num_sms / 2));
    tc::coarse_scores_kernel<PILOT><<<grid, tc::THREADS, tc::SMEM_BYTES, s>>>(mv, mq, p);
    return cudaGetLastError();
}
} // namespace

uint32_t pilot_tiles(uint32_t n_rows) {
    const uint32_t row_tiles = (n_rows + 2 * tc::BM - 1) / (2 * tc::BM);
    return std::min<uint32_t>(row_tiles, kPilotTiles);
}

uint64_t pilot_cols(uint32_t n_rows) { return (uint64_t)pilot_tiles(n_rows) * 2 * tc::BM; }

cudaError_t launch_coarse_pilot(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                uint32_t k_dim, void* scores, int num_sms, cudaStream_t s) {
    if (k_dim % tc::BK != 0) return cudaErrorInvalidValue;
    CUtensorMap mv, mq;
    if (!make_map(&mv, v_half, n_rows, k_dim, tc::BM) || !make_map(&mq, q_half, n_queries, k_dim, tc::BN_HALF))
        return cudaErrorInvalidValue;
    const uint32_t row_tiles = (n_rows + 2 * tc::BM - 1) / (2 * tc::BM);
    tc::CoarseParams p{};
    p.n_rows = n_rows;
    p.n_queries = n_queries;
    p.k_dim = k_dim;
    p.row_tiles_iter = pilot_tiles(n_rows);
    p.rt_stride = row_tiles / p.row_tiles_iter;
    p.scores = static_cast<__half*>(scores);
    p.ld = pilot_cols(n_rows);
    return coarse_launch<true>(mv, mq, p, num_sms, s);
}

cudaError_t launch_pilot_threshold(const void* scores, uint32_t n_rows, uint32_t nq, uint32_t k, float eps2,
                                   float* thr, cudaStream_t s) {
    const uint64_t cols = pilot_cols(n_rows);
    tc::pilot_threshold_kernel<<<nq, tc::SEL_THREADS, 0, s>>>(static_cast<const __half*>(scores), cols,
                                                              (uint32_t)cols, k, eps2, thr);
    return cudaGetLastError();
}

cudaError_t launch_coarse_candidates(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                     uint32_t k_dim, const float* thr, uint32_t* cand, float* cand_val,
                                     uint32_t cand_cap, uint32_t* cand_count, int num_sms, cudaStream_t s) {
    if (k_dim % tc::BK != 0) return cudaErrorInvalidValue;
    CUtensorMap mv, mq;
    if (!make_map(&mv, v_half, n_rows, k_dim, tc::BM) || !make_map(&mq, q_half, n_queries, k_dim, tc::BN_HALF))
        return cudaErrorInvalidValue;
    tc::CoarseParams p{};
    p.n_rows = n_rows;
    p.n_queries = n_queries;
    p.k_dim = k_dim;
    p.row_tiles_iter = (n_rows + 2 * tc::BM - 1) / (2 * tc::BM);
    p.rt_stride = 1;
    p.thr = thr;
    p.cand = cand;
    p.cand_val = cand_val;
    p.cand_cap = cand_cap;
    p.cand_count = cand_count;
    return coarse_launch<false>(mv, mq, p, num_sms, s);
}

cudaError_t launch_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn, uint32_t nq,
                           const uint32_t* cand, const float* cand_val, uint32_t cand_cap, uint32_t* cand_count,
                           uint32_t k, float eps2, uint32_t* out_ids, float* out_sims, cudaStream_t s) {
    if (dim % 8 != 0) return cudaErrorInvalidValue;
    const size_t smem = (size_t)dim * 4 + (size_t)cand_cap * 8;
    static SmemDone done = {};
    cudaError_t e = ensure_smem(tc::rescore_kernel, smem, done);
    if (e != cudaSuccess) return e;
    tc::rescore_kernel<<<nq, tc::RS_THREADS, smem, s>>>(rows, ids, dim, qn, cand, cand_val, cand_cap, cand_count, k,
                                                        eps2, out_ids, out_sims);
    return cudaGetLastError();
}

cudaError_t launch_threshold_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn,
                                     const uint32_t* cand, uint32_t cand_cap, const uint32_t* cand_count, float tau,
                                     uint32_t* out_ids, float* out_sims, uint64_t out_cap, uint32_t* out_count,
                                     cudaStream_t s) {
    if (dim % 8 != 0) return cudaErrorInvalidValue;
    const size_t smem = (size_t)dim * 4 + (size_t)cand_cap * 8;
    static SmemDone done = {};
    cudaError_t e = ensure_smem(tc::threshold_rescore_kernel, smem, done);
    if (e != cudaSuccess) return e;
    tc::threshold_rescore_kernel<<<1, tc::RS_THREADS, smem, s>>>(rows, ids, dim, qn, cand, cand_cap, cand_count, tau,
                                                                 out_ids, out_sims, out_cap, out_count);
    return cudaGetLastError();
}

} // namespace ss
