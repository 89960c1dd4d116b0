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

#include "ss_query_tc.cuh"

namespace ss {
namespace tc {

constexpr uint32_t BM = 128;        // store rows per tile (UMMA M)
constexpr uint32_t BN = 256;        // queries per tile (UMMA N)
constexpr uint32_t BK = 64;         // fp16 per 128-byte swizzle row
constexpr uint32_t UK = 16;         // UMMA K for kind::f16
constexpr uint32_t STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2; // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2; // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t ACC_STAGES = 2;
constexpr uint32_t TMEM_COLS = 512; // 2 x 256 fp32 accumulator columns
constexpr uint32_t THREADS = 192;   // 6 warps
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;

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

// kind::f16 instruction descriptor: D fp32, A/B fp16, both K-major, M=128, N=256
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4)            // c_format = F32
           | (0u << 7)          // a_format = F16
           | (0u << 10)         // b_format = F16
           | ((BN >> 3) << 17)  // N >> 3
           | ((BM >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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

// ------------------------------------------------------------ coarse GEMM
// scores[q * ld + r] = fp16 coarse cosine of query q and store row r.
__global__ void __launch_bounds__(THREADS, 1)
    coarse_scores_kernel(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_q,
                         uint32_t n_rows, uint32_t n_queries, uint32_t k_dim, __half* scores, uint64_t ld) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stage_a = smem;
    unsigned char* stage_b = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;                       // [STAGES]
    uint64_t* empty = bars + STAGES;             // [STAGES]
    uint64_t* tfull = bars + 2 * STAGES;         // [ACC_STAGES]
    uint64_t* tempty = bars + 2 * STAGES + ACC_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * ACC_STAGES);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t row_tiles = (n_rows + BM - 1) / BM, q_tiles = (n_queries + BN - 1) / BN;
    const uint32_t n_tiles = row_tiles * q_tiles;
    const uint32_t k_blocks = k_dim / BK;

    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (uint32_t a = 0; a < ACC_STAGES; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 4); // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_v) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_q) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                // query tile fastest: a store tile is reused from L2 by the q_tiles passes
                const uint32_t rt = t / q_tiles, qt = t % q_tiles;
                for (uint32_t kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1u);
                    mbar_expect_tx(full + stage, STAGE_BYTES);
                    tma_load_2d(stage_a + stage * A_BYTES, &map_v, full + stage, (int32_t)(kb * BK),
                                (int32_t)(rt * BM));
                    tma_load_2d(stage_b + stage * B_BYTES, &map_q, full + stage, (int32_t)(kb * BK),
                                (int32_t)(qt * BN));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = instr_desc();
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                mbar_wait(tempty + acc, acc_phase ^ 1u);
                fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (uint32_t kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(full + stage, phase);
                    fence_after();
                    const uint32_t a0 = smem_u32(stage_a + stage * A_BYTES), b0 = smem_u32(stage_b + stage * B_BYTES);
#pragma unroll
                    for (uint32_t k = 0; k < BK / UK; ++k)
                        mma_f16(d, smem_desc(a0 + k * UK * 2), smem_desc(b0 + k * UK * 2), idesc, (kb | k) != 0);
                    mma_commit(empty + stage); // frees the smem slot once these MMAs retire
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                mma_commit(tfull + acc); // accumulator ready for the epilogue
                if (++acc == ACC_STAGES) {
                    acc = 0;
                    acc_phase ^= 1u;
                }
            }
        }
    } else {
        // ===== epilogue: TMEM lane (= store row) per thread, 256 query columns
        const uint32_t quarter = warp & 3u; // TMEM lanes 32*quarter .. +31 are this warp's
        const uint32_t row_in_tile = quarter * 32u + lane;
        uint32_t acc = 0, acc_phase = 0;
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            const uint32_t rt = t / q_tiles, qt = t % q_tiles;
            mbar_wait(tfull + acc, acc_phase);
            fence_after();
            const uint32_t row = rt * BM + row_in_tile;
            const uint32_t q0 = qt * BN;
#pragma unroll 1
            for (uint32_t c = 0; c < BN; c += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN + c;
                SS_TMEM_LD32(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (row < n_rows) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t q = q0 + c + (uint32_t)j;
                        if (q < n_queries) scores[(uint64_t)q * ld + row] = __float2half_rn(__uint_as_float(r[j]));
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
            if (++acc == ACC_STAGES) {
                acc = 0;
                acc_phase ^= 1u;
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
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

// One CTA per query.  Pass 1: 4096-bin histogram of the top 12 bits of the
// orderable fp16 key; the bin holding the k-th largest coarse score c_k gives
// a lower bound lo <= c_k.  Pass 2: every row with coarse >= lo - 2*eps is a
// candidate -- a superset of {c >= c_k - 2*eps}, which holds the exact top-k.
constexpr uint32_t SEL_THREADS = 1024;
constexpr uint32_t SEL_BINS = 4096;
__global__ void __launch_bounds__(SEL_THREADS) select_candidates_kernel(const __half* scores, uint64_t ld,
                                                                        uint32_t n_rows, uint32_t k, float eps2,
                                                                        uint32_t* cand, uint32_t cand_cap,
                                                                        uint32_t* cand_count) {
    __shared__ uint32_t hist[SEL_BINS];
    __shared__ uint32_t s_bin;
    __shared__ uint32_t s_count;
    const uint32_t q = blockIdx.x;
    const __half* sc = scores + (uint64_t)q * ld;
    for (uint32_t i = threadIdx.x; i < SEL_BINS; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const uint32_t nvec = n_rows / 8;
    const uint4* sv = reinterpret_cast<const uint4*>(sc);
    for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
        const uint4 pk = __ldg(sv + v);
        const __half* h = reinterpret_cast<const __half*>(&pk);
#pragma unroll
        for (int j = 0; j < 8; ++j) atomicAdd(hist + (half_key(h[j]) >> 4), 1u);
    }
    for (uint32_t r = nvec * 8 + threadIdx.x; r < n_rows; r += blockDim.x) atomicAdd(hist + (half_key(sc[r]) >> 4), 1u);
    __syncthreads();
    // bin of the k-th largest: warp 0 scans the bins from the top, 32 at a time
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint32_t above = 0, found = 0xffffffffu;
        for (int b0 = (int)SEL_BINS - 32; b0 >= 0 && found == 0xffffffffu; b0 -= 32) {
            const uint32_t b = (uint32_t)b0 + 31u - lane; // lane 0 = highest bin of the group
            const uint32_t h = hist[b];
            uint32_t incl = h;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            const uint32_t hit = __ballot_sync(0xffffffffu, above + incl >= k);
            if (hit) found = (uint32_t)b0 + 31u - (uint32_t)(__ffs(hit) - 1);
            above += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_bin = found;
    }
    __syncthreads();
    const float thr = s_bin == 0xffffffffu ? -INFINITY : key_half(s_bin << 4) - eps2;
    uint32_t* out = cand + (uint64_t)q * cand_cap;
    for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
        const uint4 pk = __ldg(sv + v);
        const __half* h = reinterpret_cast<const __half*>(&pk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (__half2float(h[j]) >= thr) {
                const uint32_t slot = atomicAdd(&s_count, 1u);
                if (slot < cand_cap) out[slot] = v * 8u + (uint32_t)j;
            }
        }
    }
    for (uint32_t r = nvec * 8 + threadIdx.x; r < n_rows; r += blockDim.x) {
        if (__half2float(sc[r]) >= thr) {
            const uint32_t slot = atomicAdd(&s_count, 1u);
            if (slot < cand_cap) out[slot] = r;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cand_count[q] = s_count;
}

__device__ __forceinline__ bool scored_before(float sa, uint32_t ia, float sb, uint32_t ib) {
    if (sa != sb) return sa > sb; // vecstore.hpp:107-110
    return ia < ib;
}

// One warp per query: exact dot_lanes of every candidate (vecstore.hpp:21-31:
// eight fp32 lanes, separate rounded multiply and add, pairwise combine),
// then (sim desc, id asc) selection of the first k.
__global__ void __launch_bounds__(256) rescore_kernel(const float* rows, const uint32_t* ids, uint32_t dim,
                                                      const float* qn, uint32_t nq, const uint32_t* cand,
                                                      uint32_t cand_cap, const uint32_t* cand_count, uint32_t k,
                                                      float* cand_sim, uint32_t* out_ids, float* out_sims) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (q >= nq) return;
    const uint32_t nc = cand_count[q];
    if (nc > cand_cap) return; // overflow: the host answers this batch with the exact scan
    const uint32_t* cq = cand + (uint64_t)q * cand_cap;
    float* sq = cand_sim + (uint64_t)q * cand_cap;
    const float* qv = qn + (uint64_t)q * dim;
    for (uint32_t c = lane; c < nc; c += 32) {
        const float* a = rows + (uint64_t)cq[c] * dim;
        float l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t i = 0;
        for (; i + 8 <= dim; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) l[j] = __fadd_rn(l[j], __fmul_rn(a[i + j], qv[i + j]));
        float tail = 0.0f;
        for (; i < dim; ++i) tail = __fadd_rn(tail, __fmul_rn(a[i], qv[i]));
        const float s01 = __fadd_rn(l[0], l[1]), s23 = __fadd_rn(l[2], l[3]);
        const float s45 = __fadd_rn(l[4], l[5]), s67 = __fadd_rn(l[6], l[7]);
        sq[c] = __fadd_rn(__fadd_rn(__fadd_rn(s01, s23), __fadd_rn(s45, s67)), tail);
    }
    __syncwarp();
    // k rounds of warp arg-max by (sim desc, id asc); candidates are few
    const uint32_t take = min(k, nc);
    for (uint32_t o = 0; o < take; ++o) {
        float bs = -INFINITY;
        uint32_t bi = 0xffffffffu, bc = 0xffffffffu;
        for (uint32_t c = lane; c < nc; c += 32) {
            const float s = sq[c];
            const uint32_t id = ids[cq[c]];
            if (!isnan(s) && (bc == 0xffffffffu || scored_before(s, id, bs, bi))) {
                bs = s;
                bi = id;
                bc = c;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float os = __shfl_xor_sync(0xffffffffu, bs, off);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            const uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, off);
            if (oc != 0xffffffffu && (bc == 0xffffffffu || scored_before(os, oi, bs, bi))) {
                bs = os;
                bi = oi;
                bc = oc;
            }
        }
        if (lane == 0) {
            out_ids[(uint64_t)q * k + o] = bi;
            out_sims[(uint64_t)q * k + o] = bs;
            sq[bc] = NAN; // taken
        }
        __syncwarp();
    }
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

size_t tc_scores_smem() { return tc::SMEM_BYTES; }

cudaError_t launch_to_half(const float* in, uint64_t n, void* out, cudaStream_t s) {
    if (!n) return cudaSuccess;
    tc::to_half_kernel<<<148 * 8, 256, 0, s>>>(in, n, static_cast<__half*>(out));
    return cudaGetLastError();
}

cudaError_t launch_coarse_scores(const void* v_half, uint32_t n_rows, const void* q_half, uint32_t n_queries,
                                 uint32_t k_dim, void* scores, uint64_t ld, int num_sms, cudaStream_t s) {
    if (k_dim % tc::BK != 0) return cudaErrorInvalidValue;
    CUtensorMap mv, mq;
    if (!make_map(&mv, v_half, n_rows, k_dim, tc::BM) || !make_map(&mq, q_half, n_queries, k_dim, tc::BN))
        return cudaErrorInvalidValue;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tc::coarse_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)tc::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const uint32_t tiles = ((n_rows + tc::BM - 1) / tc::BM) * ((n_queries + tc::BN - 1) / tc::BN);
    const uint32_t grid = std::min<uint32_t>(tiles, (uint32_t)num_sms);
    tc::coarse_scores_kernel<<<grid, tc::THREADS, tc::SMEM_BYTES, s>>>(mv, mq, n_rows, n_queries, k_dim,
                                                                       static_cast<__half*>(scores), ld);
    return cudaGetLastError();
}

cudaError_t launch_select_candidates(const void* scores, uint64_t ld, uint32_t n_rows, uint32_t nq, uint32_t k,
                                     float eps2, uint32_t* cand, uint32_t cand_cap, uint32_t* cand_count,
                                     cudaStream_t s) {
    tc::select_candidates_kernel<<<nq, tc::SEL_THREADS, 0, s>>>(static_cast<const __half*>(scores), ld, n_rows, k,
                                                                eps2, cand, cand_cap, cand_count);
    return cudaGetLastError();
}

cudaError_t launch_rescore(const float* rows, const uint32_t* ids, uint32_t dim, const float* qn, uint32_t nq,
                           const uint32_t* cand, uint32_t cand_cap, const uint32_t* cand_count, uint32_t k,
                           float* cand_sim, uint32_t* out_ids, float* out_sims, cudaStream_t s) {
    tc::rescore_kernel<<<(nq * 32 + 255) / 256, 256, 0, s>>>(rows, ids, dim, qn, nq, cand, cand_cap, cand_count, k,
                                                             cand_sim, out_ids, out_sims);
    return cudaGetLastError();
}

} // namespace ss
