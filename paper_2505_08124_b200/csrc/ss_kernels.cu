// Integer / fp32 kernels of the embedding pass and the vector query:
// mask decode, tile binning helpers, the sparse 512-d contraction,
// normalisation, store build and exact cosine scoring / top-k.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "ss_kernels.cuh"

namespace ss {
namespace {

// ------------------------------------------------------------ mask decode
// providers.hpp:95-109 rle_decode (alternating runs, zeros first) straight
// into a per-pixel mask bitset.  Pass 1 (one CTA per mask): a block scan turns
// run lengths into start positions and emits every "ones" run as a (start,
// len, mask) span.  Pass 2: one warp per span, lanes stride its pixels and
// OR bit m into the pixel's bitset word (spans of different masks share words).
__global__ void __launch_bounds__(256) rle_spans_kernel(const uint32_t* runs, const uint64_t* run_offsets,
                                                        uint4* spans, unsigned int* n_spans) {
    using Scan = cub::BlockScan<unsigned long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long carry;
    const uint32_t m = blockIdx.x;
    const uint64_t r0 = run_offsets[m], r1 = run_offsets[m + 1];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = r0; base < r1; base += 256) {
        const uint64_t k = base + threadIdx.x;
        const unsigned long long len = k < r1 ? runs[k] : 0ull;
        unsigned long long pos, agg;
        Scan(tmp).ExclusiveSum(len, pos, agg);
        pos += carry;
        const bool ones = k < r1 && ((k - r0) & 1ull) && len > 0;
        const unsigned int bal = __ballot_sync(0xffffffffu, ones);
        unsigned int slot0 = 0;
        if ((threadIdx.x & 31) == 0 && bal) slot0 = atomicAdd(n_spans, (unsigned int)__popc(bal));
        slot0 = __shfl_sync(0xffffffffu, slot0, 0);
        if (ones) {
            const unsigned int slot = slot0 + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
            spans[slot] = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)len, m);
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) spans_to_bits_kernel(const uint4* spans, const unsigned int* n_spans,
                                                            uint32_t words, uint32_t* bits) {
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned int n = *n_spans;
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
         w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint4 sp = spans[w];
        const unsigned long long pos = ((unsigned long long)sp.y << 32) | sp.x;
        const uint32_t word = sp.w >> 5, bit = 1u << (sp.w & 31u);
        for (uint32_t i = lane; i < sp.z; i += 32) atomicOr(bits + (pos + i) * words + word, bit);
    }
}

// providers.hpp:359-373 resample_mask (nearest neighbour, u64 index math)
__global__ void resample_bits_kernel(const uint32_t* src, uint32_t sw, uint32_t sh, uint32_t* dst, uint32_t tw,
                                     uint32_t th, uint32_t words) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (uint64_t)tw * th) return;
    const uint32_t x = (uint32_t)(i % tw), y = (uint32_t)(i / tw);
    uint32_t sy = (uint32_t)((2ull * y + 1) * sh / (2ull * th));
    uint32_t sx = (uint32_t)((2ull * x + 1) * sw / (2ull * tw));
    sy = sy < sh - 1 ? sy : sh - 1;
    sx = sx < sw - 1 ? sx : sw - 1;
    const uint32_t* s = src + ((uint64_t)sy * sw + sx) * words;
    for (uint32_t w = 0; w < words; ++w) dst[i * words + w] = s[w];
}

// ------------------------------------------------------------- binning
// rasterizer.hpp:181-194 builds, per 16x16 tile, the depth-ordered list of
// splats whose padded box covers the tile.  Here, with no host round trip:
//  1. narrow_keys: survivors' depth bit patterns -> 32-bit keys
//     (bits - min) >> shift (monotone in depth); culled -> 0xffffffff;
//  2. one stable radix sort of (key32, id) over all N Gaussians (CUB);
//  3. tie_fixup: exact (depth bits, id) order inside runs of equal key32;
//     => order[] is the reference's depth_sort order (projection.hpp:59-64);
//  4. count / offsets / scatter over CHUNKS OF CONSECUTIVE RANKS, with the
//     per-chunk tile histogram in shared memory: tile t's list is the
//     concatenation, in chunk order, of one small segment per chunk;
//  5. segment_sort: each (chunk, tile) segment (~8 entries) is put in depth
//     order -- the whole tile list is then in global depth order.
__device__ __forceinline__ uint32_t narrow_shift(const ViewInfo* info) {
    const unsigned long long span = info->min_key ^ info->max_key;
    const uint32_t hb = span ? 64u - (uint32_t)__clzll((long long)span) : 0u;
    return hb > 32u ? hb - 32u : 0u;
}

// (depth bits, id) ordering of the reference's comparator
__device__ __forceinline__ bool depth_before(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__global__ void narrow_keys_kernel(const unsigned long long* keys, uint64_t n, const ViewInfo* info, uint32_t* k32) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    if (k == ~0ull) {
        k32[i] = 0xffffffffu;
        return;
    }
    const uint32_t v = (uint32_t)((k - info->min_key) >> narrow_shift(info));
    k32[i] = v == 0xffffffffu ? 0xfffffffeu : v; // culled Gaussians alone sort last
}

__global__ void tie_fixup_kernel(const uint32_t* k32, uint64_t n, const unsigned long long* keys, uint32_t* order) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 >= n) return;
    const uint32_t k = k32[i];
    if (k == 0xffffffffu) return;                // culled tail
    if (i > 0 && k32[i - 1] == k) return;       // not a run start
    if (k32[i + 1] != k) return;                // singleton
    uint64_t e = i + 2;
    while (e < n && k32[e] == k) ++e;
    for (uint64_t a = i + 1; a < e; ++a) {      // insertion sort by (depth bits, id)
        const uint32_t id = order[a];
        const unsigned long long key = keys[id];
        uint64_t b = a;
        while (b > i && depth_before(key, id, keys[order[b - 1]], order[b - 1])) {
            order[b] = order[b - 1];
            --b;
        }
        order[b] = id;
    }
}

__device__ __forceinline__ bool rank_box(const SplatRec* rec, const uint32_t* k32s, const uint32_t* order, uint64_t r,
                                         uint32_t& id, uint32_t& tx0, uint32_t& tx1, uint32_t& ty0, uint32_t& ty1) {
    if (k32s[r] == 0xffffffffu) return false; // culled (projection.hpp:38 / rasterizer.hpp:177)
    id = order[r];
    const uint2 box = __ldg(reinterpret_cast<const uint2*>(&rec[id].x0));
    tx0 = (box.x & 0xffffu) / kTile;
    tx1 = (box.x >> 16) / kTile;
    ty0 = (box.y & 0xffffu) / kTile;
    ty1 = (box.y >> 16) / kTile;
    return true;
}

__global__ void __launch_bounds__(1024) tile_count_kernel(const SplatRec* rec, const uint32_t* k32s,
                                                         const uint32_t* order, uint64_t n, uint64_t chunk,
                                                         uint32_t tiles, uint32_t tiles_x, uint32_t* chunk_counts) {
    extern __shared__ uint32_t hist[];
    for (uint32_t t = threadIdx.x; t < tiles; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    const uint64_t lo = (uint64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    for (uint64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        uint32_t id, tx0, tx1, ty0, ty1;
        if (!rank_box(rec, k32s, order, r, id, tx0, tx1, ty0, ty1)) continue;
        for (uint32_t ty = ty0; ty <= ty1; ++ty)
            for (uint32_t tx = tx0; tx <= tx1; ++tx) atomicAdd(hist + ty * tiles_x + tx, 1u);
    }
    __syncthreads();
    uint32_t* row = chunk_counts + (uint64_t)blockIdx.x * tiles;
    for (uint32_t t = threadIdx.x; t < tiles; t += blockDim.x) row[t] = hist[t];
}

// Per tile (one thread each): exclusive prefix of the chunk counts down the
// tile's column (in place, coalesced across threads) and the tile total.
__global__ void __launch_bounds__(128) tile_column_prefix_kernel(uint32_t* chunk_counts, uint32_t n_chunks,
                                                                 uint32_t tiles, uint32_t* totals) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tiles) return;
    uint32_t run = 0;
    uint32_t c = 0;
    for (; c + 8 <= n_chunks; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = chunk_counts[(uint64_t)(c + j) * tiles + t];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            chunk_counts[(uint64_t)(c + j) * tiles + t] = run;
            run += v[j];
        }
    }
    for (; c < n_chunks; ++c) {
        const uint32_t v = chunk_counts[(uint64_t)c * tiles + t];
        chunk_counts[(uint64_t)c * tiles + t] = run;
        run += v;
    }
    totals[t] = run;
}

// One CTA: exclusive scan of the tile totals -> tile_start[0..tiles].
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* totals, uint32_t tiles, uint32_t* tile_start,
                                                        ViewInfo* info) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < tiles; base += 1024) {
        const uint32_t t = base + threadIdx.x;
        const uint32_t v = t < tiles ? totals[t] : 0u;
        uint32_t ex, agg;
        Scan(tmp).ExclusiveSum(v, ex, agg);
        if (t < tiles) tile_start[t] = ex + carry;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tile_start[tiles] = carry;
        info->n_instances = carry;
    }
}

__global__ void __launch_bounds__(1024) tile_scatter_kernel(const SplatRec* rec, const uint32_t* k32s,
                                                           const uint32_t* order, uint64_t n, uint64_t chunk,
                                                           uint32_t tiles, uint32_t tiles_x,
                                                           const uint32_t* chunk_prefix, const uint32_t* tile_start,
                                                           uint32_t* list, uint64_t cap, ViewInfo* info) {
    extern __shared__ uint32_t cursor[];
    if (info->n_instances > cap) { // the tile lists do not fit: the host re-runs the view
        if (threadIdx.x == 0) info->overflow = 1u;
        return;
    }
    const uint32_t* pre = chunk_prefix + (uint64_t)blockIdx.x * tiles;
    for (uint32_t t = threadIdx.x; t < tiles; t += blockDim.x) cursor[t] = tile_start[t] + pre[t];
    __syncthreads();
    const uint64_t lo = (uint64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    for (uint64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        uint32_t id, tx0, tx1, ty0, ty1;
        if (!rank_box(rec, k32s, order, r, id, tx0, tx1, ty0, ty1)) continue;
        for (uint32_t ty = ty0; ty <= ty1; ++ty)
            for (uint32_t tx = tx0; tx <= tx1; ++tx) list[atomicAdd(cursor + ty * tiles_x + tx, 1u)] = (uint32_t)r;
    }
}

// Warp bitonic sort of 32*R u32; element lane + 32*r lives in v[r] of `lane`.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[R], uint32_t lane) {
#pragma unroll
    for (uint32_t k = 2; k <= 32u * R; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const uint32_t jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if ((r & jr) != 0) continue;
                    const bool asc = ((lane + 32u * r) & k) == 0;
                    const uint32_t lo = min(v[r], v[r | jr]), hi = max(v[r], v[r | jr]);
                    v[r] = asc ? lo : hi;
                    v[r | jr] = asc ? hi : lo;
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t pv = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool asc = ((lane + 32u * r) & k) == 0;
                    v[r] = (lower == asc) ? min(v[r], pv) : max(v[r], pv);
                }
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void warp_sort_segment(uint32_t* seg, uint32_t m, uint32_t lane) {
    uint32_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = lane + 32u * r < m ? seg[lane + 32u * r] : 0xffffffffu;
    warp_bitonic<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (lane + 32u * r < m) seg[lane + 32u * r] = v[r];
}

// One CTA per tile: the tile's list (depth ranks, one segment per rank chunk,
// segments already in chunk order) is loaded coalesced into shared memory,
// each warp sorts segments with a register bitonic network of up to 512
// (longer segments: insertion sort by one lane), and the ranks are replaced by
// Gaussian ids (order[rank]) on the way out, so the compositor reads records
// directly.  Tiles larger than the shared-memory slice sort in global memory.
constexpr uint32_t kSegSmem = 12288; // ranks per tile held in shared memory (48 KB)
__global__ void __launch_bounds__(512) segment_sort_kernel(const uint32_t* chunk_prefix, uint32_t n_chunks,
                                                           uint32_t tiles, const uint32_t* tile_start,
                                                           const uint32_t* order, uint32_t* list,
                                                           const ViewInfo* info) {
    extern __shared__ uint32_t sl[];
    const uint32_t t = blockIdx.x;
    const uint32_t ts = tile_start[t], n = tile_start[t + 1] - ts;
    if (n == 0 || info->overflow) return;
    const bool in_smem = n <= kSegSmem;
    uint32_t* base = in_smem ? sl : list + ts;
    if (in_smem) {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sl[i] = list[ts + i];
        __syncthreads();
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t c = warp; c < n_chunks; c += nw) {
        const uint32_t s0 = chunk_prefix[(uint64_t)c * tiles + t];
        const uint32_t s1 = c + 1 < n_chunks ? chunk_prefix[(uint64_t)(c + 1) * tiles + t] : n;
        const uint32_t m = s1 - s0;
        if (m < 2) continue;
        if (m <= 64) {
            warp_sort_segment<2>(base + s0, m, lane);
        } else if (m <= 128) {
            warp_sort_segment<4>(base + s0, m, lane);
        } else if (m <= 256) {
            warp_sort_segment<8>(base + s0, m, lane);
        } else if (m <= 512) {
            warp_sort_segment<16>(base + s0, m, lane);
        } else if (lane == 0) {
            for (uint32_t x = s0 + 1; x < s1; ++x) {
                const uint32_t r = base[x];
                uint32_t y = x;
                while (y > s0 && base[y - 1] > r) {
                    base[y] = base[y - 1];
                    --y;
                }
                base[y] = r;
            }
        }
        __syncwarp();
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) list[ts + i] = __ldg(order + base[i]);
}

// --------------------------------------------------------- contraction
// pipeline.hpp:70-80 accumulate, per view: for every rank the compositor
// touched, row[gid] += sum_m acc[rank, m] * CLIP_m and total[gid] +=
// sum_m acc[rank, m]; then the scalars are cleared for the next view.  One
// warp per touched Gaussian; the 2 KB fp32 row moves as four coalesced
// float4 sweeps; CLIP rows stay L1/L2-resident (M x 2 KB per view).
template <bool DIM512>
__global__ void __launch_bounds__(256) contract_kernel(ContractParams p) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned long long n_touched = p.info->n_touched;
    unsigned long long pairs = 0;
    for (uint64_t t = warp0; t < n_touched; t += nwarps) {
        const uint32_t gid = p.touched_list[t];
        float* accrow = p.acc + (size_t)gid * p.n_masks;
        float* row = p.sums + (size_t)gid * p.dim;
        float4 racc[4];
        if constexpr (DIM512) {
#pragma unroll
            for (int q = 0; q < 4; ++q) racc[q] = reinterpret_cast<const float4*>(row)[lane + 32 * q];
        }
        float wsum = 0.0f;
        for (uint32_t c = 0; c < p.n_masks; c += 32) {
            const uint32_t mi = c + lane;
            float v = 0.0f;
            if (mi < p.n_masks) {
                v = accrow[mi];
                if (v != 0.0f) accrow[mi] = 0.0f;
            }
            wsum += v;
            uint32_t bal = __ballot_sync(0xffffffffu, v != 0.0f);
            pairs += __popc(bal);
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const float w = __shfl_sync(0xffffffffu, v, src);
                const float* e = p.clip + (size_t)(c + src) * p.dim;
                if constexpr (DIM512) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 ev = __ldg(reinterpret_cast<const float4*>(e) + lane + 32 * q);
                        racc[q].x += w * ev.x;
                        racc[q].y += w * ev.y;
                        racc[q].z += w * ev.z;
                        racc[q].w += w * ev.w;
                    }
                } else {
                    for (uint32_t d = lane; d < p.dim; d += 32) row[d] += w * __ldg(e + d);
                }
            }
        }
        if constexpr (DIM512) {
#pragma unroll
            for (int q = 0; q < 4; ++q) reinterpret_cast<float4*>(row)[lane + 32 * q] = racc[q];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        if (lane == 0) {
            p.totals[gid] += wsum;
            p.touched[gid] = 0u;
        }
    }
    if (p.count_pairs) {
        // pairs is warp-uniform (ballot popcounts); count once per warp
        if (lane == 0 && pairs) atomicAdd(p.cum + 1, pairs);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(p.cum, n_touched);
    }
}

// pipeline.hpp:120-135 finalize_into: covered rows (total > 1e-8) become
// sum/total, coverage = total; uncovered rows are exactly zero.
__global__ void __launch_bounds__(256) normalize_kernel(const float* sums, const float* totals, uint64_t n,
                                                        uint32_t dim, float* rows, float* coverage) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec = (dim & 3u) == 0;
    for (uint64_t k = warp0; k < n; k += nwarps) {
        const float t = totals[k];
        const bool cov = (double)t > 1e-8;
        const double inv = cov ? 1.0 / (double)t : 0.0;
        const float* s = sums + k * dim;
        float* o = rows + k * dim;
        if (vec) {
            for (uint32_t d = lane * 4; d < dim; d += 128) {
                float4 v = *reinterpret_cast<const float4*>(s + d);
                if (cov) {
                    v.x = __double2float_rn((double)v.x * inv);
                    v.y = __double2float_rn((double)v.y * inv);
                    v.z = __double2float_rn((double)v.z * inv);
                    v.w = __double2float_rn((double)v.w * inv);
                } else {
                    v = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                *reinterpret_cast<float4*>(o + d) = v;
            }
        } else {
            for (uint32_t d = lane; d < dim; d += 32) o[d] = cov ? __double2float_rn((double)s[d] * inv) : 0.0f;
        }
        if (lane == 0) coverage[k] = cov ? t : 0.0f;
    }
}

// ---------------------------------------------------------------- query
// vecstore.hpp:34-42 normalized_copy, one warp per row: the f64 square sum is
// accumulated strictly sequentially (lane 0 walks the row staged in
// registers via shuffles) so the unit rows are bit-identical.
__global__ void __launch_bounds__(256) normalize_rows_kernel(const float* in, const uint32_t* select, uint64_t n,
                                                             uint32_t dim, float* out, int* zero_flag) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp0; k < n; k += nwarps) {
        const uint64_t src = select ? select[k] : k;
        const float* v = in + src * dim;
        double ns = 0.0;
        for (uint32_t c = 0; c < dim; c += 32) {
            const float x = (c + lane < dim) ? v[c + lane] : 0.0f;
            const double sq = (double)x * (double)x; // exact
            const uint32_t cnt = min(32u, dim - c);
            for (uint32_t j = 0; j < cnt; ++j) ns = __dadd_rn(ns, __shfl_sync(0xffffffffu, sq, j));
        }
        if (!(ns > 0.0)) {
            if (lane == 0) atomicExch(zero_flag, 1);
            continue;
        }
        const double inv = __ddiv_rn(1.0, __dsqrt_rn(ns));
        for (uint32_t d = lane; d < dim; d += 32) out[k * dim + d] = __double2float_rn(__dmul_rn((double)v[d], inv));
    }
}

// vecstore.hpp:21-31 dot_lanes, exactly: eight fp32 lanes accumulated in
// index order with separate rounded multiply and add (no FMA), pairwise
// combine, then the tail.  One thread per store row, QT queries per block
// held in shared memory, so each row is read once per query tile.
template <int QT>
__global__ void __launch_bounds__(256) score_kernel(const float* rows, uint64_t count, uint32_t dim,
                                                    const float* queries, uint32_t nq, uint32_t q0, float* scores) {
    extern __shared__ float sq[]; // QT x dim
    const uint32_t qn = min((uint32_t)QT, nq - q0);
    for (uint32_t i = threadIdx.x; i < QT * dim; i += blockDim.x) {
        const uint32_t qi = i / dim;
        sq[i] = qi < qn ? queries[(size_t)(q0 + qi) * dim + (i % dim)] : 0.0f;
    }
    __syncthreads();
    const uint32_t d8 = dim & ~7u;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (uint64_t)gridDim.x * blockDim.x) {
        const float* a = rows + r * dim;
        float lanes[QT][8];
#pragma unroll
        for (int q = 0; q < QT; ++q)
#pragma unroll
            for (int l = 0; l < 8; ++l) lanes[q][l] = 0.0f;
        for (uint32_t i = 0; i < d8; i += 8) {
            float av[8];
            if ((dim & 3u) == 0) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(a + i));
                const float4 y = __ldg(reinterpret_cast<const float4*>(a + i + 4));
                av[0] = x.x; av[1] = x.y; av[2] = x.z; av[3] = x.w;
                av[4] = y.x; av[5] = y.y; av[6] = y.z; av[7] = y.w;
            } else {
#pragma unroll
                for (int l = 0; l < 8; ++l) av[l] = __ldg(a + i + l);
            }
#pragma unroll
            for (int q = 0; q < QT; ++q)
#pragma unroll
                for (int l = 0; l < 8; ++l) lanes[q][l] = __fadd_rn(lanes[q][l], __fmul_rn(av[l], sq[q * dim + i + l]));
        }
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            if ((uint32_t)q >= qn) break;
            float tail = 0.0f;
            for (uint32_t i = d8; i < dim; ++i) tail = __fadd_rn(tail, __fmul_rn(__ldg(a + i), sq[q * dim + i]));
            const float s01 = __fadd_rn(lanes[q][0], lanes[q][1]), s23 = __fadd_rn(lanes[q][2], lanes[q][3]);
            const float s45 = __fadd_rn(lanes[q][4], lanes[q][5]), s67 = __fadd_rn(lanes[q][6], lanes[q][7]);
            scores[(size_t)q * count + r] = __fadd_rn(__fadd_rn(__fadd_rn(s01, s23), __fadd_rn(s45, s67)), tail);
        }
    }
}

__device__ __forceinline__ bool scored_before(float sa, uint32_t ia, float sb, uint32_t ib) {
    // vecstore.hpp:107-110
    if (sa != sb) return sa > sb;
    return ia < ib;
}

// Per-query exact top-k over a score row: each thread keeps a sorted local
// list of the best k it has seen, then the block merges the 256 lists in
// shared memory.  k <= kMaxK.
constexpr int kMaxK = 64;
__global__ void __launch_bounds__(256) topk_kernel(const float* scores, const uint32_t* ids, uint64_t count,
                                                   uint32_t k, uint32_t q0, uint32_t* out_ids, float* out_sims) {
    const uint32_t qi = blockIdx.x;
    const float* s = scores + (size_t)qi * count;
    float bs[kMaxK];
    uint32_t bi[kMaxK];
    uint32_t have = 0;
    const uint32_t take = (uint32_t)min((uint64_t)k, count);
    for (uint64_t r = threadIdx.x; r < count; r += blockDim.x) {
        const float v = s[r];
        const uint32_t id = ids[r];
        if (have == take && !scored_before(v, id, bs[take - 1], bi[take - 1])) continue;
        uint32_t pos = have < take ? have : take - 1;
        while (pos > 0 && scored_before(v, id, bs[pos - 1], bi[pos - 1])) {
            bs[pos] = bs[pos - 1];
            bi[pos] = bi[pos - 1];
            --pos;
        }
        bs[pos] = v;
        bi[pos] = id;
        if (have < take) ++have;
    }
    // block merge: repeatedly extract the best head among the threads
    __shared__ float hs[256];
    __shared__ uint32_t hi[256];
    __shared__ int hwin;
    uint32_t head = 0;
    for (uint32_t outk = 0; outk < take; ++outk) {
        hs[threadIdx.x] = head < have ? bs[head] : -INFINITY;
        hi[threadIdx.x] = head < have ? bi[head] : 0xffffffffu;
        const bool valid = head < have;
        __syncthreads();
        if (threadIdx.x == 0) {
            int best = -1;
            for (int t = 0; t < (int)blockDim.x; ++t) {
                const bool tv = hi[t] != 0xffffffffu || hs[t] != -INFINITY;
                if (!tv) continue;
                if (best < 0 || scored_before(hs[t], hi[t], hs[best], hi[best])) best = t;
            }
            hwin = best;
            if (best >= 0) {
                out_ids[(size_t)(q0 + qi) * k + outk] = hi[best];
                out_sims[(size_t)(q0 + qi) * k + outk] = hs[best];
            }
        }
        __syncthreads();
        if ((int)threadIdx.x == hwin && valid) ++head;
        __syncthreads();
    }
}

__global__ void flag_covered_kernel(const float* coverage, uint64_t n, uint8_t* flags) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = coverage[i] > 1e-8f ? 1 : 0; // EmbeddingTable::covered, pipeline.hpp:115
}

// (sim desc, id asc) as one ascending u64 radix key
__global__ void threshold_keys_kernel(const float* scores, const uint32_t* ids, uint64_t count, float tau,
                                      unsigned long long* keys, uint8_t* flags) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const float v = scores[i];
    flags[i] = v >= tau ? 1 : 0;
    uint32_t b = __float_as_uint(v);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u); // ascending-orderable
    b = ~b;                                          // descending
    keys[i] = ((unsigned long long)b << 32) | ids[i];
}

} // namespace

// ---------------------------------------------------------------- launchers
static inline unsigned blocks_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }
static inline unsigned warp_grid(uint64_t n) {
    const uint64_t b = (n + 7) / 8; // 8 warps per 256-thread block
    return (unsigned)(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16);
}

cudaError_t launch_rle_to_bits(const uint32_t* runs, const uint64_t* run_offsets, uint32_t n_masks, uint32_t words,
                               uint32_t* bits, uint4* spans, unsigned int* n_spans, cudaStream_t s) {
    if (n_masks == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(n_spans, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    rle_spans_kernel<<<n_masks, 256, 0, s>>>(runs, run_offsets, spans, n_spans);
    spans_to_bits_kernel<<<148 * 8, 256, 0, s>>>(spans, n_spans, words, bits);
    return cudaGetLastError();
}
cudaError_t launch_resample_bits(const uint32_t* src, uint32_t sw, uint32_t sh, uint32_t* dst, uint32_t tw,
                                 uint32_t th, uint32_t words, cudaStream_t s) {
    const uint64_t n = (uint64_t)tw * th;
    if (!n) return cudaSuccess;
    resample_bits_kernel<<<blocks_for(n, 256), 256, 0, s>>>(src, sw, sh, dst, tw, th, words);
    return cudaGetLastError();
}
uint32_t tile_chunks(uint64_t n, uint64_t* chunk) {
    // ~128 rank chunks: per-chunk tile histograms stay small and the
    // per-tile segments short
    uint64_t c = (n + 127) / 128;
    c = std::max<uint64_t>(1024, (c + 1023) / 1024 * 1024);
    *chunk = c;
    return (uint32_t)std::max<uint64_t>(1, (n + c - 1) / c);
}

cudaError_t launch_narrow_keys(const unsigned long long* keys, uint64_t n, const ViewInfo* info, uint32_t* k32,
                               cudaStream_t s) {
    if (!n) return cudaSuccess;
    narrow_keys_kernel<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, info, k32);
    return cudaGetLastError();
}

cudaError_t launch_tie_fixup(const uint32_t* k32s, uint64_t n, const unsigned long long* keys, uint32_t* order,
                             cudaStream_t s) {
    if (n < 2) return cudaSuccess;
    tie_fixup_kernel<<<blocks_for(n, 256), 256, 0, s>>>(k32s, n, keys, order);
    return cudaGetLastError();
}

cudaError_t launch_tile_bins(const SplatRec* rec, const uint32_t* k32s, const uint32_t* order,
                             const unsigned long long* keys, uint64_t n, uint32_t tiles, uint32_t tiles_x,
                             uint32_t* chunk_counts, uint32_t* totals, uint32_t* tile_start, uint32_t* list,
                             uint64_t cap, ViewInfo* info, cudaStream_t s) {
    uint64_t chunk = 0;
    const uint32_t nch = tile_chunks(n, &chunk);
    const size_t smem = (size_t)tiles * 4;
    // raise the dynamic shared-memory limit once per device (the call is not free)
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        const int lim = 50000 * 4;
        cudaError_t e = cudaFuncSetAttribute(tile_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
        if (e != cudaSuccess) return e;
        configured_dev = dev;
    }
    tile_count_kernel<<<nch, 1024, smem, s>>>(rec, k32s, order, n, chunk, tiles, tiles_x, chunk_counts);
    tile_column_prefix_kernel<<<blocks_for(tiles, 128), 128, 0, s>>>(chunk_counts, nch, tiles, totals);
    tile_scan_kernel<<<1, 1024, 0, s>>>(totals, tiles, tile_start, info);
    tile_scatter_kernel<<<nch, 1024, smem, s>>>(rec, k32s, order, n, chunk, tiles, tiles_x, chunk_counts, tile_start,
                                                list, cap, info);
    segment_sort_kernel<<<tiles, 512, kSegSmem * 4, s>>>(chunk_counts, nch, tiles, tile_start, order, list, info);
    return cudaGetLastError();
}

cudaError_t launch_contract(const ContractParams& p, uint64_t max_touched, cudaStream_t s) {
    if (!max_touched) return cudaSuccess;
    if (p.dim == 512)
        contract_kernel<true><<<warp_grid(max_touched), 256, 0, s>>>(p);
    else
        contract_kernel<false><<<warp_grid(max_touched), 256, 0, s>>>(p);
    return cudaGetLastError();
}
cudaError_t launch_normalize(const float* sums, const float* totals, uint64_t n, uint32_t dim, float* rows,
                             float* coverage, cudaStream_t s) {
    if (!n) return cudaSuccess;
    normalize_kernel<<<warp_grid(n), 256, 0, s>>>(sums, totals, n, dim, rows, coverage);
    return cudaGetLastError();
}
cudaError_t launch_normalize_rows(const float* in, const uint32_t* select, uint64_t n, uint32_t dim, float* out,
                                  int* zero_flag, cudaStream_t s) {
    if (!n) return cudaSuccess;
    normalize_rows_kernel<<<warp_grid(n), 256, 0, s>>>(in, select, n, dim, out, zero_flag);
    return cudaGetLastError();
}
cudaError_t launch_flag_covered(const float* coverage, uint64_t n, uint8_t* flags, cudaStream_t s) {
    if (!n) return cudaSuccess;
    flag_covered_kernel<<<blocks_for(n, 256), 256, 0, s>>>(coverage, n, flags);
    return cudaGetLastError();
}
constexpr int kScoreQT = 8;
int score_query_tile() { return kScoreQT; }
cudaError_t launch_score(const float* rows, uint64_t count, uint32_t dim, const float* queries, uint32_t nq, uint32_t q0,
                         float* scores, cudaStream_t s) {
    if (!count) return cudaSuccess;
    const size_t smem = (size_t)kScoreQT * dim * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(score_kernel<kScoreQT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    unsigned g = blocks_for(count, 256);
    if (g > 148u * 8) g = 148u * 8;
    score_kernel<kScoreQT><<<g, 256, smem, s>>>(rows, count, dim, queries, nq, q0, scores);
    return cudaGetLastError();
}
cudaError_t launch_topk(const float* scores, const uint32_t* ids, uint64_t count, uint32_t k, uint32_t nq_tile,
                        uint32_t q0, uint32_t* out_ids, float* out_sims, cudaStream_t s) {
    if (!nq_tile || !count || !k) return cudaSuccess;
    if (k > (uint32_t)kMaxK) return cudaErrorInvalidValue;
    topk_kernel<<<nq_tile, 256, 0, s>>>(scores, ids, count, k, q0, out_ids, out_sims);
    return cudaGetLastError();
}
cudaError_t launch_threshold_keys(const float* scores, const uint32_t* ids, uint64_t count, float tau,
                                  unsigned long long* keys, uint8_t* flags, cudaStream_t s) {
    if (!count) return cudaSuccess;
    threshold_keys_kernel<<<blocks_for(count, 256), 256, 0, s>>>(scores, ids, count, tau, keys, flags);
    return cudaGetLastError();
}

} // namespace ss
