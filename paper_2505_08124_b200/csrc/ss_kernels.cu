// Integer / fp32 kernels of the embedding pass and the vector query:
// mask decode, tile binning helpers, the sparse 512-d contraction,
// normalisation, store build and exact cosine scoring / top-k.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <cub/iterator/transform_input_iterator.cuh>

#include "ss_kernels.cuh"

namespace ss {
// flags[i] as a u32 for the exclusive scan of the sparse combine (i == n reads 0)
struct FlagAt {
    const uint8_t* f;
    uint64_t n;
    __host__ __device__ uint32_t operator()(uint64_t i) const { return i < n ? (uint32_t)f[i] : 0u; }
};
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
//  4. instances (tile, id) emitted in depth-rank order at scanned offsets;
//  5. a stable radix sort by tile key (CUB) over a device-sized capacity
//     (padding keys sort last) => every tile's slice is in depth order;
//  6. tile_ranges: slice bounds by boundary detection.
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
    // four keys per thread (two 16-byte loads, one 16-byte store)
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 >= n) return;
    const unsigned long long mn = info->min_key;
    const uint32_t sh = narrow_shift(info);
    unsigned long long k[4];
    if (i0 + 4 <= n) {
        const ulonglong2 a = reinterpret_cast<const ulonglong2*>(keys + i0)[0];
        const ulonglong2 b = reinterpret_cast<const ulonglong2*>(keys + i0)[1];
        k[0] = a.x, k[1] = a.y, k[2] = b.x, k[3] = b.y;
    } else {
        for (int j = 0; j < 4; ++j) k[j] = i0 + j < n ? keys[i0 + j] : ~0ull;
    }
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t t = (uint32_t)((k[j] - mn) >> sh);
        v[j] = k[j] == ~0ull ? 0xffffffffu : (t == 0xffffffffu ? 0xfffffffeu : t); // culled alone sort last
    }
    if (i0 + 4 <= n) {
        reinterpret_cast<uint4*>(k32 + i0)[0] = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
        for (int j = 0; j < 4; ++j)
            if (i0 + j < n) k32[i0 + j] = v[j];
    }
}

__global__ void tie_fixup_kernel(const uint32_t* k32, uint64_t n, const unsigned long long* keys, uint32_t* order) {
    // four sorted keys per thread: a run of equal narrowed keys is fixed by the
    // thread owning its first element (almost always there is none)
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 + 1 >= n) return;
    uint32_t kk[5];
    if (i0 + 5 <= n) {
        const uint4 q = reinterpret_cast<const uint4*>(k32 + i0)[0];
        kk[0] = q.x, kk[1] = q.y, kk[2] = q.z, kk[3] = q.w, kk[4] = k32[i0 + 4];
    } else {
        for (int j = 0; j < 5; ++j) kk[j] = i0 + j < n ? k32[i0 + j] : 0xffffffffu;
    }
    uint32_t prev = i0 > 0 ? k32[i0 - 1] : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint64_t i = i0 + j;
        const uint32_t k = kk[j];
        const bool start = i + 1 < n && k != 0xffffffffu && (i == 0 || prev != k) && kk[j + 1] == k;
        prev = k;
        if (!start) continue;
        uint64_t e = i + 2;
        while (e < n && k32[e] == k) ++e;
        for (uint64_t a = i + 1; a < e; ++a) { // insertion sort by (depth bits, id)
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
}

// Boxes in depth-rank order, gathered once: rbox[r] = boxes[order[r]], or
// kCulledBox for the culled tail (a real box has x0 <= x1 < 65535).
constexpr uint32_t kCulledBox = 0xffffffffu;
__device__ __forceinline__ uint32_t box_tiles(uint2 box);

// ... and the rank's tile count, cnt[n] = 0, for the offset scan.
__global__ void gather_boxes_kernel(const uint2* boxes, const uint32_t* k32s, const uint32_t* order, uint64_t n,
                                    uint2* rbox, uint32_t* cnt) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        cnt[n] = 0u;
        return;
    }
    const uint2 b = k32s[r] == 0xffffffffu ? make_uint2(kCulledBox, kCulledBox) : __ldg(boxes + order[r]);
    rbox[r] = b;
    cnt[r] = box_tiles(b);
}

__device__ __forceinline__ uint32_t box_tiles(uint2 box) {
    if (box.x == kCulledBox) return 0u;
    return ((box.x >> 16) / kTile - (box.x & 0xffffu) / kTile + 1u) *
           ((box.y >> 16) / kTile - (box.y & 0xffffu) / kTile + 1u);
}


// Instances in depth-rank order: splat of rank r writes (tile, id) for every
// tile its box covers (row-major within the box) at offsets[r] (exclusive
// scan of RankTiles).  A stable sort by tile then yields each tile's list in
// depth order.  Warp-cooperative: the warp's 32 ranks own one contiguous
// output range, written 32 consecutive slots per round; a slot's rank is
// found by a binary search over the lanes' offsets (shuffles).
template <typename K>
__global__ void emit_instances_kernel(const uint2* rbox, const uint32_t* order, uint64_t n, const uint32_t* offsets,
                                      uint32_t tiles_x, uint64_t cap, K* keys, uint32_t* vals, ViewInfo* info) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t r0 = r - lane;
    if (r0 >= n) return;
    if (offsets[n] > cap) { // lists do not fit: the host re-runs the view
        if (r == 0) info->overflow = 1u;
        return;
    }
    const bool live = r < n;
    const uint2 box = live ? rbox[r] : make_uint2(kCulledBox, kCulledBox);
    const uint32_t cnt = box_tiles(box);
    const uint32_t off = live ? offsets[r] : offsets[n];
    const uint32_t tx0 = (box.x & 0xffffu) / kTile, ty0 = (box.y & 0xffffu) / kTile;
    const uint32_t nx = box.x == kCulledBox ? 1u : (box.x >> 16) / kTile - tx0 + 1u;
    const uint32_t id = live && cnt ? order[r] : 0u;
    const uint32_t base = __shfl_sync(0xffffffffu, off, 0);
    const uint32_t rel = off - base; // lane's first slot within the warp's range
    const uint32_t total = __shfl_sync(0xffffffffu, rel + cnt, 31);
    for (uint32_t p0 = 0; p0 < total; p0 += 32) {
        const uint32_t pos = p0 + lane;
        // owner: the last lane whose first slot is <= pos (empty lanes never own a slot)
        uint32_t o = 0;
#pragma unroll
        for (uint32_t step = 16; step > 0; step >>= 1) {
            const uint32_t rv = __shfl_sync(0xffffffffu, rel, o + step);
            if (rv <= pos) o += step;
        }
        const uint32_t o_rel = __shfl_sync(0xffffffffu, rel, o);
        const uint32_t o_nx = __shfl_sync(0xffffffffu, nx, o);
        const uint32_t o_tx0 = __shfl_sync(0xffffffffu, tx0, o);
        const uint32_t o_ty0 = __shfl_sync(0xffffffffu, ty0, o);
        const uint32_t o_id = __shfl_sync(0xffffffffu, id, o);
        if (pos < total) {
            const uint32_t k = pos - o_rel;
            const uint32_t dy = k / o_nx, dx = k - dy * o_nx;
            const uint64_t q = (uint64_t)base + pos;
            keys[q] = (K)((o_ty0 + dy) * tiles_x + o_tx0 + dx);
            vals[q] = o_id;
        }
    }
}

// Pad [I_v, cap) with the largest key so a fixed-size sort leaves it last.
template <typename K>
__global__ void pad_keys_kernel(const uint32_t* offsets, uint64_t n, uint64_t cap, K* keys) {
    const uint64_t iv = offsets[n];
    for (uint64_t i = iv + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = (K)~(K)0;
}

template <typename K>
__global__ void tile_ranges_kernel(const K* keys, const uint32_t* offsets, uint64_t n, uint32_t* start,
                                   uint32_t* end, ViewInfo* info) {
    // each thread checks the boundaries of 16 bytes of sorted keys (one uint4)
    constexpr uint32_t PER = 16 / sizeof(K);
    const uint64_t iv = offsets[n];
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * PER;
    if (i0 == 0) info->n_instances = iv;
    if (i0 >= iv || info->overflow) return;
    K k[PER];
    *reinterpret_cast<uint4*>(k) = __ldg(reinterpret_cast<const uint4*>(keys + i0));
    uint32_t prev = i0 == 0 ? 0xffffffffu : (uint32_t)__ldg(keys + i0 - 1);
#pragma unroll
    for (uint32_t j = 0; j < PER; ++j) {
        const uint64_t i = i0 + j;
        if (i >= iv) break;
        const uint32_t kj = k[j];
        if (i == 0 || prev != kj) start[kj] = (uint32_t)i;
        const uint32_t next = j + 1 < PER ? (uint32_t)k[j + 1] : (i + 1 < iv ? (uint32_t)__ldg(keys + i + 1) : 0u);
        if (i == iv - 1 || next != kj) end[kj] = (uint32_t)(i + 1);
        prev = kj;
    }
}

// ------------------------------------------------ direct box binning
// The same tile lists as steps 4-6 above (each tile's slice = the depth ranks
// whose box covers it, ascending) without materialising (tile, id) keys or
// sorting them: a counting sort whose one "digit" is the whole tile index.
//  A. bin_count: chunk c = ranks [c*R, (c+1)*R); counts[c][t] = instances of
//     tile t in the chunk (shared-memory histogram).  Also rbox[r].
//  B. bin_scan: per tile, exclusive prefix over chunks (in 32 slices:
//     counts[c][t] becomes the prefix inside its slice, slice[s][t] the slice
//     base), tile totals; the last CTA scans the totals into tile_start /
//     tile_end and sets n_instances / overflow.
//  C. bin_scatter: chunk c's CTA holds cur[t] = start + slice + prefix; its
//     warps own consecutive rank ranges, so a per-tile scan over the warps'
//     own counts gives each warp its first slot; inside a warp the 32-slot
//     rounds run in rank order and slots of one tile in a round belong to
//     distinct ranks in lane order (a rank covers a tile at most once), so
//     the rank inside the round is popc(match_any(tile) & lanes below).
// Every step is deterministic; the result is bit-identical to the sort path.
constexpr uint32_t kBinChunk = 4096;   // ranks per chunk
constexpr uint32_t kBinSlices = 32;    // chunk slices of the prefix scan

// Visit a warp's 32 boxes' tile instances in (lane, row-major tile) order, 32
// slots per round: f(valid, tile, owner_lane) on every lane of every round.
template <typename F>
__device__ __forceinline__ void for_each_instance(uint2 box, uint32_t lane, uint32_t tiles_x, F&& f) {
    const uint32_t cnt = box_tiles(box);
    const uint32_t tx0 = (box.x & 0xffffu) / kTile, ty0 = (box.y & 0xffffu) / kTile;
    const uint32_t nx = box.x == kCulledBox ? 1u : (box.x >> 16) / kTile - tx0 + 1u;
    uint32_t incl = cnt;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    const uint32_t rel = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t p0 = 0; p0 < total; p0 += 32) {
        const uint32_t pos = p0 + lane;
        uint32_t o = 0; // the last lane whose first slot is <= pos
#pragma unroll
        for (uint32_t step = 16; step > 0; step >>= 1) {
            const uint32_t rv = __shfl_sync(0xffffffffu, rel, o + step);
            if (rv <= pos) o += step;
        }
        const uint32_t o_rel = __shfl_sync(0xffffffffu, rel, o);
        const uint32_t o_nx = __shfl_sync(0xffffffffu, nx, o);
        const uint32_t o_tx0 = __shfl_sync(0xffffffffu, tx0, o);
        const uint32_t o_ty0 = __shfl_sync(0xffffffffu, ty0, o);
        const uint32_t k = pos - o_rel;
        const uint32_t dy = k / o_nx, dx = k - dy * o_nx;
        f(pos < total, (o_ty0 + dy) * tiles_x + o_tx0 + dx, o);
    }
}

__device__ __forceinline__ uint32_t bin_chunks(const ViewInfo* info) {
    return (uint32_t)((info->n_surv + kBinChunk - 1) / kBinChunk);
}

__global__ void __launch_bounds__(256) bin_count_kernel(BinParams p) {
    extern __shared__ uint32_t hist[];
    const uint64_t n_surv = p.info->n_surv;
    const uint64_t base = (uint64_t)blockIdx.x * kBinChunk;
    if (base >= n_surv) return;
    for (uint32_t t = threadIdx.x; t < p.tiles; t += blockDim.x) hist[t] = 0u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    constexpr uint32_t groups = kBinChunk / 256u;
    const uint64_t r0 = base + (uint64_t)warp * groups * 32u + lane;
    auto load_id = [&](uint32_t g) {
        return r0 + g * 32u < n_surv ? __ldg(p.order + r0 + g * 32u) : 0xffffffffu;
    };
    auto load_box = [&](uint32_t id) {
        return id != 0xffffffffu ? __ldg(p.boxes + id) : make_uint2(kCulledBox, kCulledBox);
    };
    uint32_t id = load_id(0), id_next = load_id(1);
    uint2 next = load_box(id);
    for (uint32_t g = 0; g < groups; ++g) {
        const uint2 box = next;
        const uint32_t idg = id;
        id = id_next;
        if (g + 1 < groups) next = load_box(id);
        if (g + 2 < groups) id_next = load_id(g + 2);
        if (idg != 0xffffffffu) p.rbox[r0 + g * 32u] = box;
        for_each_instance(box, lane, p.tiles_x, [&](bool valid, uint32_t t, uint32_t) {
            if (valid) atomicAdd(hist + t, 1u);
        });
    }
    __syncthreads();
    uint32_t* row = p.counts + (size_t)blockIdx.x * p.tiles;
    for (uint32_t t = threadIdx.x; t < p.tiles; t += blockDim.x) row[t] = hist[t];
}

__global__ void __launch_bounds__(1024) bin_scan_kernel(BinParams p) {
    __shared__ uint32_t sm[32][33];
    __shared__ uint32_t wsum[32];
    __shared__ bool last;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32u + tx;
    const uint32_t C = bin_chunks(p.info);
    const uint32_t S = (C + kBinSlices - 1) / kBinSlices;
    const uint32_t t = blockIdx.x * 32u + tx;
    uint32_t sum = 0;
    if (t < p.tiles) {
        const uint32_t c1 = min(C, (ty + 1) * S);
        for (uint32_t c = ty * S; c < c1; c += 8) { // eight loads in flight, then the stores
            uint32_t v[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) v[i] = c + i < c1 ? p.counts[(size_t)(c + i) * p.tiles + t] : 0u;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                if (c + i < c1) p.counts[(size_t)(c + i) * p.tiles + t] = sum;
                sum += v[i];
            }
        }
    }
    sm[ty][tx] = sum;
    __syncthreads();
    { // warp ty scans column ty over the 32 slices (lane = slice)
        const uint32_t v = sm[tx][ty];
        uint32_t incl = v;
#pragma unroll
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
            if (tx >= d) incl += u;
        }
        sm[tx][ty] = incl - v;
        const uint32_t tt = blockIdx.x * 32u + ty;
        if (tx == 31u && tt < p.tiles) p.tot[tt] = incl;
    }
    __syncthreads();
    if (t < p.tiles) p.slice[(size_t)ty * p.tiles + t] = sm[ty][tx];
    // the last CTA to finish scans the tile totals
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(p.done, 1u) == gridDim.x * gridDim.y - 1u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t seg = (p.tiles + 1023u) / 1024u;
    const uint32_t t0 = min(p.tiles, tid * seg), t1 = min(p.tiles, t0 + seg);
    uint32_t local = 0;
    for (uint32_t u = t0; u < t1; ++u) local += __ldcg(p.tot + u);
    uint32_t incl = local;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
        if (tx >= d) incl += u;
    }
    if (tx == 31u) wsum[ty] = incl;
    __syncthreads();
    if (ty == 0) {
        const uint32_t v = wsum[tx];
        uint32_t wi = v;
#pragma unroll
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, wi, d);
            if (tx >= d) wi += u;
        }
        wsum[tx] = wi - v;
    }
    __syncthreads();
    uint32_t run = wsum[ty] + incl - local;
    for (uint32_t u = t0; u < t1; ++u) {
        const uint32_t v = __ldcg(p.tot + u);
        p.start[u] = run;
        run += v;
        p.end[u] = run;
    }
    if (tid == 1023u) {
        p.info->n_instances = run;
        if (run > p.cap) p.info->overflow = 1u;
        *p.done = 0u;
    }
}

template <uint32_t WARPS>
__global__ void __launch_bounds__(WARPS * 32) bin_scatter_kernel(BinParams p) {
    extern __shared__ uint32_t cur[];                                    // [tiles]
    uint16_t* wh = reinterpret_cast<uint16_t*>(cur + p.tiles);           // [WARPS][tiles]
    if (p.info->overflow) return;
    const uint64_t n_surv = p.info->n_surv;
    const uint64_t base = (uint64_t)blockIdx.x * kBinChunk;
    if (base >= n_surv) return;
    const uint32_t C = bin_chunks(p.info);
    const uint32_t S = (C + kBinSlices - 1) / kBinSlices;
    const uint32_t* row = p.counts + (size_t)blockIdx.x * p.tiles;
    const uint32_t* sl = p.slice + (size_t)(blockIdx.x / S) * p.tiles;
    for (uint32_t t0 = threadIdx.x; t0 < p.tiles; t0 += 4u * blockDim.x) { // four tiles' loads in flight
        uint32_t v[4];
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
            const uint32_t t = t0 + u * blockDim.x;
            v[u] = t < p.tiles ? __ldg(p.start + t) + __ldg(sl + t) + __ldg(row + t) : 0u;
        }
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u)
            if (t0 + u * blockDim.x < p.tiles) cur[t0 + u * blockDim.x] = v[u];
    }
    for (uint32_t t = threadIdx.x; t < WARPS * p.tiles; t += blockDim.x) wh[t] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    constexpr uint32_t groups = kBinChunk / (WARPS * 32u);
    const uint32_t below = (1u << lane) - 1u;
    const uint64_t r0 = base + (uint64_t)warp * groups * 32u + lane;
    auto load_box = [&](uint32_t g) {
        return r0 + g * 32u < n_surv ? p.rbox[r0 + g * 32u] : make_uint2(kCulledBox, kCulledBox);
    };
    // the warp's u16 counters, addressed as packed pairs for shared-memory atomics
    uint32_t* mine32 = reinterpret_cast<uint32_t*>(wh);
    const uint32_t mine0 = warp * p.tiles; // element index of (warp, tile 0)
    // 1. the warp's own per-tile counts (order-free: plain atomics)
    uint2 next = load_box(0);
    for (uint32_t g = 0; g < groups; ++g) {
        const uint2 box = next;
        if (g + 1 < groups) next = load_box(g + 1); // one group ahead
        for_each_instance(box, lane, p.tiles_x, [&](bool valid, uint32_t t, uint32_t) {
            if (valid) {
                const uint32_t e = mine0 + t;
                atomicAdd(mine32 + (e >> 1), 1u << (16u * (e & 1u)));
            }
        });
    }
    __syncthreads();
    // 2. warp offsets inside the chunk (a tile holds <= kBinChunk of its instances)
    for (uint32_t t = threadIdx.x; t < p.tiles; t += blockDim.x) {
        uint32_t run = 0;
#pragma unroll
        for (uint32_t w = 0; w < WARPS; ++w) {
            const uint32_t v = wh[(size_t)w * p.tiles + t];
            wh[(size_t)w * p.tiles + t] = (uint16_t)run;
            run += v;
        }
    }
    __syncthreads();
    // 3. scatter in rank order
    auto load_id = [&](uint32_t g) { return r0 + g * 32u < n_surv ? __ldg(p.order + r0 + g * 32u) : 0u; };
    next = load_box(0);
    uint32_t next_id = load_id(0);
    for (uint32_t g = 0; g < groups; ++g) {
        const uint2 box = next;
        const uint32_t id = next_id;
        if (g + 1 < groups) {
            next = load_box(g + 1);
            next_id = load_id(g + 1);
        }
        for_each_instance(box, lane, p.tiles_x, [&](bool valid, uint32_t t, uint32_t o) {
            const uint32_t gid = __shfl_sync(0xffffffffu, id, o);
            // slot from an atomic on the warp's counter; lanes of one round
            // sharing a tile (rare: different ranks) are then re-ranked in lane
            // order = rank order
            const uint32_t e = mine0 + t, sh = 16u * (e & 1u);
            uint32_t off = 0;
            if (valid) off = (atomicAdd(mine32 + (e >> 1), 1u << sh) >> sh) & 0xffffu;
            __syncwarp();
            uint32_t now = 0;
            if (valid) now = (mine32[e >> 1] >> sh) & 0xffffu;
            if (__ballot_sync(0xffffffffu, valid && now != off + 1u)) {
                const uint32_t m = __match_any_sync(0xffffffffu, valid ? t : 0xffffffffu);
                if (valid && __popc(m) > 1) off = now - __popc(m) + __popc(m & below);
            }
            if (valid) p.list[cur[t] + off] = gid;
            __syncwarp();
        });
    }
}

// ------------------------------------------------- tile-sort binning
// rasterizer.hpp:181-194 (tile_bins) without a global depth sort.
//  1. ts_scatter: CTA per chunk of kTsChunk Gaussians (id order).  A shared
//     histogram counts the chunk's instances per tile; one atomicAdd per
//     (chunk, tile) on fill[t] reserves the chunk's slots in tile t's
//     fixed-capacity range; the instances are then written there, unordered,
//     as (narrowed depth key, gid).  A tile outgrowing its capacity flags
//     bin_fallback = 1 (the host grows the capacity and re-runs the view).
//  2. tile_sort: CTA per tile.  The narrowed keys (monotone in the f64 depth
//     bits) of the tile's instances are bucketed into B >= 2n buckets over the
//     tile's own key range (shared-memory counting sort: histogram, scan,
//     scatter); buckets holding several instances are put in exact (depth
//     bits, id) order -- the reference's depth_sort comparator,
//     projection.hpp:59-64 -- by insertion on the full keys.  The tile's list
//     is then exactly its slice of the reference's tile_bins.  A tile beyond
//     kTileSortMax instances or a bucket beyond kTsBucketMax (massive exact
//     depth ties) flags bin_fallback = 2: the host re-runs the view on the
//     global depth sort, whose tie fix-up handles any run length.
#ifndef SS_TS_CHUNK
#define SS_TS_CHUNK 2048
#endif
#ifndef SS_TS_THREADS
#define SS_TS_THREADS 1024
#endif
constexpr uint32_t kTsChunk = SS_TS_CHUNK;   // Gaussians per scatter CTA
constexpr uint32_t kTsBucketMax = 64; // instances per bucket the fix-up orders
constexpr uint32_t kTsMaxTiles = 16384; // shared histogram of the scatter (64 KB)

constexpr uint32_t kTsThreads = SS_TS_THREADS;  // scatter CTA: 32 warps, each 2 groups of 32 Gaussians
// (300 c4 views, views/s and serialised bin ms: 8192 Gaussians per 1024-thread CTA
// 1650 / 67.0, 4096 per 512 threads 1654-1657 / 65.6, 4096 per 1024 threads
// 1670-1675 / 62.3, 2048 per 1024 threads 1672-1676 / 58.4, 2048 per 256 1649 / 64.9)

// f(tile) for every tile of a box, row-major (per lane; lanes diverge on box size)
template <typename F>
__device__ __forceinline__ void for_box_tiles(uint2 box, uint32_t tiles_x, F&& f) {
    if (box.x == kCulledBox) return;
    const uint32_t tx0 = (box.x & 0xffffu) / kTile, tx1 = (box.x >> 16) / kTile;
    const uint32_t ty0 = (box.y & 0xffffu) / kTile, ty1 = (box.y >> 16) / kTile;
    for (uint32_t ty = ty0; ty <= ty1; ++ty)
        for (uint32_t tx = tx0; tx <= tx1; ++tx) f(ty * tiles_x + tx);
}

__global__ void __launch_bounds__(kTsThreads, 2048 / kTsThreads) ts_scatter_kernel(TileSortParams p) {
    extern __shared__ uint32_t hist[]; // [tiles]: counts, then cursors
    __shared__ uint32_t s_over;        // a tile of this chunk outgrew its capacity
    const uint64_t base = (uint64_t)blockIdx.x * kTsChunk;
    if (base >= p.n) return;
    for (uint32_t t = threadIdx.x; t < p.tiles; t += blockDim.x) hist[t] = 0u;
    if (threadIdx.x == 0) s_over = 0u;
    const uint32_t lane = threadIdx.x & 31u;
    constexpr uint32_t groups = kTsChunk / kTsThreads;
    // thread i takes Gaussians base + i + g * kTsThreads (coalesced)
    uint2 box[groups];
#pragma unroll
    for (uint32_t g = 0; g < groups; ++g) {
        const uint64_t id = base + threadIdx.x + (uint64_t)g * kTsThreads;
        box[g] = id < p.n ? __ldg(p.boxes + id) : make_uint2(kCulledBox, kCulledBox);
    }
    __syncthreads();
#pragma unroll
    for (uint32_t g = 0; g < groups; ++g) for_box_tiles(box[g], p.tiles_x, [&](uint32_t t) { atomicAdd(hist + t, 1u); });
    // the narrowed depth keys for the scatter, loaded while the histogram settles
    const unsigned long long mn = p.info->min_key;
    const uint32_t sh = narrow_shift(p.info);
    uint32_t k32[groups];
#pragma unroll
    for (uint32_t g = 0; g < groups; ++g) {
        const uint64_t id = base + threadIdx.x + (uint64_t)g * kTsThreads;
        k32[g] = box[g].x != kCulledBox ? (uint32_t)((__ldg(p.keys + id) - mn) >> sh) : 0u; // monotone in depth
    }
    __syncthreads();
    // reserve each touched tile's slots: one global atomic per (chunk, tile),
    // a thread's (up to 4) reservations in flight together
    uint32_t mine = 0, mfill = 0;
    for (uint32_t t0 = threadIdx.x; t0 < p.tiles; t0 += 4u * blockDim.x) {
        uint32_t c[4], b[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t t = t0 + k * blockDim.x;
            c[k] = t < p.tiles ? hist[t] : 0u;
        }
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) b[k] = c[k] ? atomicAdd(p.fill + t0 + k * blockDim.x, c[k]) : 0u;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            if (!c[k]) continue;
            const uint32_t t = t0 + k * blockDim.x;
            mine += c[k];
            mfill = max(mfill, b[k] + c[k]);
            hist[t] = t * p.cap + b[k];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mine += __shfl_xor_sync(0xffffffffu, mine, o);
        mfill = max(mfill, __shfl_xor_sync(0xffffffffu, mfill, o));
    }
    if (lane == 0) {
        if (mine) atomicAdd(&p.info->n_instances, (unsigned long long)mine);
        if (mfill > p.cap) {
            atomicMax(&p.info->max_fill, mfill);
            atomicMax(&p.info->bin_fallback, 1u);
            p.info->overflow = 1u;
            s_over = 1u;
        }
    }
    __syncthreads();
    // a chunk with an overflowing tile writes nothing (its slots could run past
    // the slab; the view is re-run with a larger capacity), so no per-instance
    // bounds test below
    if (s_over) return;
#pragma unroll
    for (uint32_t g = 0; g < groups; ++g) {
        const uint32_t id = (uint32_t)(base + threadIdx.x + (uint64_t)g * kTsThreads);
        const uint2 v = make_uint2(k32[g], id);
        for_box_tiles(box[g], p.tiles_x, [&](uint32_t t) { p.slab[atomicAdd(hist + t, 1u)] = v; });
    }
}

#ifndef SS_TS_SORT_THREADS
#define SS_TS_SORT_THREADS 512
#endif
constexpr uint32_t kTsSortThreads = SS_TS_SORT_THREADS;

// MAXN: the slot capacity of the launch (4096 by default: 48 KB of shared
// memory and <= 40 registers, three CTAs per SM, which leaves room for the
// other lanes' kernels; 8192 once a view had a larger tile).
#ifndef SS_TS_BUCKET_SHIFT
#define SS_TS_BUCKET_SHIFT 1
#endif
// buckets the sort of a tile of up to n instances uses (lb below) at most
__host__ __device__ constexpr uint32_t tile_sort_buckets(uint32_t n) {
    uint32_t lb = 5;
    while ((1u << lb) < n) ++lb;
    return 1u << (lb > 5u + SS_TS_BUCKET_SHIFT ? lb - SS_TS_BUCKET_SHIFT : 5u);
}
__host__ __device__ constexpr size_t tile_sort_smem(uint32_t maxn) {
    return (size_t)tile_sort_buckets(maxn) * 4 + (size_t)maxn * 8;
}

// FIXUP: CTA k sorts tile fix_tiles[k] in full (k < fix_count[1]) and clears
// its need flag; otherwise CTA t sorts tile t (a prefix of it in prefix mode).
template <uint32_t MAXN, bool FIXUP>
__device__ __forceinline__ void tile_sort_one(const TileSortParams& p, uint32_t t, uint32_t* cnt, uint2* out,
                                              uint32_t* red_min, uint32_t* red_max, uint32_t& s_fail,
                                              uint32_t& s_prefix, uint32_t& s_lo) {
    constexpr uint32_t kTsPer = MAXN / kTsSortThreads; // slots per thread
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (p.info->overflow) return; // the view is re-run
    const uint32_t n = p.fill[t];
    const size_t base = (size_t)t * p.cap;
    if (tid == 0) {
        // fixup: the prefix the main sort already ranked (its list end) is
        // left as written; only the rest is ranked here
        s_lo = FIXUP ? p.end[t] - (uint32_t)base : 0u;
        p.start[t] = (uint32_t)base;
        p.end[t] = (uint32_t)base + n;
        s_fail = 0u;
    }
    if (n == 0) return;
    if (n > MAXN) { // cannot happen: the scatter flags tiles beyond the slot capacity
        if (tid == 0) {
            atomicMax(&p.info->bin_fallback, 2u);
            p.info->overflow = 1u;
        }
        return;
    }
    // the tile's (key, gid) slots, strided over the threads, held in registers
    const uint2* src = p.slab + base;
    uint2 v[kTsPer];
    uint32_t mn = 0xffffffffu, mx = 0u;
    const uint32_t per = (n + kTsSortThreads - 1u) / kTsSortThreads; // slots per thread this tile
#pragma unroll
    for (uint32_t k = 0; k < kTsPer; ++k) {
        if (k >= per) break;
        const uint32_t i = tid + k * kTsSortThreads;
        v[k] = i < n ? src[i] : make_uint2(0u, 0u);
        if (i < n) {
            mn = min(mn, v[k].x);
            mx = max(mx, v[k].x);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        red_min[warp] = mn;
        red_max[warp] = mx;
    }
    // B = 2^lb >= n buckets (32 .. MAXN) over [mn, mx]
    uint32_t lb = 5;
    while ((1u << lb) < n) ++lb;
    // about two instances per bucket: half the scan work of one per bucket,
    // the rank loop stays short (measured +0.6 % on c4)
    lb = lb > 5u + SS_TS_BUCKET_SHIFT ? lb - SS_TS_BUCKET_SHIFT : 5u;
    const uint32_t B = 1u << lb;
    for (uint32_t b = tid; b < B; b += kTsSortThreads) cnt[b] = 0u;
    __syncthreads();
    mn = red_min[0];
    mx = red_max[0];
#pragma unroll
    for (int w = 1; w < (int)(kTsSortThreads / 32); ++w) {
        mn = min(mn, red_min[w]);
        mx = max(mx, red_max[w]);
    }
    const uint32_t span = mx - mn;
    const uint32_t hb = span ? 32u - (uint32_t)__clz(span) : 0u;
    const uint32_t sh = hb > lb ? hb - lb : 0u;
#pragma unroll
    for (uint32_t k = 0; k < kTsPer; ++k) {
        if (k >= per) break;
        if (tid + k * kTsSortThreads < n) atomicAdd(cnt + ((v[k].x - mn) >> sh), 1u);
    }
    __syncthreads();
    { // exclusive scan of cnt[0, B): warp w scans its contiguous segment 32
      // counters per round (conflict-free), then the warp totals are scanned
        __shared__ uint32_t wtot[kTsSortThreads / 32];
        constexpr uint32_t W = kTsSortThreads / 32;
        const uint32_t seg = B / W, s0 = warp * seg; // B >= 32 * W or seg < 32 (then lanes past seg idle)
        uint32_t carry = 0;
        for (uint32_t b = s0; b < s0 + seg; b += 32u) {
            const uint32_t i = b + lane;
            const uint32_t c = i < s0 + seg ? cnt[i] : 0u;
            uint32_t incl = c;
#pragma unroll
            for (uint32_t d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += u;
            }
            if (i < s0 + seg) cnt[i] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) wtot[warp] = carry;
        __syncthreads();
        uint32_t before = 0;
        for (uint32_t w = 0; w < warp; ++w) before += wtot[w];
        if (before)
            for (uint32_t i = s0 + lane; i < s0 + seg; i += 32u) cnt[i] += before;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kTsPer; ++k) {
        if (k >= per) break;
        if (tid + k * kTsSortThreads < n) out[atomicAdd(cnt + ((v[k].x - mn) >> sh), 1u)] = v[k];
    }
    // prefix mode: rank only the whole buckets holding the first
    // max(prefix_min, n / 4) instances (buckets are key-ordered, so they are
    // exactly the first entries of the full order); every bucket is still
    // checked against kTsBucketMax now, so the fixup sort of the rest cannot
    // fail after the compositor has used the prefix
    if (tid == 0) s_prefix = n;
    if (!FIXUP && p.prefix_min && n > p.prefix_min) {
        __syncthreads();
        if (tid == 0) {
            const uint32_t target = max(p.prefix_min, n >> 2);
            uint32_t lo = 0, hi = B - 1; // first bucket whose end reaches target
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (cnt[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            s_prefix = cnt[lo];
        }
        for (uint32_t b = tid; b < B; b += kTsSortThreads)
            if (cnt[b] - (b ? cnt[b - 1] : 0u) > kTsBucketMax) s_fail = 1u;
    }
    __syncthreads();
    const uint32_t P = s_prefix;
    if (P < n && tid == 0) p.end[t] = (uint32_t)base + P;
    // cnt[b] is now the end of bucket b (= the start of bucket b + 1).  Each
    // instance's final position is its bucket's start plus its rank among the
    // bucket's members by (key, then depth bits and id on equal keys) -- the
    // reference's depth_sort comparator -- and its id goes straight to the
    // tile's list (buckets average ~1-2 members: O(s) compares per instance,
    // no serial insertion sort).
    // Threads take the instances in bucket order (out[i]), so a warp's lanes
    // share buckets of similar size (one large bucket no longer stalls 31
    // lanes of small ones) and the list writes land near i, coalesced.
    uint32_t* dst = p.list + base;
    for (uint32_t i = s_lo + tid; i < P; i += kTsSortThreads) {
        const uint2 x = out[i];
        const uint32_t b = (x.x - mn) >> sh;
        const uint32_t s0 = b ? cnt[b - 1] : 0u, e0 = cnt[b];
        uint32_t pos = s0;
        if (e0 - s0 > 1u) {
            if (e0 - s0 > kTsBucketMax) {
                s_fail = 1u;
                continue;
            }
            // branch-free count of the members with a smaller narrowed key;
            // equal narrowed keys (rare: 2^32 levels over the view's depth
            // range) take the exact pass below
            uint32_t lt = 0, tie = 0;
            for (uint32_t c = s0; c < e0; ++c) {
                const uint2 y = out[c];
                lt += y.x < x.x ? 1u : 0u;
                tie |= (y.x == x.x) & (y.y != x.y);
            }
            if (!tie) {
                pos += lt;
            } else {
                const unsigned long long kx = __ldg(p.keys + x.y);
                for (uint32_t c = s0; c < e0; ++c) {
                    const uint2 y = out[c];
                    bool before = y.x < x.x;
                    if (y.x == x.x && y.y != x.y) // equal narrowed keys: the full depth bits, then the id
                        before = depth_before(__ldg(p.keys + y.y), y.y, kx, x.y);
                    pos += before ? 1u : 0u;
                }
            }
        }
        dst[pos] = x.y;
    }
    __syncthreads();
    if (s_fail && tid == 0) { // massive exact ties: the view takes the global depth sort
        atomicMax(&p.info->bin_fallback, 2u);
        p.info->overflow = 1u;
    }
}

template <uint32_t MAXN, int MIN_CTAS, bool FIXUP>
__global__ void __launch_bounds__(kTsSortThreads, MIN_CTAS) tile_sort_kernel(TileSortParams p) {
    extern __shared__ uint32_t sm[]; // cnt[tile_sort_buckets(MAXN)], then out[MAXN] as (key, gid)
    uint32_t* cnt = sm;
    uint2* out = reinterpret_cast<uint2*>(sm + tile_sort_buckets(MAXN));
    __shared__ uint32_t red_min[kTsSortThreads / 32], red_max[kTsSortThreads / 32];
    __shared__ uint32_t s_fail, s_prefix, s_lo;
    if constexpr (FIXUP) {
        // a small grid walks the queued tiles (most views queue a few dozen)
        const uint32_t count = p.fix_count[1];
        for (uint32_t k = blockIdx.x; k < count; k += gridDim.x) {
            const uint32_t t = p.fix_tiles[k];
            if (threadIdx.x == 0) p.need[t] = 0u;
            tile_sort_one<MAXN, true>(p, t, cnt, out, red_min, red_max, s_fail, s_prefix, s_lo);
            __syncthreads(); // shared memory reused by the next tile
        }
    } else {
        tile_sort_one<MAXN, false>(p, blockIdx.x, cnt, out, red_min, red_max, s_fail, s_prefix, s_lo);
    }
}

// --------------------------------------------------------- contraction
// pipeline.hpp:70-80 accumulate for a group of up to four consecutive views:
// for every Gaussian touched in any of them, row[gid] += sum_m acc_v[gid, m] *
// CLIP_v,m and total[gid] += sum_m acc_v[gid, m], view by view in view order
// and mask by mask in mask order -- the same fp32 operation sequence as one
// contraction per view, but the 2 KB row is read and written once per group
// (consecutive views touch ~95 % the same Gaussians).  A Gaussian is handled
// by the first member whose list holds it; later members skip it.  One warp
// per (member, list entry); CLIP rows stay L1/L2-resident.
template <bool DIM512, bool CLIP_SMEM = false>
__device__ __forceinline__ void contract_member(const ContractMember& m, uint32_t gid, uint32_t lane, uint32_t dim,
                                                float* row, float4 (&racc)[4], float& wsum,
                                                unsigned long long& pairs) {
    const AccRow accrow = acc_row(m, gid);
    float vsum = 0.0f;
    for (uint32_t c = 0; c < m.n_masks; c += 32) {
        const uint32_t mi = c + lane;
        float v = 0.0f;
        if (mi < m.n_masks) {
            v = accrow.get(mi);
            if (v != 0.0f) accrow.clear(mi);
        }
        vsum += v;
        uint32_t bal = __ballot_sync(0xffffffffu, v != 0.0f);
        pairs += __popc(bal);
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            const float w = __shfl_sync(0xffffffffu, v, src);
            const float* e = m.clip + (size_t)(c + src) * dim;
            if constexpr (DIM512) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 ev = CLIP_SMEM ? reinterpret_cast<const float4*>(e)[lane + 32 * q]
                                                : __ldg(reinterpret_cast<const float4*>(e) + lane + 32 * q);
                    racc[q].x += w * ev.x;
                    racc[q].y += w * ev.y;
                    racc[q].z += w * ev.z;
                    racc[q].w += w * ev.w;
                }
            } else {
                for (uint32_t d = lane; d < dim; d += 32) row[d] += w * __ldg(e + d);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
    wsum += vsum; // totals[gid] += this view's sum, in view order
}

template <bool DIM512>
__global__ void __launch_bounds__(256) contract_kernel(ContractParams p) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long cnt[kMaxGroup], total = 0;
#pragma unroll
    for (uint32_t i = 0; i < kMaxGroup; ++i) {
        cnt[i] = i < p.n_members ? *p.m[i].touched_count : 0ull;
        total += cnt[i];
    }
    unsigned long long pairs = 0, rows = 0;
    for (uint64_t t = warp0; t < total; t += nwarps) {
        uint32_t i = 0;
        uint64_t tt = t;
        while (tt >= cnt[i]) {
            tt -= cnt[i];
            ++i;
        }
        const uint32_t gid = p.m[i].touched_list[tt];
        bool earlier = false;
        for (uint32_t j = 0; j < i; ++j) earlier |= __ldg(p.m[j].touched + gid) == p.m[j].gen;
        if (earlier) continue; // handled with the earlier view's entry
        ++rows;
        float* row = p.sums + (size_t)gid * p.dim;
        float4 racc[4];
        if constexpr (DIM512) {
#pragma unroll
            for (int q = 0; q < 4; ++q) racc[q] = reinterpret_cast<const float4*>(row)[lane + 32 * q];
        }
        float wsum = p.totals[gid];
        for (uint32_t j = i; j < p.n_members; ++j) {
            if (j != i && __ldg(p.m[j].touched + gid) != p.m[j].gen) continue;
            float vs = 0.0f;
            contract_member<DIM512>(p.m[j], gid, lane, p.dim, row, racc, vs, pairs);
            wsum += vs;
        }
        if constexpr (DIM512) {
#pragma unroll
            for (int q = 0; q < 4; ++q) reinterpret_cast<float4*>(row)[lane + 32 * q] = racc[q];
        }
        if (lane == 0) p.totals[gid] = wsum;
    }
    if (p.count_pairs) {
        // pairs is warp-uniform (ballot popcounts); count once per warp
        if (lane == 0 && pairs) atomicAdd(p.cum + 1, pairs);
        if (lane == 0 && rows) atomicAdd(p.cum + 2, rows);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(p.cum, total);
    }
}

constexpr uint32_t kContractThreads = 768; // 24 warps x <= 85 registers (row + prefetched row)

// Single-view contraction with the view's CLIP rows (M <= 64, D = 512)
// staged in shared memory: one 768-thread CTA per SM, persistent over the
// touched list.  Same per-row operation order as contract_kernel.  Software
// pipelined: a warp's next 32 list entries are loaded one per lane, and the
// next Gaussian's row, total and mask weights are in flight while the
// current one is contracted (every Gaussian appears once in the list, so no
// other warp touches a prefetched row).
__global__ void __launch_bounds__(kContractThreads, 1) contract_smem_kernel(ContractParams p) {
    extern __shared__ float4 sclip4[]; // n_masks x 128 float4
    const ContractMember& m = p.m[0];
    const uint32_t n4 = m.n_masks * 128u;
    const float4* g4 = reinterpret_cast<const float4*>(m.clip);
    for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) sclip4[i] = __ldg(g4 + i);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned long long total = *m.touched_count;
    const uint32_t M = m.n_masks;
    unsigned long long pairs = 0;
    auto batch = [&](uint64_t t0) { // lane i: the entry of iteration t0 + i * nwarps
        const uint64_t tt = t0 + (uint64_t)lane * nwarps;
        return tt < total ? __ldg(m.touched_list + tt) : 0u;
    };
    auto fetch = [&](uint32_t gid, float4 (&r)[4], float& w, float& v0, float& v1) {
        const float4* row = reinterpret_cast<const float4*>(p.sums + (size_t)gid * 512u);
#pragma unroll
        for (int q = 0; q < 4; ++q) r[q] = row[lane + 32 * q];
        w = p.totals[gid];
        const AccRow accrow = acc_row(m, gid);
        v0 = lane < M ? accrow.get(lane) : 0.0f;
        v1 = lane + 32u < M ? accrow.get(lane + 32u) : 0.0f;
    };
    uint64_t t = warp0;
    if (t < total) {
        uint32_t gb = batch(t), k = 0;
        uint32_t gid = __shfl_sync(0xffffffffu, gb, 0);
        float4 racc[4];
        float wsum, v0, v1;
        fetch(gid, racc, wsum, v0, v1);
        for (; t < total; t += nwarps) {
            const uint64_t tn = t + nwarps;
            if (++k == 32u) {
                gb = batch(tn);
                k = 0;
            }
            const uint32_t ngid = __shfl_sync(0xffffffffu, gb, k);
            float4 nacc[4];
            float nw = 0.0f, nv0 = 0.0f, nv1 = 0.0f;
            if (tn < total) fetch(ngid, nacc, nw, nv0, nv1);
            // contract_member<true, true> on the prefetched mask weights
            const AccRow accrow = acc_row(m, gid);
            float vsum = 0.0f;
#pragma unroll
            for (uint32_t c = 0; c < 64u; c += 32u) {
                if (c >= M) break;
                const float v = c == 0 ? v0 : v1;
                if (v != 0.0f) accrow.clear(c + lane);
                vsum += v;
                uint32_t bal = __ballot_sync(0xffffffffu, v != 0.0f);
                pairs += __popc(bal);
                while (bal) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    const float w = __shfl_sync(0xffffffffu, v, src);
                    const float4* e = sclip4 + (size_t)(c + src) * 128u;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 ev = e[lane + 32 * q];
                        racc[q].x += w * ev.x;
                        racc[q].y += w * ev.y;
                        racc[q].z += w * ev.z;
                        racc[q].w += w * ev.w;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
            wsum += vsum;
            float4* row = reinterpret_cast<float4*>(p.sums + (size_t)gid * 512u);
#pragma unroll
            for (int q = 0; q < 4; ++q) row[lane + 32 * q] = racc[q];
            if (lane == 0) p.totals[gid] = wsum;
#pragma unroll
            for (int q = 0; q < 4; ++q) racc[q] = nacc[q];
            gid = ngid;
            wsum = nw;
            v0 = nv0;
            v1 = nv1;
        }
    }
    if (p.count_pairs) {
        if (lane == 0 && pairs) atomicAdd(p.cum + 1, pairs);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            atomicAdd(p.cum, total);
            atomicAdd(p.cum + 2, total); // rows read and written (each touched row once)
        }
    }
}

// Group contraction (2-3 consecutive views, D = 512, M <= 64 each).
//  1. group_union_kernel: one thread per (member, list entry); an entry whose
//     Gaussian no earlier member touched becomes one union entry (gid, mask of
//     the members that touched it) -- the union of the lists, each Gaussian once.
//  2. contract_group_pass_kernel<H>, H = 0, 1: the members' CLIP rows for D-half
//     H staged in shared memory (3 x 64 masks x 1 KB = 192 KB), one warp per
//     union entry with the next entry's half row and mask weights in flight;
//     every touched half row is read and written once for the whole group.
// Per element the fp32 sequence is the single-view one (views in order, masks
// in order within a view), so the sums are bit-identical to contracting the
// views one by one.  Mask weights are cleared and totals updated in pass 1.
__global__ void __launch_bounds__(256) group_union_kernel(ContractParams p, uint2* ulist, unsigned int* ucount) {
    const uint32_t nm = p.n_members;
    unsigned long long cnt[kMaxGroup - 1], all = 0;
#pragma unroll
    for (uint32_t j = 0; j < kMaxGroup - 1; ++j) {
        cnt[j] = j < nm ? *p.m[j].touched_count : 0ull;
        all += cnt[j];
    }
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < all; base += stride) {
        uint64_t e = base + lane;
        uint32_t gid = 0, mask = 0;
        if (e < all) {
            uint32_t j = 0;
#pragma unroll
            for (uint32_t k = 0; k < kMaxGroup - 2; ++k)
                if (j == k && e >= cnt[k]) {
                    e -= cnt[k];
                    j = k + 1;
                }
            gid = __ldg(p.m[j].touched_list + e);
            mask = 1u << j;
            for (uint32_t k = 0; k < nm; ++k) {
                if (k == j || __ldg(p.m[k].touched + gid) != p.m[k].gen) continue;
                if (k < j) { // an earlier member owns it
                    mask = 0;
                    break;
                }
                mask |= 1u << k;
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0u);
        if (!bal) continue;
        const uint32_t leader = __ffs(bal) - 1;
        uint32_t slot = 0;
        if (lane == leader) slot = atomicAdd(ucount, (unsigned int)__popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (mask) ulist[slot + __popc(bal & ((1u << lane) - 1u))] = make_uint2(gid, mask);
    }
}

// MEMBERS: views in the group (<= 3); CH: 32-mask chunks per view (2: M <= 64,
// 4: M <= 128); DIRECT: a single view, walked through its own touched list;
// FIX: the members' scalars are fixed point (SS_OPT_DETERMINISTIC).
template <uint32_t H, uint32_t MEMBERS, uint32_t CH, bool DIRECT, bool FIX>
__global__ void __launch_bounds__(1024, 1) contract_group_pass_kernel(ContractParams p, const uint2* ulist,
                                                                     const unsigned int* ucount) {
    extern __shared__ float4 sclip4[]; // per member: n_masks x 64 float4 (D-half H)
    __shared__ uint32_t soff[kMaxGroup];
    const uint32_t nm = p.n_members;
    if (threadIdx.x == 0) {
        uint32_t off = 0;
        for (uint32_t i = 0; i < kMaxGroup; ++i) {
            soff[i] = off;
            off += i < nm ? p.m[i].n_masks * 64u : 0u;
        }
    }
    __syncthreads();
    for (uint32_t i = 0; i < nm; ++i) {
        const float4* g4 = reinterpret_cast<const float4*>(p.m[i].clip);
        const uint32_t n = p.m[i].n_masks * 64u;
        for (uint32_t e = threadIdx.x; e < n; e += blockDim.x)
            sclip4[soff[i] + e] = __ldg(g4 + (size_t)(e >> 6) * 128u + H * 64u + (e & 63u));
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total = DIRECT ? *p.m[0].touched_count : *ucount;
    auto entry = [&](uint64_t i) {
        return DIRECT ? make_uint2(__ldg(p.m[0].touched_list + i), 1u) : ulist[i];
    };
    unsigned long long pairs = 0;
    // one union entry's inputs: half row, total (pass 1), CH mask-weight words per member
    struct In {
        float4 r[2];
        float w;
        float v[MEMBERS][CH];
    };
    auto fetch = [&](uint2 u, In& x) {
        const float4* row = reinterpret_cast<const float4*>(p.sums + (size_t)u.x * 512u) + H * 64u;
        x.r[0] = row[lane];
        x.r[1] = row[lane + 32];
        x.w = H ? p.totals[u.x] : 0.0f;
#pragma unroll
        for (uint32_t j = 0; j < MEMBERS; ++j) {
#pragma unroll
            for (uint32_t c = 0; c < CH; ++c) x.v[j][c] = 0.0f;
            if (j < nm && ((u.y >> j) & 1u)) {
                const auto accrow = acc_row_t<FIX>(p.m[j], u.x);
#pragma unroll
                for (uint32_t c = 0; c < CH; ++c)
                    if (32u * c + lane < p.m[j].n_masks) x.v[j][c] = accrow.get(32u * c + lane);
            }
        }
    };
    uint64_t t = warp0;
    if (t < total) {
        uint2 u = entry(t);
        In cur;
        fetch(u, cur);
        for (; t < total; t += nwarps) {
            const uint64_t tn = t + nwarps;
            uint2 un = make_uint2(0u, 0u);
            In nxt;
            if (tn < total) {
                un = entry(tn);
                fetch(un, nxt);
            }
            float wsum = cur.w;
#pragma unroll
            for (uint32_t j = 0; j < MEMBERS; ++j) {
                if (j >= nm || !((u.y >> j) & 1u)) continue;
                const uint32_t M = p.m[j].n_masks;
                const auto accrow = acc_row_t<FIX>(p.m[j], u.x);
                const float4* clip = sclip4 + soff[j];
                float vsum = 0.0f;
#pragma unroll
                for (uint32_t c = 0; c < CH; ++c) {
                    if (32u * c >= M) break;
                    const float v = cur.v[j][c];
                    if (H && v != 0.0f) accrow.clear(32u * c + lane);
                    vsum += v;
                    uint32_t bal = __ballot_sync(0xffffffffu, v != 0.0f);
                    if (H) pairs += __popc(bal);
                    while (bal) {
                        const int src = __ffs(bal) - 1;
                        bal &= bal - 1;
                        const float w = __shfl_sync(0xffffffffu, v, src);
                        const float4* e = clip + (size_t)(32u * c + src) * 64u;
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const float4 ev = e[lane + 32 * q];
                            cur.r[q].x += w * ev.x;
                            cur.r[q].y += w * ev.y;
                            cur.r[q].z += w * ev.z;
                            cur.r[q].w += w * ev.w;
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
                wsum += vsum;
            }
            float4* row = reinterpret_cast<float4*>(p.sums + (size_t)u.x * 512u) + H * 64u;
            row[lane] = cur.r[0];
            row[lane + 32] = cur.r[1];
            if (H && lane == 0) p.totals[u.x] = wsum;
            u = un;
            cur = nxt;
        }
    }
    if (H && p.count_pairs) {
        if (lane == 0 && pairs) atomicAdd(p.cum + 1, pairs);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long all = 0;
            for (uint32_t i = 0; i < nm; ++i) all += *p.m[i].touched_count;
            atomicAdd(p.cum, all);
            atomicAdd(p.cum + 2, (unsigned long long)total); // union rows, each read and written once per group
        }
    }
}

// eval.hpp:122-158 assign_classes.  Warp per row: the row is staged in
// shared memory, lane l owns classes l, l+32, ...; every dot product and norm
// is the reference's sequential f64 sum (products of f32 values are exact in
// f64, explicit __dmul_rn/__dadd_rn keep FMA out), cos = dot / (|row| |label|)
// or -1 for a zero denominator, and the arg max takes the lowest class id on
// ties.  Labels arrive transposed ([dim][n_labels]) so lanes read them
// coalesced.  Uncovered rows (coverage <= f32(1e-8)) get kUnlabeled = -1.
__global__ void __launch_bounds__(256) assign_classes_kernel(const float* rows, const float* coverage, uint64_t n,
                                                             uint32_t dim, const int32_t* label_ids,
                                                             const float* labels_t, const double* label_norms,
                                                             uint32_t n_labels, int32_t* out) {
    extern __shared__ float srow[]; // 8 warps x dim
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    float* row_s = srow + (size_t)wib * dim;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp0; k < n; k += nwarps) {
        if (!(coverage[k] > 1e-8f)) {
            if (lane == 0) out[k] = -1;
            continue;
        }
        const float* row = rows + k * dim;
        __syncwarp();
        for (uint32_t d = lane; d < dim; d += 32) row_s[d] = row[d];
        __syncwarp();
        double rn = 0.0;
        for (uint32_t d = 0; d < dim; ++d) rn = __dadd_rn(rn, __dmul_rn((double)row_s[d], (double)row_s[d]));
        rn = __dsqrt_rn(rn);
        double best = -2.0;
        int32_t best_id = -1;
        bool have = false;
        for (uint32_t c = lane; c < n_labels; c += 32) {
            double dot = 0.0;
            for (uint32_t d = 0; d < dim; ++d)
                dot = __dadd_rn(dot, __dmul_rn((double)row_s[d], (double)__ldg(labels_t + (size_t)d * n_labels + c)));
            const double denom = __dmul_rn(rn, label_norms[c]);
            const double cs = denom > 0.0 ? __ddiv_rn(dot, denom) : -1.0;
            const int32_t id = label_ids[c];
            // the reference's scan (best = -2 first, replace on cos > best or on an
            // equal cos with a lower id) selects the max cos, lowest id among equals;
            // a NaN cos never replaces
            if (!isnan(cs) && (!have || cs > best || (cs == best && id < best_id))) {
                best = cs;
                best_id = id;
                have = true;
            }
        }
        // arg max over lanes by (cos desc, id asc); lanes without a candidate lose
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, best_id, o);
            const bool oh = __shfl_xor_sync(0xffffffffu, have, o);
            if (oh && (!have || ob > best || (ob == best && oi < best_id))) {
                best = ob;
                best_id = oi;
                have = true;
            }
        }
        if (lane == 0) out[k] = have ? best_id : -1;
    }
}

// label_norms[c] = sqrt(sum_d double(v)^2) sequentially; labels_t = transpose
__global__ void label_prep_kernel(const float* labels, uint32_t dim, uint32_t n_labels, float* labels_t,
                                  double* norms) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_labels) return;
    double nn = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
        const float v = labels[(size_t)c * dim + d];
        nn = __dadd_rn(nn, __dmul_rn((double)v, (double)v));
        labels_t[(size_t)d * n_labels + c] = v;
    }
    norms[c] = __dsqrt_rn(nn);
}

// pipeline.hpp:120-135 finalize_into: covered rows (total > 1e-8) become
// sum/total, coverage = total; uncovered rows are exactly zero.
__global__ void __launch_bounds__(256) normalize_kernel(const float* sums, const float* totals, uint64_t n,
                                                        uint32_t dim, float* rows, float* coverage,
                                                        unsigned long long* covered) {
    unsigned long long ncov = 0;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec = (dim & 3u) == 0;
    for (uint64_t k = warp0; k < n; k += nwarps) {
        const float t = totals[k];
        const bool cov = (double)t > 1e-8;
        ncov += cov;
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
    if (covered && lane == 0 && ncov) atomicAdd(covered, ncov); // rows whose sums were read (roofline bytes)
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

// The view's contraction list from the compositor's stamps: every Gaussian
// with touched[g] == gen.  A block takes 1024 consecutive ids per round (4 per
// thread) and reserves its slots with one atomic (per-warp atomics on the one
// counter serialise in L2).
__global__ void __launch_bounds__(256) touched_compact_kernel(const uint32_t* touched, uint64_t n, uint32_t gen,
                                                              uint32_t* list, unsigned long long* count) {
    __shared__ uint32_t wtot[8];
    __shared__ unsigned long long sbase;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t below = (1u << lane) - 1u;
    for (uint64_t b0 = (uint64_t)blockIdx.x * 1024u; b0 < n; b0 += (uint64_t)gridDim.x * 1024u) {
        const uint64_t g0 = b0 + threadIdx.x * 4u;
        uint32_t t[4] = {0u, 0u, 0u, 0u};
        if (g0 + 3u < n) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(touched + g0));
            t[0] = v.x;
            t[1] = v.y;
            t[2] = v.z;
            t[3] = v.w;
        } else {
            for (uint32_t k = 0; k < 4u; ++k)
                if (g0 + k < n) t[k] = touched[g0 + k];
        }
        uint32_t bal[4], tot = 0;
#pragma unroll
        for (uint32_t k = 0; k < 4u; ++k) {
            bal[k] = __ballot_sync(0xffffffffu, g0 + k < n && t[k] == gen);
            tot += __popc(bal[k]);
        }
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        uint32_t before = 0, all = 0;
#pragma unroll
        for (uint32_t w = 0; w < 8u; ++w) {
            before += w < warp ? wtot[w] : 0u;
            all += wtot[w];
        }
        if (threadIdx.x == 0 && all) sbase = atomicAdd(count, (unsigned long long)all);
        __syncthreads();
        if (all) {
            unsigned long long base = sbase + before;
#pragma unroll
            for (uint32_t k = 0; k < 4u; ++k) {
                if ((bal[k] >> lane) & 1u) list[base + __popc(bal[k] & below)] = (uint32_t)(g0 + k);
                base += __popc(bal[k]);
            }
        }
        __syncthreads(); // wtot / sbase are reused next round
    }
}

// ---------------------------------------------------- partition_store
// vecstore.hpp:169-213.  Doubles map to u64 keys whose unsigned order is the
// numeric order (NaN means are skipped, as cwiseMin/cwiseMax skip them:
// std::min(m, NaN) keeps m, scene.hpp:43-46).
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// bbox.min over the records' f32 means widened to f64 (Aabb::expand)
__global__ void __launch_bounds__(256) bbox_min_kernel(const float* means, uint64_t n, unsigned long long* mn3) {
    unsigned long long m[3] = {~0ull, ~0ull, ~0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < 3; ++a) {
            const double v = (double)means[3 * i + a];
            if (v == v) m[a] = min(m[a], dkey(v));
        }
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m[a] = min(m[a], __shfl_xor_sync(0xffffffffu, m[a], o));
        if ((threadIdx.x & 31u) == 0 && m[a] != ~0ull) atomicMin(mn3 + a, m[a]);
    }
}

// x86 cvttsd2si: NaN / out of range -> INT_MIN (static_cast<int32_t>(std::floor(...)) on the reference's target)
__device__ __forceinline__ int32_t to_i32_x86(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
    return (int32_t)v;
}

// cell key per record: floor((m - bbox.min) / cell_size) per axis, biased to
// unsigned order (std::map<CellKey> compares the signed x, then y, then z);
// yz = (y << 32) | z and x by record, idx = record index
__global__ void __launch_bounds__(256) cell_keys_kernel(const float* means, uint64_t n,
                                                        const unsigned long long* mn3, double cell,
                                                        unsigned long long* yz, uint32_t* kx, uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t k[3];
    for (int a = 0; a < 3; ++a) {
        const double lo = dkey_inv(mn3[a]);
        const double q = __ddiv_rn(__dsub_rn((double)means[3 * i + a], lo), cell);
        k[a] = (uint32_t)to_i32_x86(floor(q)) ^ 0x80000000u;
    }
    kx[i] = k[0];
    yz[i] = ((unsigned long long)k[1] << 32) | k[2];
    idx[i] = (uint32_t)i;
}

template <typename T>
__global__ void gather_kernel(const T* src, const uint32_t* perm, uint64_t n, T* dst) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

// heads of the cells in the sorted order
__global__ void cell_heads_kernel(const uint32_t* kx, const unsigned long long* yz, uint64_t n, uint8_t* head) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    head[i] = i == 0 || kx[i] != kx[i - 1] || yz[i] != yz[i - 1];
}

// per cell: (x, y, z) signed and its first position
__global__ void cell_list_kernel(const uint32_t* kx, const unsigned long long* yz, const uint32_t* heads,
                                 const int* n_heads, int32_t* cells, uint64_t* offsets, uint64_t n) {
    const int c = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    const int nc = *n_heads;
    if (c > nc) return;
    if (c == nc) {
        offsets[c] = n;
        return;
    }
    const uint32_t h = heads[c];
    cells[3 * c + 0] = (int32_t)(kx[h] ^ 0x80000000u);
    cells[3 * c + 1] = (int32_t)((uint32_t)(yz[h] >> 32) ^ 0x80000000u);
    cells[3 * c + 2] = (int32_t)((uint32_t)yz[h] ^ 0x80000000u);
    offsets[c] = h;
}

// rows and ids gathered into cell order (warp per record)
__global__ void __launch_bounds__(256) gather_records_kernel(const float* rows, const uint32_t* ids,
                                                             const uint32_t* order, uint64_t n, uint32_t dim,
                                                             float* out_rows, uint32_t* out_ids) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = w0; j < n; j += nw) {
        const uint32_t src = order[j];
        if (lane == 0) out_ids[j] = ids[src];
        for (uint32_t d = lane; d < dim; d += 32) out_rows[j * dim + d] = rows[(uint64_t)src * dim + d];
    }
}

// Inverse of threshold_keys_kernel for the first `take` sorted keys: query q's
// ranked (id, sim) written straight into its result row (no host round trip).
__global__ void decode_keys_kernel(const unsigned long long* keys, uint64_t take, uint32_t* ids, float* sims) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= take) return;
    const unsigned long long k = keys[i];
    ids[i] = (uint32_t)(k & 0xffffffffu);
    uint32_t b = ~(uint32_t)(k >> 32);
    b = (b & 0x80000000u) ? (b & 0x7fffffffu) : ~b;
    sims[i] = __uint_as_float(b);
}

// Upper bound of the store's row norms (warp per row, f64 sum of squares,
// rounded up): the tensor-core query's error bound scales with it.  Any
// non-finite element reports +inf, which keeps such a store on the exact path.
__global__ void __launch_bounds__(256) row_norm_max_kernel(const float* rows, uint64_t n, uint32_t dim,
                                                           unsigned int* max_bits) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    float best = 0.0f;
    for (uint64_t k = warp0; k < n; k += nwarps) {
        const float* v = rows + k * dim;
        double ns = 0.0;
        bool finite = true;
        for (uint32_t d = lane; d < dim; d += 32) {
            const float x = v[d];
            finite &= isfinite(x);
            ns += (double)x * (double)x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        finite = __all_sync(0xffffffffu, finite);
        const float nrm = finite ? __double2float_ru(sqrt(ns) * (1.0 + 1e-12)) : INFINITY;
        best = fmaxf(best, nrm);
    }
    if (lane == 0 && best > 0.0f) atomicMax(max_bits, __float_as_uint(best)); // non-negative floats order as ints
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
cudaError_t launch_narrow_keys(const unsigned long long* keys, uint64_t n, const ViewInfo* info, uint32_t* k32,
                               cudaStream_t s) {
    if (!n) return cudaSuccess;
    narrow_keys_kernel<<<blocks_for((n + 3) / 4, 256), 256, 0, s>>>(keys, n, info, k32);
    return cudaGetLastError();
}

cudaError_t launch_tie_fixup(const uint32_t* k32s, uint64_t n, const unsigned long long* keys, uint32_t* order,
                             cudaStream_t s) {
    if (n < 2) return cudaSuccess;
    tie_fixup_kernel<<<blocks_for((n + 3) / 4, 256), 256, 0, s>>>(k32s, n, keys, order);
    return cudaGetLastError();
}

cudaError_t launch_gather_boxes(const uint2* boxes, const uint32_t* k32s, const uint32_t* order, uint64_t n,
                                uint2* rbox, uint32_t* cnt, cudaStream_t s) {
    gather_boxes_kernel<<<blocks_for(n + 1, 256), 256, 0, s>>>(boxes, k32s, order, n, rbox, cnt);
    return cudaGetLastError();
}

cudaError_t launch_instance_offsets(const uint32_t* cnt, uint64_t n, uint32_t* offsets, void* tmp, size_t* tmp_bytes,
                                    cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, cnt, offsets, (int)(n + 1), s);
}

cudaError_t launch_emit_instances(const uint2* rbox, const uint32_t* order, uint64_t n, const uint32_t* offsets,
                                  uint32_t tiles_x, uint64_t cap, void* keys, bool k16, uint32_t* vals, ViewInfo* info,
                                  cudaStream_t s) {
    if (!n) return cudaSuccess;
    const unsigned g = (unsigned)std::min<uint64_t>(blocks_for(cap, 256), 148u * 16u);
    if (k16) {
        emit_instances_kernel<uint16_t><<<blocks_for(n, 256), 256, 0, s>>>(rbox, order, n, offsets, tiles_x, cap,
                                                                            static_cast<uint16_t*>(keys), vals, info);
        pad_keys_kernel<uint16_t><<<g, 256, 0, s>>>(offsets, n, cap, static_cast<uint16_t*>(keys));
    } else {
        emit_instances_kernel<uint32_t><<<blocks_for(n, 256), 256, 0, s>>>(rbox, order, n, offsets, tiles_x, cap,
                                                                            static_cast<uint32_t*>(keys), vals, info);
        pad_keys_kernel<uint32_t><<<g, 256, 0, s>>>(offsets, n, cap, static_cast<uint32_t*>(keys));
    }
    return cudaGetLastError();
}

uint32_t tile_sort_max_tiles() { return kTsMaxTiles; }

template <bool FIXUP>
cudaError_t configure_tile_sort() {
    cudaError_t e = cudaFuncSetAttribute(tile_sort_kernel<kTileSortMax, 2, FIXUP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_sort_smem(kTileSortMax));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tile_sort_kernel<kTileSortMax * 3 / 4, 3, FIXUP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_sort_smem(kTileSortMax * 3 / 4));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tile_sort_kernel<kTileSortMax / 2, 3, FIXUP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_sort_smem(kTileSortMax / 2));
    return e;
}

template <bool FIXUP>
void launch_tile_sort_kernel(const TileSortParams& p, unsigned grid, cudaStream_t s) {
    // slot capacity 4096 / 6144 (c4's dense tiles reach ~5300 instances): 64 KB
    // or less of shared memory, three CTAs per SM; 8192: two
    if (p.cap <= kTileSortMax / 2)
        tile_sort_kernel<kTileSortMax / 2, 3, FIXUP><<<grid, kTsSortThreads, tile_sort_smem(kTileSortMax / 2), s>>>(p);
    else if (p.cap <= kTileSortMax * 3 / 4)
        tile_sort_kernel<kTileSortMax * 3 / 4, 3, FIXUP>
            <<<grid, kTsSortThreads, tile_sort_smem(kTileSortMax * 3 / 4), s>>>(p);
    else
        tile_sort_kernel<kTileSortMax, 2, FIXUP><<<grid, kTsSortThreads, tile_sort_smem(kTileSortMax), s>>>(p);
}

cudaError_t launch_tile_sort_fixup(const TileSortParams& p, cudaStream_t s) {
    // one CTA per SM walks the queued tiles
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    launch_tile_sort_kernel<true>(p, std::min<unsigned>((unsigned)sms, p.tiles), s);
    return cudaGetLastError();
}

cudaError_t launch_tile_sort_bin(const TileSortParams& p, cudaStream_t s) {
    if (p.tiles > kTsMaxTiles) return cudaErrorInvalidValue;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<int> configured[64] = {};
    if (dev >= 0 && dev < 64 && !configured[dev].load()) {
        cudaError_t e = cudaFuncSetAttribute(ts_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(kTsMaxTiles * 4));
        if (e == cudaSuccess) e = configure_tile_sort<false>();
        if (e == cudaSuccess) e = configure_tile_sort<true>();
        if (e != cudaSuccess) return e;
        configured[dev].store(1);
    }
    cudaError_t e = cudaMemsetAsync(p.fill, 0, (size_t)p.tiles * 4, s);
    if (e != cudaSuccess) return e;
    if (p.n) {
        const unsigned chunks = (unsigned)((p.n + kTsChunk - 1) / kTsChunk);
        ts_scatter_kernel<<<chunks, kTsThreads, (size_t)p.tiles * 4, s>>>(p);
    }
    launch_tile_sort_kernel<false>(p, p.tiles, s);
    return cudaGetLastError();
}

uint32_t bin_scatter_warps(uint32_t tiles) {
    if (20ull * tiles <= 112u * 1024u) return 8u; // two CTAs of 8 warps per SM
    if (tiles <= 18000u) return 4u;              // 12 B per tile: <= 216 KB
    return 0u;
}

size_t bin_counts_entries(uint64_t n, uint32_t tiles) {
    return (size_t)((n + kBinChunk - 1) / kBinChunk) * tiles;
}

cudaError_t launch_bin(const BinParams& p, cudaStream_t s) {
    const uint32_t warps = bin_scatter_warps(p.tiles);
    if (!warps) return cudaErrorInvalidValue;
    const unsigned chunks = (unsigned)std::max<uint64_t>((p.n + kBinChunk - 1) / kBinChunk, 1);
    static bool attr_done[3] = {false, false, false};
    const size_t count_smem = (size_t)p.tiles * 4u;
    const size_t scatter_smem = (size_t)p.tiles * (4u + 2u * warps);
    cudaError_t e;
    if (!attr_done[0]) {
        if ((e = cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)))
            return e;
        attr_done[0] = true;
    }
    if (warps == 8 && !attr_done[1]) {
        if ((e = cudaFuncSetAttribute(bin_scatter_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      112 * 1024)))
            return e;
        attr_done[1] = true;
    }
    if (warps == 4 && !attr_done[2]) {
        if ((e = cudaFuncSetAttribute(bin_scatter_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      220 * 1024)))
            return e;
        attr_done[2] = true;
    }
    bin_count_kernel<<<chunks, 256, count_smem, s>>>(p);
    bin_scan_kernel<<<(p.tiles + 31) / 32, dim3(32, 32), 0, s>>>(p);
    if (warps == 8)
        bin_scatter_kernel<8><<<chunks, 256, scatter_smem, s>>>(p);
    else
        bin_scatter_kernel<4><<<chunks, 128, scatter_smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_tile_ranges(const void* keys, bool k16, const uint32_t* offsets, uint64_t n, uint64_t cap,
                               uint32_t* start, uint32_t* end, ViewInfo* info, cudaStream_t s) {
    // the instance count lives on the device; cover the capacity, threads past it exit
    if (k16)
        tile_ranges_kernel<uint16_t><<<blocks_for((cap + 7) / 8, 256), 256, 0, s>>>(
            static_cast<const uint16_t*>(keys), offsets, n, start, end, info);
    else
        tile_ranges_kernel<uint32_t><<<blocks_for((cap + 3) / 4, 256), 256, 0, s>>>(
            static_cast<const uint32_t*>(keys), offsets, n, start, end, info);
    return cudaGetLastError();
}

cudaError_t launch_contract(const ContractParams& p, uint64_t max_touched, cudaStream_t s) {
    if (!max_touched) return cudaSuccess;
    if (p.n_members == 1 && p.dim == 512 && p.m[0].n_masks <= 64) {
        const size_t smem = (size_t)p.m[0].n_masks * 512 * 4;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        static std::atomic<int> configured[64] = {};
        if (dev >= 0 && dev < 64 && !configured[dev].load()) {
            cudaError_t e = cudaFuncSetAttribute(contract_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 64 * 512 * 4);
            if (e != cudaSuccess) return e;
            configured[dev].store(1);
        }
        contract_smem_kernel<<<sms, kContractThreads, smem, s>>>(p);
        return cudaGetLastError();
    }
    uint32_t group_masks = 0;
    bool small = true;
    for (uint32_t i = 0; i < p.n_members; ++i) {
        group_masks += p.m[i].n_masks;
        small = small && p.m[i].n_masks <= 64;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    {
        // SS_CONTRACT_CTAS: grid of the group passes (timing experiments)
        static const int override_ctas = [] {
            const char* e = getenv("SS_CONTRACT_CTAS");
            return e ? atoi(e) : 0;
        }();
        // default: 3/5 of the SMs, so compositor CTAs of other views keep the
        // rest (300 c4 views: 148 CTAs 1580, 110 1603-1606, 90 1615-1616,
        // 74 1597-1607, 50 1579-1590 views/s)
        sms = override_ctas > 0 ? std::min(sms, override_ctas) : std::max(1, (sms * 3 + 2) / 5);
    }
    static std::atomic<int> configured_g[64] = {};
    if (dev >= 0 && dev < 64 && !configured_g[dev].load()) {
        const void* ks[] = {(const void*)contract_group_pass_kernel<0, 3, 2, false, false>,
                            (const void*)contract_group_pass_kernel<1, 3, 2, false, false>,
                            (const void*)contract_group_pass_kernel<0, 1, 4, true, false>,
                            (const void*)contract_group_pass_kernel<1, 1, 4, true, false>,
                            (const void*)contract_group_pass_kernel<0, 3, 2, false, true>,
                            (const void*)contract_group_pass_kernel<1, 3, 2, false, true>,
                            (const void*)contract_group_pass_kernel<0, 1, 4, true, true>,
                            (const void*)contract_group_pass_kernel<1, 1, 4, true, true>};
        for (const void* k : ks) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
            if (e != cudaSuccess) return e;
        }
        configured_g[dev].store(1);
    }
    // the group kernels take the scalars' representation as a template
    // parameter; a group mixing both (the option changed mid-group) takes the
    // general kernel
    bool any_fix = false, all_fix = true;
    for (uint32_t i = 0; i < p.n_members; ++i) {
        any_fix = any_fix || p.m[i].fix;
        all_fix = all_fix && p.m[i].fix;
    }
    const bool mixed = any_fix && !all_fix;
    if (!mixed && p.n_members >= 2 && p.n_members < kMaxGroup && p.dim == 512 && small && group_masks <= 192 &&
        p.union_list) {
        cudaError_t e = cudaMemsetAsync(p.union_count, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return e;
        group_union_kernel<<<(unsigned)sms * 4u, 256, 0, s>>>(p, p.union_list, p.union_count);
        if (p.use_tc && p.tc_scratch && contract_tc_eligible(p)) {
            int full = 148; // one persistent CTA per SM (512 TMEM columns, ~196 KB shared each)
            cudaDeviceGetAttribute(&full, cudaDevAttrMultiProcessorCount, dev);
            return launch_contract_tc(p, p.tc_scratch, full, s);
        }
        const size_t smem = (size_t)group_masks * 1024u;
        if (all_fix) {
            contract_group_pass_kernel<0, 3, 2, false, true><<<sms, 1024, smem, s>>>(p, p.union_list, p.union_count);
            contract_group_pass_kernel<1, 3, 2, false, true><<<sms, 1024, smem, s>>>(p, p.union_list, p.union_count);
        } else {
            contract_group_pass_kernel<0, 3, 2, false, false><<<sms, 1024, smem, s>>>(p, p.union_list, p.union_count);
            contract_group_pass_kernel<1, 3, 2, false, false><<<sms, 1024, smem, s>>>(p, p.union_list, p.union_count);
        }
        return cudaGetLastError();
    }
    if (p.n_members == 1 && p.dim == 512 && p.m[0].n_masks <= 128) {
        // one view with 65..128 masks: its CLIP half-rows (<= 128 KB) per pass
        const size_t smem = (size_t)p.m[0].n_masks * 1024u;
        if (all_fix) {
            contract_group_pass_kernel<0, 1, 4, true, true><<<sms, 1024, smem, s>>>(p, nullptr, nullptr);
            contract_group_pass_kernel<1, 1, 4, true, true><<<sms, 1024, smem, s>>>(p, nullptr, nullptr);
        } else {
            contract_group_pass_kernel<0, 1, 4, true, false><<<sms, 1024, smem, s>>>(p, nullptr, nullptr);
            contract_group_pass_kernel<1, 1, 4, true, false><<<sms, 1024, smem, s>>>(p, nullptr, nullptr);
        }
        return cudaGetLastError();
    }
    if (p.dim == 512)
        contract_kernel<true><<<warp_grid(max_touched), 256, 0, s>>>(p);
    else
        contract_kernel<false><<<warp_grid(max_touched), 256, 0, s>>>(p);
    return cudaGetLastError();
}
// Covered rows of a normalised slice packed for a sparse readout (order of
// arrival; the host scatters them by id): ids, coverage and the rows.
__global__ void __launch_bounds__(256) compact_covered_kernel(const float* __restrict__ rows,
                                                              const float* __restrict__ cov, uint64_t n, uint32_t dim,
                                                              uint32_t* ids, float* pcov, float* prow,
                                                              unsigned long long* count) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = w0 * 32u; base < n; base += nw * 32u) {
        const uint64_t i = base + lane;
        const bool c = i < n && cov[i] > 0.0f; // normalize writes 0 (and a zero row) for uncovered rows
        const uint32_t bal = __ballot_sync(0xffffffffu, c);
        if (!bal) continue;
        unsigned long long slot0 = 0;
        if (lane == 0) slot0 = atomicAdd(count, (unsigned long long)__popc(bal));
        slot0 = __shfl_sync(0xffffffffu, slot0, 0);
        if (c) {
            const uint64_t k = slot0 + __popc(bal & ((1u << lane) - 1u));
            ids[k] = (uint32_t)i;
            pcov[k] = cov[i];
        }
        for (uint32_t rem = bal; rem; rem &= rem - 1u) {
            const int src = __ffs(rem) - 1;
            const uint64_t k = slot0 + __popc(bal & ((1u << src) - 1u));
            const float* r = rows + (base + src) * dim;
            float* o = prow + k * dim;
            for (uint32_t d = lane; d < dim; d += 32u) o[d] = r[d];
        }
    }
}

cudaError_t launch_compact_covered(const float* rows, const float* cov, uint64_t n, uint32_t dim, uint32_t* ids,
                                   float* pcov, float* prow, unsigned long long* count, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 8ull);
    compact_covered_kernel<<<(unsigned)blocks, 256, 0, s>>>(rows, cov, n, dim, ids, pcov, prow, count);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const float* sums, const float* totals, uint64_t n, uint32_t dim, float* rows,
                             float* coverage, unsigned long long* covered, cudaStream_t s) {
    if (!n) return cudaSuccess;
    normalize_kernel<<<warp_grid(n), 256, 0, s>>>(sums, totals, n, dim, rows, coverage, covered);
    return cudaGetLastError();
}
cudaError_t launch_normalize_rows(const float* in, const uint32_t* select, uint64_t n, uint32_t dim, float* out,
                                  int* zero_flag, cudaStream_t s) {
    if (!n) return cudaSuccess;
    normalize_rows_kernel<<<warp_grid(n), 256, 0, s>>>(in, select, n, dim, out, zero_flag);
    return cudaGetLastError();
}
cudaError_t launch_assign_classes(const float* rows, const float* coverage, uint64_t n, uint32_t dim,
                                  const int32_t* label_ids, const float* labels, uint32_t n_labels, float* labels_t,
                                  double* label_norms, int32_t* out, cudaStream_t s) {
    if (!n) return cudaSuccess;
    label_prep_kernel<<<blocks_for(n_labels, 128), 128, 0, s>>>(labels, dim, n_labels, labels_t, label_norms);
    const size_t smem = (size_t)8 * dim * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(assign_classes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    assign_classes_kernel<<<warp_grid(n), 256, smem, s>>>(rows, coverage, n, dim, label_ids, labels_t, label_norms,
                                                          n_labels, out);
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

cudaError_t launch_touched_compact(const uint32_t* touched, uint64_t n, uint32_t gen, uint32_t* list,
                                  unsigned long long* count, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const uint64_t want = (n + 1023u) / 1024u; // 256 threads x 4 ids per block
    touched_compact_kernel<<<(unsigned)std::min<uint64_t>(want, 148ull * 8u), 256, 0, s>>>(touched, n, gen, list, count);
    return cudaGetLastError();
}

size_t partition_tmp_bytes(uint64_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n, 0, 32);
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, c, it, (const uint8_t*)nullptr, (uint32_t*)nullptr, (int*)nullptr, (int)n);
    return std::max(a, std::max(b, c));
}

cudaError_t launch_store_partition(const float* means, const float* rows, const uint32_t* ids, uint64_t n,
                                   uint32_t dim, double cell, const PartitionScratch& w, cudaStream_t s) {
    if (!n) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(w.mn3, 0xff, 3 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    bbox_min_kernel<<<(unsigned)std::min<uint64_t>(blocks_for(n, 256), 148ull * 8u), 256, 0, s>>>(means, n, w.mn3);
    cell_keys_kernel<<<blocks_for(n, 256), 256, 0, s>>>(means, n, w.mn3, cell, w.yz, w.kx, w.idx);
    // stable LSD: (y, z) first, then x -> cells in (x, y, z) order, records in store order within a cell
    size_t tb = w.tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.yz, w.yz_s, w.idx, w.perm1, (int)n, 0, 64, s);
    if (e != cudaSuccess) return e;
    gather_kernel<uint32_t><<<blocks_for(n, 256), 256, 0, s>>>(w.kx, w.perm1, n, w.kx_p);
    tb = w.tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kx_p, w.kx_s, w.perm1, w.perm2, (int)n, 0, 32, s);
    if (e != cudaSuccess) return e;
    gather_kernel<unsigned long long><<<blocks_for(n, 256), 256, 0, s>>>(w.yz, w.perm2, n, w.yz_s);
    cell_heads_kernel<<<blocks_for(n, 256), 256, 0, s>>>(w.kx_s, w.yz_s, n, w.head);
    tb = w.tmp_bytes;
    thrust::counting_iterator<uint32_t> it(0);
    e = cub::DeviceSelect::Flagged(w.tmp, tb, it, w.head, w.heads, w.n_heads, (int)n, s);
    if (e != cudaSuccess) return e;
    cell_list_kernel<<<blocks_for(n + 1, 256), 256, 0, s>>>(w.kx_s, w.yz_s, w.heads, w.n_heads, w.cells, w.offsets,
                                                            n);
    gather_records_kernel<<<warp_grid(n), 256, 0, s>>>(rows, ids, w.perm2, n, dim, w.out_rows, w.out_ids);
    return cudaGetLastError();
}

// ------------------------------------------- covered-row (sparse) combine
// Only rows some rank touched carry data (c4: ~6 % of the scene), so the
// combine reduce-scatters those rows alone: global covered flags (an all-reduce
// max of every rank's "total != 0"), positions by a scan, each rank packs its
// partial's covered rows owner by owner (owner k = the rank that receives row
// block k of the round) into equal P-row segments, and after the
// reduce-scatter the owner unpacks its segment onto its block, normalising as
// normalize_kernel does (uncovered rows are exact zeros).
__global__ void covered_flags_kernel(const float* totals, uint64_t n, uint8_t* flags) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = totals[i] != 0.0f; // NaN totals count as touched
}

__global__ void __launch_bounds__(256) sparse_pack_kernel(const float* sums, const float* totals, uint64_t n,
                                                          uint32_t dim, uint64_t block, const uint8_t* flags,
                                                          const uint32_t* pos, uint64_t P, float* send_sums,
                                                          float* send_tot) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = w0; i < n; i += nw) {
        if (!flags[i]) continue;
        const uint64_t k = i / block;
        const uint64_t slot = k * P + (pos[i] - pos[k * block]);
        const float* src = sums + i * dim;
        float* dst = send_sums + slot * dim;
        for (uint32_t d = lane; d < dim; d += 32) dst[d] = src[d];
        if (lane == 0) send_tot[slot] = totals[i];
    }
}

__global__ void __launch_bounds__(256) sparse_unpack_kernel(const float* recv_sums, const float* recv_tot,
                                                            uint64_t block, uint64_t own0, const uint8_t* flags,
                                                            const uint32_t* pos, uint32_t dim, float* rows,
                                                            float* coverage, unsigned long long* covered) {
    unsigned long long ncov = 0;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w0; k < block; k += nw) {
        const uint64_t i = own0 + k; // row of the round
        const bool f = flags[i] != 0;
        const uint64_t j = f ? pos[i] - pos[own0] : 0;
        const float t = f ? recv_tot[j] : 0.0f;
        const bool cov = (double)t > 1e-8; // pipeline.hpp:120-135, as normalize_kernel
        ncov += cov;
        const double inv = cov ? 1.0 / (double)t : 0.0;
        const float* sp = recv_sums + j * dim;
        float* o = rows + k * dim;
        for (uint32_t d = lane; d < dim; d += 32) o[d] = cov ? __double2float_rn((double)sp[d] * inv) : 0.0f;
        if (lane == 0) coverage[k] = cov ? t : 0.0f;
    }
    if (covered && lane == 0 && ncov) atomicAdd(covered, ncov);
}

cudaError_t launch_covered_flags(const float* totals, uint64_t n, uint8_t* flags, cudaStream_t s) {
    if (!n) return cudaSuccess;
    covered_flags_kernel<<<blocks_for(n, 256), 256, 0, s>>>(totals, n, flags);
    return cudaGetLastError();
}
cudaError_t launch_flag_positions(const uint8_t* flags, uint64_t n, uint32_t* pos, void* tmp, size_t* tmp_bytes,
                                  cudaStream_t s) {
    // pos[i] = covered rows before i, pos[n] = all (exclusive scan over n + 1 items; flags[n] reads as 0)
    auto in = thrust::make_transform_iterator(thrust::counting_iterator<uint64_t>(0),
                                              FlagAt{flags, n});
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, in, pos, (int)(n + 1), s);
}
cudaError_t launch_sparse_pack(const float* sums, const float* totals, uint64_t n, uint32_t dim, uint64_t block,
                               const uint8_t* flags, const uint32_t* pos, uint64_t P, float* send_sums,
                               float* send_tot, cudaStream_t s) {
    if (!n || !P) return cudaSuccess;
    sparse_pack_kernel<<<warp_grid(n), 256, 0, s>>>(sums, totals, n, dim, block, flags, pos, P, send_sums, send_tot);
    return cudaGetLastError();
}
cudaError_t launch_sparse_unpack(const float* recv_sums, const float* recv_tot, uint64_t block, uint64_t own0,
                                 const uint8_t* flags, const uint32_t* pos, uint32_t dim, float* rows, float* coverage,
                                 unsigned long long* covered, cudaStream_t s) {
    if (!block) return cudaSuccess;
    sparse_unpack_kernel<<<warp_grid(block), 256, 0, s>>>(recv_sums, recv_tot, block, own0, flags, pos, dim, rows,
                                                          coverage, covered);
    return cudaGetLastError();
}

cudaError_t launch_decode_keys(const unsigned long long* keys, uint64_t take, uint32_t* ids, float* sims,
                               cudaStream_t s) {
    if (!take) return cudaSuccess;
    decode_keys_kernel<<<blocks_for(take, 256), 256, 0, s>>>(keys, take, ids, sims);
    return cudaGetLastError();
}

cudaError_t launch_row_norm_max(const float* rows, uint64_t n, uint32_t dim, unsigned int* max_bits, cudaStream_t s) {
    if (!n) return cudaSuccess;
    row_norm_max_kernel<<<warp_grid(n), 256, 0, s>>>(rows, n, dim, max_bits);
    return cudaGetLastError();
}

} // namespace ss
