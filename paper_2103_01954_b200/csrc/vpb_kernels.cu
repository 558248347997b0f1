// vpb_kernels.cu — sm_100a kernels of the B200 raymarcher (the replacement of
// volprim::render's body, march.cpp:95-132).
//
//   K0 k_repack        planar slab (k,c,z,y,x) -> channel-interleaved float4 (k,z,y,x)
//   K1 k_cull          one thread per primitive: screen-tile rectangle + depth key, per-tile
//                      counts (replaces primitiveAabb/mortonCode/buildLbvh, lbvh.cpp:13-156)
//   K2 k_scan          exclusive scan of tile counts -> per-tile ranges, key capacity check
//   K3 k_emit          (tile, depth<<32|prim) keys scattered into their tile buckets
//   K3 k_tile_sort     per-bucket ascending sort of (depth<<32|prim): MSD radix by tile
//                      (K1-K3 counting pass) + in-bucket bitonic network
//   K5 k_march_tiles   16x16-pixel tile per CTA: candidate transforms staged in shared memory,
//                      exact per-ray segment window (intersect, lbvh.cpp:207-234) and the
//                      fused quadrature (march, march.cpp:18-93)
//   K5b k_march_fallback  wide-window re-march of the rare rays whose live segments overflow
//                      the shared-memory window
//   k_march_rays       march() over caller-provided rays, all primitives as candidates
//   k_composite        composite(), march.cpp:134-147
//
// Compiled with -fmad=false: see vpb_device.cuh for the arithmetic contract.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "vpb_device.cuh"
#include "vpb_kernels.h"
#include "vpb_march.cuh"

namespace vpb {


// ----------------------------------------------------------------------------------------
// K0: planar -> interleaved. One thread per voxel; the four planar reads are coalesced
// across the warp (consecutive voxels), the float4 write is coalesced.
__global__ void k_repack(const float *__restrict__ planar, float4 *__restrict__ inter,
                         int64_t n_prim, int64_t m3) {
    const int64_t total = n_prim * m3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / m3, v = i - k * m3;
        const float *src = planar + k * 4 * m3 + v;
        inter[i] = make_float4(__ldg(src), __ldg(src + m3), __ldg(src + 2 * m3), __ldg(src + 3 * m3));
    }
}

// Pads 15-float AffineXf records to 16 floats (aligned float4 staging).
__global__ void k_pad_xf(const float *__restrict__ xf15, float *__restrict__ xf16, int n_prim) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_prim * kXfStride) return;
    const int k = i / kXfStride, j = i - k * kXfStride;
    xf16[i] = j < 15 ? xf15[k * 15 + j] : 0.0f;
}

// ----------------------------------------------------------------------------------------
// K1: cull. Same float operation sequence as the CPU restatement (oracle/vp_oracle.c,
// cull_one), so rectangles and keys are bit-identical. `prect` is the conservative pixel
// rectangle the tile rectangle is derived from (empty = {0, 0, -1, -1}); the raymarch uses it
// to skip the exact box test for candidates whose rectangle excludes the pixel.
__device__ __forceinline__ void cull_rect(const float *xf, const CamDev &cam, int4 &rect,
                                          int4 &prect, uint32_t &key) {
    const V3 s = mk3(xf[12], xf[13], xf[14]);
    const float r = sqrtf(dot3(s, s));
    const float rr = r * 1.001f + 1e-6f;
    const V3 cc = matvec(cam.R, mk3(xf[0], xf[1], xf[2])) + mk3(cam.t[0], cam.t[1], cam.t[2]);
    const float dist = sqrtf(dot3(cc, cc));
    float depth = dist - rr;
    if (!(depth > 0.0f)) depth = 0.0f;
    key = __float_as_uint(depth);
    rect = make_int4(0, 0, -1, -1);
    prect = rect;
    if (cam.width <= 0 || cam.height <= 0) return;
    if (cc.z + rr < 0.0f) return;
    if (cc.z - rr <= 1e-3f * rr) {
        rect = make_int4(0, 0, cam.tiles_x - 1, cam.tiles_y - 1);
        prect = make_int4(0, 0, cam.width - 1, cam.height - 1);
        return;
    }
    float umin = 3.402823466e+38f, umax = -3.402823466e+38f;
    float vmin = 3.402823466e+38f, vmax = -3.402823466e+38f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const V3 corner = mk3(c & 1 ? 1.0f : -1.0f, c & 2 ? 1.0f : -1.0f, c & 4 ? 1.0f : -1.0f);
        const V3 pw = mk3(xf[0], xf[1], xf[2]) +
                      matvec(xf + 3, mk3(s.x * corner.x, s.y * corner.y, s.z * corner.z));
        const V3 pc = matvec(cam.R, pw) + mk3(cam.t[0], cam.t[1], cam.t[2]);
        const V3 hp = matvec(cam.K, pc);
        const float u = hp.x / hp.z, v = hp.y / hp.z;
        umin = u < umin ? u : umin;
        umax = u > umax ? u : umax;
        vmin = v < vmin ? v : vmin;
        vmax = v > vmax ? v : vmax;
    }
    const float mu = 2.0f + 1e-3f * (fabsf(umin) + fabsf(umax));
    const float mv = 2.0f + 1e-3f * (fabsf(vmin) + fabsf(vmax));
    float x0 = floorf(umin - mu), x1 = floorf(umax + mu);
    float y0 = floorf(vmin - mv), y1 = floorf(vmax + mv);
    const float wl = (float)(cam.width - 1), hl = (float)(cam.height - 1);
    if (!(x1 >= 0.0f) || !(x0 <= wl) || !(y1 >= 0.0f) || !(y0 <= hl)) return;
    x0 = x0 > 0.0f ? x0 : 0.0f;
    y0 = y0 > 0.0f ? y0 : 0.0f;
    x1 = x1 < wl ? x1 : wl;
    y1 = y1 < hl ? y1 : hl;
    prect = make_int4((int)x0, (int)y0, (int)x1, (int)y1);
    rect = make_int4(prect.x / kTile, prect.y / kTile, prect.z / kTile, prect.w / kTile);
}

__device__ __forceinline__ void cull_body(const float *__restrict__ xf16, int n_prim, const CamDev &cam,
                       int4 *__restrict__ rects, int4 *__restrict__ prects,
                       uint32_t *__restrict__ keys, uint32_t *__restrict__ tile_counts) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_prim) return;
    float xf[15];
#pragma unroll
    for (int j = 0; j < 15; ++j) xf[j] = xf16[(size_t)k * kXfStride + j];
    int4 rc, prc;
    uint32_t key;
    cull_rect(xf, cam, rc, prc, key);
    rects[k] = rc;
    prects[k] = prc;
    keys[k] = key;
    for (int ty = rc.y; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.z; ++tx)
            if (tile_owned(cam, ty * cam.tiles_x + tx)) atomicAdd(&tile_counts[ty * cam.tiles_x + tx], 1u);
}

// K2: single-CTA exclusive scan over the tile counts (tiles <= a few 10^4). Writes the
// bucket starts twice (offsets, and the emit cursors) and flags key-capacity overflow.
// It also writes `order`: the tiles by descending candidate count (a proxy for their march
// cost), so the raymarch hands the heaviest tiles out first and the tail stays short. In a
// shard render the tiles the shard does not own go last (bucket 0), after its empty tiles.
constexpr int kOrderBuckets = 1024;
__device__ __forceinline__ void scan_body(const uint32_t *__restrict__ counts, int n_tiles,
                       uint32_t *__restrict__ offsets, uint32_t *__restrict__ cursor,
                       uint32_t *__restrict__ order, DevCounters *ctr, int64_t capacity, int n_shards,
                       int shard, unsigned long long *keys_host = nullptr) {
    const auto bucket = [&](int t) {
        return n_shards > 1 && t % n_shards != shard ? 0u : min(counts[t], (uint32_t)kOrderBuckets - 2) + 1u;
    };
    __shared__ unsigned long long warp_sums[32];
    __shared__ unsigned long long carry;
    __shared__ unsigned hist[kOrderBuckets];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n_tiles; base += blockDim.x) {
        const int i = base + tid;
        const unsigned long long v = i < n_tiles ? counts[i] : 0;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        if (lane == 31) warp_sums[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
            unsigned long long ws = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long n = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += n;
            }
            if (lane < nw) warp_sums[lane] = ws;
        }
        __syncthreads();
        const unsigned long long excl = carry + (wid ? warp_sums[wid - 1] : 0) + incl - v;
        if (i < n_tiles) {  // saturated: a bucket past 2^32 - 1 keys cannot wrap (tile_key_overflowed)
            const uint32_t e32 = excl < 0xffffffffull ? (uint32_t)excl : 0xffffffffu;
            offsets[i] = e32;
            cursor[i] = e32;
        }
        __syncthreads();
        if (tid == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (tid == 0) {
        offsets[n_tiles] = carry < 0xffffffffull ? (uint32_t)carry : 0xffffffffu;
        ctr->keys = carry;
        ctr->key_overflow = (int64_t)carry > capacity ? 1 : 0;
        ctr->key_cap = (uint32_t)min(capacity, (int64_t)0xfffffffe);
        if (keys_host) *(volatile unsigned long long *)keys_host = carry;
    }
    // counting sort of the tiles by bucket(t) (1 + min(count, 1022), 0 if not owned), descending
    for (int b = tid; b < kOrderBuckets; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    unsigned nonempty = 0;
    for (int t = tid; t < n_tiles; t += blockDim.x) {
        atomicAdd(&hist[bucket(t)], 1u);
        nonempty += counts[t] > 0;
    }
    for (int o = 16; o > 0; o >>= 1) nonempty += __shfl_down_sync(0xffffffffu, nonempty, o);
    if (lane == 0 && nonempty) atomicAdd(&ctr->nonempty_tiles, (unsigned long long)nonempty);
    __syncthreads();
    if (wid == 0) {  // exclusive scan over buckets in descending order, 32 buckets per lane
        unsigned local = 0;
        for (int q = 0; q < kOrderBuckets / 32; ++q) local += hist[kOrderBuckets - 1 - (lane * 32 + q)];
        unsigned incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        unsigned run = incl - local;
        for (int q = 0; q < kOrderBuckets / 32; ++q) {
            const int b = kOrderBuckets - 1 - (lane * 32 + q);
            const unsigned h = hist[b];
            hist[b] = run;
            run += h;
        }
    }
    __syncthreads();
    for (int t = tid; t < n_tiles; t += blockDim.x)
        order[atomicAdd(&hist[bucket(t)], 1u)] = (uint32_t)t;
}

// K3a: scatter keys into buckets, one warp per primitive: the lanes claim the slots of the
// primitive's tiles in parallel (a thread per primitive would chain its atomics' round trips).
// Order inside a bucket is arbitrary here; K3b makes it canonical.
__device__ __forceinline__ void emit_body(const int4 *__restrict__ rects, const uint32_t *__restrict__ keys,
                       int n_prim, int tiles_x, const uint32_t *__restrict__ offsets, uint32_t *__restrict__ cursor,
                       unsigned long long *__restrict__ entries, const DevCounters *ctr, int n_shards,
                       int shard) {
    const int k = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= n_prim) return;
    const int4 rc = rects[k];
    const int w = rc.z - rc.x + 1, h = rc.w - rc.y + 1;
    if (w <= 0 || h <= 0) return;
    const unsigned long long e = ((unsigned long long)keys[k] << 32) | (uint32_t)k;
    const bool ovf = ctr->key_overflow != 0;
    const unsigned cap = ctr->key_cap;
    for (int q = lane; q < w * h; q += 32) {
        const int t = (rc.y + q / w) * tiles_x + rc.x + q % w;
        if (ovf && tile_key_overflowed(offsets, t, cap)) continue;  // the fallback rebuilds its list
        if (n_shards <= 1 || t % n_shards == shard) entries[atomicAdd(&cursor[t], 1u)] = e;
    }
}

// K3b: sort each bucket ascending by (depth bits, prim).
// Buckets of up to 256 keys (all of them at the benchmark configs): one warp per bucket,
// R = 2 or 8 keys per lane in registers, a bitonic network over 32R elements with shuffles
// (no block barriers); the buckets past 256 keys are listed for k_tile_sort_big.
template <int R>
__device__ __forceinline__ void warp_bitonic(unsigned long long (&v)[R], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {  // partner in another register of the same lane
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int pr = r ^ (j >> 5);
                    if (pr > r) {
                        const bool asc = ((lane + 32 * r) & k) == 0;
                        const unsigned long long a = v[r], b = v[pr];
                        if (asc ? b < a : a < b) {
                            v[r] = b;
                            v[pr] = a;
                        }
                    }
                }
            } else {  // partner in lane ^ j
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int e = lane + 32 * r;
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool keep_min = ((e & j) == 0) == ((e & k) == 0);
                    v[r] = keep_min ? (o < v[r] ? o : v[r]) : (o > v[r] ? o : v[r]);
                }
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void warp_sort_bucket(unsigned long long *a, int n, int lane) {
    unsigned long long v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = lane + 32 * r < n ? a[lane + 32 * r] : ~0ull;
    warp_bitonic<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (lane + 32 * r < n) a[lane + 32 * r] = v[r];
}

__device__ __forceinline__ void tile_sort_warp_body(const uint32_t *__restrict__ offsets, unsigned long long *__restrict__ entries,
                 int n_tiles, uint32_t *__restrict__ big, DevCounters *ctr) {
    const int tile = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (tile >= n_tiles) return;
    if (ctr->key_overflow && tile_key_overflowed(offsets, tile, ctr->key_cap)) return;
    const uint32_t start = offsets[tile];
    const int n = (int)(offsets[tile + 1] - start);
    if (n <= 1) return;
    if (n <= 64) warp_sort_bucket<2>(entries + start, n, lane);
    else if (n <= 256) warp_sort_bucket<8>(entries + start, n, lane);
    else if (lane == 0) big[atomicAdd(&ctr->big_buckets, 1u)] = (uint32_t)tile;
}

// Buckets past 256 keys: all-ascending bitonic network (the "flip" formulation), so padding
// with +inf past n needs no special case; persistent CTAs over the list.
constexpr int kSortSmem = 2048;
__device__ __forceinline__ void tile_sort_big_body(const uint32_t *__restrict__ offsets,
                                unsigned long long *__restrict__ entries, const uint32_t *__restrict__ big,
                                const DevCounters *ctr) {
    __shared__ unsigned long long s[kSortSmem];
    for (unsigned q = blockIdx.x; q < ctr->big_buckets; q += gridDim.x) {
        const uint32_t tile = big[q];
        const uint32_t start = offsets[tile];
        const int n = (int)(offsets[tile + 1] - start);
        int p = 1;
        while (p < n) p <<= 1;
        unsigned long long *a = entries + start;
        const bool in_smem = p <= kSortSmem;
        if (in_smem) {
            for (int i = threadIdx.x; i < p; i += blockDim.x) s[i] = i < n ? a[i] : ~0ull;
            __syncthreads();
        }
        unsigned long long *v = in_smem ? s : a;
        for (int k = 2; k <= p; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < p; i += blockDim.x) {
                    const int partner = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
                    if (partner > i && (in_smem || partner < n)) {
                        const unsigned long long x = v[i], y = v[partner];
                        if (y < x) {
                            v[i] = y;
                            v[partner] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        if (in_smem)
            for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = s[i];
        __syncthreads();
    }
}

// Binning of a batch of views in one launch per stage: blockIdx.y is the view (BinBatch), so a
// batch of 8 views costs 6 launches instead of 48 and the views' single-CTA scans run side by
// side (one launch of each small kernel is latency, not work).
__global__ void k_bin_zero(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    const int n_tiles = v.cam.tiles_x * v.cam.tiles_y;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x)
        v.tile_counts[t] = 0u;
    if (blockIdx.x == 0) {
        unsigned *c = reinterpret_cast<unsigned *>(v.ctr);
        for (int i = threadIdx.x; i < (int)(sizeof(DevCounters) / 4); i += blockDim.x) c[i] = 0u;
    }
}
__global__ void k_cull(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    cull_body(bb.xf16, bb.n_prim, v.cam, v.rects, v.prects, v.keys, v.tile_counts);
}
__global__ void k_scan(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    scan_body(v.tile_counts, v.cam.tiles_x * v.cam.tiles_y, v.offsets, v.cursor, v.order, v.ctr, bb.capacity,
              v.cam.n_shards, v.cam.shard, v.keys_host);
}
__global__ void k_emit(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    emit_body(v.rects, v.keys, bb.n_prim, v.cam.tiles_x, v.offsets, v.cursor, v.entries, v.ctr, v.cam.n_shards,
              v.cam.shard);
}
__global__ void __launch_bounds__(256) k_tile_sort_warp(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    tile_sort_warp_body(v.offsets, v.entries, v.cam.tiles_x * v.cam.tiles_y, v.cursor, v.ctr);
}
__global__ void k_tile_sort_big(const __grid_constant__ BinBatch bb) {
    const BinView &v = bb.v[blockIdx.y];
    tile_sort_big_body(v.offsets, v.entries, v.cursor, v.ctr);
}

// ----------------------------------------------------------------------------------------
// K5: one CTA per 16x16 tile, heaviest tiles first (`order` from k_scan).
//   staging  the tile's candidates -> shared memory (tiles with n <= CC)
//   phase 1  every pixel: generateRay + exact segment window over the candidates
//   compact  rays with a non-empty window, in pixel order (misses write zeros and retire)
//   phase 2  the first n_hit threads march the hit rays, so warps are full of live rays
// Tiles with more than CC candidates take the same path with TileCands<false>
// (candidates read from global memory, 16-bit window indices); tiles beyond 65535
// candidates send every pixel to the fallback re-march.
// window index slots per thread (16-bit units): Window::C word-interleaves the indices, so
// the region is rounded up to whole words of every width
template <int CAP>
constexpr size_t kWcSlots = VPB_WC_INTERLEAVE ? (size_t)((CAP + 3) / 4 * 4) : (size_t)CAP;

struct TileSmem {
    float4 *xf4;       // CC * 4
    float4 *om;        // CC
    int4 *prect;       // CC
    int *prim;         // CC
    unsigned long long *tab;  // 32
    int *state;        // NT: cnt | more << 8
    int *list;         // NT
    int *warp;         // NT / 32
    float *we, *wx;    // CAP * NT each
    void *wc;          // CAP * NT window indices (uint8 or uint16)
    unsigned *mask;    // (CC + 31) / 32 words * NT per-ray candidate hit masks
};

template <int CAP, int MT, bool STAGED, int CC, bool PF, int NT>
__device__ __forceinline__ void march_tile(const TileSmem &sm, const CamDev &cam, const MarchDev &mp,
                                           const float *__restrict__ xf_g,
                                           const int4 *__restrict__ prects,
                                           const float4 *__restrict__ payload,
                                           const unsigned long long *__restrict__ entries,
                                           uint32_t start, int n, int tx, int ty, int half, const OutDev &od,
                                           DevCounters *ctr, int *__restrict__ ovf_list, int ovf_cap) {
    // NT = 256: the CTA is the whole 16x16 tile; NT = 128: the CTA is the tile's top (half 0)
    // or bottom (half 1) 16x8 pixels, and the two halves stage the same candidate list
    const int pix0 = half * NT;  // tile_pixel index of this CTA's first pixel
    using IdxT = typename std::conditional<STAGED, uint8_t, uint16_t>::type;
    const int tid = threadIdx.x;
    const int m = MT > 0 ? MT : mp.m;
    // per-primitive stride of `payload` in float4s: the x-pair layout for compile-time M
    const unsigned m3 = kPairGathers && MT >= 2 ? (unsigned)(2 * MT * MT * (MT - 1)) : (unsigned)(m * m * m);
    const V3 o = mk3(cam.center[0], cam.center[1], cam.center[2]);
    if (STAGED) {
        for (int i = tid; i < n * 4; i += NT) {
            const int c = i >> 2, q = i & 3;
            const int prim = (int)(uint32_t)(entries[start + c] & 0xffffffffull);
            if (q == 0) sm.prim[c] = prim;
            sm.xf4[q * CC + c] = __ldg(reinterpret_cast<const float4 *>(xf_g + (size_t)prim * kXfStride) + q);
        }
        __syncthreads();
        for (int c = tid; c < n; c += NT) {
            const Xf16 x = load_xf(sm.xf4 + c, CC);
            const V3 om = to_model(x.v, o);
            sm.om[c] = make_float4(om.x, om.y, om.z, 0.f);
            sm.prect[c] = prects[sm.prim[c]];
        }
        __syncthreads();
    }
    const TileCands<STAGED, PF> cands{entries, xf_g, prects, payload, m3, start, n, sm.prim,
                                  sm.xf4, sm.om, sm.prect, CC};
    IdxT *wc = reinterpret_cast<IdxT *>(sm.wc);

    // phase 1: segment windows
    const int2 px = tile_pixel(tx, ty, pix0 + tid);
    const bool valid = px.x < cam.width && px.y < cam.height;
    const int64_t pix = (int64_t)px.y * cam.width + px.x;
    int cnt = 0;
    bool more = false;
    if (!STAGED && n > 65535) {  // window indices would not fit: re-march every pixel wide
        if (valid) {
            const int slot = (int)atomicAdd(&ctr->overflow_rays, 1ull);
            if (slot < ovf_cap) ovf_list[slot] = (int)pix;
        }
        return;
    }
    if (valid && n > 0) {
        V3 rd, d;
        generate_ray(cam, (float)px.x + 0.5f, (float)px.y + 0.5f, rd, d);
        const Window<IdxT> w{sm.we, sm.wx, wc, NT, tid, STAGED ? sm.mask : nullptr, STAGED ? (CC + 31) / 32 : 0};
        window_scan<CAP>(w, cands, cnt, more, o, d, px, true, 0.f, 0);
    }
    sm.state[tid] = cnt | (more ? 256 : 0);
    if (valid && cnt == 0) write_pixel(od, pix, RayOut{});
    // compaction of hit rays (block-wide exclusive scan of the hit flags)
    const bool hit = cnt > 0;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    const int wid = tid >> 5, lane = tid & 31;
    if (lane == 0) sm.warp[wid] = __popc(bal);
    __syncthreads();
    int base = 0, n_hit = 0;
    for (int q = 0; q < NT / 32; ++q) {
        base += q < wid ? sm.warp[q] : 0;
        n_hit += sm.warp[q];
    }
    if (hit) sm.list[base + __popc(bal & ((1u << lane) - 1))] = tid;
    __syncthreads();

    // phase 2: march the hit rays
    RayOut ro{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
    const bool live = tid < n_hit;
    if (live) {
        const int r = sm.list[tid];
        const int2 rp = tile_pixel(tx, ty, pix0 + r);
        const int64_t p = (int64_t)rp.y * cam.width + rp.x;
        V3 rd, d;
        generate_ray(cam, (float)rp.x + 0.5f, (float)rp.y + 0.5f, rd, d);
        const float jit = mp.jitter ? hash_to_unit(hash_combine(mp.seed, (uint64_t)(uint32_t)(int)p)) : 0.5f;
        const int st = sm.state[r];
        const Window<IdxT> w{sm.we, sm.wx, wc, NT, r, STAGED ? sm.mask : nullptr, STAGED ? (CC + 31) / 32 : 0};
        ro = march_window<CAP, MT>(cands, w, st & 255, (st & 256) != 0, o, d, rp, jit, mp, sm.tab);
        if (ro.overflow) {
            const int slot = (int)atomicAdd(&ctr->overflow_rays, 1ull);
            if (slot < ovf_cap) ovf_list[slot] = (int)p;
        } else {
            write_pixel(od, p, ro);
        }
    }
    add_counters(ctr, ro, live && !ro.overflow);
}

template <int CAP, int MT, bool PROF, int CC, int MINB, bool PF, int NT>
__global__ void __launch_bounds__(NT, MINB)
k_march_tiles(MarchDev mp, const float *__restrict__ xf_g, const float4 *__restrict__ payload, ViewBatch views,
              const uint32_t *__restrict__ order) {
    extern __shared__ __align__(16) unsigned char smem[];
    TileSmem sm;
    sm.xf4 = reinterpret_cast<float4 *>(smem);
    sm.om = sm.xf4 + CC * 4;
    sm.prect = reinterpret_cast<int4 *>(sm.om + CC);
    sm.prim = reinterpret_cast<int *>(sm.prect + CC);
    sm.tab = reinterpret_cast<unsigned long long *>(sm.prim + CC);
    sm.state = reinterpret_cast<int *>(sm.tab + 32);
    sm.list = sm.state + NT;
    sm.warp = sm.list + NT;
    sm.we = reinterpret_cast<float *>(sm.warp + NT / 32);
    sm.wx = sm.we + CAP * NT;
    sm.wc = sm.wx + CAP * NT;
    sm.mask = reinterpret_cast<unsigned *>(reinterpret_cast<uint16_t *>(sm.wc) + kWcSlots<CAP> * NT);

    constexpr int kParts = kMarchThreads / NT;  // CTAs per tile
    const uint32_t oe = order[blockIdx.x / kParts];
    const int half = (int)(blockIdx.x % kParts);
    const ViewDev &vd = views.v[oe >> 20];
    const CamDev &cam = vd.cam;
    const OutDev &od = vd.od;
    DevCounters *ctr = vd.ctr;
    const int tile = (int)(oe & 0xfffffu);
    if (ctr->key_overflow && tile_key_overflowed(vd.offsets, tile, ctr->key_cap)) return;  // K5b marches it
    const uint32_t start = vd.offsets[tile];
    const int n = (int)(vd.offsets[tile + 1] - start);
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    load_exp_tab(sm.tab);
    unsigned long long t_start = 0;
    if (PROF && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    __syncthreads();
    if (n <= CC)
        march_tile<CAP, MT, true, CC, PF, NT>(sm, cam, mp, xf_g, vd.prects, payload, vd.entries, start, n, tx, ty, half, od, ctr,
                                      vd.ovf_list, vd.ovf_cap);
    else
        march_tile<CAP, MT, false, CC, false, NT>(sm, cam, mp, xf_g, vd.prects, payload, vd.entries, start, n, tx, ty, half, od, ctr,
                                       vd.ovf_list, vd.ovf_cap);
    if (PROF) {  // separate instantiation: per-CTA timeline for load-balance analysis
        __syncthreads();
        if (threadIdx.x == 0 && half == 0) {  // per tile: its first CTA
            unsigned long long t_end, smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            unsigned s32;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(s32));
            smid = s32;
            unsigned long long *q = od.prof + 4 * (size_t)(blockIdx.x / kParts);
            q[0] = (unsigned long long)tile;
            q[1] = smid;
            q[2] = t_start;
            q[3] = t_end;
        }
    }
}

// K5b: rays whose live segments overflowed the shared-memory window are re-marched with a
// kFallbackCap-entry window in global scratch (one window per thread of a fixed grid).
template <bool kRays>
__global__ void __launch_bounds__(kFallbackThreads)
k_march_fallback(CamDev cam, MarchDev mp, const float *__restrict__ xf_g,
                 const int4 *__restrict__ prects, int n_prim, const float4 *__restrict__ payload,
                 const uint32_t *__restrict__ offsets, const unsigned long long *__restrict__ entries,
                 OutDev od, RaysDev rays, DevCounters *ctr, const int *__restrict__ ovf_list,
                 int ovf_cap, float *scratch_e, float *scratch_x, int *scratch_c, int *huge_list, int huge_cap) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    if (!kRays && ctr->key_overflow) return;
    const int n_ovf = (int)min((unsigned long long)ovf_cap, ctr->overflow_rays);
    if (n_ovf == 0) return;  // the common case: no window overflowed (no table load, no barrier)
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const Window<int> w{scratch_e, scratch_x, scratch_c, nthreads, gtid};
    const unsigned m3 = (unsigned)(mp.m * mp.m * mp.m);
    for (int q = gtid; q < n_ovf; q += nthreads) {
        const int p = ovf_list[q];
        V3 o, d;
        float jit = 0.5f;
        RayOut ro;
        if (kRays) {
            o = mk3(rays.origins[3 * p], rays.origins[3 * p + 1], rays.origins[3 * p + 2]);
            d = mk3(rays.dirs[3 * p], rays.dirs[3 * p + 1], rays.dirs[3 * p + 2]);
            if (rays.jitter) jit = rays.jitter[p];
            const BvhCands cands{xf_g, payload, m3, n_prim, mp.bvh};
            ro = march_ray<kFallbackCap>(cands, w, o, d, make_int2(0, 0), jit, mp, s_tab);
        } else {
            const int px = p % cam.width, py = p / cam.width;
            const int tile = (py / kTile) * cam.tiles_x + px / kTile;
            generate_ray(cam, (float)px + 0.5f, (float)py + 0.5f, o, d);
            if (mp.jitter) jit = hash_to_unit(hash_combine(mp.seed, (uint64_t)(uint32_t)p));
            const uint32_t start = offsets[tile];
            const TileCands<false> cands{entries, xf_g, prects, payload, m3, start,
                                         (int)(offsets[tile + 1] - start), nullptr, nullptr, nullptr,
                                         nullptr};
            ro = march_ray<kFallbackCap>(cands, w, o, d, make_int2(px, py), jit, mp, s_tab);
        }
        if (ro.overflow) {  // more live segments than kFallbackCap: the last-resort pass
            const unsigned slot = atomicAdd(&ctr->huge_rays, 1u);
            if (huge_list && (int)slot < huge_cap) huge_list[slot] = p;
            else atomicAdd(&ctr->fallback_fail, 1);
            continue;
        }
        write_ray(od, p, ro);  // (od.state is null for camera renders)
        atomicAdd(&ctr->ray_samples, (unsigned long long)ro.samples);  // rare path: plain atomics
        atomicAdd(&ctr->prim_samples, (unsigned long long)ro.prim_samples);
        atomicAdd(&ctr->hit_rays, (unsigned long long)ro.hit);
        atomicAdd(&ctr->early_exits, (unsigned long long)ro.early);
        atomicAdd(&ctr->saturated, (unsigned long long)ro.saturated);
        atomicAdd(&ctr->refills, (unsigned long long)ro.refills);
        if (ro.numeric) atomicAdd(&ctr->numeric_fail, 1ull);
    }
}

// march() over caller rays, one warp per ray (small batches): the warp builds the ray's whole
// sorted segment list through the BVH (warp_segment_list) in shared memory, then walks
// it 32 lattice steps at a time (march_warp). Rays with more than kWarpList segments go to the
// wide-window fallback like window overflows.
constexpr int kWarpList = kRaySegs;  // segments per ray held by the warp
constexpr int kWarpCand = 256;  // BVH leaves a ray may cross before the warp path gives up
#ifndef VPB_RAYS_MINB
#define VPB_RAYS_MINB 7  // 72 registers, no spills (5: 58.4M, 6: 59.4M, 7: 60.0M, 8 spills: 60.0M backward rays/s)
#endif
// MINB: CTAs per SM. Large batches run at VPB_RAYS_MINB (more rays in flight); small ones (a
// single wave) at 5, where the extra registers shorten each ray's chain (evalLoss's 2,048 rays:
// 0.365 vs 0.38 ms); a runtime voxel count needs the registers too (no spills at 5).
template <int MT, int MINB>
__global__ void __launch_bounds__(128, MINB)
k_march_rays_warp(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
                  RaysDev rays, int64_t n_rays, OutDev od, DevCounters *ctr, int *__restrict__ ovf_list,
                  int ovf_cap) {
    __shared__ unsigned long long s_tab[32];
    __shared__ float s_e[4][kWarpList], s_x[4][kWarpList];
    __shared__ int s_c[4][kWarpList];
    __shared__ int s_cand[4][kWarpCand];
    __shared__ float s_ce[4][kWarpCand], s_cx[4][kWarpCand];
    __shared__ float s_sv[4][4 * kSvStride];  // march_warp: a chunk's per-step sums
    load_exp_tab(s_tab);
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    for (int64_t r = blockIdx.x * 4 + wid; r < n_rays; r += (int64_t)gridDim.x * 4) {
        const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
        const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        const int nh = warp_segment_list(cands, o, d, lane, s_cand[wid], s_ce[wid], s_cx[wid], kWarpCand, s_e[wid],
                                         s_x[wid], s_c[wid], kWarpList);
        const bool more = nh < 0;
        const int cnt = more ? 0 : nh;
        RayOut ro{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
        if (more) {
            ro.overflow = 1;
            if (lane == 0) {
                const int slot = (int)atomicAdd(&ctr->overflow_rays, 1ull);
                if (slot < ovf_cap) ovf_list[slot] = (int)r;
            }
        } else {
            ro = march_warp<BvhCands, MT>(cands, s_e[wid], s_x[wid], s_c[wid], cnt, o, d, jit, mp, s_tab, lane, s_sv[wid]);
            if (lane == 0) write_ray(od, r, ro);
            if (od.segs) {  // keep the list for the backward pass of the same rays
                float *sg = od.segs + (size_t)r * (3 * kRaySegs);
                for (int j = lane; j < cnt; j += 32) {
                    sg[j] = s_e[wid][j];
                    sg[kRaySegs + j] = s_x[wid][j];
                    sg[2 * kRaySegs + j] = __int_as_float(s_c[wid][j]);
                }
                if (lane == 0) od.state[8 * r + 7] = __int_as_float(cnt);
            }
        }
        add_counters(ctr, ro, lane == 0 && !ro.overflow);
        __syncwarp();
    }
}

// composite() is elementwise (march.cpp:134-147).
__global__ void k_composite(const float *__restrict__ rgb, const float *__restrict__ alpha,
                            const float *__restrict__ bg, float *__restrict__ out, int64_t n_px) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_px) return;
    const float a = alpha[p];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[3 * p + c] = a * rgb[3 * p + c] + (1.0f - a) * bg[3 * p + c];
}

__global__ void k_expf(const float *__restrict__ x, float *__restrict__ y, int64_t n) {
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = expf_glibc(x[i], s_tab);
}

// ----------------------------------------------------------------------------------------
// Host-side launchers (plain C++ signatures for vpb_api.cpp).
#ifndef VPB_WINDOW_CAP
#define VPB_WINDOW_CAP 14
#endif

// Three raymarch configurations, chosen per render from the previous render's mean
// candidates per non-empty tile (vpb_api.cpp). The kernel is bound by gather latency, so each
// keeps its shared memory small enough that the rest of the SM's 256 KB stays L1 cache for the
// payload (e.g. 3 x 52 KB -> 92 KB of L1 for Normal). Measured on the BASELINE configs
// (profiles/r01_tile_configs.txt):
//   Light  (<= 14 candidates/tile, K=512 M=32):   10-entry windows, 48 staged, 6 half-tile CTAs/SM
//   Normal (<= 40, the K=4096 M=16 headline):      14-entry windows, 56 staged, 6 half-tile CTAs/SM
//   Dense  (K=32768 M=8: long lists, many segments per ray, refills on the critical path of
//          the heaviest tiles):                    24-entry windows, 192 staged, 2 CTAs/SM
// VPB_WINDOW_CAP / VPB_CAND_CAP / VPB_MARCH_MINB override Normal for tuning builds.
#ifndef VPB_MARCH_MINB
#define VPB_MARCH_MINB 6
#endif
#ifndef VPB_CARVEOUT
#define VPB_CARVEOUT -1  // shared-memory carveout hint in percent; -1: just enough for MINB CTAs
#endif
#ifndef VPB_NORMAL_PF
#define VPB_NORMAL_PF false
#endif
// PF: line-vs-box prefilter before the exact candidate test (K=32768 M=8 launch 4.58 ->
// 4.27 ms; the K=4096 headline 6.16 -> 6.28 ms, so only the dense tier uses it).
#ifndef VPB_NORMAL_NT
#define VPB_NORMAL_NT 128
#endif
#ifndef VPB_LIGHT_NT
#define VPB_LIGHT_NT 128
#endif
#ifndef VPB_DENSE_NT
#define VPB_DENSE_NT 256
#endif
#ifndef VPB_DENSE_MINB
#define VPB_DENSE_MINB 2
#endif
#ifndef VPB_DENSE_CAP
#define VPB_DENSE_CAP 24
#endif
#ifndef VPB_DENSE_CC
#define VPB_DENSE_CC 192
#endif
#ifndef VPB_LIGHT_CAP
#define VPB_LIGHT_CAP 10
#endif
#ifndef VPB_LIGHT_CC
#define VPB_LIGHT_CC 48
#endif
// NT: threads per CTA (256: a CTA per 16x16 tile; 128: a CTA per 16x8 half tile). A CTA holds
// its warp slots until its longest ray ends; by the per-pixel sample counts of the headline,
// lanes are 67 % busy over a 16x16 CTA's lifetime and 72 % over a 16x8 one
// (tools/lane_efficiency.py). The normal tier therefore runs half tiles, 6 CTAs/SM: the
// headline launch went from 6.18 to 5.99 ms (profiles/r01_tile_configs.txt, sweeps 6-7);
// 16x4 quarter tiles at 10-12 CTAs/SM lose again (6.07-6.42 ms). Staging 56 candidates
// instead of 64 keeps 6 CTAs' shared memory under the 164 KB carveout, so L1 keeps 92 KB
// instead of 60: 5.92 ms (sweep 8). The light tier as half tiles with 10-entry windows and 48
// staged: K=512 M=32 12.61 -> 12.24 ms, K=64 M=16 at 256^2 2.63 -> 2.50 ms (sweep 10).
struct TileCfgLight {
    static constexpr int CAP = VPB_LIGHT_CAP, CC = VPB_LIGHT_CC, MINB = VPB_LIGHT_NT == 128 ? 6 : 3,
                         NT = VPB_LIGHT_NT;
    static constexpr bool PF = false;
};
struct TileCfgNormal {
    static constexpr int CAP = VPB_WINDOW_CAP, CC = kCandCap, MINB = VPB_MARCH_MINB, NT = VPB_NORMAL_NT;
    static constexpr bool PF = VPB_NORMAL_PF;
};
struct TileCfgDense {
    static constexpr int CAP = VPB_DENSE_CAP, CC = VPB_DENSE_CC, MINB = VPB_DENSE_MINB, NT = VPB_DENSE_NT;
    static constexpr bool PF = true;
};

template <int CAP, int CC, int NT>
static size_t tiles_smem() {
    return (size_t)CC * kXfStride * 4 + CC * 16 * 2 + CC * 4 + 32 * 8 + NT * 4 * 2 + (NT / 32) * 4 +
           (size_t)CAP * NT * 8 + kWcSlots<CAP> * NT * 2 + (size_t)((CC + 31) / 32) * NT * 4;
}
size_t march_tiles_smem() { return tiles_smem<TileCfgNormal::CAP, TileCfgNormal::CC, TileCfgNormal::NT>(); }

cudaError_t launch_repack(const float *planar, float4 *inter, int64_t n_prim, int64_t m3,
                          cudaStream_t st) {
    const int64_t total = n_prim * m3;
    if (total == 0) return cudaSuccess;
    const int blocks = (int)((total + 255) / 256 < 148 * 64 ? (total + 255) / 256 : 148 * 64);
    k_repack<<<blocks, 256, 0, st>>>(planar, inter, n_prim, m3);
    return cudaGetLastError();
}

cudaError_t launch_pad_xf(const float *xf15, float *xf16, int n_prim, cudaStream_t st) {
    if (n_prim == 0) return cudaSuccess;
    k_pad_xf<<<(n_prim * kXfStride + 255) / 256, 256, 0, st>>>(xf15, xf16, n_prim);
    return cudaGetLastError();
}

cudaError_t launch_binning_batch(const BinBatch &bb, cudaStream_t st) {
    int max_tiles = 0;
    for (int v = 0; v < bb.n; ++v) max_tiles = max(max_tiles, bb.v[v].cam.tiles_x * bb.v[v].cam.tiles_y);
    const unsigned nv = (unsigned)bb.n;
    k_bin_zero<<<dim3((unsigned)((max_tiles + 1023) / 1024), nv), 1024, 0, st>>>(bb);
    if (bb.n_prim > 0) k_cull<<<dim3((unsigned)((bb.n_prim + 127) / 128), nv), 128, 0, st>>>(bb);
    k_scan<<<dim3(1, nv), 1024, 0, st>>>(bb);
    if (bb.n_prim > 0) k_emit<<<dim3((unsigned)((bb.n_prim * 32ll + 255) / 256), nv), 256, 0, st>>>(bb);
    k_tile_sort_warp<<<dim3((unsigned)((max_tiles + 7) / 8), nv), 256, 0, st>>>(bb);
    k_tile_sort_big<<<dim3((unsigned)(148 / bb.n > 16 ? 148 / bb.n : 16), nv), 128, 0, st>>>(bb);
    return cudaGetLastError();
}

cudaError_t launch_binning(const CamDev &cam, const float *xf16, int n_prim, int4 *rects,
                           int4 *prects, uint32_t *keys, uint32_t *tile_counts, uint32_t *offsets,
                           uint32_t *cursor, uint32_t *order, unsigned long long *entries,
                           int64_t capacity, DevCounters *ctr, cudaStream_t st) {
    BinBatch bb{};
    bb.n = 1;
    bb.xf16 = xf16;
    bb.n_prim = n_prim;
    bb.capacity = capacity;
    bb.v[0] = BinView{cam, rects, prects, keys, tile_counts, offsets, cursor, order, entries, ctr};
    return launch_binning_batch(bb, st);
}

template <class Cfg, int MT, bool PROF>
static cudaError_t launch_tiles_m(const MarchDev &mp, const float *xf16, const float4 *payload_canon,
                                  const float4 *pairs, const ViewBatch &views, const uint32_t *order, int n_ctas,
                                  cudaStream_t st) {
    const float4 *payload = kPairGathers && MT >= 2 ? pairs : payload_canon;
    // function attributes are per device: set them once on each device this process uses
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = tiles_smem<Cfg::CAP, Cfg::CC, Cfg::NT>();
    // a runtime voxel count needs a few more registers: one CTA fewer per SM instead of spills
    constexpr int MINB = MT == 0 && Cfg::MINB > 2 ? Cfg::MINB - 1 : Cfg::MINB;
    auto kern = k_march_tiles<Cfg::CAP, MT, PROF, Cfg::CC, MINB, Cfg::PF, Cfg::NT>;
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // Ask for just the shared memory MINB resident CTAs need (each also reserves 1 KB):
        // the rest of the 256 KB unified array stays L1 cache for the payload gathers.
        int carve = VPB_CARVEOUT;
        if (carve < 0) carve = (int)((MINB * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve > 100 ? 100 : carve);
        if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    kern<<<n_ctas * (kMarchThreads / Cfg::NT), Cfg::NT, smem, st>>>(mp, xf16, payload, views, order);
    return cudaGetLastError();
}

template <class Cfg>
static cudaError_t launch_tiles_cfg(const MarchDev &mp, const float *xf16, const float4 *payload,
                                    const float4 *pairs, const ViewBatch &views, const uint32_t *order, int n_ctas,
                                    bool prof, cudaStream_t st) {
#define VPB_TILES(MT)                                                                                  \
    (prof ? launch_tiles_m<Cfg, MT, true>(mp, xf16, payload, pairs, views, order, n_ctas, st)      \
          : launch_tiles_m<Cfg, MT, false>(mp, xf16, payload, pairs, views, order, n_ctas, st))
    switch (mp.m) {  // compile-time voxel counts for the common grids
    case 1: return VPB_TILES(1);
    case 2: return VPB_TILES(2);
    case 4: return VPB_TILES(4);
    case 8: return VPB_TILES(8);
    case 16: return VPB_TILES(16);
    case 32: return VPB_TILES(32);
    default: return VPB_TILES(0);
    }
#undef VPB_TILES
}

cudaError_t launch_march_tiles(const MarchDev &mp, const float *xf16, const float4 *payload, const float4 *pairs,
                               const ViewBatch &views, const uint32_t *order, int n_ctas, bool prof, TileTier tier,
                               cudaStream_t st) {
    if (n_ctas == 0) return cudaSuccess;
    switch (tier) {
    case TileTier::Light:
        return launch_tiles_cfg<TileCfgLight>(mp, xf16, payload, pairs, views, order, n_ctas, prof, st);
    case TileTier::Dense:
        return launch_tiles_cfg<TileCfgDense>(mp, xf16, payload, pairs, views, order, n_ctas, prof, st);
    default:
        return launch_tiles_cfg<TileCfgNormal>(mp, xf16, payload, pairs, views, order, n_ctas, prof, st);
    }
}

bool march_uses_pairs(int m) { return kPairGathers && (m == 2 || m == 4 || m == 8 || m == 16 || m == 32); }

// The x-pair payload layout the raymarch gathers from (kPairGathers): for primitive k and row
// (z, y), entry x in [0, M-1) holds the interleaved voxels x and x+1 (32 B, aligned), so a
// trilinear stencil reads 4 aligned 32-byte rows. Derived from the canonical interleaved payload
// after every change of it.
__global__ void k_build_pairs(const float4 *__restrict__ payload, float4 *__restrict__ pairs, int64_t n_prim,
                              int m) {
    const int64_t rows = n_prim * m * m, per = m - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / per, x = i - row * per;
        const float4 *src = payload + row * m + x;
        pairs[2 * i] = src[0];
        pairs[2 * i + 1] = src[1];
    }
}

cudaError_t launch_build_pairs(const float4 *payload, float4 *pairs, int64_t n_prim, int m, cudaStream_t st) {
    const int64_t n = n_prim * m * m * (m - 1);
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    k_build_pairs<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(payload, pairs, n_prim, m);
    return cudaGetLastError();
}

// Candidates of a key-overflowed tile rebuilt from all K pixel rectangles (prim ids, any
// order: the window keeps the smallest (tEnter, prim) keys whatever the scan order). Same
// predicate and exact test as TileCands<false>, so the rays get the very same segment lists.
struct ListCands {
    const uint32_t *list;
    const float *xf_g;
    const int4 *prects_g;
    const float4 *payload;
    unsigned m3;
    int n;
    __device__ __forceinline__ int prim(int c) const { return (int)list[c]; }
    __device__ __forceinline__ const float *xf(int c) const { return xf_g + (size_t)prim(c) * kXfStride; }
    __device__ __forceinline__ Xf16 xfv(int c) const { return ldg_xf(xf(c)); }
    __device__ __forceinline__ const float4 *base(int c) const { return payload + (size_t)prim(c) * m3; }
    __device__ __forceinline__ bool covers(int c, int2 px) const {
        const int4 r = prects_g[prim(c)];
        return px.x >= r.x && px.x <= r.z && px.y >= r.y && px.y <= r.w;
    }
    __device__ __forceinline__ bool hit(int c, V3 o, V3 d, float &tE, float &tX) const {
        return intersect_obb(xf(c), o, d, tE, tX);
    }
};

__device__ __forceinline__ void fallback_pixel(const ViewDev &vd, const MarchDev &mp, int p, RayOut &ro,
                                               bool &ok, const ListCands *lc, const float *xf_g,
                                               const float4 *payload, unsigned m3, const Window<int> &w,
                                               const unsigned long long *tab) {
    const CamDev &cam = vd.cam;
    const int px = p % cam.width, py = p / cam.width;
    V3 o, d;
    generate_ray(cam, (float)px + 0.5f, (float)py + 0.5f, o, d);
    const float jit = mp.jitter ? hash_to_unit(hash_combine(mp.seed, (uint64_t)(uint32_t)p)) : 0.5f;
    if (lc) {
        ro = march_ray<kFallbackCap>(*lc, w, o, d, make_int2(px, py), jit, mp, tab);
    } else {
        const int tile = (py / kTile) * cam.tiles_x + px / kTile;
        const uint32_t start = vd.offsets[tile];
        const TileCands<false> cands{vd.entries, xf_g, vd.prects, payload, m3, start,
                                     (int)(vd.offsets[tile + 1] - start), nullptr, nullptr, nullptr,
                                     nullptr};
        ro = march_ray<kFallbackCap>(cands, w, o, d, make_int2(px, py), jit, mp, tab);
    }
    ok = !ro.overflow;
    if (!ok) {  // more live segments than kFallbackCap: the huge pass takes the pixel
        const unsigned slot = atomicAdd(&vd.ctr->huge_rays, 1u);
        if ((int)slot < vd.huge_cap) vd.huge_list[slot] = p;
        else atomicAdd(&vd.ctr->fallback_fail, 1);
        return;
    }
    write_pixel(vd.od, p, ro);
}

// All K primitives as candidates, filtered by their pixel rectangles (k_march_huge_views).
struct AllCands {
    const float *xf_g;
    const int4 *prects_g;
    const float4 *payload;
    unsigned m3;
    int n;
    static constexpr bool kRs = false;
    __device__ __forceinline__ int prim(int c) const { return c; }
    __device__ __forceinline__ const float *xf(int c) const { return xf_g + (size_t)c * kXfStride; }
    __device__ __forceinline__ Xf16 xfv(int c) const { return ldg_xf(xf(c)); }
    __device__ __forceinline__ const float4 *base(int c) const { return payload + (size_t)c * m3; }
    __device__ __forceinline__ bool covers(int c, int2 px) const {
        const int4 r = prects_g[c];
        return px.x >= r.x && px.x <= r.z && px.y >= r.y && px.y <= r.w;
    }
    __device__ __forceinline__ bool hit(int c, V3 o, V3 d, float &tE, float &tX) const {
        return intersect_obb(xf(c), o, d, tE, tX);
    }
};

// K5c: camera pixels with more than kFallbackCap live segments, marched with kHugeCap-entry
// windows over all primitives (the window keeps the smallest (tEnter, prim) keys whatever the
// candidate order, so the segment lists are the tile kernel's). Beyond kHugeCap: Numeric.
__global__ void __launch_bounds__(32)
k_march_huge_views(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
                   ViewBatch views, float *scratch_e, float *scratch_x, int *scratch_c) {
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const Window<int> w{scratch_e, scratch_x, scratch_c, nthreads, gtid};
    const unsigned m3 = (unsigned)(mp.m * mp.m * mp.m);
    for (int v = 0; v < views.n; ++v) {
        const ViewDev &vd = views.v[v];
        DevCounters *ctr = vd.ctr;
        const int n = (int)min((unsigned)vd.huge_cap, ctr->huge_rays);
        const CamDev &cam = vd.cam;
        const AllCands all{xf_g, vd.prects, payload, m3, n_prim};
        for (int q = gtid; q < n; q += nthreads) {
            const int p = vd.huge_list[q];
            const int px = p % cam.width, py = p / cam.width;
            V3 o, d;
            generate_ray(cam, (float)px + 0.5f, (float)py + 0.5f, o, d);
            const float jit = mp.jitter ? hash_to_unit(hash_combine(mp.seed, (uint64_t)(uint32_t)p)) : 0.5f;
            const RayOut ro = march_ray<kHugeCap>(all, w, o, d, make_int2(px, py), jit, mp, s_tab);
            if (ro.overflow) {
                atomicAdd(&ctr->fallback_fail, 1);
                continue;
            }
            write_pixel(vd.od, p, ro);
            atomicAdd(&ctr->ray_samples, (unsigned long long)ro.samples);  // rare path: plain atomics
            atomicAdd(&ctr->prim_samples, (unsigned long long)ro.prim_samples);
            atomicAdd(&ctr->hit_rays, (unsigned long long)ro.hit);
            atomicAdd(&ctr->early_exits, (unsigned long long)ro.early);
            atomicAdd(&ctr->saturated, (unsigned long long)ro.saturated);
            atomicAdd(&ctr->refills, (unsigned long long)ro.refills);
            if (ro.numeric) atomicAdd(&ctr->numeric_fail, 1ull);
        }
    }
}

cudaError_t launch_march_huge_views(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                    const ViewBatch &views, float *se, float *sx, int *sc, cudaStream_t st) {
    k_march_huge_views<<<kHugeThreads / 32, 32, 0, st>>>(mp, xf16, n_prim, payload, views, se, sx, sc);
    return cudaGetLastError();
}

// K5b over every view of a launch.
//  (1) Key-overflowed tiles (their bucket did not fit the entries buffer; K3 and K5 skipped
//      them): each CTA takes such tiles in turn, rebuilds the tile's candidate list from all K
//      pixel rectangles (the tile-rectangle test K1/K3 use) into its slice of `tile_scratch`,
//      and marches the tile's pixels with kFallbackCap-entry windows. Nothing is skipped, so an
//      async render is exact whatever the key capacity.
//  (2) The rays whose live segments overflowed K5's window, re-marched wide.
__global__ void __launch_bounds__(kFallbackThreads)
k_march_fallback_views(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
                       ViewBatch views, float *scratch_e, float *scratch_x, int *scratch_c,
                       uint32_t *__restrict__ tile_scratch) {
    __shared__ unsigned long long s_tab[32];
    __shared__ int s_warp[kFallbackThreads / 32];
    __shared__ int s_n;
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const Window<int> w{scratch_e, scratch_x, scratch_c, nthreads, gtid};
    const unsigned m3 = (unsigned)(mp.m * mp.m * mp.m);
    for (int v = 0; v < views.n; ++v) {
        const ViewDev &vd = views.v[v];
        DevCounters *ctr = vd.ctr;
        if (!ctr->key_overflow) continue;
        const CamDev &cam = vd.cam;
        const unsigned cap = ctr->key_cap;
        const int n_tiles = cam.tiles_x * cam.tiles_y;
        uint32_t *list = tile_scratch + (size_t)blockIdx.x * n_prim;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            if (!tile_key_overflowed(vd.offsets, t, cap)) continue;  // uniform over the CTA
            const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
            if (tid == 0) s_n = 0;
            __syncthreads();
            for (int base = 0; base < n_prim; base += kFallbackThreads) {  // compaction in prim order
                const int k = base + tid;
                bool in = false;
                if (k < n_prim) {
                    const int4 r = vd.prects[k];
                    in = r.z >= r.x && r.w >= r.y && tx >= r.x / kTile && tx <= r.z / kTile &&
                         ty >= r.y / kTile && ty <= r.w / kTile;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                if (lane == 0) s_warp[wid] = __popc(bal);
                __syncthreads();
                int off = s_n;
                for (int q = 0; q < wid; ++q) off += s_warp[q];
                if (in) list[off + __popc(bal & ((1u << lane) - 1))] = (uint32_t)k;
                __syncthreads();
                if (tid == 0)
                    for (int q = 0; q < kFallbackThreads / 32; ++q) s_n += s_warp[q];
                __syncthreads();
            }
            __threadfence_block();
            const ListCands lc{list, xf_g, vd.prects, payload, m3, s_n};
            for (int q = tid; q < kTile * kTile; q += kFallbackThreads) {
                const int2 pp = make_int2(tx * kTile + (q & 15), ty * kTile + (q >> 4));
                RayOut ro{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
                bool ok = false;
                if (pp.x < cam.width && pp.y < cam.height)
                    fallback_pixel(vd, mp, pp.y * cam.width + pp.x, ro, ok, &lc, xf_g, payload, m3, w, s_tab);
                add_counters(ctr, ro, ok);
            }
            __syncthreads();  // the list slice is reused by the CTA's next tile
        }
    }
    for (int v = 0; v < views.n; ++v) {
        const ViewDev &vd = views.v[v];
        DevCounters *ctr = vd.ctr;
        const int n_ovf = (int)min((unsigned long long)vd.ovf_cap, ctr->overflow_rays);
        for (int q = gtid; q < n_ovf; q += nthreads) {
            RayOut ro;
            bool ok;
            fallback_pixel(vd, mp, vd.ovf_list[q], ro, ok, nullptr, xf_g, payload, m3, w, s_tab);
            if (!ok) continue;
            atomicAdd(&ctr->ray_samples, (unsigned long long)ro.samples);  // rare path: plain atomics
            atomicAdd(&ctr->prim_samples, (unsigned long long)ro.prim_samples);
            atomicAdd(&ctr->hit_rays, (unsigned long long)ro.hit);
            atomicAdd(&ctr->early_exits, (unsigned long long)ro.early);
            atomicAdd(&ctr->saturated, (unsigned long long)ro.saturated);
            atomicAdd(&ctr->refills, (unsigned long long)ro.refills);
            if (ro.numeric) atomicAdd(&ctr->numeric_fail, 1ull);
        }
    }
}

cudaError_t launch_march_fallback_views(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                        const ViewBatch &views, float *se, float *sx, int *sc,
                                        uint32_t *tile_scratch, cudaStream_t st) {
    k_march_fallback_views<<<kOvfTileBlocks, kFallbackThreads, 0, st>>>(mp, xf16, n_prim, payload, views, se, sx,
                                                                        sc, tile_scratch);
    return cudaGetLastError();
}

// Heaviest-first order over several views' tiles: one CTA, counting sort of min(count, 1023)
// descending; entries are (view << 20 | tile).
struct BatchCounts {
    const uint32_t *counts[kMaxViews];
    int n_tiles[kMaxViews];
    int n;
};
__global__ void k_batch_order(BatchCounts bc, uint32_t *__restrict__ order) {
    __shared__ unsigned hist[kOrderBuckets];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int b = tid; b < kOrderBuckets; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int v = 0; v < bc.n; ++v)
        for (int t = tid; t < bc.n_tiles[v]; t += blockDim.x)
            atomicAdd(&hist[min(bc.counts[v][t], (uint32_t)kOrderBuckets - 1)], 1u);
    __syncthreads();
    if (wid == 0) {  // exclusive scan over buckets in descending order, 32 buckets per lane
        unsigned local = 0;
        for (int q = 0; q < kOrderBuckets / 32; ++q) local += hist[kOrderBuckets - 1 - (lane * 32 + q)];
        unsigned incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        unsigned run = incl - local;
        for (int q = 0; q < kOrderBuckets / 32; ++q) {
            const int b = kOrderBuckets - 1 - (lane * 32 + q);
            const unsigned h = hist[b];
            hist[b] = run;
            run += h;
        }
    }
    __syncthreads();
    for (int v = 0; v < bc.n; ++v)
        for (int t = tid; t < bc.n_tiles[v]; t += blockDim.x)
            order[atomicAdd(&hist[min(bc.counts[v][t], (uint32_t)kOrderBuckets - 1)], 1u)] =
                ((uint32_t)v << 20) | (uint32_t)t;
}

cudaError_t launch_batch_order(const uint32_t *const *tile_counts, const int *n_tiles, int n_views, uint32_t *order,
                               cudaStream_t st) {
    BatchCounts bc{};
    bc.n = n_views;
    for (int v = 0; v < n_views; ++v) {
        bc.counts[v] = tile_counts[v];
        bc.n_tiles[v] = n_tiles[v];
    }
    k_batch_order<<<1, 1024, 0, st>>>(bc, order);
    return cudaGetLastError();
}

cudaError_t launch_march_fallback(bool rays_mode, const CamDev &cam, const MarchDev &mp,
                                  const float *xf16, const int4 *prects, int n_prim,
                                  const float4 *payload, const uint32_t *offsets,
                                  const unsigned long long *entries, const OutDev &od,
                                  const RaysDev &rays, DevCounters *ctr, const int *ovf_list,
                                  int ovf_cap, float *se, float *sx, int *sc, cudaStream_t st, int *huge_list,
                                  int huge_cap) {
    // camera renders re-march their overflow rays in k_march_fallback_views
    if (!rays_mode) return cudaErrorInvalidValue;
    return launch_pdl(k_march_fallback<true>, dim3(kFallbackBlocks), dim3(kFallbackThreads), 0, st, cam, mp, xf16,
                      prects, n_prim, payload, offsets, entries, od, rays, ctr, ovf_list, ovf_cap, se, sx, sc,
                      huge_list, huge_cap);
}

// K5c for arbitrary rays: kHugeCap-entry windows through the BVH, one thread per ray.
__global__ void __launch_bounds__(32)
k_march_huge_rays(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
                  OutDev od, RaysDev rays, DevCounters *ctr, const int *__restrict__ huge_list, int huge_cap,
                  float *scratch_e, float *scratch_x, int *scratch_c) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    const int n = (int)min((unsigned)huge_cap, ctr->huge_rays);
    if (n == 0) return;
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const Window<int> w{scratch_e, scratch_x, scratch_c, nthreads, gtid};
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    for (int q = gtid; q < n; q += nthreads) {
        const int p = huge_list[q];
        const V3 o = mk3(rays.origins[3 * p], rays.origins[3 * p + 1], rays.origins[3 * p + 2]);
        const V3 d = mk3(rays.dirs[3 * p], rays.dirs[3 * p + 1], rays.dirs[3 * p + 2]);
        const float jit = rays.jitter ? rays.jitter[p] : 0.5f;
        const RayOut ro = march_ray<kHugeCap>(cands, w, o, d, make_int2(0, 0), jit, mp, s_tab);
        if (ro.overflow) {
            atomicAdd(&ctr->fallback_fail, 1);
            continue;
        }
        write_ray(od, p, ro);
        if (od.state) od.state[8 * (size_t)p + 7] = __int_as_float(-2);  // the backward's huge pass
        atomicAdd(&ctr->ray_samples, (unsigned long long)ro.samples);
        atomicAdd(&ctr->prim_samples, (unsigned long long)ro.prim_samples);
        atomicAdd(&ctr->hit_rays, (unsigned long long)ro.hit);
        atomicAdd(&ctr->early_exits, (unsigned long long)ro.early);
        atomicAdd(&ctr->saturated, (unsigned long long)ro.saturated);
        atomicAdd(&ctr->refills, (unsigned long long)ro.refills);
        if (ro.numeric) atomicAdd(&ctr->numeric_fail, 1ull);
    }
}

cudaError_t launch_march_huge_rays(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                   const OutDev &od, const RaysDev &rays, DevCounters *ctr, const int *huge_list,
                                   int huge_cap, float *se, float *sx, int *sc, cudaStream_t st) {
    return launch_pdl(k_march_huge_rays, dim3(kHugeThreads / 32), dim3(32), 0, st, mp, xf16, n_prim, payload, od, rays,
                      ctr, huge_list, huge_cap, se, sx, sc);
}

cudaError_t launch_march_rays(const MarchDev &mp, const float *xf16, int n_prim,
                              const float4 *payload, const RaysDev &rays, int64_t n_rays,
                              const OutDev &od, DevCounters *ctr, int *ovf_list, int ovf_cap,
                              cudaStream_t st) {
    if (n_rays == 0) return cudaSuccess;
    // Each ray is a serial latency chain, so rays are marched a warp per ray, 32 lattice steps
    // at a time. Since the warp walks the BVH cooperatively (warp_bvh_leaves) this wins at
    // every batch size measured (65,536 rays: 1.05 -> 0.7 ms against one thread per ray, a
    // kernel since removed).
    const int64_t blocks = (n_rays + 3) / 4;
#ifndef VPB_RAYS_GRID
#define VPB_RAYS_GRID 96  // CTAs per SM in the grid (backward rays/s at 5 CTAs/SM: 16 54.4M, 64 56.8M, one ray per warp 55.9M; at 7: 64 63.0M, 96 63.4M, 128 62.4M)
#endif
    const unsigned grid = (unsigned)(blocks < 148 * VPB_RAYS_GRID ? blocks : 148 * VPB_RAYS_GRID);
    const bool big = n_rays >= 8192;
#define VPB_RAYS_LAUNCH(MT, MB)                                                                               \
    k_march_rays_warp<MT, MB><<<grid, 128, 0, st>>>(mp, xf16, n_prim, payload, rays, n_rays, od, ctr, ovf_list, \
                                                    ovf_cap)
    switch (mp.m) {  // compile-time voxel counts for the common grids (immediate corner offsets)
    case 8: big ? VPB_RAYS_LAUNCH(8, VPB_RAYS_MINB) : VPB_RAYS_LAUNCH(8, 5); break;
    case 16: big ? VPB_RAYS_LAUNCH(16, VPB_RAYS_MINB) : VPB_RAYS_LAUNCH(16, 5); break;
    case 32: big ? VPB_RAYS_LAUNCH(32, VPB_RAYS_MINB) : VPB_RAYS_LAUNCH(32, 5); break;
    default: VPB_RAYS_LAUNCH(0, 5); break;
    }
#undef VPB_RAYS_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_composite(const float *rgb, const float *alpha, const float *bg, float *out,
                             int64_t n_px, cudaStream_t st) {
    if (n_px == 0) return cudaSuccess;
    k_composite<<<(unsigned)((n_px + 255) / 256), 256, 0, st>>>(rgb, alpha, bg, out, n_px);
    return cudaGetLastError();
}

cudaError_t launch_expf(const float *x, float *y, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_expf<<<148 * 8, 256, 0, st>>>(x, y, n);
    return cudaGetLastError();
}

} // namespace vpb
