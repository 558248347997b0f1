// vpb_bvh.cu — device build of the linear BVH used by arbitrary-ray marching (vpb_bvh.cuh).
// Replaces the reference's host buildLbvh (lbvh.cpp:48-156) for march() / backwardRay /
// evalLoss rays; camera renders use the tile lists instead (vpb_kernels.cu K1-K3).
//
//   k_bvh_boxes     padded world box per primitive (from the composed transform)
//   k_bvh_bounds    one CTA: bounds of the box centres
//   k_bvh_keys      (30-bit Morton code of the centre << 32) | primitive
//   k_radix_*       stable LSD radix sort of the keys on their 30 Morton bits (in-house: four
//                   8-bit digit passes of tile histogram -> digit-major scan -> stable scatter;
//                   up to 8192 keys in one CTA out of shared memory)
//   k_bvh_internal  Karras (2012) hierarchy from the sorted keys: one thread per internal node
//   k_bvh_refit     bottom-up child boxes (second arrival at a node computes it)
//
// The boxes only prune, so they are padded generously: a ray the exact model-space test
// reports as a hit must never be pruned by float rounding in the world-space slab test.
#include <cuda_runtime.h>

#include <cstdint>

#include "vpb_bvh.cuh"
#include "vpb_device.cuh"
#include "vpb_kernels.h"

namespace vpb {

__global__ void k_bvh_boxes(const float *__restrict__ xf16, int n, float4 *__restrict__ lo,
                            float4 *__restrict__ hi) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const float *x = xf16 + (size_t)k * kXfStride;
    // half extent along world axis a: sum_j |R(a, j)| s_j (R column-major: R(a, j) = x[3 + 3j + a])
    float h[3], c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        h[a] = fabsf(x[3 + a]) * x[12] + fabsf(x[6 + a]) * x[13] + fabsf(x[9 + a]) * x[14];
        c[a] = x[a];
        h[a] = h[a] * 1.001f + 1e-4f * (fabsf(c[a]) + h[a]) + 1e-7f;
    }
    lo[k] = make_float4(c[0] - h[0], c[1] - h[1], c[2] - h[2], 0.0f);
    hi[k] = make_float4(c[0] + h[0], c[1] + h[1], c[2] + h[2], 0.0f);
}

__global__ void k_bvh_bounds(const float *__restrict__ xf16, int n, float *__restrict__ bounds) {
    __shared__ float s[6][32];
    float mn[3] = {3.402823466e+38f, 3.402823466e+38f, 3.402823466e+38f};
    float mx[3] = {-3.402823466e+38f, -3.402823466e+38f, -3.402823466e+38f};
    for (int k = threadIdx.x; k < n; k += blockDim.x)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float v = xf16[(size_t)k * kXfStride + a];
            mn[a] = fminf(mn[a], v);
            mx[a] = fmaxf(mx[a], v);
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s[a][wid] = mn[a];
            s[3 + a][wid] = mx[a];
        }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int a = threadIdx.x;
        float lo = 3.402823466e+38f, hi = -3.402823466e+38f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            lo = fminf(lo, s[a][w]);
            hi = fmaxf(hi, s[3 + a][w]);
        }
        bounds[a] = lo;
        bounds[3 + a] = hi;
    }
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_bvh_keys(const float *__restrict__ xf16, int n, const float *__restrict__ bounds,
                           unsigned long long *__restrict__ keys) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float ext = bounds[3 + a] - bounds[a];
        const float u = ext > 0.0f ? (xf16[(size_t)k * kXfStride + a] - bounds[a]) / ext : 0.0f;
        q[a] = (uint32_t)fminf(fmaxf(u * 1024.0f, 0.0f), 1023.0f);
    }
    const uint32_t morton = spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
    keys[k] = ((unsigned long long)morton << 32) | (uint32_t)k;
}

__device__ __forceinline__ int bvh_delta(const unsigned long long *keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    return __clzll(keys[i] ^ keys[j]);  // keys are distinct (primitive index in the low bits)
}

// Internal node i of n - 1. parent[] holds internal nodes at [0, n-1), leaves at n-1 + position.
__global__ void k_bvh_internal(const unsigned long long *__restrict__ keys, int n, BvhNode *__restrict__ nodes,
                               int *__restrict__ parent) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = bvh_delta(keys, n, i, i + 1) - bvh_delta(keys, n, i, i - 1) > 0 ? 1 : -1;
    const int dmin = bvh_delta(keys, n, i, i - d);
    int lmax = 2;
    while (bvh_delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (bvh_delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = bvh_delta(keys, n, i, j);
    int s = 0, t = l;
    do {
        t = (t + 1) >> 1;
        if (bvh_delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    const int gamma = i + s * d + (d < 0 ? -1 : 0);
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    int left, right;
    if (lo == gamma) {
        left = -(int)(uint32_t)(keys[gamma] & 0xffffffffull) - 1;
        parent[n - 1 + gamma] = i;
    } else {
        left = gamma;
        parent[gamma] = i;
    }
    if (hi == gamma + 1) {
        right = -(int)(uint32_t)(keys[gamma + 1] & 0xffffffffull) - 1;
        parent[n - 1 + gamma + 1] = i;
    } else {
        right = gamma + 1;
        parent[gamma + 1] = i;
    }
    nodes[i].d = make_int4(left, right, 0, 0);
    if (i == 0) parent[0] = -1;
}

__global__ void k_bvh_refit(const unsigned long long *__restrict__ keys, int n, const float4 *__restrict__ lo,
                            const float4 *__restrict__ hi, BvhNode *nodes, float4 *nlo, float4 *nhi,
                            const int *__restrict__ parent, unsigned *flags) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int node = parent[n - 1 + p];
    while (node >= 0) {
        if (atomicAdd(&flags[node], 1u) == 0) return;  // the sibling subtree is not done yet
        __threadfence();
        const int4 ch = nodes[node].d;
        float4 l0, h0, l1, h1;
        if (ch.x < 0) {
            l0 = lo[-ch.x - 1];
            h0 = hi[-ch.x - 1];
        } else {
            l0 = __ldcg(nlo + ch.x);
            h0 = __ldcg(nhi + ch.x);
        }
        if (ch.y < 0) {
            l1 = lo[-ch.y - 1];
            h1 = hi[-ch.y - 1];
        } else {
            l1 = __ldcg(nlo + ch.y);
            h1 = __ldcg(nhi + ch.y);
        }
        nodes[node].a = make_float4(l0.x, l0.y, l0.z, h0.x);
        nodes[node].b = make_float4(h0.y, h0.z, l1.x, l1.y);
        nodes[node].c = make_float4(l1.z, h1.x, h1.y, h1.z);
        nlo[node] = make_float4(fminf(l0.x, l1.x), fminf(l0.y, l1.y), fminf(l0.z, l1.z), 0.0f);
        nhi[node] = make_float4(fmaxf(h0.x, h1.x), fmaxf(h0.y, h1.y), fmaxf(h0.z, h1.z), 0.0f);
        __threadfence();
        node = parent[node];
    }
}

// ---- stable LSD radix sort of 64-bit keys on bits [32, 62) ------------------------------------
// A pass sorts on one 8-bit digit (the last one on 6 bits): (1) k_radix_hist counts the digits of
// each tile of kRadixTile keys into hist[digit * n_tiles + tile]; (2) k_radix_scan, one CTA,
// turns that digit-major table into exclusive offsets (digit-major order = the stable order);
// (3) k_radix_scatter ranks each key inside its tile, in tile order, and writes it to
// offset[digit][tile] + rank. The keys start in primitive order, so equal Morton codes keep
// that order: the result is the order of the full 62-bit keys, as buildLbvh sorts them
// (lbvh.cpp:81-100).
constexpr int kRadixThreads = 256, kRadixItems = 8, kRadixTile = kRadixThreads * kRadixItems;
constexpr int kRadixBins = 256;

__device__ __forceinline__ unsigned radix_digit(unsigned long long key, int shift) {
    return (unsigned)(key >> shift) & (kRadixBins - 1);
}

__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const unsigned long long *__restrict__ keys, int n,
                                                              int shift, unsigned *__restrict__ hist, int n_tiles) {
    __shared__ unsigned h[kRadixBins];
    for (int b = threadIdx.x; b < kRadixBins; b += kRadixThreads) h[b] = 0u;
    __syncthreads();
    const int base = blockIdx.x * kRadixTile;
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const int i = base + r * kRadixThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[radix_digit(keys[i], shift)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kRadixBins; b += kRadixThreads) hist[b * n_tiles + blockIdx.x] = h[b];
}

// One CTA: exclusive scan of the m = 256 * n_tiles counts in place.
__global__ void __launch_bounds__(1024) k_radix_scan(unsigned *__restrict__ hist, int m) {
    __shared__ unsigned warp_sums[32];
    __shared__ unsigned carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < m; base += 1024) {
        const int i = base + tid;
        const unsigned v = i < m ? hist[i] : 0u;
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) warp_sums[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            unsigned ws = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += u;
            }
            warp_sums[lane] = ws;
        }
        __syncthreads();
        const unsigned excl = carry + (wid ? warp_sums[wid - 1] : 0u) + incl - v;
        if (i < m) hist[i] = excl;
        __syncthreads();
        if (tid == 1023) carry = excl + v;
        __syncthreads();
    }
}

// Stable scatter of one tile: kRadixItems rounds of kRadixThreads keys in index order. Inside a
// round a key's rank among equal digits = its rank in its warp (__match_any_sync) + the counts of
// the earlier warps + the keys of earlier rounds.
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const unsigned long long *__restrict__ in,
                                                                 unsigned long long *__restrict__ out, int n,
                                                                 int shift, const unsigned *__restrict__ offs,
                                                                 int n_tiles) {
    constexpr int kWarps = kRadixThreads / 32;
    __shared__ unsigned run[kRadixBins];           // offset of the next key of each digit
    __shared__ unsigned wcnt[kWarps][kRadixBins];  // per warp: its count, then its exclusive prefix
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int b = tid; b < kRadixBins; b += kRadixThreads) run[b] = offs[b * n_tiles + blockIdx.x];
    const int base = blockIdx.x * kRadixTile;
    for (int r = 0; r < kRadixItems; ++r) {
        for (int b = tid; b < kWarps * kRadixBins; b += kRadixThreads) (&wcnt[0][0])[b] = 0u;
        __syncthreads();
        const int i = base + r * kRadixThreads + tid;
        const bool valid = i < n;
        const unsigned long long key = valid ? in[i] : 0ull;
        const unsigned dg = valid ? radix_digit(key, shift) : kRadixBins;  // kRadixBins: no key
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const unsigned below = __popc(peers & ((1u << lane) - 1u));
        if (valid && below == 0) wcnt[wid][dg] = __popc(peers);  // the group's lowest lane
        __syncthreads();
        for (int b = tid; b < kRadixBins; b += kRadixThreads) {  // exclusive prefix over warps
            unsigned acc = run[b];
            for (int w = 0; w < kWarps; ++w) {
                const unsigned c = wcnt[w][b];
                wcnt[w][b] = acc;
                acc += c;
            }
            run[b] = acc;
        }
        __syncthreads();
        if (valid) out[wcnt[wid][dg] + below] = key;
        __syncthreads();
    }
}

// Up to kSmallSort keys: the whole sort in ONE CTA out of shared memory (the four passes of
// the same stable LSD scheme: histogram, scan, warp-ranked scatter), so a per-pose rebuild at
// K = 4096 costs one launch instead of twelve (the multi-CTA path is launch-latency bound there).
constexpr int kSmallSort = 8192, kSmallThreads = 1024, kSmallWarps = kSmallThreads / 32;

size_t small_sort_smem(int n) { return (size_t)2 * n * 8 + (size_t)kSmallWarps * kRadixBins * 4; }

__global__ void __launch_bounds__(kSmallThreads) k_radix_sort_small(unsigned long long *keys, int n) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long *a = reinterpret_cast<unsigned long long *>(smem), *b = a + n;
    unsigned *wcnt = reinterpret_cast<unsigned *>(b + n);  // [kSmallWarps][kRadixBins]
    __shared__ unsigned run[kRadixBins];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < n; i += kSmallThreads) a[i] = keys[i];
    for (int shift = 32; shift < 62; shift += 8) {
        for (int q = tid; q < kRadixBins; q += kSmallThreads) run[q] = 0u;
        __syncthreads();
        for (int i = tid; i < n; i += kSmallThreads) atomicAdd(&run[radix_digit(a[i], shift)], 1u);
        __syncthreads();
        if (wid == 0) {  // exclusive scan of the 256 counts, 8 per lane
            unsigned v[kRadixBins / 32], sum = 0;
#pragma unroll
            for (int q = 0; q < kRadixBins / 32; ++q) {
                v[q] = run[lane * (kRadixBins / 32) + q];
                sum += v[q];
            }
            unsigned incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            unsigned acc = incl - sum;
#pragma unroll
            for (int q = 0; q < kRadixBins / 32; ++q) {
                run[lane * (kRadixBins / 32) + q] = acc;
                acc += v[q];
            }
        }
        __syncthreads();
        for (int base = 0; base < n; base += kSmallThreads) {  // stable: chunks in index order
            for (int q = tid; q < kSmallWarps * kRadixBins; q += kSmallThreads) wcnt[q] = 0u;
            __syncthreads();
            const int i = base + tid;
            const bool valid = i < n;
            const unsigned long long key = valid ? a[i] : 0ull;
            const unsigned dg = valid ? radix_digit(key, shift) : kRadixBins;
            const unsigned peers = __match_any_sync(0xffffffffu, dg);
            const unsigned below = __popc(peers & ((1u << lane) - 1u));
            if (valid && below == 0) wcnt[wid * kRadixBins + dg] = __popc(peers);
            __syncthreads();
            for (int q = tid; q < kRadixBins; q += kSmallThreads) {
                unsigned acc = run[q];
                for (int w = 0; w < kSmallWarps; ++w) {
                    const unsigned c = wcnt[w * kRadixBins + q];
                    wcnt[w * kRadixBins + q] = acc;
                    acc += c;
                }
                run[q] = acc;
            }
            __syncthreads();
            if (valid) b[wcnt[wid * kRadixBins + dg] + below] = key;
            __syncthreads();
        }
        unsigned long long *t = a;
        a = b;
        b = t;
    }
    for (int i = tid; i < n; i += kSmallThreads) keys[i] = a[i];  // four passes: back in the first buffer
}

// Stable sort of n keys on bits [32, 62) into `keys` (tmp / hist: the multi-CTA path's scratch).
cudaError_t radix_sort30(unsigned long long *keys, unsigned long long *tmp, unsigned *hist, int n, cudaStream_t st) {
    if (n <= 1) return cudaSuccess;
    if (n <= kSmallSort) {
        static bool attr_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr_set[dev]) {
            cudaFuncSetAttribute(k_radix_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)small_sort_smem(kSmallSort));
            if (dev >= 0 && dev < 64) attr_set[dev] = true;
        }
        k_radix_sort_small<<<1, kSmallThreads, small_sort_smem(n), st>>>(keys, n);
        return cudaGetLastError();
    }
    const int nt = (n + kRadixTile - 1) / kRadixTile;
    unsigned long long *src = keys, *dst = tmp;
    for (int shift = 32; shift < 62; shift += 8) {
        k_radix_hist<<<nt, kRadixThreads, 0, st>>>(src, n, shift, hist, nt);
        k_radix_scan<<<1, 1024, 0, st>>>(hist, kRadixBins * nt);
        k_radix_scatter<<<nt, kRadixThreads, 0, st>>>(src, dst, n, shift, hist, nt);
        unsigned long long *t = src;
        src = dst;
        dst = t;
    }
    return cudaGetLastError();  // an even number of passes: the result is back in keys
}

// Scratch carve-up, shared by the size query and the build.
struct BvhScratch {
    float4 *lo, *hi, *nlo, *nhi;
    unsigned long long *k0, *k1;
    int *parent;
    unsigned *flags;
    float *bounds;
    unsigned *hist;  // radix sort: 256 digits x tiles
    int n_tiles;
    size_t total;
};
static BvhScratch bvh_layout(int n, void *base) {
    BvhScratch s{};
    unsigned char *p = static_cast<unsigned char *>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        void *q = p ? p + off : nullptr;
        off += (bytes + 255) / 256 * 256;
        return q;
    };
    s.lo = static_cast<float4 *>(take((size_t)n * 16));
    s.hi = static_cast<float4 *>(take((size_t)n * 16));
    s.nlo = static_cast<float4 *>(take((size_t)n * 16));
    s.nhi = static_cast<float4 *>(take((size_t)n * 16));
    s.k0 = static_cast<unsigned long long *>(take((size_t)n * 8));
    s.k1 = static_cast<unsigned long long *>(take((size_t)n * 8));
    s.parent = static_cast<int *>(take((size_t)(2 * n) * 4));
    s.flags = static_cast<unsigned *>(take((size_t)n * 4));
    s.bounds = static_cast<float *>(take(64));
    s.n_tiles = (n + kRadixTile - 1) / kRadixTile;
    s.hist = static_cast<unsigned *>(take((size_t)kRadixBins * s.n_tiles * 4));
    s.total = off;
    return s;
}

size_t bvh_scratch_bytes(int n) { return n > 1 ? bvh_layout(n, nullptr).total : 0; }

// The BVH's key sort alone (testing): sorts n keys on bits [32, 62), stable; keys/tmp device.
cudaError_t launch_radix_sort30(unsigned long long *keys, unsigned long long *tmp, unsigned *hist, int n,
                                cudaStream_t st) {
    return radix_sort30(keys, tmp, hist, n, st);
}

// BvhWide record of every internal node (after the refit): its eight great-grandchild slots.
__device__ __forceinline__ void wide_slot(BvhWide &w, int q, float4 a, float2 hyz, int id, bool valid) {
    w.s[2 * q] = a;
    w.s[2 * q + 1] = make_float4(hyz.x, hyz.y, __int_as_float(id), valid ? 1.0f : 0.0f);
}
// child c of a binary node: its box (lo.xyz hi.x | hi.yz) and index
__device__ __forceinline__ void node_child(const BvhNode &nd, int c, float4 &a, float2 &hyz, int &id) {
    if (c) {
        a = make_float4(nd.b.z, nd.b.w, nd.c.x, nd.c.y);
        hyz = make_float2(nd.c.z, nd.c.w);
        id = nd.d.y;
    } else {
        a = nd.a;
        hyz = make_float2(nd.b.x, nd.b.y);
        id = nd.d.x;
    }
}
__global__ void k_bvh_widen(const BvhNode *__restrict__ nodes, int n_internal, BvhWide *__restrict__ wide) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_internal) return;
    const float inf = __int_as_float(0x7f800000);
    const float4 ea = make_float4(inf, inf, inf, -inf);
    const float2 eh = make_float2(-inf, -inf);
    const BvhNode nd = nodes[i];
    BvhWide w;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        float4 ca;
        float2 ch;
        int cid;
        node_child(nd, c, ca, ch, cid);
        if (cid < 0) {  // a leaf child: slot 4c, the rest of its group empty
            wide_slot(w, 4 * c, ca, ch, cid, true);
            for (int q = 1; q < 4; ++q) wide_slot(w, 4 * c + q, ea, eh, 0, false);
            continue;
        }
        const BvhNode cn = nodes[cid];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            float4 ga;
            float2 gh;
            int gid;
            node_child(cn, g, ga, gh, gid);
            if (gid < 0) {  // a leaf grandchild: slot 4c + 2g, its pair empty
                wide_slot(w, 4 * c + 2 * g, ga, gh, gid, true);
                wide_slot(w, 4 * c + 2 * g + 1, ea, eh, 0, false);
                continue;
            }
            const BvhNode gn = nodes[gid];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float4 ha;
                float2 hh;
                int hid;
                node_child(gn, h, ha, hh, hid);
                wide_slot(w, 4 * c + 2 * g + h, ha, hh, hid, true);
            }
        }
    }
    wide[i] = w;
}

// New boxes in the topology of the last launch_bvh_build over the same n primitives (its sorted
// keys and parent links are still in the scratch): the leaves' boxes from the current
// transforms, then the bottom-up refit and the wide records. The hierarchy stays exact (every
// box bounds its subtree), so walks find the same leaves; only its quality ages.
cudaError_t launch_bvh_refit(const float *xf16, int n, BvhNode *nodes, BvhWide *wide, void *scratch,
                             size_t scratch_bytes, cudaStream_t st) {
    if (n <= 1) return cudaSuccess;
    const BvhScratch sc = bvh_layout(n, scratch);
    if (sc.total > scratch_bytes) return cudaErrorInvalidValue;
    const int b = (n + 255) / 256;
    k_bvh_boxes<<<b, 256, 0, st>>>(xf16, n, sc.lo, sc.hi);
    cudaMemsetAsync(sc.flags, 0, (size_t)n * 4, st);
    k_bvh_refit<<<b, 256, 0, st>>>(sc.k0, n, sc.lo, sc.hi, nodes, sc.nlo, sc.nhi, sc.parent, sc.flags);
    if (wide) k_bvh_widen<<<(n - 1 + 255) / 256, 256, 0, st>>>(nodes, n - 1, wide);
    return cudaGetLastError();
}

cudaError_t launch_bvh_build(const float *xf16, int n, BvhNode *nodes, BvhWide *wide, void *scratch,
                             size_t scratch_bytes, cudaStream_t st) {
    if (n <= 1) return cudaSuccess;
    const BvhScratch sc = bvh_layout(n, scratch);
    if (sc.total > scratch_bytes) return cudaErrorInvalidValue;
    float4 *lo = sc.lo, *hi = sc.hi, *nlo = sc.nlo, *nhi = sc.nhi;
    unsigned long long *k0 = sc.k0, *k1 = sc.k1;  // radix ping-pong buffers
    int *parent = sc.parent;
    unsigned *flags = sc.flags;
    float *bounds = sc.bounds;
    const int b = (n + 255) / 256;
    k_bvh_boxes<<<b, 256, 0, st>>>(xf16, n, lo, hi);
    k_bvh_bounds<<<1, 1024, 0, st>>>(xf16, n, bounds);
    k_bvh_keys<<<b, 256, 0, st>>>(xf16, n, bounds, k0);
    // Only the 30 Morton bits are sorted (digits at bits 32, 40, 48, 56): the keys start in
    // primitive order and the sort is stable, so equal codes stay in index order, which is the
    // full 62-bit key order. The sorted keys end up in k0.
    if (cudaError_t e = radix_sort30(k0, k1, sc.hist, n, st)) return e;
    k_bvh_internal<<<(n - 1 + 255) / 256, 256, 0, st>>>(k0, n, nodes, parent);
    cudaMemsetAsync(flags, 0, (size_t)n * 4, st);
    k_bvh_refit<<<b, 256, 0, st>>>(k0, n, lo, hi, nodes, nlo, nhi, parent, flags);
    if (wide) k_bvh_widen<<<(n - 1 + 255) / 256, 256, 0, st>>>(nodes, n - 1, wide);
    return cudaGetLastError();
}

}  // namespace vpb
