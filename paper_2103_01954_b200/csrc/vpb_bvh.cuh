// vpb_bvh.cuh — candidate source for arbitrary rays (march(), backwardRay, evalLoss rays):
// a linear BVH over padded world boxes of the primitives, built on the device per frame
// (vpb_bvh.cu). It only prunes: every leaf it reaches gets the exact intersectObb test
// (lbvh.cpp:177-205), and the boxes are padded so a true hit is never pruned, so the hit lists
// equal brute force, which is what the reference's intersect() returns (lbvh.cpp:207-234;
// test_lbvh.cpp:184-210 checks intersect == brute force).
#pragma once

#include <cstdint>

#include "vpb_device.cuh"
#include "vpb_kernels.h"  // BvhNode, BvhDev

namespace vpb {

// Slab test of a ray (t >= 0) against an axis-aligned box; d components of 0 test the origin.
__device__ __forceinline__ bool ray_box(V3 o, V3 d, V3 inv, float lx, float ly, float lz, float hx, float hy,
                                        float hz) {
    float t0 = 0.0f, t1 = __int_as_float(0x7f800000);
#define VPB_SLAB(oa, da, ia, lo, hi)                                    \
    if (da == 0.0f) {                                                  \
        if (oa < lo || oa > hi) return false;                          \
    } else {                                                           \
        float ta = (lo - oa) * ia, tb = (hi - oa) * ia;                \
        if (ta > tb) {                                                 \
            const float s = ta;                                        \
            ta = tb;                                                   \
            tb = s;                                                    \
        }                                                              \
        t0 = ta > t0 ? ta : t0;                                        \
        t1 = tb < t1 ? tb : t1;                                        \
    }
    VPB_SLAB(o.x, d.x, inv.x, lx, hx)
    VPB_SLAB(o.y, d.y, inv.y, ly, hy)
    VPB_SLAB(o.z, d.z, inv.z, lz, hz)
#undef VPB_SLAB
    return t0 <= t1;
}

// Calls f(prim) for every primitive whose padded box the ray (t >= 0) passes through.
// Stack bound: the 62-bit keys (30-bit Morton code, 32-bit primitive index) are distinct, and
// a Karras child's key range shares a strictly longer prefix than its parent's, so the depth
// is at most 62; depth-first with one pending sibling per level needs at most 63 slots.
template <class F>
__device__ __forceinline__ void bvh_for_each(const BvhDev &bvh, V3 o, V3 d, F &&f) {
    if (bvh.n_prim <= 0) return;
    if (bvh.n_prim == 1) {
        f(0);
        return;
    }
    const V3 inv = mk3(1.0f / d.x, 1.0f / d.y, 1.0f / d.z);
    constexpr int kStack = 64;
    int stack[kStack];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const BvhNode n = bvh.nodes[stack[--sp]];
        const bool hl = ray_box(o, d, inv, n.a.x, n.a.y, n.a.z, n.a.w, n.b.x, n.b.y);
        const bool hr = ray_box(o, d, inv, n.b.z, n.b.w, n.c.x, n.c.y, n.c.z, n.c.w);
        if (hl) {
            if (n.d.x < 0) f(-n.d.x - 1);
            else stack[sp++ & (kStack - 1)] = n.d.x;
        }
        if (hr) {
            if (n.d.y < 0) f(-n.d.y - 1);
            else stack[sp++ & (kStack - 1)] = n.d.y;
        }
    }
}

}  // namespace vpb
