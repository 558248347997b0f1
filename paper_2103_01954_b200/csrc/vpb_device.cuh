// vpb_device.cuh — device-side arithmetic of the raymarcher, bit-faithful to the reference.
//
// The whole translation unit is compiled with -fmad=false (no FMA contraction), IEEE
// division and square root (no --use_fast_math), so each expression below rounds exactly
// like the reference's binary32 SSE code (which contains no vfmadd). Every
// helper keeps the reference's operation order; the cited lines are the ones restated.
#pragma once

#include <cstdint>

#include "vpb_camdev.h"

namespace vpb {

struct V3 {
    float x, y, z;
};

__device__ __forceinline__ V3 mk3(float x, float y, float z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(V3 a, float s) { return V3{a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ float dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float comp(V3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

// math.h:122-124 — col(0)*v.x + col(1)*v.y + col(2)*v.z on a column-major matrix.
__device__ __forceinline__ V3 matvec(const float *m, V3 v) {
    return (mk3(m[0], m[1], m[2]) * v.x + mk3(m[3], m[4], m[5]) * v.y) + mk3(m[6], m[7], m[8]) * v.z;
}
// Mat3::transpose() * v: column j of R^T is row j of R.
__device__ __forceinline__ V3 matTvec(const float *m, V3 v) {
    return (mk3(m[0], m[3], m[6]) * v.x + mk3(m[1], m[4], m[7]) * v.y) + mk3(m[2], m[5], m[8]) * v.z;
}

// Composed primitive transform, 16-float padded record: t[3] rot[9] scale[3] pad.
constexpr int kXfStride = 16;

// primitive.h:61-63 — AffineXf::toModel = (R^T (p - t)) ./ s
__device__ __forceinline__ V3 to_model(const float *xf, V3 p) {
    const V3 q = matTvec(xf + 3, p - mk3(xf[0], xf[1], xf[2]));
    return V3{q.x / xf[12], q.y / xf[13], q.z / xf[14]};
}

// lbvh.cpp:177-205 — exact oriented slab test in model space, with om = toModel(origin)
// supplied by the caller (it depends only on the primitive and the ray origin).
__device__ __forceinline__ bool intersect_obb_om(const float *xf, V3 om, V3 d, float &tEnterOut,
                                                 float &tExitOut) {
    const V3 q = matTvec(xf + 3, d);
    const V3 dm = V3{q.x / xf[12], q.y / xf[13], q.z / xf[14]};
    float tEnter = -3.402823466e+38f, tExit = 3.402823466e+38f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float oa = comp(om, a), da = comp(dm, a);
        if (da == 0.0f) {
            if (oa < -1.0f || oa > 1.0f) return false;
            continue;
        }
        const float inv = 1.0f / da;
        const float cNear = da > 0.0f ? -1.0f : 1.0f;
        const float t1 = (cNear - oa) * inv;
        const float t2 = (-cNear - oa) * inv;
        if (t1 > tEnter) tEnter = t1;
        tExit = t2 < tExit ? t2 : tExit;
    }
    if (tEnter < 0.0f) tEnter = 0.0f;
    if (tEnter >= tExit || tExit <= 0.0f) return false;
    tEnterOut = tEnter;
    tExitOut = tExit;
    return true;
}

// Conservative line-vs-box rejection in the primitive's rotated, unscaled frame, run before
// intersect_obb_om's six divisions: the ray's line misses the box of half-extents s iff one
// of the three axes e_a x q separates them, |o'_a q_b - o'_b q_a| > s_a |q_b| + s_b |q_a|, with
// o' = om * s and q = R^T d. It never rejects a hit of the exact test: a rejection needs the
// line to clear the box by a margin of 2^-15 of the terms' magnitudes (relative rounding of
// every quantity involved, om's and the slab test's t-values included, is below 2^-20), so a
// rejected candidate misses by far more than intersect_obb_om's rounding can bridge.
// Returns true when the exact test is still needed.
__device__ __forceinline__ bool line_may_hit_box(const float *xf, V3 om, V3 q) {
    const float sx = xf[12], sy = xf[13], sz = xf[14];
    const float ox = om.x * sx, oy = om.y * sy, oz = om.z * sz;
    const float ax = fabsf(q.x), ay = fabsf(q.y), az = fabsf(q.z);
    const float kRel = 3.0517578125e-05f;  // 2^-15
    const float a1 = ox * q.y, b1 = oy * q.x;
    const float a2 = oy * q.z, b2 = oz * q.y;
    const float a3 = oz * q.x, b3 = ox * q.z;
    const float r1 = sx * ay + sy * ax, r2 = sy * az + sz * ay, r3 = sz * ax + sx * az;
    const bool miss = fabsf(a1 - b1) > r1 + kRel * ((fabsf(a1) + fabsf(b1)) + r1) ||
                      fabsf(a2 - b2) > r2 + kRel * ((fabsf(a2) + fabsf(b2)) + r2) ||
                      fabsf(a3 - b3) > r3 + kRel * ((fabsf(a3) + fabsf(b3)) + r3);
    return !miss;
}

__device__ __forceinline__ bool intersect_obb(const float *xf, V3 o, V3 d, float &tEnterOut,
                                              float &tExitOut) {
    return intersect_obb_om(xf, to_model(xf, o), d, tEnterOut, tExitOut);
}

// camera.cpp:14-23 — pixel (px, py) is x + 0.5, y + 0.5.
__device__ __forceinline__ void generate_ray(const CamDev &cam, float px, float py, V3 &o, V3 &d) {
    const V3 dirCam = matvec(cam.kinv, mk3(px, py, 1.0f));
    const V3 v = matTvec(cam.R, dirCam);
    const float len = sqrtf(dot3(v, v));
    d = V3{v.x / len, v.y / len, v.z / len};
    o = mk3(cam.center[0], cam.center[1], cam.center[2]);
}

// math.h:170-179
__device__ __forceinline__ uint64_t hash_combine(uint64_t seed, uint64_t value) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull + value;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float hash_to_unit(uint64_t h) {
    return __ull2float_rn(h >> 11) * 1.1102230246251565e-16f; // real(1.0 / 2^53)
}

// ---------------------------------------------------------------------------------------
// glibc 2.39 expf, bit-exact port (std::exp(float) in window(), primitive.cpp:27).
// Algorithm: sysdeps/ieee754/flt-32/e_expf.c (ARM optimized-routines): k = round(x*32/ln2),
// 2^(k/32) from a 32-entry table, cubic correction, all in binary64, one final rounding.
// glibc's x86-64 ifunc selects the FMA build on FMA-capable hosts; the FMA and non-FMA
// builds agree on every float in [-104, 88] (checked exhaustively on the host), as does
// this port except at the two inputs patched below. The table lives in shared memory
// (lanes index it divergently).
#ifndef VPB_EXPTAB_SPLIT
#define VPB_EXPTAB_SPLIT 1
#endif
__constant__ unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

// The binary64 core, valid on [-0x1.9fe368p6, 0x1.62e42ep6] minus the two patched inputs.
__device__ __forceinline__ float expf_core(float x, const unsigned long long *tab) {
    const double InvLn2N = 0x1.71547652b82fep+0 * 32, Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
                 C2 = 0x1.62e42ff0c52d6p-1 / 32;
    const double z = __dmul_rn(InvLn2N, (double)x);
    double kd = __dadd_rn(z, Shift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, Shift);
    const double r = __dsub_rn(z, kd);
    // the table is staged as two 32-bit halves (load_exp_tab): two conflict-free LDS.32 instead
    // of an LDS.64 whose entries i and i + 16 share banks
#if VPB_EXPTAB_SPLIT
    const unsigned *tw = reinterpret_cast<const unsigned *>(tab);
    const unsigned j = (unsigned)(ki & 31);
    const unsigned long long t = (((unsigned long long)tw[32 + j] << 32) | tw[j]) + (ki << 47);
#else
    const unsigned long long t = tab[ki & 31] + (ki << 47);
#endif
    const double s = __longlong_as_double((long long)t);
    const double zz = __fma_rn(C0, r, C1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(C2, r, 1.0);
    y = __fma_rn(zz, r2, y);
    return __double2float_rn(__dmul_rn(y, s));
}

// Stages kExp2fTab into 32 shared u64 slots (64 words) as lo[32] then hi[32]; threads 0..31 of
// the block write it (a __syncthreads must follow before expf_core reads it).
__device__ __forceinline__ void load_exp_tab(unsigned long long *s_tab) {
    if (threadIdx.x < 32) {
        const unsigned long long v = kExp2fTab[threadIdx.x];
#if VPB_EXPTAB_SPLIT
        unsigned *w = reinterpret_cast<unsigned *>(s_tab);
        w[threadIdx.x] = (unsigned)v;
        w[32 + threadIdx.x] = (unsigned)(v >> 32);
#else
        s_tab[threadIdx.x] = v;
#endif
    }
}

__device__ __forceinline__ float expf_glibc(float x, const unsigned long long *tab) {
    if (!(x == x)) return x + x;
    if (x < -0x1.9fe368p6f) return 0.0f;
    if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
    if (x == -0x1.f8cbb2p+5f) return 0x1.f45326p-92f;
    if (x == 0x1.04845ep+5f) return 0x1.f93e38p+46f;
    return expf_core(x, tab);
}

// primitive.cpp:12-22
__device__ __forceinline__ float pow_even(float x, int beta) {
    float r = 1.0f, b = fabsf(x);
    int e = beta;
    while (e > 0) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}
__device__ __forceinline__ float pow8(float x) { // pow_even(x, 8): r = 1 * b^8 exactly
    const float b = fabsf(x);
    const float b2 = b * b;
    const float b4 = b2 * b2;
    return b4 * b4;
}
__device__ __forceinline__ float pow6(float x) { // pow_even(x, 6): r = (1 * b^2) * b^4
    const float b = fabsf(x);
    const float b2 = b * b;
    return b2 * (b2 * b2);
}

// primitive.cpp:25-28
__device__ __forceinline__ float window_value(V3 p, float alpha, int beta,
                                              const unsigned long long *tab) {
    if (alpha == 0.0f) return 1.0f;
    float s;
    if (beta == 8)
        s = (pow8(p.x) + pow8(p.y)) + pow8(p.z);
    else
        s = (pow_even(p.x, beta) + pow_even(p.y, beta)) + pow_even(p.z, beta);
    const float x = -alpha * s;
    // |p| <= 1 makes s a finite value in [0, 3], so for 0 < alpha <= 34.6 the argument lies in
    // [-103.8, 0]: no NaN, overflow or underflow cases; only the -63.1 patch can apply.
    if (alpha > 0.0f && alpha <= 34.6f) return x == -0x1.f8cbb2p+5f ? 0x1.f45326p-92f : expf_core(x, tab);
    return expf_glibc(x, tab);
}

// march.cpp:14-16 — cwiseMax(-1, cwiseMin(1, p)) with std::min/std::max semantics.
__device__ __forceinline__ float clamp_unit(float v) {
    const float lo = v < 1.0f ? v : 1.0f;
    return -1.0f < lo ? lo : -1.0f;
}

// One primitive-sample: march.cpp:64-69 with trilinearStencil (primitive.cpp:51-69),
// gatherChannel/cornerWeight (primitive.cpp:71-99) over the channel-interleaved float4
// payload (k, z, y, x, rgba), and window(). Each channel accumulates its 8 corners in the
// reference order (z, y, x loops, x fastest; weight (wx*wy)*wz, starting from 0).
//
// pbase is the primitive's first voxel (payload + k * M^3). MT > 0 makes the voxel count a compile-time constant: the stencil folds to constants and
// the eight corner loads become one address plus immediate offsets. Because
// trilinearStencil clamps lo to [0, M-2], the upper corner is always lo+1 for M >= 2
// (gatherChannel's min(lo+c, M-1) never bites); for M == 1 all corners are voxel 0.
#ifndef VPB_PAIRS
#define VPB_PAIRS 0
#endif
// Compile-time voxel counts (MT >= 2) gather from the x-pair payload layout (vpb_kernels.cu
// k_build_pairs): 4 x 256-bit loads per sample instead of 8 x 128-bit.
constexpr bool kPairGathers = VPB_PAIRS != 0;

__device__ __forceinline__ void ldg_pair(const float4 *p, float4 &a, float4 &b) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

template <int MT>
__device__ __forceinline__ void sample_primitive(const float4 *__restrict__ pbase, int m_rt,
                                                 const float *xf, V3 pw, float alpha,
                                                 int beta, const unsigned long long *tab,
                                                 float &sigma, float &r, float &g, float &b) {
    const int m = MT > 0 ? MT : m_rt;
    const V3 q = to_model(xf, pw);
    const V3 pm = mk3(clamp_unit(q.x), clamp_unit(q.y), clamp_unit(q.z));
    int lo[3];
    float fr[3];
    const float mf = (float)m;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float u = (comp(pm, a) + 1.0f) * 0.5f * mf - 0.5f;
        if (u <= 0.0f) u = 0.0f;
        else if (u >= (float)(m - 1)) u = (float)(m - 1);
        int i0 = (int)floorf(u);
        if (i0 > m - 2) i0 = (m - 2) > 0 ? (m - 2) : 0;
        lo[a] = i0;
        fr[a] = m > 1 ? u - (float)i0 : 0.0f;
    }
    float4 c000, c001, c010, c011, c100, c101, c110, c111;
    if (kPairGathers && MT >= 2) {
        // x-pair layout (build_pairs): entry (z, y, x) of the primitive holds voxels x and x+1,
        // 32 B aligned, so each (z, y) row of the stencil is ONE 256-bit load (LDG.256)
        constexpr int R = 2 * (MT - 1);  // float4s per row of pairs
        const float4 *p = pbase + (unsigned)(2 * ((lo[2] * MT + lo[1]) * (MT - 1) + lo[0]));
        ldg_pair(p, c000, c001);
        ldg_pair(p + R, c010, c011);
        ldg_pair(p + MT * R, c100, c101);
        ldg_pair(p + MT * R + R, c110, c111);
    } else if (MT >= 2) {  // immediate offsets
        const float4 *p = pbase + (unsigned)((lo[2] * m + lo[1]) * m + lo[0]);
        c000 = __ldg(p);
        c001 = __ldg(p + 1);
        c010 = __ldg(p + MT);
        c011 = __ldg(p + MT + 1);
        c100 = __ldg(p + MT * MT);
        c101 = __ldg(p + MT * MT + 1);
        c110 = __ldg(p + MT * MT + MT);
        c111 = __ldg(p + MT * MT + MT + 1);
    } else {
        const float4 *p = pbase + (unsigned)((lo[2] * m + lo[1]) * m + lo[0]);
        const int dx = m > 1 ? 1 : 0, dy = m > 1 ? m : 0, dz = m > 1 ? m * m : 0;
        c000 = __ldg(p);
        c001 = __ldg(p + dx);
        c010 = __ldg(p + dy);
        c011 = __ldg(p + dy + dx);
        c100 = __ldg(p + dz);
        c101 = __ldg(p + dz + dx);
        c110 = __ldg(p + dz + dy);
        c111 = __ldg(p + dz + dy + dx);
    }
    const float wx0 = 1.0f - fr[0], wx1 = fr[0];
    const float wy0 = 1.0f - fr[1], wy1 = fr[1];
    const float wz0 = 1.0f - fr[2], wz1 = fr[2];
    const float w00 = wx0 * wy0, w01 = wx1 * wy0, w10 = wx0 * wy1, w11 = wx1 * wy1;
    const float w000 = w00 * wz0, w001 = w01 * wz0, w010 = w10 * wz0, w011 = w11 * wz0;
    const float w100 = w00 * wz1, w101 = w01 * wz1, w110 = w10 * wz1, w111 = w11 * wz1;
#define VPB_GATHER(ch)                                                                        \
    (((((((0.0f + w000 * c000.ch) + w001 * c001.ch) + w010 * c010.ch) + w011 * c011.ch) +     \
        w100 * c100.ch) + w101 * c101.ch) + w110 * c110.ch) + w111 * c111.ch
    const float s_raw = VPB_GATHER(w);
    r = VPB_GATHER(x);
    g = VPB_GATHER(y);
    b = VPB_GATHER(z);
#undef VPB_GATHER
    sigma = s_raw * window_value(pm, alpha, beta, tab);
}

} // namespace vpb
