// vpb_compose.cu — Frame::composed() on the device (primitive.cpp:41-49, rotation.cpp:8-27):
// PrimitiveTransform records (tBase, rBase, sBase, deltaT, deltaR, deltaS) -> the resident
// 16-float AffineXf records the raymarch reads, without a host round trip. Bit-exact with the
// reference's binary32 host code: the same operation order as vpb_hostmath.hpp compose()
// (-fmad=false), and glibc 2.39 sinf / cosf restated below.
//
//   k_compose        one thread per primitive; optionally first writes Adam's updated deltas
//                    back into the records with the scale projection of losses.cpp:97-103
//   k_gather_deltas  the 9 deltas per primitive, contiguous (Adam's GradBuffer order)
//   k_pose36         backwardRay's pose data: rBase and rotationDerivative (rotation.cpp:30-38)
//   k_sincos         test hook: the sinf / cosf port over an array
#include <cuda_runtime.h>

#include <cstdint>

#include "vpb_device.cuh"
#include "vpb_kernels.h"

namespace vpb {

// ----------------------------------------------------------------------------------------
// glibc 2.39 sinf / cosf (sysdeps/ieee754/flt-32/s_sinf.c, s_cosf.c, sincosf.h; the ARM
// optimized-routines algorithm). The polynomials run in binary64 with fused multiply-adds, as
// in the FMA build glibc's ifunc selects on x86-64 hosts with FMA (where the reference runs),
// and round once to float. Table rows: c0 c1 s1 c2 s2 c3 s3 c4 (__sincosf_table; the second
// row negates the cosine coefficients). kInvPio4 holds 4/pi in 24 overlapping 32-bit windows
// (__inv_pio4). The C restatement is oracle/vp_oracle.c sc_eval, checked against libm on every
// float of [0, 120] and strided beyond; tests/test_gpu_train.py checks this port against libm.
__constant__ double kSinCosTab[2][8] = {
    {0x1p0, -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, 0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, 0x1.99343027bf8c3p-16},
    {-0x1p0, 0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, -0x1.99343027bf8c3p-16}};
__constant__ uint32_t kInvPio4[24] = {
    0xa2,       0xa2f9,     0xa2f983,   0xa2f9836e, 0xf9836e4e, 0x836e4e44, 0x6e4e4415, 0x4e441529,
    0x441529fc, 0x1529fc27, 0x29fc2757, 0xfc2757d1, 0x2757d1f5, 0x57d1f534, 0xd1f534dd, 0xf534ddc0,
    0x34ddc0db, 0xddc0db62, 0xc0db6295, 0xdb629599, 0x6295993c, 0x95993c43, 0x993c4390, 0x3c439041};

__device__ __forceinline__ uint32_t abstop12(float x) { return (__float_as_uint(x) >> 20) & 0x7ffu; }

// sinf_poly: n even -> the sine polynomial, odd -> the cosine polynomial
__device__ __forceinline__ float sc_poly(double x, double x2, int row, int n) {
    const double *c = kSinCosTab[row];
    if ((n & 1) == 0) {
        const double x3 = __dmul_rn(x, x2);
        const double s1 = fma(x2, c[6], c[4]);
        const double x7 = __dmul_rn(x3, x2);
        const double s = fma(x3, c[2], x);
        return __double2float_rn(fma(x7, s1, s));
    }
    const double x4 = __dmul_rn(x2, x2);
    const double c2 = fma(x2, c[7], c[5]);
    const double c1 = fma(x2, c[1], c[0]);
    const double x6 = __dmul_rn(x4, x2);
    const double cc = fma(x4, c[3], c1);
    return __double2float_rn(fma(x6, c2, cc));
}

// reduce_fast: |x| < 120, one multiply by 2/pi * 2^24 and a fused x - n * pi/2
__device__ __forceinline__ double sc_reduce_fast(double x, int &n) {
    const double r = __dmul_rn(x, 0x1.45f306dc9c883p+23);
    n = (__double2int_rz(r) + 0x800000) >> 24;
    return fma(-(double)n, 0x1.921fb54442d18p0, x);
}

// reduce_large: 4/pi with 192 bits, a 32x96 -> 128-bit product modulo 2^62
__device__ __forceinline__ double sc_reduce_large(uint32_t xi, int &n) {
    const uint32_t *arr = &kInvPio4[(xi >> 26) & 15];
    const int shift = (xi >> 23) & 7;
    xi = (xi & 0xffffffu) | 0x800000u;
    xi <<= shift;
    uint64_t res0 = (uint64_t)(uint32_t)(xi * arr[0]);
    const uint64_t res1 = (uint64_t)xi * arr[4];
    const uint64_t res2 = (uint64_t)xi * arr[8];
    res0 = (res2 >> 32) | (res0 << 32);
    res0 += res1;
    const uint64_t q = (res0 + (1ull << 61)) >> 62;
    res0 -= q << 62;
    n = (int)q;
    return __dmul_rn((double)(int64_t)res0, 0x1.921fb54442d18p-62);
}

__device__ float sincosf_glibc(float y, bool want_cos) {
    double x = y;
    int n = 0, row = 0;
    if (abstop12(y) < abstop12(0x1.921fb6p-1f)) {  // |y| < pi/4 (top-12-bit compare)
        const double x2 = __dmul_rn(x, x);
        if (abstop12(y) < abstop12(0x1p-12f)) return want_cos ? 1.0f : y;
        return sc_poly(x, x2, 0, want_cos ? 1 : 0);
    }
    if (abstop12(y) < abstop12(120.0f)) {
        x = sc_reduce_fast(x, n);
        const double s = ((n + 1) & 2) ? -1.0 : 1.0;  // sign[n & 3] = {1, -1, -1, 1}
        if (n & 2) row = 1;
        return sc_poly(__dmul_rn(x, s), __dmul_rn(x, x), row, want_cos ? n ^ 1 : n);
    }
    if (abstop12(y) < abstop12(__int_as_float(0x7f800000))) {
        const uint32_t xi = __float_as_uint(y);
        const int sgn = (int)(xi >> 31);
        x = sc_reduce_large(xi, n);
        const double s = ((n + sgn + 1) & 2) ? -1.0 : 1.0;
        if ((n + sgn) & 2) row = 1;
        return sc_poly(__dmul_rn(x, s), __dmul_rn(x, x), row, want_cos ? n ^ 1 : n);
    }
    return __fdiv_rn(y - y, y - y);  // inf / nan -> nan
}

// ----------------------------------------------------------------------------------------
// Column-major 3x3 (element (r, c) at m[3c + r]), math.h:71-124 operation order.
struct Mat3d {
    float m[9];
};

// Mat3 * Mat3, accumulating each element from zero with k in the middle (math.h:115-121)
__device__ __forceinline__ Mat3d mat_mul(const Mat3d &a, const Mat3d &o) {
    Mat3d r;
#pragma unroll
    for (int i = 0; i < 9; ++i) r.m[i] = 0.0f;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int i = 0; i < 3; ++i) r.m[c * 3 + i] = r.m[c * 3 + i] + a.m[k * 3 + i] * o.m[c * 3 + k];
    return r;
}

__device__ __forceinline__ Mat3d skew_dev(float x, float y, float z) {  // math.h:94-100
    Mat3d k;
    k.m[0] = 0.0f; k.m[1] = z;    k.m[2] = -y;
    k.m[3] = -z;   k.m[4] = 0.0f; k.m[5] = x;
    k.m[6] = y;    k.m[7] = -x;   k.m[8] = 0.0f;
    return k;
}

// rotationFromAxisAngle (rotation.cpp:8-27): Rodrigues, I + K a + K^2 b
__device__ __forceinline__ Mat3d rotation_from_axis_angle_dev(float vx, float vy, float vz) {
    Mat3d r;
    const float t2 = (vx * vx + vy * vy) + vz * vz;
#pragma unroll
    for (int i = 0; i < 9; ++i) r.m[i] = (i % 4 == 0) ? 1.0f : 0.0f;
    if (t2 == 0.0f) return r;
    const float theta = __fsqrt_rn(t2);
    float a, b;
    if (theta < 1e-4f) {
        a = 1.0f - __fdiv_rn(t2, 6.0f);
        b = 0.5f - __fdiv_rn(t2, 24.0f);
    } else {
        a = __fdiv_rn(sincosf_glibc(theta, false), theta);
        b = __fdiv_rn(1.0f - sincosf_glibc(theta, true), t2);
    }
    const Mat3d k = skew_dev(vx, vy, vz);
    const Mat3d kk = mat_mul(k, k);
#pragma unroll
    for (int i = 0; i < 9; ++i) r.m[i] = (r.m[i] + k.m[i] * a) + kk.m[i] * b;
    return r;
}

// rotationDerivative (rotation.cpp:30-38): dR(v)/dv_i, the vpb_hostmath.hpp operation order
__device__ Mat3d rotation_derivative_dev(float vx, float vy, float vz, int i) {
    const float t2 = (vx * vx + vy * vy) + vz * vz;
    const float ex = i == 0 ? 1.0f : 0.0f, ey = i == 1 ? 1.0f : 0.0f, ez = i == 2 ? 1.0f : 0.0f;
    if (t2 < 1e-14f) return skew_dev(ex, ey, ez);
    const Mat3d r = rotation_from_axis_angle_dev(vx, vy, vz);
    Mat3d imr;
#pragma unroll
    for (int q = 0; q < 9; ++q) imr.m[q] = ((q % 4 == 0) ? 1.0f : 0.0f) - r.m[q];
    // (I - R) e, math.h:122-124: (col0 * e.x + col1 * e.y) + col2 * e.z
    const float ux = (imr.m[0] * ex + imr.m[3] * ey) + imr.m[6] * ez;
    const float uy = (imr.m[1] * ex + imr.m[4] * ey) + imr.m[7] * ez;
    const float uz = (imr.m[2] * ex + imr.m[5] * ey) + imr.m[8] * ez;
    // cross(v, u), math.h:54-56
    const float wx = vy * uz - vz * uy, wy = vz * ux - vx * uz, wz = vx * uy - vy * ux;
    const Mat3d sv = skew_dev(vx, vy, vz), sw = skew_dev(wx, wy, wz);
    const float vi = i == 0 ? vx : (i == 1 ? vy : vz);
    const float s = __fdiv_rn(1.0f, t2);
    Mat3d c;
#pragma unroll
    for (int q = 0; q < 9; ++q) c.m[q] = (sv.m[q] * vi + sw.m[q]) * s;
    return mat_mul(c, r);
}

// backwardRay's per-primitive pose data: rBase[9], then dR(deltaR)/dv_0..2 (27 floats).
__global__ void k_pose36(const float *__restrict__ tr24, int n_prim, float *__restrict__ p36) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_prim) return;
    const float *t = tr24 + (size_t)k * 24;
    float *o = p36 + (size_t)k * 36;
#pragma unroll
    for (int i = 0; i < 9; ++i) o[i] = t[3 + i];
    for (int q = 0; q < 3; ++q) {
        const Mat3d d = rotation_derivative_dev(t[18], t[19], t[20], q);
#pragma unroll
        for (int i = 0; i < 9; ++i) o[9 + 9 * q + i] = d.m[i];
    }
}

cudaError_t launch_pose36(const float *tr24, int n_prim, float *p36, cudaStream_t st) {
    if (n_prim <= 0) return cudaSuccess;
    k_pose36<<<(n_prim + 127) / 128, 128, 0, st>>>(tr24, n_prim, p36);
    return cudaGetLastError();
}

// One primitive: [optional: deltas from Adam + the scale projection] then compose.
// tr24: tBase[3] rBase[9] sBase[3] deltaT[3] deltaR[3] deltaS[3].
__global__ void k_compose(float *__restrict__ tr24, const float *__restrict__ deltas, int n_prim,
                          float *__restrict__ xf16, int *__restrict__ bad, const int *__restrict__ skip) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_prim) return;
    if (skip && *skip) return;  // adamStep found a non-finite gradient: nothing is touched
    float t[24];
#pragma unroll
    for (int i = 0; i < 24; ++i) t[i] = tr24[(size_t)k * 24 + i];
    if (deltas) {  // adamStep's deltas, then the feasibility projection (losses.cpp:97-103)
        constexpr float kMinScale = 1e-4f;  // losses.h:61
#pragma unroll
        for (int i = 0; i < 9; ++i) t[15 + i] = deltas[(size_t)k * 9 + i];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float composed = t[12 + a] + t[21 + a];
            if (composed < kMinScale) t[21 + a] = kMinScale - t[12 + a];
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) tr24[(size_t)k * 24 + 15 + i] = t[15 + i];
    }
    const float sx = t[12] + t[21], sy = t[13] + t[22], sz = t[14] + t[23];
    if (sx <= 0.0f || sy <= 0.0f || sz <= 0.0f) atomicExch(bad, 1);  // primitive.cpp:44-45
    const Mat3d rd = rotation_from_axis_angle_dev(t[18], t[19], t[20]);
    Mat3d rb;
#pragma unroll
    for (int i = 0; i < 9; ++i) rb.m[i] = t[3 + i];
    const Mat3d rot = mat_mul(rd, rb);
    float *o = xf16 + (size_t)k * kXfStride;
    o[0] = t[0] + t[15];
    o[1] = t[1] + t[16];
    o[2] = t[2] + t[17];
#pragma unroll
    for (int i = 0; i < 9; ++i) o[3 + i] = rot.m[i];
    o[12] = sx;
    o[13] = sy;
    o[14] = sz;
    o[15] = 0.0f;
}

__global__ void k_gather_deltas(const float *__restrict__ tr24, int n_prim, float *__restrict__ deltas) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_prim * 9) return;
    deltas[i] = tr24[(size_t)(i / 9) * 24 + 15 + i % 9];
}

__global__ void k_sincos(const float *__restrict__ x, float *__restrict__ y, int64_t n, int want_cos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = sincosf_glibc(x[i], want_cos != 0);
}

cudaError_t launch_compose(float *tr24, const float *deltas, int n_prim, float *xf16, int *bad, cudaStream_t st,
                           const int *skip) {
    if (n_prim <= 0) return cudaSuccess;
    k_compose<<<(n_prim + 127) / 128, 128, 0, st>>>(tr24, deltas, n_prim, xf16, bad, skip);
    return cudaGetLastError();
}

cudaError_t launch_gather_deltas(const float *tr24, int n_prim, float *deltas, cudaStream_t st) {
    if (n_prim <= 0) return cudaSuccess;
    k_gather_deltas<<<(n_prim * 9 + 255) / 256, 256, 0, st>>>(tr24, n_prim, deltas);
    return cudaGetLastError();
}

cudaError_t launch_sincos(const float *x, float *y, int64_t n, bool want_cos, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    k_sincos<<<blocks, 256, 0, st>>>(x, y, n, want_cos ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace vpb
