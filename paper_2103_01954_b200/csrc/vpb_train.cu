// vpb_train.cu — the training-side rows of SURVEY.md §8(f): the evalLoss ray-batch driver
// (grad.cpp:197-251) and Adam with the feasibility projection (losses.cpp:70-104), both on
// the resident frame so a fit iteration keeps the payload on the device.
//
//   k_eval_rays        RaySample -> Ray: generateRay per sample camera (camera.cpp:14-23) and
//                      evalLoss's jitter hash (grad.cpp:222-225)
//   k_loss_adjoints    composite with the sample background, the photometric residual and the
//                      adjoints evalLoss hands to backwardRay (grad.cpp:228-247)
//   k_adam_check /     adamStep: non-finite gradient check, then the bias-corrected update
//   k_adam_update      over [payload | deltas] and the payload projection (>= 0); the
//                      payload lives channel-interleaved on the device
// Same arithmetic contract as the renderer (-fmad=false): element-wise results equal the
// reference's bit for bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "vpb_device.cuh"
#include "vpb_kernels.h"

namespace vpb {

__global__ void k_eval_rays(const CamDev *__restrict__ cams, int n_cams, const int *__restrict__ cam_index,
                            const float *__restrict__ pixel_xy, const int *__restrict__ pixel_id,
                            int64_t n, int jitter, unsigned long long seed, float *__restrict__ origins,
                            float *__restrict__ dirs, float *__restrict__ jit, int *__restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ci = cam_index[i];
    if (ci < 0 || ci >= n_cams) {
        atomicExch(bad, 1);
        return;
    }
    const CamDev cam = cams[ci];
    const float px = pixel_xy[2 * i], py = pixel_xy[2 * i + 1];
    if (px < 0.0f || py < 0.0f || px > (float)cam.width || py > (float)cam.height) atomicExch(bad, 2);
    V3 o, d;
    generate_ray(cam, px, py, o, d);
    origins[3 * i] = o.x;
    origins[3 * i + 1] = o.y;
    origins[3 * i + 2] = o.z;
    dirs[3 * i] = d.x;
    dirs[3 * i + 1] = d.y;
    dirs[3 * i + 2] = d.z;
    jit[i] = jitter ? hash_to_unit(hash_combine(seed, (uint64_t)(uint32_t)ci * 0x100000001b3ull +
                                                          (uint64_t)(uint32_t)pixel_id[i]))
                    : 0.5f;
}

// composited = rgb * a + bg * (1 - a); e = composited - target; aI = e * (2 lambda / n);
// aRgb = aI * a; aAlpha = dot(aI, rgb - bg)   (grad.cpp:227-247, losses.cpp:12-25)
__global__ void k_loss_adjoints(const float *__restrict__ rgb, const float *__restrict__ alpha,
                                const float *__restrict__ target, const float *__restrict__ bg,
                                int64_t n, float scale, float *__restrict__ composited,
                                float *__restrict__ resid, float *__restrict__ adj_rgb,
                                float *__restrict__ adj_alpha) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float a = alpha[i];
    const V3 c = mk3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
    const V3 b = mk3(bg[3 * i], bg[3 * i + 1], bg[3 * i + 2]);
    const V3 comp = c * a + b * (1.0f - a);
    const V3 e = comp - mk3(target[3 * i], target[3 * i + 1], target[3 * i + 2]);
    const V3 aI = e * scale;
    const V3 aRgb = aI * a;
    composited[3 * i] = comp.x;
    composited[3 * i + 1] = comp.y;
    composited[3 * i + 2] = comp.z;
    resid[3 * i] = e.x;
    resid[3 * i + 1] = e.y;
    resid[3 * i + 2] = e.z;
    adj_rgb[3 * i] = aRgb.x;
    adj_rgb[3 * i + 1] = aRgb.y;
    adj_rgb[3 * i + 2] = aRgb.z;
    adj_alpha[i] = dot3(aI, c - b);
}

__global__ void k_adam_check(const float *__restrict__ g, int64_t n, int *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(g[i])) atomicExch(bad, 1);
}
// The same over a 16-byte aligned gradient: four float4 loads in flight per thread per round,
// one flag store per thread that saw a non-finite value.
__global__ void __launch_bounds__(256) k_adam_check4(const float4 *__restrict__ g4, int64_t n4,
                                                     const float *__restrict__ tail, int n_tail,
                                                     int *__restrict__ bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool ok = true;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(g4 + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) ok &= isfinite(v[u].x) && isfinite(v[u].y) && isfinite(v[u].z) && isfinite(v[u].w);
    }
    for (; i < n4; i += stride) {
        const float4 v = __ldcs(g4 + i);
        ok &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
    if (blockIdx.x == 0 && (int)threadIdx.x < n_tail) ok &= isfinite(tail[threadIdx.x]);
    if (!ok) atomicExch(bad, 1);
}

// lr * (a / bc1) / (sqrt(b / bc2) + eps) (losses.cpp:88-90). Most parameters of a fit step
// have zero moments (voxels no ray touched), and a zero dividend sends the IEEE division down
// its slow path (FCHK flags it; ncu put half of the update's instructions there). A zero over a positive divisor is that zero with its sign, and sqrt(+-0) is
// +-0, so returning the operand itself gives the same bits; NaN, infinite and non-positive
// divisors still divide.
// An opaque copy: the compiler may not replace it by an operand it knows to be discarded.
__device__ __forceinline__ float opaque(float x) {
    float y;
    asm("mov.b32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float adam_quot(float a, float b, float lr, const AdamDev &c) {
    // The division runs speculatively under a select, so a zero operand is replaced by 1 (a
    // fast-path division whose result is discarded) through an opaque copy.
    const bool za = a == 0.0f && c.bc1 > 0.0f, zb = b == 0.0f && c.bc2 > 0.0f;
    const float qa = opaque(za ? 1.0f : a) / c.bc1, qb = opaque(zb ? 1.0f : b) / c.bc2;
    const float mHat = za ? a : qa, vHat = zb ? b : qb;
    const bool zv = vHat == 0.0f;
    const float rv = sqrtf(opaque(zv ? 1.0f : vHat));
    const float root = zv ? vHat : rv;
    const float num = lr * mHat, den = root + c.eps;
    const bool zn = num == 0.0f && den > 0.0f;
    const float q = opaque(zn ? 1.0f : num) / den;
    return zn ? num : q;
}

// One Adam step over [payload (planar GradBuffer order) | 9K deltas] (losses.cpp:81-92). The
// payload parameter with planar index (k, ch, v) lives at payload[k * m3 + v].ch
// (channel-interleaved), so a thread takes one voxel: its float4 is read and written once,
// and the four channels' gradient and moments are coalesced across the warp (consecutive v).
__device__ __forceinline__ float adam_one(const float *__restrict__ g, float *__restrict__ m1, float *__restrict__ m2,
                                          int64_t i, float lr, const AdamDev &c) {
    const float gi = g[i];
    const float a = c.beta1 * m1[i] + (1.0f - c.beta1) * gi;
    const float b = c.beta2 * m2[i] + (1.0f - c.beta2) * gi * gi;
    m1[i] = a;
    m2[i] = b;
    return adam_quot(a, b, lr, c);
}

__global__ void k_adam_update(const float *__restrict__ g, float *__restrict__ m1, float *__restrict__ m2,
                              float4 *__restrict__ payload, float *__restrict__ deltas, int64_t n_pay,
                              int64_t n, unsigned m3, AdamDev c, const int *__restrict__ skip) {
    if (*skip) return;  // the check pass found a non-finite gradient (losses.cpp:74-75)
    const int64_t n_vox = n_pay / 4, total = n_vox + (n - n_pay);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        if (q < n_vox) {
            const int64_t k = q / m3, v = q - k * m3;
            float4 pv = payload[q];
            float *pf = &pv.x;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                const float step = adam_one(g, m1, m2, (k * 4 + ch) * (int64_t)m3 + v, c.lr * 1.0f, c);
                float nv = pf[ch] - step;
                if (nv < 0.0f) nv = 0.0f;  // feasibility projection (losses.cpp:95-96)
                pf[ch] = nv;
            }
            payload[q] = pv;
        } else {
            const int64_t i = n_pay + (q - n_vox);
            float *p = deltas + (i - n_pay);
            *p = *p - adam_one(g, m1, m2, i, c.lr * c.lr_delta_scale, c);
        }
    }
}

// The same update with 16-byte accesses (m3 % 4 == 0, i.e. even M): a thread takes four
// consecutive voxels of one primitive, so each channel's gradient and moments are one float4
// each and the payload four consecutive float4 (64 contiguous bytes per lane). Every element
// goes through adam_one's arithmetic unchanged; only the access width differs. 629 -> 573 us
// at 67 M parameters (ncu); the pass is bound by the three IEEE divisions and the square root
// per parameter (~170 thread-instructions each, fixed-latency stalls), not by HBM.
__device__ __forceinline__ float adam_elem(float gi, float &m1, float &m2, float lr, const AdamDev &c) {
    const float a = c.beta1 * m1 + (1.0f - c.beta1) * gi;
    const float b = c.beta2 * m2 + (1.0f - c.beta2) * gi * gi;
    m1 = a;
    m2 = b;
    return adam_quot(a, b, lr, c);
}

#ifndef VPB_ADAM_PRELOAD
#define VPB_ADAM_PRELOAD 1  // 334 -> 301 us per update (0.92 of the HBM peak)
#endif
__global__ void __launch_bounds__(256)
k_adam_update4(const float *__restrict__ g, float *__restrict__ m1, float *__restrict__ m2,
               float4 *__restrict__ payload, float *__restrict__ deltas, int64_t n_pay, int64_t n, unsigned m3,
               AdamDev c, const int *__restrict__ skip) {
    if (*skip) return;  // the check pass found a non-finite gradient (losses.cpp:74-75)
    const int64_t q4 = m3 / 4, n_quads = n_pay / 16, total = n_quads + (n - n_pay);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        if (q < n_quads) {
            const int64_t k = q / q4, v0 = (q - k * q4) * 4;
            float4 *pp = payload + k * m3 + v0;
            float4 pv[4] = {pp[0], pp[1], pp[2], pp[3]};
#if VPB_ADAM_PRELOAD
            // every load of the quad in flight before the arithmetic (16 x 16 B per thread)
            float4 gq[4], aq[4], bq[4];
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                const int64_t i = (k * 4 + ch) * (int64_t)m3 + v0;
                gq[ch] = __ldcs(reinterpret_cast<const float4 *>(g + i));
                aq[ch] = __ldcs(reinterpret_cast<const float4 *>(m1 + i));
                bq[ch] = __ldcs(reinterpret_cast<const float4 *>(m2 + i));
            }
#endif
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                const int64_t i = (k * 4 + ch) * (int64_t)m3 + v0;
#if VPB_ADAM_PRELOAD
                const float4 g4 = gq[ch];
                float4 a4 = aq[ch];
                float4 b4 = bq[ch];
#else
                const float4 g4 = *reinterpret_cast<const float4 *>(g + i);
                float4 a4 = *reinterpret_cast<const float4 *>(m1 + i);
                float4 b4 = *reinterpret_cast<const float4 *>(m2 + i);
#endif
                const float gs[4] = {g4.x, g4.y, g4.z, g4.w};
                float *as = &a4.x, *bs = &b4.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float *pf = &pv[e].x;
                    float nv = pf[ch] - adam_elem(gs[e], as[e], bs[e], c.lr * 1.0f, c);
                    if (nv < 0.0f) nv = 0.0f;  // feasibility projection (losses.cpp:95-96)
                    pf[ch] = nv;
                }
                *reinterpret_cast<float4 *>(m1 + i) = a4;
                *reinterpret_cast<float4 *>(m2 + i) = b4;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) pp[e] = pv[e];
        } else {
            const int64_t i = n_pay + (q - n_quads);
            float *p = deltas + (i - n_pay);
            *p = *p - adam_one(g, m1, m2, i, c.lr * c.lr_delta_scale, c);
        }
    }
}

cudaError_t launch_eval_rays(const CamDev *cams, int n_cams, const int *cam_index, const float *pixel_xy,
                             const int *pixel_id, int64_t n, int jitter, unsigned long long seed,
                             float *origins, float *dirs, float *jit, int *bad, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_eval_rays<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(cams, n_cams, cam_index, pixel_xy, pixel_id, n,
                                                             jitter, seed, origins, dirs, jit, bad);
    return cudaGetLastError();
}

cudaError_t launch_loss_adjoints(const float *rgb, const float *alpha, const float *target, const float *bg,
                                 int64_t n, float scale, float *composited, float *resid, float *adj_rgb,
                                 float *adj_alpha, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_loss_adjoints<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(rgb, alpha, target, bg, n, scale, composited,
                                                                 resid, adj_rgb, adj_alpha);
    return cudaGetLastError();
}

cudaError_t launch_adam(const float *g, float *m1, float *m2, float4 *payload, float *deltas, int64_t n_pay,
                        int64_t n, unsigned m3, const AdamDev &c, int *bad, bool check, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    if (check) {
        if ((reinterpret_cast<uintptr_t>(g) & 15) == 0)
            k_adam_check4<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const float4 *>(g), n / 4, g + (n / 4) * 4,
                                                  (int)(n % 4), bad);
        else
            k_adam_check<<<blocks, 256, 0, st>>>(g, n, bad);
    } else if (m3 % 4 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
        // 16-byte gradient loads: only for an aligned caller pointer (a view at an offset into a
        // flat buffer may be 4-byte aligned; a misaligned LDG.128 would kill the context)
        const int64_t items = n_pay / 16 + (n - n_pay);
        const unsigned b4 = (unsigned)((items + 255) / 256 < 148 * 8 ? (items + 255) / 256 : 148 * 8);
        k_adam_update4<<<b4, 256, 0, st>>>(g, m1, m2, payload, deltas, n_pay, n, m3, c, bad);
    } else {
        k_adam_update<<<blocks, 256, 0, st>>>(g, m1, m2, payload, deltas, n_pay, n, m3, c, bad);
    }
    return cudaGetLastError();
}

}  // namespace vpb
