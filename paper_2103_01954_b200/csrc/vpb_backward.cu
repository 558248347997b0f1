// vpb_backward.cu — K6, the backward pass: backwardRay (grad.cpp:34-195) for a batch of rays.
//
// backwardRay per ray: (1) the ray's sorted segment list (intersect, lbvh.cpp:207-234) and
// (2) march()'s bookkeeping the adjoints need (lastStep, saturated, satTPrev, satSigmaSum,
// satRgbWeighted; march.h:22-33) come from the forward march of the same rays
// (k_march_rays_warp keeps them); (3) the adjoint walk over steps 0..lastStep (grad.cpp:66-164):
// per primitive-sample the colour/opacity adjoints, the payload scatter over 8 corners x 4
// channels, the spatial gradient through the stencil and the fade window, and the pose
// Jacobians (deltaT, deltaS, deltaR via rotationDerivative); (4) the t_min anchor chain onto the
// first-hit primitive (grad.cpp:166-194).
//
// Paths: batches of >= 8,192 rays run K6a-c, passes over primitive-samples (k_bwd_plan,
// k_bwd_scan_*, k_bwd_records, k_bwd_pairs, k_bwd_fold); smaller batches, and rays that find no
// room in the pair arrays, the warp-per-ray walk (k_backward_rays_warp); rays the forward could
// not keep a list for, the per-thread walks (k_backward_rays_list / _huge).
// Every per-sample value is computed with the reference's operation order (same bits), and so
// is gTmin; the global sums use device reductions, so only their summation order differs from
// the reference's sequential loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "vpb_device.cuh"
#include "vpb_kernels.h"
#include "vpb_march.cuh"

namespace vpb {

// Lattice walk shared by the replay and the adjoint pass (the stepping of march.cpp:27-58:
// admission, retirement, gap skip, window refill). F::step_begin(i, ts, pw), F::prim(k, c),
// F::step_end(i) -> bool stop. Returns 0, or 1 when the window overflowed, 2 on a runaway.
template <int CAP, class Cands, class Win, class F>
__device__ int walk_steps(const Cands &cands, const Win &w, int cnt, bool more, V3 o, V3 d,
                          int2 px, float jit, float dt, long long i_end, F &f) {
    if (cnt == 0) return 0;
    const float t0 = w.E(0);
    int nxt = 0, lo = 0;
    for (long long i = 0; i <= i_end; ++i) {
        if (i > (1ll << 40)) return 2;
        const float ts = t0 + (__ll2float_rn(i) + jit) * dt;
        for (;;) {
            while (nxt < cnt && w.E(nxt) <= ts) ++nxt;
            if (nxt < cnt || !more) break;
            const float lastE = w.E(cnt - 1);
            const int lastP = cands.prim(w.C(cnt - 1));
            int live = 0;
            for (int q = 0; q < nxt; ++q) {
                if (w.X(q) > ts) {
                    if (live != q) {
                        w.E(live) = w.E(q);
                        w.X(live) = w.X(q);
                        w.C(live) = w.C(q);
                    }
                    ++live;
                }
            }
            if (live == CAP) return 1;
            cnt = live;
            nxt = live;
            lo = 0;
            more = false;
            window_scan<CAP>(w, cands, cnt, more, o, d, px, false, lastE, lastP);
        }
        while (lo < nxt && w.X(lo) <= ts) ++lo;
        bool any = false;
        for (int j = lo; j < nxt; ++j)
            if (w.X(j) > ts) {
                any = true;
                break;
            }
        if (!any) {
            if (nxt >= cnt) break;
            const float tNext = w.E(nxt);
            const long long skipTo = (long long)ceil((double)((tNext - t0) / dt) - (double)jit);
            if (skipTo > i + 1) i = skipTo - 1;
            continue;
        }
        f.step_begin(i, ts, o + d * ts);
        for (int j = lo; j < nxt; ++j)
            if (w.X(j) > ts) f.prim(cands.prim(w.C(j)), w.C(j));
        if (f.step_end(i)) break;
    }
    return 0;
}

// Everything one primitive-sample exposes to the adjoints (PrimSample, grad.cpp:16-25).
struct PrimEval {
    V3 pm;
    bool cube[3];
    int lo[3];
    float fr[3];
    bool clamped[3];
    float sigmaRaw, win;
    V3 rgb;
    // stencilRgbGradient sums (primitive.cpp:101-127) per channel (rgb, sigma) before the
    // 0.5*M scale and the clamped-axis zeroing
    float sgx[4], sgy[4], sgz[4];
};

// The sample's trilinear stencil (primitive.cpp:51-99) and, in the same pass over the 8
// corners, the four channels' stencil-gradient sums: a corner's value is used as soon as it
// arrives and no corner stays live in registers. Each sum runs over the corners in the
// reference's order with the reference's products ((wx*wy)*wz, ((dx*wy)*wz)*v), so the bits
// are the reference's.
__device__ __forceinline__ void eval_primitive(const float4 *__restrict__ pbase, int m,
                                               const float *xf, V3 pw, float alpha, int beta,
                                               const unsigned long long *tab, PrimEval &e) {
    const V3 raw = to_model(xf, pw);
#pragma unroll
    for (int a = 0; a < 3; ++a) e.cube[a] = comp(raw, a) <= -1.0f || comp(raw, a) >= 1.0f;
    e.pm = mk3(clamp_unit(raw.x), clamp_unit(raw.y), clamp_unit(raw.z));
    const float mf = (float)m;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float u = (comp(e.pm, a) + 1.0f) * 0.5f * mf - 0.5f;
        e.clamped[a] = false;
        if (u <= 0.0f) {
            u = 0.0f;
            e.clamped[a] = true;
        } else if (u >= (float)(m - 1)) {
            u = (float)(m - 1);
            e.clamped[a] = true;
        }
        int i0 = (int)floorf(u);
        if (i0 > m - 2) i0 = (m - 2) > 0 ? (m - 2) : 0;
        e.lo[a] = i0;
        e.fr[a] = m > 1 ? u - (float)i0 : 0.0f;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) e.sgx[ch] = e.sgy[ch] = e.sgz[ch] = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
        const int z = min(e.lo[2] + cz, m - 1), y = min(e.lo[1] + cy, m - 1), x = min(e.lo[0] + cx, m - 1);
        const float4 c = __ldg(pbase + (z * m + y) * m + x);
        const float wx = cx ? e.fr[0] : 1.0f - e.fr[0];
        const float wy = cy ? e.fr[1] : 1.0f - e.fr[1];
        const float wz = cz ? e.fr[2] : 1.0f - e.fr[2];
        const float wgt = wx * wy * wz;
        acc[0] += wgt * c.x;
        acc[1] += wgt * c.y;
        acc[2] += wgt * c.z;
        acc[3] += wgt * c.w;
        const float a0 = (cx ? 1.0f : -1.0f) * wy * wz;
        const float a1 = wx * (cy ? 1.0f : -1.0f) * wz;
        const float a2 = wx * wy * (cz ? 1.0f : -1.0f);
        const float v[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            e.sgx[ch] += a0 * v[ch];
            e.sgy[ch] += a1 * v[ch];
            e.sgz[ch] += a2 * v[ch];
        }
    }
    e.rgb = mk3(acc[0], acc[1], acc[2]);
    e.sigmaRaw = acc[3];
    e.win = window_value(e.pm, alpha, beta, tab);
}


// windowGradient (primitive.cpp:30-39)
__device__ __forceinline__ V3 window_gradient(V3 p, float alpha, int beta, float wv) {
    if (alpha == 0.0f) return mk3(0.f, 0.f, 0.f);
    const float c = -alpha * (float)beta * wv;
    if (beta == 8)  // pow_even(x, 6) multiplies out to b^2 * b^4 (same products, same bits)
        return mk3(c * (pow6(p.x) * p.x), c * (pow6(p.y) * p.y), c * (pow6(p.z) * p.z));
    return mk3(c * (pow_even(p.x, beta - 2) * p.x), c * (pow_even(p.y, beta - 2) * p.y),
               c * (pow_even(p.z, beta - 2) * p.z));
}

// Step 2: bit-exact replay of march() keeping the backward bookkeeping.
template <class Cands>
struct FwdReplay {
    const Cands &cands;
    const MarchDev &mp;
    const unsigned long long *tab;
    float transmittance = 0.f, sigmaSum = 0.f, rw = 0.f, gw = 0.f, bw = 0.f;
    V3 pw;
    long long lastStep = -1;
    bool saturated = false;
    float satTPrev = 0.f, satSigmaSum = 0.f, satR = 0.f, satG = 0.f, satB = 0.f;
    __device__ FwdReplay(const Cands &c, const MarchDev &m, const unsigned long long *t)
        : cands(c), mp(m), tab(t) {}
    __device__ void step_begin(long long, float, V3 p) {
        pw = p;
        sigmaSum = rw = gw = bw = 0.f;
    }
    __device__ void prim(int k, int c) {
        float sg, r, g, b;
        sample_primitive<0>(cands.base(c), mp.m, cands.xf(c), pw, mp.alpha, mp.beta, tab, sg, r, g, b);
        sigmaSum += sg;
        rw += r * sg;
        gw += g * sg;
        bw += b * sg;
    }
    __device__ bool step_end(long long i) {
        lastStep = i;
        const float dT = sigmaSum * mp.dt;
        if (transmittance + dT >= 1.0f) {
            satTPrev = transmittance;
            satSigmaSum = sigmaSum;
            satR = rw;
            satG = gw;
            satB = bw;
            transmittance = 1.0f;
            saturated = true;
            return true;
        }
        transmittance += dT;
        return transmittance > 1.0f - mp.eps;
    }
};

__device__ __forceinline__ void red_add(float *p, float v) { atomicAdd(p, v); }

// One corner's payload gradient (rgb, sigma) of primitive k at voxel v. Planar GradBuffer
// (params.h:12-27): four scalar reductions, one per channel plane. With VPB_BWD_V4 the device
// gradient is channel-interleaved like the payload (k, z, y, x, c) and the corner is ONE
// 16-byte vector reduction (red.global.add.v4.f32); vp_backward_rays transposes it to the
// planar layout at the C-ABI.
__device__ __forceinline__ void scatter_payload(const BwdDev &bd, int k, size_t m3, size_t v, float r, float g,
                                                float b, float s) {
    if (bd.g_pay4) {
        float *p = bd.g_pay4 + 4 * ((size_t)k * m3 + v);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(r), "f"(g), "f"(b), "f"(s)
                     : "memory");
        return;
    }
    float *gk = bd.g_pay + (size_t)k * 4 * m3;
    red_add(gk + v, r);
    red_add(gk + m3 + v, g);
    red_add(gk + 2 * m3 + v, b);
    red_add(gk + 3 * m3 + v, s);
}

// One primitive-sample's adjoint (grad.cpp:96-161): the colour/opacity adjoints, the payload
// scatter over the 8 corners, the spatial gradient through the stencil and the fade window,
// and the pose terms: rotG = R (gP ./ s) (deltaT gets -rotG, gPWorldStep +rotG), the rotation
// term (deltaR) and the scale term (deltaS). Returns false when gP == 0 (no pose terms).
template <class Cands>
__device__ __forceinline__ bool sample_adjoint(const Cands &cands, const MarchDev &mp, const unsigned long long *tab,
                                               const FwdReplay<Cands> &fwd, const BwdDev &bd, V3 aRgb, float aAlpha,
                                               bool satStep, int k, int c, V3 pw, V3 &rotG, V3 &rTerm, V3 &sTerm) {
    const int m = mp.m;
    const float *xf = cands.xf(c);
    PrimEval e;
    eval_primitive(cands.base(c), m, xf, pw, mp.alpha, mp.beta, tab, e);
    const float dt = mp.dt;
    const float sigmaW = e.sigmaRaw * e.win;
    V3 gRgb;
    float gSigmaW;
    if (satStep) {  // grad.cpp:104-108 (rgbWeighted of this step == satRgbWeighted)
        const float budget = 1.0f - fwd.satTPrev;
        const float inv = 1.0f / fwd.satSigmaSum;
        gRgb = aRgb * (sigmaW * budget * inv);
        const V3 diff = e.rgb * fwd.satSigmaSum - mk3(fwd.satR, fwd.satG, fwd.satB);
        gSigmaW = dot3(aRgb, diff) * budget * inv * inv;
    } else {  // grad.cpp:109-118
        gRgb = aRgb * (sigmaW * dt);
        gSigmaW = dot3(aRgb, e.rgb) * dt;
        if (fwd.saturated)
            gSigmaW -= dot3(aRgb, mk3(fwd.satR, fwd.satG, fwd.satB)) / fwd.satSigmaSum * dt;
        else
            gSigmaW += aAlpha * dt;
    }
    // payload scatter (grad.cpp:121-134): corner weights in the reference's product order
    const size_t m3 = (size_t)m * m * m;
    const float gsw = gSigmaW * e.win;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
        const float wx = cx ? e.fr[0] : 1.0f - e.fr[0];
        const float wy = cy ? e.fr[1] : 1.0f - e.fr[1];
        const float wz = cz ? e.fr[2] : 1.0f - e.fr[2];
        const float wgt = wx * wy * wz;
        if (wgt == 0.0f) continue;
        const int z = min(e.lo[2] + cz, m - 1), y = min(e.lo[1] + cy, m - 1), x = min(e.lo[0] + cx, m - 1);
        scatter_payload(bd, k, m3, ((size_t)z * m + y) * m + x, gRgb.x * wgt, gRgb.y * wgt, gRgb.z * wgt,
                        gsw * wgt);
    }
    V3 sgrad[4];
    const float sh = 0.5f * (float)m;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
        sgrad[ch] = m == 1 ? mk3(0.f, 0.f, 0.f)
                           : mk3(e.clamped[0] ? 0.f : e.sgx[ch] * sh, e.clamped[1] ? 0.f : e.sgy[ch] * sh,
                                 e.clamped[2] ? 0.f : e.sgz[ch] * sh);
    // spatial gradient (grad.cpp:136-145)
    const V3 gradW = window_gradient(e.pm, mp.alpha, mp.beta, e.win);
    V3 gP = (sgrad[3] * e.win + gradW * e.sigmaRaw) * gSigmaW;
    gP = gP + sgrad[0] * gRgb.x;
    gP = gP + sgrad[1] * gRgb.y;
    gP = gP + sgrad[2] * gRgb.z;
    if (e.cube[0]) gP.x = 0.f;
    if (e.cube[1]) gP.y = 0.f;
    if (e.cube[2]) gP.z = 0.f;
    if (gP.x == 0.f && gP.y == 0.f && gP.z == 0.f) return false;
    // pose Jacobians (grad.cpp:147-161)
    const V3 gOverS = mk3(gP.x / xf[12], gP.y / xf[13], gP.z / xf[14]);
    rotG = matvec(xf + 3, gOverS);
    sTerm = mk3(-gP.x * e.pm.x / xf[12], -gP.y * e.pm.y / xf[13], -gP.z * e.pm.z / xf[14]);
    const V3 u = pw - mk3(xf[0], xf[1], xf[2]);
    const float *pose = bd.pose36 + 36 * (size_t)k;  // rBase[9], dR/dv_i [3][9]
    const V3 v = matvec(pose, gOverS);
    rTerm = mk3(dot3(matvec(pose + 9, v), u), dot3(matvec(pose + 18, v), u), dot3(matvec(pose + 27, v), u));
    return true;
}

#ifndef VPB_BWD_WARP_AGG
#define VPB_BWD_WARP_AGG 1  // warp-aggregated pose atomics at the end of each ray
#endif

// Step 3: the adjoint walk.
template <class Cands>
struct BwdWalk {
    const Cands &cands;
    const MarchDev &mp;
    const unsigned long long *tab;
    const FwdReplay<Cands> &fwd;
    const BwdDev &bd;
    V3 d, aRgb;
    float aAlpha;
    float ts = 0.f;
    V3 pw, gPWorldStep;
    float gTmin = 0.f;
    bool satStep = false;
    int cur = -1;      // primitive whose pose gradients are being summed in registers
    int last_touched = -1;
    float acc[9];      // deltaT[3] deltaR[3] deltaS[3]
    __device__ BwdWalk(const Cands &c, const MarchDev &m, const unsigned long long *t,
                       const FwdReplay<Cands> &f, const BwdDev &b, V3 dir, V3 ar, float aa)
        : cands(c), mp(m), tab(t), fwd(f), bd(b), d(dir), aRgb(ar), aAlpha(aa) {
        for (float &v : acc) v = 0.f;
    }
    // End of a warp-per-ray walk (all 32 lanes converged): lanes summing the same primitive
    // are reduced with a masked butterfly, one group at a time, and the group's lowest lane
    // issues the 9 pose atomics (warp-aggregated atomics).
    __device__ void flush_warp(int lane) {
#if VPB_BWD_WARP_AGG
        unsigned left = __ballot_sync(0xffffffffu, cur >= 0);
        while (left) {
            const int lead = __ffs(left) - 1;
            const int k = __shfl_sync(0xffffffffu, cur, lead);
            const unsigned grp = __ballot_sync(0xffffffffu, cur == k);
            const bool in = (grp >> lane) & 1u;
            float v[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) v[q] = in ? acc[q] : 0.f;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int q = 0; q < 9; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
            if (lane == lead) {
                float *g = bd.g_pose + 9 * (size_t)k;
                for (int q = 0; q < 9; ++q)
                    if (v[q] != 0.f) red_add(g + q, v[q]);
            }
            left &= ~grp;
        }
        cur = -1;
        for (float &x : acc) x = 0.f;
#else
        (void)lane;
        flush();
#endif
    }
    __device__ void flush() {
        if (cur < 0) return;
        float *g = bd.g_pose + 9 * (size_t)cur;
        for (int q = 0; q < 9; ++q)
            if (acc[q] != 0.f) red_add(g + q, acc[q]);
        for (float &v : acc) v = 0.f;
    }
    __device__ void pose_add(int k, int off, V3 v) {
        if (k != cur) {
            flush();
            cur = k;
        }
        acc[off] += v.x;
        acc[off + 1] += v.y;
        acc[off + 2] += v.z;
    }
    __device__ void step_begin(long long i, float t, V3 p) {
        ts = t;
        pw = p;
        gPWorldStep = mk3(0.f, 0.f, 0.f);
        satStep = fwd.saturated && i == fwd.lastStep;
    }
    __device__ void prim(int k, int c) {
        if (bd.touched && k != last_touched) {  // primitives with gradient entries (the transpose's set)
            bd.touched[k] = 1u;
            last_touched = k;
        }
        V3 rotG, rTerm, sTerm;
        if (!sample_adjoint(cands, mp, tab, fwd, bd, aRgb, aAlpha, satStep, k, c, pw, rotG, rTerm, sTerm)) return;
        pose_add(k, 0, mk3(-rotG.x, -rotG.y, -rotG.z));
        pose_add(k, 6, sTerm);
        pose_add(k, 3, rTerm);
        gPWorldStep = gPWorldStep + rotG;
    }
    __device__ bool step_end(long long) {
        gTmin += dot3(gPWorldStep, d);
        return false;
    }
};

// lbvh.cpp:177-205 keeping the entry face
__device__ __forceinline__ bool intersect_face(const float *xf, V3 o, V3 d, int &axis, int &sign,
                                               bool &clamped) {
    const V3 om = to_model(xf, o);
    const V3 q = matTvec(xf + 3, d);
    const V3 dm = V3{q.x / xf[12], q.y / xf[13], q.z / xf[14]};
    float tEnter = -3.402823466e+38f, tExit = 3.402823466e+38f;
    axis = -1;
    sign = 0;
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
        if (t1 > tEnter) {
            tEnter = t1;
            axis = a;
            sign = (int)cNear;
        }
        tExit = t2 < tExit ? t2 : tExit;
    }
    clamped = tEnter < 0.0f;
    if (clamped) tEnter = 0.0f;
    return !(tEnter >= tExit || tExit <= 0.0f);
}

// The t_min anchor chain (grad.cpp:166-194): the first hit's entry depends on the pose of the
// first primitive (k0) through its entry face. Returns false when it contributes nothing;
// otherwise the deltaT, deltaR and deltaS terms of k0.
__device__ __forceinline__ bool anchor_terms(const float *xf, const float *pose, float tMin, float gTmin, V3 o,
                                             V3 d, V3 &gT3, V3 &gR3, V3 &gS3) {
    if (gTmin == 0.f) return false;
    int axis, sign;
    bool clamped;
    if (!intersect_face(xf, o, d, axis, sign, clamped) || clamped) return false;
    const int j = axis;
    const float c = (float)sign;
    const V3 q = mk3(xf[3 + 3 * j], xf[4 + 3 * j], xf[5 + 3 * j]);
    const float qd = dot3(q, d);
    if (qd == 0.0f) return false;
    const float gT = gTmin;
    gT3 = q * (gT / qd);
    gS3 = mk3(0.f, 0.f, 0.f);
    const float gsj = gT * c / qd;
    if (j == 0) gS3.x = gsj;
    else if (j == 1) gS3.y = gsj;
    else gS3.z = gsj;
    const V3 toT = mk3(xf[0], xf[1], xf[2]) - o;
    const V3 rj = mk3(pose[3 * j], pose[3 * j + 1], pose[3 * j + 2]);
    float gR[3];
#pragma unroll
    for (int ii = 0; ii < 3; ++ii) {
        const V3 qp = matvec(pose + 9 + 9 * ii, rj);
        gR[ii] = gT * (dot3(qp, toT) - tMin * dot3(qp, d)) / qd;
    }
    gR3 = mk3(gR[0], gR[1], gR[2]);
    return true;
}

template <class Cands>
__device__ void anchor_chain(BwdWalk<Cands> &bw, const Cands &cands, const BwdDev &bd, int k0, float tMin,
                             float gTmin, V3 o, V3 d) {
    V3 gT3, gR3, gS3;
    if (!anchor_terms(cands.xf(k0), bd.pose36 + 36 * (size_t)k0, tMin, gTmin, o, d, gT3, gR3, gS3)) return;
    bw.pose_add(k0, 0, gT3);
    bw.pose_add(k0, 6, gS3);
    bw.pose_add(k0, 3, gR3);
}

__device__ __forceinline__ void load_fwd_state(FwdReplay<BvhCands> &fwd, const float *s) {
    fwd.lastStep = __float_as_int(s[0]);
    fwd.saturated = __float_as_int(s[1]) != 0;
    fwd.satTPrev = s[2];
    fwd.satSigmaSum = s[3];
    fwd.satR = s[4];
    fwd.satG = s[5];
    fwd.satB = s[6];
}

// backwardRay of one ray by one thread with a kFallbackCap-entry window; returns 0, or 1 / 2
// (window overflow / runaway walk).
template <int CAP, class Win>
__device__ int backward_one_ray(const BvhCands &cands, const Win &w, const MarchDev &mp,
                                const unsigned long long *tab, const BwdDev &bd, V3 o, V3 d, float jit,
                                int64_t r) {
    const int2 px = make_int2(0, 0);
    int cnt = 0;
    bool more = false;
    window_scan<CAP>(w, cands, cnt, more, o, d, px, true, 0.f, 0);
    if (cnt == 0) return 0;
    const int k0 = cands.prim(w.C(0));
    const float tMin = w.E(0);
    FwdReplay<BvhCands> fwd(cands, mp, tab);
    int st = 0;
    const bool have_fwd = bd.fwd_state != nullptr;
    if (have_fwd)  // the forward pass of this very ray recorded the replay's results
        load_fwd_state(fwd, bd.fwd_state + 8 * r);
    else
        st = walk_steps<CAP>(cands, w, cnt, more, o, d, px, jit, mp.dt, 1ll << 62, fwd);
    if (st != 0 || fwd.lastStep < 0) return st;
    const V3 aRgb = mk3(bd.adj_rgb[3 * r], bd.adj_rgb[3 * r + 1], bd.adj_rgb[3 * r + 2]);
    BwdWalk<BvhCands> bw(cands, mp, tab, fwd, bd, d, aRgb, bd.adj_alpha[r]);
    if (!have_fwd) {  // the replay consumed the window
        cnt = 0;
        more = false;
        window_scan<CAP>(w, cands, cnt, more, o, d, px, true, 0.f, 0);
    }
    st = walk_steps<CAP>(cands, w, cnt, more, o, d, px, jit, mp.dt, fwd.lastStep, bw);
    if (st == 0) anchor_chain(bw, cands, bd, k0, tMin, bw.gTmin, o, d);
    bw.flush();
    return st;
}

// The rays whose segment list the forward could not keep (more than kRaySegs segments; none
// at the benchmark configs): one thread per ray with a kFallbackCap-entry global window,
// rebuilding the list through the BVH. The warp kernel lists them (ray_list, ctr->bwd_long).
__global__ void __launch_bounds__(32, 12)
k_backward_rays_list(MarchDev mp, const float *__restrict__ xf_g, int n_prim,
                     const float4 *__restrict__ payload, RaysDev rays, BwdDev bd, DevCounters *ctr,
                     const int *__restrict__ ray_list, int list_cap, float *se, float *sx, int *sc) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    const int n = (int)min((unsigned)list_cap, ctr->bwd_long);
    if (n == 0) return;  // the common case: every list fit (no table load, no barrier)
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const Window<int> w{se, sx, sc, nthreads, gtid};
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    for (int q = gtid; q < n; q += nthreads) {
        const int64_t r = ray_list[q];
        const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
        const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        const int st = backward_one_ray<kFallbackCap>(cands, w, mp, s_tab, bd, o, d, jit, r);
        if (st == 1) atomicAdd(&ctr->fallback_fail, 1);
        if (st == 2) atomicAdd(&ctr->numeric_fail, 1ull);
    }
}

// The rays whose forward needed the last-resort pass (more than kFallbackCap live segments:
// forward state[7] == -2): the per-thread walk with kHugeCap-entry windows.
__global__ void __launch_bounds__(32)
k_backward_rays_huge(MarchDev mp, const float *__restrict__ xf_g, int n_prim,
                     const float4 *__restrict__ payload, RaysDev rays, BwdDev bd, DevCounters *ctr,
                     const int *__restrict__ ray_list, int list_cap, float *se, float *sx, int *sc) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    const int n = (int)min((unsigned)list_cap, ctr->bwd_huge);
    if (n == 0) return;
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const int nthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const Window<int> w{se, sx, sc, nthreads, gtid};
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    for (int q = gtid; q < n; q += nthreads) {
        const int64_t r = ray_list[q];
        const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
        const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        const int st = backward_one_ray<kHugeCap>(cands, w, mp, s_tab, bd, o, d, jit, r);
        if (st == 1) atomicAdd(&ctr->fallback_fail, 1);
        if (st == 2) atomicAdd(&ctr->numeric_fail, 1ull);
    }
}

// backwardRay for small batches with the forward's per-ray state (evalLoss): one warp per ray,
// 32 lattice steps at a time. The warp builds the ray's sorted segment list
// (warp_segment_list); each lane takes
// one step of the visited sequence (the march_warp replay of the lattice walk) and runs the
// adjoint of its active primitives (the payload scatter and pose sums are atomics, as in the
// per-thread walk); gTmin, the only sequential sum, is accumulated over the chunk's steps in
// step order. Rays with more than kWarpListBwd segments take the per-thread path.
constexpr int kWarpListBwd = kRaySegs;
// 3 CTAs/SM (162 registers, no spills). 4 CTAs (128 registers, 28 B of spills) and 5 (96,
// 180 B) measured 2.05 and 2.14 ms for the 65,536-ray row against 2.03: more resident warps
// do not help this walk (K6, tools/bwd_sweep.sh)
#ifndef VPB_BWD_PAIRS
#define VPB_BWD_PAIRS 1  // deal primitive-samples (not steps) out to the lanes
#endif
#ifndef VPB_TR_GRID
#define VPB_TR_GRID 64  // CTAs per SM of k_grad_transpose4 (16 -> 64: +0.8 %)
#endif
#ifndef VPB_BWD_RAY_GRID
#define VPB_BWD_RAY_GRID 96  // CTAs per SM of the warp-per-ray passes (K6a walk, records; 16 -> 64: +1.5 %, 96: +0.5 %)
#endif
#ifndef VPB_BWD_PAIR_GRID
#define VPB_BWD_PAIR_GRID 24  // CTAs per SM of K6b (samples grid-strided; 8: 57.0M, 20-24: 62.2M, 32: 61.4M, 48: 60.3M)
#endif
#ifndef VPB_BWD_PAIRS_NT
#define VPB_BWD_PAIRS_NT 256  // threads per CTA of K6b
#endif
#ifndef VPB_BWD_PAIRS_MINB
#define VPB_BWD_PAIRS_MINB 3  // 80 registers (12 B of spills): 1.50 vs 1.52 ms for the backward row
#endif
#ifndef VPB_BWD_WARP_MINB
#define VPB_BWD_WARP_MINB 3
#endif
__global__ void __launch_bounds__(128, VPB_BWD_WARP_MINB)
k_backward_rays_warp(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
                     RaysDev rays, int64_t n_rays, BwdDev bd, DevCounters *ctr, int *__restrict__ ray_list,
                     int list_cap, int *__restrict__ huge_list, int huge_cap, const int *__restrict__ only) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    if (only && ctr->bwd_fb == 0) return;  // no spilled rays (the common case)
    __shared__ unsigned long long s_tab[32];
    __shared__ float s_e[4][kWarpListBwd], s_x[4][kWarpListBwd];
    __shared__ int s_c[4][kWarpListBwd];
    load_exp_tab(s_tab);
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * 4, gw = blockIdx.x * 4 + wid;
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    const float dt = mp.dt;
    // only: the rays K6a left to this walk (ctr->bwd_fb of them), else every ray
    const int64_t n_iter = only ? (int64_t)min((unsigned long long)ctr->bwd_fb, (unsigned long long)n_rays) : n_rays;
    for (int64_t q = gw; q < n_iter; q += nwarps) {
        const int64_t r = only ? (int64_t)only[q] : q;
        const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
        const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        // the forward of these rays kept the ray's segment list (count >= 0), or marked it as
        // too long (-1): those rays go to k_backward_rays_list
        const int nh = __float_as_int(bd.fwd_state[8 * r + 7]);
        if (nh < 0) {
            if (lane == 0) {
                if (nh == -2 && huge_list) {  // the forward needed more than kFallbackCap live segments
                    const unsigned slot = atomicAdd(&ctr->bwd_huge, 1u);
                    if ((int)slot < huge_cap) huge_list[slot] = (int)r;
                    else atomicAdd(&ctr->fallback_fail, 1);
                } else {
                    const unsigned slot = atomicAdd(&ctr->bwd_long, 1u);
                    if ((int)slot < list_cap) ray_list[slot] = (int)r;
                }
            }
            continue;
        }
        {
            const float *sg = bd.fwd_segs + (size_t)r * (3 * kRaySegs);
            for (int j = lane; j < nh; j += 32) {
                s_e[wid][j] = sg[j];
                s_x[wid][j] = sg[kRaySegs + j];
                s_c[wid][j] = __float_as_int(sg[2 * kRaySegs + j]);
            }
            __syncwarp();
        }
        const int cnt = nh;
        if (cnt == 0) continue;
        const float *E = s_e[wid], *X = s_x[wid];
        const int *P = s_c[wid];
        FwdReplay<BvhCands> fwd(cands, mp, s_tab);
        load_fwd_state(fwd, bd.fwd_state + 8 * r);
        const int lastStep = (int)fwd.lastStep;
        if (lastStep < 0) continue;
        const V3 aRgb = mk3(bd.adj_rgb[3 * r], bd.adj_rgb[3 * r + 1], bd.adj_rgb[3 * r + 2]);
        BwdWalk<BvhCands> bw(cands, mp, s_tab, fwd, bd, d, aRgb, bd.adj_alpha[r]);
        const float t0 = E[0];
        float gTmin = 0.f;
        int base = 0;
        for (;;) {
            const int i = base + lane;
            const bool valid = i <= lastStep;
            const float ts = t0 + (__int2float_rn(i) + jit) * dt;
            int na = 0, nadm = 0;
            for (int j = 0; j < cnt && valid; ++j) {
                if (!(E[j] <= ts)) break;
                nadm = j + 1;
                na += X[j] > ts;
            }
            const unsigned empty = __ballot_sync(0xffffffffu, !(valid && na > 0));
            const int L = empty ? __ffs(empty) - 1 : 32;
            float contrib = 0.f;
#if VPB_BWD_PAIRS
            // The chunk's primitive-samples (step s < L, k-th active entry of s), step-major,
            // are dealt out one per lane, 32 at a time. Each step's sum of rotG is then folded
            // in list order, starting from the carry of the previous batch, exactly as
            // gPWorldStep accumulates in the per-step walk (grad.cpp:66-164).
            const int myna = lane < L ? na : 0;
            int incl = myna;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            const int excl = incl - myna;
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            V3 acc = mk3(0.f, 0.f, 0.f);  // gPWorldStep of this lane's step
            for (int p0 = 0; p0 < total; p0 += 32) {
                const int p = p0 + lane;
                const bool has = p < total;
                int s = 0;  // the pair's step: the number of lanes with incl <= p
#pragma unroll
                for (int h = 16; h > 0; h >>= 1)
                    if (__shfl_sync(0xffffffffu, incl, s + h - 1) <= p) s += h;
                const int k = p - __shfl_sync(0xffffffffu, excl, s);
                const int incl_s = __shfl_sync(0xffffffffu, incl, s);
                const float tsp = __shfl_sync(0xffffffffu, ts, s);
                V3 rg = mk3(0.f, 0.f, 0.f);
                if (has) {
                    int j = 0;
                    for (int left = k;; ++j)
                        if (X[j] > tsp) {
                            if (left == 0) break;
                            --left;
                        }
                    bw.step_begin(base + s, tsp, o + d * tsp);
                    bw.prim(P[j], P[j]);
                    rg = bw.gPWorldStep;
                }
                const bool lead = has && (lane == 0 || k == 0);
                const int run = lead ? min(incl_s - p, 32 - lane) : 0;
                // a run leader starts from its step's carry (the sum over earlier batches)
                V3 c = mk3(__shfl_sync(0xffffffffu, acc.x, s), __shfl_sync(0xffffffffu, acc.y, s),
                           __shfl_sync(0xffffffffu, acc.z, s));
                c = c + rg;
                const int maxrun = __reduce_max_sync(0xffffffffu, run);
                for (int t = 1; t < maxrun; ++t) {
                    const V3 v = mk3(__shfl_down_sync(0xffffffffu, rg.x, t), __shfl_down_sync(0xffffffffu, rg.y, t),
                                     __shfl_down_sync(0xffffffffu, rg.z, t));
                    if (t < run) c = c + v;
                }
                // lane s < L takes its step's fold from the lane holding the step's first pair here
                const int f = excl > p0 ? excl - p0 : 0;
                const bool mine = lane < L && excl < p0 + 32 && incl > p0;
                const int fl = f < 32 ? f : 31;
                const V3 nv = mk3(__shfl_sync(0xffffffffu, c.x, fl), __shfl_sync(0xffffffffu, c.y, fl),
                                  __shfl_sync(0xffffffffu, c.z, fl));
                if (mine) acc = nv;
            }
            if (lane < L) contrib = dot3(acc, d);
#else
            if (lane < L) {  // a visited step with samples (grad.cpp:66-164)
                bw.step_begin(i, ts, o + d * ts);
                for (int j = 0; j < nadm; ++j)
                    if (X[j] > ts) bw.prim(P[j], P[j]);
                contrib = dot3(bw.gPWorldStep, d);
            }
#endif
            for (int s = 0; s < L; ++s) gTmin += __shfl_sync(0xffffffffu, contrib, s);  // step order
            if (base + L - 1 >= lastStep) break;
            if (L == 32) {
                base += 32;
                continue;
            }
            const int iL = base + L;
            const int nadmL = __shfl_sync(0xffffffffu, nadm, L);
            if (nadmL >= cnt) break;
            const float nextE = E[nadmL];
            const double sk = ceil((double)((nextE - t0) / dt) - (double)jit);  // gap skip, march.cpp:45-49
            const int skipTo = sk > (double)(1 << 30) ? (1 << 30) + 1 : (int)sk;
            base = skipTo > iL + 1 ? skipTo : iL + 1;
        }
        if (lane == 0) anchor_chain(bw, cands, bd, P[0], t0, gTmin, o, d);
        __syncwarp();
        bw.flush_warp(lane);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// K6a-c: the backward as passes over primitive-samples (the default path). The warp-per-ray
// walk above keeps its lanes busy only 60 % of the time (19 threads per instruction): a ray
// has ~50 samples spread over chunks of 32 lattice steps. Here one thread evaluates one
// sample, so every lane works, and the per-ray bookkeeping is two light thread-per-ray passes.

// Rays the forward could not keep a list for go to the per-thread kernels (as in the warp walk).
__device__ __forceinline__ void route_long_ray(int nh, int64_t r, DevCounters *ctr, int *ray_list, int list_cap,
                                               int *huge_list, int huge_cap) {
    if (nh == -2 && huge_list) {  // the forward needed more than kFallbackCap live segments
        const unsigned slot = atomicAdd(&ctr->bwd_huge, 1u);
        if ((int)slot < huge_cap) huge_list[slot] = (int)r;
        else atomicAdd(&ctr->fallback_fail, 1);
    } else {
        const unsigned slot = atomicAdd(&ctr->bwd_long, 1u);
        if ((int)slot < list_cap) ray_list[slot] = (int)r;
    }
}

// K6a's walk for one ray by its warp: the lattice walk of march.cpp:27-58 over the ray's segment
// list E/X (admission, gap skip; steps 0..lastStep), 32 steps per round, without sampling.
// Entry j is admitted at step A[j] (-1: never) and is live on the n_j consecutive steps from
// there; OFF[j] is the exclusive prefix of n_j in entry order, OFF[nh] the total (returned).
__device__ __forceinline__ int plan_ray_walk(int lane, const float *E, const float *X, int *A, int *OFF, int nh,
                                             int lastStep, float jit, float dt) {
    for (int j = lane; j < nh; j += 32) A[j] = -1;
    __syncwarp();
    const float t0 = E[0];
    int base = 0, nadm_prev = 0;  // entries admitted before this round
    for (;;) {
        const int i = base + lane;
        const bool valid = i <= lastStep;
        const float ts = t0 + (__int2float_rn(i) + jit) * dt;
        int na = 0, nadm = 0;
        for (int j = 0; j < nh && valid; ++j) {
            if (!(E[j] <= ts)) break;  // sorted by tEnter: the admitted entries are a prefix
            nadm = j + 1;
            na += X[j] > ts;
        }
        const unsigned empty = __ballot_sync(0xffffffffu, !(valid && na > 0));
        const int L = empty ? __ffs(empty) - 1 : 32;
        // the steps visited this round: s < L, and s == L when it is a real (empty) step
        int before = __shfl_up_sync(0xffffffffu, nadm, 1);
        if (lane == 0) before = nadm_prev;
        if (valid && lane <= L)
            for (int j = before; j < nadm; ++j) A[j] = base + lane;
        if (L == 32) {
            nadm_prev = __shfl_sync(0xffffffffu, nadm, 31);
            base += 32;
            if (base > lastStep) break;
            continue;
        }
        const int iL = base + L;
        if (iL > lastStep) break;
        const int nadmL = __shfl_sync(0xffffffffu, nadm, L);
        if (nadmL >= nh) break;  // nothing left to admit: march.cpp:43-44
        nadm_prev = nadmL;
        const double sk = ceil((double)((E[nadmL] - t0) / dt) - (double)jit);  // gap skip, march.cpp:45-49
        const int skipTo = sk > (double)(1 << 30) ? (1 << 30) + 1 : (int)sk;
        base = skipTo > iL + 1 ? skipTo : iL + 1;
        if (base > lastStep) break;
    }
    __syncwarp();
    // n_j (the live steps from a_j, up to lastStep), then offsets in entry order
    int carry = 0;
    for (int j0 = 0; j0 < nh; j0 += 32) {
        const int j = j0 + lane;
        int n = 0;
        if (j < nh && A[j] >= 0) {
            // e = the first step >= a_j with ts(e) >= X_j (or lastStep + 1): ts is
            // nondecreasing in e, so start from the real-valued estimate and correct it
            const int a = A[j];
            const float x = X[j];
            const double est = ceil((double)((x - t0) / dt) - (double)jit);
            int e = est < (double)a ? a : est > (double)lastStep + 1.0 ? lastStep + 1 : (int)est;
            while (e > a && t0 + (__int2float_rn(e - 1) + jit) * dt >= x) --e;
            while (e <= lastStep && t0 + (__int2float_rn(e) + jit) * dt < x) ++e;
            n = e - a;
        }
        int incl = n;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        if (j < nh) OFF[j] = carry + incl - n;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    const int total = carry;
    if (lane == 0) OFF[nh] = total;
    __syncwarp();
    return total;
}

// K6a, one warp per ray: the lattice walk of march.cpp:27-58 over the forward's segment list
// (admission, gap skip; steps 0..lastStep), 32 steps per round as march_warp steps it, without
// sampling. Entry j is admitted at step a_j and is live on the n_j consecutive steps from there
// (while it is live the active set is not empty, so no gap skip intervenes), so the ray's
// primitive-samples are (j, a_j + t), t < n_j. They get the range [base, base + sum n_j) of
// the pair arrays, entry-major; each record carries what K6b needs without further lookups.
__global__ void __launch_bounds__(128)
k_bwd_plan(MarchDev mp, RaysDev rays, int64_t n_rays, BwdDev bd, BwdPairs pp, DevCounters *ctr,
           int *__restrict__ ray_list, int list_cap, int *__restrict__ huge_list, int huge_cap) {
    __shared__ float s_E[4][kRaySegs], s_X[4][kRaySegs];
    __shared__ int s_a[4][kRaySegs], s_off[4][kRaySegs + 1];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *E = s_E[wid], *X = s_X[wid];
    int *A = s_a[wid], *OFF = s_off[wid];
    const float dt = mp.dt;
    const int64_t nwarps = (int64_t)gridDim.x * 4;
    for (int64_t r = (int64_t)blockIdx.x * 4 + wid; r < n_rays; r += nwarps) {
        const float *state = bd.fwd_state + 8 * r;
        const int nh = __float_as_int(state[7]);
        const int lastStep = __float_as_int(state[0]);
        if (nh < 0 || nh == 0 || lastStep < 0) {
            if (lane == 0) {
                if (nh < 0) route_long_ray(nh, r, ctr, ray_list, list_cap, huge_list, huge_cap);
                pp.span[r] = make_int4(0, nh < 0 ? -1 : 0, 0, 0);
            }
            continue;
        }
        const float *sg = bd.fwd_segs + (size_t)r * (3 * kRaySegs);
        for (int j = lane; j < nh; j += 32) {
            E[j] = sg[j];
            X[j] = sg[kRaySegs + j];
        }
        __syncwarp();
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        const int total = plan_ray_walk(lane, E, X, A, OFF, nh, lastStep, jit, dt);
        int2 *ent = pp.ent + (size_t)r * kRaySegs;
        for (int j = lane; j < nh; j += 32) ent[j] = make_int2(A[j], OFF[j]);
        const int4 sp = make_int4(0, total, nh, 0);  // base: k_bwd_scan_* (ray order)
        if (lane == 0) pp.span[r] = sp;
        __syncwarp();
    }
}

// Pair bases in ray order (so K6b's lanes and resident warps walk neighbouring rays, whose
// samples share payload and gradient lines in L2): an exclusive scan of the rays' sample
// counts. k_bwd_scan_tiles scans 1024 rays per CTA (span.x = offset within the tile, tile_sums
// = the tile's total); k_bwd_scan_top turns tile_sums into tile bases and stores the grand
// total as the pair count.
constexpr int kScanTile = 4096;  // rays per CTA of k_bwd_scan_tiles: 1024 threads x 4
__global__ void __launch_bounds__(1024) k_bwd_scan_tiles(int64_t n_rays, BwdPairs pp, DevCounters *ctr) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    __shared__ int s_w[32];
    const int64_t r0 = (int64_t)blockIdx.x * kScanTile + 4 * threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int v[4], mine = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        v[u] = r0 + u < n_rays ? max(pp.span[r0 + u].y, 0) : 0;
        mine += v[u];
    }
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += u;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = s_w[lane], wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += u;
        }
        s_w[lane] = wi - w;  // exclusive warp bases
        if (lane == 31) {
            pp.tile_sums[blockIdx.x] = gridDim.x == 1 ? 0 : wi;
            if (gridDim.x == 1) ctr->bwd_pairs = (unsigned long long)wi;  // one tile: no k_bwd_scan_top
        }
    }
    __syncthreads();
    int off = s_w[wid] + incl - mine;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (r0 + u < n_rays) pp.span[r0 + u].x = off;
        off += v[u];
    }
}

__global__ void __launch_bounds__(1024) k_bwd_scan_top(int n_tiles, BwdPairs pp, DevCounters *ctr) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    __shared__ long long s_w[32];
    __shared__ long long s_carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int t0 = 0; t0 < n_tiles; t0 += 1024) {
        const int t = t0 + threadIdx.x;
        const long long v = t < n_tiles ? pp.tile_sums[t] : 0;
        long long incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long u = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += u;
        }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            long long w = s_w[lane], wi = w;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const long long u = __shfl_up_sync(0xffffffffu, wi, off);
                if (lane >= off) wi += u;
            }
            s_w[lane] = wi - w;
        }
        __syncthreads();
        const long long base = s_carry + s_w[wid] + incl - v;
        // bases past 2^31 cannot be pair indices: those rays take the warp walk (capacity < 2^31)
        if (t < n_tiles) pp.tile_sums[t] = (int)min(base, (long long)0x7fffffff);
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = base + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) ctr->bwd_pairs = (unsigned long long)s_carry;
}

// K6a (records), one warp per ray: the ray's samples (j, a_j + t), entry-major, at its base in
// ray order; a ray past the capacity goes to the warp walk (the one straddling it leaves
// sentinels that K6b skips).
__global__ void __launch_bounds__(128)
k_bwd_records(MarchDev mp, RaysDev rays, int64_t n_rays, BwdDev bd, BwdPairs pp, DevCounters *ctr) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    __shared__ int s_a[4][kRaySegs], s_off[4][kRaySegs + 1];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int *A = s_a[wid], *OFF = s_off[wid];
    const float dt = mp.dt;
    const int64_t nwarps = (int64_t)gridDim.x * 4;
    for (int64_t r = (int64_t)blockIdx.x * 4 + wid; r < n_rays; r += nwarps) {
        int4 sp = pp.span[r];
        if (sp.y <= 0) continue;
        const int total = sp.y, nh = sp.z;
        const long long base = (long long)pp.tile_sums[r / kScanTile] + sp.x;
        if (base + total > (long long)pp.cap) {  // no room: the warp walk takes the ray
            if (lane == 0) {
                pp.fb_list[atomicAdd(&ctr->bwd_fb, 1u)] = (int)r;
                pp.span[r] = make_int4(0, -1, nh, 0);
            }
            for (long long t = base + lane; t < (long long)pp.cap; t += 32) pp.rec[t] = make_int4(-1, 0, 0, 0);
            continue;
        }
        const int2 *ent = pp.ent + (size_t)r * kRaySegs;
        for (int j = lane; j < nh; j += 32) {
            const int2 e = ent[j];
            A[j] = e.x;
            OFF[j] = e.y;
        }
        __syncwarp();
        const float *state = bd.fwd_state + 8 * r;
        const int lastStep = __float_as_int(state[0]);
        const bool sat = __float_as_int(state[1]) != 0;
        const float *sg = bd.fwd_segs + (size_t)r * (3 * kRaySegs);
        const float t0 = sg[0];
        const float jit = rays.jitter ? rays.jitter[r] : 0.5f;
        if (lane == 0) OFF[nh] = total;
        __syncwarp();
        for (int p = lane; p < total; p += 32) {
            int lo = 0, hi = nh - 1;  // the last entry with OFF[j] <= p
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (OFF[mid] <= p) lo = mid;
                else hi = mid - 1;
            }
            const int step = A[lo] + (p - OFF[lo]);
            // the sample's place in step-major order (steps in order, each step's live entries
            // in list order): samples of every entry at earlier steps, then the entries before
            // this one live at this step
            int sm = 0;
            for (int j = 0; j < nh; ++j) {
                const int a = A[j];
                if (a < 0 || a > step) break;  // admission steps grow with j; unadmitted entries last
                const int n = OFF[j + 1] - OFF[j];
                sm += min(step - a, n) + (j < lo && step < a + n ? 1 : 0);
            }
            const float ts = t0 + (__int2float_rn(step) + jit) * dt;
            const int c = __float_as_int(sg[2 * kRaySegs + lo]);
            const unsigned w = (unsigned)(base + sm) | ((sat && step == lastStep) ? 0x80000000u : 0u);
            pp.rec[base + p] = make_int4((int)r, c, __float_as_int(ts), (int)w);
            pp.terms[base + sm].w = __int_as_float(step);  // K6b fills in rotG
        }
        if (lane == 0) pp.span[r].x = (int)base;
        __syncwarp();
    }
}

// K6b, one thread per primitive-sample: the sample's adjoint (sample_adjoint: payload scatter
// as reductions). The pose terms go to the primitive's deltaT/deltaR/deltaS: the samples are
// entry-major, so a warp's lanes form runs of one (ray, primitive); each run is summed with a
// segmented shuffle scan and its last lane issues the nine reductions (SURVEY.md §8 a-20:
// warp-aggregated atomics). rotG is kept for K6c's t_min chain (terms, step-major).
__global__ void __launch_bounds__(VPB_BWD_PAIRS_NT, VPB_BWD_PAIRS_MINB)
k_bwd_pairs(MarchDev mp, const float *__restrict__ xf_g, int n_prim, const float4 *__restrict__ payload,
            RaysDev rays, BwdDev bd, BwdPairs pp, const DevCounters *__restrict__ ctr) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    __shared__ unsigned long long s_tab[32];
    load_exp_tab(s_tab);
    __syncthreads();
    const BvhCands cands{xf_g, payload, (unsigned)(mp.m * mp.m * mp.m), n_prim, mp.bvh};
    const unsigned long long n = min(ctr->bwd_pairs, (unsigned long long)pp.cap);
    const size_t cap = pp.cap;
    const int lane = threadIdx.x & 31;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    // warp-uniform loop: every lane takes part in the shuffles
    for (size_t p0 = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); p0 < n; p0 += stride) {
        const size_t p = p0 + lane;
        int4 rec = make_int4(-1, -1, 0, 0);
        if (p < n) rec = pp.rec[p];
        float v[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) v[q] = 0.f;
        if (rec.x >= 0) {  // (rec.x < 0: the unwritten part of a ray that did not fit, k_bwd_plan)
            const int64_t r = rec.x;
            const int c = rec.y;
            const float ts = __int_as_float(rec.z);
            const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
            const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
            FwdReplay<BvhCands> fwd(cands, mp, s_tab);
            load_fwd_state(fwd, bd.fwd_state + 8 * r);
            const V3 aRgb = mk3(bd.adj_rgb[3 * r], bd.adj_rgb[3 * r + 1], bd.adj_rgb[3 * r + 2]);
            if (bd.touched) bd.touched[c] = 1u;
            V3 rotG, rTerm, sTerm;
            if (sample_adjoint(cands, mp, s_tab, fwd, bd, aRgb, bd.adj_alpha[r], rec.w < 0, c, c, o + d * ts, rotG,
                               rTerm, sTerm)) {
                v[0] = -rotG.x;
                v[1] = -rotG.y;
                v[2] = -rotG.z;
                v[3] = rTerm.x;
                v[4] = rTerm.y;
                v[5] = rTerm.z;
                v[6] = sTerm.x;
                v[7] = sTerm.y;
                v[8] = sTerm.z;
            }
            // rotG (+0 without pose terms) at the sample's step-major place, with its step
            float4 *t = pp.terms + (rec.w & 0x7fffffff);
            t->x = -v[0];
            t->y = -v[1];
            t->z = -v[2];
        }
        // runs of equal (ray, primitive) over the lanes: segmented inclusive scan
        const int prev_x = __shfl_up_sync(0xffffffffu, rec.x, 1), prev_y = __shfl_up_sync(0xffffffffu, rec.y, 1);
        const bool head = lane == 0 || prev_x != rec.x || prev_y != rec.y;
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        const int seg = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));  // this lane's run starts here
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                const float u = __shfl_up_sync(0xffffffffu, v[q], off);
                if (lane - off >= seg) v[q] += u;
            }
        }
        const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
        if (tail && rec.x >= 0) {
            float *g = bd.g_pose + 9 * (size_t)rec.y;
#pragma unroll
            for (int q = 0; q < 9; ++q)
                if (v[q] != 0.f) red_add(g + q, v[q]);
        }
    }
}

// K6c, one thread per ray: gTmin = the sum over the visited steps, in step order, of
// dot(gPWorldStep, d), gPWorldStep = the step's rotG summed in list order from 0 (grad.cpp:66-
// 164). The ray's samples are read in step-major order (k_bwd_records placed each sample's
// rotG there, with its step), so both sums are one sequential pass (a sample without pose
// terms adds +0, which leaves a sum that started at +0 unchanged). Then the t_min anchor chain
// (grad.cpp:166-194) onto the first hit's primitive.
__global__ void __launch_bounds__(128)
k_bwd_fold(const float *__restrict__ xf_g, RaysDev rays, int64_t n_rays, BwdDev bd, BwdPairs pp) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int4 sp = pp.span[r];
        if (sp.y <= 0) continue;
        const float4 *T = pp.terms + (size_t)sp.x;
        const V3 d = mk3(rays.dirs[3 * r], rays.dirs[3 * r + 1], rays.dirs[3 * r + 2]);
        float gTmin = 0.f;
        V3 g = mk3(0.f, 0.f, 0.f);
        int cur = __float_as_int(T[0].w);
        for (int t = 0; t < sp.y; ++t) {
            const float4 v = T[t];
            const int step = __float_as_int(v.w);
            if (step != cur) {  // the previous step is complete
                gTmin += dot3(g, d);
                g = mk3(0.f, 0.f, 0.f);
                cur = step;
            }
            g = g + mk3(v.x, v.y, v.z);
        }
        gTmin += dot3(g, d);
        if (gTmin == 0.f) continue;
        const float *sg = bd.fwd_segs + (size_t)r * (3 * kRaySegs);
        const int k0 = __float_as_int(sg[2 * kRaySegs]);
        const V3 o = mk3(rays.origins[3 * r], rays.origins[3 * r + 1], rays.origins[3 * r + 2]);
        V3 gT3, gR3, gS3;
        if (!anchor_terms(xf_g + (size_t)k0 * kXfStride, bd.pose36 + 36 * (size_t)k0, sg[0], gTmin, o, d, gT3, gR3,
                          gS3))
            continue;
        float *gp = bd.g_pose + 9 * (size_t)k0;
        const float an[9] = {gT3.x, gT3.y, gT3.z, gR3.x, gR3.y, gR3.z, gS3.x, gS3.y, gS3.z};
#pragma unroll
        for (int q = 0; q < 9; ++q)
            if (an[q] != 0.f) red_add(gp + q, an[q]);
    }
}

// The channel-interleaved payload gradient (VPB_BWD_V4 layout) into the caller's planar
// GradBuffer (params.h:12-27): primitives the walk touched are transposed (assigned, or added
// when accumulating) and their interleaved slots cleared for the next call; untouched ones get
// zeros (or keep the caller's values when accumulating). One thread per voxel.
__global__ void __launch_bounds__(256) k_grad_transpose(float4 *__restrict__ g4, float *__restrict__ planar,
                                                        const unsigned *__restrict__ touched, int n_prim,
                                                        unsigned m3, int accumulate) {
    for (int k = blockIdx.x; k < n_prim; k += gridDim.x) {  // one primitive per CTA iteration
        float *dst = planar + (size_t)k * 4 * m3;
        float4 *src = g4 + (size_t)k * m3;
        if (!touched[k]) {
            if (!accumulate)
                for (unsigned i = threadIdx.x; i < 4 * m3; i += blockDim.x) dst[i] = 0.f;
            continue;
        }
        // four voxels per thread per round, all loads issued before the stores (one load in
        // flight per thread left the kernel latency-bound at 12 % of DRAM bandwidth)
        constexpr int U = 4;
        for (unsigned v0 = threadIdx.x; v0 < m3; v0 += U * blockDim.x) {
            float4 g[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned v = v0 + u * blockDim.x;
                g[u] = v < m3 ? src[v] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned v = v0 + u * blockDim.x;
                if (v >= m3) break;
                src[v] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (accumulate) {
                    dst[v] += g[u].x;
                    dst[m3 + v] += g[u].y;
                    dst[2 * m3 + v] += g[u].z;
                    dst[3 * m3 + v] += g[u].w;
                } else {
                    dst[v] = g[u].x;
                    dst[m3 + v] = g[u].y;
                    dst[2 * m3 + v] = g[u].z;
                    dst[3 * m3 + v] = g[u].w;
                }
            }
        }
    }
}

// The same for m3 % 4 == 0, flattened over (primitive, 4 consecutive voxels) in tiles of 256
// quads per CTA (untouched primitives: zero vectors, or nothing when accumulating; touched
// ones): the tile's interleaved voxels are loaded with coalesced 16-byte accesses and
// staged in shared memory; after the barrier the slots are cleared (a store to an address
// whose load is still in flight stalls the warp: 6x slower when the clear followed each load)
// and each thread writes its quad as one 16-byte vector per channel plane.
__global__ void __launch_bounds__(256) k_grad_transpose4(float4 *__restrict__ g4, float4 *__restrict__ planar,
                                                         const unsigned *__restrict__ touched, unsigned nq,
                                                         unsigned q3, int accumulate, int clear) {
    VPB_PDL_WAIT();  // launched after its producer with programmatic serialization
    __shared__ float4 sm[4 * 256 + 4 * 8];  // padded: a float4 every 8 keeps the quad reads conflict-light
    const int t = threadIdx.x;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned i0 = blockIdx.x * 256u; i0 < nq; i0 += gridDim.x * 256u) {
        const unsigned k_first = i0 / q3, k_last = min(i0 + 255u, nq - 1) / q3;
        bool any = false;  // block-uniform: is a primitive of this tile touched?
        for (unsigned k = k_first; k <= k_last && !any; ++k) any = touched[k] != 0u;
        if (!any) {  // untouched primitives: zeros (or the caller's values when accumulating)
            const unsigned i = i0 + t;
            if (!accumulate && i < nq) {
                const unsigned k = i / q3;
                float4 *dst = planar + (size_t)k * 4 * q3 + (i - k * q3);
                dst[0] = z;
                dst[q3] = z;
                dst[2 * q3] = z;
                dst[3 * q3] = z;
            }
            continue;
        }
        bool tch[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned l = t + 256 * u, iq = i0 + (l >> 2);  // voxel 4 * i0 + l is in quad iq
            tch[u] = iq < nq && touched[iq / q3];
            sm[l + (l >> 5)] = tch[u] ? g4[4 * (size_t)i0 + l] : z;
        }
        __syncthreads();
        if (clear)
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (tch[u]) g4[4 * (size_t)i0 + t + 256 * u] = z;
        const unsigned i = i0 + t;
        if (i < nq) {
            const unsigned k = i / q3, qv = i - k * q3;
            float4 *dst = planar + (size_t)k * 4 * q3 + qv;  // plane c at dst[c * q3]
            if (touched[k]) {
                const int l = 4 * t;
                const float4 a = sm[l + (l >> 5)], b = sm[l + 1 + ((l + 1) >> 5)], c = sm[l + 2 + ((l + 2) >> 5)],
                             d = sm[l + 3 + ((l + 3) >> 5)];
                float4 p0 = make_float4(a.x, b.x, c.x, d.x), p1 = make_float4(a.y, b.y, c.y, d.y);
                float4 p2 = make_float4(a.z, b.z, c.z, d.z), p3 = make_float4(a.w, b.w, c.w, d.w);
                if (accumulate) {
                    const float4 o0 = dst[0], o1 = dst[q3], o2 = dst[2 * q3], o3 = dst[3 * q3];
                    p0 = make_float4(o0.x + p0.x, o0.y + p0.y, o0.z + p0.z, o0.w + p0.w);
                    p1 = make_float4(o1.x + p1.x, o1.y + p1.y, o1.z + p1.z, o1.w + p1.w);
                    p2 = make_float4(o2.x + p2.x, o2.y + p2.y, o2.z + p2.z, o2.w + p2.w);
                    p3 = make_float4(o3.x + p3.x, o3.y + p3.y, o3.z + p3.z, o3.w + p3.w);
                }
                dst[0] = p0;
                dst[q3] = p1;
                dst[2 * q3] = p2;
                dst[3 * q3] = p3;
            } else if (!accumulate) {
                dst[0] = z;
                dst[q3] = z;
                dst[2 * q3] = z;
                dst[3 * q3] = z;
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_grad_transpose(float4 *g4, float *planar, const unsigned *touched, int n_prim, unsigned m3,
                                  bool accumulate, cudaStream_t st, bool clear) {
    if (n_prim == 0 || m3 == 0) return cudaSuccess;
    const size_t nq = size_t(n_prim) * (m3 / 4);
    if (m3 % 4 == 0 && (reinterpret_cast<uintptr_t>(planar) & 15) == 0 && nq < (size_t(1) << 32) - 256) {
        return launch_pdl(k_grad_transpose4, dim3(148 * VPB_TR_GRID), dim3(256), 0, st, g4,
                          reinterpret_cast<float4 *>(planar), touched, unsigned(nq), m3 / 4, accumulate ? 1 : 0,
                          clear ? 1 : 0);
    }
    const int blocks = n_prim < 148 * 8 ? n_prim : 148 * 8;
    k_grad_transpose<<<blocks, 256, 0, st>>>(g4, planar, touched, n_prim, m3, accumulate ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_backward_rays(const MarchDev &mp, const float *xf16, int n_prim,
                                 const float4 *payload, const RaysDev &rays, int64_t n_rays,
                                 const BwdDev &bd, DevCounters *ctr, int *ray_list, int list_cap, float *se,
                                 float *sx, int *sc, cudaStream_t st, int *huge_list, int huge_cap, float *he,
                                 float *hx, int *hc, const BwdPairs *pairs, cudaStream_t st2, cudaEvent_t ev_fork,
                                 cudaEvent_t ev_join) {
    if (n_rays == 0 || n_prim == 0) return cudaSuccess;
    // The adjoint walk goes warp-per-ray for every batch size (the forward's state and segment
    // lists are required): one ray per thread leaves 27 % of the lanes busy (the rays' walks
    // diverge); then the rays with lists too long for the forward to keep, one per thread.
    if (!bd.fwd_state || !bd.fwd_segs) return cudaErrorInvalidValue;
    const int64_t blocks = (n_rays + 3) / 4;
    if (pairs) {
        const unsigned ray_blocks = (unsigned)(blocks < 148 * VPB_BWD_RAY_GRID ? blocks : 148 * VPB_BWD_RAY_GRID);
        k_bwd_plan<<<ray_blocks, 128, 0, st>>>(mp, rays, n_rays, bd, *pairs, ctr, ray_list, list_cap, huge_list,
                                               huge_cap);
        const int64_t n_tiles = (n_rays + kScanTile - 1) / kScanTile;
        // the chain from here on launches programmatically (each kernel waits for its producer)
        if (cudaError_t e = cudaGetLastError()) return e;
        if (cudaError_t e = launch_pdl(k_bwd_scan_tiles, dim3((unsigned)n_tiles), dim3(1024), 0, st, n_rays, *pairs, ctr))
            return e;
        if (n_tiles > 1)
            if (cudaError_t e = launch_pdl(k_bwd_scan_top, dim3(1), dim3(1024), 0, st, (int)n_tiles, *pairs, ctr))
                return e;
        if (cudaError_t e = launch_pdl(k_bwd_records, dim3(ray_blocks), dim3(128), 0, st, mp, rays, n_rays, bd, *pairs,
                                       ctr))
            return e;
        if (cudaError_t e = launch_pdl(k_bwd_pairs, dim3(148 * VPB_BWD_PAIR_GRID), dim3(VPB_BWD_PAIRS_NT), 0, st, mp,
                                       xf16, n_prim, payload, rays, bd, *pairs, ctr))
            return e;
        const int64_t tb = (n_rays + 127) / 128;
        // K6c reads only K6b's rotG and writes pose reductions: it runs beside the walk for the
        // spilled rays and the gradient transpose (the caller joins ev_join)
        cudaStream_t sf = st;
        if (st2 && ev_fork && ev_join) {
            cudaEventRecord(ev_fork, st);
            cudaStreamWaitEvent(st2, ev_fork, 0);
            sf = st2;
        }
        k_bwd_fold<<<(unsigned)(tb < 148 * 16 ? tb : 148 * 16), 128, 0, sf>>>(xf16, rays, n_rays, bd, *pairs);
        if (sf != st) cudaEventRecord(ev_join, sf);
        // the rays that found no room in the pair arrays (none once the capacity has grown)
        k_backward_rays_warp<<<(unsigned)(blocks < 148 * 4 ? blocks : 148 * 4), 128, 0, st>>>(
            mp, xf16, n_prim, payload, rays, n_rays, bd, ctr, ray_list, list_cap, huge_list, huge_cap, pairs->fb_list);
    } else {
        k_backward_rays_warp<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 128, 0, st>>>(
            mp, xf16, n_prim, payload, rays, n_rays, bd, ctr, ray_list, list_cap, huge_list, huge_cap, nullptr);
    }
    if (cudaError_t e = cudaGetLastError()) return e;
    if (cudaError_t e = launch_pdl(k_backward_rays_list, dim3(kBackwardWarps), dim3(32), 0, st, mp, xf16, n_prim,
                                   payload, rays, bd, ctr, ray_list, list_cap, se, sx, sc))
        return e;
    if (huge_list)
        return launch_pdl(k_backward_rays_huge, dim3(kHugeThreads / 32), dim3(32), 0, st, mp, xf16, n_prim, payload,
                          rays, bd, ctr, huge_list, huge_cap, he, hx, hc);
    return cudaSuccess;
}

}  // namespace vpb
