// vpb_losses.cpp — the O(K) regularisers of evalLoss (losses.cpp:27-68), host side with the
// reference's binary32 operation order (built with -ffp-contract=off). They touch only the
// pose deltas and the guide-mesh offsets, so they stay on the host next to compose().
#include <cstdint>

#include "../../include/vpb.h"
#include "vpb_hostmath.hpp"

using namespace vpb::host;

// lossVol (losses.cpp:45-55) + lossDel (losses.cpp:57-68). grad_pose (nullable) receives
// += deltaT[3] deltaR[3] deltaS[3] per primitive, in the reference's accumulation order
// (lossVol's deltaS term first, then lossDel's).
extern "C" int vp_loss_pose(int32_t n_prim, const float *tr24, float lambda_vol, float lambda_del,
                            float *loss_vol, float *loss_del, float *grad_pose) {
    if (n_prim < 0 || (n_prim > 0 && !tr24)) return VP_ERR_USAGE;
    float accv = 0, accd = 0;
    for (int32_t k = 0; k < n_prim; ++k) {
        const float *t = tr24 + 24 * size_t(k);
        const F3 s = add(load3(t + 12), load3(t + 21));
        accv += s.x * s.y * s.z;
        if (grad_pose) {
            float *g = grad_pose + 9 * size_t(k);
            const F3 gs = mul(f3(s.y * s.z, s.x * s.z, s.x * s.y), lambda_vol);
            g[6] += gs.x;
            g[7] += gs.y;
            g[8] += gs.z;
        }
    }
    const float two_l = 2 * lambda_del;
    for (int32_t k = 0; k < n_prim; ++k) {
        const float *t = tr24 + 24 * size_t(k);
        const F3 dT = load3(t + 15), dR = load3(t + 18), dS = load3(t + 21);
        accd += dot(dT, dT) + dot(dR, dR) + dot(dS, dS);
        if (grad_pose) {
            float *g = grad_pose + 9 * size_t(k);
            const F3 a = mul(dT, two_l), b = mul(dR, two_l), c = mul(dS, two_l);
            g[0] += a.x; g[1] += a.y; g[2] += a.z;
            g[3] += b.x; g[4] += b.y; g[5] += b.z;
            g[6] += c.x; g[7] += c.y; g[8] += c.z;
        }
    }
    if (loss_vol) *loss_vol = lambda_vol * accv;
    if (loss_del) *loss_del = lambda_del * accd;
    return VP_OK;
}

// lossGeo (losses.cpp:27-43): base/offsets/tracked are n_verts*3; offsets nullable (zero).
extern "C" int vp_loss_geo(int32_t n_verts, const float *base, const float *offsets,
                           const float *tracked, float lambda, float *loss, float *grad_verts) {
    if (n_verts <= 0 || !base || !tracked) return VP_ERR_USAGE;
    const float invN = 1.0f / float(n_verts);
    const float scale = 2 * lambda * invN;
    float acc = 0;
    for (int32_t i = 0; i < n_verts; ++i) {
        F3 fitted = load3(base + 3 * size_t(i));
        if (offsets) fitted = add(fitted, load3(offsets + 3 * size_t(i)));
        const F3 e = sub(fitted, load3(tracked + 3 * size_t(i)));
        acc += dot(e, e);
        if (grad_verts) {
            const F3 g = mul(e, scale);
            grad_verts[3 * size_t(i)] += g.x;
            grad_verts[3 * size_t(i) + 1] += g.y;
            grad_verts[3 * size_t(i) + 2] += g.z;
        }
    }
    if (loss) *loss = lambda * invN * acc;
    return VP_OK;
}
