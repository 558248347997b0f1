// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" glue around the *unmodified* reference core built in double precision
// (-DVOLPRIM_USE_DOUBLE, the reference's own f64 configuration of acceptance_f64.cpp), compiled
// by oracle/Makefile into oracle/_ref/libvolprim_ref_f64.so. It exposes only the reference's
// gradcheck (grad.cpp:293-370): Richardson-extrapolated central differences of evalLoss on
// sampled coordinates of every parameter group, with the f64 analytic gradient beside them.
// oracle/gen_gradcheck.py stores the result as tests/golden/gradcheck.npz; the GPU test checks
// the device's f32 analytic gradient against these finite differences (an independent
// gradient check: no part of it is the device's own backward pass).
//
// Inputs are float32 arrays (exactly representable in double): tr24 = K PrimitiveTransform
// records (tBase[3] rBase[9] column-major sBase[3] deltaT[3] deltaR[3] deltaS[3]), the planar
// payload, cams23 = n_cams * {K[9] R[9] t[3] w h} (column-major), and the ray batch.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "volprim/errors.h"
#include "volprim/grad.h"
#include "volprim/params.h"
#include "volprim/scene.h"

using namespace volprim;

namespace {
thread_local std::string g_err64;
Vec3 v3(const float *p) { return Vec3(real(p[0]), real(p[1]), real(p[2])); }
Mat3 m3(const float *p) {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.m[i] = real(p[i]);
    return m;
}
}  // namespace

extern "C" {

const char *vpref64_last_error() { return g_err64.c_str(); }
int vpref64_sizeof_real() { return int(sizeof(real)); }

// Runs gradcheck(scene, 0, cams, batch, {}, weights, cfg, n_params, seed) and writes up to
// cap entries: index (GradBuffer order), group, analytic (f64), finite difference (f64).
int vpref64_gradcheck(int32_t nPrim, int32_t m, const float *tr24, const float *payload, float wAlpha,
                      int32_t wBeta, int32_t nCams, const float *cams23, int64_t n, const int32_t *camIndex,
                      const int32_t *pixelId, const float *target, const float *background, const float *weights4,
                      float stepSize, float earlyEps, int32_t nParams, uint64_t seed, int64_t cap, int64_t *nOut,
                      int64_t *index, int32_t *group, double *analytic, double *finiteDiff) {
    try {
        Scene scene;
        scene.window = WindowParams{real(wAlpha), wBeta};
        Frame fr;
        for (int k = 0; k < nPrim; ++k) {
            const float *p = tr24 + 24 * size_t(k);
            PrimitiveTransform xf;
            xf.tBase = v3(p);
            xf.rBase = m3(p + 3);
            xf.sBase = v3(p + 12);
            xf.deltaT = v3(p + 15);
            xf.deltaR = v3(p + 18);
            xf.deltaS = v3(p + 21);
            fr.transforms.push_back(xf);
        }
        fr.slab.resize(nPrim, m);
        for (size_t i = 0; i < fr.slab.payload.size(); ++i) fr.slab.payload[i] = real(payload[i]);
        scene.frames.push_back(fr);
        std::vector<Camera> cams;
        for (int c = 0; c < nCams; ++c) {
            const float *q = cams23 + 23 * size_t(c);
            Camera cam;
            cam.intrinsics = m3(q);
            cam.rotation.matrix = m3(q + 9);
            cam.translation = v3(q + 18);
            cam.width = int(q[21]);
            cam.height = int(q[22]);
            cams.push_back(cam);
        }
        std::vector<RaySample> batch(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            RaySample &rs = batch[size_t(i)];
            rs.cameraIndex = camIndex[i];
            rs.pixelId = pixelId[i];
            const int w = cams[size_t(rs.cameraIndex)].width;
            rs.pixel = Vec2(real(pixelId[i] % w) + real(0.5), real(pixelId[i] / w) + real(0.5));
            rs.target = v3(target + 3 * i);
            rs.background = v3(background + 3 * i);
        }
        LossWeights lw;
        lw.pho = real(weights4[0]);
        lw.geo = real(weights4[1]);
        lw.vol = real(weights4[2]);
        lw.del = real(weights4[3]);
        MarchConfig cfg;
        cfg.stepSize = real(stepSize);
        cfg.earlyEps = real(earlyEps);
        const GradcheckReport rep = gradcheck(scene, 0, cams, batch, {}, lw, cfg, nParams, seed);
        *nOut = int64_t(rep.entries.size());
        for (size_t i = 0; i < rep.entries.size() && int64_t(i) < cap; ++i) {
            index[i] = int64_t(rep.entries[i].index);
            group[i] = int32_t(rep.entries[i].group);
            analytic[i] = double(rep.entries[i].analytic);
            finiteDiff[i] = double(rep.entries[i].finiteDiff);
        }
        return 0;
    } catch (const Error &e) {
        g_err64 = e.what();
        return int(e.category());
    } catch (const std::exception &e) {
        g_err64 = e.what();
        return 1;
    }
}

}  // extern "C"
