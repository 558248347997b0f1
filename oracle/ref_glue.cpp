// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" glue around the *unmodified* reference volprim core
// (/root/reference/proj/src/volprim/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libvolprim_ref.so). It only marshals flat arrays into the reference's own
// types and calls the reference's own functions, so tests and bench.py's cpu_baseline /
// --impl reference legs can drive the real reference through ctypes:
//
//   vpref_render        -> volprim::render            (march.h:59, march.cpp:95-132)
//   vpref_compose       -> volprim::compose           (primitive.cpp:41-49)
//   vpref_look_at       -> volprim::lookAtCamera      (synthetic.cpp:15-38)
//   vpref_intersect     -> buildLbvh + intersect      (lbvh.cpp:81-156, 207-234)
//   vpref_march_rays    -> intersect + march          (march.cpp:18-93)
//   vpref_generate_ray  -> generateRay                (camera.cpp:14-23)
//   vpref_window        -> window                     (primitive.cpp:25-28)
//   vpref_backward_rays -> intersect + backwardRay    (grad.cpp:34-195) into a GradBuffer
//   vpref_load_slab     -> loadSlab                   (scene_io.cpp:43-66)
//   vpref_shell_scene   -> the §8d "mvp_shell" bench inputs, built with the reference's own
//                          compose() / AffineXf::toWorld (primitive.cpp:41-49, primitive.h:60)
//   vpref_shell_camera  -> lookAtCamera on the §8d headline view / 64-view ring
//   vpref_scene_*       -> a resident Scene (built once), so the reference arm of bench.py times
//                          volprim::render (march.cpp:95-132) and nothing else per call
//
// Flat layouts (shared with include/vpb.h):
//   PrimitiveTransform = 24 floats: tBase[3] rBase[9] (column-major) sBase[3] deltaT[3]
//                        deltaR[3] deltaS[3]
//   AffineXf           = 15 floats: t[3] rot[9] (column-major) scale[3]
//   Camera             = K[9] (column-major), R[9] (column-major), t[3], width, height
// Return codes: 0 ok, volprim::ErrorCategory value on volprim::Error, 1 on other exceptions.
#include <cstdint>
#include <algorithm>
#include <cmath>
#include <random>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "volprim/errors.h"
#include "volprim/grad.h"
#include "volprim/params.h"
#include "volprim/lbvh.h"
#include "volprim/march.h"
#include "volprim/primitive.h"
#include "volprim/scene.h"
#include "volprim/scene_io.h"
#include "volprim/synthetic.h"

using namespace volprim;

namespace {

thread_local std::string g_err;

Vec3 v3(const float *p) { return Vec3(p[0], p[1], p[2]); }
Mat3 m3(const float *p) {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.m[i] = p[i];
    return m;
}
void put3(float *o, const Vec3 &v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
void put9(float *o, const Mat3 &m) { for (int i = 0; i < 9; ++i) o[i] = m.m[i]; }

PrimitiveTransform transformFrom24(const float *p) {
    PrimitiveTransform xf;
    xf.tBase = v3(p + 0);
    xf.rBase = m3(p + 3);
    xf.sBase = v3(p + 12);
    xf.deltaT = v3(p + 15);
    xf.deltaR = v3(p + 18);
    xf.deltaS = v3(p + 21);
    return xf;
}

AffineXf xfFrom15(const float *p) {
    AffineXf xf;
    xf.t = v3(p + 0);
    xf.rot = m3(p + 3);
    xf.scale = v3(p + 12);
    return xf;
}

Camera cameraFrom(const float *k9, const float *r9, const float *t3, int w, int h) {
    Camera cam;
    cam.intrinsics = m3(k9);
    cam.rotation.matrix = m3(r9); // render() only reads rotation.matrix
    cam.translation = v3(t3);
    cam.width = w;
    cam.height = h;
    return cam;
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const Error &e) {
        g_err = e.what();
        return int(e.category());
    } catch (const std::exception &e) {
        g_err = e.what();
        return 1;
    }
}

} // namespace

extern "C" {

const char *vpref_last_error() { return g_err.c_str(); }

int vpref_sizeof_real() { return int(sizeof(real)); }

int vpref_compose(int32_t n, const float *tr24, float *xf15) {
    return guarded([&] {
        for (int k = 0; k < n; ++k) {
            const AffineXf xf = compose(transformFrom24(tr24 + 24 * size_t(k)));
            put3(xf15 + 15 * size_t(k) + 0, xf.t);
            put9(xf15 + 15 * size_t(k) + 3, xf.rot);
            put3(xf15 + 15 * size_t(k) + 12, xf.scale);
        }
    });
}

int vpref_render(int32_t nPrim, int32_t m, const float *tr24, const float *payload, float wAlpha,
                 int32_t wBeta, const float *k9, const float *r9, const float *t3, int32_t width,
                 int32_t height, float stepSize, float earlyEps, int32_t jitter, uint64_t seed,
                 uint64_t perm, float *rgb, float *alpha, int32_t *samples) {
    return guarded([&] {
        Scene scene;
        scene.window = WindowParams{wAlpha, wBeta};
        Frame fr;
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        scene.frames.push_back(std::move(fr));
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        cfg.jitter = jitter != 0;
        cfg.seed = seed;
        cfg.accumulationPermutation = perm;
        const Camera cam = cameraFrom(k9, r9, t3, width, height);
        const RenderOutput out = render(scene, 0, cam, cfg);
        std::memcpy(rgb, out.color.data.data(), out.color.data.size() * sizeof(float));
        std::memcpy(alpha, out.alpha.data.data(), out.alpha.data.size() * sizeof(float));
        for (size_t i = 0; i < out.sampleCounts.size(); ++i) samples[i] = out.sampleCounts[i];
    });
}

int vpref_look_at(const float *pos, const float *target, const float *up, float focalPx,
                  int32_t width, int32_t height, float *k9, float *r9, float *t3,
                  float *axisAngle3) {
    return guarded([&] {
        const Camera cam = lookAtCamera(v3(pos), v3(target), v3(up), focalPx, width, height);
        put9(k9, cam.intrinsics);
        put9(r9, cam.rotation.matrix);
        put3(t3, cam.translation);
        put3(axisAngle3, cam.rotation.axisAngle);
    });
}

int vpref_generate_ray(const float *k9, const float *r9, const float *t3, int32_t width,
                       int32_t height, float px, float py, float *origin, float *dir) {
    return guarded([&] {
        const Camera cam = cameraFrom(k9, r9, t3, width, height);
        const Ray ray = generateRay(cam, Vec2(px, py));
        put3(origin, ray.origin);
        put3(dir, ray.direction);
    });
}

// Segment list of one ray via the reference's LBVH traversal. Writes up to cap entries and
// returns the total count in *nSeg.
int vpref_intersect(int32_t nPrim, const float *xf15, const float *origin, const float *dir,
                    int32_t cap, int32_t *nSeg, int32_t *prims, float *tEnter, float *tExit,
                    float *tMin, float *tMax) {
    return guarded([&] {
        std::vector<AffineXf> xfs;
        std::vector<Aabb> boxes;
        for (int k = 0; k < nPrim; ++k) {
            xfs.push_back(xfFrom15(xf15 + 15 * size_t(k)));
            boxes.push_back(primitiveAabb(xfs.back()));
        }
        Ray ray;
        ray.origin = v3(origin);
        ray.direction = v3(dir);
        const RaySegmentList segs = intersect(buildLbvh(boxes), xfs, ray);
        *nSeg = int32_t(segs.segments.size());
        for (int i = 0; i < int(segs.segments.size()) && i < cap; ++i) {
            prims[i] = segs.segments[i].primitive;
            tEnter[i] = segs.segments[i].tEnter;
            tExit[i] = segs.segments[i].tExit;
        }
        *tMin = segs.tMin;
        *tMax = segs.tMax;
    });
}

// Per-pixel prim-sample counts of render(): the reference's own generateRay,
// intersect and march per pixel (march.cpp:112-126); march() reports where it stopped
// (MarchResult::lastStep), and the step loop of march.cpp:34-49 is replayed on the reference's
// segment list up to that step, adding the size of the active set at every visited step
// (the executions of march.cpp:63-70). Single-threaded; composes the frame like render().
int vpref_render_prim_counts(int32_t nPrim, int32_t m, const float *tr24, const float *payload, float wAlpha,
                             int32_t wBeta, const float *k9, const float *r9, const float *t3, int32_t width,
                             int32_t height, float stepSize, float earlyEps, int32_t jitter, uint64_t seed,
                             int32_t *prim) {
    return guarded([&] {
        Frame fr;
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        const std::vector<AffineXf> xfs = fr.composed();
        std::vector<Aabb> boxes;
        for (const auto &xf : xfs) boxes.push_back(primitiveAabb(xf));
        const Lbvh bvh = buildLbvh(boxes);
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        const WindowParams w{wAlpha, wBeta};
        const Camera cam = cameraFrom(k9, r9, t3, width, height);
        for (int y = 0; y < height; ++y)
            for (int x = 0; x < width; ++x) {
                const int pixelId = y * width + x;
                const Ray ray = generateRay(cam, Vec2(real(x) + real(0.5), real(y) + real(0.5)));
                const RaySegmentList segs = intersect(bvh, xfs, ray);
                real jitter01 = real(0.5);
                if (jitter) jitter01 = hashToUnit(hashCombine(seed, uint64_t(pixelId)));
                const MarchResult mr = march(ray, segs, fr.slab, xfs, w, cfg, jitter01);
                int64_t count = 0;
                if (!segs.segments.empty() && mr.lastStep >= 0) {
                    const real dt = cfg.stepSize, t0 = segs.tMin;
                    const int nSegs = int(segs.segments.size());
                    std::vector<int> active;
                    int next = 0;
                    for (int64_t i = 0; i <= mr.lastStep; ++i) {
                        const real ts = t0 + (real(i) + jitter01) * dt;
                        if (ts >= segs.tMax) break;
                        while (next < nSegs && segs.segments[next].tEnter <= ts) active.push_back(next++);
                        active.erase(std::remove_if(active.begin(), active.end(),
                                                    [&](int q) { return segs.segments[q].tExit <= ts; }),
                                     active.end());
                        if (active.empty()) {
                            if (next >= nSegs) break;
                            const real tNext = segs.segments[next].tEnter;
                            const int64_t skipTo = int64_t(std::ceil((tNext - t0) / dt - double(jitter01)));
                            if (skipTo > i + 1) i = skipTo - 1;
                            continue;
                        }
                        count += int64_t(active.size());
                    }
                }
                prim[pixelId] = int32_t(count);
            }
    });
}

// march() over arbitrary rays (the reference's lower-level entry point, march.h:42-44).
int vpref_march_rays(int32_t nPrim, int32_t m, const float *xf15, const float *payload,
                     float wAlpha, int32_t wBeta, int64_t nRays, const float *origins,
                     const float *dirs, const float *jitter01, float stepSize, float earlyEps,
                     uint64_t perm, float *rgb, float *alpha, int32_t *samples) {
    return guarded([&] {
        std::vector<AffineXf> xfs;
        std::vector<Aabb> boxes;
        for (int k = 0; k < nPrim; ++k) {
            xfs.push_back(xfFrom15(xf15 + 15 * size_t(k)));
            boxes.push_back(primitiveAabb(xfs.back()));
        }
        PrimitiveSlab slab;
        slab.resize(nPrim, m);
        std::memcpy(slab.payload.data(), payload, slab.payload.size() * sizeof(float));
        const Lbvh bvh = buildLbvh(boxes);
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        cfg.accumulationPermutation = perm;
        const WindowParams w{wAlpha, wBeta};
        for (int64_t r = 0; r < nRays; ++r) {
            Ray ray;
            ray.origin = v3(origins + 3 * r);
            ray.direction = v3(dirs + 3 * r);
            const RaySegmentList segs = intersect(bvh, xfs, ray);
            const MarchResult mr =
                march(ray, segs, slab, xfs, w, cfg, jitter01 ? jitter01[r] : real(0.5));
            put3(rgb + 3 * r, mr.rgb);
            alpha[r] = mr.alpha;
            samples[r] = mr.samples;
        }
    });
}

// backwardRay over explicit rays with given output adjoints; grads (K*4*M^3 + 9K floats,
// the GradBuffer layout of params.h:12-27 with no vertices) are overwritten.
int vpref_backward_rays(int32_t nPrim, int32_t m, const float *tr24, const float *payload,
                        float wAlpha, int32_t wBeta, int64_t nRays, const float *origins,
                        const float *dirs, const float *jitter01, const float *adjRgb,
                        const float *adjAlpha, float stepSize, float earlyEps, float *grads) {
    return guarded([&] {
        Frame fr;
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        const std::vector<AffineXf> xfs = fr.composed();
        std::vector<Aabb> boxes;
        for (const auto &xf : xfs) boxes.push_back(primitiveAabb(xf));
        const Lbvh bvh = buildLbvh(boxes);
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        const WindowParams w{wAlpha, wBeta};
        GradBuffer gb(layoutOf(fr, 0));
        for (int64_t r = 0; r < nRays; ++r) {
            Ray ray;
            ray.origin = v3(origins + 3 * r);
            ray.direction = v3(dirs + 3 * r);
            const RaySegmentList segs = intersect(bvh, xfs, ray);
            backwardRay(ray, segs, fr, xfs, w, cfg, jitter01 ? jitter01[r] : real(0.5),
                        v3(adjRgb + 3 * r), adjAlpha[r], gb);
        }
        std::memcpy(grads, gb.values.data(), gb.values.size() * sizeof(float));
    });
}

// evalLoss (grad.cpp:197-251) with no tracked vertices: cams23 = n_cams * {K[9] R[9] t[3] w h};
// RaySamples given as arrays. terms4 = {pho, geo, vol, del}; grads (nullable) overwritten with
// the GradBuffer (K*4*M^3 + 9K).
int vpref_eval_loss(int32_t nPrim, int32_t m, const float *tr24, const float *payload,
                    float wAlpha, int32_t wBeta, int32_t nCams, const float *cams23, int64_t n,
                    const int32_t *camIndex, const float *pixelXY, const int32_t *pixelId,
                    const float *target, const float *background, float lPho, float lVol,
                    float lDel, float stepSize, float earlyEps, int32_t jitter, uint64_t seed,
                    float *terms4, float *grads) {
    return guarded([&] {
        Scene scene;
        scene.window = WindowParams{wAlpha, wBeta};
        Frame fr;
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        scene.frames.push_back(fr);
        std::vector<Camera> cams;
        for (int c = 0; c < nCams; ++c) {
            const float *q = cams23 + 23 * size_t(c);
            cams.push_back(cameraFrom(q, q + 9, q + 18, int(q[21]), int(q[22])));
        }
        std::vector<RaySample> batch(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            RaySample &rs = batch[size_t(i)];
            rs.cameraIndex = camIndex[i];
            rs.pixel = Vec2(pixelXY[2 * i], pixelXY[2 * i + 1]);
            rs.pixelId = pixelId[i];
            rs.target = v3(target + 3 * i);
            rs.background = v3(background + 3 * i);
        }
        LossWeights w;
        w.pho = lPho;
        w.vol = lVol;
        w.del = lDel;
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        cfg.jitter = jitter != 0;
        cfg.seed = seed;
        GradBuffer gb(layoutOf(scene.frames[0], 0));
        const LossTerms t = evalLoss(scene, 0, cams, batch, {}, w, cfg, grads ? &gb : nullptr);
        terms4[0] = t.pho;
        terms4[1] = t.geo;
        terms4[2] = t.vol;
        terms4[3] = t.del;
        if (grads) std::memcpy(grads, gb.values.data(), gb.values.size() * sizeof(float));
    });
}

// nSteps adamStep calls (losses.cpp:70-104) with the given gradient sequence
// (nSteps * (K*4*M^3 + 9K)); tr24 and the planar payload are updated in place.
int vpref_adam_run(int32_t nPrim, int32_t m, float *tr24, float *payload, int32_t nSteps,
                   const float *grads, const float *cfg6) {
    return guarded([&] {
        Frame fr;
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        const ParamLayout layout = layoutOf(fr, 0);
        AdamConfig c;
        c.lr = cfg6[0];
        c.beta1 = cfg6[1];
        c.beta2 = cfg6[2];
        c.eps = cfg6[3];
        c.lrDeltaScale = cfg6[4];
        c.lrVertexScale = cfg6[5];
        AdamState state(layout.total(), c);
        GradBuffer gb(layout);
        for (int s = 0; s < nSteps; ++s) {
            std::memcpy(gb.values.data(), grads + size_t(s) * layout.total(), layout.total() * sizeof(float));
            adamStep(fr, layout, gb, state);
        }
        std::memcpy(payload, fr.slab.payload.data(), fr.slab.payload.size() * sizeof(float));
        for (int k = 0; k < nPrim; ++k) {
            float *o = tr24 + 24 * size_t(k);
            put3(o + 15, fr.transforms[size_t(k)].deltaT);
            put3(o + 18, fr.transforms[size_t(k)].deltaR);
            put3(o + 21, fr.transforms[size_t(k)].deltaS);
        }
    });
}

// loadSlab into caller memory: *k, *m always; the planar payload when `payload` holds at
// least `cap` floats >= K*4*M^3.
int vpref_load_slab(const char *path, int32_t *k, int32_t *m, float *payload, int64_t cap) {
    return guarded([&] {
        const PrimitiveSlab slab = loadSlab(path);
        *k = slab.numPrimitives;
        *m = slab.voxelsPerAxis;
        if (payload && int64_t(slab.payload.size()) <= cap)
            std::memcpy(payload, slab.payload.data(), slab.payload.size() * sizeof(float));
    });
}

// The §8d synthetic scene ("mvp_shell"), restated on the reference's own types so the reference
// arm never loads the product library. K primitives on a Fibonacci sphere (R = 0.35 m,
// h = R*sqrt(4*pi/K)), frame R_hat = [t b n], pose deltas from mt19937_64(1234) drawn six at a
// time in a fixed order, analytic RGB/sigma fields sampled at voxel-centre world points of the
// composed frame. tests/test_oracle_golden.py pins its output to digests.json["generator"].
int vpref_shell_scene(int32_t nPrim, int32_t m, float *tr24, float *payload) {
    return guarded([&] {
        if (nPrim < 0 || m < 1) throw Error(ErrorCategory::Usage, "shell scene: bad K or M");
        constexpr double pi = 3.14159265358979323846;
        const double radius = 0.35;
        const double h = nPrim > 0 ? radius * std::sqrt(4.0 * pi / nPrim) : 0.0;
        const double sigma0 = nPrim > 0 ? 1.5 / (0.7 * h) : 0.0;
        const double goldenAngle = pi * (3.0 - std::sqrt(5.0));
        std::mt19937_64 gen(1234);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        const size_t vox = size_t(m) * m * m;
        for (int32_t k = 0; k < nPrim; ++k) {
            const double nz = 1.0 - (2.0 * k + 1.0) / nPrim;
            const double rr = std::sqrt(std::max(0.0, 1.0 - nz * nz));
            const double ph = k * goldenAngle;
            const double nx = rr * std::cos(ph), ny = rr * std::sin(ph);
            // tangent = normalize(e_z x n) (fallback e_y), bitangent = n x tangent
            double tx = -ny, ty = nx, tz = 0.0;
            const double len = std::sqrt(tx * tx + ty * ty + tz * tz);
            if (len < 1e-12) {
                tx = 0.0; ty = 1.0; tz = 0.0;
            } else {
                tx /= len; ty /= len; tz /= len;
            }
            const double bx = ny * tz - nz * ty, by = nz * tx - nx * tz, bz = nx * ty - ny * tx;
            double d[6];
            for (double &v : d) v = u(gen);
            PrimitiveTransform pt;
            pt.tBase = Vec3(float(radius * nx), float(radius * ny), float(radius * nz));
            const float cols[9] = {float(tx), float(ty), float(tz), float(bx), float(by), float(bz),
                                   float(nx), float(ny), float(nz)};
            pt.rBase = m3(cols);
            pt.sBase = Vec3(float(0.6 * h), float(0.6 * h), float(0.35 * h));
            pt.deltaT = Vec3(float(0.05 * h * d[3]), float(0.05 * h * d[4]), float(0.05 * h * d[5]));
            pt.deltaR = Vec3(float(0.1 * d[0]), float(0.1 * d[1]), float(0.1 * d[2]));
            pt.deltaS = Vec3(0, 0, 0);
            if (tr24) {
                float *o = tr24 + 24 * size_t(k);
                put3(o + 0, pt.tBase);
                put9(o + 3, pt.rBase);
                put3(o + 12, pt.sBase);
                put3(o + 15, pt.deltaT);
                put3(o + 18, pt.deltaR);
                put3(o + 21, pt.deltaS);
            }
            if (!payload) continue;
            const AffineXf xf = compose(pt);
            float *dst = payload + size_t(k) * 4 * vox;
            for (int zi = 0; zi < m; ++zi)
                for (int yi = 0; yi < m; ++yi)
                    for (int xi = 0; xi < m; ++xi) {
                        const Vec3 pm(-1 + float(2 * xi + 1) / m, -1 + float(2 * yi + 1) / m,
                                      -1 + float(2 * zi + 1) / m);
                        const Vec3 pw = xf.toWorld(pm);
                        const double x = pw.x, y = pw.y, z = pw.z;
                        const size_t at = (size_t(zi) * m + yi) * m + xi;
                        for (int c = 0; c < 3; ++c)
                            dst[c * vox + at] = float(0.5 + 0.45 * std::sin(9 * x + 7 * y * (c + 1) + 5 * z));
                        dst[3 * vox + at] = float(sigma0 * (0.5 + 0.5 * std::sin(11 * x + 13 * y + 3 * z)));
                    }
        }
    });
}

// lookAtCamera (synthetic.cpp:15-38) at the §8d positions: view < 0 is the headline camera at
// (0.25, 0.15, -1.1); otherwise view v of an n-view ring (az = 2*pi*v/n, el = 0.35*sin(3*az),
// radius 1.1). Target the origin, up +y, f = 1.2*W, square W x W image.
int vpref_shell_camera(int32_t view, int32_t nViews, int32_t width, float *k9, float *r9, float *t3) {
    return guarded([&] {
        if (width <= 0 || (view >= 0 && (nViews <= 0 || view >= nViews)))
            throw Error(ErrorCategory::Usage, "shell camera: bad view");
        Vec3 pos(0.25f, 0.15f, -1.1f);
        if (view >= 0) {
            constexpr double pi = 3.14159265358979323846;
            const double az = 2.0 * pi * view / nViews;
            const double el = 0.35 * std::sin(3.0 * az);
            pos = Vec3(float(1.1 * std::cos(el) * std::sin(az)), float(1.1 * std::sin(el)),
                       float(-1.1 * std::cos(el) * std::cos(az)));
        }
        const Camera cam = lookAtCamera(pos, Vec3(0, 0, 0), Vec3(0, 1, 0), float(1.2 * width), width, width);
        put9(k9, cam.intrinsics);
        put9(r9, cam.rotation.matrix);
        put3(t3, cam.translation);
    });
}

// A resident one-frame Scene. The handle owns a volprim::Scene built once; vpref_scene_render
// then runs volprim::render on it and nothing else is inside the call except the optional
// copies into caller arrays (null pointers skip them) and the sum of the sample counts.
struct RefScene {
    Scene scene;
};

void *vpref_scene_new(int32_t nPrim, int32_t m, const float *tr24, const float *payload, float wAlpha,
                      int32_t wBeta) {
    RefScene *rs = nullptr;
    const int rc = guarded([&] {
        auto owned = std::make_unique<RefScene>();
        owned->scene.window = WindowParams{wAlpha, wBeta};
        Frame fr;
        fr.transforms.reserve(size_t(nPrim));
        for (int k = 0; k < nPrim; ++k) fr.transforms.push_back(transformFrom24(tr24 + 24 * size_t(k)));
        fr.slab.resize(nPrim, m);
        std::memcpy(fr.slab.payload.data(), payload, fr.slab.payload.size() * sizeof(float));
        owned->scene.frames.push_back(std::move(fr));
        rs = owned.release();
    });
    return rc == 0 ? rs : nullptr;
}

// The shell scene generated straight into a resident Scene (no 268 MB round trip through Python).
void *vpref_scene_new_shell(int32_t nPrim, int32_t m, float wAlpha, int32_t wBeta) {
    std::vector<float> tr(size_t(nPrim) * 24), pay(size_t(nPrim) * 4 * size_t(m) * m * m);
    if (vpref_shell_scene(nPrim, m, tr.data(), pay.data()) != 0) return nullptr;
    return vpref_scene_new(nPrim, m, tr.data(), pay.data(), wAlpha, wBeta);
}

void vpref_scene_free(void *h) { delete static_cast<RefScene *>(h); }

int vpref_scene_render(void *h, const float *k9, const float *r9, const float *t3, int32_t width,
                       int32_t height, float stepSize, float earlyEps, int32_t jitter, uint64_t seed,
                       float *rgb, float *alpha, int32_t *samples, int64_t *totalSamples) {
    return guarded([&] {
        if (!h) throw Error(ErrorCategory::Usage, "null scene");
        MarchConfig cfg;
        cfg.stepSize = stepSize;
        cfg.earlyEps = earlyEps;
        cfg.jitter = jitter != 0;
        cfg.seed = seed;
        const Camera cam = cameraFrom(k9, r9, t3, width, height);
        const RenderOutput out = render(static_cast<RefScene *>(h)->scene, 0, cam, cfg);
        if (totalSamples) *totalSamples = int64_t(out.totalSamples());
        if (rgb) std::memcpy(rgb, out.color.data.data(), out.color.data.size() * sizeof(float));
        if (alpha) std::memcpy(alpha, out.alpha.data.data(), out.alpha.data.size() * sizeof(float));
        if (samples)
            for (size_t i = 0; i < out.sampleCounts.size(); ++i) samples[i] = out.sampleCounts[i];
    });
}

float vpref_window(float x, float y, float z, float wAlpha, int32_t wBeta) {
    return window(Vec3(x, y, z), WindowParams{wAlpha, wBeta});
}

} // extern "C"
