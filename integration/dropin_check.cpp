// dropin_check.cpp — renders the same scene with the reference's volprim::render (CPU) and
// with volprim::render_b200 (the adapter over libvpb.so) and compares the outputs bitwise.
// Built by oracle/Makefile (target `dropin`) against the reference sources; run on a B200:
//     oracle/_ref/dropin_check [K M W]
#include <algorithm>
#include <chrono>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "volprim/errors.h"
#include "volprim/march.h"
#include "volprim/scene.h"
#include "volprim/synthetic.h"
#include "vpb.h"

namespace volprim {
RenderOutput render_b200(const Scene &scene, int frame, const Camera &cam, const MarchConfig &cfg);
}
using namespace volprim;

int main(int argc, char **argv) {
    const int k = argc > 1 ? std::atoi(argv[1]) : 64;
    const int m = argc > 2 ? std::atoi(argv[2]) : 16;
    const int w = argc > 3 ? std::atoi(argv[3]) : 256;
    std::vector<float> tr(size_t(k) * 24), pay(size_t(k) * 4 * m * m * m);
    if (vp_make_shell_scene(k, m, tr.data(), pay.data()) != VP_OK) return 2;
    Scene scene;
    Frame fr;
    for (int i = 0; i < k; ++i) {
        const float *r = tr.data() + size_t(i) * 24;
        PrimitiveTransform t;
        t.tBase = Vec3(r[0], r[1], r[2]);
        for (int q = 0; q < 9; ++q) t.rBase.m[q] = r[3 + q];
        t.sBase = Vec3(r[12], r[13], r[14]);
        t.deltaT = Vec3(r[15], r[16], r[17]);
        t.deltaR = Vec3(r[18], r[19], r[20]);
        t.deltaS = Vec3(r[21], r[22], r[23]);
        fr.transforms.push_back(t);
    }
    fr.slab.resize(k, m);
    std::memcpy(fr.slab.payload.data(), pay.data(), pay.size() * sizeof(float));
    scene.frames.push_back(fr);
    const Camera cam = lookAtCamera(Vec3(0.25f, 0.15f, -1.1f), Vec3(0, 0, 0), Vec3(0, 1, 0),
                                    real(1.2) * w, w, w);
    const MarchConfig cfg;
    auto t0 = std::chrono::steady_clock::now();
    const RenderOutput a = render(scene, 0, cam, cfg);
    auto t1 = std::chrono::steady_clock::now();
    const RenderOutput b = render_b200(scene, 0, cam, cfg);  // cold: context, buffers, threads
    // warm calls as a render loop makes them: each call's RenderOutput replaces the last one
    std::vector<double> warm;
    RenderOutput c;
    for (int i = 0; i < 7; ++i) {
        auto t2 = std::chrono::steady_clock::now();
        c = render_b200(scene, 0, cam, cfg);
        auto t3 = std::chrono::steady_clock::now();
        warm.push_back(std::chrono::duration<double, std::milli>(t3 - t2).count());
    }
    std::sort(warm.begin(), warm.end());
    const bool same = a.color.data == c.color.data && a.alpha.data == c.alpha.data &&
                      a.sampleCounts == c.sampleCounts && b.color.data == c.color.data;
    std::printf("dropin K=%d M=%d %dx%d: reference %.1f ms, render_b200 %.3f ms (warm, median of 7, incl. "
                "payload upload and RenderOutput allocation), samples %lld vs %lld, bitwise %s\n",
                k, m, w, w, std::chrono::duration<double, std::milli>(t1 - t0).count(), warm[3],
                (long long)a.totalSamples(), (long long)c.totalSamples(), same ? "IDENTICAL" : "DIFFERENT");
    bool threw = false;
    try {
        render_b200(scene, 1, cam, cfg);
    } catch (const Error &e) {
        threw = e.category() == ErrorCategory::Usage;
    }
    std::printf("bad frame index -> volprim::Error(Usage): %s\n", threw ? "yes" : "NO");
    return same && threw ? 0 : 1;
}
