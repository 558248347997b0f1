// volprim_render_b200.cpp — the adapter a volprim maintainer adds to route the reference's
// renderer through libvpb.so. It is compiled against the reference's
// own headers and types; nothing here is copied from the reference.
//
//   RenderOutput volprim::render_b200(const Scene&, int frame, const Camera&, const MarchConfig&)
//
// has exactly the contract of volprim::render (march.h:59, march.cpp:95-132): same inputs,
// same RenderOutput layout, volprim::Error(Usage) for a bad frame index or a non-positive
// composed scale (march.cpp:96-97, primitive.cpp:44-45). Device failures surface as
// std::runtime_error. To make it *the* render(), rename it and drop march.cpp's definition.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "vpb.h"
#include "volprim/errors.h"
#include "volprim/march.h"
#include "volprim/scene.h"

static_assert(sizeof(volprim::real) == sizeof(float),
              "libvpb renders the binary32 build of volprim (VOLPRIM_USE_DOUBLE is not supported)");

namespace volprim {

namespace {

void check(int rc, const vp_ctx *ctx) {
    if (rc == VP_OK) return;
    const std::string msg = vp_last_error(ctx);
    if (rc == VP_ERR_USAGE) throw Error(ErrorCategory::Usage, msg);
    if (rc == VP_ERR_NUMERIC) throw Error(ErrorCategory::Numeric, msg);
    throw std::runtime_error("libvpb: " + msg);
}

struct Context {  // one context per host thread (a vp_ctx is not thread-safe)
    vp_ctx *ctx = nullptr;
    Context() { check(vp_create(0, &ctx), nullptr); }
    ~Context() { vp_destroy(ctx); }
};

void put(float *dst, const Vec3 &v) {
    dst[0] = v.x;
    dst[1] = v.y;
    dst[2] = v.z;
}

}  // namespace

RenderOutput render_b200(const Scene &scene, int frame, const Camera &cam, const MarchConfig &cfg) {
    if (frame < 0 || frame >= int(scene.frames.size()))
        throw Error(ErrorCategory::Usage, "frame index out of range");
    const Frame &fr = scene.frames[frame];
    const int k = int(fr.transforms.size());
    std::vector<float> tr(size_t(k) * 24), xf(size_t(k) * 15);
    for (int i = 0; i < k; ++i) {
        const PrimitiveTransform &t = fr.transforms[size_t(i)];
        float *r = tr.data() + size_t(i) * 24;
        put(r + 0, t.tBase);
        std::memcpy(r + 3, t.rBase.m, 9 * sizeof(float));
        put(r + 12, t.sBase);
        put(r + 15, t.deltaT);
        put(r + 18, t.deltaR);
        put(r + 21, t.deltaS);
    }
    check(vp_compose(k, tr.data(), xf.data()), nullptr);  // Frame::composed()

    static thread_local Context c;
    check(vp_set_scene(c.ctx, k, fr.slab.voxelsPerAxis, xf.data(), fr.slab.payload.data(),
                       scene.window.alpha, scene.window.beta),
          c.ctx);
    vp_camera vc{};
    std::memcpy(vc.K, cam.intrinsics.m, sizeof vc.K);
    std::memcpy(vc.R, cam.rotation.matrix.m, sizeof vc.R);
    put(vc.t, cam.translation);
    vc.width = cam.width;
    vc.height = cam.height;
    vp_march vm{};
    vm.step_size = cfg.stepSize;
    vm.early_eps = cfg.earlyEps;
    vm.jitter = cfg.jitter ? 1 : 0;
    vm.seed = cfg.seed;
    vm.accumulation_permutation = cfg.accumulationPermutation;

    RenderOutput out;
    out.color = Image(cam.width, cam.height, 3);
    out.alpha = Image(cam.width, cam.height, 1);
    out.sampleCounts.assign(size_t(cam.width) * cam.height, 0);
    static_assert(sizeof(int) == sizeof(int32_t), "sample counts are int32 on the boundary");
    check(vp_render(c.ctx, &vc, &vm, out.color.data.data(), out.alpha.data.data(),
                    reinterpret_cast<int32_t *>(out.sampleCounts.data()), nullptr),
          c.ctx);
    return out;
}

}  // namespace volprim
