// vpb_ctx_internal.h — the narrow view of a vp_ctx that the other host modules of libvpb
// (vpb_comm.cpp) use; the context itself stays private to vpb_api.cpp. Internal header.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

struct vp_ctx;
struct float4;

namespace vpb {

// The resident scene's device buffers (composed transforms, 16 floats per primitive; the
// channel-interleaved payload, K * M^3 float4s) and the context's device / stream.
struct CtxScene {
    float *xf16;
    float4 *payload;
    int n_prim, m, device;
    cudaStream_t stream;
};
// The CUDA device the context was created on.
int ctx_device(const vp_ctx *ctx);
// VP_ERR_USAGE when the context holds no scene (vp_set_scene first).
int ctx_scene(vp_ctx *ctx, CtxScene *out);
// The scene's transforms and payload are written on `st` by another agent (a broadcast): the
// context's derived state (BVH, the raymarch's pair layout) is stale, the transforms count as
// set, and the context's next call that uses the scene makes its streams wait for `st`'s work
// enqueued by then (so a broadcast launched only at a caller's vp_group_end is covered).
int ctx_scene_written(vp_ctx *ctx, cudaStream_t st);
// `st` (a former scene writer) is about to be destroyed after a synchronize: forget it.
void ctx_drop_writer(vp_ctx *ctx, cudaStream_t st);
// Make `st` wait for the context's renders enqueued so far (their device outputs complete).
int ctx_wait_renders(vp_ctx *ctx, cudaStream_t st);
// Error reporting shared with vpb_api.cpp (vp_last_error).
int ctx_fail(vp_ctx *ctx, int code, const std::string &msg);

}  // namespace vpb
