/* vpb.h — C-ABI of the B200-native MVP raymarcher (libvpb.so).
 *
 * Drop-in boundary for the reference's forward raymarcher:
 *
 *   RenderOutput volprim::render(const Scene &, int frame, const Camera &, const MarchConfig &)
 *     (/root/reference/proj/src/volprim/march.h:59, body march.cpp:95-132)
 *
 * The reference has no FFI of its own (it is a C++ library); these are the
 * entry points a C++ caller binds through a thin adapter. Plain
 * pointers and sizes only. Every entry point returns an int status that mirrors
 * volprim::ErrorCategory (errors.h:11-17): 0 ok, 2 usage, 6 numeric, plus 7 for a CUDA /
 * device failure. vp_last_error() returns the message of the last failure on a context
 * (or of the last context-free call when ctx is NULL).
 *
 * Flat layouts (matrices are column-major exactly like volprim::Mat3::m, math.h:71-73):
 *   PrimitiveTransform (primitive.h:45-52) = 24 floats
 *       tBase[3] rBase[9] sBase[3] deltaT[3] deltaR[3] deltaS[3]
 *   AffineXf (primitive.h:56-64)           = 15 floats  t[3] rot[9] scale[3]
 *   PrimitiveSlab payload (primitive.h:25-41) = K*4*M^3 floats, planar (k, channel, z, y, x)
 *   Image outputs (image.h:14-25): rgb H*W*3 interleaved, alpha H*W, samples H*W (int32)
 *
 * Output / input pointers may be host memory (pageable or pinned) or device memory of the
 * context's device; the library detects which (cudaPointerGetAttributes). A context is not
 * thread-safe: use one context per device per host thread (the reference render() is
 * re-entrant because it holds no state; here the state is the resident scene).
 */
#ifndef VPB_H
#define VPB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPB_VERSION 1

enum {
    VP_OK = 0,
    VP_ERR_USAGE = 2,   /* ErrorCategory::Usage   (errors.h:12) */
    VP_ERR_IO = 3,      /* ErrorCategory::Io      (errors.h:13) */
    VP_ERR_FORMAT = 4,  /* ErrorCategory::Format  (errors.h:14) */
    VP_ERR_VERSION = 5, /* ErrorCategory::Version (errors.h:15) */
    VP_ERR_NUMERIC = 6, /* ErrorCategory::Numeric (errors.h:16) */
    VP_ERR_DEVICE = 7   /* CUDA / device failure (no reference counterpart) */
};

typedef struct vp_ctx vp_ctx;

/* volprim::Camera (camera.h:21-29): intrinsics K, world-to-camera rotation R and
 * translation t (x_cam = R x_world + t), image size. Rotation::axisAngle is not read by
 * render() and is therefore not part of the boundary. */
typedef struct vp_camera {
    float K[9];
    float R[9];
    float t[3];
    int32_t width;
    int32_t height;
} vp_camera;

/* volprim::MarchConfig (march.h:11-20). accumulation_permutation is the reference's test
 * hook; a non-zero value returns VP_ERR_USAGE. */
typedef struct vp_march {
    float step_size;   /* metres, > 0 */
    float early_eps;   /* terminate once T > 1 - early_eps */
    int32_t jitter;    /* 0/1: per-pixel hashToUnit(hashCombine(seed, pixelId)) offset */
    int32_t reserved;
    uint64_t seed;
    uint64_t accumulation_permutation;
} vp_march;

/* Per-render counters (device atomics; the reference's only diagnostic is the per-pixel
 * sample count, march.h:49-55). */
typedef struct vp_stats {
    int64_t ray_samples;   /* sum of per-pixel samples (RenderOutput::totalSamples) */
    int64_t prim_samples;  /* primitive evaluations (body of march.cpp:63-70) */
    int64_t hit_rays;      /* rays with a non-empty segment list */
    int64_t early_exits;   /* rays stopped by T > 1 - eps (march.cpp:87) */
    int64_t saturated;     /* rays stopped by the saturation clamp (march.cpp:75-84) */
    int64_t overflow_rays; /* rays re-marched by the wide-window fallback kernel */
    int64_t keys;          /* (tile, depth) keys emitted by the binning pass */
    int64_t refills;       /* per-ray window refills (rays with > window hits) */
    float ms;              /* device time of the render (CUDA events), ms */
    int32_t huge_rays;     /* rays marched by the last-resort pass (> 256 live segments) */
} vp_stats;

int vp_version(void);

/* ---- context ------------------------------------------------------------------------- */
int vp_create(int32_t device, vp_ctx **out);
int vp_destroy(vp_ctx *ctx);
const char *vp_last_error(const vp_ctx *ctx);
/* The CUDA stream the context launches on (cudaStream_t as void*). */
void *vp_stream(vp_ctx *ctx);

/* ---- host-side scene preparation (exact reference arithmetic, no device work) --------- */
/* Frame::composed() / compose() (scene.h:19-24, primitive.cpp:41-49): 24 -> 15 floats per
 * primitive. VP_ERR_USAGE on a non-positive composed scale, like the reference. */
int vp_compose(int32_t n_prim, const float *transforms24, float *xf15);

/* ---- resident scene ---------------------------------------------------------------------
 * Uploads a frame: composed transforms and the planar slab, which kernel K0 repacks on the
 * device into channel-interleaved float4 voxels (k, z, y, x, rgba). window = WindowParams
 * (primitive.h:14-17). VP_ERR_USAGE on K < 0, M < 1 (when K > 0), odd or negative beta,
 * non-positive scale. xf15 may be NULL: the transforms then come from vp_set_frame (or
 * vp_set_transforms) before the first render. */
int vp_set_scene(vp_ctx *ctx, int32_t n_prim, int32_t m, const float *xf15,
                 const float *payload_planar, float window_alpha, int32_t window_beta);
/* Replace only the transforms (same K), e.g. a new frame with the same payload. */
int vp_set_transforms(vp_ctx *ctx, int32_t n_prim, const float *xf15);
/* Stream-ordered variant (cudaStream_t `stream`, NULL = the context's): the upload waits for
 * the binning and raymarch of the previous render (they read the old transforms), and later
 * renders wait for it. xf15 host (page-locked for
 * overlap) or device; it must stay valid until the copy has run. Unlike vp_set_transforms
 * it does not re-check the scales (the caller's records were composed by vp_compose). */
int vp_set_transforms_async(vp_ctx *ctx, int32_t n_prim, const float *xf15, void *stream);
/* Frame::composed() on the device (scene.h:19-24, primitive.cpp:41-49, rotation.cpp:8-27):
 * takes the frame's PrimitiveTransform records (K*24 floats, host or device) and composes
 * them into the resident transforms, bit-identical to vp_compose (the device restates glibc
 * sinf/cosf). The records stay resident for vp_adam_step. Same K as the resident scene;
 * vp_set_scene may be called with xf15 = NULL first. VP_ERR_USAGE on a non-positive
 * composed scale. */
int vp_set_frame(vp_ctx *ctx, int32_t n_prim, const float *transforms24);
/* Copy the resident composed transforms out as K*15 floats (host or device). */
int vp_get_transforms(vp_ctx *ctx, float *xf15);
/* Adopt an already-interleaved payload (K*M^3 float4 = K*M^3*4 floats, host or device),
 * e.g. after an NCCL broadcast of the repacked buffer. Keeps the current transforms. */
int vp_set_payload_interleaved(vp_ctx *ctx, int32_t n_prim, int32_t m,
                               const float *payload_interleaved);
/* loadSlab (scene_io.cpp:43-66; VPSL format, README.md:96-104) straight into the device
 * layout: the file is streamed through double-buffered pinned chunks, copied and repacked
 * (K0) chunk by chunk, so the planar slab never exists whole in host or device memory.
 * xf15 are the frame's composed transforms (n_prim must equal the file's K). Errors as the
 * reference: VP_ERR_IO (cannot open), VP_ERR_FORMAT (magic, truncation, implausible header:
 * K = 0 or > 2^20, M = 0 or > 512), VP_ERR_VERSION (version != 1). */
int vp_load_slab(vp_ctx *ctx, const char *path, int32_t n_prim, const float *xf15,
                 float window_alpha, int32_t window_beta);

/* Device pointer / float count of the resident interleaved payload (for broadcasts). */
int vp_payload_device(vp_ctx *ctx, float **dev_ptr, int64_t *n_floats);
/* Copy the resident interleaved payload to dst (host or device, K*M^3*4 floats). */
int vp_copy_payload(vp_ctx *ctx, float *dst);
/* (vp_set_scene accepts payload_planar == NULL: the payload is then allocated but
 *  undefined until vp_set_payload_interleaved.) */

/* ---- render (the drop-in for volprim::render) --------------------------------------------
 * Synchronous. rgb: H*W*3, alpha: H*W, samples: H*W (nullable), stats nullable. */
int vp_render(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, float *rgb,
              float *alpha, int32_t *samples, vp_stats *stats);
/* Asynchronous variant, enqueued on `stream` (cudaStream_t; NULL = the context's stream).
 * Outputs are all device pointers (stream-ordered) or all host pointers (page-locked for
 * overlap): then the view renders into one of two device slots and its device->host copy
 * runs on an internal copy stream while the next view renders; call vp_sync before reading
 * them. samples nullable. Counters can be read afterwards with vp_read_stats. */
int vp_render_async(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, float *rgb,
                    float *alpha, int32_t *samples, void *stream);
/* A batch of 1..16 views of the resident frame in ONE raymarch launch (the tiles of all views
 * heaviest first, so the batch pays the launch's tail once; e.g. the 64-view ring in 4..8
 * calls), enqueued on `stream`. Outputs are arrays of all device or all host pointers (samples
 * may be NULL); host outputs (page-locked for overlap) are copied out while the next batch
 * renders: call vp_sync before reading them. vp_read_stats afterwards reports the last view. */
int vp_render_batch_async(vp_ctx *ctx, int32_t n_views, const vp_camera *cams, const vp_march *cfg,
                          float *const *rgb, float *const *alpha, int32_t *const *samples, void *stream);
/* One shard of a view split over n_shards renders (tile sharding across GPUs, SURVEY.md §8e;
 * the reference renders a view in one call, march.cpp:95-132, and parallelises over rows,
 * threads.h:16-36). The shard owns the 16x16 tiles t (row-major tile index, tiles_x =
 * ceil(W/16)) with t % n_shards == shard: it culls every primitive, but bins and marches only
 * its tiles, heaviest first. Outputs are DEVICE pointers in a tile-major layout of
 * vp_shard_tiles() slots of 256 pixels: pixel (x, y) of owned tile t is at slot t / n_shards,
 * offset (y % 16) * 16 + x % 16 (rgb 3 floats, alpha 1 float, samples 1 int32 per pixel);
 * pixels of partial edge tiles outside the image are not written. Every pixel value is
 * bitwise the one vp_render_async produces. Enqueued on `stream` (NULL: the context's). */
int vp_render_shard_async(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, int32_t shard,
                          int32_t n_shards, float *rgb, float *alpha, int32_t *samples, void *stream);
/* Number of tile slots of shard `shard` of n_shards for a width x height view. */
int64_t vp_shard_tiles(int32_t width, int32_t height, int32_t shard, int32_t n_shards);
/* Capacity (keys) of each view's tile-key buffer (K3's (tile, depth) entries); 0 restores the
 * default max(2^20, 16 K). A view whose keys do not all fit still renders exactly: the tiles
 * whose buckets overflow are marched by the fallback kernel from all K primitives' pixel
 * rectangles (slower). With grow != 0 the capacity then follows the largest key count seen
 * (without waiting on the device); grow == 0 keeps it fixed (memory-bounded callers, tests). */
int vp_set_key_capacity(vp_ctx *ctx, int64_t keys, int32_t grow);
/* Waits for every render and output copy the context has enqueued. */
int vp_sync(vp_ctx *ctx);
int vp_read_stats(vp_ctx *ctx, vp_stats *stats);
/* Device durations (CUDA events on the launching stream) of the raymarch kernels (K5 + K5b)
 * of the renders enqueued since the previous call, oldest first, at most the last 256.
 * Synchronises on those events; *n receives the count written. */
int vp_kernel_times(vp_ctx *ctx, int64_t max, float *march_ms, int64_t *n);

/* march() over arbitrary rays (march.h:42-44 with intersect(), lbvh.cpp:207-234, as the
 * candidate source over all K primitives). jitter01 nullable (0.5). Synchronous. */
int vp_march_rays(vp_ctx *ctx, int64_t n_rays, const float *origins, const float *dirs,
                  const float *jitter01, const vp_march *cfg, float *rgb, float *alpha,
                  int32_t *samples);

/* backwardRay (grad.cpp:34-195) for a batch of rays through the resident frame, given the
 * output adjoints adj_rgb (n*3, dLoss/d rgb) and adj_alpha (n, dLoss/d alpha), exactly the
 * values evalLoss passes (grad.cpp:240-248). transforms24 are the frame's PrimitiveTransform
 * records (K*24): rBase and deltaR enter the rotation Jacobians; they must compose to the
 * resident transforms. grads (host or device) holds K*4*M^3 + 9*K floats in the GradBuffer
 * layout (params.h:12-27): the planar payload gradient, then deltaT[3] deltaR[3] deltaS[3]
 * per primitive. accumulate != 0 adds into it, else it is overwritten. Per-sample terms
 * match the reference bit for bit; the global sums use device atomics, so their summation
 * order (and last bits) differ from the reference's sequential loop. Synchronous. */
int vp_backward_rays(vp_ctx *ctx, int64_t n_rays, const float *origins, const float *dirs,
                     const float *jitter01, const float *adj_rgb, const float *adj_alpha,
                     const vp_march *cfg, const float *transforms24, float *grads,
                     int32_t accumulate);

/* ---- training rows ------------------------------------------------------
 * evalLoss's ray-batch part (grad.cpp:197-251): for each RaySample i (fit.cpp:85-113) the ray
 * of camera cams[cam_index[i]] through pixel_xy[i] (generateRay, camera.cpp:14-23), evalLoss's
 * jitter hash of (cam_index, pixel_id) (grad.cpp:222-225), march(), composite with
 * background[i], L_pho = lambda * mean |composited - target|^2 (losses.cpp:12-25) into
 * *loss_pho, the composited pixels (nullable), and, when grads != NULL, backwardRay of every
 * ray with the photometric adjoints into grads (layout and accumulate as vp_backward_rays).
 * VP_ERR_USAGE on an empty batch, a bad camera index or a pixel outside its image. */
int vp_eval_loss_pho(vp_ctx *ctx, int32_t n_cams, const vp_camera *cams, int64_t n,
                     const int32_t *cam_index, const float *pixel_xy, const int32_t *pixel_id,
                     const float *target, const float *background, float lambda_pho,
                     const vp_march *cfg, const float *transforms24, float *loss_pho,
                     float *composited, float *grads, int32_t accumulate);

/* lossVol + lossDel (losses.cpp:45-68) on the host; grad_pose (9 floats per primitive,
 * nullable) accumulates +=. */
int vp_loss_pose(int32_t n_prim, const float *transforms24, float lambda_vol, float lambda_del,
                 float *loss_vol, float *loss_del, float *grad_pose);
/* lossGeo (losses.cpp:27-43) on the host; offsets nullable; grad_verts (n*3) accumulates. */
int vp_loss_geo(int32_t n_verts, const float *base, const float *offsets, const float *tracked,
                float lambda, float *loss, float *grad_verts);

/* AdamConfig (losses.h:34-44). */
typedef struct vp_adam {
    float lr, beta1, beta2, eps, lr_delta_scale, lr_vertex_scale;
} vp_adam;
/* adamStep (losses.cpp:70-104) on the resident frame over [payload | 9K deltas] (no guide-
 * mesh vertices): grads (host or device, vp_backward_rays layout). The payload is updated and
 * projected (>= 0) in place on the device; the deltas are updated in transforms24 (host,
 * K*24, in/out), composed scales projected to >= 1e-4, and the frame recomposed and
 * re-uploaded. Moments persist in the context (AdamState) until vp_adam_reset or a frame of
 * a different size. VP_ERR_NUMERIC (and no update) on a non-finite gradient: the payload,
 * moments, step count and transforms24 are untouched, and the resident records are the
 * caller's (the resident composition is unchanged). VP_ERR_USAGE when a composed scale is
 * still non-positive after the projection (the reference's Frame::composed() would throw at the
 * next use, primitive.cpp:44-45): the step IS committed (payload, moments, step count and the
 * deltas in transforms24), but the frame is not recomposed and renders fail until valid
 * transforms are set. grads: device pointers need no alignment (16-byte aligned ones take the
 * vectorised update). */
int vp_adam_step(vp_ctx *ctx, const vp_adam *cfg, const float *grads, float *transforms24);
int vp_adam_reset(vp_ctx *ctx);

/* composite() (march.cpp:134-147): out = A*I + (1-A)*B, all H*W(*3) arrays. */
int vp_composite(vp_ctx *ctx, int32_t width, int32_t height, const float *rgb,
                 const float *alpha, const float *background, float *out);

/* ---- binning artefacts (parity checks of cull / keys / per-tile sorted lists) -----------
 * rect4: K*4 {tx0,ty0,tx1,ty1} (empty = {0,0,-1,-1}); depth_key: K; tile_offsets:
 * n_tiles+1; tile_prims: up to cap entries. *n_keys receives the total. Synchronous. */
int vp_debug_tiles(vp_ctx *ctx, const vp_camera *cam, int32_t *rect4, uint32_t *depth_key,
                   int32_t *tile_offsets, int32_t *tile_prims, int64_t cap, int64_t *n_keys);

/* Profiling hook: renders the view with a per-CTA timeline of the raymarch kernel; out gets
 * 4 uint64 per CTA in launch order: tile index, SM id, start and end (%globaltimer ns).
 * *n_out receives the CTA count (= tiles). */
int vp_debug_tile_times(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, uint64_t *out,
                        int64_t cap, int64_t *n_out);

/* Test hook: evaluates the device port of glibc expf used by window() (primitive.cpp:27)
 * elementwise, so the port can be checked exhaustively against the host libm. */
int vp_debug_expf(vp_ctx *ctx, int64_t n, const float *x, float *y);
/* Test hook: the device LBVH's stable radix sort (vpb_bvh.cu) of n 64-bit keys on bits [32, 62),
 * host arrays (the replacement of buildLbvh's std::sort, lbvh.cpp:81-100). */
int vp_debug_radix_sort(vp_ctx *ctx, int64_t n, const uint64_t *keys_in, uint64_t *keys_out);
/* Test hook: the device port of glibc sinf (which = 0) / cosf (which = 1) used by the
 * device compose (rotationFromAxisAngle, rotation.cpp:19-22), elementwise. */
int vp_debug_sincos(vp_ctx *ctx, int64_t n, const float *x, float *y, int32_t which);
/* Test hook: backwardRay's per-primitive pose data (rBase[9], then rotationDerivative of
 * deltaR for i = 0, 1, 2, rotation.cpp:30-38; 36 floats per primitive) from K*24 host records,
 * computed by the device kernel (on_device = 1) or the host restatement (0). */
int vp_debug_pose(vp_ctx *ctx, int32_t n_prim, const float *transforms24, float *out36, int32_t on_device);

/* ---- multi-GPU: NCCL over NVLink / NVSwitch inside libvpb -----------------
 * The path shards by view or image tile with no data-path collective; the only traffic is one
 * broadcast of the scene and the gather of outputs to a root. The reference parallelises over
 * rows inside one process (threads.h:16-36, used at march.cpp:112); these calls are its
 * multi-GPU counterpart, for C++ callers of the drop-in (no torch needed). A vp_comm belongs
 * to one context (its device); collectives run on the communicator's own stream. */
#define VP_COMM_ID_BYTES 128
typedef struct vp_comm vp_comm;
/* A fresh NCCL unique id (VP_COMM_ID_BYTES); rank 0 creates it and shares it out of band. */
int vp_comm_unique_id(uint8_t *id);
/* One process per GPU: joins the n_ranks communicator as `rank` on ctx's device. max_ctas > 0
 * caps NCCL's CTAs (ncclConfig_t.maxCTAs) so a gather overlapping the next raymarch takes few
 * SMs; 0 = NCCL's default. */
int vp_comm_init(vp_ctx *ctx, const uint8_t *id, int32_t n_ranks, int32_t rank, int32_t max_ctas,
                 vp_comm **out);
/* One process driving n GPUs: ctxs[i] (created on devices[i]) becomes rank i of one
 * communicator (the ncclCommInitAll pattern); out receives n communicators. Collectives of this
 * mode are issued for every rank between vp_group_start and vp_group_end. */
int vp_comm_init_all(int32_t n, vp_ctx *const *ctxs, const int32_t *devices, int32_t max_ctas, vp_comm **out);
/* Destroy a communicator before the context it was created for. */
int vp_comm_destroy(vp_comm *comm);
int vp_group_start(void);
int vp_group_end(void);
/* Every rank first calls vp_set_scene with the same K and M: the root with its transforms and
 * payload, the others with NULL for both (shape only). Then the root's composed transforms and
 * repacked interleaved payload are broadcast, so only the root runs K0. Stream-ordered: the
 * other ranks' next renders wait for the broadcast. */
int vp_broadcast_scene(vp_comm *comm, int32_t root);
/* Gathers n_views rendered views of every rank to the root in one NCCL group, after the
 * context's renders so far. rgb/alpha/samples: this rank's n_views DEVICE outputs of n_px
 * pixels (samples NULL on every rank or on none). dst_*: on the root, n_ranks * n_views device
 * pointers (rank r's view j at r * n_views + j; the root's own views are copied on the device),
 * NULL on the other ranks. Asynchronous: see vp_comm_wait / vp_comm_sync. */
int vp_gather_views(vp_comm *comm, int32_t root, int32_t n_views, int64_t n_px, float *const *rgb,
                    float *const *alpha, int32_t *const *samples, float *const *dst_rgb, float *const *dst_alpha,
                    int32_t *const *dst_samples);
/* `stream` (NULL: the context's) waits for the communicator's work so far (e.g. before a render
 * overwrites outputs a gather is still sending). */
int vp_comm_wait(vp_comm *comm, void *stream);
/* Blocks until the communicator's work so far has completed. */
int vp_comm_sync(vp_comm *comm);
/* Message of the last failing vp_comm_* / vp_group_* call made without a context. */
const char *vp_comm_last_error(void);

/* ---- synthetic benchmark inputs ("mvp_shell"), host only ------------------ */
/* transforms24: K*24, payload_planar: K*4*M^3 (either may be NULL to skip). */
int vp_make_shell_scene(int32_t n_prim, int32_t m, float *transforms24, float *payload_planar);
/* lookAtCamera (synthetic.cpp:15-38). axis_angle nullable. */
int vp_look_at_camera(const float *position, const float *target, const float *up,
                      float focal_px, int32_t width, int32_t height, vp_camera *out,
                      float *axis_angle);
/* view < 0: the single headline view; else view v of the n_views ring. */
int vp_shell_camera(int32_t view, int32_t n_views, int32_t width, vp_camera *out);

#ifdef __cplusplus
}
#endif

#endif /* VPB_H */
