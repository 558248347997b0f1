// vpb_kernels.h — launch interface between the C-ABI host code (vpb_api.cpp) and the
// sm_100a kernels (vpb_kernels.cu). Internal header; not part of the public boundary.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "vpb_camdev.h"

namespace vpb {

// Programmatic dependent launch: a kernel launched with launch_pdl may be scheduled while its
// stream predecessor drains (hiding the launch gap); it must start with VPB_PDL_WAIT(), which
// returns once the predecessor has completed and its writes are visible (a no-op otherwise).
#define VPB_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}


struct DevCounters {
    unsigned long long ray_samples, prim_samples, hit_rays, early_exits, saturated;
    unsigned long long overflow_rays, refills, keys, numeric_fail, nonempty_tiles;
    unsigned long long bwd_pairs;  // K6a: primitive-samples planned (the pair cursor; may pass the capacity)
    int key_overflow;
    int fallback_fail;
    unsigned big_buckets;  // K3b: tile buckets past 256 keys (sorted by k_tile_sort_big)
    // key capacity of this view's entries buffer (set by K2): a tile whose bucket ends past it
    // is "key-overflowed" (tile_key_overflowed) and is marched by the fallback from all K
    // primitives' pixel rectangles instead of its (unwritten) bucket
    unsigned key_cap;
    unsigned bwd_long;  // K6: rays whose segment list the forward did not keep (k_backward_rays_list)
    unsigned huge_rays;  // pixels / rays for the last-resort passes (more than kFallbackCap live segments)
    unsigned bwd_huge;   // K6: rays whose forward took the last-resort pass (k_backward_rays_huge)
    unsigned bwd_fb;     // K6a: rays left to the warp-per-ray walk (pair capacity exhausted)
};

// A tile whose bucket [offsets[t], offsets[t+1]) does not fit the entries buffer. K2 saturates
// the offsets at 0xffffffff, so they never wrap; an empty tile past the capacity is not one.
__host__ __device__ __forceinline__ bool tile_key_overflowed(const uint32_t *offsets, int t, unsigned cap) {
    const uint32_t end = offsets[t + 1];
    return end > cap && (end > offsets[t] || end == 0xffffffffu);
}

// Raymarch kernel configuration (window length, staged candidates, CTAs/SM): vpb_kernels.cu.
enum class TileTier : int { Light = 0, Normal = 1, Dense = 2 };

// Linear BVH over the primitives for arbitrary rays (vpb_bvh.cuh / vpb_bvh.cu). Internal
// node: the boxes of both children and their indices (>= 0 internal node, < 0 leaf holding
// primitive -(c + 1)). 64 bytes.
struct BvhNode {
    float4 a;  // left lo.xyz, left hi.x
    float4 b;  // left hi.yz, right lo.xy
    float4 c;  // right lo.z, right hi.xyz
    int4 d;    // left, right, -, -
};
// The same hierarchy three levels at a time (k_bvh_widen): record i holds the eight great-
// grandchild slots of internal node i, slot 4c + 2g + h = child c's child g's child h; a leaf
// met earlier sits in the first slot of its group (h = 0, and g = 0 for a leaf child) with the
// rest of the group empty. A slot is lo.xyz hi.x | hi.yz, index (int bits), valid. One
// 256-byte record per frontier node replaces the node, child and grandchild loads of a
// three-level round of the warp walk.
struct BvhWide {
    float4 s[16];
};
struct BvhDev {
    const BvhNode *nodes;
    int n_prim;  // 1 -> the root is primitive 0 itself
    const BvhWide *wide = nullptr;
};

struct MarchDev {
    float dt, eps;
    int jitter, m;
    unsigned long long seed;
    float alpha;
    int beta;
    BvhDev bvh;  // arbitrary-ray kernels only (vp_march_rays, backward, evalLoss)
};

struct OutDev {
    float *rgb;
    float *alpha;
    int *samples;
    unsigned long long *prof = nullptr;  // per CTA: tile, SM id, start ns, end ns (debug)
    float *state = nullptr;  // arbitrary rays: 8 floats per ray of MarchResult bookkeeping
    // arbitrary rays, warp kernel: the ray's sorted segment list for a following backward,
    // kRaySegs (E) | kRaySegs (X) | kRaySegs (primitive) per ray; count in state[7] (-1: none)
    float *segs = nullptr;
    // Tile-major shard outputs (vp_render_shard_async): pixel (x, y) of owned tile t is
    // written at (t / shard_n) * 256 + (y % 16) * 16 + x % 16. 0 = the image layout.
    int shard_n = 0, width = 0, tiles_x = 0;
};

// One camera view of a raymarch launch: its camera, outputs and binning artefacts (K1-K3 of
// that view), its counters and its overflow list. A launch marches the tiles of up to
// kMaxViews views (vp_render_batch_async), passed by value as a kernel parameter.
struct ViewDev {
    CamDev cam;
    OutDev od;
    const int4 *prects;
    const uint32_t *offsets;
    const unsigned long long *entries;
    DevCounters *ctr;
    int *ovf_list;
    int ovf_cap;
    int *huge_list;  // pixels whose live segments overflow even K5b's window (k_march_huge_views)
    int huge_cap;
};
constexpr int kMaxViews = 16;
struct ViewBatch {
    ViewDev v[kMaxViews];
    int n;
};

// Binning (K1-K3) of up to kMaxViews views in one launch per stage (blockIdx.y = view).
struct BinView {
    CamDev cam;
    int4 *rects, *prects;
    uint32_t *keys, *tile_counts, *offsets, *cursor, *order;
    unsigned long long *entries;
    DevCounters *ctr;  // zeroed by the batch's first kernel
    // nullable: K2 also stores the key count here (mapped pinned host memory: a store over
    // the bus, so no copy-engine transfer queues behind the caller's output copies)
    unsigned long long *keys_host;
};
struct BinBatch {
    BinView v[kMaxViews];
    int n;
    const float *xf16;
    int n_prim;
    int64_t capacity;
};

struct RaysDev {
    const float *origins;
    const float *dirs;
    const float *jitter;
};

// Backward-pass buffers (K6): planar payload gradients + 9 pose gradients per primitive (the
// GradBuffer layout of params.h:12-27), per-primitive pose data (rBase[9] and the three
// rotationDerivative matrices [27]), and the per-ray output adjoints.
struct BwdDev {
    float *g_pay;
    float *g_pose;
    const float *pose36;
    const float *adj_rgb;
    const float *adj_alpha;
    const float *fwd_state = nullptr;  // the forward's per-ray state (skips the replay), or null
    const float *fwd_segs = nullptr;   // the forward's segment lists (OutDev::segs), or null
    float *g_pay4 = nullptr;  // non-null: channel-interleaved payload gradient (k, z, y, x, c)
    unsigned *touched = nullptr;  // with g_pay4: per primitive, set when the walk scatters into it
};

// K6 pair workspace (vpb_backward.cu): the backward as three passes over primitive-samples.
// K6a plans each ray's samples (ray, step, entry) entry-major into [base, base + total);
// K6b evaluates one sample per thread (payload scatter, pose terms); K6c folds each ray's
// pose terms per entry and the t_min chain in step order.
struct BwdPairs {
    int4 *rec;             // [cap] ray, primitive, ts (bits), step-major slot | saturating step << 31
    float4 *terms;         // [cap] rotG and the lattice step per sample, step-major per ray (K6c)
    int4 *span;            // [n_rays] base, total (-1: not planned), admitted entries, -
    int2 *ent;             // [n_rays][kRaySegs] admission step, offset in the ray's range
    int *fb_list;          // [n_rays] rays for the warp-per-ray walk
    int *tile_sums;        // [n_rays / 4096 + 1] per 4096 rays: sample count, then base
    unsigned cap;
};

// Adam step constants (losses.cpp:70-104); bc1/bc2 = 1 - beta^step computed on the host.
struct AdamDev {
    float lr, beta1, beta2, eps, lr_delta_scale, bc1, bc2;
};

constexpr int kFallbackCap = 256;      // segment window of the fallback re-march
constexpr int kRaySegs = 96;  // segments per ray held by the warp-per-ray kernels
constexpr int kFallbackBlocks = 148;   // one CTA per SM
// The last resort for camera rays: more than kFallbackCap primitives live at one sample (the
// reference has no limit). One thread per such pixel over ALL primitives (their pixel rectangles
// filter them), with kHugeCap-entry windows in global scratch: rare, so a small grid.
constexpr int kHugeCap = 4096;
constexpr int kHugeThreads = 148 * 4;
constexpr int kHugeListCap = 1 << 16;  // per view
constexpr int kFallbackThreads = 128;
// key-overflowed tiles (tile_key_overflowed): a fallback CTA rebuilds such a tile's candidate
// list from all K pixel rectangles into its own slice of K entries of global scratch
constexpr int kOvfTileBlocks = kFallbackBlocks;
// backwardRay: one-warp CTAs, 12 per SM (168 registers, no spills); the scratch
// windows (kFallbackCap entries each) are sized for the larger of the two grids
constexpr int kBackwardWarps = 148 * 12;
constexpr int kScratchThreads = kBackwardWarps * 32 > kFallbackBlocks * kFallbackThreads
                                    ? kBackwardWarps * 32 : kFallbackBlocks * kFallbackThreads;

size_t march_tiles_smem();

}  // namespace vpb

namespace vpb {

cudaError_t launch_repack(const float *planar, float4 *inter, int64_t n_prim, int64_t m3,
                          cudaStream_t st);
cudaError_t launch_pad_xf(const float *xf15, float *xf16, int n_prim, cudaStream_t st);
cudaError_t launch_binning_batch(const BinBatch &bb, cudaStream_t st);
// one view; also zeroes its counters
cudaError_t launch_binning(const CamDev &cam, const float *xf16, int n_prim, int4 *rects,
                           int4 *prects, uint32_t *keys, uint32_t *tile_counts, uint32_t *offsets,
                           uint32_t *cursor, uint32_t *order, unsigned long long *entries,
                           int64_t capacity, DevCounters *ctr, cudaStream_t st);
// K5 over the tiles of every view in `views`; `order` lists (view << 20 | tile), heaviest first.
// pairs: the x-pair layout (launch_build_pairs), read instead of payload when march_uses_pairs(M)
cudaError_t launch_march_tiles(const MarchDev &mp, const float *xf16, const float4 *payload, const float4 *pairs,
                               const ViewBatch &views, const uint32_t *order, int n_ctas, bool prof, TileTier tier,
                               cudaStream_t st);
bool march_uses_pairs(int m);
// x-pair layout: n_prim * M * M * (M - 1) entries of 2 float4s
cudaError_t launch_build_pairs(const float4 *payload, float4 *pairs, int64_t n_prim, int m, cudaStream_t st);
// K5b for the views' overflow rays (one launch for all views).
// Key-overflowed tiles are marched here too: tile_scratch holds kOvfTileBlocks * n_prim prim ids.
cudaError_t launch_march_fallback_views(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                        const ViewBatch &views, float *se, float *sx, int *sc,
                                        uint32_t *tile_scratch, cudaStream_t st);
// The views' huge pixels (ViewDev::huge_list, ctr->huge_rays), kHugeCap windows in se/sx/sc
// (kHugeThreads * kHugeCap entries each).
cudaError_t launch_march_huge_views(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                    const ViewBatch &views, float *se, float *sx, int *sc, cudaStream_t st);
// Heaviest-first order over the tiles of several views (counting sort of their candidate counts).
cudaError_t launch_batch_order(const uint32_t *const *tile_counts, const int *n_tiles, int n_views, uint32_t *order,
                               cudaStream_t st);
cudaError_t launch_march_fallback(bool rays_mode, const CamDev &cam, const MarchDev &mp,
                                  const float *xf16, const int4 *prects, int n_prim, const float4 *payload,
                                  const uint32_t *offsets, const unsigned long long *entries,
                                  const OutDev &od, const RaysDev &rays, DevCounters *ctr,
                                  const int *ovf_list, int ovf_cap, float *se, float *sx,
                                  int *sc, cudaStream_t st, int *huge_list = nullptr, int huge_cap = 0);
// Arbitrary rays the fallback could not hold (ctr->huge_rays of huge_list): kHugeCap windows
// through the BVH; a ray's forward state records it (state[7] = -2) for the backward.
cudaError_t launch_march_huge_rays(const MarchDev &mp, const float *xf16, int n_prim, const float4 *payload,
                                   const OutDev &od, const RaysDev &rays, DevCounters *ctr, const int *huge_list,
                                   int huge_cap, float *se, float *sx, int *sc, cudaStream_t st);
cudaError_t launch_march_rays(const MarchDev &mp, const float *xf16, int n_prim,
                              const float4 *payload, const RaysDev &rays, int64_t n_rays,
                              const OutDev &od, DevCounters *ctr, int *ovf_list, int ovf_cap,
                              cudaStream_t st);
// K6: needs bd.fwd_state and bd.fwd_segs (the forward of the same rays, k_march_rays_warp);
// ray_list (list_cap entries) collects the rays whose lists the forward could not keep.
// pairs: the K6a-c workspace; null runs the warp-per-ray walk over every ray. With st2 and
// both events, K6c runs on st2 after ev_fork; the caller makes st wait for ev_join.
cudaError_t launch_backward_rays(const MarchDev &mp, const float *xf16, int n_prim,
                                 const float4 *payload, const RaysDev &rays, int64_t n_rays,
                                 const BwdDev &bd, DevCounters *ctr, int *ray_list, int list_cap, float *se,
                                 float *sx, int *sc, cudaStream_t st, int *huge_list = nullptr, int huge_cap = 0,
                                 float *he = nullptr, float *hx = nullptr, int *hc = nullptr,
                                 const BwdPairs *pairs = nullptr, cudaStream_t st2 = nullptr,
                                 cudaEvent_t ev_fork = nullptr, cudaEvent_t ev_join = nullptr);
// vpb_backward.cu: interleaved payload gradient -> planar GradBuffer (touched primitives)
// clear = false: g4 is left as it is (the caller clears it later, e.g. on another stream)
cudaError_t launch_grad_transpose(float4 *g4, float *planar, const unsigned *touched, int n_prim, unsigned m3,
                                  bool accumulate, cudaStream_t st, bool clear = true);
cudaError_t launch_eval_rays(const CamDev *cams, int n_cams, const int *cam_index, const float *pixel_xy,
                             const int *pixel_id, int64_t n, int jitter, unsigned long long seed,
                             float *origins, float *dirs, float *jit, int *bad, cudaStream_t st);
cudaError_t launch_loss_adjoints(const float *rgb, const float *alpha, const float *target, const float *bg,
                                 int64_t n, float scale, float *composited, float *resid, float *adj_rgb,
                                 float *adj_alpha, cudaStream_t st);
cudaError_t launch_adam(const float *g, float *m1, float *m2, float4 *payload, float *deltas, int64_t n_pay,
                        int64_t n, unsigned m3, const AdamDev &c, int *bad, bool check, cudaStream_t st);
// check: k_adam_check sets *bad on a non-finite gradient. Otherwise the update, which reads *bad
// (non-null) first and returns without writing when it is set.
cudaError_t launch_expf(const float *x, float *y, int64_t n, cudaStream_t st);
// vpb_compose.cu: Frame::composed() on the device (+ Adam's delta write-back and projection)
// skip (nullable, device): when *skip != 0 the kernel returns without touching anything
cudaError_t launch_compose(float *tr24, const float *deltas, int n_prim, float *xf16, int *bad, cudaStream_t st,
                           const int *skip = nullptr);
cudaError_t launch_gather_deltas(const float *tr24, int n_prim, float *deltas, cudaStream_t st);
cudaError_t launch_pose36(const float *tr24, int n_prim, float *p36, cudaStream_t st);
// vpb_bvh.cu: BVH build over the resident transforms (n - 1 nodes)
size_t bvh_scratch_bytes(int n);
cudaError_t launch_bvh_build(const float *xf16, int n, BvhNode *nodes, BvhWide *wide, void *scratch,
                             size_t scratch_bytes, cudaStream_t st);
cudaError_t launch_bvh_refit(const float *xf16, int n, BvhNode *nodes, BvhWide *wide, void *scratch,
                             size_t scratch_bytes, cudaStream_t st);
// the BVH's stable radix sort on key bits [32, 62) (testing); hist: 256 * ceil(n / 2048) words
cudaError_t launch_radix_sort30(unsigned long long *keys, unsigned long long *tmp, unsigned *hist, int n,
                                cudaStream_t st);
cudaError_t launch_sincos(const float *x, float *y, int64_t n, bool want_cos, cudaStream_t st);
cudaError_t launch_composite(const float *rgb, const float *alpha, const float *bg, float *out,
                             int64_t n_px, cudaStream_t st);

}  // namespace vpb
