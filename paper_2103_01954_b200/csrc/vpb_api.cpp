// vpb_api.cpp — the C-ABI (include/vpb.h): context, resident scene, and the render
// pipeline that replaces volprim::render (march.cpp:95-132):
//
//   host:   compose (if asked) + camera constants, exact reference arithmetic
//   device: K1 cull -> K2 scan -> K3 emit + per-tile sort -> K5 tile raymarch -> K5b fallback
//
// all enqueued on one stream with no host synchronisation inside the pipeline (the
// fallback kernel reads the overflow count on the device), so vp_render_async can be
// captured or overlapped; vp_render adds the host copies and one final synchronisation.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vpb.h"
#include <nvtx3/nvToolsExt.h>

#include "vpb_ctx_internal.h"
#include "vpb_hostcopy.hpp"
#include "vpb_hostmath.hpp"
#include "vpb_kernels.h"

using namespace vpb;

namespace {

thread_local std::string g_err;  // errors of context-free calls

template <class T> struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t want) {
        if (want <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        const cudaError_t e = cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T));
        if (e == cudaSuccess) n = std::max<size_t>(want, 1);
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
};

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

constexpr int kTimingSlots = 256;  // march-kernel event pairs kept for vp_kernel_times

// NVTX range over a C-ABI call (header-only NVTX v3: free unless a profiler is attached), so a
// timeline shows each entry point around the kernels it launches.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#ifndef VPB_STAGE_MB
#define VPB_STAGE_MB 8
#endif
constexpr size_t kStageBytes = size_t(VPB_STAGE_MB) << 20;  // host slab upload chunk (upload_planar_host)

}  // namespace

// Binning artefacts of one view (K1-K3 outputs), its counters and its overflow list. Two
// groups of kMaxViews slots: a launch's views are binned on bin_stream into one group while
// the previous launch marches from the other (enqueue_views).
struct BinSlot {
    DBuf<int4> rects, prects;
    DBuf<uint32_t> keys, tile_counts, offsets, cursor, order;
    DBuf<unsigned long long> entries;
    DBuf<int> ovf, huge;  // window-overflow pixels; pixels for the huge pass (kHugeListCap)
    int ovf_cap = 0;
    DevCounters *d_ctr = nullptr;
    cudaEvent_t ev_binned = nullptr, ev_marched = nullptr;
};

struct vp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::string err;
    bool has_scene = false;
    int32_t n_prim = 0, m = 0;
    float w_alpha = 8;
    int32_t w_beta = 8;
    // composed transforms, 16 floats per primitive: double-buffered so vp_set_transforms_async
    // can upload the next frame while the current one is still binned / marched
    DBuf<float> xfb[2];
    int xfi = 0;
    cudaEvent_t ev_xf_binned[2] = {}, ev_xf_marched[2] = {};
    DBuf<float> xf15_tmp, planar_tmp;
    DBuf<float> tr24;      // resident PrimitiveTransform records (vp_set_frame, vp_adam_step)
    DBuf<int> flag;        // device error flag (compose)
    bool has_xf = false;   // resident composed transforms are set
    DBuf<float4> payload;
    // derived x-pair layout of the payload for the raymarch's 256-bit gathers (march_uses_pairs);
    // rebuilt before the next raymarch whenever the payload may have changed
    DBuf<float4> pairs;
    bool pairs_dirty = true;
    BinSlot slot[2 * kMaxViews];
    int cur = 0;    // slot of the latest render's last view
    int group = 0;  // slot group of the latest launch
    BinSlot &bs() { return slot[cur]; }
    cudaStream_t bin_stream = nullptr;
    DBuf<uint32_t> batch_order[2];  // per group: heaviest-first (view, tile) order of a batch
    // vp_render_batch_async into host memory: per slot group, device outputs of every view;
    // the group's device->host copies (copy_stream) overlap the other group's raymarch
    DBuf<float> bring_rgb[2], bring_alpha[2];
    DBuf<int> bring_samples[2];
    cudaEvent_t ev_brendered[2] = {}, ev_bcopied[2] = {};
    // vp_set_transforms_async: the upload waits for binning still reading the old transforms
    // (ev_last_binned) and the next binning waits for the upload (ev_xf)
    cudaEvent_t ev_xf = nullptr, ev_last_binned = nullptr, ev_last_marched = nullptr;
    DBuf<float> out_rgb, out_alpha;
    DBuf<int> out_samples, ovf_list;
    DBuf<float> fb_e, fb_x;
    DBuf<int> fb_c;
    DBuf<float> hg_e, hg_x;  // K5c (k_march_huge_views / _rays, k_backward_rays_huge) windows
    DBuf<int> hg_c;
    DBuf<int> huge_ray_list;  // ray batches: the rays for the last-resort passes
    DBuf<float> ray_o, ray_d, ray_j;
    DevCounters *d_ctr = nullptr, *h_ctr = nullptr;
    DevCounters *last_ctr[kMaxViews] = {};  // the counters of the latest render launch's views
    int last_n = 1;                          // 1: ctx->d_ctr alone (single view / ray calls)
    int64_t entries_cap = 0;
    bool key_cap_fixed = false;  // vp_set_key_capacity(..., grow = 0)
    int ovf_cap = 0;
    // K5b's per-CTA candidate lists for key-overflowed tiles (kOvfTileBlocks x n_prim ids)
    DBuf<uint32_t> ovf_tile_lists;
    // per slot: the key count K2 found, copied to pinned memory after each binning so the next
    // launch can grow entries_cap without waiting (h_keys_ready: that copy's event)
    unsigned long long *h_keys = nullptr, *d_keys = nullptr;  // mapped pinned: host / device view
    cudaEvent_t ev_keys[2] = {};
    cudaEvent_t t_ev[2 * kTimingSlots] = {};
    int64_t t_count = 0;
    DBuf<float> adam_m1, adam_m2;  // Adam moments over [payload | deltas] (GradBuffer order)
    // per-entry-point scratch, kept across calls (a cudaMalloc per training call costs ms)
    DBuf<float> s_loss, s_bwd_g, s_bwd_pose, s_bwd_adj, s_bwd_fwd, s_adam;
    // backward payload gradient, channel-interleaved (zero between calls) + touched flags
    DBuf<float> g_pay4;
    // batches with the auxiliary stream alternate between two interleaved gradient buffers:
    // the one a call used is cleared on the auxiliary stream during the next call's forward,
    // so the transpose only reads it (g4_dirty: holds a previous call's gradient)
    DBuf<float> g_pay4b;
    float *h_zeros = nullptr;  // page-locked zeros: small clears as copy-engine uploads (no SM slots)
    size_t h_zeros_n = 0;
    int g4_cur = 0;
    bool g4_dirty[2] = {false, false};
    DBuf<unsigned> g_touched;
    DBuf<int> bwd_list;  // K6: rays whose segment lists the forward did not keep
    // K6a-c pair workspace (BwdPairs); pair_cap grows to the planned count after a call that
    // overflowed it (the overflowing rays take the warp walk, so results never depend on it)
    DBuf<int4> bp_rec;
    DBuf<int2> bp_ent;
    DBuf<float4> bp_terms;
    DBuf<int4> bp_span;
    DBuf<int> bp_fb, bp_tiles;
    size_t pair_cap = 0;
    bool pair_cap_fixed = false;
    // backward path: 1 the warp-per-ray walk for every ray, 0 the passes over primitive-samples
    // (K6a-c), -1 auto (K6a-c from kPairsMinRays rays: below, its per-ray passes leave the GPU
    // mostly idle and the one-kernel walk is quicker); VPB_BWD_MODE=warp|pairs
    int bwd_warp_walk = -1;
    // host slab uploads (upload_planar_host): page-locked + device staging chunks, their
    // transfer events, and the host copy threads
    static constexpr int kStageSlots = 4;
    float *stage_h[kStageSlots] = {};
    size_t stage_h_floats[kStageSlots] = {};
    DBuf<float> stage_d[kStageSlots];
    cudaEvent_t ev_stage[kStageSlots] = {};
    std::unique_ptr<CopyPool> copy_pool;
    void *out_stage = nullptr;  // copy_out_host: page-locked staging of pageable outputs
    size_t out_stage_bytes = 0;
    cudaEvent_t ev_out[3] = {};
    // payload gradient layout of the backward: 0 planar, 1 interleaved + vector reductions
    // (transposed at the C-ABI), -1 auto (interleaved for batches of kV4MinRays rays or more,
    // where the 4x fewer reductions outweigh the transpose)
    int bwd_v4 = -1;
    // BVH over the resident transforms for arbitrary rays, rebuilt lazily after a pose change
    DBuf<BvhNode> bvh_nodes;
    DBuf<BvhWide> bvh_wide;  // the same hierarchy three levels per record (warp walks)
    int bvh_built_n = 0, bvh_refits = 0;  // the topology in bvh_scratch: primitives, refits since
    // vp_render_async into host memory: two device output slots; the device->host copy of
    // one view (copy_stream) overlaps the rendering of the next
    cudaStream_t copy_stream = nullptr;
    cudaStream_t aux_stream = nullptr;  // the backward's K6c beside the transpose
    float *h_loss = nullptr;  // evalLoss: page-locked staging of host ray-batch inputs
    size_t h_loss_floats = 0;
    cudaEvent_t ev_aux_fork = nullptr, ev_aux_join = nullptr, ev_aux_pose = nullptr;
    cudaEvent_t ev_rendered[2] = {}, ev_copied[2] = {};
    DBuf<float> ring_rgb[2], ring_alpha[2];
    DBuf<int> ring_samples[2];
    int ring_next = 0;
    DBuf<unsigned char> bvh_scratch;
    bool bvh_dirty = true;
    int64_t adam_step = 0;
    // Raymarch configuration for the next render, from the mean candidates per non-empty tile
    // of the last render whose counters reached the host (see note_density).
    TileTier tier = TileTier::Normal;
    bool tier_known = false;
    cudaStream_t scene_writer = nullptr;  // another agent's stream that wrote the scene (broadcast)  // false after a scene change: the next render measures the density first
    int tile_cfg = -1;  // VPB_TILE_CFG override: -1 auto, else a TileTier
};

namespace {

int fail(vp_ctx *ctx, int code, const std::string &msg) {
    (ctx ? ctx->err : g_err) = msg;
    return code;
}
int cuda_fail(vp_ctx *ctx, cudaError_t e, const char *where) {
    return fail(ctx, VP_ERR_DEVICE, std::string(where) + ": " + cudaGetErrorString(e));
}
#define VP_CUDA(ctx, call)                                   \
    do {                                                     \
        const cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

// Camera constants with the reference's host arithmetic (camera.cpp:14-23, camera.h:28).
CamDev make_cam(const vp_camera &c) {
    using namespace vpb::host;
    CamDev d{};
    const M3 K = load9(c.K), R = load9(c.R);
    const M3 kinv = inverse(K);
    const F3 center = neg(mv(transposed(R), load3(c.t)));
    std::memcpy(d.kinv, kinv.m, sizeof d.kinv);
    std::memcpy(d.R, c.R, sizeof d.R);
    std::memcpy(d.K, c.K, sizeof d.K);
    std::memcpy(d.t, c.t, sizeof d.t);
    d.center[0] = center.x;
    d.center[1] = center.y;
    d.center[2] = center.z;
    d.width = c.width;
    d.height = c.height;
    d.tiles_x = (c.width + 15) / 16;
    d.tiles_y = (c.height + 15) / 16;
    return d;
}

int check_march(vp_ctx *ctx, const vp_march *cfg) {
    if (!cfg) return fail(ctx, VP_ERR_USAGE, "null march config");
    if (!(cfg->step_size > 0) || !std::isfinite(cfg->step_size))
        return fail(ctx, VP_ERR_USAGE, "step_size must be positive and finite");
    if (!std::isfinite(cfg->early_eps)) return fail(ctx, VP_ERR_USAGE, "early_eps must be finite");
    if (cfg->accumulation_permutation != 0)
        return fail(ctx, VP_ERR_USAGE,
                    "accumulationPermutation is a march() test hook; not supported by the device path");
    return VP_OK;
}

MarchDev make_march(const vp_ctx *ctx, const vp_march *cfg) {
    MarchDev mp{};
    mp.dt = cfg->step_size;
    mp.eps = cfg->early_eps;
    mp.jitter = cfg->jitter != 0;
    mp.m = ctx->m;
    mp.seed = cfg->seed;
    mp.alpha = ctx->w_alpha;
    mp.beta = ctx->w_beta;
    return mp;
}

// The BVH of the resident transforms (built on the ctx stream if the pose changed).
int ensure_bvh(vp_ctx *ctx, MarchDev &mp) {
    const int n = ctx->n_prim;
    if (ctx->bvh_dirty && n > 1) {
        VP_CUDA(ctx, ctx->bvh_nodes.ensure(size_t(n - 1)));
        VP_CUDA(ctx, ctx->bvh_wide.ensure(size_t(n - 1)));
        const size_t bytes = bvh_scratch_bytes(n);
        VP_CUDA(ctx, ctx->bvh_scratch.ensure(bytes));
        // A pose change (an Adam step, a new frame of the same primitives) refits the last
        // build's topology; the Morton order and hierarchy are rebuilt every kBvhRefits poses
        constexpr int kBvhRefits = 16;
        if (ctx->bvh_built_n == n && ctx->bvh_refits < kBvhRefits) {
            VP_CUDA(ctx, launch_bvh_refit(ctx->xfb[ctx->xfi].p, n, ctx->bvh_nodes.p, ctx->bvh_wide.p,
                                          ctx->bvh_scratch.p, bytes, ctx->stream));
            ++ctx->bvh_refits;
        } else {
            VP_CUDA(ctx, launch_bvh_build(ctx->xfb[ctx->xfi].p, n, ctx->bvh_nodes.p, ctx->bvh_wide.p,
                                          ctx->bvh_scratch.p, bytes, ctx->stream));
            ctx->bvh_built_n = n;
            ctx->bvh_refits = 0;
        }
    }
    ctx->bvh_dirty = false;
    mp.bvh = BvhDev{ctx->bvh_nodes.p, n, ctx->bvh_wide.p};
    return VP_OK;
}

int ensure_fallback(vp_ctx *ctx) {
    const size_t n = size_t(kScratchThreads) * kFallbackCap;
    VP_CUDA(ctx, ctx->fb_e.ensure(n));
    VP_CUDA(ctx, ctx->fb_x.ensure(n));
    VP_CUDA(ctx, ctx->fb_c.ensure(n));
    const size_t nh = size_t(kHugeThreads) * kHugeCap;  // K5c windows (29 MB)
    VP_CUDA(ctx, ctx->huge_ray_list.ensure(size_t(kHugeListCap)));
    VP_CUDA(ctx, ctx->hg_e.ensure(nh));
    VP_CUDA(ctx, ctx->hg_x.ensure(nh));
    VP_CUDA(ctx, ctx->hg_c.ensure(nh));
    return VP_OK;
}

int ensure_slot(vp_ctx *ctx, BinSlot &b) {
    if (b.d_ctr) return VP_OK;
    VP_CUDA(ctx, cudaMalloc(&b.d_ctr, sizeof(DevCounters)));
    VP_CUDA(ctx, cudaMemset(b.d_ctr, 0, sizeof(DevCounters)));
    VP_CUDA(ctx, cudaEventCreateWithFlags(&b.ev_binned, cudaEventDisableTiming));
    VP_CUDA(ctx, cudaEventCreateWithFlags(&b.ev_marched, cudaEventDisableTiming));
    return VP_OK;
}

// Buffers of one slot for a view of camera `cam`.
int ensure_slot_buffers(vp_ctx *ctx, BinSlot &b, const CamDev &cam) {
    const size_t n_tiles = size_t(cam.tiles_x) * cam.tiles_y;
    const size_t n_px = size_t(cam.width) * cam.height;
    if (n_tiles >= (size_t(1) << 20)) return fail(ctx, VP_ERR_USAGE, "image too large (2^20 tiles)");
    if (ctx->entries_cap == 0) ctx->entries_cap = std::max<int64_t>(int64_t(1) << 20, int64_t(ctx->n_prim) * 16);
    if (int rc = ensure_slot(ctx, b)) return rc;
    VP_CUDA(ctx, b.tile_counts.ensure(n_tiles));
    VP_CUDA(ctx, b.offsets.ensure(n_tiles + 1));
    VP_CUDA(ctx, b.cursor.ensure(n_tiles));
    VP_CUDA(ctx, b.order.ensure(n_tiles));
    VP_CUDA(ctx, b.rects.ensure(size_t(std::max(ctx->n_prim, 1))));
    VP_CUDA(ctx, b.prects.ensure(size_t(std::max(ctx->n_prim, 1))));
    VP_CUDA(ctx, b.keys.ensure(size_t(std::max(ctx->n_prim, 1))));
    VP_CUDA(ctx, b.entries.ensure(size_t(ctx->entries_cap)));
    VP_CUDA(ctx, ctx->ovf_tile_lists.ensure(size_t(kOvfTileBlocks) * size_t(std::max(ctx->n_prim, 1))));
    if (size_t(b.ovf_cap) < n_px) {
        VP_CUDA(ctx, b.ovf.ensure(n_px));
        b.ovf_cap = int(n_px);
    }
    VP_CUDA(ctx, b.huge.ensure(size_t(kHugeListCap)));
    return ensure_fallback(ctx);
}

// Buffers for a single-view render (both slots it may land in).
int ensure_render_buffers(vp_ctx *ctx, const CamDev &cam) {
    for (int g = 0; g < 2; ++g)
        if (int rc = ensure_slot_buffers(ctx, ctx->slot[g * kMaxViews], cam)) return rc;
    return VP_OK;
}

// Key capacity for the next binning. A view whose tile buckets do not fit the entries buffer
// still renders exactly (its overflowed tiles are marched by K5b from all K pixel rectangles),
// but slower, so the capacity follows the largest key count seen: from the pinned copies of
// launches whose binning has completed (never waits) and from vp_render / vp_read_stats.
void note_keys(vp_ctx *ctx, unsigned long long keys) {
    if (!ctx->key_cap_fixed && int64_t(keys) > ctx->entries_cap) ctx->entries_cap = int64_t(keys) + int64_t(keys) / 4 + 1024;
}

void grow_key_capacity(vp_ctx *ctx) {
    for (int g = 0; g < 2; ++g) {
        if (!ctx->ev_keys[g] || cudaEventQuery(ctx->ev_keys[g]) != cudaSuccess) {
            cudaGetLastError();  // cudaErrorNotReady is not an error here
            continue;
        }
        for (int v = 0; v < kMaxViews; ++v)
            note_keys(ctx, reinterpret_cast<volatile unsigned long long *>(ctx->h_keys)[g * kMaxViews + v]);
    }
}

// The device pipeline for `n` views (no host synchronisation). Binning (K1-K3) of each view
// goes to bin_stream into the slot group the previous launch did not use, so it overlaps the
// previous launch's raymarch (whose tail leaves SMs idle); a slot is rebinned only after the
// raymarch that read it has finished. Then ONE raymarch launch covers the tiles of all the
// views, heaviest first across views (a batch pays the tail of a launch once), and one
// fallback launch their overflow rays.
// n_ctas_single: a shard render's owned tile count (its order lists them first), else -1.
void note_density(vp_ctx *ctx, const DevCounters &c);

int enqueue_views(vp_ctx *ctx, int n, const CamDev *cams, const MarchDev &mp, const OutDev *ods, cudaStream_t st,
                  int n_ctas_single = -1) {
    if (n < 1 || n > kMaxViews) return fail(ctx, VP_ERR_USAGE, "1 to 16 views per launch");
    grow_key_capacity(ctx);
    ctx->group ^= 1;
    BinSlot *grp = ctx->slot + ctx->group * kMaxViews;
    for (int v = 0; v < n; ++v)
        if (int rc = ensure_slot_buffers(ctx, grp[v], cams[v])) return rc;
    ViewBatch vb{};
    vb.n = n;
    VP_CUDA(ctx, cudaStreamWaitEvent(ctx->bin_stream, ctx->ev_xf, 0));  // vp_set_transforms_async
    const uint32_t *counts[kMaxViews];
    int n_tiles[kMaxViews];
    int total = 0;
    BinBatch bb{};  // K1-K3 of every view: one launch per stage (vpb_kernels.cu k_bin_zero ...)
    bb.n = n;
    bb.xf16 = ctx->xfb[ctx->xfi].p;
    bb.n_prim = ctx->n_prim;
    bb.capacity = ctx->entries_cap;
    for (int v = 0; v < n; ++v) {
        BinSlot &b = grp[v];
        VP_CUDA(ctx, cudaStreamWaitEvent(ctx->bin_stream, b.ev_marched, 0));
        unsigned long long *kh = ctx->h_keys + ctx->group * kMaxViews + v;  // grow_key_capacity reads it
        bb.v[v] = BinView{cams[v], b.rects.p, b.prects.p, b.keys.p, b.tile_counts.p, b.offsets.p, b.cursor.p,
                          b.order.p, b.entries.p, b.d_ctr, ctx->d_keys + (kh - ctx->h_keys)};
        vb.v[v] = ViewDev{cams[v], ods[v], b.prects.p, b.offsets.p, b.entries.p, b.d_ctr, b.ovf.p, b.ovf_cap,
                          b.huge.p, kHugeListCap};
        counts[v] = b.tile_counts.p;
        n_tiles[v] = cams[v].tiles_x * cams[v].tiles_y;
        total += n_tiles[v];
    }
    VP_CUDA(ctx, launch_binning_batch(bb, ctx->bin_stream));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_keys[ctx->group], ctx->bin_stream));  // K2 stored the key counts
    if (!ctx->tier_known && ctx->tile_cfg < 0) {
        // first render of a scene: wait for its binning (tens of µs, once) and pick the raymarch
        // tier from this scene's density instead of the previous scene's
        VP_CUDA(ctx, cudaStreamSynchronize(ctx->bin_stream));
        DevCounters sum{};
        for (int v = 0; v < n; ++v) {
            VP_CUDA(ctx, cudaMemcpy(ctx->h_ctr, grp[v].d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost));
            sum.keys += ctx->h_ctr->keys;
            sum.nonempty_tiles += ctx->h_ctr->nonempty_tiles;
        }
        note_density(ctx, sum);
        ctx->tier_known = true;
    }
    const uint32_t *order = grp[0].order.p;
    if (n > 1) {
        VP_CUDA(ctx, ctx->batch_order[ctx->group].ensure(size_t(std::max(total, 1))));
        VP_CUDA(ctx, launch_batch_order(counts, n_tiles, n, ctx->batch_order[ctx->group].p, ctx->bin_stream));
        order = ctx->batch_order[ctx->group].p;
    }
    VP_CUDA(ctx, cudaEventRecord(grp[0].ev_binned, ctx->bin_stream));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_last_binned, ctx->bin_stream));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_xf_binned[ctx->xfi], ctx->bin_stream));
    VP_CUDA(ctx, cudaStreamWaitEvent(st, grp[0].ev_binned, 0));
    const int slot = int(ctx->t_count % kTimingSlots);
    VP_CUDA(ctx, cudaEventRecord(ctx->t_ev[2 * slot], st));
    if (n == 1 && n_ctas_single >= 0) total = n_ctas_single;
    if (march_uses_pairs(ctx->m) && ctx->pairs_dirty) {  // the raymarch's x-pair layout, after a payload change
        VP_CUDA(ctx, ctx->pairs.ensure(2 * size_t(ctx->n_prim) * ctx->m * ctx->m * (ctx->m - 1)));
        VP_CUDA(ctx, launch_build_pairs(ctx->payload.p, ctx->pairs.p, ctx->n_prim, ctx->m, st));
        ctx->pairs_dirty = false;
    }
    VP_CUDA(ctx, launch_march_tiles(mp, ctx->xfb[ctx->xfi].p, ctx->payload.p, ctx->pairs.p, vb, order, total,
                                    ods[0].prof != nullptr,
                                    ctx->tile_cfg < 0 ? ctx->tier : TileTier(ctx->tile_cfg), st));
    VP_CUDA(ctx, launch_march_fallback_views(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, vb, ctx->fb_e.p,
                                             ctx->fb_x.p, ctx->fb_c.p, ctx->ovf_tile_lists.p, st));
    VP_CUDA(ctx, launch_march_huge_views(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, vb, ctx->hg_e.p,
                                         ctx->hg_x.p, ctx->hg_c.p, st));
    VP_CUDA(ctx, cudaEventRecord(ctx->t_ev[2 * slot + 1], st));
    for (int v = 0; v < n; ++v) VP_CUDA(ctx, cudaEventRecord(grp[v].ev_marched, st));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_last_marched, st));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_xf_marched[ctx->xfi], st));
    ++ctx->t_count;
    ctx->cur = ctx->group * kMaxViews + n - 1;
    ctx->d_ctr = grp[n - 1].d_ctr;
    for (int v = 0; v < n; ++v) ctx->last_ctr[v] = grp[v].d_ctr;
    ctx->last_n = n;
    return VP_OK;
}

int enqueue_render(vp_ctx *ctx, const CamDev &cam, const MarchDev &mp, const OutDev &od, cudaStream_t st) {
    return enqueue_views(ctx, 1, &cam, mp, &od, st);
}

// Mean candidates per non-empty tile: up to 14 -> Light, up to 40 -> Normal, else Dense
// (thresholds between the BASELINE configs' 11, 22 and 66; vpb_kernels.cu TileCfg*).
constexpr unsigned long long kLightKeysPerTile = 14, kDenseKeysPerTile = 40;

void note_density(vp_ctx *ctx, const DevCounters &c) {
    if (c.nonempty_tiles == 0) return;
    ctx->tier_known = true;
    ctx->tier = c.keys > kDenseKeysPerTile * c.nonempty_tiles  ? TileTier::Dense
                : c.keys > kLightKeysPerTile * c.nonempty_tiles ? TileTier::Normal
                                                                : TileTier::Light;
}

void fill_stats(const DevCounters &c, float ms, vp_stats *s) {
    if (!s) return;
    s->ray_samples = int64_t(c.ray_samples);
    s->prim_samples = int64_t(c.prim_samples);
    s->hit_rays = int64_t(c.hit_rays);
    s->early_exits = int64_t(c.early_exits);
    s->saturated = int64_t(c.saturated);
    s->overflow_rays = int64_t(c.overflow_rays);
    s->keys = int64_t(c.keys);
    s->refills = int64_t(c.refills);
    s->ms = ms;
    s->huge_rays = int32_t(c.huge_rays);
}

int check_counters(vp_ctx *ctx, const DevCounters &c) {
    if (c.fallback_fail)
        return fail(ctx, VP_ERR_NUMERIC,
                    "a ray has more simultaneously live primitive segments than the widest window holds "
                    "(4096)");
    if (c.numeric_fail) return fail(ctx, VP_ERR_NUMERIC, "quadrature did not terminate");
    return VP_OK;
}

int check_ctx(vp_ctx *ctx, bool need_scene, bool need_xf = true) {
    if (!ctx) return fail(nullptr, VP_ERR_USAGE, "null context");
    if (ctx->scene_writer) {  // ctx_scene_written: everything from now on waits for the writer
        VP_CUDA(ctx, cudaEventRecord(ctx->ev_xf, ctx->scene_writer));  // the binning waits for ev_xf
        VP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_xf, 0));
        VP_CUDA(ctx, cudaStreamWaitEvent(ctx->bin_stream, ctx->ev_xf, 0));
        ctx->scene_writer = nullptr;
    }
    if (need_scene && !ctx->has_scene) return fail(ctx, VP_ERR_USAGE, "no scene set");
    if (need_scene && need_xf && ctx->n_prim > 0 && !ctx->has_xf)
        return fail(ctx, VP_ERR_USAGE, "no transforms set (vp_set_frame / vp_set_transforms)");
    const cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    return VP_OK;
}

// Before a synchronous entry point rewrites the resident transforms or payload: wait for the
// asynchronous renders that may still read them (binning stream, last raymarch, own stream).
int quiesce(vp_ctx *ctx) {
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->bin_stream));
    VP_CUDA(ctx, cudaEventSynchronize(ctx->ev_last_marched));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int check_cam(vp_ctx *ctx, const vp_camera *cam) {
    if (!cam) return fail(ctx, VP_ERR_USAGE, "null camera");
    if (cam->width < 0 || cam->height < 0) return fail(ctx, VP_ERR_USAGE, "negative image size");
    return VP_OK;
}

}  // namespace

namespace vpb {

int ctx_device(const vp_ctx *ctx) { return ctx->device; }

int ctx_scene(vp_ctx *ctx, CtxScene *out) {
    if (!ctx) return fail(nullptr, VP_ERR_USAGE, "null context");
    if (!ctx->has_scene) return fail(ctx, VP_ERR_USAGE, "no scene set (vp_set_scene first)");
    const size_t k = size_t(ctx->n_prim);
    if (k > 0) {  // a receiving context may hold only the shape (vp_set_scene with NULL data)
        VP_CUDA(ctx, ctx->xfb[ctx->xfi].ensure(16 * k));
        VP_CUDA(ctx, ctx->payload.ensure(k * size_t(ctx->m) * ctx->m * ctx->m));
    }
    *out = CtxScene{ctx->xfb[ctx->xfi].p, ctx->payload.p, ctx->n_prim, ctx->m, ctx->device, ctx->stream};
    return VP_OK;
}

int ctx_scene_written(vp_ctx *ctx, cudaStream_t st) {
    ctx->has_xf = true;
    ctx->bvh_dirty = true;
    ctx->bvh_built_n = 0;  // a new scene: rebuild the BVH topology, not just refit it
    ctx->pairs_dirty = true;
    // The writer's work may not be enqueued yet (a broadcast inside a caller's NCCL group is
    // launched at vp_group_end), so the context waits for `st` when it next uses the scene
    // (check_ctx), not now.
    ctx->scene_writer = st;
    return VP_OK;
}

void ctx_drop_writer(vp_ctx *ctx, cudaStream_t st) {  // the writer's stream is being destroyed (synced)
    if (ctx && ctx->scene_writer == st) ctx->scene_writer = nullptr;
}

int ctx_wait_renders(vp_ctx *ctx, cudaStream_t st) {
    VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_last_marched, 0));
    return VP_OK;
}

int ctx_fail(vp_ctx *ctx, int code, const std::string &msg) { return fail(ctx, code, msg); }

}  // namespace vpb

extern "C" {

int vp_version(void) { return VPB_VERSION; }

int vp_create(int32_t device, vp_ctx **out) {
    if (!out) return fail(nullptr, VP_ERR_USAGE, "null output pointer");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDeviceCount");
    if (device < 0 || device >= n) return fail(nullptr, VP_ERR_USAGE, "device index out of range");
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(nullptr, VP_ERR_DEVICE, std::string("libvpb is built for sm_100a (B200); device is ") +
                                                prop.name);
    vp_ctx *ctx = new vp_ctx();
    ctx->device = device;
    if (const char *bl = std::getenv("VPB_BWD_LAYOUT"))  // A/B: "v4" = interleaved + vector reductions
        ctx->bwd_v4 = std::strcmp(bl, "v4") == 0 ? 1 : std::strcmp(bl, "planar") == 0 ? 0 : -1;
    if (const char *bm = std::getenv("VPB_BWD_MODE"))  // A/B: "warp" = the warp-per-ray walk for every ray
        ctx->bwd_warp_walk = std::strcmp(bm, "warp") == 0 ? 1 : std::strcmp(bm, "pairs") == 0 ? 0 : -1;
    if (const char *pc = std::getenv("VPB_BWD_PAIR_CAP")) {  // tests: a fixed (small) pair capacity
        ctx->pair_cap = size_t(std::strtoull(pc, nullptr, 10));
        ctx->pair_cap_fixed = true;
    }
    if (const char *tc = std::getenv("VPB_TILE_CFG"))  // tuning override: light | normal | dense
        ctx->tile_cfg = std::strcmp(tc, "light") == 0    ? int(TileTier::Light)
                        : std::strcmp(tc, "normal") == 0 ? int(TileTier::Normal)
                        : std::strcmp(tc, "dense") == 0  ? int(TileTier::Dense)
                                                         : -1;
    int rc = VP_OK;
    if ((e = cudaSetDevice(device)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreate(&ctx->ev0)) != cudaSuccess || (e = cudaEventCreate(&ctx->ev1)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_rendered[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_rendered[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_copied[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_copied[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->bin_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_brendered[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_brendered[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_bcopied[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_bcopied[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_xf, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_last_binned, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_last_marched, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_xf_binned[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_xf_binned[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_xf_marched[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_xf_marched[1], cudaEventDisableTiming)) != cudaSuccess ||

        (e = cudaEventCreateWithFlags(&ctx->ev_out[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_out[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_out[2], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_stage[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_stage[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_stage[2], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_stage[3], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_keys[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_keys[1], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaHostAlloc(&ctx->h_keys, sizeof(unsigned long long) * 2 * kMaxViews, cudaHostAllocMapped)) !=
            cudaSuccess ||
        (e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&ctx->d_keys), ctx->h_keys, 0)) != cudaSuccess ||
        (e = cudaMallocHost(&ctx->h_ctr, sizeof(DevCounters))) != cudaSuccess) {
        rc = cuda_fail(nullptr, e, "vp_create");
        vp_destroy(ctx);
        return rc;
    }
    std::memset(ctx->h_keys, 0, sizeof(unsigned long long) * 2 * kMaxViews);
    for (cudaEvent_t &ev : ctx->t_ev)
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) {
        rc = cuda_fail(nullptr, e, "vp_create");
        vp_destroy(ctx);
        return rc;
    }
    if ((rc = ensure_slot(ctx, ctx->slot[0])) != VP_OK) {
        g_err = ctx->err;
        vp_destroy(ctx);
        return rc;
    }
    ctx->d_ctr = ctx->slot[0].d_ctr;
    *out = ctx;
    return VP_OK;
}

int vp_destroy(vp_ctx *ctx) {
    if (!ctx) return VP_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    if (ctx->bin_stream) cudaStreamSynchronize(ctx->bin_stream);
    for (int q = 0; q < 2; ++q) {
        ctx->ring_rgb[q].release();
        ctx->ring_alpha[q].release();
        ctx->ring_samples[q].release();
        if (ctx->ev_rendered[q]) cudaEventDestroy(ctx->ev_rendered[q]);
        if (ctx->ev_copied[q]) cudaEventDestroy(ctx->ev_copied[q]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->aux_stream) {
        cudaStreamSynchronize(ctx->aux_stream);
        cudaStreamDestroy(ctx->aux_stream);
    }
    if (ctx->ev_aux_fork) cudaEventDestroy(ctx->ev_aux_fork);
    if (ctx->ev_aux_join) cudaEventDestroy(ctx->ev_aux_join);
    if (ctx->ev_aux_pose) cudaEventDestroy(ctx->ev_aux_pose);
    if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
    ctx->tr24.release();
    for (auto *b : {&ctx->s_loss, &ctx->s_bwd_g, &ctx->s_bwd_pose, &ctx->s_bwd_adj, &ctx->s_bwd_fwd, &ctx->s_adam})
        b->release();
    ctx->flag.release();
    for (auto *b : {&ctx->xfb[0], &ctx->xfb[1], &ctx->xf15_tmp, &ctx->planar_tmp, &ctx->out_rgb, &ctx->out_alpha,
                    &ctx->fb_e, &ctx->fb_x, &ctx->ray_o, &ctx->ray_d, &ctx->ray_j})
        b->release();
    ctx->payload.release();
    for (BinSlot &b : ctx->slot) {
        b.rects.release();
        b.prects.release();
        for (auto *u : {&b.keys, &b.tile_counts, &b.offsets, &b.cursor, &b.order}) u->release();
        b.entries.release();
        b.ovf.release();
        b.huge.release();
        if (b.d_ctr) cudaFree(b.d_ctr);
        if (b.ev_binned) cudaEventDestroy(b.ev_binned);
        if (b.ev_marched) cudaEventDestroy(b.ev_marched);
    }
    if (ctx->bin_stream) cudaStreamDestroy(ctx->bin_stream);
    if (ctx->ev_xf) cudaEventDestroy(ctx->ev_xf);
    if (ctx->ev_last_binned) cudaEventDestroy(ctx->ev_last_binned);
    if (ctx->ev_last_marched) cudaEventDestroy(ctx->ev_last_marched);
    for (int q = 0; q < 2; ++q) {
        if (ctx->ev_xf_binned[q]) cudaEventDestroy(ctx->ev_xf_binned[q]);
        if (ctx->ev_xf_marched[q]) cudaEventDestroy(ctx->ev_xf_marched[q]);
    }
    for (int g = 0; g < 2; ++g) {
        ctx->batch_order[g].release();
        ctx->bring_rgb[g].release();
        ctx->bring_alpha[g].release();
        ctx->bring_samples[g].release();
        if (ctx->ev_brendered[g]) cudaEventDestroy(ctx->ev_brendered[g]);
        if (ctx->ev_bcopied[g]) cudaEventDestroy(ctx->ev_bcopied[g]);
    }
    for (auto *b : {&ctx->out_samples, &ctx->ovf_list, &ctx->fb_c, &ctx->hg_c}) b->release();
    ctx->hg_e.release();
    ctx->hg_x.release();
    ctx->huge_ray_list.release();
    if (ctx->h_ctr) cudaFreeHost(ctx->h_ctr);
    if (ctx->h_keys) cudaFreeHost(ctx->h_keys);
    for (cudaEvent_t ev : ctx->ev_keys)
        if (ev) cudaEventDestroy(ev);
    ctx->ovf_tile_lists.release();
    ctx->g_pay4.release();
    ctx->g_pay4b.release();
    if (ctx->h_zeros) cudaFreeHost(ctx->h_zeros);
    ctx->h_zeros = nullptr;
    ctx->h_zeros_n = 0;
    ctx->g_touched.release();
    ctx->bwd_list.release();
    ctx->bp_rec.release();
    ctx->bp_ent.release();
    ctx->bp_terms.release();
    ctx->bp_span.release();
    ctx->bp_fb.release();
    ctx->bp_tiles.release();
    for (int i = 0; i < vp_ctx::kStageSlots; ++i) {
        if (ctx->stage_h[i]) cudaFreeHost(ctx->stage_h[i]);
        ctx->stage_d[i].release();
        if (ctx->ev_stage[i]) cudaEventDestroy(ctx->ev_stage[i]);
    }
    ctx->copy_pool.reset();
    if (ctx->out_stage) cudaFreeHost(ctx->out_stage);
    for (cudaEvent_t ev : ctx->ev_out)
        if (ev) cudaEventDestroy(ev);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (cudaEvent_t ev : ctx->t_ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return VP_OK;
}

const char *vp_last_error(const vp_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

void *vp_stream(vp_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int vp_compose(int32_t n_prim, const float *tr24, float *xf15) {
    if (n_prim < 0 || (n_prim > 0 && (!tr24 || !xf15))) return fail(nullptr, VP_ERR_USAGE, "bad arguments");
    for (int32_t k = 0; k < n_prim; ++k)
        if (!vpb::host::compose(tr24 + 24 * size_t(k), xf15 + 15 * size_t(k)))
            return fail(nullptr, VP_ERR_USAGE, "non-positive composed primitive scale");
    return VP_OK;
}

int vp_set_transforms(vp_ctx *ctx, int32_t n_prim, const float *xf15) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (int rc = quiesce(ctx)) return rc;
    if (!ctx->has_scene || n_prim != ctx->n_prim) return fail(ctx, VP_ERR_USAGE, "primitive count mismatch");
    if (n_prim == 0) return VP_OK;
    if (!xf15) return fail(ctx, VP_ERR_USAGE, "null transforms");
    const bool dev = is_device_ptr(xf15);
    if (!dev) {
        for (int32_t k = 0; k < n_prim; ++k) {
            const float *s = xf15 + 15 * size_t(k) + 12;
            if (!(s[0] > 0) || !(s[1] > 0) || !(s[2] > 0))
                return fail(ctx, VP_ERR_USAGE, "non-positive composed primitive scale");
        }
    }
    VP_CUDA(ctx, ctx->xfb[ctx->xfi].ensure(size_t(n_prim) * 16));
    const float *src = xf15;
    if (!dev) {
        VP_CUDA(ctx, ctx->xf15_tmp.ensure(size_t(n_prim) * 15));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->xf15_tmp.p, xf15, sizeof(float) * 15 * size_t(n_prim),
                                     cudaMemcpyHostToDevice, ctx->stream));
        src = ctx->xf15_tmp.p;
    }
    VP_CUDA(ctx, launch_pad_xf(src, ctx->xfb[ctx->xfi].p, n_prim, ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->has_xf = true;
    ctx->bvh_dirty = true;
    return VP_OK;
}

int vp_set_transforms_async(vp_ctx *ctx, int32_t n_prim, const float *xf15, void *stream) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (!ctx->has_scene || n_prim != ctx->n_prim) return fail(ctx, VP_ERR_USAGE, "primitive count mismatch");
    if (n_prim == 0) return VP_OK;
    if (!xf15) return fail(ctx, VP_ERR_USAGE, "null transforms");
    if (!ctx->has_xf) return fail(ctx, VP_ERR_USAGE, "set the frame's transforms synchronously first");
    // Upload into the other buffer, once the binning and raymarch that last read it are done.
    // Without a caller stream the upload goes on the binning stream: enqueued on the render
    // stream it would wait for the raymarch in flight, and the next views' binning (which
    // waits for the upload) could not overlap that raymarch.
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->bin_stream;
    const int j = ctx->xfi ^ 1;
    VP_CUDA(ctx, ctx->xfb[j].ensure(size_t(n_prim) * 16));
    VP_CUDA(ctx, ctx->xf15_tmp.ensure(size_t(n_prim) * 15));
    VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_xf_binned[j], 0));
    VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_xf_marched[j], 0));
    // xf15_tmp is shared by every upload: the previous one (possibly on another stream) must
    // have finished reading it
    VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_xf, 0));
    VP_CUDA(ctx, cudaMemcpyAsync(ctx->xf15_tmp.p, xf15, sizeof(float) * 15 * size_t(n_prim), cudaMemcpyDefault, st));
    VP_CUDA(ctx, launch_pad_xf(ctx->xf15_tmp.p, ctx->xfb[j].p, n_prim, st));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_xf, st));
    if (st != ctx->stream) VP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_xf, 0));
    ctx->xfi = j;
    ctx->bvh_dirty = true;
    return VP_OK;
}

int vp_set_frame(vp_ctx *ctx, int32_t n_prim, const float *tr24) {
    NvtxRange nvtx_("vp_set_frame");
    if (int rc = check_ctx(ctx, false)) return rc;
    if (int rc = quiesce(ctx)) return rc;
    if (!ctx->has_scene || n_prim != ctx->n_prim) return fail(ctx, VP_ERR_USAGE, "primitive count mismatch");
    if (n_prim == 0) return VP_OK;
    if (!tr24) return fail(ctx, VP_ERR_USAGE, "null transforms");
    cudaStream_t st = ctx->stream;
    VP_CUDA(ctx, ctx->tr24.ensure(size_t(n_prim) * 24));
    VP_CUDA(ctx, ctx->xfb[ctx->xfi].ensure(size_t(n_prim) * 16));
    VP_CUDA(ctx, ctx->flag.ensure(1));
    if ((const void *)tr24 != (const void *)ctx->tr24.p)
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->tr24.p, tr24, sizeof(float) * 24 * size_t(n_prim),
                                     is_device_ptr(tr24) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    VP_CUDA(ctx, cudaMemsetAsync(ctx->flag.p, 0, sizeof(int), st));
    VP_CUDA(ctx, launch_compose(ctx->tr24.p, nullptr, n_prim, ctx->xfb[ctx->xfi].p, ctx->flag.p, st));
    int bad = 0;
    VP_CUDA(ctx, cudaMemcpyAsync(&bad, ctx->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    ctx->has_xf = !bad;
    ctx->bvh_dirty = true;
    if (bad) return fail(ctx, VP_ERR_USAGE, "non-positive composed primitive scale");
    return VP_OK;
}

int vp_get_transforms(vp_ctx *ctx, float *xf15) {
    if (int rc = check_ctx(ctx, true)) return rc;
    if (ctx->n_prim == 0) return VP_OK;
    if (!xf15) return fail(ctx, VP_ERR_USAGE, "null destination");
    VP_CUDA(ctx, cudaMemcpy2DAsync(xf15, 15 * sizeof(float), ctx->xfb[ctx->xfi].p, 16 * sizeof(float), 15 * sizeof(float),
                                   size_t(ctx->n_prim),
                                   is_device_ptr(xf15) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                   ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

// A host planar slab (pageable, e.g. the reference Scene's std::vector) into the resident
// interleaved payload: chunks of whole primitives go pageable -> page-locked staging (the copy
// pool's threads) -> device staging (copy engine) -> K0 repack, double-buffered, so the host
// copies of the next chunks overlap the transfer and repack of chunk i (four slots: the host
// copy outruns PCIe, so the copy engine never waits). Page-locked callers skip the
// host copy. The staging buffers persist in the context.
// The host copy threads (up to 7 besides the caller). If threads cannot be created the pool has
// none and copies run on the calling thread (an exception must not cross the C-ABI).
static void ensure_copy_pool(vp_ctx *ctx) {
    if (ctx->copy_pool) return;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    try {
        ctx->copy_pool = std::make_unique<CopyPool>(int(std::min(7u, hw > 1 ? hw - 1 : 0u)));
    } catch (...) {
        ctx->copy_pool = std::make_unique<CopyPool>(0);
    }
}

static int upload_planar_host(vp_ctx *ctx, const float *payload, int64_t n_prim, int64_t m3) {
    cudaStream_t st = ctx->stream;
    const size_t per_prim = 4 * size_t(m3);  // floats
    const size_t chunk_prims = std::max<size_t>(1, kStageBytes / (per_prim * 4));
    const size_t chunk_floats = chunk_prims * per_prim;
    cudaPointerAttributes attr{};
    const bool pinned =
        cudaPointerGetAttributes(&attr, payload) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    for (int i = 0; i < vp_ctx::kStageSlots; ++i) {
        VP_CUDA(ctx, ctx->stage_d[i].ensure(chunk_floats));
        if (!pinned && ctx->stage_h_floats[i] < chunk_floats) {
            if (ctx->stage_h[i]) cudaFreeHost(ctx->stage_h[i]);
            ctx->stage_h[i] = nullptr;
            ctx->stage_h_floats[i] = 0;
            VP_CUDA(ctx, cudaMallocHost(&ctx->stage_h[i], chunk_floats * sizeof(float)));
            ctx->stage_h_floats[i] = chunk_floats;
        }
    }
    if (!pinned) ensure_copy_pool(ctx);
    int slot = 0;
    for (size_t k0 = 0; k0 < size_t(n_prim); k0 += chunk_prims, slot = (slot + 1) % vp_ctx::kStageSlots) {
        const size_t nk = std::min(chunk_prims, size_t(n_prim) - k0), nfl = nk * per_prim;
        const float *src = payload + k0 * per_prim;
        if (!pinned) {  // the staging slot is free once its previous transfer has run
            VP_CUDA(ctx, cudaEventSynchronize(ctx->ev_stage[slot]));
            ctx->copy_pool->copy(ctx->stage_h[slot], src, nfl * sizeof(float));
            src = ctx->stage_h[slot];
        }
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->stage_d[slot].p, src, nfl * sizeof(float), cudaMemcpyHostToDevice, st));
        VP_CUDA(ctx, cudaEventRecord(ctx->ev_stage[slot], st));
        VP_CUDA(ctx, launch_repack(ctx->stage_d[slot].p, ctx->payload.p + k0 * size_t(m3), int64_t(nk), m3, st));
    }
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    return VP_OK;
}

// Device results into caller host memory. Page-locked destinations take a direct copy;
// pageable ones (e.g. the reference's RenderOutput vectors) are staged through one page-locked
// buffer, each array copied out by the copy pool as soon as its own transfer has landed.
struct HostOut {
    void *dst;
    const void *src;
    size_t bytes;
};
static int copy_out_host(vp_ctx *ctx, const HostOut *outs, int n, cudaStream_t st) {
    size_t staged = 0;
    bool pageable[3] = {};
    for (int i = 0; i < n; ++i) {
        cudaPointerAttributes attr{};
        pageable[i] = !(cudaPointerGetAttributes(&attr, outs[i].dst) == cudaSuccess &&
                        attr.type == cudaMemoryTypeHost);
        cudaGetLastError();
        if (pageable[i]) staged += (outs[i].bytes + 255) & ~size_t(255);
    }
    if (staged > ctx->out_stage_bytes) {
        if (ctx->out_stage) cudaFreeHost(ctx->out_stage);
        ctx->out_stage = nullptr;
        ctx->out_stage_bytes = 0;
        VP_CUDA(ctx, cudaMallocHost(&ctx->out_stage, staged));
        ctx->out_stage_bytes = staged;
    }
    if (staged) ensure_copy_pool(ctx);
    size_t off = 0;
    unsigned char *stage = static_cast<unsigned char *>(ctx->out_stage);
    for (int i = 0; i < n; ++i) {
        void *dst = pageable[i] ? stage + off : outs[i].dst;
        VP_CUDA(ctx, cudaMemcpyAsync(dst, outs[i].src, outs[i].bytes, cudaMemcpyDeviceToHost, st));
        VP_CUDA(ctx, cudaEventRecord(ctx->ev_out[i], st));
        if (pageable[i]) off += (outs[i].bytes + 255) & ~size_t(255);
    }
    off = 0;
    for (int i = 0; i < n; ++i) {
        VP_CUDA(ctx, cudaEventSynchronize(ctx->ev_out[i]));
        if (!pageable[i]) continue;
        ctx->copy_pool->copy(outs[i].dst, stage + off, outs[i].bytes);
        off += (outs[i].bytes + 255) & ~size_t(255);
    }
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    return VP_OK;
}

int vp_set_scene(vp_ctx *ctx, int32_t n_prim, int32_t m, const float *xf15,
                 const float *payload, float window_alpha, int32_t window_beta) {
    NvtxRange nvtx_("vp_set_scene");
    if (int rc = check_ctx(ctx, false)) return rc;
    if (int rc = quiesce(ctx)) return rc;
    if (n_prim < 0) return fail(ctx, VP_ERR_USAGE, "negative primitive count");
    if (n_prim > 0 && m < 1) return fail(ctx, VP_ERR_USAGE, "voxels per axis must be >= 1");
    if (!std::isfinite(window_alpha)) return fail(ctx, VP_ERR_USAGE, "window alpha must be finite");
    ctx->has_scene = false;
    ctx->bvh_built_n = 0;  // a new scene: rebuild the BVH topology, not just refit it
    ctx->n_prim = n_prim;
    ctx->m = m;
    ctx->w_alpha = window_alpha;
    ctx->w_beta = window_beta;
    ctx->has_scene = true;
    ctx->has_xf = false;
    if (n_prim == 0) return VP_OK;
    if (xf15) {
        if (int rc = vp_set_transforms(ctx, n_prim, xf15)) {
            ctx->has_scene = false;
            return rc;
        }
    } else {
        VP_CUDA(ctx, ctx->xfb[ctx->xfi].ensure(size_t(n_prim) * 16));
    }
    const int64_t m3 = int64_t(m) * m * m;
    const size_t nf = size_t(n_prim) * 4 * size_t(m3);
    VP_CUDA(ctx, ctx->payload.ensure(size_t(n_prim) * size_t(m3)));
    ctx->pairs_dirty = true;
    if (!payload) return VP_OK;  // filled later by vp_set_payload_interleaved
    if (!is_device_ptr(payload)) return upload_planar_host(ctx, payload, n_prim, m3);
    VP_CUDA(ctx, launch_repack(payload, ctx->payload.p, n_prim, m3, ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    (void)nf;
    return VP_OK;
}

int vp_set_payload_interleaved(vp_ctx *ctx, int32_t n_prim, int32_t m, const float *inter) {
    if (int rc = check_ctx(ctx, true, false)) return rc;
    if (int rc = quiesce(ctx)) return rc;
    if (n_prim != ctx->n_prim || m != ctx->m) return fail(ctx, VP_ERR_USAGE, "payload shape mismatch");
    if (n_prim == 0) return VP_OK;
    if (!inter) return fail(ctx, VP_ERR_USAGE, "null payload");
    const size_t n4 = size_t(n_prim) * size_t(m) * m * m;
    VP_CUDA(ctx, ctx->payload.ensure(n4));
    ctx->pairs_dirty = true;
    if ((const void *)inter != (const void *)ctx->payload.p)
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->payload.p, inter, n4 * sizeof(float4),
                                     is_device_ptr(inter) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                     ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int vp_payload_device(vp_ctx *ctx, float **dev_ptr, int64_t *n_floats) {
    if (int rc = check_ctx(ctx, true, false)) return rc;
    ctx->pairs_dirty = true;  // the caller may write through the pointer (a broadcast's destination)
    if (dev_ptr) *dev_ptr = reinterpret_cast<float *>(ctx->payload.p);
    if (n_floats) *n_floats = int64_t(ctx->n_prim) * ctx->m * ctx->m * ctx->m * 4;
    return VP_OK;
}

int vp_copy_payload(vp_ctx *ctx, float *dst) {
    if (int rc = check_ctx(ctx, true, false)) return rc;
    const size_t n4 = size_t(ctx->n_prim) * size_t(ctx->m) * ctx->m * ctx->m;
    if (n4 == 0) return VP_OK;
    if (!dst) return fail(ctx, VP_ERR_USAGE, "null destination");
    VP_CUDA(ctx, cudaMemcpyAsync(dst, ctx->payload.p, n4 * sizeof(float4),
                                 is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int vp_kernel_times(vp_ctx *ctx, int64_t max, float *march_ms, int64_t *n) {
    if (int rc = check_ctx(ctx, false)) return rc;
    const int64_t avail = std::min<int64_t>(ctx->t_count, kTimingSlots);
    const int64_t first = ctx->t_count - avail;
    int64_t w = 0;
    for (int64_t i = first; i < ctx->t_count && w < max; ++i, ++w) {
        const int slot = int(i % kTimingSlots);
        VP_CUDA(ctx, cudaEventSynchronize(ctx->t_ev[2 * slot + 1]));
        float ms = 0.f;
        VP_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->t_ev[2 * slot], ctx->t_ev[2 * slot + 1]));
        if (march_ms) march_ms[w] = ms;
    }
    if (n) *n = w;
    ctx->t_count = 0;
    return VP_OK;
}

int vp_render_async(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, float *rgb_dev,
                    float *alpha_dev, int32_t *samples_dev, void *stream) {
    NvtxRange nvtx_("vp_render_async");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_cam(ctx, cam)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    const CamDev cd = make_cam(*cam);
    const size_t n_px = size_t(cam->width) * cam->height;
    if (n_px == 0) return VP_OK;
    if (!rgb_dev || !alpha_dev) return fail(ctx, VP_ERR_USAGE, "null output");
    if (ctx->n_prim == 0) {
        VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
        VP_CUDA(ctx, cudaMemsetAsync(rgb_dev, 0, n_px * 3 * sizeof(float), st));
        VP_CUDA(ctx, cudaMemsetAsync(alpha_dev, 0, n_px * sizeof(float), st));
        if (samples_dev) VP_CUDA(ctx, cudaMemsetAsync(samples_dev, 0, n_px * sizeof(int32_t), st));
        return VP_OK;
    }
    if (int rc = ensure_render_buffers(ctx, cd)) return rc;
    const bool host_out = !is_device_ptr(rgb_dev);
    if (!host_out) {
        if (!is_device_ptr(alpha_dev) || (samples_dev && !is_device_ptr(samples_dev)))
            return fail(ctx, VP_ERR_USAGE, "outputs must be all device or all host pointers");
        const OutDev od{rgb_dev, alpha_dev, samples_dev};
        return enqueue_render(ctx, cd, make_march(ctx, cfg), od, st);
    }
    if (is_device_ptr(alpha_dev) || (samples_dev && is_device_ptr(samples_dev)))
        return fail(ctx, VP_ERR_USAGE, "outputs must be all device or all host pointers");
    // host outputs: render into a device slot, copy it out on copy_stream while the next view
    // renders; the slot is reused only after its previous copy finished
    const int q = ctx->ring_next;
    ctx->ring_next ^= 1;
    VP_CUDA(ctx, ctx->ring_rgb[q].ensure(3 * n_px));
    VP_CUDA(ctx, ctx->ring_alpha[q].ensure(n_px));
    if (samples_dev) VP_CUDA(ctx, ctx->ring_samples[q].ensure(n_px));
    VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_copied[q], 0));
    const OutDev od{ctx->ring_rgb[q].p, ctx->ring_alpha[q].p, samples_dev ? ctx->ring_samples[q].p : nullptr};
    if (int rc = enqueue_render(ctx, cd, make_march(ctx, cfg), od, st)) return rc;
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_rendered[q], st));
    VP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_rendered[q], 0));
    VP_CUDA(ctx, cudaMemcpyAsync(rgb_dev, od.rgb, 12 * n_px, cudaMemcpyDeviceToHost, ctx->copy_stream));
    VP_CUDA(ctx, cudaMemcpyAsync(alpha_dev, od.alpha, 4 * n_px, cudaMemcpyDeviceToHost, ctx->copy_stream));
    if (samples_dev)
        VP_CUDA(ctx, cudaMemcpyAsync(samples_dev, od.samples, 4 * n_px, cudaMemcpyDeviceToHost, ctx->copy_stream));
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_copied[q], ctx->copy_stream));
    return VP_OK;
}

int64_t vp_shard_tiles(int32_t width, int32_t height, int32_t shard, int32_t n_shards) {
    if (width <= 0 || height <= 0 || n_shards < 1 || shard < 0 || shard >= n_shards) return 0;
    const int64_t n_tiles = int64_t((width + 15) / 16) * ((height + 15) / 16);
    return n_tiles > shard ? (n_tiles - shard + n_shards - 1) / n_shards : 0;
}

int vp_render_shard_async(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, int32_t shard,
                          int32_t n_shards, float *rgb, float *alpha, int32_t *samples, void *stream) {
    NvtxRange nvtx_("vp_render_shard_async");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_cam(ctx, cam)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(ctx, VP_ERR_USAGE, "bad shard index");
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    const int64_t slots = vp_shard_tiles(cam->width, cam->height, shard, n_shards);
    if (slots == 0) return VP_OK;
    if (!rgb || !alpha) return fail(ctx, VP_ERR_USAGE, "null output");
    if (!is_device_ptr(rgb) || !is_device_ptr(alpha) || (samples && !is_device_ptr(samples)))
        return fail(ctx, VP_ERR_USAGE, "shard outputs must be device pointers");
    const size_t n_px = size_t(slots) * 256;
    if (ctx->n_prim == 0) {
        VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
        VP_CUDA(ctx, cudaMemsetAsync(rgb, 0, n_px * 3 * sizeof(float), st));
        VP_CUDA(ctx, cudaMemsetAsync(alpha, 0, n_px * sizeof(float), st));
        if (samples) VP_CUDA(ctx, cudaMemsetAsync(samples, 0, n_px * sizeof(int32_t), st));
        return VP_OK;
    }
    CamDev cd = make_cam(*cam);
    cd.n_shards = n_shards;
    cd.shard = shard;
    if (int rc = ensure_render_buffers(ctx, cd)) return rc;
    OutDev od{rgb, alpha, samples};
    od.shard_n = n_shards;
    od.width = cd.width;
    od.tiles_x = cd.tiles_x;
    return enqueue_views(ctx, 1, &cd, make_march(ctx, cfg), &od, st, int(slots));
}

int vp_render_batch_async(vp_ctx *ctx, int32_t n_views, const vp_camera *cams, const vp_march *cfg,
                          float *const *rgb, float *const *alpha, int32_t *const *samples, void *stream) {
    NvtxRange nvtx_("vp_render_batch_async");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    if (n_views < 1 || n_views > kMaxViews) return fail(ctx, VP_ERR_USAGE, "1 to 16 views per batch");
    if (!cams || !rgb || !alpha || !rgb[0]) return fail(ctx, VP_ERR_USAGE, "null arguments");
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    const bool host_out = !is_device_ptr(rgb[0]);
    CamDev cds[kMaxViews];
    OutDev ods[kMaxViews];
    size_t px_off[kMaxViews + 1] = {0};
    for (int v = 0; v < n_views; ++v) {
        if (int rc = check_cam(ctx, &cams[v])) return rc;
        const size_t n_px = size_t(cams[v].width) * cams[v].height;
        if (n_px == 0) return fail(ctx, VP_ERR_USAGE, "empty view in a batch");
        int32_t *sp = samples ? samples[v] : nullptr;
        if (!rgb[v] || !alpha[v] || is_device_ptr(rgb[v]) != !host_out || is_device_ptr(alpha[v]) != !host_out ||
            (sp && is_device_ptr(sp) != !host_out))
            return fail(ctx, VP_ERR_USAGE, "batch outputs must be all device or all host pointers");
        cds[v] = make_cam(cams[v]);
        ods[v] = OutDev{rgb[v], alpha[v], sp};
        px_off[v + 1] = px_off[v] + n_px;
    }
    const int g = ctx->group ^ 1;  // the slot group enqueue_views is about to use
    if (host_out) {  // render into the group's device outputs; copied out on copy_stream
        VP_CUDA(ctx, ctx->bring_rgb[g].ensure(3 * px_off[n_views]));
        VP_CUDA(ctx, ctx->bring_alpha[g].ensure(px_off[n_views]));
        if (samples) VP_CUDA(ctx, ctx->bring_samples[g].ensure(px_off[n_views]));
        VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_bcopied[g], 0));
        for (int v = 0; v < n_views; ++v)
            ods[v] = OutDev{ctx->bring_rgb[g].p + 3 * px_off[v], ctx->bring_alpha[g].p + px_off[v],
                            samples && samples[v] ? ctx->bring_samples[g].p + px_off[v] : nullptr};
    }
    if (ctx->n_prim == 0) {
        for (int v = 0; v < n_views; ++v) {
            const size_t n_px = px_off[v + 1] - px_off[v];
            VP_CUDA(ctx, cudaMemsetAsync(ods[v].rgb, 0, 12 * n_px, st));
            VP_CUDA(ctx, cudaMemsetAsync(ods[v].alpha, 0, 4 * n_px, st));
            if (ods[v].samples) VP_CUDA(ctx, cudaMemsetAsync(ods[v].samples, 0, 4 * n_px, st));
        }
        ctx->group = g;
    } else if (int rc = enqueue_views(ctx, n_views, cds, make_march(ctx, cfg), ods, st)) {
        return rc;
    }
    if (!host_out) return VP_OK;
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_brendered[g], st));
    VP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_brendered[g], 0));
    for (int v = 0; v < n_views; ++v) {
        const size_t n_px = px_off[v + 1] - px_off[v];
        VP_CUDA(ctx, cudaMemcpyAsync(rgb[v], ods[v].rgb, 12 * n_px, cudaMemcpyDeviceToHost, ctx->copy_stream));
        VP_CUDA(ctx, cudaMemcpyAsync(alpha[v], ods[v].alpha, 4 * n_px, cudaMemcpyDeviceToHost, ctx->copy_stream));
        if (ods[v].samples)
            VP_CUDA(ctx, cudaMemcpyAsync(samples[v], ods[v].samples, 4 * n_px, cudaMemcpyDeviceToHost,
                                         ctx->copy_stream));
    }
    VP_CUDA(ctx, cudaEventRecord(ctx->ev_bcopied[g], ctx->copy_stream));
    return VP_OK;
}

int vp_sync(vp_ctx *ctx) {
    if (int rc = check_ctx(ctx, false)) return rc;
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
    return VP_OK;
}

int vp_set_key_capacity(vp_ctx *ctx, int64_t keys, int32_t grow) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (keys < 0 || keys > int64_t(0xfffffffe)) return fail(ctx, VP_ERR_USAGE, "key capacity out of range");
    ctx->entries_cap = keys;  // 0: the default, max(2^20, 16 K), at the next render
    ctx->key_cap_fixed = keys > 0 && grow == 0;
    return VP_OK;
}

int vp_read_stats(vp_ctx *ctx, vp_stats *stats) {
    if (int rc = check_ctx(ctx, false)) return rc;
    // the latest launch may still run on a caller's stream
    VP_CUDA(ctx, cudaEventSynchronize(ctx->ev_last_marched));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    DevCounters c{};
    unsigned long long max_keys = 0;  // the key capacity a single view needs
    for (int v = 0; v < (ctx->last_n > 1 ? ctx->last_n : 1); ++v) {  // a batch: summed over its views
        VP_CUDA(ctx, cudaMemcpy(ctx->h_ctr, ctx->last_n > 1 ? ctx->last_ctr[v] : ctx->d_ctr, sizeof(DevCounters),
                                cudaMemcpyDeviceToHost));
        const DevCounters &q = *ctx->h_ctr;
        c.ray_samples += q.ray_samples;
        c.prim_samples += q.prim_samples;
        c.hit_rays += q.hit_rays;
        c.early_exits += q.early_exits;
        c.saturated += q.saturated;
        c.overflow_rays += q.overflow_rays;
        c.refills += q.refills;
        c.keys += q.keys;
        max_keys = std::max(max_keys, q.keys);
        c.numeric_fail += q.numeric_fail;
        c.nonempty_tiles += q.nonempty_tiles;
        c.key_overflow |= q.key_overflow;
        c.fallback_fail |= q.fallback_fail;
        c.huge_rays += q.huge_rays;
    }
    note_density(ctx, c);
    fill_stats(c, 0.f, stats);
    note_keys(ctx, max_keys);  // key-overflowed tiles were rendered by K5b; grow for the next render
    return check_counters(ctx, c);
}

int vp_render(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, float *rgb, float *alpha,
              int32_t *samples, vp_stats *stats) {
    NvtxRange nvtx_("vp_render");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_cam(ctx, cam)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    const size_t n_px = size_t(cam->width) * cam->height;
    if (stats) std::memset(stats, 0, sizeof *stats);
    if (n_px == 0) return VP_OK;
    if (!rgb || !alpha) return fail(ctx, VP_ERR_USAGE, "null output");
    const bool d_rgb = is_device_ptr(rgb), d_alpha = is_device_ptr(alpha);
    const bool d_samp = samples && is_device_ptr(samples);
    cudaStream_t st = ctx->stream;
    if (ctx->n_prim == 0) {  // march.cpp:108: empty frame renders a zero image
        if (d_rgb) VP_CUDA(ctx, cudaMemset(rgb, 0, n_px * 3 * sizeof(float)));
        else std::memset(rgb, 0, n_px * 3 * sizeof(float));
        if (d_alpha) VP_CUDA(ctx, cudaMemset(alpha, 0, n_px * sizeof(float)));
        else std::memset(alpha, 0, n_px * sizeof(float));
        if (samples) {
            if (d_samp) VP_CUDA(ctx, cudaMemset(samples, 0, n_px * sizeof(int32_t)));
            else std::memset(samples, 0, n_px * sizeof(int32_t));
        }
        return VP_OK;
    }
    const CamDev cd = make_cam(*cam);
    const MarchDev mp = make_march(ctx, cfg);
    OutDev od{rgb, alpha, samples};
    if (!d_rgb) {
        VP_CUDA(ctx, ctx->out_rgb.ensure(n_px * 3));
        od.rgb = ctx->out_rgb.p;
    }
    if (!d_alpha) {
        VP_CUDA(ctx, ctx->out_alpha.ensure(n_px));
        od.alpha = ctx->out_alpha.p;
    }
    if (samples && !d_samp) {
        VP_CUDA(ctx, ctx->out_samples.ensure(n_px));
        od.samples = ctx->out_samples.p;
    }
    {
        if (int rc = ensure_render_buffers(ctx, cd)) return rc;
        VP_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
        if (int rc = enqueue_render(ctx, cd, mp, od, st)) return rc;
        VP_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
        VP_CUDA(ctx, cudaStreamSynchronize(st));
        const DevCounters c = *ctx->h_ctr;
        note_density(ctx, c);
        note_keys(ctx, c.keys);  // overflowed tiles were marched by K5b; size for the next render
        HostOut outs[3];
        int n_out = 0;
        if (!d_rgb) outs[n_out++] = HostOut{rgb, od.rgb, n_px * 3 * sizeof(float)};
        if (!d_alpha) outs[n_out++] = HostOut{alpha, od.alpha, n_px * sizeof(float)};
        if (samples && !d_samp) outs[n_out++] = HostOut{samples, od.samples, n_px * sizeof(int32_t)};
        if (int rc = copy_out_host(ctx, outs, n_out, st)) return rc;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        fill_stats(c, ms, stats);
        return check_counters(ctx, c);
    }
}

int vp_march_rays(vp_ctx *ctx, int64_t n_rays, const float *origins, const float *dirs,
                  const float *jitter01, const vp_march *cfg, float *rgb, float *alpha,
                  int32_t *samples) {
    NvtxRange nvtx_("vp_march_rays");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    if (n_rays < 0) return fail(ctx, VP_ERR_USAGE, "negative ray count");
    if (n_rays == 0) return VP_OK;
    if (!origins || !dirs || !rgb || !alpha) return fail(ctx, VP_ERR_USAGE, "null ray arrays");
    cudaStream_t st = ctx->stream;
    const size_t n = size_t(n_rays);
    RaysDev rays{origins, dirs, jitter01};
    if (!is_device_ptr(origins)) {
        VP_CUDA(ctx, ctx->ray_o.ensure(3 * n));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_o.p, origins, 12 * n, cudaMemcpyHostToDevice, st));
        rays.origins = ctx->ray_o.p;
    }
    if (!is_device_ptr(dirs)) {
        VP_CUDA(ctx, ctx->ray_d.ensure(3 * n));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_d.p, dirs, 12 * n, cudaMemcpyHostToDevice, st));
        rays.dirs = ctx->ray_d.p;
    }
    if (jitter01 && !is_device_ptr(jitter01)) {
        VP_CUDA(ctx, ctx->ray_j.ensure(n));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_j.p, jitter01, 4 * n, cudaMemcpyHostToDevice, st));
        rays.jitter = ctx->ray_j.p;
    }
    const bool d_rgb = is_device_ptr(rgb), d_alpha = is_device_ptr(alpha);
    const bool d_samp = samples && is_device_ptr(samples);
    OutDev od{rgb, alpha, samples};
    if (!d_rgb) { VP_CUDA(ctx, ctx->out_rgb.ensure(3 * n)); od.rgb = ctx->out_rgb.p; }
    if (!d_alpha) { VP_CUDA(ctx, ctx->out_alpha.ensure(n)); od.alpha = ctx->out_alpha.p; }
    if (samples && !d_samp) { VP_CUDA(ctx, ctx->out_samples.ensure(n)); od.samples = ctx->out_samples.p; }
    if (size_t(ctx->ovf_cap) < n) {
        VP_CUDA(ctx, ctx->ovf_list.ensure(n));
        ctx->ovf_cap = int(n);
    }
    if (int rc = ensure_fallback(ctx)) return rc;
    MarchDev mp = make_march(ctx, cfg);
    if (int rc = ensure_bvh(ctx, mp)) return rc;
    VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
    if (ctx->n_prim == 0) {
        VP_CUDA(ctx, cudaMemsetAsync(od.rgb, 0, 12 * n, st));
        VP_CUDA(ctx, cudaMemsetAsync(od.alpha, 0, 4 * n, st));
        if (od.samples) VP_CUDA(ctx, cudaMemsetAsync(od.samples, 0, 4 * n, st));
    } else {
        VP_CUDA(ctx, launch_march_rays(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, rays, n_rays, od,
                                       ctx->d_ctr, ctx->ovf_list.p, ctx->ovf_cap, st));
        const CamDev none{};
        VP_CUDA(ctx, launch_march_fallback(true, none, mp, ctx->xfb[ctx->xfi].p, nullptr, ctx->n_prim, ctx->payload.p,
                                           nullptr, nullptr, od, rays, ctx->d_ctr, ctx->ovf_list.p,
                                           ctx->ovf_cap, ctx->fb_e.p, ctx->fb_x.p, ctx->fb_c.p, st,
                                           ctx->huge_ray_list.p, kHugeListCap));
        VP_CUDA(ctx, launch_march_huge_rays(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, od, rays, ctx->d_ctr,
                                            ctx->huge_ray_list.p, kHugeListCap, ctx->hg_e.p, ctx->hg_x.p, ctx->hg_c.p,
                                            st));
    }
    if (!d_rgb) VP_CUDA(ctx, cudaMemcpyAsync(rgb, od.rgb, 12 * n, cudaMemcpyDeviceToHost, st));
    if (!d_alpha) VP_CUDA(ctx, cudaMemcpyAsync(alpha, od.alpha, 4 * n, cudaMemcpyDeviceToHost, st));
    if (samples && !d_samp) VP_CUDA(ctx, cudaMemcpyAsync(samples, od.samples, 4 * n, cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    return check_counters(ctx, *ctx->h_ctr);
}

int vp_composite(vp_ctx *ctx, int32_t width, int32_t height, const float *rgb, const float *alpha,
                 const float *background, float *out) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (width < 0 || height < 0) return fail(ctx, VP_ERR_USAGE, "background dimensions do not match render");
    const size_t n = size_t(width) * height;
    if (n == 0) return VP_OK;
    if (!rgb || !alpha || !background || !out) return fail(ctx, VP_ERR_USAGE, "null image");
    cudaStream_t st = ctx->stream;
    DBuf<float> tmp;
    const float *d_in[3] = {rgb, alpha, background};
    const size_t sz[3] = {3 * n, n, 3 * n};
    size_t total = 0;
    for (int i = 0; i < 3; ++i)
        if (!is_device_ptr(d_in[i])) total += sz[i];
    const bool d_out = is_device_ptr(out);
    if (!d_out) total += 3 * n;
    VP_CUDA(ctx, tmp.ensure(total));
    size_t off = 0;
    for (int i = 0; i < 3; ++i)
        if (!is_device_ptr(d_in[i])) {
            VP_CUDA(ctx, cudaMemcpyAsync(tmp.p + off, d_in[i], sz[i] * 4, cudaMemcpyHostToDevice, st));
            d_in[i] = tmp.p + off;
            off += sz[i];
        }
    float *o = d_out ? out : tmp.p + off;
    VP_CUDA(ctx, launch_composite(d_in[0], d_in[1], d_in[2], o, int64_t(n), st));
    if (!d_out) VP_CUDA(ctx, cudaMemcpyAsync(out, o, 12 * n, cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    tmp.release();
    return VP_OK;
}

int vp_debug_tiles(vp_ctx *ctx, const vp_camera *cam, int32_t *rect4, uint32_t *depth_key,
                   int32_t *tile_offsets, int32_t *tile_prims, int64_t cap, int64_t *n_keys) {
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_cam(ctx, cam)) return rc;
    const CamDev cd = make_cam(*cam);
    const size_t n_tiles = size_t(cd.tiles_x) * cd.tiles_y;
    cudaStream_t st = ctx->stream;
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->bin_stream));
    ctx->cur = 0;  // slot 0, synchronously on the context stream
    ctx->d_ctr = ctx->slot[0].d_ctr;
    for (int attempt = 0; attempt < 3; ++attempt) {
        if (int rc = ensure_render_buffers(ctx, cd)) return rc;
        VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
        VP_CUDA(ctx, launch_binning(cd, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->bs().rects.p, ctx->bs().prects.p, ctx->bs().keys.p,
                                    ctx->bs().tile_counts.p, ctx->bs().offsets.p, ctx->bs().cursor.p, ctx->bs().order.p, ctx->bs().entries.p,
                                    ctx->entries_cap, ctx->d_ctr, st));
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
        VP_CUDA(ctx, cudaStreamSynchronize(st));
        const DevCounters c = *ctx->h_ctr;
        if (c.key_overflow) {
            ctx->entries_cap = int64_t(c.keys) + int64_t(c.keys) / 4 + 1024;
            continue;
        }
        const size_t nk = size_t(c.keys);
        if (n_keys) *n_keys = int64_t(nk);
        if (rect4 && ctx->n_prim > 0)
            VP_CUDA(ctx, cudaMemcpy(rect4, ctx->bs().rects.p, sizeof(int4) * ctx->n_prim, cudaMemcpyDeviceToHost));
        if (depth_key && ctx->n_prim > 0)
            VP_CUDA(ctx, cudaMemcpy(depth_key, ctx->bs().keys.p, sizeof(uint32_t) * ctx->n_prim, cudaMemcpyDeviceToHost));
        if (tile_offsets)
            VP_CUDA(ctx, cudaMemcpy(tile_offsets, ctx->bs().offsets.p, sizeof(uint32_t) * (n_tiles + 1),
                                    cudaMemcpyDeviceToHost));
        if (tile_prims && cap > 0 && nk > 0) {
            std::vector<unsigned long long> e(nk);
            VP_CUDA(ctx, cudaMemcpy(e.data(), ctx->bs().entries.p, nk * 8, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < nk && int64_t(i) < cap; ++i) tile_prims[i] = int32_t(e[i] & 0xffffffffull);
        }
        return VP_OK;
    }
    return fail(ctx, VP_ERR_DEVICE, "tile key buffer could not be sized");
}

}  // extern "C"

namespace {
// backwardRay over a batch; fwd_state (device, 8 floats per ray, written by the forward march
// of the same rays) lets the kernel skip its replay of march().
int backward_rays(vp_ctx *ctx, int64_t n_rays, const float *origins, const float *dirs, const float *jitter01,
                  const float *adj_rgb, const float *adj_alpha, const vp_march *cfg, const float *transforms24,
                  float *grads, int32_t accumulate, const float *fwd_state, const float *fwd_segs) {
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    if (n_rays < 0) return fail(ctx, VP_ERR_USAGE, "negative ray count");
    const int k = ctx->n_prim, m = ctx->m;
    const size_t n_pay = size_t(k) * 4 * m * m * m, n_grad = n_pay + 9 * size_t(k);
    if (!grads) return fail(ctx, VP_ERR_USAGE, "null gradient buffer");
    if (k > 0 && !transforms24) return fail(ctx, VP_ERR_USAGE, "null transforms");
    if (n_rays > 0 && (!origins || !dirs || !adj_rgb || !adj_alpha))
        return fail(ctx, VP_ERR_USAGE, "null ray arrays");
    cudaStream_t st = ctx->stream;
    const bool d_grads = is_device_ptr(grads);
    DBuf<float> &g = ctx->s_bwd_g, &pose = ctx->s_bwd_pose, &adj = ctx->s_bwd_adj;
    float *dg = grads;
    if (!d_grads) {
        VP_CUDA(ctx, g.ensure(n_grad));
        dg = g.p;
        if (accumulate) VP_CUDA(ctx, cudaMemcpyAsync(dg, grads, n_grad * 4, cudaMemcpyHostToDevice, st));
    }
    // v4: the payload gradient is scattered channel-interleaved (one 16-byte reduction per
    // corner) into ctx->g_pay4, kept zeroed between calls, then transposed into dg
    constexpr int64_t kV4MinRays = 16384, kPairsMinRays = 8192;
    const bool pairs = ctx->bwd_warp_walk == 0 || (ctx->bwd_warp_walk < 0 && n_rays >= kPairsMinRays);
    const bool v4 = k > 0 && n_rays > 0 && (ctx->bwd_v4 == 1 || (ctx->bwd_v4 < 0 && pairs && n_rays >= kV4MinRays));
    // the gradient buffers are cleared once the forward is queued (below), or here without rays
    auto clear_grads = [&](cudaStream_t st) -> int {
        if (v4) {
            if (ctx->g_pay4.n < n_pay) {
                VP_CUDA(ctx, ctx->g_pay4.ensure(n_pay));
                VP_CUDA(ctx, cudaMemsetAsync(ctx->g_pay4.p, 0, n_pay * 4, st));
                ctx->g4_dirty[0] = false;
            }
            if (pairs && ctx->g_pay4b.n < n_pay) {
                VP_CUDA(ctx, ctx->g_pay4b.ensure(n_pay));
                VP_CUDA(ctx, cudaMemsetAsync(ctx->g_pay4b.p, 0, n_pay * 4, st));
                ctx->g4_dirty[1] = false;
            }
            if (!pairs) ctx->g4_cur = 0;  // the single-buffer path clears in the transpose
            // a dirty buffer is cleared whole: an earlier, larger scene may have written past n_pay
            DBuf<float> &g4b = ctx->g4_cur ? ctx->g_pay4b : ctx->g_pay4;
            if (ctx->g4_dirty[ctx->g4_cur]) {  // not cleared during an earlier call
                VP_CUDA(ctx, cudaMemsetAsync(g4b.p, 0, g4b.n * 4, st));
                ctx->g4_dirty[ctx->g4_cur] = false;
            }
            VP_CUDA(ctx, ctx->g_touched.ensure(size_t(k)));
            // the flags and the pose part are cleared by copies from a zero block: on the
            // auxiliary stream they then run at once instead of waiting for the forward's SMs
            if (ctx->h_zeros_n < 9 * size_t(k)) {
                if (ctx->h_zeros) cudaFreeHost(ctx->h_zeros);
                ctx->h_zeros = nullptr;
                ctx->h_zeros_n = 0;
                VP_CUDA(ctx, cudaMallocHost(&ctx->h_zeros, 9 * size_t(k) * 4));
                memset(ctx->h_zeros, 0, 9 * size_t(k) * 4);
                ctx->h_zeros_n = 9 * size_t(k);
            }
            VP_CUDA(ctx, cudaMemcpyAsync(ctx->g_touched.p, ctx->h_zeros, 4 * size_t(k), cudaMemcpyHostToDevice, st));
            if (!accumulate)
                VP_CUDA(ctx, cudaMemcpyAsync(dg + n_pay, ctx->h_zeros, (n_grad - n_pay) * 4, cudaMemcpyHostToDevice, st));
        } else if (!accumulate) {
            VP_CUDA(ctx, cudaMemsetAsync(dg, 0, n_grad * 4, st));
        }
        return VP_OK;
    };
    if (!(k > 0 && n_rays > 0))
        if (int rc = clear_grads(st)) return rc;
    if (k > 0 && n_rays > 0) {
        const size_t n = size_t(n_rays);
        RaysDev rays{origins, dirs, jitter01};
        if (!is_device_ptr(origins)) {
            VP_CUDA(ctx, ctx->ray_o.ensure(3 * n));
            VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_o.p, origins, 12 * n, cudaMemcpyHostToDevice, st));
            rays.origins = ctx->ray_o.p;
        }
        if (!is_device_ptr(dirs)) {
            VP_CUDA(ctx, ctx->ray_d.ensure(3 * n));
            VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_d.p, dirs, 12 * n, cudaMemcpyHostToDevice, st));
            rays.dirs = ctx->ray_d.p;
        }
        if (jitter01 && !is_device_ptr(jitter01)) {
            VP_CUDA(ctx, ctx->ray_j.ensure(n));
            VP_CUDA(ctx, cudaMemcpyAsync(ctx->ray_j.p, jitter01, 4 * n, cudaMemcpyHostToDevice, st));
            rays.jitter = ctx->ray_j.p;
        }
        const float *a_rgb = adj_rgb, *a_alpha = adj_alpha;
        if (!is_device_ptr(adj_rgb) || !is_device_ptr(adj_alpha)) {
            VP_CUDA(ctx, adj.ensure(4 * n));
            VP_CUDA(ctx, cudaMemcpyAsync(adj.p, adj_rgb, 12 * n, cudaMemcpyDefault, st));
            VP_CUDA(ctx, cudaMemcpyAsync(adj.p + 3 * n, adj_alpha, 4 * n, cudaMemcpyDefault, st));
            a_rgb = adj.p;
            a_alpha = adj.p + 3 * n;
        }
        if (int rc = ensure_fallback(ctx)) return rc;
        VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
        MarchDev mp = make_march(ctx, cfg);
        if (int rc = ensure_bvh(ctx, mp)) return rc;
        // the auxiliary stream (the pose data beside the forward; K6c beside the transpose):
        // ev_aux_pose marks the ray stream's work before the forward
        if (pairs) {
            if (!ctx->aux_stream) {
                VP_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
                VP_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_aux_fork, cudaEventDisableTiming));
                VP_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_aux_join, cudaEventDisableTiming));
                VP_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_aux_pose, cudaEventDisableTiming));
            }
            VP_CUDA(ctx, cudaEventRecord(ctx->ev_aux_pose, st));
        }
        if (!fwd_state) {
            // forward march of the same rays first, recording the MarchResult bookkeeping, so
            // the backward kernel does not replay march() itself
            VP_CUDA(ctx, ctx->s_bwd_fwd.ensure((12 + 3 * kRaySegs) * n));
            OutDev od{ctx->s_bwd_fwd.p, ctx->s_bwd_fwd.p + 3 * n, nullptr};
            od.state = ctx->s_bwd_fwd.p + 4 * n;
            od.segs = ctx->s_bwd_fwd.p + 12 * n;
            if (size_t(ctx->ovf_cap) < n) {
                VP_CUDA(ctx, ctx->ovf_list.ensure(n));
                ctx->ovf_cap = int(n);
            }
            VP_CUDA(ctx, launch_march_rays(mp, ctx->xfb[ctx->xfi].p, k, ctx->payload.p, rays, n_rays, od, ctx->d_ctr,
                                           ctx->ovf_list.p, ctx->ovf_cap, st));
            const CamDev none{};
            VP_CUDA(ctx, launch_march_fallback(true, none, mp, ctx->xfb[ctx->xfi].p, nullptr, k, ctx->payload.p, nullptr,
                                               nullptr, od, rays, ctx->d_ctr, ctx->ovf_list.p, ctx->ovf_cap,
                                               ctx->fb_e.p, ctx->fb_x.p, ctx->fb_c.p, st, ctx->huge_ray_list.p,
                                               kHugeListCap));
            VP_CUDA(ctx, launch_march_huge_rays(mp, ctx->xfb[ctx->xfi].p, k, ctx->payload.p, od, rays, ctx->d_ctr,
                                                ctx->huge_ray_list.p, kHugeListCap, ctx->hg_e.p, ctx->hg_x.p,
                                                ctx->hg_c.p, st));
            fwd_state = od.state;
            fwd_segs = od.segs;
        }
        // pose data on the device (k_pose36, the reference's operation order): rBase and
        // dR(deltaR)/dv_i per primitive; pose = [36 K | the records, if they are on the host].
        // Queued after the forward, on the auxiliary stream when there is one: it runs beside
        // the forward (a pageable upload of the records included), and the ray stream waits for
        // it before anything reads it.
        cudaStream_t sp = st;
        if (pairs) {
            VP_CUDA(ctx, cudaStreamWaitEvent(ctx->aux_stream, ctx->ev_aux_pose, 0));  // st before the forward
            sp = ctx->aux_stream;
        }
        // order on the auxiliary stream: the records' upload (copy engine, at once), then the
        // kernels, which find SM slots only as the forward's last CTAs retire
        VP_CUDA(ctx, pose.ensure(36 * size_t(k) + 24 * size_t(k)));
        const float *d_tr = transforms24;
        if (!is_device_ptr(transforms24)) {
            VP_CUDA(ctx, cudaMemcpyAsync(pose.p + 36 * size_t(k), transforms24, 96 * size_t(k),
                                         cudaMemcpyHostToDevice, sp));
            d_tr = pose.p + 36 * size_t(k);
        }
        if (int rc = clear_grads(sp)) return rc;  // (beside the forward: it reads none of these)
        VP_CUDA(ctx, launch_pose36(d_tr, k, pose.p, sp));
        if (v4 && sp != st && ctx->g4_dirty[ctx->g4_cur ^ 1]) {  // the idle gradient buffer, beside the forward
            DBuf<float> &idle = ctx->g4_cur ? ctx->g_pay4 : ctx->g_pay4b;
            VP_CUDA(ctx, cudaMemsetAsync(idle.p, 0, idle.n * 4, sp));
            ctx->g4_dirty[ctx->g4_cur ^ 1] = false;
        }
        if (sp != st) {
            VP_CUDA(ctx, cudaEventRecord(ctx->ev_aux_join, sp));
            VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_aux_join, 0));
        }
        BwdDev bd{dg, dg + n_pay, pose.p, a_rgb, a_alpha, fwd_state, fwd_segs};
        if (v4) {
            bd.g_pay4 = ctx->g4_cur ? ctx->g_pay4b.p : ctx->g_pay4.p;
            if (pairs) ctx->g4_dirty[ctx->g4_cur] = true;  // (before any launch: an error later leaves it marked)
            bd.touched = ctx->g_touched.p;
        }
        VP_CUDA(ctx, ctx->bwd_list.ensure(n));
        BwdPairs bp{};
        const bool aux_ok = pairs;
        if (pairs) {
            if (!ctx->pair_cap_fixed) ctx->pair_cap = std::max(ctx->pair_cap, std::max<size_t>(size_t(1) << 20, 64 * n));
            const size_t cap = std::max<size_t>(ctx->pair_cap, 1);
            VP_CUDA(ctx, ctx->bp_rec.ensure(cap));
            VP_CUDA(ctx, ctx->bp_terms.ensure(cap));
            VP_CUDA(ctx, ctx->bp_span.ensure(n));
            VP_CUDA(ctx, ctx->bp_ent.ensure(n * kRaySegs));
            VP_CUDA(ctx, ctx->bp_fb.ensure(n));
            VP_CUDA(ctx, ctx->bp_tiles.ensure(n / 4096 + 1));
            bp = BwdPairs{ctx->bp_rec.p, ctx->bp_terms.p, ctx->bp_span.p, ctx->bp_ent.p, ctx->bp_fb.p,
                          ctx->bp_tiles.p, unsigned(std::min<size_t>(cap, 0x7fffffffu))};
        }
        VP_CUDA(ctx, launch_backward_rays(mp, ctx->xfb[ctx->xfi].p, k, ctx->payload.p, rays, n_rays,
                                          bd, ctx->d_ctr, ctx->bwd_list.p, int(n), ctx->fb_e.p, ctx->fb_x.p,
                                          ctx->fb_c.p, st, ctx->huge_ray_list.p, kHugeListCap, ctx->hg_e.p,
                                          ctx->hg_x.p, ctx->hg_c.p, pairs ? &bp : nullptr, aux_ok ? ctx->aux_stream : nullptr,
                                          ctx->ev_aux_fork, ctx->ev_aux_join));
        if (v4)
            VP_CUDA(ctx, launch_grad_transpose(reinterpret_cast<float4 *>(bd.g_pay4), dg, ctx->g_touched.p, k,
                                               unsigned(size_t(m) * m * m), accumulate != 0, st, !pairs));
        if (v4 && pairs) ctx->g4_cur ^= 1;  // this call's buffer is cleared during the next call's forward
        if (aux_ok) VP_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_aux_join, 0));  // K6c joins
        VP_CUDA(ctx, cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
    }
    if (!d_grads) VP_CUDA(ctx, cudaMemcpyAsync(grads, dg, n_grad * 4, cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    if (k > 0 && n_rays > 0) {
        // the next call gets room for this call's samples (this one was exact either way)
        if (!ctx->pair_cap_fixed && ctx->h_ctr->bwd_pairs > ctx->pair_cap)
            ctx->pair_cap = size_t(ctx->h_ctr->bwd_pairs) + size_t(ctx->h_ctr->bwd_pairs) / 4;
        return check_counters(ctx, *ctx->h_ctr);
    }
    return VP_OK;
}
}  // namespace

extern "C" {

int vp_backward_rays(vp_ctx *ctx, int64_t n_rays, const float *origins, const float *dirs,
                     const float *jitter01, const float *adj_rgb, const float *adj_alpha,
                     const vp_march *cfg, const float *transforms24, float *grads,
                     int32_t accumulate) {
    NvtxRange nvtx_("vp_backward_rays");
    return backward_rays(ctx, n_rays, origins, dirs, jitter01, adj_rgb, adj_alpha, cfg, transforms24, grads,
                         accumulate, nullptr, nullptr);
}


int vp_eval_loss_pho(vp_ctx *ctx, int32_t n_cams, const vp_camera *cams, int64_t n,
                     const int32_t *cam_index, const float *pixel_xy, const int32_t *pixel_id,
                     const float *target, const float *background, float lambda_pho,
                     const vp_march *cfg, const float *transforms24, float *loss_pho,
                     float *composited, float *grads, int32_t accumulate) {
    NvtxRange nvtx_("vp_eval_loss_pho");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    if (n <= 0) return fail(ctx, VP_ERR_USAGE, "empty pixel set");  // losses.cpp:14
    if (n_cams <= 0 || !cams || !cam_index || !pixel_xy || !pixel_id || !target || !background)
        return fail(ctx, VP_ERR_USAGE, "null ray-batch arrays");
    if (grads && !transforms24) return fail(ctx, VP_ERR_USAGE, "null transforms");
    cudaStream_t st = ctx->stream;
    const size_t nn = size_t(n);
    std::vector<CamDev> cd(static_cast<size_t>(n_cams));
    for (int32_t c = 0; c < n_cams; ++c) cd[size_t(c)] = make_cam(cams[c]);
    // Host-resident pixel sets are range-checked here (the comparisons k_eval_rays makes), so
    // the device flag needs no round trip before the march; device-resident ones are checked
    // by k_eval_rays and read back below.
    const bool host_check = !is_device_ptr(cam_index) && !is_device_ptr(pixel_xy);
    if (host_check) {
        for (size_t i = 0; i < nn; ++i) {
            const int ci = cam_index[i];
            if (ci < 0 || ci >= n_cams) return fail(ctx, VP_ERR_USAGE, "camera index out of range");
            const float px = pixel_xy[2 * i], py = pixel_xy[2 * i + 1];
            if (px < 0.0f || py < 0.0f || px > float(cd[size_t(ci)].width) || py > float(cd[size_t(ci)].height))
                return fail(ctx, VP_ERR_USAGE, "pixel outside image bounds");  // camera.cpp:15-16
        }
    }
    // one device block: cams | cam_index | pixel_id | pixel_xy | target | bg | o | d | jit |
    // rgb | alpha | composited | resid | adj_rgb | adj_alpha | forward state | segment lists | bad flag
    const size_t cam_f = (sizeof(CamDev) * cd.size() + 15) / 16 * 4;
    DBuf<float> &buf = ctx->s_loss;
    const size_t n_seg = grads ? size_t(3 * kRaySegs) : 0;  // segment lists kept for the backward
    const size_t total = cam_f + nn * (1 + 1 + 2 + 3 + 3 + 3 + 3 + 1 + 3 + 1 + 3 + 3 + 3 + 1 + 8 + n_seg) + 4;
    VP_CUDA(ctx, buf.ensure(total));
    float *p = buf.p;
    CamDev *d_cams = reinterpret_cast<CamDev *>(p);
    p += cam_f;
    int *d_ci = reinterpret_cast<int *>(p); p += nn;
    int *d_pid = reinterpret_cast<int *>(p); p += nn;
    float *d_xy = p; p += 2 * nn;
    float *d_tg = p; p += 3 * nn;
    float *d_bg = p; p += 3 * nn;
    float *d_o = p; p += 3 * nn;
    float *d_d = p; p += 3 * nn;
    float *d_j = p; p += nn;
    float *d_rgb = p; p += 3 * nn;
    float *d_a = p; p += nn;
    float *d_comp = p; p += 3 * nn;
    float *d_res = p; p += 3 * nn;
    float *d_ar = p; p += 3 * nn;
    float *d_aa = p; p += nn;
    float *d_state = p; p += 8 * nn;  // forward MarchResult bookkeeping for the backward
    float *d_segs = n_seg ? p : nullptr; p += n_seg * nn;
    int *d_bad = reinterpret_cast<int *>(p);
    const bool host_in = host_check && !is_device_ptr(pixel_id) && !is_device_ptr(target) &&
                         !is_device_ptr(background);
    if (host_in) {
        // host inputs packed into one page-locked block in the device layout, one transfer
        // (six pageable copies each paid the driver's staging)
        const size_t in_f = size_t(d_bg + 3 * nn - buf.p);
        if (ctx->h_loss_floats < in_f) {
            if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
            ctx->h_loss = nullptr;
            ctx->h_loss_floats = 0;
            VP_CUDA(ctx, cudaMallocHost(&ctx->h_loss, in_f * sizeof(float)));
            ctx->h_loss_floats = in_f;
        }
        float *h = ctx->h_loss;
        std::memcpy(h, cd.data(), sizeof(CamDev) * cd.size());
        std::memcpy(h + (d_ci - reinterpret_cast<int *>(buf.p)), cam_index, 4 * nn);
        std::memcpy(h + (d_pid - reinterpret_cast<int *>(buf.p)), pixel_id, 4 * nn);
        std::memcpy(h + (d_xy - buf.p), pixel_xy, 8 * nn);
        std::memcpy(h + (d_tg - buf.p), target, 12 * nn);
        std::memcpy(h + (d_bg - buf.p), background, 12 * nn);
        VP_CUDA(ctx, cudaMemcpyAsync(buf.p, h, in_f * sizeof(float), cudaMemcpyHostToDevice, st));
    } else {
        VP_CUDA(ctx, cudaMemcpyAsync(d_cams, cd.data(), sizeof(CamDev) * cd.size(), cudaMemcpyHostToDevice, st));
        VP_CUDA(ctx, cudaMemcpyAsync(d_ci, cam_index, 4 * nn, cudaMemcpyDefault, st));
        VP_CUDA(ctx, cudaMemcpyAsync(d_pid, pixel_id, 4 * nn, cudaMemcpyDefault, st));
        VP_CUDA(ctx, cudaMemcpyAsync(d_xy, pixel_xy, 8 * nn, cudaMemcpyDefault, st));
        VP_CUDA(ctx, cudaMemcpyAsync(d_tg, target, 12 * nn, cudaMemcpyDefault, st));
        VP_CUDA(ctx, cudaMemcpyAsync(d_bg, background, 12 * nn, cudaMemcpyDefault, st));
    }
    VP_CUDA(ctx, cudaMemsetAsync(d_bad, 0, 4, st));
    VP_CUDA(ctx, launch_eval_rays(d_cams, n_cams, d_ci, d_xy, d_pid, n, cfg->jitter, cfg->seed, d_o, d_d, d_j,
                                  d_bad, st));
    int h_bad = 0;
    if (!host_check) {
        VP_CUDA(ctx, cudaMemcpyAsync(&h_bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
        VP_CUDA(ctx, cudaStreamSynchronize(st));
    }
    if (h_bad == 1) return fail(ctx, VP_ERR_USAGE, "camera index out of range");
    if (h_bad == 2) return fail(ctx, VP_ERR_USAGE, "pixel outside image bounds");  // camera.cpp:15-16
    // forward march of the batch (evalLoss, grad.cpp:216-226)
    const RaysDev rays{d_o, d_d, d_j};
    OutDev od{d_rgb, d_a, nullptr};
    od.state = d_state;
    od.segs = d_segs;
    if (size_t(ctx->ovf_cap) < nn) {
        VP_CUDA(ctx, ctx->ovf_list.ensure(nn));
        ctx->ovf_cap = int(nn);
    }
    if (int rc = ensure_fallback(ctx)) return rc;
    MarchDev mp = make_march(ctx, cfg);
    if (int rc = ensure_bvh(ctx, mp)) return rc;
    VP_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), st));
        ctx->last_n = 1;
    if (ctx->n_prim == 0) {
        VP_CUDA(ctx, cudaMemsetAsync(d_rgb, 0, 12 * nn, st));
        VP_CUDA(ctx, cudaMemsetAsync(d_a, 0, 4 * nn, st));
    } else {
        VP_CUDA(ctx, launch_march_rays(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, rays, n, od, ctx->d_ctr,
                                       ctx->ovf_list.p, ctx->ovf_cap, st));
        const CamDev none{};
        VP_CUDA(ctx, launch_march_fallback(true, none, mp, ctx->xfb[ctx->xfi].p, nullptr, ctx->n_prim, ctx->payload.p,
                                           nullptr, nullptr, od, rays, ctx->d_ctr, ctx->ovf_list.p, ctx->ovf_cap,
                                           ctx->fb_e.p, ctx->fb_x.p, ctx->fb_c.p, st, ctx->huge_ray_list.p,
                                           kHugeListCap));
        VP_CUDA(ctx, launch_march_huge_rays(mp, ctx->xfb[ctx->xfi].p, ctx->n_prim, ctx->payload.p, od, rays, ctx->d_ctr,
                                            ctx->huge_ray_list.p, kHugeListCap, ctx->hg_e.p, ctx->hg_x.p, ctx->hg_c.p,
                                            st));
    }
    // lossPho (losses.cpp:12-25): residuals and adjoints on the device, the scalar sum on the
    // host in the reference's sequential order
    const float invN = 1.0f / float(nn);
    const float scale = 2 * lambda_pho * invN;
    VP_CUDA(ctx, launch_loss_adjoints(d_rgb, d_a, d_tg, d_bg, n, scale, d_comp, d_res, d_ar, d_aa, st));
    std::vector<float> res(3 * nn);
    VP_CUDA(ctx, cudaMemcpyAsync(res.data(), d_res, 12 * nn, cudaMemcpyDeviceToHost, st));
    if (composited) VP_CUDA(ctx, cudaMemcpyAsync(composited, d_comp, 12 * nn, cudaMemcpyDefault, st));
    VP_CUDA(ctx, cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    if (int rc = check_counters(ctx, *ctx->h_ctr)) return rc;
    float acc = 0;
    for (size_t i = 0; i < nn; ++i) {
        const host::F3 e = host::f3(res[3 * i], res[3 * i + 1], res[3 * i + 2]);
        acc += host::dot(e, e);
    }
    if (loss_pho) *loss_pho = lambda_pho * invN * acc;
    if (!grads) return VP_OK;
    // backwardRay for every ray with the photometric adjoints (grad.cpp:240-248)
    return backward_rays(ctx, n, d_o, d_d, d_j, d_ar, d_aa, cfg, transforms24, grads, accumulate, d_state, d_segs);
}

int vp_debug_tile_times(vp_ctx *ctx, const vp_camera *cam, const vp_march *cfg, uint64_t *out,
                        int64_t cap, int64_t *n_out) {
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = check_cam(ctx, cam)) return rc;
    if (int rc = check_march(ctx, cfg)) return rc;
    const CamDev cd = make_cam(*cam);
    const size_t n_tiles = size_t(cd.tiles_x) * cd.tiles_y, n_px = size_t(cam->width) * cam->height;
    if (n_out) *n_out = int64_t(n_tiles);
    if (n_px == 0 || ctx->n_prim == 0) return VP_OK;
    if (int rc = ensure_render_buffers(ctx, cd)) return rc;
    VP_CUDA(ctx, ctx->out_rgb.ensure(3 * n_px));
    VP_CUDA(ctx, ctx->out_alpha.ensure(n_px));
    DBuf<unsigned long long> prof;
    VP_CUDA(ctx, prof.ensure(4 * n_tiles));
    OutDev od{ctx->out_rgb.p, ctx->out_alpha.p, nullptr};
    od.prof = prof.p;
    if (int rc = enqueue_render(ctx, cd, make_march(ctx, cfg), od, ctx->stream)) return rc;
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (out && cap > 0)
        VP_CUDA(ctx, cudaMemcpy(out, prof.p, 8 * std::min<size_t>(size_t(cap), 4 * n_tiles), cudaMemcpyDeviceToHost));
    return VP_OK;
}

int vp_load_slab(vp_ctx *ctx, const char *path, int32_t n_prim, const float *xf15,
                 float window_alpha, int32_t window_beta) {
    NvtxRange nvtx_("vp_load_slab");
    if (int rc = check_ctx(ctx, false)) return rc;
    if (!path) return fail(ctx, VP_ERR_USAGE, "null path");
    std::FILE *f = std::fopen(path, "rb");
    if (!f) return fail(ctx, VP_ERR_IO, std::string("cannot open slab: ") + path);  // scene_io.cpp:44
    struct Closer {
        std::FILE *f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "VPSL", 4) != 0)
        return fail(ctx, VP_ERR_FORMAT, std::string("bad slab magic: ") + path);
    uint32_t header[3];
    if (std::fread(header, 4, 3, f) != 3)
        return fail(ctx, VP_ERR_FORMAT, std::string("truncated slab header: ") + path);
    if (header[0] != 1)
        return fail(ctx, VP_ERR_VERSION, "unsupported slab version " + std::to_string(header[0]));
    if (header[1] == 0 || header[2] == 0 || header[1] > (1u << 20) || header[2] > 512)
        return fail(ctx, VP_ERR_FORMAT, std::string("implausible slab header: ") + path);
    const int k = int(header[1]), m = int(header[2]);
    if (n_prim != k) return fail(ctx, VP_ERR_USAGE, "slab primitive count does not match the transforms");
    // transforms first (validates the scales), payload buffer allocated, filled below
    if (int rc = vp_set_scene(ctx, k, m, xf15, nullptr, window_alpha, window_beta)) return rc;
    ctx->has_scene = false;  // until the payload is complete
    const size_t m3 = size_t(m) * m * m, per_prim = 4 * m3;
    {
        // The file mapped read-only: the payload goes through the same pipeline as a pageable
        // caller slab (upload_planar_host: the copy pool's threads move page-cache pages into
        // the page-locked staging slots while the copy engine and K0 take the previous chunk).
        // A file that cannot be mapped takes the double-buffered fread path below.
        const size_t need = 16 + size_t(k) * per_prim * 4;
        struct stat stt{};
        if (fstat(fileno(f), &stt) == 0 && S_ISREG(stt.st_mode)) {
            if (size_t(stt.st_size) < need)
                return fail(ctx, VP_ERR_FORMAT, std::string("truncated slab payload: ") + path);
            void *map = mmap(nullptr, need, PROT_READ, MAP_PRIVATE, fileno(f), 0);
            if (map != MAP_FAILED) {
                madvise(map, need, MADV_SEQUENTIAL);
                madvise(map, need, MADV_WILLNEED);
                const int rc = upload_planar_host(ctx, reinterpret_cast<const float *>(
                                                           static_cast<const unsigned char *>(map) + 16),
                                                  k, int64_t(m3));
                munmap(map, need);
                if (rc) return rc;
                ctx->pairs_dirty = true;
                ctx->has_scene = true;
                return VP_OK;
            }
        }
    }
    const size_t chunk_prims = std::max<size_t>(1, (size_t(64) << 20) / (per_prim * 4));
    float *pinned[2] = {nullptr, nullptr};
    DBuf<float> dev[2];
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct PinnedFree {
        float **p;
        cudaEvent_t *e;
        ~PinnedFree() {
            for (int i = 0; i < 2; ++i) {
                if (e[i]) cudaEventSynchronize(e[i]), cudaEventDestroy(e[i]);
                if (p[i]) cudaFreeHost(p[i]);
            }
        }
    } pf{pinned, done};
    for (int i = 0; i < 2; ++i) {
        VP_CUDA(ctx, cudaMallocHost(&pinned[i], chunk_prims * per_prim * 4));
        VP_CUDA(ctx, dev[i].ensure(chunk_prims * per_prim));
        VP_CUDA(ctx, cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    // double-buffered: read chunk i+1 from the file while chunk i is copied and repacked
    int slot = 0;
    for (size_t k0 = 0; k0 < size_t(k); k0 += chunk_prims, slot ^= 1) {
        const size_t nk = std::min(chunk_prims, size_t(k) - k0), nf = nk * per_prim;
        VP_CUDA(ctx, cudaEventSynchronize(done[slot]));  // the slot's previous copy finished
        if (std::fread(pinned[slot], 4, nf, f) != nf)
            return fail(ctx, VP_ERR_FORMAT, std::string("truncated slab payload: ") + path);
        VP_CUDA(ctx, cudaMemcpyAsync(dev[slot].p, pinned[slot], nf * 4, cudaMemcpyHostToDevice, ctx->stream));
        VP_CUDA(ctx, launch_repack(dev[slot].p, ctx->payload.p + k0 * m3, int64_t(nk), int64_t(m3), ctx->stream));
        ctx->pairs_dirty = true;
        VP_CUDA(ctx, cudaEventRecord(done[slot], ctx->stream));
    }
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->has_scene = true;
    return VP_OK;
}

int vp_adam_reset(vp_ctx *ctx) {
    if (int rc = check_ctx(ctx, false)) return rc;
    ctx->adam_m1.release();
    ctx->adam_m2.release();
    ctx->adam_step = 0;
    return VP_OK;
}

int vp_adam_step(vp_ctx *ctx, const vp_adam *cfg, const float *grads, float *transforms24) {
    NvtxRange nvtx_("vp_adam_step");
    if (int rc = check_ctx(ctx, true)) return rc;
    if (int rc = quiesce(ctx)) return rc;
    if (!cfg || !grads) return fail(ctx, VP_ERR_USAGE, "null arguments");
    const int k = ctx->n_prim, m = ctx->m;
    if (k > 0 && !transforms24) return fail(ctx, VP_ERR_USAGE, "null transforms");
    const size_t m3 = size_t(m) * m * m, n_pay = size_t(k) * 4 * m3, n = n_pay + 9 * size_t(k);
    if (n == 0) return VP_OK;
    cudaStream_t st = ctx->stream;
    if (ctx->adam_m1.n != n || ctx->adam_step == 0) {  // AdamState(n): zero moments
        VP_CUDA(ctx, ctx->adam_m1.ensure(n));
        VP_CUDA(ctx, ctx->adam_m2.ensure(n));
        VP_CUDA(ctx, cudaMemsetAsync(ctx->adam_m1.p, 0, 4 * n, st));
        VP_CUDA(ctx, cudaMemsetAsync(ctx->adam_m2.p, 0, 4 * n, st));
        ctx->adam_step = 0;
    }
    // scratch: [deltas | flags: non-finite gradient, bad scale | pad to 16 B | host grads]; the
    // gradient slot exists only for host gradients (device ones are read in place)
    DBuf<float> &tmp = ctx->s_adam;
    const bool host_grads = !is_device_ptr(grads);
    const size_t g_off = (9 * size_t(k) + 2 + 3) & ~size_t(3);
    VP_CUDA(ctx, tmp.ensure(g_off + (host_grads ? n : 0)));
    const float *dg = grads;
    if (host_grads) {
        VP_CUDA(ctx, cudaMemcpyAsync(tmp.p + g_off, grads, 4 * n, cudaMemcpyHostToDevice, st));
        dg = tmp.p + g_off;
    }
    float *d_delta = tmp.p;
    int *d_bad = reinterpret_cast<int *>(tmp.p + 9 * size_t(k));  // [0] gradient, [1] scale
    // the caller's records are authoritative: resident copy, then the deltas in Adam's order
    VP_CUDA(ctx, ctx->tr24.ensure(24 * size_t(k)));
    VP_CUDA(ctx, cudaMemcpyAsync(ctx->tr24.p, transforms24, 4 * 24 * size_t(k),
                                 is_device_ptr(transforms24) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    VP_CUDA(ctx, launch_gather_deltas(ctx->tr24.p, k, d_delta, st));
    VP_CUDA(ctx, cudaMemsetAsync(d_bad, 0, 8, st));
    AdamDev c{cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->lr_delta_scale, 0.f, 0.f};
    VP_CUDA(ctx, launch_adam(dg, nullptr, nullptr, nullptr, nullptr, int64_t(n_pay), int64_t(n), unsigned(m3), c,
                             d_bad, true, st));
    // No host round trip between the check and the update: the update and the compose read the
    // check's flag on the device and touch nothing when it is set, so a non-finite gradient
    // still leaves every parameter, moment and the step count as they were (losses.cpp:74-75).
    const int step = ctx->adam_step + 1;
    c.bc1 = 1 - std::pow(cfg->beta1, float(step));  // losses.cpp:79-80
    c.bc2 = 1 - std::pow(cfg->beta2, float(step));
    ctx->pairs_dirty = true;
    VP_CUDA(ctx, launch_adam(dg, ctx->adam_m1.p, ctx->adam_m2.p, ctx->payload.p, d_delta, int64_t(n_pay),
                             int64_t(n), unsigned(m3), c, d_bad, false, st));
    // deltas back into the records with the scale projection (losses.cpp:97-103), then the
    // frame is recomposed on the device (primitive.cpp:41-49)
    VP_CUDA(ctx, ctx->xfb[ctx->xfi].ensure(16 * size_t(k)));
    VP_CUDA(ctx, launch_compose(ctx->tr24.p, d_delta, k, ctx->xfb[ctx->xfi].p, d_bad + 1, st, d_bad));
    if ((const void *)transforms24 != (const void *)ctx->tr24.p)
        VP_CUDA(ctx, cudaMemcpyAsync(transforms24, ctx->tr24.p, 4 * 24 * size_t(k),
                                     is_device_ptr(transforms24) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                     st));
    int bad[2] = {0, 0};
    VP_CUDA(ctx, cudaMemcpyAsync(bad, d_bad, 8, cudaMemcpyDeviceToHost, st));
    VP_CUDA(ctx, cudaStreamSynchronize(st));
    if (bad[0]) return fail(ctx, VP_ERR_NUMERIC, "non-finite gradient");  // losses.cpp:74-75
    ctx->adam_step = step;
    ctx->has_xf = !bad[1];
    ctx->bvh_dirty = true;
    if (bad[1]) return fail(ctx, VP_ERR_USAGE, "non-positive composed primitive scale");
    return VP_OK;
}

int vp_debug_pose(vp_ctx *ctx, int32_t n_prim, const float *tr24, float *out36, int32_t on_device) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (n_prim < 0 || (n_prim > 0 && (!tr24 || !out36))) return fail(ctx, VP_ERR_USAGE, "bad arguments");
    if (n_prim == 0) return VP_OK;
    if (!on_device) {  // the host restatement (vpb_hostmath.hpp) the device kernel replaced
        for (int i = 0; i < n_prim; ++i) {
            const float *tr = tr24 + 24 * size_t(i);
            std::memcpy(out36 + 36 * size_t(i), tr + 3, 9 * sizeof(float));
            for (int q = 0; q < 3; ++q) {
                const host::M3 r = host::rotation_derivative(host::load3(tr + 18), q);
                std::memcpy(out36 + 36 * size_t(i) + 9 + 9 * q, r.m, 9 * sizeof(float));
            }
        }
        return VP_OK;
    }
    DBuf<float> tmp;
    VP_CUDA(ctx, tmp.ensure(60 * size_t(n_prim)));
    VP_CUDA(ctx, cudaMemcpyAsync(tmp.p, tr24, 96 * size_t(n_prim), cudaMemcpyHostToDevice, ctx->stream));
    VP_CUDA(ctx, launch_pose36(tmp.p, n_prim, tmp.p + 24 * size_t(n_prim), ctx->stream));
    VP_CUDA(ctx, cudaMemcpyAsync(out36, tmp.p + 24 * size_t(n_prim), 144 * size_t(n_prim), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int vp_debug_radix_sort(vp_ctx *ctx, int64_t n, const uint64_t *keys_in, uint64_t *keys_out) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (n < 0 || n > (int64_t(1) << 26) || (n > 0 && (!keys_in || !keys_out)))
        return fail(ctx, VP_ERR_USAGE, "bad arguments");
    if (n == 0) return VP_OK;
    DBuf<unsigned long long> k;
    DBuf<unsigned> h;
    VP_CUDA(ctx, k.ensure(2 * size_t(n)));
    VP_CUDA(ctx, h.ensure(256 * size_t((n + 2047) / 2048)));
    VP_CUDA(ctx, cudaMemcpyAsync(k.p, keys_in, 8 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    VP_CUDA(ctx, launch_radix_sort30(k.p, k.p + n, h.p, int(n), ctx->stream));
    VP_CUDA(ctx, cudaMemcpyAsync(keys_out, k.p, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int vp_debug_sincos(vp_ctx *ctx, int64_t n, const float *x, float *y, int32_t which) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (n < 0 || (n > 0 && (!x || !y)) || which < 0 || which > 1) return fail(ctx, VP_ERR_USAGE, "bad arguments");
    if (n == 0) return VP_OK;
    DBuf<float> tmp;
    VP_CUDA(ctx, tmp.ensure(2 * size_t(n)));
    VP_CUDA(ctx, cudaMemcpyAsync(tmp.p, x, 4 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    VP_CUDA(ctx, launch_sincos(tmp.p, tmp.p + n, n, which == 1, ctx->stream));
    VP_CUDA(ctx, cudaMemcpyAsync(y, tmp.p + n, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return VP_OK;
}

int vp_debug_expf(vp_ctx *ctx, int64_t n, const float *x, float *y) {
    if (int rc = check_ctx(ctx, false)) return rc;
    if (n < 0 || (n > 0 && (!x || !y))) return fail(ctx, VP_ERR_USAGE, "bad arguments");
    if (n == 0) return VP_OK;
    DBuf<float> tmp;
    VP_CUDA(ctx, tmp.ensure(2 * size_t(n)));
    VP_CUDA(ctx, cudaMemcpyAsync(tmp.p, x, 4 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    VP_CUDA(ctx, launch_expf(tmp.p, tmp.p + n, n, ctx->stream));
    VP_CUDA(ctx, cudaMemcpyAsync(y, tmp.p + n, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    VP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    tmp.release();
    return VP_OK;
}

}  // extern "C"
