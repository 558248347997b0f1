// vpb_comm.cpp — multi-GPU plumbing of the C-ABI: NCCL over NVLink / NVSwitch
// inside libvpb, so a C++ caller of the drop-in can shard views or tiles over GPUs without
// torch. The path shards by view (or image tile) with no data-path collective: the only
// traffic is one broadcast of the scene (the composed transforms and the already repacked
// interleaved payload, so only the root runs K0) and the gather of rendered outputs to the
// root. The reference parallelises inside one process over rows (threads.h:16-36,
// march.cpp:112); this is its multi-GPU counterpart.
//
// Two ways to build communicators: one process per GPU (vp_comm_init with an id from
// vp_comm_unique_id, shared out of band, e.g. over torch.distributed), or one process driving
// every GPU (vp_comm_init_all, ncclCommInitAll). In the single-process mode the per-GPU calls
// of one collective are issued between vp_group_start / vp_group_end, as NCCL requires.
//
// Every collective runs on the communicator's own stream, after the context's work it depends
// on (stream-ordered, no host wait). NCCL's CTA count is capped (ncclConfig_t.maxCTAs) so a
// gather that overlaps the next raymarch takes few SMs from it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vpb.h"
#include "vpb_ctx_internal.h"

struct vp_comm {
    vp_ctx *ctx = nullptr;
    ncclComm_t nc = nullptr;
    int n_ranks = 0, rank = 0, device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev = nullptr;
};

namespace {

thread_local std::string g_comm_err;

// NCCL is bound at the first vp_comm_* call (dlopen by soname, dlsym), not linked: rendering
// never needs it, and a process that imports torch AFTER loading libvpb must get torch's own
// (newer) libnccl.so.2 — a linked system NCCL would already own that soname and break torch.
// When torch is loaded first, dlopen returns torch's library.
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)?
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto &fn, const char *name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            all = all && fn != nullptr;
        };
        sym(n.GetUniqueId, "ncclGetUniqueId");
        sym(n.CommInitRankConfig, "ncclCommInitRankConfig");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.Broadcast, "ncclBroadcast");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
        sym(n.GetErrorString, "ncclGetErrorString");
        n.ok = all;
        if (!all) n.why = "libnccl.so.2 lacks an entry point libvpb needs";
    });
    return n;
}

int nccl_fail(vp_ctx *ctx, ncclResult_t r, const char *where) {
    const std::string msg = std::string(where) + ": " + nccl().GetErrorString(r);
    if (ctx) return vpb::ctx_fail(ctx, VP_ERR_DEVICE, msg);
    g_comm_err = msg;
    return VP_ERR_DEVICE;
}
int cuda_fail(vp_ctx *ctx, cudaError_t e, const char *where) {
    const std::string msg = std::string(where) + ": " + cudaGetErrorString(e);
    if (ctx) return vpb::ctx_fail(ctx, VP_ERR_DEVICE, msg);
    g_comm_err = msg;
    return VP_ERR_DEVICE;
}
#define VP_NCCL(ctx, call)                                           \
    do {                                                             \
        const ncclResult_t r_ = (call);                              \
        if (r_ != ncclSuccess) return nccl_fail((ctx), r_, #call);   \
    } while (0)
#define VP_NEED_NCCL(ctx)                                            \
    do {                                                             \
        if (!nccl().ok) {                                            \
            if (ctx) return vpb::ctx_fail((ctx), VP_ERR_DEVICE, nccl().why); \
            g_comm_err = nccl().why;                                 \
            return VP_ERR_DEVICE;                                    \
        }                                                            \
    } while (0)
#define VP_CU(ctx, call)                                             \
    do {                                                             \
        const cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call);   \
    } while (0)

ncclConfig_t nccl_config(int32_t max_ctas) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 1;
    if (max_ctas > 0) {
        cfg.maxCTAs = max_ctas;
        cfg.minCTAs = 1;
    }
    return cfg;
}

int finish_comm(vp_comm *c) {
    VP_CU(c->ctx, cudaSetDevice(c->device));
    VP_CU(c->ctx, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    VP_CU(c->ctx, cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming));
    return VP_OK;
}

void free_comm(vp_comm *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    vpb::ctx_drop_writer(c->ctx, c->stream);
    if (c->nc) nccl().CommDestroy(c->nc);
    if (c->ev) cudaEventDestroy(c->ev);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // namespace

extern "C" {

const char *vp_comm_last_error(void) { return g_comm_err.c_str(); }

int vp_comm_unique_id(uint8_t *id) {
    if (!id) return VP_ERR_USAGE;
    VP_NEED_NCCL(nullptr);
    static_assert(sizeof(ncclUniqueId) == VP_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    VP_NCCL(nullptr, nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof u);
    return VP_OK;
}

int vp_comm_init(vp_ctx *ctx, const uint8_t *id, int32_t n_ranks, int32_t rank, int32_t max_ctas, vp_comm **out) {
    if (!ctx || !id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks) {
        g_comm_err = "vp_comm_init: bad arguments";
        return VP_ERR_USAGE;
    }
    VP_NEED_NCCL(ctx);
    *out = nullptr;
    const int device = vpb::ctx_device(ctx);
    auto *c = new vp_comm;
    c->ctx = ctx;
    c->n_ranks = n_ranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclConfig_t cfg = nccl_config(max_ctas);
    cudaSetDevice(device);
    const ncclResult_t r = nccl().CommInitRankConfig(&c->nc, n_ranks, u, rank, &cfg);
    if (r != ncclSuccess) {
        const int rc = nccl_fail(ctx, r, "ncclCommInitRankConfig");
        c->nc = nullptr;
        free_comm(c);
        return rc;
    }
    if (int rc = finish_comm(c)) {
        free_comm(c);
        return rc;
    }
    *out = c;
    return VP_OK;
}

int vp_comm_init_all(int32_t n, vp_ctx *const *ctxs, const int32_t *devices, int32_t max_ctas, vp_comm **out) {
    if (n < 1 || !ctxs || !devices || !out) {
        g_comm_err = "vp_comm_init_all: bad arguments";
        return VP_ERR_USAGE;
    }
    VP_NEED_NCCL(nullptr);
    std::vector<ncclComm_t> ncs(size_t(n), nullptr);
    // ncclCommInitAll has no config argument: build each rank with ncclCommInitRankConfig
    // inside one group (the documented single-process equivalent), so maxCTAs applies
    ncclUniqueId u;
    VP_NCCL(nullptr, nccl().GetUniqueId(&u));
    ncclConfig_t cfg = nccl_config(max_ctas);
    VP_NCCL(nullptr, nccl().GroupStart());
    for (int i = 0; i < n; ++i) {
        VP_CU(nullptr, cudaSetDevice(devices[i]));
        VP_NCCL(nullptr, nccl().CommInitRankConfig(&ncs[size_t(i)], n, u, i, &cfg));
    }
    VP_NCCL(nullptr, nccl().GroupEnd());
    for (int i = 0; i < n; ++i) {
        auto *c = new vp_comm;
        c->ctx = ctxs[i];
        c->nc = ncs[size_t(i)];
        c->n_ranks = n;
        c->rank = i;
        c->device = devices[i];
        if (int rc = finish_comm(c)) {
            free_comm(c);
            for (int j = 0; j < i; ++j) free_comm(out[j]);
            return rc;
        }
        out[i] = c;
    }
    return VP_OK;
}

int vp_comm_destroy(vp_comm *comm) {
    free_comm(comm);
    return VP_OK;
}

int vp_group_start(void) {
    VP_NEED_NCCL(nullptr);
    VP_NCCL(nullptr, nccl().GroupStart());
    return VP_OK;
}
int vp_group_end(void) {
    VP_NEED_NCCL(nullptr);
    VP_NCCL(nullptr, nccl().GroupEnd());
    return VP_OK;
}

// Every rank: vp_set_scene with the same K, M (the root with its data, the others with NULL
// transforms and payload: shape only). Then the root's composed transforms (K x 16 floats) and
// repacked interleaved payload (K M^3 float4) go to every rank in two broadcasts.
int vp_broadcast_scene(vp_comm *comm, int32_t root) {
    nvtxRangePushA("vp_broadcast_scene");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
    if (!comm || root < 0 || root >= comm->n_ranks) {
        g_comm_err = "vp_broadcast_scene: bad arguments";
        return VP_ERR_USAGE;
    }
    vp_ctx *ctx = comm->ctx;
    vpb::CtxScene sc{};
    if (int rc = vpb::ctx_scene(ctx, &sc)) return rc;
    VP_CU(ctx, cudaSetDevice(comm->device));
    // the root's scene upload (on the context stream) must be complete
    VP_CU(ctx, cudaEventRecord(comm->ev, sc.stream));
    VP_CU(ctx, cudaStreamWaitEvent(comm->stream, comm->ev, 0));
    const size_t k = size_t(sc.n_prim);
    if (k > 0) {
        VP_NCCL(ctx, nccl().GroupStart());
        VP_NCCL(ctx, nccl().Broadcast(sc.xf16, sc.xf16, 16 * k, ncclFloat32, root, comm->nc, comm->stream));
        VP_NCCL(ctx, nccl().Broadcast(sc.payload, sc.payload, 4 * k * size_t(sc.m) * sc.m * sc.m, ncclFloat32, root,
                                   comm->nc, comm->stream));
        VP_NCCL(ctx, nccl().GroupEnd());
    }
    if (comm->rank != root) return vpb::ctx_scene_written(ctx, comm->stream);
    return VP_OK;
}

// Gather n_views rendered views (device outputs of n_px pixels: rgb 3, alpha 1, samples 1 per
// pixel; samples may be NULL on every rank) from every rank to the root, after the context's
// renders so far. dst_* (root only; NULL elsewhere) hold n_ranks * n_views device pointers,
// rank r's view j at index r * n_views + j; the root's own views are copied device to device.
// One NCCL group: every send and receive of the call in flight at once.
int vp_gather_views(vp_comm *comm, int32_t root, int32_t n_views, int64_t n_px, float *const *rgb,
                    float *const *alpha, int32_t *const *samples, float *const *dst_rgb, float *const *dst_alpha,
                    int32_t *const *dst_samples) {
    nvtxRangePushA("vp_gather_views");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
    if (!comm || root < 0 || root >= comm->n_ranks || n_views < 0 || n_px < 0 || (n_views > 0 && (!rgb || !alpha))) {
        g_comm_err = "vp_gather_views: bad arguments";
        return VP_ERR_USAGE;
    }
    vp_ctx *ctx = comm->ctx;
    const bool is_root = comm->rank == root;
    if (is_root && n_views > 0 && (!dst_rgb || !dst_alpha || (samples && !dst_samples)))
        return vpb::ctx_fail(ctx, VP_ERR_USAGE, "vp_gather_views: the root needs destination arrays");
    if (n_views == 0 || n_px == 0) return VP_OK;
    VP_CU(ctx, cudaSetDevice(comm->device));
    if (int rc = vpb::ctx_wait_renders(ctx, comm->stream)) return rc;
    const size_t px = size_t(n_px);
    cudaStream_t st = comm->stream;
    VP_NCCL(ctx, nccl().GroupStart());
    for (int j = 0; j < n_views; ++j) {
        if (!is_root) {
            VP_NCCL(ctx, nccl().Send(rgb[j], 3 * px, ncclFloat32, root, comm->nc, st));
            VP_NCCL(ctx, nccl().Send(alpha[j], px, ncclFloat32, root, comm->nc, st));
            if (samples) VP_NCCL(ctx, nccl().Send(samples[j], px, ncclInt32, root, comm->nc, st));
            continue;
        }
        for (int r = 0; r < comm->n_ranks; ++r) {
            const size_t d = size_t(r) * n_views + j;
            if (r == root) continue;
            VP_NCCL(ctx, nccl().Recv(dst_rgb[d], 3 * px, ncclFloat32, r, comm->nc, st));
            VP_NCCL(ctx, nccl().Recv(dst_alpha[d], px, ncclFloat32, r, comm->nc, st));
            if (samples) VP_NCCL(ctx, nccl().Recv(dst_samples[d], px, ncclInt32, r, comm->nc, st));
        }
    }
    VP_NCCL(ctx, nccl().GroupEnd());
    if (is_root)
        for (int j = 0; j < n_views; ++j) {
            const size_t d = size_t(root) * n_views + j;
            if (dst_rgb[d] != rgb[j])
                VP_CU(ctx, cudaMemcpyAsync(dst_rgb[d], rgb[j], 12 * px, cudaMemcpyDeviceToDevice, st));
            if (dst_alpha[d] != alpha[j])
                VP_CU(ctx, cudaMemcpyAsync(dst_alpha[d], alpha[j], 4 * px, cudaMemcpyDeviceToDevice, st));
            if (samples && dst_samples[d] != samples[j])
                VP_CU(ctx, cudaMemcpyAsync(dst_samples[d], samples[j], 4 * px, cudaMemcpyDeviceToDevice, st));
        }
    return VP_OK;
}

// Make `stream` (NULL: the context's) wait for the communicator's work so far, e.g. before a
// render overwrites outputs a gather is still sending.
int vp_comm_wait(vp_comm *comm, void *stream) {
    if (!comm) return VP_ERR_USAGE;
    vp_ctx *ctx = comm->ctx;
    VP_CU(ctx, cudaSetDevice(comm->device));
    VP_CU(ctx, cudaEventRecord(comm->ev, comm->stream));
    vpb::CtxScene sc{};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!st) {
        if (int rc = vpb::ctx_scene(ctx, &sc)) return rc;
        st = sc.stream;
    }
    VP_CU(ctx, cudaStreamWaitEvent(st, comm->ev, 0));
    return VP_OK;
}

// Blocks until the communicator's work so far has completed.
int vp_comm_sync(vp_comm *comm) {
    if (!comm) return VP_ERR_USAGE;
    VP_CU(comm->ctx, cudaSetDevice(comm->device));
    VP_CU(comm->ctx, cudaStreamSynchronize(comm->stream));
    return VP_OK;
}

}  // extern "C"
