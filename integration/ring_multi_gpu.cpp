// ring_multi_gpu.cpp — a C++ caller of libvpb rendering BASELINE config 5 (the 64-view ring around
// the 4096 x 16^3 shell at 1024^2) over every visible GPU from ONE process, with no torch: one
// context per GPU, vp_comm_init_all, the scene uploaded once on GPU 0 and broadcast
// (vp_broadcast_scene), 64 / N views per GPU rendered 8 per raymarch launch, and every view
// gathered to GPU 0 in one NCCL group per round (vp_gather_views). Prints the ray-samples and the
// wall time. Build: make ring_multi_gpu; run: ./build/ring_multi_gpu [n_gpus]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vpb.h"

#define CHECK(call)                                                                     \
    do {                                                                                \
        const int rc_ = (call);                                                         \
        if (rc_ != VP_OK) {                                                             \
            std::fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, vp_comm_last_error()); \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(int argc, char **argv) {
    int visible = 0;
    cudaGetDeviceCount(&visible);
    const int n = argc > 1 ? std::atoi(argv[1]) : visible;
    if (n < 1 || n > visible || 64 % n != 0) {
        std::fprintf(stderr, "need 1..%d GPUs dividing 64\n", visible);
        return 2;
    }
    const int K = 4096, M = 16, W = 1024, views_per_gpu = 64 / n, batch = 8;
    const size_t px = size_t(W) * W;
    std::vector<float> tr(size_t(K) * 24), pay(size_t(K) * 4 * M * M * M), xf(size_t(K) * 15);
    CHECK(vp_make_shell_scene(K, M, tr.data(), pay.data()));
    CHECK(vp_compose(K, tr.data(), xf.data()));

    std::vector<vp_ctx *> ctx(static_cast<size_t>(n));
    std::vector<int32_t> dev(static_cast<size_t>(n));
    for (int g = 0; g < n; ++g) {
        dev[size_t(g)] = g;
        CHECK(vp_create(g, &ctx[size_t(g)]));
    }
    std::vector<vp_comm *> comm(static_cast<size_t>(n));
    CHECK(vp_comm_init_all(n, ctx.data(), dev.data(), 8, comm.data()));
    CHECK(vp_set_scene(ctx[0], K, M, xf.data(), pay.data(), 8.0f, 8));
    for (int g = 1; g < n; ++g) CHECK(vp_set_scene(ctx[size_t(g)], K, M, nullptr, nullptr, 8.0f, 8));
    CHECK(vp_group_start());
    for (int g = 0; g < n; ++g) CHECK(vp_broadcast_scene(comm[size_t(g)], 0));
    CHECK(vp_group_end());
    for (int g = 0; g < n; ++g) CHECK(vp_comm_sync(comm[size_t(g)]));

    // device outputs: per GPU one batch of 8 views; on GPU 0 the gathered n x 8 views
    std::vector<std::vector<float *>> rgb(static_cast<size_t>(n)), alpha(static_cast<size_t>(n));
    std::vector<std::vector<int32_t *>> samples(static_cast<size_t>(n));
    std::vector<float *> dst_rgb(static_cast<size_t>(n) * batch), dst_alpha(static_cast<size_t>(n) * batch);
    std::vector<int32_t *> dst_samples(static_cast<size_t>(n) * batch);
    for (int g = 0; g < n; ++g) {
        cudaSetDevice(g);
        for (int j = 0; j < batch; ++j) {
            float *p;
            int32_t *s;
            cudaMalloc(&p, px * 3 * sizeof(float));
            rgb[size_t(g)].push_back(p);
            cudaMalloc(&p, px * sizeof(float));
            alpha[size_t(g)].push_back(p);
            cudaMalloc(&s, px * sizeof(int32_t));
            samples[size_t(g)].push_back(s);
        }
    }
    cudaSetDevice(0);
    for (size_t i = 0; i < dst_rgb.size(); ++i) {
        cudaMalloc(&dst_rgb[i], px * 3 * sizeof(float));
        cudaMalloc(&dst_alpha[i], px * sizeof(float));
        cudaMalloc(&dst_samples[i], px * sizeof(int32_t));
    }
    vp_march cfg{};
    cfg.step_size = 0.001f;
    cfg.early_eps = 0.01f;

    long long total = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int round = 0; round < views_per_gpu / batch; ++round) {
        for (int g = 0; g < n; ++g) {  // GPU g renders views g * views_per_gpu + round * 8 + j
            std::vector<vp_camera> cams(batch);
            for (int j = 0; j < batch; ++j)
                CHECK(vp_shell_camera(g * views_per_gpu + round * batch + j, 64, W, &cams[size_t(j)]));
            CHECK(vp_comm_wait(comm[size_t(g)], nullptr));  // the previous round's gather has sent
            CHECK(vp_render_batch_async(ctx[size_t(g)], batch, cams.data(), &cfg, rgb[size_t(g)].data(),
                                        alpha[size_t(g)].data(), samples[size_t(g)].data(), nullptr));
        }
        CHECK(vp_group_start());
        for (int g = 0; g < n; ++g)
            CHECK(vp_gather_views(comm[size_t(g)], 0, batch, int64_t(px), rgb[size_t(g)].data(),
                                  alpha[size_t(g)].data(), samples[size_t(g)].data(),
                                  g == 0 ? dst_rgb.data() : nullptr, g == 0 ? dst_alpha.data() : nullptr,
                                  g == 0 ? dst_samples.data() : nullptr));
        CHECK(vp_group_end());
    }
    for (int g = 0; g < n; ++g) CHECK(vp_comm_sync(comm[size_t(g)]));
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // ray-samples of every gathered view of the last round, summed on the host from GPU 0's copies
    std::vector<int32_t> h(px);
    for (size_t i = 0; i < dst_samples.size(); ++i) {
        cudaMemcpy(h.data(), dst_samples[i], px * sizeof(int32_t), cudaMemcpyDeviceToHost);
        for (int32_t v : h) total += v;
    }
    std::printf("ring_multi_gpu: %d GPU(s), 64 views of 4096x16^3 at 1024^2 in %.1f ms wall (incl. gathers to GPU 0); "
                "last round's %d gathered views hold %lld ray-samples\n",
                n, s * 1e3, n * batch, total);
    for (int g = 0; g < n; ++g) vp_comm_destroy(comm[size_t(g)]);
    for (int g = 0; g < n; ++g) vp_destroy(ctx[size_t(g)]);
    return 0;
}
