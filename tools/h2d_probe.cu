// Host-side upload limits on the box: pinned H2D bandwidth (one stream, 8 MB chunks) and the
// pageable -> page-locked memcpy rate with T host threads (the drop-in's staging step).
// nvcc -O2 -o build/h2d_probe tools/h2d_probe.cu -lpthread
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t bytes = size_t(256) << 20, chunk = size_t(8) << 20;
    char *pin = nullptr, *dev = nullptr;
    cudaMallocHost(&pin, bytes);
    cudaMalloc(&dev, bytes);
    std::vector<char> pageable(bytes, 1);
    memset(pin, 2, bytes);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int rep = 0; rep < 3; ++rep) {
        const double t0 = now();
        for (size_t o = 0; o < bytes; o += chunk) cudaMemcpyAsync(dev + o, pin + o, chunk, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        printf("pinned H2D: %.1f GB/s\n", bytes / (now() - t0) / 1e9);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    printf("hardware_concurrency %u\n", hw);
    for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
        if (T > (int)hw) break;
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            const double t0 = now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    const size_t per = bytes / T, o = per * t;
                    memcpy(pin + o, pageable.data() + o, t == T - 1 ? bytes - o : per);
                });
            for (auto &x : th) x.join();
            best = std::min(best, now() - t0);
        }
        printf("memcpy pageable->pinned, %2d threads: %.1f GB/s\n", T, bytes / best / 1e9);
    }
    return 0;
}
