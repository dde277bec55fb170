// pack_probe.cu -- can the config-4 batch cross PCIe as upper-triangle word
// tails packed by host threads, faster than the full-row DMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pack_probe tools/pack_probe.cu -lpthread
// Measures: (1) host copy bandwidth, (2) the packing rate with T threads,
// (3) packing pipelined with the H2D DMA of the packed chunks (no kernels),
// against (4) the full-row DMA.  Not part of the library.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
#include <functional>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// n = 512, 64-byte rows: row i keeps 64-bit words [i / 64, 8)
static inline size_t pack_one(const uint64_t *src, uint64_t *dst) {
    uint64_t *d = dst;
    for (int g = 0; g < 8; ++g) {
        const int L = 8 - g;
        for (int r = 0; r < 64; ++r) {
            const uint64_t *s = src + (size_t)(64 * g + r) * 8 + g;
            for (int w = 0; w < L; ++w) d[w] = s[w];
            d += L;
        }
    }
    return (size_t)(d - dst);
}

static void pack_range(const uint8_t *in, uint8_t *out, int64_t g0, int64_t g1, size_t pk) {
    for (int64_t g = g0; g < g1; ++g)
        pack_one(reinterpret_cast<const uint64_t *>(in + (size_t)(g - g0) * 32768), reinterpret_cast<uint64_t *>(out + (size_t)(g - g0) * pk));
}

static void par(int T, int64_t cnt, const std::function<void(int64_t, int64_t)> &f) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
        int64_t a = cnt * t / T, b = cnt * (t + 1) / T;
        th.emplace_back([=, &f] { f(a, b); });
    }
    for (auto &x : th) x.join();
}

int main() {
    const int64_t G = 65536, GB = 32768;
    const size_t pk = 18432;  // packed bytes per graph
    uint8_t *in, *st;
    if (cudaHostAlloc((void **)&in, G * GB, 0) != cudaSuccess || cudaHostAlloc((void **)&st, G * pk, 0) != cudaSuccess) {
        printf("cudaHostAlloc failed: plain malloc (host-only run)\n");
        in = (uint8_t *)malloc(G * GB);
        st = (uint8_t *)malloc(G * pk);
    }
    for (size_t i = 0; i < (size_t)G * GB; i += 4096) in[i] = (uint8_t)i;
    memset(st, 0, G * pk);
    uint8_t *dev;
    if (cudaMalloc(&dev, G * GB) != cudaSuccess) { printf("no device: host part only\n"); dev = nullptr; }
    setvbuf(stdout, nullptr, _IONBF, 0);
    setvbuf(stdout, nullptr, _IONBF, 0);
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    for (int T : {1, 8, 16, 32}) {
        double t0 = now();
        par(T, G, [&](int64_t a, int64_t b) { memcpy(st + a * pk, in + a * pk, (b - a) * pk); });
        double t1 = now();
        par(T, G, [&](int64_t a, int64_t b) { pack_range(in + a * GB, st + a * pk, a, b, pk); });
        double t2 = now();
        printf("T=%2d memcpy %.1f GB/s | pack %.2f ms = %.1f GB/s of input\n", T, G * pk / (t1 - t0) / 1e9,
               (t2 - t1) * 1e3, G * GB / (t2 - t1) / 1e9);
    }
    if (!dev) return 0;
    // pipelined: chunks packed by T threads into a ring of staging slots, each DMA'd as soon as packed
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s);
        cudaMemcpyAsync(dev, in, G * GB, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("full DMA %.2f ms (%.1f GB/s)\n", ms, G * GB / ms / 1e6);
        cudaEventRecord(a, s);
        cudaMemcpyAsync(dev, st, G * pk, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("packed DMA alone %.2f ms (%.1f GB/s)\n", ms, G * pk / ms / 1e6);
    }
    for (int T : {8, 16}) {
        for (int64_t chunk : {1024, 4096}) {
            const int64_t nc = G / chunk;
            std::vector<std::atomic<int>> done(nc);
            for (auto &d : done) d = 0;
            double t0 = now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    for (int64_t c = 0; c < nc; ++c) {
                        const int64_t x = c * chunk + chunk * t / T, y = c * chunk + chunk * (t + 1) / T;
                        pack_range(in + x * GB, st + x * pk, x, y, pk);
                        done[c].fetch_add(1);
                    }
                });
            for (int64_t c = 0; c < nc; ++c) {
                while (done[c].load() < T) {
                }
                cudaMemcpyAsync(dev + c * chunk * pk, st + c * chunk * pk, chunk * pk, cudaMemcpyHostToDevice, s);
            }
            for (auto &x : th) x.join();
            cudaStreamSynchronize(s);
            double t1 = now();
            printf("pipelined T=%d chunk=%lld: %.2f ms per batch (%.2f M graphs/s)\n", T, (long long)chunk,
                   (t1 - t0) * 1e3, G / (t1 - t0) / 1e6);
        }
    }
    return 0;
}
