// host_call_probe.cu -- where does the host-buffer single-graph call spend its
// time at n = 1000 (configuration 1)?  Pageable host rows (125 B, the
// reference's packing) into 128-byte device rows.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/host_call_probe \
//        tools/host_call_probe.cu -Lpaper_1508_06329_b200/lib -lchordal_b200 -Xlinker -rpath=$PWD/paper_1508_06329_b200/lib
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "chordal_b200.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

template <typename F>
static double wall_us(F f, int reps = 50) {
    f();
    cudaDeviceSynchronize();
    double t0 = now();
    for (int i = 0; i < reps; ++i) f();
    return (now() - t0) / reps * 1e6;
}

int main() {
    const int n = 1000, rb = 125, stride = 128;
    std::vector<uint8_t> host((size_t)n * rb);
    // a path graph: chordal, cheap search
    for (int v = 0; v + 1 < n; ++v) {
        host[(size_t)v * rb + (v + 1) / 8] |= 1u << ((v + 1) & 7);
        host[(size_t)(v + 1) * rb + v / 8] |= 1u << (v & 7);
    }
    uint8_t *dev, *flat;
    cudaMalloc(&dev, (size_t)n * stride);
    cudaMalloc(&flat, (size_t)n * stride);
    cudaStream_t s = cudaStreamPerThread;
    std::vector<int32_t> ord(n);
    int32_t wit[3], ch;
    printf("flat pageable H2D %d B + sync: %.1f us\n", n * rb, wall_us([&] {
               cudaMemcpyAsync(flat, host.data(), (size_t)n * rb, cudaMemcpyHostToDevice, s);
               cudaStreamSynchronize(s);
           }));
    printf("2D pageable H2D + sync:          %.1f us\n", wall_us([&] {
               cudaMemcpy2DAsync(dev, stride, host.data(), rb, rb, n, cudaMemcpyHostToDevice, s);
               cudaStreamSynchronize(s);
           }));
    printf("D2H order (pageable) + sync:     %.1f us\n", wall_us([&] {
               cudaMemcpyAsync(ord.data(), flat, 4 * n, cudaMemcpyDeviceToHost, s);
               cudaStreamSynchronize(s);
           }));
    const size_t wsb = chordal_dense_host_workspace_bytes(n, n - 1);
    void *ws;
    cudaMalloc(&ws, wsb + 256);
    printf("whole host_ws call:              %.1f us\n", wall_us([&] {
               chordal_is_chordal_dense_host_ws(host.data(), n, rb, n - 1, 0, 0, ord.data(), wit, &ch, ws, wsb);
           }));
    const size_t dwsb = chordal_dense_workspace_bytes(n, n - 1);
    void *dws;
    int32_t *dord, *dwit;
    cudaMalloc(&dws, dwsb);
    cudaMalloc(&dord, 8 * n + 16);
    cudaMalloc(&dwit, 16);
    cudaMemcpy2D(dev, stride, host.data(), rb, rb, n, cudaMemcpyHostToDevice);
    printf("device is_chordal + sync:        %.1f us\n", wall_us([&] {
               chordal_is_chordal_dense(dev, n, stride, n - 1, 0, 0, dord, dord + n, dws, dwsb, dwit, s);
               cudaStreamSynchronize(s);
           }));
    printf("rc check: %s chordal=%d\n", cudaGetErrorString(cudaGetLastError()), ch);
    return 0;
}
