// seg_time.cu -- times launch_lexbfs_seg (the CTA engine, no profiling counters)
// on a dumped graph with its edge count known, as the library pipeline calls it;
// SEG_THREADS=T overrides the thread count.  Not part of the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/seg_time tools/seg_time.cu
//   SEG_THREADS=256 tools/seg_time graph.bin      (file from tools/dump_graph.py)
#include <cstdio>
#include <cstdlib>
#define SEG_THREADS_ENV
#include <vector>

#include "../paper_1508_06329_b200/csrc/lexbfs_seg.cu"

int main(int argc, char **argv) {
    if (argc < 2) return 1;
    FILE *f = fopen(argv[1], "rb");
    long long hdr[2];
    if (!f || fread(hdr, 8, 2, f) != 2) return 1;
    const long long n = hdr[0], stride = hdr[1];
    std::vector<uint8_t> h((size_t)(n * stride));
    if (fread(h.data(), 1, h.size(), f) != h.size()) return 1;
    fclose(f);
    long long deg2 = 0;
    for (uint8_t b : h) deg2 += __builtin_popcount(b);
    uint8_t *adj;
    int32_t *ord;
    cudaMalloc(&adj, h.size());
    cudaMalloc(&ord, sizeof(int32_t) * 2 * n);
    cudaMemcpy(adj, h.data(), h.size(), cudaMemcpyHostToDevice);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        int rc = chordal::launch_lexbfs_seg(adj, n, stride, deg2 / 2, CHORDAL_TIE_ASCENDING, 0, 0, ord, ord + n, nullptr, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rc) printf("rc=%d\n", rc);
        if (rep && ms < best) best = ms;
    }
    printf("n=%lld m=%lld T=%s best of 3: %.3f ms (%.1f ns/step)\n", n, deg2 / 2, getenv("SEG_THREADS") ? getenv("SEG_THREADS") : "auto",
           best, best * 1e6 / n);
    return 0;
}
