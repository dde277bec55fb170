// seg_profile.cu -- per-phase cycle breakdown of the touched-segment LexBFS
// kernel (lexbfs_seg.cu compiled with -DSEG_PROFILE).  Not part of the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSEG_PROFILE \
//        -o tools/seg_profile tools/seg_profile.cu
//   tools/seg_profile graph.bin      (int64 n, int64 stride, then n*stride bytes)
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
    uint8_t *adj;
    int32_t *ord;
    cudaMalloc(&adj, h.size());
    cudaMalloc(&ord, sizeof(int32_t) * 3 * n);
    cudaMemcpy(adj, h.data(), h.size(), cudaMemcpyHostToDevice);
    const uint64_t cell = 0;
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(chordal::seg_prof, z, sizeof(z));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        int rc = chordal::launch_lexbfs_seg(adj, n, stride, -1, CHORDAL_TIE_ASCENDING, 0, cell, ord, ord + n,
                                            getenv("NOPARENT") ? nullptr : ord + 2 * n,
                                            0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long p[16];
        cudaMemcpyFromSymbol(p, chordal::seg_prof, sizeof(p));
        const char *const names[] = {"steps", "full", "phase1", "short-tail", "scan", "3a", "3b", "3c+end", "guess-hit", "ntouch", "movers(full)", "splits", "3b-own", "3b-wait", "max-thr-mov", "3b-rounds(w0)"};
        printf("rc=%d n=%lld %.3f ms (%.1f ns/step)\n", rc, n, ms, ms * 1e6 / n);
        for (int k = 0; k < 16; ++k)
            printf("  %-10s %14llu  %8.1f per step\n", names[k], p[k], (double)p[k] / (double)(p[0] ? p[0] : 1));
    }
    return 0;
}
