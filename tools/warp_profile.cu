// warp_profile.cu -- counters of the one-warp LexBFS engine (warp_seg.cuh built
// with -DWSEG_PROFILE).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DWSEG_PROFILE \
//        -o tools/warp_profile tools/warp_profile.cu
//   tools/warp_profile graph.bin      (int64 n, int64 stride, then n*stride bytes; n <= 1024)
#include <cstdio>
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
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(chordal::wseg_prof, z, sizeof(z));
        cudaMemcpyToSymbol(chordal::wseg_ph, z, sizeof(z));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        int rc = chordal::launch_lexbfs_seg(adj, n, stride, -1, CHORDAL_TIE_ASCENDING, 0, 0, ord, ord + n, ord + 2 * n, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long p[8];
        cudaMemcpyFromSymbol(p, chordal::wseg_prof, sizeof(p));
        printf("rc=%d n=%lld %.3f ms (%.1f ns/step)\n", rc, n, ms, ms * 1e6 / n);
        const char *const names[] = {"steps", "guess-hit", "row-wait-cyc", "total-cyc", "split-steps"};
        for (int k = 0; k < 5; ++k)
            printf("  %-13s %12llu  %8.1f per step\n", names[k], p[k], (double)p[k] / (double)(p[0] ? p[0] : 1));
        unsigned long long q[8];
        cudaMemcpyFromSymbol(q, chordal::wseg_ph, sizeof(q));
        const char *const ph[] = {"pivot+row", "movers", "reached+scan", "split-decide", "split", "append+tail"};
        for (int k = 0; k < 6; ++k)
            printf("  %-13s %12llu  %8.1f per step\n", ph[k], q[k], (double)q[k] / (double)(p[0] ? p[0] : 1));
    }
    return 0;
}
