// slot_profile.cu -- per-phase cycle counters of the CSR slot engine (csr.cu
// built with -DSLOT_PROFILE).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSLOT_PROFILE -I include \
//        -o tools/slot_profile tools/slot_profile.cu
//   tools/slot_profile indptr.bin indices.bin     (int64 indptr[n+1], int32 indices)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1508_06329_b200/csrc/csr.cu"

int main(int argc, char **argv) {
    if (argc < 3) return 1;
    FILE *f = fopen(argv[1], "rb");
    std::vector<int64_t> ip;
    int64_t x;
    while (f && fread(&x, 8, 1, f) == 1) ip.push_back(x);
    if (f) fclose(f);
    const long long n = (long long)ip.size() - 1, nnz = ip.back();
    std::vector<int32_t> ix((size_t)nnz);
    f = fopen(argv[2], "rb");
    if (!f || fread(ix.data(), 4, ix.size(), f) != ix.size()) return 1;
    fclose(f);
    int64_t *dip;
    int32_t *dix, *out;
    cudaMalloc(&dip, 8 * (n + 1));
    cudaMalloc(&dix, 4 * (nnz + 1));
    cudaMalloc(&out, 4 * 3 * n);
    cudaMemcpy(dip, ip.data(), 8 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dix, ix.data(), 4 * nnz, cudaMemcpyHostToDevice);
    const size_t wsb = chordal::csr_workspace_bytes(n, nnz / 2);
    void *ws;
    cudaMalloc(&ws, wsb);
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(chordal::slot_prof, z, sizeof(z));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        int rc = chordal::launch_lexbfs_csr(dip, dix, n, nnz / 2, CHORDAL_TIE_ASCENDING, 0, 0, out, out + n,
                                            getenv("NOPARENT") ? nullptr : out + 2 * n, ws, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long p[16];
        cudaMemcpyFromSymbol(p, chordal::slot_prof, sizeof(p));
        printf("rc=%d n=%lld %.3f ms (%.1f ns/step) err=%s\n", rc, n, ms, ms * 1e6 / n,
               cudaGetErrorString(cudaGetLastError()));
        const char *const names[] = {"steps", "pivot", "bounds+pass1", "allocate", "pass2+restore", "touched", "pivot-known", "bounds-ahead", "fast", "bounds-wait", "list-avail", "cls-avail", "match", "fields", "scan", "alloc-done"};
        for (int k = 0; k < 16; ++k)
            printf("  %-14s %14llu  %8.1f per step\n", names[k], p[k], (double)p[k] / (double)(p[0] ? p[0] : 1));
    }
    return 0;
}
