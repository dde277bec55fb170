#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(1024, 1) toy(int iters, const unsigned *rows, int n, unsigned long long *out) {
    __shared__ unsigned long long best[2][32];
    __shared__ unsigned long long cbest[2];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    unsigned long long key = (unsigned long long)(t * 7919 + rank * 104729) * 2654435761ULL;
    int x = 0;
    for (int i = 0; i < iters; ++i) {
        const int par = i & 1;
        // row word of pivot x for this thread
        unsigned w = NOLOAD ? (unsigned)x : rows[(long long)x * (n / 32) + ((rank * 1024 + t) & (n / 32 - 1))];
        key = (key << 1) ^ (w & 1) ^ i;
        unsigned long long k = key;
        for (int d = 16; d; d >>= 1) { unsigned long long o = __shfl_xor_sync(~0u, k, d); k = o > k ? o : k; }
        if (lane == 0) best[par][warp] = k;
        __syncthreads();
        if (warp == 0) {
            k = best[par][lane];
            for (int d = 16; d; d >>= 1) { unsigned long long o = __shfl_xor_sync(~0u, k, d); k = o > k ? o : k; }
            if (lane == 0) cbest[par] = k;
        }
        cl.sync();
        unsigned long long g = 0;
        if (warp == 0) {
            if (lane < CS) g = *cl.map_shared_rank(&cbest[par], lane);
            for (int d = 16; d; d >>= 1) { unsigned long long o = __shfl_xor_sync(~0u, g, d); g = o > g ? o : g; }
            if (lane == 0) best[par][31] = g;
        }
        __syncthreads();
        g = best[par][31];
        x = (int)(g % n);
    }
    if (t == 0 && rank == 0) out[0] = key;
}

int main() {
    int n = 32768;
    unsigned *rows; unsigned long long *out;
    cudaMalloc(&rows, (size_t)n * n / 8); cudaMemset(rows, 0x5a, (size_t)n * n / 8);
    cudaMalloc(&out, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        int iters = 20000;
        cudaEventRecord(a);
        toy<8><<<8, 1024>>>(iters, rows, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cluster 8: %.1f ns/iter err=%s\n", ms * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
        cudaFuncSetAttribute(toy<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaEventRecord(a);
        toy<16><<<16, 1024>>>(iters, rows, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster 16: %.1f ns/iter err=%s\n", ms * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
