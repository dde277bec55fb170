// zc_probe.cu -- how fast can the batch's graphs cross PCIe?
//   (1) cudaMemcpyAsync of the whole batch (what batch_host_run does today)
//   (2) zero-copy kernel reading all of it from mapped pinned memory
//   (3) zero-copy kernel reading only the 32-byte sectors at or right of the
//       diagonal (rows v < 256: both sectors, rows v >= 256: the second) at N=512
//   (4) DMA 3D copy of the same sectors (narrow rows)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_probe tools/zc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 512, RB = 64, GB = N * RB;  // 32 KiB per graph

// one CTA per graph, 256 threads: full copy, uint4 per thread x 8
__global__ void zc_all(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int graphs) {
    for (int g = blockIdx.x; g < graphs; g += gridDim.x) {
        const uint4 *s = src + (size_t)g * (GB / 16);
        uint4 *d = dst + (size_t)g * (GB / 16);
        uint4 r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = s[threadIdx.x + 256 * k];
#pragma unroll
        for (int k = 0; k < 8; ++k) d[threadIdx.x + 256 * k] = r[k];
    }
}

// upper-triangle sectors only: rows 0..255 whole (16 KiB contiguous), rows
// 256..511 bytes 32..63 (32 B of every 64)
__global__ void zc_upper(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int graphs) {
    for (int g = blockIdx.x; g < graphs; g += gridDim.x) {
        const uint4 *s = src + (size_t)g * (GB / 16);
        uint4 *d = dst + (size_t)g * (GB / 16);
        uint4 r[6];
        // 1024 uint4 of rows 0..255 + 512 uint4 (2 per row) of rows 256..511 = 1536 = 6 x 256
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = s[threadIdx.x + 256 * k];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            int q = threadIdx.x + 256 * k;  // 0..511
            int row = 256 + (q >> 1), half = q & 1;
            r[4 + k] = s[row * 4 + 2 + half];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) d[threadIdx.x + 256 * k] = r[k];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            int q = threadIdx.x + 256 * k;
            int row = 256 + (q >> 1), half = q & 1;
            d[row * 4 + 2 + half] = r[4 + k];
        }
    }
}

int main(int argc, char **argv) {
    const int graphs = argc > 1 ? atoi(argv[1]) : 65536;
    const size_t bytes = (size_t)graphs * GB;
    uint8_t *h, *d;
    CK(cudaHostAlloc((void **)&h, bytes, cudaHostAllocMapped));
    memset(h, 0x5A, bytes);
    CK(cudaMalloc((void **)&d, bytes));
    uint8_t *hd;
    CK(cudaHostGetDevicePointer((void **)&hd, h, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("memcpy all        : %8.2f ms  %6.1f GB/s\n", ms, bytes / ms / 1e6);
    }
    int grids[] = {148, 296, 592, 1184, 2368};
    for (int gi = 0; gi < 5; ++gi) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            zc_all<<<grids[gi], 256>>>((const uint4 *)hd, (uint4 *)d, graphs);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            CK(cudaGetLastError());
            cudaEventElapsedTime(&ms, a, b);
            printf("zc all   grid %5d: %8.2f ms  %6.1f GB/s of bytes\n", grids[gi], ms, bytes / ms / 1e6);
        }
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            zc_upper<<<grids[gi], 256>>>((const uint4 *)hd, (uint4 *)d, graphs);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            CK(cudaGetLastError());
            cudaEventElapsedTime(&ms, a, b);
            printf("zc upper grid %5d: %8.2f ms  %6.1f GB/s of sectors read (%.1f GB/s equiv full)\n", grids[gi], ms,
                   0.75 * bytes / ms / 1e6, bytes / ms / 1e6);
        }
    }
    // DMA: rows 0..255 of every graph (16 KiB each, pitch 32 KiB) + 32 B of rows 256..511
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaMemcpy2DAsync(d, GB, h, GB, GB / 2, graphs, cudaMemcpyHostToDevice);
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(h + GB / 2 + 32, RB, 32, 256);
        p.dstPtr = make_cudaPitchedPtr(d + GB / 2 + 32, RB, 32, 256);
        // depth stride = pitch * ysize = 64 * 512 -> use height 512 rows per slice, copy 256
        p.srcPtr = make_cudaPitchedPtr(h + GB / 2 + 32, RB, 32, 512);
        p.dstPtr = make_cudaPitchedPtr(d + GB / 2 + 32, RB, 32, 512);
        p.extent = make_cudaExtent(32, 256, graphs);
        p.kind = cudaMemcpyHostToDevice;
        cudaError_t e = cudaMemcpy3DAsync(&p);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("dma 2D+3D upper   : %8.2f ms  %6.1f GB/s of sectors (%s)\n", ms, 0.75 * bytes / ms / 1e6,
               cudaGetErrorString(e));
    }
    return 0;
}
