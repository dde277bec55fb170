// e2e_api_probe.cu -- which per-call resource handling makes the host-buffer batch
// call stall?  Same copy pattern as chordal_is_chordal_batch_host (8 chunks of
// 256 MiB H2D + a dummy kernel + 16 MiB D2H over 3 streams), with
//   A: streams created / destroyed per call, pool block allocated per call
//   B: streams per call, device buffer allocated once
//   C: persistent streams, pool block per call
//   D: persistent streams and buffer
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void touch(unsigned char *p, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] ^= 1;
}

int main() {
    const size_t B = 65536, G = 32768, CH = 8192, NB = 3, per = CH * G + CH * 4 * 515 + 1024;
    unsigned char *host, *outh, *dbuf;
    cudaMallocHost(&host, B * G);
    cudaMallocHost(&outh, B * 4 * 515);
    cudaMalloc(&dbuf, NB * per);
    cudaStream_t ps[NB];
    for (int k = 0; k < NB; ++k) cudaStreamCreateWithFlags(&ps[k], cudaStreamNonBlocking);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = NB * per;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    for (int variant = 0; variant < 4; ++variant) {
        double t[12];
        for (int call = -3; call < 12; ++call) {
            auto t0 = std::chrono::steady_clock::now();
            const bool per_streams = variant == 0 || variant == 1, per_alloc = variant == 0 || variant == 2;
            cudaStream_t st[NB];
            for (int k = 0; k < NB; ++k) {
                if (per_streams) cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking); else st[k] = ps[k];
            }
            unsigned char *blk = dbuf;
            if (per_alloc) cudaMallocAsync((void **)&blk, NB * per, cudaStreamPerThread);
            cudaEvent_t ev;
            cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            cudaEventRecord(ev, cudaStreamPerThread);
            for (int k = 0; k < NB; ++k) cudaStreamWaitEvent(st[k], ev, 0);
            for (size_t b0 = 0, c = 0; b0 < B; b0 += CH, ++c) {
                const int k = c % NB;
                unsigned char *d = blk + k * per;
                cudaMemcpyAsync(d, host + b0 * G, CH * G, cudaMemcpyHostToDevice, st[k]);
                touch<<<1024, 256, 0, st[k]>>>(d, CH * G);
                cudaMemcpyAsync(outh + b0 * 4 * 515, d + CH * G, CH * 4 * 515, cudaMemcpyDeviceToHost, st[k]);
            }
            for (int k = 0; k < NB; ++k) {
                cudaStreamSynchronize(st[k]);
                if (per_streams) cudaStreamDestroy(st[k]);
            }
            cudaEventDestroy(ev);
            if (per_alloc) {
                cudaFreeAsync(blk, cudaStreamPerThread);
                cudaStreamSynchronize(cudaStreamPerThread);
            }
            auto t1 = std::chrono::steady_clock::now();
            if (call >= 0) t[call] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
        printf("%c:", "ABCD"[variant]);
        for (int i = 0; i < 12; ++i) printf(" %.1f", t[i]);
        printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
