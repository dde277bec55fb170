// batch.cu -- is_chordal over many small independent graphs (n <= 1024).
//
// One warp per graph, four graphs per CTA (graph b + w * gridDim.x for warp w of
// CTA b), no CTA-level synchronisation.
// The warp runs the register-resident touched-segment LexBFS of warp_seg.cuh
// (any density; ~4 KB of shared state per graph at n = 512, so ~40 graphs are
// in flight per SM to hide the per-step latency) and then the PEO check.
// Replaces is_chordal (peo.py:177-202) called once per graph by the
// reference's bench loop (bench.py:86-95).
// PEO check: lanes stride over vertices; parent from the search (or a short
// backward scan over the order for vertices placed by the early exit); stray =
// A[v] & ~A[p] & ~{p} confirmed by pos < pos(p); the minimum (p << 32 | v) key
// is the reference's witness (peo.py:81-85).
#include "common.cuh"
#include "warp_seg.cuh"

namespace chordal {

namespace {


struct BatchLayout {  // shared memory per graph (one warp); the adjacency stays in global memory
    size_t A, An, P, par, F, NB, total;
    __host__ __device__ static size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
    __host__ __device__ BatchLayout(int n) {
        const size_t np = size_t((n + 31) >> 5) * 32;
        size_t o = 0;
        A = o; o = a16(o + np * 2);
        An = o; o = a16(o + np * 2);
        P = o; o = a16(o + np * 2);
        par = o; o = a16(o + np * 2);
        F = o; o = a16(o + 32 * 4);
        NB = o; o = a16(o + 32 * 4);
        total = o;
    }
};

}  // namespace

// (A single-graph form -- rows staged in shared memory, search, PEO check and
// witness in one launch -- measured slower than the separate one-warp search
// kernel + the grid-wide dense PEO kernels once the latter record the parents:
// config 1 is_chordal 0.62 -> 0.52 ms; a single warp checks 1000 vertices
// serially, and warps parked at a barrier beside the searching warp slow it
// down by 18 %.  Removed.)
template <int WPC, int MINB>
__global__ void __launch_bounds__(32 * WPC, MINB)
batch_chordal_kernel(const uint8_t *__restrict__ adj_all, long long batch, int n, int stride,
                     int32_t *__restrict__ orders, int32_t *__restrict__ witness) {
    extern __shared__ __align__(16) uint8_t smem[];
    const BatchLayout L(n);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w of CTA b takes graph b + w * gridDim.x
    const long long g = (long long)blockIdx.x + (long long)warp * gridDim.x;
    if (g >= batch) return;  // whole warp; the CTA never synchronises
    const int W = (n + 31) >> 5;
    const int sw = stride >> 2;  // row pitch in 32-bit words
    const uint32_t *A32 = reinterpret_cast<const uint32_t *>(adj_all + g * (long long)n * stride);
    uint8_t *ws = smem + warp * L.total;
    WarpSegMem M;
    M.A = (uint16_t *)(ws + L.A);
    M.An = (uint16_t *)(ws + L.An);
    M.P = (uint16_t *)(ws + L.P);
    M.par = (uint16_t *)(ws + L.par);
    M.F = (uint32_t *)(ws + L.F);
    M.NB = (uint32_t *)(ws + L.NB);
    const uint16_t *ord = M.A, *pos = M.P, *par = M.par;

    // ---- LexBFS -------------------------------------------------------------------
    if (n <= 512)
        warp_seg_lexbfs<CHORDAL_TIE_ASCENDING, false, false, 16>(A32, sw, n, M);
    else
        warp_seg_lexbfs<CHORDAL_TIE_ASCENDING, false, false, 32>(A32, sw, n, M);
    const bool have_parent = true;

    // ---- write the order ---------------------------------------------------
    int32_t *og = orders + g * n;
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(og) & 15) == 0) {  // 4 entries per 64-bit load / 128-bit store
        const uint2 *o2 = reinterpret_cast<const uint2 *>(ord);
        int4 *g4 = reinterpret_cast<int4 *>(og);
        for (int k = lane; k < (n >> 2); k += 32) {
            const uint2 w = o2[k];
            g4[k] = make_int4((int)(w.x & 0xFFFFu), (int)(w.x >> 16), (int)(w.y & 0xFFFFu), (int)(w.y >> 16));
        }
    } else {
        for (int k = lane; k < n; k += 32) og[k] = ord[k];
    }

    // ---- PEO check: lanes stride over vertices -----------------------------------
    unsigned long long best = ~0ULL;
    // the warp's smallest violation key so far, shared through the (now idle)
    // mover-flag words so that every lane skips the vertices it cannot beat
    unsigned long long *sbest = reinterpret_cast<unsigned long long *>(M.F);
    if (lane == 0) *sbest = ~0ULL;
    __syncwarp();
    for (int v = lane; v < n; v += 32) {
        const int pv = pos[v];
        if (pv == 0) continue;
        const uint32_t *__restrict__ rv = A32 + v * sw;
        int parent = have_parent ? (int)(int16_t)par[v] : -2;
        if (parent == -2) {  // not produced by the search: backward scan, then full pass
            parent = -1;
            const int lim = pv > 64 ? pv - 64 : 0;
            for (int q0 = pv - 1; q0 >= lim && parent < 0; q0 -= 4) {  // four probes per round trip
                int u[4];
                uint32_t w[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) u[k] = q0 - k >= lim ? (int)ord[q0 - k] : 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = q0 - k >= lim ? rv[u[k] >> 5] : 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (parent < 0 && ((w[k] >> (u[k] & 31)) & 1u)) parent = u[k];
            }
            if (parent < 0 && lim > 0) {
                int bp = -1;
                for (int w = 0; w < W; ++w) {
                    uint32_t m = rv[w];
                    while (m) {
                        int b = __ffs(m) - 1;
                        m &= m - 1;
                        int pu = pos[32 * w + b];
                        if (pu < pv && pu > bp) bp = pu;
                    }
                }
                if (bp >= 0) parent = ord[bp];
            }
        }
        if (parent < 0) continue;
        const unsigned long long k64 = ((unsigned long long)parent << 32) | (unsigned)v;
        if (k64 >= best || k64 >= *(volatile unsigned long long *)sbest) continue;
        const int pp = pos[parent];
        const uint4 *rv4 = reinterpret_cast<const uint4 *>(rv);
        const uint4 *rp4 = reinterpret_cast<const uint4 *>(A32 + parent * sw);
        bool viol = false;
        // 16 words (two rows x four 128-bit loads, all in flight) per round
        for (int w0 = 0; w0 < W && !viol; w0 += 16) {
            uint32_t a[16], b[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
                if (w0 + 4 * j < W) {
                    x = __ldg(rv4 + (w0 >> 2) + j);
                    y = __ldg(rp4 + (w0 >> 2) + j);
                }
                a[4 * j] = x.x; a[4 * j + 1] = x.y; a[4 * j + 2] = x.z; a[4 * j + 3] = x.w;
                b[4 * j] = y.x; b[4 * j + 1] = y.y; b[4 * j + 2] = y.z; b[4 * j + 3] = y.w;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int w = w0 + j;
                uint32_t m = a[j] & ~b[j];
                if ((parent >> 5) == w) m &= ~(1u << (parent & 31));
                while (m && !viol) {
                    const int bb = __ffs(m) - 1;
                    m &= m - 1;
                    if (pos[32 * w + bb] < pp) viol = true;
                }
            }
        }
        if (viol) {
            best = k64;
            atomicMin(sbest, k64);
        }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(CH_FULL, best, d);
        best = o < best ? o : best;
    }
    int32_t *wg = witness + 3 * g;
    if (best == ~0ULL) {
        if (lane < 3) wg[lane] = -1;
        return;
    }
    const int p = (int)(best >> 32), v = (int)(best & 0xFFFFFFFFu);
    const int pp = pos[p];
    const uint32_t *rv = A32 + v * sw, *rp = A32 + p * sw;
    uint32_t cand = 0;
    if (lane < W) {
        uint32_t m = rv[lane] & ~rp[lane];
        if ((p >> 5) == lane) m &= ~(1u << (p & 31));
        while (m) {
            int b = __ffs(m) - 1;
            m &= m - 1;
            if (pos[32 * lane + b] < pp) cand |= 1u << b;
        }
    }
    uint32_t any = __ballot_sync(CH_FULL, cand != 0);
    int src = __ffs(any) - 1;
    uint32_t c = __shfl_sync(CH_FULL, cand, src);
    if (lane == 0) {
        wg[0] = v;
        wg[1] = p;
        wg[2] = 32 * src + __ffs(c) - 1;
    }
}

template <int WPC, int MINB>
static int launch_batch_cfg(const uint8_t *adj, int64_t batch, int64_t n, int64_t stride, int32_t *orders,
                            int32_t *witness, cudaStream_t stream) {
    const BatchLayout L((int)n);
    const size_t smem = L.total * WPC;
    cudaError_t e = cudaFuncSetAttribute(batch_chordal_kernel<WPC, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return CHORDAL_ECUDA;
    const long long blocks = (batch + WPC - 1) / WPC;
    batch_chordal_kernel<WPC, MINB><<<(unsigned)blocks, 32 * WPC, smem, stream>>>(adj, batch, (int)n, (int)stride,
                                                                                  orders, witness);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_batch(const uint8_t *adj, int64_t batch, int64_t n, int64_t stride, int32_t *orders,
                 int32_t *witness, cudaStream_t stream) {
    if (batch <= 0) return CHORDAL_OK;
    if (n > 1024) return CHORDAL_ETOOLARGE;
    // Four warps per CTA, warp w of CTA b on graph b + w * gridDim.x, registers
    // capped at 56 per thread (9 CTAs = 36 warps per SM, 12 bytes of spill):
    // 7.56 ms per config-4 batch uncapped (71 registers, 28 warps), 7.12 at 64
    // (<4, 8>), 7.02 here, 7.20 at 48 (<4, 10>), 8.58 at 40; <2, 18> 7.40,
    // <8, 4> 7.25 (tools/ab_multi.sh).
#ifndef BATCH_MINB
#define BATCH_MINB 9  // round 2 re-check: 8 (64 registers) 6.25 ms, 10 (48, spills) 6.29 ms, 9: 5.95 ms
#endif
    return launch_batch_cfg<4, BATCH_MINB>(adj, batch, n, stride, orders, witness, stream);
}

}  // namespace chordal
