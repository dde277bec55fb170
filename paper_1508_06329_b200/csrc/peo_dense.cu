// peo_dense.cu -- vertex-parallel perfect-elimination-order check on bitsets.
//
// Replaces is_peo (peo.py:72-174: _is_peo_lists, peo_holds_array via
// _left_rows_packed, _first_witness_big) and parallel_peo_test
// (parallel/peo.py:37-95: preparationLNandP + testing).
//
// One warp per vertex v, grid-stride over v in [v_begin, v_end):
//   parent   p(v) = the left neighbour with the greatest position.  A warp
//            scans positions pos(v)-1, pos(v)-2, ... 32 at a time testing the
//            adjacency bit A[v][order[q]] (ballot -> first hit).  After a few
//            rounds without a hit it switches to a pass over the set bits of
//            row v keeping max pos(u) < pos(v) (cost = deg(v) lookups).
//   stray    LN(v)\{p} subset of LN(p)  <=>  no z in A[v] & ~A[p] & ~{p} with
//            pos(z) < pos(p)  (every z in LN(v)\{p} precedes p because p is
//            the latest left neighbour).  Rows are streamed with 128-bit loads;
//            candidates are confirmed with a pos[] lookup; the warp stops at
//            its first stray (ballot).
//   key      violating v lowers a global 64-bit key (p << 32) | v with
//            atomicMin; the minimum is exactly the reference's first witness
//            pair (parents ascending, then children ascending, peo.py:81-85).
//            Warps whose key already exceeds the running minimum skip the
//            subset test.
// The witness kernel then resolves z = min id of the stray set for the
// winning pair (peo.py:126-141).
#include "common.cuh"

namespace chordal {

namespace {

constexpr int kBackRounds = 4;  // 128 candidate positions before the full pass
constexpr int kRowU4 = 8;       // uint4 per lane per row chunk: 32 x 8 x 16 B = 4 KB (n = 32768) per round

__device__ __forceinline__ bool row_bit(const uint32_t *row, int v) {
    return (__ldg(row + (v >> 5)) >> (v & 31)) & 1u;
}

}  // namespace

__global__ void __launch_bounds__(256)
peo_dense_key_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                     const int32_t *__restrict__ order, const int32_t *__restrict__ pos,
                     const int32_t *__restrict__ parent_in, int v_begin, int v_end,
                     unsigned long long *__restrict__ key) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n4 = (n + 127) >> 7;  // uint4 per row holding vertex bits
    for (int v = v_begin + gw; v < v_end; v += nwarps) {
        const int pv = __ldg(pos + v);
        if (pv == 0) continue;
        const uint32_t *rowv = reinterpret_cast<const uint32_t *>(adj + (long long)v * stride);
        // ---- parent: given by the search, else backward scan ---------------
        int parent = parent_in ? __ldg(parent_in + v) : -2;  // -2: unknown, search it
        bool exhausted = parent != -2;
        if (parent == -2) parent = -1;
        for (int r = 0; r < kBackRounds && !exhausted; ++r) {
            int q = pv - 1 - (32 * r + lane);
            bool hit = q >= 0 && row_bit(rowv, __ldg(order + q));
            uint32_t m = __ballot_sync(CH_FULL, hit);
            if (m) {
                parent = __ldg(order + pv - 1 - (32 * r + __ffs(m) - 1));
                break;
            }
            if (pv - 1 - 32 * (r + 1) < 0) { exhausted = true; break; }
        }
        if (parent < 0 && !exhausted) {
            // full pass: max position among neighbours that precede v
            int best = -1;
            const uint4 *r4 = reinterpret_cast<const uint4 *>(rowv);
            for (int k = lane; k < n4; k += 32) {
                uint4 w4 = __ldg(r4 + k);
                uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t w = ws[j];
                    while (w) {
                        int b = __ffs(w) - 1;
                        w &= w - 1;
                        int u = 128 * k + 32 * j + b;
                        int pu = __ldg(pos + u);
                        if (pu < pv && pu > best) best = pu;
                    }
                }
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) best = max(best, __shfl_xor_sync(CH_FULL, best, d));
            if (best >= 0) parent = __ldg(order + best);
        }
        if (parent < 0) continue;
        const unsigned long long k64 = ((unsigned long long)parent << 32) | (unsigned)v;
        if (k64 >= *(volatile unsigned long long *)key) continue;
        // ---- stray test: A[v] & ~A[p] & ~{p}, confirmed by pos < pos(p) ---
        // Rows go in chunks of 32 x kRowU4 uint4 per warp with every load of a
        // chunk issued before any is used (one memory round trip per 4 KB of
        // row per warp); p is excluded by setting its bit in the copy of A[p];
        // candidate positions are looked up eight at a time.
        const int pp = __ldg(pos + parent);
        const uint4 *rv4 = reinterpret_cast<const uint4 *>(rowv);
        const uint4 *rp4 = reinterpret_cast<const uint4 *>(adj + (long long)parent * stride);
        bool viol = false;
        for (int k0 = 0; k0 < n4 && !viol; k0 += 32 * kRowU4) {
            uint4 a[kRowU4], b[kRowU4];
#pragma unroll
            for (int j = 0; j < kRowU4; ++j) {
                const int k = k0 + 32 * j + lane;
                a[j] = make_uint4(0, 0, 0, 0);
                b[j] = make_uint4(0, 0, 0, 0);
                if (k < n4) {
                    a[j] = __ldg(rv4 + k);
                    b[j] = __ldg(rp4 + k);
                }
            }
#pragma unroll
            for (int j = 0; j < kRowU4; ++j) {
                const int k = k0 + 32 * j + lane;
                if ((parent >> 7) == k) {  // exclude p itself
                    const uint32_t pb = 1u << (parent & 31);
                    switch ((parent >> 5) & 3) {
                        case 0: b[j].x |= pb; break;
                        case 1: b[j].y |= pb; break;
                        case 2: b[j].z |= pb; break;
                        default: b[j].w |= pb; break;
                    }
                }
                const uint32_t ws[4] = {a[j].x & ~b[j].x, a[j].y & ~b[j].y, a[j].z & ~b[j].z, a[j].w & ~b[j].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t w = ws[q];
                    const int base = 128 * k + 32 * q;
                    while (w && !viol) {  // up to eight position lookups in flight
                        int z[8], pz[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            z[u] = w ? base + __ffs(w) - 1 : -1;
                            w &= w - 1;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) pz[u] = z[u] >= 0 ? __ldg(pos + z[u]) : 0x7FFFFFFF;
#pragma unroll
                        for (int u = 0; u < 8; ++u) viol |= pz[u] < pp;
                    }
                }
            }
            viol = __any_sync(CH_FULL, viol);
        }
        if (viol && lane == 0) atomicMin(key, k64);
    }
}

// One warp: resolve the minimum key to (v, p, z).
__global__ void peo_dense_witness_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                                         const int32_t *__restrict__ pos,
                                         const unsigned long long *__restrict__ key,
                                         int32_t *__restrict__ witness) {
    const int lane = threadIdx.x & 31;
    const unsigned long long k64 = *key;
    if (k64 == ~0ULL) {
        if (lane < 3) witness[lane] = -1;
        return;
    }
    const int p = (int)(k64 >> 32), v = (int)(k64 & 0xFFFFFFFFu);
    const int pp = pos[p];
    const uint32_t *rv = reinterpret_cast<const uint32_t *>(adj + (long long)v * stride);
    const uint32_t *rp = reinterpret_cast<const uint32_t *>(adj + (long long)p * stride);
    const int nw = (n + 31) >> 5;
    int z = -1;
    for (int w0 = 0; w0 < nw; w0 += 32) {
        int w = w0 + lane;
        uint32_t cand = 0;
        if (w < nw) {
            uint32_t s = rv[w] & ~rp[w];
            if (p >> 5 == w) s &= ~(1u << (p & 31));
            while (s) {
                int b = __ffs(s) - 1;
                s &= s - 1;
                if (pos[32 * w + b] < pp) cand |= 1u << b;
            }
        }
        uint32_t any = __ballot_sync(CH_FULL, cand != 0);
        if (any) {
            int src = __ffs(any) - 1;
            uint32_t c = __shfl_sync(CH_FULL, cand, src);
            z = 32 * (w0 + src) + __ffs(c) - 1;
            break;
        }
    }
    if (lane == 0) {
        witness[0] = v;
        witness[1] = p;
        witness[2] = z;
    }
}

__global__ void key_init_kernel(unsigned long long *key) { *key = ~0ULL; }

int launch_key_init(uint64_t *key, cudaStream_t stream) {
    key_init_kernel<<<1, 1, 0, stream>>>(reinterpret_cast<unsigned long long *>(key));
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_peo_dense_key(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *order,
                         const int32_t *pos, const int32_t *parent, int64_t v_begin, int64_t v_end, uint64_t *key,
                         cudaStream_t stream) {
    if (v_begin < 0) v_begin = 0;
    if (v_end > n) v_end = n;
    if (v_end <= v_begin) return CHORDAL_OK;
    const int64_t nv = v_end - v_begin;
    const int threads = 256;
    int64_t blocks = (nv * 32 + threads - 1) / threads;
    const int64_t cap = 148LL * 16;
    if (blocks > cap) blocks = cap;
    peo_dense_key_kernel<<<(int)blocks, threads, 0, stream>>>(
        adj, (int)n, stride, order, pos, parent, (int)v_begin, (int)v_end,
        reinterpret_cast<unsigned long long *>(key));
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_peo_dense_witness(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *pos,
                             const uint64_t *key, int32_t *witness, cudaStream_t stream) {
    peo_dense_witness_kernel<<<1, 32, 0, stream>>>(
        adj, (int)n, stride, pos, reinterpret_cast<const unsigned long long *>(key), witness);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
