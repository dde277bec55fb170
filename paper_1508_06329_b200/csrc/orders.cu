// orders.cu -- the reference's other vertex orderings on the GPU:
//   mcs_order  (search.py:113-145)  maximum cardinality search, the ordering
//              whose PEO test is Tarjan-Yannakakis' chordality test (the
//              reference's test_peo.py:127-147 pairs it with is_peo);
//   bfs_order  (search.py:79-110)   breadth-first order with component
//              restarts.
// Both with LOWEST_INDEX ties or a seeded TieBreak replayed from the same
// Philox streams ("mcs" / "bfs", rng.py:18-21).
//
// MCS: one persistent CTA; the weight of every vertex (#visited neighbours,
// stored +1, 0 = visited) lives in shared memory as u16 (n <= 65535).  A step
// is one block-wide max over packed keys (w+1) << 16 | (0xFFFF - v) -- the
// largest weight, ties to the smallest id, exactly the reference's scan --
// then the pivot's row words bump its unvisited neighbours.  Seeded ties:
// count the vertices at the maximum weight (block scan over contiguous
// ranges, i.e. ascending id), draw Generator.integers(count), take that one.
//
// BFS: one warp on CSR rows.  The output order is the queue itself; a
// shared-memory bitset marks queued vertices.  Each popped vertex appends its
// unqueued neighbours in adjacency order (ballot + prefix per 32-neighbour
// chunk); seeded runs shuffle them with Generator.shuffle (Fisher-Yates,
// random_interval) and restart at pool[integers(len(pool))].
#include "common.cuh"
#include "philox.cuh"

namespace chordal {

namespace {

constexpr int kMcsMaxThreads = 1024;

// block-wide max of a u32, broadcast to every thread (two barriers)
__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = __reduce_max_sync(CH_FULL, v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    uint32_t r = lane < nw ? red[lane] : 0u;
    r = __reduce_max_sync(CH_FULL, r);
    __syncthreads();
    return r;
}

// block-wide exclusive sum (every thread gets its prefix and the total)
__device__ __forceinline__ int block_scan_excl(int v, int *red, int &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(CH_FULL, incl, d);
        if (lane >= d) incl += o;
    }
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    int w = lane < nw ? red[lane] : 0, wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(CH_FULL, wi, d);
        if (lane >= d) wi += o;
    }
    total = __shfl_sync(CH_FULL, wi, 31);
    const int before = __shfl_sync(CH_FULL, wi - w, warp);
    __syncthreads();
    return before + incl - v;
}

}  // namespace

template <bool SEEDED>
__global__ void __launch_bounds__(kMcsMaxThreads, 1)
mcs_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride, uint64_t key, int32_t *__restrict__ order,
                 int32_t *__restrict__ pos) {
    extern __shared__ __align__(16) uint16_t wsm[];  // weight + 1, 0 = visited
    __shared__ uint32_t red[32];
    __shared__ int redi[32];
    const int t = threadIdx.x, T = blockDim.x;
    const int C = ((n + T - 1) / T + 7) & ~7;  // contiguous vertex range per thread, multiple of 8
    const int v0 = t * C, v1 = min(n, v0 + C);
    const int npad = ((n + 7) & ~7);
    for (int v = t; v < npad; v += T) wsm[v] = v < n ? 1 : 0;
    __syncthreads();
    PhiloxStream rs(key);
    const uint32_t *rows = reinterpret_cast<const uint32_t *>(adj);
    const long long sw = stride >> 2;
    const int W = (n + 31) >> 5;
    for (int i = 0; i < n; ++i) {
        // ---- the unvisited vertex with the most visited neighbours -------------
        uint32_t best = 0;
        for (int v = v0; v < v1; v += 8) {
            const uint4 q = *reinterpret_cast<const uint4 *>(wsm + v);
            const uint32_t h[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t lo = h[k] & 0xFFFFu, hi = h[k] >> 16;
                const int va = v + 2 * k, vb = va + 1;
                if (lo) best = max(best, (lo << 16) | (uint32_t)(0xFFFF - va));
                if (hi && vb < v1) best = max(best, (hi << 16) | (uint32_t)(0xFFFF - vb));
            }
        }
        best = block_max_u32(best, red);
        int x = 0xFFFF - (int)(best & 0xFFFFu);
        if (SEEDED) {
            // ties = every unvisited vertex at the maximum weight, ascending id
            const uint32_t wmax = best >> 16;
            int c = 0;
            for (int v = v0; v < v1; ++v) c += wsm[v] == wmax;
            int total;
            const int before = block_scan_excl(c, redi, total);
            const int k = (int)rs.bounded(0, (uint64_t)(total - 1));
            if (k >= before && k < before + c) {
                int r = k - before;
                for (int v = v0; v < v1; ++v)
                    if (wsm[v] == wmax && r-- == 0) {
                        redi[0] = v;
                        break;
                    }
            }
            __syncthreads();
            x = redi[0];
            __syncthreads();
        }
        if (t == 0) {
            order[i] = x;
            pos[x] = i;
            wsm[x] = 0;
        }
        __syncthreads();
        // ---- visited-neighbour counts of x's unvisited neighbours -------------
        const uint32_t *rx = rows + (long long)x * sw;
        for (int w = t; w < W; w += T) {
            uint32_t b = __ldg(rx + w);
            while (b) {
                const int y = 32 * w + __ffs(b) - 1;
                b &= b - 1;
                const uint16_t cur = wsm[y];
                if (cur) wsm[y] = (uint16_t)(cur + 1);
            }
        }
        __syncthreads();
    }
}

// BFS on CSR rows, one warp.  `queued` is an n-bit bitset (shared or global).
// Neighbour sources of the BFS: append x's unqueued neighbours, ascending, at
// order[tail...] and mark them queued; returns the new tail.
struct BfsCsrRows {
    const int64_t *indptr;
    const int32_t *indices;
    __device__ __forceinline__ int append(int x, uint32_t *queued, int32_t *order, int tail) const {
        const int lane = threadIdx.x & 31;
        const uint32_t lt = (1u << lane) - 1u;
        const int64_t b = __ldg(indptr + x), e = __ldg(indptr + x + 1);
        for (int64_t c0 = b; c0 < e; c0 += 32) {
            const int64_t k = c0 + lane;
            const int y = k < e ? __ldg(indices + k) : 0;
            const bool fresh = k < e && !((queued[y >> 5] >> (y & 31)) & 1u);
            const uint32_t fm = __ballot_sync(CH_FULL, fresh);
            if (fresh) {
                order[tail + __popc(fm & lt)] = y;
                atomicOr(&queued[y >> 5], 1u << (y & 31));
            }
            tail += __popc(fm);
            __syncwarp();
        }
        return tail;
    }
};

// Dense rows: fresh = row & ~queued word by word, lane l owning a contiguous run
// of words so that one warp prefix sum places the fresh vertices in id order.
struct BfsDenseRows {
    const uint32_t *rows;
    long long sw;  // pitch in words
    int W;         // words holding vertex bits
    __device__ __forceinline__ int append(int x, uint32_t *queued, int32_t *order, int tail) const {
        const int lane = threadIdx.x & 31;
        const uint32_t *r = rows + (long long)x * sw;
        for (int base = 0; base < W; base += 32 * 8) {  // 8 words per lane per round
            const int w0 = base + 8 * lane;
            uint32_t f[8];
            int c = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int w = w0 + j;
                f[j] = w < W ? (__ldg(r + w) & ~queued[w]) : 0u;
                c += __popc(f[j]);
            }
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(CH_FULL, incl, d);
                if (lane >= d) incl += o;
            }
            int at = tail + incl - c;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint32_t m = f[j];
                if (m) queued[w0 + j] |= m;
                while (m) {
                    order[at++] = 32 * (w0 + j) + __ffs(m) - 1;
                    m &= m - 1;
                }
            }
            tail += __shfl_sync(CH_FULL, incl, 31);
            __syncwarp();
        }
        return tail;
    }
};

template <bool SEEDED, typename Rows>
__device__ void bfs_warp(const Rows &R, int n, uint64_t key, uint32_t *queued, int32_t *__restrict__ order,
                         int32_t *__restrict__ pos) {
    const int lane = threadIdx.x & 31;
    const int W = (n + 31) >> 5;
    for (int w = lane; w < W; w += 32) queued[w] = 0;
    __syncwarp();
    PhiloxStream rs(key);
    int head = 0, tail = 0, next_start = 0, nqueued = 0;
    while (head < n) {
        if (head == tail) {  // queue empty: restart (search.py:90-100)
            int s;
            if (!SEEDED) {
                while ((queued[next_start >> 5] >> (next_start & 31)) & 1u) ++next_start;
                s = next_start;
            } else {
                // pool = unqueued vertices ascending; s = pool[integers(len(pool))]
                int k = (int)rs.bounded(0, (uint64_t)(n - nqueued - 1));
                s = -1;
                for (int w0 = 0; w0 < W && s < 0; w0 += 32) {
                    const int w = w0 + lane;
                    uint32_t free_bits = 0;
                    if (w < W) {
                        free_bits = ~queued[w];
                        if (w == W - 1 && (n & 31)) free_bits &= mask_below(n & 31);
                    }
                    const int c = __popc(free_bits);
                    int incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int o = __shfl_up_sync(CH_FULL, incl, d);
                        if (lane >= d) incl += o;
                    }
                    const int excl = incl - c;
                    const bool mine = k >= excl && k < incl;
                    const uint32_t bm = __ballot_sync(CH_FULL, mine);
                    if (bm) {
                        const int src = __ffs(bm) - 1;
                        int v = -1;
                        if (mine) v = 32 * w + (int)__fns(free_bits, 0, k - excl + 1);
                        s = __shfl_sync(CH_FULL, v, src);
                    } else {
                        k -= __shfl_sync(CH_FULL, incl, 31);
                    }
                }
            }
            __syncwarp();  // the lanes' queued[] reads above precede lane 0's write
            if (lane == 0) {
                queued[s >> 5] |= 1u << (s & 31);
                order[tail] = s;
                pos[s] = tail;
            }
            ++tail;
            ++nqueued;
            __syncwarp();
        }
        const int x = order[head];
        ++head;
        const int t0 = tail;
        tail = R.append(x, queued, order, tail);
        if (SEEDED && tail - t0 > 1) {  // gen.shuffle(fresh) (search.py:104-105)
            // every lane draws (the stream stays identical across lanes), lane 0 swaps
            for (int i2 = tail - t0 - 1; i2 >= 1; --i2) {
                uint32_t mask = (uint32_t)i2;
                mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
                uint32_t j;
                while ((j = rs.next32() & mask) > (uint32_t)i2) {
                }
                if (lane == 0) {
                    const int32_t tmp = order[t0 + i2];
                    order[t0 + i2] = order[t0 + (int)j];
                    order[t0 + (int)j] = tmp;
                }
            }
        }
        nqueued += tail - t0;
        __syncwarp();
        for (int k = t0 + lane; k < tail; k += 32) pos[order[k]] = k;
        __syncwarp();
    }
}

constexpr int kBfsSmemMaxN = 227 * 1024 * 8 - 1024;

template <bool SEEDED>
__global__ void __launch_bounds__(32, 1)
bfs_csr_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n, uint64_t key,
               uint32_t *gqueued, int32_t *__restrict__ order, int32_t *__restrict__ pos) {
    extern __shared__ uint32_t squeued[];
    bfs_warp<SEEDED>(BfsCsrRows{indptr, indices}, n, key, gqueued ? gqueued : squeued, order, pos);
}

template <bool SEEDED>
__global__ void __launch_bounds__(32, 1)
bfs_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride, uint64_t key, int32_t *__restrict__ order,
                 int32_t *__restrict__ pos) {
    extern __shared__ uint32_t squeued[];
    bfs_warp<SEEDED>(BfsDenseRows{reinterpret_cast<const uint32_t *>(adj), stride >> 2, (n + 31) >> 5}, n, key,
                     squeued, order, pos);
}

int launch_bfs_dense(const uint8_t *adj, int64_t n, int64_t stride, bool seeded, uint64_t key, int32_t *order,
                     int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    if (n > 65535) return CHORDAL_ETOOLARGE;
    const size_t smem = (size_t)((n + 31) / 32) * sizeof(uint32_t);
    if (seeded)
        bfs_dense_kernel<true><<<1, 32, smem, stream>>>(adj, (int)n, stride, key, order, pos);
    else
        bfs_dense_kernel<false><<<1, 32, smem, stream>>>(adj, (int)n, stride, key, order, pos);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_mcs_dense(const uint8_t *adj, int64_t n, int64_t stride, bool seeded, uint64_t key, int32_t *order,
                     int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    if (n > 65535) return CHORDAL_ETOOLARGE;
    int T = (int)(((n + 7) / 8 + 31) / 32 * 32);
    T = T < 32 ? 32 : (T > kMcsMaxThreads ? kMcsMaxThreads : T);
    const size_t smem = (size_t)(((n + 7) & ~7LL) + 8) * sizeof(uint16_t);
    cudaError_t e;
    if (seeded) {
        e = cudaFuncSetAttribute(mcs_dense_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return CHORDAL_ECUDA;
        mcs_dense_kernel<true><<<1, T, smem, stream>>>(adj, (int)n, stride, key, order, pos);
    } else {
        e = cudaFuncSetAttribute(mcs_dense_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return CHORDAL_ECUDA;
        mcs_dense_kernel<false><<<1, T, smem, stream>>>(adj, (int)n, stride, key, order, pos);
    }
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

size_t bfs_csr_workspace_bytes(int64_t n) {
    return n > kBfsSmemMaxN ? (size_t)((n + 31) / 32) * sizeof(uint32_t) : 0;
}

int launch_bfs_csr(const int64_t *indptr, const int32_t *indices, int64_t n, bool seeded, uint64_t key,
                   uint32_t *ws, int32_t *order, int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    if (n > 0x7FFFFFF0LL) return CHORDAL_ETOOLARGE;
    const bool global = n > kBfsSmemMaxN;
    const size_t smem = global ? 0 : (size_t)((n + 31) / 32) * sizeof(uint32_t);
    uint32_t *gq = global ? ws : nullptr;
    if (global && !ws) return CHORDAL_EINVAL;
    cudaError_t e;
    if (seeded) {
        e = cudaFuncSetAttribute(bfs_csr_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return CHORDAL_ECUDA;
        bfs_csr_kernel<true><<<1, 32, smem, stream>>>(indptr, indices, (int)n, key, gq, order, pos);
    } else {
        e = cudaFuncSetAttribute(bfs_csr_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return CHORDAL_ECUDA;
        bfs_csr_kernel<false><<<1, 32, smem, stream>>>(indptr, indices, (int)n, key, gq, order, pos);
    }
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
