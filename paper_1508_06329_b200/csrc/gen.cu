// gen.cu -- device-side, bit-exact replay of the reference's dense generator.
//
// gen_dense_random(n, p, seed) (generate.py:32-56) draws one uniform double
// per ordered cell of each 1024-row block, row-major, from the Philox4x64-10
// stream keyed by mix64(seed, crc32("dense-random")) (rng.py:18-21), keeps
// the strict upper triangle (cols > row) and mirrors it.  Because the blocks
// are consecutive full rows, draw number k = u*n + v decides edge {u, v},
// u < v.  numpy's Philox increments its 256-bit counter before producing
// each 4-word block, so block c = k/4 + 1, word k%4; the double is
// (x >> 11) * 2^-53 (numpy random_standard_uniform).
//
// Kernel 1 writes every row word (upper-triangle bits only); kernel 2 ORs in
// the mirrored lower triangle with a 32x32 ballot bit-transpose per warp.
#include "common.cuh"
#include "philox.cuh"

namespace chordal {

namespace {

__device__ __forceinline__ uint64_t dense_key(long long seed, uint32_t crc) {
    // mix64(seed, crc32("dense-random")) -- _bitops.py:51-57
    return splitmix64(splitmix64((uint64_t)seed) ^ (uint64_t)crc);
}

}  // namespace

// One thread per (graph, row u, 32-bit word w).
__global__ void gen_dense_upper_kernel(uint8_t *__restrict__ adj, long long batch, int n, int stride,
                                       double p, long long seed0, long long seed_step, uint32_t crc) {
    const int words = stride >> 2;
    const long long total = batch * (long long)n * words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(t % words);
        const long long r = t / words;
        const int u = (int)(r % n);
        const long long b = r / n;
        uint32_t bits = 0;
        const int v0 = 32 * w;
        if (v0 + 31 > u && v0 < n) {
            const uint64_t key = dense_key(seed0 + b * seed_step, crc);
            const int vlo = max(v0, u + 1), vhi = min(v0 + 32, n);
            long long k = (long long)u * n + vlo;
            const long long kend = (long long)u * n + vhi;
            while (k < kend) {
                U4 blk = philox4x64_10((uint64_t)(k >> 2) + 1, key);
                for (int j = (int)(k & 3); j < 4 && k < kend; ++j, ++k) {
                    double d = (double)(blk.v[j] >> 11) * (1.0 / 9007199254740992.0);
                    if (d < p) bits |= 1u << ((int)(k - (long long)u * n) - v0);
                }
            }
        }
        reinterpret_cast<uint32_t *>(adj + r * stride)[w] = bits;
    }
}

// One warp per 32x32 lower tile (I >= J) of one graph: rows 32I+c, word J
// receive bit r = A[32J + r][32I + c] (upper triangle, written by kernel 1).
__global__ void gen_mirror_kernel(uint8_t *__restrict__ adj, long long batch, int n, int stride) {
    const int lane = threadIdx.x & 31;
    const int RB = (n + 31) >> 5;
    const long long tiles = (long long)RB * (RB + 1) / 2;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarp = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = gw; t < batch * tiles; t += nwarp) {
        const long long b = t / tiles;
        long long k = t % tiles;
        // tile index k -> (I, J) with 0 <= J <= I
        int I = (int)((sqrt(8.0 * (double)k + 1.0) - 1.0) * 0.5);
        while ((long long)I * (I + 1) / 2 > k) --I;
        while ((long long)(I + 1) * (I + 2) / 2 <= k) ++I;
        const int J = (int)(k - (long long)I * (I + 1) / 2);
        uint8_t *g = adj + b * (long long)n * stride;
        const int srow = 32 * J + lane;
        uint32_t src = srow < n ? reinterpret_cast<const uint32_t *>(g + (long long)srow * stride)[I] : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            uint32_t bal = __ballot_sync(CH_FULL, (src >> c) & 1u);
            if (lane == c) mine = bal;
        }
        const int drow = 32 * I + lane;
        if (drow < n && mine) {
            // each destination word has exactly one writer; on the diagonal
            // tile this warp is also the only reader of the word (read above)
            uint32_t *dst = reinterpret_cast<uint32_t *>(g + (long long)drow * stride) + J;
            *dst |= mine;
        }
    }
}

int launch_gen_dense_random(uint8_t *adj, int64_t batch, int64_t n, int64_t stride, double p,
                            int64_t seed0, int64_t seed_step, uint32_t crc, cudaStream_t stream) {
    const int threads = 256;
    long long total = batch * n * (stride >> 2);
    long long blocks = (total + threads - 1) / threads;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    gen_dense_upper_kernel<<<(int)blocks, threads, 0, stream>>>(adj, batch, (int)n, (int)stride, p, seed0,
                                                                seed_step, crc);
    CH_LAUNCH_CHECK();
    const long long RB = (n + 31) / 32;
    long long warps = batch * RB * (RB + 1) / 2;
    long long mblocks = (warps * 32 + threads - 1) / threads;
    if (mblocks > 148LL * 64) mblocks = 148LL * 64;
    gen_mirror_kernel<<<(int)mblocks, threads, 0, stream>>>(adj, batch, (int)n, (int)stride);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

// ---------------------------------------------------------------------------
// gen_chordal_random (generate.py:118-155) bit for bit, one thread per graph.
//
// numpy's Generator draws replayed exactly:
//   integers(lo, hi)  -> random_bounded_uint64(off=lo, rng=hi-1-lo): rng == 0
//                        draws nothing; rng < 2^32-1 uses Lemire's 32-bit
//                        rejection on next_uint32, which hands out the low
//                        then the high half of each 64-bit Philox output.
//   choice(P, size=w, replace=False) with P <= 10000 -> Floyd's algorithm
//                        over j = P-w .. P-1 with an open-addressing hash set
//                        of 2^ceil(log2(1.2 w)) slots, then an in-place
//                        Fisher-Yates shuffle (j = bounded(0, i), i = w-1..1).
// (Verified against numpy 2.3 on every configuration generator call.)
namespace chordal {

namespace {

__device__ __forceinline__ uint64_t chordal_key(long long seed, uint32_t crc) {
    return splitmix64(splitmix64((uint64_t)seed) ^ (uint64_t)crc);
}

__device__ __forceinline__ void set_edge(uint8_t *g, long long stride, int a, int b) {
    if (!g) return;  // edge-list mode: the attachment lists are the output
    reinterpret_cast<uint32_t *>(g + (long long)a * stride)[b >> 5] |= 1u << (b & 31);
    reinterpret_cast<uint32_t *>(g + (long long)b * stride)[a >> 5] |= 1u << (a & 31);
}

}  // namespace

__global__ void gen_chordal_kernel(uint8_t *__restrict__ adj, long long batch, int n, long long stride, int k,
                                   long long seed0, long long seed_step, uint32_t crc, int32_t *__restrict__ scratch,
                                   long long scratch_words, int hmask) {
    const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (b >= batch) return;
    uint8_t *g = adj ? adj + b * (long long)n * stride : nullptr;
    int32_t *att_off = scratch + b * scratch_words;
    int32_t *att_len = att_off + n;
    int32_t *hs = att_len + n;
    int32_t *lst = hs + (hmask + 1);
    PhiloxStream rs(chordal_key(seed0 + b * seed_step, crc));
    int32_t top = 0;
    att_off[0] = 0;
    att_len[0] = 0;
    for (int i = 1; i < n; ++i) {
        int32_t *out = lst + top;
        int cnt;
        if (k >= i) {
            for (int c = 0; c < i; ++c) {
                out[c] = c;
                set_edge(g, stride, i, c);
            }
            cnt = i;
        } else {
            long long want = (long long)k + (long long)(int64_t)rs.bounded((uint64_t)(int64_t)-1, 2);
            want = want < 1 ? 1 : (want > i ? i : want);
            const int j = (int)rs.bounded(0, (uint64_t)(i - 1));
            const int32_t *src = lst + att_off[j];
            const int plen = att_len[j];
            const int P = plen + 1;  // pool = att[j] ++ [j]
            if (want >= P) {
                for (int c = 0; c < plen; ++c) {
                    int v = src[c];
                    out[c] = v;
                    set_edge(g, stride, i, v);
                }
                out[plen] = j;
                set_edge(g, stride, i, j);
                cnt = P;
            } else {
                const int w = (int)want;
                // Floyd sampling of w distinct indices out of P
                const int setsize = (int)(1.2 * (double)w);
                int mask = setsize;
                mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
                for (int t = 0; t <= mask; ++t) hs[t] = -1;
                for (int jj = P - w; jj < P; ++jj) {
                    int val = (int)rs.bounded(0, (uint64_t)jj);
                    int loc = val & mask;
                    while (hs[loc] != -1 && hs[loc] != val) loc = (loc + 1) & mask;
                    if (hs[loc] == -1) {
                        hs[loc] = val;
                        out[jj - P + w] = val;
                    } else {
                        loc = jj & mask;
                        while (hs[loc] != -1) loc = (loc + 1) & mask;
                        hs[loc] = jj;
                        out[jj - P + w] = jj;
                    }
                }
                for (int t = w - 1; t >= 1; --t) {  // Fisher-Yates (shuffle=True)
                    int r = (int)rs.bounded(0, (uint64_t)t);
                    int tmp = out[r];
                    out[r] = out[t];
                    out[t] = tmp;
                }
                for (int c = 0; c < w; ++c) {  // pool[idx]
                    int id = out[c];
                    int v = id < plen ? src[id] : j;
                    out[c] = v;
                    set_edge(g, stride, i, v);
                }
                cnt = w;
            }
        }
        att_off[i] = top;
        att_len[i] = cnt;
        top += cnt;
    }
}

long long gen_chordal_scratch_words(int64_t n, int64_t k, int *hmask_out) {
    int setsize = (int)(1.2 * (double)(k + 2));
    int mask = setsize;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    if (hmask_out) *hmask_out = mask;
    // att_off[n] + att_len[n] + hash[mask+1] + lists (vertex i keeps <= min(i, k+1) entries)
    return 2 * n + (mask + 1) + n * (k + 1) + 4;
}

int launch_gen_chordal_random(uint8_t *adj, int64_t batch, int64_t n, int64_t stride, int64_t k, int64_t seed0,
                              int64_t seed_step, uint32_t crc, int32_t *scratch, cudaStream_t stream) {
    int hmask = 0;
    const long long words = gen_chordal_scratch_words(n, k, &hmask);
    if (cudaMemsetAsync(adj, 0, (size_t)batch * n * stride, stream) != cudaSuccess) return CHORDAL_ECUDA;
    if (k == 0 || n == 1) return CHORDAL_OK;  // edgeless, no draws (generate.py:133-134)
    const int threads = 64;
    const long long blocks = (batch + threads - 1) / threads;
    gen_chordal_kernel<<<(unsigned)blocks, threads, 0, stream>>>(adj, batch, (int)n, stride, (int)k, seed0, seed_step,
                                                                 crc, scratch, words, hmask);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

// Undirected edge list (0-based u[i], v[i]) -> packed rows; duplicates collapse
// (Graph._from_numpy_edges, graph.py:78-88, built in HBM instead of on the host).
__global__ void edges_to_dense_kernel(const int32_t *__restrict__ u, const int32_t *__restrict__ v, long long m,
                                      uint8_t *__restrict__ adj, long long stride) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m; e += (long long)gridDim.x * blockDim.x) {
        const int a = __ldg(u + e), b = __ldg(v + e);
        atomicOr(reinterpret_cast<unsigned int *>(adj + (long long)a * stride) + (b >> 5), 1u << (b & 31));
        atomicOr(reinterpret_cast<unsigned int *>(adj + (long long)b * stride) + (a >> 5), 1u << (a & 31));
    }
}

int launch_edges_to_dense(const int32_t *u, const int32_t *v, int64_t m, uint8_t *adj, int64_t n, int64_t stride,
                          cudaStream_t stream) {
    if (cudaMemsetAsync(adj, 0, (size_t)n * stride, stream) != cudaSuccess) return CHORDAL_ECUDA;
    if (m <= 0) return CHORDAL_OK;
    long long blocks = (m + 255) / 256;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    edges_to_dense_kernel<<<(int)blocks, 256, 0, stream>>>(u, v, m, adj, stride);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

// Edge list of gen_chordal_random from the generator's attachment lists:
// vertex i attached to lst[att_off[i] .. att_off[i] + att_len[i]) -> (i, v).
__global__ void edges_from_lists_kernel(const int32_t *__restrict__ att_off, const int32_t *__restrict__ att_len,
                                        const int32_t *__restrict__ lst, int n, int32_t *__restrict__ u,
                                        int32_t *__restrict__ v, long long *__restrict__ m_out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int o = i == 0 ? 0 : att_off[i], c = i == 0 ? 0 : att_len[i];
        for (int j = 0; j < c; ++j) {
            u[o + j] = i;
            v[o + j] = lst[o + j];
        }
        if (i == n - 1) *m_out = (long long)o + c;
    }
}

int launch_gen_chordal_edges(int64_t n, int64_t k, int64_t seed, uint32_t crc, int32_t *scratch, int32_t *u,
                             int32_t *v, long long *m_out, cudaStream_t stream) {
    int hmask = 0;
    const long long words = gen_chordal_scratch_words(n, k, &hmask);
    if (k == 0 || n == 1) {
        return cudaMemsetAsync(m_out, 0, sizeof(long long), stream) == cudaSuccess ? CHORDAL_OK : CHORDAL_ECUDA;
    }
    gen_chordal_kernel<<<1, 32, 0, stream>>>(nullptr, 1, (int)n, 0, (int)k, seed, 1, crc, scratch, words, hmask);
    CH_LAUNCH_CHECK();
    const int32_t *att_off = scratch, *att_len = scratch + n, *lst = scratch + 2 * n + (hmask + 1);
    long long blocks = (n + 255) / 256;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    edges_from_lists_kernel<<<(int)blocks, 256, 0, stream>>>(att_off, att_len, lst, (int)n, u, v, m_out);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
