// lexbfs_dense.cu -- single-CTA persistent LexBFS over a packed adjacency bitset.
//
// Replaces the reference's LexBFS implementations for dense graphs:
//   lexbfs_partition / PartitionList   search.py:328-532
//   lexbfs_labels / _LabelChain        search.py:152-310
//   lexbfs_array                        _arraylex.py:22-65
//   parallel_lexbfs + kernels 1-4      parallel/lexbfs.py:37-262 (paper kernels
//                                      PAPER.md:810-840, one launch per step)
// with one persistent CTA that keeps the whole search state in shared memory
// and runs every LexBFS step between four __syncthreads barriers.
//
// State (all in SMEM, n <= 32768 so vertex ids and positions fit uint16):
//   arr[2][n]  the arrangement of *reached* unvisited vertices by priority:
//              positions [i+1, tail) are the label classes in descending label
//              order, each class a contiguous window sorted by the tie rule
//              (the _arraylex.py:17-19 invariant: the first unconsumed position
//              is the next pivot).  Double-buffered: step i reads one buffer
//              and scatters the refined arrangement into the other.
//   bnd[]      class-start bitmask over positions.
//   U[]        bitset (by vertex id) of unreached vertices -- the empty-label
//              class, always the lowest-priority class.  It is never stored in
//              arr, so a step costs O(|reached region|), not O(n).
//   segtot[]   per-segment count of pivot neighbours (scratch).
//
// Step i (pivot x = arr[i]):
//   phase 1  warp per 32 positions: flag F = adj(x, arr[p]) (ballot), class
//            starts B (ballot).  Thread per vertex word: ext = row_x & U.
//   phase 2  thread per 32-position word: block-wide segmented scan of the
//            flag counts (reset at class starts) and plain scan of |ext|;
//            segment ends publish their flagged totals and the new class
//            boundary s + T (the neighbour part C_x is placed before the
//            remainder, SPEC "replace C by C_x, C_2", search.py:440-463).
//            ext is appended at the tail as one new class (ascending id).
//   phase 3  warp per 32 positions: stable-partition scatter into the other
//            buffer: flagged -> s + rank_f, unflagged -> s + T + rank_u.
// Early exit: once U is empty and every reached position is a singleton
// class, the remaining order is the arrangement itself.
#include "common.cuh"

namespace chordal {

namespace {

struct Red {  // (score, id) max-reduction element
    uint64_t score;
    int32_t id;
};

__device__ __forceinline__ bool red_better(uint64_t s1, int32_t i1, uint64_t s2, int32_t i2) {
    return s1 > s2 || (s1 == s2 && i1 > i2);
}

// Tie score of candidate vertex v: larger wins.  ASCENDING -> smallest id,
// DESCENDING -> largest id, SEEDED_ARB -> splitmix64(prefix ^ (v+1)) with
// ties to the larger id (Arbitration.choose, parallel/engine.py:47-53).
template <int MODE>
__device__ __forceinline__ uint64_t tie_score(int32_t v, uint64_t prefix) {
    if (MODE == CHORDAL_TIE_ASCENDING) return (uint64_t)(0x7FFFFFFF - v);
    if (MODE == CHORDAL_TIE_DESCENDING) return (uint64_t)v;
    return splitmix64(prefix ^ (uint64_t)(v + 1));
}

__device__ __forceinline__ void warp_red(uint64_t &s, int32_t &id) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        uint64_t s2 = __shfl_xor_sync(CH_FULL, s, d);
        int32_t i2 = __shfl_xor_sync(CH_FULL, id, d);
        if (red_better(s2, i2, s, id)) { s = s2; id = i2; }
    }
}

// Block-wide (score,id) max; result broadcast to all threads.  Two barriers.
__device__ __forceinline__ void block_red(uint64_t &s, int32_t &id, uint64_t *rs, int32_t *ri) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_red(s, id);
    if (lane == 0) { rs[warp] = s; ri[warp] = id; }
    __syncthreads();
    s = lane < nw ? rs[lane] : 0;
    id = lane < nw ? ri[lane] : -1;
    warp_red(s, id);
    __syncthreads();
}

}  // namespace

// Shared-memory carve-up (bytes), W = ceil(n/32) position/vertex words.
struct LexLayout {
    size_t arrA, arrB, segtot, U, bnd, Fw, Bw, cin, lbin, red_s, red_i, wt, total;
    __host__ __device__ static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
    __host__ __device__ LexLayout(int W) {
        size_t np = size_t(W) * 32, o = 0;
        arrA = o; o = align16(o + np * 2);
        arrB = o; o = align16(o + np * 2);
        segtot = o; o = align16(o + np * 2);
        U = o; o = align16(o + size_t(W) * 4);
        bnd = o; o = align16(o + size_t(W + 2) * 4);
        Fw = o; o = align16(o + size_t(W) * 4);
        Bw = o; o = align16(o + size_t(W + 1) * 4);
        cin = o; o = align16(o + size_t(W) * 4);
        lbin = o; o = align16(o + size_t(W) * 4);
        red_s = o; o = align16(o + 32 * 8);
        red_i = o; o = align16(o + 32 * 4);
        wt = o; o = align16(o + 32 * 16);  // warp totals: cnt, flag, lb, ext
        total = o;
    }
};

template <int MODE>
__global__ void __launch_bounds__(1024, 1)
lexbfs_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride, uint64_t seed,
                    uint64_t cell, int32_t *__restrict__ order, int32_t *__restrict__ pos) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int W = (n + 31) >> 5;
    const LexLayout L(W);
    uint16_t *arrA = (uint16_t *)(smem + L.arrA);
    uint16_t *arrB = (uint16_t *)(smem + L.arrB);
    uint16_t *segtot = (uint16_t *)(smem + L.segtot);
    uint32_t *U = (uint32_t *)(smem + L.U);
    uint32_t *bnd = (uint32_t *)(smem + L.bnd);
    uint32_t *Fw = (uint32_t *)(smem + L.Fw);
    uint32_t *Bw = (uint32_t *)(smem + L.Bw);
    uint32_t *cin = (uint32_t *)(smem + L.cin);
    int32_t *lbin = (int32_t *)(smem + L.lbin);
    uint64_t *red_s = (uint64_t *)(smem + L.red_s);
    int32_t *red_i = (int32_t *)(smem + L.red_i);
    int32_t *wt = (int32_t *)(smem + L.wt);  // [4][32]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = blockDim.x, NW = T >> 5;

    for (int w = tid; w < W; w += T) {
        uint32_t full = (w == W - 1 && (n & 31)) ? mask_below(n & 31) : CH_FULL;
        U[w] = full;
        bnd[w] = 0;
    }
    if (tid < 2) bnd[W + tid] = 0;
    __syncthreads();
    // Every rule starts at vertex 0 (vertex 1 in the reference: the smallest id
    // for LOWEST_INDEX, pinned for parallel_lexbfs, parallel/lexbfs.py:173).
    if (tid == 0) {
        arrA[0] = 0;
        U[0] &= ~1u;
        bnd[0] |= 1u;
    }
    __syncthreads();

    int tail = 1;
    uint16_t *A = arrA, *An = arrB;
    for (int i = 0; i < n; ++i) {
        uint64_t prefix = 0;
        if (MODE == CHORDAL_TIE_SEEDED_ARB) prefix = mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell);
        if (i == tail) {
            // Reached region empty: the next pivot comes from the unreached
            // (empty-label) class -- a new component.
            uint64_t s = 0;
            int32_t id = -1;
            for (int w = tid; w < W; w += T) {
                uint32_t u = U[w];
                if (!u) continue;
                if (MODE == CHORDAL_TIE_ASCENDING) {
                    int32_t v = 32 * w + __ffs(u) - 1;
                    uint64_t sc = tie_score<MODE>(v, prefix);
                    if (id < 0 || red_better(sc, v, s, id)) { s = sc; id = v; }
                } else if (MODE == CHORDAL_TIE_DESCENDING) {
                    int32_t v = 32 * w + highest_bit(u);
                    uint64_t sc = tie_score<MODE>(v, prefix);
                    if (id < 0 || red_better(sc, v, s, id)) { s = sc; id = v; }
                } else {
                    while (u) {
                        int b = __ffs(u) - 1;
                        u &= u - 1;
                        int32_t v = 32 * w + b;
                        uint64_t sc = tie_score<MODE>(v, prefix);
                        if (id < 0 || red_better(sc, v, s, id)) { s = sc; id = v; }
                    }
                }
            }
            if (id < 0) s = 0;
            block_red(s, id, red_s, red_i);
            if (tid == 0) {
                A[i] = (uint16_t)id;
                U[id >> 5] &= ~(1u << (id & 31));
                bnd[i >> 5] |= 1u << (i & 31);
            }
            tail = i + 1;
            __syncthreads();
        } else if (MODE == CHORDAL_TIE_SEEDED_ARB && i > 0) {
            // Elect within the max-label class [i, e): all its members offer
            // themselves as `current` (parallel/lexbfs.py:216-225).
            __shared__ int s_e;
            if (warp == 0) {
                int e = tail;
                for (int w0 = (i + 1) >> 5; w0 * 32 < tail; w0 += 32) {
                    int w = w0 + lane;
                    uint32_t m = 0;
                    if (w * 32 < tail) {
                        m = bnd[w];
                        if (w == ((i + 1) >> 5)) m &= ~mask_below((i + 1) & 31);
                    }
                    uint32_t any = __ballot_sync(CH_FULL, m != 0);
                    if (any) {
                        int src = __ffs(any) - 1;
                        uint32_t mm = __shfl_sync(CH_FULL, m, src);
                        e = min(tail, (w0 + src) * 32 + __ffs(mm) - 1);
                        break;
                    }
                }
                if (lane == 0) s_e = e;
            }
            __syncthreads();
            const int e = s_e;
            uint64_t s = 0;
            int32_t id = -1, bp = -1;
            for (int p = i + tid; p < e; p += T) {
                int32_t v = A[p];
                uint64_t sc = tie_score<MODE>(v, prefix);
                if (id < 0 || red_better(sc, v, s, id)) { s = sc; id = v; bp = p; }
            }
            const int32_t my_id = id;
            block_red(s, id, red_s, red_i);
            __shared__ int s_bp;
            if (my_id == id && bp >= 0) s_bp = bp;
            __syncthreads();
            if (tid == 0 && s_bp != i) {
                uint16_t t0 = A[i];
                A[i] = A[s_bp];
                A[s_bp] = t0;
            }
            __syncthreads();
        }

        const int x = A[i];
        if (tid == 0) {
            order[i] = x;
            pos[x] = i;
        }
        const uint32_t *rowx = reinterpret_cast<const uint32_t *>(adj + (long long)x * stride);
        const int R = tail - (i + 1);
        const int Q = (R + 31) >> 5;

        // ---- phase 1: flags and class starts, warp per 32 positions ------
        for (int q = warp; q < Q; q += NW) {
            int p = i + 1 + 32 * q + lane;
            bool valid = p < tail;
            int v = valid ? A[p] : 0;
            bool f = valid && ((__ldg(rowx + (v >> 5)) >> (v & 31)) & 1u);
            bool b = valid && (((bnd[p >> 5] >> (p & 31)) & 1u) || p == i + 1);
            uint32_t fw = __ballot_sync(CH_FULL, f);
            uint32_t bw = __ballot_sync(CH_FULL, b);
            if (lane == 0) { Fw[q] = fw; Bw[q] = bw; }
        }
        uint32_t ext = 0;
        if (tid < W) ext = __ldg(rowx + tid) & U[tid];
        // Early-exit predicate on the state at the start of this step.
        bool pred = true;
        if (tid < W) {
            if (U[tid]) pred = false;
            int lo = max(i + 1, 32 * tid), hi = min(tail, 32 * tid + 32);
            if (lo < hi) {
                uint32_t live = mask_below(hi - 32 * tid) & ~mask_below(lo - 32 * tid);
                uint32_t B = bnd[tid];
                if (i + 1 >= 32 * tid && i + 1 < 32 * tid + 32) B |= 1u << ((i + 1) & 31);
                uint32_t E = (B >> 1) | (bnd[tid + 1] << 31);
                if (tail - 1 >= 32 * tid && tail - 1 < 32 * tid + 32) E |= 1u << ((tail - 1) & 31);
                if (live & ~(B & E)) pred = false;
            }
        }
        if (__syncthreads_and(pred)) {
            for (int p = i + 1 + tid; p < n; p += T) {
                int v = A[p];
                order[p] = v;
                pos[v] = p;
            }
            break;
        }

        // ---- phase 2: word-level segmented scan --------------------------
        uint32_t F = 0, B = 0;
        if (tid < Q) { F = Fw[tid]; B = Bw[tid]; }
        int flag = B != 0;
        int hb = flag ? highest_bit(B) : 0;
        int cnt = flag ? __popc(F & ~mask_below(hb)) : __popc(F);
        int lb = flag ? 32 * tid + hb : -1;
        int extc = __popc(ext);
        // inclusive warp scan: (cnt reset at flag) / max(lb) / sum(extc)
        int icnt = cnt, iflag = flag, ilb = lb, iext = extc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int oc = __shfl_up_sync(CH_FULL, icnt, d);
            int of = __shfl_up_sync(CH_FULL, iflag, d);
            int ol = __shfl_up_sync(CH_FULL, ilb, d);
            int oe = __shfl_up_sync(CH_FULL, iext, d);
            if (lane >= d) {
                if (!iflag) icnt += oc;
                iflag |= of;
                ilb = max(ilb, ol);
                iext += oe;
            }
        }
        if (lane == 31) { wt[warp] = icnt; wt[32 + warp] = iflag; wt[64 + warp] = ilb; wt[96 + warp] = iext; }
        // exclusive-in-warp
        int xcnt = __shfl_up_sync(CH_FULL, icnt, 1), xflag = __shfl_up_sync(CH_FULL, iflag, 1);
        int xlb = __shfl_up_sync(CH_FULL, ilb, 1), xext = __shfl_up_sync(CH_FULL, iext, 1);
        if (lane == 0) { xcnt = 0; xflag = 0; xlb = -1; xext = 0; }
        __syncthreads();
        // warp prefixes: lane j holds warp j's total; inclusive scan over warps
        int pc = lane < NW ? wt[lane] : 0, pf = lane < NW ? wt[32 + lane] : 0;
        int pl = lane < NW ? wt[64 + lane] : -1, pe = lane < NW ? wt[96 + lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int oc = __shfl_up_sync(CH_FULL, pc, d);
            int of = __shfl_up_sync(CH_FULL, pf, d);
            int ol = __shfl_up_sync(CH_FULL, pl, d);
            int oe = __shfl_up_sync(CH_FULL, pe, d);
            if (lane >= d) {
                if (!pf) pc += oc;
                pf |= of;
                pl = max(pl, ol);
                pe += oe;
            }
        }
        const int ktot = __shfl_sync(CH_FULL, pe, NW - 1);
        int wpc = __shfl_sync(CH_FULL, pc, (warp + 31) & 31), wpf = __shfl_sync(CH_FULL, pf, (warp + 31) & 31);
        int wpl = __shfl_sync(CH_FULL, pl, (warp + 31) & 31), wpe = __shfl_sync(CH_FULL, pe, (warp + 31) & 31);
        if (warp == 0) { wpc = 0; wpf = 0; wpl = -1; wpe = 0; }
        // combine(warp prefix, exclusive-in-warp)
        const int cnt_in = xflag ? xcnt : wpc + xcnt;
        const int lb_in = max(wpl, xlb);
        const int ext_pref = wpe + xext;

        if (tid < Q) {
            cin[tid] = cnt_in;
            lbin[tid] = lb_in;
            const uint32_t vb = mask_below(R - 32 * tid);
            const uint32_t Bn = (tid + 1 < Q) ? Bw[tid + 1] : 0u;
            uint32_t E = (B >> 1) | (Bn << 31);
            if (((R - 1) >> 5) == tid) E |= 1u << ((R - 1) & 31);
            E &= vb;
            uint32_t ends = E & ~B;  // ends of non-singleton segments
            while (ends) {
                int e = __ffs(ends) - 1;
                ends &= ends - 1;
                uint32_t below = B & mask_below(e + 1);
                int s, fb;
                if (below) {
                    int h = highest_bit(below);
                    s = 32 * tid + h;
                    fb = __popc(F & mask_below(e) & ~mask_below(h));
                } else {
                    s = lb_in;
                    fb = cnt_in + __popc(F & mask_below(e));
                }
                int Tt = fb + ((F >> e) & 1u);
                segtot[s] = (uint16_t)Tt;
                int len = 32 * tid + e - s + 1;
                if (Tt > 0 && Tt < len) {
                    int nb = i + 1 + s + Tt;
                    atomicOr(&bnd[nb >> 5], 1u << (nb & 31));
                }
            }
        }
        // Append the newly reached vertices as one class after the tail.
        if (ext) {
            int r = 0;
            uint32_t e2 = ext;
            while (e2) {
                int b = __ffs(e2) - 1;
                e2 &= e2 - 1;
                int idx = ext_pref + r++;
                int dst = (MODE == CHORDAL_TIE_DESCENDING) ? tail + (ktot - 1 - idx) : tail + idx;
                An[dst] = (uint16_t)(32 * tid + b);
            }
            U[tid] &= ~ext;
        }
        if (tid == 0 && ktot > 0) atomicOr(&bnd[tail >> 5], 1u << (tail & 31));
        __syncthreads();

        // ---- phase 3: stable-partition scatter into the other buffer -----
        for (int q = warp; q < Q; q += NW) {
            int rel = 32 * q + lane;
            if (rel < R) {
                int p = i + 1 + rel;
                int v = A[p];
                uint32_t Fq = Fw[q], Bq = Bw[q];
                uint32_t Bn = (q + 1 < Q) ? Bw[q + 1] : 0u;
                uint32_t E = (Bq >> 1) | (Bn << 31);
                if (((R - 1) >> 5) == q) E |= 1u << ((R - 1) & 31);
                int nrel = rel;
                bool single = ((Bq & E) >> lane) & 1u;
                if (!single) {
                    uint32_t below = Bq & mask_below(lane + 1);
                    int s, fb;
                    if (below) {
                        int h = highest_bit(below);
                        s = 32 * q + h;
                        fb = __popc(Fq & mask_below(lane) & ~mask_below(h));
                    } else {
                        s = lbin[q];
                        fb = (int)cin[q] + __popc(Fq & mask_below(lane));
                    }
                    int Tt = segtot[s];
                    nrel = ((Fq >> lane) & 1u) ? s + fb : s + Tt + (rel - s - fb);
                }
                An[i + 1 + nrel] = (uint16_t)v;
            }
        }
        tail += ktot;
        __syncthreads();
        uint16_t *t2 = A;
        A = An;
        An = t2;
    }
}

__global__ void positions_kernel(const int32_t *__restrict__ order, int n, int32_t *__restrict__ pos) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        pos[order[i]] = i;
}

int launch_lexbfs_dense(const uint8_t *adj, int64_t n, int64_t stride, int32_t tie_rule, uint64_t seed,
                        uint64_t cell, int32_t *order, int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    if (n > CHORDAL_DENSE_LEXBFS_MAX_N) return CHORDAL_ETOOLARGE;
    const int W = (int)((n + 31) >> 5);
    int T = ((W + 31) / 32) * 32;
    if (T < 32) T = 32;
    if (n > 2048 && T < 256) T = 256;
    if (T > 1024) T = 1024;
    const LexLayout L(W);
    const size_t smem = L.total;
    cudaError_t e;
    switch (tie_rule) {
        case CHORDAL_TIE_ASCENDING:
            e = cudaFuncSetAttribute(lexbfs_dense_kernel<CHORDAL_TIE_ASCENDING>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return CHORDAL_ECUDA;
            lexbfs_dense_kernel<CHORDAL_TIE_ASCENDING>
                <<<1, T, smem, stream>>>(adj, (int)n, stride, seed, cell, order, pos);
            break;
        case CHORDAL_TIE_DESCENDING:
            e = cudaFuncSetAttribute(lexbfs_dense_kernel<CHORDAL_TIE_DESCENDING>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return CHORDAL_ECUDA;
            lexbfs_dense_kernel<CHORDAL_TIE_DESCENDING>
                <<<1, T, smem, stream>>>(adj, (int)n, stride, seed, cell, order, pos);
            break;
        case CHORDAL_TIE_SEEDED_ARB:
            e = cudaFuncSetAttribute(lexbfs_dense_kernel<CHORDAL_TIE_SEEDED_ARB>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return CHORDAL_ECUDA;
            lexbfs_dense_kernel<CHORDAL_TIE_SEEDED_ARB>
                <<<1, T, smem, stream>>>(adj, (int)n, stride, seed, cell, order, pos);
            break;
        default:
            return CHORDAL_EINVAL;
    }
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_positions(const int32_t *order, int64_t n, int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    positions_kernel<<<blocks, 256, 0, stream>>>(order, (int)n, pos);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

// Relabel: out[r] bit s = adj[perm[r]][perm[s]].  Used to replay the
// reference's seeded array tie-break (search.py:535-541: ties go to the
// earliest vertex of a Philox permutation) with the ascending kernel.
__global__ void permute_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                                     const int32_t *__restrict__ perm, uint8_t *__restrict__ out) {
    const int words = (int)(stride >> 2);
    const long long total = (long long)n * words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(t / words), w = (int)(t % words);
        uint32_t bits = 0;
        if (32 * w < n) {
            const uint32_t *row = reinterpret_cast<const uint32_t *>(adj + (long long)__ldg(perm + r) * stride);
            const int hi = min(32, n - 32 * w);
            for (int j = 0; j < hi; ++j) {
                int u = __ldg(perm + 32 * w + j);
                bits |= ((__ldg(row + (u >> 5)) >> (u & 31)) & 1u) << j;
            }
        }
        reinterpret_cast<uint32_t *>(out + (long long)r * stride)[w] = bits;
    }
}

int launch_permute_dense(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *perm, uint8_t *out,
                         cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    long long total = n * (stride >> 2);
    long long blocks = (total + 255) / 256;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    permute_dense_kernel<<<(int)blocks, 256, 0, stream>>>(adj, (int)n, stride, perm, out);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

__global__ void fill_i32_kernel(int32_t *__restrict__ p, long long n, int32_t value) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = value;
}

int launch_fill_i32(int32_t *p, int64_t n, int32_t value, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    long long blocks = (n + 255) / 256;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    fill_i32_kernel<<<(int)blocks, 256, 0, stream>>>(p, n, value);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
