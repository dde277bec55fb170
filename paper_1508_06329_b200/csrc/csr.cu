// csr.cu -- sparse (CSR) LexBFS via the slot engine with its state in global
// memory (L2-resident), and the bitset -> CSR conversion used to route sparse
// dense-stored graphs here.  The CSR PEO check is in peo_csr.cu.
//
// Replaces, for adjacency-list inputs, lexbfs_partition(method="linked")
// (search.py:500-532) and _is_peo_lists (peo.py:100-149) -- the pair the
// reference runs on graphs that only expose n, m and adjacency_lists0()
// (the N = 10^6 configuration).
#include <cstdlib>

#include "common.cuh"
#include "slot_engine.cuh"

namespace chordal {

namespace {

// Workspace carve-up (bytes) of the slot engine's global-memory state: isz /
// ssz = bytes of the vertex/class (I) and slot (S) index types.  The slot
// capacity n + m + 64 covers every move of the search (each edge moves at most
// one endpoint, once), so compaction never runs for single graphs.
struct CsrWs {
    size_t cls, slot, c_head, c_end, c_live, c_prev, c_next, c_tgt, c_cnt, freel, touched, scratch, prog, total;
    long long cap;
    __host__ __device__ CsrWs(long long n, long long m, int isz, int ssz) {
        const long long nc = n + 2;
        cap = n + m + 64;
        size_t o = 0;
        auto take = [&](long long elems, int sz) { size_t r = o; o += ((size_t)elems * sz + 15) & ~size_t(15); return r; };
        cls = take(n, isz);
        slot = take(cap + slot_detail::kSlotPad, isz);
        c_head = take(nc, ssz);
        c_end = take(nc, ssz);
        c_live = take(nc, isz);
        c_prev = take(nc, isz);
        c_next = take(nc, isz);
        c_tgt = take(nc, isz);
        c_cnt = take(nc, isz);
        freel = take(nc, isz);
        touched = take(nc, isz);
        scratch = take(n, isz);
        prog = take(4, 4);  // search -> look-ahead warp hand-off (head class, done, step)
        total = o;
    }
};

// u16 vertex/class ids (NIL = 0xFFFF) for n <= 32768; the per-neighbour arrays
// (cls, c_cnt, c_tgt) then fit in shared memory next to the staging buffer.
constexpr long long kSmemMaxN = 32768;
constexpr int kNbrBuf = 4096;  // neighbour-list staging entries
inline size_t smem16_bytes(long long n) { return (size_t)(3 * n + 24 + kNbrBuf) * sizeof(uint16_t) + 64; }

}  // namespace

template <typename I, typename S>
__device__ __forceinline__ SlotMem<I, S> carve(uint8_t *ws, const CsrWs &L) {
    SlotMem<I, S> M;
    M.cls = reinterpret_cast<I *>(ws + L.cls);
    M.slot_v = reinterpret_cast<I *>(ws + L.slot);
    M.c_head = reinterpret_cast<S *>(ws + L.c_head);
    M.c_end = reinterpret_cast<S *>(ws + L.c_end);
    M.c_live = reinterpret_cast<I *>(ws + L.c_live);
    M.c_prev = reinterpret_cast<I *>(ws + L.c_prev);
    M.c_next = reinterpret_cast<I *>(ws + L.c_next);
    M.c_tgt = reinterpret_cast<I *>(ws + L.c_tgt);
    M.c_cnt = reinterpret_cast<I *>(ws + L.c_cnt);
    M.freel = reinterpret_cast<I *>(ws + L.freel);
    M.touched = reinterpret_cast<I *>(ws + L.touched);
    M.scratch = reinterpret_cast<I *>(ws + L.scratch);
    M.cap = L.cap;
    return M;
}

// Look-ahead warp (slot_lookahead): the next CSR_LOOKAHEAD live vertices of the
// class list, re-walked every CSR_LOOKAHEAD_EVERY steps (0: no look-ahead warp).
// Config 5: 1.85 s without, 1.615 s with 64 / 8, 1.67 s with 128 / 8, 1.595 s
// with 32 / 4 (tools/ab_variants.sh).  Re-measured after the fast-step early
// exits (profiles/r02_ab_la_final.txt): 32 / 4 1.316 s, 32 / 2 1.317 s, 64 / 4
// 1.321 s, 16 / 2 1.364 s -- 32 / 4 kept.
#ifndef CSR_LOOKAHEAD
#define CSR_LOOKAHEAD 32
#endif
#ifndef CSR_LOOKAHEAD_EVERY
#define CSR_LOOKAHEAD_EVERY 4
#endif

// Any n: all state in global memory (L2-resident), int32 ids; neighbour lists
// staged through shared memory.  Warp 0 runs the search; with CSR_LOOKAHEAD a
// second warp prefetches the next pivots' lists (slot_lookahead).
template <int MODE>
__global__ void __launch_bounds__(64, 1)
lexbfs_csr_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n, long long m,
                  uint8_t *ws, int32_t *__restrict__ order, int32_t *__restrict__ pos, int32_t *__restrict__ parent,
                  uint64_t seed, uint64_t cell) {
    __shared__ int32_t nbuf[kNbrBuf];
    // The hand-off to the look-ahead warp lives in global memory (the
    // workspace) and is read racily on purpose: the look-ahead only needs a
    // recent head class / step, and a stale one costs a useless prefetch.
    const CsrWs L(n, m, 4, 4);
    volatile int *prog = reinterpret_cast<volatile int *>(ws + L.prog);
    SlotMem<int32_t, int32_t> M = carve<int32_t, int32_t>(ws, L);
    slot_set_bounds(M, n, slot_detail::kSlotPad);
    if (threadIdx.x == 0) prog[0] = prog[1] = prog[2] = 0;
    __syncthreads();
    if (threadIdx.x >= 32) {
        if (CSR_LOOKAHEAD > 0)
            slot_lookahead<int32_t, int32_t>(indptr, indices, n, M, prog, CSR_LOOKAHEAD, CSR_LOOKAHEAD_EVERY);
        return;
    }
    CsrStagedSource<int32_t> src{indptr, indices, nbuf, kNbrBuf, 0};
    slot_lexbfs<int32_t, int32_t, MODE, CsrStagedSource<int32_t>, int32_t>(src, n, M, order, pos, parent, seed, cell,
                                                                           CSR_LOOKAHEAD > 0 ? prog : nullptr);
}

// n <= 32768: u16 ids; cls / c_cnt / c_tgt (192 KB at n = 32768) and the
// neighbour staging buffer live in shared memory, so a 32-neighbour chunk
// costs shared-memory latency only; class bookkeeping stays in global memory.
template <int MODE>
__global__ void __launch_bounds__(32, 1)
lexbfs_csr_smem_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n, long long m,
                       uint8_t *ws, int32_t *__restrict__ order, int32_t *__restrict__ pos,
                       int32_t *__restrict__ parent, uint64_t seed, uint64_t cell) {
    extern __shared__ __align__(16) uint16_t sm16[];
    const CsrWs L(n, m, 2, 4);
    SlotMem<uint16_t, int32_t> M = carve<uint16_t, int32_t>(ws, L);
    M.cls = sm16;
    M.c_cnt = sm16 + ((n + 7) & ~7);
    M.c_tgt = M.c_cnt + ((n + 2 + 7) & ~7);
    uint16_t *nbuf = M.c_tgt + ((n + 2 + 7) & ~7);
    slot_set_bounds(M, n, slot_detail::kSlotPad);
    CsrStagedSource<uint16_t> src{indptr, indices, nbuf, kNbrBuf, 0};
    slot_lexbfs<uint16_t, int32_t, MODE, CsrStagedSource<uint16_t>, int32_t>(src, n, M, order, pos, parent, seed,
                                                                              cell);
}

// Small sparse graphs: the whole engine state -- class bookkeeping and the slot
// array included -- in shared memory with u16 ids and u16 slot indices, so a
// step's chain of dependent reads (pivot slot -> neighbour classes -> class
// fields -> next head slot) costs shared-memory latency instead of L2 round
// trips.  Only the neighbour lists stay in global memory.  The slot array holds
// as many slots as fit (>= 2n + 64); when the bump pointer would overflow, the
// live slots are compacted (slot_detail::compact).
constexpr int kAllNbrBuf = 1024;
struct AllSmemLayout {
    size_t cls, slot, c_head, c_end, c_live, c_prev, c_next, c_tgt, c_cnt, freel, touched, scratch, nbuf, total;
    long long cap;
    __host__ __device__ AllSmemLayout(long long n, long long cap_) : cap(cap_) {
        const long long nc = n + 2;
        size_t o = 0;
        auto take = [&](long long elems) { size_t r = o; o += ((size_t)elems * 2 + 15) & ~size_t(15); return r; };
        cls = take(n);
        c_head = take(nc);
        c_end = take(nc);
        c_live = take(nc);
        c_prev = take(nc);
        c_next = take(nc);
        c_tgt = take(nc);
        c_cnt = take(nc);
        freel = take(nc);
        touched = take(nc);
        scratch = take(n);
        nbuf = take(kAllNbrBuf);
        slot = take(cap + slot_detail::kSlotPad);
        total = o;
    }
};
constexpr size_t kAllSmemMax = 232448;  // 227 KB of dynamic shared memory per block
// slot capacity for all-in-shared-memory state, or 0 when it does not fit
inline long long all_smem_cap(long long n, long long m) {
    if (n > 8836) return 0;  // 26 n + ~3 KB bytes must fit
    const AllSmemLayout L0(n, 0);
    const long long room = ((long long)kAllSmemMax - (long long)L0.total) / 2 - slot_detail::kSlotPad - 8;
    long long cap = n + m + 64 < room ? n + m + 64 : room;
    if (cap > 65000) cap = 65000;  // u16 slot indices
    return cap >= 2 * n + 64 ? cap : 0;
}

template <int MODE>
__global__ void __launch_bounds__(32, 1)
lexbfs_csr_allsmem_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n,
                          long long cap, int32_t *__restrict__ order, int32_t *__restrict__ pos,
                          int32_t *__restrict__ parent, uint64_t seed, uint64_t cell) {
    extern __shared__ __align__(16) uint8_t smb[];
    const AllSmemLayout L(n, cap);
    SlotMem<uint16_t, uint16_t> M;
    M.cls = reinterpret_cast<uint16_t *>(smb + L.cls);
    M.slot_v = reinterpret_cast<uint16_t *>(smb + L.slot);
    M.c_head = reinterpret_cast<uint16_t *>(smb + L.c_head);
    M.c_end = reinterpret_cast<uint16_t *>(smb + L.c_end);
    M.c_live = reinterpret_cast<uint16_t *>(smb + L.c_live);
    M.c_prev = reinterpret_cast<uint16_t *>(smb + L.c_prev);
    M.c_next = reinterpret_cast<uint16_t *>(smb + L.c_next);
    M.c_tgt = reinterpret_cast<uint16_t *>(smb + L.c_tgt);
    M.c_cnt = reinterpret_cast<uint16_t *>(smb + L.c_cnt);
    M.freel = reinterpret_cast<uint16_t *>(smb + L.freel);
    M.touched = reinterpret_cast<uint16_t *>(smb + L.touched);
    M.scratch = reinterpret_cast<uint16_t *>(smb + L.scratch);
    M.cap = cap;
    slot_set_bounds(M, n, slot_detail::kSlotPad);
    uint16_t *nbuf = reinterpret_cast<uint16_t *>(smb + L.nbuf);
    CsrStagedSource<uint16_t> src{indptr, indices, nbuf, kAllNbrBuf, 0};
    slot_lexbfs<uint16_t, uint16_t, MODE, CsrStagedSource<uint16_t>, int32_t>(src, n, M, order, pos, parent, seed,
                                                                               cell);
}

// ---------------------------------------------------------------------------
// bitset rows -> CSR (ascending per row)
__global__ void row_degrees_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                                   int64_t *__restrict__ deg) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int words = (n + 31) >> 5;
    for (int r = gw; r < n; r += nw) {
        const uint32_t *row = reinterpret_cast<const uint32_t *>(adj + (long long)r * stride);
        int c = 0;
        for (int w = lane; w < words; w += 32) c += __popc(__ldg(row + w));
        c = __reduce_add_sync(CH_FULL, c);
        if (lane == 0) deg[r + 1] = c;
    }
}

// single-block inclusive scan of deg[1..n] in place -> indptr (deg[0] = 0)
__global__ void scan_degrees_kernel(int64_t *__restrict__ indptr, int n) {
    __shared__ int64_t wsum[32];
    __shared__ int64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { carry = 0; indptr[0] = 0; }
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        int i = base + tid;
        int64_t v = i < n ? indptr[i + 1] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int64_t o = __shfl_up_sync(CH_FULL, v, d);
            if (lane >= d) v += o;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        if (warp == 0) {
            int64_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int64_t o = __shfl_up_sync(CH_FULL, s, d);
                if (lane >= d) s += o;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        int64_t pre = carry + (warp > 0 ? wsum[warp - 1] : 0);
        if (i < n) indptr[i + 1] = v + pre;
        __syncthreads();
        if (tid == blockDim.x - 1) carry = pre + v;
        __syncthreads();
    }
}

__global__ void fill_indices_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                                    const int64_t *__restrict__ indptr, int32_t *__restrict__ indices,
                                    long long cap) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int words = (n + 31) >> 5;
    for (int r = gw; r < n; r += nw) {
        const uint32_t *row = reinterpret_cast<const uint32_t *>(adj + (long long)r * stride);
        int64_t at = indptr[r];
        for (int w0 = 0; w0 < words; w0 += 32) {
            int w = w0 + lane;
            uint32_t x = w < words ? __ldg(row + w) : 0u;
            int c = __popc(x), incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int o = __shfl_up_sync(CH_FULL, incl, d);
                if (lane >= d) incl += o;
            }
            int64_t o = at + incl - c;
            while (x) {
                int b = __ffs(x) - 1;
                x &= x - 1;
                if (o < cap) indices[o] = 32 * w + b;  // never write past the caller's buffer
                ++o;
            }
            at += __shfl_sync(CH_FULL, incl, 31);
        }
    }
}

// ---------------------------------------------------------------------------
size_t csr_workspace_bytes(int64_t n, int64_t m) { return CsrWs(n, m, 4, 4).total; }

template <int MODE>
static int launch_csr_mode(const int64_t *indptr, const int32_t *indices, int64_t n, int64_t m, uint64_t seed,
                           uint64_t cell, int32_t *order, int32_t *pos, int32_t *parent, void *ws,
                           cudaStream_t stream) {
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    const long long acap = getenv("CSR_NO_ALLSMEM") ? 0 : all_smem_cap(n, m);
    if (acap > 0) {
        const size_t sm = AllSmemLayout(n, acap).total;
        if (cudaFuncSetAttribute(lexbfs_csr_allsmem_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm) != cudaSuccess)
            return CHORDAL_ECUDA;
        lexbfs_csr_allsmem_kernel<MODE><<<1, 32, sm, stream>>>(indptr, indices, (int)n, acap, order, pos, parent,
                                                               seed, cell);
    } else if (n <= kSmemMaxN) {
        const size_t sm = smem16_bytes(n);
        if (cudaFuncSetAttribute(lexbfs_csr_smem_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm) != cudaSuccess)
            return CHORDAL_ECUDA;
        lexbfs_csr_smem_kernel<MODE><<<1, 32, sm, stream>>>(indptr, indices, (int)n, m, w, order, pos, parent, seed,
                                                            cell);
    } else {
        lexbfs_csr_kernel<MODE><<<1, CSR_LOOKAHEAD > 0 ? 64 : 32, 0, stream>>>(indptr, indices, (int)n, m, w, order,
                                                                               pos, parent, seed, cell);
    }
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_lexbfs_csr(const int64_t *indptr, const int32_t *indices, int64_t n, int64_t m, int32_t tie_rule,
                      uint64_t seed, uint64_t cell, int32_t *order, int32_t *pos, int32_t *parent, void *ws,
                      cudaStream_t stream) {
    switch (tie_rule) {
        case CHORDAL_TIE_ASCENDING:
            return launch_csr_mode<CHORDAL_TIE_ASCENDING>(indptr, indices, n, m, seed, cell, order, pos, parent, ws,
                                                          stream);
        case CHORDAL_TIE_DESCENDING:
            return launch_csr_mode<CHORDAL_TIE_DESCENDING>(indptr, indices, n, m, seed, cell, order, pos, parent, ws,
                                                           stream);
        case CHORDAL_TIE_SEEDED_ARB:
            return launch_csr_mode<CHORDAL_TIE_SEEDED_ARB>(indptr, indices, n, m, seed, cell, order, pos, parent, ws,
                                                           stream);
        case CHORDAL_TIE_SEEDED_PARTITION:  // seed: the Philox key of (seed, "lexbfs-partition")
            return launch_csr_mode<CHORDAL_TIE_SEEDED_PARTITION>(indptr, indices, n, m, seed, cell, order, pos, parent,
                                                                 ws, stream);
        case CHORDAL_TIE_SEEDED_LABELS:  // seed: the Philox key of (seed, "lexbfs-labels")
            return launch_csr_mode<CHORDAL_TIE_SEEDED_LABELS>(indptr, indices, n, m, seed, cell, order, pos, parent,
                                                              ws, stream);
        default:
            return CHORDAL_EINVAL;
    }
}

int launch_dense_degrees(const uint8_t *adj, int64_t n, int64_t stride, int64_t *indptr, cudaStream_t stream) {
    long long blocks = (n * 32 + 255) / 256;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    row_degrees_kernel<<<(int)blocks, 256, 0, stream>>>(adj, (int)n, stride, indptr);
    CH_LAUNCH_CHECK();
    scan_degrees_kernel<<<1, 1024, 0, stream>>>(indptr, (int)n);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_dense_fill(const uint8_t *adj, int64_t n, int64_t stride, const int64_t *indptr, int32_t *indices,
                      int64_t cap, cudaStream_t stream) {
    long long blocks = (n * 32 + 255) / 256;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    fill_indices_kernel<<<(int)blocks, 256, 0, stream>>>(adj, (int)n, stride, indptr, indices, cap);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
