// csr.cu -- sparse (CSR) chordality test: LexBFS via the slot engine with its
// state in global memory (L2-resident), a vertex-parallel CSR PEO check, and
// the bitset -> CSR conversion used to route sparse dense-stored graphs here.
//
// Replaces, for adjacency-list inputs, lexbfs_partition(method="linked")
// (search.py:500-532) and _is_peo_lists (peo.py:100-149) -- the pair the
// reference runs on graphs that only expose n, m and adjacency_lists0()
// (the N = 10^6 configuration).
#include <mutex>

#include "common.cuh"
#include "slot_engine.cuh"

namespace chordal {

namespace {

// Workspace carve-up (bytes) of the slot engine's global-memory state: isz /
// ssz = bytes of the vertex/class (I) and slot (S) index types.  The slot
// capacity n + m + 64 covers every move of the search (each edge moves at most
// one endpoint, once), so compaction never runs for single graphs.
struct CsrWs {
    size_t cls, slot, c_head, c_end, c_live, c_prev, c_next, c_tgt, c_cnt, freel, touched, scratch, total;
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
        total = o;
    }
};

// u16 vertex/class ids (NIL = 0xFFFF) for n <= 32768; the per-neighbour arrays
// (cls, c_cnt, c_tgt) then fit in shared memory next to the staging buffer.
constexpr long long kSmemMaxN = 32768;
constexpr int kPeoHeavy = 4096;     // rows longer than this are checked by the whole grid
constexpr int kPeoHeavyMax = 4096;  // capacity of the heavy-row list

// rows with more neighbours than this are "heavy"; at least kPeoHeavy, raised
// with the edge count so that at most nnz / threshold < kPeoHeavyMax rows qualify
__device__ __forceinline__ int64_t heavy_threshold(const int64_t *__restrict__ indptr, int n) {
    const int64_t t = __ldg(indptr + n) / kPeoHeavyMax + 1;
    return t > kPeoHeavy ? t : (int64_t)kPeoHeavy;
}
constexpr int kNbrBuf = 4096;  // neighbour-list staging entries
inline size_t smem16_bytes(long long n) { return (size_t)(3 * n + 24 + kNbrBuf) * sizeof(uint16_t) + 64; }

__device__ __forceinline__ bool contains(const int32_t *__restrict__ a, int64_t lo, int64_t hi, int key) {
    // lower_bound then equality test
    int64_t l = lo, h = hi;
    while (l < h) {
        int64_t mid = (l + h) >> 1;
        if (__ldg(a + mid) < key) l = mid + 1; else h = mid;
    }
    return l < hi && __ldg(a + l) == key;
}

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

// Any n: all state in global memory (L2-resident), int32 ids; neighbour lists
// staged through shared memory.
template <int MODE>
__global__ void __launch_bounds__(32, 1)
lexbfs_csr_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n, long long m,
                  uint8_t *ws, int32_t *__restrict__ order, int32_t *__restrict__ pos, int32_t *__restrict__ parent,
                  uint64_t seed, uint64_t cell) {
    __shared__ int32_t nbuf[kNbrBuf];
    const CsrWs L(n, m, 4, 4);
    const SlotMem<int32_t, int32_t> M = carve<int32_t, int32_t>(ws, L);
    CsrStagedSource<int32_t> src{indptr, indices, nbuf, kNbrBuf, 0};
    slot_lexbfs<int32_t, int32_t, MODE, CsrStagedSource<int32_t>, int32_t>(src, n, M, order, pos, parent, seed, cell);
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
    CsrStagedSource<uint16_t> src{indptr, indices, nbuf, kNbrBuf, 0};
    slot_lexbfs<uint16_t, int32_t, MODE, CsrStagedSource<uint16_t>, int32_t>(src, n, M, order, pos, parent, seed,
                                                                              cell);
}

// ---------------------------------------------------------------------------
// PEO check on CSR: one warp per vertex v in [v_begin, v_end).
//   parent  given (from LexBFS) or the neighbour with the greatest position
//           before pos(v) (peo.py:106-121);
//   stray   some z in N(v), z != p, pos(z) < pos(p), z not in N(p) -- each
//           candidate is looked up in p's sorted list by binary search.
__global__ void __launch_bounds__(256)
peo_csr_key_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n,
                   const int32_t *__restrict__ pos, const int32_t *__restrict__ parent_in, int v_begin, int v_end,
                   unsigned long long *__restrict__ key) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int64_t heavy = heavy_threshold(indptr, n);
    // The current minimum key, refreshed every 16 vertices of this warp: read per
    // vertex, a million warps' loads of one address queued at one L2 slice and
    // made the check's time swing 0.8-1.8 ms between runs on configuration 5.
    unsigned long long kmin = ~0ULL;
    int it = 0;
    for (int v = v_begin + gw; v < v_end; v += nw, ++it) {
        if ((it & 15) == 0) kmin = *(volatile unsigned long long *)key;
        const int pv = __ldg(pos + v);
        const int64_t b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
        if (e - b > heavy) continue;  // heavy rows: split over the grid (peo_csr_heavy_*)
        int p = parent_in ? __ldg(parent_in + v) : -2;
        if (p == -2) {  // unknown: max position among the neighbours preceding v
            int best = -1;
            for (int64_t k = b + lane; k < e; k += 32) {
                int pu = __ldg(pos + __ldg(indices + k));
                if (pu < pv && pu > best) best = pu;
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) best = max(best, __shfl_xor_sync(CH_FULL, best, d));
            p = -1;
            if (best >= 0) {
                // the neighbour at that position
                for (int64_t k = b + lane; k < e; k += 32) {
                    int u = __ldg(indices + k);
                    if (__ldg(pos + u) == best) p = u;
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) p = max(p, __shfl_xor_sync(CH_FULL, p, d));
            }
        }
        if (p < 0) continue;
        const unsigned long long k64 = ((unsigned long long)p << 32) | (unsigned)v;
        if (k64 >= kmin) continue;
        const int pp = __ldg(pos + p);
        const int64_t pb = __ldg(indptr + p), pe = __ldg(indptr + p + 1);
        bool viol = false;
        for (int64_t k0 = b; k0 < e; k0 += 32) {
            int64_t k = k0 + lane;
            if (k < e) {
                int z = __ldg(indices + k);
                if (z != p && __ldg(pos + z) < pp && !contains(indices, pb, pe, z)) viol = true;
            }
            if (__any_sync(CH_FULL, viol)) { viol = true; break; }
        }
        if (viol) {
            if (lane == 0) atomicMin(key, k64);
            kmin = min(kmin, k64);
        }
    }
}

// ---- rows with more than kPeoHeavy neighbours (config 5: vertex 0 has 419,309)
// One warp per row would serialise the whole check behind them, so their
// neighbour lists are split into 1024-entry slices spread over the grid:
//   collect  list the heavy rows of [v_begin, v_end)
//   parent   (only where the search left it unknown) max position before
//            pos(v) over the slices (atomicMax), then the neighbour holding it
//   stray    every slice tests its candidates (z != p, pos(z) < pos(p),
//            z not in N(p)) and lowers the key on a hit.
struct PeoHeavy {
    int count;
    int pad;
    int v[kPeoHeavyMax];
    int best[kPeoHeavyMax];    // max position before pos(v) (parent search)
    int parent[kPeoHeavyMax];  // resolved parent, -1 none
};

constexpr int kHeavySlots = 4;
__device__ PeoHeavy g_peo_heavy[kHeavySlots];  // 4 x 48 KB per device

struct HeavySlots {
    std::mutex mu;
    PeoHeavy *base = nullptr;
    cudaEvent_t ev[kHeavySlots] = {};
    unsigned next = 0;
};

// one set per device (the module's __device__ array is per device too)
HeavySlots &heavy_slots() {
    static HeavySlots sets[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return sets[dev & 63];
}

__global__ void peo_csr_heavy_collect(const int64_t *__restrict__ indptr, int n, const int32_t *__restrict__ parent_in,
                                      int v_begin, int v_end, PeoHeavy *H) {
    const int64_t heavy = heavy_threshold(indptr, n);
    for (int v = v_begin + blockIdx.x * blockDim.x + threadIdx.x; v < v_end; v += gridDim.x * blockDim.x) {
        if (__ldg(indptr + v + 1) - __ldg(indptr + v) > heavy) {
            const int k = atomicAdd(&H->count, 1);
            if (k < kPeoHeavyMax) {
                H->v[k] = v;
                H->best[k] = -1;
                H->parent[k] = parent_in ? __ldg(parent_in + v) : -2;
            }
        }
    }
}

constexpr int kSlice = 1024;  // neighbours per warp work item

// every warp of the grid walks the (heavy row, slice) items
template <typename Fn>
__device__ __forceinline__ void for_each_heavy_slice(const int64_t *__restrict__ indptr, const PeoHeavy *H, Fn &&fn) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int cnt = min(H->count, kPeoHeavyMax);
    long long item = 0;
    for (int j = 0; j < cnt; ++j) {
        const int v = H->v[j];
        const int64_t b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
        const long long ns = (e - b + kSlice - 1) / kSlice;
        for (long long sidx = ((gw - item) % nw + nw) % nw; sidx < ns; sidx += nw) {
            const int64_t lo = b + sidx * kSlice, hi = min(e, lo + kSlice);
            fn(j, v, lo, hi);
        }
        item += ns;
    }
}

__global__ void __launch_bounds__(256) peo_csr_heavy_parent_max(const int64_t *__restrict__ indptr,
                                                                const int32_t *__restrict__ indices,
                                                                const int32_t *__restrict__ pos, PeoHeavy *H) {
    const int lane = threadIdx.x & 31;
    for_each_heavy_slice(indptr, H, [&](int j, int v, int64_t lo, int64_t hi) {
        if (H->parent[j] != -2) return;  // given by the search
        const int pv = __ldg(pos + v);
        int best = -1;
        for (int64_t k = lo + lane; k < hi; k += 32) {
            const int pu = __ldg(pos + __ldg(indices + k));
            if (pu < pv && pu > best) best = pu;
        }
        best = __reduce_max_sync(CH_FULL, best);
        if (lane == 0 && best >= 0) atomicMax(&H->best[j], best);
    });
}

__global__ void __launch_bounds__(256) peo_csr_heavy_parent_pick(const int64_t *__restrict__ indptr,
                                                                 const int32_t *__restrict__ indices,
                                                                 const int32_t *__restrict__ pos, PeoHeavy *H) {
    const int lane = threadIdx.x & 31;
    for_each_heavy_slice(indptr, H, [&](int j, int v, int64_t lo, int64_t hi) {
        if (H->parent[j] != -2) return;
        const int best = H->best[j];
        if (best < 0) {
            if (lo == __ldg(indptr + v) && lane == 0) H->parent[j] = -1;  // no left neighbour
            return;
        }
        for (int64_t k = lo + lane; k < hi; k += 32) {
            const int u = __ldg(indices + k);
            if (__ldg(pos + u) == best) H->parent[j] = u;  // unique: positions are distinct
        }
    });
}

__global__ void __launch_bounds__(256) peo_csr_heavy_stray(const int64_t *__restrict__ indptr,
                                                           const int32_t *__restrict__ indices,
                                                           const int32_t *__restrict__ pos, const PeoHeavy *H,
                                                           unsigned long long *__restrict__ key) {
    const int lane = threadIdx.x & 31;
    for_each_heavy_slice(indptr, H, [&](int j, int v, int64_t lo, int64_t hi) {
        const int p = H->parent[j];
        if (p < 0 || __ldg(pos + v) == 0) return;
        const unsigned long long k64 = ((unsigned long long)p << 32) | (unsigned)v;
        if (k64 >= *(volatile unsigned long long *)key) return;
        const int pp = __ldg(pos + p);
        const int64_t pb = __ldg(indptr + p), pe = __ldg(indptr + p + 1);
        bool viol = false;
        for (int64_t k0 = lo; k0 < hi; k0 += 32) {
            const int64_t k = k0 + lane;
            if (k < hi) {
                const int z = __ldg(indices + k);
                if (z != p && __ldg(pos + z) < pp && !contains(indices, pb, pe, z)) viol = true;
            }
            if (__any_sync(CH_FULL, viol)) { viol = true; break; }
        }
        if (viol && lane == 0) atomicMin(key, k64);
    });
}

__global__ void peo_csr_witness_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                                       const int32_t *__restrict__ pos, const unsigned long long *__restrict__ key,
                                       int32_t *__restrict__ witness) {
    const int lane = threadIdx.x & 31;
    const unsigned long long k64 = *key;
    if (k64 == ~0ULL) {
        if (lane < 3) witness[lane] = -1;
        return;
    }
    const int p = (int)(k64 >> 32), v = (int)(k64 & 0xFFFFFFFFu);
    const int pp = pos[p];
    const int64_t b = indptr[v], e = indptr[v + 1], pb = indptr[p], pe = indptr[p + 1];
    int z = -1;
    for (int64_t k0 = b; k0 < e; k0 += 32) {  // N(v) ascending: the first hit is the smallest z
        int64_t k = k0 + lane;
        bool hit = false;
        int zz = 0;
        if (k < e) {
            zz = indices[k];
            hit = zz != p && pos[zz] < pp && !contains(indices, pb, pe, zz);
        }
        uint32_t m = __ballot_sync(CH_FULL, hit);
        if (m) {
            z = __shfl_sync(CH_FULL, zz, __ffs(m) - 1);
            break;
        }
    }
    if (lane == 0) {
        witness[0] = v;
        witness[1] = p;
        witness[2] = z;
    }
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
    if (n <= kSmemMaxN) {
        const size_t sm = smem16_bytes(n);
        if (cudaFuncSetAttribute(lexbfs_csr_smem_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm) != cudaSuccess)
            return CHORDAL_ECUDA;
        lexbfs_csr_smem_kernel<MODE><<<1, 32, sm, stream>>>(indptr, indices, (int)n, m, w, order, pos, parent, seed,
                                                            cell);
    } else {
        lexbfs_csr_kernel<MODE><<<1, 32, 0, stream>>>(indptr, indices, (int)n, m, w, order, pos, parent, seed, cell);
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

int launch_peo_csr_key(const int64_t *indptr, const int32_t *indices, int64_t n, const int32_t *pos,
                       const int32_t *parent, int64_t v_begin, int64_t v_end, uint64_t *key, cudaStream_t stream) {
    if (v_begin < 0) v_begin = 0;
    if (v_end > n) v_end = n;
    if (v_end <= v_begin) return CHORDAL_OK;
    long long blocks = ((v_end - v_begin) * 32 + 255) / 256;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    peo_csr_key_kernel<<<(int)blocks, 256, 0, stream>>>(indptr, indices, (int)n, pos, parent, (int)v_begin,
                                                        (int)v_end, reinterpret_cast<unsigned long long *>(key));
    CH_LAUNCH_CHECK();
    // heavy rows: their list lives in one of a few static device slots, handed
    // out round robin; a slot's next user waits (on the device) for the event
    // its previous user recorded.  No allocation per call -- stream-ordered
    // pool blocks made single calls milliseconds slower at random.
    HeavySlots &hs = heavy_slots();
    std::lock_guard<std::mutex> lock(hs.mu);
    if (!hs.base && cudaGetSymbolAddress(reinterpret_cast<void **>(&hs.base), g_peo_heavy) != cudaSuccess)
        return CHORDAL_ECUDA;
    const int slot = (int)(hs.next++ % kHeavySlots);
    if (!hs.ev[slot]) {
        if (cudaEventCreateWithFlags(&hs.ev[slot], cudaEventDisableTiming) != cudaSuccess) return CHORDAL_ECUDA;
    } else if (cudaStreamWaitEvent(stream, hs.ev[slot], 0) != cudaSuccess) {
        return CHORDAL_ECUDA;
    }
    PeoHeavy *H = hs.base + slot;
    cudaMemsetAsync(H, 0, sizeof(int) * 2, stream);
    long long cb = (v_end - v_begin + 255) / 256;
    if (cb > 148LL * 8) cb = 148LL * 8;
    peo_csr_heavy_collect<<<(int)cb, 256, 0, stream>>>(indptr, (int)n, parent, (int)v_begin, (int)v_end, H);
    const int hb = 148 * 8;
    peo_csr_heavy_parent_max<<<hb, 256, 0, stream>>>(indptr, indices, pos, H);
    peo_csr_heavy_parent_pick<<<hb, 256, 0, stream>>>(indptr, indices, pos, H);
    peo_csr_heavy_stray<<<hb, 256, 0, stream>>>(indptr, indices, pos, H, reinterpret_cast<unsigned long long *>(key));
    const cudaError_t le = cudaGetLastError();
    if (cudaEventRecord(hs.ev[slot], stream) != cudaSuccess) return CHORDAL_ECUDA;
    return le == cudaSuccess ? CHORDAL_OK : CHORDAL_ECUDA;
}

int launch_peo_csr_witness(const int64_t *indptr, const int32_t *indices, const int32_t *pos, const uint64_t *key,
                           int32_t *witness, cudaStream_t stream) {
    peo_csr_witness_kernel<<<1, 32, 0, stream>>>(indptr, indices, pos,
                                                 reinterpret_cast<const unsigned long long *>(key), witness);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
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
