// peo_csr.cu -- the PEO check on CSR adjacency (the N = 10^6 configuration).
//
// Replaces _is_peo_lists (peo.py:100-149) and _first_witness_big (peo.py:152-174)
// for graphs that only expose adjacency lists.  For every v with a
// left neighbour: p = parent(v) = the left neighbour with the greatest position
// (given by the LexBFS, or searched here); v violates iff some z in N(v),
// z != p, pos(z) < pos(p), is not adjacent to p.  Violators lower one 64-bit
// key (p << 32 | v) with atomicMin -- the reference's first witness pair
// (parents ascending, then children ascending, peo.py:124-145); a one-warp
// kernel then resolves z (the smallest such z, adjacency lists ascending).
//
// One cooperative launch (peo_csr_kernel), grid = the resident CTAs:
//   light rows (deg <= kHeavy): kG = 8 lanes per vertex, four vertices in flight
//     per warp, every load of a round issued before any is used: the vertex's
//     header (prefetched one round ahead), then pos(p), N(p)'s bounds and 16
//     entries of N(v), then pos(z) and N(p) itself -- three dependent memory
//     round trips per vertex.  Membership z in N(p): when |N(p)| <= 32 the group
//     holds N(p) in registers and compares by shuffles; otherwise a binary
//     search in the shorter of N(p) and N(z) (z in N(p) <=> p in N(z)), all of a
//     lane's searches advancing in lockstep so their loads overlap.
//   heavy rows (deg > kHeavy; config 5: 2,211 rows, vertex 0 has 419,309
//     neighbours): listed in a queue in the caller's workspace during the light
//     phase; after a grid sync every CTA builds the rows' slice prefix in shared
//     memory and the grid takes kSlice-entry slices round robin (a parent pass
//     by 64-bit atomicMax of (pos + 1) << 32 | u, and one more grid sync, only
//     when some heavy row's parent is unknown).
// No global state: the queue lives in the workspace (chordal_peo_csr_workspace_bytes),
// its header cleared by a memset on the caller's stream.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace chordal {

namespace {

constexpr int kG = 8;            // lanes per light vertex
constexpr int kNG = 32 / kG;     // light vertices in flight per warp
constexpr int kU = 2;            // N(v) entries per lane per round (kG * kU = 16 per round)
constexpr int kUP = 4;           // N(p) entries per lane held in registers (kG * kUP = 32)
constexpr int kHeavy = 256;      // rows longer than this go to the queue
constexpr int kQueueCap = 4096;  // queued rows (further heavy rows: the light path checks them)
constexpr int kSlice = 256;      // entries per heavy work item (8 per lane)
constexpr int kSliceU = kSlice / 32;

struct HeavyQueue {
    int count;        // queued rows
    int need_parent;  // some queued row's parent is unknown
    int next_item;    // work-item claims (parent slices, stray slices, light chunks)
    int parent_done;  // parent slices finished
    int pad[4];
    int v[kQueueCap];
    int parent[kQueueCap];               // given, or -2
    unsigned long long pkey[kQueueCap];  // max (pos + 1) << 32 | u over left neighbours, 0 = none
};

// lockstep lower_bound of key_i in a[lo_i, hi_i) for the K searches of a lane
// (loads of one step are independent); found_i = key_i present.
template <int K>
__device__ __forceinline__ void lockstep_contains(const int32_t *__restrict__ a, const int64_t (&lo)[K],
                                                  const int64_t (&hi)[K], const int (&key)[K], bool (&found)[K]) {
    int64_t l[K], h[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        l[i] = lo[i];
        h[i] = hi[i];
    }
    for (;;) {
        bool any = false;
#pragma unroll
        for (int i = 0; i < K; ++i) any |= l[i] < h[i];
        if (!any) break;
        int val[K];
        int64_t mid[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            mid[i] = (l[i] + h[i]) >> 1;
            val[i] = l[i] < h[i] ? __ldg(a + mid[i]) : 0;
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (l[i] < h[i]) {
                if (val[i] < key[i]) l[i] = mid[i] + 1; else h[i] = mid[i];
            }
        }
    }
    int val[K];
#pragma unroll
    for (int i = 0; i < K; ++i) val[i] = l[i] < hi[i] ? __ldg(a + l[i]) : -1;
#pragma unroll
    for (int i = 0; i < K; ++i) found[i] = l[i] < hi[i] && val[i] == key[i];
}

// membership of the candidates z_i (cand_i) in N(p) = indices[pb, pe): binary
// search in N(p), or -- for a long N(p) -- for p in N(z_i) when that is shorter
template <int K>
__device__ __forceinline__ void adjacent_k(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                                           int p, int64_t pb, int64_t pe, const int (&z)[K], const bool (&cand)[K],
                                           bool (&adj)[K]) {
    int64_t lo[K], hi[K], zb[K], ze[K];
    int key[K];
    const bool longp = pe - pb > 64;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        zb[i] = (longp && cand[i]) ? __ldg(indptr + z[i]) : 0;
        ze[i] = (longp && cand[i]) ? __ldg(indptr + z[i] + 1) : 0;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (longp && ze[i] - zb[i] < pe - pb) {
            lo[i] = zb[i];
            hi[i] = ze[i];
            key[i] = p;
        } else {
            lo[i] = pb;
            hi[i] = pe;
            key[i] = z[i];
        }
        if (!cand[i]) lo[i] = hi[i] = 0;
    }
    lockstep_contains<K>(indices, lo, hi, key, adj);
}

}  // namespace

size_t peo_csr_workspace_bytes() { return (sizeof(HeavyQueue) + 255) & ~size_t(255); }

// The light path for one round of kNG vertices (one per kG-lane group):
// returns the group's violation in `viol` (lanes of the group agree).
__device__ __forceinline__ void light_round(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                                            const int32_t *__restrict__ pos, int v, bool act, int pv, int64_t b,
                                            int64_t e, int p, unsigned long long kmin, int sub, int sl,
                                            unsigned gmask, unsigned long long &k64, bool &viol) {
    // parent search where the LexBFS did not record it
    const bool need = act && p == -2;
    if (__any_sync(CH_FULL, need)) {
        unsigned long long best = 0;
        for (int64_t k0 = b; __any_sync(CH_FULL, need && k0 < e); k0 += kG * kU) {
            int u[kU], pu[kU];
#pragma unroll
            for (int i = 0; i < kU; ++i) {
                const int64_t k = k0 + sl + kG * i;
                u[i] = (need && k < e) ? __ldg(indices + k) : -1;
            }
#pragma unroll
            for (int i = 0; i < kU; ++i) pu[i] = u[i] >= 0 ? __ldg(pos + u[i]) : 0x7FFFFFFF;
#pragma unroll
            for (int i = 0; i < kU; ++i)
                if (pu[i] < pv) best = max(best, ((unsigned long long)(pu[i] + 1) << 32) | (unsigned)u[i]);
        }
#pragma unroll
        for (int d = kG / 2; d >= 1; d >>= 1) best = max(best, __shfl_xor_sync(CH_FULL, best, d));
        if (need) p = best ? (int)(best & 0xFFFFFFFFu) : -1;
    }
    act = act && p >= 0;
    k64 = ((unsigned long long)(unsigned)p << 32) | (unsigned)v;
    act = act && k64 < kmin;
    // round trip 2: p's position and bounds, the first entries of N(v)
    int z[kU];
#pragma unroll
    for (int i = 0; i < kU; ++i) {
        const int64_t k = b + sl + kG * i;
        z[i] = (act && k < e) ? __ldg(indices + k) : -1;
    }
    int pp = 0;
    int64_t pb = 0, pe = 0;
    if (act) {
        pp = __ldg(pos + p);
        pb = __ldg(indptr + p);
        pe = __ldg(indptr + p + 1);
    }
    const int dp = (int)(pe - pb);
    // N(p) in the group's registers when it is short: lane sl holds the block
    // N(p)[kUP*sl, kUP*sl + kUP) (INT_MAX padding)
    const bool shortp = act && dp <= kG * kUP;
    int np[kUP];
#pragma unroll
    for (int i = 0; i < kUP; ++i) {
        const int j = kUP * sl + i;
        np[i] = (shortp && j < dp) ? __ldg(indices + pb + j) : 0x7FFFFFFF;
    }
    const bool any_short = __any_sync(CH_FULL, shortp);
    viol = false;
    for (int64_t k0 = b; __any_sync(CH_FULL, act && k0 < e); k0 += kG * kU) {
        if (k0 != b) {
#pragma unroll
            for (int i = 0; i < kU; ++i) {
                const int64_t k = k0 + sl + kG * i;
                z[i] = (act && k < e) ? __ldg(indices + k) : -1;
            }
        }
        int pz[kU];
#pragma unroll
        for (int i = 0; i < kU; ++i) pz[i] = (z[i] >= 0 && z[i] != p) ? __ldg(pos + z[i]) : 0x7FFFFFFF;
        bool cand[kU], adj[kU];
#pragma unroll
        for (int i = 0; i < kU; ++i) {
            cand[i] = pz[i] < pp;
            adj[i] = false;
        }
        if (any_short) {  // find z's block by the block starts, then compare within it
            int nb[kU];
#pragma unroll
            for (int r = 0; r < kU; ++r) nb[r] = 0;
#pragma unroll
            for (int t = 0; t < kG; ++t) {
                const int s = __shfl_sync(CH_FULL, np[0], sub * kG + t);
#pragma unroll
                for (int r = 0; r < kU; ++r) nb[r] += s <= z[r];
            }
#pragma unroll
            for (int r = 0; r < kU; ++r) {
                const int src = sub * kG + max(nb[r] - 1, 0);
#pragma unroll
                for (int i = 0; i < kUP; ++i) adj[r] |= __shfl_sync(CH_FULL, np[i], src) == z[r];
            }
        }
        if (!shortp) adjacent_k<kU>(indptr, indices, p, pb, pe, z, cand, adj);
#pragma unroll
        for (int i = 0; i < kU; ++i) viol |= cand[i] && !adj[i];
        if (__ballot_sync(CH_FULL, viol) & gmask) act = false;  // this group is done
    }
    viol = (__ballot_sync(CH_FULL, viol) & gmask) != 0;
}

__global__ void __launch_bounds__(256, 4)
peo_csr_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
               const int32_t *__restrict__ pos, const int32_t *__restrict__ parent_in, int v_begin, int v_end,
               unsigned long long *__restrict__ key, HeavyQueue *__restrict__ Q, int heavy_thr) {
    __shared__ int pre[kQueueCap + 1];
    __shared__ int wsum[8];
    const int lane = threadIdx.x & 31;
    const int sub = lane / kG, sl = lane % kG;
    const unsigned gmask = ((1u << kG) - 1u) << (sub * kG);
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    cg::grid_group grid = cg::this_grid();

    // ---- phase 0: list the heavy rows --------------------------------------
    for (int v = v_begin + gtid; v < v_end; v += nthreads) {
        if (__ldg(indptr + v + 1) - __ldg(indptr + v) > heavy_thr) {
            const int slot = atomicAdd(&Q->count, 1);
            if (slot < kQueueCap) {
                const int p = parent_in ? __ldg(parent_in + v) : -2;
                Q->v[slot] = v;
                Q->parent[slot] = p;
                Q->pkey[slot] = 0;
                if (p == -2) Q->need_parent = 1;
            }
        }
    }
    grid.sync();
    const int cnt = min(*(volatile int *)&Q->count, kQueueCap);
    {  // slice prefix of the queued rows (every CTA builds its own copy)
        const int tid = threadIdx.x, w = tid >> 5;
        int carry = 0;
        for (int j0 = 0; j0 < cnt; j0 += blockDim.x) {
            const int j = j0 + tid;
            int s = 0;
            if (j < cnt) {
                const int vv = Q->v[j];
                s = (int)((__ldg(indptr + vv + 1) - __ldg(indptr + vv) + kSlice - 1) / kSlice);
            }
            int incl = s;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(CH_FULL, incl, d);
                if (lane >= d) incl += o;
            }
            if (lane == 31) wsum[w] = incl;
            __syncthreads();
            int off = carry, tot = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
                if (k < w) off += wsum[k];
                tot += wsum[k];
            }
            if (j < cnt) pre[j + 1] = off + incl;
            __syncthreads();
            carry += tot;
        }
        if (tid == 0) pre[0] = 0;
        __syncthreads();
    }
    auto row_of = [&](int item) {  // the row holding slice `item`: last j with pre[j] <= item
        int l = 0, h = cnt;
        while (h - l > 1) {
            const int mid = (l + h) >> 1;
            if (pre[mid] <= item) l = mid; else h = mid;
        }
        return l;
    };
    // ---- work items, claimed in order: heavy parent slices (only when some
    // parent is unknown), heavy stray slices, light chunks of kChunk vertices
    const int H = cnt ? pre[cnt] : 0;
    const int P = *(volatile int *)&Q->need_parent ? H : 0;
    constexpr int kChunk = 8 * kNG;  // eight rounds of kNG vertices
    const int L = (v_end - v_begin + kChunk - 1) / kChunk;
    const int total = P + H + L;
    unsigned long long kmin = ~0ULL;
    int item = 0;
    if (lane == 0) item = atomicAdd(&Q->next_item, 1);
    item = __shfl_sync(CH_FULL, item, 0);
    while (item < total) {
        int next = 0;  // the next claim, in flight while this item runs
        if (lane == 0) next = atomicAdd(&Q->next_item, 1);
        if (item < P + H) {
            const bool parent_pass = item < P;
            const int s = parent_pass ? item : item - P;
            const int j = row_of(s);
            const int vv = Q->v[j];
            const int pv = __ldg(pos + vv);
            const int64_t lo = __ldg(indptr + vv) + (int64_t)(s - pre[j]) * kSlice;
            const int64_t hi = min(__ldg(indptr + vv + 1), lo + kSlice);
            if (parent_pass) {
                if (Q->parent[j] == -2) {
                    int u[kSliceU], pu[kSliceU];
#pragma unroll
                    for (int i = 0; i < kSliceU; ++i) {
                        const int64_t k = lo + lane + 32 * i;
                        u[i] = k < hi ? __ldg(indices + k) : -1;
                    }
#pragma unroll
                    for (int i = 0; i < kSliceU; ++i) pu[i] = u[i] >= 0 ? __ldg(pos + u[i]) : 0x7FFFFFFF;
                    unsigned long long best = 0;
#pragma unroll
                    for (int i = 0; i < kSliceU; ++i)
                        if (pu[i] < pv) best = max(best, ((unsigned long long)(pu[i] + 1) << 32) | (unsigned)u[i]);
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) best = max(best, __shfl_xor_sync(CH_FULL, best, d));
                    if (lane == 0 && best) atomicMax(&Q->pkey[j], best);
                }
                if (lane == 0) {
                    __threadfence();
                    atomicAdd(&Q->parent_done, 1);
                }
            } else {
                if (P) {  // parent slices were all claimed before this one, by running warps
                    while (*(volatile int *)&Q->parent_done < P) __nanosleep(256);
                    __threadfence();
                }
                int p = Q->parent[j];
                if (p == -2) {
                    const unsigned long long pk = *(volatile unsigned long long *)&Q->pkey[j];
                    p = pk ? (int)(pk & 0xFFFFFFFFu) : -1;
                }
                const unsigned long long k64 = ((unsigned long long)(unsigned)p << 32) | (unsigned)vv;
                if (p >= 0 && k64 < *(volatile unsigned long long *)key) {
                    const int pp = __ldg(pos + p);
                    const int64_t pb = __ldg(indptr + p), pe = __ldg(indptr + p + 1);
                    int zz[kSliceU], pz[kSliceU];
#pragma unroll
                    for (int i = 0; i < kSliceU; ++i) {
                        const int64_t k = lo + lane + 32 * i;
                        zz[i] = k < hi ? __ldg(indices + k) : -1;
                    }
#pragma unroll
                    for (int i = 0; i < kSliceU; ++i)
                        pz[i] = (zz[i] >= 0 && zz[i] != p) ? __ldg(pos + zz[i]) : 0x7FFFFFFF;
                    bool viol = false;
#pragma unroll
                    for (int h = 0; h < kSliceU; h += 4) {  // four searches in flight per lane (register budget)
                        const int z4[4] = {zz[h], zz[h + 1], zz[h + 2], zz[h + 3]};
                        const bool c4[4] = {pz[h] < pp, pz[h + 1] < pp, pz[h + 2] < pp, pz[h + 3] < pp};
                        bool a4[4];
                        adjacent_k<4>(indptr, indices, p, pb, pe, z4, c4, a4);
#pragma unroll
                        for (int i = 0; i < 4; ++i) viol |= c4[i] && !a4[i];
                    }
                    if (__any_sync(CH_FULL, viol) && lane == 0) atomicMin(key, k64);
                }
            }
        } else {
            // light chunk: eight rounds, each round's vertex header loaded one round ahead
            kmin = *(volatile unsigned long long *)key;
            const int c0 = v_begin + (item - P - H) * kChunk;
            const int c1 = min(v_end, c0 + kChunk);
            int hv_pos = 0, hv_par = -1;
            int64_t hv_b = 0, hv_e = 0;
            if (c0 + sub < c1) {
                hv_pos = __ldg(pos + c0 + sub);
                hv_b = __ldg(indptr + c0 + sub);
                hv_e = __ldg(indptr + c0 + sub + 1);
                hv_par = parent_in ? __ldg(parent_in + c0 + sub) : -2;
            }
            for (int base = c0; base < c1; base += kNG) {
                const int v = base + sub;
                const bool in = v < c1;
                const int pv = hv_pos, p = hv_par;
                const int64_t b = hv_b, e = hv_e;
                const int vn = v + kNG;
                if (vn < c1) {
                    hv_pos = __ldg(pos + vn);
                    hv_b = __ldg(indptr + vn);
                    hv_e = __ldg(indptr + vn + 1);
                    hv_par = parent_in ? __ldg(parent_in + vn) : -2;
                }
                // queued rows were checked above (a full queue leaves the rest here)
                bool act = in && !(e - b > heavy_thr && cnt < kQueueCap);
                unsigned long long k64;
                bool viol;
                light_round(indptr, indices, pos, v, act, pv, b, e, p, kmin, sub, sl, gmask, k64, viol);
                if (viol && sl == 0) atomicMin(key, k64);
                const unsigned vm = __ballot_sync(CH_FULL, viol);
                if (vm) {
                    unsigned long long km = viol ? k64 : ~0ULL;
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) km = min(km, __shfl_xor_sync(CH_FULL, km, d));
                    kmin = min(kmin, km);
                }
            }
        }
        item = __shfl_sync(CH_FULL, next, 0);
    }
}

// One warp: resolve the minimum key to (v, p, z), z the smallest stray of N(v).
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
        const int64_t k = k0 + lane;
        const int zz[1] = {k < e ? indices[k] : -1};
        const bool cand[1] = {zz[0] >= 0 && zz[0] != p && pos[zz[0]] < pp};
        bool adj[1];
        adjacent_k<1>(indptr, indices, p, pb, pe, zz, cand, adj);
        const uint32_t m = __ballot_sync(CH_FULL, cand[0] && !adj[0]);
        if (m) {
            z = __shfl_sync(CH_FULL, zz[0], __ffs(m) - 1);
            break;
        }
    }
    if (lane == 0) {
        witness[0] = v;
        witness[1] = p;
        witness[2] = z;
    }
}

int launch_peo_csr_key(const int64_t *indptr, const int32_t *indices, int64_t n, const int32_t *pos,
                       const int32_t *parent, int64_t v_begin, int64_t v_end, uint64_t *key, void *ws,
                       cudaStream_t stream) {
    if (v_begin < 0) v_begin = 0;
    if (v_end > n) v_end = n;
    if (v_end <= v_begin) return CHORDAL_OK;
    HeavyQueue *Q = reinterpret_cast<HeavyQueue *>(ws);
    if (cudaMemsetAsync(Q, 0, 32, stream) != cudaSuccess) return CHORDAL_ECUDA;
    int dev = 0, sms = 148, occ = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, peo_csr_kernel, 256, 0);
    if (occ < 1) occ = 1;
    long long blocks = ((v_end - v_begin + kNG - 1) / kNG * 32 + 255) / 256;
    if (blocks > (long long)sms * occ) blocks = (long long)sms * occ;
    int vb = (int)v_begin, ve = (int)v_end, thr = kHeavy;
    unsigned long long *k = reinterpret_cast<unsigned long long *>(key);
    void *args[] = {(void *)&indptr, (void *)&indices, (void *)&pos, (void *)&parent, &vb, &ve, &k, &Q, &thr};
    if (cudaLaunchCooperativeKernel((const void *)peo_csr_kernel, dim3((unsigned)blocks), dim3(256), args, 0,
                                    stream) != cudaSuccess)
        return CHORDAL_ECUDA;
    return CHORDAL_OK;
}

int launch_peo_csr_witness(const int64_t *indptr, const int32_t *indices, const int32_t *pos, const uint64_t *key,
                           int32_t *witness, cudaStream_t stream) {
    peo_csr_witness_kernel<<<1, 32, 0, stream>>>(indptr, indices, pos,
                                                 reinterpret_cast<const unsigned long long *>(key), witness);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
