// slot_engine.cuh -- warp-level LexBFS by partition refinement in O(deg) per step.
//
// This is the reference's PartitionList algorithm (search.py:328-532:
// classes in priority order, each visited vertex x moves its unvisited
// neighbours y out of their class c into a new class placed immediately
// before c, neighbours handled in ascending id so every class stays sorted)
// re-expressed so one warp processes the 32 neighbours of a chunk at once:
//
//   slots     every class owns a segment [head, end) of a slot array holding
//             its members in tie order (ascending id; descending for the
//             DESCENDING rule).  A vertex that moves out is *not* removed:
//             its old slot simply becomes dead (cls[v] no longer names the
//             segment's class), so a split costs O(#moved), not O(|class|).
//             The class head pointer only moves forward past dead slots.
//   classes   doubly linked in label order (chead = largest label); ids are
//             recycled through a free list.
//   step i    pivot x = first live slot of the head class (a warp ballot
//             skips dead slots 32 at a time);
//             pass 1 over x's unvisited neighbours (chunks of 32 lanes):
//               __match_any_sync groups lanes by class, leaders accumulate
//               per-class move counts;
//             allocate: a class whose members all move keeps its place (the
//               "whole class moves in one hop" case, search.py:448-453);
//               otherwise a new class d with a fresh segment of exactly the
//               moved count is linked before c;
//             pass 2 places each mover at d.head + (running count of earlier
//               movers of c) -- the ascending-id order of the reference.
//   early exit once #classes == #unvisited (every class a singleton): the
//             rest of the order is the class list.
// parent[y] = x is recorded for every unvisited neighbour y of x, so after
// the search parent[y] is the last visited neighbour of y, i.e. the PEO
// parent (left neighbour with the greatest position, peo.py:106-121) -- except
// for vertices placed by the early exit, whose parent is left as -2 (unknown)
// for the PEO check to compute.
//
// All state is addressed through plain pointers: the batch kernel passes
// shared-memory arrays, the single-graph kernel global (L2-resident) ones.
#pragma once
#include "common.cuh"

namespace chordal {

template <typename I>
struct SlotMem {
    I *cls;       // [n]   class of vertex, VISITED once consumed
    I *slot_v;    // [cap] vertex stored in a slot
    I *c_head, *c_end;              // [n+2] segment bounds (slot indices < cap)
    I *c_live, *c_prev, *c_next;    // [n+2]
    I *c_tgt, *c_cnt;               // [n+2] per-step split target / mover count
    I *c_split;                     // [n+2] step that last touched the class
    I *freel;     // [n+2] free class ids
    I *touched;   // [n+2] classes touched in the current step
    I *scratch;   // [n]   compaction / neighbour staging buffer
    int32_t cap;  // slot capacity (>= 2n + 32: compaction leaves <= n live slots)
};

template <typename I>
struct SlotConst {
    static constexpr I NIL = (I)~(I)0;      // no class / no link
    static constexpr I VISITED = (I)~(I)0;
};

// Neighbour sources.  prepare(x, b, e) is warp-collective and yields the
// ascending neighbour list of x as entries [b, e) read back with get(e).
struct CsrSource {  // CSR rows in global memory
    const int64_t *indptr;
    const int32_t *indices;
    __device__ __forceinline__ void prepare(int x, int64_t &b, int64_t &e) const {
        b = __ldg(indptr + x);
        e = __ldg(indptr + x + 1);
    }
    __device__ __forceinline__ int get(int64_t e) const { return __ldg(indices + e); }
};

template <typename I>
struct BitsetSource {  // packed row of n <= 1024 bits (generic pointer: smem or global)
    const uint32_t *rows;
    int sw;      // row pitch in 32-bit words
    int words;   // ceil(n/32) <= 32
    I *nbuf;     // [n] staging of the compacted neighbour ids
    __device__ __forceinline__ void prepare(int x, int64_t &b, int64_t &e) const {
        const int lane = threadIdx.x & 31;
        uint32_t w = lane < words ? rows[x * sw + lane] : 0u;
        int c = __popc(w), incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(CH_FULL, incl, d);
            if (lane >= d) incl += o;
        }
        int at = incl - c;
        while (w) {
            int bit = __ffs(w) - 1;
            w &= w - 1;
            nbuf[at++] = (I)(32 * lane + bit);
        }
        b = 0;
        e = __shfl_sync(CH_FULL, incl, 31);
        __syncwarp();
    }
    __device__ __forceinline__ int get(int64_t e) const { return (int)nbuf[e]; }
};

namespace slot_detail {

template <typename I>
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Compacts the live members of every class (in class order) to the front of
// the slot array.  Runs when the bump pointer would overflow.  Live members
// are first gathered into scratch (size n) and then copied back, so segments
// of classes not yet visited are never overwritten.
template <typename I>
__device__ int compact(const SlotMem<I> &M, int chead, int lane) {
    int top = 0;
    for (int c = chead; c != (int)SlotConst<I>::NIL; c = (int)M.c_next[c]) {
        const int h = M.c_head[c], e = M.c_end[c];
        const int start = top;
        for (int s0 = h; s0 < e; s0 += 32) {
            int s = s0 + lane;
            bool live = false;
            int v = 0;
            if (s < e) {
                v = (int)M.slot_v[s];
                live = (int)M.cls[v] == c;
            }
            uint32_t m = __ballot_sync(CH_FULL, live);
            if (live) M.scratch[top + __popc(m & lanemask_lt<I>())] = (I)v;
            top += __popc(m);
        }
        __syncwarp();
        if (lane == 0) {
            M.c_head[c] = (I)start;
            M.c_end[c] = (I)top;
        }
    }
    __syncwarp();
    for (int t = lane; t < top; t += 32) M.slot_v[t] = M.scratch[t];
    __syncwarp();
    return top;
}

}  // namespace slot_detail

// One warp runs the whole search.  order[i], pos[v] (optional) and parent[v]
// (optional; (I)-1 for roots, (I)-2 when left to the PEO check) are written,
// in the engine's index type I.
// MODE: CHORDAL_TIE_ASCENDING / DESCENDING / SEEDED_ARB.
template <typename I, int MODE, typename Src>
__device__ void slot_lexbfs(const Src &src, int n, const SlotMem<I> &M, I *__restrict__ order, I *__restrict__ pos,
                            I *__restrict__ parent, uint64_t seed, uint64_t cell) {
    using C = SlotConst<I>;
    const int lane = threadIdx.x & 31;
    // ---- initial partition: one class, segment in tie order ------------------
    for (int v = lane; v < n; v += 32) {
        M.cls[v] = 0;
        int sv = v;
        if (MODE == CHORDAL_TIE_DESCENDING) sv = v == 0 ? 0 : n - v;  // [0, n-1, ..., 1]
        M.slot_v[v] = (I)sv;
        if (parent) parent[v] = (I)-1;
    }
    for (int c = lane; c < n + 1; c += 32) M.freel[c] = (I)(n - c);  // pop from the top -> 1, 2, ...
    if (lane == 0) {
        M.c_head[0] = (I)0;
        M.c_end[0] = (I)n;
        M.c_live[0] = (I)n;
        M.c_prev[0] = C::NIL;
        M.c_next[0] = C::NIL;
        M.c_split[0] = C::NIL;  // never equals a step index
    }
    __syncwarp();
    int chead = 0, nfree = n, top = n, nclasses = 1, nunv = n;
    const uint32_t lt = slot_detail::lanemask_lt<I>();

    for (int i = 0; i < n; ++i) {
        // ---- pivot: first live slot of the head class (or hash election) ----
        const int c0 = chead;
        int h = M.c_head[c0];
        const int e0 = M.c_end[c0];
        int xs = -1;
        if (MODE == CHORDAL_TIE_SEEDED_ARB && i > 0) {
            const uint64_t prefix = mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell);
            uint64_t best = 0;
            int bs = -1, bv = -1;
            for (int s0 = h; s0 < e0; s0 += 32) {
                int s = s0 + lane;
                if (s < e0) {
                    int v = (int)M.slot_v[s];
                    if ((int)M.cls[v] == c0) {
                        uint64_t k = splitmix64(prefix ^ (uint64_t)(v + 1));
                        if (bs < 0 || k > best || (k == best && v > bv)) { best = k; bs = s; bv = v; }
                    }
                }
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                uint64_t b2 = __shfl_xor_sync(CH_FULL, best, d);
                int s2 = __shfl_xor_sync(CH_FULL, bs, d), v2 = __shfl_xor_sync(CH_FULL, bv, d);
                if (s2 >= 0 && (bs < 0 || b2 > best || (b2 == best && v2 > bv))) { best = b2; bs = s2; bv = v2; }
            }
            xs = bs;
        } else {
            for (;; h += 32) {
                int s = h + lane;
                bool live = false;
                if (s < e0) live = (int)M.cls[(int)M.slot_v[s]] == c0;
                uint32_t m = __ballot_sync(CH_FULL, live);
                if (m) {
                    xs = h + __ffs(m) - 1;
                    break;
                }
            }
        }
        const int x = (int)M.slot_v[xs];
        __syncwarp();
        if (lane == 0) {
            if (MODE != CHORDAL_TIE_SEEDED_ARB || xs == (int)M.c_head[c0]) M.c_head[c0] = (I)(xs + 1);
            M.cls[x] = C::VISITED;
            order[i] = (I)x;
            if (pos) pos[x] = (I)i;
        }
        --nunv;
        const int live0 = (int)M.c_live[c0] - 1;
        if (live0 == 0) {  // unlink the emptied head class
            chead = (int)M.c_next[c0];
            if (lane == 0) {
                if (chead != (int)C::NIL) M.c_prev[chead] = C::NIL;
                M.freel[nfree] = (I)c0;
            }
            ++nfree;
            --nclasses;
        } else if (lane == 0) {
            M.c_live[c0] = (I)live0;
        }
        __syncwarp();
        if (nunv == 0) break;
        // ---- early exit: every class is a singleton ------------------------
        if (nclasses == nunv) {
            int k = i + 1;
            for (int c = chead; c != (int)C::NIL; c = (int)M.c_next[c], ++k) {
                int hh = M.c_head[c];
                int xs2 = -1;
                for (;; hh += 32) {
                    int s = hh + lane;
                    bool live = s < M.c_end[c] && (int)M.cls[(int)M.slot_v[s]] == c;
                    uint32_t m = __ballot_sync(CH_FULL, live);
                    if (m) {
                        xs2 = hh + __ffs(m) - 1;
                        break;
                    }
                }
                if (lane == 0) {
                    int v = (int)M.slot_v[xs2];
                    order[k] = (I)v;
                    if (pos) pos[v] = (I)k;
                    // the skipped steps would still have refreshed this vertex's
                    // parent: leave it to the PEO check (PARENT_UNKNOWN)
                    if (parent) parent[v] = (I)-2;
                    M.cls[v] = C::VISITED;
                }
            }
            __syncwarp();
            break;
        }
        // ---- pass 1: count movers per class ----------------------------------
        int64_t nb0, nb1;
        src.prepare(x, nb0, nb1);
        int ntouch = 0;
        for (int64_t e0c = nb0; e0c < nb1; e0c += 32) {
            int64_t e = (MODE == CHORDAL_TIE_DESCENDING) ? nb1 - 1 - (e0c - nb0) - lane : e0c + lane;
            bool ok = (MODE == CHORDAL_TIE_DESCENDING) ? e >= nb0 : e < nb1;
            int y = ok ? src.get(e) : 0;
            int c = ok ? (int)M.cls[y] : (int)C::VISITED;
            ok = ok && c != (int)C::VISITED;
            if (ok && parent) parent[y] = (I)x;
            uint32_t vm = __ballot_sync(CH_FULL, ok);
            uint32_t peers = __match_any_sync(CH_FULL, ok ? c : -1) & vm;
            bool leader = ok && (peers & lt) == 0;
            // first touch of a class in this step?
            bool fresh = leader && (int)M.c_split[c] != i;
            uint32_t fm = __ballot_sync(CH_FULL, fresh);
            if (fresh) {
                M.c_split[c] = (I)i;
                M.c_cnt[c] = (I)0;
                M.touched[ntouch + __popc(fm & lt)] = (I)c;
            }
            ntouch += __popc(fm);
            __syncwarp();
            if (leader) M.c_cnt[c] = (I)((int)M.c_cnt[c] + __popc(peers));
            __syncwarp();
        }
        if (ntouch == 0) continue;
        // ---- allocate new classes (lanes over touched classes) -----------------
        int need = 0;
        for (int t0 = 0; t0 < ntouch; t0 += 32) {
            int t = t0 + lane;
            int k = 0;
            if (t < ntouch) {
                int c = (int)M.touched[t];
                k = (int)M.c_cnt[c];
                if (k == (int)M.c_live[c]) k = 0;  // whole class moves: stays in place
            }
            need += __reduce_add_sync(CH_FULL, k);
        }
        if (top + need > M.cap) {
            top = slot_detail::compact<I>(M, chead, lane);
        }
        for (int t0 = 0; t0 < ntouch; t0 += 32) {
            int t = t0 + lane;
            int c = 0, k = 0;
            bool split = false;
            if (t < ntouch) {
                c = (int)M.touched[t];
                k = (int)M.c_cnt[c];
                split = k != (int)M.c_live[c];
            }
            uint32_t sm = __ballot_sync(CH_FULL, split);
            int rank = __popc(sm & lt);
            // segment offsets: exclusive prefix of k over splitting lanes
            int kk = split ? k : 0, incl = kk;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int o = __shfl_up_sync(CH_FULL, incl, d);
                if (lane >= d) incl += o;
            }
            if (t < ntouch) {
                if (split) {
                    const int d = (int)M.freel[nfree - 1 - rank];
                    const int start = top + incl - kk;
                    M.c_head[d] = (I)start;
                    M.c_end[d] = (I)(start + k);
                    M.c_live[d] = (I)k;
                    M.c_split[d] = (I)i;
                    M.c_cnt[d] = (I)0;
                    M.c_live[c] = (I)((int)M.c_live[c] - k);
                    M.c_tgt[c] = (I)d;
                    M.c_cnt[c] = (I)0;  // becomes the running rank of pass 2
                } else {
                    M.c_tgt[c] = (I)c;
                }
            }
            const int nsplit = __popc(sm);
            top += __shfl_sync(CH_FULL, incl, 31);
            nfree -= nsplit;
            nclasses += nsplit;
            __syncwarp();
            // link d before c (sequential over the splitting lanes keeps the
            // list consistent when neighbouring classes split together)
            for (uint32_t m = sm; m; m &= m - 1) {
                const int src_lane = __ffs(m) - 1;
                if (lane == src_lane) {
                    const int d = (int)M.c_tgt[c];
                    const int p = (int)M.c_prev[c];
                    M.c_prev[d] = (I)p;
                    M.c_next[d] = (I)c;
                    M.c_prev[c] = (I)d;
                    if (p != (int)C::NIL) M.c_next[p] = (I)d;
                }
                __syncwarp();
            }
            __syncwarp();
            // chead may have been split: the new class precedes it
            if (sm) {
                int ch = chead;
                if (M.c_prev[ch] != C::NIL) chead = (int)M.c_prev[ch];
            }
        }
        __syncwarp();
        // ---- pass 2: place the movers in ascending (tie) order -----------------
        for (int64_t e0c = nb0; e0c < nb1; e0c += 32) {
            int64_t e = (MODE == CHORDAL_TIE_DESCENDING) ? nb1 - 1 - (e0c - nb0) - lane : e0c + lane;
            bool ok = (MODE == CHORDAL_TIE_DESCENDING) ? e >= nb0 : e < nb1;
            int y = ok ? src.get(e) : 0;
            int c = ok ? (int)M.cls[y] : (int)C::VISITED;
            ok = ok && c != (int)C::VISITED;
            int d = ok ? (int)M.c_tgt[c] : 0;
            ok = ok && d != c;  // whole-class moves need no slot change
            uint32_t vm = __ballot_sync(CH_FULL, ok);
            uint32_t peers = __match_any_sync(CH_FULL, ok ? c : -1) & vm;
            if (ok) {
                int r = (int)M.c_cnt[c] + __popc(peers & lt);
                M.slot_v[(int)M.c_head[d] + r] = (I)y;
            }
            __syncwarp();
            if (ok) {
                M.cls[y] = (I)d;
                if ((peers & lt) == 0) M.c_cnt[c] = (I)((int)M.c_cnt[c] + __popc(peers));
            }
            __syncwarp();
        }
    }
}

}  // namespace chordal
