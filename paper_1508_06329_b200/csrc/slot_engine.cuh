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
//               per-class move counts (c_cnt == 0 marks an untouched class);
//             allocate: a class whose members all move keeps its place (the
//               "whole class moves in one hop" case, search.py:448-453);
//               otherwise a new class d with a fresh segment of exactly the
//               moved count is linked before c -- all splits of a step at
//               once (each insertion touches only its own cells);
//             pass 2 places each mover at d's next free slot -- chunk order is
//               ascending id, the reference's insertion order;
//             a pivot with <= 32 neighbours (one chunk) takes a fast step that
//               does both passes in registers (no per-class counters in memory).
//   early exit once #classes == #unvisited (every class a singleton): the
//             rest of the order is the class list.
// parent[y] = x is recorded for every unvisited neighbour y of x, so after
// the search parent[y] is the last visited neighbour of y, i.e. the PEO
// parent (left neighbour with the greatest position, peo.py:106-121) -- except
// for vertices placed by the early exit, whose parent is left as -2 (unknown)
// for the PEO check to compute.
//
// All state is addressed through plain pointers: the batch kernel passes
// shared-memory arrays, the single-graph kernels a mix of shared (the arrays
// touched per neighbour) and global ones.  I is the vertex/class index type,
// S the slot index type.
#pragma once
#include <type_traits>
#ifdef CHORDAL_SLOT_BOUNDS
#include <cstdio>
#endif

#include "common.cuh"
#include "philox.cuh"

namespace chordal {

// Bounds-checked build (-DCHORDAL_SLOT_BOUNDS, tools/bounds_check.sh): every
// subscript and pointer offset of the slot state is range-checked against its
// array length and traps with the array's name.  It stands in for
// compute-sanitizer memcheck, which this pool no longer runs; the product
// build compiles the fields as plain pointers.
#ifdef CHORDAL_SLOT_BOUNDS
template <typename T>
struct ChkPtr {
    T *p = nullptr;
    long long len = 0x7fffffffffffffffLL;  // unchecked until slot_set_bounds
    const char *name = "?";
    __host__ __device__ ChkPtr() {}
    __host__ __device__ ChkPtr(T *q) : p(q) {}
    __device__ __forceinline__ void check(long long i) const {
        if (i < 0 || i >= len) {
            printf("slot bounds: %s[%lld] outside [0, %lld) (block %d lane %d)\n", name, i, len, blockIdx.x,
                   threadIdx.x);
            __trap();
        }
    }
    template <typename J>
    __device__ __forceinline__ T &operator[](J i) const { check((long long)i); return p[i]; }
    template <typename J>
    __device__ __forceinline__ T *operator+(J i) const { check((long long)i); return p + i; }
    __host__ __device__ operator T *() const { return p; }
};
template <typename T>
using SlotPtr = ChkPtr<T>;
#else
template <typename T>
using SlotPtr = T *;
#endif

template <typename I, typename S>
struct SlotMem {
    SlotPtr<I> cls;                        // [n]   class of vertex, VISITED once consumed
    SlotPtr<I> slot_v;                     // [cap + kSlotPad] vertex stored in a slot (16-byte aligned)
    SlotPtr<S> c_head, c_end;              // [n+2] segment bounds (slot indices < cap)
    SlotPtr<I> c_live, c_prev, c_next;     // [n+2]
    SlotPtr<I> c_tgt;                      // [n+2] split target of a touched class
    SlotPtr<I> c_cnt;                      // [n+2] movers (pass 1) / next free slot - step base (pass 2); 0 between steps
    SlotPtr<I> freel;                      // [n+2] free class ids
    SlotPtr<I> touched;                    // [n+2] classes touched in the current step
    SlotPtr<I> scratch;                    // [n]   compaction buffer
    long long cap;                          // slot capacity (>= 2n + 32: compaction leaves <= n live slots)
};

// Array lengths for the checked build (no-op otherwise); pad = slot_v's tail
// beyond cap (slot_detail::kSlotPad).
template <typename I, typename S>
__device__ __forceinline__ void slot_set_bounds(SlotMem<I, S> &M, long long n, long long pad) {
#ifdef CHORDAL_SLOT_BOUNDS
    const long long nc = n + 2;
    M.cls.len = n; M.cls.name = "cls";
    M.slot_v.len = M.cap + pad; M.slot_v.name = "slot_v";
    M.c_head.len = nc; M.c_head.name = "c_head";
    M.c_end.len = nc; M.c_end.name = "c_end";
    M.c_live.len = nc; M.c_live.name = "c_live";
    M.c_prev.len = nc; M.c_prev.name = "c_prev";
    M.c_next.len = nc; M.c_next.name = "c_next";
    M.c_tgt.len = nc; M.c_tgt.name = "c_tgt";
    M.c_cnt.len = nc; M.c_cnt.name = "c_cnt";
    M.freel.len = nc; M.freel.name = "freel";
    M.touched.len = nc; M.touched.name = "touched";
    M.scratch.len = n; M.scratch.name = "scratch";
#else
    (void)M; (void)n; (void)pad;
#endif
}

template <typename I>
struct SlotConst {
    static constexpr I NIL = (I)~(I)0;  // no class / no link
    static constexpr I VISITED = (I)~(I)0;
};

// ---------------------------------------------------------------------------
// Neighbour source: bounds(x) gives the ascending list as entries [b, e);
// the engine walks it in blocks of at most capacity() entries, calling the
// warp-collective stage(lo, hi) before reading entries of [lo, hi) with get().

// CSR rows staged through a shared-memory buffer: each block of the pivot's
// list is fetched with one burst of independent loads (one memory round trip
// per block instead of one per 32-neighbour chunk).
template <typename T>
struct CsrStagedSource {
    const int64_t *indptr;
    const int32_t *indices;
    T *buf;      // shared memory, bufcap entries
    int bufcap;
    mutable int64_t base;
    __device__ __forceinline__ void bounds(int x, int64_t &b, int64_t &e) const {
        b = __ldg(indptr + x);
        e = __ldg(indptr + x + 1);
    }
    __device__ __forceinline__ int capacity() const { return bufcap; }
    __device__ __forceinline__ void stage(int64_t lo, int64_t hi) const {
        const int lane = threadIdx.x & 31;
        const int cnt = (int)(hi - lo);
        const int32_t *src = indices + lo;
        int k = lane;
        for (; k + 224 < cnt; k += 256) {
            int32_t a[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __ldg(src + k + 32 * j);
#pragma unroll
            for (int j = 0; j < 8; ++j) buf[k + 32 * j] = (T)a[j];
        }
        for (; k < cnt; k += 32) buf[k] = (T)__ldg(src + k);
        base = lo;
        __syncwarp();
    }
    __device__ __forceinline__ int get(int64_t e) const { return (int)buf[e - base]; }
    // one list entry straight from global memory (the <= 32-neighbour fast step)
    // (an L2 evict-first hint on these list loads measured slower: config 5
    // 1.88 -> 1.97 s)
    __device__ __forceinline__ int fetch(int64_t k) const { return __ldg(indices + k); }
    // Row bounds of a likely next pivot, issued where they stand (their values
    // are used a step later), and an L2 prefetch of the row itself once they
    // have arrived: the next step's row fetch then skips the indptr round trip
    // and finds the list in L2.
    __device__ __forceinline__ void bounds_issue(int v, int64_t &b, int64_t &e) const {
        asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(b) : "l"(indptr + v));
        asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(e) : "l"(indptr + v + 1));
    }
    __device__ __forceinline__ void prefetch_row(int64_t b, int64_t e) const {
        const int lane = threadIdx.x & 31;
        const int64_t k = b + 32 * (int64_t)lane;
        if (k < e) asm volatile("prefetch.global.L2 [%0];" ::"l"(indices + k));
    }
};

#ifdef SLOT_PROFILE
// lane-0 cycle counters (tools/slot_profile.cu only): [0] steps [1] pivot
// [2] bounds + pass 1 [3] allocate [4] pass 2 + restore [5] touched classes
// [6] steps with the pivot known ahead [7] steps with its row bounds fetched ahead
// [8] fast steps (<= 32 neighbours) [9] (unused)
__device__ unsigned long long slot_prof[16];
#define SLOT_T(k)                                           \
    do {                                                    \
        const long long _c = clock64();                     \
        slot_acc[k] += (unsigned long long)(_c - slot_t0);  \
        slot_t0 = _c;                                       \
    } while (0)
#else
#define SLOT_T(k) \
    do {          \
    } while (0)
#endif

namespace slot_detail {

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Visits x's neighbour list in tie order (ascending; descending for the
// DESCENDING rule) as chunks of 32 lanes: fn(valid, y).
template <int MODE, typename Src, typename Fn>
__device__ __forceinline__ void for_each_chunk(const Src &src, int64_t b, int64_t e, Fn &&fn) {
    const int lane = threadIdx.x & 31;
    const int64_t cap = src.capacity();
    int chunk = 0;
    if (MODE == CHORDAL_TIE_DESCENDING) {
        for (int64_t hi = e; hi > b; hi -= cap) {
            const int64_t lo = hi - cap > b ? hi - cap : b;
            src.stage(lo, hi);
            for (int64_t c0 = hi; c0 > lo; c0 -= 32, ++chunk) {
                const int64_t k = c0 - 1 - lane;
                const bool ok = k >= lo;
                fn(ok, ok ? src.get(k) : 0, chunk);
            }
        }
    } else {
        for (int64_t lo = b; lo < e; lo += cap) {
            const int64_t hi = lo + cap < e ? lo + cap : e;
            src.stage(lo, hi);
            for (int64_t c0 = lo; c0 < hi; c0 += 32, ++chunk) {
                const int64_t k = c0 + lane;
                const bool ok = k < hi;
                fn(ok, ok ? src.get(k) : 0, chunk);
            }
        }
    }
}

// First live slot of class c in [h, e): each lane tests V = 16/sizeof(I)
// consecutive slots fetched with one 16-byte load, so a warp skips 32*V dead
// slots per memory round trip.  The slot array is padded by kSlotPad entries
// and 16-byte aligned, so the over-read past e stays inside the allocation.
constexpr int kSlotPad = 256;  // >= 32 * V for V = 8 (u16) and 4 (int32); 32 * 8 int32 for a 32-byte window
template <typename I, typename S>
__device__ __forceinline__ long long first_live(const SlotMem<I, S> &M, int c, long long h, long long e,
                                               int *vert = nullptr) {
    constexpr int V = 16 / sizeof(I);
    const int lane = threadIdx.x & 31;
    for (long long base = h & ~(long long)(V - 1);; base += 32 * V) {
        const long long s0 = base + (long long)lane * V;
        const uint4 raw = *reinterpret_cast<const uint4 *>(M.slot_v + s0);
        const I *vals = reinterpret_cast<const I *>(&raw);
        int first = V, v1 = -1;
#pragma unroll
        for (int j = V - 1; j >= 0; --j) {
            const long long s = s0 + j;
            if (s >= h && s < e && (int)M.cls[(int)vals[j]] == c) {
                first = j;
                v1 = (int)vals[j];
            }
        }
        const uint32_t m = __ballot_sync(CH_FULL, first < V);
        if (m) {
            const int src = __ffs(m) - 1;
            if (vert) *vert = __shfl_sync(CH_FULL, v1, src);
            return base + (long long)src * V + __shfl_sync(CH_FULL, first, src);
        }
    }
}

// Compacts the live members of every class (in class order) to the front of
// the slot array.  Runs when the bump pointer would overflow.  Live members
// are first gathered into scratch (size n) and then copied back, so segments
// of classes not yet visited are never overwritten.
template <typename I, typename S>
__device__ long long compact(const SlotMem<I, S> &M, int chead, int lane) {
    long long top = 0;
    for (int c = chead; c != (int)SlotConst<I>::NIL; c = (int)M.c_next[c]) {
        const long long h = (long long)M.c_head[c], e = (long long)M.c_end[c];
        const long long start = top;
        for (long long s0 = h; s0 < e; s0 += 32) {
            const long long s = s0 + lane;
            bool live = false;
            int v = 0;
            if (s < e) {
                v = (int)M.slot_v[s];
                live = (int)M.cls[v] == c;
            }
            uint32_t m = __ballot_sync(CH_FULL, live);
            if (live) M.scratch[top + __popc(m & lanemask_lt())] = (I)v;
            top += __popc(m);
        }
        __syncwarp();
        if (lane == 0) {
            M.c_head[c] = (S)start;
            M.c_end[c] = (S)top;
        }
    }
    __syncwarp();
    for (long long t = lane; t < top; t += 32) M.slot_v[t] = M.scratch[t];
    __syncwarp();
    return top;
}

}  // namespace slot_detail

// One warp runs the whole search.  order[i], pos[v] (optional) and parent[v]
// (optional; (O)-1 for roots, (O)-2 when left to the PEO check) are written
// in the output type O.  MODE: CHORDAL_TIE_ASCENDING / DESCENDING / SEEDED_ARB.
template <typename I, typename S, int MODE, typename Src, typename O>
__device__ void slot_lexbfs(const Src &src, int n, const SlotMem<I, S> &M, O *__restrict__ order, O *__restrict__ pos,
                            O *__restrict__ parent, uint64_t seed, uint64_t cell,
                            volatile int *progress = nullptr) {
    using C = SlotConst<I>;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = slot_detail::lanemask_lt();
    // ---- initial partition: one class, segment in tie order ------------------
    for (int v = lane; v < n; v += 32) {
        M.cls[v] = 0;
        int sv = v;
        if (MODE == CHORDAL_TIE_DESCENDING) sv = v == 0 ? 0 : n - v;  // [0, n-1, ..., 1]
        M.slot_v[v] = (I)sv;
        if (parent) parent[v] = (O)-1;
    }
    for (int c = lane; c < n + 1; c += 32) M.freel[c] = (I)(n - c);  // pop from the top -> 1, 2, ...
    for (int c = lane; c < n + 2; c += 32) M.c_cnt[c] = (I)0;       // "untouched" outside a step
    if (lane == 0) {
        M.c_head[0] = (S)0;
        M.c_end[0] = (S)n;
        M.c_live[0] = (I)n;
        M.c_prev[0] = C::NIL;
        M.c_next[0] = C::NIL;
    }
    __syncwarp();
    if (MODE == CHORDAL_TIE_SEEDED_PARTITION) {
        // lexbfs_partition(seeded, method="linked") (search.py:515-518): the one
        // initial class holds range(n) shuffled by Generator.shuffle -- Fisher-
        // Yates with random_interval (masked rejection on next_uint32), i = n-1..1,
        // on the stream keyed by `seed` (= mix64(seed, crc32("lexbfs-partition"))).
        if (lane == 0) {
            PhiloxStream rs(seed);
            for (int i2 = n - 1; i2 >= 1; --i2) {
                uint32_t mask = (uint32_t)i2;
                mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
                uint32_t j;
                while ((j = rs.next32() & mask) > (uint32_t)i2) {
                }
                const I t = M.slot_v[i2];
                M.slot_v[i2] = M.slot_v[j];
                M.slot_v[j] = t;
            }
        }
        __syncwarp();
    }
    // lexbfs_labels(seeded, method="linked") (search.py:285-290): the pivot is
    // member Generator.integers(|C|) of the max-label class C, members in chain
    // order (= ascending id here); every lane keeps the same stream.
    PhiloxStream lab(seed);
    int chead = 0, nfree = n, nclasses = 1, nunv = n;
    long long top = n;
    int gv = -1;  // vertex whose row bounds (gb0, gb1) were fetched ahead
    int64_t gb0 = 0, gb1 = 0;
    // Next-pivot tracking (ascending / descending / seeded-partition ties): the
    // next pivot is the first live member of the head class after the step,
    // i.e. the head class's next live slot after x -- unless the step gives the
    // head class a new segment, when it is the head class's first mover in tie
    // order.  Both are known by the end of the step, so the next step skips the
    // first-live scan; -1 = unknown (fall back to the scan).
    constexpr bool kTrack = MODE == CHORDAL_TIE_ASCENDING || MODE == CHORDAL_TIE_DESCENDING ||
                            MODE == CHORDAL_TIE_SEEDED_PARTITION;
    constexpr int V = 16 / sizeof(I);
#ifndef SLOT_WIN_BYTES
#define SLOT_WIN_BYTES 16
#endif
    // the int32 form's next-pivot window: VW slots per lane (16 bytes; 8 bytes
    // measured 1.466 -> 1.517 s on configuration 5, 32 bytes 1.578 s)
    constexpr int VW = SLOT_WIN_BYTES / sizeof(I);
    struct alignas(16) Win32 { uint4 a, b; };
    using WinT = typename std::conditional<SLOT_WIN_BYTES == 32, Win32,
                                           typename std::conditional<SLOT_WIN_BYTES == 16, uint4, uint2>::type>::type;
    constexpr bool kProbeWin = sizeof(I) == 2;  // next-pivot candidates: 32-slot probe (u16) or wide window
    int nx = -1;
    long long nxs = -1;

#ifdef SLOT_PROFILE
    unsigned long long slot_acc[16] = {0};
    long long slot_t0 = clock64();
#endif
    for (int i = 0; i < n; ++i) {
#ifdef SLOT_PROFILE
        slot_acc[0]++;
        slot_t0 = clock64();
#endif
        // The pivot known with its row bounds and <= 32 neighbours: its list is
        // fetched first, so that round trip overlaps the head-class reads below
        // (config 5: 1.98 -> 1.94 s).
        constexpr bool kFast = MODE == CHORDAL_TIE_ASCENDING || MODE == CHORDAL_TIE_DESCENDING;
        const bool pre = kFast && nx >= 0 && nx == gv && gb1 - gb0 <= 32;
#ifdef SLOT_PROFILE
        if (__any_sync(CH_FULL, pre)) slot_acc[9] += clock64() - slot_t0;  // wait for the row bounds
#endif
        int ypre = 0;
        if (pre && lane < (int)(gb1 - gb0))
            ypre = src.fetch(MODE == CHORDAL_TIE_DESCENDING ? gb1 - 1 - lane : gb0 + lane);
        // ---- pivot: first live slot of the head class (or hash election) ----
        const int c0 = chead;
        if (progress && lane == 0 && (i & 3) == 0) {  // for the look-ahead warp (slot_lookahead): head class, step
            progress[0] = c0;
            progress[2] = i;
        }
        const long long e0 = (long long)M.c_end[c0];
        const int live_c0 = (int)M.c_live[c0], next_c0 = (int)M.c_next[c0];  // one round trip
        long long xs = -1;
        int x = -1;
#ifdef SLOT_PROFILE
        if (kTrack && nx >= 0) slot_acc[6]++;
        if (kTrack && nx >= 0 && nx == gv) slot_acc[7]++;
#endif
        if (kTrack && nx >= 0) {
            xs = nxs;
            x = nx;
        } else if (MODE == CHORDAL_TIE_SEEDED_ARB && i > 0) {
            const long long h = (long long)M.c_head[c0];
            const uint64_t prefix = mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell);
            uint64_t best = 0;
            long long bs = -1;
            int bv = -1;
            for (long long s0 = h; s0 < e0; s0 += 32) {
                const long long s = s0 + lane;
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
                long long s2 = __shfl_xor_sync(CH_FULL, bs, d);
                int v2 = __shfl_xor_sync(CH_FULL, bv, d);
                if (s2 >= 0 && (bs < 0 || b2 > best || (b2 == best && v2 > bv))) { best = b2; bs = s2; bv = v2; }
            }
            xs = bs;
        } else if (MODE == CHORDAL_TIE_SEEDED_LABELS) {
            const long long h = (long long)M.c_head[c0];
            int rem = (int)lab.bounded(0, (uint64_t)((int)M.c_live[c0] - 1));
            for (long long s0 = h;; s0 += 32) {
                const long long s = s0 + lane;
                const bool live = s < e0 && (int)M.cls[(int)M.slot_v[s]] == c0;
                const uint32_t bm = __ballot_sync(CH_FULL, live);
                const int c = __popc(bm);
                if (rem < c) {
                    xs = s0 + (long long)__fns(bm, 0, rem + 1);
                    break;
                }
                rem -= c;
            }
        } else {
            xs = slot_detail::first_live<I, S>(M, c0, (long long)M.c_head[c0], e0, &x);
        }
        if (x < 0) x = (int)M.slot_v[xs];
        // the 32 slots after x (bounded by x's segment later): candidates for
        // the next pivot, and their classes (slots below `top` all hold vertices)
        // (u16 state -- shared memory -- probes 32 slots, one per lane; int32
        // state in global memory reads a 32 * V-slot window with 16-byte loads:
        // its classes are fragmented by dead slots, and the probe measured
        // slower there: configuration 5 1.46 -> 1.65 s, CSR n = 8192 8.38 ->
        // 7.21 ms with it)
        int pA = -1, pclA = -1;
        if (kTrack && kProbeWin && xs + 1 + lane < top) {
            pA = (int)M.slot_v[xs + 1 + lane];
            pclA = (int)M.cls[pA];
        }
        const long long cand_base = (xs + 1) & ~(long long)(VW - 1);
        WinT cand_raw{};
        if (kTrack && !kProbeWin) cand_raw = *reinterpret_cast<const WinT *>(M.slot_v + cand_base + (long long)lane * VW);
        __syncwarp();
        if (lane == 0) {
            if ((MODE != CHORDAL_TIE_SEEDED_ARB && MODE != CHORDAL_TIE_SEEDED_LABELS) || xs == (long long)M.c_head[c0])
                M.c_head[c0] = (S)(xs + 1);
            M.cls[x] = C::VISITED;
            order[i] = (O)x;
            if (pos) pos[x] = (O)i;
        }
        --nunv;
        const int live0 = live_c0 - 1;
        if (live0 == 0) {  // unlink the emptied head class
            chead = next_c0;
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
                const long long xs2 = slot_detail::first_live<I, S>(M, c, (long long)M.c_head[c],
                                                                   (long long)M.c_end[c]);
                __syncwarp();  // every lane's cls[] reads in first_live precede lane 0's write
                if (lane == 0) {
                    int v = (int)M.slot_v[xs2];
                    order[k] = (O)v;
                    if (pos) pos[v] = (O)k;
                    // the skipped steps would still have refreshed this vertex's
                    // parent: leave it to the PEO check (unknown = -2)
                    if (parent) parent[v] = (O)-2;
                    M.cls[v] = C::VISITED;
                }
                __syncwarp();  // the next class's first_live reads cls[] after this write
            }
            __syncwarp();
            break;
        }
        SLOT_T(1);
        // ---- pass 1: count movers per class ----------------------------------
        int64_t nb0, nb1;
        if (x == gv) {  // bounds fetched a step ago
            nb0 = gb0;
            nb1 = gb1;
        } else {
            src.bounds(x, nb0, nb1);
        }
        const int hc = chead;  // head class before this step's splits
        // The next-pivot candidates: the head class after x's removal -- x's
        // class (the 32 slots after x, read with x) or, when x emptied it, the
        // next class (the first 32 slots of its segment) -- with their classes,
        // read once for the fast step and the general path.
        const bool alt = hc != c0 && hc != (int)C::NIL;  // head class after x: not x's class
        long long wlo = xs + 1, whi = e0;
        int pv = pA, pcl = xs + 1 + lane < e0 ? pclA : -1;
        if (kTrack && kProbeWin && alt) {
            wlo = (long long)M.c_head[hc];
            whi = (long long)M.c_end[hc];
            pv = pcl = -1;
            if (wlo + lane < whi) {
                pv = (int)M.slot_v[wlo + lane];
                pcl = (int)M.cls[pv];
            }
        }
        // the head class's first live slot (its classes as read before this
        // step's moves: a head class that loses members to a split gets a new
        // segment and its first mover is the next pivot instead)
        auto window_probe = [&](int &gv_out, long long &gs_out) {
            gv_out = -1;
            gs_out = -1;
            const uint32_t gm = __ballot_sync(CH_FULL, pcl == hc);
            if (gm) {
                const int src_l = __ffs(gm) - 1;
                gv_out = __shfl_sync(CH_FULL, pv, src_l);
                gs_out = wlo + src_l;
                return;
            }
            // none of the first 32 is live: the 32 * V slots behind them
            const long long wb = (wlo + 32) & ~(long long)(V - 1), l0 = wb + (long long)lane * V;
            const uint4 raw = *reinterpret_cast<const uint4 *>(M.slot_v + l0);
            const int rlo = (int)(wlo - l0 < 0 ? 0 : (wlo - l0 > V ? V : wlo - l0));
            const int rhi = (int)(whi - l0 < 0 ? 0 : (whi - l0 > V ? V : whi - l0));
            const I *cv = reinterpret_cast<const I *>(&raw);
            int fj = V, fv = -1;
#pragma unroll
            for (int j = V - 1; j >= 0; --j)
                if (j >= rlo && j < rhi && (int)M.cls[(int)cv[j]] == hc) {
                    fj = j;
                    fv = (int)cv[j];
                }
            const uint32_t gm2 = __ballot_sync(CH_FULL, fj < V);
            if (gm2) {
                const int src_l = __ffs(gm2) - 1;
                gv_out = __shfl_sync(CH_FULL, fv, src_l);
                gs_out = wb + (long long)src_l * V + __shfl_sync(CH_FULL, fj, src_l);
            }
        };
        // int32 state: the same candidates as a 32 * V-slot window (16-byte
        // loads), bounds lane-relative so each slot costs 32-bit compares only.
        long long wb = cand_base, wlo2 = xs + 1, whi2 = e0;
        WinT wraw = cand_raw;
        if (kTrack && !kProbeWin && alt) {
            wlo2 = (long long)M.c_head[hc];
            whi2 = (long long)M.c_end[hc];
            wb = wlo2 & ~(long long)(VW - 1);
            wraw = *reinterpret_cast<const WinT *>(M.slot_v + wb + (long long)lane * VW);
        }
        int wcl[VW];  // class of each window slot inside [wlo, whi), else -1
        if (kTrack && !kProbeWin) {
            const long long l0 = wb + (long long)lane * VW;
            const int rlo = (int)(wlo2 - l0 < 0 ? 0 : (wlo2 - l0 > VW ? VW : wlo2 - l0));
            const int rhi = (int)(whi2 - l0 < 0 ? 0 : (whi2 - l0 > VW ? VW : whi2 - l0));
            const I *cv = reinterpret_cast<const I *>(&wraw);
#pragma unroll
            for (int j = 0; j < VW; ++j) wcl[j] = (j >= rlo && j < rhi) ? (int)M.cls[(int)cv[j]] : -1;
        }
        // the head class's first live slot in the window (its classes as read
        // before this step's moves: a head class that loses members to a split
        // gets a new segment and its first mover is the next pivot instead)
        auto window_wide = [&](int &gv_out, long long &gs_out) {
            const I *cv = reinterpret_cast<const I *>(&wraw);
            int fj = VW, fv = -1;
#pragma unroll
            for (int j = VW - 1; j >= 0; --j)
                if (wcl[j] == hc) {
                    fj = j;
                    fv = (int)cv[j];
                }
            const uint32_t gm = __ballot_sync(CH_FULL, fj < VW);
            gv_out = -1;
            gs_out = -1;
            if (gm) {
                const int src_l = __ffs(gm) - 1;
                gv_out = __shfl_sync(CH_FULL, fv, src_l);
                gs_out = wb + (long long)src_l * VW + __shfl_sync(CH_FULL, fj, src_l);
            }
        };
        auto window_first = [&](int &gv_out, long long &gs_out) {
            if constexpr (kProbeWin)
                window_probe(gv_out, gs_out);
            else
                window_wide(gv_out, gs_out);
        };
        // ---- fast step: at most 32 neighbours (97 % of the configuration-5 steps) --
        // One chunk holds every mover of the step, so a class's group in the
        // chunk is its whole move set: counts come from __match_any_sync, each
        // leader reads its class's fields once, the new segments are laid out
        // in registers -- no c_cnt / touched round trips and no restore pass.
        // When x's class emptied, the new head class's first live slot is
        // fetched too, so the next pivot stays known.
        if constexpr (kFast) {
            if (nb1 - nb0 <= 32 && top + 32 <= M.cap) {
#ifdef SLOT_PROFILE
                slot_acc[8]++;
#endif
                const int deg = (int)(nb1 - nb0);
                const int y = pre ? ypre
                                  : (lane < deg ? src.fetch(MODE == CHORDAL_TIE_DESCENDING ? nb1 - 1 - lane : nb0 + lane) : 0);
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)y) != 0xFFFFFFFFu) slot_acc[10] += clock64() - slot_t0;  // list
#endif
                const int frl = nfree - 1 - lane >= 0 ? (int)M.freel[nfree - 1 - lane] : 0;
                const int c = lane < deg ? (int)M.cls[y] : (int)C::VISITED;
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)c) != 0xFFFFFFFEu) slot_acc[11] += clock64() - slot_t0;  // classes
#endif
                const bool ok = c != (int)C::VISITED;
                // every mover reads its class's fields (same address within a
                // group: one broadcast), so the reads do not wait for the grouping
#ifndef SLOT_LEADER_FIELDS
                int live_c = 0, pold = 0;
                if (ok) {
                    live_c = (int)M.c_live[c];
                    pold = (int)M.c_prev[c];
                }
#endif
                if (ok && parent) parent[y] = (O)x;
                const uint32_t vm = __ballot_sync(CH_FULL, ok);
                if (vm == 0) {  // no unvisited neighbour: nothing moves, only the next pivot
                    int guess;
                    long long gslot;
                    window_first(guess, gslot);
                    nx = guess;
                    nxs = gslot;
                    if (nx >= 0 && nx != gv) {
                        src.bounds_issue(nx, gb0, gb1);
                        gv = nx;
                    }
                    __syncwarp();
                    SLOT_T(2);
                    continue;
                }
                const uint32_t peers = __match_any_sync(CH_FULL, ok ? c : -1) & vm;
                const bool leader = ok && (peers & lt) == 0;
                const int cnt = __popc(peers);
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)(cnt)) != 0xFFFFFFF3u) slot_acc[12] += clock64() - slot_t0;
#endif
#ifdef SLOT_LEADER_FIELDS
                int live_c = 0, pold = 0;
                if (leader) {
                    live_c = (int)M.c_live[c];
                    pold = (int)M.c_prev[c];
                }
#endif
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)(live_c + pold)) != 0xFFFFFFF3u) slot_acc[13] += clock64() - slot_t0;
#endif
                int hmv = ok && c == hc ? y : (MODE == CHORDAL_TIE_DESCENDING ? -1 : 0x7FFFFFFF);
                const int hmf = MODE == CHORDAL_TIE_DESCENDING ? __reduce_max_sync(CH_FULL, hmv)
                                                               : (int)__reduce_min_sync(CH_FULL, (unsigned)hmv);
                // next pivot if the head class keeps its segment
                int guess = -1;
                long long gslot = -1;
                window_first(guess, gslot);
                // new classes: one per split group, segments laid out in lane order
                const bool split = leader && cnt != live_c;
                const uint32_t sm = __ballot_sync(CH_FULL, split);
                if (sm == 0) {  // only whole classes move (they keep their place): the next pivot only
                    nx = guess;
                    nxs = gslot;
                    if (nx >= 0 && nx != gv) {
                        src.bounds_issue(nx, gb0, gb1);
                        gv = nx;
                    }
                    __syncwarp();
                    SLOT_T(2);
                    continue;
                }
                const int d = __shfl_sync(CH_FULL, frl, __popc(sm & lt));
                const int kk = split ? cnt : 0;
#ifndef SLOT_SCAN_SHFL
                // segment offsets: kk <= 32, so six independent bit-plane ballots
                // give the exclusive prefix and the total (a shorter chain than a
                // five-round shuffle scan)
                int excl = 0, ktot = 0;
                if ((sm & (sm - 1)) == 0) {  // at most one class splits (most steps): no scan
                    ktot = sm ? __shfl_sync(CH_FULL, kk, __ffs(sm) - 1) : 0;
                } else {
#pragma unroll
                    for (int bit = 0; bit < 6; ++bit) {
                        const uint32_t bm = __ballot_sync(CH_FULL, (kk >> bit) & 1);
                        excl += __popc(bm & lt) << bit;
                        ktot += __popc(bm) << bit;
                    }
                }
                const int incl = excl + kk;
#else
                int incl = kk;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const int o = __shfl_up_sync(CH_FULL, incl, dd);
                    if (lane >= dd) incl += o;
                }
                const int ktot = __shfl_sync(CH_FULL, incl, 31);
#endif
                const int start = (int)top + incl - kk;
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)(start)) != 0xFFFFFFF3u) slot_acc[14] += clock64() - slot_t0;
#endif
                if (split) {
                    M.c_head[d] = (S)start;
                    M.c_end[d] = (S)(start + cnt);
                    M.c_live[d] = (I)cnt;
                    M.c_cnt[d] = (I)0;
                    M.c_live[c] = (I)(live_c - cnt);
                    // link d before c (pold read above, before any link write)
                    M.c_prev[d] = (I)pold;
                    M.c_next[d] = (I)c;
                    M.c_prev[c] = (I)d;
                    if (pold != (int)C::NIL) M.c_next[pold] = (I)d;
                }
                int hstart = -1;
                const uint32_t hb = __ballot_sync(CH_FULL, split && c == hc);
                if (hb) {  // the head class split: its movers' class is the new head
                    const int src_l = __ffs(hb) - 1;
                    chead = __shfl_sync(CH_FULL, d, src_l);
                    hstart = __shfl_sync(CH_FULL, start, src_l);
                }
                top += ktot;
                nfree -= __popc(sm);
#ifdef SLOT_PROFILE
                if (__reduce_or_sync(CH_FULL, (unsigned)(top + nfree)) != 0xFFFFFFF3u) slot_acc[15] += clock64() - slot_t0;
#endif
                nclasses += __popc(sm);
                // movers of split classes into their new segment, in lane (tie) order
                const int ls = ok ? __ffs(peers) - 1 : 0;
                const int dl = __shfl_sync(CH_FULL, d, ls);
                const int stl = __shfl_sync(CH_FULL, start, ls);
                __syncwarp();  // the candidate-class reads above precede these writes (racecheck)
                if (ok && ((sm >> ls) & 1u)) {
                    M.slot_v[stl + __popc(peers & lt)] = (I)y;
                    M.cls[y] = (I)dl;
                }
                nx = hstart >= 0 ? hmf : guess;
                nxs = hstart >= 0 ? hstart : gslot;
                if (nx >= 0 && nx != gv) {  // issuing these earlier (on the window guess) or adding an
                    src.bounds_issue(nx, gb0, gb1);  // L2 prefetch of the row measured slower
                    gv = nx;
                }
                __syncwarp();
                SLOT_T(2);
                continue;
            }
        }
        int ntouch = 0;
        int hm = MODE == CHORDAL_TIE_DESCENDING ? -1 : 0x7FFFFFFF;  // first mover of hc in tie order
        int cls_c0 = (int)C::VISITED;  // the first chunk's classes, reused by pass 2
        slot_detail::for_each_chunk<MODE>(src, nb0, nb1, [&](bool ok, int y, int chunk) {
            int c = ok ? (int)M.cls[y] : (int)C::VISITED;
            if (chunk == 0) cls_c0 = c;
            ok = ok && c != (int)C::VISITED;
            if (kTrack && ok && c == hc) hm = MODE == CHORDAL_TIE_DESCENDING ? max(hm, y) : min(hm, y);
            if (ok && parent) parent[y] = (O)x;
            const uint32_t vm = __ballot_sync(CH_FULL, ok);
            const uint32_t peers = __match_any_sync(CH_FULL, ok ? c : -1) & vm;
            const bool leader = ok && (peers & lt) == 0;
            const int old = leader ? (int)M.c_cnt[c] : 0;
            const bool fresh = leader && old == 0;  // first touch in this step
            const uint32_t fm = __ballot_sync(CH_FULL, fresh);
            if (fresh) M.touched[ntouch + __popc(fm & lt)] = (I)c;
            ntouch += __popc(fm);
            if (leader) M.c_cnt[c] = (I)(old + __popc(peers));
            __syncwarp();
        });
        // next pivot if the head class keeps its segment: its next live slot in the window
        int guess = -1;
        long long gslot = -1;
        if (kTrack) {
            window_first(guess, gslot);
            hm = MODE == CHORDAL_TIE_DESCENDING ? __reduce_max_sync(CH_FULL, hm)
                                                : (int)__reduce_min_sync(CH_FULL, (unsigned)hm);
        }
        SLOT_T(2);
#ifdef SLOT_PROFILE
        slot_acc[5] += ntouch;
#endif
        if (ntouch == 0) {
            nx = guess;
            nxs = gslot;
            if (nx >= 0 && nx != gv) {
                src.bounds_issue(nx, gb0, gb1);
                gv = nx;
            }
            continue;
        }
        // ---- allocate new classes (lanes over touched classes) -----------------
        if (top + (nb1 - nb0) > M.cap) {  // the movers need at most deg(x) slots
            int need = 0;
            for (int t0 = 0; t0 < ntouch; t0 += 32) {
                const int t = t0 + lane;
                int k = 0;
                if (t < ntouch) {
                    const int c = (int)M.touched[t];
                    k = (int)M.c_cnt[c];
                    if (k == (int)M.c_live[c] && MODE != CHORDAL_TIE_SEEDED_PARTITION) k = 0;  // whole class moves: stays in place
                }
                need += __reduce_add_sync(CH_FULL, k);
            }
            if (top + need > M.cap) {
                top = slot_detail::compact<I, S>(M, chead, lane);
                gslot = -1;  // slots moved: the guess's slot is stale
                guess = -1;
            }
        }
        const long long top0 = top;  // pass 2 slots are top0 + c_cnt[c] + rank
        long long hstart = -1;        // first slot of the segment hc's movers go to, if any
        for (int t0 = 0; t0 < ntouch; t0 += 32) {
            const int t = t0 + lane;
            int c = 0, k = 0;
            bool split = false, resort = false;
            if (t < ntouch) {
                c = (int)M.touched[t];
                k = (int)M.c_cnt[c];
                split = k != (int)M.c_live[c];
                // PartitionList moves every member, so a class whose members all
                // move is re-ordered by adjacency (search.py:440-463); with the
                // seeded initial shuffle that order differs from the slot order
                resort = !split && MODE == CHORDAL_TIE_SEEDED_PARTITION;
            }
            const uint32_t sm = __ballot_sync(CH_FULL, split);
            const int rank = __popc(sm & lt);
            // segment offsets: inclusive prefix of k over the splitting (and re-sorted) lanes
            const int kk = (split || resort) ? k : 0;
            int incl = kk;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int o = __shfl_up_sync(CH_FULL, incl, d);
                if (lane >= d) incl += o;
            }
            int pold = 0;
            if (split) {
                const int d = (int)M.freel[nfree - 1 - rank];
                const long long start = top + incl - kk;
                M.c_head[d] = (S)start;
                M.c_end[d] = (S)(start + k);
                M.c_live[d] = (I)k;
                M.c_cnt[d] = (I)0;
                M.c_live[c] = (I)((int)M.c_live[c] - k);
                M.c_tgt[c] = (I)d;
                M.c_cnt[c] = (I)(start - top0);  // pass 2: next free slot of the new segment
                pold = (int)M.c_prev[c];
            } else if (resort) {
                const long long start = top + incl - kk;
                M.c_head[c] = (S)start;
                M.c_end[c] = (S)(start + k);
                M.c_tgt[c] = (I)c;
                M.c_cnt[c] = (I)(start - top0);
            } else if (t < ntouch) {
                M.c_tgt[c] = (I)c;
            }
            if (kTrack) {  // did hc get a new segment?
                const uint32_t hb = __ballot_sync(CH_FULL, (split || resort) && c == hc);
                if (hb) hstart = __shfl_sync(CH_FULL, top + incl - kk, __ffs(hb) - 1);
            }
            const int nsplit = __popc(sm);
            top += __shfl_sync(CH_FULL, incl, 31);
            nfree -= nsplit;
            nclasses += nsplit;
            __syncwarp();
            // link d before c, all splitting lanes at once: inserting d before
            // c reads only c.prev and writes d.prev, d.next, c.prev and
            // (old c.prev).next -- disjoint cells for distinct c, and no
            // insertion writes another class's .prev, so concurrent inserts
            // (even of adjacent classes) leave a consistent list.
            if (split) {
                const int d = (int)M.c_tgt[c];
                M.c_prev[d] = (I)pold;
                M.c_next[d] = (I)c;
                M.c_prev[c] = (I)d;
                if (pold != (int)C::NIL) M.c_next[pold] = (I)d;
            }
            __syncwarp();
            // chead may have been split: the new class precedes it
            if (sm && M.c_prev[chead] != C::NIL) chead = (int)M.c_prev[chead];
        }
        __syncwarp();
        if (kTrack) {
            nx = hstart >= 0 ? hm : guess;
            nxs = hstart >= 0 ? hstart : gslot;
            if (nx >= 0 && nx != gv) {  // its row bounds arrive during pass 2
                src.bounds_issue(nx, gb0, gb1);
                gv = nx;
            }
        }
        SLOT_T(3);
        // ---- pass 2: place the movers in ascending (tie) order -----------------
        slot_detail::for_each_chunk<MODE>(src, nb0, nb1, [&](bool ok, int y, int chunk) {
            int c = chunk == 0 ? cls_c0 : (ok ? (int)M.cls[y] : (int)C::VISITED);
            ok = ok && c != (int)C::VISITED;
            const int d = ok ? (int)M.c_tgt[c] : 0;
            if (MODE != CHORDAL_TIE_SEEDED_PARTITION) ok = ok && d != c;  // whole-class moves need no slot change
            const uint32_t vm = __ballot_sync(CH_FULL, ok);
            const uint32_t peers = __match_any_sync(CH_FULL, ok ? c : -1) & vm;
            const int rel = ok ? (int)M.c_cnt[c] : 0;
            __syncwarp();  // every peer has read c_cnt[c] before its leader advances it
            if (ok) {
                M.slot_v[top0 + rel + __popc(peers & lt)] = (I)y;
                M.cls[y] = (I)d;
                if ((peers & lt) == 0) M.c_cnt[c] = (I)(rel + __popc(peers));
            }
            __syncwarp();
        });
        // ---- restore c_cnt = 0 on the classes touched in this step -------------
        for (int t = lane; t < ntouch; t += 32) M.c_cnt[(int)M.touched[t]] = (I)0;
        if (kTrack && nx >= 0) src.prefetch_row(gb0, gb1);  // the next pivot's row into L2
        __syncwarp();
        SLOT_T(4);
    }
#ifdef SLOT_PROFILE
    if (lane == 0)
        for (int k = 0; k < 16; ++k) atomicAdd(&slot_prof[k], slot_acc[k]);
#endif
    if (progress && lane == 0) progress[1] = 1;
}

// Look-ahead warp of the global-state slot engine: every few steps it walks the
// class list from the current head class and, for the next `ahead` live
// vertices (the next pivots, in order, unless a split reorders them), loads
// their row bounds and prefetches their neighbour lists into L2 -- each list is
// read once per search, so without this the pivot's list fetch is a DRAM round
// trip on the search's critical path.  It only reads (racy reads of structures
// the search is mutating are harmless: a wrong guess costs one useless prefetch).
// the nearest SLOT_LOOKAHEAD_L1 of the look-ahead vertices also get their list
// entries read and their neighbours' class ids prefetched into L1 (config 5:
// 1.626 -> 1.552 s with 16; 32: 1.553 s; re-measured on the current kernel,
// profiles/r02_ab_l1_final.txt: 16 1.317 s, 8 1.324 s, 32 1.328 s)
#ifndef SLOT_LOOKAHEAD_L1
#define SLOT_LOOKAHEAD_L1 16
#endif
#ifndef SLOT_LOOKAHEAD_FIELDS
#define SLOT_LOOKAHEAD_FIELDS 1  // config 5: 1.568 -> 1.523 s
#endif
template <typename I, typename S>
__device__ void slot_lookahead(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n,
                               const SlotMem<I, S> &M, volatile int *progress, int ahead, int every) {
    using C = SlotConst<I>;
    const int lane = threadIdx.x & 31;
    int last = -every;
    while (true) {
        if (progress[1]) break;
        const int step = progress[2];
        if (step - last < every) {
            __nanosleep(32);  // (256 ns: the look-ahead lags, 1.528 -> 1.553 s)
            continue;
        }
        last = step;
        int c = progress[0];
        int budget = ahead;
        // every value read here may be stale (the search is mutating it): ids
        // and slot ranges are range-checked so a stale read never leaves the arrays
        while (budget > 0 && c >= 0 && c < n + 2) {
            long long h = (long long)M.c_head[c], e = (long long)M.c_end[c];
            const int next = (int)M.c_next[c];
            if (h < 0 || e > M.cap || h >= e) break;
            if (e - h > 4096) e = h + 4096;
            for (long long s0 = h; s0 < e && budget > 0; s0 += 32) {
                const long long sl = s0 + lane;
                const int v = sl < e ? (int)M.slot_v[sl] : -1;
                const bool live = v >= 0 && v < n && (int)M.cls[v] == c;
                const int before = ahead - budget;  // live vertices of earlier rounds
                const uint32_t lm = __ballot_sync(CH_FULL, live);
                int64_t b = 0, en = 0;
                if (live) {
                    b = __ldg(indptr + v);
                    en = __ldg(indptr + v + 1);
                    for (int64_t k = b; k < en && k < b + 64; k += 32)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(indices + k));
                }
#if SLOT_LOOKAHEAD_L1 > 0
                // the nearest pivots: their lists and their neighbours' class ids
                // into this SM's L1 (the search warp shares it), one warp-wide
                // round trip per pivot
                for (uint32_t mm = lm; mm && before + __popc(lm & ~mm) < SLOT_LOOKAHEAD_L1; mm &= mm - 1) {
                    const int src = __ffs(mm) - 1;
                    const int64_t bb = __shfl_sync(CH_FULL, b, src), ee = __shfl_sync(CH_FULL, en, src);
                    if (ee - bb > 32) continue;
                    if (lane < (int)(ee - bb)) {
                        const int y = __ldg(indices + bb + lane);
                        if (y >= 0 && y < n) {
#if SLOT_LOOKAHEAD_FIELDS
                            // and the fields of y's class the fast step reads
                            const int cy = (int)M.cls[y];
                            if (cy >= 0 && cy < n + 2) {
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(M.c_live + cy));
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(M.c_prev + cy));
                            }
#else
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(M.cls + y));
#endif
                        }
                    }
                }
#endif
                budget -= __popc(lm);
            }
            c = next;
        }
    }
}

}  // namespace chordal
