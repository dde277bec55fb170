// lexbfs_seg.cu -- single-CTA persistent LexBFS over a packed adjacency bitset
// whose per-step cost is O(deg(x)/32 + movers + |split classes|), not O(n).
//
// Replaces, for dense-stored graphs with n <= 32768:
//   lexbfs_partition / PartitionList   search.py:328-532
//   lexbfs_labels / _LabelChain        search.py:152-310
//   lexbfs_array                        _arraylex.py:22-65
//   parallel_lexbfs + kernels 1-4      parallel/lexbfs.py:37-262 (the paper's
//                                      one-launch-per-step loop)
//
// State, all in shared memory (u16 vertex ids and positions, 215 KB at n=32768):
//   A[]    the arrangement: A[0..i) is the order so far, A[i..tail) the
//          reached unvisited vertices in priority order -- label classes in
//          descending label order, each a contiguous run sorted by the tie
//          rule (the _arraylex.py:17-19 invariant: the first unconsumed
//          position is the next pivot).
//   P[]    position of every reached vertex in A.
//   U, RA  vertex bitsets: unreached (the empty-label class, never stored in
//          A) and reached-unvisited.
//   bnd    class-start bits over positions.
//
// Step i, pivot x = A[i], one thread per 32-bit word of x's row:
//   1. movers: row & RA -> flag bit P[y] in F (positions); row & U = the newly
//      reached vertices (appended after the tail as one class, tie order);
//      parent[y] = x for both (the PEO parent: last visited neighbour).
//   2. (only if some reached vertex moved) word-level scans over positions:
//      prefix count of F, last class start before each word, first class
//      start after it.  Any class [s, e) then knows its mover count
//      T = cnt(e) - cnt(s) in O(1).
//   3. words of classes with 0 < T < |class| (a real split; T == |class| is
//      the "whole class moves" case of search.py:448-453 and needs nothing)
//      are listed and stably partitioned: movers first (they form the new,
//      higher class placed before the remainder, search.py:440-463).
// Early exit: once every vertex is reached and every class is a singleton the
// rest of the order is the arrangement itself (G(n, 0.5) exits after a few
// dozen steps).
//
// The next pivot's row is loaded speculatively (guess: A[i+1] as it stands at
// the start of step i -- right whenever the head class is not split), so the
// row fetch of step i+1 overlaps step i.
#include "common.cuh"
#include "warp_seg.cuh"

namespace chordal {

#ifdef SEG_PROFILE
// Per-phase cycle counters of thread 0 (tools/seg_profile.cu only):
// [0] steps [1] full-path steps [2] phase 1 [3] short tail [4] scans [5] 3a
// [6] 3b [7] 3c + end [8] steps with a row-guess hit
__device__ unsigned long long seg_prof[16];
#define SEG_T(k)                                          \
    do {                                                  \
        const long long _c = clock64();                   \
        seg_acc[k] += (unsigned long long)(_c - seg_t0);  \
        seg_t0 = _c;                                      \
    } while (0)
#else
#define SEG_T(k) \
    do {         \
    } while (0)
#endif

namespace {

constexpr int kSegBig = 0x7FFFFFFF;
// Internal mode (not an ABI tie rule): replay a given order, pivot i forced to
// forced[i], and report the first step whose pivot is not in the maximum-label
// class (the LexBFS invariant the reference's debug / audit modes assert:
// search.py:270-271 / 313-322, parallel/lexbfs.py:82-129) and the first step
// whose pivot differs from the LOWEST_INDEX choice.
constexpr int kTieCertify = 5;
#ifndef SEG_SPARSE_SPLIT
#define SEG_SPARSE_SPLIT 1
#endif
constexpr bool kSparseSplit = SEG_SPARSE_SPLIT;
// A step that splits no class and reaches no new vertex writes nothing the next
// step reads except the mover flags and the per-warp slots, which can alternate
// between two buffers by step parity -- so its closing barrier (B4) could be
// skipped.  Measured slower (c3 chordal 58.8 -> 60.3 ms, config 2 chordal 8.20
// -> 9.34 ms: warps that run ahead into the next step's phase 1 lengthen the
// waits at its B1), so off (-DSEG_ELIDE_B4=1 builds it; correct either way).
#ifndef SEG_ELIDE_B4
#define SEG_ELIDE_B4 0
#endif
constexpr int kFBufs = SEG_ELIDE_B4 ? 2 : 1;
#ifndef SEG_SPARSE_WT
#define SEG_SPARSE_WT 2     // only the two-word form (0: any)
#endif
#ifndef SEG_SPARSE_MAXMOV
#define SEG_SPARSE_MAXMOV 32
#endif
#ifndef SEG_SPARSE_SPAN
#define SEG_SPARSE_SPAN 32  // words
#endif
constexpr int kSegDenseFrac = 8;  // edge density (2m / n^2) from which the kernel runs 512 threads: 1 / 8
// The one-warp form (ONEWARP, 4 G words per lane) for sparse graphs up to this
// n: no block barriers, but measured slower -- config 2 chordal 11.9 -> 18.4 ms
// with one warp of 8 words per lane against two warps of 4 (the second warp's
// independent work hides more latency than the barriers cost).  Off by default
// (-DSEG_ONEWARP_MAX_N=16384 builds it).
#ifndef SEG_ONEWARP_MAX_N
#define SEG_ONEWARP_MAX_N 0
#endif
constexpr int kOneWarpMaxN = SEG_ONEWARP_MAX_N;

struct SegLayout {
    size_t A, An, P, U, RA, F, NB, bnd, Pc, LB, NBq, TW, wt, misc, wslot, total;
    __host__ __device__ static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
    __host__ __device__ SegLayout(int W) {
        const size_t np = size_t(W) * 32;
        size_t o = 0;
        A = o; o = align16(o + np * 2);
        An = o; o = align16(o + np * 2);
        P = o; o = align16(o + np * 2);
        const size_t WP = size_t(W + 31) & ~size_t(31);  // words rounded up to a thread's word group (<= 32)
        U = o; o = align16(o + WP * 4);
        RA = o; o = align16(o + WP * 4);
        F = o; o = align16(o + WP * 4 * kFBufs);  // mover flags, double-buffered by step parity
        NB = o; o = align16(o + WP * 4);
        bnd = o; o = align16(o + (WP + 4) * 4);
        Pc = o; o = align16(o + WP * 2);
        LB = o; o = align16(o + WP * 2);
        NBq = o; o = align16(o + WP * 2);
        TW = o; o = align16(o + WP * 2);
        wt = o; o = align16(o + 4 * 32 * 4);
        misc = o; o = align16(o + 24 * 4);
        wslot = o; o = align16(o + 3 * 32 * 4 * kFBufs);  // per-warp mover count / min / max position (by parity)
        total = o;
    }
};

__device__ __forceinline__ uint4 ld_nc_v4(const uint32_t *p) {
    return __ldg(reinterpret_cast<const uint4 *>(p));
}

__device__ __forceinline__ bool seg_better(uint64_t s1, int32_t i1, uint64_t s2, int32_t i2) {
    return s1 > s2 || (s1 == s2 && i1 > i2);
}

template <int MODE>
__device__ __forceinline__ uint64_t seg_tie_score(int32_t v, uint64_t prefix) {
    if (MODE == CHORDAL_TIE_ASCENDING || MODE == kTieCertify) return (uint64_t)(0x7FFFFFFF - v);
    if (MODE == CHORDAL_TIE_DESCENDING) return (uint64_t)v;
    return splitmix64(prefix ^ (uint64_t)(v + 1));  // Arbitration.choose, parallel/engine.py:47-53
}

// Block-wide (score, id) max, broadcast to every thread.  Two barriers (none
// for a one-warp block).
template <bool ONEWARP>
__device__ __forceinline__ void seg_block_max(uint64_t &s, int32_t &id, uint64_t *rs, int32_t *ri) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        uint64_t s2 = __shfl_xor_sync(CH_FULL, s, d);
        int32_t i2 = __shfl_xor_sync(CH_FULL, id, d);
        if (seg_better(s2, i2, s, id)) { s = s2; id = i2; }
    }
    if (ONEWARP) return;
    if (lane == 0) { rs[warp] = s; ri[warp] = id; }
    __syncthreads();
    s = lane < nw ? rs[lane] : 0;
    id = lane < nw ? ri[lane] : -1;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        uint64_t s2 = __shfl_xor_sync(CH_FULL, s, d);
        int32_t i2 = __shfl_xor_sync(CH_FULL, id, d);
        if (seg_better(s2, i2, s, id)) { s = s2; id = i2; }
    }
    __syncthreads();
}

// Block-wide exclusive scans, thread t = word t: sums of a and e, max of h
// (identity 0), suffix min of l (identity kSegBig).  Totals of a and e are
// returned to every thread.  One barrier (none for a one-warp block); wt (4 x
// 32 ints) is free again after the caller's next barrier.
template <bool ONEWARP>
__device__ __forceinline__ void seg_scan4(int a, int e, int h, int l, int *wt, int &xa, int &xe, int &xh, int &xl,
                                          int &ta, int &te) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    int ia = a, ie = e, ih = h, il = l;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int oa = __shfl_up_sync(CH_FULL, ia, d), oe = __shfl_up_sync(CH_FULL, ie, d);
        const int oh = __shfl_up_sync(CH_FULL, ih, d), ol = __shfl_down_sync(CH_FULL, il, d);
        if (lane >= d) { ia += oa; ie += oe; ih = max(ih, oh); }
        if (lane + d < 32) il = min(il, ol);
    }
    if (lane == 31) { wt[warp] = ia; wt[32 + warp] = ie; wt[64 + warp] = ih; }
    if (lane == 0) wt[96 + warp] = il;
    xa = ia - a;
    xe = ie - e;
    xh = __shfl_up_sync(CH_FULL, ih, 1);
    xl = __shfl_down_sync(CH_FULL, il, 1);
    if (lane == 0) xh = 0;
    if (lane == 31) xl = kSegBig;
    if (ONEWARP) {
        ta = __shfl_sync(CH_FULL, ia, 31);
        te = __shfl_sync(CH_FULL, ie, 31);
        return;
    }
    __syncthreads();
    int pa = lane < NW ? wt[lane] : 0, pe = lane < NW ? wt[32 + lane] : 0;
    int ph = lane < NW ? wt[64 + lane] : 0, pl = lane < NW ? wt[96 + lane] : kSegBig;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int oa = __shfl_up_sync(CH_FULL, pa, d), oe = __shfl_up_sync(CH_FULL, pe, d);
        const int oh = __shfl_up_sync(CH_FULL, ph, d), ol = __shfl_down_sync(CH_FULL, pl, d);
        if (lane >= d) { pa += oa; pe += oe; ph = max(ph, oh); }
        if (lane + d < 32) pl = min(pl, ol);
    }
    ta = __shfl_sync(CH_FULL, pa, NW - 1);
    te = __shfl_sync(CH_FULL, pe, NW - 1);
    const int wa = __shfl_sync(CH_FULL, pa, (warp + 31) & 31), we = __shfl_sync(CH_FULL, pe, (warp + 31) & 31);
    const int wh = __shfl_sync(CH_FULL, ph, (warp + 31) & 31), wl = __shfl_sync(CH_FULL, pl, (warp + 1) & 31);
    if (warp > 0) { xa += wa; xe += we; xh = max(xh, wh); }
    if (warp + 1 < NW) xl = min(xl, wl);
}

// Exclusive sum scan of e only (the append-only steps).  One barrier (none for
// a one-warp block).
template <bool ONEWARP>
__device__ __forceinline__ int seg_scan1(int e, int *wt, int &te) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    int ie = e;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int oe = __shfl_up_sync(CH_FULL, ie, d);
        if (lane >= d) ie += oe;
    }
    int xe = ie - e;
    if (ONEWARP) {
        te = __shfl_sync(CH_FULL, ie, 31);
        return xe;
    }
    if (lane == 31) wt[32 + warp] = ie;
    __syncthreads();
    int pe = lane < NW ? wt[32 + lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int oe = __shfl_up_sync(CH_FULL, pe, d);
        if (lane >= d) pe += oe;
    }
    te = __shfl_sync(CH_FULL, pe, NW - 1);
    const int we = __shfl_sync(CH_FULL, pe, (warp + 31) & 31);
    if (warp > 0) xe += we;
    return xe;
}

// Loads / stores of a thread's WT consecutive 32-bit words (WT = 1, 2 or a
// multiple of 4), vectorised to 128 / 64 / 32-bit accesses.
template <int WT>
__device__ __forceinline__ void ld_words(const uint32_t *p, uint32_t (&o)[WT]) {
    if constexpr (WT >= 4) {
#pragma unroll
        for (int g = 0; g < WT / 4; ++g) {
            const uint4 v = reinterpret_cast<const uint4 *>(p)[g];
            o[4 * g] = v.x; o[4 * g + 1] = v.y; o[4 * g + 2] = v.z; o[4 * g + 3] = v.w;
        }
    } else if constexpr (WT == 2) {
        const uint2 v = *reinterpret_cast<const uint2 *>(p);
        o[0] = v.x; o[1] = v.y;
    } else {
        o[0] = *p;
    }
}
template <int WT>
__device__ __forceinline__ void ld_words_nc(const uint32_t *p, uint32_t (&o)[WT]) {
    if constexpr (WT >= 4) {
#pragma unroll
        for (int g = 0; g < WT / 4; ++g) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p) + g);
            o[4 * g] = v.x; o[4 * g + 1] = v.y; o[4 * g + 2] = v.z; o[4 * g + 3] = v.w;
        }
    } else if constexpr (WT == 2) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        o[0] = v.x; o[1] = v.y;
    } else {
        o[0] = __ldg(p);
    }
}
template <int WT>
__device__ __forceinline__ void st_words(uint32_t *p, const uint32_t (&v)[WT]) {
    if constexpr (WT >= 4) {
#pragma unroll
        for (int g = 0; g < WT / 4; ++g)
            reinterpret_cast<uint4 *>(p)[g] = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    } else if constexpr (WT == 2) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(v[0], v[1]);
    } else {
        *p = v[0];
    }
}
template <int WT>
__device__ __forceinline__ void st_zero(uint32_t *p) {
    uint32_t z[WT];
#pragma unroll
    for (int k = 0; k < WT; ++k) z[k] = 0u;
    st_words<WT>(p, z);
}
// WT 16-bit values (all < 65536), packed.
template <int WT>
__device__ __forceinline__ void st_u16(uint16_t *p, const int (&v)[WT]) {
    if constexpr (WT >= 4) {
#pragma unroll
        for (int g = 0; g < WT / 4; ++g)
            reinterpret_cast<uint2 *>(p)[g] =
                make_uint2((uint32_t)v[4 * g] | ((uint32_t)v[4 * g + 1] << 16),
                           (uint32_t)v[4 * g + 2] | ((uint32_t)v[4 * g + 3] << 16));
    } else if constexpr (WT == 2) {
        *reinterpret_cast<uint32_t *>(p) = (uint32_t)v[0] | ((uint32_t)v[1] << 16);
    } else {
        *p = (uint16_t)v[0];
    }
}

// Sparse split (one warp): stably partition, movers first, every split class
// inside the position span [S, E) -- S and E class bounds, at most 32 words --
// the one-warp engine's split (warp_seg.cuh) on a window of position words:
// lane l owns word (S >> 5) + l.  New class starts go to NB; returns the
// number of new classes (warp-uniform).  Used when a step's movers are few
// (<= 32) and their classes are short, so the block-wide scans and the two
// extra barriers of the general split path are not needed.
__device__ __forceinline__ int span_split_warp(int S, int E, const uint32_t *__restrict__ F,
                                               const uint32_t *__restrict__ bnd, uint16_t *A, uint16_t *An,
                                               uint16_t *P, uint32_t *NB) {
    const int l = threadIdx.x & 31;
    const uint32_t ltm = wseg::lanemask_lt();
    const int q0 = S >> 5, nwd = ((E - 1) >> 5) - q0 + 1;
    const int q = q0 + l;
    const int lo = max(32 * q, S), hi = min(32 * q + 32, E);
    const bool inr = l < nwd && lo < hi;
    const int lob = inr ? lo - 32 * q : 0, hib = inr ? hi - 32 * q : 0;
    const uint32_t vm = inr ? (mask_below(hib) & ~mask_below(lob)) : 0u;
    const uint32_t Fl = inr ? (F[q] & vm) : 0u;
    uint32_t b = inr ? (bnd[q] & vm) : 0u;
    if (l == 0) b |= 1u << (S & 31);  // S starts a class (hpos's bit is only set at the step's end)
    int tot;
    const int Pc = wseg::excl_prefix6(__popc(Fl), ltm, tot);
    const int hb = b ? 32 * q + highest_bit(b) : 0;
    const int lb = b ? 32 * q + __ffs(b) - 1 : kSegBig;
    const uint32_t bw = __ballot_sync(CH_FULL, b != 0);
    const uint32_t below = bw & ltm, above = bw & ~ltm & ~(1u << l);
    int LBr = __shfl_sync(CH_FULL, hb, below ? highest_bit(below) : 0);
    int NBr = __shfl_sync(CH_FULL, lb, above ? __ffs(above) - 1 : 0);
    if (!below) LBr = S;
    if (!above) NBr = E;
    NBr = min(NBr, E);
    // movers at positions in [S, pp) (all lanes must call: shuffles)
    auto cntb = [&](int pp) -> int {
        const int qq = (pp >> 5) - q0;
        const int pcq = __shfl_sync(CH_FULL, Pc, qq & 31);
        const uint32_t fq = __shfl_sync(CH_FULL, Fl, qq & 31);
        return qq >= nwd ? tot : pcq + __popc(fq & mask_below(pp & 31));
    };
    // words of split classes (the touched-word test of warp_seg.cuh)
    bool touched = (((Fl ^ (Fl >> 1)) & ~(b >> 1)) & vm & (vm >> 1)) != 0;
    const int s_in = LBr, e_in = b ? 32 * q + __ffs(b) - 1 : NBr;
    const int s_out = b ? 32 * q + highest_bit(b) : 0, e_out = NBr;
    const int c1 = cntb(s_in), c4 = cntb(e_out);
    const int c2 = b ? Pc + __popc(Fl & mask_below(e_in & 31)) : c4;
    const int c3 = Pc + __popc(Fl & mask_below(s_out & 31));
    if (inr && !touched && !((b >> lob) & 1u)) {
        const int T = c2 - c1;
        touched = T > 0 && T < e_in - s_in;
    }
    if (inr && !touched && hib == 32 && NBr > 32 * q + 32 && b) {
        const int T = c4 - c3;
        touched = T > 0 && T < e_out - s_out;
    }
    const uint32_t pkb = (uint32_t)LBr | ((uint32_t)NBr << 16);
    const uint32_t pkc = (uint32_t)c1 | ((uint32_t)c4 << 16);
    const uint32_t tmask = __ballot_sync(CH_FULL, touched);
    int nsp = 0;
#ifndef SEG_SPAN_K
#define SEG_SPAN_K 2
#endif
    // K touched words per round, branch-free up to the stores, so their shuffle /
    // shared-memory chains overlap (the other warps wait: this is latency-bound,
    // as in the one-warp engine's single-graph form)
    constexpr int K = SEG_SPAN_K;
    auto word = [&](int qq, int &v, int &dst, bool &ok, bool &start, int &ns) {
        const uint32_t bq = __shfl_sync(CH_FULL, b, qq), fq = __shfl_sync(CH_FULL, Fl, qq);
        const uint32_t pbq = __shfl_sync(CH_FULL, pkb, qq), pcq2 = __shfl_sync(CH_FULL, pkc, qq);
        const int pcq = __shfl_sync(CH_FULL, Pc, qq);
        const int wq = q0 + qq;
        const int p = 32 * wq + l;
        ok = p >= S && p < E;
        const uint32_t bl = bq & mask_below(l + 1), ab = bq & ~mask_below(l + 1);
        const int s = bl ? 32 * wq + highest_bit(bl) : (int)(pbq & 0xFFFFu);
        const int e = ab ? 32 * wq + __ffs(ab) - 1 : (int)(pbq >> 16);
        const int cs = bl ? pcq + __popc(fq & mask_below(s & 31)) : (int)(pcq2 & 0xFFFFu);
        const int T = (ab ? pcq + __popc(fq & mask_below(e & 31)) : (int)(pcq2 >> 16)) - cs;
        v = ok ? (int)A[p] : 0;
        const bool split = T > 0 && T < e - s;
        const int fb = pcq + __popc(fq & mask_below(l)) - cs;
        const int to = ((fq >> l) & 1u) ? s + fb : s + T + (p - s - fb);
        dst = split ? to : p;
        start = ok && split && p == s;
        ns = s + T;
    };
    for (uint32_t tm = tmask; tm;) {
        int qv[K], v[K], dst[K], ns[K];
        bool has[K], ok[K], st[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            has[u] = tm != 0;
            qv[u] = has[u] ? __ffs(tm) - 1 : 0;
            tm &= tm - 1;
        }
#pragma unroll
        for (int u = 0; u < K; ++u) word(qv[u], v[u], dst[u], ok[u], st[u], ns[u]);
#pragma unroll
        for (int u = 0; u < K; ++u)
            if (has[u] && ok[u]) An[dst[u]] = (uint16_t)v[u];
#pragma unroll
        for (int u = 0; u < K; ++u)
            if (has[u] && st[u]) {
                atomicOr(&NB[ns[u] >> 5], 1u << (ns[u] & 31));
                ++nsp;
            }
    }
    __syncwarp();
    for (uint32_t tm = tmask; tm;) {
        int p[K], v[K];
        bool ok[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const bool h = tm != 0;
            p[u] = h ? 32 * (q0 + __ffs(tm) - 1) + l : 32 * q0 + l;
            tm &= tm - 1;
            ok[u] = h && p[u] >= S && p[u] < E;
            v[u] = An[p[u]];
        }
#pragma unroll
        for (int u = 0; u < K; ++u)
            if (ok[u]) {
                A[p[u]] = (uint16_t)v[u];
                P[v[u]] = (uint16_t)p[u];
            }
    }
    return __reduce_add_sync(CH_FULL, nsp);
}

}  // namespace

// MV: movers handled per round of a thread's mover loop (their position loads
// overlap): 4 for dense graphs (many movers per thread), 2 otherwise (config 2
// chordal 12.53 -> 12.07 ms; G(8192, 0.5) would go 0.260 -> 0.274 ms with 2;
// 4 on the sparse path: c3 chordal 69.8 -> 72.0 ms).
// WT: 32-bit words per thread (thread t owns vertex / position words
// [WT t, WT (t + 1)); 1, 2 or a multiple of 4).
// ONEWARP: the block is one warp -- every barrier is a __syncwarp and the
// block scans are warp scans.
// MAXT: the largest block the instance is launched with (register budget).
template <int MODE, int MV, int WT, bool ONEWARP, int MAXT>
__global__ void __launch_bounds__(ONEWARP ? 32 : MAXT, 1)
lexbfs_seg_kernel(const uint8_t *__restrict__ adj, int n, long long stride, uint64_t seed, uint64_t cell,
                  int32_t *__restrict__ order, int32_t *__restrict__ pos_out, int32_t *__restrict__ parent,
                  const int32_t *__restrict__ forced, int32_t *__restrict__ status) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int W = (n + 31) >> 5;
    const int WP = (W + 3) & ~3;
    const SegLayout L(W);
    uint16_t *A = (uint16_t *)(smem + L.A);
    uint16_t *An = (uint16_t *)(smem + L.An);
    uint16_t *P = (uint16_t *)(smem + L.P);
    uint32_t *U = (uint32_t *)(smem + L.U);
    uint32_t *RA = (uint32_t *)(smem + L.RA);
    uint32_t *const F0 = (uint32_t *)(smem + L.F);
    uint32_t *NB = (uint32_t *)(smem + L.NB);
    uint32_t *bnd = (uint32_t *)(smem + L.bnd);
    // (packing F + Pc into one 64-bit word and LB + NBq into one 32-bit word, so
    // the split phases issue 6 shared loads per word instead of 10, measured
    // c3 chordal 63.3 -> 63.8 ms, config 2 chordal 8.20 -> 8.08 ms: 3b is issue-
    // bound across the block's warps, not shared-memory bound; not used)
    uint16_t *Pc = (uint16_t *)(smem + L.Pc);
    uint16_t *LB = (uint16_t *)(smem + L.LB);
    uint16_t *NBq = (uint16_t *)(smem + L.NBq);
    uint16_t *TW = (uint16_t *)(smem + L.TW);
    int *wt = (int *)(smem + L.wt);
    // Per-step counters in 3 rotating sets of 8: [0] any vertex newly reached,
    // [4] #split-class words, [5] #splits, [6] re-aimed row guess (the mover
    // count and range come from per-warp slots, L.wslot).  Step i uses set
    // i % 3 and resets set (i + 1) % 3, whose last readers (step i - 2) are two
    // barriers behind.
    int *misc = (int *)(smem + L.misc);
    uint64_t *red_s = (uint64_t *)(smem + L.wt);  // block_max scratch aliases wt (never live at once)
    int32_t *red_i = (int32_t *)(smem + L.wt + 32 * 8);

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int NT = ONEWARP ? 32 : blockDim.x, NW = NT >> 5;
    constexpr int LG = WT == 1 ? 0 : (WT == 2 ? 1 : (WT == 4 ? 2 : (WT == 8 ? 3 : (WT == 16 ? 4 : 5))));  // log2(WT)
    static_assert(WT == 1 || WT == 2 || WT == 4 || WT == 8 || WT == 16 || WT == 32, "WT");
    const int w0 = WT * t;  // this thread owns vertex / position words [w0, w0 + WT)
    const bool own = w0 < W;
#define SEG_SYNC()                   \
    do {                             \
        if (ONEWARP) __syncwarp();   \
        else __syncthreads();        \
    } while (0)

    for (int w = t; w < WP; w += NT) {
        U[w] = w < W - 1 ? CH_FULL : (w == W - 1 ? ((n & 31) ? mask_below(n & 31) : CH_FULL) : 0u);
        RA[w] = 0;
        for (int b = 0; b < kFBufs; ++b) F0[b * WP + w] = 0;
        NB[w] = 0;
        bnd[w] = 0;
    }
    if (t < 4) bnd[WP + t] = 0;
    if (t < 24) misc[t] = (t & 7) == 2 ? kSegBig : ((t & 7) == 3 ? -1 : 0);
    if (parent)
        for (int v = t; v < n; v += NT) parent[v] = -1;
    SEG_SYNC();
    // Every rule starts at vertex 0 (vertex 1 in the reference: the smallest id
    // for LOWEST_INDEX, pinned for parallel_lexbfs, parallel/lexbfs.py:173).
    if (t == 0) {
        const int v0 = MODE == kTieCertify ? forced[0] : 0;
        A[0] = (uint16_t)v0;
        P[v0] = 0;
        U[v0 >> 5] &= ~(1u << (v0 & 31));
        bnd[0] = 1u;
        if (MODE == kTieCertify) {
            status[0] = kSegBig;
            status[1] = v0 != 0 ? 0 : kSegBig;
        }
    }
    SEG_SYNC();

    const uint32_t *rows = reinterpret_cast<const uint32_t *>(adj);
    const long long sw = stride >> 2;  // row pitch in words (a multiple of 4)
#ifdef SEG_PROFILE
    unsigned long long seg_acc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
    int tail = 1, nclasses = 1;
    int guess = -1;
    uint32_t nxt[WT];
#pragma unroll
    for (int k = 0; k < WT; ++k) nxt[k] = 0u;

    for (int i = 0; i < n; ++i) {
        // ---- pivot ---------------------------------------------------------
        if (i == tail) {
            // Reached region empty: the next pivot comes from the unreached
            // (empty-label) class -- a new component.
            const uint64_t prefix = MODE == CHORDAL_TIE_SEEDED_ARB ? mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell) : 0;
            uint64_t s = 0;
            int32_t id = -1;
            for (int w = t; w < W; w += NT) {
                uint32_t u = U[w];
                if (!u) continue;
                if (MODE == CHORDAL_TIE_ASCENDING) {
                    const int32_t v = 32 * w + __ffs(u) - 1;
                    const uint64_t sc = seg_tie_score<MODE>(v, prefix);
                    if (id < 0 || seg_better(sc, v, s, id)) { s = sc; id = v; }
                } else if (MODE == CHORDAL_TIE_DESCENDING) {
                    const int32_t v = 32 * w + highest_bit(u);
                    const uint64_t sc = seg_tie_score<MODE>(v, prefix);
                    if (id < 0 || seg_better(sc, v, s, id)) { s = sc; id = v; }
                } else {
                    while (u) {
                        const int b = __ffs(u) - 1;
                        u &= u - 1;
                        const int32_t v = 32 * w + b;
                        const uint64_t sc = seg_tie_score<MODE>(v, prefix);
                        if (id < 0 || seg_better(sc, v, s, id)) { s = sc; id = v; }
                    }
                }
            }
            if (id < 0) s = 0;
            // certify: the forced pivot must be unreached (every unreached vertex
            // has the empty label); U is read before thread 0 updates it
            const int fx = MODE == kTieCertify ? forced[i] : -1;
            const bool fbad = MODE == kTieCertify && !((U[fx >> 5] >> (fx & 31)) & 1u);
            seg_block_max<ONEWARP>(s, id, red_s, red_i);
            if (MODE == kTieCertify) {
                if (fbad) {
                    if (t == 0) {
                        status[0] = i;
                        atomicMin(status + 1, i);
                    }
                    break;
                }
                if (t == 0 && fx != id) atomicMin(status + 1, i);
                id = fx;
            }
            if (t == 0) {
                A[i] = (uint16_t)id;
                P[id] = (uint16_t)i;
                U[id >> 5] &= ~(1u << (id & 31));
                bnd[i >> 5] |= 1u << (i & 31);
            }
            tail = i + 1;
            nclasses = 1;
            SEG_SYNC();
        } else if ((MODE == CHORDAL_TIE_SEEDED_ARB || MODE == kTieCertify) && i > 0) {
            // Elect within the max-label class [i, e): all its members offer
            // themselves as `current` (parallel/lexbfs.py:216-225).
            int e = tail;
            for (int v0 = (i + 1) >> 5; v0 * 32 < tail; v0 += 32) {
                const int w = v0 + lane;
                uint32_t m = 0;
                if (w * 32 < tail) {
                    m = bnd[w];
                    if (w == ((i + 1) >> 5)) m &= ~mask_below((i + 1) & 31);
                }
                const uint32_t any = __ballot_sync(CH_FULL, m != 0);
                if (any) {
                    const int src = __ffs(any) - 1;
                    const uint32_t mm = __shfl_sync(CH_FULL, m, src);
                    e = min(tail, (v0 + src) * 32 + __ffs(mm) - 1);
                    break;
                }
            }
            if (MODE == kTieCertify) {
                // the forced pivot must be a reached vertex of the head class [i, e)
                const int fx = forced[i];
                const bool reached = ((RA[fx >> 5] >> (fx & 31)) & 1u) != 0;
                const int fp = reached ? (int)P[fx] : -1;
                const int a0 = A[i];
                if (fp < i || fp >= e) {
                    if (t == 0) {
                        status[0] = i;
                        atomicMin(status + 1, i);
                    }
                    break;
                }
                SEG_SYNC();  // everyone has read A[i] / P[fx]
                if (t == 0 && fp != i) {
                    atomicMin(status + 1, i);
                    A[i] = (uint16_t)fx;
                    A[fp] = (uint16_t)a0;
                    P[fx] = (uint16_t)i;
                    P[a0] = (uint16_t)fp;
                }
                SEG_SYNC();
            } else {
            const uint64_t prefix = mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell);
            uint64_t s = 0;
            int32_t id = -1, bp = -1;
            for (int p = i + t; p < e; p += NT) {
                const int32_t v = A[p];
                const uint64_t sc = seg_tie_score<MODE>(v, prefix);
                if (id < 0 || seg_better(sc, v, s, id)) { s = sc; id = v; bp = p; }
            }
            const int32_t my_id = id;
            seg_block_max<ONEWARP>(s, id, red_s, red_i);
            if (my_id == id && bp >= 0 && bp != i) {  // exactly one thread holds the winner
                const uint16_t t0 = A[i];
                A[i] = (uint16_t)id;
                A[bp] = t0;
                P[id] = (uint16_t)i;
                P[t0] = (uint16_t)bp;
            }
            SEG_SYNC();
            }
        }

#ifdef SEG_PROFILE
        long long seg_t0 = clock64();
        seg_acc[0]++;
#endif
        const int x = A[i];
        const int tail0 = tail;
        const int hpos = i + 1;  // first region position (the rest of x's class starts here)
        // x's class was the singleton {x} iff the next position starts a class
        const bool head_single = hpos >= tail0 || ((bnd[hpos >> 5] >> (hpos & 31)) & 1u);
        if (head_single) --nclasses;
        if (t == 0) {
            order[i] = x;
            pos_out[x] = i;
        }
        int *fl = misc + 8 * (i % 3);
        uint32_t *const F = F0 + (kFBufs > 1 ? (i & 1) * WP : 0);
        // ---- phase 1: movers and newly reached vertices, 128-bit row loads --
        uint32_t r[WT], ext[WT];
#pragma unroll
        for (int k = 0; k < WT; ++k) r[k] = ext[k] = 0u;
        int extc = 0, cnt = 0, pmn = kSegBig, pmx = -1;
        if (own) {
            if (x == guess) {
#pragma unroll
                for (int k = 0; k < WT; ++k) r[k] = nxt[k];
            } else {
                ld_words_nc<WT>(rows + (long long)x * sw + w0, r);
            }
        }
#ifdef SEG_PROFILE
        const int guess_prev = guess;
#endif
        guess = hpos < tail0 ? (int)A[hpos] : -1;
        // (an L2 prefetch of the row two positions ahead measured slower: c3
        // chordal 68.9 -> 69.8 ms, c2 chordal 12.04 -> 12.42 ms)
        if (own) {
            if (((x >> 5) >> LG) == t) RA[x >> 5] &= ~(1u << (x & 31));
            uint32_t ra[WT], uu[WT];
            ld_words<WT>(RA + w0, ra);
            ld_words<WT>(U + w0, uu);
#pragma unroll
            for (int k = 0; k < WT; ++k) {
                uint32_t m2 = r[k] & ra[k];
                ext[k] = r[k] & uu[k];
                extc += __popc(ext[k]);
                while (m2) {  // MV movers per round: their position loads overlap
                    int y[MV], pp[MV], c = 0;
#pragma unroll
                    for (int u = 0; u < MV; ++u) {
                        y[u] = 32 * (w0 + k) + __ffs(m2) - 1;
                        if (m2) ++c;
                        m2 &= m2 - 1;
                    }
#pragma unroll
                    for (int u = 0; u < MV; ++u) pp[u] = u < c ? (int)P[y[u]] : 0;
#pragma unroll
                    for (int u = 0; u < MV; ++u) {
                        if (u < c) {
                            // (combining the bits of lanes that flag the same word
                            // -- match_any + reduce_or, one atomic per word -- measured
                            // 2x slower: c3 chordal 58.7 -> 128 ms)
                            atomicOr(&F[pp[u] >> 5], 1u << (pp[u] & 31));
                            if (parent) parent[y[u]] = x;
                            pmn = min(pmn, pp[u]);
                            pmx = max(pmx, pp[u]);
                        }
                    }
                    cnt += c;
                }
            }
            if (extc) {
                if (parent) {
#pragma unroll
                    for (int k = 0; k < WT; ++k) {
                        uint32_t m3 = ext[k];
                        while (m3) {
                            const int b = __ffs(m3) - 1;
                            m3 &= m3 - 1;
                            parent[32 * (w0 + k) + b] = x;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < WT; ++k) {
                    uu[k] &= ~ext[k];
                    ra[k] |= ext[k];
                }
                st_words<WT>(U + w0, uu);
                st_words<WT>(RA + w0, ra);
                fl[0] = 1;
            }
        }
#ifdef SEG_PROFILE
        if (cnt) atomicMax(fl + 7, cnt);  // [14]: most movers handled by one thread
#endif
        // The next pivot's row, issued only now: issued before the mover loop
        // (into the registers the current row just left) it stalled that loop
        // (c3 chordal 90.5 -> 86.5 ms; re-measured at two words per thread: 58.9
        // -> 67.3 ms); an extra L2 prefetch of the row after it no longer pays
        // once the load sits here.
        if (guess >= 0 && own) ld_words_nc<WT>(rows + (long long)guess * sw + w0, nxt);
        // mover count and position range: per-warp slots, reduced after B1 by
        // every warp (lane w reads warp w's slot) -- same-address shared atomics
        // from every warp cost ~1 % of a step at N = 32768
        int *ws_ = (int *)(smem + L.wslot) + (kFBufs > 1 ? (i & 1) * 96 : 0);
        {
            const int wc = __reduce_add_sync(CH_FULL, cnt);
            const int wmn = (int)__reduce_min_sync(CH_FULL, (unsigned)pmn);
            const int wmx = __reduce_max_sync(CH_FULL, pmx);
            if (lane == 0) {
                ws_[warp] = wc;
                ws_[32 + warp] = wmn;
                ws_[64 + warp] = wmx;
            }
        }
        if (t < 8) misc[8 * ((i + 1) % 3) + t] = t == 2 ? kSegBig : (t == 3 ? -1 : 0);
        SEG_SYNC();  // B1
        SEG_T(2);
#ifdef SEG_PROFILE
        if (x == guess_prev) seg_acc[8]++;
        seg_acc[14] += fl[7];
#endif
        const bool anyE = fl[0] != 0;
        const int cntA = __reduce_add_sync(CH_FULL, lane < NW ? ws_[lane] : 0);
        const int gmn = (int)__reduce_min_sync(CH_FULL, lane < NW ? (unsigned)ws_[32 + lane] : (unsigned)kSegBig);
        const int gmx = __reduce_max_sync(CH_FULL, lane < NW ? ws_[64 + lane] : -1);
        // Movers that fill a run of whole classes change nothing (every class
        // they touch moves in one hop, search.py:448-453).
        const bool full = cntA > 0 &&
                          !(cntA == gmx - gmn + 1 && (gmn == hpos || ((bnd[gmn >> 5] >> (gmn & 31)) & 1u)) &&
                            (gmx + 1 >= tail0 || ((bnd[(gmx + 1) >> 5] >> ((gmx + 1) & 31)) & 1u)));
        int ktot = 0, xe = 0;
        uint32_t nbadd[WT];
#pragma unroll
        for (int k = 0; k < WT; ++k) nbadd[k] = 0u;
        // Region class starts of position word q: bnd bits in [hpos, tail0)
        // with hpos forced.
        auto breg = [&](int q) -> uint32_t {
            uint32_t b = bnd[q];
            const int lo = hpos - 32 * q;
            if (lo > 0) b = lo >= 32 ? 0u : (b & ~mask_below(lo));
            if (lo >= 0 && lo < 32) b |= 1u << lo;
            return b;
        };
        // Sparse split: few movers (<= 32) whose classes span at most 32 words
        // [S, E) -- one warp partitions them (span_split_warp) while the others
        // wait at one barrier, instead of the block scans and three barriers of
        // the general path.  Every warp finds S and E itself (same loads).
        // Measured: c3 chordal 63.0 -> 58.9 ms, chord-removed 80.4 -> 81.3 ms;
        // with one word per thread (8 warps) it does not pay (config 2 chordal
        // 8.20 -> 8.27 ms), hence two-word form only; mover caps 16 / 128 / 1024
        // and an 8-word span: within 1 %.
        bool sparse = false;
        int spS = -1, spE = -1;
        if (kSparseSplit && (SEG_SPARSE_WT == 0 || WT == SEG_SPARSE_WT) && full && cntA <= SEG_SPARSE_MAXMOV &&
            (gmx >> 5) - (gmn >> 5) < SEG_SPARSE_SPAN) {
            for (int r = 0, qb = gmn >> 5; r < 2 && spS < 0 && qb >= (hpos >> 5); ++r, qb -= 32) {
                const int q = qb - lane;
                uint32_t bw = 0u;
                if (q >= (hpos >> 5)) {
                    bw = breg(q);
                    if (q == (gmn >> 5)) bw &= mask_below((gmn & 31) + 1);
                }
                const uint32_t any = __ballot_sync(CH_FULL, bw != 0u);
                if (any) {
                    const int src = __ffs(any) - 1;
                    spS = 32 * (qb - src) + highest_bit(__shfl_sync(CH_FULL, bw, src));
                }
            }
            const int q1 = (gmx + 1) >> 5;
            if (gmx + 1 >= tail0) spE = tail0;
            for (int r = 0, qb = q1; r < 2 && spE < 0; ++r, qb += 32) {
                if (32 * qb >= tail0) {
                    spE = tail0;
                    break;
                }
                const int q = qb + lane;
                uint32_t bw = 0u;
                if (32 * q < tail0) {
                    bw = breg(q);
                    if (q == q1) bw &= ~mask_below((gmx + 1) & 31);
                }
                const uint32_t any = __ballot_sync(CH_FULL, bw != 0u);
                if (any) {
                    const int src = __ffs(any) - 1;
                    spE = min(tail0, 32 * (qb + src) + __ffs(__shfl_sync(CH_FULL, bw, src)) - 1);
                }
            }
            sparse = spS >= 0 && spE > spS && ((spE - 1) >> 5) - (spS >> 5) < SEG_SPARSE_SPAN;
        }

        if (!full) {
            if (anyE) xe = seg_scan1<ONEWARP>(extc, wt, ktot);
        } else if (sparse) {
            if (t == 0) {  // re-aim the speculative row load (as in the general path below)
                int g = -1;
                if (gmn > hpos && (gmn >> 5) - (hpos >> 5) < 4) {
                    bool inhead = true;
                    for (int q = hpos >> 5; q <= (gmn >> 5); ++q) {
                        uint32_t bw = bnd[q];
                        if (q == (hpos >> 5)) bw &= ~mask_below((hpos & 31) + 1);
                        if (q == (gmn >> 5)) bw &= mask_below((gmn & 31) + 1);
                        if (bw) inhead = false;
                    }
                    if (inhead) g = A[gmn];
                }
                fl[6] = g;
            }
            if (anyE) xe = seg_scan1<ONEWARP>(extc, wt, ktot);
            if (warp == 0) {
                const int ns = span_split_warp(spS, spE, F, bnd, A, An, P, NB);
                if (lane == 0) fl[5] = ns;
            }
            SEG_SYNC();  // B3' (polling a flag instead measured slower: c3 chordal 58.1 -> 60.5 ms)
            {
                const int g = fl[6];
                if (g >= 0 && g != guess) {
                    guess = g;
                    if (own) ld_words_nc<WT>(rows + (long long)g * sw + w0, nxt);
                }
            }
            nclasses += fl[5];
            if (own) {
                ld_words<WT>(NB + w0, nbadd);
                uint32_t any = 0u;
#pragma unroll
                for (int k = 0; k < WT; ++k) any |= nbadd[k];
                if (any) st_zero<WT>(NB + w0);
            }
        } else {
#ifdef SEG_PROFILE
            seg_acc[1]++;
#endif
            // A split of the head class puts its first mover (the smallest
            // mover position gmn, if the head class reaches that far) at hpos:
            // that is the next pivot.  Re-aim the speculative row load.
            if (t == 0) {
                int g = -1;
                if (gmn > hpos && (gmn >> 5) - (hpos >> 5) < 4) {
                    bool inhead = true;
                    for (int q = hpos >> 5; q <= (gmn >> 5); ++q) {
                        uint32_t bw = bnd[q];
                        if (q == (hpos >> 5)) bw &= ~mask_below((hpos & 31) + 1);
                        if (q == (gmn >> 5)) bw &= mask_below((gmn & 31) + 1);
                        if (bw) inhead = false;
                    }
                    if (inhead) g = A[gmn];
                }
                fl[6] = g;
            }
            // ---- phase 2: word-level scans over positions -------------------------
            uint32_t f[WT], b[WT];
            int cpre[WT], hb[WT], lbw[WT];
            int ctot = 0, hmax = 0, lmin = kSegBig;
#pragma unroll
            for (int k = 0; k < WT; ++k) f[k] = b[k] = 0u;
            if (own) ld_words<WT>(F + w0, f);
#pragma unroll
            for (int k = 0; k < WT; ++k) {
                if (own) b[k] = breg(w0 + k);
                cpre[k] = ctot;
                ctot += __popc(f[k]);
                hb[k] = b[k] ? 32 * (w0 + k) + highest_bit(b[k]) : 0;
                lbw[k] = b[k] ? 32 * (w0 + k) + __ffs(b[k]) - 1 : kSegBig;
                hmax = max(hmax, hb[k]);
                lmin = min(lmin, lbw[k]);
            }
            int xa, xh, xl, ta;
            seg_scan4<ONEWARP>(ctot, extc, hmax, lmin, wt, xa, xe, xh, xl, ta, ktot);
            int nbq[WT], lbq[WT];
            {
                int run = xh;
#pragma unroll
                for (int k = 0; k < WT; ++k) { lbq[k] = run; run = max(run, hb[k]); }
                run = min(xl, tail0);
#pragma unroll
                for (int k = WT - 1; k >= 0; --k) { nbq[k] = run; run = min(run, lbw[k]); }
            }
            if (own) {
                int pcv[WT];
#pragma unroll
                for (int k = 0; k < WT; ++k) pcv[k] = xa + cpre[k];
                st_u16<WT>(Pc + w0, pcv);
                st_u16<WT>(LB + w0, lbq);
                st_u16<WT>(NBq + w0, nbq);
            }
            SEG_SYNC();  // B2
            SEG_T(4);
            {
                const int g = fl[6];
                if (g >= 0 && g != guess) {
                    guess = g;
                    if (own) ld_words_nc<WT>(rows + (long long)g * sw + w0, nxt);
                }
            }
            // ---- phase 3a: list the words of split classes ------------------------
            // Split classes hold movers, so they lie inside [span_s, span_e): from
            // the start of the class of the first mover to the end of the class
            // of the last one; words outside are never rewritten.
            int span_s, span_e;
            {
                const int qn = gmn >> 5, qx = (gmx + 1) >> 5;
                const uint32_t bn = breg(qn) & mask_below((gmn & 31) + 1);
                span_s = bn ? 32 * qn + highest_bit(bn) : (int)LB[qn];
                span_e = tail0;
                if (gmx + 1 < tail0) {
                    const uint32_t bx = qx < W ? breg(qx) & ~mask_below((gmx + 1) & 31) : 0u;
                    span_e = bx ? 32 * qx + __ffs(bx) - 1 : min((int)NBq[qx], tail0);
                }
            }
            // movers at positions < pp
            auto cntb = [&](int pp) -> int {
                const int q = pp >> 5;
                if (q >= W) return ta;
                return (int)Pc[q] + __popc(F[q] & mask_below(pp & 31));
            };
            auto is_split = [&](int s, int e) -> bool {
                const int T = cntb(e) - cntb(s);
                return T > 0 && T < e - s;
            };
            if (own) {
#pragma unroll
                for (int k = 0; k < WT; ++k) {
                    const int q = w0 + k;
                    const int lo = max(32 * q, max(hpos, span_s)), hi = min(32 * q + 32, min(tail0, span_e));
                    if (lo >= hi) continue;
                    const int lob = lo - 32 * q, hib = hi - 32 * q;
                    const uint32_t vm = mask_below(hib) & ~mask_below(lob);
                    // two neighbouring positions of one class, one mover and one not
                    bool touched = (((f[k] ^ (f[k] >> 1)) & ~(b[k] >> 1)) & vm & (vm >> 1)) != 0;
                    // a class entering from the previous word
                    if (!touched && !((b[k] >> lob) & 1u))
                        touched = is_split(lbq[k], b[k] ? 32 * q + __ffs(b[k]) - 1 : nbq[k]);
                    // a class leaving into the next word
                    if (!touched && hib == 32 && nbq[k] > 32 * q + 32 && b[k])
                        touched = is_split(32 * q + highest_bit(b[k]), nbq[k]);
                    if (touched) TW[atomicAdd(fl + 4, 1)] = (uint16_t)q;
                }
            }
            SEG_SYNC();  // B2.5
            SEG_T(5);
            const int ntouch = fl[4];
#ifdef SEG_PROFILE
            seg_acc[9] += ntouch;
            seg_acc[10] += cntA;
#endif
            // ---- phase 3b: stable partition of split classes into An --------------
#ifdef SEG_PROFILE
            const long long own0 = clock64();
#endif
            // Branch-free and staged: every round issues its shared-memory loads in
            // three waves (word data; class bounds; mover counts at the bounds)
            // for all four words at once -- written with data-dependent branches
            // the compiler serialised the words, ~2000 cycles per round.
            for (int j0 = 4 * warp; j0 < ntouch; j0 += 4 * NW) {
#ifdef SEG_PROFILE
                seg_acc[15]++;  // 3b rounds of this warp
#endif
                int q[4], p[4], v[4], lbw[4], nbw[4], pcw[4];
                uint32_t bw[4], fw[4];
                bool ok[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) q[u] = (int)TW[j0 + u < ntouch ? j0 + u : j0];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    p[u] = 32 * q[u] + lane;
                    ok[u] = j0 + u < ntouch && p[u] >= hpos && p[u] < tail0;
                    v[u] = A[p[u]];
                    bw[u] = bnd[q[u]];
                    lbw[u] = LB[q[u]];
                    nbw[u] = NBq[q[u]];
                    fw[u] = F[q[u]];
                    pcw[u] = Pc[q[u]];
                }
                int s[4], e[4], ps[4], pe[4];
                uint32_t fs[4], fe[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t b = bw[u];
                    const int lo = hpos - 32 * q[u];
                    b = lo <= 0 ? b : (lo >= 32 ? 0u : (b & ~mask_below(lo)));
                    b = (lo >= 0 && lo < 32) ? (b | (1u << lo)) : b;
                    const uint32_t bl = b & mask_below(lane + 1), above = b & ~mask_below(lane + 1);
                    s[u] = bl ? 32 * q[u] + highest_bit(bl) : lbw[u];
                    e[u] = above ? 32 * q[u] + __ffs(above) - 1 : nbw[u];
                    const int qs = min(s[u] >> 5, W - 1), qe = min(e[u] >> 5, W - 1);
                    ps[u] = Pc[qs];
                    fs[u] = F[qs];
                    pe[u] = Pc[qe];
                    fe[u] = F[qe];
                }
                int dst[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cs = (s[u] >> 5) >= W ? ta : ps[u] + __popc(fs[u] & mask_below(s[u] & 31));
                    const int ce = (e[u] >> 5) >= W ? ta : pe[u] + __popc(fe[u] & mask_below(e[u] & 31));
                    const int T = ce - cs;
                    const bool split = ok[u] && T > 0 && T < e[u] - s[u];
                    const int fb = pcw[u] + __popc(fw[u] & mask_below(lane)) - cs;
                    const int to = ((fw[u] >> lane) & 1u) ? s[u] + fb : s[u] + T + (p[u] - s[u] - fb);
                    dst[u] = split ? to : p[u];
                    if (split && p[u] == s[u]) {
                        atomicOr(&NB[(s[u] + T) >> 5], 1u << ((s[u] + T) & 31));
                        atomicAdd(fl + 5, 1);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (ok[u]) An[dst[u]] = (uint16_t)v[u];
            }
#ifdef SEG_PROFILE
            const long long own1 = clock64();
#endif
            SEG_SYNC();  // B3
#ifdef SEG_PROFILE
            {  // 3b: [12] thread 0's own loop cycles, [13] cycles waiting at B3 for the others
                seg_acc[12] += (unsigned long long)(own1 - own0);
                seg_acc[13] += (unsigned long long)(clock64() - own1);
            }
#endif
            SEG_T(6);
            nclasses += fl[5];
#ifdef SEG_PROFILE
            seg_acc[11] += fl[5];
#endif
            // ---- phase 3c: copy back and positions --------------------------------
            for (int j0 = 4 * warp; j0 < ntouch; j0 += 4 * NW) {
                int p[4], v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    p[u] = j0 + u < ntouch ? 32 * (int)TW[j0 + u] + lane : -1;
                    v[u] = p[u] >= hpos && p[u] < tail0 ? (int)An[p[u]] : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (v[u] >= 0) {
                        A[p[u]] = (uint16_t)v[u];
                        P[v[u]] = (uint16_t)p[u];
                    }
                }
            }
            if (own) {
                ld_words<WT>(NB + w0, nbadd);
                uint32_t any = 0u;
#pragma unroll
                for (int k = 0; k < WT; ++k) any |= nbadd[k];
                if (any) st_zero<WT>(NB + w0);
            }
        }
        // ---- end of step: clear flags, new class starts, append -----------------
        if (own) {
            if (cntA && (w0 + WT - 1) >= (gmn >> 5) && w0 <= (gmx >> 5)) st_zero<WT>(F + w0);
#pragma unroll
            for (int k = 0; k < WT; ++k) {
                // (the hpos bit is never read again -- later steps force their own
                // region start -- so elided steps skip it: no shared write then)
                if (hpos < tail0 && (hpos >> 5) == w0 + k && !(SEG_ELIDE_B4 && !full && ktot == 0))
                    nbadd[k] |= 1u << (hpos & 31);
                if (ktot > 0 && (tail0 >> 5) == w0 + k) nbadd[k] |= 1u << (tail0 & 31);
            }
#pragma unroll
            for (int k = 0; k < WT; ++k)
                if (nbadd[k]) bnd[w0 + k] |= nbadd[k];
            if (extc) {  // the newly reached vertices: one class after the tail, tie order
                int idx = xe;
#pragma unroll
                for (int k = 0; k < WT; ++k) {
                    uint32_t e2 = ext[k];
                    while (e2) {
                        const int b = __ffs(e2) - 1;
                        e2 &= e2 - 1;
                        const int dst = (MODE == CHORDAL_TIE_DESCENDING) ? tail0 + (ktot - 1 - idx) : tail0 + idx;
                        ++idx;
                        A[dst] = (uint16_t)(32 * (w0 + k) + b);
                        P[32 * (w0 + k) + b] = (uint16_t)dst;
                    }
                }
            }
        }
        if (ktot > 0) {
            tail = tail0 + ktot;
            ++nclasses;
        }
        if (!(SEG_ELIDE_B4 && !full && ktot == 0)) SEG_SYNC();  // B4
        SEG_T(full ? 7 : 3);
        // ---- early exit: everything reached, every class a singleton ----------
        if (tail == n && nclasses == tail - hpos) {
            for (int p = hpos + t; p < n; p += NT) {
                const int v = A[p];
                if (MODE == kTieCertify && forced[p] != v) {  // every class a singleton: the order is fixed
                    atomicMin(status, p);
                    atomicMin(status + 1, p);
                }
                order[p] = v;
                pos_out[v] = p;
                // the skipped steps would still have refreshed this vertex's
                // parent: leave it to the PEO check (unknown = -2)
                if (parent) parent[v] = -2;
            }
            break;
        }
    }
    if (MODE == kTieCertify) {  // "no such step" -> -1
        SEG_SYNC();
        if (t < 2 && status[t] == kSegBig) status[t] = -1;
    }
#ifdef SEG_PROFILE
    if (t == 0)
        for (int k = 0; k < 16; ++k) seg_prof[k] = seg_acc[k];
#endif
#undef SEG_SYNC
}

size_t seg_smem_bytes(int64_t n) { return SegLayout((int)((n + 31) >> 5)).total; }

// n <= 1024, LOWEST_INDEX / descending ties: the one-warp engine (warp_seg.cuh),
// bitsets in registers; the arrays are copied out at the end.
// Launched with kWarpKernelWarps warps: all stage the rows (more loads in
// flight); warp 0 runs the search and copies the arrays out.
constexpr int kWarpKernelWarps = 8;
template <int MODE, bool STAGE>
__global__ void __launch_bounds__(32 * kWarpKernelWarps, 1)
lexbfs_warp_kernel(const uint8_t *__restrict__ adj, int n, long long stride, int32_t *__restrict__ order,
                   int32_t *__restrict__ pos_out, int32_t *__restrict__ parent) {
    extern __shared__ __align__(16) uint8_t smem[];
    const size_t np = size_t((n + 31) >> 5) * 32;
    WarpSegMem M;
    M.A = (uint16_t *)smem;
    M.An = M.A + np;
    M.P = M.An + np;
    M.par = M.P + np;
    M.F = (uint32_t *)(M.par + np);
    M.NB = M.F + 32;
    const uint32_t *rows = reinterpret_cast<const uint32_t *>(adj);
    const int nthr = blockDim.x;
    if (STAGE) {  // rows into shared memory after the state (16-byte aligned), eight copies in flight per thread
        uint4 *dst = reinterpret_cast<uint4 *>(smem + ((np * 8 + 256 + 15) & ~size_t(15)));
        const uint4 *src = reinterpret_cast<const uint4 *>(adj);
        const int n16 = n * (int)(stride >> 4);
        int k = threadIdx.x;
        for (; k + 7 * nthr < n16; k += 8 * nthr) {
            uint4 t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) t[j] = __ldg(src + k + nthr * j);
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[k + nthr * j] = t[j];
        }
        for (; k < n16; k += nthr) dst[k] = __ldg(src + k);
        rows = reinterpret_cast<const uint32_t *>(dst);
    }
    __syncthreads();
    // the staging warps leave: parked at a barrier beside the searching warp they
    // slow it down (config 1: 0.50 -> 0.59 ms)
    if (threadIdx.x >= 32) return;
    warp_seg_lexbfs<MODE, true, STAGE>(rows, (int)(stride >> 2), n, M);
    for (int k = threadIdx.x; k < n; k += 32) {
        order[k] = M.A[k];
        pos_out[k] = M.P[k];
        if (parent) parent[k] = (int)(int16_t)M.par[k];
    }
}

int launch_lexbfs_seg(const uint8_t *adj, int64_t n, int64_t stride, int64_t m, int32_t tie_rule, uint64_t seed, uint64_t cell,
                      int32_t *order, int32_t *pos, int32_t *parent, cudaStream_t stream,
                      const int32_t *forced = nullptr, int32_t *status = nullptr) {
    if (n <= 0) return CHORDAL_OK;
    if (n > CHORDAL_DENSE_LEXBFS_MAX_N) return CHORDAL_ETOOLARGE;
    if (tie_rule == kTieCertify && (!forced || !status)) return CHORDAL_EINVAL;
    // (the CTA engine below with one word per thread takes 0.99-1.16 ms for
    // config 1's LexBFS on 32-512 threads; the one-warp engine 0.51 ms)
    if (n <= 1024 && tie_rule != CHORDAL_TIE_SEEDED_ARB && tie_rule != kTieCertify) {
        const size_t state = (size_t((n + 31) >> 5) * 32 * 2 * 4 + 256 + 15) & ~size_t(15);
        const size_t rows = (size_t)n * stride;
        const bool stage = state + rows <= 200 * 1024;  // rows staged in shared memory when they fit
        const size_t wsmem = stage ? state + rows : state;
#define WARP_LAUNCH(M, S)                                                                                    \
    if (cudaFuncSetAttribute(lexbfs_warp_kernel<M, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                             (int)wsmem) != cudaSuccess)                                                      \
        return CHORDAL_ECUDA;                                                                                 \
    lexbfs_warp_kernel<M, S><<<1, 32 * kWarpKernelWarps, wsmem, stream>>>(adj, (int)n, stride, order, pos, parent);
        if (tie_rule == CHORDAL_TIE_DESCENDING) {
            if (stage) { WARP_LAUNCH(CHORDAL_TIE_DESCENDING, true) } else { WARP_LAUNCH(CHORDAL_TIE_DESCENDING, false) }
        } else {
            if (stage) { WARP_LAUNCH(CHORDAL_TIE_ASCENDING, true) } else { WARP_LAUNCH(CHORDAL_TIE_ASCENDING, false) }
        }
#undef WARP_LAUNCH
        CH_LAUNCH_CHECK();
        return CHORDAL_OK;
    }
    const int W = (int)((n + 31) >> 5);
    // Words per thread (WT) and threads (T).  Every phase of a step has a
    // per-thread loop over the thread's words and ends at a block barrier, so
    // the step's latency follows the per-thread work: fewer words per thread
    // until the block barrier / register budget bites (config 3 chordal, sparse:
    // WT = 4 on 256 threads 68.2 ms, WT = 2 on 512 63.0 ms, WT = 1 on 1024 99 ms
    // (64 registers, spills); config 2 chordal: WT 4 / 2 / 1 11.9 / 9.07 / 8.20
    // ms; G(8192, 0.5): 0.452 / 0.250 / 0.176 ms; G(32768, 0.5): WT 4 / 2 / 1
    // 0.68 / 0.556 / 0.616 ms; WT = 8 / 16 (fewer warps) 103 / 180 ms on
    // config 3 chordal).  Dense graphs (m known, 2m >= n^2 / 8: G(n, 0.5) splits
    // classes of thousands of vertices in each of its few steps) keep at least
    // 512 threads for their partition phases (3b / 3c, one warp per four
    // split-class words); extra threads for sparse graphs do not pay (config 2
    // chordal on 512 threads: 8.20 -> 9.20 ms).
    const bool dense = m >= 0 && n > 1024 && 2 * m * kSegDenseFrac >= n * n;
    const bool onewarp = m > 0 && !dense && n <= kOneWarpMaxN;
    int T1 = max(32, (W + 31) / 32 * 32), T2 = max(32, ((W + 1) / 2 + 31) / 32 * 32);
    if (dense) {
        T1 = max(T1, 512);
        T2 = max(T2, 512);
    }
#ifdef SEG_THREADS_ENV
    if (const char *ev = getenv("SEG_THREADS")) T2 = max(T2, atoi(ev));
#endif
#ifndef SEG_MV_DENSE
#define SEG_MV_DENSE 4
#endif
// movers per round, sparse graphs: 2 with two words per thread, 1 with one
// (config 2 chordal 8.20 -> 7.96 ms; c3 chordal with 1: 58.6 -> 59.0 ms);
// dense graphs: 4 (2: unchanged)
#ifndef SEG_MV_SPARSE
#define SEG_MV_SPARSE 2
#endif
    const bool wt1 = W <= (dense ? 512 : 256);  // one word per thread within a 512-thread register budget
    const size_t smem = seg_smem_bytes(n);
    cudaError_t e;
#define SEG_LAUNCH_K(M, K, WTN, OW, NTH, MT)                                                                     \
    e = cudaFuncSetAttribute(lexbfs_seg_kernel<M, K, WTN, OW, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)smem);                                                                         \
    if (e != cudaSuccess) return CHORDAL_ECUDA;                                                                  \
    lexbfs_seg_kernel<M, K, WTN, OW, MT><<<1, NTH, smem, stream>>>(adj, (int)n, stride, seed, cell, order, pos,  \
                                                                   parent, forced, status);
#if SEG_ONEWARP_MAX_N > 0
#define SEG_LAUNCH_OW(M)                               \
    if (onewarp && W <= 128) {                         \
        SEG_LAUNCH_K(M, 2, 4, true, 32, 32)            \
    } else if (onewarp && W <= 256) {                  \
        SEG_LAUNCH_K(M, 2, 8, true, 32, 32)            \
    } else if (onewarp) {                              \
        SEG_LAUNCH_K(M, 2, 16, true, 32, 32)           \
    } else
#else
#define SEG_LAUNCH_OW(M)
#endif
#define SEG_LAUNCH(M)                                   \
    SEG_LAUNCH_OW(M)                                    \
    if (dense && wt1) {                                 \
        SEG_LAUNCH_K(M, SEG_MV_DENSE, 1, false, T1, 512) \
    } else if (dense) {                                 \
        SEG_LAUNCH_K(M, SEG_MV_DENSE, 2, false, T2, 512) \
    } else if (wt1) {                                   \
        SEG_LAUNCH_K(M, 1, 1, false, T1, 512)           \
    } else {                                            \
        SEG_LAUNCH_K(M, SEG_MV_SPARSE, 2, false, T2, 512) \
    }
    switch (tie_rule) {
        case CHORDAL_TIE_ASCENDING: SEG_LAUNCH(CHORDAL_TIE_ASCENDING); break;
        case CHORDAL_TIE_DESCENDING: SEG_LAUNCH(CHORDAL_TIE_DESCENDING); break;
        case CHORDAL_TIE_SEEDED_ARB: SEG_LAUNCH(CHORDAL_TIE_SEEDED_ARB); break;
        case kTieCertify: SEG_LAUNCH(kTieCertify); break;
        default: return CHORDAL_EINVAL;
    }
#undef SEG_LAUNCH
#undef SEG_LAUNCH_OW
#undef SEG_LAUNCH_K
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
