// warp_seg.cuh -- one-warp LexBFS for graphs with n <= 1024 (the batch
// kernel's engine and the single-graph path for small n).
//
// The touched-segment arrangement algorithm of lexbfs_seg.cu (search.py:328-532
// / _arraylex.py:17-65 semantics, LOWEST_INDEX or fixed-descending ties) with
// lane l owning 32-bit word l of every bitset, so that the per-step scans are
// warp shuffles and the bitsets live in registers:
//   registers  U (unreached), RA (reached unvisited), B (class starts over
//              positions) and the row word of the pivot (rows are read from
//              global memory in the batch, from a shared-memory copy for single
//              graphs);
//   shared     A / An (arrangement and its scatter buffer), P (positions),
//              par (PEO parents), F / NB (32-word mover and new-start bitsets
//              written with shared atomics) -- 8 * 32W + 256 bytes per graph.
// A step with no split class costs a few dozen instructions; a split step adds
// three shuffle scans and one pass per touched word.  At the end A is the
// order and P the positions.
#pragma once
#include "common.cuh"

namespace chordal {

#ifdef WSEG_PROFILE
// [0] steps [1] (unused) [2] cycles waiting for the row [3] total cycles
// [4] split steps (tools/warp_profile.cu only)
__device__ unsigned long long wseg_prof[8];
// per-phase cycles: [0] pivot + row [1] movers [2] newly reached + scan
// [3] split decision [4] split [5] append + tail
__device__ unsigned long long wseg_ph[8];
#define WSEG_T(k)                                              \
    do {                                                       \
        const long long _c = clock64();                        \
        ph[k] += (unsigned long long)(_c - ph_t0);             \
        ph_t0 = _c;                                            \
    } while (0)
#else
#define WSEG_T(k) \
    do {          \
    } while (0)
#endif

struct WarpSegMem {
    uint16_t *A, *An, *P;  // [32 W]
    uint16_t *par;         // [32 W] PEO parents (required); 0xFFFF = no parent, 0xFFFE = left to the PEO check
    uint32_t *F, *NB;      // [32]
};

namespace wseg {

constexpr int kBig = 0x7FFFFFFF;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exclusive prefix sum over the warp of small values c in [0, 63], and their total:
// six independent ballots of the bit planes instead of a five-round shuffle scan
// (the per-step chain is latency-bound).
__device__ __forceinline__ int excl_prefix6(int c, uint32_t lt, int &total) {
    int pre = 0, tot = 0;
#pragma unroll
    for (int bit = 0; bit < 6; ++bit) {
        const uint32_t bm = __ballot_sync(CH_FULL, (c >> bit) & 1);
        pre += __popc(bm & lt) << bit;
        tot += __popc(bm) << bit;
    }
    total = tot;
    return pre;
}


}  // namespace wseg

// rows: the graph's packed rows (global), sw: row pitch in 32-bit words.
// SPAN: lanes that can hold words (32; 16 for graphs of <= 512 vertices, whose
// shuffle scans then need four rounds instead of five)
template <int MODE, bool LATENCY = false, bool SMEM_ROWS = false, int SPAN = 32>
__device__ void warp_seg_lexbfs(const uint32_t *__restrict__ rows, int sw, int n, const WarpSegMem &M) {
    using namespace wseg;
    const int l = threadIdx.x & 31;
    const uint32_t ltm = lanemask_lt();
    const int W = (n + 31) >> 5;
    uint32_t Ul = l < W ? ((l < W - 1 || !(n & 31)) ? CH_FULL : mask_below(n & 31)) : 0u;
    uint32_t RAl = 0, Bl = 0;
    M.F[l] = 0;
    M.NB[l] = 0;
    {  // par: 0xFFFF over the whole (16-byte aligned, 32 W entries) array: 128-bit stores
        uint4 *p4 = reinterpret_cast<uint4 *>(M.par);
        for (int k = l; k < 4 * W; k += 32) p4[k] = make_uint4(CH_FULL, CH_FULL, CH_FULL, CH_FULL);
    }
    // every rule starts at vertex 0 (parallel/lexbfs.py:173)
    if (l == 0) {
        M.A[0] = 0;
        M.P[0] = 0;
        Ul &= ~1u;
        Bl = 1u;
    }
    __syncwarp();
    int tail = 1, nclasses = 1;
#ifdef WSEG_PROFILE
    unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long ph_t0 = clock64();
    const long long pstart = clock64();
#endif
    for (int i = 0; i < n; ++i) {
        if (i == tail) {  // reached region empty: a new component from the unreached class
            const uint32_t any = __ballot_sync(CH_FULL, Ul != 0);
            int v;
            if (MODE == CHORDAL_TIE_DESCENDING) {
                const int src = highest_bit(any);
                v = 32 * src + highest_bit(__shfl_sync(CH_FULL, Ul, src));
            } else {
                const int src = __ffs(any) - 1;
                v = 32 * src + __ffs(__shfl_sync(CH_FULL, Ul, src)) - 1;
            }
            if (l == 0) {
                M.A[i] = (uint16_t)v;
                M.P[v] = (uint16_t)i;
            }
            if (l == (v >> 5)) Ul &= ~(1u << (v & 31));
            if (l == (i >> 5)) Bl |= 1u << (i & 31);
            tail = i + 1;
            nclasses = 1;
            __syncwarp();
        }
        const int x = M.A[i];
        const int tail0 = tail, hpos = i + 1;
        if (LATENCY) {  // class count for the early exit (the batch tests the class starts instead)
            const uint32_t bh = __shfl_sync(CH_FULL, Bl, (hpos >> 5) & 31);
            if (hpos >= tail0 || ((bh >> (hpos & 31)) & 1u)) --nclasses;  // x's class was {x}
        }
        // ---- row of x ---------------------------------------------------------
        uint32_t r = 0;
#ifdef WSEG_PROFILE
        pacc[0]++;
        const long long pw0 = clock64();
#endif
        // The row of x: shared memory when staged (single graphs), else the
        // read-only path.  No speculative next-row load: it cost the batch more
        // issue slots than the latency it hid (36 graphs per SM hide it anyway).
        if (l < W) r = SMEM_ROWS ? rows[x * sw + l] : __ldg(rows + x * sw + l);
#ifdef WSEG_PROFILE
        {
            const uint32_t any_r = __reduce_or_sync(CH_FULL, r);
            if (any_r == 0xDEADBEEFu) pacc[7]++;  // forces the wait here
            pacc[2] += clock64() - pw0;
        }
#endif
        if (l == (x >> 5)) RAl &= ~(1u << (x & 31));
        WSEG_T(0);
        uint32_t mv = r & RAl;
        const uint32_t ext = r & Ul;
        // ---- movers: flag their positions, record x as their parent ------------
        // (Letting the idle upper lanes of a <= 16-word graph walk the high half
        // of each word -- per-lane mover loops half as long on dense graphs --
        // measured slower in the batch: 5.93 -> 6.07 ms; -DWSEG_HALVES builds it.)
#ifdef WSEG_HALVES
        const bool halves = !LATENCY && W <= 16;
#else
        constexpr bool halves = false;
#endif
        int wbase = 32 * l;
        if (halves) {
            const uint32_t mvw = __shfl_sync(CH_FULL, mv, l & 15);
            mv = l < 16 ? (mvw & 0xFFFFu) : (mvw & 0xFFFF0000u);
            wbase = 32 * (l & 15);
        }
        const int cnt = __popc(mv);
        int pmn = kBig, pmx = -1;
        // one mover per iteration: lanes hold few movers per step, and wider
        // rounds (four, position loads overlapped) only issued predicated-off
        // work -- a config-4 batch 6.45 -> 6.13 ms, config 1 1180 -> 1134
        // cycles per step
        while (mv) {
            const int y = wbase + __ffs(mv) - 1;
            mv &= mv - 1;
            const int pp = (int)M.P[y];
            atomicOr(&M.F[pp >> 5], 1u << (pp & 31));
            M.par[y] = (uint16_t)x;
            pmn = min(pmn, pp);
            pmx = max(pmx, pp);
        }
        WSEG_T(1);
        {
            uint32_t m3 = ext;
            if (halves) {
                const uint32_t ew = __shfl_sync(CH_FULL, ext, l & 15);
                m3 = l < 16 ? (ew & 0xFFFFu) : (ew & 0xFFFF0000u);
            }
            while (m3) {
                M.par[wbase + __ffs(m3) - 1] = (uint16_t)x;
                m3 &= m3 - 1;
            }
        }
        if (ext) {
            Ul &= ~ext;
            RAl |= ext;
        }
        const int cntA = __reduce_add_sync(CH_FULL, cnt);
        // newly reached vertices: exclusive prefix over lanes (= id order).  Most
        // steps reach nothing new or only within one word: no scan then; otherwise
        // the single-graph kernel takes the shorter-latency ballot form, the batch
        // the cheaper shuffle scan (more graphs in flight hide its latency)
        int ktot, xe;
        const uint32_t extw = __ballot_sync(CH_FULL, ext != 0);
        if (__popc(extw) <= 1) {
            xe = 0;
            ktot = extw ? __popc(__shfl_sync(CH_FULL, ext, __ffs(extw) - 1)) : 0;
        } else if (LATENCY) {
            xe = excl_prefix6(__popc(ext), ltm, ktot);
        } else {
            const int ec = __popc(ext);
            int incl = ec;
#pragma unroll
            for (int d = 1; d < SPAN; d <<= 1) {
                const int o = __shfl_up_sync(CH_FULL, incl, d);
                if (l >= d) incl += o;
            }
            xe = incl - ec;
            ktot = __shfl_sync(CH_FULL, incl, SPAN - 1);
        }

        WSEG_T(2);
        if (cntA) {
            __syncwarp();  // the mover flags are in F
            const uint32_t Fl = M.F[l];
            M.F[l] = 0;
            const int gmn = (int)__reduce_min_sync(CH_FULL, (unsigned)pmn);
            const int gmx = __reduce_max_sync(CH_FULL, pmx);
            const uint32_t bmn = __shfl_sync(CH_FULL, Bl, (gmn >> 5) & 31);
            const uint32_t bmx = __shfl_sync(CH_FULL, Bl, ((gmx + 1) >> 5) & 31);
            // movers that fill a run of whole classes change nothing (search.py:448-453)
            const bool whole = cntA == gmx - gmn + 1 && (gmn == hpos || ((bmn >> (gmn & 31)) & 1u)) &&
                               (gmx + 1 >= tail0 || ((bmx >> ((gmx + 1) & 31)) & 1u));
#ifdef WSEG_PROFILE
            if (!whole) pacc[4]++;
#endif
            WSEG_T(3);
            if (!whole) {
                // region class starts of word l: [hpos, tail0) with hpos forced
                uint32_t b = Bl;
                {
                    const int lo = hpos - 32 * l;
                    if (lo > 0) b = lo >= 32 ? 0u : (b & ~mask_below(lo));
                    if (lo >= 0 && lo < 32) b |= 1u << lo;
                }
                const int fc = __popc(Fl);
                const int hb = b ? 32 * l + highest_bit(b) : 0;
                const int lb = b ? 32 * l + __ffs(b) - 1 : kBig;
                int Pc, LBr, NBr;  // movers before word l; last class start before it, first after it
                if (LATENCY) {
                    int fct;
                    Pc = excl_prefix6(fc, ltm, fct);
                    // the starts grow with the word: the nearest words with a start
                    const uint32_t bw = __ballot_sync(CH_FULL, b != 0);
                    const uint32_t below = bw & ltm, above = bw & ~ltm & ~(1u << l);
                    LBr = __shfl_sync(CH_FULL, hb, below ? highest_bit(below) : 0);
                    NBr = __shfl_sync(CH_FULL, lb, above ? __ffs(above) - 1 : 0);
                    if (!below) LBr = 0;
                    if (!above) NBr = kBig;
                } else {
                    // (lanes >= SPAN hold no class start: il = kBig there, so
                    // the suffix minima of lanes < SPAN are complete)
                    int ia = fc, ih = hb, il = lb;
#pragma unroll
                    for (int d = 1; d < SPAN; d <<= 1) {
                        const int oa = __shfl_up_sync(CH_FULL, ia, d), oh = __shfl_up_sync(CH_FULL, ih, d);
                        const int ol = __shfl_down_sync(CH_FULL, il, d);
                        if (l >= d) { ia += oa; ih = max(ih, oh); }
                        if (l + d < 32) il = min(il, ol);
                    }
                    Pc = ia - fc;
                    LBr = __shfl_up_sync(CH_FULL, ih, 1);
                    NBr = __shfl_down_sync(CH_FULL, il, 1);
                    if (l == 0) LBr = 0;
                    if (l == 31) NBr = kBig;
                }
                NBr = min(NBr, tail0);
                // movers at positions < pp (all lanes must call: shuffles)
                auto cntb = [&](int pp) -> int {
                    const int q = pp >> 5;
                    const int pcq = __shfl_sync(CH_FULL, Pc, q & 31);
                    const uint32_t fq = __shfl_sync(CH_FULL, Fl, q & 31);
                    return q >= W ? cntA : pcq + __popc(fq & mask_below(pp & 31));
                };
                // ---- words of split classes ---------------------------------------
                const int lo = max(32 * l, hpos), hi = min(32 * l + 32, tail0);
                const bool inr = lo < hi;
                const int lob = inr ? lo - 32 * l : 0, hib = inr ? hi - 32 * l : 0;
                const uint32_t vm = inr ? (mask_below(hib) & ~mask_below(lob)) : 0u;
                bool touched = (((Fl ^ (Fl >> 1)) & ~(b >> 1)) & vm & (vm >> 1)) != 0;
                // a class entering from the previous word / leaving into the next one
                const int s_in = LBr, e_in = b ? 32 * l + __ffs(b) - 1 : NBr;
                const int s_out = b ? 32 * l + highest_bit(b) : 0, e_out = NBr;
                // bounds inside this lane's own word need no shuffle; e_in is NBr
                // (= e_out) when the word has no class start
                const int c1 = cntb(s_in), c4 = cntb(e_out);
                const int c2 = b ? Pc + __popc(Fl & mask_below(e_in & 31)) : c4;
                const int c3 = Pc + __popc(Fl & mask_below(s_out & 31));
                // the word's class bounds outside it and their mover counts, packed
                // 16 + 16 bits (all <= n <= 1024) so a touched word costs two shuffles
                const uint32_t pkb = (uint32_t)LBr | ((uint32_t)NBr << 16);
                const uint32_t pkc = (uint32_t)c1 | ((uint32_t)c4 << 16);
                if (inr && !touched && !((b >> lob) & 1u)) {
                    const int T = c2 - c1;
                    touched = T > 0 && T < e_in - s_in;
                }
                if (inr && !touched && hib == 32 && NBr > 32 * l + 32 && b) {
                    const int T = c4 - c3;
                    touched = T > 0 && T < e_out - s_out;
                }
                const uint32_t tmask = __ballot_sync(CH_FULL, touched);
                // ---- stable partition of every split class: movers first -----------
                int nsp = 0;
                if (LATENCY) {
                    // Several touched words per round, branch-free up to the stores, so
                    // their shuffle / shared-memory chains overlap (single graphs:
                    // the step is a latency chain; the batch keeps one word per
                    // round -- fewer instructions, its latency is hidden).
                    auto word = [&](int q, int &v, int &dst, bool &ok, bool &start, int &ns) {
                        const uint32_t bq = __shfl_sync(CH_FULL, b, q), fq = __shfl_sync(CH_FULL, Fl, q);
                        const uint32_t pbq = __shfl_sync(CH_FULL, pkb, q), pcq2 = __shfl_sync(CH_FULL, pkc, q);
                        const int pcq = __shfl_sync(CH_FULL, Pc, q);
                        const int p = 32 * q + l;
                        ok = p >= hpos && p < tail0;
                        const uint32_t bl = bq & mask_below(l + 1), ab = bq & ~mask_below(l + 1);
                        const int s = bl ? 32 * q + highest_bit(bl) : (int)(pbq & 0xFFFFu);
                        const int e = ab ? 32 * q + __ffs(ab) - 1 : (int)(pbq >> 16);
                        const int cs = bl ? pcq + __popc(fq & mask_below(s & 31)) : (int)(pcq2 & 0xFFFFu);
                        const int T = (ab ? pcq + __popc(fq & mask_below(e & 31)) : (int)(pcq2 >> 16)) - cs;
                        v = M.A[p];
                        const bool split = T > 0 && T < e - s;
                        const int fb = pcq + __popc(fq & mask_below(l)) - cs;
                        const int to = ((fq >> l) & 1u) ? s + fb : s + T + (p - s - fb);
                        dst = split ? to : p;
                        start = ok && split && p == s;
                        ns = s + T;
                    };
#ifndef WSEG_SPLIT_K
#define WSEG_SPLIT_K 2
#endif
                    // words per round: 2 on config 1 (chordal n = 1000: split steps 633 ->
                    // 446 cycles per step; 4 words: 468, 8: 631, tools/warp_profile.cu);
                    // the batch kernel with 2: 7.52 -> 8.01 ms (tools/ab_batch.sh)
                    constexpr int K = WSEG_SPLIT_K;
                    for (uint32_t tm = tmask; tm;) {
                        int q[K], v[K], dst[K], ns[K];
                        bool has[K], ok[K], st[K];
#pragma unroll
                        for (int u = 0; u < K; ++u) {
                            has[u] = tm != 0;
                            q[u] = has[u] ? __ffs(tm) - 1 : q[0];
                            tm &= tm - 1;
                        }
#pragma unroll
                        for (int u = 0; u < K; ++u) word(q[u], v[u], dst[u], ok[u], st[u], ns[u]);
#pragma unroll
                        for (int u = 0; u < K; ++u)
                            if (has[u] && ok[u]) M.An[dst[u]] = (uint16_t)v[u];
#pragma unroll
                        for (int u = 0; u < K; ++u)
                            if (has[u] && st[u]) {
                                atomicOr(&M.NB[ns[u] >> 5], 1u << (ns[u] & 31));
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
                            p[u] = h ? 32 * (__ffs(tm) - 1) + l : p[0];
                            tm &= tm - 1;
                            ok[u] = h && p[u] >= hpos && p[u] < tail0;
                            v[u] = M.An[p[u]];
                        }
#pragma unroll
                        for (int u = 0; u < K; ++u)
                            if (ok[u]) {
                                M.A[p[u]] = (uint16_t)v[u];
                                M.P[v[u]] = (uint16_t)p[u];
                            }
                    }
                } else {
                    for (uint32_t tm = tmask; tm; tm &= tm - 1) {
                        const int q = __ffs(tm) - 1;
                        const uint32_t bq = __shfl_sync(CH_FULL, b, q), fq = __shfl_sync(CH_FULL, Fl, q);
                        const uint32_t pbq = __shfl_sync(CH_FULL, pkb, q), pcq2 = __shfl_sync(CH_FULL, pkc, q);
                        const int pcq = __shfl_sync(CH_FULL, Pc, q);
                        const int p = 32 * q + l;
                        const bool ok = p >= hpos && p < tail0;
                        const uint32_t bl = bq & mask_below(l + 1), ab = bq & ~mask_below(l + 1);
                        const int s = bl ? 32 * q + highest_bit(bl) : (int)(pbq & 0xFFFFu);
                        const int e = ab ? 32 * q + __ffs(ab) - 1 : (int)(pbq >> 16);
                        const int cs = bl ? pcq + __popc(fq & mask_below(s & 31)) : (int)(pcq2 & 0xFFFFu);
                        const int T = (ab ? pcq + __popc(fq & mask_below(e & 31)) : (int)(pcq2 >> 16)) - cs;
                        const int v = M.A[p];
                        if (ok) {
                            int dst = p;
                            if (T > 0 && T < e - s) {
                                const int fb = pcq + __popc(fq & mask_below(l)) - cs;
                                dst = ((fq >> l) & 1u) ? s + fb : s + T + (p - s - fb);
                                if (p == s) {
                                    atomicOr(&M.NB[(s + T) >> 5], 1u << ((s + T) & 31));
                                    ++nsp;
                                }
                            }
                            M.An[dst] = (uint16_t)v;
                        }
                    }
                    __syncwarp();
                    for (uint32_t tm = tmask; tm; tm &= tm - 1) {
                        const int p = 32 * (__ffs(tm) - 1) + l;
                        if (p >= hpos && p < tail0) {
                            const int v = M.An[p];
                            M.A[p] = (uint16_t)v;
                            M.P[v] = (uint16_t)p;
                        }
                    }
                }
                if (LATENCY) nclasses += __reduce_add_sync(CH_FULL, nsp);
                __syncwarp();
                Bl |= M.NB[l];
                M.NB[l] = 0;
            }
        }
        WSEG_T(4);
        // ---- append the newly reached vertices as one class (tie order) ---------
        if (ext) {
            int idx = xe;
            uint32_t e2 = ext;
            while (e2) {
                const int y = 32 * l + __ffs(e2) - 1;
                e2 &= e2 - 1;
                const int dst = (MODE == CHORDAL_TIE_DESCENDING) ? tail0 + (ktot - 1 - idx) : tail0 + idx;
                ++idx;
                M.A[dst] = (uint16_t)y;
                M.P[y] = (uint16_t)dst;
            }
        }
        // The start bit at hpos is never read again (every later step forces its
        // own region start); the batch skips it (config 4: 6.13 -> 6.01 ms), the
        // latency form keeps it (dropping it measured 0.504 -> 0.513 ms there).
        if (LATENCY && hpos < tail0 && l == (hpos >> 5)) Bl |= 1u << (hpos & 31);
        if (ktot > 0 && l == (tail0 >> 5)) Bl |= 1u << (tail0 & 31);
        if (ktot > 0) {
            tail = tail0 + ktot;
            if (LATENCY) ++nclasses;
        }
        __syncwarp();
        WSEG_T(5);
        // ---- early exit: everything reached, every class a singleton ---------------
        // batch form: with everything reached, test the class starts of [hpos, n)
        // directly (cheaper than keeping a class count every step)
        bool singletons = false;
        if (LATENCY) {
            singletons = tail == n && nclasses == tail - hpos;
        } else if (tail == n) {
            const int lo = hpos + 1 - 32 * l;  // positions <= hpos count as starts
            uint32_t m = Bl | (lo <= 0 ? 0u : mask_below(lo > 32 ? 32 : lo));
            if (32 * l + 32 > n) m |= ~mask_below(n - 32 * l > 0 ? n - 32 * l : 0);
            singletons = __all_sync(CH_FULL, m == CH_FULL);
        }
        if (singletons) {
            for (int p = hpos + l; p < n; p += 32) M.par[M.A[p]] = 0xFFFE;
            break;
        }
    }
    __syncwarp();
#ifdef WSEG_PROFILE
    pacc[3] = clock64() - pstart;
    if (l == 0)
        for (int k = 0; k < 8; ++k) {
            atomicAdd(&wseg_prof[k], pacc[k]);
            atomicAdd(&wseg_ph[k], ph[k]);
        }
#endif
}

}  // namespace chordal
