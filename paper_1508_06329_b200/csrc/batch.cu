// batch.cu -- is_chordal over many small independent graphs (n <= 1024).
//
// One warp (= one CTA) per graph.  A first coalesced pass over the graph's
// packed rows counts the edges and pulls the rows from HBM into L2; the warp
// then runs one of two LexBFS engines and the PEO check, reading rows through
// L1/L2 while only the ~19 KB of search state lives in shared memory (so ~11
// graphs are in flight per SM to hide the per-step latency).  Replaces
// is_chordal (peo.py:177-202) called once per graph by the reference's bench
// loop (bench.py:86-95).
//
//   dense graphs (m > n^2/16): a one-warp arrangement engine
//     (reached-region arrangement + unreached bitset, stable segmented
//     partition per step) -- random dense graphs split into singleton classes
//     after O(log n) steps and the search exits early;
//   other graphs: the O(deg)-per-step slot engine (slot_engine.cuh), which
//     also yields every vertex's PEO parent.
// PEO check: lanes stride over vertices; parent from the engine (or a short
// backward scan over the order); stray = A[v] & ~A[p] & ~{p} confirmed by
// pos < pos(p); the minimum (p << 32 | v) key is the reference's witness.
#include "common.cuh"
#include "slot_engine.cuh"

namespace chordal {

namespace {

struct BatchLayout {  // shared memory per graph (one warp); the adjacency stays in global memory
    size_t ord, pos, par, uni, total;
    // arrangement engine (inside uni)
    size_t arrA, arrB, segtot, U, bnd, Fw, Bw, cin, lbin, rowbuf, arr_end;
    // slot engine (inside uni)
    size_t cls, slot, c_head, c_end, c_live, c_prev, c_next, c_tgt, c_cnt, freel, touched, scratch, nbuf,
        slot_end;
    int cap;
    __host__ __device__ static size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
    __host__ __device__ BatchLayout(int n) {
        const int W = (n + 31) >> 5;
        const size_t np = size_t(W) * 32, nc = size_t(n) + 2;
        size_t o = 0;
        ord = o; o = a16(o + size_t(n) * 2);
        pos = o; o = a16(o + size_t(n) * 2);
        par = o; o = a16(o + size_t(n) * 2);
        uni = o;
        size_t u = o;
        arrA = u; u = a16(u + np * 2);
        arrB = u; u = a16(u + np * 2);
        segtot = u; u = a16(u + np * 2);
        U = u; u = a16(u + size_t(W) * 4);
        bnd = u; u = a16(u + size_t(W + 2) * 4);
        Fw = u; u = a16(u + size_t(W) * 4);
        Bw = u; u = a16(u + size_t(W + 1) * 4);
        cin = u; u = a16(u + size_t(W) * 4);
        lbin = u; u = a16(u + size_t(W) * 4);
        rowbuf = u; u = a16(u + size_t(W) * 4);
        arr_end = u;
        cap = 2 * n + 64;
        u = o;
        cls = u; u = a16(u + size_t(n) * 2);
        slot = u; u = a16(u + size_t(cap + slot_detail::kSlotPad) * 2);
        c_head = u; u = a16(u + nc * 2);
        c_end = u; u = a16(u + nc * 2);
        c_live = u; u = a16(u + nc * 2);
        c_prev = u; u = a16(u + nc * 2);
        c_next = u; u = a16(u + nc * 2);
        c_tgt = u; u = a16(u + nc * 2);
        c_cnt = u; u = a16(u + nc * 2);
        freel = u; u = a16(u + nc * 2);
        touched = u; u = a16(u + nc * 2);
        scratch = u; u = a16(u + size_t(n) * 2);
        nbuf = u; u = a16(u + size_t(n) * 2);
        slot_end = u;
        total = arr_end > slot_end ? arr_end : slot_end;
    }
};

// Arrangement LexBFS (LOWEST_INDEX) for one graph in one warp (the _arraylex.py:17-19
// invariant; lexbfs_seg.cu is the single-graph form).
__device__ void arrangement_lexbfs_warp(const uint32_t *__restrict__ A32, int n, int sw, uint8_t *smem,
                                        const BatchLayout &L, uint16_t *ord, uint16_t *pos) {
    const int lane = threadIdx.x & 31;
    const int W = (n + 31) >> 5;
    uint16_t *arrA = (uint16_t *)(smem + L.arrA);
    uint16_t *arrB = (uint16_t *)(smem + L.arrB);
    uint16_t *segtot = (uint16_t *)(smem + L.segtot);
    uint32_t *U = (uint32_t *)(smem + L.U);
    uint32_t *bnd = (uint32_t *)(smem + L.bnd);
    uint32_t *Fw = (uint32_t *)(smem + L.Fw);
    uint32_t *Bw = (uint32_t *)(smem + L.Bw);
    uint32_t *cin = (uint32_t *)(smem + L.cin);
    int32_t *lbin = (int32_t *)(smem + L.lbin);
    uint32_t *rowbuf = (uint32_t *)(smem + L.rowbuf);
    for (int w = lane; w < W; w += 32) {
        U[w] = (w == W - 1 && (n & 31)) ? mask_below(n & 31) : CH_FULL;
        bnd[w] = 0;
    }
    if (lane < 2) bnd[W + lane] = 0;
    __syncwarp();
    if (lane == 0) {
        arrA[0] = 0;
        U[0] &= ~1u;
        bnd[0] |= 1u;
    }
    __syncwarp();
    int tail = 1;
    uint16_t *A = arrA, *An = arrB;
    for (int i = 0; i < n; ++i) {
        if (i == tail) {
            uint32_t u = lane < W ? U[lane] : 0u;
            uint32_t any = __ballot_sync(CH_FULL, u != 0);
            int src = __ffs(any) - 1;
            uint32_t uw = __shfl_sync(CH_FULL, u, src);
            int id = 32 * src + __ffs(uw) - 1;
            if (lane == 0) {
                A[i] = (uint16_t)id;
                U[id >> 5] &= ~(1u << (id & 31));
                bnd[i >> 5] |= 1u << (i & 31);
            }
            tail = i + 1;
            __syncwarp();
        }
        const int x = A[i];
        if (lane == 0) {
            ord[i] = (uint16_t)x;
            pos[x] = (uint16_t)i;
        }
        if (lane < W) rowbuf[lane] = __ldg(A32 + x * sw + lane);  // pivot row: one L2 round trip
        // speculative L1 prefetch of the row of the vertex now at position i+1
        // (it is the next pivot whenever the refinement leaves that slot alone,
        // e.g. once the leading classes are singletons)
        if (lane < W && i + 1 < tail)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A32 + (int)A[i + 1] * sw + lane));
        __syncwarp();
        const uint32_t *rowx = rowbuf;
        const int R = tail - (i + 1);
        const int Q = (R + 31) >> 5;
        for (int q = 0; q < Q; ++q) {
            int p = i + 1 + 32 * q + lane;
            bool valid = p < tail;
            int v = valid ? A[p] : 0;
            bool f = valid && ((rowx[v >> 5] >> (v & 31)) & 1u);
            bool b = valid && (((bnd[p >> 5] >> (p & 31)) & 1u) || p == i + 1);
            uint32_t fw = __ballot_sync(CH_FULL, f), bw = __ballot_sync(CH_FULL, b);
            if (lane == 0) { Fw[q] = fw; Bw[q] = bw; }
        }
        uint32_t ext = lane < W ? (rowx[lane] & U[lane]) : 0u;
        bool pred = true;
        if (lane < W) {
            if (U[lane]) pred = false;
            int lo = max(i + 1, 32 * lane), hi = min(tail, 32 * lane + 32);
            if (lo < hi) {
                uint32_t live = mask_below(hi - 32 * lane) & ~mask_below(lo - 32 * lane);
                uint32_t B = bnd[lane];
                if (i + 1 >= 32 * lane && i + 1 < 32 * lane + 32) B |= 1u << ((i + 1) & 31);
                uint32_t E = (B >> 1) | (bnd[lane + 1] << 31);
                if (tail - 1 >= 32 * lane && tail - 1 < 32 * lane + 32) E |= 1u << ((tail - 1) & 31);
                if (live & ~(B & E)) pred = false;
            }
        }
        if (__all_sync(CH_FULL, pred)) {
            for (int p = i + 1 + lane; p < n; p += 32) {
                int v = A[p];
                ord[p] = (uint16_t)v;
                pos[v] = (uint16_t)p;
            }
            break;
        }
        __syncwarp();
        uint32_t F = 0, B = 0;
        if (lane < Q) { F = Fw[lane]; B = Bw[lane]; }
        int iflag = B != 0;
        int hb = iflag ? highest_bit(B) : 0;
        int icnt = iflag ? __popc(F & ~mask_below(hb)) : __popc(F);
        int ilb = iflag ? 32 * lane + hb : -1;
        int iext = __popc(ext);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int oc = __shfl_up_sync(CH_FULL, icnt, d), of = __shfl_up_sync(CH_FULL, iflag, d);
            int ol = __shfl_up_sync(CH_FULL, ilb, d), oe = __shfl_up_sync(CH_FULL, iext, d);
            if (lane >= d) {
                if (!iflag) icnt += oc;
                iflag |= of;
                ilb = max(ilb, ol);
                iext += oe;
            }
        }
        const int ktot = __shfl_sync(CH_FULL, iext, 31);
        int cnt_in = __shfl_up_sync(CH_FULL, icnt, 1), lb_in = __shfl_up_sync(CH_FULL, ilb, 1);
        int ext_pref = __shfl_up_sync(CH_FULL, iext, 1);
        if (lane == 0) { cnt_in = 0; lb_in = -1; ext_pref = 0; }
        if (lane < Q) {
            cin[lane] = cnt_in;
            lbin[lane] = lb_in;
            const uint32_t vb = mask_below(R - 32 * lane);
            const uint32_t Bn = (lane + 1 < Q) ? Bw[lane + 1] : 0u;
            uint32_t E = (B >> 1) | (Bn << 31);
            if (((R - 1) >> 5) == lane) E |= 1u << ((R - 1) & 31);
            E &= vb;
            uint32_t ends = E & ~B;
            while (ends) {
                int e = __ffs(ends) - 1;
                ends &= ends - 1;
                uint32_t below = B & mask_below(e + 1);
                int s, fb;
                if (below) {
                    int h = highest_bit(below);
                    s = 32 * lane + h;
                    fb = __popc(F & mask_below(e) & ~mask_below(h));
                } else {
                    s = lb_in;
                    fb = cnt_in + __popc(F & mask_below(e));
                }
                int Tt = fb + ((F >> e) & 1u);
                segtot[s] = (uint16_t)Tt;
                int len = 32 * lane + e - s + 1;
                if (Tt > 0 && Tt < len) {
                    int nb = i + 1 + s + Tt;
                    atomicOr(&bnd[nb >> 5], 1u << (nb & 31));
                }
            }
        }
        if (ext) {
            int r = 0;
            uint32_t e2 = ext;
            while (e2) {
                int b = __ffs(e2) - 1;
                e2 &= e2 - 1;
                An[tail + ext_pref + r++] = (uint16_t)(32 * lane + b);
            }
            U[lane] &= ~ext;
        }
        if (lane == 0 && ktot > 0) atomicOr(&bnd[tail >> 5], 1u << (tail & 31));
        __syncwarp();
        for (int q = 0; q < Q; ++q) {
            int rel = 32 * q + lane;
            if (rel < R) {
                int v = A[i + 1 + rel];
                uint32_t Fq = Fw[q], Bq = Bw[q];
                uint32_t Bn = (q + 1 < Q) ? Bw[q + 1] : 0u;
                uint32_t E = (Bq >> 1) | (Bn << 31);
                if (((R - 1) >> 5) == q) E |= 1u << ((R - 1) & 31);
                int nrel = rel;
                if (!(((Bq & E) >> lane) & 1u)) {
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
        __syncwarp();
        uint16_t *t2 = A;
        A = An;
        An = t2;
    }
    __syncwarp();
}

}  // namespace

__global__ void __launch_bounds__(32)
batch_chordal_kernel(const uint8_t *__restrict__ adj_all, int n, int stride, int32_t *__restrict__ orders,
                     int32_t *__restrict__ witness) {
    extern __shared__ __align__(16) uint8_t smem[];
    const BatchLayout L(n);
    const int lane = threadIdx.x;
    const int W = (n + 31) >> 5;
    const int sw = stride >> 2;  // row pitch in 32-bit words
    const long long g = blockIdx.x;
    const uint32_t *A32 = reinterpret_cast<const uint32_t *>(adj_all + g * (long long)n * stride);
    uint16_t *ord = (uint16_t *)(smem + L.ord);
    uint16_t *pos = (uint16_t *)(smem + L.pos);
    uint16_t *par = (uint16_t *)(smem + L.par);

    // ---- one coalesced 128-bit pass over the graph: edge count (engine choice)
    //      and the HBM -> L2 fill for the row reads that follow ------------------
    int bits = 0;
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(A32);
        const int n16 = (n * stride) >> 4;
        int k = lane;
        for (; k + 96 < n16; k += 128) {
            uint4 a = __ldg(src + k), b = __ldg(src + k + 32), c = __ldg(src + k + 64), d = __ldg(src + k + 96);
            bits += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) +
                    __popc(b.z) + __popc(b.w) + __popc(c.x) + __popc(c.y) + __popc(c.z) + __popc(c.w) +
                    __popc(d.x) + __popc(d.y) + __popc(d.z) + __popc(d.w);
        }
        for (; k < n16; k += 32) {
            uint4 a = __ldg(src + k);
            bits += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
        }
    }
    bits = __reduce_add_sync(CH_FULL, bits);  // = 2m

    // ---- LexBFS -------------------------------------------------------------------
    const bool dense = (long long)bits * 8 > (long long)n * n;  // m > n^2/16
    bool have_parent = false;
    if (dense) {
        arrangement_lexbfs_warp(A32, n, sw, smem, L, ord, pos);
    } else {
        SlotMem<uint16_t, uint16_t> M;
        M.cls = (uint16_t *)(smem + L.cls);
        M.slot_v = (uint16_t *)(smem + L.slot);
        M.c_head = (uint16_t *)(smem + L.c_head);
        M.c_end = (uint16_t *)(smem + L.c_end);
        M.c_live = (uint16_t *)(smem + L.c_live);
        M.c_prev = (uint16_t *)(smem + L.c_prev);
        M.c_next = (uint16_t *)(smem + L.c_next);
        M.c_tgt = (uint16_t *)(smem + L.c_tgt);
        M.c_cnt = (uint16_t *)(smem + L.c_cnt);
        M.freel = (uint16_t *)(smem + L.freel);
        M.touched = (uint16_t *)(smem + L.touched);
        M.scratch = (uint16_t *)(smem + L.scratch);
        M.cap = L.cap;
        BitsetSource<uint16_t> src{A32, sw, W, (uint16_t *)(smem + L.nbuf)};
        slot_lexbfs<uint16_t, uint16_t, CHORDAL_TIE_ASCENDING, BitsetSource<uint16_t>, uint16_t>(src, n, M, ord, pos,
                                                                                                 par, 0, 0);
        have_parent = true;
    }
    __syncwarp();

    // ---- write the order ---------------------------------------------------
    int32_t *og = orders + g * n;
    for (int k = lane; k < n; k += 32) og[k] = ord[k];

    // ---- PEO check: lanes stride over vertices -----------------------------------
    unsigned long long best = ~0ULL;
    for (int v = lane; v < n; v += 32) {
        const int pv = pos[v];
        if (pv == 0) continue;
        const uint32_t *__restrict__ rv = A32 + v * sw;
        int parent = have_parent ? (int)(int16_t)par[v] : -2;
        if (parent == -2) {  // not produced by the search: backward scan, then full pass
            parent = -1;
            const int lim = pv > 64 ? pv - 64 : 0;
            for (int q = pv - 1; q >= lim; --q) {
                int u = ord[q];
                if ((rv[u >> 5] >> (u & 31)) & 1u) { parent = u; break; }
            }
            if (parent < 0 && lim > 0) {
                int bp = -1;
                for (int w = 0; w < W; ++w) {
                    uint32_t m = rv[w];
                    while (m) {
                        int b = __ffs(m) - 1;
                        m &= m - 1;
                        int pu = pos[32 * w + b];
                        if (pu < pv && pu > bp) bp = pu;
                    }
                }
                if (bp >= 0) parent = ord[bp];
            }
        }
        if (parent < 0) continue;
        const unsigned long long k64 = ((unsigned long long)parent << 32) | (unsigned)v;
        if (k64 >= best) continue;
        const int pp = pos[parent];
        const uint4 *rv4 = reinterpret_cast<const uint4 *>(rv);
        const uint4 *rp4 = reinterpret_cast<const uint4 *>(A32 + parent * sw);
        bool viol = false;
        // 16 words (two rows x four 128-bit loads, all in flight) per round
        for (int w0 = 0; w0 < W && !viol; w0 += 16) {
            uint32_t a[16], b[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
                if (w0 + 4 * j < W) {
                    x = __ldg(rv4 + (w0 >> 2) + j);
                    y = __ldg(rp4 + (w0 >> 2) + j);
                }
                a[4 * j] = x.x; a[4 * j + 1] = x.y; a[4 * j + 2] = x.z; a[4 * j + 3] = x.w;
                b[4 * j] = y.x; b[4 * j + 1] = y.y; b[4 * j + 2] = y.z; b[4 * j + 3] = y.w;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int w = w0 + j;
                uint32_t m = a[j] & ~b[j];
                if ((parent >> 5) == w) m &= ~(1u << (parent & 31));
                while (m && !viol) {
                    const int bb = __ffs(m) - 1;
                    m &= m - 1;
                    if (pos[32 * w + bb] < pp) viol = true;
                }
            }
        }
        if (viol) best = k64;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(CH_FULL, best, d);
        best = o < best ? o : best;
    }
    int32_t *wg = witness + 3 * g;
    if (best == ~0ULL) {
        if (lane < 3) wg[lane] = -1;
        return;
    }
    const int p = (int)(best >> 32), v = (int)(best & 0xFFFFFFFFu);
    const int pp = pos[p];
    const uint32_t *rv = A32 + v * sw, *rp = A32 + p * sw;
    uint32_t cand = 0;
    if (lane < W) {
        uint32_t m = rv[lane] & ~rp[lane];
        if ((p >> 5) == lane) m &= ~(1u << (p & 31));
        while (m) {
            int b = __ffs(m) - 1;
            m &= m - 1;
            if (pos[32 * lane + b] < pp) cand |= 1u << b;
        }
    }
    uint32_t any = __ballot_sync(CH_FULL, cand != 0);
    int src = __ffs(any) - 1;
    uint32_t c = __shfl_sync(CH_FULL, cand, src);
    if (lane == 0) {
        wg[0] = v;
        wg[1] = p;
        wg[2] = 32 * src + __ffs(c) - 1;
    }
}

int launch_batch(const uint8_t *adj, int64_t batch, int64_t n, int64_t stride, int32_t *orders,
                 int32_t *witness, cudaStream_t stream) {
    const BatchLayout L((int)n);
    if (L.total > 227 * 1024) return CHORDAL_ETOOLARGE;
    cudaError_t e = cudaFuncSetAttribute(batch_chordal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.total);
    if (e != cudaSuccess) return CHORDAL_ECUDA;
    // grid.x limit is 2^31-1: one CTA per graph
    batch_chordal_kernel<<<(unsigned)batch, 32, L.total, stream>>>(adj, (int)n, (int)stride, orders, witness);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
