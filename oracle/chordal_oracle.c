/*
 * chordal_oracle.c -- CPU restatement of the reference's chordality-test path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1508_06329_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never routes through it (there is no CPU fallback).
 *
 * Reference: /root/reference/pkg/src/chordalkit (pure Python + numpy,
 * "chordalkit" 0.1.0).  Every function below cites the file:line it restates.
 * Parity pinning: tests/golden/ holds fixtures produced by running the
 * reference itself (tests/golden/make_golden.py); tests/test_oracle_golden.py
 * checks this oracle against every one of them.
 *
 * Conventions: vertices are 0-based int32 here (the reference is 1-based at
 * its API edge and 0-based internally, graph.py:1-7).  Dense graphs are
 * packed little-endian bit rows exactly like Graph._packed (graph.py:78-88):
 * bit (j & 7) of byte (j >> 3) of row i <=> edge i-j; `stride` is the row
 * pitch in bytes (>= ceil(n/8)).  CSR graphs use int64 indptr / int32 sorted
 * indices (the adjacency_lists0() shape, graph.py:152-158).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

#define ORACLE_OK 0
#define ORACLE_ENOMEM 4

static inline int dbit(const uint8_t *row, int64_t j) { return (row[j >> 3] >> (j & 7)) & 1; }

/* ---------------------------------------------------------------------------
 * splitmix64 / mix64 -- _bitops.py:43-57
 */
uint64_t oracle_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t mix64_2(uint64_t a, uint64_t b) {
    uint64_t h = oracle_splitmix64(0 ^ a);
    return oracle_splitmix64(h ^ b);
}

static uint64_t mix64_3(uint64_t a, uint64_t b, uint64_t c) {
    return oracle_splitmix64(mix64_2(a, b) ^ c);
}

/* zlib crc32 of "current" -- label_hash, _bitops.py:77-79 */
static uint32_t crc32_str(const char *s) {
    uint32_t c = 0xFFFFFFFFu;
    for (; *s; ++s) {
        c ^= (uint8_t)*s;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return c ^ 0xFFFFFFFFu;
}

/* ---------------------------------------------------------------------------
 * Partition-refinement LexBFS over a linked vertex chain --
 * PartitionList (search.py:328-463) driven by lexbfs_partition's linked
 * method (search.py:515-532).  `members` is the initial chain order (the
 * reference passes range(n), or a shuffled list for seeded tie-breaks,
 * search.py:516-518).  Neighbours are visited in ascending id, as
 * adjacency_lists0() yields them.  Class ids are recycled through a free list
 * (the reference appends forever); ids are internal and never observable.
 */
typedef struct {
    int32_t *vprev, *vnext, *class_of;
    int32_t *cfirst, *clast, *cprev, *cnext, *csplit_iter, *csplit_target;
    int32_t *freelist;
    int32_t nfree, vhead, chead;
} plist_t;

static int plist_init(plist_t *P, int64_t n, const int32_t *members) {
    int64_t cap = 2 * n + 4;
    P->vprev = malloc(sizeof(int32_t) * (n + 1));
    P->vnext = malloc(sizeof(int32_t) * (n + 1));
    P->class_of = malloc(sizeof(int32_t) * (n + 1));
    P->cfirst = malloc(sizeof(int32_t) * cap);
    P->clast = malloc(sizeof(int32_t) * cap);
    P->cprev = malloc(sizeof(int32_t) * cap);
    P->cnext = malloc(sizeof(int32_t) * cap);
    P->csplit_iter = malloc(sizeof(int32_t) * cap);
    P->csplit_target = malloc(sizeof(int32_t) * cap);
    P->freelist = malloc(sizeof(int32_t) * cap);
    if (!P->vprev || !P->vnext || !P->class_of || !P->cfirst || !P->clast || !P->cprev ||
        !P->cnext || !P->csplit_iter || !P->csplit_target || !P->freelist)
        return ORACLE_ENOMEM;
    /* search.py:343-362 */
    int32_t prev = -1;
    for (int64_t k = 0; k < n; ++k) {
        int32_t v = members ? members[k] : (int32_t)k;
        P->vprev[v] = prev;
        P->vnext[v] = -1;
        if (prev >= 0) P->vnext[prev] = v;
        P->class_of[v] = 0;
        prev = v;
    }
    P->vhead = n ? (members ? members[0] : 0) : -1;
    P->cfirst[0] = P->vhead;
    P->clast[0] = prev;
    P->cprev[0] = -1;
    P->cnext[0] = -1;
    P->chead = 0;
    P->csplit_iter[0] = -1;
    P->csplit_target[0] = -1;
    P->nfree = 0;
    for (int64_t c = cap - 1; c >= 1; --c) P->freelist[P->nfree++] = (int32_t)c;
    return ORACLE_OK;
}

static void plist_free(plist_t *P) {
    free(P->vprev); free(P->vnext); free(P->class_of); free(P->cfirst); free(P->clast);
    free(P->cprev); free(P->cnext); free(P->csplit_iter); free(P->csplit_target); free(P->freelist);
}

/* _new_class_before, search.py:366-380 */
static int32_t plist_new_class_before(plist_t *P, int32_t c) {
    int32_t d = P->freelist[--P->nfree];
    P->cfirst[d] = -1;
    P->clast[d] = -1;
    int32_t prev = P->cprev[c];
    P->cprev[d] = prev;
    P->cnext[d] = c;
    P->cprev[c] = d;
    if (prev >= 0) P->cnext[prev] = d; else P->chead = d;
    P->csplit_iter[d] = -1;
    P->csplit_target[d] = -1;
    return d;
}

/* _unlink_class, search.py:382-389 (+ id recycling) */
static void plist_unlink_class(plist_t *P, int32_t c) {
    int32_t p = P->cprev[c], x = P->cnext[c];
    if (p >= 0) P->cnext[p] = x; else P->chead = x;
    if (x >= 0) P->cprev[x] = p;
    P->freelist[P->nfree++] = c;
}

/* _detach, search.py:393-409 */
static void plist_detach(plist_t *P, int32_t v) {
    int32_t c = P->class_of[v];
    int32_t p = P->vprev[v], x = P->vnext[v];
    if (p >= 0) P->vnext[p] = x; else P->vhead = x;
    if (x >= 0) P->vprev[x] = p;
    int sole = P->cfirst[c] == v && P->clast[c] == v;
    if (sole) { P->cfirst[c] = P->clast[c] = -1; }
    else if (P->cfirst[c] == v) P->cfirst[c] = x;
    else if (P->clast[c] == v) P->clast[c] = p;
    P->vprev[v] = P->vnext[v] = -1;
}

/* _insert_before / _insert_after, search.py:411-427 */
static void plist_insert_before(plist_t *P, int32_t v, int32_t anchor) {
    int32_t p = P->vprev[anchor];
    P->vprev[v] = p;
    P->vnext[v] = anchor;
    P->vprev[anchor] = v;
    if (p >= 0) P->vnext[p] = v; else P->vhead = v;
}

static void plist_insert_after(plist_t *P, int32_t v, int32_t anchor) {
    int32_t x = P->vnext[anchor];
    P->vnext[v] = x;
    P->vprev[v] = anchor;
    P->vnext[anchor] = v;
    if (x >= 0) P->vprev[x] = v;
}

/* pop_first, search.py:431-438 */
static int32_t plist_pop_first(plist_t *P) {
    int32_t c = P->chead;
    int32_t x = P->cfirst[c];
    plist_detach(P, x);
    if (P->cfirst[c] == -1) plist_unlink_class(P, c);
    P->class_of[x] = -1;
    return x;
}

/* move_to_splitter, search.py:440-463 */
static void plist_move_to_splitter(plist_t *P, int32_t y, int32_t iteration) {
    int32_t c = P->class_of[y];
    int32_t d;
    if (P->csplit_iter[c] != iteration) {
        d = plist_new_class_before(P, c);
        P->csplit_iter[c] = iteration;
        P->csplit_target[c] = d;
    } else {
        d = P->csplit_target[c];
    }
    if (P->cfirst[c] == y && P->clast[c] == y && P->cfirst[d] == -1) {
        P->class_of[y] = d;
        P->cfirst[d] = P->clast[d] = y;
        plist_unlink_class(P, c);
        return;
    }
    plist_detach(P, y);
    if (P->cfirst[d] == -1) {
        plist_insert_before(P, y, P->cfirst[c]);
        P->cfirst[d] = P->clast[d] = y;
    } else {
        plist_insert_after(P, y, P->clast[d]);
        P->clast[d] = y;
    }
    P->class_of[y] = d;
    if (P->cfirst[c] == -1) plist_unlink_class(P, c);
}

/* lexbfs_partition(g, method="linked") on packed rows, search.py:515-532 */
int oracle_lexbfs_partition(const uint8_t *adj, int64_t n, int64_t stride,
                            const int32_t *members, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    plist_t P;
    if (plist_init(&P, n, members) != ORACLE_OK) { plist_free(&P); return ORACLE_ENOMEM; }
    uint8_t *visited = calloc((size_t)n, 1);
    if (!visited) { plist_free(&P); return ORACLE_ENOMEM; }
    int64_t rowbytes = (n + 7) >> 3;
    for (int64_t i = 1; i <= n; ++i) {
        int32_t x = plist_pop_first(&P);
        visited[x] = 1;
        order[i - 1] = x;
        const uint8_t *row = adj + (int64_t)x * stride;
        for (int64_t b = 0; b < rowbytes; ++b) {
            uint8_t byte = row[b];
            while (byte) {
                int k = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t y = (b << 3) + k;
                if (y < n && !visited[y]) plist_move_to_splitter(&P, (int32_t)y, (int32_t)i);
            }
        }
    }
    free(visited);
    plist_free(&P);
    return ORACLE_OK;
}

/* Same algorithm on CSR adjacency -- the duck-typed CSR shim of SURVEY 8(c),
 * i.e. lexbfs_partition(g, method="linked") fed by adjacency_lists0(). */
int oracle_lexbfs_partition_csr(const int64_t *indptr, const int32_t *indices, int64_t n,
                                int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    plist_t P;
    if (plist_init(&P, n, NULL) != ORACLE_OK) { plist_free(&P); return ORACLE_ENOMEM; }
    uint8_t *visited = calloc((size_t)n, 1);
    if (!visited) { plist_free(&P); return ORACLE_ENOMEM; }
    for (int64_t i = 1; i <= n; ++i) {
        int32_t x = plist_pop_first(&P);
        visited[x] = 1;
        order[i - 1] = x;
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t y = indices[e];
            if (!visited[y]) plist_move_to_splitter(&P, y, (int32_t)i);
        }
    }
    free(visited);
    plist_free(&P);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * numpy's Philox4x64-10 bit generator and the two Generator draws the seeded
 * linked LexBFS variants use (rng.py:18-21: key = mix64(seed, crc32(label)),
 * 256-bit counter starting at 0, incremented before each 4-word block;
 * next_uint32 hands out the low then the high half of a 64-bit output and
 * keeps the other half buffered across calls).
 *   random_interval(max)   masked rejection (Generator.shuffle's Fisher-Yates)
 *   bounded(rng)           Lemire 32-bit rejection (Generator.integers)
 */
typedef struct {
    uint64_t key, ctr, blk[4];
    int pos, has32;
    uint32_t u32;
} philox_t;

static void philox_init(philox_t *r, uint64_t key) {
    memset(r, 0, sizeof *r);
    r->key = key;
    r->pos = 4;
}

static uint64_t philox_next64(philox_t *r) {
    if (r->pos >= 4) {
        uint64_t c[4] = {++r->ctr, 0, 0, 0}, k0 = r->key, k1 = 0;
        for (int i = 0; i < 10; ++i) {
            __uint128_t p0 = (__uint128_t)0xD2E7470EE14C6C93ULL * c[0];
            __uint128_t p1 = (__uint128_t)0xCA5A826395121157ULL * c[2];
            uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
            uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
            uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
            c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        memcpy(r->blk, c, sizeof c);
        r->pos = 0;
    }
    return r->blk[r->pos++];
}

static uint32_t philox_next32(philox_t *r) {
    if (r->has32) { r->has32 = 0; return r->u32; }
    uint64_t x = philox_next64(r);
    r->has32 = 1;
    r->u32 = (uint32_t)(x >> 32);
    return (uint32_t)x;
}

static uint32_t philox_interval(philox_t *r, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max, v;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    while ((v = philox_next32(r) & mask) > max) {
    }
    return v;
}

static uint32_t philox_bounded(philox_t *r, uint32_t rng) { /* [0, rng], rng < 2^32 - 1 */
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)philox_next32(r) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        const uint32_t th = (0xFFFFFFFFu - rng) % excl;
        while (left < th) {
            m = (uint64_t)philox_next32(r) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

static uint64_t stream_key(uint64_t seed, const char *label) {
    return oracle_splitmix64(oracle_splitmix64(seed) ^ (uint64_t)crc32_str(label));
}

/* lexbfs_partition(g, seeded(seed), method="linked"), search.py:515-532: the
 * members are range(n) after Generator.shuffle (Fisher-Yates, i = n-1..1,
 * j = random_interval(i)) on the stream (seed, "lexbfs-partition"). */
int oracle_lexbfs_partition_seeded(const uint8_t *adj, int64_t n, int64_t stride, uint64_t seed,
                                   int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    int32_t *members = malloc(sizeof(int32_t) * (size_t)n);
    if (!members) return ORACLE_ENOMEM;
    for (int64_t k = 0; k < n; ++k) members[k] = (int32_t)k;
    philox_t r;
    philox_init(&r, stream_key(seed, "lexbfs-partition"));
    for (int64_t i = n - 1; i >= 1; --i) {
        uint32_t j = philox_interval(&r, (uint32_t)i);
        int32_t t = members[i];
        members[i] = members[j];
        members[j] = t;
    }
    int rc = oracle_lexbfs_partition(adj, n, stride, members, order);
    free(members);
    return rc;
}

/* lexbfs_labels(g, seeded(seed), method="linked"), search.py:283-310: the
 * pivot is member Generator.integers(|C|) of the max-label class C in chain
 * order.  The chain starts as range(n) and receives movers in adjacency
 * order, so every class lists its members by ascending id -- the order of a
 * PartitionList started from range(n), whose first class is the chain tail. */
int oracle_lexbfs_labels_seeded(const uint8_t *adj, int64_t n, int64_t stride, uint64_t seed, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    plist_t P;
    if (plist_init(&P, n, NULL) != ORACLE_OK) { plist_free(&P); return ORACLE_ENOMEM; }
    uint8_t *visited = calloc((size_t)n, 1);
    if (!visited) { plist_free(&P); return ORACLE_ENOMEM; }
    philox_t r;
    philox_init(&r, stream_key(seed, "lexbfs-labels"));
    int64_t rowbytes = (n + 7) >> 3;
    for (int64_t i = 1; i <= n; ++i) {
        int32_t c = P.chead, size = 0;
        for (int32_t v = P.cfirst[c];; v = P.vnext[v]) {
            ++size;
            if (v == P.clast[c]) break;
        }
        uint32_t k = philox_bounded(&r, (uint32_t)(size - 1));
        int32_t x = P.cfirst[c];
        while (k--) x = P.vnext[x];
        plist_detach(&P, x);  /* detach_vertex, search.py:215-227 */
        if (P.cfirst[c] == -1) plist_unlink_class(&P, c);
        P.class_of[x] = -1;
        visited[x] = 1;
        order[i - 1] = x;
        const uint8_t *row = adj + (int64_t)x * stride;
        for (int64_t b = 0; b < rowbytes; ++b) {
            uint8_t byte = row[b];
            while (byte) {
                int kk = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t y = (b << 3) + kk;
                if (y < n && !visited[y]) plist_move_to_splitter(&P, (int32_t)y, (int32_t)i);
            }
        }
    }
    free(visited);
    plist_free(&P);
    return ORACLE_OK;
}

/* mcs_order, search.py:113-145: scan for the unvisited vertex of largest
 * weight (first = smallest id); seeded: ties[integers(len(ties))] on the
 * stream (seed, "mcs").  O(n^2 / 8 + n^2) like the reference. */
int oracle_mcs_order(const uint8_t *adj, int64_t n, int64_t stride, int seeded, uint64_t seed, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    int32_t *weight = calloc((size_t)n, sizeof(int32_t)), *ties = malloc(sizeof(int32_t) * (size_t)n);
    uint8_t *done = calloc((size_t)n, 1);
    if (!weight || !ties || !done) { free(weight); free(ties); free(done); return ORACLE_ENOMEM; }
    philox_t r;
    philox_init(&r, stream_key(seed, "mcs"));
    for (int64_t i = 0; i < n; ++i) {
        int32_t best = -1, x = -1, nt = 0;
        for (int32_t v = 0; v < n; ++v) {
            if (done[v]) continue;
            if (weight[v] > best) { best = weight[v]; x = v; nt = 0; ties[nt++] = v; }
            else if (weight[v] == best) ties[nt++] = v;
        }
        if (seeded) x = ties[philox_bounded(&r, (uint32_t)(nt - 1))];
        done[x] = 1;
        order[i] = x;
        const uint8_t *row = adj + (int64_t)x * stride;
        for (int32_t y = 0; y < n; ++y)
            if (dbit(row, y) && !done[y]) ++weight[y];
    }
    free(weight); free(ties); free(done);
    return ORACLE_OK;
}

/* bfs_order, search.py:79-110: FIFO queue, restarts at the smallest unqueued
 * vertex; seeded: restart at pool[integers(len(pool))], fresh neighbours
 * shuffled (Fisher-Yates, random_interval) on the stream (seed, "bfs"). */
int oracle_bfs_order(const uint8_t *adj, int64_t n, int64_t stride, int seeded, uint64_t seed, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    uint8_t *queued = calloc((size_t)n, 1);
    if (!queued) return ORACLE_ENOMEM;
    philox_t r;
    philox_init(&r, stream_key(seed, "bfs"));
    int64_t head = 0, tail = 0, next_start = 0, nq = 0;
    while (head < n) {
        if (head == tail) {
            int64_t s;
            if (!seeded) {
                while (queued[next_start]) ++next_start;
                s = next_start;
            } else {
                uint32_t k = philox_bounded(&r, (uint32_t)(n - nq - 1));
                for (s = 0;; ++s)
                    if (!queued[s] && k-- == 0) break;
            }
            queued[s] = 1;
            order[tail++] = (int32_t)s;
            ++nq;
        }
        int32_t x = order[head++];
        int64_t t0 = tail;
        const uint8_t *row = adj + (int64_t)x * stride;
        for (int32_t y = 0; y < n; ++y)
            if (dbit(row, y) && !queued[y]) { queued[y] = 1; order[tail++] = y; }
        if (seeded && tail - t0 > 1)
            for (int64_t i = tail - t0 - 1; i >= 1; --i) {
                uint32_t j = philox_interval(&r, (uint32_t)i);
                int32_t tmp = order[t0 + i];
                order[t0 + i] = order[t0 + j];
                order[t0 + j] = tmp;
            }
        nq += tail - t0;
    }
    free(queued);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * Array partition refinement -- lexbfs_array, _arraylex.py:22-65.  Ties are
 * broken by position in `initial` (identity => LOWEST_INDEX; a Philox
 * permutation => the seeded array path, search.py:535-541).
 */
int oracle_lexbfs_array(const uint8_t *adj, int64_t n, int64_t stride,
                        const int32_t *initial, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    int64_t ccap = 2 * n + 4;
    int32_t *arr = malloc(sizeof(int32_t) * n);
    int32_t *class_id = calloc((size_t)n, sizeof(int32_t));
    int32_t *starts = malloc(sizeof(int32_t) * ccap);
    int32_t *ends = malloc(sizeof(int32_t) * ccap);
    int32_t *touched = malloc(sizeof(int32_t) * ccap);
    int32_t *tmark = calloc((size_t)ccap, sizeof(int32_t));
    int32_t *ys = malloc(sizeof(int32_t) * n);
    int32_t *win = malloc(sizeof(int32_t) * n);
    uint8_t *flag = calloc((size_t)n, 1);
    uint8_t *visited = calloc((size_t)n, 1);
    if (!arr || !class_id || !starts || !ends || !touched || !tmark || !ys || !win || !flag || !visited) {
        free(arr); free(class_id); free(starts); free(ends); free(touched); free(tmark);
        free(ys); free(win); free(flag); free(visited);
        return ORACLE_ENOMEM;
    }
    for (int64_t k = 0; k < n; ++k) arr[k] = initial ? initial[k] : (int32_t)k;
    int64_t nclass = 1;
    starts[0] = 0;
    ends[0] = (int32_t)n;
    int64_t rowbytes = (n + 7) >> 3;
    for (int64_t i = 0; i < n; ++i) {
        int32_t x = arr[i];
        order[i] = x;
        visited[x] = 1;
        starts[class_id[x]] += 1;
        const uint8_t *row = adj + (int64_t)x * stride;
        int64_t ny = 0;
        for (int64_t b = 0; b < rowbytes; ++b) {
            uint8_t byte = row[b];
            while (byte) {
                int k = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t y = (b << 3) + k;
                if (y < n && !visited[y]) ys[ny++] = (int32_t)y;
            }
        }
        if (ny == 0) continue;
        /* np.unique(class_id[ys]) -- windows are disjoint, so visiting the
         * touched classes in first-touch order gives the same result. */
        int64_t nt = 0;
        for (int64_t k = 0; k < ny; ++k) {
            flag[ys[k]] = 1;
            int32_t c = class_id[ys[k]];
            if (tmark[c] != (int32_t)(i + 1)) { tmark[c] = (int32_t)(i + 1); touched[nt++] = c; }
        }
        for (int64_t t = 0; t < nt; ++t) {
            int32_t c = touched[t];
            int32_t s = starts[c], e = ends[c];
            if (e - s <= 1) continue;
            int32_t kf = 0;
            for (int32_t q = s; q < e; ++q) { win[q - s] = arr[q]; kf += flag[arr[q]]; }
            if (kf == e - s) continue;
            int32_t a = s, bpos = s + kf;
            for (int32_t q = 0; q < e - s; ++q) {
                if (flag[win[q]]) arr[a++] = win[q]; else arr[bpos++] = win[q];
            }
            int64_t nc = nclass++;
            starts[nc] = s;
            ends[nc] = s + kf;
            for (int32_t q = s; q < s + kf; ++q) class_id[arr[q]] = (int32_t)nc;
            starts[c] = s + kf;
        }
        for (int64_t k = 0; k < ny; ++k) flag[ys[k]] = 0;
    }
    free(arr); free(class_id); free(starts); free(ends); free(touched); free(tmark);
    free(ys); free(win); free(flag); free(visited);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * Barrier-phase LexBFS election rule -- parallel_lexbfs (parallel/lexbfs.py:
 * 234-262).  Current starts at vertex 1 (lexbfs.py:173); at iteration i the
 * electors are the members of the tail (max-label) set (lexbfs.py:211-225)
 * and Arbitration picks the winner (engine.py:47-53):
 *   mode 0 fixed ascending  -> min id,   mode 1 fixed descending -> max id,
 *   mode 2 seeded(s) -> argmax_w (splitmix64(prefix_i ^ w), w), w 1-based,
 *   prefix_i = mix64(s, 4(i-1)+3, mix64(crc32("current"), 0)).
 * The set structure is kept as the same array refinement as above (a label
 * class is a window; which member heads it is irrelevant because the rule
 * picks from the whole window).
 */
int oracle_lexbfs_arbitrated(const uint8_t *adj, int64_t n, int64_t stride, int mode,
                             uint64_t seed, int32_t *order) {
    if (n <= 0) return ORACLE_OK;
    int64_t ccap = 2 * n + 4;
    int32_t *arr = malloc(sizeof(int32_t) * n);
    int32_t *class_id = calloc((size_t)n, sizeof(int32_t));
    int32_t *starts = malloc(sizeof(int32_t) * ccap);
    int32_t *ends = malloc(sizeof(int32_t) * ccap);
    int32_t *touched = malloc(sizeof(int32_t) * ccap);
    int32_t *tmark = calloc((size_t)ccap, sizeof(int32_t));
    int32_t *ys = malloc(sizeof(int32_t) * n);
    int32_t *win = malloc(sizeof(int32_t) * n);
    uint8_t *flag = calloc((size_t)n, 1);
    uint8_t *visited = calloc((size_t)n, 1);
    if (!arr || !class_id || !starts || !ends || !touched || !tmark || !ys || !win || !flag || !visited) {
        free(arr); free(class_id); free(starts); free(ends); free(touched); free(tmark);
        free(ys); free(win); free(flag); free(visited);
        return ORACLE_ENOMEM;
    }
    for (int64_t k = 0; k < n; ++k) arr[k] = (int32_t)k;
    int64_t nclass = 1;
    starts[0] = 0;
    ends[0] = (int32_t)n;
    uint64_t cell = mix64_2(crc32_str("current"), 0);
    int64_t rowbytes = (n + 7) >> 3;
    for (int64_t i = 0; i < n; ++i) {
        if (i > 0) {
            /* elect within the head window [i, end of its class) */
            int32_t c0 = class_id[arr[i]];
            int32_t s = starts[c0], e = ends[c0];
            int32_t best = s;
            if (mode == 0) {
                for (int32_t q = s; q < e; ++q) if (arr[q] < arr[best]) best = q;
            } else if (mode == 1) {
                for (int32_t q = s; q < e; ++q) if (arr[q] > arr[best]) best = q;
            } else {
                /* iteration i (1-based) elects position i+1 at epoch 4(i-1)+3 */
                uint64_t prefix = mix64_3(seed, (uint64_t)(4 * (i - 1) + 3), cell);
                uint64_t bk = oracle_splitmix64(prefix ^ (uint64_t)(arr[best] + 1));
                for (int32_t q = s; q < e; ++q) {
                    uint64_t k = oracle_splitmix64(prefix ^ (uint64_t)(arr[q] + 1));
                    if (k > bk || (k == bk && arr[q] > arr[best])) { bk = k; best = q; }
                }
            }
            int32_t tmp = arr[s]; arr[s] = arr[best]; arr[best] = tmp;
        }
        int32_t x = arr[i];
        order[i] = x;
        visited[x] = 1;
        starts[class_id[x]] += 1;
        const uint8_t *row = adj + (int64_t)x * stride;
        int64_t ny = 0;
        for (int64_t b = 0; b < rowbytes; ++b) {
            uint8_t byte = row[b];
            while (byte) {
                int k = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t y = (b << 3) + k;
                if (y < n && !visited[y]) ys[ny++] = (int32_t)y;
            }
        }
        if (ny == 0) continue;
        int64_t nt = 0;
        for (int64_t k = 0; k < ny; ++k) {
            flag[ys[k]] = 1;
            int32_t c = class_id[ys[k]];
            if (tmark[c] != (int32_t)(i + 1)) { tmark[c] = (int32_t)(i + 1); touched[nt++] = c; }
        }
        for (int64_t t = 0; t < nt; ++t) {
            int32_t c = touched[t];
            int32_t s = starts[c], e = ends[c];
            if (e - s <= 1) continue;
            int32_t kf = 0;
            for (int32_t q = s; q < e; ++q) { win[q - s] = arr[q]; kf += flag[arr[q]]; }
            if (kf == e - s) continue;
            int32_t a = s, bpos = s + kf;
            for (int32_t q = 0; q < e - s; ++q) {
                if (flag[win[q]]) arr[a++] = win[q]; else arr[bpos++] = win[q];
            }
            int64_t nc = nclass++;
            starts[nc] = s;
            ends[nc] = s + kf;
            for (int32_t q = s; q < s + kf; ++q) class_id[arr[q]] = (int32_t)nc;
            starts[c] = s + kf;
        }
        for (int64_t k = 0; k < ny; ++k) flag[ys[k]] = 0;
    }
    free(arr); free(class_id); free(starts); free(ends); free(touched); free(tmark);
    free(ys); free(win); free(flag); free(visited);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * PEO test with the deterministic first witness -- _is_peo_lists
 * (peo.py:100-149); identical result to peo_holds_array + _first_witness_big
 * (_arraylex.py:104-124, peo.py:152-174).
 *   scan 1: parent[v] = left neighbour with the greatest position (peo.py:106-121)
 *   scans 2-4: for x ascending, mark ln[x]; for children y of x (y in adj[x]
 *   ascending with parent[y] == x), the first z in ln[y] (ascending) with
 *   z != x and z not marked is the witness (v=y, p=x, z) (peo.py:124-142).
 * Writes witness[0..2] = (v, p, z) 0-based, or (-1,-1,-1) for a PEO.
 * Returns 1 if `order` is a PEO, 0 if not, <0 on allocation failure.
 */
int oracle_is_peo(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *order,
                  int32_t *witness) {
    witness[0] = witness[1] = witness[2] = -1;
    if (n <= 0) return 1;
    int32_t *pos = malloc(sizeof(int32_t) * n);
    int32_t *parent = malloc(sizeof(int32_t) * n);
    if (!pos || !parent) { free(pos); free(parent); return -ORACLE_ENOMEM; }
    for (int64_t k = 0; k < n; ++k) pos[order[k]] = (int32_t)k;
    int64_t rowbytes = (n + 7) >> 3;
    /* scan 1 */
    for (int64_t v = 0; v < n; ++v) {
        const uint8_t *row = adj + v * stride;
        int32_t best = -1, best_pos = -1;
        for (int64_t b = 0; b < rowbytes; ++b) {
            uint8_t byte = row[b];
            while (byte) {
                int k = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t w = (b << 3) + k;
                if (w < n && pos[w] < pos[v] && pos[w] > best_pos) { best_pos = pos[w]; best = (int32_t)w; }
            }
        }
        parent[v] = best;
    }
    /* scans 2-4: "visited" = ln[x] membership, tested on the fly */
    int ok = 1;
    for (int64_t x = 0; x < n && ok; ++x) {
        const uint8_t *rowx = adj + x * stride;
        for (int64_t b = 0; b < rowbytes && ok; ++b) {
            uint8_t byte = rowx[b];
            while (byte && ok) {
                int k = __builtin_ctz(byte);
                byte &= (uint8_t)(byte - 1);
                int64_t y = (b << 3) + k;
                if (y >= n || parent[y] != x) continue;
                const uint8_t *rowy = adj + y * stride;
                for (int64_t zb = 0; zb < rowbytes && ok; ++zb) {
                    uint8_t zbyte = rowy[zb];
                    while (zbyte) {
                        int kk = __builtin_ctz(zbyte);
                        zbyte &= (uint8_t)(zbyte - 1);
                        int64_t z = (zb << 3) + kk;
                        if (z >= n || pos[z] >= pos[y]) continue; /* z in ln[y] */
                        int marked = dbit(rowx, z) && pos[z] < pos[x]; /* z in ln[x] */
                        if (z != x && !marked) {
                            witness[0] = (int32_t)y;
                            witness[1] = (int32_t)x;
                            witness[2] = (int32_t)z;
                            ok = 0;
                            break;
                        }
                    }
                }
            }
        }
    }
    free(pos);
    free(parent);
    return ok;
}

/* _is_peo_lists on CSR adjacency (literal list form, peo.py:100-149) */
int oracle_is_peo_csr(const int64_t *indptr, const int32_t *indices, int64_t n,
                      const int32_t *order, int32_t *witness) {
    witness[0] = witness[1] = witness[2] = -1;
    if (n <= 0) return 1;
    int32_t *pos = malloc(sizeof(int32_t) * n);
    int32_t *parent = malloc(sizeof(int32_t) * n);
    uint8_t *visited = calloc((size_t)n, 1);
    if (!pos || !parent || !visited) { free(pos); free(parent); free(visited); return -ORACLE_ENOMEM; }
    for (int64_t k = 0; k < n; ++k) pos[order[k]] = (int32_t)k;
    for (int64_t v = 0; v < n; ++v) {
        int32_t best = -1, best_pos = -1;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t w = indices[e];
            if (pos[w] < pos[v] && pos[w] > best_pos) { best_pos = pos[w]; best = w; }
        }
        parent[v] = best;
    }
    int ok = 1;
    for (int64_t x = 0; x < n && ok; ++x) {
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t w = indices[e];
            if (pos[w] < pos[x]) visited[w] = 1;
        }
        for (int64_t e = indptr[x]; e < indptr[x + 1] && ok; ++e) {
            int32_t y = indices[e];
            if (parent[y] != x) continue;
            for (int64_t f = indptr[y]; f < indptr[y + 1]; ++f) {
                int32_t z = indices[f];
                if (pos[z] >= pos[y]) continue;
                if (z != x && !visited[z]) {
                    witness[0] = y; witness[1] = (int32_t)x; witness[2] = z;
                    ok = 0;
                    break;
                }
            }
        }
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t w = indices[e];
            if (pos[w] < pos[x]) visited[w] = 0;
        }
    }
    free(pos); free(parent); free(visited);
    return ok;
}

/* _is_peo_lists with its instrumentation (peo.py:100-149), literally: the
 * list-element reads of the four scans (ScanStats.reads, peo.py:48-56,
 * 146-148), and scan 1's parents and left-list sizes -- what
 * left_neighborhoods (graph.py:284-302) defines as parent(v) and |LN(v)|.
 * parent_out / ln_size_out / reads_out may be NULL. */
int oracle_peo_lists_stats(const int64_t *indptr, const int32_t *indices, int64_t n, const int32_t *order,
                           int32_t *witness, int32_t *parent_out, int32_t *ln_size_out, int64_t *reads_out) {
    witness[0] = witness[1] = witness[2] = -1;
    if (reads_out) *reads_out = 0;
    if (n <= 0) return 1;
    int32_t *pos = malloc(sizeof(int32_t) * n);
    int32_t *parent = malloc(sizeof(int32_t) * n);
    int32_t *lnsz = calloc((size_t)n, sizeof(int32_t));
    uint8_t *visited = calloc((size_t)n, 1);
    if (!pos || !parent || !lnsz || !visited) {
        free(pos); free(parent); free(lnsz); free(visited);
        return -ORACLE_ENOMEM;
    }
    for (int64_t k = 0; k < n; ++k) pos[order[k]] = (int32_t)k;
    int64_t reads = 0;
    /* scan 1 (peo.py:106-121) */
    for (int64_t v = 0; v < n; ++v) {
        int32_t best = -1, best_pos = -1;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t w = indices[e];
            reads += 1;
            if (pos[w] < pos[v]) {
                lnsz[v] += 1;
                if (pos[w] > best_pos) { best_pos = pos[w]; best = w; }
            }
        }
        parent[v] = best;
    }
    /* scans 2-4 (peo.py:124-145); ln[y] holds y's left neighbours in adjacency order */
    int ok = 1;
    for (int64_t x = 0; x < n && ok; ++x) {
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t w = indices[e];
            if (pos[w] < pos[x]) { visited[w] = 1; reads += 1; }
        }
        for (int64_t e = indptr[x]; e < indptr[x + 1] && ok; ++e) {
            int32_t y = indices[e];
            reads += 1;
            if (parent[y] != x) continue;
            for (int64_t f = indptr[y]; f < indptr[y + 1]; ++f) {
                int32_t z = indices[f];
                if (pos[z] >= pos[y]) continue;
                reads += 1;
                if (z != x && !visited[z]) {
                    witness[0] = y; witness[1] = (int32_t)x; witness[2] = z;
                    ok = 0;
                    break;
                }
            }
        }
        if (!ok) break;
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t w = indices[e];
            if (pos[w] < pos[x]) { visited[w] = 0; reads += 1; }
        }
    }
    if (parent_out) memcpy(parent_out, parent, sizeof(int32_t) * n);
    if (ln_size_out) memcpy(ln_size_out, lnsz, sizeof(int32_t) * n);
    if (reads_out) *reads_out = reads;
    free(pos); free(parent); free(lnsz); free(visited);
    return ok;
}

/* ---------------------------------------------------------------------------
 * is_chordal (peo.py:177-202) over a batch of independent dense graphs, with
 * `nthreads` host threads (the CPU baseline for the batched configuration).
 * Graph b lives at adj + b * graph_bytes.  verdict[b] = 1 chordal / 0 not.
 */
typedef struct {
    const uint8_t *adj;
    int64_t batch, n, stride, graph_bytes;
    int32_t *orders, *witness, *verdict;
    int64_t next;
    pthread_mutex_t lock;
    int err;
} batch_job_t;

static void *batch_worker(void *arg) {
    batch_job_t *J = (batch_job_t *)arg;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        int64_t b = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (b >= J->batch) break;
        const uint8_t *g = J->adj + b * J->graph_bytes;
        int32_t *ord = J->orders + b * J->n;
        int r = oracle_lexbfs_partition(g, J->n, J->stride, NULL, ord);
        if (r == ORACLE_OK) r = oracle_is_peo(g, J->n, J->stride, ord, J->witness + 3 * b);
        else r = -1;
        if (r < 0) { pthread_mutex_lock(&J->lock); J->err = 1; pthread_mutex_unlock(&J->lock); continue; }
        J->verdict[b] = r;
    }
    return NULL;
}

int oracle_is_chordal_batch(const uint8_t *adj, int64_t batch, int64_t n, int64_t stride,
                            int64_t graph_bytes, int32_t *orders, int32_t *witness,
                            int32_t *verdict, int nthreads) {
    batch_job_t J = {adj, batch, n, stride, graph_bytes, orders, witness, verdict, 0,
                     PTHREAD_MUTEX_INITIALIZER, 0};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t tid[1024];
    for (int t = 1; t < nthreads; ++t) pthread_create(&tid[t], NULL, batch_worker, &J);
    batch_worker(&J);
    for (int t = 1; t < nthreads; ++t) pthread_join(tid[t], NULL);
    return J.err ? ORACLE_ENOMEM : ORACLE_OK;
}

int oracle_max_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* ---------------------------------------------------------------------------
 * The benchmark generators, so that the CPU legs of bench.py draw their inputs
 * without the product library.  Streams: rng.stream(seed, label) (rng.py:18-21).
 *
 * gen_dense_random (generate.py:32-56): one Generator.random() double per cell
 * of each 1024-row block, row-major over full rows, so draw number u*n + v
 * decides edge {u, v} for u < v; random() = (next64 >> 11) * 2^-53.
 */
int oracle_gen_dense_random(int64_t n, double p, uint64_t seed, int64_t stride, uint8_t *out) {
    memset(out, 0, (size_t)(n * stride));
    if (n <= 1) return ORACLE_OK;
    philox_t r;
    philox_init(&r, stream_key(seed, "dense-random"));
    /* draws below the diagonal are skipped by seeking the counter: numpy's
     * Philox increments it before each 4-word block, so draw k is word k % 4
     * of block k / 4 + 1 */
    for (int64_t u = 0; u + 1 < n; ++u) {
        int64_t kk = u * n + u + 1;
        r.ctr = (uint64_t)(kk >> 2);
        r.pos = 4;
        philox_next64(&r);
        r.pos = (int)(kk & 3);
        for (int64_t v = u + 1; v < n; ++v) {
            double d = (double)(philox_next64(&r) >> 11) * (1.0 / 9007199254740992.0);
            if (d < p) {
                out[u * stride + (v >> 3)] |= (uint8_t)(1u << (v & 7));
                out[v * stride + (u >> 3)] |= (uint8_t)(1u << (u & 7));
            }
        }
    }
    return ORACLE_OK;
}

/* gen_chordal_random (generate.py:118-155).  Draws, as numpy's Generator makes
 * them:
 *   integers(-1, 2)  = -1 + bounded(2)         (random_bounded_uint64, Lemire)
 *   integers(0, i)   = bounded(i - 1)
 *   choice(P, size=w, replace=False), P <= 10000: Floyd's algorithm over
 *     j = P-w .. P-1 with an open-addressing set of 2^ceil(log2(1.2 w)) slots
 *     (a collision takes j itself), then Fisher-Yates over the w picks with
 *     bounded(t) for t = w-1 .. 1.
 * Vertex i attaches to pool[idx] for the picked idx, pool = cliques[j] ++ [j]. */
int oracle_gen_chordal_random(int64_t n, int64_t k, uint64_t seed, int64_t stride, uint8_t *out) {
    memset(out, 0, (size_t)(n * stride));
    if (k == 0 || n <= 1) return ORACLE_OK;
    int setsize = (int)(1.2 * (double)(k + 2)), mask0 = setsize;
    mask0 |= mask0 >> 1; mask0 |= mask0 >> 2; mask0 |= mask0 >> 4; mask0 |= mask0 >> 8; mask0 |= mask0 >> 16;
    int32_t *att_off = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *att_len = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *hs = malloc(sizeof(int32_t) * (size_t)(mask0 + 1));
    /* vertex i keeps min(i, k + 1) entries */
    int32_t *lst = malloc(sizeof(int32_t) * (size_t)(n * (k + 1) + 4));
    if (!att_off || !att_len || !hs || !lst) {
        free(att_off); free(att_len); free(hs); free(lst);
        return ORACLE_ENOMEM;
    }
    philox_t r;
    philox_init(&r, stream_key(seed, "chordal-random"));
#define SET_EDGE(a, b)                                                      \
    do {                                                                    \
        out[(int64_t)(a) * stride + ((b) >> 3)] |= (uint8_t)(1u << ((b) & 7)); \
        out[(int64_t)(b) * stride + ((a) >> 3)] |= (uint8_t)(1u << ((a) & 7)); \
    } while (0)
    int64_t top = 0;
    att_off[0] = 0;
    att_len[0] = 0;
    for (int64_t i = 1; i < n; ++i) {
        int32_t *o = lst + top;
        int cnt;
        if (k >= i) { /* join the whole prefix clique, no draws */
            for (int c = 0; c < i; ++c) { o[c] = c; SET_EDGE(i, c); }
            cnt = (int)i;
        } else {
            int64_t want = k - 1 + (int64_t)philox_bounded(&r, 2);
            if (want < 1) want = 1;
            if (want > i) want = i;
            const int j = (int)philox_bounded(&r, (uint32_t)(i - 1));
            const int32_t *src = lst + att_off[j];
            const int plen = att_len[j], P = plen + 1;
            if (want >= P) {
                for (int c = 0; c < plen; ++c) { o[c] = src[c]; SET_EDGE(i, src[c]); }
                o[plen] = j;
                SET_EDGE(i, j);
                cnt = P;
            } else {
                const int w = (int)want;
                int mask = (int)(1.2 * (double)w);
                mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
                for (int t = 0; t <= mask; ++t) hs[t] = -1;
                for (int jj = P - w; jj < P; ++jj) {
                    int val = (int)philox_bounded(&r, (uint32_t)jj);
                    int loc = val & mask;
                    while (hs[loc] != -1 && hs[loc] != val) loc = (loc + 1) & mask;
                    if (hs[loc] == -1) {
                        hs[loc] = val;
                        o[jj - P + w] = val;
                    } else {
                        loc = jj & mask;
                        while (hs[loc] != -1) loc = (loc + 1) & mask;
                        hs[loc] = jj;
                        o[jj - P + w] = jj;
                    }
                }
                for (int t = w - 1; t >= 1; --t) {
                    int rr = (int)philox_bounded(&r, (uint32_t)t);
                    int tmp = o[rr]; o[rr] = o[t]; o[t] = tmp;
                }
                for (int c = 0; c < w; ++c) {
                    int v = o[c] < plen ? src[o[c]] : j;
                    o[c] = v;
                    SET_EDGE(i, v);
                }
                cnt = w;
            }
        }
        att_off[i] = (int32_t)top;
        att_len[i] = cnt;
        top += cnt;
    }
#undef SET_EDGE
    free(att_off); free(att_len); free(hs); free(lst);
    return ORACLE_OK;
}

/* Configuration 4's batch: seed s in [seed_lo, seed_lo + count):
 * gen_dense_random(n, p, s) if s is even, else gen_chordal_random(n, k, s),
 * graph s - seed_lo at out + (s - seed_lo) * n * stride; nthreads host threads. */
typedef struct {
    int64_t n, k, seed_lo, count, stride, next;
    double p;
    uint8_t *out;
    pthread_mutex_t lock;
    int err;
} gen_job_t;

static void *gen_worker(void *arg) {
    gen_job_t *J = (gen_job_t *)arg;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        int64_t b = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (b >= J->count) break;
        int64_t s = J->seed_lo + b;
        uint8_t *g = J->out + b * J->n * J->stride;
        int rc = (s % 2 == 0) ? oracle_gen_dense_random(J->n, J->p, (uint64_t)s, J->stride, g)
                              : oracle_gen_chordal_random(J->n, J->k, (uint64_t)s, J->stride, g);
        if (rc) { pthread_mutex_lock(&J->lock); J->err = rc; pthread_mutex_unlock(&J->lock); }
    }
    return NULL;
}

int oracle_gen_config4_batch(int64_t n, double p, int64_t k, int64_t seed_lo, int64_t count, int64_t stride,
                             uint8_t *out, int nthreads) {
    gen_job_t J = {n, k, seed_lo, count, stride, 0, p, out, PTHREAD_MUTEX_INITIALIZER, 0};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t tid[1024];
    for (int t = 1; t < nthreads; ++t) pthread_create(&tid[t], NULL, gen_worker, &J);
    gen_worker(&J);
    for (int t = 1; t < nthreads; ++t) pthread_join(tid[t], NULL);
    return J.err;
}
