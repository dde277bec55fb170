/*
 * chordal_b200.h -- C ABI of libchordal_b200.so, the sm_100a chordality test.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 1508.06329,
 * package "chordalkit", /root/reference/pkg/src/chordalkit).  The reference is
 * pure Python; its "FFI" for this path is the set of Python entry points listed
 * next to each function.  The Python mirror in paper_1508_06329_b200/ binds
 * these symbols with ctypes (see INTEGRATION.md for the binding a chordalkit
 * maintainer would add).
 *
 * Conventions
 *  - Vertices are 0-based int32 (the reference is 1-based only at its API
 *    edge, graph.py:1-7; the Python layer converts).
 *  - Dense graphs: packed little-endian bit rows exactly like Graph._packed
 *    (graph.py:78-88: bit j&7 of byte j>>3 of row i <=> edge i-j), with a row
 *    pitch `stride` in bytes: stride % 16 == 0, stride >= ceil(n/8), padding
 *    bits zero, base pointer 16-byte aligned.
 *  - CSR graphs: int64 indptr[n+1], int32 indices (sorted ascending per row,
 *    symmetric, no self loops) -- the adjacency_lists0() shape (graph.py:152).
 *  - "_dev" arguments are device pointers; every call is asynchronous on
 *    `stream` (a cudaStream_t; NULL = legacy default stream) unless the name
 *    ends in _host.  The library holds no caller pointer after return and is
 *    reentrant per stream; it keeps no global state of its own (scratch space
 *    comes from caller workspaces).  The _host entry points without a workspace
 *    argument allocate stream-ordered from the device's default memory pool
 *    and free before returning (the pool's settings are left to the caller);
 *    repeated callers use the _ws forms with a workspace they keep.
 *  - Witness triples are int32[3] = (v, p, z) -- WitnessTriple (peo.py:26-45),
 *    0-based -- or (-1, -1, -1) when the ordering is a PEO.
 *  - Every function returns a chordal status code (CHORDAL_OK == 0).
 */
#ifndef CHORDAL_B200_H
#define CHORDAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHORDAL_OK 0
#define CHORDAL_EINVAL 1     /* bad argument (maps to ValueError / InvalidOrdering) */
#define CHORDAL_ETOOLARGE 2  /* n beyond this kernel's capacity (maps to GraphTooLarge) */
#define CHORDAL_ECUDA 3      /* CUDA launch/runtime failure */
#define CHORDAL_ENOMEM 4     /* device allocation failed (host-buffer entry points) */
#define CHORDAL_EPARSE 5     /* text input rejected (maps to ParseError; line + message returned) */
#define CHORDAL_EUTF8 6      /* text input is not valid UTF-8 (maps to ParseError) */
#define CHORDAL_ENCCL 7      /* NCCL not loadable in the process, or a collective failed */

/* LexBFS tie rules.
 *  ASCENDING  : max label, ties -> smallest vertex id.  = lexbfs_partition /
 *               lexbfs_labels with LOWEST_INDEX (search.py:262-310, 500-532,
 *               _arraylex.py:22-65) = parallel_lexbfs(Arbitration.fixed_priority())
 *               (parallel/lexbfs.py:234-262).
 *  DESCENDING : parallel_lexbfs(Arbitration.fixed_priority("descending")):
 *               starts at vertex 0, ties -> largest id.
 *  SEEDED_ARB : parallel_lexbfs(Arbitration.seeded(seed)): starts at vertex 0;
 *               at iteration i the winner among the max-label set is
 *               argmax_w (splitmix64(prefix_i ^ w), w), w 1-based,
 *               prefix_i = mix64(seed, 4(i-1)+3, mix64(crc32("current"), 0))
 *               (parallel/engine.py:47-53, parallel/lexbfs.py:211-225).
 *  SEEDED_PARTITION (CSR entry point only): lexbfs_partition(seeded(seed),
 *               method="linked") (search.py:515-532): the initial class is
 *               range(n) shuffled by Generator.shuffle on the stream
 *               (seed, "lexbfs-partition"); split-off and fully moved classes
 *               hold their members in adjacency order.
 *  SEEDED_LABELS (CSR entry point only): lexbfs_labels(seeded(seed),
 *               method="linked") (search.py:283-290): the pivot is member
 *               Generator.integers(|C|) of the max-label class C (ascending id
 *               order) on the stream (seed, "lexbfs-labels").                  */
#define CHORDAL_TIE_ASCENDING 0
#define CHORDAL_TIE_DESCENDING 1
#define CHORDAL_TIE_SEEDED_ARB 2
#define CHORDAL_TIE_SEEDED_PARTITION 3
#define CHORDAL_TIE_SEEDED_LABELS 4

/* Largest n the single-CTA dense LexBFS kernel accepts (state lives in SMEM). */
#define CHORDAL_DENSE_LEXBFS_MAX_N 32768

int chordal_abi_version(void);
const char *chordal_strerror(int status);

/* ---- dense single graph ------------------------------------------------ */

/* Workspace (device bytes) of chordal_lexbfs_dense / chordal_is_chordal_dense
 * for a graph of n vertices and m edges. */
size_t chordal_dense_workspace_bytes(int64_t n, int64_t m);

/* LexBFS ordering.  Replaces lexbfs_partition (search.py:500-506),
 * lexbfs_labels (search.py:262-268) and parallel_lexbfs (parallel/lexbfs.py:
 * 234-243).  Writes order_dev[n] (vertex at each position), pos_dev[n]
 * (position of each vertex) and, if parent_dev is not NULL, the PEO parent of
 * every vertex (-1 for none, -2 for "not computed": vertices placed by the
 * early exit once every class is a singleton); the PEO checks accept -2
 * entries and search those parents themselves.
 * Engines: n <= 1024 (LOWEST_INDEX / descending) runs the one-warp engine; up to
 * n <= 32768 the persistent single-CTA touched-segment kernel (state in shared
 * memory, any density; m, when known, picks its dense or sparse form -- pass
 * m < 0 or 0 if unknown: the sparse form is then used) -- except sparse graphs
 * with 1024 < n <= 8836 and a known m of average degree <= 20, which like all
 * larger graphs are converted to CSR on the device and run the O(deg)-per-step
 * slot kernel (for n <= 8836 with all its state in shared memory).  The CSR route
 * needs the edge count m (Graph.m; the workspace is sized from it, and an
 * understated m is rejected): for n > 32768 pass m < 0 to let the call count the
 * edges, which synchronises `stream` once. */
int chordal_lexbfs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                         uint64_t seed, int32_t *order_dev, int32_t *pos_dev, int32_t *parent_dev, void *ws,
                         size_t ws_bytes, void *stream);

/* LexBFS certificate of a given order (the invariant behind lexbfs_labels(debug=True),
 * search.py:270-271, 313-322, and parallel_lexbfs(audit=True), parallel/lexbfs.py:82-129:
 * every pivot carries the lexicographically largest label of the unvisited
 * vertices).  Replays the search with pivot i forced to order_dev[i] (a
 * permutation of 0..n-1) and writes status_dev[0] = the first step whose pivot
 * is not in the maximum-label class (-1: order_dev is a LexBFS order) and
 * status_dev[1] = the first step whose pivot differs from the LOWEST_INDEX
 * choice (-1: it is the LOWEST_INDEX order).  n <= 32768 (single-CTA engine);
 * ws >= chordal_lexbfs_certify_workspace_bytes(n). */
size_t chordal_lexbfs_certify_workspace_bytes(int64_t n);
int chordal_lexbfs_certify_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m,
                                 const int32_t *order_dev, int32_t *status_dev, void *ws, size_t ws_bytes,
                                 void *stream);

/* pos_dev[order_dev[i]] = i  (VertexOrdering.pos0, graph.py:224-230). */
int chordal_positions(const int32_t *order_dev, int64_t n, int32_t *pos_dev, void *stream);

/* Sets *key_dev = UINT64_MAX (the "no violation" key). */
int chordal_key_init(uint64_t *key_dev, void *stream);

/* Vertex-parallel PEO check over v in [v_begin, v_end): for each v takes the
 * parent p (parent_dev[v] if given, else the left neighbour with the greatest
 * position, peo.py:106-121) and tests LN(v)\{p} subset of LN(p) (peo.py:
 * 124-142, parallel/peo.py:57-65); atomically lowers *key_dev to
 * min((p << 32) | v) over violating v.  The minimum key is the reference's
 * deterministic witness pair (ascending p, then ascending v, peo.py:81-85).
 * Row shards of one graph can run on different GPUs and be combined with an
 * integer MIN all-reduce of the key. */
int chordal_peo_dense_key(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                          const int32_t *pos_dev, const int32_t *parent_dev, int64_t v_begin, int64_t v_end,
                          uint64_t *key_dev, void *stream);

/* Resolves the key to the witness triple: z = smallest vertex id in
 * LN(v) \ {p} \ N(p)  (peo.py:126-141 / _first_witness_big peo.py:167-173). */
int chordal_peo_dense_witness(const uint8_t *adj_dev, int64_t n, int64_t stride,
                              const int32_t *pos_dev, const uint64_t *key_dev,
                              int32_t *witness_dev, void *stream);

/* is_peo (peo.py:72-97): key_init + peo_dense_key over all v + witness. */
int chordal_peo_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                      const int32_t *pos_dev, const int32_t *parent_dev, uint64_t *key_dev, int32_t *witness_dev,
                      void *stream);

/* is_chordal (peo.py:177-202) / parallel_is_chordal (parallel/peo.py:98-114):
 * LexBFS then the PEO check (parents handed over when the slot engine ran),
 * all on `stream`.  ws: chordal_dense_workspace_bytes(n, m) bytes. */
int chordal_is_chordal_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                             uint64_t seed, int32_t *order_dev, int32_t *pos_dev, void *ws, size_t ws_bytes,
                             int32_t *witness_dev, void *stream);

/* Host-buffer form of is_chordal: copies the unpadded packed rows
 * (row_bytes = ceil(n/8), exactly Graph._packed) to the device, runs the
 * pipeline, copies order (n int32) and witness back and synchronises.
 * *chordal_out = 1 chordal / 0 not.  Allocates and frees its own device
 * memory (stream-ordered). */
int chordal_is_chordal_dense_host(const uint8_t *adj_host, int64_t n, int64_t row_bytes,
                                  int32_t tie_rule, uint64_t seed, int32_t *order_host,
                                  int32_t *witness_host, int32_t *chordal_out);

/* ---- CSR single graph (the N = 10^6 configuration) ---------------------- */

/* Workspace of chordal_lexbfs_csr for n vertices and m edges (m = indptr[n]/2;
 * about 50 bytes per vertex + 4 per edge). */
size_t chordal_lexbfs_csr_workspace_bytes(int64_t n, int64_t m);

/* LexBFS on CSR adjacency with the slot engine:
 * lexbfs_partition(g, method="linked") (search.py:500-532) on a graph that
 * exposes adjacency_lists0().  For n <= 32768 the per-neighbour state lives in
 * shared memory, above that in global memory.  parent_dev optional. */
int chordal_lexbfs_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int64_t m, int32_t tie_rule,
                       uint64_t seed, int32_t *order_dev, int32_t *pos_dev, int32_t *parent_dev, void *ws,
                       size_t ws_bytes, void *stream);

/* Workspace (device bytes, 16-byte aligned) of the CSR PEO check: the queue of
 * heavy rows (more than 1024 neighbours) whose lists the whole grid splits. */
size_t chordal_peo_csr_workspace_bytes(int64_t n);

/* PEO check on CSR over v in [v_begin, v_end) (row shards), as
 * chordal_peo_dense_key: parent_dev optional (NULL or -2 entries: searched);
 * membership z in N(p) by binary search in the shorter of N(p), N(z).  ws:
 * chordal_peo_csr_workspace_bytes(n) bytes, cleared on `stream` by the call;
 * one workspace per concurrent call. */
int chordal_peo_csr_key(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *pos_dev,
                        const int32_t *parent_dev, int64_t v_begin, int64_t v_end, uint64_t *key_dev, void *ws,
                        size_t ws_bytes, void *stream);
int chordal_peo_csr_witness(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n,
                            const int32_t *pos_dev, const uint64_t *key_dev, int32_t *witness_dev, void *stream);
/* _is_peo_lists (peo.py:100-149) on CSR: init + key over all v + witness. */
int chordal_peo_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *pos_dev,
                    const int32_t *parent_dev, uint64_t *key_dev, int32_t *witness_dev, void *ws, size_t ws_bytes,
                    void *stream);

/* ---- left neighbourhoods (graph.py:284-302) ----------------------------- */

/* left_neighborhoods(g, ordering): LN(v) = the neighbours of v placed before
 * it, parent(v) = the member of LN(v) with the greatest position (-1 if
 * none).  order_dev/pos_dev: a 0-based permutation and its inverse.  Each
 * output is optional (NULL = not written): ln_rows_dev uint8[n][stride] (LN
 * rows in the input's packed layout, padding zero), parent_dev int32[n],
 * ln_size_dev int32[n] = |LN(v)|, deg_dev int32[n] = deg(v).  The sizes feed
 * the reference's list-scan read count (ScanStats, peo.py:100-149). */
int chordal_left_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                       const int32_t *pos_dev, uint8_t *ln_rows_dev, int32_t *parent_dev, int32_t *ln_size_dev,
                       int32_t *deg_dev, void *stream);
/* The same on CSR adjacency (deg(v) = indptr[v+1] - indptr[v]). */
int chordal_left_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *order_dev,
                     const int32_t *pos_dev, int32_t *parent_dev, int32_t *ln_size_dev, void *stream);

/* The host-buffer pipeline over a caller-provided device workspace of
 * chordal_dense_host_workspace_bytes(n, m) bytes (256-byte aligned; m = the edge
 * count, Graph.m), reused across calls, on the calling thread's default stream. */
size_t chordal_dense_host_workspace_bytes(int64_t n, int64_t m);
int chordal_is_chordal_dense_host_ws(const uint8_t *adj_host, int64_t n, int64_t row_bytes, int64_t m,
                                     int32_t tie_rule, uint64_t seed, int32_t *order_host, int32_t *witness_host,
                                     int32_t *chordal_out, void *ws_dev, size_t ws_bytes);

/* Packed rows -> CSR (ascending rows).  indptr_dev[n+1] is always written;
 * indices_dev (capacity indptr[n]) is filled when not NULL, so a caller can
 * size it from indptr[n] first. */
int chordal_dense_to_csr(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t *indptr_dev,
                         int32_t *indices_dev, void *stream);

/* Relabel: out row r, bit s = adj[perm[r]][perm[s]] (perm a 0-based
 * permutation, out distinct from adj, same stride).  Lets the ascending
 * kernel replay lexbfs_array with a seeded initial arrangement
 * (search.py:535-541, _arraylex.py:22-27): order = perm[order_relabelled]. */
int chordal_permute_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *perm_dev,
                          uint8_t *out_dev, void *stream);

/* ---- batches of small dense graphs (one warp-resident search per graph) - */

/* Largest n per graph the batched kernel accepts. */
#define CHORDAL_BATCH_MAX_N 1024

/* is_chordal over `batch` independent graphs of n vertices, graph b at
 * adj_dev + b * n * stride.  Writes orders_dev[b*n + i] and
 * witness_dev[3*b + k]; verdict = witness[3*b] < 0.  LOWEST_INDEX ties. */
int chordal_is_chordal_batch(const uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride,
                             int32_t *orders_dev, int32_t *witness_dev, void *stream);

/* Host-buffer form of the batch (the end-to-end call a host application
 * makes): graph b at adj_host + b * n * row_bytes (row_bytes >= ceil(n/8); use
 * pinned memory for full copy bandwidth).  Chunks of `chunk` graphs (<= 0:
 * 4096) rotate over three streams so the H2D copy of one chunk and the D2H of
 * another overlap the search of a third.  Synchronous: returns when
 * orders_host[b*n + i] and witness_host[3*b + k] are written. */
int chordal_is_chordal_batch_host(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes,
                                  int32_t *orders_host, int32_t *witness_host, int64_t chunk);

/* The same with a caller-provided device workspace of
 * chordal_batch_host_workspace_bytes(n, chunk) bytes (256-byte aligned), reused
 * across calls: the form to call repeatedly.  (Each call of the form above
 * takes and returns a ~1 GB pool block, which costs some calls 10-600 ms.) */
size_t chordal_batch_host_workspace_bytes(int64_t n, int64_t chunk);
int chordal_is_chordal_batch_host_ws(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes,
                                     int32_t *orders_host, int32_t *witness_host, int64_t chunk, void *ws_dev,
                                     size_t ws_bytes);

/* ---- synthetic inputs --------------------------------------------------- */

/* gen_dense_random (generate.py:32-56) bit for bit: Philox4x64-10 keyed by
 * key = mix64(seed, crc32("dense-random")) (rng.py:18-21), uniform doubles
 * (x >> 11) * 2^-53 drawn row-major over the upper triangle (draw u*n+v
 * decides edge u<v), mirrored.  Graph b (seed = seed0 + b * seed_step) is
 * written at adj_dev + b * n * stride; rows are fully overwritten. */
int chordal_gen_dense_random(uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride, double p,
                             int64_t seed0, int64_t seed_step, void *stream);

/* Build packed rows from an undirected edge list (0-based endpoints, vertex
 * ids < n, no self loops; duplicates collapse) -- Graph._from_numpy_edges
 * (graph.py:78-88) in HBM.  Rows are zeroed first. */
int chordal_edges_to_dense(const int32_t *u_dev, const int32_t *v_dev, int64_t m, uint8_t *adj_dev, int64_t n,
                           int64_t stride, void *stream);

/* gen_chordal_random (generate.py:118-155) bit for bit, one GPU thread per
 * graph: Philox4x64-10 keyed by mix64(seed, crc32("chordal-random")), with
 * numpy's integers() (Lemire 32-bit bounded draws on split 64-bit outputs)
 * and choice(replace=False) (Floyd + shuffle) replayed exactly.  Graph b uses
 * seed0 + b * seed_step.  Needs k + 2 <= 10000 and a device scratch of
 * chordal_gen_chordal_random_scratch_bytes(batch, n, k) bytes. */
size_t chordal_gen_chordal_random_scratch_bytes(int64_t batch, int64_t n, int64_t k);

/* Edge-list form for one large graph (the N = 10^6 configuration, whose
 * dense matrix would not fit): the same draws, run by one GPU thread; writes
 * the m attachment edges (u_dev[e], v_dev[e]) -- capacity n * (k + 1) -- and
 * *m_dev.  scratch: chordal_gen_chordal_random_scratch_bytes(1, n, k). */
int chordal_gen_chordal_random_edges(int64_t n, int64_t k, int64_t seed, int32_t *u_dev, int32_t *v_dev,
                                     int64_t *m_dev, void *scratch_dev, size_t scratch_bytes, void *stream);
int chordal_gen_chordal_random(uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride, int64_t k, int64_t seed0,
                               int64_t seed_step, void *scratch_dev, size_t scratch_bytes, void *stream);

/* ---- other vertex orderings (search.py:79-145) ----------------------------- */

/* mcs_order (search.py:113-145) on dense rows, n <= 65535: maximum cardinality
 * search, ties to the smallest id; seeded != 0 replays TieBreak(seed): the
 * winner is ties[Generator.integers(len(ties))] on the stream (seed, "mcs"),
 * ties ascending.  One persistent CTA, weights in shared memory. */
int chordal_mcs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int32_t seeded, uint64_t seed,
                      int32_t *order_dev, int32_t *pos_dev, void *stream);

/* bfs_order (search.py:79-110) on CSR rows: FIFO order with restarts at the
 * smallest unqueued vertex; seeded != 0 replays TieBreak(seed) (restart at
 * pool[integers(len(pool))], fresh neighbours Generator.shuffle'd) on the
 * stream (seed, "bfs").  ws: chordal_bfs_csr_workspace_bytes(n) bytes (0
 * unless n exceeds the shared-memory bitset). */
size_t chordal_bfs_csr_workspace_bytes(int64_t n);
/* bfs_order on dense rows (n <= 65535): fresh neighbours = row & ~queued, one
 * warp, word-parallel -- the form for dense-stored graphs. */
int chordal_bfs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int32_t seeded, uint64_t seed,
                      int32_t *order_dev, int32_t *pos_dev, void *stream);
int chordal_bfs_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int32_t seeded, uint64_t seed,
                    int32_t *order_dev, int32_t *pos_dev, void *ws, size_t ws_bytes, void *stream);

/* ---- plain-text formats (host side, textio.py) ---------------------------- */

/* parse_graph_text (textio.py:30-86) straight into packed rows.  Two calls:
 * with rows_out == NULL the text is scanned up to its header and *n_out /
 * *m_out are returned (errors before or on the header are reported); the
 * caller then passes zeroed rows_out[n * row_bytes] (row_bytes >= ceil(n/8))
 * and the whole text is validated while the bits are set.  cap: the vertex cap
 * of _check_size (graph.py:23-28), < 0 = none.  Errors: CHORDAL_EPARSE with
 * *err_line (1-based, -1 = no line) and err_msg = the reference's message;
 * CHORDAL_ETOOLARGE with err_msg = n in decimal (GraphTooLarge);
 * CHORDAL_EUTF8.  Host memory only; no CUDA. */
int chordal_parse_graph_text(const char *text, int64_t len, int64_t cap, int64_t *n_out, int64_t *m_out,
                             uint8_t *rows_out, int64_t row_bytes, int64_t *err_line, char *err_msg,
                             int64_t err_cap);

/* write_graph_text (textio.py:89-93): "p n m" then "e u v" for u < v
 * ascending.  Returns the text length; writes it to out when out_cap is large
 * enough (call with out = NULL to size the buffer); -1 on bad arguments. */
int64_t chordal_write_graph_text(const uint8_t *rows, int64_t n, int64_t row_bytes, int64_t m, char *out,
                                 int64_t out_cap);

/* parse_ordering_text's field scan (textio.py:96-106): whitespace-separated
 * integers; the first n go to order_out (1-based ids as written), *count_out =
 * the number of fields.  The caller raises InvalidOrdering on a count or
 * permutation mismatch. */
int chordal_parse_ordering_text(const char *text, int64_t len, int64_t n, int64_t *order_out, int64_t *count_out,
                                int64_t *err_line, char *err_msg, int64_t err_cap);

/* ---- multi-GPU: row-sharded chordality test over NCCL ----------------- */

/* is_chordal of one graph replicated on every rank of `nccl_comm` (the caller's
 * ncclComm_t, one GPU per rank), the protocol of distributed.sharded_is_chordal:
 * rank `root` runs LexBFS (a single graph's step chain stays on one GPU),
 * broadcasts order + PEO parents, every rank checks its row shard (contiguous,
 * rank r of W gets n / W rows, +1 for r < n % W; chordal_peo_*_key), one 8-byte MIN all-reduce of
 * the witness key, z resolved on every rank.  On return (stream order) every
 * rank holds order_dev, pos_dev and witness_dev.  NCCL is resolved from the
 * process by soname (libnccl.so.2, the library that created the communicator)
 * at the first call: CHORDAL_ENCCL if it cannot be.  Dense graphs with
 * n > 32768 need m >= 0.  ws: chordal_{dense,csr}_nccl_workspace_bytes(n, m). */
size_t chordal_dense_nccl_workspace_bytes(int64_t n, int64_t m);
int chordal_is_chordal_dense_nccl(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                                  uint64_t seed, int32_t root, void *nccl_comm, int32_t *order_dev, int32_t *pos_dev,
                                  int32_t *witness_dev, void *ws, size_t ws_bytes, void *stream);
size_t chordal_csr_nccl_workspace_bytes(int64_t n, int64_t m);
int chordal_is_chordal_csr_nccl(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int64_t m,
                                int32_t tie_rule, uint64_t seed, int32_t root, void *nccl_comm, int32_t *order_dev,
                                int32_t *pos_dev, int32_t *witness_dev, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CHORDAL_B200_H */
