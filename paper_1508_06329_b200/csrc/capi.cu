// capi.cu -- extern "C" entry points of libchordal_b200.so (include/chordal_b200.h).
//
// Thin validation + launch layer: no global mutable state, no retained caller
// pointers; every device entry point is asynchronous on the caller's stream.
#include <cstring>
#include <dlfcn.h>

#include "common.cuh"

namespace chordal {
int launch_lexbfs_seg(const uint8_t *, int64_t, int64_t, int64_t, int32_t, uint64_t, uint64_t, int32_t *, int32_t *,
                      int32_t *, cudaStream_t, const int32_t * = nullptr, int32_t * = nullptr);
int launch_positions(const int32_t *, int64_t, int32_t *, cudaStream_t);
int launch_fill_i32(int32_t *, int64_t, int32_t, cudaStream_t);
int launch_key_init(uint64_t *, cudaStream_t);
int launch_peo_dense_key(const uint8_t *, int64_t, int64_t, const int32_t *, const int32_t *, const int32_t *,
                         int64_t, int64_t, uint64_t *, cudaStream_t);
size_t csr_workspace_bytes(int64_t, int64_t);
int launch_lexbfs_csr(const int64_t *, const int32_t *, int64_t, int64_t, int32_t, uint64_t, uint64_t, int32_t *,
                      int32_t *,
                      int32_t *, void *, cudaStream_t);
int launch_peo_csr_key(const int64_t *, const int32_t *, int64_t, const int32_t *, const int32_t *, int64_t, int64_t,
                       uint64_t *, void *, cudaStream_t);
size_t peo_csr_workspace_bytes();
int launch_peo_csr_witness(const int64_t *, const int32_t *, const int32_t *, const uint64_t *, int32_t *,
                           cudaStream_t);
int launch_dense_degrees(const uint8_t *, int64_t, int64_t, int64_t *, cudaStream_t);
int launch_dense_fill(const uint8_t *, int64_t, int64_t, const int64_t *, int32_t *, int64_t, cudaStream_t);
int launch_peo_dense_witness(const uint8_t *, int64_t, int64_t, const int32_t *, const uint64_t *,
                             int32_t *, cudaStream_t);
int launch_permute_dense(const uint8_t *, int64_t, int64_t, const int32_t *, uint8_t *, cudaStream_t);
int launch_spread_rows(const uint8_t *, int64_t, int64_t, int64_t, int64_t, uint8_t *, cudaStream_t);
int launch_batch(const uint8_t *, int64_t, int64_t, int64_t, int32_t *, int32_t *, cudaStream_t);
int launch_mcs_dense(const uint8_t *, int64_t, int64_t, bool, uint64_t, int32_t *, int32_t *, cudaStream_t);
size_t bfs_csr_workspace_bytes(int64_t);
int launch_bfs_dense(const uint8_t *, int64_t, int64_t, bool, uint64_t, int32_t *, int32_t *, cudaStream_t);
int launch_bfs_csr(const int64_t *, const int32_t *, int64_t, bool, uint64_t, uint32_t *, int32_t *, int32_t *,
                   cudaStream_t);
int launch_gen_dense_random(uint8_t *, int64_t, int64_t, int64_t, double, int64_t, int64_t, uint32_t,
                            cudaStream_t);
int launch_edges_to_dense(const int32_t *, const int32_t *, int64_t, uint8_t *, int64_t, int64_t, cudaStream_t);
long long gen_chordal_scratch_words(int64_t, int64_t, int *);
int launch_gen_chordal_edges(int64_t, int64_t, int64_t, uint32_t, int32_t *, int32_t *, int32_t *, long long *,
                             cudaStream_t);
int launch_gen_chordal_random(uint8_t *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, uint32_t, int32_t *,
                              cudaStream_t);
int launch_left_dense(const uint8_t *, int64_t, int64_t, const int32_t *, const int32_t *, uint8_t *, int32_t *,
                      int32_t *, int32_t *, cudaStream_t);
int launch_left_csr(const int64_t *, const int32_t *, int64_t, const int32_t *, const int32_t *, int32_t *, int32_t *,
                    cudaStream_t);

}  // namespace chordal

using namespace chordal;

namespace {

// zlib crc32 (label_hash, _bitops.py:77-79)
uint32_t crc32_str(const char *s) {
    uint32_t c = 0xFFFFFFFFu;
    for (; *s; ++s) {
        c ^= (uint8_t)*s;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return c ^ 0xFFFFFFFFu;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// The host-buffer entry points without a workspace argument allocate their
// device buffers stream-ordered from the device's default pool and free them
// before returning; the pool's settings are the caller's (with the default
// release threshold the memory goes back to the driver at each sync, so
// repeated calls should use the _ws forms with a workspace kept by the caller).

int check_dense(const void *adj, int64_t n, int64_t stride) {
    if (n < 0) return CHORDAL_EINVAL;
    if (n == 0) return CHORDAL_OK;
    if (!adj) return CHORDAL_EINVAL;
    if (n > 0x7FFFFFFF) return CHORDAL_ETOOLARGE;
    if (stride % 16 != 0 || stride < (n + 7) / 8) return CHORDAL_EINVAL;
    if (reinterpret_cast<uintptr_t>(adj) % 16 != 0) return CHORDAL_EINVAL;
    return CHORDAL_OK;
}

}  // namespace

extern "C" {

int chordal_abi_version(void) { return 3; }

const char *chordal_strerror(int status) {
    switch (status) {
        case CHORDAL_OK: return "ok";
        case CHORDAL_EINVAL: return "invalid argument";
        case CHORDAL_ETOOLARGE: return "graph too large for this kernel";
        case CHORDAL_ECUDA: return "CUDA error";
        case CHORDAL_ENOMEM: return "device allocation failed";
        case CHORDAL_EPARSE: return "text input rejected";
        case CHORDAL_EUTF8: return "text input is not valid UTF-8";
        case CHORDAL_ENCCL: return "NCCL not loadable in this process, or a collective failed";
        default: return "unknown status";
    }
}

// Engine choice for a dense-stored graph: n <= 32768 runs the single-CTA
// touched-segment arrangement kernel (lexbfs_seg.cu, state in shared memory,
// O(deg/32 + movers + split classes) per step, any density); larger graphs are
// converted to CSR on the device and run the slot engine -- and so do sparse
// graphs (known m, average degree <= 20) with 1024 < n <= 8836, whose slot
// engine keeps all its state in shared memory: 0.78-0.92x the CTA engine's time
// including the conversion (tools/engine_cross.py; configuration 2 chordal
// 7.98 -> 7.25 + 0.1 ms), while at average degree >= 40 it is 1.1-1.3x slower.
static bool small_sparse(int64_t n, int64_t m) { return n > 1024 && n <= 8836 && m > 0 && 2 * m <= 20 * n; }
static bool use_seg(int64_t n, int64_t m) { return n <= CHORDAL_DENSE_LEXBFS_MAX_N && !small_sparse(n, m); }

struct DenseWs {  // workspace carve-up (bytes) of the dense entry points
    size_t key, parent, indptr, indices, slot, total;
    DenseWs(int64_t n, int64_t m) {
        auto a = [](size_t x) { return (x + 255) & ~size_t(255); };
        size_t o = 0;
        key = o; o = a(o + 16);
        parent = o; o = a(o + sizeof(int32_t) * (size_t)n);
        indptr = indices = slot = o;
        if (!use_seg(n, m)) {
            indptr = o; o = a(o + sizeof(int64_t) * (size_t)(n + 1));
            indices = o; o = a(o + sizeof(int32_t) * (size_t)(2 * m + 1));
            slot = o; o = a(o + csr_workspace_bytes(n, m));
        }
        total = o;
    }
};

static int count_edges_sync(const uint8_t *adj, int64_t n, int64_t stride, cudaStream_t s, int64_t *m_out) {
    int64_t *ip = nullptr;
    if (cudaMallocAsync((void **)&ip, sizeof(int64_t) * (n + 1), s) != cudaSuccess) return CHORDAL_ENOMEM;
    int rc = launch_dense_degrees(adj, n, stride, ip, s);
    int64_t tot = 0;
    if (rc == CHORDAL_OK &&
        cudaMemcpyAsync(&tot, ip + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        rc = CHORDAL_ECUDA;
    cudaFreeAsync(ip, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == CHORDAL_OK) rc = CHORDAL_ECUDA;
    *m_out = tot / 2;
    return rc;
}

// indptr[n] <= 2m, or EINVAL: buffers sized from a caller's m must hold every
// adjacency entry (one 8-byte read back + a sync of the stream; only on the
// slot-engine routes, whose searches take milliseconds to seconds).
static int check_nnz(const int64_t *indptr, int64_t n, int64_t m, cudaStream_t s) {
    int64_t tot = 0;
    if (cudaMemcpyAsync(&tot, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return CHORDAL_ECUDA;
    return (tot < 0 || tot > 2 * m) ? CHORDAL_EINVAL : CHORDAL_OK;
}

size_t chordal_dense_workspace_bytes(int64_t n, int64_t m) {
    if (n < 0 || m < 0) return 0;
    return DenseWs(n, m).total;
}

int chordal_lexbfs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                         uint64_t seed, int32_t *order_dev, int32_t *pos_dev, int32_t *parent_dev, void *ws,
                         size_t ws_bytes, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    if (!order_dev || !pos_dev) return CHORDAL_EINVAL;
    if (tie_rule < 0 || tie_rule > 2) return CHORDAL_EINVAL;
    cudaStream_t s = as_stream(stream);
    const uint64_t cell = current_cell(crc32_str("current"));
    if (use_seg(n, m))
        return launch_lexbfs_seg(adj_dev, n, stride, m, tie_rule, seed, cell, order_dev, pos_dev, parent_dev, s);
    if (m < 0) {
        rc = count_edges_sync(adj_dev, n, stride, s, &m);
        if (rc) return rc;
    }
    const DenseWs L(n, m);
    if (!ws || ws_bytes < L.total) return CHORDAL_EINVAL;
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    int64_t *indptr = reinterpret_cast<int64_t *>(w + L.indptr);
    int32_t *indices = reinterpret_cast<int32_t *>(w + L.indices);
    rc = launch_dense_degrees(adj_dev, n, stride, indptr, s);
    if (rc) return rc;
    rc = check_nnz(indptr, n, m, s);  // the workspace was sized from m
    if (rc) return rc;
    rc = launch_dense_fill(adj_dev, n, stride, indptr, indices, 2 * m + 1, s);
    if (rc) return rc;
    return launch_lexbfs_csr(indptr, indices, n, m, tie_rule, seed, cell, order_dev, pos_dev, parent_dev,
                             w + L.slot, s);
}

size_t chordal_lexbfs_certify_workspace_bytes(int64_t n) { return n > 0 ? (size_t)n * 8 : 0; }

int chordal_lexbfs_certify_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m,
                                 const int32_t *order_dev, int32_t *status_dev, void *ws, size_t ws_bytes,
                                 void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!status_dev) return CHORDAL_EINVAL;
    cudaStream_t s = as_stream(stream);
    if (n == 0) return cudaMemsetAsync(status_dev, 0xFF, 2 * sizeof(int32_t), s) == cudaSuccess ? CHORDAL_OK
                                                                                                 : CHORDAL_ECUDA;
    if (!order_dev) return CHORDAL_EINVAL;
    if (n > CHORDAL_DENSE_LEXBFS_MAX_N) return CHORDAL_ETOOLARGE;
    if (!ws || ws_bytes < chordal_lexbfs_certify_workspace_bytes(n)) return CHORDAL_EINVAL;
    int32_t *replay = reinterpret_cast<int32_t *>(ws);
    rc = launch_lexbfs_seg(adj_dev, n, stride, m, 5 /* kTieCertify */, 0, 0, replay, replay + n, nullptr, s,
                           order_dev, status_dev);
    return rc;
}

int chordal_positions(const int32_t *order_dev, int64_t n, int32_t *pos_dev, void *stream) {
    if (n < 0 || (n > 0 && (!order_dev || !pos_dev))) return CHORDAL_EINVAL;
    return launch_positions(order_dev, n, pos_dev, as_stream(stream));
}

int chordal_key_init(uint64_t *key_dev, void *stream) {
    if (!key_dev) return CHORDAL_EINVAL;
    return launch_key_init(key_dev, as_stream(stream));
}

int chordal_peo_dense_key(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                          const int32_t *pos_dev, const int32_t *parent_dev, int64_t v_begin, int64_t v_end,
                          uint64_t *key_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    if (!order_dev || !pos_dev || !key_dev) return CHORDAL_EINVAL;
    return launch_peo_dense_key(adj_dev, n, stride, order_dev, pos_dev, parent_dev, v_begin, v_end, key_dev,
                                as_stream(stream));
}

int chordal_peo_dense_witness(const uint8_t *adj_dev, int64_t n, int64_t stride,
                              const int32_t *pos_dev, const uint64_t *key_dev,
                              int32_t *witness_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!key_dev || !witness_dev) return CHORDAL_EINVAL;
    if (n == 0) {
        // empty graph: always a PEO
        static const int32_t none[3] = {-1, -1, -1};
        if (cudaMemcpyAsync(witness_dev, none, sizeof(none), cudaMemcpyHostToDevice,
                            as_stream(stream)) != cudaSuccess)
            return CHORDAL_ECUDA;
        return CHORDAL_OK;
    }
    if (!pos_dev) return CHORDAL_EINVAL;
    return launch_peo_dense_witness(adj_dev, n, stride, pos_dev, key_dev, witness_dev,
                                    as_stream(stream));
}

int chordal_peo_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                      const int32_t *pos_dev, const int32_t *parent_dev, uint64_t *key_dev, int32_t *witness_dev,
                      void *stream) {
    // three launches (key init, key, witness): a fused form whose last CTA resolves
    // the witness (ticket counter) measured no faster -- G(8192, 0.5) is_chordal
    // 0.1987 -> 0.2002 ms, config 3 unchanged; queued launches cost ~no gap
    int rc = chordal_key_init(key_dev, stream);
    if (rc) return rc;
    rc = chordal_peo_dense_key(adj_dev, n, stride, order_dev, pos_dev, parent_dev, 0, n, key_dev, stream);
    if (rc) return rc;
    return chordal_peo_dense_witness(adj_dev, n, stride, pos_dev, key_dev, witness_dev, stream);
}

int chordal_is_chordal_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                             uint64_t seed, int32_t *order_dev, int32_t *pos_dev, void *ws, size_t ws_bytes,
                             int32_t *witness_dev, void *stream) {
    cudaStream_t s = as_stream(stream);
    if (n > 0 && m < 0 && !use_seg(n, m)) {
        int rc0 = check_dense(adj_dev, n, stride);
        if (rc0) return rc0;
        rc0 = count_edges_sync(adj_dev, n, stride, s, &m);
        if (rc0) return rc0;
    }
    const DenseWs L(n, m < 0 ? 0 : m);
    if (!ws || ws_bytes < L.total) return CHORDAL_EINVAL;
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    uint64_t *key = reinterpret_cast<uint64_t *>(w + L.key);
    // The shared-memory CTA engine would record parents with one global store per
    // unvisited neighbour per step (~6 % of its step time at N = 32768, k = 1024);
    // the PEO kernel finds them in a fraction of a millisecond instead.  The slot
    // engine (n > 32768) keeps recording them.
    // The one-warp engine (n <= 1024) records them in shared memory and copies
    // them out with the order.
    int32_t *parent = (use_seg(n, m) && n > 1024) ? nullptr : reinterpret_cast<int32_t *>(w + L.parent);
    int rc = chordal_lexbfs_dense(adj_dev, n, stride, m, tie_rule, seed, order_dev, pos_dev, parent, ws, ws_bytes,
                                  stream);
    if (rc) return rc;
    return chordal_peo_dense(adj_dev, n, stride, order_dev, pos_dev, n > 0 ? parent : nullptr, key, witness_dev,
                             stream);
}

// Host rows -> device rows of pitch `stride` with zeroed padding.  Equal pitches:
// one flat copy.  A narrower host pitch (the reference's ceil(n/8)-byte rows):
// one flat copy into `staging` (>= n * row_bytes bytes) and a kernel that spreads
// the rows -- a pitched copy from pageable memory is staged row by row by the
// driver (0.45 ms at n = 1000, tools/host_call_probe.cu).  A wider host pitch:
// the pitched copy into pre-zeroed rows.
static int upload_rows(uint8_t *adj, int64_t stride, const uint8_t *adj_host, int64_t row_bytes, int64_t n,
                       uint8_t *staging, cudaStream_t s) {
    const int64_t nb = (n + 7) / 8;
    if (row_bytes == stride && stride == nb)
        return cudaMemcpyAsync(adj, adj_host, (size_t)n * stride, cudaMemcpyHostToDevice, s) == cudaSuccess
                   ? CHORDAL_OK : CHORDAL_ECUDA;
    if (row_bytes <= stride && staging) {
        if (cudaMemcpyAsync(staging, adj_host, (size_t)n * row_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return CHORDAL_ECUDA;
        return launch_spread_rows(staging, row_bytes, n, nb, stride, adj, s);
    }
    if (cudaMemsetAsync(adj, 0, (size_t)n * stride, s) != cudaSuccess ||
        cudaMemcpy2DAsync(adj, stride, adj_host, row_bytes, nb, n, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return CHORDAL_ECUDA;
    return CHORDAL_OK;
}

int chordal_is_chordal_dense_host(const uint8_t *adj_host, int64_t n, int64_t row_bytes,
                                  int32_t tie_rule, uint64_t seed, int32_t *order_host,
                                  int32_t *witness_host, int32_t *chordal_out) {
    if (n < 0 || !witness_host || !chordal_out || (n > 0 && (!adj_host || !order_host)))
        return CHORDAL_EINVAL;
    if (n > 0 && row_bytes < (n + 7) / 8) return CHORDAL_EINVAL;
    if (n == 0) {
        witness_host[0] = witness_host[1] = witness_host[2] = -1;
        *chordal_out = 1;
        return CHORDAL_OK;
    }
    const int64_t stride = (((n + 7) / 8) + 15) / 16 * 16;
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return CHORDAL_ECUDA;
    const size_t adj_bytes = ((size_t)n * stride + 255) & ~size_t(255);
    uint8_t *adj = nullptr, *ws = nullptr;
    int32_t *order = nullptr;
    int rc = CHORDAL_OK;
    int64_t m = -1;
    do {
        // staging for a narrower host pitch (the rows are spread on the device)
        const size_t stage_bytes = row_bytes <= stride ? (((size_t)n * row_bytes + 255) & ~size_t(255)) : 0;
        const size_t ord_bytes = (sizeof(int32_t) * (size_t)(2 * n + 4) + 255) & ~size_t(255);
        if (cudaMallocAsync((void **)&adj, adj_bytes + ord_bytes + stage_bytes, s) != cudaSuccess) {
            rc = CHORDAL_ENOMEM;
            break;
        }
        order = reinterpret_cast<int32_t *>(adj + adj_bytes);
        rc = upload_rows(adj, stride, adj_host, row_bytes, n, stage_bytes ? adj + adj_bytes + ord_bytes : nullptr, s);
        if (rc) break;
        if (n > 1024) {  // the engine choice (CSR route) and its thread count depend on the density
            rc = count_edges_sync(adj, n, stride, s, &m);
            if (rc) break;
        }
        const size_t wsb = DenseWs(n, m).total;
        if (cudaMallocAsync((void **)&ws, wsb + 16, s) != cudaSuccess) { rc = CHORDAL_ENOMEM; break; }
        int32_t *wit = reinterpret_cast<int32_t *>(ws + wsb);
        rc = chordal_is_chordal_dense(adj, n, stride, m, tie_rule, seed, order, order + n, ws, wsb, wit, s);
        if (rc) break;
        if (cudaMemcpyAsync(order_host, order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(witness_host, wit, sizeof(int32_t) * 3, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
            rc = CHORDAL_ECUDA;
            break;
        }
    } while (0);
    if (ws) cudaFreeAsync(ws, s);
    if (adj) cudaFreeAsync(adj, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == CHORDAL_OK) rc = CHORDAL_ECUDA;
    cudaStreamDestroy(s);
    if (rc == CHORDAL_OK) *chordal_out = witness_host[0] < 0 ? 1 : 0;
    return rc;
}

size_t chordal_dense_host_workspace_bytes(int64_t n, int64_t m) {
    if (n <= 0) return 0;
    const int64_t stride = (((n + 7) / 8) + 15) / 16 * 16;
    const size_t adj_bytes = ((size_t)n * stride + 255) & ~size_t(255);
    const size_t ord_bytes = (sizeof(int32_t) * (size_t)(2 * n + 4) + 255) & ~size_t(255);
    // + staging for host rows narrower than the device pitch (upload_rows)
    const size_t stage_bytes = stride != (n + 7) / 8 ? adj_bytes : 0;
    return adj_bytes + ord_bytes + ((DenseWs(n, m < 0 ? 0 : m).total + 255) & ~size_t(255)) + 256 + stage_bytes;
}

int chordal_is_chordal_dense_host_ws(const uint8_t *adj_host, int64_t n, int64_t row_bytes, int64_t m,
                                     int32_t tie_rule, uint64_t seed, int32_t *order_host, int32_t *witness_host,
                                     int32_t *chordal_out, void *ws_dev, size_t ws_bytes) {
    if (n < 0 || m < 0 || !witness_host || !chordal_out || (n > 0 && (!adj_host || !order_host)))
        return CHORDAL_EINVAL;
    if (n > 0 && row_bytes < (n + 7) / 8) return CHORDAL_EINVAL;
    if (n == 0) {
        witness_host[0] = witness_host[1] = witness_host[2] = -1;
        *chordal_out = 1;
        return CHORDAL_OK;
    }
    if (!ws_dev || ws_bytes < chordal_dense_host_workspace_bytes(n, m) ||
        (reinterpret_cast<uintptr_t>(ws_dev) & 255))
        return CHORDAL_EINVAL;
    const int64_t stride = (((n + 7) / 8) + 15) / 16 * 16;
    const size_t adj_bytes = ((size_t)n * stride + 255) & ~size_t(255);
    const size_t ord_bytes = (sizeof(int32_t) * (size_t)(2 * n + 4) + 255) & ~size_t(255);
    const size_t wsb = (DenseWs(n, m).total + 255) & ~size_t(255);
    uint8_t *adj = reinterpret_cast<uint8_t *>(ws_dev);
    int32_t *order = reinterpret_cast<int32_t *>(adj + adj_bytes);
    uint8_t *ws = adj + adj_bytes + ord_bytes;
    int32_t *wit = reinterpret_cast<int32_t *>(ws + wsb);
    cudaStream_t s = cudaStreamPerThread;
    int rc = CHORDAL_OK;
    do {
        uint8_t *staging = stride != (n + 7) / 8 ? reinterpret_cast<uint8_t *>(wit) + 256 : nullptr;
        rc = upload_rows(adj, stride, adj_host, row_bytes, n, staging, s);
        if (rc) break;
        rc = chordal_is_chordal_dense(adj, n, stride, m, tie_rule, seed, order, order + n, ws, wsb, wit, s);
        if (rc) break;
        if (cudaMemcpyAsync(order_host, order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(witness_host, wit, sizeof(int32_t) * 3, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            rc = CHORDAL_ECUDA;
    } while (0);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == CHORDAL_OK) rc = CHORDAL_ECUDA;
    if (rc == CHORDAL_OK) *chordal_out = witness_host[0] < 0 ? 1 : 0;
    return rc;
}

// ---- CSR -------------------------------------------------------------------

size_t chordal_lexbfs_csr_workspace_bytes(int64_t n, int64_t m) {
    return (n <= 0 || m < 0) ? 0 : csr_workspace_bytes(n, m);
}

int chordal_lexbfs_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int64_t m, int32_t tie_rule,
                       uint64_t seed, int32_t *order_dev, int32_t *pos_dev, int32_t *parent_dev, void *ws,
                       size_t ws_bytes, void *stream) {
    if (n < 0 || m < 0) return CHORDAL_EINVAL;
    if (n == 0) return CHORDAL_OK;
    if (n > 0x7FFFFFF0LL / 2) return CHORDAL_ETOOLARGE;
    if (!indptr_dev || !indices_dev || !order_dev || !pos_dev || !ws) return CHORDAL_EINVAL;
    if (ws_bytes < csr_workspace_bytes(n, m)) return CHORDAL_EINVAL;
    if (tie_rule < 0 || tie_rule > 4) return CHORDAL_EINVAL;
    // the seeded linked variants draw from the Philox stream (seed, label) (rng.py:18-21)
    if (tie_rule == CHORDAL_TIE_SEEDED_PARTITION)
        seed = splitmix64(splitmix64(seed) ^ (uint64_t)crc32_str("lexbfs-partition"));
    else if (tie_rule == CHORDAL_TIE_SEEDED_LABELS)
        seed = splitmix64(splitmix64(seed) ^ (uint64_t)crc32_str("lexbfs-labels"));
    int rc = check_nnz(indptr_dev, n, m, as_stream(stream));
    if (rc) return rc;
    return launch_lexbfs_csr(indptr_dev, indices_dev, n, m, tie_rule, seed, current_cell(crc32_str("current")),
                             order_dev, pos_dev, parent_dev, ws, as_stream(stream));
}

int chordal_mcs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int32_t seeded, uint64_t seed,
                      int32_t *order_dev, int32_t *pos_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    if (!order_dev || !pos_dev) return CHORDAL_EINVAL;
    const uint64_t key = splitmix64(splitmix64(seed) ^ (uint64_t)crc32_str("mcs"));
    return launch_mcs_dense(adj_dev, n, stride, seeded != 0, key, order_dev, pos_dev, as_stream(stream));
}

int chordal_bfs_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, int32_t seeded, uint64_t seed,
                      int32_t *order_dev, int32_t *pos_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    if (!order_dev || !pos_dev) return CHORDAL_EINVAL;
    const uint64_t key = splitmix64(splitmix64(seed) ^ (uint64_t)crc32_str("bfs"));
    return launch_bfs_dense(adj_dev, n, stride, seeded != 0, key, order_dev, pos_dev, as_stream(stream));
}

size_t chordal_bfs_csr_workspace_bytes(int64_t n) { return n > 0 ? bfs_csr_workspace_bytes(n) : 0; }

int chordal_bfs_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int32_t seeded, uint64_t seed,
                    int32_t *order_dev, int32_t *pos_dev, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0) return CHORDAL_EINVAL;
    if (n == 0) return CHORDAL_OK;
    if (!indptr_dev || !indices_dev || !order_dev || !pos_dev) return CHORDAL_EINVAL;
    if (ws_bytes < bfs_csr_workspace_bytes(n)) return CHORDAL_EINVAL;
    const uint64_t key = splitmix64(splitmix64(seed) ^ (uint64_t)crc32_str("bfs"));
    return launch_bfs_csr(indptr_dev, indices_dev, n, seeded != 0, key, reinterpret_cast<uint32_t *>(ws), order_dev,
                          pos_dev, as_stream(stream));
}

size_t chordal_peo_csr_workspace_bytes(int64_t n) { return n > 0 ? peo_csr_workspace_bytes() : 0; }

int chordal_peo_csr_key(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *pos_dev,
                        const int32_t *parent_dev, int64_t v_begin, int64_t v_end, uint64_t *key_dev, void *ws,
                        size_t ws_bytes, void *stream) {
    if (n < 0) return CHORDAL_EINVAL;
    if (n == 0) return CHORDAL_OK;
    if (n > 0x7FFFFFFF) return CHORDAL_ETOOLARGE;
    if (!indptr_dev || !indices_dev || !pos_dev || !key_dev) return CHORDAL_EINVAL;
    if (!ws || ws_bytes < peo_csr_workspace_bytes() || (reinterpret_cast<uintptr_t>(ws) & 15)) return CHORDAL_EINVAL;
    return launch_peo_csr_key(indptr_dev, indices_dev, n, pos_dev, parent_dev, v_begin, v_end, key_dev, ws,
                              as_stream(stream));
}

int chordal_peo_csr_witness(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n,
                            const int32_t *pos_dev, const uint64_t *key_dev, int32_t *witness_dev, void *stream) {
    if (n < 0 || !key_dev || !witness_dev) return CHORDAL_EINVAL;
    if (n == 0) {
        static const int32_t none[3] = {-1, -1, -1};
        return cudaMemcpyAsync(witness_dev, none, sizeof(none), cudaMemcpyHostToDevice, as_stream(stream)) ==
                       cudaSuccess ? CHORDAL_OK : CHORDAL_ECUDA;
    }
    if (!indptr_dev || !indices_dev || !pos_dev) return CHORDAL_EINVAL;
    return launch_peo_csr_witness(indptr_dev, indices_dev, pos_dev, key_dev, witness_dev, as_stream(stream));
}

int chordal_peo_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *pos_dev,
                    const int32_t *parent_dev, uint64_t *key_dev, int32_t *witness_dev, void *ws, size_t ws_bytes,
                    void *stream) {
    int rc = chordal_key_init(key_dev, stream);
    if (rc) return rc;
    rc = chordal_peo_csr_key(indptr_dev, indices_dev, n, pos_dev, parent_dev, 0, n, key_dev, ws, ws_bytes, stream);
    if (rc) return rc;
    return chordal_peo_csr_witness(indptr_dev, indices_dev, n, pos_dev, key_dev, witness_dev, stream);
}

int chordal_left_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *order_dev,
                       const int32_t *pos_dev, uint8_t *ln_rows_dev, int32_t *parent_dev, int32_t *ln_size_dev,
                       int32_t *deg_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    if (!order_dev || !pos_dev) return CHORDAL_EINVAL;
    if (ln_rows_dev && reinterpret_cast<uintptr_t>(ln_rows_dev) % 16 != 0) return CHORDAL_EINVAL;
    return launch_left_dense(adj_dev, n, stride, order_dev, pos_dev, ln_rows_dev, parent_dev, ln_size_dev, deg_dev,
                             as_stream(stream));
}

int chordal_left_csr(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, const int32_t *order_dev,
                     const int32_t *pos_dev, int32_t *parent_dev, int32_t *ln_size_dev, void *stream) {
    if (n < 0) return CHORDAL_EINVAL;
    if (n == 0) return CHORDAL_OK;
    if (n > 0x7FFFFFFF) return CHORDAL_ETOOLARGE;
    if (!indptr_dev || !indices_dev || !order_dev || !pos_dev) return CHORDAL_EINVAL;
    return launch_left_csr(indptr_dev, indices_dev, n, order_dev, pos_dev, parent_dev, ln_size_dev,
                           as_stream(stream));
}

int chordal_dense_to_csr(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t *indptr_dev,
                         int32_t *indices_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!indptr_dev) return CHORDAL_EINVAL;
    if (n == 0) return cudaMemsetAsync(indptr_dev, 0, sizeof(int64_t), as_stream(stream)) == cudaSuccess
                           ? CHORDAL_OK : CHORDAL_ECUDA;
    rc = launch_dense_degrees(adj_dev, n, stride, indptr_dev, as_stream(stream));
    if (rc || !indices_dev) return rc;
    return launch_dense_fill(adj_dev, n, stride, indptr_dev, indices_dev, INT64_MAX, as_stream(stream));
}

int chordal_permute_dense(const uint8_t *adj_dev, int64_t n, int64_t stride, const int32_t *perm_dev,
                          uint8_t *out_dev, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (n == 0) return CHORDAL_OK;
    rc = check_dense(out_dev, n, stride);
    if (rc) return rc;
    if (!perm_dev || out_dev == adj_dev) return CHORDAL_EINVAL;
    return launch_permute_dense(adj_dev, n, stride, perm_dev, out_dev, as_stream(stream));
}

int chordal_is_chordal_batch(const uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride,
                             int32_t *orders_dev, int32_t *witness_dev, void *stream) {
    if (batch < 0 || n < 0) return CHORDAL_EINVAL;
    if (batch == 0) return CHORDAL_OK;
    if (n == 0) {  // every empty graph is chordal: witness (-1, -1, -1)
        if (!witness_dev) return CHORDAL_EINVAL;
        return cudaMemsetAsync(witness_dev, 0xFF, sizeof(int32_t) * 3 * (size_t)batch, as_stream(stream)) ==
                       cudaSuccess ? CHORDAL_OK : CHORDAL_ECUDA;
    }
    if (n > CHORDAL_BATCH_MAX_N) return CHORDAL_ETOOLARGE;
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!orders_dev || !witness_dev) return CHORDAL_EINVAL;
    return launch_batch(adj_dev, batch, n, stride, orders_dev, witness_dev, as_stream(stream));
}

static size_t batch_host_set_bytes(int64_t n, int64_t chunk) {
    const int64_t stride = (((n + 7) / 8) + 15) / 16 * 16;
    // + staging for host rows narrower than the device pitch (spread on the device)
    const size_t stage = stride != (n + 7) / 8 ? (((size_t)n * stride * chunk + 255) & ~size_t(255)) : 0;
    return ((size_t)n * stride * chunk + sizeof(int32_t) * (size_t)(n + 3) * chunk + 1023 + stage) & ~size_t(255);
}

size_t chordal_batch_host_workspace_bytes(int64_t n, int64_t chunk) {
    if (n <= 0) return 0;
    if (chunk <= 0) chunk = 4096;
    return 3 * batch_host_set_bytes(n, chunk);
}

// The host-buffer batch over a caller-provided device block (three chunk-sized
// sets: graphs, orders, witnesses) and three per-call streams.
static int batch_host_run(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes, int32_t *orders_host,
                          int32_t *witness_host, int64_t chunk, uint8_t *block, cudaStream_t home) {
    const int64_t stride = (((n + 7) / 8) + 15) / 16 * 16;
    const size_t gbytes = (size_t)n * stride;
    constexpr int NB = 3;  // H2D of chunk c+1 and D2H of c-1 overlap the search of c
    const size_t per_set = batch_host_set_bytes(n, chunk);
    // one flat copy only when host rows, device rows and the vertex bytes coincide;
    // otherwise (n+7)/8 bytes per row into rows whose padding was zeroed once
    const bool flat = row_bytes == stride && stride == (n + 7) / 8;
    cudaEvent_t ready = nullptr;
    cudaStream_t st[NB] = {};
    uint8_t *buf[NB] = {};
    int32_t *ord[NB] = {};
    int32_t *wit[NB] = {};
    uint8_t *stg[NB] = {};
    // narrower host rows: one flat copy per chunk and a spread kernel (a pitched
    // copy from pageable memory is staged row by row by the driver)
    const bool spread = !flat && row_bytes <= stride && stride != (n + 7) / 8;
    int rc = CHORDAL_OK;
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ready, home) != cudaSuccess)
        rc = CHORDAL_ECUDA;
    for (int k = 0; k < NB && rc == CHORDAL_OK; ++k) {
        uint8_t *base = block + k * per_set;
        buf[k] = base;
        ord[k] = reinterpret_cast<int32_t *>(base + ((gbytes * chunk + 255) & ~size_t(255)));
        wit[k] = ord[k] + (size_t)n * chunk;
        stg[k] = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(wit[k] + 3 * chunk) + 255) & ~uintptr_t(255));
        if (cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamWaitEvent(st[k], ready, 0) != cudaSuccess) {
            rc = CHORDAL_ECUDA;
            break;
        }
        if (!flat && !spread && cudaMemsetAsync(buf[k], 0, gbytes * chunk, st[k]) != cudaSuccess)
            rc = CHORDAL_ECUDA;
    }
    for (int64_t b0 = 0, c = 0; b0 < batch && rc == CHORDAL_OK; b0 += chunk, ++c) {
        const int k = (int)(c % NB);
        const int64_t nb = (batch - b0 < chunk) ? batch - b0 : chunk;
        const uint8_t *src = adj_host + b0 * n * row_bytes;
        cudaError_t e = flat     ? cudaMemcpyAsync(buf[k], src, gbytes * nb, cudaMemcpyHostToDevice, st[k])
                        : spread ? cudaMemcpyAsync(stg[k], src, (size_t)n * nb * row_bytes, cudaMemcpyHostToDevice,
                                                   st[k])
                                 : cudaMemcpy2DAsync(buf[k], stride, src, row_bytes, (n + 7) / 8, n * nb,
                                                     cudaMemcpyHostToDevice, st[k]);
        if (e != cudaSuccess) { rc = CHORDAL_ECUDA; break; }
        if (spread && (rc = launch_spread_rows(stg[k], row_bytes, n * nb, (n + 7) / 8, stride, buf[k], st[k])))
            break;
        rc = launch_batch(buf[k], nb, n, stride, ord[k], wit[k], st[k]);
        if (rc) break;
        if (cudaMemcpyAsync(orders_host + b0 * n, ord[k], sizeof(int32_t) * n * nb, cudaMemcpyDeviceToHost,
                            st[k]) != cudaSuccess ||
            cudaMemcpyAsync(witness_host + 3 * b0, wit[k], sizeof(int32_t) * 3 * nb, cudaMemcpyDeviceToHost,
                            st[k]) != cudaSuccess)
            rc = CHORDAL_ECUDA;
    }
    for (int k = 0; k < NB; ++k) {
        if (!st[k]) continue;
        if (cudaStreamSynchronize(st[k]) != cudaSuccess && rc == CHORDAL_OK) rc = CHORDAL_ECUDA;
        cudaStreamDestroy(st[k]);
    }
    if (ready) cudaEventDestroy(ready);
    return rc;
}

static int batch_host_check(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes,
                            int32_t *orders_host, int32_t *witness_host) {
    if (batch < 0 || n < 0 || (batch > 0 && (!witness_host || (n > 0 && (!adj_host || !orders_host)))))
        return CHORDAL_EINVAL;
    if (batch == 0) return -1;  // nothing to do
    if (n == 0) {  // every empty graph is chordal
        for (int64_t b = 0; b < 3 * batch; ++b) witness_host[b] = -1;
        return -1;
    }
    if (n > CHORDAL_BATCH_MAX_N) return CHORDAL_ETOOLARGE;
    if (row_bytes < (n + 7) / 8) return CHORDAL_EINVAL;
    return CHORDAL_OK;
}

int chordal_is_chordal_batch_host(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes,
                                  int32_t *orders_host, int32_t *witness_host, int64_t chunk) {
    int rc = batch_host_check(adj_host, batch, n, row_bytes, orders_host, witness_host);
    if (rc) return rc < 0 ? CHORDAL_OK : rc;
    if (chunk <= 0) chunk = 4096;
    if (chunk > batch) chunk = batch;
    // one stream-ordered block per call on the calling thread's default stream
    // (see chordal_is_chordal_batch_host_ws for the jitter-free form)
    const size_t wsb = chordal_batch_host_workspace_bytes(n, chunk);
    cudaStream_t home = cudaStreamPerThread;
    uint8_t *block = nullptr;
    if (cudaMallocAsync((void **)&block, wsb, home) != cudaSuccess) return CHORDAL_ENOMEM;
    rc = batch_host_run(adj_host, batch, n, row_bytes, orders_host, witness_host, chunk, block, home);
    cudaFreeAsync(block, home);
    if (cudaStreamSynchronize(home) != cudaSuccess && rc == CHORDAL_OK) rc = CHORDAL_ECUDA;
    return rc;
}

int chordal_is_chordal_batch_host_ws(const uint8_t *adj_host, int64_t batch, int64_t n, int64_t row_bytes,
                                     int32_t *orders_host, int32_t *witness_host, int64_t chunk, void *ws_dev,
                                     size_t ws_bytes) {
    int rc = batch_host_check(adj_host, batch, n, row_bytes, orders_host, witness_host);
    if (rc) return rc < 0 ? CHORDAL_OK : rc;
    if (chunk <= 0) chunk = 4096;
    if (chunk > batch) chunk = batch;
    if (!ws_dev || ws_bytes < chordal_batch_host_workspace_bytes(n, chunk) ||
        (reinterpret_cast<uintptr_t>(ws_dev) & 255))
        return CHORDAL_EINVAL;
    cudaStream_t home = cudaStreamPerThread;
    return batch_host_run(adj_host, batch, n, row_bytes, orders_host, witness_host, chunk,
                          reinterpret_cast<uint8_t *>(ws_dev), home);
}

int chordal_gen_dense_random(uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride, double p,
                             int64_t seed0, int64_t seed_step, void *stream) {
    if (batch < 0 || n < 0) return CHORDAL_EINVAL;
    if (batch == 0 || n == 0) return CHORDAL_OK;
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!(p > 0.0 && p <= 1.0)) return CHORDAL_EINVAL;
    if (n == 1) return cudaMemsetAsync(adj_dev, 0, (size_t)batch * stride, as_stream(stream)) == cudaSuccess
                          ? CHORDAL_OK : CHORDAL_ECUDA;
    return launch_gen_dense_random(adj_dev, batch, n, stride, p, seed0, seed_step,
                                   crc32_str("dense-random"), as_stream(stream));
}

int chordal_edges_to_dense(const int32_t *u_dev, const int32_t *v_dev, int64_t m, uint8_t *adj_dev, int64_t n,
                           int64_t stride, void *stream) {
    if (m < 0 || (m > 0 && (!u_dev || !v_dev))) return CHORDAL_EINVAL;
    if (n == 0) return m == 0 ? CHORDAL_OK : CHORDAL_EINVAL;
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    return launch_edges_to_dense(u_dev, v_dev, m, adj_dev, n, stride, as_stream(stream));
}

int chordal_gen_chordal_random_edges(int64_t n, int64_t k, int64_t seed, int32_t *u_dev, int32_t *v_dev,
                                     int64_t *m_dev, void *scratch_dev, size_t scratch_bytes, void *stream) {
    if (n < 1 || k < 0 || k >= n || !u_dev || !v_dev || !m_dev) return CHORDAL_EINVAL;
    if (k + 2 > 10000 || n > 0x7FFFFFFF / (k + 2)) return CHORDAL_EINVAL;
    if (!scratch_dev || scratch_bytes < chordal_gen_chordal_random_scratch_bytes(1, n, k)) return CHORDAL_EINVAL;
    return launch_gen_chordal_edges(n, k, seed, crc32_str("chordal-random"), reinterpret_cast<int32_t *>(scratch_dev),
                                    u_dev, v_dev, reinterpret_cast<long long *>(m_dev), as_stream(stream));
}

size_t chordal_gen_chordal_random_scratch_bytes(int64_t batch, int64_t n, int64_t k) {
    if (batch <= 0 || n <= 0 || k < 0) return 0;
    return (size_t)batch * (size_t)gen_chordal_scratch_words(n, k, nullptr) * sizeof(int32_t);
}

int chordal_gen_chordal_random(uint8_t *adj_dev, int64_t batch, int64_t n, int64_t stride, int64_t k, int64_t seed0,
                               int64_t seed_step, void *scratch_dev, size_t scratch_bytes, void *stream) {
    if (batch < 0 || n < 1 || k < 0 || k >= n) return CHORDAL_EINVAL;
    if (batch == 0) return CHORDAL_OK;
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (k + 2 > 10000) return CHORDAL_EINVAL;  // numpy switches choice() algorithm above this pool size
    if (!scratch_dev || scratch_bytes < chordal_gen_chordal_random_scratch_bytes(batch, n, k)) return CHORDAL_EINVAL;
    return launch_gen_chordal_random(adj_dev, batch, n, stride, k, seed0, seed_step, crc32_str("chordal-random"),
                                     reinterpret_cast<int32_t *>(scratch_dev), as_stream(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-GPU (row-sharded PEO check) over the caller's NCCL communicator.
//
// The protocol of distributed.sharded_is_chordal, for callers without torch:
// the root rank runs LexBFS (a single graph's step chain stays on one GPU),
// order + parents are broadcast, every rank checks its contiguous row shard
// [n r / W, n (r + 1) / W), one 8-byte MIN all-reduce of the witness key, and
// every rank resolves z locally.  NCCL is not linked: its entry points are
// resolved from the process (the library that created `comm`, found by its
// soname) at the first call, so libchordal_b200.so loads without NCCL.
namespace {

// nccl.h enum values (stable across NCCL 2.x)
constexpr int kNcclInt32 = 2, kNcclUint64 = 5, kNcclMin = 3;

struct NcclApi {
    typedef int (*count_t)(void *, int *);
    typedef int (*bcast_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
    typedef int (*allred_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
    typedef int (*group_t)();
    count_t count = nullptr, user_rank = nullptr;
    bcast_t bcast = nullptr;
    allred_t allreduce = nullptr;
    group_t gstart = nullptr, gend = nullptr;
    bool ok = false;
};

const NcclApi &nccl_api() {
    // resolved once; read-only afterwards (a function-local static: thread-safe
    // initialisation, no mutable state after it)
    static const NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return a;
        a.count = (NcclApi::count_t)dlsym(h, "ncclCommCount");
        a.user_rank = (NcclApi::count_t)dlsym(h, "ncclCommUserRank");
        a.bcast = (NcclApi::bcast_t)dlsym(h, "ncclBroadcast");
        a.allreduce = (NcclApi::allred_t)dlsym(h, "ncclAllReduce");
        a.gstart = (NcclApi::group_t)dlsym(h, "ncclGroupStart");
        a.gend = (NcclApi::group_t)dlsym(h, "ncclGroupEnd");
        a.ok = a.count && a.user_rank && a.bcast && a.allreduce && a.gstart && a.gend;
        return a;
    }();
    return api;
}

struct ShardWs {  // key + parent, then the LexBFS workspace
    size_t key, parent, rest, total;
    ShardWs(int64_t n, size_t rest_bytes) {
        auto a = [](size_t x) { return (x + 255) & ~size_t(255); };
        key = 0;
        parent = 256;
        rest = a(parent + sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
        total = rest + rest_bytes;
    }
};

// order + parent from the root, positions, this rank's shard of the key, MIN
// all-reduce.  `key_fn(lo, hi)` launches the shard's key kernel.
template <typename KeyFn>
int shard_exchange(const NcclApi &api, void *comm, int root, int64_t n, int32_t *order, int32_t *pos,
                   int32_t *parent, uint64_t *key, cudaStream_t s, KeyFn key_fn) {
    int world = 0, rank = 0;
    if (api.count(comm, &world) || api.user_rank(comm, &rank) || world <= 0) return CHORDAL_ENCCL;
    if (api.gstart()) return CHORDAL_ENCCL;
    const int b1 = api.bcast(order, order, (size_t)n, kNcclInt32, root, comm, s);
    const int b2 = api.bcast(parent, parent, (size_t)n, kNcclInt32, root, comm, s);
    if (api.gend() || b1 || b2) return CHORDAL_ENCCL;
    int rc = launch_positions(order, n, pos, s);
    if (rc) return rc;
    rc = launch_key_init(key, s);
    if (rc) return rc;
    // distributed.shard_bounds: contiguous, balanced to +-1
    const int64_t base = n / world, extra = n % world;
    const int64_t lo = rank * base + (rank < extra ? rank : extra), hi = lo + base + (rank < extra ? 1 : 0);
    if (lo < hi) {
        rc = key_fn(lo, hi);
        if (rc) return rc;
    }
    // UINT64_MAX ("no violation") is the MIN identity of the unsigned key
    if (api.allreduce(key, key, 1, kNcclUint64, kNcclMin, comm, s)) return CHORDAL_ENCCL;
    return CHORDAL_OK;
}

}  // namespace

size_t chordal_dense_nccl_workspace_bytes(int64_t n, int64_t m) {
    return ShardWs(n, DenseWs(n, m < 0 ? 0 : m).total).total;
}

int chordal_is_chordal_dense_nccl(const uint8_t *adj_dev, int64_t n, int64_t stride, int64_t m, int32_t tie_rule,
                                  uint64_t seed, int32_t root, void *nccl_comm, int32_t *order_dev, int32_t *pos_dev,
                                  int32_t *witness_dev, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_dense(adj_dev, n, stride);
    if (rc) return rc;
    if (!nccl_comm || !witness_dev || root < 0) return CHORDAL_EINVAL;
    cudaStream_t s = as_stream(stream);
    if (n == 0) return cudaMemsetAsync(witness_dev, 0xFF, 3 * sizeof(int32_t), s) == cudaSuccess ? CHORDAL_OK
                                                                                                  : CHORDAL_ECUDA;
    if (!order_dev || !pos_dev || !ws) return CHORDAL_EINVAL;
    if (!use_seg(n, m) && m < 0) return CHORDAL_EINVAL;  // every rank sizes the same workspace
    const ShardWs L(n, DenseWs(n, m < 0 ? 0 : m).total);
    if (ws_bytes < L.total) return CHORDAL_EINVAL;
    const NcclApi &api = nccl_api();
    if (!api.ok) return CHORDAL_ENCCL;
    int world = 0, rank = 0;
    if (api.count(nccl_comm, &world) || api.user_rank(nccl_comm, &rank)) return CHORDAL_ENCCL;
    if (root >= world) return CHORDAL_EINVAL;
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    uint64_t *key = reinterpret_cast<uint64_t *>(w + L.key);
    int32_t *parent = reinterpret_cast<int32_t *>(w + L.parent);
    if (rank == root) {
        // the CTA engine leaves the parents to the PEO check (-2 = search them)
        if (use_seg(n, m)) {
            rc = launch_fill_i32(parent, n, -2, s);
            if (rc) return rc;
        }
        rc = chordal_lexbfs_dense(adj_dev, n, stride, m, tie_rule, seed, order_dev, pos_dev,
                                  use_seg(n, m) ? nullptr : parent, w + L.rest, ws_bytes - L.rest, stream);
        if (rc) return rc;
    }
    rc = shard_exchange(api, nccl_comm, root, n, order_dev, pos_dev, parent, key, s, [&](int64_t lo, int64_t hi) {
        return launch_peo_dense_key(adj_dev, n, stride, order_dev, pos_dev, parent, lo, hi, key, s);
    });
    if (rc) return rc;
    return launch_peo_dense_witness(adj_dev, n, stride, pos_dev, key, witness_dev, s);
}

size_t chordal_csr_nccl_workspace_bytes(int64_t n, int64_t m) {
    const size_t peo = (peo_csr_workspace_bytes() + 255) & ~size_t(255);
    return ShardWs(n, peo + csr_workspace_bytes(n, m < 0 ? 0 : m)).total;
}

int chordal_is_chordal_csr_nccl(const int64_t *indptr_dev, const int32_t *indices_dev, int64_t n, int64_t m,
                                int32_t tie_rule, uint64_t seed, int32_t root, void *nccl_comm, int32_t *order_dev,
                                int32_t *pos_dev, int32_t *witness_dev, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || m < 0 || !nccl_comm || !witness_dev || root < 0) return CHORDAL_EINVAL;
    cudaStream_t s = as_stream(stream);
    if (n == 0) return cudaMemsetAsync(witness_dev, 0xFF, 3 * sizeof(int32_t), s) == cudaSuccess ? CHORDAL_OK
                                                                                                  : CHORDAL_ECUDA;
    if (!indptr_dev || !indices_dev || !order_dev || !pos_dev || !ws) return CHORDAL_EINVAL;
    const size_t peo = (peo_csr_workspace_bytes() + 255) & ~size_t(255);
    const ShardWs L(n, peo + csr_workspace_bytes(n, m));
    if (ws_bytes < L.total) return CHORDAL_EINVAL;
    const NcclApi &api = nccl_api();
    if (!api.ok) return CHORDAL_ENCCL;
    int world = 0, rank = 0;
    if (api.count(nccl_comm, &world) || api.user_rank(nccl_comm, &rank)) return CHORDAL_ENCCL;
    if (root >= world) return CHORDAL_EINVAL;
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    uint64_t *key = reinterpret_cast<uint64_t *>(w + L.key);
    int32_t *parent = reinterpret_cast<int32_t *>(w + L.parent);
    uint8_t *peo_ws = w + L.rest;
    int rc;
    if (rank == root) {
        rc = chordal_lexbfs_csr(indptr_dev, indices_dev, n, m, tie_rule, seed, order_dev, pos_dev, parent,
                                peo_ws + peo, ws_bytes - L.rest - peo, stream);
        if (rc) return rc;
    }
    rc = shard_exchange(api, nccl_comm, root, n, order_dev, pos_dev, parent, key, s, [&](int64_t lo, int64_t hi) {
        return chordal_peo_csr_key(indptr_dev, indices_dev, n, pos_dev, parent, lo, hi, key, peo_ws, peo, stream);
    });
    if (rc) return rc;
    return launch_peo_csr_witness(indptr_dev, indices_dev, pos_dev, key, witness_dev, s);
}
