// api.cu -- C-ABI entry points of libnnqs (include/nnqs.h): argument
// validation, handle lifetime, device selection, error reporting.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "internal.h"

namespace {
thread_local std::string g_last_error;

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// The library's own stream-ordered memory pool, one per device, created once
// (thread-safe).  Its release threshold keeps freed blocks for reuse by the next
// call (the per-call scratch is large and the call repeats every VMC step); the
// device's default pool -- shared with PyTorch / NCCL -- is not touched.
std::once_flag g_pool_once[64];
cudaMemPool_t g_pool[64] = {};

cudaMemPool_t library_pool(int device) {
    if (device < 0 || device >= 64) return nullptr;
    std::call_once(g_pool_once[device], [device]() {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            g_pool[device] = pool;
        }
    });
    return g_pool[device];
}

int check_symmetry(const double *h1, const double *h2, int n) {
    double mx = 0.0;
    for (size_t i = 0; i < (size_t)n * n; ++i) mx = std::fmax(mx, std::fabs(h1[i]));
    const size_t n4 = (size_t)n * n * n * n;
    for (size_t i = 0; i < n4; ++i) mx = std::fmax(mx, std::fabs(h2[i]));
    for (size_t i = 0; i < (size_t)n * n; ++i)
        if (!std::isfinite(h1[i])) return nnqs_set_error(NNQS_E_ARG, "h1 has a non-finite entry");
    for (size_t i = 0; i < n4; ++i)
        if (!std::isfinite(h2[i])) return nnqs_set_error(NNQS_E_ARG, "h2 has a non-finite entry");
    const double tol = 1e-12 * (mx > 0 ? mx : 1.0);
    for (int p = 0; p < n; ++p)
        for (int q = 0; q < n; ++q)
            if (std::fabs(h1[p * n + q] - h1[q * n + p]) > tol)
                return nnqs_set_error(NNQS_E_SYMMETRY, "h1 is not symmetric");
    auto G = [&](int p, int q, int r, int s) { return h2[(((size_t)p * n + q) * n + r) * n + s]; };
    for (int p = 0; p < n; ++p)
        for (int q = 0; q < n; ++q)
            for (int r = 0; r < n; ++r)
                for (int s = 0; s < n; ++s) {
                    const double v = G(p, q, r, s);
                    const double o[7] = {G(q, p, r, s), G(p, q, s, r), G(q, p, s, r), G(r, s, p, q),
                                         G(s, r, p, q), G(r, s, q, p), G(s, r, q, p)};
                    for (double w : o)
                        if (std::fabs(v - w) > tol)
                            return nnqs_set_error(NNQS_E_SYMMETRY, "h2 lacks the 8-fold symmetry of real orbitals");
                }
    return NNQS_OK;
}

int finish_ham(nnqs_ham h, int device, nnqs_ham *out) {
    h->device = device;
    nnqs_spin_index_build(h->host, h->spin);
    h->n_groups = (int64_t)h->host.off.size() - 1;
    h->n_terms = (int64_t)h->host.d.size();
    if (device < 0) {          // host-only handle: export / info only
        *out = h;
        return NNQS_OK;
    }
    DeviceGuard g(device);
    if (!g.ok) return nnqs_set_error(NNQS_E_CUDA, "cudaSetDevice failed");
    int rc = nnqs_ham_upload(h);
    if (!rc) rc = nnqs_spin_index_upload(h);
    if (rc) {
        nnqs_spin_index_release(h);
        nnqs_ham_release(h);
        delete h;
        return rc;
    }
    *out = h;
    return NNQS_OK;
}
}  // namespace

cudaError_t nnqs_malloc_async(void **p, size_t bytes, cudaStream_t st) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = library_pool(dev);
    if (!pool) return cudaMallocAsync(p, bytes, st);   // pool creation failed: the default pool
    return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

int nnqs_set_error(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

void nnqs_hash_columns(u64 cols[128]) {
    u64 s = 0x5EED0F2306167050ULL;
    for (int j = 0; j < 128; ++j) cols[j] = nnqs_splitmix64(s);
}

void nnqs_filter_columns(uint32_t cols[128]) {
    u64 s = 0xF117E2306167051ULL;
    for (int j = 0; j < 128; ++j) cols[j] = (uint32_t)(nnqs_splitmix64(s) >> 32);
}

u64 nnqs_hash_host(const u64 cols[128], u64 lo, u64 hi) {
    u64 h = 0;
    for (int j = 0; j < 64; ++j)
        if (lo >> j & 1) h ^= cols[j];
    for (int j = 0; j < 64; ++j)
        if (hi >> j & 1) h ^= cols[64 + j];
    return h;
}

extern "C" {

const char *nnqs_last_error(void) { return g_last_error.c_str(); }

const char *nnqs_version(void) { return "libnnqs 0.1 (sm_100a; local-energy hot path of arXiv 2306.16705)"; }

int nnqs_ham_compress(const double *h1, const double *h2, int n_spin_orbitals, double e_core,
                      double tol, int device, nnqs_ham *out) {
    if (!h1 || !h2 || !out) return nnqs_set_error(NNQS_E_ARG, "nnqs_ham_compress: null pointer");
    *out = nullptr;
    if (n_spin_orbitals <= 0 || (n_spin_orbitals & 1) || n_spin_orbitals > 128)
        return nnqs_set_error(NNQS_E_SIZE, "n_spin_orbitals must be even and in [2, 128]");
    if (!(tol >= 0.0) || !std::isfinite(e_core))
        return nnqs_set_error(NNQS_E_ARG, "tol must be >= 0 and e_core finite");
    const int n = n_spin_orbitals / 2;
    int rc = check_symmetry(h1, h2, n);
    if (rc) return rc;
    nnqs_ham h = new (std::nothrow) nnqs_ham_s();
    if (!h) return nnqs_set_error(NNQS_E_NOMEM, "host allocation failed");
    try {
        rc = nnqs_compress_host(h1, h2, n, e_core, tol, h->host);
    } catch (const std::bad_alloc &) {
        rc = nnqs_set_error(NNQS_E_NOMEM, "host allocation failed in compress");
    }
    if (rc) {
        delete h;
        return rc;
    }
    return finish_ham(h, device, out);
}

int nnqs_ham_from_pauli(const uint64_t *xmask, const uint64_t *zmask, const double *coeff_re,
                        const double *coeff_im, int64_t n_terms, int n_qubits, double tol,
                        int device, nnqs_ham *out) {
    if (!out || n_terms < 0 || (n_terms > 0 && (!xmask || !zmask || !coeff_re)))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_ham_from_pauli: bad arguments");
    *out = nullptr;
    if (n_qubits <= 0 || n_qubits > 128) return nnqs_set_error(NNQS_E_SIZE, "n_qubits must be in [1, 128]");
    if (!(tol >= 0.0)) return nnqs_set_error(NNQS_E_ARG, "tol must be >= 0");
    nnqs_ham h = new (std::nothrow) nnqs_ham_s();
    if (!h) return nnqs_set_error(NNQS_E_NOMEM, "host allocation failed");
    int rc = nnqs_from_pauli_host((const u64 *)xmask, (const u64 *)zmask, coeff_re, coeff_im, n_terms,
                                  n_qubits, tol, h->host);
    if (rc) {
        delete h;
        return rc;
    }
    return finish_ham(h, device, out);
}

int nnqs_ham_info(nnqs_ham h, int *n_qubits, int64_t *n_groups, int64_t *n_terms, int64_t *device_bytes) {
    if (!h) return nnqs_set_error(NNQS_E_ARG, "nnqs_ham_info: null handle");
    if (n_qubits) *n_qubits = h->host.n_qubits;
    if (n_groups) *n_groups = h->n_groups;
    if (n_terms) *n_terms = h->n_terms;
    if (device_bytes) *device_bytes = h->dev.bytes;
    return NNQS_OK;
}

int nnqs_ham_export(nnqs_ham h, uint64_t *xmask, int64_t *offsets, uint64_t *zmask, double *coeff) {
    if (!h) return nnqs_set_error(NNQS_E_ARG, "nnqs_ham_export: null handle");
    const HostTable &H = h->host;
    if (xmask) std::memcpy(xmask, H.x.data(), H.x.size() * 8);
    if (offsets) std::memcpy(offsets, H.off.data(), H.off.size() * 8);
    if (zmask) std::memcpy(zmask, H.z.data(), H.z.size() * 8);
    if (coeff) std::memcpy(coeff, H.d.data(), H.d.size() * 8);
    return NNQS_OK;
}

int nnqs_ham_free(nnqs_ham h) {
    if (!h) return NNQS_OK;
    if (h->device >= 0) {
        DeviceGuard g(h->device);
        nnqs_spin_index_release(h);     // before nnqs_ham_release resets the DeviceHam
        nnqs_ham_release(h);
    }
    delete h;
    return NNQS_OK;
}

void nnqs_options_default(nnqs_options *opt) {
    if (!opt) return;
    std::memset(opt, 0, sizeof(*opt));
    opt->algorithm = NNQS_ALGO_AUTO;
    opt->thr_single = 128;     // measured (step ms): 96 63.52, 128 63.45, 192 63.67, 256 64.15
    opt->thr_double = 8192;    // measured (step ms): 2048 69.46, 4096 63.51, 8192 63.15
    opt->thr_rowheavy = 16384; // DESIGN.md Sec. 7 (entry-driven join below 16384 rows: slower)
}

int nnqs_table_prepare(nnqs_ham h, int mode, const uint64_t *keys, const double *logpsi, int64_t n,
                       void *cuda_stream, nnqs_table *out) {
    return nnqs_table_prepare_ex(h, mode, keys, logpsi, n, nullptr, cuda_stream, out);
}

int nnqs_table_prepare_ex(nnqs_ham h, int mode, const uint64_t *keys, const double *logpsi, int64_t n,
                          const nnqs_options *opt, void *cuda_stream, nnqs_table *out) {
    if (!h || !out || n < 0 || (mode != 0 && mode != 1) || (n > 0 && !logpsi))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_table_prepare: bad arguments");
    if (h->device < 0) return nnqs_set_error(NNQS_E_ARG, "host-only Hamiltonian (device < 0)");
    *out = nullptr;
    nnqs_options o;
    nnqs_options_default(&o);
    if (opt) {
        for (int32_t r : opt->reserved)
            if (r) return nnqs_set_error(NNQS_E_ARG, "nnqs_options.reserved must be zero");
        if (opt->algorithm != NNQS_ALGO_AUTO && opt->algorithm != NNQS_ALGO_LITERAL)
            return nnqs_set_error(NNQS_E_ARG, "nnqs_options.algorithm must be 0 or 1");
        if (opt->literal_kernel < 0 || opt->literal_kernel > NNQS_LIT_PLAIN)
            return nnqs_set_error(NNQS_E_ARG, "nnqs_options.literal_kernel must be 0, 1 or 2");
        o.literal_kernel = opt->literal_kernel;
        if (opt->thr_single < 0 || opt->thr_double < 0 || opt->thr_rowheavy < 0)
            return nnqs_set_error(NNQS_E_ARG, "nnqs_options thresholds must be >= 0");
        o.algorithm = opt->algorithm;
        if (opt->thr_single) o.thr_single = opt->thr_single;
        if (opt->thr_double) o.thr_double = opt->thr_double;
        if (opt->thr_rowheavy) o.thr_rowheavy = opt->thr_rowheavy;
    }
    if (o.thr_rowheavy < o.thr_single) o.thr_rowheavy = o.thr_single;   // join rows must be in the multimap
    if (mode == 0 && n > 0 && !keys) return nnqs_set_error(NNQS_E_ARG, "sample-aware mode needs keys");
    if (mode == 0 && n >= (int64_t)0xFFFFFFFFLL) return nnqs_set_error(NNQS_E_SIZE, "table larger than 2^32-1 keys");
    if (mode == 1) {
        const int N = h->host.n_qubits;
        if (N > 30) return nnqs_set_error(NNQS_E_SIZE, "exact mode needs N <= 30");
        if (n != ((int64_t)1 << N)) return nnqs_set_error(NNQS_E_ARG, "exact mode needs n = 2^N");
    }
    nnqs_table t = new (std::nothrow) nnqs_table_s();
    if (!t) return nnqs_set_error(NNQS_E_NOMEM, "host allocation failed");
    t->mode = mode;
    t->n = n;
    t->device = h->device;
    t->stream = cuda_stream;
    t->opt = o;
    DeviceGuard g(h->device);
    if (!g.ok) {
        delete t;
        return nnqs_set_error(NNQS_E_CUDA, "cudaSetDevice failed");
    }
    int rc = NNQS_OK;
    for (int i = 0; i < 3 && !rc; ++i) {
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
            rc = nnqs_set_error(NNQS_E_CUDA, "cudaStreamCreate failed");
        t->own[i] = s;
    }
    cudaEvent_t ev = nullptr;
    if (!rc && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        rc = nnqs_set_error(NNQS_E_CUDA, "cudaEventCreate failed");
    t->last_use = ev;
    bool checked = false;   // the order / exp-ratio flags are read at the spin build's first sync
    if (!rc) rc = nnqs_table_build(t, keys, logpsi, cuda_stream, /*defer_check=*/mode == 0);
    if (!rc && mode == 0) rc = nnqs_table_build_spin(h, t, cuda_stream, &checked);
    if (!rc && mode == 0 && !checked && n) rc = nnqs_table_check(t, nullptr, cuda_stream);
    if (!rc) cudaEventRecord((cudaEvent_t)t->last_use, (cudaStream_t)cuda_stream);
    if (rc) {
        cudaStreamSynchronize((cudaStream_t)cuda_stream);
        nnqs_table_free(t);
        return rc;
    }
    *out = t;
    return NNQS_OK;
}

int nnqs_table_free(nnqs_table t) {
    if (!t) return NNQS_OK;
    {
        DeviceGuard g(t->device);
        // release on the table's own stream, ordered after the last call that used it
        cudaStream_t rs = (cudaStream_t)t->own[0];
        if (rs && t->last_use) cudaStreamWaitEvent(rs, (cudaEvent_t)t->last_use, 0);
        t->stream = rs;
        nnqs_table_release_spin(t);
        nnqs_table_release(t);
        for (void *&s : t->own)
            if (s) { cudaStreamDestroy((cudaStream_t)s); s = nullptr; }   // pending frees still complete
        if (t->last_use) cudaEventDestroy((cudaEvent_t)t->last_use);
        t->last_use = nullptr;
    }
    delete t;
    return NNQS_OK;
}

int nnqs_table_set_algorithm(nnqs_table t, int algorithm) {
    if (!t) return nnqs_set_error(NNQS_E_ARG, "nnqs_table_set_algorithm: null table");
    if (algorithm != NNQS_ALGO_AUTO && algorithm != NNQS_ALGO_LITERAL)
        return nnqs_set_error(NNQS_E_ARG, "algorithm must be 0 or 1");
    t->opt.algorithm = algorithm;
    return NNQS_OK;
}

int nnqs_table_info(nnqs_table t, int64_t *n, double *shift, int64_t *device_bytes) {
    if (!t) return nnqs_set_error(NNQS_E_ARG, "nnqs_table_info: null handle");
    if (n) *n = t->n;
    if (device_bytes) *device_bytes = t->bytes;
    if (shift) {
        DeviceGuard g(t->device);
        cudaStream_t rs = (cudaStream_t)t->own[0];
        u64 k = 0;
        cudaError_t e = cudaStreamWaitEvent(rs, (cudaEvent_t)t->last_use, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&k, t->shift_key, 8, cudaMemcpyDeviceToHost, rs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(rs);
        if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
        if (k == 0) *shift = 0.0;
        else {
            u64 b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
            std::memcpy(shift, &b, 8);
        }
    }
    return NNQS_OK;
}

namespace {
bool structured_rows(nnqs_ham h, nnqs_table t, const uint64_t *rows) {
    return !rows && t->spin_ready && h->spin.ok && t->opt.algorithm != NNQS_ALGO_LITERAL;
}

// One local-energy launch sequence (both algorithms), the fused Eq. (6) chunk
// partials and the hit log included; records the table's last-use event.
int local_energy_impl(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows, const double *row_logpsi,
                      int64_t n_rows, double *eloc_out, const int64_t *counts, double *partials_out,
                      int64_t *stats_out, const HitLogHost &lg, void *cuda_stream) {
    cudaStream_t st = (cudaStream_t)cuda_stream;
    ChunkSink cs;
    unsigned *ctr = nullptr;
    int rc = NNQS_OK;
    if (partials_out && n_rows > 0) {
        const int64_t nch = (n_rows + NNQS_REDUCE_CHUNK - 1) / NNQS_REDUCE_CHUNK;
        cudaError_t e = nnqs_malloc_async((void **)&ctr, 4 * (size_t)nch, st);
        if (e != cudaSuccess) return nnqs_set_error(NNQS_E_NOMEM, cudaGetErrorString(e));
        cudaMemsetAsync(ctr, 0, 4 * (size_t)nch, st);
        cs.counts = counts;
        cs.partials = partials_out;
        cs.ctr = ctr;
    }
    if (n_rows > 0) {
        if (structured_rows(h, t, rows))
            rc = nnqs_launch_local_energy_spin(h, t, row_begin, n_rows, eloc_out, stats_out, cs, lg, cuda_stream);
        else
            rc = nnqs_launch_local_energy(h, t, row_begin, rows, row_logpsi, n_rows, eloc_out, stats_out, cs,
                                          cuda_stream);
    }
    if (ctr) cudaFreeAsync(ctr, st);
    cudaEventRecord((cudaEvent_t)t->last_use, st);
    return rc;
}

int local_energy_args(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows, const double *row_logpsi,
                      int64_t n_rows, double *eloc_out, const int64_t *counts, double *partials_out) {
    if (!h || !t || n_rows < 0 || (n_rows > 0 && !eloc_out) || (!counts != !partials_out))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_local_energy: bad arguments");
    if (t->device != h->device) return nnqs_set_error(NNQS_E_ARG, "table and Hamiltonian on different devices");
    if (rows) {
        if (n_rows > 0 && !row_logpsi) return nnqs_set_error(NNQS_E_ARG, "explicit rows need row_logpsi");
    } else if (row_begin < 0 || row_begin + n_rows > t->n) {
        return nnqs_set_error(NNQS_E_TABLE, "row range outside the table");
    }
    return NNQS_OK;
}
}  // namespace

int nnqs_local_energy(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows,
                      const double *row_logpsi, int64_t n_rows, double *eloc_out, const int64_t *counts,
                      double *partials_out, int64_t *stats_out, void *cuda_stream) {
    int rc = local_energy_args(h, t, row_begin, rows, row_logpsi, n_rows, eloc_out, counts, partials_out);
    if (rc) return rc;
    DeviceGuard g(h->device);
    if (!g.ok) return nnqs_set_error(NNQS_E_CUDA, "cudaSetDevice failed");
    return local_energy_impl(h, t, row_begin, rows, row_logpsi, n_rows, eloc_out, counts, partials_out, stats_out,
                             HitLogHost{}, cuda_stream);
}

int nnqs_chunk_work(nnqs_table t, int64_t chunk, int64_t *work_out, int64_t *floor_out, void *cuda_stream) {
    if (!t || chunk <= 0 || (t->n > 0 && !work_out)) return nnqs_set_error(NNQS_E_ARG, "nnqs_chunk_work: bad arguments");
    DeviceGuard g(t->device);
    if (!g.ok) return nnqs_set_error(NNQS_E_CUDA, "cudaSetDevice failed");
    if (t->spin_ready && t->opt.algorithm != NNQS_ALGO_LITERAL) {
        const int rc = nnqs_chunk_work_spin(t, chunk, work_out, floor_out, cuda_stream);
        cudaEventRecord((cudaEvent_t)t->last_use, (cudaStream_t)cuda_stream);
        return rc;
    }
    const int64_t nch = (t->n + chunk - 1) / chunk;   // literal loop: every row costs K' pair tests
    for (int64_t c = 0; c < nch; ++c) {
        work_out[c] = std::min(chunk, t->n - c * chunk);
        if (floor_out) floor_out[c] = 0;
    }
    return NNQS_OK;
}

int nnqs_coupled_debug_rows(nnqs_ham h, nnqs_table t, int64_t row_begin, int64_t n_rows, int64_t max_pairs,
                            int64_t *row_id, int64_t *group_id, uint64_t *xprime, int64_t *table_idx,
                            double *h_xxp, int64_t *n_pairs_out) {
    if (!n_pairs_out || max_pairs < 0) return nnqs_set_error(NNQS_E_ARG, "nnqs_coupled_debug_rows: bad arguments");
    int rc = local_energy_args(h, t, row_begin, nullptr, nullptr, n_rows, (double *)1, nullptr, nullptr);
    if (rc) return rc;
    DeviceGuard g(h->device);
    if (!g.ok) return nnqs_set_error(NNQS_E_CUDA, "cudaSetDevice failed");
    cudaStream_t st = (cudaStream_t)t->own[0];
    cudaStreamWaitEvent(st, (cudaEvent_t)t->last_use, 0);
    const size_t cap = (size_t)(max_pairs > 0 ? max_pairs : 1);
    const size_t bytes = 16 * (size_t)(n_rows + 1) + cap * 24 + 64;
    char *buf = nullptr;
    cudaError_t e = cudaMalloc((void **)&buf, bytes);
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_NOMEM, cudaGetErrorString(e));
    double *eloc = (double *)buf;
    HitLogHost lg;
    lg.count = (unsigned long long *)(buf + 16 * (size_t)(n_rows + 1));
    lg.cap = (long long)cap;
    lg.row = (long long *)((char *)lg.count + 64);
    lg.idx = lg.row + cap;
    lg.h = (double *)(lg.idx + cap);
    cudaMemsetAsync(lg.count, 0, 8, st);
    rc = local_energy_impl(h, t, row_begin, nullptr, nullptr, n_rows, eloc, nullptr, nullptr, nullptr, lg, st);
    unsigned long long cnt = 0;
    if (!rc) rc = cudaMemcpyAsync(&cnt, lg.count, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess ? NNQS_OK
                  : nnqs_set_error(NNQS_E_CUDA, "read hit count");
    if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = nnqs_set_error(NNQS_E_CUDA, "sync");
    if (!rc) {
        const size_t m = std::min<size_t>((size_t)cnt, cap);
        std::vector<long long> hr(m), hi(m);
        std::vector<double> hh(m);
        if (m) {
            cudaMemcpy(hr.data(), lg.row, 8 * m, cudaMemcpyDeviceToHost);
            cudaMemcpy(hi.data(), lg.idx, 8 * m, cudaMemcpyDeviceToHost);
            cudaMemcpy(hh.data(), lg.h, 8 * m, cudaMemcpyDeviceToHost);
        }
        // keys of the rows and of x' (mode 0: the table's keys; mode 1: the index)
        std::vector<u64> keys;
        if (t->mode == 0 && t->n > 0) {
            keys.resize(2 * (size_t)t->n);
            cudaMemcpy(keys.data(), t->keys, 16 * (size_t)t->n, cudaMemcpyDeviceToHost);
        }
        const HostTable &H = h->host;
        const int64_t K = (int64_t)H.off.size() - 1;
        auto key_of = [&](long long i, u64 &lo, u64 &hi2) {
            if (t->mode == 0) { lo = keys[2 * i]; hi2 = keys[2 * i + 1]; }
            else { lo = (u64)i; hi2 = 0; }
        };
        for (size_t j = 0; j < m && j < (size_t)max_pairs; ++j) {
            u64 x0, x1, y0, y1;
            key_of(hr[j], x0, x1);
            key_of(hi[j], y0, y1);
            if (row_id) row_id[j] = hr[j];
            if (table_idx) table_idx[j] = hi[j];
            if (h_xxp) h_xxp[j] = hh[j];
            if (xprime) { xprime[2 * j] = y0; xprime[2 * j + 1] = y1; }
            if (group_id) {   // groups ascending by 128-bit X (word1, then word0)
                const u64 X0 = x0 ^ y0, X1 = x1 ^ y1;
                int64_t lo = 0, hi3 = K - 1, found = -1;
                while (lo <= hi3) {
                    const int64_t mid = (lo + hi3) / 2;
                    const u64 m0 = H.x[2 * mid], m1 = H.x[2 * mid + 1];
                    if (m1 == X1 && m0 == X0) { found = mid; break; }
                    if (m1 < X1 || (m1 == X1 && m0 < X0)) lo = mid + 1; else hi3 = mid - 1;
                }
                group_id[j] = found;
            }
        }
        *n_pairs_out = (int64_t)cnt;
        if ((int64_t)cnt > max_pairs) rc = nnqs_set_error(NNQS_E_SIZE, "max_pairs too small");
    }
    cudaStreamSynchronize(st);
    cudaFree(buf);
    return rc;
}

int nnqs_coupled_debug(nnqs_ham h, nnqs_table t, const uint64_t *rows_host, int64_t n_rows,
                       int64_t max_pairs, int64_t *row_id, int64_t *group_id, uint64_t *xprime,
                       int64_t *table_idx, double *h_xxp, int64_t *n_pairs_out) {
    if (!h || !t || !rows_host || n_rows < 0 || max_pairs < 0 || !n_pairs_out)
        return nnqs_set_error(NNQS_E_ARG, "nnqs_coupled_debug: bad arguments");
    DeviceGuard g(h->device);
    cudaStream_t st = (cudaStream_t)t->own[0];
    cudaStreamWaitEvent(st, (cudaEvent_t)t->last_use, 0);
    void *buf = nullptr;
    const size_t cap = (size_t)(max_pairs > 0 ? max_pairs : 1);
    const size_t bytes = 16 * (size_t)n_rows + cap * (24 + 16 + 8) + 16;
    cudaError_t e = cudaMalloc(&buf, bytes);
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_NOMEM, cudaGetErrorString(e));
    char *p = (char *)buf;
    uint64_t *rows_d = (uint64_t *)p; p += 16 * (size_t)n_rows;
    int64_t *oi = (int64_t *)p; p += 24 * cap;
    u64 *ox = (u64 *)p; p += 16 * cap;
    double *oh = (double *)p; p += 8 * cap;
    unsigned long long *counter = (unsigned long long *)p;
    cudaMemcpyAsync(rows_d, rows_host, 16 * (size_t)n_rows, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(counter, 0, 8, st);
    int rc = nnqs_launch_coupled_debug(h, t, rows_d, n_rows, max_pairs, oi, ox, oh, counter, st);
    unsigned long long cnt = 0;
    if (!rc) {
        cudaMemcpyAsync(&cnt, counter, 8, cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    }
    if (!rc) {
        const size_t m = cnt < cap ? (size_t)cnt : cap;
        std::vector<int64_t> hi(3 * m);
        std::vector<u64> hx(2 * m);
        std::vector<double> hh(m);
        if (m) {
            cudaMemcpy(hi.data(), oi, 24 * m, cudaMemcpyDeviceToHost);
            cudaMemcpy(hx.data(), ox, 16 * m, cudaMemcpyDeviceToHost);
            cudaMemcpy(hh.data(), oh, 8 * m, cudaMemcpyDeviceToHost);
        }
        for (size_t i = 0; i < m && i < (size_t)max_pairs; ++i) {
            if (row_id) row_id[i] = hi[3 * i];
            if (group_id) group_id[i] = hi[3 * i + 1];
            if (table_idx) table_idx[i] = hi[3 * i + 2];
            if (xprime) { xprime[2 * i] = hx[2 * i]; xprime[2 * i + 1] = hx[2 * i + 1]; }
            if (h_xxp) h_xxp[i] = hh[i];
        }
        *n_pairs_out = (int64_t)cnt;
        if ((int64_t)cnt > max_pairs) rc = nnqs_set_error(NNQS_E_SIZE, "max_pairs too small");
    }
    cudaFree(buf);
    return rc;
}

}  // extern "C"
