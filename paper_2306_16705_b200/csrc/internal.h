// Internal declarations of libnnqs (not part of the C-ABI; see include/nnqs.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/nnqs.h"

typedef unsigned long long u64;

// ----------------------------------------------------------------- errors
int nnqs_set_error(int code, const std::string &msg);

// ---------------------------------------------------------- GF(2) hash
// h(x) = XOR_{j : bit j of x set} col[j]: linear over GF(2), so
// h(x ^ X) = h(x) ^ h(X) and one XOR per (row, group) gives the bucket
// of x' = x ^ X_k.  Columns come from splitmix64 with a fixed seed.
static inline u64 nnqs_splitmix64(u64 &s) {
    u64 z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
void nnqs_hash_columns(u64 cols[128]);
// 32-bit GF(2)-linear filter hash columns of the bit-sliced literal kernel
// (per-spin string filters: f_alpha(x) = XOR over the set alpha bits of x, f_beta likewise)
void nnqs_filter_columns(uint32_t cols[128]);
u64 nnqs_hash_host(const u64 cols[128], u64 lo, u64 hi);

// ------------------------------------------------------------ Hamiltonian
struct HostTable {
    int n_qubits = 0;
    bool conserving = false;          // H conserves N_alpha and N_beta (compress)
    std::vector<u64> x;               // [K][2]
    std::vector<int64_t> off;         // [K+1]
    std::vector<u64> z;               // [Nh][2]
    std::vector<double> d;            // [Nh]
};

// host compress (compress.cpp): Eq. (9) -> grouped fused Pauli table
int nnqs_compress_host(const double *h1, const double *h2, int n, double e_core, double tol,
                       HostTable &out);
int nnqs_from_pauli_host(const u64 *xm, const u64 *zm, const double *cre, const double *cim,
                         int64_t n_terms, int n_qubits, double tol, HostTable &out);

// alpha/beta-factorised index of a spin-conserving table (structured.cu):
// every flip group is X = 0, an alpha pair, a beta pair, an alpha quad, a
// beta quad, or alpha pair x beta pair (the single / double excitations of
// Eq. (9)); group ids are reachable from the orbital indices without a search.
struct SpinIndex {
    bool ok = false;
    int n = 0;                        // spatial orbitals (<= 64)
    int64_t P = 0, Q = 0;             // n(n-1)/2, C(n,4)
    int32_t diag_k = -1;
    std::vector<int32_t> pair_k[2];   // [P]   2-site groups per spin
    std::vector<int32_t> quad_k[2];   // [Q]   4-site same-spin groups
    std::vector<int32_t> ab_k;        // [P*P] alpha pair x beta pair groups
    std::vector<int32_t> ab_rec;      // [P*P] the same, or 0x40000000 | folded string for one-string groups
    std::vector<int32_t> quad_rec[2]; // [Q] quads: 0x40000000 | (count-1) << 28 | first folded string, or k
    // In-sector folded Pauli table (same groups, CSR): for a hit x' = x ^ X with
    // x and x' in one (N_alpha, N_beta) sector, (-1)^{popc(x & F)} is a known
    // constant for F = the pair masks of X (-1 each) or a same-spin quad (+1),
    // so the strings Z and Z ^ F of a group merge into one.
    // Diagonal group X = 0 in occupation form (all its strings have |Z| <= 2):
    // sum_i d_i (-1)^{popc(x & Z_i)} = K + sum_{p occ} u_p + sum_{p<q occ} v_pq
    bool diag_ok = false;
    double diag_K = 0.0;
    std::vector<double> diag_uv;      // [N + N*N]: u_p, then v (symmetric, zero diagonal)
    // Single-excitation groups (alpha / beta pairs) in occupation form: their
    // folded strings are B ^ {0 or one Z_R}, so the group value at an in-sector
    // x is (-1)^{popc(x & B)} (T - 2 sum_{R occupied} c_R).  Record per pair
    // slot (spin * P + pair rank): {B.lo, B.hi (as bits), T, 0, c_0 .. c_{N-1}}.
    bool occ_ok = false;
    std::vector<double> occ_rec;      // [2P][4 + N]
    // Alpha pair x beta pair groups in closed form: every such group folds to one
    // string Z = canon(J), J = JW(2p, 2q) ^ JW(2r+1, 2s+1) (the qubits strictly
    // between each pair's sites), so its value at an in-sector x is
    // ab_d[U * P + V] * (-1)^{popc(x & J)} (U, V the pair ranks; the canonical
    // representative's flips are folded into ab_d).  Existence bit per slot.
    bool ab_ok = false;
    int64_t ab_w = 0;                 // 64-bit words per U row of ab_bits
    std::vector<double> ab_d;         // [P*P]
    std::vector<u64> ab_bits;         // [P * ab_w]
    std::vector<uint32_t> pair_sites; // [P] p | q << 8 (p < q) of pair rank U
    std::vector<u64> pair_J;          // [2][P][2] JW string masks: alpha pair U, beta pair V
    std::vector<uint32_t> foff;       // [K+1]
    std::vector<u64> fz;              // [M][2]
    std::vector<double> fd;           // [M]
};
int nnqs_spin_index_build(const HostTable &H, SpinIndex &S);
struct nnqs_ham_s;
int nnqs_spin_index_upload(struct nnqs_ham_s *h);
void nnqs_spin_index_release(struct nnqs_ham_s *h);

struct DeviceHam {
    // group arrays [K]
    void *gx = nullptr;       // ulonglong2 X mask
    u64 *ghx = nullptr;       // h(X)
    uint32_t *ginfo = nullptr;// bits 0..7: popc(X & alpha)/2, 8..15: popc(X & beta)/2
    uint32_t *goff = nullptr; // [K+1] term offsets
    // term arrays [Nh]
    void *tz = nullptr;       // ulonglong2 Z mask
    double *td = nullptr;     // fused coefficient d
    void *glit = nullptr;     // [K] 32-B {X, h(X), info} records of the literal kernel
    void *gbs = nullptr;      // [K] 32-B records of the bit-sliced literal kernel (k_eloc_bs), or null
    // spin index (structured path)
    int32_t *pair_k[2] = {nullptr, nullptr};
    int32_t *quad_k[2] = {nullptr, nullptr};
    int32_t *quad_rec[2] = {nullptr, nullptr};
    int32_t *ab_k = nullptr;
    int32_t *ab_rec = nullptr;
    double *ab_d = nullptr;    // alpha x beta groups in closed form (SpinIndex::ab_ok)
    u64 *ab_bits = nullptr;
    u64 *pair_J = nullptr;
    double *diag_uv = nullptr; // diagonal group in occupation form (structured path)
    double *occ_rec = nullptr; // single-excitation groups in occupation form
    void *frng = nullptr;      // folded table (structured path): uint2 range per group,
    void *frec = nullptr;      // 32-B {Z lo, Z hi, d, 0} per string
    int64_t bytes = 0;
};

struct nnqs_ham_s {
    HostTable host;
    SpinIndex spin;
    DeviceHam dev;
    int device = 0;
    int64_t n_groups = 0, n_terms = 0;
};

struct nnqs_table_s {
    int mode = 0;             // 0 sample-aware, 1 exact
    int device = 0;
    int64_t n = 0;
    void *stream = nullptr;   // the prepare stream (build only)
    nnqs_options opt{};       // per-table options (include/nnqs.h)
    void *own[3] = {nullptr, nullptr, nullptr};   // private streams: release, join, phase (ii)
    void *last_use = nullptr; // cudaEvent_t recorded after every call using the table
    void *keys = nullptr;     // ulonglong2 [n] (mode 0)
    void *logpsi = nullptr;   // double2 [n]
    void *psi_hat = nullptr;  // double2 [n]
    u64 *slots = nullptr;     // hash slots [4 * n_buckets] (mode 0)
    uint32_t *bsbm = nullptr; // alpha- and beta-string filter bitmaps of k_eloc_bs (mode 0)
    u64 bucket_mask = 0;
    u64 *shift_key = nullptr; // device: order-preserving key of s = max Re logpsi
    int *flag = nullptr;      // device: [0] order violation flag, [1] rows with psi_hat(x) < e^-600
    int64_t n_direct = 0;     // host copy of flag[1]
    int64_t bytes = 0;
    // alpha/beta string index (structured path, mode 0)
    bool spin_ready = false;
    void *spin_buf = nullptr; // one allocation holding the arrays below
    u64 *sa = nullptr, *sb = nullptr;          // [n] alpha / beta occupation strings
    int32_t *ga_of = nullptr, *gb_of = nullptr;// [n] alpha-group / beta-group of entry i
    int32_t *offA = nullptr, *offB = nullptr;  // [n+1] CSR over alpha / beta groups
    u64 *listA_b = nullptr;                    // [n] entries sorted by (a, b): beta string
    int32_t *listA_idx = nullptr;              //     ... and table index
    u64 *listB_a = nullptr;                    // [n] entries sorted by (b, a): alpha string
    int32_t *listB_idx = nullptr;
    u64 *ah_keys = nullptr;                    // alpha string -> alpha group (open addressing)
    int32_t *ah_vals = nullptr;
    u64 ah_mask = 0;
    // deletion-key multimap for heavy string groups (see structured.cu)
    void *mm = nullptr;                        // unique-key hash slots, 32 B: {u64 key, u32 meta, u32 beg | u32 end, pad}
    u64 mm_mask = 0;
    u64 *mm_bloom = nullptr;                   // blocked Bloom filter over (key, meta): 2 bits in one word
    u64 mm_bloom_mask = 0;                     // words - 1
    void *mm_ent = nullptr;                    // [m] {u64 varying string, u64 entry index}, sorted by (meta, key, entry)
    void *mm_buf = nullptr;
    int32_t thr_single = 0, thr_double = 0;    // list-length thresholds
    bool uniform_pc = false;                   // one popcount per spin over the table (set by the multimap build)
    int32_t thr_rowheavy = 0;                  // alpha groups with more rows: entry-driven phase (iii)
    int32_t *heavy_groups = nullptr;           // [n_heavy] those alpha group ids (device)
    int64_t n_alpha_groups = 0;
    int spin_n = 0;                            // spatial orbitals (the Hamiltonian's SpinIndex::n)
    void *nl_rng = nullptr;                    // int2 [n_alpha_groups]: adjacent-alpha list range (structured.cu k_nl)
    void *nl = nullptr;                        // int4 {g', u rank, offA[g'], len}
    int32_t *nl_cost = nullptr;                // [n_alpha_groups] phase (iii) work estimate of a row
    void *nl_buf = nullptr;
    int n_heavy = 0;
};

// checked: set when the spin build has read and checked the table flags (nnqs_table_check)
int nnqs_table_build_spin(nnqs_ham h, nnqs_table t, void *stream, bool *checked);
void nnqs_table_release_spin(nnqs_table t);
// fused first pass of Eq. (6) per chunk of NNQS_REDUCE_CHUNK rows (nnqs_local_energy's
// counts / partials_out): ctr = device u32[n_chunks] zeroed by the caller
struct ChunkSink {
    const int64_t *counts = nullptr;
    double *partials = nullptr;
    unsigned *ctr = nullptr;
};
// parity hit log of the production path (nnqs_coupled_debug_rows); count == nullptr: off
struct HitLogHost {
    unsigned long long *count = nullptr;
    long long cap = 0;
    long long *row = nullptr, *idx = nullptr;
    double *h = nullptr;
};
int nnqs_launch_local_energy_spin(nnqs_ham h, nnqs_table t, int64_t row_begin, int64_t n_rows,
                                  double *eloc, int64_t *stats, const ChunkSink &cs, const HitLogHost &lg,
                                  void *stream);
int nnqs_chunk_work_spin(nnqs_table t, int64_t chunk, int64_t *work_host, int64_t *floor_host, void *stream);

// device side (kernels.cu)
int nnqs_ham_upload(nnqs_ham h);
void nnqs_ham_release(nnqs_ham h);
// defer_check: leave the read of the order / exp-ratio flags (a host sync) to the caller,
// which must then call nnqs_table_check (nnqs_table_build_spin folds it into its first sync)
int nnqs_table_build(nnqs_table t, const uint64_t *keys, const double *logpsi, void *stream, bool defer_check);
int nnqs_table_check(nnqs_table t, const int *host_flags, void *stream);
void nnqs_table_release(nnqs_table t);
int nnqs_launch_local_energy(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows,
                             const double *row_logpsi, int64_t n_rows, double *eloc,
                             int64_t *stats, const ChunkSink &cs, void *stream);
// stream-ordered allocation from the library's own memory pool (one per device,
// created once, thread-safe; the device's default pool is left untouched)
cudaError_t nnqs_malloc_async(void **p, size_t bytes, cudaStream_t st);
template <class T> inline cudaError_t nnqs_malloc_async(T **p, size_t bytes, cudaStream_t st) {
    return nnqs_malloc_async(reinterpret_cast<void **>(p), bytes, st);
}
int nnqs_launch_coupled_debug(nnqs_ham h, nnqs_table t, const uint64_t *rows_dev, int64_t n_rows,
                              int64_t max_pairs, int64_t *out_i64 /*[max][3]*/, u64 *out_x /*[max][2]*/,
                              double *out_h, unsigned long long *counter, void *stream);
