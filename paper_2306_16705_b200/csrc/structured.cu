// structured.cu -- the alpha/beta-factorised ("string-driven") local-energy
// path: same sum as Algorithm 2, same set of
// (row, group) pairs with x' = x ^ X_k in the sample table,
// enumerated from the table side instead of the group side.
//
// A row x = (a, b) (alpha / beta occupation strings) couples through a group
// of the compressed table (Fig. 6(c)) only to
//   (i)   x' = (a'', b): a'' in A(b) = {alpha strings paired with b in T},
//         X = alpha pair (2-site group) or alpha quad (4-site same-spin);
//   (ii)  x' = (a, b''): b'' in B(a), X = beta pair or beta quad;
//   (iii) x' = (a ^ u, b ^ v): u an alpha single (one occupied, one empty),
//         v a beta single, X = u x v (4-site opposite-spin);
// plus the diagonal group (X = 0, x' = x).  Scanning the table-side lists
// A(b), B(a) and B(a ^ u) visits every x' of the table that some group can
// reach, so the hit set equals the literal loop's (tests: P3 parity), while
// the work per row drops from K' (2.06e6 groups at 120 qubits) to the list
// lengths.  H_xx' itself is still the group's Pauli sum
// sum_i d_i (-1)^{popc(x & Z_i)} (reading R1).
//
// Accumulation order of a row depends on the row and the table only (fixed
// lane assignment, fixed butterfly reduction): bit-identical for any row
// slicing / number of GPUs.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <mutex>
#include <limits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

__constant__ u64 c_hs[128];   // same GF(2) hash columns as kernels.cu (per translation unit)

namespace {

std::mutex g_hs_ready_mu;
bool g_hs_ready[64] = {false};

// the hash columns in constant memory of `device` (the current device), once per device
int ensure_hs(int device) {
    if (device < 0 || device >= 64) return NNQS_E_ARG;
    std::lock_guard<std::mutex> lk(g_hs_ready_mu);
    if (g_hs_ready[device]) return NNQS_OK;
    u64 cols[128];
    nnqs_hash_columns(cols);
    cudaError_t e = cudaMemcpyToSymbol(c_hs, cols, sizeof(cols));
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    g_hs_ready[device] = true;
    return NNQS_OK;
}

int ensure_binom(int device);

inline int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return NNQS_OK;
    return nnqs_set_error(e == cudaErrorMemoryAllocation ? NNQS_E_NOMEM : NNQS_E_CUDA,
                          std::string(what) + ": " + cudaGetErrorString(e));
}

inline int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return (int)g;
}

__host__ __device__ __forceinline__ int pair_rank(int p, int q, int n) {   // p < q < n <= 64
    return ((p * (2 * n - p - 1)) >> 1) + (q - p - 1);
}

__host__ __device__ __forceinline__ int quad_rank(int p1, int p2, int p3, int p4) {  // colex, p1<p2<p3<p4<64
    return p1 + ((p2 * (p2 - 1)) >> 1) + (p3 * (p3 - 1) * (p3 - 2)) / 6 + (p4 * (p4 - 1) * (p4 - 2) * (p4 - 3)) / 24;
}

__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}


// ------------------------------------------------------------- device views
struct SpinView {
    int n;
    int64_t P;
    const int32_t *pair_k0, *pair_k1, *quad_k0, *quad_k1, *ab_k;
    const int32_t *ab_rec;    // alpha pair x beta pair -> REC_TAG | folded string (single-string groups) or k
    const int32_t *quad_rec0, *quad_rec1;   // same-spin quads -> REC_TAG | count | first string, or k
    int32_t diag_k;
    int nq;                   // qubits
    const double *occ_rec;    // single-excitation records (SpinIndex::occ_rec) or nullptr
    double diag_K;            // diagonal group in occupation form (SpinIndex), or
    const double *diag_uv;    // nullptr: evaluate its Pauli strings
    const double *ab_d;       // alpha x beta groups in closed form (SpinIndex::ab_ok), or nullptr
    const u64 *ab_bits;       //   existence bit per (U, V) slot, rows of ab_w words
    int64_t ab_w;
    const ulonglong2 *pair_J;     // [2][P] JW string masks of alpha / beta pairs
};

// x' = x ^ X with X = alpha pair U (qubits 2p, 2q) x beta pair V (2r+1, 2s+1):
// H_{x'x} = ab_d[U P + V] (-1)^{popc(x & J)}, J = the qubits strictly between
// each pair's sites (the JW strings; SpinIndex::ab_d).
__device__ __forceinline__ double ab_value(const double *ab_d, const ulonglong2 *pair_J, int64_t P, uint32_t U,
                                           uint32_t V, u64 x0, u64 x1) {
    const ulonglong2 ja = __ldg(pair_J + U), jb = __ldg(pair_J + P + V);   // JW strings of the two pairs
    const u64 m0 = ja.x ^ jb.x, m1 = ja.y ^ jb.y;
    const double d = __ldg(ab_d + (int64_t)U * P + V);
    return __longlong_as_double(__double_as_longlong(d) ^
                                ((long long)((__popcll(x0 & m0) + __popcll(x1 & m1)) & 1) << 63));
}
// existence of the alpha x beta group (U, V): its queue key AB_TAG | U << 11 | V, or -1
#define AB_TAG 0x20000000
__device__ __forceinline__ int32_t ab_key(const SpinView &S, int32_t U, int32_t V) {
    if (S.ab_d) {
        const u64 w = __ldg(S.ab_bits + (int64_t)U * S.ab_w + (V >> 6));
        return ((w >> (V & 63)) & 1) ? (int32_t)(AB_TAG | (U << 11) | V) : -1;
    }
    return __ldg(S.ab_rec + (int64_t)U * S.P + V);
}

// folded table on the device: per group its string range, per string one 32-B
// record {Z lo, Z hi}, {d bits, 0} (one sector per string instead of two)
struct GroupView {
    const uint2 *grng;
    const ulonglong2 *rec;
};
__device__ __forceinline__ uint2 g_range(const GroupView &G, int32_t k) { return __ldg(G.grng + k); }
__device__ __forceinline__ ulonglong2 g_z(const GroupView &G, uint32_t i) { return __ldg(G.rec + 2 * i); }
__device__ __forceinline__ double g_d(const GroupView &G, uint32_t i) {
    return __longlong_as_double((long long)__ldg(G.rec + 2 * i + 1).x);
}

// Parity/debug hit log (nnqs_coupled_debug_rows): every hit the production
// kernels evaluate is appended as (row, x' table index, H_xx').  count == nullptr
// (the normal call) disables it: one warp-uniform branch per evaluated batch.
struct HitLog {
    unsigned long long *count;
    long long cap;
    long long *row, *idx;
    double *h;
};
__device__ __forceinline__ void log_hit(const HitLog &L, int row, long long idx, double hv) {
    const unsigned long long s = atomicAdd(L.count, 1ULL);
    if ((long long)s < L.cap) {
        L.row[s] = row;
        L.idx[s] = idx;
        L.h[s] = hv;
    }
}

struct TabSpin {
    int64_t n;
    const ulonglong2 *keys;
    const double2 *logpsi;
    const double2 *psi_hat;
    const u64 *slots;
    u64 bucket_mask;
    const u64 *shift_key;
    const u64 *sa, *sb;
    const int32_t *ga_of, *gb_of, *offA, *offB;
    const u64 *listA_b, *listB_a;
    const int32_t *listA_idx, *listB_idx;
    const u64 *ah_keys;
    const int32_t *ah_vals;
    u64 ah_mask;
    const ulonglong2 *mm;     // deletion multimap: unique (key, meta) -> run id (y = meta | run << 32)
    u64 mm_mask;
    const u64 *mm_bloom;      // ~8 bits per run: most probes miss (C5: ~80%) and stop here, in L2
    u64 mm_bloom_mask;
    const ulonglong2 *mm_ent;  // {varying string, entry index} per multimap entry
    const int2 *nl_rng;        // [alpha groups] -> [begin, end) in nl
    const int4 *nl;            // {g', u rank, offA[g'], |list(g')|} of the present a' = a ^ u
    int32_t thr_single, thr_double;
    int uniform_pc;           // every alpha (beta) string of the table has one popcount: XOR
                              // distance 2 / 4 already implies a balanced excitation
    HitLog log;               // parity hit log (count == nullptr: off)
};

// ---------------------------------------------------------------- multimap
// Deletion keys: two occupation strings of one spin differ by a single
// excitation iff they share a 1-deletion (the string minus one occupied
// orbital), by a double iff they share a 2-deletion.  For heavy groups the
// table entries are indexed by (tag, group id, deletion) so that a row finds
// its coupled x' with 15 (singles) or 105 (doubles) probes instead of a scan.
//   tag 0: (alpha group, beta string minus 1 orbital)   tag 1: minus 2
//   tag 2: (beta group, alpha string minus 1 orbital)   tag 3: minus 2
#define MM_EMPTY 0xFFFFFFFFu
__host__ __device__ __forceinline__ uint32_t mm_meta(int tag, int32_t g) { return ((uint32_t)tag << 30) | (uint32_t)g; }
__host__ __device__ __forceinline__ u64 mm_hash(u64 key, uint32_t meta) {
    return mix64(key ^ ((u64)meta * 0x9E3779B97F4A7C15ULL));
}

__device__ __forceinline__ double dkey_inv2(u64 k) {
    if (k == 0) return 0.0;
    u64 b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double((long long)b);
}

__device__ __forceinline__ double flip_sign2(double d, int parity) {
    return __longlong_as_double(__double_as_longlong(d) ^ ((long long)parity << 63));
}

// H_{x', x} = sum_{i in group k} d_i (-1)^{popc(x & Z_i)}  (one lane)
__device__ __forceinline__ double group_value1(const GroupView &G, int32_t k, u64 x0, u64 x1,
                                               unsigned long long &n_str) {
    const uint2 be = g_range(G, k);
    const uint32_t b = be.x, e = be.y;
    double hv = 0.0;
#pragma unroll 4
    for (uint32_t i = b; i < e; ++i) {
        const ulonglong2 Z = g_z(G, i);
        hv += flip_sign2(g_d(G, i), (__popcll(x0 & Z.x) + __popcll(x1 & Z.y)) & 1);
    }
    n_str += e - b;
    return hv;
}

// Warp-cooperative Pauli sum of strings [b, e): lane l takes b+l, b+l+32, ...
// in ascending order (4 loads in flight), then a fixed butterfly.  Every lane
// returns the group value.
__device__ __forceinline__ double warp_strided_sum(const GroupView &G, uint32_t b, uint32_t e, u64 x0, u64 x1) {
    const int lane = threadIdx.x & 31;
    double hv = 0.0;
    for (uint32_t t0 = b + lane; t0 < e; t0 += 128) {
        ulonglong2 Z[4];
        double d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool ok = t0 + 32 * u < e;
            Z[u] = ok ? g_z(G, t0 + 32 * u) : make_ulonglong2(0, 0);
            d[u] = ok ? g_d(G, t0 + 32 * u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t0 + 32 * u < e) hv += flip_sign2(d[u], (__popcll(x0 & Z[u].x) + __popcll(x1 & Z[u].y)) & 1);
    }
    for (int o = 16; o; o >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, o);
    return hv;
}

__device__ __forceinline__ int32_t alpha_lookup(const TabSpin &T, u64 a) {
    u64 s = mix64(a) & T.ah_mask;
    while (true) {
        const int32_t v = __ldg(T.ah_vals + s);
        if (v < 0) return -1;
        if (__ldg(T.ah_keys + s) == a) return v;
        s = (s + 1) & T.ah_mask;
    }
}

// index of the o-th set bit (0-based) of a 64-bit word
__device__ __forceinline__ int nth_set(u64 w, int o) {
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    const int c = __popc(lo);
    if (o < c) return (int)__fns(lo, 0, o + 1);
    return 32 + (int)__fns(hi, 0, o - c + 1);
}

// group id of the same-spin excitation d (2 or 4 bits, within one spin string)
// lut: shared C(p,2), C(p,3), C(p,4) for p < 64 (colex rank of a quad without
// divisions); the extreme bits by ffs / clz, the middle two from what remains
__device__ __forceinline__ int32_t same_spin_group(const SpinView &S, int spin, u64 d, int c, const uint32_t *lut) {
    const int p1 = __ffsll((long long)d) - 1;
    const int p4 = 63 - __clzll((long long)d);
    if (c == 2) return __ldg((spin ? S.pair_k1 : S.pair_k0) + pair_rank(p1, p4, S.n));
    const u64 m = d & (d - 1) & ~(1ULL << p4);
    const int p2 = __ffsll((long long)m) - 1;
    const int p3 = 63 - __clzll((long long)m);
    return __ldg((spin ? S.quad_rec1 : S.quad_rec0) + (p1 + (int)(lut[p2] + lut[64 + p3] + lut[128 + p4])));
}

// Queue tag of a same-spin excitation: singles with an occupation-form record
// are queued as 0x80000000 | (spin * P + pair rank), everything else as k.
#define OCC_TAG 0x80000000u
#define REC_TAG 0x40000000   // queue key = REC_TAG | (count - 1) << 28 | first folded string (1-4 strings)
__device__ __forceinline__ int32_t same_spin_tag(const SpinView &S, int spin, u64 d, int c, const uint32_t *lut) {
    if (c == 2 && S.occ_rec) {
        const int p1 = __ffsll((long long)d) - 1;
        const int p2 = 63 - __clzll((long long)d);
        const int32_t rk = pair_rank(p1, p2, S.n);
        if (__ldg((spin ? S.pair_k1 : S.pair_k0) + rk) < 0) return -1;
        return (int32_t)(OCC_TAG | (uint32_t)(spin * S.P + rk));
    }
    return same_spin_group(S, spin, d, c, lut);
}

// multimap lookup: [beg, end) into mm_ent of the entries stored under (key, meta).
// A slot is 32 B (one sector): {key, meta | beg << 32}, {end, -}.
__device__ __forceinline__ bool mm_bloom_pass(const TabSpin &T, u64 h) {
    const u64 bw = __ldg(T.mm_bloom + ((h >> 32) & T.mm_bloom_mask));
    return (bw >> ((h >> 20) & 63)) & (bw >> ((h >> 26) & 63)) & 1;
}

// slot probe of a key that passed the Bloom filter
__device__ __forceinline__ void mm_find_slots(const TabSpin &T, u64 h, u64 key, uint32_t meta, int32_t &beg,
                                              int32_t &end) {
    beg = end = 0;
    u64 pos = h & T.mm_mask;
    while (true) {
        const ulonglong2 v = __ldg(T.mm + 2 * pos);
        const ulonglong2 w = __ldg(T.mm + 2 * pos + 1);
        const uint32_t sm = (uint32_t)v.y;
        if (sm == MM_EMPTY) return;
        if (v.x == key && sm == meta) {
            beg = (int32_t)(v.y >> 32);
            end = (int32_t)w.x;
            return;
        }
        pos = (pos + 1) & T.mm_mask;
    }
}

__device__ __forceinline__ void mm_find(const TabSpin &T, u64 key, uint32_t meta, int32_t &beg, int32_t &end) {
    const u64 h = mm_hash(key, meta);
    beg = end = 0;
    const u64 bw = __ldg(T.mm_bloom + ((h >> 32) & T.mm_bloom_mask));
    if (!((bw >> ((h >> 20) & 63)) & (bw >> ((h >> 26) & 63)) & 1)) return;
    u64 pos = h & T.mm_mask;
    while (true) {
        const ulonglong2 v = __ldg(T.mm + 2 * pos);
        const ulonglong2 w = __ldg(T.mm + 2 * pos + 1);
        const uint32_t sm = (uint32_t)v.y;
        if (sm == MM_EMPTY) return;
        if (v.x == key && sm == meta) {
            beg = (int32_t)(v.y >> 32);
            end = (int32_t)w.x;
            return;
        }
        pos = (pos + 1) & T.mm_mask;
    }
}

// (i, j) = the c-th index pair i < j in colex order (c = j(j-1)/2 + i)
__device__ __forceinline__ void nth_pair(int c, int &i, int &j) {
    j = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)c)) * 0.5f);
    while (j * (j - 1) / 2 > c) --j;
    while ((j + 1) * j / 2 <= c) ++j;
    i = c - j * (j - 1) / 2;
}

// Evaluate the first cnt queued hits (lane l takes slot l), add their
// contributions H * psi(x') to the lane accumulators, and shift the queue.
// Out of line: it is reached from every candidate site, and inlining it there
// overflowed the instruction cache.  Everything is passed and returned by value
// (views by value, accumulators in/out): a reference argument of a call that
// is not inlined forces the referenced object -- e.g. a kernel-parameter
// struct -- into local memory.
#define QCAP 256   // per-warp hit ring (power of two >= 32 + 4 * 32)

// The row being evaluated by a warp, and its per-lane accumulators, live in
// shared memory: they are touched only here and at the row's start and end,
// which keeps the scanning loops' register footprint (and spills) down.
struct RowState {
    u64 x0, x1;
    double2 lx;
    int direct;
    int row;        // table index of the row (hit log)
};

// Inlined at every push site: the ratio psi(x')/psi(x) of the rare rows with
// psi_hat(x) < e^-600 (exp / sincos, large code) is a separate instantiation
// (DIRECT), so this stays small and no ABI call forces the kernel's live
// registers to local memory.
template <bool DIRECT, bool OCC, bool AB, bool LOG>
__device__ __forceinline__ uint2 flush_queue(const GroupView &G, const double2 *psi_hat, const double2 *logpsi,
                                             const int2 *q, int qh, int cnt, const RowState *rs, double2 *acc,
                                             const double *occ_rec, int nq, const HitLog &lg, const double *ab_d,
                                             const ulonglong2 *pair_J, int64_t P, const int32_t *listA_idx) {
    const int lane = threadIdx.x & 31;
    uint32_t c_hit = 0, c_str = 0;
    __syncwarp();
    const u64 x0 = rs->x0, x1 = rs->x1;
    constexpr bool direct = DIRECT;
    int2 e = make_int2(-1, 0);
    uint32_t gb0 = 0, ge0 = 0;
    double2 ps0 = make_double2(0.0, 0.0);
    bool occ = false, ab = false;
    if (lane < cnt) {
        e = q[(qh + lane) & (QCAP - 1)];          // ring buffer: no shifting after a flush
        occ = OCC && e.x < 0;                      // single excitation, occupation-form record
        ab = AB && !occ && !(e.x & REC_TAG) && (e.x & AB_TAG);   // alpha x beta, closed form
        if (!occ && !ab) {
            if (e.x & REC_TAG) {                   // 1-4 folded strings, start and count carried in the tag
                gb0 = (uint32_t)(e.x & 0x0FFFFFFF);
                ge0 = gb0 + 1 + ((e.x >> 28) & 3);
            } else {
                const uint2 be = g_range(G, e.x);
                gb0 = be.x;
                ge0 = be.y;
            }
        }
        if (AB && ab && e.x < 0) e.y = __ldg(listA_idx + e.y);   // lazy alpha x beta entry: list position
        if (!direct) ps0 = __ldg(psi_hat + e.y);   // issued with the offsets, used after the sum
        ++c_hit;
    }
    auto add = [&](double hv, int64_t idx) {
        if (LOG && lg.count) log_hit(lg, rs->row, idx, hv);
        double2 ps = ps0;
        if (direct) {
            const double2 lx = rs->lx;
            const double2 l = logpsi[idx];
            const double m = exp(l.x - lx.x);
            double sn, cs;
            sincos(l.y - lx.y, &sn, &cs);
            ps = make_double2(m * cs, m * sn);
        }
        double2 a = acc[lane];
        a.x = fma(hv, ps.x, a.x);
        a.y = fma(hv, ps.y, a.y);
        acc[lane] = a;
    };
    if (OCC && occ) {
        // (-1)^{popc(x & B)} (T - 2 sum_{R occupied} c_R): the folded strings B ^ Z_R summed
        // in occupation form (SpinIndex::occ_rec)
        const double *rr = occ_rec + (size_t)(e.x & 0x7FFFFFFF) * (4 + nq);
        const u64 B0 = (u64)__double_as_longlong(__ldg(rr)), B1 = (u64)__double_as_longlong(__ldg(rr + 1));
        const double Tg = __ldg(rr + 2);
        double sum = 0.0;
        for (int hw = 0; hw < 4; ++hw) {           // 32-bit halves: one FLO per occupied qubit
            uint32_t w = (uint32_t)((hw < 2 ? x0 : x1) >> (32 * (hw & 1)));
            const double *rb = rr + 4 + 32 * hw;
            while (w) {                            // 4 loads in flight, added in ascending R as before
                double v[4];
                bool has[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    has[u] = w != 0;
                    v[u] = has[u] ? __ldg(rb + (__ffs(w) - 1)) : 0.0;
                    w &= w - 1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (has[u]) sum += v[u];
            }
        }
        const double hv = flip_sign2(fma(-2.0, sum, Tg), (__popcll(x0 & B0) + __popcll(x1 & B1)) & 1);
        if (hv == hv) {                            // NaN: the pair has no group (SpinIndex::occ_rec)
            c_str += __popcll(x0) + __popcll(x1) + 1;
            add(hv, e.y);
        } else {
            --c_hit;
        }
    }
    const bool big = lane < cnt && !occ && ge0 - gb0 > 32;
    if (AB && ab) {
        const double hv = ab_value(ab_d, pair_J, P, ((uint32_t)e.x >> 11) & 0x7FF, (uint32_t)e.x & 0x7FF, x0, x1);
        if (hv == hv) {                            // NaN: no alpha x beta group (lazy entries only)
            add(hv, e.y);
            ++c_str;
        } else {
            --c_hit;
        }
    }
    if (lane < cnt && !occ && !big && !ab) {
        // 4 strings in flight per lane (loads issued before the sums; same order)
        double hv = 0.0;
        for (uint32_t i0 = gb0; i0 < ge0; i0 += 4) {
            ulonglong2 Z[4];
            double d[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ok = i0 + u < ge0;
                Z[u] = ok ? g_z(G, i0 + u) : make_ulonglong2(0, 0);
                d[u] = ok ? g_d(G, i0 + u) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < ge0) hv += flip_sign2(d[u], (__popcll(x0 & Z[u].x) + __popcll(x1 & Z[u].y)) & 1);
        }
        c_str += ge0 - gb0;
        add(hv, e.y);
    }
    unsigned bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {                               // long groups: whole warp, fixed reduction
        const int src = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        const uint32_t b1 = __shfl_sync(0xffffffffu, gb0, src), e1 = __shfl_sync(0xffffffffu, ge0, src);
        double hv = warp_strided_sum(G, b1, e1, x0, x1);
        if (lane == src) {
            add(hv, e.y);
            c_str += e1 - b1;
        }
    }
    __syncwarp();
    return make_uint2(c_hit, c_str);
}

// section cycle counters (build with -DNNQS_PROFILE; nnqs_debug_counters)
#ifdef NNQS_PROFILE
__device__ unsigned long long g_prof[16];
#define PROF_DECL unsigned long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define PROF_T(v) const long long v = clock64();
#define PROF_ADD(slot, v) prof[slot] += (unsigned long long)(clock64() - (v));
#define PROF_FLUSH                                                            \
    if ((threadIdx.x & 31) == 0)                                              \
        for (int ps_ = 0; ps_ < 12; ++ps_) atomicAdd(g_prof + ps_, prof[ps_]);
#else
#define PROF_DECL
#define PROF_T(v)
#define PROF_ADD(slot, v)
#define PROF_FLUSH
#endif

#define SCAN_LIMIT 8192
// multimap sizing (measured): slots >= 4 x runs, 8 Bloom bits per run
#define MM_LOAD 4.0
#define MM_BLOOM_BITS 8
// phases compiled into the launch sequence (profiling builds may mask some: -DNNQS_PHASE_MASK=...)
#ifndef NNQS_PHASE_MASK
#define NNQS_PHASE_MASK 15
#endif
#define WARPS_PER_BLOCK 8
#ifndef NNQS_P3_MINB
#define NNQS_P3_MINB 4   // CTAs per SM of the phase-(iii) kernel (launch bounds)
#endif
#ifndef NNQS_AB
#define NNQS_AB 1      // alpha x beta groups in closed form (SpinIndex::ab_ok)
#endif
#ifndef NNQS_LAZY_AB
#define NNQS_LAZY_AB 1 // light phase (iii) candidates: existence + index resolved in the flush
#endif
#ifndef NNQS_SPIN_MINB
#define NNQS_SPIN_MINB 4
#endif
#define HCAP 96

// one warp per row; rows are table entries [row_begin, row_begin + n_rows).
// Candidate x' are found by warp-uniform, 4-way unrolled scans of the table's
// string lists; hits (group k, table index) go to a per-warp queue and are
// evaluated 32 at a time, one per lane (slot s -> lane s mod 32, so the
// summation order of a row is fixed by the row and the table).
// PH selects the phases compiled into this instantiation: 1 diagonal, 2/4 same-
// spin lists, 8 alpha x beta.  PH = 7 writes the row's partial sum to
// `partial`; PH = 8 starts from it and finalises E_loc (two smaller kernels:
// fewer registers, more resident warps, less instruction-cache pressure).
// partial2 != NULL: phase (ii) (PH = 20) runs concurrently with PH = 3 on its own
// stream, starts from zero and writes partial2; PH = 24 starts from
// partial + partial2 (a row's order is still fixed by the row and the table).
template <int PH, int MINB, bool DIRECT, bool LOG>
__global__ void __launch_bounds__(256, MINB) k_eloc_spin(SpinView S, GroupView G, TabSpin T, int64_t row_begin,
                                                   int64_t n_rows, double2 *out,
                                                   unsigned long long *stats, unsigned long long pairs,
                                                   int phase_mask, const double2 *acc_heavy, int32_t thr_rowheavy,
                                                   double2 *partial, unsigned long long *row_ctr,
                                                   const int32_t *perm, double2 *partial2, ChunkSink cs) {
    __shared__ int2 s_q[WARPS_PER_BLOCK][QCAP];
    __shared__ uint8_t s_orb[WARPS_PER_BLOCK][4][64];   // occ(a), vir(a), occ(b), vir(b) of the row
    __shared__ int2 s_h[(PH & 8) ? WARPS_PER_BLOCK : 1][HCAP];   // heavy adjacent alpha groups (g, u rank)
    __shared__ int32_t s_pl[(PH & 8) ? WARPS_PER_BLOCK : 1][64];    // Bloom-passing probe tasks
    __shared__ RowState s_row[WARPS_PER_BLOCK];
    __shared__ uint32_t s_lut[(PH & 6) ? 192 : 1];   // C(p,2), C(p,3), C(p,4), p < 64
    if (PH & 6) {
        for (int i = threadIdx.x; i < 192; i += blockDim.x) {
            const uint32_t p = i & 63, k = 2 + (i >> 6);
            uint32_t v = 1;
            for (uint32_t j = 1; j <= k; ++j) v = v * (p >= k ? p - k + j : 0) / j;
            s_lut[i] = p >= k ? v : 0;
        }
        __syncthreads();
    }
    __shared__ uint8_t s_oq[(PH & 1) ? WARPS_PER_BLOCK : 1][128];   // occupied qubits (diagonal)
    __shared__ double2 s_acc[WARPS_PER_BLOCK][32];
    if ((PH & 8) && !DIRECT && stats && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats, pairs);
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    int2 *q = s_q[threadIdx.x >> 5];
    uint8_t *occA = s_orb[threadIdx.x >> 5][0], *virA = s_orb[threadIdx.x >> 5][1];
    uint8_t *occB = s_orb[threadIdx.x >> 5][2], *virB = s_orb[threadIdx.x >> 5][3];
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double s = dkey_inv2(*T.shift_key);
    const u64 nmask = S.n >= 64 ? ~0ULL : ((1ULL << S.n) - 1);
    RowState *rs = &s_row[threadIdx.x >> 5];
    double2 *acc = s_acc[threadIdx.x >> 5];
    uint32_t c_cand = 0, c_hit = 0, c_str = 0;
    // rows: grid-stride, or (row_ctr != nullptr) handed out one at a time from a
    // global counter, so a few expensive rows do not leave other warps idle
    auto next_row = [&](int64_t cur) -> int64_t {
        if (!row_ctr) return cur + nwarps;
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(row_ctr, 1ULL);
        const int64_t w = (int64_t)__shfl_sync(0xffffffffu, v, 0);
        return (perm && w < n_rows) ? (int64_t)__ldg(perm + w) : w;   // costliest rows first
    };
    PROF_DECL
    for (int64_t r = row_ctr ? next_row(0) : warp; r < n_rows; r = next_row(r)) {
        PROF_T(t_row)
#ifdef NNQS_PROFILE
        bool prof_in_ss = false;
#endif
        const int64_t i = row_begin + r;
        const double2 lx0 = T.logpsi[i];
        if (!(lx0.x > -INFINITY)) {
            if (lane == 0 && (PH & 8) && !DIRECT) out[r] = make_double2(NAN, NAN);
            if ((PH & 8) && !DIRECT) chunk_done_warp(cs, out, r, n_rows);
            continue;
        }
        if (((lx0.x - s) < -600.0) != DIRECT) continue;   // the other instantiation's row
        const u64 a = T.sa[i], b = T.sb[i];
        __syncwarp();
        if (lane == 0) {
            const ulonglong2 xk = T.keys[i];
            rs->x0 = xk.x;
            rs->x1 = xk.y;
            rs->lx = lx0;
            rs->direct = DIRECT;
            rs->row = (int)i;
        }
        double2 a0 = make_double2(0.0, 0.0);         // 16: continue a row
        if ((PH & 16) && lane == 0) {
            if (!(PH & 8) && partial2) {
                // phase (ii) concurrent with (i): starts from zero
            } else if ((PH & 8) && partial2) {
                const double2 p1 = partial[r], p2 = partial2[r];
                a0 = make_double2(p1.x + p2.x, p1.y + p2.y);
            } else {
                a0 = partial[r];
            }
        }
        acc[lane] = a0;
        for (int j = lane; j < S.n; j += 32) {       // orbital lists (replace nth-set-bit searches)
            const u64 below = (1ULL << j) - 1;
            if ((a >> j) & 1) occA[__popcll(a & below)] = (uint8_t)j;
            else virA[j - __popcll(a & below)] = (uint8_t)j;
            if ((b >> j) & 1) occB[__popcll(b & below)] = (uint8_t)j;
            else virB[j - __popcll(b & below)] = (uint8_t)j;
        }
        __syncwarp();
        int qn = 0, qh = 0;                          // warp-uniform ring length and head
        auto flush = [&](int cnt) {                  // lanes < cnt evaluate q[qh + lane]
            if (phase_mask & 64) {                   // profiling builds only: hits found, not evaluated
                qh = (qh + cnt) & (QCAP - 1);
                qn -= cnt;
                return;
            }
            PROF_T(t_fl)
            const uint2 fo = flush_queue<DIRECT, (PH & 6) != 0, (PH & 8) != 0, LOG>(G, T.psi_hat, T.logpsi, q, qh, cnt, rs, acc,
                                                                                S.occ_rec, S.nq, T.log, S.ab_d,
                                                                                S.pair_J, S.P, T.listA_idx);
            c_hit += fo.x;
            c_str += fo.y;
            qh = (qh + cnt) & (QCAP - 1);
            qn -= cnt;
            PROF_ADD(5, t_fl)
#ifdef NNQS_PROFILE
            if (prof_in_ss) prof[9] += (unsigned long long)(clock64() - t_fl);
#endif
        };
        auto push = [&](int32_t k, int32_t idx) {    // all lanes; k == -1 = no hit (OCC_TAG keys are negative)
            const unsigned m = __ballot_sync(0xffffffffu, k != -1);
            if (k != -1) q[(qh + qn + __popc(m & lt_mask)) & (QCAP - 1)] = make_int2(k, idx);
            qn += __popc(m);
            if (qn >= 32) flush(32);
        };
        // four candidates per lane at once (same queue order as four push calls:
        // u-major, then lane), one flush check
        auto push4 = [&](const int32_t *kk, const int32_t *ix) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned m = __ballot_sync(0xffffffffu, kk[u] != -1);
                if (kk[u] != -1) q[(qh + qn + __popc(m & lt_mask)) & (QCAP - 1)] = make_int2(kk[u], ix[u]);
                qn += __popc(m);
            }
            while (qn >= 32) flush(32);
        };
        // Every lane holds a multimap match range [mb, me) and a tag; all matches of
        // the warp are evaluated 32 at a time in (lane, position) order -- parallel
        // dependent loads instead of one matching lane at a time.
        auto drain = [&](int32_t mb, int32_t me, int32_t tag, auto &&eval) {
            const int32_t len = me - mb;
            int32_t incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int32_t excl = incl - len;
            const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
            for (int32_t f0 = 0; f0 < total; f0 += 32) {
                const int32_t f = f0 + lane;
                int lo = 0;
#pragma unroll
                for (int st = 16; st; st >>= 1) {
                    const int c = lo + st;
                    const int32_t ex = __shfl_sync(0xffffffffu, excl, c & 31);
                    if (c < 32 && ex <= f) lo = c;
                }
                const int32_t smb = __shfl_sync(0xffffffffu, mb, lo);
                const int32_t sex = __shfl_sync(0xffffffffu, excl, lo);
                const int32_t stag = __shfl_sync(0xffffffffu, tag, lo);
                int32_t k = -1, idx = 0;
                if (f < total) eval(smb + (f - sex), stag, k, idx);
                push(k, idx);
            }
        };
        PROF_ADD(6, t_row)
        PROF_T(t_diag)
        // ---- diagonal group: warp-cooperative Pauli sum, fixed reduction
        if ((PH & 1) && S.diag_k >= 0 && (phase_mask & 1)) {
            uint32_t gb = 0, ge = 0;
            double hv;
            if (S.diag_uv) {
                // occupation form: K + sum_{p occ} u_p + sum_{p<q occ} v_pq over the
                // row's occupied qubits (lane l: qubit l, l+32, .. and its partners above)
                const int nocc = __popcll(rs->x0) + __popcll(rs->x1);
                uint8_t *oq = s_oq[(PH & 1) ? (threadIdx.x >> 5) : 0];
                __syncwarp();
                for (int j = lane; j < S.nq; j += 32) {
                    const u64 w = j < 64 ? rs->x0 : rs->x1;
                    const int jb = j & 63;
                    if ((w >> jb) & 1)
                        oq[(j < 64 ? 0 : __popcll(rs->x0)) + __popcll(w & ((1ULL << jb) - 1))] = (uint8_t)j;
                }
                __syncwarp();
                hv = 0.0;
                for (int l = lane; l < nocc; l += 32) {
                    const int p = oq[l];
                    const double *vp = S.diag_uv + S.nq + (size_t)p * S.nq;
                    double t = __ldg(S.diag_uv + p);
                    int m = l + 1;
                    for (; m + 3 < nocc; m += 4) {       // 4 loads in flight, same order of additions
                        const double v0 = __ldg(vp + oq[m]), v1 = __ldg(vp + oq[m + 1]);
                        const double v2 = __ldg(vp + oq[m + 2]), v3 = __ldg(vp + oq[m + 3]);
                        t += v0;
                        t += v1;
                        t += v2;
                        t += v3;
                    }
                    for (; m < nocc; ++m) t += __ldg(vp + oq[m]);
                    hv += t;
                }
                for (int o = 16; o; o >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, o);
                hv += S.diag_K;
                gb = 0;
                ge = (uint32_t)(nocc + nocc * (nocc - 1) / 2);
                __syncwarp();
            } else {
                const uint2 be = g_range(G, S.diag_k);
                gb = be.x;
                ge = be.y;
                hv = warp_strided_sum(G, gb, ge, rs->x0, rs->x1);
            }
            if (lane == 0) {   // x' = x: psi_hat(x) (or 1 on the direct path)
                if (LOG && T.log.count) log_hit(T.log, (int)i, i, hv);
                double2 ps = make_double2(1.0, 0.0);
                if (!DIRECT) ps = __ldg(T.psi_hat + i);
                double2 ac = acc[0];
                ac.x = fma(hv, ps.x, ac.x);
                ac.y = fma(hv, ps.y, ac.y);
                acc[0] = ac;
                c_str += ge - gb;
                ++c_hit;
            }
        }
        PROF_ADD(0, t_diag)
        // ---- (i) same beta string: x' = (a'', b), a'' in A(b);  (ii) same alpha string
        for (int ph = 0; ph < 2; ++ph) {
            if (!(PH & (2 << ph)) || !(phase_mask & (2 << ph))) continue;
            PROF_T(t_ph)
#ifdef NNQS_PROFILE
            prof_in_ss = true;
#endif
            const int32_t g = ph == 0 ? T.gb_of[i] : T.ga_of[i];
            const int32_t *off = ph == 0 ? T.offB : T.offA;
            const u64 *lst = ph == 0 ? T.listB_a : T.listA_b;
            const int32_t *lidx = ph == 0 ? T.listB_idx : T.listA_idx;
            const u64 mine = ph == 0 ? a : b;
            const int32_t jb = off[g], je = off[g + 1];
            if (je - jb <= T.thr_double) {
                for (int32_t j0 = jb; j0 < je; j0 += 128) {
                    u64 v[4];
                    int32_t ix[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t j = j0 + 32 * u + lane;
                        v[u] = j < je ? __ldg(lst + j) : mine;
                    }
                    int32_t kk[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {           // group-id loads of all four issued before any push
                        const int32_t j = j0 + 32 * u + lane;
                        const u64 d = mine ^ v[u];
                        const int c = __popcll(d);
                        kk[u] = -1;
                        ix[u] = 0;
                        if ((c == 2 || c == 4) && (T.uniform_pc || 2 * __popcll(mine & d) == c)) {
                            kk[u] = same_spin_tag(S, ph, d, c, s_lut);
                            ix[u] = __ldg(lidx + j);
                        }
                        c_cand += j < je;
                    }
                    push4(kk, ix);
                }
            } else {
                PROF_T(t_ssh)
                // heavy group: 1-deletion (singles) and 2-deletion (doubles) probes
                const int no = __popcll(mine);
                const int ntask = no + no * (no - 1) / 2;
                const int tag1 = ph == 0 ? 2 : 0;
                for (int t0 = 0; t0 < ntask; t0 += 32) {
                    const int t = t0 + lane;
                    const bool live = t < ntask;
                    u64 key = 0;
                    uint32_t meta = 0;
                    int want = 2;
                    if (live) {
                        const uint8_t *occ = ph == 0 ? occA : occB;
                        if (t < no) {
                            key = mine ^ (1ULL << occ[t]);
                            meta = mm_meta(tag1, g);
                        } else {
                            int i1, i2;
                            nth_pair(t - no, i1, i2);
                            const int p1 = occ[i1], p2 = occ[i2];
                            key = mine ^ (1ULL << p1) ^ (1ULL << p2);
                            meta = mm_meta(tag1 + 1, g);
                            want = 4;
                        }
                        ++c_cand;
                    }
                    int32_t mb = 0, me = 0;
                    if (live) mm_find(T, key, meta, mb, me);
                    drain(mb, me, want, [&](int32_t mj, int32_t swant, int32_t &k, int32_t &idx) {
                        const ulonglong2 en = __ldg(T.mm_ent + mj);
                        idx = (int32_t)en.y;
                        const u64 d = mine ^ en.x;
                        if (__popcll(d) == swant) k = same_spin_tag(S, ph, d, swant, s_lut);
                    });
                }
                PROF_ADD(8, t_ssh)
            }
            PROF_ADD(1 + ph, t_ph)
        }
        PROF_T(t_iii)
#ifdef NNQS_PROFILE
        prof_in_ss = false;
#endif
        // ---- (iii) alpha single u x beta single v
        const int32_t ga_row = T.ga_of[i];
        const bool row_heavy = (PH & 8) && acc_heavy && (T.offA[ga_row + 1] - T.offA[ga_row] > thr_rowheavy);
        if (row_heavy && lane == 0) {              // precomputed by the entry-driven join
            const double2 h = acc_heavy[r];
            double2 ac = acc[0];
            ac.x += h.x;
            ac.y += h.y;
            acc[0] = ac;
        }
        if ((PH & 8) && (phase_mask & 8) && !row_heavy) {
            const u64 va = ~a & nmask, vb = ~b & nmask;
            const int noa = __popcll(a), nva = __popcll(va);
            const int nob = __popcll(b), nvb = __popcll(vb);
            const int combos = noa * nva;
            (void)nvb;
            int nheavy = 0;                          // warp-uniform
            int2 *hl = s_h[(PH & 8) ? (threadIdx.x >> 5) : 0];
            int32_t *pl = s_pl[(PH & 8) ? (threadIdx.x >> 5) : 0];
            // heavy alpha groups a' = a ^ u: probe (a', b - e_r) for every occupied beta r,
            // nheavy x nob probes spread over the lanes, matches drained warp-wide
            auto probe_heavy = [&]() {
                PROF_T(t_hv)
                __syncwarp();
                const int ntask = nheavy * nob;
                // Bloom words first; the probes that pass (~25 %) are compacted (task ids)
                // and only they run the dependent slot -> record -> group chain, 32 at a time
                int np = 0;
                for (int t0 = 0; t0 < ntask || np > 0; t0 += 32) {
                    if (t0 < ntask) {
                        const int t = t0 + lane;
                        bool pass = false;
                        if (t < ntask) {
                            const int h = t / nob, rr = t - h * nob;
                            pass = mm_bloom_pass(T, mm_hash(b ^ (1ULL << occB[rr]), mm_meta(0, hl[h].x)));
                            ++c_cand;
                        }
                        const unsigned pm = __ballot_sync(0xffffffffu, pass);
                        if (pass) pl[np + __popc(pm & lt_mask)] = t;
                        np += __popc(pm);
                        if (np < 32 && t0 + 32 < ntask) continue;
                    }
                    const int cnt = min(np, 32);
                    __syncwarp();
                    int32_t mb = 0, me = 0, ur = 0;
                    if (lane < cnt) {
                        const int t = pl[lane];
                        const int h = t / nob, rr = t - h * nob;
                        const int2 hv = hl[h];
                        ur = hv.y;
                        const u64 key = b ^ (1ULL << occB[rr]);
                        const uint32_t meta = mm_meta(0, hv.x);
                        mm_find_slots(T, mm_hash(key, meta), key, meta, mb, me);
                    }
                    __syncwarp();
                    if (lane < np - cnt) pl[lane] = pl[lane + cnt];
                    np -= cnt;
                    drain(mb, me, ur, [&](int32_t mj, int32_t sur, int32_t &k, int32_t &idx) {
                        const ulonglong2 en = __ldg(T.mm_ent + mj);
                        idx = (int32_t)en.y;
                        const u64 d = b ^ en.x;
                        if (d) {
                            const int r1 = __ffsll((long long)d) - 1;
                            const int r2 = 63 - __clzll((long long)d);
                            k = ab_key(S, sur, pair_rank(r1, r2, S.n));
                        }
                    });
                }
                nheavy = 0;
                __syncwarp();
                PROF_ADD(4, t_hv)
            };
            (void)combos;
            // the alpha strings a' = a ^ u present in the table, with their list ranges:
            // precomputed once per alpha group by nnqs_table_prepare (k_nl_fill)
            const int2 nbr = __ldg(T.nl_rng + ga_row);
            const int32_t nb0 = nbr.x, nb1 = nbr.y;
            for (int32_t c0 = nb0; c0 < nb1; c0 += 32) {
                const int32_t cidx = c0 + lane;
                int32_t g2 = -1, ljb = 0, llen = 0, urank = 0;
                if (cidx < nb1) {
                    const int4 nl = __ldg(T.nl + cidx);
                    g2 = nl.x;
                    urank = nl.y;
                    ljb = nl.z;
                    llen = nl.w;
                    ++c_cand;
                }
                const bool heavy = g2 >= 0 && llen > T.thr_single;
                const int32_t ll = (g2 >= 0 && !heavy) ? llen : 0;
                int32_t incl = ll;                       // warp prefix sum of the light list lengths
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const int32_t excl = incl - ll;
                const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
                // flattened scan of all light lists of this chunk: 128 entries per warp step
                for (int32_t f0 = 0; f0 < ((phase_mask & 16) ? 0 : total); f0 += 128) {
                    u64 v[4];
                    int32_t jj[4], ur[4], ix[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t f = f0 + 32 * u + lane;
                        int lo = 0;
#pragma unroll
                        for (int st = 16; st; st >>= 1) {
                            const int c = lo + st;
                            const int32_t ex = __shfl_sync(0xffffffffu, excl, c & 31);
                            if (c < 32 && ex <= f) lo = c;
                        }
                        const int32_t ob = __shfl_sync(0xffffffffu, ljb, lo);
                        const int32_t oe = __shfl_sync(0xffffffffu, excl, lo);
                        ur[u] = __shfl_sync(0xffffffffu, urank, lo);
                        jj[u] = ob + (f - oe);
                        v[u] = f < total ? __ldg(T.listA_b + jj[u]) : b;
                    }
                    int32_t kk[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {           // group-id and index loads of all four issued
                        const u64 d = b ^ v[u];             // before any push (candidates passing the test)
                        kk[u] = -1;
                        ix[u] = 0;
                        if (__popcll(d) == 2 && (T.uniform_pc || __popcll(b & d) == 1)) {
                            const int r1 = __ffsll((long long)d) - 1;
                            const int r2 = 63 - __clzll((long long)d);
                            if (NNQS_LAZY_AB && S.ab_d) {
                                // existence and table index resolved at evaluation (no dependent
                                // load on the scan): the queue carries the alpha-list position
                                kk[u] = (int32_t)(0x80000000u | AB_TAG | ((uint32_t)ur[u] << 11) |
                                                  (uint32_t)pair_rank(r1, r2, S.n));
                                ix[u] = jj[u];
                            } else {
                                kk[u] = ab_key(S, ur[u], pair_rank(r1, r2, S.n));
                                ix[u] = __ldg(T.listA_idx + jj[u]);
                            }
                        }
                        c_cand += (f0 + 32 * u + lane) < total;
                    }
                    push4(kk, ix);
                }
                // heavy adjacent alpha strings: deferred to the warp's heavy list
                const unsigned hb = __ballot_sync(0xffffffffu, heavy && !(phase_mask & 32));
                if (heavy && !(phase_mask & 32)) hl[nheavy + __popc(hb & lt_mask)] = make_int2(g2, urank);
                nheavy += __popc(hb);
                if (nheavy > HCAP - 32) probe_heavy();
            }
            probe_heavy();
        }
        if (qn > 0) flush(qn);
        PROF_ADD(3, t_iii)
        __syncwarp();
        double ar = acc[lane].x, ai = acc[lane].y;
        const double2 lx = rs->lx;
        constexpr bool direct = DIRECT;
        const double rel = lx.x - s;
        for (int o = 16; o; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
        }
        if (lane == 0 && !(PH & 8)) (((PH & 16) && partial2) ? partial2 : partial)[r] = make_double2(ar, ai);
        if (lane == 0 && (PH & 8)) {
            double2 e;
            if (direct) {
                e = make_double2(ar, ai);
            } else {
                const double m = exp(-rel);
                double sn, cs;
                sincos(-lx.y, &sn, &cs);
                const double ir = m * cs, ii = m * sn;
                e = make_double2(ar * ir - ai * ii, ar * ii + ai * ir);
            }
            out[r] = e;
        }
        if (PH & 8) chunk_done_warp(cs, out, r, n_rows);   // fused first pass of Eq. (6)
        PROF_ADD(7, t_row)
    }
    PROF_FLUSH
    if (stats) {
        for (int o = 16; o; o >>= 1) {
            c_cand += __shfl_xor_sync(0xffffffffu, c_cand, o);
            c_hit += __shfl_xor_sync(0xffffffffu, c_hit, o);
            c_str += __shfl_xor_sync(0xffffffffu, c_str, o);
        }
        if (lane == 0) {
            atomicAdd((unsigned long long *)stats + 1, (unsigned long long)c_cand);
            atomicAdd((unsigned long long *)stats + 2, (unsigned long long)c_hit);
            atomicAdd((unsigned long long *)stats + 3, (unsigned long long)c_str);
        }
    }
}

// ------------------------------------------------------ table-side index build
__device__ __forceinline__ u64 gather_spin(u64 w, int s) {     // bits s, s+2, ... of w -> 32 bits
    w = (w >> s) & 0x5555555555555555ULL;
    w = (w | (w >> 1)) & 0x3333333333333333ULL;
    w = (w | (w >> 2)) & 0x0F0F0F0F0F0F0F0FULL;
    w = (w | (w >> 4)) & 0x00FF00FF00FF00FFULL;
    w = (w | (w >> 8)) & 0x0000FFFF0000FFFFULL;
    w = (w | (w >> 16)) & 0x00000000FFFFFFFFULL;
    return w;
}

__global__ void k_split(const ulonglong2 *keys, int64_t n, u64 *sa, u64 *sb, int32_t *iota) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 k = keys[i];
        sa[i] = gather_spin(k.x, 0) | (gather_spin(k.y, 0) << 32);
        sb[i] = gather_spin(k.x, 1) | (gather_spin(k.y, 1) << 32);
        iota[i] = (int32_t)i;
    }
}

__global__ void k_iota(int32_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

__global__ void k_gather64(const u64 *src, const int32_t *perm, int64_t n, u64 *dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void k_heads(const u64 *ksorted, int64_t n, int32_t *flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        flag[j] = (j == 0 || ksorted[j] != ksorted[j - 1]) ? 1 : 0;
}

// gid = inclusive scan of heads - 1; lists + CSR + group-of-entry
__global__ void k_csr(const u64 *ksorted, const int32_t *perm, const int32_t *incl, int64_t n,
                      const u64 *other, int32_t *off, int32_t *g_of, u64 *list_other, int32_t *list_idx,
                      u64 *hkeys, int32_t *hvals, u64 hmask) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = incl[j] - 1;
        const int32_t e = perm[j];
        g_of[e] = g;
        list_other[j] = other[e];
        list_idx[j] = e;
        const bool head = (j == 0 || ksorted[j] != ksorted[j - 1]);
        if (head) {
            off[g] = (int32_t)j;
            if (hkeys) {
                const u64 key = ksorted[j];
                u64 s = mix64(key) & hmask;
                while (atomicCAS((int *)(hvals + s), -1, g) != -1) s = (s + 1) & hmask;
                hkeys[s] = key;
            }
        }
        if (j == n - 1) off[g + 1] = (int32_t)n;
    }
}

// keys per entry (heavy groups only)
__device__ __forceinline__ int mm_keys_of(int32_t la, int32_t lb, int na, int nb, int32_t thr_s, int32_t thr_d) {
    int c = 0;
    if (la > thr_s) c += nb;
    if (la > thr_d) c += nb * (nb - 1) / 2;
    if (lb > thr_d) c += na;                 // beta groups are probed (phase (i)) only above thr_d
    if (lb > thr_d) c += na * (na - 1) / 2;
    return c;
}

__global__ void k_mm_count(const u64 *sa, const u64 *sb, const int32_t *ga_of, const int32_t *gb_of,
                           const int32_t *offA, const int32_t *offB, int64_t n, int32_t thr_s, int32_t thr_d,
                           int32_t *counts, int *pc_range, int32_t *flagB) {
    // also: popcount range of the alpha / beta strings (min a, max a, min b, max b) and
    // the beta groups that receive keys (for the compact sort key)
    int mna = 64, mxa = 0, mnb = 64, mxb = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t la = offA[ga_of[e] + 1] - offA[ga_of[e]];
        const int32_t lb = offB[gb_of[e] + 1] - offB[gb_of[e]];
        const int pa = __popcll(sa[e]), pb = __popcll(sb[e]);
        counts[e] = mm_keys_of(la, lb, pa, pb, thr_s, thr_d);
        if (lb > thr_d) flagB[gb_of[e]] = 1;
        mna = min(mna, pa); mxa = max(mxa, pa);
        mnb = min(mnb, pb); mxb = max(mxb, pb);
    }
    atomicMin(pc_range + 0, mna);
    atomicMax(pc_range + 1, mxa);
    atomicMin(pc_range + 2, mnb);
    atomicMax(pc_range + 3, mxb);
}

__global__ void k_flag_alpha(const int32_t *offA, int64_t ng, int32_t thr_s, int32_t *flagA) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng;
         g += (int64_t)gridDim.x * blockDim.x)
        flagA[g] = offA[g + 1] - offA[g] > thr_s ? 1 : 0;
}

// binomials C(p, k), p < 64, k < 32 (colex rank of a deletion string)
__device__ u64 d_binom[64 * 32];

// Compact sort key of a multimap record: (meta rank << rbits) | colex rank of the key
// among strings of its popcount -- injective when every alpha (beta) string of the
// table has one popcount, so one radix sort on ~55 bits groups the runs.
__device__ __forceinline__ u64 mm_sort_key(u64 key, uint32_t meta, const int32_t *rankA, const int32_t *rankB,
                                           int32_t NA, int32_t NB, int rbits) {
    const int tag = (int)(meta >> 30);
    const int32_t g = (int32_t)(meta & 0x3FFFFFFFu);
    const u64 mr = tag < 2 ? (u64)(rankA[g] + (tag == 1 ? NA : 0)) : (u64)(2 * NA + rankB[g] + (tag == 3 ? NB : 0));
    u64 r = 0;
    int i = 0;
    for (u64 w = key; w; w &= w - 1, ++i) r += d_binom[(__ffsll((long long)w) - 1) * 32 + i + 1];
    return (mr << rbits) | r;
}

// Balanced emission: block of 256 entries, their keys (up to 15 + 105 + 15 + 105
// each) flattened through a block prefix sum and written by all threads, coalesced.
// Same key set and the same entry order per run as k_mm_emit (a run's entries are
// ordered by entry index; each entry contributes at most one key to a run).
__global__ void __launch_bounds__(256) k_mm_emit_flat(const u64 *sa, const u64 *sb, const int32_t *ga_of,
                                                      const int32_t *gb_of, const int32_t *offA, const int32_t *offB,
                                                      int64_t n, int32_t thr_s, int32_t thr_d, const int32_t *counts,
                                                      const int64_t *eoff, u64 *K, uint32_t *M, int32_t *V,
                                                      u64 *SV, u64 *SK, const int32_t *rankA, const int32_t *rankB,
                                                      int32_t NA, int32_t NB, int rbits) {
    typedef cub::BlockScan<int32_t, 256> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int32_t s_pre[257];
    __shared__ u64 s_a[256], s_b[256];
    __shared__ int32_t s_ga[256], s_gb[256];
    __shared__ uint8_t s_f[256];
    const int64_t e0 = (int64_t)blockIdx.x * 256;
    const int64_t e = e0 + threadIdx.x;
    int32_t c = 0;
    if (e < n) {
        c = counts[e];
        const int32_t ga = ga_of[e], gb = gb_of[e];
        const int32_t la = offA[ga + 1] - offA[ga], lb = offB[gb + 1] - offB[gb];
        s_a[threadIdx.x] = sa[e];
        s_b[threadIdx.x] = sb[e];
        s_ga[threadIdx.x] = ga;
        s_gb[threadIdx.x] = gb;
        s_f[threadIdx.x] = (uint8_t)((la > thr_s ? 1 : 0) | (la > thr_d ? 2 : 0) | (lb > thr_d ? 12 : 0));
    }
    int32_t ex, total;
    Scan(tmp).ExclusiveSum(c, ex, total);
    s_pre[threadIdx.x] = ex;
    if (threadIdx.x == 0) s_pre[256] = total;
    __syncthreads();
    if (e0 >= n) return;
    const int64_t base = eoff[e0];
    for (int32_t p = threadIdx.x; p < total; p += 256) {
        int lo = 0, hi = 256;                          // last t with s_pre[t] <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_pre[mid] <= p) lo = mid; else hi = mid;
        }
        int32_t l = p - s_pre[lo];
        const uint8_t f = s_f[lo];
        u64 key = 0, w = 0;
        uint32_t meta = 0;
        for (int side = 0; side < 2; ++side) {
            const u64 ws = side == 0 ? s_b[lo] : s_a[lo];      // side 0: beta deletions keyed by the alpha group
            const int32_t gs = side == 0 ? s_ga[lo] : s_gb[lo];
            const int tag = side == 0 ? 0 : 2;
            const int ns = __popcll(ws);
            if (f & (side == 0 ? 1 : 4)) {
                if (l < ns) { key = ws ^ (1ULL << nth_set(ws, l)); meta = mm_meta(tag, gs); w = ws; break; }
                l -= ns;
            }
            if (f & (side == 0 ? 2 : 8)) {
                const int np = ns * (ns - 1) / 2;
                if (l < np) {
                    int i1, i2;
                    nth_pair(l, i1, i2);
                    key = ws ^ (1ULL << nth_set(ws, i1)) ^ (1ULL << nth_set(ws, i2));
                    meta = mm_meta(tag + 1, gs);
                    w = ws;
                    break;
                }
                l -= np;
            }
        }
        const int64_t o = base + p;
        K[o] = key;
        M[o] = meta;
        V[o] = (int32_t)(e0 + lo);
        SV[o] = w;
        if (SK) SK[o] = mm_sort_key(key, meta, rankA, rankB, NA, NB, rbits);
    }
}

__global__ void k_gather32(const uint32_t *src, const int32_t *perm, int64_t n, uint32_t *dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void k_mm_heads(const u64 *K2, const uint32_t *M2, int64_t m, int32_t *flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        flag[j] = (j == 0 || K2[j] != K2[j - 1] || M2[j] != M2[j - 1]) ? 1 : 0;
}

__global__ void k_mm_runs(const u64 *K2, const uint32_t *M2, const int32_t *P2, const int32_t *V, const u64 *SV,
                          const int32_t *rid, int64_t m, int32_t *run_start, ulonglong2 *ent) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        ent[j] = make_ulonglong2(SV[P2[j]], (u64)(uint32_t)V[P2[j]]);
        const int32_t r = rid[j] - 1;
        if (j == 0 || K2[j] != K2[j - 1] || M2[j] != M2[j - 1]) run_start[r] = (int32_t)j;
        if (j == m - 1) run_start[r + 1] = (int32_t)m;
    }
}

// one slot per run: claimed by CAS on the meta word, then key and bounds written
__global__ void k_mm_slots(const u64 *K2, const uint32_t *M2, const int32_t *run_start, int64_t nruns,
                           ulonglong2 *slots, u64 mask, u64 *bloom, u64 bmask) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = run_start[r], je = run_start[r + 1];
        const u64 key = K2[j];
        const uint32_t meta = M2[j];
        const u64 h = mm_hash(key, meta);
        atomicOr(bloom + ((h >> 32) & bmask), (1ULL << ((h >> 20) & 63)) | (1ULL << ((h >> 26) & 63)));
        u64 s = h & mask;
        while (true) {
            uint32_t *w = reinterpret_cast<uint32_t *>(slots + 2 * s);
            if (atomicCAS(w + 2, MM_EMPTY, meta) == MM_EMPTY) {
                slots[2 * s].x = key;
                w[3] = (uint32_t)j;
                slots[2 * s + 1] = make_ulonglong2((u64)(uint32_t)je, 0);
                break;
            }
            s = (s + 1) & mask;
        }
    }
}

// ---------------------------------------------- entry-driven phase (iii) join
// For an alpha group g with very many rows (the Hartree-Fock alpha string pairs
// with ~10^5 rows at 120 qubits), phase (iii) is evaluated from the neighbour
// side: every entry (a', b'') of every adjacent alpha string a' = a ^ u probes
// the 1-deletions b'' - e_s in g's multimap (tag 0) and finds the rows (a, b)
// with b - e_r = b'' - e_s.  Hits are emitted as (row, x' index) keys, sorted,
// and summed per row in that order (k_hj_eval), so the result is deterministic.
// Hit key of the join: (row - row_begin) << ibits | table index of x'; sorting
// the keys on their used bits orders every row's hits by x' (deterministic sums).
#ifndef HJ_FLIGHT
#define HJ_FLIGHT 4   // matches per lane in flight (k_hj_emit)
#endif
__global__ void __launch_bounds__(256) k_hj_emit(SpinView S, TabSpin T, const int32_t *heavy_groups, int n_heavy,
                                                 int64_t row_begin, int64_t row_end, int clip, int ibits,
                                                 int kbits, unsigned long long *counter, u64 *keys_out, int64_t cap,
                                                 unsigned long long *stats) {
    // (heavy group g = blockIdx.y): the tasks (adjacent alpha string a', entry of
    // list(a'), occupied beta orbital of the entry) of all of g's adjacent strings
    // are flattened through a block-local prefix sum and spread over the whole grid
    // (list lengths differ by 100x: one block per a' left most SMs idle)
    const int hg = blockIdx.y;
    if (hg >= n_heavy) return;
    const int32_t g = heavy_groups[hg];
    const int32_t nb0 = T.nl_rng[g].x, nb1 = T.nl_rng[g].y;
    const int nc = nb1 - nb0;                        // <= n_alpha * n_empty <= 1024 (n <= 64)
    __shared__ long long s_pre[1025];
    __shared__ int4 s_nl[1024];
    __shared__ int s_nob[1024];
    typedef cub::BlockScan<long long, 256> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    long long cnt4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int c = 4 * threadIdx.x + u;
        cnt4[u] = 0;
        if (c < nc) {
            const int4 nl = T.nl[nb0 + c];
            const int nob = __popcll(T.listA_b[nl.z]);     // all entries of one table sector share it
            s_nl[c] = nl;
            s_nob[c] = nob;
            cnt4[u] = (long long)nl.w * nob;
        }
    }
    long long tot = 0;
    Scan(scan_tmp).ExclusiveSum(cnt4, cnt4, tot);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (4 * threadIdx.x + u < nc) s_pre[4 * threadIdx.x + u] = cnt4[u];
    if (threadIdx.x == 0) s_pre[nc] = tot;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t meta = mm_meta(0, g);
    unsigned long long probes = 0;
    for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < tot; t0 += (long long)gridDim.x * blockDim.x) {
        const long long t = t0 + threadIdx.x;
        int32_t mb = 0, me = 0, idx2 = 0, abo = 0;
        u64 b2 = 0;
        if (t < tot) {
            int lo = 0, hi = nc;                         // last c with s_pre[c] <= t
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= t) lo = mid; else hi = mid;
            }
            const int4 nl = s_nl[lo];
            const int nob = s_nob[lo];
            const long long loc = t - s_pre[lo];
            const int32_t j = nl.z + (int32_t)(loc / nob);
            const int sb = (int)(loc % nob);
            abo = nl.y;
            b2 = T.listA_b[j];
            idx2 = T.listA_idx[j];
            mm_find(T, b2 ^ (1ULL << nth_set(b2, sb)), meta, mb, me);
            ++probes;
            if (clip && me > mb) {
                // a run's records are in table-entry order: keep only this rank's rows
                // (the same matches the filter below keeps, without loading the others)
                int32_t lo = mb, hi = me;
                while (lo < hi) {
                    const int32_t mid = (lo + hi) >> 1;
                    if ((int64_t)(int32_t)T.mm_ent[mid].y < row_begin) lo = mid + 1; else hi = mid;
                }
                int32_t lo2 = lo, hi2 = me;
                while (lo2 < hi2) {
                    const int32_t mid = (lo2 + hi2) >> 1;
                    if ((int64_t)(int32_t)T.mm_ent[mid].y < row_end) lo2 = mid + 1; else hi2 = mid;
                }
                mb = lo;
                me = lo2;
            }
        }
        // the warp's matches, flattened over the lanes (run lengths differ widely):
        // lane f of a step takes the f-th match in (lane, position) order
        const int32_t len = me - mb;
        int32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int32_t excl = incl - len;
        const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (int32_t f0 = 0; f0 < total; f0 += 32 * HJ_FLIGHT) {
            // HJ_FLIGHT matches per lane: records, then group ids, loaded before any use
            ulonglong2 en[HJ_FLIGHT];
            u64 bo[HJ_FLIGHT];
            int32_t io[HJ_FLIGHT], ao[HJ_FLIGHT];
#pragma unroll
            for (int u = 0; u < HJ_FLIGHT; ++u) {
                const int32_t f = f0 + 32 * u + lane;
                int lo = 0;
#pragma unroll
                for (int st = 16; st; st >>= 1) {
                    const int c = lo + st;
                    const int32_t ex = __shfl_sync(0xffffffffu, excl, c & 31);
                    if (c < 32 && ex <= f) lo = c;
                }
                const int32_t mj = __shfl_sync(0xffffffffu, mb, lo) + (f - __shfl_sync(0xffffffffu, excl, lo));
                bo[u] = __shfl_sync(0xffffffffu, b2, lo);
                io[u] = __shfl_sync(0xffffffffu, idx2, lo);
                ao[u] = __shfl_sync(0xffffffffu, abo, lo);
                en[u] = f < total ? T.mm_ent[mj] : make_ulonglong2(bo[u], 0);   // d = 0: no hit
            }
            int32_t kk[HJ_FLIGHT];
#pragma unroll
            for (int u = 0; u < HJ_FLIGHT; ++u) {
                const int32_t e = (int32_t)en[u].y;
                const u64 d = en[u].x ^ bo[u];
                kk[u] = -1;
                if (e >= row_begin && e < row_end && d != 0) {
                    const int r1 = __ffsll((long long)d) - 1, r2 = 63 - __clzll((long long)d);
                    kk[u] = S.ab_k[(int64_t)ao[u] * S.P + pair_rank(r1, r2, S.n)];
                }
            }
            // one warp-aggregated slot reservation for all HJ_FLIGHT x 32 matches
            unsigned m[HJ_FLIGHT];
            int nok = 0;
#pragma unroll
            for (int u = 0; u < HJ_FLIGHT; ++u) {
                m[u] = __ballot_sync(0xffffffffu, kk[u] >= 0);
                nok += __popc(m[u]);
            }
            unsigned long long base = 0;
            if (lane == 0 && nok) base = atomicAdd(counter, (unsigned long long)nok);
            base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
            for (int u = 0; u < HJ_FLIGHT; ++u) {
                if (kk[u] >= 0) {
                    const unsigned long long slot = base + __popc(m[u] & ((1u << lane) - 1u));
                    if ((int64_t)slot < cap)
                        keys_out[slot] =
                            ((((u64)((int32_t)en[u].y - row_begin) << ibits) | (u64)(uint32_t)io[u]) << kbits) |
                            (kbits ? (u64)(uint32_t)kk[u] : 0);
                }
                base += __popc(m[u]);
            }
        }
    }
    if (stats) {
        for (int o = 16; o; o >>= 1) probes += __shfl_xor_sync(0xffffffffu, probes, o);
        if (lane == 0) atomicAdd(stats + 1, probes);
    }
}

// first / one-past-last position of every row's run in the sorted keys
__global__ void k_hj_bounds(const u64 *keys, int64_t m, int shift, int32_t *kb, int32_t *ke) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const u64 r = keys[j] >> shift;
        if (j == 0 || (keys[j - 1] >> shift) != r) kb[r] = (int32_t)j;
        if (j == m - 1 || (keys[j + 1] >> shift) != r) ke[r] = (int32_t)(j + 1);
    }
}

// one warp per row of the heavy groups: sum its sorted hits (fixed lane order)
template <bool LOG>
__global__ void k_hj_eval(SpinView S, GroupView G, TabSpin T, const int32_t *heavy_groups, int n_heavy,
                          int64_t row_begin, int64_t row_end, const u64 *keys, int ibits, int kbits, const int32_t *kb,
                          const int32_t *ke, double2 *acc, unsigned long long *stats) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double s = dkey_inv2(*T.shift_key);
    const u64 imask = (1ULL << ibits) - 1, kmask = (1ULL << kbits) - 1;
    unsigned long long c_hit = 0, c_str = 0;
    for (int hg = 0; hg < n_heavy; ++hg) {
        const int32_t g = heavy_groups[hg];
        const int32_t rb = T.offA[g], re = T.offA[g + 1];
        for (int64_t t = warp; t < re - rb; t += nwarps) {
            const int32_t e = T.listA_idx[rb + t];
            if (e < row_begin || e >= row_end) continue;
            const u64 rloc = (u64)(e - row_begin);
            const int32_t hb = kb[rloc], he = ke[rloc];
            const ulonglong2 xk = T.keys[e];
            const u64 a = T.sa[e], b = T.sb[e];
            const double2 lx = T.logpsi[e];
            const bool direct = (lx.x - s) < -600.0;
            double ar = 0.0, ai = 0.0;
            int32_t j = hb + lane;
            if (kbits && !direct) {
                // four hits per lane in flight: keys -> (offsets, psi_hat) -> strings;
                // accumulation order unchanged (j ascending per lane)
                for (; j + 96 < he; j += 128) {
                    int32_t kk[4], ix[4];
                    uint32_t b0[4], b1[4];
                    double2 ps[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const u64 key = keys[j + 32 * u];
                        ix[u] = (int32_t)((key >> kbits) & imask);
                        kk[u] = (int32_t)(key & kmask);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint2 be = g_range(G, kk[u]);
                        b0[u] = be.x;
                        b1[u] = be.y;
                        ps[u] = __ldg(T.psi_hat + ix[u]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        double hv = 0.0;
                        for (uint32_t i = b0[u]; i < b1[u]; ++i) {
                            const ulonglong2 Z = g_z(G, i);
                            hv += flip_sign2(g_d(G, i), (__popcll(xk.x & Z.x) + __popcll(xk.y & Z.y)) & 1);
                        }
                        c_str += b1[u] - b0[u];
                        if (LOG && T.log.count) log_hit(T.log, e, ix[u], hv);
                        ar = fma(hv, ps[u].x, ar);
                        ai = fma(hv, ps[u].y, ai);
                        ++c_hit;
                    }
                }
            }
            for (; j < he; j += 32) {
                const u64 key = keys[j];
                const int32_t idx = (int32_t)((key >> kbits) & imask);
                int32_t k;
                if (kbits) {
                    k = (int32_t)(key & kmask);       // group id carried in the key's low bits
                } else {
                    const u64 du = a ^ T.sa[idx], dv = b ^ T.sb[idx];
                    const int p1 = __ffsll((long long)du) - 1, p2 = 63 - __clzll((long long)du);
                    const int r1 = __ffsll((long long)dv) - 1, r2 = 63 - __clzll((long long)dv);
                    k = S.ab_k[pair_rank(p1, p2, S.n) * S.P + pair_rank(r1, r2, S.n)];
                }
                const double hv = group_value1(G, k, xk.x, xk.y, c_str);
                if (LOG && T.log.count) log_hit(T.log, e, idx, hv);
                double2 ps;
                if (!direct) {
                    ps = T.psi_hat[idx];
                } else {
                    const double2 l = T.logpsi[idx];
                    const double mg = exp(l.x - lx.x);
                    double sn, cs;
                    sincos(l.y - lx.y, &sn, &cs);
                    ps = make_double2(mg * cs, mg * sn);
                }
                ar = fma(hv, ps.x, ar);
                ai = fma(hv, ps.y, ai);
                ++c_hit;
            }
            for (int o = 16; o; o >>= 1) {
                ar += __shfl_xor_sync(0xffffffffu, ar, o);
                ai += __shfl_xor_sync(0xffffffffu, ai, o);
            }
            if (lane == 0) acc[rloc] = make_double2(ar, ai);
        }
    }
    if (stats) {
        for (int o = 16; o; o >>= 1) {
            c_hit += __shfl_xor_sync(0xffffffffu, c_hit, o);
            c_str += __shfl_xor_sync(0xffffffffu, c_str, o);
        }
        if (lane == 0) {
            atomicAdd(stats + 2, c_hit);
            atomicAdd(stats + 3, c_str);
        }
    }
}

// Adjacent alpha strings of each alpha group g (a' = a ^ u, u = one occupied ->
// one empty orbital, a' present in the table), warp per group, in (occupied,
// empty) order.
#define NL_WARPS 4
__global__ void __launch_bounds__(32 * NL_WARPS) k_nl(TabSpin T, int n_orb, int64_t n_groups, int2 *rng, int4 *nl,
                                                     unsigned long long *cursor, int32_t thr_single, int32_t *cost) {
    // one pass: the present a' are compacted into the warp's shared buffer, one
    // atomic reserves the group's block, the buffer is written out.  Block
    // positions depend on scheduling; each group's list (and its order) does not.
    __shared__ int2 s_nl[NL_WARPS][1024];          // (g', u rank); occupied x empty <= 1024 for n <= 64
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    int2 *buf = s_nl[threadIdx.x >> 5];
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const u64 nmask = n_orb >= 64 ? ~0ULL : ((1ULL << n_orb) - 1);
    for (int64_t g = warp; g < n_groups; g += nwarps) {
        const u64 a = T.sa[T.listA_idx[T.offA[g]]];
        const u64 va = ~a & nmask;
        const int noa = __popcll(a), nva = __popcll(va);
        const int combos = noa * nva;
        int32_t cnt = 0;
        for (int c0 = 0; c0 < combos; c0 += 32) {
            const int c = c0 + lane;
            int32_t g2 = -1;
            int p = 0, q = 0;
            if (c < combos) {
                p = nth_set(a, c / nva);
                q = nth_set(va, c % nva);
                g2 = alpha_lookup(T, a ^ (1ULL << p) ^ (1ULL << q));
            }
            const unsigned m = __ballot_sync(0xffffffffu, g2 >= 0);
            if (g2 >= 0) buf[cnt + __popc(m & lt_mask)] = make_int2(g2, pair_rank(min(p, q), max(p, q), n_orb));
            cnt += __popc(m);
        }
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(cursor, (unsigned long long)cnt);
        const int32_t pos = (int32_t)__shfl_sync(0xffffffffu, base, 0);
        if (lane == 0) rng[g] = make_int2(pos, pos + cnt);
        int32_t work = 0;                            // phase (iii) work estimate of a row of g
        for (int c = lane; c < cnt; c += 32) {
            const int2 e = buf[c];
            const int32_t b0 = T.offA[e.x], len = T.offA[e.x + 1] - b0;
            nl[pos + c] = make_int4(e.x, e.y, b0, len);
            work += len > thr_single ? 64 : len;
        }
        for (int o = 16; o; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
        if (lane == 0) cost[g] = work;
        __syncwarp();
    }
}

// ---- adjacent-alpha lists by a deletion join: two alpha strings of the table are
// one single excitation apart iff they share a 1-deletion, and they share exactly
// one.  Each group emits its n_alpha deletions; after a sort on the deletion, every
// run lists strings that are pairwise adjacent.
__global__ void k_adel_count(const u64 *sa, const int32_t *listA_idx, const int32_t *offA, int64_t ng,
                             int32_t *cnt) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x)
        cnt[g] = __popcll(sa[listA_idx[offA[g]]]);
}

__global__ void k_adel_emit(const u64 *sa, const int32_t *listA_idx, const int32_t *offA, int64_t ng,
                            const int32_t *eoff, u64 *DK, int32_t *DV) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
        const u64 a = sa[listA_idx[offA[g]]];
        int32_t o = eoff[g];
        for (u64 w = a; w; w &= w - 1, ++o) {
            DK[o] = a ^ (w & (~w + 1));
            DV[o] = (int32_t)g;
        }
    }
}

// run bounds of every sorted element, and its neighbour count (run size - 1)
__global__ void k_adel_runs(const u64 *DK2, int64_t m, int32_t *rb, int32_t *re, int32_t *nn) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = j, e = j + 1;
        while (b > 0 && DK2[b - 1] == DK2[j]) --b;      // runs are short (<= n_empty + 1)
        while (e < m && DK2[e] == DK2[j]) ++e;
        rb[j] = (int32_t)b;
        re[j] = (int32_t)e;
        nn[j] = (int32_t)(e - b - 1);
    }
}

__global__ void k_adel_gcount(const int32_t *G2, const int32_t *nn_g, int64_t m, int32_t *gcnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if (nn_g[i]) atomicAdd(gcnt + G2[i], nn_g[i]);
}

__global__ void k_adel_rng(const int32_t *beg, int64_t ng, int2 *rng) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x)
        rng[g] = make_int2(beg[g], beg[g + 1]);
}

// element order i (sorted by group, then by deletion): write the run's other members
__global__ void k_adel_fill(const u64 *sa, const int32_t *listA_idx, const int32_t *offA, int n_orb, int64_t m,
                            const int32_t *G2, const int32_t *J2, const int32_t *within, const int32_t *gbeg,
                            const int32_t *DV2, const int32_t *rb, const int32_t *re, int32_t thr_single, int4 *nl,
                            int32_t *cost) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = G2[i], j = J2[i];
        const u64 a = sa[listA_idx[offA[g]]];
        int32_t pos = gbeg[g] + within[i];
        int32_t work = 0;
        for (int32_t jj = rb[j]; jj < re[j]; ++jj) {
            if (jj == j) continue;
            const int32_t g2 = DV2[jj];
            const u64 a2 = sa[listA_idx[offA[g2]]];
            const int p = __ffsll((long long)(a & ~a2)) - 1, q = __ffsll((long long)(a2 & ~a)) - 1;
            const int32_t b0 = offA[g2], len = offA[g2 + 1] - b0;
            nl[pos++] = make_int4(g2, pair_rank(min(p, q), max(p, q), n_orb), b0, len);
            work += len > thr_single ? 64 : len;
        }
        if (work) atomicAdd(cost + g, work);
    }
}

// per-row work estimates of the three row kernels (sort keys for a longest-first
// row order): same-spin list lengths (probes above thr_d), adjacent-alpha work
__global__ void k_row_cost(TabSpin T, int64_t row_begin, int64_t n_rows, int32_t thr_d, int32_t thr_rowheavy,
                           const int32_t *nl_cost, uint32_t *c3, uint32_t *c20, uint32_t *c24, int32_t *iota) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = row_begin + r;
        const int32_t ga = T.ga_of[i], gb = T.gb_of[i];
        const int32_t la = T.offA[ga + 1] - T.offA[ga], lb = T.offB[gb + 1] - T.offB[gb];
        c3[r] = (uint32_t)(lb > thr_d ? 4096 : lb);
        c20[r] = (uint32_t)(la > thr_d ? 4096 : la);
        // phase (iii): longest first by cost class (two octaves of the adjacent-alpha work),
        // rows of one beta string together within a class -- rows (a1, b), (a2, b) next to a
        // common heavy a' repeat the same (a', b - e_r) probes, which then hit in L2
        // (measured: 45.2 -> 44.2 ms per C5 call; exact longest-first or pure beta order: 45.1)
        const uint32_t c = la > thr_rowheavy ? 0u : (uint32_t)nl_cost[ga];
#ifndef NNQS_P3_CLASS
#define NNQS_P3_CLASS 2                           // octaves per cost class
#endif
        const uint32_t cls = c ? (uint32_t)((31 - __clz(c)) / NNQS_P3_CLASS) + 1u : 0u;
        c24[r] = (cls << 22) | ((uint32_t)gb & 0x3FFFFFu);
        iota[r] = (int32_t)r;
    }
}

// per-chunk work estimate of the three row kernels and the entry-driven join (for
// cost-balanced rank slices): per row base + beta-side list (phase i) + alpha-side
// list (phase ii) + adjacent-alpha work (phase iii); lists above thr_d are probed
// (cost pd), rows of join-evaluated alpha groups cost pj.  One block per chunk.
__global__ void __launch_bounds__(256) k_chunk_work(TabSpin T, int64_t chunk, int32_t thr_d, int32_t thr_rowheavy,
                                                    const int32_t *nl_cost, int32_t w0, int32_t pd, int32_t pj,
                                                    int32_t px, int32_t pf, long long *work, long long *floor_out) {
    const int64_t r0 = (int64_t)blockIdx.x * chunk;
    const int64_t r1 = (r0 + chunk < T.n) ? r0 + chunk : T.n;
    long long w = 0, fl = 0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const int32_t ga = T.ga_of[i], gb = T.gb_of[i];
        const int32_t la = T.offA[ga + 1] - T.offA[ga], lb = T.offB[gb + 1] - T.offB[gb];
        w += w0 + (lb > thr_d ? pd : lb) + (la > thr_d ? pd : la) + (la > thr_rowheavy ? pj : (nl_cost ? nl_cost[ga] : 0));
        // rows whose alpha and beta lists are both probed (the Hartree-Fock row and its
        // like) drain matches near both strings in one warp: ~ la * lb / n, a latency floor
        if (la > thr_d && lb > thr_d) {
            w += (long long)px * la * lb / T.n;
            fl = max(fl, (long long)pf * la * lb / T.n);
        }
    }
    typedef cub::BlockReduce<long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    const long long tot = Red(tmp).Sum(w);
    __syncthreads();
    const long long mx = Red(tmp).Reduce(fl, cub::Max());
    if (threadIdx.x == 0) {
        work[blockIdx.x] = tot;
        if (floor_out) floor_out[blockIdx.x] = mx;
    }
}

// predicate of the heavy alpha groups (more than thr rows) for cub::DeviceSelect::If
struct HeavyGroup {
    const int32_t *offA;
    int32_t thr;
    __device__ __forceinline__ bool operator()(const int32_t g) const { return offA[g + 1] - offA[g] > thr; }
};

}  // namespace

// ============================================================== host side
int nnqs_spin_index_build(const HostTable &H, SpinIndex &S) {
    S = SpinIndex();
    const int N = H.n_qubits;
    if (!H.conserving || N > 128 || (N & 1)) return NNQS_OK;
    const int n = N / 2;
    S.n = n;
    S.P = (int64_t)n * (n - 1) / 2;
    S.Q = n >= 4 ? (int64_t)n * (n - 1) * (n - 2) * (n - 3) / 24 : 0;
    for (int s = 0; s < 2; ++s) {
        S.pair_k[s].assign(std::max<int64_t>(S.P, 1), -1);
        S.quad_k[s].assign(std::max<int64_t>(S.Q, 1), -1);
    }
    S.ab_k.assign(std::max<int64_t>(S.P * S.P, 1), -1);
    const int64_t K = (int64_t)H.off.size() - 1;
    for (int64_t k = 0; k < K; ++k) {
        int pos[2][4], cnt[2] = {0, 0};
        bool bad = false;
        for (int w = 0; w < 2 && !bad; ++w) {
            u64 x = H.x[2 * k + w];
            while (x) {
                const int j = 64 * w + __builtin_ctzll(x);
                x &= x - 1;
                const int s = j & 1, p = j >> 1;
                if (cnt[s] == 4) { bad = true; break; }
                pos[s][cnt[s]++] = p;        // ascending (qubits ascend)
            }
        }
        if (bad) return NNQS_OK;
        const int ca = cnt[0], cb = cnt[1];
        if (ca == 0 && cb == 0) S.diag_k = (int32_t)k;
        else if (ca == 2 && cb == 0) S.pair_k[0][pair_rank(pos[0][0], pos[0][1], n)] = (int32_t)k;
        else if (ca == 0 && cb == 2) S.pair_k[1][pair_rank(pos[1][0], pos[1][1], n)] = (int32_t)k;
        else if (ca == 4 && cb == 0) S.quad_k[0][quad_rank(pos[0][0], pos[0][1], pos[0][2], pos[0][3])] = (int32_t)k;
        else if (ca == 0 && cb == 4) S.quad_k[1][quad_rank(pos[1][0], pos[1][1], pos[1][2], pos[1][3])] = (int32_t)k;
        else if (ca == 2 && cb == 2)
            S.ab_k[pair_rank(pos[0][0], pos[0][1], n) * S.P + pair_rank(pos[1][0], pos[1][1], n)] = (int32_t)k;
        else return NNQS_OK;               // not a single/double excitation pattern
    }
    // ---- in-sector folding (see SpinIndex): generators F of each group type
    S.foff.assign(K + 1, 0);
    S.fz.clear();
    S.fd.clear();
    for (int64_t k = 0; k < K; ++k) {
        u64 X[2] = {H.x[2 * k], H.x[2 * k + 1]};
        u64 F[2][2] = {{0, 0}, {0, 0}};
        int nf = 0;
        u64 xs[2][2] = {{0, 0}, {0, 0}};        // X restricted to spin s (qubits 2p+s)
        for (int w = 0; w < 2; ++w) {
            xs[0][w] = X[w] & 0x5555555555555555ULL;
            xs[1][w] = X[w] & 0xAAAAAAAAAAAAAAAAULL;
        }
        const int ca = __builtin_popcountll(xs[0][0]) + __builtin_popcountll(xs[0][1]);
        const int cb = __builtin_popcountll(xs[1][0]) + __builtin_popcountll(xs[1][1]);
        if (ca == 2 || ca == 4) { F[nf][0] = xs[0][0]; F[nf][1] = xs[0][1]; ++nf; }   // sign (-1)^{ca/2}
        if (cb == 2 || cb == 4) { F[nf][0] = xs[1][0]; F[nf][1] = xs[1][1]; ++nf; }
        std::vector<std::pair<std::pair<u64, u64>, long double>> acc;
        for (int64_t t = H.off[k]; t < H.off[k + 1]; ++t) {
            u64 z0 = H.z[2 * t], z1 = H.z[2 * t + 1];
            long double d = H.d[t];
            // canonical representative: clear the lowest set bit of each generator
            for (int g = 0; g < nf; ++g) {
                const int cnt = __builtin_popcountll(F[g][0]) + __builtin_popcountll(F[g][1]);
                const u64 lowbit0 = F[g][0] ? (F[g][0] & (~F[g][0] + 1)) : 0;
                const u64 lowbit1 = F[g][0] ? 0 : (F[g][1] & (~F[g][1] + 1));
                const bool has = (z0 & lowbit0) || (z1 & lowbit1);
                if (has) {
                    z0 ^= F[g][0];
                    z1 ^= F[g][1];
                    if (cnt == 2) d = -d;      // (-1)^{popc(x & F)} = -1 in sector (one of the pair set)
                }                              // cnt == 4: +1 (two of the quad set)
            }
            acc.push_back({{z1, z0}, d});
        }
        std::sort(acc.begin(), acc.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
        for (size_t u = 0; u < acc.size();) {
            size_t v = u;
            long double sum = 0.0L;
            while (v < acc.size() && acc[v].first == acc[u].first) sum += acc[v++].second;
            if ((double)sum != 0.0) {
                S.fz.push_back(acc[u].first.second);
                S.fz.push_back(acc[u].first.first);
                S.fd.push_back((double)sum);
            }
            u = v;
        }
        S.foff[k + 1] = (uint32_t)S.fd.size();
    }
    // ---- alpha x beta slots whose folded group is one string: the string's index
    S.ab_rec.assign(S.ab_k.size(), -1);
    for (size_t i = 0; i < S.ab_k.size(); ++i) {
        const int32_t k = S.ab_k[i];
        if (k < 0) continue;
        const uint32_t b0 = S.foff[k], b1 = S.foff[k + 1];
        S.ab_rec[i] = (b1 == b0 + 1 && b0 < 0x10000000u && k < 0x40000000) ? (int32_t)(0x40000000u | b0) : k;
    }
    // ---- alpha x beta groups in closed form (SpinIndex::ab_ok): the folded group is
    // one string equal to canon(J) (or none: the strings cancelled, value 0); any
    // other shape leaves the path on the per-string records
    S.ab_ok = N <= 128 && S.P <= 2048 && K < 0x20000000;
    if (S.ab_ok) {
        S.pair_sites.assign(std::max<int64_t>(S.P, 1), 0);
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) S.pair_sites[pair_rank(p, q, n)] = (uint32_t)p | ((uint32_t)q << 8);
        S.ab_w = (S.P + 63) / 64;
        S.ab_d.assign(std::max<int64_t>(S.P * S.P, 1), std::numeric_limits<double>::quiet_NaN());   // NaN: no group
        S.ab_bits.assign(std::max<int64_t>(S.P * S.ab_w, 1), 0);
        auto between = [](int lo, int hi, u64 &m0, u64 &m1) {   // qubits lo < j < hi
            for (int j = lo + 1; j < hi; ++j) (j < 64 ? m0 : m1) ^= 1ULL << (j & 63);
        };
        S.pair_J.assign(4 * std::max<int64_t>(S.P, 1), 0);
        for (int64_t U = 0; U < S.P; ++U) {
            const int p = S.pair_sites[U] & 0xFF, q = S.pair_sites[U] >> 8;
            between(2 * p, 2 * q, S.pair_J[2 * U], S.pair_J[2 * U + 1]);
            between(2 * p + 1, 2 * q + 1, S.pair_J[2 * (S.P + U)], S.pair_J[2 * (S.P + U) + 1]);
        }
        for (int64_t U = 0; U < S.P && S.ab_ok; ++U)
            for (int64_t V = 0; V < S.P; ++V) {
                const int32_t k = S.ab_k[U * S.P + V];
                if (k < 0) continue;
                const int p = S.pair_sites[U] & 0xFF, q = S.pair_sites[U] >> 8;
                const int r = S.pair_sites[V] & 0xFF, s2 = S.pair_sites[V] >> 8;
                const int qa = 2 * p, qb = 2 * q, qc = 2 * r + 1, qd = 2 * s2 + 1;
                u64 Z0 = S.pair_J[2 * U] ^ S.pair_J[2 * (S.P + V)];
                u64 Z1 = S.pair_J[2 * U + 1] ^ S.pair_J[2 * (S.P + V) + 1];
                double sign = 1.0;
                for (int g2 = 0; g2 < 2; ++g2) {           // canonical representative: clear the low site
                    const int lo = g2 == 0 ? qa : qc, hi = g2 == 0 ? qb : qd;
                    if (((lo < 64 ? Z0 : Z1) >> (lo & 63)) & 1) {
                        (lo < 64 ? Z0 : Z1) ^= 1ULL << (lo & 63);
                        (hi < 64 ? Z0 : Z1) ^= 1ULL << (hi & 63);
                        sign = -sign;                      // popc(x & pair) is odd in sector
                    }
                }
                const uint32_t b0 = S.foff[k], b1 = S.foff[k + 1];
                double v = 0.0;
                if (b1 == b0 + 1 && S.fz[2 * b0] == Z0 && S.fz[2 * b0 + 1] == Z1) v = sign * S.fd[b0];
                else if (b1 != b0) { S.ab_ok = false; break; }
                S.ab_d[U * S.P + V] = v;
                S.ab_bits[U * S.ab_w + (V >> 6)] |= 1ULL << (V & 63);
            }
        if (!S.ab_ok) { S.ab_d.clear(); S.ab_bits.clear(); S.pair_sites.clear(); S.pair_J.clear(); }
    }
    // ---- same-spin quads likewise (their folded groups hold up to 3 strings)
    for (int sp = 0; sp < 2; ++sp) {
        S.quad_rec[sp].assign(S.quad_k[sp].size(), -1);
        for (size_t i = 0; i < S.quad_k[sp].size(); ++i) {
            const int32_t k = S.quad_k[sp][i];
            if (k < 0) continue;
            const uint32_t b0 = S.foff[k], b1 = S.foff[k + 1];
            S.quad_rec[sp][i] = (b1 > b0 && b1 - b0 <= 4 && b0 < 0x10000000u && k < 0x40000000)
                                    ? (int32_t)(0x40000000u | ((b1 - b0 - 1) << 28) | b0) : k;
        }
    }
    // ---- single-excitation groups in occupation form (see SpinIndex::occ_rec)
    S.occ_ok = N <= 128;
    if (S.occ_ok) {
        const int stride = 4 + N;
        S.occ_rec.assign((size_t)2 * S.P * stride, 0.0);
        for (int sp = 0; sp < 2 && S.occ_ok; ++sp)
            for (int64_t rk = 0; rk < S.P && S.occ_ok; ++rk) {
                const int32_t k = S.pair_k[sp][rk];
                if (k < 0) {                        // no group: NaN total, the kernels drop such hits
                    S.occ_rec[((size_t)sp * S.P + rk) * stride + 2] = std::numeric_limits<double>::quiet_NaN();
                    continue;
                }
                // base B = bitwise majority of the group's strings (the JW string J of
                // the pair; every other string is J ^ Z_R)
                int cnt[128] = {0};
                const uint32_t ns = S.foff[k + 1] - S.foff[k];
                for (uint32_t t = S.foff[k]; t < S.foff[k + 1]; ++t)
                    for (int w = 0; w < 2; ++w)
                        for (u64 z = S.fz[2 * t + w]; z; z &= z - 1) ++cnt[64 * w + __builtin_ctzll(z)];
                u64 B0 = 0, B1 = 0;
                for (int j = 0; j < 128; ++j)
                    if (2 * (uint32_t)cnt[j] > ns) (j < 64 ? B0 : B1) |= 1ULL << (j & 63);
                double *rec = &S.occ_rec[((size_t)sp * S.P + rk) * stride];
                long double Tg = 0.0L;
                for (uint32_t t = S.foff[k]; t < S.foff[k + 1]; ++t) {
                    const u64 w0 = S.fz[2 * t] ^ B0, w1 = S.fz[2 * t + 1] ^ B1;
                    const int pc = __builtin_popcountll(w0) + __builtin_popcountll(w1);
                    if (pc > 1) { S.occ_ok = false; break; }
                    Tg += S.fd[t];
                    if (pc == 1) rec[4 + (w0 ? __builtin_ctzll(w0) : 64 + __builtin_ctzll(w1))] += S.fd[t];
                }
                std::memcpy(&rec[0], &B0, 8);
                std::memcpy(&rec[1], &B1, 8);
                rec[2] = (double)Tg;
            }
        if (!S.occ_ok) S.occ_rec.clear();
    }
    // ---- diagonal group in occupation form (s_p = 1 - 2 n_p):
    //   c0 + sum_p c_p s_p + sum_{p<q} c_pq s_p s_q
    //   = K + sum_{p occ} u_p + sum_{p<q occ} v_pq,
    //   K = c0 + sum c_p + sum c_pq,  u_p = -2 (c_p + sum_{q != p} c_pq),  v_pq = 4 c_pq
    S.diag_ok = false;
    if (S.diag_k >= 0 && N <= 128) {
        std::vector<long double> c1(N, 0.0L), c2((size_t)N * N, 0.0L);
        long double c0 = 0.0L;
        bool ok = true;
        for (int64_t t = H.off[S.diag_k]; t < H.off[S.diag_k + 1] && ok; ++t) {
            int q[3], nb = 0;
            for (int w = 0; w < 2; ++w)
                for (u64 z = H.z[2 * t + w]; z; z &= z - 1) {
                    if (nb == 2) { ok = false; break; }
                    q[nb++] = 64 * w + __builtin_ctzll(z);
                }
            if (!ok) break;
            if (nb == 0) c0 += H.d[t];
            else if (nb == 1) c1[q[0]] += H.d[t];
            else { c2[(size_t)q[0] * N + q[1]] += H.d[t]; c2[(size_t)q[1] * N + q[0]] += H.d[t]; }
        }
        if (ok) {
            long double K = c0;
            for (int p = 0; p < N; ++p) {
                K += c1[p];
                for (int q = p + 1; q < N; ++q) K += c2[(size_t)p * N + q];
            }
            S.diag_uv.assign((size_t)N + (size_t)N * N, 0.0);
            for (int p = 0; p < N; ++p) {
                long double R = 0.0L;
                for (int q = 0; q < N; ++q) R += c2[(size_t)p * N + q];
                S.diag_uv[p] = (double)(-2.0L * (c1[p] + R));
                for (int q = 0; q < N; ++q) S.diag_uv[N + (size_t)p * N + q] = (double)(4.0L * c2[(size_t)p * N + q]);
            }
            S.diag_K = (double)K;
            S.diag_ok = true;
        }
    }
    S.ok = true;
    return NNQS_OK;
}

int nnqs_spin_index_upload(nnqs_ham h) {
    SpinIndex &S = h->spin;
    DeviceHam &D = h->dev;
    if (!S.ok) return NNQS_OK;
    int rc;
    for (int s = 0; s < 2; ++s) {
        size_t bp = 4 * S.pair_k[s].size(), bq = 4 * S.quad_k[s].size();
        if ((rc = cuda_check(cudaMalloc((void **)&D.pair_k[s], bp), "alloc pair_k"))) return rc;
        if ((rc = cuda_check(cudaMalloc((void **)&D.quad_k[s], bq), "alloc quad_k"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.pair_k[s], S.pair_k[s].data(), bp, cudaMemcpyHostToDevice), "copy pair_k"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.quad_k[s], S.quad_k[s].data(), bq, cudaMemcpyHostToDevice), "copy quad_k"))) return rc;
        if (S.quad_rec[s].size() == S.quad_k[s].size()) {
            if ((rc = cuda_check(cudaMalloc((void **)&D.quad_rec[s], bq), "alloc quad_rec"))) return rc;
            if ((rc = cuda_check(cudaMemcpy(D.quad_rec[s], S.quad_rec[s].data(), bq, cudaMemcpyHostToDevice),
                                 "copy quad_rec"))) return rc;
            D.bytes += (int64_t)bq;
        }
        D.bytes += (int64_t)(bp + bq);
    }
    size_t bab = 4 * S.ab_k.size();
    if ((rc = cuda_check(cudaMalloc((void **)&D.ab_k, bab), "alloc ab_k"))) return rc;
    if ((rc = cuda_check(cudaMemcpy(D.ab_k, S.ab_k.data(), bab, cudaMemcpyHostToDevice), "copy ab_k"))) return rc;
    D.bytes += (int64_t)bab;
    if (S.ab_rec.size() == S.ab_k.size()) {
        if ((rc = cuda_check(cudaMalloc((void **)&D.ab_rec, bab), "alloc ab_rec"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.ab_rec, S.ab_rec.data(), bab, cudaMemcpyHostToDevice), "copy ab_rec"))) return rc;
        D.bytes += (int64_t)bab;
    }
    if (S.ab_ok) {
        const size_t bd = 8 * S.ab_d.size(), bb = 8 * S.ab_bits.size();
        const size_t bj = 8 * S.pair_J.size();
        if ((rc = cuda_check(cudaMalloc((void **)&D.pair_J, bj), "alloc pair_J"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.pair_J, S.pair_J.data(), bj, cudaMemcpyHostToDevice), "copy pair_J"))) return rc;
        D.bytes += (int64_t)bj;
        if ((rc = cuda_check(cudaMalloc((void **)&D.ab_d, bd), "alloc ab_d"))) return rc;
        if ((rc = cuda_check(cudaMalloc((void **)&D.ab_bits, bb), "alloc ab_bits"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.ab_d, S.ab_d.data(), bd, cudaMemcpyHostToDevice), "copy ab_d"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.ab_bits, S.ab_bits.data(), bb, cudaMemcpyHostToDevice), "copy ab_bits"))) return rc;
        D.bytes += (int64_t)(bd + bb);
    }
    if (S.occ_ok) {
        const size_t bo2 = 8 * S.occ_rec.size();
        if ((rc = cuda_check(cudaMalloc((void **)&D.occ_rec, bo2), "alloc occ"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.occ_rec, S.occ_rec.data(), bo2, cudaMemcpyHostToDevice), "copy occ"))) return rc;
        D.bytes += (int64_t)bo2;
    }
    if (S.diag_ok) {
        const size_t bu = 8 * S.diag_uv.size();
        if ((rc = cuda_check(cudaMalloc((void **)&D.diag_uv, bu), "alloc diag"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.diag_uv, S.diag_uv.data(), bu, cudaMemcpyHostToDevice), "copy diag"))) return rc;
        D.bytes += (int64_t)bu;
    }
    {
        const int64_t K = (int64_t)S.foff.size() - 1, M = (int64_t)S.fd.size();
        std::vector<uint32_t> rng(2 * std::max<int64_t>(K, 1), 0);
        for (int64_t k = 0; k < K; ++k) {
            rng[2 * k] = S.foff[k];
            rng[2 * k + 1] = S.foff[k + 1];
        }
        std::vector<u64> rec(4 * std::max<int64_t>(M, 1), 0);
        for (int64_t i = 0; i < M; ++i) {
            rec[4 * i] = S.fz[2 * i];
            rec[4 * i + 1] = S.fz[2 * i + 1];
            std::memcpy(&rec[4 * i + 2], &S.fd[i], 8);
        }
        const size_t br = 4 * rng.size(), bq = 8 * rec.size();
        if ((rc = cuda_check(cudaMalloc((void **)&D.frng, br), "alloc folded ranges"))) return rc;
        if ((rc = cuda_check(cudaMalloc((void **)&D.frec, bq), "alloc folded strings"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.frng, rng.data(), br, cudaMemcpyHostToDevice), "copy folded ranges"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.frec, rec.data(), bq, cudaMemcpyHostToDevice), "copy folded strings"))) return rc;
        D.bytes += (int64_t)(br + bq);
    }
    return NNQS_OK;
}

void nnqs_spin_index_release(nnqs_ham h) {
    DeviceHam &D = h->dev;
    for (int s = 0; s < 2; ++s) {
        cudaFree(D.pair_k[s]);
        cudaFree(D.quad_k[s]);
        cudaFree(D.quad_rec[s]);
        D.pair_k[s] = D.quad_k[s] = D.quad_rec[s] = nullptr;
    }
    cudaFree(D.ab_k);
    D.ab_k = nullptr;
    cudaFree(D.ab_rec);
    D.ab_rec = nullptr;
    cudaFree(D.ab_d);
    cudaFree(D.ab_bits);
    cudaFree(D.pair_J);
    D.pair_J = nullptr;
    D.ab_d = nullptr;
    D.ab_bits = nullptr;
    cudaFree(D.diag_uv);
    D.diag_uv = nullptr;
    cudaFree(D.occ_rec);
    D.occ_rec = nullptr;
    cudaFree(D.frng);
    cudaFree(D.frec);
    D.frng = nullptr;
    D.frec = nullptr;
}

namespace {
int ensure_binom(int device) {
    static bool ready[64] = {false};
    static std::mutex mu;
    if (device < 0 || device >= 64) return NNQS_E_ARG;
    std::lock_guard<std::mutex> lk(mu);
    if (ready[device]) return NNQS_OK;
    static u64 tab[64 * 32];
    for (int p = 0; p < 64; ++p)
        for (int k = 0; k < 32; ++k) {
            long double r = (k > p) ? 0.0L : 1.0L;
            for (int i = 1; i <= k && k <= p; ++i) r = r * (p - k + i) / i;
            tab[p * 32 + k] = (u64)(r + 0.5L);
        }
    cudaError_t e = cudaMemcpyToSymbol(d_binom, tab, sizeof(tab));
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    ready[device] = true;
    return NNQS_OK;
}

int build_multimap(nnqs_table t, int64_t n, cudaStream_t st, int32_t *counts, void *, size_t) {
    const int g = grid_for(n, 256);
    int64_t *eoff = nullptr;
    int rc = cuda_check(nnqs_malloc_async((void **)&eoff, 8 * (n + 1), st), "alloc mm offsets");
    if (rc) return rc;
    // compact-key support: popcount range, dense ranks of the groups that receive keys
    const int64_t nga = t->n_alpha_groups;
    int32_t *rk = nullptr;                       // [pc_range 4 | flagA nga+1 | rankA | flagB n+1 | rankB]
    rc = cuda_check(nnqs_malloc_async((void **)&rk, 4 * (4 + 2 * (nga + 1) + 2 * (n + 1)) + 64, st), "alloc mm ranks");
    if (rc) { cudaFreeAsync(eoff, st); return rc; }
    int *pcr = rk;
    int32_t *flagA = rk + 4, *rankA = flagA + nga + 1, *flagB = rankA + nga + 1, *rankB = flagB + n + 1;
    {
        const int init[4] = {64, 0, 64, 0};
        cudaMemcpyAsync(pcr, init, sizeof(init), cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(flagB, 0, 4 * (n + 1), st);
        cudaMemsetAsync(flagA + nga, 0, 4, st);
    }
    k_mm_count<<<g, 256, 0, st>>>(t->sa, t->sb, t->ga_of, t->gb_of, t->offA, t->offB, n, t->thr_single,
                                  t->thr_double, counts, pcr, flagB);
    k_flag_alpha<<<grid_for(nga, 256), 256, 0, st>>>(t->offA, nga, t->thr_single, flagA);
    {
        size_t ts1 = 0, ts2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, ts1, flagA, rankA, (int)nga + 1, st);
        cub::DeviceScan::ExclusiveSum(nullptr, ts2, flagB, rankB, (int)n + 1, st);
        void *tsc = nullptr;
        rc = cuda_check(nnqs_malloc_async(&tsc, std::max(ts1, ts2), st), "alloc rank scan");
        if (rc) { cudaFreeAsync(rk, st); cudaFreeAsync(eoff, st); return rc; }
        cub::DeviceScan::ExclusiveSum(tsc, ts1, flagA, rankA, (int)nga + 1, st);
        cub::DeviceScan::ExclusiveSum(tsc, ts2, flagB, rankB, (int)n + 1, st);
        cudaFreeAsync(tsc, st);
    }
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, eoff, (int)n + 1, st);
    void *stmp = nullptr;
    cudaMemsetAsync(eoff + n, 0, 8, st);
    rc = cuda_check(nnqs_malloc_async(&stmp, tb, st), "alloc scan tmp");
    if (rc) { cudaFreeAsync(eoff, st); return rc; }
    // counts has n entries; scan n+1 with a zero appended (counts[n] read as 0)
    int32_t *cz = nullptr;
    nnqs_malloc_async((void **)&cz, 4 * (n + 1), st);
    cudaMemcpyAsync(cz, counts, 4 * n, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(cz + n, 0, 4, st);
    cub::DeviceScan::ExclusiveSum(stmp, tb, cz, eoff, (int)n + 1, st);
    int64_t m = 0;
    int hpc[4] = {0, 0, 0, 0};
    int32_t NA = 0, NB = 0;
    rc = cuda_check(cudaMemcpyAsync(&m, eoff + n, 8, cudaMemcpyDeviceToHost, st), "read mm size");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(hpc, pcr, sizeof(hpc), cudaMemcpyDeviceToHost, st), "read pc range");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(&NA, rankA + nga, 4, cudaMemcpyDeviceToHost, st), "read NA");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(&NB, rankB + n, 4, cudaMemcpyDeviceToHost, st), "read NB");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
    cudaFreeAsync(stmp, st);
    cudaFreeAsync(cz, st);
    // compact key: one popcount per side, meta rank and colex rank in <= 64 bits
    int rbits = 0, kbits_all = 65;
    if (!rc && hpc[0] == hpc[1] && hpc[2] == hpc[3] && t->spin_n <= 64) {
        auto binom = [](int nn, int kk) -> long double {
            if (kk < 0 || kk > nn) return 0.0L;
            long double r = 1.0L;
            for (int i = 1; i <= kk; ++i) r = r * (nn - kk + i) / i;
            return r;
        };
        long double mx = 1.0L;
        for (int pc : {hpc[0], hpc[2]})
            for (int d = 1; d <= 2; ++d) mx = std::max(mx, binom(t->spin_n, pc - d));
        while (rbits < 64 && (long double)(1ULL << rbits) < mx) ++rbits;
        int mbits = 0;
        while ((1LL << mbits) < 2LL * NA + 2LL * NB + 1) ++mbits;
        kbits_all = rbits + mbits;
    }
    const bool compact = kbits_all <= 64 && ensure_binom(t->device) == NNQS_OK;
    t->uniform_pc = !rc && hpc[0] == hpc[1] && hpc[2] == hpc[3];
    if (rc || m == 0) {
        cudaFreeAsync(rk, st);
        cudaFreeAsync(eoff, st);
        if (!rc) {   // empty multimap: one empty slot
            rc = cuda_check(nnqs_malloc_async(&t->mm_buf, 128, st), "alloc mm");
            if (rc) return rc;
            t->mm = t->mm_buf;
            t->mm_mask = 0;
            t->mm_ent = (char *)t->mm_buf + 64;
            t->mm_bloom = (u64 *)((char *)t->mm_buf + 96);
            t->mm_bloom_mask = 0;
            cudaMemsetAsync(t->mm, 0xFF, 32, st);
            cudaMemsetAsync(t->mm_bloom, 0, 8, st);
        }
        return rc;
    }
    if (m >= (1LL << 31)) {
        cudaFreeAsync(rk, st);
        cudaFreeAsync(eoff, st);
        return nnqs_set_error(NNQS_E_SIZE, "multimap too large");
    }
    // scratch for the sort
    auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (const u64 *)nullptr, (u64 *)nullptr, (const int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)m, 0, 64, st);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)m, 0, 32, st);
    cub::DeviceScan::InclusiveSum(nullptr, t3, (const int32_t *)nullptr, (int32_t *)nullptr, (int)m, st);
    const size_t ctb = std::max(t1, std::max(t2, t3));
    const size_t sbytes = 4 * r16(8 * m) + 3 * r16(4 * m) + 4 * r16(4 * m) + r16(ctb) + 64;
    char *sc = nullptr;
    rc = cuda_check(nnqs_malloc_async((void **)&sc, sbytes, st), "alloc mm scratch");
    if (rc) { cudaFreeAsync(rk, st); cudaFreeAsync(eoff, st); return rc; }
    char *sp = sc;
    auto take = [&](size_t b) { char *p = sp; sp += r16(b); return p; };
    u64 *K = (u64 *)take(8 * m), *K1 = (u64 *)take(8 * m), *K2 = (u64 *)take(8 * m), *SV = (u64 *)take(8 * m);
    uint32_t *M = (uint32_t *)take(4 * m), *M1 = (uint32_t *)take(4 * m), *M2 = (uint32_t *)take(4 * m);
    int32_t *V = (int32_t *)take(4 * m), *io = (int32_t *)take(4 * (m + 1)), *P1 = (int32_t *)take(4 * m),
            *P2 = (int32_t *)take(4 * m);
    void *ct = take(ctb);
    const int gm = grid_for(m, 256);
    k_mm_emit_flat<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(t->sa, t->sb, t->ga_of, t->gb_of, t->offA, t->offB,
                                                               n, t->thr_single, t->thr_double, counts, eoff, K, M,
                                                               V, SV, compact ? K1 : nullptr, rankA, rankB, NA, NB,
                                                               rbits);
    k_iota<<<gm, 256, 0, st>>>(io, m);
    size_t tb1 = ctb;
    if (compact) {
        // one stable sort on (meta rank, colex rank): runs grouped by (meta, key), a
        // run's records in emission (entry) order -- the same order as the two sorts
        cub::DeviceRadixSort::SortPairs(ct, tb1, K1, K2, io, P2, (int)m, 0, kbits_all, st);
        k_gather32<<<gm, 256, 0, st>>>(M, P2, m, M2);
        k_gather64<<<gm, 256, 0, st>>>(K, P2, m, K2);
    } else {
        cub::DeviceRadixSort::SortPairs(ct, tb1, K, K1, io, P1, (int)m, 0, 64, st);
        k_gather32<<<gm, 256, 0, st>>>(M, P1, m, M1);
        tb1 = ctb;
        cub::DeviceRadixSort::SortPairs(ct, tb1, M1, M2, P1, P2, (int)m, 0, 32, st);
        k_gather64<<<gm, 256, 0, st>>>(K, P2, m, K2);
    }
    k_mm_heads<<<gm, 256, 0, st>>>(K2, M2, m, io);        // io reused as head flags
    tb1 = ctb;
    cub::DeviceScan::InclusiveSum(ct, tb1, io, P1, (int)m, st);   // P1 reused as run ids (1-based)
    int32_t nruns = 0;
    rc = cuda_check(cudaMemcpyAsync(&nruns, P1 + m - 1, 4, cudaMemcpyDeviceToHost, st), "read runs");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
    if (rc) { cudaFreeAsync(sc, st); cudaFreeAsync(eoff, st); return rc; }
    u64 slots = 2;   // slots >= MM_LOAD * runs (power of two)
    while ((double)slots < MM_LOAD * (double)nruns) slots <<= 1;
    u64 bwords = 1;
    while (bwords * 64 < (u64)MM_BLOOM_BITS * (u64)nruns) bwords <<= 1;
    const size_t pbytes = r16(32 * slots) + r16(16 * m) + r16(8 * bwords);
    rc = cuda_check(nnqs_malloc_async(&t->mm_buf, pbytes, st), "alloc multimap");
    if (rc) { cudaFreeAsync(sc, st); cudaFreeAsync(eoff, st); return rc; }
    t->mm = t->mm_buf;
    t->mm_mask = slots - 1;
    t->mm_ent = (char *)t->mm_buf + r16(32 * slots);
    t->mm_bloom = (u64 *)((char *)t->mm_ent + r16(16 * m));
    t->mm_bloom_mask = bwords - 1;
    t->bytes += (int64_t)pbytes;
    cudaMemsetAsync(t->mm, 0xFF, 32 * slots, st);
    cudaMemsetAsync(t->mm_bloom, 0, 8 * bwords, st);
    int32_t *run_start = io;   // head flags are dead after the scan; io holds m + 1 ints >= nruns + 1
    k_mm_runs<<<gm, 256, 0, st>>>(K2, M2, P2, V, SV, P1, m, run_start, (ulonglong2 *)t->mm_ent);
    k_mm_slots<<<grid_for(nruns, 256), 256, 0, st>>>(K2, M2, run_start, nruns, (ulonglong2 *)t->mm, t->mm_mask,
                                                         t->mm_bloom, t->mm_bloom_mask);
    cudaFreeAsync(sc, st);
    cudaFreeAsync(eoff, st);
    cudaFreeAsync(rk, st);
    return cuda_check(cudaGetLastError(), "multimap kernels");
}
}  // namespace

int nnqs_table_build_spin(nnqs_ham h, nnqs_table t, void *stream, bool *checked) {
    if (!h->spin.ok || t->mode != 0 || t->n == 0) return NNQS_OK;
    t->spin_n = h->spin.n;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = t->n;
    if (n >= (1LL << 31) - 2) return NNQS_OK;
    u64 hs = 1;
    while (hs < 2 * (u64)n) hs <<= 1;
    // temp storage for the two sorts
    size_t tmp_sort = 0, tmp_scan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const u64 *)nullptr, (u64 *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 64, st);
    cub::DeviceScan::InclusiveSum(nullptr, tmp_scan, (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, st);
    const size_t tmp = std::max(tmp_sort, tmp_scan);
    // persistent arrays
    auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
    const size_t pers = 2 * r16(8 * n) + 2 * r16(4 * n) + 2 * r16(4 * (n + 1)) + 2 * r16(8 * n) + 2 * r16(4 * n) +
                        r16(8 * hs) + r16(4 * hs) + 16;
    // scratch: iota, perm1, perm2 (int32), k1, k2 (u64), flags, incl (int32), cub temp
    const size_t scr = 5 * r16(4 * n) + 2 * r16(8 * n) + r16(tmp) + 16;
    char *buf = nullptr;
    int rc = cuda_check(nnqs_malloc_async((void **)&buf, pers, st), "alloc spin index");
    if (rc) return rc;
    char *scratch = nullptr;
    rc = cuda_check(nnqs_malloc_async((void **)&scratch, scr, st), "alloc spin scratch");
    if (rc) { cudaFreeAsync(buf, st); return rc; }
    t->spin_buf = buf;
    auto take = [&](size_t bytes) { char *p = buf; buf += (bytes + 15) & ~size_t(15); return p; };
    t->sa = (u64 *)take(8 * n);
    t->sb = (u64 *)take(8 * n);
    t->ga_of = (int32_t *)take(4 * n);
    t->gb_of = (int32_t *)take(4 * n);
    t->offA = (int32_t *)take(4 * (n + 1));
    t->offB = (int32_t *)take(4 * (n + 1));
    t->listA_b = (u64 *)take(8 * n);
    t->listA_idx = (int32_t *)take(4 * n);
    t->listB_a = (u64 *)take(8 * n);
    t->listB_idx = (int32_t *)take(4 * n);
    t->ah_keys = (u64 *)take(8 * hs);
    t->ah_vals = (int32_t *)take(4 * hs);
    t->ah_mask = hs - 1;
    t->bytes += (int64_t)pers;
    char *sp = scratch;
    auto stake = [&](size_t bytes) { char *p = sp; sp += (bytes + 15) & ~size_t(15); return p; };
    int32_t *iota = (int32_t *)stake(4 * n), *perm1 = (int32_t *)stake(4 * n), *perm2 = (int32_t *)stake(4 * n);
    u64 *k1 = (u64 *)stake(8 * n), *k2 = (u64 *)stake(8 * n);
    int32_t *flags = (int32_t *)stake(4 * n), *incl = (int32_t *)stake(4 * n);
    void *ctmp = stake(tmp);
    const int g = grid_for(n, 256);
    k_split<<<g, 256, 0, st>>>((const ulonglong2 *)t->keys, n, t->sa, t->sb, iota);
    cudaMemsetAsync(t->ah_vals, 0xFF, 4 * hs, st);
    for (int pass = 0; pass < 2; ++pass) {
        // pass 0: sort by (a, b) -> alpha groups, lists of b;  pass 1: by (b, a)
        const u64 *primary = pass == 0 ? t->sa : t->sb;
        const u64 *secondary = pass == 0 ? t->sb : t->sa;
        size_t tb = tmp;
        cub::DeviceRadixSort::SortPairs(ctmp, tb, secondary, k1, iota, perm1, (int)n, 0, 64, st);
        k_gather64<<<g, 256, 0, st>>>(primary, perm1, n, k2);
        tb = tmp;
        cub::DeviceRadixSort::SortPairs(ctmp, tb, k2, k1, perm1, perm2, (int)n, 0, 64, st);
        k_heads<<<g, 256, 0, st>>>(k1, n, flags);
        tb = tmp;
        cub::DeviceScan::InclusiveSum(ctmp, tb, flags, incl, (int)n, st);
        if (pass == 0) {
            k_csr<<<g, 256, 0, st>>>(k1, perm2, incl, n, t->sb, t->offA, t->ga_of, t->listA_b, t->listA_idx,
                                     t->ah_keys, t->ah_vals, t->ah_mask);
            int32_t nga = 0;
            int tflag[2] = {0, 0};   // nnqs_table_build's flags, read at the same sync
            rc = cuda_check(cudaMemcpyAsync(&nga, incl + n - 1, 4, cudaMemcpyDeviceToHost, st), "read alpha groups");
            if (!rc) rc = cuda_check(cudaMemcpyAsync(tflag, t->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st), "read flag");
            if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
            if (!rc) rc = nnqs_table_check(t, tflag, st);
            if (checked) *checked = true;
            if (rc) { cudaFreeAsync(scratch, st); return rc; }
            t->n_alpha_groups = nga;
        }
        else
            k_csr<<<g, 256, 0, st>>>(k1, perm2, incl, n, t->sa, t->offB, t->gb_of, t->listB_a, t->listB_idx,
                                     nullptr, nullptr, 0);
    }
    t->thr_single = t->opt.thr_single;   // per-table options (nnqs_options; defaults measured in DESIGN.md Sec. 7)
    t->thr_double = t->opt.thr_double;
    // adjacent-alpha lists per alpha group (phase (iii) streams them instead of
    // repeating the 675 alpha-string lookups for every row of the group)
    {
        const int64_t ng = t->n_alpha_groups;
        const int n_orb = h->spin.n;
        const int64_t maxc = (int64_t)(n_orb / 2) * (n_orb - n_orb / 2);   // max occupied x empty
        const size_t rb = (8 * (size_t)ng + 15) & ~size_t(15);            // 16-B aligned regions
        const size_t cb = (4 * (size_t)ng + 15) & ~size_t(15);
        const size_t bytes = rb + 64 + cb + 16 * (size_t)(ng * maxc + 1);
        rc = cuda_check(nnqs_malloc_async(&t->nl_buf, bytes, st), "alloc nl");
        if (rc) { cudaFreeAsync(scratch, st); return rc; }
        t->nl_rng = t->nl_buf;
        unsigned long long *cursor = (unsigned long long *)((char *)t->nl_buf + rb);
        t->nl_cost = (int32_t *)((char *)t->nl_buf + rb + 64);
        t->nl = (char *)t->nl_buf + rb + 64 + cb;
        t->bytes += (int64_t)bytes;
        if (n_orb < 64) {
            // deletion join (see k_adel_*): ~n_alpha keys per group instead of
            // n_alpha x n_empty hash lookups
            int32_t *cnt = nullptr;
            rc = cuda_check(nnqs_malloc_async((void **)&cnt, 8 * (ng + 2), st), "alloc nl join counts");
            if (rc) { cudaFreeAsync(scratch, st); return rc; }
            int32_t *eoff = cnt + ng + 1;
            cudaMemsetAsync(cnt + ng, 0, 4, st);
            k_adel_count<<<grid_for(ng, 256), 256, 0, st>>>(t->sa, t->listA_idx, t->offA, ng, cnt);
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, eoff, (int)ng + 1, st);
            void *tmp0 = nullptr;
            rc = cuda_check(nnqs_malloc_async(&tmp0, tb, st), "alloc nl join scan");
            if (rc) { cudaFreeAsync(cnt, st); cudaFreeAsync(scratch, st); return rc; }
            cub::DeviceScan::ExclusiveSum(tmp0, tb, cnt, eoff, (int)ng + 1, st);
            cudaFreeAsync(tmp0, st);
            int32_t m32 = 0;
            rc = cuda_check(cudaMemcpyAsync(&m32, eoff + ng, 4, cudaMemcpyDeviceToHost, st), "read nl join size");
            if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
            if (rc) { cudaFreeAsync(cnt, st); cudaFreeAsync(scratch, st); return rc; }
            const int64_t m = m32;
            size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, t1, (const u64 *)nullptr, (u64 *)nullptr, (const int32_t *)nullptr,
                                            (int32_t *)nullptr, (int)m, 0, n_orb, st);
            cub::DeviceRadixSort::SortPairs(nullptr, t2, (const int32_t *)nullptr, (int32_t *)nullptr,
                                            (const int32_t *)nullptr, (int32_t *)nullptr, (int)m, 0, 32, st);
            cub::DeviceScan::ExclusiveSumByKey(nullptr, t3, (const int32_t *)nullptr, (const int32_t *)nullptr,
                                               (int32_t *)nullptr, (int)m, cub::Equality(), st);
            cub::DeviceScan::ExclusiveSum(nullptr, t4, (const int32_t *)nullptr, (int32_t *)nullptr, (int)ng + 1, st);
            const size_t tt = std::max(std::max(t1, t2), std::max(t3, t4));
            auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
            char *w = nullptr;
            const size_t wb = 2 * al(8 * m) + 9 * al(4 * (m + 1)) + al(4 * (ng + 1)) + al(tt);
            rc = cuda_check(nnqs_malloc_async((void **)&w, wb, st), "alloc nl join work");
            if (rc) { cudaFreeAsync(cnt, st); cudaFreeAsync(scratch, st); return rc; }
            char *wp = w;
            auto tk = [&](size_t x) { char *p0 = wp; wp += al(x); return p0; };
            u64 *DK = (u64 *)tk(8 * m), *DK2 = (u64 *)tk(8 * m);
            int32_t *DV = (int32_t *)tk(4 * (m + 1)), *DV2 = (int32_t *)tk(4 * (m + 1));
            int32_t *rbv = (int32_t *)tk(4 * (m + 1)), *rev = (int32_t *)tk(4 * (m + 1)), *nn = (int32_t *)tk(4 * (m + 1));
            int32_t *io = (int32_t *)tk(4 * (m + 1)), *G2 = (int32_t *)tk(4 * (m + 1)), *J2 = (int32_t *)tk(4 * (m + 1));
            int32_t *within = (int32_t *)tk(4 * (m + 1));
            int32_t *gcnt = (int32_t *)tk(4 * (ng + 1));
            void *ctmp2 = tk(tt);
            const int gm = grid_for(m, 256);
            k_adel_emit<<<grid_for(ng, 256), 256, 0, st>>>(t->sa, t->listA_idx, t->offA, ng, eoff, DK, DV);
            size_t tb1 = tt;
            cub::DeviceRadixSort::SortPairs(ctmp2, tb1, DK, DK2, DV, DV2, (int)m, 0, n_orb, st);
            k_adel_runs<<<gm, 256, 0, st>>>(DK2, m, rbv, rev, nn);
            k_iota<<<gm, 256, 0, st>>>(io, m);
            tb1 = tt;   // element order by group (stable: by deletion within a group)
            cub::DeviceRadixSort::SortPairs(ctmp2, tb1, DV2, G2, io, J2, (int)m, 0, 32, st);
            k_gather32<<<gm, 256, 0, st>>>((const uint32_t *)nn, J2, m, (uint32_t *)io);
            tb1 = tt;   // io = nn in group order; within = its exclusive sum per group
            cub::DeviceScan::ExclusiveSumByKey(ctmp2, tb1, G2, io, within, (int)m, cub::Equality(), st);
            cudaMemsetAsync(gcnt, 0, 4 * (ng + 1), st);
            k_adel_gcount<<<gm, 256, 0, st>>>(G2, io, m, gcnt);
            tb1 = tt;
            cub::DeviceScan::ExclusiveSum(ctmp2, tb1, gcnt, cnt, (int)ng + 1, st);   // cnt = group begin
            k_adel_rng<<<grid_for(ng, 256), 256, 0, st>>>(cnt, ng, (int2 *)t->nl_rng);
            cudaMemsetAsync(t->nl_cost, 0, 4 * ng, st);
            k_adel_fill<<<gm, 256, 0, st>>>(t->sa, t->listA_idx, t->offA, n_orb, m, G2, J2, within, cnt, DV2, rbv, rev,
                                            t->thr_single, (int4 *)t->nl, t->nl_cost);
            cudaFreeAsync(w, st);
            cudaFreeAsync(cnt, st);
        } else {
            cudaMemsetAsync(cursor, 0, 8, st);
            TabSpin tv{};
            tv.sa = t->sa; tv.listA_idx = t->listA_idx; tv.offA = t->offA;
            tv.ah_keys = t->ah_keys; tv.ah_vals = t->ah_vals; tv.ah_mask = t->ah_mask;
            const int gw = (int)std::min<int64_t>((ng + NL_WARPS - 1) / NL_WARPS, 148 * 48);
            k_nl<<<std::max(gw, 1), 32 * NL_WARPS, 0, st>>>(tv, n_orb, ng, (int2 *)t->nl_rng, (int4 *)t->nl, cursor,
                                                            t->thr_single, t->nl_cost);
        }
    }
    // deletion multimap for heavy groups (sorted CSR + unique-key hash)
    rc = build_multimap(t, n, st, flags, ctmp, tmp);
    if (rc) { cudaFreeAsync(scratch, st); return rc; }
    t->thr_rowheavy = t->opt.thr_rowheavy;
    if (t->thr_rowheavy < t->thr_single) t->thr_rowheavy = t->thr_single;   // rows must be in the multimap
    {
        // heavy alpha groups (more than thr_rowheavy rows) in ascending id order, written
        // on the device: one read of their count (at most n / (thr_rowheavy + 1) of them)
        int *cnt_d = (int *)incl;   // scratch reuse
        const int cap = (int)std::min<int64_t>(t->n_alpha_groups, n / ((int64_t)t->thr_rowheavy + 1) + 1);
        rc = cuda_check(nnqs_malloc_async((void **)&t->heavy_groups, 4 * (size_t)std::max(cap, 1), st), "alloc heavy");
        if (rc) { cudaFreeAsync(scratch, st); return rc; }
        const HeavyGroup pred{t->offA, t->thr_rowheavy};
        const int ng = (int)t->n_alpha_groups;
        size_t tsel = 0;
        cub::DeviceSelect::If(nullptr, tsel, thrust::counting_iterator<int32_t>(0), t->heavy_groups, cnt_d, ng, pred, st);
        void *tmp_sel = nullptr;
        rc = cuda_check(nnqs_malloc_async(&tmp_sel, std::max<size_t>(tsel, 16), st), "alloc heavy select");
        if (rc) { cudaFreeAsync(scratch, st); return rc; }
        cub::DeviceSelect::If(tmp_sel, tsel, thrust::counting_iterator<int32_t>(0), t->heavy_groups, cnt_d, ng, pred,
                              st);
        cudaFreeAsync(tmp_sel, st);
        int nh = 0;
        rc = cuda_check(cudaMemcpyAsync(&nh, cnt_d, sizeof(int), cudaMemcpyDeviceToHost, st), "read heavy");
        if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
        if (rc) { cudaFreeAsync(scratch, st); return rc; }
        if (nh > cap) { cudaFreeAsync(scratch, st); return nnqs_set_error(NNQS_E_TABLE, "internal: heavy group bound"); }
        t->n_heavy = nh;
    }
    cudaFreeAsync(scratch, st);
    rc = cuda_check(cudaGetLastError(), "spin index kernels");
    if (rc) return rc;
    t->spin_ready = true;
    return NNQS_OK;
}

void nnqs_table_release_spin(nnqs_table t) {
    if (t->spin_buf) cudaFreeAsync(t->spin_buf, (cudaStream_t)t->stream);
    if (t->mm_buf) cudaFreeAsync(t->mm_buf, (cudaStream_t)t->stream);
    if (t->heavy_groups) cudaFreeAsync(t->heavy_groups, (cudaStream_t)t->stream);
    if (t->nl_buf) cudaFreeAsync(t->nl_buf, (cudaStream_t)t->stream);
    t->nl_rng = nullptr;
    t->nl_cost = nullptr;
    t->nl = t->nl_buf = nullptr;
    t->heavy_groups = nullptr;
    t->n_heavy = 0;
    t->mm = t->mm_buf = nullptr;
    t->spin_buf = nullptr;
    t->spin_ready = false;
}

int nnqs_chunk_work_spin(nnqs_table t, int64_t chunk, int64_t *work_host, int64_t *floor_host, void *stream) {
    const int64_t nch = (t->n + chunk - 1) / chunk;
    if (nch == 0) return NNQS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // estimate weights: base per row, probed list, join row,
    // probed x probed product, latency floor
    const int w0 = 256, pd = 4096, pj = 4096, px = 0, pf = 32768;
    TabSpin tv{};
    tv.n = t->n;
    tv.ga_of = t->ga_of;
    tv.gb_of = t->gb_of;
    tv.offA = t->offA;
    tv.offB = t->offB;
    long long *wd = nullptr;
    int rc = cuda_check(nnqs_malloc_async((void **)&wd, 16 * nch, st), "alloc chunk work");
    if (rc) return rc;
    k_chunk_work<<<(unsigned)nch, 256, 0, st>>>(tv, chunk, t->thr_double, t->thr_rowheavy, t->nl_cost, w0, pd, pj, px,
                                                pf, wd, wd + nch);
    rc = cuda_check(cudaMemcpyAsync(work_host, wd, 8 * nch, cudaMemcpyDeviceToHost, st), "read chunk work");
    if (!rc && floor_host)
        rc = cuda_check(cudaMemcpyAsync(floor_host, wd + nch, 8 * nch, cudaMemcpyDeviceToHost, st), "read chunk floor");
    cudaFreeAsync(wd, st);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync chunk work");
    return rc;
}

int nnqs_launch_local_energy_spin(nnqs_ham h, nnqs_table t, int64_t row_begin, int64_t n_rows, double *eloc,
                                  int64_t *stats, const ChunkSink &cs, const HitLogHost &lg, void *stream) {
    const SpinIndex &S = h->spin;
    const DeviceHam &D = h->dev;
    SpinView sv{S.n, S.P, D.pair_k[0], D.pair_k[1], D.quad_k[0], D.quad_k[1], D.ab_k, D.ab_rec ? D.ab_rec : D.ab_k,
                D.quad_rec[0] ? D.quad_rec[0] : D.quad_k[0], D.quad_rec[1] ? D.quad_rec[1] : D.quad_k[1],
                S.diag_k,
                h->host.n_qubits, S.occ_ok ? D.occ_rec : nullptr, S.diag_K, S.diag_ok ? D.diag_uv : nullptr,
                (S.ab_ok && NNQS_AB) ? D.ab_d : nullptr, D.ab_bits, S.ab_w, (const ulonglong2 *)D.pair_J};
    GroupView gv{(const uint2 *)D.frng, (const ulonglong2 *)D.frec};   // in-sector folded strings
    TabSpin tv{t->n, (const ulonglong2 *)t->keys, (const double2 *)t->logpsi, (const double2 *)t->psi_hat,
               t->slots, t->bucket_mask, t->shift_key, t->sa, t->sb, t->ga_of, t->gb_of, t->offA, t->offB,
               t->listA_b, t->listB_a, t->listA_idx, t->listB_idx, t->ah_keys, t->ah_vals, t->ah_mask,
               (const ulonglong2 *)t->mm, t->mm_mask, t->mm_bloom, t->mm_bloom_mask,
               (const ulonglong2 *)t->mm_ent, (const int2 *)t->nl_rng, (const int4 *)t->nl, t->thr_single,
               t->thr_double, t->uniform_pc ? 1 : 0, HitLog{lg.count, lg.cap, lg.row, lg.idx, lg.h}};
    cudaStream_t st = (cudaStream_t)stream;
    int rc = ensure_hs(h->device);
    if (rc) return rc;
    // stats[0] = row-group pairs resolved (the literal loop's R * K', by definition)
    const unsigned long long pairs = (unsigned long long)n_rows * (unsigned long long)h->n_groups;
    constexpr int phase_mask = NNQS_PHASE_MASK;
    const bool do_hj = t->n_heavy > 0 && (phase_mask & 8);
    const int64_t row_end = row_begin + n_rows;
    // Streams: st (caller) runs the diagonal + phase (i) and the phase (iii) kernel;
    // hs (table-owned) the entry-driven join of the heavy alpha groups; s2 (table-owned)
    // phase (ii), concurrently with phase (i).  Both start after everything queued on st
    // so far and are joined back into st by events before phase (iii).
    cudaStream_t hs = (cudaStream_t)t->own[1], s2 = (cudaStream_t)t->own[2];
    // every buffer and event of the call; released on every exit path (stream-ordered)
    double2 *acc_heavy = nullptr, *partial = nullptr;
    unsigned long long *hcnt = nullptr, *ctr = nullptr;
    u64 *hkeys = nullptr;
    void *pbuf = nullptr;
    cudaEvent_t ev_start = nullptr, ev_hj = nullptr, ev_p2 = nullptr;
    auto cleanup = [&](int code) -> int {
        if (hkeys) cudaFreeAsync(hkeys, hs);
        if (pbuf) cudaFreeAsync(pbuf, st);
        if (ctr) cudaFreeAsync(ctr, st);
        if (partial) cudaFreeAsync(partial, st);
        if (acc_heavy) cudaFreeAsync(acc_heavy, st);
        if (hcnt) cudaFreeAsync(hcnt, st);
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_hj) cudaEventDestroy(ev_hj);
        if (ev_p2) cudaEventDestroy(ev_p2);
        if (code) return code;
        return cuda_check(cudaGetLastError(), "structured local energy launch");
    };
    if (do_hj) {
        rc = cuda_check(nnqs_malloc_async((void **)&acc_heavy, 16 * n_rows + 16, st), "alloc acc_heavy");
        if (!rc) rc = cuda_check(nnqs_malloc_async((void **)&hcnt, 16, st), "alloc hj counter");
        if (rc) return cleanup(rc);
        cudaMemsetAsync(acc_heavy, 0, 16 * n_rows, st);
        cudaMemsetAsync(hcnt, 0, 16, st);
    }
    rc = cuda_check(nnqs_malloc_async((void **)&partial, 32 * n_rows + 32, st), "alloc partial");
    if (rc) return cleanup(rc);
    double2 *partial2 = partial + n_rows + 1;
    // longest-first row orders for the three row kernels (work estimates, one
    // descending sort each); results do not depend on the order
    int32_t *perm3 = nullptr, *perm20 = nullptr, *perm24 = nullptr;
    if (t->nl_cost) {
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n_rows, 0,
                                                  32, st);
        const size_t nb = ((size_t)4 * n_rows + 255) & ~size_t(255);
        rc = cuda_check(nnqs_malloc_async(&pbuf, 8 * nb + tb + 256, st), "alloc row orders");
        if (rc) return cleanup(rc);
        char *pp = (char *)pbuf;
        uint32_t *c3 = (uint32_t *)pp, *c20 = (uint32_t *)(pp + nb), *c24 = (uint32_t *)(pp + 2 * nb);
        int32_t *io = (int32_t *)(pp + 3 * nb);
        perm3 = (int32_t *)(pp + 4 * nb);
        perm20 = (int32_t *)(pp + 5 * nb);
        perm24 = (int32_t *)(pp + 6 * nb);
        uint32_t *ks = (uint32_t *)(pp + 7 * nb);
        void *tmp = pp + 8 * nb;
        k_row_cost<<<grid_for(n_rows, 256), 256, 0, st>>>(tv, row_begin, n_rows, t->thr_double, t->thr_rowheavy,
                                                         t->nl_cost, c3, c20, c24, io);
        uint32_t *cs3[3] = {c3, c20, c24};
        int32_t *ps[3] = {perm3, perm20, perm24};
        for (int k = 0; k < 3; ++k) {
            size_t tb1 = tb;
            cub::DeviceRadixSort::SortPairsDescending(tmp, tb1, cs3[k], ks, io, ps[k], (int)n_rows, 0, 32, st);
        }
    }
    rc = cuda_check(nnqs_malloc_async((void **)&ctr, 128, st), "alloc row counters");
    if (rc) return cleanup(rc);
    cudaMemsetAsync(ctr, 0, 128, st);   // [0, 6): the row kernels' row counters
    rc = cuda_check(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_check(cudaEventCreateWithFlags(&ev_hj, cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_check(cudaEventCreateWithFlags(&ev_p2, cudaEventDisableTiming), "event");
    if (rc) return cleanup(rc);
    cudaEventRecord(ev_start, st);        // s2 and hs start after everything queued on st
    cudaStreamWaitEvent(s2, ev_start, 0);
    cudaStreamWaitEvent(hs, ev_start, 0);
    int nl = 0;
    auto launch = [&](auto kern, const int32_t *perm, cudaStream_t ks) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        const int gg = std::max(1, per_sm) * 148;   // persistent grid, rows from the counter
        kern<<<gg, 256, 0, ks>>>(sv, gv, tv, row_begin, n_rows, (double2 *)eloc, (unsigned long long *)stats, pairs,
                                 phase_mask, acc_heavy, t->thr_rowheavy, partial, ctr + nl, perm, partial2, cs);
        ++nl;
    };
    // three launches, each a smaller kernel (instruction cache): diagonal + phase (i)
    // -> partial; phase (ii) (s2, concurrent) -> partial2; phase (iii) starts from
    // partial + partial2 and finalises (fused chunk partials of Eq. (6) included)
    // the parity hit log (nnqs_coupled_debug_rows) has instantiations of its own, so
    // the production kernels carry none of its code
    const bool lg_on = lg.count != nullptr;
    if (lg_on) {
        launch(k_eloc_spin<3, 4, false, true>, perm3, st);
        launch(k_eloc_spin<20, 4, false, true>, perm20, s2);
    } else {
        launch(k_eloc_spin<3, 4, false, false>, perm3, st);
        launch(k_eloc_spin<20, 4, false, false>, perm20, s2);
    }
    if (t->n_direct) {
        if (lg_on) {
            launch(k_eloc_spin<3, 4, true, true>, perm3, st);
            launch(k_eloc_spin<20, 4, true, true>, perm20, s2);
        } else {
            launch(k_eloc_spin<3, 4, true, false>, perm3, st);
            launch(k_eloc_spin<20, 4, true, false>, perm20, s2);
        }
    }
    cudaEventRecord(ev_p2, s2);
    cudaStreamWaitEvent(st, ev_p2, 0);
    if (do_hj) {
        // entry-driven join (phase (iii) of the rows of very heavy alpha groups) on hs
        int ibits = 1, rbits = 1;
        while ((1LL << ibits) < t->n) ++ibits;
        while ((1LL << rbits) < n_rows) ++rbits;
        int kbits = 1;
        while ((1LL << kbits) < h->n_groups) ++kbits;
        if (rbits + ibits + kbits > 64) kbits = 0;   // no room: k is recomputed from the strings
        constexpr int hj_gx = 1184, hj_ev = 8;       // grid shapes (measured)
        const dim3 hgrid(hj_gx, t->n_heavy);
        const int clip = (int)(row_begin > 0 || row_end < t->n);   // keep only this slice's rows
        int64_t cap = std::max<int64_t>(1 << 20, std::min<int64_t>((int64_t)1 << 26, 64 * n_rows));
        for (int attempt = 0; attempt < 2 && !rc; ++attempt) {
            size_t tb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, (const u64 *)nullptr, (u64 *)nullptr, (int)cap, kbits,
                                           kbits + ibits + rbits, hs);
            rc = cuda_check(nnqs_malloc_async((void **)&hkeys, 16 * cap + tb + 8 * n_rows + 1024, hs), "alloc hj keys");
            if (rc) break;
            cudaMemsetAsync(hcnt, 0, 8, hs);
            k_hj_emit<<<hgrid, 256, 0, hs>>>(sv, tv, t->heavy_groups, t->n_heavy, row_begin, row_end, clip, ibits,
                                             kbits, hcnt, hkeys, cap, attempt == 0 ? (unsigned long long *)stats : nullptr);
            unsigned long long m = 0;
            rc = cuda_check(cudaMemcpyAsync(&m, hcnt, 8, cudaMemcpyDeviceToHost, hs), "read hj count");
            if (!rc) rc = cuda_check(cudaStreamSynchronize(hs), "sync");
            if (rc) break;
            if ((int64_t)m > cap) {              // buffer too small: size exactly and redo
                if (m >= (1ULL << 31)) { rc = nnqs_set_error(NNQS_E_SIZE, "entry-driven join larger than 2^31 hits"); break; }
                cudaFreeAsync(hkeys, hs);
                hkeys = nullptr;
                cap = (int64_t)m;
                continue;
            }
            if (m) {
                u64 *k2 = hkeys + cap;
                int32_t *kb = (int32_t *)(hkeys + 2 * cap), *ke = kb + n_rows;
                void *htmp = (void *)(((uintptr_t)(ke + n_rows) + 511) & ~(uintptr_t)255);   // 256-B aligned
                cudaMemsetAsync(kb, 0, 8 * n_rows, hs);
                tb = 0;
                // order by (row, x' index) only: the group id rides along in the low bits
                cub::DeviceRadixSort::SortKeys(nullptr, tb, (const u64 *)nullptr, (u64 *)nullptr, (int)m, kbits,
                                               kbits + ibits + rbits, hs);
                cub::DeviceRadixSort::SortKeys(htmp, tb, hkeys, k2, (int)m, kbits, kbits + ibits + rbits, hs);
                k_hj_bounds<<<grid_for((int64_t)m, 256), 256, 0, hs>>>(k2, (int64_t)m, ibits + kbits, kb, ke);
                auto hj_eval = lg_on ? k_hj_eval<true> : k_hj_eval<false>;
                hj_eval<<<148 * hj_ev, 256, 0, hs>>>(sv, gv, tv, t->heavy_groups, t->n_heavy, row_begin, row_end, k2,
                                                   ibits, kbits, kb, ke, acc_heavy, (unsigned long long *)stats);
            }
            break;
        }
    }
    if (do_hj) {
        cudaEventRecord(ev_hj, hs);
        cudaStreamWaitEvent(st, ev_hj, 0);
    }
    if (!rc) {
        if (lg_on) {
            launch(k_eloc_spin<24, NNQS_P3_MINB, false, true>, perm24, st);
            if (t->n_direct) launch(k_eloc_spin<24, NNQS_P3_MINB, true, true>, perm24, st);
        } else {
            launch(k_eloc_spin<24, NNQS_P3_MINB, false, false>, perm24, st);
            if (t->n_direct) launch(k_eloc_spin<24, NNQS_P3_MINB, true, false>, perm24, st);
        }
    }
    return cleanup(rc);
}

int nnqs_debug_counters(uint64_t *out, int reset) {
    if (!out) return nnqs_set_error(NNQS_E_ARG, "nnqs_debug_counters: null out");
    for (int i = 0; i < 16; ++i) out[i] = 0;
#ifdef NNQS_PROFILE
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 16);
    if (e == cudaSuccess && reset) {
        unsigned long long z[16] = {0};
        e = cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
#else
    (void)reset;
#endif
    return NNQS_OK;
}
