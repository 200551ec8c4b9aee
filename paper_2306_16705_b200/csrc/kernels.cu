// kernels.cu -- device side of libnnqs (sm_100a).
//
//   table build      id_lut / wf_lut of Algorithm 2: order check,
//                    psi_hat = exp(logpsi - s), GF(2)-linear hash index
//   local energy     Eq. (4) over the grouped table of Fig. 6(c),
//                    fused entry evaluation + sample-aware lookup
//                    (PAPER.md:379-381); Algorithm 2
//   energy reduce    Eq. (6) with counts
#include <cuda_runtime.h>

#include <mutex>

#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

#define NNQS_EMPTY_SLOT 0xFFFFFFFFFFFFFFFFULL
#define ALPHA_MASK 0x5555555555555555ULL
#define BETA_MASK 0xAAAAAAAAAAAAAAAAULL

__constant__ u64 c_hash[128];
__constant__ uint32_t c_filt[128];

namespace {

std::mutex g_hash_ready_mu;
bool g_hash_ready[64] = {false};

// the hash columns in constant memory of `device` (the current device), once per device
int ensure_hash(int device) {
    if (device < 0 || device >= 64) return NNQS_E_ARG;
    std::lock_guard<std::mutex> lk(g_hash_ready_mu);
    if (g_hash_ready[device]) return NNQS_OK;
    u64 cols[128];
    nnqs_hash_columns(cols);
    cudaError_t e = cudaMemcpyToSymbol(c_hash, cols, sizeof(cols));
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    uint32_t fcols[128];
    nnqs_filter_columns(fcols);
    e = cudaMemcpyToSymbol(c_filt, fcols, sizeof(fcols));
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    g_hash_ready[device] = true;
    return NNQS_OK;
}

inline int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return NNQS_OK;
    return nnqs_set_error(e == cudaErrorMemoryAllocation ? NNQS_E_NOMEM : NNQS_E_CUDA,
                          std::string(what) + ": " + cudaGetErrorString(e));
}

struct HamView {
    const ulonglong2 *gx;
    const u64 *ghx;
    const uint32_t *ginfo;
    const uint32_t *goff;
    const ulonglong2 *tz;
    const double *td;
    int64_t K;
};

struct TabView {
    int64_t n;
    const ulonglong2 *keys;
    const double2 *logpsi;
    const double2 *psi_hat;
    const u64 *slots;
    u64 bucket_mask;
    const u64 *shift_key;
};

HamView ham_view(nnqs_ham h) {
    return {(const ulonglong2 *)h->dev.gx, h->dev.ghx, h->dev.ginfo, h->dev.goff,
            (const ulonglong2 *)h->dev.tz, h->dev.td, h->n_groups};
}

TabView tab_view(nnqs_table t) {
    return {t->n, (const ulonglong2 *)t->keys, (const double2 *)t->logpsi,
            (const double2 *)t->psi_hat, t->slots, t->bucket_mask, t->shift_key};
}

// ------------------------------------------------------------ device helpers
__device__ __forceinline__ u64 hash128(u64 lo, u64 hi) {
    u64 h = 0;
    while (lo) {
        h ^= c_hash[__ffsll((long long)lo) - 1];
        lo &= lo - 1;
    }
    while (hi) {
        h ^= c_hash[64 + __ffsll((long long)hi) - 1];
        hi &= hi - 1;
    }
    return h;
}

// order-preserving map double -> u64 (for atomicMax)
__device__ __forceinline__ u64 dkey(double v) {
    u64 b = (u64)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(u64 k) {
    if (k == 0) return 0.0;                       // no finite entry
    u64 b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double((long long)b);
}

// bucketised linear probing: 4 slots (32 B) per bucket, slot = fp32 << 32 | rank
__device__ __forceinline__ int64_t probe(const TabView &T, u64 h, u64 p0, u64 p1) {
    u64 b = h & T.bucket_mask;
    const uint32_t fp = (uint32_t)(h >> 32);
    while (true) {
        const ulonglong2 *bk = reinterpret_cast<const ulonglong2 *>(T.slots + 4 * b);
        const ulonglong2 s01 = __ldg(bk), s23 = __ldg(bk + 1);
        const u64 s[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (s[i] == NNQS_EMPTY_SLOT) return -1;
            if ((uint32_t)(s[i] >> 32) == fp) {
                const uint32_t r = (uint32_t)s[i];
                const ulonglong2 k = __ldg(T.keys + r);
                if (k.x == p0 && k.y == p1) return (int64_t)r;
            }
        }
        b = (b + 1) & T.bucket_mask;
    }
}

__device__ __forceinline__ double flip_sign(double d, int parity) {
    return __longlong_as_double(__double_as_longlong(d) ^ ((long long)parity << 63));
}

// H_{x', x} = sum_{i in group k} d_i (-1)^{popc(x & Z_i)}   (reading R1/R2)
__device__ __forceinline__ double group_value(const HamView &H, int64_t k, u64 x0, u64 x1,
                                              u64 &n_str) {
    const uint32_t b = __ldg(H.goff + k), e = __ldg(H.goff + k + 1);
    double hv = 0.0;
    for (uint32_t i = b; i < e; ++i) {
        const ulonglong2 Z = __ldg(H.tz + i);
        const int par = (__popcll(x0 & Z.x) + __popcll(x1 & Z.y)) & 1;
        hv += flip_sign(__ldg(H.td + i), par);
    }
    n_str += e - b;
    return hv;
}

// ------------------------------------------------------------ table build
__global__ void k_check_order(const ulonglong2 *keys, int64_t n, int *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 a = keys[i - 1], b = keys[i];
        if (!(a.y < b.y || (a.y == b.y && a.x < b.x))) atomicOr(flag, 1);
    }
}

__global__ void k_max_re(const double2 *lp, int64_t n, u64 *shift_key) {
    u64 m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = lp[i].x;
        if (isfinite(v)) m = max(m, dkey(v));
    }
    for (int o = 16; o; o >>= 1) m = max(m, (u64)__shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax((unsigned long long *)shift_key, (unsigned long long)m);
}

__global__ void k_psi_hat(const double2 *lp, int64_t n, const u64 *shift_key, double2 *ph, int *n_direct) {
    const double s = dkey_inv(*shift_key);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 l = lp[i];
        if (l.x > -INFINITY && l.x - s < -600.0) atomicAdd(n_direct, 1);   // rows on the exp-ratio path (R11)
        const double m = exp(l.x - s);
        double sn, cs;
        sincos(l.y, &sn, &cs);
        ph[i] = make_double2(m * cs, m * sn);
    }
}

__global__ void k_hash_insert(const ulonglong2 *keys, int64_t n, u64 *slots, u64 mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 k = keys[i];
        const u64 h = hash128(k.x, k.y);
        const u64 val = ((h >> 32) << 32) | (u64)(uint32_t)i;
        u64 b = h & mask;
        bool done = false;
        while (!done) {
            for (int s = 0; s < 4 && !done; ++s) {
                const u64 old = atomicCAS((unsigned long long *)(slots + 4 * b + s),
                                          (unsigned long long)NNQS_EMPTY_SLOT, (unsigned long long)val);
                done = old == NNQS_EMPTY_SLOT;
            }
            b = (b + 1) & mask;
        }
    }
}

// ------------------------------------------------------------ local energy
// v1: one thread per row, grid-stride over rows, groups in
// ascending order, per-row accumulation order = ascending k.
template <int MODE, bool CONS>
__global__ void __launch_bounds__(256) k_eloc_v1(HamView H, TabView T, int64_t row_begin,
                                                 const ulonglong2 *rows, const double2 *row_lp,
                                                 int64_t n_rows, double2 *out,
                                                 unsigned long long *stats, ChunkSink cs) {
    const double s = dkey_inv(*T.shift_key);
    u64 c_pairs = 0, c_sec = 0, c_hit = 0, c_str = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        u64 x0, x1;
        double2 lx;
        if (rows) {
            const ulonglong2 k = rows[r];
            x0 = k.x; x1 = k.y;
            lx = row_lp[r];
        } else {
            const int64_t i = row_begin + r;
            if (MODE == 0) {
                const ulonglong2 k = T.keys[i];
                x0 = k.x; x1 = k.y;
            } else {
                x0 = (u64)i; x1 = 0;
            }
            lx = T.logpsi[i];
        }
        if (!(lx.x > -INFINITY)) {                 // psi(x) = 0: 0/0 (reading R10)
            out[r] = make_double2(NAN, NAN);
            chunk_done_thread(cs, out, r, n_rows);
            continue;
        }
        const double rel = lx.x - s;
        const bool direct = rel < -600.0;          // reading R11 fallback
        const u64 hx = (MODE == 0) ? hash128(x0, x1) : 0;
        double ar = 0.0, ai = 0.0;
        for (int64_t k = 0; k < H.K; ++k) {
            const ulonglong2 X = __ldg(H.gx + k);
            if (CONS) {
                const uint32_t info = __ldg(H.ginfo + k);
                const int na = __popcll(x0 & X.x & ALPHA_MASK) + __popcll(x1 & X.y & ALPHA_MASK);
                const int nb = __popcll(x0 & X.x & BETA_MASK) + __popcll(x1 & X.y & BETA_MASK);
                if (na != (int)(info & 0xff) || nb != (int)((info >> 8) & 0xff)) continue;
            }
            ++c_sec;
            const u64 p0 = x0 ^ X.x, p1 = x1 ^ X.y;
            int64_t idx;
            if (MODE == 1) idx = (p1 == 0 && p0 < (u64)T.n) ? (int64_t)p0 : -1;
            else idx = probe(T, hx ^ __ldg(H.ghx + k), p0, p1);
            if (idx < 0) continue;
            ++c_hit;
            const double hv = group_value(H, k, x0, x1, c_str);
            double2 ps;
            if (!direct) {
                ps = __ldg(T.psi_hat + idx);
            } else {
                const double2 l = T.logpsi[idx];
                const double m = exp(l.x - lx.x);
                double sn, cs;
                sincos(l.y - lx.y, &sn, &cs);
                ps = make_double2(m * cs, m * sn);
            }
            ar = fma(hv, ps.x, ar);
            ai = fma(hv, ps.y, ai);
        }
        c_pairs += (u64)H.K;
        double2 e;
        if (direct) {
            e = make_double2(ar, ai);
        } else {
            // E = acc / psi_hat(x) = acc * exp(-(logpsi(x) - s))
            const double m = exp(-rel);
            double sn, cs;
            sincos(-lx.y, &sn, &cs);
            const double ir = m * cs, ii = m * sn;
            e = make_double2(ar * ir - ai * ii, ar * ii + ai * ir);
        }
        out[r] = e;
        chunk_done_thread(cs, out, r, n_rows);   // fused first pass of Eq. (6)
    }
    if (stats) {
        for (int o = 16; o; o >>= 1) {
            c_pairs += __shfl_xor_sync(0xffffffffu, c_pairs, o);
            c_sec += __shfl_xor_sync(0xffffffffu, c_sec, o);
            c_hit += __shfl_xor_sync(0xffffffffu, c_hit, o);
            c_str += __shfl_xor_sync(0xffffffffu, c_str, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(stats + 0, c_pairs);
            atomicAdd(stats + 1, c_sec);
            atomicAdd(stats + 2, c_hit);
            atomicAdd(stats + 3, c_str);
        }
    }
}

// ------------------------------------------ literal Algorithm 2, staged (v2)
// The same loop as k_eloc_v1 (every row x every group, ascending k; sector
// test, lookup, string sum on a hit) with the group table
// streamed through shared memory: 32-B records {X, h(X), sector info} in tiles of
// LIT_TILE groups, fetched by the bulk-copy engine (cp.async.bulk + mbarrier,
// LIT_STAGES deep) while the CTA works on the previous tiles, each tile read by
// the LIT_THREADS rows of the CTA (one row per thread; one tile load per 1024
// rows instead of one broadcast load per warp and group).  Hits are applied in
// ascending k, so a row's sum is bit-identical to k_eloc_v1's.
#define LIT_THREADS 512
#define LIT_TILE 1024
#define LIT_STAGES 4

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct LitRec {
    ulonglong2 x;      // flip mask X_k
    u64 hx;            // h(X_k)
    uint32_t info;     // popc(X & alpha) / 2 | popc(X & beta) / 2 << 8 | odd << 16
    uint32_t pad;
};

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MODE, bool CONS>
__global__ void __launch_bounds__(LIT_THREADS, 1) k_eloc_lit(HamView H, const LitRec *rec, TabView T,
                                                             int64_t row_begin, const ulonglong2 *rows,
                                                             const double2 *row_lp, int64_t n_rows, double2 *out,
                                                             unsigned long long *stats, ChunkSink cs) {
    extern __shared__ __align__(128) unsigned char lit_smem[];
    LitRec *tile = reinterpret_cast<LitRec *>(lit_smem);                    // [LIT_STAGES][LIT_TILE]
    __shared__ __align__(8) unsigned long long full[LIT_STAGES], empty[LIT_STAGES];
    const int kWarps = blockDim.x / 32;           // blockDim: a multiple of 32, <= LIT_THREADS
    const double s = dkey_inv(*T.shift_key);
    const int64_t K = H.K;
    const int64_t n_tiles = (K + LIT_TILE - 1) / LIT_TILE;
    const int lane = threadIdx.x & 31;
    u64 c_pairs = 0, c_sec = 0, c_hit = 0, c_str = 0;
    // every row block of this CTA streams the whole table: one continuous ring of
    // tiles (global tile counter q = block * n_tiles + t, stage q % S, phase q / S)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t first = (int64_t)blockIdx.x * blockDim.x;
    const int64_t n_blocks = first < n_rows ? (n_rows - first + stride - 1) / stride : 0;
    const int64_t q_end = n_blocks * n_tiles;
    auto issue = [&](int64_t q) {                 // producer: tile q % n_tiles into stage q % S
        const int st = (int)(q % LIT_STAGES);
        const int64_t g0 = (q % n_tiles) * LIT_TILE;
        const unsigned bytes = (unsigned)(min((int64_t)LIT_TILE, K - g0) * (int64_t)sizeof(LitRec));
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(tile + st * LIT_TILE, rec + g0, bytes, &full[st]);
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < LIT_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int64_t q = 0; q < LIT_STAGES && q < q_end; ++q) issue(q);
    int64_t q = 0;
    for (int64_t blk = 0; blk < n_blocks; ++blk) {
        const int64_t r = first + blk * stride + threadIdx.x;
        u64 x0 = 0, x1 = 0;
        double2 lx = make_double2(-INFINITY, 0.0);
        if (r < n_rows) {
            if (rows) {
                const ulonglong2 k = rows[r];
                x0 = k.x;
                x1 = k.y;
                lx = row_lp[r];
            } else {
                const int64_t i = row_begin + r;
                if (MODE == 0) {
                    const ulonglong2 k = T.keys[i];
                    x0 = k.x;
                    x1 = k.y;
                } else {
                    x0 = (u64)i;
                }
                lx = T.logpsi[i];
            }
        }
        const bool live = lx.x > -INFINITY;      // psi(x) = 0 (reading R10) or past the end: no pairs
        const bool direct = (lx.x - s) < -600.0;
        const u64 hx = (MODE == 0 && live) ? hash128(x0, x1) : 0;
        double ar = 0.0, ai = 0.0;
        for (int64_t t = 0; t < n_tiles; ++t, ++q) {
            const int st = (int)(q % LIT_STAGES);
            const unsigned ph = (unsigned)((q / LIT_STAGES) & 1);
            mbar_wait(&full[st], ph);
            const LitRec *tl = tile + st * LIT_TILE;
            const int gn = live ? (int)min((int64_t)LIT_TILE, K - t * LIT_TILE) : 0;
            for (int g = 0; g < gn; ++g) {
                const LitRec R = tl[g];
                if (CONS) {
                    const int na = __popcll(x0 & R.x.x & ALPHA_MASK) + __popcll(x1 & R.x.y & ALPHA_MASK);
                    const int nb = __popcll(x0 & R.x.x & BETA_MASK) + __popcll(x1 & R.x.y & BETA_MASK);
                    if (na != (int)(R.info & 0xff) || nb != (int)((R.info >> 8) & 0xff)) continue;
                }
                ++c_sec;
                const u64 p0 = x0 ^ R.x.x, p1 = x1 ^ R.x.y;
                int64_t idx;
                if (MODE == 1) idx = (p1 == 0 && p0 < (u64)T.n) ? (int64_t)p0 : -1;
                else idx = probe(T, hx ^ R.hx, p0, p1);
                if (idx < 0) continue;
                ++c_hit;
                const double hv = group_value(H, t * LIT_TILE + g, x0, x1, c_str);
                double2 ps;
                if (!direct) {
                    ps = __ldg(T.psi_hat + idx);
                } else {
                    const double2 l = T.logpsi[idx];
                    const double m = exp(l.x - lx.x);
                    double sn, cs2;
                    sincos(l.y - lx.y, &sn, &cs2);
                    ps = make_double2(m * cs2, m * sn);
                }
                ar = fma(hv, ps.x, ar);
                ai = fma(hv, ps.y, ai);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);   // this warp is done with stage st
            if (threadIdx.x == 0 && q + LIT_STAGES < q_end) {
                mbar_wait(&empty[st], ph);            // every warp released it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(q + LIT_STAGES);
            }
        }
        if (r < n_rows) {
            double2 e;
            if (!live) {
                e = make_double2(NAN, NAN);
            } else if (direct) {
                e = make_double2(ar, ai);
            } else {
                // E = acc / psi_hat(x) = acc * exp(-(logpsi(x) - s))
                const double m = exp(-(lx.x - s));
                double sn, cs2;
                sincos(-lx.y, &sn, &cs2);
                const double ir = m * cs2, ii = m * sn;
                e = make_double2(ar * ir - ai * ii, ar * ii + ai * ir);
            }
            if (live) c_pairs += (u64)K;
            out[r] = e;
            chunk_done_thread(cs, out, r, n_rows);
        }
    }
    if (stats) {
        for (int o = 16; o; o >>= 1) {
            c_pairs += __shfl_xor_sync(0xffffffffu, c_pairs, o);
            c_sec += __shfl_xor_sync(0xffffffffu, c_sec, o);
            c_hit += __shfl_xor_sync(0xffffffffu, c_hit, o);
            c_str += __shfl_xor_sync(0xffffffffu, c_str, o);
        }
        if (lane == 0) {
            atomicAdd(stats + 0, c_pairs);
            atomicAdd(stats + 1, c_sec);
            atomicAdd(stats + 2, c_hit);
            atomicAdd(stats + 3, c_str);
        }
    }
}

// ------------------------------ literal Algorithm 2, bit-sliced over rows (v3)
// The same loop again -- every row x every group, ascending k; sector test,
// lookup, string sum on a hit -- with the sector test of 32
// rows x 32 groups done in a few logic instructions.  A warp owns 32 rows and
// keeps them bit-sliced in shared memory (plane p = bit p of the 32 keys, one
// word); lane l takes group k0 + l, whose flip mask X_k has at most four bits
// for a number-conserving H (Eq. 9: singles and doubles), and forms the 32-row
// mask of rows x with x ^ X_k in x's (N_alpha, N_beta) sector:
//   one pair per spin   bit_i(x) != bit_j(x)        (P_i ^ P_j)
//   a pair per spin     (P_i ^ P_j) & (P_k ^ P_l)
//   a same-spin quad    exactly two of P_i, P_j, P_k, P_l set.
// The in-sector (group, row) pairs of the 32 x 32 block (~16 % at C5) are then
// queued in shared memory in (group, row) order and taken 32 at a time, so every
// lane has a pair and its lookup in flight: a per-spin string filter (f_alpha(x'),
// f_beta(x') in shared-memory bitmaps of the table's alpha and beta strings --
// GF(2)-linear, f(x ^ X) = f(x) ^ f(X); no false negatives), then the hash
// probe of Algorithm 2's lookup, then, on a hit, the string sum.  Each row's
// lane adds its hits in ascending k with the same arithmetic as k_eloc_v1, so
// the result is bit-identical to it.
#ifndef BS_WARPS
#define BS_WARPS 16
#endif
#ifndef BS_TILE
#define BS_TILE 256
#endif
#ifndef BS_STAGES
#define BS_STAGES 3
#endif
#ifndef BS_LF
#define BS_LF 2                                   // lookups in flight per lane
#endif
#ifndef BS_FQ
#define BS_FQ 512                                 // pair-queue entries per warp (a batch has <= 32 x 32 BS_P)
#endif
#ifndef BS_P
#define BS_P 1                                    // 32-row blocks per warp (2 and 4 measured slower)
#endif
#define BS_FB 19                                  // filter bits per spin (2^19-bit bitmaps, 64 KB each)
#define BS_BM_WORDS (2u << (BS_FB - 5))           // both bitmaps, 32-bit words
#define BS_SMEM ((size_t)BS_BM_WORDS * 4 + (size_t)BS_STAGES * BS_TILE * sizeof(BsRec) + BS_WARPS * sizeof(BsWarp))

struct BsRec {
    ulonglong2 x;      // X_k
    u64 hx;            // h(X_k)
    uint32_t fa, fb;   // f_alpha(X_k), f_beta(X_k)
    uint32_t pos;      // flip sites, alpha ones first; 128 = the zero plane, 129 = the ones plane
    uint32_t sb;       // strings [sb, se) of group k
    uint32_t se;       // bit 31: same-spin quad (two-of-four test)
    uint32_t pad;
};

// per-warp shared state of k_eloc_bs (in the dynamic shared memory, after the tile ring)
struct __align__(16) BsWarp {
    ulonglong2 rx[BS_P * 32];   // the warp's rows: key
    uint4 rh[BS_P * 32];        //   h(x) lo, hi, f_alpha(x), f_beta(x)
    double2 rl[BS_P * 32];      //   log psi(x)
    double qh[32];              // hits of one round: H_xx', psi(x')/psi-hat factor, row
    double2 qp[32];
    uint32_t pl[BS_P][132];     // bit planes of the warp's rows (+ zero, ones)
    int32_t qr[32];
    uint16_t fq[BS_FQ];         // in-sector pairs of a batch in (group, row) order: group | row << 8
};

// Algorithm 2's lookup of x' (the probe above) with each 32-B bucket decided from one
// load: the slots whose fingerprint matches are compared with the key; the bucket
// ends the search unless it is full (slots fill in order, so slot 3 tells)
__device__ __forceinline__ int64_t probe_fast(const TabView &T, u64 h, u64 p0, u64 p1) {
    u64 b = h & T.bucket_mask;
    const uint32_t fp = (uint32_t)(h >> 32);
    while (true) {
        const ulonglong2 *bk = reinterpret_cast<const ulonglong2 *>(T.slots + 4 * b);
        const ulonglong2 s01 = __ldg(bk), s23 = __ldg(bk + 1);
        const u64 sl[4] = {s01.x, s01.y, s23.x, s23.y};
        unsigned m = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            m |= (unsigned)((uint32_t)(sl[i] >> 32) == fp && sl[i] != NNQS_EMPTY_SLOT) << i;
        while (m) {
            const int i = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t r = (uint32_t)(i == 0 ? s01.x : i == 1 ? s01.y : i == 2 ? s23.x : s23.y);
            const ulonglong2 k = __ldg(T.keys + r);
            if (k.x == p0 && k.y == p1) return (int64_t)r;
        }
        if (s23.y == NNQS_EMPTY_SLOT) return -1;
        b = (b + 1) & T.bucket_mask;
    }
}

// probe_fast with the first bucket's 32 B already loaded (s01, s23)
__device__ __forceinline__ int64_t probe_resolve(const TabView &T, u64 h, u64 p0, u64 p1, ulonglong2 s01,
                                                 ulonglong2 s23) {
    const uint32_t fp = (uint32_t)(h >> 32);
    const u64 sl[4] = {s01.x, s01.y, s23.x, s23.y};
    unsigned m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) m |= (unsigned)((uint32_t)(sl[i] >> 32) == fp && sl[i] != NNQS_EMPTY_SLOT) << i;
    while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t r = (uint32_t)(i == 0 ? s01.x : i == 1 ? s01.y : i == 2 ? s23.x : s23.y);
        const ulonglong2 k = __ldg(T.keys + r);
        if (k.x == p0 && k.y == p1) return (int64_t)r;
    }
    if (s23.y == NNQS_EMPTY_SLOT) return -1;
    // full bucket: continue with the next one (the same walk as probe_fast)
    const u64 h2 = (h & ~T.bucket_mask) | ((h + 1) & T.bucket_mask);
    return probe_fast(T, h2, p0, p1);
}

__device__ __forceinline__ uint32_t ffilt(u64 w, int base) {
    uint32_t f = 0;
    while (w) {
        f ^= c_filt[base + __ffsll((long long)w) - 1];
        w &= w - 1;
    }
    return f;
}

__device__ __forceinline__ bool bm_test(const uint32_t *bm, uint32_t f) {
    const uint32_t b = f & ((1u << BS_FB) - 1);
    return (bm[b >> 5] >> (b & 31)) & 1u;
}

__global__ void __launch_bounds__(BS_WARPS * 32, 1) k_eloc_bs(HamView H, const BsRec *rec, TabView T,
                                                              const uint32_t *bm, int64_t row_begin,
                                                              const ulonglong2 *rows, const double2 *row_lp,
                                                              int64_t n_rows, double2 *out,
                                                              unsigned long long *stats, ChunkSink cs) {
    constexpr int NP = BS_P;                        // 32-row blocks per warp (one group tile feeds 32 NP rows)
    extern __shared__ __align__(128) unsigned char bs_smem[];
    uint32_t *s_bm = reinterpret_cast<uint32_t *>(bs_smem);                          // [2][2^BS_FB / 32]
    BsRec *tile = reinterpret_cast<BsRec *>(bs_smem + (size_t)BS_BM_WORDS * 4);    // [BS_STAGES][BS_TILE]
    BsWarp *s_w = reinterpret_cast<BsWarp *>(bs_smem + (size_t)BS_BM_WORDS * 4 +
                                             (size_t)BS_STAGES * BS_TILE * sizeof(BsRec));   // [BS_WARPS]
    __shared__ __align__(8) unsigned long long full[BS_STAGES];
    __shared__ unsigned s_done[BS_STAGES];          // warps done with the stage's current tile
    const int kWarps = blockDim.x / 32;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    BsWarp &W = s_w[wid];
    const double s = dkey_inv(*T.shift_key);
    const int64_t K = H.K;
    const int64_t n_tiles = (K + BS_TILE - 1) / BS_TILE;
    u64 c_pairs = 0, c_sec = 0, c_hit = 0, c_str = 0;
    const int64_t per_cta = (int64_t)blockDim.x * NP;
    const int64_t stride = (int64_t)gridDim.x * per_cta;
    const int64_t first = (int64_t)blockIdx.x * per_cta;
    const int64_t n_blocks = first < n_rows ? (n_rows - first + stride - 1) / stride : 0;
    const int64_t q_end = n_blocks * n_tiles;
    auto issue = [&](int64_t q) {
        const int st = (int)(q % BS_STAGES);
        const int64_t g0 = (q % n_tiles) * BS_TILE;
        const unsigned bytes = (unsigned)(min((int64_t)BS_TILE, K - g0) * (int64_t)sizeof(BsRec));
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(tile + st * BS_TILE, rec + g0, bytes, &full[st]);
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < BS_STAGES; ++st) {
            mbar_init(&full[st], 1);
            s_done[st] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t i = threadIdx.x; i < BS_BM_WORDS / 4; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_bm)[i] = __ldg(reinterpret_cast<const uint4 *>(bm) + i);
    if (lane < NP) {
        W.pl[lane][128] = 0u;
        W.pl[lane][129] = ~0u;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int64_t q = 0; q < BS_STAGES && q < q_end; ++q) issue(q);
    const uint32_t *bmA = s_bm, *bmB = s_bm + BS_BM_WORDS / 2;
    int64_t q = 0;
    for (int64_t blk = 0; blk < n_blocks; ++blk) {
        const int64_t r0 = first + blk * stride + (int64_t)wid * 32 * NP;   // the warp's NP x 32 rows
        double2 lx[NP];
        uint32_t live_m[NP];
        __syncwarp();
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int64_t r = r0 + 32 * p + lane;
            u64 x0 = 0, x1 = 0;
            lx[p] = make_double2(-INFINITY, 0.0);
            if (r < n_rows) {
                if (rows) {
                    const ulonglong2 k = rows[r];
                    x0 = k.x;
                    x1 = k.y;
                    lx[p] = row_lp[r];
                } else {
                    const ulonglong2 k = T.keys[row_begin + r];
                    x0 = k.x;
                    x1 = k.y;
                    lx[p] = T.logpsi[row_begin + r];
                }
            }
            const bool live = lx[p].x > -INFINITY;   // psi(x) = 0 (reading R10) or past the end: no pairs
            live_m[p] = __ballot_sync(FULL, live);
            const u64 hx = live ? hash128(x0, x1) : 0;
            const uint32_t fa = live ? ffilt(x0 & ALPHA_MASK, 0) ^ ffilt(x1 & ALPHA_MASK, 64) : 0;
            const uint32_t fb = live ? ffilt(x0 & BETA_MASK, 0) ^ ffilt(x1 & BETA_MASK, 64) : 0;
            W.rx[32 * p + lane] = make_ulonglong2(x0, x1);
            W.rh[32 * p + lane] = make_uint4((uint32_t)hx, (uint32_t)(hx >> 32), fa, fb);
            W.rl[32 * p + lane] = lx[p];
            for (int b = 0; b < 128; ++b) {          // bit planes of the block's rows
                const uint32_t v = __ballot_sync(FULL, ((b < 64 ? x0 >> b : x1 >> (b - 64)) & 1ULL) != 0);
                if (lane == (b & 31)) W.pl[p][b] = v;
            }
        }
        uint32_t any_live = 0;
#pragma unroll
        for (int p = 0; p < NP; ++p) any_live |= live_m[p];
        __syncwarp();
        double ar[NP], ai[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) ar[p] = ai[p] = 0.0;
        for (int64_t t = 0; t < n_tiles; ++t, ++q) {
            const int st = (int)(q % BS_STAGES);
            const unsigned ph = (unsigned)((q / BS_STAGES) & 1);
            mbar_wait(&full[st], ph);
            const BsRec *tl = tile + st * BS_TILE;
            const int gn = any_live ? (int)min((int64_t)BS_TILE, K - t * BS_TILE) : 0;
            for (int g0 = 0; g0 < gn; g0 += 32) {
                // lane = group g0 + lane: the in-sector masks of the NP row blocks
                uint32_t m[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) m[p] = 0;
                if (g0 + lane < gn) {
                    const uint32_t pos = tl[g0 + lane].pos, se = tl[g0 + lane].se;
                    const uint32_t i0 = pos & 0xff, i1 = (pos >> 8) & 0xff, i2 = (pos >> 16) & 0xff, i3 = pos >> 24;
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        const uint32_t *pl = W.pl[p];
                        const uint32_t P0 = pl[i0], P1 = pl[i1], P2 = pl[i2], P3 = pl[i3];
                        const uint32_t s1 = P0 ^ P1, s2 = P2 ^ P3;
                        m[p] = ((se >> 31) ? (s1 & s2) | (((P0 & P1) ^ (P2 & P3)) & ~(s1 | s2)) : (s1 & s2)) &
                               live_m[p];
                    }
                }
                // the in-sector (group, row) pairs, flattened over the warp in (group, block, row) order
                int cnt = 0;
#pragma unroll
                for (int p = 0; p < NP; ++p) cnt += __popc(m[p]);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += v;
                }
                const int excl = incl - cnt;
                const int total = __shfl_sync(FULL, incl, 31);
                c_sec += cnt;
                for (int base = 0; base < total; base += BS_FQ) {
                    {   // this lane's pairs (ascending row) at positions excl.. of the (group, row) order
                        int j = excl;
#pragma unroll
                        for (int p = 0; p < NP; ++p) {
                            uint32_t v = m[p];
                            while (v) {
                                const int r = __ffs(v) - 1;
                                v &= v - 1;
                                if (j >= base && j < base + BS_FQ) W.fq[j - base] = (uint16_t)(lane | ((32 * p + r) << 8));
                                ++j;
                            }
                        }
                    }
                    __syncwarp();
                    const int lim = min(total, base + BS_FQ);
                    // a pair's lookup: the filter, then its first bucket (the loads are issued for
                    // BS_LF pairs per lane before any is resolved: BS_LF lookups in flight)
                    auto prep = [&](int f, int &lo, int &row, u64 &h, u64 &p0, u64 &p1) -> bool {
                        if (f >= lim) return false;
                        const uint32_t e = W.fq[f - base];
                        lo = (int)(e & 0xff);
                        row = (int)(e >> 8);
                        const uint4 rh = W.rh[row];
                        const BsRec &G = tl[g0 + lo];
                        if (!(bm_test(bmA, rh.z ^ G.fa) && bm_test(bmB, rh.w ^ G.fb))) return false;
                        const ulonglong2 xr = W.rx[row];
                        const ulonglong2 X = G.x;
                        h = ((u64)rh.x | ((u64)rh.y << 32)) ^ G.hx;
                        p0 = xr.x ^ X.x;
                        p1 = xr.y ^ X.y;
                        return true;
                    };
                    // a round's hits: H_xx' and psi(x')/psi-hat by the finding lane, then each
                    // row's lane adds its hits in (group) order
                    auto apply = [&](int64_t idx, int lo, int row) {
                        const unsigned hm = __ballot_sync(FULL, idx >= 0);
                        if (!hm) return;                     // rare: ~0.4 hits per 32 x 32 pairs at C5
                        if (idx >= 0) {                      // H_xx': the group's strings in order
                            const BsRec &G = tl[g0 + lo];
                            const ulonglong2 xr = W.rx[row];
                            const uint32_t b = G.sb, e = G.se & 0x7FFFFFFFu;
                            double hv = 0.0;
                            for (uint32_t i = b; i < e; ++i) {
                                const ulonglong2 Z = __ldg(H.tz + i);
                                const int par = (__popcll(xr.x & Z.x) + __popcll(xr.y & Z.y)) & 1;
                                hv += flip_sign(__ldg(H.td + i), par);
                            }
                            c_str += e - b;
                            const double2 lr = W.rl[row];
                            double2 ps;
                            if (!((lr.x - s) < -600.0)) {
                                ps = __ldg(T.psi_hat + idx);
                            } else {                         // reading R11
                                const double2 l2 = T.logpsi[idx];
                                const double mm = exp(l2.x - lr.x);
                                double sn, cs2;
                                sincos(l2.y - lr.y, &sn, &cs2);
                                ps = make_double2(mm * cs2, mm * sn);
                            }
                            W.qh[lane] = hv;
                            W.qp[lane] = ps;
                            W.qr[lane] = row;
                        }
                        __syncwarp();
                        unsigned h2 = hm;
                        while (h2) {
                            const int l = __ffs(h2) - 1;
                            h2 &= h2 - 1;
                            const int rw = W.qr[l];
                            if ((rw & 31) == lane) {
                                const double hv = W.qh[l];
                                const double2 ps = W.qp[l];
#pragma unroll
                                for (int p = 0; p < NP; ++p) {
                                    if ((rw >> 5) != p) continue;
                                    ar[p] = fma(hv, ps.x, ar[p]);
                                    ai[p] = fma(hv, ps.y, ai[p]);
                                }
                                ++c_hit;
                            }
                        }
                        __syncwarp();
                    };
                    for (int f0 = base; f0 < lim; f0 += 32 * BS_LF) {
                        int lo[BS_LF], rw[BS_LF];
                        u64 hh[BS_LF], a0[BS_LF], a1[BS_LF];
                        bool w[BS_LF];
                        ulonglong2 s01[BS_LF], s23[BS_LF];
                        int64_t idx[BS_LF];
#pragma unroll
                        for (int u = 0; u < BS_LF; ++u) {
                            lo[u] = rw[u] = 0;
                            hh[u] = a0[u] = a1[u] = 0;
                            w[u] = prep(f0 + 32 * u + lane, lo[u], rw[u], hh[u], a0[u], a1[u]);
                        }
#pragma unroll
                        for (int u = 0; u < BS_LF; ++u)
                            if (w[u]) {
                                const ulonglong2 *bk =
                                    reinterpret_cast<const ulonglong2 *>(T.slots + 4 * (hh[u] & T.bucket_mask));
                                s01[u] = __ldg(bk);
                                s23[u] = __ldg(bk + 1);
                            }
#pragma unroll
                        for (int u = 0; u < BS_LF; ++u)
                            idx[u] = w[u] ? probe_resolve(T, hh[u], a0[u], a1[u], s01[u], s23[u]) : -1;
#pragma unroll
                        for (int u = 0; u < BS_LF; ++u) apply(idx[u], lo[u], rw[u]);   // (group, row) order
                    }
                    __syncwarp();                        // the queue is refilled by the next pass / batch
                }
            }
            __syncwarp();
            if (lane == 0) {                         // the last warp done with the tile refills the stage
                __threadfence_block();
                if (atomicAdd(&s_done[st], 1u) == (unsigned)kWarps - 1) {
                    atomicExch(&s_done[st], 0u);
                    if (q + BS_STAGES < q_end) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue(q + BS_STAGES);
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int64_t r = r0 + 32 * p + lane;
            if (r < n_rows) {
                const bool live = lx[p].x > -INFINITY;
                double2 e;
                if (!live) {
                    e = make_double2(NAN, NAN);
                } else if ((lx[p].x - s) < -600.0) {
                    e = make_double2(ar[p], ai[p]);
                } else {
                    // E = acc / psi_hat(x) = acc * exp(-(logpsi(x) - s))
                    const double mm = exp(-(lx[p].x - s));
                    double sn, cs2;
                    sincos(-lx[p].y, &sn, &cs2);
                    const double ir = mm * cs2, ii = mm * sn;
                    e = make_double2(ar[p] * ir - ai[p] * ii, ar[p] * ii + ai[p] * ir);
                }
                if (live) c_pairs += (u64)K;
                out[r] = e;
                chunk_done_thread(cs, out, r, n_rows);
            }
        }
    }
    if (stats) {
        for (int o = 16; o; o >>= 1) {
            c_pairs += __shfl_xor_sync(0xffffffffu, c_pairs, o);
            c_sec += __shfl_xor_sync(0xffffffffu, c_sec, o);
            c_hit += __shfl_xor_sync(0xffffffffu, c_hit, o);
            c_str += __shfl_xor_sync(0xffffffffu, c_str, o);
        }
        if (lane == 0) {
            atomicAdd(stats + 0, c_pairs);
            atomicAdd(stats + 1, c_sec);
            atomicAdd(stats + 2, c_hit);
            atomicAdd(stats + 3, c_str);
        }
    }
}

// per-spin string filter bitmaps of a mode-0 table (k_eloc_bs): bit f_alpha(key) and bit f_beta(key)
__global__ void k_bs_bitmap(const ulonglong2 *keys, int64_t n, uint32_t *bm) {
    __shared__ uint32_t col[128];                   // the filter columns (per-lane bit loops: no
    if (threadIdx.x < 128) col[threadIdx.x] = c_filt[threadIdx.x];   // serialised constant reads)
    __syncthreads();
    auto f = [&](u64 w, int base) {
        uint32_t v = 0;
        while (w) {
            v ^= col[base + __ffsll((long long)w) - 1];
            w &= w - 1;
        }
        return v;
    };
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 k = keys[i];
        const uint32_t fa = f(k.x & ALPHA_MASK, 0) ^ f(k.y & ALPHA_MASK, 64);
        const uint32_t fb = f(k.x & BETA_MASK, 0) ^ f(k.y & BETA_MASK, 64);
        const uint32_t ba = fa & ((1u << BS_FB) - 1), bb = fb & ((1u << BS_FB) - 1);
        // most keys share their alpha or beta string with many others: read before the atomic
        if (!(__ldcg(bm + (ba >> 5)) >> (ba & 31) & 1u)) atomicOr(bm + (ba >> 5), 1u << (ba & 31));
        if (!(__ldcg(bm + BS_BM_WORDS / 2 + (bb >> 5)) >> (bb & 31) & 1u))
            atomicOr(bm + BS_BM_WORDS / 2 + (bb >> 5), 1u << (bb & 31));
    }
}

template <int MODE, bool CONS>
__global__ void k_coupled_debug(HamView H, TabView T, const ulonglong2 *rows, int64_t n_rows,
                                int64_t max_pairs, int64_t *oi, u64 *ox, double *oh,
                                unsigned long long *counter) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const u64 x0 = rows[r].x, x1 = rows[r].y;
        const u64 hx = (MODE == 0) ? hash128(x0, x1) : 0;
        u64 dummy = 0;
        for (int64_t k = 0; k < H.K; ++k) {
            const ulonglong2 X = H.gx[k];
            if (CONS) {
                const uint32_t info = H.ginfo[k];
                const int na = __popcll(x0 & X.x & ALPHA_MASK) + __popcll(x1 & X.y & ALPHA_MASK);
                const int nb = __popcll(x0 & X.x & BETA_MASK) + __popcll(x1 & X.y & BETA_MASK);
                if (na != (int)(info & 0xff) || nb != (int)((info >> 8) & 0xff)) continue;
            }
            const u64 p0 = x0 ^ X.x, p1 = x1 ^ X.y;
            int64_t idx;
            if (MODE == 1) idx = (p1 == 0 && p0 < (u64)T.n) ? (int64_t)p0 : -1;
            else idx = probe(T, hx ^ H.ghx[k], p0, p1);
            if (idx < 0) continue;
            const double hv = group_value(H, k, x0, x1, dummy);
            const unsigned long long slot = atomicAdd(counter, 1ULL);
            if ((int64_t)slot < max_pairs) {
                oi[3 * slot] = r;
                oi[3 * slot + 1] = k;
                oi[3 * slot + 2] = idx;
                ox[2 * slot] = p0;
                ox[2 * slot + 1] = p1;
                oh[slot] = hv;
            }
        }
    }
}

// ------------------------------------------------------------ energy reduce
// one warp per chunk of NNQS_REDUCE_CHUNK rows, 8 chunks per block; the fixed
// order of chunk_partial_warp (common.cuh), shared with the fused epilogues
__global__ void __launch_bounds__(256) k_chunk_partials(const double2 *eloc, const int64_t *counts,
                                                        int64_t n, const double *mean,
                                                        double *partials) {
    const int64_t ch = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t base = ch * NNQS_REDUCE_CHUNK;
    if (base >= n) return;
    const int len = (int)min((int64_t)NNQS_REDUCE_CHUNK, n - base);
    const double3 p = chunk_partial_warp<false>(eloc, counts, base, len, mean);
    if ((threadIdx.x & 31) == 0) {
        partials[3 * ch] = p.x;
        partials[3 * ch + 1] = p.y;
        partials[3 * ch + 2] = mean ? 0.0 : p.z;
    }
}

// one block of COMBINE_T threads: thread t sums chunks t, t + T, ... (ascending), then a
// fixed binary tree -- an order set by the global chunk grid alone (any rank split)
#define COMBINE_T 1024
__global__ void __launch_bounds__(COMBINE_T) k_combine(const double *partials, int64_t n_chunks, int pass,
                                                       double *out) {
    __shared__ double sw[COMBINE_T], s1[COMBINE_T], s2[COMBINE_T];
    const int t = threadIdx.x;
    double W = 0.0, S1 = 0.0, S2 = 0.0;
    for (int64_t c = t; c < n_chunks; c += COMBINE_T) {
        W += partials[3 * c];
        S1 += partials[3 * c + 1];
        S2 += partials[3 * c + 2];
    }
    sw[t] = W;
    s1[t] = S1;
    s2[t] = S2;
    __syncthreads();
    for (int h = COMBINE_T / 2; h; h >>= 1) {
        if (t < h) {
            sw[t] += sw[t + h];
            s1[t] += s1[t + h];
            s2[t] += s2[t + h];
        }
        __syncthreads();
    }
    if (t != 0) return;
    W = sw[0];
    S1 = s1[0];
    S2 = s2[0];
    if (pass == 1) {
        out[0] = S1 / W; out[1] = S2 / W; out[2] = W; out[3] = 0.0;
    } else {
        out[0] = S1 / W; out[1] = W; out[2] = 0.0; out[3] = 0.0;
    }
}

__global__ void k_any_nan(const double *x, int64_t n, int *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (isnan(x[i])) atomicOr(flag, 1);
}

inline int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

}  // namespace

// ======================================================================= host
int nnqs_ham_upload(nnqs_ham h) {
    int rc = ensure_hash(h->device);
    if (rc) return rc;
    const HostTable &H = h->host;
    const int64_t K = (int64_t)H.off.size() - 1, Nh = (int64_t)H.d.size();
    if (Nh >= (int64_t)0xFFFFFFFFLL)
        return nnqs_set_error(NNQS_E_SIZE, "more than 2^32-1 Pauli strings");
    u64 cols[128];
    nnqs_hash_columns(cols);
    std::vector<u64> hx(K);
    std::vector<uint32_t> info(K), off(K + 1);
    for (int64_t k = 0; k < K; ++k) {
        const u64 x0 = H.x[2 * k], x1 = H.x[2 * k + 1];
        hx[k] = nnqs_hash_host(cols, x0, x1);
        const int na = __builtin_popcountll(x0 & ALPHA_MASK) + __builtin_popcountll(x1 & ALPHA_MASK);
        const int nb = __builtin_popcountll(x0 & BETA_MASK) + __builtin_popcountll(x1 & BETA_MASK);
        info[k] = (uint32_t)(na / 2) | ((uint32_t)(nb / 2) << 8) | ((uint32_t)((na & 1) | (nb & 1)) << 16);
        off[k] = (uint32_t)H.off[k];
    }
    off[K] = (uint32_t)H.off[K];
    DeviceHam &D = h->dev;
    size_t bx = 16 * (size_t)K, bh = 8 * (size_t)K, bi = 4 * (size_t)K, bo = 4 * (size_t)(K + 1),
           bz = 16 * (size_t)Nh, bd = 8 * (size_t)Nh;
    if ((rc = cuda_check(cudaMalloc(&D.gx, bx ? bx : 16), "cudaMalloc gx"))) return rc;
    if ((rc = cuda_check(cudaMalloc((void **)&D.ghx, bh ? bh : 8), "cudaMalloc ghx"))) return rc;
    if ((rc = cuda_check(cudaMalloc((void **)&D.ginfo, bi ? bi : 4), "cudaMalloc ginfo"))) return rc;
    if ((rc = cuda_check(cudaMalloc((void **)&D.goff, bo), "cudaMalloc goff"))) return rc;
    if ((rc = cuda_check(cudaMalloc(&D.tz, bz ? bz : 16), "cudaMalloc tz"))) return rc;
    if ((rc = cuda_check(cudaMalloc((void **)&D.td, bd ? bd : 8), "cudaMalloc td"))) return rc;
    if (K) {
        if ((rc = cuda_check(cudaMemcpy(D.gx, H.x.data(), bx, cudaMemcpyHostToDevice), "copy gx"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.ghx, hx.data(), bh, cudaMemcpyHostToDevice), "copy ghx"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.ginfo, info.data(), bi, cudaMemcpyHostToDevice), "copy ginfo"))) return rc;
    }
    if ((rc = cuda_check(cudaMemcpy(D.goff, off.data(), bo, cudaMemcpyHostToDevice), "copy goff"))) return rc;
    if (Nh) {
        if ((rc = cuda_check(cudaMemcpy(D.tz, H.z.data(), bz, cudaMemcpyHostToDevice), "copy tz"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.td, H.d.data(), bd, cudaMemcpyHostToDevice), "copy td"))) return rc;
    }
    // the literal kernel's 32-B group records {X, h(X), info} (k_eloc_lit streams them)
    std::vector<LitRec> lit(std::max<int64_t>(K, 1));
    for (int64_t k = 0; k < K; ++k) lit[k] = LitRec{make_ulonglong2(H.x[2 * k], H.x[2 * k + 1]), hx[k], info[k], 0};
    const size_t bl = sizeof(LitRec) * lit.size();
    if ((rc = cuda_check(cudaMalloc(&D.glit, bl), "cudaMalloc glit"))) return rc;
    if ((rc = cuda_check(cudaMemcpy(D.glit, lit.data(), bl, cudaMemcpyHostToDevice), "copy glit"))) return rc;
    // the bit-sliced kernel's records: only when every flip mask has at most four
    // sites with an even count per spin (a number-conserving H: Eq. 9's singles and
    // doubles), so the 32-row sector test is one of the three forms of k_eloc_bs
    size_t bb = 0;
    bool bs_ok = H.conserving && K > 0 && Nh < 0x7FFFFFFFLL;
    for (int64_t k = 0; k < K && bs_ok; ++k) {
        const u64 x0 = H.x[2 * k], x1 = H.x[2 * k + 1];
        const int na = __builtin_popcountll(x0 & ALPHA_MASK) + __builtin_popcountll(x1 & ALPHA_MASK);
        const int nb = __builtin_popcountll(x0 & BETA_MASK) + __builtin_popcountll(x1 & BETA_MASK);
        bs_ok = (na & 1) == 0 && (nb & 1) == 0 && na + nb <= 4;
    }
    if (bs_ok) {
        uint32_t fcol[128];
        nnqs_filter_columns(fcol);
        std::vector<BsRec> bs(K);
        for (int64_t k = 0; k < K; ++k) {
            const u64 x[2] = {H.x[2 * k], H.x[2 * k + 1]};
            uint32_t fa = 0, fb = 0, pos = 0;
            int np = 0, na = 0;
            for (int spin = 0; spin < 2; ++spin)          // alpha sites (even qubits) first
                for (int j = 0; j < 128; ++j)
                    if ((x[j >> 6] >> (j & 63) & 1) && (j & 1) == spin) {
                        (spin ? fb : fa) ^= fcol[j];
                        pos |= (uint32_t)j << (8 * np++);
                        na += spin == 0;
                    }
            const bool quad = na == 4 || np - na == 4;
            if (np == 0) pos = 128u | 129u << 8 | 128u << 16 | 129u << 24;
            else if (np == 2) pos |= 128u << 16 | 129u << 24;
            bs[k] = BsRec{make_ulonglong2(x[0], x[1]), hx[k], fa, fb, pos, off[k],
                          off[k + 1] | (quad ? 0x80000000u : 0u), 0};
        }
        bb = sizeof(BsRec) * bs.size();
        if ((rc = cuda_check(cudaMalloc(&D.gbs, bb), "cudaMalloc gbs"))) return rc;
        if ((rc = cuda_check(cudaMemcpy(D.gbs, bs.data(), bb, cudaMemcpyHostToDevice), "copy gbs"))) return rc;
    }
    D.bytes = (int64_t)(bx + bh + bi + bo + bz + bd + bl + bb);
    return NNQS_OK;
}

void nnqs_ham_release(nnqs_ham h) {
    DeviceHam &D = h->dev;
    cudaFree(D.gx); cudaFree(D.ghx); cudaFree(D.ginfo); cudaFree(D.goff); cudaFree(D.tz); cudaFree(D.td);
    cudaFree(D.glit);
    cudaFree(D.gbs);
    D = DeviceHam();
}

int nnqs_table_build(nnqs_table t, const uint64_t *keys, const double *logpsi, void *stream, bool defer_check) {
    int rc = ensure_hash(t->device);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = t->n;
    size_t bk = 16 * (size_t)n;
    // shift key + flag in one small allocation
    if ((rc = cuda_check(nnqs_malloc_async((void **)&t->shift_key, 16, st), "alloc shift"))) return rc;
    t->flag = (int *)(t->shift_key + 1);
    if ((rc = cuda_check(cudaMemsetAsync(t->shift_key, 0, 16, st), "memset shift"))) return rc;
    if ((rc = cuda_check(nnqs_malloc_async(&t->logpsi, bk ? bk : 16, st), "alloc logpsi"))) return rc;
    if ((rc = cuda_check(nnqs_malloc_async(&t->psi_hat, bk ? bk : 16, st), "alloc psi_hat"))) return rc;
    if (n) {
        if ((rc = cuda_check(cudaMemcpyAsync(t->logpsi, logpsi, bk, cudaMemcpyDeviceToDevice, st), "copy logpsi"))) return rc;
    }
    t->bytes = 16 + 2 * (int64_t)bk;
    if (t->mode == 0) {
        u64 nb = 1;
        while (nb * 4 < 4 * (u64)(n > 0 ? n : 1)) nb <<= 1;   // load factor <= 1/4: ~2 % of buckets full
        t->bucket_mask = nb - 1;
        if ((rc = cuda_check(nnqs_malloc_async(&t->keys, bk ? bk : 16, st), "alloc keys"))) return rc;
        if ((rc = cuda_check(nnqs_malloc_async((void **)&t->slots, 32 * nb, st), "alloc slots"))) return rc;
        if (n) {
            if ((rc = cuda_check(cudaMemcpyAsync(t->keys, keys, bk, cudaMemcpyDeviceToDevice, st), "copy keys"))) return rc;
        }
        if ((rc = cuda_check(cudaMemsetAsync(t->slots, 0xFF, 32 * nb, st), "memset slots"))) return rc;
        t->bytes += (int64_t)bk + 32 * (int64_t)nb;
        if ((rc = cuda_check(nnqs_malloc_async((void **)&t->bsbm, 4 * (size_t)BS_BM_WORDS, st), "alloc bsbm"))) return rc;
        if ((rc = cuda_check(cudaMemsetAsync(t->bsbm, 0, 4 * (size_t)BS_BM_WORDS, st), "memset bsbm"))) return rc;
        t->bytes += 4 * (int64_t)BS_BM_WORDS;
        if (n > 1) k_check_order<<<grid_for(n, 256), 256, 0, st>>>((const ulonglong2 *)t->keys, n, t->flag);
        if (n) k_hash_insert<<<grid_for(n, 256), 256, 0, st>>>((const ulonglong2 *)t->keys, n, t->slots, t->bucket_mask);
        if (n) k_bs_bitmap<<<grid_for(n, 256), 256, 0, st>>>((const ulonglong2 *)t->keys, n, t->bsbm);
    }
    if (n) {
        k_max_re<<<grid_for(n, 256), 256, 0, st>>>((const double2 *)t->logpsi, n, t->shift_key);
        k_psi_hat<<<grid_for(n, 256), 256, 0, st>>>((const double2 *)t->logpsi, n, t->shift_key,
                                                     (double2 *)t->psi_hat, t->flag + 1);
    }
    if ((rc = cuda_check(cudaGetLastError(), "table kernels"))) return rc;
    if (n && !defer_check) return nnqs_table_check(t, nullptr, stream);
    return NNQS_OK;
}

// the build's flags (order violation, rows on the exp-ratio path): read with a sync of
// `stream`, or (host != nullptr) already copied there by a caller that synchronised
int nnqs_table_check(nnqs_table t, const int *host, void *stream) {
    int flag[2] = {0, 0};   // order violation, rows with psi_hat(x) < e^-600
    if (!host) {
        cudaStream_t st = (cudaStream_t)stream;
        int rc;
        if ((rc = cuda_check(cudaMemcpyAsync(flag, t->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st), "read flag"))) return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(st), "sync"))) return rc;
        host = flag;
    }
    t->n_direct = host[1];
    if (t->mode == 0 && host[0]) return nnqs_set_error(NNQS_E_TABLE, "keys are not strictly increasing as 128-bit integers");
    return NNQS_OK;
}

void nnqs_table_release(nnqs_table t) {
    cudaStream_t st = (cudaStream_t)t->stream;
    if (t->keys) cudaFreeAsync(t->keys, st);
    if (t->logpsi) cudaFreeAsync(t->logpsi, st);
    if (t->psi_hat) cudaFreeAsync(t->psi_hat, st);
    if (t->slots) cudaFreeAsync(t->slots, st);
    if (t->bsbm) cudaFreeAsync(t->bsbm, st);
    t->bsbm = nullptr;
    if (t->shift_key) cudaFreeAsync(t->shift_key, st);
    t->keys = t->logpsi = t->psi_hat = nullptr;
    t->slots = t->shift_key = nullptr;
}

int nnqs_launch_local_energy(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows,
                             const double *row_logpsi, int64_t n_rows, double *eloc,
                             int64_t *stats, const ChunkSink &cs, void *stream) {
    if (n_rows == 0) return NNQS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    HamView H = ham_view(h);
    TabView T = tab_view(t);
    const bool cons = h->host.conserving;
    const int g = grid_for(n_rows, 256);
    auto *r = (const ulonglong2 *)rows;
    auto *rl = (const double2 *)row_logpsi;
    auto *o = (double2 *)eloc;
    auto *s = (unsigned long long *)stats;
    const int lk = t->opt.literal_kernel;
    if (lk == NNQS_LIT_AUTO && t->mode == 0 && cons && h->dev.gbs && t->bsbm) {   // bit-sliced (k_eloc_bs)
        cudaFuncSetAttribute(k_eloc_bs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BS_SMEM);
        // one CTA per SM, 32 rows per warp; fewer warps per CTA when the rows would not fill 148 CTAs
        const int64_t warps_needed = (n_rows + 32 * BS_P - 1) / (32 * BS_P);
        const int64_t per = std::min<int64_t>(BS_WARPS, std::max<int64_t>(1, (warps_needed + 147) / 148)) * 32;
        const int gl = (int)std::min<int64_t>((n_rows + per * BS_P - 1) / (per * BS_P), 148);
        k_eloc_bs<<<gl, (unsigned)per, BS_SMEM, st>>>(H, (const BsRec *)h->dev.gbs, T, t->bsbm, row_begin, r, rl,
                                                       n_rows, o, s, cs);
        return cuda_check(cudaGetLastError(), "local energy launch");
    }
    if (h->dev.glit && lk != NNQS_LIT_PLAIN) {    // staged literal kernel (k_eloc_lit)
        auto kern = t->mode == 0 ? (cons ? k_eloc_lit<0, true> : k_eloc_lit<0, false>)
                                 : (cons ? k_eloc_lit<1, true> : k_eloc_lit<1, false>);
        const size_t smem = (size_t)LIT_STAGES * LIT_TILE * sizeof(LitRec);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // one CTA per SM; fewer threads per CTA when the rows would not fill 148 CTAs
        const int64_t per = std::min<int64_t>(LIT_THREADS, std::max<int64_t>(64, ((n_rows + 147) / 148 + 31) / 32 * 32));
        const int64_t blocks = (n_rows + per - 1) / per;
        const int gl = (int)std::min<int64_t>(blocks, 148);
        kern<<<gl, (unsigned)per, smem, st>>>(H, (const LitRec *)h->dev.glit, T, row_begin, r, rl, n_rows, o, s, cs);
        return cuda_check(cudaGetLastError(), "local energy launch");
    }
    if (t->mode == 0) {
        if (cons) k_eloc_v1<0, true><<<g, 256, 0, st>>>(H, T, row_begin, r, rl, n_rows, o, s, cs);
        else k_eloc_v1<0, false><<<g, 256, 0, st>>>(H, T, row_begin, r, rl, n_rows, o, s, cs);
    } else {
        if (cons) k_eloc_v1<1, true><<<g, 256, 0, st>>>(H, T, row_begin, r, rl, n_rows, o, s, cs);
        else k_eloc_v1<1, false><<<g, 256, 0, st>>>(H, T, row_begin, r, rl, n_rows, o, s, cs);
    }
    return cuda_check(cudaGetLastError(), "local energy launch");
}

int nnqs_launch_coupled_debug(nnqs_ham h, nnqs_table t, const uint64_t *rows_dev, int64_t n_rows,
                              int64_t max_pairs, int64_t *oi, u64 *ox, double *oh,
                              unsigned long long *counter, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    HamView H = ham_view(h);
    TabView T = tab_view(t);
    const bool cons = h->host.conserving;
    const int g = grid_for(n_rows, 128);
    auto *r = (const ulonglong2 *)rows_dev;
    if (t->mode == 0) {
        if (cons) k_coupled_debug<0, true><<<g, 128, 0, st>>>(H, T, r, n_rows, max_pairs, oi, ox, oh, counter);
        else k_coupled_debug<0, false><<<g, 128, 0, st>>>(H, T, r, n_rows, max_pairs, oi, ox, oh, counter);
    } else {
        if (cons) k_coupled_debug<1, true><<<g, 128, 0, st>>>(H, T, r, n_rows, max_pairs, oi, ox, oh, counter);
        else k_coupled_debug<1, false><<<g, 128, 0, st>>>(H, T, r, n_rows, max_pairs, oi, ox, oh, counter);
    }
    return cuda_check(cudaGetLastError(), "coupled debug launch");
}

// ----------------------------------------------------------- C-ABI: reduce
extern "C" int nnqs_energy_chunk_partials(const double *eloc, const int64_t *counts, int64_t n,
                                          const double *mean_dev, double *partials,
                                          void *cuda_stream) {
    if (n < 0 || (n > 0 && (!eloc || !counts || !partials)))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_energy_chunk_partials: bad arguments");
    if (n == 0) return NNQS_OK;
    const int64_t chunks = (n + NNQS_REDUCE_CHUNK - 1) / NNQS_REDUCE_CHUNK;
    k_chunk_partials<<<(unsigned)((chunks + 7) / 8), 256, 0, (cudaStream_t)cuda_stream>>>(
        (const double2 *)eloc, counts, n, mean_dev, partials);
    return cuda_check(cudaGetLastError(), "chunk partials launch");
}

extern "C" int nnqs_energy_combine(const double *partials, int64_t n_chunks, int pass,
                                   double *out_dev, void *cuda_stream) {
    if (!partials || !out_dev || n_chunks <= 0 || (pass != 1 && pass != 2))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_energy_combine: bad arguments");
    k_combine<<<1, COMBINE_T, 0, (cudaStream_t)cuda_stream>>>(partials, n_chunks, pass, out_dev);
    return cuda_check(cudaGetLastError(), "combine launch");
}

// Eq. (7) weights: a_u = 2 w_u Re(E_u - mean) / W,
// b_u = 2 w_u Im(E_u - mean) / W; energy = (mean_re, mean_im, W).
__global__ void k_grad_weights(const double2 *eloc, const int64_t *counts, int64_t n, const double *energy,
                               double2 *ab) {
    const double mre = energy[0], mim = energy[1], W = energy[2];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 e = eloc[i];
        const double f = 2.0 * (double)counts[i] / W;
        ab[i] = make_double2(f * (e.x - mre), f * (e.y - mim));
    }
}

extern "C" int nnqs_grad_weights(const double *eloc, const int64_t *counts, int64_t n, const double *energy_dev,
                                 double *ab_out, void *cuda_stream) {
    if (n < 0 || (n > 0 && (!eloc || !counts || !energy_dev || !ab_out)))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_grad_weights: bad arguments");
    if (n == 0) return NNQS_OK;
    k_grad_weights<<<grid_for(n, 256), 256, 0, (cudaStream_t)cuda_stream>>>((const double2 *)eloc, counts, n,
                                                                          energy_dev, (double2 *)ab_out);
    return cuda_check(cudaGetLastError(), "grad weights launch");
}

extern "C" int nnqs_energy_reduce(const double *eloc, const int64_t *counts, int64_t n,
                                  double out[4], void *cuda_stream) {
    if (n <= 0 || !eloc || !counts || !out)
        return nnqs_set_error(NNQS_E_ARG, "nnqs_energy_reduce: bad arguments");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int64_t chunks = (n + NNQS_REDUCE_CHUNK - 1) / NNQS_REDUCE_CHUNK;
    double *buf = nullptr;
    int rc = cuda_check(nnqs_malloc_async((void **)&buf, sizeof(double) * (3 * chunks + 8), st), "alloc reduce");
    if (rc) return rc;
    double *part = buf, *o1 = buf + 3 * chunks, *o2 = o1 + 4;
    k_chunk_partials<<<(unsigned)((chunks + 7) / 8), 256, 0, st>>>((const double2 *)eloc, counts, n, nullptr, part);
    k_combine<<<1, COMBINE_T, 0, st>>>(part, chunks, 1, o1);
    k_chunk_partials<<<(unsigned)((chunks + 7) / 8), 256, 0, st>>>((const double2 *)eloc, counts, n, o1, part);
    k_combine<<<1, COMBINE_T, 0, st>>>(part, chunks, 2, o2);
    double h[8];
    rc = cuda_check(cudaMemcpyAsync(h, o1, sizeof(h), cudaMemcpyDeviceToHost, st), "read reduce");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync reduce");
    cudaFreeAsync(buf, st);
    if (rc) return rc;
    out[0] = h[0]; out[1] = h[1]; out[2] = h[4]; out[3] = h[2];
    if (!(h[2] > 0.0)) return nnqs_set_error(NNQS_E_EMPTY, "sum of counts is zero");
    return NNQS_OK;
}

extern "C" int nnqs_local_energy_check(const double *eloc, int64_t n, void *cuda_stream) {
    if (n < 0 || (n > 0 && !eloc)) return nnqs_set_error(NNQS_E_ARG, "nnqs_local_energy_check: bad arguments");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int *flag = nullptr;
    int rc = cuda_check(nnqs_malloc_async((void **)&flag, sizeof(int), st), "alloc flag");
    if (rc) return rc;
    cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (n) k_any_nan<<<grid_for(2 * n, 256), 256, 0, st>>>(eloc, 2 * n, flag);
    int h = 0;
    rc = cuda_check(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "read flag");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
    cudaFreeAsync(flag, st);
    if (rc) return rc;
    if (h) return nnqs_set_error(NNQS_E_ZERO_PSI, "some row has psi(x) = 0 (E_loc set to NaN)");
    return NNQS_OK;
}
