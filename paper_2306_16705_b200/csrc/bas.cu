// bas.cu -- one layer of batch autoregressive sampling (BAS, PAPER.md:224-229,
// Fig. 3(b)) with the number-conservation mask (Eq. 12): every
// unique prefix of the layer splits its weight w among its four children (the
// two qubits of spatial orbital i: outcome o -> alpha bit o & 1 at qubit 2i, beta
// bit o >> 1 at qubit 2i+1; orbitals are sampled from n-1 down to 0, "the reverse
// order of the qubits") by a multinomial draw of exactly w samples from the
// masked conditional distribution; zero-weight children are pruned.
//
// The draw is a chain of conditional binomials (reading R24): inversion
// (BINV) when n * min(p, 1 - p) < 10, else Hormann's transformed rejection (BTRS).
// Its uniforms come from a counter-based generator keyed by (seed, orbital, parent
// key), so a node's children depend on the node alone: any partition of a layer
// over ranks (parallel BAS) reproduces the serial samples exactly.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include "internal.h"

namespace {

__device__ __forceinline__ u64 bas_mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// uniform stream of one node: U_t = 53 high bits of mix(base + (t + 1) * golden) / 2^53
struct Stream {
    u64 base;
    u64 t;
    __device__ double next() {
        ++t;
        return (double)(bas_mix(base + t * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
    }
};

__device__ __forceinline__ double log_fact(double k) {   // log(k!), k >= 0 integral
    const double tab[10] = {0.0, 0.0, 0.6931471805599453, 1.791759469228055, 3.1780538303479458,
                            4.787491742782046, 6.579251212010101, 8.525161361065415, 10.60460290274525,
                            12.801827480081469};
    if (k < 10.0) return tab[(int)k];
    const double z = k + 1.0;
    return (k + 0.5) * log(z) - z + 0.9189385332046727 + (1.0 / 12.0 - 1.0 / (360.0 * z * z)) / z;
}

// Binomial(n, p) with 0 < p <= 1/2
__device__ long long binom_half(long long n, double p, Stream &S) {
    const double nd = (double)n, q = 1.0 - p;
    if (nd * p < 10.0) {                                   // BINV: inversion of the CDF
        const double s = p / q, a = (nd + 1.0) * s;
        while (true) {
            double r = exp(nd * log1p(-p));                // q^n
            double u = S.next();
            long long x = 0;
            while (x <= n && x < 256) {
                if (u < r) return x;
                u -= r;
                ++x;
                r *= a / (double)x - s;
            }
        }
    }
    const double spq = sqrt(nd * p * q);                  // BTRS (Hormann 1993)
    const double b = 1.15 + 2.53 * spq;
    const double a = -0.0873 + 0.0248 * b + 0.01 * p;
    const double c = nd * p + 0.5;
    const double vr = 0.92 - 4.2 / b;
    const double alpha = (2.83 + 5.1 / b) * spq;
    const double lpq = log(p / q);
    const double m = floor((nd + 1.0) * p);
    const double h = log_fact(m) + log_fact(nd - m);
    while (true) {
        const double u = S.next() - 0.5;
        double v = S.next();
        const double us = 0.5 - fabs(u);
        const double k = floor((2.0 * a / us + b) * u + c);
        if (!(k >= 0.0 && k <= nd)) continue;
        if (us >= 0.07 && v <= vr) return (long long)k;
        v = log(v * alpha / (a / (us * us) + b));
        if (v <= h - log_fact(k) - log_fact(nd - k) + (k - m) * lpq) return (long long)k;
    }
}

__device__ long long binom(long long n, double p, Stream &S) {
    if (n <= 0 || p <= 0.0) return 0;
    if (p >= 1.0) return n;
    if (p > 0.5) return n - binom_half(n, 1.0 - p, S);
    return binom_half(n, p, S);
}

// one thread per parent: masked multinomial split of its weight into 4 children
__global__ void k_bas_split(const ulonglong2 *keys, const long long *counts, const double *probs, int64_t m,
                            int orbital, int n_up, int n_dn, u64 seed, long long *child, int32_t *flag,
                            int *err) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 k = keys[j];
        const long long w = counts[j];
        const int na = __popcll(k.x & 0x5555555555555555ULL) + __popcll(k.y & 0x5555555555555555ULL);
        const int nb = __popcll(k.x & 0xAAAAAAAAAAAAAAAAULL) + __popcll(k.y & 0xAAAAAAAAAAAAAAAAULL);
        double q[4];
        for (int o = 0; o < 4; ++o) {
            const int a2 = na + (o & 1), b2 = nb + (o >> 1);
            const bool ok = a2 <= n_up && b2 <= n_dn && a2 + orbital >= n_up && b2 + orbital >= n_dn;
            const double pr = probs[4 * j + o];
            q[o] = ok ? pr : 0.0;
        }
        const double S3 = q[3], S2 = q[2] + S3, S1 = q[1] + S2, S0 = q[0] + S1;
        const double tail[4] = {S0, S1, S2, S3};
        long long c[4] = {0, 0, 0, 0};
        if (w > 0 && !(S0 > 0.0)) {
            atomicExch(err, 1);                            // no feasible continuation (caller bug)
        } else {
            Stream st{bas_mix(bas_mix(bas_mix(bas_mix(seed) ^ (u64)(orbital + 1)) ^ k.x) ^ k.y), 0};
            long long rem = w;
            for (int o = 0; o < 3; ++o) {
                if (rem > 0 && q[o] > 0.0) c[o] = binom(rem, q[o] / tail[o], st);
                rem -= c[o];
            }
            c[3] = rem;
        }
        for (int o = 0; o < 4; ++o) {
            child[4 * j + o] = c[o];
            flag[4 * j + o] = c[o] > 0 ? 1 : 0;
        }
    }
}

__global__ void k_bas_scatter(const ulonglong2 *keys, const long long *child, const int32_t *pos, int64_t m,
                              int orbital, ulonglong2 *keys_out, long long *counts_out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 4 * m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const long long c = child[e];
        if (c <= 0) continue;
        const int o = (int)(e & 3);
        ulonglong2 k = keys[e >> 2];
        const int qa = 2 * orbital, qb = 2 * orbital + 1;
        if (o & 1) (qa < 64 ? k.x : k.y) |= 1ULL << (qa & 63);
        if (o >> 1) (qb < 64 ? k.x : k.y) |= 1ULL << (qb & 63);
        keys_out[pos[e]] = k;
        counts_out[pos[e]] = c;
    }
}

inline int grid_of(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

int nnqs_bas_layer(const uint64_t *keys, const int64_t *counts, const double *probs, int64_t m, int orbital,
                   int n_orbitals, int n_up, int n_dn, uint64_t seed, uint64_t *keys_out, int64_t *counts_out,
                   int64_t *m_out, void *cuda_stream) {
    if (!m_out || m < 0 || (m > 0 && (!keys || !counts || !probs || !keys_out || !counts_out)))
        return nnqs_set_error(NNQS_E_ARG, "nnqs_bas_layer: bad arguments");
    if (n_orbitals < 1 || n_orbitals > 64 || orbital < 0 || orbital >= n_orbitals || n_up < 0 || n_dn < 0 ||
        n_up > n_orbitals || n_dn > n_orbitals)
        return nnqs_set_error(NNQS_E_SIZE, "nnqs_bas_layer: need 0 <= orbital < n_orbitals <= 64, electrons <= n");
    if (m >= (1LL << 29)) return nnqs_set_error(NNQS_E_SIZE, "nnqs_bas_layer: layer wider than 2^29 nodes");
    *m_out = 0;
    if (m == 0) return NNQS_OK;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t *)nullptr, (int32_t *)nullptr, (int)(4 * m + 1), st);
    const size_t bc = 8 * 4 * (size_t)m, bf = 4 * (4 * (size_t)m + 1);
    char *buf = nullptr;
    cudaError_t e = nnqs_malloc_async((void **)&buf, bc + 2 * bf + tb + 64, st);
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_NOMEM, cudaGetErrorString(e));
    long long *child = (long long *)buf;
    int32_t *flag = (int32_t *)(buf + bc), *pos = (int32_t *)(buf + bc + bf);
    int *err = (int *)(buf + bc + 2 * bf);
    void *tmp = buf + bc + 2 * bf + 16;
    cudaMemsetAsync(err, 0, 4, st);
    cudaMemsetAsync(flag + 4 * m, 0, 4, st);
    k_bas_split<<<grid_of(m), 256, 0, st>>>((const ulonglong2 *)keys, (const long long *)counts, probs, m, orbital,
                                           n_up, n_dn, seed, child, flag, err);
    cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)(4 * m + 1), st);
    int32_t tot = 0;
    int herr = 0;
    cudaMemcpyAsync(&tot, pos + 4 * m, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st);
    k_bas_scatter<<<grid_of(4 * m), 256, 0, st>>>((const ulonglong2 *)keys, child, pos, m, orbital,
                                                 (ulonglong2 *)keys_out, (long long *)counts_out);
    e = cudaStreamSynchronize(st);
    cudaFreeAsync(buf, st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return nnqs_set_error(NNQS_E_CUDA, cudaGetErrorString(e));
    if (herr) return nnqs_set_error(NNQS_E_ARG, "nnqs_bas_layer: a node has no feasible continuation (all masked)");
    *m_out = tot;
    return NNQS_OK;
}
