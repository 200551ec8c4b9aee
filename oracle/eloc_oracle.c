/*
 * oracle/eloc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow CPU definition of the local energy of PAPER.md Eq. (4)
 * (Sec. 2.1) for the second-quantised Hamiltonian of
 * Eq. (9) (Sec. 2.3) under the Jordan-Wigner sign rules
 * (the paper uses OpenFermion's convention):
 *
 *   a_j |x>  = 0 if x_j = 0, else (-1)^{popc(x & (2^j - 1))} |x - 2^j>
 *   a+_j |x> = 0 if x_j = 1, else (-1)^{popc(x & (2^j - 1))} |x + 2^j>
 *
 *   H = e_core + sum_{pq,s} h_pq a+_{ps} a_{qs}
 *       + 1/2 sum_{pqrs,s,t} (pq|rs) a+_{ps} a+_{rt} a_{st} a_{qs}
 *
 * (spatial chemists' integrals; spin orbital (p,s) = qubit 2p+s, PAPER.md:287;
 * DESIGN.md readings R7, R8).  H|x> is built by applying every term right to
 * left (terms whose annihilator meets an empty orbital are zero and are
 * skipped, as are terms with a zero integral).  H is real symmetric, so the
 * coefficient of |x'> in H|x>, <x'|H|x>, equals H_{x x'}.
 *
 *   E_loc(x) = sum_{x' in T} H_{x x'} psi(x') / psi(x),
 *   psi(y)/psi(x) = exp(logpsi(y) - logpsi(x))      (complex)
 *
 * T = the sorted unique-sample table (sample-aware mode: x'
 * not in T contributes zero; membership by bisection) or all
 * 2^N configurations (exact mode, logpsi indexed by x).  Accumulation in
 * long double with Neumaier compensation, terms in ascending table index.
 *
 * This file shares no code with the CUDA library; only tests/, bench.py's
 * cpu_baseline leg and __graft_entry__.smoke() may call it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { uint64_t w[2]; } det_t;

static int occupied(const det_t *x, int j) { return (int)((x->w[j >> 6] >> (j & 63)) & 1u); }

/* popc(x & (2^j - 1)) mod 2: the Jordan-Wigner string of qubit j */
static int parity_below(const det_t *x, int j) {
    int c;
    if (j >= 64)
        c = __builtin_popcountll(x->w[0]) + __builtin_popcountll(x->w[1] & ((1ULL << (j - 64)) - 1));
    else
        c = __builtin_popcountll(x->w[0] & ((1ULL << j) - 1));
    return c & 1;
}

/* a_j: returns 0 if the result is the zero vector */
static int annihilate(det_t *x, int j, int *sign) {
    if (!occupied(x, j)) return 0;
    *sign ^= parity_below(x, j);
    x->w[j >> 6] &= ~(1ULL << (j & 63));
    return 1;
}

/* a+_j */
static int create(det_t *x, int j, int *sign) {
    if (occupied(x, j)) return 0;
    *sign ^= parity_below(x, j);
    x->w[j >> 6] |= (1ULL << (j & 63));
    return 1;
}

static int det_cmp(const det_t *a, const uint64_t *k) {
    if (a->w[1] != k[1]) return a->w[1] < k[1] ? -1 : 1;
    if (a->w[0] != k[0]) return a->w[0] < k[0] ? -1 : 1;
    return 0;
}

typedef struct {
    int exact;
    const uint64_t *keys;   /* sorted [n_keys][2] (sample mode) */
    int64_t n_keys;
    long double *acc;       /* [n_keys] */
    unsigned char *touched; /* [n_keys] */
    int64_t *list;          /* touched indices */
    int64_t n_list;
} row_ctx_t;

static int64_t table_index(const row_ctx_t *c, const det_t *y) {
    if (c->exact) {
        if (y->w[1] != 0 || (c->n_keys < (1LL << 62) && y->w[0] >= (uint64_t)c->n_keys)) return -1;
        return (int64_t)y->w[0];
    }
    int64_t lo = 0, hi = c->n_keys - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        int r = det_cmp(y, c->keys + 2 * mid);
        if (r == 0) return mid;
        if (r < 0) hi = mid - 1; else lo = mid + 1;
    }
    return -1;
}

static void emit(row_ctx_t *c, const det_t *y, long double v) {
    int64_t idx = table_index(c, y);
    if (idx < 0) return;
    if (!c->touched[idx]) {
        c->touched[idx] = 1;
        c->acc[idx] = 0.0L;
        c->list[c->n_list++] = idx;
    }
    c->acc[idx] += v;
}

/* Apply every term of Eq. (9) to |x> (O2a) and accumulate <x'|H|x> for x' in T. */
static void apply_hamiltonian(int n, const double *h1, const double *h2, double e_core,
                              const det_t *x, row_ctx_t *c) {
    emit(c, x, (long double)e_core);
    for (int sq = 0; sq < 2; ++sq)
        for (int q = 0; q < n; ++q) {
            det_t y = *x; int s1 = 0;
            if (!annihilate(&y, 2 * q + sq, &s1)) continue;
            for (int p = 0; p < n; ++p) {
                double v = h1[p * n + q];
                if (v == 0.0) continue;
                det_t z = y; int s2 = s1;
                if (!create(&z, 2 * p + sq, &s2)) continue;
                emit(c, &z, s2 ? -(long double)v : (long double)v);
            }
        }
    for (int sg = 0; sg < 2; ++sg)
        for (int q = 0; q < n; ++q) {
            det_t y1 = *x; int s1 = 0;
            if (!annihilate(&y1, 2 * q + sg, &s1)) continue;
            for (int tau = 0; tau < 2; ++tau)
                for (int s = 0; s < n; ++s) {
                    det_t y2 = y1; int s2 = s1;
                    if (!annihilate(&y2, 2 * s + tau, &s2)) continue;
                    for (int r = 0; r < n; ++r) {
                        det_t y3 = y2; int s3 = s2;
                        if (!create(&y3, 2 * r + tau, &s3)) continue;
                        for (int p = 0; p < n; ++p) {
                            double v = h2[(((size_t)p * n + q) * n + r) * n + s];
                            if (v == 0.0) continue;
                            det_t y4 = y3; int s4 = s3;
                            if (!create(&y4, 2 * p + sg, &s4)) continue;
                            long double hv = 0.5L * (long double)v;
                            emit(c, &y4, s4 ? -hv : hv);
                        }
                    }
                }
        }
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static void neumaier(long double *sum, long double *comp, long double v) {
    long double t = *sum + v;
    if (fabsl(*sum) >= fabsl(v)) *comp += (*sum - t) + v;
    else *comp += (v - t) + *sum;
    *sum = t;
}

static int check_sorted(const uint64_t *keys, int64_t n) {
    for (int64_t i = 1; i < n; ++i) {
        const uint64_t *a = keys + 2 * (i - 1), *b = keys + 2 * i;
        if (!(a[1] < b[1] || (a[1] == b[1] && a[0] < b[0]))) return 0;
    }
    return 1;
}

static int ctx_init(row_ctx_t *c, int exact, const uint64_t *keys, int64_t n_keys) {
    c->exact = exact; c->keys = keys; c->n_keys = n_keys; c->n_list = 0;
    c->acc = (long double *)malloc(sizeof(long double) * (size_t)n_keys);
    c->touched = (unsigned char *)calloc((size_t)n_keys, 1);
    c->list = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_keys);
    return c->acc && c->touched && c->list;
}

static void ctx_reset(row_ctx_t *c) {
    for (int64_t i = 0; i < c->n_list; ++i) c->touched[c->list[i]] = 0;
    c->n_list = 0;
}

static void ctx_free(row_ctx_t *c) { free(c->acc); free(c->touched); free(c->list); }

/*
 * Hits of one row: every x' in T reached by a term of H from x, with
 * H_{x x'} (the long-double sum rounded to double), ascending table index.
 * exact != 0: T = all 2^N states, index = x'.  Returns 0, or -4 if keys are not
 * strictly increasing, -7 on allocation failure, -2 if max_hits is too small.
 */
int oracle_row_hits(int n, const double *h1, const double *h2, double e_core,
                    int exact, const uint64_t *keys, int64_t n_keys, const uint64_t *x,
                    int64_t max_hits, int64_t *hit_idx, double *hit_h, int64_t *n_hits) {
    if (!exact && !check_sorted(keys, n_keys)) return -4;
    row_ctx_t c;
    if (!ctx_init(&c, exact, keys, n_keys)) { ctx_free(&c); return -7; }
    det_t d = {{x[0], x[1]}};
    apply_hamiltonian(n, h1, h2, e_core, &d, &c);
    qsort(c.list, (size_t)c.n_list, sizeof(int64_t), cmp_i64);
    int rc = 0;
    if (c.n_list > max_hits) rc = -2;
    for (int64_t i = 0; i < c.n_list && i < max_hits; ++i) {
        hit_idx[i] = c.list[i];
        hit_h[i] = (double)c.acc[c.list[i]];
    }
    *n_hits = c.n_list;
    ctx_free(&c);
    return rc;
}

/*
 * E_loc for n_rows rows (explicit keys + their log psi) against table T.
 * eloc_out [n_rows][2] = (Re, Im); NaN for a row with psi(x) = 0.
 * scale_out (optional) [n_rows] = sum_x' |H_xx'| |psi(x')/psi(x)|, the scale of
 * the parity tolerance (reading R14).
 */
int oracle_eloc(int n, const double *h1, const double *h2, double e_core,
                int exact, const uint64_t *keys, const double *logpsi, int64_t n_keys,
                const uint64_t *rows, const double *row_logpsi, int64_t n_rows,
                double *eloc_out, double *scale_out, int n_threads) {
    if (!exact && !check_sorted(keys, n_keys)) return -4;
    int rc = 0;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel num_threads(n_threads)
#endif
    {
        row_ctx_t c;
        int ok = ctx_init(&c, exact, keys, n_keys);
        if (!ok) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            rc = -7;
        }
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < n_rows; ++i) {
            if (!ok) continue;
            double lre = row_logpsi[2 * i], lim = row_logpsi[2 * i + 1];
            if (isinf(lre) && lre < 0) {
                eloc_out[2 * i] = NAN; eloc_out[2 * i + 1] = NAN;
                if (scale_out) scale_out[i] = NAN;
                continue;
            }
            det_t d = {{rows[2 * i], rows[2 * i + 1]}};
            apply_hamiltonian(n, h1, h2, e_core, &d, &c);
            qsort(c.list, (size_t)c.n_list, sizeof(int64_t), cmp_i64);
            long double sr = 0, cr = 0, si = 0, ci = 0, sa = 0;
            for (int64_t t = 0; t < c.n_list; ++t) {
                int64_t idx = c.list[t];
                long double h = c.acc[idx];
                long double mag = expl((long double)logpsi[2 * idx] - (long double)lre);
                long double ph = (long double)logpsi[2 * idx + 1] - (long double)lim;
                neumaier(&sr, &cr, h * mag * cosl(ph));
                neumaier(&si, &ci, h * mag * sinl(ph));
                sa += fabsl(h) * mag;
            }
            if (scale_out) scale_out[i] = (double)sa;
            eloc_out[2 * i] = (double)(sr + cr);
            eloc_out[2 * i + 1] = (double)(si + ci);
            ctx_reset(&c);
        }
        ctx_free(&c);
    }
    return rc;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
