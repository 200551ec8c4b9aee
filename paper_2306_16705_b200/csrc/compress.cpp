// compress.cpp -- host side of nnqs_ham_compress / nnqs_ham_from_pauli.
//
// Builds the grouped Pauli table of Fig. 6(c) (Algorithm 1,
// PAPER.md:319-363) for the JW image of Eq. (9)
// (PAPER.md:174-176).  Instead of expanding O(N^4) symbolic Pauli products
// and merging them in a dictionary, every flip group is generated directly:
// for a flip mask X the off-diagonal function f_X(x) = <x^X|H|x> is, by the
// Slater-Condon rules, (JW string) x (a function of a few occupation bits), and
// its Walsh expansion f_X(x) = sum_Z d(X,Z) (-1)^{popc(x&Z)} IS the fused
// coefficient list of the group (d = c * Re((-i)^{Y_occ})).
//
//   X = 0            f = H_xx = e_core + sum_P eps_P n_P + sum_{P<Q} V_PQ n_P n_Q
//   X = {P,Q}        f = [x_P != x_Q] (-1)^{popc(x & (P,Q))} (h_pq + sum_R W_R n_R)
//   X = {S0<..<S3}   f = (-1)^{popc(x & ((S0,S1) u (S2,S3)))} g(x_S0..x_S3)
// with n_R = (1 - Z_R)/2.  4-site coefficients are carried as integer
// combinations of the three distinct integrals of the site set, so the
// structural zeros of the Walsh transform are exact zeros.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "internal.h"

namespace {

struct Builder {
    std::vector<u64> gx;            // [2 * groups]
    std::vector<int64_t> gstart;    // first term
    std::vector<int32_t> gcount;
    std::vector<u64> tz;            // [2 * terms]
    std::vector<double> td;
    double tol = 0.0;

    void begin(u64 x0, u64 x1) {
        gx.push_back(x0);
        gx.push_back(x1);
        gstart.push_back((int64_t)td.size());
        gcount.push_back(0);
    }
    void add(u64 z0, u64 z1, double d) {
        if (!(std::fabs(d) > tol)) return;
        tz.push_back(z0);
        tz.push_back(z1);
        td.push_back(d);
        gcount.back() += 1;
    }
    void end() {
        if (gcount.back() == 0) {
            gx.pop_back();
            gx.pop_back();
            gstart.pop_back();
            gcount.pop_back();
        }
    }
};

inline void set_bit(u64 &lo, u64 &hi, int j) {
    if (j < 64) lo ^= 1ULL << j;
    else hi ^= 1ULL << (j - 64);
}

// bits strictly between a < b
inline void between(int a, int b, u64 &lo, u64 &hi) {
    lo = hi = 0;
    for (int j = a + 1; j < b; ++j) set_bit(lo, hi, j);
}

struct Ints {
    const double *h1, *h2;
    int n;
    double e(int p, int q) const { return h1[(size_t)p * n + q]; }
    double g(int p, int q, int r, int s) const {
        return h2[(((size_t)p * n + q) * n + r) * n + s];
    }
};

// ---------------------------------------------------------------- X = 0
void diagonal_group(const Ints &I, int N, double e_core, Builder &b) {
    std::vector<double> eps(N), V((size_t)N * N, 0.0);
    for (int P = 0; P < N; ++P) eps[P] = I.e(P >> 1, P >> 1);
    for (int P = 0; P < N; ++P)
        for (int Q = P + 1; Q < N; ++Q) {
            int p = P >> 1, q = Q >> 1;
            double v = I.g(p, p, q, q);
            if ((P & 1) == (Q & 1)) v -= I.g(p, q, q, p);
            V[(size_t)P * N + Q] = V[(size_t)Q * N + P] = v;
        }
    b.begin(0, 0);
    double c0 = e_core;
    for (int P = 0; P < N; ++P) c0 += 0.5 * eps[P];
    for (int P = 0; P < N; ++P)
        for (int Q = P + 1; Q < N; ++Q) c0 += 0.25 * V[(size_t)P * N + Q];
    b.add(0, 0, c0);
    for (int P = 0; P < N; ++P) {
        double c = -0.5 * eps[P];
        for (int Q = 0; Q < N; ++Q)
            if (Q != P) c -= 0.25 * V[(size_t)P * N + Q];
        u64 lo = 0, hi = 0;
        set_bit(lo, hi, P);
        b.add(lo, hi, c);
    }
    for (int P = 0; P < N; ++P)
        for (int Q = P + 1; Q < N; ++Q) {
            u64 lo = 0, hi = 0;
            set_bit(lo, hi, P);
            set_bit(lo, hi, Q);
            b.add(lo, hi, 0.25 * V[(size_t)P * N + Q]);
        }
    b.end();
}

// ---------------------------------------------------------- X = {P, Q}
void two_site_group(const Ints &I, int N, int P, int Q, Builder &b, std::vector<double> &W) {
    const int p = P >> 1, q = Q >> 1, sg = P & 1;
    double h = I.e(p, q);
    bool any = h != 0.0;
    for (int R = 0; R < N; ++R) {
        W[R] = 0.0;
        if (R == P || R == Q) continue;
        int r = R >> 1;
        double w = I.g(p, q, r, r);
        if ((R & 1) == sg) w -= I.g(p, r, r, q);
        W[R] = w;
        any |= w != 0.0;
    }
    if (!any) return;
    double C = h;
    for (int R = 0; R < N; ++R)
        if (R != P && R != Q) C += 0.5 * W[R];
    u64 x0 = 0, x1 = 0;
    set_bit(x0, x1, P);
    set_bit(x0, x1, Q);
    u64 m0, m1;
    between(P, Q, m0, m1);
    b.begin(x0, x1);
    b.add(m0, m1, 0.5 * C);
    b.add(m0 ^ x0, m1 ^ x1, -0.5 * C);
    for (int R = 0; R < N; ++R) {
        if (R == P || R == Q) continue;
        u64 r0 = 0, r1 = 0;
        set_bit(r0, r1, R);
        b.add(m0 ^ r0, m1 ^ r1, -0.25 * W[R]);
        b.add(m0 ^ r0 ^ x0, m1 ^ r1 ^ x1, 0.25 * W[R]);
    }
    b.end();
}

// ------------------------------------------------ X = {S0 < S1 < S2 < S3}
inline int pairing_id(int u, int v) {       // pairing of {0,1,2,3} containing (u, v)
    int partner0 = (u == 0) ? v : (v == 0) ? u : 6 - u - v;
    return partner0 - 1;
}

struct FourSiteTables {
    // per pattern (4-bit, 2 set): sign-folded integer vectors over the 3 atoms
    int coef[16][3];
    bool valid[16];
};

// JW sign, restricted to the four sites, of a+_a a+_b a_j a_i on local state st
inline int local_sign(int st, int i, int j, int a, int bb) {
    int s = 0;
    s ^= __builtin_popcount(st & ((1 << i) - 1)) & 1; st &= ~(1 << i);
    s ^= __builtin_popcount(st & ((1 << j) - 1)) & 1; st &= ~(1 << j);
    s ^= __builtin_popcount(st & ((1 << bb) - 1)) & 1; st |= 1 << bb;
    s ^= __builtin_popcount(st & ((1 << a) - 1)) & 1; st |= 1 << a;
    return s;
}

void four_site_group(const Ints &I, const int S[4], Builder &b, long &odd_violations) {
    int o[4], sp[4];
    for (int t = 0; t < 4; ++t) { o[t] = S[t] >> 1; sp[t] = S[t] & 1; }
    const double A[3] = {I.g(o[0], o[1], o[2], o[3]), I.g(o[0], o[2], o[1], o[3]),
                         I.g(o[0], o[3], o[1], o[2])};
    if (A[0] == 0.0 && A[1] == 0.0 && A[2] == 0.0) return;
    int g[16][3];
    std::memset(g, 0, sizeof(g));
    for (int pat = 0; pat < 16; ++pat) {
        if (__builtin_popcount(pat) != 2) continue;
        int occ[2], emp[2], no = 0, ne = 0;
        for (int t = 0; t < 4; ++t) {
            if (pat >> t & 1) occ[no++] = t; else emp[ne++] = t;
        }
        const int i = occ[0], j = occ[1], a = emp[0], bb = emp[1];
        // <x'|H|x> = ([ai|bj] - [aj|bi]) <x'| a+_a a+_b a_j a_i |x>
        int c[3] = {0, 0, 0};
        if (sp[a] == sp[i] && sp[bb] == sp[j]) c[pairing_id(a, i)] += 1;
        if (sp[a] == sp[j] && sp[bb] == sp[i]) c[pairing_id(a, j)] -= 1;
        const int s = local_sign(pat, i, j, a, bb);
        for (int k = 0; k < 3; ++k) g[pat][k] = s ? -c[k] : c[k];
    }
    u64 x0 = 0, x1 = 0;
    for (int t = 0; t < 4; ++t) set_bit(x0, x1, S[t]);
    u64 m0, m1, n0, n1;
    between(S[0], S[1], m0, m1);
    between(S[2], S[3], n0, n1);
    m0 |= n0;
    m1 |= n1;
    b.begin(x0, x1);
    for (int z = 0; z < 16; ++z) {
        int cz[3] = {0, 0, 0};
        for (int pat = 0; pat < 16; ++pat) {
            int sgn = (__builtin_popcount(pat & z) & 1) ? -1 : 1;
            for (int k = 0; k < 3; ++k) cz[k] += sgn * g[pat][k];
        }
        if (__builtin_popcount(z) & 1) {   // odd Y_occ: zero by hermiticity (reading R3)
            if (cz[0] || cz[1] || cz[2]) ++odd_violations;
            continue;
        }
        if (!cz[0] && !cz[1] && !cz[2]) continue;
        double d = ((double)cz[0] * A[0] + (double)cz[1] * A[1] + (double)cz[2] * A[2]) / 16.0;
        u64 z0 = m0, z1 = m1;
        for (int t = 0; t < 4; ++t)
            if (z >> t & 1) set_bit(z0, z1, S[t]);
        b.add(z0, z1, d);
    }
    b.end();
}

bool less128(u64 a0, u64 a1, u64 b0, u64 b1) { return a1 != b1 ? a1 < b1 : a0 < b0; }

void assemble(std::vector<Builder> &bs, int n_qubits, HostTable &out) {
    struct Ref { u64 x0, x1; int b; int64_t g; };
    std::vector<Ref> refs;
    size_t nt = 0;
    for (int t = 0; t < (int)bs.size(); ++t) {
        for (size_t g = 0; g < bs[t].gstart.size(); ++g)
            refs.push_back({bs[t].gx[2 * g], bs[t].gx[2 * g + 1], t, (int64_t)g});
        nt += bs[t].td.size();
    }
    std::sort(refs.begin(), refs.end(), [](const Ref &a, const Ref &b) {
        return less128(a.x0, a.x1, b.x0, b.x1);
    });
    out.n_qubits = n_qubits;
    out.x.resize(2 * refs.size());
    out.off.resize(refs.size() + 1);
    out.z.resize(2 * nt);
    out.d.resize(nt);
    int64_t pos = 0;
    std::vector<int64_t> perm;
    for (size_t k = 0; k < refs.size(); ++k) {
        const Builder &B = bs[refs[k].b];
        int64_t s = B.gstart[refs[k].g], c = B.gcount[refs[k].g];
        out.x[2 * k] = refs[k].x0;
        out.x[2 * k + 1] = refs[k].x1;
        out.off[k] = pos;
        perm.resize(c);
        std::iota(perm.begin(), perm.end(), s);
        std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
            return less128(B.tz[2 * a], B.tz[2 * a + 1], B.tz[2 * b], B.tz[2 * b + 1]);
        });
        for (int64_t i = 0; i < c; ++i) {
            out.z[2 * (pos + i)] = B.tz[2 * perm[i]];
            out.z[2 * (pos + i) + 1] = B.tz[2 * perm[i] + 1];
            out.d[pos + i] = B.td[perm[i]];
        }
        pos += c;
    }
    out.off[refs.size()] = pos;
}

}  // namespace

int nnqs_compress_host(const double *h1, const double *h2, int n, double e_core, double tol,
                       HostTable &out) {
    const int N = 2 * n;
    Ints I{h1, h2, n};
    int nthreads = 1;
#ifdef _OPENMP
    nthreads = omp_get_max_threads();
#endif
    std::vector<Builder> bs(nthreads + 1);
    for (auto &b : bs) b.tol = tol;
    long odd_violations = 0;
    diagonal_group(I, N, e_core, bs[nthreads]);
    // 2-site groups X = {P, Q}, same spin
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : odd_violations)
    for (int P = 0; P < N; ++P) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        std::vector<double> W(N);
        for (int Q = P + 2; Q < N; Q += 2) two_site_group(I, N, P, Q, bs[tid], W);
        // 4-site same-spin groups with lowest site P
        const int sg = P & 1, p1 = P >> 1;
        for (int p2 = p1 + 1; p2 < n; ++p2)
            for (int p3 = p2 + 1; p3 < n; ++p3)
                for (int p4 = p3 + 1; p4 < n; ++p4) {
                    int S[4] = {2 * p1 + sg, 2 * p2 + sg, 2 * p3 + sg, 2 * p4 + sg};
                    four_site_group(I, S, bs[tid], odd_violations);
                }
    }
    // 4-site opposite-spin groups: alpha pair (p<q) x beta pair (r<s)
    const int npair = n * (n - 1) / 2;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads) reduction(+ : odd_violations)
    for (int a = 0; a < npair; ++a) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        int p = 0, rem = a;
        while (rem >= n - 1 - p) { rem -= n - 1 - p; ++p; }
        int q = p + 1 + rem;
        for (int r = 0; r < n; ++r)
            for (int s = r + 1; s < n; ++s) {
                int S[4] = {2 * p, 2 * q, 2 * r + 1, 2 * s + 1};
                std::sort(S, S + 4);
                four_site_group(I, S, bs[tid], odd_violations);
            }
    }
    if (odd_violations)
        return nnqs_set_error(NNQS_E_SYMMETRY, "internal: odd-Y Walsh coefficient not structurally zero");
    assemble(bs, N, out);
    out.conserving = true;
    return NNQS_OK;
}

int nnqs_from_pauli_host(const u64 *xm, const u64 *zm, const double *cre, const double *cim,
                         int64_t n_terms, int n_qubits, double tol, HostTable &out) {
    (void)cim;
    struct T { u64 x0, x1, z0, z1; double d; };
    std::vector<T> ts;
    ts.reserve(n_terms);
    for (int64_t i = 0; i < n_terms; ++i) {
        u64 x0 = xm[2 * i], x1 = xm[2 * i + 1], z0 = zm[2 * i], z1 = zm[2 * i + 1];
        if (n_qubits < 128) {
            u64 lim0 = n_qubits >= 64 ? ~0ULL : ((1ULL << n_qubits) - 1);
            u64 lim1 = n_qubits <= 64 ? 0ULL : ((1ULL << (n_qubits - 64)) - 1);
            if ((x0 & ~lim0) || (x1 & ~lim1) || (z0 & ~lim0) || (z1 & ~lim1))
                return nnqs_set_error(NNQS_E_ARG, "Pauli mask has bits beyond n_qubits (term " +
                                                      std::to_string(i) + ")");
        }
        int ny = __builtin_popcountll(x0 & z0) + __builtin_popcountll(x1 & z1);
        if (ny & 1) {
            if (std::fabs(cre[i]) > tol)
                return nnqs_set_error(NNQS_E_ODD_Y, "odd Y count with |Re c| > tol at term " +
                                                        std::to_string(i));
            continue;
        }
        // Algorithm 1: coeff <- Re(c) * Re((-i)^{Y_occ})
        double d = (ny & 2) ? -cre[i] : cre[i];
        ts.push_back({x0, x1, z0, z1, d});
    }
    std::sort(ts.begin(), ts.end(), [](const T &a, const T &b) {
        if (a.x1 != b.x1) return a.x1 < b.x1;
        if (a.x0 != b.x0) return a.x0 < b.x0;
        return less128(a.z0, a.z1, b.z0, b.z1);
    });
    // merge duplicates
    std::vector<T> m;
    for (auto &t : ts) {
        if (!m.empty() && m.back().x0 == t.x0 && m.back().x1 == t.x1 && m.back().z0 == t.z0 &&
            m.back().z1 == t.z1)
            m.back().d += t.d;
        else
            m.push_back(t);
    }
    Builder b;
    b.tol = tol;
    for (size_t i = 0; i < m.size();) {
        size_t j = i;
        b.begin(m[i].x0, m[i].x1);
        while (j < m.size() && m[j].x0 == m[i].x0 && m[j].x1 == m[i].x1) {
            b.add(m[j].z0, m[j].z1, m[j].d);
            ++j;
        }
        b.end();
        i = j;
    }
    std::vector<Builder> bs(1, b);
    assemble(bs, n_qubits, out);
    out.conserving = false;
    return NNQS_OK;
}
