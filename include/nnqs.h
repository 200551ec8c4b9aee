/*
 * nnqs.h -- C-ABI of libnnqs: the local-energy hot path of NNQS-Transformer
 * (arXiv 2306.16705) on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n (arXiv 2306.16705 LaTeX source).
 *
 * The path (Sec. 3.4; stages 2-4 of Sec. 3.2):
 *   nnqs_ham_compress    Eq. (9) integrals -> JW Pauli table grouped by flip
 *                        mask with fused coefficients (Fig. 6(c), Algorithm 1,
 *                        P:309-363).  Host, once per molecule.
 *   nnqs_table_prepare   the unique-sample lookup table ("bits of a
 *                        64-bit integer ... two integers") + psi table (wf_lut,
 *                        P:383).  Device.
 *   nnqs_local_energy    E_loc(x) = sum_x' H_xx' psi(x')/psi(x), Eq. (4)
 *                        (P:139-141), fused entry evaluation,
 *                        sample-aware: x' not in the table contributes 0
 *                        (P:379); Algorithm 2.  Device.
 *   nnqs_chunk_work      per-chunk work estimate for cost-balanced rank
 *                        slices (the data-centric split).  Device.
 *   nnqs_energy_reduce   count-weighted mean and variance, Eq. (6)
 *                        over unique samples with weights.  Device.
 *
 * Conventions:
 *   - Spin orbital (p, s) of spatial orbital p, spin s (0 = alpha, 1 = beta) is
 *     qubit 2p+s (0-indexed reading of P:287).  Occupied = bit 1.
 *   - Configuration keys are uint64[2]: word0 = qubits 0..63, word1 = qubits
 *     64..127; tables are strictly increasing as 128-bit integers
 *     (compare word1, then word0).  N = n_spin_orbitals <= 128.
 *   - Pauli table: H = sum_k sum_{i in group k} d_i X^{X_k} Z^{Z_i}, where
 *     X^a Z^b flips the bits a after applying the sign (-1)^{popc(x & b)}; so
 *     <x ^ X_k | H | x> = sum_i d_i (-1)^{popc(x & Z_i)}.  d_i is Algorithm 1's
 *     fused coefficient c_i * Re((-i)^{Y_occ}) with the sign reading
 *     R1 (Algorithm 2's literal "(sum & 1) ? 1 : -1", builds -H).
 *   - log psi is complex, (Re, Im) interleaved float64; Re may be -inf (psi = 0).
 *
 * Memory: "host" / "device" is stated per pointer.  Device pointers are
 * borrowed for the duration of a stream-ordered call only.  Handles own all
 * their memory.  Every call returns a status; errors never abort the process.
 * The message of the last error on the calling thread is nnqs_last_error().
 */
#ifndef NNQS_H
#define NNQS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    NNQS_OK = 0,
    NNQS_E_ARG = -1,       /* null / inconsistent argument */
    NNQS_E_SIZE = -2,      /* N odd, N > 128, exact mode with N > 30, n < 0 */
    NNQS_E_SYMMETRY = -3,  /* h1 not symmetric / h2 not 8-fold symmetric (1e-12 rel) */
    NNQS_E_TABLE = -4,     /* keys not strictly increasing, rows out of range */
    NNQS_E_ZERO_PSI = -5,  /* some row has psi(x) = 0: its E_loc is NaN, others valid */
    NNQS_E_CUDA = -6,      /* CUDA runtime error */
    NNQS_E_NOMEM = -7,     /* host or device allocation failed */
    NNQS_E_EMPTY = -8,     /* sum of counts == 0 (Eq. 6 undefined) */
    NNQS_E_ODD_Y = -9      /* Pauli input: odd-Y term with |Re c| > tol (SPEC reading) */
};

/* thread-local, static storage; "" if no error yet */
const char *nnqs_last_error(void);
/* library version / build string */
const char *nnqs_version(void);

typedef struct nnqs_ham_s *nnqs_ham;     /* immutable after creation; owns host + device copies */
typedef struct nnqs_table_s *nnqs_table; /* owns its device copies; borrows nothing */

/*
 * nnqs_ham_compress -- Eq. (9) under Jordan-Wigner
 * into the grouped table of Fig. 6(c) (Algorithm 1).
 *   h1  host f64[n*n], row-major h_pq (n = n_spin_orbitals/2 spatial orbitals)
 *   h2  host f64[n^4], chemists' (pq|rs) at ((p*n+q)*n+r)*n+s; the Eq. (9)
 *       two-body term is 1/2 sum (pq|rs) a+_{ps} a+_{rt} a_{st} a_{qs}
 *   e_core  constant (nuclear repulsion / frozen core) -> identity string
 *   tol     drop strings with |d| <= tol (0 keeps every non-zero)
 *   device  CUDA device ordinal that receives the device copy; device < 0
 *           builds a host-only handle (info / export only, no CUDA calls)
 * Validates symmetry (NNQS_E_SYMMETRY) and N (NNQS_E_SIZE).  Copies h1/h2; the
 * caller keeps ownership.  Groups are ascending by 128-bit X, strings within a
 * group ascending by Z.  The handle records that H conserves N_alpha and N_beta.
 */
int nnqs_ham_compress(const double *h1, const double *h2, int n_spin_orbitals, double e_core,
                      double tol, int device, nnqs_ham *out);

/*
 * nnqs_ham_from_pauli -- Algorithm 1 on an explicit Pauli list
 * (Fig. 6(a)): string i has X/Y mask xmask[i] (host u64[n][2]), Y/Z
 * mask zmask[i] (host u64[n][2]) and complex coefficient (coeff_re, coeff_im)
 * (host f64[n]); fused d = Re(c) * Re((-i)^{Y_occ}).  Duplicate strings are
 * summed.  Odd Y_occ with |Re c| > tol -> NNQS_E_ODD_Y.  No sector assumption
 * is recorded (every group is evaluated for every row).
 */
int nnqs_ham_from_pauli(const uint64_t *xmask, const uint64_t *zmask, const double *coeff_re,
                        const double *coeff_im, int64_t n_terms, int n_qubits, double tol,
                        int device, nnqs_ham *out);

/* counts and device footprint (any pointer may be NULL) */
int nnqs_ham_info(nnqs_ham h, int *n_qubits, int64_t *n_groups, int64_t *n_terms,
                  int64_t *device_bytes);

/*
 * Export the grouped table to host buffers sized from nnqs_ham_info:
 *   xmask u64[K][2], offsets i64[K+1] (offsets[0] = 0, CSR), zmask u64[Nh][2],
 *   coeff f64[Nh] (fused d_i).  Any pointer may be NULL.
 */
int nnqs_ham_export(nnqs_ham h, uint64_t *xmask, int64_t *offsets, uint64_t *zmask, double *coeff);
int nnqs_ham_free(nnqs_ham h);

/*
 * Per-table options (no process-wide state: every knob lives in the table).
 *   algorithm    0 (NNQS_ALGO_AUTO): table rows (rows == NULL) of a sample-aware
 *                table over a Hamiltonian from nnqs_ham_compress use the
 *                alpha/beta-factorised enumeration (DESIGN.md "structured
 *                path"): the same (row, group) pairs with x' in the table as
 *                the literal loop, found by scanning the table's alpha-/beta-
 *                string lists and probing a deletion-key multimap for heavy
 *                strings; H_xx' is the group's Pauli sum on the in-sector folded
 *                table (R21; diagonal and single-excitation groups in
 *                occupation form, R22), so E_loc agrees with the literal loop to
 *                rounding (R14), not bit for bit.  Every other call (explicit
 *                rows, exact mode, nnqs_ham_from_pauli tables) uses the literal
 *                loop.  1 (NNQS_ALGO_LITERAL): always the literal loop of
 *                Algorithm 2 (every row x every group, sector test, hash lookup).
 *   thr_single   structured path: adjacent alpha strings with more table rows
 *                than this are probed through the deletion multimap instead of
 *                scanned (0 = default 128)
 *   thr_double   same-spin lists longer than this are probed (0 = default 8192)
 *   thr_rowheavy alpha groups with more rows than this take phase (iii) through
 *                the entry-driven join (0 = default 16384; raised to thr_single)
 *   literal_kernel  which kernel runs the literal loop: 0 (NNQS_LIT_AUTO) the
 *                bit-sliced one (32 rows x 32 groups per sector test, per-spin
 *                string filter before the lookup) on sample-aware tables of a
 *                number-conserving H, else the staged one; 1 (NNQS_LIT_STAGED)
 *                the group-tile-staged one-row-per-thread kernel; 2
 *                (NNQS_LIT_PLAIN) the unstaged one.  All three visit every
 *                (row, group) pair in ascending k with the same arithmetic:
 *                bit-identical results.
 * The thresholds change the work split, never the hit set or a row's value
 * beyond rounding order.  nnqs_options_default fills the defaults.
 */
#define NNQS_ALGO_AUTO 0
#define NNQS_ALGO_LITERAL 1
#define NNQS_LIT_AUTO 0
#define NNQS_LIT_STAGED 1
#define NNQS_LIT_PLAIN 2
typedef struct {
    int32_t algorithm;
    int32_t thr_single;
    int32_t thr_double;
    int32_t thr_rowheavy;
    int32_t literal_kernel;
    int32_t reserved[11];   /* must be zero */
} nnqs_options;
void nnqs_options_default(nnqs_options *opt);

/*
 * nnqs_table_prepare -- the lookup tables of Algorithm 2 (id_lut / wf_lut,
 * P:383): validates strict 128-bit order, builds psi_hat(y) =
 * exp(logpsi(y) - s), s = max Re logpsi, and a GF(2)-linear hash index over the
 * keys (the lookup that replaces binary_find); sample-aware tables over a
 * spin-conserving Hamiltonian also get the alpha/beta string index of the
 * structured path (CSR by alpha / beta string, adjacent-alpha lists, deletion
 * multimap).
 *   mode 0 (sample-aware): keys device u64[n][2] (sorted), logpsi device f64[n][2]
 *   mode 1 (exact): keys == NULL, n = 2^N (N <= 30), logpsi indexed by configuration
 *   opt          NULL = defaults (nnqs_options_default)
 *   cuda_stream  cudaStream_t (NULL = legacy default stream); keys / logpsi are
 *                read in stream order; the table copies what it keeps.
 * The table owns its device memory and two private CUDA streams (used inside
 * nnqs_local_energy, joined back by events).  It records an event after every
 * call that uses it; nnqs_table_free orders the release after that event on a
 * private stream, so the caller's streams need not outlive the table.  A table
 * may be used by one call at a time (calls on one thread, or serialised).
 * Synchronises cuda_stream (table sizes); returns NNQS_E_TABLE if the order
 * check fails, NNQS_E_NOMEM / NNQS_E_CUDA on device errors (nothing leaks).
 */
int nnqs_table_prepare(nnqs_ham h, int mode, const uint64_t *keys, const double *logpsi,
                       int64_t n, void *cuda_stream, nnqs_table *out);
int nnqs_table_prepare_ex(nnqs_ham h, int mode, const uint64_t *keys, const double *logpsi,
                          int64_t n, const nnqs_options *opt, void *cuda_stream, nnqs_table *out);
int nnqs_table_free(nnqs_table t);
/* the table's algorithm (NNQS_ALGO_*); not concurrently with a call using t */
int nnqs_table_set_algorithm(nnqs_table t, int algorithm);
/* table size and the log-psi shift s (host out; may be NULL) */
int nnqs_table_info(nnqs_table t, int64_t *n, double *shift, int64_t *device_bytes);

/*
 * nnqs_local_energy -- Eq. (4) for n_rows rows (Algorithm 2).
 *   rows == NULL: the rows are table entries [row_begin, row_begin + n_rows)
 *                 (the paper's ist / batch_size_cur_rank; in
 *                 exact mode, the configurations row_begin...);
 *   rows != NULL: explicit device u64[n_rows][2] with row_logpsi device
 *                 f64[n_rows][2] (any configurations).
 *   eloc_out  device f64[n_rows][2] = (Re, Im) E_loc
 *   counts, partials_out  optional (both or neither): counts device i64[n_rows]
 *             (sample weights w); partials_out device
 *             f64[ceil(n_rows/NNQS_REDUCE_CHUNK)][3] receives the first pass of
 *             Eq. (6) per chunk of NNQS_REDUCE_CHUNK rows of this call, (W,
 *             sum w Re E, sum w Im E), fused into the E_loc epilogue: the warp
 *             that completes a chunk's last row reduces the chunk in the fixed
 *             order of nnqs_energy_chunk_partials (bit-identical to it), so
 *             chunk-aligned rank slices combine bit for bit (stage 4).
 *   stats_out optional device i64[4] (zeroed by the caller) accumulating
 *             (row-group pairs, pairs whose x' shares x's particle sector,
 *              lookups that hit, Pauli strings evaluated); NULL to skip.  On the
 *             structured path stats_out[0] is R x K' by definition (the pairs
 *             the enumeration resolves, not a counter), stats_out[1] counts
 *             list entries / probes examined and stats_out[3] folded terms.
 * x' absent from the table contributes zero.  For Hamiltonians from
 * nnqs_ham_compress, groups whose x' leaves x's (N_alpha, N_beta) sector are
 * skipped (their exact H_xx' is 0).  A row with psi(x) = 0 gets NaN; this is
 * reported by nnqs_local_energy_check().  Asynchronous on cuda_stream, except
 * that the structured path synchronises once (size of its entry-driven join).
 * E_loc of a row is bit-identical for any row_begin / n_rows slicing, across
 * runs, and (structured path) independent of the row schedule.
 */
int nnqs_local_energy(nnqs_ham h, nnqs_table t, int64_t row_begin, const uint64_t *rows,
                      const double *row_logpsi, int64_t n_rows, double *eloc_out,
                      const int64_t *counts, double *partials_out, int64_t *stats_out,
                      void *cuda_stream);

/*
 * Profiling aid (not part of the method): cycle counters of the structured
 * kernel's sections, summed over warps, when libnnqs was compiled with
 * -DNNQS_PROFILE (NNQS_NVCC_DEFINES); all zero otherwise.  out: host u64[16]
 * = {diagonal, phase (i), phase (ii), (iii) list scans, (iii) heavy probes,
 * hit flushes, row setup, total}; reset != 0 zeroes the device counters after
 * reading.  Synchronises the device.  Returns NNQS_OK or NNQS_E_CUDA.
 */
int nnqs_debug_counters(uint64_t *out, int reset);

/*
 * Work estimate of nnqs_local_energy per chunk of table rows, for cost-balanced
 * contiguous rank slices (the paper's ist / batch_size_cur_rank, P:389, P:425,
 * with slice lengths chosen by work instead of by count: rows near the
 * Hartree-Fock string couple to far more table entries than the rest, and the
 * sorted table puts them together).  work_out: host i64[ceil(n/chunk)], chunk c
 * covering rows [c*chunk, min((c+1)*chunk, n)); relative units (list lengths
 * the row kernels scan, fixed costs for probed lists and join rows; the literal
 * Algorithm 2 path: rows per chunk).  floor_out (NULL to skip): host
 * i64[ceil(n/chunk)], in the same units, the largest single-row latency floor in
 * the chunk (one warp evaluates one row: a row whose alpha and beta lists are
 * both probed, the Hartree-Fock row, bounds its slice's time from below); 0 on
 * the literal path.  Deterministic for a given table, so every rank derives the
 * same slices.  Synchronises cuda_stream.  NNQS_E_ARG on bad arguments
 * (chunk <= 0), NNQS_E_CUDA on a launch or copy failure.
 */
int nnqs_chunk_work(nnqs_table t, int64_t chunk, int64_t *work_out, int64_t *floor_out, void *cuda_stream);

/* Synchronises cuda_stream; NNQS_E_ZERO_PSI if any of eloc (device f64[n][2]) is NaN. */
int nnqs_local_energy_check(const double *eloc, int64_t n, void *cuda_stream);

/*
 * Energy reduction, Eq. (6) with weights:
 *   mean = sum w E / W,  var = sum w |E - mean|^2 / W,  W = sum w  (two passes,
 *   population variance).  Chunks of NNQS_REDUCE_CHUNK rows are reduced in a
 *   fixed tree order and combined in ascending chunk order, so results are
 *   bit-identical however the rows are split over devices (chunk-aligned).
 *
 * nnqs_energy_chunk_partials: partials device f64[n_chunks][3],
 *   n_chunks = ceil(n / NNQS_REDUCE_CHUNK);  mean_dev == NULL: pass 1,
 *   (W, sum w Re E, sum w Im E) per chunk;  mean_dev device f64[2]: pass 2,
 *   (W, sum w |E - mean|^2, 0) per chunk.  eloc device f64[n][2], counts device i64[n].
 * nnqs_energy_combine: partials device f64[n_chunks][3] -> out_dev device f64[4]:
 *   pass 1: (mean_re, mean_im, W, 0);  pass 2: (var, W, 0, 0).
 * nnqs_energy_reduce: single-device convenience, out host f64[4] =
 *   (mean_re, mean_im, var, W); synchronises; NNQS_E_EMPTY if W == 0.
 */
#define NNQS_REDUCE_CHUNK 1024
int nnqs_energy_chunk_partials(const double *eloc, const int64_t *counts, int64_t n,
                               const double *mean_dev, double *partials, void *cuda_stream);
int nnqs_energy_combine(const double *partials, int64_t n_chunks, int pass, double *out_dev,
                        void *cuda_stream);
int nnqs_energy_reduce(const double *eloc, const int64_t *counts, int64_t n, double out[4],
                       void *cuda_stream);

/*
 * Gradient weights of Eq. (7): with
 * ln Psi* = ln|Psi| - i phi, the estimator 2 Re E_p[(E_loc - E) grad ln Psi*]
 * over the unique samples with counts w_u is sum_u a_u grad ln|Psi(x_u)| +
 * b_u grad phi(x_u), where
 *   a_u = 2 w_u Re(E_loc(x_u) - mean) / W,   b_u = 2 w_u Im(E_loc(x_u) - mean) / W.
 * eloc device f64[n][2], counts device i64[n], energy_dev device f64[3] =
 * (mean_re, mean_im, W) -- e.g. nnqs_energy_combine's pass-1 output, global over
 * all ranks; ab_out device f64[n][2] = (a_u, b_u).  Stream-ordered;
 * NNQS_E_ARG on bad arguments.  The ansatz backward that consumes the weights
 * is outside this library.
 */
int nnqs_grad_weights(const double *eloc, const int64_t *counts, int64_t n, const double *energy_dev,
                      double *ab_out, void *cuda_stream);

/*
 * Parity/debug (small inputs): every (row, group) whose x' = x ^ X_k is found
 * in the table, with its index and H_xx', by the literal loop (Algorithm 2,
 * P:399-418).  rows: host u64[n_rows][2].  Outputs host arrays of capacity
 * max_pairs; n_pairs_out = number found (may exceed max_pairs, then
 * NNQS_E_SIZE).  Order unspecified.
 */
int nnqs_coupled_debug(nnqs_ham h, nnqs_table t, const uint64_t *rows_host, int64_t n_rows,
                       int64_t max_pairs, int64_t *row_id, int64_t *group_id, uint64_t *xprime,
                       int64_t *table_idx, double *h_xxp, int64_t *n_pairs_out);

/*
 * Parity/debug of the production path (P3 of DESIGN.md Sec. 4): runs exactly
 * the launch sequence nnqs_local_energy uses for the table rows
 * [row_begin, row_begin + n_rows) (the table's algorithm; the structured
 * kernels with their multimap probes, entry-driven join and occupation forms)
 * with a hit log enabled, and returns every hit those kernels evaluate:
 * row_id = table index of the row, table_idx = table index of x' (the lookup
 * index), xprime = the key of x' (read from the table), group_id = k with
 * X_k = x ^ x' (host search of the grouped table, -1 if X is not a group),
 * h_xxp = the H_xx' the kernel multiplied with psi(x') (the diagonal x' = x
 * included).  Host outputs of capacity max_pairs (any may be NULL);
 * n_pairs_out = hits found (> max_pairs: NNQS_E_SIZE, the first max_pairs in
 * unspecified order are written).  Synchronises; for tests on small slices.
 */
int nnqs_coupled_debug_rows(nnqs_ham h, nnqs_table t, int64_t row_begin, int64_t n_rows, int64_t max_pairs,
                            int64_t *row_id, int64_t *group_id, uint64_t *xprime, int64_t *table_idx,
                            double *h_xxp, int64_t *n_pairs_out);

/*
 * nnqs_bas_layer -- one local sampling step of batch autoregressive sampling
 * (BAS, Fig. 3(b); stage 1 of the data-centric iteration).
 * Input: the m unique prefixes of the current layer (device keys u64[m][2] in
 * the sample-key layout: qubit 2p = spin-up orbital p, 2p+1 = spin-down; only
 * orbitals > `orbital` set), their weights (device i64[m], >= 0) and the model's
 * conditional distribution over the next two qubits (device f64[m][4], outcome
 * o: up bit o & 1, down bit o >> 1; unnormalised values are fine).  Orbitals are
 * sampled from n_orbitals - 1 down to 0 (the reverse qubit order).
 * Each prefix's weight w is split among its 4 children by a multinomial draw of
 * exactly w samples from the masked, renormalised distribution (Eq. 12, P:290:
 * outcomes exceeding n_up / n_dn are zeroed; so are outcomes that can no longer
 * reach them -- DESIGN.md R24), as a chain of conditional binomials with
 * uniforms from a counter-based generator keyed by (seed, orbital, prefix key):
 * a node's children depend on the node alone, so any split of a layer over
 * ranks (parallel BAS) reproduces the serial result exactly.
 * Output: the children with weight > 0 (zero-weight leaves pruned),
 * device keys_out u64[4m][2] / counts_out i64[4m] (capacity 4m), in (parent,
 * outcome) order -- ascending keys when the input is ascending; *m_out (host)
 * = how many.  Synchronises cuda_stream.  Errors: NNQS_E_ARG (bad pointers, or
 * a prefix with weight > 0 and no feasible outcome), NNQS_E_SIZE (orbital
 * outside [0, n_orbitals), n_orbitals > 64, m >= 2^29), NNQS_E_NOMEM/_CUDA.
 */
int nnqs_bas_layer(const uint64_t *keys, const int64_t *counts, const double *probs, int64_t m, int orbital,
                   int n_orbitals, int n_up, int n_dn, uint64_t seed, uint64_t *keys_out, int64_t *counts_out,
                   int64_t *m_out, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* NNQS_H */
