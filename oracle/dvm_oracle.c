/*
 * dvm_oracle.c -- CPU ORACLE for the periodized, direction-truncated DVM
 * collision operator D^{Ñ,N̄}(f,f) of Mouhot, Pareschi & Rey (arXiv 1201.3986).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load or call it.  It shares no source, header, table or helper with the
 * CUDA library under paper_1201_3986_b200/ and must never be linked into it.
 *
 * What it computes (a plain direct double sum, written out from the paper):
 *
 *   eq:DR with the Carleman kernel of PAPER.md:355-365,
 *   the decoupled weights of eq:decoup and the direction
 *   truncation of beta^{N̄} / eq:decD:
 *
 *   Q_i = sum_{k in [-Ñ,Ñ]^d, k != 0, ||k/gcd(k)||_inf <= N̄}
 *         sum_{l in [-Ñ,Ñ]^d, k.l = 0}
 *             a(k) * ( f_{i+k} f_{i+l} - f_i f_{i+k+l} )        (indices mod N)
 *
 *   a(k) = h^{d+1} |k|_2 / gcd(|k_1|,...,|k_d|),   b(l) = 1,    h = 2L/N
 *
 *   dvm_oracle_collide_w takes general decoupled weights instead (eq:decoup,
 *   B̃(|k|,|l|) w_{k,l} = a(k) b(l)): caller-given a(k) and
 *   b(l) tabulated over the box [-Ñ,Ñ]^d, and Γ̃_{k,l} = a(k) b(l) on the same
 *   truncated pair set.
 *
 *   - "−Ñ ≤ k,l ≤ Ñ" is read componentwise (multi-index convention,
 *     PAPER.md:372-373): DESIGN.md reading R8.
 *   - A nonzero k lies on exactly one line e Z through 0, e = ±k/gcd(k); the
 *     fast operator keeps line e iff e is a "primal representant" of order
 *     ||e||_inf <= N̄ and then keeps every multiple of e in
 *     the box and every l of e^⊥ in the box (not
 *     truncated by N̄): DESIGN.md readings R7, R9.
 *   - k = 0 contributes nothing: a(0) := 0 (reading R6; the bracket vanishes
 *     anyway).
 *   - Periodic indices: reading R10.
 *   - No extra physical prefactor: Γ̃_{k,l} = a(k) b(l) exactly as printed
 *     (reading R5).
 *
 * Algorithm (step by step, no blocking, fusion or reordering):
 *   1. Build the pair list by brute force: k in lexicographic order over the
 *      box, then l in lexicographic order, keeping orthogonal pairs whose k has
 *      an allowed line (optionally restricted to a caller-given subset of lines,
 *      used only to test direction sharding).
 *   2. For every requested node i (OpenMP over nodes; the per-node order is
 *      fixed and independent of the thread count), accumulate with Neumaier
 *      compensated summation:
 *        Q_i  = sum a (f_{i+k} f_{i+l} - f_i f_{i+k+l})
 *        G_i  = sum a  f_{i+k} f_{i+l}                 (gain, diagnostic)
 *        Lo_i = f_i * sum a f_{i+k+l}                  (loss, diagnostic)
 *
 * Layout: f is [ncells][N]...[N] (d axes), row-major, last axis fastest; node
 * index i = sum_j x_j N^{d-1-j}.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC dvm_oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXD 3

static int orc_gcd(int a, int b)
{
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

static int orc_gcd_vec(int d, const int *k)
{
    int g = 0;
    for (int j = 0; j < d; ++j) g = orc_gcd(g, k[j]);
    return g;
}

/* Reading R2: Ñ = max(floor(N/(3+sqrt2)), N̄)
 * states Ñ = [2N/(3+√2)] with N the half-width, which gives Ñ = 1,3,7,14 for
 * N = 8,16,32,64 points. */
int dvm_oracle_ntilde_rule(int N, int Nbar)
{
    int nt = (int)floor((double)N / (3.0 + sqrt(2.0)));
    return nt > Nbar ? nt : Nbar;
}

/* Canonical primitive directions with ||e||_inf <= N̄ ("primal
 * representants"): gcd = 1 and first nonzero component
 * positive.  Brute force over [-N̄,N̄]^d in lexicographic order (reading R7).
 * Returns the count; writes them to dirs[count*d] when dirs != NULL. */
int64_t dvm_oracle_directions(int d, int Nbar, int *dirs)
{
    if (d < 1 || d > ORC_MAXD || Nbar < 0) return -1;
    int side = 2 * Nbar + 1;
    int64_t total = 1;
    for (int j = 0; j < d; ++j) total *= side;
    int64_t count = 0;
    int e[ORC_MAXD];
    for (int64_t c = 0; c < total; ++c) {
        int64_t r = c;
        for (int j = d - 1; j >= 0; --j) {
            e[j] = (int)(r % side) - Nbar;
            r /= side;
        }
        int first = 0;
        for (int j = 0; j < d; ++j)
            if (e[j] != 0) {
                first = e[j];
                break;
            }
        if (first <= 0) continue;                /* zero vector or non-canonical sign */
        if (orc_gcd_vec(d, e) != 1) continue;    /* not primitive */
        if (dirs)
            for (int j = 0; j < d; ++j) dirs[count * d + j] = e[j];
        ++count;
    }
    return count;
}

/* Is k allowed as the "k" of a pair?  Its line must be of order <= N̄, and (if
 * a subset of lines is given) its canonical direction must be in the subset. */
static int orc_k_allowed(int d, const int *k, int Nbar, int ndirs, const int *dirs)
{
    int g = orc_gcd_vec(d, k);
    if (g == 0) return 0; /* k = 0: a(0) := 0 (reading R6) */
    int e[ORC_MAXD];
    int first = 0;
    for (int j = 0; j < d; ++j) {
        e[j] = k[j] / g;
        if (!first && e[j] != 0) first = e[j];
    }
    if (first < 0)
        for (int j = 0; j < d; ++j) e[j] = -e[j];
    for (int j = 0; j < d; ++j)
        if (abs(e[j]) > Nbar) return 0;
    if (ndirs < 0) return 1;
    for (int t = 0; t < ndirs; ++t) {
        int same = 1;
        for (int j = 0; j < d; ++j)
            if (dirs[t * d + j] != e[j]) {
                same = 0;
                break;
            }
        if (same) return 1;
    }
    return 0;
}

/* Index of an offset v in [-Ñ,Ñ]^d in a box table (row-major, last axis fastest). */
static int64_t orc_box_index(int d, int Ntilde, const int *v)
{
    int64_t idx = 0;
    for (int j = 0; j < d; ++j) idx = idx * (2 * Ntilde + 1) + (v[j] + Ntilde);
    return idx;
}

/* Step 1: the pair list.  Returns the number of pairs; fills k[], l[] (npairs*d)
 * and the pair weights w[] when they are non-NULL and cap is large enough.
 * wa/wb NULL: Γ̃_{k,l} = a(k) = h^{d+1}|k|/gcd(k) (b = 1); otherwise
 * Γ̃_{k,l} = wa[k] * wb[l] (eq:decoup), box tables over [-Ñ,Ñ]^d. */
static int64_t orc_pairs(int d, int Ntilde, int Nbar, double h, int ndirs, const int *dirs, const double *wa,
                         const double *wb, int64_t cap, int *kout, int *lout, double *aout)
{
    if (d < 1 || d > ORC_MAXD || Ntilde < 0) return -1;
    int side = 2 * Ntilde + 1;
    int64_t box = 1;
    for (int j = 0; j < d; ++j) box *= side;
    double hd1 = pow(h, d + 1);
    /* the box points in lexicographic order, decoded once */
    int *boxv = (int *)malloc(sizeof(int) * (size_t)(box * d));
    if (!boxv) return -1;
    for (int64_t c = 0; c < box; ++c) {
        int64_t r = c;
        for (int j = d - 1; j >= 0; --j) {
            boxv[c * d + j] = (int)(r % side) - Ntilde;
            r /= side;
        }
    }
    int64_t n = 0;
    for (int64_t ck = 0; ck < box; ++ck) {
        const int *k = boxv + ck * d;
        if (!orc_k_allowed(d, k, Nbar, ndirs, dirs)) continue;
        int g = orc_gcd_vec(d, k);
        double norm = 0.0;
        for (int j = 0; j < d; ++j) norm += (double)k[j] * (double)k[j];
        double a = hd1 * sqrt(norm) / (double)g; /* a(k) = h^{d+1}|k|/gcd(k) */
        if (wa) a = wa[orc_box_index(d, Ntilde, k)];
        for (int64_t cl = 0; cl < box; ++cl) {
            const int *l = boxv + cl * d;
            long dot = 0;
            for (int j = 0; j < d; ++j) dot += (long)k[j] * l[j];
            if (dot != 0) continue; /* 1(k.l) */
            if (n < cap && kout && lout && aout) {
                for (int j = 0; j < d; ++j) {
                    kout[n * d + j] = k[j];
                    lout[n * d + j] = l[j];
                }
                aout[n] = wb ? a * wb[orc_box_index(d, Ntilde, l)] : a;
            }
            ++n;
        }
    }
    free(boxv);
    return n;
}

int64_t dvm_oracle_pairs(int d, int Ntilde, int Nbar, double h, int ndirs, const int *dirs,
                         int64_t cap, int *kout, int *lout, double *aout)
{
    return orc_pairs(d, Ntilde, Nbar, h, ndirs, dirs, NULL, NULL, cap, kout, lout, aout);
}

static inline void neu_add(double *s, double *c, double x)
{
    double t = *s + x;
    if (fabs(*s) >= fabs(x))
        *c += (*s - t) + x;
    else
        *c += (x - t) + *s;
    *s = t;
}

/* Periodic index of node x + o (reading R10) from per-node
 * tables: wrap[j][o_j + 2Ñ] = ((x_j + o_j) mod N) * N^{d-1-j}, filled once per
 * node for every offset |o_j| <= 2Ñ (k, l and k + l all lie in [-2Ñ,2Ñ]^d).
 * The table is only a precomputed "mod N"; the floating-point work and its
 * order are those of the sum written above. */
#define ORC_MAXW (4 * 64 + 1) /* 4Ñ + 1 entries per axis; Ñ <= 64 */
#define ORC_NB 16               /* nodes evaluated side by side per pass over the pair list */
static inline int64_t orc_wrap_index(int d, const int32_t (*wrap)[ORC_MAXW], int twoNt, const int *o)
{
    int64_t idx = 0;
    for (int j = 0; j < d; ++j) idx += wrap[j][o[j] + twoNt];
    return idx;
}

/* Step 2.  Evaluate Q (and diagnostics G, Lo) at npts nodes of every cell
 * (npts < 0: all N^d nodes in storage order; otherwise pts[] holds node
 * indices, the same npts for every cell, or with pts_per_cell = 1 a
 * [ncells][npts] table of each cell's own nodes).  Outputs are
 * [ncells][npts]; any of Q, G, Lo may be NULL (G = Lo = NULL skips the
 * diagnostics; Q is accumulated the same way either way).
 * h = 2L/N (reading R3).  ndirs < 0: all lines of order <= N̄; otherwise only
 * the given canonical lines.  wa/wb: optional box tables of a(k), b(l)
 * (see orc_pairs).  Returns 0 on success, negative on bad input. */
int dvm_oracle_collide_w(int d, int N, int Nbar, int Ntilde, double L, const double *f,
                         int64_t ncells, int64_t npts, const int64_t *pts, int pts_per_cell, int ndirs,
                         const int *dirs, const double *wa, const double *wb, double *Q, double *G,
                         double *Lo, int nthreads)
{
    if (d < 1 || d > ORC_MAXD || N < 1 || Ntilde < 0 || ncells < 0 || !f) return -1;
    { int64_t nn = 1; for (int j = 0; j < d; ++j) nn *= N; if (nn > 2147483647) return -1; } /* int32 node tables */
    if (npts >= 0 && npts > 0 && !pts) return -1;
    if (4 * Ntilde + 1 > ORC_MAXW) return -1;
    double h = 2.0 * L / (double)N;
    int64_t cap = orc_pairs(d, Ntilde, Nbar, h, ndirs, dirs, wa, wb, 0, NULL, NULL, NULL);
    if (cap < 0) return -2;
    int *k = (int *)malloc(sizeof(int) * (size_t)(cap * d + 1));
    int *l = (int *)malloc(sizeof(int) * (size_t)(cap * d + 1));
    int *kl = (int *)malloc(sizeof(int) * (size_t)(cap * d + 1));
    double *a = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
    if (!k || !l || !kl || !a) {
        free(k); free(l); free(kl); free(a);
        return -3;
    }
    orc_pairs(d, Ntilde, Nbar, h, ndirs, dirs, wa, wb, cap, k, l, a);
    for (int64_t p = 0; p < cap * d; ++p) kl[p] = k[p] + l[p];

    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    int64_t nout = npts < 0 ? nodes : npts;
    int64_t total = ncells * nout;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const int twoNt = 2 * Ntilde;
    /* Work items are blocks of ORC_NB consecutive outputs: the pair list is read
     * once per block and applied to each node of the block in turn.  Every node
     * still accumulates its own terms in pair-list order with its own
     * compensated sums, so each result is exactly that of a one-node loop
     * (the blocking only saves re-reading the list from memory). */
    int64_t nblocks = (total + ORC_NB - 1) / ORC_NB;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t blk = 0; blk < nblocks; ++blk) {
        int64_t t0 = blk * ORC_NB;
        int nb = (int)(total - t0 < ORC_NB ? total - t0 : ORC_NB);
        int32_t wrap[ORC_NB][ORC_MAXD][ORC_MAXW];
        const double *fcs[ORC_NB];
        double fi[ORC_NB];
        double qs[ORC_NB], qc[ORC_NB], gs[ORC_NB], gc[ORC_NB], ls[ORC_NB], lc[ORC_NB];
        for (int b = 0; b < nb; ++b) {
            int64_t t = t0 + b;
            int64_t cell = t / nout;
            int64_t node = npts < 0 ? (t % nout) : (pts_per_cell ? pts[t] : pts[t % nout]);
            const double *fc = f + cell * nodes;
            int x[ORC_MAXD];
            int64_t r = node;
            for (int j = d - 1; j >= 0; --j) {
                x[j] = (int)(r % N);
                r /= N;
            }
            int64_t stride = 1;
            for (int j = d - 1; j >= 0; --j) {
                for (int o = -twoNt; o <= twoNt; ++o) {
                    int c = (x[j] + o) % N;
                    if (c < 0) c += N;
                    wrap[b][j][o + twoNt] = (int32_t)(c * stride);
                }
                stride *= N;
            }
            fcs[b] = fc;
            fi[b] = fc[node];
            qs[b] = qc[b] = gs[b] = gc[b] = ls[b] = lc[b] = 0.0;
        }
        const int diag = G || Lo;
        for (int64_t p = 0; p < cap; ++p) {
            const int *kp = k + p * d, *lp = l + p * d, *klp = kl + p * d;
            for (int b = 0; b < nb; ++b) {
                const int32_t(*w)[ORC_MAXW] = (const int32_t(*)[ORC_MAXW])wrap[b];
                double fk = fcs[b][orc_wrap_index(d, w, twoNt, kp)];
                double fl = fcs[b][orc_wrap_index(d, w, twoNt, lp)];
                double fkl = fcs[b][orc_wrap_index(d, w, twoNt, klp)];
                neu_add(&qs[b], &qc[b], a[p] * (fk * fl - fi[b] * fkl));
                if (diag) {
                    neu_add(&gs[b], &gc[b], a[p] * (fk * fl)); /* gain */
                    neu_add(&ls[b], &lc[b], a[p] * fkl);       /* loss (times f_i below) */
                }
            }
        }
        for (int b = 0; b < nb; ++b) {
            int64_t t = t0 + b;
            if (Q) Q[t] = qs[b] + qc[b];
            if (G) G[t] = gs[b] + gc[b];
            if (Lo) Lo[t] = fi[b] * (ls[b] + lc[b]);
        }
    }
    free(k);
    free(l);
    free(kl);
    free(a);
    return 0;
}

int dvm_oracle_collide(int d, int N, int Nbar, int Ntilde, double L, const double *f,
                       int64_t ncells, int64_t npts, const int64_t *pts, int ndirs,
                       const int *dirs, double *Q, double *G, double *Lo, int nthreads)
{
    return dvm_oracle_collide_w(d, N, Nbar, Ntilde, L, f, ncells, npts, pts, 0, ndirs, dirs, NULL, NULL, Q,
                                G, Lo, nthreads);
}
