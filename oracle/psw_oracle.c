/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the parsweep hot path
 * (see psw_oracle.h for the contract and the parity pin). Compiled with
 * -ffp-contract=off so every product/sum rounds exactly like the reference
 * compiled the same way (oracle/Makefile builds both with identical flags).
 *
 * Reference paths are relative to /root/reference/proj/include/parsweep/.
 */
#include "psw_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* core/thomas.hpp:22-45 — forward elimination with alpha/beta coefficients,
 * then back substitution. Pivot floor check before every division (:32,:38). */
static int thomas_scratch(int64_t n, const double* sub, const double* diag, const double* sup,
                          const double* f, double* x, double* alpha, double* beta,
                          int64_t* bad) {
    double piv = diag[0];
    if (fabs(piv) < ORC_PIVOT_FLOOR) {
        if (bad) *bad = 0;
        return ORC_PIVOT_BREAKDOWN;
    }
    alpha[0] = (n > 1) ? -sup[0] / piv : 0.0;
    beta[0] = f[0] / piv;
    for (int64_t i = 1; i < n; ++i) {
        piv = diag[i] + sub[i - 1] * alpha[i - 1];
        if (fabs(piv) < ORC_PIVOT_FLOOR) {
            if (bad) *bad = i;
            return ORC_PIVOT_BREAKDOWN;
        }
        alpha[i] = (i + 1 < n) ? -sup[i] / piv : 0.0;
        beta[i] = (f[i] - sub[i - 1] * beta[i - 1]) / piv;
    }
    x[n - 1] = beta[n - 1];
    for (int64_t i = n - 1; i-- > 0;) x[i] = beta[i] + alpha[i] * x[i + 1];
    return ORC_OK;
}

int orc_thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* f, double* x, int64_t* bad) {
    double* ws = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    if (!ws) return ORC_NO_MEMORY;
    int rc = thomas_scratch(n, sub, diag, sup, f, x, ws, ws + n, bad);
    free(ws);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* runtime/decompose.hpp:33-47: sizes base+1 for the first n%P ranges, base
 * for the rest; induced_partition (:23-29) keeps every range's right end but
 * the last one. */
int orc_decompose(int64_t n, int64_t P, int64_t* boundaries) {
    if (P <= 0 || n < 2 * P) return ORC_TOO_MANY_PES;
    int64_t base = n / P, rem = n % P, last = 0;
    for (int64_t i = 0; i + 1 < P; ++i) {
        last += base + (i < rem ? 1 : 0);
        boundaries[i] = last; /* 1-based right endpoint */
    }
    return ORC_OK;
}

/* dichotomy/partition.hpp:31-42 */
int orc_partition_validate(int64_t n, int64_t p, const int64_t* b) {
    if (n < 2) return ORC_INVALID_ARGUMENT;
    int64_t prev = 0;
    for (int64_t j = 0; j < p; ++j) {
        if (b[j] < 2 || b[j] > n - 1) return ORC_INVALID_ARGUMENT;
        if (b[j] <= prev) return ORC_INVALID_ARGUMENT;
        prev = b[j];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* dichotomy/level_sets.hpp:18-37: depth = floor(log2 p) + 1; level i takes
 * multiples of 2^(depth-i) not claimed by an earlier level, ascending. */
int64_t orc_level_sets(int64_t p, int64_t* order, int64_t* level_off) {
    int64_t depth = 1;
    while (((int64_t)1 << depth) <= p) ++depth;
    char* taken = (char*)calloc((size_t)p + 1, 1);
    int64_t w = 0;
    for (int64_t i = 1; i <= depth; ++i) {
        level_off[i - 1] = w;
        int64_t stride = (int64_t)1 << (depth - i);
        for (int64_t k = 1; k < ((int64_t)1 << i); ++k) {
            int64_t j = stride * k;
            if (j > p) break;
            if (taken[j]) continue;
            taken[j] = 1;
            order[w++] = j;
        }
    }
    level_off[depth] = w;
    free(taken);
    return depth;
}

uint64_t orc_comm_rounds(int64_t p) {
    if (p <= 0) return 0;
    int64_t depth = 1;
    while (((int64_t)1 << depth) <= p) ++depth;
    return (uint64_t)depth + 2;
}

/* ------------------------------------------------------------------------ */
/* dichotomy/preliminary.hpp:171-199 with the DirectSymmetric provider
 * (:139-143: g = thomas(A, e_r)); one-sided systems b_left_matrix (:29-37)
 * and b_right_matrix (:41-49); samples as in build_samples (:85-96). */
/* ------------------------------------------------------------------------ */
/* GRowProvider (dichotomy/preliminary.hpp:108-157): inverse rows under a
 * strategy, with the Auto fallbacks of its constructor (:111-132). */
#define ORC_INVERSE_SCALE_LIMIT 1e280 /* core/inverse_rows.hpp:14 */

typedef struct {
    int strategy;
    double *scale, *ssub, *ssup;      /* Symmetrize: core/symmetrize.hpp:21-37 */
    double *y, *z, *y_rho, *z_rho;    /* ExplicitInverse: core/inverse_rows.hpp:21-80 */
} grow_ctx;

static void grow_free(grow_ctx* c) {
    free(c->scale); free(c->ssub); free(c->ssup);
    free(c->y); free(c->z); free(c->y_rho); free(c->z_rho);
    memset(c, 0, sizeof(*c));
}

/* core/symmetrize.hpp:21-37; returns the failing k or -1 */
static int64_t symmetrize_into(int64_t n, const double* sub, const double* sup, grow_ctx* c) {
    c->scale[0] = 1.0;
    for (int64_t k = 1; k < n; ++k) c->scale[k] = 1.0;
    for (int64_t k = 0; k + 1 < n; ++k) {
        const double product = sub[k] * sup[k];
        if (!(product > 0.0)) return k;
        c->scale[k + 1] = c->scale[k] * sqrt(sub[k] / sup[k]);
        const double off = copysign(sqrt(product), sup[k]);
        c->ssub[k] = off;
        c->ssup[k] = off;
    }
    return -1;
}

/* core/inverse_rows.hpp:46-80; ORC_OK, ORC_ORACLE_FALLBACK or a pivot breakdown */
static int inverse_factors(int64_t n, const double* sub, const double* diag, const double* sup,
                           grow_ctx* c, double* e, double* al, double* be, int64_t* bad) {
    for (int64_t k = 0; k + 1 < n; ++k)
        if (sub[k] == 0.0 || sup[k] == 0.0) return ORC_ORACLE_FALLBACK;
    memset(e, 0, sizeof(double) * (size_t)n);
    e[n - 1] = 1.0;
    int rc = thomas_scratch(n, sub, diag, sup, e, c->y, al, be, bad);
    if (rc) return rc;
    if (!(fabs(c->y[0]) >= 1.0 / ORC_INVERSE_SCALE_LIMIT)) return ORC_ORACLE_FALLBACK;
    memset(e, 0, sizeof(double) * (size_t)n);
    e[0] = 1.0 / c->y[0];
    rc = thomas_scratch(n, sub, diag, sup, e, c->z, al, be, bad);
    if (rc) return rc;
    double rho = 1.0;
    for (int64_t j = 0; j < n; ++j) {
        if (j > 0) rho *= sup[j - 1] / sub[j - 1];
        if (!(fabs(rho) <= ORC_INVERSE_SCALE_LIMIT && fabs(rho) >= 1.0 / ORC_INVERSE_SCALE_LIMIT))
            return ORC_ORACLE_FALLBACK;
        c->y_rho[j] = c->y[j] * rho;
        c->z_rho[j] = c->z[j] * rho;
        if (!isfinite(c->y_rho[j]) || !isfinite(c->z_rho[j])) return ORC_ORACLE_FALLBACK;
    }
    return ORC_OK;
}

static int grow_init(int64_t n, const double* sub, const double* diag, const double* sup,
                     int requested, grow_ctx* c, double* e, double* al, double* be,
                     int64_t* bad) {
    memset(c, 0, sizeof(*c));
    int s = requested;
    if (s == ORC_GROW_AUTO) {
        int sym = 1;
        for (int64_t k = 0; k + 1 < n && sym; ++k) sym = sub[k] == sup[k];
        s = sym ? ORC_GROW_DIRECT_SYMMETRIC : ORC_GROW_SYMMETRIZE;
    }
    const size_t sz = (size_t)n;
    if (s == ORC_GROW_SYMMETRIZE) {
        c->scale = (double*)malloc(sizeof(double) * sz);
        c->ssub = (double*)malloc(sizeof(double) * sz);
        c->ssup = (double*)malloc(sizeof(double) * sz);
        if (!c->scale || !c->ssub || !c->ssup) return ORC_NO_MEMORY;
        int64_t k = symmetrize_into(n, sub, sup, c);
        if (k < 0)
            for (int64_t i = 0; i < n; ++i)
                if (!(isfinite(c->scale[i]) && c->scale[i] > 0.0)) { k = 0; break; }
        if (k >= 0) {
            if (requested != ORC_GROW_AUTO) {
                if (bad) *bad = k;
                return ORC_NOT_SYMMETRIZABLE;
            }
            s = ORC_GROW_EXPLICIT_INVERSE;
        }
    }
    if (s == ORC_GROW_EXPLICIT_INVERSE) {
        c->y = (double*)malloc(sizeof(double) * sz);
        c->z = (double*)malloc(sizeof(double) * sz);
        c->y_rho = (double*)malloc(sizeof(double) * sz);
        c->z_rho = (double*)malloc(sizeof(double) * sz);
        if (!c->y || !c->z || !c->y_rho || !c->z_rho) return ORC_NO_MEMORY;
        const int rc = inverse_factors(n, sub, diag, sup, c, e, al, be, bad);
        if (rc == ORC_ORACLE_FALLBACK) {
            if (requested != ORC_GROW_AUTO) return ORC_ORACLE_FALLBACK;
            s = ORC_GROW_TRANSPOSE_SOLVE;
        } else if (rc) {
            return rc;
        }
    }
    c->strategy = s;
    return ORC_OK;
}

/* GRowProvider::row (preliminary.hpp:136-156): row r0 (0-based) of inv(A) */
static int grow_row(const grow_ctx* c, int64_t n, const double* sub, const double* diag,
                    const double* sup, int64_t r0, double* g, double* e, double* al, double* be,
                    int64_t* bad) {
    switch (c->strategy) {
        case ORC_GROW_DIRECT_SYMMETRIC:
            memset(e, 0, sizeof(double) * (size_t)n);
            e[r0] = 1.0;
            return thomas_scratch(n, sub, diag, sup, e, g, al, be, bad);
        case ORC_GROW_SYMMETRIZE: {
            memset(e, 0, sizeof(double) * (size_t)n);
            e[r0] = 1.0;
            const int rc = thomas_scratch(n, c->ssub, diag, c->ssup, e, g, al, be, bad);
            if (rc) return rc;
            for (int64_t j = 0; j < n; ++j) g[j] *= c->scale[r0] / c->scale[j];
            return ORC_OK;
        }
        case ORC_GROW_EXPLICIT_INVERSE:
            for (int64_t j = 0; j < r0; ++j) g[j] = c->z[r0] * c->y_rho[j];
            for (int64_t j = r0; j < n; ++j) g[j] = c->y[r0] * c->z_rho[j];
            return ORC_OK;
        default: /* TransposeSolve: inverse_row_transpose (core/inverse_rows.hpp:99-104) */
            memset(e, 0, sizeof(double) * (size_t)n);
            e[r0] = 1.0;
            return thomas_scratch(n, sup, diag, sub, e, g, al, be, bad);
    }
}

int orc_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, double* g, double* zr_s, double* zl_s,
                    double* max_z, int64_t* bad) {
    return orc_preliminary_ex(n, sub, diag, sup, p, bnd, ORC_GROW_AUTO, NULL, g, zr_s, zl_s,
                              max_z, bad);
}

int orc_preliminary_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int* used, double* g,
                       double* zr_s, double* zl_s, double* max_z, int64_t* bad) {
    size_t sz = (size_t)n;
    double* e = (double*)malloc(sizeof(double) * sz);
    double* al = (double*)malloc(sizeof(double) * sz);
    double* be = (double*)malloc(sizeof(double) * sz);
    double* bd = (double*)malloc(sizeof(double) * sz);
    double* bs = (double*)malloc(sizeof(double) * sz);
    double* bu = (double*)malloc(sizeof(double) * sz);
    double* zl_all = (double*)malloc(sizeof(double) * sz * (size_t)(p > 0 ? p : 1));
    double* zr_all = (double*)malloc(sizeof(double) * sz * (size_t)(p > 0 ? p : 1));
    int rc = ORC_OK;
    double mz = 0.0;
    grow_ctx gc;
    memset(&gc, 0, sizeof(gc));
    if (!e || !al || !be || !bd || !bs || !bu || !zl_all || !zr_all) { rc = ORC_NO_MEMORY; goto out; }
    rc = grow_init(n, sub, diag, sup, strategy, &gc, e, al, be, bad);
    if (rc) goto out;
    if (used) *used = gc.strategy;

    for (int64_t j = 0; j < p; ++j) {
        const int64_t r = bnd[j];
        /* inverse row r (0-based r-1) */
        rc = grow_row(&gc, n, sub, diag, sup, r - 1, g + (size_t)j * sz, e, al, be, bad);
        if (rc) goto out;

        /* z_left: rows 1..r, row r unit, rhs e_last */
        memcpy(bd, diag, sizeof(double) * (size_t)r);
        bd[r - 1] = 1.0;
        memcpy(bs, sub, sizeof(double) * (size_t)(r - 1));
        bs[r - 2] = 0.0;
        memcpy(bu, sup, sizeof(double) * (size_t)(r - 1));
        memset(e, 0, sizeof(double) * (size_t)r);
        e[r - 1] = 1.0;
        double* zl = zl_all + (size_t)j * sz;
        rc = thomas_scratch(r, bs, bd, bu, e, zl, al, be, bad);
        if (rc) goto out;

        /* z_right: rows r..n, row r unit, rhs e_first */
        const int64_t m = n - r + 1;
        memcpy(bd, diag + (r - 1), sizeof(double) * (size_t)m);
        bd[0] = 1.0;
        memcpy(bs, sub + (r - 1), sizeof(double) * (size_t)(m - 1));
        memcpy(bu, sup + (r - 1), sizeof(double) * (size_t)(m - 1));
        bu[0] = 0.0;
        memset(e, 0, sizeof(double) * (size_t)m);
        e[0] = 1.0;
        double* zr = zr_all + (size_t)j * sz;
        rc = thomas_scratch(m, bs, bd, bu, e, zr, al, be, bad);
        if (rc) goto out;

        for (int64_t q = 0; q < r; ++q) mz = fmax(mz, fabs(zl[q]));
        for (int64_t q = 0; q < m; ++q) mz = fmax(mz, fabs(zr[q]));
    }
    if (zr_s && zl_s) {
        memset(zr_s, 0, sizeof(double) * (size_t)(p * p));
        memset(zl_s, 0, sizeof(double) * (size_t)(p * p));
        for (int64_t j = 0; j < p; ++j) {
            const int64_t rj = bnd[j];
            for (int64_t i = j; i < p; ++i) zr_s[j * p + i] = zr_all[(size_t)j * sz + (size_t)(bnd[i] - rj)];
            for (int64_t i = 0; i <= j; ++i) zl_s[j * p + i] = zl_all[(size_t)j * sz + (size_t)(bnd[i] - 1)];
        }
    }
    if (max_z) *max_z = mz;
out:
    grow_free(&gc);
    free(e); free(al); free(be); free(bd); free(bs); free(bu); free(zl_all); free(zr_all);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* dichotomy/partition.hpp:26-29 (1-based half-open block range). */
static int64_t block_begin(int64_t p, const int64_t* bnd, int64_t t) { return t == 0 ? 1 : bnd[t - 1]; }
static int64_t block_end(int64_t n, int64_t p, const int64_t* bnd, int64_t t) { return t == p ? n + 1 : bnd[t]; }

/* dichotomy/betas.hpp:34-59: ascending-row dot products of f against the
 * inverse rows of the block's right (g_t) and left (g_{t-1}) boundaries. */
void orc_betas(int64_t n, int64_t p, const int64_t* bnd, const double* g, const double* f,
               double* left, double* right) {
    for (int64_t t = 0; t <= p; ++t) { left[t] = 0.0; right[t] = 0.0; }
    for (int64_t t = 0; t <= p; ++t) {
        const int64_t lo = block_begin(p, bnd, t), hi = block_end(n, p, bnd, t);
        if (t < p) {
            const double* gr = g + (size_t)t * (size_t)n;
            double s = 0.0;
            for (int64_t q = lo; q < hi; ++q) s += f[q - 1] * gr[q - 1];
            right[t] = s;
        }
        if (t > 0) {
            const double* gl = g + (size_t)(t - 1) * (size_t)n;
            double s = 0.0;
            for (int64_t q = lo; q < hi; ++q) s += f[q - 1] * gl[q - 1];
            left[t] = s;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* boundary_solve.hpp:42-55: in-segment particular sum at boundary e. */
static double seg_sum(int64_t p, const double* zr_s, const double* zl_s, const double* left,
                      const double* right, int64_t kl, int64_t kr, int64_t e, uint64_t* terms) {
    double s = 0.0;
    for (int64_t t = kl + 1; t <= e; ++t) { s += right[t] * zr_s[t * p + e]; ++*terms; }
    for (int64_t t = e + 1; t <= kr; ++t) { s += left[t] * zl_s[(t - 1) * p + e]; ++*terms; }
    return s;
}

/* boundary_solve.hpp:61-88: one component with the 2x2 endpoint match. */
static double seg_component(int64_t p, const double* zr_s, const double* zl_s, const double* left,
                            const double* right, const double* value, int64_t kl, int64_t kr,
                            int64_t i, uint64_t* terms) {
    const double vi = seg_sum(p, zr_s, zl_s, left, right, kl, kr, i, terms);
    const int lk = kl >= 0, rk = kr < p;
    if (lk && rk) {
        const double b1 = value[kl] - seg_sum(p, zr_s, zl_s, left, right, kl, kr, kl, terms);
        const double b2 = value[kr] - seg_sum(p, zr_s, zl_s, left, right, kl, kr, kr, terms);
        const double m12 = zl_s[kr * p + kl];
        const double m21 = zr_s[kl * p + kr];
        const double det = 1.0 - m12 * m21;
        const double cl = (b1 - m12 * b2) / det;
        const double cr = (b2 - m21 * b1) / det;
        return vi + cl * zr_s[kl * p + i] + cr * zl_s[kr * p + i];
    }
    if (rk) {
        const double cr = value[kr] - seg_sum(p, zr_s, zl_s, left, right, kl, kr, kr, terms);
        return vi + cr * zl_s[kr * p + i];
    }
    if (lk) {
        const double cl = value[kl] - seg_sum(p, zr_s, zl_s, left, right, kl, kr, kl, terms);
        return vi + cl * zr_s[kl * p + i];
    }
    return vi;
}

/* boundary_solve.hpp:96-121: levels in dichotomy order, nearest known
 * neighbours found by scanning (:108-111). */
void orc_solve_boundaries(int64_t p, const double* zr_s, const double* zl_s,
                          const double* left, const double* right, double* value,
                          uint64_t* terms) {
    uint64_t local_terms = 0;
    if (!terms) terms = &local_terms;
    if (p == 0) return;
    for (int64_t j = 0; j < p; ++j) value[j] = 0.0;
    char* known = (char*)calloc((size_t)p, 1);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * 70);
    int64_t depth = orc_level_sets(p, order, off);
    for (int64_t l = 0; l < depth; ++l) {
        for (int64_t w = off[l]; w < off[l + 1]; ++w) {
            const int64_t i = order[w] - 1;
            int64_t kl = i - 1;
            while (kl >= 0 && !known[kl]) --kl;
            int64_t kr = i + 1;
            while (kr < p && !known[kr]) ++kr;
            value[i] = seg_component(p, zr_s, zl_s, left, right, value, kl, kr, i, terms);
        }
        for (int64_t w = off[l]; w < off[l + 1]; ++w) known[order[w] - 1] = 1;
    }
    free(known); free(order); free(off);
}

/* boundary_solve.hpp:126-136 */
void orc_solve_boundaries_two_sided(int64_t p, const double* zr_s, const double* zl_s,
                                    const double* left, const double* right, double* value,
                                    uint64_t* terms) {
    uint64_t local_terms = 0;
    if (!terms) terms = &local_terms;
    for (int64_t i = 0; i < p; ++i) value[i] = seg_sum(p, zr_s, zl_s, left, right, -1, p, i, terms);
}

/* ------------------------------------------------------------------------ */
/* local_solve.hpp:25-50: copy the closed block's rows, turn known boundary
 * rows into unit rows, sweep. Scratch: 5*(hi-lo+1) doubles. */
static int solve_local_scratch(int64_t n, const double* sub, const double* diag, const double* sup,
                               int64_t p, const int64_t* bnd, int64_t t, const double* f,
                               int has_first, double first_val, int has_last, double last_val,
                               double* out, double* ws, int64_t* bad) {
    const int64_t lo = t == 0 ? 1 : bnd[t - 1];
    const int64_t hi = t == p ? n : bnd[t];
    const int64_t m = hi - lo + 1;
    double* bd = ws;
    double* bs = ws + m;
    double* bu = ws + 2 * m;
    double* rhs = ws + 3 * m;
    double* al = ws + 4 * m;
    double* be = ws + 5 * m;
    memcpy(bd, diag + (lo - 1), sizeof(double) * (size_t)m);
    memcpy(bs, sub + (lo - 1), sizeof(double) * (size_t)(m - 1));
    memcpy(bu, sup + (lo - 1), sizeof(double) * (size_t)(m - 1));
    memcpy(rhs, f + (lo - 1), sizeof(double) * (size_t)m);
    if (has_first) { bd[0] = 1.0; bu[0] = 0.0; rhs[0] = first_val; }
    if (has_last) { bd[m - 1] = 1.0; bs[m - 2] = 0.0; rhs[m - 1] = last_val; }
    return thomas_scratch(m, bs, bd, bu, rhs, out, al, be, bad);
}

int orc_solve_local(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, int64_t t, const double* f, int has_first,
                    double first_val, int has_last, double last_val, double* out, int64_t* bad) {
    double* ws = (double*)malloc(sizeof(double) * 6 * (size_t)n);
    if (!ws) return ORC_NO_MEMORY;
    int rc = solve_local_scratch(n, sub, diag, sup, p, bnd, t, f, has_first, first_val, has_last,
                                 last_val, out, ws, bad);
    free(ws);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* dichotomy/batch.hpp:20-51: betas -> boundaries -> per-block sweeps; each
 * block writes its owned rows [n_t, n_{t+1}). `ws` holds 7n + 4(p+1) doubles. */
static int solve_one(int64_t n, const double* sub, const double* diag, const double* sup,
                     int64_t p, const int64_t* bnd, const double* g, const double* zr_s,
                     const double* zl_s, const double* f, double* out, double* ws,
                     uint64_t* terms, int64_t* bad) {
    double* left = ws;
    double* right = ws + (p + 1);
    double* value = ws + 2 * (p + 1);
    double* xb = ws + 3 * (p + 1) + 1;
    double* scratch = xb + n;
    orc_betas(n, p, bnd, g, f, left, right);
    orc_solve_boundaries(p, zr_s, zl_s, left, right, value, terms);
    for (int64_t t = 0; t <= p; ++t) {
        const int64_t lo = block_begin(p, bnd, t);
        const int64_t hi_owned = block_end(n, p, bnd, t) - 1;
        int rc = solve_local_scratch(n, sub, diag, sup, p, bnd, t, f, t > 0,
                                     t > 0 ? value[t - 1] : 0.0, t < p, t < p ? value[t] : 0.0,
                                     xb, scratch, bad);
        if (rc) return rc;
        for (int64_t row = lo; row <= hi_owned; ++row) out[row - 1] = xb[row - lo];
    }
    return ORC_OK;
}

static size_t solve_ws_doubles(int64_t n, int64_t p) { return (size_t)(7 * n + 4 * (p + 1) + 8); }

int orc_solve_with_preliminary(int64_t n, const double* sub, const double* diag,
                               const double* sup, int64_t p, const int64_t* bnd,
                               const double* g, const double* zr_s, const double* zl_s,
                               const double* f, double* out, uint64_t* terms, int64_t* bad) {
    double* ws = (double*)malloc(sizeof(double) * solve_ws_doubles(n, p));
    if (!ws) return ORC_NO_MEMORY;
    int rc = solve_one(n, sub, diag, sup, p, bnd, g, zr_s, zl_s, f, out, ws, terms, bad);
    free(ws);
    return rc;
}

/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n, p, k0, k1, ldf, ldx;
    const double *sub, *diag, *sup, *g, *zr, *zl, *F;
    const int64_t* bnd;
    double* X;
    int rc;
    int64_t bad;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    double* ws = (double*)malloc(sizeof(double) * solve_ws_doubles(j->n, j->p));
    if (!ws) { j->rc = ORC_NO_MEMORY; return NULL; }
    for (int64_t k = j->k0; k < j->k1 && j->rc == ORC_OK; ++k)
        j->rc = solve_one(j->n, j->sub, j->diag, j->sup, j->p, j->bnd, j->g, j->zr, j->zl,
                          j->F + (size_t)k * (size_t)j->ldf, j->X + (size_t)k * (size_t)j->ldx, ws,
                          NULL, &j->bad);
    free(ws);
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int solve_batch_impl(int64_t n, const double* sub, const double* diag, const double* sup,
                            int64_t p, const int64_t* bnd, int strategy, int64_t nrhs,
                            const double* F, int64_t ldf, double* X, int64_t ldx, int nthreads,
                            double* setup_s, double* solve_s, int64_t* bad);

int orc_solve_batch_threads(int64_t n, const double* sub, const double* diag, const double* sup,
                            int64_t p, const int64_t* bnd, int64_t nrhs, const double* F,
                            int64_t ldf, double* X, int64_t ldx, int nthreads,
                            double* setup_s, double* solve_s, int64_t* bad) {
    return solve_batch_impl(n, sub, diag, sup, p, bnd, ORC_GROW_AUTO, nrhs, F, ldf, X, ldx,
                            nthreads, setup_s, solve_s, bad);
}

int orc_solve_batch_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int64_t nrhs,
                       const double* F, int64_t ldf, double* X, int64_t ldx, int64_t* bad) {
    return solve_batch_impl(n, sub, diag, sup, p, bnd, strategy, nrhs, F, ldf, X, ldx, 1, NULL,
                            NULL, bad);
}

static int solve_batch_impl(int64_t n, const double* sub, const double* diag, const double* sup,
                            int64_t p, const int64_t* bnd, int strategy, int64_t nrhs,
                            const double* F, int64_t ldf, double* X, int64_t ldx, int nthreads,
                            double* setup_s, double* solve_s, int64_t* bad) {
    int rc = orc_partition_validate(n, p, bnd);
    if (rc) return rc;
    const double t0 = now_s();
    double* g = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(p > 0 ? p : 1));
    double* zr = (double*)malloc(sizeof(double) * (size_t)(p * p + 1));
    double* zl = (double*)malloc(sizeof(double) * (size_t)(p * p + 1));
    if (!g || !zr || !zl) { free(g); free(zr); free(zl); return ORC_NO_MEMORY; }
    rc = orc_preliminary_ex(n, sub, diag, sup, p, bnd, strategy, NULL, g, zr, zl, NULL, bad);
    const double t1 = now_s();
    if (rc == ORC_OK) {
        if (nthreads < 1) nthreads = 1;
        if (nthreads > nrhs) nthreads = (int)(nrhs > 0 ? nrhs : 1);
        batch_job* jobs = (batch_job*)calloc((size_t)nthreads, sizeof(batch_job));
        pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
        const int64_t chunk = (nrhs + nthreads - 1) / nthreads;
        for (int w = 0; w < nthreads; ++w) {
            batch_job* j = &jobs[w];
            j->n = n; j->p = p; j->ldf = ldf; j->ldx = ldx;
            j->sub = sub; j->diag = diag; j->sup = sup; j->g = g; j->zr = zr; j->zl = zl;
            j->F = F; j->X = X; j->bnd = bnd; j->rc = ORC_OK; j->bad = 0;
            j->k0 = (int64_t)w * chunk;
            j->k1 = j->k0 + chunk < nrhs ? j->k0 + chunk : nrhs;
            if (w == 0 || nthreads == 1) continue;
            pthread_create(&th[w], NULL, batch_worker, j);
        }
        batch_worker(&jobs[0]);
        for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
        for (int w = 0; w < nthreads; ++w)
            if (jobs[w].rc && rc == ORC_OK) { rc = jobs[w].rc; if (bad) *bad = jobs[w].bad; }
        free(jobs); free(th);
    }
    const double t2 = now_s();
    if (setup_s) *setup_s = t1 - t0;
    if (solve_s) *solve_s = t2 - t1;
    free(g); free(zr); free(zl);
    return rc;
}

int orc_solve_batch(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, int64_t nrhs, const double* F, int64_t ldf,
                    double* X, int64_t ldx, int64_t* bad) {
    return orc_solve_batch_threads(n, sub, diag, sup, p, bnd, nrhs, F, ldf, X, ldx, 1, NULL, NULL, bad);
}

/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void orc_fill_uniform(double* out, int64_t count, uint64_t seed, uint64_t offset, double lo,
                      double hi) {
    const double scale = 1.0 / 9007199254740992.0; /* 2^-53 */
    const double span = hi - lo;
    for (int64_t i = 0; i < count; ++i) {
        const double u = (double)(splitmix64(seed ^ (offset + (uint64_t)i)) >> 11) * scale;
        out[i] = lo + span * u;
    }
}
