/* TEST INFRASTRUCTURE ONLY — CPU oracle; see sslref.h.  Never linked into the
 * product library (paper_2504_03373_b200/), never called on its hot path.
 *
 * Restates the reference double-precision GSVD-MUSIC path in C99.  Arithmetic
 * follows the reference's operation order with contraction disabled
 * (-ffp-contract=off) and the textbook complex formulas that
 * -fcx-limited-range selects (proj/CMakeLists.txt:15-18), so on x86-64 the
 * results are expected to match the compiled reference bit for bit; the tests
 * pin that against oracle/_ref and tests/golden/.
 */
#include "sslref.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---------------------------------------------------------------------------
 * complex helpers: plain formulas, one rounding per operation
 * ------------------------------------------------------------------------- */
typedef struct { double re, im; } cd;

static inline cd c_make(double re, double im) { cd z = {re, im}; return z; }
static inline cd c_add(cd a, cd b) { return c_make(a.re + b.re, a.im + b.im); }
static inline cd c_sub(cd a, cd b) { return c_make(a.re - b.re, a.im - b.im); }
static inline cd c_mul(cd a, cd b) { return c_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cd c_conj(cd a) { return c_make(a.re, -a.im); }
static inline cd c_scale(double s, cd a) { return c_make(s * a.re, s * a.im); }
static inline cd c_rdiv(cd a, double s) { return c_make(a.re / s, a.im / s); }
static inline double c_norm(cd a) { return a.re * a.re + a.im * a.im; }
static inline double c_abs(cd a) { return hypot(a.re, a.im); }
/* (1,0)/z under limited range: conj(z)/|z|^2 computed per component */
static inline cd c_recip(cd z) {
    const double den = z.re * z.re + z.im * z.im;
    return c_make((1.0 * z.re + 0.0 * z.im) / den, (0.0 * z.re - 1.0 * z.im) / den);
}

/* dense complex matrix, row major */
typedef struct { uint32_t rows, cols; cd* v; } cmat;

static cmat cm_new(uint32_t r, uint32_t c) {
    cmat m; m.rows = r; m.cols = c;
    m.v = (cd*)calloc((size_t)r * c + 1, sizeof(cd));
    return m;
}
static void cm_free(cmat* m) { free(m->v); m->v = NULL; }
#define AT(m, i, j) ((m).v[(size_t)(i) * (m).cols + (j)])

/* matmul with the zero skip of mat.hpp:31-44: c(i,j) accumulates over k in order */
static cmat cm_mul(cmat a, cmat b) {
    cmat c = cm_new(a.rows, b.cols);
    for (uint32_t i = 0; i < a.rows; ++i)
        for (uint32_t k = 0; k < a.cols; ++k) {
            const cd aik = AT(a, i, k);
            if (aik.re == 0.0 && aik.im == 0.0) continue;
            for (uint32_t j = 0; j < b.cols; ++j) AT(c, i, j) = c_add(AT(c, i, j), c_mul(aik, AT(b, k, j)));
        }
    return c;
}

static cmat cm_adj(cmat a) {
    cmat c = cm_new(a.cols, a.rows);
    for (uint32_t i = 0; i < a.rows; ++i)
        for (uint32_t j = 0; j < a.cols; ++j) AT(c, j, i) = c_conj(AT(a, i, j));
    return c;
}

static double col_norm2(cmat m, uint32_t col) {
    double s = 0;
    for (uint32_t i = 0; i < m.rows; ++i) s += c_norm(AT(m, i, col));
    return s;
}

/* ---------------------------------------------------------------------------
 * correlation window (correlation.cpp:53-130)
 * ------------------------------------------------------------------------- */

/* running sum += sign * x x^H over every bin (correlation.cpp:60-73) */
static void corr_accumulate(cd* sum, const float* frame, uint32_t m, uint32_t bins, double sign) {
    for (uint32_t b = 0; b < bins; ++b) {
        cd* acc = sum + (size_t)b * m * m;
        for (uint32_t i = 0; i < m; ++i) {
            const float* pi = frame + ((size_t)i * bins + b) * 2;
            const cd xi = c_make((double)pi[0], (double)pi[1]);
            for (uint32_t j = 0; j < m; ++j) {
                const float* pj = frame + ((size_t)j * bins + b) * 2;
                const cd xj = c_make((double)pj[0], (double)pj[1]);
                acc[(size_t)i * m + j] = c_add(acc[(size_t)i * m + j], c_scale(sign, c_mul(xi, c_conj(xj))));
            }
        }
    }
}

int orc_correlation(const float* x, uint32_t frames, uint32_t m, uint32_t bins, uint32_t t,
                    uint32_t rebuild_interval, float* r_out, uint32_t* written) {
    if (t < 1) return set_err(2, "correlation window length must be >= 1");
    if (m == 0) return set_err(2, "empty spectrum frame");
    if (rebuild_interval < 1) rebuild_interval = 1;
    const size_t fsz = (size_t)m * bins * 2;
    for (size_t i = 0; i < fsz * frames; ++i)
        if (!isfinite(x[i])) return set_err(2, "non-finite spectrum value");
    cd* sum = (cd*)calloc((size_t)bins * m * m, sizeof(cd));
    uint64_t pushed = 0, since = 0;
    const double inv_t = 1.0 / (double)t;
    uint32_t out = 0;
    for (uint32_t f = 0; f < frames; ++f) {
        /* push (correlation.cpp:86-110): the ring slot of the frame leaving
         * the window is the frame pushed T pushes ago */
        if (pushed >= t) corr_accumulate(sum, x + (size_t)(f - t) * fsz, m, bins, -1.0);
        corr_accumulate(sum, x + (size_t)f * fsz, m, bins, 1.0);
        ++pushed;
        if (++since >= rebuild_interval) {
            /* rebuild oldest first (correlation.cpp:75-84) */
            memset(sum, 0, (size_t)bins * m * m * sizeof(cd));
            const uint64_t have = pushed < t ? pushed : t;
            for (uint64_t k = 0; k < have; ++k) {
                const uint64_t g = pushed - have + k; /* global frame index */
                corr_accumulate(sum, x + (size_t)g * fsz, m, bins, 1.0);
            }
            since = 0;
        }
        if (pushed < t) continue;
        /* normalized (correlation.cpp:112-130) */
        float* r = r_out + (size_t)out * bins * m * m * 2;
        for (size_t i = 0; i < (size_t)bins * m * m; ++i) {
            r[2 * i] = (float)(sum[i].re * inv_t);
            r[2 * i + 1] = (float)(sum[i].im * inv_t);
        }
        ++out;
    }
    free(sum);
    *written = out;
    return 0;
}

/* ---------------------------------------------------------------------------
 * Gauss-Jordan inverse with partial pivoting (gsvd.cpp:21-62)
 * ------------------------------------------------------------------------- */
static int inverse_d(cmat a, cmat inv, int pivoting, uint32_t bin_label) {
    const uint32_t n = a.rows;
    double scale = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i) {
        const double v = c_abs(a.v[i]);
        if (v > scale) scale = v;
    }
    const double floor_ = scale * 2.220446049250313080847e-16 * (double)n;
    for (uint32_t col = 0; col < n; ++col) {
        uint32_t piv = col;
        if (pivoting)
            for (uint32_t row = col + 1; row < n; ++row)
                if (c_abs(AT(a, row, col)) > c_abs(AT(a, piv, col))) piv = row;
        if (!(c_abs(AT(a, piv, col)) > floor_)) {
            char msg[96];
            snprintf(msg, sizeof msg, "noise matrix is singular at bin %u", bin_label);
            return set_err(3, msg);
        }
        if (piv != col)
            for (uint32_t j = 0; j < n; ++j) {
                cd t0 = AT(a, col, j); AT(a, col, j) = AT(a, piv, j); AT(a, piv, j) = t0;
                cd t1 = AT(inv, col, j); AT(inv, col, j) = AT(inv, piv, j); AT(inv, piv, j) = t1;
            }
        const cd d = c_recip(AT(a, col, col));
        for (uint32_t j = 0; j < n; ++j) {
            AT(a, col, j) = c_mul(AT(a, col, j), d);
            AT(inv, col, j) = c_mul(AT(inv, col, j), d);
        }
        for (uint32_t row = 0; row < n; ++row) {
            if (row == col) continue;
            const cd f = AT(a, row, col);
            if (f.re == 0.0 && f.im == 0.0) continue;
            for (uint32_t j = 0; j < n; ++j) {
                AT(a, row, j) = c_sub(AT(a, row, j), c_mul(f, AT(a, col, j)));
                AT(inv, row, j) = c_sub(AT(inv, row, j), c_mul(f, AT(inv, col, j)));
            }
        }
    }
    return 0;
}

int orc_mat_inverse(const float* k, uint32_t m, int pivoting, uint32_t bin_label, double* out) {
    cmat a = cm_new(m, m), inv = cm_new(m, m);
    for (size_t i = 0; i < (size_t)m * m; ++i) a.v[i] = c_make(k[2 * i], k[2 * i + 1]);
    for (uint32_t i = 0; i < m; ++i) AT(inv, i, i) = c_make(1, 0);
    const int rc = inverse_d(a, inv, pivoting, bin_label);
    if (rc == 0) memcpy(out, inv.v, (size_t)m * m * sizeof(cd));
    cm_free(&a);
    cm_free(&inv);
    return rc;
}

/* ---------------------------------------------------------------------------
 * one-sided Jacobi (gsvd.cpp:622-695)
 * ------------------------------------------------------------------------- */

/* stable descending order of values (gsvd.cpp:331-338): insertion sort keeps
 * equal keys in index order */
static void desc_perm(const double* v, uint32_t n, uint32_t* perm) {
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    for (uint32_t i = 1; i < n; ++i) {
        const uint32_t p = perm[i];
        uint32_t j = i;
        while (j > 0 && v[p] > v[perm[j - 1]]) {
            perm[j] = perm[j - 1];
            --j;
        }
        perm[j] = p;
    }
}

static void jacobi(cmat a, double* sigma, cmat u, cmat* vh, uint32_t* sweeps_out, uint8_t* conv_out) {
    const uint32_t n = a.rows;
    cmat w = cm_new(n, n), v = cm_new(n, n);
    memcpy(w.v, a.v, (size_t)n * n * sizeof(cd));
    for (uint32_t i = 0; i < n; ++i) AT(v, i, i) = c_make(1, 0);
    double* cn = (double*)malloc(sizeof(double) * (n + 1));
    int converged = 0;
    uint32_t sweeps = 0;
    for (uint32_t sweep = 0; sweep < 60 && !converged; ++sweep) {
        sweeps = sweep + 1;
        double cn_max = 0;
        for (uint32_t j = 0; j < n; ++j) {
            cn[j] = col_norm2(w, j);
            if (cn[j] > cn_max) cn_max = cn[j];
        }
        const double drop = 1e-20 * cn_max;
        int rotated = 0;
        for (uint32_t p = 0; p + 1 < n; ++p)
            for (uint32_t q = p + 1; q < n; ++q) {
                if (cn[p] <= drop || cn[q] <= drop) continue;
                cd apq = c_make(0, 0);
                for (uint32_t i = 0; i < n; ++i) apq = c_add(apq, c_mul(c_conj(AT(w, i, p)), AT(w, i, q)));
                const double mag = c_abs(apq);
                if (mag * mag <= 1e-28 * cn[p] * cn[q]) continue;
                rotated = 1;
                const cd ph = c_rdiv(apq, mag);
                const double tau = (cn[q] - cn[p]) / (2.0 * mag);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = t * c;
                const cd sphc = c_scale(s, c_conj(ph));
                for (uint32_t i = 0; i < n; ++i) {
                    const cd wp = AT(w, i, p), wq = AT(w, i, q);
                    AT(w, i, p) = c_sub(c_scale(c, wp), c_mul(sphc, wq));
                    AT(w, i, q) = c_add(c_scale(s, wp), c_mul(c_scale(c, c_conj(ph)), wq));
                }
                for (uint32_t i = 0; i < n; ++i) {
                    const cd vp = AT(v, i, p), vq = AT(v, i, q);
                    AT(v, i, p) = c_sub(c_scale(c, vp), c_mul(sphc, vq));
                    AT(v, i, q) = c_add(c_scale(s, vp), c_mul(c_scale(c, c_conj(ph)), vq));
                }
                const double old_p = cn[p];
                cn[p] = c * c * old_p - 2.0 * c * s * mag + s * s * cn[q];
                cn[q] = s * s * old_p + 2.0 * c * s * mag + c * c * cn[q];
            }
        if (!rotated) converged = 1;
    }
    double* raw = (double*)malloc(sizeof(double) * (n + 1));
    cmat uu = cm_new(n, n);
    for (uint32_t j = 0; j < n; ++j) {
        const double nrm = sqrt(col_norm2(w, j));
        raw[j] = nrm;
        if (nrm > 0) {
            const double inv = 1.0 / nrm;
            for (uint32_t i = 0; i < n; ++i) AT(uu, i, j) = c_scale(inv, AT(w, i, j));
        }
    }
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    desc_perm(raw, n, perm);
    for (uint32_t i = 0; i < n; ++i) sigma[i] = raw[perm[i]];
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < n; ++j) AT(u, i, j) = AT(uu, i, perm[j]);
    if (vh)
        for (uint32_t r = 0; r < n; ++r)
            for (uint32_t j = 0; j < n; ++j) AT(*vh, r, j) = c_conj(AT(v, j, perm[r]));
    if (sweeps_out) *sweeps_out = sweeps;
    if (conv_out) *conv_out = (uint8_t)converged;
    free(perm);
    free(raw);
    free(cn);
    cm_free(&uu);
    cm_free(&w);
    cm_free(&v);
}

int orc_jacobi_svd(const double* a, uint32_t m, double* sigma, double* u, double* vh, uint32_t* sweeps,
                   uint8_t* conv) {
    cmat am = cm_new(m, m), um = cm_new(m, m), vm = cm_new(m, m);
    memcpy(am.v, a, (size_t)m * m * sizeof(cd));
    jacobi(am, sigma, um, &vm, sweeps, conv);
    memcpy(u, um.v, (size_t)m * m * sizeof(cd));
    if (vh) memcpy(vh, vm.v, (size_t)m * m * sizeof(cd));
    cm_free(&am);
    cm_free(&um);
    cm_free(&vm);
    return 0;
}

/* ---------------------------------------------------------------------------
 * canonical bases for degenerate groups (gsvd.cpp:377-565)
 * ------------------------------------------------------------------------- */
#define DEGENERATE_GAP 1e-5 /* gsvd.cpp:381 */

/* c -= sum_k (b_k^H c) b_k over the first `cols` columns, sequentially (389-396) */
static void project_out(cd* c, cmat basis, uint32_t cols) {
    for (uint32_t k = 0; k < cols; ++k) {
        cd dot = c_make(0, 0);
        for (uint32_t i = 0; i < basis.rows; ++i) dot = c_add(dot, c_mul(c_conj(AT(basis, i, k)), c[i]));
        for (uint32_t i = 0; i < basis.rows; ++i) c[i] = c_sub(c[i], c_mul(dot, AT(basis, i, k)));
    }
}

typedef void (*make_fn)(uint32_t j, cd* c, void* ctx);

/* fixed-order orthonormal pick with relaxation passes (gsvd.cpp:404-436) */
static cmat pick_orthonormal(uint32_t n, uint32_t need, const cmat* exclude, make_fn make, void* ctx) {
    cmat out = cm_new(n, need);
    uint32_t taken = 0;
    char* used = (char*)calloc(n + 1, 1);
    cd* c = (cd*)malloc(sizeof(cd) * (n + 1));
    static const double thresholds[3] = {0.05, 1e-8, 0.0};
    for (int pass_t = 0; pass_t < 3; ++pass_t) {
        const double thr = thresholds[pass_t];
        for (uint32_t j = 0; j < n && taken < need; ++j) {
            if (used[j]) continue;
            make(j, c, ctx);
            double norm0 = 0;
            for (uint32_t i = 0; i < n; ++i) norm0 += c_norm(c[i]);
            norm0 = sqrt(norm0);
            if (!(norm0 > 1e-140)) continue;
            for (int pass = 0; pass < 2; ++pass) {
                if (exclude) project_out(c, *exclude, exclude->cols);
                project_out(c, out, taken);
            }
            double nrm = 0;
            for (uint32_t i = 0; i < n; ++i) nrm += c_norm(c[i]);
            nrm = sqrt(nrm);
            if (!(nrm > thr * norm0) || !(nrm > 0)) continue;
            const double inv = 1.0 / nrm;
            for (uint32_t i = 0; i < n; ++i) AT(out, i, taken) = c_scale(inv, c[i]);
            used[j] = 1;
            ++taken;
        }
        if (taken == need) break;
    }
    free(c);
    free(used);
    return out;
}

static void make_unit(uint32_t j, cd* c, void* ctx) {
    const uint32_t n = *(const uint32_t*)ctx;
    for (uint32_t i = 0; i < n; ++i) c[i] = c_make(0, 0);
    c[j] = c_make(1, 0);
}

typedef struct { cmat group; } group_ctx;

/* candidate = projector of the group applied to delta_j (gsvd.cpp:518-526) */
static void make_group(uint32_t j, cd* c, void* ctx) {
    const cmat g = ((group_ctx*)ctx)->group;
    for (uint32_t r = 0; r < g.rows; ++r) {
        cd acc = c_make(0, 0);
        for (uint32_t kk = 0; kk < g.cols; ++kk) acc = c_add(acc, c_mul(AT(g, r, kk), c_conj(AT(g, j, kk))));
        c[r] = acc;
    }
}

/* one step of A A^H subspace iteration with 2-pass MGS (gsvd.cpp:440-466) */
static cmat refine_leading(cmat a, cmat lead) {
    cmat ah = cm_adj(a);
    cmat t = cm_mul(ah, lead);
    cmat s = cm_mul(a, t);
    cm_free(&ah);
    cm_free(&t);
    for (uint32_t j = 0; j < s.cols; ++j) {
        for (int pass = 0; pass < 2; ++pass)
            for (uint32_t k = 0; k < j; ++k) {
                cd dot = c_make(0, 0);
                for (uint32_t i = 0; i < s.rows; ++i) dot = c_add(dot, c_mul(c_conj(AT(s, i, k)), AT(s, i, j)));
                for (uint32_t i = 0; i < s.rows; ++i) AT(s, i, j) = c_sub(AT(s, i, j), c_mul(dot, AT(s, i, k)));
            }
        double nrm = sqrt(col_norm2(s, j));
        if (!(nrm > 1e-200)) {
            for (uint32_t i = 0; i < s.rows; ++i) AT(s, i, j) = AT(lead, i, j);
            for (uint32_t k = 0; k < j; ++k) {
                cd dot = c_make(0, 0);
                for (uint32_t i = 0; i < s.rows; ++i) dot = c_add(dot, c_mul(c_conj(AT(s, i, k)), AT(s, i, j)));
                for (uint32_t i = 0; i < s.rows; ++i) AT(s, i, j) = c_sub(AT(s, i, j), c_mul(dot, AT(s, i, k)));
            }
            nrm = sqrt(col_norm2(s, j));
            if (!(nrm > 0)) continue;
        }
        const double inv = 1.0 / nrm;
        for (uint32_t i = 0; i < s.rows; ++i) AT(s, i, j) = c_scale(inv, AT(s, i, j));
    }
    return s;
}

static void canonicalize(cmat a, const double* values, cmat e, cmat* er) {
    const uint32_t n = a.rows;
    if (n == 0) return;
    const double smax = values[0] > 0 ? values[0] : 0.0;
    uint32_t z = 0;
    while (z < n && values[n - 1 - z] <= DEGENERATE_GAP * smax) ++z;
    if (z > 0) {
        const uint32_t lead = n - z;
        cmat basis = cm_new(n, lead);
        if (lead > 0) {
            cmat v = cm_new(n, lead);
            for (uint32_t i = 0; i < n; ++i)
                for (uint32_t j = 0; j < lead; ++j) AT(v, i, j) = AT(e, i, j);
            cm_free(&basis);
            basis = refine_leading(a, v);
            cm_free(&v);
        }
        uint32_t nn = n;
        cmat comp = pick_orthonormal(n, z, lead > 0 ? &basis : NULL, make_unit, &nn);
        for (uint32_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < z; ++j) AT(e, i, lead + j) = AT(comp, i, j);
        cm_free(&comp);
        cm_free(&basis);
    }
    const uint32_t lead_end = n - z;
    for (uint32_t i = 0; i < lead_end;) {
        uint32_t end = i;
        while (end + 1 < lead_end && values[end] - values[end + 1] <= DEGENERATE_GAP * smax) ++end;
        if (end > i) {
            const uint32_t kdim = end - i + 1;
            group_ctx g;
            g.group = cm_new(n, kdim);
            for (uint32_t r = 0; r < n; ++r)
                for (uint32_t j = 0; j < kdim; ++j) AT(g.group, r, j) = AT(e, r, i + j);
            cmat b = pick_orthonormal(n, kdim, NULL, make_group, &g);
            cmat gh = cm_adj(g.group);
            cmat w = cm_mul(gh, b);
            for (uint32_t r = 0; r < n; ++r)
                for (uint32_t j = 0; j < kdim; ++j) AT(e, r, i + j) = AT(b, r, j);
            if (er) {
                cmat rows = cm_new(kdim, er->cols);
                for (uint32_t j = 0; j < kdim; ++j)
                    for (uint32_t cc = 0; cc < er->cols; ++cc) AT(rows, j, cc) = AT(*er, i + j, cc);
                cmat wh = cm_adj(w);
                cmat mixed = cm_mul(wh, rows);
                for (uint32_t j = 0; j < kdim; ++j)
                    for (uint32_t cc = 0; cc < er->cols; ++cc) AT(*er, i + j, cc) = AT(mixed, j, cc);
                cm_free(&rows);
                cm_free(&wh);
                cm_free(&mixed);
            }
            cm_free(&gh);
            cm_free(&w);
            cm_free(&b);
            cm_free(&g.group);
        }
        i = end + 1;
    }
    /* phase of each left vector (gsvd.cpp:545-564) */
    for (uint32_t j = 0; j < n; ++j) {
        uint32_t piv = 0;
        double best = -1;
        for (uint32_t i = 0; i < n; ++i) {
            const double mg = c_abs(AT(e, i, j));
            if (mg > best) {
                best = mg;
                piv = i;
            }
        }
        if (!(best > 0)) continue;
        const cd val = AT(e, piv, j);
        const cd ph = c_rdiv(val, c_abs(val));
        const cd up = c_conj(ph);
        for (uint32_t i = 0; i < n; ++i) AT(e, i, j) = c_mul(AT(e, i, j), up);
        if (er)
            for (uint32_t cc = 0; cc < er->cols; ++cc) AT(*er, j, cc) = c_mul(AT(*er, j, cc), ph);
    }
}

void orc_canonicalize(const double* a, uint32_t m, const double* sigma, double* e, double* er) {
    cmat am = cm_new(m, m), em, erm;
    memcpy(am.v, a, (size_t)m * m * sizeof(cd));
    em.rows = em.cols = m;
    em.v = (cd*)e;
    erm.rows = erm.cols = m;
    erm.v = (cd*)er;
    canonicalize(am, sigma, em, er ? &erm : NULL);
    cm_free(&am);
}

/* gsvd_reference_matrix (gsvd.cpp:697-716) on A = K^-1 R */
static void reference_bin(cmat kinv, const float* r, uint32_t m, int canonical, double* sigma, double* e,
                          double* er, uint32_t* sweeps, uint8_t* conv) {
    cmat rm = cm_new(m, m);
    for (size_t i = 0; i < (size_t)m * m; ++i) rm.v[i] = c_make(r[2 * i], r[2 * i + 1]);
    cmat a = cm_mul(kinv, rm);
    cmat u = cm_new(m, m), vh = cm_new(m, m);
    jacobi(a, sigma, u, &vh, sweeps, conv);
    if (canonical) canonicalize(a, sigma, u, &vh);
    memcpy(e, u.v, (size_t)m * m * sizeof(cd));
    if (er) memcpy(er, vh.v, (size_t)m * m * sizeof(cd));
    cm_free(&rm);
    cm_free(&a);
    cm_free(&u);
    cm_free(&vh);
}

int orc_gsvd_reference(const float* k, const double* kinv, const float* r, uint32_t m, uint32_t bins,
                       int canonical, int threads, double* sigma, double* e, double* er, uint32_t* sweeps,
                       uint8_t* conv) {
    int status = 0;
    char first_err[256] = {0};
    for (size_t i = 0; i < (size_t)bins * m * m * 2; ++i)
        if (!isfinite(r[i])) return set_err(2, "non-finite correlation entry");
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (uint32_t b = 0; b < bins; ++b) {
        cmat ki = cm_new(m, m);
        int rc = 0;
        if (kinv) {
            memcpy(ki.v, kinv + (size_t)b * m * m * 2, (size_t)m * m * sizeof(cd));
        } else {
            cmat ka = cm_new(m, m);
            const float* kb = k + (size_t)b * m * m * 2;
            for (size_t i = 0; i < (size_t)m * m; ++i) ka.v[i] = c_make(kb[2 * i], kb[2 * i + 1]);
            for (uint32_t i = 0; i < m; ++i) AT(ki, i, i) = c_make(1, 0);
            rc = inverse_d(ka, ki, 1, b);
            cm_free(&ka);
        }
        if (rc) {
#pragma omp critical
            {
                if (!status) {
                    status = rc;
                    snprintf(first_err, sizeof first_err, "%s", g_err);
                }
            }
        } else {
            const size_t mm = (size_t)m * m * 2;
            reference_bin(ki, r + (size_t)b * mm, m, canonical, sigma + (size_t)b * m, e + (size_t)b * mm,
                          er ? er + (size_t)b * mm : NULL, sweeps ? sweeps + b : NULL, conv ? conv + b : NULL);
        }
        cm_free(&ki);
    }
    if (status) return set_err(status, first_err);
    return 0;
}

/* ---------------------------------------------------------------------------
 * spectrum (music.cpp:112-165)
 * ------------------------------------------------------------------------- */
int orc_spectrum(const double* e, uint32_t m, uint32_t bins, const float* h, uint32_t dirs,
                 uint32_t num_sources, float floor_f, int squared, int threads, double* power,
                 double* bin_power) {
    if (num_sources == 0) return set_err(2, "num_sources must be at least 1");
    if (!(floor_f > 0)) return set_err(2, "denominator_floor must be positive");
    if (num_sources >= m) return set_err(2, "num_sources must be smaller than the channel count");
    const uint32_t nn = m - num_sources;
    const double floor_ = (double)floor_f;
    /* noise columns gathered [bin][vector][mic] (music.cpp:127-135) */
    cd* noise = (cd*)malloc(sizeof(cd) * ((size_t)bins * nn * m + 1));
    for (uint32_t b = 0; b < bins; ++b) {
        const cd* eb = (const cd*)(e + (size_t)b * m * m * 2);
        for (uint32_t i = 0; i < nn; ++i)
            for (uint32_t mic = 0; mic < m; ++mic)
                noise[((size_t)b * nn + i) * m + mic] = eb[(size_t)mic * m + num_sources + i];
    }
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (uint32_t d = 0; d < dirs; ++d) {
        double acc = 0.0;
        for (uint32_t b = 0; b < bins; ++b) {
            const float* hv = h + (((size_t)d * bins + b) * m) * 2;
            double num = 0;
            for (uint32_t mic = 0; mic < m; ++mic)
                num += (double)hv[2 * mic] * (double)hv[2 * mic] + (double)hv[2 * mic + 1] * (double)hv[2 * mic + 1];
            double den = 0;
            const cd* nv = noise + (size_t)b * nn * m;
            for (uint32_t i = 0; i < nn; ++i, nv += m) {
                cd dot = c_make(0, 0);
                for (uint32_t mic = 0; mic < m; ++mic)
                    dot = c_add(dot, c_mul(c_conj(c_make(hv[2 * mic], hv[2 * mic + 1])), nv[mic]));
                const double mag = c_abs(dot);
                den += squared ? mag * mag : mag;
            }
            if (den < floor_) den = floor_;
            const double p = num / den;
            acc += p;
            if (bin_power) bin_power[(size_t)b * dirs + d] = p;
        }
        power[d] = acc;
    }
    free(noise);
    return 0;
}

/* ---------------------------------------------------------------------------
 * topology and peaks (music.cpp:15-19, 176-236)
 * ------------------------------------------------------------------------- */
static void unit_vec(double az_deg, double el_deg, double* u) {
    const double az = az_deg * M_PI / 180.0;
    const double el = el_deg * M_PI / 180.0;
    u[0] = cos(el) * cos(az);
    u[1] = cos(el) * sin(az);
    u[2] = sin(el);
}

int orc_topology(const double* dirs, uint32_t n, double radius_deg, uint32_t* offsets, uint32_t* nbr,
                 uint32_t cap) {
    double* u = (double*)malloc(sizeof(double) * 3 * (n + 1));
    uint32_t* deg = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    for (uint32_t i = 0; i < n; ++i) unit_vec(dirs[2 * i], dirs[2 * i + 1], u + 3 * i);
    const double cr = cos(radius_deg * M_PI / 180.0);
    /* pass 1: degrees; pass 2: fill in ascending neighbor order */
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = i + 1; j < n; ++j) {
            const double dot = u[3 * i] * u[3 * j] + u[3 * i + 1] * u[3 * j + 1] + u[3 * i + 2] * u[3 * j + 2];
            if (dot >= cr) {
                ++deg[i];
                ++deg[j];
            }
        }
    uint32_t total = 0;
    for (uint32_t i = 0; i < n; ++i) {
        offsets[i] = total;
        total += deg[i];
    }
    offsets[n] = total;
    if (total > cap) {
        free(u);
        free(deg);
        return set_err(2, "topology capacity exceeded");
    }
    memset(deg, 0, sizeof(uint32_t) * (n + 1));
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = i + 1; j < n; ++j) {
            const double dot = u[3 * i] * u[3 * j] + u[3 * i + 1] * u[3 * j + 1] + u[3 * i + 2] * u[3 * j + 2];
            if (dot >= cr) {
                nbr[offsets[i] + deg[i]++] = j;
                nbr[offsets[j] + deg[j]++] = i;
            }
        }
    free(u);
    free(deg);
    return 0;
}

int orc_peaks(const double* power, uint32_t n, const uint32_t* offsets, const uint32_t* nbr,
              uint32_t num_sources, float low_power_ratio, uint32_t* idx, double* pw, uint8_t* low,
              uint32_t* count) {
    if (num_sources == 0) return set_err(2, "num_sources must be at least 1");
    double mean = 0;
    for (uint32_t d = 0; d < n; ++d) mean += power[d];
    if (n) mean /= (double)n;
    uint32_t* peaks = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t np = 0;
    for (uint32_t d = 0; d < n; ++d) {
        int is_peak = 1;
        for (uint32_t k = offsets[d]; k < offsets[d + 1]; ++k)
            if (power[d] < power[nbr[k]]) {
                is_peak = 0;
                break;
            }
        if (is_peak) peaks[np++] = d;
    }
    /* stable order (power desc, index asc), then truncate (music.cpp:220-224) */
    for (uint32_t i = 1; i < np; ++i) {
        const uint32_t p = peaks[i];
        uint32_t j = i;
        while (j > 0 && (power[p] > power[peaks[j - 1]] ||
                         (power[p] == power[peaks[j - 1]] && p < peaks[j - 1]))) {
            peaks[j] = peaks[j - 1];
            --j;
        }
        peaks[j] = p;
    }
    if (np > num_sources) np = num_sources;
    const double thr = (double)low_power_ratio * mean;
    for (uint32_t i = 0; i < np; ++i) {
        idx[i] = peaks[i];
        pw[i] = power[peaks[i]];
        low[i] = power[peaks[i]] < thr ? 1 : 0;
    }
    *count = np;
    free(peaks);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* STFT front end                                                            */
/* ------------------------------------------------------------------------- */

/* make_window (stft.cpp:28-36): periodic Hann evaluated in double, rounded
 * to float once. */
void orc_window(int kind, uint32_t length, float* w) {
    for (uint32_t n = 0; n < length; ++n)
        w[n] = kind == 0 ? (float)(0.5 - 0.5 * cos(2.0 * M_PI * (double)n / (double)length)) : 1.0f;
}

/* fft_pow2<float> (fft.hpp:15-44): bit-reversal permutation, then radix-2
 * stages with the twiddle advanced by w *= wlen (complex<double>, textbook
 * product under -fcx-limited-range), butterflies in double, results rounded
 * to float after every stage. */
static void fft_pow2_f(float* re, float* im, uint32_t n) {
    for (uint32_t i = 1, j = 0; i < n; ++i) {
        uint32_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            float t = re[i]; re[i] = re[j]; re[j] = t;
            t = im[i]; im[i] = im[j]; im[j] = t;
        }
    }
    for (uint32_t len = 2; len <= n; len <<= 1) {
        const double ang = -2.0 * M_PI / (double)len;
        const cd wlen = c_make(cos(ang), sin(ang));
        for (uint32_t i = 0; i < n; i += len) {
            cd w = c_make(1.0, 0.0);
            for (uint32_t k = 0; k < len / 2; ++k) {
                const cd u = c_make(re[i + k], im[i + k]);
                const cd v = c_mul(c_make(re[i + k + len / 2], im[i + k + len / 2]), w);
                re[i + k] = (float)(u.re + v.re);
                im[i + k] = (float)(u.im + v.im);
                re[i + k + len / 2] = (float)(u.re - v.re);
                im[i + k + len / 2] = (float)(u.im - v.im);
                w = c_mul(w, wlen);
            }
        }
    }
}

int orc_stft(const float* pcm, uint32_t m, uint64_t nsamples, uint32_t frame_length, uint32_t shift, int window,
             uint32_t bin_min, uint32_t bin_max, float* frames, uint32_t* nframes) {
    /* StftConfig::validate (stft.cpp:9-16) */
    if (frame_length == 0) return set_err(2, "frame_length must be positive");
    if (shift == 0) return set_err(2, "shift must be positive");
    if (shift > frame_length) return set_err(2, "shift must not exceed frame_length");
    if (bin_min > bin_max) return set_err(2, "bin_min must not exceed bin_max");
    if (bin_max > frame_length / 2) return set_err(2, "bin_max exceeds the half spectrum of frame_length");
    /* stft_frame_count (stft.cpp:38-42) */
    const uint64_t nf = nsamples < frame_length ? 0 : (nsamples - frame_length) / shift + 1;
    if (nframes) *nframes = (uint32_t)nf;
    if (!frames) return 0;
    const uint32_t nb = bin_max - bin_min + 1;
    float* w = (float*)malloc(sizeof(float) * frame_length);
    float* re = (float*)malloc(sizeof(float) * frame_length);
    float* im = (float*)malloc(sizeof(float) * frame_length);
    orc_window(window, frame_length, w);
    for (uint64_t f = 0; f < nf; ++f)
        for (uint32_t c = 0; c < m; ++c) {
            const float* src = pcm + (uint64_t)c * nsamples + f * shift;  /* stft.cpp:49-53 */
            for (uint32_t i = 0; i < frame_length; ++i) {
                re[i] = src[i] * w[i];
                im[i] = 0.0f;
            }
            if (frame_length & (frame_length - 1)) {
                /* real_dft_half's direct sum for other lengths (fft.hpp:55-65):
                   FP64 accumulation in i order, the angle as the reference writes it */
                for (uint32_t b = 0; b < nb; ++b) {
                    const uint32_t k = bin_min + b;
                    double sr = 0, si = 0;
                    for (uint32_t i = 0; i < frame_length; ++i) {
                        const double ang = -2.0 * M_PI * (double)k * (double)i / (double)frame_length;
                        sr += (double)re[i] * cos(ang);
                        si += (double)re[i] * sin(ang);
                    }
                    frames[((f * m + c) * (uint64_t)nb + b) * 2] = (float)sr;
                    frames[((f * m + c) * (uint64_t)nb + b) * 2 + 1] = (float)si;
                }
                continue;
            }
            fft_pow2_f(re, im, frame_length);
            float* dst = frames + ((f * m + c) * (uint64_t)nb) * 2;  /* retained band (stft.cpp:55-56) */
            for (uint32_t b = 0; b < nb; ++b) {
                dst[2 * b] = re[bin_min + b];
                dst[2 * b + 1] = im[bin_min + b];
            }
        }
    free(w);
    free(re);
    free(im);
    return 0;
}
