/*
 * pn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference package's Gauss-Newton hot path
 * (polynewt, /root/reference/pkg/src/polynewt).  It exists to CHECK the CUDA
 * product path and to provide the CPU baseline timed by bench.py; it is never
 * linked into, loaded by, or called from the product library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (see oracle/Makefile).  -ffp-contract=off is essential: every product
 *        and sum of the reference is an individually rounded binary64 op.
 *
 * Parity is pinned against golden vectors produced by the Python reference
 * itself (tests/golden/make_golden.py) and against the reference's
 * known-answer tests (tests/test_oracle.py).
 *
 * Element layout (matches one column of polynewt.varith.VecContext planes):
 *   real    : c[0..nc-1]
 *   complex : re c[0..nc-1], im c[0..nc-1]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXC 8 /* doubles per element, complex qd */

/* ------------------------------------------------------------------------ */
/* L0: error-free transformations                       _eft.py:22-65        */

static const double kSplit = 134217729.0; /* 2^27 + 1, _eft.py:19 */

static inline void two_sum(double a, double b, double *s, double *e) {
    /* _eft.py:22-27 */
    double x = a + b;
    double bb = x - a;
    *e = (a - (x - bb)) + (b - bb);
    *s = x;
}

static inline void quick_two_sum(double a, double b, double *s, double *e) {
    /* _eft.py:30-34 */
    double x = a + b;
    *e = b - (x - a);
    *s = x;
}

static inline void dekker_split(double a, double *hi, double *lo) {
    /* _eft.py:37-41 */
    double t = kSplit * a;
    double h = t - (t - a);
    *hi = h;
    *lo = a - h;
}

static inline void two_prod(double a, double b, double *p, double *e) {
    /* _eft.py:44-50 -- Dekker form kept on purpose: the CUDA path uses the
     * FMA form, so agreement cross-checks SURVEY P1. */
    double x = a * b;
    double ah, al, bh, bl;
    dekker_split(a, &ah, &al);
    dekker_split(b, &bh, &bl);
    *e = (((ah * bh - x) + ah * bl) + al * bh) + al * bl;
    *p = x;
}

static inline void three_sum(double *a, double *b, double *c) {
    /* _eft.py:53-58: in/out (a,b,c) -> (s,u,v) */
    double t1, t2, s, t3, u, v;
    two_sum(*a, *b, &t1, &t2);
    two_sum(*c, t1, &s, &t3);
    two_sum(t2, t3, &u, &v);
    *a = s; *b = u; *c = v;
}

static inline void three_sum2(double *a, double *b, double c) {
    /* _eft.py:61-65: (a,b,c) -> (s, t2+t3) */
    double t1, t2, s, t3;
    two_sum(*a, *b, &t1, &t2);
    two_sum(c, t1, &s, &t3);
    *a = s; *b = t2 + t3;
}

/* ------------------------------------------------------------------------ */
/* double-double                                         _eft.py:72-126      */

static inline void dd_add(const double *a, const double *b, double *o) {
    /* _eft.py:72-78 */
    double s1, s2, t1, t2;
    two_sum(a[0], b[0], &s1, &s2);
    two_sum(a[1], b[1], &t1, &t2);
    s2 = s2 + t1;
    quick_two_sum(s1, s2, &s1, &s2);
    s2 = s2 + t2;
    quick_two_sum(s1, s2, &o[0], &o[1]);
}

static inline void dd_sub(const double *a, const double *b, double *o) {
    /* _eft.py:85-86 */
    double nb[2] = {-b[0], -b[1]};
    dd_add(a, nb, o);
}

static inline void dd_mul(const double *a, const double *b, double *o) {
    /* _eft.py:89-92 */
    double p, e;
    two_prod(a[0], b[0], &p, &e);
    e = e + (a[0] * b[1] + a[1] * b[0]);
    quick_two_sum(p, e, &o[0], &o[1]);
}

static void dd_div(const double *a, const double *b, double *o) {
    /* _eft.py:105-111 */
    static const double one[2] = {1.0, 0.0};
    double r[2] = {1.0 / b[0], 0.0}, t[2], e[2];
    for (int it = 0; it < 2; ++it) {
        dd_mul(b, r, t);
        dd_sub(one, t, e);
        dd_mul(r, e, t);
        dd_add(r, t, r);
    }
    dd_mul(a, r, o);
}

static void dd_sqrt(const double *a, double *o) {
    /* _eft.py:114-126 (caller filters a == 0) */
    static const double one[2] = {1.0, 0.0};
    static const double half[2] = {0.5, 0.0};
    double seed = 1.0 / sqrt(a[0]);
    double r[2] = {seed, 0.0 * seed}, t[2], u[2], e[2];
    for (int it = 0; it < 2; ++it) {
        dd_mul(r, r, t);
        dd_mul(a, t, u);
        dd_sub(one, u, e);
        dd_mul(r, e, t);
        dd_mul(half, t, u);
        dd_add(r, u, r);
    }
    dd_mul(a, r, o);
}

/* ------------------------------------------------------------------------ */
/* quad-double                                           _eft.py:134-275     */

static inline void renorm5(double c0, double c1, double c2, double c3, double c4,
                           double *o) {
    /* _eft.py:134-151 (scalar form; the masked array form 154-173 is equal) */
    double s, t1, t2, t3, t4, cur, e;
    quick_two_sum(c3, c4, &s, &t4);
    quick_two_sum(c2, s, &s, &t3);
    quick_two_sum(c1, s, &s, &t2);
    quick_two_sum(c0, s, &cur, &t1);
    double out[4] = {0.0, 0.0, 0.0, 0.0};
    int k = 0;
    double ts_[4] = {t1, t2, t3, t4};
    for (int i = 0; i < 4; ++i) {
        quick_two_sum(cur, ts_[i], &s, &e);
        if (e != 0.0 && k < 3) {
            out[k] = s;
            cur = e;
            k += 1;
        } else {
            cur = s;
        }
    }
    out[k] = cur;
    o[0] = out[0]; o[1] = out[1]; o[2] = out[2]; o[3] = out[3];
}

static void qd_add(const double *a, const double *b, double *o) {
    /* _eft.py:186-196 */
    double s1, s2, s3, s4, t1, t2, t3, t4;
    two_sum(a[0], b[0], &s1, &t1);
    two_sum(a[1], b[1], &s2, &t2);
    two_sum(a[2], b[2], &s3, &t3);
    two_sum(a[3], b[3], &s4, &t4);
    two_sum(s2, t1, &s2, &t1);
    three_sum(&s3, &t2, &t1);
    three_sum2(&s4, &t3, t2);
    t4 = (t4 + t3) + t1;
    renorm5(s1, s2, s3, s4, t4, o);
}

static void qd_sub(const double *a, const double *b, double *o) {
    /* _eft.py:203-204 */
    double nb[4] = {-b[0], -b[1], -b[2], -b[3]};
    qd_add(a, nb, o);
}

static void qd_mul(const double *a, const double *b, double *o) {
    /* _eft.py:207-250 */
    double a0 = a[0], a1 = a[1], a2 = a[2], a3 = a[3];
    double b0 = b[0], b1 = b[1], b2 = b[2], b3 = b[3];
    double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
    two_prod(a0, b0, &p0, &q0);
    two_prod(a0, b1, &p1, &q1);
    two_prod(a1, b0, &p2, &q2);
    two_prod(a0, b2, &p3, &q3);
    two_prod(a1, b1, &p4, &q4);
    two_prod(a2, b0, &p5, &q5);

    three_sum(&p1, &p2, &q0);

    three_sum(&p2, &q1, &q2);
    three_sum(&p3, &p4, &p5);
    double s0, t0, s1, t1, s2;
    two_sum(p2, p3, &s0, &t0);
    two_sum(q1, p4, &s1, &t1);
    s2 = q2 + p5;
    two_sum(s1, t0, &s1, &t0);
    s2 = s2 + (t0 + t1);

    double p6, q6, p7, q7, p8, q8, p9, q9;
    two_prod(a0, b3, &p6, &q6);
    two_prod(a1, b2, &p7, &q7);
    two_prod(a2, b1, &p8, &q8);
    two_prod(a3, b0, &p9, &q9);

    two_sum(q0, q3, &q0, &q3);
    two_sum(q4, q5, &q4, &q5);
    two_sum(p6, p7, &p6, &p7);
    two_sum(p8, p9, &p8, &p9);
    two_sum(q0, q4, &t0, &t1);
    t1 = t1 + (q3 + q5);
    double r0, r1;
    two_sum(p6, p8, &r0, &r1);
    r1 = r1 + (p7 + p9);
    two_sum(t0, r0, &q3, &q4);
    q4 = q4 + (t1 + r1);
    two_sum(q3, s1, &t0, &t1);
    t1 = t1 + q4;

    t1 = ((t1 + ((a1 * b3 + a2 * b2) + a3 * b1)) + (((q6 + q7) + q8) + q9)) + s2;

    renorm5(p0, p1, s0, t0, t1, o);
}

static void qd_div(const double *a, const double *b, double *o) {
    /* _eft.py:257-264 */
    static const double one[4] = {1.0, 0.0, 0.0, 0.0};
    double z = 0.0 * b[0];
    double r[4] = {1.0 / b[0], z, z, z}, t[4], e[4];
    for (int it = 0; it < 3; ++it) {
        qd_mul(b, r, t);
        qd_sub(one, t, e);
        qd_mul(r, e, t);
        qd_add(r, t, r);
    }
    qd_mul(a, r, o);
}

static void qd_sqrt(const double *a, double *o) {
    /* _eft.py:267-275 */
    static const double one[4] = {1.0, 0.0, 0.0, 0.0};
    static const double half[4] = {0.5, 0.0, 0.0, 0.0};
    double seed = 1.0 / sqrt(a[0]);
    double z = 0.0 * seed;
    double r[4] = {seed, z, z, z}, t[4], u[4], e[4];
    for (int it = 0; it < 3; ++it) {
        qd_mul(r, r, t);
        qd_mul(a, t, u);
        qd_sub(one, u, e);
        qd_mul(r, e, t);
        qd_mul(half, t, u);
        qd_add(r, u, r);
    }
    qd_mul(a, r, o);
}

/* ------------------------------------------------------------------------ */
/* L1: real field ops at nc components                   varith.py:19-62     */

static inline void f_add(int nc, const double *a, const double *b, double *o) {
    double t[4];
    if (nc == 1) { o[0] = a[0] + b[0]; return; }
    if (nc == 2) { dd_add(a, b, t); o[0] = t[0]; o[1] = t[1]; return; }
    qd_add(a, b, t); memcpy(o, t, sizeof(t));
}

static inline void f_sub(int nc, const double *a, const double *b, double *o) {
    double t[4];
    if (nc == 1) { o[0] = a[0] - b[0]; return; }
    if (nc == 2) { dd_sub(a, b, t); o[0] = t[0]; o[1] = t[1]; return; }
    qd_sub(a, b, t); memcpy(o, t, sizeof(t));
}

static inline void f_mul(int nc, const double *a, const double *b, double *o) {
    double t[4];
    if (nc == 1) { o[0] = a[0] * b[0]; return; }
    if (nc == 2) { dd_mul(a, b, t); o[0] = t[0]; o[1] = t[1]; return; }
    qd_mul(a, b, t); memcpy(o, t, sizeof(t));
}

static inline void f_div(int nc, const double *a, const double *b, double *o) {
    double t[4];
    if (nc == 1) { o[0] = a[0] / b[0]; return; }
    if (nc == 2) { dd_div(a, b, t); o[0] = t[0]; o[1] = t[1]; return; }
    qd_div(a, b, t); memcpy(o, t, sizeof(t));
}

static inline void f_sqrt(int nc, const double *a, double *o) {
    /* varith.py:51-62: zero is filtered to an all-zero result */
    double t[4];
    if (nc == 1) { o[0] = sqrt(a[0]); return; }
    if (a[0] == 0.0) { for (int c = 0; c < nc; ++c) o[c] = 0.0; return; }
    if (nc == 2) { dd_sqrt(a, t); o[0] = t[0]; o[1] = t[1]; return; }
    qd_sqrt(a, t); memcpy(o, t, sizeof(t));
}

/* ------------------------------------------------------------------------ */
/* element ops (real or complex)                  varith.py:104-156,        */
/*                                                xprec.py:287-328           */

typedef struct { int nc, cplx, es; } lvl_t;

static inline lvl_t mk_lvl(int nc, int cplx) {
    lvl_t L = {nc, cplx, cplx ? 2 * nc : nc};
    return L;
}

static inline void e_copy(lvl_t L, const double *a, double *o) { memcpy(o, a, sizeof(double) * L.es); }

static inline void e_add(lvl_t L, const double *a, const double *b, double *o) {
    f_add(L.nc, a, b, o);
    if (L.cplx) f_add(L.nc, a + L.nc, b + L.nc, o + L.nc);
}

static inline void e_sub(lvl_t L, const double *a, const double *b, double *o) {
    f_sub(L.nc, a, b, o);
    if (L.cplx) f_sub(L.nc, a + L.nc, b + L.nc, o + L.nc);
}

static inline void e_mul(lvl_t L, const double *a, const double *b, double *o) {
    /* varith.py:114-120 / xprec.py:302-306:
     * (ar*br - ai*bi, ar*bi + ai*br) */
    if (!L.cplx) { f_mul(L.nc, a, b, o); return; }
    int nc = L.nc;
    double t1[4], t2[4], re[4], im[4];
    f_mul(nc, a, b, t1);
    f_mul(nc, a + nc, b + nc, t2);
    f_sub(nc, t1, t2, re);
    f_mul(nc, a, b + nc, t1);
    f_mul(nc, a + nc, b, t2);
    f_add(nc, t1, t2, im);
    memcpy(o, re, sizeof(double) * nc);
    memcpy(o + nc, im, sizeof(double) * nc);
}

static inline void e_conj(lvl_t L, const double *a, double *o) {
    memcpy(o, a, sizeof(double) * L.es);
    if (L.cplx) for (int c = 0; c < L.nc; ++c) o[L.nc + c] = -a[L.nc + c];
}

static inline void e_div(lvl_t L, const double *a, const double *b, double *o) {
    /* varith.py:130-136 / xprec.py:310-317: (a*conj b)/(br^2+bi^2) */
    if (!L.cplx) { f_div(L.nc, a, b, o); return; }
    int nc = L.nc;
    double t1[4], t2[4], den[4], cb[8], num[8];
    f_mul(nc, b, b, t1);
    f_mul(nc, b + nc, b + nc, t2);
    f_add(nc, t1, t2, den);
    e_conj(L, b, cb);
    e_mul(L, a, cb, num);
    f_div(nc, num, den, o);
    f_div(nc, num + nc, den, o + nc);
}

static inline void e_div_real(lvl_t L, const double *a, const double *r, double *o) {
    /* varith.py:138-142 */
    f_div(L.nc, a, r, o);
    if (L.cplx) f_div(L.nc, a + L.nc, r, o + L.nc);
}

static inline void e_abs2(lvl_t L, const double *a, double *o) {
    /* varith.py:149-153: real component array */
    if (!L.cplx) { f_mul(L.nc, a, a, o); return; }
    double t1[4], t2[4];
    f_mul(L.nc, a, a, t1);
    f_mul(L.nc, a + L.nc, a + L.nc, t2);
    f_add(L.nc, t1, t2, o);
}

static inline void e_mul_int(lvl_t L, const double *a, int d, double *o) {
    /* xprec.py:36-49 + 302-304: scalar * int promotes d to (float(d), 0, ..)
     * and multiplies each part in the field */
    double dv[4] = {(double)d, 0.0, 0.0, 0.0};
    f_mul(L.nc, a, dv, o);
    if (L.cplx) f_mul(L.nc, a + L.nc, dv, o + L.nc);
}

/* tree_sum over n elements at stride `stride` (in elements).
 * varith.py:169-191 / evaldiff.py:205-212: level-by-level pairwise sum with
 * the odd tail carried to the next level. */
static void e_tree_sum(lvl_t L, long n, const double *a, long stride, double *o, double *scratch) {
    if (n <= 0) { memset(o, 0, sizeof(double) * L.es); return; }
    for (long i = 0; i < n; ++i) e_copy(L, a + i * stride * L.es, scratch + i * L.es);
    long len = n;
    while (len > 1) {
        long even = 2 * (len / 2), w = 0;
        for (long i = 0; i < even; i += 2, ++w)
            e_add(L, scratch + i * L.es, scratch + (i + 1) * L.es, scratch + w * L.es);
        if (len % 2) { e_copy(L, scratch + (len - 1) * L.es, scratch + w * L.es); ++w; }
        len = w;
    }
    e_copy(L, scratch, o);
}

static inline void r_tree_sum(int nc, long n, const double *a, double *o, double *scratch) {
    lvl_t R = mk_lvl(nc, 0);
    e_tree_sum(R, n, a, 1, o, scratch);
}

/* ------------------------------------------------------------------------ */
/* exported scalar/vector entry points (tests: varith parity)               */

int or_vec_op(int nc, int cplx, int op, long n, const double *a, const double *b, double *o) {
    lvl_t L = mk_lvl(nc, cplx);
    for (long i = 0; i < n; ++i) {
        const double *x = a + i * L.es, *y = b ? b + i * L.es : NULL;
        double *z = o + i * ((op == 4 || op == 5) ? L.nc : L.es); /* abs2/sqrt: real out */
        switch (op) {
        case 0: e_add(L, x, y, z); break;
        case 1: e_sub(L, x, y, z); break;
        case 2: e_mul(L, x, y, z); break;
        case 3: e_div(L, x, y, z); break;
        case 4: e_abs2(L, x, z); break;               /* writes nc doubles */
        case 5: f_sqrt(nc, x, z); break;              /* real input, nc doubles */
        case 6: e_conj(L, x, z); break;
        default: return -1;
        }
    }
    return 0;
}

int or_tree_sum(int nc, int cplx, long n, const double *a, double *o) {
    lvl_t L = mk_lvl(nc, cplx);
    double *scratch = (double *)malloc(sizeof(double) * L.es * (n > 0 ? n : 1));
    e_tree_sum(L, n, a, 1, o, scratch);
    free(scratch);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* L3 (1)+(2): monomial evaluation, product tree, gradient, accumulation     */

/* eval_product_tree + gradient_from_tree, evaldiff.py:53-108.
 * v: k input elements; root: product; grads: k elements.
 * work: scratch of at least 4*k elements.  Returns eval/grad mult counts. */
static void tree_eval_grad(lvl_t L, int k, const double *v, double *root, double *grads,
                           double *work, long long *em, long long *gm) {
    const int es = L.es;
    int base = 1;
    while (base * 2 <= k) base *= 2;
    int ell = k - base;
    /* levels stored back to back: level 0 has base slots, level j has base>>j */
    double *lv = work;
    for (int t = 0; t < base; ++t) e_copy(L, v + t * es, lv + t * es);
    for (int t = 0; t < ell; ++t) e_mul(L, v + t * es, v + (base + t) * es, lv + t * es);
    *em += ell;
    int nlev = 1;
    long off[32];
    off[0] = 0;
    long cur = 0, size = base;
    while (size > 1) {
        long s = size / 2, nxt = cur + size;
        for (long t = 0; t < s; ++t)
            e_mul(L, lv + (cur + t) * es, lv + (cur + t + s) * es, lv + (nxt + t) * es);
        *em += s;
        off[nlev++] = nxt;
        cur = nxt;
        size = s;
    }
    e_copy(L, lv + off[nlev - 1] * es, root);
    if (k == 1) { /* gradient of a single factor is one (never reached: k==1 bypass) */
        memset(grads, 0, sizeof(double) * es);
        grads[0] = 1.0;
        return;
    }
    /* comp = [levels[-2][1], levels[-2][0]] */
    double *comp = work + (2 * (long)base) * es;   /* base elements */
    double *nxtc = comp + (long)base * es;         /* base elements */
    long l2 = off[nlev - 2];
    e_copy(L, lv + (l2 + 1) * es, comp);
    e_copy(L, lv + l2 * es, comp + es);
    for (int j = nlev - 2; j >= 1; --j) {
        long prev = off[j - 1];
        long s = (long)base >> j; /* len(levels[j]) */
        for (long t = 0; t < s; ++t) {
            e_mul(L, comp + t * es, lv + (prev + t + s) * es, nxtc + t * es);
            e_mul(L, comp + t * es, lv + (prev + t) * es, nxtc + (t + s) * es);
        }
        *gm += 2 * s;
        memcpy(comp, nxtc, sizeof(double) * es * 2 * s);
    }
    for (int t = 0; t < base; ++t) {
        if (t < ell) {
            e_mul(L, comp + t * es, v + (base + t) * es, grads + t * es);
            e_mul(L, comp + t * es, v + t * es, grads + (base + t) * es);
            *gm += 2;
        } else {
            e_copy(L, comp + t * es, grads + t * es);
        }
    }
}

/*
 * Evaluate a canonicalised system (monomials of each poly already in
 * canonical order, polyrep.py:103-107) at x.  Restates evaluate_system,
 * evaldiff.py:215-266 with eval_monomial_and_derivs 142-180 and
 * build_power_table / eval_common_factor polyrep.py:120-139.
 *
 * poly_ptr[m+1] -> monomial ranges; mon_ptr[M+1] -> support ranges;
 * var_idx/exps[nnz]; coeffs[M*es]; x[n*es]; f[m*es]; J[m*n*es] row-major.
 * counts[2] += (eval_mults, grad_mults).
 */
int or_evaluate(int nc, int cplx, int m, int n, const int *poly_ptr, const int *mon_ptr,
                const int *var_idx, const int *exps, const double *coeffs, const double *x,
                double *f, double *J, long long *counts, int nthreads) {
    lvl_t L = mk_lvl(nc, cplx);
    const int es = L.es;
    long M = poly_ptr[m];
    long nnz = mon_ptr[M];
    /* power table: max exponent per variable over the system */
    int *maxdeg = (int *)calloc(n, sizeof(int));
    for (long t = 0; t < nnz; ++t)
        if (exps[t] > maxdeg[var_idx[t]]) maxdeg[var_idx[t]] = exps[t];
    long *toff = (long *)malloc(sizeof(long) * (n + 1));
    toff[0] = 0;
    for (int v = 0; v < n; ++v) toff[v + 1] = toff[v] + maxdeg[v];
    double *table = (double *)malloc(sizeof(double) * es * (toff[n] > 0 ? toff[n] : 1));
    for (int v = 0; v < n; ++v) {
        if (maxdeg[v] == 0) continue;
        double *row = table + toff[v] * es; /* row[d-1] = x^d */
        e_copy(L, x + (long)v * es, row);
        for (int d = 2; d <= maxdeg[v]; ++d)
            e_mul(L, row + (d - 2) * es, x + (long)v * es, row + (d - 1) * es);
    }
    /* per monomial: value + derivative contributions (in support order) */
    double *mval = (double *)malloc(sizeof(double) * es * (M > 0 ? M : 1));
    double *dval = (double *)malloc(sizeof(double) * es * (nnz > 0 ? nnz : 1));
    int kmax = 1;
    for (long i = 0; i < M; ++i) {
        int k = mon_ptr[i + 1] - mon_ptr[i];
        if (k > kmax) kmax = k;
    }
    long long em = 0, gm = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads) reduction(+ : em, gm)
#endif
    {
        double *vals = (double *)malloc(sizeof(double) * es * kmax);
        double *grads = (double *)malloc(sizeof(double) * es * kmax);
        double *work = (double *)malloc(sizeof(double) * es * 4 * (kmax + 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
        for (long i = 0; i < M; ++i) {
            const int lo = mon_ptr[i], k = mon_ptr[i + 1] - lo;
            const double *coeff = coeffs + i * es;
            double *value = mval + i * es;
            if (k == 0) { e_copy(L, coeff, value); continue; }
            if (k == 1) {
                int v = var_idx[lo], d = exps[lo];
                const double *row = table + toff[v] * es;
                e_mul(L, coeff, row + (d - 1) * es, value);
                em += 1;
                double dco[8];
                e_mul_int(L, coeff, d, dco);
                if (d == 1) e_copy(L, dco, dval + (long)lo * es);
                else { e_mul(L, dco, row + (d - 2) * es, dval + (long)lo * es); gm += 1; }
                continue;
            }
            /* common factor: left fold of table[var][d-1] over d >= 2 */
            double common[8], t8[8];
            int have_common = 0, c = 0;
            for (int p = 0; p < k; ++p) {
                int v = var_idx[lo + p], d = exps[lo + p];
                if (d < 2) continue;
                const double *pw = table + (toff[v] + d - 2) * es;
                if (!have_common) { e_copy(L, pw, common); have_common = 1; }
                else { e_mul(L, common, pw, t8); e_copy(L, t8, common); }
                ++c;
            }
            for (int p = 0; p < k; ++p) e_copy(L, x + (long)var_idx[lo + p] * es, vals + p * es);
            double root[8], scale[8];
            tree_eval_grad(L, k, vals, root, grads, work, &em, &gm);
            if (have_common) { e_mul(L, coeff, common, scale); em += 1 + (c - 1 > 0 ? c - 1 : 0); }
            else e_copy(L, coeff, scale);
            e_mul(L, scale, root, value);
            em += 1;
            for (int p = 0; p < k; ++p) {
                int d = exps[lo + p];
                double ds[8];
                if (d == 1) e_copy(L, scale, ds);
                else e_mul_int(L, scale, d, ds);
                e_mul(L, ds, grads + p * es, dval + (long)(lo + p) * es);
                gm += 1 + (d > 1 ? 1 : 0);
            }
        }
        free(vals); free(grads); free(work);
    }
    /* accumulate per polynomial: values and Jacobian rows */
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int *cnt = (int *)malloc(sizeof(int) * (n + 1));
        int *pos = (int *)malloc(sizeof(int) * (n + 1));
        long cap = 1024;
        long *lst = (long *)malloc(sizeof(long) * cap);
        double *buf = (double *)malloc(sizeof(double) * es * cap);
        double *scr = (double *)malloc(sizeof(double) * es * cap);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int i = 0; i < m; ++i) {
            long m0 = poly_ptr[i], m1 = poly_ptr[i + 1];
            long T = m1 - m0;
            long need = T;
            long nz = mon_ptr[m1] - mon_ptr[m0];
            if (nz > need) need = nz;
            if (need > cap) {
                cap = need;
                lst = (long *)realloc(lst, sizeof(long) * cap);
                buf = (double *)realloc(buf, sizeof(double) * es * cap);
                scr = (double *)realloc(scr, sizeof(double) * es * cap);
            }
            /* value: tree over monomial values in canonical order */
            if (T > 0) e_tree_sum(L, T, mval + m0 * es, 1, f + (long)i * es, scr);
            else memset(f + (long)i * es, 0, sizeof(double) * es);
            double *row = J + (long)i * n * es;
            memset(row, 0, sizeof(double) * es * n);
            memset(cnt, 0, sizeof(int) * (n + 1));
            for (long t = mon_ptr[m0]; t < mon_ptr[m1]; ++t) cnt[var_idx[t] + 1]++;
            for (int v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
            memcpy(pos, cnt, sizeof(int) * (n + 1));
            for (long t = mon_ptr[m0]; t < mon_ptr[m1]; ++t) lst[pos[var_idx[t]]++] = t;
            for (int v = 0; v < n; ++v) {
                int a = cnt[v], b = cnt[v + 1];
                if (b == a) continue;
                for (int q = a; q < b; ++q) e_copy(L, dval + lst[q] * es, buf + (q - a) * es);
                e_tree_sum(L, b - a, buf, 1, row + (long)v * es, scr);
            }
        }
        free(cnt); free(pos); free(lst); free(buf); free(scr);
    }
    if (counts) { counts[0] += em; counts[1] += gm; }
    free(maxdeg); free(toff); free(table); free(mval); free(dval);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* L3 (3): modified Gram-Schmidt least squares                mgs.py:145-305 */

static double eps_of(int nc) { return nc == 1 ? ldexp(1.0, -53) : nc == 2 ? ldexp(1.0, -104) : ldexp(1.0, -209); }

/* column norm: sqrt(tree_sum(abs2(col))), mgs.py:128-137.  A is row-major
 * m x ncols elements; column j. */
static void col_norm(lvl_t L, int m, int ncols, const double *A, int j, double *out, double *scr) {
    double *a2 = scr;                 /* m real elements */
    double *s2 = scr + (long)m * L.nc; /* tree scratch */
    for (int i = 0; i < m; ++i) e_abs2(L, A + ((long)i * ncols + j) * L.es, a2 + (long)i * L.nc);
    double t[4];
    r_tree_sum(L.nc, m, a2, t, s2);
    f_sqrt(L.nc, t, out);
}

/*
 * aug: m x (n+1) row-major elements (modified copy made internally).
 * Q: m x n row-major (nullable); R: (n+1) x (n+1) row-major (zeroed here).
 * Returns 0, or 1 on MgsBreakdownError with info[0]=k, info[1]=rkk_hi,
 * info[2]=threshold.  Restates mgs_qr (immediate variant), mgs.py:145-221.
 */
int or_mgs_qr(int nc, int cplx, int m, int n, const double *aug, double *Q, double *R, double *info,
              int nthreads) {
    lvl_t L = mk_lvl(nc, cplx);
    const int es = L.es, nc1 = n + 1;
    if (!(m >= n && n >= 1)) return -1;
    double *A = (double *)malloc(sizeof(double) * es * (long)m * nc1);
    memcpy(A, aug, sizeof(double) * es * (long)m * nc1);
    if (Q) memset(Q, 0, sizeof(double) * es * (long)m * n);
    memset(R, 0, sizeof(double) * es * (long)nc1 * nc1);
    double *orig = (double *)malloc(sizeof(double) * n);
    double *scr = (double *)malloc(sizeof(double) * es * 2 * ((long)m + 1));
    const double eps = eps_of(nc);
    for (int k = 0; k < n; ++k) {
        double t[4];
        col_norm(L, m, nc1, A, k, t, scr);
        orig[k] = t[0];
    }
    double *q = (double *)malloc(sizeof(double) * es * (long)m);
    int rc = 0;
    for (int k = 0; k <= n; ++k) {
        double rkk[4];
        col_norm(L, m, nc1, A, k, rkk, scr);
        if (k < n) {
            double thr = ((1.0 * (double)n) * eps) * orig[k];
            if (rkk[0] <= thr) {
                if (info) { info[0] = k; info[1] = rkk[0]; info[2] = thr; }
                rc = 1;
                break;
            }
        }
        double *Rkk = R + ((long)k * nc1 + k) * es;
        memcpy(Rkk, rkk, sizeof(double) * nc);
        if (k >= n) break;
        for (int i = 0; i < m; ++i) e_div_real(L, A + ((long)i * nc1 + k) * es, rkk, q + (long)i * es);
        if (Q)
            for (int i = 0; i < m; ++i) e_copy(L, q + (long)i * es, Q + ((long)i * n + k) * es);
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
#endif
        {
            double *pr = (double *)malloc(sizeof(double) * es * 2 * ((long)m + 1));
            double *sc = pr + (long)m * es + es;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
            for (int j = k + 1; j <= n; ++j) {
                double qc[8], r[8], t[8];
                for (int i = 0; i < m; ++i) {
                    e_conj(L, q + (long)i * es, qc);
                    e_mul(L, qc, A + ((long)i * nc1 + j) * es, pr + (long)i * es);
                }
                e_tree_sum(L, m, pr, 1, r, sc);
                for (int i = 0; i < m; ++i) {
                    double *aij = A + ((long)i * nc1 + j) * es;
                    e_mul(L, q + (long)i * es, r, t);
                    e_sub(L, aij, t, aij);
                }
                e_copy(L, r, R + ((long)k * nc1 + j) * es);
            }
            free(pr);
        }
    }
    free(A); free(orig); free(scr); free(q);
    return rc;
}

/* back substitution R x = y, mgs.py:229-247 (staged variant 250-289 is
 * bit-identical).  R: (n+1)x(n+1) augmented factor (leading n x n used),
 * y = R[:n, n].  Returns 0, or 2 on SingularMatrixError (info[0] = j). */
int or_back_substitute(int nc, int cplx, int n, const double *R, double *x, double *info) {
    lvl_t L = mk_lvl(nc, cplx);
    const int es = L.es, nc1 = n + 1;
    double *yw = (double *)malloc(sizeof(double) * es * n);
    for (int i = 0; i < n; ++i) e_copy(L, R + ((long)i * nc1 + n) * es, yw + (long)i * es);
    int rc = 0;
    for (int j = n - 1; j >= 0; --j) {
        const double *diag = R + ((long)j * nc1 + j) * es;
        int nz = 0;
        for (int c = 0; c < es; ++c) nz |= diag[c] != 0.0;
        if (!nz) { if (info) info[0] = j; rc = 2; break; }
        e_div(L, yw + (long)j * es, diag, x + (long)j * es);
        for (int i = 0; i < j; ++i) {
            double t[8];
            e_mul(L, R + ((long)i * nc1 + j) * es, x + (long)j * es, t);
            e_sub(L, yw + (long)i * es, t, yw + (long)i * es);
        }
    }
    free(yw);
    return rc;
}

/* least_squares_solve, mgs.py:299-305.  z_out = hi(R[n,n].re). */
int or_least_squares(int nc, int cplx, int m, int n, const double *aug, double *Q, double *R, double *x,
                     double *z_out, double *info, int nthreads) {
    int rc = or_mgs_qr(nc, cplx, m, n, aug, Q, R, info, nthreads);
    if (rc) return rc;
    lvl_t L = mk_lvl(nc, cplx);
    if (z_out) *z_out = R[((long)n * (n + 1) + n) * L.es];
    return or_back_substitute(nc, cplx, n, R, x, info);
}

/* newton_step, newton.py:82-103: f, J at x; [J | -f]; LSQ; x_next = x + dx.
 * Outputs f (m), dx (n), x_next (n).  work must hold m*(n+1) + (n+1)^2 elems. */
int or_newton_step(int nc, int cplx, int m, int n, const int *poly_ptr, const int *mon_ptr,
                   const int *var_idx, const int *exps, const double *coeffs, const double *x,
                   double *f, double *dx, double *x_next, double *info, long long *counts, int nthreads) {
    lvl_t L = mk_lvl(nc, cplx);
    const int es = L.es, nc1 = n + 1;
    double *J = (double *)malloc(sizeof(double) * es * (long)m * n);
    double *aug = (double *)malloc(sizeof(double) * es * (long)m * nc1);
    double *R = (double *)malloc(sizeof(double) * es * (long)nc1 * nc1);
    or_evaluate(nc, cplx, m, n, poly_ptr, mon_ptr, var_idx, exps, coeffs, x, f, J, counts, nthreads);
    for (int i = 0; i < m; ++i) {
        memcpy(aug + (long)i * nc1 * es, J + (long)i * n * es, sizeof(double) * es * n);
        double *b = aug + ((long)i * nc1 + n) * es;
        for (int c = 0; c < es; ++c) b[c] = -f[(long)i * es + c];
    }
    int rc = or_least_squares(nc, cplx, m, n, aug, NULL, R, dx, NULL, info, nthreads);
    if (!rc)
        for (int j = 0; j < n; ++j) e_add(L, x + (long)j * es, dx + (long)j * es, x_next + (long)j * es);
    free(J); free(aug); free(R);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Synthetic input family F(n, T, k, seed, maxexp, m[, kmin]).
 * The reference has no random sparse generator (its bench.py:98-110 only
 * builds full-product stress monomials); this is an independent C
 * restatement of the builder-defined family so that bench.py's
 * --impl reference arm builds its inputs without loading the product
 * library.  splitmix64 stream, Floyd's k-subset, sorted variables, exponents
 * 1 + below(maxexp), coefficient parts (0.5 + 1.5 u) with a random sign.
 * kmin < k: the variable count is drawn first, uniform in [kmin, k].
 * tests/test_host.py checks it array-for-array against the product's
 * pn_generate_random_system. */
static uint64_t sm_state;
static uint64_t sm_next(void) {
    uint64_t z = (sm_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint32_t sm_below(uint32_t bound) { return (uint32_t)(((unsigned __int128)sm_next() * bound) >> 64); }
static double sm_uniform(void) { return (double)(sm_next() >> 11) * 0x1.0p-53; }

int or_generate_random_system(int m, int n, int T, int kmin, int k, int maxexp, uint64_t seed, int *poly_ptr,
                              int *mon_ptr, int *var_idx, int *exps, double *coef_re, double *coef_im) {
    if (m < 0 || n < 1 || T < 0 || kmin < 0 || kmin > k || k > n || maxexp < 1) return -1;
    sm_state = seed * 0x2545F4914F6CDD1Dull + 0x1234567ull;
    int *pick = (int *)malloc(sizeof(int) * (k > 0 ? k : 1));
    long mon = 0, ent = 0;
    poly_ptr[0] = 0;
    mon_ptr[0] = 0;
    for (int i = 0; i < m; ++i) {
        for (int t = 0; t < T; ++t) {
            int kt = kmin < k ? kmin + (int)sm_below((uint32_t)(k - kmin + 1)) : k;
            int cnt = 0;
            for (int j = n - kt; j < n; ++j) {
                int r = (int)sm_below((uint32_t)j + 1), seen = 0;
                for (int q = 0; q < cnt; ++q) seen |= pick[q] == r;
                /* insertion keeps pick sorted */
                int v = seen ? j : r, q = cnt++;
                while (q > 0 && pick[q - 1] > v) { pick[q] = pick[q - 1]; --q; }
                pick[q] = v;
            }
            for (int q = 0; q < cnt; ++q) {
                var_idx[ent] = pick[q];
                exps[ent] = 1 + (int)sm_below((uint32_t)maxexp);
                ++ent;
            }
            double re = 0.5 + 1.5 * sm_uniform();
            if (sm_next() & 1) re = -re;
            double im = 0.5 + 1.5 * sm_uniform();
            if (sm_next() & 1) im = -im;
            coef_re[mon] = re;
            if (coef_im) coef_im[mon] = im;
            mon_ptr[++mon] = (int)ent;
        }
        poly_ptr[i + 1] = (int)mon;
    }
    free(pick);
    return 0;
}

int or_version(void) { return 1; }
