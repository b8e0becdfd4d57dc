// xprec.cuh -- device extended-precision arithmetic (double, double-double,
// quad-double; real and complex) replaying the reference's exact binary64
// operation sequence.
//
// Reference semantics: /root/reference/pkg/src/polynewt/_eft.py (L0),
// varith.py:19-156 and xprec.py:278-328 (L1).  Parity rules (SURVEY 8(a')):
//  * every sum/product is an individually rounded binary64 op: we use the
//    __dadd_rn/__dsub_rn/__dmul_rn intrinsics, which ptxas never contracts
//    into FMA, independently of -fmad;
//  * two_prod is p = a*b, e = fma(a, b, -p): bit-identical to the reference's
//    Dekker split form, 2 instructions instead of 17;
//  * reciprocal seeds use IEEE division/sqrt (__ddiv_rn, __dsqrt_rn), never
//    rsqrt or fast reciprocals;
//  * dd/qd division is mul(a, recip(b)) with recip depending on b only
//    (_eft.py:105-111, 257-264), so callers may hoist the reciprocal;
//    complex-double division stays per-element IEEE (varith.py:43-46);
//  * renorm5's data-dependent branch is reproduced by predication
//    (_eft.py:134-173);
//  * operand order follows the reference everywhere.
#pragma once
#include <cuda_runtime.h>

namespace pn {

#define PN_DI __device__ __forceinline__
#define PN_HDI __host__ __device__ __forceinline__

PN_DI double dadd(double a, double b) { return __dadd_rn(a, b); }
PN_DI double dsub(double a, double b) { return __dsub_rn(a, b); }
PN_DI double dmul(double a, double b) { return __dmul_rn(a, b); }
PN_DI double ddiv(double a, double b) { return __ddiv_rn(a, b); }
PN_DI double dsqrt(double a) { return __dsqrt_rn(a); }
// sign flip and "!= 0.0" on the integer pipes: exact, and they keep the FP64
// pipe (the bottleneck of every dd/qd kernel) for the arithmetic itself
PN_DI double dneg(double x) { return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x)); }
PN_DI bool dnz(double x) { return ((__double2hiint(x) & 0x7fffffff) | __double2loint(x)) != 0; }

// ---------------------------------------------------------------------------
// L0 error-free transforms (_eft.py:22-65)

PN_DI void two_sum(double a, double b, double &s, double &e) {
  double x = dadd(a, b);
  double bb = dsub(x, a);
  e = dadd(dsub(a, dsub(x, bb)), dsub(b, bb));
  s = x;
}

PN_DI void quick_two_sum(double a, double b, double &s, double &e) {
  double x = dadd(a, b);
  e = dsub(b, dsub(x, a));
  s = x;
}

PN_DI void two_prod(double a, double b, double &p, double &e) {
  double x = dmul(a, b);
  e = fma(a, b, -x);
  p = x;
}

// (a,b,c) -> (s,u,v)
PN_DI void three_sum(double &a, double &b, double &c) {
  double t1, t2, s, t3, u, v;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, s, t3);
  two_sum(t2, t3, u, v);
  a = s; b = u; c = v;
}

// (a,b,c) -> (s, t2+t3)
PN_DI void three_sum2(double &a, double &b, double c) {
  double t1, t2, s, t3;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, s, t3);
  a = s; b = dadd(t2, t3);
}

// ---------------------------------------------------------------------------
// real field elements with NC binary64 components

template <int NC> struct F { double c[NC]; };

template <int NC> PN_DI F<NC> fzero() { F<NC> r; _Pragma("unroll") for (int i = 0; i < NC; ++i) r.c[i] = 0.0; return r; }
template <int NC> PN_DI F<NC> fconst(double v) { F<NC> r = fzero<NC>(); r.c[0] = v; return r; }
template <int NC> PN_DI F<NC> fneg(const F<NC> &a) { F<NC> r; _Pragma("unroll") for (int i = 0; i < NC; ++i) r.c[i] = dneg(a.c[i]); return r; }

// ---- double (NC = 1): plain IEEE ops ------------------------------------
PN_DI F<1> fadd(const F<1> &a, const F<1> &b) { F<1> r; r.c[0] = dadd(a.c[0], b.c[0]); return r; }
PN_DI F<1> fsub(const F<1> &a, const F<1> &b) { F<1> r; r.c[0] = dsub(a.c[0], b.c[0]); return r; }
PN_DI F<1> fmul(const F<1> &a, const F<1> &b) { F<1> r; r.c[0] = dmul(a.c[0], b.c[0]); return r; }

// ---- double-double (_eft.py:72-126) -------------------------------------
PN_DI F<2> fadd(const F<2> &a, const F<2> &b) {
  double s1, s2, t1, t2;
  two_sum(a.c[0], b.c[0], s1, s2);
  two_sum(a.c[1], b.c[1], t1, t2);
  s2 = dadd(s2, t1);
  quick_two_sum(s1, s2, s1, s2);
  s2 = dadd(s2, t2);
  F<2> r;
  quick_two_sum(s1, s2, r.c[0], r.c[1]);
  return r;
}
PN_DI F<2> fsub(const F<2> &a, const F<2> &b) { return fadd(a, fneg(b)); }
PN_DI F<2> fmul(const F<2> &a, const F<2> &b) {
  double p, e;
  two_prod(a.c[0], b.c[0], p, e);
  e = dadd(e, dadd(dmul(a.c[0], b.c[1]), dmul(a.c[1], b.c[0])));
  F<2> r;
  quick_two_sum(p, e, r.c[0], r.c[1]);
  return r;
}

// ---- quad-double (_eft.py:134-275) --------------------------------------
PN_DI F<4> renorm5(double c0, double c1, double c2, double c3, double c4) {
  double s, t1, t2, t3, t4, cur, e;
  quick_two_sum(c3, c4, s, t4);
  quick_two_sum(c2, s, s, t3);
  quick_two_sum(c1, s, s, t2);
  quick_two_sum(c0, s, cur, t1);
  F<4> r;
  // Common case: the first three steps all leave a nonzero error term, so
  // every step "advances" and the fourth folds into the last slot
  // (_eft.py:142-150 with k reaching 3).  Same operations as the general
  // path below; the branch is warp-uniform on generic data.
  {
    double s1, e1, s2, e2, s3, e3;
    quick_two_sum(cur, t1, s1, e1);
    quick_two_sum(e1, t2, s2, e2);
    quick_two_sum(e2, t3, s3, e3);
    if (dnz(e1) && dnz(e2) && dnz(e3)) {
      r.c[0] = s1; r.c[1] = s2; r.c[2] = s3; r.c[3] = dadd(e3, t4);
      return r;
    }
  }
  double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
  int k = 0;
  const double tv[4] = {t1, t2, t3, t4};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    quick_two_sum(cur, tv[i], s, e);
    const bool adv = dnz(e) && (k < 3);
    o0 = (adv && k == 0) ? s : o0;
    o1 = (adv && k == 1) ? s : o1;
    o2 = (adv && k == 2) ? s : o2;
    cur = adv ? e : s;
    k += adv ? 1 : 0;
  }
  o0 = (k == 0) ? cur : o0;
  o1 = (k == 1) ? cur : o1;
  o2 = (k == 2) ? cur : o2;
  o3 = (k == 3) ? cur : o3;
  r.c[0] = o0; r.c[1] = o1; r.c[2] = o2; r.c[3] = o3;
  return r;
}

#ifndef PN_QD_CALL
#define PN_QD_CALL static __device__ __noinline__
#endif

PN_DI F<4> qd_add_body(const F<4> &a, const F<4> &b) {
  double s1, s2, s3, s4, t1, t2, t3, t4;
  two_sum(a.c[0], b.c[0], s1, t1);
  two_sum(a.c[1], b.c[1], s2, t2);
  two_sum(a.c[2], b.c[2], s3, t3);
  two_sum(a.c[3], b.c[3], s4, t4);
  two_sum(s2, t1, s2, t1);
  three_sum(s3, t2, t1);
  three_sum2(s4, t3, t2);
  t4 = dadd(dadd(t4, t3), t1);
  return renorm5(s1, s2, s3, s4, t4);
}
PN_DI F<4> qd_mul_body(const F<4> &a, const F<4> &b) {
  const double a0 = a.c[0], a1 = a.c[1], a2 = a.c[2], a3 = a.c[3];
  const double b0 = b.c[0], b1 = b.c[1], b2 = b.c[2], b3 = b.c[3];
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
  two_prod(a0, b0, p0, q0);
  two_prod(a0, b1, p1, q1);
  two_prod(a1, b0, p2, q2);
  two_prod(a0, b2, p3, q3);
  two_prod(a1, b1, p4, q4);
  two_prod(a2, b0, p5, q5);
  three_sum(p1, p2, q0);
  // six-three sum of p2, q1, q2, p3, p4, p5
  three_sum(p2, q1, q2);
  three_sum(p3, p4, p5);
  double s0, t0, s1, t1, s2;
  two_sum(p2, p3, s0, t0);
  two_sum(q1, p4, s1, t1);
  s2 = dadd(q2, p5);
  two_sum(s1, t0, s1, t0);
  s2 = dadd(s2, dadd(t0, t1));
  double p6, q6, p7, q7, p8, q8, p9, q9;
  two_prod(a0, b3, p6, q6);
  two_prod(a1, b2, p7, q7);
  two_prod(a2, b1, p8, q8);
  two_prod(a3, b0, p9, q9);
  // nine-two sum of q0, s1, q3..q5, p6..p9
  two_sum(q0, q3, q0, q3);
  two_sum(q4, q5, q4, q5);
  two_sum(p6, p7, p6, p7);
  two_sum(p8, p9, p8, p9);
  two_sum(q0, q4, t0, t1);
  t1 = dadd(t1, dadd(q3, q5));
  double r0, r1;
  two_sum(p6, p8, r0, r1);
  r1 = dadd(r1, dadd(p7, p9));
  two_sum(t0, r0, q3, q4);
  q4 = dadd(q4, dadd(t1, r1));
  two_sum(q3, s1, t0, t1);
  t1 = dadd(t1, q4);
  // O(eps^4) terms
  const double u = dadd(dadd(dmul(a1, b3), dmul(a2, b2)), dmul(a3, b1));
  const double w = dadd(dadd(dadd(q6, q7), q8), q9);
  t1 = dadd(dadd(dadd(t1, u), w), s2);
  return renorm5(p0, p1, s0, t0, t1);
}

// The quad-double primitives are out-of-line calls by default: a fully
// inlined complex-qd kernel is >1 MB of SASS and stalls on instruction fetch
// (ncu: stall_no_inst 35-45%); one shared copy of each primitive fits the
// instruction cache.
PN_QD_CALL F<4> qd_add_call(F<4> a, F<4> b) { return qd_add_body(a, b); }
PN_QD_CALL F<4> qd_mul_call(F<4> a, F<4> b) { return qd_mul_body(a, b); }
PN_DI F<4> fadd(const F<4> &a, const F<4> &b) { return qd_add_call(a, b); }
PN_DI F<4> fsub(const F<4> &a, const F<4> &b) { return qd_add_call(a, fneg(b)); }
PN_DI F<4> fmul(const F<4> &a, const F<4> &b) { return qd_mul_call(a, b); }

// ---- reciprocal / division / sqrt ---------------------------------------
// recip(b) is the Newton-refined reciprocal of the reference's division;
// div(a, b) == mul(a, recip(b)) bit-for-bit (_eft.py:105-111, 257-264).
PN_DI F<2> frecip(const F<2> &b) {
  F<2> r; r.c[0] = ddiv(1.0, b.c[0]); r.c[1] = 0.0;
  const F<2> one = fconst<2>(1.0);
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    F<2> e = fsub(one, fmul(b, r));
    r = fadd(r, fmul(r, e));
  }
  return r;
}
PN_DI F<4> frecip(const F<4> &b) {
  const double z = dmul(0.0, b.c[0]);
  F<4> r; r.c[0] = ddiv(1.0, b.c[0]); r.c[1] = z; r.c[2] = z; r.c[3] = z;
  const F<4> one = fconst<4>(1.0);
#pragma unroll 1
  for (int it = 0; it < 3; ++it) {
    F<4> e = fsub(one, fmul(b, r));
    r = fadd(r, fmul(r, e));
  }
  return r;
}
PN_DI F<1> fdiv(const F<1> &a, const F<1> &b) { F<1> r; r.c[0] = ddiv(a.c[0], b.c[0]); return r; }
PN_DI F<2> fdiv(const F<2> &a, const F<2> &b) { return fmul(a, frecip(b)); }
PN_DI F<4> fdiv(const F<4> &a, const F<4> &b) { return fmul(a, frecip(b)); }

// sqrt_real semantics (varith.py:51-62): nc == 1 -> IEEE sqrt; otherwise an
// exact zero hi component maps to all-zero, else the rsqrt Newton iteration.
PN_DI F<1> fsqrt(const F<1> &a) { F<1> r; r.c[0] = dsqrt(a.c[0]); return r; }
PN_DI F<2> fsqrt(const F<2> &a) {
  if (a.c[0] == 0.0) return fzero<2>();
  const double seed = ddiv(1.0, dsqrt(a.c[0]));
  F<2> r; r.c[0] = seed; r.c[1] = dmul(0.0, seed);
  const F<2> one = fconst<2>(1.0), half = fconst<2>(0.5);
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    F<2> e = fsub(one, fmul(a, fmul(r, r)));
    r = fadd(r, fmul(half, fmul(r, e)));
  }
  return fmul(a, r);
}
PN_DI F<4> fsqrt(const F<4> &a) {
  if (a.c[0] == 0.0) return fzero<4>();
  const double seed = ddiv(1.0, dsqrt(a.c[0]));
  const double z = dmul(0.0, seed);
  F<4> r; r.c[0] = seed; r.c[1] = z; r.c[2] = z; r.c[3] = z;
  const F<4> one = fconst<4>(1.0), half = fconst<4>(0.5);
#pragma unroll 1
  for (int it = 0; it < 3; ++it) {
    F<4> e = fsub(one, fmul(a, fmul(r, r)));
    r = fadd(r, fmul(half, fmul(r, e)));
  }
  return fmul(a, r);
}

// ---------------------------------------------------------------------------
// complex elements over F<NC> (varith.py:104-156, xprec.py:287-328)

template <int NC> struct C { F<NC> re, im; };

template <int NC> PN_DI C<NC> cadd(const C<NC> &a, const C<NC> &b) { return {fadd(a.re, b.re), fadd(a.im, b.im)}; }
template <int NC> PN_DI C<NC> csub(const C<NC> &a, const C<NC> &b) { return {fsub(a.re, b.re), fsub(a.im, b.im)}; }
// (ar*br - ai*bi, ar*bi + ai*br), evaluated in exactly that order
template <int NC> PN_DI C<NC> cmul(const C<NC> &a, const C<NC> &b) {
  F<NC> t1 = fmul(a.re, b.re);
  F<NC> t2 = fmul(a.im, b.im);
  F<NC> re = fsub(t1, t2);
  F<NC> t3 = fmul(a.re, b.im);
  F<NC> t4 = fmul(a.im, b.re);
  return {re, fadd(t3, t4)};
}
template <int NC> PN_DI C<NC> cconj(const C<NC> &a) { return {a.re, fneg(a.im)}; }

#ifndef PN_QD_MODE
#define PN_QD_MODE 1
#endif
#if PN_QD_MODE == 1
// Complex quad-double ops as single out-of-line units: the four real products
// of a complex multiply are independent, so inlining them inside one call
// lets the scheduler interleave them, while each kernel keeps one copy of the
// code (instruction-cache friendly) and pays one call per 914 FP64 instr.
PN_QD_CALL C<4> c4_mul_call(C<4> a, C<4> b) {
  const F<4> t1 = qd_mul_body(a.re, b.re);
  const F<4> t2 = qd_mul_body(a.im, b.im);
  const F<4> t3 = qd_mul_body(a.re, b.im);
  const F<4> t4 = qd_mul_body(a.im, b.re);
  return {qd_add_body(t1, fneg(t2)), qd_add_body(t3, t4)};
}
PN_QD_CALL C<4> c4_add_call(C<4> a, C<4> b) { return {qd_add_body(a.re, b.re), qd_add_body(a.im, b.im)}; }
template <> PN_DI C<4> cmul<4>(const C<4> &a, const C<4> &b) { return c4_mul_call(a, b); }
template <> PN_DI C<4> cadd<4>(const C<4> &a, const C<4> &b) { return c4_add_call(a, b); }
template <> PN_DI C<4> csub<4>(const C<4> &a, const C<4> &b) { return c4_add_call(a, {fneg(b.re), fneg(b.im)}); }
#endif

// ---------------------------------------------------------------------------
// generic element interface: E = F<NC> (real level) or C<NC> (complex level)

template <class E> struct Traits;
template <int NC> struct Traits<F<NC>> {
  static constexpr int nc = NC, es = NC;
  static constexpr bool cplx = false;
  using R = F<NC>;
};
template <int NC> struct Traits<C<NC>> {
  static constexpr int nc = NC, es = 2 * NC;
  static constexpr bool cplx = true;
  using R = F<NC>;
};

template <int NC> PN_DI F<NC> eadd(const F<NC> &a, const F<NC> &b) { return fadd(a, b); }
template <int NC> PN_DI F<NC> esub(const F<NC> &a, const F<NC> &b) { return fsub(a, b); }
template <int NC> PN_DI F<NC> emul(const F<NC> &a, const F<NC> &b) { return fmul(a, b); }
template <int NC> PN_DI F<NC> econj(const F<NC> &a) { return a; }
template <int NC> PN_DI C<NC> eadd(const C<NC> &a, const C<NC> &b) { return cadd(a, b); }
template <int NC> PN_DI C<NC> esub(const C<NC> &a, const C<NC> &b) { return csub(a, b); }
template <int NC> PN_DI C<NC> emul(const C<NC> &a, const C<NC> &b) { return cmul(a, b); }
template <int NC> PN_DI C<NC> econj(const C<NC> &a) { return cconj(a); }

template <class E> PN_DI E ezero() { E r; double *p = reinterpret_cast<double *>(&r); _Pragma("unroll") for (int i = 0; i < Traits<E>::es; ++i) p[i] = 0.0; return r; }
template <class E> PN_DI E eneg(const E &a) { E r; const double *s = reinterpret_cast<const double *>(&a); double *p = reinterpret_cast<double *>(&r); _Pragma("unroll") for (int i = 0; i < Traits<E>::es; ++i) p[i] = dneg(s[i]); return r; }
// one_like (xprec.py:376-383)
template <class E> PN_DI E eone() { E r = ezero<E>(); reinterpret_cast<double *>(&r)[0] = 1.0; return r; }

// scalar * int: the int is promoted to (float(d), 0, ...) and each part is
// multiplied in the field (xprec.py:36-49, 302-304)
template <int NC> PN_DI F<NC> emul_int(const F<NC> &a, int d) { return fmul(a, fconst<NC>((double)d)); }
template <int NC> PN_DI C<NC> emul_int(const C<NC> &a, int d) {
  const F<NC> dv = fconst<NC>((double)d);
  return {fmul(a.re, dv), fmul(a.im, dv)};
}

// squared modulus (varith.py:149-153), a real element
template <int NC> PN_DI F<NC> eabs2(const F<NC> &a) { return fmul(a, a); }
template <int NC> PN_DI F<NC> eabs2(const C<NC> &a) { return fadd(fmul(a.re, a.re), fmul(a.im, a.im)); }

// divide by a real element (varith.py:138-142); dd/qd take a hoisted recip
template <int NC> PN_DI F<NC> ediv_real(const F<NC> &a, const F<NC> &r) { return fdiv(a, r); }
template <int NC> PN_DI C<NC> ediv_real(const C<NC> &a, const F<NC> &r) { return {fdiv(a.re, r), fdiv(a.im, r)}; }

// "division prepared from the divisor": for NC>1 the reciprocal of the real
// divisor is computed once and applied with mul; for NC==1 the IEEE quotient
// is kept (varith.py:43-46).
template <int NC> struct RDiv {
  F<NC> v;  // recip (NC>1) or the divisor itself (NC==1)
};
PN_DI RDiv<1> rdiv_prepare(const F<1> &d) { return {d}; }
PN_DI RDiv<2> rdiv_prepare(const F<2> &d) { return {frecip(d)}; }
PN_DI RDiv<4> rdiv_prepare(const F<4> &d) { return {frecip(d)}; }
PN_DI F<1> rdiv_apply(const F<1> &a, const RDiv<1> &p) { return fdiv(a, p.v); }
PN_DI F<2> rdiv_apply(const F<2> &a, const RDiv<2> &p) { return fmul(a, p.v); }
PN_DI F<4> rdiv_apply(const F<4> &a, const RDiv<4> &p) { return fmul(a, p.v); }
template <int NC> PN_DI F<NC> ediv_prepared(const F<NC> &a, const RDiv<NC> &p) { return rdiv_apply(a, p); }
template <int NC> PN_DI C<NC> ediv_prepared(const C<NC> &a, const RDiv<NC> &p) { return {rdiv_apply(a.re, p), rdiv_apply(a.im, p)}; }

// full element division (varith.py:130-136): real -> field division;
// complex -> (a * conj b) / (br^2 + bi^2), both parts divided by den.
template <int NC> PN_DI F<NC> ediv(const F<NC> &a, const F<NC> &b) { return fdiv(a, b); }
template <int NC> PN_DI C<NC> ediv(const C<NC> &a, const C<NC> &b) {
  F<NC> den = fadd(fmul(b.re, b.re), fmul(b.im, b.im));
  C<NC> num = cmul(a, cconj(b));
  RDiv<NC> p = rdiv_prepare(den);
  return {rdiv_apply(num.re, p), rdiv_apply(num.im, p)};
}
// the denominator of ediv, for hoisting the reciprocal (back substitution)
template <int NC> PN_DI F<NC> ediv_den(const F<NC> &b) { return b; }
template <int NC> PN_DI F<NC> ediv_den(const C<NC> &b) { return fadd(fmul(b.re, b.re), fmul(b.im, b.im)); }
template <int NC> PN_DI F<NC> ediv_with(const F<NC> &a, const F<NC> &, const RDiv<NC> &p) { return rdiv_apply(a, p); }
template <int NC> PN_DI C<NC> ediv_with(const C<NC> &a, const C<NC> &b, const RDiv<NC> &p) {
  C<NC> num = cmul(a, cconj(b));
  return {rdiv_apply(num.re, p), rdiv_apply(num.im, p)};
}

// embed a real element as a level element (real_embed, varith.py:158-162)
template <int NC> PN_DI F<NC> eembed(const F<NC> &r, F<NC> *) { return r; }
template <int NC> PN_DI C<NC> eembed(const F<NC> &r, C<NC> *) { return {r, fzero<NC>()}; }

// the real part's leading component (hi of re)
template <int NC> PN_DI double ehi(const F<NC> &a) { return a.c[0]; }
template <int NC> PN_DI double ehi(const C<NC> &a) { return a.re.c[0]; }

// ---------------------------------------------------------------------------
// memory access: elements are stored as ES contiguous doubles (AoS)

template <class E> PN_DI E eload(const double *__restrict__ p) {
  E r;
  double *d = reinterpret_cast<double *>(&r);
  constexpr int es = Traits<E>::es;
  if constexpr (es % 2 == 0) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int i = 0; i < es / 2; ++i) { double2 v = q[i]; d[2 * i] = v.x; d[2 * i + 1] = v.y; }
  } else {
#pragma unroll
    for (int i = 0; i < es; ++i) d[i] = p[i];
  }
  return r;
}
template <class E> PN_DI E eload_ldg(const double *__restrict__ p) {
  E r;
  double *d = reinterpret_cast<double *>(&r);
  constexpr int es = Traits<E>::es;
  if constexpr (es % 2 == 0) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int i = 0; i < es / 2; ++i) { double2 v = __ldg(q + i); d[2 * i] = v.x; d[2 * i + 1] = v.y; }
  } else {
#pragma unroll
    for (int i = 0; i < es; ++i) d[i] = __ldg(p + i);
  }
  return r;
}
template <class E> PN_DI void estore(double *__restrict__ p, const E &v) {
  const double *d = reinterpret_cast<const double *>(&v);
  constexpr int es = Traits<E>::es;
  if constexpr (es % 2 == 0) {
    double2 *q = reinterpret_cast<double2 *>(p);
#pragma unroll
    for (int i = 0; i < es / 2; ++i) q[i] = make_double2(d[2 * i], d[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < es; ++i) p[i] = d[i];
  }
}

// warp shuffle of a whole element
template <class E> PN_DI E eshfl_xor(const E &v, int mask) {
  E r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *d = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < Traits<E>::es; ++i) d[i] = __shfl_xor_sync(0xffffffffu, s[i], mask);
  return r;
}
template <class E> PN_DI E eshfl_idx(const E &v, int src) {
  E r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *d = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < Traits<E>::es; ++i) d[i] = __shfl_sync(0xffffffffu, s[i], src);
  return r;
}
template <class E> PN_DI E eshfl_down(const E &v, int delta) {
  E r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *d = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < Traits<E>::es; ++i) d[i] = __shfl_down_sync(0xffffffffu, s[i], delta);
  return r;
}

}  // namespace pn
