// textfmt.cpp -- native ingestion of the system text format (polyrep.py:
// 140-304) straight into CSR arrays and coefficient planes, for systems of
// 10^6 monomials where building Monomial objects in Python takes minutes.
//
// Grammar (parse_system / _parse_poly / _parse_term): line 1 "m n"; then m
// polynomials, each a '+'/'-'-separated list of terms closed by ';'; a term
// is a '*'-product of at most one coefficient ("2.5", ".5", "(re,im)") and
// variable factors "x<i>" / "x<i>^<d>" (repeated variables add exponents,
// the coefficient defaults to one, a leading '-' negates every component).
//
// Coefficients are converted exactly as parse_decimal (xprec.py:432-446):
// the literal is the rational D * 10^E, components are split off by
// repeated exact subtraction of the correctly rounded (round-half-even)
// double, and quad doubles finish with renorm5(c0, c1, c2, c3, 0)
// (_eft.py:134-179).  The rational arithmetic runs on a small fixed-point
// bignum: Q = floor(|D| 2^S / 10^-E) with a sticky bit, S chosen so that
// every component's last bit lies above 2^-S (so each subtraction is exact
// and guard + sticky decide every rounding).
//
// Anything outside the common grammar -- every error, non-ASCII input
// (the reference also accepts the sign U+2212 and Unicode digits), decimal
// forms Python's Decimal accepts but this scanner does not, values that
// overflow -- returns PN_E_ARG and the Python layer re-parses the text with
// its own parser, which raises the reference's exact SystemParseError.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/polynewt_b200.h"

namespace {

// ---- minimal unsigned bignum (little-endian 32-bit limbs) ------------------
struct Big {
  std::vector<uint32_t> d;
  void trim() {
    while (!d.empty() && d.back() == 0) d.pop_back();
  }
  bool zero() const { return d.empty(); }
  int bits() const {
    if (d.empty()) return 0;
    return 32 * ((int)d.size() - 1) + (32 - __builtin_clz(d.back()));
  }
  void mul_small(uint32_t m, uint32_t add = 0) {
    uint64_t carry = add;
    for (auto &x : d) {
      const uint64_t t = (uint64_t)x * m + carry;
      x = (uint32_t)t;
      carry = t >> 32;
    }
    if (carry) d.push_back((uint32_t)carry);
  }
  void shl(int s) {
    if (d.empty() || s == 0) return;
    const int w = s / 32, b = s % 32;
    if (b) {
      uint32_t carry = 0;
      for (auto &x : d) {
        const uint32_t nx = (x << b) | carry;
        carry = x >> (32 - b);
        x = nx;
      }
      if (carry) d.push_back(carry);
    }
    d.insert(d.begin(), w, 0u);
  }
  bool bit(int i) const {
    const int w = i / 32;
    return w < (int)d.size() && ((d[w] >> (i % 32)) & 1);
  }
  bool any_below(int i) const {  // any set bit at positions < i
    for (int w = 0; w < (int)d.size() && 32 * w < i; ++w) {
      const int hi = std::min(32, i - 32 * w);
      const uint32_t mask = hi == 32 ? 0xffffffffu : ((1u << hi) - 1);
      if (d[w] & mask) return true;
    }
    return false;
  }
};

int cmp(const Big &a, const Big &b) {
  if (a.d.size() != b.d.size()) return a.d.size() < b.d.size() ? -1 : 1;
  for (int i = (int)a.d.size() - 1; i >= 0; --i)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}
void sub_in(Big &a, const Big &b) {  // a -= b, a >= b
  int64_t borrow = 0;
  for (size_t i = 0; i < a.d.size(); ++i) {
    int64_t t = (int64_t)a.d[i] - borrow - (i < b.d.size() ? (int64_t)b.d[i] : 0);
    borrow = t < 0;
    a.d[i] = (uint32_t)(t + (borrow << 32));
  }
  a.trim();
}
void add_in(Big &a, const Big &b) {
  if (a.d.size() < b.d.size()) a.d.resize(b.d.size(), 0);
  uint64_t carry = 0;
  for (size_t i = 0; i < a.d.size(); ++i) {
    const uint64_t t = (uint64_t)a.d[i] + (i < b.d.size() ? b.d[i] : 0) + carry;
    a.d[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) a.d.push_back((uint32_t)carry);
}
// q = floor(a / b), r = a mod b: Knuth's algorithm D on 32-bit limbs
// (Hacker's Delight, divmnu), O(len(a) * len(b))
void divmod(const Big &a, const Big &b, Big &q, Big &r) {
  q.d.clear();
  if (cmp(a, b) < 0) {
    r = a;
    return;
  }
  const int n = (int)b.d.size(), m = (int)a.d.size();
  if (n == 1) {  // short division
    const uint64_t v = b.d[0];
    q.d.assign(m, 0);
    uint64_t rem = 0;
    for (int j = m - 1; j >= 0; --j) {
      const uint64_t cur = (rem << 32) | a.d[j];
      q.d[j] = (uint32_t)(cur / v);
      rem = cur % v;
    }
    q.trim();
    r.d = {(uint32_t)rem};
    r.trim();
    return;
  }
  const int sft = __builtin_clz(b.d[n - 1]);  // normalise the divisor's top limb
  std::vector<uint32_t> vn(n), un(m + 1);
  for (int i = n - 1; i > 0; --i) vn[i] = (b.d[i] << sft) | (sft ? (uint32_t)((uint64_t)b.d[i - 1] >> (32 - sft)) : 0);
  vn[0] = b.d[0] << sft;
  un[m] = sft ? (uint32_t)((uint64_t)a.d[m - 1] >> (32 - sft)) : 0;
  for (int i = m - 1; i > 0; --i) un[i] = (a.d[i] << sft) | (sft ? (uint32_t)((uint64_t)a.d[i - 1] >> (32 - sft)) : 0);
  un[0] = a.d[0] << sft;
  q.d.assign(m - n + 1, 0);
  const uint64_t base = 1ull << 32;
  for (int j = m - n; j >= 0; --j) {
    const uint64_t num = ((uint64_t)un[j + n] << 32) | un[j + n - 1];
    uint64_t qhat = num / vn[n - 1], rhat = num % vn[n - 1];
    while (qhat >= base || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
      --qhat;
      rhat += vn[n - 1];
      if (rhat >= base) break;
    }
    int64_t borrow = 0;
    uint64_t carry = 0;
    for (int i = 0; i < n; ++i) {
      const uint64_t p = qhat * vn[i] + carry;
      carry = p >> 32;
      const int64_t t = (int64_t)un[i + j] - borrow - (int64_t)(p & 0xffffffffu);
      un[i + j] = (uint32_t)t;
      borrow = t < 0 ? 1 : 0;
    }
    const int64_t t = (int64_t)un[j + n] - borrow - (int64_t)carry;
    un[j + n] = (uint32_t)t;
    if (t < 0) {  // qhat was one too large: add the divisor back
      --qhat;
      uint64_t c = 0;
      for (int i = 0; i < n; ++i) {
        const uint64_t s2 = (uint64_t)un[i + j] + vn[i] + c;
        un[i + j] = (uint32_t)s2;
        c = s2 >> 32;
      }
      un[j + n] += (uint32_t)c;
    }
    q.d[j] = (uint32_t)qhat;
  }
  q.trim();
  r.d.assign(n, 0);
  for (int i = 0; i < n; ++i) r.d[i] = (un[i] >> sft) | (sft ? (uint32_t)((uint64_t)un[i + 1] << (32 - sft)) : 0);
  r.trim();
}

// signed fixed-point value v = sign * Q * 2^-S (+ sticky: a positive
// remainder below Q's last bit, same sign)
struct Fixed {
  Big q;
  bool neg = false, sticky = false;
  int S = 0;
};

// round-half-even of v to a double (subnormals included); false on overflow
bool round_double(const Fixed &v, double &out) {
  if (v.q.zero()) {
    out = 0.0;  // float(Fraction(0)) is +0.0 whatever the sign of the residual before it
    return !v.sticky;  // sticky alone cannot occur: S keeps every nonzero residual visible
  }
  const int nb = v.q.bits();
  const int e0 = nb - 1 - v.S;  // value in [2^e0, 2^(e0+1))
  if (e0 > 1023) return false;
  // keep p significant bits: 53 for normals, fewer below 2^-1022
  int p = 53;
  if (e0 < -1022) p = 53 - (-1022 - e0);
  if (p <= 0) p = 0;
  const int drop = nb - p;  // bits of Q below the kept ones
  uint64_t mant = 0;
  for (int i = nb - 1; i >= drop && i >= 0; --i) mant = (mant << 1) | (uint64_t)v.q.bit(i);
  bool up = false;
  if (drop > 0) {
    const bool guard = v.q.bit(drop - 1);
    const bool rest = v.q.any_below(drop - 1) || v.sticky;
    up = guard && (rest || (mant & 1));
  } else if (v.sticky) {
    return false;  // cannot happen with the chosen S
  }
  if (up) ++mant;
  double r = std::ldexp((double)mant, drop - v.S);
  if (std::isinf(r)) return false;
  out = v.neg ? -r : r;
  return true;
}

// v -= c exactly (c's last bit must lie above 2^-S)
bool subtract(Fixed &v, double c) {
  if (c == 0.0) return true;
  int ex;
  const double fr = std::frexp(std::fabs(c), &ex);  // |c| = fr * 2^ex, fr in [0.5, 1)
  const uint64_t m = (uint64_t)std::ldexp(fr, 53);  // |c| = m * 2^(ex-53)
  const int sh = ex - 53 + v.S;                    // |c| * 2^S = m * 2^sh
  if (sh < 0) return false;
  Big C;
  C.d = {(uint32_t)m, (uint32_t)(m >> 32)};
  C.trim();
  C.shl(sh);
  const bool cneg = c < 0;
  if (cneg == v.neg) {  // same sign: |v| - |c|
    if (cmp(v.q, C) >= 0) {
      sub_in(v.q, C);
    } else {  // |c| > |v|: the residual flips sign.  With a sticky part
      // e in (0, 1) ulp: |c| - (Q + e) = (|c| - Q - 1) + (1 - e), so the
      // new magnitude is |c| - Q - 1 with the sticky bit still set
      Big t = C;
      sub_in(t, v.q);
      if (v.sticky) {
        Big one;
        one.d = {1};
        sub_in(t, one);
      }
      v.q = t;
      v.neg = !v.neg;
    }
  } else {
    add_in(v.q, C);
  }
  return true;
}

// --- the reference's renorm5 (_eft.py:134-179), host binary64 -----------------
inline void quick_two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  e = b - (s - a);
}
inline void renorm5(double c0, double c1, double c2, double c3, double c4, double out[4]) {
  double s, t0, t1, t2, t3;
  quick_two_sum(c3, c4, s, t3);
  quick_two_sum(c2, s, s, t2);
  quick_two_sum(c1, s, s, t1);
  quick_two_sum(c0, s, c0, t0);
  // second pass: accumulate the non-zero tails in order
  const double tv[4] = {t0, t1, t2, t3};
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  double cur = c0;
  int k = 0;
  for (int i = 0; i < 4; ++i) {
    double e;
    quick_two_sum(cur, tv[i], s, e);
    if (e != 0.0 && k < 3) {
      o[k++] = s;
      cur = e;
    } else {
      cur = s;
    }
  }
  o[k] = cur;
  for (int i = 0; i < 4; ++i) out[i] = o[i];
}

// parse_decimal (xprec.py:432-446) for the literal text[a, b): components
// into out (nc of them); false if the literal is outside the grammar here
bool parse_decimal(const char *t, size_t a, size_t b, int nc, double *out) {
  while (a < b && (t[a] == ' ' || t[a] == '\t')) ++a;  // level.parse strips
  while (b > a && (t[b - 1] == ' ' || t[b - 1] == '\t')) --b;
  if (a >= b) return false;
  bool neg = false;
  if (t[a] == '+' || t[a] == '-') {  // only inside "(re,im)"
    neg = t[a] == '-';
    ++a;
  }
  Big D;
  int ndig = 0, frac = 0;
  bool seen_dot = false, last_digit = false;
  size_t i = a;
  for (; i < b; ++i) {
    const char ch = t[i];
    if (ch >= '0' && ch <= '9') {
      D.mul_small(10, (uint32_t)(ch - '0'));
      ++ndig;
      if (seen_dot) ++frac;
      last_digit = true;
    } else if (ch == '_') {  // Decimal accepts single underscores between digits
      if (!last_digit || i + 1 >= b || !(t[i + 1] >= '0' && t[i + 1] <= '9')) return false;
      last_digit = false;
    } else if (ch == '.') {
      if (seen_dot) return false;
      seen_dot = true;
      last_digit = false;
    } else {
      break;
    }
  }
  if (ndig == 0) return false;
  long exp10 = 0;
  if (i < b) {
    if (t[i] != 'e' && t[i] != 'E') return false;
    ++i;
    bool eneg = false;
    if (i < b && (t[i] == '+' || t[i] == '-')) eneg = t[i++] == '-';
    if (i >= b) return false;
    bool lastd = false;
    for (; i < b; ++i) {
      if (t[i] >= '0' && t[i] <= '9') {
        exp10 = exp10 * 10 + (t[i] - '0');
        if (exp10 > 100000) return false;
        lastd = true;
      } else if (t[i] == '_' && lastd && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
        lastd = false;
      } else {
        return false;
      }
    }
    if (eneg) exp10 = -exp10;
  }
  exp10 -= frac;
  D.trim();
  if (D.zero()) {  // an exact zero: all components +-0 (Fraction(0) -> 0.0)
    for (int c = 0; c < nc; ++c) out[c] = 0.0;
    (void)neg;  // Fraction(Decimal("-0")) == 0: float(0) is +0.0
    return true;
  }
  if (exp10 > 400 || exp10 < -800) return false;
  // value = D * 10^exp10 as Fixed with S bits below the point
  Fixed v;
  v.neg = neg;
  const int k = exp10 < 0 ? (int)-exp10 : 0;
  const int dbits = D.bits();
  // S: the last bit of every component (ulps down to 2^(e0 - 53 nc), each
  // nonzero residual >= 2^-(S0 + log2 10^k) apart) stays above 2^-S
  const int lg10k = (int)std::ceil(k * 3.3219280948873626) + 1;
  const int e0_est = dbits - lg10k;  // ~ log2 of the value
  int S = 64 * nc + nc * (lg10k + 8) + (e0_est < 0 ? -e0_est : 0) + 64;
  if (exp10 >= 0) {
    Big P = D;
    for (long j = 0; j < exp10; ++j) P.mul_small(10);
    P.shl(S);
    v.q = P;
  } else {
    Big num = D, den;
    den.d = {1};
    for (int j = 0; j < k; ++j) den.mul_small(10);
    num.shl(S);
    Big r;
    divmod(num, den, v.q, r);
    v.sticky = !r.zero();
  }
  v.S = S;
  double c[4] = {0, 0, 0, 0};
  for (int j = 0; j < nc; ++j) {
    if (!round_double(v, c[j])) return false;
    if (j + 1 < nc && !subtract(v, c[j])) return false;
  }
  if (nc == 4) {
    double r[4];
    renorm5(c[0], c[1], c[2], c[3], 0.0, r);
    for (int j = 0; j < 4; ++j) out[j] = r[j];
  } else {
    for (int j = 0; j < nc; ++j) out[j] = c[j];
  }
  return true;
}

bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\f' || ch == '\v'; }

}  // namespace

struct pn_text_system {
  int nc = 1, cplx = 0, m = 0, n = 0;
  std::vector<int32_t> poly_ptr{0}, mon_ptr{0}, var_idx, exps;
  std::vector<double> comps;  // es per monomial (generation order)
};

extern "C" int pn_parse_system(const char *text, int64_t len, int nc, int cplx, pn_text_system **out) {
  if (!out || !text || len < 0 || !(nc == 1 || nc == 2 || nc == 4)) return PN_E_ARG;
  *out = nullptr;
  for (int64_t i = 0; i < len; ++i)
    if ((unsigned char)text[i] >= 0x80) return PN_E_ARG;  // Unicode signs / digits / spaces: Python path
  const int es = nc * (cplx ? 2 : 1);
  auto S = new pn_text_system;
  S->nc = nc;
  S->cplx = cplx;
  auto fail = [&]() {
    delete S;
    return PN_E_ARG;
  };
  const char *t = text;
  const size_t L = (size_t)len;
  // header: the first line split on whitespace, exactly two integers
  size_t nl = 0;
  while (nl < L && t[nl] != '\n') ++nl;
  {
    std::vector<std::string> tok;
    size_t i = 0;
    while (i < nl) {
      while (i < nl && is_ws(t[i])) ++i;
      size_t j = i;
      while (j < nl && !is_ws(t[j])) ++j;
      if (j > i) tok.emplace_back(t + i, j - i);
      i = j;
    }
    if (tok.size() != 2) return fail();
    for (auto &s : tok)
      for (char ch : s)
        if (ch < '0' || ch > '9') return fail();  // int() also takes signs/underscores: Python path
    if (tok[0].size() > 9 || tok[1].size() > 9) return fail();
    S->m = std::stoi(tok[0]);
    S->n = std::stoi(tok[1]);
  }
  size_t p = nl < L ? nl + 1 : L;
  auto skip = [&]() {
    while (p < L && is_ws(t[p])) ++p;
  };
  std::vector<int64_t> acc;  // exponent per variable of the current term (sparse reset)
  acc.assign((size_t)S->n, 0);
  std::vector<int32_t> touched;
  std::vector<double> coeff(es);
  for (int i = 0; i < S->m; ++i) {
    bool negate = false, pending = false, first = true, any_term = false;
    for (;;) {
      skip();
      if (p >= L) return fail();
      const char ch = t[p];
      if (ch == ';') {
        if (pending || first) return fail();
        ++p;
        break;
      }
      if (ch == '+' || ch == '-') {
        if (pending) return fail();
        negate = ch == '-';
        pending = true;
        first = false;
        ++p;
        continue;
      }
      if (any_term && !pending) return fail();
      // ---- a term: factors joined by '*'
      bool have_coeff = false;
      touched.clear();
      for (;;) {
        skip();
        if (p >= L) return fail();
        if (t[p] == 'x') {
          size_t q = p + 1;
          int64_t idx = 0;
          if (q >= L || t[q] < '0' || t[q] > '9') return fail();
          while (q < L && t[q] >= '0' && t[q] <= '9') {
            idx = idx * 10 + (t[q] - '0');
            if (idx > (1ll << 31)) return fail();
            ++q;
          }
          int64_t d = 1;
          if (q < L && t[q] == '^') {
            ++q;
            if (q >= L || t[q] < '0' || t[q] > '9') return fail();
            d = 0;
            while (q < L && t[q] >= '0' && t[q] <= '9') {
              d = d * 10 + (t[q] - '0');
              if (d > (1ll << 30)) return fail();
              ++q;
            }
            if (d < 1) return fail();
          }
          if (idx >= S->n) return fail();
          if (acc[idx] == 0) touched.push_back((int32_t)idx);
          acc[idx] += d;
          if (acc[idx] > (1ll << 31) - 1) return fail();
          p = q;
        } else if (t[p] == '(') {
          if (!cplx || have_coeff) return fail();
          size_t q = p + 1;
          while (q < L && t[q] != ')' && t[q] != '(') ++q;
          if (q >= L || t[q] != ')') return fail();
          size_t comma = p + 1, ncomma = 0;
          for (size_t r = p + 1; r < q; ++r)
            if (t[r] == ',') {
              comma = r;
              ++ncomma;
            }
          if (ncomma != 1) return fail();
          if (!parse_decimal(t, p + 1, comma, nc, coeff.data())) return fail();
          if (!parse_decimal(t, comma + 1, q, nc, coeff.data() + nc)) return fail();
          have_coeff = true;
          p = q + 1;
        } else if ((t[p] >= '0' && t[p] <= '9') || t[p] == '.') {
          if (have_coeff) return fail();
          size_t q = p + (t[p] == '.' ? 1 : 0);
          if (t[p] == '.' && (q >= L || t[q] < '0' || t[q] > '9')) return fail();
          while (q < L && ((t[q] >= '0' && t[q] <= '9') || t[q] == '_' || t[q] == '.' || t[q] == 'e' || t[q] == 'E' ||
                           t[q] == '+' || t[q] == '-'))
            ++q;
          if (!parse_decimal(t, p, q, nc, coeff.data())) return fail();
          for (int c = nc; c < es; ++c) coeff[c] = 0.0;  // level.parse: Complex(x, real_zero())
          have_coeff = true;
          p = q;
        } else {
          return fail();
        }
        skip();
        if (p < L && t[p] == '*') {
          ++p;
          continue;
        }
        break;
      }
      if (p < L && t[p] == '^') return fail();
      if (!have_coeff) {  // level.one()
        for (int c = 0; c < es; ++c) coeff[c] = 0.0;
        coeff[0] = 1.0;
      }
      if (negate)
        for (int c = 0; c < es; ++c) coeff[c] = -coeff[c];
      bool nonzero = false;
      for (int c = 0; c < es; ++c) nonzero |= coeff[c] != 0.0;
      if (!nonzero) return fail();  // Monomial refuses a zero coefficient
      std::sort(touched.begin(), touched.end());
      for (int32_t v : touched) {
        S->var_idx.push_back(v);
        S->exps.push_back((int32_t)acc[v]);
        acc[v] = 0;
      }
      S->mon_ptr.push_back((int32_t)S->var_idx.size());
      S->comps.insert(S->comps.end(), coeff.begin(), coeff.end());
      negate = false;
      pending = false;
      first = false;
      any_term = true;
    }
    S->poly_ptr.push_back((int32_t)(S->mon_ptr.size() - 1));
    if (S->var_idx.size() >= (1ull << 31)) return fail();
  }
  skip();
  if (p < L) return fail();
  *out = S;
  return PN_OK;
}

extern "C" int pn_text_system_sizes(const pn_text_system *s, int32_t *m, int32_t *n, int64_t *M, int64_t *nnz) {
  if (!s || !m || !n || !M || !nnz) return PN_E_ARG;
  *m = s->m;
  *n = s->n;
  *M = (int64_t)s->mon_ptr.size() - 1;
  *nnz = (int64_t)s->var_idx.size();
  return PN_OK;
}

// CSR in generation order and the coefficients as planes (es, M)
extern "C" int pn_text_system_export(const pn_text_system *s, int32_t *poly_ptr, int32_t *mon_ptr, int32_t *var_idx,
                                     int32_t *exps, double *coeff_planes) {
  if (!s || !poly_ptr || !mon_ptr || (!s->var_idx.empty() && (!var_idx || !exps)) || !coeff_planes) return PN_E_ARG;
  const int es = s->nc * (s->cplx ? 2 : 1);
  const size_t M = s->mon_ptr.size() - 1;
  std::copy(s->poly_ptr.begin(), s->poly_ptr.end(), poly_ptr);
  std::copy(s->mon_ptr.begin(), s->mon_ptr.end(), mon_ptr);
  std::copy(s->var_idx.begin(), s->var_idx.end(), var_idx);
  std::copy(s->exps.begin(), s->exps.end(), exps);
  for (size_t c = 0; c < M; ++c)
    for (int e = 0; e < es; ++e) coeff_planes[(size_t)e * M + c] = s->comps[c * es + e];
  return PN_OK;
}

extern "C" int pn_text_system_free(pn_text_system *s) {
  delete s;
  return PN_OK;
}
