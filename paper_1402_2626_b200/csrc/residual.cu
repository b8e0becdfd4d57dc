// residual.cu -- residual_check (mgs.py:311-357): max componentwise |A - QR|
// of a factorisation, recomputed in the next-higher precision (d -> dd,
// dd -> qd) with the reference's exact operation sequence:
//   acc = 0; for k: acc = acc + promote(Q[:, k]) * promote(R[k, :n]);
//   diff = promote(A) - acc; result = sqrt(max hi(abs2(diff))).
// promote() pads the extra components with +0.0 (varith.py:200-209), so the
// value is bit-identical to the reference.
//
// Quad double: the reference uses 320-bit mpfr (mgs.py:334-357).  Here every
// product of components is split exactly (two_prod) and all terms of
// A - sum_k Q_ik R_kj are accumulated EXACTLY in a 576-bit fixed-point
// integer (LSB 2^-512; terms below it, far under any qd factorisation's
// residual, are truncated), then the exact difference is rounded to a qd
// value, squared and maxed in qd, and square-rooted; float() is math.fsum.
// The reference's 320-bit rounding differs from the exact value by ~2^-100
// relative, so both round to the same binary64 except within ~1e-30 of a
// rounding boundary.
//
// Tiled like a GEMM (16 x 16 outputs per CTA, Q and R tiles staged in shared
// memory), but every output keeps its sequential k order: there is no
// tensor-core shortcut for individually rounded extended-precision sums.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace pn {

template <class E> struct NextLevel;
template <> struct NextLevel<F<1>> { using T = F<2>; };
template <> struct NextLevel<F<2>> { using T = F<4>; };
template <> struct NextLevel<C<1>> { using T = C<2>; };
template <> struct NextLevel<C<2>> { using T = C<4>; };

template <int NC> __device__ __forceinline__ F<2 * NC> promote_f(const F<NC> &v) {
  F<2 * NC> r;
#pragma unroll
  for (int i = 0; i < 2 * NC; ++i) r.c[i] = i < NC ? v.c[i] : 0.0;
  return r;
}
template <int NC> __device__ __forceinline__ F<2 * NC> promote(const F<NC> &v) { return promote_f(v); }
template <int NC> __device__ __forceinline__ C<2 * NC> promote(const C<NC> &v) {
  return {promote_f(v.re), promote_f(v.im)};
}

// element (r, c) of a (rows, cols) component-plane array
template <class E>
__device__ __forceinline__ E plane_get(const double *__restrict__ a, long long rows, long long cols, long long r,
                                       long long c) {
  return eload_planes<E>(a, rows * cols, r * cols + c);
}

template <class E, int T>
__global__ void __launch_bounds__(T *T) k_residual(int m, int n, const double *__restrict__ A,
                                                    const double *__restrict__ Q, const double *__restrict__ R,
                                                    unsigned long long *__restrict__ maxbits) {
  using H = typename NextLevel<E>::T;
  __shared__ E sQ[T][T + 1];
  __shared__ E sR[T][T + 1];
  __shared__ double smax[T * T / 32];
  const int tx = threadIdx.x % T, ty = threadIdx.x / T;
  const int i = blockIdx.y * T + ty, j = blockIdx.x * T + tx;
  H acc = ezero<H>();
  for (int k0 = 0; k0 < n; k0 += T) {
    sQ[ty][tx] = (i < m && k0 + tx < n) ? plane_get<E>(Q, m, n, i, k0 + tx) : ezero<E>();
    sR[ty][tx] = (k0 + ty < n && j < n) ? plane_get<E>(R, n, n, k0 + ty, j) : ezero<E>();
    __syncthreads();
    const int kk_end = min(T, n - k0);
    for (int kk = 0; kk < kk_end; ++kk) acc = eadd(acc, emul(promote(sQ[ty][kk]), promote(sR[kk][tx])));
    __syncthreads();
  }
  double mag = 0.0;
  if (i < m && j < n) mag = eabs2(esub(promote(plane_get<E>(A, m, n, i, j)), acc)).c[0];
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) mag = fmax(mag, __shfl_xor_sync(0xffffffffu, mag, s));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = mag;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = smax[0];
    for (int w = 1; w < T * T / 32; ++w) b = fmax(b, smax[w]);
    // magnitudes are >= 0: their IEEE bit patterns order like unsigned ints
    atomicMax(maxbits, (unsigned long long)__double_as_longlong(b));
  }
}

// ---- exact fixed-point accumulation for quad double -----------------------
constexpr int XL = 9;        // 64-bit limbs
constexpr int XOFF = 512;    // bit position of 2^0 (LSB = 2^-512)

struct Fix {
  unsigned long long w[XL];
};
__device__ __forceinline__ void fix_zero(Fix &a) {
#pragma unroll
  for (int l = 0; l < XL; ++l) a.w[l] = 0ull;
}
// a += |x| (exactly, bits below 2^-512 truncated)
__device__ __forceinline__ void fix_add_abs(Fix &a, double x) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int ex = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & ((1ull << 52) - 1);
  if (ex == 0 && mant == 0) return;
  int p;  // bit position of the mantissa's LSB
  if (ex == 0) p = 1 - 1075 + XOFF;
  else {
    mant |= 1ull << 52;
    p = ex - 1075 + XOFF;
  }
  if (p < 0) {
    if (p <= -64) return;
    mant >>= -p;
    p = 0;
  }
  const int L = p >> 6, sh = p & 63;
  const unsigned long long w0 = mant << sh, w1 = sh ? (mant >> (64 - sh)) : 0ull;
  unsigned long long carry = 0;
#pragma unroll
  for (int l = 0; l < XL; ++l) {
    const unsigned long long add = (l == L) ? w0 : (l == L + 1) ? w1 : 0ull;
    const unsigned long long s1 = a.w[l] + add;
    const unsigned long long c1 = s1 < add;
    const unsigned long long s2 = s1 + carry;
    const unsigned long long c2 = s2 < carry;
    a.w[l] = s2;
    carry = c1 | c2;
  }
}
// signed term: positive into P, negative into N
__device__ __forceinline__ void fix_term(Fix &P, Fix &N, double x, bool neg) {
  const bool n = (x < 0.0) != neg;
  if (n) fix_add_abs(N, x);
  else fix_add_abs(P, x);
}
// P += sign * (a * b) exactly: all 16 component products split by two_prod
__device__ __forceinline__ void fix_prod(Fix &P, Fix &N, const F<4> &a, const F<4> &b, bool neg) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double p, e;
      two_prod(a.c[i], b.c[j], p, e);
      fix_term(P, N, p, neg);
      fix_term(P, N, e, neg);
    }
}
// P - N rounded to a quad double (magnitude from the top 256 bits)
__device__ __forceinline__ F<4> fix_to_qd(const Fix &P, const Fix &N) {
  Fix d;
  unsigned long long borrow = 0;
#pragma unroll
  for (int l = 0; l < XL; ++l) {
    const unsigned long long s1 = P.w[l] - N.w[l];
    const unsigned long long b1 = P.w[l] < N.w[l];
    const unsigned long long s2 = s1 - borrow;
    const unsigned long long b2 = s1 < borrow;
    d.w[l] = s2;
    borrow = b1 | b2;
  }
  const bool negv = borrow != 0;  // two's complement sign
  if (negv) {
    unsigned long long c = 1;
#pragma unroll
    for (int l = 0; l < XL; ++l) {
      const unsigned long long v = ~d.w[l] + c;
      c = (c && v == 0) ? 1 : 0;
      d.w[l] = v;
    }
  }
  int h = -1;
#pragma unroll
  for (int l = 0; l < XL; ++l)
    if (d.w[l]) h = l;
  F<4> r = fzero<4>();
  if (h < 0) return r;
  for (int l = h; l >= 0 && l >= h - 3; --l) {
    const double hi = ldexp((double)(d.w[l] >> 32), 64 * l + 32 - XOFF);
    const double lo = ldexp((double)(d.w[l] & 0xffffffffull), 64 * l - XOFF);
    r = fadd(r, fconst<4>(hi));
    r = fadd(r, fconst<4>(lo));
  }
  return negv ? fneg(r) : r;
}
__device__ __forceinline__ bool qd_less(const F<4> &a, const F<4> &b) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (a.c[i] != b.c[i]) return a.c[i] < b.c[i];
  return false;
}

template <class E>
__global__ void __launch_bounds__(128) k_residual_qd(int m, int n, const double *__restrict__ A,
                                                     const double *__restrict__ Q, const double *__restrict__ R,
                                                     double *__restrict__ blockmax) {
  constexpr bool CPLX = Traits<E>::cplx;
  const int idx = blockIdx.x * 128 + threadIdx.x;
  F<4> mag = fzero<4>();
  if (idx < m * n) {
    const int i = idx / n, j = idx % n;
    Fix Pr, Nr, Pi, Ni;
    fix_zero(Pr);
    fix_zero(Nr);
    fix_zero(Pi);
    fix_zero(Ni);
    const E a = plane_get<E>(A, m, n, i, j);
    if constexpr (CPLX) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        fix_term(Pr, Nr, a.re.c[c], false);
        fix_term(Pi, Ni, a.im.c[c], false);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) fix_term(Pr, Nr, a.c[c], false);
    }
    for (int k = 0; k < n; ++k) {
      const E q = plane_get<E>(Q, m, n, i, k);
      const E r = plane_get<E>(R, n, n, k, j);
      if constexpr (CPLX) {
        // re: A - (qr rr - qi ri);  im: A - (qr ri + qi rr)
        fix_prod(Pr, Nr, q.re, r.re, true);
        fix_prod(Pr, Nr, q.im, r.im, false);
        fix_prod(Pi, Ni, q.re, r.im, true);
        fix_prod(Pi, Ni, q.im, r.re, true);
      } else {
        fix_prod(Pr, Nr, q, r, true);
      }
    }
    const F<4> dr = fix_to_qd(Pr, Nr);
    mag = fmul(dr, dr);
    if constexpr (CPLX) {
      const F<4> di = fix_to_qd(Pi, Ni);
      mag = fadd(mag, fmul(di, di));
    }
  }
  __shared__ F<4> sm[128];
  sm[threadIdx.x] = mag;
  __syncthreads();
  for (int s = 64; s > 0; s >>= 1) {
    if (threadIdx.x < s && qd_less(sm[threadIdx.x], sm[threadIdx.x + s])) sm[threadIdx.x] = sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int c = 0; c < 4; ++c) blockmax[blockIdx.x * 4 + c] = sm[0].c[c];
}

// max over the block maxima, sqrt, float() (math.fsum of the components)
static __global__ void k_residual_qd_final(int nblocks, const double *__restrict__ blockmax, double *__restrict__ out) {
  F<4> best = fzero<4>();
  for (int b = 0; b < nblocks; ++b) {
    F<4> v;
#pragma unroll
    for (int c = 0; c < 4; ++c) v.c[c] = blockmax[b * 4 + c];
    if (qd_less(best, v)) best = v;
  }
  const F<4> s = fsqrt(best);
  // math.fsum of four non-overlapping components: exact sum rounded once
  double p[4];
  int np = 0;
  for (int t = 0; t < 4; ++t) {
    double x = s.c[t];
    int i2 = 0;
    for (int j = 0; j < np; ++j) {
      double y = p[j];
      if (fabs(x) < fabs(y)) {
        const double tmp = x;
        x = y;
        y = tmp;
      }
      const double hi = __dadd_rn(x, y), yr = __dsub_rn(hi, x), lo = __dsub_rn(y, yr);
      if (lo != 0.0) p[i2++] = lo;
      x = hi;
    }
    np = i2;
    if (x != 0.0) p[np++] = x;
  }
  double hi = 0.0, lo = 0.0;
  if (np > 0) {
    hi = p[--np];
    while (np > 0) {
      const double x = hi, y = p[--np];
      hi = __dadd_rn(x, y);
      const double yr = __dsub_rn(hi, x);
      lo = __dsub_rn(y, yr);
      if (lo != 0.0) break;
    }
    if (np > 0 && ((lo < 0.0 && p[np - 1] < 0.0) || (lo > 0.0 && p[np - 1] > 0.0))) {
      const double y = __dmul_rn(lo, 2.0), x = __dadd_rn(hi, y), yr = __dsub_rn(x, hi);
      if (y == yr) hi = x;
    }
  }
  *out = hi;
}

template <class E>
double residual_impl(int m, int n, const double *A, const double *Q, const double *R, cudaStream_t st) {
  if constexpr (Traits<E>::nc == 4) {
    const long long cnt = (long long)m * n;
    const int nblocks = (int)((cnt + 127) / 128);
    DevBuf bm((size_t)nblocks * 4 * sizeof(double) + 16, st), out(16, st);
    k_residual_qd<E><<<nblocks, 128, 0, st>>>(m, n, A, Q, R, bm.d());
    PN_CHECK_LAUNCH();
    k_residual_qd_final<<<1, 1, 0, st>>>(nblocks, bm.d(), out.d());
    PN_CHECK_LAUNCH();
    count_launch(2);
    double r = 0.0;
    PN_CHECK_CUDA(cudaMemcpyAsync(&r, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    PN_CHECK_CUDA(cudaStreamSynchronize(st));
    return r;
  } else {
    constexpr int T = 16;
    DevBuf mx(sizeof(unsigned long long), st);
    PN_CHECK_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
    const dim3 grid((n + T - 1) / T, (m + T - 1) / T);
    k_residual<E, T><<<grid, T * T, 0, st>>>(m, n, A, Q, R, mx.as<unsigned long long>());
    PN_CHECK_LAUNCH();
    count_launch(1);
    unsigned long long bits = 0;
    PN_CHECK_CUDA(cudaMemcpyAsync(&bits, mx.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
    PN_CHECK_CUDA(cudaStreamSynchronize(st));
    double worst;
    memcpy(&worst, &bits, sizeof(worst));
    return std::sqrt(worst);  // float(np.sqrt(np.max(mags)))
  }
}

#ifdef PN_NC
template double residual_impl<PnLevel>(int, int, const double *, const double *, const double *, cudaStream_t);
#endif

}  // namespace pn
