// batch.cu -- config C5: the least-squares half of many independent Newton
// steps at once, one CTA per start.
//
// k_solve_batch factors [J | -f] of one start with modified Gram-Schmidt
// (mgs.py:145-221), back-substitutes (mgs.py:229-289), forms x + dx
// (newton.py:92) and applies run_newton's convergence test
// (newton.py:121-130) -- all inside one CTA, so a whole batch of starts is
// one launch with no inter-CTA synchronisation.
//
// Schedule: left-looking over panels of P columns.  A panel is loaded into
// shared memory, receives the updates of every earlier pivot q_k (streamed
// from global memory, prefetched one sweep ahead), and is then factored in
// place.  Column j still receives sweeps k = 0..j-1 in order with the
// reference's dot products and updates, and the panel order only changes
// when each column is touched, so R, Q and x are bit-identical to the
// right-looking reference.  Compared with sweeping the trailing matrix per
// pivot this reads the matrix once and Q once per panel instead of
// n(n+1)/2 column passes: the kernel stays on the FP64 pipes instead of HBM.
//
// Rows: thread t owns the aligned block [t*B, t*B+B) of every column, so
// all panel traffic is thread-private (shared memory as a register
// extension) and the only synchronisation is in the reductions.  The P dot
// products of a sweep are reduced together by a warp reduce-scatter (each
// shuffle level halves the columns a lane carries, so no addition is done
// twice) followed by a tree over warps; every reduction keeps tree_sum's
// right-pruned pairwise order.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace pn {

// panel width: P element accumulators (P*es doubles) must fit in registers
template <class E> struct PanelMax {
  static constexpr int v = 64 / Traits<E>::es > 32 ? 32 : 64 / Traits<E>::es;
};

// float() of a field element (xprec.py:153-154, 261-262); quad double uses
// Python's math.fsum (CPython msum with its half-even fix-up)
__device__ __forceinline__ double to_float(const F<1> &a) { return a.c[0]; }
__device__ __forceinline__ double to_float(const F<2> &a) { return __dadd_rn(a.c[0], a.c[1]); }
__device__ inline double to_float(const F<4> &a) {
  double p[4];
  int np = 0;
  for (int t = 0; t < 4; ++t) {
    double x = a.c[t];
    int i = 0;
    for (int j = 0; j < np; ++j) {
      double y = p[j];
      if (fabs(x) < fabs(y)) {
        const double tmp = x;
        x = y;
        y = tmp;
      }
      const double hi = __dadd_rn(x, y), yr = __dsub_rn(hi, x), lo = __dsub_rn(y, yr);
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    np = i;
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
  return hi;
}

// float(modulus(v)) (newton.py:33-34; xprec.py:327-328 complex, abs real)
template <int NC> __device__ __forceinline__ double mod_float(const C<NC> &v) { return to_float(fsqrt(eabs2(v))); }
template <int NC> __device__ __forceinline__ double mod_float(const F<NC> &v) {
  return to_float(ehi(v) < 0.0 ? fneg(v) : v);
}

// max over the CTA (exact, order independent); result in every thread
template <int NT> __device__ __forceinline__ double block_max(double v, double *sm) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, s));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = sm[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) r = fmax(r, sm[w]);
  return r;
}

template <class E, int B, int P, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_solve_batch(const int32_t *__restrict__ slots, int m, int n, double *__restrict__ Aall, long long As,
                  double *__restrict__ Qall, long long Qs, double *__restrict__ Rall, long long Rs,
                  double *__restrict__ xall, long long xs, double *__restrict__ dxall, double eps, double tol,
                  int32_t *__restrict__ flags) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  constexpr int NC = Traits<E>::nc;
  constexpr int MP = NT * B;  // padded rows of a panel column
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double smem[];
  double *pan = smem;                                              // P x es planes x MP
  E *sred = reinterpret_cast<E *>(pan + (size_t)P * es * MP);      // 2 x NW * P
  E *sres = sred + 2 * NW * P;                                     // 2 x P
  int par = 0;  // parity of the double-buffered reduction slots
  __shared__ double s_orig[P];
  __shared__ double s_max[NW];
  __shared__ int s_sing;

  const int slot = slots[blockIdx.x];
  const double *A = Aall + slot * As;
  double *Q = Qall + slot * Qs;
  double *R = Rall + slot * Rs;
  double *x = xall + slot * xs;
  double *dx = dxall + (long long)slot * n * es;
  const int t = threadIdx.x;
  const int nparts = (m + B - 1) / B;
  const int valid = m - t * B <= 0 ? 0 : (m - t * B >= B ? B : m - t * B);
  const long long ldR = n + 1;

  // panel element (column c, this thread's q-th row); planes, row slot q*NT+t
  auto pget = [&](int c, int q) -> E {
    E v;
    double *d = reinterpret_cast<double *>(&v);
#pragma unroll
    for (int p = 0; p < es; ++p) d[p] = pan[((size_t)c * es + p) * MP + q * NT + t];
    return v;
  };
  auto pput = [&](int c, int q, const E &v) {
    const double *d = reinterpret_cast<const double *>(&v);
#pragma unroll
    for (int p = 0; p < es; ++p) pan[((size_t)c * es + p) * MP + q * NT + t] = d[p];
  };
  auto qrow = [&](int k, E (&qv)[B]) {
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int r = t * B + q;
      qv[q] = r < m ? eload<E>(Q + ((long long)k * m + r) * es) : ezero<E>();
    }
  };
  // one sweep: r_c = tree_sum(conj(q) a_c), a_c -= q r_c for the panel
  // columns c in [c0, np) (mgs.py:201-215); R[k, j0+c] = r_c
  auto sweep = [&](const E (&qv)[B], int k, int j0, int c0, int np) {
    E part[P];
#pragma unroll
    for (int c = 0; c < P; ++c) {
      E pr[B];
#pragma unroll
      for (int q = 0; q < B; ++q) pr[q] = emul(econj(qv[q]), pget(c, q));
      part[c] = local_tree<E, B>(pr, valid);
    }
    const E *res = sres + par * P;
    multi_tree_reduce<E, P, NT>(part, nparts, sred, sres, par);
#pragma unroll
    for (int c = 0; c < P; ++c) {
      if (c < c0 || c >= np) continue;
      const E rk = res[c];
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q < valid) pput(c, q, esub(pget(c, q), emul(qv[q], rk)));
    }
    if (t >= c0 && t < np) estore(R + ((long long)(j0 + t) * ldR + k) * es, res[t]);
  };

  for (int j0 = 0; j0 <= n; j0 += P) {
    const int np = min(P, n + 1 - j0);
    // ---- load the panel; original norms of its columns (mgs.py:171-172)
#pragma unroll
    for (int c = 0; c < P; ++c)
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int r = t * B + q;
        pput(c, q, (c < np && r < m) ? eload<E>(A + ((long long)(j0 + c) * m + r) * es) : ezero<E>());
      }
    {
      Rl part[P];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        Rl a2[B];
#pragma unroll
        for (int q = 0; q < B; ++q) a2[q] = eabs2(pget(c, q));
        part[c] = local_tree<Rl, B>(a2, valid);
      }
      Rl *rred = reinterpret_cast<Rl *>(sred), *rres = reinterpret_cast<Rl *>(sres);
      const Rl *res = rres + par * P;
      multi_tree_reduce<Rl, P, NT>(part, nparts, rred, rres, par);
      if (t < np) s_orig[t] = fsqrt(res[t]).c[0];
      __syncthreads();
    }
    // ---- left-looking: sweeps of every earlier pivot, q prefetched one ahead
    if (j0 > 0) {
      E qv[B], qn[B];
      qrow(0, qv);
      for (int k = 0; k < j0; ++k) {
        if (k + 1 < j0) qrow(k + 1, qn);
        sweep(qv, k, j0, 0, np);
#pragma unroll
        for (int q = 0; q < B; ++q) qv[q] = qn[q];
      }
    }
    // ---- factor the panel in place
    for (int kk = 0; kk < np; ++kk) {
      const int k = j0 + kk;
      Rl a2[B];
#pragma unroll
      for (int q = 0; q < B; ++q) a2[q] = eabs2(pget(kk, q));
      Rl *rred = reinterpret_cast<Rl *>(sred);
      const Rl rkk = fsqrt(block_tree_reduce<Rl, NT>(local_tree<Rl, B>(a2, valid), nparts, rred));
      if (k < n) {
        // breakdown: rkk_hi <= BREAKDOWN_FACTOR * n * eps * orig (mgs.py:176-181)
        const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), s_orig[kk]);
        if (rkk.c[0] <= thr) {
          if (t == 0) flags[slot] = 2;
          return;  // uniform across the CTA
        }
      }
      if (t == 0) estore(R + ((long long)k * ldR + k) * es, eembed(rkk, (E *)nullptr));
      if (k == n) break;  // R[n, n] = z
      const RDiv<NC> p = rdiv_prepare(rkk);
      E qv[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int r = t * B + q;
        qv[q] = ediv_prepared(pget(kk, q), p);
        if (r < m) estore(Q + ((long long)k * m + r) * es, qv[q]);
      }
      if (kk + 1 < np) sweep(qv, k, j0, kk + 1, np);
    }
    __syncthreads();
  }

  // ---- back substitution R dx = y, y = R[:n, n] (mgs.py:229-289) --------
  // y and the reciprocals of r_jj's squared modulus live in the panel area
  using RD = RDiv<NC>;
  E *ys = reinterpret_cast<E *>(pan);                  // n elements
  E *xsol = ys + n;                                    // n elements
  RD *prep = reinterpret_cast<RD *>(xsol + n);         // n reciprocals
  if (t == 0) s_sing = -1;
  __syncthreads();
  for (int j = t; j < n; j += NT) {
    ys[j] = eload<E>(R + ((long long)n * ldR + j) * es);
    const double *dg = R + ((long long)j * ldR + j) * es;
    bool nz = false;
#pragma unroll
    for (int c = 0; c < es; ++c) nz |= dg[c] != 0.0;
    if (!nz) atomicMax(&s_sing, j);
    else prep[j] = rdiv_prepare(ediv_den(eload<E>(dg)));
  }
  __syncthreads();
  if (s_sing >= 0) {
    if (t == 0) flags[slot] = 3;  // SingularMatrixError (mgs.py:241-242)
    return;
  }
  const int lane = t & 31;
  for (int hi = n; hi > 0; hi -= 32) {
    const int lo = hi - 32 > 0 ? hi - 32 : 0;
    if (t < 32) {  // warp 0 solves the diagonal block; lane l holds row lo+l
      E yr = lo + lane < hi ? ys[lo + lane] : ezero<E>();
      E xl = ezero<E>();
      for (int j = hi - 1; j >= lo; --j) {
        const int jl = j - lo;
        if (lane == jl) xl = ediv_with(yr, eload<E>(R + ((long long)j * ldR + j) * es), prep[j]);
        const E xj = eshfl_idx(xl, jl);
        if (lane < jl) yr = esub(yr, emul(eload<E>(R + ((long long)j * ldR + lo + lane) * es), xj));
      }
      if (lo + lane < hi) xsol[lo + lane] = xl;
    }
    __syncthreads();
    // rows above the block, subtractions in descending column order
    for (int r = t; r < lo; r += NT) {
      E v = ys[r];
      for (int j = hi - 1; j >= lo; --j) v = esub(v, emul(eload<E>(R + ((long long)j * ldR + r) * es), xsol[j]));
      ys[r] = v;
    }
    __syncthreads();
  }

  // ---- x_next = x + dx, norms, convergence (newton.py:92, 121-130) ------
  double dmax = 0.0, xmax = 0.0;
  for (int i = t; i < n; i += NT) {
    const E d = xsol[i];
    const E xn = eadd(eload<E>(x + (long long)i * es), d);
    estore(x + (long long)i * es, xn);
    estore(dx + (long long)i * es, d);
    dmax = fmax(dmax, mod_float(d));
    xmax = fmax(xmax, mod_float(xn));
  }
  const double dxn = block_max<NT>(dmax, s_max);
  const double xnn = block_max<NT>(xmax, s_max);
  if (t == 0) {
    const double tl = tol > 0.0 ? tol : __dmul_rn(__dmul_rn(10.0, eps), __dadd_rn(1.0, xnn));
    flags[slot] = dxn <= tl ? 1 : 0;
  }
}

template <class E, int B, int P, int MINB>
static void launch_solve(int nb, const int32_t *slots, int m, int n, double *A, long long As, double *Q,
                         long long Qs, double *R, long long Rs, double *x, long long xs, double *dx, double eps,
                         double tol, int32_t *flags, cudaStream_t st) {
  constexpr int NT = 256;
  constexpr int es = Traits<E>::es;
  const size_t pan = (size_t)P * es * NT * B * sizeof(double);
  const size_t bsub = (size_t)n * (2 * es + Traits<E>::nc) * sizeof(double);
  const size_t smem = std::max(pan, bsub) + (size_t)2 * (NT / 32 + 1) * P * es * sizeof(double);
  PN_REQUIRE(smem <= 227 * 1024, PN_E_ARG, "batched solve: n=%d needs %zu B of shared memory", n, smem);
  auto kern = k_solve_batch<E, B, P, NT, MINB>;
  PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nb, NT, smem, st>>>(slots, m, n, A, As, Q, Qs, R, Rs, x, xs, dx, eps, tol, flags);
  PN_CHECK_LAUNCH();
  count_launch(1);
}

template <class E>
void solve_batch_impl(int nb, const int32_t *slots, int m, int n, double *A, long long As, double *Q, long long Qs,
                      double *R, long long Rs, double *x, long long xs, double *dx, double tol, int32_t *flags,
                      cudaStream_t st) {
  constexpr int PM = PanelMax<E>::v;
  const double eps = Traits<E>::nc == 1 ? 0x1p-53 : Traits<E>::nc == 2 ? 0x1p-104 : 0x1p-209;
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  PN_REQUIRE(m <= 1024, PN_E_ARG, "batched solve supports m <= 1024 rows (got %d)", m);
  if (nb <= 0) return;
  // half the panel width and two CTAs per SM at m <= 256 (more warps to hide
  // FP64 latency, twice the Q traffic): 3524 vs 3120 start-iterations/s on
  // C5 against the full panel (r01)
  if (m <= 256) {
    launch_solve<E, 1, PM / 2, 2>(nb, slots, m, n, A, As, Q, Qs, R, Rs, x, xs, dx, eps, tol, flags, st);
  } else if (m <= 512) {
    launch_solve<E, 2, PM / 2, 1>(nb, slots, m, n, A, As, Q, Qs, R, Rs, x, xs, dx, eps, tol, flags, st);
  } else {
    launch_solve<E, 4, PM / 4, 1>(nb, slots, m, n, A, As, Q, Qs, R, Rs, x, xs, dx, eps, tol, flags, st);
  }
}

#ifdef PN_NC
template void solve_batch_impl<PnLevel>(int, const int32_t *, int, int, double *, long long, double *, long long,
                                        double *, long long, double *, long long, double *, double, int32_t *,
                                        cudaStream_t);
#endif

}  // namespace pn
