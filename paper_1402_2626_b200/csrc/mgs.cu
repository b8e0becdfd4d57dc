// mgs.cu -- subsystem (3): right-looking modified Gram-Schmidt on [A b] and
// back substitution, on the FP64 pipes (no tensor cores: every product of the
// extended-precision EFT sequence is individually rounded, so this is not a
// DGEMM contraction).
//
// Reference: mgs_qr (mgs.py:145-221; the delayed variant is bit-identical),
// _column_norm (128-137), back_substitute(_staged) (229-289),
// least_squares_solve (299-305), MgsBreakdownError / SingularMatrixError
// (22-36), BREAKDOWN_FACTOR (118-119).
//
// Layout: A and Q are AoS column-major (ld = m): a column is one contiguous
// run of m elements, so a CTA streams its column with coalesced 16-64 B
// element loads.  R is AoS column-major with ld = n+1.
//
// Schedule: one launch per sweep k.  The CTA that updates column k+1 in
// sweep k immediately forms its norm, checks breakdown and writes q_{k+1}
// (look-ahead normalisation), so sweep k+1 starts from a published pivot.
// Each CTA handles one column at a time; thread t owns the aligned row block
// [t*B, t*B+B), so dot products and norms reduce in the reference's
// canonical pairwise order (block_tree_reduce) and are bit-identical.
#include "common.cuh"
#include "internal.h"

namespace pn {


template <class E, int B>
__device__ __forceinline__ void load_rows(E (&v)[B], const double *__restrict__ col, int row0, int m) {
  constexpr int es = Traits<E>::es;
#pragma unroll
  for (int q = 0; q < B; ++q) v[q] = (row0 + q < m) ? eload<E>(col + (long long)(row0 + q) * es) : ezero<E>();
}

template <class E, int B>
__device__ __forceinline__ void store_rows(double *__restrict__ col, const E (&v)[B], int row0, int m) {
  constexpr int es = Traits<E>::es;
#pragma unroll
  for (int q = 0; q < B; ++q)
    if (row0 + q < m) estore(col + (long long)(row0 + q) * es, v[q]);
}

// ||col||_2 = sqrt(tree_sum(abs2(col))) as a real element (mgs.py:128-137)
template <class E, int B>
__device__ __forceinline__ typename Traits<E>::R column_norm(const E (&v)[B], int row0, int m,
                                                             typename Traits<E>::R *sm) {
  using R = typename Traits<E>::R;
  R a2[B];
#pragma unroll
  for (int q = 0; q < B; ++q) a2[q] = eabs2(v[q]);
  const int valid = m - row0 < 0 ? 0 : (m - row0 > B ? B : m - row0);
  R part = local_tree<R, B>(a2, valid);
  const int nparts = (m + B - 1) / B;
  R s = block_tree_reduce<R, kMgsThreads>(part, nparts, sm);
  return fsqrt(s);
}

// pivot handling shared by the first pivot and the look-ahead: breakdown
// test (mgs.py:176-181), R[k,k] = real_embed(rkk), Q[:,k] = col / rkk
template <class E, int B>
__device__ __forceinline__ bool finish_pivot(const E (&v)[B], int row0, int m, int n, int k,
                                             const typename Traits<E>::R &rkk, const double *__restrict__ orig,
                                             double eps, double *__restrict__ Q, double *__restrict__ R,
                                             MgsStatus *status) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  if (k < n) {
    // threshold = BREAKDOWN_FACTOR * n * eps * orig_norms[k], left to right
    const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), orig[k]);
    if (rkk.c[0] <= thr) {
      if (threadIdx.x == 0) {
        status->k = k;
        status->rkk = rkk.c[0];
        status->thr = thr;
        __threadfence();
        status->code = PN_E_BREAKDOWN;
      }
      return false;
    }
  }
  if (threadIdx.x == 0) estore(R + ((long long)k * (n + 1) + k) * es, eembed(rkk, (E *)nullptr));
  if (k < n) {
    const RDiv<Traits<E>::nc> p = rdiv_prepare(rkk);
    double *qc = Q + (long long)k * m * es;
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (row0 + q < m) estore(qc + (long long)(row0 + q) * es, ediv_prepared(v[q], p));
  }
  return true;
  (void)sizeof(Rl);
}

// hi component of the initial column norms (mgs.py:171-172)
template <class E, int B>
__global__ void __launch_bounds__(kMgsThreads) k_mgs_orig(const double *__restrict__ A, int m, int n,
                                                          double *__restrict__ orig) {
  using R = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  __shared__ R sm[kMgsThreads / 32];
  const int row0 = threadIdx.x * B;
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    E v[B];
    load_rows<E, B>(v, A + (long long)j * m * es, row0, m);
    R nrm = column_norm<E, B>(v, row0, m, sm);
    if (threadIdx.x == 0) orig[j] = nrm.c[0];
  }
}

// the first pivot (k = 0)
template <class E, int B>
__global__ void __launch_bounds__(kMgsThreads) k_mgs_pivot(const double *__restrict__ A, int m, int n, int k,
                                                           const double *__restrict__ orig, double eps,
                                                           double *__restrict__ Q, double *__restrict__ R,
                                                           MgsStatus *status) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  __shared__ Rl sm[kMgsThreads / 32];
  if (status->code) return;
  const int row0 = threadIdx.x * B;
  E v[B];
  load_rows<E, B>(v, A + (long long)k * m * es, row0, m);
  Rl rkk = column_norm<E, B>(v, row0, m, sm);
  finish_pivot<E, B>(v, row0, m, n, k, rkk, orig, eps, Q, R, status);
}

// sweep k: columns j = k+1..n get r_kj = tree_sum(conj(q) a_j) and
// a_j -= q r_kj (mgs.py:201-215); column k+1 also becomes the next pivot
template <class E, int B>
__global__ void __launch_bounds__(kMgsThreads) k_mgs_sweep(double *__restrict__ A, int m, int n, int k,
                                                           const double *__restrict__ orig, double eps,
                                                           double *__restrict__ Q, double *__restrict__ R,
                                                           MgsStatus *status) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  __shared__ E sme[kMgsThreads / 32];
  __shared__ Rl smr[kMgsThreads / 32];
  if (status->code) return;
  const int row0 = threadIdx.x * B;
  const int valid = m - row0 < 0 ? 0 : (m - row0 > B ? B : m - row0);
  const int nparts = (m + B - 1) / B;
  E qv[B];
  load_rows<E, B>(qv, Q + (long long)k * m * es, row0, m);
  for (int j = k + 1 + blockIdx.x; j <= n; j += gridDim.x) {
    double *col = A + (long long)j * m * es;
    E a[B], pr[B];
    load_rows<E, B>(a, col, row0, m);
#pragma unroll
    for (int q = 0; q < B; ++q) pr[q] = emul(econj(qv[q]), a[q]);
    E part = local_tree<E, B>(pr, valid);
    const E r = block_tree_reduce<E, kMgsThreads>(part, nparts, sme);
#pragma unroll
    for (int q = 0; q < B; ++q) a[q] = esub(a[q], emul(qv[q], r));
    store_rows<E, B>(col, a, row0, m);
    if (threadIdx.x == 0) estore(R + ((long long)j * (n + 1) + k) * es, r);
    if (j == k + 1) {
      Rl rkk = column_norm<E, B>(a, row0, m, smr);
      finish_pivot<E, B>(a, row0, m, n, k + 1, rkk, orig, eps, Q, R, status);
    }
  }
}

// back substitution R x = y, y = R[:n, n] (mgs.py:229-247): descending j,
// x_j = y_j / r_jj (full complex division), y[:j] -= R[:j, j] x_j.  The
// division's reciprocal depends on r_jj only, so it is prepared for all j
// in parallel first; the sequential chain is one multiply per step.
template <class E, int NT>
__global__ void __launch_bounds__(NT) k_backsub(const double *__restrict__ R, int n, double *__restrict__ x,
                                                RDiv<Traits<E>::nc> *__restrict__ prep, E *__restrict__ xs,
                                                MgsStatus *status) {
  constexpr int es = Traits<E>::es;
  constexpr int NC = Traits<E>::nc;
  const long long ld = n + 1;
  __shared__ int s_sing;
  if (status->code) return;  // the factorization already failed
  if (threadIdx.x == 0) s_sing = -1;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += NT) {
    const double *dg = R + ((long long)j * ld + j) * es;
    bool nz = false;
#pragma unroll
    for (int p = 0; p < es; ++p) nz |= dg[p] != 0.0;
    if (!nz) atomicMax(&s_sing, j);
    else prep[j] = rdiv_prepare(ediv_den(eload<E>(dg)));
  }
  __syncthreads();
  if (s_sing >= 0) {
    if (threadIdx.x == 0) {
      status->k = s_sing;
      status->code = PN_E_SINGULAR;
    }
    return;
  }
  // rows i owned by thread i % NT, kept in registers (up to RPT rows)
  constexpr int RPT = 4;
  E y[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = threadIdx.x + q * NT;
    y[q] = i < n ? eload<E>(R + ((long long)n * ld + i) * es) : ezero<E>();
  }
  for (int j = n - 1; j >= 0; --j) {
    if ((j % NT) == (int)threadIdx.x) {
      const int q = j / NT;
      E yj = y[0];
#pragma unroll
      for (int qq = 1; qq < RPT; ++qq) yj = (qq == q) ? y[qq] : yj;
      const E rjj = eload<E>(R + ((long long)j * ld + j) * es);
      xs[j] = ediv_with(yj, rjj, prep[j]);
    }
    __syncthreads();
    const E xj = xs[j];
    const double *rc = R + (long long)j * ld * es;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = threadIdx.x + q * NT;
      if (i < j) y[q] = esub(y[q], emul(eload<E>(rc + (long long)i * es), xj));
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += NT) estore(x + (long long)j * es, xs[j]);
  (void)sizeof(RDiv<NC>);
}

static double level_eps(int nc) { return nc == 1 ? 0x1p-53 : nc == 2 ? 0x1p-104 : 0x1p-209; }

template <class E, int B>
static void mgs_run(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  constexpr int es = Traits<E>::es;
  MgsStatus *status = w.status.as<MgsStatus>();
  double *orig = w.orig.d();
  const double eps = level_eps(Traits<E>::nc);
  const int sms = num_sms();
  k_mgs_orig<E, B><<<std::min(n, sms * 4), kMgsThreads, 0, st>>>(A, m, n, orig);
  PN_CHECK_LAUNCH();
  k_mgs_pivot<E, B><<<1, kMgsThreads, 0, st>>>(A, m, n, 0, orig, eps, Q, R, status);
  PN_CHECK_LAUNCH();
  count_launch(2);
  for (int k = 0; k < n; ++k) {
    const int cols = n - k;
    const int grid = std::min(cols, sms * 4);
    k_mgs_sweep<E, B><<<grid, kMgsThreads, 0, st>>>(A, m, n, k, orig, eps, Q, R, status);
  }
  PN_CHECK_LAUNCH();
  count_launch(n);
  (void)es;
}

template <class E>
void mgs_impl(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  switch (rows_per_thread(m)) {
    case 1: mgs_run<E, 1>(m, n, A, Q, R, w, st); break;
    case 2: mgs_run<E, 2>(m, n, A, Q, R, w, st); break;
    case 4: mgs_run<E, 4>(m, n, A, Q, R, w, st); break;
    case 8: mgs_run<E, 8>(m, n, A, Q, R, w, st); break;
    default: mgs_run<E, 16>(m, n, A, Q, R, w, st); break;
  }
}

template <class E>
void backsub_impl(int n, const double *R, double *x, MgsWork &w, cudaStream_t st) {
  constexpr int NT = kBacksubThreads;
  constexpr int es = Traits<E>::es;
  DevBuf prep((size_t)n * Traits<E>::nc * sizeof(double) + 16, st);
  DevBuf xs((size_t)n * es * sizeof(double) + 16, st);
  k_backsub<E, NT><<<1, NT, 0, st>>>(R, n, x, prep.as<RDiv<Traits<E>::nc>>(), xs.as<E>(), w.status.as<MgsStatus>());
  PN_CHECK_LAUNCH();
  count_launch(1);
}

// one translation unit per precision level (see Makefile)
#ifdef PN_NC
template void mgs_impl<PnLevel>(int, int, double *, double *, double *, MgsWork &, cudaStream_t);
template void backsub_impl<PnLevel>(int, const double *, double *, MgsWork &, cudaStream_t);
#endif

}  // namespace pn
