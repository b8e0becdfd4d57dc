// residual.cu -- residual_check (mgs.py:311-357): max componentwise |A - QR|
// of a factorisation, recomputed in the next-higher precision (d -> dd,
// dd -> qd) with the reference's exact operation sequence:
//   acc = 0; for k: acc = acc + promote(Q[:, k]) * promote(R[k, :n]);
//   diff = promote(A) - acc; result = sqrt(max hi(abs2(diff))).
// promote() pads the extra components with +0.0 (varith.py:200-209), so the
// value is bit-identical to the reference.  The qd check runs in 320-bit
// mpfr in the reference and is not offered here.
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

template <class E>
double residual_impl(int m, int n, const double *A, const double *Q, const double *R, cudaStream_t st) {
  if constexpr (Traits<E>::nc == 4) {
    PN_REQUIRE(false, PN_E_ARG, "residual_check of a quad-double factorisation needs 320-bit arithmetic "
                                "(mgs.py:334-357); only d and dd are checked on the GPU");
    return 0.0;
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
