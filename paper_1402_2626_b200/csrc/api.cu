// api.cu -- level dispatch and the C-ABI entry points of the evaluation and
// least-squares subsystems (the per-level kernels live in evaldiff.cu and
// mgs.cu, compiled once per precision level).
#include "common.cuh"
#include "internal.h"
#include "nvtx.h"

namespace pn {

void evaldiff_device(pn_system *sys, const double *x, double *f, double *A, long long ldA, int negf_col,
                     cudaStream_t st) {
  dispatch_level(sys->nc, sys->cplx,
                 [&]<class E>() { evaldiff_impl<E>(sys, x, f, A, ldA, negf_col, st); });
}



void mgs_factor_device(int nc, int cplx, int m, int n, double *A, double *Q, double *R, MgsWork &w,
                       cudaStream_t st) {
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  const int B = rows_per_thread(m);
  PN_REQUIRE(B <= 16, PN_E_ARG, "MGS supports at most %d rows (got m=%d)", 16 * kMgsThreads, m);
  const int es = nc * (cplx ? 2 : 1);
  w.orig.ensure((size_t)n * sizeof(double));
  w.status.ensure(sizeof(MgsStatus));
  PN_CHECK_CUDA(cudaMemsetAsync(w.status.p, 0, sizeof(MgsStatus), st));
  PN_CHECK_CUDA(cudaMemsetAsync(R, 0, (size_t)(n + 1) * (n + 1) * es * sizeof(double), st));
  dispatch_level(nc, cplx, [&]<class E>() { mgs_impl<E>(m, n, A, Q, R, w, st); });
}

void backsub_device(int nc, int cplx, int n, const double *R, double *x, MgsWork &w, cudaStream_t st) {
  PN_REQUIRE(n >= 1, PN_E_ARG, "back substitution needs n >= 1");
  w.status.ensure(sizeof(MgsStatus));
  dispatch_level(nc, cplx, [&]<class E>() { backsub_impl<E>(n, R, x, w, st); });
}


int mgs_read_status(MgsWork &w, pn_numinfo *info, cudaStream_t st) {
  MgsStatus s;
  PN_CHECK_CUDA(cudaMemcpyAsync(&s, w.status.p, sizeof(s), cudaMemcpyDeviceToHost, st));
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  if (info) {
    if (s.code == PN_E_BREAKDOWN) {
      info->k = s.k;
      info->rkk = s.rkk;
      info->threshold = s.thr;
    } else if (s.code == PN_E_SINGULAR) {
      info->index = s.k;
    }
  }
  if (s.code == PN_E_BREAKDOWN)
    set_error("MGS breakdown at column %d: r_kk=%.3e <= %.3e", s.k, s.rkk, s.thr);
  else if (s.code == PN_E_SINGULAR)
    set_error("zero diagonal entry at index %d", s.k);
  return s.code;
}



}  // namespace pn

using namespace pn;


extern "C" int pn_evaldiff(pn_system *sys, const double *x, double *f, double *J, pn_counts *counts, void *stream) {
  PN_API_BEGIN
  NvtxRange range("pn_evaldiff");
  PN_REQUIRE(sys && x, PN_E_ARG, "pn_evaldiff: NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int es = sys->es, m = sys->m, n = sys->n;
  DevIn dx(x, (size_t)n * es, st);
  sys->xbuf.ensure((size_t)n * es * sizeof(double));
  planes_to_aos(es, n, dx.d, sys->xbuf.d(), st);
  sys->Abuf.ensure((size_t)std::max(m, 1) * (n + 1) * es * sizeof(double));
  sys->fbuf.ensure((size_t)std::max(m, 1) * es * sizeof(double));
  evaldiff_device(sys, sys->xbuf.d(), sys->fbuf.d(), sys->Abuf.d(), m, -1, st);
  DevOut df(f, (size_t)m * es, st);
  DevOut dJ(J, (size_t)m * n * es, st);
  if (df.d) aos_to_planes(es, m, sys->fbuf.d(), df.d, st);
  if (dJ.d) aos_colmajor_to_planes(es, m, n, sys->Abuf.d(), m, dJ.d, st);
  df.finish(st);
  dJ.finish(st);
  if (counts) *counts = sys->counts;
  if (df.host || dJ.host) PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}



namespace {
struct LsqBuffers {
  DevBuf A, Q, R;
};
}  // namespace

extern "C" int pn_mgs_qr(int nc, int cplx, int32_t m, int32_t n, const double *aug, double *Q, double *R,
                         pn_numinfo *info, void *stream) {
  PN_API_BEGIN
  NvtxRange range("pn_mgs_qr");
  check_level(nc, cplx);
  PN_REQUIRE(aug, PN_E_ARG, "pn_mgs_qr: aug is NULL");
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  DevIn din(aug, (size_t)m * (n + 1) * es, st);
  DevBuf A((size_t)m * (n + 1) * es * sizeof(double), st);
  DevBuf Qd((size_t)m * n * es * sizeof(double), st);
  DevBuf Rd((size_t)(n + 1) * (n + 1) * es * sizeof(double), st);
  PN_CHECK_CUDA(cudaMemsetAsync(Qd.p, 0, Qd.bytes, st));
  planes_to_aos_colmajor(es, m, n + 1, din.d, A.d(), m, st);
  MgsWork w;
  mgs_factor_device(nc, cplx, m, n, A.d(), Qd.d(), Rd.d(), w, st);
  const int rc = mgs_read_status(w, info, st);
  if (rc) return rc;
  DevOut dq(Q, (size_t)m * n * es, st);
  DevOut dr(R, (size_t)(n + 1) * (n + 1) * es, st);
  if (dq.d) aos_colmajor_to_planes(es, m, n, Qd.d(), m, dq.d, st);
  if (dr.d) aos_colmajor_to_planes(es, n + 1, n + 1, Rd.d(), n + 1, dr.d, st);
  dq.finish(st);
  dr.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}

extern "C" int pn_back_substitute(int nc, int cplx, int32_t n, const double *R, double *x, pn_numinfo *info,
                                  void *stream) {
  PN_API_BEGIN
  check_level(nc, cplx);
  PN_REQUIRE(R && x && n >= 1, PN_E_ARG, "pn_back_substitute: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  DevIn din(R, (size_t)(n + 1) * (n + 1) * es, st);
  DevBuf Rd((size_t)(n + 1) * (n + 1) * es * sizeof(double), st);
  planes_to_aos_colmajor(es, n + 1, n + 1, din.d, Rd.d(), n + 1, st);
  DevBuf xd((size_t)n * es * sizeof(double), st);
  MgsWork w;
  w.status.ensure(sizeof(MgsStatus));
  PN_CHECK_CUDA(cudaMemsetAsync(w.status.p, 0, sizeof(MgsStatus), st));
  backsub_device(nc, cplx, n, Rd.d(), xd.d(), w, st);
  const int rc = mgs_read_status(w, info, st);
  if (rc) return rc;
  DevOut dx(x, (size_t)n * es, st);
  aos_to_planes(es, n, xd.d(), dx.d, st);
  dx.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}

extern "C" int pn_least_squares(int nc, int cplx, int32_t m, int32_t n, const double *aug, double *x, double *z,
                                double *Q, double *R, pn_numinfo *info, void *stream) {
  PN_API_BEGIN
  NvtxRange range("pn_least_squares");
  check_level(nc, cplx);
  PN_REQUIRE(aug && x, PN_E_ARG, "pn_least_squares: NULL argument");
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  DevIn din(aug, (size_t)m * (n + 1) * es, st);
  DevBuf A((size_t)m * (n + 1) * es * sizeof(double), st);
  DevBuf Qd((size_t)m * n * es * sizeof(double), st);
  DevBuf Rd((size_t)(n + 1) * (n + 1) * es * sizeof(double), st);
  PN_CHECK_CUDA(cudaMemsetAsync(Qd.p, 0, Qd.bytes, st));
  planes_to_aos_colmajor(es, m, n + 1, din.d, A.d(), m, st);
  MgsWork w;
  mgs_factor_device(nc, cplx, m, n, A.d(), Qd.d(), Rd.d(), w, st);
  int rc = mgs_read_status(w, info, st);
  if (rc) return rc;
  DevBuf xd((size_t)n * es * sizeof(double), st);
  backsub_device(nc, cplx, n, Rd.d(), xd.d(), w, st);
  rc = mgs_read_status(w, info, st);
  if (rc) return rc;
  double zhi = 0.0;
  PN_CHECK_CUDA(cudaMemcpyAsync(&zhi, Rd.d() + ((size_t)n * (n + 1) + n) * es, sizeof(double),
                                cudaMemcpyDeviceToHost, st));
  DevOut dx(x, (size_t)n * es, st);
  DevOut dq(Q, (size_t)m * n * es, st);
  DevOut dr(R, (size_t)(n + 1) * (n + 1) * es, st);
  aos_to_planes(es, n, xd.d(), dx.d, st);
  if (dq.d) aos_colmajor_to_planes(es, m, n, Qd.d(), m, dq.d, st);
  if (dr.d) aos_colmajor_to_planes(es, n + 1, n + 1, Rd.d(), n + 1, dr.d, st);
  dx.finish(st);
  dq.finish(st);
  dr.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  if (z) *z = zhi;
  if (info) info->z = zhi;
  PN_API_END
}

// residual_check (mgs.py:311-357) for d and dd factorisations
extern "C" int pn_residual_check(int nc, int cplx, int32_t m, int32_t n, const double *A, const double *Q,
                                 const double *R, double *out, void *stream) {
  PN_API_BEGIN
  check_level(nc, cplx);
  PN_REQUIRE(A && Q && R && out && m >= n && n >= 1, PN_E_ARG, "pn_residual_check: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  DevIn da(A, (size_t)m * n * es, st), dq(Q, (size_t)m * n * es, st), dr(R, (size_t)n * n * es, st);
  double r = 0.0;
  dispatch_level(nc, cplx, [&]<class E>() { r = residual_impl<E>(m, n, da.d, dq.d, dr.d, st); });
  *out = r;
  PN_API_END
}
