// newton.cu -- one Gauss-Newton correction, device resident end to end
// (newton.py:82-103): f, J at x -> [J | -f] -> MGS least squares -> x + dx,
// plus the field moduli the host turns into the reference's float norms.
#include "common.cuh"
#include "internal.h"

using namespace pn;

extern "C" int pn_newton_step(pn_system *sys, const double *x, double *x_next, double *f, double *dx,
                              double *fmod, double *dxmod, double *xmod, pn_numinfo *info, void *stream) {
  PN_API_BEGIN
  PN_REQUIRE(sys && x, PN_E_ARG, "pn_newton_step: NULL argument");
  const int m = sys->m, n = sys->n, es = sys->es, nc = sys->nc, cplx = sys->cplx;
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t ebytes = (size_t)es * sizeof(double);
  DevIn din(x, (size_t)n * es, st);
  sys->xbuf.ensure((size_t)n * ebytes);
  sys->Abuf.ensure((size_t)m * (n + 1) * ebytes);
  sys->fbuf.ensure((size_t)m * ebytes);
  sys->vbuf.ensure((size_t)m * n * ebytes);           // Q
  sys->Rbuf.ensure((size_t)(n + 1) * (n + 1) * ebytes);
  sys->xsol.ensure((size_t)2 * n * ebytes);           // dx, x_next
  double *xa = sys->xbuf.d(), *A = sys->Abuf.d(), *fa = sys->fbuf.d();
  double *Q = sys->vbuf.d(), *R = sys->Rbuf.d(), *dxa = sys->xsol.d(), *xn = dxa + (size_t)n * es;

  cudaEvent_t ev[4];
  for (auto &e : ev) PN_CHECK_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  planes_to_aos(es, n, din.d, xa, st);
  PN_CHECK_CUDA(cudaEventRecord(ev[0], st));
  // A = J(x) with b = -f(x) in column n (newton.py:84-87)
  evaldiff_device(sys, xa, fa, A, m, n, st);
  PN_CHECK_CUDA(cudaEventRecord(ev[1], st));
  mgs_factor_device(nc, cplx, m, n, A, Q, R, sys->mgs, st);
  backsub_device(nc, cplx, n, R, dxa, sys->mgs, st);
  PN_CHECK_CUDA(cudaEventRecord(ev[2], st));
  // x_next = x + dx (newton.py:92)
  vec_op_aos(nc, cplx, PN_OP_ADD, n, xa, dxa, xn, st);
  PN_CHECK_CUDA(cudaEventRecord(ev[3], st));

  DevOut o_x(x_next, (size_t)n * es, st), o_f(f, (size_t)m * es, st), o_dx(dx, (size_t)n * es, st);
  DevOut o_fm(fmod, (size_t)m * nc, st), o_dm(dxmod, (size_t)n * nc, st), o_xm(xmod, (size_t)n * nc, st);
  if (o_x.d) aos_to_planes(es, n, xn, o_x.d, st);
  if (o_f.d) aos_to_planes(es, m, fa, o_f.d, st);
  if (o_dx.d) aos_to_planes(es, n, dxa, o_dx.d, st);
  // moduli: computed AoS (nc doubles per element) into scratch, then planes
  const int len[3] = {m, n, n};
  const double *src[3] = {fa, dxa, xn};
  DevOut *dst[3] = {&o_fm, &o_dm, &o_xm};
  size_t need = 0;
  for (int i = 0; i < 3; ++i) need += dst[i]->d ? (size_t)len[i] * nc : 0;
  DevBuf mod(need * sizeof(double) + 8, st);
  size_t off = 0;
  for (int i = 0; i < 3; ++i) {
    if (!dst[i]->d) continue;
    vec_op_aos(nc, cplx, PN_OP_MODULUS, len[i], src[i], nullptr, mod.d() + off, st);
    aos_to_planes(nc, len[i], mod.d() + off, dst[i]->d, st);
    off += (size_t)len[i] * nc;
  }
  const int rc = mgs_read_status(sys->mgs, info, st);  // synchronises
  if (rc) return rc;
  o_x.finish(st);
  o_f.finish(st);
  o_dx.finish(st);
  o_fm.finish(st);
  o_dm.finish(st);
  o_xm.finish(st);
  if (info) {
    double zhi = 0.0;
    PN_CHECK_CUDA(cudaMemcpyAsync(&zhi, R + ((size_t)n * (n + 1) + n) * es, sizeof(double),
                                  cudaMemcpyDeviceToHost, st));
    PN_CHECK_CUDA(cudaStreamSynchronize(st));
    info->z = zhi;
    float ms[3] = {0, 0, 0};
    for (int i = 0; i < 3; ++i) PN_CHECK_CUDA(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
    info->t_evaluate = ms[0] * 1e-3;
    info->t_solve = ms[1] * 1e-3;
    info->t_update = ms[2] * 1e-3;
  }
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}
