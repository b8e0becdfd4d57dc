// newton.cu -- one Gauss-Newton correction, device resident end to end
// (newton.py:82-103): f, J at x -> [J | -f] -> MGS least squares -> x + dx,
// plus the field moduli the host turns into the reference's float norms.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "nvtx.h"

using namespace pn;

// Graph replay of the device step for small systems (PN_GRAPH=1 always, 0
// never; default m*(n+1) <= 128*129, where the step is a few dozen short,
// launch-bound kernels).  The buffers of the step live in the system, so the
// captured pointers stay valid; per-call scratch inside the step becomes
// graph allocation nodes.
static bool use_step_graph(const pn_system *sys) {
  const char *v = getenv("PN_GRAPH");
  if (v) return strcmp(v, "0") != 0;
  return (long long)sys->m * (sys->n + 1) <= 128LL * 129;
}

// Capture the device step once, after a direct step has sized every arena
// and cached every table (so nothing inside allocates synchronously).  If
// the runtime refuses any call under capture, the system keeps the direct
// path (graph_state = -1); both paths launch the same kernels.
template <class F>
static void capture_step_graph(pn_system *sys, F &&device_step) {
  sys->graph_state = -1;
  if (!sys->graph_stream) {
    if (cudaStreamCreateWithFlags(&sys->graph_stream, cudaStreamNonBlocking) != cudaSuccess) return;
    for (auto &e : sys->gev)
      if (cudaEventCreate(&e) != cudaSuccess) return;
  }
  cudaStream_t gs = sys->graph_stream;
  if (cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return;
  const long long before = pn_launch_count();
  bool ok = true;
  try {
    device_step(gs, sys->gev, true);
  } catch (const Fail &) {
    ok = false;
  }
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(gs, &g);
  sys->graph_launches = pn_launch_count() - before;
  count_launch(-(int)sys->graph_launches);  // captured, not launched
  if (ok && e == cudaSuccess && g) {
    cudaGraphExec_t exec = nullptr;
    if (cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
      sys->step_graph = exec;
      sys->graph_state = 1;
    }
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();  // a refused capture leaves no sticky error
}

extern "C" int pn_newton_step(pn_system *sys, const double *x, double *x_next, double *f, double *dx,
                              double *fmod, double *dxmod, double *xmod, pn_numinfo *info, void *stream) {
  PN_API_BEGIN
  NvtxRange range("pn_newton_step");
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

  // phase events: created once per system and reused by every step
  if (!sys->pev[0])
    for (auto &e : sys->pev) PN_CHECK_CUDA(cudaEventCreate(&e));
  cudaEvent_t *evl = sys->pev;
  // the device step from x (AoS in xa) to x_next; `external` records the
  // phase events as graph nodes visible outside the graph
  auto device_step = [&](cudaStream_t s, cudaEvent_t *e, bool external) {
    auto rec = [&](cudaEvent_t ev) {
      PN_CHECK_CUDA(external ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal) : cudaEventRecord(ev, s));
    };
    rec(e[0]);
    // A = J(x) with b = -f(x) in column n (newton.py:84-87)
    {
      NvtxRange r("evaluate");
      evaldiff_device(sys, xa, fa, A, m, n, s);
    }
    rec(e[1]);
    {
      NvtxRange r("factor");
      mgs_factor_device(nc, cplx, m, n, A, Q, R, sys->mgs, s);
    }
    rec(e[4]);
    {
      NvtxRange r("back_substitute");
      backsub_device(nc, cplx, n, R, dxa, sys->mgs, s);
    }
    rec(e[2]);
    // x_next = x + dx (newton.py:92)
    vec_op_aos(nc, cplx, PN_OP_ADD, n, xa, dxa, xn, s);
    rec(e[3]);
  };
  planes_to_aos(es, n, din.d, xa, st);
  const bool graph = sys->graph_state == 1 && use_step_graph(sys);
  cudaEvent_t *ev = graph ? sys->gev : evl;
  if (graph) {
    PN_CHECK_CUDA(cudaGraphLaunch(sys->step_graph, st));
    count_launch((int)sys->graph_launches);
  } else {
    device_step(st, evl, false);
  }

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
    float mf = 0.f;
    PN_CHECK_CUDA(cudaEventElapsedTime(&mf, ev[1], ev[4]));
    info->t_factor = mf * 1e-3;
  }
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  if (sys->graph_state == 0 && use_step_graph(sys)) capture_step_graph(sys, device_step);
  PN_API_END
}

// ---------------------------------------------------------------------------
// Batched Newton runs: B independent run_newton
// calls (newton.py:106-132) on one system whose constant terms differ per
// start (the homotopy shift of newton.py:144-158).  The system's supports and
// coefficients stay resident; per start only the m constant coefficients
// and x change.  Starts are independent units, so multi-GPU runs shard them
// with no collective on the data path (bench.py gathers the results once).

namespace {

template <class E>
__global__ void k_scatter_consts(int m, const int32_t *__restrict__ cpos, const double *__restrict__ src,
                                 double *__restrict__ coeff) {
  constexpr int es = Traits<E>::es;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) estore(coeff + (long long)cpos[i] * es, eload<E>(src + (long long)i * es));
}

template <class E>
__global__ void k_gather_consts(int m, const int32_t *__restrict__ cpos, const double *__restrict__ coeff,
                                double *__restrict__ dst) {
  constexpr int es = Traits<E>::es;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) estore(dst + (long long)i * es, eload<E>(coeff + (long long)cpos[i] * es));
}

// Python's math.fsum (CPython's msum with the half-even fix-up): the float()
// of a quad double (xprec.py:261-262) used by the convergence test.
double host_fsum(const double *v, int n) {
  double p[16];
  int np = 0;
  for (int t = 0; t < n; ++t) {
    double x = v[t];
    int i = 0;
    for (int j = 0; j < np; ++j) {
      double y = p[j];
      if (std::fabs(x) < std::fabs(y)) std::swap(x, y);
      const double hi = x + y, yr = hi - x, lo = y - yr;
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
      hi = x + y;
      const double yr = hi - x;
      lo = y - yr;
      if (lo != 0.0) break;
    }
    if (np > 0 && ((lo < 0.0 && p[np - 1] < 0.0) || (lo > 0.0 && p[np - 1] > 0.0))) {
      const double y = lo * 2.0, x = hi + y, yr = x - hi;
      if (y == yr) hi = x;
    }
  }
  return hi;
}

// max over float(modulus(v)) (newton.py:33-34) from AoS real moduli
double host_inf_norm(const std::vector<double> &mod, int nc, int len) {
  double best = 0.0;
  for (int i = 0; i < len; ++i) {
    const double *c = mod.data() + (size_t)i * nc;
    const double v = nc == 1 ? c[0] : nc == 2 ? c[0] + c[1] : host_fsum(c, 4);
    if (v > best) best = v;
  }
  return best;
}

}  // namespace

static void newton_batch_serial(pn_system *sys, int64_t B, const double *x0, const double *consts, int max_iters,
                                double tol, double *x_out, int32_t *iters, int32_t *status, cudaStream_t st,
                                const DevBuf &cpos_d) {
  NvtxRange range("newton_batch_serial");
  PN_REQUIRE(sys && x0 && x_out && iters && status && B >= 0 && max_iters >= 1, PN_E_ARG,
             "pn_newton_batch: bad arguments");
  const int m = sys->m, n = sys->n, es = sys->es, nc = sys->nc, cplx = sys->cplx;
  const size_t ebytes = (size_t)es * sizeof(double);
  DevIn xin(x0, (size_t)B * n * es, st);
  DevIn cin(consts, consts ? (size_t)B * m * es : 0, st);
  DevBuf xa_all((size_t)B * n * ebytes + 16, st), ca_all(consts ? (size_t)B * m * ebytes + 16 : 16, st);
  if (B) planes_to_aos(es, B * n, xin.d, xa_all.d(), st);
  if (consts && B) planes_to_aos(es, B * m, cin.d, ca_all.d(), st);
  sys->Abuf.ensure((size_t)m * (n + 1) * ebytes);
  sys->fbuf.ensure((size_t)m * ebytes);
  sys->vbuf.ensure((size_t)m * n * ebytes);
  sys->Rbuf.ensure((size_t)(n + 1) * (n + 1) * ebytes);
  sys->xsol.ensure((size_t)2 * n * ebytes);
  double *A = sys->Abuf.d(), *fa = sys->fbuf.d(), *Q = sys->vbuf.d(), *R = sys->Rbuf.d();
  double *dxa = sys->xsol.d(), *xn = dxa + (size_t)n * es;
  DevBuf mod((size_t)2 * n * nc * sizeof(double) + 16, st);
  std::vector<double> hmod((size_t)2 * n * nc);
  const double eps = nc == 1 ? 0x1p-53 : nc == 2 ? 0x1p-104 : 0x1p-209;
  // the per-start constants are written into the system's coefficients;
  // keep the originals and restore them afterwards (no side effect on sys)
  DevBuf saved(consts ? (size_t)m * ebytes + 16 : 16, st);
  if (consts) {
    dispatch_level(nc, cplx, [&]<class E>() {
      k_gather_consts<E><<<(m + 127) / 128, 128, 0, st>>>(m, cpos_d.as<int32_t>(), sys->d_coeff, saved.d());
    });
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
  for (int64_t b = 0; b < B; ++b) {
    double *xb = xa_all.d() + (size_t)b * n * es;
    if (consts) {
      dispatch_level(nc, cplx, [&]<class E>() {
        k_scatter_consts<E><<<(m + 127) / 128, 128, 0, st>>>(m, cpos_d.as<int32_t>(),
                                                             ca_all.d() + (size_t)b * m * es, sys->d_coeff);
      });
      PN_CHECK_LAUNCH();
      count_launch(1);
    }
    int it = 0, stat = 1;
    for (it = 1; it <= max_iters; ++it) {
      evaldiff_device(sys, xb, fa, A, m, n, st);
      mgs_factor_device(nc, cplx, m, n, A, Q, R, sys->mgs, st);
      backsub_device(nc, cplx, n, R, dxa, sys->mgs, st);
      vec_op_aos(nc, cplx, PN_OP_ADD, n, xb, dxa, xn, st);
      vec_op_aos(nc, cplx, PN_OP_MODULUS, n, dxa, nullptr, mod.d(), st);
      vec_op_aos(nc, cplx, PN_OP_MODULUS, n, xn, nullptr, mod.d() + (size_t)n * nc, st);
      const int rc = mgs_read_status(sys->mgs, nullptr, st);
      if (rc) {
        stat = rc == PN_E_BREAKDOWN ? 2 : 3;
        break;
      }
      PN_CHECK_CUDA(cudaMemcpyAsync(xb, xn, (size_t)n * ebytes, cudaMemcpyDeviceToDevice, st));
      PN_CHECK_CUDA(cudaMemcpyAsync(hmod.data(), mod.d(), hmod.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      PN_CHECK_CUDA(cudaStreamSynchronize(st));
      const double dxn = host_inf_norm(hmod, nc, n);
      std::vector<double> xm(hmod.begin() + (size_t)n * nc, hmod.end());
      const double t = tol > 0.0 ? tol : 10.0 * eps * (1.0 + host_inf_norm(xm, nc, n));
      if (dxn <= t) {
        stat = 0;
        break;
      }
    }
    iters[b] = it > max_iters ? max_iters : it;
    status[b] = stat;
  }
  if (consts) {
    dispatch_level(nc, cplx, [&]<class E>() {
      k_scatter_consts<E><<<(m + 127) / 128, 128, 0, st>>>(m, cpos_d.as<int32_t>(), saved.d(), sys->d_coeff);
    });
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
  DevOut xo(x_out, (size_t)B * n * es, st);
  if (B) aos_to_planes(es, B * n, xa_all.d(), xo.d, st);
  xo.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
}


// position of every polynomial's constant monomial in canonical order
static void constant_positions(pn_system *sys, DevBuf &cpos_d, cudaStream_t st) {
  const int m = sys->m;
  std::vector<int32_t> mon_ptr(sys->M + 1), cpos(m, -1);
  PN_CHECK_CUDA(cudaMemcpy(mon_ptr.data(), sys->d_mon_ptr, sizeof(int32_t) * (sys->M + 1), cudaMemcpyDeviceToHost));
  // poly boundaries come from the value segments (seg_ptr[0..m])
  std::vector<int64_t> seg(m + 1);
  PN_CHECK_CUDA(cudaMemcpy(seg.data(), sys->d_seg_ptr, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost));
  for (int i = 0; i < m; ++i) {
    for (int64_t c = seg[i]; c < seg[i + 1]; ++c)
      if (mon_ptr[c + 1] == mon_ptr[c]) {
        PN_REQUIRE(cpos[i] < 0, PN_E_ARG, "polynomial %d has more than one constant term", i);
        cpos[i] = (int32_t)c;
      }
    PN_REQUIRE(cpos[i] >= 0, PN_E_ARG, "per-start constants need a constant term in every polynomial (row %d)", i);
  }
  PN_CHECK_CUDA(cudaMemcpyAsync(cpos_d.p, cpos.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
}

// slots of a batched run: per-slot device state, all strides in doubles
struct BatchSlots {
  int W = 0;
  long long xs = 0, ts = 0, cs = 0, as = 0, qs = 0, rs = 0, ks = 0;
  DevBuf x, dx, table, contrib, A, Q, R, k, flags, list;
};

static long long batch_slot_doubles(const pn_system *sys) {
  const long long es = sys->es, m = sys->m, n = sys->n;
  return (sys->M + sys->nnz) * es + std::max(sys->table_len, 1LL) * es + m * (n + 1) * es + m * n * es +
         (n + 1) * (n + 1) * es + 2 * n * es + m * es;
}

static int batch_width(const pn_system *sys, int64_t B) {
  size_t fr = 0, tot = 0;
  PN_CHECK_CUDA(cudaMemGetInfo(&fr, &tot));
  const double per = (double)batch_slot_doubles(sys) * sizeof(double);
  long long W = std::min<long long>(B, 4LL * num_sms());
  W = std::min<long long>(W, (long long)(0.6 * (double)fr / per));
  if (const char *v = getenv("PN_BATCH_SLOTS")) W = std::min<long long>(B, std::max(1, atoi(v)));
  PN_REQUIRE(W >= 1 || B == 0, PN_E_NOMEM, "not enough device memory for one batch slot (%.0f MB)", per / 1e6);
  return (int)W;
}

static void batch_alloc(pn_system *sys, BatchSlots &s, int W, cudaStream_t st) {
  const long long es = sys->es, m = sys->m, n = sys->n;
  s.W = W;
  s.xs = n * es;
  s.ts = std::max(sys->table_len, 1LL) * es;
  s.cs = (sys->M + sys->nnz) * es;
  s.as = m * (n + 1) * es;
  s.qs = m * n * es;
  s.rs = (n + 1) * (n + 1) * es;
  s.ks = m * es;
  auto mk = [&](DevBuf &b, long long per) { b = DevBuf((size_t)W * per * sizeof(double) + 16, st); };
  mk(s.x, s.xs);
  mk(s.dx, s.xs);
  mk(s.table, s.ts);
  mk(s.contrib, s.cs);
  mk(s.A, s.as);
  mk(s.Q, s.qs);
  mk(s.R, s.rs);
  mk(s.k, s.ks);
  s.flags = DevBuf((size_t)W * sizeof(int32_t) + 16, st);
  s.list = DevBuf((size_t)W * sizeof(int32_t) + 16, st);
}

// Batched runs: W slots hold W starts at a time.  Every iteration evaluates
// all busy slots in one pass of the evaluation kernels (blockIdx.y = slot)
// and solves them with one k_solve_batch launch (one CTA per start); the
// host then retires converged / failed / exhausted starts and refills their
// slots from the queue, so the GPU stays full until the queue drains.
extern "C" int pn_newton_batch(pn_system *sys, int64_t B, const double *x0, const double *consts, int max_iters,
                               double tol, double *x_out, int32_t *iters, int32_t *status, void *stream) {
  PN_API_BEGIN
  NvtxRange range("pn_newton_batch");
  PN_REQUIRE(sys && x0 && x_out && iters && status && B >= 0 && max_iters >= 1, PN_E_ARG,
             "pn_newton_batch: bad arguments");
  const int m = sys->m, n = sys->n, es = sys->es;
  PN_REQUIRE(m >= n && n >= 1, PN_E_ARG, "need m >= n >= 1, got m=%d, n=%d", m, n);
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf cpos_d(sizeof(int32_t) * (m + 1), st);
  if (consts) constant_positions(sys, cpos_d, st);
  const char *mode = getenv("PN_BATCH_MODE");
  if ((mode && strcmp(mode, "serial") == 0) || m > 1024) {
    newton_batch_serial(sys, B, x0, consts, max_iters, tol, x_out, iters, status, st, cpos_d);
    return PN_OK;
  }
  const size_t ebytes = (size_t)es * sizeof(double);
  DevIn xin(x0, (size_t)B * n * es, st);
  DevIn cin(consts, consts ? (size_t)B * m * es : 0, st);
  DevBuf xa_all((size_t)B * n * ebytes + 16, st), ca_all(consts ? (size_t)B * m * ebytes + 16 : 16, st);
  if (B) planes_to_aos(es, B * n, xin.d, xa_all.d(), st);
  if (consts && B) planes_to_aos(es, B * m, cin.d, ca_all.d(), st);
  const int W = B ? batch_width(sys, B) : 0;
  BatchSlots s;
  if (W) batch_alloc(sys, s, W, st);
  // Slot groups on their own streams: while the host retires and refills one
  // group, the other groups' kernels run, and one group's evaluation (HBM
  // and latency heavy) overlaps another's FP64-bound solve.
  constexpr int MAXG = 4;
  int NG = 4;  // C5 2048 starts: 3848 / 3984 / 4040 / 4051 start-iter/s for 1..4 groups
  if (const char *v = getenv("PN_BATCH_GROUPS")) NG = std::max(1, std::min(MAXG, atoi(v)));
  NG = std::max(1, std::min(NG, W));
  int gsplit[MAXG + 1];
  for (int g = 0; g <= NG; ++g) gsplit[g] = (int)((long long)W * g / NG);
  cudaStream_t gs[MAXG] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ready_ev = nullptr;
  struct StreamGuard {
    cudaStream_t *s;
    cudaEvent_t *e;
    ~StreamGuard() {
      for (int g = 0; g < MAXG; ++g)
        if (s[g]) cudaStreamDestroy(s[g]);
      if (*e) cudaEventDestroy(*e);
    }
  } guard{gs, &ready_ev};
  PN_CHECK_CUDA(cudaEventCreateWithFlags(&ready_ev, cudaEventDisableTiming));
  PN_CHECK_CUDA(cudaEventRecord(ready_ev, st));
  for (int g = 0; g < NG; ++g) {
    PN_CHECK_CUDA(cudaStreamCreateWithFlags(&gs[g], cudaStreamNonBlocking));
    PN_CHECK_CUDA(cudaStreamWaitEvent(gs[g], ready_ev, 0));
  }
  std::vector<int64_t> owner(W, -1);
  std::vector<int32_t> it((size_t)B, 0);
  // pinned host buffers, so the per-group copies stay asynchronous
  int32_t *hbuf = nullptr;
  PN_CHECK_CUDA(cudaMallocHost(&hbuf, sizeof(int32_t) * (2 * (size_t)W + 2)));
  struct HostGuard {
    int32_t *p;
    ~HostGuard() { cudaFreeHost(p); }
  } hguard{hbuf};
  int32_t *flags = hbuf, *hlist = hbuf + W + 1;
  std::vector<int32_t> list[MAXG];
  bool pending[MAXG] = {false, false, false, false};
  int64_t next = 0;
  auto load = [&](int slot, cudaStream_t sg) {
    if (next >= B) {
      owner[slot] = -1;
      return;
    }
    const int64_t b = next++;
    owner[slot] = b;
    PN_CHECK_CUDA(cudaMemcpyAsync(s.x.d() + slot * s.xs, xa_all.d() + b * n * es, n * ebytes,
                                  cudaMemcpyDeviceToDevice, sg));
    if (consts)
      PN_CHECK_CUDA(cudaMemcpyAsync(s.k.d() + slot * s.ks, ca_all.d() + b * m * es, m * ebytes,
                                    cudaMemcpyDeviceToDevice, sg));
  };
  for (int g = 0; g < NG; ++g)
    for (int w = gsplit[g]; w < gsplit[g + 1]; ++w) load(w, gs[g]);
  // retire finished starts of group g (its stream is synchronised)
  auto retire = [&](int g) {
    for (int w : list[g]) {
      const int64_t b = owner[w];
      const int f = flags[w];
      ++it[b];
      int stat = -1;
      if (f == 1) stat = 0;
      else if (f == 2) stat = 2;
      else if (f == 3) stat = 3;
      else if (it[b] >= max_iters) stat = 1;
      if (stat < 0) continue;
      iters[b] = it[b];
      status[b] = stat;
      PN_CHECK_CUDA(cudaMemcpyAsync(xa_all.d() + b * n * es, s.x.d() + w * s.xs, n * ebytes,
                                    cudaMemcpyDeviceToDevice, gs[g]));
      load(w, gs[g]);
    }
  };
  while (true) {
    bool any = false;
    for (int g = 0; g < NG; ++g) {
      if (pending[g]) {
        PN_CHECK_CUDA(cudaStreamSynchronize(gs[g]));
        pending[g] = false;
        retire(g);
      }
      list[g].clear();
      for (int w = gsplit[g]; w < gsplit[g + 1]; ++w)
        if (owner[w] >= 0) list[g].push_back(w);
      if (list[g].empty()) continue;
      any = true;
      const int nb = (int)list[g].size();
      int32_t *sl = s.list.as<int32_t>() + gsplit[g];
      std::copy(list[g].begin(), list[g].end(), hlist + gsplit[g]);
      PN_CHECK_CUDA(cudaMemcpyAsync(sl, hlist + gsplit[g], sizeof(int32_t) * nb, cudaMemcpyHostToDevice, gs[g]));
      const BView bv{sl, s.xs, s.ts, s.cs, s.as, 0};
      dispatch_level(sys->nc, sys->cplx, [&]<class E>() {
        evaldiff_batch_impl<E>(sys, nb, bv, s.x.d(), s.table.d(), s.contrib.d(), nullptr, s.A.d(), n,
                               cpos_d.as<int32_t>(), consts ? s.k.d() : nullptr, s.ks, gs[g]);
        solve_batch_impl<E>(nb, sl, m, n, s.A.d(), s.as, s.Q.d(), s.qs, s.R.d(), s.rs, s.x.d(), s.xs, s.dx.d(),
                            tol, s.flags.as<int32_t>(), gs[g]);
      });
      PN_CHECK_CUDA(cudaMemcpyAsync(flags + gsplit[g], s.flags.as<int32_t>() + gsplit[g],
                                    sizeof(int32_t) * (gsplit[g + 1] - gsplit[g]), cudaMemcpyDeviceToHost, gs[g]));
      pending[g] = true;
    }
    if (!any) break;
  }
  for (int g = 0; g < NG; ++g) {
    PN_CHECK_CUDA(cudaEventRecord(ready_ev, gs[g]));
    PN_CHECK_CUDA(cudaStreamWaitEvent(st, ready_ev, 0));
  }
  DevOut xo(x_out, (size_t)B * n * es, st);
  if (B) aos_to_planes(es, B * n, xa_all.d(), xo.d, st);
  xo.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}

// values f(x_b) of a batch of points (planes (cshape, B, n) -> (cshape, B, m)),
// evaluated W points at a time through the batched evaluation kernels
extern "C" int pn_evaldiff_batch(pn_system *sys, int64_t B, const double *x, double *f, void *stream) {
  PN_API_BEGIN
  PN_REQUIRE(sys && x && f && B >= 0, PN_E_ARG, "pn_evaldiff_batch: bad arguments");
  const int m = sys->m, n = sys->n, es = sys->es;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t ebytes = (size_t)es * sizeof(double);
  DevIn xin(x, (size_t)B * n * es, st);
  DevBuf xa((size_t)B * n * ebytes + 16, st), fa((size_t)B * m * ebytes + 16, st);
  if (B) planes_to_aos(es, B * n, xin.d, xa.d(), st);
  const int W = B ? batch_width(sys, B) : 0;
  if (W) {
    const long long ts = std::max(sys->table_len, 1LL) * es, cs = (sys->M + sys->nnz) * es;
    const long long as = (long long)std::max(m, 1) * (n + 1) * es;
    DevBuf table((size_t)W * ts * sizeof(double) + 16, st), contrib((size_t)W * cs * sizeof(double) + 16, st);
    DevBuf A((size_t)W * as * sizeof(double) + 16, st);
    for (int64_t b0 = 0; b0 < B; b0 += W) {
      const int nb = (int)std::min<int64_t>(W, B - b0);
      const BView bv{nullptr, (long long)n * es, ts, cs, as, (long long)m * es};
      dispatch_level(sys->nc, sys->cplx, [&]<class E>() {
        evaldiff_batch_impl<E>(sys, nb, bv, xa.d() + b0 * n * es, table.d(), contrib.d(), fa.d() + b0 * m * es,
                               A.d(), -1, nullptr, nullptr, 0, st);
      });
    }
  }
  DevOut fo(f, (size_t)B * m * es, st);
  if (B) aos_to_planes(es, B * m, fa.d(), fo.d, st);
  fo.finish(st);
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}
