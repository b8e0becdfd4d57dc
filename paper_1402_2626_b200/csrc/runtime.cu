// runtime.cu -- error plumbing, memory staging, layout conversion and the
// element-wise VecContext kernels (varith.py:104-191).
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <new>

#include "common.cuh"
#include "internal.h"

namespace pn {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// keep freed stream-ordered memory in the device pool instead of returning
// it at every synchronisation: batched runs allocate tens of GB of slots per
// call, and re-mapping them each time costs more than a Newton iteration
static void keep_pool_memory() {
  static const bool done = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    return true;
  }();
  (void)done;
}

DevBuf::DevBuf(size_t nbytes, cudaStream_t st) : bytes(nbytes), s(st) {
  keep_pool_memory();
  if (nbytes) PN_CHECK_CUDA(cudaMallocAsync(&p, nbytes, st));
}
DevBuf::~DevBuf() {
  if (p) cudaFreeAsync(p, s);
}

void DevArena::ensure(size_t nbytes) {
  if (nbytes <= bytes) return;
  if (p) {
    cudaDeviceSynchronize();
    cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t e = cudaMalloc(&p, nbytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed: %s", nbytes, cudaGetErrorString(e));
    throw Fail{PN_E_NOMEM};
  }
  bytes = nbytes;
}
DevArena::~DevArena() {
  if (p) cudaFree(p);
}

DevIn::DevIn(const double *src, size_t ndoubles, cudaStream_t st) {
  if (!src || is_device_ptr(src)) {
    d = src;
    return;
  }
  DevBuf b(ndoubles * sizeof(double), st);
  if (ndoubles) PN_CHECK_CUDA(cudaMemcpyAsync(b.p, src, ndoubles * sizeof(double), cudaMemcpyHostToDevice, st));
  d = b.d();
  own = std::move(b);
}

DevOut::DevOut(double *dst, size_t ndoubles, cudaStream_t st) : n(ndoubles) {
  if (!dst) return;
  if (is_device_ptr(dst)) {
    d = dst;
    return;
  }
  host = dst;
  DevBuf b(ndoubles * sizeof(double), st);
  d = b.d();
  own = std::move(b);
}
void DevOut::finish(cudaStream_t st) {
  if (host && n) PN_CHECK_CUDA(cudaMemcpyAsync(host, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
}

// ---------------------------------------------------------------------------
// layout conversion

__global__ void k_planes_to_aos_cm(int es, int rows, int cols, const double *__restrict__ src,
                                   double *__restrict__ dst, long long ld) {
  const long long total = (long long)rows * cols;
  const long long plane = total;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;  // source is row-major
    double *o = dst + (j * ld + i) * es;
    for (int p = 0; p < es; ++p) o[p] = src[p * plane + e];
  }
}

__global__ void k_aos_cm_to_planes(int es, int rows, int cols, const double *__restrict__ src, long long ld,
                                   double *__restrict__ dst) {
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;
    const double *s = src + (j * ld + i) * es;
    for (int p = 0; p < es; ++p) dst[p * total + e] = s[p];
  }
}

static int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = (long long)num_sms() * 32;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

void planes_to_aos_colmajor(int es, int rows, int cols, const double *src, double *dst, long long ld,
                            cudaStream_t st) {
  long long total = (long long)rows * cols;
  if (!total) return;
  k_planes_to_aos_cm<<<grid_for(total, 256), 256, 0, st>>>(es, rows, cols, src, dst, ld);
  PN_CHECK_LAUNCH();
  count_launch(1);
}

void aos_colmajor_to_planes(int es, int rows, int cols, const double *src, long long ld, double *dst,
                            cudaStream_t st) {
  long long total = (long long)rows * cols;
  if (!total) return;
  k_aos_cm_to_planes<<<grid_for(total, 256), 256, 0, st>>>(es, rows, cols, src, ld, dst);
  PN_CHECK_LAUNCH();
  count_launch(1);
}

// a 1-D array is a (n x 1) matrix: row-major index i; column-major ld = n
void planes_to_aos(int es, long long n, const double *src, double *dst, cudaStream_t st) {
  planes_to_aos_colmajor(es, (int)n, 1, src, dst, n, st);
}
void aos_to_planes(int es, long long n, const double *src, double *dst, cudaStream_t st) {
  aos_colmajor_to_planes(es, (int)n, 1, src, n, dst, st);
}

// ---------------------------------------------------------------------------
// element-wise ops (VecContext), on planes or AoS

template <class E, bool PLANES>
__global__ void k_vec_op(int op, long long n, const double *__restrict__ a, const double *__restrict__ b,
                         double *__restrict__ out) {
  using R = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    E x = PLANES ? eload_planes<E>(a, n, i) : eload<E>(a + i * es);
    switch (op) {
      case PN_OP_ADD:
      case PN_OP_SUB:
      case PN_OP_MUL:
      case PN_OP_DIV: {
        E y = PLANES ? eload_planes<E>(b, n, i) : eload<E>(b + i * es);
        E z = op == PN_OP_ADD ? eadd(x, y) : op == PN_OP_SUB ? esub(x, y) : op == PN_OP_MUL ? emul(x, y) : ediv(x, y);
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * es, z);
        break;
      }
      case PN_OP_DIV_REAL: {
        R r = PLANES ? eload_planes<R>(b, n, i) : eload<R>(b + i * Traits<R>::es);
        E z = ediv_real(x, r);
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * es, z);
        break;
      }
      case PN_OP_CONJ: {
        E z = econj(x);
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * es, z);
        break;
      }
      case PN_OP_ABS2: {
        R z = eabs2(x);
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * Traits<R>::es, z);
        break;
      }
      case PN_OP_SQRT: {
        // input is a real element: reinterpret the leading nc components
        R r = PLANES ? eload_planes<R>(a, n, i) : eload<R>(a + i * Traits<R>::es);
        R z = fsqrt(r);
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * Traits<R>::es, z);
        break;
      }
      case PN_OP_MODULUS: {
        // xprec.modulus: complex -> sqrt(re*re + im*im) (xprec.py:327-328,
        // 348-354); real -> abs (xprec.py:121-122, 231-232)
        R z;
        if constexpr (Traits<E>::cplx) {
          z = fsqrt(eabs2(x));
        } else {
          z = (ehi(x) < 0.0) ? fneg(x) : x;
        }
        if (PLANES) estore_planes(out, n, i, z); else estore(out + i * Traits<R>::es, z);
        break;
      }
      default:
        break;
    }
  }
}

template <bool PLANES>
static void launch_vec_op(int nc, int cplx, int op, long long n, const double *a, const double *b, double *out,
                          cudaStream_t st) {
  if (n <= 0) return;
  const int threads = 128;
  const int grid = grid_for(n, threads);
  dispatch_level(nc, cplx, [&]<class E>() {
    if (op == PN_OP_SQRT) {
      // sqrt operates on real planes regardless of the level's cplx flag
      using R = typename Traits<E>::R;
      k_vec_op<R, PLANES><<<grid, threads, 0, st>>>(op, n, a, b, out);
    } else {
      k_vec_op<E, PLANES><<<grid, threads, 0, st>>>(op, n, a, b, out);
    }
  });
  PN_CHECK_LAUNCH();
  count_launch(1);
}

void vec_op_aos(int nc, int cplx, int op, long long n, const double *a, const double *b, double *out,
                cudaStream_t st) {
  launch_vec_op<false>(nc, cplx, op, n, a, b, out, st);
}

// ---------------------------------------------------------------------------
// tree_sum over one axis (varith.py:169-191) with a single CTA: thread t
// folds the aligned block [t*B, t*B+B) sequentially (pairwise), then the
// block partials are combined by block_tree_reduce.  Large n loops over
// chunks of NT*B elements, which are themselves aligned blocks, and the chunk
// partials are combined with the same stride-doubling rule.
template <class E, int NT>
__global__ void k_tree_sum(long long n, const double *__restrict__ a, double *__restrict__ out) {
  __shared__ E sm[NT / 32];
  // chunk partials are kept in a binary-counter stack (right-pruned tree)
  E stack[40];
  const long long per = (n + NT - 1) / NT;
  long long B = 1;
  while (B < per) B <<= 1;
  if (B > (1ll << 20)) B = 1ll << 20;
  const long long chunk = B * NT;
  const long long nchunks = (n + chunk - 1) / chunk;
  for (long long c = 0; c < nchunks; ++c) {
    const long long base = c * chunk + threadIdx.x * B;
    // sequential binary-counter fold of this thread's aligned block
    E st[40];
    long long cnt = 0;
    for (long long q = 0; q < B && base + q < n; ++q) {
      E carry = eload_planes<E>(a, n, base + q);
      int lvl = 0;
      for (long long p = cnt; p & 1; p >>= 1, ++lvl) carry = eadd(st[lvl], carry);
      st[lvl] = carry;
      ++cnt;
    }
    E part = ezero<E>();
    if (cnt > 0) {
      int lo = __ffsll(cnt) - 1;
      part = st[lo];
      for (int l = lo + 1; l < 63; ++l)
        if ((cnt >> l) & 1) part = eadd(st[l], part);
    }
    const long long rem = n - c * chunk;
    const int nparts = (int)((rem + B - 1) / B < NT ? (rem + B - 1) / B : NT);
    E cp = block_tree_reduce<E, NT>(part, nparts, sm);
    if (threadIdx.x == 0) {
      int lvl = 0;
      for (long long p = c; p & 1; p >>= 1, ++lvl) cp = eadd(stack[lvl], cp);
      stack[lvl] = cp;
    }
  }
  if (threadIdx.x == 0) {
    E r = ezero<E>();
    if (nchunks > 0) {
      int lo = __ffsll(nchunks) - 1;
      r = stack[lo];
      for (int l = lo + 1; l < 63; ++l)
        if ((nchunks >> l) & 1) r = eadd(stack[l], r);
    }
    estore_planes(out, 1, 0, r);
  }
}

// FP64 pipe throughput probe: every thread runs 8 independent DFMA chains;
// one DFMA is counted as one FP64 instruction (the unit of the roofline's
// work counts).  The result is written so the chains cannot be elided.
__global__ void __launch_bounds__(256) k_fp64_probe(int iters, double seed, double *out) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

}  // namespace pn

using namespace pn;

extern "C" int pn_fp64_peak(double *instr_per_s, void *stream) {
  PN_API_BEGIN
  PN_REQUIRE(instr_per_s, PN_E_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf sink(64, st);
  const int iters = 1 << 14, threads = 256, blocks = num_sms() * 8;
  cudaEvent_t e0, e1;
  PN_CHECK_CUDA(cudaEventCreate(&e0));
  PN_CHECK_CUDA(cudaEventCreate(&e1));
  k_fp64_probe<<<blocks, threads, 0, st>>>(iters / 8, 1.0, sink.d());  // warm-up
  PN_CHECK_CUDA(cudaEventRecord(e0, st));
  k_fp64_probe<<<blocks, threads, 0, st>>>(iters, 1.0, sink.d());
  PN_CHECK_CUDA(cudaEventRecord(e1, st));
  PN_CHECK_LAUNCH();
  count_launch(2);
  PN_CHECK_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  PN_CHECK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *instr_per_s = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
  PN_API_END
}

extern "C" {

int pn_version(void) { return 100; }

const char *pn_last_error(void) { return g_err; }

int pn_device_count(int *count) {
  PN_API_BEGIN
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  if (count) *count = c;
  PN_API_END
}

int64_t pn_launch_count(void) { return g_launches.load(); }

int pn_vec_op(int nc, int cplx, int op, int64_t n, const double *a, const double *b, double *out, void *stream) {
  PN_API_BEGIN
  check_level(nc, cplx);
  PN_REQUIRE(n >= 0 && a && out, PN_E_ARG, "pn_vec_op: bad arguments");
  PN_REQUIRE(op >= 0 && op <= PN_OP_DIV_REAL, PN_E_ARG, "pn_vec_op: unknown op %d", op);
  const bool binary = op == PN_OP_ADD || op == PN_OP_SUB || op == PN_OP_MUL || op == PN_OP_DIV || op == PN_OP_DIV_REAL;
  PN_REQUIRE(!binary || b, PN_E_ARG, "pn_vec_op: op %d needs a second operand", op);
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  const int in_es = (op == PN_OP_SQRT) ? nc : es;
  const int b_es = (op == PN_OP_DIV_REAL) ? nc : es;
  const int out_es = (op == PN_OP_ABS2 || op == PN_OP_SQRT || op == PN_OP_MODULUS) ? nc : es;
  DevIn da(a, (size_t)n * in_es, st);
  DevIn db(binary ? b : nullptr, binary ? (size_t)n * b_es : 0, st);
  DevOut dout(out, (size_t)n * out_es, st);
  launch_vec_op<true>(nc, cplx, op, n, da.d, db.d, dout.d, st);
  dout.finish(st);
  if (dout.host) PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}

int pn_tree_sum(int nc, int cplx, int64_t n, const double *a, double *out, void *stream) {
  PN_API_BEGIN
  check_level(nc, cplx);
  PN_REQUIRE(n >= 1 && a && out, PN_E_ARG, "pn_tree_sum: need n >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1);
  DevIn da(a, (size_t)n * es, st);
  DevOut dout(out, (size_t)es, st);
  dispatch_level(nc, cplx, [&]<class E>() { k_tree_sum<E, 256><<<1, 256, 0, st>>>(n, da.d, dout.d); });
  PN_CHECK_LAUNCH();
  count_launch(1);
  dout.finish(st);
  if (dout.host) PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}

}  // extern "C"
