// internal.h -- declarations shared by the translation units of
// libpolynewt_b200.so (not part of the public C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../include/polynewt_b200.h"

namespace pn {

// batch view of the evaluation kernels: slot b = slots[blockIdx.y] (or
// blockIdx.y) works on x + b*x, table + b*t, contrib + b*c, A + b*a, f + b*f
// (strides in doubles)
struct BView {
  const int32_t *slots;
  long long x, t, c, a, f;
};

void set_error(const char *fmt, ...);
void count_launch(int n);

// ---------------------------------------------------------------------------
// device memory helpers

bool is_device_ptr(const void *p);

// stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync)
struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t nbytes, cudaStream_t st);
  ~DevBuf();
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; }
  DevBuf &operator=(DevBuf &&o) noexcept {
    if (this != &o) {
      if (p) cudaFreeAsync(p, s);
      p = o.p;
      bytes = o.bytes;
      s = o.s;
      o.p = nullptr;
    }
    return *this;
  }
  double *d() const { return static_cast<double *>(p); }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

// persistent device allocation (cudaMalloc), grown on demand
struct DevArena {
  void *p = nullptr;
  size_t bytes = 0;
  void ensure(size_t nbytes);
  ~DevArena();
  double *d() const { return static_cast<double *>(p); }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

// read-only input on the device: either the caller's device pointer or a
// staged copy of a host buffer
struct DevIn {
  const double *d = nullptr;
  DevBuf own;
  DevIn(const double *src, size_t ndoubles, cudaStream_t st);
};

// output: device pointer of the caller or a scratch buffer copied back by finish()
struct DevOut {
  double *d = nullptr;
  double *host = nullptr;
  size_t n = 0;
  DevBuf own;
  DevOut(double *dst, size_t ndoubles, cudaStream_t st);
  void finish(cudaStream_t st);  // enqueue D2H copy if host
};

// ---------------------------------------------------------------------------
// layout conversion (component planes <-> AoS elements)

// planes (es, rows, cols) row-major  ->  AoS column-major with leading dim ld
void planes_to_aos_colmajor(int es, int rows, int cols, const double *src, double *dst, long long ld,
                            cudaStream_t st);
// AoS column-major (ld)  ->  planes (es, rows, cols) row-major
void aos_colmajor_to_planes(int es, int rows, int cols, const double *src, long long ld, double *dst,
                            cudaStream_t st);
// 1-D: planes (es, n) <-> AoS (n, es)
void planes_to_aos(int es, long long n, const double *src, double *dst, cudaStream_t st);
void aos_to_planes(int es, long long n, const double *src, double *dst, cudaStream_t st);

// element-wise op on AoS arrays (used inside the Newton step)
void vec_op_aos(int nc, int cplx, int op, long long n, const double *a, const double *b, double *out,
                cudaStream_t st);

// ---------------------------------------------------------------------------
// MGS least squares on a device-resident augmented matrix
//   A : AoS column-major (m rows, n+1 cols, ld = m), overwritten
//   Q : AoS column-major (m, n) or NULL
//   R : AoS column-major ((n+1) x (n+1), ld = n+1), zero-initialised here
// status (device int[4]) + info (device double[4]) receive the breakdown
// record; the call enqueues work on st and returns without synchronising.
constexpr int kMgsThreads = 256;     // CTA size of the MGS sweeps
constexpr int kBacksubThreads = 256;  // CTA size of back substitution (n <= 4 * this)
inline int rows_per_thread(int m) {
  int per = (m + kMgsThreads - 1) / kMgsThreads, B = 1;
  while (B < per) B <<= 1;
  return B;
}
struct MgsStatus {
  int code;  // 0 ok, PN_E_BREAKDOWN, PN_E_SINGULAR
  int k;
  double rkk, thr;
};
struct MgsWork {
  DevArena qbuf;    // normalized pivot columns when Q is not requested
  DevArena orig;    // orig column norms (hi)
  DevArena status;  // MgsStatus
  DevArena ready;   // dataflow schedule: pivot-published flags (n+1 ints)
  DevArena own;     // flow schedule: column ownership table (G x maxo ints)
  long long own_key = -1;
  int own_maxo = 0;
};
void mgs_factor_device(int nc, int cplx, int m, int n, double *A, double *Q, double *R, MgsWork &w,
                       cudaStream_t st);
// back substitution on the device-resident R (column-major, ld = n+1); x AoS
void backsub_device(int nc, int cplx, int n, const double *R, double *x, MgsWork &w, cudaStream_t st);
// read the status record written by mgs/backsub; returns PN_OK / PN_E_BREAKDOWN / PN_E_SINGULAR
int mgs_read_status(MgsWork &w, pn_numinfo *info, cudaStream_t st);

// k_eval_rows geometry: CTA size and lanes per monomial (chunk = NT / G
// monomials).  Plain double: 8 lanes per monomial so 1024 threads fit the
// register file (twice the warps to hide the stack pushes' latency).
__host__ __device__ constexpr int rows_nt(int nc) { return nc == 1 ? 1024 : 512; }
__host__ __device__ constexpr int rows_g(int nc, bool cplx, int base) {
  return (nc == 1 || nc == 4 || (nc == 2 && cplx) ? 8 : 4) < base ? (nc == 1 || nc == 4 || (nc == 2 && cplx) ? 8 : 4)
                                                                     : base;
}

// shared-memory carve-up of k_eval_rows (byte offsets, 16-byte aligned),
// shared by the plan (system.cu) and the kernel (evaldiff.cu)
constexpr size_t kRowsSmemMax = 226 * 1024;
struct RowsLayout {
  static constexpr int VL = 24;  // value-stack levels
  static constexpr __host__ __device__ int le(int CH, int K) { return CH * K + 8; }  // staged entries per buffer
  size_t xs, stk, buf, vals, wpart, vstk, cnt, sent, smp, scf, sro, pad, total;
  int lmp, lcf, rs;  // per-buffer lengths: mon_ptr ints, coefficient doubles, run starts (uint16)
};
__host__ __device__ inline RowsLayout rows_layout(int n, int D, int K, int es, int CH, int BASE, int NW, bool xsm) {
  RowsLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 15) & ~(size_t)15;
    return at;
  };
  const size_t eb = (size_t)es * 8;
  L.xs = take(xsm ? (size_t)n * eb : 0);
  L.stk = take((size_t)D * n * eb);
  L.buf = take((size_t)CH * K * eb);
  L.vals = take((size_t)CH * eb);
  L.wpart = take((size_t)NW * eb);
  L.vstk = take((size_t)RowsLayout::VL * eb);
  L.cnt = take((size_t)n * 4);
  L.sent = take((size_t)2 * RowsLayout::le(CH, K) * 4);
  L.lmp = CH + 8;
  L.lcf = ((CH + 1) * es + 3) & ~1;
  L.rs = (n + 1 + 7) & ~7;
  L.smp = take((size_t)2 * L.lmp * 4);
  L.scf = take((size_t)2 * L.lcf * 8);
  L.sro = take((size_t)2 * L.rs * 2);
  L.pad = take((size_t)2 * BASE * 4);
  L.total = o;
  return L;
}

}  // namespace pn

// ---------------------------------------------------------------------------
// the packed, device-resident system (evaldiff.py:183-194 PreparedSystem)
struct pn_system {
  int nc = 0, cplx = 0, es = 0;
  int m = 0, n = 0;
  long long M = 0, nnz = 0;
  long long nseg = 0;  // Jacobian segments (nonzero entries)
  int max_k = 0, max_deg = 0;
  std::vector<long long> perm;  // canonical position -> input monomial
  pn_counts counts{};
  pn_system_stats stats{};

  // device arrays (canonical order)
  int32_t *d_mon_ptr = nullptr;  // M+1
  int32_t *d_var = nullptr;      // nnz
  int32_t *d_exp = nullptr;      // nnz
  int32_t *d_dst = nullptr;      // nnz: contribution slot of each support entry
  double *d_coeff = nullptr;     // M * es (AoS)
  int32_t *d_toff = nullptr;     // n: power-table row offset per variable
  int32_t *d_tdeg = nullptr;     // n: max exponent per variable (0 = absent)
  int64_t *d_seg_ptr = nullptr;  // m + nseg + 1 segment starts in the contribution buffer
  int64_t *d_seg_out = nullptr;  // nseg: output index (column-major j*m + i) of J segments
  long long table_len = 0;

  // monomial buckets by kind, device lists of canonical monomial indices
  struct Bucket {
    int kind;        // 0: k<=1, 1: tree with BASE=base, 2: large tree
    int base;
    long long count;
    int32_t *d_list;
    // dense uniform bucket: every monomial has k = dense_k and the bucket's
    // support entries are the contiguous block [e0, e0 + count*dense_k)
    // (lets k_mono_tree_tma stage whole chunks with bulk copies); 0 if not
    int dense_k = 0;
    long long e0 = 0;
    bool unit_exp = false;  // dense bucket whose exponents are all 1
  };
  std::vector<Bucket> buckets;


  // plan of the row evaluation (k_eval_rows): one CTA per polynomial at a
  // time, chunks of CH canonical monomials, per-variable binary-counter
  // stacks of depth D in shared memory.  Applies when every non-constant
  // monomial has the same k = K (2..32), n <= 65536, exponents <= 15 and the
  // stacks fit.
  struct Rows {
    bool ok = false;
    int K = 0, base = 0, CH = 0, D = 0;
    long long nchunks = 0;
    bool unit = false;             // every exponent is 1
    uint32_t *d_ent = nullptr;     // nnz: var | (slot in the chunk buffer) << 16 | exponent << 28
    int32_t *d_poly_chunk = nullptr;  // m + 1: first chunk of each polynomial
    int4 *d_desc = nullptr;        // nchunks: {first monomial, monomials, first entry, end entry}
    uint16_t *d_runoff = nullptr;  // nchunks * rs (rs = n + 1 rounded up to 8): start of variable j's run
  } rows;

  // scratch reused across evaluations
  pn::DevArena contrib;  // (M + nnz) * es
  pn::DevArena table;    // table_len * es
  pn::DevArena tree_scratch;  // k_mono_large levels when 3*base elements exceed shared memory
  pn::DevArena xbuf;     // n * es
  pn::DevArena Abuf;     // m * (n+1) * es (Newton / evaldiff output)
  pn::DevArena Rbuf, xsol, fbuf, vbuf;
  pn::MgsWork mgs;
  cudaEvent_t ev = nullptr;

  // CUDA graph of the device part of pn_newton_step (evaluation,
  // factorisation, back substitution, update) for small systems, where the
  // step is launch-bound: captured after the first direct step, replayed
  // afterwards.  graph_state: 0 not tried, 1 captured, -1 capture refused
  cudaGraphExec_t step_graph = nullptr;
  cudaStream_t graph_stream = nullptr;
  cudaEvent_t gev[5] = {};
  cudaEvent_t pev[5] = {};  // phase events of the direct (non-graph) step
  long long graph_launches = 0;  // kernels inside the graph (launch counter)
  int graph_state = 0;

  ~pn_system();
};

namespace pn {
// evaluate at x (AoS, device) into f (AoS, device, may be NULL) and the
// Jacobian, written column-major with leading dimension ldA into A (zeroed
// entries included).  If negf_col >= 0, -f is additionally written into
// column negf_col of A (the b column of [J -f]).
void evaldiff_device(pn_system *sys, const double *x, double *f, double *A, long long ldA, int negf_col,
                     cudaStream_t st);

// per-level implementations (explicitly instantiated in one TU per level)
template <class E>
void evaldiff_impl(pn_system *sys, const double *x, double *f, double *A, long long ldA, int negf_col,
                   cudaStream_t st);
template <class E>
void evaldiff_batch_impl(pn_system *sys, int nb, const BView &bv, const double *x, double *table, double *contrib,
                         double *f, double *A, int negf_col, const int32_t *cpos, const double *consts,
                         long long cstride, cudaStream_t st);
template <class E>
void solve_batch_impl(int nb, const int32_t *slots, int m, int n, double *A, long long As, double *Q, long long Qs,
                      double *R, long long Rs, double *x, long long xs, double *dx, double tol, int32_t *flags,
                      cudaStream_t st);
template <class E>
double residual_impl(int m, int n, const double *A, const double *Q, const double *R, cudaStream_t st);
template <class E>
void mgs_impl(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st);
template <class E>
void backsub_impl(int n, const double *R, double *x, MgsWork &w, cudaStream_t st);
}  // namespace pn
