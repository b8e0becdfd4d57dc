// comm.cu -- the one collective of the batched path in the C ABI: an NCCL
// communicator and the all-gather of a sharded batch's results (status,
// iteration counts, final x of every start), so a non-torch host can run
// config C5 over several GPUs through this library alone (SURVEY 8(b)
// pn_comm_*, 8(e)).  The reference runs its starts one process at a time
// (newton.py:106-159); here each rank solves the contiguous block of starts
// shard_range assigns it and this gather is the only communication.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy
// already mapped by the process -- e.g. PyTorch's -- when there is one), so
// the library has no link-time NCCL dependency and cannot pull a second
// NCCL into a process that already has one.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[PN_COMM_ID_BYTES];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0 };

struct Nccl {
  void *h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
};

Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
    n.getErrorString = (decltype(n.getErrorString))dlsym(h, "ncclGetErrorString");
    if (n.getUniqueId && n.commInitRank && n.commDestroy && n.allGather) n.h = h;
  });
  if (!n.h) {
    pn::set_error("NCCL (libnccl.so.2) is not available");
    throw pn::Fail{PN_E_COMM};
  }
  return n;
}

#define PN_CHECK_NCCL(expr)                                                                           \
  do {                                                                                                \
    const ncclResult_t r_ = (expr);                                                                   \
    if (r_ != 0) {                                                                                    \
      pn::set_error("NCCL error %d (%s) at %s:%d", r_, nccl().getErrorString ? nccl().getErrorString(r_) : "", \
                    __FILE__, __LINE__);                                                              \
      throw pn::Fail{PN_E_COMM};                                                                      \
    }                                                                                                 \
  } while (0)

// batch.shard_range: contiguous, balanced blocks of starts
void shard_range(int64_t B, int world, int rank, int64_t &lo, int64_t &hi) {
  const int64_t base = B / world, extra = B % world;
  lo = rank * base + std::min<int64_t>(rank, extra);
  hi = lo + base + (rank < extra ? 1 : 0);
}

}  // namespace

struct pn_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

extern "C" int pn_comm_unique_id(unsigned char *id) {
  PN_API_BEGIN
  PN_REQUIRE(id, PN_E_ARG, "pn_comm_unique_id: NULL id");
  ncclUniqueId u;
  PN_CHECK_NCCL(nccl().getUniqueId(&u));
  memcpy(id, u.internal, PN_COMM_ID_BYTES);
  PN_API_END
}

extern "C" int pn_comm_init(int world, int rank, const unsigned char *id, int device, pn_comm **out) {
  PN_API_BEGIN
  PN_REQUIRE(out && id, PN_E_ARG, "pn_comm_init: NULL argument");
  PN_REQUIRE(world >= 1 && rank >= 0 && rank < world, PN_E_ARG, "pn_comm_init: rank %d of world %d", rank, world);
  *out = nullptr;
  PN_CHECK_CUDA(cudaSetDevice(device));
  auto c = new pn_comm;
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  memcpy(u.internal, id, PN_COMM_ID_BYTES);
  const ncclResult_t r = nccl().commInitRank(&c->comm, world, u, rank);
  if (r != 0) {
    delete c;
    PN_CHECK_NCCL(r);
  }
  *out = c;
  PN_API_END
}

extern "C" int pn_comm_destroy(pn_comm *c) {
  PN_API_BEGIN
  if (c) {
    if (c->comm) nccl().commDestroy(c->comm);
    delete c;
  }
  PN_API_END
}

// Gather every rank's shard of a batch result into the full batch on every
// rank.  x_shard: planes (es, cnt, n) of this rank's starts [lo, hi) (cnt =
// hi - lo by shard_range); x_all: planes (es, B, n); iters / status: int32
// per start.  Host or device pointers.  Shards are padded to the widest
// shard and packed into one buffer: a single ncclAllGather, the only
// collective of the run.
extern "C" int pn_batch_allgather(pn_comm *c, int nc, int cplx, int32_t n, int64_t B, const double *x_shard,
                                  const int32_t *iters_shard, const int32_t *status_shard, double *x_all,
                                  int32_t *iters_all, int32_t *status_all, void *stream) {
  PN_API_BEGIN
  PN_REQUIRE(c, PN_E_ARG, "pn_batch_allgather: NULL communicator");
  pn::check_level(nc, cplx);
  PN_REQUIRE(n >= 1 && B >= 0, PN_E_ARG, "pn_batch_allgather: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  const int es = nc * (cplx ? 2 : 1), W = c->world;
  int64_t lo, hi;
  shard_range(B, W, c->rank, lo, hi);
  const int64_t cnt = hi - lo, width = (B + W - 1) / W;
  const size_t xrow = (size_t)n * sizeof(double);
  // send: [es][width][n] doubles, then [width] iters, [width] status
  const size_t xsend = (size_t)es * width * xrow, isend = (size_t)width * sizeof(int32_t);
  const size_t per_rank = xsend + 2 * isend;
  pn::DevBuf send(per_rank + 16, st), recv(per_rank * W + 16, st);
  PN_CHECK_CUDA(cudaMemsetAsync(send.p, 0, per_rank, st));
  char *sp = send.as<char>();
  if (cnt > 0) {
    // one strided copy: es planes of cnt rows of n doubles
    PN_CHECK_CUDA(cudaMemcpy2DAsync(sp, (size_t)width * xrow, x_shard, (size_t)cnt * xrow, (size_t)cnt * xrow, es,
                                    cudaMemcpyDefault, st));
    PN_CHECK_CUDA(cudaMemcpyAsync(sp + xsend, iters_shard, (size_t)cnt * sizeof(int32_t), cudaMemcpyDefault, st));
    PN_CHECK_CUDA(cudaMemcpyAsync(sp + xsend + isend, status_shard, (size_t)cnt * sizeof(int32_t),
                                  cudaMemcpyDefault, st));
  }
  PN_CHECK_NCCL(nccl().allGather(sp, recv.p, per_rank, ncclInt8, c->comm, st));
  const char *rp = recv.as<char>();
  for (int r = 0; r < W; ++r) {
    int64_t rlo, rhi;
    shard_range(B, W, r, rlo, rhi);
    const int64_t rc = rhi - rlo;
    if (rc <= 0) continue;
    const char *src = rp + (size_t)r * per_rank;
    if (x_all)
      PN_CHECK_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char *>(x_all) + (size_t)rlo * xrow, (size_t)B * xrow, src,
                                      (size_t)width * xrow, (size_t)rc * xrow, es, cudaMemcpyDefault, st));
    if (iters_all)
      PN_CHECK_CUDA(cudaMemcpyAsync(iters_all + rlo, src + xsend, (size_t)rc * sizeof(int32_t), cudaMemcpyDefault, st));
    if (status_all)
      PN_CHECK_CUDA(cudaMemcpyAsync(status_all + rlo, src + xsend + isend, (size_t)rc * sizeof(int32_t),
                                    cudaMemcpyDefault, st));
  }
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  PN_API_END
}
