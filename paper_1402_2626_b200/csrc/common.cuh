// common.cuh -- shared host/device helpers for the polynewt_b200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <type_traits>

#include "../../include/polynewt_b200.h"
#include "xprec.cuh"

namespace pn {

// ---------------------------------------------------------------------------
// host error plumbing: every C-ABI entry point returns a status and leaves a
// message in a thread-local buffer (pn_last_error)

void set_error(const char *fmt, ...);

struct Fail {
  int code;
};

#define PN_CHECK_CUDA(expr)                                                            \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::pn::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,  \
                      __LINE__, cudaGetErrorString(_e));                               \
      throw ::pn::Fail{PN_E_CUDA};                                                     \
    }                                                                                  \
  } while (0)

#define PN_CHECK_LAUNCH() PN_CHECK_CUDA(cudaGetLastError())

#define PN_REQUIRE(cond, code, ...)        \
  do {                                     \
    if (!(cond)) {                         \
      ::pn::set_error(__VA_ARGS__);        \
      throw ::pn::Fail{code};              \
    }                                      \
  } while (0)

// convert exceptions to status codes at the C boundary
#define PN_API_BEGIN try {
#define PN_API_END                                             \
  }                                                            \
  catch (const ::pn::Fail &f) {                                \
    return f.code;                                             \
  }                                                            \
  catch (const std::bad_alloc &) {                             \
    ::pn::set_error("host allocation failed");                 \
    return PN_E_NOMEM;                                         \
  }                                                            \
  catch (...) {                                                \
    ::pn::set_error("unexpected C++ exception");               \
    return PN_E_CUDA;                                          \
  }                                                            \
  return PN_OK;

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// kernel-launch bookkeeping: bench.py reports how many of our kernels ran
void count_launch(int n = 1);

// ---------------------------------------------------------------------------
// device: canonical pairwise tree reduction over per-thread partials.
//
// tree_sum (varith.py:169-191) pairs (0,1),(2,3),... level by level and
// carries an odd tail; that equals stride-doubling: at stride s, index t
// (a multiple of 2s) absorbs t+s when t+s < n.  Thread t holds
// the partial of the aligned block t; nparts = number of blocks.  The result
// is returned in every thread.  sm must hold NT/32 elements.
template <class E, int NT>
__device__ __forceinline__ E block_tree_reduce(E v, int nparts, E *sm) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    E o = eshfl_down(v, s);
    if ((lane & (2 * s - 1)) == 0 && t + s < nparts) v = eadd(v, o);
  }
  constexpr int NW = NT / 32;
  if constexpr (NW > 1) {
    if (lane == 0) sm[w] = v;
    __syncthreads();
    if (w == 0) {
      const int nw = (nparts + 31) / 32;
      E x = (lane < NW) ? sm[lane] : sm[0];
#pragma unroll
      for (int s = 1; s < NW; s <<= 1) {
        E o = eshfl_down(x, s);
        if ((lane & (2 * s - 1)) == 0 && lane + s < nw) x = eadd(x, o);
      }
      __syncwarp();  // every lane has read sm[] before lane 0 overwrites sm[0]
      if (lane == 0) sm[0] = x;
    }
    __syncthreads();
    v = sm[0];
    __syncthreads();
  } else {
    const double *s = reinterpret_cast<const double *>(&v);
    E r;
    double *d = reinterpret_cast<double *>(&r);
#pragma unroll
    for (int i = 0; i < Traits<E>::es; ++i) d[i] = __shfl_sync(0xffffffffu, s[i], 0);
    v = r;
  }
  return v;
}

// The same tree with a single barrier: every warp writes its partial into
// half `parity` of sm (2*NT/32 elements), and after one __syncthreads every
// warp reduces the NT/32 partials itself with the same absorb rule.  The
// redundant cross-warp levels cost log2(NT/32) additions per warp but remove
// two barriers from the critical path; alternating `parity` between
// consecutive calls makes the reuse of sm race-free without a trailing
// barrier.
template <class E, int NT>
__device__ __forceinline__ E block_tree_reduce_1bar(E v, int nparts, E *sm, int parity) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    E o = eshfl_down(v, s);
    if ((lane & (2 * s - 1)) == 0 && t + s < nparts) v = eadd(v, o);
  }
  constexpr int NW = NT / 32;
  if constexpr (NW > 1) {
    E *h = sm + (parity & 1) * NW;
    if (lane == 0) h[w] = v;
    __syncthreads();
    const int nw = (nparts + 31) / 32;
    E x = h[lane < NW ? lane : 0];
#pragma unroll
    for (int s = 1; s < NW; s <<= 1) {
      E o = eshfl_down(x, s);
      if ((lane & (2 * s - 1)) == 0 && lane + s < nw) x = eadd(x, o);
    }
    v = x;
  }
  return eshfl_idx(v, 0);
}

// ---------------------------------------------------------------------------
// TMA 1-D bulk copies (cp.async.bulk global -> shared) completing on an
// mbarrier; sizes and addresses must be multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// ---------------------------------------------------------------------------
// multi-column tree reductions (warp reduce-scatter), shared by the batched
// solve and the pipelined MGS
// column carried by `lane` after the reduce-scatter levels of a P-wide reduction
template <int P> __device__ __forceinline__ int rs_col(int lane) {
  int c = 0;
#pragma unroll
  for (int l = 0; (1 << l) < P; ++l) c += ((lane >> l) & 1) * (P >> (l + 1));
  return c;
}

// level LV of the warp phase: lanes t and t^s combine the nodes t&~(2s-1)
// and (t&~(2s-1))+s; the lower node is the left operand, a missing upper
// node (index >= nparts) passes the lower one through
template <class E, int P, int LV>
__device__ __forceinline__ void rs_level(E (&v)[P], int t, int nparts) {
  constexpr int s = 1 << LV;
  constexpr int cnt = (P >> LV) > 0 ? (P >> LV) : 1;
  const bool upper = (t & s) != 0;
  const bool absorb = ((t & ~(2 * s - 1)) + s) < nparts;
  if constexpr (cnt > 1) {
    constexpr int h = cnt / 2;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const E mine = upper ? v[h + i] : v[i];
      const E send = upper ? v[i] : v[h + i];
      const E recv = eshfl_xor(send, s);
      const E lhs = upper ? recv : mine;
      const E rhs = upper ? mine : recv;
      v[i] = absorb ? eadd(lhs, rhs) : lhs;
    }
  } else {
    const E recv = eshfl_xor(v[0], s);
    const E lhs = upper ? recv : v[0];
    const E rhs = upper ? v[0] : recv;
    v[0] = absorb ? eadd(lhs, rhs) : lhs;
  }
  if constexpr (LV < 4) rs_level<E, P, LV + 1>(v, t, nparts);
}

// P simultaneous tree_sums over the CTA's row blocks; thread t holds the
// partial of its block for each column.  Results land in sout[par*P + c].
// sred holds 2 * NT/32 * P elements, sout 2 * P: the buffers alternate with
// the CTA-uniform parity `par` (flipped here), so consecutive reductions
// need no trailing barrier.  The tree over the warps' partials runs on warp
// 0 with 32/P lanes per column (a local pairwise tree over each lane's warp
// partials, then shuffle levels), not serially in one thread.  `mid` runs on
// every thread right after the first barrier (every thread has finished all
// earlier work of the CTA there).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// FOLD > 0: the P column results are the sums of FOLD consecutive aligned
// row blocks of one column; warp 0 also folds them by their pairwise tree
// (two shuffle levels for P = 4) and sout[par * P] gets the one total, so
// the other warps read one value instead of each repeating the fold.
template <class E, int P, int NT, int FOLD = 0, class Hook = NoHook>
__device__ __forceinline__ void multi_tree_reduce(E (&v)[P], int nparts, E *sred, E *sout, int &par,
                                                  const Hook &mid = Hook()) {
  constexpr int NW = NT / 32;
  constexpr int LPC0 = 32 / P;
  constexpr int LPC = LPC0 < NW ? LPC0 : NW;  // lanes per column
  constexpr int WPL = NW / LPC;               // warp partials per lane
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  E *sr = sred + par * NW * P;
  E *so = sout + par * P;
  rs_level<E, P, 0>(v, t, nparts);
  if (lane < P) sr[w * P + rs_col<P>(lane)] = v[0];
  __syncthreads();
  mid();
  if (w == 0) {
    const int nw = (nparts + 31) / 32;
    const int c = lane / LPC, jl = lane % LPC;
    const int cc = c < P ? c : 0;
    E x[WPL];
#pragma unroll
    for (int i = 0; i < WPL; ++i) x[i] = sr[(jl * WPL + i) * P + cc];
#pragma unroll
    for (int s = 1; s < WPL; s <<= 1)
#pragma unroll
      for (int i = 0; i + s < WPL; i += 2 * s)
        if (jl * WPL + i + s < nw) x[i] = eadd(x[i], x[i + s]);
    E acc = x[0];
#pragma unroll
    for (int s2 = 1; s2 < LPC; s2 <<= 1) {
      const E o = eshfl_xor(acc, s2);
      const bool upper = (jl & s2) != 0;
      const bool absorb = ((jl & ~(2 * s2 - 1)) + s2) * WPL < nw;
      const E lhs = upper ? o : acc;
      const E rhs = upper ? acc : o;
      acc = absorb ? eadd(lhs, rhs) : lhs;
    }
    if constexpr (FOLD > 0) {
      // every lane of a column group holds its total; combine the groups
#pragma unroll
      for (int f = 1; f < P; f <<= 1) {
        const E o = eshfl_xor(acc, f * LPC);
        const bool upper = (c & f) != 0;
        const bool absorb = ((c & ~(2 * f - 1)) + f) < FOLD;
        const E lhs = upper ? o : acc;
        const E rhs = upper ? acc : o;
        acc = absorb ? eadd(lhs, rhs) : lhs;
      }
      if (lane == 0) so[0] = acc;
    } else {
      if (jl == 0 && c < P) so[c] = acc;
    }
  }
  __syncthreads();
  par ^= 1;
}

// sequential pairwise tree over a register array of B elements where only
// the first `valid` are present (aligned block; right-pruned)
template <class E, int B>
__device__ __forceinline__ E local_tree(E (&v)[B], int valid) {
#pragma unroll
  for (int s = 1; s < B; s <<= 1) {
#pragma unroll
    for (int t = 0; t + s < B; t += 2 * s) {
      if (t + s < valid) v[t] = eadd(v[t], v[t + s]);
    }
  }
  return v[0];
}

// element load/store on component planes: plane p of a (cshape, count)
// array lives at base + p*count
template <class E>
__device__ __forceinline__ E eload_planes(const double *__restrict__ base, long long count, long long i) {
  E r;
  double *d = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int p = 0; p < Traits<E>::es; ++p) d[p] = base[p * count + i];
  return r;
}
template <class E>
__device__ __forceinline__ void estore_planes(double *__restrict__ base, long long count, long long i, const E &v) {
  const double *d = reinterpret_cast<const double *>(&v);
#pragma unroll
  for (int p = 0; p < Traits<E>::es; ++p) base[p * count + i] = d[p];
}

// level dispatch: calls f.template operator()<E>() for the level's element type
template <class Fn>
inline void dispatch_level(int nc, int cplx, Fn &&f) {
  if (cplx) {
    if (nc == 1) f.template operator()<C<1>>();
    else if (nc == 2) f.template operator()<C<2>>();
    else f.template operator()<C<4>>();
  } else {
    if (nc == 1) f.template operator()<F<1>>();
    else if (nc == 2) f.template operator()<F<2>>();
    else f.template operator()<F<4>>();
  }
}

inline void check_level(int nc, int cplx) {
  PN_REQUIRE((nc == 1 || nc == 2 || nc == 4) && (cplx == 0 || cplx == 1), PN_E_ARG,
             "precision level must have nc in {1,2,4} and cplx in {0,1} (got nc=%d cplx=%d)", nc, cplx);
}

#ifdef PN_NC
// the precision level compiled by this translation unit
using PnLevel = std::conditional_t<PN_CPLX, C<PN_NC>, F<PN_NC>>;
#endif

}  // namespace pn
