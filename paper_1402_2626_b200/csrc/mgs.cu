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
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

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

// ---------------------------------------------------------------------------
// Persistent dataflow form of the same sweeps: one launch for the whole
// factorisation.  Column j is owned by CTA j mod G; a CTA applies sweep k to
// its columns as soon as pivot q_k is published (ready[k]), and the owner of
// column k+1 updates that column first, normalises it and publishes q_{k+1}.
// Every column still receives its updates in sweep order with the same
// reductions, so the result is bit-identical to the launch-per-sweep path;
// only the idle gaps between sweeps disappear.  All CTAs are co-resident
// (cooperative launch), so the waits cannot deadlock; a clock64 watchdog
// turns a stuck wait into an error instead of a hang.

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <class E, int B>
__device__ __forceinline__ void load_rows_cg(E (&v)[B], const double *__restrict__ col, int row0, int m) {
  constexpr int es = Traits<E>::es;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    E x = ezero<E>();
    if (row0 + q < m) {
      double *d = reinterpret_cast<double *>(&x);
      const double2 *s = reinterpret_cast<const double2 *>(col + (long long)(row0 + q) * es);
      if constexpr (es % 2 == 0) {
#pragma unroll
        for (int i = 0; i < es / 2; ++i) {
          double2 t = __ldcg(s + i);
          d[2 * i] = t.x;
          d[2 * i + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < es; ++i) d[i] = __ldcg(col + (long long)(row0 + q) * es + i);
      }
    }
    v[q] = x;
  }
}

// Intra-CTA step counter of the back-substitution lookahead: the solver
// publishes x_j in shared memory and then the step count with a block-scope
// release store; the lookahead group spins on an acquire load (libcu++
// atomic_ref, so the ordering is explicit to the compiler and the tools).
// Step hand-off of the back-substitution kernels: one mbarrier per step slot
// of a 32-row block (count 1: the thread that stores x_j arrives with release
// semantics; the lookahead group waits on the slot's phase with acquire).
// Only blocks with a lookahead group (b > 0) arrive, so every completed phase
// has its waiter; slot s has completed one phase per earlier block that used
// it (the first block, processed first, is the short one: n0 rows), so block
// number p (in processing order) waits for parity (p - (s >= n0)) & 1.  An
// mbarrier is a synchronisation object the sanitizers track, unlike an atomic
// counter.
__device__ __forceinline__ void xslot_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ uint32_t xslot_parity(int p, int s, int n0) { return (uint32_t)(p - (s >= n0 ? 1 : 0)) & 1; }
__device__ __forceinline__ void xslot_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// publish pivot k: make this CTA's Q/R writes visible, then raise the flag
// diagnostics (PN_MGS_TRACE=file): global-timer stamp of every published pivot
__device__ unsigned long long *g_mgs_trace = nullptr;
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The CTA barrier orders every thread's Q/R stores before thread 0's
// release store (gpu scope, cumulative), so one fence in thread 0 suffices
// instead of a MEMBAR.GPU in every thread (the CUTLASS semaphore pattern).
__device__ __forceinline__ void red_release_add(int *p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void publish(int *ready, int k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    st_release(ready + k, 1);
    if (g_mgs_trace) g_mgs_trace[k] = globaltimer();
  }
}

// wait for pivot k; false on failure (breakdown elsewhere or watchdog)
__device__ __forceinline__ bool wait_pivot(const int *ready, int k, MgsStatus *status) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    int ok = 1;
    while (ld_acquire(ready + k) == 0) {
      __nanosleep(64);
      if (ld_acquire(&status->code) != 0) {  // a breakdown ended the factorisation
        ok = 0;
        break;
      }
      if (clock64() - t0 > (1ll << 36)) {  // ~30 s at 2 GHz: never on a healthy run
        status->k = k;
        atomicExch(&status->code, PN_E_CUDA);
        ok = 0;
        break;
      }
    }
    if (ok && ld_acquire(&status->code) != 0) ok = 0;
    s_ok = ok;
  }
  __syncthreads();
  const bool ok = s_ok;
  __syncthreads();
  return ok;
}

#ifndef PN_DATAFLOW_MINB
#define PN_DATAFLOW_MINB 2  // two CTAs per SM (128 regs, no spills): cdd MGS 21.3 -> 20.0 ms
#endif
template <class E, int B>
__global__ void __launch_bounds__(kMgsThreads, PN_DATAFLOW_MINB) k_mgs_dataflow(double *__restrict__ A, int m, int n,
                                                              double *__restrict__ orig, double eps,
                                                              double *__restrict__ Q, double *__restrict__ R,
                                                              MgsStatus *status, int *ready) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  __shared__ E sme[kMgsThreads / 32];
  __shared__ Rl smr[kMgsThreads / 32];
  const int G = gridDim.x, cta = blockIdx.x;
  const int row0 = threadIdx.x * B;
  const int valid = m - row0 < 0 ? 0 : (m - row0 > B ? B : m - row0);
  const int nparts = (m + B - 1) / B;
  // initial column norms of the owned columns (mgs.py:171-172)
  for (int j = cta; j < n; j += G) {
    E v[B];
    load_rows<E, B>(v, A + (long long)j * m * es, row0, m);
    Rl nrm = column_norm<E, B>(v, row0, m, smr);
    if (threadIdx.x == 0) orig[j] = nrm.c[0];
  }
  __syncthreads();
  if (cta == 0) {  // pivot 0
    E v[B];
    load_rows<E, B>(v, A, row0, m);
    Rl rkk = column_norm<E, B>(v, row0, m, smr);
    finish_pivot<E, B>(v, row0, m, n, 0, rkk, orig, eps, Q, R, status);
    publish(ready, 0);
  }
  if constexpr (Traits<E>::nc == 1) {
    // Every thread only ever reads back the rows it stored itself, so the next
    // (sweep, column) pair's rows can be loaded while the current one computes
    // (also across the wait for the next pivot); the L2 latency of the column
    // load leaves the critical path.
    auto first_after = [&](int k) { return k + 1 + (((cta - (k + 1)) % G) + G) % G; };
    E cur[B];
    int have = -1;  // column whose current rows are in cur
    for (int k = 0; k < n; ++k) {
      const int j0 = first_after(k);
      if (j0 > n) break;
      if (!wait_pivot(ready, k, status)) return;
      E qv[B];
      load_rows_cg<E, B>(qv, Q + (long long)k * m * es, row0, m);
      for (int j = j0; j <= n; j += G) {
        double *col = A + (long long)j * m * es;
        if (have != j) load_rows<E, B>(cur, col, row0, m);
        // next pair: (k, j+G) or (k+1, first column after k+1)
        int jn = j + G;
        if (jn > n) jn = k + 1 < n ? first_after(k + 1) : n + 1;
        const bool pf = jn <= n && jn != j;
        E nxt[B];
        if (pf) load_rows<E, B>(nxt, A + (long long)jn * m * es, row0, m);
        E pr[B];
  #pragma unroll
        for (int q = 0; q < B; ++q) pr[q] = emul(econj(qv[q]), cur[q]);
        E part = local_tree<E, B>(pr, valid);
        const E r = block_tree_reduce<E, kMgsThreads>(part, nparts, sme);
  #pragma unroll
        for (int q = 0; q < B; ++q) cur[q] = esub(cur[q], emul(qv[q], r));
        store_rows<E, B>(col, cur, row0, m);
        if (threadIdx.x == 0) estore(R + ((long long)j * (n + 1) + k) * es, r);
        if (j == k + 1) {
          Rl rkk = column_norm<E, B>(cur, row0, m, smr);
          const bool ok = finish_pivot<E, B>(cur, row0, m, n, k + 1, rkk, orig, eps, Q, R, status);
          publish(ready, k + 1);  // also on breakdown, so that waiters wake up
          if (!ok) return;
        }
        if (pf) {
  #pragma unroll
          for (int q = 0; q < B; ++q) cur[q] = nxt[q];
          have = jn;
        } else {
          have = (jn == j) ? j : -1;  // the same column again next sweep: cur is current
        }
      }
    }
  } else {
    // dd/qd: the prefetch registers would cost the second CTA per SM (measured slower)
    for (int k = 0; k < n; ++k) {
      // first owned column after k
      int j0 = k + 1 + (((cta - (k + 1)) % G) + G) % G;
      if (j0 > n) break;
      if (!wait_pivot(ready, k, status)) return;
      E qv[B];
      load_rows_cg<E, B>(qv, Q + (long long)k * m * es, row0, m);
      for (int j = j0; j <= n; j += G) {
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
          const bool ok = finish_pivot<E, B>(a, row0, m, n, k + 1, rkk, orig, eps, Q, R, status);
          publish(ready, k + 1);  // also on breakdown, so that waiters wake up
          if (!ok) return;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_mgs_flow: the production schedule.  Same dataflow as k_mgs_dataflow, plus
//  * priority: each CTA always serves its lowest unfinished column first (the
//    next pivot on the critical path); while that column waits for a pivot,
//    the CTA catches its other columns up on every published sweep, checking
//    between sweeps whether the critical column can move again;
//  * the working column lives in shared memory (component planes, XOR
//    swizzled so thread t's aligned row block is bank-conflict free) and
//    stays there across consecutive sweeps; q_k rows stream from L2.  Few
//    live registers -> two CTAs per SM even in complex quad double.
// Per column the operation sequence is exactly the reference's, so results
// are bit-identical to both other schedules.

// element load through L2 only (pivots written by other CTAs in this launch)
template <class E>
__device__ __forceinline__ E eload_cg(const double *p) {
  E r;
  double *d = reinterpret_cast<double *>(&r);
  constexpr int es = Traits<E>::es;
  if constexpr (es % 2 == 0) {
#pragma unroll
    for (int i = 0; i < es / 2; ++i) {
      const double2 t = __ldcg(reinterpret_cast<const double2 *>(p) + i);
      d[2 * i] = t.x;
      d[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < es; ++i) d[i] = __ldcg(p + i);
  }
  return r;
}

template <class E, int B>
struct SmemCol {
  double *base;  // es planes of NT*B doubles
  int plane;
  __device__ __forceinline__ int pos(int r) const {
    // a 64-bit warp access is served per half-warp (16 doubles = 32 banks):
    // XOR the in-block index with the thread's position among the 16/B
    // threads that share a wavefront's bank row
    constexpr int W = (16 / B) > 0 ? 16 / B : 1;
    const int t = r / B, i = r % B;
    return t * B + (i ^ ((t / W) % B));
  }
  __device__ __forceinline__ E get(int r) const {
    E v;
    double *d = reinterpret_cast<double *>(&v);
    const int p = pos(r);
#pragma unroll
    for (int c = 0; c < Traits<E>::es; ++c) d[c] = base[c * plane + p];
    return v;
  }
  __device__ __forceinline__ void put(int r, const E &v) const {
    const double *d = reinterpret_cast<const double *>(&v);
    const int p = pos(r);
#pragma unroll
    for (int c = 0; c < Traits<E>::es; ++c) base[c * plane + p] = d[c];
  }
};

// streaming pairwise tree (binary counter) over a thread's aligned row block
template <class E, int D>
struct Pairwise {
  E st[D];
  int cnt = 0;
  __device__ __forceinline__ void push(E v) {
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (!((cnt >> l) & 1)) {
        st[l] = v;
        break;
      }
      v = eadd(st[l], v);
    }
    ++cnt;
  }
  __device__ __forceinline__ E fold() const {
    E acc = ezero<E>();
    bool have = false;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if ((cnt >> l) & 1) {
        acc = have ? eadd(st[l], acc) : st[l];
        have = true;
      }
    }
    return acc;
  }
};

template <int B> struct Depth { static constexpr int value = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 3 : B <= 8 ? 4 : 5; };

template <class E, int B, int NT>
__global__ void __launch_bounds__(NT, NT <= 128 ? 3 : NT <= 256 ? 2 : 1) k_mgs_flow(double *__restrict__ A, int m, int n, double *__restrict__ orig,
                                                    double eps, double *__restrict__ Q, double *__restrict__ R,
                                                    MgsStatus *status, int *ready, int kstop, int hold, int lag,
                                                    const int *__restrict__ own, int maxo, int pickrule,
                                                    bool qcache) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  constexpr int D = Depth<B>::value;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double smem_col[];
  // Broadcast slots are double-buffered by a CTA-uniform parity `par`: a slot
  // written by use #a is only rewritten by use #a+2, and every thread has
  // passed use #a+1's barrier (after reading #a) by then -- so a reduction
  // needs two barriers instead of three, and the pivot poll rides along.
  __shared__ E s_pe[2][NW], s_re[2];
  __shared__ Rl s_pr[2][NW], s_rr[2];
  __shared__ int s_kn[2], s_fl[2];
  const int cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int row0 = tid * B;
  const int nparts = (m + B - 1) / B;
  const int row = cta;  // the CTA's row of the ownership table
  // the CTA's columns, ascending (own: maxo per CTA, -1 padded)
  int cols[64];
  int nown = 0;
  for (int i = 0; i < maxo && i < 64; ++i) {
    const int j = own[row * maxo + i];
    if (j < 0) break;
    cols[nown++] = j;
  }
  const SmemCol<E, B> col{smem_col, NT * B};
  if (nown == 0) return;
  // CTA-uniform state (every thread holds the same values) and thread 0's
  // private poll cursor
  int known = 0, fail = 0, par = 0, res = -1;
  int kn0 = 0, f0 = 0;
  int done[64];
  for (int i = 0; i < 64; ++i) done[i] = 0;

  auto t0_poll = [&]() {  // thread 0: advance past every published pivot
    while (kn0 < n && ld_acquire(ready + kn0)) ++kn0;
    if (ld_acquire(&status->code)) f0 = 1;
  };
  auto poll = [&]() {  // one barrier
    if (tid == 0) {
      t0_poll();
      s_kn[par] = kn0;
      s_fl[par] = f0;
    }
    __syncthreads();
    known = s_kn[par];
    fail = s_fl[par];
    par ^= 1;
  };
  // tree_sum over the CTA's row blocks (two barriers, poll included)
  auto reduce2 = [&](auto v, auto *part, auto *out) {
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const auto o = eshfl_down(v, s);
      if ((lane & (2 * s - 1)) == 0 && tid + s < nparts) v = eadd(v, o);
    }
    if (lane == 0) part[par * NW + w] = v;
    if (tid == 0) {
      t0_poll();
      s_kn[par] = kn0;
      s_fl[par] = f0;
    }
    __syncthreads();
    if (w == 0) {
      const int nw = (nparts + 31) / 32;
      auto x = part[par * NW + (lane < NW ? lane : 0)];
#pragma unroll
      for (int s = 1; s < NW; s <<= 1) {
        const auto o = eshfl_down(x, s);
        if ((lane & (2 * s - 1)) == 0 && lane + s < nw) x = eadd(x, o);
      }
      if (lane == 0) out[par] = x;
    }
    __syncthreads();
    const auto r = out[par];
    known = s_kn[par];
    fail = s_fl[par];
    par ^= 1;
    return r;
  };
  auto make_resident = [&](int idx) {
    if (res == idx) return;
    __syncthreads();  // the current column's sweeps are done with the smem rows
    if (res >= 0) {
      double *g = A + (long long)cols[res] * m * es;
      for (int r = tid; r < m; r += NT) estore(g + (long long)r * es, col.get(r));
    }
    const double *g = A + (long long)cols[idx] * m * es;
    for (int r = tid; r < m; r += NT) col.put(r, eload<E>(g + (long long)r * es));
    __syncthreads();
    res = idx;
  };
  auto block_wait = [&](int k) {
    if (tid == 0) {
      long long t0 = clock64();
      while (!ld_acquire(ready + k)) {
        if (ld_acquire(&status->code)) break;
        __nanosleep(100);
        if (clock64() - t0 > (1ll << 36)) {
          status->k = k;
          atomicExch(&status->code, PN_E_CUDA);
          break;
        }
      }
    }
    poll();
  };
  // q rows: through L1 when qcache (the second read of a row and the other
  // half of each 32-byte sector hit L1), else L2 only.  Safe: a q column is
  // written once per launch before its release flag, nobody reads it earlier,
  // and its lines are whole (the column is a multiple of 128 bytes).
  auto qload = [&](const double *p) -> E { return qcache ? eload<E>(p) : eload_cg<E>(p); };
  // one sweep k applied to the resident column j (mgs.py:201-215)
  auto apply = [&](int k, int j) {
    const double *qk = Q + (long long)k * m * es;
    Pairwise<E, D> pw;
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int r = row0 + q;
      if (r < m) pw.push(emul(econj(qload(qk + (long long)r * es)), col.get(r)));
    }
    const E rk = reduce2(pw.fold(), &s_pe[0][0], s_re);
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int r = row0 + q;
      if (r < m) col.put(r, esub(col.get(r), emul(qload(qk + (long long)r * es), rk)));
    }
    if (tid == 0) estore(R + ((long long)j * (n + 1) + k) * es, rk);
  };
  // norm of the resident column (mgs.py:128-137)
  auto norm = [&]() -> Rl {
    Pairwise<Rl, D> pw;
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (row0 + q < m) pw.push(eabs2(col.get(row0 + q)));
    return fsqrt(reduce2(pw.fold(), &s_pr[0][0], s_rr));
  };

  // phase 0: initial norms of the owned columns (mgs.py:171-172)
  for (int i = 0; i < nown; ++i) {
    const int j = cols[i];
    if (j >= n) break;
    make_resident(i);
    const Rl nrm = norm();
    if (tid == 0) orig[j] = nrm.c[0];
  }

  // Columns c >= kstop only receive the sweeps k < kstop here and are
  // written back to A; k_mgs_tail finishes them (pivots kstop..n).
  poll();
  int lo = 0;
  while (lo < nown) {
    const int c = cols[lo];
    const int tgt = c < kstop ? c : kstop;
    if (fail) return;
    const int dlo = done[lo];
    if (dlo < tgt && dlo >= known) {
      // critical column blocked on pivot dlo: catch a lagging column up --
      // unless c pivots within `hold` sweeps of the one in flight: then this
      // CTA is on the critical path and a lagging apply would delay it
      int pick = -1;
      if (pickrule == 0) {  // earliest deadline: the lowest lagging column
        for (int i = lo + 1; i < nown; ++i)
          if (done[i] < known) {
            pick = i;
            break;
          }
      } else {  // longest remaining chain (cols[i] - done[i]) first
        int best = -1;
        for (int i = lo + 1; i < nown; ++i)
          if (done[i] < known && cols[i] - done[i] > best) {
            best = cols[i] - done[i];
            pick = i;
          }
      }
      // ... but a column lagging more than `lag` sweeps is caught up anyway:
      // its sweeps are a sequential chain that must not pile up
      if (pick >= 0 && c - dlo <= hold && known - done[pick] <= lag) pick = -1;
      if (pick < 0) {
        block_wait(dlo);
        continue;
      }
      make_resident(pick);
      const int cj = cols[pick];
      int d = done[pick];
      while (d < known && d < cj) {
        apply(d, cj);
        ++d;
        if (fail) return;
        if (known > dlo) break;  // the critical column can move again
      }
      done[pick] = d;
      continue;
    }
    // serve the critical column with every published sweep
    make_resident(lo);
    int d = dlo;
    while (d < tgt) {
      if (d >= known) {
        poll();
        if (fail) return;
        if (d >= known) break;  // next pivot not out yet: reconsider the work list
      }
      apply(d, c);
      ++d;
    }
    done[lo] = d;
    if (d < tgt) continue;
    if (c >= kstop) {  // hand the column to the tail kernel
      __syncthreads();
      double *g = A + (long long)c * m * es;
      for (int r = tid; r < m; r += NT) estore(g + (long long)r * es, col.get(r));
      __syncthreads();
      res = -1;
      ++lo;
      continue;
    }
    // pivot c (mgs.py:176-193); c == n is the residual norm z
    const Rl rkk = norm();
    if (c < n) {
      const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), orig[c]);
      if (rkk.c[0] <= thr) {
        if (tid == 0) {
          status->k = c;
          status->rkk = rkk.c[0];
          status->thr = thr;
          __threadfence();
          atomicExch(&status->code, PN_E_BREAKDOWN);
        }
        publish(ready, c);
        return;
      }
    }
    if (tid == 0) estore(R + ((long long)c * (n + 1) + c) * es, eembed(rkk, (E *)nullptr));
    if (c < n) {
      const RDiv<Traits<E>::nc> p = rdiv_prepare(rkk);
      double *qc = Q + (long long)c * m * es;
      for (int r = tid; r < m; r += NT) estore(qc + (long long)r * es, ediv_prepared(col.get(r), p));
      publish(ready, c);
    } else {
      __syncthreads();
    }
    res = -1;  // column c is final; nothing to write back
    ++lo;
  }
}

// ---------------------------------------------------------------------------
// k_mgs_tail: the last C sweeps of the quad-double factorisation.  There the
// flow kernel is critical-path bound (one pivot per ~64 us while only C
// columns remain, profiles/r01 trace), so every remaining column is split
// over S CTAs by aligned row blocks of RQ = NT*B rows.  Each part reduces its
// block (the lower levels of tree_sum's tree), the S partials are exchanged
// through global memory with release/acquire flags and combined in the same
// pairwise order (the top levels), so r_kj, the norms and therefore Q and R
// stay bit-identical.  Pivot j is published when all S parts have stored
// their rows of q_j (ready[j] counts to S).
template <class E, int B, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_mgs_tail(double *__restrict__ A, int m, int n, const double *__restrict__ orig,
                                                 double eps, double *__restrict__ Q, double *__restrict__ R,
                                                 MgsStatus *status, int *ready, int kstop, int S,
                                                 double *__restrict__ xch, int *__restrict__ xflag) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  constexpr int RQ = NT * B;
  __shared__ E sme[NT / 32];
  __shared__ Rl smr[NT / 32];
  __shared__ E s_r;
  __shared__ Rl s_n;
  __shared__ int s_ok;
  const int ci = blockIdx.x / S, part = blockIdx.x % S;
  const int j = kstop + ci;
  if (g_mgs_trace && blockIdx.x == 0 && threadIdx.x == 0) g_mgs_trace[n + 1] = globaltimer();  // tail start
  const int tid = threadIdx.x;
  const int row0 = part * RQ + tid * B;
  const int valid = m - row0 <= 0 ? 0 : (m - row0 >= B ? B : m - row0);
  const int prow = m - part * RQ;  // rows of this part (may exceed RQ)
  const int nparts = prow <= 0 ? 0 : ((prow >= RQ ? RQ : prow) + B - 1) / B;
  const int sparts = (m + RQ - 1) / RQ;  // parts with rows
  const long long ldR = n + 1;
  const double *col = A + (long long)j * m * es;
  E a[B];
#pragma unroll
  for (int q = 0; q < B; ++q) a[q] = q < valid ? eload<E>(col + (long long)(row0 + q) * es) : ezero<E>();
  // exchange slot of column ci: [2 parity][S] elements (E units) + flags
  E *xe = reinterpret_cast<E *>(xch) + (long long)ci * 2 * S;
  int *xf = xflag + (long long)ci * 2 * S;
  // publish this part's partial with tag, gather all S, combine in tree order
  auto exchange = [&](auto v, int tag) {
    using T = decltype(v);
    T *slot = reinterpret_cast<T *>(xe + (tag & 1) * S);
    if (tid == 0) {
      slot[part] = v;
      __threadfence();
      st_release(xf + (tag & 1) * S + part, tag);
      bool ok = true;
      long long t0 = clock64();
      for (int p = 0; p < sparts && ok; ++p)
        while (ld_acquire(xf + (tag & 1) * S + p) != tag) {
          if (ld_acquire(&status->code)) { ok = false; break; }
          if (clock64() - t0 > (1ll << 36)) {
            atomicExch(&status->code, PN_E_CUDA);
            ok = false;
            break;
          }
        }
      T acc = v;
      if (ok) {
        T w[8];
        for (int p = 0; p < sparts; ++p) w[p] = eload_cg<T>(reinterpret_cast<const double *>(slot + p));
        for (int st = 1; st < sparts; st <<= 1)
          for (int p = 0; p + st < sparts; p += 2 * st) w[p] = eadd(w[p], w[p + st]);
        acc = w[0];
      }
      s_ok = ok;
      return acc;
    }
    return v;
  };
  for (int k = kstop; k <= j && k <= n; ++k) {
    if (k < j) {
      // wait for pivot k (all S parts of its column stored q_k)
      if (tid == 0) {
        long long t0 = clock64();
        int ok = 1;
        while (ld_acquire(ready + k) < S) {
          if (ld_acquire(&status->code)) { ok = 0; break; }
          __nanosleep(32);
          if (clock64() - t0 > (1ll << 36)) {
            atomicExch(&status->code, PN_E_CUDA);
            ok = 0;
            break;
          }
        }
        s_ok = ok;
      }
      __syncthreads();
      if (!s_ok) return;  // every part of a column waits on the same flag: all leave here
      const double *qk = Q + (long long)k * m * es;
      E qv[B];
#pragma unroll
      for (int q = 0; q < B; ++q) qv[q] = q < valid ? eload_cg<E>(qk + (long long)(row0 + q) * es) : ezero<E>();
      E pr[B];
#pragma unroll
      for (int q = 0; q < B; ++q) pr[q] = emul(econj(qv[q]), a[q]);
      const E part_sum = block_tree_reduce<E, NT>(local_tree<E, B>(pr, valid), nparts, sme);
      const E r = exchange(part_sum, k + 1);
      if (tid == 0) s_r = r;
      __syncthreads();
      if (!s_ok) return;
      const E rk = s_r;
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q < valid) a[q] = esub(a[q], emul(qv[q], rk));
      if (part == 0 && tid == 0) estore(R + ((long long)j * ldR + k) * es, rk);
      __syncthreads();  // s_r / s_ok reuse
      continue;
    }
    // pivot j (mgs.py:176-193); j == n is the residual norm z
    Rl a2[B];
#pragma unroll
    for (int q = 0; q < B; ++q) a2[q] = eabs2(a[q]);
    const Rl part_n = block_tree_reduce<Rl, NT>(local_tree<Rl, B>(a2, valid), nparts, smr);
    const Rl tot = exchange(part_n, j + 1 + (1 << 30));
    if (tid == 0) s_n = tot;
    __syncthreads();
    if (!s_ok) return;
    const Rl rkk = fsqrt(s_n);
    if (j < n) {
      const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), orig[j]);
      if (rkk.c[0] <= thr) {
        if (part == 0 && tid == 0) {
          status->k = j;
          status->rkk = rkk.c[0];
          status->thr = thr;
          __threadfence();
          atomicExch(&status->code, PN_E_BREAKDOWN);
        }
        return;
      }
    }
    if (part == 0 && tid == 0) estore(R + ((long long)j * ldR + j) * es, eembed(rkk, (E *)nullptr));
    if (j < n) {
      const RDiv<Traits<E>::nc> p = rdiv_prepare(rkk);
      double *qc = Q + (long long)j * m * es;
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q < valid) estore(qc + (long long)(row0 + q) * es, ediv_prepared(a[q], p));
      __syncthreads();
      if (tid == 0) {
        red_release_add(ready + j, 1);
        if (g_mgs_trace && part == 0) g_mgs_trace[j] = globaltimer();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_mgs_pipe: the dataflow schedule with TMA-pipelined operands (d, dd; m a
// multiple of 256).  The dataflow kernel stalls on the L2 latency of every
// column it streams (ncu: long_scoreboard is its top stall for cdd).  Here a
// CTA knows the order of its (sweep, column) applies in advance, so the next
// column is brought into a second shared-memory buffer by a cp.async.bulk
// (TMA) while the current one computes, and q_k arrives the same way once per
// sweep.  Thread t owns rows t, t+256, ... (one row of each 256-row block).
// For double double the element accesses conflict (ncu r01: 570 M excess
// wavefronts); a lane-rotated 16-byte access order removed 88 % of them but
// made the kernel 6 % slower (the selects cost more than the conflicts: it is
// barrier and FP64 bound, ncu r02), so the plain layout stays;
// each block's dot product is a block tree, reduced for all blocks at once by
// the warp reduce-scatter, and the block sums are combined pairwise (aligned
// 256-row blocks: the top levels of tree_sum's tree).  Column updates are
// written back to A (and a generic->async proxy fence orders them before the
// later bulk copy of the same column).
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// block sums of NQ aligned 256-row blocks (reduce-scatter), then their
// pairwise tree (absorb rule over the blocks)
template <class T, int P, int NQ, int NT, class Hook = NoHook>
__device__ __forceinline__ T pipe_block_sum(T (&v)[P], T *part, T *out, int &par, bool fold,
                                            const Hook &mid = Hook()) {
  const T *res = out + par * P;
  if (fold) {
    multi_tree_reduce<T, P, NT, NQ>(v, NT, part, out, par, mid);
    return res[0];
  }
  multi_tree_reduce<T, P, NT>(v, NT, part, out, par, mid);
  T acc = res[0];
  if constexpr (NQ == 2) acc = eadd(res[0], res[1]);
  if constexpr (NQ == 3) acc = eadd(eadd(res[0], res[1]), res[2]);
  if constexpr (NQ == 4) acc = eadd(eadd(res[0], res[1]), eadd(res[2], res[3]));
  return acc;
}

// thread-block cluster helpers (the PAIR variant of k_mgs_pipe)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_peer(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
// one element to the peer's shared memory, completing bytes on its mbarrier
template <class E>
__device__ __forceinline__ void st_async_elem(uint32_t addr, const E &v, uint32_t peer_bar) {
  const double *d = reinterpret_cast<const double *>(&v);
  constexpr int es = Traits<E>::es;
  if constexpr (es % 2 == 0) {
#pragma unroll
    for (int i = 0; i < es; i += 2)
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                       addr + 8 * i),
                   "d"(d[i]), "d"(d[i + 1]), "r"(peer_bar)
                   : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < es; ++i)
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr + 8 * i),
                   "d"(d[i]), "r"(peer_bar)
                   : "memory");
  }
}
__device__ __forceinline__ void remote_arrive(uint32_t peer_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(peer_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool mbar_try_cluster(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <class E, int NQ, int QB, bool PAIR = false>
__global__ void __launch_bounds__(256, 2) k_mgs_pipe(double *__restrict__ A, int m, int n, double *__restrict__ orig,
                                                     double eps, double *__restrict__ Q, double *__restrict__ R,
                                                     MgsStatus *status, int *ready, int late) {
  using Rl = typename Traits<E>::R;
  constexpr int NT = 256;
  constexpr int es = Traits<E>::es;
  constexpr int P = NQ == 1 ? 1 : (NQ == 2 ? 2 : 4);  // reduce-scatter width (power of two)
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) double pipe_smem[];
  E *colb = reinterpret_cast<E *>(pipe_smem);  // [2][m]
  E *qbuf = colb + 2 * m;                      // [QB][m] (QB = 2: q_{k+1} prefetched)
  E *qd = qbuf + (size_t)QB * m;               // PAIR: q_k pushed by the cluster partner
  __shared__ E s_pe[2 * NW * P], s_oe[2 * P];
  __shared__ Rl s_pr[2 * NW * P], s_or[2 * P];
  __shared__ __align__(8) uint64_t bar[6];     // col0, col1, q0, q1; PAIR: q pushed, pair buffer free
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const uint32_t cbytes = (uint32_t)m * es * sizeof(double);
  // warp 0 folds the block sums (dd at m = 1024: cdd factorisation 15.9 ->
  // 15.67 ms); complex double keeps the per-thread fold (5.05 -> 5.15 ms with
  // warp 0's two extra shuffle levels on its pivot chain), and so do fewer
  // than four blocks (0.5 % at m = 512 / 768), profiles/r02/exp ab17/ab18/ab52
  constexpr bool fold = Traits<E>::nc >= 2 && NQ == 4;
  int par = 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[3], 1);
    if (PAIR) {
      mbar_init(&bar[4], 1);
      mbar_init(&bar[5], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph[4] = {0, 0, 0, 0};
  // PAIR (cluster of two CTAs, 2i and 2i+1): column c of rank 0 is followed
  // by column c+1 of rank 1, so rank 0 pushes every q_c it pivots straight
  // into rank 1's shared memory (st.async, completing on rank 1's mbarrier)
  // and rank 1 starts its pivot sweep without the flag poll and bulk copy
  uint32_t rank = 0, ph4 = 0, ph5 = 0, peer_qd = 0, peer_b4 = 0, peer_b5 = 0;
  if constexpr (PAIR) {
    rank = cluster_rank();
    peer_qd = map_peer(qd, rank ^ 1);
    peer_b4 = map_peer(&bar[4], rank ^ 1);
    peer_b5 = map_peer(&bar[5], rank ^ 1);
    cluster_sync_all();  // the partner's barriers are initialised
    if (rank == 1 && tid == 0) remote_arrive(peer_b5);  // the pair buffer starts free
  }
  // every exit: no remote operation may target a CTA that has left
  auto leave = [&]() {
    if constexpr (PAIR) cluster_sync_all();
  };
  __shared__ int s_pok;
  // thread 0 waits on a cluster-scope mbarrier phase, giving up on a failure
  // status; the result is broadcast (one barrier)
  auto wait_cluster_bar = [&](uint64_t *b, uint32_t parity) -> bool {
    if (tid == 0) {
      int ok = 1;
      long long t0 = clock64();
      while (!mbar_try_cluster(b, parity)) {
        if (ld_acquire(&status->code) != 0) {
          ok = 0;
          break;
        }
        if (clock64() - t0 > (1ll << 36)) {
          atomicExch(&status->code, PN_E_CUDA);
          ok = 0;
          break;
        }
      }
      s_pok = ok;
    }
    __syncthreads();
    return s_pok != 0;
  };
  auto col_norm = [&](const E (&a)[NQ]) -> Rl {
    Rl v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = q < NQ ? eabs2(a[q]) : ezero<Rl>();
    return fsqrt(pipe_block_sum<Rl, P, NQ, NT>(v, s_pr, s_or, par, fold));
  };
  // initial column norms of the owned columns (mgs.py:171-172)
  for (int j = cta; j < n; j += G) {
    E a[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a[q] = eload<E>(A + ((long long)j * m + q * NT + tid) * es);
    const Rl nrm = col_norm(a);
    if (tid == 0) orig[j] = nrm.c[0];
  }
  __syncthreads();
  auto pivot = [&](int c, const E (&a)[NQ]) -> bool {  // (mgs.py:176-193)
    const Rl rkk = col_norm(a);
    if (c < n) {
      const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), orig[c]);
      if (rkk.c[0] <= thr) {
        if (tid == 0) {
          status->k = c;
          status->rkk = rkk.c[0];
          status->thr = thr;
          __threadfence();
          atomicExch(&status->code, PN_E_BREAKDOWN);
        }
        publish(ready, c);
        return false;
      }
    }
    if (tid == 0) estore(R + ((long long)c * (n + 1) + c) * es, eembed(rkk, (E *)nullptr));
    if (c < n) {
      const RDiv<Traits<E>::nc> p = rdiv_prepare(rkk);
      E qv[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        qv[q] = ediv_prepared(a[q], p);
        estore(Q + ((long long)c * m + q * NT + tid) * es, qv[q]);
      }
      fence_proxy_async();
      if constexpr (PAIR) {
        if (rank == 0) {  // push q_c to the partner, which pivots c+1 next
          if (!wait_cluster_bar(&bar[5], ph5)) return false;
          ph5 ^= 1;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            st_async_elem<E>(peer_qd + (uint32_t)((q * NT + tid) * es * sizeof(double)), qv[q], peer_b4);
        }
      }
      publish(ready, c);
    }
    return true;
  };
  if (cta == 0) {  // pivot 0
    E a[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a[q] = eload<E>(A + ((long long)q * NT + tid) * es);
    if (!pivot(0, a)) {
      leave();
      return;
    }
  }
  auto first_after = [&](int k) { return k + 1 + (((cta - (k + 1)) % G) + G) % G; };
  // No proxy fence at the issue: every generic write of A and Q is followed
  // by its writer's own fence.proxy.async (after the column update, before a
  // pivot's publish) and a barrier or release/acquire separates it from the
  // bulk copy, so a fence here would only stall thread 0 -- and with it warp
  // 0's part of the reduction the other warps wait for (ncu: barrier stalls)
  auto issue_col = [&](int j, int b) {  // thread 0
    mbar_expect_tx(&bar[b], cbytes);
    bulk_g2s(colb + (size_t)b * m, A + (long long)j * m * es, cbytes, &bar[b]);
  };
  int s = 0;
  int inbuf = -1;  // column whose current rows are in colb[s] (no copy pending)
  int qs = 0;      // q buffer of the current sweep
  int qpre = -1;   // (thread 0) sweep whose q is already being copied into the other buffer
  auto issue_q = [&](int k, int b) {  // thread 0
    mbar_expect_tx(&bar[2 + b], cbytes);
    bulk_g2s(qbuf + (size_t)b * m, Q + (long long)k * m * es, cbytes, &bar[2 + b]);
  };
  if (tid == 0 && first_after(0) <= n) issue_col(first_after(0), 0);
  // pivot wait with one barrier: s_ok is rewritten only at the next sweep's
  // wait, and every sweep has at least one apply (two reduction barriers) in
  // between
  __shared__ int s_ok;
  auto wait1 = [&](int k) -> bool {
    if (tid == 0) {
      long long t0 = clock64();
      int ok = 1;
      while (ld_acquire(ready + k) == 0) {
        __nanosleep(64);
        if (ld_acquire(&status->code) != 0) {
          ok = 0;
          break;
        }
        if (clock64() - t0 > (1ll << 36)) {
          status->k = k;
          atomicExch(&status->code, PN_E_CUDA);
          ok = 0;
          break;
        }
      }
      if (ok && ld_acquire(&status->code) != 0) ok = 0;
      s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
  };
  for (int k = 0; k < n; ++k) {
    const int j0 = first_after(k);
    if (j0 > n) break;
    // PAIR: rank 1's pivot sweep takes q_k from its partner's push
    const bool pair = PAIR && rank == 1 && j0 == k + 1;
    const E *qb;
    if (pair) {
      if (tid == 0) mbar_expect_tx(&bar[4], cbytes);
      const bool ok = wait_cluster_bar(&bar[4], ph4);
      ph4 ^= 1;
      if (!ok) {
        leave();
        return;
      }
      qb = qd;
    } else {
      if ((late & 2) ? !wait_pivot(ready, k, status) : !wait1(k)) {
        leave();
        return;
      }
      if (QB == 2) qs = k & 1;
      if (tid == 0 && qpre != k) issue_q(k, qs);
      mbar_wait(&bar[2 + qs], ph[2 + qs]);
      ph[2 + qs] ^= 1;
      qb = qbuf + (size_t)qs * m;
    }
    for (int j = j0; j <= n; j += G) {
      int jn = j + G;
      if (jn > n) jn = k + 1 < n ? first_after(k + 1) : n + 1;
      const bool pf = jn <= n && jn != j;
      // late: the prefetch goes out after the first barrier of this apply's
      // reduction (everyone is done with the other buffer there), so no
      // barrier closes the apply
      if (!(late & 1) && pf && tid == 0) issue_col(jn, s ^ 1);
      // q_{k+1} into the other buffer as soon as it is published (its last
      // reader, sweep k-1, finished before this sweep's first barrier)
      if (QB == 2 && tid == 0 && qpre != k + 1 && k + 1 < n && first_after(k + 1) <= n &&
          ld_acquire(ready + k + 1)) {
        issue_q(k + 1, qs ^ 1);
        qpre = k + 1;
      }
      if (inbuf != j) {
        mbar_wait(&bar[s], ph[s]);
        ph[s] ^= 1;
      }
      E a[NQ];
      E *cb = colb + (size_t)s * m;
      E v[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        if (q < NQ) {
          a[q] = cb[q * NT + tid];
          v[q] = emul(econj(qb[q * NT + tid]), a[q]);
        } else {
          v[q] = ezero<E>();
        }
      }
      const auto mid = [&]() {
        if ((late & 1) && pf && tid == 0) issue_col(jn, s ^ 1);
      };
      const E r = pipe_block_sum<E, P, NQ, NT>(v, s_pe, s_oe, par, fold, mid);
      double *col = A + (long long)j * m * es;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        a[q] = esub(a[q], emul(qb[q * NT + tid], r));
        cb[q * NT + tid] = a[q];
        estore(col + ((long long)q * NT + tid) * es, a[q]);
      }
      fence_proxy_async();
      if (tid == 0) estore(R + ((long long)j * (n + 1) + k) * es, r);
      if (j == k + 1 && !pivot(k + 1, a)) {
        leave();
        return;
      }
      if (!(late & 1)) __syncthreads();  // colb[s] and the reduction slots are free
      if (pf) {
        s ^= 1;
        inbuf = -1;
      } else {
        inbuf = (jn == j) ? j : -1;
      }
    }
    if constexpr (PAIR) {
      if (pair) {
        __syncthreads();  // every thread is done with the pushed q_k
        if (tid == 0) remote_arrive(peer_b5);
      }
    }
  }
  leave();
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

// PN_MGS_MODE=sweeps selects the launch-per-sweep schedule (kept as the
// reference schedule for tests); the default is the persistent dataflow kernel.
// 0 flow, 1 dataflow, 2 sweeps, 4 pipe, 5 small (the warp-per-column
// schedule, 2-3x slower for cd/cdd in r01, was removed).  Default by measurement
// (profiles/r01): the priority/smem schedule wins when sweeps are
// compute-heavy (quad double); for d/dd the TMA-pipelined dataflow kernel
// (k_mgs_pipe, m a multiple of 256 up to 1024) and otherwise the plain
// dataflow kernel have the shorter per-sweep latency.
static int mgs_mode(int nc) {
  const char *v = getenv("PN_MGS_MODE");
  if (v && strcmp(v, "sweeps") == 0) return 2;
  if (v && strcmp(v, "dataflow") == 0) return 1;
  if (v && strcmp(v, "flow") == 0) return 0;
  if (v && strcmp(v, "pipe") == 0) return 4;
  if (v && strcmp(v, "small") == 0) return 5;
  return nc == 4 ? 0 : 4;
}

static void trace_begin(int n, unsigned long long **buf) {
  *buf = nullptr;
  if (!getenv("PN_MGS_TRACE")) return;
  PN_CHECK_CUDA(cudaMalloc(buf, sizeof(unsigned long long) * (n + 2)));
  PN_CHECK_CUDA(cudaMemset(*buf, 0, sizeof(unsigned long long) * (n + 2)));
  PN_CHECK_CUDA(cudaMemcpyToSymbol(g_mgs_trace, buf, sizeof(*buf)));
}
static void trace_end(int n, unsigned long long *buf, cudaStream_t st) {
  if (!buf) return;
  PN_CHECK_CUDA(cudaStreamSynchronize(st));
  std::vector<unsigned long long> h(n + 2);
  PN_CHECK_CUDA(cudaMemcpy(h.data(), buf, sizeof(unsigned long long) * (n + 2), cudaMemcpyDeviceToHost));
  unsigned long long *null = nullptr;
  PN_CHECK_CUDA(cudaMemcpyToSymbol(g_mgs_trace, &null, sizeof(null)));
  cudaFree(buf);
  if (FILE *f = fopen(getenv("PN_MGS_TRACE"), "w")) {
    for (int k = 0; k <= n + 1; ++k) fprintf(f, "%d %llu\n", k, h[k]);
    fclose(f);
  }
}

// Column ownership of the flow kernel.  A CTA applies its columns' sweeps
// one at a time and shares its SM with one other CTA (c and c + S, S SMs),
// so what has to be balanced is the sweep count per SM over time.
// "smsnake" (default with two CTAs per SM): rounds of S columns are dealt to
// the SMs in alternating direction (SM s gets s, 2S-1-s, 2S+s, ...), which
// gives every SM the same total over the full rounds (max/mean 1.02 at
// n = 1024 vs 1.13 for round robin), and an SM's columns alternate between
// its two CTAs; cqd MGS 106.3 -> 102.9 ms.  "rr": CTA c owns c, c+G, ...;
// "snake": CTA-level alternating direction (pivot n-C 14 ms sooner but the
// tail kernel's columns are left behind: +4 ms).  Other in-SM splits
// (greedy by load, ABBA) were slower (scripts/own/*.txt, profiles/r01).
// PN_FLOW_OWN=smsnake|rr|snake.
static void flow_owner_table(int n, int G, MgsWork &w, cudaStream_t st) {
  const char *v = getenv("PN_FLOW_OWN");
  const int S = num_sms();
  const bool pairs = G == 2 * S;  // two CTAs per SM: c and c + S share one
  const int var = v && strcmp(v, "rr") == 0 ? 0 : v && strcmp(v, "snake") == 0 ? 1 : (pairs ? 3 : 0);
  const long long key = ((long long)n << 32) | ((long long)G << 4) | var;
  if (w.own_key == key) return;
  std::vector<std::vector<int>> lists(G);
  if (var == 3) {
    // SM-level snake: round r of S columns goes to SMs 0..S-1, alternating
    // direction; an SM's r-th column goes to its CTA s (r even) or s + S
    for (int j = 0; j <= n; ++j) {
      const int r = j / S, i = j % S;
      const int sm = (r & 1) ? S - 1 - i : i;
      lists[sm + ((r & 1) ? S : 0)].push_back(j);
    }
  } else {
    for (int j = 0; j <= n; ++j) {
      const int r = j / G, i = j % G;
      lists[var == 1 && (r & 1) ? G - 1 - i : i].push_back(j);
    }
  }
  int maxo = 1;
  std::vector<int> seen(n + 1, 0);
  for (auto &l : lists) {
    std::sort(l.begin(), l.end());
    maxo = std::max(maxo, (int)l.size());
    for (int j : l) ++seen[j];
  }
  for (int j = 0; j <= n; ++j)
    if (seen[j] != 1) {  // an unowned column would stall every pivot after it
      set_error("flow schedule: column %d owned %d times", j, seen[j]);
      throw Fail{PN_E_ARG};
    }
  if (maxo > 64) {
    set_error("flow schedule: more than 64 columns per CTA");
    throw Fail{PN_E_ARG};
  }
  std::vector<int> tab((size_t)G * maxo, -1);
  for (int c = 0; c < G; ++c)
    for (size_t i = 0; i < lists[c].size(); ++i) tab[(size_t)c * maxo + i] = lists[c][i];
  w.own.ensure(tab.size() * sizeof(int));
  PN_CHECK_CUDA(cudaMemcpyAsync(w.own.p, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  PN_CHECK_CUDA(cudaStreamSynchronize(st));  // tab is pageable and goes out of scope
  w.own_key = key;
  w.own_maxo = maxo;
}

template <class E, int B, int NT>
static bool flow_launch(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  MgsStatus *status = w.status.as<MgsStatus>();
  double *orig = w.orig.d();
  const double eps = level_eps(Traits<E>::nc);
  const size_t smem = (size_t)Traits<E>::es * NT * B * sizeof(double);
  auto kern = k_mgs_flow<E, B, NT>;
  PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  const int grid = std::min(per_sm * num_sms(), n + 1);
  if (per_sm <= 0 || (n + 1 + grid - 1) / grid > 64) return false;
  // row-split tail (quad double): the last C columns, S CTAs each, parts of
  // RQ = 256 rows (128 threads x 2 rows, four CTAs per SM; 64 x 4 and
  // 128 x 4-row variants and a cluster/DSMEM exchange were measured slower
  // or equal in r01 and removed)
  const char *tv = getenv("PN_MGS_TAIL");
  const void *tk = (const void *)k_mgs_tail<E, 2, 128>;
  const int tnt = 128, RQ = 256;
  int kstop = n + 1, S = (m + RQ - 1) / RQ, C = 0;
  if (Traits<E>::nc == 4 && S >= 2 && S <= 8 && !(tv && strcmp(tv, "0") == 0)) {
    int tper = 0;
    PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tper, tk, tnt, 0));
    C = std::min(n + 1, tper * num_sms() / S);
    if (tv && atoi(tv) > 0) C = std::min(C, atoi(tv));
    if (C >= 16) kstop = n + 1 - C;
    else C = 0;
  }
  w.ready.ensure((size_t)(n + 1) * sizeof(int));
  PN_CHECK_CUDA(cudaMemsetAsync(w.ready.p, 0, (size_t)(n + 1) * sizeof(int), st));
  int *ready = w.ready.as<int>();
  // hold: a CTA whose critical column pivots within `hold` sweeps of the
  // pivot in flight does no lagging work (PN_FLOW_HOLD, 0 = off; round 1: 1
  // measured 129.5 -> 124.2 ms per cqd step; round 2, final kernels: cqd
  // factorisation 111.8 / 102.70 / 102.40 / 102.42 / 102.43 ms for hold =
  // 0 / 1 / 2 / 3 / 4, profiles/r02/exp ab60/ab61)
  const char *hv = getenv("PN_FLOW_HOLD");
  int hold = hv ? atoi(hv) : 2;
  const char *lv = getenv("PN_FLOW_LAG");
  int lag = lv ? atoi(lv) : 1 << 30;
  flow_owner_table(n, grid, w, st);
  const int *own = w.own.as<int>();
  int maxo = w.own_maxo;
  // lagging column to catch up: 1 = longest remaining chain (default,
  // cqd MGS 107.5 -> 106.8 ms), 0 = lowest index (earliest deadline)
  const char *pv = getenv("PN_FLOW_PICK");
  int pickrule = pv ? atoi(pv) : 1;
  // q rows through L1 (cqd factorisation 103.25 -> 102.72 ms, profiles/r02/exp
  // ab7); PN_FLOW_QCACHE=0 streams them from L2 only
  const char *qc = getenv("PN_FLOW_QCACHE");
  bool qcache = !(qc && strcmp(qc, "0") == 0) && ((long long)m * Traits<E>::es * 8) % 128 == 0;
  void *args[] = {&A, &m, &n, &orig, (void *)&eps, &Q, &R, &status, &ready, &kstop, &hold, &lag, &own, &maxo, &pickrule,
                  &qcache};
  unsigned long long *tr = nullptr;
  trace_begin(n, &tr);
  PN_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)kern, grid, NT, args, smem, st));
  count_launch(1);
  if (C > 0) {
    constexpr int es = Traits<E>::es;
    DevBuf xch((size_t)C * 2 * S * es * sizeof(double) + 16, st), xfl((size_t)C * 2 * S * sizeof(int) + 16, st);
    PN_CHECK_CUDA(cudaMemsetAsync(xfl.p, 0, (size_t)C * 2 * S * sizeof(int), st));
    double *xp = xch.d();
    int *xf = xfl.as<int>();
    void *targs[] = {&A, &m, &n, &orig, (void *)&eps, &Q, &R, &status, &ready, &kstop, &S, &xp, &xf};
    PN_CHECK_CUDA(cudaLaunchCooperativeKernel(tk, C * S, tnt, targs, 0, st));
    count_launch(1);
  }
  trace_end(n, tr, st);
  return true;
}

// PAIR launch of k_mgs_pipe (complex/real double): clusters of two CTAs,
// cooperative; false when the clusters cannot all be resident
template <class E, int NQ>
static bool pipe_launch_pair(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  MgsStatus *status = w.status.as<MgsStatus>();
  double *orig = w.orig.d();
  double eps = level_eps(Traits<E>::nc);
  constexpr int QB = 1;
  const size_t smem = (size_t)(2 + QB + 1) * m * Traits<E>::es * sizeof(double);
  auto kern = k_mgs_pipe<E, NQ, QB, true>;
  PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  if (per_sm <= 0) return false;
  int grid = std::min(per_sm * num_sms(), n + 1) & ~1;  // even: whole clusters, G even
  if (grid < 2) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void *)kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (2 * nclusters < grid) grid = 2 * nclusters;
  if (grid < 2) return false;
  cfg.gridDim = dim3(grid);
  cfg.numAttrs = 2;
  w.ready.ensure((size_t)(n + 1) * sizeof(int));
  PN_CHECK_CUDA(cudaMemsetAsync(w.ready.p, 0, (size_t)(n + 1) * sizeof(int), st));
  int *ready = w.ready.as<int>();
  int late = 0;
  unsigned long long *tr = nullptr;
  trace_begin(n, &tr);
  PN_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, A, m, n, orig, eps, Q, R, status, ready, late));
  trace_end(n, tr, st);
  count_launch(1);
  return true;
}

template <class E, int NQ>
static bool pipe_launch(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  if constexpr (Traits<E>::nc == 1) {
    const char *pv = getenv("PN_PIPE_PAIR");
    if (pv && atoi(pv) == 1 && pipe_launch_pair<E, NQ>(m, n, A, Q, R, w, st)) return true;
  }
  MgsStatus *status = w.status.as<MgsStatus>();
  double *orig = w.orig.d();
  const double eps = level_eps(Traits<E>::nc);
  // QB = 2 (q_{k+1} prefetched as soon as it is published) measured slower
  // for cd (5.3 -> 5.7 ms: thread 0's per-apply flag poll delays every apply)
  constexpr int QB = 1;
  const size_t smem = (size_t)(2 + QB) * m * Traits<E>::es * sizeof(double);
  auto kern = k_mgs_pipe<E, NQ, QB>;
  PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  if (per_sm <= 0) return false;
  const int grid = std::min(per_sm * num_sms(), n + 1);
  w.ready.ensure((size_t)(n + 1) * sizeof(int));
  PN_CHECK_CUDA(cudaMemsetAsync(w.ready.p, 0, (size_t)(n + 1) * sizeof(int), st));
  int *ready = w.ready.as<int>();
  // PN_PIPE_LATE bit 0: late prefetch (no closing barrier per apply): cdd
  // factorisation 16.13 -> 15.99 ms at m = 1024; but cd 5.05 -> 7.46 ms and
  // cdd at m = 512 / 768 4.14 -> 5.65 / 9.05 -> 13.94 ms (shorter applies no
  // longer cover the column copy), so double double with four row blocks
  // only (profiles/r02/exp ab8/ab9/ab51).  Bit 1: the two-barrier pivot wait
  // instead of the one-barrier one.
  const char *lv = getenv("PN_PIPE_LATE");
  int late = lv ? atoi(lv) : (Traits<E>::nc == 2 && NQ == 4 ? 1 : 0);
  void *args[] = {&A, &m, &n, &orig, (void *)&eps, &Q, &R, &status, &ready, &late};
  unsigned long long *tr = nullptr;
  trace_begin(n, &tr);
  PN_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)kern, grid, 256, args, smem, st));
  trace_end(n, tr, st);
  count_launch(1);
  return true;
}

// k_mgs_small: the whole factorisation in one CTA for m <= 32 (config C1
// and the small systems of the tests).  [A b] sits in shared memory as
// component planes (row = lane, conflict-free); warp w owns columns w,
// w + NW, ...; per pivot the owner computes r_kk and q_k, one barrier, every
// warp sweeps its later columns, one barrier.  Sums over rows are the warp
// shuffle tree with right pruning = tree_sum's order (mgs.py:145-221); no
// inter-CTA flags, so a pivot costs its arithmetic chain plus two barriers.
template <class E, int NT>
__global__ void __launch_bounds__(NT) k_mgs_small(const double *__restrict__ A, int m, int n, double eps,
                                                   double *__restrict__ Q, double *__restrict__ R,
                                                   MgsStatus *status) {
  using Rl = typename Traits<E>::R;
  constexpr int es = Traits<E>::es;
  extern __shared__ __align__(16) double ms_smem[];
  __shared__ double s_orig[64];
  __shared__ int s_fail;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int ncol = n + 1, P = ncol * 32;
  auto get = [&](int j) {
    E v;
    double *d = reinterpret_cast<double *>(&v);
#pragma unroll
    for (int c = 0; c < es; ++c) d[c] = ms_smem[c * P + j * 32 + lane];
    return v;
  };
  auto put = [&](int j, const E &v) {
    const double *d = reinterpret_cast<const double *>(&v);
#pragma unroll
    for (int c = 0; c < es; ++c) ms_smem[c * P + j * 32 + lane] = d[c];
  };
  // tree_sum over rows 0..m-1 of one value per lane, result on every lane
  auto wsum = [&](auto v) {
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const auto o = eshfl_down(v, s);
      if ((lane & (2 * s - 1)) == 0 && lane + s < m) v = eadd(v, o);
    }
    return eshfl_idx(v, 0);
  };
  auto norm = [&](int j) -> Rl { return fsqrt(wsum(lane < m ? eabs2(get(j)) : ezero<Rl>())); };
  if (threadIdx.x == 0) s_fail = 0;
  for (int j = w; j < ncol; j += NW) put(j, lane < m ? eload<E>(A + ((long long)j * m + lane) * es) : ezero<E>());
  __syncthreads();
  for (int j = w; j < n; j += NW) {  // initial column norms (mgs.py:171-172)
    const Rl nrm = norm(j);
    if (lane == 0) s_orig[j] = nrm.c[0];
  }
  __syncthreads();
  for (int k = 0; k <= n; ++k) {
    if (w == k % NW) {  // pivot k (mgs.py:176-193); k == n is the residual norm z
      const Rl rkk = norm(k);
      bool ok = true;
      if (k < n) {
        const double thr = __dmul_rn(__dmul_rn(__dmul_rn(1.0, (double)n), eps), s_orig[k]);
        if (rkk.c[0] <= thr) {
          ok = false;
          if (lane == 0) {
            status->k = k;
            status->rkk = rkk.c[0];
            status->thr = thr;
            status->code = PN_E_BREAKDOWN;
            s_fail = 1;
          }
        }
      }
      if (ok) {
        if (lane == 0) estore(R + ((long long)k * ncol + k) * es, eembed(rkk, (E *)nullptr));
        if (k < n) {
          const RDiv<Traits<E>::nc> p = rdiv_prepare(rkk);
          const E q = ediv_prepared(get(k), p);
          put(k, q);
          if (lane < m) estore(Q + ((long long)k * m + lane) * es, q);
        }
      }
    }
    __syncthreads();
    if (s_fail || k == n) break;
    for (int j = w; j < ncol; j += NW) {  // sweep k over the later columns (mgs.py:201-215)
      if (j <= k) continue;
      const E q = get(k), a = get(j);
      const E r = wsum(lane < m ? emul(econj(q), a) : ezero<E>());
      if (lane < m) put(j, esub(a, emul(q, r)));
      if (lane == 0) estore(R + ((long long)j * ncol + k) * es, r);
    }
    __syncthreads();
  }
}

template <class E, int B>
static void mgs_run(int m, int n, double *A, double *Q, double *R, MgsWork &w, cudaStream_t st) {
  MgsStatus *status = w.status.as<MgsStatus>();
  double *orig = w.orig.d();
  const double eps = level_eps(Traits<E>::nc);
  const int sms = num_sms();
  int mode = mgs_mode(Traits<E>::nc);
  // one CTA for m <= 32 (default for d/dd: C1 cd step 0.231 -> 0.176 ms;
  // qd keeps the dataflow kernel, whose 33 CTAs sweep the columns in
  // parallel: 1.07 vs 1.14 ms; PN_MGS_MODE=small forces it, larger m take
  // the default schedule)
  const bool mode_set = getenv("PN_MGS_MODE") != nullptr;
  if (m <= 32 && (mode == 5 || (!mode_set && Traits<E>::nc <= 2))) {
    const size_t smem = (size_t)Traits<E>::es * (n + 1) * 32 * sizeof(double);
    // plain double: a warp per column (up to 32); dd/qd: 16 warps (registers)
    constexpr int NT = Traits<E>::nc == 1 ? 1024 : 512;
    auto kern = k_mgs_small<E, NT>;
    if (smem > 48 * 1024) PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nt = std::min(NT, 32 * (n + 1));
    kern<<<1, nt, smem, st>>>(A, m, n, eps, Q, R, status);
    PN_CHECK_LAUNCH();
    count_launch(1);
    return;
  }
  if (mode == 5) mode = Traits<E>::nc == 4 ? 0 : 4;
  if (mode == 4 && Traits<E>::nc <= 2 && m % 256 == 0 && m <= 1024) {
    bool done = false;
    switch (m / 256) {
      case 1: done = pipe_launch<E, 1>(m, n, A, Q, R, w, st); break;
      case 2: done = pipe_launch<E, 2>(m, n, A, Q, R, w, st); break;
      case 3: done = pipe_launch<E, 3>(m, n, A, Q, R, w, st); break;
      default: done = pipe_launch<E, 4>(m, n, A, Q, R, w, st); break;
    }
    if (done) return;
  }
  // complex dd with 1024 < m <= 2048 rows: the flow kernel (8 rows per
  // thread, two CTAs per SM) instead of the dataflow kernel: factorisation
  // 80.3 -> 57.3 ms at 1536 rows, 153 -> 115 ms at 2048, Chandrasekhar
  // n = 2048 cdd (6 steps) 0.944 -> 0.718 s; complex double stays on the
  // dataflow kernel (24.3 vs 29.5 ms at 1536), above 2048 rows the wide flow
  // kernel wins (profiles/r02/exp ab43/ab44).  PN_FLOW_TALL=0 keeps dataflow.
  if (mode == 4 && Traits<E>::nc == 2 && Traits<E>::cplx && m > 1024 && m <= 2048) {
    const char *ft = getenv("PN_FLOW_TALL"), *fw = getenv("PN_FLOW_WIDE");
    if (!(ft && strcmp(ft, "0") == 0) && !(fw && strcmp(fw, "1") == 0)) mode = 0;
  }
  if (mode == 0) {
    // 6 warps x 8 rows for 1024 < m <= 1536 (the C4 overdetermined shape):
    // a 96 KB column, two CTAs per SM instead of one 128 KB CTA
    if constexpr (B == 8) {
      if (m <= 1536 && flow_launch<E, B, 192>(m, n, A, Q, R, w, st)) return;
    }
    // qd with 3/4 of the CTA's rows used (256 < m <= 384, 512 < m <= 768):
    // 192-thread CTAs instead of 256 with a quarter of the threads idle --
    // cqd factorisation at 768 rows 71.4 -> 61.0 ms (profiles/r02/exp ab62).
    // PN_FLOW_192=0 keeps 256 threads.
    if constexpr ((B == 4 || B == 2) && Traits<E>::nc == 4) {
      const char *f3 = getenv("PN_FLOW_192");
      if (!(f3 && atoi(f3) == 0) && m > 128 * B && m <= 192 * B && flow_launch<E, B, 192>(m, n, A, Q, R, w, st))
        return;
    }
    // real qd, 2048 < m <= 4096 (Chandrasekhar real qd): the column fills
    // one CTA's shared memory either way; 16 warps x 8 rows instead of 8 x 16
    // (PN_FLOW_WIDE=0 keeps the 256-thread CTA)
    if constexpr (B == 16 && Traits<E>::nc == 4 && !Traits<E>::cplx) {
      const char *fw = getenv("PN_FLOW_WIDE");
      const bool wide = fw ? strcmp(fw, "0") != 0 : true;
      // up to 3072 rows: 384 threads x 8 rows fill the CTA (Chandrasekhar
      // real qd n = 3048: 5.75 -> 5.59 s; PN_FLOW_384=0 keeps 512)
      const char *f3 = getenv("PN_FLOW_384");
      if (wide && m > 2048 && m <= 3072 && !(f3 && atoi(f3) == 0) && flow_launch<E, 8, 384>(m, n, A, Q, R, w, st))
        return;
      if (wide && m > 2048 && flow_launch<E, 8, 512>(m, n, A, Q, R, w, st)) return;
    }
    if (flow_launch<E, B, kMgsThreads>(m, n, A, Q, R, w, st)) return;
  }
  // d/dd columns of 2048 < m <= 4096 rows: the flow kernel with 1024-thread
  // CTAs (4 rows per thread, the working column in shared memory, one CTA
  // per SM) instead of the streaming dataflow kernel -- Chandrasekhar
  // n = 4096 cdd, 6 Newton steps 9.9 -> 6.2 s (equal at 2048).  Complex dd:
  // 512 threads x 8 rows (128 registers instead of 64): factorisation 3072
  // rows 431.7 -> 408.6 ms, 4096 rows 951 -> 890 ms; complex double keeps
  // 1024 x 4 (154.6 vs 212.8 ms at 3072; profiles/r02/exp ab46).
  // PN_FLOW_WIDE=0|1|2 forces dataflow / 1024 threads / 512 threads.
  if (mode == 4 && Traits<E>::nc <= 2 && m > 1024 && m <= 4096) {
    const char *fw = getenv("PN_FLOW_WIDE");
    const int wide = fw ? atoi(fw) : (m > 2048 ? (Traits<E>::nc == 2 && Traits<E>::cplx ? 2 : 1) : 0);
    if constexpr (B == 16 && Traits<E>::nc == 2) {
      // up to 3072 rows: 384 threads x 8 rows (Chandrasekhar cdd n = 3072:
      // 2.50 -> 2.45 s; PN_FLOW_384=0 keeps 512)
      const char *f3 = getenv("PN_FLOW_384");
      if (wide == 2 && m <= 3072 && !(f3 && atoi(f3) == 0) && flow_launch<E, 8, 384>(m, n, A, Q, R, w, st)) return;
      if (wide == 2 && flow_launch<E, 8, 512>(m, n, A, Q, R, w, st)) return;
    }
    if (wide && flow_launch<E, 4, 1024>(m, n, A, Q, R, w, st)) return;
  }
  if (mode <= 1 || mode == 4) {
    int per_sm = 0;
    PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs_dataflow<E, B>, kMgsThreads, 0));
    if (per_sm > 0) {
      w.ready.ensure((size_t)(n + 1) * sizeof(int));
      PN_CHECK_CUDA(cudaMemsetAsync(w.ready.p, 0, (size_t)(n + 1) * sizeof(int), st));
      int *ready = w.ready.as<int>();
      const int grid = std::min(per_sm * sms, n + 1);
      void *args[] = {&A, &m, &n, &orig, (void *)&eps, &Q, &R, &status, &ready};
      unsigned long long *tr = nullptr;
      trace_begin(n, &tr);
      PN_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_mgs_dataflow<E, B>, grid, kMgsThreads, args, 0, st));
      trace_end(n, tr, st);
      count_launch(1);
      return;
    }
  }
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


// ---------------------------------------------------------------------------
// Back substitution R x = y, y = R[:n, n] (mgs.py:229-247), over 32-row
// diagonal blocks from the bottom, one cooperative launch with one grid
// barrier per block.  Every row receives its subtractions in descending
// column order, so x is bit-identical to the reference's sequential solve.
//
// Lane-parallel arithmetic for complex quad double: the solve is a chain of
// n dependent complex-qd operations; a single lane issues a complex multiply
// in ~4300 cycles (profiles/r01/micro_fp64.txt) because its four qd products
// share one instruction stream.  In k_backsub_look four lanes own a row and
// compute the four real products of every complex multiply side by side
// (then two lanes form re = t1 - t2 and im = t3 + t4), which shortens the
// chain about 2.5x.  The reference's operation sequence is unchanged
// (xprec.py:302-306, varith.py:130-136).

template <int NC>
__device__ __forceinline__ F<NC> shfl_fn(const F<NC> &v, int src) {
  F<NC> r;
#pragma unroll
  for (int i = 0; i < NC; ++i) r.c[i] = __shfl_sync(0xffffffffu, v.c[i], src);
  return r;
}
template <int NC>
__device__ __forceinline__ F<NC> shfl_xor_fn(const F<NC> &v, int mask) {
  F<NC> r;
#pragma unroll
  for (int i = 0; i < NC; ++i) r.c[i] = __shfl_xor_sync(0xffffffffu, v.c[i], mask);
  return r;
}
// a*b on a group of four lanes (p = lane & 3): p0 ar*br, p1 ai*bi, p2 ar*bi,
// p3 ai*br; re = t1 - t2 on p0, im = t3 + t4 on p2.  Every lane of the warp
// must call it (full-mask shuffles); all four lanes get the result.
template <int NC>
__device__ __forceinline__ C<NC> lp_cmul(const C<NC> &a, const C<NC> &b, int p, int g4) {
  const F<NC> x = (p == 0 || p == 2) ? a.re : a.im;
  const F<NC> y = (p == 0 || p == 3) ? b.re : b.im;
  const F<NC> prod = fmul(x, y);
  const F<NC> other = shfl_xor_fn(prod, 1);
  const F<NC> v = fadd(prod, p == 0 ? fneg(other) : other);
  return {shfl_fn(v, g4), shfl_fn(v, g4 + 2)};
}
// a - b: p0 re, p1 im
template <int NC>
__device__ __forceinline__ C<NC> lp_csub(const C<NC> &a, const C<NC> &b, int p, int g4) {
  const F<NC> v = fadd((p & 1) ? a.im : a.re, fneg((p & 1) ? b.im : b.re));
  return {shfl_fn(v, g4), shfl_fn(v, g4 + 1)};
}
// y / r as (y * conj r) * recip(|r|^2) (varith.py:130-136 with the hoisted reciprocal)
template <int NC>
__device__ __forceinline__ C<NC> lp_div(const C<NC> &yv, const C<NC> &r, const RDiv<NC> &pr, int p, int g4) {
  const C<NC> num = lp_cmul(yv, cconj(r), p, g4);
  const F<NC> v = rdiv_apply((p & 1) ? num.im : num.re, pr);
  return {shfl_fn(v, g4), shfl_fn(v, g4 + 1)};
}


// k_backsub_look (complex qd): CTA 0 has two 128-thread groups: the solver
// (rows of block b,
// four lanes per row) and a lookahead group holding the 32 rows of block b-1,
// which subtracts R[i, j] x_j for each x_j of block b as soon as the solver
// has it (two updates per solver step), after first catching up on block
// b+1's x.  The other CTAs apply block b+1's x to every row below block b-1
// meanwhile.  Every row still takes its updates in descending j (blocks b+2..
// from the other CTAs in earlier rounds, then b+1 and b from the lookahead
// group); the solver never waits for a separate next-block pass
// (mgs.py:229-247).  (The plain lanes kernel without the lookahead group:
// 5.2 vs 3.7 ms at n = 1024, removed.)
template <int NC>
__global__ void __launch_bounds__(256) k_backsub_look(const double *__restrict__ R, int n, double *__restrict__ x,
                                                      RDiv<NC> *__restrict__ prep, double *__restrict__ y,
                                                      int *sing, MgsStatus *status) {
  namespace cg = cooperative_groups;
  using E = C<NC>;
  constexpr int es = 2 * NC;
  constexpr int NT = 256;
  extern __shared__ __align__(16) double lk_smem[];
  E *sD = reinterpret_cast<E *>(lk_smem);  // R[lo+ii, lo+jj] at jj*32+ii (diagonal block b)
  E *sU = sD + 32 * 32;                     // R[lo-32+ii, lo+jj]    (block b-1 rows, block b columns)
  E *sV = sU + 32 * 32;                     // R[lo-32+ii, lo+32+jj] (block b-1 rows, block b+1 columns)
  E *sX = sV + 32 * 32;                     // [2][32]: x of block b at parity b & 1
  E *sY = sX + 64;                          // block b-1 rows after the lookahead
  RDiv<NC> *sP = reinterpret_cast<RDiv<NC> *>(sY + 32);
  __shared__ __align__(8) uint64_t s_xbar[32];  // x_j of step s of a block is in sX
  cg::grid_group grid = cg::this_grid();
  if (status->code) return;
  if (blockIdx.x == 0 && threadIdx.x < 32) mbar_init(&s_xbar[threadIdx.x], 1);  // only CTA 0 hands off
  const long long ld = n + 1;
  const int gtid = blockIdx.x * NT + threadIdx.x, gsize = gridDim.x * NT;
  for (int j = gtid; j < n; j += gsize) {
    estore(y + (long long)j * es, eload<E>(R + ((long long)n * ld + j) * es));
    const double *dg = R + ((long long)j * ld + j) * es;
    bool nz = false;
#pragma unroll
    for (int q = 0; q < es; ++q) nz |= dg[q] != 0.0;
    if (!nz) atomicMax(sing, j);
    else prep[j] = rdiv_prepare(ediv_den(eload<E>(dg)));
  }
  grid.sync();
  if (*(volatile int *)sing >= 0) {
    if (gtid == 0) {
      status->k = *sing;
      status->code = PN_E_SINGULAR;
    }
    return;
  }
  const int t = threadIdx.x, tt = t & 127, lane = t & 31, p = lane & 3, g4 = lane & ~3;
  const bool solver = t < 128;
  const int rl = tt >> 2;
  const int nb = (n + 31) / 32;
  for (int b = nb - 1; b >= 0; --b) {
    const int lo = b * 32, hi = min(n, lo + 32), nbk = hi - lo;
    const int par = b & 1;
    if (blockIdx.x == 0) {
      // catch-up columns (block b+1) and lookahead rows exist only for b > 0
      const int ncu = (b > 0 && b + 1 < nb) ? min(n, lo + 64) - (lo + 32) : 0;
      if (solver) {
        for (int e = tt; e < 32 * 32; e += 128) {
          const int jj = e >> 5, ii = e & 31;
          if (jj < nbk && ii <= jj) sD[e] = eload<E>(R + ((long long)(lo + jj) * ld + lo + ii) * es);
        }
        if (tt < nbk) sP[tt] = prep[lo + tt];
      } else if (b > 0) {
        for (int e = tt; e < 32 * 32; e += 128) {
          const int jj = e >> 5, ii = e & 31;
          if (jj < nbk) sU[e] = eload<E>(R + ((long long)(lo + jj) * ld + lo - 32 + ii) * es);
          if (jj < ncu) sV[e] = eload<E>(R + ((long long)(lo + 32 + jj) * ld + lo - 32 + ii) * es);
        }
      }
      __syncthreads();
      E yr = ezero<E>(), v = ezero<E>();
      if (solver) {
        if (rl < nbk) yr = b == nb - 1 ? eload<E>(y + (long long)(lo + rl) * es) : sY[rl];
      } else if (b > 0) {
        v = eload<E>(y + (long long)(lo - 32 + rl) * es);
      }
      int q = 0;  // lookahead group's next update
      auto look = [&]() {
        if (q < ncu) {
          const int jj = ncu - 1 - q;
          v = lp_csub(v, lp_cmul(sV[jj * 32 + rl], sX[(par ^ 1) * 32 + jj], p, g4), p, g4);
        } else {
          const int jj = nbk - 1 - (q - ncu);
          v = lp_csub(v, lp_cmul(sU[jj * 32 + rl], sX[par * 32 + jj], p, g4), p, g4);
        }
        ++q;
      };
      __syncthreads();  // sY was read before the lookahead group rewrites it
      const int pblk = nb - 1 - b, n0 = n - 32 * (nb - 1);  // processing index; rows of the first block
      if (solver) {
        // the solver's steps sync on a named barrier of its 128 threads; the
        // lookahead group follows the step slots instead
        for (int s = 0; s < nbk; ++s) {
          const int jl = nbk - 1 - s;
          if ((jl >> 3) == (tt >> 5)) {
            const E xj = lp_div(yr, sD[jl * 32 + jl], sP[jl], p, g4);
            if (rl == jl && p == 0) {
              sX[par * 32 + jl] = xj;
              if (b > 0) xslot_arrive(&s_xbar[s]);  // block 0 has no lookahead group
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if ((tt >> 5) * 8 < jl) {
            const E u = lp_csub(yr, lp_cmul(sD[jl * 32 + rl], sX[par * 32 + jl], p, g4), p, g4);
            if (rl < jl) yr = u;
          }
        }
      } else if (b > 0) {
        // block b+1's x first, then block b's as the solver publishes them
        while (q < ncu) look();
        for (int s = 0; s < nbk; ++s) {
          xslot_wait(&s_xbar[s], xslot_parity(pblk, s, n0));
          look();
        }
        if (p == 0) sY[rl] = v;
      }
      __syncthreads();
      if (solver && tt < nbk) estore(x + (long long)(lo + tt) * es, sX[par * 32 + tt]);
    } else if (b + 1 < nb) {
      // rows below block b-1 take block b+1's x (descending columns)
      const int c0 = lo + 32, nc1 = min(n, lo + 64) - c0;
      for (int r = gtid - NT; r < lo - 32; r += gsize - NT) {
        E v = eload<E>(y + (long long)r * es);
#pragma unroll 4
        for (int jj = 31; jj >= 0; --jj)
          if (jj < nc1)
            v = esub(v, emul(eload<E>(R + ((long long)(c0 + jj) * ld + r) * es), eload<E>(x + (long long)(c0 + jj) * es)));
        estore(y + (long long)r * es, v);
      }
    }
    grid.sync();
  }
}

// k_backsub_blocked_look (d, dd, real qd): one lane per row with the
// lookahead of k_backsub_look: warp 0 of CTA 0 solves block b, warp 1 holds
// block b-1's rows, applies block b+1's x and then block b's x_j as warp 0
// publishes them; the rest of the grid applies block b+1's x to the rows
// below block b-1.  The solver's operands (diagonal block, the blocks above
// it, the hoisted reciprocals) are staged in shared memory with all loads in
// flight at once, so the sequential chain never waits on L2.
template <class E, int NT>
__global__ void __launch_bounds__(NT) k_backsub_blocked_look(const double *__restrict__ R, int n,
                                                             double *__restrict__ x,
                                                             RDiv<Traits<E>::nc> *__restrict__ prep,
                                                             double *__restrict__ y, int *sing, MgsStatus *status) {
  namespace cg = cooperative_groups;
  using RD = RDiv<Traits<E>::nc>;
  constexpr int es = Traits<E>::es;
  extern __shared__ __align__(16) double bk_smem[];
  E *sD = reinterpret_cast<E *>(bk_smem);  // R[lo+ii, lo+jj] at jj*32+ii
  E *sU = sD + 32 * 32;                     // R[lo-32+ii, lo+jj]
  E *sV = sU + 32 * 32;                     // R[lo-32+ii, lo+32+jj]
  E *sX = sV + 32 * 32;                     // [2][32]
  E *sY = sX + 64;                          // block b-1 rows after the lookahead
  RD *sP = reinterpret_cast<RD *>(sY + 32);
  __shared__ __align__(8) uint64_t s_xbar[32];  // x_j of step s of a block is in sX
  cg::grid_group grid = cg::this_grid();
  if (status->code) return;
  if (blockIdx.x == 0 && threadIdx.x < 32) mbar_init(&s_xbar[threadIdx.x], 1);  // only CTA 0 hands off
  const long long ld = n + 1;
  const int gtid = blockIdx.x * NT + threadIdx.x, gsize = gridDim.x * NT;
  for (int j = gtid; j < n; j += gsize) {
    estore(y + (long long)j * es, eload<E>(R + ((long long)n * ld + j) * es));
    const double *dg = R + ((long long)j * ld + j) * es;
    bool nz = false;
#pragma unroll
    for (int p = 0; p < es; ++p) nz |= dg[p] != 0.0;
    if (!nz) atomicMax(sing, j);
    else prep[j] = rdiv_prepare(ediv_den(eload<E>(dg)));
  }
  grid.sync();
  if (*(volatile int *)sing >= 0) {
    if (gtid == 0) {
      status->k = *sing;
      status->code = PN_E_SINGULAR;
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (n + 31) / 32;
  for (int b = nb - 1; b >= 0; --b) {
    const int lo = b * 32, hi = min(n, lo + 32), nbk = hi - lo;
    const int par = b & 1;
    if (blockIdx.x == 0) {
      const int ncu = (b > 0 && b + 1 < nb) ? min(n, lo + 64) - (lo + 32) : 0;
      // stage the blocks with every thread of the CTA, all loads independent
      for (int e = threadIdx.x; e < 32 * 32; e += NT) {
        const int jj = e >> 5, ii = e & 31;
        if (jj < nbk && ii <= jj) sD[e] = eload<E>(R + ((long long)(lo + jj) * ld + lo + ii) * es);
        if (b > 0 && jj < nbk) sU[e] = eload<E>(R + ((long long)(lo + jj) * ld + lo - 32 + ii) * es);
        if (jj < ncu) sV[e] = eload<E>(R + ((long long)(lo + 32 + jj) * ld + lo - 32 + ii) * es);
      }
      if (threadIdx.x < nbk) sP[threadIdx.x] = prep[lo + threadIdx.x];
      __syncthreads();
      const int pblk = nb - 1 - b, n0 = n - 32 * (nb - 1);  // processing index; rows of the first block
      if (warp == 0) {
        E yr = ezero<E>();
        if (lane < nbk) yr = b == nb - 1 ? eload<E>(y + (long long)(lo + lane) * es) : sY[lane];
        __syncwarp();
        E xl = ezero<E>();
        for (int s = 0; s < nbk; ++s) {
          const int jl = nbk - 1 - s;
          if (lane == jl) {
            xl = ediv_with(yr, sD[jl * 32 + jl], sP[jl]);
            sX[par * 32 + jl] = xl;
            if (b > 0) xslot_arrive(&s_xbar[s]);  // block 0 has no lookahead warp
          }
          const E xj = eshfl_idx(xl, jl);
          if (lane < jl) yr = esub(yr, emul(sD[jl * 32 + lane], xj));
        }
        if (lane < nbk) estore(x + (long long)(lo + lane) * es, xl);
      } else if (warp == 1 && b > 0) {
        E v = eload<E>(y + (long long)(lo - 32 + lane) * es);
        for (int jj = ncu - 1; jj >= 0; --jj) v = esub(v, emul(sV[jj * 32 + lane], sX[(par ^ 1) * 32 + jj]));
        for (int s = 0; s < nbk; ++s) {
          const int jl = nbk - 1 - s;
          xslot_wait(&s_xbar[s], xslot_parity(pblk, s, n0));
          v = esub(v, emul(sU[jl * 32 + lane], sX[par * 32 + jl]));
        }
        sY[lane] = v;
      }
      __syncthreads();
    } else if (b + 1 < nb) {
      const int c0 = lo + 32, nc1 = min(n, lo + 64) - c0;
      for (int r = gtid - NT; r < lo - 32; r += gsize - NT) {
        E v = eload<E>(y + (long long)r * es);
#pragma unroll 4
        for (int jj = 31; jj >= 0; --jj)
          if (jj < nc1)
            v = esub(v, emul(eload<E>(R + ((long long)(c0 + jj) * ld + r) * es), eload<E>(x + (long long)(c0 + jj) * es)));
        estore(y + (long long)r * es, v);
      }
    }
    grid.sync();
  }
}

template <class E>
void backsub_impl(int n, const double *R, double *x, MgsWork &w, cudaStream_t st) {
  constexpr int es = Traits<E>::es;
  DevBuf prep((size_t)n * Traits<E>::nc * sizeof(double) + 16, st);
  // PN_BACKSUB_MODE=single: one CTA, n <= 1024 (tests); default: lookahead
  const char *mode = getenv("PN_BACKSUB_MODE");
  const bool look = !(mode && strcmp(mode, "single") == 0);
  // complex qd: four lanes per row.  Complex dd measured slower with lanes
  // (1.18 vs 1.0 ms at n = 1024): its chain is short already.
  if constexpr (Traits<E>::cplx && Traits<E>::nc == 4) {
    constexpr int NC = Traits<E>::nc;
    if (look) {
      constexpr int NT = 256;
      DevBuf yw((size_t)n * es * sizeof(double) + 16, st);
      DevBuf sbuf(16, st);
      int *sing = sbuf.as<int>();
      PN_CHECK_CUDA(cudaMemsetAsync(sing, 0xff, sizeof(int), st));
      const int grid = std::max(2, std::min(num_sms(), (n + NT - 1) / NT + 1));
      RDiv<NC> *pp = prep.as<RDiv<NC>>();
      double *yp = yw.d();
      MgsStatus *status = w.status.as<MgsStatus>();
      void *args[] = {(void *)&R, &n, &x, &pp, &yp, &sing, &status};
      const size_t smem = (size_t)(3 * 32 * 32 + 96) * es * sizeof(double) + 32 * sizeof(RDiv<NC>);
      PN_CHECK_CUDA(cudaFuncSetAttribute(k_backsub_look<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      PN_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_backsub_look<NC>, grid, NT, args, smem, st));
      count_launch(1);
      return;
    }
  }
  if (look) {
    constexpr int NT = 128;
    DevBuf yw((size_t)n * es * sizeof(double) + 16, st);
    DevBuf sbuf(16, st);
    int *sing = sbuf.as<int>();
    PN_CHECK_CUDA(cudaMemsetAsync(sing, 0xff, sizeof(int), st));
    const int grid = std::max(2, std::min(num_sms(), (n + NT - 1) / NT + 1));
    RDiv<Traits<E>::nc> *pp = prep.as<RDiv<Traits<E>::nc>>();
    double *yp = yw.d();
    MgsStatus *status = w.status.as<MgsStatus>();
    void *args[] = {(void *)&R, &n, &x, &pp, &yp, &sing, &status};
    const size_t smem = (size_t)(3 * 32 * 32 + 96) * es * sizeof(double) + 32 * sizeof(RDiv<Traits<E>::nc>);
    auto kern = k_backsub_blocked_look<E, NT>;
    PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PN_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)kern, grid, NT, args, smem, st));
    count_launch(1);
    return;
  }
  constexpr int NT = kBacksubThreads;
  PN_REQUIRE(n <= NT * 4, PN_E_ARG, "single-CTA back substitution supports n <= %d", NT * 4);
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
