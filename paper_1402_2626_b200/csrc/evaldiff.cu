// evaldiff.cu -- subsystems (1)+(2): monomial evaluation with reverse-mode
// differentiation on binary product trees, and the fixed-order accumulation
// of values and Jacobian entries.
//
// Reference: evaluate_system (evaldiff.py:215-266), eval_monomial_and_derivs
// (142-180), eval_product_tree (53-73), gradient_from_tree (76-108),
// _tree_reduce (205-212), build_power_table / eval_common_factor
// (polyrep.py:120-139).
//
// Kernels
//   K0 k_power_table : x_v^d for d = 1..maxdeg_v (one thread per variable)
//   K1 k_mono_small  : k <= 1 monomials (constant, single-variable bypass)
//   K1 k_mono_tree   : 2 <= k <= 32; a group of G lanes per monomial.  Lane
//                      r owns tree nodes t == r (mod G): the low levels of
//                      the sequential-addressing tree are lane-local, the top
//                      log2(G) levels are butterflies over warp shuffles
//                      (every lane computes its node redundantly, so no lane
//                      idles and the downward sweep needs one shuffle per
//                      level).  Operand order is the reference's (lower index
//                      on the left), so results are bit-identical.
//   K1 k_mono_large  : k > 32 (e.g. cyclic n-roots): one CTA per monomial,
//                      tree levels in shared memory (the paper's scheme)
//   K2 k_segments    : one thread per output entry; a binary-counter fold of
//                      the entry's contributions reproduces tree_sum's
//                      right-pruned pairwise order exactly.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace pn {

// Batched evaluation (config C5): blockIdx.y selects a batch slot; each slot
// has its own point, power table, contribution buffer, f and [J | -f].  The
// single-system path uses one slot with zero strides.
__device__ __forceinline__ long long bslot(const BView &v) {
  return v.slots ? (long long)v.slots[blockIdx.y] : (long long)blockIdx.y;
}

// ---------------------------------------------------------------------------
// K0

template <class E>
__global__ void k_power_table(int n, const double *__restrict__ x, const int32_t *__restrict__ toff,
                              const int32_t *__restrict__ tdeg, double *__restrict__ table, BView bv) {
  constexpr int es = Traits<E>::es;
  const long long b = bslot(bv);
  x += b * bv.x;
  table += b * bv.t;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int deg = tdeg[v];
  if (deg == 0) return;
  const E xv = eload<E>(x + (long long)v * es);
  double *row = table + (long long)toff[v] * es;
  E cur = xv;
  estore(row, cur);
  for (int d = 2; d <= deg; ++d) {
    cur = emul(cur, xv);  // row[d] = row[d-1] * x (polyrep.py:128)
    estore(row + (long long)(d - 1) * es, cur);
  }
}

// ---------------------------------------------------------------------------
// K1, k <= 1

template <class E>
__global__ void k_mono_small(const int32_t *__restrict__ list, long long count, const int32_t *__restrict__ mon_ptr,
                             const int32_t *__restrict__ var, const int32_t *__restrict__ exps,
                             const int32_t *__restrict__ dst, const double *__restrict__ coeff,
                             const double *__restrict__ table, const int32_t *__restrict__ toff,
                             double *__restrict__ contrib, BView bv) {
  constexpr int es = Traits<E>::es;
  const long long b = bslot(bv);
  table += b * bv.t;
  contrib += b * bv.c;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < count;
       g += (long long)gridDim.x * blockDim.x) {
    const int c = list[g];
    const int lo = mon_ptr[c], k = mon_ptr[c + 1] - lo;
    const E co = eload<E>(coeff + (long long)c * es);
    if (k == 0) {  // evaldiff.py:152-153
      estore(contrib + (long long)c * es, co);
      continue;
    }
    // single-variable bypass, evaldiff.py:156-165
    const int v = var[lo], d = exps[lo];
    const double *row = table + (long long)toff[v] * es;
    const E value = emul(co, eload<E>(row + (long long)(d - 1) * es));
    const E dco = emul_int(co, d);
    const E deriv = (d == 1) ? dco : emul(dco, eload<E>(row + (long long)(d - 2) * es));
    estore(contrib + (long long)c * es, value);
    estore(contrib + (long long)dst[lo] * es, deriv);
  }
}

// scale = coeff [* common]; common = left fold of x_v^(d-1) over d >= 2
// (polyrep.py:133-139, evaldiff.py:168)
// support entries: plain (PK = 0: variable / exponent arrays) or packed
// (PK = 1, k_eval_rows: var | chunk slot << 16 | exponent << 28)
template <int PK> __device__ __forceinline__ int ent_var(int e) { return PK ? (e & 0xffff) : e; }
template <int PK> __device__ __forceinline__ int ent_exp(int e) { return PK ? (int)((unsigned)e >> 28) : e; }
template <int PK> __device__ __forceinline__ int ent_slot(int e) { return PK ? (int)(((unsigned)e >> 16) & 0xfff) : e; }

template <class E, int PK = 0>
__device__ __forceinline__ E monomial_scale(const E &co, int lo, int k, const int32_t *__restrict__ var,
                                            const int32_t *__restrict__ exps, const double *__restrict__ table,
                                            const int32_t *__restrict__ toff) {
  constexpr int es = Traits<E>::es;
  bool have = false;
  E common;
  for (int p = 0; p < k; ++p) {
    const int d = ent_exp<PK>(exps[lo + p]);
    if (d < 2) continue;
    const E pw = eload<E>(table + ((long long)toff[ent_var<PK>(var[lo + p])] + d - 2) * es);
    common = have ? emul(common, pw) : pw;
    have = true;
  }
  return have ? emul(co, common) : co;
}

// ---------------------------------------------------------------------------
// K1, 2 <= k <= 32: G lanes per monomial, BASE = 2^floor(log2 k)

template <int V> struct Log2 { static constexpr int value = 1 + Log2<V / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

// One monomial with 2 <= k <= 32 on a group of G lanes (lane r of the group
// passes r).  mv / me: the monomial's variable indices and exponents (global
// or shared memory).
// Results go through two sinks: value(v) on lane 0 of the group and
// deriv(t, v) for every support position t of the monomial.  Inactive
// groups (active == false) run the shuffles but emit nothing.
template <class E, int BASE, int G, int PK = 0, bool XSM = false, class VSink, class DSink>
__device__ __forceinline__ void mono_tree_eval(int r, bool active, int k, const int32_t *mv, const int32_t *me,
                                               const E &co, const double *__restrict__ x,
                                               const double *__restrict__ table, const int32_t *__restrict__ toff,
                                               VSink &&value_sink, DSink &&deriv_sink, bool unit = false) {
  constexpr int es = Traits<E>::es;
  constexpr int SL = BASE / G;            // slots per lane
  constexpr int NLOC = Log2<SL>::value;   // lane-local levels above the slots
  constexpr int NX = Log2<G>::value;      // butterfly levels
  constexpr int NLV = SL > 1 ? SL - 1 : 1;
  static_assert(BASE >= G && G >= 2 && G <= 32, "bad tree config");
  const int ell = k - BASE;

  // PK: mv / me hold packed entries (ent_var / ent_exp); XSM: x is in shared memory
  auto leaf = [&](int t) -> E {
    const double *p = x + (long long)ent_var<PK>(mv[t]) * es;
    if constexpr (XSM) return eload<E>(p);
    else return eload_ldg<E>(p);
  };
  // slot t of level 0: v[t] * v[BASE+t] for t < ell, else v[t] (evaldiff.py:63-65)
  auto slot = [&](int t) -> E {
    E v = leaf(t);
    if (t < ell) v = emul(v, leaf(BASE + t));
    return v;
  };

  // ---- upward sweep (evaldiff.py:67-72) --------------------------------
  // lv holds lane-local levels 1..NLOC; level j has SL>>j entries at
  // offset SL - (SL >> (j-1)); entry u is global node r + G*u.
  E lv[NLV];
  E X[NX + 1];
  if constexpr (NLOC == 0) {
    X[0] = slot(r);
  } else {
#pragma unroll
    for (int u = 0; u < SL / 2; ++u) lv[u] = emul(slot(r + G * u), slot(r + G * (u + SL / 2)));
#pragma unroll
    for (int j = 2; j <= NLOC; ++j) {
      const int oprev = SL - (SL >> (j - 2)), ocur = SL - (SL >> (j - 1)), h = SL >> j;
#pragma unroll
      for (int u = 0; u < h; ++u) lv[ocur + u] = emul(lv[oprev + u], lv[oprev + u + h]);
    }
    X[0] = lv[SL - 2];
  }
  // butterflies: level of size S = G >> q; lane r holds node r mod S
#pragma unroll
  for (int q = 1; q <= NX; ++q) {
    const int S = G >> q;
    const E other = eshfl_xor(X[q - 1], S);
    const bool low = (r & (2 * S - 1)) < S;  // lower index stays the left operand
    X[q] = emul(low ? X[q - 1] : other, low ? other : X[q - 1]);
  }
  const E root = X[NX];

  // ---- value (evaldiff.py:166-172) ---------------------------------------
  // unit: every exponent is 1 (the bucket was checked on upload), so the
  // common factor is empty and scale == co
  const E scale = unit ? co : monomial_scale<E, PK>(co, 0, k, mv, me, table, toff);
  if (active && r == 0) value_sink(emul(scale, root));

  // ---- downward sweep of complements (evaldiff.py:89-98) -----------------
  // complement of this lane's node at the current level
  E cmp = eshfl_xor(X[NX - 1], 1);  // comp = [L[1], L[0]] at the size-2 level
#pragma unroll
  for (int q = NX - 2; q >= 0; --q) {
    const int S = G >> (q + 1);
    cmp = emul(cmp, eshfl_xor(X[q], S));
  }
  // lane-local levels: comp_{j-1}[u] = comp_j[u] * L_{j-1}[u+h],
  //                    comp_{j-1}[u+h] = comp_j[u] * L_{j-1}[u]
  E cl[SL];
  if constexpr (NLOC == 0) {
    cl[0] = cmp;
  } else {
    lv[SL - 2] = cmp;  // complement of the level-NLOC node (size G)
#pragma unroll
    for (int j = NLOC; j >= 2; --j) {
      const int ocur = SL - (SL >> (j - 1)), oprev = SL - (SL >> (j - 2)), h = SL >> j;
#pragma unroll
      for (int u = 0; u < h; ++u) {
        const E cu = lv[ocur + u];
        const E lo_ = emul(cu, lv[oprev + u + h]);
        const E hi_ = emul(cu, lv[oprev + u]);
        lv[oprev + u] = lo_;
        lv[oprev + u + h] = hi_;
      }
    }
    // level 1 -> slots
#pragma unroll
    for (int u = 0; u < SL / 2; ++u) {
      const E cu = lv[u];
      cl[u] = emul(cu, slot(r + G * (u + SL / 2)));
      cl[u + SL / 2] = emul(cu, slot(r + G * u));
    }
  }

  // ---- unfold folded pairs and scale (evaldiff.py:100-108, 174-180) -------
  if (!active) return;
#pragma unroll
  for (int u = 0; u < SL; ++u) {
    const int t = r + G * u;
    if (t < ell) {
      const int t2 = BASE + t;
      const E g1 = emul(cl[u], leaf(t2));
      const E g2 = emul(cl[u], leaf(t));
      const int d1 = unit ? 1 : ent_exp<PK>(me[t]), d2 = unit ? 1 : ent_exp<PK>(me[t2]);
      const E s1 = d1 == 1 ? scale : emul_int(scale, d1);
      const E s2 = d2 == 1 ? scale : emul_int(scale, d2);
      deriv_sink(t, emul(s1, g1));
      deriv_sink(t2, emul(s2, g2));
    } else {
      const int d1 = unit ? 1 : ent_exp<PK>(me[t]);
      const E s1 = d1 == 1 ? scale : emul_int(scale, d1);
      deriv_sink(t, emul(s1, cl[u]));
    }
  }
}

template <class E, int BASE, int G, int NT>
__global__ void __launch_bounds__(NT) k_mono_tree(const int32_t *__restrict__ list, long long count,
                                                  const int32_t *__restrict__ mon_ptr,
                                                  const int32_t *__restrict__ var, const int32_t *__restrict__ exps,
                                                  const int32_t *__restrict__ dst, const double *__restrict__ coeff,
                                                  const double *__restrict__ x, const double *__restrict__ table,
                                                  const int32_t *__restrict__ toff, double *__restrict__ contrib,
                                                  BView bv) {
  constexpr int es = Traits<E>::es;
  {
    const long long b = bslot(bv);
    x += b * bv.x;
    table += b * bv.t;
    contrib += b * bv.c;
  }
  const long long grp = (blockIdx.x * (long long)NT + threadIdx.x) / G;
  const int r = threadIdx.x % G;
  const bool active = grp < count;
  const int c = list[active ? grp : count - 1];
  const int lo = mon_ptr[c], k = mon_ptr[c + 1] - lo;
  const E co = eload<E>(coeff + (long long)c * es);
  mono_tree_eval<E, BASE, G>(
      r, active, k, var + lo, exps + lo, co, x, table, toff,
      [&](const E &v) { estore(contrib + (long long)c * es, v); },
      [&](int t, const E &v) { estore(contrib + (long long)dst[lo + t] * es, v); });
}

// ---------------------------------------------------------------------------
// lanes per monomial of the K1 trees, by precision

template <class E> struct TreeG;  // lanes per monomial, by precision
#ifndef PN_TREE_G_DD
#define PN_TREE_G_DD 8  // cdd: 8 lanes per monomial (fewer registers, 3 CTAs/SM) measured faster than 4
#endif
template <int NC> struct TreeG<F<NC>> { static constexpr int value = NC == 4 ? 8 : 4; };
template <int NC> struct TreeG<C<NC>> { static constexpr int value = NC == 4 ? 8 : NC == 2 ? PN_TREE_G_DD : 4; };

// binary-counter stack: level l of the stack lives at st[l * stride]
template <class E>
__device__ __forceinline__ void stack_push(E *st, int stride, int cnt, E v) {
  int l = 0;
  while ((cnt >> l) & 1) {
    v = eadd(st[l * stride], v);  // the older (lower-index) block stays on the left
    ++l;
  }
  st[l * stride] = v;
}

template <class E>
__device__ __forceinline__ E stack_fold(const E *st, int stride, int cnt) {
  int l = __ffs(cnt) - 1;
  E acc = st[l * stride];
  for (++l; l < 31; ++l)
    if ((cnt >> l) & 1) acc = eadd(st[l * stride], acc);
  return acc;
}

// ---------------------------------------------------------------------------
// K1 with TMA-staged supports (dense uniform buckets: every monomial of the
// bucket has k = K and the bucket's support entries are one contiguous block,
// as for the C2/C4/C5 systems).  Persistent CTAs walk chunks of CH = NT/G
// monomials; a chunk's variable indices, exponents, contribution slots and
// canonical indices arrive in shared memory by cp.async.bulk on an mbarrier,
// double buffered, so the next chunk's supports stream in while the current
// chunk's trees compute and no lane waits on a dependent index load.  The
// arithmetic is mono_tree_eval, identical to k_mono_tree.
template <class E, int BASE, int G, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) k_mono_tree_tma(const int32_t *__restrict__ list, long long count, int K,
                                                      long long e0, const int32_t *__restrict__ var,
                                                      const int32_t *__restrict__ exps,
                                                      const int32_t *__restrict__ dst, const double *__restrict__ coeff,
                                                      const double *__restrict__ x, const double *__restrict__ table,
                                                      const int32_t *__restrict__ toff, double *__restrict__ contrib,
                                                      BView bv, bool unit) {
  constexpr int es = Traits<E>::es;
  constexpr int CH = NT / G;
  extern __shared__ __align__(16) int tma_smem[];
  __shared__ __align__(8) uint64_t bar[2];
  const int L = CH * K;                        // ints per array per stage (multiple of 4)
  int *st_var = tma_smem;                      // [2][L]
  int *st_exp = st_var + 2 * L;                // [2][L]
  int *st_dst = st_exp + 2 * L;                // [2][L]
  int *st_lst = st_dst + 2 * L;                // [2][CH]
  {
    const long long b = bslot(bv);
    x += b * bv.x;
    table += b * bv.t;
    contrib += b * bv.c;
  }
  const long long nchunks = (count + CH - 1) / CH;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long long ch, int s) {  // thread 0: stage chunk ch into buffer s
    const long long m0 = ch * CH;
    const int cnt = (int)min((long long)CH, count - m0);
    const uint32_t lb = (uint32_t)((cnt * 4 + 15) & ~15);
    const long long ebeg = e0 + m0 * K;
    const uint32_t sb = (uint32_t)(((long long)cnt * K * 4 + 15) & ~15LL);
    mbar_expect_tx(&bar[s], 3 * sb + lb);
    bulk_g2s(st_var + s * L, var + ebeg, sb, &bar[s]);
    bulk_g2s(st_exp + s * L, exps + ebeg, sb, &bar[s]);
    bulk_g2s(st_dst + s * L, dst + ebeg, sb, &bar[s]);
    bulk_g2s(st_lst + s * CH, list + m0, lb, &bar[s]);
  };
  long long ch = blockIdx.x;
  if (ch < nchunks && tid == 0) issue(ch, 0);
  uint32_t phase[2] = {0, 0};
  for (int s = 0; ch < nchunks; ch += gridDim.x, s ^= 1) {
    const long long nxt = ch + gridDim.x;
    if (nxt < nchunks && tid == 0) issue(nxt, s ^ 1);  // buffer s^1 was released by the last barrier
    mbar_wait(&bar[s], phase[s]);
    phase[s] ^= 1;
    const long long m0 = ch * CH;
    const int u = tid / G, r = tid % G;
    const bool active = m0 + u < count;
    const int uu = active ? u : 0;
    const int *mv = st_var + s * L + uu * K;
    const int *me = st_exp + s * L + uu * K;
    const int *md = st_dst + s * L + uu * K;
    const int c = st_lst[s * CH + uu];
    const E co = eload<E>(coeff + (long long)c * es);
    mono_tree_eval<E, BASE, G>(
        r, active, K, mv, me, co, x, table, toff, [&](const E &v) { estore(contrib + (long long)c * es, v); },
        [&](int t, const E &v) { estore(contrib + (long long)md[t] * es, v); }, unit);
    __syncthreads();  // buffer s is free for the chunk after next
  }
}

// ---------------------------------------------------------------------------
// K1, k > 32: one CTA per monomial, tree levels in shared memory

template <class E, int NT>
__global__ void __launch_bounds__(NT) k_mono_large(const int32_t *__restrict__ list, long long count,
                                                   const int32_t *__restrict__ mon_ptr,
                                                   const int32_t *__restrict__ var, const int32_t *__restrict__ exps,
                                                   const int32_t *__restrict__ dst, const double *__restrict__ coeff,
                                                   const double *__restrict__ x, const double *__restrict__ table,
                                                   const int32_t *__restrict__ toff, double *__restrict__ contrib,
                                                   BView bv, double *__restrict__ gscratch, long long gstride) {
  constexpr int es = Traits<E>::es;
  {
    const long long b = bslot(bv);
    x += b * bv.x;
    table += b * bv.t;
    contrib += b * bv.c;
  }
  extern __shared__ __align__(16) double smem[];
  // levels back to back (2*base entries) then base complements; in shared
  // memory when 3*base elements fit, otherwise in a per-CTA slice of global
  // scratch (L2 resident: 3*base*es*8 bytes per CTA), so k is bounded by n only
  E *lvl = gscratch ? reinterpret_cast<E *>(gscratch + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * gstride)
                    : reinterpret_cast<E *>(smem);
  __shared__ E s_scale;
  for (long long g = blockIdx.x; g < count; g += gridDim.x) {
    const int c = list[g];
    const int lo = mon_ptr[c], k = mon_ptr[c + 1] - lo;
    int base = 1;
    while (base * 2 <= k) base *= 2;
    const int ell = k - base;
    const int32_t *__restrict__ mv = var + lo;
    auto leaf = [&](int t) -> E { return eload_ldg<E>(x + (long long)mv[t] * es); };
    for (int t = threadIdx.x; t < base; t += NT) {
      E v = leaf(t);
      if (t < ell) v = emul(v, leaf(base + t));
      lvl[t] = v;
    }
    __syncthreads();
    // level offsets: level j starts at 2*base - (2*base >> j)
    int off = 0;
    for (int size = base; size > 1; size >>= 1) {
      const int s = size / 2;
      for (int t = threadIdx.x; t < s; t += NT) lvl[off + size + t] = emul(lvl[off + t], lvl[off + t + s]);
      off += size;
      __syncthreads();
    }
    const E root = lvl[off];
    // common factor only when some exponent is >= 2 (one parallel pass)
    bool multi_t = false;
    for (int t = threadIdx.x; t < k; t += NT) multi_t |= exps[lo + t] >= 2;
    const bool multi = __syncthreads_or(multi_t);
    if (threadIdx.x == 0) {
      const E co = eload<E>(coeff + (long long)c * es);
      const E scale = multi ? monomial_scale<E>(co, lo, k, var, exps, table, toff) : co;
      s_scale = scale;
      estore(contrib + (long long)c * es, emul(scale, root));
    }
    // complements, in place over a separate buffer of base entries
    E *cmp = lvl + 2 * base;
    // size-2 level starts at off - 2
    if (threadIdx.x == 0) {
      cmp[0] = lvl[off - 2 + 1];
      cmp[1] = lvl[off - 2];
    }
    __syncthreads();
    int o2 = off - 2;  // offset of the size-2 level
    for (int s = 2; s < base; s <<= 1) {
      const int oprev = o2 - 2 * s;  // level of size 2s
      for (int t = threadIdx.x; t < s; t += NT) {
        const E ct = cmp[t];
        const E a = emul(ct, lvl[oprev + t + s]);
        const E b = emul(ct, lvl[oprev + t]);
        cmp[t] = a;
        cmp[t + s] = b;
      }
      o2 = oprev;
      __syncthreads();
    }
    const E scale = s_scale;
    for (int t = threadIdx.x; t < base; t += NT) {
      if (t < ell) {
        const int t2 = base + t;
        const E g1 = emul(cmp[t], leaf(t2));
        const E g2 = emul(cmp[t], leaf(t));
        const int d1 = exps[lo + t], d2 = exps[lo + t2];
        estore(contrib + (long long)dst[lo + t] * es, emul(d1 == 1 ? scale : emul_int(scale, d1), g1));
        estore(contrib + (long long)dst[lo + t2] * es, emul(d2 == 1 ? scale : emul_int(scale, d2), g2));
      } else {
        const int d1 = exps[lo + t];
        estore(contrib + (long long)dst[lo + t] * es, emul(d1 == 1 ? scale : emul_int(scale, d1), cmp[t]));
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K1, 32 < k: one WARP per monomial (cyclic n-roots, the paper's large
// products).  Same tree and operand order as k_mono_large, but the levels
// live in a warp-private slice of shared memory and the warp synchronises
// with __syncwarp only, so monomials of different warps proceed
// independently and no CTA-wide barrier idles 256 threads on the top levels
// of one tree.  The complements overwrite the levels in place (both
// children of a node are read before either is written); for dd/qd level 0
// is recomputed from x instead of stored, so a monomial needs base - 1
// elements (qd base 256: 16 KB, twelve warps per SM; cyclic 448-roots qd
// 23.6 -> 20.6 ms), for d 2 * base; trees too wide for six warps per SM
// take k_mono_large.
template <class E, int NW, bool LEAN>
__global__ void __launch_bounds__(NW * 32) k_mono_warp(const int32_t *__restrict__ list, long long count, int base,
                                                       const int32_t *__restrict__ mon_ptr,
                                                       const int32_t *__restrict__ var, const int32_t *__restrict__ exps,
                                                       const int32_t *__restrict__ dst, const double *__restrict__ coeff,
                                                       const double *__restrict__ x, const double *__restrict__ table,
                                                       const int32_t *__restrict__ toff, double *__restrict__ contrib,
                                                       BView bv) {
  constexpr int es = Traits<E>::es;
  {
    const long long b = bslot(bv);
    x += b * bv.x;
    table += b * bv.t;
    contrib += b * bv.c;
  }
  extern __shared__ __align__(16) double wsmem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // LEAN (dd, qd): levels 1.. only (base - 1 elements; level 0 -- the slots --
  // is recomputed from x when the complements reach it); otherwise (d,
  // where the extra loads cost more than the storage saves) levels 0.. in
  // 2 * base elements.  The complements then overwrite the levels in place.
  E *lvl = reinterpret_cast<E *>(wsmem) + (size_t)w * (LEAN ? base : 2 * base);
  const long long nwarps = (long long)gridDim.x * NW;
  const int h0 = base / 2;  // size of level 1 (base >= 64 here)
  for (long long g = blockIdx.x * (long long)NW + w; g < count; g += nwarps) {
    const int c = list[g];
    const int lo = mon_ptr[c], k = mon_ptr[c + 1] - lo;
    const int ell = k - base;  // every monomial of the bucket has floor_pow2(k) == base
    const int32_t *__restrict__ mv = var + lo;
    auto leaf = [&](int t) -> E { return eload_ldg<E>(x + (long long)mv[t] * es); };
    // slot t of level 0 (evaldiff.py:63-65): v[t] * v[base+t] for t < ell
    auto slot = [&](int t) -> E {
      E v = leaf(t);
      if (t < ell) v = emul(v, leaf(base + t));
      return v;
    };
    // upward sweep (evaldiff.py:67-72): each level stored right after the
    // previous one, starting with level 1 (LEAN) or level 0
    int off = 0;
    if constexpr (LEAN) {
      for (int t = lane; t < h0; t += 32) lvl[t] = emul(slot(t), slot(t + h0));
    } else {
      for (int t = lane; t < base; t += 32) lvl[t] = slot(t);
    }
    __syncwarp();
    for (int size = LEAN ? h0 : base; size > 1; size >>= 1) {
      const int h = size / 2;
      for (int t = lane; t < h; t += 32) lvl[off + size + t] = emul(lvl[off + t], lvl[off + t + h]);
      off += size;
      __syncwarp();
    }
    const E root = lvl[off];
    const E co = eload<E>(coeff + (long long)c * es);
    // the common factor (polyrep.py:133-139) only when an exponent is >= 2:
    // one coalesced pass of the warp over the exponents decides it
    bool multi = false;
    for (int t = lane; t < k; t += 32) multi |= exps[lo + t] >= 2;
    const E scale = __any_sync(0xffffffffu, multi) ? monomial_scale<E>(co, lo, k, var, exps, table, toff) : co;
    if (lane == 0) estore(contrib + (long long)c * es, emul(scale, root));
    // downward sweep of complements (evaldiff.py:89-98), in place: the
    // size-2 level's pair becomes [L1, L0], then each level's pair (t, t+h)
    // is replaced by (cmp[t] * L[t+h], cmp[t] * L[t]) down to level 1
    int o2 = off - 2;
    if (lane == 0) {
      const E a0 = lvl[o2], a1 = lvl[o2 + 1];
      lvl[o2] = a1;
      lvl[o2 + 1] = a0;
    }
    __syncwarp();
    for (int h = 2; h < (LEAN ? h0 : base); h <<= 1) {
      const int oprev = o2 - 2 * h;  // level of size 2h
      for (int t = lane; t < h; t += 32) {
        const E ct = lvl[o2 + t];
        const E a = lvl[oprev + t], b2 = lvl[oprev + t + h];
        lvl[oprev + t] = emul(ct, b2);
        lvl[oprev + t + h] = emul(ct, a);
      }
      o2 = oprev;
      __syncwarp();
    }
    // level 0's complements from level 1's and the recomputed slots, then
    // unfold folded pairs and scale (evaldiff.py:100-108, 174-180)
    auto emit = [&](int t, const E &cm) {
      if (t < ell) {
        const int t2 = base + t;
        const E g1 = emul(cm, leaf(t2));
        const E g2 = emul(cm, leaf(t));
        const int d1 = exps[lo + t], d2 = exps[lo + t2];
        estore(contrib + (long long)dst[lo + t] * es, emul(d1 == 1 ? scale : emul_int(scale, d1), g1));
        estore(contrib + (long long)dst[lo + t2] * es, emul(d2 == 1 ? scale : emul_int(scale, d2), g2));
      } else {
        const int d1 = exps[lo + t];
        estore(contrib + (long long)dst[lo + t] * es, emul(d1 == 1 ? scale : emul_int(scale, d1), cm));
      }
    };
    if constexpr (LEAN) {
      for (int t = lane; t < h0; t += 32) {
        const E c1 = lvl[t];
        const E s0 = slot(t), s1 = slot(t + h0);
        emit(t, emul(c1, s1));
        emit(t + h0, emul(c1, s0));
      }
    } else {
      for (int t = lane; t < base; t += 32) emit(t, lvl[t]);
    }
    __syncwarp();  // the levels are rewritten by the warp's next monomial
  }
}

// ---------------------------------------------------------------------------
// K2: one thread per output entry

template <class E>
__global__ void __launch_bounds__(128) k_segments(long long nseg_total, int m, const int64_t *__restrict__ seg_ptr,
                                                  const int64_t *__restrict__ seg_out,
                                                  const double *__restrict__ contrib, double *__restrict__ f,
                                                  double *__restrict__ A, long long negf_off, BView bv) {
  constexpr int es = Traits<E>::es;
  {
    const long long b = bslot(bv);
    contrib += b * bv.c;
    if (f) f += b * bv.f;
    A += b * bv.a;
  }
  E stk[32];
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nseg_total;
       s += (long long)gridDim.x * blockDim.x) {
    const long long a = seg_ptr[s], b = seg_ptr[s + 1];
    const long long L = b - a;
    E acc;
    if (L == 0) {
      acc = ezero<E>();  // zero_like(point[0]) for an empty polynomial (evaldiff.py:261)
    } else {
      // aligned blocks of 8: eight independent loads in flight, their
      // pairwise tree, pushed at level 3 -- the same as eight level-0 pushes
      long long p = 0;
      for (; p + 8 <= L; p += 8) {
        E v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = eload<E>(contrib + (a + p + q) * es);
#pragma unroll
        for (int q = 0; q < 8; q += 2) v[q] = eadd(v[q], v[q + 1]);
        v[0] = eadd(v[0], v[2]);
        v[4] = eadd(v[4], v[6]);
        E carry = eadd(v[0], v[4]);
        int lvl = 3;
        for (long long q = p >> 3; q & 1; q >>= 1, ++lvl) carry = eadd(stk[lvl], carry);
        stk[lvl] = carry;
      }
      for (; p < L; ++p) {
        E carry = eload<E>(contrib + (a + p) * es);
        int lvl = 0;
        for (long long q = p; q & 1; q >>= 1, ++lvl) carry = eadd(stk[lvl], carry);
        stk[lvl] = carry;
      }
      int l = __ffsll(L) - 1;
      acc = stk[l];
      for (++l; l < 32; ++l)
        if ((L >> l) & 1) acc = eadd(stk[l], acc);
    }
    if (s < m) {
      if (f) estore(f + s * es, acc);
      if (negf_off >= 0) estore(A + (negf_off + s) * es, eneg(acc));
    } else {
      estore(A + seg_out[s - m] * es, acc);
    }
  }
}

// ---------------------------------------------------------------------------
// K1+K2 per polynomial in one CTA (k_eval_rows, plan in pn_system::Rows):
// no contribution buffer in HBM.  A persistent CTA takes whole polynomials;
// polynomial i is evaluated in chunks of CH = NT/G canonical monomials
// (aligned power-of-two blocks):
//   * the chunk's packed support entries (var | slot << 16) arrive in shared
//     memory by a bulk copy issued one chunk ahead (double buffered, mbarrier);
//   * mono_tree_eval (identical arithmetic to K1, x staged in shared memory)
//     stores every derivative at its slot of the chunk buffer, where the
//     chunk's contributions are ordered by (variable, canonical monomial);
//   * every variable j then pushes its run of the chunk, in order, onto its
//     own binary-counter stack in shared memory (level l of variable j at
//     stk[l * n + j]) -- the streaming form of tree_sum's right-pruned
//     pairwise order, so the Jacobian entry folded from the stack
//     at the end is bit-identical to K2's fold of the contiguous run;
//   * the chunk's monomial values are reduced by the tree's lower levels
//     (warp shuffles, then the warps' partials) and pushed at chunk
//     granularity onto a value stack.
// The row of J is written once (exact zeros included, evaldiff.py:262), f_i
// and -f_i once.  HBM traffic is the packed supports, the coefficients and
// the row: the memory-bound complex-double evaluation no longer writes and
// re-reads (M + nnz) contributions.

// push the run p[0, L) onto a binary-counter stack whose count is c: in
// aligned blocks of up to 8 (the pairwise node of an aligned block is what
// the element-wise pushes would build), each block pushed at its level --
// bit-identical to L element pushes with fewer stack round trips
template <class E>
__device__ __forceinline__ void run_push(E *st, int stride, int c, const E *p, int L) {
  int q = 0;
  while (q < L) {
    const int cq = c + q;
    int l = 0;
    while (l < 3 && ((cq >> l) & 1) == 0 && q + (2 << l) <= L) ++l;
    E v;
    if (l == 0) {
      v = p[q];
    } else if (l == 1) {
      v = eadd(p[q], p[q + 1]);
    } else if (l == 2) {
      v = eadd(eadd(p[q], p[q + 1]), eadd(p[q + 2], p[q + 3]));
    } else {
      v = eadd(eadd(eadd(p[q], p[q + 1]), eadd(p[q + 2], p[q + 3])),
               eadd(eadd(p[q + 4], p[q + 5]), eadd(p[q + 6], p[q + 7])));
    }
    int lvl = l;
    for (int k = cq >> l; k & 1; k >>= 1, ++lvl) v = eadd(st[lvl * stride], v);
    st[lvl * stride] = v;
    q += 1 << l;
  }
}

// in-place right-pruned pairwise tree over p[0, L) (tree_sum order, P4)
template <class E>
__device__ __forceinline__ E run_tree_inplace(E *p, int L) {
  for (int s = 1; s < L; s <<= 1)
    for (int a = 0; a + s < L; a += 2 * s) p[a] = eadd(p[a], p[a + s]);
  return p[0];
}

template <class E, int BASE, int G, int NT, bool XSM>
__global__ void __launch_bounds__(NT) k_eval_rows(int m, int n, int K, int D, const int64_t *__restrict__ poly_ptr,
                                                  const int32_t *__restrict__ mon_ptr,
                                                  const uint32_t *__restrict__ ent, const int32_t *__restrict__ exps,
                                                  const int32_t *__restrict__ poly_chunk,
                                                  const int4 *__restrict__ desc,
                                                  const uint16_t *__restrict__ runoff,
                                                  const double *__restrict__ coeff, const double *__restrict__ x,
                                                  const double *__restrict__ table, const int32_t *__restrict__ toff,
                                                  const double *__restrict__ consts, long long cstride,
                                                  double *__restrict__ f, double *__restrict__ A, int negf_col,
                                                  bool unit, BView bv) {
  constexpr int es = Traits<E>::es;
  constexpr int CH = NT / G;           // monomials per chunk
  constexpr int NW = NT / 32;
  constexpr int VL = RowsLayout::VL;  // value-stack levels (chunk granularity)
  const int LE = RowsLayout::le(CH, K);  // staged entries per buffer
  extern __shared__ __align__(16) double rows_smem[];
  __shared__ __align__(8) uint64_t bar[2];
  const RowsLayout Lo = rows_layout(n, D, K, es, CH, BASE, NW, XSM);
  char *sb = reinterpret_cast<char *>(rows_smem);
  E *xs = reinterpret_cast<E *>(sb + Lo.xs);            // n (when XSM)
  E *stk = reinterpret_cast<E *>(sb + Lo.stk);          // D x n
  E *buf = reinterpret_cast<E *>(sb + Lo.buf);          // CH * K chunk contributions (by variable, monomial)
  E *vals = reinterpret_cast<E *>(sb + Lo.vals);        // CH monomial values
  E *wpart = reinterpret_cast<E *>(sb + Lo.wpart);      // NW warp partials
  E *vstk = reinterpret_cast<E *>(sb + Lo.vstk);        // VL
  int *cnt = reinterpret_cast<int *>(sb + Lo.cnt);      // n
  uint32_t *sent = reinterpret_cast<uint32_t *>(sb + Lo.sent);  // [2][LE] packed entries
  int *smp = reinterpret_cast<int *>(sb + Lo.smp);      // [2][lmp] mon_ptr of the chunk
  double *scf = reinterpret_cast<double *>(sb + Lo.scf);  // [2][lcf] coefficients of the chunk
  uint16_t *sro = reinterpret_cast<uint16_t *>(sb + Lo.sro);  // [2][rs] run starts of the chunk
  int *pad = reinterpret_cast<int *>(sb + Lo.pad);      // 2 * BASE: var 0 / exponent 1 for idle groups
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long b = bslot(bv);
  x += b * bv.x;
  table += b * bv.t;
  A += b * bv.a;
  if (XSM)
    for (int v = tid; v < n; v += NT) xs[v] = eload<E>(x + (long long)v * es);
  if (tid < 2 * BASE) pad[tid] = 1 << 28;  // packed: variable 0, slot 0, exponent 1
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const double *xsrc = XSM ? reinterpret_cast<const double *>(xs) : x;

  // Producer (thread 0): stages the CTA's chunks (polynomials blockIdx.x,
  // +gridDim.x, ...) one chunk ahead -- packed entries, mon_ptr, coefficients
  // and the variables' run starts, four bulk copies on one mbarrier -- with
  // the next chunk's descriptor and the next polynomial's chunk range loaded
  // one step earlier still, so no dependent global load sits on the path.
  int q_i = blockIdx.x - (int)gridDim.x, q_g = 0, q_ge = 0;
  int q_ni = blockIdx.x, q_nlo = 0, q_nhi = 0;
  bool have = false;
  int4 dnext = make_int4(0, 0, 0, 0);
  auto prod_next = [&]() -> bool {
    if (q_g + 1 < q_ge) {
      ++q_g;
      return true;
    }
    for (;;) {
      q_i = q_ni;
      if (q_i >= m) return false;
      q_g = q_nlo;
      q_ge = q_nhi;
      q_ni = q_i + gridDim.x;
      if (q_ni < m) {
        q_nlo = poly_chunk[q_ni];
        q_nhi = poly_chunk[q_ni + 1];
      }
      if (q_g < q_ge) return true;
    }
  };
  auto issue = [&](int s) {  // stage chunk q_g (descriptor dnext) into buffer s
    if (!have) return;
    const int4 d = dnext;  // {c0, U, e0, e1}
    const long long c0 = d.x, a0 = d.z & ~3LL, m0 = c0 & ~3LL, f0 = (c0 * es) & ~1LL;
    // at least 16 bytes (a chunk of constants has no entries; every array carries 16 bytes of padding)
    const uint32_t be = (uint32_t)max(16LL, ((d.w - a0) * 4 + 15) & ~15LL);
    const uint32_t bm = (uint32_t)(((c0 + d.y + 1 - m0) * 4 + 15) & ~15LL);
    const uint32_t bc = (uint32_t)((((c0 + d.y) * es - f0) * 8 + 15) & ~15LL);
    const uint32_t br = (uint32_t)(Lo.rs * 2);
    // the buffer's previous contents were read through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[s], be + bm + bc + br);
    bulk_g2s(sent + s * LE, ent + a0, be, &bar[s]);
    bulk_g2s(smp + s * Lo.lmp, mon_ptr + m0, bm, &bar[s]);
    bulk_g2s(scf + s * Lo.lcf, coeff + f0, bc, &bar[s]);
    bulk_g2s(sro + s * Lo.rs, runoff + (long long)q_g * Lo.rs, br, &bar[s]);
    have = prod_next();
    if (have) dnext = desc[q_g];
  };
  if (tid == 0) {
    if (q_ni < m) {
      q_nlo = poly_chunk[q_ni];
      q_nhi = poly_chunk[q_ni + 1];
    }
    have = prod_next();
    if (have) dnext = desc[q_g];
    issue(0);
  }
  uint32_t phase[2] = {0, 0};
  int s = 0;

  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const long long p0 = poly_ptr[i];
    const int T = (int)(poly_ptr[i + 1] - p0);
    const int nch = (T + CH - 1) / CH;
    for (int j = tid; j < n; j += NT) cnt[j] = 0;
    E value = ezero<E>();  // f_i; zero_like for an empty polynomial (evaldiff.py:261)
    for (int c = 0; c < nch; ++c, s ^= 1) {
      // stage the chunk after this one into the other buffer (released by the
      // barrier that ended the previous chunk)
      if (tid == 0) issue(s ^ 1);
      const long long c0 = p0 + (long long)c * CH;
      const int U = min(CH, T - c * CH);
      mbar_wait(&bar[s], phase[s]);
      phase[s] ^= 1;
      const int *mp = smp + s * Lo.lmp + (int)(c0 & 3);        // mon_ptr[c0 + u] = mp[u]
      const double *cf = scf + s * Lo.lcf + (int)((c0 * es) & 1);  // coefficient u at cf + u * es
      const int e0 = mp[0], shift = e0 & 3;
      // ---- trees: group u of G lanes takes monomial u of the chunk
      const int u = tid / G, r = tid % G;
      const int uu = u < U ? u : 0;
      const int lo = mp[uu] - e0 + shift, k = mp[uu + 1] - mp[uu];
      const bool tree = u < U && k > 0;
      if (u < U && k == 0 && r == 0)  // constant term (evaldiff.py:152-153); per-start shift if given
        vals[u] = consts ? eload<E>(consts + b * cstride + (long long)i * es) : eload<E>(cf + uu * es);
      const int32_t *mv = tree ? reinterpret_cast<const int32_t *>(sent + s * LE + lo) : pad;
      const E co = tree ? eload<E>(cf + uu * es) : ezero<E>();
      mono_tree_eval<E, BASE, G, 1, XSM>(
          r, tree, tree ? k : BASE, mv, mv, co, xsrc, table, toff, [&](const E &v) { vals[u] = v; },
          [&](int t, const E &v) { buf[ent_slot<1>(mv[t])] = v; }, unit);
      __syncthreads();
      // ---- pushes: variable j's run of this chunk, in canonical order
      const uint16_t *ro = sro + s * Lo.rs;
      for (int j = tid; j < n; j += NT) {
        const int a = ro[j], L = ro[j + 1] - a;
        if (L == 0) continue;
        run_push(stk + j, n, cnt[j], buf + a, L);
        cnt[j] += L;
      }
      // ---- values: the chunk's node of tree_sum (aligned block of CH)
      {
        E v = tid < U ? vals[tid] : ezero<E>();
        if (warp * 32 < U) {
#pragma unroll
          for (int w = 1; w < 32; w <<= 1) {
            const E o = eshfl_down(v, w);
            if ((lane & (2 * w - 1)) == 0 && lane + w < U - warp * 32) v = eadd(v, o);
          }
          if (lane == 0) wpart[warp] = v;
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int P = (U + 31) / 32;
        E v = run_tree_inplace(wpart, P);
        if (c + 1 < nch) {
          stack_push(vstk, 1, c, v);
        } else {  // last chunk: fold the chunk-level counter (c full chunks)
          E acc = v;
          for (int l = 0; l < VL; ++l)
            if ((c >> l) & 1) acc = eadd(vstk[l], acc);
          value = acc;
        }
      }
    }
    __syncthreads();
    // ---- the row: J[i, :] column-major (ld = m), f_i, -f_i
    for (int j = tid; j < n; j += NT) {
      const int L = cnt[j];
      estore(A + ((long long)j * m + i) * es, L ? stack_fold(stk + j, n, L) : ezero<E>());
    }
    if (tid == 0) {
      if (f) estore(f + b * bv.f + (long long)i * es, value);
      if (negf_col >= 0) estore(A + ((long long)negf_col * m + i) * es, eneg(value));
    }
    __syncthreads();  // cnt / stacks are reset by the next polynomial
  }
}

template <class E, int BASE>
static size_t rows_smem(const pn_system *sys, int NT, int G, bool xsm) {
  return rows_layout(sys->n, sys->rows.D, sys->rows.K, Traits<E>::es, NT / G, BASE, NT / 32, xsm).total;
}

template <class E, int BASE>
static void launch_rows(pn_system *sys, const double *x, const double *table, double *f, double *A, int negf_col,
                        int nb, const BView &bv, const double *consts, long long cstride, cudaStream_t st) {
  constexpr int G = rows_g(Traits<E>::nc, Traits<E>::cplx, BASE);
  constexpr int NT = rows_nt(Traits<E>::nc);
  const auto &R = sys->rows;
  // x in shared memory when it fits beside the stacks
  const bool xsm = rows_smem<E, BASE>(sys, NT, G, true) <= kRowsSmemMax;
  const size_t smem = rows_smem<E, BASE>(sys, NT, G, xsm);
  auto kern = xsm ? k_eval_rows<E, BASE, G, NT, true> : k_eval_rows<E, BASE, G, NT, false>;
  PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  const int want = std::max(1, per_sm * num_sms() / std::max(nb, 1));
  const dim3 grid((unsigned)std::min(sys->m, want), (unsigned)nb);
  kern<<<grid, NT, smem, st>>>(sys->m, sys->n, R.K, R.D, sys->d_seg_ptr, sys->d_mon_ptr, R.d_ent, sys->d_exp,
                               R.d_poly_chunk, R.d_desc, R.d_runoff, sys->d_coeff, x, table, sys->d_toff, consts, cstride, f,
                               A, negf_col, R.unit, bv);
  PN_CHECK_LAUNCH();
  count_launch(1);
}

// the row path serves systems it was planned for (uniform k, stacks fit);
// PN_EVAL_ROWS=0|1 at call time overrides the default (complex/real
// double: memory-bound; dd/qd keep the FP64-bound K1 + K2 unless forced)
template <class E>
static bool use_rows(const pn_system *sys) {
  if (!sys->rows.ok) return false;
  const char *v = getenv("PN_EVAL_ROWS");
  if (v) return strcmp(v, "0") != 0;
  return Traits<E>::nc == 1;
}

template <class E, int BASE>
static void launch_tree(const pn_system::Bucket &b, pn_system *sys, const double *x, const double *table,
                        double *contrib, int nb, const BView &bv, cudaStream_t st) {
  constexpr int G = TreeG<E>::value < BASE ? TreeG<E>::value : BASE;
  constexpr int NT = 128;
  // dd/qd (compute-bound trees): 4 % faster on the cqd step; plain double is
  // memory-bound and faster with one CTA per chunk (measured, profiles/r01)
  const char *tv = getenv("PN_TREE_TMA");
  const bool tma = tv ? strcmp(tv, "0") != 0 : Traits<E>::nc >= 2;
  if (b.dense_k && tma) {
    constexpr int CH = NT / G;
    // the chunk's supports arrive as one contiguous copy per array (padded
    // rows, KS = G mod 32, removed the 4-way conflicts of the support reads
    // but the per-row bulk copies cost more: C5 4158 -> 3900 start-iter/s,
    // r01; removed)
    const size_t smem = (size_t)(6 * CH * b.dense_k + 2 * CH) * sizeof(int);
    auto kern = k_mono_tree_tma<E, BASE, G, NT>;
    if constexpr (Traits<E>::nc >= 2 && BASE == 32) {
      // register cap for occupancy: qd 3 CTAs per SM (168 registers, cqd
      // eval 11.9 -> 11.3 ms), dd 4 (128 registers, C5 4190 -> 4260
      // start-iterations/s); PN_TREE_MINB=1|3|4 overrides
      const char *mb = getenv("PN_TREE_MINB");
      const int minb = mb ? atoi(mb) : (Traits<E>::nc == 4 ? 3 : 4);
      if (minb == 3) kern = k_mono_tree_tma<E, BASE, G, NT, 3>;
      if (minb == 4) kern = k_mono_tree_tma<E, BASE, G, NT, 4>;
    }
    if (smem > 48 * 1024) PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    const long long nchunks = (b.count + CH - 1) / CH;
    // one resident wave of persistent CTAs (per slot share when batched)
    const long long want = std::max(1LL, (long long)std::max(per_sm, 1) * num_sms() / std::max(nb, 1));
    const dim3 grid((unsigned)std::min(nchunks, want), (unsigned)nb);
    kern<<<grid, NT, smem, st>>>(b.d_list, b.count, b.dense_k, b.e0, sys->d_var, sys->d_exp, sys->d_dst, sys->d_coeff,
                                 x, table, sys->d_toff, contrib, bv, b.unit_exp);
    PN_CHECK_LAUNCH();
    count_launch(1);
    return;
  }
  const long long threads = b.count * G;
  const dim3 grid((unsigned)((threads + NT - 1) / NT), (unsigned)nb);
  k_mono_tree<E, BASE, G, NT><<<grid, NT, 0, st>>>(b.d_list, b.count, sys->d_mon_ptr, sys->d_var, sys->d_exp,
                                                   sys->d_dst, sys->d_coeff, x, table, sys->d_toff, contrib, bv);
  PN_CHECK_LAUNCH();
  count_launch(1);
}

// per-start constant terms (homotopy shifts, newton.py:144-158): after the
// k <= 1 kernel has written every constant monomial's value, slot b's
// constant of polynomial i is replaced by consts[b][i]
template <class E>
__global__ void k_scatter_consts_batch(int m, const int32_t *__restrict__ cpos, const double *__restrict__ consts,
                                       long long cstride, double *__restrict__ contrib, BView bv) {
  constexpr int es = Traits<E>::es;
  const long long b = bslot(bv);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) estore(contrib + b * bv.c + (long long)cpos[i] * es, eload<E>(consts + b * cstride + (long long)i * es));
}

// zero the Jacobian columns of every slot (absent entries are exact zeros,
// evaldiff.py:262); column n (-f) is fully written by k_segments
template <class E>
__global__ void k_zero_jac(long long count, double *__restrict__ A, BView bv) {
  double2 *a = reinterpret_cast<double2 *>(A + bslot(bv) * bv.a);
  const long long n2 = count * Traits<E>::es / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    a[i] = make_double2(0.0, 0.0);
}

// the evaluation pipeline for nb slots (nb = 1, zero strides: one system)
template <class E>
static void evaldiff_run(pn_system *sys, const double *x, double *table, double *contrib, double *f, double *A,
                         long long ldA, int negf_col, int nb, const BView &bv, const int32_t *cpos,
                         const double *consts, long long cstride, cudaStream_t st) {
  constexpr int es = Traits<E>::es;
  if (nb <= 0) return;
  if (sys->table_len > 0) {
    k_power_table<E><<<dim3((sys->n + 127) / 128, nb), 128, 0, st>>>(sys->n, x, sys->d_toff, sys->d_tdeg, table, bv);
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
  if (use_rows<E>(sys)) {
    switch (sys->rows.base) {
      case 2: launch_rows<E, 2>(sys, x, table, f, A, negf_col, nb, bv, consts, cstride, st); break;
      case 4: launch_rows<E, 4>(sys, x, table, f, A, negf_col, nb, bv, consts, cstride, st); break;
      case 8: launch_rows<E, 8>(sys, x, table, f, A, negf_col, nb, bv, consts, cstride, st); break;
      case 16: launch_rows<E, 16>(sys, x, table, f, A, negf_col, nb, bv, consts, cstride, st); break;
      default: launch_rows<E, 32>(sys, x, table, f, A, negf_col, nb, bv, consts, cstride, st); break;
    }
    return;
  }
  for (const auto &b : sys->buckets) {
    if (b.count == 0) continue;
    if (b.kind == 0) {
      const int gx = (int)std::min<long long>((b.count + 127) / 128, std::max(1LL, (long long)num_sms() * 16 / nb));
      k_mono_small<E><<<dim3(gx, nb), 128, 0, st>>>(b.d_list, b.count, sys->d_mon_ptr, sys->d_var, sys->d_exp,
                                                    sys->d_dst, sys->d_coeff, table, sys->d_toff, contrib, bv);
      PN_CHECK_LAUNCH();
      count_launch(1);
    } else if (b.kind == 1) {
      switch (b.base) {
        case 2: launch_tree<E, 2>(b, sys, x, table, contrib, nb, bv, st); break;
        case 4: launch_tree<E, 4>(b, sys, x, table, contrib, nb, bv, st); break;
        case 8: launch_tree<E, 8>(b, sys, x, table, contrib, nb, bv, st); break;
        case 16: launch_tree<E, 16>(b, sys, x, table, contrib, nb, bv, st); break;
        case 32: launch_tree<E, 32>(b, sys, x, table, contrib, nb, bv, st); break;
        default: PN_REQUIRE(false, PN_E_ARG, "internal: bad bucket base %d", b.base);
      }
    } else {
      const int base = b.base;
      // warp per monomial while a warp's levels (2*base elements) leave room
      // for six warps per SM (PN_LARGE_WARP=0: CTA per monomial)
      const char *wv = getenv("PN_LARGE_WARP");
      constexpr bool lean = Traits<E>::nc >= 2;
      const size_t wbytes = (size_t)(lean ? base : 2 * base) * es * sizeof(double);
      if (!(wv && strcmp(wv, "0") == 0) && wbytes * 6 <= 224 * 1024) {
        auto launch = [&](auto kern, int NW) {
          const size_t smem = NW * wbytes;
          if (smem > 48 * 1024)
            PN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int per_sm = 0;
          PN_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem));
          const long long blocks = (b.count + NW - 1) / NW;
          const int gx =
              (int)std::min<long long>(blocks, std::max(1LL, (long long)std::max(per_sm, 1) * num_sms() / nb));
          kern<<<dim3(gx, nb), NW * 32, smem, st>>>(b.d_list, b.count, base, sys->d_mon_ptr, sys->d_var,
                                                    sys->d_exp, sys->d_dst, sys->d_coeff, x, table, sys->d_toff,
                                                    contrib, bv);
        };
        if (wbytes * 8 <= 224 * 1024) launch(k_mono_warp<E, 4, lean>, 4);  // 4 warps per CTA
        else launch(k_mono_warp<E, 2, lean>, 2);                            // 2 per CTA, 3 CTAs per SM
        PN_CHECK_LAUNCH();
        count_launch(1);
        continue;
      }
      size_t smem = (size_t)3 * base * es * sizeof(double);
      constexpr int NT = 256;
      const int gx = (int)std::min<long long>(b.count, std::max(1LL, (long long)num_sms() * 8 / nb));
      double *gscratch = nullptr;
      const long long gstride = 3LL * base * es;
      if (smem > 227 * 1024) {  // levels in global memory (see k_mono_large)
        sys->tree_scratch.ensure((size_t)gx * nb * gstride * sizeof(double));
        gscratch = sys->tree_scratch.d();
        smem = 0;
      } else {
        PN_CHECK_CUDA(cudaFuncSetAttribute(k_mono_large<E, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
      }
      k_mono_large<E, NT><<<dim3(gx, nb), NT, smem, st>>>(b.d_list, b.count, sys->d_mon_ptr, sys->d_var,
                                                          sys->d_exp, sys->d_dst, sys->d_coeff, x, table,
                                                          sys->d_toff, contrib, bv, gscratch, gstride);
      PN_CHECK_LAUNCH();
      count_launch(1);
    }
  }
  if (consts) {
    k_scatter_consts_batch<E><<<dim3((sys->m + 127) / 128, nb), 128, 0, st>>>(sys->m, cpos, consts, cstride, contrib,
                                                                               bv);
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
  // dense Jacobian: absent entries are exact zeros (evaldiff.py:262)
  if (nb == 1 && !bv.slots) {
    PN_CHECK_CUDA(cudaMemsetAsync(A, 0, (size_t)sys->n * ldA * es * sizeof(double), st));
  } else {
    const long long cnt = (long long)sys->n * ldA;
    const int gx = (int)std::min<long long>((cnt * es / 2 + 255) / 256, std::max(1LL, (long long)num_sms() * 8 / nb));
    k_zero_jac<E><<<dim3(gx, nb), 256, 0, st>>>(cnt, A, bv);
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
  const long long total = sys->m + sys->nseg;
  if (total > 0) {
    const int gx = (int)std::min<long long>((total + 127) / 128, std::max(1LL, (long long)num_sms() * 32 / nb));
    k_segments<E><<<dim3(gx, nb), 128, 0, st>>>(total, sys->m, sys->d_seg_ptr, sys->d_seg_out, contrib, f, A,
                                                negf_col >= 0 ? (long long)negf_col * ldA : -1, bv);
    PN_CHECK_LAUNCH();
    count_launch(1);
  }
}

template <class E>
void evaldiff_impl(pn_system *sys, const double *x, double *f, double *A, long long ldA, int negf_col,
                   cudaStream_t st) {
  constexpr int es = Traits<E>::es;
  PN_REQUIRE(ldA == sys->m, PN_E_ARG, "internal: Jacobian leading dimension must equal m");
  sys->contrib.ensure((size_t)(sys->M + sys->nnz) * es * sizeof(double) + 16);
  sys->table.ensure((size_t)(sys->table_len > 0 ? sys->table_len : 1) * es * sizeof(double));
  const BView bv{nullptr, 0, 0, 0, 0, 0};
  evaldiff_run<E>(sys, x, sys->table.d(), sys->contrib.d(), f, A, ldA, negf_col, 1, bv, nullptr, nullptr, 0, st);
}

template <class E>
void evaldiff_batch_impl(pn_system *sys, int nb, const BView &bv, const double *x, double *table, double *contrib,
                         double *f, double *A, int negf_col, const int32_t *cpos, const double *consts,
                         long long cstride, cudaStream_t st) {
  evaldiff_run<E>(sys, x, table, contrib, f, A, sys->m, negf_col, nb, bv, cpos, consts, cstride, st);
}

// one translation unit per precision level (see Makefile): explicit
// instantiation for the level selected by PN_NC / PN_CPLX
#ifdef PN_NC
template void evaldiff_impl<PnLevel>(pn_system *, const double *, double *, double *, long long, int,
                                      cudaStream_t);
template void evaldiff_batch_impl<PnLevel>(pn_system *, int, const BView &, const double *, double *, double *,
                                           double *, double *, int, const int32_t *, const double *, long long,
                                           cudaStream_t);
#endif

}  // namespace pn
