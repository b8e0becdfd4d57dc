// system.cu -- host-side packer for pn_system: validation, canonical monomial
// order, power-table layout, the Jacobian segment map and the k-buckets, plus
// the synthetic system generator.  Integer work only; every floating-point
// operation of the hot path runs in the CUDA kernels.
//
// Reference: PolySystem / Monomial validation (polyrep.py:23-48, 71-107),
// PreparedSystem (evaldiff.py:183-194), decompose (polyrep.py:59-62),
// max_exponent / build_power_table (polyrep.py:92-101, 120-130), the per
// (poly, var) contribution lists of evaluate_system (evaldiff.py:248-265) and
// OpCounter's tallies (evaldiff.py:155-180).
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "internal.h"

using namespace pn;

pn_system::~pn_system() {
  cudaFree(d_mon_ptr);
  cudaFree(d_var);
  cudaFree(d_exp);
  cudaFree(d_dst);
  cudaFree(d_coeff);
  cudaFree(d_toff);
  cudaFree(d_tdeg);
  cudaFree(d_seg_ptr);
  cudaFree(d_seg_out);
  for (auto &b : buckets) cudaFree(b.d_list);
  cudaFree(rows.d_ent);
  cudaFree(rows.d_poly_chunk);
  cudaFree(rows.d_desc);
  cudaFree(rows.d_runoff);
  if (ev) cudaEventDestroy(ev);
  if (step_graph) cudaGraphExecDestroy(step_graph);
  for (auto e : gev)
    if (e) cudaEventDestroy(e);
  for (auto e : pev)
    if (e) cudaEventDestroy(e);
  if (graph_stream) cudaStreamDestroy(graph_stream);
}

namespace {

template <class T>
T *upload(const std::vector<T> &v) {
  T *p = nullptr;
  // +16 bytes: bulk copies of a last partial chunk round their size up to 16
  size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T) + 16;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    throw Fail{PN_E_NOMEM};
  }
  if (!v.empty()) PN_CHECK_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// canonical order (polyrep.py:103-107): ascending dense exponent vector.
// Equivalent sparse comparison: walk the supports in increasing
// variable order; at the first difference the monomial whose variable index
// is larger (i.e. lacks the smaller variable) is smaller; with equal
// variables the smaller exponent is smaller; a proper prefix is smaller.
struct CanonLess {
  const int32_t *mon_ptr, *var, *exp;
  bool operator()(int64_t a, int64_t b) const {
    int32_t pa = mon_ptr[a], ea = mon_ptr[a + 1], pb = mon_ptr[b], eb = mon_ptr[b + 1];
    for (; pa < ea && pb < eb; ++pa, ++pb) {
      if (var[pa] != var[pb]) return var[pa] > var[pb];
      if (exp[pa] != exp[pb]) return exp[pa] < exp[pb];
    }
    return (ea - pa) < (eb - pb);
  }
};

inline int floor_pow2(int k) {
  int b = 1;
  while (b * 2 <= k) b *= 2;
  return b;
}

// Plan of the row evaluation (evaldiff.cu, k_eval_rows).  Eligible when
// every non-constant monomial has the same k = K (2 <= K <= 32), n fits 16
// bits and the per-variable stacks (n x D elements, D = bit length of the
// longest Jacobian-entry run) fit in shared memory.  Chunks are CH = 512/G
// consecutive canonical monomials of a polynomial (rows_nt / rows_g in
// internal.h); inside a chunk the support entries are ranked by
// (variable, monomial) -- the reference's summation order restricted to the
// chunk (evaldiff.py:252-265) -- and each entry is packed as
// var | rank << 16 | exponent << 28 (rank < CH * K <= 4096); per chunk the
// run start of every variable (uint16).
void build_rows_plan(pn_system &S, const int32_t *poly_ptr, const std::vector<int32_t> &cptr,
                     const std::vector<int32_t> &cvar, const std::vector<int32_t> &cexp) {
  const char *env = getenv("PN_EVAL_ROWS");
  if (env && strcmp(env, "0") == 0) return;
  const int m = S.m, n = S.n, es = S.es;
  if (m == 0 || n > 65536) return;
  int K = -1;
  for (int64_t c = 0; c < S.M; ++c) {
    const int k = cptr[c + 1] - cptr[c];
    if (k == 0) continue;
    if (K < 0) K = k;
    else if (k != K) return;
  }
  if (K < 2 || K > 32) return;
  const int base = floor_pow2(K);
  const int G = rows_g(S.nc, S.cplx, base), NT = rows_nt(S.nc);
  const int CH = NT / G;
  // stack depth
  std::vector<int32_t> cnt(n, 0);
  int maxL = 0;
  for (int i = 0; i < m; ++i) {
    for (int32_t t = cptr[poly_ptr[i]]; t < cptr[poly_ptr[i + 1]]; ++t) maxL = std::max(maxL, ++cnt[cvar[t]]);
    for (int32_t t = cptr[poly_ptr[i]]; t < cptr[poly_ptr[i + 1]]; ++t) cnt[cvar[t]] = 0;
  }
  int D = 1;
  while ((1 << D) <= maxL) ++D;
  for (int64_t t = 0; t < S.nnz; ++t)
    if (cexp[t] > 15) return;  // 4 exponent bits in the packed entry
  // shared memory without x staged (evaldiff.cu decides whether x fits too)
  if (rows_layout(n, D, K, es, CH, base, NT / 32, false).total > kRowsSmemMax) return;
  std::vector<int32_t> poly_chunk(m + 1, 0);
  for (int i = 0; i < m; ++i) poly_chunk[i + 1] = poly_chunk[i] + (poly_ptr[i + 1] - poly_ptr[i] + CH - 1) / CH;
  const long long nchunks = poly_chunk[m];
  const int RS = (n + 1 + 7) & ~7;
  std::vector<uint32_t> ent(S.nnz);
  std::vector<uint16_t> runoff((size_t)nchunks * RS);
  std::vector<int4> desc(nchunks);
  std::vector<int32_t> pos(n);
  for (int i = 0; i < m; ++i) {
    const int T = poly_ptr[i + 1] - poly_ptr[i];
    for (int c = 0; c * CH < T; ++c) {
      const int64_t c0 = poly_ptr[i] + (int64_t)c * CH, c1 = std::min<int64_t>(poly_ptr[i + 1], c0 + CH);
      const int32_t e0 = cptr[c0], e1 = cptr[c1];
      for (int32_t t = e0; t < e1; ++t) cnt[cvar[t]]++;
      desc[poly_chunk[i] + c] = make_int4((int)c0, (int)(c1 - c0), e0, e1);
      uint16_t *ro = &runoff[(size_t)(poly_chunk[i] + c) * RS];
      int acc = 0;
      for (int j = 0; j < n; ++j) {
        ro[j] = (uint16_t)acc;
        pos[j] = acc;
        acc += cnt[j];
        cnt[j] = 0;
      }
      ro[n] = (uint16_t)acc;
      for (int32_t t = e0; t < e1; ++t)
        ent[t] = (uint32_t)cvar[t] | ((uint32_t)pos[cvar[t]]++ << 16) | ((uint32_t)cexp[t] << 28);
    }
  }
  bool unit = true;
  for (int64_t t = 0; unit && t < S.nnz; ++t) unit = cexp[t] == 1;
  auto &R = S.rows;
  R.K = K;
  R.base = base;
  R.CH = CH;
  R.D = D;
  R.nchunks = nchunks;
  R.unit = unit;
  R.d_ent = upload(ent);
  R.d_poly_chunk = upload(poly_chunk);
  R.d_runoff = upload(runoff);
  R.d_desc = upload(desc);
  R.ok = true;
}

}  // namespace

extern "C" int pn_system_create(int nc, int cplx, int32_t m, int32_t n, int64_t M, int64_t nnz,
                                const int32_t *poly_ptr, const int32_t *mon_ptr, const int32_t *var_idx,
                                const int32_t *exps, const double *coeffs, int already_canonical,
                                pn_system **out) {
  PN_API_BEGIN
  check_level(nc, cplx);
  PN_REQUIRE(out, PN_E_ARG, "pn_system_create: out is NULL");
  *out = nullptr;
  PN_REQUIRE(m >= 0 && n >= 1 && M >= 0 && nnz >= 0, PN_E_ARG, "pn_system_create: bad sizes");
  PN_REQUIRE(M + nnz < (int64_t)1 << 31, PN_E_ARG, "pn_system_create: more than 2^31 terms");
  PN_REQUIRE(poly_ptr && mon_ptr && (nnz == 0 || (var_idx && exps)) && (M == 0 || coeffs), PN_E_ARG,
             "pn_system_create: NULL array");
  PN_REQUIRE(poly_ptr[0] == 0 && poly_ptr[m] == M, PN_E_ARG, "poly_ptr must span [0, M]");
  PN_REQUIRE(mon_ptr[0] == 0 && mon_ptr[M] == nnz, PN_E_ARG, "mon_ptr must span [0, nnz]");
  for (int i = 0; i < m; ++i) PN_REQUIRE(poly_ptr[i] <= poly_ptr[i + 1], PN_E_ARG, "poly_ptr not monotone");
  for (int64_t t = 0; t < M; ++t) {
    PN_REQUIRE(mon_ptr[t] <= mon_ptr[t + 1], PN_E_ARG, "mon_ptr not monotone");
    int prev = -1;
    for (int32_t p = mon_ptr[t]; p < mon_ptr[t + 1]; ++p) {
      PN_REQUIRE(var_idx[p] >= 0 && var_idx[p] < n, PN_E_ARG,
                 "variable index %d out of range for n_vars=%d", var_idx[p], n);
      PN_REQUIRE(var_idx[p] > prev, PN_E_ARG, "variable indices must be strictly increasing");
      PN_REQUIRE(exps[p] >= 1, PN_E_ARG, "listed exponents must be >= 1");
      prev = var_idx[p];
    }
  }

  auto sys = std::make_unique<pn_system>();
  pn_system &S = *sys;
  S.nc = nc;
  S.cplx = cplx;
  S.es = nc * (cplx ? 2 : 1);
  S.m = m;
  S.n = n;
  S.M = M;
  S.nnz = nnz;
  const int es = S.es;

  // 1. canonical order within each polynomial (stable: duplicates keep order)
  S.perm.resize(M);
  std::iota(S.perm.begin(), S.perm.end(), 0);
  if (!already_canonical) {
    CanonLess less{mon_ptr, var_idx, exps};
    for (int i = 0; i < m; ++i)
      std::stable_sort(S.perm.begin() + poly_ptr[i], S.perm.begin() + poly_ptr[i + 1], less);
  }

  // 2. canonical CSR + AoS coefficients
  std::vector<int32_t> cptr(M + 1), cvar(nnz), cexp(nnz);
  std::vector<double> ccoef((size_t)M * es);
  cptr[0] = 0;
  for (int64_t c = 0; c < M; ++c) {
    const int64_t src = S.perm[c];
    const int32_t a = mon_ptr[src], b = mon_ptr[src + 1];
    std::copy(var_idx + a, var_idx + b, cvar.begin() + cptr[c]);
    std::copy(exps + a, exps + b, cexp.begin() + cptr[c]);
    cptr[c + 1] = cptr[c] + (b - a);
    for (int p = 0; p < es; ++p) ccoef[(size_t)c * es + p] = coeffs[(size_t)p * M + src];
  }

  // 3. power table layout: x^1..x^maxdeg per variable present
  std::vector<int32_t> tdeg(n, 0), toff(n, 0);
  for (int64_t t = 0; t < nnz; ++t) tdeg[cvar[t]] = std::max(tdeg[cvar[t]], cexp[t]);
  long long tl = 0;
  int maxdeg = 0;
  int64_t table_muls = 0;
  for (int v = 0; v < n; ++v) {
    toff[v] = (int32_t)tl;
    tl += tdeg[v];
    maxdeg = std::max(maxdeg, tdeg[v]);
    if (tdeg[v] > 1) table_muls += tdeg[v] - 1;
  }
  S.table_len = tl;
  S.max_deg = maxdeg;

  // 4. contribution slots: [0, M) monomial values (canonical order), then the
  // support entries stably sorted by variable -> within a variable ordered by
  // (poly, canonical monomial), so each Jacobian entry (i, j) is one
  // contiguous run in the reference's summation order
  std::vector<int64_t> vcount(n + 1, 0);
  for (int64_t t = 0; t < nnz; ++t) vcount[cvar[t] + 1]++;
  for (int v = 0; v < n; ++v) vcount[v + 1] += vcount[v];
  std::vector<int32_t> dst(nnz);
  std::vector<int32_t> entry_poly(nnz);
  {
    std::vector<int64_t> pos(vcount.begin(), vcount.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int32_t c = poly_ptr[i]; c < poly_ptr[i + 1]; ++c)
        for (int32_t t = cptr[c]; t < cptr[c + 1]; ++t) {
          const int64_t slot = pos[cvar[t]]++;
          dst[t] = (int32_t)(M + slot);
          entry_poly[slot] = i;
        }
  }
  std::vector<int64_t> seg_ptr;
  std::vector<int64_t> seg_out;
  seg_ptr.reserve((size_t)m + 1);
  for (int i = 0; i < m; ++i) seg_ptr.push_back(poly_ptr[i]);
  int64_t add_ops = 0;
  for (int i = 0; i < m; ++i)
    if (poly_ptr[i + 1] > poly_ptr[i]) add_ops += poly_ptr[i + 1] - poly_ptr[i] - 1;
  for (int v = 0; v < n; ++v) {
    int64_t a = vcount[v];
    while (a < vcount[v + 1]) {
      int64_t b = a + 1;
      while (b < vcount[v + 1] && entry_poly[b] == entry_poly[a]) ++b;
      seg_ptr.push_back(M + a);
      seg_out.push_back((int64_t)v * m + entry_poly[a]);
      add_ops += b - a - 1;
      a = b;
    }
  }
  seg_ptr.push_back(M + nnz);
  S.nseg = (long long)seg_out.size();

  // 5. buckets + analytic OpCounter + work counts
  // 0: k <= 1; 1..5: base 2..32; 6 + j: large trees of base 2^(6 + j)
  std::vector<std::vector<int32_t>> lists(6 + 26);
  int64_t em = 0, gm = 0, mul_ops = 0, int_ops = 0;
  int max_k = 0;
  for (int64_t c = 0; c < M; ++c) {
    const int k = cptr[c + 1] - cptr[c];
    max_k = std::max(max_k, k);
    int cc = 0;
    for (int32_t t = cptr[c]; t < cptr[c + 1]; ++t) cc += cexp[t] >= 2;
    if (k == 0) {
      lists[0].push_back((int32_t)c);
      continue;
    }
    if (k == 1) {
      lists[0].push_back((int32_t)c);
      const int d = cexp[cptr[c]];
      em += 1;
      gm += d > 1 ? 1 : 0;
      mul_ops += 1 + (d > 1 ? 1 : 0);
      int_ops += 1;
      continue;
    }
    const int base = floor_pow2(k), ell = k - base;
    em += (k - 1) + cc + 1;                          // tree, common fold + scale, value
    gm += (2 * base - 4) + 2 * ell + k + cc;         // gradient circuit + derivative scaling
    mul_ops += (k - 1) + cc + 1 + (2 * base - 4) + 2 * ell + k;
    int_ops += cc;
    const int lst = __builtin_ctz(base);  // base 2 -> 1, ..., 32 -> 5, 64 -> 6, ...
    lists[lst].push_back((int32_t)c);
  }
  S.counts.eval_mults = em;
  S.counts.grad_mults = gm;
  S.max_k = max_k;
  for (int b = 0; b < (int)lists.size(); ++b) {
    if (lists[b].empty()) continue;
    pn_system::Bucket bk;
    bk.kind = b == 0 ? 0 : (b >= 6 ? 2 : 1);
    bk.base = b >= 1 ? (1 << b) : 0;
    bk.count = (long long)lists[b].size();
    bk.d_list = upload(lists[b]);
    if (bk.kind == 1) {
      const auto &L = lists[b];
      const int K = cptr[L[0] + 1] - cptr[L[0]];
      bool dense = cptr[L[0]] % 4 == 0;
      for (size_t i = 0; dense && i < L.size(); ++i)
        dense = cptr[L[i] + 1] - cptr[L[i]] == K && (int64_t)cptr[L[i]] == (int64_t)cptr[L[0]] + (int64_t)i * K;
      if (dense) {
        bk.dense_k = K;
        bk.e0 = cptr[L[0]];
        bool unit = true;
        for (int64_t t = bk.e0; unit && t < bk.e0 + bk.count * K; ++t) unit = cexp[t] == 1;
        bk.unit_exp = unit;
      }
    }
    S.buckets.push_back(bk);
  }

  S.stats.nc = nc;
  S.stats.cplx = cplx;
  S.stats.m = m;
  S.stats.n = n;
  S.stats.monomials = M;
  S.stats.support = nnz;
  S.stats.segments = S.nseg;
  S.stats.mul_ops = mul_ops;
  S.stats.int_mul_ops = int_ops;
  S.stats.add_ops = add_ops;
  S.stats.table_mul_ops = table_muls;
  S.stats.max_k = max_k;
  S.stats.max_deg = maxdeg;

  // 6. upload
  S.d_mon_ptr = upload(cptr);
  S.d_var = upload(cvar);
  S.d_exp = upload(cexp);
  S.d_dst = upload(dst);
  S.d_coeff = upload(ccoef);
  S.d_toff = upload(toff);
  S.d_tdeg = upload(tdeg);
  S.d_seg_ptr = upload(seg_ptr);
  S.d_seg_out = upload(seg_out);
  build_rows_plan(S, poly_ptr, cptr, cvar, cexp);
  PN_CHECK_CUDA(cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming));
  *out = sys.release();
  PN_API_END
}

extern "C" int pn_system_destroy(pn_system *sys) {
  PN_API_BEGIN
  if (sys) {
    cudaDeviceSynchronize();
    delete sys;
  }
  PN_API_END
}

extern "C" int pn_system_get_stats(const pn_system *sys, pn_system_stats *stats) {
  PN_API_BEGIN
  PN_REQUIRE(sys && stats, PN_E_ARG, "NULL argument");
  *stats = sys->stats;
  PN_API_END
}

extern "C" int pn_system_plan_info(const pn_system *sys, pn_plan_info *info) {
  PN_API_BEGIN
  PN_REQUIRE(sys && info, PN_E_ARG, "NULL argument");
  const auto &R = sys->rows;
  *info = pn_plan_info{R.ok ? 1 : 0, R.K, R.CH, R.D, (int64_t)R.nchunks};
  PN_API_END
}

extern "C" int pn_system_canonical_order(const pn_system *sys, int64_t *perm) {
  PN_API_BEGIN
  PN_REQUIRE(sys && perm, PN_E_ARG, "NULL argument");
  for (size_t i = 0; i < sys->perm.size(); ++i) perm[i] = sys->perm[i];
  PN_API_END
}

extern "C" int pn_system_counts(const pn_system *sys, pn_counts *counts) {
  PN_API_BEGIN
  PN_REQUIRE(sys && counts, PN_E_ARG, "NULL argument");
  *counts = sys->counts;
  PN_API_END
}

// ---------------------------------------------------------------------------
// synthetic generator F(n, T, k, seed, maxexp, m) -- SURVEY 8(d)

namespace {
struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  uint32_t below(uint32_t bound) { return (uint32_t)(((unsigned __int128)next() * bound) >> 64); }
};
}  // namespace

extern "C" int pn_generate_random_system(int32_t m, int32_t n, int32_t T, int32_t kmin, int32_t k, int32_t maxexp,
                                         uint64_t seed, int32_t *poly_ptr, int32_t *mon_ptr, int32_t *var_idx,
                                         int32_t *exps, double *coef_re, double *coef_im) {
  PN_API_BEGIN
  PN_REQUIRE(m >= 0 && n >= 1 && T >= 0 && kmin >= 0 && kmin <= k && k <= n && maxexp >= 1, PN_E_ARG,
             "pn_generate_random_system: need 0 <= kmin <= k <= n, maxexp >= 1");
  PN_REQUIRE((int64_t)m * T * k < (int64_t)1 << 31, PN_E_ARG, "pn_generate_random_system: too many terms");
  SplitMix rng{seed * 0x2545F4914F6CDD1Dull + 0x1234567ull};
  std::vector<int32_t> pick(k);
  int64_t mon = 0, ent = 0;
  poly_ptr[0] = 0;
  mon_ptr[0] = 0;
  for (int32_t i = 0; i < m; ++i) {
    for (int32_t t = 0; t < T; ++t) {
      // "mixed" variant: k_t uniform in [kmin, k]; no draw when kmin == k, so
      // the uniform family's stream is unchanged
      const int32_t kt = kmin < k ? kmin + (int32_t)rng.below((uint32_t)(k - kmin + 1)) : k;
      // Floyd's algorithm: kt distinct values of [0, n)
      int cnt = 0;
      for (int32_t j = n - kt; j < n; ++j) {
        int32_t r = (int32_t)rng.below((uint32_t)j + 1);
        bool seen = false;
        for (int q = 0; q < cnt; ++q)
          if (pick[q] == r) { seen = true; break; }
        pick[cnt++] = seen ? j : r;
      }
      std::sort(pick.begin(), pick.begin() + cnt);
      for (int q = 0; q < cnt; ++q) {
        var_idx[ent] = pick[q];
        exps[ent] = 1 + (int32_t)rng.below((uint32_t)maxexp);
        ++ent;
      }
      double re = 0.5 + 1.5 * rng.uniform();
      if (rng.next() & 1) re = -re;
      double im = 0.5 + 1.5 * rng.uniform();
      if (rng.next() & 1) im = -im;
      coef_re[mon] = re;
      if (coef_im) coef_im[mon] = im;
      ++mon;
      mon_ptr[mon] = (int32_t)ent;
    }
    poly_ptr[i + 1] = (int32_t)mon;
  }
  PN_API_END
}
