/*
 * polynewt_b200.h -- C ABI of libpolynewt_b200.so, the B200-native
 * Gauss-Newton hot path (evaluation + reverse-mode differentiation of sparse
 * polynomial systems, Jacobian accumulation, modified Gram-Schmidt least
 * squares, Newton step) in complex/real double, double-double, quad-double.
 *
 * Every entry point replaces one function of the reference package
 * `polynewt` (paths relative to /root/reference/pkg/src/polynewt):
 *
 *   pn_vec_op / pn_tree_sum  <- varith.VecContext.add/sub/mul/div/abs2/
 *                               sqrt_real/conj, tree_sum   (varith.py:104-191)
 *   pn_system_create         <- evaldiff.PreparedSystem    (evaldiff.py:183-194)
 *                               + PolySystem.canonicalized (polyrep.py:103-107)
 *   pn_evaldiff              <- evaldiff.evaluate_system   (evaldiff.py:215-266)
 *   pn_mgs_qr                <- mgs.mgs_qr                 (mgs.py:145-221)
 *   pn_back_substitute       <- mgs.back_substitute(_staged) (mgs.py:229-289)
 *   pn_least_squares         <- mgs.least_squares_solve    (mgs.py:299-305)
 *   pn_newton_step           <- newton.newton_step         (newton.py:82-103)
 *   pn_newton_batch          <- newton.run_newton over homotopy_start_system
 *                               starts                     (newton.py:106-159)
 *   pn_residual_check        <- mgs.residual_check         (mgs.py:311-357)
 *
 * Conventions
 *  - A precision level is (nc, cplx): nc in {1,2,4} binary64 components
 *    (d, dd, qd); cplx in {0,1}.  es = nc * (cplx ? 2 : 1) doubles/element.
 *  - Array arguments use the reference's component-plane layout
 *    (varith.py:3-8, 73): a complex array of data shape S is float64
 *    C-contiguous with shape (2, nc, *S); a real one (nc, *S).
 *  - Pointers may be host (pageable or pinned) or device memory; the kind is
 *    detected per pointer.  Host buffers are staged through device memory on
 *    `stream` and the call returns after the results are back on the host.
 *    With device pointers the call is asynchronous on `stream` (NULL = the
 *    legacy default stream) unless it must report a numerical status.
 *  - Results are bit-identical to the reference on the same inputs.
 *  - Return value: PN_OK or an error code; pn_last_error() describes the
 *    last failure of the calling thread.
 */
#ifndef POLYNEWT_B200_H
#define POLYNEWT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PN_OK 0
#define PN_E_ARG 1       /* ValueError: shape / argument mismatch          */
#define PN_E_BREAKDOWN 2 /* mgs.MgsBreakdownError(k, rkk, threshold)       */
#define PN_E_SINGULAR 3  /* mgs.SingularMatrixError(index)                 */
#define PN_E_DOMAIN 4    /* xprec.DomainError                              */
#define PN_E_CUDA 5      /* CUDA runtime failure (RuntimeError)            */
#define PN_E_NOMEM 6     /* device or host allocation failure              */
#define PN_E_COMM 7      /* NCCL unavailable or failed (RuntimeError)      */

/* element-wise op codes for pn_vec_op (VecContext methods) */
#define PN_OP_ADD 0
#define PN_OP_SUB 1
#define PN_OP_MUL 2
#define PN_OP_DIV 3
#define PN_OP_ABS2 4     /* complex/real -> real element (nc doubles)     */
#define PN_OP_SQRT 5     /* real -> real, sqrt_real semantics             */
#define PN_OP_CONJ 6
#define PN_OP_MODULUS 7  /* xprec.modulus in the field: sqrt(re^2+im^2)
                            for complex, |x| for real (nc doubles out)   */
#define PN_OP_DIV_REAL 8 /* a / r with r a real array (VecContext.div_real) */

typedef struct pn_system pn_system;

/* numerical status details (MgsBreakdownError / SingularMatrixError) */
typedef struct {
  int32_t k;         /* breakdown column                                 */
  int32_t index;     /* singular diagonal index                          */
  double rkk;        /* hi component of r_kk at breakdown                */
  double threshold;  /* 1.0*n*eps*||a_k||_hi                             */
  double z;          /* least-squares residual norm hi(R[n,n])           */
  double t_evaluate; /* pn_newton_step phase times (seconds, CUDA events) */
  double t_solve;
  double t_update;
  double t_factor;  /* MGS factorisation alone (part of t_solve), seconds */
} pn_numinfo;

/* OpCounter (evaldiff.py:21-30): multiplication tallies of one evaluation */
typedef struct {
  int64_t eval_mults;
  int64_t grad_mults;
} pn_counts;

/* static description of a packed system (host-side analytic counts used
 * for the roofline: complex/real field multiplies, int multiplies, adds) */
typedef struct {
  int32_t nc, cplx, m, n;
  int64_t monomials;      /* M                                            */
  int64_t support;        /* nnz = sum of k over monomials                */
  int64_t segments;       /* nonzero Jacobian entries                     */
  int64_t mul_ops;        /* element x element multiplies per evaluation  */
  int64_t int_mul_ops;    /* element x small-integer multiplies           */
  int64_t add_ops;        /* element adds in the value/Jacobian trees     */
  int64_t table_mul_ops;  /* power-table multiplies                       */
  int32_t max_k;          /* largest monomial support                     */
  int32_t max_deg;        /* largest exponent                             */
} pn_system_stats;

int pn_version(void);
const char *pn_last_error(void);
int pn_device_count(int *count);
/* number of kernels this library launched since load (bench evidence) */
int64_t pn_launch_count(void);
/* measured FP64 pipe throughput of the current device (DFMA instructions/s),
 * the roofline denominator for the FP64-bound kernels */
int pn_fp64_peak(double *instr_per_s, void *stream);

/* ---- element-wise arithmetic on component planes ---------------------- */
/* a, b, out: planes of n elements.  b may be NULL for unary ops.  For
 * PN_OP_DIV_REAL, b is a real-plane array (nc, n). */
int pn_vec_op(int nc, int cplx, int op, int64_t n, const double *a, const double *b, double *out,
              void *stream);
/* canonical pairwise sum over the n elements of a (planes) -> out (one element) */
int pn_tree_sum(int nc, int cplx, int64_t n, const double *a, double *out, void *stream);

/* ---- systems ------------------------------------------------------------ */
/* Supports in CSR: poly_ptr[m+1] over monomials, mon_ptr[M+1] over the
 * support entries var_idx/exps[nnz] (strictly increasing vars, d >= 1, per
 * Monomial, polyrep.py:23-48).  coeffs: planes (cshape, M).  The monomials of
 * each polynomial are put into canonical order (stable sort on the dense
 * exponent vector, polyrep.py:103-107) unless already_canonical != 0.
 * The system lives on the current device until pn_system_destroy. */
int pn_system_create(int nc, int cplx, int32_t m, int32_t n, int64_t M, int64_t nnz,
                     const int32_t *poly_ptr, const int32_t *mon_ptr, const int32_t *var_idx,
                     const int32_t *exps, const double *coeffs, int already_canonical,
                     pn_system **out);
int pn_system_destroy(pn_system *sys);
int pn_system_get_stats(const pn_system *sys, pn_system_stats *stats);
/* the evaluation plan chosen for the system (diagnostics and tests):
 * rows_ok = 1 when the row kernel (k_eval_rows) can serve it, with its
 * uniform monomial size K, monomials per chunk, per-variable stack depth and
 * number of chunks */
typedef struct {
  int32_t rows_ok, K, chunk, depth;
  int64_t nchunks;
} pn_plan_info;
int pn_system_plan_info(const pn_system *sys, pn_plan_info *info);
/* canonical position -> input monomial index (M entries) */
int pn_system_canonical_order(const pn_system *sys, int64_t *perm);
/* analytic OpCounter of one evaluation (equals the reference's tallies) */
int pn_system_counts(const pn_system *sys, pn_counts *counts);

/* f = values (planes (cshape, m)); J = Jacobian (planes (cshape, m, n),
 * row-major).  Either output may be NULL.  counts (optional) receives the
 * OpCounter tallies. */
int pn_evaldiff(pn_system *sys, const double *x, double *f, double *J, pn_counts *counts, void *stream);

/* ---- least squares -------------------------------------------------------- */
/* aug: planes (cshape, m, n+1) = [A b].  Q: planes (cshape, m, n) or NULL;
 * R: planes (cshape, n+1, n+1) or NULL.  Returns PN_E_BREAKDOWN with info
 * filled on rank deficiency. */
int pn_mgs_qr(int nc, int cplx, int32_t m, int32_t n, const double *aug, double *Q, double *R,
              pn_numinfo *info, void *stream);
/* R: planes (cshape, n+1, n+1) (augmented factor; y = R[:n, n]).  x: (cshape, n). */
int pn_back_substitute(int nc, int cplx, int32_t n, const double *R, double *x, pn_numinfo *info,
                       void *stream);
/* x: planes (cshape, n); z receives hi(R[n,n]); Q, R optional as above. */
int pn_least_squares(int nc, int cplx, int32_t m, int32_t n, const double *aug, double *x, double *z,
                     double *Q, double *R, pn_numinfo *info, void *stream);

/* max componentwise |A - QR| recomputed in the next precision (d -> dd,
 * dd -> qd), bit-identical to mgs.residual_check.  A, Q: planes (cshape, m, n);
 * R: planes (cshape, n, n) (the leading block of the augmented factor).
 * Quad-double factorisations (320-bit mpfr in the reference) are evaluated by
 * exact fixed-point accumulation of all component products. */
int pn_residual_check(int nc, int cplx, int32_t m, int32_t n, const double *A, const double *Q, const double *R,
                      double *out, void *stream);

/* ---- Newton ---------------------------------------------------------------- */
/* One Gauss-Newton correction at x (planes (cshape, n)):
 *   x_next = x + dx,  dx = argmin ||J dx + f||, f = F(x), J = F'(x).
 * Optional outputs (planes): f (m), dx (n), and field moduli (real planes
 * (nc, len)) fmod (m), dxmod (n), xmod (n) of f, dx and x_next, from which the
 * host forms the reference's float norms (newton.py:33-34, 94-101). */
int pn_newton_step(pn_system *sys, const double *x, double *x_next, double *f, double *dx,
                   double *fmod, double *dxmod, double *xmod, pn_numinfo *info, void *stream);

/* Batched Newton runs (config C5): B independent run_newton calls
 * (newton.py:106-132) sharing the system's supports and coefficients.
 * x0, x_out: planes (cshape, B, n).  consts: planes (cshape, B, m) with the
 * coefficient of polynomial i's constant term for start b (the homotopy
 * shift of newton.py:135-159, already added to any base constant), or NULL;
 * with consts every polynomial must have exactly one constant term.
 * tol <= 0 selects the reference default 10*eps*(1+||x||_inf).
 * iters[b] = iterations run; status[b] = 0 converged, 1 max_iters reached,
 * 2 MGS breakdown, 3 singular back substitution. */
int pn_newton_batch(pn_system *sys, int64_t B, const double *x0, const double *consts, int max_iters, double tol,
                    double *x_out, int32_t *iters, int32_t *status, void *stream);
/* values f(x_b) for a batch of points: x planes (cshape, B, n) -> f planes (cshape, B, m) */
int pn_evaldiff_batch(pn_system *sys, int64_t B, const double *x, double *f, void *stream);

/* ---- synthetic inputs -------------------------------------------------------- */
/* SURVEY 8(d) F(n, T, k, seed, maxexp, m): m polynomials in n variables, T
 * monomials each of k distinct variables (uniform subset), exponents uniform
 * in [1, maxexp], coefficient parts uniform in +-[0.5, 2).  kmin < k gives
 * the C2 "mixed" variant: each monomial's variable count is uniform in
 * [kmin, k] (kmin == k draws nothing extra, so the uniform family is
 * unchanged).  Outputs CSR in generation order plus binary64 coefficients
 * coef_re/coef_im (M each; coef_im may be NULL for real systems).  Arrays
 * must be preallocated: poly_ptr[m+1], mon_ptr[m*T+1], var_idx/exps[m*T*k]
 * (the actual entry count is mon_ptr[m*T]).  The oracle carries an
 * independent restatement (or_generate_random_system) that the reference
 * arm of bench.py uses, so that arm never loads this library. */
int pn_generate_random_system(int32_t m, int32_t n, int32_t T, int32_t kmin, int32_t k, int32_t maxexp,
                              uint64_t seed, int32_t *poly_ptr, int32_t *mon_ptr, int32_t *var_idx, int32_t *exps,
                              double *coef_re, double *coef_im);

/* ---- system text format (polyrep.py:140-304) ------------------------------- */
/* Native ingestion of the text format into CSR (generation order) and
 * coefficient planes (es, M), the components converted exactly as
 * parse_decimal (xprec.py:432-446).  PN_E_ARG for malformed input and for
 * constructs outside the native scanner (non-ASCII text, unusual numeric
 * forms): the host then re-parses with polyrep.parse_system, which raises
 * the reference's SystemParseError or builds the system. */
typedef struct pn_text_system pn_text_system;
int pn_parse_system(const char *text, int64_t len, int nc, int cplx, pn_text_system **out);
int pn_text_system_sizes(const pn_text_system *s, int32_t *m, int32_t *n, int64_t *M, int64_t *nnz);
int pn_text_system_export(const pn_text_system *s, int32_t *poly_ptr, int32_t *mon_ptr, int32_t *var_idx,
                          int32_t *exps, double *coeff_planes);
int pn_text_system_free(pn_text_system *s);

/* ---- the batched path's collective (config C5 over several GPUs) ------------- */
/* SURVEY 8(b) pn_comm_* / 8(e).  One process per GPU: rank 0 creates an id
 * with pn_comm_unique_id and the host hands its 128 bytes to every rank (any
 * out-of-band channel); each rank calls pn_comm_init.  pn_batch_allgather
 * is the run's only collective: every rank contributes the results of its
 * block of starts [lo, hi) = batch.shard_range(B, world, rank) -- x planes
 * (cshape, hi - lo, n), iteration counts and status words as
 * pn_newton_batch returns them -- and receives the full batch (x planes
 * (cshape, B, n)).  Host or device pointers.  NCCL is loaded at run time
 * (the process's own copy when it has one); PN_E_COMM if unavailable.
 * Replaces batch.gather_batch's torch.distributed all_gather for hosts
 * without PyTorch. */
#define PN_COMM_ID_BYTES 128
typedef struct pn_comm pn_comm;
int pn_comm_unique_id(unsigned char *id);
int pn_comm_init(int world, int rank, const unsigned char *id, int device, pn_comm **out);
int pn_comm_destroy(pn_comm *comm);
int pn_batch_allgather(pn_comm *comm, int nc, int cplx, int32_t n, int64_t B, const double *x_shard,
                       const int32_t *iters_shard, const int32_t *status_shard, double *x_all, int32_t *iters_all,
                       int32_t *status_all, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* POLYNEWT_B200_H */
