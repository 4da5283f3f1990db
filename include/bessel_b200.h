/*
 * bessel_b200.h -- C ABI of the B200-native hot path of arXiv 2409.08729
 * ("Robust and efficient computation of the logarithm of modified Bessel
 * functions", PAPER.md).  Shared library: libbessel_b200.so (sm_100a).
 *
 * Conventions for every entry point
 *   - Pointers named *_d are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors), pointers named *_h are HOST pointers (pinned recommended).
 *     The library never takes ownership; the caller allocates and frees.
 *   - Arrays are dense, contiguous, element i of every array belongs to the
 *     same (v_i, x_i) pair.  n may be 0 (no-op, returns B200_OK).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device
 *     calls are asynchronous w.r.t. the host; host-buffer (_h) calls return
 *     after the results are in the host buffer.
 *   - Return value: 0 (B200_OK) on success, otherwise a b200_status code;
 *     b200_last_error() returns a static string describing the last failure.
 *     Invalid arguments (n < 0, NULL pointer with n > 0) are rejected before
 *     any launch.  Out-of-domain inputs are NOT errors: they produce NaN in
 *     that element only (see each function).
 *   - Alignment: 16-byte aligned arrays (any cudaMalloc / torch allocation)
 *     move through the bulk-copy (TMA) engine; 8-byte aligned ones (e.g. a
 *     view starting at an odd element) take a per-thread cp.async path with
 *     identical results.
 *   - Operating range: 1e-140 <= x <= 1e140, |v| <= 1e140 (f64) and
 *     1e-18 <= x <= 1e18, |v| <= 1e18 (f32) run on the fast table-driven
 *     paths; finite arguments outside it (subnormals included) are evaluated
 *     by the same formulas with library functions, rescaling and scaled
 *     recurrences (slower, same accuracy); IEEE special values follow each
 *     function's description.
 *   - Thread safety: device entry points may be called concurrently from
 *     several host threads and streams; host-buffer entry points serialise
 *     per device on an internal pipeline (4 streams, 512 MB of device
 *     staging allocated on first use and kept for the process lifetime).
 *   - Determinism: results depend only on (v_i, x_i) -- not on n, the
 *     position in the array, the stream or the alignment.
 */
#ifndef BESSEL_B200_H
#define BESSEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    B200_OK = 0,
    B200_ERR_INVALID_ARGUMENT = 1,
    B200_ERR_CUDA = 2,
    B200_ERR_NO_DEVICE = 3
} b200_status;

/* Region ids written by b200_classify_* (Algorithm 1, PAPER.md lines 359-386,
 * GPU branch set {mu, U13, fallback} per the Algorithm 1 caption). */
enum {
    B200_METHOD_MU = 0,        /* large-argument expansion, Eqs. (log Iv mu k)/(log Kv mu k) */
    B200_METHOD_U13 = 1,       /* uniform large-order (Debye) expansion, Eqs. (log Iv u k)/(log Kv u k) */
    B200_METHOD_FALLBACK = 2   /* I: log-domain power series, Eq. (log Iv); K: small-argument method */
};

/* ------------------------------------------------------------------------
 * log I_v(x) -- PAPER.md §3.1 (Eq. (Iv infinite series), line 127) evaluated by
 * Algorithm 1 (lines 359-386) on the GPU branch set.
 *   v_d, x_d : n orders / arguments.  Domain v >= 0, x >= 0 (paper line 125).
 *   out_d    : n results, log I_v(x).  log I_0(0) = 0; log I_v(0) = -inf (v>0);
 *              NaN where v < 0, x < 0 or an input is NaN.
 * Accuracy (f64): |out - exact| <= 1e-13 * max(|exact|, 1) on the tested
 * domain; f32: 1e-5.
 */
int b200_log_iv_f64(const double *v_d, const double *x_d, double *out_d, int64_t n, void *stream);
int b200_log_iv_f32(const float *v_d, const float *x_d, float *out_d, int64_t n, void *stream);

/* ------------------------------------------------------------------------
 * log K_v(x) -- PAPER.md §3.2 (Eqs. (log Kv mu k), (log Kv u k), lines 233-246)
 * by Algorithm 1; the small-argument fallback replaces the paper's Simpson
 * integral (line 251-269) by the trapezoidal rule on the same integral
 * representation (2 < x <= 30) or Temme's series (x <= 2), each followed by
 * the forward recurrence in the order -- DESIGN.md §5.
 *   Domain: x > 0, any real v (K_{-v} = K_v).  x = 0 -> +inf (pole);
 *   x < 0 or NaN input -> NaN.
 */
int b200_log_kv_f64(const double *v_d, const double *x_d, double *out_d, int64_t n, void *stream);
int b200_log_kv_f32(const float *v_d, const float *x_d, float *out_d, int64_t n, void *stream);

/* ------------------------------------------------------------------------
 * log I_v(x) AND log K_v(x) of the same pairs in one pass (fused): the inputs
 * are read once, classification / binning is shared, and inside the mu and U
 * regions the expansions share every term (I and K differ only by the sign
 * pattern (-1)^k, Eqs. (log Iv mu k)/(log Kv mu k), (log Iv u k)/(log Kv u k)).
 * In the small-argument fallback region (1e-6 <= x <= 30 for f64, 2 < x <= 30
 * for f32) log I is taken from the K values by the Wronskian
 * I_v K_{v+1} + I_{v+1} K_v = 1/x with I_{v+1}/I_v from Miller's backward
 * recurrence instead of the power series of Eq. (Iv infinite series).
 *   out_i_d[i] = log I_{v_i}(x_i), out_k_d[i] = log K_{v_i}(x_i), with the
 *   domains and special values of the two functions above (v < 0: out_i NaN,
 *   out_k = log K_{|v|}).  Results equal the separate calls to the stated
 *   accuracy (not bit for bit: the fused sums round differently).
 */
int b200_log_ivkv_f64(const double *v_d, const double *x_d, double *out_i_d, double *out_k_d, int64_t n,
                      void *stream);
int b200_log_ivkv_f32(const float *v_d, const float *x_d, float *out_i_d, float *out_k_d, int64_t n,
                      void *stream);

/* The paper's own K fallback (log-domain Rothwell integral, Simpson N=600,
 * heuristic maxima) on the same dispatch -- kept for
 * fidelity studies; accuracy is the paper's (~1e-9, Table 2), not 1e-13. */
int b200_log_kv_paper_f64(const double *v_d, const double *x_d, double *out_d, int64_t n, void *stream);

/* Region id (B200_METHOD_*) per element, as int8 -- the dispatch of
 * Algorithm 1 / Table 1 (lines 338-352) with the GPU branch set. */
int b200_classify_f64(const double *v_d, const double *x_d, int8_t *method_d, int64_t n, void *stream);

/* ------------------------------------------------------------------------
 * Host-buffer variants (end-to-end): v_h, x_h, out_h are HOST arrays; the
 * library stages them through device memory in chunks, overlapping
 * H2D copy / kernel / D2H copy on internal streams.  Blocking.
 */
int b200_log_iv_f64_host(const double *v_h, const double *x_h, double *out_h, int64_t n);
int b200_log_kv_f64_host(const double *v_h, const double *x_h, double *out_h, int64_t n);
int b200_log_ivkv_f64_host(const double *v_h, const double *x_h, double *out_i_h, double *out_k_h, int64_t n);

/* ------------------------------------------------------------------------
 * von Mises-Fisher fit, §6.3 (lines 663-693).
 *
 * b200_vmf_colsum_*: colsum_d[j] (+)= sum_i X[i, j] over the n rows of the
 *   row-major n x d matrix X_d (leading dimension ld >= d elements), fp64
 *   accumulation.  If accumulate == 0 colsum_d is overwritten, else added to.
 *   This is the data-parallel part (Eq. (mean direction estimate), line 672).
 *   with_count != 0: colsum_d holds d + 1 doubles and colsum_d[d] (+)= n, so
 *   with rows sharded over GPUs ONE all-reduce of the d + 1 doubles carries
 *   both the column sums and the global row count.  Deterministic for a given
 *   (n, d, device).  Scratch: the per-slab partials use a library-owned device
 *   buffer per (device, stream), grown on demand and kept for the process;
 *   concurrent calls on different streams or host threads are safe.  A call
 *   on a stream that has not used the library yet allocates that buffer
 *   (cudaMalloc): before capturing into a CUDA graph, make one call on the
 *   capture stream.  The partial -> reduce -> fit kernels are chained by
 *   programmatic dependent launch (captured as programmatic graph edges).
 *   Errors: n < 0, d < 0, ld < d, NULL X with n > 0, NULL colsum_d.
 *
 * b200_vmf_fit_from_colsum: given the global column sum (d doubles) and the
 *   global row count n_total, computes on the device
 *     mu_d[0..d)   = xbar / Rbar                      (line 672)
 *     stats_d[0]   = Rbar
 *     stats_d[1..3]= kappa0, kappa1, kappa2            (Eq. (kappa estimates), lines 676-680)
 *     stats_d[4]   = kappa_mle  (root of Rbar - A_p(kappa), the maximiser of
 *                                the log-likelihood, lines 684-691)
 *     stats_d[5]   = logLik(kappa_mle)                 (lines 685-689)
 *     stats_d[6]   = A_p(kappa_mle) - Rbar  (stationarity residual)
 *     stats_d[7]   = number of MLE iterations
 *   stats_d must hold 8 doubles.  p = d.  n_total == 0: the row count is read
 *   from colsum_d[d] (a with_count column sum).  Rbar outside (0,1) -> stats NaN.
 *   Errors: d < 2, n_total < 0, NULL pointers.
 *
 * b200_vmf_fit_*: both steps on one device (workspace: d doubles, device); n >= 1.
 */
int b200_vmf_colsum_f32(const float *X_d, int64_t n, int64_t d, int64_t ld, double *colsum_d,
                        int accumulate, int with_count, void *stream);
int b200_vmf_colsum_f64(const double *X_d, int64_t n, int64_t d, int64_t ld, double *colsum_d,
                        int accumulate, int with_count, void *stream);
int b200_vmf_fit_from_colsum(const double *colsum_d, int64_t n_total, int64_t d, double *mu_d,
                             double *stats_d, void *stream);
int b200_vmf_fit_f32(const float *X_d, int64_t n, int64_t d, double *workspace_d, double *mu_d,
                     double *stats_d, void *stream);
int b200_vmf_fit_f64(const double *X_d, int64_t n, int64_t d, double *workspace_d, double *mu_d,
                     double *stats_d, void *stream);

/* ------------------------------------------------------------------------ */
const char *b200_last_error(void);
/* Number of kernel launches issued by this library since load (diagnostic;
 * bench.py reports it as gpu_launches). */
int64_t b200_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BESSEL_B200_H */
