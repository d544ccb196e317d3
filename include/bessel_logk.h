/*
 * bessel_logk.h -- C ABI of the B200 (sm_100a) fixed-bin integral method for
 * log K_v(x) and its derivatives (Takekawa, arXiv 2108.11560).
 *
 * Operation (PAPER.md, cited as P:<line>):
 *   K_v(x) = int_0^inf cosh(vt) exp(-x cosh t) dt,  v in R, x > 0   (Eq. 1-2)
 *   For every element i the library finds the peak t_p of
 *   g(t) = log cosh(vt) - x cosh t (t_p = 0 when v^2 <= x,
 *   P:103-110) and the range [t0, t1] where g >= g(t_p) + log eps
 *    with Alg. 1 FindRange and Alg. 2 FindZero (at most
 *   10 iterations, ending on the paper's "until" clause with a working
 *   tolerance, R4), then integrates with a FIXED number of trapezoid
 *   intervals n = nbins (Eq. (int)) in log-sum-exp form:
 *     logk[i]     = log K_v(x)
 *     dlogk_dv[i] = d log K_v(x) / dv   (integrand t sinh(vt) e^{-x cosh t})
 *     dlogk_dx[i] = d log K_v(x) / dx   (integrand -cosh t cosh(vt) e^{-x cosh t})
 *   The three sums share f's range and nodes (one pass).
 *
 * Conventions shared by every entry point
 *   - v, x, logk, dlogk_dv, dlogk_dx of the device entry points are DEVICE
 *     pointers to n contiguous elements, owned by the caller.  The library
 *     never allocates, frees or synchronises on those paths; the call enqueues
 *     one kernel on `stream` (NULL = legacy default stream) and returns.
 *   - Any of logk / dlogk_dv / dlogk_dx may be NULL to skip that output (a
 *     compile-time kernel variant; skipped outputs cost nothing and do not
 *     change the others bit-wise).  At least one must be non-NULL.  Outputs
 *     must not alias the inputs or each other.
 *   - Per-element domain (never fails the batch): x <= 0, x or v NaN/inf ->
 *     all requested outputs NaN.  v < 0 -> evaluated at |v| with dlogk_dv
 *     negated (K is even in v).  The FindRange doubling cap (t <= t_s + 2^12)
 *     exceeded -> NaN.  FP64 entry points: an integration range reaching
 *     t = 709 (e^t overflows double; x near or below DBL_MIN for small orders)
 *     -> NaN, as in the oracle (R23).  Meaningful derivatives need
 *     eps (x + v t_p) << 1 (R22).
 *   - Results are a pure function of (v[i], x[i], nbins, entry point,
 *     options, lanes per element): bit-identical across runs, batch
 *     permutations, shard counts and output subsets.  (lanes_per_element = 0
 *     picks the lane count from n, which can change the last ulps; pass an
 *     explicit value for n-independent bits.)
 *   - Reentrant and thread-safe; no global mutable state except the one-time
 *     lazily created helper streams of the *_host entry points.
 *
 * Errors: BLK_EINVAL (no CUDA call made) when nbins < 2 or nbins >
 * BLK_MAX_NBINS, an option is out of range, or n > 0 and v or x is NULL or all
 * outputs are NULL; otherwise n == 0 is a no-op returning BLK_OK (pointers are
 * not inspected).  BLK_ECUDA when a CUDA call or the
 * kernel launch fails (message via bessel_logk_last_error()).
 */
#ifndef BESSEL_LOGK_H
#define BESSEL_LOGK_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BLK_API __attribute__((visibility("default")))
#else
#define BLK_API
#endif

/* Same type as the CUDA runtime's cudaStream_t (an opaque CUstream handle). */
struct CUstream_st;
typedef struct CUstream_st *cudaStream_t;

typedef enum {
    BLK_OK = 0,
    BLK_EINVAL = 1,
    BLK_ECUDA = 2
} blk_status;

/* Largest accepted nbins (the paper fixes none). */
#define BLK_MAX_NBINS 65536

/* Range-finding precision (options.range_mode). */
#define BLK_RANGE_AUTO 0  /* FP32 (FMA + MUFU pipes) when nbins >= 48 and the element is
                             inside the FP32-safe domain (x in [1e-30, 1e4], |v| <= 1e4),
                             else FP64 as below: coarse grids are sensitive to the
                             node placement (R20) */
#define BLK_RANGE_F64 1   /* working-precision range finding, as the paper does: FP64,
                             FindZero until the Newton step is below 2^-45 of the
                             scale (the oracle's fixed-10-iteration ranges) */

typedef struct {
    /* Lanes cooperating on one element (1 = one element per thread; 2..32,
     * a power of two, splits the n+1 bins across lanes with a warp-shuffle
     * reduction).  0 = automatic choice from n (documented in DESIGN.md). */
    int lanes_per_element;
    /* BLK_RANGE_AUTO or BLK_RANGE_F64. */
    int range_mode;
    /* Threads per block of the simple kernel (0 = default 128; else a
     * multiple of 32 in [32, 128]). */
    int block_threads;
    /* Kernel variant: BLK_KERNEL_AUTO or BLK_KERNEL_SIMPLE (the same
     * kernel: one element -- or lanes_per_element lanes -- per thread, both
     * phases in every warp), or BLK_KERNEL_VEC128 (below).  Any other value
     * is BLK_EINVAL.  (A warp-specialised producer/consumer variant was
     * measured 10-20% slower and removed.) */
    int kernel;
} blk_options;

#define BLK_KERNEL_AUTO 0
#define BLK_KERNEL_SIMPLE 1
/* One element per thread with warp-cooperative 128-bit loads and stores of
 * the v / x / output streams (BASELINE.json north_star (3)): each warp moves
 * its 32 elements as 16-byte vectors and transposes them through shared
 * memory.  lanes_per_element must be 0 or 1 (else BLK_EINVAL).  Needs every
 * non-NULL stream 16-byte aligned; otherwise the scalar-I/O kernel runs.
 * Results are bit-identical to BLK_KERNEL_SIMPLE with one lane per element.
 * Not the default: measured 0.8% (FP64) / 1.7% (FP32) slower on B200, the
 * kernels being compute-bound at ~3% of HBM bandwidth. */
#define BLK_KERNEL_VEC128 2

/*
 * FP64 entry point.  eps = 2^-52 (log eps = -36.0437, R9).
 * v, x: device, n doubles each.  logk, dlogk_dv, dlogk_dx: device, n doubles
 * each, or NULL.  nbins: number of trapezoid INTERVALS n (n+1 nodes).
 */
BLK_API blk_status bessel_logk_f64(const double *v, const double *x, size_t n,
                           double *logk, double *dlogk_dv, double *dlogk_dx,
                           int nbins, cudaStream_t stream);

/* FP32 entry point: same contract, float arrays, eps = 2^-23. */
BLK_API blk_status bessel_logk_f32(const float *v, const float *x, size_t n,
                           float *logk, float *dlogk_dv, float *dlogk_dx,
                           int nbins, cudaStream_t stream);

/* Same as above with explicit options (opts may be NULL = all defaults). */
BLK_API blk_status bessel_logk_f64_ex(const double *v, const double *x, size_t n,
                              double *logk, double *dlogk_dv, double *dlogk_dx,
                              int nbins, const blk_options *opts,
                              cudaStream_t stream);
BLK_API blk_status bessel_logk_f32_ex(const float *v, const float *x, size_t n,
                              float *logk, float *dlogk_dv, float *dlogk_dx,
                              int nbins, const blk_options *opts,
                              cudaStream_t stream);

/*
 * Host-buffer entry point (end-to-end use).  v, x, logk, dlogk_dv, dlogk_dx
 * are HOST pointers.  Two transports, same results:
 *  - zero-copy: when every non-NULL buffer is page-locked host memory mapped
 *    into the device address space (cudaHostAlloc / cudaMallocHost /
 *    cudaHostRegister under unified addressing -- e.g. torch pin_memory), one
 *    kernel launch reads the inputs and writes the outputs over PCIe
 *    directly, so the transfers overlap the computation element by element
 *    (the workspace is not used and may be NULL);
 *  - staged: otherwise (pageable memory works but serialises), the batch is
 *    split into chunks of `chunk` elements (0 = default 2^20) that are copied
 *    host->device, computed and copied device->host on a small pool of
 *    streams so that transfers of one chunk overlap the kernel of another.
 *    (BLK_HOST_PIPELINE=1 in the environment forces this path; measurement
 *    only.)
 * workspace: DEVICE buffer of at least bessel_logk_host_workspace_bytes(chunk,
 * 8) bytes, owned by the caller; required (BLK_EINVAL if NULL or too small)
 * only when the staged transport is taken.
 * Blocking: returns after all results are in host memory (the work is ordered
 * after prior work on `stream`).  Both transports run the simple kernel with
 * one element per lane, so results equal bessel_logk_f64_ex with
 * lanes_per_element = 1 bit for bit, whatever the transport or chunking.
 */
BLK_API size_t bessel_logk_host_workspace_bytes(size_t chunk, size_t elem_bytes);
BLK_API blk_status bessel_logk_f64_host(const double *v, const double *x, size_t n,
                                double *logk, double *dlogk_dv, double *dlogk_dx,
                                int nbins, void *workspace, size_t workspace_bytes,
                                size_t chunk, cudaStream_t stream);
/* The same for the FP32 entry point: float host arrays; workspace of at
 * least bessel_logk_host_workspace_bytes(chunk, 4) bytes. */
BLK_API blk_status bessel_logk_f32_host(const float *v, const float *x, size_t n,
                                float *logk, float *dlogk_dv, float *dlogk_dx,
                                int nbins, void *workspace, size_t workspace_bytes,
                                size_t chunk, cudaStream_t stream);

/*
 * The integration plan alone: Alg. 3 lines 2-9 (Alg. 1 FindRange,
 * Alg. 2 FindZero) exactly as bessel_logk_f64 / _f64_ex find it
 * for the same nbins and options (range_mode selects the finder as there;
 * lanes_per_element does not change the plan):
 *   tp[i] = t_p (0 when v^2 <= x), gp[i] = g(t_p) (the log-sum-exp
 *   shift of Eq. (int)), t0[i], t1[i] = the ends of the range where
 *   g >= g(t_p) + log eps, eps = 2^-52.
 * bessel_logk_f64 integrates Eq. (int) with n = nbins intervals over exactly
 * [t0[i], t1[i]] with shift gp[i].  All pointers DEVICE, n doubles each; any
 * output may be NULL (at least one not).  NaN where the element has no plan
 * (invalid input, FindRange cap).  Several plans are equally correct (any
 * conservative range, R20); this one lets a caller check the
 * quadrature against a reference on the same range.
 */
BLK_API blk_status bessel_logk_plan_f64(const double *v, const double *x, size_t n, double *tp,
                                        double *gp, double *t0, double *t1, int nbins,
                                        const blk_options *opts, cudaStream_t stream);

/*
 * Second derivatives in the same pass: from the
 * second-order differentiated integrands of Sec. 4.1 (f^{(n,m)},
 * n+m = 2) over f's range and nodes,
 *   d2_dv2  = d^2 log K / dv^2   = S11/S0 - (S1/S0)^2,   S11 = sum w t^2
 *   d2_dx2  = d^2 log K / dx^2   = S22/S0 - (S2/S0)^2,   S22 = sum w cosh^2 t
 *   d2_dvdx = d^2 log K / dv dx  = S1 S2/S0^2 - S12/S0,   S12 = sum w t tanh(vt) cosh t
 * plus log K, dlogK/dv, dlogK/dx as bessel_logk_f64.  All pointers DEVICE,
 * n doubles each, any may be NULL (at least one not).  d2_dvdx is odd in v.
 * The differences of moments lose |S11/S0|/|d2_dv2| (and alike) in relative
 * precision -- the conditioning of the quantities themselves.  Options as for
 * bessel_logk_f64_ex (the WS kernel variant is not available).
 */
BLK_API blk_status bessel_logk_hess_f64(const double *v, const double *x, size_t n,
                                        double *logk, double *dlogk_dv, double *dlogk_dx,
                                        double *d2_dv2, double *d2_dx2, double *d2_dvdx,
                                        int nbins, const blk_options *opts,
                                        cudaStream_t stream);

/*
 * Normal-inverse-Gaussian log-likelihood of a sample and its gradient, the
 * application the paper motivates:
 *   out[0] = sum_i log p(y_i),  out[1..4] = d/d(alpha, beta, delta, mu) of it,
 *   log p(y) = log alpha + log delta - log pi + delta*gamma + beta*(y-mu)
 *              - log q + log K_1(alpha*q),  q = sqrt(delta^2+(y-mu)^2),
 *              gamma = sqrt(alpha^2 - beta^2),
 * with log K_1 and dlogK_1/dz from the same plan + fixed-bin quadrature (v=1).
 * y: DEVICE, n doubles.  out: DEVICE, 5 doubles (written, not accumulated).
 * workspace: DEVICE, >= bessel_nig_workspace_bytes(n) bytes, caller-owned.
 * Two kernels on `stream`; the block partials are reduced in a fixed order,
 * so the result is bit-reproducible.  BLK_EINVAL unless |beta| < alpha,
 * delta > 0 and all parameters finite.  n == 0 writes zeros.
 */
BLK_API size_t bessel_nig_workspace_bytes(size_t n);
BLK_API blk_status bessel_nig_loglik_f64(const double *y, size_t n, double alpha,
                                         double beta, double delta, double mu, int nbins,
                                         double *out, void *workspace,
                                         size_t workspace_bytes, cudaStream_t stream);

/* Human-readable message for the last non-OK status on this thread. */
BLK_API const char *bessel_logk_last_error(void);

/* Library version string. */
BLK_API const char *bessel_logk_version(void);

/*
 * Peak-rate microbenchmarks used as the roofline denominators (bench.py):
 * each thread runs `iters` iterations of BLK_MB_UNROLL instructions spread
 * over 8 independent dependency chains; out (device, blocks*threads
 * elements) receives a data-dependent value so the work cannot be elided.
 *   ops = blocks * threads * iters * BLK_MB_UNROLL
 *   fp64: DFMA (2 flops each); fp32: FFMA (2 flops each); mufu: MUFU.EX2
 */
#define BLK_MB_UNROLL 16
BLK_API blk_status blk_microbench_fp64(int blocks, int threads, int iters, double *out,
                               cudaStream_t stream);
BLK_API blk_status blk_microbench_fp32(int blocks, int threads, int iters, float *out,
                               cudaStream_t stream);
BLK_API blk_status blk_microbench_mufu(int blocks, int threads, int iters, float *out,
                               cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* BESSEL_LOGK_H */
