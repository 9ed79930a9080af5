/*
 * nlk_b200.h — C ABI of the B200 batched small-system nonlinear solver.
 *
 * This is the drop-in boundary for the reference's per-system solve path
 * (/root/reference/pkg/src/nlkit).  The reference is pure Python, so its
 * "interface" is the Python call
 *     nlkit.solvers.run_preset(name, Problem(residual, u0, params), SolveOptions(abstol, maxiters))
 *         -> SolveResult(u_star, resid_norm, retcode, stats)
 * (solvers.py:640-655, core.py:27-91, 158-169); each entry point below names the
 * reference piece it replaces.  The Python shim paper_2403_16341_b200 binds
 * these symbols with ctypes (see INTEGRATION.md for the nlkit-side binding).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch or CUDA types cross the boundary
 *     (streams are passed as void*; NULL = the legacy default stream);
 *   - a call with a stream runs on that stream's device (the current device
 *     is switched for the call and restored); with the NULL stream it runs
 *     on the current device;
 *   - batch arrays are structure-of-arrays: u0/u_out are [n][B] (element i of
 *     system b at i*B + b), p is [m][B];
 *   - dtype 0 = IEEE binary64 (the reference's arithmetic), 1 = binary32;
 *   - retcode values are nlkit's RetCode in declaration order
 *     (core.py:17-24): 0 Success, 1 MaxIters, 2 LineSearchFailed,
 *     3 LinearSolveFailed, 4 Stalled, 5 NonFinite;
 *   - per-system numerical failures are NEVER errors (they are retcodes);
 *     API misuse returns a negative status and sets nlk_last_error().
 *   - entry points are re-entrant; the registry is immutable; the library keeps
 *     no pointer after a call returns.
 */
#ifndef NLK_B200_H
#define NLK_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define NLK_API __attribute__((visibility("default")))
#else
#define NLK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NLK_OK 0
#define NLK_ERR_UNKNOWN_PROBLEM (-1)  /* KeyError in problems.get_problem (problems.py:459,474) */
#define NLK_ERR_BAD_SIZE (-2)         /* n not compiled for this problem */
#define NLK_ERR_UNKNOWN_ALG (-3)      /* KeyError in run_preset (solvers.py:649-650) */
#define NLK_ERR_BAD_OPTIONS (-4)      /* ValueError in SolveOptions (core.py:61-65) */
#define NLK_ERR_BAD_ARGUMENT (-5)     /* null buffer, negative B, missing params */
#define NLK_ERR_NOT_COMPILED (-6)     /* (problem, n, alg, dtype) has no kernel */
#define NLK_ERR_CUDA (-7)             /* CUDA runtime error (message in nlk_last_error) */

/* algorithm ids; names match ALGORITHM_PRESETS (solvers.py:610-637) */
#define NLK_ALG_NEWTON_RAPHSON 0     /* "newton-raphson"      = SimpleNewtonRaphson */
#define NLK_ALG_TRUST_REGION 1       /* "trust-region"        = SimpleTrustRegion   */
#define NLK_ALG_BROYDEN 2            /* "broyden"             = SimpleBroyden       */
#define NLK_ALG_KLEMENT 3            /* "klement"             = SimpleKlement       */
#define NLK_ALG_DFSANE 4             /* "dfsane"              = SimpleDFSane (no nlkit counterpart) */
#define NLK_ALG_NEWTON_BACKTRACKING 5 /* "newton-backtracking" (solvers.py:613) */

#define NLK_F64 0
#define NLK_F32 1

/* Library version (major*10000 + minor*100 + patch). */
NLK_API int nlk_version(void);

/* Hash of the sources the library was built from (csrc/, include/):
 * the first 16 hex digits of the SHA-256 over the sorted file names and
 * contents, computed by paper_2403_16341_b200/build.py at build time.
 * _lib.source_build_id() recomputes it from a source tree, so a caller can
 * prove that the loaded binary is the one its sources describe. */
NLK_API const char* nlk_build_id(void);

/* Message of the last failed call on this thread ("" if none). */
NLK_API const char* nlk_last_error(void);

/* Resolve a preset name to an algorithm id (replaces the ALGORITHM_PRESETS
 * lookup in run_preset, solvers.py:649-651).  Returns NLK_ERR_UNKNOWN_ALG
 * for names without a batched kernel. */
NLK_API int nlk_alg_lookup(const char* name);

/* Number of compiled (problem, n) instances and their description. */
NLK_API int nlk_num_problems(void);
NLK_API int nlk_problem_info(int32_t handle, const char** id, int32_t* n, int32_t* m);

/* Resolve an nlkit problem id (problems.py:450-474 naming: "test23/<name>",
 * "quadratic", "generalized_rosenbrock") at size n (0 = the problem's fixed
 * size).  Replaces binding Problem.residual to a Python callable
 * (core.py:35): the residual is a compiled device function. */
NLK_API int nlk_problem_lookup(const char* id, int32_t n, int32_t* handle, int32_t* n_out, int32_t* m_out);

/* Solve B independent systems already resident on the current device.
 * Replaces B calls of run_preset(alg, Problem(residual, u0_b, p_b),
 * SolveOptions(abstol, maxiters)) (solvers.py:640-655): writes u_star
 * (u_out), resid_norm = max|f(u_star)| (resid_out), retcode and the
 * Stats counters nsteps/nf/njac/nlinsolve (core.py:68-91).  Counter
 * pointers may be NULL.  Asynchronous on `stream`. */
NLK_API int nlk_solve_batch(int32_t handle, int32_t alg, int32_t dtype, int64_t B,
                    const void* u0_soa, const void* p_soa, double abstol, int32_t maxiters,
                    void* u_out, void* resid_out, int8_t* retcode_out, int32_t* nsteps_out,
                    int32_t* nf_out, int32_t* njac_out, int32_t* nlinsolve_out, void* stream);

/* The default poly-algorithm for a batch: replaces B calls of
 * nlkit.solve(Problem(...)) / run_polyalgorithm(problem, options)
 * (core.py:158-169, solvers.py:570-599).  Every registered problem has
 * n <= QN_SKIP_THRESHOLD = 25, so the quasi-Newton stages are skipped and
 * the stages are newton-raphson -> newton-backtracking -> trust-region
 * (solvers.py:553-565), each with the full iteration budget.  A stage runs
 * only on the systems no earlier stage solved; outputs are the first
 * success, else the stage result with the smallest residual max-norm (the
 * earliest on ties); the four counters are summed over the stages that ran.
 * stage_retcodes_out is int8 [3][B]: the RetCode of stage s for system b at
 * s*B + b, -1 where the stage did not run (SolveResult.stage_retcodes).
 * Device buffers, asynchronous on `stream` (three launches, no host sync). */
NLK_API int nlk_solve_batch_poly(int32_t handle, int32_t dtype, int64_t B, const void* u0_soa,
                                 const void* p_soa, double abstol, int32_t maxiters,
                                 void* u_out, void* resid_out, int8_t* retcode_out,
                                 int32_t* nsteps_out, int32_t* nf_out, int32_t* njac_out,
                                 int32_t* nlinsolve_out, int8_t* stage_retcodes_out,
                                 void* stream);

/* Same contract with HOST buffers (pageable or pinned): the library stages
 * the batch through device memory in chunks, overlapping host<->device copies
 * with the solve on `num_streams` streams, and returns when results are in
 * the host buffers.  This is the call a CPU caller of nlkit switches to. */
NLK_API int nlk_solve_batch_host(int32_t handle, int32_t alg, int32_t dtype, int64_t B,
                         const void* u0_soa, const void* p_soa, double abstol, int32_t maxiters,
                         void* u_out, void* resid_out, int8_t* retcode_out, int32_t* nsteps_out,
                         int32_t* nf_out, int32_t* njac_out, int32_t* nlinsolve_out,
                         int64_t chunk, int32_t num_streams);

/* Asynchronous host-buffer solve: enqueues on `stream` the stream-ordered
 * allocation of a device staging area, the host->device copy of u0/p, the
 * solve, the device->host copy of every output and the release of the
 * staging area, then returns.  Host buffers must stay valid until the stream
 * reaches that point (synchronise it, or record an event); with pinned host
 * memory the copies overlap other work on other streams, so a caller can keep
 * several batches in flight (e.g. one stream per problem batch).  Same
 * outputs as nlk_solve_batch_host. */
NLK_API int nlk_solve_batch_host_async(int32_t handle, int32_t alg, int32_t dtype, int64_t B,
                         const void* u0_soa, const void* p_soa, double abstol, int32_t maxiters,
                         void* u_out, void* resid_out, int8_t* retcode_out, int32_t* nsteps_out,
                         int32_t* nf_out, int32_t* njac_out, int32_t* nlinsolve_out,
                         void* stream);

/* Number of blocks the last nlk_solve_batch launch on this thread used
 * (diagnostics for the persistent grid). */
NLK_API int nlk_last_grid(void);

/* Number of kernels the last nlk_solve_batch launch on this thread issued: 1,
 * or 2 where a closed-form problem's fast Newton / trust-region kernel is
 * followed by the kernel that completes its deferred systems (diagnostics;
 * bench.py's gpu_launches). */
NLK_API int nlk_last_launches(void);

/* Measured FP64 FMA-pipe throughput of the current device in TFLOP/s (8
 * independent DFMA chains per thread, all SMs; synchronous on `stream`).
 * The roofline denominator for the solve kernels, which are FP64-issue
 * bound rather than HBM- or tensor-bound. */
NLK_API int nlk_fp64_peak(int64_t iters, double* tflops_out, void* stream);
/* The same for the FP32 FMA pipe (FFMA chains): the roofline denominator of
 * the fp32 instantiations. */
NLK_API int nlk_fp32_peak(int64_t iters, double* tflops_out, void* stream);

/* Implicit-function-theorem sensitivities at B roots of one parametrised
 * problem (m > 0), device buffers, asynchronous on `stream`.
 *   nlk_ift_forward_batch  replaces sensitivity.ift_forward(problem, u_star,
 *     theta, abstol, full) (sensitivity.py:40-57): S_out = d(u_star)/d(theta),
 *     [n*m][B] with S[i][j] of system b at (i*m + j)*B + b;
 *   nlk_ift_adjoint_batch  replaces sensitivity.ift_adjoint(problem, u_star,
 *     theta, gbar, abstol, full) (sensitivity.py:60-80): grad_out [m][B].
 * u_star_soa [n][B], theta_soa [m][B], gbar_soa [n][B].  solve_resid_out
 * ([B], may be NULL) is the `full=True` SensitivityResult.solve_residual.
 * status_out[b]: 0 ok, 1 not a root (the reference raises ValueError,
 * sensitivity.py:31-36), 2 SingularMatrix (strict LU, linalg.py:87-105),
 * 3 NonFiniteValue (dual evaluation); outputs of a failed system are NaN.
 * dtype must be 0 (f64). */
NLK_API int nlk_ift_forward_batch(int32_t handle, int32_t dtype, int64_t B, const void* u_star_soa,
                                  const void* theta_soa, double abstol, void* S_out,
                                  void* solve_resid_out, int8_t* status_out, void* stream);
NLK_API int nlk_ift_adjoint_batch(int32_t handle, int32_t dtype, int64_t B, const void* u_star_soa,
                                  const void* theta_soa, const void* gbar_soa, double abstol,
                                  void* grad_out, void* solve_resid_out, int8_t* status_out,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NLK_B200_H */
