/*
 * smnn.h -- C ABI of the B200-native S-MNN hot path (arXiv 2410.06074).
 *
 * One *instance* is one (batch, ODE-dim) pair of the paper's linear ODE
 * (PAPER.md:68-80 with V = Q = 1): a single variable y of derivative order
 * R = `order`, T time points, initial values at the first time point only
 * (T_init = 1, R_init = n_iv - 1).  Instances are
 * independent; a call processes `n_inst` = B*D of them.
 *
 * Tensor layouts (row-major, instance outermost, "paper layout" of
 * BASELINE.json north_star; b = R + 1 is the block size of PAPER.md:158):
 *   coeffs [n_inst, T, b]     c_{t,r}  of sum_r c_{t,r} y^{(r)}_t = d_t
 *   rhs    [n_inst, T]        d_t
 *   iv     [n_inst, n_iv]     u_r, r < n_iv, at t = 0
 *   steps  [n_inst, T-1]      s_t = span between t and t+1, > 0
 *   y      [n_inst, T, b]     y_{t,r}, the solution of Eq. least_squares
 *   grad_* same shape as the tensor they differentiate.
 *   M_diag [n_inst, T, b, b]  M_t = M_{t,t}        (App. A.1 :625-634)
 *   N_sub  [n_inst, T-1, b, b] N_t = M_{t+1,t}     (lower off-diagonal block)
 *   beta   [n_inst, T, b]     beta_t
 *   L      [n_inst, T, b, b]  lower-triangular Cholesky blocks, zeros above the diagonal
 *   P      [n_inst, T-1, b, b] LDL multipliers, P L L^T P^T = M
 *
 * Element type: `dtype` selects storage and arithmetic:
 *   SMNN_F32      float storage, float arithmetic
 *   SMNN_F64      double storage, double arithmetic
 *   SMNN_F32_C64  float storage, double arithmetic (fp32 HBM traffic,
 *                 fp64-accurate normal equations)
 *
 * Memory: unless stated otherwise every pointer is a DEVICE pointer on the
 * current CUDA device, owned by the caller, not retained after the call;
 * inputs are read-only, outputs are fully overwritten.  Calls are
 * asynchronous on `stream` (a cudaStream_t, NULL = legacy default stream).
 *
 * Errors: every entry point returns SMNN_OK (0) or a negative code; the
 * message of the last failure on the calling thread is returned by
 * smnn_last_error().  Argument errors are detected before any launch.
 * Numerical breakdown (a non-positive or non-finite Cholesky pivot, i.e.
 * M not numerically SPD) is reported per instance in `info` (may be NULL):
 * info[i] = 0 on success, else 1 + a time index t0 <= t of the failing block
 * t (like LAPACK potrf, which reports t itself): the time-parallel solver
 * checks its pivots once per time chunk and reports the chunk's first point,
 * or the separator point when the breakdown is in the separator system.  The
 * outputs of such an instance are undefined.
 */
#ifndef SMNN_H_
#define SMNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMNN_F32 0
#define SMNN_F64 1
#define SMNN_F32_C64 2

#define SMNN_OK 0
#define SMNN_ERR_ARG (-1)         /* invalid argument / shape / null pointer      */
#define SMNN_ERR_CUDA (-2)        /* a CUDA runtime call or launch failed        */
#define SMNN_ERR_UNSUPPORTED (-3) /* order > 3, or dtype unknown                 */
#define SMNN_ERR_WORKSPACE (-4)   /* workspace_bytes < smnn_workspace_bytes()    */

#define SMNN_MAX_ORDER 3

typedef struct smnn_problem {
  int64_t n_inst;   /* number of independent instances (B*D), >= 1              */
  int32_t T;        /* time points per instance, >= 1                            */
  int32_t order;    /* R in 0..3; block size b = R + 1                           */
  int32_t n_iv;     /* initial values per instance, 1..R+1 (R_init = n_iv - 1)   */
  int32_t dtype;    /* SMNN_F32 | SMNN_F64 | SMNN_F32_C64                        */
  int32_t threads_per_inst; /* time-chunks (= CUDA threads) per instance; 0 = auto */
  int32_t path;     /* kernel path: 0 = automatic (recommended), or an SMNN_PATH_*
                       code to force one (tests / measurements; a forced path the
                       problem does not fit falls back to the automatic order)    */
  double w_gov;     /* importance weights of PAPER.md:130, all > 0               */
  double w_init;
  double w_smooth;
} smnn_problem;

/* Library identification and the last error message of this thread. */
const char* smnn_version(void);
const char* smnn_last_error(void);

/* Which kernels smnn_factor_solve_fwd (bwd = 0) / smnn_solve_bwd (bwd = 1)
 * run for `p` on this build (p->path = 0: the automatic choice):
 *   SMNN_PATH_RF          one launch: resident register-factor kernel (one CTA
 *                         per instance, whole instance in shared memory; fp32)
 *   SMNN_PATH_PIPE        three launches: chunk pass 1, separator reduction,
 *                         chunk pass 2 (long horizons; needs the workspace)
 *   SMNN_PATH_CHECKPOINT  one launch: checkpointing resident / streaming kernel
 *   SMNN_PATH_X64         one cluster launch: fp64-arithmetic cluster-resident
 *                         kernel (SMNN_F64, SMNN_F32_C64)
 * SMNN_PATH_STREAM is accepted in p->path only: the checkpoint path with its
 * streaming (non-resident) kernel.  Returns a negative SMNN_ERR_* code on an
 * invalid `p`. */
#define SMNN_PATH_RF 1
#define SMNN_PATH_PIPE 2
#define SMNN_PATH_CHECKPOINT 3
#define SMNN_PATH_X64 4
#define SMNN_PATH_STREAM 5
int smnn_kernel_path(const smnn_problem* p, int bwd);

/* Number of kernel launches one smnn_factor_solve_fwd (bwd = 0) /
 * smnn_solve_bwd (bwd = 1) call makes for `p` with every output requested
 * (SMNN_F32_C64 backward on a path that reads y from storage runs as SMNN_F64
 * on promoted copies: widening, fp64 forward + backward, narrowing; see
 * smnn_solve_bwd).  Negative SMNN_ERR_* code on an invalid `p`. */
int smnn_launch_count(const smnn_problem* p, int bwd);

/* Bytes of device workspace the fused kernels need for `p` on the current
 * device (checkpoint scratch of the time-parallel solver, one slot per
 * resident CTA).  Pass at least this much to smnn_factor_solve_fwd /
 * smnn_solve_bwd.  Returns 0 and sets the error on invalid `p`. */
size_t smnn_workspace_bytes(const smnn_problem* p);

/* Appendix A.1: assemble the non-zero blocks of
 * M = A^T W A and beta = A^T W b for every instance.  Outputs M_diag, N_sub,
 * beta in the storage type of `dtype`.  N_sub may be NULL when T == 1. */
int smnn_assemble(const smnn_problem* p, const void* coeffs, const void* rhs,
                  const void* iv, const void* steps, void* M_diag, void* N_sub,
                  void* beta, void* stream);

/* Fused forward pass (Algorithm 1 = assemble + Decompose + Substitute,
 * PAPER.md:216-234, 239-263, 293-315): y = M^{-1} beta per instance, with M
 * and beta assembled in registers (never written to HBM) and the block
 * Cholesky / substitution split over time chunks (DESIGN.md "Time-parallel
 * partition solver").  `workspace` must hold smnn_workspace_bytes(p). */
int smnn_factor_solve_fwd(const smnn_problem* p, const void* coeffs, const void* rhs,
                          const void* iv, const void* steps, void* y, int32_t* info,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Fused backward pass (Algorithm 2, chained
 * through Appendix A.1): given y from the forward pass and grad_y = dl/dy,
 * computes dl/dbeta = M^{-1} dl/dy by re-factoring M in registers, then
 * dl/dcoeffs, dl/drhs, dl/div, dl/dsteps.  Any grad_* output may be NULL to
 * skip it.  The gradients are those of the exact solution y(c, d, u, s):
 * SMNN_F32 and SMNN_F64 read y from `y`; SMNN_F32_C64 does not trust the
 * fp32 rounding of y (the residual terms of the chain amplify it ~1e4x) and
 * recomputes y in fp64 -- the x64 kernel solves for y and dl/dbeta together,
 * every other path runs the backward as SMNN_F64 on fp64 copies of the
 * inputs widened in the workspace (smnn_launch_count reports the launches). */
int smnn_solve_bwd(const smnn_problem* p, const void* coeffs, const void* rhs,
                   const void* iv, const void* steps, const void* y, const void* grad_y,
                   void* grad_coeffs, void* grad_rhs, void* grad_iv, void* grad_steps,
                   int32_t* info, void* workspace, size_t workspace_bytes, void* stream);

/* The same two calls with the fp32 REMAINDER of y (SMNN_F32_C64 only).
 * The f32c64 forward computes y in fp64 and rounds it into the fp32 `y`; with
 * y_lo (device, [n_inst, T, b] float, nullable) it also writes
 * y_lo = fl32(y_fp64 - (double)y), so that (double)y + (double)y_lo carries
 * the fp64 solution to ~2^-48 relative.  smnn_solve_bwd_ex given that pair
 * reads y = y + y_lo in fp64 for the gradient chain (Algorithm 2's
 * dl/dM = -dl/dbeta y^T and the residual terms of Appendix A.1), instead of
 * re-solving y beside dl/dbeta: one right-hand side instead of two (the
 * same gradients up to rounding).  The pair is used only where
 * smnn_ylo_used(p) returns 1 (both directions on the pipeline); otherwise
 * the forward fills y_lo with zeros and the backward ignores it (y is then
 * re-solved as in smnn_solve_bwd).  For SMNN_F32 / SMNN_F64 y_lo must be
 * NULL-or-ignored: it is not read or written.  A y_lo that does not come
 * from the forward of the same inputs gives wrong gradients (not detected). */
int smnn_ylo_used(const smnn_problem* p);
int smnn_factor_solve_fwd_ex(const smnn_problem* p, const void* coeffs, const void* rhs,
                             const void* iv, const void* steps, void* y, void* y_lo, int32_t* info,
                             void* workspace, size_t workspace_bytes, void* stream);
int smnn_solve_bwd_ex(const smnn_problem* p, const void* coeffs, const void* rhs,
                      const void* iv, const void* steps, const void* y, const void* y_lo,
                      const void* grad_y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                      void* grad_steps, int32_t* info, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Algorithm 3 "Decompose", materialised: one sequential
 * sweep per instance writing L [n,T,b,b] and P [n,T-1,b,b] to HBM (the
 * paper's own data flow; used for parity and as the sequential baseline).
 * P may be NULL when T == 1. */
int smnn_factor(const smnn_problem* p, const void* coeffs, const void* steps,
                void* L, void* P, int32_t* info, void* stream);

/* Algorithm 4 "Substitute": out = M^{-1} alpha from the
 * materialised L, P of smnn_factor.  alpha, out: [n_inst, T, b]; may alias. */
int smnn_substitute(const smnn_problem* p, const void* L, const void* P,
                    const void* alpha, void* out, void* stream);

/* ------------------------------------------------------------------------
 * Host-buffer end-to-end plan (the call a user makes with data in host RAM).
 * A plan owns device buffers for one batch of shape `p`.  fwd_bwd_host copies
 * the HOST inputs in, runs smnn_factor_solve_fwd then smnn_solve_bwd, and
 * copies y and all gradients back to HOST memory.  The batch is split into up
 * to 8 groups of instances (about one per 16 MiB of input) pipelined over the
 * plan's own copy-in, compute and copy-out streams (H2D of a group overlaps the kernels of the previous one
 * and the D2H of the one before), ordered after the work already on `stream`,
 * and `stream` waits for the last copy-out: the call returns once the work is
 * enqueued (synchronise `stream` before reading the outputs).  A call is also
 * ordered after the plan's previous call, whatever stream that one used (the
 * device buffers are the plan's).  Host buffers must be page-locked for the
 * copies to overlap; each holds exactly the batch's elements of the plan's
 * storage type (the library copies that many bytes; no size is passed).
 * info (nullable, n_inst int32): the forward pass's breakdown code where it
 * reports one, else the backward pass's (same convention as
 * smnn_factor_solve_fwd).
 * ---------------------------------------------------------------------- */
typedef struct smnn_plan smnn_plan;

int smnn_plan_create(smnn_plan** plan, const smnn_problem* p);
int smnn_plan_destroy(smnn_plan* plan);
int smnn_plan_fwd_bwd_host(smnn_plan* plan, const void* coeffs, const void* rhs,
                           const void* iv, const void* steps, const void* grad_y,
                           void* y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                           void* grad_steps, int32_t* info, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SMNN_H_ */
