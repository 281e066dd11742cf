/*
 * pint.h -- C ABI of libpint.so, the B200 (sm_100a) implementation of the
 * inexact-Uzawa hot path of arXiv 1802.08126 (reference package `pintsolve`,
 * /root/reference/pkg/src/pintsolve).
 *
 * The reference exposes this path as a duck-typed Python operator protocol
 * (SURVEY.md 8(b)); every entry point below replaces one reference callable,
 * cited as file:line relative to pkg/src/pintsolve/.  The Python package
 * paper_1802_08126_b200 binds these with ctypes, and any
 * other FFI (cffi, JNI, cgo) can bind them the same way: plain pointers and
 * sizes, no torch or numpy types.
 *
 * Data layout.  A "block vector" is a time-major slab of N_local x n fp64
 * values, row r = time step (or DST mode) r, column = interior spatial node
 * in the reference numbering (2D: j*(c-1)+i, x fastest; 3D: (k*(c-1)+j)*(c-1)+i),
 * i.e. exactly the C-order numpy array of shape (N, dim) the reference uses.
 *
 * Pointers.  Every `const double* in` / `double* out` argument may be a host
 * pointer (pageable or pinned) or a device pointer on the context's device;
 * the library detects which (cudaPointerGetAttributes) and stages host
 * buffers through context-owned device memory.  All work is ordered on the
 * context's stream; calls return after the result is in `out`.
 *
 * Status codes map one-to-one onto the reference exception taxonomy
 * (errors.py:4-25): PINT_INPUT -> InputError, PINT_DIMENSION ->
 * DimensionMismatchError, PINT_NOT_SPD -> NotSpdError, PINT_DIVERGED ->
 * SolverDivergenceError.  pint_last_error() returns the message.
 */
#ifndef PINT_H
#define PINT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PINT_OK 0
#define PINT_INPUT 1       /* errors.py:4  InputError */
#define PINT_DIMENSION 2   /* errors.py:8  DimensionMismatchError */
#define PINT_NOT_SPD 3     /* errors.py:12 NotSpdError */
#define PINT_DIVERGED 4    /* errors.py:20 SolverDivergenceError */
#define PINT_CUDA 5        /* device / driver / NCCL failure */

/* which batched multigrid set a call refers to */
#define PINT_MG_ATILDE 0   /* per-step blocks of A~ (solvers.py:127-155) */
#define PINT_MG_HTILDE 1   /* per-mode blocks H_k of H~ (schur.py:30-52) */
#define PINT_MG_EULER 2    /* per-step M + tau_n A_n of the sequential oracle (solvers.py:166-170) */

typedef struct pint_ctx pint_ctx;

/* Version of the ABI described by this header. */
int pint_abi_version(void);

/* Create a context on CUDA device `device`.  `rank`/`world` describe the
 * time-axis partition (rank r owns steps [n0, n0+N_local)); world must be 1
 * in this build.  `nccl_id` is reserved (NULL).  Replaces the process-global
 * thread pool of parallel.py:19-43 as the unit of execution. */
int pint_ctx_create(int device, int rank, int world, const void* nccl_id, pint_ctx** out);
int pint_ctx_destroy(pint_ctx* ctx);
const char* pint_last_error(const pint_ctx* ctx);
/* Synchronise the context stream. */
int pint_sync(pint_ctx* ctx);
/* Order all further work on a caller-owned cudaStream_t (e.g. the current
 * torch stream; 0 = the legacy default stream); own != 0 restores the
 * context's own stream. */
int pint_set_stream(pint_ctx* ctx, void* stream, int own);
/* Arithmetic of the 2D band kernels (time operators, multigrid):
 * exact != 0: no FMA contraction, every stencil / V-cycle row sum in scipy's
 *             CSR order, bit-identical to the reference (linalg.py:96-97,
 *             spatial.py:148-161);
 * exact == 0: FMA-contracted (the default; <= 1e-15 relative per operator,
 *             Uzawa histories within the reference's own DST-path noise).
 * The initial value is taken from the environment variable PINT_EXACT. */
int pint_set_arith(pint_ctx* ctx, int exact);
int pint_get_arith(const pint_ctx* ctx);

/* ---------------------------------------------------------------------------
 * Problem: the spatial stencils, step sizes and stiffness scales of one
 * ProblemSpec (problems.py:153-182) as consumed by TimeGlobalSystem
 * (operators.py:29-99).
 *
 *   dims        2 or 3 (3: unit cube, Kuhn-split P1, 27-point tables; ops3d.cu)
 *   m           interior points per side (cells - 1)
 *   N           time steps owned by this context
 *   steps[N]    tau_n (TimeGrid.steps, problems.py:49-51)
 *   mass[S]     mass stencil, S = 3^dims coefficients in CSR column order
 *               (2D: SW,S,SE,W,C,E,NW,N,NE); absent entries are 0
 *   n_a         number of distinct stiffness stencils
 *   a_st[n_a*S] stiffness stencils
 *   a_sid[N]    stencil used by step n
 *   a_scale[N]  factor s_n with  A-block_n u = s_n * (a_st[a_sid[n]] u)
 *               (operators.py:92-99: c_n*tau_n when proportional, else tau_n)
 *   aref[S]     reference stiffness A_ref stencil (schur.py:72)
 *   tau_ref     reference step (problems.py:283)
 * ------------------------------------------------------------------------- */
int pint_problem_set(pint_ctx* ctx, int dims, int m, int N,
                     const double* steps, const double* mass,
                     int n_a, const double* a_st, const int* a_sid, const double* a_scale,
                     const double* aref, double tau_ref);

/* fold_rhs (operators.py:22-26): f_n = tau_n load_n, f_1 += M u_init. */
int pint_fold_rhs(pint_ctx* ctx, const double* load, const double* u_init, double* f);

/* apply_K / apply_Kt / apply_Abd (operators.py:78-99). */
int pint_apply_K(pint_ctx* ctx, const double* in, double* out);
int pint_apply_Kt(pint_ctx* ctx, const double* in, double* out);
int pint_apply_Abd(pint_ctx* ctx, const double* in, double* out);

/* ---------------------------------------------------------------------------
 * Batched multigrid sets (spatial.py:116-169, one V-cycle, 1 pre + 1 post
 * damped-Jacobi sweep, Galerkin coarse operators, direct coarsest solve).
 *
 *   levels        number of grids, fine to coarse (spatial.py:100-113)
 *   level_m[L]    interior points per side on each level
 *   n_sets        number of distinct operators (hierarchies)
 *   tables[L*n_sets*(S+1)]  per (level, set): S stencil coefficients in CSR
 *                 order followed by dinv = damping/diag (spatial.py:142);
 *                 on the coarsest level only the centre coefficient is used
 *                 (1x1 direct solve, spatial.py:143,149-150)
 *   sid[B]        operator set of each batch plane (B = N: steps or modes)
 * ------------------------------------------------------------------------- */
int pint_mg_set(pint_ctx* ctx, int which, int levels, const int* level_m,
                int n_sets, const double* tables, const int* sid);
/* V-cycle options of a configured set (MgVCycleSolver(cycles=, smooth_steps=),
 * spatial.py:116-169): `cycles` V-cycles with residual correction
 * (spatial.py:163-169) and `smooth_steps` damped-Jacobi sweeps before and
 * after the coarse correction (spatial.py:152-160).  (1, 1), the setting of
 * every BASELINE config and the default after pint_mg_set, runs the fused
 * band kernels; anything else runs general thread-per-point kernels
 * (mg_generic.cu), bit-identical to the reference's products.  Not available
 * for field mode. */
int pint_mg_set_options(pint_ctx* ctx, int which, int cycles, int smooth_steps);

/* ---------------------------------------------------------------------------
 * Field mode (EXTENSION, BASELINE config 4): 2D stiffness operators that are
 * not translation invariant, e.g. -div(a(x, t) grad u).  Replaces, for the
 * structured 2D grids, the reference's general per-step branch: a list of
 * distinct A_n (problems.py:153-165), tau_n A_n u_n (operators.py:92-99) and
 * one multigrid hierarchy per distinct A_n (solvers.py:134-140).  Once any
 * field is set, the stiffness stencils given to pint_problem_set are unused.
 *
 * Compact fields of a symmetric P1 operator: three planes [3][n] holding the
 * centre, east (i, i+1) and north (i, i+m) coefficient of every row.
 * ------------------------------------------------------------------------- */
/* fields[count][3][n] (host or device) -> steps [step0, step0 + count). */
int pint_field_set(pint_ctx* ctx, int step0, int count, const double* fields);
/* Assemble steps [step0, step0 + count) on the GPU from per-cell weights
 * cell_w[count][cells][cells] ([j][i] for cell (i, j)), the element loop of
 * problems.py:99-138 with w_e K_e (bit-identical to the scipy assembly). */
int pint_field_assemble(pint_ctx* ctx, int step0, int count, const double* cell_w);
/* Separable family (instead of pint_field_set / pint_field_assemble): the
 * cell weight of step n is sum_r weights[n][r] * cell_w[r] (terms <=
 * PINT_FSEP_MAX = 3; config 4: a = (1 + 0.1 U) + (0.5 sin 2 pi t_n) r^2).
 * The stiffness is linear in the weight, so A_n = sum_r weights[n][r] A(w_r)
 * and, because the Galerkin product is linear too, every coarse operator is
 * the same combination of `terms` coarse tables: the device keeps
 * [terms][3][n] fine and [terms][9][m_l^2] coarse tables (cache resident)
 * instead of [N][3][n] / [N][9][m_l^2] slabs (25.7 + 2 x 25.6 GB at config 4)
 * and forms every coefficient in registers.  The H~ set of such a problem
 * uses the same form with the two terms (M, A_ref) and weights (mu_k,
 * tau_ref).  Each coefficient differs from the per-step assembly by
 * rounding (a few ulps), so this path is held to a tolerance, not to bit
 * equality (tests/test_gpu_field.py). */
int pint_field_separable(pint_ctx* ctx, int terms, const double* cell_w, const double* weights);
/* A_ref (schur.py:41-47): fields[3][n], or (fields == NULL) a copy of step `step`. */
int pint_field_aref(pint_ctx* ctx, int step, const double* fields);
/* Field multigrid set: Galerkin coarse rows of every step (A~) or mode
 * (H~, mu[N] = frequency weights) built on the GPU, bit-identical to
 * (P^T A) P of spatial.py:140; damping as spatial.py:136. */
int pint_mg_set_field(pint_ctx* ctx, int which, int levels, const int* level_m, double damping,
                      const double* mu);

/* One V-cycle per plane, planes [0, count) of the set (spatial.py:163-169). */
int pint_vcycle(pint_ctx* ctx, int which, int count, const double* in, double* out);

/* A~^{-1}: out_n = V_n(in_n) / tau_n  (BlockDiagSolver.apply_inverse, solvers.py:143-150). */
int pint_atilde_inv(pint_ctx* ctx, const double* in, double* out);

/* H~^{-1}: DST^T, per-mode V-cycle / A_ref / V-cycle scaled by 2 tau_ref / N,
 * DST  (SchurPreconditioner.apply_inverse, schur.py:62-76). */
int pint_htilde_inv(pint_ctx* ctx, const double* in, double* out);

/* Sine transforms along the time axis (dst.py:57-93).
 *   kind 0 inverse            u_n  = sum_k uh_k sin((2k-1) n pi / 2N)     dst.py:67-73
 *   kind 1 inverse_transpose  rh_k = sum_n r_n  sin((2k-1) n pi / 2N)     dst.py:86-93
 *   kind 2 forward            (2/N) * kind1 with the last input row halved dst.py:57-65
 *   kind 3 forward_transpose  (2/N) * kind0, last output row halved        dst.py:75-84  */
int pint_dst(pint_ctx* ctx, int kind, const double* in, double* out);
/* Same transforms on any (N, ncols) slab, independent of the problem
 * (DstPlan(N) used standalone, dst.py:31-55). */
int pint_dst_raw(pint_ctx* ctx, int kind, int N, long long ncols, const double* in, double* out);
/* out = base + alpha * T(in) in one pass (the Uzawa u += omega S^T w of a
 * time partition whose columns are complete, solvers.py:231); device only. */
int pint_dst_raw_axpy(pint_ctx* ctx, int kind, int N, long long ncols, const double* in,
                      double* out, const double* base, double alpha);

/* ---------------------------------------------------------------------------
 * Uzawa iteration (uzawa_solve, solvers.py:177-264), state resident on the
 * device.  begin() copies f, p, u in (p, u may be NULL for zeros) and
 * returns ref = sqrt(max(f.A~^-1 f + f.H~^-1 f, 0)) (solvers.py:212-217).
 * step() runs one iteration (solvers.py:224-233) and returns
 * the residual numerator sqrt(max(sum r1.dp + sum z.y, 0)) (not divided by ref).
 * end() copies p, u out.  pint_uzawa() is the whole loop, with the
 * reference's stopping rule (res < tol after recording) and divergence guard
 * (res > 1e6*first_res -> PINT_DIVERGED); res_hist[max_iter] receives the
 * residuals, *iters the count, phase_ms[3] = {dst, multigrid, other} device ms.
 * ------------------------------------------------------------------------- */
int pint_uzawa_begin(pint_ctx* ctx, const double* f, const double* p0, const double* u0,
                     double* ref_out);
int pint_uzawa_step(pint_ctx* ctx, double omega, double* res_num_out);
int pint_uzawa_end(pint_ctx* ctx, double* p, double* u);
/* Host output buffers (p, u of pint_uzawa_end) may be fresh pageable
 * allocations; this starts background first-touch of their pages so the
 * device-to-host copy later runs at copy-engine rate.  Asynchronous; the next
 * host copy out of this context waits for it.  Device pointers are ignored.
 * (No reference counterpart: a transfer-path detail of uzawa_solve's
 * numpy-in/numpy-out contract, solvers.py:177-264.) */
int pint_host_prefault(pint_ctx* ctx, void* host, long long bytes);
/* Wait for every background first-touch started by pint_host_prefault.  Call
 * before releasing a prefaulted buffer that no copy-out has consumed (error
 * paths of the caller's loop). */
int pint_host_prefault_join(pint_ctx* ctx);
int pint_uzawa(pint_ctx* ctx, const double* f, double* p, double* u, double omega,
               double tol, int max_iter, int use_initial, double* res_hist, int* iters,
               int* converged, double* phase_ms);

/* ---------------------------------------------------------------------------
 * MINRES building blocks (minres_solve, solvers.py:267-327).  Device pointers.
 * apply_saddle: top = Abd p - K u, bottom = -Kt p - ((K u + Kt u) + Abd u)
 *   (TimeGlobalSystem.apply_saddle, operators.py:107-111), bit-identical.
 * lincomb: out[i] = ((x0[i] + a1*x1[i]) + a2*x2[i]) * (use_scale ? scale : 1),
 *   x1/x2 may be NULL (term skipped): the operation order of numpy's
 *   v - a*w1 - b*w2, s*y and x + phi*w in scipy's minres.
 * dot: sum a[i]*b[i] (deterministic tree order; not numpy's BLAS order).
 * ------------------------------------------------------------------------- */
int pint_apply_saddle(pint_ctx* ctx, const double* p, const double* u, double* top,
                      double* bottom);
int pint_lincomb(pint_ctx* ctx, double* out, long long count, const double* x0, double a1,
                 const double* x1, double a2, const double* x2, double scale, int use_scale);
int pint_dot(pint_ctx* ctx, const double* a, const double* b, long long count, double* out);

/* ---------------------------------------------------------------------------
 * Time-partitioned building blocks (one context per rank).  The
 * driver (paper_1802_08126_b200/distributed.py) moves ghost planes and
 * transposes with torch.distributed; these calls do the arithmetic.  All
 * pointers must be device pointers.  Every call is stream-ordered on the
 * context stream (pint_set_stream: the caller's, so NCCL and these kernels
 * order without host waits); none blocks the host except when a `dot`
 * output is a host pointer.
 *
 * pint_set_partition: this context's N steps are global steps [n0, n0+N) of
 *   N_global.  With has_prev / has_next the u and p slabs passed to the
 *   residual calls carry the neighbours' boundary planes at local plane -1 / N
 *   (the pointer still addresses local plane 0).
 * pint_residual_r1 / _z: r1 = K u - A p - f, z = f - K^T p - (K u + K^T u + A u)
 *   over the local steps (solvers.py:224, 227-229).
 * pint_atilde_update: p += A~^{-1} r1, *dot = sum r1.dp over the local steps
 *   (solvers.py:225-226, 233); p == NULL: only *dot = sum r1.(A~^{-1} r1).
 *   `dot` may be a device pointer (stream-ordered copy) or a host pointer
 *   (the call then waits for the stream), or NULL; same for htilde_modes.
 * pint_htilde_modes: for this rank's DST modes zh, w = (2 tau_ref/N_global)
 *   V_H(A_ref V_H(zh)) and *dot = sum zh.w (schur.py:69-75); w == NULL: dot only.
 * pint_axpy: u = u + omega*y on `count` values (solvers.py:231).
 * ------------------------------------------------------------------------- */
int pint_set_partition(pint_ctx* ctx, int n0, int N_global, int has_prev, int has_next);
int pint_residual_r1(pint_ctx* ctx, const double* u, const double* p, const double* f, double* r1);
int pint_residual_z(pint_ctx* ctx, const double* u, const double* p, const double* f, double* z);
int pint_atilde_update(pint_ctx* ctx, const double* r1, double* p, double* dot);
int pint_htilde_modes(pint_ctx* ctx, const double* zh, double* w, double* dot);
int pint_axpy(pint_ctx* ctx, double* u, const double* y, double omega, long long count);

/* Enable per-phase CUDA-event timing of pint_uzawa_step (on != 0) and read
 * the cumulative device milliseconds {dst, multigrid, other} since begin()
 * (the fft_seconds / spatial_seconds columns of ConvergenceHistory,
 * solvers.py:245-253). */
int pint_set_timing(pint_ctx* ctx, int on);
int pint_phase_ms(pint_ctx* ctx, double* ms3);

/* Per-kernel profiling: with on != 0 every launch is bracketed by CUDA
 * events on the context stream; pint_kernel_stat() returns, for kernel family
 * id in [0, pint_kernel_count()), its name, total device ms, launch count and
 * total algorithmic bytes.  Turning it on resets them. */
int pint_profile(pint_ctx* ctx, int on);
int pint_kernel_count(void);
int pint_kernel_stat(pint_ctx* ctx, int id, const char** name, double* ms_total,
                     long long* launches, double* alg_bytes_total);

/* Run `iters` Uzawa iterations (as pint_uzawa_step, residual numerators to
 * res_num[iters]) and return their device time in ms, measured with CUDA
 * events on the context stream (the bench's timed region). */
int pint_uzawa_run(pint_ctx* ctx, double omega, int iters, double* res_num, double* ms_out);

/* Number of kernel launches issued by this context so far (bench evidence). */
long long pint_launch_count(const pint_ctx* ctx);


/* ---------------------------------------------------------------------------
 * Diagnostic mode on the device: the reference's exact-solve oracles.
 * Every SPD spatial solve is multigrid-preconditioned CG to relative residual
 * <= tol (1e-14 typical; it stops earlier only at the rounding floor),
 * batched over planes.  Not available for per-point stiffness fields.
 *
 * pint_sequential_euler: forward implicit-Euler sweep
 *   (M + tau_n A_n) u_n = M u_{n-1} + tau_n load_n        (solvers.py:158-174)
 *   needs the PINT_MG_EULER set (tables of M + tau_n A_n, sid per step);
 *   *iters = most CG iterations of any step, *worst_rel = largest final
 *   relative residual.
 * pint_s_norm: |a - b|_S (b may be NULL), the discrete parabolic norm
 *   s(v,v) = sum tau_n (M dv_n/tau_n).A_n^{-1}(M dv_n/tau_n) + sum v.A_bd v
 *            + v_N.M v_N + sum dv.M dv                   (operators.py:141-183)
 *   needs the A~ set (its level-0 operators are the A_n).
 * pint_uzawa_s_error: |u_j - u_star|_S of the context's Uzawa iterate
 *   (uzawa_solve's diagnostic branch, solvers.py:236-244).
 * pint_abd_inverse: out = A_bd^{-1} in, A_bd = diag(tau_n A_n)  (operators.py:113-122)
 * ------------------------------------------------------------------------- */
int pint_sequential_euler(pint_ctx* ctx, const double* load, const double* u_init,
                          double* u_out, double tol, int max_iter, int* iters,
                          double* worst_rel);
int pint_s_norm(pint_ctx* ctx, const double* a, const double* b, double tol, int max_iter,
                double* out);
int pint_uzawa_s_error(pint_ctx* ctx, const double* u_star, double tol, int max_iter,
                       double* out);
int pint_abd_inverse(pint_ctx* ctx, const double* in, double* out, double tol, int max_iter);

#ifdef __cplusplus
}
#endif
#endif /* PINT_H */
