/*
 * toepreg_b200.h - C ABI of the B200 superfast Tikhonov-Toeplitz solver.
 *
 * The reference package (toepreg 0.1.0, /root/reference/pkg) is pure Python;
 * its boundary for this path is the Python call
 *     solve_tikhonov(problem, config=None) -> SolveReport
 * (ref: pkg/src/toepreg/solver.py:58-78, re-exported at __init__.py:5-14),
 * with the inner operator rec_tan_int(system, ...) (ref: tanint.py:457-467).
 * The entry points below are what that boundary binds to through ctypes
 * (see INTEGRATION.md); the Python shim paper_1302_6945_b200.solve_tikhonov
 * mirrors the reference signature on top of them.
 *
 * Conventions
 *  - complex values are interleaved (re, im) float64, all pointers passed to
 *    tr_solve_batch are DEVICE pointers owned by the caller;
 *  - Toeplitz generators follow the reference layout: length rows+cols-1,
 *    top-right -> bottom-left, entry (i,j) = gen[i - j + cols - 1]
 *    (ref: toeplitz.py:1-7);
 *  - a batch stride of 0 means "shared by every system of the batch"
 *    (e.g. config 2: one T, 64 right-hand sides);
 *  - the library keeps no pointer after return; concurrent calls are safe
 *    on distinct streams and workspaces.
 *
 * Return codes: 0 ok; 2 invalid arguments (-> ValueError); 3 at least one
 * system singular (-> SingularSystemError, per-system status in tr_diag);
 * 4 CUDA error (-> RuntimeError); 5 capacity exceeded (too many deferred
 * conditions for the workspace, or a basis product longer than planned:
 * status 5 / 6 in tr_diag; -> RuntimeError).
 */
#ifndef TOEPREG_B200_H
#define TOEPREG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TR_GENERAL = 0, TR_L2 = 1, TR_GRAMIAN = 2 };
enum { TR_FILL_AUTO = 0, TR_FILL_ZERO = 1, TR_FILL_ECHO = 2 };

/* Problem shape + SolverConfig (ref: solver.py:39-45, toeplitz.py:167-233). */
typedef struct tr_desc {
  int32_t variant;          /* TR_GENERAL / TR_L2 / TR_GRAMIAN */
  int64_t m;                /* rows of T (gramian: = n) */
  int64_t n;                /* unknowns */
  int64_t p_rows;           /* rows of L (general/gramian; l2: = n) */
  int32_t n_lim;            /* SolverConfig.n_lim (256) */
  double pivot_threshold;   /* SolverConfig.pivot_threshold (1e-8) */
  int32_t fill;             /* SolverConfig.fill */
  int32_t paired;           /* SolverConfig.paired */
  int32_t force_even;       /* SolverConfig.force_even */
  int32_t refine;           /* iterative refinement on (> 0) / off (0 = reference's single pass) */
  int32_t refine_cg;        /* refinement by up to this many CG iterations warm-started at the
                               direct solution; systems CG leaves unfinished (and every system
                               when 0) get `refine` direct refinement solves instead */
  int32_t real_data;        /* 1: every input (T, b / normal rhs) has a zero imaginary part; the CG
                               refinement of the l2 variant then runs on real vectors with
                               half-length transforms.  0: unknown / complex (always valid) */
} tr_desc;

/* Per-system report (ref: SolveReport solver.py:48-55, TanIntDiagnostics
 * tanint.py:72-85). */
typedef struct tr_diag {
  int32_t status;               /* 0 ok, 3 singular, 5 too many deferred conditions,
                                   6 a basis product exceeded its planned length (x untrusted) */
  int32_t difficult_points;
  int64_t conditions_total;
  int32_t recursion_depth;
  int32_t retried_leaves;
  double max_column_scale;
  int64_t final_col_degrees[8];
  double relative_residual;
  int32_t trim_overflow;        /* products truncated at the degree bound */
  int32_t refine_cg_iterations; /* CG refinement iterations run (0: none / direct refinement) */
  double wall_time_s;           /* device time of the solve (assemble -> extract, + refinement),
                                   excluding the residual evaluation; the whole batch's time */
  int32_t rescued;              /* 1: the direct solve failed under FP64 rounding (singular, or no
                                   better than x = 0) and x comes from CG from zero (refine > 0) */
} tr_diag;

/* Bytes of device workspace tr_solve_batch needs for `batch` systems. */
size_t tr_workspace_bytes(const tr_desc* d, int64_t batch);

/* Circulant order N = n_tilde + k of the extended system (ref
 * extension.py:42-68, :190-193) and the tree shape, for diagnostics. */
int tr_plan_info(const tr_desc* d, int64_t* order, int64_t* leaves, int32_t* depth,
                 int64_t* max_leaf_conditions);

/* Solve `batch` independent systems.  Device inputs:
 *   T_gen  [batch][m+n-1]     (general, l2)          stride T_bs
 *   L_gen  [batch][p_rows+n-1](general, gramian)     stride L_bs
 *   G_col  [batch][n]         (gramian: first column of T^H T)  stride G_bs
 *   beta_sq[batch]            (l2: |beta|^2, real)   stride beta_bs
 *   rhs    [batch][m] = b, or [batch][n] = normal rhs y = T^H b when
 *          rhs_is_normal (always for gramian)        stride rhs_bs
 * Outputs: x_out [batch][n] (device), diag_host [batch] (host, may be NULL).
 * The call is stream-ordered; when diag_host is non-NULL it synchronises the
 * stream to fill it. */
int tr_solve_batch(const tr_desc* d, int64_t batch,
                   const double* T_gen, int64_t T_bs,
                   const double* L_gen, int64_t L_bs,
                   const double* G_col, int64_t G_bs,
                   const double* beta_sq, int64_t beta_bs,
                   const double* rhs, int64_t rhs_bs, int32_t rhs_is_normal,
                   double* x_out, tr_diag* diag_host,
                   void* workspace, size_t ws_bytes, void* stream);

/* Host-buffer convenience entry (what a non-CUDA caller binds): copies the
 * inputs in, solves, copies x out.  Same argument meaning, HOST pointers. */
int tr_solve_batch_host(const tr_desc* d, int64_t batch,
                        const double* T_gen, int64_t T_bs,
                        const double* L_gen, int64_t L_bs,
                        const double* G_col, int64_t G_bs,
                        const double* beta_sq, int64_t beta_bs,
                        const double* rhs, int64_t rhs_bs, int32_t rhs_is_normal,
                        double* x_out, tr_diag* diag_host);

/* Conjugate gradients from a zero start on the normal equations, batched
 * (replaces toepreg.solver.cg_solve, pkg/src/toepreg/solver.py:184-215).
 * Same inputs as tr_solve_batch; max_iterations <= 0 means the reference
 * default max(10 n, 100); systems stop individually at
 * ||r|| <= tolerance ||rhs||; time_budget >= 0 is checked after completed
 * iterations (time_budget < 0: none).  x_out [batch][n] device, iterations [batch] host.  The
 * workspace is tr_cg_workspace_bytes(d, batch). */
size_t tr_cg_workspace_bytes(const tr_desc* d, int64_t batch);
int tr_cg_batch(const tr_desc* d, int64_t batch,
                const double* T_gen, int64_t T_bs,
                const double* L_gen, int64_t L_bs,
                const double* G_col, int64_t G_bs,
                const double* beta_sq, int64_t beta_bs,
                const double* rhs, int64_t rhs_bs, int32_t rhs_is_normal,
                int64_t max_iterations, double tolerance, double time_budget,
                double* x_out, int64_t* iterations,
                void* workspace, size_t ws_bytes, void* stream);

/* y = A x with A the normal matrix (replaces NormalOperator.apply,
 * pkg/src/toepreg/solver.py:104-167): T^H T + |beta|^2 I (l2),
 * T^H T + L^H L (general), G + L^H L (gramian).  x, y [batch][n] device;
 * workspace as tr_cg_workspace_bytes. */
int tr_normal_apply(const tr_desc* d, int64_t batch,
                    const double* T_gen, int64_t T_bs,
                    const double* L_gen, int64_t L_bs,
                    const double* G_col, int64_t G_bs,
                    const double* beta_sq, int64_t beta_bs,
                    const double* x, double* y,
                    void* workspace, size_t ws_bytes, void* stream);

/* Nonuniform Fourier sums for the Gramian setup (replaces the dense
 * exp(outer(...)) forms of pkg/src/toepreg/nufft.py:60-72 and :106-114):
 *   adjoint != 0: out[d] = sum_{k<K} in[k] exp(sign 2 pi i freqs[k] d), d < n
 *   adjoint == 0: out[k] = sum_{j<n} in[j] exp(sign 2 pi i freqs[k] j), k < K
 * freqs [K] float64, in / out complex128 (interleaved); device pointers. */
int tr_nudft(const double* freqs, int64_t K, int64_t n, const double* in, int32_t adjoint,
             int32_t sign, double* out, void* stream);

/* Stage entry points mirroring reference helpers, for stage-level parity:
 *  tr_grid_eval   ~ fftpoly.grid_eval(coeffs, N, offset, stride) (:64-89)
 *  tr_fft         ~ batched unnormalised DFT, sign +1/-1
 *  tr_matpoly_mul ~ fftpoly.matpoly_multiply(a, b) (:233-249), untrimmed
 *  tr_assemble    ~ extension.assemble(problem).weights (:267-273)
 * All pointers are device pointers; all are stream-ordered on `stream`. */
int tr_fft(const double* in, double* out, int64_t n, int64_t lines, int32_t sign, void* stream);
int tr_grid_eval(const double* coeffs, int64_t lines, int64_t length, int64_t n_nodes,
                 int64_t offset, int64_t stride, double* out, void* stream);
int tr_matpoly_mul(const double* a, int64_t la, const double* b, int64_t lb, int32_t p,
                   double* out, void* stream);
int tr_assemble(const tr_desc* d, const double* T_gen, const double* L_gen, const double* G_col,
                const double* beta_sq, const double* rhs, int32_t rhs_is_normal,
                double* weights_out, void* stream);

/* One leaf sweep ~ tanint._Engine._serial_leaf (:395-434): the
 * `leaf_index`-th leaf of the plan on device weights [N][rows][p] with the
 * degree ledger col_degrees[p] (host, in/out).  basis_out (device) receives
 * the normalised p x p x cap coefficient cube (cap >= conditions + 1). */
int tr_leaf(const tr_desc* d, const double* weights, int64_t leaf_index, int64_t* col_degrees,
            double* basis_out, int64_t cap, int32_t* ndeferred, double* self_residual,
            int32_t* attempts, void* stream);

/* Instrumentation: total kernel launches issued by this library; optional
 * per-class CUDA-event timing (classes: 0 assemble, 1 fft, 2 leaf pivot
 * chain, 3 leaf basis replay, 4 leaf self-check, 5 leaf exact, 6 coset update,
 * 7 combine, 8 normal operator, 9 finish); measured FP64 FMA peak. */
int64_t tr_launch_count(void);
int tr_kernel_timing(int32_t enable);
int tr_kernel_stats(int32_t cls, double* total_ms, int64_t* launches);
/* Algorithmic bytes / flops issued per class while timing was enabled
 * (minimal HBM traffic and useful FP64 flops, SURVEY 8(d) counting). */
int tr_kernel_work_stats(int32_t cls, double* alg_bytes, double* alg_flops);
int tr_fp64_peak(double* tflops);
/* FFT device time by (length, lines) while timing was enabled, largest
 * first: rows[3k..3k+2] = {n, lines, launches}, ms[k]; returns the count. */
int tr_fft_breakdown(int64_t* rows, double* ms, int cap);

/* Last error message of the calling thread. */
const char* tr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TOEPREG_B200_H */
