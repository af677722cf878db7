/*
 * t2s2.h — C ABI of the B200-native T^2S^2 hot path.
 *
 * Drop-in boundary for the reference's Python host API (pkg/src/ttss/).
 * The reference is pure Python/numpy, so its FFI for this path is a ctypes
 * binding; every entry point below replaces one
 * reference function and keeps its argument meaning and error behaviour:
 *
 *   t2s2_round     <- tensor_train.tt_round      (tensor_train.py:327)
 *                     tensor_train.tt_op_round   (tensor_train.py:616)
 *   t2s2_norm      <- tensor_train.tt_norm       (tensor_train.py:319)
 *   t2s2_dot       <- tensor_train.tt_dot        (tensor_train.py:296)
 *   t2s2_add       <- tensor_train.tt_add        (tensor_train.py:253)
 *   t2s2_scale     <- tensor_train.tt_scale      (tensor_train.py:277)
 *   t2s2_apply     <- tensor_train.tt_apply      (tensor_train.py:359)
 *   t2s2_full      <- tensor_train.tt_full       (tensor_train.py:186)
 *   t2s2_solve     <- tt_solver.solve            (tt_solver.py:445)
 *   t2s2_residual  <- tt_solver.residual         (tt_solver.py:80)
 *   t2s2_march     <- time_integration._march    (time_integration.py:149)
 *
 * Instrumentation without a reference counterpart: t2s2_stats_reset /
 * t2s2_stats_read / t2s2_launch_log (per-family and per-launch kernel
 * accounting), t2s2_dense_solve / t2s2_gemm (kernel test hooks).
 *
 * Trains cross the boundary as plain arrays: d, per-core row (and, for
 * operators, column) mode sizes, d+1 bond ranks, and all cores
 * concatenated row-major in float64 — the layout of the reference's
 * "TTS2" container payload (tensor_train.py:648).  Inside the library a
 * train is device resident (t2s2_train handle).
 *
 * All functions return 0 on success or a T2S2_ERR_* code; the message is
 * available from t2s2_last_error().  Shape errors correspond to the
 * reference's ShapeError, value errors to ValueError, stagnation to
 * MarchStepError.
 */
#ifndef T2S2_H_
#define T2S2_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define T2S2_OK 0
#define T2S2_ERR_ARG 1
#define T2S2_ERR_CUDA 2
#define T2S2_ERR_SHAPE 3
#define T2S2_ERR_VALUE 4
#define T2S2_ERR_STAGNATION 5
#define T2S2_ERR_CAPACITY 6

#define T2S2_MAX_SWEEPS 1024

typedef struct t2s2_context t2s2_context;
typedef struct t2s2_train t2s2_train;

/* SolverConfig (tt_solver.py:39-59). local_solver: 0 auto, 1 direct, 2 iterative. */
typedef struct {
  int max_sweeps;
  double residual_tol;
  double rounding_tol;
  int enrichment_rank;
  int max_rank;
  int local_solver;
  int local_direct_size;
  double inner_tol_factor;
  int stagnation_window;
  double stagnation_drop;
} t2s2_solver_config;

/* SolveReport (tt_solver.py:62-76); histories hold n_sweeps entries. */
typedef struct {
  int n_sweeps;
  double residuals[T2S2_MAX_SWEEPS];
  int ranks[T2S2_MAX_SWEEPS];
  double compression[T2S2_MAX_SWEEPS];
  double wall_time;
  int converged;
  int stagnated;
} t2s2_solve_report;

/* One row of MarchDiagnostics (time_integration.py:76-115) minus peak. */
typedef struct {
  int step;
  int max_rank;
  double compression;
  double residual;
  int sweeps;
} t2s2_step_report;

/* Per-family launch accounting: launches, algorithmic flops/bytes, and
 * (while profile_events is on) summed CUDA-event device time. */
typedef struct {
  char family[32];
  long long launches;
  double device_ms;
  double flops;
  double bytes;
} t2s2_kernel_stat;

int t2s2_context_create(int device, t2s2_context** out);
/* SM partitions (no reference counterpart: B200 throughput feature for
 * independent solves, BASELINE config 4).  t2s2_sm_partitions splits the
 * device's SMs into `count` disjoint green contexts once per process and
 * writes each partition's SM count to sms_out[count]; a context created on
 * partition `part` runs all its kernels on those SMs only, so independent
 * solves in different host threads cannot block each other's cooperative
 * kernels. */
int t2s2_sm_partitions(int device, int count, int* sms_out);
int t2s2_context_create_on_partition(int device, int part, t2s2_context** out);
/* Instrumentation: the device's global nanosecond timer, read by a kernel
 * on the context's stream once its earlier work has run (blocking); one
 * clock for all contexts and partitions of the device. */
int t2s2_device_clock(t2s2_context* ctx, unsigned long long* out_ns);
void t2s2_context_destroy(t2s2_context* ctx);
const char* t2s2_last_error(const t2s2_context* ctx);
/* Limit whole-GPU cooperative kernels (the local dense solves) to `sms`
 * CTAs (0 = all SMs), so several contexts on one device — one per host
 * thread, e.g. independent solves of a parameter sweep — can run their
 * local solves concurrently. */
int t2s2_context_set_sm_budget(t2s2_context* ctx, int sms);
/* The cudaStream_t every kernel of the context is launched on (for
 * callers that time or order work around the engine). */
void* t2s2_stream(t2s2_context* ctx);
/* Wait for all device work of the context. */
int t2s2_synchronize(t2s2_context* ctx);

/* Reset the counters; profile_events != 0 also records a CUDA event pair
 * around every launch (adds ~2 us per launch). */
int t2s2_stats_reset(t2s2_context* ctx, int profile_events);
int t2s2_stats_read(t2s2_context* ctx, t2s2_kernel_stat* out, int capacity, int* count);

/* Instrumentation (no reference counterpart): while profile_events is on,
 * one record per launch in launch order — family index (the order of
 * t2s2_stats_read), algorithmic flops and bytes, CUDA-event duration.  At
 * most T2S2_LAUNCH_LOG_CAP records are kept per reset. */
#define T2S2_LAUNCH_LOG_CAP 1000000
typedef struct {
  int family;
  double flops;
  double bytes;
  double device_ms;
} t2s2_launch_record;
int t2s2_launch_log(t2s2_context* ctx, t2s2_launch_record* out, int capacity, int* count);

/* Instrumentation (no reference counterpart): the device->host reads that
 * steer the host (ranks, candidate scores, residuals, solver flags).
 * mode 1 records the values every such read returns, mode 2 hands the
 * recorded values back to an IDENTICAL run without synchronising (the host
 * then runs ahead of the device; a run that asks for a different read
 * fails with T2S2_ERR_ARG), mode 3 runs normally and reports (stderr) the
 * first read whose value differs from the recorded run (a determinism
 * check), mode 0 switches everything off.  *count = reads recorded.  Used to
 * measure what the synchronising reads cost. */
int t2s2_read_trace(t2s2_context* ctx, int mode, int* count);

/* cols == NULL uploads a vector train (cores r0 x rows x r1), otherwise an
 * operator train (cores r0 x rows x cols x r1).  host_cores holds the
 * concatenated cores; device_cores (second form) is a device pointer. */
int t2s2_train_upload(t2s2_context* ctx, int d, const int* rows, const int* cols,
                      const int* ranks, const double* host_cores, t2s2_train** out);
int t2s2_train_upload_device(t2s2_context* ctx, int d, const int* rows, const int* cols,
                             const int* ranks, const double* device_cores, t2s2_train** out);
/* Shape query: d, rows[d], cols[d] (zeros for vectors), ranks[d+1], and the
 * total number of float64 entries of all cores. */
int t2s2_train_shape(const t2s2_train* t, int* d, int* rows, int* cols, int* ranks,
                     size_t* n_entries);
int t2s2_train_download(t2s2_context* ctx, const t2s2_train* t, double* host_cores,
                        size_t capacity);
void t2s2_train_free(t2s2_train* t);

int t2s2_round(t2s2_context* ctx, const t2s2_train* v, double tol, int max_rank,
               t2s2_train** out);
int t2s2_norm(t2s2_context* ctx, const t2s2_train* v, double* out);
int t2s2_dot(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* b, double* out);
/* out = sa * a + sb * b (tt_add of tt_scale'd operands). */
int t2s2_add(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* b, double sa, double sb,
             t2s2_train** out);
int t2s2_scale(t2s2_context* ctx, const t2s2_train* a, double s, t2s2_train** out);
int t2s2_apply(t2s2_context* ctx, const t2s2_train* op, const t2s2_train* v, t2s2_train** out);
int t2s2_full(t2s2_context* ctx, const t2s2_train* v, double* host_dense, size_t capacity);

/* x0 is required (the host layer builds the reference's default guess). */
int t2s2_solve(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* rhs,
               const t2s2_train* x0, const t2s2_solver_config* cfg, t2s2_train** x,
               t2s2_solve_report* report);
/* Dense solve of one local system (column-major n x n) — the kernels behind
 * the direct local solves (tt_solver.py:357-366, 392-397), exposed for
 * testing: the verified block Gauss-Jordan kernel (threshold partial
 * pivoting: no interchange while every multiplier is <= 8 in magnitude;
 * GEPP's factors when none exceeds 1), else the partial-pivoting kernel; returns T2S2_ERR_VALUE on an exactly singular
 * matrix (numpy.linalg.solve's LinAlgError). */
int t2s2_dense_solve(t2s2_context* ctx, int n, const double* a_colmajor, const double* b,
                     double* x);
/* Row-major fp64 GEMM on device pointers, C = op(A) op(B) (op = transpose
 * when the flag is set), through the engine's GEMM-program kernel — the
 * contraction engine behind every tensordot of tt_solver.py, exposed for
 * testing and benchmarking.  Enqueued on the context stream. */
int t2s2_gemm(t2s2_context* ctx, int ta, int tb, int m, int n, int k, const double* a, int lda,
              const double* b, int ldb, double* c, int ldc);
int t2s2_residual(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* x,
                  const t2s2_train* rhs, double tol, double* out);

/* Implicit step-and-truncate march (time_integration.py:149-191):
 *   rhs_k = round(right @ state + bc_k + src_k, 0.01 * step_tol)
 *   state = round(solve(left, rhs_k, x0=state), step_tol)
 * bc/src hold n_forcing entries (1: the same pair every step, as in the
 * reference; n_steps: per-step data for time-dependent problems); either
 * array or entry may be NULL.  states_out (optional, n_steps entries)
 * receives every stride-th state and the final one (NULL elsewhere);
 * reports (optional) n_steps rows.  On inner stagnation returns
 * T2S2_ERR_STAGNATION and *failed_step (optional) names the step. */
int t2s2_march(t2s2_context* ctx, const t2s2_train* left, const t2s2_train* right,
               const t2s2_train* state0, int n_steps, const t2s2_train* const* bc,
               const t2s2_train* const* src, int n_forcing, double step_tol,
               const t2s2_solver_config* cfg, int store_stride, t2s2_train** states_out,
               t2s2_step_report* reports, int* failed_step);

#ifdef __cplusplus
}
#endif

#endif /* T2S2_H_ */
