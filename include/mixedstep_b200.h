/*
 * mixedstep_b200.h — C-ABI of the B200-native mixed-precision BS3(2) integrator.
 *
 * This is the drop-in boundary for the reference's hot path.
 * The reference (mixedstep, C++20, CPU-only) reaches its hot path through two
 * seams; every entry point below replaces one of them:
 *
 *   1. the model plugin  CoupledSystem::eval_rhs(t, x, StagePrecision, out)
 *        (proj/include/mixedstep/systems.hpp:79-80, implemented by
 *         PairwiseSystem<Kernel>, proj/src/systems.cpp:91-110)        -> ms_eval_rhs
 *      and the factories make_lco / make_kuramoto / make_cc
 *        (systems.hpp:107-119, systems.cpp:209-268)                   -> ms_system_create
 *   2. the solver API (proj/include/mixedstep/solver.hpp:128-163):
 *        solve(...)           solver.hpp:154-156, solver.cpp:462-470 -> ms_solve
 *        bs32_step(...)       solver.hpp:147-149, solver.cpp:453-460 -> ms_bs32_step
 *        estimate_error(...)  solver.hpp:130-131, solver.cpp:399-411 -> ms_estimate_error
 *        adjust_step(...)     solver.hpp:135,     solver.cpp:413-418 -> ms_adjust_step
 *        initial_step(...)    solver.hpp:140-142, solver.cpp:420-451 -> ms_initial_step
 *        dp54_reference(...)  solver.hpp:161-163, solver.cpp:472-483 -> ms_dp54_reference
 *        policy_for(...)      precision.hpp:77,   precision.cpp:22-42 -> ms_policy_for
 *
 * Conventions (SURVEY.md §8(b) "Error conventions"):
 *   - return codes: MS_OK (0), MS_EINVAL (1) where the reference throws
 *     std::invalid_argument, MS_ECUDA (2) for CUDA failures; no C++ exception
 *     ever crosses this boundary; ms_last_error() holds a thread-local message;
 *   - numerical failure is never an error code: it is SolveResult::status;
 *   - all host-side vectors are fp64, agent-major interleaved (agent i occupies
 *     slots [i*d, (i+1)*d), systems.hpp:56-58);
 *   - a system handle owns its device memory; K is converted to its storage
 *     format and uploaded once, at creation, and is read-only afterwards.
 *
 * There is no CPU fallback behind this ABI: every compute entry point runs
 * sm_100a kernels and fails with MS_ECUDA when no B200 is present.
 */
#ifndef MIXEDSTEP_B200_H
#define MIXEDSTEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MS_ABI_VERSION 3

/* ---- return codes ---------------------------------------------------- */
#define MS_OK 0
#define MS_EINVAL 1
#define MS_ECUDA 2

/* ---- FloatFormat, precision.hpp:11 (same order) ------------------------ */
enum { MS_BINARY32 = 0, MS_BINARY64 = 1 };

/* ---- PolicyVariant, precision.hpp:51 (same order) + custom ------------- */
enum { MS_SINGLE = 0, MS_MIXED1 = 1, MS_MIXED2 = 2, MS_DOUBLE = 3, MS_CUSTOM = 4 };

/* ---- SolveStatus, solver.hpp:63-71 (same order) ------------------------ */
enum {
  MS_COMPLETED = 0,
  MS_MAX_ITERATIONS = 1,
  MS_MAX_FAILED_STEPS = 2,
  MS_WALL_CLOCK = 3,
  MS_SLOW_SOLVER = 4,
  MS_STEP_TOO_SMALL = 5,
  MS_NON_FINITE = 6
};

/* ---- models ------------------------------------------------------------
 * LCO/KURAMOTO/CC are the reference's three kernels (systems.cpp:112-189),
 * extended with a dense per-pair coupling K_ij applied inside G exactly where
 * the reference multiplies by coupling_k.
 * SCALAR_* are the reference's test fixtures ScalarExp / ScalarZero /
 * ScalarNan (proj/tests/test_support.hpp:21-53), N = 1, d = 1. */
enum {
  MS_MODEL_LCO = 0,
  MS_MODEL_KURAMOTO = 1,
  MS_MODEL_CC = 2,
  MS_MODEL_SCALAR_EXP = 16,
  MS_MODEL_SCALAR_ZERO = 17,
  MS_MODEL_SCALAR_NAN = 18
};

/* storage format of the coupling matrix K on the device */
enum { MS_K_SCALAR = 0, MS_K_F32 = 1, MS_K_F16 = 2, MS_K_BF16 = 3 };
/* element type of a host K buffer handed to ms_system_create */
enum { MS_HOST_F64 = 0, MS_HOST_F32 = 1 };
/* coupling-sum evaluation order:
 *   FAST      — warp-parallel blocked sum per row, Kuramoto via the sin/cos
 *               split; tolerance parity;
 *   FAITHFUL  — one thread per row, ascending j including j = i, per-pair G,
 *               exactly the order of eval_core (systems.cpp:50-57). */
/* RHS evaluation order: FAST = blocked/tree sums (tolerance parity; Kuramoto
 * split into K sin / K cos); FAITHFUL = eval_core's sequential order with
 * per-pair G (systems.cpp:30-64); ORDERED = the Kuramoto split summed in
 * sequential order (the oracle's split form bit for bit; other models: as
 * FAITHFUL) */
enum { MS_RHS_FAST = 0, MS_RHS_FAITHFUL = 1, MS_RHS_ORDERED = 2 };

/* StagePrecision, precision.hpp:36-42 */
typedef struct {
  uint8_t f_prec;
  uint8_t sum_prec;
  uint8_t g_prec;
  uint8_t _pad;
} ms_stage_prec;

/* PrecisionPolicy, precision.hpp:61-74 (per_stage = rows for k2, k3, k4) */
typedef struct {
  ms_stage_prec per_stage[3];
  ms_stage_prec first_step_k1;
  uint8_t storage;
  uint8_t variant;
  uint8_t _pad[2];
} ms_policy;

/* SolverConfig, solver.hpp:39-61 (defaults from ms_default_config) */
typedef struct {
  double rel_tol;
  double abs_tol;
  double h_min_factor;
  int64_t max_iterations;
  int64_t max_failed_steps;
  int32_t time_limits_enabled;
  int32_t record_step_log;
  double wall_clock_limit;
  double slow_solver_elapsed;
  double slow_solver_progress;
  double safety;
  double fac_min;
  double fac_max;
  double controller_exponent;
  int32_t record_snapshots; /* StepSnapshot per accepted step (solver.cpp:324-327), see ms_solve_result */
  int32_t _pad;
} ms_solver_config;

/* StepRecord, solver.hpp:88-93 */
typedef struct {
  double t;
  double h;
  double err;
  int32_t accepted;
  int32_t _pad;
} ms_step_record;

/* Model description: the arguments of make_lco / make_kuramoto / make_cc
 * plus the dense-coupling extension. NULL arrays take the reference values. */
typedef struct {
  int32_t model;        /* MS_MODEL_* */
  int32_t n_agents;     /* N >= 1 */
  int32_t coupled_slot; /* LCO only: 0 = reference form (position), 1 = config-1 form (velocity) */
  int32_t k_storage;    /* MS_K_* */
  int32_t rhs_mode;     /* MS_RHS_* */
  int32_t device;       /* CUDA device ordinal */
  int32_t row_begin;    /* rows of K evaluated by this handle: [row_begin, row_end); 0,0 = all */
  int32_t row_end;
  double coupling_k;    /* scalar coupling (MS_K_SCALAR): the reference's coupling_k */
  double stimulus_i0;   /* CC stimulus I0 */
  const double* m;          /* [d] per-slot weights; NULL = 1/N on the coupled slot */
  const double* omega;      /* Kuramoto [N] natural frequencies */
  const double* w2;         /* LCO config-1 [N] squared frequencies; NULL = 1 */
  const double* cc_k1;      /* CC [N] */
  const double* cc_theta_h; /* CC [N] */
  const double* cc_k0;      /* CC [N] per-cell constants; NULL = CcConstants (systems.hpp:32-43) */
  const double* cc_k2;
  const double* cc_a;
  const double* cc_b;
  const double* cc_c;
  const double* cc_eps;
  const void* K;            /* host row-major N x N (k_host_dtype) or NULL */
  int32_t k_host_dtype;     /* MS_HOST_F64 / MS_HOST_F32 */
  int32_t _pad;
} ms_system_desc;

/* SolveResult, solver.hpp:115-126 (final_state / step_log are caller buffers) */
typedef struct {
  int32_t status;
  int32_t _pad;
  double t_reached;
  int64_t n_accepted;
  int64_t n_failed;
  int64_t rhs_evals;         /* FlopTally::rhs_evals */
  int64_t flops_low;         /* FlopTally::low  */
  int64_t flops_high;        /* FlopTally::high */
  double* final_state;       /* [dN] or NULL (host, or device for ms_solve_device) */
  ms_step_record* step_log;  /* [step_log_capacity] host buffer or NULL */
  int64_t step_log_capacity; /* in */
  int64_t step_log_count;    /* out: records produced (may exceed capacity) */
  double device_ms;          /* out: device time of the adaptive loop (CUDA events) */
  /* StepSnapshot (solver.hpp:96-100) when cfg->record_snapshots: host buffer of
   * (snapshot_capacity + 1) x dN doubles. Row 0 is the loop's starting state
   * (x0, rounded to binary32 under binary32 storage, solver.cpp:263); row k+1
   * is the state after accepted step k, so snapshot k = (row k, row k+1,
   * snapshot_h[k]). NULL = not recorded. */
  double* snapshots;
  double* snapshot_h;          /* [snapshot_capacity] step sizes */
  int64_t snapshot_capacity;   /* in */
  int64_t snapshot_count;      /* out: accepted steps (may exceed capacity) */
  /* Dense output (D6 extension; the reference has none): the cubic
   * Hermite interpolant of each accepted step from (x_n, k1) to (x_{n+1}, k_last)
   * at the sorted output times t_eval[n_eval] in [t0, t_final]; y_eval is a host
   * buffer of n_eval x dN doubles. Times <= t0 get the starting state. NULL =
   * none. n_eval_done: rows written (< n_eval if the solve stopped early). */
  const double* t_eval;
  int64_t n_eval;
  double* y_eval;
  int64_t n_eval_done;
} ms_solve_result;

/* StepOutcome, solver.hpp:75-86 (vectors are caller buffers of length dN) */
typedef struct {
  double* x_next;
  double* x_tilde;
  double* k4;
  double* x_store;
  double err;
  int32_t accepted;
  int32_t _pad;
  double h_used;
  double h_next;
  int64_t rhs_evals;
  int64_t flops_low;
  int64_t flops_high;
} ms_step_outcome;

typedef struct ms_system* ms_system_t;

/* ---- library ---------------------------------------------------------- */
int ms_abi_version(void);
const char* ms_last_error(void);
/* sizeof of the ABI structs, in declaration order: ms_stage_prec, ms_policy,
 * ms_solver_config, ms_step_record, ms_system_desc, ms_solve_result,
 * ms_step_outcome, ms_exchange (binding self-check) */
int ms_abi_sizes(int64_t out[8]);
/* device count visible to the library (0 without a GPU; never an error) */
int ms_device_count(void);
/* number of this library's kernels that have run on the current device since
 * the library was loaded (every kernel counts itself once, CUDA-graph replays
 * included); synchronizes the device; -1 on a CUDA error or without a GPU.
 * Bench/driver evidence, no reference counterpart. */
int64_t ms_launch_count(void);
void ms_default_config(ms_solver_config* cfg);
/* policy_for, precision.cpp:22-42 */
int ms_policy_for(int variant, ms_policy* out);
/* PrecisionPolicy::lowest_format, precision.cpp:9-20 */
int ms_policy_lowest_format(const ms_policy* p);

/* ---- seeded inputs (SplitMix64, rng.hpp:13-52) --------------------------
 * n sequential draws of one (seed, stream) generator. */
int ms_rng_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, double* out);
int ms_rng_normal(uint64_t seed, uint64_t stream, int64_t n, double* out);

/* ---- systems ----------------------------------------------------------
 * ms_system_create uploads K once, converted to k_storage (read-only from then
 * on). A Kuramoto handle with f16 K also keeps K as MMA tile images for the
 * tensor-core sweep (another f16 copy of its rows: 2 GiB at N = 32768), used
 * by binary32 rows at N >= 16384; without room for them the
 * CUDA-core sweeps serve it. */
int ms_system_create(const ms_system_desc* desc, ms_system_t* out);
int ms_system_destroy(ms_system_t sys);
/* K_ij = lo + (hi - lo) * uniform01() of SplitMix64(seed, stream), row-major
 * draw order, generated on the device (bit-identical to the host generator),
 * then rounded to the storage format. Replaces a host upload for large N. */
int ms_system_fill_k_uniform(ms_system_t sys, uint64_t seed, uint64_t stream, double lo, double hi);
/* copy K back as fp64 in storage precision (test hook; rows x N row-major) */
int ms_system_get_k(ms_system_t sys, double* out);
int ms_system_dim(ms_system_t sys);
int ms_system_agents(ms_system_t sys);
/* FlopProfile {theta_f, theta_g, theta_w, d} (systems.hpp:24-29) */
int ms_system_flop_profile(ms_system_t sys, int64_t out[4]);

/* CoupledSystem::eval_rhs (systems.hpp:79-80): host in, host out, synchronous */
int ms_eval_rhs(ms_system_t sys, double t, const double* x, ms_stage_prec sp, double* out);

/* ---- solver ----------------------------------------------------------- */
int ms_estimate_error(int64_t n, const double* x_n, const double* x_next, const double* x_tilde,
                      double ab, double rel, double* err);
int ms_adjust_step(double h, double err, double rel_tol, const ms_solver_config* cfg, double* h_next);
int ms_initial_step(ms_system_t sys, double t0, double t_final, const double* x0,
                    const ms_solver_config* cfg, int order, double* h0, int64_t* rhs_evals);
int ms_bs32_step(ms_system_t sys, double t, const double* x_n, double h, const double* k1,
                 const ms_policy* policy, const ms_solver_config* cfg, ms_step_outcome* out);
/* solve(): host x0, host final_state; H2D/D2H inside */
int ms_solve(ms_system_t sys, const double* x0, double t0, double t_final, const ms_policy* policy,
             const ms_solver_config* cfg, ms_solve_result* res);
/* solve() on device-resident buffers: x0 and res->final_state are device
 * pointers; stream is a cudaStream_t (NULL = the handle's own stream). */
int ms_solve_device(ms_system_t sys, const double* x0_dev, double t0, double t_final,
                    const ms_policy* policy, const ms_solver_config* cfg, ms_solve_result* res,
                    void* stream);
/* ---- host-driven loop with exchange points (row-sharded solves) --------
 * The same attempt as ms_solve, cut into segments so a caller can all-gather
 * the stage derivative rows of a row-sharded handle between sweeps (NCCL).
 * Segments of list 0 (start-up: initial_step + cold k1) run once; those of
 * list 1 form one attempt. After a segment with exch->needed = 1 the caller
 * must make buf[0, total) identical on every rank (each rank owns
 * [offset, offset + count)); the next segment re-checks finiteness on the
 * gathered vector, so every rank takes identical decisions. Kernels are
 * enqueued on `stream` (cudaStream_t, NULL = the handle's stream); nothing
 * in a segment synchronizes, so segments and collectives can be captured into
 * a CUDA graph. ms_loop_done synchronizes and reads the loop flag. */
typedef struct {
  int32_t needed;
  int32_t _pad;
  double* buf;    /* device pointer, dN doubles */
  int64_t offset; /* first element owned by this handle */
  int64_t count;  /* elements owned by this handle */
  int64_t total;  /* dN */
} ms_exchange;
int ms_loop_begin(ms_system_t sys, const double* x0, int x0_on_device, double t0, double t_final,
                  const ms_policy* policy, const ms_solver_config* cfg, int64_t step_log_capacity,
                  void* stream);
int ms_loop_segment_count(ms_system_t sys, int list, int* count);
int ms_loop_run_segment(ms_system_t sys, int list, int index, void* stream, ms_exchange* exch);
int ms_loop_done(ms_system_t sys, void* stream, int* done);
int ms_loop_end(ms_system_t sys, ms_solve_result* res, int final_on_device, void* stream);

/* Push exchange (no reference counterpart; replaces the all-gather of the
 * row-sharded loop). Each rank's sweeps store their output rows into their own
 * workspace AND at the same offset into every peer's workspace (peer memory:
 * NVLink P2P or CUDA IPC mappings), so the exchange rides on the sweep's own
 * stores. Every segment then ends with a release-store of the rank's epoch into
 * each peer's mailbox (ms_loop_run_segment returns exch->needed = 0), and the
 * caller runs ms_loop_push_wait before the next segment (an acquire spin until
 * every peer's slot reaches the epoch; a peer missing for 20 s traps).
 * Sequence per solve: ms_loop_begin; ms_loop_push_info (this rank's workspace
 * base and mailbox, to export); exchange them (ms_ipc_export / ms_ipc_import
 * across processes); ms_loop_push_setup on every rank; synchronize the ranks;
 * then the segments. The workspace must not move afterwards (same step-log
 * capacity on every begin). world <= 8. */
int ms_loop_push_info(ms_system_t sys, void** ws_base, size_t* ws_bytes, void** mailbox);
int ms_loop_push_setup(ms_system_t sys, int world, int rank, void* const* peer_ws /* [world] */,
                       void* const* peer_mailbox /* [world] */);
int ms_loop_push_wait(ms_system_t sys, void* stream);
/* CUDA IPC of a device allocation's base pointer (64-byte handle) */
int ms_ipc_export(void* dev_ptr, unsigned char* handle64);
int ms_ipc_import(const unsigned char* handle64, void** dev_ptr);
int ms_ipc_close(void* dev_ptr);

/* ---- concurrent policy variants ------------------------
 * Up to four solves of one system from the same x0, one policy each (the
 * harness's Single/Mixed1/Mixed2/Double, harness.cpp:113-121), advanced in
 * lock-step attempts on the device. For the split Kuramoto over a stored K
 * each stage is ONE K sweep for all variants. Every variant's result (state,
 * counts, step log) is bit-identical to its own ms_solve; device_ms is the
 * shared loop time. Snapshots are not recorded here. */
typedef struct ms_variants* ms_variants_t;
int ms_variants_create(ms_system_t sys, int32_t count, ms_variants_t* out);
int ms_variants_destroy(ms_variants_t v);
int ms_variants_solve(ms_variants_t v, const double* x0, double t0, double t_final, const ms_policy* policies,
                      const ms_solver_config* cfg, ms_solve_result* results);

/* ---- batched ensembles sharing one K (BASELINE.json configs[4]) ---------
 * B Kuramoto trajectories (own omega_b, theta0_b, own adaptive controller)
 * over the K of a Kuramoto system handle. Each trajectory follows the
 * reference's solve (solver.cpp:226-347) exactly; all advance in lock-step
 * attempts so that one stage evaluates the whole ensemble as one dense
 * contraction K [S|C]. With tensor_cores = 1 (K stored f16 or bf16), stage
 * rows with F, sum and G in binary32 run as a tcgen05 GEMM: sin/cos operands
 * rounded to K's 16-bit format, exact products, binary32 accumulation; other
 * rows (binary64 sums, initial_step) run the exact split on CUDA cores.
 * Arrays are trajectory-major [B][N]; result arrays are caller-owned. */
typedef struct ms_batch* ms_batch_t;
typedef struct {
  int32_t* status;     /* [B] or NULL */
  double* t_reached;   /* [B] or NULL */
  int64_t* n_accepted; /* [B] or NULL */
  int64_t* n_failed;   /* [B] or NULL */
  int64_t* rhs_evals;  /* [B] or NULL */
  double* final_state; /* [B][N] host or NULL */
  int64_t attempts;    /* out: lock-step attempts */
  double device_ms;    /* out */
} ms_batch_result;
int ms_batch_create(ms_system_t sys, int32_t batch, const double* omega, int32_t tensor_cores, ms_batch_t* out);
int ms_batch_destroy(ms_batch_t b);
int ms_batch_eval_rhs(ms_batch_t b, const double* x, ms_stage_prec sp, double* out);
int ms_batch_solve(ms_batch_t b, const double* x0, double t0, double t_final, const ms_policy* policy,
                   const ms_solver_config* cfg, ms_batch_result* res);
/* measurement hook: mean device ms of the ensemble's contraction kernel and
 * of its stage-prep kernel over `iters` evaluations at host state x */
int ms_batch_profile_rhs(ms_batch_t b, const double* x, ms_stage_prec sp, int iters, double* rhs_ms,
                         double* prep_ms);

/* Measurement hook (no reference counterpart): times `iters` evaluations of
 * the RHS at host state x under row sp with CUDA events on the handle's
 * stream, returning the mean device time of the coupling sweep kernel and of
 * the stage-prep kernel (milliseconds per launch). */
int ms_profile_rhs(ms_system_t sys, const double* x, ms_stage_prec sp, int iters, double* rhs_ms,
                   double* prep_ms);
/* dp54_reference (solver.cpp:472-483): all-binary64 DP5(4) at rel = abs = 1e-9 */
int ms_dp54_reference(ms_system_t sys, const double* x0, double t0, double t_final,
                      const ms_solver_config* cfg, ms_solve_result* res);

#ifdef __cplusplus
}
#endif
#endif /* MIXEDSTEP_B200_H */
