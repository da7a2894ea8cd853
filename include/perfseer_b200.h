/* perfseer_b200.h — the drop-in C ABI of the B200 measured-kernel and
 * calibration path.
 *
 * The reference exposes this path as C++ virtuals and free functions; this
 * header is what a binding (cgo / JNI / ctypes / plain C++) links against.
 * Every entry point returns int status (0 = OK); on failure the message is
 * available from ps_last_error() (thread-local, valid until the next call on
 * the same thread). No torch or C++ types cross this boundary.
 *
 * Reference interfaces replaced (paths relative to the reference's proj/):
 *   ps_init / ps_destroy / ps_measure
 *       perfseer::Executor::id/measure        include/perfseer/executor.hpp:16-23
 *       (the GPU executor the reference leaves as an extension point)
 *   ps_measure_summary
 *       perfseer::measure_kernel + summarize  src/executor.cpp:14-48
 *   ps_desc_from_id
 *       variant_id() parsing (the executor dispatches on Kernel::name, which is
 *       the generator variant id)             src/uipick.cpp:149-154,197-198
 *   ps_run_verify
 *       parity hook: runs one generated kernel on caller-owned HOST buffers
 *       (the reference's own interpreter is tests/support.hpp:50-162)
 *   ps_fit_lm_batched
 *       perfseer::fit_model (Levenberg-Marquardt) src/model.cpp:485-606
 *   ps_eval_batched
 *       perfseer::predict + report ranking     src/model.cpp:615-623,
 *                                              tools/perfseer.cpp:452-469
 *   ps_run_host / ps_run_host_batch
 *       `perfseer measure` over a kernel directory through host data
 *       (tools/perfseer.cpp:211-240), one kernel / a pipelined sweep
 *   ps_enumerate
 *       perfseer::brute_force_count            src/oracle.cpp:76-425
 *   ps_catalog / ps_feature_table / ps_fit_cpu / ps_predict_cpu / ...
 *       the C++ port's KernelCollection::generate, gather_feature_values,
 *       fit_model, predict (uipick.cpp:71-119, features.cpp:417-493,
 *       model.cpp:485-623) for non-C++ hosts
 *   ps_prepare / ps_trim / ps_mark / ps_elapsed / ps_host_alloc
 *       new: residency, step timing and pinned staging for the B200 sweep
 *
 * Threading: one ps_ctx per GPU; a ps_ctx must not be used concurrently
 * (executors are exclusive resources, executor.hpp:13-15).
 * Different contexts may be driven from different host threads.
 */
#ifndef PERFSEER_B200_H_
#define PERFSEER_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_ERR_ARG 1      /* bad argument / unknown generator (SemanticError-like) */
#define PS_ERR_CUDA 2     /* CUDA runtime failure (mapped to EvalError by CudaExecutor) */
#define PS_ERR_NOMEM 3    /* device allocation failed */
#define PS_ERR_STATE 4    /* call out of order */

typedef struct ps_ctx ps_ctx;

/* Generators: one per UIPiCK builder (src/uipick.cpp:295-664) plus the DG
 * application variants designed from PAPER.md:2341-2442. */
enum ps_generator {
  PS_GEN_GMEM_PATTERN = 1,   /* make_gmem_pattern      uipick.cpp:295-315 */
  PS_GEN_FLOPS = 2,          /* make_flops_pattern     uipick.cpp:317-378 */
  PS_GEN_LMEM_SHUFFLE = 3,   /* make_lmem_shuffle      uipick.cpp:380-404 */
  PS_GEN_BARRIER = 4,        /* make_barrier_knl       uipick.cpp:406-423 */
  PS_GEN_EMPTY = 5,          /* make_empty_knl         uipick.cpp:425-432 */
  PS_GEN_OVERLAP = 6,        /* make_overlap_knl       uipick.cpp:434-462 */
  PS_GEN_MATMUL = 7,         /* make_matmul_sq         uipick.cpp:464-554 */
  PS_GEN_MATMUL_RM = 8,      /* make_matmul_sq_rm      uipick.cpp:556-581 */
  PS_GEN_FD = 9,             /* make_fd_stencil        uipick.cpp:583-639 */
  PS_GEN_FD_RM = 10,         /* make_fd_stencil_rm     uipick.cpp:641-664 */
  PS_GEN_DG = 11,            /* DG differentiation */
  PS_GEN_DG_RM = 12,         /* DG work-removed */
  PS_GEN_MATMUL_TC = 13,     /* extra: tcgen05 dense contraction (not a paper variant) */
  PS_GEN_DG_TC = 14          /* extra: DG as a tcgen05 contraction (not a paper variant) */
};

enum ps_dtype { PS_F32 = 0, PS_F64 = 1 };
enum ps_flop_op { PS_OP_ADD = 0, PS_OP_MUL = 1, PS_OP_MADD = 2 };
/* keep argument of the *_rm generators */
enum ps_keep { PS_KEEP_NONE = 0, PS_KEEP_A = 1, PS_KEEP_B = 2, PS_KEEP_U = 3, PS_KEEP_RES = 4,
               PS_KEEP_DM = 5 };
/* DG variants */
enum ps_dg_variant { PS_DG_NOPF = 0, PS_DG_UPF = 1, PS_DG_DMPF = 2, PS_DG_DMPF_T = 3 };
/* input fill modes */
enum ps_fill { PS_FILL_SEED17 = 0, PS_FILL_UNIFORM = 1 };

/* Plain-old-data description of one generated measurement kernel, parsed
 * from its variant id ("gen__arg-value__..."). Unused fields are 0. */
typedef struct ps_kernel_desc {
  int32_t gen;          /* enum ps_generator */
  int32_t dtype;        /* enum ps_dtype */
  int32_t op;           /* flops: enum ps_flop_op */
  int32_t keep;         /* *_rm: enum ps_keep */
  int64_t nelements;    /* pattern generators: E */
  int64_t lsize0, lsize1;
  int64_t lid_stride0, lid_stride1;
  int64_t n_inputs;     /* gmem_pattern: n_input_arrays */
  int64_t m;            /* flops/lmem/barrier/overlap iteration count */
  int64_t num_groups;   /* empty_knl */
  int64_t n;            /* matmul / finite_diff size */
  int32_t prefetch;     /* matmul: 1 = PF, 0 = noPF */
  int32_t tile;         /* finite_diff: 16 or 18 */
  int64_t nel;          /* DG: number of elements */
  int64_t np;           /* DG: padded nodes per element (multiple of 16) */
  int64_t nmat;         /* DG: number of derivative matrices (3) */
  int32_t dg_variant;   /* enum ps_dg_variant */
  int32_t reserved;
} ps_kernel_desc;

/* Buffer layout of a kernel's global arrays (host side, no GPU needed). */
#define PS_MAX_ARRAYS 4
typedef struct ps_io_info {
  int32_t n_inputs;
  int32_t n_outputs;
  int32_t elem_bytes;
  int32_t reserved;
  int64_t input_elems[PS_MAX_ARRAYS];
  int64_t output_elems[PS_MAX_ARRAYS];
  /* algorithmic work per launch, for roofline reporting */
  double bytes_global;   /* compulsory DRAM bytes (each array touched once) */
  double flops;          /* floating-point operations (madd = 2) */
  double bytes_shared;   /* shared-memory bytes moved */
} ps_io_info;

const char* ps_last_error(void);
const char* ps_version(void);

/* --- host-only helpers (no GPU required) -------------------------------- */
int ps_desc_from_id(const char* variant_id, ps_kernel_desc* out);
int ps_kernel_io(const ps_kernel_desc* desc, ps_io_info* out);

/* --- device context ------------------------------------------------------ */
int ps_init(int device, ps_ctx** out);
int ps_destroy(ps_ctx* ctx);
int ps_device_info(ps_ctx* ctx, int* sm_count, int* sm_clock_khz, size_t* l2_bytes,
                   size_t* free_bytes);

/* Allocates (grow-only, cached) device buffers for desc and fills inputs on
 * the device with the deterministic pattern (PS_FILL_SEED17: the reference
 * test fixture's 1 + FNV1a(array, flat) % 17, tests/support.hpp:35-44;
 * PS_FILL_UNIFORM: U[-1,1) from `seed`). */
int ps_prepare(ps_ctx* ctx, const ps_kernel_desc* desc, int fill_mode, uint64_t seed);

/* Executor::measure: `warmup` untimed launches then `trials` launches each
 * bracketed by CUDA events on the context stream; per-trial seconds into the
 * caller-owned out_seconds[trials]. Prepares buffers on first use. */
int ps_measure(ps_ctx* ctx, const ps_kernel_desc* desc, int warmup, int trials,
               double* out_seconds);

/* measure_kernel + summarize (drop trials > filter_factor * median, mean of
 * survivors, src/executor.cpp:14-38). */
int ps_measure_summary(ps_ctx* ctx, const ps_kernel_desc* desc, int warmup, int trials,
                       double filter_factor, double* mean_seconds, int* kept_trials);

/* Launch `launches` back-to-back kernels on prepared buffers and return the
 * total device time (CUDA events) — used by the bench's timed region. */
int ps_run_timed(ps_ctx* ctx, const ps_kernel_desc* desc, int launches, double* seconds);

/* Parity hook: host inputs -> device, one launch, device -> host outputs.
 * inputs[i] has input_elems[i] elements of the kernel dtype; outputs are
 * zero-initialised on the device before the launch. */
int ps_run_verify(ps_ctx* ctx, const ps_kernel_desc* desc, const void* const* inputs,
                  int n_inputs, void* const* outputs, int n_outputs);

/* Device pointer of the prepared input/output i (for zero-copy callers). */
int ps_buffer(ps_ctx* ctx, int is_output, int index, void** dev_ptr, int64_t* elems);

/* End to end through host buffers: H2D of every input, one launch, D2H of
 * every output, bracketed by CUDA events; seconds = the whole sequence. */
int ps_run_host(ps_ctx* ctx, const ps_kernel_desc* desc, const void* const* inputs, int n_inputs,
                void* const* outputs, int n_outputs, double* seconds);
/* End to end over a batch of kernels, pipelined: the H2D copies of kernel
 * i+1, the launch of kernel i and the D2H copies of kernel i-1 overlap (three
 * streams, four device slots; PCIe is full duplex). inputs / outputs hold, for
 * each kernel in order, its n_inputs / n_outputs host pointers (pinned for
 * overlap) back to back. seconds = first H2D to last D2H, CUDA events.
 * (New; the batched form of ps_run_host for sweeps through host data.) */
int ps_run_host_batch(ps_ctx* ctx, int n, const ps_kernel_desc* descs, const void* const* inputs,
                      void* const* outputs, double* seconds);
/* The same with the step's result instead of (or besides) the output arrays:
 * checksums[i] (n entries, may be NULL) = wrapping 64-bit sum of the 32-bit
 * words of kernel i's outputs, computed on the device and read back once at
 * the end of the batch; outputs may be NULL (no output copies). */
int ps_run_host_batch_ex(ps_ctx* ctx, int n, const ps_kernel_desc* descs, const void* const* inputs,
                         void* const* outputs, uint64_t* checksums, double* seconds);
/* Releases every resident prepared variant and staging buffer of the context
 * (the context, its stream and events stay valid; later calls re-prepare). */
int ps_trim(ps_ctx* ctx);
/* Pinned host memory for ps_run_host callers. */
int ps_host_alloc(size_t bytes, void** ptr);
int ps_host_free(void* ptr);

/* Event markers on the context stream (slots 0..63) for timing whole steps. */
int ps_mark(ps_ctx* ctx, int slot);
int ps_elapsed(ps_ctx* ctx, int from_slot, int to_slot, double* seconds);

/* --- calibration (K17) and prediction (K18) ------------------------------ */

/* Compiled model expression: postfix bytecode over params/features/constants
 * (compiled host-side from the reference model grammar, model.cpp:50-234). */
#define PS_BC_NUM 0     /* push consts[arg]            */
#define PS_BC_PARAM 1   /* push params[arg]            */
#define PS_BC_FEAT 2    /* push features[arg]          */
#define PS_BC_ADD 3
#define PS_BC_SUB 4
#define PS_BC_MUL 5
#define PS_BC_DIV 6
#define PS_BC_TANH 7
typedef struct ps_bytecode {
  int32_t n_ops;
  int32_t n_consts;
  const int32_t* ops;     /* [n_ops] opcode << 16 | arg */
  const double* consts;   /* [n_consts] */
} ps_bytecode;

typedef struct ps_fit_opts {
  double lambda0, lambda_decrease, lambda_increase, step_tol, grad_tol;
  int32_t max_iterations;
  int32_t nonnegative;
} ps_fit_opts;

typedef struct ps_fit_stats {
  double residual_norm;
  int32_t iterations;
  int32_t converged;
  int32_t status;        /* 0 ok, 1 damping overflow (divergence) */
  int32_t trials;        /* damped solves tried (K17 v2; 0 elsewhere) */
} ps_fit_stats;

/* Batched LM: `nbatch` independent fits of one model (np params, nf
 * features) over nr rows each. features: [nbatch][nr][nf], t: [nbatch][nr],
 * params_inout: [nbatch][np] (initial point in, fitted out), stats[nbatch].
 * jac holds np bytecodes (dg/dp_i). Host buffers. */
int ps_fit_lm_batched(ps_ctx* ctx, const ps_bytecode* model, const ps_bytecode* jac, int np,
                      int nf, const double* features, const double* t, int nr, int nbatch,
                      const ps_fit_opts* opts, double* params_inout, ps_fit_stats* stats);
/* Same with mode bits: 1 = column equilibration (iterate on q = p / |p0|),
 * 2 = warp-shuffle reductions (default: per-entry sums in the reference's
 * row order, which makes linear fits bit-identical to fit_model). */
int ps_fit_lm_batched_ex(ps_ctx* ctx, const ps_bytecode* model, const ps_bytecode* jac, int np,
                         int nf, const double* features, const double* t, int nr, int nbatch,
                         const ps_fit_opts* opts, int mode, double* params_inout,
                         ps_fit_stats* stats);

/* K17 v2: every fit of a calibration round in one launch. A job is one model
 * (model file text: output id line + expression, model.cpp:625-644) fitted
 * from nbatch starts to nr rows; the library compiles the model and its
 * derivatives into one straight-line program with shared subexpressions.
 * mode bits: 1 column equilibration, 2 warp-shuffle sums (default: row-order
 * sums, bit-identical to fit_model), 4 residuals relative to t.
 * shared_rows = 1: features [nr][nf] and t [nr] are shared by every start
 * (else [nbatch][nr][nf], [nbatch][nr]). Host buffers; kernel_seconds (may
 * be NULL) is the device time of the one launch. */
typedef struct ps_lm_job {
  const char* model_text;
  int32_t nf, nr, nbatch, mode, shared_rows, reserved;
  const double* features;
  const double* t;
  ps_fit_opts opts;
  double* params_inout;   /* [nbatch][np] */
  ps_fit_stats* stats;    /* [nbatch] */
} ps_lm_job;
int ps_fit_lm_jobs(ps_ctx* ctx, int njobs, const ps_lm_job* jobs, double* kernel_seconds);

/* The device tanh K17 and K18 evaluate sstep/tanh with (csrc/cuda/libm_glibc.cuh):
 * the host glibc's std::tanh (model.cpp:253) restated bit for bit, so device
 * and reference model evaluations agree exactly. x, out: n host doubles. */
int ps_math_tanh(ps_ctx* ctx, const double* x, int64_t n, double* out);

/* K18 batched prediction over a variant space. A table set is compiled
 * host-side from JSON {"variants": [{"id": variant id, "model": model text,
 * "params": [fitted values], "group": application index, "coords":
 * {"<size parameter>": point coordinate 0..3}}]}: every model feature of
 * every variant becomes an exact integer polynomial in the point coordinates
 * (checked against evaluate_feature at several admissible sizes, so a
 * parameter-dependent match is an error rather than a silent freeze).
 * points: [npts][4] int64; pred: [npts][nvar] seconds; argmin:
 * [npts][ngroups] winning variant index per application group (strict '<'
 * first minimum in variant order, tools/perfseer.cpp:458-467). */
typedef struct ps_tables ps_tables;
int ps_tables_build(const char* spec_json, ps_tables** out);
int ps_tables_info(const ps_tables* tables, int* nvar, int* ngroups, int64_t* nterms);
int ps_tables_free(ps_tables* tables);
int ps_eval_batched(ps_ctx* ctx, const ps_tables* tables, const int64_t* points, int64_t npts,
                    double* pred, uint8_t* argmin, double* kernel_seconds);
/* K18 specialised to one table set: the tables' feature polynomials and
 * model programs as one kernel compiled at run time (NVRTC, sm_100a) and
 * cached per device — what ps_eval_batched launches unless the option
 * "k18_jit" is off (then the table interpreter). ps_eval_prepare compiles
 * and loads it ahead of the first evaluation (jit_seconds: the time this
 * call spent); ps_eval_jit_source returns the generated CUDA source;
 * ps_eval_jit_compile compiles it without a device (cubin size out). Same
 * bits as the interpreter and ps_eval_cpu. Table sets whose generated source
 * exceeds 512 KB (~150 variants) keep the interpreter. */
int ps_eval_prepare(ps_ctx* ctx, const ps_tables* tables, double* jit_seconds);
int ps_eval_jit_source(const ps_tables* tables, char* out, size_t cap, size_t* needed);
int ps_eval_jit_compile(const ps_tables* tables, size_t* cubin_bytes);
/* The same evaluation on `threads` host threads (CPU port of K18). */
int ps_eval_cpu(const ps_tables* tables, const int64_t* points, int64_t npts, double* pred,
                uint8_t* argmin, int threads);

/* --- host pipeline over the C++ port (no GPU) ----------------------------
 * Text in, caller-owned buffers out. Lists are newline-separated. */

/* KernelCollection::generate (uipick.cpp:71-119) over catalog "reference"
 * (builtin_generators, uipick.cpp:669-804) or "b200" (B200 ladders + DG);
 * tags one per line, match = identical|subset|superset|intersect. Output:
 * "variant_id\tbindings\n" per kernel. */
int ps_catalog(const char* catalog, const char* tags, const char* match, char* out, size_t cap,
               size_t* needed);
/* parse_model_file (model.cpp:625-644) -> JSON {output, expression, params,
 * features, cost_params}. */
/* One catalog kernel as {"id", "kernel": perfseer-kernel/1 JSON
 * (kernel_json.cpp:135-196), "bindings"} — what the reference's
 * kernel_from_json + analyze consume (stage-file interop). */
int ps_kernel_json(const char* variant_id, char* out, size_t cap, size_t* needed);
int ps_model_info(const char* model_text, char* out, size_t cap, size_t* needed);
/* gather_feature_values (features.cpp:473-493) for the model's features over
 * kernels given by variant id: out[k * nf + f]. */
int ps_feature_table(const char* model_text, const char* variant_ids, int sub_group_size,
                     double* out, int64_t cap_values);
/* fit_model (model.cpp:485-606), bit-identical to the reference; scale != 0
 * applies scale_features_by_output (model.cpp:421-435) first. */
int ps_fit_cpu(const char* model_text, const double* features, const double* t, int nr, int scale,
               const ps_fit_opts* opts, double* params_out, ps_fit_stats* stats);
/* The reference's deterministic LM start (model.cpp:439-481). */
int ps_initial_point(const char* model_text, const double* features, const double* t, int nr,
                     int scale, double* params_out);
/* predict (model.cpp:615-623) per kernel variant id. */
int ps_predict_cpu(const char* model_text, const double* params, const char* variant_ids,
                   int sub_group_size, double* out, int64_t cap);
/* Postfix bytecode of the model (which = -1) or of d model / d p_which. */
int ps_model_bytecode(const char* model_text, int which, int32_t* ops, int cap_ops, double* consts,
                      int cap_consts, int* n_ops, int* n_consts, int* max_stack);
/* Process-wide options of the host port. "partial_subgroups" = "strict"
 * (reference: sub-group counts need wg % 32 == 0, features.cpp:318-326) or
 * "round_up" (a work-group issues ceil(wg/32) sub-groups). */
/* Exact counts of a generated variant at its own bindings (SPEC acceptance 1
 * at any size), as JSON {"ops", "access_counts", "access_footprints",
 * "footprints", "barrier_local", "group_launch"}: mode 0 = symbolic
 * (counting.cpp analyze), 1 = CPU enumeration (oracle.cpp:429-443
 * brute_force_count), 2 = the same enumeration on the GPU of ctx. */
int ps_enumerate(ps_ctx* ctx, const char* variant_id, int mode, char* out, size_t cap,
                 size_t* needed);
/* The model (and with_jacobian, its np symbolic derivatives, diff_expr
 * model.cpp:289-330) as one straight-line register program with common
 * subexpressions computed once (what K17/K18 execute): JSON {"insns": [op <<
 * 16 | dst, a << 16 | b, ...], "consts", "outputs": [slot per expression],
 * "n_slots", "n_nodes"}. */
int ps_model_program(const char* model_text, int with_jacobian, char* out, size_t cap,
                     size_t* needed);
/* Process-wide options: "partial_subgroups" = strict (the reference: raise
 * when a work-group is not a whole number of sub-groups) | round_up
 * (ceil(wg/32) sub-groups); "launch_geometry" = realised
 * (vectorised row sweeps, FD strips) | literal (one CTA per IR work-group,
 * the grid/block of launch_geometry, transforms.cpp:242-275);
 * "k18_jit" = on (default: ps_eval_batched runs the tables' run-time
 * specialised kernel) | off (the table interpreter);
 * "measure_queue_ahead" = on (default: ps_measure enqueues a short idle
 * kernel before the timed trials so each event pair brackets device work
 * only, like the OpenCL profiling timestamps the paper reads) | off. */
int ps_set_option(const char* key, const char* value);
/* NVTX ranges for a host pipeline's stages (sweep, e2e, fits, predictions:
 * visible in nsys / ncu timelines; free without a profiler). The library
 * opens its own ranges around ps_measure, the e2e batch, K17, K18 and the K18
 * compile. */
int ps_trace_push(const char* name);
int ps_trace_pop(void);
/* geo_mean_rel_error (executor.cpp:50-61). */
int ps_geo_mean_rel_error(const double* pred, const double* meas, int n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PERFSEER_B200_H_ */
