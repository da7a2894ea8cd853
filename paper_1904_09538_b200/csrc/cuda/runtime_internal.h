// Internal state of a ps_ctx (one per GPU) and the launch helpers shared by
// the suite, DG, tensor-core and model translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../../include/perfseer_b200.h"

namespace ps {

// NVTX range over a host-side stage (header-only NVTX v3: free unless a
// profiler is attached); shows ps_measure / fits / evaluations in nsys/ncu
// timelines (SURVEY §5 tracing).
struct TraceRange {
  explicit TraceRange(const char* name) { nvtxRangePushA(name); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange&) = delete;
  TraceRange& operator=(const TraceRange&) = delete;
};

struct DevBuf {
  void* ptr = nullptr;
  size_t cap = 0;
};

// Device arrays of one prepared kernel variant. Slots stay resident (inputs
// filled once, in HBM) until the LRU cache exceeds its byte budget.
struct Slot {
  DevBuf in[PS_MAX_ARRAYS];
  DevBuf out[PS_MAX_ARRAYS];
  ps_io_info io{};
  int fill_mode = -1;
  uint64_t seed = 0;
  uint64_t last_use = 0;
  size_t bytes = 0;
};

struct Ctx {
  int device = 0;
  int sm_count = 0;
  int sm_clock_khz = 0;
  size_t l2_bytes = 0;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<cudaEvent_t> marks;  // ps_mark slots
  DevBuf in[PS_MAX_ARRAYS];   // views of the active slot (not owned)
  DevBuf out[PS_MAX_ARRAYS];
  DevBuf scratch[8];
  std::map<std::string, Slot> slots;  // keyed by the raw descriptor bytes
  Slot host_slot;                     // caller-data runs (verify / run_host)
  // ps_run_host_batch: one device arena the kernels' arrays are placed in as
  // a ring (byte-level lookahead for the copy engines), copy-in / copy-out
  // streams and per-kernel events ordering them against the launches
  DevBuf arena;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> pipe_ev[3];  // [h2d done, launch done, d2h done][kernel]
  size_t cache_bytes = 0, cache_cap = 0;
  uint64_t tick = 0;
  bool prepared = false;
  ps_kernel_desc desc{};
  ps_io_info io{};
  int fill_mode = 0;
  uint64_t seed = 0;
  bool force_generic = false;
  // flops_pattern initial values v_j = base + step*j (uipick.cpp:339-343)
  float flop_base = 0.5f;
  float flop_step = 0.015625f;

  int ensure(DevBuf& b, size_t bytes, const std::string* keep = nullptr);
  void activate(Slot& s);
  void release(Slot& s);
};

int set_error(int code, const char* fmt, ...);
int validate_desc(const ps_kernel_desc* d);
int kernel_io(const ps_kernel_desc* d, ps_io_info* io);
int parse_variant_id(const char* id, ps_kernel_desc* d);
int launch(Ctx* c, const ps_kernel_desc* d);
int events(Ctx* c, int n);

int dg_validate(const ps_kernel_desc* d);
int dg_io(const ps_kernel_desc* d, ps_io_info* io);
const char* dg_input_name(const ps_kernel_desc* d, int i);
int dg_launch(Ctx* c, const ps_kernel_desc* d);
int tc_launch(Ctx* c, const ps_kernel_desc* d);
int dg_tc_launch(Ctx* c, const ps_kernel_desc* d);

}  // namespace ps

namespace ps {

// Flat view of compiled prediction tables (built host-side by
// perfseer::build_variant_tables, consumed by the K18 kernel).
struct FlatTables {
  int nvar, ngroups, nmodels;
  const int32_t *var_group, *var_model, *var_feat_base;
  const int32_t *feat_begin, *feat_end;
  const int64_t *feat_den, *term_coef;
  const int8_t* term_exp;  // [nterms][4]
  int nslots, nterms;
  const int32_t* model_nf;          // [nmodels]
  const int32_t* model_insn_begin;  // [nmodels + 1] into insns (instruction index)
  const uint32_t* insns;            // [n][2]: op << 16 | dst, a << 16 | b
  const int32_t* model_out;         // [nmodels] result register
  const int32_t* model_regs;        // [nmodels] registers used
  const int32_t* model_const_begin;  // [nmodels + 1] into consts
  const double* consts;
  const int32_t* model_param_begin;  // [nmodels + 1] into params
  const double* params;
};

// Device evaluator limits (K18 eval.cu, K17 lm.cu); the C ABI rejects inputs
// beyond them before any launch.
constexpr int kEvalMaxFeat = 48;
constexpr int kEvalMaxGroups = 8;
constexpr int kEvalMaxStack = 48;
constexpr int kEvalMaxRegs = 64;
constexpr int kEvalMaxVariants = 256;  // argmin is one byte per group
constexpr int kLmMaxParams = 24;
constexpr int kLmMaxStack = 48;
constexpr int kDualStack = 24;

// Deepest stack a postfix program reaches; -1 when it underflows, ends with
// other than one value, or references a constant/parameter/feature outside
// [0, n_consts) / [0, np) / [0, nf).
int bytecode_depth(const int32_t* ops, int n_ops, int n_consts, int np, int nf);

// Launch geometry switch (runtime.cu): literal = one CTA per IR work-group.
void set_literal_geometry(bool on);
bool literal_geometry();
// Queue-ahead kernel before ps_measure's timed trials (on by default).
void set_queue_ahead(bool on);
// K18 run-time specialisation (eval_jit.cu): the tables as one NVRTC-compiled
// kernel (on by default; off = the table interpreter in eval.cu).
struct JitKernels {
  cudaKernel_t predict = nullptr;  // grid.y = variant: pred[pt][v]
  cudaKernel_t rank = nullptr;     // argmin per group from pred
  int lanes = 1;                   // points per thread of predict
};
void set_k18_jit(bool on);
bool k18_jit_enabled();
std::string k18_jit_source(const struct FlatTables& h);
int k18_jit_compile(const std::string& src, std::vector<char>* cubin);
int k18_jit_kernel(Ctx* c, const struct FlatTables& h, void** kernel, double* compile_seconds);

// K17 v2 (lm_jobs.cu): straight-line model programs (host-compiled,
// perfseer::compile_program) and one fit job per (model, problem, starts).
struct LmProgramHost {
  const uint32_t* insns;  // [n_insns][2]
  const double* consts;
  const int32_t* outputs;
  int n_insns, n_consts, n_outputs, n_slots;
};
struct LmJobHost {
  LmProgramHost value, full;  // value: the model; full: the model and its np derivatives
  int np, nf, nr, nbatch, mode, shared_rows;
  const double* features;  // [shared_rows ? 1 : nbatch][nr][nf]
  const double* t;         // [shared_rows ? 1 : nbatch][nr]
  ps_fit_opts opts;
  double* params;          // [nbatch][np] in/out
  ps_fit_stats* stats;     // [nbatch]
};
int fit_lm_jobs_gpu(Ctx* c, int njobs, const LmJobHost* jobs, double* kernel_seconds);

// jit_kernel: the tables' specialised kernel (k18_jit_kernel), or null for
// the table interpreter
int eval_tables_gpu(Ctx* c, const FlatTables& t, const int64_t* points, int64_t npts, double* pred,
                    uint8_t* argmin, double* kernel_seconds, void* jit_kernel = nullptr);

}  // namespace ps
