// K17 (v2): every Levenberg-Marquardt fit of a calibration round in ONE
// launch — applications x models x starts, one CTA per fit.
//
// Algorithm = the reference fit_model (model.cpp:485-606), as in lm.cu: r =
// t - g(p), stop when |J^T r|_inf < grad_tol, damped normal equations
// (J^T J + lambda I) delta = J^T r by Gaussian elimination with partial
// pivoting (pivot < 1e-300 -> raise lambda), accept when the candidate cost
// is finite and <= the current one (lambda *= decrease, relative-step stop),
// else lambda *= increase; lambda > 1e100 is divergence.
//
// What is B200-shaped here:
// * the model and its np symbolic derivatives run as ONE straight-line
//   register program with shared subexpressions (ps_model.cpp
//   compile_program: e.g. the DG ldst_g model + Jacobian is 866 instructions
//   instead of 3 million tree-walk operations per row), bit-identical to the
//   tree walk; a value-only program evaluates candidate steps;
// * the Jacobian rows (nr x (np + 1) doubles) live in shared memory when they
//   fit (the whole calibration table of one application does), so J^T J is
//   formed from shared memory;
// * J^T J / J^T r: in reference mode one thread per entry sums the rows in
//   row order (the reference's loop order, bitwise); in shuffle mode one warp
//   per entry with a shuffle tree;
// * the damped solve is warp-cooperative: lane r owns row r of the
//   augmented matrix, the pivot is a warp arg-max (first maximum, the
//   reference's strict '>' scan), eliminations run on all rows at once with
//   each element's operation sequence unchanged; back substitution on lane 0
//   in the reference's order.
// Compiled with -fmad=false (Makefile): no contraction, so reference-mode
// fits are bit-identical to fit_model (tests/test_gpu_lm.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "libm_glibc.cuh"
#include "runtime_internal.h"

namespace ps {

constexpr int kJobThreads = 256;
constexpr int kJobMaxParams = 32;  // one warp lane per row of the solve
constexpr int kJobMaxSlots = 96;

struct DevProgram {
  const uint32_t* insns;  // [n_insns][2]
  const double* consts;
  const int32_t* outputs;
  int n_insns, n_outputs, n_slots;
};

struct DevJob {
  DevProgram value, full;
  int np, nf, nr, nbatch, mode, shared_rows;
  const double* features;
  const double* t;
  ps_fit_opts opt;
  double* params;
  ps_fit_stats* stats;
  double* work;  // global J rows when they do not fit in shared memory (else null)
  int first_cta;
};

// Runs the program at (p, f); its registers live at s[slot * stride]:
// shared memory (stride = blockDim.x, one column per thread) when the CTA
// has room, else the thread's local array (stride 1). The results stay in
// the slots named by pr.outputs.
template <int kStride>
__device__ __forceinline__ void exec_program(const DevProgram& pr, const double* __restrict__ p,
                                             const double* __restrict__ f, double* s, int stride) {
  const int st = kStride ? kStride : stride;
  // one 8-byte load per instruction, fetched one instruction ahead so the
  // fetch latency overlaps the current instruction's operands and operation
  const uint2* ins = reinterpret_cast<const uint2*>(pr.insns);
  const int n = pr.n_insns;
  uint2 next = n > 0 ? __ldg(ins) : make_uint2(0u, 0u);
  for (int i = 0; i < n; ++i) {
    const uint2 w = next;
    if (i + 1 < n) next = __ldg(ins + i + 1);
    const uint32_t w0 = w.x, w1 = w.y;
    const int op = int(w0 >> 16), d = int(w0 & 0xffff), a = int(w1 >> 16), b = int(w1 & 0xffff);
    double v;
    switch (op) {
      case PS_BC_NUM: v = __ldg(pr.consts + a); break;
      case PS_BC_PARAM: v = p[a]; break;
      case PS_BC_FEAT: v = f[a]; break;
      case PS_BC_TANH: v = glibc_tanh(s[a * st]); break;
      case PS_BC_ADD: v = __dadd_rn(s[a * st], s[b * st]); break;
      case PS_BC_SUB: v = __dsub_rn(s[a * st], s[b * st]); break;
      case PS_BC_MUL: v = __dmul_rn(s[a * st], s[b * st]); break;
      default: v = __ddiv_rn(s[a * st], s[b * st]);
    }
    s[d * st] = v;
  }
}

struct Fit {
  const DevJob* J;
  const double* f;  // [nr][nf]
  const double* t;  // [nr]
  double* w;        // [nr][np + 1]: scaled J row, then the residual
  double* slots;    // program registers in shared memory ([slot][thread]) or null
  int np, nr, stride;
  bool ordered, relative;
};

// Residuals (and, with jacobian, the scaled Jacobian) of every row.
__device__ void rows_eval(const Fit& F, const double* p, const double* scale, bool jacobian) {
  double local[kJobMaxSlots];
  const DevProgram& pr = jacobian ? F.J->full : F.J->value;
  double* s = F.slots ? F.slots + threadIdx.x : local;
  const int stride = F.slots ? (int)blockDim.x : 1;
  for (int k = threadIdx.x; k < F.nr; k += blockDim.x) {
    const double* fk = F.f + (size_t)k * F.J->nf;
    double* wk = F.w + (size_t)k * F.stride;
    // relative mode: r = (t - g) / t and J / t (the paper's output scaling
    // applied to the model; see lm.cu)
    const double tk = F.t[k];
    const double w_row = F.relative ? 1.0 / tk : 1.0;
    if (F.slots)
      exec_program<0>(pr, p, fk, s, stride);
    else
      exec_program<1>(pr, p, fk, s, 1);
    wk[F.np] = __dmul_rn(__dsub_rn(tk, s[pr.outputs[0] * stride]), w_row);
    if (jacobian)
      for (int i = 0; i < F.np; ++i)
        wk[i] = __dmul_rn(__dmul_rn(s[pr.outputs[1 + i] * stride], scale[i]), w_row);
  }
  __syncthreads();
}

// sum_k x(k): row order by one thread, or a warp shuffle tree.
template <class X>
__device__ double row_reduce(int nr, bool ordered, X&& x) {
  if (ordered) {
    double s = 0.0;
    for (int k = 0; k < nr; ++k) s = __dadd_rn(s, x(k));
    return s;
  }
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int k = lane; k < nr; k += 32) s = __dadd_rn(s, x(k));
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

__device__ double cost_of(const Fit& F, double* red) {
  if (threadIdx.x < 32) {
    const double s = row_reduce(F.nr, F.ordered, [&](int k) {
      const double r = F.w[(size_t)k * F.stride + F.np];
      return __dmul_rn(r, r);
    });
    if (threadIdx.x == 0) *red = s;
  }
  __syncthreads();
  const double c = *red;
  __syncthreads();
  return c;
}

// Warp 0: solve (jtj + lambda I) x = jtr by Gaussian elimination with partial
// pivoting, the reference's arithmetic (solve_dense, model.cpp:367-391).
// Returns 0 ok, 3 singular. a: [np][np + 1] shared scratch.
__device__ int warp_solve(int np, const double* jtj, const double* jtr, double lambda, double* a, double* x) {
  const int lane = threadIdx.x & 31;
  const int ld = np + 1;
  if (lane < np) {
    for (int c = 0; c < np; ++c) a[lane * ld + c] = jtj[lane * np + c];
    a[lane * ld + lane] = __dadd_rn(a[lane * ld + lane], lambda);
    a[lane * ld + np] = jtr[lane];
  }
  __syncwarp();
  for (int col = 0; col < np; ++col) {
    // pivot: the first row in col.. with the largest |a[r][col]| (the
    // reference keeps the earlier row on ties: strict '>')
    double v = lane >= col && lane < np ? fabs(a[lane * ld + col]) : -1.0;
    int idx = lane;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    if (v < 1e-300) return 3;  // singular (a NaN pivot is not, as in the reference)
    if (idx != col) {
      for (int c = lane; c <= np; c += 32) {
        const double tmp = a[idx * ld + c];
        a[idx * ld + c] = a[col * ld + c];
        a[col * ld + c] = tmp;
      }
    }
    __syncwarp();
    if (lane > col && lane < np) {
      const double fct = __ddiv_rn(a[lane * ld + col], a[col * ld + col]);
      if (fct != 0.0) {
        for (int c = col; c < np; ++c)
          a[lane * ld + c] = __dsub_rn(a[lane * ld + c], __dmul_rn(fct, a[col * ld + c]));
        a[lane * ld + np] = __dsub_rn(a[lane * ld + np], __dmul_rn(fct, a[col * ld + np]));
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    for (int col = np - 1; col >= 0; --col) {
      double acc = a[col * ld + np];
      for (int c = col + 1; c < np; ++c) acc = __dsub_rn(acc, __dmul_rn(a[col * ld + c], x[c]));
      x[col] = __ddiv_rn(acc, a[col * ld + col]);
    }
  }
  __syncwarp();
  return 0;
}

__global__ void __launch_bounds__(kJobThreads) lm_jobs_kernel(const DevJob* __restrict__ jobs, int njobs,
                                                              size_t rows_bytes, int slots_in_smem) {
  // the job of this CTA: the last job whose first CTA is <= blockIdx.x
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (jobs[mid].first_cta <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const DevJob& J = jobs[lo];
  const int b = (int)blockIdx.x - J.first_cta;
  const int np = J.np;
  extern __shared__ double smem[];
  __shared__ double p[kJobMaxParams], cand[kJobMaxParams], scale[kJobMaxParams], x[kJobMaxParams];
  __shared__ double jtj[kJobMaxParams * kJobMaxParams], jtr[kJobMaxParams];
  __shared__ double aug[kJobMaxParams * (kJobMaxParams + 1)];
  __shared__ double red;
  __shared__ int flag_sh;   // gradient / step test: 1 converged
  __shared__ int solve_sh;  // damped solve: 0 ok, 2 diverged, 3 singular (its own word: warp 0
                            // writes it while other warps may still read flag_sh)

  Fit F;
  F.J = &J;
  F.np = np;
  F.nr = J.nr;
  F.stride = np + 1;
  F.f = J.features + (J.shared_rows ? 0 : (size_t)b * J.nr * J.nf);
  F.t = J.t + (J.shared_rows ? 0 : (size_t)b * J.nr);
  F.w = J.work ? J.work + (size_t)b * J.nr * F.stride : smem;
  // program registers after the J rows (dynamic shared memory), when they fit
  F.slots = slots_in_smem ? smem + rows_bytes / sizeof(double) : nullptr;
  F.ordered = (J.mode & 2) == 0;
  F.relative = (J.mode & 4) != 0;
  const ps_fit_opts& opt = J.opt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;

  if (threadIdx.x < np) {
    const double p0 = J.params[(size_t)b * np + threadIdx.x];
    scale[threadIdx.x] = 1.0;
    p[threadIdx.x] = opt.nonnegative ? fmax(p0, 0.0) : p0;
  }
  __syncthreads();
  if (J.mode & 1) {
    // column equilibration: q = p / s with s_i = 1 / |J[:, i]| at the start
    rows_eval(F, p, scale, true);
    if (threadIdx.x < np) {
      double s2 = 0.0;
      for (int k = 0; k < F.nr; ++k) {
        const double v = F.w[(size_t)k * F.stride + threadIdx.x];
        s2 = __dadd_rn(s2, __dmul_rn(v, v));
      }
      scale[threadIdx.x] = s2 > 0.0 && isfinite(s2) ? 1.0 / sqrt(s2) : 1.0;
    }
    __syncthreads();
  }
  rows_eval(F, p, scale, false);
  double cost = cost_of(F, &red);
  double lambda = opt.lambda0;
  int iter = 0, converged = 0, status = 0, trials = 0;
  if (!isfinite(cost)) status = 3;

  for (; !status && iter < opt.max_iterations; ++iter) {
    rows_eval(F, p, scale, true);
    const int entries = np + np * np;
    if (F.ordered) {
      for (int e = threadIdx.x; e < entries; e += blockDim.x) {
        const int i = e < np ? e : (e - np) / np, j = e < np ? np : (e - np) % np;
        double s = 0.0;
        for (int k = 0; k < F.nr; ++k)
          s = __dadd_rn(s, __dmul_rn(F.w[(size_t)k * F.stride + i], F.w[(size_t)k * F.stride + j]));
        (e < np ? jtr[i] : jtj[e - np]) = s;
      }
    } else {
      for (int e = warp; e < entries; e += nwarps) {
        const int i = e < np ? e : (e - np) / np, j = e < np ? np : (e - np) % np;
        const double s = row_reduce(F.nr, false, [&](int k) {
          return __dmul_rn(F.w[(size_t)k * F.stride + i], F.w[(size_t)k * F.stride + j]);
        });
        if (lane == 0) (e < np ? jtr[i] : jtj[e - np]) = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double gmax = 0.0;  // |gradient| of 0.5 |r|^2 in p coordinates: J^T r / s
      for (int i = 0; i < np; ++i) gmax = fmax(gmax, fabs(__ddiv_rn(jtr[i], scale[i])));
      flag_sh = gmax < opt.grad_tol ? 1 : 0;
    }
    __syncthreads();
    if (flag_sh == 1) {
      converged = 1;
      break;
    }
    bool accepted = false;
    while (!accepted) {
      ++trials;
      if (warp == 0) {
        int fl = 0;
        if (lambda > 1e100) {
          fl = 2;
        } else {
          fl = warp_solve(np, jtj, jtr, lambda, aug, x);
          if (fl == 0 && lane < np) {
            double v = __dadd_rn(p[lane], __dmul_rn(x[lane], scale[lane]));
            if (opt.nonnegative) v = fmax(v, 0.0);
            cand[lane] = v;
          }
        }
        if (lane == 0) solve_sh = fl;
      }
      __syncthreads();
      if (solve_sh == 2) {
        status = 1;
        break;
      }
      if (solve_sh == 3) {
        lambda *= opt.lambda_increase;
        __syncthreads();
        continue;
      }
      rows_eval(F, cand, scale, false);
      const double cand_cost = cost_of(F, &red);
      if (isfinite(cand_cost) && cand_cost <= cost) {
        if (threadIdx.x == 0) {
          double step = 0.0, sc = 0.0;
          for (int i = 0; i < np; ++i) {
            const double dq = __ddiv_rn(__dsub_rn(cand[i], p[i]), scale[i]);
            const double q = __ddiv_rn(p[i], scale[i]);
            step = __dadd_rn(step, __dmul_rn(dq, dq));
            sc = __dadd_rn(sc, __dmul_rn(q, q));
          }
          for (int i = 0; i < np; ++i) p[i] = cand[i];
          flag_sh = sqrt(step) < opt.step_tol * (sqrt(sc) + opt.step_tol) ? 1 : 0;
        }
        __syncthreads();
        cost = cand_cost;
        lambda *= opt.lambda_decrease;
        accepted = true;
        if (flag_sh == 1) converged = 1;
      } else {
        lambda *= opt.lambda_increase;
      }
      __syncthreads();
    }
    if (status) break;
    if (converged) {
      ++iter;
      break;
    }
  }
  if (threadIdx.x < np) J.params[(size_t)b * np + threadIdx.x] = p[threadIdx.x];
  if (threadIdx.x == 0) {
    J.stats[b].residual_norm = sqrt(cost);
    J.stats[b].iterations = iter;
    J.stats[b].converged = converged;
    J.stats[b].status = status;
    J.stats[b].trials = trials;
  }
}

int fit_lm_jobs_gpu(Ctx* c, int njobs, const LmJobHost* jobs, double* kernel_seconds) {
  TraceRange trace("K17 fit_lm_jobs");
  if (njobs < 1) return set_error(PS_ERR_ARG, "ps_fit_lm_jobs: no jobs");
  int dev_smem = 0;
  cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  const size_t static_smem = sizeof(double) * (4 * kJobMaxParams + kJobMaxParams * kJobMaxParams + kJobMaxParams +
                                               kJobMaxParams * (kJobMaxParams + 1) + 1) + 64;
  const size_t smem_cap = (size_t)dev_smem > static_smem ? (size_t)dev_smem - static_smem : 0;
  // J rows in shared memory when every job's fits: the largest job decides
  size_t rows_bytes = 0;
  for (int j = 0; j < njobs; ++j) {
    const LmJobHost& h = jobs[j];
    if (h.np < 1 || h.np > kJobMaxParams)
      return set_error(PS_ERR_ARG, "job %d: np must be in 1..%d", j, kJobMaxParams);
    if (h.nr < h.np)
      return set_error(PS_ERR_ARG,
                       "job %d: rank deficiency: %d measurement rows for %d parameters; the feature "
                       "matrix cannot have full column rank", j, h.nr, h.np);
    if (h.nbatch < 1) return set_error(PS_ERR_ARG, "job %d: nbatch must be >= 1", j);
    if (h.full.n_outputs != h.np + 1 || h.value.n_outputs != 1)
      return set_error(PS_ERR_ARG, "job %d: programs do not match np", j);
    if (h.full.n_slots > kJobMaxSlots || h.value.n_slots > kJobMaxSlots)
      return set_error(PS_ERR_ARG, "job %d: model program needs %d registers (device: %d)", j,
                       std::max(h.full.n_slots, h.value.n_slots), kJobMaxSlots);
    rows_bytes = std::max(rows_bytes, sizeof(double) * (size_t)h.nr * (h.np + 1));
  }
  const bool rows_in_smem = rows_bytes <= smem_cap;
  cudaSetDevice(c->device);
  // one device block: programs, features, t, params, stats, job table (+ global J rows)
  size_t total = 4096 + sizeof(DevJob) * njobs;
  auto al = [](size_t n) { return (n + 255) & ~size_t(255); };
  for (int j = 0; j < njobs; ++j) {
    const LmJobHost& h = jobs[j];
    for (const LmProgramHost* pr : {&h.value, &h.full})
      total += al(sizeof(uint32_t) * 2 * pr->n_insns) + al(sizeof(double) * std::max(1, pr->n_consts)) +
               al(sizeof(int32_t) * pr->n_outputs);
    const size_t rows = h.shared_rows ? 1 : (size_t)h.nbatch;
    total += al(sizeof(double) * rows * h.nr * h.nf) + al(sizeof(double) * rows * h.nr) +
             al(sizeof(double) * h.nbatch * h.np) + al(sizeof(ps_fit_stats) * h.nbatch);
    if (!rows_in_smem) total += al(sizeof(double) * (size_t)h.nbatch * h.nr * (h.np + 1));
  }
  int rc = c->ensure(c->scratch[2], total);
  if (rc) return rc;
  char* base = static_cast<char*>(c->scratch[2].ptr);
  size_t off = 0;
  auto carve = [&](size_t n) {
    char* q = base + off;
    off += al(n);
    return q;
  };
  auto up = [&](const void* src, size_t n) -> void* {
    void* d = carve(n);
    if (n) cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, c->stream);
    return d;
  };
  std::vector<DevJob> dj((size_t)njobs);
  int ctas = 0;
  for (int j = 0; j < njobs; ++j) {
    const LmJobHost& h = jobs[j];
    DevJob& d = dj[(size_t)j];
    auto prog = [&](const LmProgramHost& pr) {
      DevProgram out;
      out.insns = static_cast<const uint32_t*>(up(pr.insns, sizeof(uint32_t) * 2 * pr.n_insns));
      out.consts = static_cast<const double*>(up(pr.consts, sizeof(double) * pr.n_consts));
      out.outputs = static_cast<const int32_t*>(up(pr.outputs, sizeof(int32_t) * pr.n_outputs));
      out.n_insns = pr.n_insns;
      out.n_outputs = pr.n_outputs;
      out.n_slots = pr.n_slots;
      return out;
    };
    d.value = prog(h.value);
    d.full = prog(h.full);
    d.np = h.np;
    d.nf = h.nf;
    d.nr = h.nr;
    d.nbatch = h.nbatch;
    d.mode = h.mode;
    d.shared_rows = h.shared_rows;
    const size_t rows = h.shared_rows ? 1 : (size_t)h.nbatch;
    d.features = static_cast<const double*>(up(h.features, sizeof(double) * rows * h.nr * h.nf));
    d.t = static_cast<const double*>(up(h.t, sizeof(double) * rows * h.nr));
    d.opt = h.opts;
    d.params = static_cast<double*>(up(h.params, sizeof(double) * h.nbatch * h.np));
    d.stats = reinterpret_cast<ps_fit_stats*>(carve(sizeof(ps_fit_stats) * h.nbatch));
    d.work = rows_in_smem ? nullptr
                          : reinterpret_cast<double*>(carve(sizeof(double) * (size_t)h.nbatch * h.nr * (h.np + 1)));
    d.first_cta = ctas;
    ctas += h.nbatch;
  }
  DevJob* djobs = static_cast<DevJob*>(up(dj.data(), sizeof(DevJob) * njobs));
  const size_t rows_dyn = rows_in_smem ? rows_bytes : 0;
  // program registers in shared memory ([slot][thread], every thread its
  // column) when they fit beside the J rows: the interpreter's operand
  // traffic stays on chip instead of in local memory
  int max_slots = 1;
  for (int j = 0; j < njobs; ++j) max_slots = std::max({max_slots, jobs[j].full.n_slots, jobs[j].value.n_slots});
  const size_t slots_bytes = sizeof(double) * (size_t)max_slots * kJobThreads;
  const bool slots_in_smem = rows_dyn + slots_bytes <= smem_cap && !std::getenv("PS_LM_LOCAL_SLOTS");
  const size_t dyn = rows_dyn + (slots_in_smem ? slots_bytes : 0);
  // static + dynamic above 48 KB needs the opt-in limit raised
  if (cudaFuncSetAttribute(lm_jobs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess)
    return set_error(PS_ERR_CUDA, "LM jobs: cannot reserve %zu B of shared memory", dyn);
  if ((rc = events(c, 2))) return rc;
  cudaEventRecord(c->ev[0], c->stream);
  lm_jobs_kernel<<<ctas, kJobThreads, dyn, c->stream>>>(djobs, njobs, rows_dyn, slots_in_smem ? 1 : 0);
  cudaEventRecord(c->ev[1], c->stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "LM jobs launch failed: %s", cudaGetErrorString(e));
  for (int j = 0; j < njobs; ++j) {
    const LmJobHost& h = jobs[j];
    cudaMemcpyAsync(h.params, dj[(size_t)j].params, sizeof(double) * h.nbatch * h.np, cudaMemcpyDeviceToHost,
                    c->stream);
    cudaMemcpyAsync(h.stats, dj[(size_t)j].stats, sizeof(ps_fit_stats) * h.nbatch, cudaMemcpyDeviceToHost,
                    c->stream);
  }
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "LM jobs failed: %s", cudaGetErrorString(e));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
  if (kernel_seconds) *kernel_seconds = ms * 1e-3;
  return PS_OK;
}

}  // namespace ps
