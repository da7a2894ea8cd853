// K17: batched Levenberg-Marquardt calibration on the GPU.
//
// Algorithm = the reference fit_model (model.cpp:485-606): residual
// r = t - g(p); gradient -J^T r with an infinity-norm stop at grad_tol;
// damped normal equations (J^T J + lambda I) delta = J^T r solved by Gaussian
// elimination with partial pivoting (pivot < 1e-300 -> singular -> raise
// lambda); accept when the new cost is finite and <= the old one (lambda *=
// decrease, relative-step stop), else lambda *= increase; lambda > 1e100 is
// divergence. One CTA per fit (a batch = independent fits: models x starts);
// rows are spread over the CTA's threads, J^T J / J^T r / cost are formed
// with warp-shuffle reductions in a fixed order (deterministic run to run;
// summation order differs from the CPU's sequential loop, hence the 1e-4
// parity tolerance of the spec). Optional column equilibration p = s * q
// (s = |initial p|) runs the same iteration in scaled coordinates.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "libm_glibc.cuh"
#include "runtime_internal.h"

namespace ps {

constexpr int kLmThreads = 256;

struct LmProgram {
  const int32_t* ops;
  const double* consts;
  int n_ops;
};

__device__ double run_program(const LmProgram& pr, const double* p, const double* f) {
  double st[kLmMaxStack];
  int sp = 0;
  for (int i = 0; i < pr.n_ops; ++i) {
    const int32_t w = pr.ops[i];
    const int code = w >> 16, arg = w & 0xffff;
    switch (code) {
      case PS_BC_NUM: st[sp++] = pr.consts[arg]; break;
      case PS_BC_PARAM: st[sp++] = p[arg]; break;
      case PS_BC_FEAT: st[sp++] = f[arg]; break;
      case PS_BC_TANH: st[sp - 1] = glibc_tanh(st[sp - 1]); break;
      default: {
        const double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = code == PS_BC_ADD ? __dadd_rn(a, b)
                     : code == PS_BC_SUB ? __dsub_rn(a, b)
                     : code == PS_BC_MUL ? __dmul_rn(a, b)
                                         : __ddiv_rn(a, b);
      }
    }
  }
  return st[0];
}

// Forward-mode differentiation of the model bytecode: every stack slot
// carries its value and its gradient with respect to the np parameters, so
// one pass yields g and dg/dp without the symbolic derivative trees (which
// grow combinatorially for nested overlap steps). The product, quotient and
// tanh rules are the ones diff_expr applies (model.cpp:289-330).
__device__ void run_dual(const LmProgram& pr, const double* p, const double* f, int np, double* val,
                         double* grad) {
  double sv[kDualStack];
  double sg[kDualStack][kLmMaxParams];
  int sp = 0;
  for (int i = 0; i < pr.n_ops; ++i) {
    const int32_t w = pr.ops[i];
    const int code = w >> 16, arg = w & 0xffff;
    switch (code) {
      case PS_BC_NUM:
      case PS_BC_FEAT:
        sv[sp] = code == PS_BC_NUM ? pr.consts[arg] : f[arg];
        for (int j = 0; j < np; ++j) sg[sp][j] = 0.0;
        ++sp;
        break;
      case PS_BC_PARAM:
        sv[sp] = p[arg];
        for (int j = 0; j < np; ++j) sg[sp][j] = j == arg ? 1.0 : 0.0;
        ++sp;
        break;
      case PS_BC_TANH: {
        const double t = glibc_tanh(sv[sp - 1]);
        const double d = 1.0 - t * t;
        sv[sp - 1] = t;
        for (int j = 0; j < np; ++j) sg[sp - 1][j] = d * sg[sp - 1][j];
        break;
      }
      default: {
        const int bi = --sp, ai = sp - 1;
        const double a = sv[ai], b = sv[bi];
        if (code == PS_BC_ADD || code == PS_BC_SUB) {
          const double s = code == PS_BC_ADD ? 1.0 : -1.0;
          for (int j = 0; j < np; ++j) sg[ai][j] = sg[ai][j] + s * sg[bi][j];
          sv[ai] = code == PS_BC_ADD ? a + b : a - b;
        } else if (code == PS_BC_MUL) {
          for (int j = 0; j < np; ++j) sg[ai][j] = sg[ai][j] * b + a * sg[bi][j];
          sv[ai] = a * b;
        } else {
          for (int j = 0; j < np; ++j) sg[ai][j] = sg[ai][j] / b - a * sg[bi][j] / (b * b);
          sv[ai] = a / b;
        }
      }
    }
  }
  *val = sv[0];
  for (int j = 0; j < np; ++j) grad[j] = sg[0][j];
}

struct LmArgs {
  LmProgram model;
  const LmProgram* jac;  // [np]
  int np, nf, nr, nbatch;
  const double* features;  // [nbatch][nr][nf]
  const double* t;         // [nbatch][nr]
  double* params;          // [nbatch][np] in/out
  ps_fit_stats* stats;
  double* work;            // [nbatch][nr][np + 1]: J rows and residuals
  ps_fit_opts opt;
  int equilibrate;
  int ordered;             // 1: per-entry sums in row order (reference order)
  int relative;            // 1: residuals relative to t (weights 1/t)
  int dual;                // 1: forward-mode derivatives (jac programs unused)
};

// Sum over rows k of x(k), either sequentially in row order by one thread
// (the reference's loop order) or by one warp with a shuffle tree.
template <class F>
__device__ double row_sum(int nr, bool ordered, F&& x) {
  if (ordered) {
    double s = 0.0;
    for (int k = 0; k < nr; ++k) s += x(k);
    return s;
  }
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int k = lane; k < nr; k += 32) s += x(k);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Residuals (and optionally the scaled Jacobian) of every row into `w`.
__device__ void eval_rows(const LmArgs& A, const double* f, const double* t, const double* p,
                          const double* scale, double* w, bool jacobian) {
  const int stride = A.np + 1;
  for (int k = threadIdx.x; k < A.nr; k += blockDim.x) {
    const double* fk = f + (size_t)k * A.nf;
    double* wk = w + (size_t)k * stride;
    // Relative mode: r = (t - g) / t, J = dg/dp / t — the output scaling of
    // model.cpp:421-435 applied to the model rather than to each feature, so
    // product terms (p_bar * f_barrier * f_groups) scale correctly.
    const double w_row = A.relative ? 1.0 / t[k] : 1.0;
    if (jacobian && A.dual) {
      double g, grad[kLmMaxParams];
      run_dual(A.model, p, fk, A.np, &g, grad);
      wk[A.np] = (t[k] - g) * w_row;
      for (int i = 0; i < A.np; ++i) wk[i] = grad[i] * scale[i] * w_row;
      continue;
    }
    wk[A.np] = (t[k] - run_program(A.model, p, fk)) * w_row;
    if (jacobian)
      for (int i = 0; i < A.np; ++i) wk[i] = run_program(A.jac[i], p, fk) * scale[i] * w_row;
  }
  __syncthreads();
}

// Sum of squared residuals; entry order k ascending (or warp tree).
__device__ double cost_of(const LmArgs& A, const double* w, double* red) {
  const int stride = A.np + 1;
  const bool ordered = A.ordered != 0;
  if (threadIdx.x < 32) {
    const double s = row_sum(A.nr, ordered, [&](int k) {
      const double r = w[(size_t)k * stride + A.np];
      return r * r;
    });
    if (threadIdx.x == 0) *red = s;
  }
  __syncthreads();
  const double c = *red;
  __syncthreads();
  return c;
}

__global__ void __launch_bounds__(kLmThreads) lm_batched_kernel(LmArgs A) {
  const int b = blockIdx.x;
  const int np = A.np, stride = np + 1;
  const double* f = A.features + (size_t)b * A.nr * A.nf;
  const double* t = A.t + (size_t)b * A.nr;
  double* w = A.work + (size_t)b * A.nr * stride;
  const bool ordered = A.ordered != 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;

  __shared__ double p[kLmMaxParams], cand[kLmMaxParams], scale[kLmMaxParams];
  __shared__ double jtj[kLmMaxParams * kLmMaxParams], jtr[kLmMaxParams];
  __shared__ double red;
  __shared__ int flag_sh;   // gradient / step test: 1 converged
  __shared__ int solve_sh;  // damped solve: 0 ok, 2 diverged, 3 singular (own word: thread 0
                            // writes it while other threads may still read flag_sh)

  if (threadIdx.x < np) {
    const double p0 = A.params[(size_t)b * np + threadIdx.x];
    scale[threadIdx.x] = 1.0;
    p[threadIdx.x] = A.opt.nonnegative ? fmax(p0, 0.0) : p0;
  }
  __syncthreads();
  if (A.equilibrate) {
    // Column equilibration: iterate on q = p / s with s_i = 1 / ||J[:, i]||
    // at the start, so every column of the scaled Jacobian has unit norm and
    // lambda I damps all directions alike (features span ~12 decades).
    eval_rows(A, f, t, p, scale, w, true);
    if (threadIdx.x < np) {
      double s2 = 0.0;
      for (int k = 0; k < A.nr; ++k) {
        const double v = w[(size_t)k * stride + threadIdx.x];
        s2 += v * v;
      }
      scale[threadIdx.x] = s2 > 0.0 && isfinite(s2) ? 1.0 / sqrt(s2) : 1.0;
    }
    __syncthreads();
  }
  eval_rows(A, f, t, p, scale, w, false);
  double cost = cost_of(A, w, &red);
  double lambda = A.opt.lambda0;
  int iter = 0, converged = 0, status = 0;
  if (!isfinite(cost)) status = 3;

  for (; !status && iter < A.opt.max_iterations; ++iter) {
    eval_rows(A, f, t, p, scale, w, true);
    // J^T r (entries 0..np-1) and J^T J (np..np+np^2-1): one entry per
    // thread (ordered) or per warp (shuffle tree).
    const int entries = np + np * np;
    if (ordered) {
      for (int e = threadIdx.x; e < entries; e += blockDim.x) {
        const int i = e < np ? e : (e - np) / np, j = e < np ? np : (e - np) % np;
        double s = 0.0;
        for (int k = 0; k < A.nr; ++k) s += w[(size_t)k * stride + i] * w[(size_t)k * stride + j];
        (e < np ? jtr[i] : jtj[e - np]) = s;
      }
    } else {
      for (int e = warp; e < entries; e += nwarps) {
        const int i = e < np ? e : (e - np) / np, j = e < np ? np : (e - np) % np;
        const double s = row_sum(A.nr, false, [&](int k) {
          return w[(size_t)k * stride + i] * w[(size_t)k * stride + j];
        });
        if (lane == 0) (e < np ? jtr[i] : jtj[e - np]) = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double gmax = 0.0;  // gradient of 0.5 |r|^2 in p coordinates: -J^T r / s
      for (int i = 0; i < np; ++i) gmax = fmax(gmax, fabs(jtr[i] / scale[i]));
      flag_sh = gmax < A.opt.grad_tol ? 1 : 0;
    }
    __syncthreads();
    if (flag_sh == 1) {
      converged = 1;
      break;
    }
    bool accepted = false;
    while (!accepted) {
      if (threadIdx.x == 0) {
        solve_sh = 0;
        if (lambda > 1e100) {
          solve_sh = 2;
        } else {
          double a[kLmMaxParams][kLmMaxParams + 1];
          for (int i = 0; i < np; ++i) {
            for (int c = 0; c < np; ++c) a[i][c] = jtj[i * np + c];
            a[i][i] += lambda;
            a[i][np] = jtr[i];
          }
          for (int col = 0; col < np && solve_sh == 0; ++col) {
            int piv = col;
            for (int r = col + 1; r < np; ++r)
              if (fabs(a[r][col]) > fabs(a[piv][col])) piv = r;
            if (fabs(a[piv][col]) < 1e-300) {
              solve_sh = 3;
              break;
            }
            if (piv != col)
              for (int c = 0; c <= np; ++c) {
                const double tmp = a[piv][c];
                a[piv][c] = a[col][c];
                a[col][c] = tmp;
              }
            for (int r = col + 1; r < np; ++r) {
              const double fct = a[r][col] / a[col][col];
              if (fct == 0.0) continue;
              for (int c = col; c < np; ++c) a[r][c] -= fct * a[col][c];
              a[r][np] -= fct * a[col][np];
            }
          }
          if (solve_sh == 0) {
            double x[kLmMaxParams];
            for (int col = np - 1; col >= 0; --col) {
              double acc = a[col][np];
              for (int c = col + 1; c < np; ++c) acc -= a[col][c] * x[c];
              x[col] = acc / a[col][col];
            }
            for (int i = 0; i < np; ++i) {
              double v = p[i] + x[i] * scale[i];
              if (A.opt.nonnegative) v = fmax(v, 0.0);
              cand[i] = v;
            }
          }
        }
      }
      __syncthreads();
      if (solve_sh == 2) {
        status = 1;
        break;
      }
      if (solve_sh == 3) {
        lambda *= A.opt.lambda_increase;
        __syncthreads();
        continue;
      }
      eval_rows(A, f, t, cand, scale, w, false);
      const double cand_cost = cost_of(A, w, &red);
      if (isfinite(cand_cost) && cand_cost <= cost) {
        if (threadIdx.x == 0) {
          double step = 0.0, sc = 0.0;
          for (int i = 0; i < np; ++i) {
            const double dq = (cand[i] - p[i]) / scale[i], q = p[i] / scale[i];
            step += dq * dq;
            sc += q * q;
          }
          for (int i = 0; i < np; ++i) p[i] = cand[i];
          flag_sh = sqrt(step) < A.opt.step_tol * (sqrt(sc) + A.opt.step_tol) ? 1 : 0;
        }
        __syncthreads();
        cost = cand_cost;
        lambda *= A.opt.lambda_decrease;
        accepted = true;
        if (flag_sh == 1) converged = 1;
      } else {
        lambda *= A.opt.lambda_increase;
      }
      __syncthreads();
    }
    if (status) break;
    if (converged) {
      ++iter;
      break;
    }
  }
  if (threadIdx.x < np) A.params[(size_t)b * np + threadIdx.x] = p[threadIdx.x];
  if (threadIdx.x == 0) {
    A.stats[b].residual_norm = sqrt(cost);
    A.stats[b].iterations = iter;
    A.stats[b].converged = converged;
    A.stats[b].status = status;
    A.stats[b].trials = 0;
  }
}

}  // namespace ps

namespace ps {

int bytecode_depth(const int32_t* ops, int n_ops, int n_consts, int np, int nf) {
  if (n_ops < 1 || !ops) return -1;
  int sp = 0, depth = 0;
  for (int i = 0; i < n_ops; ++i) {
    const int code = ops[i] >> 16, arg = ops[i] & 0xffff;
    switch (code) {
      case PS_BC_NUM:
      case PS_BC_PARAM:
      case PS_BC_FEAT:
        if (arg >= (code == PS_BC_NUM ? n_consts : code == PS_BC_PARAM ? np : nf)) return -1;
        depth = std::max(depth, ++sp);
        break;
      case PS_BC_TANH:
        if (sp < 1) return -1;
        break;
      case PS_BC_ADD:
      case PS_BC_SUB:
      case PS_BC_MUL:
      case PS_BC_DIV:
        if (sp < 2) return -1;
        --sp;
        break;
      default:
        return -1;
    }
  }
  return sp == 1 ? depth : -1;
}

__global__ void tanh_kernel(const double* x, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = glibc_tanh(x[i]);
}

}  // namespace ps

using namespace ps;

extern "C" int ps_math_tanh(ps_ctx* ctx, const double* x, int64_t n, double* out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !x || !out || n < 0) return set_error(PS_ERR_ARG, "ps_math_tanh: bad argument");
  if (n == 0) return PS_OK;
  cudaSetDevice(c->device);
  const size_t bytes = sizeof(double) * (size_t)n;
  int rc = c->ensure(c->scratch[0], 2 * bytes + 256);
  if (rc) return rc;
  double* dx = static_cast<double*>(c->scratch[0].ptr);
  double* dy = dx + n;
  cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, c->stream);
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  tanh_kernel<<<blocks, 256, 0, c->stream>>>(dx, n, dy);
  cudaMemcpyAsync(out, dy, bytes, cudaMemcpyDeviceToHost, c->stream);
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "tanh kernel failed: %s", cudaGetErrorString(e));
  return PS_OK;
}

extern "C" int ps_fit_lm_batched_ex(ps_ctx* ctx, const ps_bytecode* model, const ps_bytecode* jac,
                                    int np, int nf, const double* features, const double* t, int nr,
                                    int nbatch, const ps_fit_opts* opts, int equilibrate,
                                    double* params_inout, ps_fit_stats* stats) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  const bool dual = (equilibrate & 8) != 0;
  if (!c || !model || (!jac && !dual) || !features || !t || !opts || !params_inout || !stats)
    return set_error(PS_ERR_ARG, "ps_fit_lm_batched: null argument");
  if (np < 1 || np > kLmMaxParams) return set_error(PS_ERR_ARG, "np must be in 1..%d", kLmMaxParams);
  if (nr < np)
    return set_error(PS_ERR_ARG,
                     "rank deficiency: %d measurement rows for %d parameters; the feature matrix "
                     "cannot have full column rank",
                     nr, np);
  if (nbatch < 1) return set_error(PS_ERR_ARG, "nbatch must be >= 1");
  if (nf < 1 || nf > 0xffff) return set_error(PS_ERR_ARG, "nf must be in 1..65535");
  {
    // the device interpreters keep fixed stacks: reject deeper programs here
    const int dm = bytecode_depth(model->ops, model->n_ops, model->n_consts, np, nf);
    if (dm < 0) return set_error(PS_ERR_ARG, "malformed model bytecode");
    const int lim = dual ? kDualStack : kLmMaxStack;
    if (dm > lim)
      return set_error(PS_ERR_ARG, "model expression needs a stack of %d (device %s evaluator: %d)", dm,
                       dual ? "forward-mode" : "bytecode", lim);
    if (!dual)
      for (int i = 0; i < np; ++i) {
        const int dj = bytecode_depth(jac[i].ops, jac[i].n_ops, jac[i].n_consts, np, nf);
        if (dj < 0) return set_error(PS_ERR_ARG, "malformed derivative bytecode for parameter %d", i);
        if (dj > kLmMaxStack)
          return set_error(PS_ERR_ARG, "derivative %d needs a stack of %d (device evaluator: %d)", i, dj,
                           kLmMaxStack);
      }
  }
  cudaSetDevice(c->device);
  // Device copies: programs, features, t, params, stats.
  std::vector<const ps_bytecode*> progs{model};
  if (!dual)
    for (int i = 0; i < np; ++i) progs.push_back(&jac[i]);
  size_t op_words = 0, const_words = 0;
  for (auto* p : progs) {
    op_words += (size_t)p->n_ops;
    const_words += (size_t)p->n_consts;
  }
  const size_t fbytes = sizeof(double) * (size_t)nbatch * nr * nf;
  const size_t tbytes = sizeof(double) * (size_t)nbatch * nr;
  const size_t pbytes = sizeof(double) * (size_t)nbatch * np;
  const size_t sbytes = sizeof(ps_fit_stats) * (size_t)nbatch;
  const size_t wbytes = sizeof(double) * (size_t)nbatch * nr * (np + 1);
  const size_t total = op_words * 4 + const_words * 8 + sizeof(LmProgram) * (np + 1) + fbytes +
                       tbytes + pbytes + sbytes + wbytes + 2048;
  int rc = c->ensure(c->scratch[0], total);
  if (rc) return rc;
  char* base = static_cast<char*>(c->scratch[0].ptr);
  size_t off = 0;
  auto carve = [&](size_t n) {
    off = (off + 15) & ~size_t(15);
    char* p = base + off;
    off += n;
    return p;
  };
  std::vector<LmProgram> host_progs;
  for (auto* p : progs) {
    int32_t* dops = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * (size_t)p->n_ops));
    double* dconst = reinterpret_cast<double*>(carve(sizeof(double) * (size_t)std::max(1, p->n_consts)));
    if (cudaMemcpyAsync(dops, p->ops, sizeof(int32_t) * p->n_ops, cudaMemcpyHostToDevice, c->stream) ||
        (p->n_consts && cudaMemcpyAsync(dconst, p->consts, sizeof(double) * p->n_consts,
                                        cudaMemcpyHostToDevice, c->stream)))
      return set_error(PS_ERR_CUDA, "bytecode upload failed");
    host_progs.push_back(LmProgram{dops, dconst, p->n_ops});
  }
  LmProgram* djac = reinterpret_cast<LmProgram*>(carve(sizeof(LmProgram) * np));
  double* df = reinterpret_cast<double*>(carve(fbytes));
  double* dt = reinterpret_cast<double*>(carve(tbytes));
  double* dp = reinterpret_cast<double*>(carve(pbytes));
  ps_fit_stats* ds = reinterpret_cast<ps_fit_stats*>(carve(sbytes));
  double* dw = reinterpret_cast<double*>(carve(wbytes));
  if (!dual)
    cudaMemcpyAsync(djac, host_progs.data() + 1, sizeof(LmProgram) * np, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(df, features, fbytes, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(dt, t, tbytes, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(dp, params_inout, pbytes, cudaMemcpyHostToDevice, c->stream);
  LmArgs a{host_progs[0], djac, np, nf, nr, nbatch, df, dt, dp, ds, dw, *opts, equilibrate & 1,
           (equilibrate & 2) ? 0 : 1, (equilibrate & 4) ? 1 : 0, (equilibrate & 8) ? 1 : 0};
  lm_batched_kernel<<<nbatch, kLmThreads, 0, c->stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "LM launch failed: %s", cudaGetErrorString(e));
  cudaMemcpyAsync(params_inout, dp, pbytes, cudaMemcpyDeviceToHost, c->stream);
  cudaMemcpyAsync(stats, ds, sbytes, cudaMemcpyDeviceToHost, c->stream);
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "LM failed: %s", cudaGetErrorString(e));
  return PS_OK;
}

extern "C" int ps_fit_lm_batched(ps_ctx* ctx, const ps_bytecode* model, const ps_bytecode* jac,
                                 int np, int nf, const double* features, const double* t, int nr,
                                 int nbatch, const ps_fit_opts* opts, double* params_inout,
                                 ps_fit_stats* stats) {
  return ps_fit_lm_batched_ex(ctx, model, jac, np, nf, features, t, nr, nbatch, opts, 0,
                              params_inout, stats);
}
