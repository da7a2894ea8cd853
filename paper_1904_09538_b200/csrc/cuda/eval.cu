// K18: batched prediction and ranking over a variant space.
//
// One thread per parameter point. For every variant the model's count
// features are evaluated exactly (128-bit integer polynomial / common
// denominator, the reference's exact-rational evaluation, features.cpp:342-415),
// converted to double, and the calibrated model is evaluated by a bytecode
// interpreter (eval_model, model.cpp:409-419). Per application group the
// winner is the strict '<' first minimum in variant order
// (tools/perfseer.cpp:458-467). Points are read once (32 B) and predictions
// written once (8 B per variant): the kernel is integer/FP64 compute bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "libm_glibc.cuh"
#include "runtime_internal.h"

namespace ps {


struct DevTables {
  FlatTables t;  // pointers are device pointers
};

// The model's straight-line register program (common subexpressions once,
// ps_model.cpp compile_program): the same IEEE operations on the same
// operands as eval_model's tree walk, so the same bits.
__device__ double eval_model_prog(const uint32_t* __restrict__ insns, int n, const double* __restrict__ consts,
                                  const double* __restrict__ p, const double* f, int out) {
  double s[kEvalMaxRegs];
  for (int i = 0; i < n; ++i) {
    const uint32_t w0 = __ldg(insns + 2 * i), w1 = __ldg(insns + 2 * i + 1);
    const int op = int(w0 >> 16), d = int(w0 & 0xffff), a = int(w1 >> 16), b = int(w1 & 0xffff);
    double v;
    switch (op) {
      case PS_BC_NUM: v = __ldg(consts + a); break;
      case PS_BC_PARAM: v = __ldg(p + a); break;
      case PS_BC_FEAT: v = f[a]; break;
      case PS_BC_TANH: v = glibc_tanh(s[a]); break;
      case PS_BC_ADD: v = __dadd_rn(s[a], s[b]); break;
      case PS_BC_SUB: v = __dsub_rn(s[a], s[b]); break;
      case PS_BC_MUL: v = __dmul_rn(s[a], s[b]); break;
      default: v = __ddiv_rn(s[a], s[b]);
    }
    s[d] = v;
  }
  return s[out];
}

__global__ void __launch_bounds__(128) eval_points_kernel(FlatTables t, const int64_t* __restrict__ points,
                                                          int64_t npts, double* __restrict__ pred,
                                                          uint8_t* __restrict__ argmin) {
  for (int64_t pt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pt < npts;
       pt += (int64_t)gridDim.x * blockDim.x) {
    int64_t x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = points[pt * 4 + c];
    double best[kEvalMaxGroups];
    int besti[kEvalMaxGroups];
    for (int g = 0; g < t.ngroups; ++g) besti[g] = -1;
    for (int v = 0; v < t.nvar; ++v) {
      const int m = t.var_model[v];
      const int nf = t.model_nf[m];
      double f[kEvalMaxFeat];
      for (int j = 0; j < nf; ++j) {
        const int slot = t.var_feat_base[v] + j;
        __int128 acc = 0;
        for (int k = t.feat_begin[slot]; k < t.feat_end[slot]; ++k) {
          __int128 term = t.term_coef[k];
          for (int c = 0; c < 4; ++c)
            for (int e = 0; e < t.term_exp[k * 4 + c]; ++e) term *= x[c];
          acc += term;
        }
        const long long den = t.feat_den[slot];
        const __int128 lim = (__int128)1 << 53;
        if (den == 1) {
          f[j] = (double)acc;
        } else if (acc < lim && acc > -lim && den < (1LL << 53)) {
          // both exact doubles: one correctly rounded division of the same
          // real quotient the lowest-terms form divides, so the same bits
          f[j] = (double)(long long)acc / (double)den;
        } else {  // Rational -> double as the host does: lowest terms, one division
          __int128 a = acc < 0 ? -acc : acc, b = den;
          while (b) {
            const __int128 r = a % b;
            a = b;
            b = r;
          }
          f[j] = (a > 1) ? (double)(acc / a) / (double)(den / (long long)a)
                         : (double)acc / (double)den;
        }
      }
      const double y = eval_model_prog(t.insns + 2 * (size_t)t.model_insn_begin[m],
                                       t.model_insn_begin[m + 1] - t.model_insn_begin[m],
                                       t.consts + t.model_const_begin[m], t.params + t.model_param_begin[m], f,
                                       t.model_out[m]);
      pred[pt * t.nvar + v] = y;
      const int g = t.var_group[v];
      if (besti[g] < 0 || y < best[g]) {
        best[g] = y;
        besti[g] = v;
      }
    }
    for (int g = 0; g < t.ngroups; ++g) argmin[pt * t.ngroups + g] = (uint8_t)besti[g];
  }
}

int eval_tables_gpu(Ctx* c, const FlatTables& h, const int64_t* points, int64_t npts, double* pred,
                    uint8_t* argmin, double* kernel_seconds, void* jit_kernel) {
  TraceRange trace(jit_kernel ? "K18 eval (specialised)" : "K18 eval (interpreter)");
  if (h.ngroups > kEvalMaxGroups) return set_error(PS_ERR_ARG, "at most %d application groups", kEvalMaxGroups);
  if (h.nvar > kEvalMaxVariants) return set_error(PS_ERR_ARG, "at most %d variants", kEvalMaxVariants);
  for (int m = 0; m < h.nmodels; ++m) {
    if (h.model_nf[m] > kEvalMaxFeat) return set_error(PS_ERR_ARG, "model with more than %d features", kEvalMaxFeat);
    if (h.model_regs[m] > kEvalMaxRegs)
      return set_error(PS_ERR_ARG, "model %d: program needs %d registers (device evaluator: %d)", m,
                       h.model_regs[m], kEvalMaxRegs);
  }
  if (cudaSetDevice(c->device) != cudaSuccess) return set_error(PS_ERR_CUDA, "cudaSetDevice failed");
  // Pack every table array into one device allocation.
  struct Part {
    const void* src;
    size_t bytes;
    void** dst;
  };
  FlatTables d = h;
  std::vector<Part> parts;
  if (jit_kernel) {
    // the specialised kernel carries the tables in its code: only the
    // fitted parameters travel
    parts = {{h.params, sizeof(double) * h.model_param_begin[h.nmodels], (void**)&d.params}};
  } else parts = {
      {h.var_group, sizeof(int32_t) * h.nvar, (void**)&d.var_group},
      {h.var_model, sizeof(int32_t) * h.nvar, (void**)&d.var_model},
      {h.var_feat_base, sizeof(int32_t) * h.nvar, (void**)&d.var_feat_base},
      {h.feat_begin, sizeof(int32_t) * h.nslots, (void**)&d.feat_begin},
      {h.feat_end, sizeof(int32_t) * h.nslots, (void**)&d.feat_end},
      {h.feat_den, sizeof(int64_t) * h.nslots, (void**)&d.feat_den},
      {h.term_coef, sizeof(int64_t) * h.nterms, (void**)&d.term_coef},
      {h.term_exp, (size_t)4 * h.nterms, (void**)&d.term_exp},
      {h.model_nf, sizeof(int32_t) * h.nmodels, (void**)&d.model_nf},
      {h.model_insn_begin, sizeof(int32_t) * (h.nmodels + 1), (void**)&d.model_insn_begin},
      {h.insns, sizeof(uint32_t) * 2 * (size_t)h.model_insn_begin[h.nmodels], (void**)&d.insns},
      {h.model_out, sizeof(int32_t) * h.nmodels, (void**)&d.model_out},
      {h.model_regs, sizeof(int32_t) * h.nmodels, (void**)&d.model_regs},
      {h.model_const_begin, sizeof(int32_t) * (h.nmodels + 1), (void**)&d.model_const_begin},
      {h.consts, sizeof(double) * std::max(1, h.model_const_begin[h.nmodels]), (void**)&d.consts},
      {h.model_param_begin, sizeof(int32_t) * (h.nmodels + 1), (void**)&d.model_param_begin},
      {h.params, sizeof(double) * h.model_param_begin[h.nmodels], (void**)&d.params},
  };
  size_t total = 0;
  for (auto& p : parts) total += (p.bytes + 255) & ~size_t(255);
  const size_t pts_bytes = sizeof(int64_t) * 4 * (size_t)npts;
  const size_t pred_bytes = sizeof(double) * (size_t)npts * h.nvar;
  const size_t arg_bytes = (size_t)npts * h.ngroups;
  int rc = c->ensure(c->scratch[1], total + pts_bytes + pred_bytes + arg_bytes + 1024);
  if (rc) return rc;
  char* base = static_cast<char*>(c->scratch[1].ptr);
  size_t off = 0;
  for (auto& p : parts) {
    *p.dst = base + off;
    if (p.bytes && cudaMemcpyAsync(base + off, p.src, p.bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      return set_error(PS_ERR_CUDA, "table upload failed");
    off += (p.bytes + 255) & ~size_t(255);
  }
  int64_t* dpts = reinterpret_cast<int64_t*>(base + off);
  off += (pts_bytes + 255) & ~size_t(255);
  double* dpred = reinterpret_cast<double*>(base + off);
  off += (pred_bytes + 255) & ~size_t(255);
  uint8_t* darg = reinterpret_cast<uint8_t*>(base + off);
  const int threads = 128;
  const int64_t wave = (int64_t)c->sm_count * threads * 8;  // points one chunk launch covers
  // Chunked pipeline: the points of chunk i+1 copy in (h2d stream) while
  // chunk i evaluates (context stream) and chunk i-1's predictions copy out
  // (d2h stream) — the two copy engines and the SMs overlap, so an
  // end-to-end call costs about max(kernel, copy-out) instead of their sum.
  // Each chunk is a whole number of 8-CTA-per-SM waves; kernel_seconds is the
  // sum of the chunk kernels' own event times.
  const int64_t chunk = npts >= 3 * wave ? std::max<int64_t>(wave, (npts / 8 + wave - 1) / wave * wave) : npts;
  const int nchunks = (int)((npts + chunk - 1) / chunk);
  if ((rc = events(c, 1 + 3 * nchunks))) return rc;
  if (nchunks > 1) {
    if (!c->h2d_stream && cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking) != cudaSuccess)
      return set_error(PS_ERR_CUDA, "stream creation failed");
    if (!c->d2h_stream && cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking) != cudaSuccess)
      return set_error(PS_ERR_CUDA, "stream creation failed");
    // the copy streams start after everything already on the context stream
    cudaEventRecord(c->ev[0], c->stream);
    cudaStreamWaitEvent(c->h2d_stream, c->ev[0], 0);
    cudaStreamWaitEvent(c->d2h_stream, c->ev[0], 0);
  }
  cudaStream_t in_st = nchunks > 1 ? c->h2d_stream : c->stream;
  cudaStream_t out_st = nchunks > 1 ? c->d2h_stream : c->stream;
  for (int i = 0; i < nchunks; ++i) {
    const int64_t lo = (int64_t)i * chunk, n = std::min<int64_t>(chunk, npts - lo);
    cudaEvent_t in_done = c->ev[1 + 3 * i], k0 = c->ev[2 + 3 * i], k1 = c->ev[3 + 3 * i];
    cudaMemcpyAsync(dpts + 4 * lo, points + 4 * lo, sizeof(int64_t) * 4 * (size_t)n, cudaMemcpyHostToDevice,
                    in_st);
    if (nchunks > 1) {
      cudaEventRecord(in_done, in_st);
      cudaStreamWaitEvent(c->stream, in_done, 0);
    }
    const unsigned blocks =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)c->sm_count * 16));
    cudaEventRecord(k0, c->stream);
    if (jit_kernel) {  // the tables compiled into kernels (eval_jit.cu)
      const JitKernels* jk = static_cast<const JitKernels*>(jit_kernel);
      const int64_t* kp = dpts + 4 * lo;
      double* kpred = dpred + (size_t)lo * h.nvar;
      uint8_t* karg = darg + (size_t)lo * h.ngroups;
      const double* kparams = d.params;
      int64_t kn = n;
      const int64_t per_cta = (int64_t)threads * jk->lanes;
      const unsigned bx = std::max(1u, (unsigned)std::min<int64_t>((n + per_cta - 1) / per_cta,
                                                                    (int64_t)c->sm_count * 16));
      void* pargs[] = {&kp, &kn, &kpred, &kparams};
      cudaLaunchKernel(reinterpret_cast<const void*>(jk->predict), dim3(bx, (unsigned)h.nvar), dim3(threads),
                       pargs, 0, c->stream);
      void* rargs[] = {&kpred, &kn, &karg};
      cudaLaunchKernel(reinterpret_cast<const void*>(jk->rank), dim3(blocks), dim3(threads), rargs, 0, c->stream);
    } else {
      eval_points_kernel<<<blocks, threads, 0, c->stream>>>(d, dpts + 4 * lo, n, dpred + (size_t)lo * h.nvar,
                                                            darg + (size_t)lo * h.ngroups);
    }
    cudaEventRecord(k1, c->stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "eval launch failed: %s", cudaGetErrorString(e));
    if (nchunks > 1) cudaStreamWaitEvent(out_st, k1, 0);
    cudaMemcpyAsync(pred + (size_t)lo * h.nvar, dpred + (size_t)lo * h.nvar, sizeof(double) * (size_t)n * h.nvar,
                    cudaMemcpyDeviceToHost, out_st);
    cudaMemcpyAsync(argmin + (size_t)lo * h.ngroups, darg + (size_t)lo * h.ngroups, (size_t)n * h.ngroups,
                    cudaMemcpyDeviceToHost, out_st);
  }
  cudaError_t e = cudaStreamSynchronize(out_st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && nchunks > 1) e = cudaStreamSynchronize(in_st);
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "eval failed: %s", cudaGetErrorString(e));
  double secs = 0.0;
  for (int i = 0; i < nchunks; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2 + 3 * i], c->ev[3 + 3 * i]);
    secs += ms * 1e-3;
  }
  if (kernel_seconds) *kernel_seconds = secs;
  return PS_OK;
}

}  // namespace ps
