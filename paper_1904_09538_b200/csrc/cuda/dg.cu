// Launch/IO glue for the DG kernels (dg_kernels.cuh).
#include <cstring>

#include "dg_kernels.cuh"
#include "runtime_internal.h"

namespace ps {

int dg_validate(const ps_kernel_desc* d) {
  if (d->dtype != PS_F32) return set_error(PS_ERR_ARG, "DG variants are float32");
  if (d->nel < 16 || d->nel % 16 != 0)
    return set_error(PS_ERR_ARG, "DG requires nelements to be a multiple of 16");
  if (d->np < 16 || d->np % 16 != 0)
    return set_error(PS_ERR_ARG, "DG requires nunit_nodes to be a multiple of 16 (pad)");
  if (d->nmat < 1 || d->nmat > 4) return set_error(PS_ERR_ARG, "DG supports 1..4 matrices");
  if (d->dg_variant < PS_DG_NOPF || d->dg_variant > PS_DG_DMPF_T)
    return set_error(PS_ERR_ARG, "unknown DG variant");
  if (d->gen == PS_GEN_DG_RM && d->keep != PS_KEEP_U && d->keep != PS_KEEP_DM &&
      d->keep != PS_KEEP_RES)
    return set_error(PS_ERR_ARG, "DG rm keep must be u, dm or res");
  if (d->nel / 16 > 2147483647LL) return set_error(PS_ERR_ARG, "nelements too large");
  return PS_OK;
}

int dg_io(const ps_kernel_desc* d, ps_io_info* io) {
  const int64_t dm = d->nmat * d->np * d->np, u = d->nel * d->np, res = d->nmat * d->nel * d->np;
  const double eb = 4.0;
  auto in = [&](int64_t n) { io->input_elems[io->n_inputs++] = n; };
  auto out = [&](int64_t n) { io->output_elems[io->n_outputs++] = n; };
  if (d->gen == PS_GEN_DG || d->gen == PS_GEN_DG_TC) {
    in(dm);
    in(u);
    out(res);
    io->bytes_global = eb * (double)(dm + u + res);
    io->flops = 2.0 * (double)d->nmat * (double)d->nel * (double)d->np * (double)d->np;
    if (d->gen == PS_GEN_DG_TC)
      io->bytes_shared = 0;
    else if (d->dg_variant == PS_DG_UPF)
      io->bytes_shared = eb * ((double)u * (1.0 + (double)d->np));
    else if (d->dg_variant != PS_DG_NOPF)
      io->bytes_shared = eb * (double)d->nmat * (double)d->np * (double)d->np *
                         ((double)d->nel / 16.0) * (1.0 / 16.0 + 1.0);
    return PS_OK;
  }
  if (d->keep == PS_KEEP_RES) {
    out(res);
    io->bytes_global = eb * (double)res;
  } else {
    in(d->keep == PS_KEEP_U ? u : dm);
    out(d->np * d->nel);
    io->bytes_global = eb * (double)((d->keep == PS_KEEP_U ? u : dm) + d->np * d->nel);
  }
  return PS_OK;
}

const char* dg_input_name(const ps_kernel_desc* d, int i) {
  if (d->gen == PS_GEN_DG || d->gen == PS_GEN_DG_TC) return i == 0 ? "diff_mat" : "u";
  return d->keep == PS_KEEP_U ? "u" : "diff_mat";
}

template <int V>
static void launch_rm(const ps_kernel_desc* d, dim3 g, dim3 b, cudaStream_t st, const float* src,
                      float* dst, DgDims dims) {
  if (d->keep == PS_KEEP_U)
    dg_rm<V, 3><<<g, b, 0, st>>>(src, dst, dims);
  else if (d->keep == PS_KEEP_DM)
    dg_rm<V, 5><<<g, b, 0, st>>>(src, dst, dims);
  else
    dg_rm<V, 4><<<g, b, 0, st>>>(src, dst, dims);
}

int dg_launch(Ctx* c, const ps_kernel_desc* d) {
  DgDims dims{d->nel, (int)d->np, (int)d->nmat};
  dim3 grid((unsigned)(d->nel / 16), (unsigned)(d->np / 16)), block(16, 16);
  cudaStream_t st = c->stream;
  const float* in0 = (const float*)c->in[0].ptr;
  const float* in1 = (const float*)c->in[1].ptr;
  float* out0 = (float*)c->out[0].ptr;
  if (d->gen == PS_GEN_DG) {
    switch (d->dg_variant) {
      case PS_DG_NOPF: dg_nopf<<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
      case PS_DG_UPF:
        switch (d->nmat) {
          case 1: dg_upf<1><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
          case 2: dg_upf<2><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
          case 3: dg_upf<3><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
          default: dg_upf<4><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
        }
        break;
      case PS_DG_DMPF: dg_dmpf<false><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
      default: dg_dmpf<true><<<grid, block, 0, st>>>(in0, in1, out0, dims); break;
    }
  } else {
    switch (d->dg_variant) {
      case PS_DG_NOPF: launch_rm<0>(d, grid, block, st, in0, out0, dims); break;
      case PS_DG_UPF: launch_rm<1>(d, grid, block, st, in0, out0, dims); break;
      case PS_DG_DMPF: launch_rm<2>(d, grid, block, st, in0, out0, dims); break;
      default: launch_rm<3>(d, grid, block, st, in0, out0, dims); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(PS_ERR_CUDA, "DG launch failed: %s", cudaGetErrorString(e));
  return PS_OK;
}

}  // namespace ps
