// Experiment: the DG dmPF u-row loads. A work-item reads its u row k (pitch
// Np*4 B) one 64-byte tile at a time; the 16 k of a warp are one pitch apart.
// When the pitch is a multiple of 128 B every tile segment of a warp lies in
// the same half of its cache line and the 32-byte loads of one instruction
// reach only 2 (of 4) sector offsets: dmPF runs ~1.35x slower per flop at
// Np = 32/64/96/128 than at Np = 16/48 (odd multiple of 64 B: 4 offsets),
// which the count features cannot express. Variants timed here (nel = 1e6):
//   A  current realisation (dg_kernels.cuh dg_dmpf<false>)
//   B  u loads with L1::no_allocate (served from L2, no L1 bank grouping)
//   C  tile pairs: each lane loads its 128-byte two-tile segment as four
//      32-byte chunks in lane-rotated order (4 offsets at every pitch), the
//      second tile's half held across the barrier; selects undo the rotation
//   D  tile pairs without rotation (4 loads in flight, same offset per instr)
// Every variant is checked bitwise against A.
#include <cstdio>
#include <vector>

#include "../../paper_1904_09538_b200/csrc/cuda/dg_kernels.cuh"
using namespace ps;

__device__ __forceinline__ f8 ldg256_na(const float* p) {
  f8 r;
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
        "=f"(r.v[6]), "=f"(r.v[7])
      : "l"(p));
  return r;
}

__global__ void __launch_bounds__(256) dmpf_B(const float* __restrict__ dm, const float* __restrict__ u,
                                              float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    for (int jo = 0; jo < d.np / 16; ++jo) {
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      const float* ur = u + k * d.np + jo * 16;
      const f8 b0 = ldg256_na(ur), b1 = ldg256_na(ur + 8);
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 a = *reinterpret_cast<const float4*>(&dmf[ly][4 * j4]);
        const f8& b = j4 < 2 ? b0 : b1;
        const int o = 4 * (j4 & 1);
        acc = __fmaf_rn(a.x, b.v[o], acc);
        acc = __fmaf_rn(a.y, b.v[o + 1], acc);
        acc = __fmaf_rn(a.z, b.v[o + 2], acc);
        acc = __fmaf_rn(a.w, b.v[o + 3], acc);
      }
    }
    res[dg_res_idx(false, d, m, k, i0 + ly)] = acc;
  }
}

template <bool ROT>
__global__ void __launch_bounds__(256) dmpf_CD(const float* __restrict__ dm, const float* __restrict__ u,
                                               float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  const int r = ROT ? (lx & 3) : 0;
  const int njo = d.np / 16;
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    f8 c[4];
    for (int jo = 0; jo < njo; ++jo) {
      if ((jo & 1) == 0) {
        const float* ur = u + k * d.np + jo * 16;
        if (jo + 1 < njo) {
          f8 x[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) x[t] = ldg256(ur + 8 * ((t + r) & 3));
#pragma unroll
          for (int q = 0; q < 4; ++q)  // chunk q sits in x[(q - r) & 3]
#pragma unroll
            for (int e = 0; e < 8; ++e)
              c[q].v[e] = r == 0 ? x[q].v[e] : r == 1 ? x[(q + 3) & 3].v[e]
                          : r == 2 ? x[(q + 2) & 3].v[e] : x[(q + 1) & 3].v[e];
        } else {
          c[0] = ldg256(ur);
          c[1] = ldg256(ur + 8);
        }
      }
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      const f8& b0 = (jo & 1) ? c[2] : c[0];
      const f8& b1 = (jo & 1) ? c[3] : c[1];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 a = *reinterpret_cast<const float4*>(&dmf[ly][4 * j4]);
        const f8& b = j4 < 2 ? b0 : b1;
        const int o = 4 * (j4 & 1);
        acc = __fmaf_rn(a.x, b.v[o], acc);
        acc = __fmaf_rn(a.y, b.v[o + 1], acc);
        acc = __fmaf_rn(a.z, b.v[o + 2], acc);
        acc = __fmaf_rn(a.w, b.v[o + 3], acc);
      }
    }
    res[dg_res_idx(false, d, m, k, i0 + ly)] = acc;
  }
}

int main() {
  const int64_t nel = 1000000;
  const int nmat = 3;
  for (int np : {16, 32, 48, 64, 96, 128}) {
    DgDims d{nel, np, nmat};
    const size_t nu = nel * np, ndm = (size_t)nmat * np * np, nres = (size_t)nmat * nel * np;
    std::vector<float> hu(nu), hdm(ndm);
    for (size_t i = 0; i < nu; ++i) hu[i] = (float)((i * 2654435761u) % 17) - 8.f;
    for (size_t i = 0; i < ndm; ++i) hdm[i] = (float)((i * 40503u) % 13) - 6.f;
    float *du, *ddm, *r0, *r1;
    cudaMalloc(&du, nu * 4);
    cudaMalloc(&ddm, ndm * 4);
    cudaMalloc(&r0, nres * 4);
    cudaMalloc(&r1, nres * 4);
    cudaMemcpy(du, hu.data(), nu * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ddm, hdm.data(), ndm * 4, cudaMemcpyHostToDevice);
    dim3 grid(nel / 16, np / 16), block(16, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> a(nres), b(nres);
    auto run = [&](int v, float* out) {
      if (v == 0) dg_dmpf<false><<<grid, block>>>(ddm, du, out, d);
      if (v == 1) dmpf_B<<<grid, block>>>(ddm, du, out, d);
      if (v == 2) dmpf_CD<true><<<grid, block>>>(ddm, du, out, d);
      if (v == 3) dmpf_CD<false><<<grid, block>>>(ddm, du, out, d);
    };
    printf("Np %3d:", np);
    for (int v = 0; v < 4; ++v) {
      float* out = v == 0 ? r0 : r1;
      for (int w = 0; w < 3; ++w) run(v, out);
      cudaEventRecord(e0);
      for (int t = 0; t < 10; ++t) run(v, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      bool same = true;
      if (v) {
        cudaMemcpy(a.data(), r0, nres * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), r1, nres * 4, cudaMemcpyDeviceToHost);
        same = memcmp(a.data(), b.data(), nres * 4) == 0;
      }
      const double tf = 2.0 * nmat * nel * np * np / (ms * 1e-3) / 1e12;
      printf("  %c %8.1f us %5.2f TF/s%s", 'A' + v, ms * 1e3, tf, same ? "" : " MISMATCH");
    }
    printf("\n");
    cudaFree(du);
    cudaFree(ddm);
    cudaFree(r0);
    cudaFree(r1);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
