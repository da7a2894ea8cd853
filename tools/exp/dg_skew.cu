// Experiment: DG noPF u-row loads with a per-lane skew of the (m, j8) chunk
// stream, so one warp-wide 32-byte load spreads over 4 (addr mod 128) sector
// groups instead of 1 when the row pitch is a multiple of 128 B.
#include <cstdio>
#include <vector>
#include "../../paper_1904_09538_b200/csrc/cuda/dg_kernels.cuh"
using namespace ps;

template <int UNR>
__global__ void __launch_bounds__(256) dg_nopf_skew(const float* __restrict__ dm,
                                                    const float* __restrict__ u,
                                                    float* __restrict__ res, DgDims d) {
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i = blockIdx.y * 16 + ly;
  const int nj8 = d.np / 8;
  const bool four = (nj8 & 3) == 0;
  const int s = four ? (lx & 3) : ((lx >> 1) & 1);
  const int smax = four ? 3 : 1;
  const int S = d.nmat * nj8;
  const float* urow = u + k * d.np;
  const float* dmrow = dm + (int64_t)i * d.np;
  const int64_t mstride = (int64_t)d.np * d.np;
  int m = 0, j8 = 0;
  float acc = 0.f;
  for (int t = 0; t < S + smax; ++t) {
    const int idx = t - s;
    if (idx >= 0 && idx < S) {
      const f8 a = ldg256(dmrow + 8 * j8), b = ldg256(urow + 8 * j8);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = __fmaf_rn(a.v[q], b.v[q], acc);
      if (++j8 == nj8) {
        res[((int64_t)m * d.nel + k) * d.np + i] = acc;
        acc = 0.f;
        j8 = 0;
        ++m;
        dmrow += mstride;
      }
    }
  }
}

// branch-free steady state: every lane active for t in [smax, S)
__global__ void __launch_bounds__(256) dg_nopf_skew2(const float* __restrict__ dm,
                                                     const float* __restrict__ u,
                                                     float* __restrict__ res, DgDims d) {
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i = blockIdx.y * 16 + ly;
  const int nj8 = d.np / 8;
  const bool four = (nj8 & 3) == 0;
  const int s = four ? (lx & 3) : ((lx >> 1) & 1);
  const int smax = four ? 3 : 1;
  const int S = d.nmat * nj8;
  const float* urow = u + k * d.np;
  const float* up = urow;
  const float* dmp = dm + (int64_t)i * d.np;
  const int64_t mstep = (int64_t)d.np * d.np - (d.np - 8);
  float* rp = res + k * d.np + i;
  const int64_t rstep = d.nel * d.np;
  int j8 = 0;
  float acc = 0.f;
  auto step = [&]() {
    const f8 a = ldg256(dmp), b = ldg256(up);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __fmaf_rn(a.v[q], b.v[q], acc);
    const bool wrap = j8 == nj8 - 1;
    if (wrap) *rp = acc;
    acc = wrap ? 0.f : acc;
    j8 = wrap ? 0 : j8 + 1;
    rp += wrap ? rstep : 0;
    dmp += wrap ? mstep : 8;
    up = wrap ? urow : up + 8;
  };
  // prologue: lane starts at t = s
  for (int t = 0; t < smax; ++t) if (t >= s) step();
#pragma unroll 2
  for (int t = smax; t < S; ++t) step();
  for (int t = S; t < S + smax; ++t) if (t - s < S) step();
}

// dmPF with the two 32-byte u chunks of a tile issued in lane-dependent order
template <bool SWAP>
__global__ void __launch_bounds__(256) dg_dmpf_swap(const float* __restrict__ dm,
                                                    const float* __restrict__ u,
                                                    float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  const int nj8 = d.np / 8;
  const bool sw = ((nj8 & 3) == 0) ? (lx & 1) : ((lx >> 1) & 1);
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    for (int jo = 0; jo < d.np / 16; ++jo) {
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      const float* ur = u + k * d.np + jo * 16;
      f8 x0, x1;
      if (SWAP) {
        x0 = ldg256(ur + (sw ? 8 : 0));
        x1 = ldg256(ur + (sw ? 0 : 8));
      } else {
        x0 = ldg256(ur); x1 = ldg256(ur + 8);
      }
      f8 b0, b1;
#pragma unroll
      for (int q = 0; q < 8; ++q) { b0.v[q] = (SWAP && sw) ? x1.v[q] : x0.v[q]; b1.v[q] = (SWAP && sw) ? x0.v[q] : x1.v[q]; }
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
    res[((int64_t)m * d.nel + k) * d.np + i0 + ly] = acc;
  }
}

// dmPF, 4 line offsets at pitch % 128 == 0: lanes with (lx & 2) load their u
// chunks one tile ahead (a 16-float register buffer), and lanes with (lx & 1)
// load the two chunks of a tile in reverse order.
__global__ void __launch_bounds__(256) dg_dmpf_ahead(const float* __restrict__ dm,
                                                     const float* __restrict__ u,
                                                     float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  const int nj8 = d.np / 8, njo = d.np / 16;
  const bool four = (nj8 & 3) == 0;
  const bool sw = four ? (lx & 1) : ((lx >> 1) & 1);
  const bool ahead = four && (lx & 2);
  const float* urow = u + k * d.np;
  const int o0 = sw ? 8 : 0, o1 = sw ? 0 : 8;
  f8 n0, n1;
  if (ahead) { n0 = ldg256(urow + o0); n1 = ldg256(urow + o1); }
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    for (int jo = 0; jo < njo; ++jo) {
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      const int jl = ahead ? (jo + 1 == njo ? 0 : jo + 1) : jo;
      const bool last = ahead && m == d.nmat - 1 && jo == njo - 1;
      f8 x0, x1;
      if (!last) { x0 = ldg256(urow + 16 * jl + o0); x1 = ldg256(urow + 16 * jl + o1); }
      f8 b0, b1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float c0 = ahead ? n0.v[q] : x0.v[q], c1 = ahead ? n1.v[q] : x1.v[q];
        b0.v[q] = sw ? c1 : c0;
        b1.v[q] = sw ? c0 : c1;
      }
      if (ahead) { n0 = x0; n1 = x1; }
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
    res[((int64_t)m * d.nel + k) * d.np + i0 + ly] = acc;
  }
}

// dmPF with 16-byte u loads: lane l loads the tile's four quarters starting
// at quarter ROT ? (l & 3) : 0 (4 line offsets per instruction at any pitch),
// then un-rotates them with selects so the FMAs still run in j order.
// Measured (B200, nel 1e6, Np 16..128): unrotated 16-byte loads 2.0-3.5 TF/s;
// rotated 4.6-5.9 TF/s — flatter in Np than the shipped 32-byte lane swap
// (5.3-8.0 TF/s) but slower at every Np except 64/128 (within 4%): rejected.
template <bool ROT>
__global__ void __launch_bounds__(256) dg_dmpf_rot4(const float* __restrict__ dm,
                                                    const float* __restrict__ u,
                                                    float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  const int rot = ROT ? (lx & 3) : 0;
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    for (int jo = 0; jo < d.np / 16; ++jo) {
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      const float4* ur = reinterpret_cast<const float4*>(u + k * d.np + jo * 16);
      float4 x[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) x[s] = __ldg(ur + ((s + rot) & 3));
      // x[s] holds quarter (s + rot) & 3; quarter q is x[(q - rot) & 3]
      float4 b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = (q - rot) & 3;
        const float4 lo = (s & 1) ? x[1] : x[0], hi = (s & 1) ? x[3] : x[2];
        b[q] = (s & 2) ? hi : lo;
      }
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 a = *reinterpret_cast<const float4*>(&dmf[ly][4 * j4]);
        acc = __fmaf_rn(a.x, b[j4].x, acc);
        acc = __fmaf_rn(a.y, b[j4].y, acc);
        acc = __fmaf_rn(a.z, b[j4].z, acc);
        acc = __fmaf_rn(a.w, b[j4].w, acc);
      }
    }
    res[((int64_t)m * d.nel + k) * d.np + i0 + ly] = acc;
  }
}

int main() {
  const int64_t nel = 1000000;
  const int nps[] = {16, 32, 48, 64, 96, 128};
  for (int np : nps) {
    DgDims d{nel, np, 3};
    size_t nu = nel * np, ndm = 3 * np * np, nr = 3 * nel * np;
    std::vector<float> hu(nu), hdm(ndm);
    for (size_t x = 0; x < nu; ++x) hu[x] = (float)((x * 2654435761u) % 17) - 8.f;
    for (size_t x = 0; x < ndm; ++x) hdm[x] = (float)((x * 40503u) % 13) * 0.25f;
    float *u, *dm, *r0, *r1;
    cudaMalloc(&u, nu * 4); cudaMalloc(&dm, ndm * 4); cudaMalloc(&r0, nr * 4); cudaMalloc(&r1, nr * 4);
    cudaMemcpy(u, hu.data(), nu * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, hdm.data(), ndm * 4, cudaMemcpyHostToDevice);
    dim3 grid(nel / 16, np / 16), block(16, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](auto launch) {
      for (int w = 0; w < 3; ++w) launch();
      cudaEventRecord(e0);
      for (int w = 0; w < 20; ++w) launch();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 20;
    };
    float t0 = time([&] { dg_nopf<<<grid, block>>>(dm, u, r0, d); });
    float t1 = time([&] { dg_nopf_skew<1><<<grid, block>>>(dm, u, r1, d); });
    float *r2; cudaMalloc(&r2, nr * 4);
    float t2 = time([&] { dg_nopf_skew2<<<grid, block>>>(dm, u, r2, d); });
    float t3 = time([&] { dg_dmpf<false><<<grid, block>>>(dm, u, r2, d); });
    float t4 = time([&] { dg_dmpf_swap<true><<<grid, block>>>(dm, u, r2, d); });
    std::vector<float> c(nr);
    cudaMemcpy(c.data(), r2, nr * 4, cudaMemcpyDeviceToHost);
    size_t bad2 = 0;
    dg_nopf_skew2<<<grid, block>>>(dm, u, r2, d);
    cudaMemcpy(c.data(), r2, nr * 4, cudaMemcpyDeviceToHost);
    for (size_t x = 0; x < nr; ++x) bad2 += c[x] != 0 && false;
    {
      std::vector<float> ref(nr); cudaMemcpy(ref.data(), r0, nr*4, cudaMemcpyDeviceToHost);
      for (size_t x = 0; x < nr; ++x) bad2 += memcmp(&ref[x], &c[x], 4) != 0;
      dg_dmpf_swap<true><<<grid, block>>>(dm, u, r2, d);
      cudaMemcpy(c.data(), r2, nr * 4, cudaMemcpyDeviceToHost);
      for (size_t x = 0; x < nr; ++x) bad2 += memcmp(&ref[x], &c[x], 4) != 0;
    }
    float t5 = time([&] { dg_dmpf_ahead<<<grid, block>>>(dm, u, r2, d); });
    {
      std::vector<float> ref(nr); cudaMemcpy(ref.data(), r0, nr*4, cudaMemcpyDeviceToHost);
      cudaMemcpy(c.data(), r2, nr * 4, cudaMemcpyDeviceToHost);
      for (size_t x = 0; x < nr; ++x) bad2 += memcmp(&ref[x], &c[x], 4) != 0;
    }
    double fl2 = 2.0 * 3 * nel * np * np;
    printf("np %3d  dmPF-ahead %.2f TF\n", np, fl2/t5/1e9);
    for (int v = 0; v < 2; ++v) {
      float t6 = v ? time([&] { dg_dmpf_rot4<true><<<grid, block>>>(dm, u, r2, d); })
                   : time([&] { dg_dmpf_rot4<false><<<grid, block>>>(dm, u, r2, d); });
      std::vector<float> ref(nr); cudaMemcpy(ref.data(), r0, nr*4, cudaMemcpyDeviceToHost);
      cudaMemcpy(c.data(), r2, nr * 4, cudaMemcpyDeviceToHost);
      size_t b6 = 0;
      for (size_t x = 0; x < nr; ++x) b6 += memcmp(&ref[x], &c[x], 4) != 0;
      printf("np %3d  dmPF-16B%s %.2f TF  mism %zu\n", np, v ? "-rot4" : "", fl2/t6/1e9, b6);
    }
    printf("np %3d  skew2 %.2f TF  dmPF %.2f TF  dmPF-swap %.2f TF  mism %zu\n", np, fl2/t2/1e9, fl2/t3/1e9, fl2/t4/1e9, bad2);
    cudaFree(r2);
    std::vector<float> a(nr), b(nr);
    cudaMemcpy(a.data(), r0, nr * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), r1, nr * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0; for (size_t x = 0; x < nr; ++x) bad += memcmp(&a[x], &b[x], 4) != 0;
    double fl = 2.0 * 3 * nel * np * np;
    printf("np %3d  orig %.4f ms %.2f TF   skew %.4f ms %.2f TF  mismatches %zu  err=%s\n", np, t0,
           fl / t0 / 1e9, t1, fl / t1 / 1e9, bad, cudaGetErrorString(cudaGetLastError()));
    cudaFree(u); cudaFree(dm); cudaFree(r0); cudaFree(r1);
  }
}
