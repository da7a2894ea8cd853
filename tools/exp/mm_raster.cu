// Experiment: CTA raster order of the 16x16 noPF/PF matmul (and the b-column
// work-removed kernel) vs DRAM re-reads at n = 4096/8192. Grid remap only:
// every CTA still computes its own 16x16 work-group, bitwise the same.
#include <cstdio>
#include <cstring>
#include <vector>
#include "../../paper_1904_09538_b200/csrc/cuda/suite_kernels.cuh"
using namespace ps;

// group-M raster: GM block rows per group, column-major inside a group
__device__ __forceinline__ void raster(int GM, int nb, int& bx, int& by) {
  const int id = blockIdx.y * gridDim.x + blockIdx.x;
  if (GM <= 0) { bx = blockIdx.x; by = blockIdx.y; return; }
  const int per_group = GM * nb;
  const int g = id / per_group, r = id % per_group;
  const int rows = min(GM, nb - g * GM);
  by = g * GM + r % rows;
  bx = r / rows;
}

__global__ void __launch_bounds__(256) nopf_r(const float* __restrict__ a, const float* __restrict__ b,
                                              float* __restrict__ c, int n, int GM) {
  int bx, by;
  raster(GM, n / 16, bx, by);
  const int i = by * 16 + threadIdx.y, j = bx * 16 + threadIdx.x;
  const float4* arow4 = reinterpret_cast<const float4*>(a + (int64_t)i * n);
  const float* bcol = b + j;
  const int64_t n64 = n;
  float acc = 0.f;
  for (int k8 = 0; k8 < n / 8; ++k8) {
    const float4 a0 = __ldg(arow4 + 2 * k8), a1 = __ldg(arow4 + 2 * k8 + 1);
    const float* bk = bcol + 8 * (int64_t)k8 * n64;
    float bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) bv[q] = __ldg(bk + q * n64);
    acc = __fmaf_rn(a0.x, bv[0], acc); acc = __fmaf_rn(a0.y, bv[1], acc);
    acc = __fmaf_rn(a0.z, bv[2], acc); acc = __fmaf_rn(a0.w, bv[3], acc);
    acc = __fmaf_rn(a1.x, bv[4], acc); acc = __fmaf_rn(a1.y, bv[5], acc);
    acc = __fmaf_rn(a1.z, bv[6], acc); acc = __fmaf_rn(a1.w, bv[7], acc);
  }
  c[(int64_t)i * n + j] = acc;
}

template <int GM>
__global__ void __launch_bounds__(256) nopf_p(const float* __restrict__ a,
                                              const float* __restrict__ b, float* __restrict__ c,
                                              int n, int tile) {
  int bx, by;
  raster(GM, n / 16, bx, by);
  const int i = by * tile + threadIdx.y;
  const int j = bx * tile + threadIdx.x;
  const float* arow = a + (int64_t)i * n;
  const float* bcol = b + j;
  float acc = 0.f;
  const float4* arow4 = reinterpret_cast<const float4*>(arow);
  const int64_t n64 = n;
  for (int k8 = 0; k8 < n / 8; ++k8) {
    const float4 a0 = __ldg(arow4 + 2 * k8), a1 = __ldg(arow4 + 2 * k8 + 1);
    const float* bk = bcol + 8 * (int64_t)k8 * n64;
    float bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) bv[q] = __ldg(bk + q * n64);
    acc = fma_t(a0.x, bv[0], acc);
    acc = fma_t(a0.y, bv[1], acc);
    acc = fma_t(a0.z, bv[2], acc);
    acc = fma_t(a0.w, bv[3], acc);
    acc = fma_t(a1.x, bv[4], acc);
    acc = fma_t(a1.y, bv[5], acc);
    acc = fma_t(a1.z, bv[6], acc);
    acc = fma_t(a1.w, bv[7], acc);
  }
  c[(int64_t)i * n + j] = acc;
}

__global__ void __launch_bounds__(256) pf_r(const float* __restrict__ a, const float* __restrict__ b,
                                            float* __restrict__ c, int n, int GM) {
  __shared__ __align__(16) float af[16][16];
  __shared__ float bf[16][16];
  int bx, by;
  raster(GM, n / 16, bx, by);
  const int ti = threadIdx.y, tj = threadIdx.x;
  const int row = by * 16 + ti, col = bx * 16 + tj;
  float acc = 0.f;
  for (int kt = 0; kt < n / 16; ++kt) {
    bar_sync();
    af[ti][tj] = a[(int64_t)row * n + kt * 16 + tj];
    bf[ti][tj] = b[(int64_t)(kt * 16 + ti) * n + col];
    bar_sync();
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const float4 av = *reinterpret_cast<const float4*>(&af[ti][4 * k4]);
      acc = __fmaf_rn(av.x, bf[4 * k4][tj], acc);
      acc = __fmaf_rn(av.y, bf[4 * k4 + 1][tj], acc);
      acc = __fmaf_rn(av.z, bf[4 * k4 + 2][tj], acc);
      acc = __fmaf_rn(av.w, bf[4 * k4 + 3][tj], acc);
    }
  }
  c[(int64_t)row * n + col] = acc;
}

__global__ void __launch_bounds__(256) rmb_r(const float* __restrict__ b, float* __restrict__ dest, int n, int GM) {
  int bx, by;
  raster(GM, n / 16, bx, by);
  const int row = by * 16 + threadIdx.y, col = bx * 16 + threadIdx.x;
  const float* bcol = b + col;
  const int64_t n64 = n;
  float acc = 0.f;
  for (int k8 = 0; k8 < n / 8; ++k8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(bcol + (8 * (int64_t)k8 + q) * n64);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __fadd_rn(acc, v[q]);
  }
  dest[(int64_t)row * n + col] = acc;
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;  // for ncu: run one GM once
  for (int n : {4096, 8192}) {
    size_t N = (size_t)n * n;
    std::vector<float> h(N);
    for (size_t x = 0; x < N; ++x) h[x] = (float)((x * 2654435761u) % 17);
    float *a, *b, *c, *c0;
    cudaMalloc(&a, N * 4); cudaMalloc(&b, N * 4); cudaMalloc(&c, N * 4); cudaMalloc(&c0, N * 4);
    cudaMemcpy(a, h.data(), N * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h.data(), N * 4, cudaMemcpyHostToDevice);
    dim3 grid(n / 16, n / 16), block(16, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](auto f, int reps) {
      f(); cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) f();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / reps;
    };
    if (only >= 0) {
      nopf_r<<<grid, block>>>(a, b, c, n, only); rmb_r<<<grid, block>>>(b, c, n, only);
      cudaDeviceSynchronize(); continue;
    }
    nopf_r<<<grid, block>>>(a, b, c0, n, 0);
    std::vector<float> r0(N), r1(N);
    cudaMemcpy(r0.data(), c0, N * 4, cudaMemcpyDeviceToHost);
    int reps = n == 8192 ? 3 : 10;
    {
      float tp0 = time([&] { matmul_nopf<float><<<grid, block>>>(a, b, c, n, 16, 0); }, reps);
      float tp1 = time([&] { matmul_pf<float, 16><<<grid, block>>>(a, b, c, n); }, reps);
      printf("n %d product noPF %.3f ms  PF %.3f ms\n", n, tp0, tp1);
      float g0 = time([&] { nopf_p<0><<<grid, block>>>(a, b, c, n, 16); }, reps);
      float g64 = time([&] { nopf_p<64><<<grid, block>>>(a, b, c, n, 16); }, reps);
      float g128 = time([&] { nopf_p<128><<<grid, block>>>(a, b, c, n, 16); }, reps);
      float g256 = time([&] { nopf_p<256><<<grid, block>>>(a, b, c, n, 16); }, reps);
      printf("n %d product-style raster GM0 %.3f  GM64 %.3f  GM128 %.3f  GM256 %.3f ms\n", n, g0, g64, g128, g256);
      // group heights dividing the SM count (148 = 4 x 37): CTAs s, s+148, ...
      // of a wave share a block row (and its a rows in L1) when CTAs are
      // dealt to SMs in id order, while each group streams b from L2 once
      float g37 = time([&] { nopf_p<37><<<grid, block>>>(a, b, c, n, 16); }, reps);
      float g74 = time([&] { nopf_p<74><<<grid, block>>>(a, b, c, n, 16); }, reps);
      float g148 = time([&] { nopf_p<148><<<grid, block>>>(a, b, c, n, 16); }, reps);
      printf("n %d product-style raster GM37 %.3f  GM74 %.3f  GM148 %.3f ms\n", n, g37, g74, g148);
    }
    for (int GM : {0, 37, 74, 128, 148}) {
      float tn = time([&] { nopf_r<<<grid, block>>>(a, b, c, n, GM); }, reps);
      cudaMemcpy(r1.data(), c, N * 4, cudaMemcpyDeviceToHost);
      bool same = memcmp(r0.data(), r1.data(), N * 4) == 0;
      float tp = time([&] { pf_r<<<grid, block>>>(a, b, c, n, GM); }, reps);
      float tr = time([&] { rmb_r<<<grid, block>>>(b, c, n, GM); }, reps);
      printf("n %d GM %2d  noPF %.3f ms (%s)  PF %.3f ms  rm-b %.3f ms  %s\n", n, GM, tn, same ? "same" : "DIFF", tp, tr,
             cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(a); cudaFree(b); cudaFree(c); cudaFree(c0);
  }
}
