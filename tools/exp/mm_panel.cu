// Experiment: PANEL raster of the 16x16 noPF/PF matmul and the b-column
// work-removed kernel — the grid walked row-major inside panels of W block
// columns (co-resident CTAs keep sharing a block row's a rows in L1, as in
// the default order, while a wave's b working set shrinks from all of b to W
// block columns). Grid remap only: every CTA computes its own work-group.
// (tools/exp/mm_raster.cu tried column-major group-M rasters: slower.)
#include <cstdio>
#include <cstring>
#include <vector>
#include "../../paper_1904_09538_b200/csrc/cuda/suite_kernels.cuh"
using namespace ps;

__device__ __forceinline__ void panel(int W, int nb, int& bx, int& by) {
  const int id = blockIdx.y * gridDim.x + blockIdx.x;
  if (W <= 0) { bx = blockIdx.x; by = blockIdx.y; return; }
  const int per = W * nb, p = id / per, r = id % per;
  const int w = min(W, nb - p * W);
  by = r / w;
  bx = p * W + r % w;
}

__global__ void __launch_bounds__(256) nopf_w(const float* __restrict__ a, const float* __restrict__ b,
                                              float* __restrict__ c, int n, int W) {
  int bx, by;
  panel(W, n / 16, bx, by);
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
    acc = fma_t(a0.x, bv[0], acc); acc = fma_t(a0.y, bv[1], acc);
    acc = fma_t(a0.z, bv[2], acc); acc = fma_t(a0.w, bv[3], acc);
    acc = fma_t(a1.x, bv[4], acc); acc = fma_t(a1.y, bv[5], acc);
    acc = fma_t(a1.z, bv[6], acc); acc = fma_t(a1.w, bv[7], acc);
  }
  c[(int64_t)i * n + j] = acc;
}

__global__ void __launch_bounds__(256) pf_w(const float* __restrict__ a, const float* __restrict__ b,
                                            float* __restrict__ c, int n, int W) {
  __shared__ __align__(16) float af[16][16];
  __shared__ float bf[16][16];
  int bx, by;
  panel(W, n / 16, bx, by);
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

__global__ void __launch_bounds__(256) rmb_w(const float* __restrict__ b, float* __restrict__ dest, int n, int W) {
  int bx, by;
  panel(W, n / 16, bx, by);
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

int main() {
  for (int n : {2048, 4096, 8192}) {
    size_t N = (size_t)n * n;
    std::vector<float> h(N);
    for (size_t x = 0; x < N; ++x) h[x] = (float)((x * 2654435761u) % 17);
    float *a, *b, *c;
    cudaMalloc(&a, N * 4); cudaMalloc(&b, N * 4); cudaMalloc(&c, N * 4);
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
    const int reps = n == 8192 ? 3 : 10;
    std::vector<float> r0(N), r1(N);
    nopf_w<<<grid, block>>>(a, b, c, n, 0);
    cudaMemcpy(r0.data(), c, N * 4, cudaMemcpyDeviceToHost);
    for (int W : {0, 16, 32, 64, 128, 256}) {
      if (W >= n / 16) continue;
      float tn = time([&] { nopf_w<<<grid, block>>>(a, b, c, n, W); }, reps);
      cudaMemcpy(r1.data(), c, N * 4, cudaMemcpyDeviceToHost);
      const bool same = memcmp(r0.data(), r1.data(), N * 4) == 0;
      float tp = time([&] { pf_w<<<grid, block>>>(a, b, c, n, W); }, reps);
      float tr = time([&] { rmb_w<<<grid, block>>>(b, c, n, W); }, reps);
      printf("n %d W %3d  noPF %8.3f ms (%s)  PF %8.3f ms  rm-b %8.3f ms\\n", n, W, tn, same ? "same" : "DIFF", tp, tr);
    }
    cudaFree(a); cudaFree(b); cudaFree(c);
  }
}
