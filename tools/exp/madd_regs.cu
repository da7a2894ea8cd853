// Experiment: flops_madd (SHOC chain v_j = fma(v_{j+27}, v_{j+21}, v_j)) rate
// vs operand order / unroll shape; all variants compute identical bits.
#include <cstdio>
#include <cstring>
#include <vector>

template <int VAR>
__global__ void __launch_bounds__(256) madd_k(float* out, int m, float base, float step) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(base, __fmul_rn(step, (float)j));
  for (int t = 0; t < m; ++t) {
#pragma unroll
    for (int u = 0; u < 64; ++u) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (VAR == 0) v[j] = __fmaf_rn(v[(j + 27) & 31], v[(j + 21) & 31], v[j]);
        else v[j] = __fmaf_rn(v[(j + 21) & 31], v[(j + 27) & 31], v[j]);  // commuted product
      }
    }
  }
  float r = v[0];
#pragma unroll
  for (int j = 1; j < 32; ++j) r = __fadd_rn(r, v[j]);
  out[blockIdx.x * 256 + threadIdx.x] = r;
}

// independent FFMAs with three distinct registers each (no operand shared with
// the previous instruction) vs with two operands shared (reuse cache)
template <int SHARE>
__global__ void __launch_bounds__(256) ffma_k(float* out, int m, float base, float step) {
  float a[16], b[16], c[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    a[j] = base + step * j;
    b[j] = base - step * j;
    c[j] = step * (j + 1);
  }
  for (int t = 0; t < m * 128; ++t) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (SHARE) a[j] = __fmaf_rn(b[0], c[0], a[j]);
      else a[j] = __fmaf_rn(b[j], c[j], a[j]);
    }
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) r += a[j] + b[j] + c[j];
  out[blockIdx.x * 256 + threadIdx.x] = r;
}

int main() {
  const int blocks = 8192, m = 64;
  float* o;
  cudaMalloc(&o, blocks * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> r0(blocks * 256), r1(blocks * 256);
  auto run = [&](auto k, std::vector<float>& r) {
    k<<<blocks, 256>>>(o, m, 0.5f, 0.015625f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) k<<<blocks, 256>>>(o, m, 0.5f, 0.015625f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost);
    const double ffma = 2048.0 * m * blocks * 256;
    return ffma / (ms / 5 * 1e-3) / 1e12;
  };
  double t0 = run(madd_k<0>, r0), t1 = run(madd_k<1>, r1);
  const double f3 = run(ffma_k<0>, r0), f2 = run(ffma_k<1>, r1);
  printf("indep-3reg %.2f  shared-operands %.2f Tffma/s (x m*128*16 vs 2048 m: same count)\n", f3, f2);
  printf("var0 %.2f Tffma/s  var1 %.2f Tffma/s  same=%d  peak %.2f\n", t0, t1,
         memcmp(r0.data(), r1.data(), r0.size() * 4) == 0, 148 * 128 * 1.965e9 / 1e12);
}
