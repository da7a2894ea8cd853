// Experiment: flops_madd with W work-items per thread, their SHOC updates
// interleaved (each work-item's own operation order unchanged), against the
// one-work-item realisation. Work-items get their base from separate
// runtime arguments so the compiler cannot merge their identical chains.
// Reports the FFMA rate as a fraction of 148 SMs x 128 lanes x clock.
#include <cstdio>
#include <cstring>
#include <vector>

template <int W, int BLK>
__global__ void __launch_bounds__(BLK) madd_w(float* out, int m, const float* __restrict__ bases, float step) {
  float v[W][32];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const float base = bases[w];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[w][j] = __fadd_rn(base, __fmul_rn(step, (float)j));
  }
  for (int t = 0; t < m; ++t) {
#pragma unroll
    for (int u = 0; u < 64; ++u) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
#pragma unroll
        for (int w = 0; w < W; ++w) v[w][j] = __fmaf_rn(v[w][(j + 27) & 31], v[w][(j + 21) & 31], v[w][j]);
      }
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    float r = v[w][0];
#pragma unroll
    for (int j = 1; j < 32; ++j) r = __fadd_rn(r, v[w][j]);
    out[((size_t)blockIdx.x * BLK + threadIdx.x) * W + w] = r;
  }
}

template <int W, int BLK>
void run(const char* name, float* out, const float* bases, int sms, int clk_khz) {
  const int m = 64;
  const long long wis = (1LL << 21);
  const int blocks = (int)(wis / W / BLK);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) madd_w<W, BLK><<<blocks, BLK>>>(out, m, bases, 0.015625f);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) madd_w<W, BLK><<<blocks, BLK>>>(out, m, bases, 0.015625f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  const double ffma = 2048.0 * m * wis;
  const double peak = (double)sms * 128 * clk_khz * 1e3;
  printf("%-12s %8.3f ms  %6.2f TFFMA/s  %.3f of FFMA peak\n", name, ms, ffma / (ms * 1e-3) / 1e12,
         ffma / (ms * 1e-3) / peak);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out, *bases;
  cudaMalloc(&out, (1 << 21) * 4);
  cudaMalloc(&bases, 16);
  float hb[4] = {0.5f, 0.5f, 0.5f, 0.5f};
  cudaMemcpy(bases, hb, 16, cudaMemcpyHostToDevice);
  run<1, 256>("W1 blk256", out, bases, sms, clk);
  run<2, 256>("W2 blk256", out, bases, sms, clk);
  run<2, 128>("W2 blk128", out, bases, sms, clk);
  run<3, 128>("W3 blk128", out, bases, sms, clk);
  run<4, 128>("W4 blk128", out, bases, sms, clk);
  run<4, 64>("W4 blk64", out, bases, sms, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
