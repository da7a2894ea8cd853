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

// two work-items per thread packed into the lanes of one 64-bit register
// pair: each FFMA2 (fma.rn.f32x2, sm_100) executes the same fused
// multiply-add of both work-items' chains, every lane exactly fmaf.
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int BLK>
__global__ void __launch_bounds__(BLK) madd_f2(float* out, int m, const float* __restrict__ bases, float step) {
  unsigned long long v[32];
  const float b0 = bases[0], b1 = bases[1];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float2 x = make_float2(__fadd_rn(b0, __fmul_rn(step, (float)j)), __fadd_rn(b1, __fmul_rn(step, (float)j)));
    v[j] = *reinterpret_cast<unsigned long long*>(&x);
  }
  for (int t = 0; t < m; ++t) {
#pragma unroll
    for (int u = 0; u < 64; ++u) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ffma2(v[(j + 27) & 31], v[(j + 21) & 31], v[j]);
    }
  }
  float r0, r1;
  {
    float2 x = *reinterpret_cast<float2*>(&v[0]);
    r0 = x.x;
    r1 = x.y;
  }
#pragma unroll
  for (int j = 1; j < 32; ++j) {
    float2 x = *reinterpret_cast<float2*>(&v[j]);
    r0 = __fadd_rn(r0, x.x);
    r1 = __fadd_rn(r1, x.y);
  }
  out[((size_t)blockIdx.x * BLK + threadIdx.x) * 2] = r0;
  out[((size_t)blockIdx.x * BLK + threadIdx.x) * 2 + 1] = r1;
}

template <int BLK>
void run_f2(const char* name, float* out, const float* bases, int sms, int clk_khz) {
  const int m = 64;
  const long long wis = (1LL << 21);
  const int blocks = (int)(wis / 2 / BLK);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) madd_f2<BLK><<<blocks, BLK>>>(out, m, bases, 0.015625f);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) madd_f2<BLK><<<blocks, BLK>>>(out, m, bases, 0.015625f);
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
  run_f2<256>("F2 blk256", out, bases, sms, clk);
  run_f2<128>("F2 blk128", out, bases, sms, clk);
  // bitwise: the packed kernel's work-item results equal the scalar kernel's
  {
    std::vector<float> a(1 << 21), b(1 << 21);
    madd_w<1, 256><<<(1 << 21) / 256, 256>>>(out, 3, bases, 0.015625f);
    cudaMemcpy(a.data(), out, (1 << 21) * 4, cudaMemcpyDeviceToHost);
    madd_f2<256><<<(1 << 20) / 256, 256>>>(out, 3, bases, 0.015625f);
    cudaMemcpy(b.data(), out, (1 << 21) * 4, cudaMemcpyDeviceToHost);
    printf("F2 bitwise equal to scalar: %s\n", memcmp(a.data(), b.data(), a.size() * 4) == 0 ? "yes" : "NO");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
