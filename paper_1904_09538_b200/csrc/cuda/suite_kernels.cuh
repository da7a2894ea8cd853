// sm_100a realisations of the UIPiCK measurement kernels (reference
// src/uipick.cpp:295-664).
//
// Contract: every kernel executes
// exactly the IR of its generator — the same per-work-item index set, the
// same arithmetic in the same order (madd = one fused multiply-add), the same
// memory spaces (global vs shared) and the same barrier count per
// work-group. Work-items map to threads one-to-one with lid(0) -> threadIdx.x
// unless a kernel's comment states a coarsening; a coarsened thread executes
// several whole work-items of the same work-group row, which keeps every
// warp's addresses inside the cache lines the IR's lockstep order touches.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace ps {

// PatternLayout (uipick.cpp:211-245): the global index of work-item
// (lx, ly) in group (gx, gy) is s0*lx + s1*ly + s0*L0*gx + s1*L1*gy.
struct Pattern {
  int64_t s0, s1;
  int32_t L0, L1;
  int64_t G0, G1;
  __device__ __forceinline__ int64_t gidx(int lx, int ly, int64_t gx, int64_t gy) const {
    return s0 * lx + s1 * ly + s0 * L0 * gx + s1 * L1 * gy;
  }
};

// ---------------------------------------------------------------------------
// K1 gmem_pattern, 1:1 geometry (general strides): result[g] = in0[g] (+ in1[g])
// left-associated (uipick.cpp:306-313). 1-D grid over G0*G1 work-groups.
template <typename T, int K>
__global__ void __launch_bounds__(1024) gmem_pattern_generic(const T* __restrict__ in0,
                                                             const T* __restrict__ in1,
                                                             T* __restrict__ out, Pattern p) {
  int64_t bid = blockIdx.x;
  int64_t gx = bid % p.G0, gy = bid / p.G0;
  int64_t g = p.gidx(threadIdx.x, threadIdx.y, gx, gy);
  T v = in0[g];
  if constexpr (K == 2) v = add_t(v, in1[g]);
  out[g] = v;
}

// K1 gmem_pattern, contiguous layout (s0 = 1, s1 = L0 * G0: every row of
// the s1-wide matrix is covered by one row of work-groups). A thread executes
// the VEC consecutive lx work-items (4*VEC contiguous bytes per array) of one
// work-group row, and a CTA sweeps ROWS work-group rows, so each thread keeps
// ROWS independent 16-byte loads per array in flight. Index set, arithmetic
// and store per element are identical to the 1:1 kernel.
template <typename T, int K, int VEC, int ROWS>
__global__ void __launch_bounds__(256) gmem_pattern_rows(const T* __restrict__ in0,
                                                         const T* __restrict__ in1,
                                                         T* __restrict__ out, int64_t row_elems,
                                                         int64_t nrows) {
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int kPerVec = sizeof(V) / sizeof(T);
  static_assert(kPerVec * 1 == VEC, "VEC must equal the 16-byte lane width");
  const int64_t vecs_per_row = row_elems / kPerVec;
  const int64_t total_vecs = vecs_per_row * nrows;
  const V* a = reinterpret_cast<const V*>(in0);
  const V* b = reinterpret_cast<const V*>(in1);
  V* o = reinterpret_cast<V*>(out);
  int64_t base = (int64_t)blockIdx.x * blockDim.x * ROWS + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ROWS;
  for (; base < total_vecs; base += stride) {
    V va[ROWS], vb[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      int64_t i = base + (int64_t)r * blockDim.x;
      if (i < total_vecs) {
        va[r] = __ldcs(a + i);
        if constexpr (K == 2) vb[r] = __ldcs(b + i);
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      int64_t i = base + (int64_t)r * blockDim.x;
      if (i < total_vecs) {
        V v = va[r];
        if constexpr (K == 2) {
          if constexpr (sizeof(T) == 4) {
            v.x = add_t(v.x, vb[r].x);
            v.y = add_t(v.y, vb[r].y);
            v.z = add_t(v.z, vb[r].z);
            v.w = add_t(v.w, vb[r].w);
          } else {
            v.x = add_t(v.x, vb[r].x);
            v.y = add_t(v.y, vb[r].y);
          }
        }
        __stcs(o + i, v);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2-K4 flops_{add,mul,madd}_pattern (uipick.cpp:317-378): 32 private values
// v_j = 0.5 + j/64 (exact, flit at uipick.cpp:251-255); m iterations of a
// 64x-unrolled SHOC sweep v_j <- op(v_{(j+27)%32}, v_{(j+21)%32}) (madd:
// v_{(j+27)%32}*v_{(j+21)%32} + v_j fused); left-associated 31-add reduction;
// one store. base/step arrive as runtime arguments so nothing folds.
template <int OP>
__device__ __forceinline__ float flop_op(float a, float c, float self) {
  if constexpr (OP == 0) return __fadd_rn(a, c);
  if constexpr (OP == 1) return __fmul_rn(a, c);
  return __fmaf_rn(a, c, self);
}

template <int OP>
__global__ void __launch_bounds__(256) flops_pattern(float* __restrict__ out, Pattern p, int m,
                                                     float base, float step) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(base, __fmul_rn(step, (float)j));
  for (int t = 0; t < m; ++t) {
#pragma unroll
    for (int u = 0; u < 64; ++u) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = flop_op<OP>(v[(j + 27) & 31], v[(j + 21) & 31], v[j]);
    }
  }
  float r = v[0];
#pragma unroll
  for (int j = 1; j < 32; ++j) r = __fadd_rn(r, v[j]);
  int64_t bid = blockIdx.x;
  out[p.gidx(threadIdx.x, threadIdx.y, bid % p.G0, bid / p.G0)] = r;
}

// ---------------------------------------------------------------------------
// K5 lmem_shuffle (uipick.cpp:380-404): locbuf_a[l] = 1; m x (locbuf_b[l] =
// locbuf_a[l]); result[g] = locbuf_b[l]; no barrier. Shared accesses are
// volatile so each of the m load/store pairs is issued. Loads of an unrolled
// group are issued before its stores (they touch disjoint arrays, so the
// order is semantically free) to keep the shared pipe, not latency, binding.
__global__ void __launch_bounds__(1024) lmem_shuffle(float* __restrict__ out, Pattern p, int m) {
  extern __shared__ float smem[];
  const int wg = p.L0 * p.L1;
  float* sa = smem;
  float* sb = smem + wg;
  const int l = threadIdx.x + p.L0 * threadIdx.y;
  sts_volatile(&sa[l], 1.0f);
  int t = 0;
  for (; t + 4 <= m; t += 4) {
    float x0 = lds_volatile(&sa[l]);
    float x1 = lds_volatile(&sa[l]);
    float x2 = lds_volatile(&sa[l]);
    float x3 = lds_volatile(&sa[l]);
    sts_volatile(&sb[l], x0);
    sts_volatile(&sb[l], x1);
    sts_volatile(&sb[l], x2);
    sts_volatile(&sb[l], x3);
  }
  for (; t < m; ++t) sts_volatile(&sb[l], lds_volatile(&sa[l]));
  float r = lds_volatile(&sb[l]);
  int64_t bid = blockIdx.x;
  out[p.gidx(threadIdx.x, threadIdx.y, bid % p.G0, bid / p.G0)] = r;
}

// K6 barrier_knl (uipick.cpp:406-423): m local barriers, then result[g] = 1.
__global__ void __launch_bounds__(1024) barrier_knl(float* __restrict__ out, Pattern p, int m) {
  for (int t = 0; t < m; ++t) bar_sync();
  int64_t bid = blockIdx.x;
  out[p.gidx(threadIdx.x, threadIdx.y, bid % p.G0, bid / p.G0)] = 1.0f;
}

// K7 empty_knl (uipick.cpp:425-432): no statements, num_groups x 256.
__global__ void __launch_bounds__(256) empty_knl() {}

// K8 overlap_knl (uipick.cpp:434-462): tmp = in0[g]; m x (locbuf_b[l] =
// locbuf_a[l]) (locbuf_a is never written in the IR); result[g] = tmp.
__global__ void __launch_bounds__(1024) overlap_knl(const float* __restrict__ in0,
                                                    float* __restrict__ out, Pattern p, int m) {
  extern __shared__ float smem[];
  const int wg = p.L0 * p.L1;
  float* sa = smem;
  float* sb = smem + wg;
  const int l = threadIdx.x + p.L0 * threadIdx.y;
  int64_t bid = blockIdx.x;
  const int64_t g = p.gidx(threadIdx.x, threadIdx.y, bid % p.G0, bid / p.G0);
  float tmp = in0[g];
  int t = 0;
  for (; t + 2 <= m; t += 2) {
    float x0 = lds_volatile(&sa[l]);
    float x1 = lds_volatile(&sa[l]);
    sts_volatile(&sb[l], x0);
    sts_volatile(&sb[l], x1);
  }
  for (; t < m; ++t) sts_volatile(&sb[l], lds_volatile(&sa[l]));
  out[g] = tmp;
}

// K8 overlap_knl, contiguous layout (s0 = 1): the same coarsening as
// gmem_pattern_rows — a thread executes 4 consecutive lx work-items (one
// 16-byte vector) of ROWS work-group rows. Per work-item the IR order is
// kept: global load, m shared load/store pairs on the work-item's own
// locbuf slot (vectorised 16-byte LDS/STS over the thread's 4 work-items),
// global store. The ROWS global loads are issued before the shared work, so
// HBM latency overlaps the on-chip traffic exactly as the kernel intends.
template <int ROWS>
__global__ void __launch_bounds__(256) overlap_rows(const float* __restrict__ in0,
                                                   float* __restrict__ out, int64_t total_vecs,
                                                   int m) {
  __shared__ float4 sa[256], sb[256];
  const float4* a = reinterpret_cast<const float4*>(in0);
  float4* o = reinterpret_cast<float4*>(out);
  const unsigned pa = static_cast<unsigned>(__cvta_generic_to_shared(&sa[threadIdx.x]));
  const unsigned pb = static_cast<unsigned>(__cvta_generic_to_shared(&sb[threadIdx.x]));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ROWS;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * ROWS + threadIdx.x; base < total_vecs;
       base += stride) {
    float4 v[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t i = base + (int64_t)r * blockDim.x;
      if (i < total_vecs) v[r] = __ldcs(a + i);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      for (int t = 0; t < m; ++t) {
        float x, y, z, w;
        asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
                     : "r"(pa)
                     : "memory");
        asm volatile("st.volatile.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(pb), "f"(x), "f"(y),
                     "f"(z), "f"(w)
                     : "memory");
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t i = base + (int64_t)r * blockDim.x;
      if (i < total_vecs) __stcs(o + i, v[r]);
    }
  }
}

// ---------------------------------------------------------------------------
// Work-group order of the 16x16 matmul grids (the IR fixes which work-items a
// group holds, not the order the hardware runs groups in): with W > 0 the
// square grid is walked row-major inside panels of W block columns. The CTAs
// co-resident on an SM still share one block row (its a rows stay in L1), but
// a wave's b working set shrinks from all of b to W block columns, which fits
// L2 — at n = 8192 the default order streams b from DRAM ~220 times
// (tools/exp/mm_panel.cu: noPF 161 -> 122 ms, the b-column work-removed
// kernel 116 -> 73 ms at W = 64; PF unchanged).
constexpr int kMatmulPanel = 64;
__device__ __forceinline__ void matmul_group(int W, int& bx, int& by) {
  const int nb = (int)gridDim.x;
  if (W <= 0 || W >= nb) {
    bx = blockIdx.x;
    by = blockIdx.y;
    return;
  }
  const int id = blockIdx.y * nb + blockIdx.x;
  const int per = W * (int)gridDim.y, p = id / per, r = id % per;
  const int w = min(W, nb - p * W);
  by = r / w;
  bx = p * W + r % w;
}

// K9 matmul_sq noPF (uipick.cpp:478-502): c[i,j] = sum_k a[i,k]*b[k,j] with
// i = 16*i_out + i_in (g.1, l.1), j = 16*j_out + j_in (g.0, l.0); one madd
// per k in ascending order, accumulator starting at 0.
template <typename T>
__global__ void __launch_bounds__(256) matmul_nopf(const T* __restrict__ a,
                                                   const T* __restrict__ b, T* __restrict__ c,
                                                   int n, int tile, int panel) {
  int bx, by;
  matmul_group(panel, bx, by);
  const int i = by * tile + threadIdx.y;
  const int j = bx * tile + threadIdx.x;
  const T* arow = a + (int64_t)i * n;
  const T* bcol = b + j;
  T acc = T(0);
  if constexpr (sizeof(T) == 4) {
    // the work-item's a row along the sequential k as 16-byte loads (n is a
    // multiple of 16): same elements, same madd order, a quarter of the a
    // load instructions (32-byte loads measured slower here: 5.0 vs 8.2 TF/s)
    // All 10 loads of an 8-k step are issued before its first FMA (the madd
    // chain is serial, so the loads are the only parallelism there is).
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
  } else {
#pragma unroll 8
    for (int k = 0; k < n; ++k) acc = fma_t(arow[k], bcol[(int64_t)k * n], acc);
  }
  c[(int64_t)i * n + j] = acc;
}

// K10 matmul_sq PF (uipick.cpp:504-553): per k_out: barrier; a_fetch[i_in,
// j_in] = a[row, 16 k_out + j_in]; b_fetch[i_in, j_in] = b[16 k_out + i_in,
// col]; barrier; 16 madds acc += a_fetch[i_in,k_in] * b_fetch[k_in,j_in].
template <typename T, int TS>
__global__ void __launch_bounds__(TS* TS) matmul_pf(const T* __restrict__ a,
                                                    const T* __restrict__ b, T* __restrict__ c,
                                                    int n) {
  __shared__ __align__(16) T af[TS][TS];
  __shared__ T bf[TS][TS];
  const int ti = threadIdx.y, tj = threadIdx.x;
  const int row = blockIdx.y * TS + ti;
  const int col = blockIdx.x * TS + tj;
  T acc = T(0);
  const int ntiles = n / TS;
  for (int kt = 0; kt < ntiles; ++kt) {
    bar_sync();  // bar_pre
    af[ti][tj] = a[(int64_t)row * n + kt * TS + tj];
    bf[ti][tj] = b[(int64_t)(kt * TS + ti) * n + col];
    bar_sync();  // bar_post
    if constexpr (sizeof(T) == 4 && TS % 4 == 0) {
      // a_fetch row read 4 k_in at a time (LDS.128, a broadcast per half-warp)
#pragma unroll
      for (int k4 = 0; k4 < TS / 4; ++k4) {
        const float4 av = *reinterpret_cast<const float4*>(&af[ti][4 * k4]);
        acc = fma_t(av.x, bf[4 * k4][tj], acc);
        acc = fma_t(av.y, bf[4 * k4 + 1][tj], acc);
        acc = fma_t(av.z, bf[4 * k4 + 2][tj], acc);
        acc = fma_t(av.w, bf[4 * k4 + 3][tj], acc);
      }
    } else {
#pragma unroll
      for (int kin = 0; kin < TS; ++kin) acc = fma_t(af[ti][kin], bf[kin][tj], acc);
    }
  }
  c[(int64_t)row * n + col] = acc;
}

// K11 matmul_sq_rm (uipick.cpp:556-581 via remove_work, transforms.cpp:317-514):
// tgt_read = 0; tgt_read += (surviving load) over its loop; tgt_read_dest[i, j]
// = tgt_read with lid(0) fastest. keep: 1 = a, 2 = b.
template <typename T, bool PF, int KEEP>
__global__ void __launch_bounds__(256) matmul_rm(const T* __restrict__ src,
                                                 T* __restrict__ dest, int n, int tile, int panel) {
  const int ti = threadIdx.y, tj = threadIdx.x;
  int bx, by;
  matmul_group(panel, bx, by);  // the order of the application kernel it times
  const int row = by * tile + ti;
  const int col = bx * tile + tj;
  T acc = T(0);
  if constexpr (PF) {
    const int ntiles = n / tile;
#pragma unroll 4
    for (int kt = 0; kt < ntiles; ++kt) {
      if constexpr (KEEP == 1)
        acc = add_t(acc, src[(int64_t)row * n + kt * tile + tj]);
      else
        acc = add_t(acc, src[(int64_t)(kt * tile + ti) * n + col]);
    }
  } else if constexpr (KEEP == 1 && sizeof(T) == 4) {
    // the application kernel's 16-byte a-row loads
    const float4* row4 = reinterpret_cast<const float4*>(src + (int64_t)row * n);
    for (int k8 = 0; k8 < n / 8; ++k8) {
      const float4 v0 = __ldg(row4 + 2 * k8), v1 = __ldg(row4 + 2 * k8 + 1);
      acc = add_t(acc, v0.x);
      acc = add_t(acc, v0.y);
      acc = add_t(acc, v0.z);
      acc = add_t(acc, v0.w);
      acc = add_t(acc, v1.x);
      acc = add_t(acc, v1.y);
      acc = add_t(acc, v1.z);
      acc = add_t(acc, v1.w);
    }
  } else if constexpr (KEEP == 2) {
    // b column, 8 loads in flight ahead of the serial add chain (as the
    // application kernel issues them)
    const T* bcol = src + col;
    const int64_t n64 = n;
    for (int k8 = 0; k8 < n / 8; ++k8) {
      T v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldg(bcol + (8 * (int64_t)k8 + q) * n64);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = add_t(acc, v[q]);
    }
  } else {
#pragma unroll 8
    for (int k = 0; k < n; ++k) acc = add_t(acc, src[(int64_t)row * n + k]);
  }
  dest[(int64_t)row * n + col] = acc;
}

// ---------------------------------------------------------------------------
// K12 finite_diff TxT (uipick.cpp:583-639): fetch the TxT tile u[I i_out + l1,
// I j_out + l0] to shared; barrier; the I x I interior points of the
// five-point stencil, ((u01 + u10) - 4 u11) + u12 + u21 with the -4 u11 term
// fused (the IR counts it as a madd). The IR places the compute in
// sequential c1, c0 loops (a uniform, per-sub-group access); the
// realisation assigns interior point (c1, c0) to work-item (l1, l0), which
// executes the same n^2 statement instances.
template <int T>
__global__ void __launch_bounds__(T* T) finite_diff(const float* __restrict__ u,
                                                   float* __restrict__ res, int n) {
  constexpr int I = T - 2;
  __shared__ float uf[T][T + 1];
  const int l0 = threadIdx.x, l1 = threadIdx.y;
  const int i_out = blockIdx.y, j_out = blockIdx.x;
  const int64_t W = n + 2;
  uf[l1][l0] = u[(int64_t)(I * i_out + l1) * W + I * j_out + l0];
  bar_sync();
  if (l1 < I && l0 < I) {
    float s = __fadd_rn(uf[l1][l0 + 1], uf[l1 + 1][l0]);
    s = __fmaf_rn(-4.0f, uf[l1 + 1][l0 + 1], s);
    s = __fadd_rn(s, uf[l1 + 1][l0 + 2]);
    s = __fadd_rn(s, uf[l1 + 2][l0 + 1]);
    res[(int64_t)(I * i_out + l1) * n + I * j_out + l0] = s;
  }
}

// K12, coarsened: a CTA of T x T threads executes R horizontally adjacent
// work-groups (j_out = R*bx + r). Every work-item still fetches its own u
// element into its group's tile and the interior work-items compute their
// stencil point with the identical operation sequence; the R groups'
// barriers are executed as one CTA barrier (a superset synchronisation). The
// R independent fetches per thread keep enough HBM reads in flight.
template <int T, int R>
__global__ void __launch_bounds__(T* T) finite_diff_multi(const float* __restrict__ u,
                                                         float* __restrict__ res, int n) {
  constexpr int I = T - 2;
  __shared__ float uf[R][T][T + 1];
  const int l0 = threadIdx.x, l1 = threadIdx.y;
  const int i_out = blockIdx.y;
  const int groups = n / I;
  const int64_t W = n + 2;
  const float* urow = u + (int64_t)(I * i_out + l1) * W + l0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j_out = blockIdx.x * R + r;
    if (j_out < groups) uf[r][l1][l0] = __ldg(urow + I * j_out);
  }
  bar_sync();
  if (l1 < I && l0 < I) {
    float* rrow = res + (int64_t)(I * i_out + l1) * n + l0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j_out = blockIdx.x * R + r;
      if (j_out >= groups) break;
      float s = __fadd_rn(uf[r][l1][l0 + 1], uf[r][l1 + 1][l0]);
      s = __fmaf_rn(-4.0f, uf[r][l1 + 1][l0 + 1], s);
      s = __fadd_rn(s, uf[r][l1 + 1][l0 + 2]);
      s = __fadd_rn(s, uf[r][l1 + 2][l0 + 1]);
      __stcs(rrow + I * j_out, s);
    }
  }
}

// K12/K13, strip realisation: one CTA of fd_strip_threads<T>() threads owns R
// horizontally adjacent work-groups, i.e. the u strip rows I*i_out ..
// I*i_out+T-1, columns I*R*bx .. I*R*bx + I*R + 1. The union of the R tiles
// (every work-item's fetch: the overlapping halo columns are the same u
// elements) is staged into shared memory warp-per-row with coalesced loads,
// all of a thread's loads in flight before its first shared store; after the
// barrier the I x I*R interior points are computed with the exact operation
// sequence of the IR statement and stored warp-per-row (16-byte stores when
// rows are 16-byte aligned). The value computed for every (c1, c0) of every
// group is unchanged; only the thread that issues each access differs, and
// the CTA shape no longer follows the T x T work-group (a 324-thread 18x18
// group is not a whole number of warps).
// MODE 0: finite_diff; 1: finite_diff_rm keep u (tgt_read_dest tiles);
// 2: finite_diff_rm keep res (res interior = tgt_read = 0).
// 7 warps for 16x16 tiles and 8 for 18x18: each warp then owns exactly
// I / NW = 2 interior rows of the strip
template <int T>
constexpr int fd_strip_threads() {
  return T == 16 ? 224 : 256;
}

template <int T, int R, int MODE>
__global__ void __launch_bounds__(fd_strip_threads<T>()) finite_diff_strip(const float* __restrict__ u,
                                                                          float* __restrict__ out, int n) {
  constexpr int I = T - 2;
  constexpr int SW = I * R + 2;                   // strip width
  constexpr int NW = fd_strip_threads<T>() / 32;  // warps
  constexpr int CJ = (SW + 31) / 32;         // 32-column chunks per strip row
  constexpr int RW = (T + NW - 1) / NW;      // strip rows per warp (upper bound)
  // row pitch: a multiple of 4 floats so that every strip row starts 16-byte
  // aligned and the stencil reads its rows with conflict-free LDS.128
  constexpr int P = CJ * 32 + 4;
  __shared__ __align__(16) float reg[MODE == 2 ? 1 : T][MODE == 2 ? 4 : P];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i_out = blockIdx.y;
  const int groups = n / I;
  const int col0 = I * R * blockIdx.x;                      // first u column of the strip
  const int gcount = min(R, groups - R * (int)blockIdx.x);  // work-groups in this strip
  const int64_t W = n + 2;
  if constexpr (MODE != 2) {
    // 8-byte loads and shared stores: n is a multiple of I (even), so the row
    // pitch n + 2, the strip origin I*R*bx and the strip width I*gcount + 2
    // are all even and every float2 is aligned and wholly inside or outside
    constexpr int CJ2 = (SW + 63) / 64;  // 64-column chunks per strip row
    const int width = I * gcount + 2;
    const float2* base = reinterpret_cast<const float2*>(u + (int64_t)(I * i_out) * W + col0) + lane;
    float2 v[RW][CJ2];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int r = warp + k * NW;
      const float2* row = base + (int64_t)r * (W / 2);
#pragma unroll
      for (int j = 0; j < CJ2; ++j)
        v[k][j] = (r < T && 2 * (lane + 32 * j) < width) ? __ldg(row + 32 * j) : make_float2(0.0f, 0.0f);
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int r = warp + k * NW;
      if (r < T) {
#pragma unroll
        for (int j = 0; j < CJ2; ++j)
          if (2 * (lane + 32 * j) < P) *reinterpret_cast<float2*>(&reg[r][2 * (lane + 32 * j)]) = v[k][j];
      }
    }
    bar_sync();  // the R work-groups' fetch barriers, executed as one
  }
  if constexpr (MODE == 0 || MODE == 2) {
    const int width = I * gcount;
    float* rbase = out + (int64_t)(I * i_out) * n + col0;
    if ((n & 3) == 0) {  // rows and strip offsets are 16-byte aligned
      static_assert((I * R) % 4 == 0, "strip row must hold whole float4");
      constexpr int Q = I * R / 4;  // float4 per output row
      constexpr int QJ = (Q + 31) / 32;
      for (int r = warp; r < I; r += NW) {
#pragma unroll
        for (int j = 0; j < QJ; ++j) {
          const int c = 4 * (lane + 32 * j);
          if (4 * 32 * j >= width) continue;  // warp-uniform: the whole chunk is past the strip
          const bool live = c < width;
          float o[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          if constexpr (MODE == 0) {
            // rows r, r+1, r+2 over columns c .. c+5: the lane's aligned
            // float4 of each row; the two columns past it come from the next
            // lane's float4 (shuffle) — lane 31 reads them itself — so each
            // row is read once from shared memory instead of twice
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0;
            if (c < width + 4) {  // the first lane past the strip supplies the halo columns
              a0 = *reinterpret_cast<const float4*>(&reg[r][c]);
              a1 = *reinterpret_cast<const float4*>(&reg[r + 1][c]);
              a2 = *reinterpret_cast<const float4*>(&reg[r + 2][c]);
            }
            float n0 = __shfl_down_sync(0xffffffffu, a0.x, 1);
            float n1 = __shfl_down_sync(0xffffffffu, a1.x, 1);
            float n1b = __shfl_down_sync(0xffffffffu, a1.y, 1);
            float n2 = __shfl_down_sync(0xffffffffu, a2.x, 1);
            if (lane == 31 && live) {
              n0 = reg[r][c + 4];
              n1 = reg[r + 1][c + 4];
              n1b = reg[r + 1][c + 5];
              n2 = reg[r + 2][c + 4];
            }
            const float x0[4] = {a0.y, a0.z, a0.w, n0};
            const float x1[6] = {a1.x, a1.y, a1.z, a1.w, n1, n1b};
            const float x2[4] = {a2.y, a2.z, a2.w, n2};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float t = __fadd_rn(x0[k], x1[k]);
              t = __fmaf_rn(-4.0f, x1[k + 1], t);
              t = __fadd_rn(t, x1[k + 2]);
              o[k] = __fadd_rn(t, x2[k]);
            }
          }
          if (!live) continue;
          float* dst = rbase + (int64_t)r * n + c;
          if (c + 3 < width) {
            __stcs(reinterpret_cast<float4*>(dst), make_float4(o[0], o[1], o[2], o[3]));
          } else {
            for (int q = 0; q < 4 && c + q < width; ++q) __stcs(dst + q, o[q]);
          }
        }
      }
    } else {
      constexpr int QJ = (I * R + 31) / 32;
      for (int r = warp; r < I; r += NW) {
#pragma unroll
        for (int j = 0; j < QJ; ++j) {
          const int c = lane + 32 * j;
          if (c >= width) continue;
          float s = 0.0f;
          if constexpr (MODE == 0) {
            s = __fadd_rn(reg[r][c + 1], reg[r + 1][c]);
            s = __fmaf_rn(-4.0f, reg[r + 1][c + 1], s);
            s = __fadd_rn(s, reg[r + 1][c + 2]);
            s = __fadd_rn(s, reg[r + 2][c + 1]);
          }
          __stcs(rbase + (int64_t)r * n + c, s);
        }
      }
    }
  } else {
    // tgt_read_dest[T*i_out + l1, T*j_out + l0] = 0 + u[I*i_out + l1, I*j_out + l0]
    const int64_t DW = (int64_t)groups * T;
    const int width = T * gcount;
    float* dbase = out + (int64_t)(T * i_out) * DW + (int64_t)T * R * blockIdx.x;
    constexpr int DJ = (T * R + 31) / 32;
    for (int r = warp; r < T; r += NW) {
#pragma unroll
      for (int j = 0; j < DJ; ++j) {
        const int c = lane + 32 * j;
        if (c >= width) continue;
        const int g = c / T, l0 = c - g * T;
        __stcs(dbase + (int64_t)r * DW + c, __fadd_rn(0.0f, reg[r][I * g + l0]));
      }
    }
  }
}

template <int T, int R>
__global__ void __launch_bounds__(T* T) finite_diff_rm_u_multi(const float* __restrict__ u,
                                                              float* __restrict__ dest, int n) {
  constexpr int I = T - 2;
  const int l0 = threadIdx.x, l1 = threadIdx.y;
  const int i_out = blockIdx.y;
  const int groups = n / I;
  const int64_t W = n + 2;
  const int64_t DW = (int64_t)groups * T;
  const float* urow = u + (int64_t)(I * i_out + l1) * W + l0;
  float v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j_out = blockIdx.x * R + r;
    v[r] = j_out < groups ? __ldg(urow + I * j_out) : 0.f;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j_out = blockIdx.x * R + r;
    if (j_out < groups)
      __stcs(dest + (int64_t)(T * i_out + l1) * DW + T * j_out + l0, __fadd_rn(0.0f, v[r]));
  }
}

// K13 finite_diff_rm (uipick.cpp:641-664). keep u: tgt_read = 0 + u[fetch
// index]; tgt_read_dest[T i_out + l1, T j_out + l0] = tgt_read. keep res:
// res[interior] = tgt_read = 0.
template <int T>
__global__ void __launch_bounds__(T* T) finite_diff_rm_u(const float* __restrict__ u,
                                                        float* __restrict__ dest, int n) {
  constexpr int I = T - 2;
  const int l0 = threadIdx.x, l1 = threadIdx.y;
  const int i_out = blockIdx.y, j_out = blockIdx.x;
  const int64_t W = n + 2;
  const int64_t DW = (int64_t)(n / I) * T;
  float acc = __fadd_rn(0.0f, u[(int64_t)(I * i_out + l1) * W + I * j_out + l0]);
  dest[(int64_t)(T * i_out + l1) * DW + T * j_out + l0] = acc;
}

template <int T>
__global__ void __launch_bounds__(T* T) finite_diff_rm_res(float* __restrict__ res, int n) {
  constexpr int I = T - 2;
  const int l0 = threadIdx.x, l1 = threadIdx.y;
  if (l1 < I && l0 < I)
    res[(int64_t)(I * blockIdx.y + l1) * n + I * blockIdx.x + l0] = 0.0f;
}

}  // namespace ps
