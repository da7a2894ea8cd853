// K14/K15: DG element-wise differentiation, res[m,k,i] = sum_j dm[m,i,j] u[k,j]
// (the reference ships no DG generator, SPEC.md:16,536 —
// the IR these kernels realise is defined by this repo's dg_diff builder,
// DESIGN.md "DG variants").
//
// Common geometry: i split by 16 (g.1/l.1), k split by 16 (g.0/l.0); a
// work-item owns (k, i) and loops over m and j. Layouts (row-major):
//   dm  [nmat][Np][Np]
//   u   [nel][Np]         (dmPFtrans: [Np][nel], k fastest)
//   res [nmat][nel][Np]   (dmPFtrans: [nmat][Np][nel], k fastest)
// Accumulation order per (m, k, i): j ascending from 0, fused multiply-add,
// identical in all four variants (so all four produce the same bits).
#pragma once

#include "device_common.cuh"

namespace ps {

struct DgDims {
  int64_t nel;
  int np;
  int nmat;
};

__device__ __forceinline__ int64_t dg_u_idx(bool trans, const DgDims& d, int64_t k, int j) {
  return trans ? (int64_t)j * d.nel + k : k * d.np + j;
}
__device__ __forceinline__ int64_t dg_res_idx(bool trans, const DgDims& d, int m, int64_t k,
                                              int i) {
  return trans ? ((int64_t)m * d.np + i) * d.nel + k : ((int64_t)m * d.nel + k) * d.np + i;
}

// Lane skew of the u-row loads (noPF, dmPF and their work-removed kernels).
// A work-item reads its own u row k (pitch Np floats) 32 bytes at a time; the
// 16 k of a warp sit Np*4 bytes apart, so when that pitch is a multiple of
// 128 B every lane's sector of one load instruction lies at the same offset
// within its cache line, and the warp's 16 sectors are served one per L1
// cycle (measured on B200: Np = 32, 64, 96, 128 run at ~3.4 TF/s, Np = 16, 48
// — pitch an odd multiple of 64 B — at ~5 TF/s). Skewing which chunk a lane
// loads in a given instruction spreads the sectors over 4 (2 for dmPF) line
// offsets. Only the issue schedule changes: each work-item still loads the
// same elements and accumulates them in the same order.
//   pitch % 128 == 0  (Np/8 % 4 == 0): skew = lx & 3, offsets 0..3 from the skew
//   pitch % 128 == 64 (Np/8 % 4 == 2): skew = (lx >> 1) & 1, the row parity
//                                      supplies the other factor of 2
__device__ __forceinline__ int dg_lane_skew(int lx, int nj8, int* smax) {
  const bool four = (nj8 & 3) == 0;
  *smax = four ? 3 : 1;
  return four ? (lx & 3) : ((lx >> 1) & 1);
}
// dmPF: a tile's u row is two 32-byte chunks; half the lanes load them in
// reverse order (2 line offsets, 4 with the row parity when Np/8 % 4 == 2).
__device__ __forceinline__ bool dg_lane_swap(int lx, int nj8) {
  return ((nj8 & 3) == 0) ? (lx & 1) : ((lx >> 1) & 1);
}

// noPF: no local memory; m outermost, reduction over j. The work-item's own
// row reads along the sequential j are issued as 32-byte loads (Np is a
// multiple of 16, so rows are 64-byte aligned): the same thread reads the same
// elements and accumulates them in the same order. The (m, j8) chunk sequence
// of a work-item runs as one stream, lane l starting dg_lane_skew(l) steps
// late; a work-item stores res[m, k, i] when its m-th row completes.
__global__ void __launch_bounds__(256) dg_nopf(const float* __restrict__ dm,
                                               const float* __restrict__ u,
                                               float* __restrict__ res, DgDims d) {
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i = blockIdx.y * 16 + ly;
  const int nj8 = d.np / 8;
  int smax;
  const int s = dg_lane_skew(lx, nj8, &smax);
  const int S = d.nmat * nj8;
  const float* urow = u + k * d.np;
  const float* dmrow = dm + (int64_t)i * d.np;
  int m = 0, j8 = 0;
  float acc = 0.f;
  for (int t = 0; t < S + smax; ++t) {
    const int c = t - s;
    if (c >= 0 && c < S) {
      const f8 a = ldg256(dmrow + 8 * j8), b = ldg256(urow + 8 * j8);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = __fmaf_rn(a.v[q], b.v[q], acc);
      if (++j8 == nj8) {
        res[dg_res_idx(false, d, m, k, i)] = acc;
        acc = 0.f;
        j8 = 0;
        ++m;
        dmrow += (int64_t)d.np * d.np;
      }
    }
  }
}

// uPF: 16x16 tiles of u staged in shared memory per j_out (two barriers per
// tile), m privatised into NMAT accumulators, loop order j_out, j_in, m.
// Row pitch 20 keeps u_fetch rows 16-byte aligned (conflict-free LDS.128 per
// quarter warp); the work-item's dm row and u_fetch row are read 4 j_in at a
// time, the FMAs still run in j_in, m order.
template <int NMAT>
__global__ void __launch_bounds__(256) dg_upf(const float* __restrict__ dm,
                                              const float* __restrict__ u,
                                              float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float uf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * 16;
  const int i = blockIdx.y * 16 + ly;
  float acc[NMAT];
#pragma unroll
  for (int m = 0; m < NMAT; ++m) acc[m] = 0.f;
  for (int jo = 0; jo < d.np / 16; ++jo) {
    bar_sync();
    uf[ly][lx] = u[(k0 + ly) * d.np + jo * 16 + lx];  // u_fetch[k_in, j_in], j_in -> l.0
    bar_sync();
    // the work-item's dm rows for this j_out: 2 x 32-byte loads per m, the
    // same load shape as noPF's (dg-uPFnoPF-dm is one tag for both)
    f8 dv[NMAT][2];
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const float* row = dm + ((int64_t)m * d.np + i) * d.np + jo * 16;
      dv[m][0] = ldg256(row);
      dv[m][1] = ldg256(row + 8);
    }
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 uv = *reinterpret_cast<const float4*>(&uf[lx][4 * j4]);
      const float u4[4] = {uv.x, uv.y, uv.z, uv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * j4 + q;
#pragma unroll
        for (int m = 0; m < NMAT; ++m) acc[m] = __fmaf_rn(dv[m][j >> 3].v[j & 7], u4[q], acc[m]);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < NMAT; ++m) res[dg_res_idx(false, d, m, k0 + lx, i)] = acc[m];
}

// dmPF / dmPFtrans: per m and j_out, a 16x16 tile of dm staged in shared
// memory (two barriers per tile); u read directly (strided by Np in dmPF,
// unit-stride across lid(0) in the transposed layout). The work-item's
// dm_fetch row is read 4 j_in at a time (LDS.128, pitch 20), and in dmPF its
// u row 8 at a time (32-byte loads, the two chunks of a tile in lane-swapped
// order, dg_lane_swap); all 16 u loads of a j_out tile are issued before its
// FMAs, which run in j_in order.
template <bool TRANS>
__global__ void __launch_bounds__(256) dg_dmpf(const float* __restrict__ dm,
                                               const float* __restrict__ u,
                                               float* __restrict__ res, DgDims d) {
  __shared__ __align__(16) float dmf[16][20];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 16 + lx;
  const int i0 = blockIdx.y * 16;
  const bool sw = !TRANS && dg_lane_swap(lx, d.np / 8);
  for (int m = 0; m < d.nmat; ++m) {
    float acc = 0.f;
    for (int jo = 0; jo < d.np / 16; ++jo) {
      bar_sync();
      dmf[ly][lx] = dm[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx];
      bar_sync();
      if constexpr (TRANS) {
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 a = *reinterpret_cast<const float4*>(&dmf[ly][4 * j4]);
          const int j = jo * 16 + 4 * j4;
          const float b0 = __ldg(u + (int64_t)j * d.nel + k);
          const float b1 = __ldg(u + (int64_t)(j + 1) * d.nel + k);
          const float b2 = __ldg(u + (int64_t)(j + 2) * d.nel + k);
          const float b3 = __ldg(u + (int64_t)(j + 3) * d.nel + k);
          acc = __fmaf_rn(a.x, b0, acc);
          acc = __fmaf_rn(a.y, b1, acc);
          acc = __fmaf_rn(a.z, b2, acc);
          acc = __fmaf_rn(a.w, b3, acc);
        }
      } else {
        const float* ur = u + k * d.np + jo * 16;
        const f8 x0 = ldg256(ur + (sw ? 8 : 0)), x1 = ldg256(ur + (sw ? 0 : 8));
        f8 b0, b1;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          b0.v[q] = sw ? x1.v[q] : x0.v[q];
          b1.v[q] = sw ? x0.v[q] : x1.v[q];
        }
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
    }
    res[dg_res_idx(TRANS, d, m, k, i0 + ly)] = acc;
  }
}

// Work-removed DG (remove_work semantics, transforms.cpp:317-514): the kept
// global load accumulates into tgt_read in the variant's statement order; a
// kept res store writes tgt_read (= 0); otherwise tgt_read_dest[i, k] (lid(0)
// fastest) receives tgt_read.
// keep: 3 = u, 5 = dm, 4 = res.  variant: 0 noPF, 1 uPF, 2 dmPF, 3 dmPFtrans.
template <int VARIANT, int KEEP>
__global__ void __launch_bounds__(256) dg_rm(const float* __restrict__ src,
                                             float* __restrict__ dst, DgDims d) {
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * 16;
  const int64_t k = k0 + lx;
  const int i0 = blockIdx.y * 16;
  const int i = i0 + ly;
  constexpr bool TRANS = VARIANT == 3;
  if constexpr (KEEP == 4) {
    for (int m = 0; m < d.nmat; ++m) dst[dg_res_idx(TRANS, d, m, k, i)] = 0.f;
    return;
  } else {
    float acc = 0.f;
    const int njo = d.np / 16;
    // row reads along the sequential j use the same 16-byte loads as the
    // application kernels (same accesses, same fadd order)
    auto add4 = [&](float4 v) {
      acc = __fadd_rn(acc, v.x);
      acc = __fadd_rn(acc, v.y);
      acc = __fadd_rn(acc, v.z);
      acc = __fadd_rn(acc, v.w);
    };
    if constexpr (VARIANT == 0) {
      // statement within (m, k, i), reduction j; the application kernel's
      // lane-skewed (m, j8) chunk stream
      const int nj8 = d.np / 8;
      int smax;
      const int s = dg_lane_skew(lx, nj8, &smax);
      const int S = d.nmat * nj8;
      const float* row0 = KEEP == 3 ? src + k * d.np : src + (int64_t)i * d.np;
      const float* row = row0;
      int j8 = 0;
      for (int t = 0; t < S + smax; ++t) {
        const int c = t - s;
        if (c >= 0 && c < S) {
          const f8 v = ldg256(row + 8 * j8);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc = __fadd_rn(acc, v.v[q]);
          if (++j8 == nj8) {
            j8 = 0;
            if (KEEP != 3) row += (int64_t)d.np * d.np;
          }
        }
      }
    } else if constexpr (VARIANT == 1) {
      if constexpr (KEEP == 3) {
        // fetch: one u load per (work-item, j_out)
        for (int jo = 0; jo < njo; ++jo) acc = __fadd_rn(acc, src[(k0 + ly) * d.np + jo * 16 + lx]);
      } else {
        // the uPF update's dm reads: per j_out, 2 x 32-byte loads per m
        for (int jo = 0; jo < njo; ++jo) {
          f8 v[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (m < d.nmat) {
              const float* row = src + ((int64_t)m * d.np + i) * d.np + jo * 16;
              v[m][0] = ldg256(row);
              v[m][1] = ldg256(row + 8);
            }
#pragma unroll
          for (int j = 0; j < 16; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (m < d.nmat) acc = __fadd_rn(acc, v[m][j >> 3].v[j & 7]);
        }
      }
    } else {
      if constexpr (KEEP == 3) {
        for (int m = 0; m < d.nmat; ++m)
          for (int jo = 0; jo < njo; ++jo) {
            if constexpr (TRANS) {
              for (int j4 = 0; j4 < 4; ++j4)
                for (int q = 0; q < 4; ++q)
                  acc = __fadd_rn(acc, src[dg_u_idx(true, d, k, jo * 16 + 4 * j4 + q)]);
            } else {
              const bool sw = dg_lane_swap(lx, d.np / 8);
              const float* ur = src + k * d.np + jo * 16;
              const f8 x0 = ldg256(ur + (sw ? 8 : 0)), x1 = ldg256(ur + (sw ? 0 : 8));
#pragma unroll
              for (int q = 0; q < 8; ++q) acc = __fadd_rn(acc, sw ? x1.v[q] : x0.v[q]);
#pragma unroll
              for (int q = 0; q < 8; ++q) acc = __fadd_rn(acc, sw ? x0.v[q] : x1.v[q]);
            }
          }
      } else {
        for (int m = 0; m < d.nmat; ++m)
          for (int jo = 0; jo < njo; ++jo)
            acc = __fadd_rn(acc, src[((int64_t)m * d.np + i0 + ly) * d.np + jo * 16 + lx]);
      }
    }
    dst[(int64_t)i * d.nel + k] = acc;
  }
}

}  // namespace ps
