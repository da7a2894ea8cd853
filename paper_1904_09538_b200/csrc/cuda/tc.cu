// K16: matmul_sq_tc — the extra dense-contraction variant on the 5th-gen
// tensor cores (not a paper variant; BASELINE north_star "tensor cores appear
// only in an extra tcgen05 matmul/DG variant flagged as a dense contraction").
//
// C[n][n] = A[n][n] . B[n][n], fp32 row-major in HBM, computed with
// tcgen05.mma kind::tf32 (A and B read as TF32, FP32 accumulation in TMEM).
// With the suite's seed-pattern inputs (small integers, tests/support.hpp:35-44)
// every product and partial sum is exact, so the result equals the fp32
// oracle bit for bit; on U[-1,1) inputs the TF32 operand rounding bounds the
// error (stated in tests/test_gpu_parity.py).
//
// A is read K-major (row-major A[m][k]); B is read N-major straight from
// row-major B[k][n] (instruction descriptor b_major = MN). For tf32 the only
// MN-major shared-memory layout the tensor core accepts is the 128-byte
// swizzle with 32-byte atomicity (SWIZZLE_128B_BASE32B, TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; with the plain 128-byte swizzle the
// accumulator silently stays zero — measured). PS_TC_B=k selects the older
// path that first writes Bt = B^T and reads both operands K-major (~11% slower
// at n = 8192: 0.2 ms of transpose traffic per launch).
//
// Persistent CTAs (one per SM) over 128x256 output tiles, 6 warps:
//   warp 0 lane 0  TMA producer: per 32-wide K block, A 128x32 (K-major) and
//                  B 32x256 (N-major, one 3-D box) into a 4-stage ring,
//                  mbarrier complete_tx;
//   warp 1 lane 0  MMA issuer: 4 x tcgen05.mma (M=128, N=256, K=8) per stage
//                  into one of two TMEM accumulators, tcgen05.commit frees
//                  the stage / publishes the accumulator;
//   warps 2-5      epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes
//                  32(w%4)..+31 = tile rows), 16-byte streaming stores,
//                  overlapping the next tile's MMAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "runtime_internal.h"

namespace ps {
namespace {

constexpr int BM = 128, BN = 256, BK = 32;  // BK: 32 fp32 = one 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int UMMA_K = 8;                   // K per tcgen05.mma for kind::tf32
constexpr int A_BYTES = BM * BK * 4;        // 16 KB
constexpr int B_BYTES = BN * BK * 4;        // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 256;         // 128 lanes x 256 fp32 columns

// Instruction descriptor (cute/arch/mma_sm100_desc.hpp InstrDescriptor):
// D f32, A/B tf32, both K-major, N>>3 at bit 17, M>>4 at bit 24.
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                           (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
// Same with B N-major (b_major bit 16): B read straight from row-major [k][n].
constexpr uint32_t IDESC_BMN = IDESC | (1u << 16);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TC_WAIT;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// Shared-memory matrix descriptor, 128-byte swizzle (cute UMMA::SmemDescriptor):
// start >> 4 at [0,14), LBO >> 4 at [16,30), SBO >> 4 at [32,46), version 1 at
// [46,48), layout SWIZZLE_128B (2) at [61,64).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// MN-major tf32 operands take the 128-byte swizzle with 32-byte atomicity
// (layout type 1, SWIZZLE_128B_BASE32B; cute Layout_MN_SW128_32B_Atom: rows of
// 128 B along N, 4-row K groups of 512 B, Swizzle<2,5,2>).
__device__ __forceinline__ uint64_t desc_sw128_32b(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(1) << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc,
                                         uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u)  // no output lanes disabled
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Persistent: one CTA per SM walks the output tiles (tile = blockIdx.x +
// k * gridDim.x, 128-row blocks fastest inside bands of TILE_BAND column
// blocks for L2 reuse). Two 256-column TMEM accumulators let the epilogue of
// tile i drain while the MMAs of tile i+1 run. 6 warps: 0 TMA, 1 MMA,
// 2-5 epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
constexpr int TILE_BAND = 8;

__device__ __forceinline__ void tile_coords(int t, int mt, int& m0, int& n0) {
  const int per_band = TILE_BAND * mt;
  const int band = t / per_band, r = t - band * per_band;
  m0 = (r % mt) * BM;
  n0 = (band * TILE_BAND + r / mt) * BN;
}

__device__ __forceinline__ void tile_coords2(int t, int mt, int& m0, int& n0) {
  const int per_band = TILE_BAND * mt;
  const int band = t / per_band, r = t - band * per_band;
  m0 = (r % mt) * 256;
  n0 = (band * TILE_BAND + r / mt) * BN;
}

// BMN: B is loaded N-major straight from row-major B[k][n] — one 3-D TMA box
// of 8 N-atoms x 32 k-rows x 32 n (128 B rows, 128B swizzle with 32-byte
// atomicity, the only MN-major layout tf32 accepts), atoms 4 KB apart (LBO),
// 4-row K groups 512 B apart (SBO), start + 1024 B per 8-deep K step.
template <bool BMN>
__global__ void __launch_bounds__(192, 1)
    matmul_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     float* __restrict__ C, int n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;                                    // STAGES x A tile (1024-aligned)
  uint8_t* sb = smem + STAGES * A_BYTES;                 // STAGES x Bt tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = n / BK;
  const int mt = n / BM, ntiles = mt * (n / BN);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 128);  // every epilogue thread arrives
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // one warp allocates (and later frees) both accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer, stage ring continues across tiles
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0;
        tile_coords(t, mt, m0, n0);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty0 + 8 * s, ((it / STAGES) - 1) & 1);
          const uint32_t fb = full0 + 8 * s;
          mbar_expect_tx(fb, STAGE_BYTES);
          tma_load_2d(smem_u32(sa + s * A_BYTES), &tmA, fb, kb * BK, m0);
          if constexpr (BMN)
            tma_load_3d(smem_u32(sb + s * B_BYTES), &tmB, fb, 0, kb * BK, n0 / 32);
          else
            tma_load_2d(smem_u32(sb + s * B_BYTES), &tmB, fb, kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t d = tmem + uint32_t(acc * TMEM_COLS);
        if (local >= 2) mbar_wait(tempty0 + 8 * acc, ((local >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full0 + 8 * s, (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(sa + s * A_BYTES), b_base = smem_u32(sb + s * B_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            // K-major, 128 B swizzle rows: advance 8 tf32 (32 B) inside the
            // row; 8-row groups 1024 B apart (SBO); LBO unused (16 B)
            const uint64_t da = desc_sw128(a_base + ks * UMMA_K * 4, 16, 1024);
            if constexpr (BMN) {
              // N-major: 32-n atoms 4096 B apart (LBO), 4-row K groups 512 B
              // apart (SBO); one K step of 8 rows starts 1024 B further
              const uint64_t db = desc_sw128_32b(b_base + ks * 1024, 4096, 512);
              mma_tf32(d, da, db, (kb | ks) != 0, IDESC_BMN);
            } else {
              const uint64_t db = desc_sw128(b_base + ks * UMMA_K * 4, 16, 1024);
              mma_tf32(d, da, db, (kb | ks) != 0, IDESC);
            }
          }
          mma_commit(empty0 + 8 * s);  // stage s free once these MMAs have read it
        }
        mma_commit(tfull0 + 8 * acc);  // accumulator complete
      }
    }
  } else {
    // epilogue warps 2-5: TMEM lanes 32*(warp%4) .. +31 are tile rows
    const int q4 = warp & 3;
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      int m0, n0;
      tile_coords(t, mt, m0, n0);
      const int acc = local & 1;
      mbar_wait(tfull0 + 8 * acc, (local >> 1) & 1);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + 32 * q4 + lane;
      float* crow = C + (int64_t)row * n + n0;
      const uint32_t tbase = tmem + (uint32_t(32 * q4) << 16) + uint32_t(acc * TMEM_COLS);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + uint32_t(32 * c), v);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          __stcs(reinterpret_cast<float4*>(crow + 32 * c + 4 * q),
                 make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * acc) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * TMEM_COLS)
                 : "memory");
}

// ---------------------------------------------------------------------------
// CTA-pair version (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile with M = 256 MMAs issued by the leader (rank 0). Each CTA
// stages its own 128 rows of A and its own 128-column half of B (N-major)
// per 32-deep K block, so a pair reads 2 x (128 + 128) x 32 operands per K
// block for a 256 x 256 tile instead of 2 x (128 + 256) x 32 for two 128 x 256
// tiles: a third less L2 -> SM traffic. Both CTAs' TMA loads complete on the
// leader's stage barrier (.cta_group::2, peer bit cleared); the leader's
// tcgen05.commit multicasts stage-free / accumulator-ready to both CTAs; both
// epilogues drain their own TMEM rows and arrive on the leader's
// accumulator-free barrier through its cluster address.
constexpr int BM2 = 256, STAGES2 = 6;
constexpr int A2_BYTES = 128 * BK * 4;        // this CTA's 128 rows of A
constexpr int B2_BYTES = (BN / 2) * BK * 4;   // this CTA's 128 columns of B
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + 1024 + 256;
constexpr uint32_t IDESC2 = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM2 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(uint32_t local) {  // same offset in cluster rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
  return r;
}
__device__ __forceinline__ void tma2_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void tma2_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mma2_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC2), "r"(acc), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((unsigned short)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    matmul_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      float* __restrict__ C, int n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                            // STAGES2 x (128 x 32) A
  uint8_t* sb = smem + STAGES2 * A2_BYTES;       // STAGES2 x (32 x 128) B half, N-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + STAGES2 * B2_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES2 + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nk = n / BK;
  const int mt = n / BM2, ntiles = mt * (n / BN);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES2);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES2), tempty0 = smem_u32(bars + 2 * STAGES2 + 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 256);  // both CTAs' epilogue threads (leader's copy)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own A rows and own B half
      int it = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int m0, n0;
        tile_coords2(t, mt, m0, n0);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES2;
          if (it >= STAGES2) mbar_wait(empty0 + 8 * s, ((it / STAGES2) - 1) & 1);
          const uint32_t fb = full0 + 8 * s;
          if (leader) mbar_expect_tx(fb, 2 * STAGE2_BYTES);
          tma2_2d(smem_u32(sa + s * A2_BYTES), &tmA, fb, kb * BK, m0 + 128 * int(rank));
          tma2_3d(smem_u32(sb + s * B2_BYTES), &tmB, fb, 0, kb * BK, (n0 + 128 * int(rank)) / 32);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer for the pair
      int it = 0, local = 0;
      for (int t = pair; t < ntiles; t += npairs, ++local) {
        const int acc = local & 1;
        const uint32_t d = tmem + uint32_t(acc * TMEM_COLS);
        if (local >= 2) mbar_wait(tempty0 + 8 * acc, ((local >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES2;
          mbar_wait(full0 + 8 * s, (it / STAGES2) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(sa + s * A2_BYTES), b_base = smem_u32(sb + s * B2_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks)
            mma2_tf32(d, desc_sw128(a_base + ks * UMMA_K * 4, 16, 1024), desc_sw128_32b(b_base + ks * 1024, 4096, 512),
                      (kb | ks) != 0);
          commit2(empty0 + 8 * s);
        }
        commit2(tfull0 + 8 * acc);
      }
    }
  } else {  // epilogue (both CTAs): this CTA's 128 rows of the 256 x 256 tile
    const int q4 = warp & 3;
    int local = 0;
    for (int t = pair; t < ntiles; t += npairs, ++local) {
      int m0, n0;
      tile_coords2(t, mt, m0, n0);
      const int acc = local & 1;
      mbar_wait(tfull0 + 8 * acc, (local >> 1) & 1);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + 128 * int(rank) + 32 * q4 + lane;
      float* crow = C + (int64_t)row * n + n0;
      const uint32_t tbase = tmem + (uint32_t(32 * q4) << 16) + uint32_t(acc * TMEM_COLS);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + uint32_t(32 * c), v);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          __stcs(reinterpret_cast<float4*>(crow + 32 * c + 4 * q),
                 make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(tempty0 + 8 * acc))
                   : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TMEM_COLS) : "memory");
}

// Bt[j][i] = B[i][j], 32x32 tiles through shared memory (coalesced both ways).
__global__ void __launch_bounds__(256) transpose_f32(const float* __restrict__ b,
                                                     float* __restrict__ bt, int n) {
  __shared__ float t[32][33];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows per pass
#pragma unroll
  for (int r = ty; r < 32; r += 8) t[r][tx] = __ldg(b + (int64_t)(y0 + r) * n + x0 + tx);
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) __stcs(bt + (int64_t)(x0 + r) * n + y0 + tx, t[tx][r]);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 row-major [rows][cols] map with a box of box_cols x box_rows.
int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, uint32_t box_cols,
             uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_error(PS_ERR_CUDA, "matmul_sq_tc: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(PS_ERR_CUDA, "matmul_sq_tc: cuTensorMapEncodeTiled failed (%d)", int(r));
  return PS_OK;
}

// B[k][n] row-major viewed as 3-D (32 n, k, n/32 atoms) for N-major boxes.
int make_map_bmn(CUtensorMap* m, const void* base, int64_t n) {
  auto fn = encode_fn();
  if (!fn) return set_error(PS_ERR_CUDA, "matmul_sq_tc: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {32, cuuint64_t(n), cuuint64_t(n / 32)};
  const cuuint64_t strides[2] = {cuuint64_t(n) * 4, 128};
  const cuuint32_t box[3] = {32, BK, BN / 32};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(PS_ERR_CUDA, "matmul_sq_tc: cuTensorMapEncodeTiled (B N-major) failed (%d)", int(r));
  return PS_OK;
}

// B half for the CTA pair: box 32 n x 32 k x 4 atoms (128 columns)
int make_map_bmn_half(CUtensorMap* m, const void* base, int64_t n) {
  auto fn = encode_fn();
  if (!fn) return set_error(PS_ERR_CUDA, "matmul_sq_tc: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {32, cuuint64_t(n), cuuint64_t(n / 32)};
  const cuuint64_t strides[2] = {cuuint64_t(n) * 4, 128};
  const cuuint32_t box[3] = {32, BK, (BN / 2) / 32};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PS_ERR_CUDA, "matmul_sq_tc: B half map failed (%d)", int(r));
  return PS_OK;
}

int tc_mode() {  // 2 = CTA pairs (default), 1 = single CTA, 0 = transpose path
  const char* e = std::getenv("PS_TC_B");
  if (e && std::string(e) == "k") return 0;
  const char* p = std::getenv("PS_TC_PAIR");
  return (p && std::string(p) == "0") ? 1 : 2;
}

bool b_n_major() {
  const char* e = std::getenv("PS_TC_B");
  return !(e && std::string(e) == "k");
}

}  // namespace

int tc_launch(Ctx* c, const ps_kernel_desc* d) {
  if (d->dtype != PS_F32) return set_error(PS_ERR_ARG, "matmul_sq_tc is float32 (tf32 tensor cores)");
  const int n = (int)d->n;
  if (n % BN != 0) return set_error(PS_ERR_ARG, "matmul_sq_tc requires n to be a multiple of %d", BN);
  static std::once_flag attr;
  std::call_once(attr, [] {
    cudaFuncSetAttribute(matmul_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(matmul_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(matmul_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES);
  });
  if (tc_mode() == 2) {
    CUtensorMap ta2, tb2;
    int rc2 = make_map(&ta2, c->in[0].ptr, n, n, BK, 128);  // A: box 32 (k) x 128 (m)
    if (rc2) return rc2;
    rc2 = make_map_bmn_half(&tb2, c->in[1].ptr, n);
    if (rc2) return rc2;
    const int ntiles2 = (n / BM2) * (n / BN);
    const int pairs = ntiles2 < c->sm_count / 2 ? ntiles2 : c->sm_count / 2;
    matmul_tc2_kernel<<<2 * pairs, 192, SMEM2_BYTES, c->stream>>>(ta2, tb2, (float*)c->out[0].ptr, n);
    return PS_OK;
  }
  const int ntiles = (n / BM) * (n / BN);
  const int grid = ntiles < c->sm_count ? ntiles : c->sm_count;
  CUtensorMap ta, tb;
  int rc = make_map(&ta, c->in[0].ptr, n, n, BK, BM);  // A [m][k]: box 32 (k) x 128 (m)
  if (rc) return rc;
  if (b_n_major()) {
    rc = make_map_bmn(&tb, c->in[1].ptr, n);
    if (rc) return rc;
    matmul_tc_kernel<true><<<grid, 192, SMEM_BYTES, c->stream>>>(ta, tb, (float*)c->out[0].ptr, n);
    return PS_OK;
  }
  DevBuf& bt = c->scratch[7];
  if (int rc2 = c->ensure(bt, size_t(n) * n * sizeof(float))) return rc2;
  rc = make_map(&tb, bt.ptr, n, n, BK, BN);            // Bt [n][k]: box 32 (k) x 256 (n)
  if (rc) return rc;
  transpose_f32<<<dim3(n / 32, n / 32), 256, 0, c->stream>>>((const float*)c->in[1].ptr,
                                                             (float*)bt.ptr, n);
  matmul_tc_kernel<false><<<grid, 192, SMEM_BYTES, c->stream>>>(ta, tb, (float*)c->out[0].ptr, n);
  return PS_OK;
}

}  // namespace ps
