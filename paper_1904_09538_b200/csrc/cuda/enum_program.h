/* Flat enumeration program for the GPU brute-force counter (
 * reference oracle.cpp:76-443). Built host-side from a kernel IR at concrete
 * bindings (csrc/host/ps_enumerate_gpu.cpp), run by csrc/cuda/enum.cu.
 * Plain C so both g++ and nvcc share it. */
#pragma once
#include <stdint.h>

#define PS_ENUM_MAXD 10 /* loop levels of one nest (statement inames + reduction binders) */
#define PS_ENUM_MAXR 4  /* array rank */

/* A loop nest: level d runs over [lo_d, hi_d], both affine in the outer
 * levels: v = c[PS_ENUM_MAXD] + sum_{e<d} c[e] * x_e. The box bounds the
 * levels for the flat thread index; points outside lo/hi are skipped. */
typedef struct {
  int depth;
  int64_t lo[PS_ENUM_MAXD][PS_ENUM_MAXD + 1];
  int64_t hi[PS_ENUM_MAXD][PS_ENUM_MAXD + 1];
  int64_t box_lo[PS_ENUM_MAXD];
  int64_t box_ext[PS_ENUM_MAXD];
} ps_enum_nest;

/* An access site visited once per point of its nest: rank subscripts, each
 * affine in the nest levels; the flat row-major index marks two bitmaps (its
 * pattern-group x array footprint and the array's footprint). */
typedef struct {
  int nest;
  int rank;
  int bitmap_group;
  int bitmap_array;
  int64_t sub[PS_ENUM_MAXR][PS_ENUM_MAXD + 1];
  int64_t dim[PS_ENUM_MAXR];
} ps_enum_site;

typedef struct {
  int n_nests;
  const ps_enum_nest* nests;
  int n_sites;
  const ps_enum_site* sites;
  int n_bitmaps;
  const int64_t* bitmap_bits; /* bits (array elements) per bitmap */
} ps_enum_program;

#ifdef __cplusplus
extern "C" {
#endif
struct ps_ctx;
/* nest_points[n_nests], bitmap_pop[n_bitmaps]; returns a ps status code. */
int ps_enum_gpu_run(struct ps_ctx* ctx, const ps_enum_program* prog, int64_t* nest_points,
                    int64_t* bitmap_pop);
#ifdef __cplusplus
}
#endif
