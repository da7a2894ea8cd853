// GPU brute-force counter: every point of every loop nest is
// one thread-index in a grid-stride loop; points are counted (warp-reduced
// atomics) and every access site of the nest sets its element's bit in two
// footprint bitmaps (atomicOr), popcounted at the end. Exact integer work,
// no floating point; the host folds the tallies into OracleCounts
// (csrc/host/ps_enumerate_gpu.cpp).
#include <vector>

#include "enum_program.h"
#include "runtime_internal.h"

namespace ps {
namespace {

__device__ __forceinline__ int64_t affine_at(const int64_t* c, const int64_t* x, int n) {
  int64_t v = c[PS_ENUM_MAXD];
  for (int e = 0; e < n; ++e) v += c[e] * x[e];
  return v;
}

__global__ void __launch_bounds__(256) enum_nest_kernel(const ps_enum_nest* __restrict__ nest,
                                                        const ps_enum_site* __restrict__ sites,
                                                        int site_begin, int site_end, int64_t volume,
                                                        unsigned long long* __restrict__ points,
                                                        unsigned int* const* __restrict__ bitmaps,
                                                        unsigned int* __restrict__ oob) {
  __shared__ ps_enum_nest sn;
  if (threadIdx.x == 0) sn = *nest;
  __syncthreads();
  unsigned long long local = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < volume; t += stride) {
    int64_t x[PS_ENUM_MAXD];
    int64_t r = t;
    for (int d = sn.depth - 1; d >= 0; --d) {  // innermost level fastest
      x[d] = sn.box_lo[d] + r % sn.box_ext[d];
      r /= sn.box_ext[d];
    }
    bool in = true;
    for (int d = 0; d < sn.depth && in; ++d)
      in = x[d] >= affine_at(sn.lo[d], x, d) && x[d] <= affine_at(sn.hi[d], x, d);
    if (!in) continue;
    ++local;
    for (int si = site_begin; si < site_end; ++si) {
      const ps_enum_site& s = sites[si];
      int64_t flat = 0;
      bool ok = true;
      for (int q = 0; q < s.rank; ++q) {
        const int64_t v = affine_at(s.sub[q], x, sn.depth);
        ok = ok && v >= 0 && v < s.dim[q];
        flat = flat * s.dim[q] + v;
      }
      if (!ok) {
        atomicOr(oob, 1u);
        continue;
      }
      atomicOr(bitmaps[s.bitmap_group] + (flat >> 5), 1u << (flat & 31));
      atomicOr(bitmaps[s.bitmap_array] + (flat >> 5), 1u << (flat & 31));
    }
  }
  // warp-reduce the point count, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(points, local);
}

__global__ void popcount_kernel(const unsigned int* __restrict__ bits, int64_t words,
                                unsigned long long* __restrict__ out) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x)
    local += __popc(bits[i]);
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

#define ENUM_CUDA(x)                                                              \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      for (void* p : owned) cudaFree(p);                                          \
      return set_error(PS_ERR_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
    }                                                                             \
  } while (0)

}  // namespace
}  // namespace ps

extern "C" int ps_enum_gpu_run(ps_ctx* ctx, const ps_enum_program* prog, int64_t* nest_points,
                               int64_t* bitmap_pop) {
  using namespace ps;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !prog) return set_error(PS_ERR_ARG, "ps_enum_gpu_run: null argument");
  cudaStream_t st = c->stream;
  std::vector<void*> owned;
  auto alloc = [&](size_t bytes, void** p) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
    if (e == cudaSuccess) owned.push_back(*p);
    return e;
  };
  ps_enum_nest* d_nests = nullptr;
  ps_enum_site* d_sites = nullptr;
  unsigned long long* d_counts = nullptr;  // [n_nests] points, then [n_bitmaps] popcounts
  unsigned int* d_oob = nullptr;
  unsigned int** d_bitmap_ptrs = nullptr;
  ENUM_CUDA(alloc(sizeof(ps_enum_nest) * prog->n_nests, (void**)&d_nests));
  ENUM_CUDA(alloc(sizeof(ps_enum_site) * prog->n_sites, (void**)&d_sites));
  ENUM_CUDA(alloc(sizeof(unsigned long long) * (prog->n_nests + prog->n_bitmaps),
                  (void**)&d_counts));
  ENUM_CUDA(alloc(sizeof(unsigned int), (void**)&d_oob));
  std::vector<unsigned int*> bm(prog->n_bitmaps, nullptr);
  for (int i = 0; i < prog->n_bitmaps; ++i) {
    const size_t words = (size_t)((prog->bitmap_bits[i] + 31) / 32);
    ENUM_CUDA(alloc(words * 4, (void**)&bm[i]));
    ENUM_CUDA(cudaMemsetAsync(bm[i], 0, words * 4, st));
  }
  ENUM_CUDA(alloc(sizeof(unsigned int*) * (prog->n_bitmaps ? prog->n_bitmaps : 1),
                  (void**)&d_bitmap_ptrs));
  ENUM_CUDA(cudaMemcpyAsync(d_nests, prog->nests, sizeof(ps_enum_nest) * prog->n_nests,
                            cudaMemcpyHostToDevice, st));
  ENUM_CUDA(cudaMemcpyAsync(d_sites, prog->sites, sizeof(ps_enum_site) * prog->n_sites,
                            cudaMemcpyHostToDevice, st));
  ENUM_CUDA(cudaMemcpyAsync(d_bitmap_ptrs, bm.data(), sizeof(unsigned int*) * prog->n_bitmaps,
                            cudaMemcpyHostToDevice, st));
  ENUM_CUDA(cudaMemsetAsync(d_counts, 0,
                            sizeof(unsigned long long) * (prog->n_nests + prog->n_bitmaps), st));
  ENUM_CUDA(cudaMemsetAsync(d_oob, 0, sizeof(unsigned int), st));
  // sites are grouped by nest in the program (host guarantees ascending nest)
  int s0 = 0;
  for (int n = 0; n < prog->n_nests; ++n) {
    int s1 = s0;
    while (s1 < prog->n_sites && prog->sites[s1].nest == n) ++s1;
    int64_t volume = 1;
    for (int d = 0; d < prog->nests[n].depth; ++d) volume *= prog->nests[n].box_ext[d];
    if (volume > 0) {
      const int64_t blocks64 = (volume + 255) / 256;
      const int blocks = (int)(blocks64 < (int64_t)c->sm_count * 64 ? blocks64 : (int64_t)c->sm_count * 64);
      enum_nest_kernel<<<blocks, 256, 0, st>>>(d_nests + n, d_sites, s0, s1, volume, d_counts + n,
                                               d_bitmap_ptrs, d_oob);
      ENUM_CUDA(cudaGetLastError());
    }
    s0 = s1;
  }
  for (int i = 0; i < prog->n_bitmaps; ++i) {
    const int64_t words = (prog->bitmap_bits[i] + 31) / 32;
    popcount_kernel<<<c->sm_count * 4, 256, 0, st>>>(bm[i], words, d_counts + prog->n_nests + i);
    ENUM_CUDA(cudaGetLastError());
  }
  std::vector<unsigned long long> h(prog->n_nests + prog->n_bitmaps);
  unsigned int oob = 0;
  ENUM_CUDA(cudaMemcpyAsync(h.data(), d_counts, sizeof(unsigned long long) * h.size(),
                            cudaMemcpyDeviceToHost, st));
  ENUM_CUDA(cudaMemcpyAsync(&oob, d_oob, sizeof(oob), cudaMemcpyDeviceToHost, st));
  ENUM_CUDA(cudaStreamSynchronize(st));
  for (void* p : owned) cudaFree(p);
  if (oob) return set_error(PS_ERR_ARG, "enumeration: an access subscript leaves its array bounds");
  for (int n = 0; n < prog->n_nests; ++n) nest_points[n] = (int64_t)h[n];
  for (int i = 0; i < prog->n_bitmaps; ++i) bitmap_pop[i] = (int64_t)h[prog->n_nests + i];
  return PS_OK;
}
