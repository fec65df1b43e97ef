// Shared helpers for the sm_100a kernels: error state, geometry, keys, hashing.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <string>

#include "sparseconv_b200.h"

namespace scb {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);

#define SCB_CHECK_ARG(cond, msg)                                   \
  do {                                                             \
    if (!(cond)) {                                                 \
      ::scb::set_error(std::string(__func__) + ": " + (msg));      \
      return SCB_EINVAL;                                           \
    }                                                              \
  } while (0)

#define SCB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t err_ = (call);                                                      \
    if (err_ != cudaSuccess) {                                                      \
      ::scb::set_error(std::string(__func__) + ": " #call ": " + cudaGetErrorString(err_)); \
      return SCB_ECUDA;                                                             \
    }                                                                               \
  } while (0)

// Every kernel launch site of the library is followed by SCB_LAUNCHED(), which
// checks the launch and bumps the process-wide launch counter
// (scb_launch_count, used by bench.py's gpu_launches).
void count_launch();
#define SCB_LAUNCHED()          \
  do {                          \
    ::scb::count_launch();      \
    SCB_CUDA(cudaGetLastError()); \
  } while (0)

inline cudaStream_t as_stream(scb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------ geometry
// Device-side copy of scb_grid_t passed by value to kernels.
struct Grid {
  int dim;
  long long batch;
  long long ext[4];
};

inline Grid to_grid(const scb_grid_t* g) {
  Grid r;
  r.dim = g->dim;
  r.batch = g->batch_size;
  for (int d = 0; d < 4; ++d) r.ext[d] = d < g->dim ? g->extent[d] : 1;
  return r;
}

inline long long total_cells(const Grid& g) {
  long long t = g.batch;
  for (int d = 0; d < g.dim; ++d) t *= g.ext[d];
  return t;
}

constexpr long long EMPTY_KEY = -1;

// Batch-major flat key (core.py:46-66) of a coordinate known to be in bounds.
template <int D>
__device__ __forceinline__ long long flat_key(const int* c, const Grid& g) {
  long long k = c[0];
#pragma unroll
  for (int d = 0; d < D; ++d) k = k * g.ext[d] + c[d + 1];
  return k;
}

template <int D>
__device__ __forceinline__ bool in_bounds(const int* c, const Grid& g) {
  if (c[0] < 0 || c[0] >= g.batch) return false;
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (c[d + 1] < 0 || c[d + 1] >= g.ext[d]) return false;
  return true;
}

// 64-bit finaliser (murmur3 fmix64); the slot layout never reaches any
// output, only probe lengths.
__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// Lexicographic offset n of a K^D window (mapping.py:63-79): digit of dim 0 is
// most significant; `lo` is the window base (-(K-1)/2 for odd K, the
// reference's EVEN_KERNEL_OFFSET_BASE = 0 for even K, mapping.py:26).
template <int D>
__device__ __forceinline__ void offset_of(int n, int K, int lo, int* delta) {
#pragma unroll
  for (int d = D - 1; d >= 0; --d) {
    delta[d] = lo + n % K;
    n /= K;
  }
}

// Look a (possibly out-of-bounds) coordinate up in the index.  Returns the
// row or -1 (MISS).
template <int D>
__device__ __forceinline__ int index_lookup(int kind, const int* c, const Grid& g,
                                            const long long* __restrict__ keys,
                                            const int* __restrict__ rows,
                                            unsigned long long mask) {
  if (!in_bounds<D>(c, g)) return -1;
  const long long key = flat_key<D>(c, g);
  if (kind == SCB_INDEX_GRID) return __ldg(rows + key);
  unsigned long long slot = mix64((unsigned long long)key) & mask;
  while (true) {
    const long long k = __ldg(keys + slot);
    if (k == key) return __ldg(rows + slot);
    if (k == EMPTY_KEY) return -1;
    slot = (slot + 1) & mask;
  }
}

inline int ceil_div_i(long long a, long long b) { return (int)((a + b - 1) / b); }

// Row stride of a [V][n] hit matrix: n rounded up to 4 entries so every row
// starts 16-byte aligned (1-D TMA loads of a tile's neighbour rows need it).
__host__ __device__ __forceinline__ long long hits_ld(long long n) { return (n + 3) & ~3LL; }

// GEMM problem table of one layer (segments = scheduled offsets + centre).
// Built on the host (scb_grouped_gemm) or on the device straight from a hit
// matrix (scb_plan_from_hits), in which case the GEMM reads it from global
// memory and no map size ever crosses to the host.
struct SegDesc {
  long long a_row, c_row;
  int rows, b_index, a_src, _pad;
};
struct SegTable {
  int n_segs, total_tiles;
  long long rows_pad;  // gather-buffer rows in use (device-built tables)
  int tile_start[SCB_MAX_SEGMENTS + 1];
  SegDesc seg[SCB_MAX_SEGMENTS];
};

// Dispatch on the spatial rank.
#define SCB_DISPATCH_DIM(dim, ...)          \
  switch (dim) {                            \
    case 1: { constexpr int D = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int D = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int D = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int D = 4; __VA_ARGS__; } break; \
    default: set_error("spatial rank must be between 1 and 4"); return SCB_EINVAL; \
  }

}  // namespace scb
