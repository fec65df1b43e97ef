// Point cloud -> sparse voxels on the device (reference core.py:174-216,
// SURVEY.md §8(f) row 2): the step in front of the hot path, so a batch of
// raw scans never round-trips through host numpy.  A batch of B scans is
// voxelised in one pass into one packed tensor: scan b is voxelised exactly
// as the reference voxelises it alone (its own min corner), gets batch
// column b, and the boundary is the per-dimension max over the scans (the
// packing the bench and SURVEY.md §8(e) use; bit-identical to B separate
// calls + concatenation).
//
//   cells = floor((p - min_corner[b]) / voxel_size)     (f64, like numpy)
//   boundary = max_b max(cells) + 1, key = flat(b, cells)
//   stable radix sort of (key, point index) -> runs of equal keys = voxels,
//   ascending key order (np.unique order)
//   reduce "mean": f64 sum of each voxel's points in point order (what
//   np.bincount accumulates), / count, one round to f32; "first": the
//   voxel's first point in input order.
//
// Bit-exact with the reference: the same f64 operations in the same order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace scb {
namespace vox {

// Order-preserving map of doubles onto unsigned 64-bit integers (for atomicMin).
__device__ __forceinline__ unsigned long long ordered(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unordered(unsigned long long u) {
  const unsigned long long b = (u & 0x8000000000000000ull) ? (u & ~0x8000000000000000ull) : ~u;
  return __longlong_as_double((long long)b);
}

// Scan b's points are [scan_ptr[b], scan_ptr[b + 1]) (scan_ptr NULL: one
// scan of n points).  Kernels over points run blockIdx.y = scan, so the scan
// of a point is block-uniform and the min / max reductions stay warp-local.
__device__ __forceinline__ void scan_range(const long long* __restrict__ scan_ptr, long long n,
                                           long long& lo, long long& hi) {
  const int b = blockIdx.y;
  lo = scan_ptr ? __ldg(scan_ptr + b) : 0;
  hi = scan_ptr ? __ldg(scan_ptr + b + 1) : n;
}

__global__ void init_kernel(unsigned long long* mins, long long* maxs, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    mins[i] = ~0ull;
    maxs[i] = 0;
  }
}

// per-scan minimum corner: mins[b][d]
__global__ void min_kernel(const double* __restrict__ pts, long long n, int cols, int dims,
                           const long long* __restrict__ scan_ptr, unsigned long long* mins) {
  long long lo, hi;
  scan_range(scan_ptr, n, lo, hi);
  for (int d = 0; d < dims; ++d) {
    unsigned long long m = ~0ull;
    for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
         i += (long long)gridDim.x * blockDim.x)
      m = min(m, ordered(pts[i * cols + d]));
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMin(mins + blockIdx.y * dims + d, m);
  }
}

// cells (kept in `cell`, [n][dims]) and their per-scan, per-dimension maxima
__global__ void cells_kernel(const double* __restrict__ pts, long long n, int cols, int dims,
                             double voxel, const long long* __restrict__ scan_ptr,
                             const unsigned long long* mins, long long* __restrict__ cell,
                             long long* maxs) {
  long long lo, hi;
  scan_range(scan_ptr, n, lo, hi);
  for (int d = 0; d < dims; ++d) {
    const double base = unordered(mins[blockIdx.y * dims + d]);
    long long m = 0;
    for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
         i += (long long)gridDim.x * blockDim.x) {
      const double q = __ddiv_rn(__dsub_rn(pts[i * cols + d], base), voxel);
      const long long c = (long long)floor(q);
      cell[i * dims + d] = c;
      m = max(m, c);
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
      atomicMax((unsigned long long*)(maxs + blockIdx.y * dims + d), (unsigned long long)m);
  }
}

// shared boundary: ext[d] = max over scans of (max cell + 1)
__global__ void extent_kernel(const long long* maxs, int B, int dims, long long* ext) {
  const int d = threadIdx.x;
  if (d < dims) {
    long long e = 0;
    for (int b = 0; b < B; ++b) e = max(e, maxs[b * dims + d] + 1);
    ext[d] = e;
  }
}

// key = flat(batch = scan, cells) over the shared boundary
__global__ void keys_kernel(const long long* __restrict__ cell, long long n, int dims,
                            const long long* __restrict__ scan_ptr, const long long* ext,
                            unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  long long lo, hi;
  scan_range(scan_ptr, n, lo, hi);
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
       i += (long long)gridDim.x * blockDim.x) {
    long long k = blockIdx.y;
    for (int d = 0; d < dims; ++d) k = k * ext[d] + cell[i * dims + d];
    keys[i] = (unsigned long long)k;
    idx[i] = (int)i;
  }
}

// one thread per voxel: run [start, start + count) of the sorted points
__global__ void reduce_kernel(const double* __restrict__ pts, int cols, int dims,
                              const int* __restrict__ sidx, const int* __restrict__ counts,
                              const int* __restrict__ starts, const long long* n_vox,
                              int first, float* __restrict__ out) {
  const int C = cols - dims;
  const long long nv = *n_vox;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    const int s = starts[v], cnt = counts[v];
    for (int c = 0; c < C; ++c) {
      double acc;
      if (first) {
        acc = pts[(long long)sidx[s] * cols + dims + c];
      } else {
        acc = 0.0;
        for (int j = 0; j < cnt; ++j) acc = __dadd_rn(acc, pts[(long long)sidx[s + j] * cols + dims + c]);
        acc = __ddiv_rn(acc, (double)cnt);
      }
      out[v * C + c] = (float)acc;
    }
  }
}

__global__ void coords_kernel(const unsigned long long* __restrict__ ukeys, const long long* n_vox,
                              int dims, const long long* ext, int* __restrict__ coords,
                              long long* __restrict__ meta) {
  const long long nv = *n_vox;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    long long r = (long long)ukeys[v];
    for (int d = dims - 1; d >= 0; --d) {
      const long long b = ext[d];
      coords[v * (dims + 1) + d + 1] = (int)(r % b);
      r /= b;
    }
    coords[v * (dims + 1)] = (int)r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    meta[0] = nv;
    for (int d = 0; d < dims; ++d) meta[1 + d] = ext[d];
  }
}

struct Ws {
  size_t mins, maxs, ext, cell, keys, keys2, idx, idx2, ukeys, counts, starts, nvox, tmp, total;
};

static Ws layout(long long n, int dims, int B = 64) {
  auto r = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t sort_tmp = 0, rle_tmp = 0, scan_tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr,
                                  (int64_t)n);
  cub::DeviceRunLengthEncode::Encode(nullptr, rle_tmp, (unsigned long long*)nullptr,
                                     (unsigned long long*)nullptr, (int*)nullptr,
                                     (long long*)nullptr, (int64_t)n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (int*)nullptr, (int*)nullptr, (int64_t)n);
  Ws w{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += r(bytes); return o; };
  w.mins = take(8 * (size_t)B * 4);
  w.maxs = take(8 * (size_t)B * 4);
  w.ext = take(8 * 4);
  w.cell = take((size_t)n * dims * 8);
  w.keys = take((size_t)n * 8);
  w.keys2 = take((size_t)n * 8);
  w.idx = take((size_t)n * 4);
  w.idx2 = take((size_t)n * 4);
  w.ukeys = take((size_t)n * 8);
  w.counts = take((size_t)n * 4);
  w.starts = take((size_t)n * 4);
  w.nvox = take(8);
  w.tmp = take(std::max(sort_tmp, std::max(rle_tmp, scan_tmp)));
  w.total = off;
  return w;
}

}  // namespace vox
}  // namespace scb

using namespace scb;

extern "C" int64_t scb_voxelize_workspace(int64_t n_points, int32_t spatial_dims) {
  return (int64_t)vox::layout(n_points, spatial_dims).total;
}

extern "C" int32_t scb_voxelize_batch(const double* points, const int64_t* scan_ptr,
                                      int32_t n_scans, int64_t n_points, int32_t cols,
                                      int32_t spatial_dims, double voxel_size,
                                      int32_t reduce_first, void* workspace, int64_t ws_bytes,
                                      int32_t* out_coords, float* out_features, int64_t* meta,
                                      scb_stream_t stream) {
  using namespace vox;
  SCB_CHECK_ARG(n_points > 0, "empty cloud");
  SCB_CHECK_ARG(n_scans >= 1 && n_scans <= 64, "1..64 scans per batch");
  SCB_CHECK_ARG(n_scans == 1 || scan_ptr != nullptr, "scan offsets required for a batch");
  SCB_CHECK_ARG(spatial_dims >= 1 && spatial_dims <= 4, "spatial rank must be between 1 and 4");
  SCB_CHECK_ARG(cols >= spatial_dims, "points need at least spatial_dims columns");
  SCB_CHECK_ARG(voxel_size > 0, "voxel_size must be positive");
  SCB_CHECK_ARG(n_points < (1LL << 31), "too many points");
  Ws w = layout(n_points, spatial_dims);
  SCB_CHECK_ARG(ws_bytes >= (int64_t)w.total, "workspace too small");
  cudaStream_t s = as_stream(stream);
  char* b = (char*)workspace;
  auto* mins = (unsigned long long*)(b + w.mins);
  auto* maxs = (long long*)(b + w.maxs);
  auto* ext = (long long*)(b + w.ext);
  auto* cell = (long long*)(b + w.cell);
  auto* keys = (unsigned long long*)(b + w.keys);
  auto* keys2 = (unsigned long long*)(b + w.keys2);
  auto* idx = (int*)(b + w.idx);
  auto* idx2 = (int*)(b + w.idx2);
  auto* ukeys = (unsigned long long*)(b + w.ukeys);
  auto* counts = (int*)(b + w.counts);
  auto* starts = (int*)(b + w.starts);
  auto* nvox = (long long*)(b + w.nvox);
  void* tmp = b + w.tmp;
  const long long* sp = (const long long*)scan_ptr;
  const int grid = (int)std::min<long long>((n_points + 255) / 256, 1184);
  // point kernels: blockIdx.y = scan, x blocks over the largest scan's share
  const dim3 pgrid((unsigned)std::max(1, (int)std::min<long long>(
                       (n_points / n_scans + 255) / 256 + 1, 1184 / n_scans + 1)),
                   (unsigned)n_scans);
  init_kernel<<<1, 256, 0, s>>>(mins, maxs, n_scans * spatial_dims);
  SCB_CUDA(cudaMemsetAsync(counts, 0, (size_t)n_points * sizeof(int), s));
  min_kernel<<<pgrid, 256, 0, s>>>(points, n_points, cols, spatial_dims, sp, mins);
  cells_kernel<<<pgrid, 256, 0, s>>>(points, n_points, cols, spatial_dims, voxel_size, sp, mins,
                                     cell, maxs);
  extent_kernel<<<1, 32, 0, s>>>(maxs, n_scans, spatial_dims, ext);
  keys_kernel<<<pgrid, 256, 0, s>>>(cell, n_points, spatial_dims, sp, ext, keys, idx);
  SCB_LAUNCHED();
  size_t tb = w.total - w.tmp;
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, idx, idx2, (int64_t)n_points, 0,
                                           63, s));
  tb = w.total - w.tmp;
  SCB_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, tb, keys2, ukeys, counts, (long long*)nvox,
                                              (int64_t)n_points, s));
  tb = w.total - w.tmp;
  SCB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, starts, (int64_t)n_points, s));
  reduce_kernel<<<grid, 256, 0, s>>>(points, cols, spatial_dims, idx2, counts, starts, nvox,
                                     reduce_first, out_features);
  coords_kernel<<<grid, 256, 0, s>>>(ukeys, nvox, spatial_dims, ext, out_coords,
                                     (long long*)meta);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_voxelize(const double* points, int64_t n_points, int32_t cols,
                                int32_t spatial_dims, double voxel_size, int32_t reduce_first,
                                void* workspace, int64_t ws_bytes, int32_t* out_coords,
                                float* out_features, int64_t* meta, scb_stream_t stream) {
  return scb_voxelize_batch(points, nullptr, 1, n_points, cols, spatial_dims, voxel_size,
                            reduce_first, workspace, ws_bytes, out_coords, out_features, meta,
                            stream);
}
