// Kernel-map construction on sm_100a: coordinate index (hash / grid), strided
// output coordinates, map search, per-offset compaction, transposed maps and
// the gather/scatter plan.  Everything here is integer work and bit-exact
// w.r.t. the reference (mapping.py); see DESIGN.md §3.
#include <cub/cub.cuh>

#include "common.cuh"

namespace scb {

// =================================================================== index

template <int D>
__global__ void hash_build_kernel(const int* __restrict__ coords, long long n, Grid g,
                                  unsigned long long* keys, int* rows, unsigned long long mask,
                                  int* status) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int c[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) c[d] = coords[i * (D + 1) + d];
    if (!in_bounds<D>(c, g)) {
      atomicAdd(status + 1, 1);
      continue;
    }
    const unsigned long long key = (unsigned long long)flat_key<D>(c, g);
    unsigned long long slot = mix64(key) & mask;
    while (true) {
      const unsigned long long prev = atomicCAS(keys + slot, (unsigned long long)EMPTY_KEY, key);
      if (prev == (unsigned long long)EMPTY_KEY) {
        rows[slot] = (int)i;
        break;
      }
      if (prev == key) {  // duplicate coordinate row
        atomicAdd(status, 1);
        break;
      }
      slot = (slot + 1) & mask;
    }
  }
}

template <int D>
__global__ void grid_build_kernel(const int* __restrict__ coords, long long n, Grid g, int* table,
                                  int* status) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int c[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) c[d] = coords[i * (D + 1) + d];
    if (!in_bounds<D>(c, g)) {
      atomicAdd(status + 1, 1);
      continue;
    }
    if (atomicCAS(table + flat_key<D>(c, g), -1, (int)i) != -1) atomicAdd(status, 1);
  }
}

template <int D>
__global__ void index_query_kernel(int kind, const int* __restrict__ probes, long long n, Grid g,
                                   const long long* __restrict__ keys,
                                   const int* __restrict__ rows, unsigned long long mask,
                                   int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int c[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) c[d] = probes[i * (D + 1) + d];
    out[i] = index_lookup<D>(kind, c, g, keys, rows, mask);
  }
}

static int grid_blocks(long long n, int threads, int cap = 148 * 16) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

}  // namespace scb

using namespace scb;

extern "C" int64_t scb_hits_ld(int64_t n) { return hits_ld(n); }

extern "C" int64_t scb_hash_slots(int64_t n) {
  int64_t t = 2;
  while (t < 2 * (n > 1 ? n : 1)) t *= 2;
  return t;
}

extern "C" int32_t scb_index_build(int32_t kind, const int32_t* coords, int64_t n,
                                   const scb_grid_t* grid, int64_t* table_keys,
                                   int32_t* table_rows, int64_t slots, int32_t* status,
                                   scb_stream_t stream) {
  SCB_CHECK_ARG(grid && grid->dim >= 1 && grid->dim <= 4, "bad grid");
  Grid g = to_grid(grid);
  cudaStream_t s = as_stream(stream);
  SCB_CUDA(cudaMemsetAsync(status, 0, 2 * sizeof(int32_t), s));
  if (kind == SCB_INDEX_HASH) {
    SCB_CHECK_ARG(slots >= 2 && (slots & (slots - 1)) == 0, "slots must be a power of two");
    SCB_CHECK_ARG(slots >= n, "hash table smaller than the key count");
    SCB_CUDA(cudaMemsetAsync(table_keys, 0xFF, slots * sizeof(int64_t), s));
    if (n == 0) return SCB_OK;
    SCB_DISPATCH_DIM(g.dim, hash_build_kernel<D><<<grid_blocks(n, 256), 256, 0, s>>>(
                                coords, n, g, (unsigned long long*)table_keys, table_rows,
                                (unsigned long long)(slots - 1), status));
  } else if (kind == SCB_INDEX_GRID) {
    SCB_CHECK_ARG(slots >= total_cells(g), "grid table smaller than the cell count");
    SCB_CUDA(cudaMemsetAsync(table_rows, 0xFF, total_cells(g) * sizeof(int32_t), s));
    if (n == 0) return SCB_OK;
    SCB_DISPATCH_DIM(g.dim, grid_build_kernel<D><<<grid_blocks(n, 256), 256, 0, s>>>(
                                coords, n, g, table_rows, status));
  } else {
    SCB_CHECK_ARG(false, "unknown index kind");
  }
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_index_query(int32_t kind, const int32_t* probes, int64_t n,
                                   const scb_grid_t* grid, const int64_t* table_keys,
                                   const int32_t* table_rows, int64_t slots, int32_t* rows_out,
                                   scb_stream_t stream) {
  SCB_CHECK_ARG(grid && grid->dim >= 1 && grid->dim <= 4, "bad grid");
  if (n == 0) return SCB_OK;
  Grid g = to_grid(grid);
  SCB_DISPATCH_DIM(g.dim, index_query_kernel<D><<<grid_blocks(n, 256), 256, 0, as_stream(stream)>>>(
                              kind, probes, n, g, (const long long*)table_keys, table_rows,
                              (unsigned long long)(slots - 1), rows_out));
  SCB_LAUNCHED();
  return SCB_OK;
}

// =================================================================== output coordinates

namespace scb {

static int cand_per_input(int dim, int K, int s) {
  int per_dim = (K + s - 1) / s;
  int c = 1;
  for (int d = 0; d < dim; ++d) c *= per_dim;
  return c;
}

// Fused stages 1-4 of the downsampling pipeline (mapping.py:237-247): every
// input proposes u = p - delta per offset, kept iff u % s == 0, 0 <= u and
// u < s * b_out; survivors are flattened over the output grid.  Empty slots
// get the sentinel (total output cells), which sorts last.  KT: the key type
// the candidates are sorted in (32-bit whenever the sentinel fits).
template <int D, typename KT>
__device__ __forceinline__ void propose(const int* p, const Grid& gout, int K, int lo, int s,
                                       int cap, KT sentinel, KT* __restrict__ out) {
  int w = 0;
  if (K == s) {
    // one candidate per input: per dimension the single delta in
    // [lo, lo + K) with (p - delta) % s == 0
    bool keep = true;
    long long key = p[0];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      int r = (p[d + 1] - lo) % s;
      r += r < 0 ? s : 0;
      const int u = p[d + 1] - lo - r;
      keep = keep && u >= 0 && u < s * gout.ext[d];
      key = key * gout.ext[d] + (u >= 0 ? u / s : 0);
    }
    if (keep && cap > 0) out[w++] = (KT)key;
  } else {
    // per dimension the valid coarse coordinates q = (p - delta) / s, delta in
    // [lo, lo + K), (p - delta) % s == 0, 0 <= q < ext, form one contiguous
    // range: q_max = floor((p - lo) / s) and the (K - 1 - r) / s below it
    // (r = (p - lo) mod s), clipped to the grid -- one division per dimension
    // instead of the K^D offset walk's; the candidates are the ranges'
    // Cartesian product (their order is irrelevant: sorted and deduplicated next)
    int qlo[D], qhi[D];
    bool any = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int x = p[d + 1] - lo;
      int r = x % s;
      r += r < 0 ? s : 0;
      const int q = (x - r) / s;
      qhi[d] = (int)min((long long)q, (long long)gout.ext[d] - 1);
      qlo[d] = max(r <= K - 1 ? q - (K - 1 - r) / s : q + 1, 0);
      any = any && qlo[d] <= qhi[d];
    }
    if (any) {
      int idx[D];
#pragma unroll
      for (int d = 0; d < D; ++d) idx[d] = qlo[d];
      while (w < cap) {
        long long key = p[0];
#pragma unroll
        for (int d = 0; d < D; ++d) key = key * gout.ext[d] + idx[d];
        out[w++] = (KT)key;
        int d = D - 1;   // odometer over the per-dimension ranges
        for (; d >= 0; --d) {
          if (++idx[d] <= qhi[d]) break;
          idx[d] = qlo[d];
        }
        if (d < 0) break;
      }
    }
  }
  for (; w < cap; ++w) out[w] = sentinel;
}

template <int D, typename KT>
__global__ void out_candidates_kernel(const int* __restrict__ coords, long long n, Grid gout,
                                      int K, int lo, int s, int cap, KT sentinel,
                                      KT* __restrict__ cand) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int p[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) p[d] = coords[i * (D + 1) + d];
    propose<D, KT>(p, gout, K, lo, s, cap, sentinel, cand + i * cap);
  }
}

// The same candidates from the previous level's sorted unique keys (input
// grid `gin`), for the first *n_dev of n_cap rows; rows past the live count
// propose only sentinels.  Lets a chain of strided levels run with the
// counts on the device (one host read for the whole chain).
template <int D, typename KT>
__global__ void out_candidates_keys_kernel(const unsigned long long* __restrict__ keys,
                                           const long long* __restrict__ n_dev, long long n_cap,
                                           Grid gin, Grid gout, int K, int lo, int s, int cap,
                                           KT sentinel, KT* __restrict__ cand) {
  const long long n = *n_dev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_cap;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < n) {
      long long r = (long long)keys[i];
      int p[D + 1];
#pragma unroll
      for (int d = D - 1; d >= 0; --d) {
        p[d + 1] = (int)(r % gin.ext[d]);
        r /= gin.ext[d];
      }
      p[0] = (int)r;
      propose<D, KT>(p, gout, K, lo, s, cap, sentinel, cand + i * cap);
    } else {
      for (int w = 0; w < cap; ++w) cand[i * cap + w] = sentinel;
    }
  }
}

// Sorted unique 32-bit keys -> the int64 output keys, dropping the sentinel.
__global__ void widen_keys_kernel(const uint32_t* __restrict__ uniq, long long* __restrict__ count,
                                  uint32_t sentinel, unsigned long long* __restrict__ out,
                                  long long cap) {
  const long long c = *count;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < c) out[i] = uniq[i];
  }
}

__global__ void drop_sentinel_kernel(const unsigned long long* uniq, long long* count,
                                     unsigned long long sentinel) {
  long long c = *count;
  if (c > 0 && uniq[c - 1] == sentinel) *count = c - 1;
}
__global__ void drop_sentinel_kernel32(const uint32_t* uniq, long long* count, uint32_t sentinel) {
  long long c = *count;
  if (c > 0 && uniq[c - 1] == sentinel) *count = c - 1;
}

template <int D>
__global__ void unflatten_kernel(const long long* __restrict__ keys, long long n, Grid g,
                                 int* __restrict__ coords) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = keys[i];
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      coords[i * (D + 1) + d + 1] = (int)(r % g.ext[d]);
      r /= g.ext[d];
    }
    coords[i * (D + 1)] = (int)r;
  }
}

struct OutCoordWs {
  size_t cand_bytes, sort_tmp, uniq_tmp, total;
};

static OutCoordWs out_coord_ws(long long n_in, int dim, int K, int s) {
  OutCoordWs w{};
  long long items = n_in * cand_per_input(dim, K, s);
  w.cand_bytes = ((size_t)items * 8 + 255) / 256 * 256;
  cub::DeviceRadixSort::SortKeys(nullptr, w.sort_tmp, (unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int64_t)items, 0, 64);
  cub::DeviceSelect::Unique(nullptr, w.uniq_tmp, (unsigned long long*)nullptr,
                            (unsigned long long*)nullptr, (long long*)nullptr, (int64_t)items);
  size_t s32 = 0, u32 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, s32, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                 (int64_t)items, 0, 32);
  cub::DeviceSelect::Unique(nullptr, u32, (uint32_t*)nullptr, (uint32_t*)nullptr,
                            (long long*)nullptr, (int64_t)items);
  w.sort_tmp = w.sort_tmp > s32 ? w.sort_tmp : s32;
  w.uniq_tmp = w.uniq_tmp > u32 ? w.uniq_tmp : u32;
  w.sort_tmp = (w.sort_tmp + 255) / 256 * 256;
  w.uniq_tmp = (w.uniq_tmp + 255) / 256 * 256;
  w.total = 2 * w.cand_bytes + (w.sort_tmp > w.uniq_tmp ? w.sort_tmp : w.uniq_tmp);
  return w;
}

}  // namespace scb

extern "C" int64_t scb_output_coords_capacity(int64_t n_in, int32_t dim, int32_t kernel_size,
                                              int32_t stride) {
  return n_in * cand_per_input(dim, kernel_size, stride);
}

extern "C" int64_t scb_output_coords_workspace(int64_t n_in, int32_t dim, int32_t kernel_size,
                                               int32_t stride) {
  return (int64_t)out_coord_ws(n_in, dim, kernel_size, stride).total;
}

namespace scb {

// Sort + unique the candidates (KT keys; 32-bit when the sentinel fits) into
// the int64 out_keys with the count on the device.
template <typename KT>
static int32_t sort_unique(void* workspace, const OutCoordWs& w, long long items,
                           unsigned long long sentinel, int end_bit, int64_t* out_keys,
                           int64_t* n_out, cudaStream_t s) {
  char* base = (char*)workspace;
  auto* cand = (KT*)base;
  auto* sorted = (KT*)(base + w.cand_bytes);
  void* tmp = base + 2 * w.cand_bytes;
  size_t tb = w.sort_tmp;
  SCB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, cand, sorted, (int64_t)items, 0, end_bit, s));
  tb = w.uniq_tmp;
  if (sizeof(KT) == 8) {
    SCB_CUDA(cub::DeviceSelect::Unique(tmp, tb, sorted, (KT*)out_keys, (long long*)n_out,
                                       (int64_t)items, s));
    drop_sentinel_kernel<<<1, 1, 0, s>>>((const unsigned long long*)out_keys, (long long*)n_out,
                                         sentinel);
    SCB_LAUNCHED();
  } else {
    KT* uniq = cand;  // the candidates are dead once sorted
    SCB_CUDA(cub::DeviceSelect::Unique(tmp, tb, sorted, uniq, (long long*)n_out, (int64_t)items, s));
    drop_sentinel_kernel32<<<1, 1, 0, s>>>((const uint32_t*)uniq, (long long*)n_out,
                                           (uint32_t)sentinel);
    SCB_LAUNCHED();
    widen_keys_kernel<<<grid_blocks(items, 256), 256, 0, s>>>(
        (const uint32_t*)uniq, (long long*)n_out, (uint32_t)sentinel,
        (unsigned long long*)out_keys, items);
    SCB_LAUNCHED();
  }
  return SCB_OK;
}

static int key_end_bit(unsigned long long sentinel) {
  int end_bit = 1;
  while (end_bit < 64 && (sentinel >> end_bit) != 0) ++end_bit;
  return end_bit;
}

}  // namespace scb

extern "C" int32_t scb_output_coords(const int32_t* in_coords, int64_t n_in,
                                     const scb_grid_t* out_grid, int32_t kernel_size,
                                     int32_t offset_base, int32_t stride, void* workspace,
                                     int64_t ws_bytes,
                                     int64_t* out_keys, int64_t* n_out, scb_stream_t stream) {
  SCB_CHECK_ARG(out_grid && out_grid->dim >= 1 && out_grid->dim <= 4, "bad grid");
  SCB_CHECK_ARG(stride >= 1 && kernel_size >= 1, "bad kernel size / stride");
  cudaStream_t s = as_stream(stream);
  Grid g = to_grid(out_grid);
  OutCoordWs w = out_coord_ws(n_in, g.dim, kernel_size, stride);
  SCB_CHECK_ARG(ws_bytes >= (int64_t)w.total, "workspace too small");
  if (n_in == 0) {
    SCB_CUDA(cudaMemsetAsync(n_out, 0, sizeof(int64_t), s));
    return SCB_OK;
  }
  const int cap = cand_per_input(g.dim, kernel_size, stride);
  const long long items = n_in * cap;
  const unsigned long long sentinel = (unsigned long long)total_cells(g);
  const int end_bit = key_end_bit(sentinel);
  if (end_bit <= 32) {
    SCB_DISPATCH_DIM(g.dim, out_candidates_kernel<D, uint32_t><<<grid_blocks(n_in, 256), 256, 0, s>>>(
                                in_coords, n_in, g, kernel_size, offset_base, stride, cap,
                                (uint32_t)sentinel, (uint32_t*)workspace));
    SCB_LAUNCHED();
    return sort_unique<uint32_t>(workspace, w, items, sentinel, end_bit, out_keys, n_out, s);
  }
  SCB_DISPATCH_DIM(g.dim, out_candidates_kernel<D, unsigned long long><<<grid_blocks(n_in, 256), 256, 0, s>>>(
                              in_coords, n_in, g, kernel_size, offset_base, stride, cap, sentinel,
                              (unsigned long long*)workspace));
  SCB_LAUNCHED();
  return sort_unique<unsigned long long>(workspace, w, items, sentinel, end_bit, out_keys, n_out, s);
}

extern "C" int32_t scb_output_keys_next(const int64_t* in_keys, const int64_t* n_in_dev,
                                        int64_t n_cap, const scb_grid_t* in_grid,
                                        const scb_grid_t* out_grid, int32_t kernel_size,
                                        int32_t offset_base, int32_t stride, void* workspace,
                                        int64_t ws_bytes, int64_t* out_keys, int64_t* n_out,
                                        scb_stream_t stream) {
  SCB_CHECK_ARG(in_grid && out_grid && in_grid->dim == out_grid->dim && out_grid->dim >= 1 &&
                    out_grid->dim <= 4, "bad grids");
  SCB_CHECK_ARG(stride >= 1 && kernel_size >= 1, "bad kernel size / stride");
  cudaStream_t s = as_stream(stream);
  Grid gi = to_grid(in_grid), g = to_grid(out_grid);
  OutCoordWs w = out_coord_ws(n_cap, g.dim, kernel_size, stride);
  SCB_CHECK_ARG(ws_bytes >= (int64_t)w.total, "workspace too small");
  if (n_cap == 0) {
    SCB_CUDA(cudaMemsetAsync(n_out, 0, sizeof(int64_t), s));
    return SCB_OK;
  }
  const int cap = cand_per_input(g.dim, kernel_size, stride);
  const long long items = n_cap * cap;
  const unsigned long long sentinel = (unsigned long long)total_cells(g);
  const int end_bit = key_end_bit(sentinel);
  if (end_bit <= 32) {
    SCB_DISPATCH_DIM(g.dim, out_candidates_keys_kernel<D, uint32_t><<<grid_blocks(n_cap, 256), 256, 0, s>>>(
                                (const unsigned long long*)in_keys, (const long long*)n_in_dev,
                                n_cap, gi, g, kernel_size, offset_base, stride, cap,
                                (uint32_t)sentinel, (uint32_t*)workspace));
    SCB_LAUNCHED();
    return sort_unique<uint32_t>(workspace, w, items, sentinel, end_bit, out_keys, n_out, s);
  }
  SCB_DISPATCH_DIM(g.dim, out_candidates_keys_kernel<D, unsigned long long><<<grid_blocks(n_cap, 256), 256, 0, s>>>(
                              (const unsigned long long*)in_keys, (const long long*)n_in_dev,
                              n_cap, gi, g, kernel_size, offset_base, stride, cap, sentinel,
                              (unsigned long long*)workspace));
  SCB_LAUNCHED();
  return sort_unique<unsigned long long>(workspace, w, items, sentinel, end_bit, out_keys, n_out, s);
}

extern "C" int32_t scb_unflatten(const int64_t* keys, int64_t n, const scb_grid_t* grid,
                                 int32_t* coords, scb_stream_t stream) {
  SCB_CHECK_ARG(grid && grid->dim >= 1 && grid->dim <= 4, "bad grid");
  if (n == 0) return SCB_OK;
  Grid g = to_grid(grid);
  SCB_DISPATCH_DIM(g.dim, unflatten_kernel<D><<<grid_blocks(n, 256), 256, 0, as_stream(stream)>>>(
                              (const long long*)keys, n, g, coords));
  SCB_LAUNCHED();
  return SCB_OK;
}

// =================================================================== map search

namespace scb {

// One thread per (output, searched offset): probe s*q + delta, record the
// input row.  blockIdx.y is the offset so hit-matrix writes are coalesced.
template <int D>
__global__ void map_search_kernel(int kind, const int* __restrict__ out_coords, long long n_out,
                                  Grid gin, int K, int lo, int s, int dil, int V, int symmetric,
                                  const long long* __restrict__ keys,
                                  const int* __restrict__ rows, unsigned long long mask,
                                  int* __restrict__ hits) {
  const int n = blockIdx.y;
  int delta[D];
  offset_of<D>(n, K, lo, delta);
#pragma unroll
  for (int d = 0; d < D; ++d) delta[d] *= dil;   // dilated window (dil = 1: the reference's)
  const int center = (V - 1) / 2;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n_out;
       k += (long long)gridDim.x * blockDim.x) {
    int p[D + 1];
    p[0] = out_coords[k * (D + 1)];
#pragma unroll
    for (int d = 0; d < D; ++d) p[d + 1] = s * out_coords[k * (D + 1) + d + 1] + delta[d];
    const int j = index_lookup<D>(kind, p, gin, keys, rows, mask);
    hits[(long long)n * hits_ld(n_out) + k] = j;
    // derive_symmetric_maps (mapping.py:322-339): M[V-1-n] holds (k, j) for
    // every (j, k) in M[n]; writing it at row j of the mirror column yields
    // the reference's "sorted by new output row" order for free.
    if (symmetric && n < center && j >= 0) hits[(long long)(V - 1 - n) * hits_ld(n_out) + j] = (int)k;
  }
}

// Stride-1 map of a set onto itself when every row's neighbour-presence word
// is already known (scb_presence_masks, carried through the presence
// reordering): a row probes only the offsets its word marks present (each
// probe is a hit), writes -1 for the others without probing, and the
// 128-row tile words (scb_tile_masks) fall out as the OR of the row words.
// One block of 128 threads per output tile, grid-stride over tiles.
template <int D>
__global__ void __launch_bounds__(128) map_search_masked_kernel(
    int kind, const int* __restrict__ coords, long long n, Grid g, int K, int lo, int V,
    const long long* __restrict__ keys, const int* __restrict__ rows, unsigned long long smask,
    const uint32_t* __restrict__ masks, int* __restrict__ hits, uint32_t* __restrict__ tmask) {
  __shared__ uint32_t acc[4];
  const long long ld = hits_ld(n);
  const long long tiles = (n + 127) / 128;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long long k = t * 128 + threadIdx.x;
    uint32_t m = 0;
    if (k < n) {
      m = __ldg(masks + k);
      int c[D + 1];
#pragma unroll
      for (int d = 0; d <= D; ++d) c[d] = __ldg(coords + k * (D + 1) + d);
      for (int v = 0; v < V; ++v) {
        int j = -1;
        if ((m >> v) & 1u) {
          int delta[D], p[D + 1];
          offset_of<D>(v, K, lo, delta);
          p[0] = c[0];
#pragma unroll
          for (int d = 0; d < D; ++d) p[d + 1] = c[d + 1] + delta[d];
          j = index_lookup<D>(kind, p, g, keys, rows, smask);
        }
        hits[(long long)v * ld + k] = j;
      }
    }
    const uint32_t w = __reduce_or_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) acc[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0 && tmask) tmask[t] = acc[0] | acc[1] | acc[2] | acc[3];
    __syncthreads();
  }
}

constexpr int CHUNK_THREADS = 256;
constexpr int CHUNK_ITEMS = 8;
constexpr int CHUNK = CHUNK_THREADS * CHUNK_ITEMS;

__global__ void __launch_bounds__(CHUNK_THREADS) map_count_kernel(const int* __restrict__ hits,
                                                                  long long n_out, int nchunks,
                                                                  int* __restrict__ counts) {
  const int n = blockIdx.y, c = blockIdx.x;
  const int* col = hits + (long long)n * hits_ld(n_out);
  const long long base = (long long)c * CHUNK;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < CHUNK_ITEMS; ++i) {
    long long k = base + i * CHUNK_THREADS + threadIdx.x;
    if (k < n_out && col[k] >= 0) ++cnt;
  }
  typedef cub::BlockReduce<int, CHUNK_THREADS> Reduce;
  __shared__ typename Reduce::TempStorage tmp;
  int total = Reduce(tmp).Sum(cnt);
  if (threadIdx.x == 0) counts[(long long)n * nchunks + c] = total;
}

// Exclusive scan of the (offset-major) chunk counts in one block; also
// emits offset_ptr[V+1].
__global__ void __launch_bounds__(1024) map_scan_kernel(const int* __restrict__ counts, int V,
                                                        int nchunks, long long* __restrict__ bases,
                                                        long long* __restrict__ offset_ptr) {
  typedef cub::BlockScan<long long, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const long long total = (long long)V * nchunks;
  for (long long start = 0; start < total; start += 1024) {
    long long i = start + threadIdx.x;
    long long v = i < total ? counts[i] : 0;
    long long excl, agg;
    Scan(tmp).ExclusiveSum(v, excl, agg);
    if (i < total) {
      bases[i] = carry + excl;
      if (i % nchunks == 0) offset_ptr[i / nchunks] = carry + excl;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) offset_ptr[V] = carry;
}

__global__ void __launch_bounds__(CHUNK_THREADS) map_compact_kernel(
    const int* __restrict__ hits, long long n_out, int nchunks, const long long* __restrict__ bases,
    int* __restrict__ in_idx, int* __restrict__ out_idx) {
  const int n = blockIdx.y, c = blockIdx.x;
  const int* col = hits + (long long)n * hits_ld(n_out);
  const long long base = (long long)c * CHUNK;
  long long out_base = bases[(long long)n * nchunks + c];
  __shared__ int warp_tot[CHUNK_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < CHUNK_ITEMS; ++i) {
    const long long k = base + i * CHUNK_THREADS + threadIdx.x;
    const int j = k < n_out ? col[k] : -1;
    const unsigned ballot = __ballot_sync(0xffffffffu, j >= 0);
    if (lane == 0) warp_tot[warp] = __popc(ballot);
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < CHUNK_THREADS / 32; ++w) {
      before += (w < warp) ? warp_tot[w] : 0;
      all += warp_tot[w];
    }
    if (j >= 0) {
      const long long r = out_base + before + __popc(ballot & ((1u << lane) - 1));
      in_idx[r] = j;
      out_idx[r] = (int)k;
    }
    out_base += all;
    __syncthreads();
  }
}

// The whole gather/scatter plan straight from a hit matrix, after
// map_count_kernel + map_scan_kernel (bases / offset_ptr): entry (j, k) of
// offset n with rank r among the offset's entries (output order) goes to
// buffer row slab[n] + r.  Writes buf_in, the full pos[n_out][V] (-1 where
// absent, so no memset), the padding rows of every slab, and — block (0,0) —
// the GEMM SegTable.  No host round trip.
__global__ void __launch_bounds__(CHUNK_THREADS) plan_from_hits_kernel(
    const int* __restrict__ hits, long long ld, int V, long long n_out, int nchunks,
    const long long* __restrict__ bases, const long long* __restrict__ offset_ptr, int skip,
    int tile, long long c_base, int gemm_bm, int gemm_ntn, int center_seg, long long center_rows,
    int* __restrict__ buf_in, int* __restrict__ pos, SegTable* __restrict__ table) {
  __shared__ long long ptr_s[SCB_MAX_SEGMENTS + 1];
  __shared__ long long slab_s[SCB_MAX_SEGMENTS + 1];
  __shared__ int warp_tot[CHUNK_THREADS / 32];
  const int n = blockIdx.y, c = blockIdx.x;
  for (int i = threadIdx.x; i <= V; i += blockDim.x) ptr_s[i] = offset_ptr[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int m = 0; m < V; ++m) {
      slab_s[m] = acc;
      const long long sz = (m == skip) ? 0 : ptr_s[m + 1] - ptr_s[m];
      acc += (sz + tile - 1) / tile * tile;
    }
    slab_s[V] = acc;
  }
  __syncthreads();
  if (c == 0 && n == 0) {
    // padding rows of every slab -> -1 (zero rows in the gather)
    for (int m = 0; m < V; ++m) {
      const long long sz = (m == skip) ? 0 : ptr_s[m + 1] - ptr_s[m];
      for (long long r = slab_s[m] + sz + threadIdx.x; r < slab_s[m + 1]; r += blockDim.x)
        buf_in[r] = -1;
    }
    if (threadIdx.x == 0) {
      int s = 0, tiles = 0;
      if (center_seg >= 0 && center_rows > 0) {
        SegDesc& d = table->seg[s];
        d.a_row = 0; d.c_row = 0; d.rows = (int)center_rows; d.b_index = center_seg; d.a_src = 1;
        table->tile_start[s++] = tiles;
        tiles += (int)((center_rows + gemm_bm - 1) / gemm_bm) * gemm_ntn;
      }
      for (int m = 0; m < V; ++m) {
        const long long sz = (m == skip) ? 0 : ptr_s[m + 1] - ptr_s[m];
        if (sz == 0 || s >= SCB_MAX_SEGMENTS) continue;
        SegDesc& d = table->seg[s];
        d.a_row = slab_s[m]; d.c_row = slab_s[m] + c_base; d.rows = (int)sz; d.b_index = m;
        d.a_src = 0;
        table->tile_start[s++] = tiles;
        tiles += (int)((sz + gemm_bm - 1) / gemm_bm) * gemm_ntn;
      }
      table->tile_start[s] = tiles;
      table->n_segs = s;
      table->total_tiles = tiles;
      table->rows_pad = slab_s[V];
    }
  }
  const int* col = hits + (long long)n * ld;
  const long long base = (long long)c * CHUNK;
  long long out_base = bases[(long long)n * nchunks + c] - ptr_s[n] + slab_s[n];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < CHUNK_ITEMS; ++i) {
    const long long k = base + i * CHUNK_THREADS + threadIdx.x;
    const int j = k < n_out ? col[k] : -1;
    const bool take = j >= 0 && n != skip;
    const unsigned ballot = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_tot[warp] = __popc(ballot);
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < CHUNK_THREADS / 32; ++w) {
      before += (w < warp) ? warp_tot[w] : 0;
      all += warp_tot[w];
    }
    if (k < n_out) {
      int r = -1;
      if (take) {
        const long long row = out_base + before + __popc(ballot & ((1u << lane) - 1));
        buf_in[row] = j;
        r = (int)(row + c_base);
      }
      pos[k * V + n] = r;
    }
    out_base += all;
    __syncthreads();
  }
}

__device__ __forceinline__ int find_offset(const long long* ptr_s, int V, long long e) {
  int lo = 0, hi = V;  // largest n with ptr[n] <= e
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (ptr_s[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void map_transpose_kernel(const long long* __restrict__ offset_ptr,
                                     const int* __restrict__ in_idx,
                                     const int* __restrict__ out_idx, int V, long long total,
                                     long long n_in, int* __restrict__ hits_t) {
  extern __shared__ long long ptr_s[];
  for (int i = threadIdx.x; i <= V; i += blockDim.x) ptr_s[i] = offset_ptr[i];
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int n = find_offset(ptr_s, V, e);
    hits_t[(long long)n * hits_ld(n_in) + in_idx[e]] = out_idx[e];
  }
}

// hits_t[n][hits[n][k]] = k: the transposed map's hit matrix straight from the
// forward hit matrix (no compaction needed).
__global__ void hits_transpose_kernel(const int* __restrict__ hits, long long total,
                                      long long n_out, long long n_in, int* __restrict__ hits_t) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long n = i / n_out, k = i - n * n_out;
    const int j = hits[n * hits_ld(n_out) + k];
    if (j >= 0) hits_t[n * hits_ld(n_in) + j] = (int)k;
  }
}

__global__ void plan_build_kernel(const long long* __restrict__ offset_ptr,
                                  const int* __restrict__ in_idx, const int* __restrict__ out_idx,
                                  int V, long long total, int skip, int tile,
                                  int* __restrict__ buf_in, int* __restrict__ pos,
                                  int* __restrict__ status) {
  extern __shared__ long long sm[];
  long long* ptr_s = sm;
  long long* slab_s = sm + V + 1;
  for (int i = threadIdx.x; i <= V; i += blockDim.x) ptr_s[i] = offset_ptr[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int n = 0; n < V; ++n) {
      slab_s[n] = acc;
      const long long sz = (n == skip) ? 0 : ptr_s[n + 1] - ptr_s[n];
      acc += (sz + tile - 1) / tile * tile;
    }
  }
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int n = find_offset(ptr_s, V, e);
    if (n == skip) continue;
    const long long r = slab_s[n] + (e - ptr_s[n]);
    buf_in[r] = in_idx[e];
    int* slot = pos + (long long)out_idx[e] * V + n;
    if (status) {
      // a real kernel map has at most one entry per (output, offset)
      if (atomicCAS(slot, -1, (int)r) != -1) atomicAdd(status, 1);
    } else {
      *slot = (int)r;
    }
  }
}

}  // namespace scb

extern "C" int32_t scb_map_search_dilated(int32_t kind, const int32_t* out_coords, int64_t n_out,
                                          const scb_grid_t* in_grid, int32_t kernel_size,
                                          int32_t offset_base, int32_t stride, int32_t dilation,
                                          int32_t symmetric, const int64_t* table_keys,
                                          const int32_t* table_rows, int64_t slots, int32_t* hits,
                                          scb_stream_t stream) {
  SCB_CHECK_ARG(in_grid && in_grid->dim >= 1 && in_grid->dim <= 4, "bad grid");
  SCB_CHECK_ARG(dilation >= 1, "dilation must be >= 1");
  Grid g = to_grid(in_grid);
  int V = 1;
  for (int d = 0; d < g.dim; ++d) V *= kernel_size;
  SCB_CHECK_ARG(V <= 65535, "kernel volume too large");
  const bool sym = symmetric != 0;
  if (sym) {
    SCB_CHECK_ARG(stride == 1, "symmetric maps exist only for stride-1 layers");
    SCB_CHECK_ARG(kernel_size % 2 == 1, "symmetric maps exist only for odd kernel sizes");
  }
  cudaStream_t s = as_stream(stream);
  if (n_out == 0) return SCB_OK;
  const int searched = sym ? (V - 1) / 2 + 1 : V;
  if (sym && V > 1) {
    const long long c = (V - 1) / 2;
    SCB_CUDA(cudaMemsetAsync(hits + (c + 1) * hits_ld(n_out), 0xFF,
                             (V - 1 - c) * hits_ld(n_out) * sizeof(int32_t), s));
  }
  dim3 grid(grid_blocks(n_out, 256, 4096), searched);
  SCB_DISPATCH_DIM(g.dim, map_search_kernel<D><<<grid, 256, 0, s>>>(
                              kind, out_coords, n_out, g, kernel_size, offset_base, stride, dilation,
                              V, sym ? 1 : 0, (const long long*)table_keys, table_rows,
                              (unsigned long long)(slots - 1), hits));
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_map_search(int32_t kind, const int32_t* out_coords, int64_t n_out,
                                  const scb_grid_t* in_grid, int32_t kernel_size,
                                  int32_t offset_base, int32_t stride, int32_t symmetric,
                                  const int64_t* table_keys, const int32_t* table_rows,
                                  int64_t slots, int32_t* hits, scb_stream_t stream) {
  return scb_map_search_dilated(kind, out_coords, n_out, in_grid, kernel_size, offset_base, stride,
                                1, symmetric, table_keys, table_rows, slots, hits, stream);
}

extern "C" int64_t scb_map_workspace(int32_t volume, int64_t n_out) {
  const long long nchunks = (n_out + CHUNK - 1) / CHUNK;
  const long long m = volume * (nchunks > 0 ? nchunks : 1);
  return (int64_t)(((m * 4 + 255) / 256 * 256) + m * 8);
}

extern "C" int32_t scb_map_count(const int32_t* hits, int32_t volume, int64_t n_out,
                                 void* workspace, int64_t* offset_ptr, scb_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  const long long nchunks = (n_out + CHUNK - 1) / CHUNK;
  if (nchunks == 0) {
    SCB_CUDA(cudaMemsetAsync(offset_ptr, 0, (volume + 1) * sizeof(int64_t), s));
    return SCB_OK;
  }
  SCB_CHECK_ARG(nchunks < (1LL << 31), "too many outputs");
  const long long m = volume * nchunks;
  int* counts = (int*)workspace;
  long long* bases = (long long*)((char*)workspace + (m * 4 + 255) / 256 * 256);
  map_count_kernel<<<dim3((unsigned)nchunks, volume), CHUNK_THREADS, 0, s>>>(hits, n_out,
                                                                           (int)nchunks, counts);
  SCB_LAUNCHED();
  map_scan_kernel<<<1, 1024, 0, s>>>(counts, volume, (int)nchunks, bases, (long long*)offset_ptr);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_map_compact(const int32_t* hits, int32_t volume, int64_t n_out,
                                   const void* workspace, const int64_t* offset_ptr,
                                   int32_t* in_idx, int32_t* out_idx, scb_stream_t stream) {
  (void)offset_ptr;
  const long long nchunks = (n_out + CHUNK - 1) / CHUNK;
  if (nchunks == 0) return SCB_OK;
  const long long m = volume * nchunks;
  const long long* bases =
      (const long long*)((const char*)workspace + (m * 4 + 255) / 256 * 256);
  map_compact_kernel<<<dim3((unsigned)nchunks, volume), CHUNK_THREADS, 0, as_stream(stream)>>>(
      hits, n_out, (int)nchunks, bases, in_idx, out_idx);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_map_transpose(const int64_t* offset_ptr, const int32_t* in_idx,
                                     const int32_t* out_idx, int32_t volume, int64_t total,
                                     int64_t n_in, int32_t* hits_t, scb_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  SCB_CUDA(cudaMemsetAsync(hits_t, 0xFF, (size_t)volume * hits_ld(n_in) * sizeof(int32_t), s));
  if (total == 0) return SCB_OK;
  map_transpose_kernel<<<grid_blocks(total, 256), 256, (volume + 1) * sizeof(long long), s>>>(
      (const long long*)offset_ptr, in_idx, out_idx, volume, total, n_in, hits_t);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int64_t scb_plan_rows_cap(int32_t volume, int64_t n_out, int32_t tile_rows) {
  return (int64_t)volume * (n_out + tile_rows);
}

extern "C" int64_t scb_segtable_bytes(void) { return (int64_t)sizeof(SegTable); }

extern "C" int32_t scb_plan_from_hits(const int32_t* hits, int32_t volume, int64_t n_out,
                                      int32_t skip_offset, int32_t tile_rows, int64_t c_base,
                                      int32_t gemm_bm, int32_t gemm_ntn, int32_t center_seg,
                                      int64_t center_rows, void* workspace, int64_t* offset_ptr,
                                      int32_t* buf_in, int32_t* pos, void* table,
                                      scb_stream_t stream) {
  SCB_CHECK_ARG(volume >= 1 && volume <= SCB_MAX_SEGMENTS - 1, "kernel volume too large");
  SCB_CHECK_ARG(tile_rows >= 1 && gemm_bm >= 1 && gemm_ntn >= 1, "bad tile sizes");
  cudaStream_t s = as_stream(stream);
  const long long nchunks = (n_out + CHUNK - 1) / CHUNK;
  if (nchunks == 0) {
    SCB_CUDA(cudaMemsetAsync(table, 0, sizeof(SegTable), s));
    SCB_CUDA(cudaMemsetAsync(offset_ptr, 0, (volume + 1) * sizeof(int64_t), s));
    return SCB_OK;
  }
  const int32_t rc = scb_map_count(hits, volume, n_out, workspace, offset_ptr, stream);
  if (rc != SCB_OK) return rc;
  const long long m = volume * nchunks;
  const long long* bases = (const long long*)((const char*)workspace + (m * 4 + 255) / 256 * 256);
  plan_from_hits_kernel<<<dim3((unsigned)nchunks, volume), CHUNK_THREADS, 0, s>>>(
      hits, hits_ld(n_out), volume, n_out, (int)nchunks, bases, (const long long*)offset_ptr,
      skip_offset, tile_rows, c_base, gemm_bm, gemm_ntn, center_seg, center_rows, buf_in, pos,
      (SegTable*)table);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_hits_transpose(const int32_t* hits, int32_t volume, int64_t n_out,
                                      int64_t n_in, int32_t* hits_t, scb_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  if (n_in) SCB_CUDA(cudaMemsetAsync(hits_t, 0xFF, (size_t)volume * hits_ld(n_in) * sizeof(int32_t), s));
  const long long total = (long long)volume * n_out;
  if (total == 0) return SCB_OK;
  hits_transpose_kernel<<<grid_blocks(total, 256), 256, 0, s>>>(hits, total, n_out, n_in, hits_t);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_plan_build(const int64_t* offset_ptr, const int32_t* in_idx,
                                  const int32_t* out_idx, int32_t volume, int64_t total,
                                  int64_t n_out, int32_t skip_offset, int32_t tile_rows,
                                  int32_t* buf_in, int64_t rows_pad, int32_t* pos,
                                  int32_t* status, scb_stream_t stream) {
  SCB_CHECK_ARG(tile_rows >= 1, "tile_rows must be positive");
  cudaStream_t s = as_stream(stream);
  if (status) SCB_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
  if (rows_pad) SCB_CUDA(cudaMemsetAsync(buf_in, 0xFF, rows_pad * sizeof(int32_t), s));
  if (n_out) SCB_CUDA(cudaMemsetAsync(pos, 0xFF, (size_t)n_out * volume * sizeof(int32_t), s));
  if (total == 0) return SCB_OK;
  plan_build_kernel<<<grid_blocks(total, 256), 256, (2 * volume + 1) * sizeof(long long), s>>>(
      (const long long*)offset_ptr, in_idx, out_idx, volume, total, skip_offset, tile_rows,
      buf_in, pos, status);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_map_search_masked(int32_t kind, const int32_t* coords, int64_t n,
                                         const scb_grid_t* grid, int32_t kernel_size,
                                         int32_t offset_base, const int64_t* table_keys,
                                         const int32_t* table_rows, int64_t slots,
                                         const uint32_t* masks, int32_t* hits,
                                         uint32_t* tile_masks, scb_stream_t stream) {
  SCB_CHECK_ARG(grid && grid->dim >= 1 && grid->dim <= 4, "bad grid");
  SCB_CHECK_ARG(masks != nullptr && hits != nullptr, "presence masks and hits are required");
  Grid g = to_grid(grid);
  int V = 1;
  for (int d = 0; d < g.dim; ++d) V *= kernel_size;
  SCB_CHECK_ARG(V <= 32, "presence masks hold at most 32 offsets");
  if (n == 0) return SCB_OK;
  const long long tiles = (n + 127) / 128;
  const int blocks = (int)(tiles < 148 * 16 ? tiles : 148 * 16);
  SCB_DISPATCH_DIM(g.dim, map_search_masked_kernel<D><<<blocks, 128, 0, as_stream(stream)>>>(
                              kind, coords, n, g, kernel_size, offset_base, V,
                              (const long long*)table_keys, table_rows,
                              (unsigned long long)(slots - 1), masks, hits, tile_masks));
  SCB_LAUNCHED();
  return SCB_OK;
}
