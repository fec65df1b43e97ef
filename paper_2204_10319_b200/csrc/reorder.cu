// Presence-mask row reordering (B200 extension; the bitmask sort of
// TorchSparse++): rows of a coordinate set are reordered so that 128-row
// tiles hold rows with similar neighbour patterns, which makes whole (tile,
// offset) blocks of the fused conv absent (scb_tile_masks).
// A reordered set is an ordinary coordinate set in another row order: its
// maps are built by the regular index + map search, so every result is the
// same set of (input, output) pairs, just relabelled.  Models un-permute
// their final output rows (scb_permute_rows), so what leaves the engine is
// in the reference's row order.
//
//   scb_presence_masks  bit n of mask[k] = coordinate k + delta_n is present
//                       (stride 1, same set), plus per-offset counts
//   scb_mask_sort       perm = stable sort of rows by their mask with the
//                       rarest offsets as the most significant bits
//   scb_permute_rows    dst[i] = src[index[i]] (gather) or dst[index[i]] = src[i]
#include <cub/cub.cuh>

#include "common.cuh"

namespace scb {
namespace {

constexpr int RT = 256;

// Symmetric probing (stride 1, odd K: q = p + delta_v  <=>  p = q + delta_{V-1-v}):
// each row probes the offsets below the centre, sets bit v of its own word
// and bit V-1-v of the neighbour's word (atomicOr; masks zeroed first), and
// the centre bit.  counts[v] = counts[V-1-v] = hits at offset v < centre.
template <int D>
__global__ void __launch_bounds__(RT) presence_masks_kernel(
    int kind, const int* __restrict__ coords, long long n, Grid g, int K, int lo, int V,
    const long long* __restrict__ keys, const int* __restrict__ rows, unsigned long long smask,
    uint32_t* __restrict__ masks, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int cnt[32];
  if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int center = (V - 1) / 2;
  for (long long base = (long long)blockIdx.x * RT; base < n; base += (long long)gridDim.x * RT) {
    const long long k = base + threadIdx.x;
    uint32_t m = 0;
    if (k < n) {
      int c[D + 1];
#pragma unroll
      for (int d = 0; d <= D; ++d) c[d] = coords[k * (D + 1) + d];
      m = 1u << center;
      for (int v = 0; v < center; ++v) {
        int delta[D], p[D + 1];
        offset_of<D>(v, K, lo, delta);
        p[0] = c[0];
#pragma unroll
        for (int d = 0; d < D; ++d) p[d + 1] = c[d + 1] + delta[d];
        const int j = index_lookup<D>(kind, p, g, keys, rows, smask);
        if (j >= 0) {
          m |= 1u << v;
          atomicOr(masks + j, 1u << (V - 1 - v));
        }
      }
      atomicOr(masks + k, m);
    }
    for (int v = 0; v < center; ++v) {
      const unsigned b = __ballot_sync(0xffffffffu, (m >> v) & 1u);
      if (lane == 0 && b) atomicAdd(&cnt[v], (unsigned)__popc(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < center && cnt[threadIdx.x]) {
    atomicAdd(counts + threadIdx.x, (unsigned long long)cnt[threadIdx.x]);
    atomicAdd(counts + V - 1 - threadIdx.x, (unsigned long long)cnt[threadIdx.x]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(counts + center, (unsigned long long)n);
}

// key = the mask with offset v moved to bit pos[v], pos[v] = number
// of offsets more frequent than v (ties: lower index first) -- the rarest
// offsets decide the order first, so rows sharing their rare neighbours
// land in the same tiles.
template <typename KeyT>
__global__ void __launch_bounds__(RT) sort_keys_kernel(const uint32_t* __restrict__ masks,
                                                       const int* __restrict__ coords, int cols,
                                                       long long n, int V,
                                                       const unsigned long long* __restrict__ counts,
                                                       KeyT* __restrict__ keys,
                                                       int* __restrict__ vals) {
  __shared__ int pos[32];
  if (threadIdx.x < V) {
    const unsigned long long c = counts[threadIdx.x];
    int r = 0;
    for (int u = 0; u < V; ++u) {
      const unsigned long long cu = counts[u];
      r += (cu > c || (cu == c && u < (int)threadIdx.x)) ? 1 : 0;
    }
    pos[threadIdx.x] = r;
  }
  __syncthreads();
  for (long long k = (long long)blockIdx.x * RT + threadIdx.x; k < n; k += (long long)gridDim.x * RT) {
    const uint32_t m = masks[k];
    KeyT key = 0;
    for (int v = 0; v < V; ++v) key |= (KeyT)((m >> v) & 1u) << pos[v];
    // the batch column is not part of the key: maps never cross batch
    // entries, so tiles may mix them, and grouping equal words across the
    // batch leaves ~19 % fewer live (tile, offset) blocks at level 0
    // ...and the words are visited in Gray-code order (sort by the word's
    // index along the reflected Gray sequence: consecutive groups differ in
    // one offset, ~3 % fewer live blocks than plain binary order)
    key ^= key >> 1;
    key ^= key >> 2;
    key ^= key >> 4;
    key ^= key >> 8;
    key ^= key >> 16;
    if (sizeof(KeyT) > 4) key ^= key >> 32;
    keys[k] = key;
    vals[k] = (int)k;
  }
}

template <typename T>
__global__ void permute_rows_kernel(const uint8_t* __restrict__ src, long long src_ld,
                                    const int* __restrict__ index, long long n, int row_words,
                                    uint8_t* __restrict__ dst, long long dst_ld, int scatter) {
  const long long total = n * row_words;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / row_words;
    const int w = (int)(e - i * row_words);
    const long long j = index[i];
    const long long si = scatter ? i : j, di = scatter ? j : i;
    reinterpret_cast<T*>(dst + di * dst_ld)[w] = __ldg(reinterpret_cast<const T*>(src + si * src_ld) + w);
  }
}

// coords_out[i] = coords[perm[i]], inv[perm[i]] = i
__global__ void apply_order_kernel(const int* __restrict__ perm, long long n,
                                   const int* __restrict__ coords, int cols,
                                   int* __restrict__ coords_out, int* __restrict__ inv) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = perm[i];
    inv[j] = (int)i;
    for (int c = 0; c < cols; ++c) coords_out[i * cols + c] = __ldg(coords + (long long)j * cols + c);
  }
}

// The same index under relabelled rows: occupied slots get inv[row].
__global__ void relabel_kernel(const long long* __restrict__ keys, const int* __restrict__ rows_in,
                               long long slots, const int* __restrict__ inv,
                               int* __restrict__ rows_out) {
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < slots;
       s += (long long)gridDim.x * blockDim.x) {
    const bool occupied = keys ? __ldg(keys + s) != EMPTY_KEY : __ldg(rows_in + s) >= 0;
    rows_out[s] = occupied ? __ldg(inv + __ldg(rows_in + s)) : -1;
  }
}

// One-hot maps (every output row has at most one entry, e.g. the transposed
// k2 s2 map: each fine voxel has one parent): key[k] = the offset of row k's
// entry (V when it has none), to be stably sorted so that 128-row tiles hold
// rows of one offset.
__global__ void onehot_keys_kernel(const int* __restrict__ hits, long long ld, int V, long long n,
                                   uint32_t* __restrict__ keys, int* __restrict__ vals) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    uint32_t off = (uint32_t)V;
    for (int v = V - 1; v >= 0; --v)
      if (__ldg(hits + (long long)v * ld + k) >= 0) off = (uint32_t)v;
    keys[k] = off;
    vals[k] = (int)k;
  }
}

// The hit matrix in the sorted row order (tile row r = output row perm[r])
// and its tile words.  128 threads per block, one tile per iteration.
__global__ void __launch_bounds__(128) onehot_apply_kernel(
    const int* __restrict__ hits, long long ld, int V, long long n, const uint32_t* __restrict__ skeys,
    const int* __restrict__ perm, int* __restrict__ hits_out, uint32_t* __restrict__ tmask) {
  __shared__ uint32_t acc[4];
  const long long tiles = (n + 127) / 128;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long long r = t * 128 + threadIdx.x;
    uint32_t m = 0;
    if (r < n) {
      const long long k = perm[r];
      const uint32_t off = skeys[r];
      for (int v = 0; v < V; ++v)
        hits_out[(long long)v * ld + r] = (uint32_t)v == off ? __ldg(hits + (long long)v * ld + k) : -1;
      m = off < (uint32_t)V ? (1u << off) : 0u;
    }
    const uint32_t w = __reduce_or_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) acc[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) tmask[t] = acc[0] | acc[1] | acc[2] | acc[3];
    __syncthreads();
  }
}

int blocks_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < 148 * 16 ? b : 148 * 16);
}

struct SortWs {
  size_t keys_in, keys_out, vals_in, tmp, total;
};
SortWs sort_ws(long long n) {
  SortWs w;
  auto a = [](size_t x) { return (x + 255) / 256 * 256; };
  w.keys_in = a(sizeof(unsigned long long) * (size_t)(n > 0 ? n : 1));
  w.keys_out = w.keys_in;
  w.vals_in = a(sizeof(int) * (size_t)(n > 0 ? n : 1));
  size_t tb = 0, tb32 = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, tb, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr,
                                  (int64_t)(n > 0 ? n : 1), 0, 64);
  cub::DeviceRadixSort::SortPairs((void*)nullptr, tb32, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int*)nullptr, (int*)nullptr, (int64_t)(n > 0 ? n : 1), 0, 32);
  w.tmp = a(tb > tb32 ? tb : tb32);
  w.total = w.keys_in + w.keys_out + w.vals_in + w.tmp + 256;
  return w;
}

}  // namespace
}  // namespace scb

using namespace scb;

extern "C" int32_t scb_presence_masks(int32_t kind, const int32_t* coords, int64_t n,
                                      const scb_grid_t* grid, int32_t kernel_size,
                                      int32_t offset_base, const int64_t* table_keys,
                                      const int32_t* table_rows, int64_t slots, uint32_t* masks,
                                      uint64_t* counts, scb_stream_t stream) {
  SCB_CHECK_ARG(grid && grid->dim >= 1 && grid->dim <= 4, "bad grid");
  Grid g = to_grid(grid);
  int V = 1;
  for (int d = 0; d < g.dim; ++d) V *= kernel_size;
  SCB_CHECK_ARG(V <= 32, "presence masks hold at most 32 offsets");
  SCB_CHECK_ARG(kernel_size % 2 == 1, "presence masks need an odd kernel size (symmetric probing)");
  cudaStream_t s = as_stream(stream);
  SCB_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * V, s));
  if (n == 0) return SCB_OK;
  SCB_CUDA(cudaMemsetAsync(masks, 0, sizeof(uint32_t) * n, s));
  SCB_DISPATCH_DIM(g.dim, presence_masks_kernel<D><<<blocks_for(n, RT), RT, 0, s>>>(
                              kind, coords, n, g, kernel_size, offset_base, V,
                              (const long long*)table_keys, table_rows,
                              (unsigned long long)(slots - 1), masks,
                              (unsigned long long*)counts));
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int64_t scb_mask_sort_workspace(int64_t n) { return (int64_t)sort_ws(n).total; }

extern "C" int32_t scb_mask_sort(const uint32_t* masks, const uint64_t* counts,
                                 const int32_t* coords, int32_t cols, int64_t n, int32_t volume,
                                 int64_t batch_size, void* workspace, int64_t ws_bytes,
                                 int32_t* perm, scb_stream_t stream) {
  SCB_CHECK_ARG(volume >= 1 && volume <= 32, "presence masks hold at most 32 offsets");
  SCB_CHECK_ARG(batch_size >= 1, "batch size must be positive");
  const SortWs w = sort_ws(n);
  SCB_CHECK_ARG(ws_bytes >= (int64_t)w.total, "workspace too small");
  if (n == 0) return SCB_OK;
  const int end_bit = volume;
  SCB_CHECK_ARG(end_bit <= 64, "batch too large for the sort key");
  cudaStream_t s = as_stream(stream);
  char* base = (char*)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
  void* kin = base;
  void* kout = base + w.keys_in;
  auto* vin = (int*)(base + w.keys_in + w.keys_out);
  void* tmp = base + w.keys_in + w.keys_out + w.vals_in;
  size_t tb = w.tmp;
  // LSD radix sort: stable, so rows with equal keys keep their (flat-key)
  // order; 32-bit keys whenever batch + mask bits fit (half the key traffic)
  if (end_bit <= 32) {
    sort_keys_kernel<uint32_t><<<blocks_for(n, RT), RT, 0, s>>>(
        masks, coords, cols, n, volume, (const unsigned long long*)counts, (uint32_t*)kin, vin);
    SCB_LAUNCHED();
    SCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, (uint32_t*)kin, (uint32_t*)kout, vin, perm,
                                             (int64_t)n, 0, end_bit, s));
  } else {
    sort_keys_kernel<unsigned long long><<<blocks_for(n, RT), RT, 0, s>>>(
        masks, coords, cols, n, volume, (const unsigned long long*)counts,
        (unsigned long long*)kin, vin);
    SCB_LAUNCHED();
    SCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, (unsigned long long*)kin,
                                             (unsigned long long*)kout, vin, perm, (int64_t)n, 0,
                                             end_bit, s));
  }
  return SCB_OK;
}

extern "C" int32_t scb_apply_order(const int32_t* perm, int64_t n, const int32_t* coords,
                                   int32_t cols, int32_t* coords_out, int32_t* inv_out,
                                   scb_stream_t stream) {
  SCB_CHECK_ARG(cols >= 1 && cols <= 5, "coordinate rows have 2..5 columns");
  if (n == 0) return SCB_OK;
  apply_order_kernel<<<blocks_for(n, RT), RT, 0, as_stream(stream)>>>(perm, n, coords, cols,
                                                                      coords_out, inv_out);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_index_relabel(int32_t kind, const int64_t* table_keys,
                                     const int32_t* rows_in, int64_t slots, const int32_t* inv,
                                     int32_t* rows_out, scb_stream_t stream) {
  SCB_CHECK_ARG(kind == SCB_INDEX_HASH || kind == SCB_INDEX_GRID, "unknown index kind");
  SCB_CHECK_ARG(kind == SCB_INDEX_GRID || table_keys != nullptr, "hash index needs its keys");
  if (slots == 0) return SCB_OK;
  relabel_kernel<<<blocks_for(slots, RT), RT, 0, as_stream(stream)>>>(
      kind == SCB_INDEX_HASH ? (const long long*)table_keys : nullptr, rows_in, slots, inv,
      rows_out);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_permute_rows(const void* src, int64_t src_ld_bytes, const int32_t* index,
                                    int64_t n, int32_t row_bytes, void* dst, int64_t dst_ld_bytes,
                                    int32_t scatter, scb_stream_t stream) {
  SCB_CHECK_ARG(row_bytes > 0 && row_bytes % 2 == 0, "row bytes must be a positive multiple of 2");
  SCB_CHECK_ARG(src_ld_bytes >= row_bytes && dst_ld_bytes >= row_bytes, "row strides too small");
  if (n == 0) return SCB_OK;
  cudaStream_t s = as_stream(stream);
  const uintptr_t align = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)src_ld_bytes |
                          (uintptr_t)dst_ld_bytes | (uintptr_t)row_bytes;
  const int vb = (align % 16 == 0) ? 16 : ((align % 8 == 0) ? 8 : ((align % 4 == 0) ? 4 : 2));
  const int words = row_bytes / vb;
  const int blocks = blocks_for(n * words, RT);
  if (vb == 16)
    permute_rows_kernel<uint4><<<blocks, RT, 0, s>>>((const uint8_t*)src, src_ld_bytes, index, n,
                                                     words, (uint8_t*)dst, dst_ld_bytes, scatter);
  else if (vb == 8)
    permute_rows_kernel<uint2><<<blocks, RT, 0, s>>>((const uint8_t*)src, src_ld_bytes, index, n,
                                                     words, (uint8_t*)dst, dst_ld_bytes, scatter);
  else if (vb == 4)
    permute_rows_kernel<uint32_t><<<blocks, RT, 0, s>>>((const uint8_t*)src, src_ld_bytes, index, n,
                                                        words, (uint8_t*)dst, dst_ld_bytes, scatter);
  else
    permute_rows_kernel<uint16_t><<<blocks, RT, 0, s>>>((const uint8_t*)src, src_ld_bytes, index, n,
                                                        words, (uint8_t*)dst, dst_ld_bytes, scatter);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int64_t scb_onehot_order_workspace(int64_t n) { return (int64_t)sort_ws(n).total; }

extern "C" int32_t scb_onehot_order(const int32_t* hits, int32_t volume, int64_t n, void* workspace,
                                    int64_t ws_bytes, int32_t* perm, int32_t* hits_out,
                                    uint32_t* tile_masks, scb_stream_t stream) {
  SCB_CHECK_ARG(volume >= 1 && volume <= 32, "one-hot order supports at most 32 offsets");
  SCB_CHECK_ARG(hits && perm && hits_out && tile_masks, "hits, perm, hits_out, tile_masks required");
  const SortWs w = sort_ws(n);
  SCB_CHECK_ARG(ws_bytes >= (int64_t)w.total, "workspace too small");
  if (n == 0) return SCB_OK;
  cudaStream_t s = as_stream(stream);
  char* base = (char*)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
  auto* kin = (uint32_t*)base;
  auto* kout = (uint32_t*)(base + w.keys_in);
  auto* vin = (int*)(base + w.keys_in + w.keys_out);
  void* tmp = base + w.keys_in + w.keys_out + w.vals_in;
  size_t tb = w.tmp;
  const long long ld = hits_ld(n);
  onehot_keys_kernel<<<blocks_for(n, RT), RT, 0, s>>>(hits, ld, volume, n, kin, vin);
  SCB_LAUNCHED();
  int end_bit = 1;
  while ((volume >> end_bit) != 0) ++end_bit;
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, perm, (int64_t)n, 0, end_bit, s));
  const long long tiles = (n + 127) / 128;
  onehot_apply_kernel<<<(int)(tiles < 148 * 16 ? tiles : 148 * 16), 128, 0, s>>>(
      hits, ld, volume, n, kout, perm, hits_out, tile_masks);
  SCB_LAUNCHED();
  return SCB_OK;
}
