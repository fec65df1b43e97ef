// Data movement on sm_100a: gather into the offset-major buffer, the
// output-stationary scatter (+ centre add + pointwise epilogue), pointwise
// ops, residual add, fp16 quantisation and fp16 weight packing.  All are
// HBM-bound streaming kernels: 128-bit vector accesses, grids
// sized in multiples of the SM count, no atomics.
#include "common.cuh"

namespace scb {

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

static int blocks_for(long long work, int threads, int per_sm = 8) {
  long long b = (work + threads - 1) / threads;
  long long cap = (long long)sm_count() * per_sm;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

// ------------------------------------------------------------------ gather
// buffer[r, :] = features[buf_in[r], :], vector type VT (16/8/4/2 bytes).
// One thread moves one vector; rows are walked in buffer order so stores are
// fully coalesced and the (L2-resident) feature rows are read with 128-bit
// loads.  Padding rows (buf_in < 0) are zero-filled so the GEMM never sees
// non-finite garbage.
template <typename VT, int UNROLL = 4>
__global__ void __launch_bounds__(256) gather_kernel(const VT* __restrict__ feat, long long ldf_v,
                                                     const int* __restrict__ buf_in,
                                                     long long rows, int vecs_per_row,
                                                     VT* __restrict__ buf, long long ldb_v,
                                                     const long long* __restrict__ rows_dev) {
  if (rows_dev) rows = min(rows, *rows_dev);  // device-built plans: rows in use
  const long long total = rows * vecs_per_row;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // UNROLL independent (index load -> row load -> store) chains per thread so
  // each warp keeps several L2 requests in flight.
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < total;
       base += UNROLL * stride) {
    long long r[UNROLL];
    int v[UNROLL], src[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const long long t = base + u * stride;
      if (total < (1LL << 31)) {  // 32-bit division (a 64-bit one is ~4x the instructions)
        const unsigned q = (unsigned)t / (unsigned)vecs_per_row;
        r[u] = q;
        v[u] = (int)((unsigned)t - q * (unsigned)vecs_per_row);
      } else {
        r[u] = t / vecs_per_row;
        v[u] = (int)(t - r[u] * vecs_per_row);
      }
      src[u] = t < total ? __ldg(buf_in + r[u]) : -1;
    }
    VT val[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (src[u] >= 0) val[u] = __ldg(feat + src[u] * ldf_v + v[u]);
      else memset(&val[u], 0, sizeof(VT));
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)  // streaming stores: the buffer is read once, by the GEMM
      if (base + u * stride < total) __stcs(buf + r[u] * ldb_v + v[u], val[u]);
  }
}

template <typename VT>
static void launch_gather(const void* f, long long ldf_b, const int* buf_in, long long rows,
                          long long row_b, void* buf, long long ldb_b, const long long* rows_dev,
                          cudaStream_t s) {
  const int vpr = (int)(row_b / sizeof(VT));
  gather_kernel<VT><<<blocks_for(rows * vpr, 256), 256, 0, s>>>(
      (const VT*)f, ldf_b / (long long)sizeof(VT), buf_in, rows, vpr, (VT*)buf,
      ldb_b / (long long)sizeof(VT), rows_dev);
}

// ------------------------------------------------------------------ scatter
template <typename T> __device__ __forceinline__ void store_out(T* p, float v);
template <> __device__ __forceinline__ void store_out<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void store_out<__half>(__half* p, float v) {
  *p = __float2half_rn(v);
}

template <typename T> __device__ __forceinline__ float ld_f(const T* p);
template <> __device__ __forceinline__ float ld_f<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_f<__half>(const __half* p) { return __half2float(*p); }

struct Epi {
  const float* scale;
  const float* shift;
  const float* bias;
  const void* residual;  // same dtype/shape as the output, nullable
  int relu;
};

template <typename T>
__device__ __forceinline__ float epilogue(float a, long long k, int c, long long ldo,
                                          const Epi& e) {
  if (e.scale) a = a * __ldg(e.scale + c) + __ldg(e.shift + c);
  if (e.bias) a = a + __ldg(e.bias + c);
  if (e.residual) a = a + ld_f<T>(reinterpret_cast<const T*>(e.residual) + k * ldo + c);
  if (e.relu) a = fmaxf(a, 0.f);
  return a;
}

// Output-stationary fold (kernels.py:38-50): one thread group owns output row
// k, walks its V buffer positions in ascending offset order (== ascending
// buffer row, the reference's fold order), accumulates in f32 registers and
// writes the row exactly once.  Each thread owns 4 consecutive channels
// (float4 loads of the partial rows).
template <typename OutT, int VEC>
__global__ void __launch_bounds__(256) scatter_kernel(const float* __restrict__ partial,
                                                      long long ldp,
                                                      const int* __restrict__ pos, int V,
                                                      long long n_out, int c_out, int groups,
                                                      long long center_row,
                                                      OutT* __restrict__ out, long long ldo,
                                                      Epi e) {
  const long long total = n_out * groups;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / groups;
    const int c0 = (int)(t - k * groups) * VEC;
    float acc[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
    const int* pk = pos + k * V;
    // Positions are read CH at a time and all their partial rows are loaded
    // before any is added, so up to CH row loads are in flight per thread;
    // the adds still run in ascending offset order (the reference's fold).
    constexpr int CH = 9;
    for (int n0 = 0; n0 < V; n0 += CH) {
      int r[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) r[u] = (n0 + u < V) ? __ldg(pk + n0 + u) : -1;
      if constexpr (VEC == 4) {
        float4 v[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u)
          v[u] = r[u] >= 0 ? __ldg(reinterpret_cast<const float4*>(partial + (long long)r[u] * ldp + c0))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          if (r[u] < 0) continue;
          acc[0] += v[u].x; acc[1] += v[u].y; acc[2] += v[u].z; acc[3] += v[u].w;
        }
      } else {
        for (int u = 0; u < CH; ++u) {
          if (r[u] < 0) continue;
          const float* src = partial + (long long)r[u] * ldp + c0;
#pragma unroll
          for (int i = 0; i < VEC; ++i)
            if (c0 + i < c_out) acc[i] += __ldg(src + i);
        }
      }
    }
    if (center_row >= 0) {
      const float* src = partial + (center_row + k) * ldp + c0;
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        if (c0 + i < c_out) acc[i] += __ldg(src + i);
    }
    if constexpr (VEC == 4 && sizeof(OutT) == 2) {
      // one 8-byte store of the four channels (row starts are 8-byte aligned
      // when the row stride is a multiple of 4; checked by the launcher)
      if (c0 + 4 <= c_out && (ldo & 3) == 0) {
        __half2 lo = __floats2half2_rn(epilogue<OutT>(acc[0], k, c0, ldo, e),
                                       epilogue<OutT>(acc[1], k, c0 + 1, ldo, e));
        __half2 hi = __floats2half2_rn(epilogue<OutT>(acc[2], k, c0 + 2, ldo, e),
                                       epilogue<OutT>(acc[3], k, c0 + 3, ldo, e));
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(out + k * ldo + c0) = w;
        continue;
      }
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      if (c0 + i < c_out)
        store_out<OutT>(out + k * ldo + c0 + i, epilogue<OutT>(acc[i], k, c0 + i, ldo, e));
  }
}

// General output-stationary fold over a CSR (reference
// scatter_accumulate with any plan, execution.py:183-218): output k sums
// buffer rows out_rows[out_ptr[k] .. out_ptr[k+1]) in that (ascending
// buffer-row) order in f32 and writes its row once.  Unlike scatter_kernel's
// fixed-width position table this takes any number of entries per
// (output, offset) pair -- maps built by hand through the reference API.
template <typename InT, typename OutT>
__global__ void __launch_bounds__(256) scatter_csr_kernel(const InT* __restrict__ buffer,
                                                          long long ldb,
                                                          const long long* __restrict__ out_ptr,
                                                          const int* __restrict__ out_rows,
                                                          long long n_out, int c,
                                                          OutT* __restrict__ out, long long ldo) {
  const long long total = n_out * c;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / c;
    const int ch = (int)(t - k * c);
    float acc = 0.f;
    for (long long e = __ldg(out_ptr + k), end = __ldg(out_ptr + k + 1); e < end; ++e)
      acc += ld_f<InT>(buffer + (long long)__ldg(out_rows + e) * ldb + ch);
    store_out<OutT>(out + k * ldo + ch, acc);
  }
}

// Small device -> pinned-host reads written by the SMs through the host
// pointer (UVA-mapped pinned memory) instead of a DMA copy: the copy engine
// may be busy with a large transfer on another stream (a batch's logits),
// and a count the compute stream needs must not queue behind it.
__global__ void store_to_host_kernel(const unsigned int* __restrict__ src,
                                     volatile unsigned int* dst, long long words) {
  for (long long i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}

// ------------------------------------------------------------------ pointwise
template <typename T>
__global__ void pointwise_kernel(T* __restrict__ x, long long n, int c, int op,
                                 const float* __restrict__ a, const float* __restrict__ b) {
  const long long total = n * c;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(i % c);
    float v = ld_f<T>(x + i);
    if (op == 0) v = fmaxf(v, 0.f);
    else if (op == 1) v = v + __ldg(a + ch);
    else v = v * __ldg(a + ch) + __ldg(b + ch);
    store_out<T>(x + i, v);
  }
}

template <typename T>
__global__ void add_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ o,
                           long long n, int relu) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float v = ld_f<T>(x + i) + ld_f<T>(y + i);
    if (relu) v = fmaxf(v, 0.f);
    store_out<T>(o + i, v);
  }
}

__global__ void quantize_kernel(const float* __restrict__ in, __half* __restrict__ out,
                                long long n, unsigned long long* sat) {
  unsigned int local = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = in[i];
    __half h = __float2half_rn(v);
    if (__hisinf(h) && isfinite(v)) {
      h = __float2half_rn(v > 0 ? 65504.f : -65504.f);
      ++local;
    }
    out[i] = h;
  }
  if (local) atomicAdd(sat, (unsigned long long)local);
}

// w[V][c_in][c_out] f32 -> packed[V][n_pad][k_pad] f16 (K-major B operand of
// the tcgen05 GEMM), zero padded.
__global__ void pack_weights_kernel(const float* __restrict__ w, int V, int c_in, int c_out,
                                    __half* __restrict__ packed, int k_pad, int n_pad) {
  const long long total = (long long)V * n_pad * k_pad;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int kk = (int)(i % k_pad);
    const int nn = (int)((i / k_pad) % n_pad);
    const int v = (int)(i / ((long long)k_pad * n_pad));
    float val = 0.f;
    if (kk < c_in && nn < c_out) val = w[((long long)v * c_in + kk) * c_out + nn];
    packed[i] = __float2half_rn(val);
  }
}

}  // namespace scb

using namespace scb;

extern "C" int32_t scb_gather(int32_t dtype, const void* features, int64_t n_in, int32_t channels,
                              int64_t ld_feat, const int32_t* buf_in, int64_t rows, void* buffer,
                              int64_t ld_buf, const int64_t* rows_dev, scb_stream_t stream) {
  (void)n_in;
  SCB_CHECK_ARG(dtype == SCB_F32 || dtype == SCB_F16, "dtype must be f32 or f16");
  SCB_CHECK_ARG(channels >= 1 && ld_feat >= channels && ld_buf >= channels, "bad strides");
  if (rows == 0) return SCB_OK;
  const int es = dtype == SCB_F32 ? 4 : 2;
  const long long row_b = (long long)channels * es, ldf_b = ld_feat * es, ldb_b = ld_buf * es;
  const uintptr_t align = (uintptr_t)features | (uintptr_t)buffer;
  auto fits = [&](long long w) {
    return row_b % w == 0 && ldf_b % w == 0 && ldb_b % w == 0 && align % w == 0;
  };
  cudaStream_t s = as_stream(stream);
  const long long* rd = (const long long*)rows_dev;
  if (fits(16)) launch_gather<int4>(features, ldf_b, buf_in, rows, row_b, buffer, ldb_b, rd, s);
  else if (fits(8)) launch_gather<int2>(features, ldf_b, buf_in, rows, row_b, buffer, ldb_b, rd, s);
  else if (fits(4)) launch_gather<int>(features, ldf_b, buf_in, rows, row_b, buffer, ldb_b, rd, s);
  else launch_gather<short>(features, ldf_b, buf_in, rows, row_b, buffer, ldb_b, rd, s);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_scatter(const float* partial, int64_t ldp, const int32_t* pos,
                               int32_t volume, int64_t n_out, int32_t c_out, int64_t center_row,
                               int32_t out_dtype, void* out, int64_t ld_out, const float* scale,
                               const float* shift, const float* bias, const void* residual,
                               int32_t relu,
                               scb_stream_t stream) {
  SCB_CHECK_ARG(out_dtype == SCB_F32 || out_dtype == SCB_F16, "dtype must be f32 or f16");
  SCB_CHECK_ARG((scale == nullptr) == (shift == nullptr), "scale and shift go together");
  if (n_out == 0) return SCB_OK;
  Epi e{scale, shift, bias, residual, relu};
  cudaStream_t s = as_stream(stream);
  const bool vec4 = (c_out % 4 == 0) && (ldp % 4 == 0) && ((uintptr_t)partial % 16 == 0);
  const int groups = vec4 ? c_out / 4 : c_out;
  const long long work = n_out * groups;
  const int nb = blocks_for(work, 256, 16);
  if (out_dtype == SCB_F32) {
    if (vec4)
      scatter_kernel<float, 4><<<nb, 256, 0, s>>>(partial, ldp, pos, volume, n_out, c_out, groups,
                                                  center_row, (float*)out, ld_out, e);
    else
      scatter_kernel<float, 1><<<nb, 256, 0, s>>>(partial, ldp, pos, volume, n_out, c_out, groups,
                                                  center_row, (float*)out, ld_out, e);
  } else {
    if (vec4)
      scatter_kernel<__half, 4><<<nb, 256, 0, s>>>(partial, ldp, pos, volume, n_out, c_out, groups,
                                                   center_row, (__half*)out, ld_out, e);
    else
      scatter_kernel<__half, 1><<<nb, 256, 0, s>>>(partial, ldp, pos, volume, n_out, c_out, groups,
                                                   center_row, (__half*)out, ld_out, e);
  }
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_scatter_csr(int32_t in_dtype, const void* buffer, int64_t ldb,
                                   const int64_t* out_ptr, const int32_t* out_rows, int64_t n_out,
                                   int32_t channels, int32_t out_dtype, void* out, int64_t ld_out,
                                   scb_stream_t stream) {
  SCB_CHECK_ARG(in_dtype == SCB_F32 || in_dtype == SCB_F16, "dtype must be f32 or f16");
  SCB_CHECK_ARG(out_dtype == SCB_F32 || out_dtype == SCB_F16, "dtype must be f32 or f16");
  SCB_CHECK_ARG(channels >= 1 && ldb >= channels && ld_out >= channels, "bad row strides");
  if (n_out == 0) return SCB_OK;
  cudaStream_t s = as_stream(stream);
  const int nb = blocks_for(n_out * channels, 256, 16);
#define SCB_SC_LAUNCH(IT, OT)                                                                  \
  scatter_csr_kernel<IT, OT><<<nb, 256, 0, s>>>((const IT*)buffer, ldb, (const long long*)out_ptr, \
                                                out_rows, n_out, channels, (OT*)out, ld_out)
  if (in_dtype == SCB_F32 && out_dtype == SCB_F32) SCB_SC_LAUNCH(float, float);
  else if (in_dtype == SCB_F32) SCB_SC_LAUNCH(float, __half);
  else if (out_dtype == SCB_F32) SCB_SC_LAUNCH(__half, float);
  else SCB_SC_LAUNCH(__half, __half);
#undef SCB_SC_LAUNCH
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_store_to_host(const void* src, void* host_dst, int64_t bytes,
                                     scb_stream_t stream) {
  SCB_CHECK_ARG(bytes >= 0 && bytes % 4 == 0 && bytes <= (1 << 20),
                "bytes must be a multiple of 4, at most 1 MiB");
  SCB_CHECK_ARG(((uintptr_t)src | (uintptr_t)host_dst) % 4 == 0, "4-byte aligned buffers");
  if (bytes == 0) return SCB_OK;
  store_to_host_kernel<<<1, 128, 0, as_stream(stream)>>>((const unsigned int*)src,
                                                         (volatile unsigned int*)host_dst,
                                                         bytes / 4);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_pointwise(int32_t dtype, void* features, int64_t n, int32_t channels,
                                 int32_t op, const float* a, const float* b,
                                 scb_stream_t stream) {
  SCB_CHECK_ARG(op >= 0 && op <= 2, "unknown pointwise op");
  SCB_CHECK_ARG(op == 0 || a, "missing parameter vector");
  SCB_CHECK_ARG(op != 2 || b, "missing shift vector");
  if (n * channels == 0) return SCB_OK;
  cudaStream_t s = as_stream(stream);
  const int nb = blocks_for(n * channels, 256);
  if (dtype == SCB_F32) pointwise_kernel<float><<<nb, 256, 0, s>>>((float*)features, n, channels, op, a, b);
  else pointwise_kernel<__half><<<nb, 256, 0, s>>>((__half*)features, n, channels, op, a, b);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_add(int32_t dtype, const void* x, const void* y, void* out, int64_t count,
                           int32_t relu, scb_stream_t stream) {
  if (count == 0) return SCB_OK;
  cudaStream_t s = as_stream(stream);
  const int nb = blocks_for(count, 256);
  if (dtype == SCB_F32) add_kernel<float><<<nb, 256, 0, s>>>((const float*)x, (const float*)y, (float*)out, count, relu);
  else add_kernel<__half><<<nb, 256, 0, s>>>((const __half*)x, (const __half*)y, (__half*)out, count, relu);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_quantize_f16(const float* in, void* out, int64_t count, int64_t* n_saturated,
                                    scb_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  SCB_CUDA(cudaMemsetAsync(n_saturated, 0, sizeof(int64_t), s));
  if (count == 0) return SCB_OK;
  quantize_kernel<<<blocks_for(count, 256), 256, 0, s>>>(in, (__half*)out, count,
                                                         (unsigned long long*)n_saturated);
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_pack_weights_f16(const float* w, int32_t volume, int32_t c_in,
                                        int32_t c_out, void* packed, int32_t k_pad, int32_t n_pad,
                                        scb_stream_t stream) {
  SCB_CHECK_ARG(k_pad >= c_in && n_pad >= c_out, "padding smaller than the weight shape");
  const long long total = (long long)volume * k_pad * n_pad;
  if (total == 0) return SCB_OK;
  pack_weights_kernel<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(
      w, volume, c_in, c_out, (__half*)packed, k_pad, n_pad);
  SCB_LAUNCHED();
  return SCB_OK;
}
