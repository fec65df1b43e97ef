// Grouped GEMM of the sparse-conv forward (execute_groups, execution.py:331-368,
// plus the centre-offset matmul, execution.py:423-424) as ONE persistent
// launch per layer.
//
// FP16-storage path: tcgen05.mma (kind::f16, f32 accumulate in TMEM), TMA
// loads of A (gather buffer slab or, for the centre offset, the feature
// matrix itself) and B (per-offset weight slice, K-major fp16), TMA stores of
// f32 partial tiles.  Warp roles (192 threads, 1 CTA / SM):
//   warp 0  : TMA producer (one elected lane)
//   warp 1  : TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5: epilogue, TMEM -> registers -> swizzled smem -> TMA store
// Pipelines: smem ring (full/empty mbarriers, `stages` deep) between TMA and
// MMA; a 2-deep TMEM accumulator ring (tmem_full/tmem_empty) between MMA and
// the epilogue so tile i's epilogue overlaps tile i+1's MMAs.
//
// FP32 path: exact-f32 SIMT FMA (see the header for why not TF32).
#include <cuda.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace scb {
namespace tc {

constexpr int BM = 128;
constexpr int THREADS = 192;
constexpr int MAX_SEG = SCB_MAX_SEGMENTS;
constexpr int EPI_BUF_BYTES = 4096;  // 32 rows x 128 B
constexpr int EPI_BYTES = 4 * 2 * EPI_BUF_BYTES;

using Seg = SegDesc;

struct Params {
  int n_pad, kc, n_kchunks, epi_cols, stages, swz;
  uint32_t idesc, tmem_cols, a_stage_bytes, b_stage_bytes, stage_bytes, tx_bytes;
  const SegTable* dtab;  // device-built problem table (scb_plan_from_hits), else null
  SegTable tab;          // host-built table (by value in parameter space)
};

using namespace ::scb::ptx;

__device__ __forceinline__ int find_seg(const SegTable& T, int t) {
  int lo = 0, hi = T.n_segs;  // largest s with tile_start[s] <= t
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (T.tile_start[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(THREADS, 1)
    grouped_gemm_f16_kernel(const __grid_constant__ CUtensorMap tmA0,
                            const __grid_constant__ CUtensorMap tmA1,
                            const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ CUtensorMap tmC,
                            const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_base = smem + (size_t)p.stages * p.stage_bytes;
  uint64_t* full = (uint64_t*)(epi_base + EPI_BYTES);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SegTable& T = p.dtab ? *p.dtab : p.tab;
  // contiguous tile range per CTA: consecutive tiles share an offset's weights
  const int t_begin = (int)((long long)T.total_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long long)T.total_tiles * (blockIdx.x + 1) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA1) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; ++t) {
        const int s = find_seg(T, t);
        const Seg& sg = T.seg[s];
        const int a_row = (int)(sg.a_row + (long long)(t - T.tile_start[s]) * BM);
        const int b_row = sg.b_index * p.n_pad;
        const CUtensorMap* ma = sg.a_src ? &tmA1 : &tmA0;
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + (size_t)stage * p.stage_bytes;
          mbar_expect_tx(full + stage, p.tx_bytes);
          tma_load_2d(sa, ma, full + stage, kk * p.kc, a_row);
          tma_load_2d(sa + p.a_stage_bytes, &tmB, full + stage, kk * p.kc, b_row);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer
    if (lane == 0) {
      const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
      const uint32_t sbo = 8u * (uint32_t)p.swz;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = t_begin; t < t_end; ++t) {
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * p.n_pad);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          mbar_wait(full + stage, phase);
          tc_after();
          const uint32_t sa = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sb = sa + p.a_stage_bytes;
          for (int k = 0; k < p.kc / 16; ++k) {
            const uint64_t da = make_sdesc(sa + k * 32, sbo, layout);
            const uint64_t db = make_sdesc(sb + k * 32, sbo, layout);
            mma_f16(d_tmem, da, db, p.idesc, (kk | k) != 0);
          }
          mma_commit(empty + stage);  // frees the smem slot once these MMAs retire
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull + acc);  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ===================== epilogue: TMEM -> regs -> swizzled smem -> TMA store
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* bufs = epi_base + (warp - 2) * 2 * EPI_BUF_BYTES;
    int acc = 0, nbuf = 0;
    uint32_t acc_phase = 0;
    const int chunks = p.n_pad / p.epi_cols;
    for (int t = t_begin; t < t_end; ++t) {
      const int s = find_seg(T, t);
      const Seg& sg = T.seg[s];
      const int c_row = (int)(sg.c_row + (long long)(t - T.tile_start[s]) * BM) + 32 * q;
      mbar_wait(tfull + acc, acc_phase);
      tc_after();
      for (int j = 0; j < chunks; ++j) {
        const uint32_t taddr =
            tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * p.n_pad + j * p.epi_cols);
        uint32_t r[32];
        TMEM_LD_X16(taddr, r);
        if (p.epi_cols == 32) TMEM_LD_X16(taddr + 16, (r + 16));
        tmem_wait_ld();
        uint8_t* buf = bufs + nbuf * EPI_BUF_BYTES;
        if (lane == 0) bulk_wait_read1();  // the store that last used `buf` has read it
        __syncwarp();
        if (p.epi_cols == 32) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 v = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
            *reinterpret_cast<uint4*>(buf + lane * 128 + ((c ^ (lane & 7)) << 4)) = v;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 v = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
            *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = v;
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, buf, j * p.epi_cols, c_row);
          bulk_commit();
        }
        nbuf ^= 1;
      }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

}  // namespace tc

// ------------------------------------------------------------------ FP32 SIMT path
namespace simt {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int MAX_SEG = SCB_MAX_SEGMENTS;

using Seg = SegDesc;
struct Params {
  int ntn;
  const SegTable* dtab;  // device-built table (tiles = m-tiles of 64 x ntn), else null
  SegTable tab;
};

__global__ void __launch_bounds__(256) grouped_gemm_f32_kernel(
    const float* __restrict__ A0, long long lda, const float* __restrict__ A1, long long ldf,
    int c_in, const float* __restrict__ W, int c_out, float* __restrict__ C, long long ldc,
    const __grid_constant__ Params p) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const SegTable& T = p.dtab ? *p.dtab : p.tab;
  for (int t = blockIdx.x; t < T.total_tiles; t += gridDim.x) {
    int lo = 0, hi = T.n_segs;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (T.tile_start[mid] <= t) lo = mid; else hi = mid;
    }
    const Seg& sg = T.seg[lo];
    const int local = t - T.tile_start[lo];
    const int mt = local / p.ntn, nt = local % p.ntn;
    const int m0 = mt * BM, n0 = nt * BN;
    const float* A = sg.a_src ? A1 : A0;
    const long long ld = sg.a_src ? ldf : lda;
    const float* Wb = W + (long long)sg.b_index * c_in * c_out;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < c_in; k0 += BK) {
      for (int i = tid; i < BM * BK; i += 256) {
        const int r = i / BK, k = i % BK;
        float v = 0.f;
        if (m0 + r < sg.rows && k0 + k < c_in) v = A[(sg.a_row + m0 + r) * ld + k0 + k];
        As[k][r] = v;
      }
      for (int i = tid; i < BK * BN; i += 256) {
        const int k = i / BN, n = i % BN;
        float v = 0.f;
        if (k0 + k < c_in && n0 + n < c_out) v = Wb[(long long)(k0 + k) * c_out + n0 + n];
        Bs[k][n] = v;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + ty * 4 + i;
      if (r >= sg.rows) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n < c_out) C[(sg.c_row + r) * ldc + n] = acc[i][j];
      }
    }
  }
}

}  // namespace simt

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)ptr;
  }();
  return fn;
}

static CUtensorMapSwizzle swizzle_of(int bytes) {
  return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                      : (bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

bool encode_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                        long long inner, long long rows, long long ld, int box_inner, int box_rows,
                        int swz_bytes, std::string& err) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(swz_bytes),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

bool encode_map_1d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, long long n, int box,
                   std::string& err) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[1] = {(cuuint64_t)(n > 0 ? n : 1)};
  cuuint64_t strides[1] = {0};
  cuuint32_t boxd[1] = {(cuuint32_t)box};
  cuuint32_t estr[1] = {1};
  CUresult r = fn(m, dt, 1, const_cast<void*>(base), dims, strides, boxd, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled (1-D) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

int device_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Host-built table from a segment list (tile = `bm` rows x `ntn` column tiles).
static int build_table(SegTable& T, const scb_segment_t* segs, int n_segs, int volume,
                       const void* a_features, long long c_rows, int bm, int ntn, bool pad_rows) {
  SCB_CHECK_ARG(n_segs <= SCB_MAX_SEGMENTS, "too many GEMM segments");
  memset(&T, 0, sizeof(T));
  int tiles = 0, used = 0;
  for (int i = 0; i < n_segs; ++i) {
    if (segs[i].rows <= 0) continue;
    SCB_CHECK_ARG(segs[i].b_index >= 0 && segs[i].b_index < volume, "segment weight index");
    SCB_CHECK_ARG(segs[i].a_src == 0 || a_features != nullptr, "centre segment needs features");
    const int mt = (segs[i].rows + bm - 1) / bm;
    SCB_CHECK_ARG(segs[i].c_row + (pad_rows ? (long long)mt * bm : segs[i].rows) <= c_rows,
                  "partial buffer too small");
    SegDesc& d = T.seg[used];
    d.a_row = segs[i].a_row;
    d.c_row = segs[i].c_row;
    d.rows = segs[i].rows;
    d.b_index = segs[i].b_index;
    d.a_src = segs[i].a_src;
    T.tile_start[used] = tiles;
    tiles += mt * ntn;
    ++used;
  }
  T.n_segs = used;
  T.tile_start[used] = tiles;
  T.total_tiles = tiles;
  return SCB_OK;
}

static int gemm_f16(const void* a_buffer, long long a_rows, long long lda, const void* a_features,
                    long long f_rows, long long ldf, int c_in, const void* w_packed, int volume,
                    int c_out, float* partial, long long c_rows, long long ldc,
                    const scb_segment_t* segs, int n_segs, const SegTable* dtab,
                    cudaStream_t stream) {
  using namespace tc;
  const int n_pad = (c_out + 15) / 16 * 16;
  const int k_pad = (c_in + 15) / 16 * 16;
  SCB_CHECK_ARG(n_pad <= 256, "c_out > 256 is not supported by the tcgen05 path");
  SCB_CHECK_ARG(ldc == n_pad, "partial stride must equal roundup(c_out, 16)");
  SCB_CHECK_ARG(lda % 8 == 0 && (ldf % 8 == 0 || a_features == nullptr),
                "A row strides must be multiples of 8 elements (16 B) for TMA");
  Params p;
  memset(&p, 0, sizeof(p));
  p.n_pad = n_pad;
  p.kc = (k_pad % 64 == 0) ? 64 : ((k_pad % 32 == 0) ? 32 : 16);
  p.swz = p.kc * 2;
  p.n_kchunks = k_pad / p.kc;
  p.epi_cols = (n_pad % 32 == 0) ? 32 : 16;
  p.idesc = (1u << 4) | ((uint32_t)(n_pad >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * n_pad)) cols *= 2;
  p.tmem_cols = cols;
  auto r1024 = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  p.a_stage_bytes = r1024((uint32_t)(BM * p.kc * 2));
  p.b_stage_bytes = r1024((uint32_t)(n_pad * p.kc * 2));
  p.stage_bytes = p.a_stage_bytes + p.b_stage_bytes;
  p.tx_bytes = (uint32_t)(BM * p.kc * 2 + n_pad * p.kc * 2);
  const int smem_cap = 227 * 1024;
  const int fixed = 1024 + EPI_BYTES + 256;
  int stages = (smem_cap - fixed) / (int)p.stage_bytes;
  if (stages > 8) stages = 8;
  SCB_CHECK_ARG(stages >= 2, "stage does not fit in shared memory");
  p.stages = stages;
  const int smem = fixed + stages * (int)p.stage_bytes;

  int grid = device_sms();
  if (dtab) {
    p.dtab = dtab;  // tile count known on the device only: one persistent CTA per SM
  } else {
    const int rc = build_table(p.tab, segs, n_segs, volume, a_features, c_rows, BM, 1, true);
    if (rc != SCB_OK) return rc;
    if (p.tab.total_tiles == 0) return SCB_OK;
    if (p.tab.total_tiles < grid) grid = p.tab.total_tiles;
  }

  CUtensorMap mA0, mA1, mB, mC;
  std::string err;
  const void* a1 = a_features ? a_features : a_buffer;
  const long long a1_rows = a_features ? f_rows : a_rows, a1_ld = a_features ? ldf : lda;
  bool ok = encode_map_2d(&mA0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a_buffer, c_in, a_rows, lda, p.kc,
                        BM, p.swz, err) &&
            encode_map_2d(&mA1, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a1, c_in, a1_rows, a1_ld, p.kc, BM,
                        p.swz, err) &&
            encode_map_2d(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, k_pad,
                        (long long)volume * n_pad, k_pad, p.kc, n_pad, p.swz, err) &&
            encode_map_2d(&mC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, partial, n_pad, c_rows, ldc,
                        p.epi_cols, 32, p.epi_cols * 4, err);
  if (!ok) {
    set_error(std::string("scb_grouped_gemm: ") + err);
    return SCB_ECUDA;
  }
  static int configured = 0;
  if (!configured) {
    SCB_CUDA(cudaFuncSetAttribute(grouped_gemm_f16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_cap));
    configured = 1;
  }
  grouped_gemm_f16_kernel<<<grid, THREADS, smem, stream>>>(mA0, mA1, mB, mC, p);
  SCB_LAUNCHED();
  return SCB_OK;
}

static int gemm_f32(const void* a_buffer, long long lda, const void* a_features, long long ldf,
                    int c_in, const void* w, int volume, int c_out, float* partial,
                    long long c_rows, long long ldc, const scb_segment_t* segs, int n_segs,
                    const SegTable* dtab, cudaStream_t stream) {
  using namespace simt;
  SCB_CHECK_ARG(ldc >= c_out, "partial stride smaller than c_out");
  Params p;
  memset(&p, 0, sizeof(p));
  p.ntn = (c_out + BN - 1) / BN;
  int grid = device_sms() * 8;
  if (dtab) {
    p.dtab = dtab;
  } else {
    const int rc = build_table(p.tab, segs, n_segs, volume, a_features, c_rows, BM, p.ntn, false);
    if (rc != SCB_OK) return rc;
    if (p.tab.total_tiles == 0) return SCB_OK;
    if (p.tab.total_tiles < grid) grid = p.tab.total_tiles;
  }
  grouped_gemm_f32_kernel<<<grid, 256, 0, stream>>>((const float*)a_buffer, lda,
                                                    (const float*)a_features, ldf, c_in,
                                                    (const float*)w, c_out, partial, ldc, p);
  SCB_LAUNCHED();
  return SCB_OK;
}

}  // namespace scb

extern "C" int32_t scb_gemm_tile_geometry(int32_t dtype, int32_t c_out, int32_t* bm,
                                          int32_t* ntn) {
  if (dtype == SCB_F16) {
    *bm = scb::tc::BM;
    *ntn = 1;
  } else {
    *bm = scb::simt::BM;
    *ntn = (c_out + scb::simt::BN - 1) / scb::simt::BN;
  }
  return SCB_OK;
}

extern "C" int32_t scb_grouped_gemm(int32_t dtype, const void* a_buffer, int64_t a_rows,
                                    int64_t lda, const void* a_features, int64_t f_rows,
                                    int64_t ldf, int32_t c_in, const void* weights, int32_t volume,
                                    int32_t c_out, float* partial, int64_t c_rows, int64_t ldc,
                                    const scb_segment_t* segments, int32_t n_segments,
                                    scb_stream_t stream) {
  SCB_CHECK_ARG(c_in >= 1 && c_out >= 1 && volume >= 1, "bad GEMM shape");
  SCB_CHECK_ARG(n_segments >= 0 && (segments || n_segments == 0), "bad segment table");
  cudaStream_t s = scb::as_stream(stream);
  if (dtype == SCB_F16)
    return scb::gemm_f16(a_buffer, a_rows, lda, a_features, f_rows, ldf, c_in, weights, volume,
                         c_out, partial, c_rows, ldc, segments, n_segments, nullptr, s);
  if (dtype == SCB_F32)
    return scb::gemm_f32(a_buffer, lda, a_features, ldf, c_in, weights, volume, c_out, partial,
                         c_rows, ldc, segments, n_segments, nullptr, s);
  scb::set_error("scb_grouped_gemm: dtype must be f32 or f16");
  return SCB_EINVAL;
}

extern "C" int32_t scb_grouped_gemm_table(int32_t dtype, const void* a_buffer, int64_t a_rows,
                                          int64_t lda, const void* a_features, int64_t f_rows,
                                          int64_t ldf, int32_t c_in, const void* weights,
                                          int32_t volume, int32_t c_out, float* partial,
                                          int64_t c_rows, int64_t ldc, const void* table,
                                          scb_stream_t stream) {
  SCB_CHECK_ARG(c_in >= 1 && c_out >= 1 && volume >= 1, "bad GEMM shape");
  SCB_CHECK_ARG(table != nullptr, "missing device problem table");
  cudaStream_t s = scb::as_stream(stream);
  const auto* t = (const scb::SegTable*)table;
  if (dtype == SCB_F16)
    return scb::gemm_f16(a_buffer, a_rows, lda, a_features, f_rows, ldf, c_in, weights, volume,
                         c_out, partial, c_rows, ldc, nullptr, 0, t, s);
  if (dtype == SCB_F32)
    return scb::gemm_f32(a_buffer, lda, a_features, ldf, c_in, weights, volume, c_out, partial,
                         c_rows, ldc, nullptr, 0, t, s);
  scb::set_error("scb_grouped_gemm_table: dtype must be f32 or f16");
  return SCB_EINVAL;
}
