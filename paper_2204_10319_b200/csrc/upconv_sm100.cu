// Transposed K = s convolution (the decoder's k2 s2 "up" layers,
// inverse_conv_forward, execution.py:530-551, on a map made by
// KernelMap.swap_roles of the encoder's k2 s2 map) in SCATTER form.
//
// The swapped map is one-hot: every fine output row k has exactly one entry
// (its coarse parent p, at the offset n with k = s p + delta_n).  The
// gather-form fused kernel therefore runs 128-row output tiles whose rows
// mostly sit at different offsets (~6 live offsets per tile, each almost all
// zero-filled).  Here the coarse side drives instead:
//
//   for each 128-row tile of coarse rows p, for each offset n:
//     acc = x[p-tile] . W[n]                        (tcgen05, A read once per tile)
//     out[child[n][p]] = epilogue(acc[p])           (child = the encoder map's
//                                                    hit matrix; -1 -> no store)
//
// A is a dense TMA tile of the input features (no gather at all) loaded with
// the tile's V x 128 child words into an A ring; B is the packed weights,
// resident in shared memory when all V slices fit beside two A slots, else
// streamed from L2 one offset slice per ring stage.  Accumulators rotate
// through TMEM (4 x n_pad columns) so the scattering epilogue of (tile, n)
// overlaps the MMAs of later offsets.  Each output row is written exactly once
// (full rows, 16-B stores by the lane that owns the coarse row): no atomics,
// no zero-init.  Executed FLOPs are V / (fine rows per coarse row) ~ 3.3x the
// useful ones at level 0.
//
// Measured (level 1 -> 0 of the bench's 8-scan pack, 96 -> 96 + BN + ReLU,
// 424k coarse rows; tools/up_probe.py, SCB_UP_DEBUG): 0.156 ms vs 0.267 ms
// for the gather-form fused kernel.  Without stores 0.141, without any
// epilogue work 0.140, without MMAs too 0.125 (ncu): the epilogue warps wait
// on the accumulator-full barrier most of the time while the MMA thread
// rarely waits; not HBM (95 MB read + 192 MB written in 0.156 ms ~ 1.8 TB/s).
// DESIGN.md §3 lists the variants measured slower.
//
// Warp roles (352 threads, persistent, 1 CTA per SM):
//   warp 0      A producer (TMA tiles of x + bulk copies of the child words)
//   warp 1      TMEM allocator + MMA issuer
//   warps 2..9  epilogue, two groups of four draining alternate (tile, n)
//               units: tcgen05.ld -> BN / bias / ReLU -> fp16 -> scattered rows
//   warp 10     B producer (weight slices)
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace scb {
namespace up {

using namespace ::scb::ptx;

constexpr int BM = 128;
constexpr int EPI_WARPS = 8;  // epilogue warps 2 .. 9
constexpr int THREADS = 32 * (3 + EPI_WARPS);  // + A producer 0, MMA 1, B producer 10
constexpr int MAX_A = 4;      // A-tile ring depth cap
constexpr int MAX_STAGES = 32;

struct Params {
  long long n_in;            // coarse rows
  long long ldc;             // child-matrix row stride
  long long ldo;             // output row stride (elements)
  int c_out, V, n_pad, kc, n_kchunks, relu;
  int nacc;                  // TMEM accumulators (each n_pad columns)
  int b_resident;            // all V x n_kchunks weight chunks live in smem
  int b_stages;              // else: ring depth
  int b_kg;                  // streamed: K chunks per ring stage
  int debug;                 // EXPERIMENT (SCB_UP_DEBUG, results wrong): 1 = no stores,
                             // 2 = no TMEM loads / math, 4 = no MMAs, 8 = no A / child copies
  int a_stages;              // A-tile ring depth (each slot: the tile + its V x 128 child words)
  int total_tiles;
  uint32_t idesc, tmem_cols, swz;
  uint32_t a_chunk_bytes;    // one K chunk of an A tile: 128 x kc fp16
  uint32_t b_chunk_bytes;    // slot stride of one K chunk of a weight slice (1024-aligned)
  uint32_t b_tx;             // bytes one weight-chunk load delivers: n_pad x kc fp16
  const int* child;          // [V][ldc] fine output row or -1; NULL = identity (V = 1)
  int a_split;               // K chunks read from x (the rest from x2, the concatenation)
  const float* scale;        // nullable (with shift)
  const float* shift;
  const float* bias;         // nullable
  __half* out;
};

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

constexpr int EPI_AFFINE = 1, EPI_BIAS = 2, EPI_RELU = 4;

// 8 accumulator columns -> BN scale/shift, bias, ReLU (the fused kernel's
// order) -> 8 fp16.  epi_s: scale[256], shift[256], bias[256] in smem.
template <int EPI>
__device__ __forceinline__ uint4 emit8(const uint32_t* r, const float* epi_s, int col) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  if (EPI & EPI_AFFINE) {
    const float4 s0 = *reinterpret_cast<const float4*>(epi_s + col);
    const float4 s1 = *reinterpret_cast<const float4*>(epi_s + col + 4);
    const float4 t0 = *reinterpret_cast<const float4*>(epi_s + 256 + col);
    const float4 t1 = *reinterpret_cast<const float4*>(epi_s + 256 + col + 4);
    v[0] = v[0] * s0.x + t0.x; v[1] = v[1] * s0.y + t0.y;
    v[2] = v[2] * s0.z + t0.z; v[3] = v[3] * s0.w + t0.w;
    v[4] = v[4] * s1.x + t1.x; v[5] = v[5] * s1.y + t1.y;
    v[6] = v[6] * s1.z + t1.z; v[7] = v[7] * s1.w + t1.w;
  }
  if (EPI & EPI_BIAS) {
    const float4 b0 = *reinterpret_cast<const float4*>(epi_s + 512 + col);
    const float4 b1 = *reinterpret_cast<const float4*>(epi_s + 512 + col + 4);
    v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
    v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
  }
  if (EPI & EPI_RELU) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  return make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                    pack_half2(v[6], v[7]));
}

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    upconv_scatter_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmA2,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base, derived from smem_raw so shared-window accesses stay LDS/STS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_tile_bytes = p.a_chunk_bytes * p.n_kchunks;
  const int AS = p.a_stages;
  uint8_t* a_base = smem;                               // AS A tiles
  uint8_t* b_base = smem + (size_t)AS * a_tile_bytes;   // weights (resident or ring)
  const int b_slots = p.b_resident ? p.V * p.n_kchunks : p.b_stages * p.b_kg;
  uint64_t* bars = (uint64_t*)(b_base + (size_t)b_slots * p.b_chunk_bytes);
  uint64_t* a_full = bars;                  // [AS] A tile + its child words landed
  uint64_t* a_empty = a_full + MAX_A;       // [AS] the tile's MMAs retired
  uint64_t* c_empty = a_empty + MAX_A;      // [AS] the epilogue is done with its child words
  uint64_t* tfull = c_empty + MAX_A;        // [nacc]
  uint64_t* tempty = tfull + 4;             // [nacc]
  uint64_t* b_full = tempty + 4;            // [b_slots] (resident: [0] only)
  uint64_t* b_empty = b_full + MAX_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(b_empty + MAX_STAGES);
  int* child_s = (int*)(tmem_slot + 4);     // [AS][V][128]
  float* epi_s = (float*)(child_s + AS * p.V * BM);   // scale[256], shift[256], bias[256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < AS; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, 1);
      mbar_init(c_empty + i, EPI_WARPS);
    }
    for (int i = 0; i < p.nacc; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 4);
    }
    for (int i = 0; i < (p.b_resident ? 1 : p.b_stages); ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA2) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < p.n_pad; i += THREADS) {   // padding columns: identity
    const bool c = i < p.c_out;
    epi_s[i] = p.scale && c ? p.scale[i] : 1.f;
    epi_s[256 + i] = p.shift && c ? p.shift[i] : 0.f;
    epi_s[512 + i] = p.bias && c ? p.bias[i] : 0.f;
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== A producer: tiles of x + their child words, AS deep
    if (lane == 0) {
      int ab = 0;
      uint32_t a_ph = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        mbar_wait(c_empty + ab, a_ph ^ 1);
        mbar_wait(a_empty + ab, a_ph ^ 1);
        // child words: V rows of 128 (bulk copies; 16-B multiples, the hit
        // matrix's row stride is a multiple of 4)
        const long long r0 = (long long)t * BM;
        const uint32_t cbytes = p.child ? (uint32_t)(min((long long)BM, p.ldc - r0) * 4) : 0u;
        if (p.debug & 8) { mbar_arrive(a_full + ab); if (++ab == AS) { ab = 0; a_ph ^= 1; } continue; }
        mbar_expect_tx(a_full + ab, a_tile_bytes + cbytes * (uint32_t)p.V);
        for (int n = 0; n < p.V && cbytes; ++n)
          bulk_load(smem_u32(child_s + (ab * p.V + n) * BM), p.child + n * p.ldc + r0, cbytes,
                    a_full + ab);
        // K chunks [0, a_split) from x, the rest from the concatenated x2
        for (int kk = 0; kk < p.n_kchunks; ++kk)
          tma_load_2d(a_base + (size_t)ab * a_tile_bytes + (size_t)kk * p.a_chunk_bytes,
                      kk < p.a_split ? &tmA : &tmA2, a_full + ab,
                      (kk < p.a_split ? kk : kk - p.a_split) * p.kc, t * BM);
        if (++ab == AS) { ab = 0; a_ph ^= 1; }
      }
    }
  } else if (warp == 2 + EPI_WARPS) {
    // ===================== B producer: weight slices, resident or streamed per (tile, n, k)
    if (lane == 0) {
      if (p.b_resident) {
        mbar_expect_tx(b_full, p.b_tx * (uint32_t)(p.V * p.n_kchunks));
        for (int n = 0; n < p.V; ++n)
          for (int kk = 0; kk < p.n_kchunks; ++kk)
            tma_load_2d(b_base + (size_t)(n * p.n_kchunks + kk) * p.b_chunk_bytes, &tmB, b_full,
                        kk * p.kc, n * p.n_pad);
      } else {
        int bs = 0;
        uint32_t b_ph = 0;
        // one ring stage = one offset's whole slice (all K chunks): one wait
        // and one commit per (tile, offset) on the MMA side
        // (b_kg K chunks when the whole slice is too large for two stages)
        const size_t stage_bytes = (size_t)p.b_kg * p.b_chunk_bytes;
        for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x)
          for (int n = 0; n < p.V; ++n)
            for (int k0 = 0; k0 < p.n_kchunks; k0 += p.b_kg) {
              mbar_wait(b_empty + bs, b_ph ^ 1);
              mbar_expect_tx(b_full + bs, p.b_tx * (uint32_t)p.b_kg);
              for (int kk = 0; kk < p.b_kg; ++kk)
                tma_load_2d(b_base + bs * stage_bytes + (size_t)kk * p.b_chunk_bytes, &tmB,
                            b_full + bs, (k0 + kk) * p.kc, n * p.n_pad);
              if (++bs == p.b_stages) { bs = 0; b_ph ^= 1; }
            }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer
    if (lane == 0) {
      const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
      const uint32_t sbo = 8u * p.swz;
      if (p.b_resident) {
        mbar_wait(b_full, 0);
        tc_after();
      }
      int ab = 0, bs = 0, acc = 0;
      uint32_t a_ph = 0, b_ph = 0, acc_ph = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        mbar_wait(a_full + ab, a_ph);
        tc_after();
        const uint32_t sa0 = smem_u32(a_base + (size_t)ab * a_tile_bytes);
        for (int n = 0; n < p.V; ++n) {
          mbar_wait(tempty + acc, acc_ph ^ 1);
          tc_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * p.n_pad);
          const int kg = p.b_resident ? p.n_kchunks : p.b_kg;
          for (int k0 = 0; k0 < p.n_kchunks; k0 += kg) {
            uint32_t sb0;
            if (p.b_resident) {
              sb0 = smem_u32(b_base + (size_t)n * p.n_kchunks * p.b_chunk_bytes);
            } else {
              mbar_wait(b_full + bs, b_ph);
              tc_after();
              sb0 = smem_u32(b_base + (size_t)bs * p.b_kg * p.b_chunk_bytes);
            }
            for (int kk = 0; kk < kg; ++kk) {
              const uint32_t sa = sa0 + (k0 + kk) * p.a_chunk_bytes;
              const uint32_t sb = sb0 + kk * p.b_chunk_bytes;
              for (int k = 0; k < p.kc / 16 && !(p.debug & 4); ++k)
                mma_f16(d_tmem, make_sdesc(sa + k * 32, sbo, layout),
                        make_sdesc(sb + k * 32, sbo, layout), p.idesc, ((k0 + kk) | k) != 0);
            }
            if (!p.b_resident) {
              mma_commit(b_empty + bs);
              if (++bs == p.b_stages) { bs = 0; b_ph ^= 1; }
            }
          }
          mma_commit(tfull + acc);
          if (++acc == p.nacc) { acc = 0; acc_ph ^= 1; }
        }
        mma_commit(a_empty + ab);  // the A tile is free once its last MMAs retire
        if (++ab == AS) { ab = 0; a_ph ^= 1; }
      }
    }
  } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
    // ===================== epilogue: two groups of four warps drain alternate
    // units (warp w reads TMEM lanes 32 (w % 4) ..; group g takes the units
    // u = g, g + 2, ... whose accumulators are u % nacc, nacc even)
    const int q = warp & 3;
    const int g = (warp - 2) >> 2;
    const int cols = p.n_pad;
    int acc = g, cb = 0, u = 0;
    uint32_t acc_ph = 0, c_ph = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      const long long prow = (long long)t * BM + 32 * q + lane;   // coarse row
      mbar_wait_sleep(a_full + cb, c_ph, 32);
      const int* cw = child_s + cb * p.V * BM + 32 * q + lane;
      for (int n = 0; n < p.V; ++n, ++u) {
        if ((u & 1) != g) continue;
        const long long k = prow >= p.n_in ? -1LL : (p.child ? (long long)cw[n * BM] : prow);
        mbar_wait_sleep(tfull + acc, acc_ph, 32);
        tc_after();
        if (!(p.debug & 2) && __any_sync(0xffffffffu, k >= 0)) {
          for (int c0 = 0; c0 < cols; c0 += 64) {
            const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * p.n_pad + c0);
            const int nc = cols - c0 >= 64 ? 64 : cols - c0;   // multiple of 16
            uint32_t r[64];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (16 * j < nc) TMEM_LD_X16(taddr + 16 * j, (r + 16 * j));
            tmem_wait_ld();
            if (k >= 0 && !(p.debug & 1)) {
              uint4* dst = reinterpret_cast<uint4*>(p.out + k * p.ldo + c0);
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                if (8 * c < nc && c0 + 8 * c < p.c_out)
                  dst[c] = emit8<EPI>(r + 8 * c, epi_s, c0 + 8 * c);
              }
            }
          }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + acc);
        acc += 2;
        if (acc >= p.nacc) { acc -= p.nacc; acc_ph ^= 1; }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(c_empty + cb);
      if (++cb == AS) { cb = 0; c_ph ^= 1; }
    }
  }

  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

}  // namespace up

bool cached_map_f16(CUtensorMap* out, const void* base, long long inner, long long rows, long long ld,
                    int box_inner, int box_rows, int swz, std::string& err);
int device_sms();

}  // namespace scb

using namespace scb;

namespace {

// Shared launcher: the transposed scatter form (child != NULL) and the dense
// pointwise form (child == NULL: identity rows, V = 1, optional concat).
int32_t launch_dense(const char* name, const void* features, int64_t ldf, int32_t c_split,
                     const void* features2, int64_t ldf2, int64_t n_in, int32_t c_in,
                     const int32_t* child, int32_t volume, const void* weights_packed,
                     int32_t c_out, void* out, int64_t ldo, const float* scale,
                     const float* shift, const float* bias, int32_t relu, scb_stream_t stream) {
  using namespace up;
  auto bad = [&](const char* msg) {
    set_error(std::string(name) + ": " + msg);
    return SCB_EINVAL;
  };
  if (!features || !weights_packed || !out) return bad("features, weights and out are required");
  if (!child && volume != 1) return bad("the identity form has volume 1");
  if (volume < 1 || volume > 32) return bad("volume must be in [1, 32]");
  if (c_in < 8 || c_in % 8 != 0 || c_in > 256) return bad("c_in must be a multiple of 8 in [8, 256]");
  if (c_out < 1 || c_out > 256) return bad("c_out must be in [1, 256]");
  if (ldf < (features2 ? c_split : c_in) || ldf % 8 != 0)
    return bad("ldf must cover the channels and be a multiple of 8");
  // rows are stored in 8-column groups: a C_out that is not a multiple of 8
  // (the 19-class head) also writes the padding columns of its 8-aligned rows
  if (ldo < (c_out + 7) / 8 * 8 || ldo % 8 != 0)
    return bad("ldo must be a multiple of 8 covering c_out rounded up to 8");
  if ((scale == nullptr) != (shift == nullptr)) return bad("scale and shift go together");
  if (n_in <= 0) return SCB_OK;
  if (n_in >= (1LL << 31) - BM) return bad("n_in too large");
  const int n_pad = (c_out + 15) / 16 * 16;
  const int k_pad = (c_in + 15) / 16 * 16;
  Params p;
  memset(&p, 0, sizeof(p));
  p.n_in = n_in;
  p.ldc = hits_ld(n_in);
  p.ldo = ldo;
  p.c_out = c_out;
  p.V = volume;
  p.n_pad = n_pad;
  // K chunk: the widest dividing k_pad (and the concat split, so no chunk
  // straddles the two sources)
  p.kc = 64;
  while (p.kc > 16 && (k_pad % p.kc != 0 || (features2 && c_split % p.kc != 0))) p.kc /= 2;
  if (features2 && c_split % p.kc != 0) {
    set_error(std::string(name) + ": the concat split must be a multiple of 16 channels");
    return SCB_EINVAL;
  }
  p.swz = (uint32_t)p.kc * 2;
  p.n_kchunks = k_pad / p.kc;
  p.a_split = features2 ? c_split / p.kc : p.n_kchunks;
  p.relu = relu;
  p.idesc = (1u << 4) | ((uint32_t)(n_pad >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  p.nacc = std::min(4, 512 / n_pad) & ~1;   // even: the two epilogue groups alternate
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.nacc * n_pad)) cols *= 2;
  p.tmem_cols = cols;
  p.total_tiles = (int)((n_in + BM - 1) / BM);
  auto r1024 = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  p.a_chunk_bytes = r1024((uint32_t)(BM * p.kc * 2));
  p.b_tx = (uint32_t)(n_pad * p.kc * 2);
  p.b_chunk_bytes = r1024(p.b_tx);
  p.child = child;
  p.scale = scale;
  p.shift = shift;
  p.bias = bias;
  p.out = (__half*)out;
  static const int dbg = [] { const char* v = getenv("SCB_UP_DEBUG"); return v ? atoi(v) : 0; }();
  p.debug = dbg;

  const int smem_cap = 227 * 1024;
  const int fixed = 1024 + (3 * MAX_A + 8 + 2 * MAX_STAGES) * 8 + 16 + 3 * 256 * 4;
  const int a_slot = (int)(p.a_chunk_bytes * p.n_kchunks) + volume * BM * 4;
  const int b_all = volume * p.n_kchunks * (int)p.b_chunk_bytes;
  // weights resident when they fit beside >= 3 A slots (the A ring hides the
  // DRAM latency of the feature tiles); else streamed from L2 through a ring
  int as_res = std::min(MAX_A, (smem_cap - fixed - b_all) / a_slot);
  if (as_res >= 2) {
    p.b_resident = 1;
    p.b_stages = 0;
    p.a_stages = as_res;
  } else {
    p.b_resident = 0;
    // a stage holds b_kg K chunks: the whole slice when two stages fit
    // beside two A slots, else the largest divisor of n_kchunks that does
    p.b_kg = p.n_kchunks;
    while (p.b_kg > 1 && (fixed + 2 * a_slot + 2 * p.b_kg * (int)p.b_chunk_bytes > smem_cap ||
                          p.n_kchunks % p.b_kg != 0))
      --p.b_kg;
    const int b_stage = p.b_kg * (int)p.b_chunk_bytes;
    p.a_stages = std::min(MAX_A, (smem_cap - fixed - 2 * b_stage) / a_slot);
    SCB_CHECK_ARG(p.a_stages >= 1, "feature tile does not fit in shared memory");
    p.b_stages = std::min(MAX_STAGES, (smem_cap - fixed - p.a_stages * a_slot) / b_stage);
    SCB_CHECK_ARG(p.b_stages >= 2, "weight ring does not fit in shared memory");
  }
  const int smem = fixed + p.a_stages * a_slot +
                   (p.b_resident ? b_all : p.b_stages * p.b_kg * (int)p.b_chunk_bytes);

  CUtensorMap mA, mA2, mB;
  std::string err;
  const int ca = features2 ? c_split : c_in;
  if (!cached_map_f16(&mA, features, ca, n_in, ldf, p.kc, BM, (int)p.swz, err) ||
      !cached_map_f16(&mA2, features2 ? features2 : features, features2 ? c_in - c_split : ca,
                      n_in, features2 ? ldf2 : ldf, p.kc, BM, (int)p.swz, err) ||
      !cached_map_f16(&mB, weights_packed, k_pad, (long long)volume * n_pad, k_pad, p.kc, n_pad,
                      (int)p.swz, err)) {
    set_error(std::string(name) + ": " + err);
    return SCB_ECUDA;
  }
  const int epi = (scale ? EPI_AFFINE : 0) | (bias ? EPI_BIAS : 0) | (relu ? EPI_RELU : 0);
  const int grid = std::min(p.total_tiles, device_sms());
  static std::once_flag attr_once[8];
  static cudaError_t attr_err[8];
  auto launch = [&](auto kernel) {
    std::call_once(attr_once[epi], [&] {
      attr_err[epi] = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_cap);
    });
    if (attr_err[epi] != cudaSuccess) return attr_err[epi];
    kernel<<<grid, THREADS, smem, as_stream(stream)>>>(mA, mA2, mB, p);
    return cudaSuccess;
  };
  cudaError_t e;
  switch (epi) {
    case 0: e = launch(upconv_scatter_kernel<0>); break;
    case 1: e = launch(upconv_scatter_kernel<1>); break;
    case 2: e = launch(upconv_scatter_kernel<2>); break;
    case 3: e = launch(upconv_scatter_kernel<3>); break;
    case 4: e = launch(upconv_scatter_kernel<4>); break;
    case 5: e = launch(upconv_scatter_kernel<5>); break;
    case 6: e = launch(upconv_scatter_kernel<6>); break;
    default: e = launch(upconv_scatter_kernel<7>); break;
  }
  SCB_CUDA(e);
  SCB_LAUNCHED();
  return SCB_OK;
}

}  // namespace

extern "C" int32_t scb_conv_transposed_scatter(const void* features, int64_t ldf, int64_t n_in,
                                               int32_t c_in, const int32_t* child, int32_t volume,
                                               const void* weights_packed, int32_t c_out,
                                               void* out, int64_t ldo, int64_t n_out,
                                               const float* scale, const float* shift,
                                               const float* bias, int32_t relu,
                                               scb_stream_t stream) {
  SCB_CHECK_ARG(child != nullptr, "child is required");
  if (n_out <= 0) return SCB_OK;
  return launch_dense("scb_conv_transposed_scatter", features, ldf, c_in, nullptr, 0, n_in, c_in,
                      child, volume, weights_packed, c_out, out, ldo, scale, shift, bias, relu,
                      stream);
}

extern "C" int32_t scb_conv_pointwise(const void* features, int64_t ldf, int32_t c_split,
                                      const void* features2, int64_t ldf2, int64_t n,
                                      int32_t c_in, const void* weights_packed, int32_t c_out,
                                      void* out, int64_t ldo, const float* scale,
                                      const float* shift, const float* bias, int32_t relu,
                                      scb_stream_t stream) {
  SCB_CHECK_ARG(!features2 || (c_split > 0 && c_split < c_in && c_split % 8 == 0 &&
                               ldf2 >= c_in - c_split && ldf2 % 8 == 0),
                "concat: 0 < c_split < c_in, multiples of 8");
  return launch_dense("scb_conv_pointwise", features, ldf, c_split, features2, ldf2, n, c_in,
                      nullptr, 1, weights_packed, c_out, out, ldo, scale, shift, bias, relu,
                      stream);
}
