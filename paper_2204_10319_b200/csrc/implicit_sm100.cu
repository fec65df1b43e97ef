// Fused gather -> tcgen05 GEMM -> epilogue convolution (the "implicit GEMM"
// dataflow): one persistent kernel per layer computes
//
//   out[k] = epilogue( sum_n  features[hits[n][k]] . W[n] )      (absent -> 0)
//
// for 128-row output tiles, accumulating all V offsets in TMEM (double-
// buffered accumulators, so the epilogue of tile i overlaps tile i+1).  The
// gather is fused into the operand load: cp.async moves each present
// neighbour's 16-B row chunks straight into the 128/64/32-B swizzled UMMA
// layout (absent neighbours are zero), so neither the gather buffer nor the
// f32 partials ever reach HBM.  Each output row is written once (fp16) with
// BN / bias / residual / ReLU applied in registers.  V = 1 is the K=1 layer
// (identity map, no hit matrix).
//
// Pipeline (per stage: `ops` offsets x one K chunk of A and B):
//   * producers never block on their own copies: each thread's completion is
//     tracked by cp.async.mbarrier.arrive.noinc, absent rows are zero-filled
//     by zero-size cp.async, so every write of a stage is async-tracked;
//   * copies are lane-per-chunk (the CPR lanes of a row copy its consecutive
//     16-B chunks), P threads per row split the chunks;
//   * the MMA warp runs converged (stage indices and descriptors in uniform
//     registers) and one elected lane issues; descriptors advance by
//     constant steps.
// (Measured on the MinkUNet level-0 96->96 layer: 1.27 ms for the first
// row-per-thread / wait_group version, 0.73 ms with the above.)
//
// Warp roles (64 + 128 P + 128 threads, persistent over contiguous tile
// ranges, 1 or 2 CTAs per SM):
//   warp 0        TMA producer of the weight slices (B, K-major fp16)
//   warp 1        TMEM allocator + MMA issuer
//   warps 2..     A producers (P per output row)
//   last 4 warps  epilogue: tcgen05.ld -> epilogue -> swizzled smem -> TMA store
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace scb {
namespace ic {

using namespace ::scb::ptx;

constexpr int BM = 128;
constexpr int EPI_BUF = 32 * 64;        // 32 rows x 64 B (32 fp16 columns)
constexpr int MAX_OPS = 8;              // kernel offsets per pipeline stage

struct Params {
  long long n_out;
  int n_in, c_in, c_out, V, n_pad, kc, n_kchunks, stages, swz, epi_cols, total_tiles, relu;
  int ops;                  // offsets per stage (small C_in -> several)
  int epi_bufs;             // epilogue staging buffers per warp (1 or 2)
  int nacc;                 // TMEM accumulator buffers (2: epilogue overlaps the next tile)
  int rowmode;              // 1: one producer thread per row (needs P = 1)
  int debug;                // SCB_IMPLICIT_DEBUG: 1 no A loads, 16 wait counters, 32 no B loads
  int groups;               // ceil(V / ops) offset groups per tile
  int bsleep, esleep;       // poll back-off (ns) of the weight producer / the epilogue
  int vk;                   // virtual-K: K = the V x C_in concatenation in 64-wide chunks
  int nsplit, n_unit;       // work unit = (row tile, one of nsplit n_unit-column slices)
  int nblk;                 // A/B blocks per tile: V (per-offset K chunks) or ceil(V C_in / 64)
  uint32_t idesc, tmem_cols;
  uint32_t a_off_bytes;     // one offset's A block [128 rows][kc] (1024-aligned)
  uint32_t b_off_bytes;     // one offset's B block [n_pad][kc]   (1024-aligned)
  uint32_t a_stage_bytes, stage_bytes;
  uint32_t b_tx;            // bytes one offset's B load delivers
  long long ldf, ldh;       // feature row stride, hit-matrix row stride
  const __half* feat;       // [n_in][ldf]: input channels [0, c_split)
  const __half* feat2;      // nullable: channels [c_split, c_in) (skip concat), [n_in][ldf2]
  long long ldf2;
  int c_split;
  const int* hits;          // [V][ldh] input row or -1 (unused for V = 1)
  const float* scale;       // nullable (with shift)
  const float* shift;
  const float* bias;        // nullable
  const __half* residual;   // nullable, [n_out][c_out]
};

__device__ __forceinline__ uint32_t swz_off(int row, int chunk, int swz) {
  if (swz == 128) return row * 128 + ((chunk ^ (row & 7)) << 4);
  if (swz == 64) return row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
  return row * 32 + ((chunk ^ ((row >> 2) & 1)) << 4);
}

// SCB_IMPLICIT_DEBUG bit 16: per-role cycle counters of CTA 0.
__device__ unsigned long long g_ic_prof[16];
#define IC_PROF(idx, cond, ...)                                                       \
  do {                                                                                \
    if ((p.debug & 16) && blockIdx.x == 0 && (cond)) {                                \
      const long long t0_ = clock64();                                                \
      __VA_ARGS__;                                                                    \
      atomicAdd(&g_ic_prof[idx], (unsigned long long)(clock64() - t0_));              \
    } else {                                                                          \
      __VA_ARGS__;                                                                    \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ============ epilogue role (4 warps; warp w reads TMEM lanes 32 (w % 4)..):
// accumulator acc of tile t -> scale/shift, bias, residual, ReLU -> fp16 ->
// swizzled staging buffer -> TMA store of 32 rows x epi_cols.
__device__ __forceinline__ void epilogue_role(const Params& p, const CUtensorMap* tmOut_,
                                              uint32_t tmem_base, uint64_t* tfull,
                                              uint64_t* tempty, uint8_t* epi_base, int warp,
                                              int epi0, int lane, int t_begin, int t_end) {
  // ============ epilogue
  const int q = warp & 3;
  uint8_t* bufs = epi_base + (warp - epi0) * p.epi_bufs * EPI_BUF;
  int acc = 0, nbuf = 0;
  uint32_t acc_phase = 0;
  const int chunks = p.n_unit / p.epi_cols;
  for (int t = t_begin; t < t_end; ++t) {
    IC_PROF(5, warp == epi0 && lane == 0, mbar_wait_sleep(tfull + acc, acc_phase, p.esleep));
    tc_after();
    const int rt = p.nsplit == 2 ? (t >> 1) : t;
    const int cb = p.nsplit == 2 ? (t & 1) * p.n_unit : 0;   // first output column of the unit
    const long long row0 = (long long)rt * BM + 32 * q;
    const long long k = row0 + lane;
    const bool row_ok = k < p.n_out;
    for (int j = 0; j < chunks && row0 < p.n_out; ++j) {
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * p.n_unit + j * p.epi_cols);
      const int c0 = cb + j * p.epi_cols;   // output column
      uint32_t r[32];
      TMEM_LD_X16(taddr, r);
      if (p.epi_cols == 32) TMEM_LD_X16(taddr + 16, (r + 16));
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      const int ncol = p.epi_cols;
      if (p.scale) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < ncol && c0 + i < p.c_out)
            v[i] = v[i] * __ldg(p.scale + c0 + i) + __ldg(p.shift + c0 + i);
      }
      if (p.bias) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < ncol && c0 + i < p.c_out) v[i] += __ldg(p.bias + c0 + i);
      }
      if (p.residual && row_ok) {
        const uint4* rp = reinterpret_cast<const uint4*>(p.residual + k * p.c_out + c0);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g * 8 < ncol && c0 + g * 8 < p.c_out) {
            const uint4 w = __ldg(rp + g);
            const __half2* hh = reinterpret_cast<const __half2*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(hh[e]);
              v[g * 8 + 2 * e] += f.x;
              v[g * 8 + 2 * e + 1] += f.y;
            }
          }
        }
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      uint8_t* buf = bufs + nbuf * EPI_BUF;
      if (lane == 0) {
        if (p.epi_bufs == 2) IC_PROF(6, warp == epi0, bulk_wait_read1());
        else bulk_wait_read0();
      }
      __syncwarp();
      if (ncol == 32) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 w = make_uint4(pack_half2(v[8 * c], v[8 * c + 1]), pack_half2(v[8 * c + 2], v[8 * c + 3]),
                               pack_half2(v[8 * c + 4], v[8 * c + 5]), pack_half2(v[8 * c + 6], v[8 * c + 7]));
          *reinterpret_cast<uint4*>(buf + swz_off(lane, c, 64)) = w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint4 w = make_uint4(pack_half2(v[8 * c], v[8 * c + 1]), pack_half2(v[8 * c + 2], v[8 * c + 3]),
                               pack_half2(v[8 * c + 4], v[8 * c + 5]), pack_half2(v[8 * c + 6], v[8 * c + 7]));
          *reinterpret_cast<uint4*>(buf + swz_off(lane, c, 32)) = w;
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmOut_, buf, c0, (int)row0);
        bulk_commit();
      }
      nbuf ^= p.epi_bufs - 1;
    }
    tc_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty + acc);
    if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
  }
  if (lane == 0) bulk_wait_all();
}

template <int V, int KC, int P, int MINB>
__global__ void __launch_bounds__(64 + 128 * P + 128, MINB)
    implicit_conv_f16_kernel(const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmOut,
                             const __grid_constant__ Params p) {
  constexpr int NPROD = 128 * P;           // A-producer threads
  constexpr int EPI0 = 2 + 4 * P;          // first epilogue warp
  constexpr int CPR = KC / 8;              // 16-B chunks per row per K chunk
  constexpr int IT = CPR / P;              // chunks a producer thread copies per offset
  constexpr int SWZ = KC * 2;              // swizzle span = row bytes
  constexpr int MAXO = (32 / IT) < MAX_OPS ? (32 / IT) : MAX_OPS;
  constexpr int NT = (V + P - 1) / P;      // offsets whose index a thread prefetches
  static_assert(IT >= 1 && IT * P == CPR, "P must divide the chunks per row");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_base = smem + (size_t)p.stages * p.stage_bytes;
  int* nbr_s = (int*)(epi_base + 4 * p.epi_bufs * EPI_BUF);      // [V][BM] neighbour rows of the tile
  uint64_t* full = (uint64_t*)(nbr_s + V * BM);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const long long k_t0 = clock64();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_begin = (int)((long long)p.total_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long long)p.total_tiles * (blockIdx.x + 1) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, NPROD + 1);  // one async (noinc) arrive per producer + the B expect_tx
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmOut) : "memory");
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
  // Programmatic dependent launch: the prologue above (barriers, TMEM,
  // tensor-map prefetch) overlapped the previous kernel's tail; wait for it
  // (all its writes visible) before reading any input, and let the next
  // layer's kernel start its own prologue as soon as SMs free up.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ============ B producer: the stage's weight slices via TMA
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; ++t)
        for (int g = 0; g < p.groups; ++g) {
          const int nv = min(p.ops, p.nblk - g * p.ops);
          for (int kk = 0; kk < p.n_kchunks; ++kk) {
            IC_PROF(2, true, mbar_wait_sleep(empty + stage, phase ^ 1, p.bsleep));
            if (p.debug & 32) {
              mbar_arrive(full + stage);
            } else {
              mbar_expect_tx(full + stage, nv * p.b_tx);
              uint8_t* sb = smem + (size_t)stage * p.stage_bytes + p.a_stage_bytes;
              for (int o = 0; o < nv; ++o) {
                if (p.vk)   // [n_pad][V C_in] K-major: block = 64 consecutive virtual channels
                  tma_load_2d(sb + o * p.b_off_bytes, &tmB, full + stage, (g * p.ops + o) * 64, 0);
                else
                  tma_load_2d(sb + o * p.b_off_bytes, &tmB, full + stage, kk * p.kc,
                              (g * p.ops + o) * p.n_pad + (p.nsplit == 2 ? (t & 1) * p.n_unit : 0));
              }
            }
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
          }
        }
    }
  } else if (warp >= 2 && warp < EPI0) {
    // ============ A producers.  Thread (h, row) prefetches the neighbour
    // rows of output row `row` for the offsets n = h (mod P) one tile ahead
    // and parks them in the tile's index table.  Copies are lane-per-chunk:
    // item `it` of thread pt is chunk (pt % CPR) of row it * (NPROD / CPR) +
    // pt / CPR, so consecutive lanes copy consecutive 16-B chunks of a row.
    const int pt = threadIdx.x - 64;
    const int row = pt & (BM - 1);
    const int h = pt >> 7;
    int nxt[NT];
    {
      const long long k = (long long)(p.nsplit == 2 ? (t_begin >> 1) : t_begin) * BM + row;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int n = h + i * P;
        nxt[i] = (n < V && t_begin < t_end && k < p.n_out)
                     ? (V == 1 ? (int)k : __ldg(p.hits + (long long)n * p.ldh + k)) : -1;
      }
    }
    // (no stage zeroing: every 16-B item of a stage is rewritten each use)
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t nb_s0 = smem_u32(nbr_s);
    const int cr = pt / CPR, cc = pt % CPR;   // row group / chunk of this lane
    uint32_t roff[IT];                        // smem offset of item it inside a block
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int r = it * (NPROD / CPR) + cr;
      const int rxr = SWZ == 128 ? (r & 7) : (SWZ == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
      roff[it] = (uint32_t)(r * (KC * 2)) + ((uint32_t)(cc ^ rxr) << 4);
    }
    uint32_t sw[CPR];                         // row mode: swizzled offset of chunk c in the row
#pragma unroll
    for (int c = 0; c < CPR; ++c) {
      const int rx = SWZ == 128 ? (row & 7) : (SWZ == 64 ? ((row >> 1) & 3) : ((row >> 2) & 1));
      sw[c] = (uint32_t)((c ^ rx) << 4);
    }
    const uint32_t ldfb1 = (uint32_t)(p.ldf * 2);   // row strides in bytes (host-checked < 2^32)
    const uint32_t ldfb2 = (uint32_t)(p.ldf2 * 2);
    for (int t = t_begin; t < t_end; ++t) {
      // the table is read by other threads: rewrite it only after every
      // producer finished the previous tile (the first barrier also orders
      // the zeroed stage buffers before any copy)
      asm volatile("bar.sync 1, %0;" ::"n"(NPROD) : "memory");
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int n = h + i * P;
        if (n < V)
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(nb_s0 + (uint32_t)((n * BM + row) * 4)), "r"(nxt[i]) : "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NPROD) : "memory");
      {
        const long long k = (long long)(p.nsplit == 2 ? ((t + 1) >> 1) : (t + 1)) * BM + row;
        const bool ok = (t + 1 < t_end) && k < p.n_out;
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          const int n = h + i * P;
          nxt[i] = (ok && n < V) ? (V == 1 ? (int)k : __ldg(p.hits + (long long)n * p.ldh + k)) : -1;
        }
      }
      for (int g = 0; g < p.groups; ++g) {
        const int nv = min(p.ops, p.nblk - g * p.ops);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          IC_PROF(0, pt == 0, mbar_wait(empty + stage, phase ^ 1));
          const long long a_t0 = clock64();
          const uint32_t dst = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const int col0 = kk * KC;
          const int live = p.vk ? CPR : min(CPR, (p.c_in - col0) / 8);  // chunks inside C_in
          // Every 16-B item of the stage is written each time: a copy of a
          // present neighbour's chunk or a zero-fill (absent neighbour, or a
          // chunk past C_in).  (Tracking which slots already hold zeros halves
          // the copies but costs more instructions: measured slower.)
          const uint32_t nbc = nb_s0 + (uint32_t)((g * p.ops * BM + cr) * 4);
          // this lane's 8 columns come from the first or (concat) second input
          const int col = col0 + cc * 8;
          const bool second = p.feat2 != nullptr && col >= p.c_split;
          const uint64_t fbase = second
              ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((col - p.c_split) * 2)
              : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(col * 2);
          const uint32_t ldfb = second ? ldfb2 : ldfb1;
          const bool live_c = cc < live && !(p.debug & 1);
          const bool all_live = live == CPR && !(p.debug & 1);  // warp-uniform
          if (p.rowmode) {
            // row per thread: one index load, one address and CPR cp.async
            // (immediate chunk offsets) per (row, offset) -- ~2 instructions
            // per 16-B item; chunks past C_in are skipped (they stay zero)
            const bool mixed = p.feat2 != nullptr && col0 < p.c_split && col0 + KC > p.c_split;
            const bool sec0 = p.feat2 != nullptr && col0 >= p.c_split;
            const uint64_t fb0 = sec0
                ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((col0 - p.c_split) * 2)
                : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(col0 * 2);
            const uint32_t ld0 = sec0 ? ldfb2 : ldfb1;
            const int nlive = (p.debug & 1) ? 0 : live;
            for (int o = 0; o < nv; ++o) {
              int j;
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(j) : "r"(nb_s0 + (uint32_t)(((g * p.ops + o) * BM + row) * 4)));
              const uint32_t base = dst + o * p.a_off_bytes + row * (KC * 2);
              const uint32_t jj = (uint32_t)max(j, 0);
              if (!mixed) {
                const uint64_t src = fb0 + (uint64_t)jj * (uint64_t)ld0;
#pragma unroll
                for (int c = 0; c < CPR; ++c)  // chunks past C_in: zero-filled (slots are reused)
                  asm volatile(
                      "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                      "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(base + sw[c]),
                      "l"(src + (uint64_t)(c * 16)), "r"(c < nlive ? j : -1) : "memory");
              } else {
                const uint64_t s1 = reinterpret_cast<uint64_t>(p.feat) + (uint64_t)jj * ldfb1;
                const uint64_t s2 = reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)jj * ldfb2;
#pragma unroll
                for (int c = 0; c < CPR; ++c) {
                  const int col = col0 + c * 8;
                  const uint64_t src = col < p.c_split ? s1 + (uint64_t)(col * 2)
                                                       : s2 + (uint64_t)((col - p.c_split) * 2);
                  asm volatile(
                      "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                      "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(base + sw[c]),
                      "l"(src), "r"(c < nlive ? j : -1) : "memory");
                }
              }
            }
          } else {
            // lean form: every item is one cp.async whose source size is 16
            // (present) or 0 (zero-fill) -- no presence bookkeeping; the
            // producer is issue-bound, and this is ~3x fewer instructions
            for (int o = 0; o < nv; ++o) {
              int jj[IT];
              uint64_t fb = fbase;
              uint32_t ldb = ldfb;
              if (p.vk) {
                // virtual K: this lane's 8 channels are channel ch of offset n
                const int vc = (g * p.ops + o) * 64 + cc * 8;
                const int n = vc / p.c_in, ch = vc - n * p.c_in;
                const bool sec = p.feat2 != nullptr && ch >= p.c_split;
                fb = sec ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((ch - p.c_split) * 2)
                         : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(ch * 2);
                ldb = sec ? ldfb2 : ldfb1;
                const uint32_t nbn = nb_s0 + (uint32_t)((n * BM + cr) * 4);
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                  jj[it] = -1;
                  if (n < V)
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(jj[it]) : "r"(nbn + (uint32_t)(it * (NPROD / CPR) * 4)));
                }
              } else {
#pragma unroll
                for (int it = 0; it < IT; ++it)
                  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(jj[it]) : "r"(nbc + (uint32_t)((o * BM + it * (NPROD / CPR)) * 4)));
              }
              const uint32_t blk = dst + o * p.a_off_bytes;
              if (all_live) {  // the common case: no per-item liveness select
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                  const int j = jj[it];
                  const uint64_t src = fb + (uint64_t)(uint32_t)max(j, 0) * (uint64_t)ldb;
                  // ignore-src predicate (absent neighbour): zero-fill, no read
                  asm volatile(
                      "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                      "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(blk + roff[it]),
                      "l"(src), "r"(j) : "memory");
                }
              } else {
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                  const int j = live_c ? jj[it] : -1;
                  const uint64_t src = fb + (uint64_t)(uint32_t)max(j, 0) * (uint64_t)ldb;
                  asm volatile(
                      "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                      "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(blk + roff[it]),
                      "l"(src), "r"(j) : "memory");
                }
              }
            }
          }
          if ((p.debug & 16) && blockIdx.x == 0 && pt == 0) atomicAdd(&g_ic_prof[11], (unsigned long long)(clock64() - a_t0));
          if (p.debug & 128) {  // debug: wait for the copies, then a plain arrive
            cp_async_wait<0>();
            fence_async_smem();
            mbar_arrive(full + stage);
          } else {
            cp_async_arrive_noinc(full + stage);   // fires when this thread's copies land
          }
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer.  The whole warp runs the loop (so stage
    // indices and descriptors stay warp-uniform, in uniform registers) and
    // one elected lane issues.  Every offset block of a stage is multiplied
    // (a tile rarely lacks an offset entirely, and a per-block test cost more
    // issue time than the MMAs it saved).
    const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
    const uint32_t sbo = 8u * (uint32_t)p.swz;
    const uint64_t adesc_base = make_sdesc(smem_u32(smem), sbo, layout);
    const uint32_t stage_d = p.stage_bytes >> 4, a_stage_d = p.a_stage_bytes >> 4;
    const uint32_t a_off_d = p.a_off_bytes >> 4, b_off_d = p.b_off_bytes >> 4;
    const uint32_t idesc = p.idesc, n_pad = p.n_pad;
    const uint32_t tmem0 = __shfl_sync(0xffffffffu, tmem_base, 0);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int t = t_begin; t < t_end; ++t) {
      IC_PROF(4, lane == 0, mbar_wait(tempty + acc, acc_phase ^ 1));
      tc_after();
      const uint32_t d = tmem0 + (uint32_t)acc * (uint32_t)p.n_unit;
      for (int g = 0; g < p.groups; ++g) {
        const int nv = min(p.ops, p.nblk - g * p.ops);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          IC_PROF(3, lane == 0, mbar_wait(full + stage, phase));
          const long long m_t0 = clock64();
          const uint64_t ad = adesc_base + (uint64_t)(stage * stage_d);
          const uint64_t bd = ad + a_stage_d;
          const uint32_t acc0 = (g | kk) ? 1u : 0u;
          if (elect_one()) {
            if (!(p.debug & 64)) fence_async_smem();  // cp.async (generic proxy) data -> tcgen05 reads
            tc_after();
#pragma unroll
            for (int o = 0; o < MAX_OPS; ++o) {
              if (o < nv) {
                const uint64_t a = ad + (uint64_t)(o * a_off_d);
                const uint64_t b = bd + (uint64_t)(o * b_off_d);
                if ((p.debug & 2) && (g | o)) continue;  // debug: MMAs off (first block only)
                mma_f16(d, a, b, idesc, o ? 1u : acc0);
#pragma unroll
                for (int k = 1; k < KC / 16; ++k) mma_f16(d, a + 2u * k, b + 2u * k, idesc, 1u);
              }
            }
            mma_commit(empty + stage);
            if ((p.debug & 16) && blockIdx.x == 0) atomicAdd(&g_ic_prof[10], (unsigned long long)(clock64() - m_t0));
          }
          __syncwarp();
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
      if (elect_one()) mma_commit(tfull + acc);
      __syncwarp();
      if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= EPI0) {
    epilogue_role(p, &tmOut, tmem_base, tfull, tempty, epi_base, warp, EPI0, lane, t_begin, t_end);
  }

  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
  if ((p.debug & 16) && blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&g_ic_prof[7], (unsigned long long)(clock64() - k_t0));
    atomicAdd(&g_ic_prof[9], (unsigned long long)(t_end - t_begin));
  }
}

// ------------------------------------------------------------------ TS form
// The same convolution with the gathered A operand in TENSOR memory
// (tcgen05.mma A-from-TMEM): producer threads own one output row each
// (row = TMEM lane), load its present neighbours' channels straight into
// registers and tcgen05.st them into a TMEM ring; only the weights (B) pass
// through shared memory.  The SS form's per-MMA shared-memory reads of A
// (4 KB per K = 16 step, plus the cp.async writes) were the bound at
// C_out <= 128; here shared memory carries B alone.
//
// TMEM: [0, nacc n_pad) accumulators, then `stages` A blocks of 32 columns
// (one stage = 64 / KC offsets x one K chunk = 128 rows x 64 fp16).
// Warps: 0 B TMA, 1 TMEM alloc + MMA issue, 2 .. 2 + 4 PW A producers (PW
// warps per TMEM lane quarter take stages round-robin), then 4 epilogue warps.
// absent neighbours of the TS form read this (L1-resident) zero row
__device__ __align__(128) uint4 g_zero_row[32];

template <int V, int KC, int PW>
__global__ void __launch_bounds__(64 + 128 * PW + 128, 1)
    implicit_conv_ts_kernel(const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ CUtensorMap tmOut,
                            const __grid_constant__ Params p) {
  constexpr int OPS = 64 / KC;             // offsets per stage
  constexpr int CPR = KC / 8;              // 16-B chunks per row per K chunk
  constexpr int EPI0 = 2 + 4 * PW;
  constexpr int NT = (V + PW - 1) / PW;    // offsets whose index a thread prefetches
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_base = smem + (size_t)p.stages * p.stage_bytes;
  int* nbr_s = (int*)(epi_base + 4 * p.epi_bufs * EPI_BUF);      // [V][BM]
  uint64_t* full = (uint64_t*)(nbr_s + V * BM);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const long long k_t0 = clock64();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_begin = (int)((long long)p.total_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long long)p.total_tiles * (blockIdx.x + 1) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 4 + 1);   // one arrive per lane-quarter warp + the B expect_tx
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmOut) : "memory");
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t a_col0 = (uint32_t)(p.nacc * p.n_pad);

  if (warp == 0) {
    // ============ B producer (TMA): the stage's weight slices
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; ++t)
        for (int g = 0; g < p.groups; ++g) {
          const int nv = min(OPS, V - g * OPS);
          for (int kk = 0; kk < p.n_kchunks; ++kk) {
            IC_PROF(2, true, mbar_wait_sleep(empty + stage, phase ^ 1, p.bsleep));
            if (p.debug & 4) {   // debug: no weight loads
              mbar_arrive(full + stage);
            } else {
              mbar_expect_tx(full + stage, nv * p.b_tx);
              uint8_t* sb = smem + (size_t)stage * p.stage_bytes;
              for (int o = 0; o < nv; ++o)
                tma_load_2d(sb + o * p.b_off_bytes, &tmB, full + stage, kk * KC,
                            (g * OPS + o) * p.n_pad);
            }
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
          }
        }
    }
  } else if (warp >= 2 && warp < EPI0) {
    // ============ A producers: thread = output row (TMEM lane 32 q + lane).
    // Warp (q, sub) fills stages i = sub (mod PW) of the CTA's stage
    // sequence; two stages' rows are in flight per thread (register double
    // buffer) and each stage's neighbour indices are fetched a stage-pair
    // earlier.  The producer is issue-bound, so the per-stage bookkeeping is
    // incremental (no divisions) and each 16-B chunk is one load with an
    // immediate offset; absent neighbours read a zero row.
    const int q = warp & 3, sub = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    const int nk = p.n_kchunks, ntiles = t_end - t_begin;
    const uint32_t t_row = tmem_base + ((uint32_t)(32 * q) << 16) + a_col0;
    // position of the next stage whose indices are fetched (sequence order)
    int it_t = 0, it_g = 0, it_k = sub;
    while (it_k >= nk) { it_k -= nk; if (++it_g == p.groups) { it_g = 0; ++it_t; } }
    // chunks of the K chunk: all from one input unless a concat split is inside
    const uint64_t zrow = reinterpret_cast<uint64_t>(g_zero_row);
    auto load_idx = [&](int (&j)[OPS], int& kk_out) {
      const long long k = (long long)(t_begin + it_t) * BM + row;
      const bool ok = it_t < ntiles && k < p.n_out;
#pragma unroll
      for (int o = 0; o < OPS; ++o) {
        const int n = it_g * OPS + o;
        j[o] = (ok && n < V) ? ((V == 1 || (p.debug & 32)) ? (int)k : __ldg(p.hits + (long long)n * p.ldh + k)) : -1;
      }
      kk_out = it_k;
      it_k += PW;
      while (it_k >= nk) { it_k -= nk; if (++it_g == p.groups) { it_g = 0; ++it_t; } }
    };
    auto load_rows = [&](const int (&j)[OPS], int kk, uint4 (&v)[OPS][CPR]) {
      const int col0 = kk * KC;
      const int live = (p.debug & 1) ? 0 : min(CPR, (p.c_in - col0) / 8);
      const bool split = p.feat2 != nullptr && col0 < p.c_split && col0 + KC > p.c_split;
      if (live == CPR && !split) {   // warp-uniform fast path
        const bool second = p.feat2 != nullptr && col0 >= p.c_split;
        const uint64_t base = second
            ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((col0 - p.c_split) * 2)
            : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(col0 * 2);
        const uint64_t ldb = (uint64_t)(second ? p.ldf2 : p.ldf) * 2u;
#pragma unroll
        for (int o = 0; o < OPS; ++o) {
          const uint64_t r = j[o] >= 0 ? base + (uint64_t)(uint32_t)j[o] * ldb : zrow;
          const uint4* rp = reinterpret_cast<const uint4*>(r);
#pragma unroll
          for (int c = 0; c < CPR; ++c) v[o][c] = __ldg(rp + c);
        }
      } else {
#pragma unroll
        for (int o = 0; o < OPS; ++o)
#pragma unroll
          for (int c = 0; c < CPR; ++c) {
            const int col = col0 + c * 8;
            const bool sec = p.feat2 != nullptr && col >= p.c_split;
            const uint64_t r = (j[o] >= 0 && c < live)
                ? (sec ? reinterpret_cast<uint64_t>(p.feat2) + ((uint64_t)(uint32_t)j[o] * p.ldf2 + (col - p.c_split)) * 2u
                       : reinterpret_cast<uint64_t>(p.feat) + ((uint64_t)(uint32_t)j[o] * p.ldf + col) * 2u)
                : zrow;
            v[o][c] = __ldg(reinterpret_cast<const uint4*>(r));
          }
      }
    };
    int st_stage = sub;
    uint32_t st_phase = 0;
    auto store = [&](uint4 (&v)[OPS][CPR]) {
      IC_PROF(0, row == 0, mbar_wait(empty + st_stage, st_phase ^ 1));   // the MMAs that read this slot are done
      tc_after();
      const uint32_t ta = t_row + (uint32_t)(st_stage * 32);
      if (!(p.debug & 8)) {   // debug 8: no TMEM stores
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[0][0]);
#pragma unroll
        for (int h = 0; h < 2; ++h) TMEM_ST_X16(ta + 16 * h, (w + 16 * h));
        tmem_wait_st();
      }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(full + st_stage);
      st_stage += PW;
      if (st_stage >= p.stages) { st_stage -= p.stages; st_phase ^= 1; }
    };
    const int total = ntiles * p.groups * nk;
    int ja[OPS], jb[OPS], ka, kb;
    uint4 va[OPS][CPR], vb[OPS][CPR];
    load_idx(ja, ka);
    load_idx(jb, kb);
    load_rows(ja, ka, va);
    load_rows(jb, kb, vb);
    load_idx(ja, ka);
    load_idx(jb, kb);
    for (int i = sub; i < total; i += 2 * PW) {
      store(va);
      load_rows(ja, ka, va);
      load_idx(ja, ka);
      if (i + PW < total) {
        store(vb);
        load_rows(jb, kb, vb);
        load_idx(jb, kb);
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer (A from TMEM, B from shared memory)
    const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
    const uint32_t sbo = 8u * (uint32_t)p.swz;
    const uint64_t bdesc_base = make_sdesc(smem_u32(smem), sbo, layout);
    const uint32_t stage_d = p.stage_bytes >> 4, b_off_d = p.b_off_bytes >> 4;
    const uint32_t idesc = p.idesc, n_pad = p.n_pad;
    const uint32_t tmem0 = __shfl_sync(0xffffffffu, tmem_base, 0);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int t = t_begin; t < t_end; ++t) {
      IC_PROF(4, lane == 0, mbar_wait(tempty + acc, acc_phase ^ 1));
      tc_after();
      const uint32_t d = tmem0 + (uint32_t)acc * n_pad;
      for (int g = 0; g < p.groups; ++g) {
        const int nv = min(OPS, V - g * OPS);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          IC_PROF(3, lane == 0, mbar_wait(full + stage, phase));
          tc_after();
          const uint64_t bd = bdesc_base + (uint64_t)(stage * stage_d);
          const uint32_t ta = tmem0 + a_col0 + (uint32_t)(stage * 32);
          const uint32_t acc0 = (g | kk) ? 1u : 0u;
          if (elect_one()) {
#pragma unroll
            for (int o = 0; o < OPS; ++o) {
              if (o < nv) {
                const uint64_t b = bd + (uint64_t)(o * b_off_d);
#pragma unroll
                for (int k = 0; k < KC / 16; ++k)
                  if (!(p.debug & 2) || (o | k | g | kk) == 0)   // debug 2: first MMA only
                    mma_f16_ts(d, ta + o * (KC / 2) + 8 * k, b + 2u * k, idesc, (o | k) ? 1u : acc0);
              }
            }
            if (p.debug & 64) mbar_arrive(empty + stage);   // debug (with 2): plain arrive
            else mma_commit(empty + stage);
          }
          __syncwarp();
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
      if (elect_one()) mma_commit(tfull + acc);
      __syncwarp();
      if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= EPI0) {
    epilogue_role(p, &tmOut, tmem_base, tfull, tempty, epi_base, warp, EPI0, lane, t_begin, t_end);
  }

  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
  if ((p.debug & 16) && blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&g_ic_prof[7], (unsigned long long)(clock64() - k_t0));
    atomicAdd(&g_ic_prof[9], (unsigned long long)(t_end - t_begin));
  }
}

}  // namespace ic

// ------------------------------------------------------------------ host
bool encode_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                   long long inner, long long rows, long long ld, int box_inner, int box_rows,
                   int swz_bytes, std::string& err);
int device_sms();

}  // namespace scb

using namespace scb;

extern "C" int32_t scb_conv_implicit_cat(const void* features, int64_t ldf, int32_t c_split,
                                         const void* features2, int64_t ldf2, int64_t n_in,
                                         int32_t c_in, const int32_t* hits, int32_t volume,
                                         int64_t n_out, const void* weights_packed,
                                         int32_t c_out, void* out, int64_t ldo,
                                         const float* scale, const float* shift,
                                         const float* bias, const void* residual, int32_t relu,
                                         scb_stream_t stream);

extern "C" int32_t scb_conv_implicit(const void* features, int64_t n_in, int32_t c_in,
                                     int64_t ldf, const int32_t* hits, int32_t volume,
                                     int64_t n_out, const void* weights_packed, int32_t c_out,
                                     void* out, const float* scale, const float* shift,
                                     const float* bias, const void* residual, int32_t relu,
                                     scb_stream_t stream) {
  return scb_conv_implicit_cat(features, ldf, c_in, nullptr, 0, n_in, c_in, hits, volume, n_out,
                               weights_packed, c_out, out, c_out, scale, shift, bias, residual,
                               relu, stream);
}

static int32_t conv_implicit_impl(const void* features, int64_t ldf, int32_t c_split,
                                         const void* features2, int64_t ldf2, int64_t n_in,
                                         int32_t c_in, const int32_t* hits, int32_t volume,
                                         int64_t n_out, const void* weights_packed,
                                         int32_t c_out, void* out, int64_t ldo,
                                         const float* scale, const float* shift,
                                         const float* bias, const void* residual, int32_t relu,
                                         scb_stream_t stream,
                                  int vk) {
  using namespace ic;
  SCB_CHECK_ARG(features2 == nullptr || (c_split % 8 == 0 && c_split > 0 && c_split < c_in &&
                                         ldf2 % 8 == 0 && ldf2 * 2 < (1LL << 32)),
                "concat split must be a positive multiple of 8 inside C_in, second stride % 8");
  SCB_CHECK_ARG(volume == 1 || volume == 8 || volume == 27,
                "implicit conv supports K^3 = 1, 8 or 27 offsets");
  SCB_CHECK_ARG(volume == 1 || hits != nullptr, "hit matrix required for K > 1");
  SCB_CHECK_ARG(volume != 1 || n_in == n_out, "K = 1: identity map needs n_in == n_out");
  SCB_CHECK_ARG(c_in % 8 == 0 && ldf % 8 == 0, "C_in and its row stride must be multiples of 8");
  SCB_CHECK_ARG(ldo % 8 == 0 && ldo >= c_out && ldo * 2 < (1LL << 32),
                "output row stride must be a multiple of 8 elements, >= C_out");
  SCB_CHECK_ARG(residual == nullptr || c_out % 8 == 0, "a residual needs C_out % 8 == 0");
  SCB_CHECK_ARG(ldf * 2 < (1LL << 32), "feature row stride too large");
  SCB_CHECK_ARG((scale == nullptr) == (shift == nullptr), "scale and shift go together");
  SCB_CHECK_ARG(n_in < (1LL << 31) - 1 && (long long)volume * hits_ld(n_out) < (1LL << 31),
                "too many rows for 32-bit TMA coordinates");
  const int n_pad = (c_out + 15) / 16 * 16;
  const int k_pad = (c_in + 15) / 16 * 16;
  SCB_CHECK_ARG(n_pad <= 256, "C_out > 256 not supported by the implicit conv");
  if (n_out == 0) return SCB_OK;
  Params p;
  memset(&p, 0, sizeof(p));
  p.n_out = n_out;
  p.n_in = (int)n_in;
  p.c_in = c_in;
  p.c_out = c_out;
  p.V = volume;
  p.n_pad = n_pad;
  p.kc = (k_pad % 64 == 0) ? 64 : ((k_pad % 32 == 0) ? 32 : 16);
  p.swz = p.kc * 2;
  p.n_kchunks = k_pad / p.kc;
  // virtual K (weights packed [n_pad][ceil64(V C_in)]): 64-wide chunks of the
  // offset-major channel concatenation, so every K = 16 MMA step reads a
  // 128-B-swizzled A block (measured ~84 cycles per M128 K16 step against
  // ~146 with 64-B rows, whatever N <= 128: tools/mma_probe.cu)
  const int kv = (int)(((long long)volume * c_in + 63) / 64 * 64);
  if (vk) {
    SCB_CHECK_ARG(volume > 1, "virtual K needs K > 1");
    p.kc = 64;
    p.swz = 128;
    p.n_kchunks = 1;
  }
  p.vk = vk ? 1 : 0;
  p.nblk = vk ? kv / 64 : volume;
  auto env_int = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
  };
  // Column split (opt-in, SCB_IC_NSPLIT=2, C_out = 256): work units of (row
  // tile, 128-column half), two CTAs per SM -- against the tile quantisation
  // of the deepest levels (~177 row tiles for 148 SMs).  Measured slower:
  // 0.142 vs 0.099 ms at L4 256->256 k3, 0.279 vs 0.209 at L3 (a half-width
  // unit costs nearly the MMA-issue time of a full one), step 711 vs 718.
  {
    const bool ts_req = env_int("SCB_IC_TS", 0) != 0;
    const bool split = !vk && !ts_req && n_pad == 256 && env_int("SCB_IC_NSPLIT", 1) == 2;
    p.nsplit = split ? 2 : 1;
    p.n_unit = split ? 128 : n_pad;
  }
  p.epi_cols = (p.n_unit % 32 == 0) ? 32 : 16;
  p.relu = relu;
  p.idesc = (1u << 4) | ((uint32_t)(p.n_unit >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  // Launch shape: two CTAs per SM when both accumulator pairs fit in TMEM
  // (C_out <= 128) -- one CTA's producer / MMA-issue gaps are filled by the
  // other -- else one; P producer threads per output row.
  // Two accumulators per CTA (the epilogue of tile i overlaps tile i+1).
  // SCB_IC_NACC=1 trades that for two CTAs per SM at C_out > 128: measured
  // 3-5 % slower on the 256-channel layers.
  p.nacc = 2;
  p.rowmode = (env_int("SCB_IC_ROW", 0) && !vk) ? 1 : 0;
  if (const char* e = getenv("SCB_IC_NACC")) p.nacc = atoi(e) == 1 ? 1 : 2;
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.nacc * p.n_unit)) cols *= 2;
  p.tmem_cols = cols;
  // 3 CTAs per SM measured 12 % faster for 64->64 (K chunks of 64) and
  // slower for narrower inputs; 2 whenever both accumulator pairs fit
  int ctas = (cols <= 128 && p.kc == 64) ? 3 : (cols <= 256 ? 2 : 1);
  {
    const int want = env_int("SCB_IMPLICIT_CTAS", ctas);
    ctas = (want >= 3 && cols <= 128) ? 3 : (want >= 2 && cols <= 256 ? 2 : 1);
  }
  const int cpr = p.kc / 8;
  const int P = 1;  // producer threads per row (2 measured slower: more warps, same issue stream)
  const int nprod = 128 * P;
  p.total_tiles = (int)((n_out + BM - 1) / BM) * p.nsplit;
  auto r1024 = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  p.b_tx = (uint32_t)(p.n_unit * p.kc * 2);
  p.a_off_bytes = r1024((uint32_t)(BM * p.kc * 2));
  p.b_off_bytes = r1024(p.b_tx);
  const uint32_t op_bytes = p.a_off_bytes + p.b_off_bytes;
  int ops = (int)((uint32_t)env_int("SCB_IC_STAGE_KB", ctas == 3 ? 24 : (ctas == 2 ? 42 : 96)) *
                  1024u / op_bytes);
  ops = std::max(1, std::min(ops, std::min(MAX_OPS, p.nblk)));
  if (env_int("SCB_IMPLICIT_OPS", 0) > 0) ops = std::min(env_int("SCB_IMPLICIT_OPS", 0), std::min(MAX_OPS, p.nblk));
  p.ops = ops;
  p.stage_bytes = ops * op_bytes;
  p.ldf = ldf;
  p.ldh = hits_ld(n_out);
  p.feat = (const __half*)features;
  p.feat2 = (const __half*)features2;
  p.ldf2 = ldf2;
  p.c_split = features2 ? c_split : c_in;
  p.hits = hits;
  p.scale = scale;
  p.shift = shift;
  p.bias = bias;
  p.residual = (const __half*)residual;
  if (const char* dbg = getenv("SCB_IMPLICIT_DEBUG")) p.debug = atoi(dbg);
  p.bsleep = env_int("SCB_IC_BSLEEP", 32);
  p.esleep = env_int("SCB_IC_ESLEEP", 256);
  // A-in-TMEM form (opt-in, SCB_IC_TS=1): K chunks of 32 / 64 channels only.
  // Measured faster than the shared-memory form only on the k3 C_out = 256
  // layers (0.197 vs 0.209 ms, 0.086 vs 0.097 ms), slower on the K = 1 and
  // narrower ones (0.029 vs 0.021 ms at 256->256 K=1, 0.71 vs 0.70 ms at
  // 96->96 k3), and the MinkUNet step is 0.5 % faster without it (710 vs 707).
  const bool ts = !vk && (p.kc == 64 || p.kc == 32) && env_int("SCB_IC_TS", 0) != 0;
  if (ts) {
    p.nacc = (2 * n_pad + 2 * 32 <= 512) ? 2 : 1;
    if (env_int("SCB_IC_NACC", 2) == 1) p.nacc = 1;
    p.tmem_cols = 512;
    p.ops = 64 / p.kc;
    p.groups = (volume + p.ops - 1) / p.ops;
    p.a_off_bytes = 0;
    p.a_stage_bytes = 0;
    p.stage_bytes = p.ops * p.b_off_bytes;
    p.epi_bufs = 2;
    const int fixed = 1024 + 4 * p.epi_bufs * EPI_BUF + volume * BM * 4 + 40 * 8 + 64;
    int stages = std::min((512 - p.nacc * n_pad) / 32, (227 * 1024 - fixed) / (int)p.stage_bytes);
    stages = std::min(stages, std::min(16, std::max(2, env_int("SCB_IC_STAGES", 16))));
    SCB_CHECK_ARG(stages >= 2, "TS: stage does not fit");
    p.stages = stages;
    const int smem_ts = fixed + stages * (int)p.stage_bytes;
    CUtensorMap mB, mO;
    std::string err;
    if (!encode_map_2d(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, weights_packed, k_pad,
                       (long long)volume * n_pad, k_pad, p.kc, n_pad, p.swz, err) ||
        !encode_map_2d(&mO, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, out, c_out, n_out, ldo,
                       p.epi_cols, 32, p.epi_cols * 2, err)) {
      set_error(std::string("scb_conv_implicit: ") + err);
      return SCB_ECUDA;
    }
    const int grid = std::min(p.total_tiles, device_sms());
    const int pw = std::min(4, std::max(2, env_int("SCB_IC_PW", 2)));
    cudaStream_t s = as_stream(stream);
    auto launch = [&](auto kernel, int threads) -> int {
      SCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem_ts;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = env_int("SCB_IC_PDL", 1) ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      SCB_CUDA(cudaLaunchKernelEx(&cfg, kernel, mB, mO, p));
      return SCB_OK;
    };
    int rc = SCB_EINVAL;
#define SCB_TS_LAUNCH_PW(VV, KK)                                                               \
  rc = pw == 2   ? launch(implicit_conv_ts_kernel<VV, KK, 2>, 64 + 256 + 128)                 \
       : pw == 3 ? launch(implicit_conv_ts_kernel<VV, KK, 3>, 64 + 384 + 128)                 \
                 : launch(implicit_conv_ts_kernel<VV, KK, 4>, 64 + 512 + 128);
#define SCB_TS_LAUNCH_K(VV)                                                                    \
  if (p.kc == 64) { SCB_TS_LAUNCH_PW(VV, 64) } else { SCB_TS_LAUNCH_PW(VV, 32) }
    if (volume == 27) { SCB_TS_LAUNCH_K(27) }
    else if (volume == 8) { SCB_TS_LAUNCH_K(8) }
    else { SCB_TS_LAUNCH_K(1) }
#undef SCB_TS_LAUNCH_K
#undef SCB_TS_LAUNCH_PW
    if (rc != SCB_OK) return rc;
    if (p.debug & 16) {
      unsigned long long prof[16];
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(prof, g_ic_prof, sizeof(prof));
      fprintf(stderr, "[ts prof cta0] tiles=%llu total=%llu Aempty(row0)=%llu Bempty=%llu MMAfull=%llu "
              "MMAtempty=%llu EPItfull=%llu (stages=%d pw=%d nacc=%d)\n", prof[9], prof[7], prof[0],
              prof[2], prof[3], prof[4], prof[5], p.stages, pw, p.nacc);
      static const unsigned long long zero[16] = {0};
      cudaMemcpyToSymbol(g_ic_prof, zero, sizeof(zero));
    }
    SCB_LAUNCHED();
    return SCB_OK;
  }
  // shared memory: stages (A + B blocks, one presence word per producer
  // thread) + epilogue staging + the tile's neighbour table + barriers
  auto fixed_bytes = [&](int epi_bufs) {
    return 1024 + 4 * epi_bufs * EPI_BUF + volume * BM * 4 + 40 * 8 + 64;
  };
  int smem_cap = ctas == 3 ? 75 * 1024 : (ctas == 2 ? 113 * 1024 : 227 * 1024);
  auto fit = [&](int e) { return (smem_cap - fixed_bytes(e)) / (int)p.stage_bytes; };
  while (fit(1) < 2 && p.ops > 1) {  // fewer offsets per stage, then one CTA per SM
    --p.ops;
    p.stage_bytes = p.ops * op_bytes;
  }
  if (fit(1) < 2 && ctas == 3) {
    ctas = 2;
    smem_cap = 113 * 1024;
  }
  if (fit(1) < 2 && ctas == 2) {
    ctas = 1;
    smem_cap = 227 * 1024;
  }
  // double-buffered epilogue staging unless the second buffer costs a stage
  p.epi_bufs = fit(2) >= fit(1) ? 2 : 1;
  if (const char* e = getenv("SCB_IC_EPI_BUFS")) p.epi_bufs = atoi(e) == 1 ? 1 : 2;
  p.groups = (p.nblk + p.ops - 1) / p.ops;
  p.a_stage_bytes = p.ops * p.a_off_bytes;
  int stages = std::min(fit(p.epi_bufs), 16);
  stages = std::min(stages, std::max(2, env_int("SCB_IC_STAGES", 16)));
  SCB_CHECK_ARG(stages >= 2, "stage does not fit in shared memory");
  p.stages = stages;
  const int smem = fixed_bytes(p.epi_bufs) + stages * (int)p.stage_bytes;

  CUtensorMap mB, mO;
  std::string err;
  if (!(vk ? encode_map_2d(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, weights_packed, kv, n_pad,
                           kv, 64, n_pad, 128, err)
           : encode_map_2d(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, weights_packed, k_pad,
                           (long long)volume * n_pad, k_pad, p.kc, p.n_unit, p.swz, err)) ||
      !encode_map_2d(&mO, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, out, c_out, n_out, ldo,
                     p.epi_cols, 32, p.epi_cols * 2, err)) {
    set_error(std::string("scb_conv_implicit: ") + err);
    return SCB_ECUDA;
  }
  const int grid = p.total_tiles < ctas * device_sms() ? p.total_tiles : ctas * device_sms();
  cudaStream_t s = as_stream(stream);
  auto launch = [&](auto kernel) -> int {
    SCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64 + nprod + 128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = env_int("SCB_IC_PDL", 1) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SCB_CUDA(cudaLaunchKernelEx(&cfg, kernel, mB, mO, p));
    return SCB_OK;
  };
  int rc = SCB_EINVAL;
#define SCB_IC_LAUNCH_P(VV, KK)                                                                \
  rc = ctas == 3 ? launch(implicit_conv_f16_kernel<VV, KK, 1, 3>)                              \
     : ctas == 2 ? launch(implicit_conv_f16_kernel<VV, KK, 1, 2>)                              \
                 : launch(implicit_conv_f16_kernel<VV, KK, 1, 1>);
#define SCB_IC_LAUNCH_K(VV)                                                                    \
  if (p.kc == 64) { SCB_IC_LAUNCH_P(VV, 64) }                                                  \
  else if (p.kc == 32) { SCB_IC_LAUNCH_P(VV, 32) }                                             \
  else { SCB_IC_LAUNCH_P(VV, 16) }
  if (volume == 27) {
    SCB_IC_LAUNCH_K(27)
  } else if (volume == 8) {
    SCB_IC_LAUNCH_K(8)
  } else if (volume == 1) {
    SCB_IC_LAUNCH_K(1)
  }
#undef SCB_IC_LAUNCH_K
#undef SCB_IC_LAUNCH_P
  if (rc == SCB_EINVAL) set_error("scb_conv_implicit: V must be 1, 8 or 27");
  if (rc != SCB_OK) return rc;
  if (p.debug & 16) {
    unsigned long long prof[16];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(prof, g_ic_prof, sizeof(prof));
    fprintf(stderr, "[ic prof cta0] tiles=%llu total=%llu Aempty=%llu Bempty=%llu MMAfull=%llu "
            "MMAtempty=%llu EPItfull=%llu EPIbulk=%llu MMAissue=%llu Aitems=%llu (stages=%d ops=%d "
            "P=%d ctas=%d)\n",
            prof[9], prof[7], prof[0], prof[2], prof[3], prof[4], prof[5], prof[6], prof[10],
            prof[11], p.stages, p.ops, P, ctas);
    static const unsigned long long zero[16] = {0};
    cudaMemcpyToSymbol(g_ic_prof, zero, sizeof(zero));
  }
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_conv_implicit_cat(const void* features, int64_t ldf, int32_t c_split,
                                         const void* features2, int64_t ldf2, int64_t n_in,
                                         int32_t c_in, const int32_t* hits, int32_t volume,
                                         int64_t n_out, const void* weights_packed,
                                         int32_t c_out, void* out, int64_t ldo,
                                         const float* scale, const float* shift,
                                         const float* bias, const void* residual, int32_t relu,
                                         scb_stream_t stream) {
  return conv_implicit_impl(features, ldf, c_split, features2, ldf2, n_in, c_in, hits, volume,
                            n_out, weights_packed, c_out, out, ldo, scale, shift, bias, residual,
                            relu, stream, 0);
}

extern "C" int32_t scb_conv_implicit_vk(const void* features, int64_t ldf, int32_t c_split,
                                        const void* features2, int64_t ldf2, int64_t n_in,
                                        int32_t c_in, const int32_t* hits, int32_t volume,
                                        int64_t n_out, const void* weights_vk, int32_t c_out,
                                        void* out, int64_t ldo, const float* scale,
                                        const float* shift, const float* bias,
                                        const void* residual, int32_t relu,
                                        scb_stream_t stream) {
  return conv_implicit_impl(features, ldf, c_split, features2, ldf2, n_in, c_in, hits, volume,
                            n_out, weights_vk, c_out, out, ldo, scale, shift, bias, residual,
                            relu, stream, 1);
}
