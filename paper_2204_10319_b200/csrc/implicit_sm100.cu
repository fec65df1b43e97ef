// Fused gather -> tcgen05 GEMM -> epilogue convolution (the "implicit GEMM"
// dataflow): one persistent kernel per layer computes
//
//   out[k] = epilogue( sum_n  features[hits[n][k]] . W[n] )      (absent -> 0)
//
// for 128-row output tiles, accumulating the tile's offsets in TMEM (double-
// buffered accumulators, so the epilogue of tile i overlaps tile i+1).  The
// gather is fused into the operand load: cp.async moves each present
// neighbour's 16-B row chunks straight into the 128/64/32-B swizzled UMMA
// layout (absent neighbours are zero-filled without a read), so neither the
// gather buffer nor the f32 partials ever reach HBM.  Each output row is
// written once (fp16) with BN / bias / residual / ReLU applied in registers.
//
// Sparse offset skipping: `tile_mask[t]` (scb_tile_masks) has bit n set when
// some row of tile t has a neighbour at offset n.  Every role walks only the
// set bits, `ops` offsets per pipeline stage, so an absent (tile, offset)
// block costs no weight load, no copies and no MMA.  Rows reordered by their
// presence mask (scb_presence_masks + scb_mask_sort, the TorchSparse++
// bitmask sort) turn ~94 % live blocks of a LiDAR level into ~40 %.
//
// Pipeline (per stage: up to `ops` active offsets x one K chunk of A and B):
//   * producers never block on their own copies: each thread's completion is
//     tracked by cp.async.mbarrier.arrive.noinc, absent rows are zero-filled
//     by ignore-src cp.async, so every write of a stage is async-tracked;
//   * copies are lane-per-chunk (the CPR lanes of a row copy its consecutive
//     16-B chunks);
//   * the MMA warp runs converged (stage indices and descriptors in uniform
//     registers) and one elected lane issues; descriptors advance by
//     constant steps.
//
// Warp roles (64 + 128 + 128 threads, persistent, 1-3 CTAs per SM):
//   warp 0        TMA producer of the weight slices (B, K-major fp16)
//   warp 1        TMEM allocator + MMA issuer
//   warps 2..5    A producers (one output row each)
//   warps 6..9    epilogue: tcgen05.ld -> epilogue -> swizzled smem -> TMA store
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace scb {
namespace ic {

using namespace ::scb::ptx;

constexpr int BM = 128;
constexpr int EPI_BUF = 32 * 64;        // 32 rows x 64 B (32 fp16 columns)
constexpr int MAX_OPS = 8;              // kernel offsets per pipeline stage
constexpr int NPROD = 128;              // A-producer threads (one per tile row)
constexpr int EPI0 = 6;                 // first epilogue warp

struct Params {
  long long n_out;
  int n_in, c_in, c_out, V, n_pad, kc, n_kchunks, swz, epi_cols, total_tiles, relu;
  int ops;                  // active offsets per stage (small C_in -> several)
  int a_stages, b_stages;   // ring depths: A (gathered rows) and B (weights) separately
  int epi_bufs;             // epilogue staging buffers per warp (1 or 2)
  int nacc;                 // TMEM accumulator buffers (2: epilogue overlaps the next tile)
  int interleave;           // tile order: 1 = t = blockIdx + i * gridDim, 0 = contiguous ranges
  int debug;                // EXPERIMENT (SCB_IC_DEBUG): 1 = B loaded once, 2 = no A copies, 4 = no proxy fence
  int pair;                 // CTA-pair kernel: work items are 256-row pair tiles (rows of CTA r: 2T + r)
  int idx_slots;            // pair kernel: index-ring slots (one offset group's hit rows each)
  uint32_t idx_slot_bytes;  // ops x 128 x 4
  uint32_t all_bits;        // (1 << V) - 1
  uint32_t idesc, tmem_cols;
  uint32_t a_off_bytes;     // one offset's A block [128 rows][kc] (1024-aligned)
  uint32_t b_off_bytes;     // one offset's B block [n_pad][kc]   (1024-aligned)
  uint32_t a_stage_bytes, b_stage_bytes;
  uint32_t b_tx;            // bytes one offset's B load delivers
  long long ldf, ldh;       // feature row stride, hit-matrix row stride
  const __half* feat;       // [n_in][ldf]: input channels [0, c_split)
  const __half* feat2;      // nullable: channels [c_split, c_in) (skip concat), [n_in][ldf2]
  long long ldf2;
  int c_split;
  const int* hits;          // [V][ldh] input row or -1; NULL = identity map (K = 1, s = 1)
  const uint32_t* tmask;    // nullable: [total_tiles] active-offset bits per row tile
  const float* scale;       // nullable (with shift)
  const float* shift;
  const float* bias;        // nullable
  const __half* residual;   // nullable, [n_out][c_out]
  const int* orow;          // nullable: tile row r holds output row orow[r] (stored row by row)
  long long ldo;            // output row stride (elements), for the orow stores
  __half* out;              // output base, for the orow stores
};

// Index registers a producer thread holds per offset group: ops x IT <=
// MAX_IDX (IT = K-chunk / 8 rows per thread), for the current group and the
// next; 8 at three CTAs per SM (64 registers per thread).
constexpr int MAX_IDX = 16;
__host__ __device__ constexpr int max_idx(int minb) { return minb >= 3 ? 8 : MAX_IDX; }

// Active offsets of row tile t (never empty: an all-absent tile still needs
// its accumulator zeroed, so it runs offset 0 with every row zero-filled).
__device__ __forceinline__ uint32_t tile_bits(const Params& p, int t) {
  uint32_t m = p.all_bits;
  if (p.tmask) {
    if (p.pair) {  // a pair tile runs the union of its two row tiles' offsets
      m = __ldg(p.tmask + 2 * t);
      if (2 * t + 1 < p.total_tiles) m |= __ldg(p.tmask + 2 * t + 1);
      m &= p.all_bits;
    } else {
      m = __ldg(p.tmask + t) & p.all_bits;
    }
  }
  return m ? m : 1u;
}

// The next group of up to `ops` active offsets (lowest bits first).
__device__ __forceinline__ uint32_t next_group(uint32_t& rem, int ops) {
  uint32_t g = 0;
  for (int o = 0; o < ops && rem; ++o) {
    const uint32_t b = rem & (0u - rem);
    g |= b;
    rem ^= b;
  }
  return g;
}

// The CTA's tile sequence: t0, t0 + step, ... < lim.
struct TileSeq {
  int t0, step, lim;
};
__device__ __forceinline__ TileSeq tile_seq(const Params& p) {
  if (p.pair)  // one pair tile per cluster (CTAs 2c, 2c + 1), interleaved
    return {(int)(blockIdx.x >> 1), (int)(gridDim.x >> 1), (p.total_tiles + 1) >> 1};
  if (p.interleave) return {(int)blockIdx.x, (int)gridDim.x, p.total_tiles};
  const int b = (int)((long long)p.total_tiles * blockIdx.x / gridDim.x);
  const int e = (int)((long long)p.total_tiles * (blockIdx.x + 1) / gridDim.x);
  return {b, 1, e};
}

// Walks the CTA's (tile, offset group) sequence: every role iterates it in
// the same order, so stage i of every ring refers to the same work.
struct GroupIter {
  int t;          // current tile (>= lim: done)
  uint32_t rem;   // active offsets of tile t not yet grouped
  uint32_t mg;    // current group
  uint32_t nmask; // the next tile's offsets, loaded a whole tile ahead (no
                  // dependent global load at tile boundaries)
  bool first;     // the group is tile t's first
  __device__ __forceinline__ void start(const Params& p, const TileSeq& ts) {
    t = ts.t0;
    rem = t < ts.lim ? tile_bits(p, t) : 0u;
    nmask = t + ts.step < ts.lim ? tile_bits(p, t + ts.step) : 0u;
    mg = next_group(rem, p.ops);
    first = true;
  }
  __device__ __forceinline__ void advance(const Params& p, const TileSeq& ts) {
    first = rem == 0u;
    if (first) {
      t += ts.step;
      rem = t < ts.lim ? nmask : 0u;
      nmask = t + ts.step < ts.lim ? tile_bits(p, t + ts.step) : 0u;
    }
    mg = next_group(rem, p.ops);
  }
  __device__ __forceinline__ bool done(const TileSeq& ts) const { return t >= ts.lim; }
  __device__ __forceinline__ bool last_of_tile() const { return rem == 0u; }
};

#ifdef SCB_IC_TRACE
// Per-stage timeline of the first CTAs (tools/ic_trace.py; trace builds
// only: make trace): [cta][stage][event] clock64 stamps, events
//   0 producer 0 passed the empty wait (starts issuing the stage's copies)
//   1 MMA warp passed the full wait (A + B landed)
//   2 MMA warp committed the stage's MMAs
//   3 MMA warp passed the A-full wait (before the B-full wait)
//   4 elected MMA lane passed the proxy fence, 5 issued the stage's MMAs
constexpr int TR_CTAS = 4, TR_STAGES = 512, TR_EV = 6;
__device__ long long g_ic_trace[TR_CTAS][TR_STAGES][TR_EV];
__device__ __forceinline__ void trace_stamp(int idx, int ev) {
  if (blockIdx.x < TR_CTAS && idx < TR_STAGES) g_ic_trace[blockIdx.x][idx][ev] = clock64();
}
#define IC_TRACE(idx, ev) trace_stamp((idx), (ev))
#else
#define IC_TRACE(idx, ev) ((void)0)
#endif

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
                                              int lane, const TileSeq& ts, uint32_t rank = 0) {
  const int q = warp & 3;
  uint8_t* bufs = epi_base + (warp - EPI0) * p.epi_bufs * EPI_BUF;
  int acc = 0, nbuf = 0;
  uint32_t acc_phase = 0;
  const int chunks = p.n_pad / p.epi_cols;
  for (int t = ts.t0; t < ts.lim; t += ts.step) {
    mbar_wait_sleep(tfull + acc, acc_phase, 256);
    tc_after();
    const long long row0 = (long long)(p.pair ? 2 * t + (int)rank : t) * BM + 32 * q;
    const long long r = row0 + lane;        // tile row
    const bool row_ok = r < p.n_out;
    // output row of this lane: the tile row itself, or orow[r] when the
    // tiles run over a permutation of the output rows (one-hot maps)
    const long long k = (p.orow && row_ok) ? (long long)__ldg(p.orow + r) : r;
    for (int j = 0; j < chunks && row0 < p.n_out; ++j) {
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * p.n_pad + j * p.epi_cols);
      const int c0 = j * p.epi_cols;   // output column
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
      if (p.orow) {
        // permuted rows: each lane stores its own row's columns (16-B stores)
        if (row_ok) {
          uint4* dst = reinterpret_cast<uint4*>(p.out + k * p.ldo + c0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c * 8 < ncol && c0 + c * 8 < p.c_out)
              dst[c] = make_uint4(pack_half2(v[8 * c], v[8 * c + 1]), pack_half2(v[8 * c + 2], v[8 * c + 3]),
                                  pack_half2(v[8 * c + 4], v[8 * c + 5]), pack_half2(v[8 * c + 6], v[8 * c + 7]));
          }
        }
        continue;
      }
      uint8_t* buf = bufs + nbuf * EPI_BUF;
      if (lane == 0) {
        if (p.epi_bufs == 2) bulk_wait_read1();
        else bulk_wait_read0();
      }
      __syncwarp();
      if (ncol == 32) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 w = make_uint4(pack_half2(v[8 * c], v[8 * c + 1]), pack_half2(v[8 * c + 2], v[8 * c + 3]),
                               pack_half2(v[8 * c + 4], v[8 * c + 5]), pack_half2(v[8 * c + 6], v[8 * c + 7]));
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint4 w = make_uint4(pack_half2(v[8 * c], v[8 * c + 1]), pack_half2(v[8 * c + 2], v[8 * c + 3]),
                               pack_half2(v[8 * c + 4], v[8 * c + 5]), pack_half2(v[8 * c + 6], v[8 * c + 7]));
          *reinterpret_cast<uint4*>(buf + lane * 32 + ((c ^ ((lane >> 2) & 1)) << 4)) = w;
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
    if (lane == 0) {
      if (p.pair)  // the pair's MMA issuer (CTA 0) waits on CTA 0's barrier
        mbar_arrive_cluster(mapa_shared(smem_u32(tempty + acc), 0));
      else
        mbar_arrive(tempty + acc);
    }
    if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
  }
  if (lane == 0) bulk_wait_all();
}

constexpr int PAIR_THREADS = 64 + NPROD + 128 + 32;   // + warp 10: the index loader
constexpr int IC_THREADS = PAIR_THREADS;
constexpr int IDX_WARP = 10;

template <int V, int KC, int MINB>
__global__ void __launch_bounds__(IC_THREADS, MINB)
    implicit_conv_f16_kernel(const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmOut,
                             const __grid_constant__ Params p) {
  constexpr int CPR = KC / 8;              // 16-B chunks per row per K chunk
  constexpr int IT = CPR;                  // chunks a producer thread copies per offset
  constexpr int SWZ = KC * 2;              // swizzle span = row bytes
  constexpr int RPI = NPROD / CPR;         // rows one warp-wide item sweep covers
  constexpr int MI = max_idx(MINB);
  constexpr int MAXO = MI / IT;            // offsets per stage the index registers hold
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* b_base = smem + (size_t)p.a_stages * p.a_stage_bytes;
  uint8_t* epi_base = b_base + (size_t)p.b_stages * p.b_stage_bytes;
  uint8_t* idx_base = epi_base + 4 * p.epi_bufs * EPI_BUF;   // [idx_slots][ops][128] int32
  uint64_t* afull = (uint64_t*)(idx_base + (size_t)p.idx_slots * p.idx_slot_bytes);
  uint64_t* aempty = afull + p.a_stages;
  uint64_t* bfull = aempty + p.a_stages;
  uint64_t* bempty = bfull + p.b_stages;
  uint64_t* tfull = bempty + p.b_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ifull = tempty + 2;
  uint64_t* iempty = ifull + p.idx_slots;
  uint32_t* tmem_slot = (uint32_t*)(iempty + p.idx_slots);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileSeq ts = tile_seq(p);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.a_stages; ++s) {
      mbar_init(afull + s, NPROD);  // one async (noinc) arrive per producer thread
      mbar_init(aempty + s, 1);
    }
    for (int s = 0; s < p.b_stages; ++s) {
      mbar_init(bfull + s, 1);      // the B expect_tx arrive
      mbar_init(bempty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    for (int i = 0; i < p.idx_slots; ++i) {
      mbar_init(ifull + i, 1);        // the loader's arrive.expect_tx
      mbar_init(iempty + i, NPROD);   // every producer thread has read its indices
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
    // ============ B producer: the stage's weight slices via TMA, own ring
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      GroupIter g;
      for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
        const int nv = __popc(g.mg);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          mbar_wait_sleep(bempty + stage, phase ^ 1, 32);
          if ((p.debug & 1) && (phase || g.t != ts.t0)) {
            mbar_arrive(bfull + stage);
            if (++stage == p.b_stages) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(bfull + stage, nv * p.b_tx);
          uint8_t* sb = b_base + (size_t)stage * p.b_stage_bytes;
          uint32_t x = g.mg;
          for (int o = 0; o < nv; ++o) {
            const int n = __ffs(x) - 1;
            x &= x - 1;
            tma_load_2d(sb + o * p.b_off_bytes, &tmB, bfull + stage, kk * p.kc, n * p.n_pad);
          }
          if (++stage == p.b_stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 2 && warp < EPI0) {
    // ============ A producers.  Item `it` of thread pt is 16-B chunk
    // (pt % CPR) of tile row it * RPI + pt / CPR (consecutive lanes copy
    // consecutive chunks of a row).  The input row of every item of a group
    // is loaded straight from the hit matrix into registers one group ahead
    // (no shared index table, no producer barrier); each stage is one K
    // chunk of the group's offsets, written with one cp.async per item
    // (ignore-src zero-fill for absent neighbours), completion tracked by a
    // noinc arrive on the stage's full barrier.
    const int pt = threadIdx.x - 64;
    const int cr = pt / CPR, cc = pt % CPR;
    uint32_t roff[IT];                        // smem offset of item it inside a block
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int r = it * RPI + cr;
      const int rxr = SWZ == 128 ? (r & 7) : (SWZ == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
      roff[it] = (uint32_t)(r * (KC * 2)) + ((uint32_t)(cc ^ rxr) << 4);
    }
    int cur[MI], nxt[MI];
    // input rows of group (t, mg) for this thread's items straight from the
    // hit matrix (-1 = absent): the path without the index ring, one group ahead
    auto load_idx = [&](int t, uint32_t mg, int* dst) {
      const long long r0 = (long long)t * BM + cr;
      uint32_t x = mg;
#pragma unroll
      for (int o = 0; o < MAXO; ++o) {
        const int n = x ? __ffs(x) - 1 : 0;
        const bool on = x != 0u;
        x &= x - 1;
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const long long k = r0 + it * RPI;
          int j = -1;
          if (on && k < p.n_out) j = p.hits ? __ldg(p.hits + (long long)n * p.ldh + k) : (int)k;
          dst[o * IT + it] = j;
        }
      }
    };
    const uint32_t ldfb1 = (uint32_t)(p.ldf * 2);   // row strides in bytes (host-checked < 2^32)
    const uint32_t ldfb2 = (uint32_t)(p.ldf2 * 2);
    int stage = 0, islot = 0;
    uint32_t phase = 0, iph = 0;
#ifdef SCB_IC_TRACE
    int nstage = 0;
#endif
    const bool ring = p.hits && p.idx_slots > 0;
    GroupIter g;
    g.start(p, ts);
    if (!ring && !g.done(ts)) load_idx(g.t, g.mg, nxt);
    for (; !g.done(ts); g.advance(p, ts)) {
      const int nv = __popc(g.mg);
      const long long row0 = (long long)g.t * BM;
      if (!ring) {
#pragma unroll
        for (int i = 0; i < MI; ++i) cur[i] = nxt[i];
        GroupIter gn = g;   // the next group's rows load while this one copies
        gn.advance(p, ts);
        if (!gn.done(ts)) load_idx(gn.t, gn.mg, nxt);
      } else {
        // the group's input rows from the index ring (the loader warp bulk-
        // copies the hit-matrix rows several groups ahead)
        mbar_wait(ifull + islot, iph);
        const int* tab = reinterpret_cast<const int*>(idx_base + (size_t)islot * p.idx_slot_bytes);
#pragma unroll
        for (int o = 0; o < MAXO; ++o) {
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const int r = it * RPI + cr;
            cur[o * IT + it] = (o < nv && row0 + r < p.n_out) ? tab[o * BM + r] : -1;
          }
        }
        // the slot's next fill is an async-proxy (bulk copy) write: order this
        // thread's generic reads of it before that write (WAR across proxies)
        fence_async_smem();
        mbar_arrive(iempty + islot);
        if (++islot == p.idx_slots) { islot = 0; iph ^= 1; }
      }
      for (int kk = 0; kk < p.n_kchunks; ++kk) {
        mbar_wait(aempty + stage, phase ^ 1);
        if (pt == 0) IC_TRACE(nstage, 0);
        const uint32_t dst = smem_u32(smem + (size_t)stage * p.a_stage_bytes);
        const int col0 = kk * KC;
        const int live = min(CPR, (p.c_in - col0) / 8);  // chunks inside C_in
        // this lane's 8 columns come from the first or (concat) second input
        const int col = col0 + cc * 8;
        const bool second = p.feat2 != nullptr && col >= p.c_split;
        const uint64_t fb = second
            ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((col - p.c_split) * 2)
            : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(col * 2);
        const uint32_t ldb = second ? ldfb2 : ldfb1;
        const bool live_c = cc < live;
#pragma unroll
        for (int o = 0; o < MAXO; ++o) {
          if (o < nv && !(p.debug & 2)) {
            const uint32_t blk = dst + o * p.a_off_bytes;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
              const int j = live_c ? cur[o * IT + it] : -1;
              const uint64_t src = fb + (uint64_t)(uint32_t)max(j, 0) * (uint64_t)ldb;
              // L2-only (.cg): an L1-allocating .ca gather measured 4-13 % slower
              asm volatile(
                  "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                  "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(blk + roff[it]),
                  "l"(src), "r"(j) : "memory");
            }
          }
        }
        cp_async_arrive_noinc(afull + stage);   // fires when this thread's copies land
#ifdef SCB_IC_TRACE
        ++nstage;
#endif
        if (++stage == p.a_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == IDX_WARP) {
    // ============ index loader: each group's hit-matrix rows (the tile's 128
    // rows of every active offset, contiguous in hits[n][.]) by bulk copy
    if (lane == 0 && p.hits && p.idx_slots > 0) {
      int slot = 0;
      uint32_t ph = 0;
      GroupIter g;
      for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
        mbar_wait_sleep(iempty + slot, ph ^ 1, 20);
        const long long row0 = (long long)g.t * BM;
        const long long avail = p.ldh - row0;   // entries of each hit row from row0 on
        const uint32_t bytes = avail <= 0 ? 0u : (uint32_t)((avail < BM ? avail : BM) * 4);
        if (bytes) {
          const int nv = __popc(g.mg);
          mbar_expect_tx(ifull + slot, (uint32_t)nv * bytes);
          const uint32_t dst = smem_u32(idx_base + (size_t)slot * p.idx_slot_bytes);
          uint32_t x = g.mg;
          for (int o = 0; o < nv; ++o) {
            const int n = __ffs(x) - 1;
            x &= x - 1;
            bulk_load(dst + o * BM * 4, p.hits + (long long)n * p.ldh + row0, bytes, ifull + slot);
          }
        } else {
          mbar_arrive(ifull + slot);
        }
        if (++slot == p.idx_slots) { slot = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer.  The whole warp runs the loop (so stage
    // indices and descriptors stay warp-uniform, in uniform registers) and
    // one elected lane issues; each stage's MMAs release their A and B
    // slots with one commit each.
    const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
    const uint32_t sbo = 8u * (uint32_t)p.swz;
    const uint64_t adesc_base = make_sdesc(smem_u32(smem), sbo, layout);
    const uint64_t bdesc_base = make_sdesc(smem_u32(b_base), sbo, layout);
    const uint32_t a_stage_d = p.a_stage_bytes >> 4, b_stage_d = p.b_stage_bytes >> 4;
    const uint32_t a_off_d = p.a_off_bytes >> 4, b_off_d = p.b_off_bytes >> 4;
    const uint32_t idesc = p.idesc;
    const uint32_t tmem0 = __shfl_sync(0xffffffffu, tmem_base, 0);
#ifdef SCB_IC_TRACE
    int nstage = 0;
#endif
    int as = 0, bs = 0, acc = 0;
    uint32_t aph = 0, bph = 0, acc_phase = 0;
    uint32_t d = 0, acc0 = 0;
    GroupIter g;
    for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
      if (g.first) {
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_after();
        d = tmem0 + (uint32_t)acc * (uint32_t)p.n_pad;
        acc0 = 0u;   // the tile's first MMA overwrites the accumulator
      }
      const int nv = __popc(g.mg);
      for (int kk = 0; kk < p.n_kchunks; ++kk) {
        mbar_wait(afull + as, aph);
        if (lane == 0) IC_TRACE(nstage, 3);
        mbar_wait(bfull + bs, bph);
        if (lane == 0) IC_TRACE(nstage, 1);
        const uint64_t ad = adesc_base + (uint64_t)(as * a_stage_d);
        const uint64_t bd = bdesc_base + (uint64_t)(bs * b_stage_d);
        if (elect_one()) {
          if (!(p.debug & 4)) fence_async_smem();  // cp.async (generic proxy) data -> tcgen05 reads
          tc_after();
          IC_TRACE(nstage, 4);
#pragma unroll
          for (int o = 0; o < MAX_OPS; ++o) {
            if (o < nv) {
              const uint64_t a = ad + (uint64_t)(o * a_off_d);
              const uint64_t b = bd + (uint64_t)(o * b_off_d);
              mma_f16(d, a, b, idesc, o ? 1u : acc0);
#pragma unroll
              for (int k = 1; k < KC / 16; ++k) mma_f16(d, a + 2u * k, b + 2u * k, idesc, 1u);
            }
          }
          IC_TRACE(nstage, 5);
          mma_commit(aempty + as);
          mma_commit(bempty + bs);
        }
        __syncwarp();
        if (lane == 0) IC_TRACE(nstage, 2);
#ifdef SCB_IC_TRACE
        ++nstage;
#endif
        acc0 = 1u;
        if (++as == p.a_stages) { as = 0; aph ^= 1; }
        if (++bs == p.b_stages) { bs = 0; bph ^= 1; }
      }
      if (g.last_of_tile()) {
        if (elect_one()) mma_commit(tfull + acc);
        __syncwarp();
        if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= EPI0 && warp < EPI0 + 4) {
    epilogue_role(p, &tmOut, tmem_base, tfull, tempty, epi_base, warp, lane, ts);
  }

  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

// ============ The CTA-pair form (tcgen05 cta_group::2).  A cluster of two
// CTAs on one TPC computes 256-row pair tiles: CTA r gathers rows
// (2T + r) * 128 .. + 127 of pair tile T into its own smem and holds half of
// the weight slice (N / 2 output channels); CTA 0's MMA thread issues one
// M = 256 MMA per K step for both SMs, so each instruction and each pipeline
// stage carries twice the work of the single-CTA kernel (the per-stage issue
// overhead of that kernel is what bounds it), and each SM streams half the
// weights.  One ring per CTA (a stage holds its A rows and its B half):
//   full[s]   CTA 0: its producers (noinc) + its B arrive.expect_tx + the
//             relay from CTA 1; CTA 1: its producers + its B
//   empty[s]  one arrival in both CTAs from the MMA commit (multicast)
//   tfull     MMA commit (multicast) -> both epilogues
//   tempty    4 + 4 epilogue warps of both CTAs -> CTA 0's MMA thread
// CTA 1's warp 1 relays its full barriers to CTA 0 (after a proxy fence, so
// the MMA's async-proxy reads see its cp.async data).
template <int V, int KC, int MINB>
__global__ void __launch_bounds__(PAIR_THREADS, MINB)
    implicit_conv_pair_kernel(const __grid_constant__ CUtensorMap tmB,
                              const __grid_constant__ CUtensorMap tmOut,
                              const __grid_constant__ Params p) {
  constexpr int CPR = KC / 8;
  constexpr int IT = CPR;
  constexpr int SWZ = KC * 2;
  constexpr int RPI = NPROD / CPR;
  constexpr int MI = max_idx(MINB);
  constexpr int MAXO = MI / IT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_base = smem + (size_t)p.a_stages * p.a_stage_bytes;
  uint8_t* idx_base = epi_base + 4 * p.epi_bufs * EPI_BUF;     // [idx_slots][ops][128] int32
  uint64_t* full = (uint64_t*)(idx_base + (size_t)p.idx_slots * p.idx_slot_bytes);
  uint64_t* empty = full + p.a_stages;
  uint64_t* tfull = empty + p.a_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ifull = tempty + 2;
  uint64_t* iempty = ifull + p.idx_slots;
  uint32_t* tmem_slot = (uint32_t*)(iempty + p.idx_slots);
  const uint32_t b_region = (uint32_t)p.ops * p.a_off_bytes;   // B half after the A blocks

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileSeq ts = tile_seq(p);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.a_stages; ++s) {
      mbar_init(full + s, NPROD + 1 + (rank == 0 ? 1 : 0));
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);
    }
    for (int i = 0; i < p.idx_slots; ++i) {
      mbar_init(ifull + i, 1);        // the loader's arrive.expect_tx
      mbar_init(iempty + i, NPROD);   // every producer thread has read its indices
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmOut) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_before();
  cluster_sync_all();   // both CTAs' barriers initialised, TMEM allocated
  tc_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ============ B producer: this CTA's half of the stage's weight slices
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int nrow0 = (int)rank * (p.n_pad >> 1);
      GroupIter g;
      for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
        const int nv = __popc(g.mg);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          mbar_wait_sleep(empty + stage, phase ^ 1, 32);
          mbar_expect_tx(full + stage, nv * p.b_tx);
          uint8_t* sb = smem + (size_t)stage * p.a_stage_bytes + b_region;
          uint32_t x = g.mg;
          for (int o = 0; o < nv; ++o) {
            const int n = __ffs(x) - 1;
            x &= x - 1;
            tma_load_2d(sb + o * p.b_off_bytes, &tmB, full + stage, kk * p.kc, n * p.n_pad + nrow0);
          }
          if (++stage == p.a_stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 2 && warp < EPI0) {
    // ============ A producers (as the single-CTA kernel; rows of this CTA's
    // half).  A group's input rows come from the index ring (the loader warp
    // bulk-copies the group's hit-matrix rows several groups ahead), so no
    // producer waits on a dependent global load.
    const int pt = threadIdx.x - 64;
    const int cr = pt / CPR, cc = pt % CPR;
    uint32_t roff[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int r = it * RPI + cr;
      const int rxr = SWZ == 128 ? (r & 7) : (SWZ == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
      roff[it] = (uint32_t)(r * (KC * 2)) + ((uint32_t)(cc ^ rxr) << 4);
    }
    int cur[MI];
    const uint32_t ldfb1 = (uint32_t)(p.ldf * 2);
    const uint32_t ldfb2 = (uint32_t)(p.ldf2 * 2);
    int stage = 0, islot = 0;
    uint32_t phase = 0, iph = 0;
#ifdef SCB_IC_TRACE
    int nstage = 0;
#endif
    GroupIter g;
    for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
      const int nv = __popc(g.mg);
      const long long row0 = (long long)(2 * g.t + (int)rank) * BM;
      if (p.hits) {
        mbar_wait(ifull + islot, iph);
        const int* tab = reinterpret_cast<const int*>(idx_base + (size_t)islot * p.idx_slot_bytes);
#pragma unroll
        for (int o = 0; o < MAXO; ++o) {
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const int r = it * RPI + cr;
            cur[o * IT + it] = (o < nv && row0 + r < p.n_out) ? tab[o * BM + r] : -1;
          }
        }
        // the slot's next fill is an async-proxy (bulk copy) write: order this
        // thread's generic reads of it before that write (WAR across proxies)
        fence_async_smem();
        mbar_arrive(iempty + islot);
        if (++islot == p.idx_slots) { islot = 0; iph ^= 1; }
      } else {  // identity map (K = 1, s = 1)
#pragma unroll
        for (int o = 0; o < MAXO; ++o) {
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const long long k = row0 + it * RPI + cr;
            cur[o * IT + it] = (o < nv && k < p.n_out) ? (int)k : -1;
          }
        }
      }
      for (int kk = 0; kk < p.n_kchunks; ++kk) {
        mbar_wait(empty + stage, phase ^ 1);
        if (pt == 0) IC_TRACE(nstage, 0);
        const uint32_t dst = smem_u32(smem + (size_t)stage * p.a_stage_bytes);
        const int col0 = kk * KC;
        const int live = min(CPR, (p.c_in - col0) / 8);
        const int col = col0 + cc * 8;
        const bool second = p.feat2 != nullptr && col >= p.c_split;
        const uint64_t fb = second
            ? reinterpret_cast<uint64_t>(p.feat2) + (uint64_t)((col - p.c_split) * 2)
            : reinterpret_cast<uint64_t>(p.feat) + (uint64_t)(col * 2);
        const uint32_t ldb = second ? ldfb2 : ldfb1;
        const bool live_c = cc < live;
#pragma unroll
        for (int o = 0; o < MAXO; ++o) {
          if (o < nv) {
            const uint32_t blk = dst + o * p.a_off_bytes;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
              const int j = live_c ? cur[o * IT + it] : -1;
              const uint64_t src = fb + (uint64_t)(uint32_t)max(j, 0) * (uint64_t)ldb;
              asm volatile(
                  "{ .reg .pred q; setp.lt.s32 q, %2, 0;\n"
                  "  cp.async.cg.shared.global [%0], [%1], 16, q; }" ::"r"(blk + roff[it]),
                  "l"(src), "r"(j) : "memory");
            }
          }
        }
        cp_async_arrive_noinc(full + stage);
#ifdef SCB_IC_TRACE
        ++nstage;
#endif
        if (++stage == p.a_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == IDX_WARP) {
    // ============ index loader: each group's hit-matrix rows (this CTA's 128
    // rows of every active offset, contiguous in hits[n][.]) by bulk copy
    if (lane == 0 && p.hits) {
      int slot = 0;
      uint32_t ph = 0;
      GroupIter g;
      for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
        mbar_wait_sleep(iempty + slot, ph ^ 1, 20);
        const long long row0 = (long long)(2 * g.t + (int)rank) * BM;
        const long long avail = p.ldh - row0;   // entries of each hit row from row0 on
        const uint32_t bytes = avail <= 0 ? 0u : (uint32_t)((avail < BM ? avail : BM) * 4);
        if (bytes) {
          const int nv = __popc(g.mg);
          mbar_expect_tx(ifull + slot, (uint32_t)nv * bytes);
          const uint32_t dst = smem_u32(idx_base + (size_t)slot * p.idx_slot_bytes);
          uint32_t x = g.mg;
          for (int o = 0; o < nv; ++o) {
            const int n = __ffs(x) - 1;
            x &= x - 1;
            bulk_load(dst + o * BM * 4, p.hits + (long long)n * p.ldh + row0, bytes, ifull + slot);
          }
        } else {
          mbar_arrive(ifull + slot);
        }
        if (++slot == p.idx_slots) { slot = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank != 0) {
      // ============ relay (CTA 1): each filled stage -> CTA 0's full barrier
      if (lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        GroupIter g;
        for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
          for (int kk = 0; kk < p.n_kchunks; ++kk) {
            mbar_wait(full + stage, phase);
            fence_async_smem();   // this CTA's cp.async data -> the pair MMA (async proxy)
            mbar_arrive_cluster(mapa_shared(smem_u32(full + stage), 0));
            if (++stage == p.a_stages) { stage = 0; phase ^= 1; }
          }
        }
      }
    } else {
      // ============ MMA issuer of the pair (CTA 0), warp converged, one lane issues
      const uint32_t layout = p.swz == 128 ? 2u : (p.swz == 64 ? 4u : 6u);
      const uint32_t sbo = 8u * (uint32_t)p.swz;
      const uint64_t adesc_base = make_sdesc(smem_u32(smem), sbo, layout);
      const uint64_t bdesc_base = make_sdesc(smem_u32(smem) + b_region, sbo, layout);
      const uint32_t stage_d = p.a_stage_bytes >> 4;
      const uint32_t a_off_d = p.a_off_bytes >> 4, b_off_d = p.b_off_bytes >> 4;
      const uint32_t idesc = p.idesc;
      const uint32_t tmem0 = __shfl_sync(0xffffffffu, tmem_base, 0);
      int as = 0, acc = 0;
      uint32_t aph = 0, acc_phase = 0;
      uint32_t d = 0, acc0 = 0;
#ifdef SCB_IC_TRACE
      int nstage = 0;
#endif
      GroupIter g;
      for (g.start(p, ts); !g.done(ts); g.advance(p, ts)) {
        if (g.first) {
          mbar_wait_cluster(tempty + acc, acc_phase ^ 1);
          tc_after();
          d = tmem0 + (uint32_t)acc * (uint32_t)p.n_pad;
          acc0 = 0u;
        }
        const int nv = __popc(g.mg);
        for (int kk = 0; kk < p.n_kchunks; ++kk) {
          mbar_wait_cluster(full + as, aph);
          if (lane == 0) { IC_TRACE(nstage, 3); IC_TRACE(nstage, 1); }
          const uint64_t ad = adesc_base + (uint64_t)(as * stage_d);
          const uint64_t bd = bdesc_base + (uint64_t)(as * stage_d);
          if (elect_one()) {
            fence_async_smem();
            tc_after();
            IC_TRACE(nstage, 4);
#pragma unroll
            for (int o = 0; o < MAX_OPS; ++o) {
              if (o < nv) {
                const uint64_t a = ad + (uint64_t)(o * a_off_d);
                const uint64_t b = bd + (uint64_t)(o * b_off_d);
                mma_f16_pair(d, a, b, idesc, o ? 1u : acc0);
#pragma unroll
                for (int k = 1; k < KC / 16; ++k) mma_f16_pair(d, a + 2u * k, b + 2u * k, idesc, 1u);
              }
            }
            IC_TRACE(nstage, 5);
            mma_commit_pair(empty + as, (uint16_t)3);
          }
          __syncwarp();
          if (lane == 0) IC_TRACE(nstage, 2);
#ifdef SCB_IC_TRACE
          ++nstage;
#endif
          acc0 = 1u;
          if (++as == p.a_stages) { as = 0; aph ^= 1; }
        }
        if (g.last_of_tile()) {
          if (elect_one()) mma_commit_pair(tfull + acc, (uint16_t)3);
          __syncwarp();
          if (++acc == p.nacc) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else if (warp >= EPI0 && warp < EPI0 + 4) {
    epilogue_role(p, &tmOut, tmem_base, tfull, tempty, epi_base, warp, lane, ts, rank);
  }

  __syncwarp();
  tc_before();
  cluster_sync_all();   // no CTA leaves while the pair's MMAs / arrivals target it
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

// ------------------------------------------------------------------ tile masks
// bit n of masks[t] = some row of tile t has hits[n][row] >= 0.  One block
// per tile, one thread per row.
__global__ void __launch_bounds__(BM) tile_masks_kernel(const int* __restrict__ hits, long long ld,
                                                        int V, long long n_out,
                                                        uint32_t* __restrict__ masks) {
  __shared__ uint32_t acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  const long long k = (long long)blockIdx.x * BM + threadIdx.x;
  uint32_t m = 0;
  if (k < n_out)
    for (int n = 0; n < V; ++n) m |= (__ldg(hits + (long long)n * ld + k) >= 0 ? 1u : 0u) << n;
  m = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicOr(&acc, m);
  __syncthreads();
  if (threadIdx.x == 0) masks[blockIdx.x] = acc;
}

}  // namespace ic

// ------------------------------------------------------------------ host
bool encode_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                   long long inner, long long rows, long long ld, int box_inner, int box_rows,
                   int swz_bytes, std::string& err);
int device_sms();

namespace {

// Launch-invariant settings, read once per process.
struct IcEnv {
  int interleave, pdl, debug, pair, ring;
};
const IcEnv& ic_env() {
  static const IcEnv e = [] {
    auto env_int = [](const char* name, int dflt) {
      const char* v = getenv(name);
      return v ? atoi(v) : dflt;
    };
    return IcEnv{env_int("SCB_IC_INTERLEAVE", 1), env_int("SCB_IC_PDL", 0),
                 env_int("SCB_IC_DEBUG", 0), env_int("SCB_IC_PAIR", 0), env_int("SCB_IC_RING", 1)};
  }();
  return e;
}

// Tensor maps are a pure function of (address, shape, box, swizzle): cache
// them instead of re-encoding each launch (weights never move; activation
// buffers recur through the caching allocator).
struct MapKey {
  const void* base;
  long long inner, rows, ld;
  int box_inner, box_rows, swz;
  bool operator==(const MapKey& o) const {
    return base == o.base && inner == o.inner && rows == o.rows && ld == o.ld &&
           box_inner == o.box_inner && box_rows == o.box_rows && swz == o.swz;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.base);
    for (long long v : {k.inner, k.rows, k.ld, (long long)k.box_inner, (long long)k.box_rows, (long long)k.swz})
      h = h * 1000003u ^ std::hash<long long>()(v);
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

}  // namespace

// shared with the transposed scatter conv (upconv_sm100.cu)
bool cached_map_f16(CUtensorMap* out, const void* base, long long inner, long long rows, long long ld,
                    int box_inner, int box_rows, int swz, std::string& err) {
  const MapKey key{base, inner, rows, ld, box_inner, box_rows, swz};
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) {
    *out = it->second;
    return true;
  }
  if (!encode_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, inner, rows, ld, box_inner,
                     box_rows, swz, err))
    return false;
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps.emplace(key, *out);
  return true;
}

namespace {

// cudaFuncSetAttribute once per kernel instantiation (a driver call per
// launch otherwise).
std::mutex g_attr_mu;
std::unordered_map<const void*, int> g_attr_smem;

template <typename K>
int set_smem_once(K kernel, int bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& done = g_attr_smem[(const void*)kernel];
  if (done < bytes) {
    SCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = bytes;
  }
  return SCB_OK;
}

}  // namespace

}  // namespace scb

using namespace scb;

#ifdef SCB_IC_TRACE
// trace builds only (not part of the ABI): copy the stamp table to host
extern "C" int32_t scb_ic_trace_read(long long* host, int64_t n) {
  const int64_t cap = (int64_t)ic::TR_CTAS * ic::TR_STAGES * ic::TR_EV;
  SCB_CUDA(cudaMemcpyFromSymbol(host, ic::g_ic_trace, sizeof(long long) * (n < cap ? n : cap)));
  return SCB_OK;
}
extern "C" int32_t scb_ic_trace_clear() {
  static long long zero[ic::TR_CTAS * ic::TR_STAGES * ic::TR_EV];
  SCB_CUDA(cudaMemcpyToSymbol(ic::g_ic_trace, zero, sizeof(zero)));
  return SCB_OK;
}
#endif

extern "C" int32_t scb_tile_masks(const int32_t* hits, int32_t volume, int64_t n_out,
                                  uint32_t* masks, scb_stream_t stream) {
  SCB_CHECK_ARG(volume >= 1 && volume <= 32, "tile masks hold at most 32 offsets");
  SCB_CHECK_ARG(hits != nullptr && masks != nullptr, "hits and masks are required");
  if (n_out <= 0) return SCB_OK;
  const long long tiles = (n_out + ic::BM - 1) / ic::BM;
  ic::tile_masks_kernel<<<(unsigned)tiles, ic::BM, 0, as_stream(stream)>>>(hits, hits_ld(n_out),
                                                                          volume, n_out, masks);
  SCB_LAUNCHED();
  return SCB_OK;
}

namespace {

// The CTA-pair launch (implicit_conv_pair_kernel): arguments as
// scb_conv_implicit_rows (validated there); `ctas` 0 = auto, 1..2 pairs' CTAs per SM.
int32_t launch_pair(const void* features, int64_t ldf, int32_t c_split, const void* features2,
                    int64_t ldf2, int64_t n_in, int32_t c_in, const int32_t* hits, int32_t volume,
                    int64_t n_out, const uint32_t* tile_mask, const int32_t* out_rows,
                    const void* weights_packed, int32_t c_out, void* out, int64_t ldo,
                    const float* scale, const float* shift, const float* bias,
                    const void* residual, int32_t relu, int ctas, int32_t stage_kb,
                    scb_stream_t stream) {
  using namespace ic;
  const IcEnv& env = ic_env();
  const int n_pad = (c_out + 15) / 16 * 16;
  const int k_pad = (c_in + 15) / 16 * 16;
  Params p;
  memset(&p, 0, sizeof(p));
  p.pair = 1;
  p.debug = env.debug;
  p.n_out = n_out;
  p.n_in = (int)n_in;
  p.c_in = c_in;
  p.c_out = c_out;
  p.V = volume;
  p.all_bits = volume == 32 ? 0xffffffffu : ((1u << volume) - 1u);
  p.n_pad = n_pad;
  p.kc = (k_pad % 64 == 0) ? 64 : ((k_pad % 32 == 0) ? 32 : 16);
  p.swz = p.kc * 2;
  p.n_kchunks = k_pad / p.kc;
  p.epi_cols = (n_pad % 32 == 0) ? 32 : 16;
  p.relu = relu;
  p.interleave = 1;
  // M = 256 over the pair, N = n_pad (each CTA holds n_pad / 2 weight rows)
  p.idesc = (1u << 4) | ((uint32_t)(n_pad >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  p.nacc = 2;
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.nacc * n_pad)) cols *= 2;
  p.tmem_cols = cols;
  if (ctas <= 0) ctas = cols <= 256 ? 2 : 1;
  if (ctas >= 2 && cols > 256) ctas = 1;
  p.total_tiles = (int)((n_out + BM - 1) / BM);
  auto r1024 = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  p.b_tx = (uint32_t)((n_pad / 2) * p.kc * 2);
  p.a_off_bytes = r1024((uint32_t)(BM * p.kc * 2));
  p.b_off_bytes = r1024(p.b_tx);
  const uint32_t op_bytes = p.a_off_bytes + p.b_off_bytes;
  const int it_per_op = p.kc / 8;
  const int skb = stage_kb > 0 ? stage_kb : (ctas == 2 ? 36 : 64);
  int ops = (int)((uint32_t)skb * 1024u / op_bytes);
  ops = std::max(1, std::min(ops, std::min(std::min(MAX_OPS, volume), max_idx(ctas) / it_per_op)));
  p.ldf = ldf;
  p.ldh = hits_ld(n_out);
  p.feat = (const __half*)features;
  p.feat2 = (const __half*)features2;
  p.ldf2 = ldf2;
  p.c_split = features2 ? c_split : c_in;
  p.hits = hits;
  p.tmask = hits ? tile_mask : nullptr;
  p.scale = scale;
  p.shift = shift;
  p.bias = bias;
  p.residual = (const __half*)residual;
  p.orow = out_rows;
  p.ldo = ldo;
  p.out = (__half*)out;
  const int idx_slots = hits ? 8 : 0;
  auto fixed_bytes = [&](int epi_bufs) {
    return 1024 + 4 * epi_bufs * EPI_BUF + idx_slots * ops * BM * 4 + (40 + 2 * idx_slots) * 8 + 64;
  };
  const int smem_cap = ctas == 2 ? 113 * 1024 : 227 * 1024;
  int st = 0, epi_bufs = 1;
  for (;;) {
    const int sb = ops * (int)op_bytes;
    const int s1 = (smem_cap - fixed_bytes(1)) / sb, s2 = (smem_cap - fixed_bytes(2)) / sb;
    epi_bufs = s2 == s1 ? 2 : 1;
    st = std::min(epi_bufs == 2 ? s2 : s1, 16);
    if (st >= 2 || ops == 1) break;
    --ops;
  }
  SCB_CHECK_ARG(st >= 2, "pair stage does not fit in shared memory");
  p.ops = ops;
  p.idx_slots = idx_slots;
  p.idx_slot_bytes = (uint32_t)(ops * BM * 4);
  p.a_stages = st;
  p.b_stages = 0;
  p.epi_bufs = epi_bufs;
  p.a_stage_bytes = ops * op_bytes;
  p.b_stage_bytes = 0;
  const int smem = fixed_bytes(epi_bufs) + st * (int)p.a_stage_bytes;

  CUtensorMap mB, mO;
  std::string err;
  if (!cached_map_f16(&mB, weights_packed, k_pad, (long long)volume * n_pad, k_pad, p.kc,
                      n_pad / 2, p.swz, err) ||
      !cached_map_f16(&mO, out, c_out, n_out, ldo, p.epi_cols, 32, p.epi_cols * 2, err)) {
    set_error(std::string("scb_conv_implicit (pair): ") + err);
    return SCB_ECUDA;
  }
  const int pair_tiles = (p.total_tiles + 1) / 2;
  const int clusters = std::min(pair_tiles, ctas * device_sms() / 2);
  cudaStream_t s = as_stream(stream);
  auto launch = [&](auto kernel) -> int {
    const int rc = set_smem_once(kernel, smem_cap);
    if (rc != SCB_OK) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(PAIR_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = env.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    SCB_CUDA(cudaLaunchKernelEx(&cfg, kernel, mB, mO, p));
    return SCB_OK;
  };
  int rc = SCB_EINVAL;
#define SCB_PAIR_LAUNCH_C(VV, KK)                                              \
  rc = ctas == 2 ? launch(implicit_conv_pair_kernel<VV, KK, 2>)                \
                 : launch(implicit_conv_pair_kernel<VV, KK, 1>);
#define SCB_PAIR_LAUNCH_K(VV)                                                  \
  if (p.kc == 64) { SCB_PAIR_LAUNCH_C(VV, 64) }                                \
  else if (p.kc == 32) { SCB_PAIR_LAUNCH_C(VV, 32) }                           \
  else { SCB_PAIR_LAUNCH_C(VV, 16) }
  if (volume == 27) {
    SCB_PAIR_LAUNCH_K(27)
  } else if (volume == 8) {
    SCB_PAIR_LAUNCH_K(8)
  } else {
    SCB_PAIR_LAUNCH_K(1)
  }
#undef SCB_PAIR_LAUNCH_K
#undef SCB_PAIR_LAUNCH_C
  if (rc != SCB_OK) return rc;
  SCB_LAUNCHED();
  return SCB_OK;
}

}  // namespace

extern "C" int32_t scb_conv_implicit_rows(const void* features, int64_t ldf, int32_t c_split,
                                          const void* features2, int64_t ldf2, int64_t n_in,
                                          int32_t c_in, const int32_t* hits, int32_t volume,
                                          int64_t n_out, const uint32_t* tile_mask,
                                          const int32_t* out_rows, const void* weights_packed,
                                          int32_t c_out, void* out, int64_t ldo, const float* scale,
                                          const float* shift, const float* bias,
                                          const void* residual, int32_t relu, int32_t ctas_per_sm,
                                          int32_t stage_kb, scb_stream_t stream) {
  using namespace ic;
  SCB_CHECK_ARG(out_rows == nullptr || hits != nullptr, "permuted output rows need a hit matrix");
  SCB_CHECK_ARG(ctas_per_sm >= 0 && ctas_per_sm <= 5,
                "ctas_per_sm must be 0 (auto), 1..3 (single-CTA kernel) or 4..5 (CTA pairs, 1..2 per SM)");
  SCB_CHECK_ARG(stage_kb == 0 || (stage_kb >= 8 && stage_kb <= 200),
                "stage_kb must be 0 (auto) or 8..200");
  SCB_CHECK_ARG(features2 == nullptr || (c_split % 8 == 0 && c_split > 0 && c_split < c_in &&
                                         ldf2 % 8 == 0 && ldf2 * 2 < (1LL << 32)),
                "concat split must be a positive multiple of 8 inside C_in, second stride % 8");
  SCB_CHECK_ARG(volume == 1 || volume == 8 || volume == 27,
                "implicit conv supports K^3 = 1, 8 or 27 offsets");
  SCB_CHECK_ARG(volume == 1 || hits != nullptr, "hit matrix required for K > 1");
  SCB_CHECK_ARG(hits != nullptr || n_in == n_out, "identity map (no hit matrix) needs n_in == n_out");
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
  const IcEnv& env = ic_env();
  if (ctas_per_sm >= 4 || (ctas_per_sm == 0 && env.pair))
    return launch_pair(features, ldf, c_split, features2, ldf2, n_in, c_in, hits, volume, n_out,
                       tile_mask, out_rows, weights_packed, c_out, out, ldo, scale, shift, bias,
                       residual, relu, ctas_per_sm >= 4 ? ctas_per_sm - 3 : 0, stage_kb, stream);
  Params p;
  memset(&p, 0, sizeof(p));
  p.n_out = n_out;
  p.n_in = (int)n_in;
  p.c_in = c_in;
  p.c_out = c_out;
  p.V = volume;
  p.all_bits = volume == 32 ? 0xffffffffu : ((1u << volume) - 1u);
  p.n_pad = n_pad;
  p.kc = (k_pad % 64 == 0) ? 64 : ((k_pad % 32 == 0) ? 32 : 16);
  p.swz = p.kc * 2;
  p.n_kchunks = k_pad / p.kc;
  p.epi_cols = (n_pad % 32 == 0) ? 32 : 16;
  p.relu = relu;
  p.interleave = env.interleave ? 1 : 0;
  p.debug = env.debug;
  p.idesc = (1u << 4) | ((uint32_t)(n_pad >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  // Two accumulators per CTA (the epilogue of tile i overlaps tile i+1).
  p.nacc = 2;
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.nacc * n_pad)) cols *= 2;
  p.tmem_cols = cols;
  // CTAs per SM: one for k3 gathering layers with 64-wide K chunks (deep A
  // ring; measured 5-15 % faster per layer than two or three since the index
  // ring removed the index-load stalls), two whenever both accumulator pairs
  // fit, else one (three for K = 1 / k2 layers measured the same in the
  // whole step).
  int ctas = (p.kc == 64 && hits && volume == 27) ? 1 : (cols <= 256 ? 2 : 1);
  if (ctas_per_sm > 0)  // tuned (autotune.tune_fused_layer): clamped to what TMEM allows
    ctas = (ctas_per_sm >= 3 && cols <= 128) ? 3 : (ctas_per_sm >= 2 && cols <= 256 ? 2 : 1);
  p.total_tiles = (int)((n_out + BM - 1) / BM);
  auto r1024 = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  p.b_tx = (uint32_t)(n_pad * p.kc * 2);
  p.a_off_bytes = r1024((uint32_t)(BM * p.kc * 2));
  p.b_off_bytes = r1024(p.b_tx);
  const uint32_t op_bytes = p.a_off_bytes + p.b_off_bytes;
  const int skb = stage_kb > 0 ? stage_kb : (ctas == 3 ? 24 : (ctas == 2 ? 42 : 96));
  const int it_per_op = p.kc / 8;  // index registers one offset needs per producer thread
  int ops = (int)((uint32_t)skb * 1024u / op_bytes);
  auto clamp_ops = [&]() {
    ops = std::max(1, std::min(ops, std::min(std::min(MAX_OPS, volume),
                                             max_idx(ctas) / it_per_op)));
  };
  clamp_ops();
  p.ldf = ldf;
  p.ldh = hits_ld(n_out);
  p.feat = (const __half*)features;
  p.feat2 = (const __half*)features2;
  p.ldf2 = ldf2;
  p.c_split = features2 ? c_split : c_in;
  p.hits = hits;
  p.tmask = hits ? tile_mask : nullptr;
  p.scale = scale;
  p.shift = shift;
  p.bias = bias;
  p.residual = (const __half*)residual;
  p.orow = out_rows;
  p.ldo = ldo;
  p.out = (__half*)out;
  // shared memory: the A ring (gathered rows) and the B ring (weights) with
  // their own depths -- the A ring as deep as the CTA's share allows (the
  // gather latency is what it hides), the B ring 3 deep (L2-resident weights
  // by TMA) -- + epilogue staging + barriers.
  // the index ring: 8 group slots (4 at three CTAs per SM), ops x 512 B each
  // (not for one-hot maps: one offset per tile, so a ring round trip per
  // tile costs more than the one-group-ahead register prefetch saves)
  auto idx_slots_for = [&]() { return (hits && !out_rows && env.ring) ? (ctas >= 3 ? 4 : 8) : 0; };
  auto fixed_bytes = [&](int epi_bufs) {
    return 1024 + 4 * epi_bufs * EPI_BUF + idx_slots_for() * ops * BM * 4 +
           (52 + 2 * idx_slots_for()) * 8 + 64;
  };
  int smem_cap = ctas == 3 ? 75 * 1024 : (ctas == 2 ? 113 * 1024 : 227 * 1024);
  int a_st = 0, b_st = 0, epi_bufs = 1;
  auto plan = [&]() -> bool {
    const int a_bytes = ops * (int)p.a_off_bytes, b_bytes = ops * (int)p.b_off_bytes;
    for (int bs = 3; bs >= 2; --bs) {
      for (int eb = 2; eb >= 1; --eb) {
        const int as = (smem_cap - fixed_bytes(eb) - bs * b_bytes) / a_bytes;
        // a second epilogue buffer only when it costs no A stage
        if (eb == 2 && as < (smem_cap - fixed_bytes(1) - bs * b_bytes) / a_bytes) continue;
        if (as >= std::max(2, bs)) {
          a_st = std::min(as, 16);
          b_st = bs;
          epi_bufs = eb;
          return true;
        }
      }
    }
    return false;
  };
  while (!plan()) {  // fewer offsets per stage, then fewer CTAs per SM
    if (ops > 1) {
      --ops;
    } else if (ctas > 1) {
      --ctas;
      smem_cap = ctas == 2 ? 113 * 1024 : 227 * 1024;
      clamp_ops();
    } else {
      SCB_CHECK_ARG(false, "stage does not fit in shared memory");
    }
  }
  p.ops = ops;
  p.idx_slots = idx_slots_for();
  p.idx_slot_bytes = (uint32_t)(ops * BM * 4);
  p.a_stages = a_st;
  p.b_stages = b_st;
  p.epi_bufs = epi_bufs;
  p.a_stage_bytes = ops * p.a_off_bytes;
  p.b_stage_bytes = ops * p.b_off_bytes;
  const int smem = fixed_bytes(epi_bufs) + a_st * (int)p.a_stage_bytes + b_st * (int)p.b_stage_bytes;

  CUtensorMap mB, mO;
  std::string err;
  if (!cached_map_f16(&mB, weights_packed, k_pad, (long long)volume * n_pad, k_pad, p.kc, n_pad,
                      p.swz, err) ||
      !cached_map_f16(&mO, out, c_out, n_out, ldo, p.epi_cols, 32, p.epi_cols * 2, err)) {
    set_error(std::string("scb_conv_implicit: ") + err);
    return SCB_ECUDA;
  }
  const int grid = p.total_tiles < ctas * device_sms() ? p.total_tiles : ctas * device_sms();
  cudaStream_t s = as_stream(stream);
  auto launch = [&](auto kernel) -> int {
    const int rc = set_smem_once(kernel, smem_cap);
    if (rc != SCB_OK) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(IC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = env.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SCB_CUDA(cudaLaunchKernelEx(&cfg, kernel, mB, mO, p));
    return SCB_OK;
  };
  int rc = SCB_EINVAL;
#define SCB_IC_LAUNCH_C(VV, KK)                                              \
  rc = ctas == 3 ? launch(implicit_conv_f16_kernel<VV, KK, 3>)               \
     : ctas == 2 ? launch(implicit_conv_f16_kernel<VV, KK, 2>)               \
                 : launch(implicit_conv_f16_kernel<VV, KK, 1>);
#define SCB_IC_LAUNCH_K(VV)                                                  \
  if (p.kc == 64) { SCB_IC_LAUNCH_C(VV, 64) }                                \
  else if (p.kc == 32) { SCB_IC_LAUNCH_C(VV, 32) }                           \
  else { SCB_IC_LAUNCH_C(VV, 16) }
  if (volume == 27) {
    SCB_IC_LAUNCH_K(27)
  } else if (volume == 8) {
    SCB_IC_LAUNCH_K(8)
  } else {
    SCB_IC_LAUNCH_K(1)
  }
#undef SCB_IC_LAUNCH_K
#undef SCB_IC_LAUNCH_C
  if (rc != SCB_OK) return rc;
  SCB_LAUNCHED();
  return SCB_OK;
}

extern "C" int32_t scb_conv_implicit_tuned(const void* features, int64_t ldf, int32_t c_split,
                                           const void* features2, int64_t ldf2, int64_t n_in,
                                           int32_t c_in, const int32_t* hits, int32_t volume,
                                           int64_t n_out, const uint32_t* tile_mask,
                                           const void* weights_packed, int32_t c_out, void* out,
                                           int64_t ldo, const float* scale, const float* shift,
                                           const float* bias, const void* residual,
                                           int32_t relu, int32_t ctas_per_sm, int32_t stage_kb,
                                           scb_stream_t stream) {
  return scb_conv_implicit_rows(features, ldf, c_split, features2, ldf2, n_in, c_in, hits, volume,
                                n_out, tile_mask, nullptr, weights_packed, c_out, out, ldo, scale,
                                shift, bias, residual, relu, ctas_per_sm, stage_kb, stream);
}

extern "C" int32_t scb_conv_implicit_cat(const void* features, int64_t ldf, int32_t c_split,
                                         const void* features2, int64_t ldf2, int64_t n_in,
                                         int32_t c_in, const int32_t* hits, int32_t volume,
                                         int64_t n_out, const uint32_t* tile_mask,
                                         const void* weights_packed, int32_t c_out, void* out,
                                         int64_t ldo, const float* scale, const float* shift,
                                         const float* bias, const void* residual, int32_t relu,
                                         scb_stream_t stream) {
  return scb_conv_implicit_tuned(features, ldf, c_split, features2, ldf2, n_in, c_in, hits,
                                 volume, n_out, tile_mask, weights_packed, c_out, out, ldo, scale,
                                 shift, bias, residual, relu, 0, 0, stream);
}

extern "C" int32_t scb_conv_implicit(const void* features, int64_t n_in, int32_t c_in,
                                     int64_t ldf, const int32_t* hits, int32_t volume,
                                     int64_t n_out, const void* weights_packed, int32_t c_out,
                                     void* out, const float* scale, const float* shift,
                                     const float* bias, const void* residual, int32_t relu,
                                     scb_stream_t stream) {
  return scb_conv_implicit_cat(features, ldf, c_in, nullptr, 0, n_in, c_in, hits, volume, n_out,
                               nullptr, weights_packed, c_out, out, c_out, scale, shift, bias,
                               residual, relu, stream);
}
