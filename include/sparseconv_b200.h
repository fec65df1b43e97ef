/*
 * sparseconv_b200.h — C ABI of the B200-native sparse-convolution engine.
 *
 * The reference (arxiv 2204.10319 CPU package `sparseconv`, read-only at
 * /root/reference/pkg/src/sparseconv) is pure Python: its operator API is a
 * set of numpy functions, so the "FFI" a maintainer would bind is exactly the
 * list below, one entry point per reference function on the hot path
 * (SURVEY.md §8(a)/(b)).  Each declaration cites the reference symbol it
 * replaces as file:line relative to pkg/src/sparseconv/.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers owned and allocated by the caller
 *    (torch tensors passed as raw addresses in the Python binding).  Nothing
 *    is allocated or freed across the ABI; scratch space is a caller-provided
 *    workspace whose size is queried first (…_workspace()).
 *  - Work is enqueued on the caller's stream (`scb_stream_t` = cudaStream_t)
 *    and is asynchronous unless stated otherwise.
 *  - Coordinates are int32 rows (batch, x1..xD), D = 1..4 (core.py:90,106-107).
 *  - Every function returns SCB_OK (0) or an error code; scb_last_error()
 *    returns a thread-local message (the Python layer re-raises it as the
 *    matching ValueError / KeyError of the reference).
 *  - Numerics: kernel maps, output coordinates, plans and gathers are
 *    bit-exact w.r.t. the reference; GEMM/scatter are f32-accumulated.
 */
#ifndef SPARSECONV_B200_H
#define SPARSECONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* scb_stream_t; /* cudaStream_t */

enum scb_status { SCB_OK = 0, SCB_EINVAL = 1, SCB_ECUDA = 2, SCB_EUNSUPPORTED = 3 };
enum scb_dtype { SCB_F32 = 0, SCB_F16 = 1 };
enum scb_index_kind { SCB_INDEX_HASH = 0, SCB_INDEX_GRID = 1 };

/* Geometry of one coordinate set: spatial rank, batch count and boundary.
 * Mirrors SparseTensor.{boundary,batch_size} (core.py:90-94). */
typedef struct {
  int32_t dim;        /* spatial rank D, 1..4 */
  int32_t _pad;
  int64_t batch_size; /* batch column is in [0, batch_size) */
  int64_t extent[4];  /* boundary per spatial dim */
} scb_grid_t;

/* One GEMM problem of the grouped contraction: `rows` buffer rows starting at
 * `a_row` (of the gather buffer when a_src == 0, of the feature matrix when
 * a_src == 1 — the centre offset) times weight slice `b_index`, written to
 * partial rows starting at `c_row`. */
typedef struct {
  int64_t a_row;
  int64_t c_row;
  int32_t rows;
  int32_t b_index;
  int32_t a_src;
  int32_t _pad;
} scb_segment_t;

#define SCB_MAX_SEGMENTS 128
#define SCB_TILE_ROWS 128 /* buffer slabs are padded to this many rows */

const char* scb_last_error(void);
int32_t scb_abi_version(void);
/* Number of SMs of the current device (for grid sizing in the host layer). */
int32_t scb_device_sm_count(void);
/* Kernels this library has launched in this process (CUB sort passes inside
 * scb_output_coords excluded). */
int64_t scb_launch_count(void);

/* ---------------------------------------------------------------- index
 * Replaces HashIndex (mapping.py:122-189), GridIndex (mapping.py:82-119) and
 * build_index (mapping.py:195-208).  Hash: open addressing, linear probing,
 * table = next pow2 >= 2N slots (load <= 0.5) of 64-bit keys + int32 rows.
 * Grid: dense int32 table over batch x boundary.
 * `status` (device, 2 x int32, zeroed by this call) receives the number of
 * duplicate keys and out-of-bounds rows found while building — the
 * SparseTensor validation of core.py:112-120. */
int64_t scb_hash_slots(int64_t n);
int32_t scb_index_build(int32_t kind, const int32_t* coords, int64_t n, const scb_grid_t* grid,
                        int64_t* table_keys, int32_t* table_rows, int64_t slots,
                        int32_t* status, scb_stream_t stream);
/* HashIndex.query / GridIndex.query: row per probe, -1 (MISS) when absent or
 * out of bounds (mapping.py:106-119, 166-189). */
int32_t scb_index_query(int32_t kind, const int32_t* probes, int64_t n, const scb_grid_t* grid,
                        const int64_t* table_keys, const int32_t* table_rows, int64_t slots,
                        int32_t* rows_out, scb_stream_t stream);

/* ---------------------------------------------------------------- output coordinates
 * Replaces compute_output_coords (mapping.py:216-248) for stride > 1: fused
 * candidate generation (offset subtraction, modular and boundary checks, key
 * flattening) then radix sort + unique on 64-bit keys, so the result is in
 * ascending flat-key order.  `offset_base` is the lowest per-dimension offset
 * of the window (-(K-1)/2 for odd K, 0 for even K: mapping.py:63-79 and its
 * EVEN_KERNEL_OFFSET_BASE hook, mapping.py:26).  `out_keys` needs room for
 * scb_output_coords_capacity() keys; `n_out` (device int64) receives the
 * count.  scb_unflatten turns keys back into coordinate rows. */
int64_t scb_output_coords_capacity(int64_t n_in, int32_t dim, int32_t kernel_size, int32_t stride);
int64_t scb_output_coords_workspace(int64_t n_in, int32_t dim, int32_t kernel_size, int32_t stride);
int32_t scb_output_coords(const int32_t* in_coords, int64_t n_in, const scb_grid_t* out_grid,
                          int32_t kernel_size, int32_t offset_base, int32_t stride,
                          void* workspace, int64_t ws_bytes, int64_t* out_keys, int64_t* n_out,
                          scb_stream_t stream);
/* The next strided level straight from the previous level's output keys
 * (grid `in_grid`), whose count stays on the device (`n_in_dev`, at most
 * `n_cap`): a chain of strided levels costs one host read instead of one per
 * level.  Same output as scb_output_coords on the unflattened coordinates. */
int32_t scb_output_keys_next(const int64_t* in_keys, const int64_t* n_in_dev, int64_t n_cap,
                             const scb_grid_t* in_grid, const scb_grid_t* out_grid,
                             int32_t kernel_size, int32_t offset_base, int32_t stride,
                             void* workspace, int64_t ws_bytes, int64_t* out_keys, int64_t* n_out,
                             scb_stream_t stream);
int32_t scb_unflatten(const int64_t* keys, int64_t n, const scb_grid_t* grid, int32_t* coords,
                      scb_stream_t stream);

/* ---------------------------------------------------------------- kernel map
 * Replaces map_search (mapping.py:289-319) and derive_symmetric_maps
 * (mapping.py:322-339).  One pass over outputs x searched offsets writes the
 * hit matrix hits[V][n_out] (input row or -1).  With `symmetric` (stride 1,
 * odd K) only offsets 0..centre are probed and the mirror entry
 * hits[V-1-n][j] = k is filled directly, which is exactly the order the
 * reference's stable re-sort produces.
 * Every hit matrix over n rows has row stride scb_hits_ld(n) = roundup(n, 4)
 * (16-byte aligned rows); allocate V * scb_hits_ld(n) int32. */
int64_t scb_hits_ld(int64_t n);
int32_t scb_map_search(int32_t kind, const int32_t* out_coords, int64_t n_out,
                       const scb_grid_t* in_grid, int32_t kernel_size, int32_t offset_base,
                       int32_t stride, int32_t symmetric, const int64_t* table_keys, const int32_t* table_rows,
                       int64_t slots, int32_t* hits, scb_stream_t stream);

/* scb_map_search over a dilated window (B200 extension; the reference has no
 * dilation, north_star's SparseConv3d has): entry (j, k) whenever
 * stride*q_k + dilation*delta_n is input j.  dilation = 1 is scb_map_search;
 * symmetric probing is valid for stride 1 and odd K at any dilation. */
int32_t scb_map_search_dilated(int32_t kind, const int32_t* out_coords, int64_t n_out,
                               const scb_grid_t* in_grid, int32_t kernel_size,
                               int32_t offset_base, int32_t stride, int32_t dilation,
                               int32_t symmetric, const int64_t* table_keys,
                               const int32_t* table_rows, int64_t slots, int32_t* hits,
                               scb_stream_t stream);
/* Per-offset compaction of a hit matrix into the canonical CSR map
 * (offset_ptr[V+1] int64, in_idx/out_idx int32, entries of each offset sorted
 * by output row).  Two phases so the caller can size in_idx/out_idx:
 * scb_map_count fills offset_ptr (device) — read offset_ptr[V] after a sync —
 * then scb_map_compact writes the entries. */
int64_t scb_map_workspace(int32_t volume, int64_t n_out);
int32_t scb_map_count(const int32_t* hits, int32_t volume, int64_t n_out, void* workspace,
                      int64_t* offset_ptr, scb_stream_t stream);
int32_t scb_map_compact(const int32_t* hits, int32_t volume, int64_t n_out, const void* workspace,
                        const int64_t* offset_ptr, int32_t* in_idx, int32_t* out_idx,
                        scb_stream_t stream);
/* KernelMap.swap_roles (mapping.py:277-286): scatter a CSR map into the hit
 * matrix of the transposed map, hits_t[V][n_in]; compact it with the two
 * calls above. */
int32_t scb_map_transpose(const int64_t* offset_ptr, const int32_t* in_idx, const int32_t* out_idx,
                          int32_t volume, int64_t total, int64_t n_in, int32_t* hits_t,
                          scb_stream_t stream);
/* Same transposition straight from a hit matrix: hits_t[n][hits[n][k]] = k
 * (no compaction, no host sync; used by the fused dataflow). */
int32_t scb_hits_transpose(const int32_t* hits, int32_t volume, int64_t n_out, int64_t n_in,
                           int32_t* hits_t, scb_stream_t stream);

/* ---------------------------------------------------------------- plan
 * Replaces build_gather_scatter_plan (mapping.py:377-418).  The B200 buffer
 * keeps the reference's offset-major order but starts every offset's slice
 * on a SCB_TILE_ROWS boundary so GEMM tiles never straddle offsets:
 * slab_ptr[n] = sum_{m<n, m != skip} roundup(|M_m|, tile).  Outputs:
 * buf_in[rows_pad] (input row per buffer row, -1 on padding rows) and
 * pos[n_out][V] (buffer row per (output, offset), -1 when absent) — the
 * output-stationary CSR of the reference in fixed-width form.  `skip_offset`
 * is the centre offset on stride-1 odd-K layers, else -1.  When `status`
 * (device int32, nullable) is given, entries that repeat an (output, offset)
 * pair — impossible for a searched map, possible for a hand-built one — are
 * counted there instead of silently overwriting. */
int32_t scb_plan_build(const int64_t* offset_ptr, const int32_t* in_idx, const int32_t* out_idx,
                       int32_t volume, int64_t total, int64_t n_out, int32_t skip_offset,
                       int32_t tile_rows, int32_t* buf_in, int64_t rows_pad, int32_t* pos,
                       int32_t* status, scb_stream_t stream);

/* Sync-free plan: the same layout built straight from a hit matrix on the
 * device (count + scan + placement), so the staged layer never reads map
 * sizes on the host.  Also writes the layer's GEMM problem table (`table`,
 * scb_segtable_bytes(); consumed by scb_grouped_gemm_table) with an optional
 * centre segment (a_src = 1, rows = center_rows, weight center_seg) placed at
 * partial rows [0, c_base); offset slabs go to partial rows slab + c_base.
 * `gemm_bm`/`gemm_ntn` are the GEMM's tile height and column tiles.
 * buf_in needs scb_plan_rows_cap() entries, workspace scb_map_workspace(). */
int64_t scb_plan_rows_cap(int32_t volume, int64_t n_out, int32_t tile_rows);
int64_t scb_segtable_bytes(void);
int32_t scb_plan_from_hits(const int32_t* hits, int32_t volume, int64_t n_out,
                           int32_t skip_offset, int32_t tile_rows, int64_t c_base,
                           int32_t gemm_bm, int32_t gemm_ntn, int32_t center_seg,
                           int64_t center_rows, void* workspace, int64_t* offset_ptr,
                           int32_t* buf_in, int32_t* pos, void* table, scb_stream_t stream);

/* ---------------------------------------------------------------- movement
 * gather (execution.py:159-180, kernels.py:28-35): buffer[r] =
 * features[buf_in[r]] (zero row when buf_in[r] < 0), 128-bit vector copies,
 * bit-exact.  `ld_*` are row strides in elements.  With `rows_dev`
 * (nullable, device int64 — a device-built SegTable's rows_pad) only
 * min(rows, *rows_dev) rows are moved; `rows` is then the capacity. */
int32_t scb_gather(int32_t dtype, const void* features, int64_t n_in, int32_t channels,
                   int64_t ld_feat, const int32_t* buf_in, int64_t rows, void* buffer,
                   int64_t ld_buf, const int64_t* rows_dev, scb_stream_t stream);
/* scatter_accumulate, output-stationary (execution.py:183-218,
 * kernels.py:38-50) fused with the centre-offset add (execution.py:423-428)
 * and an optional pointwise epilogue (execution.py:554-576):
 *   acc = sum_{n ascending} partial[pos[k][n]]   (f32, one write per row)
 *   acc += partial[center_row + k]               (if center_row >= 0)
 *   acc = acc * scale + shift (if scale), + bias (if bias),
 *         + residual[k] (if residual: out_dtype, same shape/stride as out),
 *         max(0,.) if relu
 *   out[k] = (out_dtype) acc */
int32_t scb_scatter(const float* partial, int64_t ldp, const int32_t* pos, int32_t volume,
                    int64_t n_out, int32_t c_out, int64_t center_row, int32_t out_dtype, void* out,
                    int64_t ld_out, const float* scale, const float* shift, const float* bias,
                    const void* residual, int32_t relu, scb_stream_t stream);
/* scatter_accumulate for ANY plan (execution.py:183-218, kernels.py:38-50):
 * out[k] = sum over e in [out_ptr[k], out_ptr[k+1]) of buffer[out_rows[e]],
 * folded in that order in f32, one write per row.  Buffer in the reference's
 * compact layout (`plan.total` rows, stride ldb).  Used where a hand-built
 * map has several entries per (output, offset) pair, which scb_scatter's
 * fixed-width position table cannot hold. */
int32_t scb_scatter_csr(int32_t in_dtype, const void* buffer, int64_t ldb, const int64_t* out_ptr,
                        const int32_t* out_rows, int64_t n_out, int32_t channels,
                        int32_t out_dtype, void* out, int64_t ld_out, scb_stream_t stream);
/* Small device -> pinned-host read (counts, status words) written by the SMs
 * through the pinned buffer's host pointer (UVA-mapped) on `stream`, so it
 * never waits behind a large DMA transfer on the copy engine; visible to
 * the host once an event recorded after it completes.  bytes % 4 == 0,
 * <= 1 MiB.  B200 plumbing (the reference reads numpy values directly). */
int32_t scb_store_to_host(const void* src, void* host_dst, int64_t bytes, scb_stream_t stream);
/* pointwise_apply (execution.py:554-576) on a feature matrix in place:
 * op 0 = relu, 1 = bias_add, 2 = bn_fold (scale, shift).  f32 compute, cast
 * back to the storage dtype. */
int32_t scb_pointwise(int32_t dtype, void* features, int64_t n, int32_t channels, int32_t op,
                      const float* a, const float* b, scb_stream_t stream);
/* Residual glue for the MinkUNet workload (not a reference layer kind):
 * out = relu?(x + y), same shape/dtype. */
int32_t scb_add(int32_t dtype, const void* x, const void* y, void* out, int64_t count, int32_t relu,
                scb_stream_t stream);
/* quantize_features FP16 path (core.py:219-238): f32 -> f16 RNE with
 * saturation to +-65504; `n_saturated` (device int64) counts clamps. */
int32_t scb_quantize_f16(const float* in, void* out, int64_t count, int64_t* n_saturated,
                         scb_stream_t stream);

/* ---------------------------------------------------------------- grouped GEMM
 * execute_groups (execution.py:331-368) + the centre matmul
 * (execution.py:423-424) as ONE persistent launch over a tile table built
 * from `segments` (one per scheduled offset / group member).
 *  - F16 (FP16-storage path): tcgen05.mma kind::f16, A/B staged by TMA,
 *    f32 accumulators in TMEM, TMA-stored f32 partials.  Weights must be
 *    packed by scb_pack_weights_f16 into [V][n_pad][k_pad] (K-major, zero
 *    padded; n_pad = roundup(c_out,16), k_pad = roundup(c_in,16)).
 *  - F32 (FP32 path): exact-f32 SIMT FMA (TF32 would miss the 1e-4 target,
 *    SURVEY.md §7.3 item 5); weights are the reference's [V][c_in][c_out] f32.
 * `a_buffer` has `a_rows` rows of stride `lda`; `a_features` (centre) has
 * `f_rows` rows of stride `ldf`.  Partials: `c_rows` rows of stride `ldc`
 * (ldc = n_pad for F16, c_out for F32). */
int32_t scb_pack_weights_f16(const float* w, int32_t volume, int32_t c_in, int32_t c_out,
                             void* packed, int32_t k_pad, int32_t n_pad, scb_stream_t stream);
int32_t scb_grouped_gemm(int32_t dtype, const void* a_buffer, int64_t a_rows, int64_t lda,
                         const void* a_features, int64_t f_rows, int64_t ldf, int32_t c_in,
                         const void* weights, int32_t volume, int32_t c_out, float* partial,
                         int64_t c_rows, int64_t ldc, const scb_segment_t* segments,
                         int32_t n_segments, scb_stream_t stream);
/* Same GEMM driven by a device-built problem table (scb_plan_from_hits):
 * a_rows / c_rows are capacities, the kernel reads the segments and tile
 * count from `table`, one persistent CTA per SM.  No host sync anywhere. */
int32_t scb_grouped_gemm_table(int32_t dtype, const void* a_buffer, int64_t a_rows, int64_t lda,
                               const void* a_features, int64_t f_rows, int64_t ldf, int32_t c_in,
                               const void* weights, int32_t volume, int32_t c_out, float* partial,
                               int64_t c_rows, int64_t ldc, const void* table,
                               scb_stream_t stream);
/* Tile height and column-tile count the GEMM of `dtype` uses (for
 * scb_plan_from_hits' gemm_bm / gemm_ntn). */
int32_t scb_gemm_tile_geometry(int32_t dtype, int32_t c_out, int32_t* bm, int32_t* ntn);

/* ---------------------------------------------------------------- fused dataflow
 * gather -> GEMM -> scatter of one layer (the whole of _run_dataflow,
 * execution.py:409-429, plus the pointwise epilogue) as ONE output-stationary
 * tcgen05 kernel ("implicit GEMM"):
 *   out[k] = epi( sum_n features[hits[n][k]] . W[n] ),  absent neighbours = 0,
 * with epi = *scale + shift, + bias, + residual[k], ReLU (each optional).
 * `hits` is the [V][n_out] hit matrix of scb_map_search / scb_map_transpose,
 * so no compaction, plan, gather buffer or partials are needed.  V = 1 is the
 * K=1 pointwise layer (execution.py:472-477): `hits` may be NULL (identity
 * map, n_in == n_out).  FP16 storage only; V in {1, 8, 27}; c_in, c_out
 * multiples of 8 (callers zero-pad narrower inputs); weights packed by
 * scb_pack_weights_f16.  Per-output accumulation runs over the offsets in
 * ascending order inside the tensor core (f32). */
int32_t scb_conv_implicit(const void* features, int64_t n_in, int32_t c_in, int64_t ldf,
                          const int32_t* hits, int32_t volume, int64_t n_out,
                          const void* weights_packed, int32_t c_out, void* out,
                          const float* scale, const float* shift, const float* bias,
                          const void* residual, int32_t relu, scb_stream_t stream);

/* scb_conv_implicit with the input split channel-wise over two row-aligned
 * matrices: channels [0, c_split) from `features` (row stride ldf), [c_split,
 * c_in) from `features2` (row stride ldf2) — the skip concatenation of a
 * U-Net decoder without materialising it.  `features2` NULL = scb_conv_implicit.
 * `hits` may be NULL only for the identity map (K = 1, s = 1, n_in == n_out);
 * a K = 1 strided map (volume 1) passes its hit matrix.
 * `tile_mask` (nullable): [ceil(n_out / 128)] words from scb_tile_masks —
 * offsets whose bit is clear in a 128-row tile's word are skipped for that
 * tile (no weight load, no copies, no MMA); NULL = every offset.
 * `ldo`: output row stride in elements (multiple of 8, >= c_out), so C_out
 * need not be a multiple of 8 (e.g. a 19-class head into 24-wide rows). */
int32_t scb_conv_implicit_cat(const void* features, int64_t ldf, int32_t c_split,
                              const void* features2, int64_t ldf2, int64_t n_in, int32_t c_in,
                              const int32_t* hits, int32_t volume, int64_t n_out,
                              const uint32_t* tile_mask, const void* weights_packed,
                              int32_t c_out, void* out, int64_t ldo, const float* scale,
                              const float* shift, const float* bias, const void* residual,
                              int32_t relu, scb_stream_t stream);
/* scb_conv_implicit_cat with the launch shape chosen by the caller (the
 * strategy files of autotune.tune_fused_layer): `ctas_per_sm` 1..3 co-resident
 * CTAs per SM (clamped to what TMEM allows; 0 = auto) and `stage_kb` the
 * target pipeline-stage size in KB, which sets the kernel offsets per stage
 * (0 = auto); `ctas_per_sm` 4..5 runs the CTA-pair kernel (tcgen05
 * cta_group::2, M = 256 over two SMs of a cluster; 1..2 pairs' CTAs per SM).
 * Maps, offsets and epilogue are the same for every shape; when C_in spans
 * several K chunks the order of the f32 (offset, chunk) partial sums follows
 * the offsets grouped per stage, so outputs agree to f32 summation order. */
int32_t scb_conv_implicit_tuned(const void* features, int64_t ldf, int32_t c_split,
                                const void* features2, int64_t ldf2, int64_t n_in, int32_t c_in,
                                const int32_t* hits, int32_t volume, int64_t n_out,
                                const uint32_t* tile_mask, const void* weights_packed,
                                int32_t c_out, void* out, int64_t ldo, const float* scale,
                                const float* shift, const float* bias, const void* residual,
                                int32_t relu, int32_t ctas_per_sm, int32_t stage_kb,
                                scb_stream_t stream);

/* scb_conv_implicit_tuned over a permutation of the output rows: tile row r
 * computes output row out_rows[r] (nullable = identity), so `hits` and
 * `tile_mask` are in tile-row order (scb_onehot_order) and the epilogue
 * stores (and reads the residual at) row out_rows[r].  Lets a one-hot map
 * (the transposed k2 s2 layer) run with one active offset per tile. */
int32_t scb_conv_implicit_rows(const void* features, int64_t ldf, int32_t c_split,
                               const void* features2, int64_t ldf2, int64_t n_in, int32_t c_in,
                               const int32_t* hits, int32_t volume, int64_t n_out,
                               const uint32_t* tile_mask, const int32_t* out_rows,
                               const void* weights_packed, int32_t c_out, void* out, int64_t ldo,
                               const float* scale, const float* shift, const float* bias,
                               const void* residual, int32_t relu, int32_t ctas_per_sm,
                               int32_t stage_kb, scb_stream_t stream);

/* Transposed K = s layer in scatter form (replaces inverse_conv_forward,
 * execution.py:512-551, for a map made by swap_roles of a K = s strided map,
 * mapping.py:277-286): `child` is that strided map's hit matrix
 * [volume][hits_ld(n_in)] (child[n][p] = the fine row k whose parent is
 * coarse row p at offset n, or -1), so out[child[n][p]] = epilogue(x[p] . W[n]).
 * Every fine row must have exactly one (p, n) (true for K = s maps); each row
 * of `out` [n_out][ldo] is written once.  features [n_in][ldf] fp16, c_in and
 * c_out multiples of 8 up to 256, weights packed as for scb_conv_implicit.
 * BN scale/shift (together), bias, ReLU as scb_conv_implicit; no residual.
 * B200 extension: one dense tcgen05 tile of x per 128 coarse rows, no gather. */
int32_t scb_conv_transposed_scatter(const void* features, int64_t ldf, int64_t n_in, int32_t c_in,
                                    const int32_t* child, int32_t volume,
                                    const void* weights_packed, int32_t c_out, void* out,
                                    int64_t ldo, int64_t n_out, const float* scale,
                                    const float* shift, const float* bias, int32_t relu,
                                    scb_stream_t stream);

/* K = 1, s = 1 layer (sparse_conv_forward on a pointwise kernel, execution.py:
 * 456-459: out = x . W[0] with the identity map) as a dense tcgen05 GEMM: TMA
 * tiles of x (channels [0, c_split) from `features`, the rest from
 * `features2` when given — the decoder's skip concatenation, read in place),
 * weights packed as for scb_conv_implicit, BN scale/shift (together), bias and
 * ReLU fused, each row of `out` [n][ldo] written once.  c_in a multiple of 8
 * up to 256, c_split a multiple of 16, c_out up to 256 (not a multiple of 8:
 * the padding columns of the 8-aligned rows are written too, ldo >= that).  B200 extension of the
 * fused dataflow (the same kernel as scb_conv_transposed_scatter). */
int32_t scb_conv_pointwise(const void* features, int64_t ldf, int32_t c_split,
                           const void* features2, int64_t ldf2, int64_t n, int32_t c_in,
                           const void* weights_packed, int32_t c_out, void* out, int64_t ldo,
                           const float* scale, const float* shift, const float* bias,
                           int32_t relu, scb_stream_t stream);

/* Row order for a one-hot hit matrix (every output row has at most one
 * entry, e.g. the transposed map of a K = s strided layer): perm = the rows
 * stably sorted by the offset of their entry (rows without one last),
 * hits_out[n][r] = hits[n][perm[r]] and tile_masks[t] its 128-row tile words.
 * B200 extension (the reference keeps output-row order); results of
 * scb_conv_implicit_rows with out_rows = perm are unchanged. */
int64_t scb_onehot_order_workspace(int64_t n);
int32_t scb_onehot_order(const int32_t* hits, int32_t volume, int64_t n, void* workspace,
                         int64_t ws_bytes, int32_t* perm, int32_t* hits_out, uint32_t* tile_masks,
                         scb_stream_t stream);

/* Active-offset words of a hit matrix per 128-row output tile: bit n of
 * masks[t] is set when some row k in [128 t, 128 t + 128) has
 * hits[n][k] >= 0.  volume <= 32.  B200 extension (no reference
 * counterpart): the per-tile skip list of scb_conv_implicit_cat. */
int32_t scb_tile_masks(const int32_t* hits, int32_t volume, int64_t n_out, uint32_t* masks,
                       scb_stream_t stream);

/* ---------------------------------------------------------------- row reordering
 * B200 extension with no reference counterpart (the reference keeps rows in
 * flat-key order; DESIGN.md §3 "presence-mask reordering").  A model may
 * relabel the rows of a coordinate level so that 128-row tiles share their
 * neighbour pattern; maps built over the relabelled set hold the same
 * (input, output) pairs under the new row numbers, and the model
 * un-permutes its output (scb_permute_rows), so results are unchanged. */

/* mask[k] bit n = coords[k] + delta_n (stride 1, offsets of a K^D window with
 * base offset_base) is a row of the indexed set; counts[n] (uint64, V words,
 * zeroed here) = rows with bit n.  Odd K (symmetric probing: each row probes
 * the lower half and sets the mirror bit of the neighbour it finds), K^D <= 32. */
int32_t scb_presence_masks(int32_t kind, const int32_t* coords, int64_t n,
                           const scb_grid_t* grid, int32_t kernel_size, int32_t offset_base,
                           const int64_t* table_keys, const int32_t* table_rows, int64_t slots,
                           uint32_t* masks, uint64_t* counts, scb_stream_t stream);

/* The stride-1 map of an indexed set onto itself from its presence words
 * (mask[k] of scb_presence_masks, in the set's row order): row k probes
 * only the offsets its word marks present, hits[n][k] = -1 elsewhere; the
 * same [V][hits_ld(n)] hit matrix as scb_map_search(..., symmetric=1) for
 * odd K.  tile_masks (nullable, [ceil(n / 128)]) receives the OR of the row
 * words of each 128-row tile — scb_tile_masks of that hit matrix.  K^D <= 32.
 * B200 extension: half the probes of a symmetric search at LiDAR occupancy,
 * and no tile-mask pass over the hit matrix. */
int32_t scb_map_search_masked(int32_t kind, const int32_t* coords, int64_t n,
                              const scb_grid_t* grid, int32_t kernel_size, int32_t offset_base,
                              const int64_t* table_keys, const int32_t* table_rows, int64_t slots,
                              const uint32_t* masks, int32_t* hits, uint32_t* tile_masks,
                              scb_stream_t stream);

int64_t scb_mask_sort_workspace(int64_t n);

/* perm[i] = the row placed at position i: a stable sort by the mask with
 * offsets re-ranked so the least frequent are the most significant bits,
 * the masks visited in reflected-Gray-code order.
 * Rows of different batch entries interleave (maps never cross batch
 * entries; grouping equal words across the batch leaves fewer live tile
 * blocks).  `coords` int32 rows of `cols` words (batch first); batch_size is
 * validated only. */
int32_t scb_mask_sort(const uint32_t* masks, const uint64_t* counts, const int32_t* coords,
                      int32_t cols, int64_t n, int32_t volume, int64_t batch_size,
                      void* workspace, int64_t ws_bytes, int32_t* perm, scb_stream_t stream);

/* coords_out[i] = coords[perm[i]] (rows of `cols` int32) and inv_out[perm[i]] = i. */
int32_t scb_apply_order(const int32_t* perm, int64_t n, const int32_t* coords, int32_t cols,
                        int32_t* coords_out, int32_t* inv_out, scb_stream_t stream);

/* An index of the same coordinates under relabelled rows (row r -> inv[r]):
 * rows_out[s] = inv[rows_in[s]] for occupied slots / cells, -1 elsewhere.
 * The hash keys (table_keys) are shared unchanged.  Replaces building a
 * second index over the relabelled set. */
int32_t scb_index_relabel(int32_t kind, const int64_t* table_keys, const int32_t* rows_in,
                          int64_t slots, const int32_t* inv, int32_t* rows_out,
                          scb_stream_t stream);

/* Row permutation of a byte matrix: scatter = 0: dst[i] = src[index[i]];
 * scatter = 1: dst[index[i]] = src[i]; row_bytes a multiple of 2. */
int32_t scb_permute_rows(const void* src, int64_t src_ld_bytes, const int32_t* index, int64_t n,
                         int32_t row_bytes, void* dst, int64_t dst_ld_bytes, int32_t scatter,
                         scb_stream_t stream);

/* ---------------------------------------------------------------- voxelisation
 * Replaces voxelize (core.py:174-216), the step in front of the path
 * (SURVEY.md §8(f) row 2): `points` f64 [n][cols] (first spatial_dims
 * columns are positions), cells = floor((p - min) / voxel_size), boundary =
 * max + 1, rows in ascending flat-key order, features merged by the f64 mean
 * in point order (reduce_first = 0) or taken from the first point (1) and
 * rounded once to f32 — bit-exact with the reference.  `out_coords` int32
 * [n][1+D] and `out_features` f32 [n][cols-D] need room for n rows; `meta`
 * (device int64 [1+D]) receives the voxel count and the boundary. */
int64_t scb_voxelize_workspace(int64_t n_points, int32_t spatial_dims);
int32_t scb_voxelize(const double* points, int64_t n_points, int32_t cols, int32_t spatial_dims,
                     double voxel_size, int32_t reduce_first, void* workspace, int64_t ws_bytes,
                     int32_t* out_coords, float* out_features, int64_t* meta,
                     scb_stream_t stream);
/* A batch of raw scans in one pass: scan b is points [scan_ptr[b],
 * scan_ptr[b+1]) (device int64 [n_scans+1], n_scans <= 64), voxelised
 * exactly as voxelize (core.py:174-216) voxelises it alone (its own min
 * corner), with batch column b; the boundary in `meta` is the per-dimension
 * max over the scans.  Rows ascend by (b, flat key): bit-identical to B
 * scb_voxelize calls concatenated with a shared boundary.
 * Workspace: scb_voxelize_workspace(n_points, spatial_dims). */
int32_t scb_voxelize_batch(const double* points, const int64_t* scan_ptr, int32_t n_scans,
                           int64_t n_points, int32_t cols, int32_t spatial_dims,
                           double voxel_size, int32_t reduce_first, void* workspace,
                           int64_t ws_bytes, int32_t* out_coords, float* out_features,
                           int64_t* meta, scb_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPARSECONV_B200_H */
