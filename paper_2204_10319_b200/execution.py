"""Gather -> grouped GEMM -> scatter on the B200, behind the reference's
execution API (reference ``execution.py``).

Layer data flow (device side):

    mapping   index + map search (+ output coords when strided), cached per
              coordinate set and (K, stride)            [mapping.py kernels]
    gather    buffer[slab rows] = features[buf_in]       [scb_gather]
    matmul    one persistent tcgen05 launch over every scheduled offset
              (+ the centre offset read straight from the features)
                                                          [scb_grouped_gemm]
    scatter   output-stationary f32 fold + centre add + optional epilogue,
              one write per output row                     [scb_scatter]

Numerics: FP16 storage rounds weights to fp16 for
the tensor cores and accumulates in f32 (tolerance 1e-2 relative L2); FP32
storage runs an exact-f32 FMA GEMM (tolerance 1e-4).  The grouping strategy
(eps, S) changes the tile order of the persistent launch, never the result.
"""

from __future__ import annotations

import warnings
from contextlib import contextmanager, nullcontext
from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _native as nat
from .core import (CoordinateSet, PrecisionMode, SparseTensor, WeightTensor,
                   flush_saturation_warnings)
from .mapping import (DEFAULT_GRID_CELL_CAP, GatherScatterPlan, GridCapacityError, KernelMap,
                      KernelOffsets, build_gather_scatter_plan, build_index,
                      compute_output_coords, compute_output_coords_chain, downsample_boundary,
                      start_output_coords_chain,
                      enumerate_offsets, map_search, map_search_masked, permute_rows,
                      reorder_by_presence, _cells)

GATHER_ORDERS = ("weight_stationary", "input_stationary")
SCATTER_ORDERS = ("weight_stationary", "output_stationary")


class StageTimer:
    """Per-(layer, stage) device time over a forward pass, measured with CUDA
    events on the compute stream (reference StageTimer, execution.py:39-58)."""

    STAGES = ("mapping", "gather", "matmul", "scatter", "fused", "other")

    def __init__(self):
        self._events: list[tuple[str, str, torch.cuda.Event, torch.cuda.Event]] = []
        self._samples: dict[tuple[str, str], float] = {}
        self._pool: list[torch.cuda.Event] = []

    def _event(self) -> torch.cuda.Event:
        return self._pool.pop() if self._pool else torch.cuda.Event(enable_timing=True)

    def section(self, layer: str, stage: str) -> "_Section":
        return _Section(self, layer, stage)

    @property
    def samples(self) -> dict[tuple[str, str], float]:
        if self._events:
            torch.cuda.synchronize()
            for layer, stage, s, e in self._events:
                key = (layer, stage)
                self._samples[key] = self._samples.get(key, 0.0) + s.elapsed_time(e) / 1e3
                self._pool += (s, e)  # events are reusable once read
            self._events.clear()
        return dict(self._samples)


class _Section:
    """CUDA-event bracket of one (layer, stage) on the current stream."""

    __slots__ = ("timer", "layer", "stage", "start")

    def __init__(self, timer: StageTimer, layer: str, stage: str):
        self.timer, self.layer, self.stage = timer, layer, stage

    def __enter__(self):
        self.start = self.timer._event()
        self.start.record()
        return self

    def __exit__(self, *exc):
        end = self.timer._event()
        end.record()
        self.timer._events.append((self.layer, self.stage, self.start, end))
        return False


def _timed(timer, layer, stage):
    return timer.section(layer, stage) if timer is not None else nullcontext()


@dataclass(frozen=True)
class LayerStrategy:
    """Tuned grouping parameters (execution.py:61-93)."""

    eps: float = 0.0
    threshold: float = 0.0
    index_kind: str | None = None

    def __post_init__(self):
        if not 0.0 <= self.eps <= 1.0:
            raise ValueError("eps must lie in [0, 1]")
        if self.threshold < 0:
            raise ValueError("threshold must be non-negative")

    @staticmethod
    def separate() -> "LayerStrategy":
        return LayerStrategy(0.0, 0.0)

    @staticmethod
    def symmetric_pairs() -> "LayerStrategy":
        return LayerStrategy(0.0, float("inf"))

    @staticmethod
    def dense_group() -> "LayerStrategy":
        return LayerStrategy(1.0, float("inf"))


@dataclass(frozen=True)
class LayerSpec:
    """Static description of a convolution layer (execution.py:96-113)."""

    kernel_size: int
    stride: int
    c_in: int
    c_out: int
    transposed: bool = False
    reuse_key: str | None = None
    index_kind: str | None = None
    strategy: LayerStrategy | None = None
    dilation: int = 1   # B200 extension (north_star SparseConv3d; the reference has none)

    def __post_init__(self):
        if self.stride not in (1, 2):
            raise ValueError(f"unsupported stride {self.stride}")
        if self.transposed and not self.reuse_key:
            raise ValueError("transposed layers need the reuse key of a strided layer")
        if int(self.dilation) < 1:
            raise ValueError("dilation must be >= 1")
        if self.dilation != 1 and (self.stride != 1 or self.transposed):
            raise ValueError("dilation > 1 is supported for stride-1 (submanifold) layers only")


def resolve_strategy(spec: LayerSpec, strategy: LayerStrategy | None) -> LayerStrategy:
    """Explicit argument, then the LayerSpec override, then separate
    (execution.py:116-123)."""
    if strategy is not None:
        return strategy
    if spec.strategy is not None:
        return spec.strategy
    return LayerStrategy.separate()


@dataclass(eq=False)
class CachedMap:
    """A strided layer's map plus its input-side geometry (execution.py:126-134)."""

    kmap: KernelMap
    in_coords: torch.Tensor
    in_boundary: tuple
    in_stride: int
    in_coordset: CoordinateSet | None = None


@dataclass
class ExecOptions:
    """Per-call knobs; numerics are invariant under all of them
    (execution.py:137-156).  ``map_reuse`` keeps maps built over a
    coordinate set for later layers at the same level (result-identical).
    ``dataflow`` selects the staged gather/GEMM/scatter pipeline (default,
    the reference's structure), the fused implicit-GEMM kernel, or ``auto``
    (per-layer roofline choice)."""

    order: str = "locality"
    fused: bool = True
    index_kind: str | None = None
    grid_cell_cap: int = DEFAULT_GRID_CELL_CAP
    layer_label: str = "layer"
    timer: StageTimer | None = None
    traffic_log: list | None = None
    workload_log: list | None = None
    plan_log: list | None = None
    map_reuse: bool = True
    dataflow: str = "staged"
    sync_free: bool = True
    # B200 extension: layer label -> (CTAs per SM, stage KB) launch shape of
    # the fused kernel, from a strategy file (autotune.tune_fused_layer);
    # absent layers use the built-in heuristic.  Results are shape-invariant.
    kernel_shapes: dict | None = None


    def __post_init__(self):
        if self.order not in ("locality", "weight"):
            raise ValueError(f"unknown order {self.order!r}")
        if self.dataflow not in ("staged", "fused", "auto"):
            raise ValueError(f"unknown dataflow {self.dataflow!r}")
        if not self.fused and self.order == "locality":
            warnings.warn("locality order requires fused movement; using weight order")
            self.order = "weight"


# ====================================================================== movement API

def _features_of(x) -> torch.Tensor:
    if isinstance(x, SparseTensor):
        return x.features
    if isinstance(x, torch.Tensor):
        return x.contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _buffer_ld(dtype, c: int) -> int:
    return (c + 7) // 8 * 8 if dtype == torch.float16 else c


def _ld(t: torch.Tensor | None) -> int:
    """Row stride in elements (torch reports odd strides for 0-row tensors)."""
    if t is None:
        return 0
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


class _Arena:
    """Per-(device, stream) scratch slots for the per-layer gather buffer and
    f32 partials.  Layers run in stream order, so one slot serves every layer
    of a forward pass; slots only grow (by >= 25%), which keeps multi-GB
    cudaMalloc/cudaFree churn out of the forward."""

    def __init__(self):
        self.slots = {}

    def tensor(self, name: str, shape, dtype, device) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= int(s)
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        key = (device.index, nat.stream_handle(), name)
        raw = self.slots.get(key)
        if raw is None or raw.numel() < nbytes:
            grow = 0 if raw is None else raw.numel() + raw.numel() // 4
            raw = torch.empty(max(nbytes, grow, 256), dtype=torch.uint8, device=device)
            self.slots[key] = raw
        return raw[:nbytes].view(dtype).view(tuple(int(s) for s in shape))


_ARENA = _Arena()


def _gather_padded(features: torch.Tensor, plan: GatherScatterPlan, c: int) -> torch.Tensor:
    ld = _buffer_ld(features.dtype, c)
    buf = _ARENA.tensor("gather", (max(plan.rows_pad, 1), ld), features.dtype, features.device)
    nat.call("scb_gather", nat.dtype_code(features.dtype), nat.ptr(features), features.shape[0], c,
             _ld(features), nat.ptr(plan.buf_in), plan.rows_pad, nat.ptr(buf), ld, None,
             nat.stream_handle())
    return buf


class DevicePlan:
    """Sync-free plan of one layer (scb_plan_from_hits): buffer rows,
    output positions and the GEMM problem table all built on the device from
    the hit matrix; sizes are capacities (upper bounds), the real row count
    lives in the device table."""

    __slots__ = ("pos", "buf_in", "table", "rows_cap", "c_base", "offset_ptr")

    def __init__(self, kmap: KernelMap, skip: int | None, dtype, c_out: int,
                 center_rows: int, center_seg: int | None):
        import ctypes
        lib = nat.load()
        dev = kmap.device
        V, n_out = kmap.offsets.volume, kmap.n_out
        bm, ntn = ctypes.c_int32(), ctypes.c_int32()
        lib.scb_gemm_tile_geometry(nat.dtype_code(dtype), c_out, ctypes.byref(bm),
                                   ctypes.byref(ntn))
        self.rows_cap = int(lib.scb_plan_rows_cap(V, n_out, nat.TILE_ROWS))
        self.c_base = (center_rows + nat.TILE_ROWS - 1) // nat.TILE_ROWS * nat.TILE_ROWS
        ws = _ARENA.tensor("map_ws", (max(int(lib.scb_map_workspace(V, n_out)), 8),),
                           torch.uint8, dev)
        self.offset_ptr = torch.empty(V + 1, dtype=torch.int64, device=dev)
        self.buf_in = torch.empty(max(self.rows_cap, 1), dtype=torch.int32, device=dev)
        self.pos = torch.empty((max(n_out, 1), V), dtype=torch.int32, device=dev)
        self.table = torch.empty(int(lib.scb_segtable_bytes()), dtype=torch.uint8, device=dev)
        nat.call("scb_plan_from_hits", nat.ptr(kmap.hits), V, n_out,
                 -1 if skip is None else skip, nat.TILE_ROWS, self.c_base, bm.value, ntn.value,
                 -1 if center_seg is None else center_seg, center_rows, nat.ptr(ws),
                 nat.ptr(self.offset_ptr), nat.ptr(self.buf_in), nat.ptr(self.pos),
                 nat.ptr(self.table), nat.stream_handle())

    @property
    def rows_pad_ptr(self) -> int:
        return self.table.data_ptr() + 8  # SegTable.rows_pad


def gather(features, plan: GatherScatterPlan, order: str = "weight_stationary") -> torch.Tensor:
    """Offset-partitioned buffer in the reference layout (execution.py:159-180);
    both orders are the same bit-exact device copy."""
    if order not in GATHER_ORDERS:
        raise ValueError(f"unknown gather order {order!r}")
    f = _features_of(features)
    if f.shape[0] != plan.n_in:
        raise ValueError("plan does not match the feature row count")
    buf = _gather_padded(f, plan, f.shape[1])
    return buf[plan.padded_rows(buf), : f.shape[1]].contiguous()


def scatter_accumulate(buffer, plan: GatherScatterPlan, n_out: int,
                       order: str = "weight_stationary", out_dtype=np.float32) -> torch.Tensor:
    """Fold buffer rows into output rows in ascending buffer-row order
    (execution.py:183-218): one f32 output-stationary pass on the device."""
    if order not in SCATTER_ORDERS:
        raise ValueError(f"unknown scatter order {order!r}")
    b = _features_of(buffer)
    if b.shape[0] != plan.total:
        raise ValueError("buffer rows do not match the plan")
    c = b.shape[1]
    odt = torch.float16 if np.dtype(out_dtype) == np.float16 else torch.float32
    if plan.general:  # several entries per (output, offset): CSR fold
        b = b.contiguous()
        out = torch.empty((n_out, c), dtype=odt, device=b.device)
        ptr, rows = plan.device_out_csr()
        nat.call("scb_scatter_csr", nat.dtype_code(b.dtype), nat.ptr(b), c, nat.ptr(ptr),
                 nat.ptr(rows), n_out, c, nat.dtype_code(odt), nat.ptr(out), c,
                 nat.stream_handle())
        return out
    b = b.to(torch.float32)
    padded = torch.zeros((max(plan.rows_pad, 1), c), dtype=torch.float32, device=b.device)
    if plan.total:
        padded[plan.padded_rows(b)] = b
    out = torch.empty((n_out, c), dtype=odt, device=b.device)
    nat.call("scb_scatter", nat.ptr(padded), c, nat.ptr(plan.pos), plan.pos.shape[1], n_out, c, -1,
             nat.dtype_code(odt), nat.ptr(out), c, None, None, None, None, 0, nat.stream_handle())
    return out


# ====================================================================== grouping (host, O(V))

def partition_groups(map_sizes, eps: float, schedule) -> list[tuple[int, int]]:
    """Alg. 3 greedy grouping of scheduled offsets (execution.py:221-247)."""
    if not 0.0 <= eps <= 1.0:
        raise ValueError("eps must lie in [0, 1]")
    sizes = np.asarray(map_sizes, dtype=np.int64)
    schedule = list(schedule)
    ranges, i = [], 0
    while i < len(schedule):
        lo = hi = int(sizes[schedule[i]])
        start = i
        i += 1
        while i < len(schedule):
            n = int(sizes[schedule[i]])
            nlo, nhi = min(lo, n), max(hi, n)
            if (0.0 if nhi == 0 else 1.0 - nlo / nhi) > eps:
                break
            lo, hi = nlo, nhi
            i += 1
        ranges.append((start, i))
    return ranges


@dataclass(frozen=True)
class MatmulGroup:
    start: int
    end: int
    mode: str
    padded_rows: int = 0


@dataclass(frozen=True)
class GroupingStrategy:
    """Partition of the scheduled offsets into matmul groups
    (execution.py:258-293)."""

    eps: float
    threshold: float
    schedule: tuple
    groups: tuple
    symmetric: bool
    volume: int

    def members(self, group: MatmulGroup) -> list[int]:
        sched = list(self.schedule[group.start:group.end])
        if self.symmetric:
            sched += [self.volume - 1 - n for n in sched]
        return sched

    def validate(self, map_sizes) -> None:
        sizes = np.asarray(map_sizes, dtype=np.int64)
        if sizes.shape[0] != self.volume:
            raise ValueError("map sizes do not match the strategy volume")
        covered = []
        for g in self.groups:
            covered.extend(range(g.start, g.end))
            mem = self.members(g)
            hi = max((int(sizes[m]) for m in mem), default=0)
            lo = min((int(sizes[m]) for m in mem), default=0)
            if (g.mode == "batched") != (hi < self.threshold):
                raise ValueError("group mode disagrees with the threshold")
            if g.mode == "batched" and hi > 0 and 1.0 - lo / hi > self.eps + 1e-12:
                raise ValueError("batched group exceeds the padding tolerance")
        if covered != list(range(len(self.schedule))):
            raise ValueError("groups do not partition the schedule")


def schedule_for(offsets: KernelOffsets, stride: int) -> tuple[list[int], bool]:
    """First half without centre + mirrors on stride-1 odd K, else all
    offsets (execution.py:296-306)."""
    c = offsets.center
    if stride == 1 and c is not None and offsets.volume > 1:
        return list(range(c)), True
    return list(range(offsets.volume)), False


def build_grouping(map_sizes, eps: float, threshold: float, schedule=None,
                   symmetric: bool = False) -> GroupingStrategy:
    """Concrete GroupingStrategy for a workload (execution.py:309-328)."""
    sizes = np.asarray(map_sizes, dtype=np.int64)
    schedule = list(range(sizes.shape[0])) if schedule is None else list(schedule)
    groups = []
    for start, end in partition_groups(sizes, eps, schedule):
        mem = list(schedule[start:end])
        if symmetric:
            mem += [sizes.shape[0] - 1 - n for n in mem]
        hi = max((int(sizes[m]) for m in mem), default=0)
        if hi < threshold:
            groups.append(MatmulGroup(start, end, "batched", sum(hi - int(sizes[m]) for m in mem)))
        else:
            groups.append(MatmulGroup(start, end, "sequential", 0))
    return GroupingStrategy(eps, threshold, tuple(schedule), tuple(groups), symmetric,
                            sizes.shape[0])


# ====================================================================== GEMM

def _segments(grouping: GroupingStrategy, slab_ptr: np.ndarray, sizes: np.ndarray,
              extra=()) -> "ctypes.Array":
    segs = []
    seen = set()
    for g in grouping.groups:
        for m in grouping.members(g):
            if m in seen or sizes[m] == 0:
                continue
            seen.add(m)
            segs.append((int(slab_ptr[m]), int(slab_ptr[m]), int(sizes[m]), int(m), 0))
    segs.extend(extra)
    if len(segs) > nat.MAX_SEGMENTS:
        raise ValueError("too many GEMM segments for one launch")
    arr = (nat.SegmentT * max(len(segs), 1))()
    for i, (a, c, r, b, src) in enumerate(segs):
        arr[i].a_row, arr[i].c_row, arr[i].rows, arr[i].b_index, arr[i].a_src = a, c, r, b, src
    return arr, len(segs)


def _weights_for(w: WeightTensor, dtype):
    if dtype == torch.float16:
        packed, _, n_pad = w.packed_f16()
        return packed, n_pad
    return w.device_f32(), w.c_out


def _grouped_gemm(dtype, buffer, rows_pad, features, w: WeightTensor, segs, nseg, c_rows):
    wt, ldc = _weights_for(w, dtype)
    partial = _ARENA.tensor("partial", (max(c_rows, 1), ldc), torch.float32, wt.device)
    nat.call("scb_grouped_gemm", nat.dtype_code(dtype), nat.ptr(buffer), max(rows_pad, 1),
             _ld(buffer), nat.ptr(features), 0 if features is None else features.shape[0],
             0 if features is None else _ld(features), w.c_in, nat.ptr(wt), w.weights.shape[0],
             w.c_out, nat.ptr(partial), max(c_rows, 1), ldc, segs, nseg, nat.stream_handle())
    return partial, ldc


def execute_groups(buffer, weights, strategy: GroupingStrategy, map_sizes) -> torch.Tensor:
    """Grouped multiplies over an offset-partitioned buffer in the reference
    layout (execution.py:331-368); returns the f32 partial buffer."""
    sizes = np.asarray(map_sizes, dtype=np.int64)
    if isinstance(weights, WeightTensor):
        w = weights
    else:
        wa = np.asarray(weights.cpu() if isinstance(weights, torch.Tensor) else weights,
                        dtype=np.float32)
        w = WeightTensor(wa, wa.shape[0], 1)  # a plain (V, C_in, C_out) stack
    if sizes.shape[0] != w.weights.shape[0]:
        raise ValueError("map sizes do not match the weight slices")
    strategy.validate(sizes)
    b = _features_of(buffer)
    starts = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
    np.cumsum(sizes, out=starts[1:])
    if b.shape[0] != starts[-1]:
        raise ValueError("buffer rows do not match the map sizes")
    tile = nat.TILE_ROWS
    slab = np.zeros_like(starts)
    np.cumsum((sizes + tile - 1) // tile * tile, out=slab[1:])
    rows_pad = int(slab[-1])
    ld = _buffer_ld(b.dtype, b.shape[1])
    padded = torch.zeros((max(rows_pad, 1), ld), dtype=b.dtype, device=b.device)
    idx = [torch.arange(int(slab[n]), int(slab[n] + sizes[n])) for n in range(sizes.shape[0])
           if sizes[n]]
    prow = torch.cat(idx).to(b.device) if idx else torch.empty(0, dtype=torch.int64, device=b.device)
    if prow.numel():
        padded[prow, : b.shape[1]] = b
    segs, nseg = _segments(strategy, slab, sizes)
    partial, _ = _grouped_gemm(b.dtype, padded, rows_pad, None, w, segs, nseg, rows_pad)
    return partial[prow, : w.c_out].contiguous()


# ====================================================================== layers

def _direct_center(dtype, c_in: int) -> bool:
    """The centre offset reads the feature matrix in place when the TMA row
    stride allows it (16-byte multiple); otherwise it is gathered too."""
    return dtype == torch.float32 or c_in % 8 == 0


def _epi_vec(x, c_out: int, name: str):
    if x is None:
        return None
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32
            and x.is_contiguous() and x.shape == (c_out,)):
        raise ValueError(f"epilogue {name} must be a contiguous CUDA float32 vector of length "
                         f"C_out = {c_out}")
    return x.data_ptr()


def _epi_args(ep: dict | None, n_out: int, c_out: int, dtype):
    """Raw epilogue operands, checked: the kernels read scale/shift/bias as
    f32[C_out] and the residual as a dense [n_out][C_out] matrix of the
    storage dtype."""
    ep = ep or {}
    res = ep.get("residual")
    if isinstance(res, SparseTensor):
        res = res.features
    if res is not None:
        if not (isinstance(res, torch.Tensor) and res.is_cuda and res.dtype == dtype
                and tuple(res.shape) == (n_out, c_out)):
            raise ValueError("residual must be a CUDA matrix of the output's shape and dtype")
        if not res.is_contiguous():
            raise ValueError("residual must be contiguous (row stride C_out)")
    return (_epi_vec(ep.get("scale"), c_out, "scale"), _epi_vec(ep.get("shift"), c_out, "shift"),
            _epi_vec(ep.get("bias"), c_out, "bias"), nat.ptr(res),
            int(bool(ep.get("relu", False))))


# Transposed K = s layers in scatter form (scb_conv_transposed_scatter);
# SCB_UPSCATTER=0 runs them through the gather-form fused kernel instead.
_UPSCATTER = os.environ.get("SCB_UPSCATTER", "1") != "0"
# K = 1 layers as dense TMA-fed GEMMs (scb_conv_pointwise); SCB_DENSE_K1=0 runs
# them through the gather-form fused kernel's identity map instead.
_DENSE_K1 = os.environ.get("SCB_DENSE_K1", "1") != "0"


def _fused_eligible(dtype, volume: int, w: WeightTensor) -> bool:
    """The implicit-GEMM kernel: FP16 storage, K^3 in {1, 8, 27}, C_out up to
    256 (C_out not a multiple of 8, e.g. the 19-class head, is written into
    8-aligned rows and returned as a view).  C_in that is not a multiple of 8
    (the 4-channel stem) is zero-padded to one.  Volume 1 covers both the
    K=1 s=1 identity map and K=1 strided maps (their hit matrix is read)."""
    return dtype == torch.float16 and volume in (1, 8, 27) and w.c_out <= 256


def choose_dataflow(opts: ExecOptions, dtype, kmap: KernelMap | None, w: WeightTensor) -> str:
    """"staged" (gather -> grouped GEMM -> scatter, the reference's structure)
    or "fused" (one implicit-GEMM kernel).  ``auto`` picks fused wherever it
    is eligible: measured on B200 per MinkUNet layer (tools/layer_compare.py,
    8 packed scans) it wins every k3 / k2 / transposed layer from 32 to 256
    channels (e.g. 96->96 at level 0: 0.82 vs 1.77 ms, 256->256: 0.22 vs
    0.35 ms) and k1 layers once their output is written by the fused
    epilogue instead of an f32 partial round trip."""
    volume = 1 if kmap is None else kmap.offsets.volume
    if opts.dataflow == "staged" or not _fused_eligible(dtype, volume, w):
        return "staged"
    return "fused"


def _pad_channels(f: torch.Tensor) -> torch.Tensor:
    """Zero-pad fp16 rows to a multiple of 8 channels (16-B cp.async chunks);
    the packed weights already carry zero rows for the padded channels."""
    c = f.shape[1]
    if c % 8 == 0 and f.is_contiguous():
        return f
    return torch.nn.functional.pad(f, (0, (-c) % 8)).contiguous()


def _run_fused(features: torch.Tensor, kmap: KernelMap | None, w: WeightTensor,
               opts: ExecOptions, epilogue: dict | None, concat: torch.Tensor | None = None
               ) -> torch.Tensor:
    """One scb_conv_implicit launch; ``kmap`` None = the K=1 identity map.
    ``concat``: more input channels (same rows), read in place."""
    label, timer = opts.layer_label, opts.timer
    packed, _, _ = w.packed_f16()
    volume = 1 if kmap is None else kmap.offsets.volume
    n_out = features.shape[0] if kmap is None else kmap.n_out
    ldo = (w.c_out + 7) // 8 * 8
    out = torch.empty((n_out, ldo), dtype=features.dtype, device=features.device)
    scale, shift, bias, res, relu = _epi_args(epilogue, n_out, w.c_out, features.dtype)
    rows = None
    scatter = (kmap is not None and kmap.onehot and kmap._parent is not None and concat is None
               and res is None and _UPSCATTER and w.c_in % 8 == 0 and w.c_out % 8 == 0
               and features.shape[1] == w.c_in and features.is_contiguous())
    cb = 0 if concat is None else concat.shape[1]
    pointwise = (kmap is None and _DENSE_K1 and res is None and not scatter
                 and w.c_in <= 256 and features.is_contiguous()
                 and features.shape[1] % (8 if concat is None else 16) == 0
                 and (concat is None or (concat.is_contiguous() and cb % 8 == 0))
                 and features.shape[1] + cb == w.c_in)
    if pointwise:
        # K = 1 layer: dense TMA tiles of x (and the concatenated skip) -> tcgen05
        with _timed(timer, label, "fused"):
            nat.call("scb_conv_pointwise", nat.ptr(features), features.shape[1],
                     features.shape[1], nat.ptr(concat), cb, features.shape[0], w.c_in,
                     nat.ptr(packed), w.c_out, nat.ptr(out), ldo, scale, shift, bias, relu,
                     nat.stream_handle())
    elif scatter:
        # transposed K = s layer: coarse tiles scattered to their one fine row each
        child = kmap._parent.hits
        with _timed(timer, label, "fused"):
            nat.call("scb_conv_transposed_scatter", nat.ptr(features), features.shape[1],
                     features.shape[0], w.c_in, nat.ptr(child), volume, nat.ptr(packed), w.c_out,
                     nat.ptr(out), ldo, n_out, scale, shift, bias, relu, nat.stream_handle())
    elif kmap is not None and kmap.onehot and os.environ.get("SCB_ONEHOT", "0") == "1":
        # one entry per output row: tiles over the rows sorted by offset
        perm, h, m = kmap.onehot_order()
        hits, masks, rows = nat.ptr(h), nat.ptr(m), nat.ptr(perm)
    else:
        hits = None if kmap is None else nat.ptr(kmap.hits)
        masks = None if kmap is None else nat.ptr(kmap.tile_masks())
    if not (scatter or pointwise):
        with _timed(timer, label, "fused"):
            if concat is not None and features.shape[1] % 8 == 0 and concat.shape[1] % 8 == 0 \
                    and features.is_contiguous() and concat.is_contiguous():
                f, ca, f2, cb = features, features.shape[1], concat, concat.shape[1]
            else:
                f = features if concat is None else torch.cat([features, concat], dim=1)
                f, ca, f2, cb = _pad_channels(f), None, None, 0
                ca = f.shape[1]
            ctas, skb = (opts.kernel_shapes or {}).get(label, (0, 0))
            nat.call("scb_conv_implicit_rows", nat.ptr(f), f.shape[1], ca, nat.ptr(f2),
                     0 if f2 is None else f2.shape[1], f.shape[0], ca + cb, hits, volume, n_out,
                     masks, rows, nat.ptr(packed), w.c_out, nat.ptr(out), ldo, scale, shift, bias,
                     res, relu, int(ctas), int(skb), nat.stream_handle())
    if ldo != w.c_out:
        out = out[:, : w.c_out]  # 8-aligned rows for the TMA store; a strided view
    if opts.traffic_log is not None:
        # algorithmic bytes: features in + out once, the
        # index words of the map entries moved (4 |M'|: the centre of a
        # stride-1 odd-K map is implicit), the weights, the residual
        e = 2
        m_total = n_out if kmap is None else kmap.total
        centre = kmap is not None and kmap.stride == 1 and kmap.offsets.center is not None
        m_moved = 0 if kmap is None else m_total - (n_out if centre else 0)
        base = (e * features.shape[0] * w.c_in + e * n_out * w.c_out
                + e * volume * w.c_in * w.c_out + (e * n_out * w.c_out if res else 0))
        if kmap is None:
            blocks = (n_out + nat.TILE_ROWS - 1) // nat.TILE_ROWS
        elif scatter:  # every (coarse tile, offset) block is multiplied
            blocks = volume * ((features.shape[0] + nat.TILE_ROWS - 1) // nat.TILE_ROWS)
        else:
            tm = (kmap.onehot_order()[2] if rows is not None else kmap.tile_masks()
                  ).cpu().numpy().astype(np.uint32)
            blocks = int(sum(bin(int(x)).count("1") for x in tm))
        opts.traffic_log.append((label, {
            "fused_bytes": base + 4 * m_moved,
            "fused_bytes_dense_index": base + (4 * volume * n_out if volume > 1 else 0),
            # useful FLOPs 2 |M| C_in C_out; executed: 128-row blocks of the
            # active (tile, offset) pairs the kernel multiplies
            "fused_flops": 2 * m_total * w.c_in * w.c_out,
            "fused_flops_executed": 2 * blocks * nat.TILE_ROWS * w.c_in * w.c_out,
            "fused_blocks": blocks, "fused_blocks_dense": volume * (
                (n_out + nat.TILE_ROWS - 1) // nat.TILE_ROWS)}))
    return out


def _run_staged_device(features: torch.Tensor, kmap: KernelMap, w: WeightTensor,
                       opts: ExecOptions, center: int | None, epilogue: dict | None):
    """Staged gather -> grouped GEMM -> scatter without any host sync: the
    plan and GEMM problem table come from scb_plan_from_hits, buffers are
    arena capacities, kernels read the live row/tile counts on the device.
    Same buffer layout and fold order as the host-planned path."""
    label, timer = opts.layer_label, opts.timer
    dt = features.dtype
    c_in, c_out = w.c_in, w.c_out
    direct = center is not None and _direct_center(dt, c_in)
    center_rows = features.shape[0] if direct else 0
    key = ("device", center if direct else None, nat.dtype_code(dt), c_out if dt == torch.float32
           else 0, center_rows)
    dp = kmap._plans.get(key)
    if dp is None:
        dp = DevicePlan(kmap, center if direct else None, dt, c_out, center_rows,
                        center if direct else None)
        kmap._plans[key] = dp
    ld = _buffer_ld(dt, c_in)
    with _timed(timer, label, "gather"):
        buf = _ARENA.tensor("gather", (max(dp.rows_cap, 1), ld), dt, features.device)
        nat.call("scb_gather", nat.dtype_code(dt), nat.ptr(features), features.shape[0], c_in,
                 _ld(features), nat.ptr(dp.buf_in), dp.rows_cap, nat.ptr(buf), ld,
                 dp.rows_pad_ptr, nat.stream_handle())
    wt, ldc = _weights_for(w, dt)
    c_rows = dp.c_base + dp.rows_cap
    with _timed(timer, label, "matmul"):
        partial = _ARENA.tensor("partial", (max(c_rows, 1), ldc), torch.float32, features.device)
        nat.call("scb_grouped_gemm_table", nat.dtype_code(dt), nat.ptr(buf), max(dp.rows_cap, 1),
                 ld, nat.ptr(features) if direct else None, features.shape[0] if direct else 0,
                 _ld(features) if direct else 0, c_in, nat.ptr(wt), w.weights.shape[0], c_out,
                 nat.ptr(partial), max(c_rows, 1), ldc, nat.ptr(dp.table), nat.stream_handle())
    out = torch.empty((kmap.n_out, c_out), dtype=dt, device=features.device)
    with _timed(timer, label, "scatter"):
        nat.call("scb_scatter", nat.ptr(partial), ldc, nat.ptr(dp.pos), kmap.offsets.volume,
                 kmap.n_out, c_out, 0 if direct else -1, nat.dtype_code(dt), nat.ptr(out), c_out,
                 *_epi_args(epilogue, kmap.n_out, c_out, dt), nat.stream_handle())
    return out


def _run_dataflow(features: torch.Tensor, kmap: KernelMap, w: WeightTensor,
                  strat: LayerStrategy, schedule, symmetric: bool, opts: ExecOptions,
                  center: int | None, epilogue: dict | None = None, record=None,
                  concat: torch.Tensor | None = None) -> torch.Tensor:
    """One layer's gather -> GEMM -> scatter; returns storage-dtype rows.
    ``concat``: more input channels of the same rows (fused: read in place)."""
    if choose_dataflow(opts, features.dtype, kmap, w) == "fused":
        if record is not None and opts.workload_log is not None:
            record(kmap.sizes)
        return _run_fused(features, kmap, w, opts, epilogue, concat)
    if concat is not None:
        features = torch.cat([features, concat], dim=1)
    if opts.sync_free and opts.workload_log is None and opts.plan_log is None \
            and opts.traffic_log is None:
        return _run_staged_device(features, kmap, w, opts, center, epilogue)
    sizes = kmap.sizes
    if center is not None:
        sizes[center] = 0
    if record is not None:
        record(sizes)
    grouping = build_grouping(sizes, strat.eps, strat.threshold, schedule, symmetric)
    label, timer = opts.layer_label, opts.timer
    dt = features.dtype
    c_in, c_out = w.c_in, w.c_out
    direct = center is not None and _direct_center(dt, c_in)
    plan = build_gather_scatter_plan(kmap, skip_center=direct)
    if opts.plan_log is not None:
        opts.plan_log.append((label, plan))
    sizes = plan.sizes
    with _timed(timer, label, "gather"):
        buf = _gather_padded(features, plan, c_in)
    extra = []
    center_row = -1
    c_rows = plan.rows_pad
    if direct:
        center_row = plan.rows_pad
        extra.append((0, center_row, features.shape[0], center, 1))
        c_rows += (features.shape[0] + nat.TILE_ROWS - 1) // nat.TILE_ROWS * nat.TILE_ROWS
    elif center is not None and sizes[center]:
        # centre gathered like any other offset (C_in not 16-byte aligned)
        extra.append((int(plan.slab_ptr[center]), int(plan.slab_ptr[center]),
                      int(sizes[center]), center, 0))
    segs, nseg = _segments(grouping, plan.slab_ptr, sizes, extra)
    with _timed(timer, label, "matmul"):
        partial, ldc = _grouped_gemm(dt, buf, plan.rows_pad, features if direct else None, w,
                                     segs, nseg, c_rows)
    out = torch.empty((kmap.n_out, c_out), dtype=dt, device=features.device)
    with _timed(timer, label, "scatter"):
        nat.call("scb_scatter", nat.ptr(partial), ldc, nat.ptr(plan.pos), plan.pos.shape[1],
                 kmap.n_out, c_out, center_row, nat.dtype_code(dt), nat.ptr(out), c_out,
                 *_epi_args(epilogue, kmap.n_out, c_out, dt), nat.stream_handle())
    if opts.traffic_log is not None:
        _record_traffic(opts, plan, c_in, c_out, dt, features.shape[0], kmap.n_out,
                        features.shape[0] if direct else 0, kmap.total)
    return out


def _pointwise_matmul(t: SparseTensor, w: WeightTensor, opts: ExecOptions, epilogue=None,
                      concat=None):
    """K=1, s=1 fast path (execution.py:472-477): out = features @ W[0]."""
    if choose_dataflow(opts, t.features.dtype, None, w) == "fused":
        return _run_fused(t.features, None, w, opts, epilogue, concat)
    f = t.features if concat is None else torch.cat([t.features, concat], dim=1)
    dt = f.dtype
    n = f.shape[0]
    n_rows = (n + nat.TILE_ROWS - 1) // nat.TILE_ROWS * nat.TILE_ROWS
    if _direct_center(dt, w.c_in):
        segs, nseg = _segments(GroupingStrategy(0, 0, (), (), False, 1), np.zeros(2, np.int64),
                               np.zeros(1, np.int64), [(0, 0, n, 0, 1)])
        partial, ldc = _grouped_gemm(dt, f, n, f, w, segs, nseg, n_rows)
    else:
        ld = _buffer_ld(dt, w.c_in)
        buf = torch.zeros((max(n_rows, 1), ld), dtype=dt, device=f.device)
        buf[:n, : w.c_in] = f
        segs, nseg = _segments(GroupingStrategy(0, 0, (), (), False, 1), np.zeros(2, np.int64),
                               np.zeros(1, np.int64), [(0, 0, n, 0, 0)])
        partial, ldc = _grouped_gemm(dt, buf, n_rows, None, w, segs, nseg, n_rows)
    out = torch.empty((n, w.c_out), dtype=dt, device=f.device)
    ident = _identity_pos(n, f.device)
    nat.call("scb_scatter", nat.ptr(partial), ldc, nat.ptr(ident), 1, n, w.c_out, -1,
             nat.dtype_code(dt), nat.ptr(out), w.c_out, *_epi_args(epilogue, n, w.c_out, dt),
             nat.stream_handle())
    return out


_IDENT = {}


def _identity_pos(n: int, device) -> torch.Tensor:
    t = _IDENT.get(device)
    if t is None or t.shape[0] < n:
        t = torch.arange(max(n, 1024) * 2, dtype=torch.int32, device=device).view(-1, 1)
        _IDENT[device] = t
    return t[:max(n, 1)]


def _record_workload(opts, spec, sizes, symmetric, schedule, in_coords, out_coords, boundary,
                     batch_size):
    if opts.workload_log is None:
        return
    opts.workload_log.append({
        "layer": opts.layer_label, "map_sizes": np.asarray(sizes, dtype=np.int64),
        "schedule": list(schedule), "symmetric": symmetric, "c_in": spec.c_in,
        "c_out": spec.c_out, "kernel_size": spec.kernel_size, "stride": spec.stride,
        "in_coords": in_coords, "out_coords": out_coords, "boundary": tuple(boundary),
        "batch_size": batch_size})


def _record_traffic(opts, plan, c_in, c_out, dtype, n_in, n_out, n_center, m_total):
    """Algorithmic bytes / FLOPs of one staged layer:
    e = storage bytes, p = 4 (f32 partials), int32 indices, padding rows
    excluded.  |M'| = plan.total (buffer rows), centre rows read in place."""
    e = 2 if dtype == torch.float16 else 4
    m = plan.total
    v = plan.volume
    opts.traffic_log.append((opts.layer_label, {
        "gather_bytes": e * n_in * c_in + e * m * c_in + 4 * m,
        "gemm_bytes": e * m * c_in + 4 * m * c_out + e * n_center * c_in
        + 4 * n_center * c_out + e * v * c_in * c_out,
        "gemm_flops": 2 * m_total * c_in * c_out,
        "scatter_bytes": 4 * m * c_out + e * n_out * c_out + 4 * m
        + 4 * n_center * c_out}))


def _check_channels(t, w, spec, msg=None, extra=0):
    c = t.num_channels + extra
    if c != spec.c_in or w.c_in != spec.c_in or w.c_out != spec.c_out:
        raise ValueError(msg or (
            f"channel mismatch: tensor {c}, spec {spec.c_in}->{spec.c_out}, "
            f"weights {w.c_in}->{w.c_out}"))


def _layer_maps(cset: CoordinateSet, spec: LayerSpec, strat: LayerStrategy,
                opts: ExecOptions) -> tuple[CoordinateSet, KernelMap]:
    """Output coordinate set and kernel map of a (non-transposed) layer over
    ``cset``, cached on the set under (K, stride, offset base) when
    ``opts.map_reuse`` (result-identical: maps depend on coordinates only)."""
    offsets = enumerate_offsets(len(cset.boundary), spec.kernel_size)
    kind = opts.index_kind or strat.index_kind or spec.index_kind or "auto"
    if kind == "grid" and _cells(cset.boundary, cset.batch_size) > opts.grid_cell_cap:
        raise GridCapacityError(
            f"grid index needs {_cells(cset.boundary, cset.batch_size)} cells "
            f"(cap {opts.grid_cell_cap}); use the hash index")
    dil = int(spec.dilation)
    key = (spec.kernel_size, spec.stride, offsets.base) + ((("dilation", dil),) if dil != 1 else ())
    hit = cset.maps.get(key) if opts.map_reuse else None
    if hit is None:
        if spec.stride == 1:
            out_cset = cset
        else:
            out_boundary = downsample_boundary(cset.boundary, spec.stride)
            oc = compute_output_coords(cset, offsets, spec.stride, out_boundary,
                                       cset.batch_size)
            out_cset = CoordinateSet(oc, out_boundary, cset.batch_size)
        index = build_index(cset, kind, cell_cap=opts.grid_cell_cap)
        pres = (cset.derived.get(("presence", spec.kernel_size))
                if spec.stride == 1 and dil == 1 else None)
        if pres is not None and offsets.center is not None and offsets.volume <= 32:
            # a presence-reordered level: probe only the present offsets
            kmap = map_search_masked(index, cset, offsets, pres)
        else:
            kmap = map_search(index, out_cset.coords, offsets, spec.stride, dilation=dil)
        # stride 1: the output set IS this set; store None, not a
        # self-reference (a cycle would pin the maps until the cyclic GC)
        hit = (None if out_cset is cset else out_cset, kmap)
        if opts.map_reuse:
            cset.maps[key] = hit
    out_cset, kmap = hit
    return (cset if out_cset is None else out_cset), kmap


def prepare_layer_maps(t, spec: LayerSpec, options: ExecOptions | None = None) -> CoordinateSet:
    """Build (and cache on the coordinate set) the maps a layer will use,
    without running it; returns the layer's output coordinate set.  B200
    extension: a model calls this for its strided layers before queueing any
    convolution, so the one host read per strided layer (the output
    coordinate count) happens while the GPU queue is empty and the forward
    itself issues without a host sync.  Result-identical."""
    opts = options or ExecOptions()
    if not opts.map_reuse:
        raise ValueError("prepared maps are kept in the map-reuse cache")
    cset = t.coordset if isinstance(t, SparseTensor) else t
    if spec.kernel_size == 1 and spec.stride == 1:
        return cset
    return _layer_maps(cset, spec, resolve_strategy(spec, None), opts)[0]


def prepare_strided_chain(t, specs, options: ExecOptions | None = None, *,
                          deferred: bool = False):
    """prepare_layer_maps for a chain of strided layers applied one after
    another (an encoder's downsampling path), with ONE host read for all
    output counts when every window proposes one candidate per input (K = s);
    otherwise level by level.  Returns the output coordinate set of each
    layer; maps are cached on the input sets as sparse_conv_forward would.
    Result-identical to running the layers.  ``deferred``: issue the chain
    and return a callable that finishes it (waits for the counts, builds the
    sets and maps) — queue other work in between so the host read costs no
    GPU idle time."""
    opts = options or ExecOptions()
    if not opts.map_reuse:
        raise ValueError("prepared maps are kept in the map-reuse cache")
    cset = t.coordset if isinstance(t, SparseTensor) else t
    if deferred:
        return _strided_chain(cset, specs, opts, True)
    return _strided_chain(cset, specs, opts, False)


def _strided_chain(cset, specs, opts, deferred):
    dim = len(cset.boundary)
    steps = [(enumerate_offsets(dim, sp.kernel_size), sp.stride) for sp in specs]
    chainable = all(sp.stride > 1 and sp.kernel_size == sp.stride for sp in specs)
    if not chainable or not specs:
        def sequential():
            out, cs = [], cset
            for sp in specs:
                cs = prepare_layer_maps(cs, sp, opts)
                out.append(cs)
            return out
        return sequential if deferred else sequential()
    finish = start_output_coords_chain(cset, steps)

    def build():
        return _chain_maps(cset, specs, steps, finish(), opts)
    return build if deferred else build()


def _chain_maps(cset, specs, steps, levels, opts):
    out, cs = [], cset
    for sp, (off, stride), (oc, ob) in zip(specs, steps, levels):
        key = (sp.kernel_size, stride, off.base)
        hit = cs.maps.get(key)
        if hit is None:
            nxt = CoordinateSet(oc, ob, cs.batch_size)
            kind = (opts.index_kind or (sp.strategy.index_kind if sp.strategy else None)
                    or sp.index_kind or "auto")
            index = build_index(cs, kind, cell_cap=opts.grid_cell_cap)
            cs.maps[key] = (nxt, map_search(index, nxt.coords, off, stride))
            hit = cs.maps[key]
        cs = hit[0]
        out.append(cs)
    return out


def link_strided_map(fine: CoordinateSet, coarse: CoordinateSet, spec: LayerSpec,
                     options: ExecOptions | None = None) -> KernelMap:
    """Cache on ``fine`` the map of the strided layer ``spec`` whose output
    coordinates are ``coarse`` (B200 extension): ``coarse`` must hold exactly
    compute_output_coords(fine, ...), in any row order — e.g. a presence-
    reordered level (mapping.reorder_by_presence).  The map is a plain map
    search over fine's index, so its pairs are the reference's under
    coarse's row numbering."""
    opts = options or ExecOptions()
    offsets = enumerate_offsets(len(fine.boundary), spec.kernel_size)
    key = (spec.kernel_size, spec.stride, offsets.base)
    hit = fine.maps.get(key)
    if hit is not None and hit[0] is coarse:
        return hit[1]
    kind = opts.index_kind or spec.index_kind or "auto"
    kmap = map_search(build_index(fine, kind, cell_cap=opts.grid_cell_cap), coarse.coords,
                      offsets, spec.stride)
    fine.maps[key] = (coarse, kmap)
    return kmap


def prepare_reordered_level(fine: CoordinateSet, spec: LayerSpec,
                            options: ExecOptions | None = None, reorder: bool = True
                            ) -> CoordinateSet:
    """Output coordinate set of the strided layer ``spec`` over ``fine``,
    relabelled by neighbour presence (reorder_by_presence) unless
    ``reorder`` is False, with the layer's map cached on ``fine``
    (B200 extension; one host read, the output count)."""
    opts = options or ExecOptions()
    offsets = enumerate_offsets(len(fine.boundary), spec.kernel_size)
    hit = fine.maps.get((spec.kernel_size, spec.stride, offsets.base))
    if hit is not None:
        return hit[0]
    ob = downsample_boundary(fine.boundary, spec.stride)
    out = CoordinateSet(compute_output_coords(fine, offsets, spec.stride, ob, fine.batch_size), ob,
                        fine.batch_size)
    if reorder:
        out = reorder_by_presence(out, 3, opts.index_kind or "auto")
    link_strided_map(fine, out, spec, opts)
    return out


class InflightLimiter:
    """Bounds how far the host runs ahead of the compute stream: a model
    records an event at the end of each forward, and the forward after next
    first waits (on the host) for it.  With maps built off the compute
    stream nothing else throttles the host, and every forward in flight
    holds its maps and activations in memory."""

    def __init__(self, depth: int = 2):
        self.depth = depth
        self.events: list[torch.cuda.Event] = []

    def before_forward(self) -> None:
        while len(self.events) >= self.depth:
            self.events.pop(0).synchronize()

    def after_forward(self) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self.events.append(ev)


def prepare_maps_on_stream(t, stream: torch.cuda.Stream, build, timer=None) -> None:
    """Run a model's map preparation ``build(coordset) -> [CoordinateSet]``
    on ``stream`` (B200 extension).  Maps depend on coordinates only, so a
    model can keep them off its compute stream: the next batch's mapping then
    overlaps this batch's convolutions, and the host reads it needs wait for
    mapping work only.  The compute (current) stream waits for the result,
    and every map tensor is recorded as in use by it."""
    cur = torch.cuda.current_stream()
    cs = t.coordset
    if stream is None or stream == cur:  # inline, on the compute stream
        with _timed(timer, "maps", "mapping"):
            build(cs)
        return
    if cs.stream is None or cs.stream != stream:
        stream.wait_stream(cur)  # coordinates produced on another stream: order after them
    with torch.cuda.stream(stream), _timed(timer, "maps", "mapping"):
        levels = build(cs)
    cur.wait_stream(stream)
    for lvl in levels:
        for x in lvl.device_tensors():
            x.record_stream(cur)


def sparse_conv_forward(t: SparseTensor, w: WeightTensor, spec: LayerSpec,
                        strategy: LayerStrategy | None = None, map_cache: dict | None = None,
                        options: ExecOptions | None = None, *,
                        epilogue: dict | None = None, concat=None) -> SparseTensor:
    """One sparse convolution layer on the B200 (execution.py:450-509).

    ``epilogue`` (B200 extension) fuses
    ``{"scale", "shift", "bias", "residual", "relu"}`` into the single write
    of each output row.  ``concat`` (B200 extension): a SparseTensor or
    feature matrix on the same coordinates whose channels follow ``t``'s —
    the layer input is their channel concatenation (a U-Net skip), which the
    fused kernel reads in place instead of materialising."""
    flush_saturation_warnings()
    opts = options or ExecOptions()
    cat = None
    if concat is not None:
        cat = concat.features if isinstance(concat, SparseTensor) else concat
        if cat.shape[0] != t.num_points or cat.dtype != t.features.dtype:
            raise ValueError("concat input must match the tensor's rows and dtype")
    _check_channels(t, w, spec, extra=0 if cat is None else cat.shape[1])
    label, timer = opts.layer_label, opts.timer
    strat = resolve_strategy(spec, strategy)
    if spec.kernel_size == 1 and spec.stride == 1:
        if choose_dataflow(opts, t.features.dtype, None, w) == "fused":
            out = _pointwise_matmul(t, w, opts, epilogue, cat)
        else:
            with _timed(timer, label, "matmul"):
                out = _pointwise_matmul(t, w, opts, epilogue, cat)
        _record_workload(opts, spec, np.array([t.num_points]), False, [0], t.coords, t.coords,
                         t.boundary, t.batch_size)
        return SparseTensor._wrap(out, t.stride, t.boundary, t.batch_size, t.coordset)

    offsets = enumerate_offsets(t.spatial_dims, spec.kernel_size)
    cset = t.coordset
    with _timed(timer, label, "mapping"):
        out_cset, kmap = _layer_maps(cset, spec, strat, opts)
        if map_cache is not None and spec.reuse_key:
            map_cache[spec.reuse_key] = CachedMap(kmap, t.coords, t.boundary, t.stride, cset)
    schedule, symmetric = schedule_for(offsets, spec.stride)
    center = offsets.center if (spec.stride == 1 and offsets.center is not None) else None
    record = lambda sizes: _record_workload(opts, spec, sizes, symmetric, schedule, t.coords,
                                            out_cset.coords, t.boundary, t.batch_size)
    out = _run_dataflow(t.features, kmap, w, strat, schedule, symmetric, opts, center, epilogue,
                        record, cat)
    with _timed(timer, label, "other"):  # result assembly (reference execution.py:503-508)
        return SparseTensor._wrap(out, t.stride * spec.stride, out_cset.boundary, t.batch_size,
                                  out_cset)


def inverse_conv_forward(t: SparseTensor, w: WeightTensor, spec: LayerSpec, map_cache: dict,
                         strategy: LayerStrategy | None = None,
                         options: ExecOptions | None = None, *,
                         epilogue: dict | None = None) -> SparseTensor:
    """Transposed layer replaying a cached strided map with roles swapped
    (execution.py:512-551)."""
    opts = options or ExecOptions()
    _check_channels(t, w, spec, "channel mismatch on inverse layer")
    if spec.reuse_key not in map_cache:
        raise KeyError(f"no cached map under reuse key {spec.reuse_key!r}")
    entry: CachedMap = map_cache[spec.reuse_key]
    if entry.kmap.n_out != t.num_points:
        raise ValueError("tensor does not match the cached map's output side")
    if entry.kmap.offsets.kernel_size != spec.kernel_size:
        raise ValueError("kernel size differs from the cached map")
    label, timer = opts.layer_label, opts.timer
    strat = resolve_strategy(spec, strategy)
    with _timed(timer, label, "mapping"):
        swapped = entry.kmap.swap_roles()
    schedule = list(range(swapped.offsets.volume))
    record = lambda sizes: _record_workload(opts, spec, sizes, False, schedule, t.coords,
                                            entry.in_coords, entry.in_boundary, t.batch_size)
    out = _run_dataflow(t.features, swapped, w, strat, schedule, False, opts, None, epilogue,
                        record)
    with _timed(timer, label, "other"):  # result assembly (reference execution.py:545-550)
        cset = entry.in_coordset or CoordinateSet(entry.in_coords, entry.in_boundary,
                                                  t.batch_size)
        return SparseTensor._wrap(out, entry.in_stride, tuple(entry.in_boundary), t.batch_size,
                                  cset)


_POINTWISE = {"relu": 0, "bias_add": 1, "bn_fold": 2}


def _param(x, c, name):
    if x is None:
        raise ValueError(f"{name} is required")
    a = np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x, dtype=np.float32)
    if a.shape != (c,):
        raise ValueError(f"{name} length must match the channel count")
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def pointwise_apply(t: SparseTensor, op: str, *, bias=None, scale=None,
                    shift=None) -> SparseTensor:
    """relu / bias_add / bn_fold on the device (execution.py:554-576)."""
    if op not in _POINTWISE:
        raise ValueError(f"unknown pointwise op {op!r}")
    c = t.num_channels
    a = b = None
    if op == "bias_add":
        try:
            a = _param(bias, c, "bias")
        except ValueError:
            raise ValueError("bias length must match the channel count")
    elif op == "bn_fold":
        try:
            a, b = _param(scale, c, "scale"), _param(shift, c, "shift")
        except ValueError:
            raise ValueError("scale/shift length must match the channel count")
    out = t.features.clone()
    nat.call("scb_pointwise", nat.dtype_code(out.dtype), nat.ptr(out), out.shape[0], c,
             _POINTWISE[op], nat.ptr(a), nat.ptr(b), nat.stream_handle())
    return t.replace_features(out)
