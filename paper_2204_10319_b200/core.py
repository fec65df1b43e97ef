"""Device-resident core types: the drop-in twins of the reference's
``SparseTensor``, ``WeightTensor`` and ``PrecisionMode`` (reference
``core.py:25-171``) plus ``quantize_features`` (``core.py:219-238``).

A ``SparseTensor`` here keeps its coordinates as an int32 ``(N, 1+D)`` CUDA
tensor (batch column first) and its features as an ``(N, C)`` float16/float32
CUDA tensor.  It accepts the reference's numpy inputs unchanged.  Tensors
that share a coordinate set (every stride-1 layer output) share one
``CoordinateSet``, which owns the device index and the kernel maps built
over it, so maps are built once per level — results
are identical to rebuilding them, as the reference does.
"""

from __future__ import annotations

import warnings
from enum import Enum

import numpy as np
import torch

from . import _native as nat

FP16_MAX = float(np.finfo(np.float16).max)


class PrecisionMode(Enum):
    """Feature storage precision (reference core.py:25-43).  Reductions always
    run in at least 32-bit."""

    FP32 = "fp32"
    FP16_STORAGE = "fp16"

    @property
    def storage_dtype(self) -> np.dtype:
        return np.dtype(np.float16) if self is PrecisionMode.FP16_STORAGE else np.dtype(np.float32)

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.float16 if self is PrecisionMode.FP16_STORAGE else torch.float32

    @property
    def element_bytes(self) -> int:
        return self.storage_dtype.itemsize


def flatten_coords(coords, boundary, batch_size: int = 1):
    """Batch-major flat key (reference core.py:46-66), numpy or torch."""
    total = int(batch_size)
    for b in boundary:
        if int(b) <= 0:
            raise ValueError("boundary extents must be positive")
        total *= int(b)
    if total >= 1 << 62:
        raise ValueError("coordinate space too large to key into int64")
    if isinstance(coords, torch.Tensor):
        c = coords.to(torch.int64)
        key = c[:, 0].clone()
    else:
        c = np.asarray(coords, dtype=np.int64)
        key = c[:, 0].copy()
    for d, b in enumerate(boundary):
        key = key * int(b) + c[:, d + 1]
    return key


def unflatten_coords(keys, boundary, batch_size: int = 1):
    """Inverse of :func:`flatten_coords` (reference core.py:69-79)."""
    is_t = isinstance(keys, torch.Tensor)
    rem = keys.to(torch.int64).clone() if is_t else np.asarray(keys, dtype=np.int64).copy()
    cols = [None] * (len(boundary) + 1)
    for d in range(len(boundary) - 1, -1, -1):
        cols[d + 1] = rem % int(boundary[d])
        rem = rem // int(boundary[d])
    cols[0] = rem
    return torch.stack(cols, 1) if is_t else np.stack(cols, 1)


class _PinnedRing:
    """Small pinned host buffers for asynchronous device->host reads of
    counts, reused round-robin (a fresh pinned allocation per read costs
    ~0.1 ms of host time at the start of every forward).  A slot is busy from
    ``take`` until its consumer calls ``release`` after reading it (deferred
    readers -- saturation warnings, async validation, the coordinate-chain
    finisher -- may read long after the copy landed); ``take`` skips busy
    slots and falls back to a fresh pinned buffer when all are busy."""

    def __init__(self, slots: int = 64, words: int = 16):
        self.buf = None
        self.busy = [False] * slots
        self.slots, self.words, self.next = slots, words, 0

    def take(self, n: int, dtype) -> torch.Tensor:
        if n * torch.empty((), dtype=dtype).element_size() > self.words * 8:
            return torch.empty(n, dtype=dtype, pin_memory=True)
        if self.buf is None:
            self.buf = torch.empty(self.slots * self.words, dtype=torch.int64, pin_memory=True)
        for _ in range(self.slots):
            i = self.next
            self.next = (i + 1) % self.slots
            if not self.busy[i]:
                self.busy[i] = True
                return self.buf[i * self.words:(i + 1) * self.words].view(dtype)[:n]
        return torch.empty(n, dtype=dtype, pin_memory=True)  # every slot still unread

    def read_async(self, src: torch.Tensor, n: int | None = None):
        """Start a read of ``src`` (a small device tensor, 4-byte elements
        or wider) into a pinned slot: the SMs write it through the slot's
        host pointer (scb_store_to_host), not a DMA copy, so it never waits
        behind a large transfer on the copy engine.  Returns (host view,
        event); read the view after ``event.synchronize()``, then
        ``release`` it."""
        n = src.numel() if n is None else n
        host = self.take(n, src.dtype)
        src = src.contiguous()
        nat.call("scb_store_to_host", nat.ptr(src), host.data_ptr(), n * src.element_size(),
                 nat.stream_handle())
        ev = torch.cuda.Event()
        ev.record()
        return host, ev

    def _slot(self, t: torch.Tensor):
        if self.buf is not None and t.untyped_storage().data_ptr() == \
                self.buf.untyped_storage().data_ptr():
            return (t.data_ptr() - self.buf.data_ptr()) // (self.words * 8)
        return None

    def release(self, t: torch.Tensor) -> None:
        """The consumer has read ``t``: its slot may be reused."""
        i = self._slot(t)
        if i is not None:
            self.busy[i] = False


PINNED = _PinnedRing()


def _device() -> torch.device:
    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def as_device_coords(coords) -> torch.Tensor:
    dev = _device()
    if isinstance(coords, torch.Tensor):
        return coords.to(device=dev, dtype=torch.int32).contiguous()
    arr = np.asarray(coords)
    if arr.size and (arr.max() > np.iinfo(np.int32).max or arr.min() < np.iinfo(np.int32).min):
        raise ValueError("coordinates exceed the int32 range of the device layout")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(dev)


def as_device_features(features) -> torch.Tensor:
    dev = _device()
    if isinstance(features, torch.Tensor):
        f = features.to(dev)
    else:
        f = torch.from_numpy(np.ascontiguousarray(features)).to(dev)
    if f.dtype not in (torch.float16, torch.float32):
        f = f.to(torch.float32)
    return f.contiguous()


class CoordinateSet:
    """One coordinate set on the device plus everything derived from it:
    indexes by kind and kernel maps by (kernel_size, stride) — the
    level-keyed map cache."""

    __slots__ = ("coords", "boundary", "batch_size", "indexes", "maps", "stream", "perm",
                 "derived", "__weakref__")

    def __init__(self, coords: torch.Tensor, boundary, batch_size: int, perm=None):
        self.coords = coords
        self.boundary = tuple(int(b) for b in boundary)
        self.batch_size = int(batch_size)
        self.indexes = {}
        self.maps = {}
        self.derived = {}   # reordered twins of this set (mapping.reorder_by_presence)
        # reordered set (mapping.reorder_by_presence): row i is row perm[i]
        # of the set it was derived from; None for sets in their own order
        self.perm = perm
        # the stream the coordinates were produced on (a model may continue
        # the mapping work there, off its compute stream)
        self.stream = torch.cuda.current_stream() if torch.cuda.is_available() else None

    def device_tensors(self):
        """Every device tensor owned by this set, its indexes and its maps
        (for Tensor.record_stream when another stream consumes them)."""
        out = [self.coords] + ([self.perm] if self.perm is not None else [])
        for idx in self.indexes.values():
            out += [t for t in (getattr(idx, "keys", None), getattr(idx, "rows", None),
                                getattr(idx, "_status", None)) if isinstance(t, torch.Tensor)]
        for _, kmap in self.maps.values():
            out += kmap.device_tensors()
        return out

    @property
    def num_points(self) -> int:
        return int(self.coords.shape[0])


class SparseTensor:
    """Unique integer coordinates paired with a feature row each
    (reference core.py:82-143), resident in HBM."""

    __slots__ = ("coords", "features", "stride", "boundary", "batch_size", "_cset")

    def __init__(self, coords, features, stride: int = 1, boundary=(), batch_size: int = 1,
                 *, validate: bool = True, coordset: CoordinateSet | None = None):
        boundary = tuple(int(b) for b in boundary)
        if coordset is not None:
            c = coordset.coords
        else:
            c = as_device_coords(coords)
        f = as_device_features(features)
        if c.ndim != 2 or c.shape[1] != 1 + len(boundary):
            raise ValueError(
                f"coords shape {tuple(c.shape)} does not match boundary of rank {len(boundary)}")
        if not 1 <= len(boundary) <= 4:
            raise ValueError("spatial rank must be between 1 and 4")
        if f.ndim != 2 or f.shape[0] != c.shape[0]:
            raise ValueError("feature rows must match coordinate rows")
        if int(stride) < 1:
            raise ValueError("stride must be a positive integer")
        if coordset is None:
            coordset = CoordinateSet(c, boundary, batch_size)
            if validate == "async" and c.shape[0]:
                _validate_async(coordset)
            elif validate and c.shape[0]:
                _validate(coordset)
        self.coords = c
        self.features = f
        self.stride = int(stride)
        self.boundary = boundary
        self.batch_size = int(batch_size)
        self._cset = coordset

    @classmethod
    def _wrap(cls, features: torch.Tensor, stride: int, boundary: tuple, batch_size: int,
              coordset: CoordinateSet) -> "SparseTensor":
        """Engine-internal constructor for layer outputs: the features are a
        fresh device tensor with one row per coordinate of ``coordset`` (no
        checks, no copies)."""
        t = object.__new__(cls)
        t.coords = coordset.coords
        t.features = features
        t.stride = stride
        t.boundary = boundary
        t.batch_size = batch_size
        t._cset = coordset
        return t

    # -- reference API --------------------------------------------------
    @property
    def num_points(self) -> int:
        return int(self.coords.shape[0])

    @property
    def num_channels(self) -> int:
        return int(self.features.shape[1])

    @property
    def spatial_dims(self) -> int:
        return len(self.boundary)

    def replace_features(self, features) -> "SparseTensor":
        """Same coordinates (and coordinate set), new feature matrix."""
        if (isinstance(features, torch.Tensor) and features.is_cuda and features.ndim == 2
                and features.dtype in (torch.float16, torch.float32)
                and features.shape[0] == self.coords.shape[0] and features.is_contiguous()):
            return SparseTensor._wrap(features, self.stride, self.boundary, self.batch_size,
                                      self._cset)
        return SparseTensor(None, features, self.stride, self.boundary, self.batch_size,
                            coordset=self._cset)

    # -- host views (tests, I/O) ------------------------------------------
    def coords_numpy(self) -> np.ndarray:
        out = self.coords.cpu().numpy().astype(np.int64)
        flush_saturation_warnings(block=True)
        return out

    def features_numpy(self) -> np.ndarray:
        out = self.features.cpu().numpy()
        flush_saturation_warnings(block=True)
        return out

    @property
    def coordset(self) -> CoordinateSet:
        return self._cset


_PENDING_VALIDATION: list = []


def _validate_async(cset: CoordinateSet) -> None:
    """``validate="async"`` (B200 extension for pipelined serving): the same
    device checks as ``_validate``, but the two counts come back through
    pinned memory and an event; the error is raised at the next engine host
    synchronisation (the forward's coordinate-pyramid read) or by
    :func:`flush_validation`, instead of stalling the constructor on the
    previous batch's queued work."""
    from .mapping import build_index
    idx = build_index(cset, "hash")
    host, ev = PINNED.read_async(idx._status, 2)
    _PENDING_VALIDATION.append((ev, host, cset))


def flush_validation() -> None:
    """Raise the reference's ValueError for any pending asynchronous
    validation that failed (waits for those checks only)."""
    pending = list(_PENDING_VALIDATION)
    _PENDING_VALIDATION.clear()
    for ev, host, cset in pending:
        ev.synchronize()
        dup, oob = (int(x) for x in host.tolist())
        PINNED.release(host)
        if oob:
            c = cset.coords
            b = c[:, 0]
            if int(b.min()) < 0 or int(b.max()) >= cset.batch_size:
                raise ValueError("batch index out of range")
            raise ValueError("coordinate outside boundary")
        if dup:
            raise ValueError("coordinate rows must be unique")


def _validate(cset: CoordinateSet) -> None:
    """Range and uniqueness checks of reference core.py:112-120, on device:
    building the hash index (which the first layer reuses) counts duplicate
    and out-of-range rows; one host read of the two counts."""
    from .mapping import build_index  # local import: mapping depends on core
    idx = build_index(cset, "hash")
    dup, oob = (int(x) for x in idx._status.tolist())
    if oob:  # rare: find which check failed for the reference's message
        c = cset.coords
        b = c[:, 0]
        if int(b.min()) < 0 or int(b.max()) >= cset.batch_size:
            raise ValueError("batch index out of range")
        raise ValueError("coordinate outside boundary")
    if dup:
        raise ValueError("coordinate rows must be unique")


class WeightTensor:
    """Convolution weights, one C_in x C_out matrix per kernel offset
    (reference core.py:146-171).  Keeps the reference's f32 host array and
    lazily materialises the device copies the kernels need: f32
    ``(V, C_in, C_out)`` for the FP32 path and the K-major padded fp16 pack of
    the tcgen05 path."""

    __slots__ = ("weights", "kernel_size", "dim", "_dev32", "_packed", "_packed_vk")

    def __init__(self, weights, kernel_size: int, dim: int):
        if isinstance(weights, torch.Tensor):
            weights = weights.detach().cpu().numpy()
        w = np.ascontiguousarray(weights, dtype=np.float32)
        if w.ndim != 3:
            raise ValueError("weights must be a (K**D, C_in, C_out) stack")
        if w.shape[0] != kernel_size ** dim:
            raise ValueError(f"expected {kernel_size ** dim} weight slices, got {w.shape[0]}")
        w.setflags(write=False)
        self.weights = w
        self.kernel_size = int(kernel_size)
        self.dim = int(dim)
        self._dev32 = None
        self._packed = None
        self._packed_vk = {}

    @property
    def c_in(self) -> int:
        return self.weights.shape[1]

    @property
    def c_out(self) -> int:
        return self.weights.shape[2]

    def device_f32(self) -> torch.Tensor:
        if self._dev32 is None:
            self._dev32 = torch.from_numpy(np.array(self.weights)).to(_device())
        return self._dev32

    def packed_f16(self) -> tuple[torch.Tensor, int, int]:
        """[V][n_pad][k_pad] fp16 (transposed, zero padded) + (k_pad, n_pad)."""
        if self._packed is None:
            v, ci, co = self.weights.shape
            k_pad, n_pad = (ci + 15) // 16 * 16, (co + 15) // 16 * 16
            out = torch.empty((v, n_pad, k_pad), dtype=torch.float16, device=_device())
            nat.call("scb_pack_weights_f16", nat.ptr(self.device_f32()), v, ci, co, nat.ptr(out),
                     k_pad, n_pad, nat.stream_handle())
            self._packed = (out, k_pad, n_pad)
        return self._packed

    def packed_vk_f16(self, c_kernel: int) -> torch.Tensor:
        """[n_pad][ceil64(V c_kernel)] fp16, K-major over the offset-major
        channel concatenation (virtual K; scb_conv_implicit_vk): element
        (col, n c_kernel + ci) = W[n][ci][col], zero for ci >= C_in (padded
        input channels) and past V c_kernel.  A one-time layout transform."""
        cache = self._packed_vk
        if c_kernel not in cache:
            v, ci, co = self.weights.shape
            n_pad = (co + 15) // 16 * 16
            kv = (v * c_kernel + 63) // 64 * 64
            w = torch.zeros((v, c_kernel, n_pad), dtype=torch.float32, device=_device())
            w[:, :ci, :co] = self.device_f32()
            flat = torch.zeros((kv, n_pad), dtype=torch.float32, device=_device())
            flat[: v * c_kernel] = w.reshape(v * c_kernel, n_pad)
            cache[c_kernel] = flat.t().contiguous().to(torch.float16)
        return cache[c_kernel]


def voxelize(points, voxel_size: float, reduce: str = "mean",
             spatial_dims: int = 3) -> SparseTensor:
    """Quantize a raw point cloud onto the voxel lattice on the device
    (reference core.py:174-216, same errors): cells = floor((p - min) /
    voxel_size), duplicates merged by the f64 mean or the first point, rows
    in ascending flat-key order — bit-exact with the reference.  ``points``:
    (n, cols) array or tensor (host or device), first ``spatial_dims``
    columns are positions.  One host read (the voxel count and boundary)."""
    if isinstance(points, torch.Tensor):
        p = points.to(device=_device(), dtype=torch.float64).contiguous()
    else:
        arr = np.asarray(points, dtype=np.float64)
        p = torch.from_numpy(np.ascontiguousarray(arr)).to(_device())
    if p.ndim != 2 or p.shape[0] == 0:
        raise ValueError("empty cloud")
    if p.shape[1] < spatial_dims:
        raise ValueError(f"points need at least {spatial_dims} columns")
    if voxel_size <= 0:
        raise ValueError("voxel_size must be positive")
    if reduce not in ("mean", "first"):
        raise ValueError(f"unknown reduce {reduce!r}")
    n, cols = p.shape
    lib = nat.load()
    ws = torch.empty(int(lib.scb_voxelize_workspace(n, spatial_dims)), dtype=torch.uint8,
                     device=p.device)
    coords = torch.empty((n, 1 + spatial_dims), dtype=torch.int32, device=p.device)
    feats = torch.empty((n, cols - spatial_dims), dtype=torch.float32, device=p.device)
    meta = torch.empty(1 + spatial_dims, dtype=torch.int64, device=p.device)
    nat.call("scb_voxelize", nat.ptr(p), n, cols, spatial_dims, float(voxel_size),
             int(reduce == "first"), nat.ptr(ws), ws.numel(), nat.ptr(coords),
             nat.ptr(feats) if feats.numel() else None, nat.ptr(meta), nat.stream_handle())
    m = meta.tolist()
    nv = int(m[0])
    boundary = tuple(int(b) for b in m[1:])
    c = coords[:nv]
    cset = CoordinateSet(c, boundary, 1)
    return SparseTensor._wrap(feats[:nv], 1, boundary, 1, cset)


def voxelize_batch(scans, voxel_size: float, reduce: str = "mean",
                   spatial_dims: int = 3) -> SparseTensor:
    """B raw scans -> one packed SparseTensor on the device in one pass
    (``scb_voxelize_batch``; B200 extension of reference core.py:174-216):
    scan b is voxelised exactly as :func:`voxelize` voxelises it alone (its
    own min corner, f64 cells and means), its rows get batch column b, and
    the boundary is the per-dimension max over the scans — bit-identical to
    B ``voxelize`` calls packed along the batch column.
    ``scans``: a list of (n_b, cols) arrays or tensors (host or device), or
    one (n, cols) tensor plus ``scans=(points, scan_ptr)``.  One host read
    (voxel count and boundary)."""
    if isinstance(scans, tuple) and len(scans) == 2 and isinstance(scans[0], torch.Tensor):
        p = scans[0].to(device=_device(), dtype=torch.float64).contiguous()
        ptr = torch.as_tensor(scans[1], dtype=torch.int64).to(p.device)
        B = int(ptr.shape[0]) - 1
    else:
        parts = [torch.as_tensor(np.asarray(x, dtype=np.float64)) if not isinstance(x, torch.Tensor)
                 else x.to(torch.float64) for x in scans]
        if not parts:
            raise ValueError("empty cloud")
        cols = {int(x.shape[1]) if x.ndim == 2 else -1 for x in parts}
        if len(cols) != 1 or -1 in cols:
            raise ValueError("every scan must be an (n, cols) array with the same columns")
        if any(x.shape[0] == 0 for x in parts):
            raise ValueError("empty cloud")
        B = len(parts)
        sizes = np.array([0] + [int(x.shape[0]) for x in parts], dtype=np.int64)
        ptr = torch.from_numpy(np.cumsum(sizes)).to(_device())
        p = torch.cat([x.cpu() if not x.is_cuda else x for x in parts]).to(_device()).contiguous() \
            if not all(x.is_cuda for x in parts) else torch.cat(parts).contiguous()
    if not 1 <= B <= 64:
        raise ValueError("1..64 scans per batch")
    if p.ndim != 2 or p.shape[0] == 0:
        raise ValueError("empty cloud")
    if p.shape[1] < spatial_dims:
        raise ValueError(f"points need at least {spatial_dims} columns")
    if voxel_size <= 0:
        raise ValueError("voxel_size must be positive")
    if reduce not in ("mean", "first"):
        raise ValueError(f"unknown reduce {reduce!r}")
    n, cols = p.shape
    lib = nat.load()
    ws = torch.empty(int(lib.scb_voxelize_workspace(n, spatial_dims)), dtype=torch.uint8,
                     device=p.device)
    coords = torch.empty((n, 1 + spatial_dims), dtype=torch.int32, device=p.device)
    feats = torch.empty((n, cols - spatial_dims), dtype=torch.float32, device=p.device)
    meta = torch.empty(1 + spatial_dims, dtype=torch.int64, device=p.device)
    nat.call("scb_voxelize_batch", nat.ptr(p), nat.ptr(ptr), B, n, cols, spatial_dims,
             float(voxel_size), int(reduce == "first"), nat.ptr(ws), ws.numel(), nat.ptr(coords),
             nat.ptr(feats) if feats.numel() else None, nat.ptr(meta), nat.stream_handle())
    m = meta.tolist()
    nv = int(m[0])
    boundary = tuple(int(b) for b in m[1:])
    cset = CoordinateSet(coords[:nv], boundary, B)
    return SparseTensor._wrap(feats[:nv], 1, boundary, B, cset)


def quantize_features(t: SparseTensor, mode: PrecisionMode) -> SparseTensor:
    """Convert feature storage precision (reference core.py:219-238): FP16
    rounds to nearest and saturates to +-65504 with a warning."""
    if mode is PrecisionMode.FP32:
        if t.features.dtype == torch.float32:
            return t
        return t.replace_features(t.features.to(torch.float32))
    if t.features.dtype == torch.float16:
        return t
    src = t.features.contiguous()
    out = torch.empty(src.shape, dtype=torch.float16, device=src.device)
    sat = torch.zeros(1, dtype=torch.int64, device=src.device)
    nat.call("scb_quantize_f16", nat.ptr(src), nat.ptr(out), src.numel(), nat.ptr(sat),
             nat.stream_handle())
    # The saturation count comes back asynchronously (pinned copy + event) so
    # quantising a network input does not stall the stream; the warning is
    # raised as soon as the count is known (next engine call, or any host read).
    host, ev = PINNED.read_async(sat, 1)
    _PENDING_SATURATION.append((ev, host))
    return t.replace_features(out)


_PENDING_SATURATION: list = []


def flush_saturation_warnings(block: bool = False) -> None:
    """Emit the fp16 saturation warnings of finished quantisations
    (reference core.py:232-237)."""
    keep = []
    for ev, host in _PENDING_SATURATION:
        if block:
            ev.synchronize()
        if block or ev.query():
            n_sat = int(host.item())
            PINNED.release(host)
            if n_sat:
                warnings.warn(f"{n_sat} feature element(s) saturated to the fp16 range")
        else:
            keep.append((ev, host))
    _PENDING_SATURATION[:] = keep
