"""``sparseconv.mapping`` on the B200 engine (reference ``mapping.py``).

Indexes are device hash tables / grids (``scb_index_build``), output
coordinates come from the fused candidate kernel + radix sort
(``scb_output_coords``), maps from ``scb_map_search`` — bit-exact with the
reference — and are handed back as the reference's per-offset numpy
``pairs``.  A :class:`KernelMap` built from host pairs (the reference's
tests do this) is uploaded as a CSR map on first device use.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2204_10319_b200 import mapping as _eng

from .core import SparseTensor

MISS = _eng.MISS
DEFAULT_GRID_CELL_CAP = _eng.DEFAULT_GRID_CELL_CAP
EVEN_KERNEL_OFFSET_BASE = _eng.EVEN_KERNEL_OFFSET_BASE
GridCapacityError = _eng.GridCapacityError
KernelOffsets = _eng.KernelOffsets
enumerate_offsets = _eng.enumerate_offsets
downsample_boundary = _eng.downsample_boundary


def _coords_of(x) -> np.ndarray:
    if isinstance(x, SparseTensor):
        return x.coords
    return np.asarray(x, dtype=np.int64)


class _Index:
    """A device coordinate index behind the reference's host interface
    (``kind``, ``boundary``, ``batch_size``, ``size``, ``query``)."""

    kind = "?"

    def _attach(self, dev) -> None:
        self._dev = dev
        self.boundary = tuple(dev.boundary)
        self.batch_size = int(dev.batch_size)
        self.size = int(dev.size)
        self._bounds = np.asarray(self.boundary, dtype=np.int64)

    def query(self, coords) -> np.ndarray:
        """Row per query coordinate; MISS (-1) where absent or out of
        bounds (``scb_index_query``)."""
        q = np.asarray(coords, dtype=np.int64)
        if q.shape[0] == 0:
            return np.empty(0, dtype=np.int64)
        return self._dev.query(q).cpu().numpy().astype(np.int64)


class GridIndex(_Index):
    """Dense device table over batch x boundary (reference mapping.py:82-119)."""

    kind = "grid"

    def __init__(self, coords, boundary, batch_size: int = 1,
                 cell_cap: int = DEFAULT_GRID_CELL_CAP):
        self._attach(_eng.build_index(_coords_of(coords), "grid", boundary, batch_size, cell_cap))


class HashIndex(_Index):
    """Open-addressing device table keyed by the flat coordinate, load factor
    <= 0.5, power-of-two size (reference mapping.py:122-189).  ``_mask`` is
    the table's slot mask, as in the reference."""

    kind = "hash"

    def __init__(self, coords, boundary, batch_size: int = 1):
        self._attach(_eng.build_index(_coords_of(coords), "hash", boundary, batch_size))
        self._mask = int(self._dev.slots) - 1


def build_index(coords, kind: str, boundary, batch_size: int = 1,
                cell_cap: int = DEFAULT_GRID_CELL_CAP):
    """``grid``, ``hash`` or ``auto`` (reference mapping.py:195-208; the
    device grid additionally stops at 2^27 cells, maps are identical)."""
    dev = _eng.build_index(_coords_of(coords), kind, boundary, batch_size, cell_cap)
    idx = object.__new__(GridIndex if dev.kind == "grid" else HashIndex)
    idx._attach(dev)
    if dev.kind == "hash":
        idx._mask = int(dev.slots) - 1
    return idx


CoordinateIndex = GridIndex | HashIndex


def compute_output_coords(in_coords, offsets: KernelOffsets, stride: int, out_boundary,
                          batch_size: int = 1, chunk: int | None = None) -> np.ndarray:
    """Active output coordinates in ascending flat-key order (reference
    mapping.py:216-248).  ``chunk`` bounded the reference's host memory;
    the device pass sizes its workspace itself, so it only is checked."""
    if chunk is not None and chunk < 1:
        raise ValueError("chunk must be positive")
    c = _coords_of(in_coords)
    if stride == 1:
        return c
    if c.shape[0] == 0:
        return np.empty((0, c.shape[1]), dtype=np.int64)
    out = _eng.compute_output_coords(c, offsets, stride, tuple(out_boundary), batch_size)
    return out.cpu().numpy().astype(np.int64)


class KernelMap:
    """Per-offset lists of (input row, output row) pairs (reference
    mapping.py:251-286).  ``pairs`` are host arrays; ``_dev`` is the engine
    map (hit matrix and/or CSR in HBM) they came from or were uploaded to."""

    def __init__(self, pairs, offsets: KernelOffsets, stride: int, n_in: int, n_out: int,
                 symmetric: bool = False):
        self.pairs = [np.asarray(p, dtype=np.int64).reshape(-1, 2) for p in pairs]
        self.offsets = offsets
        self.stride = int(stride)
        self.n_in = int(n_in)
        self.n_out = int(n_out)
        self.symmetric = bool(symmetric)
        self._dev = None

    @classmethod
    def _from_engine(cls, dev) -> "KernelMap":
        m = cls(dev.pairs, dev.offsets, dev.stride, dev.n_in, dev.n_out, dev.symmetric)
        m._dev = dev
        return m

    def _engine(self):
        """The engine map: uploaded once as a CSR (offset_ptr, in, out)."""
        if self._dev is None:
            device = torch.device("cuda", torch.cuda.current_device())
            sizes = self.sizes
            ptr = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
            np.cumsum(sizes, out=ptr[1:])
            st = np.concatenate(self.pairs, 0) if self.pairs else np.empty((0, 2), np.int64)
            if st.shape[0] and (st[:, 0].min() < 0 or st[:, 0].max() >= self.n_in
                                or st[:, 1].min() < 0 or st[:, 1].max() >= self.n_out):
                raise ValueError("kernel map entry outside the input/output row range")
            tens = [torch.from_numpy(np.ascontiguousarray(a)).to(device)
                    for a in (ptr, st[:, 0].astype(np.int32), st[:, 1].astype(np.int32))]
            self._dev = _eng.KernelMap(tens[0], sizes, tens[1], tens[2], self.offsets,
                                       self.stride, self.n_in, self.n_out, self.symmetric)
        return self._dev

    @property
    def sizes(self) -> np.ndarray:
        return np.array([p.shape[0] for p in self.pairs], dtype=np.int64)

    @property
    def buffer_offsets(self) -> np.ndarray:
        out = np.zeros(len(self.pairs) + 1, dtype=np.int64)
        np.cumsum(self.sizes, out=out[1:])
        return out

    @property
    def total(self) -> int:
        return int(self.sizes.sum())

    def swap_roles(self) -> "KernelMap":
        """Roles exchanged, entries re-sorted by the new output row
        (``scb_map_transpose``)."""
        return KernelMap._from_engine(self._engine().swap_roles())


def map_search(in_index, out_coords, offsets: KernelOffsets, stride: int,
               use_symmetry: bool | None = None) -> KernelMap:
    """Kernel map search (reference mapping.py:289-319) with
    ``scb_map_search``; symmetric stride-1 odd-K maps probe the lower half
    and fill the mirror in the same pass."""
    oc = _coords_of(out_coords)
    dev = in_index._dev if isinstance(in_index, _Index) else in_index
    return KernelMap._from_engine(_eng.map_search(dev, oc, offsets, stride, use_symmetry))


def derive_symmetric_maps(half_map: KernelMap) -> KernelMap:
    """Complete a stride-1 odd-K map from its lower half (reference
    mapping.py:322-339); the device transposes the hit matrix."""
    if half_map.stride != 1:
        raise ValueError("symmetric maps exist only for stride-1 layers")
    return KernelMap._from_engine(_eng.derive_symmetric_maps(half_map._engine()))


class GatherScatterPlan:
    """The device plan (128-row-aligned slabs, output-stationary position
    table) with the reference's host views (reference mapping.py:342-374):
    ``n_in``, ``n_out``, ``total``, ``row_input``, ``row_output``,
    ``buffer_offsets``, ``in_indptr``, ``in_rows``, ``out_indptr``,
    ``out_rows``, ``skipped_offset``, ``sizes``, ``in_counts``,
    ``out_counts``.  Holds its kernel map."""

    def __init__(self, dev, kmap: KernelMap):
        self._dev = dev
        self._kmap = kmap
        self._kmap_dev = kmap._engine()

    def __getattr__(self, name):
        if name.startswith("__"):
            raise AttributeError(name)
        return getattr(self._dev, name)


def build_gather_scatter_plan(kmap: KernelMap, skip_center: bool = False) -> GatherScatterPlan:
    """Buffer layout + both stationary indexes (reference mapping.py:377-418)
    with ``scb_plan_build``."""
    if skip_center and (kmap.offsets.center is None or kmap.stride != 1):
        raise ValueError("skip_center requires a stride-1 odd-K map")
    return GatherScatterPlan(_eng.build_gather_scatter_plan(kmap._engine(), skip_center), kmap)


class _ForwardingModule(type(_eng)):
    """Module attributes that steer the engine are forwarded to it, so
    ``monkeypatch.setattr(sparseconv.mapping, "EVEN_KERNEL_OFFSET_BASE", -1)``
    (the reference's negative control, tests/test_network.py) changes the
    offsets the device kernels enumerate, as it does in the reference."""

    _FORWARDED = ("EVEN_KERNEL_OFFSET_BASE",)

    def __setattr__(self, name, value):
        if name in self._FORWARDED:
            setattr(_eng, name, value)
        super().__setattr__(name, value)


import sys as _sys  # noqa: E402

_sys.modules[__name__].__class__ = _ForwardingModule

__all__ = [
    "MISS", "DEFAULT_GRID_CELL_CAP", "EVEN_KERNEL_OFFSET_BASE", "GridCapacityError",
    "KernelOffsets", "enumerate_offsets", "downsample_boundary", "GridIndex", "HashIndex",
    "CoordinateIndex", "build_index", "compute_output_coords", "KernelMap", "map_search",
    "derive_symmetric_maps", "GatherScatterPlan", "build_gather_scatter_plan",
]
