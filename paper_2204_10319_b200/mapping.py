"""Kernel-map construction on the device: the drop-in twin of the reference's
``mapping.py`` (offsets, indexes, output coordinates, map search, symmetric
maps, gather/scatter plans).  Every function here enqueues sm_100a kernels
from ``libsparseconv_b200.so``; the host only handles shapes and the one
data-dependent size per map.

Map entries follow the reference convention: entry ``(j, k)`` of offset ``n``
means input coordinate ``p_j == stride * q_k + delta_n``; within an offset
entries are sorted by output row ``k`` (mapping.py:289-319).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from itertools import product

import numpy as np
import torch

from . import _native as nat
from .core import CoordinateSet, as_device_coords

MISS = -1

# The reference's grid-index cell cap (mapping.py:21).  On the device "auto"
# additionally refuses grids above DEVICE_GRID_CAP cells (an int32 table of
# 512 MiB) and uses the hash index instead: maps are identical either way.
DEFAULT_GRID_CELL_CAP = 1 << 31
DEVICE_GRID_CAP = 1 << 27

# Base of the per-dimension offset window for even K (mapping.py:23-26); the
# reference's tests monkeypatch it to -1 as a negative control and so can ours.
EVEN_KERNEL_OFFSET_BASE = 0


class GridCapacityError(ValueError):
    """Grid index would exceed its cell cap; build a hash index instead."""


@dataclass(frozen=True, eq=False)
class KernelOffsets:
    """Ordered kernel offsets delta in Z^D, lexicographic (mapping.py:33-60)."""

    offsets: np.ndarray
    kernel_size: int
    dim: int

    def __post_init__(self):
        off = np.ascontiguousarray(self.offsets, dtype=np.int64)
        off.setflags(write=False)
        object.__setattr__(self, "offsets", off)

    @property
    def volume(self) -> int:
        return self.offsets.shape[0]

    @property
    def center(self) -> int | None:
        return (self.volume - 1) // 2 if self.kernel_size % 2 == 1 else None

    @property
    def base(self) -> int:
        """Lowest offset per dimension (what the kernels enumerate from)."""
        return int(self.offsets[0, 0]) if self.volume else 0


_OFFSETS_CACHE: dict = {}


def enumerate_offsets(dim: int, kernel_size: int) -> KernelOffsets:
    """All K**D offsets in lexicographic order (mapping.py:63-79).  Cached
    (immutable) per (dim, K, even-K base)."""
    key = (dim, kernel_size, EVEN_KERNEL_OFFSET_BASE)
    hit = _OFFSETS_CACHE.get(key)
    if hit is not None:
        return hit
    hit = _enumerate_offsets(dim, kernel_size)
    _OFFSETS_CACHE[key] = hit
    return hit


def _enumerate_offsets(dim: int, kernel_size: int) -> KernelOffsets:
    if not 1 <= dim <= 4:
        raise ValueError("dim must be between 1 and 4")
    if kernel_size < 1:
        raise ValueError("kernel_size must be >= 1")
    lo = -((kernel_size - 1) // 2) if kernel_size % 2 == 1 else EVEN_KERNEL_OFFSET_BASE
    axis = range(lo, lo + kernel_size)
    return KernelOffsets(np.array(list(product(axis, repeat=dim)), dtype=np.int64).reshape(-1, dim),
                         kernel_size, dim)


def _cells(boundary, batch_size) -> int:
    c = int(batch_size)
    for b in boundary:
        c *= int(b)
    return c


def _as_cset(coords, boundary, batch_size) -> CoordinateSet:
    if isinstance(coords, CoordinateSet):
        return coords
    if hasattr(coords, "coordset"):  # a SparseTensor
        return coords.coordset
    return CoordinateSet(as_device_coords(coords), tuple(boundary), batch_size)


class CoordinateIndex:
    """Device coordinate index: open-addressing hash (HashIndex,
    mapping.py:122-189) or dense grid (GridIndex, mapping.py:82-119)."""

    def __init__(self, cset: CoordinateSet, kind: str):
        self.kind = kind
        self.boundary = cset.boundary
        self.batch_size = cset.batch_size
        self.size = cset.num_points
        self._grid = nat.make_grid(self.boundary, self.batch_size)
        dev = cset.coords.device
        status = torch.empty(2, dtype=torch.int32, device=dev)  # zeroed by scb_index_build
        if kind == "hash":
            self.slots = int(nat.load().scb_hash_slots(self.size))
            self.keys = torch.empty(self.slots, dtype=torch.int64, device=dev)
            self.rows = torch.empty(self.slots, dtype=torch.int32, device=dev)
            code = nat.SCB_INDEX_HASH
        else:
            self.slots = _cells(self.boundary, self.batch_size)
            self.keys = None
            self.rows = torch.empty(self.slots, dtype=torch.int32, device=dev)
            code = nat.SCB_INDEX_GRID
        self.code = code
        nat.call("scb_index_build", code, nat.ptr(cset.coords), self.size, self._grid,
                 nat.ptr(self.keys), nat.ptr(self.rows), self.slots, nat.ptr(status),
                 nat.stream_handle())
        self._status = status

    @classmethod
    def relabelled(cls, src: "CoordinateIndex", inv: torch.Tensor) -> "CoordinateIndex":
        """``src`` under relabelled rows (row r -> inv[r]): the index of a
        reordered twin of src's set without a second build
        (scb_index_relabel; hash keys shared)."""
        idx = object.__new__(cls)
        idx.kind, idx.boundary, idx.batch_size = src.kind, src.boundary, src.batch_size
        idx.size, idx._grid, idx.slots, idx.code = src.size, src._grid, src.slots, src.code
        idx.keys = src.keys
        idx.rows = torch.empty_like(src.rows)
        idx._status = src._status
        nat.call("scb_index_relabel", src.code, nat.ptr(src.keys), nat.ptr(src.rows), src.slots,
                 nat.ptr(inv), nat.ptr(idx.rows), nat.stream_handle())
        return idx

    @property
    def duplicates(self) -> int:
        return int(self._status[0].item())

    def query(self, coords) -> torch.Tensor:
        """Row per query coordinate; MISS (-1) where absent or out of bounds."""
        q = as_device_coords(coords)
        out = torch.empty(q.shape[0], dtype=torch.int32, device=q.device)
        nat.call("scb_index_query", self.code, nat.ptr(q), q.shape[0], self._grid,
                 nat.ptr(self.keys), nat.ptr(self.rows), self.slots, nat.ptr(out),
                 nat.stream_handle())
        return out


def build_index(coords, kind: str = "auto", boundary=None, batch_size: int = 1,
                cell_cap: int = DEFAULT_GRID_CELL_CAP) -> CoordinateIndex:
    """Build (or reuse) a device coordinate index (mapping.py:195-208).
    ``coords`` may be a SparseTensor, a CoordinateSet or raw coordinates with
    ``boundary``/``batch_size``."""
    cset = _as_cset(coords, boundary, batch_size)
    cells = _cells(cset.boundary, cset.batch_size)
    if kind == "grid":
        if cells > cell_cap:
            raise GridCapacityError(
                f"grid index needs {cells} cells (cap {cell_cap}); use the hash index")
    elif kind == "auto":
        kind = "grid" if cells <= min(cell_cap, DEVICE_GRID_CAP) else "hash"
    elif kind != "hash":
        raise ValueError(f"unknown index kind {kind!r}")
    idx = cset.indexes.get(kind)
    if idx is None:
        idx = CoordinateIndex(cset, kind)
        cset.indexes[kind] = idx
    return idx


def presence_masks(cset: CoordinateSet, kernel_size: int = 3, kind: str = "auto"):
    """Neighbour-presence word per row of ``cset`` (bit n: coordinate +
    delta_n is in the set, stride 1) and the per-offset row counts, on the
    device (scb_presence_masks).  B200 extension."""
    offsets = enumerate_offsets(len(cset.boundary), kernel_size)
    if offsets.volume > 32:
        raise ValueError("presence masks hold at most 32 offsets")
    idx = build_index(cset, kind)
    dev = cset.coords.device
    n = cset.num_points
    masks = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(offsets.volume, dtype=torch.int64, device=dev)
    nat.call("scb_presence_masks", idx.code, nat.ptr(cset.coords), n, idx._grid, kernel_size,
             offsets.base, nat.ptr(idx.keys), nat.ptr(idx.rows), idx.slots, nat.ptr(masks),
             nat.ptr(counts), nat.stream_handle())
    return masks[:n], counts


def permute_rows(src: torch.Tensor, index: torch.Tensor, scatter: bool = False,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """Row permutation on the device (scb_permute_rows): ``out[i] =
    src[index[i]]``, or ``out[index[i]] = src[i]`` with ``scatter``."""
    n = index.shape[0]
    rows = src.shape[0] if scatter else n
    if out is None:
        out = torch.empty((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    rb = src.shape[1] * src.element_size()
    ld_s = (src.stride(0) if src.shape[0] > 1 else src.shape[1]) * src.element_size()
    ld_d = (out.stride(0) if out.shape[0] > 1 else out.shape[1]) * out.element_size()
    nat.call("scb_permute_rows", nat.ptr(src), ld_s, nat.ptr(index), n, rb, nat.ptr(out), ld_d,
             int(bool(scatter)), nat.stream_handle())
    return out


def reorder_by_presence(cset: CoordinateSet, kernel_size: int = 3,
                        kind: str = "auto") -> CoordinateSet:
    """The same coordinates with rows relabelled so that rows with similar
    neighbour patterns are adjacent (B200 extension, the TorchSparse++
    bitmask sort): a stable sort by the presence mask with the rarest
    offsets most significant (batch entries interleave: maps never cross
    them).  Returns a new CoordinateSet whose row i is
    row ``perm[i]`` of ``cset`` (``.perm``); maps built over it hold the same
    pairs under the new row numbers, and 128-row tiles of its k3 maps have
    far fewer active offsets (the fused kernel skips the rest).  Cached on
    ``cset``."""
    key = ("reorder", kernel_size)
    hit = cset.derived.get(key)
    if hit is not None:
        return hit
    n = cset.num_points
    dev = cset.coords.device
    masks, counts = presence_masks(cset, kernel_size, kind)
    V = counts.shape[0]
    lib = nat.load()
    ws = torch.empty(int(lib.scb_mask_sort_workspace(n)), dtype=torch.uint8, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    nat.call("scb_mask_sort", nat.ptr(masks), nat.ptr(counts), nat.ptr(cset.coords),
             cset.coords.shape[1], n, V, cset.batch_size, nat.ptr(ws), ws.numel(), nat.ptr(perm),
             nat.stream_handle())
    perm = perm[:n]
    coords = torch.empty_like(cset.coords)
    inv = torch.empty_like(perm)
    nat.call("scb_apply_order", nat.ptr(perm), n, nat.ptr(cset.coords), cset.coords.shape[1],
             nat.ptr(coords), nat.ptr(inv), nat.stream_handle())
    out = CoordinateSet(coords, cset.boundary, cset.batch_size, perm=perm)
    for k, idx in cset.indexes.items():   # the same indexes, rows relabelled
        out.indexes[k] = CoordinateIndex.relabelled(idx, inv)
    # the presence words in the new row order: the level's stride-1 map is
    # then searched from them (map_search_masked)
    out.derived[("presence", kernel_size)] = permute_rows(masks.view(n, 1), perm).view(n)
    cset.derived[key] = out
    return out


def downsample_boundary(boundary, stride: int) -> tuple[int, ...]:
    """ceil(b / stride) per dimension (mapping.py:211-213)."""
    return tuple(-(-int(b) // stride) for b in boundary)


def compute_output_coords(in_coords, offsets: KernelOffsets, stride: int, out_boundary,
                          batch_size: int = 1) -> torch.Tensor:
    """Active output coordinates (mapping.py:216-248).  Stride 1 returns the
    input coordinates; stride > 1 runs the fused candidate kernel and a radix
    sort + unique (32-bit keys whenever the output grid has < 2^32 cells, else
    64-bit), so rows come out in ascending flat-key order.
    Returns an int32 device tensor."""
    if stride < 1:
        raise ValueError("stride must be >= 1")
    c = in_coords.coords if hasattr(in_coords, "coords") else as_device_coords(in_coords)
    if stride == 1:
        return c
    dim = c.shape[1] - 1
    lib = nat.load()
    n_in = c.shape[0]
    grid = nat.make_grid(out_boundary, batch_size)
    cap = int(lib.scb_output_coords_capacity(n_in, dim, offsets.kernel_size, stride))
    ws_bytes = int(lib.scb_output_coords_workspace(n_in, dim, offsets.kernel_size, stride))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=c.device)
    keys = torch.empty(max(cap, 1), dtype=torch.int64, device=c.device)
    n_out = torch.zeros(1, dtype=torch.int64, device=c.device)
    nat.call("scb_output_coords", nat.ptr(c), n_in, grid, offsets.kernel_size, offsets.base,
             stride, nat.ptr(ws), ws_bytes, nat.ptr(keys), nat.ptr(n_out), nat.stream_handle())
    n = int(n_out.item())
    from .core import flush_validation
    flush_validation()
    out = torch.empty((n, dim + 1), dtype=torch.int32, device=c.device)
    nat.call("scb_unflatten", nat.ptr(keys), n, grid, nat.ptr(out), nat.stream_handle())
    return out


def compute_output_coords_chain(cset, steps) -> list[torch.Tensor]:
    """See start_output_coords_chain; returns the finished levels."""
    return start_output_coords_chain(cset, steps)()


def start_output_coords_chain(cset, steps):
    """Issue the output coordinates of successive strided levels, ``steps`` =
    [(offsets, stride), ...] applied one after the other from ``cset``, and
    return a finisher that waits for the counts and returns [(coords,
    boundary), ...] per level.  Level
    i+1 is generated from level i's keys with its count on the device
    (scb_output_keys_next), so the whole chain costs ONE host read.  Each
    level equals compute_output_coords of the previous one.  Only for windows
    that propose one candidate per input (K = s, e.g. k2 s2), where the
    capacity does not grow along the chain."""
    lib = nat.load()
    c = cset.coords
    dev = c.device
    dim = c.shape[1] - 1
    n_cap = c.shape[0]
    counts = torch.empty(max(len(steps), 1), dtype=torch.int64, device=dev)  # written by each level
    boundary, prev = cset.boundary, None
    levels = []
    for i, (offsets, stride) in enumerate(steps):
        out_b = downsample_boundary(boundary, stride)
        g = nat.make_grid(out_b, cset.batch_size)
        cap = int(lib.scb_output_coords_capacity(n_cap, dim, offsets.kernel_size, stride))
        if cap > n_cap and i:
            raise ValueError("chained output coordinates need one candidate per input")
        ws_bytes = int(lib.scb_output_coords_workspace(n_cap, dim, offsets.kernel_size, stride))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
        keys = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        cnt = counts.data_ptr() + 8 * i
        if prev is None:
            nat.call("scb_output_coords", nat.ptr(c), n_cap, g, offsets.kernel_size,
                     offsets.base, stride, nat.ptr(ws), ws_bytes, nat.ptr(keys), cnt,
                     nat.stream_handle())
        else:
            pkeys, pcnt, pgrid = prev
            nat.call("scb_output_keys_next", nat.ptr(pkeys), pcnt, n_cap, pgrid, g,
                     offsets.kernel_size, offsets.base, stride, nat.ptr(ws), ws_bytes,
                     nat.ptr(keys), cnt, nat.stream_handle())
        levels.append((keys, g, out_b, ws))
        prev = (keys, cnt, g)
        boundary, n_cap = out_b, cap
    # the chain's one host read, asynchronous: the caller can queue other work
    # (e.g. the first convolutions) before calling the returned finisher
    from .core import PINNED
    host, ready = PINNED.read_async(counts)

    def finish():
        ready.synchronize()
        from .core import flush_validation
        flush_validation()  # asynchronous input validations queued before the chain
        out = []
        ns = host.tolist()
        PINNED.release(host)
        for (keys, g, out_b, _), n in zip(levels, ns):
            co = torch.empty((n, dim + 1), dtype=torch.int32, device=dev)
            nat.call("scb_unflatten", nat.ptr(keys), n, g, nat.ptr(co), nat.stream_handle())
            out.append((co, out_b))
        return out

    return finish


def _hit_matrix(volume: int, n: int, device) -> torch.Tensor:
    """Uninitialised [V][ld] int32 hit matrix; ld = n rounded up to 4
    (scb_hits_ld) so each row is 16-byte aligned."""
    return torch.empty((volume, max((n + 3) // 4 * 4, 4)), dtype=torch.int32, device=device)


def _compact(hits: torch.Tensor, volume: int, n_out: int):
    """Hit matrix [V][n_out] -> CSR map (offset_ptr device, sizes host,
    in_idx, out_idx).  One D2H of V+1 int64 (the map sizes)."""
    lib = nat.load()
    dev = hits.device
    ws = torch.empty(max(int(lib.scb_map_workspace(volume, n_out)), 8), dtype=torch.uint8,
                     device=dev)
    ptr = torch.empty(volume + 1, dtype=torch.int64, device=dev)
    s = nat.stream_handle()
    nat.call("scb_map_count", nat.ptr(hits), volume, n_out, nat.ptr(ws), nat.ptr(ptr), s)
    host_ptr = ptr.cpu().numpy()
    total = int(host_ptr[-1])
    in_idx = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    out_idx = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    nat.call("scb_map_compact", nat.ptr(hits), volume, n_out, nat.ptr(ws), nat.ptr(ptr),
             nat.ptr(in_idx), nat.ptr(out_idx), s)
    return ptr, np.diff(host_ptr).astype(np.int64), in_idx[:total], out_idx[:total]


class KernelMap:
    """Per-offset (input row, output row) pairs (mapping.py:251-286).

    Two device representations, each built on demand from the other:
    the hit matrix ``hits[V][n_out]`` (input row or -1; what map search
    produces and what the fused dataflow consumes, no host sync) and the
    canonical CSR (``offset_ptr``, ``in_idx``, ``out_idx`` + host ``sizes``;
    what the staged dataflow and the reference API use, one D2H of V+1 sizes
    to build)."""

    def __init__(self, offset_ptr, sizes, in_idx, out_idx, offsets: KernelOffsets, stride: int,
                 n_in: int, n_out: int, symmetric: bool = False, trusted: bool = False,
                 hits: torch.Tensor | None = None):
        self.offsets = offsets
        self.stride = int(stride)
        self.n_in = int(n_in)
        self.n_out = int(n_out)
        self.symmetric = bool(symmetric)
        self.trusted = bool(trusted)  # produced by map search: one entry per (k, n)
        self._hits = hits
        self._csr = None
        if offset_ptr is not None:
            self._csr = (offset_ptr, np.asarray(sizes, dtype=np.int64), in_idx, out_idx)
        self._pairs = None
        self._plans = {}
        self._swapped = None
        self._tile_masks = None
        self.onehot = False   # at most one entry per output row (transposed K = s map)
        self._parent = None   # the K = s map this one-hot map was swapped from
        self._lazy_hits = None  # builds the hit matrix on first use (one-hot swapped maps)
        self._onehot_order = None

    @classmethod
    def from_hits(cls, hits, offsets, stride, n_in, n_out, symmetric=False) -> "KernelMap":
        return cls(None, None, None, None, offsets, stride, n_in, n_out, symmetric,
                   trusted=True, hits=hits)

    def device_tensors(self):
        out = [t for t in (self._hits, self._tile_masks) if t is not None]
        if self._parent is not None and self._parent._hits is not None:
            out.append(self._parent._hits)  # the scatter form's child table
        if self._csr is not None:
            out += [self._csr[0], self._csr[2], self._csr[3]]
        return out

    # ---- representations ------------------------------------------------
    def _ensure_csr(self):
        if self._csr is None:
            self._csr = _compact(self.hits, self.offsets.volume, self.n_out)
        return self._csr

    @property
    def hits(self) -> torch.Tensor:
        """[V][max(n_out,1)] int32 hit matrix on the device."""
        if self._hits is None and self._lazy_hits is not None:
            self._hits, self._lazy_hits = self._lazy_hits(), None
        if self._hits is None:
            ptr, _, ii, oi = self._ensure_csr()
            V = self.offsets.volume
            h = _hit_matrix(V, self.n_out, ii.device)
            # hits[n][out_idx[e]] = in_idx[e]: the transpose kernel with roles exchanged
            nat.call("scb_map_transpose", nat.ptr(ptr), nat.ptr(oi), nat.ptr(ii), V,
                     self.total, self.n_out, nat.ptr(h), nat.stream_handle())
            self._hits = h
        return self._hits

    def tile_masks(self) -> torch.Tensor:
        """Active-offset word per 128-row output tile (scb_tile_masks): bit n
        set when some row of the tile has a neighbour at offset n.  Built once
        per map (B200 extension; the fused kernel skips clear bits)."""
        if self._tile_masks is None:
            h = self.hits
            tiles = max((self.n_out + nat.TILE_ROWS - 1) // nat.TILE_ROWS, 1)
            m = torch.empty(tiles, dtype=torch.int32, device=h.device)
            nat.call("scb_tile_masks", nat.ptr(h), self.offsets.volume, self.n_out, nat.ptr(m),
                     nat.stream_handle())
            self._tile_masks = m
        return self._tile_masks

    def onehot_order(self):
        """(perm, hits, tile_masks) of a one-hot map in tile-row order: rows
        stably sorted by the offset of their entry, so each 128-row tile of
        the fused kernel has one active offset (scb_onehot_order; B200
        extension).  Built once per map."""
        if self._onehot_order is None:
            h = self.hits
            n, dev = self.n_out, h.device
            ws = torch.empty(int(nat.load().scb_onehot_order_workspace(n)), dtype=torch.uint8,
                             device=dev)
            perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            hp = _hit_matrix(self.offsets.volume, n, dev)
            tiles = max((n + nat.TILE_ROWS - 1) // nat.TILE_ROWS, 1)
            tm = torch.zeros(tiles, dtype=torch.int32, device=dev)
            nat.call("scb_onehot_order", nat.ptr(h), self.offsets.volume, n, nat.ptr(ws), ws.numel(),
                     nat.ptr(perm), nat.ptr(hp), nat.ptr(tm), nat.stream_handle())
            self._onehot_order = (perm, hp, tm)
        return self._onehot_order

    offset_ptr = property(lambda self: self._ensure_csr()[0])
    in_idx = property(lambda self: self._ensure_csr()[2])
    out_idx = property(lambda self: self._ensure_csr()[3])

    @property
    def sizes(self) -> np.ndarray:
        return self._ensure_csr()[1].copy()

    @property
    def buffer_offsets(self) -> np.ndarray:
        sz = self._ensure_csr()[1]
        out = np.zeros(sz.shape[0] + 1, dtype=np.int64)
        np.cumsum(sz, out=out[1:])
        return out

    @property
    def total(self) -> int:
        return int(self._ensure_csr()[1].sum())

    @property
    def device(self):
        if self._hits is None and self._csr is None and self._parent is not None:
            return self._parent.device
        return (self._hits if self._hits is not None else self._csr[2]).device

    @property
    def pairs(self) -> list[np.ndarray]:
        """Host copy in the reference layout: one (m_n, 2) int64 array per offset."""
        if self._pairs is None:
            j = self.in_idx.cpu().numpy().astype(np.int64)
            k = self.out_idx.cpu().numpy().astype(np.int64)
            st = self.buffer_offsets
            self._pairs = [np.stack([j[st[n]:st[n + 1]], k[st[n]:st[n + 1]]], axis=1)
                           for n in range(self.offsets.volume)]
        return self._pairs

    def swap_roles(self) -> "KernelMap":
        """Input/output roles exchanged, entries re-sorted by the new output
        row (mapping.py:277-286).  Transposing the hit matrix produces the
        re-sorted order directly: the new hit matrix is indexed by new output row."""
        if self._swapped is None:
            V = self.offsets.volume

            def transposed():
                ht = _hit_matrix(V, self.n_in, self.device)
                if self._hits is not None:
                    nat.call("scb_hits_transpose", nat.ptr(self._hits), V, self.n_out, self.n_in,
                             nat.ptr(ht), nat.stream_handle())
                else:
                    nat.call("scb_map_transpose", nat.ptr(self.offset_ptr), nat.ptr(self.in_idx),
                             nat.ptr(self.out_idx), V, self.total, self.n_in, nat.ptr(ht),
                             nat.stream_handle())
                return ht

            # K = s windows tile the fine grid: every fine row has one parent
            onehot = self.stride > 1 and self.offsets.kernel_size == self.stride
            self._swapped = KernelMap(None, None, None, None, self.offsets, self.stride,
                                      self.n_out, self.n_in, trusted=self.trusted,
                                      hits=None if onehot else transposed())
            self._swapped.onehot = onehot
            if onehot:
                # the scatter-form transposed layer reads this map's hit matrix
                # as its child table (scb_conv_transposed_scatter); the
                # transposed hit matrix is built only if something asks for it
                self._swapped._parent = self
                self._swapped._lazy_hits = transposed
        return self._swapped


def map_search(in_index: CoordinateIndex, out_coords, offsets: KernelOffsets, stride: int,
               use_symmetry: bool | None = None, dilation: int = 1) -> KernelMap:
    """Kernel map: entry (j, k) whenever stride*q_k + delta_n is input j
    (mapping.py:289-319).  Stride-1 odd-K maps probe only offsets up to the
    centre and fill the mirrored half in the same pass (mapping.py:322-339).
    ``dilation`` (B200 extension): the window's offsets are scaled by it.
    Returns a map holding the hit matrix; the CSR form is compacted on first
    use."""
    oc = out_coords.coords if hasattr(out_coords, "coords") else as_device_coords(out_coords)
    volume, center = offsets.volume, offsets.center
    if use_symmetry is None:
        use_symmetry = stride == 1 and center is not None and volume > 1
    if use_symmetry and (stride != 1 or center is None):
        raise ValueError("symmetric search requires stride 1 and odd kernel size")
    n_out = oc.shape[0]
    if use_symmetry and n_out != in_index.size:
        raise ValueError("symmetric search needs the output set to equal the input set")
    hits = _hit_matrix(volume, n_out, oc.device)
    grid = nat.make_grid(in_index.boundary, in_index.batch_size)
    if dilation == 1:
        nat.call("scb_map_search", in_index.code, nat.ptr(oc), n_out, grid, offsets.kernel_size,
                 offsets.base, stride, int(bool(use_symmetry)), nat.ptr(in_index.keys),
                 nat.ptr(in_index.rows), in_index.slots, nat.ptr(hits), nat.stream_handle())
    else:  # dilated window (B200 extension): probes stride*q + dilation*delta
        nat.call("scb_map_search_dilated", in_index.code, nat.ptr(oc), n_out, grid,
                 offsets.kernel_size, offsets.base, stride, int(dilation),
                 int(bool(use_symmetry)), nat.ptr(in_index.keys), nat.ptr(in_index.rows),
                 in_index.slots, nat.ptr(hits), nat.stream_handle())
    kmap = KernelMap.from_hits(hits, offsets, stride, in_index.size, n_out,
                               symmetric=bool(use_symmetry))
    kmap.dilation = int(dilation)
    return kmap


def map_search_masked(in_index: CoordinateIndex, cset: CoordinateSet, offsets: KernelOffsets,
                      masks: torch.Tensor) -> KernelMap:
    """The stride-1 map of ``cset`` onto itself (= map_search(..., stride 1),
    symmetric) from the rows' presence words (presence_masks in cset's row
    order): only present offsets are probed, and the map's tile masks come
    with it (scb_map_search_masked; B200 extension)."""
    n = cset.num_points
    if offsets.volume > 32 or offsets.center is None:
        raise ValueError("masked search needs an odd kernel of at most 32 offsets")
    if masks.shape[0] != n or n != in_index.size:
        raise ValueError("masked search needs the set's own presence words and index")
    hits = _hit_matrix(offsets.volume, n, cset.coords.device)
    tiles = max((n + nat.TILE_ROWS - 1) // nat.TILE_ROWS, 1)
    tm = torch.zeros(tiles, dtype=torch.int32, device=cset.coords.device)
    grid = nat.make_grid(in_index.boundary, in_index.batch_size)
    nat.call("scb_map_search_masked", in_index.code, nat.ptr(cset.coords), n, grid,
             offsets.kernel_size, offsets.base, nat.ptr(in_index.keys), nat.ptr(in_index.rows),
             in_index.slots, nat.ptr(masks), nat.ptr(hits), nat.ptr(tm), nat.stream_handle())
    kmap = KernelMap.from_hits(hits, offsets, 1, n, n, symmetric=True)
    kmap._tile_masks = tm
    return kmap


def derive_symmetric_maps(half_map: KernelMap) -> KernelMap:
    """Complete a stride-1 odd-K map from its lower half (mapping.py:322-339):
    M[V-1-n] = reversed M[n], sorted by the new output row."""
    if half_map.stride != 1:
        raise ValueError("symmetric maps exist only for stride-1 layers")
    center = half_map.offsets.center
    if center is None:
        raise ValueError("symmetric maps exist only for odd kernel sizes")
    V, n = half_map.offsets.volume, half_map.n_out
    direct = half_map.hits
    mirror = torch.empty_like(direct)
    nat.call("scb_hits_transpose", nat.ptr(direct), V, n, n, nat.ptr(mirror), nat.stream_handle())
    hits = direct.clone()
    lower = torch.arange(center, device=direct.device)
    hits[V - 1 - lower] = mirror[lower]
    return KernelMap.from_hits(hits, half_map.offsets, 1, half_map.n_in, n, symmetric=True)


class GatherScatterPlan:
    """Device plan over a kernel map (mapping.py:342-418).

    B200 layout: offset n's buffer slice starts at ``slab_ptr[n]``, a multiple
    of the GEMM tile height, so no tile straddles two offsets.  ``buf_in``
    (input row per buffer row, -1 on padding) drives the gather and ``pos``
    ([n_out][V], buffer row per output and offset) drives the
    output-stationary scatter.  The reference's compact CSR views
    (``row_input``, ``in_indptr``, ...) are available as host arrays."""

    def __init__(self, kmap: KernelMap, skip_center: bool = False, tile_rows: int = nat.TILE_ROWS):
        skipped = None
        if skip_center:
            skipped = kmap.offsets.center
            if skipped is None or kmap.stride != 1:
                raise ValueError("skip_center requires a stride-1 odd-K map")
        # weak: the map caches its plans, a strong back-reference would form a
        # cycle that only the cyclic GC frees (multi-100-MB device buffers)
        self._kmap = weakref.ref(kmap)
        self.volume = kmap.offsets.volume
        self.n_in, self.n_out = kmap.n_in, kmap.n_out
        self.skipped_offset = skipped
        self.tile_rows = int(tile_rows)
        sizes = kmap.sizes
        if skipped is not None:
            sizes[skipped] = 0
        self._sizes = sizes
        self.buffer_offsets = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
        np.cumsum(sizes, out=self.buffer_offsets[1:])
        self.total = int(self.buffer_offsets[-1])
        padded = (sizes + tile_rows - 1) // tile_rows * tile_rows
        self.slab_ptr = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
        np.cumsum(padded, out=self.slab_ptr[1:])
        self.rows_pad = int(self.slab_ptr[-1])
        V = sizes.shape[0]
        dev = kmap.device
        self.buf_in = torch.empty(max(self.rows_pad, 1), dtype=torch.int32, device=dev)
        self.pos = torch.empty((max(self.n_out, 1), V), dtype=torch.int32, device=dev)
        status = None if kmap.trusted else torch.zeros(1, dtype=torch.int32, device=dev)
        nat.call("scb_plan_build", nat.ptr(kmap.offset_ptr), nat.ptr(kmap.in_idx),
                 nat.ptr(kmap.out_idx), V, kmap.total, self.n_out,
                 -1 if skipped is None else skipped, self.tile_rows, nat.ptr(self.buf_in),
                 self.rows_pad, nat.ptr(self.pos), nat.ptr(status), nat.stream_handle())
        # A hand-built map (reference API) may hold several entries for one
        # (output, offset) pair; the fixed-width `pos` table cannot, so such
        # a plan scatters through the output CSR instead (scb_scatter_csr).
        self.general = bool(status is not None and int(status.item()))
        self._csr = None
        self._dev_csr = None
        if self.general:  # built now: the plan holds its map only weakly
            self.device_out_csr()

    @property
    def sizes(self) -> np.ndarray:
        return self._sizes.copy()

    @property
    def kmap(self) -> KernelMap:
        k = self._kmap()
        if k is None:
            raise RuntimeError("the kernel map of this plan has been released")
        return k

    # ---- reference CSR views (host numpy, computed on demand) -------------
    def _views(self):
        if self._csr is None:
            pairs = self.kmap.pairs
            kept = [p for n, p in enumerate(pairs) if n != self.skipped_offset and p.shape[0]]
            st = np.concatenate(kept, 0) if kept else np.empty((0, 2), np.int64)
            ri, ro = np.ascontiguousarray(st[:, 0]), np.ascontiguousarray(st[:, 1])
            ip = np.zeros(self.n_in + 1, np.int64)
            np.cumsum(np.bincount(ri, minlength=self.n_in), out=ip[1:])
            op = np.zeros(self.n_out + 1, np.int64)
            np.cumsum(np.bincount(ro, minlength=self.n_out), out=op[1:])
            self._csr = dict(row_input=ri, row_output=ro, in_indptr=ip,
                             in_rows=np.argsort(ri, kind="stable").astype(np.int64),
                             out_indptr=op, out_rows=np.argsort(ro, kind="stable").astype(np.int64))
        return self._csr

    row_input = property(lambda self: self._views()["row_input"])
    row_output = property(lambda self: self._views()["row_output"])
    in_indptr = property(lambda self: self._views()["in_indptr"])
    in_rows = property(lambda self: self._views()["in_rows"])
    out_indptr = property(lambda self: self._views()["out_indptr"])
    out_rows = property(lambda self: self._views()["out_rows"])
    in_counts = property(lambda self: np.diff(self.in_indptr))
    out_counts = property(lambda self: np.diff(self.out_indptr))

    def device_out_csr(self):
        """(out_indptr int64[n_out+1], out_rows int32[total]) on the device."""
        if self._dev_csr is None:
            dev = self.buf_in.device
            self._dev_csr = (torch.from_numpy(self.out_indptr).to(dev),
                             torch.from_numpy(self.out_rows.astype(np.int32)).to(dev))
        return self._dev_csr

    def padded_rows(self, compact: torch.Tensor) -> torch.Tensor:
        """Index of each compact (reference-layout) buffer row in the padded
        device layout."""
        idx = [torch.arange(self.slab_ptr[n], self.slab_ptr[n] + self._sizes[n])
               for n in range(self._sizes.shape[0]) if self._sizes[n]]
        if not idx:
            return torch.empty(0, dtype=torch.int64, device=compact.device)
        return torch.cat(idx).to(compact.device)


def build_gather_scatter_plan(kmap: KernelMap, skip_center: bool = False) -> GatherScatterPlan:
    """Lay out the buffer and build both stationary indexes (mapping.py:377-418);
    cached on the map."""
    key = bool(skip_center)
    plan = kmap._plans.get(key)
    if plan is None:
        plan = GatherScatterPlan(kmap, skip_center)
        kmap._plans[key] = plan
    return plan
