"""``sparseconv.core`` on the B200 engine (reference ``core.py``).

:class:`SparseTensor` keeps the reference's host contract — int64
``coords`` and f32/f16 ``features`` as read-only numpy arrays, frozen
attributes, the same ValueErrors — and carries the engine tensor it was
validated into (``_dev``: device coordinates, features and the coordinate
set whose index / maps later layers reuse).  Every operation below runs on
the engine; only the returned arrays are host copies.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from paper_2204_10319_b200 import core as _eng

PrecisionMode = _eng.PrecisionMode
WeightTensor = _eng.WeightTensor
DEFAULT_DENSE_CAP = 1 << 27
FP16_MAX = 65504.0
_FEATURE_DTYPES = (np.dtype(np.float32), np.dtype(np.float16))


def flatten_coords(coords, boundary, batch_size: int = 1) -> np.ndarray:
    """Batch-major flat key (reference core.py:46-66), as a numpy array."""
    return np.asarray(_eng.flatten_coords(np.asarray(coords, dtype=np.int64), boundary,
                                          batch_size))


def unflatten_coords(keys, boundary, batch_size: int = 1) -> np.ndarray:
    """Inverse of :func:`flatten_coords` (reference core.py:69-79)."""
    return np.asarray(_eng.unflatten_coords(np.asarray(keys, dtype=np.int64), boundary,
                                            batch_size))


def _readonly(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


class SparseTensor:
    """Unique integer coordinates paired with a feature row each
    (reference core.py:82-143).  Validation (rank, rows, batch range,
    boundary, uniqueness) runs on the device when the engine tensor is
    built; the arrays are read-only and the attributes frozen, as in the
    reference."""

    __slots__ = ("coords", "features", "stride", "boundary", "batch_size", "_dev")

    def __init__(self, coords, features, stride: int = 1, boundary=(), batch_size: int = 1):
        c = np.ascontiguousarray(coords, dtype=np.int64)
        f = np.ascontiguousarray(features)
        if f.dtype not in _FEATURE_DTYPES:
            f = f.astype(np.float32)
        boundary = tuple(int(b) for b in boundary)
        dev = _eng.SparseTensor(c, f, int(stride), boundary, int(batch_size))
        self._init(c, f, dev)   # (the reference also freezes the caller's arrays in place)

    def _init(self, c, f, dev) -> None:
        object.__setattr__(self, "coords", _readonly(c))
        object.__setattr__(self, "features", _readonly(f))
        object.__setattr__(self, "stride", int(dev.stride))
        object.__setattr__(self, "boundary", tuple(dev.boundary))
        object.__setattr__(self, "batch_size", int(dev.batch_size))
        object.__setattr__(self, "_dev", dev)

    @classmethod
    def _from_engine(cls, dev: "_eng.SparseTensor", coords: np.ndarray | None = None
                     ) -> "SparseTensor":
        """Host view of an engine result (one D2H of coordinates and features;
        ``coords``: a host copy already known to equal the device ones)."""
        t = object.__new__(cls)
        c = coords if coords is not None else dev.coords_numpy()
        t._init(c, dev.features_numpy(), dev)
        return t

    def __setattr__(self, name, value):
        raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")

    def __delattr__(self, name):
        raise dataclasses.FrozenInstanceError(f"cannot delete field {name!r}")

    def __repr__(self) -> str:
        return (f"SparseTensor(num_points={self.num_points}, num_channels={self.num_channels}, "
                f"stride={self.stride}, boundary={self.boundary}, batch_size={self.batch_size})")

    @property
    def num_points(self) -> int:
        return self.coords.shape[0]

    @property
    def num_channels(self) -> int:
        return self.features.shape[1]

    @property
    def spatial_dims(self) -> int:
        return len(self.boundary)

    def replace_features(self, features) -> "SparseTensor":
        """Same coordinates (the same device coordinate set: no re-validation,
        its index and maps stay reusable), new feature matrix."""
        f = np.ascontiguousarray(features)
        if f.dtype not in _FEATURE_DTYPES:
            f = f.astype(np.float32)
        if f.ndim != 2 or f.shape[0] != self.num_points:
            raise ValueError("feature rows must match coordinate rows")
        t = object.__new__(SparseTensor)
        t._init(self.coords, f, self._dev.replace_features(f))
        return t


def _engine_tensor(t) -> "_eng.SparseTensor":
    if isinstance(t, SparseTensor):
        return t._dev
    if isinstance(t, _eng.SparseTensor):
        return t
    raise TypeError(f"expected a SparseTensor, got {type(t).__name__}")


def _wrap_result(dev: "_eng.SparseTensor", like: SparseTensor | None = None) -> SparseTensor:
    """Engine result -> host tensor; coordinates are shared with ``like``
    when the result lives on the same coordinate set."""
    if like is not None and dev.coordset is like._dev.coordset:
        return SparseTensor._from_engine(dev, like.coords)
    return SparseTensor._from_engine(dev)


def voxelize(points, voxel_size: float, reduce: str = "mean",
             spatial_dims: int = 3) -> SparseTensor:
    """Quantise a point cloud onto the voxel lattice (reference
    core.py:174-216) with ``scb_voxelize``: bit-exact coordinates and f64
    means."""
    return SparseTensor._from_engine(_eng.voxelize(points, voxel_size, reduce, spatial_dims))


def quantize_features(t: SparseTensor, mode: PrecisionMode) -> SparseTensor:
    """Storage precision conversion (reference core.py:219-238) with
    ``scb_quantize_f16``: round to nearest, saturate to +-65504 with the
    reference's warning."""
    if not isinstance(mode, PrecisionMode):
        raise ValueError(f"unknown precision mode {mode!r}")
    return _wrap_result(_eng.quantize_features(_engine_tensor(t), mode), t)


def to_dense(t: SparseTensor, cap: int = DEFAULT_DENSE_CAP) -> np.ndarray:
    """Dense (batch, *boundary, C) grid of a tensor (reference
    core.py:241-256); a host utility of the reference's test tooling."""
    cells = t.batch_size * int(np.prod(t.boundary, dtype=np.int64))
    if cells * max(t.num_channels, 1) > cap:
        raise ValueError(f"dense grid of {cells * t.num_channels} elements exceeds cap {cap}")
    grid = np.zeros((t.batch_size, *t.boundary, t.num_channels), dtype=t.features.dtype)
    if t.num_points:
        grid[tuple(t.coords.T)] = t.features
    return grid


def sparsify(grid: np.ndarray, stride: int = 1) -> SparseTensor:
    """Rows of a dense grid with any nonzero channel (reference
    core.py:259-270)."""
    grid = np.asarray(grid)
    if grid.ndim < 3:
        raise ValueError("grid must be (batch, *spatial, C)")
    live = np.nonzero(np.any(grid != 0, axis=-1))
    return SparseTensor(np.stack(live, axis=1).astype(np.int64), grid[live], stride=stride,
                        boundary=grid.shape[1:-1], batch_size=grid.shape[0])
