"""Deterministic synthetic inputs for the benchmark configurations.

Host-side data preparation (numpy), *before* the hot path: point synthesis
and voxelisation are outside the SparseConv3d forward (SURVEY.md §2 marks
voxelize as a "next" row), so they stay on the CPU here.

* ``config1_cloud`` reproduces the reference recipe of SURVEY.md §8(d)
  config 1: ``synth_points("uniform", 60_000, 50.0, seed=0)`` followed by
  ``voxelize(·, 1.0)`` (reference ``synth.py:16-53``, ``core.py:174-216``),
  bit-identical (pinned by ``tests/golden/config1.npz``).
* ``raycast_scan`` is the SemanticKITTI-shaped raycast LiDAR generator that
  SURVEY.md §8(d) config 3 specifies (64 beams, 3600 azimuths, boxes over a
  ground plane, 0.05 m voxels): the reference's ``lidar_rings`` is far too
  sparse at that resolution.
"""

from __future__ import annotations

import numpy as np


def synth_uniform(n_points: int, extent: float, seed: int, channels: int = 4) -> np.ndarray:
    """Uniform cloud in [0, extent)^3 plus N(0,1) features, float32
    (the "uniform" branch of reference synth.py:33-51)."""
    rng = np.random.default_rng(seed)
    xyz = rng.uniform(0.0, extent, size=(n_points, 3))
    feats = rng.standard_normal((n_points, channels))
    return np.concatenate([xyz, feats], axis=1).astype(np.float32)


def voxelize(points: np.ndarray, voxel_size: float, spatial_dims: int = 3):
    """Floor-quantise, shift to the min corner, merge duplicates by mean, and
    return rows sorted by flat key (reference core.py:174-216).

    Returns ``(coords int64 (N, 1+D), features float32 (N, C), boundary)``.
    """
    pts = np.asarray(points, dtype=np.float64)
    xyz, feats = pts[:, :spatial_dims], pts[:, spatial_dims:]
    cells = np.floor((xyz - xyz.min(axis=0)) / voxel_size).astype(np.int64)
    boundary = tuple(int(m) + 1 for m in cells.max(axis=0))
    key = np.zeros(cells.shape[0], dtype=np.int64)
    for d, b in enumerate(boundary):
        key = key * b + cells[:, d]
    uniq, inverse = np.unique(key, return_inverse=True)
    counts = np.bincount(inverse, minlength=uniq.shape[0]).astype(np.float64)
    merged = np.empty((uniq.shape[0], feats.shape[1]), dtype=np.float32)
    for c in range(feats.shape[1]):
        merged[:, c] = (np.bincount(inverse, weights=feats[:, c], minlength=uniq.shape[0])
                        / counts).astype(np.float32)
    coords = np.empty((uniq.shape[0], 1 + spatial_dims), dtype=np.int64)
    rem = uniq.copy()
    for d in range(spatial_dims - 1, -1, -1):
        coords[:, d + 1] = rem % boundary[d]
        rem //= boundary[d]
    coords[:, 0] = rem
    return coords, merged, boundary


def config1_cloud():
    """N = 47,628 voxels, boundary (50, 50, 50)."""
    return voxelize(synth_uniform(60_000, 50.0, seed=0, channels=4), 1.0)


def raycast_points(seed: int, beams: int = 64, elev=(-24.9, 2.0), azimuths: int = 3600,
                   n_boxes: int = 60, max_range: float = 80.0, sensor_z: float = 1.73,
                   sweeps: int = 1, sweep_shift: float = 0.0, with_time: bool = False):
    """Raycast a spinning LiDAR against a ground plane plus axis-aligned boxes.

    Parameters follow SURVEY.md §8(d) config 3 (config 4 uses 32 beams,
    10 sweeps).  Returns float32 (P, 3 + 1 [+1]) rows: x, y, z, intensity
    [, dt].
    """
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-50, 50, size=(n_boxes * 3, 2))
    half = rng.uniform(0.3, 6.0, size=(centers.shape[0], 2))
    # no box within 4 m of the sensor (its footprint must not contain it)
    clear = ((np.abs(centers) - half) > 4.0).any(axis=1)
    centers, half = centers[clear][:n_boxes], half[clear][:n_boxes]
    height = rng.uniform(0.5, 6.0, size=centers.shape[0])
    box_lo = np.concatenate([centers - half, np.zeros((centers.shape[0], 1))], axis=1)
    box_hi = np.concatenate([centers + half, height[:, None]], axis=1)
    el = np.deg2rad(np.linspace(elev[0], elev[1], beams))
    out = []
    for sw in range(sweeps):
        phase = rng.uniform(0, 2 * np.pi / azimuths)
        az = phase + np.arange(azimuths) * (2 * np.pi / azimuths)
        origin = np.array([-sweep_shift * sw, 0.0, sensor_z])
        ce, se = np.cos(el)[:, None], np.sin(el)[:, None]
        d = np.stack([ce * np.cos(az)[None, :], ce * np.sin(az)[None, :],
                      np.broadcast_to(se, (beams, azimuths))], axis=-1).reshape(-1, 3)
        t = np.full(d.shape[0], np.inf)
        down = d[:, 2] < -1e-9
        t[down] = -origin[2] / d[down, 2]
        # slab test against every box, in chunks to bound memory
        inv = 1.0 / np.where(np.abs(d) < 1e-12, 1e-12, d)
        for b0 in range(0, box_lo.shape[0], 16):
            lo = (box_lo[None, b0:b0 + 16] - origin) * inv[:, None, :]
            hi = (box_hi[None, b0:b0 + 16] - origin) * inv[:, None, :]
            tmin = np.minimum(lo, hi).max(axis=-1)
            tmax = np.maximum(lo, hi).min(axis=-1)
            hit = (tmax >= np.maximum(tmin, 0.0))
            tt = np.where(hit, np.maximum(tmin, 0.0), np.inf).min(axis=1)
            t = np.minimum(t, tt)
        ok = np.isfinite(t) & (t < max_range) & (t > 0.5)
        p = origin + d[ok] * t[ok, None]
        p += rng.normal(0.0, 0.01, size=p.shape)
        cols = [p, rng.uniform(0, 1, size=(p.shape[0], 1))]
        if with_time:
            cols.append(np.full((p.shape[0], 1), 0.05 * sw))
        out.append(np.concatenate(cols, axis=1))
    return np.concatenate(out, axis=0).astype(np.float32)


def semantickitti_scan(seed: int, voxel: float = 0.05):
    """Config 3/5 scan: 64-beam raycast, voxel 0.05 m, features
    (x, y, z, intensity) -> C_in = 4."""
    pts = raycast_points(seed)
    # keep absolute xyz as features (the voxeliser averages all non-position columns)
    pts = np.concatenate([pts[:, :3], pts], axis=1)
    return voxelize(pts, voxel)


def nuscenes_sweeps(seed: int, azimuths: int = 2100, voxel: float = 0.075):
    """Config 4: 32 beams, 10 sweeps, voxel 0.075 m, features
    (x, y, z, intensity, dt) -> C_in = 5."""
    pts = raycast_points(seed, beams=32, elev=(-30.0, 10.0), azimuths=azimuths, n_boxes=80,
                         max_range=60.0, sweeps=10, sweep_shift=0.5, with_time=True)
    pts = np.concatenate([pts[:, :3], pts], axis=1)
    return voxelize(pts, voxel)
