"""GPU voxelisation (reference core.py:174-216)
against the unmodified reference's golden vectors and the oracle:
bit-exact coordinates, boundary and features (mean and first)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sparseconv_oracle as O

pytestmark = pytest.mark.gpu


def test_voxelize_matches_reference_golden():
    import paper_2204_10319_b200 as sc
    g = np.load(GOLDEN / "voxelize.npz")
    i = 0
    while f"v{i}_points" in g.files:
        dims, first = (int(x) for x in g[f"v{i}_meta"])
        t = sc.voxelize(g[f"v{i}_points"], float(g[f"v{i}_vs"][0]),
                        "first" if first else "mean", dims)
        np.testing.assert_array_equal(t.coords_numpy(), g[f"v{i}_coords"])
        np.testing.assert_array_equal(t.features_numpy(), g[f"v{i}_feats"])
        assert tuple(t.boundary) == tuple(int(x) for x in g[f"v{i}_boundary"])
        i += 1


@pytest.mark.parametrize("reduce", ["mean", "first"])
def test_voxelize_raycast_scan_vs_oracle(reduce):
    """A SemanticKITTI-shaped raycast scan (~125k points per voxel set):
    the GPU voxeliser equals the oracle bit for bit, and its output feeds
    the engine directly."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import workloads
    pts = workloads.raycast_points(3).astype(np.float64)
    pts = np.concatenate([pts[:, :3], pts], axis=1)
    t = sc.voxelize(pts, 0.05, reduce)
    c, f, b = O.voxelize(pts, 0.05, reduce)
    np.testing.assert_array_equal(t.coords_numpy(), c)
    np.testing.assert_array_equal(t.features_numpy(), f)
    assert tuple(t.boundary) == tuple(b)


def test_voxelize_errors():
    import paper_2204_10319_b200 as sc
    with pytest.raises(ValueError, match="empty"):
        sc.voxelize(np.zeros((0, 3)), 1.0)
    with pytest.raises(ValueError, match="columns"):
        sc.voxelize(np.zeros((4, 2)), 1.0)
    with pytest.raises(ValueError, match="positive"):
        sc.voxelize(np.zeros((4, 3)), 0.0)
    with pytest.raises(ValueError, match="reduce"):
        sc.voxelize(np.zeros((4, 3)), 1.0, "max")


@pytest.mark.parametrize("reduce", ["mean", "first"])
def test_voxelize_batch_equals_per_scan_packing(reduce):
    """8 raw raycast scans -> one packed tensor in one device pass
    (scb_voxelize_batch) is bit-identical to voxelising each scan with the
    oracle (the reference's algorithm) and packing them along the batch
    column with the shared boundary, as the bench does."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import workloads
    scans = []
    for s in range(8):
        pts = workloads.raycast_points(s).astype(np.float64)
        scans.append(np.concatenate([pts[:, :3], pts], axis=1))
    t = sc.voxelize_batch(scans, 0.05, reduce)
    per = [O.voxelize(p, 0.05, reduce) for p in scans]
    boundary = tuple(int(max(x[2][d] for x in per)) for d in range(3))
    coords = np.concatenate([np.concatenate([np.full((x[0].shape[0], 1), i, np.int64),
                                             x[0][:, 1:]], 1) for i, x in enumerate(per)])
    feats = np.concatenate([x[1] for x in per])
    assert t.batch_size == 8 and tuple(t.boundary) == boundary
    np.testing.assert_array_equal(t.coords_numpy(), coords)
    np.testing.assert_array_equal(t.features_numpy(), feats)
    # the single-scan entry point is the B = 1 case of the same kernels
    one = sc.voxelize_batch([scans[5]], 0.05, reduce)
    c5, f5, b5 = per[5]
    np.testing.assert_array_equal(one.coords_numpy(), c5)
    np.testing.assert_array_equal(one.features_numpy(), f5)
    assert tuple(one.boundary) == tuple(b5)


def test_voxelize_batch_errors():
    import paper_2204_10319_b200 as sc
    with pytest.raises(ValueError, match="empty"):
        sc.voxelize_batch([np.ones((3, 4)), np.zeros((0, 4))], 1.0)
    with pytest.raises(ValueError, match="columns"):
        sc.voxelize_batch([np.ones((3, 4)), np.ones((3, 5))], 1.0)
    with pytest.raises(ValueError, match="64"):
        sc.voxelize_batch([np.ones((2, 4))] * 65, 1.0)
