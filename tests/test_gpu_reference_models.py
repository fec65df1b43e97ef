"""Whole-network parity on the bench's OWN workloads against the UNMODIFIED
reference: the bench graphs run through the
reference package's public API (oracle/reference_runner.py over
baseline/_ref, numpy glue only for residual add / concat) on full,
uncropped clouds, and the B200 engine runs the same graphs the way the
bench does (fused dataflow, presence-reordered levels, FP16 storage).
Output coordinates must be identical and features within the FP16 budget
(1e-2 relative L2)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle.reference_runner import import_reference
    try:
        return import_reference()
    except ImportError as e:
        pytest.skip(str(e))


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("width", [1.0])
def test_minkunet_full_scan_vs_reference(ref, width):
    """MinkUNet 1.0x on an uncropped SemanticKITTI-shaped raycast scan
    (~121k voxels): the bench's model, exactly as the bench runs it."""
    import paper_2204_10319_b200 as sc
    from oracle.reference_runner import minkunet_reference
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    coords, feats, boundary = workloads.semantickitti_scan(0)
    assert coords.shape[0] > 100_000
    model = EngineMinkUNet(width, 4, 0)
    t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 1),
                             sc.PrecisionMode.FP16_STORAGE)
    out = model.forward(t, sc.ExecOptions(dataflow="auto", index_kind="hash"))
    rc, rf, rb = minkunet_reference(ref, model.params, width, coords, feats, boundary)
    np.testing.assert_array_equal(out.coords_numpy(), rc)
    assert _rel(out.features_numpy(), rf) <= 1e-2


def test_minkunet_packed_batch_vs_reference(ref):
    """Two scans packed along the batch column (the bench's multi-scan
    tensor) against the reference run on the same packed tensor."""
    import paper_2204_10319_b200 as sc
    from oracle.reference_runner import minkunet_reference
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    scans = [workloads.semantickitti_scan(s) for s in (1, 2)]
    boundary = tuple(int(max(s[2][d] for s in scans)) for d in range(3))
    coords = np.concatenate([np.concatenate([np.full((s[0].shape[0], 1), i, np.int64),
                                             s[0][:, 1:]], 1) for i, s in enumerate(scans)])
    feats = np.concatenate([s[1] for s in scans]).astype(np.float32)
    model = EngineMinkUNet(0.5, 4, 3)
    t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 2),
                             sc.PrecisionMode.FP16_STORAGE)
    out = model.forward(t, sc.ExecOptions(dataflow="auto", index_kind="hash"))
    rc, rf, _ = minkunet_reference(ref, model.params, 0.5, coords, feats, boundary, 2)
    np.testing.assert_array_equal(out.coords_numpy(), rc)
    assert _rel(out.features_numpy(), rf) <= 1e-2


def test_centerpoint_bench_size_vs_reference(ref):
    """Config 4: the CenterPoint-style encoder on the bench's nuScenes-shaped
    10-sweep cloud (3000 azimuths, ~147k voxels)."""
    import paper_2204_10319_b200 as sc
    from oracle.reference_runner import centerpoint_reference
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.centerpoint import EngineCenterPoint
    coords, feats, boundary = workloads.nuscenes_sweeps(0, azimuths=3000)
    assert coords.shape[0] > 120_000
    model = EngineCenterPoint(5, 0)
    t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 1),
                             sc.PrecisionMode.FP16_STORAGE)
    out = model.forward(t, sc.ExecOptions(dataflow="auto", index_kind="hash"))
    rc, rf, rb = centerpoint_reference(ref, model.params, coords, feats, boundary)
    np.testing.assert_array_equal(out.coords_numpy(), rc)
    assert tuple(out.boundary) == tuple(rb)
    assert _rel(out.features_numpy(), rf) <= 1e-2
