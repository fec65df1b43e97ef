"""Config 4 (BASELINE.json): the CenterPoint-style encoder on a
nuScenes-shaped multi-sweep cloud, B200 engine vs the CPU oracle (k3 s2
strided levels with up to 8 candidates per input, 5-channel stem)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sweeps():
    from paper_2204_10319_b200 import workloads
    return workloads.nuscenes_sweeps(0, azimuths=300)


def test_centerpoint_encoder_matches_oracle(sweeps):
    import paper_2204_10319_b200 as sc
    from oracle import sparseconv_oracle as O
    from paper_2204_10319_b200.centerpoint import EngineCenterPoint
    from oracle.models import centerpoint_oracle as forward_oracle
    coords, feats, boundary = sweeps
    assert coords.shape[0] > 5000 and feats.shape[1] == 5
    model = EngineCenterPoint(5, 0)
    t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 1),
                             sc.PrecisionMode.FP16_STORAGE)
    out = model.forward(t, sc.ExecOptions(dataflow="auto", index_kind="hash"))
    oc, of, ob = forward_oracle(model.params, coords, O.quantize(feats, "fp16"), boundary)
    np.testing.assert_array_equal(out.coords_numpy(), oc)
    assert tuple(out.boundary) == tuple(ob)
    got = out.features_numpy().astype(np.float64)
    rel = np.linalg.norm(got - of) / np.linalg.norm(of.astype(np.float64))
    assert rel <= 1e-2, rel


def test_centerpoint_staged_equals_fused_maps(sweeps):
    """Both dataflows see the same maps and agree within the FP16 tolerance."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200.centerpoint import EngineCenterPoint
    coords, feats, boundary = sweeps
    model = EngineCenterPoint(5, 1)
    outs = []
    for df in ("staged", "fused"):
        t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 1),
                                 sc.PrecisionMode.FP16_STORAGE)
        outs.append(model.forward(t, sc.ExecOptions(dataflow=df)))
    np.testing.assert_array_equal(outs[0].coords_numpy(), outs[1].coords_numpy())
    a = outs[0].features_numpy().astype(np.float64)
    b = outs[1].features_numpy().astype(np.float64)
    assert np.linalg.norm(a - b) / np.linalg.norm(a) <= 1e-2
