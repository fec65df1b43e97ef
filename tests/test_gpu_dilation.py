"""SparseConv3d with dilation (north_star's module; a B200 extension, the
reference's windows are dense cubes): dilated maps bit-exact against the
oracle's restatement with scaled offsets, layer outputs within the FP32 /
FP16 tolerances in both dataflows, and the module's strided/transposed pair."""

import numpy as np
import pytest
import torch

from conftest import random_coords
from oracle import sparseconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sc():
    import paper_2204_10319_b200 as sc
    return sc


@pytest.mark.parametrize("k,d", [(3, 2), (3, 3), (5, 2), (2, 2)])
def test_dilated_map_bit_exact(sc, rng, k, d):
    boundary, bs = (30, 30, 30), 2
    coords = random_coords(rng, boundary, 0.08, bs)
    t = sc.SparseTensor(coords, np.zeros((coords.shape[0], 1), np.float32), 1, boundary, bs)
    off = sc.enumerate_offsets(3, k)
    kmap = sc.map_search(sc.build_index(t, "hash"), t.coords, off, 1, dilation=d)
    want = O.kernel_map(coords, boundary, coords, k, 1, bs, dilation=d)
    for got, ref in zip(kmap.pairs, want):
        np.testing.assert_array_equal(got, ref)
    if d > 1:  # a real dilation changes the map
        plain = O.kernel_map(coords, boundary, coords, k, 1, bs)
        assert any(a.shape != b.shape or not np.array_equal(a, b) for a, b in zip(plain, want))


@pytest.mark.parametrize("precision,dataflow,tol", [("fp32", "staged", 1e-4),
                                                    ("fp16", "fused", 1e-2),
                                                    ("fp16", "staged", 1e-2)])
def test_dilated_layer_vs_oracle(sc, rng, precision, dataflow, tol):
    boundary = (40, 40, 40)
    coords = random_coords(rng, boundary, 0.05)
    f = rng.standard_normal((coords.shape[0], 32)).astype(np.float32)
    if precision == "fp16":
        f = O.quantize(f, "fp16")
    conv = sc.SparseConv3d(32, 48, 3, dilation=2, seed=3)
    t = sc.SparseTensor(coords, f, 1, boundary, 1)
    out = conv(t, options=sc.ExecOptions(dataflow=dataflow))
    oc, of, _ = O.conv_forward(coords, f, boundary, conv.weight.weights, 3, 1, dilation=2)
    np.testing.assert_array_equal(out.coords_numpy(), oc)
    got = out.features_numpy().astype(np.float64)
    rel = np.linalg.norm(got - of) / np.linalg.norm(of.astype(np.float64))
    assert rel <= tol, rel


def test_module_strided_transposed_pair_and_bias(sc, rng):
    boundary = (32, 32, 32)
    coords = random_coords(rng, boundary, 0.1)
    f = O.quantize(rng.standard_normal((coords.shape[0], 16)).astype(np.float32), "fp16")
    t = sc.SparseTensor(coords, f, 1, boundary, 1)
    down = sc.SparseConv3d(16, 32, 2, stride=2, reuse_key="d1", seed=1)
    up = sc.SparseConv3d(32, 16, 2, stride=2, transposed=True, reuse_key="d1", bias=True, seed=2)
    up.bias.fill_(0.25)
    cache = {}
    y = down(t, cache)
    z = up(y, cache)
    assert z.features.shape == (coords.shape[0], 16)
    np.testing.assert_array_equal(z.coords_numpy(), coords)
    oc, of, _, pairs = O.conv_forward(coords, f, boundary, down.weight.weights, 2, 2,
                                      return_map=True)
    np.testing.assert_array_equal(y.coords_numpy(), oc)
    want = O.inverse_forward(of, up.weight.weights, pairs, coords.shape[0]).astype(np.float64) + 0.25
    got = z.features_numpy().astype(np.float64)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-2
    with pytest.raises(ValueError):
        up(y)   # no map cache
