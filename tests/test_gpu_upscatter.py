"""Transposed K = s layers in scatter form (scb_conv_transposed_scatter):
the inverse layer replaying a k2 s2 map (reference execution.py:512-551)
computed from the coarse side, each product stored to its one fine row.
Checked against the oracle's inverse_forward and against the gather-form
fused kernel (SCB_UPSCATTER=0) on the same inputs."""

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


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _down_up(sc, coords, boundary, bs, c_fine, c_coarse, c_out, rng, ep=None, shuffle=False):
    from paper_2204_10319_b200 import execution as X
    n = coords.shape[0]
    if shuffle:
        coords = coords[rng.permutation(n)]
    f = rng.standard_normal((n, c_fine)).astype(np.float16)
    t = sc.SparseTensor(coords, np.zeros((n, 1), np.float32), 1, boundary, bs)
    t = t.replace_features(torch.from_numpy(f).cuda())
    wd = sc.WeightTensor(rng.normal(0, 0.1, (8, c_fine, c_coarse)).astype(np.float32), 2, 3)
    wu = sc.WeightTensor(rng.normal(0, 0.1, (8, c_coarse, c_out)).astype(np.float32), 2, 3)
    opts = sc.ExecOptions(dataflow="fused", index_kind="hash")
    cache = {}
    d = sc.sparse_conv_forward(t, wd, sc.LayerSpec(2, 2, c_fine, c_coarse, reuse_key="d"), None,
                               cache, opts)
    spec = sc.LayerSpec(2, 1, c_coarse, c_out, transposed=True, reuse_key="d")
    kmap = cache["d"].kmap.swap_roles()
    assert kmap.onehot and kmap._parent is not None
    got = sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep).features
    saved = X._UPSCATTER
    X._UPSCATTER = False
    try:
        gather_form = sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep).features
    finally:
        X._UPSCATTER = saved
    return coords, f, d, wd, wu, got, gather_form, cache


@pytest.mark.parametrize("c_coarse,c_out", [(32, 16), (48, 48), (64, 48), (96, 96), (128, 96), (256, 128), (256, 256)])
def test_scatter_equals_gather_form_and_oracle(sc, rng, c_coarse, c_out):
    boundary, bs = (48, 48, 16), 2
    coords = random_coords(rng, boundary, 0.08, bs)
    coords, f, d, wd, wu, got, gf, cache = _down_up(sc, coords, boundary, bs, 16, c_coarse, c_out,
                                                   rng, shuffle=True)
    assert got.shape == (coords.shape[0], c_out)
    # one product per output row: the same tcgen05 MMAs as the gather form
    assert torch.equal(got, gf)
    pairs = cache["d"].kmap.pairs
    want = O.inverse_forward(d.features.cpu().numpy(), wu.weights, pairs, coords.shape[0])
    assert _rel(got.float().cpu().numpy(), want) < 1e-2


def test_scatter_epilogue_bn_bias_relu(sc, rng):
    boundary, bs = (40, 40, 12), 1
    coords = random_coords(rng, boundary, 0.25, bs)
    ep = {"scale": torch.linspace(0.5, 1.5, 96, device="cuda"),
          "shift": torch.linspace(-0.1, 0.1, 96, device="cuda"),
          "bias": torch.full((96,), 0.02, device="cuda"), "relu": True}
    coords, f, d, wd, wu, got, gf, cache = _down_up(sc, coords, boundary, bs, 32, 64, 96, rng, ep)
    assert torch.equal(got, gf)
    pairs = cache["d"].kmap.pairs
    raw = O.inverse_forward(d.features.cpu().numpy(), wu.weights, pairs, coords.shape[0])
    want = np.maximum(raw.astype(np.float32) * np.linspace(0.5, 1.5, 96, dtype=np.float32)
                      + np.linspace(-0.1, 0.1, 96, dtype=np.float32) + 0.02, 0)
    assert _rel(got.float().cpu().numpy(), want) < 1e-2


def test_scatter_full_scan_level0(sc, rng):
    """The bench's level-0 -> level-1 -> level-0 pair on an uncropped raycast
    scan (121k fine rows): every fine row written once, equal to the gather form."""
    from paper_2204_10319_b200 import workloads
    c, _, b = workloads.semantickitti_scan(2)
    coords, f, d, wd, wu, got, gf, cache = _down_up(sc, c, b, 1, 32, 96, 96, rng)
    assert torch.equal(got, gf)
    assert torch.isfinite(got.float()).all()


def test_scatter_keeps_transposed_hits_lazy(sc, rng):
    """The scatter form reads the strided map's hit matrix; the swapped map's
    own hit matrix is only built when something asks for it (and then equals
    the transpose)."""
    boundary, bs = (32, 32, 12), 1
    coords = random_coords(rng, boundary, 0.25, bs)
    coords, f, d, wd, wu, got, gf, cache = _down_up(sc, coords, boundary, bs, 16, 32, 32, rng)
    down = cache["d"].kmap
    up = down.swap_roles()
    h = up.hits[:, : up.n_out].cpu().numpy()
    hd = down.hits[:, : down.n_out].cpu().numpy()
    for n in range(8):
        p = np.nonzero(hd[n] >= 0)[0]
        np.testing.assert_array_equal(h[n][hd[n][p]], p)
    assert ((h >= 0).sum(0) == 1).all()   # one-hot: every fine row has one parent


def _pointwise(sc, f, w, ep=None, concat=None, dense=True):
    from paper_2204_10319_b200 import execution as X
    saved = X._DENSE_K1
    X._DENSE_K1 = dense
    try:
        return X._run_fused(f, None, w, sc.ExecOptions(dataflow="fused"), ep, concat)
    finally:
        X._DENSE_K1 = saved


@pytest.mark.parametrize("c_in,c_split,c_out", [(96, None, 19), (64, None, 128), (128, None, 96), (96, None, 48),
                                                (128, 96, 96), (160, 96, 96), (256, None, 256),
                                                (48, 32, 64)])
def test_pointwise_dense_equals_gather_form_and_oracle(sc, rng, c_in, c_split, c_out):
    """K = 1 s = 1 layers through scb_conv_pointwise (dense TMA tiles, the skip
    concatenation read in place) against the gather-form kernel's identity map
    and the oracle's matmul (reference execution.py:456-459)."""
    n = 20000 + 77
    x = rng.standard_normal((n, c_in)).astype(np.float16)
    w = sc.WeightTensor(rng.normal(0, 0.1, (1, c_in, c_out)).astype(np.float32), 1, 3)
    ep = {"scale": torch.linspace(0.5, 1.5, c_out, device="cuda"),
          "shift": torch.linspace(-0.1, 0.1, c_out, device="cuda"), "relu": True}
    xt = torch.from_numpy(x).cuda()
    f, cat = (xt, None) if c_split is None else (xt[:, :c_split].contiguous(),
                                                 xt[:, c_split:].contiguous())
    got = _pointwise(sc, f, w, ep, cat)
    want = _pointwise(sc, f, w, ep, cat, dense=False)
    assert got.shape == (n, c_out)
    assert torch.equal(got, want)
    ref = np.maximum((x.astype(np.float32) @ w.weights[0]) * np.linspace(0.5, 1.5, c_out,
                     dtype=np.float32) + np.linspace(-0.1, 0.1, c_out, dtype=np.float32), 0)
    assert _rel(got.float().cpu().numpy(), ref) < 1e-2


def test_pointwise_no_epilogue_small(sc, rng):
    """Fewer rows than one tile, no epilogue operands."""
    x = torch.from_numpy(rng.standard_normal((37, 32)).astype(np.float16)).cuda()
    w = sc.WeightTensor(rng.normal(0, 0.1, (1, 32, 16)).astype(np.float32), 1, 3)
    got = _pointwise(sc, x, w)
    want = _pointwise(sc, x, w, dense=False)
    assert torch.equal(got, want)


def test_dense_forms_reject_bad_arguments(sc):
    """The C ABI validates its arguments (reference error convention: the
    Python layer re-raises the library message)."""
    from paper_2204_10319_b200 import _native as nat
    x = torch.zeros((10, 12), dtype=torch.float16, device="cuda")
    w = torch.zeros((1, 16, 16), dtype=torch.float16, device="cuda")
    out = torch.zeros((10, 16), dtype=torch.float16, device="cuda")
    with pytest.raises(Exception, match="c_in"):
        nat.call("scb_conv_pointwise", nat.ptr(x), 12, 12, None, 0, 10, 12, nat.ptr(w), 16,
                 nat.ptr(out), 16, None, None, None, 0, nat.stream_handle())
    with pytest.raises(Exception, match="child"):
        nat.call("scb_conv_transposed_scatter", nat.ptr(x), 16, 10, 16, None, 8, nat.ptr(w), 16,
                 nat.ptr(out), 16, 10, None, None, None, 0, nat.stream_handle())
