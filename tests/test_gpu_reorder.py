"""Presence-mask row reordering (B200 extension): masks, the
sort, relabelled maps and per-tile offset words against numpy restatements
of the oracle's map, and the models' outputs unchanged by the relabelling."""

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


def _oracle_masks(coords, boundary, batch_size=1):
    pairs = O.kernel_map(coords, boundary, coords, 3, 1, batch_size)
    m = np.zeros(coords.shape[0], np.int64)
    for n, p in enumerate(pairs):
        m[p[:, 1]] |= 1 << n
    return m, pairs


def _oracle_perm(masks, batch, V=27):
    """Stable sort by the mask with offsets ranked by decreasing frequency
    (most frequent -> bit 0, rarest -> bit V-1), words visited in Gray-code
    order; the batch column is not part of the key (rows of different batch
    entries interleave)."""
    counts = np.array([((masks >> n) & 1).sum() for n in range(V)])
    pos = np.array([sum(1 for u in range(V) if counts[u] > counts[n]
                        or (counts[u] == counts[n] and u < n)) for n in range(V)])
    key = np.zeros_like(masks)
    for n in range(V):
        key |= ((masks >> n) & 1) << pos[n]
    g = key.copy()   # Gray-code order: sort by the word's index along the Gray sequence
    shift = key >> 1
    while shift.any():
        g ^= shift
        shift >>= 1
    return np.argsort(g, kind="stable")


def _clouds(rng):
    from paper_2204_10319_b200 import workloads
    c, _, b = workloads.semantickitti_scan(3)
    return [(random_coords(rng, (18, 18, 18), 0.2, 2), (18, 18, 18), 2),
            (np.asarray(c, np.int64), tuple(b), 1)]


def test_presence_masks_sort_and_relabelled_map(sc, rng):
    from paper_2204_10319_b200.mapping import presence_masks, reorder_by_presence
    for coords, boundary, bs in _clouds(rng):
        t = sc.SparseTensor(coords, np.zeros((coords.shape[0], 1), np.float32), 1, boundary, bs)
        want_m, pairs = _oracle_masks(coords, boundary, bs)
        m, counts = presence_masks(t.coordset, 3, "hash")
        np.testing.assert_array_equal(m.cpu().numpy().astype(np.int64) & ((1 << 27) - 1), want_m)
        np.testing.assert_array_equal(counts.cpu().numpy(), [p.shape[0] for p in pairs])
        p = reorder_by_presence(t.coordset, 3, "hash")
        perm = p.perm.cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(perm, _oracle_perm(want_m, coords[:, 0]))
        np.testing.assert_array_equal(p.coords.cpu().numpy(), coords[perm])
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.shape[0])
        # the map over the relabelled set = the oracle's pairs, relabelled
        kmap = sc.map_search(sc.build_index(p, "hash"), p.coords, sc.enumerate_offsets(3, 3), 1)
        for n, (got, ref) in enumerate(zip(kmap.pairs, pairs)):
            rel = np.stack([inv[ref[:, 0]], inv[ref[:, 1]]], 1)
            rel = rel[np.argsort(rel[:, 1], kind="stable")]
            np.testing.assert_array_equal(got, rel)
        # per-tile active-offset words
        hits = kmap.hits[:, : perm.shape[0]].cpu().numpy()
        nt = (perm.shape[0] + 127) // 128
        pad = np.full((27, nt * 128), -1, np.int64)
        pad[:, : perm.shape[0]] = hits
        want_t = ((pad.reshape(27, nt, 128) >= 0).any(2).astype(np.int64)
                  << np.arange(27)[:, None]).sum(0)
        np.testing.assert_array_equal(kmap.tile_masks().cpu().numpy().astype(np.int64), want_t)


def test_permute_rows_gather_scatter(sc, rng):
    from paper_2204_10319_b200.mapping import permute_rows
    for c, dt in ((4, torch.float16), (5, torch.float16), (19, torch.float32), (24, torch.float16),
                  (3, torch.int32)):
        x = torch.from_numpy(rng.standard_normal((1000, c))).to(dt).cuda()
        idx = torch.from_numpy(rng.permutation(1000).astype(np.int32)).cuda()
        g = permute_rows(x, idx)
        assert torch.equal(g, x[idx.long()])
        assert torch.equal(permute_rows(g, idx, scatter=True), x)


def test_fused_skips_match_dense(sc, rng):
    """A layer over a relabelled set (sparse tile words) equals the same
    layer in flat-key order, row for row, bit for bit: a skipped block
    contributes exact zeros to every row of its tile."""
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.mapping import permute_rows, reorder_by_presence
    c, _, b = workloads.semantickitti_scan(2)
    n = c.shape[0]
    t = sc.SparseTensor(c, np.zeros((n, 1), np.float32), 1, b, 1)
    f = torch.from_numpy(rng.standard_normal((n, 64)).astype(np.float16)).cuda()
    w = sc.WeightTensor(rng.normal(0, 1 / np.sqrt(27 * 64), (27, 64, 96)).astype(np.float32), 3, 3)
    opts = sc.ExecOptions(dataflow="fused", index_kind="hash")
    dense = sc.sparse_conv_forward(t.replace_features(f), w, sc.LayerSpec(3, 1, 64, 96), None,
                                   None, opts).features
    p = reorder_by_presence(t.coordset, 3, "hash")
    x = sc.SparseTensor._wrap(permute_rows(f, p.perm), 1, b, 1, p)
    out = sc.sparse_conv_forward(x, w, sc.LayerSpec(3, 1, 64, 96), None, None, opts)
    kmap = p.maps[(3, 1, -1)][1]
    bits = kmap.tile_masks().cpu().numpy().astype(np.int64)
    frac = np.mean([bin(int(v)).count("1") for v in bits]) / 27
    assert frac < 0.6, frac  # the relabelling makes most (tile, offset) blocks absent
    back = permute_rows(out.features, p.perm, scatter=True)
    assert torch.equal(back, dense)


@pytest.mark.parametrize("model", ["minkunet", "centerpoint"])
def test_model_reorder_is_identical(sc, model):
    """The models with and without level relabelling: same coordinates, and
    features equal up to fp16 rounding (single layers are bit-identical,
    test_fused_skips_match_dense; across 50 layers a few elements land on
    the other side of an fp16 rounding boundary)."""
    from paper_2204_10319_b200 import workloads
    if model == "minkunet":
        from paper_2204_10319_b200.minkunet import EngineMinkUNet
        c, f, b = workloads.semantickitti_scan(0)
        mk = lambda r: EngineMinkUNet(0.5, 4, 0, reorder=r)
    else:
        from paper_2204_10319_b200.centerpoint import EngineCenterPoint
        c, f, b = workloads.nuscenes_sweeps(0, azimuths=1000)
        mk = lambda r: EngineCenterPoint(5, 0, reorder=r)
    outs = []
    for r in (False, True):
        t = sc.quantize_features(sc.SparseTensor(c, f, 1, b, 1), sc.PrecisionMode.FP16_STORAGE)
        o = mk(r).forward(t, sc.ExecOptions(dataflow="auto", index_kind="hash"))
        outs.append((o.coords_numpy(), o.features_numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    a, b = outs[0][1].astype(np.float64), outs[1][1].astype(np.float64)
    assert np.linalg.norm(a - b) / np.linalg.norm(a) <= 1e-3


def test_masked_search_equals_symmetric_search(sc, rng):
    """scb_map_search_masked (probe only the present offsets) = the
    symmetric map search, hit matrix and tile words, on a relabelled level."""
    from paper_2204_10319_b200.mapping import map_search_masked, reorder_by_presence
    for coords, boundary, bs in _clouds(rng):
        t = sc.SparseTensor(coords, np.zeros((coords.shape[0], 1), np.float32), 1, boundary, bs)
        p = reorder_by_presence(t.coordset, 3, "hash")
        idx = sc.build_index(p, "hash")
        off = sc.enumerate_offsets(3, 3)
        ref = sc.map_search(idx, p.coords, off, 1)
        got = map_search_masked(idx, p, off, p.derived[("presence", 3)])
        n = coords.shape[0]
        assert torch.equal(got.hits[:, :n], ref.hits[:, :n])
        assert torch.equal(got.tile_masks(), ref.tile_masks())
        # the engine's cached k3 map of a relabelled level is the masked one
        out = sc.sparse_conv_forward(
            sc.SparseTensor._wrap(torch.zeros((n, 8), dtype=torch.float16, device="cuda"), 1,
                                  boundary, bs, p),
            sc.WeightTensor(np.zeros((27, 8, 8), np.float32), 3, 3), sc.LayerSpec(3, 1, 8, 8),
            None, None, sc.ExecOptions(dataflow="fused", index_kind="hash"))
        assert out.features.shape[0] == n
        assert torch.equal(p.maps[(3, 1, -1)][1].hits[:, :n], ref.hits[:, :n])


def test_onehot_order_transposed_layer(sc, rng):
    """The transposed k2 layer runs over rows sorted by their parent offset
    (scb_onehot_order + scb_conv_implicit_rows): one active offset per tile,
    and the output equals the output-row-order run bit for bit."""
    import os
    from paper_2204_10319_b200 import workloads
    c, _, b = workloads.semantickitti_scan(1)
    n = c.shape[0]
    t = sc.SparseTensor(c, np.zeros((n, 1), np.float32), 1, b, 1)
    f = torch.from_numpy(rng.standard_normal((n, 32)).astype(np.float16)).cuda()
    wd = sc.WeightTensor(rng.normal(0, 0.1, (8, 32, 64)).astype(np.float32), 2, 3)
    wu = sc.WeightTensor(rng.normal(0, 0.1, (8, 64, 48)).astype(np.float32), 2, 3)
    opts = sc.ExecOptions(dataflow="fused", index_kind="hash")
    cache = {}
    d = sc.sparse_conv_forward(t.replace_features(f), wd,
                               sc.LayerSpec(2, 2, 32, 64, reuse_key="d"), None, cache, opts)
    kmap = cache["d"].kmap.swap_roles()
    assert kmap.onehot
    perm, hp, tm = kmap.onehot_order()
    p = perm.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(np.sort(p), np.arange(n))
    h = kmap.hits[:, :n].cpu().numpy()
    off = np.where((h >= 0).any(0), (h >= 0).argmax(0), 8)
    np.testing.assert_array_equal(off[p], np.sort(off, kind="stable"))
    np.testing.assert_array_equal(p, np.argsort(off, kind="stable"))
    np.testing.assert_array_equal(hp[:, :n].cpu().numpy(), h[:, p])
    bits = tm.cpu().numpy().astype(np.int64)
    assert np.mean([bin(int(v)).count("1") for v in bits]) < 1.1
    ep = {"scale": torch.full((48,), 1.1, device="cuda"),
          "shift": torch.full((48,), 0.01, device="cuda"), "relu": True}
    spec = sc.LayerSpec(2, 1, 64, 48, transposed=True, reuse_key="d")
    from paper_2204_10319_b200 import execution as X
    saved = X._UPSCATTER
    X._UPSCATTER = False   # the gather-form kernel (the scatter form takes precedence)
    try:
        want = sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep).features
        os.environ["SCB_ONEHOT"] = "1"   # opt-in (the whole MinkUNet step measured no gain)
        try:
            got = sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep).features
        finally:
            os.environ.pop("SCB_ONEHOT")
    finally:
        X._UPSCATTER = saved
    assert torch.equal(got, want)


@pytest.mark.parametrize("boundary,bs", [((40, 40, 12), 2), ((8192, 8192, 256), 4)])
def test_output_coords_key_widths(sc, rng, boundary, bs):
    """k2 s2 output coordinates with 32-bit sort keys (small grids) and
    64-bit keys (> 2^32 output cells) equal the oracle, incl. the chain."""
    from paper_2204_10319_b200.mapping import compute_output_coords_chain
    n = 20000
    keys = np.unique(rng.integers(0, bs * int(np.prod(boundary)), size=n))
    coords = np.empty((keys.shape[0], 4), np.int64)
    rem = keys
    for d in range(2, -1, -1):
        coords[:, d + 1] = rem % boundary[d]
        rem = rem // boundary[d]
    coords[:, 0] = rem
    t = sc.SparseTensor(coords, np.zeros((coords.shape[0], 1), np.float32), 1, boundary, bs)
    off = sc.enumerate_offsets(3, 2)
    levels = compute_output_coords_chain(t.coordset, [(off, 2)] * 3)
    cur, cb = coords, boundary
    for oc, ob in levels:
        nb = O.downsample_boundary(cb, 2)
        want = O.output_coords(cur, 2, 2, nb, bs)
        np.testing.assert_array_equal(oc.cpu().numpy(), want)
        assert tuple(ob) == tuple(nb)
        cur, cb = want, nb
    ob = O.downsample_boundary(boundary, 2)
    got = sc.compute_output_coords(t, off, 2, ob, bs)
    np.testing.assert_array_equal(got.cpu().numpy(), O.output_coords(coords, 2, 2, ob, bs))
