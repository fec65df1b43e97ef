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
    """Stable sort by (batch, mask with offsets ranked by decreasing
    frequency: most frequent -> bit 0, rarest -> bit V-1)."""
    counts = np.array([((masks >> n) & 1).sum() for n in range(V)])
    pos = np.array([sum(1 for u in range(V) if counts[u] > counts[n]
                        or (counts[u] == counts[n] and u < n)) for n in range(V)])
    key = np.zeros_like(masks)
    for n in range(V):
        key |= ((masks >> n) & 1) << pos[n]
    key |= batch.astype(np.int64) << V
    return np.argsort(key, kind="stable")


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
