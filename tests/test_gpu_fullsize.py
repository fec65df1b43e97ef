"""Parity on the bench's own clouds (BASELINE.json configs 3/5): the
SemanticKITTI-shaped raycast scans the bench runs, uncropped, one scan and
the 8-scan 1,000,366-voxel pack, against the CPU oracle — output
coordinates and kernel maps bit-exact per offset at every level of the
MinkUNet pyramid (k3 s1, k2 s2, transposed), in flat-key order and in the
presence-relabelled order the bench uses — plus size-independent
properties (map symmetry, transposition round trips)."""

import numpy as np
import pytest
import torch

from oracle import sparseconv_oracle as O

pytestmark = pytest.mark.gpu


def _pack(seeds):
    from paper_2204_10319_b200 import workloads
    scans = [workloads.semantickitti_scan(s) for s in seeds]
    boundary = tuple(int(max(s[2][d] for s in scans)) for d in range(3))
    coords = np.concatenate([np.concatenate([np.full((s[0].shape[0], 1), i, np.int64),
                                             s[0][:, 1:]], 1) for i, s in enumerate(scans)])
    feats = np.concatenate([s[1] for s in scans]).astype(np.float32)
    return coords, feats, boundary, len(seeds)


@pytest.fixture(scope="module", params=["one_scan", "pack8"])
def cloud(request):
    return _pack([0] if request.param == "one_scan" else range(8))


def _oracle_pyramid(coords, boundary, bs):
    """Per level: coords, boundary, k3 map, and the k2 s2 map to the next."""
    levels = []
    c, b = coords, boundary
    for i in range(5):
        lvl = {"coords": c, "boundary": b, "k3": O.kernel_map(c, b, c, 3, 1, bs)}
        if i < 4:
            nb = O.downsample_boundary(b, 2)
            nc = O.output_coords(c, 2, 2, nb, bs)
            lvl["down"] = O.kernel_map(c, b, nc, 2, 2, bs)
            c, b = nc, nb
        levels.append(lvl)
    return levels


@pytest.fixture(scope="module")
def oracle_levels(cloud):
    coords, _, boundary, bs = cloud
    return _oracle_pyramid(coords, boundary, bs)


def _relabel(pairs, inv_in, inv_out):
    out = []
    for p in pairs:
        q = np.stack([inv_in[p[:, 0]], inv_out[p[:, 1]]], 1)
        out.append(q[np.argsort(q[:, 1], kind="stable")])
    return out


def _inv(perm):
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    return inv


def _assert_maps(got, want):
    assert len(got) == len(want)
    for n, (g, w) in enumerate(zip(got, want)):
        np.testing.assert_array_equal(g, w, err_msg=f"offset {n}")


def _engine_levels(cloud, reorder):
    """The bench model's own pyramid (EngineMinkUNet._start + finish)."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    coords, feats, boundary, bs = cloud
    model = EngineMinkUNet(0.5, 4, 0, reorder=reorder)
    t = sc.SparseTensor(coords, feats, 1, boundary, bs)
    opts = sc.ExecOptions(index_kind="hash")
    l0, finish, _ = model._start(t.coordset, opts)
    finish()
    levels, cs = [], l0
    for i in range(5):
        levels.append(cs)
        if i < 4:
            cs = cs.maps[(2, 2, 0)][0]
    return levels


@pytest.mark.parametrize("reorder", [False, True])
def test_pyramid_maps_bit_exact(cloud, oracle_levels, reorder):
    """Every level's coordinates, k3 s1 map, k2 s2 map and transposed map
    against the oracle (relabelled by the level permutations when the
    levels are presence-reordered)."""
    levels = _engine_levels(cloud, reorder)
    invs = []
    for i, (cs, ref) in enumerate(zip(levels, oracle_levels)):
        c = cs.coords.cpu().numpy().astype(np.int64)
        if reorder:
            perm = cs.perm.cpu().numpy().astype(np.int64)
            np.testing.assert_array_equal(np.sort(perm), np.arange(perm.shape[0]))
            np.testing.assert_array_equal(c, ref["coords"][perm])
            invs.append(_inv(perm))
        else:
            assert cs.perm is None
            np.testing.assert_array_equal(c, ref["coords"])
            invs.append(np.arange(c.shape[0]))
        assert cs.boundary == tuple(ref["boundary"])
        k3 = cs.maps[(3, 1, -1)][1]
        _assert_maps(k3.pairs, _relabel(ref["k3"], invs[i], invs[i]))
    for i in range(4):
        down = levels[i].maps[(2, 2, 0)][1]
        want = _relabel(oracle_levels[i]["down"], invs[i], invs[i + 1])
        _assert_maps(down.pairs, want)
        _assert_maps(down.swap_roles().pairs, O.swap_roles(want))


def test_symmetric_map_property(cloud):
    import paper_2204_10319_b200 as sc
    coords, feats, boundary, bs = cloud
    t = sc.SparseTensor(coords, feats, 1, boundary, bs)
    offsets = sc.enumerate_offsets(3, 3)
    kmap = sc.map_search(sc.build_index(t, "hash"), t.coords, offsets, 1)
    n = coords.shape[0]
    hits = kmap.hits[:, :n].long()
    k = torch.arange(n, device=hits.device)
    assert torch.equal(hits[13], k)  # centre offset: every output is its own input
    for v in range(13):
        j = hits[v]
        present = j >= 0
        assert torch.equal(hits[26 - v][j[present]], k[present])
        assert int(present.sum()) == int((hits[26 - v] >= 0).sum())
    direct = sc.map_search(sc.build_index(t, "auto"), t.coords, offsets, 1, use_symmetry=False)
    assert torch.equal(direct.hits[:, :n], kmap.hits[:, :n])


def test_transpose_round_trip(cloud):
    import paper_2204_10319_b200 as sc
    coords, feats, boundary, bs = cloud
    t = sc.SparseTensor(coords, feats, 1, boundary, bs)
    offsets = sc.enumerate_offsets(3, 2)
    out = sc.compute_output_coords(t, offsets, 2, tuple(-(-b // 2) for b in t.boundary), bs)
    kmap = sc.map_search(sc.build_index(t, "hash"), out, offsets, 2)
    back = kmap.swap_roles().swap_roles()
    assert torch.equal(back.hits[:, : kmap.n_out], kmap.hits[:, : kmap.n_out])
    assert kmap.total == t.num_points  # k2 s2: every input in exactly one (offset, output)


def test_fused_layer_vs_oracle_fullsize(cloud, oracle_levels):
    """One 96->96 k3 layer of the bench's level 0 (presence-relabelled, as
    the bench runs it) against the oracle's f64 result, FP16 tolerance."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200.mapping import permute_rows
    coords, _, boundary, bs = cloud
    rng = np.random.default_rng(0)
    n = coords.shape[0]
    f = O.quantize(rng.standard_normal((n, 96)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(27 * 96), (27, 96, 96)).astype(np.float32)
    levels = _engine_levels((coords, f, boundary, bs), True)
    p0 = levels[0]
    x = sc.SparseTensor._wrap(permute_rows(torch.from_numpy(f).cuda(), p0.perm), 1, boundary, bs,
                              p0)
    out = sc.sparse_conv_forward(x, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, 96, 96), None,
                                 None, sc.ExecOptions(dataflow="fused"))
    got = permute_rows(out.features, p0.perm, scatter=True).float().cpu().numpy()
    want = np.zeros((n, 96), np.float64)
    for v, pr in enumerate(oracle_levels[0]["k3"]):
        want[pr[:, 1]] += f[pr[:, 0]].astype(np.float64) @ w[v].astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-2, rel
