"""Full-size (BASELINE.json config 5 shard: 8 packed SemanticKITTI-shaped
scans, ~1M voxels) checks through size-independent properties, where the
CPU oracle is too slow to run: map symmetry (derive_symmetric_maps,
mapping.py:322-339), the strided-coordinate rule (mapping.py:216-248),
transposition round trips (mapping.py:277-286), and the fused layer equal to
the staged layer within the FP16 tolerance."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch():
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import workloads
    scans = [workloads.semantickitti_scan(s) for s in range(8)]
    boundary = tuple(int(max(s[2][d] for s in scans)) for d in range(3))
    coords = np.concatenate([np.concatenate([np.full((s[0].shape[0], 1), i, np.int64),
                                             s[0][:, 1:]], 1) for i, s in enumerate(scans)])
    feats = np.concatenate([s[1] for s in scans]).astype(np.float32)
    t = sc.SparseTensor(coords, feats, 1, boundary, 8)
    return coords, feats, boundary, t


def test_fullsize_symmetric_map_property(batch):
    import paper_2204_10319_b200 as sc
    coords, _, boundary, t = batch
    assert coords.shape[0] > 900_000
    offsets = sc.enumerate_offsets(3, 3)
    kmap = sc.map_search(sc.build_index(t, "hash"), t.coords, offsets, 1)
    hits = kmap.hits[:, : coords.shape[0]].long()
    V = 27
    k = torch.arange(coords.shape[0], device=hits.device)
    assert torch.equal(hits[13], k)  # centre offset: every output is its own input
    for n in range(13):
        j = hits[n]
        present = j >= 0
        # M[V-1-n] holds (k, j) for every (j, k) in M[n]
        assert torch.equal(hits[V - 1 - n][j[present]], k[present])
        assert int(present.sum()) == int((hits[V - 1 - n] >= 0).sum())
    # the hash and the direct (non-symmetric) search agree everywhere
    direct = sc.map_search(sc.build_index(t, "hash"), t.coords, offsets, 1, use_symmetry=False)
    assert torch.equal(direct.hits[:, : coords.shape[0]], kmap.hits[:, : coords.shape[0]])


def test_fullsize_strided_chain_rule(batch):
    import paper_2204_10319_b200 as sc
    coords, _, boundary, t = batch
    levels = sc.prepare_strided_chain(t, [sc.LayerSpec(2, 2, 4, 4)] * 4, sc.ExecOptions())
    prev_c, prev_b = torch.from_numpy(coords).cuda(), boundary
    for lvl in levels:
        c = lvl.coords.long()
        want = torch.unique(torch.cat([prev_c[:, :1], prev_c[:, 1:] // 2], 1), dim=0)
        assert torch.equal(c, want)  # unique and in ascending (b, x, y, z) order
        assert lvl.boundary == tuple(-(-b // 2) for b in prev_b)
        prev_c, prev_b = c, lvl.boundary


def test_fullsize_transpose_round_trip(batch):
    import paper_2204_10319_b200 as sc
    _, _, _, t = batch
    offsets = sc.enumerate_offsets(3, 2)
    out = sc.compute_output_coords(t, offsets, 2, tuple(-(-b // 2) for b in t.boundary), 8)
    kmap = sc.map_search(sc.build_index(t, "hash"), out, offsets, 2)
    back = kmap.swap_roles().swap_roles()
    assert torch.equal(back.hits[:, : kmap.n_out], kmap.hits[:, : kmap.n_out])
    # k2 s2: every input row lands in exactly one (offset, output)
    assert kmap.total == t.num_points


def test_fullsize_fused_equals_staged(batch):
    import paper_2204_10319_b200 as sc
    coords, feats, boundary, t = batch
    rng = np.random.default_rng(0)
    f = torch.from_numpy(rng.standard_normal((coords.shape[0], 96)).astype(np.float16)).cuda()
    x = t.replace_features(f)
    w = sc.WeightTensor(rng.normal(0, 1 / np.sqrt(27 * 96), (27, 96, 96)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, 96, 96)
    a = sc.sparse_conv_forward(x, w, spec, None, None, sc.ExecOptions(dataflow="staged"))
    b = sc.sparse_conv_forward(x, w, spec, None, None, sc.ExecOptions(dataflow="fused"))
    a, b = a.features.float(), b.features.float()
    assert float((a - b).norm() / a.norm()) <= 1e-2
