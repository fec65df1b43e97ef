"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, unpack_pairs
from oracle import sparseconv_oracle as O


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _map_cases(g):
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_ptr")})
    return keys


def test_maps_and_output_coords_bit_exact(golden):
    g = golden("maps")
    cases = _map_cases(g)
    assert len(cases) >= 48
    for key in cases:
        coords = g[key + "_in"]
        bnd = tuple(int(x) for x in g[key + "_boundary"])
        boundary, batch = bnd[:-1], bnd[-1]
        dim = len(boundary)
        k = int(re.search(r"(?:^|_)k(\d+)", key).group(1))
        s = int(re.search(r"_s(\d+)", key).group(1))
        bout = boundary if s == 1 else O.downsample_boundary(boundary, s)
        out = O.output_coords(coords, k, s, bout, batch)
        np.testing.assert_array_equal(out, g[key + "_out"], err_msg=key)
        pairs = O.kernel_map(coords, boundary, out, k, s, batch)
        want = unpack_pairs(g[key + "_ptr"], g[key + "_pairs"])
        assert len(pairs) == k ** dim
        for n, (a, b) in enumerate(zip(pairs, want)):
            np.testing.assert_array_equal(a, b, err_msg=f"{key} offset {n}")
        if key + "_swptr" in g.files:
            sw = O.swap_roles(pairs)
            want_sw = unpack_pairs(g[key + "_swptr"], g[key + "_swpairs"])
            for a, b in zip(sw, want_sw):
                np.testing.assert_array_equal(a, b)


def test_worked_example_and_dense_block(golden):
    g = golden("maps")
    out = O.output_coords(np.array([[0, 3, 5]]), 2, 2, (2, 3))
    np.testing.assert_array_equal(out, g["worked2d_out"])
    np.testing.assert_array_equal(out, [[0, 1, 2]])
    block = np.array([[0, x, y, z] for x in range(8) for y in range(8) for z in range(8)])
    pairs = O.kernel_map(block, (8, 8, 8), block, 3, 1)
    sizes = [p.shape[0] for p in pairs]
    np.testing.assert_array_equal(sizes, g["block8_sizes"])
    assert sum(sizes) == 10648


def test_layers_match_reference(golden):
    g = golden("layers")
    keys = sorted({k[:-3] for k in g.files if k.endswith("_in")})
    assert len(keys) == 48
    for key in keys:
        k = int(re.search(r"(?:^|_)k(\d+)", key).group(1))
        s = int(re.search(r"_s(\d+)", key).group(1))
        coords, feat, w = g[key + "_in"], g[key + "_feat"], g[key + "_w"]
        oc, of, ob, pairs = O.conv_forward(coords, feat, (14, 13, 12), w, k, s,
                                           return_map=True)
        np.testing.assert_array_equal(oc, g[key + "_outc"], err_msg=key)
        ref = g[key + "_outf"]
        assert of.dtype == ref.dtype
        scale = max(float(np.abs(ref.astype(np.float32)).max()), 1e-6)
        tol = 1e-5 if ref.dtype == np.float32 else 2e-3
        assert np.abs(of.astype(np.float32) - ref.astype(np.float32)).max() / scale <= tol, key
        if key + "_invf" in g.files:
            inv = O.inverse_forward(of, g[key + "_w2"], pairs, coords.shape[0])
            ref2 = g[key + "_invf"]
            scale = max(float(np.abs(ref2.astype(np.float32)).max()), 1e-6)
            assert np.abs(inv.astype(np.float32) - ref2.astype(np.float32)).max() / scale <= tol


def test_plans_gather_scatter(golden):
    g = golden("plans")
    coords = g["in"]
    pairs = O.kernel_map(coords, (9, 9, 9), coords, 3, 1)
    for skip in (0, 1):
        pl = O.plan(pairs, coords.shape[0], coords.shape[0], 13 if skip else None)
        for name in ("buffer_offsets", "row_input", "row_output", "in_indptr", "in_rows",
                     "out_indptr", "out_rows"):
            np.testing.assert_array_equal(pl[name], g[f"skip{skip}_{name}"], err_msg=name)
        buf = O.gather(g[f"skip{skip}_feat"], pl)
        np.testing.assert_array_equal(buf, g[f"skip{skip}_buffer"])
        sc = O.scatter(g[f"skip{skip}_partial"], pl, coords.shape[0])
        np.testing.assert_array_equal(sc, g[f"skip{skip}_scatter"])


def test_network_toy_minkunet(golden):
    g = golden("network")
    doc = json.loads(str(g["doc"]))
    for prec in ("fp32", "fp16"):
        d = dict(doc, precision=prec)
        weights, pw = O.build_params(d)
        for lid, w in weights.items():
            np.testing.assert_array_equal(w, g[f"{prec}_w_{lid}"])
        oc, of = O.network_forward(d, g["in"], g["feat"], (16, 16, 16), params=(weights, pw))
        np.testing.assert_array_equal(oc, g[f"{prec}_outc"])
        ref = g[f"{prec}_outf"].astype(np.float32)
        rel = np.linalg.norm(of.astype(np.float32) - ref) / np.linalg.norm(ref)
        assert rel <= (1e-6 if prec == "fp32" else 2e-3), (prec, rel)


def test_config1_map_digest(golden):
    from paper_2204_10319_b200 import workloads
    g = golden("config1")
    coords, feats, boundary = workloads.config1_cloud()
    assert coords.shape[0] == int(g["n"])
    assert tuple(boundary) == tuple(int(b) for b in g["boundary"])
    assert _digest(coords) == str(g["coords_digest"])
    assert hashlib.sha256(feats.tobytes()).hexdigest() == str(g["feat_digest"])
    pairs = O.kernel_map(coords, boundary, coords, 3, 1)
    ptr = np.zeros(28, np.int64)
    np.cumsum([p.shape[0] for p in pairs], out=ptr[1:])
    flat = np.concatenate(pairs, 0)
    np.testing.assert_array_equal(np.diff(ptr), g["k3s1_sizes"])
    assert _digest(ptr, flat) == str(g["k3s1_digest"])
    bout = O.downsample_boundary(boundary, 2)
    out2 = O.output_coords(coords, 2, 2, bout)
    assert _digest(out2) == str(g["k2s2_out_digest"])
    pairs2 = O.kernel_map(coords, boundary, out2, 2, 2)
    ptr2 = np.zeros(9, np.int64)
    np.cumsum([p.shape[0] for p in pairs2], out=ptr2[1:])
    assert _digest(ptr2, np.concatenate(pairs2, 0)) == str(g["k2s2_digest"])


def test_partition_hand_trace():
    assert O.partition([100, 95, 90, 50, 48], 0.1, range(5)) == [(0, 3), (3, 5)]
    with pytest.raises(ValueError):
        O.partition([1, 2], 1.5, range(2))


def test_voxelize_matches_reference_golden():
    """oracle.voxelize == the unmodified reference's core.voxelize
    (tests/golden/voxelize.npz), bit-exact coordinates and features."""
    g = np.load(GOLDEN / "voxelize.npz")
    i = 0
    while f"v{i}_points" in g.files:
        dims, first = (int(x) for x in g[f"v{i}_meta"])
        c, f, b = O.voxelize(g[f"v{i}_points"], float(g[f"v{i}_vs"][0]),
                             "first" if first else "mean", dims)
        np.testing.assert_array_equal(c, g[f"v{i}_coords"])
        np.testing.assert_array_equal(f, g[f"v{i}_feats"])
        assert tuple(b) == tuple(int(x) for x in g[f"v{i}_boundary"])
        i += 1
    assert i >= 6


def test_minkunet_chain_oracle_vs_reference(golden):
    """The MinkUNet-shaped 43-conv chain (reference JSON schema) on a
    16k-voxel raycast crop: the oracle restatement against the unmodified
    reference's Network.forward (tests/golden/make_golden.py
    gen_minkunet_chain)."""
    import hashlib
    g = golden("minkunet_chain")
    doc = json.loads(str(g["doc"]))
    boundary = tuple(int(b) for b in g["boundary"])
    for prec in ("fp32", "fp16"):
        d = dict(doc, precision=prec)
        oc, of = O.network_forward(d, g["in"].astype(np.int64), g["feat"], boundary)
        h = hashlib.sha256()
        a = np.ascontiguousarray(oc.astype(np.int64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
        assert h.hexdigest() == str(g[f"{prec}_outc_digest"])
        ref = g[f"{prec}_outf"].astype(np.float64)
        rel = np.linalg.norm(of.astype(np.float64) - ref) / np.linalg.norm(ref)
        assert rel <= (1e-5 if prec == "fp32" else 5e-3), (prec, rel)
