"""Parity of the CUDA path with the reference (golden vectors) and the oracle.

Integer work (maps, output coordinates, plans, gathers) must be bit-exact;
features must match within 1e-4 relative L2 (FP32 storage) and 1e-2
(FP16 storage), the north-star tolerances.  All calls go through the C ABI.
"""

import re

import numpy as np
import pytest
import torch

from conftest import random_coords, unpack_pairs
from oracle import sparseconv_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "fp16": 1e-2}


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def sc():
    import paper_2204_10319_b200 as m
    assert torch.cuda.is_available()
    return m


def _map_keys(g):
    return sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_ptr")})


@pytest.mark.parametrize("kind", ["hash", "grid"])
def test_maps_bit_exact_vs_golden(sc, golden, kind):
    g = golden("maps")
    for key in _map_keys(g):
        coords = g[key + "_in"]
        bnd = tuple(int(x) for x in g[key + "_boundary"])
        boundary, batch = bnd[:-1], bnd[-1]
        k = int(re.search(r"(?:^|_)k(\d+)", key).group(1))
        s = int(re.search(r"_s(\d+)", key).group(1))
        off = sc.enumerate_offsets(len(boundary), k)
        bout = boundary if s == 1 else sc.downsample_boundary(boundary, s)
        out = sc.compute_output_coords(coords, off, s, bout, batch)
        np.testing.assert_array_equal(out.cpu().numpy(), g[key + "_out"], err_msg=key)
        idx = sc.build_index(coords, kind, boundary, batch)
        kmap = sc.map_search(idx, out, off, s)
        want = unpack_pairs(g[key + "_ptr"], g[key + "_pairs"])
        for n, (a, b) in enumerate(zip(kmap.pairs, want)):
            np.testing.assert_array_equal(a, b, err_msg=f"{key} offset {n} ({kind})")
        if key + "_swptr" in g.files:
            sw = kmap.swap_roles()
            for a, b in zip(sw.pairs, unpack_pairs(g[key + "_swptr"], g[key + "_swpairs"])):
                np.testing.assert_array_equal(a, b, err_msg=key + " swapped")


def test_direct_search_equals_symmetric(sc, rng):
    coords = random_coords(rng, (12, 12, 12), 0.15)
    off = sc.enumerate_offsets(3, 3)
    idx = sc.build_index(coords, "hash", (12, 12, 12))
    a = sc.map_search(idx, coords, off, 1, use_symmetry=True)
    b = sc.map_search(idx, coords, off, 1, use_symmetry=False)
    for x, y in zip(a.pairs, b.pairs):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a.sizes, a.sizes[::-1])
    # derive_symmetric_maps from the searched lower half reproduces the map
    half_pairs = [p if n <= 13 else np.empty((0, 2), np.int64) for n, p in enumerate(b.pairs)]
    assert sum(p.shape[0] for p in half_pairs) < b.total
    full = sc.derive_symmetric_maps(_from_pairs(sc, half_pairs, off, coords.shape[0]))
    for x, y in zip(full.pairs, b.pairs):
        np.testing.assert_array_equal(x, y)


def _from_pairs(sc, pairs, off, n, n_out=None, stride=1):
    ptr = np.zeros(len(pairs) + 1, np.int64)
    np.cumsum([p.shape[0] for p in pairs], out=ptr[1:])
    flat = np.concatenate(pairs, 0)
    return sc.KernelMap(torch.from_numpy(ptr).cuda(), np.diff(ptr),
                        torch.from_numpy(flat[:, 0].astype(np.int32)).cuda(),
                        torch.from_numpy(flat[:, 1].astype(np.int32)).cuda(), off, stride, n,
                        n if n_out is None else n_out)


def test_plan_with_duplicate_output_per_offset(sc):
    """A hand-built map with several entries for one (output, offset) pair
    (the reference's scatter tests build these) cannot use the fixed-width
    position table: the plan is marked general and scatters through the
    output CSR (scb_scatter_csr), folding 2048 x 0.5 exactly in f32
    (reference tests/test_execution.py::test_fp16_accumulates_in_fp32)."""
    m = 2048
    pairs = [np.stack([np.arange(m), np.zeros(m, np.int64)], 1)]
    off = sc.KernelOffsets(np.zeros((1, 3), np.int64), 1, 3)
    plan = sc.build_gather_scatter_plan(_from_pairs(sc, pairs, off, m, n_out=1, stride=2))
    assert plan.general
    buf = torch.full((m, 3), 0.5, dtype=torch.float16, device="cuda")
    for order in ("weight_stationary", "output_stationary"):
        out = sc.scatter_accumulate(buf, plan, 1, order).cpu().numpy()
        np.testing.assert_array_equal(out, np.full((1, 3), 1024.0, np.float32))
    # mixed: ascending buffer-row fold over a random many-to-one map
    rng = np.random.default_rng(3)
    k = np.sort(rng.integers(0, 5, 300))
    pairs = [np.stack([np.arange(300), k], 1)]
    plan = sc.build_gather_scatter_plan(_from_pairs(sc, pairs, off, 300, n_out=5, stride=2))
    vals = rng.standard_normal((300, 7)).astype(np.float32)
    got = sc.scatter_accumulate(torch.from_numpy(vals).cuda(), plan, 5).cpu().numpy()
    want = np.zeros((5, 7), np.float64)
    np.add.at(want, k, vals.astype(np.float64))
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)


def test_dense_block_and_worked_example(sc, golden):
    g = golden("maps")
    out = sc.compute_output_coords(np.array([[0, 3, 5]]), sc.enumerate_offsets(2, 2), 2, (2, 3))
    np.testing.assert_array_equal(out.cpu().numpy(), [[0, 1, 2]])
    only00 = sc.KernelOffsets(np.array([[0, 0]]), 1, 2)
    assert sc.compute_output_coords(np.array([[0, 3, 5]]), only00, 2, (2, 3)).shape[0] == 0
    block = np.array([[0, x, y, z] for x in range(8) for y in range(8) for z in range(8)])
    for kind in ("grid", "hash"):
        kmap = sc.map_search(sc.build_index(block, kind, (8, 8, 8)), block,
                             sc.enumerate_offsets(3, 3), 1)
        np.testing.assert_array_equal(kmap.sizes, g["block8_sizes"])
        assert kmap.total == 10648


def test_index_queries(sc, rng):
    boundary = (10, 10, 10)
    coords = random_coords(rng, boundary, 0.5)
    grid = sc.build_index(coords, "grid", boundary)
    hashed = sc.build_index(coords, "hash", boundary)
    probes = rng.integers(-2, 12, size=(10_000, 4))
    probes[:, 0] = rng.integers(0, 2, size=10_000)
    a, b = grid.query(probes).cpu().numpy(), hashed.query(probes).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    # oracle semantics of the query
    keys = O.flatten(coords, boundary)
    order = np.argsort(keys)
    np.testing.assert_array_equal(a, O._lookup(keys[order], order, boundary, 1, probes))
    bad = np.array([[0, -1, 0, 0], [0, 10, 0, 0], [1, 0, 0, 0]])
    np.testing.assert_array_equal(hashed.query(bad).cpu().numpy(), [-1, -1, -1])
    # forced collision: keys 1 and 5 (same low bits) both found
    two = np.array([[0, 0, 0, 1], [0, 0, 0, 5]])
    np.testing.assert_array_equal(sc.build_index(two, "hash", (1, 1, 16)).query(two).cpu().numpy(),
                                  [0, 1])
    with pytest.raises(sc.GridCapacityError, match="hash"):
        sc.build_index(np.array([[0, 0, 0, 0]]), "grid", (1024, 1024, 1024), cell_cap=1 << 20)
    assert sc.build_index(np.array([[0, 0, 0, 0]]), "auto", (1024, 1024, 1024),
                          cell_cap=1 << 20).kind == "hash"


def test_config1_maps_digest(sc, golden):
    import hashlib
    from paper_2204_10319_b200 import workloads
    g = golden("config1")
    coords, feats, boundary = workloads.config1_cloud()
    t = sc.SparseTensor(coords, feats, 1, boundary, 1)
    off = sc.enumerate_offsets(3, 3)
    kmap = sc.map_search(sc.build_index(t, "hash"), t.coords, off, 1)
    np.testing.assert_array_equal(kmap.sizes, g["k3s1_sizes"])
    ptr = np.zeros(28, np.int64)
    np.cumsum(kmap.sizes, out=ptr[1:])
    flat = np.concatenate(kmap.pairs, 0)

    def dig(*arrs):
        h = hashlib.sha256()
        for a in arrs:
            a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
            h.update(str(a.shape).encode())
            h.update(a.tobytes())
        return h.hexdigest()

    assert dig(ptr, flat) == str(g["k3s1_digest"])
    off2 = sc.enumerate_offsets(3, 2)
    bout = sc.downsample_boundary(boundary, 2)
    out2 = sc.compute_output_coords(t, off2, 2, bout)
    assert dig(out2.cpu().numpy()) == str(g["k2s2_out_digest"])
    k2 = sc.map_search(sc.build_index(t, "grid"), out2, off2, 2)
    ptr2 = np.zeros(9, np.int64)
    np.cumsum(k2.sizes, out=ptr2[1:])
    assert dig(ptr2, np.concatenate(k2.pairs, 0)) == str(g["k2s2_digest"])


def test_plans_gather_scatter_vs_golden(sc, golden):
    g = golden("plans")
    coords = g["in"]
    kmap = sc.map_search(sc.build_index(coords, "grid", (9, 9, 9)), coords,
                         sc.enumerate_offsets(3, 3), 1)
    for skip in (0, 1):
        plan = sc.build_gather_scatter_plan(kmap, skip_center=bool(skip))
        np.testing.assert_array_equal(plan.buffer_offsets, g[f"skip{skip}_buffer_offsets"])
        for name in ("row_input", "row_output", "in_indptr", "in_rows", "out_indptr", "out_rows"):
            np.testing.assert_array_equal(getattr(plan, name), g[f"skip{skip}_{name}"])
        feats = g[f"skip{skip}_feat"]
        for order in ("weight_stationary", "input_stationary"):
            buf = sc.gather(feats, plan, order).cpu().numpy()
            np.testing.assert_array_equal(buf, g[f"skip{skip}_buffer"])  # bit-exact
        out = sc.scatter_accumulate(g[f"skip{skip}_partial"], plan, coords.shape[0],
                                    "output_stationary").cpu().numpy()
        np.testing.assert_allclose(out, g[f"skip{skip}_scatter"], rtol=2e-6, atol=2e-6)


def test_fp16_gather_and_accumulate(sc, rng):
    coords = random_coords(rng, (9, 9, 9), 0.2)
    kmap = sc.map_search(sc.build_index(coords, "hash", (9, 9, 9)), coords,
                         sc.enumerate_offsets(3, 3), 1)
    plan = sc.build_gather_scatter_plan(kmap)
    for c in (3, 4, 8, 16, 24, 64):
        f = rng.standard_normal((coords.shape[0], c)).astype(np.float16)
        buf = sc.gather(f, plan).cpu().numpy()
        assert buf.dtype == np.float16
        np.testing.assert_array_equal(buf, f[plan.row_input])
    # 2048 x 0.5 accumulates exactly in >= fp32 (reference tests/test_execution.py:132-142):
    # a synthetic map with 2048 offsets each contributing input n to output 0
    pairs = [np.array([[n, 0]], np.int64) for n in range(2048)]
    off = sc.KernelOffsets(np.zeros((2048, 1), np.int64), 2048, 1)
    k2 = _from_pairs(sc, pairs, off, 2048, n_out=1, stride=2)
    p2 = sc.build_gather_scatter_plan(k2)
    out = sc.scatter_accumulate(np.full((2048, 4), 0.5, np.float16), p2, 1, "output_stationary",
                                np.float16).cpu().numpy()
    assert out.dtype == np.float16 and (out == 1024.0).all()


def _layer_keys(g):
    return sorted({k[:-3] for k in g.files if k.endswith("_in")})


def test_layers_vs_golden(sc, golden):
    g = golden("layers")
    for key in _layer_keys(g):
        k = int(re.search(r"(?:^|_)k(\d+)", key).group(1))
        s = int(re.search(r"_s(\d+)", key).group(1))
        prec = key.rsplit("_", 1)[1]
        w = g[key + "_w"]
        t = sc.SparseTensor(g[key + "_in"], g[key + "_feat"], 1, (14, 13, 12), 1)
        spec = sc.LayerSpec(k, s, w.shape[1], w.shape[2], reuse_key="L")
        cache = {}
        out = sc.sparse_conv_forward(t, sc.WeightTensor(w, k, 3), spec, None, cache)
        np.testing.assert_array_equal(out.coords_numpy(), g[key + "_outc"], err_msg=key)
        of = out.features_numpy()
        ref = g[key + "_outf"]
        assert of.dtype == ref.dtype, key
        assert rel_l2(of, ref) <= TOL[prec], (key, rel_l2(of, ref))
        if key + "_invf" in g.files:
            w2 = g[key + "_w2"]
            inv = sc.inverse_conv_forward(
                out, sc.WeightTensor(w2, k, 3),
                sc.LayerSpec(k, 1, w2.shape[1], w2.shape[2], transposed=True, reuse_key="L"),
                cache)
            np.testing.assert_array_equal(inv.coords_numpy(), g[key + "_in"])
            assert inv.stride == 1 and inv.boundary == (14, 13, 12)
            ref2 = g[key + "_invf"]
            assert rel_l2(inv.features_numpy(), ref2) <= TOL[prec], (key, "inverse")


def test_network_toy_vs_golden(sc, golden):
    import json
    g = golden("network")
    doc = json.loads(str(g["doc"]))
    for prec in ("fp32", "fp16"):
        net = sc.Network.build(sc.NetworkConfig.from_dict(dict(doc, precision=prec)))
        for lid, w in net.weights.items():
            np.testing.assert_array_equal(w.weights, g[f"{prec}_w_{lid}"])
        out = net.forward(sc.SparseTensor(g["in"], g["feat"], 1, (16, 16, 16), 1))
        np.testing.assert_array_equal(out.coords_numpy(), g[f"{prec}_outc"])
        assert rel_l2(out.features_numpy(), g[f"{prec}_outf"]) <= TOL[prec]


@pytest.mark.parametrize("prec,dataflow", [("fp32", "staged"), ("fp16", "staged"),
                                           ("fp16", "fused")])
def test_minkunet_chain_vs_reference_network(sc, golden, prec, dataflow):
    """The engine's Network.forward over the MinkUNet-shaped 43-conv chain
    in the reference's JSON schema, against the unmodified reference's own
    Network.forward (tests/golden/minkunet_chain.npz): output coordinates
    bit-exact (digest), features within the north-star tolerance (FP32
    1e-4, FP16 1e-2 relative L2)."""
    import hashlib
    import json
    g = golden("minkunet_chain")
    doc = dict(json.loads(str(g["doc"])), precision=prec)
    boundary = tuple(int(b) for b in g["boundary"])
    net = sc.Network.build(sc.NetworkConfig.from_dict(doc))
    out = net.forward(sc.SparseTensor(g["in"], g["feat"], 1, boundary, 1),
                      options=sc.ExecOptions(dataflow=dataflow))
    oc = out.coords_numpy()
    h = hashlib.sha256()
    h.update(str(oc.shape).encode())
    h.update(np.ascontiguousarray(oc.astype(np.int64)).tobytes())
    assert h.hexdigest() == str(g[f"{prec}_outc_digest"])
    assert rel_l2(out.features_numpy(), g[f"{prec}_outf"]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("c_in,c_out", [(64, 64), (32, 48), (16, 16), (128, 96), (4, 32)])
def test_config1_layer_vs_oracle(sc, prec, c_in, c_out):
    from paper_2204_10319_b200 import workloads
    coords, _, boundary = workloads.config1_cloud()
    rng = np.random.default_rng(c_in * 7 + c_out)
    feats = O.quantize(rng.standard_normal((coords.shape[0], c_in)).astype(np.float32), prec)
    w = rng.normal(0, 1 / np.sqrt(27 * c_in), (27, c_in, c_out)).astype(np.float32)
    oc, of, _ = O.conv_forward(coords, feats, boundary, w, 3, 1)
    t = sc.SparseTensor(coords, feats, 1, boundary, 1)
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, c_in, c_out))
    np.testing.assert_array_equal(out.coords_numpy(), oc)
    assert rel_l2(out.features_numpy(), of) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_config2_down_up_vs_oracle(sc, prec):
    from paper_2204_10319_b200 import workloads
    coords, _, boundary = workloads.config1_cloud()
    rng = np.random.default_rng(2)
    feats = O.quantize(rng.standard_normal((coords.shape[0], 32)).astype(np.float32), prec)
    w1 = rng.normal(0, 1 / np.sqrt(8 * 32), (8, 32, 64)).astype(np.float32)
    w2 = rng.normal(0, 1 / np.sqrt(8 * 64), (8, 64, 32)).astype(np.float32)
    oc, of, ob, pairs = O.conv_forward(coords, feats, boundary, w1, 2, 2, return_map=True)
    inv = O.inverse_forward(of, w2, pairs, coords.shape[0])
    t = sc.SparseTensor(coords, feats, 1, boundary, 1)
    cache = {}
    d = sc.sparse_conv_forward(t, sc.WeightTensor(w1, 2, 3), sc.LayerSpec(2, 2, 32, 64, reuse_key="down"),
                               None, cache)
    assert d.num_points == 15271 and d.stride == 2 and d.boundary == tuple(ob)
    np.testing.assert_array_equal(d.coords_numpy(), oc)
    assert rel_l2(d.features_numpy(), of) <= TOL[prec]
    u = sc.inverse_conv_forward(d, sc.WeightTensor(w2, 2, 3),
                                sc.LayerSpec(2, 1, 64, 32, transposed=True, reuse_key="down"), cache)
    np.testing.assert_array_equal(u.coords_numpy(), coords)
    assert rel_l2(u.features_numpy(), inv) <= TOL[prec]


def test_grouping_strategies_are_invariant(sc, rng):
    coords = random_coords(rng, (20, 20, 20), 0.1)
    feats = rng.standard_normal((coords.shape[0], 16)).astype(np.float32)
    w = sc.WeightTensor(rng.normal(0, 0.1, (27, 16, 16)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, 16, 16)
    outs = []
    for strat in (sc.LayerStrategy.separate(), sc.LayerStrategy.symmetric_pairs(),
                  sc.LayerStrategy.dense_group(), sc.LayerStrategy(0.3, 500.0)):
        for opts in (sc.ExecOptions(), sc.ExecOptions(order="weight", index_kind="hash"),
                     sc.ExecOptions(map_reuse=False, index_kind="grid")):
            t = sc.SparseTensor(coords, feats, 1, (20, 20, 20), 1)
            outs.append(sc.sparse_conv_forward(t, w, spec, strat, None, opts).features_numpy())
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


def test_execute_groups_matches_per_offset(sc, rng):
    sizes = rng.integers(0, 300, size=8)
    buf = rng.standard_normal((int(sizes.sum()), 16)).astype(np.float32)
    weights = rng.standard_normal((8, 16, 24)).astype(np.float32)
    st = np.concatenate([[0], np.cumsum(sizes)])
    want = np.concatenate([buf[st[n]:st[n + 1]] @ weights[n] for n in range(8)])
    for eps, thr in ((0.0, 0.0), (1.0, float("inf")), (0.4, 150.0)):
        for dt in (np.float32, np.float16):
            got = sc.execute_groups(buf.astype(dt), weights, sc.build_grouping(sizes, eps, thr),
                                    sizes).cpu().numpy()
            assert rel_l2(got, want) <= (1e-6 if dt == np.float32 else 2e-3)


def test_error_conventions(sc, rng):
    coords = random_coords(rng, (8, 8, 8), 0.2)
    t = sc.SparseTensor(coords, rng.standard_normal((coords.shape[0], 4)), 1, (8, 8, 8), 1)
    w = sc.WeightTensor(np.zeros((27, 4, 8), np.float32), 3, 3)
    with pytest.raises(ValueError, match="channel mismatch"):
        sc.sparse_conv_forward(t, w, sc.LayerSpec(3, 1, 5, 8))
    with pytest.raises(ValueError, match="unsupported stride"):
        sc.LayerSpec(3, 3, 4, 8)
    with pytest.raises(ValueError, match="reuse key"):
        sc.LayerSpec(2, 1, 4, 8, transposed=True)
    with pytest.raises(KeyError, match="no cached map"):
        sc.inverse_conv_forward(t, sc.WeightTensor(np.zeros((8, 4, 4), np.float32), 2, 3),
                                sc.LayerSpec(2, 1, 4, 4, transposed=True, reuse_key="x"), {})
    with pytest.raises(ValueError, match="unique"):
        sc.SparseTensor(np.array([[0, 1, 1, 1], [0, 1, 1, 1]]), np.zeros((2, 1)), 1, (4, 4, 4))
    with pytest.raises(ValueError, match="outside boundary"):
        sc.SparseTensor(np.array([[0, 4, 1, 1]]), np.zeros((1, 1)), 1, (4, 4, 4))
    with pytest.raises(ValueError, match="batch index"):
        sc.SparseTensor(np.array([[1, 0, 1, 1]]), np.zeros((1, 1)), 1, (4, 4, 4), 1)
    kmap = sc.map_search(sc.build_index(coords, "hash", (8, 8, 8)),
                         sc.compute_output_coords(coords, sc.enumerate_offsets(3, 2), 2, (4, 4, 4)),
                         sc.enumerate_offsets(3, 2), 2)
    with pytest.raises(ValueError, match="stride-1"):
        sc.derive_symmetric_maps(kmap)
    with pytest.raises(ValueError, match="unknown pointwise"):
        sc.pointwise_apply(t, "gelu")


def test_pointwise_ops(sc, rng):
    coords = random_coords(rng, (8, 8, 8), 0.2)
    f = rng.standard_normal((coords.shape[0], 6)).astype(np.float32)
    t = sc.SparseTensor(coords, f, 1, (8, 8, 8))
    b = rng.normal(size=6).astype(np.float32)
    s, h = rng.uniform(0.8, 1.2, 6).astype(np.float32), rng.normal(0, .05, 6).astype(np.float32)
    np.testing.assert_array_equal(sc.pointwise_apply(t, "relu").features_numpy(), np.maximum(f, 0))
    np.testing.assert_allclose(sc.pointwise_apply(t, "bias_add", bias=b).features_numpy(), f + b,
                               rtol=1e-6)
    np.testing.assert_allclose(sc.pointwise_apply(t, "bn_fold", scale=s, shift=h).features_numpy(),
                               f * s + h, rtol=1e-6, atol=1e-7)
    with pytest.raises(ValueError, match="channel count"):
        sc.pointwise_apply(t, "bias_add", bias=np.zeros(3))


def test_empty_and_isolated(sc):
    one = np.array([[0, 2, 2, 2]])
    t = sc.SparseTensor(one, np.ones((1, 4), np.float32), 1, (5, 5, 5))
    kmap = sc.map_search(sc.build_index(t, "hash"), t.coords, sc.enumerate_offsets(3, 3), 1)
    assert kmap.total == 1 and kmap.sizes[13] == 1
    w = np.random.default_rng(0).normal(size=(27, 4, 8)).astype(np.float32)
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, 4, 8))
    np.testing.assert_allclose(out.features_numpy(), np.ones((1, 4), np.float32) @ w[13], rtol=1e-6)
    # a strided layer whose output set is empty is not possible for non-empty
    # input; an empty input yields an empty output
    e = sc.SparseTensor(np.zeros((0, 4), np.int64), np.zeros((0, 4), np.float32), 1, (5, 5, 5))
    out = sc.sparse_conv_forward(e, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, 4, 8))
    assert out.num_points == 0
    w2 = np.zeros((8, 4, 4), np.float32)
    d = sc.sparse_conv_forward(e, sc.WeightTensor(w2, 2, 3), sc.LayerSpec(2, 2, 4, 4))
    assert d.num_points == 0


def test_4d_and_2d_layers_vs_oracle(sc):
    for dim, bnd in ((2, (30, 27)), (4, (6, 7, 5, 6))):
        rng = np.random.default_rng(dim)
        coords = random_coords(rng, bnd, 0.2)
        f = rng.standard_normal((coords.shape[0], 8)).astype(np.float32)
        for k, s in ((3, 1), (3, 2), (2, 2)):
            w = rng.normal(0, 0.2, (k ** dim, 8, 8)).astype(np.float32)
            oc, of, _ = O.conv_forward(coords, f, bnd, w, k, s)
            out = sc.sparse_conv_forward(sc.SparseTensor(coords, f, 1, bnd), sc.WeightTensor(w, k, dim),
                                         sc.LayerSpec(k, s, 8, 8))
            np.testing.assert_array_equal(out.coords_numpy(), oc)
            assert rel_l2(out.features_numpy(), of) <= 1e-4


@pytest.mark.parametrize("c_in,c_out", [(64, 64), (32, 48), (16, 16), (96, 128), (256, 256),
                                         (16, 20)])
def test_fused_dataflow_vs_oracle(sc, c_in, c_out):
    """The implicit-GEMM kernel (gather fused into the tcgen05 operand load)
    against the oracle: k3 s1, k2 s2 and the transposed k2 layer."""
    from paper_2204_10319_b200 import workloads
    coords, _, boundary = workloads.config1_cloud()
    rng = np.random.default_rng(c_in + 3 * c_out)
    feats = O.quantize(rng.standard_normal((coords.shape[0], c_in)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(27 * c_in), (27, c_in, c_out)).astype(np.float32)
    oc, of, _ = O.conv_forward(coords, feats, boundary, w, 3, 1)
    opts = sc.ExecOptions(dataflow="fused")
    t = sc.SparseTensor(coords, feats, 1, boundary, 1)
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, c_in, c_out),
                                 None, None, opts)
    assert rel_l2(out.features_numpy(), of) <= 1e-2
    w1 = rng.normal(0, 0.1, (8, c_in, c_out)).astype(np.float32)
    w2 = rng.normal(0, 0.1, (8, c_out, c_in)).astype(np.float32)
    doc, dof, _, pairs = O.conv_forward(coords, feats, boundary, w1, 2, 2, return_map=True)
    cache = {}
    d = sc.sparse_conv_forward(t, sc.WeightTensor(w1, 2, 3),
                               sc.LayerSpec(2, 2, c_in, c_out, reuse_key="d"), None, cache, opts)
    np.testing.assert_array_equal(d.coords_numpy(), doc)
    assert rel_l2(d.features_numpy(), dof) <= 1e-2
    u = sc.inverse_conv_forward(d, sc.WeightTensor(w2, 2, 3),
                                sc.LayerSpec(2, 1, c_out, c_in, transposed=True, reuse_key="d"),
                                cache, None, opts)
    uf = O.inverse_forward(dof, w2, pairs, coords.shape[0])
    assert rel_l2(u.features_numpy(), uf) <= 1e-2


@pytest.mark.parametrize("dataflow", ["staged", "fused"])
def test_epilogue_bn_residual_relu(sc, rng, dataflow):
    coords = random_coords(rng, (20, 20, 20), 0.1)
    n = coords.shape[0]
    f = O.quantize(rng.standard_normal((n, 32)).astype(np.float32), "fp16")
    r = O.quantize(rng.standard_normal((n, 48)).astype(np.float32), "fp16")
    w = rng.normal(0, 0.05, (27, 32, 48)).astype(np.float32)
    s = rng.uniform(0.8, 1.2, 48).astype(np.float32)
    h = rng.normal(0, 0.05, 48).astype(np.float32)
    _, base, _ = O.conv_forward(coords, f, (20, 20, 20), w, 3, 1)
    want = np.maximum(base.astype(np.float32) * s + h + r.astype(np.float32), 0)
    t = sc.SparseTensor(coords, f, 1, (20, 20, 20))
    res = sc.SparseTensor(coords, r, 1, (20, 20, 20))
    ep = {"scale": torch.from_numpy(s).cuda(), "shift": torch.from_numpy(h).cuda(),
          "residual": res, "relu": True}
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, 32, 48), None,
                                 None, sc.ExecOptions(dataflow=dataflow), epilogue=ep)
    got = out.features_numpy().astype(np.float32)
    assert rel_l2(got, want) <= 1e-2
    assert (got >= 0).all()


@pytest.mark.parametrize("c_in,c_out", [(64, 96), (128, 256), (32, 32), (96, 19)])
def test_fused_pointwise_layer(sc, rng, c_in, c_out):
    """K=1 layer through the implicit kernel (V = 1, identity map, BN + ReLU
    in the epilogue) against the oracle (execution.py:472-477)."""
    coords = random_coords(rng, (24, 24, 24), 0.2)
    n = coords.shape[0]
    f = O.quantize(rng.standard_normal((n, c_in)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(c_in), (1, c_in, c_out)).astype(np.float32)
    s = rng.uniform(0.8, 1.2, c_out).astype(np.float32)
    h = rng.normal(0, 0.05, c_out).astype(np.float32)
    _, base, _ = O.conv_forward(coords, f, (24, 24, 24), w, 1, 1)
    want = np.maximum(base.astype(np.float32) * s + h, 0)
    t = sc.SparseTensor(coords, f, 1, (24, 24, 24))
    ep = {"scale": torch.from_numpy(s).cuda(), "shift": torch.from_numpy(h).cuda(), "relu": True}
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 1, 3), sc.LayerSpec(1, 1, c_in, c_out),
                                 None, None, sc.ExecOptions(dataflow="fused"), epilogue=ep)
    assert rel_l2(out.features_numpy().astype(np.float32), want) <= 1e-2


@pytest.mark.parametrize("c_in", [4, 5, 12])
def test_fused_narrow_input_channels(sc, rng, c_in):
    """C_in not a multiple of 8 (the 4-channel MinkUNet stem, 5-channel
    nuScenes stem) is zero-padded for the implicit kernel."""
    coords = random_coords(rng, (20, 20, 20), 0.15)
    f = O.quantize(rng.standard_normal((coords.shape[0], c_in)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(27 * c_in), (27, c_in, 32)).astype(np.float32)
    _, want, _ = O.conv_forward(coords, f, (20, 20, 20), w, 3, 1)
    out = sc.sparse_conv_forward(sc.SparseTensor(coords, f, 1, (20, 20, 20)),
                                 sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, c_in, 32), None,
                                 None, sc.ExecOptions(dataflow="fused"))
    assert rel_l2(out.features_numpy(), want) <= 1e-2


@pytest.mark.parametrize("dataflow", ["staged", "fused"])
@pytest.mark.parametrize("k,ca,cb", [(3, 32, 16), (1, 64, 32), (3, 8, 24)])
def test_concat_input_vs_oracle(sc, rng, dataflow, k, ca, cb):
    """concat= (a U-Net skip read in place by the fused kernel) equals the
    layer on the materialised channel concatenation."""
    coords = random_coords(rng, (20, 20, 20), 0.15)
    n = coords.shape[0]
    fa = O.quantize(rng.standard_normal((n, ca)).astype(np.float32), "fp16")
    fb = O.quantize(rng.standard_normal((n, cb)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(k ** 3 * (ca + cb)), (k ** 3, ca + cb, 48)).astype(np.float32)
    _, want, _ = O.conv_forward(coords, np.concatenate([fa, fb], 1), (20, 20, 20), w, k, 1)
    t = sc.SparseTensor(coords, fa, 1, (20, 20, 20))
    skip = sc.SparseTensor(coords, fb, 1, (20, 20, 20))
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, k, 3), sc.LayerSpec(k, 1, ca + cb, 48),
                                 None, None, sc.ExecOptions(dataflow=dataflow), concat=skip)
    assert rel_l2(out.features_numpy(), want) <= 1e-2


def test_lazy_map_needs_no_compaction_for_fused(sc, rng):
    coords = random_coords(rng, (16, 16, 16), 0.1)
    t = sc.SparseTensor(coords, rng.standard_normal((coords.shape[0], 16)).astype(np.float16),
                        1, (16, 16, 16))
    w = sc.WeightTensor(rng.normal(0, 0.1, (27, 16, 16)).astype(np.float32), 3, 3)
    sc.sparse_conv_forward(t, w, sc.LayerSpec(3, 1, 16, 16), None, None,
                           sc.ExecOptions(dataflow="fused"))
    (_, kmap), = t.coordset.maps.values()
    assert kmap._csr is None  # the fused path consumed the hit matrix only
    assert kmap.total > 0 and kmap._csr is not None  # CSR on demand


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("k,s,c_in", [(3, 1, 16), (3, 1, 4), (2, 2, 32), (3, 2, 8)])
def test_sync_free_staged_is_bit_identical(sc, rng, prec, k, s, c_in):
    """The device-planned staged path (no host sync) reproduces the
    host-planned one bit for bit (same layout, same fold order)."""
    coords = random_coords(rng, (24, 22, 20), 0.08)
    f = O.quantize(rng.standard_normal((coords.shape[0], c_in)).astype(np.float32), prec)
    w = sc.WeightTensor(rng.normal(0, 0.1, (k ** 3, c_in, 24)).astype(np.float32), k, 3)
    outs = []
    for sync_free in (True, False):
        t = sc.SparseTensor(coords, f, 1, (24, 22, 20))
        cache = {}
        o = sc.sparse_conv_forward(t, w, sc.LayerSpec(k, s, c_in, 24, reuse_key="d"), None, cache,
                                   sc.ExecOptions(sync_free=sync_free, dataflow="staged"))
        outs.append(o.features_numpy())
        if s == 2:
            w2 = sc.WeightTensor(rng.normal(0, 0.1, (k ** 3, 24, 8)).astype(np.float32), k, 3) \
                if not outs[1:] else w2
            u = sc.inverse_conv_forward(o, w2, sc.LayerSpec(k, 1, 24, 8, transposed=True,
                                                            reuse_key="d"), cache, None,
                                        sc.ExecOptions(sync_free=sync_free, dataflow="staged"))
            outs.append(u.features_numpy())
    half = len(outs) // 2
    for a, b in zip(outs[:half], outs[half:]):
        np.testing.assert_array_equal(a, b)
    _, ref, _ = O.conv_forward(coords, f, (24, 22, 20), w.weights, k, s)
    assert rel_l2(outs[0], ref) <= TOL[prec]


def test_fp16_saturation_warns(sc):
    t = sc.SparseTensor(np.array([[0, 1, 1, 1]]), np.array([[1e6, -1e6, 1.0]], np.float32), 1,
                        (4, 4, 4))
    with pytest.warns(UserWarning, match="saturated"):
        q = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        f = q.features_numpy()
    assert f[0, 0] == 65504 and f[0, 1] == -65504 and f[0, 2] == 1.0


def test_strided_chain_equals_level_by_level(sc):
    """compute_output_coords_chain (device counts, one host read) gives the
    coordinates and maps of running each k2 s2 level on its own, bit-exact
    against the oracle (mapping.py:216-248)."""
    from paper_2204_10319_b200 import workloads
    coords, _, boundary = workloads.config1_cloud()
    t = sc.SparseTensor(coords, np.zeros((coords.shape[0], 8), np.float16), 1, boundary, 1)
    specs = [sc.LayerSpec(2, 2, 8, 8)] * 4
    levels = sc.prepare_strided_chain(t, specs, sc.ExecOptions())
    c, b = np.asarray(coords, np.int64), tuple(boundary)
    cs = t.coordset
    for lvl in levels:
        ob = O.downsample_boundary(b, 2)
        want = O.output_coords(c, 2, 2, ob, 1)
        np.testing.assert_array_equal(lvl.coords.cpu().numpy().astype(np.int64), want)
        kmap = cs.maps[(2, 2, 0)][1]
        pairs = O.kernel_map(c, b, want, 2, 2, 1)
        for got, ref in zip(kmap.pairs, pairs):
            np.testing.assert_array_equal(got, ref)
        c, b, cs = want, ob, lvl


def test_async_validation_raises_at_the_next_sync(sc):
    """validate="async" defers the reference's checks to the next host read."""
    bad = np.array([[0, 1, 1, 1], [0, 1, 1, 1]], dtype=np.int64)  # duplicate row
    t = sc.SparseTensor(bad, np.zeros((2, 4), np.float32), 1, (4, 4, 4), validate="async")
    with pytest.raises(ValueError, match="unique"):
        sc.flush_validation()
    oob = np.array([[0, 1, 1, 9]], dtype=np.int64)
    sc.SparseTensor(oob, np.zeros((1, 4), np.float32), 1, (4, 4, 4), validate="async")
    with pytest.raises(ValueError, match="outside boundary"):
        sc.flush_validation()
    ok = np.array([[0, 1, 1, 1], [0, 2, 1, 1]], dtype=np.int64)
    sc.SparseTensor(ok, np.zeros((2, 4), np.float32), 1, (4, 4, 4), validate="async")
    sc.flush_validation()


@pytest.mark.parametrize("c_in,c_out,split", [(64, 64, None), (96, 96, None), (24, 32, None),
                                              (256, 256, None), (48, 128, 16), (128, 96, 96),
                                              (64, 256, None), (256, 128, 64)])
def test_fused_epilogue_concat_shapes(sc, rng, c_in, c_out, split):
    """The implicit kernel against the oracle over K-chunk widths 16/32/64,
    C_out up to 256 (one CTA per SM), a BN + residual + ReLU epilogue and a
    concat split inside a K chunk."""
    coords = random_coords(rng, (20, 20, 20), 0.15)
    n = coords.shape[0]
    f = O.quantize(rng.standard_normal((n, c_in)).astype(np.float32), "fp16")
    r = O.quantize(rng.standard_normal((n, c_out)).astype(np.float32), "fp16")
    w = rng.normal(0, 1 / np.sqrt(27 * c_in), (27, c_in, c_out)).astype(np.float32)
    s = rng.uniform(0.8, 1.2, c_out).astype(np.float32)
    h = rng.normal(0, 0.05, c_out).astype(np.float32)
    _, base, _ = O.conv_forward(coords, f, (20, 20, 20), w, 3, 1)
    want = np.maximum(base.astype(np.float32) * s + h + r.astype(np.float32), 0)
    if split is None:
        t, skip = sc.SparseTensor(coords, f, 1, (20, 20, 20)), None
    else:
        t = sc.SparseTensor(coords, np.ascontiguousarray(f[:, :split]), 1, (20, 20, 20))
        skip = sc.SparseTensor(coords, np.ascontiguousarray(f[:, split:]), 1, (20, 20, 20))
    ep = {"scale": torch.from_numpy(s).cuda(), "shift": torch.from_numpy(h).cuda(),
          "residual": sc.SparseTensor(coords, r, 1, (20, 20, 20)), "relu": True}
    out = sc.sparse_conv_forward(t, sc.WeightTensor(w, 3, 3), sc.LayerSpec(3, 1, c_in, c_out),
                                 None, None, sc.ExecOptions(dataflow="fused"), epilogue=ep,
                                 concat=skip)
    assert rel_l2(out.features_numpy().astype(np.float32), want) <= 1e-2


@pytest.mark.parametrize("fused", [False, True])
def test_k1_strided_layer_and_inverse(sc, rng, fused):
    """K = 1, stride 2 (a volume-1 map that is NOT the identity, rows in
    shuffled order) and its transposed inverse, staged and fused, against
    the oracle (the fused path must read the hit matrix)."""
    coords = random_coords(rng, (16, 16, 16), 0.2)
    coords = coords[rng.permutation(coords.shape[0])]
    n = coords.shape[0]
    f = O.quantize(rng.standard_normal((n, 16)).astype(np.float32), "fp16")
    w1 = rng.normal(0, 0.25, (1, 16, 32)).astype(np.float32)
    w2 = rng.normal(0, 0.2, (1, 32, 16)).astype(np.float32)
    opts = sc.ExecOptions(dataflow="fused" if fused else "staged")
    t = sc.SparseTensor(coords, f, 1, (16, 16, 16))
    cache = {}
    d = sc.sparse_conv_forward(t, sc.WeightTensor(w1, 1, 3), sc.LayerSpec(1, 2, 16, 32,
                               reuse_key="d"), None, cache, opts)
    oc, of, _, pairs = O.conv_forward(coords, f, (16, 16, 16), w1, 1, 2, return_map=True)
    np.testing.assert_array_equal(d.coords_numpy(), oc)
    assert rel_l2(d.features_numpy().astype(np.float32), of) <= 1e-2
    u = sc.inverse_conv_forward(d, sc.WeightTensor(w2, 1, 3), sc.LayerSpec(
        1, 1, 32, 16, transposed=True, reuse_key="d"), cache, None, opts)
    uf = O.inverse_forward(d.features_numpy(), w2, pairs, n)
    assert rel_l2(u.features_numpy().astype(np.float32), uf) <= 1e-2
