"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``sparseconv`` straight from the read-only reference tree
(numba's cache is redirected to /tmp) and writes small ``.npz`` fixtures next
to this file.  Nothing under tests/ or the product reads /root/reference at
run time; the fixtures are what travel to the GPU box.

Large arrays (the ~47k-voxel config-1 map) are stored as SHA-256 digests of
the canonical int64 arrays plus the per-offset sizes, so the fixture stays
small while still pinning every entry bit-exactly.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, str(REF_SRC))

import sparseconv as sc  # noqa: E402  (the unmodified reference)
from sparseconv import mapping as scm  # noqa: E402
from sparseconv import execution as sce  # noqa: E402
from sparseconv import synth as scs  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def random_coords(rng, boundary, occupancy, batch_size=1):
    """Same recipe as the reference's tests/conftest.py:7-19."""
    cells = batch_size * int(np.prod(boundary))
    n = max(1, int(cells * occupancy))
    keys = np.sort(rng.choice(cells, size=n, replace=False))
    coords = np.empty((n, 1 + len(boundary)), dtype=np.int64)
    rem = keys
    for d in range(len(boundary) - 1, -1, -1):
        coords[:, d + 1] = rem % boundary[d]
        rem = rem // boundary[d]
    coords[:, 0] = rem
    return coords


def pack_pairs(pairs):
    sizes = np.array([p.shape[0] for p in pairs], dtype=np.int64)
    ptr = np.zeros(len(pairs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=ptr[1:])
    flat = np.concatenate([p for p in pairs] + [np.empty((0, 2), np.int64)], 0)
    return ptr, flat.astype(np.int64)


def gen_maps():
    """Kernel maps + output coords over seeded clouds (K x s x batch x kind)."""
    cases = {}
    idx = 0
    for k in (1, 2, 3):
        for s in (1, 2):
            for seed in range(4):
                for batch in (1, 2):
                    rng = np.random.default_rng(1000 + 97 * idx)
                    idx += 1
                    edge = 9 + seed
                    boundary = (edge, edge + 1, edge + 2)
                    coords = random_coords(rng, boundary, 0.12, batch)
                    # shuffle input rows: the map must not assume sorted input
                    if seed % 2 == 1:
                        coords = coords[rng.permutation(coords.shape[0])]
                    off = sc.enumerate_offsets(3, k)
                    bout = boundary if s == 1 else scm.downsample_boundary(boundary, s)
                    out = sc.compute_output_coords(coords, off, s, bout, batch)
                    index = sc.build_index(coords, "hash", boundary, batch)
                    kmap = sc.map_search(index, out, off, s)
                    ptr, flat = pack_pairs(kmap.pairs)
                    sw = kmap.swap_roles()
                    sptr, sflat = pack_pairs(sw.pairs)
                    key = f"k{k}_s{s}_seed{seed}_b{batch}"
                    cases[key + "_in"] = coords
                    cases[key + "_boundary"] = np.array(boundary + (batch,), np.int64)
                    cases[key + "_out"] = out
                    cases[key + "_ptr"] = ptr
                    cases[key + "_pairs"] = flat
                    cases[key + "_swptr"] = sptr
                    cases[key + "_swpairs"] = sflat
    # the 2-D worked example (tests/test_acceptance.py:67-80)
    in2 = np.array([[0, 3, 5]], np.int64)
    out2 = sc.compute_output_coords(in2, sc.enumerate_offsets(2, 2), 2, (2, 3))
    cases["worked2d_out"] = out2
    # dense 8^3 block (tests/test_mapping.py:163-172)
    block = np.array([[0, x, y, z] for x in range(8) for y in range(8) for z in range(8)],
                     np.int64)
    kmap = sc.map_search(sc.build_index(block, "grid", (8, 8, 8)), block,
                         sc.enumerate_offsets(3, 3), 1)
    cases["block8_sizes"] = kmap.sizes
    # 2-D and 4-D maps (the reference is rank-generic, core.py:106-107)
    for dim, bnd in ((2, (20, 23)), (4, (5, 6, 5, 4))):
        rng = np.random.default_rng(77 + dim)
        coords = random_coords(rng, bnd, 0.2)
        for k, s in ((3, 1), (3, 2), (2, 2)):
            off = sc.enumerate_offsets(dim, k)
            bout = bnd if s == 1 else scm.downsample_boundary(bnd, s)
            out = sc.compute_output_coords(coords, off, s, bout)
            kmap = sc.map_search(sc.build_index(coords, "hash", bnd), out, off, s)
            ptr, flat = pack_pairs(kmap.pairs)
            key = f"d{dim}_k{k}_s{s}"
            cases[key + "_in"] = coords
            cases[key + "_boundary"] = np.array(bnd + (1,), np.int64)
            cases[key + "_out"] = out
            cases[key + "_ptr"] = ptr
            cases[key + "_pairs"] = flat
    np.savez_compressed(OUT / "maps.npz", **cases)
    print("maps.npz", len(cases), "arrays")


def gen_layers():
    """Layer forwards (conv + inverse) at FP32 and FP16 storage."""
    cases = {}
    idx = 0
    for k, s in ((1, 1), (1, 2), (2, 1), (2, 2), (3, 1), (3, 2)):
        for c_in, c_out in ((4, 16), (16, 16), (32, 24), (5, 19)):
            for prec in ("fp32", "fp16"):
                rng = np.random.default_rng(5000 + idx)
                idx += 1
                boundary = (14, 13, 12)
                coords = random_coords(rng, boundary, 0.1)
                feats = rng.standard_normal((coords.shape[0], c_in)).astype(np.float32)
                vol = k ** 3
                w = rng.normal(0, 1.0 / np.sqrt(vol * c_in), (vol, c_in, c_out)).astype(np.float32)
                t = sc.SparseTensor(coords, feats, 1, boundary, 1)
                t = sc.quantize_features(t, sc.PrecisionMode(prec))
                spec = sc.LayerSpec(k, s, c_in, c_out, reuse_key="L")
                cache = {}
                out = sc.sparse_conv_forward(t, sc.WeightTensor(w, k, 3), spec, None, cache)
                key = f"k{k}_s{s}_c{c_in}x{c_out}_{prec}"
                cases[key + "_in"] = coords
                cases[key + "_feat"] = np.asarray(t.features)
                cases[key + "_w"] = w
                cases[key + "_outc"] = out.coords
                cases[key + "_outf"] = out.features
                if s == 2:
                    w2 = rng.normal(0, 1.0 / np.sqrt(vol * c_out), (vol, c_out, c_in)).astype(np.float32)
                    inv = sc.inverse_conv_forward(
                        out, sc.WeightTensor(w2, k, 3),
                        sc.LayerSpec(k, 1, c_out, c_in, transposed=True, reuse_key="L"), cache)
                    cases[key + "_w2"] = w2
                    cases[key + "_invf"] = inv.features
    np.savez_compressed(OUT / "layers.npz", **cases)
    print("layers.npz", len(cases), "arrays")


def gen_plans():
    """Gather/scatter plan arrays on a small map, with and without skip_center."""
    rng = np.random.default_rng(99)
    boundary = (9, 9, 9)
    coords = random_coords(rng, boundary, 0.2)
    off = sc.enumerate_offsets(3, 3)
    kmap = sc.map_search(sc.build_index(coords, "grid", boundary), coords, off, 1)
    cases = {"in": coords}
    for skip in (False, True):
        p = sc.build_gather_scatter_plan(kmap, skip_center=skip)
        for name in ("buffer_offsets", "row_input", "row_output", "in_indptr", "in_rows",
                     "out_indptr", "out_rows"):
            cases[f"skip{int(skip)}_{name}"] = getattr(p, name)
        feats = rng.standard_normal((coords.shape[0], 8)).astype(np.float32)
        buf = sc.gather(feats, p, "input_stationary")
        cases[f"skip{int(skip)}_feat"] = feats
        cases[f"skip{int(skip)}_buffer"] = buf
        part = rng.standard_normal((p.total, 8)).astype(np.float32)
        cases[f"skip{int(skip)}_partial"] = part
        cases[f"skip{int(skip)}_scatter"] = sc.scatter_accumulate(
            part, p, kmap.n_out, "output_stationary")
    np.savez_compressed(OUT / "plans.npz", **cases)
    print("plans.npz", len(cases), "arrays")


def gen_network():
    """The reference's bundled toy MinkUNet (configs/minkunet_toy.json)."""
    import json
    doc = json.loads((REF_SRC / "sparseconv/configs/minkunet_toy.json").read_text())
    cases = {"doc": np.array(json.dumps(doc))}
    rng = np.random.default_rng(4242)
    boundary = (16, 16, 16)
    coords = random_coords(rng, boundary, 0.15)
    feats = rng.standard_normal((coords.shape[0], 4)).astype(np.float32)
    cases["in"] = coords
    cases["feat"] = feats
    for prec in ("fp32", "fp16"):
        d = dict(doc, precision=prec)
        net = sc.Network.build(sc.NetworkConfig.from_dict(d))
        out = net.forward(sc.SparseTensor(coords, feats, 1, boundary, 1))
        cases[f"{prec}_outc"] = out.coords
        cases[f"{prec}_outf"] = out.features
        for lid, w in net.weights.items():
            cases[f"{prec}_w_{lid}"] = w.weights
    np.savez_compressed(OUT / "network.npz", **cases)
    print("network.npz", len(cases), "arrays")


def gen_config1():
    """Config 1 cloud: synth uniform 60k @ extent 50 -> voxel 1.0."""
    pts = scs.synth_points("uniform", 60_000, 50.0, seed=0, channels=4)
    t = sc.voxelize(pts, 1.0)
    off = sc.enumerate_offsets(3, 3)
    kmap = sc.map_search(sc.build_index(t.coords, "hash", t.boundary), t.coords, off, 1)
    ptr, flat = pack_pairs(kmap.pairs)
    bout = scm.downsample_boundary(t.boundary, 2)
    off2 = sc.enumerate_offsets(3, 2)
    out2 = sc.compute_output_coords(t.coords, off2, 2, bout)
    kmap2 = sc.map_search(sc.build_index(t.coords, "hash", t.boundary), out2, off2, 2)
    ptr2, flat2 = pack_pairs(kmap2.pairs)
    cases = {
        "n": np.array(t.num_points),
        "boundary": np.array(t.boundary),
        "coords_digest": np.array(digest(t.coords)),
        "feat_digest": np.array(hashlib.sha256(np.asarray(t.features).tobytes()).hexdigest()),
        "k3s1_sizes": kmap.sizes,
        "k3s1_digest": np.array(digest(ptr, flat)),
        "k2s2_nout": np.array(out2.shape[0]),
        "k2s2_out_digest": np.array(digest(out2)),
        "k2s2_sizes": kmap2.sizes,
        "k2s2_digest": np.array(digest(ptr2, flat2)),
    }
    np.savez_compressed(OUT / "config1.npz", **cases)
    print("config1.npz n =", t.num_points, "|M| =", int(kmap.sizes.sum()))


def gen_voxelize():
    """sparseconv.core.voxelize (core.py:174-216) on seeded clouds: mean and
    first reduction, 2-D and 3-D, clouds with many duplicate cells."""
    cases = {}
    rng = np.random.default_rng(777)
    for i, (n, dims, ch, vs, reduce) in enumerate([
            (4000, 3, 4, 4.0, "mean"), (4000, 3, 4, 4.0, "first"), (3000, 3, 2, 1.5, "mean"),
            (2000, 2, 3, 1.0, "mean"), (1, 3, 1, 1.0, "mean"), (3000, 3, 5, 8.0, "first"),
            (3000, 3, 0, 2.0, "mean")]):
        xyz = rng.uniform(-20, 20, size=(n, dims))
        pts = np.concatenate([xyz, rng.standard_normal((n, ch))], axis=1)
        t = sc.voxelize(pts, vs, reduce=reduce, spatial_dims=dims)
        cases[f"v{i}_points"] = pts
        cases[f"v{i}_meta"] = np.array([dims, 1 if reduce == "first" else 0], dtype=np.int64)
        cases[f"v{i}_vs"] = np.array([vs], dtype=np.float64)
        cases[f"v{i}_coords"] = np.asarray(t.coords, dtype=np.int64)
        cases[f"v{i}_feats"] = np.asarray(t.features, dtype=np.float32)
        cases[f"v{i}_boundary"] = np.asarray(t.boundary, dtype=np.int64)
    np.savez_compressed(OUT / "voxelize.npz", **cases)


def minkunet_chain_doc(width: float = 1.0) -> dict:
    """MinkUNet's layer sequence in the reference's own JSON schema
    (reference network.py:1-25): the 50-conv encoder/decoder with every
    residual block written as its two k3 convs and the skip concatenations
    dropped (the schema has neither add nor concat layers, SURVEY.md §0
    fact 8); BN folded (bn_fold) + ReLU after every conv but the head."""
    cs = [int(c * width) for c in (32, 32, 64, 128, 256, 256, 128, 96, 96)]
    L = []

    def conv(i, k, s, co, bn=True):
        L.append({"id": i, "kind": "conv", "kernel_size": k, "stride": s, "out_channels": co,
                  "index_kind": "hash"})
        if bn:
            L.extend([{"kind": "bn_fold", "id": i + ".bn"}, {"kind": "relu"}])

    conv("stem.0", 3, 1, cs[0])
    conv("stem.1", 3, 1, cs[0])
    for i in range(1, 5):
        conv(f"down{i}", 2, 2, cs[i - 1])
        for r in ("r0", "r1"):
            conv(f"enc{i}.{r}.c1", 3, 1, cs[i])
            conv(f"enc{i}.{r}.c2", 3, 1, cs[i])
    for j in range(1, 5):
        L.append({"id": f"up{j}", "kind": "inverse_conv", "kernel_size": 2,
                  "reuse": f"down{5 - j}", "out_channels": cs[4 + j]})
        L.extend([{"kind": "bn_fold", "id": f"up{j}.bn"}, {"kind": "relu"}])
        for r in ("r0", "r1"):
            conv(f"dec{j}.{r}.c1", 3, 1, cs[4 + j])
            conv(f"dec{j}.{r}.c2", 3, 1, cs[4 + j])
    conv("head", 1, 1, 19, bn=False)
    return {"name": "minkunet_chain", "in_channels": 4, "precision": "fp16", "param_seed": 7,
            "layers": L}


def gen_minkunet_chain():
    """The MinkUNet-shaped chain (minkunet_chain_doc) through the unmodified
    reference's Network.forward on a cropped raycast LiDAR scan (the bench's
    generator, paper_2204_10319_b200.workloads), FP32 and FP16 storage:
    output coordinates (digest) and features per precision."""
    import json
    sys.path.insert(0, str(OUT.parents[1]))
    from paper_2204_10319_b200.workloads import raycast_points
    pts = raycast_points(3)
    keep = pts[:, 0] ** 2 + pts[:, 1] ** 2 < 5.0 ** 2       # disc around the sensor
    pts = pts[keep]
    pts = np.concatenate([pts[:, :3], pts], axis=1)
    vox = sc.voxelize(pts, 0.05)
    doc = minkunet_chain_doc(1.0)
    cases = {"doc": np.array(json.dumps(doc)), "in": vox.coords.astype(np.int32),
             "feat": vox.features.astype(np.float32),
             "boundary": np.array(vox.boundary, np.int64)}
    for prec in ("fp32", "fp16"):
        net = sc.Network.build(sc.NetworkConfig.from_dict(dict(doc, precision=prec)))
        out = net.forward(vox)
        cases[f"{prec}_outc_digest"] = np.array(digest(out.coords))
        cases[f"{prec}_outc_n"] = np.array(out.coords.shape[0])
        cases[f"{prec}_outf"] = out.features
    np.savez_compressed(OUT / "minkunet_chain.npz", **cases)
    print("minkunet_chain.npz:", vox.num_points, "voxels,",
          sum(1 for l in doc["layers"] if "conv" in l["kind"]), "conv layers")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_minkunet_chain()
    gen_voxelize()
    gen_maps()
    gen_layers()
    gen_plans()
    gen_network()
    gen_config1()
