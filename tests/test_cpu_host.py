"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, the product refuses to run without a GPU (no CPU
fallback), and the host-side logic (grouping, specs, configs) matches the
oracle/reference semantics."""

import re
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import sparseconv_oracle as O

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "sparseconv_b200.h").read_text()
    return sorted(set(re.findall(r"\b(scb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2204_10319_b200 import _native
    lib = _native.load()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.exported_symbols())
    assert lib.scb_abi_version() == 2
    assert lib.scb_hash_slots(0) == 2 and lib.scb_hash_slots(5) == 16
    assert lib.scb_hash_slots(120_097) == 262_144
    assert isinstance(lib.scb_last_error(), bytes)


def test_library_is_sm100a_only():
    import subprocess
    so = ROOT / "paper_2204_10319_b200" / "libsparseconv_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnemonic in sass, mnemonic


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_2204_10319_b200 as sc
    with pytest.raises(RuntimeError, match="CUDA"):
        sc.SparseTensor(np.zeros((1, 4), np.int64), np.zeros((1, 2), np.float32), 1, (2, 2, 2))


def test_partition_and_grouping_match_oracle():
    from paper_2204_10319_b200 import execution as E
    assert E.partition_groups([100, 95, 90, 50, 48], 0.1, range(5)) == [(0, 3), (3, 5)]
    thresholds = [0.0, 64.0, 512.0, 4096.0, float("inf")]
    for case in range(2000):
        rng = np.random.default_rng(case)
        sizes = rng.integers(0, 10_000, size=rng.integers(1, 40))
        eps = float(rng.uniform(0.0, 1.0))
        thr = thresholds[case % len(thresholds)]
        sched = list(range(sizes.shape[0]))
        assert E.partition_groups(sizes, eps, sched) == O.partition(sizes, eps, sched)
        g = E.build_grouping(sizes, eps, thr)
        g.validate(sizes)
        assert [(x.start, x.end, x.mode, x.padded_rows) for x in g.groups] == \
            O.groups(sizes, eps, thr, sched, False)
    with pytest.raises(ValueError):
        E.partition_groups([1], 1.5, [0])


def test_grouping_special_cases():
    from paper_2204_10319_b200 import execution as E
    from paper_2204_10319_b200.mapping import enumerate_offsets
    sizes = np.zeros(27, dtype=np.int64)
    for i in range(13):
        sizes[i] = sizes[26 - i] = 400 - 10 * i
    schedule, symmetric = E.schedule_for(enumerate_offsets(3, 3), 1)
    assert schedule == list(range(13)) and symmetric
    dense = E.build_grouping(sizes, 1.0, float("inf"), schedule, symmetric)
    assert dense.groups == (E.MatmulGroup(0, 13, "batched",
                                          sum(2 * (400 - int(sizes[i])) for i in range(13))),)
    sep = E.build_grouping(sizes, 0.0, 0.0, schedule, symmetric)
    assert sep.groups == tuple(E.MatmulGroup(i, i + 1, "sequential", 0) for i in range(13))
    paired = E.build_grouping(sizes, 0.0, float("inf"), schedule, symmetric)
    assert all(len(paired.members(g)) == 2 for g in paired.groups)
    assert E.schedule_for(enumerate_offsets(3, 2), 2) == (list(range(8)), False)


def test_offsets_match_oracle():
    from paper_2204_10319_b200.mapping import enumerate_offsets
    for dim in (1, 2, 3, 4):
        for k in (1, 2, 3, 4, 5):
            off = enumerate_offsets(dim, k)
            np.testing.assert_array_equal(off.offsets, O.offsets(dim, k))
            assert off.center == O.center_of(k, dim)
    with pytest.raises(ValueError):
        enumerate_offsets(5, 3)
    with pytest.raises(ValueError):
        enumerate_offsets(3, 0)


def test_specs_and_strategies():
    from paper_2204_10319_b200 import execution as E
    with pytest.raises(ValueError, match="unsupported stride"):
        E.LayerSpec(3, 3, 4, 4)
    with pytest.raises(ValueError, match="reuse key"):
        E.LayerSpec(2, 1, 4, 4, transposed=True)
    with pytest.raises(ValueError):
        E.LayerStrategy(1.5, 0)
    with pytest.raises(ValueError):
        E.LayerStrategy(0.5, -1)
    spec = E.LayerSpec(3, 1, 4, 4, strategy=E.LayerStrategy(0.2, 10))
    assert E.resolve_strategy(spec, None) == E.LayerStrategy(0.2, 10)
    assert E.resolve_strategy(spec, E.LayerStrategy.dense_group()).eps == 1.0
    assert E.resolve_strategy(E.LayerSpec(3, 1, 4, 4), None) == E.LayerStrategy.separate()
    with pytest.warns(UserWarning):
        o = E.ExecOptions(fused=False)
    assert o.order == "weight"
    with pytest.raises(ValueError):
        E.ExecOptions(order="zigzag")


def test_network_config_parsing_and_params():
    import json
    from paper_2204_10319_b200 import network as N
    cfg = N.load_builtin_config("minkunet_toy")
    assert cfg.conv_layer_ids == ["stem", "down1", "enc1", "down2", "up1", "up2", "head"]
    net = N.Network.build(cfg)
    doc = json.loads((ROOT / "paper_2204_10319_b200" / "configs" / "minkunet_toy.json").read_text())
    weights, pw = O.build_params(doc)
    for lid, w in net.weights.items():
        np.testing.assert_array_equal(w.weights, weights[lid])
    for lid, p in net.pointwise.items():
        for k, v in p.items():
            np.testing.assert_array_equal(v, pw[lid][k])
    bad = dict(doc, layers=doc["layers"] + [{"kind": "inverse_conv", "id": "x", "reuse": "stem",
                                             "kernel_size": 3, "out_channels": 4}])
    with pytest.raises(N.ConfigError, match="reuse"):
        N.NetworkConfig.from_dict(bad)
    with pytest.raises(N.ConfigError, match="unknown kind"):
        N.NetworkConfig.from_dict(dict(doc, layers=[{"kind": "pool"}]))
    with pytest.raises(N.ConfigError, match="duplicate"):
        N.NetworkConfig.from_dict(dict(doc, layers=[doc["layers"][0], doc["layers"][0]]))


def test_workload_generators_are_deterministic():
    from paper_2204_10319_b200 import workloads as W
    a = W.raycast_points(3, azimuths=360)
    b = W.raycast_points(3, azimuths=360)
    np.testing.assert_array_equal(a, b)
    c, f, bnd = W.voxelize(np.concatenate([a[:, :3], a], 1), 0.2)
    keys = O.flatten(c, bnd)
    assert (np.diff(keys) > 0).all()  # unique and sorted by key
    assert f.shape == (c.shape[0], 4)


def test_dilation_spec_validation():
    """Dilation (B200 extension for north_star's SparseConv3d) is a stride-1
    option; the map cache keys keep dilated and plain maps apart."""
    import paper_2204_10319_b200 as sc
    sc.LayerSpec(3, 1, 8, 8, dilation=2)
    with pytest.raises(ValueError, match="dilation"):
        sc.LayerSpec(3, 1, 8, 8, dilation=0)
    with pytest.raises(ValueError, match="stride-1"):
        sc.LayerSpec(2, 2, 8, 8, dilation=2)


def test_cpu_arm_samples_and_torch_free_tables():
    """The reference CPU arm's bounded samples: equal-count azimuth sectors
    that partition each scan (fractions sum to one scan), and the model
    tables the workers load without importing torch or the engine."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import bench
    rng = np.random.default_rng(0)
    c = np.concatenate([np.zeros((1000, 1), np.int64), rng.integers(0, 500, (1000, 3))], 1)
    f = rng.standard_normal((1000, 4)).astype(np.float32)
    secs = bench.scan_sectors((c, f, (500, 500, 500)), 16)
    assert len(secs) == 16
    assert abs(sum(s[3] for s in secs) - 1.0) < 1e-12
    rows = np.concatenate([s[0] for s in secs])
    assert rows.shape == c.shape
    assert np.array_equal(np.unique(rows, axis=0), np.unique(c, axis=0))
    assert max(s[0].shape[0] for s in secs) - min(s[0].shape[0] for s in secs) <= 1
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from oracle.reference_runner import model_tables\n"
            "m = model_tables('minkunet'); p = m.build_params(0.5, 4, 0)\n"
            "assert len(m.layer_table(0.5)) == 50 and 'torch' not in sys.modules\n"
            "print('ok')" % str(root))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr


def test_dense_forms_validate_arguments_before_touching_the_device():
    """scb_conv_pointwise / scb_conv_transposed_scatter check their arguments
    host-side (EINVAL + a message naming the entry point) before any CUDA
    call, so the error convention holds without a GPU."""
    import ctypes
    from paper_2204_10319_b200 import _native
    lib = _native.load()
    fake = ctypes.c_void_p(0x1000)
    pw = lib.scb_conv_pointwise
    pw.restype = ctypes.c_int32
    i64, i32, P = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    # c_in not a multiple of 8
    rc = pw(fake, i64(16), i32(12), None, i64(0), i64(10), i32(12), fake, i32(16), fake,
            i64(16), None, None, None, i32(0), None)
    assert rc == 1 and b"scb_conv_pointwise" in lib.scb_last_error() and b"c_in" in lib.scb_last_error()
    # scale without shift
    rc = pw(fake, i64(16), i32(16), None, i64(0), i64(10), i32(16), fake, i32(16), fake,
            i64(16), fake, None, None, i32(0), None)
    assert rc == 1 and b"scale and shift" in lib.scb_last_error()
    # output rows narrower than C_out rounded up to 8 (the 19-class head needs 24)
    rc = pw(fake, i64(96), i32(96), None, i64(0), i64(10), i32(96), fake, i32(19), fake,
            i64(19), None, None, None, i32(0), None)
    assert rc == 1 and b"ldo" in lib.scb_last_error()
    ts = lib.scb_conv_transposed_scatter
    ts.restype = ctypes.c_int32
    rc = ts(fake, i64(16), i64(10), i32(16), None, i32(8), fake, i32(16), fake, i64(16),
            i64(10), None, None, None, i32(0), None)
    assert rc == 1 and b"child" in lib.scb_last_error()
    rc = ts(fake, i64(16), i64(10), i32(16), fake, i32(33), fake, i32(16), fake, i64(16),
            i64(10), None, None, None, i32(0), None)
    assert rc == 1 and b"volume" in lib.scb_last_error()
