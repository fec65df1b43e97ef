"""Strategy search (reference autotune.py): the
search loop, tie-breaking, analytic cost model and JSON v1 strategy files on
CPU (mirroring the reference's tests/test_autotune.py); the device cost
models on the GPU."""

import json

import numpy as np
import pytest

from paper_2204_10319_b200 import autotune as A
from paper_2204_10319_b200.autotune import (AnalyticCostModel, LayerRecord, LayerWorkload,
                                            SearchSpace, StrategyFile, load_strategy,
                                            save_strategy, tune_layer)


def make_workload(rng, volume=27, symmetric=True, c=8, big=2000, small=60):
    sizes = rng.integers(small // 2, small, size=volume).astype(np.int64)
    heavy = rng.choice(volume, size=max(volume // 4, 1), replace=False)
    sizes[heavy] = rng.integers(big // 2, big, size=heavy.shape[0])
    if symmetric:
        sizes = np.minimum(sizes, sizes[::-1])
        schedule = list(range((volume - 1) // 2))
    else:
        schedule = list(range(volume))
    return LayerWorkload(sizes, schedule, symmetric, c, c)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def test_search_space_rules():
    space = SearchSpace()
    assert space.configurations <= 1000
    assert 0.0 in space.eps_values and 1.0 in space.eps_values
    assert float("inf") in space.threshold_values
    with pytest.raises(ValueError):
        SearchSpace(tuple(np.linspace(0, 1, 101)), tuple(range(11)))
    with pytest.raises(ValueError):
        SearchSpace(eps_values=())
    s = SearchSpace((0.5, 0.0), (128.0, 0.0))
    assert s.eps_values == (0.0, 0.5) and s.threshold_values == (0.0, 128.0)


def test_tune_layer_argmin_and_ties(rng):
    wl = make_workload(rng)
    r = tune_layer([wl], SearchSpace((1.0,), (float("inf"),)), cost_fn=AnalyticCostModel([wl]))
    assert (r.eps, r.threshold, r.configurations) == (1.0, float("inf"), 1)
    one = LayerWorkload(np.array([5]), [0], False, 4, 4)
    r = tune_layer([one], SearchSpace((0.0, 0.5, 1.0), (0.0, 64.0, float("inf"))),
                   cost_fn=AnalyticCostModel([one]))
    assert (r.eps, r.threshold) == (0.0, 0.0)
    wls = [make_workload(rng) for _ in range(3)]
    space = SearchSpace((0.0, 0.3, 1.0), (0.0, 128.0, float("inf")))
    model = AnalyticCostModel(wls)
    r = tune_layer(wls, space, cost_fn=model)
    costs = {(e, t): model(e, t) for e in space.eps_values for t in space.threshold_values}
    assert r.cost == min(costs.values()) and costs[(r.eps, r.threshold)] == r.cost
    with pytest.raises(ValueError):
        tune_layer([], SearchSpace((0.0,), (0.0,)))


def test_analytic_model_matches_oracle_grouping(rng):
    """The analytic model's padded-FLOP arithmetic over the engine's
    grouping equals the same sum over the oracle's grouping (reference
    execution.py:221-328 restated in oracle.groups)."""
    from oracle import sparseconv_oracle as O
    wl = make_workload(rng)
    for eps, thr in [(0.0, 0.0), (0.3, 256.0), (1.0, float("inf"))]:
        want = 0.0
        for s, e, mode, _ in O.groups(wl.map_sizes, eps, thr, wl.schedule, wl.symmetric):
            members = list(wl.schedule[s:e])
            if wl.symmetric:
                members += [wl.map_sizes.shape[0] - 1 - n for n in members]
            n_max = max(int(wl.map_sizes[m]) for m in members)
            if mode == "batched":
                want += 5e4 + len(members) * n_max * wl.c_in * wl.c_out
            else:
                want += 5e4 * len(members) + sum(int(wl.map_sizes[m]) for m in members) \
                    * wl.c_in * wl.c_out
        assert AnalyticCostModel([wl])(eps, thr) == want


def test_strategy_files_round_trip_and_errors(tmp_path):
    s = StrategyFile((LayerRecord("stem", 0.1, 256.0, "grid"),
                      LayerRecord("enc1", 0.0, float("inf"), "hash", dataflow="fused")),
                     dataset="synthetic")
    p = tmp_path / "s.json"
    save_strategy(p, s)
    doc = json.loads(p.read_text())
    assert doc["version"] == 1 and doc["hardware"] == "B200"
    assert doc["layers"][1]["threshold"] == "inf" and "dataflow" not in doc["layers"][0]
    back = load_strategy(p, expected_layers=2)
    assert back.layers == s.layers and back.record_for("stem").eps == 0.1
    assert back.record_for("nope") is None
    with pytest.raises(ValueError, match="expected 3"):
        load_strategy(p, expected_layers=3)
    p.write_text(json.dumps({"version": 2, "layers": []}))
    with pytest.raises(ValueError, match="unsupported"):
        load_strategy(p)
    p.write_text("{not json")
    with pytest.raises(ValueError, match="malformed"):
        load_strategy(p)
    p.write_text(json.dumps({"version": 1, "layers": [{"eps": 0.1}]}))
    with pytest.raises(ValueError, match="malformed layer"):
        load_strategy(p)


def test_reference_strategy_file_loads(tmp_path):
    """A file in the reference's exact layout (no dataflow key) loads."""
    p = tmp_path / "ref.json"
    p.write_text(json.dumps({"version": 1, "engine": "0.1.0", "dataset": "kitti",
                             "hardware": "cpu", "layers": [
                                 {"id": "c1", "eps": 0.25, "threshold": 1024.0,
                                  "index_kind": "auto"}]}))
    s = load_strategy(p)
    assert s.layers[0] == LayerRecord("c1", 0.25, 1024.0, "auto", "auto")


@pytest.mark.gpu
def test_device_cost_models(rng):
    import paper_2204_10319_b200 as sc
    from conftest import random_coords
    wl = make_workload(rng, c=32)
    cost = A.ExecutionCostModel([wl])(0.2, 256.0)
    assert cost > 0.0
    r = tune_layer([wl], SearchSpace((0.0, 1.0), (0.0, float("inf"))))
    assert r.configurations == 4 and r.cost > 0
    coords = random_coords(rng, (16, 16, 16), 0.2)
    rec = dict(in_coords=coords, out_coords=coords, kernel_size=3, stride=1,
               boundary=(16, 16, 16), batch_size=1)
    d = A.tune_index_kind([rec])
    assert d.kind in ("grid", "hash") and d.grid_seconds > 0 and d.hash_seconds > 0
    d = A.tune_index_kind([rec], cell_cap=10)
    assert d.kind == "hash" and d.forced
    f = rng.standard_normal((coords.shape[0], 32)).astype(np.float16)
    t = sc.SparseTensor(coords, f, 1, (16, 16, 16))
    w = sc.WeightTensor(rng.normal(0, 0.05, (27, 32, 32)).astype(np.float32), 3, 3)
    dd = A.tune_dataflow(t, w, sc.LayerSpec(3, 1, 32, 32))
    assert dd.dataflow in ("staged", "fused") and dd.staged_seconds > 0


@pytest.mark.gpu
def test_tune_fused_layer_shapes_are_result_invariant():
    """The fused kernel's launch shapes (CTAs per SM, stage size) searched
    by tune_fused_layer give bit-identical outputs; the decision and the
    strategy file round trip carry the chosen shape."""
    import torch
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import autotune as A
    rng = np.random.default_rng(5)
    keys = np.sort(rng.choice(40 ** 3, 30_000, replace=False))
    c = np.stack([np.zeros_like(keys), keys // 1600, keys // 40 % 40, keys % 40], 1)
    f = rng.standard_normal((c.shape[0], 64)).astype(np.float16)
    t = sc.SparseTensor(c, f, 1, (40, 40, 40))
    w = sc.WeightTensor(rng.normal(0, 0.05, (27, 64, 64)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, 64, 64)
    outs = []
    for shape in A.KERNEL_SHAPES:
        o = sc.ExecOptions(dataflow="fused", layer_label="l", kernel_shapes={"l": shape})
        outs.append(sc.sparse_conv_forward(t, w, spec, None, None, o).features.clone())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    d = A.tune_fused_layer(t, w, spec, sc.ExecOptions(layer_label="l"), repeats=2)
    assert (d.ctas, d.stage_kb) in [s[:2] for s in d.tried]
    assert d.seconds <= d.default_seconds


def test_strategy_file_kernel_shape_round_trip(tmp_path):
    """B200 launch shapes ride in JSON v1 as an extra per-layer "kernel"
    object, which the reference's loader ignores (extra keys)."""
    sf = A.StrategyFile((LayerRecord("stem.0", 0.0, 0.0, "hash", "fused", 2, 42),
                         LayerRecord("head", 0.0, 0.0)))
    path = tmp_path / "s.json"
    A.save_strategy(path, sf)
    doc = json.loads(path.read_text())
    assert doc["layers"][0]["kernel"] == {"ctas": 2, "stage_kb": 42}
    assert "kernel" not in doc["layers"][1]
    back = A.load_strategy(path)
    assert (back.layers[0].ctas, back.layers[0].stage_kb) == (2, 42)
    assert (back.layers[1].ctas, back.layers[1].stage_kb) == (0, 0)
