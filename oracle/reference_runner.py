"""The bench's model graphs run through the UNMODIFIED reference package
(``sparseconv``, arXiv 2204.10319's CPU engine) via its own public API:
``SparseTensor``, ``WeightTensor``, ``LayerSpec``, ``sparse_conv_forward``,
``inverse_conv_forward``, ``pointwise_apply`` (reference
``execution.py:450-576``), with numpy glue for what the reference has no
layer kind for (residual add, skip concatenation).

BENCH / TEST INFRASTRUCTURE ONLY: bench.py's CPU arm (``--impl reference``
and the ``cpu_baseline`` leg) and whole-network parity tests.  Nothing on
the product path imports it.

Where the reference comes from: ``baseline/_ref`` (``pip install --target
baseline/_ref`` of the unmodified reference; it travels to
the GPU box) or, in the build container, ``/root/reference/pkg/src``.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def import_reference():
    """The reference package, or ImportError naming where it was looked for."""
    for p in _CANDIDATES:
        if (p / "sparseconv" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return importlib.import_module("sparseconv")
    raise ImportError("reference package `sparseconv` not found in "
                      + ", ".join(str(p) for p in _CANDIDATES))


def model_tables(name: str):
    """The engine's model module (layer table, parameters: numpy only)
    loaded standalone, so CPU worker processes never import torch or the
    engine package."""
    import importlib.util
    from pathlib import Path
    key = "_scb_tables_" + name
    mod = sys.modules.get(key)
    if mod is None:
        path = Path(__file__).resolve().parent.parent / "paper_2204_10319_b200" / f"{name}.py"
        spec = importlib.util.spec_from_file_location(key, path)
        mod = importlib.util.module_from_spec(spec)
        sys.modules[key] = mod
        spec.loader.exec_module(mod)
    return mod


def minkunet_reference(S, params: dict, width: float, coords, feats, boundary,
                       batch_size: int = 1, in_channels: int = 4):
    """MinkUNet (paper_2204_10319_b200.minkunet.layer_table) on reference
    ``S``: FP16 storage, hash index; returns (coords, logits, boundary)."""
    layer_table = model_tables("minkunet").layer_table
    names = {l["name"] for l in layer_table(width, in_channels)}
    t = S.quantize_features(S.SparseTensor(np.asarray(coords, np.int64), feats, 1,
                                           tuple(boundary), batch_size),
                            S.PrecisionMode.FP16_STORAGE)
    storage = t.features.dtype
    opts = S.ExecOptions(index_kind="hash")
    cache: dict = {}

    def conv(x, name, k, s, relu=True, residual=None, inverse_of=None):
        p = params[name]
        w = S.WeightTensor(p["w"], k, 3)
        ci, co = p["w"].shape[1], p["w"].shape[2]
        opts.layer_label = name
        if inverse_of is not None:
            y = S.inverse_conv_forward(x, w, S.LayerSpec(k, 1, ci, co, transposed=True,
                                                         reuse_key=inverse_of), cache,
                                       options=opts)
        else:
            y = S.sparse_conv_forward(x, w, S.LayerSpec(k, s, ci, co,
                                                        reuse_key=name if s > 1 else None),
                                      None, cache, opts)
        if "scale" in p:
            y = S.pointwise_apply(y, "bn_fold", scale=p["scale"], shift=p["shift"])
        if residual is not None:
            y = y.replace_features((y.features.astype(np.float32)
                                    + residual.features.astype(np.float32)).astype(storage))
        if relu:
            y = S.pointwise_apply(y, "relu")
        return y

    def res(x, prefix, has_proj):
        h = conv(x, prefix + ".c1", 3, 1)
        sc = conv(x, prefix + ".proj", 1, 1, relu=False) if has_proj else x
        return conv(h, prefix + ".c2", 3, 1, residual=sc)

    x = conv(t, "stem.0", 3, 1)
    x = conv(x, "stem.1", 3, 1)
    skips = [x]
    for i in range(1, 5):
        x = conv(x, f"down{i}", 2, 2)
        x = res(x, f"enc{i}.r0", f"enc{i}.r0.proj" in names)
        x = res(x, f"enc{i}.r1", f"enc{i}.r1.proj" in names)
        skips.append(x)
    for j in range(1, 5):
        x = conv(x, f"up{j}", 2, 1, inverse_of=f"down{5 - j}")
        x = x.replace_features(np.concatenate([x.features, skips[4 - j].features], axis=1))
        x = res(x, f"dec{j}.r0", True)
        x = res(x, f"dec{j}.r1", f"dec{j}.r1.proj" in names)
    out = conv(x, "head", 1, 1, relu=False)
    return out.coords, out.features, out.boundary


def centerpoint_reference(S, params: dict, coords, feats, boundary, batch_size: int = 1,
                          in_channels: int = 5):
    """The CenterPoint-style encoder (paper_2204_10319_b200.centerpoint) on
    reference ``S``: FP16 storage, hash index."""
    layer_table = model_tables("centerpoint").layer_table
    x = S.quantize_features(S.SparseTensor(np.asarray(coords, np.int64), feats, 1,
                                           tuple(boundary), batch_size),
                            S.PrecisionMode.FP16_STORAGE)
    opts = S.ExecOptions(index_kind="hash")
    for l in layer_table(in_channels):
        p = params[l["name"]]
        opts.layer_label = l["name"]
        x = S.sparse_conv_forward(x, S.WeightTensor(p["w"], 3, 3),
                                  S.LayerSpec(3, l["s"], l["ci"], l["co"]), None, None, opts)
        x = S.pointwise_apply(x, "bn_fold", scale=p["scale"], shift=p["shift"])
        x = S.pointwise_apply(x, "relu")
    return x.coords, x.features, x.boundary
