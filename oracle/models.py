"""The bench's model graphs (MinkUNet, CenterPoint-style encoder) on the
CPU oracle: TEST INFRASTRUCTURE ONLY.  Imported by tests/ (whole-network
parity of the B200 engine) and nothing on the product path.  Epilogue
rounding follows the engine: conv output in f32, BN (+ residual) + ReLU in
f32, one cast to the storage dtype per layer.  Layer tables and parameters
come from the product package (they are data, shared by both sides)."""

from __future__ import annotations

import numpy as np

from paper_2204_10319_b200.centerpoint import layer_table as centerpoint_layers
from paper_2204_10319_b200.minkunet import layer_table as minkunet_layers

from . import sparseconv_oracle as O


def minkunet_oracle(params: dict, width: float, coords: np.ndarray, feats: np.ndarray,
                   boundary, batch_size: int = 1, in_channels: int = 4):
    """The same graph on the CPU oracle (tests and the CPU baseline only).
    Epilogue rounding follows the engine: conv output in f32, BN + ReLU in
    f32, one cast to the storage dtype."""
    storage = feats.dtype
    names = {l["name"] for l in minkunet_layers(width, in_channels)}
    cache = {}

    def conv(x, name, k, s, relu=True):
        c, f, b = x
        p = params[name]
        oc, of, ob, pairs = O.conv_forward(c, f, b, p["w"], k, s, batch_size, return_map=True)
        if pairs is not None and s == 2:
            cache[name] = (pairs, c, b)
        return oc, _epi(of, p, relu), ob

    def inverse(x, name, reuse):
        pairs, fc, fb = cache[reuse]
        of = O.inverse_forward(x[1], params[name]["w"], pairs, fc.shape[0])
        return fc, _epi(of, params[name], True), fb

    def _epi(f, p, relu, residual=None):
        f = f.astype(np.float32)
        if "scale" in p:
            f = f * p["scale"] + p["shift"]
        if residual is not None:
            f = f + residual.astype(np.float32)
        if relu:
            f = np.maximum(f, 0)
        return f.astype(storage)

    def res(x, prefix, has_proj):
        h = conv(x, prefix + ".c1", 3, 1)
        sc = conv(x, prefix + ".proj", 1, 1, relu=False) if has_proj else x
        c, f, b = h
        p = params[prefix + ".c2"]
        oc, of, ob = O.conv_forward(c, f, b, p["w"], 3, 1, batch_size)
        return oc, _epi(of, p, True, sc[1]), ob

    x = (np.asarray(coords, np.int64), feats, tuple(boundary))
    x = conv(x, "stem.0", 3, 1)
    x = conv(x, "stem.1", 3, 1)
    skips = [x]
    for i in range(1, 5):
        x = conv(x, f"down{i}", 2, 2)
        x = res(x, f"enc{i}.r0", f"enc{i}.r0.proj" in names)
        x = res(x, f"enc{i}.r1", f"enc{i}.r1.proj" in names)
        skips.append(x)
    for j in range(1, 5):
        x = inverse(x, f"up{j}", f"down{5 - j}")
        sk = skips[4 - j]
        x = (x[0], np.concatenate([x[1], sk[1]], axis=1), x[2])
        x = res(x, f"dec{j}.r0", True)
        x = res(x, f"dec{j}.r1", f"dec{j}.r1.proj" in names)
    return conv(x, "head", 1, 1, relu=False)


def centerpoint_oracle(params: dict, coords: np.ndarray, feats: np.ndarray, boundary,
                   batch_size: int = 1, in_channels: int = 5):
    """The same graph on the CPU oracle (tests only): conv output in f32, BN
    + ReLU in f32, one cast to the storage dtype per layer."""
    storage = feats.dtype
    c, f, b = np.asarray(coords, np.int64), feats, tuple(boundary)
    for l in centerpoint_layers(in_channels):
        p = params[l["name"]]
        c, of, b = O.conv_forward(c, f, b, p["w"], 3, l["s"], batch_size)
        f = np.maximum(of.astype(np.float32) * p["scale"] + p["shift"], 0).astype(storage)
    return c, f, b
