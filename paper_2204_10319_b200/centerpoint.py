"""CenterPoint-style sparse 3-D encoder (BASELINE.json config 4, SURVEY.md
§8(d)) on the drop-in operator API.

Layer table, within the reference's layer semantics (cubic kernels, no spconv
padding; `src/core.py:150-161`):

    stem      conv3 in->16 +BN+ReLU, 4x conv3 16->16 +BN+ReLU
    stage i   conv3/s2 c->c_i +BN+ReLU, 4x conv3 c_i->c_i +BN+ReLU   c_i = 32, 64, 128
    out       conv3/s2 128->128 +BN+ReLU

21 convolution layers (17 SubM k3, 4 k3 s2).  Strided k3 layers propose up
to 8 candidates per input, so their output coordinates are computed level
by level (one host read each), all before the first convolution is queued.

``EngineCenterPoint`` runs on the B200 engine; ``forward_oracle`` runs the
same graph on the CPU oracle (tests only).
"""

from __future__ import annotations

import numpy as np

STAGES = (32, 64, 128)


def layer_table(in_channels: int = 5) -> list[dict]:
    L = []

    def conv(name, s, ci, co):
        L.append(dict(name=name, k=3, s=s, ci=ci, co=co))

    conv("stem.0", 1, in_channels, 16)
    for j in range(4):
        conv(f"stem.{j + 1}", 1, 16, 16)
    c = 16
    for i, ci in enumerate(STAGES, 1):
        conv(f"down{i}", 2, c, ci)
        for j in range(4):
            conv(f"stage{i}.{j}", 1, ci, ci)
        c = ci
    conv("out", 2, c, 128)
    return L


def build_params(in_channels: int = 5, seed: int = 0) -> dict:
    """Random-init weights N(0, 1/sqrt(27 C_in)) (reference network.py:183-193)
    and folded BN (scale U(0.8, 1.2), shift N(0, 0.05))."""
    rng = np.random.default_rng(seed)
    params = {}
    for l in layer_table(in_channels):
        w = rng.normal(0.0, 1.0 / np.sqrt(27 * l["ci"]), size=(27, l["ci"], l["co"]))
        params[l["name"]] = {
            "w": w.astype(np.float32),
            "scale": rng.uniform(0.8, 1.2, size=l["co"]).astype(np.float32),
            "shift": rng.normal(0.0, 0.05, size=l["co"]).astype(np.float32)}
    return params


class EngineCenterPoint:
    """The encoder on the B200 engine.  Parameters are uploaded once."""

    def __init__(self, in_channels: int = 5, seed: int = 0):
        import torch
        from .core import WeightTensor
        self.table = layer_table(in_channels)
        self.params = build_params(in_channels, seed)
        self.w, self.bn = {}, {}
        for l in self.table:
            p = self.params[l["name"]]
            self.w[l["name"]] = WeightTensor(p["w"], 3, 3)
            self.bn[l["name"]] = (torch.from_numpy(p["scale"]).cuda(),
                                  torch.from_numpy(p["shift"]).cuda())
            self.w[l["name"]].packed_f16()
        # SCB_MAP_STREAM=1: maps on a high-priority side stream (overlaps the
        # previous batch; measured noisier: the persistent conv kernels leave
        # no room for the short mapping kernels between their boundaries)
        self.mapping_stream = (torch.cuda.Stream(priority=-1)
                               if __import__("os").environ.get("SCB_MAP_STREAM") == "1" else None)
        from .execution import InflightLimiter
        self.inflight = InflightLimiter(2)

    def forward(self, t, options=None):
        from dataclasses import replace
        from .execution import (ExecOptions, LayerSpec, prepare_layer_maps,
                                prepare_maps_on_stream, sparse_conv_forward)
        opts = replace(options) if options is not None else ExecOptions()
        self.inflight.before_forward()
        if opts.map_reuse:  # the coordinate pyramid before any convolution is queued

            def build(cs):
                levels = [cs]
                prepare_layer_maps(cs, LayerSpec(3, 1, 1, 1), opts)
                for l in self.table:
                    if l["s"] == 2:
                        cs = prepare_layer_maps(cs, LayerSpec(3, 2, l["ci"], l["co"]), opts)
                        prepare_layer_maps(cs, LayerSpec(3, 1, 1, 1), opts)
                        levels.append(cs)
                return levels

            prepare_maps_on_stream(t, self.mapping_stream, build, opts.timer)
        x = t
        for l in self.table:
            opts.layer_label = l["name"]
            sc, sh = self.bn[l["name"]]
            x = sparse_conv_forward(x, self.w[l["name"]], LayerSpec(3, l["s"], l["ci"], l["co"]),
                                    None, None, opts,
                                    epilogue={"scale": sc, "shift": sh, "relu": True})
        self.inflight.after_forward()
        return x


def forward_oracle(params: dict, coords: np.ndarray, feats: np.ndarray, boundary,
                   batch_size: int = 1, in_channels: int = 5):
    """The same graph on the CPU oracle (tests only): conv output in f32, BN
    + ReLU in f32, one cast to the storage dtype per layer."""
    from oracle import sparseconv_oracle as O
    storage = feats.dtype
    c, f, b = np.asarray(coords, np.int64), feats, tuple(boundary)
    for l in layer_table(in_channels):
        p = params[l["name"]]
        c, of, b = O.conv_forward(c, f, b, p["w"], 3, l["s"], batch_size)
        f = np.maximum(of.astype(np.float32) * p["scale"] + p["shift"], 0).astype(storage)
    return c, f, b
