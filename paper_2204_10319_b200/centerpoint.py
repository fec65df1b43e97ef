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

``EngineCenterPoint`` runs on the B200 engine; the same graph on the CPU
oracle (test infrastructure) is ``oracle.models.centerpoint_oracle``.
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
    """The encoder on the B200 engine.  Parameters are uploaded once.  Every
    level but the output one is relabelled by neighbour presence
    (mapping.reorder_by_presence; ``reorder=False`` / SCB_REORDER=0 keeps the
    flat-key order); the output level is produced in the reference's
    ascending-key order, so the result is the same either way."""

    def __init__(self, in_channels: int = 5, seed: int = 0, reorder: bool | None = None):
        import collections
        import os
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
        self.reorder = (os.environ.get("SCB_REORDER", "1") == "1") if reorder is None else reorder
        from .execution import InflightLimiter
        self.inflight = InflightLimiter(2)
        # the coordinate pyramid on a high-priority side stream (SCB_MAP_STREAM=0: inline)
        self.map_stream = (torch.cuda.Stream(priority=-1)
                           if os.environ.get("SCB_MAP_STREAM", "1") == "1" else None)
        self._pending = {}
        self._retained = collections.deque()   # (end event, map objects) per forward
        self._deep_event = None
        self.prefetch_layer = os.environ.get("SCB_CP_PREFETCH_LAYER", "down2")

    def _pyramid(self, cset, opts):
        """Level-0 set (reordered) and every level's maps, on the current
        stream; returns (level-0 set, ready event).  Strided k3 levels need
        one host read of their output count each."""
        import torch
        from .execution import LayerSpec, prepare_layer_maps, prepare_reordered_level, _timed
        from .mapping import reorder_by_presence
        with _timed(opts.timer, "pyramid", "mapping"):
            cs0 = reorder_by_presence(cset, 3, opts.index_kind or "auto") \
                if self.reorder else cset
            prepare_layer_maps(cs0, LayerSpec(3, 1, 1, 1), opts)
            cs = cs0
            strided = [l for l in self.table if l["s"] == 2]
            for i, l in enumerate(strided):
                last = i == len(strided) - 1
                cs = prepare_reordered_level(cs, LayerSpec(3, 2, l["ci"], l["co"]), opts,
                                             reorder=self.reorder and not last)
                if not last:
                    prepare_layer_maps(cs, LayerSpec(3, 1, 1, 1), opts)
        ev = torch.cuda.Event()
        ev.record()
        return cs0, ev

    def _release_retained(self, limit: int = 8) -> None:
        r = self._retained
        while r and (r[0][0].query() or len(r) > limit):
            r[0][0].synchronize()
            r.popleft()

    def prefetch(self, t, options=None, coords_ready=None) -> None:
        """Build ``t``'s coordinate pyramid now, on the mapping stream (B200
        extension, as EngineMinkUNet.prefetch): a serving loop calls it for
        batch i+1 after forward(batch i), so the pyramid's kernels and host
        reads overlap batch i's convolutions.  ``coords_ready``: an event
        after which t's coordinates (and anything built on them) are on the
        device; default: everything queued on the current stream."""
        import torch
        from dataclasses import replace
        from .execution import ExecOptions
        opts = replace(options) if options is not None else ExecOptions()
        ms = self.map_stream
        if not opts.map_reuse or ms is None:
            return
        opts.timer = None
        key = id(t.coordset)
        if key in self._pending:
            return
        self._release_retained()
        if coords_ready is not None:
            ms.wait_event(coords_ready)
            if self._deep_event is not None:
                ms.wait_event(self._deep_event)
        else:
            ms.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(ms):
            cs0, ev = self._pyramid(t.coordset, opts)
        self._pending = {key: (t.coordset, cs0, ev)}

    def forward(self, t, options=None):
        import torch
        from dataclasses import replace
        from .core import SparseTensor
        from .execution import ExecOptions, LayerSpec, sparse_conv_forward
        from .mapping import permute_rows
        opts = replace(options) if options is not None else ExecOptions()
        self.inflight.before_forward()
        compute = torch.cuda.current_stream()
        ms = self.map_stream if opts.map_reuse else None
        x, cs0 = t, None
        if opts.map_reuse:  # the coordinate pyramid before any convolution is queued
            hit = self._pending.pop(id(t.coordset), None)
            if hit is not None and hit[0] is t.coordset:
                _, cs0, ev = hit
            elif ms is not None:
                self._release_retained()
                ms.wait_stream(compute)
                with torch.cuda.stream(ms):
                    cs0, ev = self._pyramid(t.coordset, opts)
            else:
                cs0, ev = self._pyramid(t.coordset, opts)
            if ms is not None:
                compute.wait_event(ev)
            if cs0 is not t.coordset:
                x = SparseTensor._wrap(permute_rows(t.features, cs0.perm), t.stride,
                                       t.boundary, t.batch_size, cs0)
        for l in self.table:
            opts.layer_label = l["name"]
            if l["name"] == self.prefetch_layer and ms is not None:
                # a prefetched batch's pyramid starts when this forward reaches
                # its deeper, narrower levels (prefetch waits on this event)
                self._deep_event = torch.cuda.Event()
                self._deep_event.record()
            sc, sh = self.bn[l["name"]]
            x = sparse_conv_forward(x, self.w[l["name"]], LayerSpec(3, l["s"], l["ci"], l["co"]),
                                    None, None, opts,
                                    epilogue={"scale": sc, "shift": sh, "relu": True})
        self.inflight.after_forward()
        if ms is not None and cs0 is not None:
            self._retained.append((self.inflight.events[-1], (t.coordset, cs0)))
        return x
