"""MinkUNet (the benchmark model of the paper) expressed on
the drop-in operator API.

Layer table (public TorchSparse/MinkowskiEngine definition):
cs = [32, 32, 64, 128, 256, 256, 128, 96, 96] x width.

    stem      conv3 in->cs0 +BN+ReLU, conv3 cs0->cs0 +BN+ReLU
    stage i   conv2/s2 (c->c) +BN+ReLU, Res(c->cs_i), Res(cs_i->cs_i)      i=1..4
    up j      deconv2 (transposed, map of stage 5-j's down conv) +BN+ReLU,
              concat skip, Res(cs+skip->cs), Res(cs->cs)                    j=1..4
    head      conv1 (linear) cs8 -> 19 classes
    Res(a->b) relu(BN(conv3(relu(BN(conv3 x)))) + proj(x)), proj = conv1+BN if a != b

50 convolution layers (34 k3 s1, 4 k2 s2, 4 transposed k2, 8 k1).  BatchNorm
is folded (eval mode) into the scatter epilogue; residual add and concat are
model glue (not reference layer kinds).

``EngineMinkUNet`` runs on the B200 engine; the same graph on the CPU
oracle (test infrastructure) is ``oracle.models.minkunet_oracle``.
"""

from __future__ import annotations

import numpy as np

N_CLASSES = 19
BASE_CS = (32, 32, 64, 128, 256, 256, 128, 96, 96)


def channels(width: float) -> list[int]:
    return [int(c * width) for c in BASE_CS]


def layer_table(width: float, in_channels: int = 4) -> list[dict]:
    """Flat list of conv layers with their (K, stride, c_in, c_out)."""
    cs = channels(width)
    L = []

    def conv(name, k, s, ci, co, kind="conv", reuse=None):
        L.append(dict(name=name, k=k, s=s, ci=ci, co=co, kind=kind, reuse=reuse))

    def res(prefix, ci, co):
        conv(prefix + ".c1", 3, 1, ci, co)
        conv(prefix + ".c2", 3, 1, co, co)
        if ci != co:
            conv(prefix + ".proj", 1, 1, ci, co)

    conv("stem.0", 3, 1, in_channels, cs[0])
    conv("stem.1", 3, 1, cs[0], cs[0])
    for i in range(1, 5):
        conv(f"down{i}", 2, 2, cs[i - 1], cs[i - 1])
        res(f"enc{i}.r0", cs[i - 1], cs[i])
        res(f"enc{i}.r1", cs[i], cs[i])
    skip = {1: cs[3], 2: cs[2], 3: cs[1], 4: cs[0]}
    prev = cs[4]
    for j in range(1, 5):
        c = cs[4 + j]
        conv(f"up{j}", 2, 1, prev, c, kind="inverse", reuse=f"down{5 - j}")
        res(f"dec{j}.r0", c + skip[j], c)
        res(f"dec{j}.r1", c, c)
        prev = c
    conv("head", 1, 1, prev, N_CLASSES)
    return L


def build_params(width: float, in_channels: int = 4, seed: int = 0) -> dict:
    """Random-init weights (N(0, 1/sqrt(K^3 C_in)), as reference
    network.py:183-193) and folded BN (scale U(0.8,1.2), shift N(0,0.05))."""
    rng = np.random.default_rng(seed)
    params = {}
    for l in layer_table(width, in_channels):
        vol = l["k"] ** 3
        w = rng.normal(0.0, 1.0 / np.sqrt(vol * l["ci"]), size=(vol, l["ci"], l["co"]))
        p = {"w": w.astype(np.float32)}
        if l["name"] != "head":
            p["scale"] = rng.uniform(0.8, 1.2, size=l["co"]).astype(np.float32)
            p["shift"] = rng.normal(0.0, 0.05, size=l["co"]).astype(np.float32)
        params[l["name"]] = p
    return params


# ---------------------------------------------------------------- engine

class EngineMinkUNet:
    """MinkUNet on the B200 engine.  Parameters are uploaded once.

    Coordinate levels are relabelled by neighbour presence
    (mapping.reorder_by_presence; ``reorder=False`` or SCB_REORDER=0 keeps
    the reference's flat-key row order): every layer then runs over rows
    whose 128-row tiles share their active kernel offsets, and the fused
    kernel skips the absent (tile, offset) blocks.  The input features are
    permuted once, the logits un-permuted once, so the output rows are in
    the input tensor's order — the same result either way."""

    def __init__(self, width: float, in_channels: int = 4, seed: int = 0,
                 reorder: bool | None = None):
        import os
        import torch
        from .core import WeightTensor
        self.width = width
        self.table = layer_table(width, in_channels)
        self.params = build_params(width, in_channels, seed)
        self.w = {}
        self.bn = {}
        for l in self.table:
            p = self.params[l["name"]]
            self.w[l["name"]] = WeightTensor(p["w"], l["k"], 3)
            if "scale" in p:
                self.bn[l["name"]] = (torch.from_numpy(p["scale"]).cuda(),
                                      torch.from_numpy(p["shift"]).cuda())
        # materialise device weights now (not inside a timed step)
        for name, w in self.w.items():
            w.packed_f16()
        self.reorder = (os.environ.get("SCB_REORDER", "1") == "1") if reorder is None else reorder
        from .execution import InflightLimiter
        self.inflight = InflightLimiter(int(os.environ.get("SCB_INFLIGHT", "3")))
        self._pending = {}   # id(coordset) -> (coordset, level-0 set, deferred chain)
        self._specs = {}

    def _down_specs(self):
        from .execution import LayerSpec
        return [LayerSpec(2, 2, self.w[f"down{i}"].c_in, self.w[f"down{i}"].c_out)
                for i in range(1, 5)]

    def _start(self, cset, opts):
        """Queue the level-0 set (reordered), its k3 map and the strided
        coordinate chain; returns (level-0 set, finisher).  The finisher
        collects the chain's one host read and builds the other levels."""
        from .execution import LayerSpec, link_strided_map, prepare_layer_maps, _timed
        from .mapping import enumerate_offsets, reorder_by_presence, start_output_coords_chain
        k3 = LayerSpec(3, 1, 1, 1)
        kind = opts.index_kind or "auto"
        timer = opts.timer
        with _timed(timer, "L0", "mapping"):
            l0 = reorder_by_presence(cset, 3, kind) if self.reorder else cset
            prepare_layer_maps(l0, k3, opts)
        specs = self._down_specs()
        dim = len(cset.boundary)
        with _timed(timer, "chain", "mapping"):
            chain = start_output_coords_chain(cset, [(enumerate_offsets(dim, sp.kernel_size),
                                                      sp.stride) for sp in specs])

        def finish():
            from .core import CoordinateSet
            fine = l0
            for i, (sp, (oc, ob)) in enumerate(zip(specs, chain()), 1):
                with _timed(timer, f"L{i}", "mapping"):
                    lvl = CoordinateSet(oc, ob, cset.batch_size)
                    if self.reorder:
                        lvl = reorder_by_presence(lvl, 3, kind)
                    link_strided_map(fine, lvl, sp, opts)
                    prepare_layer_maps(lvl, k3, opts)
                fine = lvl
        return l0, finish

    def prefetch(self, t, options=None) -> None:
        """Queue ``t``'s level-0 map and its strided coordinate chain now
        (B200 extension).  A serving loop calls this for batch i+1 before it
        runs batch i: the chain's one host read, collected in forward(batch
        i+1), then finds its kernels long finished instead of draining the
        compute queue each forward.  Same maps, same results.  At most one
        batch is held (a newer prefetch replaces an unused older one)."""
        from dataclasses import replace
        from .execution import ExecOptions
        opts = replace(options) if options is not None else ExecOptions()
        if not opts.map_reuse:
            return
        opts.timer = None
        key = id(t.coordset)
        if key in self._pending:
            return
        l0, finish = self._start(t.coordset, opts)
        self._pending = {key: (t.coordset, l0, finish)}

    def forward(self, t, options=None):
        from .core import SparseTensor
        from .execution import (ExecOptions, LayerSpec, inverse_conv_forward, _timed,
                                sparse_conv_forward)
        from .mapping import permute_rows
        from dataclasses import replace
        base = replace(options) if options is not None else ExecOptions()  # private copy
        cache = {}

        specs = self._specs

        def conv(x, name, k, s, relu=True, reuse=None, kind="conv", residual=None, concat=None):
            w = self.w[name]
            opts = base
            opts.layer_label = name
            ep = {"relu": relu, "residual": residual}
            if name in self.bn:
                ep["scale"], ep["shift"] = self.bn[name]
            spec = specs.get(name)
            if spec is None:  # static per layer: built once
                if kind == "inverse":
                    spec = LayerSpec(k, 1, w.c_in, w.c_out, transposed=True, reuse_key=reuse)
                else:  # only strided maps are replayed (by the transposed layers)
                    spec = LayerSpec(k, s, w.c_in, w.c_out, reuse_key=name if s > 1 else None)
                specs[name] = spec
            if kind == "inverse":
                return inverse_conv_forward(x, w, spec, cache, None, opts, epilogue=ep)
            return sparse_conv_forward(x, w, spec, None, cache, opts, epilogue=ep, concat=concat)

        def res(x, prefix, has_proj, skip=None):
            # relu(BN(conv2(h)) + shortcut): the residual add and ReLU run in
            # conv2's epilogue (one write of the block output).  ``skip``: the
            # decoder's concatenated skip input, read in place by c1 and proj
            h = conv(x, prefix + ".c1", 3, 1, concat=skip)
            sc = conv(x, prefix + ".proj", 1, 1, relu=False, concat=skip) if has_proj else x
            return conv(h, prefix + ".c2", 3, 1, relu=True, residual=sc)

        names = {l["name"] for l in self.table}
        self.inflight.before_forward()
        finish, l0 = None, t.coordset
        if base.map_reuse:
            # level-0 set and map plus the k2/s2 coordinate chain are queued
            # first (or were, by prefetch()); the chain's count read is
            # collected after the level-0 stems are queued
            hit = self._pending.pop(id(t.coordset), None)
            if hit is not None and hit[0] is t.coordset:
                _, l0, finish = hit
            else:
                l0, finish = self._start(t.coordset, base)
        x = t
        if l0 is not t.coordset:  # relabelled level 0: permute the input rows once
            with _timed(base.timer, "input", "permute"):
                x = SparseTensor._wrap(permute_rows(t.features, l0.perm), t.stride, t.boundary,
                                       t.batch_size, l0)
        x = conv(x, "stem.0", 3, 1)
        x = conv(x, "stem.1", 3, 1)
        if finish is not None:  # both level-0 stems are queued: the GPU stays busy meanwhile
            finish()
        skips = [x]
        for i in range(1, 5):
            x = conv(x, f"down{i}", 2, 2)
            x = res(x, f"enc{i}.r0", f"enc{i}.r0.proj" in names)
            x = res(x, f"enc{i}.r1", f"enc{i}.r1.proj" in names)
            skips.append(x)
        for j in range(1, 5):
            x = conv(x, f"up{j}", 2, 1, reuse=f"down{5 - j}", kind="inverse")
            x = res(x, f"dec{j}.r0", True, skip=skips[4 - j])
            x = res(x, f"dec{j}.r1", f"dec{j}.r1.proj" in names)
        out = conv(x, "head", 1, 1, relu=False)  # logits: no BN, no ReLU
        if l0 is not t.coordset:  # logits back to the input's row order
            with _timed(base.timer, "output", "permute"):
                f = out.features
                rows = f.as_strided((f.shape[0], f.stride(0)), (f.stride(0), 1))
                back = permute_rows(rows, l0.perm, scatter=True)[:, : f.shape[1]]
            out = SparseTensor._wrap(back, out.stride, out.boundary, out.batch_size, t.coordset)
        self.inflight.after_forward()
        return out
