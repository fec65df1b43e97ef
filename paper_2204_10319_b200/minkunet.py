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

``forward_engine`` runs on the B200 engine; ``forward_oracle`` runs the same
graph on the CPU oracle (tests / CPU baseline only).
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
    """MinkUNet on the B200 engine.  Parameters are uploaded once."""

    def __init__(self, width: float, in_channels: int = 4, seed: int = 0):
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
        # mapping work (coordinate pyramid, hash indexes, kernel maps) runs
        # here, off the compute stream: it depends on coordinates only, so
        # the next batch's maps overlap this batch's convolutions
        # SCB_MAP_STREAM=1: maps on a high-priority side stream (overlaps the
        # previous batch; measured noisier: the persistent conv kernels leave
        # no room for the short mapping kernels between their boundaries)
        self.mapping_stream = (torch.cuda.Stream(priority=-1)
                               if __import__("os").environ.get("SCB_MAP_STREAM") == "1" else None)
        from .execution import InflightLimiter
        self.inflight = InflightLimiter(int(__import__("os").environ.get("SCB_INFLIGHT", "3")))
        import weakref
        self._pending = weakref.WeakKeyDictionary()   # coordset -> deferred chain (prefetch)
        self._specs = {}

    def _down_specs(self):
        from .execution import LayerSpec
        return [LayerSpec(2, 2, self.w[f"down{i}"].c_in, self.w[f"down{i}"].c_out)
                for i in range(1, 5)]

    def prefetch(self, t, options=None) -> None:
        """Queue ``t``'s level-0 map and its strided coordinate chain now
        (B200 extension).  A serving loop calls this for batch i+1 before it
        runs batch i: the chain's one host read, collected in forward(batch
        i+1), then finds its kernels long finished instead of draining the
        compute queue each forward.  Same maps, same results."""
        from dataclasses import replace
        from .execution import ExecOptions, LayerSpec, prepare_layer_maps, prepare_strided_chain
        opts = replace(options) if options is not None else ExecOptions()
        if self.mapping_stream is not None or not opts.map_reuse or t.coordset in self._pending:
            return
        opts.timer = None
        prepare_layer_maps(t.coordset, LayerSpec(3, 1, 1, 1), opts)
        self._pending[t.coordset] = prepare_strided_chain(t.coordset, self._down_specs(), opts,
                                                          deferred=True)

    def _prepare_maps(self, t, opts):
        """The coordinate pyramid (one host read for the four k2 s2 levels)
        and every level's k3 map, on the mapping stream."""
        from .execution import (LayerSpec, prepare_layer_maps, prepare_maps_on_stream,
                                prepare_strided_chain)

        def build(cs):
            levels = [cs] + prepare_strided_chain(cs, self._down_specs(), opts)
            for lvl in levels:
                prepare_layer_maps(lvl, LayerSpec(3, 1, 1, 1), opts)
            return levels

        prepare_maps_on_stream(t, self.mapping_stream, build, opts.timer)

    def forward(self, t, options=None):
        from .execution import (ExecOptions, LayerSpec, inverse_conv_forward,
                                sparse_conv_forward)
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
        finish = None
        if base.map_reuse:
            if self.mapping_stream is not None:
                self._prepare_maps(t, base)
            else:
                # level-0 map and the k2/s2 coordinate chain are queued first
                # (or were, by prefetch()); the chain's count read is collected
                # after the level-0 stems are queued
                finish = self._pending.pop(t.coordset, None)
                if finish is None:
                    from .execution import LayerSpec, prepare_layer_maps, prepare_strided_chain
                    prepare_layer_maps(t.coordset, LayerSpec(3, 1, 1, 1), base)
                    finish = prepare_strided_chain(t.coordset, self._down_specs(), base,
                                                   deferred=True)
        x = conv(t, "stem.0", 3, 1)
        x = conv(x, "stem.1", 3, 1)
        if finish is not None:  # both level-0 stems are queued: the GPU stays busy meanwhile
            from .execution import LayerSpec, prepare_layer_maps
            for lvl in finish():
                prepare_layer_maps(lvl, LayerSpec(3, 1, 1, 1), base)
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
        out = conv(x, "head", 1, 1)
        self.inflight.after_forward()
        return out


# ---------------------------------------------------------------- oracle (CPU)

def forward_oracle(params: dict, width: float, coords: np.ndarray, feats: np.ndarray,
                   boundary, batch_size: int = 1, in_channels: int = 4):
    """The same graph on the CPU oracle (tests and the CPU baseline only).
    Epilogue rounding follows the engine: conv output in f32, BN + ReLU in
    f32, one cast to the storage dtype."""
    from oracle import sparseconv_oracle as O
    storage = feats.dtype
    names = {l["name"] for l in layer_table(width, in_channels)}
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
    return conv(x, "head", 1, 1)
