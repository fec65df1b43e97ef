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
                 reorder: bool | None = None, strategy=None):
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
        # a side stream for the coordinate levels' maps (SCB_MAP_STREAM=0: inline)
        prio = int(os.environ.get("SCB_MAP_PRIORITY", "-1"))
        # a prefetched batch's mapping starts when the previous batch enters
        # this level (the deeper levels leave SMs idle); measured best at 2
        # before the dense up / K = 1 forms, at 3 after them (1345-1348 vs
        # 1338-1340 scans/s, three same-box pairs)
        self.prefetch_level = int(os.environ.get("SCB_PREFETCH_LEVEL", "3"))
        self.map_stream = (torch.cuda.Stream(priority=prio)
                           if os.environ.get("SCB_MAP_STREAM", "1") == "1" else None)
        self.chain_stream = torch.cuda.Stream(priority=prio) if self.map_stream else None
        from .execution import InflightLimiter
        self.inflight = InflightLimiter(int(os.environ.get("SCB_INFLIGHT", "3")))
        self._pending = {}   # id(coordset) -> (coordset, level-0 set, deferred chain)
        self._specs = {}
        self._tune = None    # set by tune_kernel_shapes for one forward
        import collections
        self._retained = collections.deque()   # (end event, map objects) per forward
        # per-layer fused-kernel launch shapes from a JSON v1 strategy file
        # (autotune.save_strategy; the "kernel" extension of the records)
        self.kernel_shapes = {}
        if strategy is not None:
            from .autotune import StrategyFile, load_strategy
            sf = strategy if isinstance(strategy, StrategyFile) else load_strategy(strategy)
            self.kernel_shapes = {r.layer_id: (r.ctas, r.stage_kb) for r in sf.layers
                                  if r.ctas or r.stage_kb}

    def tune_kernel_shapes(self, t, options=None, shapes=None, repeats: int = 7,
                           rel_tol: float = 0.02):
        """Time every fused layer of one forward over ``t`` under each launch
        shape (autotune.KERNEL_SHAPES: CTAs per SM, stage KB, single-CTA or
        CTA-pair kernel) with CUDA events, keep a shape only when it beats the
        default by ``rel_tol``, and return the JSON v1 StrategyFile (the
        B200 counterpart of the reference's per-layer tune_layer records,
        autotune.py:147-218).  The tuned shapes also become this model's."""
        from .autotune import KERNEL_SHAPES, LayerRecord, StrategyFile
        self._tune = {"shapes": tuple(shapes or KERNEL_SHAPES), "repeats": repeats,
                      "rel_tol": rel_tol, "best": {}}
        saved = dict(self.kernel_shapes)
        self.kernel_shapes = {}
        try:
            self.forward(t, options)
        finally:
            best = self._tune["best"]
            self._tune = None
        self.kernel_shapes = {k: v for k, v in best.items() if v != (0, 0)} or saved
        recs = tuple(LayerRecord(l["name"], 0.0, float("inf"), "auto", "auto",
                                 *best.get(l["name"], (0, 0))) for l in self.table)
        return StrategyFile(layers=recs, dataset="semantickitti-shaped raycast scans")

    def _release_retained(self, limit: int = 8) -> None:
        """Drop the map objects of forwards whose end event has completed
        (their blocks may then be reused by the mapping streams)."""
        r = self._retained
        while r and (r[0][0].query() or len(r) > limit):
            r[0][0].synchronize()
            r.popleft()

    def _tuned_call(self, name, call, base):
        """Run ``call(opts)`` for layer ``name``; while tuning, first time it
        under every launch shape and keep the fastest."""
        from dataclasses import replace
        tune = self._tune
        if tune is None:
            return call(base)
        import torch
        timings = []
        for shape in tune["shapes"]:
            o = replace(base, kernel_shapes={name: shape})
            call(o)
            samples = []
            for _ in range(tune["repeats"]):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                # keep the GPU busy while the host queues the layer, so the
                # events bracket device work only (no host-issue gaps)
                torch.cuda._sleep(300_000)
                a.record()
                call(o)
                b.record()
                b.synchronize()
                samples.append(a.elapsed_time(b))
            timings.append((shape, sorted(samples)[len(samples) // 2]))
        default = dict(timings).get((0, 0), timings[0][1])
        best, best_t = (0, 0), default
        for shape, ms in timings:
            if ms < best_t * (1.0 - tune["rel_tol"]):
                best, best_t = shape, ms
        tune["best"][name] = best
        return call(replace(base, kernel_shapes={name: best}))

    def _down_specs(self):
        from .execution import LayerSpec
        return [LayerSpec(2, 2, self.w[f"down{i}"].c_in, self.w[f"down{i}"].c_out)
                for i in range(1, 5)]

    def _start(self, cset, opts):
        """Queue the level-0 set (reordered), its k3 map and the strided
        coordinate chain on the current stream; returns (level-0 set,
        finisher, level-0-ready event).  The finisher collects the chain's one
        host read and builds the other levels."""
        from .execution import LayerSpec, link_strided_map, prepare_layer_maps, _timed
        from .mapping import enumerate_offsets, reorder_by_presence, start_output_coords_chain
        k3 = LayerSpec(3, 1, 1, 1)
        kind = opts.index_kind or "auto"
        timer = opts.timer
        import torch
        l0_start = torch.cuda.Event()
        l0_start.record()
        with _timed(timer, "L0", "mapping"):
            l0 = reorder_by_presence(cset, 3, kind) if self.reorder else cset
            prepare_layer_maps(l0, k3, opts)
        l0_ready = torch.cuda.Event()   # what the level-0 convolutions need
        l0_ready.record()
        specs = self._down_specs()
        dim = len(cset.boundary)
        steps = [(enumerate_offsets(dim, sp.kernel_size), sp.stride) for sp in specs]
        if self.chain_stream is not None:
            # the coordinate pyramid needs the input coordinates only: it runs
            # beside the level-0 maps instead of behind them (the level-1 maps
            # wait for it, and the convolutions wait for those)
            cs_ = self.chain_stream
            cs_.wait_event(l0_start)
            with torch.cuda.stream(cs_), _timed(timer, "chain", "mapping"):
                chain0 = start_output_coords_chain(cset, steps)
            chain_done = torch.cuda.Event()
            chain_done.record(cs_)

            def chain():
                out = chain0()
                torch.cuda.current_stream().wait_event(chain_done)
                return out
        else:
            with _timed(timer, "chain", "mapping"):
                chain = start_output_coords_chain(cset, steps)

        def finish():
            """Build levels 1..4; returns an event per level, recorded on the
            current stream when the level's maps are queued."""
            import torch
            from .core import CoordinateSet
            fine, events = l0, []
            for i, (sp, (oc, ob)) in enumerate(zip(specs, chain()), 1):
                with _timed(timer, f"L{i}", "mapping"):
                    lvl = CoordinateSet(oc, ob, cset.batch_size)
                    if self.reorder:
                        lvl = reorder_by_presence(lvl, 3, kind)
                    link_strided_map(fine, lvl, sp, opts)
                    prepare_layer_maps(lvl, k3, opts)
                ev = torch.cuda.Event()
                ev.record()
                events.append(ev)
                fine = lvl
            return events
        finish.chain_done = chain_done if self.chain_stream is not None else None
        return l0, finish, l0_ready

    def prefetch(self, t, options=None, coords_ready=None) -> None:
        """Queue ``t``'s level-0 maps and its strided coordinate chain now, on
        the mapping streams (B200 extension).  A serving loop calls this for
        batch i+1 before forward(batch i): the mapping then runs beside batch
        i's convolutions, and forward(batch i+1) finds it done.  Same maps,
        same results.  ``coords_ready``: an event after which t's coordinates
        -- and anything already built on them, e.g. the hash index of
        ``validate="async"`` -- are on the device (default: everything queued
        on the current stream).
        Memory the mapping streams allocate is retained per forward until
        that forward's end event has completed, so prefetched mapping never
        reuses a block a queued convolution still reads.  At most one batch
        is held (a newer prefetch replaces an unused older one)."""
        import os
        import torch
        from contextlib import nullcontext
        from dataclasses import replace
        from .execution import ExecOptions
        opts = replace(options) if options is not None else ExecOptions()
        if not opts.map_reuse:
            return
        opts.timer = None
        key = id(t.coordset)
        if key in self._pending:
            return
        ms = self.map_stream
        if ms is not None:
            self._release_retained()
            if coords_ready is not None:
                ms.wait_event(coords_ready)
                deep = getattr(self, "_deep_event", None)
                if deep is not None and os.environ.get("SCB_PREFETCH_DEEP", "1") == "1":
                    ms.wait_event(deep)   # behind the last forward's shallow levels
            else:
                ms.wait_stream(torch.cuda.current_stream())
        with (torch.cuda.stream(ms) if ms is not None else nullcontext()):
            l0, finish, ready = self._start(t.coordset, opts)
        self._pending = {key: (t.coordset, l0, finish, ready)}

    def forward(self, t, options=None):
        from .core import SparseTensor
        from .execution import (ExecOptions, LayerSpec, inverse_conv_forward, _timed,
                                sparse_conv_forward)
        from .mapping import permute_rows
        from dataclasses import replace
        base = replace(options) if options is not None else ExecOptions()  # private copy
        if self.kernel_shapes:
            base.kernel_shapes = {**self.kernel_shapes, **(base.kernel_shapes or {})}
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
                call = lambda o: inverse_conv_forward(x, w, spec, cache, None, o, epilogue=ep)
            else:
                call = lambda o: sparse_conv_forward(x, w, spec, None, cache, o, epilogue=ep,
                                                     concat=concat)
            # the dense forms (K = 1 layers, transposed K = s layers) have no
            # launch-shape knobs: only gather-form layers are tuned
            from . import execution as X
            dense = (k == 1 and X._DENSE_K1) or (kind == "inverse" and X._UPSCATTER)
            return call(opts) if dense else self._tuned_call(name, call, opts)

        def res(x, prefix, has_proj, skip=None):
            # relu(BN(conv2(h)) + shortcut): the residual add and ReLU run in
            # conv2's epilogue (one write of the block output).  ``skip``: the
            # decoder's concatenated skip input, read in place by c1 and proj
            h = conv(x, prefix + ".c1", 3, 1, concat=skip)
            sc = conv(x, prefix + ".proj", 1, 1, relu=False, concat=skip) if has_proj else x
            return conv(h, prefix + ".c2", 3, 1, relu=True, residual=sc)

        import torch
        from contextlib import nullcontext
        names = {l["name"] for l in self.table}
        self.inflight.before_forward()
        finish, l0 = None, t.coordset
        compute = torch.cuda.current_stream()
        ms = self.map_stream if base.map_reuse else None
        on_maps = torch.cuda.stream(ms) if ms is not None else nullcontext()
        if ms is not None:
            self._release_retained()
        if base.map_reuse:
            # level-0 set and map plus the k2/s2 coordinate chain are queued
            # first (or were, by prefetch()); the chain's count read is
            # collected after the level-0 stems are queued
            hit = self._pending.pop(id(t.coordset), None)
            if hit is not None and hit[0] is t.coordset:
                _, l0, finish, l0_ready = hit
            else:
                if ms is not None:
                    # mapping on its own (high-priority) stream: it needs only
                    # the coordinates, and waiting for everything queued so
                    # far also keeps it from reusing blocks the previous
                    # forward still reads
                    ms.wait_stream(compute)
                with on_maps:
                    l0, finish, l0_ready = self._start(t.coordset, base)
            if ms is not None:   # the level-0 maps, not the coordinate chain behind them
                compute.wait_event(l0_ready)
        x = t
        if l0 is not t.coordset:  # relabelled level 0: permute the input rows once
            with _timed(base.timer, "input", "permute"):
                x = SparseTensor._wrap(permute_rows(t.features, l0.perm), t.stride, t.boundary,
                                       t.batch_size, l0)
        level_ready = [None] * 4
        early = (finish is not None and ms is not None
                 and getattr(finish, "chain_done", None) is not None and finish.chain_done.query())
        if early:  # a prefetched pyramid is already counted: queue levels 1-4 now
            with on_maps:
                level_ready = finish()
        x = conv(x, "stem.0", 3, 1)
        x = conv(x, "stem.1", 3, 1)
        if finish is not None and not early:  # both level-0 stems are queued first
            with on_maps:       # levels 1-4 map while the compute stream convolves
                level_ready = finish()
        skips = [x]
        for i in range(1, 5):
            if ms is not None and level_ready[i - 1] is not None:
                compute.wait_event(level_ready[i - 1])
            if i == self.prefetch_level and ms is not None:
                # the deep levels leave SMs idle (few tiles): the next batch's
                # prefetched mapping starts here (prefetch waits on this event)
                self._deep_event = torch.cuda.Event()
                self._deep_event.record()
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
        if ms is not None:
            # keep this forward's map objects (allocated on the mapping
            # streams) alive until its convolutions have run
            self._retained.append((self.inflight.events[-1], (t.coordset, l0)))
        return out
