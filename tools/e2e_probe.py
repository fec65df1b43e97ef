"""Attribute the end-to-end (host buffers) step time vs the device-resident
step: the bench's e2e loop with each host-facing piece toggled.
    python tools/e2e_probe.py"""
import collections
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402


def run(model, coords, feats, boundary, B, h2d=True, d2h=True, validate="async", steps=20,
        pad_d2h=False):
    dev = torch.device("cuda")
    h_c = torch.from_numpy(coords.astype(np.int32)).pin_memory()
    h_f = torch.from_numpy(feats).pin_memory()
    d_c, d_f = h_c.to(dev), h_f.to(dev)
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    NB = 4
    c_ring = [torch.empty_like(d_c) for _ in range(NB)]
    f_ring = [torch.empty_like(d_f) for _ in range(NB)]
    done = [None] * NB
    pending = collections.deque()
    h_out = None
    cnt = [0]

    def step():
        nonlocal h_out
        k = cnt[0] % NB
        cnt[0] += 1
        cur = torch.cuda.current_stream()
        if h2d:
            with torch.cuda.stream(h2d_s):
                if done[k] is not None:
                    h2d_s.wait_event(done[k])
                c_ring[k].copy_(h_c, non_blocking=True)
                f_ring[k].copy_(h_f, non_blocking=True)
            cur.wait_stream(h2d_s)
            c, f = c_ring[k], f_ring[k]
        else:
            c, f = d_c, d_f
        t = sc.SparseTensor(c, f, 1, boundary, B, validate=validate)
        t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        o = model.forward(t, sc.ExecOptions(index_kind="hash", dataflow="auto"))
        done[k] = cur.record_event()
        if d2h:
            src = o.features
            if pad_d2h:
                src = src.as_strided((src.shape[0], src.stride(0)), (src.stride(0), 1))
            if h_out is None:
                h_out = torch.empty(tuple(src.shape), dtype=src.dtype).pin_memory()
            d2h_s.wait_event(done[k])
            with torch.cuda.stream(d2h_s):
                h_out.copy_(src, non_blocking=True)
                pending.append((o, d2h_s.record_event()))
            while len(pending) > 3:
                pending.popleft()[1].synchronize()

    for _ in range(30):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.current_stream().wait_stream(d2h_s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, 1e3 * (time.perf_counter() - h0) / steps


def main():
    scans = load_scans(range(8))
    coords, feats, boundary = pack(scans)
    model = EngineMinkUNet(1.0, 4, 0)
    for name, kw in [("full e2e", {}), ("no D2H", dict(d2h=False)), ("no H2D", dict(h2d=False)),
                     ("no H2D no D2H", dict(h2d=False, d2h=False)),
                     ("no validation", dict(validate=False)),
                     ("device-resident", dict(h2d=False, d2h=False, validate=False)),
                     ("padded-row D2H", dict(pad_d2h=True)), ("full e2e again", {})]:
        ms, host = run(model, coords, feats, boundary, 8, **kw)
        print(f"{name:18s} {ms:7.3f} ms/step  host {host:6.3f} ms/step  {8e3 / ms:7.1f} scans/s",
              flush=True)


if __name__ == "__main__":
    main()
